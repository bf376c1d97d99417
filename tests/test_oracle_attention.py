"""Pins for the fp64 attention oracle (oracle/attn_oracle.c) -- CPU only.

Each test pins the oracle to something other than itself: finite
differences, an independent library routine (torch float64 SDPA autograd),
closed-form special cases and invariants that follow from Algorithm 1
 and the readings AMB-1..3 of SURVEY.md §8(c).
"""
import numpy as np
import pytest
import torch

import oracle


def _rand(shape, seed, gain=1.0):
    rng = np.random.default_rng(seed)
    return rng.standard_normal(shape) * gain


def _loss(q, k, v, dout, causal):
    o, _ = oracle.attn_fwd(q, k, v, causal)
    return float(np.sum(dout * o))


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("shape", [(1, 5, 1, 3), (2, 7, 2, 4), (1, 8, 1, 5)])
def test_bwd_matches_central_finite_differences(causal, shape):
    """dQ/dK/dV = gradient of sum(dO * O) (the backward pass's definition, §2.1)."""
    q, k, v, dout = (_rand(shape, s) for s in range(4))
    g = oracle.attn_bwd(q, k, v, dout, causal)
    h = 1e-6
    for name, x in (("dq", q), ("dk", k), ("dv", v)):
        num = np.zeros_like(x)
        it = np.nditer(x, flags=["multi_index"])
        for _ in it:
            idx = it.multi_index
            xp, xm = x.copy(), x.copy()
            xp[idx] += h
            xm[idx] -= h
            args_p = [xp if a is x else a for a in (q, k, v)]
            args_m = [xm if a is x else a for a in (q, k, v)]
            num[idx] = (_loss(*args_p, dout, causal) - _loss(*args_m, dout, causal)) / (2 * h)
        err = np.max(np.abs(num - g[name]))
        assert err < 1e-7, (name, err)


@pytest.mark.parametrize("causal", [False, True])
def test_fwd_bwd_match_torch_sdpa_float64_autograd(causal):
    """Cross-check against torch's float64 math SDPA (independent library code)."""
    B, N, H, d = 2, 37, 3, 16
    q, k, v, dout = (_rand((B, N, H, d), 10 + s) for s in range(4))
    tq, tk, tv = (torch.tensor(a.transpose(0, 2, 1, 3), requires_grad=True) for a in (q, k, v))
    to = torch.nn.functional.scaled_dot_product_attention(tq, tk, tv, is_causal=causal)
    to.backward(torch.tensor(dout.transpose(0, 2, 1, 3)))
    o, lse = oracle.attn_fwd(q, k, v, causal)
    g = oracle.attn_bwd(q, k, v, dout, causal)
    np.testing.assert_allclose(o, to.detach().numpy().transpose(0, 2, 1, 3), rtol=0, atol=1e-12)
    np.testing.assert_allclose(g["o"], o, rtol=0, atol=1e-13)
    np.testing.assert_allclose(g["lse"], lse, rtol=0, atol=1e-13)
    for name, t in (("dq", tq), ("dk", tk), ("dv", tv)):
        np.testing.assert_allclose(g[name], t.grad.numpy().transpose(0, 2, 1, 3), rtol=0, atol=1e-11)
    # L is the natural-log logsumexp of the scaled, masked scores (AMB-15).
    s = np.einsum("bnhd,bmhd->bhnm", q, k) / np.sqrt(d)
    if causal:
        s = np.where(np.tril(np.ones((N, N), bool)), s, -np.inf)
    ref = torch.logsumexp(torch.tensor(s), dim=-1).numpy()
    np.testing.assert_allclose(lse, ref, rtol=0, atol=1e-12)


@pytest.mark.parametrize("causal", [False, True])
def test_invariants(causal):
    """rowsum(dS) = 0 per row implies sum_c dK_c = 0, sum_c dV_c = sum_r dO_r,
    <Q,dQ>_F = <K,dK>_F per head; causal row 0 has dQ_0 = 0 (north_star)."""
    B, N, H, d = 2, 33, 2, 8
    q, k, v, dout = (_rand((B, N, H, d), 20 + s, gain=2.0 if s < 2 else 1.0) for s in range(4))
    g = oracle.attn_bwd(q, k, v, dout, causal)
    np.testing.assert_allclose(g["dk"].sum(axis=1), 0.0, atol=1e-12)
    np.testing.assert_allclose(g["dv"].sum(axis=1), dout.sum(axis=1), atol=1e-12)
    qdq = np.einsum("bnhd,bnhd->bh", q, g["dq"])
    kdk = np.einsum("bnhd,bnhd->bh", k, g["dk"])
    np.testing.assert_allclose(qdq, kdk, atol=1e-11)
    if causal:
        np.testing.assert_allclose(g["dq"][:, 0], 0.0, atol=1e-14)
        # the last key sees only the last query: dV_{N-1} = P_{N-1,N-1} dO_{N-1}
        p_last = np.exp(np.einsum("bhd,bhd->bh", q[:, -1], k[:, -1]) / np.sqrt(d)
                        - g["lse"][:, :, -1])
        np.testing.assert_allclose(g["dv"][:, -1], p_last[..., None] * dout[:, -1], atol=1e-13)


def test_special_cases():
    d = 6
    # N = 1: O = v, L = scale * q.k, all gradients but dV vanish, dV = dO.
    q, k, v, dout = (_rand((1, 1, 1, d), 30 + s) for s in range(4))
    o, lse = oracle.attn_fwd(q, k, v, False)
    np.testing.assert_allclose(o, v, atol=1e-15)
    np.testing.assert_allclose(lse[0, 0, 0], float(q.ravel() @ k.ravel()) / np.sqrt(d), atol=1e-14)
    g = oracle.attn_bwd(q, k, v, dout, False)
    np.testing.assert_allclose(g["dq"], 0.0, atol=1e-15)
    np.testing.assert_allclose(g["dk"], 0.0, atol=1e-15)
    np.testing.assert_allclose(g["dv"], dout, atol=1e-15)
    # causal row 0: O_0 = v_0
    q, k, v = (_rand((1, 9, 2, d), 40 + s) for s in range(3))
    o, _ = oracle.attn_fwd(q, k, v, True)
    np.testing.assert_allclose(o[:, 0], v[:, 0], atol=1e-15)
    # all keys equal: uniform P, O_r = mean_c v_c (full) / mean_{c<=r} v_c (causal)
    k = np.broadcast_to(_rand((1, 1, 2, d), 50), (1, 9, 2, d)).copy()
    o, lse = oracle.attn_fwd(q, k, v, False)
    np.testing.assert_allclose(o, np.broadcast_to(v.mean(axis=1, keepdims=True), o.shape), atol=1e-14)
    o, _ = oracle.attn_fwd(q, k, v, True)
    cm = np.cumsum(v, axis=1) / np.arange(1, 10)[None, :, None, None]
    np.testing.assert_allclose(o, cm, atol=1e-14)


@pytest.mark.parametrize("causal", [False, True])
def test_sampled_rows_match_full_backward(causal):
    """The row-sampled entry points (used at full bench size) equal the full pass."""
    B, N, H, d = 2, 40, 3, 8
    q, k, v, dout = (_rand((B, N, H, d), 60 + s) for s in range(4))
    g = oracle.attn_bwd(q, k, v, dout, causal)
    heads = [0, 4, 5]
    rows = [0, 1, 17, 39]
    dq = oracle.attn_bwd_dq_rows(q, k, v, dout, causal, heads, rows)
    dk, dv = oracle.attn_bwd_kv_rows(q, k, v, dout, causal, heads, rows)
    for a, hb in enumerate(heads):
        b, h = divmod(hb, H)
        for z, r in enumerate(rows):
            np.testing.assert_allclose(dq[a, z], g["dq"][b, r, h], atol=1e-13)
            np.testing.assert_allclose(dk[a, z], g["dk"][b, r, h], atol=1e-13)
            np.testing.assert_allclose(dv[a, z], g["dv"][b, r, h], atol=1e-13)


def test_thread_count_does_not_change_bits():
    q, k, v, dout = (_rand((2, 24, 3, 8), 70 + s) for s in range(4))
    n0 = oracle.max_threads()
    oracle.set_threads(1)
    a = oracle.attn_bwd(q, k, v, dout, True)
    oracle.set_threads(4)
    b = oracle.attn_bwd(q, k, v, dout, True)
    oracle.set_threads(n0)
    for name in ("dq", "dk", "dv"):
        assert np.array_equal(a[name], b[name])


def test_fp32_non_associativity_example():
    """§1: (1e8 + 1e-6) - 1e8 = 0 in fp32, while 1e8 - 1e8 + 1e-6 = 1e-6."""
    a, b = np.float32(1e8), np.float32(1e-6)
    assert (a + b) - a == np.float32(0.0)
    assert (a - a) + b == b
