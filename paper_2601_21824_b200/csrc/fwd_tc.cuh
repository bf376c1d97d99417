// Attention forward on the tensor cores: O and the
// natural-log logsumexp L, the inputs Algorithm 1 requires.
//
// One CTA per (128-row Q tile, (b, h)); 256 threads:
//   warp 0      TMA producer: Q once, then K (pass 1) and K, V (pass 2)
//               through 2-stage rings
//   warp 1      MMA issuer + TMEM owner: S = Q K^T (SS, M = 128 Q rows,
//               N = 128 keys), O += P V (TS: P from TMEM)
//   warps 4-7   softmax: thread = one Q row = one TMEM lane, so row max and
//               row sum need no cross-thread reduction
// Two passes over the keys (no O rescaling): pass 1 computes m and l of every
// row from S; pass 2 recomputes S, writes P = exp(S*scale - L) (already
// normalised) as packed bf16 into TMEM and accumulates O = P V.  Costs one
// extra Q K^T GEMM (1.5x the forward's FLOPs) and keeps every step exact in
// the order it is written.  Causal: key tiles after the diagonal are skipped,
// the diagonal tile masked (key c visible to query r iff c <= r, AMB-11).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "umma.cuh"

namespace dash {

struct FwdArgs {
  __nv_bfloat16* o;  // [B,N,H,d]
  float* lse;        // [B,H,N] natural log
  int B, N, H;
  float scale_log2;  // softmax scale * log2(e)
  int causal;
};

template <int D>
struct FwdCfg {
  static constexpr int BM = 128, BN = 128;  // Q rows, keys per tile
  static constexpr uint32_t TILE_BYTES = 128 * D * 2;
  static constexpr uint32_t OFF_Q = 0;
  static constexpr uint32_t OFF_K = OFF_Q + TILE_BYTES;       // 2 stages
  static constexpr uint32_t OFF_V = OFF_K + 2 * TILE_BYTES;   // 2 stages
  static constexpr uint32_t OFF_BAR = OFF_V + 2 * TILE_BYTES;
  static constexpr int NBAR = 16;
  static constexpr uint32_t OFF_MISC = OFF_BAR + NBAR * 8;
  static constexpr uint32_t SMEM_BYTES = OFF_MISC + 16 + 1024;  // + realignment slack
  // TMEM columns: S double-buffered (0, 384), P packed bf16 (128), O (256)
  static constexpr uint32_t T_S0 = 0, T_S1 = 384, T_P = 128, T_O = 256;
  static_assert(SMEM_BYTES <= 232448, "smem budget");
};

enum : int {
  F_Q_FULL = 0, F_K_FULL0 = 1, F_K_EMPTY0 = 3, F_V_FULL0 = 5, F_V_EMPTY0 = 7,
  F_S_FULL0 = 9, F_S_EMPTY0 = 11, F_P_FULL = 13, F_P_EMPTY = 14, F_O_FULL = 15, F_COUNT = 16
};
__device__ __forceinline__ float fwd_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int D>
__global__ void __launch_bounds__(256, 1)
    dash_fwd_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                       const __grid_constant__ CUtensorMap tm_v, const FwdArgs args) {
  using C = FwdCfg<D>;
  extern __shared__ __align__(1024) uint8_t fsmem_raw[];
  const uint32_t pad = (1024 - (ptx::smem_u32(fsmem_raw) & 1023)) & 1023;
  uint8_t* smem = fsmem_raw + pad;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::OFF_MISC);

  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int qt = blockIdx.x, bh = blockIdx.y, b = bh / args.H, h = bh % args.H;
  const int n_kv = args.causal ? qt + 1 : args.N / C::BN;  // key tiles visited

  if (tid == 0) {
    for (int i = 0; i < F_COUNT; ++i) ptx::mbar_init(&bars[i], 1);
    ptx::mbar_init(&bars[F_S_EMPTY0], 128);
    ptx::mbar_init(&bars[F_S_EMPTY0 + 1], 128);
    ptx::mbar_init(&bars[F_P_FULL], 128);
    ptx::fence_mbar_init();
    ptx::fence_async_smem();
  }
  if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    ptx::mbar_arrive_expect_tx_e(&bars[F_Q_FULL], C::TILE_BYTES);
#pragma unroll
    for (int blk = 0; blk < D / 64; ++blk)
      ptx::tma_load_2d_e(smem + C::OFF_Q + blk * 128 * 128, &tm_q, &bars[F_Q_FULL], h * D + blk * 64,
                         b * args.N + qt * C::BM);
    uint32_t kc = 0, vc = 0;
    for (int pass = 0; pass < 2; ++pass) {
      for (int j = 0; j < n_kv; ++j, ++kc) {
        const uint32_t st = kc & 1;
        if (kc >= 2) ptx::mbar_wait_u(&bars[F_K_EMPTY0 + st], ((kc >> 1) - 1) & 1);
        ptx::mbar_arrive_expect_tx_e(&bars[F_K_FULL0 + st], C::TILE_BYTES);
#pragma unroll
        for (int blk = 0; blk < D / 64; ++blk)
          ptx::tma_load_2d_e(smem + C::OFF_K + st * C::TILE_BYTES + blk * 128 * 128, &tm_k,
                             &bars[F_K_FULL0 + st], h * D + blk * 64, b * args.N + j * C::BN);
        if (pass == 1) {
          const uint32_t vs = vc & 1;
          if (vc >= 2) ptx::mbar_wait_u(&bars[F_V_EMPTY0 + vs], ((vc >> 1) - 1) & 1);
          ptx::mbar_arrive_expect_tx_e(&bars[F_V_FULL0 + vs], C::TILE_BYTES);
#pragma unroll
          for (int blk = 0; blk < D / 64; ++blk)
            ptx::tma_load_2d_e(smem + C::OFF_V + vs * C::TILE_BYTES + blk * 128 * 128, &tm_v,
                               &bars[F_V_FULL0 + vs], h * D + blk * 64, b * args.N + j * C::BN);
          ++vc;
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    const uint32_t s0 = ptx::smem_u32(smem);
    const uint64_t dq = tile_desc<false>(s0 + C::OFF_Q, 128);
    const uint64_t dk = tile_desc<false>(s0 + C::OFF_K, 128);
    const uint64_t dv = tile_desc<true>(s0 + C::OFF_V, 128);
    constexpr uint32_t TSTEP = C::TILE_BYTES / 16;
    ptx::mbar_wait_u(&bars[F_Q_FULL], 0);
    uint32_t kc = 0, sc = 0;
    // S(sc) = Q K^T into S buffer sc % 2 once the softmax has read S(sc - 2)
    auto issue_s = [&]() {
      const uint32_t st = kc & 1, sb = sc & 1;
      ptx::mbar_wait_u(&bars[F_K_FULL0 + st], (kc >> 1) & 1);
      if (sc >= 2) ptx::mbar_wait_u(&bars[F_S_EMPTY0 + sb], ((sc >> 1) - 1) & 1);
      ptx::tc_fence_after();
      umma_gemm_d<128, C::BN, D, false, false, 128, 128>(tbase + (sb ? C::T_S1 : C::T_S0), dq,
                                                         dk + st * TSTEP, false);
      ptx::mma_commit_e(&bars[F_K_EMPTY0 + st]);
      ptx::mma_commit_e(&bars[F_S_FULL0 + sb]);
      ++kc;
      ++sc;
    };
    for (int j = 0; j < n_kv; ++j) issue_s();  // pass 1: statistics
    issue_s();                                 // pass 2, key tile 0
    for (int j = 0; j < n_kv; ++j) {
      if (j + 1 < n_kv) issue_s();  // S of the next tile while the softmax writes P(j)
      ptx::mbar_wait_u(&bars[F_P_FULL], j & 1);
      const uint32_t vs = j & 1;
      ptx::mbar_wait_u(&bars[F_V_FULL0 + vs], (j >> 1) & 1);
      ptx::tc_fence_after();
      // O += P V  (A = P from TMEM [128 q x 128 keys], B = V [keys x D] MN-major)
      umma_gemm_ts_d<D, C::BN, true, 128>(tbase + C::T_O, tbase + C::T_P, dv + vs * TSTEP, j > 0);
      ptx::mma_commit_e(&bars[F_V_EMPTY0 + vs]);
      ptx::mma_commit_e(&bars[F_P_EMPTY]);
    }
    ptx::mma_commit_e(&bars[F_O_FULL]);
  } else if (warp >= 4) {
    // ---------------- softmax: thread = Q row ----------------
    const int rloc = (warp & 3) * 32 + lane;
    const int row = qt * C::BM + rloc;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const float sl2 = args.scale_log2;
    float m = -INFINITY, l = 0.f;  // log2-domain running max and sum
    uint32_t sc = 0;
    // pass 1
    for (int j = 0; j < n_kv; ++j, ++sc) {
      const uint32_t tS = tbase + lane_off + ((sc & 1) ? C::T_S1 : C::T_S0);
      ptx::mbar_wait(&bars[F_S_FULL0 + (sc & 1)], (sc >> 1) & 1);
      ptx::tc_fence_after();
      const bool diag = args.causal && j == qt;
#pragma unroll 1
      for (int c0 = 0; c0 < C::BN; c0 += 32) {
        float s[32];
        ptx::tmem_ld32(tS + c0, s);
        ptx::tmem_wait_ld();
        float mx = m;
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const float x = (diag && c0 + c > rloc) ? -INFINITY : s[c] * sl2;
          s[c] = x;
          mx = fmaxf(mx, x);
        }
        float sum = 0.f;
#pragma unroll
        for (int c = 0; c < 32; ++c) sum += fwd_exp2(s[c] - mx);
        l = l * fwd_exp2(m - mx) + sum;
        m = mx;
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&bars[F_S_EMPTY0 + (sc & 1)]);
    }
    const float L2 = m + log2f(l);  // log2-domain logsumexp of the row
    // pass 2
    for (int j = 0; j < n_kv; ++j, ++sc) {
      const uint32_t tS = tbase + lane_off + ((sc & 1) ? C::T_S1 : C::T_S0);
      ptx::mbar_wait(&bars[F_S_FULL0 + (sc & 1)], (sc >> 1) & 1);
      ptx::tc_fence_after();
      const bool diag = args.causal && j == qt;
#pragma unroll 1
      for (int c0 = 0; c0 < C::BN; c0 += 32) {
        float s[32];
        ptx::tmem_ld32(tS + c0, s);
        ptx::tmem_wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int c = 0; c < 32; c += 2) {
          float p0 = fwd_exp2(fmaf(s[c], sl2, -L2)), p1 = fwd_exp2(fmaf(s[c + 1], sl2, -L2));
          if (diag && c0 + c > rloc) p0 = 0.f;
          if (diag && c0 + c + 1 > rloc) p1 = 0.f;
          __nv_bfloat162 pv = __floats2bfloat162_rn(p0, p1);
          pk[c / 2] = *reinterpret_cast<uint32_t*>(&pv);
        }
        // P buffer free once O += P(j-1) V has completed
        if (c0 == 0 && j >= 1) ptx::mbar_wait(&bars[F_P_EMPTY], (j - 1) & 1);
        ptx::tmem_st16(tbase + lane_off + C::T_P + c0 / 2, pk);
      }
      ptx::tmem_wait_st();
      ptx::tc_fence_before();
      ptx::mbar_arrive(&bars[F_S_EMPTY0 + (sc & 1)]);
      ptx::mbar_arrive(&bars[F_P_FULL]);
    }
    // epilogue: O (already normalised) -> bf16, L -> natural log
    ptx::mbar_wait(&bars[F_O_FULL], 0);
    ptx::tc_fence_after();
    __nv_bfloat16* orow = args.o + ((static_cast<size_t>(b) * args.N + row) * args.H + h) * D;
#pragma unroll 1
    for (int c0 = 0; c0 < D; c0 += 32) {
      float ov[32];
      ptx::tmem_ld32(tbase + lane_off + C::T_O + c0, ov);
      ptx::tmem_wait_ld();
#pragma unroll
      for (int e = 0; e < 32; e += 8) {
        uint4 w;
        __nv_bfloat162 t0 = __floats2bfloat162_rn(ov[e], ov[e + 1]);
        __nv_bfloat162 t1 = __floats2bfloat162_rn(ov[e + 2], ov[e + 3]);
        __nv_bfloat162 t2 = __floats2bfloat162_rn(ov[e + 4], ov[e + 5]);
        __nv_bfloat162 t3 = __floats2bfloat162_rn(ov[e + 6], ov[e + 7]);
        w.x = *reinterpret_cast<uint32_t*>(&t0);
        w.y = *reinterpret_cast<uint32_t*>(&t1);
        w.z = *reinterpret_cast<uint32_t*>(&t2);
        w.w = *reinterpret_cast<uint32_t*>(&t3);
        *reinterpret_cast<uint4*>(orow + c0 + e) = w;
      }
    }
    args.lse[(static_cast<size_t>(bh)) * args.N + row] = L2 * 0.6931471805599453f;
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tbase);
  }
}

}  // namespace dash
