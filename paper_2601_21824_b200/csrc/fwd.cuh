// K6: attention forward producing O and L (the inputs Algorithm 1 requires,
// PAPER.md P:353).  Correctness-first fp32 SIMT kernel (not a timed path; the
// tcgen05 forward is NEXT-2 in SURVEY.md §8(f)).
//
// CTA = 64 query rows of one (b, h); 256 threads = 4 threads per row, thread
// p of a row owns dims {16m + 4p .. 16m + 4p + 3}.  K/V tiles of 64 rows are
// staged in smem as fp32; online softmax in fp32 with natural-log L.
#pragma once
#include <cuda_bf16.h>

namespace dash {

template <int D>
__global__ void __launch_bounds__(256)
    dash_fwd_kernel(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k,
                    const __nv_bfloat16* __restrict__ v, __nv_bfloat16* __restrict__ o,
                    float* __restrict__ lse, int B, int N, int H, float scale, int causal) {
  constexpr int BQ = 64, BK = 64, DP = D / 4;  // dims per thread
  extern __shared__ float4 fwd_smem[];
  float* sK = reinterpret_cast<float*>(fwd_smem);
  float* sV = sK + BK * D;
  const int tid = threadIdx.x;
  const int r = tid >> 2, p = tid & 3;
  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const int q0 = blockIdx.x * BQ;
  const int qr = q0 + r;
  float qv[DP], acc[DP];
  const size_t qoff = ((static_cast<size_t>(b) * N + qr) * H + h) * D;
#pragma unroll
  for (int m = 0; m < D / 16; ++m)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      qv[m * 4 + e] = __bfloat162float(q[qoff + 16 * m + 4 * p + e]) * scale;
      acc[m * 4 + e] = 0.f;
    }
  float mrow = -INFINITY, lrow = 0.f;
  const int kend = causal ? (q0 + BQ) : N;
  for (int k0 = 0; k0 < kend; k0 += BK) {
    __syncthreads();
    for (int e = tid; e < BK * D / 8; e += 256) {
      const int rr = e / (D / 8), cc = (e % (D / 8)) * 8;
      const size_t off = ((static_cast<size_t>(b) * N + k0 + rr) * H + h) * D + cc;
      const uint4 kk = *reinterpret_cast<const uint4*>(k + off);
      const uint4 vv = *reinterpret_cast<const uint4*>(v + off);
      const __nv_bfloat162* pk = reinterpret_cast<const __nv_bfloat162*>(&kk);
      const __nv_bfloat162* pv = reinterpret_cast<const __nv_bfloat162*>(&vv);
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const float2 fk = __bfloat1622float2(pk[t]);
        const float2 fv = __bfloat1622float2(pv[t]);
        sK[rr * D + cc + 2 * t] = fk.x;
        sK[rr * D + cc + 2 * t + 1] = fk.y;
        sV[rr * D + cc + 2 * t] = fv.x;
        sV[rr * D + cc + 2 * t + 1] = fv.y;
      }
    }
    __syncthreads();
    float s[BK];
    float tmax = -INFINITY;
#pragma unroll 8
    for (int c = 0; c < BK; ++c) {
      float part = 0.f;
#pragma unroll
      for (int m = 0; m < D / 16; ++m) {
        const float4 kk = *reinterpret_cast<const float4*>(sK + c * D + 16 * m + 4 * p);
        part = fmaf(qv[m * 4], kk.x, part);
        part = fmaf(qv[m * 4 + 1], kk.y, part);
        part = fmaf(qv[m * 4 + 2], kk.z, part);
        part = fmaf(qv[m * 4 + 3], kk.w, part);
      }
      part += __shfl_xor_sync(0xffffffffu, part, 1);
      part += __shfl_xor_sync(0xffffffffu, part, 2);
      if (causal && k0 + c > qr) part = -INFINITY;
      s[c] = part;
      tmax = fmaxf(tmax, part);
    }
    const float mnew = fmaxf(mrow, tmax);
    const float alpha = (mrow == -INFINITY) ? 0.f : __expf(mrow - mnew);
    lrow *= alpha;
#pragma unroll
    for (int e = 0; e < DP; ++e) acc[e] *= alpha;
#pragma unroll 4
    for (int c = 0; c < BK; ++c) {
      const float pc = (s[c] == -INFINITY) ? 0.f : __expf(s[c] - mnew);
      lrow += pc;
#pragma unroll
      for (int m = 0; m < D / 16; ++m) {
        const float4 vv = *reinterpret_cast<const float4*>(sV + c * D + 16 * m + 4 * p);
        acc[m * 4] = fmaf(pc, vv.x, acc[m * 4]);
        acc[m * 4 + 1] = fmaf(pc, vv.y, acc[m * 4 + 1]);
        acc[m * 4 + 2] = fmaf(pc, vv.z, acc[m * 4 + 2]);
        acc[m * 4 + 3] = fmaf(pc, vv.w, acc[m * 4 + 3]);
      }
    }
    mrow = mnew;
  }
  const float inv = 1.f / lrow;
#pragma unroll
  for (int m = 0; m < D / 16; ++m)
#pragma unroll
    for (int e = 0; e < 4; ++e) o[qoff + 16 * m + 4 * p + e] = __float2bfloat16_rn(acc[m * 4 + e] * inv);
  if (p == 0) lse[static_cast<size_t>(bh) * N + qr] = mrow + logf(lrow);
}

}  // namespace dash
