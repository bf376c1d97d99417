// Debug probes for the tcgen05 / TMA conventions the backward kernel relies
// on (built into libdash_probe.so, used only by tests/test_gpu_probe.py).
//
//  * dash_probe_umma: one CTA stores A and B into SW128 tiles (K-major or
//    MN-major, thread-written with the same swizzle formula the softmax role
//    uses), issues one tcgen05 GEMM, reads D back from TMEM.
//  * dash_probe_tma: TMA-loads a [rows x 64k] bf16 box with SWIZZLE_128B and
//    dumps the raw shared-memory bytes, to pin sw128_chunk_offset().
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "umma.cuh"

namespace dash {

template <int N, int K, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(128, 1)
    probe_umma_kernel(const __nv_bfloat16* A, const __nv_bfloat16* Bt, float* D) {
  constexpr int M = 128;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem;                      // M*K*2 bytes
  uint8_t* sB = smem + M * K * 2;          // N*K*2 bytes
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;

  // A logical [M][K] (row-major in global).  K-major: stored [M][K];
  // MN-major: stored [K][M].
  for (int e = tid; e < M * K / 8; e += blockDim.x) {
    if (!A_MN) {
      const int r = e / (K / 8), ch = e % (K / 8);
      const uint4 v = *reinterpret_cast<const uint4*>(A + r * K + ch * 8);
      *reinterpret_cast<uint4*>(sA + sw128_chunk_offset(M, r, ch)) = v;
    } else {
      const int r = e / (M / 8), ch = e % (M / 8);  // stored row r = k index
      __align__(16) __nv_bfloat16 tmp[8];
      for (int t = 0; t < 8; ++t) tmp[t] = A[(ch * 8 + t) * K + r];
      *reinterpret_cast<uint4*>(sA + sw128_chunk_offset(K, r, ch)) =
          *reinterpret_cast<uint4*>(tmp);
    }
  }
  // Bt logical [N][K] (B = Bt^T is K x N).  K-major: stored [N][K];
  // MN-major: stored [K][N].
  for (int e = tid; e < N * K / 8; e += blockDim.x) {
    if (!B_MN) {
      const int r = e / (K / 8), ch = e % (K / 8);
      const uint4 v = *reinterpret_cast<const uint4*>(Bt + r * K + ch * 8);
      *reinterpret_cast<uint4*>(sB + sw128_chunk_offset(N, r, ch)) = v;
    } else {
      const int r = e / (N / 8), ch = e % (N / 8);
      __align__(16) __nv_bfloat16 tmp[8];
      for (int t = 0; t < 8; ++t) tmp[t] = Bt[(ch * 8 + t) * K + r];
      *reinterpret_cast<uint4*>(sB + sw128_chunk_offset(K, r, ch)) =
          *reinterpret_cast<uint4*>(tmp);
    }
  }
  ptx::fence_async_smem();
  if (warp == 0) ptx::tmem_alloc<256>(&tmem_base);
  if (tid == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = tmem_base;
  if (warp == 0) {
    umma_gemm<M, N, K, A_MN, B_MN>(tbase, ptx::smem_u32(sA), A_MN ? K : M, ptx::smem_u32(sB),
                                   B_MN ? K : N, false);
    ptx::mma_commit_e(&bar);
  }
  __syncwarp();
  ptx::mbar_wait(&bar, 0);
  ptx::tc_fence_after();
  const uint32_t lane_base = static_cast<uint32_t>(warp * 32) << 16;
  for (int c = 0; c < N; c += 32) {
    float v[32];
    ptx::tmem_ld32(tbase + lane_base + c, v);
    ptx::tmem_wait_ld();
    for (int t = 0; t < 32; ++t) D[(warp * 32 + (tid & 31)) * N + c + t] = v[t];
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc<256>(tbase);
}

// A from TMEM ("TS" MMA): each thread writes its row of A (K bf16, packed)
// with tcgen05.st, B from smem.
template <int N, int K, bool B_MN>
__global__ void __launch_bounds__(128, 1)
    probe_umma_ts_kernel(const __nv_bfloat16* A, const __nv_bfloat16* Bt, float* D) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sB = smem;
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int e = tid; e < N * K / 8; e += blockDim.x) {
    if (!B_MN) {
      const int r = e / (K / 8), ch = e % (K / 8);
      *reinterpret_cast<uint4*>(sB + sw128_chunk_offset(N, r, ch)) =
          *reinterpret_cast<const uint4*>(Bt + r * K + ch * 8);
    } else {
      const int r = e / (N / 8), ch = e % (N / 8);
      __align__(16) __nv_bfloat16 tmp[8];
      for (int t = 0; t < 8; ++t) tmp[t] = Bt[(ch * 8 + t) * K + r];
      *reinterpret_cast<uint4*>(sB + sw128_chunk_offset(K, r, ch)) = *reinterpret_cast<uint4*>(tmp);
    }
  }
  ptx::fence_async_smem();
  if (warp == 0) ptx::tmem_alloc<256>(&tmem_base);
  if (tid == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = tmem_base;
  const uint32_t lane_base = static_cast<uint32_t>(warp * 32) << 16;
  // A row `tid` -> TMEM lane tid, columns 128 .. 128 + K/2
  for (int c = 0; c < K / 2; c += 16) {
    uint32_t r[16];
    for (int t = 0; t < 16; ++t) {
      __nv_bfloat162 v;
      v.x = A[tid * K + 2 * (c + t)];
      v.y = A[tid * K + 2 * (c + t) + 1];
      r[t] = *reinterpret_cast<uint32_t*>(&v);
    }
    ptx::tmem_st16(tbase + lane_base + 128 + c, r);
  }
  ptx::tmem_wait_st();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 0) {
    umma_gemm_ts<N, K, B_MN>(tbase, tbase + 128, ptx::smem_u32(sB), B_MN ? K : N, false);
    ptx::mma_commit_e(&bar);
  }
  __syncwarp();
  ptx::mbar_wait(&bar, 0);
  ptx::tc_fence_after();
  for (int c = 0; c < N; c += 32) {
    float v[32];
    ptx::tmem_ld32(tbase + lane_base + c, v);
    ptx::tmem_wait_ld();
    for (int t = 0; t < 32; ++t) D[tid * N + c + t] = v[t];
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc<256>(tbase);
}

// Throughput microbenchmark: `reps` back-to-back GEMMs of K = 128 (8 MMAs)
// of shape 128 x N, operands from smem (SS, A/B majorness as given) or A from
// TMEM (TS).  Returns clock64 cycles per GEMM via out[blockIdx.x].
template <int N, int MODE>  // MODE 0: SS K/K, 1: SS K/MN, 2: SS MN/MN, 3: TS (B MN)
__global__ void __launch_bounds__(128, 1) probe_mma_rate_kernel(int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int warp = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0);
  for (int i = threadIdx.x; i < (128 * 128 + N * 128) / 8; i += 128)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u, 0, 0x3f803f80u, 0);
  ptx::fence_async_smem();
  if (warp == 0) ptx::tmem_alloc<512>(&tmem_base);
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tb = tmem_base;
  if (warp == 0) {
    const uint32_t sA = ptx::smem_u32(smem), sB = ptx::smem_u32(smem + 128 * 128 * 2);
    const uint64_t ak = tile_desc<false>(sA, 128), amn = tile_desc<true>(sA, 128);
    const uint64_t bk = tile_desc<false>(sB, N), bmn = tile_desc<true>(sB, 128);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (MODE == 0) umma_gemm_d<128, N, 128, false, false, 128, N>(tb, ak, bk, r > 0);
      if (MODE == 1) umma_gemm_d<128, N, 128, false, true, 128, 128>(tb, ak, bmn, r > 0);
      if (MODE == 2) umma_gemm_d<128, N, 128, true, true, 128, 128>(tb, amn, bmn, r > 0);
      if (MODE == 3) umma_gemm_ts_d<N, 128, true, 128>(tb, tb + 256, bmn, r > 0);
    }
    ptx::mma_commit_e(&bar);
    ptx::mbar_wait_u(&bar, 0);
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / reps;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) ptx::tmem_dealloc<512>(tb);
}

// TMEM <-> register throughput: NW warps (warp w reads lane quarter w % 4),
// each doing `reps` rounds of `inflight` tcgen05.ld.32x32b.x32 (4 KB per warp
// each) followed by one wait::ld (MODE 0), or tcgen05.st.32x32b.x16 + wait::st
// (MODE 1).  out[blockIdx.x] = cycles per round of the slowest warp, so an
// SM-wide figure is NW * inflight * 4 KB (ld) / cycles.
template <int MODE, int INFLIGHT>
__global__ void __launch_bounds__(512, 1) probe_tmem_rate_kernel(int reps, long long* out) {
  __shared__ uint32_t tmem_base;
  __shared__ long long worst;
  const int warp = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0);
  if (warp == 0) ptx::tmem_alloc<512>(&tmem_base);
  if (threadIdx.x == 0) worst = 0;
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tb = tmem_base + (static_cast<uint32_t>((warp & 3) * 32) << 16);
  float acc = 0.f;
  const long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (MODE == 0) {
      float v[INFLIGHT][32];
#pragma unroll
      for (int i = 0; i < INFLIGHT; ++i) ptx::tmem_ld32(tb + ((warp >> 2) * 128 + i * 32) % 512, v[i]);
      ptx::tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < INFLIGHT; ++i) acc += v[i][i & 31];
    } else {
      uint32_t v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = static_cast<uint32_t>(r + i);
#pragma unroll
      for (int i = 0; i < INFLIGHT; ++i) ptx::tmem_st16(tb + ((warp >> 2) * 128 + i * 16) % 512, v);
      ptx::tmem_wait_st();
    }
  }
  const long long t1 = clock64();
  if (acc == 12345.f) out[0] = -1;  // keep the loads alive
  atomicMax(reinterpret_cast<unsigned long long*>(&worst), static_cast<unsigned long long>(t1 - t0));
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = worst / reps;
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem_base);
  }
}

// Throughput of adding a 32 KB fp32 tile (64 rows x 128) per iteration into
// a private global region: mode 0 = red.global.add.v4.f32 from 128 threads,
// mode 1 = same + membar.gl per iteration (ordered hand-off cost).
__global__ void __launch_bounds__(128, 1) probe_red_rate_kernel(float* dst, int iters, int mode,
                                                                long long* out) {
  float* base = dst + static_cast<size_t>(blockIdx.x) * 64 * 128;
  const int t = threadIdx.x;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    // thread t covers rows r = t / 32 + 4 k, float4 column (t % 32)
#pragma unroll 4
    for (int k = 0; k < 16; ++k) {
      float* p = base + (t / 32 + 4 * k) * 128 + (t % 32) * 4;
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1.f), "f"(1.f),
                   "f"(1.f), "f"(1.f)
                   : "memory");
    }
    if (mode == 1) asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
  const long long t1 = clock64();
  if (t == 0) out[blockIdx.x] = (t1 - t0) / iters;
}

// TMA load latency: each CTA repeatedly loads two 64-col x `rows` bf16 boxes
// (a Q sub-tile of [B,N,H,d] at d = 128) into smem and waits; returns the mean
// cycles from issue to mbarrier completion in out[blockIdx.x].
__global__ void probe_tma_latency_kernel(const __grid_constant__ CUtensorMap tmap, int rows,
                                         int iters, int row_stride_tiles, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  long long total = 0;
  if (threadIdx.x == 0) {
    for (int it = 0; it < iters; ++it) {
      const int r0 = ((blockIdx.x * 7 + it) % row_stride_tiles) * rows;
      const long long t0 = clock64();
      ptx::mbar_arrive_expect_tx(&bar, 2 * rows * 128);
      ptx::tma_load_2d(smem, &tmap, &bar, 0, r0);
      ptx::tma_load_2d(smem + rows * 128, &tmap, &bar, 64, r0);
      ptx::mbar_wait(&bar, it & 1);
      total += clock64() - t0;
    }
    out[blockIdx.x] = total / iters;
  }
}

__global__ void probe_tma_kernel(const __grid_constant__ CUtensorMap tmap, int rows, int cols,
                                 uint8_t* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  __shared__ uint64_t bar;
  const int bytes = rows * cols * 2;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ptx::mbar_arrive_expect_tx(&bar, bytes);
    for (int b = 0; b < cols / 64; ++b)
      ptx::tma_load_2d(smem + b * rows * 128, &tmap, &bar, b * 64, 0);
  }
  ptx::mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < bytes; i += blockDim.x) out[i] = smem[i];
}

}  // namespace dash

using namespace dash;

extern "C" __attribute__((visibility("default"))) int dash_probe_umma(int n, int k, int a_mn, int b_mn, const void* A, const void* Bt,
                               float* D) {
  const size_t smem = 1024 + (128 * k + n * k) * 2;
  auto launch = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<1, 128, smem>>>(static_cast<const __nv_bfloat16*>(A),
                           static_cast<const __nv_bfloat16*>(Bt), D);
  };
#define PROBE_CASE(NN, KK)                                                   \
  if (n == NN && k == KK) {                                                  \
    if (!a_mn && !b_mn) launch(probe_umma_kernel<NN, KK, false, false>);     \
    if (!a_mn && b_mn) launch(probe_umma_kernel<NN, KK, false, true>);       \
    if (a_mn && !b_mn) launch(probe_umma_kernel<NN, KK, true, false>);       \
    if (a_mn && b_mn) launch(probe_umma_kernel<NN, KK, true, true>);         \
  }
  PROBE_CASE(64, 64)
  PROBE_CASE(64, 128)
  PROBE_CASE(128, 64)
  PROBE_CASE(128, 128)
#undef PROBE_CASE
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) fprintf(stderr, "dash_probe_umma: %s\n", cudaGetErrorString(e));
  return static_cast<int>(e);
}

extern "C" __attribute__((visibility("default"))) int dash_probe_umma_ts(int n, int k, int b_mn,
                                                                        const void* A,
                                                                        const void* Bt, float* D) {
  const size_t smem = 1024 + n * k * 2;
  auto launch = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<1, 128, smem>>>(static_cast<const __nv_bfloat16*>(A),
                           static_cast<const __nv_bfloat16*>(Bt), D);
  };
  if (n == 128 && k == 64) b_mn ? launch(probe_umma_ts_kernel<128, 64, true>)
                                : launch(probe_umma_ts_kernel<128, 64, false>);
  if (n == 64 && k == 128) b_mn ? launch(probe_umma_ts_kernel<64, 128, true>)
                                : launch(probe_umma_ts_kernel<64, 128, false>);
  if (n == 128 && k == 128) b_mn ? launch(probe_umma_ts_kernel<128, 128, true>)
                                 : launch(probe_umma_ts_kernel<128, 128, false>);
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) fprintf(stderr, "dash_probe_umma_ts: %s\n", cudaGetErrorString(e));
  return static_cast<int>(e);
}

extern "C" __attribute__((visibility("default"))) int dash_probe_mma_rate(int n, int mode, int reps,
                                                                         int grid,
                                                                         long long* out) {
  const size_t smem = 1024 + (128 * 128 + 256 * 128) * 2;
  auto launch = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, 128, smem>>>(reps, out);
  };
#define RATE_CASE(NN)                                        \
  if (n == NN) {                                             \
    if (mode == 0) launch(probe_mma_rate_kernel<NN, 0>);     \
    if (mode == 1) launch(probe_mma_rate_kernel<NN, 1>);     \
    if (mode == 2) launch(probe_mma_rate_kernel<NN, 2>);     \
    if (mode == 3) launch(probe_mma_rate_kernel<NN, 3>);     \
  }
  RATE_CASE(64)
  RATE_CASE(128)
  RATE_CASE(256)
#undef RATE_CASE
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaGetLastError();
  return static_cast<int>(e);
}

// MUFU ex2 vs FMA-pipe polynomial exp2 throughput: each thread runs `reps`
// rounds over 8 independent values.  MODE 0: ex2.approx.ftz.f32; MODE 1: a
// degree-3 polynomial 2^x (floor/fraction split, FFMA Horner, exponent add)
// as in FlashAttention-4's software exp2.  out = cycles per round per CTA.
template <int MODE>
__global__ void __launch_bounds__(1024, 1) probe_exp_rate_kernel(int reps, float* sink, long long* out) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  const long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float y;
      if (MODE == 0) {
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[i]));
      } else {
        const float xf = fmaxf(x[i], -127.f);
        const float fl = floorf(xf);
        const float f = xf - fl;
        float p = fmaf(f, 0.0555041086648216f, 0.2402264923172050f);
        p = fmaf(p, f, 0.6931471805599453f);
        p = fmaf(p, f, 1.0f);
        y = __int_as_float(__float_as_int(p) + (static_cast<int>(fl) << 23));
      }
      x[i] = y - 1.0f;
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.f) sink[threadIdx.x] = s;
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / reps;
}

extern "C" __attribute__((visibility("default"))) int dash_probe_exp_rate(int mode, int nthreads,
                                                                         int reps, int grid,
                                                                         float* sink,
                                                                         long long* out) {
  if (mode == 0) probe_exp_rate_kernel<0><<<grid, nthreads>>>(reps, sink, out);
  else probe_exp_rate_kernel<1><<<grid, nthreads>>>(reps, sink, out);
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaGetLastError();
  return static_cast<int>(e);
}

extern "C" __attribute__((visibility("default"))) int dash_probe_tmem_rate(int mode, int inflight,
                                                                          int nwarps, int reps,
                                                                          int grid,
                                                                          long long* out) {
  auto launch = [&](auto kern) { kern<<<grid, nwarps * 32>>>(reps, out); };
  if (mode == 0 && inflight == 1) launch(probe_tmem_rate_kernel<0, 1>);
  if (mode == 0 && inflight == 2) launch(probe_tmem_rate_kernel<0, 2>);
  if (mode == 0 && inflight == 4) launch(probe_tmem_rate_kernel<0, 4>);
  if (mode == 1 && inflight == 1) launch(probe_tmem_rate_kernel<1, 1>);
  if (mode == 1 && inflight == 4) launch(probe_tmem_rate_kernel<1, 4>);
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaGetLastError();
  return static_cast<int>(e);
}

extern "C" __attribute__((visibility("default"))) int dash_probe_red_rate(float* dst, int iters,
                                                                         int mode, int grid,
                                                                         long long* out) {
  probe_red_rate_kernel<<<grid, 128>>>(dst, iters, mode, out);
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaGetLastError();
  return static_cast<int>(e);
}

extern "C" __attribute__((visibility("default"))) int dash_probe_tma_latency(
    const void* src, int total_rows, int ld_elems, int rows, int iters, int grid, long long* out) {
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  cudaDriverEntryPointQueryResult qres;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode),
                          cudaEnableDefault, &qres);
  if (!encode) return -1;
  CUtensorMap tmap;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(ld_elems), static_cast<cuuint64_t>(total_rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld_elems) * 2};
  cuuint32_t box[2] = {64, static_cast<cuuint32_t>(rows)};
  cuuint32_t estr[2] = {1, 1};
  if (encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(src), dims, strides,
             box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return -2;
  const size_t smem = 1024 + 2 * rows * 128;
  cudaFuncSetAttribute(probe_tma_latency_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  probe_tma_latency_kernel<<<grid, 32, smem>>>(tmap, rows, iters, total_rows / rows, out);
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaGetLastError();
  return static_cast<int>(e);
}

extern "C" __attribute__((visibility("default"))) int dash_probe_tma(const void* src, int rows, int cols, int ld_elems, void* out) {
  PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  cudaDriverEntryPointQueryResult qres;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode),
                          cudaEnableDefault, &qres);
  if (!encode) return -1;
  CUtensorMap tmap;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(ld_elems), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld_elems) * 2};
  cuuint32_t box[2] = {64, static_cast<cuuint32_t>(rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(src), dims,
                      strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return -2;
  const size_t smem = 1024 + rows * cols * 2;
  cudaFuncSetAttribute(probe_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  probe_tma_kernel<<<1, 128, smem>>>(tmap, rows, cols, static_cast<uint8_t*>(out));
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaGetLastError();
  return static_cast<int>(e);
}

// Pair-MMA (cta_group::2) throughput: a cluster of two CTAs, the leader issues
// `reps` rounds of one GEMM shape of the CTA-pair backward (bwd2.cuh) and
// waits for completion (multicast commit).  MODE 0: M=256 N=64 K=128 SS
// (S^T / dP^T); MODE 1: M=256 N=128 K=64 TS (dV / dK); MODE 2: M=128 N=64
// K=256 SS, A MN-major SW128, B MN-major SW64 (dQ^T).  out[cluster] = cycles
// per round.
template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    probe_pair_mma_rate_kernel(int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int warp = __shfl_sync(0xffffffffu, threadIdx.x / 32, 0);
  const uint32_t cta = ptx::cluster_ctarank();
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += 128)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  ptx::fence_async_smem();
  if (warp == 0) ptx::tmem_alloc2<512>(&tmem_base);
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tb = tmem_base;
  if (warp == 0 && cta == 0) {
    const uint32_t s0 = ptx::smem_u32(smem);
    const uint64_t aK = tile_desc<false>(s0, 128);
    const uint64_t bK = tile_desc<false>(s0 + 32768, 32);
    const uint64_t bMN = ptx::sdesc_sw128(s0 + 65536, 64 * 128, 1024);
    const uint64_t aMN = ptx::sdesc_sw128(s0, 256 * 128, 1024);
    const uint64_t bS64 = ptx::sdesc_sw64(s0 + 65536, 256 * 64, 512);
    constexpr uint32_t ID0 = ptx::idesc_bf16(256, 64, 0, 0);
    constexpr uint32_t ID1 = ptx::idesc_bf16(256, 128, 0, 1);
    constexpr uint32_t ID2 = ptx::idesc_bf16(128, 64, 1, 1);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (MODE == 0) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          ptx::mma2_bf16_e(tb, aK + kstep<false>(kk, 128), bK + kstep<false>(kk, 32), ID0, 1);
      } else if (MODE == 1) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          ptx::mma2_bf16_ts_e(tb + 128, tb + 448 + kk * 8, bMN + kstep<true>(kk, 64), ID1, 1);
      } else if (MODE == 2) {
#pragma unroll
        for (int kk = 0; kk < 16; ++kk)
          ptx::mma2_bf16_e(tb + 384, aMN + kk * 128, bS64 + kk * 64, ID2, 1);
      } else {
        // MODE 3: one sub-tile of the pair kernel in its issue order:
        // S^T, dP^T (SS), dK, dV (TS), dQ^T (SS, M = 128)
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          ptx::mma2_bf16_e(tb, aK + kstep<false>(kk, 128), bK + kstep<false>(kk, 32), ID0, 1);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          ptx::mma2_bf16_e(tb + 64, aK + kstep<false>(kk, 128), bK + kstep<false>(kk, 32), ID0, 1);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          ptx::mma2_bf16_ts_e(tb + 256, tb + 480 + kk * 8, bMN + kstep<true>(kk, 64), ID1, 1);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          ptx::mma2_bf16_ts_e(tb + 128, tb + 448 + kk * 8, bMN + kstep<true>(kk, 64), ID1, 1);
#pragma unroll
        for (int kk = 0; kk < 16; ++kk)
          ptx::mma2_bf16_e(tb + 384, aMN + kk * 128, bS64 + kk * 64, ID2, 1);
      }
    }
    ptx::mma2_commit_mc_e(&bar);
    ptx::mbar_wait_u(&bar, 0);
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x / 2] = (t1 - t0) / reps;
  } else if (warp == 0) {
    ptx::mbar_wait_u(&bar, 0);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc2<512>(tb);
  }
}

extern "C" __attribute__((visibility("default"))) int dash_probe_pair_mma_rate(int mode, int reps,
                                                                              int clusters,
                                                                              long long* out) {
  const size_t smem = 1024 + 96 * 1024;
  auto launch = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<2 * clusters, 128, smem>>>(reps, out);
  };
  if (mode == 0) launch(probe_pair_mma_rate_kernel<0>);
  if (mode == 1) launch(probe_pair_mma_rate_kernel<1>);
  if (mode == 2) launch(probe_pair_mma_rate_kernel<2>);
  if (mode == 3) launch(probe_pair_mma_rate_kernel<3>);
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaGetLastError();
  return static_cast<int>(e);
}
