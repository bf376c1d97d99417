// DASH deterministic attention backward -- sm_100a kernels (Algorithm 1,
// PAPER.md P:351-397, re-designed for tcgen05/TMEM/TMA).
//
// One persistent CTA per SM claims jobs (one KV tile, or a Symmetric-Shift
// pair of KV tiles) in head-major order (AMB-7) and walks the job's Q tiles
// in the schedule's order (Alg.1 lines 9/18/31 "[DASH]").  Per Q sub-tile of
// BR rows (the 128-row Q tile of the schedule model split in 128/BR):
//
//   S^T  = K Q^T           (TMEM, lanes = KV rows)       tcgen05 SS
//   dP^T = V dO^T          (TMEM)                         tcgen05 SS
//   P^T  = exp2(S^T*scale*log2e - L*log2e) ; dS^T = P^T o (dP^T - D)
//                          (softmax warps: TMEM -> regs -> bf16 SW128 smem)
//   dV  += P^T dO ;  dK += dS^T Q   (TMEM accumulators, whole job)
//   dQ_part = dS K  (d = 64)  or  dQ_part^T = K^T dS^T  (d = 128)   (TMEM)
//   ordered reduction: wait ticket == rank, TMA reduce-add (rank 0: store)
//   of the fp32 partial into dQacc, release ticket = rank + 1
//                          (Alg.1 lines 30-36)
//
// Warp roles (12 warps): 0 = TMA producer, 1 = MMA issuer + TMEM owner,
// 4-7 = softmax / dS / dK-dV epilogue (TMEM lane quarter = warp % 4),
// 8-11 = dQ drain + ordered reduction + job claiming.  Warps 2-3 idle.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "umma.cuh"

namespace dash {

struct BwdArgs {
  const float* lse;      // [B,H,N] natural log
  const float* Dvec;     // [B,H,N] rowsum(dO*O)
  __nv_bfloat16* dk;     // [B,N,H,d]
  __nv_bfloat16* dv;     // [B,N,H,d]
  int* tickets;          // [B*H][N/BR]
  int* job_counter;      // 1
  int* error_flag;       // 1
  const int* job_begin;  // [jobs_per_head + 1]
  const int2* tasks;     // {kv | q << 16, rank}
  int B, N, H;
  int jobs_per_head;
  int total_jobs;
  float scale;
  float scale_log2;
  int causal;
  int deterministic;
};

template <int D>
struct BwdCfg {
  static constexpr int BC = 128;                 // KV tile rows (TMEM lanes)
  static constexpr int BR = (D == 128) ? 64 : 128;  // Q sub-tile rows
  static constexpr int NSUB = 128 / BR;          // sub-tiles per schedule Q tile
  static constexpr int NP = (D == 128) ? 2 : 1;  // P/dS smem buffers
  static constexpr uint32_t KV_BYTES = BC * D * 2;
  static constexpr uint32_t Q_BYTES = BR * D * 2;
  static constexpr uint32_t P_BYTES = BC * BR * 2;
  static constexpr uint32_t DQ_BYTES = BR * D * 4;
  static constexpr uint32_t OFF_K = 0;
  static constexpr uint32_t OFF_V = OFF_K + KV_BYTES;
  static constexpr uint32_t OFF_Q = OFF_V + KV_BYTES;         // 2 stages
  static constexpr uint32_t OFF_DO = OFF_Q + 2 * Q_BYTES;     // 2 stages
  static constexpr uint32_t OFF_P = OFF_DO + 2 * Q_BYTES;     // NP buffers
  static constexpr uint32_t OFF_DS = OFF_P + NP * P_BYTES;    // NP buffers
  static constexpr uint32_t OFF_DQ = OFF_DS + NP * P_BYTES;   // fp32 SW128 staging
  static constexpr uint32_t OFF_L = OFF_DQ + DQ_BYTES;        // 2 x BR floats
  static constexpr uint32_t OFF_DV = OFF_L + 2 * BR * 4;      // 2 x BR floats
  static constexpr uint32_t OFF_BAR = OFF_DV + 2 * BR * 4;
  static constexpr int NBAR = 32;
  static constexpr uint32_t OFF_MISC = OFF_BAR + NBAR * 8;
  static constexpr uint32_t SMEM_BYTES = OFF_MISC + 64 + 1024;  // + alignment slack
  // TMEM columns
  static constexpr uint32_t T_S = 0;
  static constexpr uint32_t T_DP = BR;
  static constexpr uint32_t T_DV = 2 * BR;
  static constexpr uint32_t T_DK = 2 * BR + D;
  static constexpr uint32_t T_DQ = 2 * BR + 2 * D;  // two buffers of 64 columns
  static_assert(T_DQ + 128 == 512, "TMEM budget");
  static_assert(SMEM_BYTES <= 232448, "smem budget");
};

// Barrier slots
enum : int {
  B_JOB0 = 0, B_JOB1 = 1, B_KV_FULL = 2, B_KV_EMPTY = 3, B_Q_FULL0 = 4, B_Q_FULL1 = 5,
  B_Q_EMPTY0 = 6, B_Q_EMPTY1 = 7, B_S_FULL = 8, B_S_EMPTY = 9, B_P_FULL0 = 10, B_P_FULL1 = 11,
  B_P_EMPTY0 = 12, B_P_EMPTY1 = 13, B_DQ_FULL0 = 14, B_DQ_FULL1 = 15, B_DQ_EMPTY0 = 16,
  B_DQ_EMPTY1 = 17, B_ACC_FULL = 18, B_ACC_EMPTY = 19, B_COUNT = 20
};

__device__ __forceinline__ void tma_store_2d(const void* tmap, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(tmap)),
               "r"(ptx::smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void tma_reduce_add_2d(const void* tmap, const void* src, int c0,
                                                  int c1) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(tmap)),
      "r"(ptx::smem_u32(src)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int D>
__global__ void __launch_bounds__(384, 1)
    dash_bwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
                    const __grid_constant__ CUtensorMap tm_dqacc, const BwdArgs args) {
  using C = BwdCfg<D>;
  constexpr int BR = C::BR, NSUB = C::NSUB, NP = C::NP;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::OFF_MISC);
  int* job_slot = reinterpret_cast<int*>(smem + C::OFF_MISC + 8);  // [2]
  float* sL = reinterpret_cast<float*>(smem + C::OFF_L);
  float* sDv = reinterpret_cast<float*>(smem + C::OFF_DV);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    for (int i = 0; i < B_COUNT; ++i) ptx::mbar_init(&bars[i], 1);
    ptx::mbar_init(&bars[B_S_EMPTY], 128);
    ptx::mbar_init(&bars[B_P_FULL0], 128);
    ptx::mbar_init(&bars[B_P_FULL1], 128);
    ptx::mbar_init(&bars[B_DQ_EMPTY0], 128);
    ptx::mbar_init(&bars[B_DQ_EMPTY1], 128);
    ptx::mbar_init(&bars[B_ACC_EMPTY], 128);
    ptx::fence_mbar_init();
    ptx::fence_async_smem();
    ptx::prefetch_tmap(&tm_q);
    ptx::prefetch_tmap(&tm_k);
    ptx::prefetch_tmap(&tm_v);
    ptx::prefetch_tmap(&tm_do);
    ptx::prefetch_tmap(&tm_dqacc);
  }
  if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  const int n_sub_tiles = (args.N / 128) * NSUB;  // tickets per head

  if (warp == 0) {
    // ============================ TMA producer ============================
    if (lane == 0) {
      uint32_t it_job = 0, kv_cnt = 0, q_cnt = 0;
      while (true) {
        ptx::mbar_wait(&bars[B_JOB0 + (it_job & 1)], (it_job >> 1) & 1);
        const int g = job_slot[it_job & 1];
        ++it_job;
        if (g >= args.total_jobs) break;
        const int bh = g / args.jobs_per_head, lj = g % args.jobs_per_head;
        const int b = bh / args.H, h = bh % args.H;
        const int t0 = args.job_begin[lj], t1 = args.job_begin[lj + 1];
        int prev_kv = -1;
        for (int t = t0; t < t1; ++t) {
          const int2 tk = args.tasks[t];
          const int kv = tk.x & 0xFFFF, q = tk.x >> 16;
          if (kv != prev_kv) {
            if (kv_cnt > 0) ptx::mbar_wait(&bars[B_KV_EMPTY], (kv_cnt - 1) & 1);
            ptx::mbar_arrive_expect_tx(&bars[B_KV_FULL], 2 * C::KV_BYTES);
#pragma unroll
            for (int blk = 0; blk < D / 64; ++blk) {
              ptx::tma_load_2d(smem + C::OFF_K + blk * C::BC * 128, &tm_k, &bars[B_KV_FULL],
                               h * D + blk * 64, b * args.N + kv * 128);
              ptx::tma_load_2d(smem + C::OFF_V + blk * C::BC * 128, &tm_v, &bars[B_KV_FULL],
                               h * D + blk * 64, b * args.N + kv * 128);
            }
            ++kv_cnt;
            prev_kv = kv;
          }
          for (int sub = 0; sub < NSUB; ++sub) {
            const int stage = q_cnt & 1;
            if (q_cnt >= 2) ptx::mbar_wait(&bars[B_Q_EMPTY0 + stage], ((q_cnt >> 1) - 1) & 1);
            uint64_t* full = &bars[B_Q_FULL0 + stage];
            ptx::mbar_arrive_expect_tx(full, 2 * C::Q_BYTES + 2 * BR * 4);
            const int row0 = q * 128 + sub * BR;
#pragma unroll
            for (int blk = 0; blk < D / 64; ++blk) {
              ptx::tma_load_2d(smem + C::OFF_Q + stage * C::Q_BYTES + blk * BR * 128, &tm_q, full,
                               h * D + blk * 64, b * args.N + row0);
              ptx::tma_load_2d(smem + C::OFF_DO + stage * C::Q_BYTES + blk * BR * 128, &tm_do,
                               full, h * D + blk * 64, b * args.N + row0);
            }
            const size_t lo = static_cast<size_t>(bh) * args.N + row0;
            ptx::bulk_load(sL + stage * BR, args.lse + lo, BR * 4, full);
            ptx::bulk_load(sDv + stage * BR, args.Dvec + lo, BR * 4, full);
            ++q_cnt;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ==============================
    if (lane == 0) {
      uint32_t it_job = 0, kv_cnt = 0, x = 0, acc_cnt = 0;
      const uint32_t sK = ptx::smem_u32(smem + C::OFF_K), sV = ptx::smem_u32(smem + C::OFF_V);
      auto sQ = [&](uint32_t st) { return ptx::smem_u32(smem + C::OFF_Q + st * C::Q_BYTES); };
      auto sdO = [&](uint32_t st) { return ptx::smem_u32(smem + C::OFF_DO + st * C::Q_BYTES); };
      auto sP = [&](uint32_t pb) { return ptx::smem_u32(smem + C::OFF_P + pb * C::P_BYTES); };
      auto sdS = [&](uint32_t pb) { return ptx::smem_u32(smem + C::OFF_DS + pb * C::P_BYTES); };
      auto issue_sdp = [&](uint32_t xx) {
        const uint32_t st = xx & 1;
        ptx::mbar_wait(&bars[B_Q_FULL0 + st], (xx >> 1) & 1);
        if (xx > 0) ptx::mbar_wait(&bars[B_S_EMPTY], (xx - 1) & 1);
        ptx::tc_fence_after();
        umma_gemm<128, BR, D, false, false>(tbase + C::T_S, sK, 128, sQ(st), BR, false);
        umma_gemm<128, BR, D, false, false>(tbase + C::T_DP, sV, 128, sdO(st), BR, false);
        ptx::mma_commit(&bars[B_S_FULL]);
      };
      while (true) {
        ptx::mbar_wait(&bars[B_JOB0 + (it_job & 1)], (it_job >> 1) & 1);
        const int g = job_slot[it_job & 1];
        ++it_job;
        if (g >= args.total_jobs) break;
        const int lj = g % args.jobs_per_head;
        const int t0 = args.job_begin[lj], t1 = args.job_begin[lj + 1];
        int ts = t0;
        while (ts < t1) {
          const int kv = args.tasks[ts].x & 0xFFFF;
          int te = ts + 1;
          while (te < t1 && (args.tasks[te].x & 0xFFFF) == kv) ++te;
          const uint32_t nsub = static_cast<uint32_t>(te - ts) * NSUB;
          ptx::mbar_wait(&bars[B_KV_FULL], kv_cnt & 1);
          ++kv_cnt;
          ptx::tc_fence_after();
          const uint32_t base = x;
          issue_sdp(base);
          for (uint32_t u = 0; u < nsub; ++u) {
            const uint32_t xx = base + u;
            if (u + 1 < nsub) issue_sdp(xx + 1);
            const uint32_t pb = xx % NP, st = xx & 1, db = xx & 1;
            ptx::mbar_wait(&bars[B_P_FULL0 + pb], (xx / NP) & 1);
            if (u == 0 && acc_cnt > 0) ptx::mbar_wait(&bars[B_ACC_EMPTY], (acc_cnt - 1) & 1);
            ptx::tc_fence_after();
            // dV += P^T dO ; dK += dS^T Q   (Alg.1 lines 25-26)
            umma_gemm<128, D, BR, false, true>(tbase + C::T_DV, sP(pb), 128, sdO(st), BR, u > 0);
            umma_gemm<128, D, BR, false, true>(tbase + C::T_DK, sdS(pb), 128, sQ(st), BR, u > 0);
            if (xx >= 2) {
              ptx::mbar_wait(&bars[B_DQ_EMPTY0 + db], ((xx >> 1) - 1) & 1);
              ptx::tc_fence_after();
            }
            // dQ_local (Alg.1 line 28)
            if constexpr (D == 128) {
              umma_gemm<128, BR, 128, true, true>(tbase + C::T_DQ + db * 64, sK, 128, sdS(pb), 128,
                                                  false);
            } else {
              umma_gemm<128, D, 128, true, true>(tbase + C::T_DQ + db * 64, sdS(pb), 128, sK, 128,
                                                 false);
            }
            ptx::mma_commit(&bars[B_DQ_FULL0 + db]);
            ptx::mma_commit(&bars[B_Q_EMPTY0 + st]);
            ptx::mma_commit(&bars[B_P_EMPTY0 + pb]);
          }
          x = base + nsub;
          ptx::mma_commit(&bars[B_KV_EMPTY]);
          ptx::mma_commit(&bars[B_ACC_FULL]);
          ++acc_cnt;
          ts = te;
        }
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ======================= softmax / dS / epilogue ======================
    const int row = (warp & 3) * 32 + lane;  // KV row within the tile = TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    uint32_t it_job = 0, x = 0, acc_cnt = 0;
    while (true) {
      ptx::mbar_wait(&bars[B_JOB0 + (it_job & 1)], (it_job >> 1) & 1);
      const int g = job_slot[it_job & 1];
      ++it_job;
      if (g >= args.total_jobs) break;
      const int bh = g / args.jobs_per_head, lj = g % args.jobs_per_head;
      const int b = bh / args.H, h = bh % args.H;
      const int t0 = args.job_begin[lj], t1 = args.job_begin[lj + 1];
      for (int t = t0; t < t1; ++t) {
        const int2 tk = args.tasks[t];
        const int kv = tk.x & 0xFFFF, q = tk.x >> 16;
        const bool diag = args.causal && (kv == q);
        for (int sub = 0; sub < NSUB; ++sub, ++x) {
          const uint32_t st = x & 1, pb = x % NP;
          ptx::mbar_wait(&bars[B_S_FULL], x & 1);
          ptx::mbar_wait(&bars[B_Q_FULL0 + st], (x >> 1) & 1);
          if (x >= NP) ptx::mbar_wait(&bars[B_P_EMPTY0 + pb], ((x / NP) - 1) & 1);
          ptx::tc_fence_after();
          uint8_t* pP = smem + C::OFF_P + pb * C::P_BYTES;
          uint8_t* pdS = smem + C::OFF_DS + pb * C::P_BYTES;
          const float* Lrow = sL + st * BR;
          const float* Drow = sDv + st * BR;
#pragma unroll 1
          for (int ch = 0; ch < BR / 64; ++ch) {
            float s[64], dp[64];
            ptx::tmem_ld32(tbase + lane_off + C::T_S + ch * 64, *reinterpret_cast<float(*)[32]>(s));
            ptx::tmem_ld32(tbase + lane_off + C::T_S + ch * 64 + 32,
                           *reinterpret_cast<float(*)[32]>(s + 32));
            ptx::tmem_ld32(tbase + lane_off + C::T_DP + ch * 64, *reinterpret_cast<float(*)[32]>(dp));
            ptx::tmem_ld32(tbase + lane_off + C::T_DP + ch * 64 + 32,
                           *reinterpret_cast<float(*)[32]>(dp + 32));
            ptx::tmem_wait_ld();
            if (ch == BR / 64 - 1) {
              ptx::tc_fence_before();
              ptx::mbar_arrive(&bars[B_S_EMPTY]);
            }
#pragma unroll
            for (int c8 = 0; c8 < 8; ++c8) {
              const int col0 = ch * 64 + c8 * 8;  // Q row within the sub-tile
              const float4 la = *reinterpret_cast<const float4*>(Lrow + col0);
              const float4 lb = *reinterpret_cast<const float4*>(Lrow + col0 + 4);
              const float4 da = *reinterpret_cast<const float4*>(Drow + col0);
              const float4 db = *reinterpret_cast<const float4*>(Drow + col0 + 4);
              const float Lv[8] = {la.x, la.y, la.z, la.w, lb.x, lb.y, lb.z, lb.w};
              const float Dv[8] = {da.x, da.y, da.z, da.w, db.x, db.y, db.z, db.w};
              float p[8], ds[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const int c = c8 * 8 + e;
                float pv = fast_exp2(fmaf(s[c], args.scale_log2, -Lv[e] * 1.4426950408889634f));
                if (diag && row > sub * BR + col0 + e) pv = 0.f;
                p[e] = pv;
                ds[e] = pv * (dp[c] - Dv[e]);
              }
              uint4 pk, dk4;
              pk.x = pack_bf16(p[0], p[1]);
              pk.y = pack_bf16(p[2], p[3]);
              pk.z = pack_bf16(p[4], p[5]);
              pk.w = pack_bf16(p[6], p[7]);
              dk4.x = pack_bf16(ds[0], ds[1]);
              dk4.y = pack_bf16(ds[2], ds[3]);
              dk4.z = pack_bf16(ds[4], ds[5]);
              dk4.w = pack_bf16(ds[6], ds[7]);
              const uint32_t off = sw128_chunk_offset(128, row, col0 >> 3);
              *reinterpret_cast<uint4*>(pP + off) = pk;
              *reinterpret_cast<uint4*>(pdS + off) = dk4;
            }
          }
          ptx::fence_async_smem();
          ptx::mbar_arrive(&bars[B_P_FULL0 + pb]);
        }
        // End of a KV segment: dK/dV epilogue (local reduction done).
        const bool seg_end = (t + 1 == t1) || ((args.tasks[t + 1].x & 0xFFFF) != kv);
        if (seg_end) {
          ptx::mbar_wait(&bars[B_ACC_FULL], acc_cnt & 1);
          ++acc_cnt;
          ptx::tc_fence_after();
          const size_t grow = (static_cast<size_t>(b) * args.N + kv * 128 + row) * args.H + h;
          __nv_bfloat16* dvp = args.dv + grow * D;
          __nv_bfloat16* dkp = args.dk + grow * D;
#pragma unroll 1
          for (int c0 = 0; c0 < D; c0 += 32) {
            float a[32], k2[32];
            ptx::tmem_ld32(tbase + lane_off + C::T_DV + c0, a);
            ptx::tmem_ld32(tbase + lane_off + C::T_DK + c0, k2);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; e += 8) {
              uint4 pv, pk;
              pv.x = pack_bf16(a[e], a[e + 1]);
              pv.y = pack_bf16(a[e + 2], a[e + 3]);
              pv.z = pack_bf16(a[e + 4], a[e + 5]);
              pv.w = pack_bf16(a[e + 6], a[e + 7]);
              pk.x = pack_bf16(k2[e] * args.scale, k2[e + 1] * args.scale);
              pk.y = pack_bf16(k2[e + 2] * args.scale, k2[e + 3] * args.scale);
              pk.z = pack_bf16(k2[e + 4] * args.scale, k2[e + 5] * args.scale);
              pk.w = pack_bf16(k2[e + 6] * args.scale, k2[e + 7] * args.scale);
              *reinterpret_cast<uint4*>(dvp + c0 + e) = pv;
              *reinterpret_cast<uint4*>(dkp + c0 + e) = pk;
            }
          }
          ptx::tc_fence_before();
          ptx::mbar_arrive(&bars[B_ACC_EMPTY]);
        }
      }
    }
  } else if (warp >= 8) {
    // =============== dQ drain + ordered reduction + job claim ===============
    const int tl = (warp & 3) * 32 + lane;  // TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const bool leader = (warp == 8 && lane == 0);
    uint8_t* stg = smem + C::OFF_DQ;
    uint32_t it_job = 0, x = 0;
    if (leader) {
      job_slot[0] = atomicAdd(args.job_counter, 1);
      ptx::mbar_arrive(&bars[B_JOB0]);
    }
    while (true) {
      ptx::mbar_wait(&bars[B_JOB0 + (it_job & 1)], (it_job >> 1) & 1);
      const int g = job_slot[it_job & 1];
      ++it_job;
      if (g >= args.total_jobs) break;
      const int bh = g / args.jobs_per_head, lj = g % args.jobs_per_head;
      const int t0 = args.job_begin[lj], t1 = args.job_begin[lj + 1];
      for (int t = t0; t < t1; ++t) {
        const int2 tk = args.tasks[t];
        const int q = tk.x >> 16, rank = tk.y;
        for (int sub = 0; sub < NSUB; ++sub, ++x) {
          const uint32_t db = x & 1;
          ptx::mbar_wait(&bars[B_DQ_FULL0 + db], (x >> 1) & 1);
          ptx::tc_fence_after();
          float v[64];
          ptx::tmem_ld32(tbase + lane_off + C::T_DQ + db * 64, *reinterpret_cast<float(*)[32]>(v));
          ptx::tmem_ld32(tbase + lane_off + C::T_DQ + db * 64 + 32,
                         *reinterpret_cast<float(*)[32]>(v + 32));
          ptx::tmem_wait_ld();
          ptx::tc_fence_before();
          ptx::mbar_arrive(&bars[B_DQ_EMPTY0 + db]);
          // Stage the fp32 partial as SW128 boxes of 32 columns x BR rows.
          if constexpr (D == 128) {
            // lane tl = d index, v[c] = Q row c
            const int blk = tl >> 5, chunk = (tl & 31) >> 2, w = tl & 3;
#pragma unroll
            for (int c = 0; c < BR; ++c) {
              const uint32_t off = blk * BR * 128 + c * 128 + ((chunk ^ (c & 7)) << 4) + w * 4;
              *reinterpret_cast<float*>(stg + off) = v[c];
            }
          } else {
            // lane tl = Q row, v[c] = d column c
#pragma unroll
            for (int cc = 0; cc < 16; ++cc) {
              const int blk = cc >> 3, chunk = cc & 7;
              const uint32_t off = blk * BR * 128 + tl * 128 + ((chunk ^ (tl & 7)) << 4);
              *reinterpret_cast<float4*>(stg + off) =
                  make_float4(v[cc * 4], v[cc * 4 + 1], v[cc * 4 + 2], v[cc * 4 + 3]);
            }
          }
          ptx::fence_async_smem();
          ptx::bar_sync(1, 128);
          if (leader) {
            int* ticket = args.tickets + static_cast<size_t>(bh) * n_sub_tiles + q * NSUB + sub;
            const int grow = bh * args.N + q * 128 + sub * BR;  // row in dQacc [B*H*N, D]
            const bool det = args.deterministic != 0;
            if (det) {
              // Wait until the global order grants this block its turn (Alg.1 line 33).
              if (ptx::ld_acquire(ticket) != rank) {
                const uint64_t t_start = ptx::globaltimer();
                while (ptx::ld_acquire(ticket) != rank) {
                  __nanosleep(64);
                  if (ptx::globaltimer() - t_start > 20000000000ull) {  // 20 s bound
                    atomicExch(args.error_flag, 1);
                    break;
                  }
                }
              }
              ptx::fence_async_global();
            }
            // Add dQ_local to dQ (Alg.1 line 34); rank 0 stores (no zero-fill needed).
#pragma unroll
            for (int blk = 0; blk < D / 32; ++blk) {
              if (det && rank == 0) {
                tma_store_2d(&tm_dqacc, stg + blk * BR * 128, blk * 32, grow);
              } else {
                tma_reduce_add_2d(&tm_dqacc, stg + blk * BR * 128, blk * 32, grow);
              }
            }
            ptx::bulk_commit();
            ptx::bulk_wait_all();
            if (det) {
              ptx::fence_async_global();
              ptx::st_release(ticket, rank + 1);  // advance the global order (Alg.1 line 35)
            }
          }
          ptx::bar_sync(2, 128);
        }
      }
      // All of this job's ordered adds are released: claim the next job (AMB-7).
      if (leader) {
        job_slot[it_job & 1] = atomicAdd(args.job_counter, 1);
        ptx::mbar_arrive(&bars[B_JOB0 + (it_job & 1)]);
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tbase);
  }
}

// ----------------------------------------------------------------------------
// K1: D = rowsum(dO o O) (Alg.1 line 1; D in R^N per AMB-2), fp32 in a
// fixed order; also resets tickets / job counter and (atomic variant only)
// zero-fills the dQ accumulator.
template <int D>
__global__ void dash_preprocess_kernel(const __nv_bfloat16* __restrict__ o,
                                       const __nv_bfloat16* __restrict__ dout,
                                       float* __restrict__ Dvec, int B, int N, int H,
                                       int* __restrict__ zero_i32, int n_zero_i32,
                                       float4* __restrict__ zero_f32, size_t n_zero_f4,
                                       int* __restrict__ job_counter) {
  constexpr int T = D / 8;  // threads per row, 16 B each
  const size_t gtid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const size_t rows = static_cast<size_t>(B) * N * H;
  const size_t row = gtid / T;
  const int part = static_cast<int>(gtid % T);
  if (row < rows) {
    const uint4 a = *reinterpret_cast<const uint4*>(o + row * D + part * 8);
    const uint4 c = *reinterpret_cast<const uint4*>(dout + row * D + part * 8);
    const __nv_bfloat162* pa = reinterpret_cast<const __nv_bfloat162*>(&a);
    const __nv_bfloat162* pc = reinterpret_cast<const __nv_bfloat162*>(&c);
    float acc = 0.f;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 fa = __bfloat1622float2(pa[e]);
      const float2 fc = __bfloat1622float2(pc[e]);
      acc = fmaf(fa.x, fc.x, acc);
      acc = fmaf(fa.y, fc.y, acc);
    }
#pragma unroll
    for (int m = T / 2; m >= 1; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
    if (part == 0) {
      const int h = static_cast<int>(row % H);
      const size_t bn = row / H;
      const int n = static_cast<int>(bn % N);
      const int b = static_cast<int>(bn / N);
      Dvec[(static_cast<size_t>(b) * H + h) * N + n] = acc;
    }
  }
  const size_t nthreads = static_cast<size_t>(gridDim.x) * blockDim.x;
  if (gtid == 0) *job_counter = 0;
  for (size_t i = gtid; i < static_cast<size_t>(n_zero_i32); i += nthreads) zero_i32[i] = 0;
  for (size_t i = gtid; i < n_zero_f4; i += nthreads) zero_f32[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// K4: dQ = bf16(scale * dQacc), [B,H,N,d] fp32 -> [B,N,H,d] bf16.
template <int D>
__global__ void dash_dq_convert_kernel(const float* __restrict__ acc, __nv_bfloat16* __restrict__ dq,
                                       int B, int N, int H, float scale) {
  constexpr int T = D / 8;
  const size_t total = static_cast<size_t>(B) * H * N * T;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int part = static_cast<int>(i % T);
    const size_t r = i / T;  // (b*H + h)*N + n
    const int n = static_cast<int>(r % N);
    const size_t bh = r / N;
    const int h = static_cast<int>(bh % H);
    const int b = static_cast<int>(bh / H);
    const float4 x0 = *reinterpret_cast<const float4*>(acc + r * D + part * 8);
    const float4 x1 = *reinterpret_cast<const float4*>(acc + r * D + part * 8 + 4);
    uint4 out;
    out.x = pack_bf16(x0.x * scale, x0.y * scale);
    out.y = pack_bf16(x0.z * scale, x0.w * scale);
    out.z = pack_bf16(x1.x * scale, x1.y * scale);
    out.w = pack_bf16(x1.z * scale, x1.w * scale);
    *reinterpret_cast<uint4*>(dq + ((static_cast<size_t>(b) * N + n) * H + h) * D + part * 8) = out;
  }
}

}  // namespace dash
