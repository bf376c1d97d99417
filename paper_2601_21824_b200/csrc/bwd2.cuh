// DASH deterministic attention backward, d = 128 -- CTA-pair kernel
// (cta_group::2) with 256-row tiles.  Algorithm 1 with
// B_r = B_c = 256 (the tile size is a free parameter of the schedule model,
// AMB-11 / AMB-31): a job's KV tile of 256 rows is owned by a cluster of two
// CTAs on the two SMs of a TPC, CTA c holding KV rows [128c, 128c + 128) of
// the tile -- its dK / dV accumulate in its own TMEM -- and every Q tile of
// 256 rows is walked as four sub-tiles of BR = 64 rows.  Per sub-tile the
// leader CTA issues five pair MMAs for both SMs:
//
//   S^T  = K Q^T        M = 256 (KV rows), N = 64, K = d     SS, B split by N
//   dP^T = V dO^T       "                                    SS
//   dV  += P^T dO       M = 256, N = d = 128, K = 64         TS (P^T in TMEM)
//   dK  += dS^T Q       "                                    TS (dS^T in TMEM)
//   dQ_part^T = K^T dS^T  M = d = 128 (CTA c: d half c), N = 64, K = 256 KV rows
//
// so one dQ partial covers the whole 256-row KV tile: per SM, half the bytes
// of the fp32 ordered reduction of the single-CTA kernel (bwd.cuh), where the
// partial of each 128-row KV tile travels to L2 on its own.  CTA c then adds
// its d-half of the partial into dQacc under its own ticket (one ticket chain
// per (Q sub-tile, d half), both in the schedule's rank order -- Alg. 1 lines
// 30-36).
//
// Operand placement (identical shared-memory offsets in both CTAs -- a pair
// MMA reads the same descriptor address in each):
//   K, V     own 128 rows x 128, SW128 (A of S^T / dP^T, K-major)
//   KB       [256 KV rows][64] = block c (d cols 64c..64c+63) of both CTAs' K
//            tiles (A of dQ^T, MN-major: M = d half c, K = KV rows)
//   QS, dOS  [32 rows][128]: Q / dO rows 32c..32c+31 of the sub-tile (B of
//            S^T / dP^T, K-major, N half c)
//   QK, dOK  [64 rows][64]: block c of the sub-tile's Q / dO (B of dK / dV,
//            MN-major, N half c)
//   DS       [256 KV rows][32] bf16 SW64: dS^T columns 32c..32c+31 for both
//            CTAs' KV rows (B of dQ^T, MN-major, N half c); the softmax of CTA
//            c' writes its KV rows' column half h into CTA h's buffer
//            (distributed shared memory when h != c').
// Barriers the MMA issuer waits on live in the leader CTA (rank 0); the peer
// arrives on them remotely (release.cluster) and its TMA loads complete their
// bytes there.  MMA completions are multicast to both CTAs.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include <type_traits>

#include "bwd.cuh"

namespace dash {

template <int NQS_ = 2, int NQK_ = 2, int NDS_ = 2>
struct PairCfgT {
  static constexpr int D = 128;
  static constexpr int NTHREADS = 512;
  static constexpr int BC = 128;        // KV rows per CTA (TMEM lanes)
  static constexpr int TILE = 256;      // schedule tile (KV and Q)
  static constexpr int BR = 64;         // Q sub-tile rows
  static constexpr int NSUB = TILE / BR;
  // Two operand rings per Q sub-tile: the QS ring (Q / dO row halves and L, D:
  // read by S^T / dP^T and the softmax, free early) and the QK ring (Q / dO
  // column blocks: read by dV / dK, free late).  Splitting them lets the
  // early half be prefetched NQS sub-tiles ahead within the smem budget.
  static constexpr int NQS = NQS_;
  static constexpr int NQK = NQK_;
  static constexpr int NDS = NDS_;      // dS^T smem buffers (B of dQ^T)
  static constexpr int NLD = 3;         // L / D ring (512 B per slot): loaded far ahead
  static constexpr int NSMX = 2;        // softmax warpgroups (column halves = N halves)
  static constexpr int SMX_COLS = BR / NSMX;  // 32
  static constexpr uint32_t KV_BYTES = BC * D * 2;       // 32 KB
  static constexpr uint32_t KB_BYTES = 2 * BC * 64 * 2;  // 32 KB
  static constexpr uint32_t QS_BYTES = 32 * D * 2;       // 8 KB
  static constexpr uint32_t QK_BYTES = BR * 64 * 2;      // 8 KB
  static constexpr uint32_t SLOT_BYTES = 2 * QS_BYTES;   // one slot of either ring: Q + dO
  static constexpr uint32_t DS_BYTES = 2 * BC * 32 * 2;  // 16 KB
  static constexpr uint32_t DQ_BYTES = BR * 64 * 4;      // 16 KB: [64 Q rows][64 d] fp32
  static constexpr uint32_t OFF_K = 0;
  static constexpr uint32_t OFF_V = OFF_K + KV_BYTES;
  static constexpr uint32_t OFF_KB = OFF_V + KV_BYTES;
  static constexpr uint32_t OFF_QSR = OFF_KB + KB_BYTES;            // NQS slots {QS, dOS}
  static constexpr uint32_t OFF_QKR = OFF_QSR + NQS * SLOT_BYTES;   // NQK slots {QK, dOK}
  static constexpr uint32_t OFF_DS = OFF_QKR + NQK * SLOT_BYTES;
  // outbox: this CTA's KV rows of the peer's column half of dS^T, moved into the
  // peer's DS buffer by one bulk copy (async proxy) per sub-tile
  static constexpr uint32_t OUT_BYTES = BC * 32 * 2;  // 8 KB
  static constexpr uint32_t OFF_OUT = OFF_DS + NDS * DS_BYTES;
  static constexpr uint32_t OFF_DQ = OFF_OUT + NDS * OUT_BYTES;
  static constexpr uint32_t OFF_L = OFF_DQ + DQ_BYTES;              // NLD x BR floats
  static constexpr uint32_t OFF_DV = OFF_L + NLD * BR * 4;          // NLD x BR floats
  static constexpr uint32_t OFF_BAR = OFF_DV + NLD * BR * 4;
  static constexpr int NBAR = 56;
  static constexpr uint32_t OFF_MISC = OFF_BAR + NBAR * 8;
  static constexpr uint32_t BODY_BYTES = OFF_MISC + 64;
  static constexpr uint32_t SLACK = (BODY_BYTES + 1024 <= 232448) ? 1024 : (232448 - BODY_BYTES);
  static constexpr uint32_t SMEM_BYTES = BODY_BYTES + SLACK;
  // TMEM columns (per CTA)
  static constexpr uint32_t T_S = 0;
  static constexpr uint32_t T_DP = 64;
  static constexpr uint32_t T_DV = 128;
  static constexpr uint32_t T_DK = 256;
  static constexpr uint32_t T_DQ = 384;   // 2 buffers x 32 columns (M = 64 per SM layout)
  static constexpr uint32_t T_PT = 448;   // 32 columns packed bf16 P^T
  static constexpr uint32_t T_DST = 480;  // 32 columns packed bf16 dS^T
  static_assert(SMEM_BYTES <= 232448, "smem budget");
  static_assert(NQS <= 3 && NQK <= 2 && NDS <= 2, "barrier slots");
  static_assert(OFF_QSR % 1024 == 0 && OFF_DS % 1024 == 0 && OFF_DQ % 1024 == 0, "alignment");
};
using PairCfg = PairCfgT<>;

// Barrier slots.  (L) = lives in the leader and is waited on there only; (B) =
// one instance per CTA, arrived on by multicast commits or locally.
enum : int {
  P_JOB0 = 0, P_JOB1 = 1,        // (B) job slot filled (1; written by the leader)
  P_KV_FULL = 2,                 // (L) K / V of both CTAs loaded (1 + tx)
  P_KV_EMPTY = 3,                // (B) every MMA of the KV segment complete: KB free (commit)
  P_S_FULL = 4,                  // (B) S^T / dP^T in TMEM (commit)
  P_S_EMPTY = 5,                 // (L) both softmaxes read S^T / dP^T (16 warps)
  P_P_FULL = 6,                  // (L) both wrote P^T / dS^T to TMEM, own dS^T half to smem (16)
  P_PT_EMPTY = 7,                // (B) P^T consumed by dV (commit)
  P_DST_EMPTY = 8,               // (B) dS^T (TMEM) consumed by dK (commit)
  P_DQ_FULL0 = 9,                // (B) + buf: dQ partial in TMEM (commit)
  P_DQ_EMPTY0 = 11,              // (L) + buf: both drains read it (8 warps)
  P_ACC_FULL = 13,               // (B) dK/dV complete (commit)
  P_ACC_EMPTY = 14,              // (L) both epilogues read dK/dV (16 warps)
  P_JOB_DONE = 15,               // (L) every reducer agent of both CTAs released the job (4)
  P_MMA_DRAIN = 16,              // (L) exit: all MMAs complete (commit)
  P_QS_FULL0 = 17,               // (L) + slot (<= 3): QS / dOS of both CTAs loaded (1 + tx)
  P_QK_FULL0 = 20,               // (L) + slot (<= 2): QK / dOK of both CTAs loaded (1 + tx)
  P_LD_FULL0 = 22,               // (B) + slot (NLD = 3): this CTA's L/D loaded (1 + tx)
  P_QS_EMPTY0 = 25,              // (B) + slot: consumed by S^T / dP^T (commit)
  P_QK_EMPTY0 = 28,              // (B) + slot: consumed by dV / dK (commit)
  P_LD_EMPTY0 = 30,              // (B) + slot: L/D read by this CTA's softmax (256 threads)
  P_DS_EMPTY0 = 33,              // (B) + buf: dS^T smem consumed by dQ (commit)
  P_PF0 = 35,                    // (L) + (t-1)%2: producer's claim decision (1)
  P_SLOT_FREE0 = 37,             // (L) + j%2: all 32 warps of the pair read job j's slot (32)
  P_AGF0 = 39,                   // (B) + part * NAG + agent: staging part written (64)
  P_STG_EMPTY0 = 43,             // (B) + part: staging part read by the bulk engine (1)
  P_DSR0 = 45,                   // (B) + buf: this CTA's DS buffer is complete -- its own-half
                                 // softmax warps stored their rows (4) and the partner's 8 KB
                                 // landed (tx); in the leader also the peer's relay (+1): the
                                 // dQ issuer waits on it
  P_KB_FULL = 47,                // (L) KB of both CTAs loaded (1 + tx)
  P_KV_FREE = 48,                // (B) K / V read by the segment's last S^T / dP^T (commit):
                                 // the next segment's K / V load starts while its last
                                 // sub-tile's softmax, dK / dV and dQ still run
  P_COUNT = 49
};

template <int NQS_, int NQK_, int NDS_>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 1)
    dash_bwd_pair_kernel(const __grid_constant__ CUtensorMap tm_q32,
                         const __grid_constant__ CUtensorMap tm_q64,
                         const __grid_constant__ CUtensorMap tm_k,
                         const __grid_constant__ CUtensorMap tm_v,
                         const __grid_constant__ CUtensorMap tm_do32,
                         const __grid_constant__ CUtensorMap tm_do64,
                         const __grid_constant__ CUtensorMap tm_dqacc,
                         const __grid_constant__ CUtensorMap tm_dk,
                         const __grid_constant__ CUtensorMap tm_dv, const BwdArgs args) {
  using C = PairCfgT<NQS_, NQK_, NDS_>;
  constexpr int D = C::D, BR = C::BR, NSUB = C::NSUB, NQS = C::NQS, NQK = C::NQK;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t pad = (1024 - (ptx::smem_u32(smem_raw) & 1023)) & 1023;
  if (pad > C::SLACK) __trap();
  uint8_t* smem = smem_raw + pad;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::OFF_MISC);
  int* job_slot = reinterpret_cast<int*>(smem + C::OFF_MISC + 8);  // [2]
  volatile int* claim_mode = reinterpret_cast<volatile int*>(smem + C::OFF_MISC + 16);  // [2]
  float* sL = reinterpret_cast<float*>(smem + C::OFF_L);
  float* sDv = reinterpret_cast<float*>(smem + C::OFF_DV);

  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const uint32_t cta = ptx::cluster_ctarank();  // c: KV rows [128c, 128c + 128) of the tile
  const bool leader = cta == 0;
  // shared::cluster address of barrier slot i in the leader CTA
  auto lbar = [&](int i) { return ptx::mapa(ptx::smem_u32(&bars[i]), 0); };
  auto slot_read = [&](uint32_t j) { ptx::mbar_arrive_remote(lbar(P_SLOT_FREE0 + (j & 1))); };

  if (tid == 0) {
    for (int i = 0; i < P_COUNT; ++i) ptx::mbar_init(&bars[i], 1);
    ptx::mbar_init(&bars[P_S_EMPTY], 16);
    ptx::mbar_init(&bars[P_P_FULL], 16);
    ptx::mbar_init(&bars[P_DQ_EMPTY0], 8);
    ptx::mbar_init(&bars[P_DQ_EMPTY0 + 1], 8);
    ptx::mbar_init(&bars[P_ACC_EMPTY], 16);
    ptx::mbar_init(&bars[P_JOB_DONE], 2 * NAG);
    ptx::mbar_init(&bars[P_SLOT_FREE0], 32);
    ptx::mbar_init(&bars[P_SLOT_FREE0 + 1], 32);
    for (int i = 0; i < 2 * NAG; ++i) ptx::mbar_init(&bars[P_AGF0 + i], 64);
    for (int i = 0; i < C::NLD; ++i) ptx::mbar_init(&bars[P_LD_EMPTY0 + i], 256);
    for (int i = 0; i < 2; ++i) ptx::mbar_init(&bars[P_DSR0 + i], leader ? 5 : 4);

    ptx::fence_mbar_init();
    ptx::fence_async_smem();
    ptx::prefetch_tmap(&tm_q32);
    ptx::prefetch_tmap(&tm_q64);
    ptx::prefetch_tmap(&tm_k);
    ptx::prefetch_tmap(&tm_v);
    ptx::prefetch_tmap(&tm_do32);
    ptx::prefetch_tmap(&tm_do64);
    ptx::prefetch_tmap(&tm_dqacc);
    ptx::prefetch_tmap(&tm_dk);
    ptx::prefetch_tmap(&tm_dv);
  }
  if (warp == 1) ptx::tmem_alloc2<512>(tmem_slot);
  ptx::tc_fence_before();
  ptx::cluster_sync();  // barriers of both CTAs initialised, TMEM allocated
  ptx::tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  // The prologue above overlaps the preprocess kernel's tail (programmatic
  // dependent launch); D, lse2, tickets and the job counter are read only now.
  ptx::griddep_launch();
  ptx::griddep_wait();
  const int n_units = args.N / BR;  // Q sub-tiles per head

  if (warp == 0) {
    // ============================ TMA producer (both CTAs) ============================
    uint32_t it_job = 0, kv_cnt = 0, q_cnt = 0;
    const uint32_t kv_full = lbar(P_KV_FULL);
    while (true) {
      ptx::mbar_wait_cluster_u(&bars[P_JOB0 + (it_job & 1)], (it_job >> 1) & 1);
      const int g = __shfl_sync(0xffffffffu, job_slot[it_job & 1], 0);
      if (lane == 0) slot_read(it_job);
      ++it_job;
      if (g >= args.total_jobs || __shfl_sync(0xffffffffu, ptx::aborted(), 0)) break;
      const JobView jv = decode_job(args, g);
      // QS / L / D of sub-tile x + 1 are issued before QK of sub-tile x (within a
      // KV segment): their slots free in that order (S^T / dP^T of x - 1 complete
      // before dK of x - 2), so neither ring waits behind the other.
      uint32_t qs_cnt = q_cnt;  // next sub-tile whose QS part is to be issued
      auto load_qs = [&](const TaskView& tv, int sub) {
        const int row0 = tv.b * args.N + tv.q * C::TILE + sub * BR;
        const int qs = qs_cnt % NQS, ld = qs_cnt % C::NLD;
        if (lane == 0) DASH_TRACE_MARK(26, qs_cnt);
        if (qs_cnt >= static_cast<uint32_t>(C::NLD))
          ptx::mbar_wait_u(&bars[P_LD_EMPTY0 + ld], ((qs_cnt / C::NLD) - 1) & 1);
        if (lane == 0) DASH_TRACE_MARK(24, qs_cnt);
        uint64_t* ldf = &bars[P_LD_FULL0 + ld];
        ptx::mbar_arrive_expect_tx_e(ldf, 2 * BR * 4);
        const size_t lo = static_cast<size_t>(tv.bh) * args.N + tv.q * C::TILE + sub * BR;
        ptx::bulk_load_e(sL + ld * BR, args.lse2 + lo, BR * 4, ldf);
        ptx::bulk_load_e(sDv + ld * BR, args.Dvec + lo, BR * 4, ldf);
        if (lane == 0) DASH_TRACE_MARK(27, qs_cnt);
        if (qs_cnt >= static_cast<uint32_t>(NQS))
          ptx::mbar_wait_u(&bars[P_QS_EMPTY0 + qs], ((qs_cnt / NQS) - 1) & 1);
        if (lane == 0) DASH_TRACE_MARK(10, qs_cnt);
        const uint32_t qsfull = lbar(P_QS_FULL0 + qs);
        if (leader && lane == 0) ptx::mbar_arrive_expect_tx_local(&bars[P_QS_FULL0 + qs], 2 * C::SLOT_BYTES);
        __syncwarp();
        uint8_t* sqs = smem + C::OFF_QSR + qs * C::SLOT_BYTES;
#pragma unroll
        for (int blk = 0; blk < 2; ++blk) {
          ptx::tma_load_2d_pair_e(sqs + blk * 32 * 128, &tm_q32, qsfull, tv.h * D + blk * 64,
                                  row0 + 32 * cta);
          ptx::tma_load_2d_pair_e(sqs + C::QS_BYTES + blk * 32 * 128, &tm_do32, qsfull,
                                  tv.h * D + blk * 64, row0 + 32 * cta);
        }
        ++qs_cnt;
      };
      auto load_qk = [&](const TaskView& tv, int sub) {
        const int row0 = tv.b * args.N + tv.q * C::TILE + sub * BR;
        const int qk = q_cnt % NQK;
        if (q_cnt >= static_cast<uint32_t>(NQK))
          ptx::mbar_wait_u(&bars[P_QK_EMPTY0 + qk], ((q_cnt / NQK) - 1) & 1);
        if (lane == 0) DASH_TRACE_MARK(23, q_cnt);
        const uint32_t qkfull = lbar(P_QK_FULL0 + qk);
        if (leader && lane == 0) ptx::mbar_arrive_expect_tx_local(&bars[P_QK_FULL0 + qk], 2 * C::SLOT_BYTES);
        __syncwarp();
        uint8_t* sqk = smem + C::OFF_QKR + qk * C::SLOT_BYTES;
        ptx::tma_load_2d_pair_e(sqk, &tm_q64, qkfull, tv.h * D + cta * 64, row0);
        ptx::tma_load_2d_pair_e(sqk + C::QK_BYTES, &tm_do64, qkfull, tv.h * D + cta * 64, row0);
        if (lane == 0) DASH_TRACE_MARK(25, q_cnt);
        ++q_cnt;
      };
      int ts = jv.t0;
      while (ts < jv.t1 && !ptx::aborted()) {
        const int te = args.seg_end[ts];  // one load, not a chain of L2 round trips
        const TaskView tv0 = decode_task(args, jv, args.tasks[ts]);
        // K / V of this KV segment: free once the previous segment's last
        // S^T / dP^T completed (KV_FREE) -- before its last softmax / dK / dV / dQ
        if (kv_cnt > 0) ptx::mbar_wait_u(&bars[P_KV_FREE], (kv_cnt - 1) & 1);
        if (lane == 0) DASH_TRACE_MARK(20, q_cnt);
        if (ptx::aborted()) break;
        if (leader && lane == 0)
          ptx::mbar_arrive_expect_tx_local(&bars[P_KV_FULL], 2 * (2 * C::KV_BYTES));
        __syncwarp();
        const int r_own = tv0.b * args.N + tv0.kv * C::TILE + C::BC * cta;
        const int r_t0 = tv0.b * args.N + tv0.kv * C::TILE;
#pragma unroll
        for (int blk = 0; blk < 2; ++blk) {
          ptx::tma_load_2d_pair_e(smem + C::OFF_K + blk * C::BC * 128, &tm_k, kv_full,
                                  tv0.h * D + blk * 64, r_own);
          ptx::tma_load_2d_pair_e(smem + C::OFF_V + blk * C::BC * 128, &tm_v, kv_full,
                                  tv0.h * D + blk * 64, r_own);
        }
        ++kv_cnt;
        load_qs(tv0, 0);
        // KB (A of dQ^T): free once every MMA of the previous segment completed
        if (kv_cnt > 1) ptx::mbar_wait_u(&bars[P_KV_EMPTY], (kv_cnt - 2) & 1);
        if (leader && lane == 0)
          ptx::mbar_arrive_expect_tx_local(&bars[P_KB_FULL], 2 * C::KB_BYTES);
        __syncwarp();
#pragma unroll
        for (int blk = 0; blk < 2; ++blk) {
          // KB rows [128 blk, +128) = block `cta` of the KV rows of CTA blk
          ptx::tma_load_2d_pair_e(smem + C::OFF_KB + blk * C::BC * 128, &tm_k, lbar(P_KB_FULL),
                                  tv0.h * D + static_cast<int>(cta) * 64, r_t0 + blk * C::BC);
        }
        for (int t = ts; t < te; ++t) {
          const TaskView tv = decode_task(args, jv, args.tasks[t]);
          for (int sub = 0; sub < NSUB; ++sub) {
            if (sub + 1 < NSUB) {
              load_qs(tv, sub + 1);
            } else if (t + 1 < te) {
              load_qs(decode_task(args, jv, args.tasks[t + 1]), 0);
            }
            load_qk(tv, sub);
          }
        }
        ts = te;
      }
      // Claim of the next job (leader only) -- as in bwd.cuh: early claim
      // (prefetch) once every load of g is issued, else reducer agent 0
      // claims after the last release.
      if (leader) {
        if (lane == 0) {
          DASH_TRACE_MARK(28, q_cnt);
          int mode = 2;
          if (it_job >= 2) ptx::mbar_wait_cluster(&bars[P_SLOT_FREE0 + (it_job & 1)], ((it_job - 2) >> 1) & 1);
          DASH_TRACE_MARK(29, q_cnt);
          int next = -1;
          if (ptx::aborted()) {
            next = args.total_jobs;
            mode = 1;
          } else if (args.prefetch && !args.cyclic) {
            next = atomicAdd(args.job_counter, 1);
            mode = 1;
          } else if (args.prefetch) {
            // cyclic schedule: early claim only outside the current head (one
            // atomicAdd once the counter is seen beyond it; see bwd.cuh)
            const int peek = ptx::ld_relaxed(args.job_counter);
            if (peek / args.jobs_per_head != g / args.jobs_per_head) {
              next = atomicAdd(args.job_counter, 1);
              mode = 1;
            }
          }
          DASH_TRACE_MARK(30, q_cnt);
          claim_mode[(it_job - 1) & 1] = mode;
          ptx::mbar_arrive(&bars[P_PF0 + ((it_job - 1) & 1)]);
          if (mode == 1) {
            // publish job it_job to both CTAs
            const uint32_t off = ptx::smem_u32(&job_slot[it_job & 1]);
            job_slot[it_job & 1] = next;
            ptx::st_cluster_u32(ptx::mapa(off, 1), static_cast<uint32_t>(next));
            ptx::mbar_arrive(&bars[P_JOB0 + (it_job & 1)]);
            ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&bars[P_JOB0 + (it_job & 1)]), 1));
          }
        }
        __syncwarp();
      }
    }
    // Exit (abort path): let in-flight TMA writes land before the CTA retires.
    if (ptx::aborted()) {
      const long long t0 = clock64();
      while (clock64() - t0 < (1ll << 20)) {
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer (leader) ==============================
    uint32_t it_job = 0, kv_cnt = 0, x = 0, acc_cnt = 0;
    const uint32_t s0 = ptx::smem_u32(smem);
    const uint64_t dK_k = tile_desc<false>(s0 + C::OFF_K, 128);  // A of S^T
    const uint64_t dV_k = tile_desc<false>(s0 + C::OFF_V, 128);  // A of dP^T
    const uint64_t dKB_mn = ptx::sdesc_sw128(s0 + C::OFF_KB, 256 * 128, 1024);  // A of dQ^T
    const uint64_t dQS = tile_desc<false>(s0 + C::OFF_QSR, 32);
    const uint64_t dDOS = tile_desc<false>(s0 + C::OFF_QSR + C::QS_BYTES, 32);
    const uint64_t dQK = ptx::sdesc_sw128(s0 + C::OFF_QKR, BR * 128, 1024);
    const uint64_t dDOK = ptx::sdesc_sw128(s0 + C::OFF_QKR + C::QK_BYTES, BR * 128, 1024);
    const uint64_t dDS = ptx::sdesc_sw64(s0 + C::OFF_DS, 2 * C::BC * 64, 512);
    constexpr uint32_t ST_STEP = C::SLOT_BYTES / 16, DS_STEP = C::DS_BYTES / 16;
    constexpr uint32_t ID_S = ptx::idesc_bf16(256, BR, 0, 0);     // S^T, dP^T
    constexpr uint32_t ID_KV = ptx::idesc_bf16(256, D, 0, 1);     // dV, dK (TS, B MN-major)
    constexpr uint32_t ID_Q = ptx::idesc_bf16(128, BR, 1, 1);     // dQ^T (A, B MN-major)
    auto issue_sdp = [&](uint32_t xx, bool seg_last) {
      const uint32_t st = xx % NQS;
      ptx::mbar_wait_u(&bars[P_QS_FULL0 + st], (xx / NQS) & 1);
      if (xx > 0) ptx::mbar_wait_u(&bars[P_S_EMPTY], (xx - 1) & 1);
      ptx::tc_fence_after();
      if (lane == 0) DASH_TRACE_MARK(0, xx);
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk)
        ptx::mma2_bf16_e(tbase + C::T_S, dK_k + kstep<false>(kk, 128),
                         dQS + st * ST_STEP + kstep<false>(kk, 32), ID_S, kk > 0);
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk)
        ptx::mma2_bf16_e(tbase + C::T_DP, dV_k + kstep<false>(kk, 128),
                         dDOS + st * ST_STEP + kstep<false>(kk, 32), ID_S, kk > 0);
      ptx::mma2_commit_mc_e(&bars[P_S_FULL]);
      ptx::mma2_commit_mc_e(&bars[P_QS_EMPTY0 + st]);
      if (seg_last) ptx::mma2_commit_mc_e(&bars[P_KV_FREE]);  // K / V no longer read
    };
    bool kb_ready = false;  // KB of the current segment seen loaded
    // dQ_local^T = K^T dS^T over the 256 KV rows of the pair (Alg.1 line 28):
    // both DS buffers complete (P_DSR), the TMEM buffer drained (P_DQ_EMPTY)
    auto issue_dq = [&](uint32_t xx) {
      const uint32_t sb = xx % C::NDS, qb = xx & 1;
      if (!kb_ready) {
        ptx::mbar_wait_u(&bars[P_KB_FULL], (kv_cnt - 1) & 1);
        kb_ready = true;
      }
      if (xx >= 2) ptx::mbar_wait_u(&bars[P_DQ_EMPTY0 + qb], ((xx >> 1) - 1) & 1);
      ptx::mbar_wait_u(&bars[P_DSR0 + sb], (xx / C::NDS) & 1);
      ptx::tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < C::TILE / 16; ++kk)
        ptx::mma2_bf16_e(tbase + C::T_DQ + qb * 32, dKB_mn + kk * (2048 / 16),
                         dDS + sb * DS_STEP + kk * (1024 / 16), ID_Q, kk > 0);
      if (lane == 0) DASH_TRACE_MARK(2, xx);
      ptx::mma2_commit_mc_e(&bars[P_DQ_FULL0 + qb]);
      ptx::mma2_commit_mc_e(&bars[P_DS_EMPTY0 + sb]);
    };
    while (true) {
      ptx::mbar_wait_cluster_u(&bars[P_JOB0 + (it_job & 1)], (it_job >> 1) & 1);
      const int g = __shfl_sync(0xffffffffu, job_slot[it_job & 1], 0);
      if (lane == 0) slot_read(it_job);
      ++it_job;
      if (g >= args.total_jobs || __shfl_sync(0xffffffffu, ptx::aborted(), 0)) break;
      if (!leader) {
        // the peer's warp 1 relays "my DS buffer is complete" (local P_DSR) to
        // the leader's dQ issuer (the leader's P_DSR)
        const JobView pj = decode_job(args, g);
        const uint32_t nsub_job = static_cast<uint32_t>(pj.t1 - pj.t0) * NSUB;
        for (uint32_t u = 0; u < nsub_job; ++u, ++x) {
          const uint32_t sb = x % C::NDS;
          ptx::mbar_wait_u(&bars[P_DSR0 + sb], (x / C::NDS) & 1);
          if (lane == 0) ptx::mbar_arrive_remote(lbar(P_DSR0 + sb));
          __syncwarp();
        }
        continue;
      }
      const JobView jv = decode_job(args, g);
      const int t1 = __shfl_sync(0xffffffffu, jv.t1, 0);
      int ts = __shfl_sync(0xffffffffu, jv.t0, 0);
      while (ts < t1) {
        const int te = __shfl_sync(0xffffffffu, args.seg_end[ts], 0);
        const uint32_t nsub = static_cast<uint32_t>(te - ts) * NSUB;
        ptx::mbar_wait_u(&bars[P_KV_FULL], kv_cnt & 1);
        ++kv_cnt;
        ptx::tc_fence_after();
        const uint32_t base = x;
        if (lane == 0) DASH_TRACE_MARK(22, base);
        kb_ready = false;
        issue_sdp(base, nsub == 1);
        for (uint32_t u = 0; u < nsub; ++u) {
          const uint32_t xx = base + u;
          const uint32_t qk = xx % NQK;
          // S/dP of the next sub-tile go into the tensor pipe while the softmax
          // warps turn this one into P^T / dS^T (dQ is issued by the drain).
          if (u + 1 < nsub) issue_sdp(xx + 1, u + 2 == nsub);
          // QK operands first (normally long loaded), so the reaction to
          // P_FULL is only the MMA issue
          ptx::mbar_wait_u(&bars[P_QK_FULL0 + qk], (xx / NQK) & 1);
          if (u == 0 && acc_cnt > 0) ptx::mbar_wait_u(&bars[P_ACC_EMPTY], (acc_cnt - 1) & 1);
          ptx::mbar_wait_u(&bars[P_P_FULL], xx & 1);
          if (lane == 0) DASH_TRACE_MARK(1, xx);
          ptx::tc_fence_after();
          // dK += dS^T Q   (Alg.1 line 26) -- first: the softmax of the next
          // sub-tile writes its dS^T into this TMEM buffer first
#pragma unroll
          for (int kk = 0; kk < BR / 16; ++kk)
            ptx::mma2_bf16_ts_e(tbase + C::T_DK, tbase + C::T_DST + kk * 8,
                                dQK + qk * ST_STEP + kstep<true>(kk, BR), ID_KV, (u > 0 || kk > 0));
          ptx::mma2_commit_mc_e(&bars[P_DST_EMPTY]);
          // dV += P^T dO   (Alg.1 line 25)
#pragma unroll
          for (int kk = 0; kk < BR / 16; ++kk)
            ptx::mma2_bf16_ts_e(tbase + C::T_DV, tbase + C::T_PT + kk * 8,
                                dDOK + qk * ST_STEP + kstep<true>(kk, BR), ID_KV, (u > 0 || kk > 0));
          ptx::mma2_commit_mc_e(&bars[P_PT_EMPTY]);
          ptx::mma2_commit_mc_e(&bars[P_QK_EMPTY0 + qk]);
          if (lane == 0) DASH_TRACE_MARK(16, xx);
          // dQ of the previous sub-tile: its dS^T exchange has had a whole
          // sub-tile to complete, so it does not hold up S/dP of the next one
          if (u >= 1) issue_dq(xx - 1);
        }
        issue_dq(base + nsub - 1);
        x = base + nsub;
        ptx::mma2_commit_mc_e(&bars[P_KV_EMPTY]);
        ptx::mma2_commit_mc_e(&bars[P_ACC_FULL]);
        ++acc_cnt;
        ts = te;
      }
    }
    if (leader) {
      ptx::mma2_commit_mc_e(&bars[P_MMA_DRAIN]);
      ptx::mbar_wait_bounded(&bars[P_MMA_DRAIN], 0);
    }
  } else if (warp == 2 || warp == 3) {
    // ======================== ordered dQ reducers (both CTAs) ========================
    if (lane == 0) {
      const uint32_t agent = static_cast<uint32_t>(warp - 2);
      const bool det = args.deterministic != 0;
      uint32_t it_job = 0, x = 0;
      if (leader && agent == 0) {
        const int first = atomicAdd(args.job_counter, 1);
        job_slot[0] = first;
        ptx::st_cluster_u32(ptx::mapa(ptx::smem_u32(&job_slot[0]), 1), static_cast<uint32_t>(first));
        ptx::mbar_arrive(&bars[P_JOB0]);
        ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&bars[P_JOB0]), 1));
      }
      while (true) {
        ptx::mbar_wait_cluster(&bars[P_JOB0 + (it_job & 1)], (it_job >> 1) & 1);
        const int g = job_slot[it_job & 1];
        slot_read(it_job);
        if (g >= args.total_jobs || ptx::aborted()) break;
        const JobView jv = decode_job(args, g);
        for (int t = jv.t0; t < jv.t1; ++t) {
          const TaskView tv = decode_task(args, jv, args.tasks[t]);
          const int q = tv.q, rank = tv.rank;
          for (int sub = 0; sub < NSUB; ++sub, ++x) {
            if ((x % NAG) != agent) continue;
            const uint32_t ph = (x / NAG) & 1;
            const int urow = q * C::TILE + sub * BR;  // first Q row of the unit
            const int par = rank % args.split, rank_w = rank / args.split;  // AMB-27
            int* ticket = args.tickets + static_cast<size_t>(par) * args.n_tickets +
                          (static_cast<size_t>(tv.bh - args.bh_base) * n_units + urow / BR) * 2 + cta;
            if (det) {
              if (ptx::ld_acquire(ticket) != rank_w) {
                const long long t_start = clock64();
                uint32_t polls = 0;
                while (ptx::ld_relaxed(ticket) != rank_w) {
                  __nanosleep(32);
                  if ((++polls & ptx::kAbortPollMask) != 0) continue;
                  if (clock64() - t_start > args.spin_bound || ptx::aborted()) {
                    atomicExch(args.error_flag, 1);
                    atomicExch(&ptx::g_dash_abort, 1);
                    break;
                  }
                }
                (void)ptx::ld_acquire(ticket);
              }
              ptx::fence_async_global();
            }
            DASH_TRACE_MARK(7, x);
            // Add this CTA's d half of dQ_local into dQ (Alg.1 line 34); rank 0 stores.
            const int grow = (par * args.bh_count + tv.bh - args.bh_base) * args.N + urow;
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              ptx::mbar_wait(&bars[P_AGF0 + hh * NAG + agent], ph);
              const uint8_t* src = smem + C::OFF_DQ + hh * (BR * 128);
              const int col = static_cast<int>(cta) * 64 + hh * 32;
              if (det && rank_w == 0) tma_store_2d(&tm_dqacc, src, col, grow);
              else tma_reduce_add_2d(&tm_dqacc, src, col, grow);
              ptx::bulk_commit();
              if (hh == 1) {
                ptx::bulk_wait_read<1>();
                ptx::mbar_arrive(&bars[P_STG_EMPTY0]);
              }
            }
            DASH_TRACE_MARK(8, x);
            ptx::bulk_wait_read<0>();
            ptx::mbar_arrive(&bars[P_STG_EMPTY0 + 1]);
            DASH_TRACE_MARK(11, x);
            ptx::bulk_wait_all();
            DASH_TRACE_MARK(12, x);
            if (det) {
              ptx::fence_async_global();
              DASH_TRACE_MARK(17, x);
              ptx::st_release(ticket, rank_w + 1);
            }
            DASH_TRACE_MARK(9, x);
          }
        }
        count_job_done(args, g);
        ptx::mbar_arrive_remote(lbar(P_JOB_DONE));
        if (leader && agent == 0) {
          ptx::mbar_wait_cluster(&bars[P_JOB_DONE], it_job & 1);
          ptx::mbar_wait(&bars[P_PF0 + (it_job & 1)], (it_job >> 1) & 1);
          if (claim_mode[it_job & 1] == 2) {
            const uint32_t j1 = it_job + 1;
            if (j1 >= 2) ptx::mbar_wait_cluster(&bars[P_SLOT_FREE0 + (j1 & 1)], ((j1 - 2) >> 1) & 1);
            const int next = ptx::aborted() ? args.total_jobs : atomicAdd(args.job_counter, 1);
            DASH_TRACE_MARK(21, x);
            job_slot[j1 & 1] = next;
            ptx::st_cluster_u32(ptx::mapa(ptx::smem_u32(&job_slot[j1 & 1]), 1),
                                static_cast<uint32_t>(next));
            ptx::mbar_arrive(&bars[P_JOB0 + (j1 & 1)]);
            ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&bars[P_JOB0 + (j1 & 1)]), 1));
          }
        }
        ++it_job;
      }
    }
    __syncwarp();
  } else if (warp >= 4 && warp < 12) {
    // ===================== softmax / dS / epilogue (both CTAs) =====================
    const int wg = (warp - 4) >> 2;          // column half = N half = owner CTA of the dS^T columns
    const int row = (warp & 3) * 32 + lane;  // own KV row = TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const int c_base = wg * C::SMX_COLS;
    const int krow = C::BC * static_cast<int>(cta) + row;  // row in the 256-row K dimension
    uint32_t it_job = 0, x = 0, acc_cnt = 0;
    while (true) {
      ptx::mbar_wait_cluster(&bars[P_JOB0 + (it_job & 1)], (it_job >> 1) & 1);
      const int g = job_slot[it_job & 1];
      __syncwarp();
      if (lane == 0) slot_read(it_job);
      ++it_job;
      if (g >= args.total_jobs || ptx::aborted()) break;
      const JobView jv = decode_job(args, g);
      int2 tk_cur = args.tasks[jv.t0];
      for (int t = jv.t0; t < jv.t1; ++t) {
        const int2 tk_nxt = (t + 1 < jv.t1) ? args.tasks[t + 1] : make_int2(0, -1);
        const TaskView tv = decode_task(args, jv, tk_cur);
        const int kv = tv.kv, q = tv.q;
        const bool diag = args.causal && (kv == q);
        for (int sub = 0; sub < NSUB; ++sub, ++x) {
          const uint32_t st = x % C::NLD, sb = x % C::NDS;
          ptx::mbar_wait(&bars[P_S_FULL], x & 1);
          ptx::mbar_wait(&bars[P_LD_FULL0 + st], (x / C::NLD) & 1);
          ptx::tc_fence_after();
          if (row == 0 && wg == 0) DASH_TRACE_MARK(3, x);
          const float* Lrow = sL + st * BR;
          const float* Drow = sDv + st * BR;
          const int cc0 = c_base;
          float s[32], dp[32];
          ptx::tmem_ld32(tbase + lane_off + C::T_S + cc0, s);
          ptx::tmem_ld32(tbase + lane_off + C::T_DP + cc0, dp);
          ptx::tmem_wait_ld();
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive_remote(lbar(P_S_EMPTY));
          uint32_t pk[16], dk2[16];
          auto smx = [&](auto masked) {
            constexpr bool MASKED = decltype(masked)::value;
            // causal, diagonal tile: key (KV row krow) hidden from query (sub-tile
            // row) when krow > sub * BR + col
            const int mask_from = krow - sub * BR - cc0;  // masked: cols c < mask_from
#pragma unroll
            for (int c4 = 0; c4 < 8; ++c4) {
              const float4 l4 = *reinterpret_cast<const float4*>(Lrow + cc0 + c4 * 4);
              const float4 d4 = *reinterpret_cast<const float4*>(Drow + cc0 + c4 * 4);
              const float Lv[4] = {l4.x, l4.y, l4.z, l4.w};
              const float Dv[4] = {d4.x, d4.y, d4.z, d4.w};
              float p[4], ds[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int c = c4 * 4 + e;
                float pv = fast_exp2(fmaf(s[c], args.scale_log2, Lv[e]));
                if constexpr (MASKED) {
                  if (c < mask_from) pv = 0.f;
                }
                p[e] = pv;
                ds[e] = pv * (dp[c] - Dv[e]);
              }
              pk[c4 * 2] = pack_bf16(p[0], p[1]);
              pk[c4 * 2 + 1] = pack_bf16(p[2], p[3]);
              dk2[c4 * 2] = pack_bf16(ds[0], ds[1]);
              dk2[c4 * 2 + 1] = pack_bf16(ds[2], ds[3]);
            }
          };
          if (diag) smx(std::true_type{});
          else smx(std::false_type{});
          ptx::mbar_arrive(&bars[P_LD_EMPTY0 + st]);  // this thread's L, D reads of the slot are done
          if (x >= 1) ptx::mbar_wait(&bars[P_DST_EMPTY], (x - 1) & 1);
          ptx::tmem_st16(tbase + lane_off + C::T_DST + cc0 / 2, dk2);
          if (x >= 1) ptx::mbar_wait(&bars[P_PT_EMPTY], (x - 1) & 1);
          ptx::tmem_st16(tbase + lane_off + C::T_PT + cc0 / 2, pk);
          ptx::tmem_wait_st();
          ptx::tc_fence_before();
          __syncwarp();
          // P^T / dS^T are in TMEM: dV / dK of this sub-tile may go
          if (lane == 0) ptx::mbar_arrive_remote(lbar(P_P_FULL));
          // dS^T columns [32 wg, 32 wg + 32) of KV row krow -> CTA wg's SW64 buffer
          if (x >= C::NDS) ptx::mbar_wait(&bars[P_DS_EMPTY0 + sb], ((x / C::NDS) - 1) & 1);
          if (row == 0 && wg == 0) DASH_TRACE_MARK(13, x);
          const bool own_half = wg == static_cast<int>(cta);
          // own column half -> the local DS buffer (rows 128c + row); the peer's
          // half -> the outbox (same SW64 layout as the destination rows)
          uint8_t* dst = own_half ? smem + C::OFF_DS + sb * C::DS_BYTES + krow * 64
                                  : smem + C::OFF_OUT + sb * C::OUT_BYTES + row * 64;
#pragma unroll
          for (int c8 = 0; c8 < 4; ++c8) {
            const uint32_t off = static_cast<uint32_t>((c8 ^ ((krow >> 1) & 3)) << 4);
            *reinterpret_cast<uint4*>(dst + off) =
                make_uint4(dk2[c8 * 4], dk2[c8 * 4 + 1], dk2[c8 * 4 + 2], dk2[c8 * 4 + 3]);
          }
          ptx::fence_async_smem();
          __syncwarp();
          if (row == 0 && wg == 0) DASH_TRACE_MARK(15, x);
          if (lane == 0) {
            if (!own_half) {
              // this warp's 32 rows (2 KB) -> the partner's DS buffer rows
              // [128c + 32w, +32), completing on the partner's P_DSR[sb]
              const uint32_t peer = cta ^ 1u;
              const uint32_t r0 = static_cast<uint32_t>((warp & 3) * 32);
              const uint32_t dst_cl = ptx::mapa(
                  ptx::smem_u32(smem + C::OFF_DS + sb * C::DS_BYTES + (C::BC * cta + r0) * 64), peer);
              ptx::bulk_copy_s2cluster(dst_cl, smem + C::OFF_OUT + sb * C::OUT_BYTES + r0 * 64,
                                       C::OUT_BYTES / 4,
                                       ptx::mapa(ptx::smem_u32(&bars[P_DSR0 + sb]), peer));
            } else if ((warp & 3) == 0) {
              // own rows stored; also arms the partner's 8 KB of this use (safe:
              // the previous phase of P_DSR[sb] completed before S^T / dP^T of
              // this sub-tile were issued)
              ptx::mbar_arrive_expect_tx_local(&bars[P_DSR0 + sb], C::OUT_BYTES);
            } else {
              ptx::mbar_arrive(&bars[P_DSR0 + sb]);
            }
          }
          if (row == 0 && wg == 0) DASH_TRACE_MARK(4, x);
        }
        // End of a KV segment: dK/dV epilogue for this CTA's 128 KV rows.
        const bool seg_end = (t + 1 == jv.t1) || (task_seg(tk_nxt) != tv.seg);
        if (seg_end) {
          ptx::mbar_wait(&bars[P_ACC_FULL], acc_cnt & 1);
          ++acc_cnt;
          ptx::tc_fence_after();
          if (row == 0 && wg == 0) DASH_TRACE_MARK(18, x - 1);
          // dK, dV rows of this warp (32 KV rows x this warpgroup's 64 d columns)
          // go out through TMA stores of 32 x 32 bf16 boxes staged in the warp's
          // 2 KB of the outbox: free here -- ACC_FULL follows the last dQ MMA,
          // which waited for every dS^T copy out of it.  (Generic stores of one
          // 16 B piece per row per lane are LSU-bound -- one L2 request per
          // lane -- and keep the SM's store queue full under the reducers'
          // release fences.)
          uint8_t* ep = smem + C::OFF_OUT + (warp - 4) * 2048;
          const int grow0 = tv.b * args.N + kv * C::TILE + C::BC * static_cast<int>(cta) + (warp & 3) * 32;
          int nst = 0;
#pragma unroll 1
          for (int c0 = wg * (D / C::NSMX); c0 < (wg + 1) * (D / C::NSMX); c0 += 32) {
            float a[32], k2[32];
            ptx::tmem_ld32(tbase + lane_off + C::T_DV + c0, a);
            ptx::tmem_ld32(tbase + lane_off + C::T_DK + c0, k2);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int which = 0; which < 2; ++which) {  // dV, then dK (x scale, AMB-1)
              const float* src = which == 0 ? a : k2;
              const float sc = which == 0 ? 1.f : args.scale;
              if (nst > 0) {  // the previous box has been read out of the staging
                if (lane == 0) ptx::bulk_wait_read<0>();
                __syncwarp();
              }
#pragma unroll
              for (int e = 0; e < 32; e += 8) {
                uint4 pv;
                pv.x = pack_bf16(src[e] * sc, src[e + 1] * sc);
                pv.y = pack_bf16(src[e + 2] * sc, src[e + 3] * sc);
                pv.z = pack_bf16(src[e + 4] * sc, src[e + 5] * sc);
                pv.w = pack_bf16(src[e + 6] * sc, src[e + 7] * sc);
                *reinterpret_cast<uint4*>(ep + lane * 64 + e * 2) = pv;
              }
              ptx::fence_async_smem();
              __syncwarp();
              if (lane == 0) {
                tma_store_2d(which == 0 ? &tm_dv : &tm_dk, ep, tv.h * D + c0, grow0);
                ptx::bulk_commit();
              }
              ++nst;
            }
          }
          ptx::tc_fence_before();
          if (lane == 0) ptx::bulk_wait_read<0>();
          __syncwarp();
          if (row == 0 && wg == 0) DASH_TRACE_MARK(19, x - 1);
          if (lane == 0) ptx::mbar_arrive_remote(lbar(P_ACC_EMPTY));
          // every warp's staging has been read before any warp writes the
          // outbox again (the next sub-tile's dS^T halves)
          ptx::named_bar_sync(1, 256);
        }
        tk_cur = tk_nxt;
      }
    }
    if (lane == 0) ptx::bulk_wait_all();  // dK / dV stores complete before the CTA retires
    __syncwarp();
  } else {
    // ================== dQ drain (both CTAs): TMEM -> fp32 SW128 staging ==================
    // dQ^T of this CTA (M = 64 d rows per SM, N = 64 Q cols): lane l < 64 holds
    // d row l for Q cols 0..31, lane 64 + l the same d row for Q cols 32..63.
    const int tl = (warp & 3) * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const int dl = tl & 63;           // d index within this CTA's half
    const int q0 = (tl >> 6) * 32;    // first Q row (of the sub-tile) this thread holds
    const int part = dl >> 5;         // staging part = 32-column box of the d half
    const int dcol = dl & 31;
    uint32_t it_job = 0, x = 0;
    while (true) {
      ptx::mbar_wait_cluster(&bars[P_JOB0 + (it_job & 1)], (it_job >> 1) & 1);
      const int g = job_slot[it_job & 1];
      __syncwarp();
      if (lane == 0) slot_read(it_job);
      ++it_job;
      if (g >= args.total_jobs || ptx::aborted()) break;
      const JobView jv = decode_job(args, g);
      for (int t = jv.t0; t < jv.t1; ++t) {
        const int2 tk = args.tasks[t];
        for (int sub = 0; sub < NSUB; ++sub, ++x) {
          const uint32_t qb = x & 1;
          ptx::mbar_wait(&bars[P_DQ_FULL0 + qb], (x >> 1) & 1);
          ptx::tc_fence_after();
          if (tl == 0) DASH_TRACE_MARK(5, x);
          float v[32];
          ptx::tmem_ld32(tbase + lane_off + C::T_DQ + qb * 32, v);
          ptx::tmem_wait_ld();
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive_remote(lbar(P_DQ_EMPTY0 + qb));
          if (args.dump) {
            const TaskView tv = decode_task(args, jv, tk);
            const int urow0 = tv.q * C::TILE + sub * BR;
            float* dp = args.dump + ((static_cast<size_t>(tv.bh) * (args.N / C::TILE) + tv.kv) *
                                         args.N + urow0) * D + cta * 64 + dl;
#pragma unroll
            for (int c = 0; c < 32; ++c) dp[(q0 + c) * D] = v[c];
          }
          if (x >= 1) ptx::mbar_wait(&bars[P_STG_EMPTY0 + part], (x - 1) & 1);
          uint8_t* box = smem + C::OFF_DQ + part * (BR * 128);
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            const int r = q0 + c;
            const uint32_t off = r * 128 + ((((dcol >> 2) ^ (r & 7))) << 4) + (dcol & 3) * 4;
            *reinterpret_cast<float*>(box + off) = v[c];
          }
          ptx::fence_async_smem();
          ptx::mbar_arrive(&bars[P_AGF0 + part * NAG + (x % NAG)]);
          if (tl == 0) DASH_TRACE_MARK(6, x);
        }
      }
    }
  }

  if (ptx::aborted()) {
    // watchdog tripped: roles left their loops at different points; let every
    // asynchronous copy / load / MMA still in flight land before either CTA
    // of the pair retires (error path only; outputs are invalid anyway)
    const long long t0 = clock64();
    while (clock64() - t0 < (1ll << 22)) {
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync();  // no remote arrive / DSMEM store may target a retired CTA
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc2<512>(tbase);
  }
  if (args.fuse_dq) finalize_dq<D, C::NTHREADS>(args, reinterpret_cast<int*>(smem + C::OFF_DQ));
  if (tid == 0 && ptx::aborted()) atomicExch(args.error_flag, 2);
}

}  // namespace dash
