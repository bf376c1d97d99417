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
//   dV  += P^T dO  (P^T from TMEM, tcgen05 TS) ;  dK += dS^T Q  (SS)
//                          (TMEM accumulators, whole job)
//   dQ_part = dS K  (d = 64)  or  dQ_part^T = K^T dS^T  (d = 128)   (TMEM)
//   ordered reduction: wait ticket == rank, TMA reduce-add (rank 0: store)
//   of the fp32 partial into dQacc, release ticket = rank + 1
//                          (Alg.1 lines 30-36)
//
// Warp roles (16 warps, 512 threads):
//   0      TMA producer (K/V per KV tile, Q/dO/L/D per sub-tile, NSTAGE ring)
//   1      MMA issuer (one thread) + TMEM owner
//   2, 3   dQ reducers: one single-thread agent per warp (lane 0); staging
//          unit x belongs to agent x % 2 (acquire ticket -> bulk reduce-add ->
//          read done frees the staging -> completion -> release), so two
//          ordered adds are in flight; agent 0 also claims jobs
//   4-11   softmax / dS, then the dK/dV epilogue: two warpgroups, each owning
//          half of the sub-tile's columns (TMEM lane quarter = warp % 4)
//   12-15  dQ drain: TMEM -> registers -> SW128 fp32 staging
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include <type_traits>

#include "umma.cuh"

namespace dash {

struct BwdArgs {
  const float* lse2;     // [B,H,N]  -L * log2(e)  (written by the preprocess kernel)
  const float* Dvec;     // [B,H,N]  rowsum(dO * O)
  __nv_bfloat16* dk;     // [B,N,H,d]
  __nv_bfloat16* dv;     // [B,N,H,d]
  int* tickets;          // [B*H][N/BR]
  int* job_counter;      // 1
  int* error_flag;       // 1
  const int* job_begin;  // [jobs_per_head + 1]
  const int2* tasks;     // {kv | q << 16, rank}
  const int* seg_end;    // per task: index of the first task of the next KV segment (or job end)
  int B, N, H;
  int jobs_per_head;
  int total_jobs;
  float scale;
  float scale_log2;
  int causal;
  int deterministic;
  unsigned long long* trace;  // optional clock64 trace [grid][trace_cap][32] (measurement only)
  int trace_cap;
  long long spin_bound;  // ticket-wait watchdog, clock64 cycles (dash_attn_bwd_set_watchdog)
  float* dump;  // verification only: every dQ partial, [B*H][N/128][N][d] fp32
  // Interleaved accumulation (AMB-27): split = W in {1, 2, 4, 8}.  The contribution
  // of rank k goes into accumulator k % W (dQacc + (k % W) * B*H*N*d) in the
  // order of its ticket set k % W (value k / W); the convert kernel adds the W
  // accumulators in index order.  W = 1 is the paper's single global order.
  int split;
  int n_tickets;  // tickets per accumulator
  float* dqacc;   // the W accumulators [W][B,H,N,d] fp32 (1-D bulk reduce at d = 128)
  // Early claim of the next job (see the producer): 0 = claim only after every
  // ordered add of the current job is released; 1 = the producer claims the next
  // job as soon as it has issued the current job's last load, when that is
  // deadlock-free (cyclic = 1: the schedule has cyclic waits inside a head, so
  // the next job must belong to another head).
  int prefetch;
  int cyclic;
  // Head grouping: job g covers the same KV tile(s) of G = head_group
  // consecutive (b, h) heads, bh = (g / jobs_per_head) * G + hoff, each head's
  // tasks in its own schedule order (task.y = rank | hoff << 16).  Per-head Q
  // orders and reduction ranks are unchanged, so results are bit-identical
  // for every G; G only amortises the per-job claim / drain cost.
  int head_group;
  // Head chunk of this launch (dQ-plane budget, dash_attn_bwd_set_plane_budget):
  // jobs cover the flattened heads bh_base .. bh_base + bh_count - 1; the W
  // accumulators and ticket sets hold only those heads (local index
  // bh - bh_base, plane stride bh_count).  One launch = one chunk = B*H heads
  // unless the planes of all heads exceed the budget.
  int bh_base;
  int bh_count;
  // Fused dQ finalise: the main kernel writes dq
  // itself, so there is no K4.  Every reducer agent adds 1 to done[g /
  // jobs_per_head] (release, after its job's last ordered add completed); once
  // a job group's count reaches jobs_per_head x agents all of its heads' dQ
  // accumulators are final.  CTAs that find the job counter exhausted then
  // claim finalise tasks (done[bh_count / head_group] is the task counter,
  // 64 / 128 rows of one head per task, heads in job order) and write
  // dq = bf16(scale * (acc_0 + ... + acc_{W-1})), the sum K4 forms.
  int* done;
  __nv_bfloat16* dq;  // [B,N,H,d]
  int fuse_dq;        // 0: K4 converts (dash_attn_bwd_set_fused_dq(0))
  int acc_tile;       // schedule tile rows (128 / 256): contributions per Q tile
  int done_target;    // jobs_per_head x reducer agents per job (both CTAs of a pair)
};

// Per-(CTA, sub-tile) clock64 stamps for pipeline analysis; a null trace
// pointer makes every mark a not-taken branch.
#define DASH_TRACE_MARK(slot, xx)                                                         \
  do {                                                                                    \
    if (args.trace != nullptr && static_cast<int>(xx) < args.trace_cap)                   \
      args.trace[(static_cast<size_t>(blockIdx.x) * args.trace_cap + (xx)) * 32 + (slot)] = \
          clock64();                                                                      \
  } while (0)

// Shared-memory plan.  The fp32 dQ partial of a sub-tile (32 KB at both head
// dims) is staged once and handed to the bulk engine:
//   d = 128 (LINEAR): staged row-major and reduced with 1-D bulk copies
//     (cp.reduce.async.bulk, no tensor map) -- a sub-tile's partial is one
//     contiguous 32 KB run of dQacc.  The buffer is a ring of two halves (rows
//     0-31, 32-63): the drain writes one half while the bulk engine still
//     reads the other.
//   d = 64: staged as SW128 boxes of 32 fp32 columns and reduced with 2-D
//     tensor-map bulk reduces (a 128-row unit is not one contiguous run).
// Measured alternatives (round 1, profiles/r01_experiments/): one staging
// buffer per reducer with a 2-stage ring, half-size units with their own
// tickets, a 4-part or 3-slot ring, and half bulk / half red.global were all
// neutral or slower; they are no longer built.
template <int D>
struct BwdCfg {
  static constexpr int NTHREADS = 512;
  static constexpr int BC = 128;                    // KV tile rows (TMEM lanes)
  static constexpr int BR = (D == 128) ? 64 : 128;  // Q sub-tile rows
  static constexpr int NSUB = 128 / BR;             // sub-tiles per schedule Q tile
  static constexpr int NSTAGE = (D == 128) ? 3 : 2; // Q/dO/L/D ring depth
  static constexpr bool LINEAR = (D == 128);        // 1-D bulk reduce of a row-major partial
  static constexpr int NPART = 2;                   // linear staging: parts (= ring slots)
  static constexpr int NSMX = 2;                    // softmax warpgroups (column halves)
  static constexpr int SMX_COLS = BR / NSMX;        // columns per softmax thread
  static constexpr uint32_t KV_BYTES = BC * D * 2;
  static constexpr uint32_t Q_BYTES = BR * D * 2;
  static constexpr uint32_t P_BYTES = BC * BR * 2;
  // One staging unit (and one ticket) per Q sub-tile.
  static constexpr int STG_ROWS = BR;
  static constexpr uint32_t DQ_BYTES = STG_ROWS * D * 4;
  static constexpr uint32_t OFF_K = 0;
  static constexpr uint32_t OFF_V = OFF_K + KV_BYTES;
  static constexpr uint32_t OFF_Q = OFF_V + KV_BYTES;            // NSTAGE stages
  static constexpr uint32_t OFF_DO = OFF_Q + NSTAGE * Q_BYTES;   // NSTAGE stages
  static constexpr int NDS = 2;                                  // dS^T smem buffers
  // d = 128: dS^T also lives in TMEM so dK += dS^T Q runs as a TS MMA (A from
  // TMEM, full rate, no smem read); d = 64 has no TMEM room left for it.
  static constexpr bool DS_IN_TMEM = (D == 128);
  static constexpr uint32_t OFF_DS = OFF_DO + NSTAGE * Q_BYTES;  // NDS x dS^T bf16 SW128
  static constexpr uint32_t OFF_DQ = OFF_DS + NDS * P_BYTES;     // fp32 staging buffer
  static constexpr uint32_t STG_BYTES = DQ_BYTES;
  static constexpr uint32_t OFF_L = OFF_DQ + STG_BYTES;           // NSTAGE x BR floats
  static constexpr uint32_t OFF_DV = OFF_L + NSTAGE * BR * 4;    // NSTAGE x BR floats
  static constexpr uint32_t OFF_BAR = OFF_DV + NSTAGE * BR * 4;
  static constexpr int NBAR = 40;
  static constexpr uint32_t OFF_MISC = OFF_BAR + NBAR * 8;
  static constexpr uint32_t BODY_BYTES = OFF_MISC + 64;
  // Re-alignment slack for the 1024-B swizzle atoms (as much as fits; the
  // kernel traps if the dynamic smem base needs more than it has).
  static constexpr uint32_t SLACK = (BODY_BYTES + 1024 <= 232448) ? 1024 : (232448 - BODY_BYTES);
  static constexpr uint32_t SMEM_BYTES = BODY_BYTES + SLACK;
  // TMEM columns
  static constexpr uint32_t T_S = 0;
  static constexpr uint32_t T_DP = BR;
  static constexpr uint32_t T_DV = 2 * BR;
  static constexpr uint32_t T_DK = 2 * BR + D;
  static constexpr uint32_t T_DQ = 2 * BR + 2 * D;  // 64 columns
  static constexpr uint32_t T_PT = T_DQ + 64;       // BR/2 columns of packed bf16 P^T
  static constexpr uint32_t T_DST = T_PT + BR / 2;  // BR/2 columns of packed bf16 dS^T (d = 128)
  static_assert(T_PT + BR / 2 + (DS_IN_TMEM ? BR / 2 : 0) == 512, "TMEM budget");
  static_assert(SMEM_BYTES <= 232448, "smem budget");
  static_assert(SMX_COLS % 32 == 0, "softmax column split");
  static_assert(NDS * P_BYTES >= 8 * 4096, "dK/dV epilogue staging (4 KB per softmax warp)");
};

// Barrier slots (arrival count in parentheses)
enum : int {
  B_JOB0 = 0, B_JOB1 = 1,              // job slot filled (1)
  B_KV_FULL = 2, B_KV_EMPTY = 3,       // K/V tile loaded (tx) / consumed by MMA (commit)
  B_S_FULL = 4, B_S_EMPTY = 5,         // S^T/dP^T in TMEM (commit) / read by softmax (256)
  B_P_FULL = 6,                        // P^T (TMEM) and dS^T (smem) written (256)
  B_DQ_FULL = 7, B_DQ_EMPTY = 8,       // dQ partial in TMEM (commit) / drained (128)
  B_PT_EMPTY = 9,                      // P^T TMEM buffer consumed by dV (commit)
  B_DST_EMPTY = 10,                    // dS^T TMEM buffer consumed by dK (commit)
  B_STG_EMPTY1 = 11,                   // linear staging part 1 read by the reduce (1)
  B_ACC_FULL = 12, B_ACC_EMPTY = 13,   // dK/dV complete (commit) / drained (256)
  B_STG_EMPTY = 14,                    // staging (part 0) read by the reduce (1)
  B_JOB_DONE = 15,                     // every reducer agent released the job (NAG)
  B_MMA_DRAIN = 16,                    // exit: every issued MMA has completed (commit)
  B_Q_FULL0 = 18,                      // + stage (<= 4): Q/dO/L/D loaded (tx)
  B_DS_EMPTY0 = 22, B_DS_EMPTY1 = 23,  // dS^T smem buffer consumed by dK, dQ (commit)
  B_PF0 = 24,                          // + (t - 1) % 2: producer's claim decision for job t (1)
  B_Q_EMPTY0 = 26,                     // + stage (<= 4): stage consumed (commit)
  B_SLOT_FREE0 = 30,                   // + j % 2: every warp has read job j's slot (16)
  B_AGF0 = 32,                         // + h * NAG + agent: staging (part h) written for
                                       // the agent of unit x (x % NAG) (128)
  B_COUNT = 40
};
constexpr int NAG = 2;  // reducer agents (single threads, one per reducer warp)

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

// Job / task decode shared by every role.
struct JobView {
  int bh0, t0, t1;  // first (b, h) head of the job's group; task range
};
__device__ __forceinline__ JobView decode_job(const BwdArgs& a, int g) {
  JobView j;
  j.bh0 = a.bh_base + (g / a.jobs_per_head) * a.head_group;
  const int lj = g % a.jobs_per_head;
  j.t0 = a.job_begin[lj];
  j.t1 = a.job_begin[lj + 1];
  return j;
}
struct TaskView {
  int kv, q, rank, bh, b, h;
  int seg;  // KV segment key: (kv, head) -- K/V, dK/dV change with it
};
__device__ __forceinline__ int task_seg(int2 tk) {
  return (tk.x & 0xFFFF) | (tk.y & static_cast<int>(0xFFFF0000u));
}
__device__ __forceinline__ TaskView decode_task(const BwdArgs& a, const JobView& jv, int2 tk) {
  TaskView v;
  v.kv = tk.x & 0xFFFF;
  v.q = tk.x >> 16;
  v.rank = tk.y & 0xFFFF;
  v.bh = jv.bh0 + (static_cast<unsigned>(tk.y) >> 16);
  v.b = v.bh / a.H;
  v.h = v.bh % a.H;
  v.seg = task_seg(tk);
  return v;
}

// Reducer agent: this job's ordered adds are complete -- count it (the bulk
// groups were waited on with wait_group 0; the proxy fence orders the async
// proxy's writes before the generic release).
__device__ __forceinline__ void count_job_done(const BwdArgs& a, int g) {
  if (!a.fuse_dq) return;
  ptx::fence_async_global();
  ptx::red_release_add(a.done + g / a.jobs_per_head, 1);
}

// Fused dQ finalise, run by every thread of a CTA after its roles found no
// job left.  `slot` = one int of shared memory.  Tasks are claimed in head
// order (the order heads complete in); a task waits (acquire) for its job
// group's completion count.  Per element the arithmetic is K4's: the planes a
// Q tile was written into, added in index order, times scale, to bf16.
template <int D, int NT, int W>
__device__ __forceinline__ void finalize_dq_w(const BwdArgs& a, int* slot) {
  constexpr int T = D / 8;             // threads per row, 8 elements each
  constexpr int RPP = NT / T;          // rows per pass
  constexpr int FR = 16384 / D;        // rows per task (64 KB of fp32 per plane)
  constexpr int PASSES = FR / RPP;
  constexpr int UMAX = W <= 2 ? 4 : (W == 4 ? 2 : 1);
  constexpr int U = PASSES < UMAX ? PASSES : UMAX;  // passes with their loads in flight together
  static_assert(PASSES % U == 0, "passes");
  const int tid = threadIdx.x;
  const int nrb = (a.N + FR - 1) / FR;  // d = 64: N may end in half a task
  const int G = a.head_group;
  const int total = a.bh_count * nrb;
  int* task_counter = a.done + a.bh_count / G;
  const size_t plane = static_cast<size_t>(a.bh_count) * a.N * D;
  const int part = tid % T;
  auto group_done = [&](int task) { return a.done + (task / nrb) / G; };
  // Thread 0 claims one task ahead and, while the current task's loads are in
  // flight, checks (acquire) whether the next task's job group is complete, so
  // a finished group costs no round trip at the start of its task.  Abort
  // decisions are thread 0's, read back by all: uniform at every barrier.
  bool ready = false;
  if (tid == 0) slot[0] = ptx::aborted() ? total : atomicAdd(task_counter, 1);
  __syncthreads();
  int t = slot[0];
  while (t < total) {
    const int lh = t / nrb, rb = t % nrb;  // local head, row block
    int nxt = 0;
    if (tid == 0) {
      nxt = atomicAdd(task_counter, 1);
      const int* cnt = group_done(t);
      if (!ready && ptx::ld_acquire(cnt) < a.done_target) {
        const long long t0 = clock64();
        uint32_t polls = 0;
        while (ptx::ld_relaxed(cnt) < a.done_target) {
          __nanosleep(64);
          if ((++polls & ptx::kAbortPollMask) != 0) continue;
          if (clock64() - t0 > a.spin_bound || ptx::aborted()) {
            atomicExch(a.error_flag, 1);
            atomicExch(&ptx::g_dash_abort, 1);
            break;
          }
        }
        (void)ptx::ld_acquire(cnt);
      }
      ptx::fence_async_global();
      slot[2] = ptx::aborted() ? 1 : 0;
    }
    __syncthreads();
    if (slot[2]) break;
    const int bh = a.bh_base + lh;
    const int h = bh % a.H, b = bh / a.H;
#pragma unroll
    for (int u0 = 0; u0 < PASSES; u0 += U) {
      float4 x[U][W][2];
      int planes[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int n = rb * FR + (u0 + u) * RPP + tid / T;
        const int cnt = a.causal ? n / a.acc_tile + 1 : a.N / a.acc_tile;
        planes[u] = n >= a.N ? 0 : (W < cnt ? W : cnt);  // accumulator w holds ranks w, w + W, ...
        const float* src = a.dqacc + (static_cast<size_t>(lh) * a.N + n) * D + part * 8;
#pragma unroll
        for (int w = 0; w < W; ++w) {
          if (w < planes[u]) {
            x[u][w][0] = __ldcs(reinterpret_cast<const float4*>(src + w * plane));
            x[u][w][1] = __ldcs(reinterpret_cast<const float4*>(src + w * plane + 4));
          }
        }
      }
      if (tid == 0 && u0 == 0) {
        slot[1] = nxt;
        ready = nxt < total && ptx::ld_acquire(group_done(nxt)) >= a.done_target;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int n = rb * FR + (u0 + u) * RPP + tid / T;
        if (planes[u] == 0) continue;
        float4 s0 = x[u][0][0], s1 = x[u][0][1];
#pragma unroll
        for (int w = 1; w < W; ++w) {
          if (w < planes[u]) {
            s0 = make_float4(s0.x + x[u][w][0].x, s0.y + x[u][w][0].y, s0.z + x[u][w][0].z,
                             s0.w + x[u][w][0].w);
            s1 = make_float4(s1.x + x[u][w][1].x, s1.y + x[u][w][1].y, s1.z + x[u][w][1].z,
                             s1.w + x[u][w][1].w);
          }
        }
        uint4 out;
        out.x = pack_bf16(s0.x * a.scale, s0.y * a.scale);
        out.y = pack_bf16(s0.z * a.scale, s0.w * a.scale);
        out.z = pack_bf16(s1.x * a.scale, s1.y * a.scale);
        out.w = pack_bf16(s1.z * a.scale, s1.w * a.scale);
        *reinterpret_cast<uint4*>(a.dq + ((static_cast<size_t>(b) * a.N + n) * a.H + h) * D +
                                  part * 8) = out;
      }
    }
    __syncthreads();  // slot[1] published; slot[1] / slot[2] rewritten only after the next barrier
    t = slot[1];
  }
}
template <int D, int NT>
__device__ __forceinline__ void finalize_dq(const BwdArgs& a, int* slot) {
  switch (a.split) {
    case 1: finalize_dq_w<D, NT, 1>(a, slot); break;
    case 2: finalize_dq_w<D, NT, 2>(a, slot); break;
    case 4: finalize_dq_w<D, NT, 4>(a, slot); break;
    default: finalize_dq_w<D, NT, 8>(a, slot); break;
  }
}

template <int D>
__global__ void __launch_bounds__(512, 1)
    dash_bwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
                    const __grid_constant__ CUtensorMap tm_dqacc,
                    const __grid_constant__ CUtensorMap tm_dk,
                    const __grid_constant__ CUtensorMap tm_dv, const BwdArgs args) {
  using C = BwdCfg<D>;
  constexpr int BR = C::BR, NSUB = C::NSUB, NSTAGE = C::NSTAGE;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t pad = (1024 - (ptx::smem_u32(smem_raw) & 1023)) & 1023;
  if (pad > C::SLACK) __trap();
  uint8_t* smem = smem_raw + pad;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  // linear staging: barrier "part hh of the buffer has been read by the bulk engine"
  auto part_empty = [&](int hh) { return &bars[hh == 0 ? B_STG_EMPTY : B_STG_EMPTY1]; };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::OFF_MISC);
  int* job_slot = reinterpret_cast<int*>(smem + C::OFF_MISC + 8);  // [2]
  volatile int* claim_mode = reinterpret_cast<volatile int*>(smem + C::OFF_MISC + 16);  // [2]
  // Job j travels in slot j % 2; before slot j % 2 is rewritten for job j every
  // warp must have read job j - 2 from it (a claimed-ahead job can be written
  // while a lagging reducer agent has not yet started the previous job).
  auto slot_read = [&](uint32_t j) { ptx::mbar_arrive(&bars[B_SLOT_FREE0 + (j & 1)]); };
  auto wait_slot_free = [&](uint32_t j) {
    if (j >= 2) ptx::mbar_wait(&bars[B_SLOT_FREE0 + (j & 1)], ((j - 2) >> 1) & 1);
  };
  float* sL = reinterpret_cast<float*>(smem + C::OFF_L);
  float* sDv = reinterpret_cast<float*>(smem + C::OFF_DV);

  const int tid = threadIdx.x, lane = tid & 31;
  // Provably warp-uniform warp index (shfl broadcast): lets ptxas keep role
  // branches and everything derived from uniform values in uniform registers.
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);

  if (tid == 0) {
    for (int i = 0; i < B_COUNT; ++i) ptx::mbar_init(&bars[i], 1);
    ptx::mbar_init(&bars[B_S_EMPTY], 128 * C::NSMX);
    ptx::mbar_init(&bars[B_P_FULL], 128 * C::NSMX);
    ptx::mbar_init(&bars[B_ACC_EMPTY], 128 * C::NSMX);
    ptx::mbar_init(&bars[B_DQ_EMPTY], 128);
    for (int i = 0; i < C::NPART * NAG; ++i) ptx::mbar_init(&bars[B_AGF0 + i], 128);
    ptx::mbar_init(&bars[B_JOB_DONE], NAG);
    ptx::mbar_init(&bars[B_SLOT_FREE0], 16);
    ptx::mbar_init(&bars[B_SLOT_FREE0 + 1], 16);
    ptx::fence_mbar_init();
    ptx::fence_async_smem();
    ptx::prefetch_tmap(&tm_q);
    ptx::prefetch_tmap(&tm_k);
    ptx::prefetch_tmap(&tm_v);
    ptx::prefetch_tmap(&tm_do);
    if constexpr (!C::LINEAR) ptx::prefetch_tmap(&tm_dqacc);
    ptx::prefetch_tmap(&tm_dk);
    ptx::prefetch_tmap(&tm_dv);
  }
  if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  // The prologue above overlaps the preprocess kernel's tail (programmatic
  // dependent launch); D, lse2, tickets and the job counter are read only now.
  ptx::griddep_launch();
  ptx::griddep_wait();

  const int n_units = args.N / C::STG_ROWS;  // tickets per head (one per staging unit)

  if (warp == 0) {
    // ============================ TMA producer ============================
    {  // whole warp converged; elect.sync issues
      uint32_t it_job = 0, kv_cnt = 0, q_cnt = 0;
      while (true) {
        ptx::mbar_wait_u(&bars[B_JOB0 + (it_job & 1)], (it_job >> 1) & 1);
        const int g = __shfl_sync(0xffffffffu, job_slot[it_job & 1], 0);
        if (lane == 0) slot_read(it_job);
        ++it_job;
        if (g >= args.total_jobs || __shfl_sync(0xffffffffu, ptx::aborted(), 0)) break;
        const JobView jv = decode_job(args, g);
        int prev_seg = -1;
        for (int t = jv.t0; t < jv.t1; ++t) {
          const TaskView tv = decode_task(args, jv, args.tasks[t]);
          const int kv = tv.kv, q = tv.q;
          if (tv.seg != prev_seg) {
            if (kv_cnt > 0) ptx::mbar_wait_u(&bars[B_KV_EMPTY], (kv_cnt - 1) & 1);
            ptx::mbar_arrive_expect_tx_e(&bars[B_KV_FULL], 2 * C::KV_BYTES);
#pragma unroll
            for (int blk = 0; blk < D / 64; ++blk) {
              ptx::tma_load_2d_e(smem + C::OFF_K + blk * C::BC * 128, &tm_k, &bars[B_KV_FULL],
                               tv.h * D + blk * 64, tv.b * args.N + kv * 128);
              ptx::tma_load_2d_e(smem + C::OFF_V + blk * C::BC * 128, &tm_v, &bars[B_KV_FULL],
                               tv.h * D + blk * 64, tv.b * args.N + kv * 128);
            }
            ++kv_cnt;
            prev_seg = tv.seg;
          }
          for (int sub = 0; sub < NSUB; ++sub) {
            const int stage = q_cnt % NSTAGE;
            if (q_cnt >= NSTAGE)
              ptx::mbar_wait_u(&bars[B_Q_EMPTY0 + stage], ((q_cnt / NSTAGE) - 1) & 1);
            uint64_t* full = &bars[B_Q_FULL0 + stage];
            if (lane == 0) DASH_TRACE_MARK(10, q_cnt);
            ptx::mbar_arrive_expect_tx_e(full, 2 * C::Q_BYTES + 2 * BR * 4);
            const int row0 = q * 128 + sub * BR;
#pragma unroll
            for (int blk = 0; blk < D / 64; ++blk) {
              ptx::tma_load_2d_e(smem + C::OFF_Q + stage * C::Q_BYTES + blk * BR * 128, &tm_q, full,
                               tv.h * D + blk * 64, tv.b * args.N + row0);
              ptx::tma_load_2d_e(smem + C::OFF_DO + stage * C::Q_BYTES + blk * BR * 128, &tm_do,
                               full, tv.h * D + blk * 64, tv.b * args.N + row0);
            }
            const size_t lo = static_cast<size_t>(tv.bh) * args.N + row0;
            ptx::bulk_load_e(sL + stage * BR, args.lse2 + lo, BR * 4, full);
            ptx::bulk_load_e(sDv + stage * BR, args.Dvec + lo, BR * 4, full);
            ++q_cnt;
          }
        }
        // Every load of job g is issued: claim the next job now -- its claim
        // (an atomic that all CTAs of a SHIFT wave issue together, ~3 k cycles)
        // and its K/V load overlap g's last sub-tiles -- instead of after the
        // last ordered add of g is released (~18 k cycles per job, round 1).
        // Measured (profiles/r02_experiments_early_claim.txt): claiming here
        // beats waiting for g's MMAs (KV_EMPTY) by 1-5 %, once the claim itself
        // is a single atomic.  Deadlock-free: a CTA holds at most one
        // claimed-ahead job, queued behind g; g's remaining adds wait only on
        // jobs of g's head, all claimed earlier.  With cyclic waits inside a
        // head (SHIFT) the claimed-ahead job must belong to another head, so it
        // is never in g's wait cycle; with acyclic waits (NAIVE, DESCENDING:
        // rank = KV index, waits point to earlier-claimed jobs) any job is
        // fine.  Otherwise reducer agent 0 claims as before.
        if (lane == 0) {
          int mode = 2;
          wait_slot_free(it_job);  // slot it_job % 2 / claim_mode slot reusable
          if (ptx::aborted()) {
            // watchdog tripped: publish the terminal job so every role leaves
            job_slot[it_job & 1] = args.total_jobs;
            mode = 1;
          } else if (args.prefetch && !args.cyclic) {
            job_slot[it_job & 1] = atomicAdd(args.job_counter, 1);
            mode = 1;
          } else if (args.prefetch) {
            // cyclic schedule: claim early only outside the current head.  The
            // counter only grows, so once a (possibly stale) read of it lies
            // beyond this head, every later claim does too -- one atomicAdd,
            // no compare-and-swap loop (which serialises all CTAs' claims).
            const int peek = ptx::ld_relaxed(args.job_counter);
            if (peek / args.jobs_per_head != g / args.jobs_per_head) {
              job_slot[it_job & 1] = atomicAdd(args.job_counter, 1);
              mode = 1;
            }
          }
          // decision for job number it_job (the CTA's next job), slot (it_job - 1) % 2
          claim_mode[(it_job - 1) & 1] = mode;
          ptx::mbar_arrive(&bars[B_PF0 + ((it_job - 1) & 1)]);
          if (mode == 1) ptx::mbar_arrive(&bars[B_JOB0 + (it_job & 1)]);
        }
        __syncwarp();
      }
      // Exit: no TMA write may still be in flight when the CTA retires (matters
      // only after a watchdog abort, when consumers stop waiting for loads).
      if (q_cnt > 0) {
        for (uint32_t k = (q_cnt > NSTAGE ? q_cnt - NSTAGE : 0); k < q_cnt; ++k)
          ptx::mbar_wait_bounded(&bars[B_Q_FULL0 + k % NSTAGE], (k / NSTAGE) & 1);
      }
      if (kv_cnt > 0) ptx::mbar_wait_bounded(&bars[B_KV_FULL], (kv_cnt - 1) & 1);
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ==============================
    {  // whole warp converged; elect.sync issues (keeps descriptors uniform)
      uint32_t it_job = 0, kv_cnt = 0, x = 0, acc_cnt = 0;
      // Base descriptors of every smem operand, built once; per-stage/buffer
      // copies differ by a constant offset (in 16-B units) added per use.
      const uint32_t s0 = ptx::smem_u32(smem);
      const uint64_t dK_k = tile_desc<false>(s0 + C::OFF_K, 128);   // K as K-major A
      const uint64_t dK_mn = tile_desc<true>(s0 + C::OFF_K, 128);   // K as MN-major A/B
      const uint64_t dV_k = tile_desc<false>(s0 + C::OFF_V, 128);
      const uint64_t dQ_k = tile_desc<false>(s0 + C::OFF_Q, BR);    // stage 0
      const uint64_t dQ_mn = tile_desc<true>(s0 + C::OFF_Q, BR);
      const uint64_t ddO_k = tile_desc<false>(s0 + C::OFF_DO, BR);
      const uint64_t ddO_mn = tile_desc<true>(s0 + C::OFF_DO, BR);
      const uint64_t ddS_k = tile_desc<false>(s0 + C::OFF_DS, 128);  // buffer 0
      const uint64_t ddS_mn = tile_desc<true>(s0 + C::OFF_DS, 128);
      constexpr uint32_t Q_STEP = C::Q_BYTES / 16, DS_STEP = C::P_BYTES / 16;
      auto issue_sdp = [&](uint32_t xx) {
        const uint32_t st = xx % NSTAGE;
        ptx::mbar_wait_u(&bars[B_Q_FULL0 + st], (xx / NSTAGE) & 1);
        if (xx > 0) ptx::mbar_wait_u(&bars[B_S_EMPTY], (xx - 1) & 1);
        ptx::tc_fence_after();
        if (lane == 0) DASH_TRACE_MARK(0, xx);
        umma_gemm_d<128, BR, D, false, false, 128, BR>(tbase + C::T_S, dK_k, dQ_k + st * Q_STEP,
                                                       false);
        umma_gemm_d<128, BR, D, false, false, 128, BR>(tbase + C::T_DP, dV_k, ddO_k + st * Q_STEP,
                                                       false);
        ptx::mma_commit_e(&bars[B_S_FULL]);
      };
      while (true) {
        ptx::mbar_wait_u(&bars[B_JOB0 + (it_job & 1)], (it_job >> 1) & 1);
        const int g = __shfl_sync(0xffffffffu, job_slot[it_job & 1], 0);
        if (lane == 0) slot_read(it_job);
        ++it_job;
        if (g >= args.total_jobs || __shfl_sync(0xffffffffu, ptx::aborted(), 0)) break;
        const JobView jv = decode_job(args, g);
        const int t1 = __shfl_sync(0xffffffffu, jv.t1, 0);
        int ts = __shfl_sync(0xffffffffu, jv.t0, 0);
        while (ts < t1) {
          // one table load (a scan over the tasks would chain L2 round trips)
          const int te = __shfl_sync(0xffffffffu, args.seg_end[ts], 0);
          const uint32_t nsub = static_cast<uint32_t>(te - ts) * NSUB;
          ptx::mbar_wait_u(&bars[B_KV_FULL], kv_cnt & 1);
          ++kv_cnt;
          ptx::tc_fence_after();
          const uint32_t base = x;
          issue_sdp(base);
          for (uint32_t u = 0; u < nsub; ++u) {
            const uint32_t xx = base + u;
            // S/dP of the next sub-tile go into the tensor pipe while the
            // softmax warps turn this one into P^T / dS^T.
            if (u + 1 < nsub) issue_sdp(xx + 1);
            const uint32_t st = xx % NSTAGE, sb = xx % C::NDS;
            ptx::mbar_wait_u(&bars[B_P_FULL], xx & 1);
            if (lane == 0) DASH_TRACE_MARK(1, xx);
            if (u == 0 && acc_cnt > 0) ptx::mbar_wait_u(&bars[B_ACC_EMPTY], (acc_cnt - 1) & 1);
            ptx::tc_fence_after();
            // dV += P^T dO  (A = P^T straight from TMEM)   (Alg.1 line 25)
            umma_gemm_ts_d<D, BR, true, BR>(tbase + C::T_DV, tbase + C::T_PT, ddO_mn + st * Q_STEP,
                                            u > 0);
            ptx::mma_commit_e(&bars[B_PT_EMPTY]);
            // dK += dS^T Q   (Alg.1 line 26)
            if constexpr (C::DS_IN_TMEM) {
              umma_gemm_ts_d<D, BR, true, BR>(tbase + C::T_DK, tbase + C::T_DST, dQ_mn + st * Q_STEP,
                                              u > 0);
              ptx::mma_commit_e(&bars[B_DST_EMPTY]);
            } else {
              umma_gemm_d<128, D, BR, false, true, 128, BR>(tbase + C::T_DK, ddS_k + sb * DS_STEP,
                                                            dQ_mn + st * Q_STEP, u > 0);
            }
            ptx::mma_commit_e(&bars[B_Q_EMPTY0 + st]);  // Q/dO no longer needed
            if (xx >= 1) {
              ptx::mbar_wait_u(&bars[B_DQ_EMPTY], (xx - 1) & 1);
              ptx::tc_fence_after();
            }
            // dQ_local (Alg.1 line 28)
            if constexpr (D == 128) {
              umma_gemm_d<128, BR, 128, true, true, 128, 128>(tbase + C::T_DQ, dK_mn,
                                                              ddS_mn + sb * DS_STEP, false);
            } else {
              umma_gemm_d<128, D, 128, true, true, 128, 128>(tbase + C::T_DQ, ddS_mn + sb * DS_STEP,
                                                             dK_mn, false);
            }
            if (lane == 0) DASH_TRACE_MARK(2, xx);
            ptx::mma_commit_e(&bars[B_DQ_FULL]);
            ptx::mma_commit_e(&bars[B_DS_EMPTY0 + sb]);
          }
          x = base + nsub;
          ptx::mma_commit_e(&bars[B_KV_EMPTY]);
          ptx::mma_commit_e(&bars[B_ACC_FULL]);
          ++acc_cnt;
          ts = te;
        }
      }
      // Exit: every issued MMA has completed before TMEM is released.
      ptx::mma_commit_e(&bars[B_MMA_DRAIN]);
      ptx::mbar_wait_bounded(&bars[B_MMA_DRAIN], 0);
    }
  } else if (warp == 2 || warp == 3) {
    // ======================== ordered dQ reducers ==========================
    // NAG = 2 single-thread agents (lane 0 of warps 2 and 3), each with its
    // own bulk groups; staging unit x belongs to agent x % NAG, so two ordered
    // adds are in flight.  (Measured: four agents as lanes 0 and 16 of the
    // same two warps are slower -- divergent lanes of one warp do not run
    // concurrently, so a spinning agent stalls its lane-mate.)
    if (lane == 0) {
      const uint32_t agent = static_cast<uint32_t>(warp - 2);
      const bool det = args.deterministic != 0;
      uint32_t it_job = 0, x = 0;
      if (agent == 0) {
        job_slot[0] = atomicAdd(args.job_counter, 1);
        ptx::mbar_arrive(&bars[B_JOB0]);
      }
      while (true) {
        ptx::mbar_wait(&bars[B_JOB0 + (it_job & 1)], (it_job >> 1) & 1);
        const int g = job_slot[it_job & 1];
        slot_read(it_job);
        if (g >= args.total_jobs || ptx::aborted()) break;
        const JobView jv = decode_job(args, g);
        for (int t = jv.t0; t < jv.t1; ++t) {
          const TaskView tv = decode_task(args, jv, args.tasks[t]);
          const int q = tv.q, rank = tv.rank;
          for (int sub = 0; sub < NSUB; ++sub, ++x) {  // x counts staging units (= sub-tiles)
            if ((x % NAG) != agent) continue;
            const uint32_t ph = (x / NAG) & 1;  // this agent's phase on its FULL barriers
            const int urow = q * 128 + sub * BR;  // first Q row of the unit
            const int par = rank % args.split, rank_w = rank / args.split;  // AMB-27
            int* ticket = args.tickets + static_cast<size_t>(par) * args.n_tickets +
                          static_cast<size_t>(tv.bh - args.bh_base) * n_units + urow / C::STG_ROWS;
            if (det) {
              // Wait until the global order grants this block its turn (Alg.1 line 33).
              // Spin with relaxed loads (an acquire per poll would invalidate L1
              // every iteration); one acquire once the turn has come.
              if (ptx::ld_acquire(ticket) != rank_w) {
                const long long t_start = clock64();
                uint32_t polls = 0;
                while (ptx::ld_relaxed(ticket) != rank_w) {
                  __nanosleep(32);
                  if ((++polls & ptx::kAbortPollMask) != 0) continue;  // no extra round trip per poll
                  if (clock64() - t_start > args.spin_bound || ptx::aborted()) {
                    atomicExch(args.error_flag, 1);
                    atomicExch(&ptx::g_dash_abort, 1);
                    break;
                  }
                }
                (void)ptx::ld_acquire(ticket);
              }
              // Order the ticket acquire (generic proxy) before the reduce (async proxy).
              ptx::fence_async_global();
            }
            DASH_TRACE_MARK(7, x);
            // Add dQ_local to dQ (Alg.1 line 34); rank 0 stores (no zero-fill needed).
            // row of dQacc [W][B*H*N, D]
            const int grow = (par * args.bh_count + tv.bh - args.bh_base) * args.N + urow;
            if constexpr (C::LINEAR) {
              // NPART parts, each reduced as soon as the drain has written it;
              // a part is handed back as soon as the bulk engine has read it
              float* dst0 = args.dqacc + static_cast<size_t>(grow) * D;
              constexpr uint32_t HB = C::DQ_BYTES / C::NPART;
#pragma unroll
              for (int hh = 0; hh < C::NPART; ++hh) {
                ptx::mbar_wait(&bars[B_AGF0 + hh * NAG + agent], ph);
                if (hh == C::NPART - 1) DASH_TRACE_MARK(13, x);  // all parts staged
                float* dst = dst0 + hh * (HB / 4);
                const uint8_t* src = smem + C::OFF_DQ + hh * HB;
                if (det && rank_w == 0) ptx::bulk_store(dst, src, HB);
                else ptx::bulk_reduce_add_f32(dst, src, HB);
                ptx::bulk_commit();
                if (hh >= 1) {
                  ptx::bulk_wait_read<1>();  // part hh - 1 read: the drain may refill its slot
                  ptx::mbar_arrive(part_empty(hh - 1));
                }
              }
              DASH_TRACE_MARK(8, x);
              ptx::bulk_wait_read<0>();
              ptx::mbar_arrive(part_empty(C::NPART - 1));
            } else {
              const uint8_t* stg = smem + C::OFF_DQ;
              ptx::mbar_wait(&bars[B_AGF0 + agent], ph);
#pragma unroll
              for (int blk = 0; blk < D / 32; ++blk) {
                if (det && rank_w == 0) {
                  tma_store_2d(&tm_dqacc, stg + blk * C::STG_ROWS * 128, blk * 32, grow);
                } else {
                  tma_reduce_add_2d(&tm_dqacc, stg + blk * C::STG_ROWS * 128, blk * 32, grow);
                }
              }
              ptx::bulk_commit();
              DASH_TRACE_MARK(8, x);
              ptx::bulk_wait_read_all();  // staging may be overwritten from here on
              ptx::mbar_arrive(&bars[B_STG_EMPTY]);
            }
            DASH_TRACE_MARK(11, x);
            ptx::bulk_wait_all();
            DASH_TRACE_MARK(12, x);
            if (det) {
              // Advance the global order (Alg.1 line 35): proxy fence (the
              // reduce wrote through the async proxy) + gpu-scope release.
              // Measured: a relaxed store here is NOT safe -- completion of
              // the bulk group alone does not order the reduce's writes
              // before the flag (tests/test_gpu_bwd.py catches it).
              ptx::fence_async_global();
              ptx::st_release(ticket, rank_w + 1);
            }
            DASH_TRACE_MARK(9, x);
          }
        }
        // Every agent has released every add of this job: only now may the
        // CTA claim its next job (greedy claiming of AMB-7, deadlock-free).
        count_job_done(args, g);
        ptx::mbar_arrive(&bars[B_JOB_DONE]);
        if (agent == 0) {
          ptx::mbar_wait(&bars[B_JOB_DONE], it_job & 1);
          // did the producer already claim job it_job + 1?  (slot it_job % 2)
          ptx::mbar_wait(&bars[B_PF0 + (it_job & 1)], (it_job >> 1) & 1);
          if (claim_mode[it_job & 1] == 2) {
            wait_slot_free(it_job + 1);
            job_slot[(it_job + 1) & 1] =
                ptx::aborted() ? args.total_jobs : atomicAdd(args.job_counter, 1);
            ptx::mbar_arrive(&bars[B_JOB0 + ((it_job + 1) & 1)]);
          }
        }
        ++it_job;
      }
    }
    __syncwarp();
  } else if (warp >= 4 && warp < 4 + 4 * C::NSMX) {
    // ======================= softmax / dS / epilogue ======================
    const int wg = (warp - 4) >> 2;          // column half owned by this warpgroup
    const int row = (warp & 3) * 32 + lane;  // KV row within the tile = TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    constexpr int NC = C::SMX_COLS;
    const int c_base = wg * NC;
    uint32_t it_job = 0, x = 0, acc_cnt = 0;
    while (true) {
      ptx::mbar_wait(&bars[B_JOB0 + (it_job & 1)], (it_job >> 1) & 1);
      const int g = job_slot[it_job & 1];
      __syncwarp();
      if (lane == 0) slot_read(it_job);
      ++it_job;
      if (g >= args.total_jobs || ptx::aborted()) break;
      const JobView jv = decode_job(args, g);
      // The next task's entry is loaded one task ahead: its L2 latency (~700
      // cycles) otherwise sits between two sub-tiles on the softmax's
      // critical path (every sub-tile at d = 64, where a task is one sub-tile).
      int2 tk_cur = args.tasks[jv.t0];
      for (int t = jv.t0; t < jv.t1; ++t) {
        const int2 tk_nxt = (t + 1 < jv.t1) ? args.tasks[t + 1] : make_int2(0, -1);
        const TaskView tv = decode_task(args, jv, tk_cur);
        const int kv = tv.kv, q = tv.q;
        const bool diag = args.causal && (kv == q);
        for (int sub = 0; sub < NSUB; ++sub, ++x) {
          const uint32_t st = x % NSTAGE, sb = x % C::NDS;
          uint8_t* pdS = smem + C::OFF_DS + sb * C::P_BYTES;
          ptx::mbar_wait(&bars[B_S_FULL], x & 1);
          ptx::mbar_wait(&bars[B_Q_FULL0 + st], (x / NSTAGE) & 1);
          ptx::tc_fence_after();
          if (row == 0 && wg == 0) DASH_TRACE_MARK(3, x);
          const float* Lrow = sL + st * BR;
          const float* Drow = sDv + st * BR;
          // NC columns in chunks of 16, software-pipelined: the TMEM loads of
          // chunk ch + 1 are in flight while chunk ch is computed (wait::ld
          // covers every outstanding load, so a chunk's load is issued right
          // after the previous chunk's wait).  The S^T / dP^T columns are all
          // read -- S_EMPTY -- before the last chunk is computed.
          constexpr int CH = 16, NCH = NC / CH;
          float s2[2][CH], dp2[2][CH];
          ptx::tmem_ld16(tbase + lane_off + C::T_S + c_base, s2[0]);
          ptx::tmem_ld16(tbase + lane_off + C::T_DP + c_base, dp2[0]);
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch) {
            const int cur = ch & 1;
            const int cc0 = c_base + ch * CH;  // first Q row (column) of this chunk
            ptx::tmem_wait_ld();
            if (ch + 1 < NCH) {
              ptx::tmem_ld16(tbase + lane_off + C::T_S + cc0 + CH, s2[cur ^ 1]);
              ptx::tmem_ld16(tbase + lane_off + C::T_DP + cc0 + CH, dp2[cur ^ 1]);
            } else {
              ptx::tc_fence_before();
              ptx::mbar_arrive(&bars[B_S_EMPTY]);
            }
            const float* s = s2[cur];
            const float* dp = dp2[cur];
            uint32_t pk[CH / 2], dk2[CH / 2];
            // P = exp2(S*scale*log2e - L*log2e), dS = P o (dP - D), packed to bf16.
            // The causal mask (key row > query row) exists only on the diagonal
            // task; off the diagonal the per-element compare/select is skipped.
            const unsigned long long sc2 = ptx::f2_pack(args.scale_log2, args.scale_log2);
            auto smx = [&](auto masked) {
              constexpr bool MASKED = decltype(masked)::value;
              const int mask_from = row - sub * BR - cc0;  // masked: cols c < mask_from
#pragma unroll
              for (int c4 = 0; c4 < CH / 4; ++c4) {
                const float4 l4 = *reinterpret_cast<const float4*>(Lrow + cc0 + c4 * 4);
                const float4 d4 = *reinterpret_cast<const float4*>(Drow + cc0 + c4 * 4);
                const float Lv[4] = {l4.x, l4.y, l4.z, l4.w};
                const float Dv[4] = {d4.x, d4.y, d4.z, d4.w};
                float p[4], ds[4];
                // pairs of columns in packed fp32 (FFMA2 / FADD2 / FMUL2): the
                // same roundings as fmaf(s, scale, L), dp - D, P * (.)
#pragma unroll
                for (int e = 0; e < 4; e += 2) {
                  const int c = c4 * 4 + e;
                  float t0, t1;
                  ptx::f2_unpack(ptx::f2_fma(ptx::f2_pack(s[c], s[c + 1]), sc2,
                                             ptx::f2_pack(Lv[e], Lv[e + 1])), t0, t1);
                  float p0 = fast_exp2(t0), p1 = fast_exp2(t1);
                  if constexpr (MASKED) {
                    if (c < mask_from) p0 = 0.f;
                    if (c + 1 < mask_from) p1 = 0.f;
                  }
                  p[e] = p0;
                  p[e + 1] = p1;
                  ptx::f2_unpack(ptx::f2_mul(ptx::f2_pack(p0, p1),
                                             ptx::f2_sub(ptx::f2_pack(dp[c], dp[c + 1]),
                                                         ptx::f2_pack(Dv[e], Dv[e + 1]))),
                                 ds[e], ds[e + 1]);
                }
                pk[c4 * 2] = pack_bf16(p[0], p[1]);
                pk[c4 * 2 + 1] = pack_bf16(p[2], p[3]);
                dk2[c4 * 2] = pack_bf16(ds[0], ds[1]);
                dk2[c4 * 2 + 1] = pack_bf16(ds[2], ds[3]);
              }
            };
            if (diag) smx(std::true_type{});
            else smx(std::false_type{});
            // P^T -> TMEM once dV of sub-tile x - 1 consumed it.
            if (ch == 0 && x >= 1) ptx::mbar_wait(&bars[B_PT_EMPTY], (x - 1) & 1);
            ptx::tmem_st8(tbase + lane_off + C::T_PT + cc0 / 2, pk);
            if constexpr (C::DS_IN_TMEM) {
              // dS^T -> TMEM (A operand of the dK TS-MMA) once dK of x - 1 consumed it.
              if (ch == 0 && x >= 1) ptx::mbar_wait(&bars[B_DST_EMPTY], (x - 1) & 1);
              ptx::tmem_st8(tbase + lane_off + C::T_DST + cc0 / 2, dk2);
            }
            // dS^T -> smem buffer sb once dK, dQ of sub-tile x - NDS consumed it.
            if (ch == 0 && x >= C::NDS)
              ptx::mbar_wait(&bars[B_DS_EMPTY0 + sb], ((x / C::NDS) - 1) & 1);
#pragma unroll
            for (int c8 = 0; c8 < CH / 8; ++c8) {
              const uint32_t off = sw128_chunk_offset(128, row, (cc0 + c8 * 8) >> 3);
              *reinterpret_cast<uint4*>(pdS + off) =
                  make_uint4(dk2[c8 * 4], dk2[c8 * 4 + 1], dk2[c8 * 4 + 2], dk2[c8 * 4 + 3]);
            }
          }
          ptx::tmem_wait_st();
          ptx::tc_fence_before();
          ptx::fence_async_smem();
          ptx::mbar_arrive(&bars[B_P_FULL]);
          if (row == 0 && wg == 0) DASH_TRACE_MARK(4, x);
        }
        // End of a KV segment: dK/dV epilogue (local reduction done).
        const bool seg_end = (t + 1 == jv.t1) || (task_seg(tk_nxt) != tv.seg);
        if (seg_end) {
          ptx::mbar_wait(&bars[B_ACC_FULL], acc_cnt & 1);
          ++acc_cnt;
          ptx::tc_fence_after();
          // dK, dV rows of this warp (32 KV rows x this warpgroup's columns) go
          // out through TMA stores of 32 x 32 bf16 boxes staged in the warp's
          // 4 KB of the dS^T buffers: free here -- ACC_FULL follows every MMA
          // of the segment -- and rewritten only by these warps after the
          // named barrier below (generic stores of one 16 B piece per row per
          // lane are LSU-bound and slow the reducers' release fences).
          uint8_t* ep = smem + C::OFF_DS + (warp - 4) * 4096;
          const int grow0 = tv.b * args.N + kv * 128 + (warp & 3) * 32;
#pragma unroll 1
          for (int c0 = wg * (D / C::NSMX); c0 < (wg + 1) * (D / C::NSMX); c0 += 32) {
            float a[32], k2[32];
            ptx::tmem_ld32(tbase + lane_off + C::T_DV + c0, a);
            ptx::tmem_ld32(tbase + lane_off + C::T_DK + c0, k2);
            ptx::tmem_wait_ld();
            if (c0 != wg * (D / C::NSMX)) {  // the previous chunk's boxes have been read
              if (lane == 0) ptx::bulk_wait_read<0>();
              __syncwarp();
            }
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
              *reinterpret_cast<uint4*>(ep + lane * 64 + e * 2) = pv;
              *reinterpret_cast<uint4*>(ep + 2048 + lane * 64 + e * 2) = pk;
            }
            ptx::fence_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&tm_dv, ep, tv.h * D + c0, grow0);
              tma_store_2d(&tm_dk, ep + 2048, tv.h * D + c0, grow0);
              ptx::bulk_commit();
            }
          }
          ptx::tc_fence_before();
          if (lane == 0) ptx::bulk_wait_read<0>();
          __syncwarp();
          ptx::mbar_arrive(&bars[B_ACC_EMPTY]);
          // every warp's staging has been read before any warp writes dS^T again
          ptx::named_bar_sync(1, 128 * C::NSMX);
        }
        tk_cur = tk_nxt;
      }
    }
    if (lane == 0) ptx::bulk_wait_all();  // dK / dV stores complete before the CTA retires
    __syncwarp();
  } else {
    // ================== dQ drain: TMEM -> fp32 staging ==================
    const int tl = (warp & 3) * 32 + lane;  // TMEM lane
    const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
    uint32_t it_job = 0, x = 0;
    while (true) {
      ptx::mbar_wait(&bars[B_JOB0 + (it_job & 1)], (it_job >> 1) & 1);
      const int g = job_slot[it_job & 1];
      __syncwarp();
      if (lane == 0) slot_read(it_job);
      ++it_job;
      if (g >= args.total_jobs || ptx::aborted()) break;
      const JobView jv = decode_job(args, g);
      const int nx = (jv.t1 - jv.t0) * NSUB;
      for (int u = 0; u < nx; ++u, ++x) {
        ptx::mbar_wait(&bars[B_DQ_FULL], x & 1);
        ptx::tc_fence_after();
        if (tl == 0) DASH_TRACE_MARK(5, x);
        float v[64];
        ptx::tmem_ld32(tbase + lane_off + C::T_DQ, *reinterpret_cast<float(*)[32]>(v));
        ptx::tmem_ld32(tbase + lane_off + C::T_DQ + 32, *reinterpret_cast<float(*)[32]>(v + 32));
        ptx::tmem_wait_ld();
        ptx::tc_fence_before();
        ptx::mbar_arrive(&bars[B_DQ_EMPTY]);
        if (args.dump) {
          // verification: the partial of (KV tile kv, these Q rows) -> dump[bh][kv][row][:]
          const TaskView tv = decode_task(args, jv, args.tasks[jv.t0 + u / NSUB]);
          const int urow0 = tv.q * 128 + (u % NSUB) * BR;
          float* dp = args.dump + ((static_cast<size_t>(tv.bh) * (args.N / 128) + tv.kv) *
                                       args.N + urow0) * D;
          if constexpr (D == 128) {  // lane tl = d index, v[c] = Q row c
#pragma unroll
            for (int c = 0; c < BR; ++c) dp[c * D + tl] = v[c];
          } else {  // lane tl = Q row, v[c] = d column c
#pragma unroll
            for (int c = 0; c < 64; ++c) dp[tl * D + c] = v[c];
          }
        }
        uint8_t* stg0 = smem + C::OFF_DQ;
        const uint32_t y = x;  // staging unit (one per sub-tile)
        if constexpr (C::LINEAR) {
          // row-major [STG_ROWS][128] fp32 in NPART parts; lane tl = d index, v[c] = Q row c
          constexpr int HR = C::STG_ROWS / C::NPART;
#pragma unroll
          for (int hh = 0; hh < C::NPART; ++hh) {
            if (y >= 1) ptx::mbar_wait(part_empty(hh), (y - 1) & 1);
            float* dst = reinterpret_cast<float*>(stg0 + hh * (C::DQ_BYTES / C::NPART));
#pragma unroll
            for (int c = hh * HR; c < (hh + 1) * HR; ++c) dst[(c - hh * HR) * 128 + tl] = v[c];
            ptx::fence_async_smem();
            ptx::mbar_arrive(&bars[B_AGF0 + hh * NAG + (y % NAG)]);
          }
        } else {
          if (y >= 1) ptx::mbar_wait(&bars[B_STG_EMPTY], (y - 1) & 1);
          // Stage the partial as SW128 boxes of 32 fp32 columns:
          // lane tl = Q row, v[c] = d column c.
          const int r = tl;
#pragma unroll
          for (int cc = 0; cc < 16; ++cc) {
            const int blk = cc >> 3, chunk = cc & 7;
            const uint32_t off = blk * C::STG_ROWS * 128 + r * 128 + ((chunk ^ (r & 7)) << 4);
            *reinterpret_cast<float4*>(stg0 + off) =
                make_float4(v[cc * 4], v[cc * 4 + 1], v[cc * 4 + 2], v[cc * 4 + 3]);
          }
          ptx::fence_async_smem();
          ptx::mbar_arrive(&bars[B_AGF0 + (y % NAG)]);
        }
        if (tl == 0) DASH_TRACE_MARK(6, x);
        if (tl == 96) DASH_TRACE_MARK(14, x);  // last drain warp done staging
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tbase);
  }
  if (args.fuse_dq) finalize_dq<D, C::NTHREADS>(args, reinterpret_cast<int*>(smem + C::OFF_DQ));
  if (tid == 0 && ptx::aborted()) atomicExch(args.error_flag, 2);
}

// floor(n / d) for 0 <= n < 2^31 by one 64-bit multiply and shift (d fixed per
// launch): m = ceil(2^s / d) with s = 32 + ceil(log2 d) is exact on that range.
// The preprocess / convert kernels spend most of their issue slots on the
// (b, n, h) <-> (b, h, n) index maps otherwise (64-bit divisions).
struct FastDiv {
  uint64_t m;
  uint32_t s, d;
  __host__ static FastDiv make(uint32_t d) {
    uint32_t l = 0;
    while ((1ull << l) < d) ++l;
    FastDiv f;
    f.s = 32 + l;
    f.m = ((1ull << f.s) + d - 1) / d;
    f.d = d;
    return f;
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    return static_cast<uint32_t>((static_cast<uint64_t>(n) * m) >> s);
  }
};

// K1: D = rowsum(dO o O) (Alg.1 line 1; D in R^N per AMB-2), fp32 in a
// fixed order, and lse2 = -L * log2(e) for the exp2 form of P = exp(S - L);
// also resets tickets / job counter / error flag and (atomic variant only)
// zero-fills the dQ accumulator.  HBM-bound: rows are visited in memory order
// ([B, N, H, d]: one (b, n) covers H * d * 2 contiguous bytes -- measured 30 %
// faster than (b, h, n) order, whose 256-B rows lie 4 KB apart), T = d / 8
// threads per row with 16 B streaming loads each, two rows per thread and
// iteration (four loads in flight), grid-stride over a one-wave grid.
template <int D, int KR>
__global__ void __launch_bounds__(256) dash_preprocess_kernel(
    const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dout,
    const float* __restrict__ lse, float* __restrict__ Dvec, float* __restrict__ lse2, int B, int N,
    int H, FastDiv fN, FastDiv fH, int* __restrict__ zero_i32, int n_zero_i32,
    float4* __restrict__ zero_f32, size_t n_zero_f4, int* __restrict__ counters, int poison) {
  constexpr int T = D / 8;      // threads per row, 16 B each
  constexpr int RPB = 256 / T;  // rows per block and half-iteration
  ptx::griddep_wait();    // the previous call's kernels may still read this workspace
  ptx::griddep_launch();  // the main kernel's prologue may start on SMs this grid leaves
  const size_t rows = static_cast<size_t>(B) * N * H;
  const int part = static_cast<int>(threadIdx.x % T);
  auto row_addr = [&](size_t r) { return r * D + part * 8; };  // r = (b*N + n)*H + h
  auto vec_idx = [&](size_t r) {  // -> (b*H + h)*N + n, the index of D / lse2 / L
    const uint32_t r32 = static_cast<uint32_t>(r);  // rows < 2^31 (dash_api.cu)
    const uint32_t bn = fH.div(r32), b = fN.div(bn);
    return (static_cast<size_t>(b) * H + (r32 - bn * H)) * N + (bn - b * N);
  };
  auto dot = [](uint4 a, uint4 c) {
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
    return acc;
  };
  for (size_t base = static_cast<size_t>(blockIdx.x) * KR * RPB; base < rows;
       base += static_cast<size_t>(gridDim.x) * KR * RPB) {
    uint4 av[KR], cv[KR];
#pragma unroll
    for (int u = 0; u < KR; ++u) {  // every row's loads in flight together
      const size_t r = base + threadIdx.x / T + u * RPB;
      av[u] = cv[u] = make_uint4(0, 0, 0, 0);
      if (r < rows) {
        av[u] = __ldcs(reinterpret_cast<const uint4*>(o + row_addr(r)));
        cv[u] = __ldcs(reinterpret_cast<const uint4*>(dout + row_addr(r)));
      }
    }
#pragma unroll
    for (int u = 0; u < KR; ++u) {
      const size_t r = base + threadIdx.x / T + u * RPB;
      float sd = dot(av[u], cv[u]);
#pragma unroll
      for (int m = T / 2; m >= 1; m >>= 1) sd += __shfl_xor_sync(0xffffffffu, sd, m);
      if (part == 0 && r < rows) {
        const size_t i = vec_idx(r);
        Dvec[i] = sd;
        lse2[i] = -lse[i] * 1.4426950408889634f;
      }
    }
  }
  const size_t gtid = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const size_t nthreads = static_cast<size_t>(gridDim.x) * blockDim.x;
  if (gtid == 0) {
    counters[0] = 0;  // job counter
    counters[1] = 0;  // error flag (dash_check_workspace reports this call only)
    ptx::g_dash_abort = 0;
  }
  // tickets := 0; `poison` != 0 (fault injection, dash_attn_bwd_inject_fault
  // only) presets the first ticket to a value no add ever reaches.
  for (size_t i = gtid; i < static_cast<size_t>(n_zero_i32); i += nthreads)
    zero_i32[i] = (i == 0) ? poison : 0;
  for (size_t i = gtid; i < n_zero_f4; i += nthreads) zero_f32[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}

// K4: dQ = bf16(scale * dQacc), [chunk heads, N, d] fp32 -> [B,N,H,d] bf16.  With
// W interleaved accumulators (AMB-27) the sum is ((acc_0 + acc_1) + acc_2) + ...
// (fp32, in index order) over the min(W, cnt) accumulators a Q tile (of
// `tile` = 128 or 256 rows) with cnt contributions has written (causal: tile j
// has j + 1).  HBM-bound: W is a template parameter so every plane's loads of
// two 8-element pieces per thread are in flight together (streaming loads, a
// one-wave grid-stride grid).
template <int D, int W>
__global__ void __launch_bounds__(256) dash_dq_convert_kernel(
    const float* __restrict__ acc, __nv_bfloat16* __restrict__ dq, int N, int H, FastDiv fN,
    FastDiv fH, float scale, int causal, int tile, int bh_base, int bh_count) {
  constexpr int T = D / 8;
  ptx::griddep_wait();  // every ordered add of the main kernel has landed
  ptx::griddep_launch();
  const size_t total = static_cast<size_t>(bh_count) * N * T;
  const size_t plane = static_cast<size_t>(bh_count) * N * D;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i0 = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i0 < total;
       i0 += 2 * stride) {
    float4 x[2][W][2];
    int planes[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const size_t i = i0 + u * stride;
      planes[u] = 0;
      if (i < total) {
        const uint32_t r = static_cast<uint32_t>(i / T);  // (local head)*N + n
        const int n = static_cast<int>(r - fN.div(r) * N);
        const int cnt = causal ? n / tile + 1 : N / tile;  // contributions to this row's Q tile
        planes[u] = W < cnt ? W : cnt;  // accumulator w holds ranks w, w + W, ...
        const float* src = acc + r * D + (i % T) * 8;
#pragma unroll
        for (int w = 0; w < W; ++w) {
          if (w < planes[u]) {
            x[u][w][0] = __ldcs(reinterpret_cast<const float4*>(src + w * plane));
            x[u][w][1] = __ldcs(reinterpret_cast<const float4*>(src + w * plane + 4));
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      if (planes[u] == 0) continue;
      const size_t i = i0 + u * stride;
      float4 s0 = x[u][0][0], s1 = x[u][0][1];
#pragma unroll
      for (int w = 1; w < W; ++w) {
        if (w < planes[u]) {
          s0 = make_float4(s0.x + x[u][w][0].x, s0.y + x[u][w][0].y, s0.z + x[u][w][0].z,
                           s0.w + x[u][w][0].w);
          s1 = make_float4(s1.x + x[u][w][1].x, s1.y + x[u][w][1].y, s1.z + x[u][w][1].z,
                           s1.w + x[u][w][1].w);
        }
      }
      const uint32_t r = static_cast<uint32_t>(i / T);
      const uint32_t lh = fN.div(r);
      const int n = static_cast<int>(r - lh * N);
      const uint32_t bh = bh_base + lh;
      const int b = static_cast<int>(fH.div(bh));
      const int h = static_cast<int>(bh - b * H);
      uint4 out;
      out.x = pack_bf16(s0.x * scale, s0.y * scale);
      out.y = pack_bf16(s0.z * scale, s0.w * scale);
      out.z = pack_bf16(s1.x * scale, s1.y * scale);
      out.w = pack_bf16(s1.z * scale, s1.w * scale);
      *reinterpret_cast<uint4*>(dq + ((static_cast<size_t>(b) * N + n) * H + h) * D + (i % T) * 8) =
          out;
    }
  }
}

}  // namespace dash
