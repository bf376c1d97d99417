// libdash.so C ABI (include/dash.h): validation, workspace layout, TMA
// descriptors, schedule-table cache and kernel launches.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <map>
#include <set>
#include <mutex>
#include <tuple>
#include <vector>

#include "bwd.cuh"
#include "bwd2.cuh"
#include "dash.h"
#include "fwd_tc.cuh"
#include "schedule.h"

#define DASH_API extern "C" __attribute__((visibility("default")))

namespace dash {
namespace {

constexpr size_t kAlign = 1024;
// Interleaved dQ accumulators (AMB-27): 0 = automatic (the default), else
// fixed W in {1, 2, 4, 8}; DASH_ACC_SPLIT overrides the default at load time.
int g_acc_split = [] {
  const char* e = std::getenv("DASH_ACC_SPLIT");
  const int v = e ? std::atoi(e) : 0;
  return (v == 1 || v == 2 || v == 4 || v == 8) ? v : 0;
}();
int acc_split() { return g_acc_split; }
// DASH_SCHED_AUTO: the paper's schedule that measured fastest on B200 for
// this (mask, n, d) with the automatic accumulator split (bench sweeps in
// profiles/README.md): SHIFT while heads are short (n <= 32 tiles: whole heads
// fit the 148 SMs several times over); for longer causal heads DESCENDING
// (d = 128 from n = 64, d = 64 from n = 128), for longer full-mask heads
// NAIVE, whose dependencies all point to earlier-claimed jobs, so partially
// co-scheduled heads never stall (with W = 4 its remaining chain cost is gone).
int auto_schedule(const dash_shape* s, int causal) {
  const int n = s->seqlen / 128;
  if (n <= 32) return kShift;
  if (causal) return (n >= 128 || (s->head_dim == 128 && n >= 64)) ? kDescending : kShift;
  return kNaive;
}

// W actually used for a problem with n 128-row tiles per head.  Automatic:
// W = 4 once the per-tile chain is long (n >= 64), W = 8 from n >= 256
// (N >= 32k), else 2 -- measured on B200 (profiles/r01_experiments/acc_split.txt,
// acc_split_w8.txt): extra accumulators cost the convert kernel one more fp32
// read each, which only pays off at long sequences.  Depends on n only, so
// (b, h) sharding never changes it.
// The CTA-pair kernel (256-row tiles, n' = N / 256 per head) measured on B200
// (profiles/r02_acc_split_pair.txt): W = 1 -- the paper's single ordered
// accumulator -- is fastest up to n' = 8 (its dQ partials already cover 256
// KV rows, so the chain is short), 2 up to n' = 16, 4 below n' = 128, 8 above.
int acc_split_for(int n, int tile = 128) {
  if (g_acc_split) return g_acc_split;
  if (tile == 256) return n <= 8 ? 1 : n <= 16 ? 2 : n < 128 ? 4 : 8;
  return n >= 256 ? 8 : n >= 64 ? 4 : 2;
}
size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Entry of every launching ABI call.  A thread that has not used the CUDA
// runtime yet (e.g. PyTorch's autograd worker) may have no current context;
// the TMA tensor-map encoder validates addresses against the current context
// and fails without one, so make the device's primary context current
// (cudaSetDevice does, CUDA >= 12).  Also drops an error left in this thread
// by someone else's CUDA call, so DASH_ERR_CUDA reports only this call.
void bind_context() {
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaSetDevice(dev);
  (void)cudaGetLastError();
}

// Last CUDA error behind a DASH_ERR_CUDA of this thread (dash_last_cuda_error).
thread_local int g_last_cuda = 0;
dash_status cuda_fail(cudaError_t e) {
  g_last_cuda = static_cast<int>(e);
  return DASH_ERR_CUDA;
}
dash_status cuda_check_last() {
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? DASH_OK : cuda_fail(e);
}

// Head grouping G (bwd.cuh BwdArgs::head_group): a job covers its KV tile(s)
// in G consecutive (b, h) heads, paying the per-job claim / refill once per G
// heads; the heads' own schedules are untouched, so G never changes a bit
// (tests pass bit-exact under forced G = 2, 4).  Measured
// (profiles/r01_experiments/head_group.txt): it speeds up NAIVE at short
// sequences (+5-10 %) but not SHIFT or DESCENDING -- their per-job tail is
// the ordered-reduction pipeline draining, which grouping does not shorten --
// so the default is G = 1; DASH_HEAD_GROUP forces G (experiments).
int head_group_for(const dash_shape* s) {
  static const int forced = [] {
    const char* e = std::getenv("DASH_HEAD_GROUP");
    return e ? std::atoi(e) : 0;
  }();
  const int bh = s->batch * s->heads;
  if (forced >= 1 && forced <= 8 && bh % forced == 0) return forced;
  return 1;
}

// Early claim of the next job (AMB-28(a); the producer claims once the
// current job's MMAs have completed, before its last ordered adds are
// released; for SHIFT only a job of another head).  Measured per schedule and
// kernel (profiles/r02_experiments_early_claim.txt, both head dims, both
// masks): it pays for SHIFT everywhere (-3 to -13 %), for DESCENDING on the
// pair kernel and with the full mask, for NAIVE with the full mask, and for
// the atomic variant; it costs up to 2-3x for causal NAIVE (the staircase: a
// claimed job queued behind its CTA's reduction tail stalls the next head's
// chain) unless a head has at most 2 jobs (-18 % there), and for causal
// DESCENDING on the single-CTA kernel below W = 4.
// DASH_EARLY_CLAIM = 0 / 1 forces it off / on (experiments; bit-exact either way).
int early_claim(int schedule, int causal, int deterministic, int W, bool pair, int jobs_per_head) {
  static const int forced = [] {
    const char* e = std::getenv("DASH_EARLY_CLAIM");
    return e ? std::atoi(e) : -1;
  }();
  if (forced == 0 || forced == 1) return forced;
  if (!deterministic || schedule == kShift) return 1;
  if (schedule == kDescending) return (pair || !causal || W >= 4) ? 1 : 0;
  return (!causal || jobs_per_head <= 2) ? 1 : 0;  // NAIVE
}

bool shape_ok(const dash_shape* s) {
  if (!s) return false;
  if (s->batch < 1 || s->heads < 1 || s->seqlen < 128 || s->seqlen % 128) return false;
  if (s->head_dim != 64 && s->head_dim != 128) return false;
  if (s->seqlen / 128 > 32767) return false;
  // rows B*N*H index 32-bit maps in K1 / K4 (FastDiv)
  if (static_cast<int64_t>(s->batch) * s->seqlen * s->heads >= (int64_t(1) << 31)) return false;
  return true;
}
bool aligned16(const void* p) { return p && (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
float eff_scale(const dash_shape* s) {
  return s->softmax_scale > 0.f ? s->softmax_scale : 1.0f / std::sqrt(static_cast<float>(s->head_dim));
}
// Schedule tile size (AMB-11 / AMB-31): 256 (the CTA-pair kernel, bwd2.cuh)
// at d = 128 when N is a multiple of 256, else 128 (the single-CTA kernel);
// dash_attn_bwd_set_tile(128) forces the single-CTA kernel.
int g_tile = [] {
  const char* e = std::getenv("DASH_TILE");
  const int v = e ? std::atoi(e) : 0;
  return (v == 128 || v == 256) ? v : 0;
}();
int auto_schedule(const dash_shape* s, int causal);
int pair_cluster_bound() {  // CTA pairs co-resident on the current device
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 74;
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 2)
    return 74;
  return n / 2;
}
// `schedule` already resolved (not AUTO).  Automatic: the pair kernel from N =
// 4096 (full mask: 2048) -- below, the single-CTA kernel measured faster
// (profiles/r02_experiments_tile.txt: more, shorter jobs on 148 CTAs; e.g.
// causal SHIFT 172 vs 193 us at N = 512).  SHIFT needs a head's jobs
// co-resident (AMB-12): with 256-row tiles that is min(n', 128) CTA pairs for
// the full mask, ceil(n'/2) for causal -- beyond the device's pairs the
// single-CTA kernel (128-row tiles, up to 148 co-resident CTAs) runs instead.
int tile_for(const dash_shape* s, int causal, int schedule) {
  const bool pair_ok = s->head_dim == 128 && s->seqlen % PairCfg::TILE == 0;
  if (g_tile == 128 || !pair_ok) return 128;
  if (g_tile == 0 && s->seqlen < (causal ? 4096 : 2048)) return 128;
  if (schedule == kShift) {
    const ScheduleTable* t = cached_schedule(kShift, s->seqlen / PairCfg::TILE, causal ? kCausal : kFull);
    if (!t || t->coresident > pair_cluster_bound()) return 128;
  }
  return 256;
}

// One ticket per (accumulator, b, h, Q sub-tile of 64 / 128 rows) -- and per d
// half for the pair kernel; sized for the largest use at this head dim.
size_t tickets_per_head(int d, int N) { return d == 128 ? 2 * (N / 64) : N / 128; }

// W the backward uses: the setting (automatic: per n) when deterministic, one
// accumulator for the atomic variant.  Resolved once per call and passed to
// both the main kernel and the convert kernel.
int tile_for(const dash_shape* s, int causal, int schedule);
int auto_schedule(const dash_shape* s, int causal);
int resolve_sched(const dash_shape* s, int causal, int schedule) {
  return schedule == DASH_SCHED_AUTO ? auto_schedule(s, causal) : schedule;
}
int resolved_split(const dash_shape* s, int deterministic, int causal, int schedule) {
  if (!deterministic) return 1;
  const int tile = tile_for(s, causal, resolve_sched(s, causal, schedule));
  return acc_split_for(s->seqlen / tile, tile);
}

// dQ-plane budget (dash_attn_bwd_set_plane_budget): the W fp32 accumulators
// of all B*H heads take W * B*H*N*d*4 bytes -- 32 GiB at config 4 (B = 8,
// H = 32, N = 32k, d = 128, W = 8).  When that exceeds the budget the heads
// are processed in chunks of `chunk` consecutive flattened heads that reuse
// one set of planes (BwdArgs::bh_base / bh_count).  A chunk is a (b, h) shard:
// the per-head schedules, ranks and accumulation order are unchanged, so the
// results are bit-identical for every budget.
constexpr size_t kDefaultPlaneBudget = size_t(4) << 30;
size_t g_plane_budget = kDefaultPlaneBudget;

struct WsLayout {
  size_t dqacc = 0, dvec = 0, lse2 = 0, tickets = 0, done = 0, counters = 0, total = 0;
  size_t n_done = 0;  // fused dQ finalise: job-group completion counts + the task counter
  size_t dqacc_bytes = 0, n_tickets = 0;  // per accumulator, for one chunk of heads
  int planes = 1;
  int chunk = 1, chunks = 1;  // heads per chunk, number of chunks
};
// W interleaved fp32 accumulators (AMB-27), each with its own ticket set:
// dqacc [W][chunk heads, N, d], tickets [W][chunk heads][N / ticket_rows]; D
// and -L*log2(e) for all heads.  The accumulators come first (offset 0), so a
// verification test can read them back.  `G` = head grouping (chunks are
// multiples of it).
WsLayout ws_layout(const dash_shape* s, int W, int G = 1) {
  WsLayout w;
  w.planes = W;
  const int BH = s->batch * s->heads;
  const size_t per_head = static_cast<size_t>(W) * s->seqlen * s->head_dim * 4;
  size_t c = g_plane_budget / per_head;
  c = c / G * G;
  if (c < static_cast<size_t>(G)) c = G;
  w.chunk = c >= static_cast<size_t>(BH) ? BH : static_cast<int>(c);
  w.chunks = (BH + w.chunk - 1) / w.chunk;
  const size_t BHN = static_cast<size_t>(BH) * s->seqlen;
  w.dqacc_bytes = static_cast<size_t>(w.chunk) * s->seqlen * s->head_dim * 4;
  w.n_tickets = static_cast<size_t>(w.chunk) * tickets_per_head(s->head_dim, s->seqlen);
  size_t off = 0;
  w.dqacc = off;
  off = align_up(off + static_cast<size_t>(W) * w.dqacc_bytes, kAlign);
  w.dvec = off;
  off = align_up(off + BHN * 4, kAlign);
  w.lse2 = off;
  off = align_up(off + BHN * 4, kAlign);
  w.tickets = off;
  // done[] follows the tickets directly: K1 and reset_chunk zero both in one range
  w.done = off + static_cast<size_t>(W) * w.n_tickets * 4;
  w.n_done = static_cast<size_t>(w.chunk) + 1;
  off = align_up(w.done + w.n_done * 4, kAlign);
  w.counters = off;  // [0] job counter, [1] error flag (directly after done[])
  off = align_up(off + 64, kAlign);
  w.total = off;
  return w;
}

// The layout a call with these arguments uses (schedule may be AUTO).
WsLayout layout_for(const dash_shape* s, int deterministic, int causal, int schedule) {
  const int sch = resolve_sched(s, causal, schedule);
  const int G = tile_for(s, causal, sch) == PairCfg::TILE ? 1 : head_group_for(s);
  return ws_layout(s, resolved_split(s, deterministic, causal, schedule), G);
}

// dQ finalise (dash_attn_bwd_set_fused_dq): 0 = the separate K4 convert, 1 =
// in the main kernel from N = 2048 (default), 2 = always in the main kernel.
// Both form the same sums.  The in-kernel finalise runs on CTAs whose jobs ran
// out, so it hides in the kernel's tail; heads shorter than 2048 rows have
// short jobs and little tail, and there K4 (2048 threads per SM against the
// main kernel's 512) measured faster (profiles/r02_experiments_fused_dq.txt).
int g_fused_dq = 1;
bool fused_for(const dash_shape* s) {
  return g_fused_dq == 2 || (g_fused_dq == 1 && s->seqlen >= 2048);
}

// Ticket-wait watchdog (clock64 cycles): default ~35 s at 1.965 GHz.
long long g_spin_bound = 8 * ptx::kWatchdogCycles;
// Fault injection for the watchdog test (dash_attn_bwd_inject_fault): the
// value the first ticket is preset to by the next backward on this thread.
thread_local int g_poison = 0;

// cudaFuncSetAttribute is per device: remember which (device, kernel) pairs
// already have the large dynamic shared-memory limit.
bool ensure_smem_attr(const void* kern, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({dev, kern})) return true;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess)
    return false;
  done.insert({dev, kern});
  return true;
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

bool make_map_2d(CUtensorMap* m, CUtensorMapDataType dt, int esize, const void* base,
                 uint64_t inner, uint64_t outer, uint32_t box_inner, uint32_t box_outer,
                 CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * static_cast<uint64_t>(esize)};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  return enc(m, dt, 2, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int device_sms(int dev) {
  static std::mutex mu;
  static std::map<int, int> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  cache[dev] = n;
  return n;
}

// Device-resident schedule tables, uploaded once per (device, key).
struct DevTable {
  int* job_begin = nullptr;
  int2* tasks = nullptr;
  int* seg_end = nullptr;  // per task: first task of the next KV segment of its job
  int jobs = 0;
};
// With head grouping G (BwdArgs::head_group) job lj lists the tasks of the
// per-head job lj once per head of the group, head offset in task.y's high half.
const DevTable* device_table(int dev, const ScheduleTable* t, int G) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int, int, int>, DevTable> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_tuple(dev, t->schedule, t->n, t->mask, G);
  auto it = cache.find(key);
  if (it != cache.end()) return &it->second;
  std::vector<int> jb(1, 0);
  std::vector<int2> tk;
  tk.reserve(t->tasks.size() * G);
  for (int lj = 0; lj < t->jobs; ++lj) {
    for (int hoff = 0; hoff < G; ++hoff)
      for (int i = t->job_begin[lj]; i < t->job_begin[lj + 1]; ++i)
        tk.push_back(make_int2(t->tasks[i].kv | (t->tasks[i].q << 16),
                               t->tasks[i].rank | (hoff << 16)));
    jb.push_back(static_cast<int>(tk.size()));
  }
  // Segment ends: a KV segment is a maximal run of tasks with the same (kv,
  // head offset) -- the kernels' task_seg(); the kernels read te here instead
  // of scanning the tasks.
  std::vector<int> se(tk.size());
  for (int lj = 0; lj < t->jobs; ++lj) {
    const int b = jb[lj], e = jb[lj + 1];
    for (int i = e - 1; i >= b; --i) {
      const auto seg = [&](int k) {
        return (tk[k].x & 0xFFFF) | (tk[k].y & static_cast<int>(0xFFFF0000u));
      };
      se[i] = (i + 1 < e && seg(i + 1) == seg(i)) ? se[i + 1] : i + 1;
    }
  }
  DevTable d;
  d.jobs = t->jobs;
  void* buf = nullptr;
  const size_t jb_bytes = align_up(jb.size() * sizeof(int), 256);
  const size_t tk_bytes = align_up(tk.size() * sizeof(int2), 256);
  if (cudaMalloc(&buf, jb_bytes + tk_bytes + se.size() * sizeof(int)) != cudaSuccess) return nullptr;
  d.job_begin = static_cast<int*>(buf);
  d.tasks = reinterpret_cast<int2*>(static_cast<char*>(buf) + jb_bytes);
  d.seg_end = reinterpret_cast<int*>(static_cast<char*>(buf) + jb_bytes + tk_bytes);
  cudaMemcpy(d.job_begin, jb.data(), jb.size() * sizeof(int), cudaMemcpyHostToDevice);
  cudaMemcpy(d.tasks, tk.data(), tk.size() * sizeof(int2), cudaMemcpyHostToDevice);
  cudaMemcpy(d.seg_end, se.data(), se.size() * sizeof(int), cudaMemcpyHostToDevice);
  cache[key] = d;
  return &cache[key];
}

// Optional in-kernel clock64 trace (dash_attn_bwd_trace), host-thread-local.
thread_local unsigned long long* g_trace = nullptr;
thread_local int g_trace_cap = 0;
// Optional dump of every dQ partial (dash_attn_bwd_dump), host-thread-local.
thread_local float* g_dump = nullptr;

// Optional per-kernel event timing (dash_profile_begin/end).
// Events are recorded at the start of a call (tag 0) and after each launch
// (tag 1 = K1 preprocess, 2 = K2 main, 3 = K4 convert; a chunked call has one
// 2, 3 pair per chunk); dash_profile_end sums each interval under its tag.
struct ProfState {
  bool on = false;
  std::vector<std::pair<cudaEvent_t, int>> ev;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t get() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
};
ProfState& prof() {
  static ProfState p;
  return p;
}
void prof_mark(cudaStream_t st, int tag) {
  ProfState& p = prof();
  if (!p.on) return;
  cudaEvent_t e = p.get();
  cudaEventRecord(e, st);
  p.ev.emplace_back(e, tag);
}

// Between chunks: tickets and the job counter back to 0 (the error flag, the
// word after the counter, keeps what earlier chunks set); the atomic variant
// also re-zeroes its accumulator.
cudaError_t reset_chunk(char* ws, const WsLayout& w, int deterministic, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(ws + w.tickets, 0, w.counters + 4 - w.tickets, st);
  if (e == cudaSuccess && !deterministic) e = cudaMemsetAsync(ws + w.dqacc, 0, w.dqacc_bytes, st);
  return e;
}

// Programmatic dependent launch between the call's kernels (K1 -> K2 -> K4):
// each kernel waits (griddepcontrol.wait) before touching what its
// predecessor writes, so its launch and prologue can overlap the
// predecessor's tail.  Off by default: measured back to back with nothing
// between the kernels it is 2-2.5 % slower per step (with CUDA events recorded
// between the kernels, as in the first measurement, it is inert;
// profiles/r02_experiments_pdl.txt).  DASH_PDL=1 turns it on (experiments).
bool pdl_on() {
  static const bool on = [] {
    const char* e = std::getenv("DASH_PDL");
    return e && std::atoi(e) == 1;
  }();
  return on;
}
void set_pdl(cudaLaunchAttribute* a) {
  a->id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a->val.programmaticStreamSerializationAllowed = pdl_on() ? 1 : 0;
}

// K1 and K4 grids: one wave of 256-thread blocks (8 per SM), grid-stride.
template <int D>
void launch_preprocess(const dash_shape* s, const void* o, const void* dout, const float* lse,
                       float* dvec, float* lse2, int* tickets, int n_tickets, float* zero,
                       size_t n_zero_f4, int* counters, int poison, int sms, cudaStream_t stream) {
  constexpr int RPB = 256 / (D / 8);
  constexpr int kr = 2;  // rows per thread and iteration (4 measured 7 % slower)
  const size_t rows = static_cast<size_t>(s->batch) * s->seqlen * s->heads;
  size_t g = (rows + kr * RPB - 1) / (kr * RPB);
  if (g > static_cast<size_t>(sms) * 8) g = static_cast<size_t>(sms) * 8;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(g));
  cfg.blockDim = dim3(256);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  set_pdl(&attr[0]);
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, dash_preprocess_kernel<D, kr>, static_cast<const __nv_bfloat16*>(o),
                     static_cast<const __nv_bfloat16*>(dout), lse, dvec, lse2, s->batch, s->seqlen,
                     s->heads, FastDiv::make(s->seqlen), FastDiv::make(s->heads), tickets, n_tickets,
                     reinterpret_cast<float4*>(zero), n_zero_f4, counters, poison);
}
template <int D>
void launch_convert(const dash_shape* s, const float* dqacc, void* dq, int W, int causal, int tile,
                    int bh_base, int bh_count, int sms, cudaStream_t stream) {
  const size_t total = static_cast<size_t>(bh_count) * s->seqlen * (D / 8);
  size_t g = (total + 2 * 256 - 1) / (2 * 256);
  if (g > static_cast<size_t>(sms) * 8) g = static_cast<size_t>(sms) * 8;
  auto* out = static_cast<__nv_bfloat16*>(dq);
  const float sc = eff_scale(s);
  const int c = causal ? 1 : 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(g));
  cfg.blockDim = dim3(256);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  set_pdl(&attr[0]);
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  auto kern = W == 1 ? dash_dq_convert_kernel<D, 1>
              : W == 2 ? dash_dq_convert_kernel<D, 2>
              : W == 4 ? dash_dq_convert_kernel<D, 4>
                       : dash_dq_convert_kernel<D, 8>;
  cudaLaunchKernelEx(&cfg, kern, dqacc, out, s->seqlen, s->heads, FastDiv::make(s->seqlen),
                     FastDiv::make(s->heads), sc, c, tile, bh_base, bh_count);
}

template <int D>
dash_status launch_bwd(const dash_shape* s, const void* q, const void* k, const void* v,
                       const void* o, const void* dout, const float* lse, void* dq, void* dk,
                       void* dv, int causal, int schedule, int deterministic, void* workspace,
                       size_t workspace_bytes, cudaStream_t stream) {
  using C = BwdCfg<D>;
  const int n = s->seqlen / 128;
  const int W = resolved_split(s, deterministic, causal, schedule);  // once: K2 and K4 agree
  const int G = head_group_for(s);
  const WsLayout w = ws_layout(s, W, G);
  // The setting may have changed since the workspace was sized.
  if (workspace_bytes < w.total) return DASH_ERR_WORKSPACE;
  const ScheduleTable* tab = cached_schedule(schedule, n, causal ? kCausal : kFull);
  if (!tab) return DASH_ERR_UNSUPPORTED;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return DASH_ERR_CUDA;
  const int sms = device_sms(dev);
  const int max_jobs = tab->jobs * (w.chunk / G);  // per launch (one chunk of heads)
  const int grid = max_jobs < sms ? max_jobs : sms;

  if (schedule == kShift && tab->coresident > (tab->jobs < sms ? tab->jobs : sms))
    return DASH_ERR_UNSUPPORTED;
  const DevTable* dt = device_table(dev, tab, G);
  if (!dt) return DASH_ERR_CUDA;

  char* ws = static_cast<char*>(workspace);
  float* dqacc = reinterpret_cast<float*>(ws + w.dqacc);
  float* dvec = reinterpret_cast<float*>(ws + w.dvec);
  float* lse2 = reinterpret_cast<float*>(ws + w.lse2);
  int* tickets = reinterpret_cast<int*>(ws + w.tickets);
  int* counters = reinterpret_cast<int*>(ws + w.counters);

  const uint64_t HD = static_cast<uint64_t>(s->heads) * D;
  const uint64_t BN = static_cast<uint64_t>(s->batch) * s->seqlen;
  CUtensorMap tq, tk, tv, tdo, tacc, tdk, tdv;
  bool ok = make_map_2d(&tq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, q, HD, BN, 64, C::BR) &&
            make_map_2d(&tk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, k, HD, BN, 64, C::BC) &&
            make_map_2d(&tv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, v, HD, BN, 64, C::BC) &&
            make_map_2d(&tdo, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dout, HD, BN, 64, C::BR) &&
            make_map_2d(&tdk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dk, HD, BN, 32, 32,
                        CU_TENSOR_MAP_SWIZZLE_NONE) &&
            make_map_2d(&tdv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dv, HD, BN, 32, 32,
                        CU_TENSOR_MAP_SWIZZLE_NONE);
  if (ok && !C::LINEAR)  // d = 64 reduces through a 2-D map of the W planes
    ok = make_map_2d(&tacc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, dqacc, D,
                     static_cast<uint64_t>(W) * w.chunk * s->seqlen, 32, C::STG_ROWS);
  else
    tacc = tq;  // unused at d = 128 (1-D bulk reduces)
  if (!ok) {  // tensor map encoding (reported as -1 by dash_last_cuda_error)
    g_last_cuda = -1;
    return DASH_ERR_CUDA;
  }
  auto kern = dash_bwd_kernel<D>;
  if (!ensure_smem_attr(reinterpret_cast<const void*>(kern), static_cast<int>(C::SMEM_BYTES)))
    return cuda_check_last();

  const int poison = g_poison;
  g_poison = 0;
  prof_mark(stream, 0);
  // K1: D, ticket / counter / error-flag reset, dQacc zero-fill for the atomic variant.
  launch_preprocess<D>(s, o, dout, lse, dvec, lse2, tickets,
                       static_cast<int>(W * w.n_tickets + w.n_done),
                       deterministic ? nullptr : dqacc, deterministic ? 0 : w.dqacc_bytes / 16,
                       counters, poison, sms, stream);
  prof_mark(stream, 1);
  // Per chunk of heads (one chunk unless the planes exceed the budget):
  // K2, the persistent ordered-reduction backward, then K4.
  {
    BwdArgs a;
    a.lse2 = lse2;
    a.Dvec = dvec;
    a.dk = static_cast<__nv_bfloat16*>(dk);
    a.dv = static_cast<__nv_bfloat16*>(dv);
    a.tickets = tickets;
    a.job_counter = counters;
    a.error_flag = counters + 1;
    a.job_begin = dt->job_begin;
    a.tasks = dt->tasks;
    a.seg_end = dt->seg_end;
    a.B = s->batch;
    a.N = s->seqlen;
    a.H = s->heads;
    a.jobs_per_head = tab->jobs;
    a.scale = eff_scale(s);
    a.scale_log2 = a.scale * 1.4426950408889634f;
    a.causal = causal ? 1 : 0;
    a.deterministic = deterministic ? 1 : 0;
    a.trace = g_trace;
    a.trace_cap = g_trace_cap;
    a.spin_bound = g_spin_bound;
    a.split = W;
    a.dqacc = dqacc;
    a.n_tickets = static_cast<int>(w.n_tickets);
    a.dump = g_dump;
    a.prefetch = early_claim(schedule, causal, deterministic, W, false, tab->jobs);
    a.cyclic = (deterministic && schedule == kShift) ? 1 : 0;
    a.head_group = G;
    a.done = reinterpret_cast<int*>(ws + w.done);
    a.dq = static_cast<__nv_bfloat16*>(dq);
    a.fuse_dq = fused_for(s) ? 1 : 0;
    a.acc_tile = 128;
    a.done_target = tab->jobs * NAG;
    const int BH = s->batch * s->heads;
    for (int c = 0; c < w.chunks; ++c) {
      a.bh_base = c * w.chunk;
      a.bh_count = std::min(w.chunk, BH - a.bh_base);
      a.total_jobs = tab->jobs * (a.bh_count / G);
      if (c > 0 && reset_chunk(ws, w, deterministic, stream) != cudaSuccess) return cuda_check_last();
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(std::min(grid, a.total_jobs));
      cfg.blockDim = dim3(C::NTHREADS);
      cfg.dynamicSmemBytes = C::SMEM_BYTES;
      cfg.stream = stream;
      cudaLaunchAttribute attr[2];
      attr[0].id = cudaLaunchAttributeCooperative;  // co-residency for SHIFT (AMB-12)
      attr[0].val.cooperative = 1;
      set_pdl(&attr[1]);
      cfg.attrs = attr;
      cfg.numAttrs = 2;
      const cudaError_t le = cudaLaunchKernelEx(&cfg, kern, tq, tk, tv, tdo, tacc, tdk, tdv, a);
      if (le != cudaSuccess) {
        g_last_cuda = 10000 + static_cast<int>(le);  // launch of the main kernel
        return DASH_ERR_CUDA;
      }
      prof_mark(stream, 2);
      // K4: dQ = bf16(scale * (acc_0 + ... + acc_{W-1})) for the chunk's heads
      // (unless the main kernel finalised dQ itself).
      if (!a.fuse_dq) launch_convert<D>(s, dqacc, dq, W, causal, 128, a.bh_base, a.bh_count, sms, stream);
      prof_mark(stream, 3);
    }
  }
  return cuda_check_last();
}

template <int NQS, int NQK, int NDS>
int max_pair_clusters(int dev) {
  static std::mutex mu;
  static std::map<int, int> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * device_sms(dev));
  cfg.blockDim = dim3(PairCfg::NTHREADS);
  cfg.dynamicSmemBytes = PairCfgT<NQS, NQK, NDS>::SMEM_BYTES;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, dash_bwd_pair_kernel<NQS, NQK, NDS>, &cfg) != cudaSuccess ||
      n < 1)
    n = device_sms(dev) / 2;
  (void)cudaGetLastError();
  cache[dev] = n;
  return n;
}

// The CTA-pair backward (bwd2.cuh), d = 128, 256-row schedule tiles.
template <int NQS, int NQK, int NDS>
dash_status launch_bwd_pair(const dash_shape* s, const void* q, const void* k, const void* v,
                            const void* o, const void* dout, const float* lse, void* dq, void* dk,
                            void* dv, int causal, int schedule, int deterministic, void* workspace,
                            size_t workspace_bytes, cudaStream_t stream) {
  using C = PairCfgT<NQS, NQK, NDS>;
  constexpr int D = 128;
  const int n = s->seqlen / C::TILE;
  const int W = resolved_split(s, deterministic, causal, schedule);
  const WsLayout w = ws_layout(s, W);
  if (workspace_bytes < w.total) return DASH_ERR_WORKSPACE;
  const int BH = s->batch * s->heads;
  const ScheduleTable* tab = cached_schedule(schedule, n, causal ? kCausal : kFull);
  if (!tab) return DASH_ERR_UNSUPPORTED;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return DASH_ERR_CUDA;
  auto kern = dash_bwd_pair_kernel<NQS, NQK, NDS>;
  if (!ensure_smem_attr(reinterpret_cast<const void*>(kern), static_cast<int>(C::SMEM_BYTES)))
    return cuda_check_last();
  const int sms = device_sms(dev);
  const int max_cl = max_pair_clusters<NQS, NQK, NDS>(dev);
  const int max_jobs = tab->jobs * w.chunk;  // per launch (one chunk of heads)
  const int clusters = max_jobs < max_cl ? max_jobs : max_cl;
  if (schedule == kShift && tab->coresident > (tab->jobs < max_cl ? tab->jobs : max_cl))
    return DASH_ERR_UNSUPPORTED;
  const DevTable* dt = device_table(dev, tab, 1);
  if (!dt) return DASH_ERR_CUDA;

  char* ws = static_cast<char*>(workspace);
  float* dqacc = reinterpret_cast<float*>(ws + w.dqacc);
  float* dvec = reinterpret_cast<float*>(ws + w.dvec);
  float* lse2 = reinterpret_cast<float*>(ws + w.lse2);
  int* tickets = reinterpret_cast<int*>(ws + w.tickets);
  int* counters = reinterpret_cast<int*>(ws + w.counters);

  const uint64_t HD = static_cast<uint64_t>(s->heads) * D;
  const uint64_t BN = static_cast<uint64_t>(s->batch) * s->seqlen;
  CUtensorMap tq32, tq64, tk, tv, tdo32, tdo64, tacc, tdk, tdv;
  const bool ok =
      make_map_2d(&tq32, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, q, HD, BN, 64, 32) &&
      make_map_2d(&tq64, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, q, HD, BN, 64, 64) &&
      make_map_2d(&tk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, k, HD, BN, 64, C::BC) &&
      make_map_2d(&tv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, v, HD, BN, 64, C::BC) &&
      make_map_2d(&tdo32, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dout, HD, BN, 64, 32) &&
      make_map_2d(&tdo64, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dout, HD, BN, 64, 64) &&
      make_map_2d(&tacc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, dqacc, D,
                  static_cast<uint64_t>(W) * w.chunk * s->seqlen, 32, C::BR) &&
      // dK / dV epilogue: 32 x 32 bf16 boxes (64 B rows, unswizzled staging)
      make_map_2d(&tdk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dk, HD, BN, 32, 32,
                  CU_TENSOR_MAP_SWIZZLE_NONE) &&
      make_map_2d(&tdv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dv, HD, BN, 32, 32,
                  CU_TENSOR_MAP_SWIZZLE_NONE);
  if (!ok) {
    g_last_cuda = -1;
    return DASH_ERR_CUDA;
  }
  const int poison = g_poison;
  g_poison = 0;
  prof_mark(stream, 0);
  // K1: D, ticket / counter / error-flag reset, dQacc zero-fill for the atomic variant.
  launch_preprocess<D>(s, o, dout, lse, dvec, lse2, tickets,
                       static_cast<int>(W * w.n_tickets + w.n_done),
                       deterministic ? nullptr : dqacc, deterministic ? 0 : w.dqacc_bytes / 16,
                       counters, poison, sms, stream);
  prof_mark(stream, 1);
  {
    BwdArgs a;
    a.lse2 = lse2;
    a.Dvec = dvec;
    a.dk = static_cast<__nv_bfloat16*>(dk);
    a.dv = static_cast<__nv_bfloat16*>(dv);
    a.tickets = tickets;
    a.job_counter = counters;
    a.error_flag = counters + 1;
    a.job_begin = dt->job_begin;
    a.tasks = dt->tasks;
    a.seg_end = dt->seg_end;
    a.B = s->batch;
    a.N = s->seqlen;
    a.H = s->heads;
    a.jobs_per_head = tab->jobs;
    a.scale = eff_scale(s);
    a.scale_log2 = a.scale * 1.4426950408889634f;
    a.causal = causal ? 1 : 0;
    a.deterministic = deterministic ? 1 : 0;
    a.trace = g_trace;
    a.trace_cap = g_trace_cap;
    a.spin_bound = g_spin_bound;
    a.split = W;
    a.dqacc = dqacc;
    a.n_tickets = static_cast<int>(w.n_tickets);
    a.dump = g_dump;
    a.prefetch = early_claim(schedule, causal, deterministic, W, true, tab->jobs);
    a.cyclic = (deterministic && schedule == kShift) ? 1 : 0;
    a.head_group = 1;
    a.done = reinterpret_cast<int*>(ws + w.done);
    a.dq = static_cast<__nv_bfloat16*>(dq);
    a.fuse_dq = fused_for(s) ? 1 : 0;
    a.acc_tile = C::TILE;
    a.done_target = tab->jobs * 2 * NAG;  // both CTAs' agents
    for (int c = 0; c < w.chunks; ++c) {
      a.bh_base = c * w.chunk;
      a.bh_count = std::min(w.chunk, BH - a.bh_base);
      a.total_jobs = tab->jobs * a.bh_count;
      if (c > 0 && reset_chunk(ws, w, deterministic, stream) != cudaSuccess) return cuda_check_last();
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(2 * std::min(clusters, a.total_jobs));
      cfg.blockDim = dim3(C::NTHREADS);
      cfg.dynamicSmemBytes = C::SMEM_BYTES;
      cfg.stream = stream;
      cudaLaunchAttribute attr[1];
      set_pdl(&attr[0]);
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      const cudaError_t le =
          cudaLaunchKernelEx(&cfg, kern, tq32, tq64, tk, tv, tdo32, tdo64, tacc, tdk, tdv, a);
      if (le != cudaSuccess) {
        g_last_cuda = 10000 + static_cast<int>(le);
        return DASH_ERR_CUDA;
      }
      prof_mark(stream, 2);
      if (!a.fuse_dq)
        launch_convert<D>(s, dqacc, dq, W, causal, C::TILE, a.bh_base, a.bh_count, sms, stream);
      prof_mark(stream, 3);
    }
  }
  return cuda_check_last();
}

}  // namespace
}  // namespace dash

using namespace dash;

DASH_API int dash_last_cuda_error(void) { return g_last_cuda; }

DASH_API const char* dash_status_string(dash_status s) {
  switch (s) {
    case DASH_OK: return "DASH_OK";
    case DASH_ERR_INVALID_ARG: return "DASH_ERR_INVALID_ARG";
    case DASH_ERR_UNSUPPORTED: return "DASH_ERR_UNSUPPORTED";
    case DASH_ERR_WORKSPACE: return "DASH_ERR_WORKSPACE";
    case DASH_ERR_CUDA: return "DASH_ERR_CUDA";
    case DASH_ERR_DEADLOCK: return "DASH_ERR_DEADLOCK";
  }
  return "DASH_ERR_UNKNOWN";
}

DASH_API const char* dash_version(void) { return "dash-b200 0.1 (sm_100a)"; }

DASH_API dash_status dash_profile_begin(void) {
  ProfState& p = prof();
  for (auto& e : p.ev) p.pool.push_back(e.first);
  p.ev.clear();
  p.on = true;
  return DASH_OK;
}

DASH_API dash_status dash_profile_end(double* ms_pre, double* ms_main, double* ms_post,
                                      int* n_calls) {
  ProfState& p = prof();
  p.on = false;
  double sum[4] = {0, 0, 0, 0};
  int n = 0;
  if (!p.ev.empty() && cudaEventSynchronize(p.ev.back().first) != cudaSuccess) return DASH_ERR_CUDA;
  for (size_t i = 0; i < p.ev.size(); ++i) {
    const int tag = p.ev[i].second;
    if (tag == 0) {
      ++n;
      continue;
    }
    float t = 0;
    if (i > 0) cudaEventElapsedTime(&t, p.ev[i - 1].first, p.ev[i].first);
    sum[tag] += t;
  }
  for (auto& e : p.ev) p.pool.push_back(e.first);
  p.ev.clear();
  const double a = sum[1], b = sum[2], c = sum[3];
  if (ms_pre) *ms_pre = a;
  if (ms_main) *ms_main = b;
  if (ms_post) *ms_post = c;
  if (n_calls) *n_calls = n;
  return DASH_OK;
}

DASH_API dash_status dash_attn_bwd_set_fused_dq(int on) {
  if (on < 0 || on > 2) return DASH_ERR_INVALID_ARG;
  g_fused_dq = on;
  return DASH_OK;
}
DASH_API int dash_attn_bwd_fused_dq(void) { return g_fused_dq; }

DASH_API int dash_attn_bwd_launches(int causal, int schedule, int deterministic) {
  (void)causal;
  (void)schedule;
  (void)deterministic;
  return g_fused_dq == 2 ? 2 : 3;  // preprocess, main (+ dQ convert)
}

DASH_API int dash_attn_bwd_launch_count(const dash_shape* shape, int causal, int schedule,
                                        int deterministic) {
  if (!shape_ok(shape) || schedule < DASH_SCHED_NAIVE || schedule > DASH_SCHED_AUTO) return 0;
  const WsLayout w = layout_for(shape, deterministic, causal, schedule);
  return 1 + w.chunks * (fused_for(shape) ? 1 : 2);
}

namespace dash {
namespace {
template <int D>
dash_status launch_fwd_tc(const dash_shape* s, const void* q, const void* k, const void* v, void* o,
                          float* lse, int causal, cudaStream_t st) {
  using C = FwdCfg<D>;
  const uint64_t HD = static_cast<uint64_t>(s->heads) * D;
  const uint64_t BN = static_cast<uint64_t>(s->batch) * s->seqlen;
  CUtensorMap tq, tk, tv;
  if (!(make_map_2d(&tq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, q, HD, BN, 64, 128) &&
        make_map_2d(&tk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, k, HD, BN, 64, 128) &&
        make_map_2d(&tv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, v, HD, BN, 64, 128)))
    return DASH_ERR_CUDA;
  FwdArgs a;
  a.o = static_cast<__nv_bfloat16*>(o);
  a.lse = lse;
  a.B = s->batch;
  a.N = s->seqlen;
  a.H = s->heads;
  a.scale_log2 = eff_scale(s) * 1.4426950408889634f;
  a.causal = causal ? 1 : 0;
  if (!ensure_smem_attr(reinterpret_cast<const void*>(dash_fwd_tc_kernel<D>),
                        static_cast<int>(C::SMEM_BYTES)))
    return cuda_check_last();
  const dim3 grid(s->seqlen / 128, s->batch * s->heads);
  dash_fwd_tc_kernel<D><<<grid, 256, C::SMEM_BYTES, st>>>(tq, tk, tv, a);
  return cuda_check_last();
}
}  // namespace
}  // namespace dash

DASH_API dash_status dash_attn_fwd(const dash_shape* s, const void* q, const void* k, const void* v,
                                   void* o, float* lse, int causal, void* stream) {
  bind_context();
  if (!shape_ok(s) || !aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o) ||
      !aligned16(lse))
    return DASH_ERR_INVALID_ARG;
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  return s->head_dim == 128 ? launch_fwd_tc<128>(s, q, k, v, o, lse, causal, st)
                             : launch_fwd_tc<64>(s, q, k, v, o, lse, causal, st);
}

DASH_API size_t dash_attn_bwd_workspace_bytes(const dash_shape* s, int causal, int schedule,
                                              int deterministic) {
  if (!shape_ok(s)) return 0;
  if (schedule < DASH_SCHED_NAIVE || schedule > DASH_SCHED_AUTO) return 0;
  return layout_for(s, deterministic, causal, schedule).total;
}

DASH_API dash_status dash_attn_bwd(const dash_shape* s, const void* q, const void* k, const void* v,
                                   const void* o, const void* dout, const float* lse, void* dq,
                                   void* dk, void* dv, int causal, int schedule, int deterministic,
                                   void* workspace, size_t workspace_bytes, void* stream) {
  bind_context();
  if (!shape_ok(s)) return DASH_ERR_INVALID_ARG;
  const void* ptrs[] = {q, k, v, o, dout, lse, dq, dk, dv, workspace};
  for (const void* p : ptrs)
    if (!aligned16(p)) return DASH_ERR_INVALID_ARG;
  if (schedule < DASH_SCHED_NAIVE || schedule > DASH_SCHED_AUTO) return DASH_ERR_INVALID_ARG;
  if (schedule == DASH_SCHED_AUTO) schedule = auto_schedule(s, causal);
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (tile_for(s, causal, schedule) == PairCfg::TILE)
    return launch_bwd_pair<2, 2, 2>(s, q, k, v, o, dout, lse, dq, dk, dv, causal, schedule,
                                    deterministic, workspace, workspace_bytes, st);
  return s->head_dim == 128
             ? launch_bwd<128>(s, q, k, v, o, dout, lse, dq, dk, dv, causal, schedule,
                               deterministic, workspace, workspace_bytes, st)
             : launch_bwd<64>(s, q, k, v, o, dout, lse, dq, dk, dv, causal, schedule,
                              deterministic, workspace, workspace_bytes, st);
}

DASH_API dash_status dash_attn_bwd_set_watchdog(long long cycles) {
  if (cycles < 0) return DASH_ERR_INVALID_ARG;
  g_spin_bound = cycles == 0 ? 8 * ptx::kWatchdogCycles : cycles;
  return DASH_OK;
}

DASH_API dash_status dash_attn_bwd_inject_fault(int poison) {
  g_poison = poison;
  return DASH_OK;
}

DASH_API dash_status dash_attn_bwd_trace(const dash_shape* s, const void* q, const void* k,
                                         const void* v, const void* o, const void* dout,
                                         const float* lse, void* dq, void* dk, void* dv, int causal,
                                         int schedule, int deterministic, void* workspace,
                                         size_t workspace_bytes, unsigned long long* trace,
                                         int trace_cap, void* stream) {
  if (!trace || trace_cap < 1) return DASH_ERR_INVALID_ARG;
  g_trace = trace;
  g_trace_cap = trace_cap;
  const dash_status r = dash_attn_bwd(s, q, k, v, o, dout, lse, dq, dk, dv, causal, schedule,
                                      deterministic, workspace, workspace_bytes, stream);
  g_trace = nullptr;
  g_trace_cap = 0;
  return r;
}

DASH_API int dash_attn_bwd_acc_split(const dash_shape* s, int causal, int schedule) {
  if (!s) return acc_split();
  if (!shape_ok(s) || schedule < DASH_SCHED_NAIVE || schedule > DASH_SCHED_AUTO) return 0;
  return resolved_split(s, 1, causal, schedule);
}

DASH_API dash_status dash_attn_bwd_set_acc_split(int w) {
  if (w != 0 && w != 1 && w != 2 && w != 4 && w != 8) return DASH_ERR_INVALID_ARG;
  g_acc_split = w;
  return DASH_OK;
}

DASH_API int dash_attn_bwd_tile(const dash_shape* s, int causal, int schedule) {
  if (!shape_ok(s) || schedule < DASH_SCHED_NAIVE || schedule > DASH_SCHED_AUTO) return 0;
  if (schedule == DASH_SCHED_AUTO) schedule = auto_schedule(s, causal);
  return tile_for(s, causal, schedule);
}

DASH_API size_t dash_attn_bwd_dump_bytes(const dash_shape* s, int causal, int schedule) {
  const int tile = dash_attn_bwd_tile(s, causal, schedule);
  if (tile == 0) return 0;
  return static_cast<size_t>(s->batch) * s->heads * (s->seqlen / tile) * s->seqlen *
         s->head_dim * 4;
}

DASH_API dash_status dash_attn_bwd_set_plane_budget(size_t bytes) {
  g_plane_budget = bytes == 0 ? kDefaultPlaneBudget : bytes;
  return DASH_OK;
}

DASH_API int dash_attn_bwd_head_chunk(const dash_shape* s, int causal, int schedule,
                                      int deterministic) {
  if (!shape_ok(s) || schedule < DASH_SCHED_NAIVE || schedule > DASH_SCHED_AUTO) return 0;
  return layout_for(s, deterministic, causal, schedule).chunk;
}

DASH_API dash_status dash_attn_bwd_set_tile(int tile) {
  if (tile != 0 && tile != 128 && tile != 256) return DASH_ERR_INVALID_ARG;
  g_tile = tile;
  return DASH_OK;
}

DASH_API int dash_attn_bwd_resolve_schedule(const dash_shape* s, int causal, int schedule) {
  if (!shape_ok(s) || schedule < DASH_SCHED_NAIVE || schedule > DASH_SCHED_AUTO) return -1;
  return schedule == DASH_SCHED_AUTO ? auto_schedule(s, causal) : schedule;
}

DASH_API dash_status dash_attn_bwd_dump(const dash_shape* s, const void* q, const void* k,
                                        const void* v, const void* o, const void* dout,
                                        const float* lse, void* dq, void* dk, void* dv, int causal,
                                        int schedule, int deterministic, void* workspace,
                                        size_t workspace_bytes, float* partials,
                                        size_t partial_bytes, void* stream) {
  if (!shape_ok(s) || !aligned16(partials)) return DASH_ERR_INVALID_ARG;
  if (partial_bytes < dash_attn_bwd_dump_bytes(s, causal, schedule)) return DASH_ERR_WORKSPACE;
  g_dump = partials;
  const dash_status r = dash_attn_bwd(s, q, k, v, o, dout, lse, dq, dk, dv, causal, schedule,
                                      deterministic, workspace, workspace_bytes, stream);
  g_dump = nullptr;
  return r;
}

namespace {
// End-to-end path (dash_attn_bwd_host): the (b, h) heads are split into
// chunks -- batch ranges, or head ranges of one batch when B < 4 -- and the
// chunks stream through three device slots on three library streams:
// H2D of chunk i+1 || backward of chunk i || D2H of chunk i-1.  A chunk is a
// (b, h) shard, so its results are bit-identical to the one-shot call
// (tests/test_gpu_bwd.py::test_host_path_matches_device_path).
constexpr int kHostSlots = 3;
// target number of chunks per call (DASH_HOST_CHUNKS overrides; experiments)
int host_chunks() {
  static const int c = [] {
    const char* e = std::getenv("DASH_HOST_CHUNKS");
    const int v = e ? std::atoi(e) : 0;
    return v >= 1 ? v : 8;
  }();
  return c;
}
struct HostPlan {
  int nb, nh;          // chunk shape: nb batches x nh heads (nb == B or nh == H)
  int chunks_b, chunks_h;
  size_t in_bytes, lse_bytes;  // per chunk (largest)
  size_t q, k, v, o, dout, lse, dq, dk, dv, inner, slot, total;
};
HostPlan host_plan(const dash_shape* s, int causal, int schedule, int deterministic) {
  HostPlan h;
  const int kc = host_chunks();
  if (s->batch >= kc) {
    h.nb = (s->batch + kc - 1) / kc;
    h.nh = s->heads;
  } else {
    const int hb = (kc + s->batch - 1) / s->batch;  // head blocks per batch
    h.nb = 1;
    h.nh = (s->heads + hb - 1) / hb;
  }
  h.chunks_b = (s->batch + h.nb - 1) / h.nb;
  h.chunks_h = (s->heads + h.nh - 1) / h.nh;
  dash_shape cs = *s;
  cs.batch = h.nb;
  cs.heads = h.nh;
  h.in_bytes = static_cast<size_t>(h.nb) * s->seqlen * h.nh * s->head_dim * 2;
  h.lse_bytes = static_cast<size_t>(h.nb) * h.nh * s->seqlen * 4;
  size_t off = 0;
  size_t* slots[] = {&h.q, &h.k, &h.v, &h.o, &h.dout, &h.dq, &h.dk, &h.dv};
  for (size_t* sl : slots) {
    *sl = off;
    off = align_up(off + h.in_bytes, kAlign);
  }
  h.lse = off;
  off = align_up(off + h.lse_bytes, kAlign);
  h.inner = off;
  h.slot = align_up(off + layout_for(&cs, deterministic, causal, schedule).total, kAlign);
  h.total = kHostSlots * h.slot;
  return h;
}
struct HostStreams {
  cudaStream_t h2d, comp, d2h;
  cudaEvent_t start, in_done[kHostSlots], comp_done[kHostSlots], out_done[kHostSlots];
};
const HostStreams* host_streams(int dev) {
  static std::mutex mu;
  static std::map<int, HostStreams> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return &it->second;
  HostStreams hs;
  cudaStreamCreateWithFlags(&hs.h2d, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&hs.comp, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&hs.d2h, cudaStreamNonBlocking);
  cudaEventCreateWithFlags(&hs.start, cudaEventDisableTiming);
  for (int i = 0; i < kHostSlots; ++i) {
    cudaEventCreateWithFlags(&hs.in_done[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&hs.comp_done[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&hs.out_done[i], cudaEventDisableTiming);
  }
  cache[dev] = hs;
  return &cache[dev];
}
// Copies the chunk (b0.., h0..) of a [B,N,H,d] bf16 tensor between host and a
// packed [nb,N,nh,d] device buffer (2-D copy when the chunk is a head range).
cudaError_t copy_chunk(void* dst, const void* src, const dash_shape* s, int b0, int nb, int h0,
                       int nh, bool to_device, cudaStream_t st) {
  const size_t row = static_cast<size_t>(s->head_dim) * 2;
  if (nh == s->heads) {
    const size_t off = static_cast<size_t>(b0) * s->seqlen * s->heads * row;
    const size_t bytes = static_cast<size_t>(nb) * s->seqlen * s->heads * row;
    return to_device ? cudaMemcpyAsync(dst, static_cast<const char*>(src) + off, bytes,
                                       cudaMemcpyHostToDevice, st)
                     : cudaMemcpyAsync(static_cast<char*>(dst) + off, src, bytes,
                                       cudaMemcpyDeviceToHost, st);
  }
  const size_t hoff = (static_cast<size_t>(b0) * s->seqlen * s->heads + h0) * row;
  const size_t hpitch = s->heads * row, dpitch = nh * row;
  return to_device ? cudaMemcpy2DAsync(dst, dpitch, static_cast<const char*>(src) + hoff, hpitch,
                                       dpitch, s->seqlen, cudaMemcpyHostToDevice, st)
                   : cudaMemcpy2DAsync(static_cast<char*>(dst) + hoff, hpitch, src, dpitch, dpitch,
                                       s->seqlen, cudaMemcpyDeviceToHost, st);
}
}  // namespace

DASH_API size_t dash_attn_bwd_host_workspace_bytes(const dash_shape* s, int causal, int schedule,
                                                   int deterministic) {
  if (!shape_ok(s)) return 0;
  if (schedule < DASH_SCHED_NAIVE || schedule > DASH_SCHED_AUTO) return 0;
  return host_plan(s, causal, schedule, deterministic).total;
}

DASH_API dash_status dash_attn_bwd_host(const dash_shape* s, const void* q, const void* k,
                                        const void* v, const void* o, const void* dout,
                                        const float* lse, void* dq, void* dk, void* dv, int causal,
                                        int schedule, int deterministic, void* workspace,
                                        size_t workspace_bytes, void* stream) {
  bind_context();
  if (!shape_ok(s)) return DASH_ERR_INVALID_ARG;
  const void* hptrs[] = {q, k, v, o, dout, lse, dq, dk, dv};
  for (const void* p : hptrs)
    if (!p) return DASH_ERR_INVALID_ARG;
  if (!aligned16(workspace)) return DASH_ERR_INVALID_ARG;
  if (schedule < DASH_SCHED_NAIVE || schedule > DASH_SCHED_AUTO) return DASH_ERR_INVALID_ARG;
  const HostPlan h = host_plan(s, causal, schedule, deterministic);
  if (workspace_bytes < h.total) return DASH_ERR_WORKSPACE;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return DASH_ERR_CUDA;
  const HostStreams* hs = host_streams(dev);
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  // respect work already queued on the caller's stream
  if (cudaEventRecord(hs->start, st) != cudaSuccess) return DASH_ERR_CUDA;
  cudaStreamWaitEvent(hs->h2d, hs->start, 0);
  char* base = static_cast<char*>(workspace);
  int idx = 0;
  for (int cb = 0; cb < h.chunks_b; ++cb) {
    for (int ch = 0; ch < h.chunks_h; ++ch, ++idx) {
      const int b0 = cb * h.nb, nb = std::min(h.nb, s->batch - b0);
      const int h0 = ch * h.nh, nh = std::min(h.nh, s->heads - h0);
      const int slot = idx % kHostSlots;
      char* w = base + static_cast<size_t>(slot) * h.slot;
      // H2D (slot free once chunk idx - kHostSlots has been copied out)
      if (idx >= kHostSlots) cudaStreamWaitEvent(hs->h2d, hs->out_done[slot], 0);
      const void* ins[] = {q, k, v, o, dout};
      const size_t ioff[] = {h.q, h.k, h.v, h.o, h.dout};
      for (int t = 0; t < 5; ++t)
        if (copy_chunk(w + ioff[t], ins[t], s, b0, nb, h0, nh, true, hs->h2d) != cudaSuccess)
          return DASH_ERR_CUDA;
      const size_t loff = (static_cast<size_t>(b0) * s->heads + h0) * s->seqlen * 4;
      if (cudaMemcpy2DAsync(w + h.lse, static_cast<size_t>(nh) * s->seqlen * 4,
                            reinterpret_cast<const char*>(lse) + loff,
                            static_cast<size_t>(s->heads) * s->seqlen * 4,
                            static_cast<size_t>(nh) * s->seqlen * 4, nb, cudaMemcpyHostToDevice,
                            hs->h2d) != cudaSuccess)
        return DASH_ERR_CUDA;
      cudaEventRecord(hs->in_done[slot], hs->h2d);
      // backward of the chunk (a (b, h) shard: same bits as the full call)
      cudaStreamWaitEvent(hs->comp, hs->in_done[slot], 0);
      dash_shape cs = *s;
      cs.batch = nb;
      cs.heads = nh;
      const dash_status r =
          dash_attn_bwd(&cs, w + h.q, w + h.k, w + h.v, w + h.o, w + h.dout,
                        reinterpret_cast<const float*>(w + h.lse), w + h.dq, w + h.dk, w + h.dv,
                        causal, schedule, deterministic, w + h.inner, h.slot - h.inner, hs->comp);
      if (r != DASH_OK) return r;
      cudaEventRecord(hs->comp_done[slot], hs->comp);
      // D2H
      cudaStreamWaitEvent(hs->d2h, hs->comp_done[slot], 0);
      void* outs[] = {dq, dk, dv};
      const size_t ooff[] = {h.dq, h.dk, h.dv};
      for (int t = 0; t < 3; ++t)
        if (copy_chunk(outs[t], w + ooff[t], s, b0, nb, h0, nh, false, hs->d2h) != cudaSuccess)
          return DASH_ERR_CUDA;
      cudaEventRecord(hs->out_done[slot], hs->d2h);
    }
  }
  cudaEventRecord(hs->start, hs->d2h);
  cudaStreamWaitEvent(st, hs->start, 0);
  return cudaStreamSynchronize(hs->d2h) == cudaSuccess && cudaGetLastError() == cudaSuccess
             ? DASH_OK
             : DASH_ERR_CUDA;
}

DASH_API dash_status dash_check_workspace(const dash_shape* s, int causal, int schedule,
                                          int deterministic, const void* workspace, void* stream) {
  if (!shape_ok(s) || !workspace) return DASH_ERR_INVALID_ARG;
  if (schedule < DASH_SCHED_NAIVE || schedule > DASH_SCHED_AUTO) return DASH_ERR_INVALID_ARG;
  const WsLayout w = layout_for(s, deterministic, causal, schedule);
  int flag = 0;
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  int* dflag = reinterpret_cast<int*>(static_cast<char*>(const_cast<void*>(workspace)) + w.counters) + 1;
  if (cudaMemcpyAsync(&flag, dflag, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess)
    return DASH_ERR_CUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) return DASH_ERR_CUDA;
  return flag ? DASH_ERR_DEADLOCK : DASH_OK;
}

DASH_API dash_status dash_schedule_critical_path(int schedule, int n_q, int n_kv, int mask,
                                                 const dash_dag_params* p, int64_t* out_length) {
  if (!out_length || n_q != n_kv || n_kv < 1) return DASH_ERR_INVALID_ARG;
  if (schedule < DASH_SCHED_NAIVE || schedule > DASH_SCHED_SHIFT) return DASH_ERR_INVALID_ARG;
  if (mask != DASH_MASK_FULL && mask != DASH_MASK_CAUSAL) return DASH_ERR_INVALID_ARG;
  dash_dag_params d = p ? *p : dash_dag_params{2, n_kv, 1, 1};
  if (d.c < 1 || d.r < 1 || d.n_sm < 1 || d.n_heads < 1) return DASH_ERR_INVALID_ARG;
  const ScheduleTable* t = cached_schedule(schedule, n_kv, mask);
  if (!t) return DASH_ERR_UNSUPPORTED;
  const int64_t cp = critical_path(*t, d.n_heads, d.n_sm, d.c, d.r);
  if (cp < 0) return DASH_ERR_DEADLOCK;
  *out_length = cp;
  return DASH_OK;
}

DASH_API dash_status dash_schedule_table(int schedule, int n_kv, int mask, int capacity,
                                         int32_t* task_job, int32_t* task_kv, int32_t* task_q,
                                         int32_t* task_rank, int32_t* n_tasks, int32_t* n_jobs) {
  if (n_kv < 1 || !n_tasks || !n_jobs) return DASH_ERR_INVALID_ARG;
  if (schedule < DASH_SCHED_NAIVE || schedule > DASH_SCHED_SHIFT) return DASH_ERR_INVALID_ARG;
  if (mask != DASH_MASK_FULL && mask != DASH_MASK_CAUSAL) return DASH_ERR_INVALID_ARG;
  const ScheduleTable* t = cached_schedule(schedule, n_kv, mask);
  if (!t) return DASH_ERR_UNSUPPORTED;
  *n_tasks = static_cast<int32_t>(t->tasks.size());
  *n_jobs = t->jobs;
  if (capacity < static_cast<int>(t->tasks.size())) return DASH_ERR_WORKSPACE;
  if (!task_job || !task_kv || !task_q || !task_rank) return DASH_ERR_INVALID_ARG;
  for (int j = 0; j < t->jobs; ++j)
    for (int i = t->job_begin[j]; i < t->job_begin[j + 1]; ++i) {
      task_job[i] = j;
      task_kv[i] = t->tasks[i].kv;
      task_q[i] = t->tasks[i].q;
      task_rank[i] = t->tasks[i].rank;
    }
  return DASH_OK;
}
