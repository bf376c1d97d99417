// Schedule tables (§8(a) row a1) and the DAG critical-path model (row a8).
//
// Visiting orders: NAIVE P:37/P:55/P:85-89; DESCENDING §3.3
// P:91-103; SHIFT full §3.4 P:133 (Fig. 6); SHIFT causal = Symmetric
// Shift §3.4 P:135-139 (Fig. 7).  Reduction ranks are closed forms
// (DESIGN.md §Schedules): NAIVE/DESCENDING rank = i (ascending KV, AMB-6);
// SHIFT full rank = (j - i) mod n; SHIFT causal with h = n/2:
//   j >= h, i <  h : (j - h - i) mod h      (phase 1, cyclic rectangle)
//   j >= h, i >= h : i                      (phase 2, right triangle)
//   j <  h         : j - i                  (phase 2, left triangle)
// Odd n: the n + 1 schedule without the phantom tile n (AMB-29).  More than
// kShiftGroup KV tiles (full) / pairs (causal): groups, AMB-30 / AMB-35.
#include "schedule.h"

#include <algorithm>
#include <map>
#include <mutex>
#include <queue>
#include <tuple>

namespace dash {

int ScheduleTable::max_rank_plus1(int j) const { return mask == kFull ? n : j + 1; }

static int pos_mod(int a, int m) { return ((a % m) + m) % m; }

bool build_schedule(int schedule, int n, int mask, ScheduleTable* out) {
  ScheduleTable t;
  t.n = n;
  t.schedule = schedule;
  t.mask = mask;
  auto push_job = [&]() { t.job_begin.push_back(static_cast<int32_t>(t.tasks.size())); };
  if (n < 1) return false;
  if (schedule == kNaive || schedule == kDescending) {
    t.jobs = n;
    for (int i = 0; i < n; ++i) {
      push_job();
      const int lo = (mask == kCausal) ? i : 0;
      for (int s = 0; s < n - lo; ++s) {
        const int j = (schedule == kNaive) ? lo + s : n - 1 - s;
        t.tasks.push_back({i, j, i});
      }
    }
  } else if (schedule == kShift && mask == kFull) {
    // Groups of KV tiles [lo, hi), G = ceil(n / kShiftGroup) near-equal groups
    // (one group = the paper's cyclic shift, whenever n <= kShiftGroup).
    // KV i visits Q (i + s) mod n; dQ_j is reduced group by group, inside a
    // group in visit-step order (AMB-30):
    //   rank(i, j) = lo + (i <= j ? min(hi-1, j) - i : cnt_le + hi - 1 - i),
    //   cnt_le = #{group members <= j}.   (G = 1: rank = (j - i) mod n.)
    t.jobs = n;
    const int G = (n + kShiftGroup - 1) / kShiftGroup;
    for (int g = 0; g < G; ++g) {
      const int lo = static_cast<int>(static_cast<int64_t>(g) * n / G);
      const int hi = static_cast<int>(static_cast<int64_t>(g + 1) * n / G);
      t.coresident = std::max(t.coresident, hi - lo);
      for (int i = lo; i < hi; ++i) {
        push_job();
        for (int s = 0; s < n; ++s) {
          const int j = (i + s) % n;
          const int top = std::min(hi - 1, j);
          const int cnt_le = std::max(0, top - lo + 1);
          const int rank = lo + (i <= j ? top - i : cnt_le + (hi - 1 - i));
          t.tasks.push_back({i, j, rank});
        }
      }
    }
  } else if (schedule == kShift && mask == kCausal && n % 2) {
    // Odd n (AMB-29): the Symmetric Shift of n + 1 tiles without the phantom
    // KV tile n and Q tile n.  For a real Q tile j every contributor KV <= j
    // is real, so the n + 1 closed-form ranks are still 0..j in step order.
    ScheduleTable e;
    if (!build_schedule(schedule, n + 1, mask, &e)) return false;
    t.jobs = e.jobs;
    t.coresident = e.coresident;
    for (int p = 0; p < e.jobs; ++p) {
      push_job();
      for (int k = e.job_begin[p]; k < e.job_begin[p + 1]; ++k)
        if (e.tasks[k].kv < n && e.tasks[k].q < n) t.tasks.push_back(e.tasks[k]);
    }
  } else if (schedule == kShift && mask == kCausal) {
    // Pairs p = (KV p, KV n-1-p), h = n/2 of them.  More than kShiftGroup pairs
    // (AMB-35): G = ceil(h / kShiftGroup) consecutive near-equal groups of
    // pairs [lo, hi); the jobs are the paper's, dQ_j takes group 0's
    // contributions first, then group 1's, ..., each group in visit-step order
    // (G = 1: the paper's Symmetric Shift, ranks as in the header comment).
    // Per group, for Q tile j (a = j - h, r = n - 1 - j):
    //   rectangle, KV p -> j >= h (step (a - p) mod h):
    //     lo + max(0, lo - r) + #{q in [lo, hi): (a - q) mod h < (a - p) mod h}
    //   right triangle, KV n-1-p -> j >= n-1-p (steps after the rectangle,
    //     ascending KV):  lo + max(0, lo - r) + (hi - lo) + (hi - 1 - p)
    //   left triangle, KV p -> j < h, p <= j (KV descending):
    //     min(lo, j + 1) + min(hi - 1, j) - p
    const int h = n / 2;
    const int G = (h + kShiftGroup - 1) / kShiftGroup;
    t.jobs = h;
    for (int g = 0; g < G; ++g) {
      const int lo = static_cast<int>(static_cast<int64_t>(g) * h / G);
      const int hi = static_cast<int>(static_cast<int64_t>(g + 1) * h / G);
      const int gs = hi - lo;
      t.coresident = std::max(t.coresident, gs);
      // position of KV p's rectangle step among the group's steps for Q j:
      // the steps (a - q) mod h, q = hi-1 .. lo, are the cyclic range that
      // starts at (a - hi + 1) mod h; if it wraps past h - 1, the w smallest
      // values 0 .. w-1 (q = lo .. lo+w-1) come first
      auto rect_pos = [&](int a, int p) {
        const int start = pos_mod(a - hi + 1, h);
        const int u = pos_mod(a - p, h);
        const int w = start + gs - h;  // > 0 iff the range wraps
        if (w > 0 && u < w) return u;
        return (hi - 1 - p) + (w > 0 ? w : 0);
      };
      for (int p = lo; p < hi; ++p) {
        push_job();
        for (int s = 0; s <= n; ++s) {
          int i, j;
          if (s < h) {
            i = p;
            j = h + (p + s) % h;
          } else if (s < n - p) {
            i = p;
            j = p + (s - h);
          } else {
            i = n - 1 - p;
            j = (n - 1) - (s - (n - p));
          }
          int rank;
          if (j >= h) {
            const int base = lo + std::max(0, lo - (n - 1 - j));
            rank = (i < h) ? base + rect_pos(j - h, p) : base + gs + (hi - 1 - p);
          } else {
            rank = std::min(lo, j + 1) + std::min(hi - 1, j) - p;
          }
          t.tasks.push_back({i, j, rank});
        }
      }
    }
  } else {
    return false;
  }
  push_job();
  *out = std::move(t);
  return true;
}

const ScheduleTable* cached_schedule(int schedule, int n, int mask) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int>, ScheduleTable*> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_tuple(schedule, n, mask);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  auto* t = new ScheduleTable();
  if (!build_schedule(schedule, n, mask, t)) {
    delete t;
    t = nullptr;
  }
  cache[key] = t;
  return t;
}

// --- DAG model --------------------------------------------------------------
// Each SM alternates compute (weight c) and reduction (weight r) phases of the
// tasks of the job it claimed; the reduction of rank k on dQ_j of a head may
// start only after rank k-1's reduction ended (zero-weight edge).  A
// free SM claims the next job in head-major order; simultaneous claims go to
// the lower SM index (AMB-7).  The makespan is the critical path.
int64_t critical_path(const ScheduleTable& t, int m, int n_sm, int64_t c, int64_t r) {
  const int J = t.jobs, n = t.n;
  const int64_t total_jobs = static_cast<int64_t>(J) * m;
  // Reduction end time of (head, j, rank); -1 = not yet started.
  std::vector<int64_t> red_end(static_cast<size_t>(m) * n * n, -1);
  auto slot = [&](int head, int j, int rank) {
    return (static_cast<size_t>(head) * n + j) * n + rank;
  };
  struct SmState {
    int64_t job = -1;   // global job index (head * J + local)
    int task = 0;       // index into the job's task range
    int64_t c_end = 0;  // compute end of the blocked task
    bool blocked = false;
  };
  std::vector<SmState> sm(n_sm);
  // blocked_on[slot] = SM waiting for that reduction to start.
  std::vector<int> blocked_on(static_cast<size_t>(m) * n * n, -1);
  // Event = (time, order, sm).  order: 0 compute end, 1 reduction end, 2 free.
  using Ev = std::tuple<int64_t, int, int>;
  std::priority_queue<Ev, std::vector<Ev>, std::greater<Ev>> pq;
  for (int s = 0; s < n_sm; ++s) pq.emplace(0, 2, s);
  int64_t next_job = 0, makespan = 0;
  int64_t finished_jobs = 0;

  auto cur_task = [&](const SmState& st) -> const Task& {
    return t.tasks[t.job_begin[st.job % J] + st.task];
  };
  // Starts the reduction of SM s's current task no earlier than `ready`;
  // wakes the SM waiting for the next rank of the same dQ tile.
  std::vector<std::pair<int, int64_t>> wake;  // explicit stack (sm, ready)
  auto begin_reduction = [&](int s0, int64_t ready0) {
    wake.emplace_back(s0, ready0);
    while (!wake.empty()) {
      auto [s, ready] = wake.back();
      wake.pop_back();
      SmState& st = sm[s];
      const Task& tk = cur_task(st);
      const int head = static_cast<int>(st.job / J);
      const int64_t end = ready + r;
      red_end[slot(head, tk.q, tk.rank)] = end;
      st.blocked = false;
      pq.emplace(end, 1, s);
      const size_t nxt = slot(head, tk.q, tk.rank);
      const int w = blocked_on[nxt];
      if (w >= 0) {
        blocked_on[nxt] = -1;
        wake.emplace_back(w, std::max(sm[w].c_end, end));
      }
    }
  };

  while (!pq.empty()) {
    auto [time, order, s] = pq.top();
    pq.pop();
    if (time > makespan) makespan = time;
    SmState& st = sm[s];
    if (order == 2) {
      if (next_job >= total_jobs) {
        st.job = -1;
        continue;
      }
      st.job = next_job++;
      st.task = 0;
      pq.emplace(time + c, 0, s);
    } else if (order == 0) {
      const Task& tk = cur_task(st);
      const int head = static_cast<int>(st.job / J);
      if (tk.rank == 0) {
        begin_reduction(s, time);
      } else {
        const int64_t pred = red_end[slot(head, tk.q, tk.rank - 1)];
        if (pred >= 0) {
          begin_reduction(s, std::max(time, pred));
        } else {
          st.blocked = true;
          st.c_end = time;
          blocked_on[slot(head, tk.q, tk.rank - 1)] = s;
        }
      }
    } else {
      const int ntask = t.job_begin[st.job % J + 1] - t.job_begin[st.job % J];
      if (st.task + 1 < ntask) {
        ++st.task;
        pq.emplace(time + c, 0, s);
      } else {
        ++finished_jobs;
        pq.emplace(time, 2, s);
      }
    }
  }
  if (finished_jobs != total_jobs) return -1;
  return makespan;
}

}  // namespace dash
