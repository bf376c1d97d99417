// Host-side schedule generator and DAG model of the DASH backward (L1).
//
// PAPER.md §3.  Indices follow §3 (Fig. 2): i = KV tile,
// j = Q tile, n = tiles per head.  Independent of oracle/ by construction:
// ranks come from the closed forms of DESIGN.md §Schedules, not from a sort.
#pragma once
#include <cstdint>
#include <vector>

namespace dash {

enum Schedule : int { kNaive = 0, kDescending = 1, kShift = 2 };
enum Mask : int { kFull = 0, kCausal = 1 };

struct Task {
  int32_t kv;    // i
  int32_t q;     // j
  int32_t rank;  // position of this contribution in dQ_j's reduction order
};

struct ScheduleTable {
  int n = 0;
  int schedule = 0, mask = 0;
  int jobs = 0;                   // jobs per head (n, or n/2 for SHIFT causal)
  int coresident = 0;             // SHIFT: jobs that must be co-resident (largest group)
  std::vector<int32_t> job_begin;  // jobs + 1 offsets into tasks
  std::vector<Task> tasks;         // per job, in visiting order
  int max_rank_plus1(int j) const;  // contributions to dQ_j (n or j+1)
};

// SHIFT full with more than kShiftGroup KV tiles runs in groups of at most
// kShiftGroup tiles (AMB-30), SHIFT causal with more than kShiftGroup pairs
// in groups of at most kShiftGroup pairs (AMB-35): a fixed constant, so
// tables never depend on the device.
constexpr int kShiftGroup = 128;

// Returns false (and leaves *out empty) for an unsupported combination.
bool build_schedule(int schedule, int n, int mask, ScheduleTable* out);

// Shared, thread-safe cache of built tables keyed by (schedule, n, mask).
const ScheduleTable* cached_schedule(int schedule, int n, int mask);

// Event model of §3 on n_sm SMs with m heads; returns -1 on deadlock.
int64_t critical_path(const ScheduleTable& t, int m, int n_sm, int64_t c, int64_t r);

}  // namespace dash
