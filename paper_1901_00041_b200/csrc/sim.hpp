// Space-time driver on a virtual clock: the closed-loop semantics of the
// reference engine's run_space_time (proj/src/sim.cpp:398-581), restated over
// the planner in planner.hpp.  The B200 runtime uses its dispatch sequence as
// the plan stream it replays on the GPU; the parity tests compare it against
// the reference engine event for event.
#pragma once

#include <cstdint>
#include <optional>
#include <vector>

#include "planner.hpp"

namespace gmb {

struct Detector {  // sim.hpp:32-37
  double ewma_alpha = 0.2;
  std::int64_t min_observations = 10;
  double threshold_ratio = 1.5;
  bool evict_stragglers = true;
};

struct Degradation {  // sim.hpp:41-45
  int tenant = 0;
  double slowdown = 1.0;
  double start = 0;
};

struct SpaceTimeConfig {
  Device device;
  Policy scheduler;
  Detector detector;
  std::vector<Shape> layers;  // shared by every tenant (sim.cpp:28-31)
  int tenants = 1;
  int concurrency = 1;
  double slo_latency = 0.1;
  double duration = 1.0;
  double warmup = 0.1;
  bool microbench = false;
  std::optional<Degradation> degradation;

  void check() const;  // the space-time subset of SimConfig::validate (sim.cpp:15-58)
};

struct Dispatch {
  TimeNs start = 0, end = 0;
  std::int64_t flops = 0;
  double occupancy = 0;
  std::vector<std::uint64_t> members;
  std::string signature;
  std::vector<Request> requests;  // full member records (for GPU replay)
};

struct Completion {
  std::uint64_t id = 0;
  int tenant = 0;
  TimeNs enqueue = 0, dispatch = 0, complete = 0;
  bool slo_met = false;
  std::int64_t flops = 0;
};

struct SpaceTimeTrace {
  std::vector<Dispatch> events;
  std::vector<Completion> completions;
  std::vector<std::uint64_t> cancellations;
  std::vector<int> evicted;
  std::vector<TimeNs> eviction_times;
  std::int64_t cache_hits = 0, cache_misses = 0;
  std::int64_t dispatched_flops = 0, completed_flops = 0;
};

SpaceTimeTrace simulate_space_time(const SpaceTimeConfig& cfg);

// One closed-loop round on the virtual clock: every listed tenant submits one
// forward pass at `start`; the space-time loop (the dispatch FIFO, formation
// only when the FIFO is empty, completion fan-out, wake timer — sim.cpp:452-576)
// runs until every pass has completed.  Tenants may have different layer lists
// (the heterogeneous extension; the reference rejects them, sim.cpp:28-31).
// Returns the dispatch sequence; `cache` and `next_id` persist across rounds.
struct RoundTenant {
  int tenant = 0;
  std::vector<Shape> layers;
  TimeNs slo_ns = 0;
};
struct RoundDispatch {
  Plan plan;
  TimeNs start = 0, end = 0;
};
struct RoundResult {
  std::vector<RoundDispatch> dispatches;
  std::vector<std::pair<int, TimeNs>> pass_complete;  // (tenant, virtual completion)
};
RoundResult plan_round(const std::vector<RoundTenant>& tenants, TimeNs start, const Policy& policy, const Device& dev,
                       SignatureCache& cache, std::uint64_t& next_id);

}  // namespace gmb
