// Host-side space-time planner: domain types, cost model, request queue,
// dynamic batcher and latency monitor.
//
// Semantics follow the reference scheduler exactly (the plan parity contract,
// SURVEY §8 a1-a15); the representation is our own:
//   * plan costs are computed from integer totals (flops/bytes/blocks are
//     exact int64 sums, so run-length grouping cannot change a cost) rather
//     than by materialising KernelGroup vectors per probe;
//   * the variable-size pool keeps suffix totals so the SLO probe over "the
//     whole remaining pool" (scheduler.cpp:123-126) is O(1) per chunk.
// All double arithmetic keeps the reference expression order; the library is
// compiled with -ffp-contract=off so results are bit-identical.
#pragma once

#include <cstdint>
#include <deque>
#include <map>
#include <span>
#include <stdexcept>
#include <string>
#include <unordered_set>
#include <vector>

namespace gmb {

using TimeNs = std::int64_t;

// vtime.hpp:13-19
TimeNs to_ns(double seconds);
double to_seconds(TimeNs t);

// gemm.hpp:11-20 — ordering is lexicographic (m, n, k); the queue's group
// order depends on it.
struct Shape {
  std::int64_t m = 1, n = 1, k = 1;
  bool valid() const { return m >= 1 && n >= 1 && k >= 1; }
  bool operator==(const Shape&) const = default;
  auto operator<=>(const Shape&) const = default;
};

// gemm.hpp:23-31
struct Conv {
  std::int64_t image_h = 1, image_w = 1, kernel_h = 1, kernel_w = 1;
  std::int64_t in_channels = 1, out_channels = 1, stride = 1, padding = 0;
};

inline std::int64_t flops_of(const Shape& s) { return 2 * s.m * s.n * s.k; }        // gemm.hpp:33-35
inline std::int64_t bytes_of(const Shape& s, std::int64_t e = 4) {                   // gemm.hpp:38-40
  return e * (s.m * s.k + s.k * s.n + s.m * s.n);
}
Shape lower_conv(const Conv& c);                                                     // gemm.hpp:44-51
inline Shape with_batch(const Shape& s, std::int64_t b) { return {s.m * b, s.n, s.k}; }  // gemm.hpp:54-56
std::string key_of(const Shape& s);                                                  // gemm.hpp:58-60

// device.hpp:13-30
struct Device {
  double peak_flops = 14e12;
  double mem_bandwidth = 900e9;
  std::int64_t sm_count = 80;
  std::int64_t blocks_per_sm = 2;
  double launch_overhead = 5e-6;
  double context_switch_overhead = 1e-3;
  double planning_overhead = 50e-6;
  double mem_capacity = 16e9;
  double process_context_bytes = 800e6;
  std::int64_t tile_m = 64;
  std::int64_t tile_n = 64;
  double space_sched_penalty = 1.5;
  double launch_serialization = 0.5;
  // b200 extension (0 = the reference's pure roofline): a super-kernel lasts
  // at least its waves x (tile_latency + k-blocks of its longest-K member x
  // kblock_latency) -- few-tile, long-K plans are latency-bound on the
  // persistent kernel (a k-block = 64 of K; tools/calibrate_b200.py fits both)
  double tile_latency = 0;
  double kblock_latency = 0;

  std::int64_t slots() const { return sm_count * blocks_per_sm; }
  void check() const;  // device.cpp:19-39
};
Device v100_device();  // device.cpp:41-59
Device b200_device();  // this build's profile (see capi.cpp for provenance)

// cost_model.hpp:14-27
struct Cost {
  std::int64_t flops = 0, bytes = 0, blocks = 0;
  double duration = 0;
  std::int64_t waves = 0;
};
struct Group {
  Shape shape;
  std::int64_t count = 1;
};

std::int64_t tiles_of(const Shape& s, const Device& d);  // cost_model.cpp:14-16
// cost_model.cpp:18-46 over explicit groups (validates every group).
Cost roofline(std::span<const Group> groups, const Device& d, std::int64_t slot_budget,
              std::int64_t launches);
// Same formula from pre-validated integer totals.
// kb_max: k-blocks (64 of K) of the longest-K member (the latency term).
Cost roofline_totals(std::int64_t flops, std::int64_t bytes, std::int64_t blocks,
                     const Device& d, std::int64_t slot_budget, std::int64_t launches, std::int64_t kb_max = 0);
inline std::int64_t kblocks_of(const Shape& s) { return (s.k + 63) / 64; }

// scheduler.hpp:17-25 (+ B200 extension field `batch`, never read here)
struct Request {
  std::uint64_t id = 0;
  int tenant = 0;
  Shape shape;
  TimeNs enqueue = 0;
  TimeNs deadline = 0;
  int layer = 0;
  std::uint32_t pass = 0;
  std::uint32_t batch = 1;
};

// scheduler.hpp:28-34
struct Policy {
  double max_wait = 2e-3;
  std::int64_t target_batch = 1;
  bool allow_variable_size = false;
  double slo_safety_margin = 0.0;
  double variable_inefficiency = 1.10;
  // B200 extension (not in the reference): a formed super-kernel may fill up
  // to `max_waves` waves of block slots.  1 == the reference's one-wave cap
  // (scheduler.cpp:170-171, :135-144) and is the plan-parity setting; the
  // persistent super-kernel makes larger values meaningful ("b200 mode").
  std::int64_t max_waves = 1;
};

// scheduler.hpp:37-42
struct Plan {
  std::string signature;
  std::vector<Request> members;
  bool uniform = true;
  Cost cost;
};

// scheduler.hpp:44-50
struct Health {
  int tenant = 0;
  double ewma = 0;
  double alpha = 0.2;
  std::int64_t count = 0;
  bool evicted = false;
};

// scheduler.hpp:52-56
struct SignatureCache {
  std::map<std::string, Cost> entries;
  std::int64_t hits = 0, misses = 0;
};

// scheduler.hpp:59-80: shape-grouped FIFO.  Groups iterate in ascending shape
// order; a group's requests keep insertion order.
class Queue {
 public:
  void push(const Request& r);  // scheduler.cpp:8-16
  std::int64_t size() const { return size_; }
  bool empty() const { return size_ == 0; }
  std::vector<Request> drop_tenant(int tenant);  // scheduler.cpp:18-35
  const std::map<Shape, std::deque<Request>>& groups() const { return groups_; }

 private:
  friend std::vector<Plan> form_plans(Queue&, TimeNs, const Policy&, const Device&);
  std::map<Shape, std::deque<Request>> groups_;
  std::unordered_set<std::uint64_t> ids_;
  std::int64_t size_ = 0;
};

double headroom(const Request& r, TimeNs now, double predicted, const Policy& p);  // scheduler.cpp:37-41
Cost plan_cost(std::span<const Request> members, bool uniform, const Policy& p,
               const Device& d);                                                     // scheduler.cpp:43-61
std::vector<Plan> form_plans(Queue& q, TimeNs now, const Policy& p, const Device& d);  // scheduler.cpp:96-199
double charge(const Plan& plan, SignatureCache& cache, const Device& d);          // scheduler.cpp:201-212
void observe(Health& h, double seconds);                                             // scheduler.cpp:214-223
std::vector<int> stragglers(std::span<const Health> hs, double ratio, std::int64_t min_obs);  // :246-271
std::vector<Request> evict_tenant(std::vector<Health>& hs, Queue& q, int tenant);    // :225-244

// metrics.cpp:10-28
double geometric_mean(std::span<const double> v);
double nearest_rank(std::vector<double> v, double pct);

// Tile-dispatch table: member order, m-tile-major, n-tile.
struct Tile {
  std::uint16_t member, flags, m_tile, n_tile;
};
std::vector<Tile> tile_table(const Plan& plan, const Device& d);

}  // namespace gmb
