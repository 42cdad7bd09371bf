// Space-time planner (see planner.hpp for the parity contract).
#include "planner.hpp"

#include <algorithm>
#include <cmath>
#include <limits>

namespace gmb {

// ---------------------------------------------------------------- time/shapes

TimeNs to_ns(double seconds) { return static_cast<TimeNs>(std::llround(seconds * 1e9)); }
double to_seconds(TimeNs t) { return static_cast<double>(t) * 1e-9; }

Shape lower_conv(const Conv& c) {
  // Output extent per spatial dim; rows = output positions, cols = C_out,
  // inner = unrolled filter patch (gemm.hpp:44-51).
  const std::int64_t oh = (c.image_h + 2 * c.padding - c.kernel_h) / c.stride + 1;
  const std::int64_t ow = (c.image_w + 2 * c.padding - c.kernel_w) / c.stride + 1;
  if (oh < 1 || ow < 1) throw std::invalid_argument("im2col: non-positive output dims");
  return Shape{oh * ow, c.out_channels, c.kernel_h * c.kernel_w * c.in_channels};
}

std::string key_of(const Shape& s) {
  std::string out = std::to_string(s.m);
  out += 'x';
  out += std::to_string(s.n);
  out += 'x';
  out += std::to_string(s.k);
  return out;
}

// ---------------------------------------------------------------- device

void Device::check() const {
  if (peak_flops <= 0) throw std::invalid_argument("device: peak_flops must be > 0");
  if (mem_bandwidth <= 0) throw std::invalid_argument("device: mem_bandwidth must be > 0");
  if (sm_count * blocks_per_sm < 1)
    throw std::invalid_argument("device: sm_count*blocks_per_sm must be >= 1");
  if (launch_overhead < 0 || context_switch_overhead < 0 || planning_overhead < 0)
    throw std::invalid_argument("device: overheads must be >= 0");
  if (tile_m < 1 || tile_n < 1) throw std::invalid_argument("device: tiles must be >= 1");
  if (space_sched_penalty < 1)
    throw std::invalid_argument("device: space_sched_penalty must be >= 1");
  if (launch_serialization < 0 || launch_serialization > 1)
    throw std::invalid_argument("device: launch_serialization must be in [0,1]");
  if (mem_capacity <= 0) throw std::invalid_argument("device: mem_capacity must be > 0");
  if (process_context_bytes < 0)
    throw std::invalid_argument("device: process_context_bytes must be >= 0");
  if (tile_latency < 0 || kblock_latency < 0) throw std::invalid_argument("device: latencies must be >= 0");
}

Device v100_device() {
  Device d;  // shipped calibration fit, device.cpp:41-59 / profiles/v100.json
  d.peak_flops = 14e12;
  d.mem_bandwidth = 900e9;
  d.sm_count = 80;
  d.blocks_per_sm = 2;
  d.launch_overhead = 2.2e-06;
  d.context_switch_overhead = 0.000196875;
  d.planning_overhead = 50e-6;
  d.mem_capacity = 16e9;
  d.process_context_bytes = 800e6;
  d.tile_m = 64;
  d.tile_n = 64;
  d.space_sched_penalty = 1.55;
  d.launch_serialization = 1.0;
  return d;
}

Device b200_device() {
  Device d;
  d.peak_flops = 1388.8e12;      // measured sustained dense bf16 (MEASURED_PEAKS.json)
  d.mem_bandwidth = 6546.9e9;    // measured HBM copy bandwidth
  d.sm_count = 148;
  d.blocks_per_sm = 1;           // one persistent CTA per SM
  d.launch_overhead = 2.0e-6;
  d.context_switch_overhead = 25e-6;
  d.planning_overhead = 20e-6;   // tile table build + upload on a cache miss
  d.mem_capacity = 180e9;
  d.process_context_bytes = 500e6;
  d.tile_m = 128;                // super-kernel CTA tile (UMMA M)
  d.tile_n = 256;                // super-kernel CTA tile (max UMMA N)
  d.space_sched_penalty = 1.0;
  d.launch_serialization = 1.0;
  return d;
}

// ---------------------------------------------------------------- cost model

namespace {
inline std::int64_t cdiv(std::int64_t a, std::int64_t b) { return (a + b - 1) / b; }
}  // namespace

std::int64_t tiles_of(const Shape& s, const Device& d) {
  return cdiv(s.m, d.tile_m) * cdiv(s.n, d.tile_n);
}

Cost roofline_totals(std::int64_t flops, std::int64_t bytes, std::int64_t blocks,
                     const Device& d, std::int64_t slot_budget, std::int64_t launches, std::int64_t kb_max) {
  Cost c;
  c.flops = flops;
  c.bytes = bytes;
  c.blocks = blocks;
  c.waves = cdiv(blocks, slot_budget);
  // Compute side scaled by mean resident-block fraction; memory side sees the
  // whole device bandwidth (cost_model.cpp:36-44).  Expression order matters.
  const double eff = static_cast<double>(blocks) / static_cast<double>(c.waves * slot_budget);
  const double t_compute = static_cast<double>(flops) / (d.peak_flops * eff);
  const double t_memory = static_cast<double>(bytes) / d.mem_bandwidth;
  double t = std::max(t_compute, t_memory);
  if (d.tile_latency > 0 || d.kblock_latency > 0)  // b200 latency term (absent in the reference profiles)
    t = std::max(t, static_cast<double>(c.waves) *
                        (d.tile_latency + static_cast<double>(kb_max) * d.kblock_latency));
  c.duration = static_cast<double>(launches) * d.launch_overhead + t;
  return c;
}

Cost roofline(std::span<const Group> groups, const Device& d, std::int64_t slot_budget,
              std::int64_t launches) {
  if (groups.empty()) throw std::invalid_argument("empty dispatch");
  if (slot_budget < 1 || slot_budget > d.slots())
    throw std::invalid_argument("slot_budget out of range");
  if (launches < 1) throw std::invalid_argument("launches must be >= 1");
  std::int64_t flops = 0, bytes = 0, blocks = 0, kb_max = 0;
  for (const Group& g : groups) {
    if (g.count < 1 || !g.shape.valid()) throw std::invalid_argument("invalid kernel group");
    flops += g.count * flops_of(g.shape);
    bytes += g.count * bytes_of(g.shape);
    blocks += g.count * tiles_of(g.shape, d);
    kb_max = std::max(kb_max, kblocks_of(g.shape));
  }
  return roofline_totals(flops, bytes, blocks, d, slot_budget, launches, kb_max);
}

// ---------------------------------------------------------------- queue

void Queue::push(const Request& r) {
  if (!r.shape.valid()) throw std::invalid_argument("enqueue: invalid shape");
  if (!ids_.insert(r.id).second)
    throw std::invalid_argument("enqueue: duplicate request id " + std::to_string(r.id));
  groups_[r.shape].push_back(r);
  ++size_;
}

std::vector<Request> Queue::drop_tenant(int tenant) {
  std::vector<Request> out;
  for (auto g = groups_.begin(); g != groups_.end();) {
    std::deque<Request>& fifo = g->second;
    std::deque<Request> kept;
    for (Request& r : fifo) {
      if (r.tenant == tenant) {
        ids_.erase(r.id);
        out.push_back(r);
        --size_;
      } else {
        kept.push_back(r);
      }
    }
    fifo.swap(kept);
    g = fifo.empty() ? groups_.erase(g) : std::next(g);
  }
  return out;
}

// ---------------------------------------------------------------- batcher

double headroom(const Request& r, TimeNs now, double predicted, const Policy& p) {
  return to_seconds(r.deadline - now) - predicted * (1.0 + p.slo_safety_margin);
}

namespace {

// Integer totals of a member set; a plan's cost is a pure function of them.
struct Totals {
  std::int64_t flops = 0, bytes = 0, blocks = 0, kb_max = 0;
  void add(const Shape& s, const Device& d, std::int64_t times = 1) {
    flops += times * flops_of(s);
    bytes += times * bytes_of(s);
    blocks += times * tiles_of(s, d);
    kb_max = std::max(kb_max, kblocks_of(s));
  }
};

Cost cost_from(const Totals& t, bool uniform, const Policy& p, const Device& d) {
  if (t.blocks == 0) throw std::invalid_argument("empty dispatch");
  Cost c = roofline_totals(t.flops, t.bytes, t.blocks, d, d.slots(), 1, t.kb_max);
  if (!uniform) c.duration *= p.variable_inefficiency;
  return c;
}

std::string uniform_signature(const Shape& s, std::size_t count) {
  std::string sig = key_of(s);
  sig += '*';
  sig += std::to_string(count);
  return sig;
}

std::string variable_signature(std::span<const Request> members) {
  std::vector<Shape> shapes;
  shapes.reserve(members.size());
  for (const Request& r : members) shapes.push_back(r.shape);
  std::sort(shapes.begin(), shapes.end());
  std::string sig = "v:";
  for (const Shape& s : shapes) {
    sig += key_of(s);
    sig += ';';
  }
  return sig;
}

Plan seal(std::vector<Request> members, bool uniform, const Policy& p, const Device& d) {
  // target_batch < 1 would form an empty super-kernel (undefined in the
  // reference, which dereferences members.front()); fail loudly instead.
  if (members.empty()) throw std::invalid_argument("empty dispatch");
  Plan plan;
  plan.uniform = uniform;
  if (uniform) {
    for (const Request& r : members)
      if (!(r.shape == members.front().shape)) {
        plan.uniform = false;
        break;
      }
  }
  plan.signature = plan.uniform ? uniform_signature(members.front().shape, members.size())
                                : variable_signature(members);
  plan.cost = plan_cost(members, plan.uniform, p, d);
  plan.members = std::move(members);
  return plan;
}

}  // namespace

Cost plan_cost(std::span<const Request> members, bool uniform, const Policy& p, const Device& d) {
  if (members.empty()) throw std::invalid_argument("empty dispatch");
  Totals t;
  for (const Request& r : members) {
    if (!r.shape.valid()) throw std::invalid_argument("invalid kernel group");
    t.add(r.shape, d);
  }
  return cost_from(t, uniform, p, d);
}

std::vector<Plan> form_plans(Queue& q, TimeNs now, const Policy& p, const Device& d) {
  std::vector<Plan> out;
  const TimeNs max_wait_ns = to_ns(p.max_wait);
  // block slots one super-kernel may fill (reference: exactly one wave)
  const std::int64_t slots = d.slots() * std::max<std::int64_t>(1, p.max_waves);

  if (p.allow_variable_size) {
    // Variable-size (MAGMA-style) mode: one pool in arrival order, chunks
    // filling up to one wave of block slots (scheduler.cpp:102-164).
    std::vector<Request> pool;
    pool.reserve(static_cast<std::size_t>(q.size_));
    for (auto& [shape, fifo] : q.groups_) pool.insert(pool.end(), fifo.begin(), fifo.end());
    std::stable_sort(pool.begin(), pool.end(), [](const Request& a, const Request& b) {
      return a.enqueue != b.enqueue ? a.enqueue < b.enqueue : a.id < b.id;
    });
    // suffix totals: cost of "the whole remaining pool" from position i
    std::vector<Totals> suffix(pool.size() + 1);
    for (std::size_t i = pool.size(); i-- > 0;) {
      suffix[i] = suffix[i + 1];
      suffix[i].add(pool[i].shape, d);
    }
    // earliest deadline in the remaining pool: headroom is monotone in the
    // deadline for a fixed prediction, so the minimum decides the SLO leg.
    std::vector<TimeNs> min_deadline(pool.size() + 1, std::numeric_limits<TimeNs>::max());
    for (std::size_t i = pool.size(); i-- > 0;)
      min_deadline[i] = std::min(min_deadline[i + 1], pool[i].deadline);

    std::size_t pos = 0;
    while (pos < pool.size()) {
      const std::size_t left = pool.size() - pos;
      const bool size_ok = static_cast<std::int64_t>(left) >= p.target_batch;
      bool forced = now - pool[pos].enqueue >= max_wait_ns;
      if (!forced) {
        const double predicted = cost_from(suffix[pos], false, p, d).duration;
        Request probe;
        probe.deadline = min_deadline[pos];
        forced = headroom(probe, now, predicted, p) <= 0;
      }
      if (!size_ok && !forced) break;
      std::vector<Request> chunk;
      std::int64_t used = 0;
      while (pos < pool.size()) {
        const std::int64_t b = tiles_of(pool[pos].shape, d);
        if (!chunk.empty() && used + b > slots) break;
        if (size_ok && !forced && static_cast<std::int64_t>(chunk.size()) >= p.target_batch) break;
        used += b;
        chunk.push_back(pool[pos++]);
      }
      out.push_back(seal(std::move(chunk), false, p, d));
    }
    // Remove the dispatched members from their groups (first match by id).
    for (const Plan& plan : out) {
      for (const Request& r : plan.members) {
        auto g = q.groups_.find(r.shape);
        std::deque<Request>& fifo = g->second;
        for (auto it = fifo.begin(); it != fifo.end(); ++it) {
          if (it->id == r.id) {
            fifo.erase(it);
            q.ids_.erase(r.id);
            --q.size_;
            break;
          }
        }
        if (fifo.empty()) q.groups_.erase(g);
      }
    }
    return out;
  }

  // Uniform mode: each shape group independently, ascending shape order.
  for (auto g = q.groups_.begin(); g != q.groups_.end();) {
    const Shape shape = g->first;
    std::deque<Request>& fifo = g->second;
    const std::int64_t tiles = tiles_of(shape, d);
    const std::int64_t wave_cap = std::max<std::int64_t>(1, slots / tiles);
    Totals one;
    one.add(shape, d);
    while (!fifo.empty()) {
      const std::int64_t n = static_cast<std::int64_t>(fifo.size());
      const bool size_ok = n >= p.target_batch;
      bool forced = now - fifo.front().enqueue >= max_wait_ns;
      if (!forced) {
        // prediction = uniform plan over the first min(n, max(target,1))
        const std::int64_t probe = std::min<std::int64_t>(n, std::max<std::int64_t>(p.target_batch, 1));
        Totals t;
        t.flops = probe * one.flops;
        t.bytes = probe * one.bytes;
        t.blocks = probe * one.blocks;
        t.kb_max = one.kb_max;
        const double predicted = cost_from(t, true, p, d).duration;
        for (const Request& r : fifo) {
          if (headroom(r, now, predicted, p) <= 0) {
            forced = true;
            break;
          }
        }
      }
      if (!size_ok && !forced) break;
      const std::int64_t take = std::min(size_ok ? p.target_batch : n, wave_cap);
      if (take < 1) throw std::invalid_argument("empty dispatch");
      std::vector<Request> members(fifo.begin(), fifo.begin() + take);
      for (const Request& r : members) q.ids_.erase(r.id);
      fifo.erase(fifo.begin(), fifo.begin() + take);
      q.size_ -= take;
      out.push_back(seal(std::move(members), true, p, d));
    }
    g = fifo.empty() ? q.groups_.erase(g) : std::next(g);
  }
  return out;
}

double charge(const Plan& plan, SignatureCache& cache, const Device& d) {
  double duration = plan.cost.duration;
  if (cache.entries.emplace(plan.signature, plan.cost).second) {
    ++cache.misses;
    duration += d.planning_overhead;
  } else {
    ++cache.hits;
  }
  return duration;
}

// ---------------------------------------------------------------- monitor

void observe(Health& h, double seconds) {
  if (seconds < 0) throw std::invalid_argument("negative latency");
  h.ewma = h.count == 0 ? seconds : h.alpha * seconds + (1.0 - h.alpha) * h.ewma;
  ++h.count;
}

std::vector<int> stragglers(std::span<const Health> hs, double ratio, std::int64_t min_obs) {
  if (ratio <= 1.0) throw std::invalid_argument("threshold_ratio must be > 1");
  std::vector<double> live;
  for (const Health& h : hs)
    if (!h.evicted && h.count > 0) live.push_back(h.ewma);
  if (live.size() < 2) return {};
  std::sort(live.begin(), live.end());
  const std::size_t mid = live.size() / 2;
  const double median = live.size() % 2 ? live[mid] : 0.5 * (live[mid - 1] + live[mid]);
  std::vector<int> out;
  for (const Health& h : hs)
    if (!h.evicted && h.count >= min_obs && h.ewma > ratio * median) out.push_back(h.tenant);
  return out;
}

std::vector<Request> evict_tenant(std::vector<Health>& hs, Queue& q, int tenant) {
  auto it = std::find_if(hs.begin(), hs.end(), [&](const Health& h) { return h.tenant == tenant; });
  if (it == hs.end()) throw std::invalid_argument("evict: unknown tenant " + std::to_string(tenant));
  if (it->evicted)
    throw std::invalid_argument("evict: tenant " + std::to_string(tenant) + " already evicted");
  it->evicted = true;
  return q.drop_tenant(tenant);
}

// ---------------------------------------------------------------- metrics

double geometric_mean(std::span<const double> v) {
  if (v.empty()) throw std::invalid_argument("geomean of empty set");
  double acc = 0;
  for (double x : v) {
    if (x <= 0) throw std::invalid_argument("geomean requires positive values");
    acc += std::log(x);
  }
  return std::exp(acc / static_cast<double>(v.size()));
}

double nearest_rank(std::vector<double> v, double pct) {
  if (v.empty()) throw std::invalid_argument("percentile of empty set");
  std::sort(v.begin(), v.end());
  std::size_t rank = static_cast<std::size_t>(std::ceil(pct / 100.0 * static_cast<double>(v.size())));
  rank = std::clamp<std::size_t>(rank, 1, v.size());
  return v[rank - 1];
}

// ---------------------------------------------------------------- tile table

std::vector<Tile> tile_table(const Plan& plan, const Device& d) {
  std::vector<Tile> out;
  if (plan.members.size() > 0xFFFF) throw std::invalid_argument("tile table: too many members");
  for (std::size_t j = 0; j < plan.members.size(); ++j) {
    const Shape& s = plan.members[j].shape;
    const std::int64_t mt = cdiv(s.m, d.tile_m), nt = cdiv(s.n, d.tile_n);
    if (mt > 0xFFFF || nt > 0xFFFF) throw std::invalid_argument("tile table: tile index overflow");
    for (std::int64_t a = 0; a < mt; ++a)
      for (std::int64_t b = 0; b < nt; ++b)
        out.push_back(Tile{static_cast<std::uint16_t>(j), 0, static_cast<std::uint16_t>(a),
                           static_cast<std::uint16_t>(b)});
  }
  return out;
}

}  // namespace gmb
