// Virtual-clock space-time driver (see sim.hpp).
#include "sim.hpp"

#include <algorithm>
#include <cmath>
#include <deque>
#include <limits>
#include <map>
#include <queue>
#include <tuple>

namespace gmb {

void SpaceTimeConfig::check() const {
  device.check();
  if (tenants < 1) throw std::invalid_argument("config: tenants must be non-empty");
  if (!(duration > warmup) || warmup < 0)
    throw std::invalid_argument("config: need duration > warmup >= 0");
  if (layers.empty()) throw std::invalid_argument("config: tenant has no layers");
  for (const Shape& s : layers)
    if (!s.valid()) throw std::invalid_argument("config: invalid layer shape");
  if (concurrency < 1) throw std::invalid_argument("config: concurrency must be >= 1");
  if (slo_latency <= 0) throw std::invalid_argument("config: slo_latency must be > 0");
  if (scheduler.max_wait <= 0) throw std::invalid_argument("config: scheduler.max_wait must be > 0");
  if (scheduler.target_batch < 0)
    throw std::invalid_argument("config: scheduler.target_batch must be >= 0 (0 = auto)");
  if (detector.threshold_ratio <= 1)
    throw std::invalid_argument("config: detector.threshold_ratio must be > 1");
  if (degradation) {
    if (degradation->tenant < 0 || degradation->tenant >= tenants)
      throw std::invalid_argument("config: degradation names unknown tenant");
    if (degradation->slowdown < 1.0)
      throw std::invalid_argument("config: degradation slowdown must be >= 1");
  }
}

namespace {

// Heap entry ordered by (time, kind, tenant, seq) — sim.cpp:386-389.
struct Ev {
  TimeNs time = 0;
  int kind = 0;  // 0 request ready, 1 super-kernel done, 2 wake-up
  int tenant = 0;
  std::uint64_t seq = 0;
  Request req;
  bool operator>(const Ev& o) const {
    return std::tie(time, kind, tenant, seq) > std::tie(o.time, o.kind, o.tenant, o.seq);
  }
};

struct Progress {
  std::uint64_t pass_id = 0;
  TimeNs enqueue = 0;
  TimeNs first_dispatch = -1;
};

}  // namespace

SpaceTimeTrace simulate_space_time(const SpaceTimeConfig& cfg) {
  cfg.check();
  const Device& dev = cfg.device;
  std::vector<Shape> layers = cfg.layers;
  if (cfg.microbench) layers.resize(1);
  const int n = cfg.tenants;
  const int n_layers = static_cast<int>(layers.size());
  const TimeNs horizon = to_ns(cfg.duration);
  const TimeNs slo_ns = to_ns(cfg.slo_latency);
  std::int64_t pass_flops = 0;
  for (const Shape& s : layers) pass_flops += flops_of(s);

  SpaceTimeTrace tr;
  std::uint64_t next_id = 1;
  auto fresh = [&]() { return next_id++; };

  const bool has_deg = cfg.degradation.has_value();
  const TimeNs deg_start = has_deg ? to_ns(cfg.degradation->start) : 0;
  // Tenant-local post-dispatch stretch (sim.cpp:98-110).
  auto finish_time = [&](int tenant, TimeNs start, TimeNs exec) -> TimeNs {
    const bool hit = has_deg && cfg.degradation->tenant == tenant && cfg.degradation->slowdown > 1.0 &&
                     start >= deg_start;
    if (!hit) return start + exec;
    return start + static_cast<TimeNs>(std::llround(static_cast<double>(exec) * cfg.degradation->slowdown));
  };

  Queue queue;
  SignatureCache cache;
  std::vector<Health> health(n);
  for (int t = 0; t < n; ++t) {
    health[t].tenant = t;
    health[t].alpha = cfg.detector.ewma_alpha;
  }
  std::vector<std::map<std::uint32_t, Progress>> live(n);
  std::vector<std::uint32_t> pass_counter(n, 0);

  std::priority_queue<Ev, std::vector<Ev>, std::greater<Ev>> heap;
  std::uint64_t seq = 0;
  std::deque<Plan> fifo;
  bool busy = false;
  Plan running;
  TimeNs run_start = 0, run_end = 0;

  auto begin_pass = [&](int t, TimeNs at) {
    const std::uint32_t pi = pass_counter[t]++;
    Progress pr;
    pr.pass_id = fresh();
    pr.enqueue = at;
    live[t][pi] = pr;
    Request r;
    r.id = fresh();
    r.tenant = t;
    r.shape = layers[0];
    r.enqueue = at;
    r.deadline = at + slo_ns;
    r.layer = 0;
    r.pass = pi;
    heap.push(Ev{at, 0, t, seq++, r});
  };
  auto streams = [&]() {
    std::int64_t c = 0;
    for (int t = 0; t < n; ++t)
      if (!health[t].evicted) c += cfg.concurrency;
    return c;
  };

  for (int t = 0; t < n; ++t)
    for (int k = 0; k < cfg.concurrency; ++k) begin_pass(t, 0);

  const TimeNs max_wait_ns = to_ns(cfg.scheduler.max_wait);

  while (!heap.empty()) {
    const TimeNs now = heap.top().time;
    while (!heap.empty() && heap.top().time == now) {
      const Ev ev = heap.top();
      heap.pop();
      if (ev.kind == 0) {
        if (health[ev.tenant].evicted) {
          tr.cancellations.push_back(ev.req.id);
          continue;
        }
        queue.push(ev.req);
      } else if (ev.kind == 1) {
        busy = false;
        const TimeNs exec = run_end - run_start;
        tr.completed_flops += running.cost.flops;
        for (const Request& r : running.members) {
          const TimeNs done = finish_time(r.tenant, run_start, exec);
          observe(health[r.tenant], to_seconds(done - run_start));
          if (health[r.tenant].evicted) continue;
          auto it = live[r.tenant].find(r.pass);
          if (it == live[r.tenant].end()) continue;
          Progress& pr = it->second;
          if (pr.first_dispatch < 0) pr.first_dispatch = run_start;
          if (r.layer + 1 < n_layers) {
            Request nx = r;
            nx.id = fresh();
            nx.shape = layers[r.layer + 1];
            nx.enqueue = done;
            ++nx.layer;
            heap.push(Ev{done, 0, r.tenant, seq++, nx});
          } else {
            Completion c;
            c.id = pr.pass_id;
            c.tenant = r.tenant;
            c.enqueue = pr.enqueue;
            c.dispatch = pr.first_dispatch;
            c.complete = done;
            c.slo_met = (done - pr.enqueue) <= slo_ns;
            c.flops = pass_flops;
            tr.completions.push_back(c);
            live[r.tenant].erase(it);
            begin_pass(r.tenant, done);
          }
        }
        if (cfg.detector.evict_stragglers) {
          for (int t : stragglers(health, cfg.detector.threshold_ratio, cfg.detector.min_observations)) {
            tr.evicted.push_back(t);
            tr.eviction_times.push_back(now);
            for (const Request& r : evict_tenant(health, queue, t)) tr.cancellations.push_back(r.id);
            live[t].clear();
          }
        }
      }
      // kind 2: bare wake-up
    }

    if (busy) continue;
    if (fifo.empty() && now >= horizon) continue;

    if (fifo.empty()) {
      Policy pol = cfg.scheduler;
      const std::int64_t live_streams = std::max<std::int64_t>(1, streams());
      pol.target_batch = pol.target_batch == 0 ? live_streams : std::min(pol.target_batch, live_streams);
      for (Plan& p : form_plans(queue, now, pol, dev)) fifo.push_back(std::move(p));
    }
    if (!fifo.empty()) {
      Plan p = std::move(fifo.front());
      fifo.pop_front();
      const double secs = charge(p, cache, dev);
      const TimeNs end = now + to_ns(secs);
      Dispatch d;
      d.start = now;
      d.end = end;
      d.flops = p.cost.flops;
      d.occupancy = static_cast<double>(p.cost.blocks) / static_cast<double>(p.cost.waves * dev.slots());
      d.members.reserve(p.members.size());
      for (const Request& r : p.members) d.members.push_back(r.id);
      d.signature = p.signature;
      d.requests = p.members;
      tr.dispatched_flops += p.cost.flops;
      tr.events.push_back(std::move(d));
      busy = true;
      running = std::move(p);
      run_start = now;
      run_end = end;
      heap.push(Ev{end, 1, 0, seq++, {}});
    } else if (!queue.empty() && now < horizon) {
      // Nothing triggered: wake when the earliest age or SLO deadline lands.
      // (As in the reference, a non-zero target is NOT capped here.)
      Policy pol = cfg.scheduler;
      if (pol.target_batch == 0) pol.target_batch = std::max<std::int64_t>(1, streams());
      TimeNs wake = std::numeric_limits<TimeNs>::max();
      for (const auto& [shape, grp] : queue.groups()) {
        wake = std::min(wake, grp.front().enqueue + max_wait_ns);
        const std::int64_t probe =
            std::min<std::int64_t>(static_cast<std::int64_t>(grp.size()), std::max<std::int64_t>(pol.target_batch, 1));
        const std::int64_t tiles = tiles_of(shape, dev);
        const double predicted =
            roofline_totals(probe * flops_of(shape), probe * bytes_of(shape), probe * tiles, dev, dev.slots(), 1,
                            kblocks_of(shape))
                .duration;
        const TimeNs predicted_ns = to_ns(predicted * (1.0 + pol.slo_safety_margin));
        for (const Request& r : grp) wake = std::min(wake, r.deadline - predicted_ns);
      }
      if (wake != std::numeric_limits<TimeNs>::max()) heap.push(Ev{std::max(wake, now + 1), 2, 0, seq++, {}});
    }
  }
  tr.cache_hits = cache.hits;
  tr.cache_misses = cache.misses;
  return tr;
}

RoundResult plan_round(const std::vector<RoundTenant>& tenants, TimeNs start, const Policy& policy, const Device& dev,
                       SignatureCache& cache, std::uint64_t& next_id) {
  RoundResult out;
  if (tenants.empty()) return out;
  std::map<int, const RoundTenant*> by_id;
  for (const RoundTenant& t : tenants) {
    if (t.layers.empty()) throw std::invalid_argument("config: tenant has no layers");
    if (!by_id.emplace(t.tenant, &t).second)
      throw std::invalid_argument("plan_round: duplicate tenant " + std::to_string(t.tenant));
  }
  Queue queue;
  std::priority_queue<Ev, std::vector<Ev>, std::greater<Ev>> heap;
  std::uint64_t seq = 0;
  std::deque<Plan> fifo;
  bool busy = false;
  Plan running;
  TimeNs run_start = 0, run_end = 0;
  const TimeNs max_wait_ns = to_ns(policy.max_wait);
  const std::int64_t live_streams = static_cast<std::int64_t>(tenants.size());

  for (const RoundTenant& t : tenants) {
    Request r;
    r.id = next_id++;
    r.tenant = t.tenant;
    r.shape = t.layers[0];
    r.enqueue = start;
    r.deadline = start + t.slo_ns;
    r.layer = 0;
    heap.push(Ev{start, 0, t.tenant, seq++, r});
  }

  while (!heap.empty()) {
    const TimeNs now = heap.top().time;
    while (!heap.empty() && heap.top().time == now) {
      const Ev ev = heap.top();
      heap.pop();
      if (ev.kind == 0) {
        queue.push(ev.req);
      } else if (ev.kind == 1) {
        busy = false;
        for (const Request& r : running.members) {
          const RoundTenant& t = *by_id.at(r.tenant);
          if (r.layer + 1 < static_cast<int>(t.layers.size())) {
            Request nx = r;
            nx.id = next_id++;
            nx.shape = t.layers[r.layer + 1];
            nx.enqueue = run_end;
            ++nx.layer;
            heap.push(Ev{run_end, 0, r.tenant, seq++, nx});
          } else {
            out.pass_complete.emplace_back(r.tenant, run_end);
          }
        }
      }
    }
    if (busy) continue;
    if (fifo.empty()) {
      Policy pol = policy;
      pol.target_batch = pol.target_batch == 0 ? live_streams : std::min(pol.target_batch, live_streams);
      for (Plan& p : form_plans(queue, now, pol, dev)) fifo.push_back(std::move(p));
    }
    if (!fifo.empty()) {
      Plan p = std::move(fifo.front());
      fifo.pop_front();
      const TimeNs end = now + to_ns(charge(p, cache, dev));
      out.dispatches.push_back(RoundDispatch{p, now, end});
      busy = true;
      running = std::move(p);
      run_start = now;
      run_end = end;
      heap.push(Ev{end, 1, 0, seq++, {}});
    } else if (!queue.empty()) {
      Policy pol = policy;
      if (pol.target_batch == 0) pol.target_batch = live_streams;
      TimeNs wake = std::numeric_limits<TimeNs>::max();
      for (const auto& [shape, grp] : queue.groups()) {
        wake = std::min(wake, grp.front().enqueue + max_wait_ns);
        const std::int64_t probe =
            std::min<std::int64_t>(static_cast<std::int64_t>(grp.size()), std::max<std::int64_t>(pol.target_batch, 1));
        const double predicted = roofline_totals(probe * flops_of(shape), probe * bytes_of(shape),
                                                 probe * tiles_of(shape, dev), dev, dev.slots(), 1, kblocks_of(shape))
                                     .duration;
        const TimeNs predicted_ns = to_ns(predicted * (1.0 + pol.slo_safety_margin));
        for (const Request& r : grp) wake = std::min(wake, r.deadline - predicted_ns);
      }
      heap.push(Ev{std::max(wake, now + 1), 2, 0, seq++, {}});
    }
  }
  (void)run_start;
  return out;
}

}  // namespace gmb
