// extern "C" boundary for the host-side planner, cost model, monitor, metrics
// and the virtual-clock driver.  Device-side entry points live in runtime.cu.
#include <algorithm>
#include <chrono>
#include <cstring>

#include "abi.hpp"

namespace gmb {

namespace {
thread_local std::string g_last_error;
}

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const char* what) {
  g_last_error = what ? what : "";
  return code;
}

int fail_current(const gm_ctx* ctx) {
  int code = GM_EINTERNAL;
  try {
    throw;
  } catch (const std::invalid_argument& e) {
    code = fail(GM_EINVAL, e.what());
  } catch (const RangeError& e) {
    code = fail(GM_ERANGE, e.what());
  } catch (const CudaError& e) {
    code = fail(GM_ECUDA, e.what());
  } catch (const NoDevice& e) {
    code = fail(GM_ENODEV, e.what());
  } catch (const std::bad_alloc& e) {
    code = fail(GM_EOOM, e.what());
  } catch (const std::exception& e) {
    code = fail(GM_EINTERNAL, e.what());
  } catch (...) {
    code = fail(GM_EINTERNAL, "unknown error");
  }
  if (ctx) ctx->last_error = g_last_error;
  return code;
}

Device to_device(const gm_device_spec& d) {
  Device o;
  o.peak_flops = d.peak_flops;
  o.mem_bandwidth = d.mem_bandwidth;
  o.sm_count = d.sm_count;
  o.blocks_per_sm = d.blocks_per_sm;
  o.launch_overhead = d.launch_overhead;
  o.context_switch_overhead = d.context_switch_overhead;
  o.planning_overhead = d.planning_overhead;
  o.mem_capacity = d.mem_capacity;
  o.process_context_bytes = d.process_context_bytes;
  o.tile_m = d.tile_m;
  o.tile_n = d.tile_n;
  o.space_sched_penalty = d.space_sched_penalty;
  o.launch_serialization = d.launch_serialization;
  o.tile_latency = d.tile_latency;
  o.kblock_latency = d.kblock_latency;
  return o;
}

gm_device_spec from_device(const Device& d) {
  gm_device_spec o;
  o.peak_flops = d.peak_flops;
  o.mem_bandwidth = d.mem_bandwidth;
  o.sm_count = d.sm_count;
  o.blocks_per_sm = d.blocks_per_sm;
  o.launch_overhead = d.launch_overhead;
  o.context_switch_overhead = d.context_switch_overhead;
  o.planning_overhead = d.planning_overhead;
  o.mem_capacity = d.mem_capacity;
  o.process_context_bytes = d.process_context_bytes;
  o.tile_m = d.tile_m;
  o.tile_n = d.tile_n;
  o.space_sched_penalty = d.space_sched_penalty;
  o.launch_serialization = d.launch_serialization;
  o.tile_latency = d.tile_latency;
  o.kblock_latency = d.kblock_latency;
  return o;
}

Policy to_policy(const gm_batch_policy& p) {
  Policy o;
  o.max_wait = p.max_wait;
  o.target_batch = p.target_batch;
  o.allow_variable_size = p.allow_variable_size != 0;
  o.max_waves = p.max_waves < 1 ? 1 : p.max_waves;
  o.slo_safety_margin = p.slo_safety_margin;
  o.variable_inefficiency = p.variable_inefficiency;
  return o;
}

Detector to_detector(const gm_detector& d) {
  Detector o;
  o.ewma_alpha = d.ewma_alpha;
  o.min_observations = d.min_observations;
  o.threshold_ratio = d.threshold_ratio;
  o.evict_stragglers = d.evict_stragglers != 0;
  return o;
}

gm_kernel_cost from_cost(const Cost& c) { return gm_kernel_cost{c.flops, c.bytes, c.blocks, c.duration, c.waves}; }

Request to_request(const gm_kernel_request& r) {
  Request o;
  o.id = r.request_id;
  o.tenant = r.tenant_index;
  o.shape = to_shape(r.shape);
  o.enqueue = r.enqueue_time;
  o.deadline = r.slo_deadline;
  o.layer = r.layer_index;
  o.pass = r.pass_index;
  o.batch = r.batch == 0 ? 1 : r.batch;
  return o;
}

gm_kernel_request from_request(const Request& r) {
  gm_kernel_request o;
  std::memset(&o, 0, sizeof(o));
  o.request_id = r.id;
  o.tenant_index = r.tenant;
  o.layer_index = r.layer;
  o.shape = from_shape(r.shape);
  o.enqueue_time = r.enqueue;
  o.slo_deadline = r.deadline;
  o.pass_index = r.pass;
  o.batch = r.batch;
  return o;
}

Health to_health(const gm_tenant_health& h) {
  Health o;
  o.tenant = h.tenant_index;
  o.ewma = h.ewma_latency;
  o.alpha = h.ewma_alpha;
  o.count = h.observed_count;
  o.evicted = h.evicted != 0;
  return o;
}

gm_tenant_health from_health(const Health& h) {
  gm_tenant_health o;
  std::memset(&o, 0, sizeof(o));
  o.tenant_index = h.tenant;
  o.evicted = h.evicted ? 1 : 0;
  o.ewma_latency = h.ewma;
  o.ewma_alpha = h.alpha;
  o.observed_count = h.count;
  return o;
}

namespace {

template <class T>
void copy_out(const std::vector<T>& src, T* out, size_t cap, size_t* n) {
  if (n) *n = src.size();
  if (src.size() > cap || (!out && !src.empty())) throw RangeError("output buffer too small");
  std::copy(src.begin(), src.end(), out);
}

void need(const void* p, const char* what) {
  if (!p) throw std::invalid_argument(std::string("null argument: ") + what);
}

}  // namespace
}  // namespace gmb

using namespace gmb;

extern "C" {

const char* gm_last_error(const gm_ctx* ctx) { return ctx ? ctx->last_error.c_str() : g_last_error.c_str(); }
int gm_abi_version(void) { return GM_ABI_VERSION; }

void gm_device_spec_default(gm_device_spec* out) {
  if (out) *out = from_device(Device{});
}
void gm_device_spec_v100(gm_device_spec* out) {
  if (out) *out = from_device(v100_device());
}
void gm_device_spec_b200(gm_device_spec* out) {
  if (out) *out = from_device(b200_device());
}
int gm_device_spec_validate(const gm_device_spec* d) {
  GM_API_BEGIN
  need(d, "device");
  to_device(*d).check();
  GM_API_END
}
void gm_batch_policy_default(gm_batch_policy* out) {
  if (!out) return;
  std::memset(out, 0, sizeof(*out));
  const Policy p;
  out->max_wait = p.max_wait;
  out->target_batch = p.target_batch;
  out->allow_variable_size = p.allow_variable_size;
  out->max_waves = static_cast<int32_t>(p.max_waves);
  out->slo_safety_margin = p.slo_safety_margin;
  out->variable_inefficiency = p.variable_inefficiency;
}
void gm_detector_default(gm_detector* out) {
  if (!out) return;
  std::memset(out, 0, sizeof(*out));
  const Detector d;
  out->ewma_alpha = d.ewma_alpha;
  out->min_observations = d.min_observations;
  out->threshold_ratio = d.threshold_ratio;
  out->evict_stragglers = d.evict_stragglers;
}

// ---- shapes / cost model ---------------------------------------------------

int64_t gm_gemm_flops(const gm_gemm_shape* s) { return s ? flops_of(to_shape(*s)) : 0; }
int64_t gm_gemm_bytes(const gm_gemm_shape* s, int64_t elem) { return s ? bytes_of(to_shape(*s), elem) : 0; }

int gm_im2col_gemm_dims(const gm_conv_spec* c, gm_gemm_shape* out) {
  GM_API_BEGIN
  need(c, "conv");
  need(out, "out");
  *out = from_shape(lower_conv(to_conv(*c)));
  GM_API_END
}

void gm_batch_inputs(const gm_gemm_shape* s, int64_t batch, gm_gemm_shape* out) {
  if (s && out) *out = from_shape(with_batch(to_shape(*s), batch));
}

int gm_shape_key(const gm_gemm_shape* s, char* buf, size_t cap) {
  GM_API_BEGIN
  need(s, "shape");
  const std::string k = key_of(to_shape(*s));
  if (!buf || cap < k.size() + 1) throw RangeError("output buffer too small");
  std::memcpy(buf, k.c_str(), k.size() + 1);
  GM_API_END
}

int64_t gm_to_ns(double seconds) { return to_ns(seconds); }
double gm_to_seconds(int64_t ns) { return to_seconds(ns); }

int64_t gm_thread_blocks(const gm_gemm_shape* s, const gm_device_spec* d) {
  return (s && d) ? tiles_of(to_shape(*s), to_device(*d)) : 0;
}

int gm_dispatch_duration(const gm_kernel_group* groups, size_t n, const gm_device_spec* d,
                         int64_t slot_budget, int64_t launches, gm_kernel_cost* out) {
  GM_API_BEGIN
  need(d, "device");
  need(out, "out");
  std::vector<Group> gs;
  gs.reserve(n);
  for (size_t i = 0; i < n; ++i) gs.push_back(Group{to_shape(groups[i].shape), groups[i].count});
  *out = from_cost(roofline(gs, to_device(*d), slot_budget, launches));
  GM_API_END
}

// ---- queue / batcher -------------------------------------------------------

int gm_queue_create(gm_queue** out) {
  GM_API_BEGIN
  need(out, "out");
  *out = new gm_queue();
  GM_API_END
}
void gm_queue_destroy(gm_queue* q) { delete q; }

int gm_queue_enqueue(gm_queue* q, const gm_kernel_request* r) {
  GM_API_BEGIN
  need(q, "queue");
  need(r, "request");
  q->q.push(to_request(*r));
  GM_API_END
}

int64_t gm_queue_size(const gm_queue* q) { return q ? q->q.size() : 0; }

int gm_queue_snapshot(const gm_queue* q, gm_kernel_request* out, size_t cap, size_t* n) {
  GM_API_BEGIN
  need(q, "queue");
  std::vector<gm_kernel_request> all;
  for (const auto& [shape, fifo] : q->q.groups())
    for (const Request& r : fifo) all.push_back(from_request(r));
  copy_out(all, out, cap, n);
  GM_API_END
}

int gm_queue_group_count(const gm_queue* q, size_t* n) {
  GM_API_BEGIN
  need(q, "queue");
  need(n, "n");
  *n = q->q.groups().size();
  GM_API_END
}

int gm_queue_cancel_tenant(gm_queue* q, int32_t tenant, gm_kernel_request* out, size_t cap, size_t* n) {
  GM_API_BEGIN
  need(q, "queue");
  std::vector<Request> gone = q->q.drop_tenant(tenant);
  std::vector<gm_kernel_request> conv;
  for (const Request& r : gone) conv.push_back(from_request(r));
  // Cancellation already happened; report what fits.
  if (n) *n = conv.size();
  if (out) std::copy_n(conv.begin(), std::min(cap, conv.size()), out);
  if (conv.size() > cap && out) throw RangeError("output buffer too small");
  GM_API_END
}

int gm_form_batches(gm_queue* q, int64_t now, const gm_batch_policy* p, const gm_device_spec* d,
                    gm_plans** out) {
  GM_API_BEGIN
  need(q, "queue");
  need(p, "policy");
  need(d, "device");
  need(out, "out");
  auto* plans = new gm_plans();
  try {
    plans->plans = form_plans(q->q, now, to_policy(*p), to_device(*d));
  } catch (...) {
    delete plans;
    throw;
  }
  *out = plans;
  GM_API_END
}

size_t gm_plans_count(const gm_plans* p) { return p ? p->plans.size() : 0; }

int gm_plans_get(const gm_plans* p, size_t i, gm_plan_info* out) {
  GM_API_BEGIN
  need(p, "plans");
  need(out, "out");
  if (i >= p->plans.size()) throw std::invalid_argument("plan index out of range");
  const Plan& pl = p->plans[i];
  out->uniform = pl.uniform ? 1 : 0;
  out->reserved0 = 0;
  out->n_members = static_cast<int64_t>(pl.members.size());
  out->planned_cost = from_cost(pl.cost);
  out->signature = pl.signature.c_str();
  GM_API_END
}

int gm_plans_members(const gm_plans* p, size_t i, gm_kernel_request* out, size_t cap, size_t* n) {
  GM_API_BEGIN
  need(p, "plans");
  if (i >= p->plans.size()) throw std::invalid_argument("plan index out of range");
  std::vector<gm_kernel_request> v;
  for (const Request& r : p->plans[i].members) v.push_back(from_request(r));
  copy_out(v, out, cap, n);
  GM_API_END
}

void gm_plans_destroy(gm_plans* p) { delete p; }

int gm_plans_key(const gm_plans* p, uint64_t* key) {
  GM_API_BEGIN
  need(p, "plans");
  need(key, "key");
  // FNV-1a over every plan's signature and member (tenant, layer) identities:
  // equal keys <=> the same launch program (the CUDA-graph cache key).
  uint64_t h = 1469598103934665603ull;
  auto mix = [&h](const void* data, size_t n) {
    const unsigned char* b = static_cast<const unsigned char*>(data);
    for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
  };
  for (const Plan& plan : p->plans) {
    mix(plan.signature.data(), plan.signature.size());
    for (const Request& r : plan.members) {
      mix(&r.tenant, sizeof(r.tenant));
      mix(&r.layer, sizeof(r.layer));
    }
    const char sep = '|';
    mix(&sep, 1);
  }
  *key = h;
  GM_API_END
}

int gm_build_tile_table(const gm_plans* p, size_t i, const gm_device_spec* d, gm_tile* out, size_t cap,
                        size_t* n) {
  GM_API_BEGIN
  need(p, "plans");
  need(d, "device");
  if (i >= p->plans.size()) throw std::invalid_argument("plan index out of range");
  std::vector<Tile> t = tile_table(p->plans[i], to_device(*d));
  std::vector<gm_tile> v;
  v.reserve(t.size());
  for (const Tile& x : t) v.push_back(gm_tile{x.member, x.flags, x.m_tile, x.n_tile});
  copy_out(v, out, cap, n);
  GM_API_END
}

int gm_plan_super_kernel(const gm_kernel_request* members, size_t n, int uniform, const gm_batch_policy* p,
                         const gm_device_spec* d, gm_kernel_cost* out) {
  GM_API_BEGIN
  need(p, "policy");
  need(d, "device");
  need(out, "out");
  std::vector<Request> v;
  for (size_t i = 0; i < n; ++i) v.push_back(to_request(members[i]));
  *out = from_cost(plan_cost(v, uniform != 0, to_policy(*p), to_device(*d)));
  GM_API_END
}

double gm_slo_headroom(const gm_kernel_request* r, int64_t now, double predicted, const gm_batch_policy* p) {
  if (!r || !p) return 0.0;
  return headroom(to_request(*r), now, predicted, to_policy(*p));
}

int gm_cache_create(gm_cache** out) {
  GM_API_BEGIN
  need(out, "out");
  *out = new gm_cache();
  GM_API_END
}
void gm_cache_destroy(gm_cache* c) { delete c; }

int gm_dispatch_cost(const gm_plans* p, size_t i, gm_cache* c, const gm_device_spec* d, double* duration,
                     int* cache_hit) {
  GM_API_BEGIN
  need(p, "plans");
  need(c, "cache");
  need(d, "device");
  if (i >= p->plans.size()) throw std::invalid_argument("plan index out of range");
  const std::int64_t misses = c->c.misses;
  const double dur = charge(p->plans[i], c->c, to_device(*d));
  if (duration) *duration = dur;
  if (cache_hit) *cache_hit = c->c.misses == misses ? 1 : 0;
  GM_API_END
}

int gm_cache_stats(const gm_cache* c, int64_t* hits, int64_t* misses, int64_t* entries) {
  GM_API_BEGIN
  need(c, "cache");
  if (hits) *hits = c->c.hits;
  if (misses) *misses = c->c.misses;
  if (entries) *entries = static_cast<int64_t>(c->c.entries.size());
  GM_API_END
}

// ---- monitor ---------------------------------------------------------------

int gm_record_latency(gm_tenant_health* h, double observed_seconds) {
  GM_API_BEGIN
  need(h, "health");
  Health x = to_health(*h);
  observe(x, observed_seconds);
  *h = from_health(x);
  GM_API_END
}

int gm_detect_stragglers(const gm_tenant_health* h, size_t n, double threshold_ratio, int64_t min_observations,
                         int32_t* out, size_t cap, size_t* n_out) {
  GM_API_BEGIN
  std::vector<Health> hs;
  for (size_t i = 0; i < n; ++i) hs.push_back(to_health(h[i]));
  std::vector<int> flagged = stragglers(hs, threshold_ratio, min_observations);
  std::vector<int32_t> v(flagged.begin(), flagged.end());
  copy_out(v, out, cap, n_out);
  GM_API_END
}

int gm_evict(gm_tenant_health* h, size_t n, gm_queue* q, int32_t tenant, gm_kernel_request* out, size_t cap,
             size_t* n_out) {
  GM_API_BEGIN
  need(q, "queue");
  std::vector<Health> hs;
  for (size_t i = 0; i < n; ++i) hs.push_back(to_health(h[i]));
  std::vector<Request> gone = evict_tenant(hs, q->q, tenant);
  for (size_t i = 0; i < n; ++i) h[i] = from_health(hs[i]);
  if (n_out) *n_out = gone.size();
  if (out)
    for (size_t i = 0; i < std::min(cap, gone.size()); ++i) out[i] = from_request(gone[i]);
  if (out && gone.size() > cap) throw RangeError("output buffer too small");
  GM_API_END
}

// ---- metrics ---------------------------------------------------------------

int gm_percentile_nearest_rank(const double* v, size_t n, double pct, double* out) {
  GM_API_BEGIN
  need(out, "out");
  *out = nearest_rank(std::vector<double>(v, v + n), pct);
  GM_API_END
}

int gm_geomean(const double* v, size_t n, double* out) {
  GM_API_BEGIN
  need(out, "out");
  *out = geometric_mean(std::span<const double>(v, n));
  GM_API_END
}

// ---- virtual-clock driver --------------------------------------------------

int gm_plan_round_shapes(const gm_round_tenant* tenants, size_t n, int64_t start, const gm_batch_policy* p,
                         const gm_device_spec* d, gm_cache* cache, uint64_t* next_id, gm_plans** out) {
  GM_API_BEGIN
  need(out, "out");
  need(p, "policy");
  need(d, "device");
  if (n && !tenants) throw std::invalid_argument("null argument: tenants");
  std::vector<RoundTenant> round;
  round.reserve(n);
  for (size_t j = 0; j < n; ++j) {
    RoundTenant rt;
    rt.tenant = tenants[j].tenant;
    if (tenants[j].n_layers && !tenants[j].layers) throw std::invalid_argument("null argument: layers");
    for (size_t l = 0; l < tenants[j].n_layers; ++l) rt.layers.push_back(to_shape(tenants[j].layers[l]));
    rt.slo_ns = tenants[j].slo_ns;
    round.push_back(std::move(rt));
  }
  const Device dev = to_device(*d);
  dev.check();
  SignatureCache local;
  std::uint64_t id = next_id ? *next_id : 1;
  RoundResult res = plan_round(round, start, to_policy(*p), dev, cache ? cache->c : local, id);
  if (next_id) *next_id = id;
  auto* plans = new gm_plans();
  for (RoundDispatch& r : res.dispatches) {
    plans->plans.push_back(std::move(r.plan));
    plans->times.emplace_back(r.start, r.end);
  }
  *out = plans;
  GM_API_END
}

int gm_simulate_space_time(const gm_sim_config* cfg, gm_sim_trace** out) {
  GM_API_BEGIN
  need(cfg, "config");
  need(out, "out");
  SpaceTimeConfig c;
  c.device = to_device(cfg->device);
  c.scheduler = to_policy(cfg->scheduler);
  c.detector = to_detector(cfg->detector);
  for (size_t i = 0; i < cfg->n_layers; ++i) c.layers.push_back(to_shape(cfg->layers[i]));
  c.tenants = cfg->n_tenants;
  c.concurrency = cfg->concurrency;
  c.slo_latency = cfg->slo_latency;
  c.duration = cfg->duration;
  c.warmup = cfg->warmup;
  c.microbench = cfg->microbench != 0;
  if (cfg->degrade_tenant >= 0)
    c.degradation = Degradation{cfg->degrade_tenant, cfg->degrade_slowdown, cfg->degrade_start};
  auto* t = new gm_sim_trace();
  try {
    t->t = simulate_space_time(c);
  } catch (...) {
    delete t;
    throw;
  }
  *out = t;
  GM_API_END
}

int gm_sim_trace_counts(const gm_sim_trace* t, size_t* n_events, size_t* n_members, size_t* n_completions,
                        size_t* n_cancelled, int64_t* cache_hits, int64_t* cache_misses) {
  GM_API_BEGIN
  need(t, "trace");
  size_t members = 0;
  for (const Dispatch& d : t->t.events) members += d.members.size();
  if (n_events) *n_events = t->t.events.size();
  if (n_members) *n_members = members;
  if (n_completions) *n_completions = t->t.completions.size();
  if (n_cancelled) *n_cancelled = t->t.cancellations.size();
  if (cache_hits) *cache_hits = t->t.cache_hits;
  if (cache_misses) *cache_misses = t->t.cache_misses;
  GM_API_END
}

int gm_sim_trace_events(const gm_sim_trace* t, gm_sim_event* ev, size_t cap_ev, uint64_t* member_ids,
                        size_t cap_ids) {
  GM_API_BEGIN
  need(t, "trace");
  size_t total = 0;
  for (const Dispatch& d : t->t.events) total += d.members.size();
  if (t->t.events.size() > cap_ev || total > cap_ids) throw RangeError("output buffer too small");
  int64_t off = 0;
  for (size_t i = 0; i < t->t.events.size(); ++i) {
    const Dispatch& d = t->t.events[i];
    ev[i] = gm_sim_event{d.start, d.end, d.flops, d.occupancy, off, static_cast<int64_t>(d.members.size())};
    for (uint64_t id : d.members) member_ids[off++] = id;
  }
  GM_API_END
}

int gm_sim_trace_completions(const gm_sim_trace* t, gm_sim_completion* out, size_t cap) {
  GM_API_BEGIN
  need(t, "trace");
  if (t->t.completions.size() > cap) throw RangeError("output buffer too small");
  for (size_t i = 0; i < t->t.completions.size(); ++i) {
    const Completion& c = t->t.completions[i];
    out[i] = gm_sim_completion{c.id, c.tenant, c.slo_met ? 1 : 0, c.enqueue, c.dispatch, c.complete, c.flops};
  }
  GM_API_END
}

int gm_sim_trace_evictions(const gm_sim_trace* t, int32_t* tenants, int64_t* times, size_t cap, size_t* n) {
  GM_API_BEGIN
  need(t, "trace");
  if (n) *n = t->t.evicted.size();
  if (t->t.evicted.size() > cap) throw RangeError("output buffer too small");
  for (size_t i = 0; i < t->t.evicted.size(); ++i) {
    if (tenants) tenants[i] = t->t.evicted[i];
    if (times) times[i] = t->t.eviction_times[i];
  }
  GM_API_END
}

int gm_sim_trace_flops(const gm_sim_trace* t, int64_t* dispatched, int64_t* completed) {
  GM_API_BEGIN
  need(t, "trace");
  if (dispatched) *dispatched = t->t.dispatched_flops;
  if (completed) *completed = t->t.completed_flops;
  GM_API_END
}

void gm_sim_trace_destroy(gm_sim_trace* t) { delete t; }


// ---- host-driven loop over one ctx (header: gm_enqueue .. gm_ctx_health) ----

namespace {
gmb::Health& health_of(gm_ctx* ctx, int32_t tenant, const char* who) {
  if (tenant < 0 || tenant >= static_cast<int32_t>(ctx->health.size()))
    throw std::invalid_argument(std::string(who) + ": unknown tenant " + std::to_string(tenant));
  return ctx->health[static_cast<size_t>(tenant)];
}
}  // namespace

int gm_ctx_form_batches(gm_ctx* ctx, int64_t now, gm_plans** out) {
  GM_API_BEGIN
  if (!ctx || !out) throw std::invalid_argument("null argument");
  auto* p = new gm_plans();
  try {
    p->plans = form_plans(ctx->queue.q, now, ctx->pol, ctx->dev);
  } catch (...) {
    delete p;
    throw;
  }
  *out = p;
  GM_CTX_API_END(ctx)
}

int64_t gm_ctx_now_ns(const gm_ctx* ctx) {
  const int64_t t = std::chrono::duration_cast<std::chrono::nanoseconds>(
                        std::chrono::steady_clock::now().time_since_epoch()).count();
  return ctx ? t - ctx->clock0_ns : t;
}

int gm_ctx_record_latency(gm_ctx* ctx, int32_t tenant, double observed_seconds) {
  GM_API_BEGIN
  if (!ctx) throw std::invalid_argument("null context");
  observe(health_of(ctx, tenant, "record_latency"), observed_seconds);  // scheduler.cpp:214-223
  GM_CTX_API_END(ctx)
}

int gm_ctx_detect_stragglers(gm_ctx* ctx, int32_t* out, size_t cap, size_t* n) {
  GM_API_BEGIN
  if (!ctx || !n) throw std::invalid_argument("null argument");
  const std::vector<int> s = stragglers(ctx->health, ctx->det.threshold_ratio, ctx->det.min_observations);  // :246-271
  if (s.size() > cap) throw RangeError("detect_stragglers: " + std::to_string(s.size()) + " stragglers, cap " +
                                       std::to_string(cap));
  for (size_t i = 0; i < s.size(); ++i) out[i] = s[i];
  *n = s.size();
  GM_CTX_API_END(ctx)
}

int gm_ctx_evict(gm_ctx* ctx, int32_t tenant, uint64_t* cancelled_ids, size_t cap, size_t* n) {
  GM_API_BEGIN
  if (!ctx) throw std::invalid_argument("null context");
  const std::vector<Request> gone = evict_tenant(ctx->health, ctx->queue.q, tenant);  // scheduler.cpp:225-244
  for (size_t i = 0; i < gone.size(); ++i) {
    ctx->io.erase(gone[i].id);
    if (cancelled_ids && i < cap) cancelled_ids[i] = gone[i].id;
  }
  if (n) *n = gone.size();  // the eviction stands even when cap < *n (ids past cap are not written)
  GM_CTX_API_END(ctx)
}

int gm_ctx_health(const gm_ctx* ctx, int32_t tenant, gm_tenant_health* out) {
  GM_API_BEGIN
  if (!ctx || !out) throw std::invalid_argument("null argument");
  *out = from_health(health_of(const_cast<gm_ctx*>(ctx), tenant, "health"));
  GM_CTX_API_END(ctx)
}

}  // extern "C"
