// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// A JSON-in/JSON-out C entry point over the UNMODIFIED reference library
// (gpumux_core, compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libgpumux_ref.so).  The parity tests drive the same scripted
// inputs through this shim and through the product C-ABI and compare results
// bit for bit.  Doubles are emitted by nlohmann::json with round-trip
// precision, so Python's float() recovers the exact bits.
//
// Ops (request {"op": ..., ...}):
//   dispatch_duration  cost_model.cpp:18-46
//   thread_blocks      cost_model.cpp:14-16
//   im2col             gemm.hpp:44-51
//   session            a scripted sequence over one RequestQueue /
//                      SuperKernelCache / TenantHealth vector:
//                      enqueue, form, cost, cancel, evict, record, detect
//                      (scheduler.cpp:8-271)
//   run_space_time     run() with PolicyKind::kSpaceTime (sim.cpp:398-581)
//   percentile, geomean  metrics.cpp:10-28
#include <cstring>
#include <string>
#include <vector>

#include <json.hpp>

#include "gpumux/cost_model.hpp"
#include "gpumux/metrics.hpp"
#include "gpumux/scheduler.hpp"
#include "gpumux/sim.hpp"

using nlohmann::json;
using namespace gpumux;

namespace {

DeviceSpec device_of(const json& j) {
  DeviceSpec d;
  if (j.is_null()) return d;
  auto num = [&](const char* k, double& f) { if (j.contains(k)) f = j.at(k).get<double>(); };
  auto integer = [&](const char* k, std::int64_t& f) { if (j.contains(k)) f = j.at(k).get<std::int64_t>(); };
  num("peak_flops", d.peak_flops);
  num("mem_bandwidth", d.mem_bandwidth);
  integer("sm_count", d.sm_count);
  integer("blocks_per_sm", d.blocks_per_sm);
  num("launch_overhead", d.launch_overhead);
  num("context_switch_overhead", d.context_switch_overhead);
  num("planning_overhead", d.planning_overhead);
  num("mem_capacity", d.mem_capacity);
  num("process_context_bytes", d.process_context_bytes);
  integer("tile_m", d.tile_m);
  integer("tile_n", d.tile_n);
  num("space_sched_penalty", d.space_sched_penalty);
  num("launch_serialization", d.launch_serialization);
  return d;
}

BatchPolicy policy_of(const json& j) {
  BatchPolicy p;
  if (j.is_null()) return p;
  if (j.contains("max_wait")) p.max_wait = j.at("max_wait").get<double>();
  if (j.contains("target_batch")) p.target_batch = j.at("target_batch").get<std::int64_t>();
  if (j.contains("allow_variable_size")) p.allow_variable_size = j.at("allow_variable_size").get<bool>();
  if (j.contains("slo_safety_margin")) p.slo_safety_margin = j.at("slo_safety_margin").get<double>();
  if (j.contains("variable_inefficiency"))
    p.variable_inefficiency = j.at("variable_inefficiency").get<double>();
  return p;
}

GemmShape shape_of(const json& j) {
  return GemmShape{j.at(0).get<std::int64_t>(), j.at(1).get<std::int64_t>(), j.at(2).get<std::int64_t>()};
}

KernelRequest request_of(const json& j) {
  KernelRequest r;
  r.request_id = j.at("id").get<std::uint64_t>();
  r.tenant_index = j.value("tenant", 0);
  r.shape = shape_of(j.at("shape"));
  r.enqueue_time = j.value("enqueue", std::int64_t{0});
  r.slo_deadline = j.value("deadline", std::int64_t{0});
  r.layer_index = j.value("layer", 0);
  r.pass_index = j.value("pass", 0u);
  return r;
}

json cost_json(const KernelCost& c) {
  return json{{"flops", c.flops}, {"bytes", c.bytes}, {"blocks", c.blocks}, {"duration", c.duration},
              {"waves", c.waves}};
}

json request_json(const KernelRequest& r) {
  return json{{"id", r.request_id}, {"tenant", r.tenant_index}, {"shape", {r.shape.m, r.shape.n, r.shape.k}},
              {"enqueue", r.enqueue_time}, {"deadline", r.slo_deadline}, {"layer", r.layer_index},
              {"pass", r.pass_index}};
}

json plan_json(const SuperKernel& sk) {
  json ids = json::array();
  for (const KernelRequest& r : sk.members) ids.push_back(r.request_id);
  return json{{"signature", sk.shape_signature}, {"uniform", sk.uniform}, {"cost", cost_json(sk.planned_cost)},
              {"members", ids}};
}

json queue_json(const RequestQueue& q) {
  json ids = json::array();
  for (const auto& [shape, dq] : q.groups())
    for (const KernelRequest& r : dq) ids.push_back(r.request_id);
  return ids;
}

json session(const json& in) {
  RequestQueue q;
  SuperKernelCache cache;
  std::vector<TenantHealth> healths;
  for (int i = 0; i < in.value("tenants", 0); ++i) {
    TenantHealth h;
    h.tenant_index = i;
    h.ewma_alpha = in.value("ewma_alpha", 0.2);
    healths.push_back(h);
  }
  const DeviceSpec dev = device_of(in.value("device", json()));
  std::vector<SuperKernel> last;
  json out = json::array();
  for (const json& step : in.at("steps")) {
    const std::string kind = step.at("do").get<std::string>();
    json res;
    try {
      if (kind == "enqueue") {
        q.enqueue(request_of(step.at("request")));
        res = json{{"size", q.size()}};
      } else if (kind == "form") {
        last = form_batches(q, step.at("now").get<std::int64_t>(), policy_of(step.value("policy", json())), dev);
        json plans = json::array();
        for (const SuperKernel& sk : last) plans.push_back(plan_json(sk));
        res = json{{"plans", plans}, {"remaining", queue_json(q)}};
      } else if (kind == "cost") {
        const double d = dispatch_cost(last.at(step.at("plan").get<std::size_t>()), cache, dev);
        res = json{{"duration", d}, {"hits", cache.hits}, {"misses", cache.misses}};
      } else if (kind == "cancel") {
        json ids = json::array();
        for (const KernelRequest& r : q.cancel_tenant(step.at("tenant").get<int>())) ids.push_back(r.request_id);
        res = json{{"cancelled", ids}, {"remaining", queue_json(q)}};
      } else if (kind == "evict") {
        json ids = json::array();
        for (const KernelRequest& r : evict(healths, q, step.at("tenant").get<int>())) ids.push_back(r.request_id);
        res = json{{"cancelled", ids}, {"remaining", queue_json(q)}};
      } else if (kind == "record") {
        TenantHealth& h = healths.at(step.at("tenant").get<std::size_t>());
        record_latency(h, step.at("seconds").get<double>());
        res = json{{"ewma", h.ewma_latency}, {"count", h.observed_count}};
      } else if (kind == "detect") {
        res = json{{"flagged", detect_stragglers(healths, step.at("ratio").get<double>(),
                                                 step.at("min_obs").get<std::int64_t>())}};
      } else if (kind == "headroom") {
        res = json{{"headroom", slo_headroom(request_of(step.at("request")), step.at("now").get<std::int64_t>(),
                                             step.at("predicted").get<double>(),
                                             policy_of(step.value("policy", json())))}};
      } else {
        res = json{{"error", "unknown step " + kind}};
      }
    } catch (const std::exception& e) {
      res = json{{"error", e.what()}};
    }
    out.push_back(res);
  }
  return json{{"steps", out}};
}

json run_space_time(const json& in) {
  SimConfig cfg;
  cfg.device = device_of(in.value("device", json()));
  cfg.policy = PolicyKind::kSpaceTime;
  cfg.scheduler = policy_of(in.value("scheduler", json()));
  if (in.contains("detector")) {
    const json& d = in.at("detector");
    cfg.detector.ewma_alpha = d.value("ewma_alpha", cfg.detector.ewma_alpha);
    cfg.detector.min_observations = d.value("min_observations", cfg.detector.min_observations);
    cfg.detector.threshold_ratio = d.value("threshold_ratio", cfg.detector.threshold_ratio);
    cfg.detector.evict_stragglers = d.value("evict_stragglers", cfg.detector.evict_stragglers);
  }
  Tenant t;
  for (const json& s : in.at("layers")) t.layers.push_back(shape_of(s));
  t.slo_latency = in.value("slo_latency", 0.1);
  t.concurrency = in.value("concurrency", 1);
  t.weights_bytes = 0;
  const int n = in.at("tenants").get<int>();
  for (int i = 0; i < n; ++i) {
    t.tenant_id = "t" + std::to_string(i);
    cfg.tenants.push_back(t);
  }
  cfg.duration = in.value("duration", 1.0);
  cfg.warmup = in.value("warmup", 0.1 * cfg.duration);
  cfg.mode = in.value("microbench", false) ? SimMode::kMicrobench : SimMode::kForwardPass;
  if (in.contains("degrade")) {
    const json& d = in.at("degrade");
    cfg.degradation = DegradationSpec{d.at("tenant").get<int>(), d.at("slowdown").get<double>(),
                                      d.at("start").get<double>()};
  }
  const Trace tr = run(cfg);
  json events = json::array();
  for (const DispatchEvent& e : tr.events)
    events.push_back(json{{"start", e.start}, {"end", e.end}, {"flops", e.flops}, {"occupancy", e.occupancy},
                          {"members", e.member_requests}});
  json comps = json::array();
  for (const RequestLifecycle& c : tr.completions)
    comps.push_back(json{{"id", c.request_id}, {"tenant", c.tenant_index}, {"enqueue", c.enqueue_time},
                         {"dispatch", c.dispatch_time}, {"complete", c.complete_time}, {"slo_met", c.slo_met},
                         {"flops", c.flops}});
  return json{{"events", events},
              {"completions", comps},
              {"cancellations", tr.cancellations},
              {"evicted", tr.evicted_tenants},
              {"eviction_times", tr.eviction_times},
              {"cache_hits", tr.cache_hits},
              {"cache_misses", tr.cache_misses},
              {"dispatched_flops", tr.dispatched_flops},
              {"completed_flops", tr.completed_kernel_flops}};
}

json dispatch(const json& in) {
  const std::string op = in.at("op").get<std::string>();
  if (op == "dispatch_duration") {
    std::vector<KernelGroup> groups;
    for (const json& g : in.at("groups")) groups.push_back(KernelGroup{shape_of(g.at("shape")), g.value("count", 1)});
    return cost_json(dispatch_duration(groups, device_of(in.value("device", json())),
                                       in.at("slot_budget").get<std::int64_t>(), in.value("launches", 1)));
  }
  if (op == "thread_blocks") return json{{"blocks", thread_blocks(shape_of(in.at("shape")), device_of(in.value("device", json())))}};
  if (op == "im2col") {
    const json& c = in.at("conv");
    ConvSpec s{c.at(0).get<std::int64_t>(), c.at(1).get<std::int64_t>(), c.at(2).get<std::int64_t>(),
               c.at(3).get<std::int64_t>(), c.at(4).get<std::int64_t>(), c.at(5).get<std::int64_t>(),
               c.at(6).get<std::int64_t>(), c.at(7).get<std::int64_t>()};
    const GemmShape g = im2col_gemm_dims(s);
    return json{{"shape", {g.m, g.n, g.k}}};
  }
  if (op == "session") return session(in);
  if (op == "run_space_time") return run_space_time(in);
  if (op == "percentile")
    return json{{"value", percentile_nearest_rank(in.at("values").get<std::vector<double>>(), in.at("pct").get<double>())}};
  if (op == "geomean") {
    const auto v = in.at("values").get<std::vector<double>>();
    return json{{"value", geomean(v)}};
  }
  return json{{"error", "unknown op " + op}};
}

thread_local std::string g_out;

}  // namespace

extern "C" const char* gm_ref_call(const char* request) {
  try {
    g_out = dispatch(json::parse(request)).dump();
  } catch (const std::exception& e) {
    g_out = json{{"error", e.what()}}.dump();
  }
  return g_out.c_str();
}
