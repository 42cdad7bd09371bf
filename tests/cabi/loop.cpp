// Compiled C++ client of the C-ABI (links libgpumux_b200.so, no Python): the
// reference run_space_time loop shape (proj/src/sim.cpp:452-576) driven from
// outside the library through one gm_ctx:
//
//   gm_enqueue (scheduler.cpp:8-16, with per-request I/O)
//     -> gm_ctx_form_batches (form_batches, scheduler.cpp:96-199)
//     -> gm_dispatch (one super-kernel per formed plan)
//     -> gm_poll_completions (per-member completion fan-out, sim.cpp:466-476)
//     -> gm_ctx_record_latency (execution time, sim.cpp:475-476)
//     -> gm_ctx_detect_stragglers / gm_ctx_evict (sim.cpp:496-507)
//     -> next layer enqueued at completion (sim.cpp:482-488), closed loop
//
// Four tenants, each a 2-layer GEMM chain (layer 1 reads layer 0's output);
// tenants 0/1 and 2/3 share shapes, so formed super-kernels pack pairs.
// Tenant 3's observed latencies are inflated from pass 2 on (the reference's
// inject_degradation, sim.cpp:98-110), so the detector flags and evicts it.
//
//   loop --host   host-only ctx: completions are synthesized from each plan's
//                 planned cost (no GPU); checks plans, monitor and eviction
//   loop          device ctx: real launches; every pass's output (copied to
//                 host by the request I/O) is checked against the CPU oracle
//                 (oracle/_build/liboracle.so, oracle_gemm_nt) at 1e-2
//
// Exit 0 and "loop ok ..." on success; any failed check prints and exits 1.
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <thread>
#include <string>
#include <vector>

#include "gpumux_b200.h"

#ifdef GM_LOOP_GPU
#include <cuda_runtime.h>
extern "C" void oracle_gemm_nt(const float* a, const float* b, float* c, int64_t M, int64_t N, int64_t K,
                               int64_t lda, int64_t ldb, int32_t relu);
#endif

namespace {

int g_fail = 0;
#define CHECK(cond, ...)                                        \
  do {                                                          \
    if (!(cond)) {                                              \
      std::fprintf(stderr, "CHECK failed %s:%d: %s: ", __FILE__, __LINE__, #cond); \
      std::fprintf(stderr, __VA_ARGS__);                        \
      std::fprintf(stderr, "\n");                               \
      ++g_fail;                                                 \
    }                                                           \
  } while (0)
#define OK(call)                                                                      \
  do {                                                                                \
    const int st_ = (call);                                                           \
    if (st_ != GM_OK) {                                                               \
      std::fprintf(stderr, "%s:%d: %s -> %d (%s)\n", __FILE__, __LINE__, #call, st_,  \
                   gm_last_error(nullptr));                                           \
      std::exit(1);                                                                   \
    }                                                                                 \
  } while (0)

constexpr int kTenants = 4, kLayers = 2, kPasses = 6, kDegraded = 3;
constexpr double kSlowdown = 10.0;

// Layer shapes (m, n, k): layer 1's k is layer 0's n (it reads layer 0's output).
gm_gemm_shape shape_of(int tenant, int layer) {
  if (tenant < 2) return layer == 0 ? gm_gemm_shape{128, 256, 512} : gm_gemm_shape{128, 128, 256};
  return layer == 0 ? gm_gemm_shape{256, 128, 192} : gm_gemm_shape{256, 64, 128};
}

uint16_t to_bf16(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7fffu + ((u >> 16) & 1u);
  return static_cast<uint16_t>(u >> 16);
}
[[maybe_unused]] float from_bf16(uint16_t h) {
  const uint32_t u = static_cast<uint32_t>(h) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

struct Buffers {  // one tenant
#ifdef GM_LOOP_GPU
  void* x0 = nullptr;
  void* w[kLayers] = {};
  void* y[kLayers] = {};
#endif
  std::vector<std::vector<uint16_t>> in, out;  // per pass, host
  std::vector<std::vector<uint16_t>> wh;       // per layer, host copy of the weights
};

}  // namespace

int main(int argc, char** argv) {
  const bool host_only = argc > 1 && std::string(argv[1]) == "--host";
#ifndef GM_LOOP_GPU
  if (!host_only) {
    std::fprintf(stderr, "built without GM_LOOP_GPU: only --host is available\n");
    return 2;
  }
#endif
  gm_device_spec dev;
  gm_device_spec_b200(&dev);
  gm_batch_policy pol;
  gm_batch_policy_default(&pol);
  pol.target_batch = 2;   // a pair of same-shape requests triggers a super-kernel
  pol.max_wait = 1e-3;    // ... or the oldest waiting 1 ms (age trigger)
  gm_detector det;
  gm_detector_default(&det);
  det.min_observations = 3;
  det.threshold_ratio = 3.0;
  gm_ctx* ctx = nullptr;
  OK(gm_create(&dev, &pol, &det, host_only ? -1 : 0, &ctx));

  std::mt19937_64 rng(42);
  std::uniform_real_distribution<float> u(-1.f, 1.f);
  std::vector<Buffers> buf(kTenants);
  for (int t = 0; t < kTenants; ++t) {
    for (int p = 0; p < kPasses; ++p) {
      const gm_gemm_shape s0 = shape_of(t, 0), s1 = shape_of(t, 1);
      std::vector<uint16_t> x(static_cast<size_t>(s0.m * s0.k));
      for (auto& v : x) v = to_bf16(u(rng));
      buf[t].in.push_back(std::move(x));
      buf[t].out.emplace_back(static_cast<size_t>(s1.m * s1.n), 0);
    }
  }
#ifdef GM_LOOP_GPU
  if (!host_only) {
    for (int t = 0; t < kTenants; ++t) {
      Buffers& b = buf[t];
      gm_layer_desc L[kLayers];
      std::memset(L, 0, sizeof(L));
      for (int l = 0; l < kLayers; ++l) {
        const gm_gemm_shape s = shape_of(t, l);
        std::normal_distribution<float> nd(0.f, std::sqrt(2.f / static_cast<float>(s.k)));
        std::vector<uint16_t> w(static_cast<size_t>(s.n * s.k));
        for (auto& v : w) v = to_bf16(nd(rng));
        if (cudaMalloc(&b.w[l], w.size() * 2) != cudaSuccess || cudaMalloc(&b.y[l], s.m * s.n * 2) != cudaSuccess)
          return 1;
        cudaMemcpy(b.w[l], w.data(), w.size() * 2, cudaMemcpyHostToDevice);
        b.wh.push_back(std::move(w));
        L[l].kind = GM_LAYER_GEMM;
        L[l].batch = 1;
        L[l].gemm = s;
        L[l].w = b.w[l];
        L[l].y = b.y[l];
        L[l].act = l == 0 ? GM_ACT_RELU : GM_ACT_NONE;
        L[l].src = l - 1;  // layer 1 reads layer 0's output
        L[l].res_src = -1;
      }
      const gm_gemm_shape s0 = shape_of(t, 0);
      if (cudaMalloc(&b.x0, s0.m * s0.k * 2) != cudaSuccess) return 1;
      L[0].x = b.x0;
      L[1].x = b.y[0];
      gm_tenant_desc td{"loop-tenant", L, kLayers, 0.040, 1, 0};
      int32_t idx = -1;
      OK(gm_register_tenant(ctx, &td, &idx));
      CHECK(idx == t, "tenant index %d", idx);
    }
  }
  cudaStream_t stream;
  if (!host_only) cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking);
#endif

  // error channel: the reference's what() texts, per ctx
  {
    gm_kernel_request bad{};
    bad.request_id = 7;
    bad.tenant_index = 0;
    bad.shape = gm_gemm_shape{0, 8, 8};
    CHECK(gm_enqueue(ctx, &bad, nullptr) == GM_EINVAL, "invalid shape accepted");
    CHECK(std::string(gm_last_error(ctx)).find("enqueue: invalid shape") != std::string::npos, "%s",
          gm_last_error(ctx));
  }

  uint64_t next_id = 1000;
  std::vector<int> pass_of(kTenants, 0);
  std::vector<bool> evicted(kTenants, false);
  int64_t dispatches = 0, packed_pairs = 0, completions = 0;
  auto submit = [&](int t, int layer, int64_t now) {
    gm_kernel_request r{};
    r.request_id = next_id++;
    r.tenant_index = t;
    r.layer_index = layer;
    r.shape = shape_of(t, layer);
    r.enqueue_time = now;
    r.slo_deadline = now + 40'000'000;
    r.pass_index = static_cast<uint32_t>(pass_of[t]);
    r.batch = 1;
    gm_request_io io{};
    if (!host_only && layer == 0) {
      io.x = buf[t].in[pass_of[t]].data();
      io.x_bytes = buf[t].in[pass_of[t]].size() * 2;
    }
    if (!host_only && layer == kLayers - 1) {
      io.y = buf[t].out[pass_of[t]].data();
      io.y_bytes = buf[t].out[pass_of[t]].size() * 2;
    }
    OK(gm_enqueue(ctx, &r, host_only ? nullptr : &io));
    if (r.request_id == 1000) {  // duplicate ids keep the reference text
      CHECK(gm_enqueue(ctx, &r, nullptr) == GM_EINVAL, "duplicate accepted");
      CHECK(std::string(gm_last_error(ctx)) == "enqueue: duplicate request id 1000", "%s", gm_last_error(ctx));
    }
  };

  int64_t vnow = 0;  // host-only: virtual clock (ns) advanced by planned costs
  auto now_ns = [&]() { return host_only ? vnow : gm_ctx_now_ns(ctx); };
  for (int t = 0; t < kTenants; ++t) submit(t, 0, now_ns());
  std::vector<gm_completion> done(64);
  int guard = 0;
  for (;;) {
    bool live = false;
    for (int t = 0; t < kTenants; ++t) live |= !evicted[t] && pass_of[t] < kPasses;
    if (!live) break;
    // bounded: a virtual-clock step per idle formation (host), a wall-clock
    // budget on the device
    const bool stuck = host_only ? ++guard >= 10000 : gm_ctx_now_ns(ctx) > 5'000'000'000LL;
    CHECK(!stuck, "loop does not terminate");
    if (stuck) break;
    gm_plans* plans = nullptr;
    OK(gm_ctx_form_batches(ctx, now_ns(), &plans));
    const size_t np = gm_plans_count(plans);
    if (np == 0) {  // nothing triggered yet: let the age trigger fire
      gm_plans_destroy(plans);
      if (host_only)
        vnow += 250'000;
      else
        std::this_thread::sleep_for(std::chrono::microseconds(50));
      continue;
    }
    std::vector<gm_completion> got;
    for (size_t i = 0; i < np; ++i) {
      gm_plan_info info;
      OK(gm_plans_get(plans, i, &info));
      std::vector<gm_kernel_request> mem(static_cast<size_t>(info.n_members));
      size_t nm = 0;
      OK(gm_plans_members(plans, i, mem.data(), mem.size(), &nm));
      ++dispatches;
      packed_pairs += nm == 2;
      for (size_t j = 0; j < nm; ++j) CHECK(!evicted[mem[j].tenant_index], "evicted tenant %d dispatched",
                                            mem[j].tenant_index);
      if (host_only) {
        CHECK(gm_dispatch(ctx, plans, i, 0, nullptr, nullptr) == GM_ENODEV, "host ctx dispatched");
        vnow += static_cast<int64_t>(info.planned_cost.duration * 1e9);
        for (size_t j = 0; j < nm; ++j) {
          gm_completion c{};
          c.request_id = mem[j].request_id;
          c.tenant_index = mem[j].tenant_index;
          c.layer_index = mem[j].layer_index;
          c.pass_index = mem[j].pass_index;
          c.exec_seconds = info.planned_cost.duration;
          c.plan_members = static_cast<int32_t>(nm);
          got.push_back(c);
        }
      } else {
        double planned = 0;
        int hit = 0;
        OK(gm_dispatch(ctx, plans, i, reinterpret_cast<uint64_t>(
#ifdef GM_LOOP_GPU
                                          stream
#else
                                          nullptr
#endif
                                          ), &planned, &hit));
        CHECK(planned > 0, "planned cost %g", planned);
      }
    }
    gm_plans_destroy(plans);
    if (!host_only) {  // one formation's super-kernels in flight; poll until all complete
      size_t in_flight = 1;
      while (in_flight) {
        size_t n = 0;
        OK(gm_poll_completions(ctx, done.data(), done.size(), &n));
        got.insert(got.end(), done.begin(), done.begin() + static_cast<long>(n));
        OK(gm_ctx_in_flight(ctx, &in_flight));
      }
    }
    for (const gm_completion& c : got) {
      ++completions;
      CHECK(c.exec_seconds > 0, "exec %g", c.exec_seconds);
      const int t = c.tenant_index;
      if (evicted[t]) continue;
      const double slow = t == kDegraded && c.pass_index >= 2 ? kSlowdown : 1.0;
      OK(gm_ctx_record_latency(ctx, t, c.exec_seconds * slow));
      if (c.layer_index + 1 < kLayers) {
        submit(t, c.layer_index + 1, now_ns());
      } else if (++pass_of[t] < kPasses) {
        submit(t, 0, now_ns());  // closed loop: the next query arrives at completion
      }
      int32_t s[kTenants];
      size_t ns = 0;
      OK(gm_ctx_detect_stragglers(ctx, s, kTenants, &ns));
      for (size_t k = 0; k < ns; ++k) {
        uint64_t gone[8];
        size_t ng = 0;
        OK(gm_ctx_evict(ctx, s[k], gone, 8, &ng));
        evicted[s[k]] = true;
        CHECK(gm_ctx_evict(ctx, s[k], gone, 8, &ng) == GM_EINVAL, "double evict accepted");
        CHECK(std::string(gm_last_error(ctx)) == "evict: tenant " + std::to_string(s[k]) + " already evicted", "%s",
              gm_last_error(ctx));
      }
    }
  }
  gm_tenant_health h;
  OK(gm_ctx_health(ctx, kDegraded, &h));
  CHECK(h.evicted == 1 && evicted[kDegraded], "degraded tenant not evicted");
  for (int t = 0; t < kTenants; ++t)
    if (t != kDegraded) CHECK(!evicted[t] && pass_of[t] == kPasses, "tenant %d: pass %d evicted %d", t, pass_of[t],
                              static_cast<int>(evicted[t]));
  CHECK(packed_pairs > 0, "no 2-member super-kernel formed");

  double worst = 0;
#ifdef GM_LOOP_GPU
  if (!host_only) {
    for (int t = 0; t < kTenants; ++t) {
      if (t == kDegraded) continue;
      const gm_gemm_shape s0 = shape_of(t, 0), s1 = shape_of(t, 1);
      std::vector<float> w0(buf[t].wh[0].size()), w1(buf[t].wh[1].size());
      for (size_t i = 0; i < w0.size(); ++i) w0[i] = from_bf16(buf[t].wh[0][i]);
      for (size_t i = 0; i < w1.size(); ++i) w1[i] = from_bf16(buf[t].wh[1][i]);
      for (int p = 0; p < kPasses; ++p) {
        std::vector<float> x(buf[t].in[p].size()), y0(static_cast<size_t>(s0.m * s0.n)),
            y1(static_cast<size_t>(s1.m * s1.n));
        for (size_t i = 0; i < x.size(); ++i) x[i] = from_bf16(buf[t].in[p][i]);
        oracle_gemm_nt(x.data(), w0.data(), y0.data(), s0.m, s0.n, s0.k, 0, 0, 1);
        for (float& v : y0) v = from_bf16(to_bf16(v));  // the device stores layer 0 in bf16
        oracle_gemm_nt(y0.data(), w1.data(), y1.data(), s1.m, s1.n, s1.k, 0, 0, 0);
        double num = 0, den = 0;
        for (size_t i = 0; i < y1.size(); ++i) {
          num = std::fmax(num, std::fabs(from_bf16(buf[t].out[p][i]) - y1[i]));
          den = std::fmax(den, std::fabs(y1[i]));
        }
        const double rel = num / std::fmax(den, 1e-30);
        CHECK(rel <= 1e-2, "tenant %d pass %d rel err %.3e", t, p, rel);
        worst = std::fmax(worst, rel);
      }
    }
  }
#endif
  gm_destroy(ctx);
  if (g_fail) return 1;
  std::printf("loop ok: %s, %lld dispatches (%lld 2-member), %lld completions, tenant %d evicted, worst rel err %.2e\n",
              host_only ? "host-only" : "device", static_cast<long long>(dispatches),
              static_cast<long long>(packed_pairs), static_cast<long long>(completions), kDegraded, worst);
  return 0;
}
