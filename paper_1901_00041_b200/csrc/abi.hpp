// Internal glue between the C-ABI (include/gpumux_b200.h) and the C++ core:
// opaque handle definitions, struct conversions and the error channel.
#pragma once

#include <new>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/gpumux_b200.h"
#include "planner.hpp"
#include "sim.hpp"

struct gm_ctx;

namespace gmb {

struct Runtime;  // GPU side (runtime.cu)

// A CUDA runtime/driver failure; maps to GM_ECUDA.
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// No usable sm_100 device; maps to GM_ENODEV.
struct NoDevice : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// Output buffer too small; maps to GM_ERANGE.
struct RangeError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void set_error(const std::string& msg);
int fail(int code, const char* what);
// Classifies the in-flight exception (call inside a catch block) into a
// gm_status, records its message as this thread's last error and, when ctx
// is given, as that context's last error (gm_last_error(ctx)).
int fail_current(const gm_ctx* ctx);

inline Shape to_shape(const gm_gemm_shape& s) { return Shape{s.m, s.n, s.k}; }
inline gm_gemm_shape from_shape(const Shape& s) { return gm_gemm_shape{s.m, s.n, s.k}; }

inline Conv to_conv(const gm_conv_spec& c) {
  return Conv{c.image_h, c.image_w, c.kernel_h, c.kernel_w, c.in_channels, c.out_channels, c.stride, c.padding};
}

Device to_device(const gm_device_spec& d);
gm_device_spec from_device(const Device& d);
Policy to_policy(const gm_batch_policy& p);
Detector to_detector(const gm_detector& d);
gm_kernel_cost from_cost(const Cost& c);
Request to_request(const gm_kernel_request& r);
gm_kernel_request from_request(const Request& r);
Health to_health(const gm_tenant_health& h);
gm_tenant_health from_health(const Health& h);

}  // namespace gmb

struct gm_queue {
  gmb::Queue q;
};
struct gm_plans {
  std::vector<gmb::Plan> plans;
  std::vector<std::pair<gmb::TimeNs, gmb::TimeNs>> times;  // virtual [start, end) when planned by a round
};
struct gm_cache {
  gmb::SignatureCache c;
};
struct gm_sim_trace {
  gmb::SpaceTimeTrace t;
};

// Per-GPU context: the scheduler state the reference engine owns for one
// device (queue, signature cache, monitor) plus the device runtime.
struct gm_ctx {
  gmb::Device dev;
  gmb::Policy pol;
  gmb::Detector det;
  gm_queue queue;
  gm_cache cache;
  std::vector<gmb::Health> health;
  int cuda_device = -1;
  std::uint64_t next_request_id = 1;
  gmb::Runtime* rt = nullptr;
  std::int64_t clock0_ns = 0;           // steady-clock origin of gm_ctx_now_ns
  std::unordered_map<std::uint64_t, gm_request_io> io;  // gm_enqueue I/O by request id
  mutable std::string last_error;       // gm_last_error(ctx)
};

// Wraps an API body: maps C++ exceptions to status codes + gm_last_error().
// GM_CTX_API_END(ctx) also records the message on that context.
#define GM_API_BEGIN try {
#define GM_API_END                                         \
  }                                                        \
  catch (...) { return gmb::fail_current(nullptr); }       \
  return GM_OK;
#define GM_CTX_API_END(CTX)                                \
  }                                                        \
  catch (...) { return gmb::fail_current(CTX); }           \
  return GM_OK;
