/*
 * gpumux_b200.h — C-ABI of the B200-native space-time multiplexing path.
 *
 * This is the drop-in boundary for the reference's space-time scheduler
 * (arxiv 1901.00041, artifact "gpumux").  The reference exposes a plain C++
 * static-library API with no FFI layer; every entry point below names the
 * reference function it replaces (file:line under /root/reference/proj).
 *
 *   - plain C types only: POD structs, pointers, sizes; no torch, no STL
 *   - every function returns an int status (GM_OK == 0); the message of the
 *     last failure is gm_last_error(ctx) for calls on a context, and
 *     gm_last_error(NULL) for the calling thread's last failure of any call —
 *     messages equal the reference's std::invalid_argument::what() texts
 *   - objects (queue, plans, cache, ctx) are opaque handles; a handle is a
 *     single logical actor and is not thread-safe; use one
 *     gm_ctx per GPU on one host thread (tenant-sharded placement)
 *
 * Status codes mirror the reference's exception classes and CLI exit codes
 * (proj/tools/gpumux.cpp:26-30).
 */
#ifndef GPUMUX_B200_H
#define GPUMUX_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GM_ABI_VERSION 3

enum gm_status {
  GM_OK = 0,
  GM_EINVAL = 1,     /* std::invalid_argument (misuse)                    */
  GM_ECONFIG = 2,    /* gpumux::ConfigError      (CLI exit 1)             */
  GM_EOOM = 3,       /* gpumux::InfeasibleError / device OOM (CLI exit 2) */
  GM_EINTERNAL = 4,  /* anything else            (CLI exit 3)             */
  GM_ECUDA = 5,      /* CUDA runtime/driver failure                       */
  GM_ERANGE = 6,     /* caller-provided output buffer too small           */
  GM_ENODEV = 7      /* no sm_100 device / CUDA path unavailable          */
};

/* ---- L0 domain types (proj/include/gpumux/gemm.hpp:11-31) ---------------- */

typedef struct gm_gemm_shape {      /* GemmShape, gemm.hpp:11-20 */
  int64_t m, n, k;
} gm_gemm_shape;

typedef struct gm_conv_spec {       /* ConvSpec, gemm.hpp:23-31 */
  int64_t image_h, image_w, kernel_h, kernel_w;
  int64_t in_channels, out_channels, stride, padding;
} gm_conv_spec;

/* DeviceSpec, proj/include/gpumux/device.hpp:13-30 (field order kept). */
typedef struct gm_device_spec {
  double peak_flops;
  double mem_bandwidth;
  int64_t sm_count;
  int64_t blocks_per_sm;
  double launch_overhead;
  double context_switch_overhead;
  double planning_overhead;
  double mem_capacity;
  double process_context_bytes;
  int64_t tile_m;
  int64_t tile_n;
  double space_sched_penalty;
  double launch_serialization;
  /* b200 extension, 0 in the reference profiles: a super-kernel lasts at
   * least waves x (tile_latency + kblock_latency x k-blocks (64 of K) of its
   * longest-K member) -- the latency bound of few-tile plans on the
   * persistent kernel, fitted by tools/calibrate_b200.py. */
  double tile_latency;
  double kblock_latency;
} gm_device_spec;

typedef struct gm_kernel_cost {     /* KernelCost, cost_model.hpp:14-20 */
  int64_t flops;
  int64_t bytes;
  int64_t blocks;
  double duration;                  /* seconds */
  int64_t waves;
} gm_kernel_cost;

typedef struct gm_kernel_group {    /* KernelGroup, cost_model.hpp:24-27 */
  gm_gemm_shape shape;
  int64_t count;
} gm_kernel_group;

/* KernelRequest, scheduler.hpp:17-25.  `batch` is a B200 extension (query
 * coalescing, gemm.hpp:54-56); the planner never reads it (default 1). */
typedef struct gm_kernel_request {
  uint64_t request_id;
  int32_t tenant_index;
  int32_t layer_index;
  gm_gemm_shape shape;
  int64_t enqueue_time;             /* ns */
  int64_t slo_deadline;             /* absolute ns */
  uint32_t pass_index;
  uint32_t batch;
} gm_kernel_request;

typedef struct gm_batch_policy {    /* BatchPolicy, scheduler.hpp:28-34 */
  double max_wait;                  /* seconds */
  int64_t target_batch;
  int32_t allow_variable_size;
  int32_t max_waves;                /* B200 extension: waves one super-kernel may fill;
                                       0/1 = the reference's one-wave cap */
  double slo_safety_margin;
  double variable_inefficiency;
} gm_batch_policy;

typedef struct gm_tenant_health {   /* TenantHealth, scheduler.hpp:44-50 */
  int32_t tenant_index;
  int32_t evicted;
  double ewma_latency;
  double ewma_alpha;
  int64_t observed_count;
} gm_tenant_health;

typedef struct gm_detector {        /* DetectorParams, sim.hpp:32-37 */
  double ewma_alpha;
  int64_t min_observations;
  double threshold_ratio;
  int32_t evict_stragglers;
  int32_t reserved0;
} gm_detector;

/* One entry of the per-CTA tile-dispatch table.  Entries are
 * flattened in member order, then m-tile-major, then n-tile, so the table
 * length equals plan_super_kernel(...).blocks under the same DeviceSpec. */
typedef struct gm_tile {
  uint16_t member;                  /* index into the plan's member list */
  uint16_t flags;                   /* reserved (0) */
  uint16_t m_tile;
  uint16_t n_tile;
} gm_tile;

/* Summary of one formed SuperKernel (scheduler.hpp:37-42). */
typedef struct gm_plan_info {
  int32_t uniform;
  int32_t reserved0;
  int64_t n_members;
  gm_kernel_cost planned_cost;
  const char* signature;            /* owned by the gm_plans handle */
} gm_plan_info;

/* ---- defaults and profiles ---------------------------------------------- */

typedef struct gm_ctx gm_ctx;       /* one per GPU (see below) */

/* Message of the last failed call on ctx (NULL: of this thread's last failed
 * call).  The reference throws; its what() text is this string. */
const char* gm_last_error(const gm_ctx* ctx);
int gm_abi_version(void);

void gm_device_spec_default(gm_device_spec* out);  /* DeviceSpec{} defaults   */
void gm_device_spec_v100(gm_device_spec* out);     /* v100_profile(), device.cpp:41-59 */
/* B200 profile: tile_m/tile_n = the super-kernel CTA tile, sm_count = 148,
 * blocks_per_sm = 1 (one persistent CTA per SM).  Peaks from the measured
 * roofline (MEASURED_PEAKS.json); overheads fitted to B200 launches. */
void gm_device_spec_b200(gm_device_spec* out);
int gm_device_spec_validate(const gm_device_spec* d);  /* DeviceSpec::validate, device.cpp:19-39 */
void gm_batch_policy_default(gm_batch_policy* out);
void gm_detector_default(gm_detector* out);

/* ---- L0/L1: shapes and cost model --------------------------------------- */

int64_t gm_gemm_flops(const gm_gemm_shape* s);                 /* gemm.hpp:33-35 */
int64_t gm_gemm_bytes(const gm_gemm_shape* s, int64_t elem);   /* gemm.hpp:38-40 */
int gm_im2col_gemm_dims(const gm_conv_spec* c, gm_gemm_shape* out); /* gemm.hpp:44-51 */
void gm_batch_inputs(const gm_gemm_shape* s, int64_t batch, gm_gemm_shape* out); /* gemm.hpp:54-56 */
int gm_shape_key(const gm_gemm_shape* s, char* buf, size_t cap); /* gemm.hpp:58-60 */
int64_t gm_to_ns(double seconds);                              /* vtime.hpp:13-15 */
double gm_to_seconds(int64_t ns);                              /* vtime.hpp:17-19 */
int64_t gm_thread_blocks(const gm_gemm_shape* s, const gm_device_spec* d); /* cost_model.cpp:14-16 */
/* dispatch_duration, cost_model.cpp:18-46 */
int gm_dispatch_duration(const gm_kernel_group* groups, size_t n, const gm_device_spec* d,
                         int64_t slot_budget, int64_t launches, gm_kernel_cost* out);

/* ---- L2b: space-time scheduler (scheduler.hpp:59-122) ------------------- */

typedef struct gm_queue gm_queue;   /* RequestQueue */
typedef struct gm_plans gm_plans;   /* std::vector<SuperKernel> */
typedef struct gm_cache gm_cache;   /* SuperKernelCache */

int gm_queue_create(gm_queue** out);
void gm_queue_destroy(gm_queue* q);
int gm_queue_enqueue(gm_queue* q, const gm_kernel_request* r);  /* scheduler.cpp:8-16 */
int64_t gm_queue_size(const gm_queue* q);
/* Pending requests in group order (ascending m,n,k), FIFO within a group. */
int gm_queue_snapshot(const gm_queue* q, gm_kernel_request* out, size_t cap, size_t* n);
int gm_queue_group_count(const gm_queue* q, size_t* n);
/* RequestQueue::cancel_tenant, scheduler.cpp:18-35 */
int gm_queue_cancel_tenant(gm_queue* q, int32_t tenant, gm_kernel_request* out, size_t cap,
                           size_t* n);

/* form_batches, scheduler.cpp:96-199.  Mutates the queue; *out receives a
 * new plans handle (possibly empty) that the caller destroys. */
int gm_form_batches(gm_queue* q, int64_t now, const gm_batch_policy* p,
                    const gm_device_spec* d, gm_plans** out);
size_t gm_plans_count(const gm_plans* p);
int gm_plans_get(const gm_plans* p, size_t i, gm_plan_info* out);
int gm_plans_members(const gm_plans* p, size_t i, gm_kernel_request* out, size_t cap, size_t* n);
void gm_plans_destroy(gm_plans* p);
/* 64-bit identity of a plan list (signatures + member tenant/layer ids): the
 * key under which a captured launch program is cached and replayed. */
int gm_plans_key(const gm_plans* p, uint64_t* key);
/* Tile-dispatch table of plan i under device d. */
int gm_build_tile_table(const gm_plans* p, size_t i, const gm_device_spec* d, gm_tile* out,
                        size_t cap, size_t* n);

/* plan_super_kernel, scheduler.cpp:43-61 */
int gm_plan_super_kernel(const gm_kernel_request* members, size_t n, int uniform,
                         const gm_batch_policy* p, const gm_device_spec* d, gm_kernel_cost* out);
/* slo_headroom, scheduler.cpp:37-41 */
double gm_slo_headroom(const gm_kernel_request* r, int64_t now, double predicted,
                       const gm_batch_policy* p);

int gm_cache_create(gm_cache** out);
void gm_cache_destroy(gm_cache* c);
/* dispatch_cost, scheduler.cpp:201-212 */
int gm_dispatch_cost(const gm_plans* p, size_t i, gm_cache* c, const gm_device_spec* d,
                     double* duration, int* cache_hit);
int gm_cache_stats(const gm_cache* c, int64_t* hits, int64_t* misses, int64_t* entries);

/* record_latency / detect_stragglers / evict, scheduler.cpp:214-271 */
int gm_record_latency(gm_tenant_health* h, double observed_seconds);
int gm_detect_stragglers(const gm_tenant_health* h, size_t n, double threshold_ratio,
                         int64_t min_observations, int32_t* out, size_t cap, size_t* n_out);
int gm_evict(gm_tenant_health* h, size_t n, gm_queue* q, int32_t tenant,
             gm_kernel_request* out, size_t cap, size_t* n_out);

/* ---- L4: metrics (metrics.cpp:10-28) ------------------------------------ */
int gm_percentile_nearest_rank(const double* v, size_t n, double pct, double* out);
int gm_geomean(const double* v, size_t n, double* out);

/* ---- L3: space-time driver, virtual clock (sim.cpp:398-581) -------------
 * Closed-loop run_space_time over homogeneous tenants (same layer list).
 * Produces the dispatch sequence the reference engine produces; the B200
 * runtime replays that plan stream on the GPU. */
typedef struct gm_sim_config {
  gm_device_spec device;
  gm_batch_policy scheduler;
  gm_detector detector;
  const gm_gemm_shape* layers;      /* shared layer list */
  size_t n_layers;
  int32_t n_tenants;
  int32_t concurrency;
  double slo_latency;               /* seconds per pass */
  double duration;                  /* virtual seconds */
  double warmup;
  int32_t microbench;               /* 1 = keep layer 0 only (SimMode::kMicrobench) */
  int32_t degrade_tenant;           /* -1 = none (inject_degradation, sim.cpp:60-68) */
  double degrade_slowdown;
  double degrade_start;
} gm_sim_config;

typedef struct gm_sim_event {       /* DispatchEvent (policies.hpp) for space-time */
  int64_t start, end;
  int64_t flops;
  double occupancy;
  int64_t member_offset;            /* into the member-id array */
  int64_t n_members;
} gm_sim_event;

typedef struct gm_sim_completion {  /* RequestLifecycle, sim.hpp:62-71 */
  uint64_t request_id;
  int32_t tenant_index;
  int32_t slo_met;
  int64_t enqueue_time, dispatch_time, complete_time;
  int64_t flops;
} gm_sim_completion;

typedef struct gm_sim_trace gm_sim_trace;
int gm_simulate_space_time(const gm_sim_config* cfg, gm_sim_trace** out);
int gm_sim_trace_counts(const gm_sim_trace* t, size_t* n_events, size_t* n_members,
                        size_t* n_completions, size_t* n_cancelled, int64_t* cache_hits,
                        int64_t* cache_misses);
int gm_sim_trace_events(const gm_sim_trace* t, gm_sim_event* ev, size_t cap_ev,
                        uint64_t* member_ids, size_t cap_ids);
int gm_sim_trace_completions(const gm_sim_trace* t, gm_sim_completion* out, size_t cap);
int gm_sim_trace_evictions(const gm_sim_trace* t, int32_t* tenants, int64_t* times, size_t cap,
                           size_t* n);
int gm_sim_trace_flops(const gm_sim_trace* t, int64_t* dispatched, int64_t* completed);
void gm_sim_trace_destroy(gm_sim_trace* t);

/* One closed-loop space-time round on the virtual clock, host only (no GPU):
 * every listed tenant submits one forward pass at `start` and the
 * run_space_time loop (proj/src/sim.cpp:452-576: dispatch FIFO, formation only
 * when the FIFO is empty, completion fan-out of the next layer, wake timer)
 * runs until every pass has completed.  This is the planner behind
 * gm_plan_round (which reads the layer lists from registered tenants); for a
 * homogeneous tenant set its dispatches equal the reference engine's first-pass
 * dispatches (tests/test_round_parity.py).  `cache` (nullable) and `next_id`
 * (nullable, in/out) persist across rounds like a gm_ctx's. */
typedef struct gm_round_tenant {
  int32_t tenant;
  int32_t reserved;
  const gm_gemm_shape* layers;
  size_t n_layers;
  int64_t slo_ns;                   /* pass deadline = start + slo_ns */
} gm_round_tenant;
int gm_plan_round_shapes(const gm_round_tenant* tenants, size_t n, int64_t start, const gm_batch_policy* p,
                         const gm_device_spec* d, gm_cache* cache, uint64_t* next_id, gm_plans** out);

/* ---- B200 runtime: tenants, super-kernel dispatch ------------------------ */

/* DWCONV: depthwise conv (groups = channels; MobileNet-v2).  The planner sees
 * the reference's model of it, a K = R*S GEMM (proj/src/workload.cpp:66):
 * (b*P*Q, C, R*S); w is [C, ldw] with R*S taps per row; R*S <= 9, C % 4 == 0. */
enum gm_layer_kind { GM_LAYER_GEMM = 0, GM_LAYER_CONV = 1, GM_LAYER_DWCONV = 2, GM_LAYER_MAXPOOL = 3,
                     GM_LAYER_AVGPOOL = 4 };
/* MAXPOOL / AVGPOOL: conv = the window (kernel_h/w, stride, padding; in ==
 * out channels), w unused (may be null); planned like a depthwise conv, a
 * K = R*S GEMM; executed as CUDA-core tiles of the same persistent launch.
 * Pool FLOPs are not tensor work and are not counted by the benchmarks. */

/* Fused epilogue activations (after the residual add). */
enum gm_activation { GM_ACT_NONE = 0, GM_ACT_RELU = 1, GM_ACT_RELU6 = 2, GM_ACT_GELU = 3 };

/* One operator of a tenant's graph, with its device buffers (bf16).
 *   CONV: x = NHWC [batch, H, W, Cin]; w = KRSC [Cout, R, S, Cin] with a row
 *         stride of ldw elements (ldw >= R*S*Cin, ldw % 8 == 0);
 *         y = NHWC [batch, P, Q, Cout]  (== row-major [M, N])
 *   GEMM: x = A [m, k] row-major (row stride ldx), w = B [n, k] (row stride
 *         ldw), y = C [m, n] row-major. */
typedef struct gm_layer_desc {
  int32_t kind;
  int32_t batch;                    /* CONV only: images per query batch */
  gm_conv_spec conv;
  gm_gemm_shape gemm;
  const void* x;
  const void* w;
  void* y;
  int64_t ldx;                      /* 0 = dense */
  int64_t ldw;                      /* 0 = dense */
  int32_t act;                      /* gm_activation fused into the epilogue */
  /* Dataflow: the layer of this tenant whose output y is this layer's x
   * (-1 = an external input, e.g. the tenant's query batch).  x must then
   * point into that layer's y.  In a round program the layer runs after its
   * source by the tenant's dependency chain (a tenant's layers run in order,
   * proj/src/sim.cpp:482-488). */
  int32_t src;
  /* Fused residual add: y = act(x * W + res), res [M, N] bf16 row-major with
   * row stride ldr (0 = N; 16-byte aligned rows), null = none.  res_src: the
   * earlier layer of this tenant whose y it is (-1 = external). */
  const void* res;
  int64_t ldr;
  int32_t res_src;
  int32_t reserved0;
} gm_layer_desc;

typedef struct gm_tenant_desc {     /* Tenant, workload.hpp:14-22 */
  const char* tenant_id;
  const gm_layer_desc* layers;
  size_t n_layers;
  double slo_latency;
  int32_t concurrency;
  int32_t reserved0;
} gm_tenant_desc;

/* cuda_device < 0 creates a host-only context (planner, no launches). */
int gm_create(const gm_device_spec* d, const gm_batch_policy* p, const gm_detector* det,
              int cuda_device, gm_ctx** out);
void gm_destroy(gm_ctx* ctx);
int gm_ctx_queue(gm_ctx* ctx, gm_queue** q);
int gm_ctx_cache(gm_ctx* ctx, gm_cache** c);
int gm_ctx_device_spec(const gm_ctx* ctx, gm_device_spec* out);
/* Replace the BatchPolicy gm_plan_round uses (e.g. parity vs b200 mode). */
int gm_ctx_set_policy(gm_ctx* ctx, const gm_batch_policy* p);
/* Execution options of the device runtime (none changes results; defaults in
 * parentheses; tile-shape options apply to plans prepared afterwards):
 *   "pdl"               programmatic dependent launch between launches (1)
 *   "narrow_min_tiles"  in a plan that leaves most SMs idle, narrow a member's
 *                       N tile (256/128/64) until it has this many tiles; 0 = off (20)
 *   "tall_tiles"        256-row tiles for N <= 128 members of throughput-bound
 *                       plans (1); "tall_min_tiles": concurrent same-shape tiles
 *                       that count as throughput-bound (0 = 2 x SMs)
 *   "split_k"           round programs split few-tile long-K members (0);
 *                       "max_splits" (4), "split_min_kb" (8)
 *   "split_wide_kb"     a member narrowed below 128 columns with at least this
 *                       many k-blocks keeps 128-column tiles and splits K over
 *                       the same tile count instead; 0 = off (0)
 *   "skinny_min_mb"     round programs split weight-streaming GEMM members
 *                       (M <= 64, at least this many MB of weights, e.g. fc6)
 *                       over K across the idle SMs; 0 = off (64);
 *                       "skinny_max_splits" (8)
 *   "ring_layouts"      narrow members use a 6 x 32 KB operand ring (1)
 *   "critical_order"    round tile order: -1 auto (= 2), 0 plan, 1 remaining work,
 *                       2 chain progress (-1)
 *   "greedy_schedule"   greedy in-order tile claiming instead of static
 *                       round-robin (0); "dynamic_schedule": per-tenant queues (0)
 *   "row_fold"          row-folded im2col for RGB stems (1)
 */
int gm_ctx_set_option(gm_ctx* ctx, const char* name, int64_t value);

/* Registers a tenant and builds its per-layer member descriptors (TMA maps)
 * on the device.  Replaces make_tenants (workload.cpp:113-128). */
int gm_register_tenant(gm_ctx* ctx, const gm_tenant_desc* t, int32_t* tenant_index);
int gm_layer_shape(gm_ctx* ctx, int32_t tenant, int32_t layer, gm_gemm_shape* out);
int gm_tenant_count(const gm_ctx* ctx, int32_t* n);
/* Re-admit a tenant on another context (another GPU, or the same one): the
 * destination allocates the tenant's buffers (owned by that ctx), copies its
 * weights and external inputs with cudaMemcpyPeerAsync on `stream`, and
 * registers the layers with the same dataflow; *out_tenant = the new index.
 * Replaces the reference's terminal eviction (scheduler.cpp:225-244; SPEC.md:331
 * names re-admission as the open extension).  Errors report on `src`. */
int gm_migrate_tenant(gm_ctx* src, int32_t tenant, gm_ctx* dst, uint64_t stream, int32_t* out_tenant);
/* Several tenants at once: a source buffer several of them reference (a
 * logical tenant's batch variants are registrations over one set of buffers)
 * is placed once on the destination and shared there too. */
int gm_migrate_tenants(gm_ctx* src, const int32_t* tenants, size_t n, gm_ctx* dst, uint64_t stream,
                       int32_t* out_tenants);

/* Prepare (host→device upload on a miss, never inside graph capture) and
 * launch the super-kernel of plan i on `stream` (a cudaStream_t; 0 = legacy
 * default).  planned_s/cache_hit follow dispatch_cost (scheduler.cpp:201-212)
 * against the ctx's SuperKernelCache.  Members enqueued with gm_enqueue I/O
 * get their copies around the launch, and the dispatch is tracked for
 * gm_poll_completions (outside stream capture).  Launches are CUDA-graph
 * capturable once prepared. */
int gm_prepare(gm_ctx* ctx, const gm_plans* p, size_t i);
int gm_dispatch(gm_ctx* ctx, const gm_plans* p, size_t i, uint64_t stream, double* planned_s,
                int* cache_hit);
/* ---- host-driven loop over one ctx (the reference run_space_time shape,
 * proj/src/sim.cpp:452-576): gm_enqueue -> gm_ctx_form_batches ->
 * gm_dispatch -> gm_poll_completions -> gm_ctx_record_latency ->
 * gm_ctx_detect_stragglers -> gm_ctx_evict.  An external scheduler drives the
 * GPU asynchronously through these; gm_serve is the same loop run natively. */

/* I/O of one request (B200 extension of KernelRequest): host (pinned or
 * pageable) or device pointers.  x: copied into the layer's registered input
 * on the dispatch stream right before the super-kernel that runs the request
 * (a query batch arriving at layer 0); y: the layer's output copied out right
 * after it.  Either may be NULL / 0 bytes.  Sizes must not exceed the
 * registered buffers. */
typedef struct gm_request_io {
  const void* x;
  size_t x_bytes;
  void* y;
  size_t y_bytes;
} gm_request_io;

/* RequestQueue::enqueue (scheduler.cpp:8-16) on the ctx's queue, plus the
 * request's I/O (nullable).  On a device ctx the (tenant, layer) must be
 * registered and the request's shape equal its GEMM shape.  Errors keep the
 * reference texts ("enqueue: duplicate request id N", "enqueue: invalid shape"). */
int gm_enqueue(gm_ctx* ctx, const gm_kernel_request* r, const gm_request_io* io);
/* form_batches (scheduler.cpp:96-199) over the ctx's queue, policy and device. */
int gm_ctx_form_batches(gm_ctx* ctx, int64_t now, gm_plans** out);
/* Nanoseconds on the ctx's steady clock (origin: gm_create); the clock of
 * gm_completion's dispatch/complete stamps. */
int64_t gm_ctx_now_ns(const gm_ctx* ctx);

/* One completed member request of a dispatched super-kernel: the per-member
 * completion fan-out of run_space_time (sim.cpp:466-476). */
typedef struct gm_completion {
  uint64_t request_id;
  int32_t tenant_index;
  int32_t layer_index;
  uint32_t pass_index;
  uint32_t batch;
  int64_t enqueue_time;             /* as enqueued (caller's clock) */
  int64_t slo_deadline;
  int64_t dispatch_ns;              /* gm_ctx_now_ns at gm_dispatch */
  int64_t complete_ns;              /* gm_ctx_now_ns when the poll first saw it complete */
  double exec_seconds;              /* the super-kernel's device time (CUDA events): the
                                       execution time record_latency takes (sim.cpp:475-476) */
  int32_t plan_members;             /* members of its super-kernel */
  int32_t reserved0;
} gm_completion;

/* Non-blocking: appends the member completions of every dispatch whose work
 * (copy-in, super-kernel, copy-out) has finished, in dispatch order, whole
 * dispatches only; *n = completions written.  GM_ERANGE if the oldest
 * finished dispatch has more members than cap. */
int gm_poll_completions(gm_ctx* ctx, gm_completion* out, size_t cap, size_t* n);
/* Dispatches issued by gm_dispatch that gm_poll_completions has not yet returned. */
int gm_ctx_in_flight(const gm_ctx* ctx, size_t* n);
/* Blocks until every dispatch in flight has finished on the device. */
int gm_ctx_synchronize(gm_ctx* ctx);

/* The ctx's TenantHealth vector (one per registered tenant; on a host-only
 * ctx, one per tenant index seen by gm_enqueue):
 * record_latency / detect_stragglers / evict, scheduler.cpp:214-271, with the
 * ctx's DetectorParams.  gm_ctx_evict also drops the cancelled requests' I/O. */
int gm_ctx_record_latency(gm_ctx* ctx, int32_t tenant, double observed_seconds);
int gm_ctx_detect_stragglers(gm_ctx* ctx, int32_t* out, size_t cap, size_t* n);
int gm_ctx_evict(gm_ctx* ctx, int32_t tenant, uint64_t* cancelled_ids, size_t cap, size_t* n);
int gm_ctx_health(const gm_ctx* ctx, int32_t tenant, gm_tenant_health* out);

/* Launch an explicit member list (tenant, layer pairs) as one super-kernel;
 * n == 1 is the single-problem kernel used by the time-only / space-only
 * baseline modes.  Returns the number of kernels launched in *launches. */
int gm_launch_members(gm_ctx* ctx, const int32_t* tenants, const int32_t* layers, size_t n,
                      uint64_t stream, int32_t* launches);
/* Number of kernels one dispatch of this member list launches (the super-kernel
 * plus an explicit-im2col pre-pass when a member needs one). */
int gm_members_launch_count(gm_ctx* ctx, const int32_t* tenants, const int32_t* layers, size_t n,
                            int32_t* launches);
/* One closed-loop space-time round over registered tenants: each listed tenant
 * submits one forward pass at `now`; the run_space_time loop (sim.cpp:452-576:
 * dispatch FIFO, formation when the FIFO is empty, completion fan-out, wake
 * timer) runs on the virtual clock until every pass completes.  Uses the ctx's
 * BatchPolicy (target_batch 0 = auto), DeviceSpec and SuperKernelCache.
 * Returns the dispatch sequence as a plans handle (gm_plans_times gives each
 * dispatch's virtual window). */
int gm_plan_round(gm_ctx* ctx, const int32_t* tenants, size_t n, int64_t now, gm_plans** out);
int gm_plans_times(const gm_plans* p, size_t i, int64_t* start, int64_t* end);
/* Launch every plan of a handle in order on `stream` (prepares on a miss;
 * capturable once prepared).  *launches = kernels launched. */
int gm_dispatch_plans(gm_ctx* ctx, const gm_plans* p, uint64_t stream, int32_t* launches);
int gm_prepare_plans(gm_ctx* ctx, const gm_plans* p);
/* ---- CUDA-graph launch programs (the B200 meaning of "cache super-kernels
 * as workloads stabilize"): a steady-state plan stream is
 * captured once and replayed with one cudaGraphLaunch. */
enum gm_mode { GM_MODE_PACKED = 0, GM_MODE_TIME_ONLY = 1, GM_MODE_SPACE_ONLY = 2 };
typedef struct gm_graph gm_graph;
/* Packed: every plan of `p`, in order, one super-kernel launch each. */
int gm_graph_capture_plans(gm_ctx* ctx, const gm_plans* p, int timed, gm_graph** out);
/* Baselines over the same kernel code (run_time_mux sim.cpp:188-292 /
 * run_spatial sim.cpp:298-373 mode definitions): every layer of every listed
 * tenant as its own single-member launch — TIME_ONLY serially on one stream in
 * tenant order, SPACE_ONLY on one stream per tenant, forked and joined. */
int gm_graph_capture_serial(gm_ctx* ctx, const int32_t* tenants, size_t n, int mode, int timed,
                            gm_graph** out);
/* Round program: every plan of `p` (a round from gm_plan_round) in ONE
 * persistent super-kernel launch.  Tiles keep plan order; a member's
 * activations are loaded only after every tile of the same tenant's previous
 * layer is stored (device-side completion counters), weights stream ahead.
 * The per-plan launch boundary of the reference (one SuperKernel = one
 * launch) becomes a dependency edge, so no SM drains between plans. */
int gm_dispatch_round(gm_ctx* ctx, const gm_plans* p, uint64_t stream, int32_t* launches);
int gm_graph_capture_round(gm_ctx* ctx, const gm_plans* p, int timed, gm_graph** out);
/* Profiling: run the round program once with in-kernel %globaltimer stamps,
 * 6 per tile in round-tile order: producer first issue, activation gate
 * passed, first stage landed (MMA), last MMA committed, accumulator ready
 * (epilogue), stores issued.  gm_round_tiles lists the round's tiles
 * (member = registered slot, flags = plan index). */
int gm_trace_round(gm_ctx* ctx, const gm_plans* p, uint64_t stream, uint64_t* out, size_t cap, size_t* n_tiles);
int gm_round_tiles(gm_ctx* ctx, const gm_plans* p, gm_tile* out, size_t cap, size_t* n);
/* The executed tile table of a round program, one entry per tile in launch
 * order: which operator, which output tile, the tile variant the runtime
 * chose (tall 256-row, N width, split-K slice) and its device-side
 * dependency edges: one counter per output row block of a member instance;
 * a tile waits for the producer row blocks its input rows (and residual
 * rows) come from, -1 = none.  Differs from gm_build_tile_table (the planner's tile count,
 * thread_blocks under the b200 profile) by those variants. */
typedef struct gm_round_tile {
  int32_t tenant, layer;
  int32_t m_tile, n_tile;
  int32_t rows, cols;               /* output rows per tile (128 / 256 / 32) and N width */
  int32_t splits, kb_begin, kb_end; /* split-K slice (splits 1: the whole K, kb_end 0) */
  int32_t done;                     /* the tile's row-block counter (-1: nothing waits on it) */
  int32_t dep, dep_n;               /* waits on counters [dep, dep + dep_n): its input's row blocks */
  int32_t rdep, rdep_n;             /* and [rdep, rdep + rdep_n): its residual's row blocks */
  int32_t plan;                     /* index of the formed super-kernel it came from */
  int32_t cuda_core;                /* 1: depthwise / pool tile computed on CUDA cores */
} gm_round_tile;
int gm_round_tile_info(gm_ctx* ctx, const gm_plans* p, gm_round_tile* out, size_t cap, size_t* n);
/* End-to-end round program (the serving call with host buffers): per tenant
 * i, an H2D copy h_in[i] -> d_in[i] (its query batch) and its layer-0
 * pre-pass run on a copy branch that then opens the tenant's input gate; the
 * round kernel runs concurrently and starts each tenant's chain when its
 * gate opens; D2H copies d_out[i] -> h_out[i] follow the kernel.  Host
 * buffers should be pinned; the graph is bound to these pointers. */
int gm_graph_capture_round_e2e(gm_ctx* ctx, const gm_plans* p, size_t n, const int32_t* tenants,
                               const void* const* h_in, void* const* d_in, const size_t* in_bytes,
                               const void* const* d_out, void* const* h_out, const size_t* out_bytes,
                               gm_graph** out);
int gm_graph_launch(gm_graph* g, uint64_t stream);
int gm_graph_launch_count(const gm_graph* g, int32_t* superkernels, int32_t* kernels);
/* timed graphs: synchronizes on the last launch and returns the elapsed ms of
 * every super-kernel launch (external event pairs captured around each). */
int gm_graph_kernel_times(gm_graph* g, float* ms, size_t cap, size_t* n);
void gm_graph_destroy(gm_graph* g);

/* Total super-kernel launches and tiles issued by this ctx so far. */
int gm_ctx_launch_stats(const gm_ctx* ctx, int64_t* superkernels, int64_t* prepasses,
                        int64_t* tiles);

/* ---------------------------------------------------------------- serving
 * Real-clock space-time serving on one GPU: the B200 form of the reference's
 * run_space_time loop (proj/src/sim.cpp:398-581) with query arrivals, the
 * dynamic batcher's size/age/SLO triggers (form_batches, scheduler.cpp:166-197),
 * one round program per dispatch, CUDA-event completions feeding
 * record_latency / detect_stragglers / evict (scheduler.cpp:214-271).
 * A logical tenant registers one runtime tenant per batch variant (same
 * buffers, sized for the largest batch); a dispatch serves up to the largest
 * batch of its pending queries with the smallest variant that holds them. */
typedef struct gm_serve_tenant {
  int32_t n_variants;
  const int32_t* variant_tenant;  /* runtime tenant index per variant */
  const int32_t* variant_batch;   /* queries (images / sequences) per variant */
  double rate_qps;                /* Poisson arrivals per second; 0 = closed loop */
  int32_t concurrency;            /* closed loop: queries outstanding */
  int32_t reserved0;
  double slo_latency;             /* seconds; a query meets its SLO if latency <= slo */
  int64_t flops_per_query;        /* algorithmic FLOPs of one query (credited at completion) */
  /* Per-query data (optional; all null/0 = timestamps only).  Pinned host
   * slots of io_slots queries: query k of the tenant (arrival order) reads its
   * input from host_input slot k % io_slots (one query's rows of layer 0's x)
   * and gets its result in host_output slot k % io_slots (its rows of the last
   * layer's y).  Each dispatch copies its queries' inputs in before the round
   * and their results out after it, so a query's latency includes both. */
  const void* host_input;
  void* host_output;
  int32_t io_slots;
  int32_t reserved1;
} gm_serve_tenant;

typedef struct gm_serve_config {
  double duration;   /* seconds of real time (arrivals stop at the end) */
  double warmup;     /* seconds excluded from the statistics */
  double max_wait;   /* batcher age trigger in seconds; < 0 = the ctx policy's max_wait */
  uint64_t seed;     /* Poisson streams: per tenant, hashed from the seed */
  int32_t depth;     /* rounds in flight (1 = the reference's single dispatch in flight) */
  int32_t prewarm;   /* > 0: plan + upload every formable member set before the clock starts
                        (fails if there are more than this many); 0 = plan on first use */
  uint64_t stream;   /* cudaStream_t */
  /* inject_degradation (sim.cpp:60-68, 98-110): from degrade_start seconds on,
   * tenant degrade_tenant's observed completions stretch by degrade_slowdown
   * (a tenant-local post-dispatch delay; the device is not held).  Off when
   * degrade_slowdown == 0 or degrade_tenant < 0. */
  int32_t degrade_tenant;
  int32_t reserved1;
  double degrade_slowdown;
  double degrade_start;
  /* Member-set plan cache: > 0 bounds it (least recently used sets not in
   * flight are dropped; single-tenant sets stay).  async_plan: a set seen for
   * the first time is planned and uploaded on a worker thread while its
   * dispatch runs as back-to-back round programs of cached sub-sets, largest
   * first (single-tenant sets always exist; no dispatch waits on planning).  With more formable sets than `prewarm`, the pre-warm covers
   * the single-tenant sets and the full set only. */
  int32_t plan_cache_cap;
  int32_t async_plan;
} gm_serve_config;

typedef struct gm_serve_stats {
  int64_t queries;             /* completed inside (warmup, duration] */
  int64_t rounds;              /* dispatches (round-program launches) */
  int64_t dispatched_queries;
  double window_s, tflops, qps;
  double p50_ms, p99_ms, max_ms, mean_ms;  /* query latency: completion - arrival, nearest rank */
  double slo_violation_frac;
  double mean_queries_per_round, mean_round_ms;
  int64_t plan_hits, plan_misses;          /* member-set plan / device-table cache */
  int32_t evicted, reserved0;
  uint64_t evicted_mask;                   /* bit i: logical tenant i was evicted (i < 64) */
  int64_t plan_evictions;                  /* member sets dropped from the bounded cache */
  int64_t plan_fallbacks;                  /* dispatches run as single-tenant rounds (set being prepared) */
  int64_t plans_cached;                    /* member sets cached at the end */
  int64_t h2d_bytes, d2h_bytes;            /* per-query I/O moved inside the serving loop */
  int64_t plan_padded;                     /* fallbacks run as a cached superset (padded batches / tenants) */
} gm_serve_stats;

int gm_serve(gm_ctx* ctx, const gm_serve_tenant* tenants, size_t n, const gm_serve_config* cfg,
             gm_serve_stats* out, double* latencies_ms, size_t cap, size_t* n_lat);

/* One dispatch of the last gm_serve on this ctx: the real-clock counterpart
 * of the reference's DispatchEvent / NDJSON trace line (sim.hpp Trace,
 * gpumux.cpp:64-79).  Times are from the serving clock's start. */
typedef struct gm_dispatch_event {
  int64_t start_ns;   /* host dispatch */
  int64_t end_ns;     /* host-observed completion (CUDA event) */
  double device_ms;   /* round-program device time (CUDA events) */
  double flops;       /* the dispatched queries' FLOPs */
  int32_t queries;    /* member queries */
  int32_t tenants;    /* distinct tenants in the round */
  int32_t launches;   /* 1: one round-program launch */
  int32_t tiles;      /* tile-table entries executed */
} gm_dispatch_event;

/* Copies the last gm_serve's dispatch events (n = count; out == NULL queries
 * the count only).  GM_EINVAL when cap < count. */
int gm_serve_trace(gm_ctx* ctx, gm_dispatch_event* out, size_t cap, size_t* n);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif  /* GPUMUX_B200_H */
