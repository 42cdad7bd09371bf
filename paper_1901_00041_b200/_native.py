"""ctypes view of the C-ABI in include/gpumux_b200.h.

The shared library is built in-tree (``paper_1901_00041_b200/_lib``) by
``__graft_entry__.build()``.  Loading fails loudly: there is no Python
fallback for anything this module exposes.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GM_LIB_PATH") or os.path.join(_HERE, "_lib", "libgpumux_b200.so")

GM_OK, GM_EINVAL, GM_ECONFIG, GM_EOOM, GM_EINTERNAL, GM_ECUDA, GM_ERANGE, GM_ENODEV = range(8)
GM_LAYER_GEMM, GM_LAYER_CONV, GM_LAYER_DWCONV, GM_LAYER_MAXPOOL, GM_LAYER_AVGPOOL = 0, 1, 2, 3, 4
GM_ACT_NONE, GM_ACT_RELU, GM_ACT_RELU6, GM_ACT_GELU = 0, 1, 2, 3
GM_MODE_PACKED, GM_MODE_TIME_ONLY, GM_MODE_SPACE_ONLY = 0, 1, 2


class gm_gemm_shape(C.Structure):
    _fields_ = [("m", C.c_int64), ("n", C.c_int64), ("k", C.c_int64)]


class gm_conv_spec(C.Structure):
    _fields_ = [(f, C.c_int64) for f in ("image_h", "image_w", "kernel_h", "kernel_w", "in_channels",
                                          "out_channels", "stride", "padding")]


class gm_device_spec(C.Structure):
    _fields_ = [
        ("peak_flops", C.c_double), ("mem_bandwidth", C.c_double), ("sm_count", C.c_int64),
        ("blocks_per_sm", C.c_int64), ("launch_overhead", C.c_double), ("context_switch_overhead", C.c_double),
        ("planning_overhead", C.c_double), ("mem_capacity", C.c_double), ("process_context_bytes", C.c_double),
        ("tile_m", C.c_int64), ("tile_n", C.c_int64), ("space_sched_penalty", C.c_double),
        ("launch_serialization", C.c_double), ("tile_latency", C.c_double), ("kblock_latency", C.c_double),
    ]


class gm_kernel_cost(C.Structure):
    _fields_ = [("flops", C.c_int64), ("bytes", C.c_int64), ("blocks", C.c_int64), ("duration", C.c_double),
                ("waves", C.c_int64)]


class gm_kernel_group(C.Structure):
    _fields_ = [("shape", gm_gemm_shape), ("count", C.c_int64)]


class gm_kernel_request(C.Structure):
    _fields_ = [("request_id", C.c_uint64), ("tenant_index", C.c_int32), ("layer_index", C.c_int32),
                ("shape", gm_gemm_shape), ("enqueue_time", C.c_int64), ("slo_deadline", C.c_int64),
                ("pass_index", C.c_uint32), ("batch", C.c_uint32)]


class gm_round_tenant(C.Structure):
    _fields_ = [("tenant", C.c_int32), ("reserved", C.c_int32), ("layers", C.POINTER(gm_gemm_shape)),
                ("n_layers", C.c_size_t), ("slo_ns", C.c_int64)]


class gm_round_tile(C.Structure):
    _fields_ = [(f, C.c_int32) for f in ("tenant", "layer", "m_tile", "n_tile", "rows", "cols", "splits",
                                          "kb_begin", "kb_end", "done", "dep", "dep_n", "rdep", "rdep_n", "plan",
                                          "cuda_core")]


class gm_batch_policy(C.Structure):
    _fields_ = [("max_wait", C.c_double), ("target_batch", C.c_int64), ("allow_variable_size", C.c_int32),
                ("max_waves", C.c_int32), ("slo_safety_margin", C.c_double), ("variable_inefficiency", C.c_double)]


class gm_tenant_health(C.Structure):
    _fields_ = [("tenant_index", C.c_int32), ("evicted", C.c_int32), ("ewma_latency", C.c_double),
                ("ewma_alpha", C.c_double), ("observed_count", C.c_int64)]


class gm_detector(C.Structure):
    _fields_ = [("ewma_alpha", C.c_double), ("min_observations", C.c_int64), ("threshold_ratio", C.c_double),
                ("evict_stragglers", C.c_int32), ("reserved0", C.c_int32)]


class gm_tile(C.Structure):
    _fields_ = [("member", C.c_uint16), ("flags", C.c_uint16), ("m_tile", C.c_uint16), ("n_tile", C.c_uint16)]


class gm_plan_info(C.Structure):
    _fields_ = [("uniform", C.c_int32), ("reserved0", C.c_int32), ("n_members", C.c_int64),
                ("planned_cost", gm_kernel_cost), ("signature", C.c_char_p)]


class gm_sim_config(C.Structure):
    _fields_ = [("device", gm_device_spec), ("scheduler", gm_batch_policy), ("detector", gm_detector),
                ("layers", C.POINTER(gm_gemm_shape)), ("n_layers", C.c_size_t), ("n_tenants", C.c_int32),
                ("concurrency", C.c_int32), ("slo_latency", C.c_double), ("duration", C.c_double),
                ("warmup", C.c_double), ("microbench", C.c_int32), ("degrade_tenant", C.c_int32),
                ("degrade_slowdown", C.c_double), ("degrade_start", C.c_double)]


class gm_sim_event(C.Structure):
    _fields_ = [("start", C.c_int64), ("end", C.c_int64), ("flops", C.c_int64), ("occupancy", C.c_double),
                ("member_offset", C.c_int64), ("n_members", C.c_int64)]


class gm_sim_completion(C.Structure):
    _fields_ = [("request_id", C.c_uint64), ("tenant_index", C.c_int32), ("slo_met", C.c_int32),
                ("enqueue_time", C.c_int64), ("dispatch_time", C.c_int64), ("complete_time", C.c_int64),
                ("flops", C.c_int64)]


class gm_layer_desc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("batch", C.c_int32), ("conv", gm_conv_spec), ("gemm", gm_gemm_shape),
                ("x", C.c_void_p), ("w", C.c_void_p), ("y", C.c_void_p), ("ldx", C.c_int64), ("ldw", C.c_int64),
                ("act", C.c_int32), ("src", C.c_int32), ("res", C.c_void_p), ("ldr", C.c_int64),
                ("res_src", C.c_int32), ("reserved0", C.c_int32)]


class gm_tenant_desc(C.Structure):
    _fields_ = [("tenant_id", C.c_char_p), ("layers", C.POINTER(gm_layer_desc)), ("n_layers", C.c_size_t),
                ("slo_latency", C.c_double), ("concurrency", C.c_int32), ("reserved0", C.c_int32)]


P = C.POINTER
class gm_serve_tenant(C.Structure):
    _fields_ = [("n_variants", C.c_int32), ("variant_tenant", C.POINTER(C.c_int32)),
                ("variant_batch", C.POINTER(C.c_int32)), ("rate_qps", C.c_double), ("concurrency", C.c_int32),
                ("reserved0", C.c_int32), ("slo_latency", C.c_double), ("flops_per_query", C.c_int64),
                ("host_input", C.c_void_p), ("host_output", C.c_void_p), ("io_slots", C.c_int32),
                ("reserved1", C.c_int32)]


class gm_serve_config(C.Structure):
    _fields_ = [("duration", C.c_double), ("warmup", C.c_double), ("max_wait", C.c_double), ("seed", C.c_uint64),
                ("depth", C.c_int32), ("prewarm", C.c_int32), ("stream", C.c_uint64),
                ("degrade_tenant", C.c_int32), ("reserved1", C.c_int32), ("degrade_slowdown", C.c_double),
                ("degrade_start", C.c_double), ("plan_cache_cap", C.c_int32), ("async_plan", C.c_int32)]


class gm_serve_stats(C.Structure):
    _fields_ = [("queries", C.c_int64), ("rounds", C.c_int64), ("dispatched_queries", C.c_int64),
                ("window_s", C.c_double), ("tflops", C.c_double), ("qps", C.c_double), ("p50_ms", C.c_double),
                ("p99_ms", C.c_double), ("max_ms", C.c_double), ("mean_ms", C.c_double),
                ("slo_violation_frac", C.c_double), ("mean_queries_per_round", C.c_double),
                ("mean_round_ms", C.c_double), ("plan_hits", C.c_int64), ("plan_misses", C.c_int64),
                ("evicted", C.c_int32), ("reserved0", C.c_int32), ("evicted_mask", C.c_uint64),
                ("plan_evictions", C.c_int64), ("plan_fallbacks", C.c_int64), ("plans_cached", C.c_int64),
                ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64), ("plan_padded", C.c_int64)]


class gm_request_io(C.Structure):
    _fields_ = [("x", C.c_void_p), ("x_bytes", C.c_size_t), ("y", C.c_void_p), ("y_bytes", C.c_size_t)]


class gm_completion(C.Structure):
    _fields_ = [("request_id", C.c_uint64), ("tenant_index", C.c_int32), ("layer_index", C.c_int32),
                ("pass_index", C.c_uint32), ("batch", C.c_uint32), ("enqueue_time", C.c_int64),
                ("slo_deadline", C.c_int64), ("dispatch_ns", C.c_int64), ("complete_ns", C.c_int64),
                ("exec_seconds", C.c_double), ("plan_members", C.c_int32), ("reserved0", C.c_int32)]


class gm_dispatch_event(C.Structure):
    _fields_ = [("start_ns", C.c_int64), ("end_ns", C.c_int64), ("device_ms", C.c_double), ("flops", C.c_double),
                ("queries", C.c_int32), ("tenants", C.c_int32), ("launches", C.c_int32), ("tiles", C.c_int32)]


_SIGS = {
    "gm_last_error": (C.c_char_p, [C.c_void_p]),
    "gm_abi_version": (C.c_int, []),
    "gm_device_spec_default": (None, [P(gm_device_spec)]),
    "gm_device_spec_v100": (None, [P(gm_device_spec)]),
    "gm_device_spec_b200": (None, [P(gm_device_spec)]),
    "gm_device_spec_validate": (C.c_int, [P(gm_device_spec)]),
    "gm_batch_policy_default": (None, [P(gm_batch_policy)]),
    "gm_detector_default": (None, [P(gm_detector)]),
    "gm_gemm_flops": (C.c_int64, [P(gm_gemm_shape)]),
    "gm_gemm_bytes": (C.c_int64, [P(gm_gemm_shape), C.c_int64]),
    "gm_im2col_gemm_dims": (C.c_int, [P(gm_conv_spec), P(gm_gemm_shape)]),
    "gm_batch_inputs": (None, [P(gm_gemm_shape), C.c_int64, P(gm_gemm_shape)]),
    "gm_shape_key": (C.c_int, [P(gm_gemm_shape), C.c_char_p, C.c_size_t]),
    "gm_to_ns": (C.c_int64, [C.c_double]),
    "gm_to_seconds": (C.c_double, [C.c_int64]),
    "gm_thread_blocks": (C.c_int64, [P(gm_gemm_shape), P(gm_device_spec)]),
    "gm_dispatch_duration": (C.c_int, [P(gm_kernel_group), C.c_size_t, P(gm_device_spec), C.c_int64, C.c_int64,
                                       P(gm_kernel_cost)]),
    "gm_queue_create": (C.c_int, [P(C.c_void_p)]),
    "gm_queue_destroy": (None, [C.c_void_p]),
    "gm_queue_enqueue": (C.c_int, [C.c_void_p, P(gm_kernel_request)]),
    "gm_queue_size": (C.c_int64, [C.c_void_p]),
    "gm_queue_snapshot": (C.c_int, [C.c_void_p, P(gm_kernel_request), C.c_size_t, P(C.c_size_t)]),
    "gm_queue_group_count": (C.c_int, [C.c_void_p, P(C.c_size_t)]),
    "gm_queue_cancel_tenant": (C.c_int, [C.c_void_p, C.c_int32, P(gm_kernel_request), C.c_size_t, P(C.c_size_t)]),
    "gm_form_batches": (C.c_int, [C.c_void_p, C.c_int64, P(gm_batch_policy), P(gm_device_spec), P(C.c_void_p)]),
    "gm_plans_count": (C.c_size_t, [C.c_void_p]),
    "gm_plans_get": (C.c_int, [C.c_void_p, C.c_size_t, P(gm_plan_info)]),
    "gm_plans_members": (C.c_int, [C.c_void_p, C.c_size_t, P(gm_kernel_request), C.c_size_t, P(C.c_size_t)]),
    "gm_plans_destroy": (None, [C.c_void_p]),
    "gm_plans_key": (C.c_int, [C.c_void_p, P(C.c_uint64)]),
    "gm_build_tile_table": (C.c_int, [C.c_void_p, C.c_size_t, P(gm_device_spec), P(gm_tile), C.c_size_t,
                                      P(C.c_size_t)]),
    "gm_plan_super_kernel": (C.c_int, [P(gm_kernel_request), C.c_size_t, C.c_int, P(gm_batch_policy),
                                       P(gm_device_spec), P(gm_kernel_cost)]),
    "gm_slo_headroom": (C.c_double, [P(gm_kernel_request), C.c_int64, C.c_double, P(gm_batch_policy)]),
    "gm_cache_create": (C.c_int, [P(C.c_void_p)]),
    "gm_cache_destroy": (None, [C.c_void_p]),
    "gm_dispatch_cost": (C.c_int, [C.c_void_p, C.c_size_t, C.c_void_p, P(gm_device_spec), P(C.c_double),
                                   P(C.c_int)]),
    "gm_cache_stats": (C.c_int, [C.c_void_p, P(C.c_int64), P(C.c_int64), P(C.c_int64)]),
    "gm_record_latency": (C.c_int, [P(gm_tenant_health), C.c_double]),
    "gm_detect_stragglers": (C.c_int, [P(gm_tenant_health), C.c_size_t, C.c_double, C.c_int64, P(C.c_int32),
                                       C.c_size_t, P(C.c_size_t)]),
    "gm_evict": (C.c_int, [P(gm_tenant_health), C.c_size_t, C.c_void_p, C.c_int32, P(gm_kernel_request),
                           C.c_size_t, P(C.c_size_t)]),
    "gm_percentile_nearest_rank": (C.c_int, [P(C.c_double), C.c_size_t, C.c_double, P(C.c_double)]),
    "gm_geomean": (C.c_int, [P(C.c_double), C.c_size_t, P(C.c_double)]),
    "gm_simulate_space_time": (C.c_int, [P(gm_sim_config), P(C.c_void_p)]),
    "gm_sim_trace_counts": (C.c_int, [C.c_void_p, P(C.c_size_t), P(C.c_size_t), P(C.c_size_t), P(C.c_size_t),
                                      P(C.c_int64), P(C.c_int64)]),
    "gm_sim_trace_events": (C.c_int, [C.c_void_p, P(gm_sim_event), C.c_size_t, P(C.c_uint64), C.c_size_t]),
    "gm_sim_trace_completions": (C.c_int, [C.c_void_p, P(gm_sim_completion), C.c_size_t]),
    "gm_sim_trace_evictions": (C.c_int, [C.c_void_p, P(C.c_int32), P(C.c_int64), C.c_size_t, P(C.c_size_t)]),
    "gm_sim_trace_flops": (C.c_int, [C.c_void_p, P(C.c_int64), P(C.c_int64)]),
    "gm_sim_trace_destroy": (None, [C.c_void_p]),
    "gm_create": (C.c_int, [P(gm_device_spec), P(gm_batch_policy), P(gm_detector), C.c_int, P(C.c_void_p)]),
    "gm_destroy": (None, [C.c_void_p]),
    "gm_ctx_queue": (C.c_int, [C.c_void_p, P(C.c_void_p)]),
    "gm_ctx_cache": (C.c_int, [C.c_void_p, P(C.c_void_p)]),
    "gm_ctx_device_spec": (C.c_int, [C.c_void_p, P(gm_device_spec)]),
    "gm_ctx_set_policy": (C.c_int, [C.c_void_p, P(gm_batch_policy)]),
    "gm_ctx_set_option": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int64]),
    "gm_register_tenant": (C.c_int, [C.c_void_p, P(gm_tenant_desc), P(C.c_int32)]),
    "gm_layer_shape": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, P(gm_gemm_shape)]),
    "gm_tenant_count": (C.c_int, [C.c_void_p, P(C.c_int32)]),
    "gm_migrate_tenant": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_uint64, P(C.c_int32)]),
    "gm_migrate_tenants": (C.c_int, [C.c_void_p, P(C.c_int32), C.c_size_t, C.c_void_p, C.c_uint64, P(C.c_int32)]),
    "gm_prepare": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t]),
    "gm_dispatch": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_uint64, P(C.c_double), P(C.c_int)]),
    "gm_enqueue": (C.c_int, [C.c_void_p, P(gm_kernel_request), P(gm_request_io)]),
    "gm_ctx_form_batches": (C.c_int, [C.c_void_p, C.c_int64, P(C.c_void_p)]),
    "gm_ctx_now_ns": (C.c_int64, [C.c_void_p]),
    "gm_poll_completions": (C.c_int, [C.c_void_p, P(gm_completion), C.c_size_t, P(C.c_size_t)]),
    "gm_ctx_in_flight": (C.c_int, [C.c_void_p, P(C.c_size_t)]),
    "gm_ctx_synchronize": (C.c_int, [C.c_void_p]),
    "gm_ctx_record_latency": (C.c_int, [C.c_void_p, C.c_int32, C.c_double]),
    "gm_ctx_detect_stragglers": (C.c_int, [C.c_void_p, P(C.c_int32), C.c_size_t, P(C.c_size_t)]),
    "gm_ctx_evict": (C.c_int, [C.c_void_p, C.c_int32, P(C.c_uint64), C.c_size_t, P(C.c_size_t)]),
    "gm_ctx_health": (C.c_int, [C.c_void_p, C.c_int32, P(gm_tenant_health)]),
    "gm_launch_members": (C.c_int, [C.c_void_p, P(C.c_int32), P(C.c_int32), C.c_size_t, C.c_uint64,
                                    P(C.c_int32)]),
    "gm_members_launch_count": (C.c_int, [C.c_void_p, P(C.c_int32), P(C.c_int32), C.c_size_t, P(C.c_int32)]),
    "gm_plan_round": (C.c_int, [C.c_void_p, P(C.c_int32), C.c_size_t, C.c_int64, P(C.c_void_p)]),
    "gm_plans_times": (C.c_int, [C.c_void_p, C.c_size_t, P(C.c_int64), P(C.c_int64)]),
    "gm_plan_round_shapes": (C.c_int, [P(gm_round_tenant), C.c_size_t, C.c_int64, P(gm_batch_policy),
                                       P(gm_device_spec), C.c_void_p, P(C.c_uint64), P(C.c_void_p)]),
    "gm_prepare_plans": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gm_dispatch_plans": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, P(C.c_int32)]),
    "gm_graph_capture_plans": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, P(C.c_void_p)]),
    "gm_graph_capture_serial": (C.c_int, [C.c_void_p, P(C.c_int32), C.c_size_t, C.c_int, C.c_int,
                                          P(C.c_void_p)]),
    "gm_dispatch_round": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, P(C.c_int32)]),
    "gm_graph_capture_round": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, P(C.c_void_p)]),
    "gm_trace_round": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, P(C.c_uint64), C.c_size_t, P(C.c_size_t)]),
    "gm_round_tiles": (C.c_int, [C.c_void_p, C.c_void_p, P(gm_tile), C.c_size_t, P(C.c_size_t)]),
    "gm_round_tile_info": (C.c_int, [C.c_void_p, C.c_void_p, P(gm_round_tile), C.c_size_t, P(C.c_size_t)]),
    "gm_graph_capture_round_e2e": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, P(C.c_int32), P(C.c_void_p),
                                             P(C.c_void_p), P(C.c_size_t), P(C.c_void_p), P(C.c_void_p),
                                             P(C.c_size_t), P(C.c_void_p)]),
    "gm_graph_launch": (C.c_int, [C.c_void_p, C.c_uint64]),
    "gm_graph_launch_count": (C.c_int, [C.c_void_p, P(C.c_int32), P(C.c_int32)]),
    "gm_graph_kernel_times": (C.c_int, [C.c_void_p, P(C.c_float), C.c_size_t, P(C.c_size_t)]),
    "gm_graph_destroy": (None, [C.c_void_p]),
    "gm_ctx_launch_stats": (C.c_int, [C.c_void_p, P(C.c_int64), P(C.c_int64), P(C.c_int64)]),
    "gm_serve": (C.c_int, [C.c_void_p, P(gm_serve_tenant), C.c_size_t, P(gm_serve_config), P(gm_serve_stats),
                           P(C.c_double), C.c_size_t, P(C.c_size_t)]),
    "gm_serve_trace": (C.c_int, [C.c_void_p, P(gm_dispatch_event), C.c_size_t, P(C.c_size_t)]),
}

_lib = None


class NativeError(RuntimeError):
    """A failure status from the C-ABI that has no closer Python analogue."""

    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


class CudaUnavailable(NativeError):
    pass


def lib() -> C.CDLL:
    """The loaded product library; raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() (no fallback path exists)")
        handle = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            if os.environ.get("GM_LIB_PATH") and not hasattr(handle, name):
                continue  # an older build loaded for A/B comparisons (debug)
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(status: int) -> None:
    """Map a gm_status to the Python exception of the matching reference class."""
    if status == GM_OK:
        return
    msg = lib().gm_last_error(None).decode()
    if status == GM_EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    if status == GM_ENODEV:
        raise CudaUnavailable(status, msg)
    if status == GM_EOOM:
        raise MemoryError(msg)
    raise NativeError(status, msg)
