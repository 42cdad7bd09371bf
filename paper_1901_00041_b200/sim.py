"""Virtual-clock space-time driver (run_space_time, proj/src/sim.cpp:398-581).

``simulate_space_time`` returns the reference engine's dispatch sequence for a
closed-loop homogeneous tenant set; the B200 engine replays that plan stream
on the GPU (engine.py).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

from . import _native as N
from ._native import check, lib
from .scheduler import BatchPolicy, DeviceSpec, GemmShape


@dataclass
class DetectorParams:
    """sim.hpp:32-37."""
    ewma_alpha: float = 0.2
    min_observations: int = 10
    threshold_ratio: float = 1.5
    evict_stragglers: bool = True

    def _c(self) -> N.gm_detector:
        return N.gm_detector(self.ewma_alpha, self.min_observations, self.threshold_ratio,
                             int(bool(self.evict_stragglers)), 0)


@dataclass
class DegradationSpec:
    """sim.hpp:41-45."""
    tenant_index: int = 0
    slowdown: float = 1.0
    start: float = 0.0


@dataclass
class SpaceTimeConfig:
    device: DeviceSpec
    layers: Sequence[GemmShape]
    tenants: int
    scheduler: BatchPolicy = field(default_factory=lambda: BatchPolicy(target_batch=0))
    detector: DetectorParams = field(default_factory=DetectorParams)
    concurrency: int = 1
    slo_latency: float = 0.1
    duration: float = 1.0
    warmup: Optional[float] = None
    microbench: bool = False
    degradation: Optional[DegradationSpec] = None


@dataclass
class DispatchEvent:
    start: int
    end: int
    flops: int
    occupancy: float
    member_requests: List[int]


@dataclass
class RequestLifecycle:
    request_id: int
    tenant_index: int
    enqueue_time: int
    dispatch_time: int
    complete_time: int
    slo_met: bool
    flops: int


@dataclass
class Trace:
    events: List[DispatchEvent]
    completions: List[RequestLifecycle]
    cancellations: int
    evicted_tenants: List[int]
    eviction_times: List[int]
    cache_hits: int
    cache_misses: int
    dispatched_flops: int
    completed_kernel_flops: int


def simulate_space_time(cfg: SpaceTimeConfig) -> Trace:
    layers = (N.gm_gemm_shape * len(cfg.layers))(*[s._c() for s in cfg.layers])
    c = N.gm_sim_config()
    c.device = cfg.device._c()
    c.scheduler = cfg.scheduler._c()
    c.detector = cfg.detector._c()
    c.layers = layers
    c.n_layers = len(cfg.layers)
    c.n_tenants = cfg.tenants
    c.concurrency = cfg.concurrency
    c.slo_latency = cfg.slo_latency
    c.duration = cfg.duration
    c.warmup = 0.1 * cfg.duration if cfg.warmup is None else cfg.warmup
    c.microbench = int(cfg.microbench)
    deg = cfg.degradation
    c.degrade_tenant = -1 if deg is None else deg.tenant_index
    c.degrade_slowdown = 1.0 if deg is None else deg.slowdown
    c.degrade_start = 0.0 if deg is None else deg.start
    h = C.c_void_p()
    check(lib().gm_simulate_space_time(C.byref(c), C.byref(h)))
    try:
        ne, nm, nc, nx = C.c_size_t(), C.c_size_t(), C.c_size_t(), C.c_size_t()
        hits, misses = C.c_int64(), C.c_int64()
        check(lib().gm_sim_trace_counts(h, C.byref(ne), C.byref(nm), C.byref(nc), C.byref(nx), C.byref(hits),
                                        C.byref(misses)))
        ev = (N.gm_sim_event * max(1, ne.value))()
        ids = (C.c_uint64 * max(1, nm.value))()
        check(lib().gm_sim_trace_events(h, ev, ne.value, ids, nm.value))
        comps = (N.gm_sim_completion * max(1, nc.value))()
        check(lib().gm_sim_trace_completions(h, comps, nc.value))
        n_ev = C.c_size_t()
        ten = (C.c_int32 * max(1, cfg.tenants))()
        tim = (C.c_int64 * max(1, cfg.tenants))()
        check(lib().gm_sim_trace_evictions(h, ten, tim, cfg.tenants, C.byref(n_ev)))
        disp, comp = C.c_int64(), C.c_int64()
        check(lib().gm_sim_trace_flops(h, C.byref(disp), C.byref(comp)))
        events = [DispatchEvent(int(e.start), int(e.end), int(e.flops), float(e.occupancy),
                                [int(x) for x in ids[e.member_offset:e.member_offset + e.n_members]])
                  for e in ev[: ne.value]]
        completions = [RequestLifecycle(int(x.request_id), int(x.tenant_index), int(x.enqueue_time),
                                        int(x.dispatch_time), int(x.complete_time), bool(x.slo_met), int(x.flops))
                       for x in comps[: nc.value]]
        return Trace(events, completions, int(nx.value), [int(t) for t in ten[: n_ev.value]],
                     [int(t) for t in tim[: n_ev.value]], int(hits.value), int(misses.value), int(disp.value),
                     int(comp.value))
    finally:
        lib().gm_sim_trace_destroy(h)


@dataclass
class RoundDispatch:
    """One dispatch of a planned round: the formed super-kernel and its
    virtual [start, end)."""
    kernel: object  # scheduler.SuperKernel
    start: int
    end: int


def plan_round_shapes(tenants: Sequence[tuple], start: int, policy: BatchPolicy, device: DeviceSpec,
                      cache=None) -> List[RoundDispatch]:
    """gm_plan_round_shapes: one closed-loop round on the virtual clock, host
    only.  ``tenants`` = [(tenant_index, [GemmShape, ...], slo_seconds), ...].
    The run_space_time loop of proj/src/sim.cpp:452-576 for one pass per
    tenant; heterogeneous layer lists are allowed (B200 extension)."""
    from .scheduler import _Plans, _unpack_plans
    keep = []
    arr = (N.gm_round_tenant * max(1, len(tenants)))()
    for i, (t, layers, slo) in enumerate(tenants):
        ls = (N.gm_gemm_shape * max(1, len(layers)))(*[N.gm_gemm_shape(s.m, s.n, s.k) for s in layers])
        keep.append(ls)
        arr[i] = N.gm_round_tenant(int(t), 0, ls, len(layers), int(lib().gm_to_ns(float(slo))))
    h = C.c_void_p()
    check(lib().gm_plan_round_shapes(arr, len(tenants), int(start), C.byref(policy._c()), C.byref(device._c()),
                                     cache.handle if cache is not None else None, None, C.byref(h)))
    owner = _Plans(h.value)
    kernels = _unpack_plans(h.value, owner)
    out = []
    for i, k in enumerate(kernels):
        s_, e_ = C.c_int64(), C.c_int64()
        check(lib().gm_plans_times(h.value, i, C.byref(s_), C.byref(e_)))
        out.append(RoundDispatch(k, int(s_.value), int(e_.value)))
    return out
