"""Python mirror of the reference's space-time scheduler API.

Names, argument meaning and error behaviour follow
``proj/include/gpumux/{gemm,vtime,device,cost_model,scheduler}.hpp`` so code
and tests written against the reference read the same here; every call goes
through the C-ABI (``include/gpumux_b200.h``).  ``std::invalid_argument``
surfaces as ``ValueError`` with the reference's exact message.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field, fields
from typing import Iterable, List, Optional, Sequence

from . import _native as N
from ._native import check, lib


# ---------------------------------------------------------------- L0 types

@dataclass(frozen=True, order=True)
class GemmShape:
    """gemm.hpp:11-20; ordering is lexicographic (m, n, k) like operator<=>."""
    m: int = 1
    n: int = 1
    k: int = 1

    def valid(self) -> bool:
        return self.m >= 1 and self.n >= 1 and self.k >= 1

    def _c(self) -> N.gm_gemm_shape:
        return N.gm_gemm_shape(self.m, self.n, self.k)

    @staticmethod
    def _from(c: N.gm_gemm_shape) -> "GemmShape":
        return GemmShape(int(c.m), int(c.n), int(c.k))


@dataclass(frozen=True)
class ConvSpec:
    """gemm.hpp:23-31."""
    image_h: int = 1
    image_w: int = 1
    kernel_h: int = 1
    kernel_w: int = 1
    in_channels: int = 1
    out_channels: int = 1
    stride: int = 1
    padding: int = 0

    def _c(self) -> N.gm_conv_spec:
        return N.gm_conv_spec(*(getattr(self, f.name) for f in fields(self)))


def gemm_flops(s: GemmShape) -> int:
    return int(lib().gm_gemm_flops(C.byref(s._c())))


def gemm_bytes(s: GemmShape, element_size: int = 4) -> int:
    return int(lib().gm_gemm_bytes(C.byref(s._c()), element_size))


def im2col_gemm_dims(c: ConvSpec) -> GemmShape:
    out = N.gm_gemm_shape()
    check(lib().gm_im2col_gemm_dims(C.byref(c._c()), C.byref(out)))
    return GemmShape._from(out)


def batch_inputs(s: GemmShape, batch: int) -> GemmShape:
    out = N.gm_gemm_shape()
    lib().gm_batch_inputs(C.byref(s._c()), batch, C.byref(out))
    return GemmShape._from(out)


def shape_key(s: GemmShape) -> str:
    buf = C.create_string_buffer(96)
    check(lib().gm_shape_key(C.byref(s._c()), buf, len(buf)))
    return buf.value.decode()


def to_ns(seconds: float) -> int:
    return int(lib().gm_to_ns(float(seconds)))


def to_seconds(ns: int) -> float:
    return float(lib().gm_to_seconds(int(ns)))


# ---------------------------------------------------------------- device

@dataclass
class DeviceSpec:
    """device.hpp:13-30 (defaults are the struct's in-class defaults)."""
    peak_flops: float = 14e12
    mem_bandwidth: float = 900e9
    sm_count: int = 80
    blocks_per_sm: int = 2
    launch_overhead: float = 5e-6
    context_switch_overhead: float = 1e-3
    planning_overhead: float = 50e-6
    mem_capacity: float = 16e9
    process_context_bytes: float = 800e6
    tile_m: int = 64
    tile_n: int = 64
    space_sched_penalty: float = 1.5
    launch_serialization: float = 0.5
    # b200 extension (0 = the reference's roofline): latency floor per wave
    tile_latency: float = 0.0
    kblock_latency: float = 0.0

    def slot_total(self) -> int:
        return self.sm_count * self.blocks_per_sm

    def validate(self) -> None:
        check(lib().gm_device_spec_validate(C.byref(self._c())))

    def _c(self) -> N.gm_device_spec:
        return N.gm_device_spec(*(getattr(self, f.name) for f in fields(self)))

    @staticmethod
    def _from(c: N.gm_device_spec) -> "DeviceSpec":
        return DeviceSpec(*(getattr(c, f.name) for f in fields(DeviceSpec)))

    def as_dict(self) -> dict:
        return {f.name: getattr(self, f.name) for f in fields(self)}


def v100_profile() -> DeviceSpec:
    c = N.gm_device_spec()
    lib().gm_device_spec_v100(C.byref(c))
    return DeviceSpec._from(c)


def b200_profile() -> DeviceSpec:
    c = N.gm_device_spec()
    lib().gm_device_spec_b200(C.byref(c))
    return DeviceSpec._from(c)


def b200_calibrated_profile(path: Optional[str] = None) -> DeviceSpec:
    """The b200 profile with measured physical peaks and the latency floor
    (launch_overhead, tile_latency, kblock_latency) fitted to measured
    super-kernel times (tools/calibrate_b200.py writes
    profiles/b200_calibrated.json).  Falls back to the
    nominal profile when no calibration exists.  Tile shape and slot count are
    the kernel's, so the member sets of a plan stay those of b200_profile()."""
    import json
    import os
    path = path or os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                                "b200_calibrated.json")
    spec = b200_profile()
    if os.path.exists(path):
        with open(path) as f:
            for k, v in json.load(f)["fitted"].items():
                setattr(spec, k, v)
    return spec


# ---------------------------------------------------------------- cost model

@dataclass
class KernelCost:
    """cost_model.hpp:14-20."""
    flops: int = 0
    bytes: int = 0
    blocks: int = 0
    duration: float = 0.0
    waves: int = 0

    @staticmethod
    def _from(c: N.gm_kernel_cost) -> "KernelCost":
        return KernelCost(int(c.flops), int(c.bytes), int(c.blocks), float(c.duration), int(c.waves))


@dataclass
class KernelGroup:
    shape: GemmShape
    count: int = 1


def thread_blocks(shape: GemmShape, device: DeviceSpec) -> int:
    return int(lib().gm_thread_blocks(C.byref(shape._c()), C.byref(device._c())))


def dispatch_duration(kernels, device: DeviceSpec, slot_budget: int, launches: int) -> KernelCost:
    """cost_model.cpp:18-46; ``kernels`` is a GemmShape or a list of KernelGroup."""
    if isinstance(kernels, GemmShape):
        kernels = [KernelGroup(kernels, 1)]
    arr = (N.gm_kernel_group * max(1, len(kernels)))()
    for i, g in enumerate(kernels):
        arr[i] = N.gm_kernel_group(g.shape._c(), g.count)
    out = N.gm_kernel_cost()
    check(lib().gm_dispatch_duration(arr, len(kernels), C.byref(device._c()), slot_budget, launches, C.byref(out)))
    return KernelCost._from(out)


# ---------------------------------------------------------------- scheduler

@dataclass
class KernelRequest:
    """scheduler.hpp:17-25 (+ ``batch``, a B200 extension the planner ignores)."""
    request_id: int = 0
    tenant_index: int = 0
    shape: GemmShape = field(default_factory=GemmShape)
    enqueue_time: int = 0
    slo_deadline: int = 0
    layer_index: int = 0
    pass_index: int = 0
    batch: int = 1

    def _c(self) -> N.gm_kernel_request:
        return N.gm_kernel_request(self.request_id, self.tenant_index, self.layer_index, self.shape._c(),
                                   self.enqueue_time, self.slo_deadline, self.pass_index, self.batch)

    @staticmethod
    def _from(c: N.gm_kernel_request) -> "KernelRequest":
        return KernelRequest(int(c.request_id), int(c.tenant_index), GemmShape._from(c.shape), int(c.enqueue_time),
                             int(c.slo_deadline), int(c.layer_index), int(c.pass_index), int(c.batch))


@dataclass
class BatchPolicy:
    """scheduler.hpp:28-34."""
    max_wait: float = 2e-3
    target_batch: int = 1
    allow_variable_size: bool = False
    slo_safety_margin: float = 0.0
    variable_inefficiency: float = 1.10
    max_waves: int = 1  # B200 extension; 1 = the reference's one-wave cap (plan parity)

    def _c(self) -> N.gm_batch_policy:
        return N.gm_batch_policy(self.max_wait, self.target_batch, int(bool(self.allow_variable_size)),
                                 int(self.max_waves), self.slo_safety_margin, self.variable_inefficiency)


@dataclass
class SuperKernel:
    """scheduler.hpp:37-42 plus the handle needed to dispatch it on a GPU."""
    shape_signature: str
    members: List[KernelRequest]
    uniform: bool
    planned_cost: KernelCost
    _plans: Optional["_Plans"] = field(default=None, repr=False, compare=False)
    _index: int = field(default=-1, repr=False, compare=False)

    def tile_table(self, device: DeviceSpec):
        """Per-CTA tile-dispatch table: list of (member, m_tile, n_tile)."""
        n = C.c_size_t()
        dev = device._c()
        # first call sizes the table (GM_ERANGE with *n set), second fills it
        status = lib().gm_build_tile_table(self._plans.handle, self._index, C.byref(dev), None, 0, C.byref(n))
        if status not in (N.GM_OK, N.GM_ERANGE):
            check(status)
        arr = (N.gm_tile * max(1, n.value))()
        check(lib().gm_build_tile_table(self._plans.handle, self._index, C.byref(dev), arr, n.value, C.byref(n)))
        return [(int(t.member), int(t.m_tile), int(t.n_tile)) for t in arr[: n.value]]


class _Plans:
    """Owns a gm_plans handle (the formed super-kernels of one call)."""

    def __init__(self, handle: int):
        self.handle = handle

    def __del__(self):
        if self.handle:
            try:  # (at interpreter exit the module globals may already be gone)
                lib().gm_plans_destroy(self.handle)
            except Exception:
                pass
            self.handle = None


class RequestQueue:
    """scheduler.hpp:59-80 — shape-grouped FIFO."""

    def __init__(self, _borrowed: Optional[int] = None):
        if _borrowed is not None:
            self.handle, self._owned = _borrowed, False
        else:
            h = C.c_void_p()
            check(lib().gm_queue_create(C.byref(h)))
            self.handle, self._owned = h.value, True

    def __del__(self):
        if getattr(self, "_owned", False) and self.handle:
            try:  # (at interpreter exit the module globals may already be gone)
                lib().gm_queue_destroy(self.handle)
            except Exception:
                pass
            self.handle = None

    def enqueue(self, request: KernelRequest) -> None:
        check(lib().gm_queue_enqueue(self.handle, C.byref(request._c())))

    def size(self) -> int:
        return int(lib().gm_queue_size(self.handle))

    def empty(self) -> bool:
        return self.size() == 0

    def _snapshot(self) -> List[KernelRequest]:
        n = C.c_size_t(self.size())
        arr = (N.gm_kernel_request * max(1, n.value))()
        check(lib().gm_queue_snapshot(self.handle, arr, n.value, C.byref(n)))
        return [KernelRequest._from(arr[i]) for i in range(n.value)]

    def groups(self) -> dict:
        """{GemmShape: [KernelRequest...]} in ascending shape order, FIFO within."""
        out: dict = {}
        for r in self._snapshot():
            out.setdefault(r.shape, []).append(r)
        return out

    def cancel_tenant(self, tenant_index: int) -> List[KernelRequest]:
        n = C.c_size_t(self.size())
        arr = (N.gm_kernel_request * max(1, n.value))()
        check(lib().gm_queue_cancel_tenant(self.handle, tenant_index, arr, n.value, C.byref(n)))
        return [KernelRequest._from(arr[i]) for i in range(n.value)]


def _unpack_plans(handle: int, plans: Optional[_Plans] = None) -> List[SuperKernel]:
    plans = plans or _Plans(handle)
    out = []
    for i in range(int(lib().gm_plans_count(handle))):
        info = N.gm_plan_info()
        check(lib().gm_plans_get(handle, i, C.byref(info)))
        n = C.c_size_t(int(info.n_members))
        arr = (N.gm_kernel_request * max(1, n.value))()
        check(lib().gm_plans_members(handle, i, arr, n.value, C.byref(n)))
        out.append(SuperKernel(info.signature.decode(), [KernelRequest._from(arr[j]) for j in range(n.value)],
                               bool(info.uniform), KernelCost._from(info.planned_cost), plans, i))
    return out


def form_batches(queue: RequestQueue, now: int, policy: BatchPolicy, device: DeviceSpec) -> List[SuperKernel]:
    """scheduler.cpp:96-199 (mutates ``queue``)."""
    h = C.c_void_p()
    check(lib().gm_form_batches(queue.handle, int(now), C.byref(policy._c()), C.byref(device._c()), C.byref(h)))
    return _unpack_plans(h.value)


def plan_super_kernel(members: Sequence[KernelRequest], uniform: bool, policy: BatchPolicy,
                      device: DeviceSpec) -> KernelCost:
    arr = (N.gm_kernel_request * max(1, len(members)))(*[m._c() for m in members])
    out = N.gm_kernel_cost()
    check(lib().gm_plan_super_kernel(arr, len(members), int(bool(uniform)), C.byref(policy._c()),
                                     C.byref(device._c()), C.byref(out)))
    return KernelCost._from(out)


def slo_headroom(request: KernelRequest, now: int, predicted_duration: float, policy: BatchPolicy) -> float:
    return float(lib().gm_slo_headroom(C.byref(request._c()), int(now), float(predicted_duration),
                                       C.byref(policy._c())))


class SuperKernelCache:
    """scheduler.hpp:52-56."""

    def __init__(self, _borrowed: Optional[int] = None):
        if _borrowed is not None:
            self.handle, self._owned = _borrowed, False
        else:
            h = C.c_void_p()
            check(lib().gm_cache_create(C.byref(h)))
            self.handle, self._owned = h.value, True

    def __del__(self):
        if getattr(self, "_owned", False) and self.handle:
            try:  # (at interpreter exit the module globals may already be gone)
                lib().gm_cache_destroy(self.handle)
            except Exception:
                pass
            self.handle = None

    def _stats(self):
        h, m, e = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib().gm_cache_stats(self.handle, C.byref(h), C.byref(m), C.byref(e)))
        return int(h.value), int(m.value), int(e.value)

    @property
    def hits(self) -> int:
        return self._stats()[0]

    @property
    def misses(self) -> int:
        return self._stats()[1]

    @property
    def entries(self) -> int:
        return self._stats()[2]


def dispatch_cost(sk: SuperKernel, cache: SuperKernelCache, device: DeviceSpec) -> float:
    """scheduler.cpp:201-212."""
    d, hit = C.c_double(), C.c_int()
    check(lib().gm_dispatch_cost(sk._plans.handle, sk._index, cache.handle, C.byref(device._c()), C.byref(d),
                                 C.byref(hit)))
    return float(d.value)


# ---------------------------------------------------------------- monitor

@dataclass
class TenantHealth:
    """scheduler.hpp:44-50."""
    tenant_index: int = 0
    ewma_latency: float = 0.0
    ewma_alpha: float = 0.2
    observed_count: int = 0
    evicted: bool = False

    def _c(self) -> N.gm_tenant_health:
        return N.gm_tenant_health(self.tenant_index, int(self.evicted), self.ewma_latency, self.ewma_alpha,
                                  self.observed_count)

    def _load(self, c: N.gm_tenant_health) -> None:
        self.tenant_index, self.evicted = int(c.tenant_index), bool(c.evicted)
        self.ewma_latency, self.ewma_alpha = float(c.ewma_latency), float(c.ewma_alpha)
        self.observed_count = int(c.observed_count)


def record_latency(health: TenantHealth, observed_seconds: float) -> None:
    c = health._c()
    check(lib().gm_record_latency(C.byref(c), float(observed_seconds)))
    health._load(c)


def _health_array(healths: Sequence[TenantHealth]):
    arr = (N.gm_tenant_health * max(1, len(healths)))()
    for i, h in enumerate(healths):
        arr[i] = h._c()
    return arr


def detect_stragglers(healths: Sequence[TenantHealth], threshold_ratio: float, min_observations: int) -> List[int]:
    arr = _health_array(healths)
    out = (C.c_int32 * max(1, len(healths)))()
    n = C.c_size_t()
    check(lib().gm_detect_stragglers(arr, len(healths), float(threshold_ratio), int(min_observations), out,
                                     len(healths), C.byref(n)))
    return [int(out[i]) for i in range(n.value)]


def evict(healths: List[TenantHealth], queue: RequestQueue, tenant_index: int) -> List[KernelRequest]:
    arr = _health_array(healths)
    cap = queue.size()
    out = (N.gm_kernel_request * max(1, cap))()
    n = C.c_size_t()
    check(lib().gm_evict(arr, len(healths), queue.handle, int(tenant_index), out, cap, C.byref(n)))
    for i, h in enumerate(healths):
        h._load(arr[i])
    return [KernelRequest._from(out[i]) for i in range(n.value)]


# ---------------------------------------------------------------- metrics

def percentile_nearest_rank(values: Iterable[float], pct: float) -> float:
    v = list(values)
    arr = (C.c_double * max(1, len(v)))(*v)
    out = C.c_double()
    check(lib().gm_percentile_nearest_rank(arr, len(v), float(pct), C.byref(out)))
    return float(out.value)


def geomean(values: Iterable[float]) -> float:
    v = list(values)
    arr = (C.c_double * max(1, len(v)))(*v)
    out = C.c_double()
    check(lib().gm_geomean(arr, len(v), C.byref(out)))
    return float(out.value)
