"""Per-GPU context (gm_ctx): tenant registration and super-kernel dispatch.

Device buffers are torch tensors (PyTorch is plumbing here: allocation,
streams, graphs); all compute runs in the sm_100a kernels of
``libgpumux_b200.so``.  There is no CPU or PyTorch fallback: a missing
library or a non-sm_100 device raises.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

from . import _native as N
from ._native import check, lib
from .scheduler import (BatchPolicy, ConvSpec, DeviceSpec, GemmShape, RequestQueue, SuperKernel, SuperKernelCache,
                        TenantHealth, _Plans, _unpack_plans, b200_profile)
from .sim import DetectorParams


@dataclass
class LayerBuffers:
    """One operator of a tenant graph with its device tensors (bf16).

    conv: x NHWC [b, H, W, Cin], w [Cout, ldw] (KRSC rows), y NHWC [b, P, Q, Cout]
    dwconv: x NHWC [b, H, W, C], w [C, ldw] (R*S taps per row), y NHWC [b, P, Q, C]
    maxpool / avgpool: x NHWC [b, H, W, C], y NHWC [b, P, Q, C], w unused
    gemm: x [M, ldx], w [N, ldw], y [M, N]

    ``act`` (gm_activation; ``relu=True`` is act 1) runs after the optional
    residual add ``res`` ([M, N] rows, row stride ``res.stride(0)``).  ``src``
    / ``res_src``: the tenant's earlier layer whose output ``x`` / ``res``
    views (-1 = an external buffer).
    """
    kind: str
    x: object
    w: object
    y: object
    conv: Optional[ConvSpec] = None
    batch: int = 1
    gemm: Optional[GemmShape] = None
    relu: bool = False
    act: Optional[int] = None
    src: int = -1
    res: object = None
    res_src: int = -1

    @property
    def activation(self) -> int:
        return self.act if self.act is not None else (1 if self.relu else 0)


class Context:
    """gm_ctx: one scheduler + device runtime per GPU."""

    def __init__(self, device_index: int = 0, device: Optional[DeviceSpec] = None,
                 policy: Optional[BatchPolicy] = None, detector: Optional[DetectorParams] = None):
        self.device = device or b200_profile()
        self.policy = policy or BatchPolicy(target_batch=0)
        self.detector = detector or DetectorParams()
        h = C.c_void_p()
        check(lib().gm_create(C.byref(self.device._c()), C.byref(self.policy._c()), C.byref(self.detector._c()),
                              int(device_index), C.byref(h)))
        self.handle = h.value
        self.device_index = device_index
        self._keepalive: List[object] = []
        q, c = C.c_void_p(), C.c_void_p()
        check(lib().gm_ctx_queue(self.handle, C.byref(q)))
        check(lib().gm_ctx_cache(self.handle, C.byref(c)))
        self.queue = RequestQueue(_borrowed=q.value)
        self.cache = SuperKernelCache(_borrowed=c.value)

    def close(self) -> None:
        if getattr(self, "handle", None):
            lib().gm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:  # (at interpreter exit the module globals may already be gone)
            self.close()
        except Exception:
            pass

    def set_option(self, name: str, value: int) -> None:
        """Runtime execution option (see gm_ctx_set_option in the header)."""
        check(lib().gm_ctx_set_option(self.handle, name.encode(), int(value)))

    def set_policy(self, policy: BatchPolicy) -> None:
        check(lib().gm_ctx_set_policy(self.handle, C.byref(policy._c())))
        self.policy = policy

    # ------------------------------------------------------------ tenants
    def migrate_tenant(self, tenant: int, dst: "Context", stream: int = 0) -> int:
        """Re-admit ``tenant`` on ``dst`` (gm_migrate_tenant): its weights and
        external inputs move to buffers the destination owns (peer copies over
        NVLink between GPUs); returns its index in ``dst``."""
        out = C.c_int32()
        check(lib().gm_migrate_tenant(self.handle, int(tenant), dst.handle, int(stream), C.byref(out)))
        return out.value

    def migrate_tenants(self, tenants: Sequence[int], dst: "Context", stream: int = 0) -> List[int]:
        """gm_migrate_tenants: buffers shared among ``tenants`` (batch
        variants of one logical tenant) stay shared on ``dst``."""
        n = len(tenants)
        src = (C.c_int32 * n)(*tenants)
        out = (C.c_int32 * n)()
        check(lib().gm_migrate_tenants(self.handle, src, n, dst.handle, int(stream), out))
        return list(out)

    def register_tenant(self, layers: Sequence[LayerBuffers], slo_latency: float = 0.1, concurrency: int = 1,
                        tenant_id: str = "") -> int:
        descs = (N.gm_layer_desc * len(layers))()
        for i, L in enumerate(layers):
            d = descs[i]
            d.x, d.y = L.x.data_ptr(), L.y.data_ptr()
            d.w = L.w.data_ptr() if L.w is not None else None
            d.act = L.activation
            d.src = L.src
            d.res_src = L.res_src
            if L.res is not None:
                d.res = L.res.data_ptr()
                d.ldr = L.res.stride(0)
            if L.kind in ("maxpool", "avgpool"):
                d.kind = N.GM_LAYER_MAXPOOL if L.kind == "maxpool" else N.GM_LAYER_AVGPOOL
                d.batch = L.batch
                d.conv = L.conv._c()
            elif L.kind == "conv":
                d.kind = N.GM_LAYER_CONV
                d.batch = L.batch
                d.conv = L.conv._c()
                d.ldw = L.w.stride(0)
                d.ldx = L.x.stride(2)  # NHWC pixel pitch in channels (8 selects the narrow im2col path)
            elif L.kind == "dwconv":
                d.kind = N.GM_LAYER_DWCONV
                d.batch = L.batch
                d.conv = L.conv._c()
                d.ldw = L.w.stride(0)
            elif L.kind == "gemm":
                d.kind = N.GM_LAYER_GEMM
                d.gemm = L.gemm._c()
                d.ldx = L.x.stride(0)
                d.ldw = L.w.stride(0)
            else:
                raise ValueError(f"unknown layer kind {L.kind!r}")
        t = N.gm_tenant_desc(tenant_id.encode(), descs, len(layers), float(slo_latency), int(concurrency), 0)
        idx = C.c_int32()
        check(lib().gm_register_tenant(self.handle, C.byref(t), C.byref(idx)))
        self._keepalive.append(list(layers))
        return int(idx.value)

    def layer_shape(self, tenant: int, layer: int) -> GemmShape:
        out = N.gm_gemm_shape()
        check(lib().gm_layer_shape(self.handle, tenant, layer, C.byref(out)))
        return GemmShape._from(out)

    # ------------------------------------------------------------ dispatch
    def dispatch(self, sk: SuperKernel, stream: int = 0):
        """Launch one formed SuperKernel; returns (planned seconds, cache hit)."""
        d, hit = C.c_double(), C.c_int()
        check(lib().gm_dispatch(self.handle, sk._plans.handle, sk._index, int(stream), C.byref(d), C.byref(hit)))
        return float(d.value), bool(hit.value)

    def launch_members(self, members: Sequence[tuple], stream: int = 0) -> int:
        """Launch an explicit (tenant, layer) list as one super-kernel."""
        n = len(members)
        ts = (C.c_int32 * n)(*[m[0] for m in members])
        ls = (C.c_int32 * n)(*[m[1] for m in members])
        out = C.c_int32()
        check(lib().gm_launch_members(self.handle, ts, ls, n, int(stream), C.byref(out)))
        return int(out.value)

    def launch_count(self, members: Sequence[tuple]) -> int:
        n = len(members)
        ts = (C.c_int32 * n)(*[m[0] for m in members])
        ls = (C.c_int32 * n)(*[m[1] for m in members])
        out = C.c_int32()
        check(lib().gm_members_launch_count(self.handle, ts, ls, n, C.byref(out)))
        return int(out.value)

    def plan_round(self, tenants: Sequence[int], now: int = 0) -> "Round":
        arr = (C.c_int32 * max(1, len(tenants)))(*tenants)
        h = C.c_void_p()
        check(lib().gm_plan_round(self.handle, arr, len(tenants), int(now), C.byref(h)))
        return Round(self, h.value)

    def launch_stats(self):
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib().gm_ctx_launch_stats(self.handle, C.byref(a), C.byref(b), C.byref(c)))
        return {"superkernels": a.value, "prepasses": b.value, "tiles": c.value}


class Round:
    """The dispatch sequence of one space-time round (gm_plan_round)."""

    def __init__(self, ctx: Context, handle: int):
        self.ctx = ctx
        self._owner = _Plans(handle)
        self.handle = handle
        self.count = int(lib().gm_plans_count(handle))
        k = C.c_uint64()
        check(lib().gm_plans_key(handle, C.byref(k)))
        self.key = int(k.value)
        self._kernels: Optional[List[SuperKernel]] = None
        self._times: Optional[List[tuple]] = None

    @property
    def kernels(self) -> List[SuperKernel]:
        """The formed super-kernels (unpacked on first use)."""
        if self._kernels is None:
            self._kernels = _unpack_plans(self.handle, self._owner)
        return self._kernels

    @property
    def times(self) -> List[tuple]:
        """Virtual [start, end) of every dispatch of the round."""
        if self._times is None:
            self._times = []
            for i in range(self.count):
                s, e = C.c_int64(), C.c_int64()
                check(lib().gm_plans_times(self.handle, i, C.byref(s), C.byref(e)))
                self._times.append((int(s.value), int(e.value)))
        return self._times

    def end_time(self) -> int:
        if not self.count:
            return 0
        s, e = C.c_int64(), C.c_int64()
        check(lib().gm_plans_times(self.handle, self.count - 1, C.byref(s), C.byref(e)))
        return int(e.value)

    @property
    def signatures(self) -> List[str]:
        return [k.shape_signature for k in self.kernels]

    def prepare(self) -> None:
        check(lib().gm_prepare_plans(self.ctx.handle, self.handle))

    def launch(self, stream: int = 0) -> int:
        """One launch per formed super-kernel (the reference's dispatch unit)."""
        out = C.c_int32()
        check(lib().gm_dispatch_plans(self.ctx.handle, self.handle, int(stream), C.byref(out)))
        return int(out.value)

    def tile_info(self) -> List[dict]:
        """The executed tile table of this round's program (gm_round_tile_info)."""
        n = C.c_size_t()
        arr = (N.gm_round_tile * max(1, self._n_round_tiles()))()
        check(lib().gm_round_tile_info(self.ctx.handle, self.handle, arr, len(arr), C.byref(n)))
        return [{f: getattr(arr[i], f) for f, _ in N.gm_round_tile._fields_} for i in range(n.value)]

    def _n_round_tiles(self) -> int:
        n = C.c_size_t()
        st = lib().gm_round_tile_info(self.ctx.handle, self.handle, None, 0, C.byref(n))
        if st not in (N.GM_OK, N.GM_ERANGE):
            check(st)
        return int(n.value)

    def launch_round(self, stream: int = 0) -> int:
        """The whole round as one persistent launch (round program)."""
        out = C.c_int32()
        check(lib().gm_dispatch_round(self.ctx.handle, self.handle, int(stream), C.byref(out)))
        return int(out.value)
