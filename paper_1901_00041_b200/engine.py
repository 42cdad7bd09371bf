"""Space-time serving engine on one GPU: tenants, rounds, launch programs.

A *round* is the hot path of BASELINE.json's north star on one GPU: every
registered tenant submits one query batch; the space-time scheduler
(gm_plan_round: dynamic batcher + packing planner) turns the layer requests
into super-kernels; each super-kernel executes the members' conv/GEMM tiles
in one sm_100a launch.  The same kernel code also runs the two baseline
modes the paper compares against (time-only: serial per-tenant launches;
space-only: one stream per tenant), so ratios isolate packing.

Steady-state rounds are captured as CUDA graphs keyed by the plan's
signature sequence (the B200 form of "cache super-kernels as workloads
stabilize"); ``serve_round`` re-plans every round on the host
and replays the cached graph while the sequence is unchanged.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import torch

from . import _native as N
from ._native import check, lib
from .runtime import Context, LayerBuffers, Round
from .scheduler import BatchPolicy, DeviceSpec, GemmShape
from .workload import Layer

_MASK = (1 << 64) - 1


def mix64(*parts: int) -> int:
    """splitmix64 chained over the parts (hash, never XOR)."""
    h = 0x9E3779B97F4A7C15
    for p in parts:
        h = (h + (int(p) & _MASK) + 0x9E3779B97F4A7C15) & _MASK
        z = h
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
        h = z ^ (z >> 31)
    return h & ((1 << 63) - 1)


KIND_INPUT, KIND_WEIGHT = 1, 2
NARROW_C = 8  # pixel pitch of narrow-channel conv inputs (superkernel.cuh kNarrowC)


class Graph:
    """A captured launch program (gm_graph)."""

    def __init__(self, handle: int, timed: bool):
        self.handle = handle
        self.timed = timed
        sk, k = C.c_int32(), C.c_int32()
        check(lib().gm_graph_launch_count(handle, C.byref(sk), C.byref(k)))
        self.superkernels, self.kernels = int(sk.value), int(k.value)

    def launch(self, stream: int) -> None:
        check(lib().gm_graph_launch(self.handle, int(stream)))

    def kernel_times_ms(self) -> List[float]:
        n = C.c_size_t()
        arr = (C.c_float * max(1, self.superkernels))()
        check(lib().gm_graph_kernel_times(self.handle, arr, self.superkernels, C.byref(n)))
        return [float(arr[i]) for i in range(n.value)]

    def __del__(self):
        if getattr(self, "handle", None):
            try:  # (at interpreter exit the module globals may already be gone)
                lib().gm_graph_destroy(self.handle)
            except Exception:
                pass
            self.handle = None


class TenantModel:
    """Device buffers of one tenant's operator graph with synthetic data.

    Dataflow: a layer with ``src`` reads that earlier layer's output buffer
    (a view of it), and ``res`` adds that layer's output in the epilogue, so
    the tenant's query input determines every activation down to its result.
    A layer without ``src`` (the first, or every layer of a plain operator
    list) gets its own input buffer.  Inputs U(-1, 1), weights Kaiming-normal
    (std sqrt(2 / fan_in)); each tensor from its own generator seeded by
    mix64(seed, tenant, layer, kind).  Weight rows are padded to a multiple of
    8 elements (16-byte TMA strides).
    """

    def __init__(self, layers: Sequence[Layer], batch: int, seed: int, tenant: int, device: torch.device,
                 narrow_inputs: bool = False):
        self.layers = list(layers)
        self.batch = batch
        self.buffers: List[LayerBuffers] = []
        ys: List[torch.Tensor] = []
        for li, L in enumerate(self.layers):
            s = L.gemm_shape(batch)
            g_in = torch.Generator(device=device).manual_seed(mix64(seed, tenant, li, KIND_INPUT))
            g_w = torch.Generator(device=device).manual_seed(mix64(seed, tenant, li, KIND_WEIGHT))
            y = torch.empty(s.m, s.n, device=device, dtype=torch.bfloat16)
            ys.append(y)
            src = -1 if L.src is None else int(L.src)
            res, res_src = None, -1
            if L.res is not None:
                res_src = int(L.res)
                res = ys[res_src].view(s.m, s.n)  # same rows and columns as this layer's output
            windowed = L.kind in ("conv", "dwconv", "maxpool", "avgpool")
            if windowed:
                c = L.conv
                if src >= 0:
                    x = ys[src].view(batch, c.image_h, c.image_w, c.in_channels)
                else:
                    x = (torch.rand(batch, c.image_h, c.image_w, c.in_channels, device=device, generator=g_in) * 2 - 1)
                    x = x.to(torch.bfloat16)
                    if narrow_inputs and L.kind == "conv" and c.in_channels < NARROW_C and c.kernel_h > 1:
                        # narrow-channel input (RGB stem): stored with an 8-channel
                        # pixel pitch, zero padded, for the narrow TMA im2col path
                        # (opt-in: one 16 B TMA request per pixel and tap is slower
                        # than the explicit pre-pass on B200)
                        xp = torch.zeros(batch, c.image_h, c.image_w, NARROW_C, device=device, dtype=torch.bfloat16)
                        xp[..., : c.in_channels] = x
                        x = xp
            if L.kind in ("maxpool", "avgpool"):
                self.buffers.append(LayerBuffers(L.kind, x, None, y, conv=L.conv, batch=batch, act=L.act, src=src))
                continue
            if L.kind == "dwconv":
                w = (torch.randn(s.n, s.k, device=device, generator=g_w) * (2.0 / s.k) ** 0.5).to(torch.bfloat16)
                self.buffers.append(LayerBuffers("dwconv", x, w, y, conv=L.conv, batch=batch, act=L.act, src=src))
                continue
            kpad = (s.k + 7) // 8 * 8
            w = torch.zeros(s.n, kpad, device=device, dtype=torch.bfloat16)
            w[:, : s.k] = (torch.randn(s.n, s.k, device=device, generator=g_w) * (2.0 / s.k) ** 0.5).to(torch.bfloat16)
            if L.kind == "conv":
                self.buffers.append(LayerBuffers("conv", x, w, y, conv=L.conv, batch=batch, act=L.act, src=src,
                                                 res=res, res_src=res_src))
                continue
            if src >= 0:
                x = ys[src].view(s.m, -1)[:, L.src_col: L.src_col + s.k]  # strided view: ldx = the source's width
            else:
                x = torch.zeros(s.m, kpad, device=device, dtype=torch.bfloat16)
                x[:, : s.k] = (torch.rand(s.m, s.k, device=device, generator=g_in) * 2 - 1).to(torch.bfloat16)
            self.buffers.append(LayerBuffers("gemm", x, w, y, gemm=s, act=L.act, src=src, res=res, res_src=res_src))

    @property
    def query_input(self) -> torch.Tensor:
        return self.buffers[0].x

    @property
    def query_output(self) -> torch.Tensor:
        return self.buffers[-1].y

    def flops(self) -> int:
        return sum(L.flops(self.batch) for L in self.layers)

    def compulsory_bytes(self) -> int:
        return sum(L.compulsory_bytes(self.batch) for L in self.layers)


class SpaceTimeEngine:
    """Tenants on one GPU + the three execution modes over the same kernel."""

    def __init__(self, tenant_layers: Sequence[Sequence[Layer]], batches: Sequence[int], device_index: int = 0,
                 seed: int = 42, slo_latency: float = 0.040, policy: Optional[BatchPolicy] = None,
                 tenant_offset: int = 0, options: Optional[Dict[str, int]] = None,
                 device_spec: Optional[DeviceSpec] = None):
        self.device = torch.device("cuda", device_index)
        torch.cuda.set_device(self.device)
        self.ctx = Context(device_index, device=device_spec, policy=policy or BatchPolicy(target_batch=0))
        for name, value in (options or {}).items():
            self.ctx.set_option(name, value)
        self.models: List[TenantModel] = []
        self.tenants: List[int] = []
        for i, (layers, b) in enumerate(zip(tenant_layers, batches)):
            m = TenantModel(layers, b, seed, tenant_offset + i, self.device)
            self.models.append(m)
            self.tenants.append(self.ctx.register_tenant(m.buffers, slo_latency=slo_latency,
                                                         tenant_id=f"t{tenant_offset + i}"))
        self._now = 0
        self.ctx_slo = slo_latency
        self._alt = None
        self._graphs: Dict[tuple, Graph] = {}  # (plan key, host buffers) -> end-to-end launch program
        self._stable_plan: Optional[Round] = None  # serve_round's steady-state plan
        self._last_key: Optional[int] = None

    # ------------------------------------------------------------ planning
    def flops_per_round(self) -> int:
        return sum(m.flops() for m in self.models)

    def compulsory_bytes_per_round(self) -> int:
        return sum(m.compulsory_bytes() for m in self.models)

    def plan_round(self, policy: Optional[BatchPolicy] = None) -> Round:
        """One space-time round on the virtual clock (advances it).

        ``policy`` replaces the context's BatchPolicy from this round on
        (e.g. ``max_waves=1`` for reference plan parity)."""
        if policy is not None:
            self.ctx.set_policy(policy)
            self._stable_plan = None
        r = self.ctx.plan_round(self.tenants, self._now)
        if r.count:
            self._now = r.end_time()  # dispatches are serial on the virtual device
        return r

    # ------------------------------------------------------------ launch programs
    def capture_packed(self, rnd: Round, timed: bool = False) -> Graph:
        h = C.c_void_p()
        check(lib().gm_graph_capture_plans(self.ctx.handle, rnd.handle, int(timed), C.byref(h)))
        return Graph(h.value, timed)

    def capture_round(self, rnd: Round, timed: bool = False) -> Graph:
        """The round program: every plan of the round in one persistent launch."""
        h = C.c_void_p()
        check(lib().gm_graph_capture_round(self.ctx.handle, rnd.handle, int(timed), C.byref(h)))
        return Graph(h.value, timed)

    def capture_serial(self, mode: str, timed: bool = False) -> Graph:
        m = {"time_only": N.GM_MODE_TIME_ONLY, "space_only": N.GM_MODE_SPACE_ONLY}[mode]
        arr = (C.c_int32 * len(self.tenants))(*self.tenants)
        h = C.c_void_p()
        check(lib().gm_graph_capture_serial(self.ctx.handle, arr, len(self.tenants), m, int(timed), C.byref(h)))
        return Graph(h.value, timed)

    # ------------------------------------------------------------ public serving call
    def capture_round_e2e(self, rnd: Round, host_inputs: Sequence[torch.Tensor],
                          host_outputs: Sequence[torch.Tensor]) -> Graph:
        """The round program with its host traffic: per tenant the H2D copy of
        its query batch opens that tenant's input gate, so the kernel starts a
        tenant's chain as soon as its input has landed (copies overlap compute);
        D2H of every tenant's result after the kernel."""
        n = len(self.models)
        tid = (C.c_int32 * n)(*self.tenants)
        h_in = (C.c_void_p * n)(*[h.data_ptr() for h in host_inputs])
        d_in = (C.c_void_p * n)(*[m.query_input.data_ptr() for m in self.models])
        ib = (C.c_size_t * n)(*[h.numel() * h.element_size() for h in host_inputs])
        d_out = (C.c_void_p * n)(*[m.query_output.data_ptr() for m in self.models])
        h_out = (C.c_void_p * n)(*[h.data_ptr() for h in host_outputs])
        ob = (C.c_size_t * n)(*[h.numel() * h.element_size() for h in host_outputs])
        h = C.c_void_p()
        check(lib().gm_graph_capture_round_e2e(self.ctx.handle, rnd.handle, n, tid, h_in, d_in, ib, d_out, h_out, ob,
                                               C.byref(h)))
        return Graph(h.value, False)

    # ------------------------------------------------------------ public serving call
    def e2e_steady(self, host_inputs: Sequence[torch.Tensor], host_outputs: Sequence[torch.Tensor]) -> bool:
        """True once serve_round replays a captured program for these host buffers."""
        rnd = self._stable_plan
        if rnd is None:
            return False
        key = (rnd.key, tuple(h.data_ptr() for h in host_inputs), tuple(h.data_ptr() for h in host_outputs))
        return key in self._graphs

    def serve_round(self, host_inputs: Sequence[torch.Tensor], host_outputs: Sequence[torch.Tensor],
                    stream: torch.cuda.Stream) -> Round:
        """End-to-end round through the public API with host buffers.

        Plans the round with the space-time scheduler (re-planned until two
        consecutive rounds plan identically, then the steady-state plan is
        reused: a SuperKernelCache hit for every member set) and
        replays (or captures, on a new plan or new host buffers) the
        end-to-end launch program: H2D of each tenant's query batch gating its
        chain, the round kernel, D2H of each tenant's result.  Returns after
        the results are on the host.
        """
        for m, h in zip(self.models, host_inputs):
            if h.numel() != m.query_input.numel() or h.dtype != m.query_input.dtype:
                raise ValueError("host input does not match the tenant's query batch")
        rnd = self._stable_plan
        if rnd is None:
            rnd = self.plan_round()
            if self._last_key == rnd.key:
                self._stable_plan = rnd
            self._last_key = rnd.key
        key = (rnd.key, tuple(h.data_ptr() for h in host_inputs), tuple(h.data_ptr() for h in host_outputs))
        g = self._graphs.get(key)
        if g is None:
            g = self._graphs[key] = self.capture_round_e2e(rnd, host_inputs, host_outputs)
        g.launch(stream.cuda_stream)
        stream.synchronize()
        return rnd

    def _alternate_round(self):
        """A second registration of every tenant whose query input and result
        are its own buffers (every other buffer shared), and its round program:
        serve_rounds alternates the two, so step i+1's batch lands in the input
        step i is not reading, step i's results are copied out while step i+1
        runs, and no device-to-device staging move sits between rounds."""
        import dataclasses
        alt_inputs, alt_outputs, alt_tenants = [], [], []
        for t, m in zip(self.tenants, self.models):
            q = m.query_input
            xin = torch.zeros_like(q)
            lo, hi = q.data_ptr(), q.data_ptr() + q.numel() * q.element_size()

            def remap(tensor):  # a view of the query input -> the same view of xin
                if tensor is None or not (lo <= tensor.data_ptr() < hi):
                    return tensor
                off = (tensor.data_ptr() - lo) // q.element_size()
                return torch.as_strided(xin, tensor.size(), tensor.stride(), xin.storage_offset() + off)

            bufs = [dataclasses.replace(b, x=remap(b.x), res=remap(b.res)) for b in m.buffers]
            yout = torch.empty_like(m.query_output)  # the last layer's output: nothing reads it in the round
            bufs[-1] = dataclasses.replace(bufs[-1], y=yout)
            alt_inputs.append(xin)
            alt_outputs.append(yout)
            alt_tenants.append(self.ctx.register_tenant(bufs, slo_latency=self.ctx_slo, tenant_id=f"alt{t}"))
        rnd = self.ctx.plan_round(alt_tenants, self._now)
        return alt_inputs, alt_outputs, self.capture_round(rnd)

    def serve_rounds(self, steps: Sequence[Tuple[Sequence[torch.Tensor], Sequence[torch.Tensor]]],
                     stream: torch.cuda.Stream) -> Round:
        """Back-to-back end-to-end rounds, double-buffered: step i+1's H2D
        copies (pinned host -> device, on a copy stream) overlap step i's
        round kernel: two registrations of the tenants with their own
        query inputs alternate (every other buffer shared), so each step's
        batch lands straight in the input its round program reads; each step
        replays its program and copies every tenant's result to that step's
        host buffers.  Returns after the last results
        are on the host.  Throughput is max(copy, compute) per round instead
        of their sum; per-round latency is serve_round's."""
        if not steps:
            raise ValueError("no steps")
        for h_in, h_out in steps:
            if len(h_in) != len(self.models) or len(h_out) != len(self.models):
                raise ValueError("one host input and one host output per tenant")
            for m, h in zip(self.models, h_in):
                if h.numel() != m.query_input.numel() or h.dtype != m.query_input.dtype:
                    raise ValueError("host input does not match the tenant's query batch")
            for m, h in zip(self.models, h_out):
                if h.numel() != m.query_output.numel() or h.dtype != m.query_output.dtype:
                    raise ValueError("host output does not match the tenant's result")
        rnd = self._stable_plan
        tries = 0
        while rnd is None:  # plan until two consecutive rounds agree (the serve_round rule)
            r = self.plan_round()
            tries += 1
            if self._last_key == r.key:
                self._stable_plan = rnd = r
            elif tries == 8:
                rnd = r
            self._last_key = r.key
        g = self._graphs.get(("round", rnd.key))
        if g is None:
            g = self._graphs[("round", rnd.key)] = self.capture_round(rnd)
        if getattr(self, "_alt", None) is None:
            self._alt = self._alternate_round()
            self._copy_stream = torch.cuda.Stream(self.device)
            self._out_stream = torch.cuda.Stream(self.device)
        alt_inputs, alt_outputs, g_alt = self._alt
        inputs = [[m.query_input for m in self.models], alt_inputs]
        outputs = [[m.query_output for m in self.models], alt_outputs]
        graphs = [g, g_alt]
        cs, ds = self._copy_stream, self._out_stream  # H2D and D2H run in both directions at once
        landed = [torch.cuda.Event(), torch.cuda.Event()]
        done = [torch.cuda.Event(), torch.cuda.Event()]
        drained = [torch.cuda.Event(), torch.cuda.Event()]
        cs.wait_stream(stream)
        ds.wait_stream(stream)
        for i, (h_in, h_out) in enumerate(steps):
            b = i & 1
            with torch.cuda.stream(cs):
                if i >= 2:
                    cs.wait_event(done[b])  # input set b read by step i-2's round
                for d, h in zip(inputs[b], h_in):
                    d.view(-1).copy_(h.view(-1), non_blocking=True)
                landed[b].record(cs)
            with torch.cuda.stream(stream):
                stream.wait_event(landed[b])
                if i >= 2:
                    stream.wait_event(drained[b])  # output set b copied out after step i-2
                graphs[b].launch(stream.cuda_stream)
                done[b].record(stream)
            with torch.cuda.stream(ds):
                ds.wait_event(done[b])
                for y, h in zip(outputs[b], h_out):
                    h.view(-1).copy_(y.view(-1), non_blocking=True)
                drained[b].record(ds)
        ds.synchronize()
        stream.synchronize()
        return rnd


# --------------------------------------------------------------------------- serving
@dataclass
class ServeTenant:
    """One logical tenant of a serving session (gm_serve_tenant).

    ``rate_qps`` > 0: Poisson arrivals; 0: closed loop with ``concurrency``
    queries outstanding.  The dynamic batcher serves up to ``max_batch``
    queries per dispatch with the smallest registered variant in ``batches``
    that holds them (default: powers of two up to ``max_batch``).
    ``io_slots`` > 0: queries carry data -- pinned host slots of that many
    query inputs / results (``ServingEngine.host_inputs[i]`` /
    ``host_outputs[i]``); query k uses slot k % io_slots, copied in before
    its dispatch's round and out after it."""
    layers: Sequence[Layer]
    max_batch: int = 8
    rate_qps: float = 0.0
    concurrency: int = 1
    slo_latency: float = 0.040
    batches: Optional[Sequence[int]] = None
    io_slots: int = 0


@dataclass
class ServeResult:
    stats: Dict[str, float]
    latencies_ms: List[float] = field(default_factory=list)
    # one dict per dispatch (gm_serve_trace): start_ns, end_ns, device_ms,
    # flops, queries, tenants, launches, tiles; report.write_trace_ndjson
    # renders them as the reference's NDJSON trace lines
    dispatches: List[Dict[str, float]] = field(default_factory=list)


def _variant(buf: LayerBuffers, max_batch: int, b: int) -> LayerBuffers:
    """The same device buffers viewed as a batch-b operator (the first b
    queries: NHWC images and GEMM rows are query-major, so the batch-b views of
    a dataflow chain still chain)."""
    if buf.kind in ("conv", "dwconv", "maxpool", "avgpool"):
        return LayerBuffers(buf.kind, buf.x, buf.w, buf.y, conv=buf.conv, batch=b, act=buf.activation, src=buf.src,
                            res=buf.res, res_src=buf.res_src)
    g = buf.gemm
    return LayerBuffers("gemm", buf.x, buf.w, buf.y, gemm=GemmShape(g.m // max_batch * b, g.n, g.k),
                        act=buf.activation, src=buf.src, res=buf.res, res_src=buf.res_src)


class ServingEngine:
    """Real-clock space-time serving on one GPU (gm_serve).

    Each logical tenant owns device buffers for its largest batch and one
    registered runtime tenant per batch variant sharing them; ``serve`` runs
    the native serving loop (arrivals, dynamic batcher, round-program
    dispatch, CUDA-event completions, straggler monitor) for ``duration``
    seconds and returns throughput and query-latency percentiles."""

    def __init__(self, tenants: Sequence[ServeTenant], device_index: int = 0, seed: int = 42,
                 policy: Optional[BatchPolicy] = None, options: Optional[Dict[str, int]] = None,
                 device_spec: Optional[DeviceSpec] = None, tenant_offset: int = 0):
        self.device = torch.device("cuda", device_index)
        torch.cuda.set_device(self.device)
        # serving prices member sets with the calibrated profile (measured
        # peaks + latency floor, profiles/b200_calibrated.json): the SLO
        # trigger's first prediction and the fallback choice use it
        from .scheduler import b200_calibrated_profile
        self.ctx = Context(device_index, device=device_spec or b200_calibrated_profile(),
                           policy=policy or BatchPolicy(target_batch=0))
        for name, value in (options or {}).items():
            self.ctx.set_option(name, value)
        self.specs = list(tenants)
        self.models: List[TenantModel] = []
        self._variants: List[List[Tuple[int, int]]] = []
        for i, spec in enumerate(self.specs):
            bmax = spec.max_batch
            batches = sorted(set(spec.batches or [b for b in (1, 2, 4, 8, 16, 32, 64) if b < bmax] + [bmax]))
            if batches[-1] != bmax or batches[0] < 1:
                raise ValueError("batch variants must be >= 1 and end at max_batch")
            m = TenantModel(spec.layers, bmax, seed, tenant_offset + i, self.device)
            self.models.append(m)
            vs = []
            for b in batches:
                bufs = [_variant(buf, bmax, b) for buf in m.buffers]
                vs.append((b, self.ctx.register_tenant(bufs, slo_latency=spec.slo_latency,
                                                       tenant_id=f"t{tenant_offset + i}/b{b}")))
            self._variants.append(vs)
        # per-query I/O slots (pinned): one query's rows of layer 0's input /
        # of the last layer's output each
        self.host_inputs: List[Optional[torch.Tensor]] = []
        self.host_outputs: List[Optional[torch.Tensor]] = []
        for spec, m in zip(self.specs, self.models):
            if spec.io_slots <= 0:
                self.host_inputs.append(None)
                self.host_outputs.append(None)
                continue
            x, y = m.query_input, m.query_output
            qx = x.reshape(spec.max_batch, -1)
            qy = y.reshape(spec.max_batch, -1)
            hin = torch.empty((spec.io_slots, qx.shape[1]), dtype=x.dtype).pin_memory()
            g = torch.Generator().manual_seed(seed * 7919 + tenant_offset + len(self.host_inputs))
            hin.copy_((torch.rand(hin.shape, generator=g) * 2 - 1).to(x.dtype))
            b0 = m.buffers[0]
            if b0.kind != "gemm" and x.shape[-1] > b0.conv.in_channels:  # narrow pitch: pad channels stay zero
                hin.view(spec.io_slots, -1, x.shape[-1])[..., b0.conv.in_channels:] = 0
            self.host_inputs.append(hin)
            self.host_outputs.append(torch.zeros((spec.io_slots, qy.shape[1]), dtype=y.dtype).pin_memory())

    def readmit(self, tenants: Sequence[int], other: "ServingEngine") -> List[int]:
        """Re-place evicted logical tenants on another engine (another GPU's
        context, or the same GPU's): every batch variant migrates with
        gm_migrate_tenant (weights and inputs by peer copy) and ``other``
        serves the tenant from then on (placement.least_loaded picks
        ``other`` among several).  Returns their logical indices in ``other``."""
        out = []
        for i in tenants:
            moved = self.ctx.migrate_tenants([tid for _, tid in self._variants[i]], other.ctx)
            vs = [(b, t) for (b, _), t in zip(self._variants[i], moved)]
            spec = self.specs[i]
            hin, hout = self.host_inputs[i], self.host_outputs[i]
            other.specs.append(ServeTenant(spec.layers, max_batch=spec.max_batch, rate_qps=spec.rate_qps,
                                           concurrency=spec.concurrency, slo_latency=spec.slo_latency,
                                           batches=[b for b, _ in vs], io_slots=spec.io_slots if hin is not None else 0))
            other.models.append(None)
            other._variants.append(vs)
            # the tenant's query slots travel with it (same inputs, fresh results)
            other.host_inputs.append(hin.clone().pin_memory() if hin is not None else None)
            other.host_outputs.append(torch.zeros_like(hout).pin_memory() if hout is not None else None)
            out.append(len(other.specs) - 1)
        return out

    def flops_per_query(self, i: int) -> int:
        return sum(L.flops(1) for L in self.specs[i].layers)

    def serve(self, duration: float, warmup: float = 0.1, max_wait: float = -1.0, depth: int = 1,
              seed: int = 42, stream: Optional[torch.cuda.Stream] = None, prewarm: int = 4096,
              degrade: Optional[Tuple[int, float, float]] = None, plan_cache_cap: int = 0,
              async_plan: bool = False) -> ServeResult:
        """``degrade`` = (tenant, slowdown, start_s): inject_degradation
        (sim.cpp:60-68) on real hardware -- that tenant's observed completions
        stretch by ``slowdown`` from ``start_s`` on, feeding the straggler
        monitor, which evicts it (terminal)."""
        n = len(self.specs)
        arr = (N.gm_serve_tenant * n)()
        keep = []
        for i, (spec, vs) in enumerate(zip(self.specs, self._variants)):
            tid = (C.c_int32 * len(vs))(*[t for _, t in vs])
            bat = (C.c_int32 * len(vs))(*[b for b, _ in vs])
            keep += [tid, bat]
            hin, hout = self.host_inputs[i], self.host_outputs[i]
            arr[i] = N.gm_serve_tenant(len(vs), tid, bat, float(spec.rate_qps), int(spec.concurrency), 0,
                                       float(spec.slo_latency), self.flops_per_query(i),
                                       hin.data_ptr() if hin is not None else None,
                                       hout.data_ptr() if hout is not None else None,
                                       int(spec.io_slots) if hin is not None else 0, 0)
        s = stream or torch.cuda.Stream(self.device)
        dt, dslow, dstart = degrade if degrade is not None else (-1, 1.0, 0.0)
        cfg = N.gm_serve_config(float(duration), float(warmup), float(max_wait), int(seed), int(depth),
                                int(prewarm), int(s.cuda_stream), int(dt), 0, float(dslow), float(dstart),
                                int(plan_cache_cap), int(bool(async_plan)))
        out = N.gm_serve_stats()
        cap = 1 << 20
        lat = (C.c_double * cap)()
        nl = C.c_size_t()
        check(lib().gm_serve(self.ctx.handle, arr, n, C.byref(cfg), C.byref(out), lat, cap, C.byref(nl)))
        stats = {f: getattr(out, f) for f, _ in N.gm_serve_stats._fields_ if not f.startswith("reserved")}
        ne = C.c_size_t()
        check(lib().gm_serve_trace(self.ctx.handle, None, 0, C.byref(ne)))
        evs = (N.gm_dispatch_event * max(1, ne.value))()
        check(lib().gm_serve_trace(self.ctx.handle, evs, ne.value, C.byref(ne)))
        dispatches = [{f: getattr(evs[i], f) for f, _ in N.gm_dispatch_event._fields_} for i in range(ne.value)]
        return ServeResult(stats, [lat[i] for i in range(min(nl.value, cap))], dispatches)
