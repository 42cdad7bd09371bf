"""TEST INFRASTRUCTURE ONLY — a pure-Python restatement of the reference's
space-time planner, used as the checker for the product's C++ planner.

Only tests/ import this module.  It restates, function by function:
  gemm_flops / gemm_bytes / im2col / batch_inputs  proj/include/gpumux/gemm.hpp:33-56
  to_ns / to_seconds                               proj/include/gpumux/vtime.hpp:13-19
  thread_blocks / dispatch_duration                proj/src/cost_model.cpp:14-46
  RequestQueue.enqueue / cancel_tenant             proj/src/scheduler.cpp:8-35
  slo_headroom                                     proj/src/scheduler.cpp:37-41
  plan_super_kernel / signature                    proj/src/scheduler.cpp:43-92
  form_batches                                     proj/src/scheduler.cpp:96-199
  dispatch_cost                                    proj/src/scheduler.cpp:201-212
  record_latency / detect_stragglers / evict       proj/src/scheduler.cpp:214-271
  percentile_nearest_rank / geomean                proj/src/metrics.cpp:10-28
  run_space_time (closed loop)                     proj/src/sim.cpp:398-581
Python floats are IEEE doubles and every expression keeps the reference's
operand order, so results are bit-identical for the small cases it is
used on (pinned in tests/test_oracle.py against tests/golden/*.json, which
oracle/_ref — the compiled reference — produced).
"""
from __future__ import annotations

import heapq
import math
from bisect import insort
from dataclasses import dataclass, field, replace
from typing import Dict, List, Optional, Sequence, Tuple

Shape = Tuple[int, int, int]


def round_half_away(x: float) -> int:
    """std::llround: nearest, halfway cases away from zero."""
    f = math.floor(x)
    d = x - f
    if d > 0.5 or (d == 0.5 and x > 0):
        return int(f) + 1
    if d == 0.5 and x < 0:
        return int(f)
    return int(f) if d < 0.5 else int(f) + 1


def to_ns(seconds: float) -> int:
    return round_half_away(seconds * 1e9)


def to_seconds(ns: int) -> float:
    return float(ns) * 1e-9


def gemm_flops(s: Shape) -> int:
    return 2 * s[0] * s[1] * s[2]


def gemm_bytes(s: Shape, elem: int = 4) -> int:
    m, n, k = s
    return elem * (m * k + k * n + m * n)


def im2col(h, w, kh, kw, cin, cout, stride, pad) -> Shape:
    oh = (h + 2 * pad - kh) // stride + 1
    ow = (w + 2 * pad - kw) // stride + 1
    if oh < 1 or ow < 1:
        raise ValueError("im2col: non-positive output dims")
    return (oh * ow, cout, kh * kw * cin)


def batch_inputs(s: Shape, b: int) -> Shape:
    return (s[0] * b, s[1], s[2])


def shape_key(s: Shape) -> str:
    return f"{s[0]}x{s[1]}x{s[2]}"


@dataclass
class Device:
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

    def slot_total(self) -> int:
        return self.sm_count * self.blocks_per_sm


def cdiv(a: int, b: int) -> int:
    return (a + b - 1) // b


def thread_blocks(s: Shape, d: Device) -> int:
    return cdiv(s[0], d.tile_m) * cdiv(s[1], d.tile_n)


@dataclass
class Cost:
    flops: int = 0
    bytes: int = 0
    blocks: int = 0
    duration: float = 0.0
    waves: int = 0


def dispatch_duration(groups: Sequence[Tuple[Shape, int]], d: Device, slot_budget: int, launches: int) -> Cost:
    if not groups:
        raise ValueError("empty dispatch")
    if slot_budget < 1 or slot_budget > d.slot_total():
        raise ValueError("slot_budget out of range")
    if launches < 1:
        raise ValueError("launches must be >= 1")
    c = Cost()
    for s, count in groups:
        if count < 1 or min(s) < 1:
            raise ValueError("invalid kernel group")
        c.flops += count * gemm_flops(s)
        c.bytes += count * gemm_bytes(s)
        c.blocks += count * thread_blocks(s, d)
    c.waves = cdiv(c.blocks, slot_budget)
    eff = float(c.blocks) / float(c.waves * slot_budget)
    compute = float(c.flops) / (d.peak_flops * eff)
    memory = float(c.bytes) / d.mem_bandwidth
    c.duration = float(launches) * d.launch_overhead + max(compute, memory)
    return c


@dataclass
class Request:
    id: int
    tenant: int
    shape: Shape
    enqueue: int = 0
    deadline: int = 0
    layer: int = 0
    pass_index: int = 0


@dataclass
class Policy:
    max_wait: float = 2e-3
    target_batch: int = 1
    allow_variable_size: bool = False
    slo_safety_margin: float = 0.0
    variable_inefficiency: float = 1.10


@dataclass
class SuperKernel:
    signature: str
    members: List[Request]
    uniform: bool
    cost: Cost


class Queue:
    """Shape-grouped FIFO; groups iterate in ascending (m, n, k)."""

    def __init__(self):
        self.groups: Dict[Shape, List[Request]] = {}
        self.order: List[Shape] = []
        self.ids = set()

    def size(self) -> int:
        return sum(len(g) for g in self.groups.values())

    def enqueue(self, r: Request) -> None:
        if min(r.shape) < 1:
            raise ValueError("enqueue: invalid shape")
        if r.id in self.ids:
            raise ValueError(f"enqueue: duplicate request id {r.id}")
        self.ids.add(r.id)
        if r.shape not in self.groups:
            self.groups[r.shape] = []
            insort(self.order, r.shape)
        self.groups[r.shape].append(r)

    def _drop_group(self, s: Shape) -> None:
        del self.groups[s]
        self.order.remove(s)

    def cancel_tenant(self, tenant: int) -> List[Request]:
        out = []
        for s in list(self.order):
            keep = []
            for r in self.groups[s]:
                if r.tenant == tenant:
                    out.append(r)
                    self.ids.discard(r.id)
                else:
                    keep.append(r)
            self.groups[s] = keep
            if not keep:
                self._drop_group(s)
        return out

    def snapshot(self) -> List[Request]:
        return [r for s in self.order for r in self.groups[s]]


def slo_headroom(r: Request, now: int, predicted: float, p: Policy) -> float:
    return to_seconds(r.deadline - now) - predicted * (1.0 + p.slo_safety_margin)


def plan_super_kernel(members: Sequence[Request], uniform: bool, p: Policy, d: Device) -> Cost:
    groups: List[List] = []
    for r in members:
        if groups and groups[-1][0] == r.shape:
            groups[-1][1] += 1
        else:
            groups.append([r.shape, 1])
    c = dispatch_duration([(g[0], g[1]) for g in groups], d, d.slot_total(), 1)
    if not uniform:
        c.duration *= p.variable_inefficiency
    return c


def _signature(members: Sequence[Request], uniform: bool) -> str:
    if uniform:
        return shape_key(members[0].shape) + "*" + str(len(members))
    return "v:" + "".join(shape_key(s) + ";" for s in sorted(r.shape for r in members))


def _make(members: List[Request], uniform: bool, p: Policy, d: Device) -> SuperKernel:
    if uniform:
        uniform = all(r.shape == members[0].shape for r in members)
    return SuperKernel(_signature(members, uniform), members, uniform, plan_super_kernel(members, uniform, p, d))


def form_batches(q: Queue, now: int, p: Policy, d: Device) -> List[SuperKernel]:
    formed: List[SuperKernel] = []
    max_wait_ns = to_ns(p.max_wait)
    if p.allow_variable_size:
        pool = sorted(q.snapshot(), key=lambda r: (r.enqueue, r.id))
        taken = 0
        while taken < len(pool):
            remaining = len(pool) - taken
            size_ok = remaining >= p.target_batch
            forced = now - pool[taken].enqueue >= max_wait_ns
            if not forced:
                predicted = plan_super_kernel(pool[taken:], False, p, d).duration
                for r in pool[taken:]:
                    if slo_headroom(r, now, predicted, p) <= 0:
                        forced = True
                        break
            if not size_ok and not forced:
                break
            chunk: List[Request] = []
            blocks = 0
            while taken < len(pool):
                b = thread_blocks(pool[taken].shape, d)
                if chunk and blocks + b > d.slot_total():
                    break
                if size_ok and not forced and len(chunk) >= p.target_batch:
                    break
                blocks += b
                chunk.append(pool[taken])
                taken += 1
            formed.append(_make(chunk, False, p, d))
        for sk in formed:
            for r in sk.members:
                g = q.groups[r.shape]
                for i, x in enumerate(g):
                    if x.id == r.id:
                        del g[i]
                        q.ids.discard(r.id)
                        break
                if not g:
                    q._drop_group(r.shape)
        return formed
    for s in list(q.order):
        g = q.groups[s]
        wave_cap = max(1, d.slot_total() // thread_blocks(s, d))
        while g:
            n = len(g)
            size_ok = n >= p.target_batch
            forced = now - g[0].enqueue >= max_wait_ns
            if not forced:
                probe = min(n, max(p.target_batch, 1))
                predicted = plan_super_kernel(g[:probe], True, p, d).duration
                forced = any(slo_headroom(r, now, predicted, p) <= 0 for r in g)
            if not size_ok and not forced:
                break
            take = min(p.target_batch if size_ok else n, wave_cap)
            members = g[:take]
            del g[:take]
            for r in members:
                q.ids.discard(r.id)
            formed.append(_make(members, True, p, d))
        if not g:
            q._drop_group(s)
    return formed


@dataclass
class Cache:
    entries: Dict[str, Cost] = field(default_factory=dict)
    hits: int = 0
    misses: int = 0


def dispatch_cost(sk: SuperKernel, cache: Cache, d: Device) -> float:
    dur = sk.cost.duration
    if sk.signature not in cache.entries:
        cache.entries[sk.signature] = sk.cost
        cache.misses += 1
        dur += d.planning_overhead
    else:
        cache.hits += 1
    return dur


@dataclass
class Health:
    tenant: int = 0
    ewma: float = 0.0
    alpha: float = 0.2
    count: int = 0
    evicted: bool = False


def record_latency(h: Health, s: float) -> None:
    if s < 0:
        raise ValueError("negative latency")
    h.ewma = s if h.count == 0 else h.alpha * s + (1.0 - h.alpha) * h.ewma
    h.count += 1


def detect_stragglers(hs: Sequence[Health], ratio: float, min_obs: int) -> List[int]:
    if ratio <= 1.0:
        raise ValueError("threshold_ratio must be > 1")
    peers = sorted(h.ewma for h in hs if not h.evicted and h.count > 0)
    if len(peers) < 2:
        return []
    mid = len(peers) // 2
    median = peers[mid] if len(peers) % 2 else 0.5 * (peers[mid - 1] + peers[mid])
    return [h.tenant for h in hs if not h.evicted and h.count >= min_obs and h.ewma > ratio * median]


def evict(hs: List[Health], q: Queue, tenant: int) -> List[Request]:
    for h in hs:
        if h.tenant == tenant:
            if h.evicted:
                raise ValueError(f"evict: tenant {tenant} already evicted")
            h.evicted = True
            return q.cancel_tenant(tenant)
    raise ValueError(f"evict: unknown tenant {tenant}")


def percentile_nearest_rank(values: Sequence[float], pct: float) -> float:
    if not values:
        raise ValueError("percentile of empty set")
    v = sorted(values)
    rank = int(math.ceil(pct / 100.0 * len(v)))
    rank = min(max(rank, 1), len(v))
    return v[rank - 1]


def geomean(values: Sequence[float]) -> float:
    if not values:
        raise ValueError("geomean of empty set")
    acc = 0.0
    for x in values:
        if x <= 0:
            raise ValueError("geomean requires positive values")
        acc += math.log(x)
    return math.exp(acc / len(values))


def run_space_time(layers: Sequence[Shape], tenants: int, d: Device, policy: Policy, slo: float = 0.1,
                   duration: float = 1.0, concurrency: int = 1, microbench: bool = False,
                   ewma_alpha: float = 0.2, min_obs: int = 10, ratio: float = 1.5, evict_on: bool = True,
                   degrade: Optional[Tuple[int, float, float]] = None) -> dict:
    """Closed-loop space-time engine (sim.cpp:398-581) on a virtual clock."""
    layers = list(layers)[:1] if microbench else list(layers)
    horizon = to_ns(duration)
    slo_ns = to_ns(slo)
    pass_flops = sum(gemm_flops(s) for s in layers)
    state = {"next": 1, "seq": 0}

    def fresh():
        v = state["next"]
        state["next"] += 1
        return v

    def finish(tenant, start, exec_ns):
        if degrade and degrade[0] == tenant and degrade[1] > 1.0 and start >= to_ns(degrade[2]):
            return start + round_half_away(float(exec_ns) * degrade[1])
        return start + exec_ns

    q, cache = Queue(), Cache()
    health = [Health(t, 0.0, ewma_alpha) for t in range(tenants)]
    live: List[Dict[int, list]] = [dict() for _ in range(tenants)]
    counter = [0] * tenants
    heap: list = []
    out = {"events": [], "completions": [], "cancellations": [], "evicted": [], "eviction_times": []}

    def push(time, kind, tenant, req):
        heapq.heappush(heap, (time, kind, tenant, state["seq"], req))
        state["seq"] += 1

    def begin(t, at):
        pi = counter[t]
        counter[t] += 1
        live[t][pi] = [fresh(), at, -1]
        push(at, 0, t, Request(fresh(), t, layers[0], at, at + slo_ns, 0, pi))

    def streams():
        return sum(concurrency for t in range(tenants) if not health[t].evicted)

    for t in range(tenants):
        for _ in range(concurrency):
            begin(t, 0)
    fifo: List[SuperKernel] = []
    busy = False
    running, rs, re_ = None, 0, 0
    max_wait_ns = to_ns(policy.max_wait)
    while heap:
        now = heap[0][0]
        while heap and heap[0][0] == now:
            _, kind, tenant, _, req = heapq.heappop(heap)
            if kind == 0:
                if health[tenant].evicted:
                    out["cancellations"].append(req.id)
                    continue
                q.enqueue(req)
            elif kind == 1:
                busy = False
                exec_ns = re_ - rs
                for r in running.members:
                    done = finish(r.tenant, rs, exec_ns)
                    record_latency(health[r.tenant], to_seconds(done - rs))
                    if health[r.tenant].evicted:
                        continue
                    pr = live[r.tenant].get(r.pass_index)
                    if pr is None:
                        continue
                    if pr[2] < 0:
                        pr[2] = rs
                    if r.layer + 1 < len(layers):
                        push(done, 0, r.tenant, replace(r, id=fresh(), shape=layers[r.layer + 1], enqueue=done,
                                                        layer=r.layer + 1))
                    else:
                        out["completions"].append({"id": pr[0], "tenant": r.tenant, "enqueue": pr[1],
                                                   "dispatch": pr[2], "complete": done,
                                                   "slo_met": (done - pr[1]) <= slo_ns, "flops": pass_flops})
                        del live[r.tenant][r.pass_index]
                        begin(r.tenant, done)
                if evict_on:
                    for t in detect_stragglers(health, ratio, min_obs):
                        out["evicted"].append(t)
                        out["eviction_times"].append(now)
                        for r in evict(health, q, t):
                            out["cancellations"].append(r.id)
                        live[t].clear()
        if busy:
            continue
        if not fifo and now >= horizon:
            continue
        if not fifo:
            pol = replace(policy)
            live_streams = max(1, streams())
            pol.target_batch = live_streams if pol.target_batch == 0 else min(pol.target_batch, live_streams)
            fifo.extend(form_batches(q, now, pol, d))
        if fifo:
            sk = fifo.pop(0)
            end = now + to_ns(dispatch_cost(sk, cache, d))
            out["events"].append({"start": now, "end": end, "flops": sk.cost.flops,
                                  "occupancy": float(sk.cost.blocks) / float(sk.cost.waves * d.slot_total()),
                                  "members": [r.id for r in sk.members]})
            busy, running, rs, re_ = True, sk, now, end
            push(end, 1, 0, None)
        elif q.size() and now < horizon:
            pol = replace(policy)
            if pol.target_batch == 0:
                pol.target_batch = max(1, streams())
            wake = None
            for s in q.order:
                g = q.groups[s]
                w = g[0].enqueue + max_wait_ns
                wake = w if wake is None else min(wake, w)
                probe = min(len(g), max(pol.target_batch, 1))
                pred = plan_super_kernel(g[:probe], True, pol, d).duration
                pred_ns = to_ns(pred * (1.0 + pol.slo_safety_margin))
                for r in g:
                    wake = min(wake, r.deadline - pred_ns)
            if wake is not None:
                push(max(wake, now + 1), 2, 0, None)
    out["cache_hits"], out["cache_misses"] = cache.hits, cache.misses
    return out
