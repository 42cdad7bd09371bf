"""Scheduler behaviour (proj/tests/test_scheduler.cpp, all 15 cases) through the C-ABI."""
import random

import pytest

from paper_1901_00041_b200.scheduler import (BatchPolicy, DeviceSpec, GemmShape, KernelGroup, KernelRequest,
                                             RequestQueue, SuperKernelCache, TenantHealth, detect_stragglers,
                                             dispatch_cost, dispatch_duration, evict, form_batches, record_latency,
                                             slo_headroom, to_ns)

CONV = GemmShape(256, 128, 1152)


def sched_device():  # test_scheduler.cpp:11-16
    return DeviceSpec(launch_overhead=5e-6, planning_overhead=50e-6)


def req(i, tenant, shape, enqueue, deadline):
    return KernelRequest(request_id=i, tenant_index=tenant, shape=shape, enqueue_time=enqueue, slo_deadline=deadline)


def pol(target, max_wait=2e-3):
    return BatchPolicy(max_wait=max_wait, target_batch=target)


def test_enqueue_groups_by_shape_and_rejects_duplicates():
    q = RequestQueue()
    q.enqueue(req(1, 0, GemmShape(8, 8, 8), 0, 1000000))
    assert q.size() == 1
    with pytest.raises(ValueError):
        q.enqueue(req(1, 1, GemmShape(8, 8, 8), 0, 1000000))
    q.enqueue(req(2, 1, GemmShape(8, 8, 8), 10, 1000000))
    assert len(q.groups()) == 1
    q.enqueue(req(3, 0, GemmShape(16, 16, 16), 20, 1000000))
    assert len(q.groups()) == 2


def test_twenty_same_shape_fuse_into_one_launch():
    q = RequestQueue()
    for i in range(20):
        q.enqueue(req(i + 1, i, CONV, 0, to_ns(0.05)))
    f = form_batches(q, 0, pol(20), sched_device())
    assert len(f) == 1 and len(f[0].members) == 20 and f[0].uniform
    assert f[0].planned_cost.blocks == 160 and q.empty()


def test_aged_singleton_dispatches_alone():
    q = RequestQueue()
    q.enqueue(req(1, 0, CONV, 0, to_ns(0.05)))
    assert form_batches(q, to_ns(1e-3), pol(20), sched_device()) == []
    f = form_batches(q, to_ns(2e-3), pol(20), sched_device())
    assert len(f) == 1 and len(f[0].members) == 1


def test_groups_trigger_independently():
    q = RequestQueue()
    q.enqueue(req(1, 0, GemmShape(64, 64, 64), 0, to_ns(0.05)))
    q.enqueue(req(2, 1, CONV, 0, to_ns(0.05)))
    q.enqueue(req(3, 2, CONV, 0, to_ns(0.05)))
    f = form_batches(q, 0, pol(2), sched_device())
    assert len(f) == 1 and len(f[0].members) == 2 and f[0].members[0].shape == CONV
    assert q.size() == 1


def test_oldest_first_within_a_group():
    q = RequestQueue()
    for i in range(6):
        q.enqueue(req(i + 1, i, CONV, i * 100, to_ns(0.05)))
    f = form_batches(q, 1000, pol(4), sched_device())
    assert [m.request_id for m in f[0].members] == [1, 2, 3, 4]
    left = [r for g in q.groups().values() for r in g]
    assert all(t.enqueue_time <= w.enqueue_time for t in f[0].members for w in left)


def test_chunks_cap_at_one_wave():
    q = RequestQueue()
    for i in range(30):
        q.enqueue(req(i + 1, i, CONV, 0, to_ns(0.05)))
    f = form_batches(q, 0, pol(30), sched_device())
    assert len(f) == 1 and len(f[0].members) == 20 and q.size() == 10


def test_aged_group_flushes_in_capped_chunks():  # aged 45 at target 64 -> 20, 20, 5
    q = RequestQueue()
    for i in range(45):
        q.enqueue(req(i + 1, i, CONV, 0, to_ns(0.05)))
    f = form_batches(q, to_ns(2e-3), pol(64), sched_device())
    assert [len(s.members) for s in f] == [20, 20, 5]


def test_slo_headroom_arithmetic():
    p = BatchPolicy()
    r = req(1, 0, GemmShape(8, 8, 8), 0, to_ns(10e-3))
    assert slo_headroom(r, 0, 1e-3, p) == pytest.approx(9e-3)
    r.slo_deadline = 0
    assert slo_headroom(r, 0, 1e-3, p) < 0
    p.slo_safety_margin = 0.5
    r.slo_deadline = to_ns(3e-3)
    assert slo_headroom(r, 0, 2e-3, p) == pytest.approx(0.0)


def test_slo_breach_forces_formation():
    q = RequestQueue()
    q.enqueue(req(1, 0, CONV, 0, 1000))
    f = form_batches(q, 500, pol(20), sched_device())
    assert len(f) == 1 and len(f[0].members) == 1


def test_variable_size_batching_tax():
    d = sched_device()
    p = pol(2)
    p.allow_variable_size = True
    q = RequestQueue()
    q.enqueue(req(1, 0, CONV, 0, to_ns(0.05)))
    q.enqueue(req(2, 1, GemmShape(64, 64, 64), 0, to_ns(0.05)))
    f = form_batches(q, 0, p, d)
    assert len(f) == 1 and len(f[0].members) == 2 and not f[0].uniform
    raw = dispatch_duration([KernelGroup(CONV, 1), KernelGroup(GemmShape(64, 64, 64), 1)], d, d.slot_total(), 1)
    assert f[0].planned_cost.duration == pytest.approx(raw.duration * 1.10)
    assert f[0].shape_signature == "v:64x64x64;256x128x1152;"


def test_dispatch_cost_planning_on_miss_only():
    d = sched_device()
    q = RequestQueue()
    for i in range(4):
        q.enqueue(req(i + 1, i, CONV, 0, to_ns(0.05)))
    f = form_batches(q, 0, pol(2), d)
    assert len(f) == 2
    cache = SuperKernelCache()
    first, second = dispatch_cost(f[0], cache, d), dispatch_cost(f[1], cache, d)
    assert first == pytest.approx(second + d.planning_overhead)
    assert (cache.hits, cache.misses) == (1, 1)


def test_ewma_monitor():
    h = TenantHealth(ewma_alpha=0.5)
    record_latency(h, 4e-3)
    assert h.ewma_latency == pytest.approx(4e-3)
    record_latency(h, 8e-3)
    assert h.ewma_latency == pytest.approx(6e-3)
    for _ in range(100):
        record_latency(h, 2e-3)
    assert h.ewma_latency == pytest.approx(2e-3, rel=1e-6) and h.observed_count == 102
    with pytest.raises(ValueError, match="negative latency"):
        record_latency(h, -1.0)


def mk(idx, ewma, count, evicted=False):
    return TenantHealth(tenant_index=idx, ewma_latency=ewma, observed_count=count, evicted=evicted)


def test_straggler_detector():
    base = [mk(i, 1e-3, 50) for i in range(9)]
    assert detect_stragglers(base, 1.5, 10) == []
    assert detect_stragglers(base + [mk(9, 2e-3, 50)], 1.5, 10) == [9]
    assert detect_stragglers(base + [mk(9, 2e-3, 5)], 1.5, 10) == []
    assert detect_stragglers([mk(0, 5e-3, 50)], 1.5, 10) == []
    assert detect_stragglers([mk(0, 5e-3, 50), mk(1, 1e-3, 50, True)], 1.5, 10) == []
    with pytest.raises(ValueError, match="threshold_ratio must be > 1"):
        detect_stragglers(base, 1.0, 10)


def test_evict_is_terminal_and_guarded():
    hs = [TenantHealth(tenant_index=i) for i in range(3)]
    q = RequestQueue()
    q.enqueue(req(1, 0, GemmShape(8, 8, 8), 0, 1000000))
    q.enqueue(req(2, 1, GemmShape(8, 8, 8), 0, 1000000))
    q.enqueue(req(3, 1, GemmShape(16, 16, 16), 0, 1000000))
    assert len(evict(hs, q, 1)) == 2 and hs[1].evicted and q.size() == 1
    with pytest.raises(ValueError, match="evict: tenant 1 already evicted"):
        evict(hs, q, 1)
    with pytest.raises(ValueError, match="evict: unknown tenant 9"):
        evict(hs, q, 9)


def test_cancel_tenant_removes_only_that_tenant():
    q = RequestQueue()
    for i in range(10):
        q.enqueue(req(i + 1, i % 2, GemmShape(8, 8, 8), i, 1000000))
    assert len(q.cancel_tenant(0)) == 5 and q.size() == 5
    assert all(r.tenant_index == 1 for g in q.groups().values() for r in g)


def test_randomized_traffic_never_waits_beyond_max_wait():  # test_scheduler.cpp:259-301, seed 1234
    d = sched_device()
    p = pol(16, 1e-3)
    mw = to_ns(p.max_wait)
    rng = random.Random(1234)
    q = RequestQueue()
    nid, now, dispatched = 1, 0, 0
    shapes = [CONV, GemmShape(64, 64, 64), GemmShape(512, 1, 512)]
    for _ in range(3000):
        for _ in range(rng.randrange(6)):
            q.enqueue(req(nid, rng.randrange(8), shapes[rng.randrange(3)], now, now + to_ns(0.1)))
            nid += 1
        for sk in form_batches(q, now, p, d):
            for r in sk.members:
                assert now - r.enqueue_time <= mw
                dispatched += 1
        nxt = now + rng.randrange(200000)
        for g in q.groups().values():
            nxt = min(nxt, g[0].enqueue_time + mw)
        now = max(nxt, now + 1)
    assert dispatched > 5000
    assert all(now - r.enqueue_time <= mw for g in q.groups().values() for r in g)


def test_max_waves_extension_lifts_the_cap_and_defaults_to_parity():
    q = RequestQueue()
    for i in range(30):
        q.enqueue(req(i + 1, i, CONV, 0, to_ns(0.05)))
    f = form_batches(q, 0, BatchPolicy(target_batch=30, max_waves=2), sched_device())
    assert [len(s.members) for s in f] == [30]
    assert BatchPolicy().max_waves == 1
