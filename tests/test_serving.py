"""Real-clock serving (gm_serve): the run_space_time loop of the reference
(proj/src/sim.cpp:398-581) driven by real arrivals and CUDA-event
completions.  Checks the accounting invariants, the dynamic batcher's
triggers, and that served outputs are the round program's (bit-identical to
a directly launched round of the same members)."""
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _layers():
    from paper_1901_00041_b200 import workload as W
    return W.resnet18(128, classifier=False)[:6]


def _engine(**kw):
    from paper_1901_00041_b200.engine import ServeTenant, ServingEngine
    specs = [ServeTenant(_layers(), max_batch=4, **kw) for _ in range(3)]
    return ServingEngine(specs, device_index=0)


def test_closed_loop_accounting():
    eng = _engine(concurrency=2, slo_latency=0.05)
    r = eng.serve(duration=0.6, warmup=0.1)
    s = r.stats
    assert s["queries"] > 50 and s["rounds"] > 10
    assert len(r.latencies_ms) == s["queries"]
    assert s["dispatched_queries"] >= s["queries"]
    assert 0 < s["p50_ms"] <= s["p99_ms"] <= s["max_ms"]
    # closed loop, concurrency 2 per tenant: a dispatch never holds more than 2 queries of a tenant
    assert 1 <= s["mean_queries_per_round"] <= 6
    assert 0.0 <= s["slo_violation_frac"] <= 1.0
    # member sets repeat: plans and device tables come from the cache after the first few
    assert s["plan_misses"] <= 16 and s["plan_hits"] > s["plan_misses"]
    flops = sum(eng.flops_per_query(i) for i in range(3)) / 3
    assert s["tflops"] == pytest.approx(s["queries"] * flops / s["window_s"] / 1e12, rel=1e-6)
    # the dispatch trace (gm_serve_trace): one event per round, in dispatch order
    ev = r.dispatches
    assert len(ev) == s["rounds"]
    assert all(e["launches"] == 1 and e["tiles"] > 0 and 1 <= e["tenants"] <= 3 for e in ev)
    assert all(0 < e["device_ms"] and e["start_ns"] < e["end_ns"] for e in ev)
    assert [e["start_ns"] for e in ev] == sorted(e["start_ns"] for e in ev)
    assert sum(e["queries"] for e in ev) == s["dispatched_queries"]


def test_poisson_low_rate_dispatches_singletons_after_max_wait():
    # 40 queries/s per tenant with a 1 ms age trigger: queries rarely coincide,
    # so almost every dispatch carries one query and waits ~max_wait first
    eng = _engine(rate_qps=40.0, slo_latency=0.5)
    r = eng.serve(duration=1.0, warmup=0.1, max_wait=0.001, seed=7)
    s = r.stats
    assert s["queries"] > 40
    assert s["mean_queries_per_round"] < 1.5
    assert s["p50_ms"] >= 1.0  # the age trigger held each lone query ~1 ms
    assert s["slo_violation_frac"] == 0.0


def test_served_outputs_match_direct_round():
    """The serving loop launches the same round programs as gm_dispatch_round."""
    from paper_1901_00041_b200.engine import ServeTenant, ServingEngine
    specs = [ServeTenant(_layers(), max_batch=2, batches=[2], concurrency=2) for _ in range(2)]
    eng = ServingEngine(specs, device_index=0)
    eng.serve(duration=0.2, warmup=0.05)
    torch.cuda.synchronize()
    served = [m.query_output.clone() for m in eng.models]
    for m in eng.models:
        m.query_output.zero_()
    tids = [vs[0][1] for vs in eng._variants]
    rnd = eng.ctx.plan_round(tids, 0)
    s = torch.cuda.Stream()
    rnd.launch_round(s.cuda_stream)
    torch.cuda.synchronize()
    for a, m in zip(served, eng.models):
        assert torch.equal(a, m.query_output)


def test_degraded_tenant_is_detected_and_evicted():
    """inject_degradation on real hardware (sim.cpp:60-68, 98-110): tenant 1's
    observed completions stretch x3 after 0.1 s; the EWMA monitor flags it
    against the median of its peers (detect_stragglers, scheduler.cpp:246-271)
    and evicts it -- terminal, its queries stop while the others keep serving."""
    eng = _engine(concurrency=1, slo_latency=0.5)
    r = eng.serve(duration=0.8, warmup=0.05, degrade=(1, 3.0, 0.1))
    s = r.stats
    assert s["evicted"] == 1 and s["evicted_mask"] == 0b10
    assert s["queries"] > 50  # tenants 0 and 2 kept serving
    clean = eng.serve(duration=0.4, warmup=0.05)
    assert clean.stats["evicted"] == 0


def _expected_slot_outputs(eng, i):
    """Every I/O slot's result as a directly launched max-batch round of tenant
    i computes it (slot inputs copied in bmax at a time)."""
    spec, m = eng.specs[i], eng.models[i]
    bmax = spec.max_batch
    assert spec.io_slots % bmax == 0
    rnd = eng.ctx.plan_round([eng._variants[i][-1][1]], 0)
    s = torch.cuda.Stream()
    out = []
    for j0 in range(0, spec.io_slots, bmax):
        m.query_input.view(bmax, -1).copy_(eng.host_inputs[i][j0:j0 + bmax])
        torch.cuda.synchronize()
        rnd.launch_round(s.cuda_stream)
        torch.cuda.synchronize()
        out.append(m.query_output.reshape(bmax, -1).cpu().clone())
    return torch.cat(out)


def test_data_bearing_queries_get_their_own_results():
    """Per-query I/O inside gm_serve: each query's input is copied in from its
    host slot before its dispatch and its result copied out after, so every
    slot ends up holding the model applied to that slot's input, whatever
    batch / dispatch the query rode in."""
    from paper_1901_00041_b200.engine import ServeTenant, ServingEngine
    specs = [ServeTenant(_layers(), max_batch=4, concurrency=3, io_slots=8) for _ in range(3)]
    eng = ServingEngine(specs, device_index=0)
    r = eng.serve(duration=0.5, warmup=0.05)
    s = r.stats
    assert s["queries"] > 30
    qin = eng.host_inputs[0][0].numel() * 2
    qout = eng.host_outputs[0][0].numel() * 2
    assert s["h2d_bytes"] == s["dispatched_queries"] * qin
    assert s["d2h_bytes"] == s["dispatched_queries"] * qout
    for i in range(3):
        got = eng.host_outputs[i].clone()
        exp = _expected_slot_outputs(eng, i)
        assert torch.equal(got, exp), f"tenant {i}"


def test_bounded_plan_cache_with_background_planning():
    """Many tenants x batch variants: the formable member sets (3^6 - 1) are
    not pre-warmed; each new set is planned on the worker thread while its
    dispatch runs as single-tenant rounds, and the cache stays bounded (least
    recently used sets dropped).  Results stay correct throughout."""
    from paper_1901_00041_b200.engine import ServeTenant, ServingEngine
    specs = [ServeTenant(_layers(), max_batch=2, batches=[1, 2], rate_qps=900.0, slo_latency=0.2, io_slots=4)
             for _ in range(6)]
    eng = ServingEngine(specs, device_index=0)
    # cap 13: the 12 pinned single-tenant sets plus one, so a second admitted
    # set already evicts (sets are admitted on their second sighting)
    r = eng.serve(duration=1.0, warmup=0.05, max_wait=0.0005, prewarm=0, plan_cache_cap=13, async_plan=True)
    s = r.stats
    assert s["queries"] > 500
    assert s["plan_fallbacks"] > 0 and s["plan_misses"] >= s["plan_fallbacks"]
    assert s["plan_evictions"] > 0 and s["plans_cached"] <= 14  # (+1: a victim may still be in flight)
    launches = [e["launches"] for e in r.dispatches]
    # fallbacks ran as a padded cached superset (one round) or a cover of cached sub-sets
    assert min(launches) == 1 and sum(n > 1 for n in launches) + s["plan_padded"] == s["plan_fallbacks"]
    for i in range(6):
        assert torch.equal(eng.host_outputs[i].clone(), _expected_slot_outputs(eng, i)), f"tenant {i}"


def test_prewarm_scales_past_exhaustive_sets():
    """16 tenants x 2 variants (3^16 sets): pre-warm falls back to the
    single-tenant sets plus the full set instead of refusing."""
    from paper_1901_00041_b200.engine import ServeTenant, ServingEngine
    specs = [ServeTenant(_layers()[:3], max_batch=2, batches=[1, 2], concurrency=2) for _ in range(16)]
    eng = ServingEngine(specs, device_index=0)
    r = eng.serve(duration=0.3, warmup=0.05, prewarm=4096, async_plan=True)
    assert r.stats["queries"] > 50 and r.stats["plans_cached"] >= 33


def test_evicted_tenant_is_readmitted_on_another_gpu():
    """Re-placement instead of terminal eviction (SPEC.md:331's open extension):
    the monitor evicts the degraded tenant on engine A; its variants migrate
    (gm_migrate_tenant: buffers owned by the destination context, weights and
    inputs by peer copy -- NVLink between two GPUs, a device copy on one) to
    engine B on the least-loaded other GPU (GPU 1 when the box has it, else a
    second context on GPU 0), which serves its data-bearing queries; every
    query slot's result equals what the tenant computed on A."""
    from paper_1901_00041_b200.engine import ServeTenant, ServingEngine
    from paper_1901_00041_b200.placement import least_loaded
    specs = [ServeTenant(_layers(), max_batch=4, concurrency=1, slo_latency=0.5, io_slots=4) for _ in range(3)]
    a = ServingEngine(specs, device_index=0)
    r = a.serve(duration=0.8, warmup=0.05, degrade=(1, 3.0, 0.1))
    assert r.stats["evicted_mask"] == 0b10
    n_gpu = torch.cuda.device_count()
    target = least_loaded([(3, 0)] + [(0, 0)] * (n_gpu - 1), exclude=[0]) if n_gpu > 1 else 0
    b = ServingEngine([ServeTenant(_layers(), max_batch=4, concurrency=2)], device_index=target)
    (j,) = a.readmit([1], b)
    rb = b.serve(duration=0.4, warmup=0.05)
    assert rb.stats["queries"] > 20 and rb.stats["evicted"] == 0
    assert torch.equal(b.host_outputs[j].clone(), _expected_slot_outputs(a, 1))
