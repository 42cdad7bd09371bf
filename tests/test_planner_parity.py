"""Plan parity: product planner == compiled reference == Python oracle.

Goldens (tests/golden/*.json) were produced by the unmodified reference
(tests/golden/make_golden.py); the live tests re-run the reference through
oracle/_ref when it is built and cover larger randomized inputs.
"""
import json
import os
import random

import pytest

import refshim
from refshim import DEVICES, GOLDEN, random_groups, random_session
from replay import oracle_session, product_device, product_session, same
from paper_1901_00041_b200 import scheduler as S
from paper_1901_00041_b200.sim import DegradationSpec, SpaceTimeConfig, simulate_space_time


def load(name):
    with open(os.path.join(GOLDEN, name + ".json")) as f:
        return json.load(f)


def product_cost(case):
    c = case["input"]
    groups = [S.KernelGroup(S.GemmShape(*g["shape"]), g.get("count", 1)) for g in c["groups"]]
    try:
        k = S.dispatch_duration(groups, product_device(c["device"]), c["slot_budget"], c.get("launches", 1))
        return {"flops": k.flops, "bytes": k.bytes, "blocks": k.blocks, "duration": k.duration, "waves": k.waves}
    except ValueError as e:
        return {"error": str(e)}


@pytest.mark.parametrize("i", range(len(load("cost"))))
def test_dispatch_duration_golden(i):
    case = load("cost")[i]
    assert product_cost(case) == case["output"]  # bit-exact doubles


@pytest.mark.parametrize("i", range(len(load("sessions"))))
def test_scheduler_session_golden(i):
    case = load("sessions")[i]
    got = product_session(case["steps"], case["device"])
    ok, at, x, y = same(got, case["output"])
    assert ok, f"step {at}: product {x} != reference {y}"


def product_trace(c):
    layers = [S.GemmShape(*s) for s in c["layers"]]
    deg = c.get("degrade")
    cfg = SpaceTimeConfig(device=product_device(c["device"]), layers=layers, tenants=c["tenants"],
                          duration=c["duration"], warmup=0.1 * c["duration"], microbench=c.get("microbench", False),
                          slo_latency=0.05, scheduler=S.BatchPolicy(target_batch=0),
                          degradation=DegradationSpec(deg["tenant"], deg["slowdown"], deg["start"]) if deg else None)
    return simulate_space_time(cfg)


def assert_trace_equal(tr, ref):
    assert len(tr.events) == len(ref["events"])
    for a, b in zip(tr.events, ref["events"]):
        assert (a.start, a.end, a.flops, a.occupancy, a.member_requests) == \
            (b["start"], b["end"], b["flops"], b["occupancy"], b["members"])
    assert len(tr.completions) == len(ref["completions"])
    for a, b in zip(tr.completions, ref["completions"]):
        assert (a.request_id, a.tenant_index, a.enqueue_time, a.dispatch_time, a.complete_time, a.slo_met,
                a.flops) == (b["id"], b["tenant"], b["enqueue"], b["dispatch"], b["complete"], b["slo_met"],
                             b["flops"])
    assert tr.cancellations == len(ref["cancellations"])
    assert tr.evicted_tenants == ref["evicted"] and tr.eviction_times == ref["eviction_times"]
    assert (tr.cache_hits, tr.cache_misses) == (ref["cache_hits"], ref["cache_misses"])
    assert (tr.dispatched_flops, tr.completed_kernel_flops) == (ref["dispatched_flops"], ref["completed_flops"])


@pytest.mark.parametrize("i", range(len(load("sim"))))
def test_space_time_driver_golden(i):
    case = load("sim")[i]
    assert_trace_equal(product_trace(case["input"]), case["output"])


def test_metrics_and_shapes_golden():
    g = load("misc")
    for c in g["percentile"]:
        assert S.percentile_nearest_rank(c["values"], c["pct"]) == c["output"]["value"]
    for c in g["geomean"]:
        assert S.geomean(c["values"]) == c["output"]["value"]
    for c in g["im2col"]:
        try:
            got = list(S.im2col_gemm_dims(S.ConvSpec(*c["conv"])).__dict__.values())
            assert got == c["output"]["shape"]
        except ValueError as e:
            assert c["output"]["error"] == str(e)
    for c in g["thread_blocks"]:
        assert S.thread_blocks(S.GemmShape(*c["shape"]), product_device(c["device"])) == c["output"]["blocks"]


# ------------------------------------------------------------ live reference A/B

def test_live_dispatch_duration_randomized(ref):
    rng = random.Random(99)
    for _ in range(300):
        dev = rng.choice(list(DEVICES))
        case = {"input": {"device": dev, "groups": random_groups(rng), "slot_budget": rng.randint(1, 148)}}
        out = ref({"op": "dispatch_duration", "groups": case["input"]["groups"], "device": DEVICES[dev],
                   "slot_budget": case["input"]["slot_budget"]})
        assert product_cost(case) == out


@pytest.mark.parametrize("seed", range(100, 112))
def test_live_sessions_randomized(ref, seed):
    dev = list(DEVICES)[seed % len(DEVICES)]
    steps = random_session(seed, n_steps=250)
    out = ref({"op": "session", "device": DEVICES[dev], "tenants": 8, "steps": steps})["steps"]
    ok, at, x, y = same(product_session(steps, dev), out)
    assert ok, f"seed {seed} step {at}: product {x} != reference {y}"


@pytest.mark.parametrize("tenants,layers,dev,dur", [
    (10, "resnet50", "v100", 0.2),     # the wave-cap / max_wait stall case (SURVEY §7 hard part 5)
    (4, "mobilenetv2", "v100", 0.05),
    (64, "conv2_2", "v100", 0.02),
    (120, "conv2_2", "v100", 0.02),
    (4, "resnet50", "b200", 0.01),
])
def test_live_space_time_driver(ref, tenants, layers, dev, dur):
    from paper_1901_00041_b200.workload import find_preset
    name = {"conv2_2": "resnet18-conv2_2"}.get(layers, layers)
    shapes = [[s.m, s.n, s.k] for s in find_preset(name).layers]
    c = {"layers": shapes, "tenants": tenants, "duration": dur, "device": dev, "microbench": layers == "conv2_2"}
    out = ref({"op": "run_space_time", "layers": shapes, "tenants": tenants, "duration": dur, "warmup": 0.1 * dur,
               "microbench": c["microbench"], "device": DEVICES[dev], "scheduler": {"target_batch": 0},
               "slo_latency": 0.05})
    assert_trace_equal(product_trace(c), out)


def test_oracle_restatement_matches_goldens():
    """The Python oracle (oracle/planner_ref.py) is pinned to the reference."""
    for case in load("sessions"):
        ok, at, x, y = same(oracle_session(case["steps"], case["device"]), case["output"])
        assert ok, f"oracle step {at}: {x} != {y}"
