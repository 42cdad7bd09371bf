"""Plan parity of the planner that drives the GPU (gm_plan_round) against the
reference engine's own driver, run_space_time (proj/src/sim.cpp:398-581),
compiled unmodified in oracle/_ref.

gm_plan_round plans one closed-loop pass per tenant; the reference runs
passes back to back.  For a homogeneous tenant set the reference's first-pass
dispatches must be the product's round, dispatch for dispatch: member
(tenant, layer) lists in order, FLOPs, occupancy, planned duration, and the
virtual start times up to the first pass completion (after it the reference
also forms the next pass's layer-0 super-kernels, which can reorder the tail).
The reference runs with straggler eviction off: a round's plan does not
include the monitor (record_latency / detect_stragglers / evict are pinned by
tests/test_planner_parity.py), and in these saturated closed loops the
reference evicts tenants whose pass lags by one-wave-cap stalls.

The reference trace names members by request id only.  Ids come from one
counter (sim.cpp:87,125): each tenant's first pass takes a pass id and a
request id (start_pass, sim.cpp:419-433); each member completion takes the
next layer's id, or a pass id + request id when the pass ends (sim.cpp:
481-494).  Events complete in dispatch order (one super-kernel in flight,
sim.cpp:512-549), so replaying that id assignment over the trace recovers
every member's (tenant, layer, pass).
"""
import pytest

from refshim import DEVICES
from replay import product_device
from paper_1901_00041_b200 import scheduler as S
from paper_1901_00041_b200 import workload as W
from paper_1901_00041_b200.sim import plan_round_shapes


def reference_first_pass(ref, shapes, tenants, dev, slo, duration):
    out = ref({"op": "run_space_time", "layers": [list(s) for s in shapes], "tenants": tenants,
               "duration": duration, "warmup": 0.0, "microbench": False, "device": DEVICES[dev],
               "scheduler": {"target_batch": 0}, "slo_latency": slo,
               # the monitor is not part of a round's plan (gm_plan_round
               # plans; gm_serve / the C-ABI monitor evict): keep every tenant
               "detector": {"evict_stragglers": False}})
    L = len(shapes)
    nxt = 1
    info = {}
    for t in range(tenants):  # start_pass: pass id, then request id
        info[nxt + 1] = (t, 0, 0)
        nxt += 2
    events = []
    for ev in out["events"]:
        members = [info[i] for i in ev["members"]]
        events.append(dict(ev, who=members))
        for t, l, p in members:  # completion fan-out in member order
            if l + 1 < L:
                info[nxt] = (t, l + 1, p)
                nxt += 1
            else:
                info[nxt + 1] = (t, 0, p + 1)
                nxt += 2
    first_done = min(c["complete"] for c in out["completions"])
    return events, first_done


def product_round(shapes, tenants, dev, slo):
    layers = [S.GemmShape(*s) for s in shapes]
    return plan_round_shapes([(t, layers, slo) for t in range(tenants)], 0, S.BatchPolicy(target_batch=0),
                             product_device(dev))


def occupancy(cost, dev):
    return cost.blocks / (cost.waves * dev.sm_count * dev.blocks_per_sm)


def gemm_list(model, batch):
    if model == "bert":
        layers = W.bert_base_gemms(128, layers=12)
    elif model == "resnet18@128":
        layers = W.resnet18(128, classifier=False)
    elif model == "ref-resnet50":
        return [(s.m, s.n, s.k) for s in W.find_preset("resnet50").layers]
    else:
        layers = W.resnet50(224)
    return [tuple(L.gemm_shape(batch).__dict__.values()) for L in layers]


@pytest.mark.parametrize("model,batch,tenants,dev", [
    ("resnet50@224", 8, 4, "b200"),      # BASELINE configs[1], the headline round
    ("resnet50@224", 1, 4, "b200"),
    ("bert", 4, 16, "b200"),             # configs[3]
    ("bert", 1, 16, "b200"),
    ("resnet18@128", 1, 2, "b200"),      # configs[0] (C1)
    ("resnet18@128", 1, 2, "v100"),
    ("ref-resnet50", 1, 10, "v100"),     # the reference preset, wave-cap stall
    ("resnet50@224", 8, 8, "b200"),      # C5 shard: 8 tenants per GPU
])
def test_plan_round_equals_reference_first_pass(ref, model, batch, tenants, dev):
    shapes = gemm_list(model, batch)
    slo = 0.040
    got = product_round(shapes, tenants, dev, slo)
    span = got[-1].end if got else 0
    events, first_done = reference_first_pass(ref, shapes, tenants, dev, slo, duration=max(4 * span * 1e-9, 1e-3))
    first = [e for e in events if all(p == 0 for _, _, p in e["who"])]
    mixed = [e for e in events if any(p == 0 for _, _, p in e["who"]) and any(p != 0 for _, _, p in e["who"])]
    assert not mixed, "a super-kernel mixed passes (not expected for these layer lists)"
    assert len(first) == len(got)
    d = product_device(dev)
    before = 0
    for i, (g, e) in enumerate(zip(got, first)):
        who = [(r.tenant_index, r.layer_index) for r in g.kernel.members]
        assert who == [(t, l) for t, l, _ in e["who"]], f"dispatch {i}: members differ"
        assert g.kernel.planned_cost.flops == e["flops"]
        assert occupancy(g.kernel.planned_cost, d) == e["occupancy"]
        assert g.end - g.start == e["end"] - e["start"], f"dispatch {i}: planned duration differs"
        if e["start"] < first_done:
            assert (g.start, g.end) == (e["start"], e["end"]), f"dispatch {i}: virtual time differs"
            before += 1
    assert before >= len(got) // 2  # most of the round is time-checked


def test_plan_round_shapes_validates():
    with pytest.raises(ValueError, match="duplicate tenant"):
        plan_round_shapes([(0, [S.GemmShape(8, 8, 8)], 0.1), (0, [S.GemmShape(8, 8, 8)], 0.1)], 0,
                          S.BatchPolicy(), S.b200_profile())
    assert plan_round_shapes([], 0, S.BatchPolicy(), S.b200_profile()) == []


def test_plan_round_heterogeneous_is_topological():
    """The heterogeneous extension (the reference rejects mixed layer lists,
    sim.cpp:28-31): every tenant's layers are dispatched in order, each after
    the previous one's virtual completion."""
    mix = {0: W.resnet50(224), 1: W.vgg16(224), 2: W.mobilenet_v2(224)}
    tenants = [(t, [L.gemm_shape(4) for L in layers], 0.04) for t, layers in mix.items()]
    got = plan_round_shapes(tenants, 0, S.BatchPolicy(target_batch=0), S.b200_profile())
    done = {}
    for g in got:
        for r in g.kernel.members:
            prev = done.get((r.tenant_index, r.layer_index - 1))
            assert r.layer_index == 0 or (prev is not None and prev <= g.start)
            done[(r.tenant_index, r.layer_index)] = g.end
    assert sorted(done) == sorted((t, l) for t, layers in mix.items() for l in range(len(layers)))
