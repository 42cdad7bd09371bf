"""Regenerate tests/golden/*.json from the compiled, unmodified reference
(oracle/_ref/libgpumux_ref.so; build it with `make -C oracle ref`).

The fixtures pin the oracle restatement (oracle/planner_ref.py) and the
product planner to the reference's own outputs.  They are small on purpose;
the live A/B tests in tests/test_planner_parity.py cover larger inputs
whenever oracle/_ref is present.

  python tests/golden/make_golden.py
"""
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from refshim import DEVICES, SHAPES, random_groups, random_session, ref_call  # noqa: E402


def cost_cases():
    rng = random.Random(20190101)
    cases = []
    # the reference unit tests' known answers (test_cost_model.cpp:25-132)
    for r in (1, 2, 10, 20, 21, 40, 120):
        cases.append({"device": "v100", "groups": [{"shape": [256, 128, 1152], "count": r}], "slot_budget": 160})
    for _ in range(60):
        dev = rng.choice(list(DEVICES))
        slots = {"b200": 148, "default": 160}.get(dev, 160)
        cases.append({"device": dev, "groups": random_groups(rng), "slot_budget": rng.randint(1, slots),
                      "launches": rng.randint(1, 4)})
    out = []
    for c in cases:
        res = ref_call({"op": "dispatch_duration", "groups": c["groups"], "device": DEVICES[c["device"]],
                        "slot_budget": c["slot_budget"], "launches": c.get("launches", 1)})
        out.append({"input": c, "output": res})
    return out


def session_cases():
    out = []
    for seed, dev, var in [(1, "sched", False), (2, "sched", True), (3, "v100", None), (4, "b200", None),
                           (5, "default", None), (6, "b200", True)]:
        steps = random_session(seed, n_steps=90)
        res = ref_call({"op": "session", "device": DEVICES[dev], "tenants": 8, "steps": steps})
        out.append({"device": dev, "steps": steps, "output": res["steps"]})
    return out


def sim_cases():
    cases = [
        {"name": "conv2_2 microbench R=16", "layers": [[256, 128, 1152]], "tenants": 16, "duration": 0.01,
         "microbench": True, "device": "v100"},
        {"name": "conv2_2 microbench R=40", "layers": [[256, 128, 1152]], "tenants": 40, "duration": 0.01,
         "microbench": True, "device": "v100"},
        {"name": "resnet18@128 x2 (C1 twin)", "layers": [[4096, 64, 147]] + [[1024, 64, 576]] * 4 +
         [[256, 128, 576], [256, 128, 1152], [256, 128, 64], [256, 128, 1152], [256, 128, 1152],
          [64, 256, 1152], [64, 256, 2304], [64, 256, 128], [64, 256, 2304], [64, 256, 2304],
          [16, 512, 2304], [16, 512, 4608], [16, 512, 256], [16, 512, 4608], [16, 512, 4608]],
         "tenants": 2, "duration": 0.005, "device": "v100"},
        {"name": "mixed 3 tenants, degraded tenant 1, eviction", "layers": [[256, 128, 1152], [64, 64, 64]],
         "tenants": 3, "duration": 0.01, "device": "sched",
         "degrade": {"tenant": 1, "slowdown": 3.0, "start": 0.002}},
        {"name": "b200 profile, 4 tenants", "layers": [[100352, 64, 147], [25088, 64, 576], [392, 512, 4608]],
         "tenants": 4, "duration": 0.003, "device": "b200"},
    ]
    out = []
    for c in cases:
        req = {"op": "run_space_time", "layers": c["layers"], "tenants": c["tenants"], "duration": c["duration"],
               "warmup": 0.1 * c["duration"], "microbench": c.get("microbench", False),
               "device": DEVICES[c["device"]], "scheduler": {"target_batch": 0}, "slo_latency": 0.05}
        if "degrade" in c:
            req["degrade"] = c["degrade"]
        out.append({"input": c, "output": ref_call(req)})
    return out


def misc_cases():
    rng = random.Random(7)
    vals = [[rng.uniform(1e-4, 1e-2) for _ in range(rng.randint(1, 200))] for _ in range(10)]
    return {
        "percentile": [{"values": v, "pct": p, "output": ref_call({"op": "percentile", "values": v, "pct": p})}
                       for v in vals for p in (50.0, 99.0)],
        "geomean": [{"values": v, "output": ref_call({"op": "geomean", "values": v})} for v in vals],
        "im2col": [{"conv": c, "output": ref_call({"op": "im2col", "conv": c})}
                   for c in ([16, 16, 3, 3, 128, 128, 1, 1], [224, 224, 7, 7, 3, 64, 2, 3], [56, 56, 3, 3, 64, 128, 2, 1],
                             [3, 3, 3, 3, 1, 1, 1, 0], [2, 2, 5, 5, 1, 1, 1, 0])],
        "thread_blocks": [{"shape": s, "device": d, "output": ref_call({"op": "thread_blocks", "shape": s,
                                                                       "device": DEVICES[d]})}
                          for s in SHAPES for d in ("v100", "b200")],
    }


def main():
    for name, fn in (("cost", cost_cases), ("sessions", session_cases), ("sim", sim_cases), ("misc", misc_cases)):
        path = os.path.join(HERE, f"{name}.json")
        with open(path, "w") as f:
            json.dump(fn(), f, separators=(",", ":"))
        print(f"wrote {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    main()
