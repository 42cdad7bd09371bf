"""Test helpers: the compiled reference (oracle/_ref/libgpumux_ref.so) through
its JSON shim, scripted-input generators shared by the golden generator and
the parity tests, and a driver that replays a session on the product."""
from __future__ import annotations

import ctypes
import json
import os
import random
from typing import List, Optional

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libgpumux_ref.so")
GOLDEN = os.path.join(HERE, "golden")

_ref = None


def have_ref() -> bool:
    return os.path.exists(REF_LIB)


def ref_call(req: dict) -> dict:
    """One call into the unmodified reference library (JSON in, JSON out)."""
    global _ref
    if _ref is None:
        _ref = ctypes.CDLL(REF_LIB)
        _ref.gm_ref_call.restype = ctypes.c_char_p
        _ref.gm_ref_call.argtypes = [ctypes.c_char_p]
    return json.loads(_ref.gm_ref_call(json.dumps(req).encode()))


# ------------------------------------------------------------------ inputs

DEVICES = {
    "default": {},
    "sched": {"launch_overhead": 5e-6, "planning_overhead": 50e-6},  # test_scheduler.cpp:11-16
    "v100": {"launch_overhead": 2.2e-06, "context_switch_overhead": 0.000196875, "space_sched_penalty": 1.55,
             "launch_serialization": 1.0},  # device.cpp:41-59
    "b200": {"peak_flops": 1388.8e12, "mem_bandwidth": 6546.9e9, "sm_count": 148, "blocks_per_sm": 1,
             "launch_overhead": 2.0e-6, "context_switch_overhead": 25e-6, "planning_overhead": 20e-6,
             "mem_capacity": 180e9, "process_context_bytes": 500e6, "tile_m": 128, "tile_n": 256,
             "space_sched_penalty": 1.0, "launch_serialization": 1.0},
}

SHAPES = [[256, 128, 1152], [64, 64, 64], [512, 1, 512], [256, 256, 256], [1024, 64, 147], [16, 256, 2304],
          [4, 2048, 512], [1, 1000, 2048], [6272, 128, 1152], [392, 512, 4608], [100352, 64, 147]]


def random_groups(rng: random.Random) -> list:
    n = rng.randint(1, 5)
    return [{"shape": [rng.randint(1, 3000), rng.randint(1, 3000), rng.randint(1, 5000)], "count": rng.randint(1, 40)}
            for _ in range(n)]


def random_session(seed: int, n_steps: int = 120, tenants: int = 8, variable: Optional[bool] = None) -> List[dict]:
    """A scripted queue session: bursty enqueues, formations at advancing
    times with random policies, cost lookups, monitor updates, evictions."""
    rng = random.Random(seed)
    steps: List[dict] = []
    now = 0
    next_id = 1
    evicted = set()
    shapes = rng.sample(SHAPES, 4)
    for _ in range(n_steps):
        op = rng.random()
        if op < 0.55:
            for _ in range(rng.randint(1, 6)):
                steps.append({"do": "enqueue", "request": {
                    "id": next_id, "tenant": rng.randrange(tenants), "shape": rng.choice(shapes),
                    "enqueue": now - rng.randrange(0, 3_000_000), "deadline": now + rng.randrange(-500_000, 60_000_000),
                    "layer": rng.randrange(4), "pass": rng.randrange(3)}})
                next_id += 1
        elif op < 0.80:
            now += rng.randrange(0, 2_500_000)
            var = rng.random() < 0.4 if variable is None else variable
            pol = {"max_wait": rng.choice([1e-3, 2e-3, 5e-4]), "target_batch": rng.randint(1, 24),
                   "allow_variable_size": var, "slo_safety_margin": rng.choice([0.0, 0.25, 0.5]),
                   "variable_inefficiency": rng.choice([1.10, 1.25])}
            steps.append({"do": "form", "now": now, "policy": pol})
            for i in range(rng.randint(0, 3)):
                steps.append({"do": "cost", "plan": i})
        elif op < 0.88:
            steps.append({"do": "record", "tenant": rng.randrange(tenants), "seconds": rng.uniform(1e-4, 5e-3)})
        elif op < 0.93:
            steps.append({"do": "detect", "ratio": rng.choice([1.2, 1.5, 2.0]), "min_obs": rng.randint(1, 4)})
        elif op < 0.97:
            t = rng.randrange(tenants)
            steps.append({"do": "cancel", "tenant": t})
        else:
            t = rng.randrange(tenants + 1)
            steps.append({"do": "evict", "tenant": t})
            evicted.add(t)
    return steps
