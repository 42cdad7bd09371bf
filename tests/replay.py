"""Replay a scripted scheduler session (tests/refshim.random_session) on the
product C-ABI or on the Python oracle, producing results in the reference
shim's JSON shape so the three can be compared field for field."""
from __future__ import annotations

import os
import sys

from refshim import DEVICES, ROOT

sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import planner_ref as O  # noqa: E402  (test infrastructure)
from paper_1901_00041_b200 import scheduler as S  # noqa: E402


def _cost(c) -> dict:
    return {"flops": c.flops, "bytes": c.bytes, "blocks": c.blocks, "duration": c.duration, "waves": c.waves}


def product_device(name: str) -> S.DeviceSpec:
    return S.DeviceSpec(**DEVICES[name])


def product_session(steps, device: str = "sched", tenants: int = 8, ewma_alpha: float = 0.2) -> list:
    d = product_device(device)
    q = S.RequestQueue()
    cache = S.SuperKernelCache()
    healths = [S.TenantHealth(tenant_index=i, ewma_alpha=ewma_alpha) for i in range(tenants)]
    last = []
    out = []
    for st in steps:
        kind = st["do"]
        try:
            if kind == "enqueue":
                r = st["request"]
                q.enqueue(S.KernelRequest(r["id"], r.get("tenant", 0), S.GemmShape(*r["shape"]), r.get("enqueue", 0),
                                          r.get("deadline", 0), r.get("layer", 0), r.get("pass", 0)))
                res = {"size": q.size()}
            elif kind == "form":
                p = st.get("policy", {})
                last = S.form_batches(q, st["now"], S.BatchPolicy(**p), d)
                res = {"plans": [{"signature": sk.shape_signature, "uniform": sk.uniform,
                                  "cost": _cost(sk.planned_cost), "members": [m.request_id for m in sk.members]}
                                 for sk in last],
                       "remaining": [r.request_id for r in q._snapshot()]}
            elif kind == "cost":
                i = st["plan"]
                if i >= len(last):
                    raise IndexError("vector::_M_range_check")
                dur = S.dispatch_cost(last[i], cache, d)
                res = {"duration": dur, "hits": cache.hits, "misses": cache.misses}
            elif kind == "cancel":
                gone = q.cancel_tenant(st["tenant"])
                res = {"cancelled": [r.request_id for r in gone], "remaining": [r.request_id for r in q._snapshot()]}
            elif kind == "evict":
                gone = S.evict(healths, q, st["tenant"])
                res = {"cancelled": [r.request_id for r in gone], "remaining": [r.request_id for r in q._snapshot()]}
            elif kind == "record":
                h = healths[st["tenant"]]
                S.record_latency(h, st["seconds"])
                res = {"ewma": h.ewma_latency, "count": h.observed_count}
            elif kind == "detect":
                res = {"flagged": S.detect_stragglers(healths, st["ratio"], st["min_obs"])}
            else:
                res = {"error": "unknown step " + kind}
        except (ValueError, IndexError) as e:
            res = {"error": str(e)}
        out.append(res)
    return out


def oracle_device(name: str) -> O.Device:
    return O.Device(**DEVICES[name])


def oracle_session(steps, device: str = "sched", tenants: int = 8, ewma_alpha: float = 0.2) -> list:
    d = oracle_device(device)
    q = O.Queue()
    cache = O.Cache()
    healths = [O.Health(i, 0.0, ewma_alpha) for i in range(tenants)]
    last = []
    out = []
    for st in steps:
        kind = st["do"]
        try:
            if kind == "enqueue":
                r = st["request"]
                q.enqueue(O.Request(r["id"], r.get("tenant", 0), tuple(r["shape"]), r.get("enqueue", 0),
                                    r.get("deadline", 0), r.get("layer", 0), r.get("pass", 0)))
                res = {"size": q.size()}
            elif kind == "form":
                p = st.get("policy", {})
                last = O.form_batches(q, st["now"], O.Policy(**p), d)
                res = {"plans": [{"signature": sk.signature, "uniform": sk.uniform,
                                  "cost": {"flops": sk.cost.flops, "bytes": sk.cost.bytes, "blocks": sk.cost.blocks,
                                           "duration": sk.cost.duration, "waves": sk.cost.waves},
                                  "members": [m.id for m in sk.members]} for sk in last],
                       "remaining": [r.id for r in q.snapshot()]}
            elif kind == "cost":
                i = st["plan"]
                if i >= len(last):
                    raise IndexError("vector::_M_range_check")
                dur = O.dispatch_cost(last[i], cache, d)
                res = {"duration": dur, "hits": cache.hits, "misses": cache.misses}
            elif kind == "cancel":
                gone = q.cancel_tenant(st["tenant"])
                res = {"cancelled": [r.id for r in gone], "remaining": [r.id for r in q.snapshot()]}
            elif kind == "evict":
                gone = O.evict(healths, q, st["tenant"])
                res = {"cancelled": [r.id for r in gone], "remaining": [r.id for r in q.snapshot()]}
            elif kind == "record":
                h = healths[st["tenant"]]
                O.record_latency(h, st["seconds"])
                res = {"ewma": h.ewma, "count": h.count}
            elif kind == "detect":
                res = {"flagged": O.detect_stragglers(healths, st["ratio"], st["min_obs"])}
            else:
                res = {"error": "unknown step " + kind}
        except (ValueError, IndexError) as e:
            res = {"error": str(e)}
        out.append(res)
    return out


def same(a: list, b: list) -> tuple:
    """Compare two result lists; error texts only need to agree on 'is an error'
    except for std::invalid_argument messages, which must match exactly."""
    for i, (x, y) in enumerate(zip(a, b)):
        if "error" in x or "error" in y:
            if ("error" in x) != ("error" in y):
                return False, i, x, y
            if not (x["error"].startswith("vector") or y["error"].startswith("vector")) and x["error"] != y["error"]:
                return False, i, x, y
            continue
        if x != y:
            return False, i, x, y
    return len(a) == len(b), -1, None, None
