"""Print the serving sections of a bench JSON line (debug aid)."""
import json
import sys

d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][-1])


def show(name, pts):
    for k, v in pts.items():
        if isinstance(v, dict) and "qps" in v:
            print(f"  {name}.{k}: tflops {v['tflops']:.1f} qps {v['qps']:.0f} p50 {v['p50_ms']:.2f} p99 {v['p99_ms']:.2f}"
                  f" slo_viol {v['slo_violation_frac']:.3f} q/round {v['mean_queries_per_round']:.1f}"
                  f" round_ms {v['mean_round_ms']:.3f} hit {v['plan_hits']} miss {v['plan_misses']}"
                  f" pad {v.get('plan_padded')} ev {v['plan_evictions']} slo_ms {v.get('slo_ms')}")


print("headline", d["value"], "e2e", d["e2e"]["value"])
if "serving" in d:
    show("serving", d["serving"])
for c in ("config_mix", "config_bert"):
    if c in d and d[c].get("serving"):
        show(c, d[c]["serving"])
if "config_c5" in d:
    show("c5", d["config_c5"])
