"""Serving probe (debug aid): gm_serve on the headline tenants, closed loop
and Poisson at given rates; prints the stats dicts."""
import argparse
import json
import sys

sys.path.insert(0, ".")
from paper_1901_00041_b200 import workload as W  # noqa: E402
from paper_1901_00041_b200.engine import ServeTenant, ServingEngine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tenants", type=int, default=4)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--rates", default="0")
    ap.add_argument("--duration", type=float, default=2.0)
    ap.add_argument("--depth", type=int, default=1)
    ap.add_argument("--max-wait", type=float, default=-1)
    a = ap.parse_args()
    for rate in [float(x) for x in a.rates.split(",")]:
        specs = [ServeTenant(W.resnet50(224), max_batch=a.batch, rate_qps=rate, concurrency=a.batch,
                             slo_latency=0.040) for _ in range(a.tenants)]
        eng = ServingEngine(specs)
        eng.serve(duration=0.5, warmup=0.1, depth=a.depth, max_wait=a.max_wait)  # warm plan cache
        r = eng.serve(duration=a.duration, warmup=0.2, depth=a.depth, max_wait=a.max_wait)
        print(json.dumps({"rate": rate, **{k: round(v, 4) if isinstance(v, float) else v for k, v in r.stats.items()}}))


if __name__ == "__main__":
    main()
