"""Serving knobs probe (debug aid): rounds in flight and the batcher's age
trigger vs p50/p99 at 50% / 80% of saturation, 4 x ResNet-50 b<=8."""
import sys
sys.path.insert(0, ".")
from paper_1901_00041_b200 import workload as W  # noqa: E402
from paper_1901_00041_b200.engine import ServeTenant, ServingEngine  # noqa: E402

for rate in (5900.0, 9450.0):
    specs = [ServeTenant(W.resnet50(224), max_batch=8, batches=[2, 8], rate_qps=rate, slo_latency=0.04)
             for _ in range(4)]
    eng = ServingEngine(specs, device_index=0)
    for depth, mw in ((1, -1.0), (1, 0.0), (1, 0.0002), (1, 0.0005), (1, 0.001)):
        s = eng.serve(duration=1.5, warmup=0.2, depth=depth, max_wait=mw).stats
        print(rate, depth, mw, round(s["p50_ms"], 3), round(s["p99_ms"], 3), round(s["tflops"], 1),
              round(s["mean_queries_per_round"], 1), flush=True)
