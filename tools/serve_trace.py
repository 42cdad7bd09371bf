"""Serve 4 x ResNet-50 (Poisson, 50% of saturation) for a short window and
write the dispatch trace as the reference's NDJSON lines (gpumux.cpp:64-79).

  python tools/serve_trace.py out.ndjson [seconds]
"""
import sys

sys.path.insert(0, ".")
from paper_1901_00041_b200 import report  # noqa: E402
from paper_1901_00041_b200 import workload as W  # noqa: E402
from paper_1901_00041_b200.engine import ServeTenant, ServingEngine  # noqa: E402


def main():
    out = sys.argv[1]
    secs = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
    specs = [ServeTenant(W.resnet50(224), max_batch=8, batches=[2, 8], rate_qps=5900.0, slo_latency=0.04)
             for _ in range(4)]
    eng = ServingEngine(specs, device_index=0)
    r = eng.serve(duration=secs, warmup=0.1)
    report.write_trace_ndjson(out, r.dispatches)
    print({k: r.stats[k] for k in ("queries", "rounds", "p99_ms", "tflops")}, len(r.dispatches), "events")


if __name__ == "__main__":
    main()
