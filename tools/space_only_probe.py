"""Why is the space-only baseline (one stream per tenant) bimodal at large R?
Times the captured graph and eager multi-stream launches of R conv2_2 b1
tenants.  Run with CUDA_DEVICE_MAX_CONNECTIONS set to compare."""
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_1901_00041_b200 import workload as W  # noqa: E402
from paper_1901_00041_b200.engine import SpaceTimeEngine  # noqa: E402


def timeit(fn, stream, flush, reps=10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out = []
    for _ in range(reps):
        flush()
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            e0.record()
        fn()
        with torch.cuda.stream(stream):
            e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    out.sort()
    return out[len(out) // 2]


def main():
    dev = torch.device("cuda", 0)
    buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.Stream()
    print("CUDA_DEVICE_MAX_CONNECTIONS", os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS"))
    opts = {a.split("=")[0]: int(a.split("=")[1]) for a in sys.argv[1:] if "=" in a}
    flush = (lambda: None) if "noflush" in sys.argv else (lambda: buf.fill_(1))
    for r in [int(x) for x in sys.argv[1:] if "=" not in x and x.isdigit()] or [16, 32, 64, 80, 100, 120]:
        eng = SpaceTimeEngine([W.conv2_2()] * r, [1] * r, device_index=0, options=opts)
        flops = eng.flops_per_round()
        gsp = eng.capture_serial("space_only")
        gpk = eng.capture_round(eng.plan_round())
        for _ in range(3):
            gsp.launch(stream.cuda_stream)
            gpk.launch(stream.cuda_stream)
        res = {}
        for name, g in (("space_graph", gsp), ("packed", gpk)):
            ms = timeit(lambda: g.launch(stream.cuda_stream), stream, flush)
            res[name] = round(flops / ms / 1e9, 1)
        print("R", r, "tflops", res, "kernels", gsp.kernels, flush=True)
        del eng, gsp, gpk


if __name__ == "__main__":
    main()
