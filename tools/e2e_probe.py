"""Where does the e2e round time go?  H2D bandwidth of pinned buffers with and
without binding the process to the GPU's NUMA-local cores, then e2e rounds."""
import os
import sys
import time

import torch

sys.path.insert(0, ".")


def h2d_bw(nbytes=9633792, reps=50):
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    for _ in range(5):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record()
        for _ in range(reps):
            d.copy_(h, non_blocking=True)
        e1.record()
    torch.cuda.synchronize()
    return nbytes * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9


def main():
    import pynvml
    pynvml.nvmlInit()
    hnd = pynvml.nvmlDeviceGetHandleByIndex(0)
    mask = pynvml.nvmlDeviceGetCpuAffinity(hnd, 16)
    cpus = [w * 64 + b for w, m in enumerate(mask) for b in range(64) if (m >> b) & 1]
    print("ncpu", os.cpu_count(), "gpu-local cpus", len(cpus), cpus[:4], "...", "affinity now", len(os.sched_getaffinity(0)))
    torch.cuda.init()
    print("h2d GB/s default", h2d_bw())
    if "--bind" in sys.argv:
        os.sched_setaffinity(0, cpus)
        print("h2d GB/s bound", h2d_bw())
    from paper_1901_00041_b200 import workload as W
    from paper_1901_00041_b200.engine import SpaceTimeEngine
    eng = SpaceTimeEngine([W.resnet50(224)] * 4, [8] * 4)
    for a in sys.argv[1:]:
        if "=" in a:
            k, v = a.split("=")
            eng.ctx.set_option(k, int(v))
    stream = torch.cuda.Stream()
    h_in = [m.query_input.cpu().pin_memory() for m in eng.models]
    h_out = [torch.empty_like(m.query_output, device="cpu").pin_memory() for m in eng.models]
    for _ in range(10):
        eng.serve_round(h_in, h_out, stream)
    ts = []
    for _ in range(40):
        t0 = time.perf_counter()
        eng.serve_round(h_in, h_out, stream)
        ts.append((time.perf_counter() - t0) * 1e3)
    ts.sort()
    print("e2e ms min/med/mean", ts[0], ts[len(ts) // 2], sum(ts) / len(ts))
    # device-side view of the same graph
    rnd = eng._stable_plan
    g = eng.capture_round_e2e(rnd, h_in, h_out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dev = []
    for _ in range(20):
        with torch.cuda.stream(stream):
            e0.record()
        g.launch(stream.cuda_stream)
        with torch.cuda.stream(stream):
            e1.record()
        stream.synchronize()
        dev.append(e0.elapsed_time(e1))
    dev.sort()
    print("e2e graph device ms med", dev[len(dev) // 2])
    gp = eng.capture_packed(rnd)
    kt = []
    for _ in range(20):
        with torch.cuda.stream(stream):
            e0.record()
        gp.launch(stream.cuda_stream)
        with torch.cuda.stream(stream):
            e1.record()
        stream.synchronize()
        kt.append(e0.elapsed_time(e1))
    kt.sort()
    print("packed graph device ms med", kt[len(kt) // 2])
    ct = []
    for _ in range(20):
        with torch.cuda.stream(stream):
            e0.record()
            for h, m in zip(h_in, eng.models):
                m.query_input.copy_(h.view_as(m.query_input), non_blocking=True)
            e1.record()
        stream.synchronize()
        ct.append(e0.elapsed_time(e1))
    ct.sort()
    print("H2D only ms med", ct[len(ct) // 2])
    wt = []
    for _ in range(20):
        t0 = time.perf_counter()
        gp.launch(stream.cuda_stream)
        stream.synchronize()
        wt.append((time.perf_counter() - t0) * 1e3)
    wt.sort()
    print("packed graph wall ms med", wt[len(wt) // 2])


if __name__ == "__main__":
    main()
