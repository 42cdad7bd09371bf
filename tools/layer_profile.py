"""Per-super-kernel timing of one packed round (debug/profiling aid).

Prints, for each launch of the packed round: signature, members, tiles,
event-timed duration, TFLOP/s and compulsory-bytes GB/s, next to the
per-launch roofline time max(F/P, B/BW).
"""
import argparse
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1901_00041_b200 import workload as W  # noqa: E402
from paper_1901_00041_b200.engine import SpaceTimeEngine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--tenants", type=int, default=4)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--json", default="")
    a = ap.parse_args()
    peaks = json.load(open("MEASURED_PEAKS.json"))
    P, BW = peaks["bf16_tflops"] * 1e12, peaks["hbm_gbs"] * 1e9
    layers = W.resnet50(224) if a.model == "resnet50" else W.MODELS[a.model]()
    eng = SpaceTimeEngine([layers] * a.tenants, [a.batch] * a.tenants)
    rnd = eng.plan_round()
    g = eng.capture_packed(rnd, timed=True)
    s = torch.cuda.Stream()
    tot = [0.0] * g.superkernels
    for i in range(a.reps + 2):
        g.launch(s.cuda_stream)
        t = g.kernel_times_ms()
        if i >= 2:
            tot = [x + y for x, y in zip(tot, t)]
    by_layer = {(L.gemm_shape(a.batch).m, L.gemm_shape(a.batch).n, L.gemm_shape(a.batch).k): L for L in layers}
    rows = []
    sum_ms = sum_roof = 0.0
    for k, ms in zip(rnd.kernels, tot):
        ms /= a.reps
        sh = k.members[0].shape
        L = by_layer[(sh.m, sh.n, sh.k)]
        n = len(k.members)
        F = n * L.flops(a.batch)
        B = n * L.compulsory_bytes(a.batch)
        roof = max(F / P, B / BW) * 1e3
        sum_ms += ms
        sum_roof += roof
        rows.append({"layer": L.name, "sig": k.shape_signature, "members": n, "tiles": k.planned_cost.blocks,
                     "ms": ms, "tflops": F / ms / 1e9, "gbs": B / ms / 1e6, "roof_ms": roof, "eff": roof / ms})
        print(f"{L.name:24s} {k.shape_signature:22s} m={n} tiles={k.planned_cost.blocks:4d} {ms*1e3:8.1f}us "
              f"{F/ms/1e9:7.1f}TF {B/ms/1e6:7.1f}GB/s roof={roof*1e3:7.1f}us eff={roof/ms:.2f}")
    print(f"total {sum_ms*1e3:.1f}us roofline {sum_roof*1e3:.1f}us eff {sum_roof/sum_ms:.3f} "
          f"TF={eng.flops_per_round()/sum_ms/1e9:.1f}")
    if a.json:
        json.dump(rows, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
