"""Per-tile timeline of one round program (in-kernel %globaltimer stamps).

For each plan (super-kernel) of the round: wall span, and the mean per-tile
durations of gate wait / first-load latency / MMA issue / MMA drain /
epilogue, next to the plan's roofline time.  Debug/profiling aid.
"""
import argparse
import ctypes as C
import json
import sys
from collections import defaultdict

import torch

sys.path.insert(0, ".")
from paper_1901_00041_b200 import _native as N  # noqa: E402
from paper_1901_00041_b200 import workload as W  # noqa: E402
from paper_1901_00041_b200._native import check, lib  # noqa: E402
from paper_1901_00041_b200.engine import SpaceTimeEngine  # noqa: E402
from paper_1901_00041_b200.scheduler import BatchPolicy  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="resnet50")
    ap.add_argument("--tenants", type=int, default=4)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--max-waves", type=int, default=1)
    ap.add_argument("--out", default="")
    ap.add_argument("--opt", action="append", default=[], help="runtime option name=value")
    ap.add_argument("--tile-n", type=int, default=256)
    ap.add_argument("--raw", default="", help="also save raw per-tile stamps (npz: stamps, plan, cta)")
    a = ap.parse_args()
    peaks = json.load(open("MEASURED_PEAKS.json"))
    P, BW = peaks["bf16_tflops"] * 1e12, peaks["hbm_gbs"] * 1e9
    if a.model == "bert":  # BASELINE configs[3]: 12-layer BERT-base GEMM chain, seq 128
        layers = W.bert_base_gemms(128, layers=12)
    else:
        layers = W.resnet50(224) if a.model in ("resnet50", "mix") else W.MODELS[a.model]()
    opts = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in a.opt}
    from paper_1901_00041_b200.scheduler import b200_profile
    spec = b200_profile()
    spec.tile_n = a.tile_n
    if a.model == "mix":  # BASELINE configs[2]: ResNet-50 + VGG-16 + MobileNet-v2 @224, two each
        tl = [W.resnet50(224), W.vgg16(224), W.mobilenet_v2(224)] * 2
    else:
        tl = [layers] * a.tenants
    eng = SpaceTimeEngine(tl, [a.batch] * len(tl), options=opts, device_spec=spec)
    rnd = eng.plan_round(BatchPolicy(target_batch=0, max_waves=a.max_waves))
    s = torch.cuda.Stream()
    for _ in range(3):
        rnd.launch_round(s.cuda_stream)
    torch.cuda.synchronize()
    n = C.c_size_t()
    lib().gm_round_tiles(eng.ctx.handle, rnd.handle, None, 0, C.byref(n))
    tiles = (N.gm_tile * n.value)()
    check(lib().gm_round_tiles(eng.ctx.handle, rnd.handle, tiles, n.value, C.byref(n)))
    buf = (C.c_uint64 * (6 * n.value + 6 * 148))()
    nt = C.c_size_t()
    check(lib().gm_trace_round(eng.ctx.handle, rnd.handle, s.cuda_stream, buf, len(buf), C.byref(nt)))
    t = [[buf[6 * i + j] for j in range(6)] for i in range(n.value)]
    t0 = min(x[0] for x in t)
    by_plan = defaultdict(list)
    for i, tile in enumerate(tiles):
        by_plan[tile.flags].append(t[i])
    rows = []
    tot_roof = 0.0
    pos_of = {t: i for i, t in enumerate(eng.tenants)}
    for pi, k in enumerate(rnd.kernels):
        ts = by_plan[pi]
        span = (max(x[5] for x in ts) - min(x[0] for x in ts)) / 1e3
        start = (min(x[0] for x in ts) - t0) / 1e3
        mean = lambda a, b: sum(x[b] - x[a] for x in ts) / len(ts) / 1e3  # noqa: E731
        mlayers = [eng.models[pos_of[r.tenant_index]].layers[r.layer_index] for r in k.members]
        F = sum(L.flops(a.batch) for L in mlayers)
        B = sum(L.compulsory_bytes(a.batch) for L in mlayers)
        roof = max(F / P, B / BW) * 1e6
        tot_roof += roof
        row = dict(plan=pi, sig=k.shape_signature, tiles=len(ts), start_us=start, span_us=span, roof_us=roof,
                   gate=mean(0, 1), load=mean(1, 2), mma=mean(2, 3), drain=mean(3, 4), epi=mean(4, 5))
        rows.append(row)
        print(f"{pi:3d} {k.shape_signature:22s} tiles={len(ts):4d} start={start:7.1f} span={span:6.1f}us "
              f"roof={roof:5.1f} | gate={row['gate']:5.2f} load={row['load']:5.2f} mma={row['mma']:5.2f} "
              f"drain={row['drain']:5.2f} epi={row['epi']:5.2f}")
    grid = min(n.value, 148)
    cta = [[buf[6 * n.value + 6 * c + j] for j in range(6)] for c in range(grid)]
    if all(x[0] for x in cta):
        # SM cycles from each CTA's own entry (clock64; not comparable across SMs)
        names = ["setup", "producer-done", "barrier", "tmem-freed", "exit"]
        print("CTA phases, cycles from entry (min/med/max): " + ", ".join(
            "%s %d/%d/%d" % (nm, *(lambda v: (v[0], v[len(v) // 2], v[-1]))(
                sorted(x[j + 1] - x[0] for x in cta))) for j, nm in enumerate(names)))
    total = (max(x[5] for x in t) - t0) / 1e3
    print(f"kernel span {total:.1f}us, roofline {tot_roof:.1f}us, tiles {n.value}")
    if a.raw:
        import numpy as np
        np.savez_compressed(a.raw, stamps=np.array(t, dtype=np.uint64) - np.uint64(t0),
                            plan=np.array([tile.flags for tile in tiles], dtype=np.int32),
                            cta=np.arange(n.value, dtype=np.int32) % grid)
    if a.out:
        json.dump({"rows": rows, "span_us": total, "roof_us": tot_roof}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
