"""Repeated-launch dependency probe (debug aid): one round program launched
N times, each on a new query batch, every layer's sampled rows checked against
the oracle after each launch; reports the layers that fail and how often."""
import argparse
import sys
from collections import Counter

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
import oracle_check  # noqa: E402
from paper_1901_00041_b200 import workload as W  # noqa: E402
from paper_1901_00041_b200.engine import SpaceTimeEngine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mix")
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--launches", type=int, default=6)
    ap.add_argument("--opt", action="append", default=[])
    a = ap.parse_args()
    opts = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in a.opt}
    if a.config == "mix":
        models = [W.resnet50(224), W.vgg16(224), W.mobilenet_v2(224)] * 2
    else:
        models = [W.resnet50(224)] * 4
    eng = SpaceTimeEngine(models, [a.batch] * len(models), options=opts)
    rnd = eng.plan_round()
    g = eng.capture_round(rnd)
    s = torch.cuda.Stream()
    bad = Counter()
    gen = torch.Generator(device="cuda").manual_seed(7)
    for launch in range(a.launches):
        oracle_check.poison(eng.models)
        for m in eng.models:
            q = m.query_input
            q.copy_((torch.rand(q.shape, device="cuda", generator=gen) * 2 - 1).to(q.dtype))
        s.wait_stream(torch.cuda.current_stream())
        g.launch(s.cuda_stream)
        torch.cuda.synchronize()
        nbad = 0
        for ti, m in enumerate(eng.models):
            for li, (L, buf) in enumerate(zip(m.layers, m.buffers)):
                M, _ = oracle_check.layer_dims(buf)
                rows = oracle_check.sample_rows(M, tile=32, extra=8, seed=li, full_below=256)
                err = oracle_check.rel_err(buf, rows)
                if err > oracle_check.TOL:
                    if bad[(ti, li, L.name)] == 0:
                        ref = oracle_check.expect(buf, rows)
                        got = oracle_check.got_rows(buf, rows)
                        import numpy as np
                        rbad = rows[np.abs(got - ref).max(1) > 0.05 * np.abs(ref).max()]
                        print(f"   ({ti},{li},{L.name}) M={M} err={err:.3g} bad rows {len(rbad)}/{len(rows)}: {rbad[:12]}")
                        sel = np.abs(got - ref).max(1) > 0.05 * np.abs(ref).max()
                        gb, rb = got[sel], ref[sel]
                        badc = np.where((np.abs(gb - rb) > 0.05 * np.abs(ref).max()).any(0))[0]
                        print(f"      got==0 frac {np.mean(gb == 0):.3f}, |got| mean {np.abs(gb).mean():.3g} vs |ref| {np.abs(rb).mean():.3g}; bad channels {len(badc)}: {badc[:8]}..{badc[-4:]}")
                    bad[(ti, li, L.name)] += 1
                    nbad += 1
        print(f"launch {launch}: {nbad} bad layers", flush=True)
    for k, v in sorted(bad.items())[:40]:
        print("  bad", k, v)
    print(f"opts={opts} total bad layer-launches {sum(bad.values())}")


if __name__ == "__main__":
    main()
