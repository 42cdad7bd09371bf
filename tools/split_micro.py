"""Split-K micro-profile: one GEMM member as a 1-plan round program, per-tile
%globaltimer stamps printed for each split setting (debug aid)."""
import argparse
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_1901_00041_b200 import _native as N  # noqa: E402
from paper_1901_00041_b200._native import check, lib  # noqa: E402
from paper_1901_00041_b200.runtime import Context, LayerBuffers  # noqa: E402
from paper_1901_00041_b200.scheduler import BatchPolicy, GemmShape  # noqa: E402


def run(m, n, k, opts, tenants):
    ctx = Context(0, policy=BatchPolicy(target_batch=0))
    for kk, v in opts.items():
        ctx.set_option(kk, v)
    ids = []
    for _ in range(tenants):
        x = torch.randn(m, k, device="cuda").to(torch.bfloat16)
        w = torch.randn(n, k, device="cuda").to(torch.bfloat16)
        y = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        ids.append(ctx.register_tenant([LayerBuffers("gemm", x, w, y, gemm=GemmShape(m, n, k))]))
        ctx._keepalive.append((x, w, y))
    rnd = ctx.plan_round(ids, 0)
    s = torch.cuda.Stream()
    for _ in range(3):
        rnd.launch_round(s.cuda_stream)
    torch.cuda.synchronize()
    nt = C.c_size_t()
    lib().gm_round_tiles(ctx.handle, rnd.handle, None, 0, C.byref(nt))
    buf = (C.c_uint64 * (6 * nt.value))()
    check(lib().gm_trace_round(ctx.handle, rnd.handle, s.cuda_stream, buf, len(buf), C.byref(nt)))
    t = [[buf[6 * i + j] for j in range(6)] for i in range(nt.value)]
    t0 = min(x[0] for x in t)
    span = (max(x[5] for x in t) - t0) / 1e3
    print(f"{m}x{n}x{k} x{tenants} {opts}: tiles {nt.value} span {span:.1f}us")
    for i, x in enumerate(t[:12]):
        print(f"   tile {i:3d} start {(x[0]-t0)/1e3:6.2f} data {(x[2]-x[0])/1e3:5.2f} mma {(x[3]-x[2])/1e3:6.2f} "
              f"drain {(x[4]-x[3])/1e3:5.2f} epi {(x[5]-x[4])/1e3:5.2f} end {(x[5]-t0)/1e3:6.2f}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="392x512x4608")
    ap.add_argument("--tenants", type=int, default=4)
    a = ap.parse_args()
    m, n, k = (int(v) for v in a.shape.split("x"))
    for opts in ({"split_k": 0}, {"split_k": 1, "max_splits": 2}, {"split_k": 1, "max_splits": 4},
                 {"split_k": 1, "max_splits": 8}):
        run(m, n, k, opts, a.tenants)


if __name__ == "__main__":
    main()
