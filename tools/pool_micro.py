"""Isolated CUDA-core tile micro-benchmark: R tenants' pool / depthwise layers
as ONE super-kernel launch (no other work), CUDA-event timed.  Debug aid."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1901_00041_b200.runtime import Context, LayerBuffers  # noqa: E402
from paper_1901_00041_b200.scheduler import ConvSpec  # noqa: E402


def bench(kind, hw, c, r, st, pad, b=8, tenants=4, reps=20):
    ctx = Context(0)
    ts = []
    keep = []
    for _ in range(tenants):
        x = torch.randn(b, hw, hw, c, device="cuda").to(torch.bfloat16)
        P = (hw + 2 * pad - r) // st + 1
        y = torch.empty(b * P * P, c, device="cuda", dtype=torch.bfloat16)
        w = (torch.randn(c, r * r, device="cuda") * 0.3).to(torch.bfloat16) if kind == "dwconv" else None
        L = LayerBuffers(kind, x, w, y, conv=ConvSpec(hw, hw, r, r, c, c, st, pad), batch=b)
        keep.append(L)
        ts.append(ctx.register_tenant([L]))
    s = torch.cuda.Stream()
    members = [(t, 0) for t in ts]
    for _ in range(3):
        ctx.launch_members(members, s.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(reps):
            ctx.launch_members(members, s.cuda_stream)
        e1.record(s)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    byt = tenants * (b * hw * hw * c + keep[0].y.numel()) * 2
    print(f"{kind:8s} {hw}x{hw}x{c} r{r} s{st} b{b} x{tenants}: {us:7.1f} us/launch, {byt / us / 1e3:7.1f} GB/s compulsory")


CASES = {
    "maxpool112": ("maxpool", 112, 64, 3, 2, 1),
    "maxpool224": ("maxpool", 224, 64, 2, 2, 0),
    "avgpool7": ("avgpool", 7, 2048, 7, 1, 0),
    "dw112s2": ("dwconv", 112, 96, 3, 2, 1),
    "dw56": ("dwconv", 56, 144, 3, 1, 1),
}
for name in (sys.argv[1:] or CASES):
    bench(*CASES[name], reps=int(__import__("os").environ.get("REPS", "20")))
