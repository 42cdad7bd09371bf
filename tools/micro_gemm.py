"""Single-member GEMM / conv micro-benchmark of the super-kernel vs cuBLAS
(debug/profiling aid; numbers here are not bench values)."""
import argparse
import sys

import torch

sys.path.insert(0, ".")
from paper_1901_00041_b200.runtime import Context, LayerBuffers  # noqa: E402
from paper_1901_00041_b200.scheduler import ConvSpec, GemmShape, b200_profile  # noqa: E402


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tile-n", type=int, default=256)
    ap.add_argument("--shapes", default="18944x256x4096,18944x128x4096,8192x8192x8192,25088x64x576c,6272x128x1152c")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    spec = b200_profile()
    spec.tile_n = a.tile_n
    ctx = Context(0, device=spec)
    for sh in a.shapes.split(","):
        conv = sh.endswith("c")
        M, N, K = (int(v) for v in sh.rstrip("c").split("x"))
        if conv:  # 3x3 s1 p1 conv with Cin = K/9 on a square image giving M pixels
            cin = K // 9
            hw = int(round((M / 8) ** 0.5)) if M > 10000 else int(round((M / 8) ** 0.5))
            b = M // (hw * hw)
            x = torch.randn(b, hw, hw, cin, device=dev).to(torch.bfloat16)
            w = torch.randn(N, K, device=dev).to(torch.bfloat16)
            y = torch.empty(b * hw * hw, N, device=dev, dtype=torch.bfloat16)
            L = LayerBuffers("conv", x, w, y, conv=ConvSpec(hw, hw, 3, 3, cin, N, 1, 1), batch=b)
        else:
            x = torch.randn(M, K, device=dev).to(torch.bfloat16)
            w = torch.randn(N, K, device=dev).to(torch.bfloat16)
            y = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
            L = LayerBuffers("gemm", x, w, y, gemm=GemmShape(M, N, K))
        t = ctx.register_tenant([L])
        s = ctx.layer_shape(t, 0)
        ms = timeit(lambda: ctx.launch_members([(t, 0)]))
        fl = 2 * s.m * s.n * s.k
        xa = x.reshape(-1, K) if not conv else torch.randn(s.m, s.k, device=dev).to(torch.bfloat16)
        ms_ref = timeit(lambda: torch.matmul(xa, w.t()))
        print(f"{sh:18s} ours {ms*1e3:8.1f}us {fl/ms/1e9:7.1f} TF | cuBLAS(gemm) {ms_ref*1e3:8.1f}us "
              f"{fl/ms_ref/1e9:7.1f} TF", flush=True)


if __name__ == "__main__":
    main()
