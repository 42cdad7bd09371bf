"""Quick on-GPU correctness probe of the super-kernel (debug aid, not a test).

Runs a handful of conv/GEMM members through the C-ABI and prints the relative
error against torch fp32 on the same bf16-rounded inputs.
"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1901_00041_b200.runtime import Context, LayerBuffers  # noqa: E402
from paper_1901_00041_b200.scheduler import ConvSpec, GemmShape  # noqa: E402


def conv_case(b, H, W, Cin, Cout, R, stride, pad, dev):
    x = (torch.rand(b, H, W, Cin, device=dev) * 2 - 1).to(torch.bfloat16)
    K = R * R * Cin
    ldw = (K + 7) // 8 * 8
    wfull = torch.zeros(Cout, ldw, device=dev, dtype=torch.bfloat16)
    w = (torch.randn(Cout, R, R, Cin, device=dev) * (2.0 / K) ** 0.5).to(torch.bfloat16)
    wfull[:, :K] = w.reshape(Cout, K)
    P = (H + 2 * pad - R) // stride + 1
    y = torch.full((b, P, P, Cout), float("nan"), device=dev, dtype=torch.bfloat16)
    ref = torch.nn.functional.conv2d(x.float().permute(0, 3, 1, 2), w.float().permute(0, 3, 1, 2), stride=stride,
                                     padding=pad).permute(0, 2, 3, 1)
    return LayerBuffers("conv", x, wfull, y, conv=ConvSpec(H, W, R, R, Cin, Cout, stride, pad), batch=b), ref


def gemm_case(M, N, K, dev):
    ld = (K + 7) // 8 * 8
    x = (torch.rand(M, ld, device=dev) * 2 - 1).to(torch.bfloat16)[:, :K]
    w = (torch.randn(N, ld, device=dev) / K ** 0.5).to(torch.bfloat16)[:, :K]
    y = torch.full((M, N), float("nan"), device=dev, dtype=torch.bfloat16)
    return LayerBuffers("gemm", x, w, y, gemm=GemmShape(M, N, K)), x.float() @ w.float().t()


def main():
    import argparse
    from paper_1901_00041_b200.scheduler import b200_profile
    ap = argparse.ArgumentParser()
    ap.add_argument("--tile-n", type=int, default=256)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    torch.manual_seed(0)
    spec = b200_profile()
    spec.tile_n = a.tile_n
    ctx = Context(0, device=spec)
    cases = {
        "gemm 256x128x1152": gemm_case(256, 128, 1152, dev),
        "gemm 200x72x100 (tails)": gemm_case(200, 72, 100, dev),
        "gemm 1000x1000x520": gemm_case(1000, 1000, 520, dev),
        "conv 3x3 s1 16x16x128->128 b2": conv_case(2, 16, 16, 128, 128, 3, 1, 1, dev),
        "conv 3x3 s2 56x56x64->128 b1": conv_case(1, 56, 56, 64, 128, 3, 2, 1, dev),
        "conv 1x1 s1 28x28x256->512 b2": conv_case(2, 28, 28, 256, 512, 1, 1, 0, dev),
        "conv 1x1 s2 56x56x256->512 b1": conv_case(1, 56, 56, 256, 512, 1, 2, 0, dev),
        "conv 7x7 s2 stem 224->64 b2": conv_case(2, 224, 224, 3, 64, 7, 2, 3, dev),
        "conv 3x3 s1 7x7x512->512 b3": conv_case(3, 7, 7, 512, 512, 3, 1, 1, dev),
        "conv 3x3 s1 7x7x512->512 b1 (M=49)": conv_case(1, 7, 7, 512, 512, 3, 1, 1, dev),
        "gemm 8x1000x2048 (fc b8)": gemm_case(8, 1000, 2048, dev),
        "gemm 384x2304x768 (bert qkv)": gemm_case(384, 2304, 768, dev),
    }
    names = list(cases)
    tenant = ctx.register_tenant([cases[n][0] for n in names])
    ok = True
    for i, n in enumerate(names):
        t0 = time.time()
        ctx.launch_members([(tenant, i)])
        torch.cuda.synchronize()
        L, ref = cases[n]
        y = L.y.float().reshape(ref.shape)
        err = ((y - ref).abs().max() / ref.abs().max()).item()
        nan = torch.isnan(y).any().item()
        print(f"{n:36s} rel_err={err:.3e} nan={nan} shape={tuple(ctx.layer_shape(tenant, i).__dict__.values())} "
              f"{(time.time()-t0)*1e3:.1f} ms", flush=True)
        ok &= (err < 1e-2) and not nan
    # packed: all members in one launch
    for L, _ in cases.values():
        L.y.fill_(float("nan"))
    ctx.launch_members([(tenant, i) for i in range(len(names))])
    torch.cuda.synchronize()
    for i, n in enumerate(names):
        L, ref = cases[n]
        y = L.y.float().reshape(ref.shape)
        err = ((y - ref).abs().max() / ref.abs().max()).item()
        print(f"packed {n:29s} rel_err={err:.3e}", flush=True)
        ok &= err < 1e-2
    # round program: a 3-tenant ResNet-18@64 round in one persistent launch
    from paper_1901_00041_b200 import workload as W
    from paper_1901_00041_b200.engine import SpaceTimeEngine
    layers = W.resnet18(64)
    eng = SpaceTimeEngine([layers] * 3, [2, 2, 2])
    rnd = eng.plan_round()
    refs = []
    for m in eng.models:
        for L, buf in zip(m.layers, m.buffers):
            if L.kind == "conv":
                c = L.conv
                w = buf.w[:, : c.kernel_h * c.kernel_w * c.in_channels].reshape(
                    c.out_channels, c.kernel_h, c.kernel_w, c.in_channels)
                r = torch.nn.functional.conv2d(buf.x.float().permute(0, 3, 1, 2), w.float().permute(0, 3, 1, 2),
                                               stride=c.stride, padding=c.padding).permute(0, 2, 3, 1).reshape(
                    buf.y.shape)
            else:
                r = buf.x.float() @ buf.w.float().t()
            refs.append((buf.y, r))
            buf.y.fill_(float("nan"))
    s = torch.cuda.Stream()
    rnd.launch_round(s.cuda_stream)
    torch.cuda.synchronize()
    worst = max(((y.float() - r).abs().max() / r.abs().max()).item() for y, r in refs)
    print(f"round program: {len(rnd.kernels)} plans in 1 launch, worst rel err {worst:.3e}")
    ok &= worst < 1e-2
    print("ALL OK" if ok else "FAIL")


if __name__ == "__main__":
    main()
