"""The oracles themselves are pinned before they are trusted.

* oracle/planner_ref.py (planner restatement) == the reference's goldens
* oracle/conv_oracle.c (fp32 conv/GEMM checker) == torch conv2d/matmul on CPU
* oracle/cpu_conv.py (numpy port, CPU baseline) == oracle/conv_oracle.c
"""
import ctypes
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from refshim import DEVICES, GOLDEN, ROOT

sys.path.insert(0, os.path.join(ROOT, "oracle"))
import cpu_conv  # noqa: E402
import planner_ref as O  # noqa: E402

LIB = os.path.join(ROOT, "oracle", "_build", "liboracle.so")


@pytest.fixture(scope="module")
def oracle():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True, capture_output=True)
    lib = ctypes.CDLL(LIB)
    f = ctypes.POINTER(ctypes.c_float)
    i = ctypes.c_int64
    lib.oracle_conv2d_nhwc.argtypes = [f, f, f] + [i] * 10 + [ctypes.c_int32]
    lib.oracle_gemm_nt.argtypes = [f, f, f, i, i, i, i, i, ctypes.c_int32]
    lib.oracle_round_bf16.argtypes = [f, i]
    lib.oracle_im2col_nhwc.argtypes = [f, f] + [i] * 9
    lib.oracle_dwconv2d_nhwc.argtypes = [f, f, f] + [i] * 9 + [ctypes.c_int32]
    return lib


def fp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def run_conv(lib, x, w, stride, pad, relu=0):
    b, H, W, C = x.shape
    O_, R, S, _ = w.shape
    P, Q = (H + 2 * pad - R) // stride + 1, (W + 2 * pad - S) // stride + 1
    y = np.zeros((b, P, Q, O_), np.float32)
    w2 = np.ascontiguousarray(w.reshape(O_, -1))
    lib.oracle_conv2d_nhwc(fp(x), fp(w2), fp(y), b, H, W, C, O_, R, S, stride, pad, w2.shape[1], relu)
    return y


@pytest.mark.parametrize("b,hw,cin,cout,r,stride,pad", [
    (1, 16, 128, 128, 3, 1, 1), (2, 9, 3, 8, 7, 2, 3), (1, 14, 64, 16, 1, 2, 0), (3, 7, 32, 24, 3, 1, 1),
    (2, 8, 16, 8, 5, 3, 2)])
def test_conv_oracle_matches_torch(oracle, b, hw, cin, cout, r, stride, pad):
    rng = np.random.default_rng(b * 1000 + hw)
    x = rng.uniform(-1, 1, (b, hw, hw, cin)).astype(np.float32)
    w = rng.standard_normal((cout, r, r, cin)).astype(np.float32)
    y = run_conv(oracle, x, w, stride, pad)
    t = torch.nn.functional.conv2d(torch.from_numpy(x).permute(0, 3, 1, 2).double(),
                                   torch.from_numpy(w).permute(0, 3, 1, 2).double(), stride=stride,
                                   padding=pad).permute(0, 2, 3, 1).float().numpy()
    np.testing.assert_allclose(y, t, rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(cpu_conv.conv2d_nhwc(x, w, stride, pad), y, rtol=1e-4, atol=1e-4)


def test_conv_oracle_relu_and_im2col(oracle):
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, (2, 10, 10, 3)).astype(np.float32)
    w = rng.standard_normal((8, 3, 3, 3)).astype(np.float32)
    np.testing.assert_array_equal(run_conv(oracle, x, w, 1, 1, relu=1), np.maximum(run_conv(oracle, x, w, 1, 1), 0))
    K = 27
    cols = np.zeros((2 * 10 * 10, 32), np.float32)
    oracle.oracle_im2col_nhwc(fp(x), fp(cols), 2, 10, 10, 3, 3, 3, 1, 1, 32)
    y = cols[:, :K] @ w.reshape(8, K).T
    np.testing.assert_allclose(y.reshape(2, 10, 10, 8), run_conv(oracle, x, w, 1, 1), rtol=1e-5, atol=1e-5)
    assert not cols[:, K:].any()


@pytest.mark.parametrize("b,hw,c,stride", [(1, 14, 96, 1), (2, 15, 144, 2), (3, 7, 32, 1), (1, 112, 32, 1)])
def test_dwconv_oracle_matches_torch_groups(oracle, b, hw, c, stride):
    rng = np.random.default_rng(b * 100 + hw + c)
    x = rng.uniform(-1, 1, (b, hw, hw, c)).astype(np.float32)
    w = rng.standard_normal((c, 3, 3)).astype(np.float32)
    P = (hw + 2 - 3) // stride + 1
    y = np.zeros((b, P, P, c), np.float32)
    oracle.oracle_dwconv2d_nhwc(fp(x), fp(np.ascontiguousarray(w.reshape(c, 9))), fp(y), b, hw, hw, c, 3, 3, stride,
                                1, 9, 0)
    t = torch.nn.functional.conv2d(torch.from_numpy(x).permute(0, 3, 1, 2).double(),
                                   torch.from_numpy(w).unsqueeze(1).double(), stride=stride, padding=1,
                                   groups=c).permute(0, 2, 3, 1).float().numpy()
    np.testing.assert_allclose(y, t, rtol=1e-5, atol=1e-5)


def test_gemm_oracle_matches_numpy(oracle):
    rng = np.random.default_rng(5)
    a = rng.standard_normal((37, 72)).astype(np.float32)
    b = rng.standard_normal((19, 80)).astype(np.float32)
    c = np.zeros((37, 19), np.float32)
    oracle.oracle_gemm_nt(fp(a), fp(b), fp(c), 37, 19, 64, 72, 80, 0)
    np.testing.assert_allclose(c, a[:, :64] @ b[:, :64].T, rtol=1e-5, atol=1e-5)


def test_bf16_rounding_matches_torch(oracle):
    v = np.random.default_rng(9).standard_normal(10000).astype(np.float32) * 100
    v[:4] = [np.inf, -np.inf, 0.0, -0.0]
    w = v.copy()
    oracle.oracle_round_bf16(fp(w), w.size)
    np.testing.assert_array_equal(w, torch.from_numpy(v).to(torch.bfloat16).float().numpy())


def test_planner_oracle_pinned_to_reference_sim_goldens():
    with open(os.path.join(GOLDEN, "sim.json")) as f:
        cases = json.load(f)
    for case in cases:
        c, ref = case["input"], case["output"]
        deg = c.get("degrade")
        got = O.run_space_time([tuple(s) for s in c["layers"]], c["tenants"], O.Device(**DEVICES[c["device"]]),
                               O.Policy(target_batch=0), slo=0.05, duration=c["duration"],
                               microbench=c.get("microbench", False),
                               degrade=(deg["tenant"], deg["slowdown"], deg["start"]) if deg else None)
        assert got["events"] == ref["events"], c["name"]
        assert got["completions"] == ref["completions"], c["name"]
        assert got["cancellations"] == ref["cancellations"]
        assert (got["evicted"], got["eviction_times"]) == (ref["evicted"], ref["eviction_times"])
        assert (got["cache_hits"], got["cache_misses"]) == (ref["cache_hits"], ref["cache_misses"])


def test_planner_oracle_pinned_to_reference_cost_goldens():
    with open(os.path.join(GOLDEN, "cost.json")) as f:
        cases = json.load(f)
    for case in cases:
        c = case["input"]
        try:
            k = O.dispatch_duration([(tuple(g["shape"]), g.get("count", 1)) for g in c["groups"]],
                                    O.Device(**DEVICES[c["device"]]), c["slot_budget"], c.get("launches", 1))
            got = {"flops": k.flops, "bytes": k.bytes, "blocks": k.blocks, "duration": k.duration, "waves": k.waves}
        except ValueError as e:
            got = {"error": str(e)}
        assert got == case["output"]


# ------------------------------------------------------------------ dataflow operators

def _torch_act(y, act):
    if act == 1:
        return torch.relu(y)
    if act == 2:
        return torch.clamp(y, 0.0, 6.0)
    if act == 3:
        return torch.nn.functional.gelu(y)  # erf form
    return y


@pytest.mark.parametrize("act", [0, 1, 2, 3])
@pytest.mark.parametrize("with_res,with_rows", [(False, False), (True, False), (True, True)])
def test_oracle_ex_ops_match_torch(act, with_res, with_rows):
    """conv / GEMM with fused residual add and activation, depthwise, pools,
    and row sampling (oracle_check.expect) == torch float64 on CPU."""
    import oracle_check
    from paper_1901_00041_b200.runtime import LayerBuffers
    from paper_1901_00041_b200.scheduler import ConvSpec, GemmShape
    g = torch.Generator().manual_seed(act * 7 + with_res)
    b, hw, cin, cout = 2, 9, 16, 24
    x = (torch.rand(b, hw, hw, cin, generator=g) * 2 - 1).to(torch.bfloat16)
    w = (torch.randn(cout, 3 * 3 * cin, generator=g) * 0.2).to(torch.bfloat16)
    M = b * 5 * 5  # 3x3 s2 p1: 9 -> 5
    res = (torch.rand(M, cout, generator=g) * 2 - 1).to(torch.bfloat16) if with_res else None
    buf = LayerBuffers("conv", x, w, torch.empty(M, cout, dtype=torch.bfloat16),
                       conv=ConvSpec(hw, hw, 3, 3, cin, cout, 2, 1), batch=b, act=act, res=res)
    rows = np.array([0, 7, 13, M - 1], dtype=np.int64) if with_rows else None
    got = oracle_check.expect(buf, rows)
    ref = torch.nn.functional.conv2d(x.double().permute(0, 3, 1, 2), w.double().reshape(cout, 3, 3, cin)
                                     .permute(0, 3, 1, 2), stride=2, padding=1).permute(0, 2, 3, 1).reshape(M, cout)
    if res is not None:
        ref = ref + res.double()
    ref = _torch_act(ref, act).numpy()
    if rows is not None:
        ref = ref[rows]
    np.testing.assert_allclose(got, ref, rtol=1e-5, atol=1e-5)
    # GEMM with a strided (column-slice) input, like BERT's attn_out reading V
    a = (torch.rand(10, 48, generator=g) * 2 - 1).to(torch.bfloat16)[:, 16:40]
    wb = (torch.randn(8, 24, generator=g) * 0.3).to(torch.bfloat16)
    r2 = (torch.rand(10, 8, generator=g) * 2 - 1).to(torch.bfloat16) if with_res else None
    gb = LayerBuffers("gemm", a, wb, torch.empty(10, 8, dtype=torch.bfloat16), gemm=GemmShape(10, 8, 24), act=act,
                      res=r2)
    ref2 = a.double() @ wb.double().T + (r2.double() if r2 is not None else 0)
    np.testing.assert_allclose(oracle_check.expect(gb), _torch_act(ref2, act).numpy(), rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("kind,r,stride,pad", [("maxpool", 3, 2, 1), ("maxpool", 2, 2, 0), ("avgpool", 7, 1, 0)])
def test_oracle_pools_match_torch(kind, r, stride, pad):
    import oracle_check
    from paper_1901_00041_b200.runtime import LayerBuffers
    from paper_1901_00041_b200.scheduler import ConvSpec
    hw = 7 if kind == "avgpool" else 12
    x = (torch.randn(2, hw, hw, 8) * 3).to(torch.bfloat16)
    P = (hw + 2 * pad - r) // stride + 1
    buf = LayerBuffers(kind, x, None, None, conv=ConvSpec(hw, hw, r, r, 8, 8, stride, pad), batch=2)
    xt = x.double().permute(0, 3, 1, 2)
    f = torch.nn.functional.max_pool2d if kind == "maxpool" else torch.nn.functional.avg_pool2d
    ref = f(xt, r, stride, pad).permute(0, 2, 3, 1).reshape(2 * P * P, 8).numpy()
    np.testing.assert_allclose(oracle_check.expect(buf), ref, rtol=1e-6, atol=1e-6)
