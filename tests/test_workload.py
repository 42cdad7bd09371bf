"""Model graphs (workload.py): dataflow structure, the exported package-free
copies (oracle/graphs/*.json), and the numpy graph runner (oracle/cpu_conv.py,
the CPU baseline) against a float64 torch run of the same graph."""
import json
import os
import sys

import numpy as np
import pytest
import torch

from refshim import ROOT
from paper_1901_00041_b200 import workload as W

sys.path.insert(0, os.path.join(ROOT, "oracle"))
import cpu_conv  # noqa: E402


def out_numel(L, b):
    s = L.gemm_shape(b)
    return s.m * s.n


@pytest.mark.parametrize("name", sorted(W.EXPORTED_GRAPHS))
def test_exported_graph_is_current(name):
    with open(os.path.join(ROOT, "oracle", "graphs", name + ".json")) as f:
        assert json.load(f) == json.loads(json.dumps(W.graph_json(W.EXPORTED_GRAPHS[name]())))


@pytest.mark.parametrize("build", [lambda: W.resnet50(224), lambda: W.resnet18(224), lambda: W.vgg16(224),
                                   lambda: W.mobilenet_v2(224), lambda: W.bert_base_gemms(128, 3),
                                   lambda: W.resnet18(64), lambda: W.mobilenet_v2(64)])
def test_dataflow_shapes_chain(build):
    layers = build()
    b = 3
    for i, L in enumerate(layers):
        if L.src is not None:
            assert 0 <= L.src < i
            P = layers[L.src]
            if L.kind == "gemm":
                s = L.gemm_shape(b)
                assert out_numel(P, b) % s.m == 0 and out_numel(P, b) // s.m >= L.src_col + s.k
            else:
                c = L.conv
                assert out_numel(P, b) == b * c.image_h * c.image_w * c.in_channels
                assert P.gemm_shape(b).n == c.in_channels
        if L.res is not None:
            assert 0 <= L.res < i and L.kind in ("conv", "gemm")
            assert layers[L.res].gemm_shape(b).n == L.gemm_shape(b).n
            assert out_numel(layers[L.res], b) == out_numel(L, b)
    assert layers[0].src is None


def test_resnet50_structure():
    L = W.resnet50(224)
    kinds = [x.kind for x in L]
    assert kinds.count("conv") == 53 and kinds.count("maxpool") == 1 and kinds.count("avgpool") == 1
    assert kinds[-1] == "gemm" and sum(x.res is not None for x in L) == 16  # one residual add per bottleneck
    flops = sum(x.flops(1) for x in L)
    assert abs(flops / 1e9 - 8.18) < 0.05  # torchvision ResNet-50 @224: 4.09 GMACs


def _torch_graph(g, graph, b):
    ys = []
    for L, x, w in zip(graph, g.inputs, g.weights):
        if L["kind"] == "gemm":
            rows = L["rows"] * b
            a = torch.from_numpy(x).double() if L["src"] is None else \
                ys[L["src"]].reshape(rows, -1)[:, L["src_col"]:L["src_col"] + L["k"]]
            y = a @ torch.from_numpy(w).double().T
        else:
            H, W_, R, S, Cin, Cout, st, pad = L["conv"]
            a = (torch.from_numpy(x).double() if L["src"] is None else ys[L["src"]].reshape(b, H, W_, Cin))
            a = a.permute(0, 3, 1, 2)
            if L["kind"] == "conv":
                y = torch.nn.functional.conv2d(a, torch.from_numpy(w).double().permute(0, 3, 1, 2), stride=st,
                                               padding=pad)
            elif L["kind"] == "dwconv":
                y = torch.nn.functional.conv2d(a, torch.from_numpy(w).double()[:, None], stride=st, padding=pad,
                                               groups=Cin)
            elif L["kind"] == "maxpool":
                y = torch.nn.functional.max_pool2d(a, R, st, pad)
            else:
                y = torch.nn.functional.avg_pool2d(a, R, st, pad)
            y = y.permute(0, 2, 3, 1).reshape(-1, Cout)
        if L["res"] is not None:
            y = y + ys[L["res"]].reshape(y.shape)
        y = {0: y, 1: torch.relu(y), 2: torch.clamp(y, 0, 6), 3: torch.nn.functional.gelu(y)}[L["act"]]
        ys.append(y)
    return ys[-1]


@pytest.mark.parametrize("build,b", [(lambda: W.resnet18(32), 2), (lambda: W.mobilenet_v2(32), 2),
                                     (lambda: W.vgg16(32), 1), (lambda: W.bert_base_gemms(8, 2), 2)])
def test_cpu_graph_matches_torch(build, b):
    graph = json.loads(json.dumps(W.graph_json(build())))
    g = cpu_conv.CpuGraph(graph, b, seed=1)
    got = g.run_pass()
    ref = _torch_graph(g, graph, b).numpy()
    np.testing.assert_allclose(got, ref, rtol=2e-3, atol=2e-3 * np.abs(ref).max())
    assert g.flops_pass == sum(x.flops(b) for x in build())
