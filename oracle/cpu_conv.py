"""TEST INFRASTRUCTURE / CPU BASELINE ONLY — never imported by the product.

A numpy fp32 port of the operator semantics the reference models: a conv is
its im2col GEMM (proj/include/gpumux/gemm.hpp:42-51: rows = output positions,
cols = C_out, inner = the (r, s, c) filter patch), batching multiplies the
rows (gemm.hpp:54-56), and a GEMM is C = A @ B^T with B stored K-major.
The im2col view is built with stride tricks (no copy until the matmul packs
it) and the GEMM runs on numpy's multithreaded BLAS, so this is the fastest
plain-CPU fp32 restatement of the path; bench.py times it as the CPU
baseline (kind "port") and the reference arm.  tests/test_oracle.py checks it
against oracle/conv_oracle.c (double accumulation) and torch's conv2d.
"""
from __future__ import annotations

import os

import numpy as np


def conv2d_nhwc(x: np.ndarray, w: np.ndarray, stride: int, pad: int) -> np.ndarray:
    """x [b, H, W, C] fp32, w [O, R, S, C] fp32 -> y [b, P, Q, O] fp32."""
    b, H, W, Cin = x.shape
    O, R, S, _ = w.shape
    if pad:
        x = np.pad(x, ((0, 0), (pad, pad), (pad, pad), (0, 0)))
    P = (H + 2 * pad - R) // stride + 1
    Q = (W + 2 * pad - S) // stride + 1
    sb, sh, sw, sc = x.strides
    cols = np.lib.stride_tricks.as_strided(x, shape=(b, P, Q, R, S, Cin),
                                           strides=(sb, sh * stride, sw * stride, sh, sw, sc), writeable=False)
    a = np.ascontiguousarray(cols).reshape(b * P * Q, R * S * Cin)
    return (a @ w.reshape(O, R * S * Cin).T).reshape(b, P, Q, O)


def dwconv2d_nhwc(x: np.ndarray, w: np.ndarray, stride: int, pad: int) -> np.ndarray:
    """Depthwise (groups = C): x [b, H, W, C], w [C, R, S] -> y [b, P, Q, C] (torchvision MobileNet-v2)."""
    b, H, W, C = x.shape
    _, R, S = w.shape
    if pad:
        x = np.pad(x, ((0, 0), (pad, pad), (pad, pad), (0, 0)))
    P = (H + 2 * pad - R) // stride + 1
    Q = (W + 2 * pad - S) // stride + 1
    y = np.zeros((b, P, Q, C), np.float32)
    for r in range(R):
        for s in range(S):
            y += x[:, r:r + stride * P:stride, s:s + stride * Q:stride, :] * w[:, r, s]
    return y


def gemm_nt(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    return a @ b.T


def threads() -> int:
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS"):
        if os.environ.get(var):
            return int(os.environ[var])
    return os.cpu_count() or 1


# ------------------------------------------------------------------ dataflow graphs

def _act(y: np.ndarray, act: int) -> np.ndarray:
    if act == 1:
        return np.maximum(y, 0.0, out=y)
    if act == 2:
        return np.clip(y, 0.0, 6.0, out=y)
    if act == 3:
        from math import sqrt
        try:
            from scipy.special import erf
        except Exception:  # pragma: no cover - scipy is in the image
            erf = np.vectorize(__import__("math").erf)
        return 0.5 * y * (1.0 + erf(y / sqrt(2.0)))
    return y


def pool2d_nhwc(x: np.ndarray, r: int, stride: int, pad: int, is_max: bool) -> np.ndarray:
    b, H, W, C = x.shape
    if pad:
        x = np.pad(x, ((0, 0), (pad, pad), (pad, pad), (0, 0)), constant_values=-np.inf if is_max else 0.0)
    P = (H + 2 * pad - r) // stride + 1
    Q = (W + 2 * pad - r) // stride + 1
    y = np.full((b, P, Q, C), -np.inf if is_max else 0.0, np.float32)
    for i in range(r):
        for j in range(r):
            v = x[:, i:i + stride * P:stride, j:j + stride * Q:stride, :]
            y = np.maximum(y, v) if is_max else y + v
    return y if is_max else y / float(r * r)


class CpuGraph:
    """A tenant's dataflow graph (oracle/graphs/*.json, exported from the
    product's workload builders by tools/export_graphs.py) in numpy fp32:
    each layer reads its ``src`` layer's output (or its own input), adds its
    ``res`` layer's output, applies ``act`` -- the semantics the GPU path runs.
    Synthetic U(-1, 1) inputs, Kaiming-scaled weights; timed as the CPU
    baseline and the reference arm's tensor work."""

    def __init__(self, graph: list, batch: int, seed: int = 42):
        rng = np.random.default_rng(seed)
        self.graph, self.batch = graph, batch
        self.inputs, self.weights = [], []
        for L in graph:
            x = w = None
            if L["kind"] in ("conv", "dwconv", "maxpool", "avgpool"):
                H, W_, R, S, Cin, Cout, st, pad = L["conv"]
                if L["src"] is None:
                    x = rng.uniform(-1, 1, (batch, H, W_, Cin)).astype(np.float32)
                if L["kind"] == "conv":
                    w = (rng.standard_normal((Cout, R, S, Cin)) * (2.0 / (R * S * Cin)) ** 0.5).astype(np.float32)
                elif L["kind"] == "dwconv":
                    w = (rng.standard_normal((Cout, R, S)) * (2.0 / (R * S)) ** 0.5).astype(np.float32)
            else:
                if L["src"] is None:
                    x = rng.uniform(-1, 1, (L["rows"] * batch, L["k"])).astype(np.float32)
                w = (rng.standard_normal((L["n"], L["k"])) * (2.0 / L["k"]) ** 0.5).astype(np.float32)
            self.inputs.append(x)
            self.weights.append(w)
        self.flops_pass = sum(layer_flops(L, batch) for L in graph)

    def run_pass(self) -> np.ndarray:
        ys = []
        b = self.batch
        for L, x, w in zip(self.graph, self.inputs, self.weights):
            kind = L["kind"]
            if kind == "gemm":
                rows = L["rows"] * b
                a = x if L["src"] is None else ys[L["src"]].reshape(rows, -1)[:, L["src_col"]:L["src_col"] + L["k"]]
                y = gemm_nt(a, w)
            else:
                H, W_, R, S, Cin, Cout, st, pad = L["conv"]
                a = x if L["src"] is None else ys[L["src"]].reshape(b, H, W_, Cin)
                if kind == "conv":
                    y = conv2d_nhwc(a, w, st, pad)
                elif kind == "dwconv":
                    y = dwconv2d_nhwc(a, w, st, pad)
                else:
                    y = pool2d_nhwc(a, R, st, pad, kind == "maxpool")
                y = y.reshape(-1, Cout)
            if L["res"] is not None:
                y = y + ys[L["res"]].reshape(y.shape)
            ys.append(_act(y, L["act"]))
        return ys[-1]

    def sample(self, seconds: float):
        import time
        done, t0 = 0, time.perf_counter()
        while True:
            self.run_pass()
            done += 1
            el = time.perf_counter() - t0
            if el >= seconds:
                return done * self.flops_pass / el / 1e12, done, el


def layer_flops(L: dict, batch: int) -> int:
    """2mnk of the layer's GEMM view (pools: 0), gemm.hpp:33-35 / 54-56."""
    if L["kind"] in ("maxpool", "avgpool"):
        return 0
    if L["kind"] == "gemm":
        return 2 * L["rows"] * batch * L["n"] * L["k"]
    H, W_, R, S, Cin, Cout, st, pad = L["conv"]
    P = (H + 2 * pad - R) // st + 1
    Q = (W_ + 2 * pad - S) // st + 1
    k = R * S if L["kind"] == "dwconv" else R * S * Cin
    return 2 * batch * P * Q * Cout * k


def load_graph(name: str) -> list:
    import json
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "graphs", name + ".json")) as f:
        return json.load(f)
