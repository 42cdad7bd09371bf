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
