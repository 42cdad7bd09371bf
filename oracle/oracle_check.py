"""TEST INFRASTRUCTURE ONLY (tests/ and __graft_entry__.smoke()): the CPU
oracle (oracle/conv_oracle.c) applied to one operator of the GPU path, on the
device's own bf16 inputs.

For a dataflow layer the input is the previous layer's device output, so the
check is per layer: a layer that read a stale or partially written input (a
broken dependency) disagrees with the oracle computed from the final input.
Large layers are checked on sampled output rows: the first and last row of
every 128-row tile (every tile of the launch is covered), the last row, and
random rows; ``rows=None`` checks all of them.

Tolerance (BASELINE north star): ||y - y_ref||_inf / ||y_ref||_inf <= 1e-2
per operator output, bf16 in / fp32 accumulate / bf16 out.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
TOL = 1e-2

_lib = None


def oracle_lib():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(os.path.join(HERE, "_build", "liboracle.so"))
        f = ctypes.POINTER(ctypes.c_float)
        i = ctypes.c_int64
        ip = ctypes.POINTER(ctypes.c_int64)
        i32 = ctypes.c_int32
        lib.oracle_conv2d_ex.argtypes = [f, f, f, i, f, ip, i] + [i] * 10 + [i32]
        lib.oracle_gemm_ex.argtypes = [f, f, f, i, f, ip, i, i, i, i, i, i, i32]
        lib.oracle_dwconv2d_ex.argtypes = [f, f, f, ip, i] + [i] * 9 + [i32]
        lib.oracle_pool2d.argtypes = [f, f, ip, i] + [i] * 8 + [i32]
        _lib = lib
    return _lib


def _fp(a):
    return None if a is None else a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def _host(t):
    return np.ascontiguousarray(t.float().cpu().numpy())


def sample_rows(m: int, tile: int = 128, extra: int = 64, seed: int = 0, full_below: int = 1024):
    """None (every row) for small outputs, else tile-edge rows + random rows."""
    if m <= full_below:
        return None
    rows = set()
    for t0 in range(0, m, tile):
        rows.add(t0)
        rows.add(min(m, t0 + tile) - 1)
    rows.add(m - 1)
    rng = np.random.default_rng(seed)
    rows.update(int(r) for r in rng.integers(0, m, extra))
    return np.array(sorted(rows), dtype=np.int64)


def layer_dims(buf):
    """(M, N) of a LayerBuffers' output."""
    if buf.kind == "gemm":
        return buf.gemm.m, buf.gemm.n
    c = buf.conv
    P = (c.image_h + 2 * c.padding - c.kernel_h) // c.stride + 1
    Q = (c.image_w + 2 * c.padding - c.kernel_w) // c.stride + 1
    return buf.batch * P * Q, c.out_channels


def expect(buf, rows=None):
    """The oracle's fp32 output of one LayerBuffers ([len(rows) or M, N])."""
    lib = oracle_lib()
    M, N = layer_dims(buf)
    n = M if rows is None else len(rows)
    y = np.zeros((n, N), np.float32)
    rp = None if rows is None else rows.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
    act = buf.activation
    x = _host(buf.x)
    if buf.kind in ("maxpool", "avgpool"):
        c = buf.conv
        lib.oracle_pool2d(_fp(x), _fp(y), rp, n, buf.batch, c.image_h, c.image_w, c.in_channels, c.kernel_h,
                          c.kernel_w, c.stride, c.padding, int(buf.kind == "maxpool"))
        return y
    w = _host(buf.w)
    if buf.kind == "dwconv":
        c = buf.conv
        lib.oracle_dwconv2d_ex(_fp(x), _fp(w), _fp(y), rp, n, buf.batch, c.image_h, c.image_w, c.in_channels,
                               c.kernel_h, c.kernel_w, c.stride, c.padding, w.shape[1], act)
        return y
    res = None if buf.res is None else np.ascontiguousarray(_host(buf.res).reshape(M, N))
    if buf.kind == "conv":
        c = buf.conv
        x = np.ascontiguousarray(x[..., :c.in_channels])  # narrow inputs carry zero pad channels
        lib.oracle_conv2d_ex(_fp(x), _fp(w), _fp(res), N, _fp(y), rp, n, buf.batch, c.image_h, c.image_w,
                             c.in_channels, c.out_channels, c.kernel_h, c.kernel_w, c.stride, c.padding, w.shape[1],
                             act)
        return y
    g = buf.gemm
    lib.oracle_gemm_ex(_fp(x), _fp(w), _fp(res), N, _fp(y), rp, n, g.m, g.n, g.k, x.shape[1], w.shape[1], act)
    return y


def got_rows(buf, rows=None):
    M, N = layer_dims(buf)
    y = buf.y.reshape(M, N)
    if rows is not None:
        import torch
        y = y[torch.as_tensor(rows, device=y.device)]
    return y.float().cpu().numpy()


def rel_err(buf, rows=None):
    ref = expect(buf, rows)
    got = got_rows(buf, rows)
    if not np.isfinite(got).all():
        return float("inf")
    return float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30))


def check_model(model, names=None, sample=True, seed=0, tol=TOL):
    """Every layer of a TenantModel against the oracle; returns the worst error.
    ``sample`` False checks every row of every layer."""
    worst = 0.0
    for i, (L, buf) in enumerate(zip(model.layers, model.buffers)):
        M, _ = layer_dims(buf)
        tile = 32 if buf.kind in ("dwconv", "maxpool", "avgpool") else 128
        rows = sample_rows(M, tile=tile, seed=seed + i) if sample else None
        err = rel_err(buf, rows)
        assert err <= tol, f"{names or ''} layer {i} {L.name}: rel err {err:.3e} > {tol}"
        worst = max(worst, err)
    return worst


def poison(models):
    """NaN-fill every layer output, so a layer that reads its input before the
    producing layer stored it cannot pass the check."""
    for m in models:
        for buf in m.buffers:
            buf.y.fill_(float("nan"))
