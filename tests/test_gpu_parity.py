"""Super-kernel parity on the GPU: every output of the sm_100a path (through
the C-ABI) against oracle/conv_oracle.c on the same bf16-rounded inputs.

Tolerance (BASELINE north star): ||y - y_ref||_inf / ||y_ref||_inf <= 1e-2
per operator output, bf16 in / fp32 accumulate / bf16 out.
"""
import ctypes
import os

import numpy as np
import pytest

from refshim import ROOT

pytestmark = pytest.mark.gpu
TOL = 1e-2

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def oracle():
    lib = ctypes.CDLL(os.path.join(ROOT, "oracle", "_build", "liboracle.so"))
    f = ctypes.POINTER(ctypes.c_float)
    i = ctypes.c_int64
    lib.oracle_conv2d_nhwc.argtypes = [f, f, f] + [i] * 10 + [ctypes.c_int32]
    lib.oracle_gemm_nt.argtypes = [f, f, f, i, i, i, i, i, ctypes.c_int32]
    lib.oracle_dwconv2d_nhwc.argtypes = [f, f, f] + [i] * 9 + [ctypes.c_int32]
    return lib


def fp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def expect(oracle, L, relu=False):
    """fp32 oracle output of one LayerBuffers (reads the device tensors' bf16 values)."""
    if L.kind in ("maxpool", "avgpool"):
        import oracle_check
        return oracle_check.expect(L)
    x = np.ascontiguousarray(L.x.float().cpu().numpy())
    w = np.ascontiguousarray(L.w.float().cpu().numpy())
    if L.kind == "dwconv":
        c = L.conv
        P = (c.image_h + 2 * c.padding - c.kernel_h) // c.stride + 1
        Q = (c.image_w + 2 * c.padding - c.kernel_w) // c.stride + 1
        y = np.zeros((L.batch * P * Q, c.out_channels), np.float32)
        oracle.oracle_dwconv2d_nhwc(fp(x), fp(w), fp(y), L.batch, c.image_h, c.image_w, c.in_channels, c.kernel_h,
                                    c.kernel_w, c.stride, c.padding, w.shape[1], int(relu))
    elif L.kind == "conv":
        c = L.conv
        x = np.ascontiguousarray(x[..., :c.in_channels])  # narrow inputs carry zero pad channels
        P = (c.image_h + 2 * c.padding - c.kernel_h) // c.stride + 1
        Q = (c.image_w + 2 * c.padding - c.kernel_w) // c.stride + 1
        y = np.zeros((L.batch * P * Q, c.out_channels), np.float32)
        oracle.oracle_conv2d_nhwc(fp(x), fp(w), fp(y), L.batch, c.image_h, c.image_w, c.in_channels,
                                  c.out_channels, c.kernel_h, c.kernel_w, c.stride, c.padding, w.shape[1], int(relu))
    else:
        g = L.gemm
        y = np.zeros((g.m, g.n), np.float32)
        oracle.oracle_gemm_nt(fp(x), fp(w), fp(y), g.m, g.n, g.k, x.shape[1], w.shape[1], int(relu))
    return y


def rel_err(L, ref):
    got = L.y.float().cpu().numpy().reshape(ref.shape)
    assert np.isfinite(got).all()
    return float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30))


def conv_layer(b, hw, cin, cout, r, stride, pad, relu=False, seed=0, pitch=0):
    from paper_1901_00041_b200.runtime import LayerBuffers
    from paper_1901_00041_b200.scheduler import ConvSpec
    g = torch.Generator().manual_seed(seed)
    K = r * r * cin
    ldw = (K + 7) // 8 * 8
    x = (torch.rand(b, hw, hw, cin, generator=g) * 2 - 1).to(torch.bfloat16)
    if pitch:
        xp = torch.zeros(b, hw, hw, pitch, dtype=torch.bfloat16)
        xp[..., :cin] = x
        x = xp
    x = x.cuda()
    w = torch.zeros(cout, ldw, dtype=torch.bfloat16)
    w[:, :K] = (torch.randn(cout, K, generator=g) * (2.0 / K) ** 0.5).to(torch.bfloat16)
    P = (hw + 2 * pad - r) // stride + 1
    y = torch.full((b * P * P, cout), float("nan"), dtype=torch.bfloat16, device="cuda")
    return LayerBuffers("conv", x, w.cuda(), y, conv=ConvSpec(hw, hw, r, r, cin, cout, stride, pad), batch=b, relu=relu)


def dw_layer(b, hw, c, stride, relu=False, seed=0):
    """Depthwise 3x3 pad 1 (MobileNet-v2): the super-kernel's CUDA-core tile type."""
    from paper_1901_00041_b200.runtime import LayerBuffers
    from paper_1901_00041_b200.scheduler import ConvSpec
    g = torch.Generator().manual_seed(seed)
    x = (torch.rand(b, hw, hw, c, generator=g) * 2 - 1).to(torch.bfloat16).cuda()
    w = (torch.randn(c, 9, generator=g) * (2.0 / 9) ** 0.5).to(torch.bfloat16).cuda()
    P = (hw + 2 - 3) // stride + 1
    y = torch.full((b * P * P, c), float("nan"), dtype=torch.bfloat16, device="cuda")
    return LayerBuffers("dwconv", x, w, y, conv=ConvSpec(hw, hw, 3, 3, c, c, stride, 1), batch=b, relu=relu)


def pool_layer(kind, b, hw, c, r, stride, pad, seed=0):
    """Max / average pool: a CUDA-core tile type (staged through the operand
    ring when its input window fits one TMA box, else the register path)."""
    from paper_1901_00041_b200.runtime import LayerBuffers
    from paper_1901_00041_b200.scheduler import ConvSpec
    g = torch.Generator().manual_seed(seed)
    x = (torch.rand(b, hw, hw, c, generator=g) * 2 - 1).to(torch.bfloat16).cuda()
    P = (hw + 2 * pad - r) // stride + 1
    y = torch.full((b * P * P, c), float("nan"), dtype=torch.bfloat16, device="cuda")
    return LayerBuffers(kind, x, None, y, conv=ConvSpec(hw, hw, r, r, c, c, stride, pad), batch=b)


def gemm_layer(m, n, k, relu=False, seed=0):
    from paper_1901_00041_b200.runtime import LayerBuffers
    from paper_1901_00041_b200.scheduler import GemmShape
    g = torch.Generator().manual_seed(seed)
    ld = (k + 7) // 8 * 8
    x = torch.zeros(m, ld, dtype=torch.bfloat16)
    x[:, :k] = (torch.rand(m, k, generator=g) * 2 - 1).to(torch.bfloat16)
    w = torch.zeros(n, ld, dtype=torch.bfloat16)
    w[:, :k] = (torch.randn(n, k, generator=g) / k ** 0.5).to(torch.bfloat16)
    y = torch.full((m, n), float("nan"), dtype=torch.bfloat16, device="cuda")
    return LayerBuffers("gemm", x.cuda(), w.cuda(), y, gemm=GemmShape(m, n, k), relu=relu)


CASES = {
    "gemm conv2_2 256x128x1152": lambda: gemm_layer(256, 128, 1152),
    "gemm tails 200x72x100": lambda: gemm_layer(200, 72, 100),
    "gemm 1000x1000x520": lambda: gemm_layer(1000, 1000, 520),
    "gemm M=1 (fc b1)": lambda: gemm_layer(1, 1000, 2048),
    "gemm bert qkv 128x2304x768": lambda: gemm_layer(128, 2304, 768),
    "gemm relu": lambda: gemm_layer(130, 136, 200, relu=True),
    "gemm N=8 (rnn-matvec at N=8) 512x8x512": lambda: gemm_layer(512, 8, 512),
    "gemm square-256": lambda: gemm_layer(256, 256, 256),
    "conv 3x3 s1 p1 16x16x128->128 b2 (im2col TMA)": lambda: conv_layer(2, 16, 128, 128, 3, 1, 1),
    "conv 3x3 s2 p1 28x28x64->128": lambda: conv_layer(1, 28, 64, 128, 3, 2, 1),
    "conv 1x1 s1 14x14x256->512 b3 (tiled GEMM)": lambda: conv_layer(3, 14, 256, 512, 1, 1, 0),
    "conv 1x1 s2 28x28x256->512 (im2col stride)": lambda: conv_layer(1, 28, 256, 512, 1, 2, 0),
    "conv 7x7 s2 p3 stem 64x64x3->64 b2 (row fold)": lambda: conv_layer(2, 64, 3, 64, 7, 2, 3),
    "conv 7x7 s2 p3 row fold odd 37x37x3->64": lambda: conv_layer(1, 37, 3, 64, 7, 2, 3),
    "conv 3x3 s2 p1 row fold 33x33x3->32 b3": lambda: conv_layer(3, 33, 3, 32, 3, 2, 1),
    "conv 3x3 s1 p1 row fold Cin=8 9x9->16 (M<128)": lambda: conv_layer(1, 9, 8, 16, 3, 1, 1),
    "conv 7x7 s2 p3 stem 64x64x3->64 b2 (narrow im2col)": lambda: conv_layer(2, 64, 3, 64, 7, 2, 3, pitch=8),
    "conv 3x3 s2 p1 narrow 33x33x3->32": lambda: conv_layer(3, 33, 3, 32, 3, 2, 1, pitch=8),
    "conv 3x3 s1 p1 narrow Cin=8 9x9->16 (M<128)": lambda: conv_layer(1, 9, 8, 16, 3, 1, 1, pitch=8),
    "conv 3x3 s1 7x7x512->512 b1 (M=49)": lambda: conv_layer(1, 7, 512, 512, 3, 1, 1),
    "conv 5x5 s1 p2 12x12x64->96": lambda: conv_layer(2, 12, 64, 96, 5, 1, 2),
    "conv 3x3 Cin=32 (pre-pass) 10x10x32->64": lambda: conv_layer(1, 10, 32, 64, 3, 1, 1),
    "conv 3x3 relu": lambda: conv_layer(1, 12, 64, 64, 3, 1, 1, relu=True),
    "dwconv 3x3 s1 14x14x96 b2": lambda: dw_layer(2, 14, 96, 1),
    "dwconv 3x3 s2 15x15x144 (odd, stride 2)": lambda: dw_layer(1, 15, 144, 2),
    "dwconv 3x3 s1 56x56x32 b3 (many tiles)": lambda: dw_layer(3, 56, 32, 1),
    "dwconv 3x3 s1 7x7x200 relu (partial channel tile)": lambda: dw_layer(1, 7, 200, 1, relu=True),
    "dwconv 3x3 s2 300x300x16 (register path: window wider than a box)": lambda: dw_layer(1, 300, 16, 2),
    "dwconv 3x3 s2 112x112x96 b1 (staged, 48 KB ring slots)": lambda: dw_layer(1, 112, 96, 2),
    "maxpool 3x3 s2 p1 30x30x64 b2 (stem pool, staged)": lambda: pool_layer("maxpool", 2, 30, 64, 3, 2, 1),
    "maxpool 3x3 s2 p1 13x13x24 b2 (8-channel tiles)": lambda: pool_layer("maxpool", 2, 13, 24, 3, 2, 1),
    "maxpool 2x2 s2 16x16x128 (VGG pool)": lambda: pool_layer("maxpool", 1, 16, 128, 2, 2, 0),
    "maxpool 2x2 s2 300x300x8 (register path: window wider than a box)": lambda: pool_layer("maxpool", 1, 300, 8, 2, 2, 0),
    "avgpool 7x7 global 7x7x2048 b3": lambda: pool_layer("avgpool", 3, 7, 2048, 7, 1, 0),
}


@pytest.fixture(scope="module")
def registered():
    from paper_1901_00041_b200.runtime import Context
    ctx = Context(0)
    names = list(CASES)
    layers = [CASES[n]() for n in names]
    tenant = ctx.register_tenant(layers)
    return ctx, tenant, names, layers


@pytest.mark.parametrize("idx", range(len(CASES)))
def test_single_member_matches_oracle(registered, oracle, idx):
    ctx, tenant, names, layers = registered
    L = layers[idx]
    L.y.fill_(float("nan"))
    assert ctx.launch_members([(tenant, idx)]) >= 1
    torch.cuda.synchronize()
    err = rel_err(L, expect(oracle, L, L.relu))
    assert err <= TOL, f"{names[idx]}: {err:.3e}"


def test_heterogeneous_members_in_one_launch(registered, oracle):
    """Every case above as members of ONE super-kernel (variable-size packing)."""
    ctx, tenant, names, layers = registered
    for L in layers:
        L.y.fill_(float("nan"))
    ctx.launch_members([(tenant, i) for i in range(len(layers))])
    torch.cuda.synchronize()
    for n, L in zip(names, layers):
        assert rel_err(L, expect(oracle, L, L.relu)) <= TOL, n


def test_tile_table_matches_planner_blocks(registered):
    """gm_build_tile_table == thread_blocks under the b200 profile (member, m, n order)."""
    from paper_1901_00041_b200 import scheduler as S
    ctx, tenant, _, layers = registered
    q = S.RequestQueue()
    shapes = [ctx.layer_shape(tenant, i) for i in range(4)]
    for i, s in enumerate(shapes):
        q.enqueue(S.KernelRequest(i + 1, tenant, s, 0, 10**9, i))
    p = S.BatchPolicy(target_batch=1, allow_variable_size=True)
    sks = S.form_batches(q, 10**8, p, ctx.device)
    for sk in sks:
        tt = sk.tile_table(ctx.device)
        assert len(tt) == sk.planned_cost.blocks
        expect_tt = [(j, a, b) for j, r in enumerate(sk.members)
                     for a in range(-(-r.shape.m // ctx.device.tile_m)) for b in range(-(-r.shape.n // ctx.device.tile_n))]
        assert tt == expect_tt


def small_engine(tenants=3, batch=2, image=64, options=None):
    from paper_1901_00041_b200 import workload as W
    from paper_1901_00041_b200.engine import SpaceTimeEngine
    return SpaceTimeEngine([W.resnet18(image)] * tenants, [batch] * tenants, options=options or {})


def check_engine(eng, oracle=None):
    """Every layer of every tenant (dataflow graphs: each layer on the device's
    own input, i.e. its producer's output) against the oracle, every row."""
    import oracle_check
    for i, m in enumerate(eng.models):
        oracle_check.check_model(m, names=f"tenant {i}", sample=False)


def clear(eng):
    import oracle_check
    oracle_check.poison(eng.models)


def test_round_program_matches_oracle(oracle):
    """A whole 3-tenant ResNet-18 round as ONE persistent launch (device-side deps)."""
    eng = small_engine()
    rnd = eng.plan_round()
    assert all(len(k.members) == 3 for k in rnd.kernels)
    clear(eng)
    s = torch.cuda.Stream()
    rnd.launch_round(s.cuda_stream)
    torch.cuda.synchronize()
    check_engine(eng, oracle)


def test_modes_compute_identical_bits(oracle):
    """Packed (per plan), round program, time-only and space-only run the same
    kernel code: outputs are bit-identical across modes."""
    eng = small_engine(tenants=2)
    rnd = eng.plan_round()
    s = torch.cuda.Stream()
    outs = []
    for launch in (lambda: rnd.launch_round(s.cuda_stream), lambda: rnd.launch(s.cuda_stream),
                   lambda: eng.capture_serial("time_only").launch(s.cuda_stream),
                   lambda: eng.capture_serial("space_only").launch(s.cuda_stream),
                   lambda: eng.capture_round(rnd).launch(s.cuda_stream)):
        clear(eng)
        launch()
        torch.cuda.synchronize()
        outs.append([b.y.clone() for m in eng.models for b in m.buffers])
    for other in outs[1:]:
        for a, b in zip(outs[0], other):
            assert torch.equal(a, b)
    check_engine(eng, oracle)


def test_heterogeneous_models_round_program(oracle):
    """BASELINE configs[2]'s model mix in one round program: MobileNet-v2
    (depthwise CUDA-core tiles + 1x1 tensor-core tiles), ResNet-18 and VGG-16
    tenants with different layer lists, per-tenant device-side layer deps."""
    from paper_1901_00041_b200 import workload as W
    from paper_1901_00041_b200.engine import SpaceTimeEngine
    eng = SpaceTimeEngine([W.mobilenet_v2(64, classifier=False), W.resnet18(64), W.vgg16(32, classifier=False)],
                          [2, 2, 1])
    rnd = eng.plan_round()
    clear(eng)
    s = torch.cuda.Stream()
    rnd.launch_round(s.cuda_stream)
    torch.cuda.synchronize()
    check_engine(eng, oracle)
    # and the same members one launch per formed super-kernel
    clear(eng)
    rnd.launch(s.cuda_stream)
    torch.cuda.synchronize()
    check_engine(eng, oracle)


@pytest.mark.parametrize("options", [{"split_k": 1}, {"narrow_min_tiles": 32}, {"pdl": 0}, {"row_fold": 0},
                                     {"split_k": 1, "max_splits": 8, "narrow_min_tiles": 64},
                                     {"tall_min_tiles": 1}, {"tall_min_tiles": 1, "narrow_min_tiles": 0},
                                     {"tall_tiles": 0, "narrow_min_tiles": 0}, {"critical_order": 0},
                                     {"critical_order": 1}, {"critical_order": 2, "greedy_schedule": 1},
                                     {"ring_layouts": 0}, {"skinny_min_mb": 0},
                                     {"skinny_min_mb": 1, "split_min_kb": 2},
                                     {"skinny_min_mb": 1, "split_min_kb": 1, "skinny_max_splits": 64},
                                     {"split_wide_kb": 2, "narrow_min_tiles": 64},
                                     {"split_wide_kb": 2, "narrow_min_tiles": 64, "split_min_kb": 1, "max_splits": 8}])
def test_execution_options_keep_results(oracle, options):
    eng = small_engine(tenants=2, batch=4, options=options)
    rnd = eng.plan_round()
    if "split_wide_kb" in options:  # the option took effect: 128-column split tiles
        assert any(t["splits"] > 1 and t["cols"] == 128 for t in rnd.tile_info())
    clear(eng)
    s = torch.cuda.Stream()
    rnd.launch_round(s.cuda_stream)
    torch.cuda.synchronize()
    check_engine(eng, oracle)


def test_serve_round_e2e_host_buffers(oracle):
    """The gated e2e program (per-tenant H2D opens that tenant's chain): the
    host results are the dataflow chain of the host inputs."""
    eng = small_engine(tenants=2)
    s = torch.cuda.Stream()
    h_in = [m.query_input.cpu().pin_memory() for m in eng.models]
    h_out = [torch.empty_like(m.query_output, device="cpu").pin_memory() for m in eng.models]
    clear(eng)
    for _ in range(3):
        rnd = eng.serve_round(h_in, h_out, s)
    assert len(eng._graphs) == 1  # steady state: one cached launch program
    for m, h in zip(eng.models, h_out):
        assert torch.equal(h, m.query_output.cpu())
    check_engine(eng, oracle)
    # a new host batch through the cached program: new results, still the oracle's
    first = [h.clone() for h in h_out]
    g = torch.Generator().manual_seed(7)
    for h in h_in:
        h.copy_((torch.rand(h.shape, generator=g) * 2 - 1).to(h.dtype))
    clear(eng)
    eng.serve_round(h_in, h_out, s)
    assert len(eng._graphs) == 1
    for a, b, m, hi in zip(first, h_out, eng.models, h_in):
        assert not torch.equal(a, b)
        assert torch.equal(m.query_input.cpu(), hi)
    check_engine(eng, oracle)


def _producer_rows(L, P, b, r0, r1, residual):
    """Python restatement of Runtime::producer_rows for the test: rows of
    producer layer P's output that consumer L's output rows [r0, r1) read."""
    np_ = P.gemm_shape(b).n
    mp = P.gemm_shape(b).m
    if residual:
        n = L.gemm_shape(b).n
        lo, hi = r0 * n // np_, ((r1 - 1) * n + n - 1) // np_
    elif L.kind == "gemm":
        s = L.gemm_shape(b)
        pitch = np_ * mp // s.m  # the source viewed as [rows, -1]
        lo = (L.src_col + r0 * pitch) // np_
        hi = (L.src_col + (r1 - 1) * pitch + s.k - 1) // np_
    else:
        c = L.conv
        P_ = (c.image_h + 2 * c.padding - c.kernel_h) // c.stride + 1
        Q_ = (c.image_w + 2 * c.padding - c.kernel_w) // c.stride + 1

        def row(m, last):
            bb, p = m // (P_ * Q_), (m % (P_ * Q_)) // Q_
            ih = min(c.image_h - 1, p * c.stride - c.padding + c.kernel_h - 1) if last else \
                max(0, p * c.stride - c.padding)
            return (bb * c.image_h + ih) * c.image_w + (c.image_w - 1 if last else 0)
        lo, hi = row(r0, False), row(r1 - 1, True)
    return max(0, lo), min(mp - 1, hi)


def test_round_dependency_graph():
    """Device tile table edges (gm_round_tile_info): every tile waits on
    exactly the producer row blocks its input rows and residual rows come
    from (re-derived here from the layer geometry), never on its own counter,
    and the counters anything waits on are published."""
    from paper_1901_00041_b200 import workload as W
    from paper_1901_00041_b200.engine import SpaceTimeEngine
    models = [W.resnet18(64), W.mobilenet_v2(64, classifier=False), W.bert_base_gemms(16, 2)]
    eng = SpaceTimeEngine(models, [2, 2, 2])
    rnd = eng.plan_round()
    info = rnd.tile_info()
    base, rows = {}, {}
    for t in info:
        key = (t["tenant"], t["layer"])
        rows[key] = t["rows"]
        if t["m_tile"] == 0 and t["done"] >= 0:
            base[key] = t["done"]
    needed = set()
    for t in info:
        L = models[t["tenant"]][t["layer"]]
        for d, n in ((t["dep"], t["dep_n"]), (t["rdep"], t["rdep_n"])):
            if d >= 0:
                needed.update(range(d, d + n))
                assert not (d <= t["done"] < d + n)
        r0 = t["m_tile"] * t["rows"]
        r1 = min(L.gemm_shape(2).m, r0 + t["rows"])
        for which, (d, n) in (("src", (t["dep"], t["dep_n"])), ("res", (t["rdep"], t["rdep_n"]))):
            j = L.src if which == "src" else L.res
            if j is None:
                assert which == "res" or t["layer"] == 0 or d == base[(t["tenant"], t["layer"] - 1)]
                if which == "res":
                    assert d == -1
                continue
            P = models[t["tenant"]][j]
            lo, hi = _producer_rows(L, P, 2, r0, r1, which == "res")
            pr = rows[(t["tenant"], j)]
            assert (d, n) == (base[(t["tenant"], j)] + lo // pr, hi // pr - lo // pr + 1), (t, which)
    published = {t["done"] for t in info if t["done"] >= 0}
    assert needed <= published


@pytest.mark.parametrize("options", [{}, {"greedy_schedule": 1}, {"dynamic_schedule": 1}, {"critical_order": 0},
                                     {"split_k": 1, "narrow_min_tiles": 64}, {"staged_cc": 0},
                                     {"split_wide_kb": 2, "narrow_min_tiles": 64, "split_min_kb": 1}])
def test_dataflow_chain_every_schedule(oracle, options):
    """A chained ResNet-18 + MobileNet-v2 round (layer l reads layer l-1's
    output, residual adds read earlier layers) under every tile schedule,
    outputs poisoned first: results depend on dependency order."""
    from paper_1901_00041_b200 import workload as W
    from paper_1901_00041_b200.engine import SpaceTimeEngine
    eng = SpaceTimeEngine([W.resnet18(64), W.mobilenet_v2(64)], [2, 3], options=options)
    rnd = eng.plan_round()
    s = torch.cuda.Stream()
    for launch in (lambda: rnd.launch_round(s.cuda_stream), lambda: rnd.launch(s.cuda_stream)):
        clear(eng)
        launch()
        torch.cuda.synchronize()
        check_engine(eng, oracle)


def test_serve_rounds_pipelined_matches_single_rounds():
    """Double-buffered back-to-back rounds: every step's host results equal a
    synchronous serve_round of the same host batch (no staging-buffer race)."""
    eng = small_engine(tenants=2)
    s = torch.cuda.Stream()
    g = torch.Generator().manual_seed(3)
    steps = []
    for _ in range(5):
        h_in = [(torch.randn(m.query_input.shape, generator=g) * 0.5).to(torch.bfloat16).pin_memory()
                for m in eng.models]
        h_out = [torch.empty_like(m.query_output, device="cpu").pin_memory() for m in eng.models]
        steps.append((h_in, h_out))
    eng.serve_rounds(steps, s)
    for h_in, h_out in steps:
        ref = [torch.empty_like(h).pin_memory() for h in h_out]
        eng.serve_round(h_in, ref, s)
        for a, b in zip(h_out, ref):
            assert torch.equal(a, b)
    with pytest.raises(ValueError):
        eng.serve_rounds([(steps[0][0][:1], steps[0][1])], s)


def test_no_silent_fallback_on_bad_registration():
    from paper_1901_00041_b200.runtime import Context, LayerBuffers
    from paper_1901_00041_b200.scheduler import GemmShape
    ctx = Context(0)
    x = torch.zeros(64, 100, dtype=torch.bfloat16, device="cuda")  # 200 B rows: not 16 B aligned strides
    w = torch.zeros(64, 100, dtype=torch.bfloat16, device="cuda")
    y = torch.zeros(64, 64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError, match="multiple of 8"):
        ctx.register_tenant([LayerBuffers("gemm", x, w, y, gemm=GemmShape(64, 64, 100))])
