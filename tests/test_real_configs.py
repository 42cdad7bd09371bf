"""Parity at the BASELINE.json configurations, on the exact programs bench.py
times: default execution options, the reference planner (max_waves 1), the
round program in one persistent launch.  Every layer of every tenant is
compared with the CPU oracle (oracle/conv_oracle.c) on the device's own
inputs, which for these dataflow graphs are the previous layers' device
outputs: tenant 0 on every row, the others on sampled rows that cover every
output tile.  Outputs are NaN-poisoned before the first launch, and a second
launch runs on a new query batch, so a tile that read its input before the
producing layer stored it cannot pass.

Tolerance: ||y - y_ref||_inf / ||y_ref||_inf <= 1e-2 per layer output.
"""
import pytest

import oracle_check

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def run_and_check(eng, rnd, full_tenants=(0,), extra=16):
    s = torch.cuda.Stream()
    g = eng.capture_round(rnd)
    oracle_check.poison(eng.models)
    worst = 0.0
    for launch in range(2):
        if launch:  # a new query batch: every activation changes
            gen = torch.Generator(device="cuda").manual_seed(1234)
            for m in eng.models:
                q = m.query_input
                q.copy_((torch.rand(q.shape, device="cuda", generator=gen) * 2 - 1).to(q.dtype))
            prev = [m.query_output.clone() for m in eng.models]
        s.wait_stream(torch.cuda.current_stream())  # the poison / query writes above
        g.launch(s.cuda_stream)
        torch.cuda.synchronize()
        for i, m in enumerate(eng.models):
            full = i in full_tenants and launch == 0
            worst = max(worst, check(m, f"tenant {i} launch {launch}", full, extra, seed=i))
        if launch:
            assert any(not torch.equal(p, m.query_output) for p, m in zip(prev, eng.models)), \
                "outputs did not change with the query input"
    return worst


def check(model, name, full, extra, seed):
    worst = 0.0
    for li, (L, buf) in enumerate(zip(model.layers, model.buffers)):
        M, _ = oracle_check.layer_dims(buf)
        tile = 32 if buf.kind in ("dwconv", "maxpool", "avgpool") else 128
        rows = None if full else oracle_check.sample_rows(M, tile=tile, extra=extra, seed=seed * 1000 + li,
                                                          full_below=256)
        err = oracle_check.rel_err(buf, rows)
        assert err <= oracle_check.TOL, f"{name} layer {li} {L.name}: rel err {err:.3e}"
        worst = max(worst, err)
    return worst


def variants(rnd):
    info = rnd.tile_info()
    return {"tiles": len(info), "tall": sum(t["rows"] == 256 for t in info),
            "narrow": sum(t["cols"] < 256 and not t["cuda_core"] for t in info),
            "split": sum(t["splits"] > 1 for t in info), "cuda_core": sum(t["cuda_core"] for t in info)}


def assert_plan_matches_host_planner(eng, rnd, policy):
    """gm_plan_round (registered tenants) == gm_plan_round_shapes (the
    host-only planner pinned to the reference in test_round_parity.py)."""
    from paper_1901_00041_b200.sim import plan_round_shapes
    from paper_1901_00041_b200.scheduler import b200_profile
    tenants = [(t, [L.gemm_shape(m.batch) for L in m.layers], 0.040) for t, m in zip(eng.tenants, eng.models)]
    host = plan_round_shapes(tenants, 0, policy, b200_profile())
    assert len(host) == rnd.count
    for h, k, (s, e) in zip(host, rnd.kernels, rnd.times):
        assert [(r.tenant_index, r.layer_index) for r in h.kernel.members] == \
            [(r.tenant_index, r.layer_index) for r in k.members]
        assert h.kernel.planned_cost == k.planned_cost
        assert (h.start, h.end) == (s, e)


def test_headline_config_resnet50_b8():
    """BASELINE configs[1]: 4 tenants x ResNet-50@224, batch 8 (bench.py's headline)."""
    from paper_1901_00041_b200 import workload as W
    from paper_1901_00041_b200.engine import SpaceTimeEngine
    from paper_1901_00041_b200.scheduler import BatchPolicy
    eng = SpaceTimeEngine([W.resnet50(224)] * 4, [8] * 4)
    policy = BatchPolicy(target_batch=0, max_waves=1)
    rnd = eng.plan_round(policy)
    assert_plan_matches_host_planner(eng, rnd, policy)
    v = variants(rnd)
    assert v["tall"] > 0 and v["narrow"] > 0  # the default tile variants are what runs
    run_and_check(eng, rnd)


def test_bert_config_16_tenants_b4():
    """BASELINE configs[3]: 16 tenants x BERT-base 12-layer GEMM chains, seq 128, batch 4."""
    from paper_1901_00041_b200 import workload as W
    from paper_1901_00041_b200.engine import SpaceTimeEngine
    eng = SpaceTimeEngine([W.bert_base_gemms(128, layers=12)] * 16, [4] * 16)
    rnd = eng.plan_round()
    run_and_check(eng, rnd, extra=8)


@pytest.mark.parametrize("batch", [4, 8])
def test_mix_config_224(batch):
    """BASELINE configs[2]: ResNet-50 + VGG-16 + MobileNet-v2 @224 (two each),
    one round program; VGG's fc6 runs split over K (default skinny_min_mb),
    MobileNet's depthwise layers and every pool as CUDA-core tiles."""
    from paper_1901_00041_b200 import workload as W
    from paper_1901_00041_b200.engine import SpaceTimeEngine
    models = [W.resnet50(224), W.vgg16(224), W.mobilenet_v2(224)] * 2
    eng = SpaceTimeEngine(models, [batch] * len(models))
    rnd = eng.plan_round()
    info = rnd.tile_info()
    fc6 = [t for t in info if t["tenant"] == 1 and t["layer"] == len(W.vgg16(224)) - 3]
    assert fc6 and all(t["splits"] > 1 for t in fc6), "VGG fc6 should run split over K by default"
    assert any(t["cuda_core"] for t in info)
    run_and_check(eng, rnd, full_tenants=(2,), extra=8)
