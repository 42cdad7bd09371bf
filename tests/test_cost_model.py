"""Cost model known answers (proj/tests/test_cost_model.cpp) through the C-ABI."""
import random

import pytest

from paper_1901_00041_b200.scheduler import (ConvSpec, DeviceSpec, GemmShape, KernelGroup, batch_inputs,
                                             dispatch_duration, gemm_bytes, gemm_flops, im2col_gemm_dims,
                                             thread_blocks, to_ns, b200_profile, v100_profile)


def cost_device():  # test_cost_model.cpp:11-21
    return DeviceSpec(peak_flops=14e12, mem_bandwidth=900e9, sm_count=80, blocks_per_sm=2, launch_overhead=5e-6,
                      tile_m=64, tile_n=64)


D = cost_device()
CONV = GemmShape(256, 128, 1152)


def test_gemm_flops_and_bytes():  # :25-35
    assert gemm_flops(CONV) == 75497472
    assert gemm_flops(GemmShape(1, 1, 1)) == 2
    assert gemm_flops(GemmShape(512, 1, 512)) == 524288
    assert gemm_bytes(GemmShape(1, 1, 1), 4) == 12
    assert gemm_bytes(CONV, 4) == 1900544
    assert gemm_bytes(GemmShape(512, 1, 512), 4) == 1052672


def test_thread_blocks():  # :37-42
    assert thread_blocks(CONV, D) == 8
    assert thread_blocks(GemmShape(64, 64, 999), D) == 1
    assert thread_blocks(GemmShape(65, 64, 999), D) == 2


def test_single_kernel_low_occupancy():  # :44-52
    c = dispatch_duration(CONV, D, 160, 1)
    assert (c.blocks, c.waves) == (8, 1)
    assert c.duration == pytest.approx(75497472.0 / (14e12 * 0.05) + 5e-6, rel=1e-12)


def test_full_wave_same_time():  # :54-65
    one = dispatch_duration(CONV, D, 160, 1)
    twenty = dispatch_duration([KernelGroup(CONV, 20)], D, 160, 1)
    assert (twenty.blocks, twenty.waves, twenty.flops) == (160, 1, 20 * one.flops)
    assert twenty.duration - 5e-6 == pytest.approx(one.duration - 5e-6, rel=1e-12)


def test_exact_fill_and_bad_inputs():  # :67-87
    c = dispatch_duration([KernelGroup(GemmShape(64, 64, 64), 160)], D, 160, 1)
    assert c.waves == 1
    assert c.duration == pytest.approx(5e-6 + max(c.flops / 14e12, c.bytes / 900e9), rel=1e-12)
    with pytest.raises(ValueError, match="^empty dispatch$"):
        dispatch_duration([], D, 160, 1)
    with pytest.raises(ValueError, match="slot_budget out of range"):
        dispatch_duration(GemmShape(1, 1, 1), D, 0, 1)
    with pytest.raises(ValueError, match="slot_budget out of range"):
        dispatch_duration(GemmShape(1, 1, 1), D, 161, 1)


def test_duration_exceeds_launch_overhead():  # :89-100 (seeded property)
    rng = random.Random(7)
    for _ in range(200):
        s = GemmShape(rng.randint(1, 512), rng.randint(1, 512), rng.randint(1, 512))
        launches = rng.randint(1, 4)
        assert dispatch_duration(s, D, 160, launches).duration > launches * D.launch_overhead


def test_wave_quantization():  # :102-132
    prev_d, prev_t = 0.0, 0.0
    for r in range(1, 61):
        c = dispatch_duration([KernelGroup(CONV, r)], D, 160, 1)
        assert c.waves == (r * 8 + 159) // 160
        assert c.duration >= prev_d * (1 - 1e-12)
        prev_d = c.duration
        eff = c.blocks / (c.waves * 160)
        assert (eff == 1.0) == ((r * 8) % 160 == 0)
        t = c.flops / c.duration
        if r <= 20:
            assert t >= prev_t
            prev_t = t
        assert t < D.peak_flops


def test_im2col_and_batching():  # :134-159
    assert im2col_gemm_dims(ConvSpec(3, 3, 3, 3, 1, 1, 1, 0)) == GemmShape(1, 1, 9)
    assert im2col_gemm_dims(ConvSpec(16, 16, 3, 3, 128, 128, 1, 1)) == CONV
    with pytest.raises(ValueError, match="im2col: non-positive output dims"):
        im2col_gemm_dims(ConvSpec(2, 2, 5, 5, 1, 1, 1, 0))
    assert batch_inputs(CONV, 26) == GemmShape(6656, 128, 1152)
    rng = random.Random(21)
    for _ in range(100):
        s = GemmShape(rng.randint(1, 300), rng.randint(1, 300), rng.randint(1, 300))
        b = rng.randint(1, 40)
        assert gemm_flops(batch_inputs(s, b)) == b * gemm_flops(s)


def test_reference_goldens_v100():  # SURVEY §8(c) probes
    d = v100_profile()
    for r in (1, 2, 10, 20):
        assert dispatch_duration([KernelGroup(CONV, r)], d, 160, 1).duration == 1.1005353142857142e-4
    for r in (21, 40):
        assert dispatch_duration([KernelGroup(CONV, r)], d, 160, 1).duration == 2.1790706285714284e-4
    assert dispatch_duration([KernelGroup(CONV, 120)], d, 160, 1).duration == 6.4932118857142867e-4


def test_to_ns_rounds_half_away():
    assert to_ns(1.5e-9) == 2 and to_ns(2.5e-9) == 3 and to_ns(0.05) == 50_000_000


def test_b200_profile_is_the_kernel_tile():
    d = b200_profile()
    assert (d.tile_m, d.tile_n, d.sm_count, d.blocks_per_sm) == (128, 256, 148, 1)
    d.validate()


def test_latency_floor_extension():
    """The b200 latency term: zero in every reference profile (parity), else a
    plan lasts at least waves x (tile_latency + kblocks(K_max) x kblock_latency)."""
    from paper_1901_00041_b200.scheduler import GemmShape, KernelGroup, b200_profile, dispatch_duration
    d = b200_profile()
    assert d.tile_latency == 0 and d.kblock_latency == 0
    g = [KernelGroup(GemmShape(392, 512, 4608), 1), KernelGroup(GemmShape(392, 512, 512), 2)]
    base = dispatch_duration(g, d, d.slot_total(), 1)
    d.tile_latency, d.kblock_latency = 3e-6, 0.2e-6
    lat = dispatch_duration(g, d, d.slot_total(), 1)
    assert lat.waves == base.waves == 1
    assert lat.duration == pytest.approx(d.launch_overhead + 3e-6 + 72 * 0.2e-6)
    d.kblock_latency = 0.0
    d.tile_latency = 1e-12  # below the roofline: unchanged
    assert dispatch_duration(g, d, d.slot_total(), 1).duration == base.duration
    d.tile_latency = -1.0
    with pytest.raises(ValueError):
        d.validate()


def test_calibrated_b200_profile_keeps_physical_peaks():
    """profiles/b200_calibrated.json (tools/calibrate_b200.py on a B200): the
    peaks are the measured dense bf16 burst and HBM copy bandwidth, the latency
    floor is fitted, and the held-out error is what DESIGN reports."""
    import json
    import os
    from paper_1901_00041_b200.scheduler import GemmShape, KernelGroup, b200_calibrated_profile, b200_profile, \
        dispatch_duration
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                        "b200_calibrated.json")
    cal = json.load(open(path))
    d = b200_calibrated_profile()
    assert d.peak_flops == cal["fitted"]["peak_flops"] and 1.5e15 < d.peak_flops < 2.3e15
    assert d.mem_bandwidth == cal["fitted"]["mem_bandwidth"] and 5e12 < d.mem_bandwidth < 8.5e12
    assert d.tile_latency > 0 and d.kblock_latency > 0
    assert cal["median_rel_err_held_out"]["calibrated"] < 0.15 < cal["median_rel_err_held_out"]["nominal"]
    # a one-wave, narrow, long-K plan is latency-bound on the device: the
    # calibrated floor (waves x (tile + 72 k-blocks)) exceeds its roofline
    g = [KernelGroup(GemmShape(128 * 148, 64, 4608), 1)]
    cal_d = dispatch_duration(g, d, d.slot_total(), 1)
    assert cal_d.duration >= cal_d.waves * (d.tile_latency + 72 * d.kblock_latency)
    assert cal_d.duration > dispatch_duration(g, b200_profile(), d.slot_total(), 1).duration
