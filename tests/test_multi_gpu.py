"""Tenant-sharded multi-GPU host logic, world_size 2 over gloo on CPU.

Each rank owns a placement shard, runs the space-time driver for its tenants
only (no data-path collective), and the p99 is merged with one all-gather.
The merged result must equal the single-process computation over all tenants.
"""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1901_00041_b200.placement import merged_percentile, place_tenants, tenants_of


def test_placement_homogeneous_is_mod_g():
    assert place_tenants([(100, 10)] * 64, 8) == [t % 8 for t in range(64)]


def test_placement_lpt_balances_heterogeneous():
    demands = [(8, 1), (30, 2), (1, 1), (30, 2), (8, 1), (1, 1)]
    p = place_tenants(demands, 2)
    loads = [sum(d[0] for d, g in zip(demands, p) if g == k) for k in range(2)]
    assert sorted(loads) == [39, 39] and p == place_tenants(demands, 2)  # deterministic
    with pytest.raises(ValueError):
        place_tenants(demands, 0)


def _latencies(tenant_ids):
    """Per-pass latencies of a tenant subset from the space-time driver."""
    from paper_1901_00041_b200.scheduler import BatchPolicy, GemmShape, v100_profile
    from paper_1901_00041_b200.sim import SpaceTimeConfig, simulate_space_time
    tr = simulate_space_time(SpaceTimeConfig(device=v100_profile(), layers=[GemmShape(256, 128, 1152)] * 3,
                                             tenants=len(tenant_ids), duration=0.01, scheduler=BatchPolicy(target_batch=0)))
    return [(c.complete_time - c.enqueue_time) * 1e-9 for c in tr.completions]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    placement = place_tenants([(1000, 10)] * 8, world)
    mine = tenants_of(rank, placement)
    lat = _latencies(mine)
    p99 = merged_percentile(lat, 99.0)
    q.put((rank, mine, p99, lat))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shards_and_merged_p99():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    shards = [r[1] for r in res]
    assert sorted(shards[0] + shards[1]) == list(range(8)) and not set(shards[0]) & set(shards[1])
    from paper_1901_00041_b200.scheduler import percentile_nearest_rank
    union = res[0][3] + res[1][3]
    assert res[0][2] == res[1][2] == percentile_nearest_rank(union, 99.0)


def _shard_plan_parity(rank, world, port, q):
    """One rank of a C5-style job: 16 ResNet-50 b8 tenants placed over the
    ranks (homogeneous: tenant mod G), this rank's shard planned by the product
    planner (gm_plan_round) and by the unmodified reference run_space_time
    (oracle/_ref); the dispatch streams must agree member for member."""
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    for p in (here, os.path.dirname(here)):
        if p not in sys.path:
            sys.path.insert(0, p)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import refshim
    from test_round_parity import gemm_list, product_round, reference_first_pass
    placement = place_tenants([(1000, 10)] * 16, world)
    mine = tenants_of(rank, placement)
    shapes = gemm_list("resnet50@224", 8)
    got = product_round(shapes, len(mine), "b200", 0.040)
    span = got[-1].end if got else 0
    events, _ = reference_first_pass(refshim.ref_call, shapes, len(mine), "b200", 0.040,
                                     duration=max(4 * span * 1e-9, 1e-3))
    first = [e for e in events if all(p == 0 for _, _, p in e["who"])]
    same = len(first) == len(got) and all(
        [(r.tenant_index, r.layer_index) for r in g.kernel.members] == [(t, l) for t, l, _ in e["who"]] and
        g.kernel.planned_cost.flops == e["flops"] and g.end - g.start == e["end"] - e["start"]
        for g, e in zip(got, first))
    # the shards' plan streams are gathered once (off the hot path) for the report
    sizes = [None] * world
    dist.all_gather_object(sizes, len(got))
    q.put((rank, mine, same, sizes))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shard_plans_equal_reference():
    import refshim
    if not refshim.have_ref():
        pytest.skip("oracle/_ref not built (make -C oracle ref)")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_shard_plan_parity, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [list(range(0, 16, 2)), list(range(1, 16, 2))]
    assert all(r[2] for r in res), "a shard's plan differs from the reference planner on that shard"
    assert res[0][3] == res[1][3] and res[0][3][0] > 0  # identical shards, identical plan lengths


def test_least_loaded_readmission_target():
    from paper_1901_00041_b200.placement import least_loaded
    loads = [(40, 5), (10, 9), (10, 2), (30, 1)]
    assert least_loaded(loads) == 2
    assert least_loaded(loads, exclude=[2]) == 1
    assert least_loaded([(5, 5), (5, 5)], exclude=[0]) == 1
    with pytest.raises(ValueError):
        least_loaded([(1, 1)], exclude=[0])
