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
