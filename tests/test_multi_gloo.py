"""N>1 host logic of the bench on CPU (two gloo ranks): one rank drives the
whole fleet with one decision authority, the others only join the barriers
and the max over ranks; the fleet mix is one seeded mix for all GPUs."""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2107_08538_b200.multi import fleet_mix, fleet_plan, max_over_ranks, rate


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    driver, devices = fleet_plan(world, world, rank)
    # the driving rank times the fleet's step; idle ranks report 0 ms
    local_ms = [250.0, 900.0] if driver else [0.0, 0.0]
    ms = max_over_ranks(local_ms, dist)
    mix = fleet_mix("3:1", 32, world) if driver else []
    out[rank] = (driver, devices, ms, [m.job_id for m in mix], rate(len(mix), ms[0]) if driver else None)
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_one_fleet_driver():
    world = 2
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
        res = dict(out)
    assert res[0][0] and not res[1][0]
    assert res[0][1] == [0, 1] and res[1][1] == []
    assert res[0][2] == res[1][2] == [250.0, 900.0]   # the driver's clock wins the max
    assert len(res[0][3]) == 64 and len(set(res[0][3])) == 64  # 32 jobs per GPU, one mix
    assert res[0][4] == 64 / 0.250


def test_fleet_plan_rules():
    assert fleet_plan(4, 1, 0) == (True, [0, 1, 2, 3])   # one process drives 4 GPUs
    assert fleet_plan(8, 8, 0) == (True, list(range(8)))
    assert fleet_plan(8, 8, 3) == (False, [])
    with pytest.raises(ValueError):
        fleet_plan(4, 2, 0)


def test_fleet_mix_is_the_reference_selection_at_32_per_gpu():
    from paper_2107_08538_b200.catalog import gen_mix

    assert [m.job_id for m in fleet_mix("3:1", 32, 4)] == [m.job_id for m in gen_mix("3:1", 128, seed=1)]
    assert [m.template for m in fleet_mix("3:1", 32, 2)] == [m.template for m in gen_mix("3:1", 64, seed=1)]


def test_single_process_is_identity():
    assert max_over_ranks([3.0, 4.0], None) == [3.0, 4.0]
