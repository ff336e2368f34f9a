"""N>1 host logic of the bench on CPU: two gloo ranks, each with its own
seeded mix (disjoint inputs), combine device-timed step times by max."""

import os
import socket

import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2107_08538_b200.multi import max_over_ranks, rank_mix, whole_job_rate


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mix = rank_mix("3:1", 32, rank)
    local_ms = [100.0 + 50.0 * rank, 900.0 - 10.0 * rank]  # (device step, e2e step) of this rank
    ms = max_over_ranks(local_ms, dist)
    out[rank] = (ms, [m.job.seed for m in mix], whole_job_rate(len(mix), world, ms[0]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_take_the_max_and_run_disjoint_mixes():
    world = 2
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
        res = dict(out)
    assert res[0][0] == res[1][0] == [150.0, 900.0]
    assert not set(res[0][1]) & set(res[1][1])  # different seeds -> different inputs
    assert res[0][2] == res[1][2] == 64 / 0.150


def test_single_process_is_identity():
    assert max_over_ranks([3.0, 4.0], None) == [3.0, 4.0]
