"""World-size-2 gloo test of the replica plumbing used by bench.py on N GPUs."""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, size, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(size))
    from paper_1707_07598_b200 import dist
    r, s = dist.init("gloo")
    dist.barrier()
    m = dist.max_over_ranks(1.5 + r)          # rank-dependent "step time"
    seed = dist.replica_seed(7, r)
    q.put((r, s, m, seed, dist.aggregate_seconds_per_iter(m, s)))
    import torch.distributed as td
    td.destroy_process_group()


def test_replicas_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert [o[0] for o in out] == [0, 1]
    assert all(o[1] == 2 for o in out)
    assert all(o[2] == 2.5 for o in out)              # max over ranks
    assert out[0][3] != out[1][3]                     # independent replica models
    assert all(o[4] == 1.25 for o in out)             # whole-job s/iter


def test_single_process_defaults():
    from paper_1707_07598_b200 import dist
    assert dist.max_over_ranks(3.0) == 3.0
    assert dist.aggregate_seconds_per_iter(2.0, 1) == 2.0
