"""World-size-2 gloo tests of the multi-GPU host path (the bench's model-array
sharding and the per-model loss gather, C1) on CPU."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2102_02344_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, B_total, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard.model_range(rank, world, B_total)
    # each rank's "losses" are a deterministic function of the global model index
    local = torch.tensor([1000.0 + b for b in range(lo, hi)], dtype=torch.float32)
    allv = shard.gather_losses(local, B_total, world)
    # the double-buffered gatherer of the bench: two consecutive steps, each in global order
    g = shard.LossGather(B_total, world, "cpu")
    g1 = g.launch(local).clone()
    g2 = g.launch(local + 1.0).clone()
    assert np.array_equal(g1.numpy(), allv.numpy()) and np.array_equal(g2.numpy(), allv.numpy() + 1.0)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)                 # the bench's max-over-ranks timing
    q.put((rank, lo, hi, allv.numpy().tolist(), float(t.item())))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("B_total", [8, 7])
def test_shard_and_gather_gloo_world2(B_total):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, B_total, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ranges = [(o[1], o[2]) for o in outs]
    assert ranges[0][0] == 0 and ranges[-1][1] == B_total and ranges[0][1] == ranges[1][0]   # disjoint, covering
    for o in outs:
        assert np.array_equal(np.array(o[3]), 1000.0 + np.arange(B_total))                     # global model order
        assert o[4] == float(world)                                                               # max over ranks


def test_model_range_single():
    assert shard.model_range(0, 1, 5) == (0, 5)
    hp = {"lr": np.arange(6.0)}
    assert np.array_equal(shard.slice_hparams(hp, 2, 4)["lr"], [2.0, 3.0])
