"""Multi-process (gloo, world_size 2) tests of the sample-sharded hypergradient
reduction: each rank owns a contiguous block of samples, the
per-sample hypergradients (here the CPU oracle's, since no GPU is present) are
all-gathered and summed in global sample order -- bitwise equal to the
single-process sum and identical on every rank."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2412_08264_b200.distributed import allgather_sum, allreduce_cost, ordered_sum, shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _per_sample_hypergradients(batch):
    from oracle import cpu_bilevel as ob
    from oracle import cpu_imaging as im

    cfg = im.DeblurConfig(12, batch, 3, 1.0, 0.01, "filters", 2, 3, eps=0.3, alpha0=-1.0)
    th = im.deblur_theta0(cfg)
    out = []
    for k in range(batch):
        model, xt = im.deblur_sample(cfg, k)
        xh = xt + 0.01 * np.random.default_rng(k).standard_normal(xt.size)
        from oracle import cpu_krylov as ok

        d, _ = ob.hypergradient(model, th, xh, xt, opts=ok.Options(stop_rule=ok.ResidualRule(1e-10), max_iter=800))
        out.append(d)
    return np.stack(out)


def _worker(rank, world, port, hg, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    B = hg.shape[0]
    mine = torch.from_numpy(hg[list(shard(B, world, rank))])
    total = allgather_sum(mine, B)
    cost = allreduce_cost(float(rank + 1), torch.device("cpu"))
    q.put((rank, total.numpy(), cost))
    dist.destroy_process_group()


def test_shard_partitions_samples():
    for B in (1, 5, 8, 64):
        for W in (1, 2, 3, 8):
            got = [list(shard(B, W, r)) for r in range(W)]
            assert sum(got, []) == list(range(B))
            assert max(map(len, got)) - min(map(len, got)) <= 1


@pytest.mark.parametrize("world", [2])
def test_gloo_allgather_sum_is_bitwise_single_process(world):
    hg = _per_sample_hypergradients(5)
    ref = ordered_sum(torch.from_numpy(hg)).numpy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, hg, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, total, cost in res:
        assert np.array_equal(total, ref), rank
        assert cost == sum(range(1, world + 1))
