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


def _ls_worker(rank, world, port, q):
    """The upper loop's distributed pieces (lower.gradient_descent): per-sample costs of
    this rank's shard gathered and summed in sample order for every Armijo trial
    (backtracking_linesearch, bilevel.py:326-358), theta updated redundantly."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    q.put((rank,) + _upper_step(rank, world))
    if world > 1:
        dist.destroy_process_group()


def _upper_step(rank, world):
    from paper_2412_08264_b200.lower import LinesearchParams, UpperState, backtracking_linesearch

    B, p, n = 7, 5, 11
    rng = np.random.default_rng(4)
    A = rng.standard_normal((B, n, p))
    xt = rng.standard_normal((B, n))
    mine = list(shard(B, world, rank))

    def evaluate(theta, warm):  # x_k(theta) = x_true_k + A_k theta: F = sum_k 1/2 |A_k theta|^2
        x = torch.from_numpy(np.stack([xt[k] + A[k] @ theta for k in mine]))
        per = 0.5 * ((x - torch.from_numpy(xt[mine])) ** 2).sum(dim=1)
        return float(allgather_sum(per.unsqueeze(1), B)[0]), x

    theta0 = rng.standard_normal(p)
    c0, x0 = evaluate(theta0, None)
    d = sum(A[k].T @ (A[k] @ theta0) for k in range(B))  # exact gradient of F
    state, trials = backtracking_linesearch(UpperState(theta0, x0, c0, 8.0), d, LinesearchParams(beta=8.0), evaluate)
    return state.theta, state.cost, trials


def test_gloo_upper_linesearch_is_bitwise_single_process():
    ref_theta, ref_cost, ref_trials = _upper_step(0, 1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ls_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for pr in procs:
        pr.join(timeout=60)
    assert ref_trials > 1  # the step had to backtrack
    for rank, theta, cost, trials in res:
        assert np.array_equal(theta, ref_theta) and cost == ref_cost and trials == ref_trials, rank
