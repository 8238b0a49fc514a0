"""Multi-rank host logic on CPU (gloo, world_size 2/4): the quadrature points are sharded with
the library's own partition (sssvd_shard_range, host mirror of the GPU path) and each rank's
partial moment blocks S_k^(r) = sum_{j in shard r} 2 Re(w_j t_j^k X_j) are summed with one
all-reduce - the exchange the GPU path performs with ncclAllReduce. The sum must reproduce the
single-process ascending-j accumulation (moments.hpp:132-147) to rounding, and the refinement
pass (ell = 2) must do the same with one all-reduce per pass."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import sssvd_oracle as orc


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def problem():
    a = orc.random_matrix(60, 24, 5)
    g = orc.form_gram(orc.ProblemMatrix(a))
    rule = orc.ContourRule(6.0, 9.0, 32, 0.1, orc.SpectralTransform(orc.IDENTITY))  # holds part of the spectrum
    s0 = orc.random_start(24, 4, 42)
    return g, rule, s0


def worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2109_13655_b200 import sssvd
    g, rule, s0 = problem()
    h = rule.count // 2
    jb, je = sssvd.shard_range(h, world, rank)
    acc = orc.MomentAccumulator(g, rule)
    # refinement pass (ell = 2): partial S0 over the shard, one all-reduce
    part = np.zeros(s0.shape)
    sols = acc.solve_all(s0, range(jb, je))
    for idx, j in enumerate(range(jb, je)):
        part += 2.0 * (rule.weights[j] * sols[idx]).real
    t = torch.from_numpy(part)
    dist.all_reduce(t)
    s1 = t.numpy()
    # moment pass over the shard, one all-reduce of all M+1 blocks
    blocks = acc.accumulate(s1, 3, shifts=range(jb, je)).blocks
    t = torch.from_numpy(np.stack(blocks))
    dist.all_reduce(t)
    if rank == 0:
        q.put((jb, je, t.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_moments_allreduce(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    jb, je, got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    g, rule, s0 = problem()
    acc = orc.MomentAccumulator(g, rule)
    ref = acc.accumulate(acc.refine(s0), 3).blocks
    for k in range(4):
        assert np.linalg.norm(got[k] - ref[k]) <= 1e-13 * np.linalg.norm(ref[k])
    assert jb == 0 and je == 16 // world
