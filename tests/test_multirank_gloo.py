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


def gram_worker(rank, world, port, q):
    """form_gram sharded as on the GPU: this rank forms only the 64 x 64 lower-triangle tiles the
    library assigns it (sssvd_gram_tiles, the kernel's own decode), zeros elsewhere; one all-reduce
    (sum) assembles G, which must be bitwise A^T A with each tile written by exactly one rank."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2109_13655_b200 import sssvd
    a = orc.random_matrix(300, 333, 9)
    n = a.shape[1]
    g = np.zeros((n, n))
    owner = np.zeros((n, n), dtype=np.int64)
    for ti, tj in sssvd.gram_tiles(n, world, rank):
        ri, rj = slice(64 * ti, min(n, 64 * ti + 64)), slice(64 * tj, min(n, 64 * tj + 64))
        g[ri, rj] = a[:, ri].T @ a[:, rj]
        owner[ri, rj] += 1
    t, o = torch.from_numpy(g), torch.from_numpy(owner)
    dist.all_reduce(t)
    dist.all_reduce(o)
    if rank == 0:
        q.put((t.numpy(), o.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_gram_tiles_allreduce(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=gram_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    g, owner = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    a = orc.random_matrix(300, 333, 9)
    tile_lower = np.add.outer(np.arange(333) // 64, -(np.arange(333) // 64)) >= 0
    assert np.all(owner[tile_lower] == 1) and np.all(owner[~tile_lower] == 0)
    full = a.T @ a
    assert np.allclose(g[tile_lower], full[tile_lower], rtol=0, atol=1e-12)
    assert np.all(g[~tile_lower] == 0.0)


def test_bench_gpus_flag_spawns_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself with 2 ranks (torch.distributed.run);
    the reference arm runs on rank 0 only and reports the world size (CPU-only: config 1)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--gpus", "2",
                          "--config", "1", "--steps", "1", "--warmup", "3"], capture_output=True, text=True,
                         timeout=600, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout
    assert lines[0]["n_gpus"] == 2 and lines[0]["impl"] == "reference"
    assert "rank 1" not in out.stdout


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
