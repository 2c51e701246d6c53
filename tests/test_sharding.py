"""Multi-rank host logic (gloo, world size 2, CPU): the product's shard plan
(sharding.ShardedRun) and its final gather reproduce the single-process result
bitwise.  The per-rank compute here is the oracle (CPU stand-in for the GPU
engine, used only as the checker)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2112_15445_b200.sharding import shard_range, shard_sizes


def test_shard_ranges_partition():
    for n in (0, 1, 7, 32, 100, 256, 1024, 1000):
        for world in (1, 2, 3, 4, 8):
            for align in (1, 32):
                rs = [shard_range(n, r, world, align) for r in range(world)]
                assert rs[0][0] == 0 and rs[-1][1] == n
                assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
                if align == 32:
                    assert all(a % 32 == 0 or a == n for a, _ in rs)
    assert shard_sizes(256, 8, 32) == [32] * 8
    assert shard_sizes(1024, 8) == [128] * 8
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2112_15445_b200.sharding import ShardedRun
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = oracle.bench_rng("shard-cfg1", 0.9)
    g = (64, 32, 3, 3, 8, 8, (1, 1), (1, 1))
    w = oracle.synthesize_masked_weights((32, 64, 3, 3), 0.9, rng)
    x = rng.standard_normal((n, 64, 8, 8)).astype(np.float32)
    csr = oracle.build_csr(w, g)
    # the product's shard plan + final gather; the per-rank compute is the oracle (CPU)
    job = ShardedRun.from_env(n)
    assert (job.rank, job.world) == (rank, world)
    full = job.run(torch.from_numpy(x),
                   lambda xl: torch.from_numpy(oracle.sparse_conv_forward(xl.numpy(), csr, g))).numpy()
    if rank == 0:
        ref = oracle.sparse_conv_forward(x, csr, g)
        q.put(bool(np.array_equal(full, ref)) and job.local_batch == (n + 1) // 2)
    dist.barrier()
    dist.destroy_process_group()


def _weak_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2112_15445_b200.sharding import ShardedRun
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    job = ShardedRun.weak(4, rank, world)
    local = torch.full((4, 3), float(rank))
    full = job.gather(local)
    if rank == 0:
        q.put(full[:, 0].tolist() == [0.0] * 4 + [1.0] * 4 and job.global_batch == 8)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_weak_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_weak_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True


@pytest.mark.parametrize("n", [8, 13])
def test_gloo_world2_gather_matches_single_process(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True
