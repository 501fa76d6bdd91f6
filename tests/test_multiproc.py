"""World-size-2 CPU tests (gloo) of the N>1 host path: env partitioning and the
marker-field all-gather.  The per-env compute is the oracle (no GPU here); the
check is that 2 ranks x their env ranges + gather reproduce a single-process run
of all envs byte for byte (determinism contract S:672)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_28475_b200.dist import MarkerGather, env_range


def test_env_range_partitions():
    for n in (0, 1, 7, 8, 1024, 8192, 1001):
        for ws in (1, 2, 3, 4, 8):
            ids = []
            for r in range(ws):
                a, b = env_range(r, ws, n)
                assert 0 <= a <= b <= n
                ids += list(range(a, b))
            assert ids == list(range(n))
            sizes = [env_range(r, ws, n)[1] - env_range(r, ws, n)[0] for r in range(ws)]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_total, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as O
    import workloads as w
    s = w.scene_small_peg(n_envs=n_total, n_steps=2)
    s.params.fixed_iters = 20
    a, b = env_range(rank, world, n_total)
    o = O.Oracle(s, init_poses=s.init_poses[a:b])
    for k in range(2):
        o.step(s.poses[k][a:b])
    g = MarkerGather(b - a, 63, 2, rank, world, "cpu")
    for e in range(b - a):
        g.slot[e] = torch.from_numpy(o.markers(e).astype(np.float32))
    buf = g.gather()
    if rank == 0:
        np.save(out_path, buf.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gather_matches_single_process(tmp_path):
    import oracle as O
    import workloads as w
    n_total = 4
    out = str(tmp_path / "gathered.npy")
    mp.start_processes(_worker, args=(2, _free_port(), n_total, out), nprocs=2, join=True, start_method="spawn")
    got = np.load(out)
    s = w.scene_small_peg(n_envs=n_total, n_steps=2)
    s.params.fixed_iters = 20
    o = O.Oracle(s)
    for k in range(2):
        o.step(s.poses[k])
    ref = np.stack([o.markers(e).astype(np.float32) for e in range(n_total)])
    assert got.shape == ref.shape
    assert np.array_equal(got, ref)
    assert np.abs(ref).max() > 0
