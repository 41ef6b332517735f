"""Host-side multi-rank logic on CPU (gloo, world_size 2): sharding tiles the selections
exactly, the shared vector broadcast (C1), the histogram reduce (C2) and max-over-ranks
(C3) compose to the single-process result.  The per-rank selections are computed with the
oracle (this is a test of the host logic; the GPU path is covered by -m gpu)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1404_0027_b200.dist import broadcast_vector, max_over_ranks, reduce_validation, shard, weak_shard


def test_shard_tiles_range():
    for K in (0, 1, 7, 10_000, 2**20 + 3):
        for world in (1, 2, 3, 8):
            spans = [shard(K, r, world) for r in range(world)]
            pos = 0
            for s0, n in spans:
                assert s0 == pos
                pos += n
            assert pos == K
            assert max(n for _, n in spans) - min(n for _, n in spans) <= 1
    assert weak_shard(1 << 20, 3) == (3 << 20, 1 << 20)
    with pytest.raises(ValueError):
        shard(10, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, K, result_dir):
    import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        M = 37
        alpha = torch.zeros(M, dtype=torch.float32)
        if rank == 0:
            alpha = torch.from_numpy(np.random.default_rng(5).exponential(size=M).astype(np.float32))
        broadcast_vector(alpha)
        s0, n = shard(K, rank, world)
        r = oracle.ar_select(alpha.numpy(), n, seed=99, s0=s0, epoch=2)
        hist = torch.from_numpy(np.bincount(np.where(r["idx"] < 0, M, r["idx"]), minlength=M + 1).astype(np.int64))
        totals = torch.tensor([int(r["trials"].sum()), int((r["idx"] < 0).sum())], dtype=torch.int64)
        reduce_validation(hist, totals)
        t = max_over_ranks(float(rank + 1))
        np.save(os.path.join(result_dir, f"idx{rank}.npy"), r["idx"])
        np.save(os.path.join(result_dir, f"trials{rank}.npy"), r["trials"])
        if rank == 0:
            np.save(os.path.join(result_dir, "hist.npy"), hist.numpy())
            np.save(os.path.join(result_dir, "totals.npy"), totals.numpy())
            np.save(os.path.join(result_dir, "alpha.npy"), alpha.numpy())
            np.save(os.path.join(result_dir, "tmax.npy"), np.array([t]))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharded_equals_whole(tmp_path):
    import oracle
    world, K = 2, 1001
    mp.spawn(_worker, args=(world, _free_port(), K, str(tmp_path)), nprocs=world, join=True)
    alpha = np.load(tmp_path / "alpha.npy")
    whole = oracle.ar_select(alpha, K, seed=99, epoch=2)
    idx = np.concatenate([np.load(tmp_path / f"idx{r}.npy") for r in range(world)])
    trials = np.concatenate([np.load(tmp_path / f"trials{r}.npy") for r in range(world)])
    np.testing.assert_array_equal(idx, whole["idx"])
    np.testing.assert_array_equal(trials, whole["trials"])
    M = alpha.size
    hist = np.load(tmp_path / "hist.npy")
    np.testing.assert_array_equal(hist, np.bincount(whole["idx"], minlength=M + 1))
    totals = np.load(tmp_path / "totals.npy")
    assert totals[0] == whole["trials"].sum() and totals[1] == 0
    assert float(np.load(tmp_path / "tmax.npy")[0]) == 2.0
