"""Multi-rank runs of libgpuar itself (not the oracle) on the one GPU a test box has:
two processes, each its own Selector on cuda:0, joined by a gloo process group over CUDA
tensors (NCCL refuses two ranks on one GPU; the collectives are the same calls).  The
sharded outputs must be byte-identical to a one-rank run and to the oracle (R13:
a selection depends only on (seed, global index s, epoch, alpha)), C1 must deliver rank
0's vector, and the C2-reduced histogram must equal the sum.  Also bench.py --gpus 2
launching its own ranks."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SEED = synth.SELECT_SEED


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, kind, K_total, result_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1404_0027_b200 import Selector
        from paper_1404_0027_b200.dist import broadcast_vector, max_over_ranks, reduce_validation, shard
        import synth.gpu as sg
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        s0, n = shard(K_total, rank, world)
        if kind == "shared":
            M = 1029
            alpha = torch.zeros(M, dtype=torch.float32, device=dev)
            if rank == 0:
                alpha.copy_(torch.from_numpy(synth.yeast_like()))
            broadcast_vector(alpha)                                  # C1 over CUDA tensors
        else:
            M = synth.YEAST_M
            alpha = torch.empty((n, M), dtype=torch.float32, device=dev)
            sg.fill_rows(alpha, torch.from_numpy(synth.yeast_rates(M)).to(dev), synth.GEN_SEED, s0)
        sel = Selector(M, max(n, 1), SEED, device=0)
        sel.set_selection_offset(s0)
        sel.epoch = 5
        sel.set_propensities(alpha)
        idx, tau, trials = sel.select(n)
        hist, totals = sel.histogram(idx, trials)
        sel.sync()
        np.save(os.path.join(result_dir, f"hist{rank}.npy"), hist.cpu().numpy())
        reduce_validation(hist, totals, dst=0)                      # C2
        t = max_over_ranks(float(rank + 1), dev)                    # C3
        for name, v in (("idx", idx), ("tau", tau), ("trials", trials)):
            np.save(os.path.join(result_dir, f"{name}{rank}.npy"), v.cpu().numpy())
        if rank == 0:
            np.save(os.path.join(result_dir, "alpha0.npy"), alpha.cpu().numpy() if kind == "shared" else np.zeros(1))
            np.save(os.path.join(result_dir, "hist.npy"), hist.cpu().numpy())
            np.save(os.path.join(result_dir, "totals.npy"), totals.cpu().numpy())
            np.save(os.path.join(result_dir, "tmax.npy"), np.array([t]))
        sel.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,K_total", [("shared", 65_537), ("rows", 4_099)])
def test_two_ranks_libgpuar_equals_one_rank_and_oracle(kind, K_total, tmp_path):
    from paper_1404_0027_b200 import Selector
    import synth.gpu as sg
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), kind, K_total, str(tmp_path)), nprocs=world, join=True)
    cat = {k: np.concatenate([np.load(tmp_path / f"{k}{r}.npy") for r in range(world)]) for k in ("idx", "tau", "trials")}
    # the same selections from one rank, one call
    if kind == "shared":
        a = synth.yeast_like()
        np.testing.assert_array_equal(np.load(tmp_path / "alpha0.npy"), a)   # C1 delivered rank 0's vector
        dev_alpha = torch.from_numpy(a).cuda()
        host = a
    else:
        M = synth.YEAST_M
        dev_alpha = torch.empty((K_total, M), dtype=torch.float32, device="cuda")
        sg.fill_rows(dev_alpha, torch.from_numpy(synth.yeast_rates(M)).cuda(), synth.GEN_SEED, 0)
        host = dev_alpha.cpu().numpy()
    M = host.shape[-1]
    sel = Selector(M, K_total, SEED)
    sel.epoch = 5
    sel.set_propensities(dev_alpha)
    one = [t.cpu().numpy() for t in sel.select(K_total)]
    sel.sync()
    assert cat["idx"].tobytes() == one[0].tobytes()
    assert cat["tau"].tobytes() == one[1].tobytes()
    assert cat["trials"].tobytes() == one[2].tobytes()
    ref = oracle.ar_select(host, K_total, seed=SEED, epoch=5, nthreads=8)
    np.testing.assert_array_equal(cat["idx"], ref["idx"])
    np.testing.assert_array_equal(cat["trials"].view(np.uint32), ref["trials"])
    rel = np.abs(cat["tau"].astype(np.float64) - ref["tau_ref"]) / ref["tau_ref"]
    assert rel.max() <= 1e-6
    # C2: the reduced histogram is the sum of the ranks' histograms and the whole run's
    hist = np.load(tmp_path / "hist.npy")
    np.testing.assert_array_equal(hist, np.load(tmp_path / "hist0.npy") + np.load(tmp_path / "hist1.npy"))
    np.testing.assert_array_equal(hist, np.bincount(np.where(ref["idx"] < 0, M, ref["idx"]), minlength=M + 1))
    totals = np.load(tmp_path / "totals.npy")
    assert totals[0] == int(ref["trials"].sum()) and totals[1] == int((ref["idx"] < 0).sum())
    assert float(np.load(tmp_path / "tmax.npy")[0]) == 2.0


def _bench(*args, timeout=900):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    return out


@pytest.mark.parametrize("config,extra", [("c2", []), ("c4", ["--K", "131072"])])
def test_bench_gpus2_launches_its_own_ranks(config, extra):
    """bench.py --gpus 2 with no launcher in the environment runs two ranks (here sharing the
    box's one GPU over gloo, which the line must say) and reports n_gpus = 2, the C1/C2 times
    and the strong-scaling split."""
    out = _bench("--gpus", "2", "--oversubscribe", "--config", config, *extra, "--steps", "3", "--warmup", "3",
                 "--no-e2e", "--no-cpu", "--sustain-s", "0")
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["oversubscribed"]["gpus_visible"] >= 1
    assert d["config"]["K_total"] == 2 * d["config"]["K_per_gpu"]
    assert d["collectives"]["c2_reduce_ms"] > 0 and d["collectives"]["backend"] == "gloo"
    if config == "c2":
        assert d["collectives"]["c1_broadcast_ms"] > 0 and d["collectives"]["c1_bytes"] == 4 * 1029
    assert d["strong_scaling"]["K_total"] > 0 and d["strong_scaling"]["value"] > 0
    assert d["validation"]["rejected_last_step"] == 0
    assert d["validation"]["chi2_vs_exact_law"]["p"] > 1e-4
    assert abs(d["validation"]["acceptance"]["z_trials_sum"]) < 6


def test_bench_gpus_n_refuses_missing_gpus():
    n = torch.cuda.device_count()
    out = _bench("--gpus", str(n + 1), "--config", "c1", "--steps", "1", "--warmup", "3", timeout=300)
    assert out.returncode != 0 and "visible GPUs" in out.stderr
    assert not any(l.startswith("{") for l in out.stdout.splitlines())
