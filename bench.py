#!/usr/bin/env python
"""bench.py -- GPU-AR next-reaction selections/sec on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl gpuar|reference]
                    [--scaling weak|strong]

One JSON line on rank 0.  Default workload (config c4, the per-realization K x M matrix
named by BASELINE.json for 1/2/4/8 B200): M = 1029 yeast-like reactions, K = 2^20
realizations PER GPU (weak scaling: each rank owns global rows [r*K, (r+1)*K), generated in
its own HBM by libsynth -- no data-path collective); --scaling strong splits K = 2^20 in
total over the ranks, and an N > 1 weak run also reports that strong
split as a sub-record.  A step is one gpuar_select over the K resident rows: per-row
alpha_max / alpha_0 reductions, AR trials, tau (one kernel).  The 4.3 GB matrix is > L2
(126 MB), so no L2 flush is needed between steps.

--gpus N without a torch.distributed launcher (no WORLD_SIZE in the environment) re-runs
this script under `python -m torch.distributed.run --nproc-per-node N` itself, one rank per
GPU; fewer than N visible GPUs is an error (--oversubscribe allows ranks to share GPUs over
gloo, for dry runs and tests only, and says so in the JSON line).

--impl reference times the CPU oracle (oracle/, the parity reference) on rank 0 on a
bounded sample of the same workload per step; the other ranks exit 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "next-reaction selections/sec at 1/2/4/8 B200; % of ALU/HBM roofline"
UNIT = "selections/s"
SSA_UNIT = "SSA events/s (one selection each)"


def unit_of(w: dict) -> str:
    """The metric's unit for a workload: SSA events for s1, selections otherwise."""
    return SSA_UNIT if w["kind"] == "ssa" else UNIT
# ALU roofline: the fma pipe takes one warp instruction per 2 cycles per SMSP
# (B300_MICROARCH.md "Pipe rates", rt_SMSP = 2) = 64 lane-slots/clk/SM; a Philox4x32-10 call
# is 20 mul.wide.u32 = 20 IMAD.WIDE.U32 (SASS), each writing a register pair = 2 slots.
FMA_SLOTS_PER_CLK_PER_SM = 64
FMA_SLOTS_PER_PHILOX = 40
SM_COUNT = 148

CONFIGS = {
    "c1": dict(kind="shared", dist="hand", M=4, K=10_000,
               desc="c1: M=4 hand-set {1,2,3,4}, K=10^4 selections, shared vector"),
    "c2": dict(kind="shared", dist="yeast", M=1029, K=65_536,
               desc="c2: M=1029 yeast-like shared vector in smem, K=65536 selections"),
    "c3": dict(kind="shared", dist="pareto", M=10_000, K=1 << 20,
               desc="c3: shared simulated distribution, K=2^20 selections"),
    "c4": dict(kind="rows", dist="yeast", M=1029, K=1 << 20,
               desc="c4: per-realization KxM matrix, M=1029 yeast-like rows, K=2^20 realizations per GPU"),
    # max_trials 2^24: this seed's Pareto vector has p = 1.03e-5 (E[trials] ~ 9.7e4), so the
    # default cap 2^20 would reject (1-p)^(2^20) ~ 2e-5 of the selections -- ~340 of 2^24 at
    # 8 GPUs; at 2^24 P(reject) = e^-173 per selection and the run shows the paper's zero
    # rejection
    "c5": dict(kind="shared", dist="pareto", M=1_000_000, K=1 << 21, max_trials=1 << 24,
               desc="c5: M=1e6 Pareto(1.5) shared vector, K=2^21 selections per GPU (2^24 at 8 GPUs)"),
    # NEXT-2: the full SSA loop (propensities + selection + state update) on chip
    "s1": dict(kind="ssa", dist="yeast-network", M=1029, N=641, K=1 << 17, inner=16,
               desc="s1: full SSA steps, yeast-like mass-action network (641 species, 1029 reactions), "
                    "K=2^17 realizations per GPU, 16 steps per launch"),
    # NEXT-1: the paper's printed election + argmin rule on its own Table 1 / Fig. 2 workload
    "p1": dict(kind="shared", dist="gaussian", M=1024, K=62_500, rule="argmin",
               desc="p1: paper's argmin rule, discrete Gaussian M=1024, K=62500 parallel realizations"),
}

# The paper's own GPU timing for its argmin rule: 10^7 selections at
# M=1024, K=62500 (timed unit assumed) in 1326.78 ms on a Tesla K20.
PAPER_K20_SEL_PER_S = 1e7 / 1.32678


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="gpuar", choices=["gpuar", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--dist", default=None, help="c3: uniform|exponential|pareto")
    ap.add_argument("--M", type=int, default=None)
    ap.add_argument("--K", type=int, default=None, help="selections per GPU")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--max-trials", type=int, default=None, help="per-selection trial cap (default 2^20)")
    ap.add_argument("--rule", default=None, choices=["classic", "argmin", "it", "it_scan"])
    ap.add_argument("--w", type=float, default=1.0, help="argmin rule threshold multiplier T = w alpha_max")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-it", action="store_true", help="skip the inverse-transform comparison (matrix configs)")
    ap.add_argument("--no-stream-ceiling", action="store_true",
                    help="skip the row-stats stream diagnostics (matrix configs; ncu launch lists)")
    ap.add_argument("--epochs", type=int, default=0,
                    help="epochs per gpuar_select_epochs launch for the multi_epoch record (0: auto, 1: skip)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", help="nccl (default); gloo only to dry-run N ranks on one GPU")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: K selections per GPU (default); strong: K selections in total, split over the ranks")
    ap.add_argument("--oversubscribe", action="store_true",
                    help="allow more ranks than visible GPUs (ranks share GPUs over gloo; dry runs and tests only)")
    ap.add_argument("--sustain-s", type=float, default=2.0,
                    help="seconds of the sustained-loop sub-record (0: skip)")
    return ap.parse_args()


def workload(args) -> dict:
    w = dict(CONFIGS[args.config])
    if args.dist:
        w["dist"] = args.dist
    if args.M:
        w["M"] = args.M
    if args.K:
        w["K"] = args.K
    if args.rule:
        w["rule"] = args.rule
    w.setdefault("rule", "classic")
    w["w"] = args.w
    if args.max_trials:
        w["max_trials"] = args.max_trials
    w.setdefault("max_trials", 1 << 20)
    return w


# ----------------------------------------------------------------- clocks during the timed region

class ClockSampler:
    FIELDS = ["index", "clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu_index: int):
        # nvidia-smi -i takes the physical index / UUID: map through CUDA_VISIBLE_DEVICES
        vis = [v.strip() for v in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if v.strip()]
        self.gpu = vis[gpu_index] if gpu_index < len(vis) else str(gpu_index)
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={','.join(self.FIELDS)}", "--format=csv,noheader,nounits",
                 "-i", str(self.gpu), "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.rows.append((time.perf_counter(), parts))

    def wait_first(self, timeout: float = 5.0) -> None:
        t0 = time.perf_counter()
        while self.proc and not self.rows and time.perf_counter() - t0 < timeout:
            time.sleep(0.01)

    def mark(self, start: float, end: float) -> None:
        """Keep the samples taken inside [start, end] (plus the nearest one on each side)."""
        inside = [r for r in self.rows if start <= r[0] <= end]
        before = [r for r in self.rows if r[0] < start][-1:]
        after = [r for r in self.rows if r[0] > end][:1]
        self.window = before + inside + after

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        rows = [r[1] for r in getattr(self, "window", [])]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        reasons = sorted({n for r in rows for n, v in zip(self.NAMES, r[3:]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------------- helpers

def measured_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        d["_source"] = "measured"
        return d
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "_source": "fallback"}


def ncu_traffic(config: str):
    """dram bytes per launch of the dominant kernel from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    e = d.get(config)
    return None if e is None else e.get("dram_bytes_per_launch")


def make_inputs(w: dict, s0: int, K: int, device):
    """Synthetic, seeded inputs (synth/) already resident in HBM: the shared vector, or the
    matrix rows of global selections s0 .. s0+K-1 (each rank generates its own rows)."""
    import numpy as np
    import torch

    import synth
    M = w["M"]
    if w["kind"] == "ssa":
        net = synth.yeast_like_network(M=M)
        dev = {k: torch.from_numpy(np.ascontiguousarray(net[k])).to(device) for k in ("reac", "rate", "didx", "dval")}
        X = torch.from_numpy(synth.initial_state(net["N"], K)).to(device)
        t = torch.zeros(K, dtype=torch.float64, device=device)
        return dict(net=dev, N=net["N"], X=X, t=t)
    if w["kind"] == "rows":
        import synth.gpu as sg
        rates = torch.from_numpy(synth.yeast_rates(M)).to(device)
        mat = torch.empty((K, M), dtype=torch.float32, device=device)
        sg.fill_rows(mat, rates, synth.GEN_SEED, s0)
        return mat
    if w["dist"] == "hand":
        a = synth.hand([1, 2, 3, 4])
    else:
        a = synth.distribution(w["dist"], M)
    return torch.from_numpy(np.ascontiguousarray(a)).to(device)


def host_sample(w: dict, rank: int, n: int):
    import numpy as np

    import synth
    if w["kind"] == "ssa":
        net = synth.yeast_like_network(M=w["M"])
        return net, synth.initial_state(net["N"], n)
    if w["kind"] == "rows":
        return synth.rows(synth.yeast_rates(w["M"]), synth.GEN_SEED, rank * w["K"], n)
    if w["dist"] == "hand":
        return synth.hand([1, 2, 3, 4])
    return np.ascontiguousarray(synth.distribution(w["dist"], w["M"]))


def oracle_pass(w: dict, data, nn: int, epoch: int, threads: int):
    """One timed oracle pass over the first nn selections of a host sample -> (seconds, units)."""
    import numpy as np

    import oracle
    t0 = time.perf_counter()
    if w["kind"] == "ssa":
        net, X0 = data
        r = oracle.ssa_run(net, X0[:nn], np.zeros(nn), w["inner"], seed=20140327, epoch0=epoch, nthreads=threads)
        return time.perf_counter() - t0, int(r["steps"].sum())
    alpha = data[:nn] if w["kind"] == "rows" else data
    if w.get("rule") == "argmin":
        oracle.argmin_select(alpha, nn, seed=20140327, w=w["w"], epoch=epoch, nthreads=threads)
    elif w.get("rule") in ("it", "it_scan"):
        oracle.it_select(alpha, nn, seed=20140327, epoch=epoch, nthreads=threads)
    else:
        oracle.ar_select(alpha, nn, seed=20140327, epoch=epoch, max_trials=w["max_trials"], nthreads=threads)
    return time.perf_counter() - t0, nn


def oracle_rate(w: dict, seconds: float, threads: int, max_rows: int | None = None):
    """Oracle selections/s on a bounded sample of the workload (rank 0's first selections):
    the sample is at most max_rows selections; it is re-run on successive epochs until about
    `seconds` of work have been timed.  Returns (rate, sample size, seconds timed)."""
    import numpy as np

    import oracle

    K = w["K"]
    n = min(K, max_rows or K)
    data = host_sample(w, 0, n)

    def run(nn, epoch):
        return oracle_pass(w, data, nn, epoch, threads)

    # probe with a growing prefix, then time whole passes over the sample
    probe = 256
    while True:
        nn = min(probe, n)
        dt, _ = run(nn, 0)
        if dt > 0.25 or nn == n:
            break
        probe *= 4
    if nn < n:
        nn = max(1, min(n, int(nn * seconds / max(dt, 1e-9))))
    total_t, total_u, epoch = 0.0, 0, 1
    while total_t < seconds or total_u == 0:
        dt, units = run(nn, epoch)
        total_t += dt
        total_u += units
        epoch += 1
    return total_u / total_t, nn, total_t


# ----------------------------------------------------------------- the workload's config record

def bench_config(w: dict, args, world: int) -> dict:
    """The `config` object of the JSON line -- identical for our arm and the reference arm
    (the driver compares them): the workload and its sizes only."""
    from paper_1404_0027_b200.dist import shard
    M = w["M"]
    if w["kind"] == "ssa":
        return {"workload": w["desc"], "M": M, "N": w["N"], "K_per_gpu": w["K"], "steps_per_launch": w["inner"]}
    if args.scaling == "strong":
        K_total = w["K"]
        K = shard(K_total, 0, world)[1]          # rank 0's shard, the largest
        desc = w["desc"].replace("per GPU", "in total")
    else:
        K, K_total, desc = w["K"], w["K"] * world, w["desc"]
    return {"workload": desc, "M": M, "K_per_gpu": K, "K_total": K_total, "dist": w["dist"], "rule": w["rule"],
            "max_trials": w["max_trials"],
            "parallelism": f"selections sharded over {world} GPU(s) ({args.scaling} scaling), no data-path collective",
            "l2": ("inputs larger than L2 (%.2f GB/GPU), no flush" % (K * M * 4 / 1e9)) if w["kind"] == "rows"
            else "shared vector resident in smem/L2 by design; outputs 12 B/selection"}


# ----------------------------------------------------------------- the reference (oracle) arm

def run_reference(args, w, rank, world):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    # each step: a bounded sample sized so the whole run takes ~2 minutes
    budget = 120.0 / max(1, args.steps + args.warmup)
    # host memory bound: at most 2^17 matrix rows (540 MB) per sample
    rate, n, _ = oracle_rate(w, min(budget, 2.0), threads, max_rows=(1 << 17) if w["kind"] == "rows" else None)
    n = max(1, min(n, int(rate * budget)))   # one step's sample: ~budget seconds of oracle work
    data = host_sample(w, 0, n)
    warm = max(args.warmup, 3)
    for e in range(warm):
        oracle_pass(w, data, n, e, threads)
    dt, units = 0.0, 0
    for e in range(args.steps):
        t, u = oracle_pass(w, data, n, warm + e, threads)
        dt += t
        units += u
    value = units / dt
    sample = f"{n} of the {w['K']} selections per step ({'rows' if w['kind'] == 'rows' else 'selections'} 0..{n - 1})"
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": unit_of(w), "n_gpus": args.gpus,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": args.scaling if w["kind"] != "ssa" else "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic", "config": bench_config(w, args, world),
        "cpu_baseline": {"value": value, "unit": unit_of(w), "cores": threads, "kind": "oracle", "sample": sample,
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": unit_of(w), "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


# ----------------------------------------------------------------- validation (statistics, off the clock)

def chi2_pooled(counts, expected, min_expected: float = 5.0) -> dict:
    """Pearson chi^2 of observed counts against expected counts, the bins with an expected
    count < min_expected pooled into one (SURVEY.md §8(c) "law").  Statistics of the
    outputs only (scipy), not the selection method."""
    import numpy as np
    from scipy.stats import chi2

    o = np.asarray(counts, np.float64)
    e = np.asarray(expected, np.float64)
    keep = e >= min_expected
    oo, ee = list(o[keep]), list(e[keep])
    if (~keep).any():
        oo.append(o[~keep].sum())
        ee.append(e[~keep].sum())
    oo, ee = np.array(oo), np.array(ee)
    if ((ee == 0) & (oo > 0)).any():
        return {"stat": float("inf"), "dof": int(oo.size - 1), "p": 0.0, "bins": int(oo.size)}
    nz = ee > 0
    stat = float((((oo - ee) ** 2)[nz] / ee[nz]).sum())
    dof = int(nz.sum() - 1)
    return {"stat": stat, "dof": dof, "p": float(chi2.sf(stat, dof)) if dof > 0 else 1.0, "bins": int(nz.sum())}


def law_and_trials(w: dict, sel, alpha):
    """(sum over this rank's selections of the exact law alpha_j / alpha_0 as an M-vector,
    expected sum of trials, its variance) -- float64 CUDA tensors.  Shared vector: one law
    for every selection; matrix: the row laws summed (chunked, the matrix is 4.3 GB), and
    E[trials] = 1/p_r, Var = (1 - p_r)/p_r^2 with p_r = alpha_0,r / (M alpha_max,r) from
    gpuar_row_stats."""
    import numpy as np
    import torch

    M = w["M"]
    if alpha.dim() == 1:
        # The exact law of the discrete draws (R3/R5): candidate j has
        # n_j = #{x < 2^32 : (x M) >> 32 = j} of the 2^32 index words and is accepted for
        # T_j = #{v < 2^24 : fl32(v 2^-24 alpha_max) < alpha_j} of the 2^24 uniforms, so a
        # trial accepts j with probability n_j T_j / 2^56.  (alpha_j / alpha_0 and
        # a0 / (M alpha_max) are its continuum limits; on the heavy-tailed c5 vector the
        # 2^-24 quantisation of u moves p by +0.3 %, 5.7 sigma over 2^21 selections.)
        a = alpha.detach().cpu().numpy().astype(np.float32)
        amax = np.float32(a.max())
        lo = np.zeros(M, np.int64)                 # T_j by bisection: the first v whose
        hi = np.full(M, 1 << 24, np.int64)         # fl32(v 2^-24 amax) >= alpha_j
        while np.any(lo < hi):
            mid = (lo + hi) >> 1
            u = (mid.astype(np.float32) * np.float32(2.0 ** -24)) * amax
            ge = u >= a
            hi = np.where(ge, mid, hi)
            lo = np.where(ge, lo, mid + 1)
        T = lo.astype(np.float64)
        j = np.arange(M + 1, dtype=np.uint64)
        edge = (j * np.uint64(1 << 32) + np.uint64(M - 1)) // np.uint64(M)   # first x mapping to j
        n = np.diff(edge).astype(np.float64)
        wgt = n * T
        law = torch.as_tensor(wgt / wgt.sum(), device=alpha.device)
        p = float(wgt.sum() / 2.0 ** 56)
        return law, 1.0 / p, (1.0 - p) / (p * p), p
    amax_r, a0_r = sel.row_stats()
    law = torch.zeros(M, dtype=torch.float64, device=alpha.device)
    step = 1 << 16
    for r in range(0, alpha.shape[0], step):
        blk = alpha[r:r + step].double()
        d = a0_r[r:r + step].clone()
        d[d == 0] = 1.0                       # all-zero rows contribute nothing (and are rejected)
        law += (blk / d[:, None]).sum(0)
    ok = amax_r > 0
    p = a0_r[ok] / (M * amax_r[ok].double())
    return law, (1.0 / p).sum(), ((1.0 - p) / (p * p)).sum(), None


# ----------------------------------------------------------------- our arm

def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_gpuar(args, w, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1404_0027_b200 import Selector
    from paper_1404_0027_b200.dist import broadcast_vector, max_over_ranks, reduce_validation, shard, weak_shard

    device = torch.device("cuda", local_rank)
    torch.cuda.set_device(device)
    M = w["M"]
    seed = 20140327
    # weak: K selections per rank at [r K, (r+1) K); strong: K in total, contiguous shards
    if args.scaling == "strong":
        K_total = w["K"]
        s0, K = shard(K_total, rank, world)
    else:
        s0, K = weak_shard(w["K"], rank)
        K_total = K * world
    alpha = make_inputs(w, s0, K, device)
    sel = Selector(M, K, seed, device=local_rank)
    sel.set_max_trials(w["max_trials"])
    sel.set_rule(w["rule"], w["w"] if w["rule"] == "argmin" else 1.0)
    sel.set_selection_offset(s0)
    stream = torch.cuda.current_stream(device)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def ev_pair():
        return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    collectives = None
    if w["kind"] == "shared":
        if world > 1:
            # C1: one shared vector for all ranks (warm call, then the timed broadcast)
            scratch = alpha.clone()
            broadcast_vector(scratch, src=0)
            barrier()
            e0, e1 = ev_pair()
            e0.record(stream)
            broadcast_vector(alpha, src=0)
            e1.record(stream)
            e1.synchronize()
            collectives = {"c1_broadcast_ms": max_over_ranks(e0.elapsed_time(e1), device),
                           "c1_bytes": 4 * M}
        else:
            broadcast_vector(alpha, src=0)
    sel.set_propensities(alpha)
    out = (torch.empty(K, dtype=torch.int32, device=device), torch.empty(K, dtype=torch.float32, device=device),
           torch.empty(K, dtype=torch.int32, device=device))
    for _ in range(max(args.warmup, 3)):
        sel.select(K, out=out)
    sel.sync()

    def timed(n_steps, k=K, o=out):
        """n_steps consecutive selects between a barrier + synchronize on both sides; CUDA
        events on the launching stream; (ms of this rank, perf_counter window)."""
        barrier()
        t_start = time.perf_counter()
        e0, e1 = ev_pair()
        e0.record(stream)
        for _ in range(n_steps):
            sel.select(k, out=o)
        e1.record(stream)
        e1.synchronize()
        t_end = time.perf_counter()
        return e0.elapsed_time(e1), t_start, t_end

    path = sel.path
    with ClockSampler(local_rank) as clk:
        clk.wait_first()
        for _ in range(max(args.warmup, 3)):      # re-warm after the sampler start-up
            sel.select(K, out=out)
        ms, t_start, t_end = timed(args.steps)
        time.sleep(0.06)
        clk.mark(t_start, t_end)
    barrier()
    sel.sync()
    ms_max = max_over_ranks(ms, device)        # C3
    ms_step = ms_max / args.steps
    value = K_total * args.steps / (ms_max * 1e-3)
    clocks = clk.summary()

    # Sustained loop (the paper averages over runs): the same step back to
    # back for >= sustain_s seconds, its own clocks -- the power-capped steady state, next to
    # the short burst above.
    sustained = None
    if args.sustain_s > 0:
        n_sus = max(args.steps, int(math.ceil(args.sustain_s * 1e3 / max(ms_step, 1e-3))))
        with ClockSampler(local_rank) as clk2:
            clk2.wait_first()
            ms2, ts0, ts1 = timed(n_sus)
            time.sleep(0.06)
            clk2.mark(ts0, ts1)
        ms2_max = max_over_ranks(ms2, device)
        sus_ms_rank = ms2
        sustained = {"value": K_total * n_sus / (ms2_max * 1e-3), "unit": UNIT, "steps": n_sus,
                     "seconds": ms2_max * 1e-3, "ms_per_step": ms2_max / n_sus, "clocks": clk2.summary()}
        sel.sync()

    # ---- validation of the last step (untimed): histogram, C2 reduce (timed), the law
    hist, totals = sel.histogram(out[0], out[2])
    law, e_trials, v_trials, p_shared = (None, None, None, None)
    if w["rule"] != "argmin":
        law, e_trials, v_trials, p_shared = law_and_trials(w, sel, alpha)
    if world > 1:
        h_s, t_s = hist.clone(), totals.clone()
        reduce_validation(h_s, t_s, dst=0)    # warm
        barrier()
        e0, e1 = ev_pair()
        e0.record(stream)
        reduce_validation(hist, totals, dst=0)     # C2
        e1.record(stream)
        e1.synchronize()
        collectives = dict(collectives or {})
        collectives.update({"c2_reduce_ms": max_over_ranks(e0.elapsed_time(e1), device),
                            "c2_bytes": 8 * (M + 1) + 16, "backend": dist.get_backend()})
        if law is not None and w["kind"] == "rows":
            # per-rank row laws and trial expectations: summed (a shared vector's law is
            # the same on every rank)
            extra = torch.stack([torch.as_tensor(e_trials, dtype=torch.float64, device=device),
                                 torch.as_tensor(v_trials, dtype=torch.float64, device=device)])
            dist.all_reduce(law)
            dist.all_reduce(extra)
            e_trials, v_trials = extra[0], extra[1]
    if law is not None and w["kind"] == "shared":
        e_trials, v_trials = e_trials * K_total, v_trials * K_total   # per selection -> all ranks
    trials_sum = int(totals[0].item())
    rejected = int(totals[1].item())
    if w["rule"] == "argmin":
        calls = K * ((M + 3) // 4 + 1)          # M election draws (4 per call) + tau
    else:
        calls = int(((out[2].to(torch.int64) + 1) // 2).sum().item()) + K   # Philox calls of the last launch

    validation = {"seed": seed, "gen_seed": 14040027, "max_trials": w["max_trials"],
                  "trials_sum_last_step": trials_sum, "rejected_last_step": rejected,
                  "mean_trials": trials_sum / K_total}
    if law is not None and rank == 0:
        h = hist.double().cpu().numpy()
        lw = law.cpu().numpy()
        # the law is over the selections that can fire (all-zero rows are rejected by definition)
        validation["chi2_vs_exact_law"] = chi2_pooled(h[:M], lw * (h[:M].sum() / max(lw.sum(), 1e-300)))
        n = h[:M].sum()
        pj = lw / lw.sum()
        validation["mse"] = float(np.mean((pj - h[:M] / max(n, 1)) ** 2))
        validation["mse_exact_sampler_expectation"] = float(np.sum(pj * (1 - pj)) / (M * max(n, 1)))
        if w["rule"] == "classic":
            e_t, v_t = float(e_trials), float(v_trials)
            acc = {"p_hat": (K_total - rejected) / trials_sum if trials_sum else None,
                   "expected_trials_sum": e_t, "z_trials_sum": (trials_sum - e_t) / math.sqrt(v_t) if v_t > 0 else None}
            if p_shared is not None:
                acc["p"] = float(p_shared)       # exact per-trial acceptance of the discrete draws
                acc["p_continuum"] = float(alpha.double().sum() / (M * alpha.double().max()))  # a0 / (M alpha_max), BASELINE.json configs[2]
            else:
                acc["p_harmonic"] = K_total / e_t   # K / sum_r 1/p_r over the rows
            validation["acceptance"] = acc

    # useful-trial fraction = sum(trials) / trials computed; a team of g lanes
    # computes whole rounds of 2g canonical trials (g = 32 on the matrix path)
    trials_info = None
    if w["rule"] == "classic":
        g = 32 if w["kind"] == "rows" else sel.last_team
        if g > 0:
            t = out[2].to(torch.int64)
            computed = int((((t + 2 * g - 1) // (2 * g)) * (2 * g)).sum().item())
            useful = int(t.sum().item())
            trials_info = {"team": g, "trials_useful": useful, "trials_computed": computed,
                           "useful_trial_fraction": useful / computed if computed else None}

    # NEXT-3 beside the hot path: the classic inverse
    # transform on the same rows, as prefix sums + search and as the paper's linear scan,
    # timed like `value` (the same matrix, events on the launching stream, max over ranks)
    it_cmp = None
    if w["kind"] == "rows" and w["rule"] == "classic" and not args.no_it:
        it_cmp = {}
        n_it = max(3, min(args.steps, 50))
        for rule in ("it", "it_scan"):
            sel.set_rule(rule)
            for _ in range(3):
                sel.select(K, out=out)
            ms_it, _, _ = timed(n_it)
            ms_it = max_over_ranks(ms_it, device)
            it_cmp[rule] = {"value": K_total * n_it / (ms_it * 1e-3), "ms_per_step": ms_it / n_it, "steps": n_it,
                            "hbm_frac": K * (4 * M + 12) / (ms_it / n_it * 1e-3) / 1e9 / float(measured_peaks()["hbm_gbs"])}
        sel.set_rule("classic")
        it_cmp["ar_over_it"] = value / it_cmp["it"]["value"]
        it_cmp["ar_over_it_scan"] = value / it_cmp["it_scan"]["value"]

    # Multi-epoch launches (gpuar_select_epochs): n consecutive selects of the same shared
    # vector in ONE launch, bit-identical to n calls -- an SSA driver keeping the vector for n
    # steps.  Amortises the per-launch ramp, staging and drain; reported beside `value`.
    multi = None
    # (auto: n K ~ 2^24 selections per launch, up to 256 epochs; skipped for calls of >= 10 ms,
    # which have no launch overhead to amortise)
    if w["kind"] == "shared" and w["rule"] == "classic" and args.epochs != 1 and (args.epochs > 1 or ms_step < 10.0):
        n_ep = args.epochs if args.epochs > 1 else max(2, min(256, (1 << 24) // K))
        o_ep = tuple(torch.empty((n_ep, K), dtype=dt, device=device) for dt in (torch.int32, torch.float32, torch.int32))
        for _ in range(3):
            sel.select_epochs(n_ep, K, out=o_ep)
        n_calls = max(3, args.steps // n_ep)
        barrier()
        e0, e1 = ev_pair()
        e0.record(stream)
        for _ in range(n_calls):
            sel.select_epochs(n_ep, K, out=o_ep)
        e1.record(stream)
        e1.synchronize()
        ms_ep = max_over_ranks(e0.elapsed_time(e1), device)
        multi = {"value": K_total * n_ep * n_calls / (ms_ep * 1e-3), "unit": UNIT, "epochs_per_launch": n_ep,
                 "launches": n_calls, "us_per_launch": ms_ep / n_calls * 1e3}

    peaks = measured_peaks()
    if w["kind"] == "rows":
        bytes_per_launch = K * (4 * M + 12)
        ms_rank_step = ms / args.steps
        achieved = bytes_per_launch / (ms_rank_step * 1e-3) / 1e9
        peak = float(peaks["hbm_gbs"])
        traffic = ncu_traffic(args.config) if w["rule"] == "classic" else None
        # diagnostic: the same row pipeline streaming the matrix with only the alpha_max /
        # alpha_0 reduction (gpuar_row_stats, no trials) -- what the pipeline itself can read
        e0, e1 = ev_pair()
        n_rs = 0 if args.no_stream_ceiling else 20
        if n_rs:
            sel.row_stats()
        e0.record(stream)
        for _ in range(n_rs):
            sel.row_stats()
        e1.record(stream)
        e1.synchronize()
        rs_gbs = K * 4 * M / (e0.elapsed_time(e1) / n_rs * 1e-3) / 1e9 if n_rs else None
        # ... and the same stream sustained (>= sustain_s, power-capped like `sustained`): the
        # ceiling the sustained selection rate is compared with
        rs_sus = None
        if sustained and n_rs:
            n_rs2 = max(20, int(args.sustain_s * 1e3 / max(e0.elapsed_time(e1) / n_rs, 1e-3)))
            with ClockSampler(local_rank) as clk3:
                clk3.wait_first()
                t3 = time.perf_counter()
                e0.record(stream)
                for _ in range(n_rs2):
                    sel.row_stats()
                e1.record(stream)
                e1.synchronize()
                t4 = time.perf_counter()
                time.sleep(0.06)
                clk3.mark(t3, t4)
            rs_sus = {"gbs": K * 4 * M / (e0.elapsed_time(e1) / n_rs2 * 1e-3) / 1e9, "launches": n_rs2,
                      "clocks": clk3.summary()}
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": traffic, "peak_source": peaks["_source"] + " hbm_gbs (copy)",
                    "bytes_per_selection": 4 * M + 12, "frac_of_8TBs": achieved / 8000.0,
                    "row_stats_stream_gbs": rs_gbs, "row_stats_stream_sustained": rs_sus,
                    "per": "rank 0's launches (CUDA events on its stream)"}
        if w["rule"] == "argmin":
            # the paper's rule draws ceil(M/4) Philox calls per row (plus one for tau): ALU-bound,
            # so its roofline is the Philox peak; the HBM fraction stays beside it
            mhz = float(peaks.get("sm_max_mhz", 1965.0))
            alu_peak = SM_COUNT * FMA_SLOTS_PER_CLK_PER_SM / FMA_SLOTS_PER_PHILOX * mhz * 1e6 / 1e9
            alu_ach = K * ((M + 3) // 4 + 1) / (ms_rank_step * 1e-3) / 1e9
            hbm = {k: roofline[k] for k in ("achieved", "peak", "unit", "frac", "peak_source", "bytes_per_selection")}
            roofline = {"bound": "alu", "achieved": alu_ach, "peak": alu_peak, "unit": "G Philox calls/s",
                        "frac": alu_ach / alu_peak, "traffic": None,
                        "peak_source": f"148 SM x 64 fma-pipe slots/clk / (20 IMAD.WIDE x 2 slots) per Philox4x32-10 x {mhz:.0f} MHz",
                        "calls_per_selection": (M + 3) // 4 + 1, "hbm": hbm,
                        "per": "rank 0's launches (CUDA events on its stream)"}
        if sustained:
            sustained["roofline_frac"] = K * (4 * M + 12) / (sus_ms_rank / sustained["steps"] * 1e-3) / 1e9 / peak
            if rs_sus:
                # selection bytes/s over the no-trials stream's bytes/s, both sustained
                sustained["frac_of_row_stats_stream"] = (K * 4 * M / (sus_ms_rank / sustained["steps"] * 1e-3) / 1e9
                                                         / rs_sus["gbs"])
    else:
        achieved = calls / (ms_step * 1e-3) / 1e9
        mhz = float(peaks.get("sm_max_mhz", 1965.0))
        peak = SM_COUNT * FMA_SLOTS_PER_CLK_PER_SM / FMA_SLOTS_PER_PHILOX * mhz * 1e6 / 1e9
        roofline = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "G Philox calls/s",
                    "frac": achieved / peak, "traffic": ncu_traffic(args.config),
                    "peak_source": f"148 SM x 64 fma-pipe slots/clk / (20 IMAD.WIDE x 2 slots) per Philox4x32-10 x {mhz:.0f} MHz",
                    "useful_trials_per_launch": trials_sum}
        if multi:
            # the same Philox work per selection (outputs are identical in law), n_ep times per launch
            multi["frac"] = achieved * (multi["value"] / value) / peak

    # e2e: host buffers through gpuar_select_host (H2D + select + D2H inside the timed region)
    e2e = None
    if not args.no_e2e:
        if w["kind"] == "rows":
            host = torch.empty((K, M), dtype=torch.float32, pin_memory=True)
            host.copy_(alpha)
            h2d = host.numel() * 4
        else:
            host = alpha.cpu().pin_memory()
            h2d = host.numel() * 4
        hout = tuple(torch.empty(K, dtype=dt, pin_memory=True) for dt in (torch.int32, torch.float32, torch.int32))
        sel.select_host(host, K=K, out=hout)      # warm-up (allocates staging)
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            sel.select_host(host, K=K, out=hout)
        dt = time.perf_counter() - t0
        dt_max = max_over_ranks(dt, device)
        e2e = {"value": K_total * args.e2e_steps / dt_max, "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 12 * K, "steps": args.e2e_steps,
               # the bound of this number: host<->device bytes per second through PCIe
               "pcie_gbs_per_rank": (h2d + 12 * K) * args.e2e_steps / dt_max / 1e9,
               "timer": "host wall clock around synchronous gpuar_select_host, max over ranks"}
        if w["kind"] == "rows":
            # the link's own ceiling: a plain pinned host->device copy of 1 GiB of the same
            # host buffer (CUDA events), and the e2e loop's fraction of it
            nb = min(host.numel(), 1 << 28)
            src = host.view(-1)[:nb]
            dst = torch.empty(nb, dtype=torch.float32, device=device)
            dst.copy_(src, non_blocking=True)
            e0, e1 = ev_pair()
            e0.record(stream)
            for _ in range(3):
                dst.copy_(src, non_blocking=True)
            e1.record(stream)
            e1.synchronize()
            h2d_peak = 3 * 4 * nb / (e0.elapsed_time(e1) * 1e-3) / 1e9
            e2e["h2d_copy_gbs"] = h2d_peak
            e2e["pcie_frac"] = e2e["pcie_gbs_per_rank"] / h2d_peak
            del dst
        del host
        if w["kind"] == "shared":
            sel.set_propensities(alpha)           # select_host registered its own staged copy

    # Short calls: the same selections replayed from a CUDA graph of
    # consecutive gpuar_select launches (an even number: alternate launches use alternate
    # ticket sets) -- device throughput without the per-call host launch cost.  Secondary
    # figure; `value` above is the plain per-call loop.
    graph = None
    if w["kind"] == "shared" and ms_step < 0.1 and world == 1:
        try:
            n_calls = 100
            gs = torch.cuda.Stream(device)
            gs.wait_stream(stream)
            with torch.cuda.stream(gs):
                sel.select(K, out=out)             # moves the handle to gs outside the capture
                gs.synchronize()
                cg = torch.cuda.CUDAGraph()
                with torch.cuda.graph(cg, stream=gs):
                    for _ in range(n_calls):
                        sel.select(K, out=out)
                cg.replay()
                g0, g1 = ev_pair()
                reps = 20
                g0.record(gs)
                for _ in range(reps):
                    cg.replay()
                g1.record(gs)
                g1.synchronize()
            gms = g0.elapsed_time(g1) / (reps * n_calls)
            graph = {"value": K / (gms * 1e-3), "unit": UNIT, "us_per_call": gms * 1e3, "calls_per_graph": n_calls,
                     "note": "CUDA-graph replay of consecutive selects (same epochs each replay)"}
            sel._stream()                          # back to the default stream for what follows
        except Exception as exc:                   # informational only
            graph = {"error": str(exc)[:200]}

    # Strong-scaling split beside a weak N > 1 run: K = the config's K in TOTAL over the
    # ranks (SURVEY.md §8(d) c4 "strong-scaled over G"), contiguous shards of the global
    # selections; the matrix rows are regenerated for the shard (each rank its own).
    strong = None
    if world > 1 and args.scaling == "weak":
        s0s, Ks = shard(w["K"], rank, world)
        if w["kind"] == "rows":
            import synth
            import synth.gpu as sg
            sub = alpha[:Ks]
            sg.fill_rows(sub, torch.from_numpy(synth.yeast_rates(M)).to(device), synth.GEN_SEED, s0s)
            sel.set_propensities(sub)
        sel.set_selection_offset(s0s)
        o2 = tuple(t[:Ks] for t in out)
        for _ in range(3):
            sel.select(Ks, out=o2)
        ms_s, _, _ = timed(args.steps, Ks, o2)
        ms_s = max_over_ranks(ms_s, device)
        strong = {"value": w["K"] * args.steps / (ms_s * 1e-3), "unit": UNIT, "K_total": w["K"],
                  "K_per_gpu_max": max(shard(w["K"], r, world)[1] for r in range(world)),
                  "ms_per_step": ms_s / args.steps, "steps": args.steps}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        rate, n, dt = oracle_rate(w, args.cpu_seconds, threads,
                                  max_rows=(1 << 17) if w["kind"] == "rows" else None)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "oracle", "cpu_model": cpu_model(),
               "sample": f"first {n} of {K} selections of the same workload, re-run on successive epochs "
                         f"for {dt:.1f} s (OpenMP over selections)"}
        # the same oracle on one host thread (a shorter sample)
        rate1, n1, dt1 = oracle_rate(w, min(3.0, args.cpu_seconds), 1,
                                     max_rows=(1 << 14) if w["kind"] == "rows" else None)
        cpu["value_1thread"] = rate1
        cpu["sample_1thread"] = f"first {n1} selections, {dt1:.1f} s, one thread"
        # the oracle's inverse-transform linear search on the same
        # workload, all cores and one thread -- the classic method the paper argues against
        if w["rule"] == "classic":
            wi = dict(w, rule="it")
            r_it, n_it, dt_it = oracle_rate(wi, min(3.0, args.cpu_seconds), threads,
                                            max_rows=(1 << 17) if w["kind"] == "rows" else None)
            r_it1, n_it1, dt_it1 = oracle_rate(wi, min(2.0, args.cpu_seconds), 1,
                                               max_rows=(1 << 14) if w["kind"] == "rows" else None)
            cpu["it_linear_search"] = {"value": r_it, "cores": threads, "value_1thread": r_it1,
                                       "sample": f"first {n_it} selections ({dt_it:.1f} s, all cores); "
                                                 f"first {n_it1} ({dt_it1:.1f} s, one thread)"}

    if rank == 0:
        res = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded synth/ generators)",
            "config": bench_config(w, args, world),
            "path": path,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": args.steps,
            "clocks": clocks,
            "sustained": sustained,
            "graph_steady_state": graph,
            "it_comparison": it_cmp,
            "multi_epoch": multi,
            "collectives": collectives,
            "strong_scaling": strong,
            "validation": validation,
            "trials": trials_info,
        }
        if args.oversubscribe:
            res["oversubscribed"] = {"gpus_visible": torch.cuda.device_count(),
                                     "note": "ranks share GPUs (dry run): not a scaling measurement"}
        if w["rule"] == "argmin":
            # the paper's Table 1 metric on the last step's histogram and
            # its own K20 timing as context
            h = hist[:M].double().cpu().numpy()
            a = alpha.double().cpu().numpy()
            res["rule_desc"] = f"argmin (paper's printed election + selection), w={w['w']}"
            res["paper_context"] = {
                "mse_vs_normalised_propensities_last_step": float(np.mean((a / a.sum() - h / h.sum()) ** 2)),
                "paper_k20_sel_per_s": PAPER_K20_SEL_PER_S,
                "ratio_to_paper_k20": value / PAPER_K20_SEL_PER_S,
                "note": "paper: 10^7 selections, M=1024, K=62500 in 1326.78 ms on a K20 (timed unit assumed)"}
        print(json.dumps(res), flush=True)
    sel.close()


def ssa_roofline(events_per_s: float) -> dict:
    """Issue-slot roofline of the on-chip SSA loop: warp instructions per event from the
    committed ncu capture of ssa_kernel x events/s, against 148 SM x 4 issue/clk x clock."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    e = json.load(open(p)).get("s1") if os.path.exists(p) else None
    mhz = float(measured_peaks().get("sm_max_mhz", 1965.0))
    peak = SM_COUNT * 4 * mhz * 1e6 / 1e12
    if not e:
        return {"bound": "alu", "achieved": None, "peak": peak, "unit": "T warp-instr/s", "frac": None, "traffic": None}
    ipe = e["warp_instructions_per_launch"] / e["events_per_launch"]
    ach = events_per_s * ipe / 1e12
    return {"bound": "alu", "achieved": ach, "peak": peak, "unit": "T warp-instr/s (issue slots)", "frac": ach / peak,
            "traffic": None, "instructions_per_event": ipe, "source": e["report"],
            "note": f"148 SM x 4 issue/clk x {mhz:.0f} MHz; per event: M mass-action propensities, "
                    "alpha_max/a0, AR trials, state update, all on chip"}


def run_ssa(args, w, rank, world, local_rank):
    """NEXT-2 workload: K realizations advance `inner` SSA steps per launch (gpuar_ssa_run)."""
    import torch

    from paper_1404_0027_b200 import Selector
    from paper_1404_0027_b200.dist import max_over_ranks, weak_shard

    device = torch.device("cuda", local_rank)
    torch.cuda.set_device(device)
    M, K, inner = w["M"], w["K"], w["inner"]
    inp = make_inputs(w, weak_shard(K, rank)[0], K, device)
    sel = Selector(M, K, 20140327, device=local_rank)
    sel.set_selection_offset(weak_shard(K, rank)[0])
    n = inp["net"]
    sel.set_network(n["reac"], n["rate"], n["didx"], n["dval"], inp["N"])
    X, t = inp["X"], inp["t"]
    steps = torch.zeros(K, dtype=torch.int32, device=device)
    total = torch.zeros(K, dtype=torch.int64, device=device)
    for _ in range(max(args.warmup, 3)):
        sel.ssa_run(X, t, inner, steps=steps)
        total += steps  # warms torch's add kernel too: lazy module loading cost ~18 ms on first use
    sel.sync()
    total.zero_()
    stream = torch.cuda.current_stream(device)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        clk.wait_first()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        t_start = time.perf_counter()
        ev0.record(stream)
        for _ in range(args.steps):
            sel.ssa_run(X, t, inner, steps=steps)
            total += steps
        ev1.record(stream)
        ev1.synchronize()
        t_end = time.perf_counter()
        time.sleep(0.06)
        clk.mark(t_start, t_end)
    sel.sync()
    ms = max_over_ranks(ev0.elapsed_time(ev1), device)
    events = int(total.sum().item())
    # realizations halt or reject at different times on each rank: sum the ranks' events
    ev_t = torch.tensor([events], dtype=torch.int64, device=device)
    if world > 1:
        torch.distributed.all_reduce(ev_t)
    events_all = int(ev_t.item())
    value = events_all / (ms * 1e-3)
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu:
            threads = os.cpu_count() or 1
            rate, nn, dt = oracle_rate(w, args.cpu_seconds, threads)
            cpu = {"value": rate, "unit": SSA_UNIT, "cores": threads, "kind": "oracle",
                   "sample": f"{nn} realizations x {inner} steps from the initial state ({dt:.1f} s)"}
        res = {"metric": METRIC, "value": value, "unit": SSA_UNIT, "n_gpus": world,
               "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms / args.steps,
               "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
               "data": "synthetic (seeded synth/ network and initial state)",
               "config": bench_config(w, args, world),
               "roofline": ssa_roofline(value),
               "cpu_baseline": cpu, "e2e": None, "gpu_launches": args.steps, "clocks": clk.summary(),
               "validation": {"events": events, "events_per_realization_per_launch": events / K / args.steps}}
        print(json.dumps(res), flush=True)
    sel.close()


def free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def self_launch(args) -> int:
    """--gpus N without a launcher: run this script as N ranks under torch.distributed.run
    (one process per GPU, rendezvous on 127.0.0.1) and return its exit code.  Refuses when
    fewer than N GPUs are visible, unless --oversubscribe (ranks then share GPUs over gloo)."""
    import torch
    n_vis = torch.cuda.device_count()
    if n_vis < args.gpus and not args.oversubscribe:
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {n_vis} "
              "(--oversubscribe shares GPUs between ranks for a dry run)", file=sys.stderr, flush=True)
        return 2
    argv = list(sys.argv[1:])
    if n_vis < args.gpus and "--dist-backend" not in " ".join(argv):
        argv += ["--dist-backend", "gloo"]      # NCCL refuses two ranks on one GPU
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *argv]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


def main():
    args = parse()
    w = workload(args)
    if args.gpus < 1:
        raise SystemExit("bench.py: --gpus must be >= 1")
    launched = "WORLD_SIZE" in os.environ
    if args.impl == "reference":
        # the oracle arm runs on rank 0's host cores only; without a launcher there is
        # nothing to spawn (the other ranks would exit at once)
        run_reference(args, w, int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", str(args.gpus))))
        return
    if not launched and args.gpus > 1:
        sys.exit(self_launch(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but the launcher started WORLD_SIZE={world} ranks")
    import torch
    import torch.distributed as dist
    n_vis = torch.cuda.device_count()
    if n_vis < 1:
        raise SystemExit("bench.py: no CUDA device visible (the GPU-AR arm has no CPU fallback)")
    if local_rank >= n_vis:
        if not args.oversubscribe:
            raise SystemExit(f"bench.py: local rank {local_rank} has no GPU of its own ({n_vis} visible); "
                             "--oversubscribe for a shared-GPU dry run")
        local_rank %= n_vis
    if world > 1:
        torch.cuda.set_device(local_rank)
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(args.dist_backend)
    try:
        if w["kind"] == "ssa":
            run_ssa(args, w, rank, world, local_rank)
        else:
            run_gpuar(args, w, rank, world, local_rank)
    finally:
        if world > 1:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
