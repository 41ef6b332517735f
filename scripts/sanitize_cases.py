"""Small invocations of every libgpuar kernel, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck).  Exits non-zero if any result differs from the oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_1404_0027_b200 import Selector  # noqa: E402

SEED = 7


def check(a, b, what):
    if not np.array_equal(a, b):
        print("MISMATCH", what)
        sys.exit(1)


def main():
    # shared vector, all three smem paths + argmin + IT
    for a in (synth.yeast_like(), synth.exponential(70_000), synth.pareto(300_000)):
        K = 3000
        sel = Selector(a.size, K, SEED)
        sel.set_propensities(torch.from_numpy(a).cuda())
        idx, tau, tr = sel.select(K)
        sel.sync()
        check(idx.cpu().numpy(), oracle.ar_select(a, K, seed=SEED, nthreads=8)["idx"], f"shared {sel.path}")
        hist, tot = sel.histogram(idx, tr)
        sel.set_rule("argmin", 1.5)
        idx, _, _ = sel.select(K)
        sel.sync()
        check(idx.cpu().numpy(), oracle.argmin_select(a, K, seed=SEED, w=1.5, epoch=1, nthreads=8)["idx"], "argmin")
        sel.set_rule("it")
        idx, _, _ = sel.select(K)
        sel.sync()
        check(idx.cpu().numpy(), oracle.it_select(a, K, seed=SEED, epoch=2, nthreads=8), "it")
    # rows (odd M: misaligned rows), stats, argmin rows
    M, K = 1029, 700
    host = synth.rows(synth.yeast_rates(M), synth.GEN_SEED, 0, K)
    sel = Selector(M, K, SEED)
    sel.set_propensities(torch.from_numpy(host).cuda())
    idx, tau, tr = sel.select(K)
    amax, a0 = sel.row_stats()
    sel.sync()
    check(idx.cpu().numpy(), oracle.ar_select(host, K, seed=SEED, nthreads=8)["idx"], "rows")
    sel.set_rule("argmin", 1.0)
    idx, _, _ = sel.select(K)
    sel.sync()
    check(idx.cpu().numpy(), oracle.argmin_select(host, K, seed=SEED, epoch=1, nthreads=8)["idx"], "rows argmin")
    # argmin rows: the partial last call reads past M inside the ring slot (masked)
    for Mo in (5, 1030, 1031):
        ho = synth.rows(synth.yeast_rates(Mo), synth.GEN_SEED, 0, 300)
        so = Selector(Mo, 300, SEED)
        so.set_rule("argmin", 1.0)
        so.set_propensities(torch.from_numpy(ho).cuda())
        io, _, _ = so.select(300)
        so.sync()
        check(io.cpu().numpy(), oracle.argmin_select(ho, 300, seed=SEED, nthreads=8)["idx"], f"rows argmin M={Mo}")
    # inverse transform on the rows: yeast rows (parallel exact path) mixed with wide-range rows
    # (sequential fallback), both forms
    hw = host.copy()
    rng = np.random.default_rng(3)
    hw[1::4] = (2.0 ** rng.uniform(-40, 40, hw[1::4].shape)).astype(np.float32)
    for rule in ("it", "it_scan"):
        sel = Selector(M, K, SEED)
        sel.set_rule(rule)
        sel.set_propensities(torch.from_numpy(hw).cuda())
        idx, _, _ = sel.select(K)
        sel.sync()
        check(idx.cpu().numpy(), oracle.it_select(hw, K, seed=SEED, nthreads=8), f"rows {rule}")
    # shared IT prefix: parallel (Pareto) and sequential (wide range) paths
    for a in (synth.pareto(5000), (2.0 ** rng.uniform(-40, 40, 3000)).astype(np.float32)):
        sel = Selector(a.size, 500, SEED)
        sel.set_rule("it")
        sel.set_propensities(torch.from_numpy(a).cuda())
        idx, _, _ = sel.select(500)
        sel.sync()
        check(idx.cpu().numpy(), oracle.it_select(a, 500, seed=SEED, nthreads=8), "shared it prefix")
    # every shared-vector loop (lane loop with one and two calls, sub-warp teams, warp loop),
    # three back-to-back launches each (PDL overlap, alternating ticket sets), then a forced
    # team size and the non-PDL launch
    for a in (synth.uniform(1000), synth.exponential(10_000), synth.pareto(1000), synth.yeast_like()):
        K = 20_000
        sel = Selector(a.size, K, SEED)
        sel.set_propensities(torch.from_numpy(a).cuda())
        outs = [sel.select(K) for _ in range(3)]
        sel.sync()
        for e, o in enumerate(outs):
            check(o[0].cpu().numpy(), oracle.ar_select(a, K, seed=SEED, epoch=e, nthreads=8)["idx"], f"shared team {sel.last_team}")
    # multi-epoch launches (gpuar_select_epochs) on every loop: equal to consecutive selects
    for a in (synth.uniform(1000), synth.exponential(10_000), synth.pareto(1000), synth.yeast_like(),
              synth.exponential(70_000)):
        K = 3000
        s1, s2 = Selector(a.size, K, SEED), Selector(a.size, K, SEED)
        for s_ in (s1, s2):
            s_.set_propensities(torch.from_numpy(a).cuda())
        ie, _, _ = s1.select_epochs(5, K)
        seq = [s2.select(K)[0] for _ in range(5)]
        s1.sync()
        s2.sync()
        check(ie.cpu().numpy(), torch.stack(seq).cpu().numpy(), f"select_epochs {a.size}")
    for env in ({"GPUAR_TEAM": "16"}, {"GPUAR_TEAM": "8", "GPUAR_NO_PDL": "1", "GPUAR_SH_BLOCK": "256"}):
        os.environ.update(env)
        a = synth.pareto(1000)
        sel = Selector(a.size, 5000, SEED)
        sel.set_propensities(torch.from_numpy(a).cuda())
        outs = [sel.select(5000) for _ in range(2)]
        sel.sync()
        for e, o in enumerate(outs):
            check(o[0].cpu().numpy(), oracle.ar_select(a, 5000, seed=SEED, epoch=e, nthreads=8)["idx"], f"forced {env}")
        for k in env:
            del os.environ[k]
    # host pipeline
    Kh = host.shape[0]
    sel = Selector(M, Kh, SEED)
    hi, _, _ = sel.select_host(torch.from_numpy(host).pin_memory())
    check(hi.numpy(), oracle.ar_select(host, Kh, seed=SEED, nthreads=8)["idx"], "select_host")
    # SSA
    net = synth.yeast_like_network()
    X0 = synth.initial_state(641, 100)
    sel = Selector(net["rate"].size, 100, SEED)
    dev = {k: torch.from_numpy(np.ascontiguousarray(net[k])).cuda() for k in ("reac", "rate", "didx", "dval")}
    sel.set_network(dev["reac"], dev["rate"], dev["didx"], dev["dval"], net["N"])
    X = torch.from_numpy(X0).cuda()
    t = torch.zeros(100, dtype=torch.float64, device="cuda")
    sel.ssa_run(X, t, 10)
    sel.sync()
    check(X.cpu().numpy(), oracle.ssa_run(net, X0, np.zeros(100), 10, seed=SEED)["X"], "ssa")
    # Philox microkernel
    sink = torch.zeros(4096, dtype=torch.int32, device="cuda")
    sel.bench_philox(4096, 4, sink)
    sel.sync()
    print("sanitize cases ok")


if __name__ == "__main__":
    main()
