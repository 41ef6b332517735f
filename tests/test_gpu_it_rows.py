"""NEXT-3 on the per-realization matrix: the classic inverse transform (PAPER.md:270-275,
§Methods "The SSA") in its two GPU forms -- prefix sums + search (rule "it") and the linear
scan from j = 0 (rule "it_scan") -- bit-exact against oracle.it_select on
the same rows (the oracle's SEQUENTIAL binary64 prefix sums, R24).  Rows whose
partial sums round take the kernel's sequential fallback; both kinds are mixed here."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

SEED = synth.SELECT_SEED
TAU_RTOL = 1e-6


def _run(host, rule, K=None, s0=0, epoch=0, ld=None):
    from paper_1404_0027_b200 import Selector
    K = host.shape[0] if K is None else K
    M = host.shape[1] if ld is None else ld
    sel = Selector(M, K, SEED)
    sel.set_rule(rule)
    sel.set_selection_offset(s0)
    sel.epoch = epoch
    dev = torch.from_numpy(np.ascontiguousarray(host)).cuda()
    if ld is not None:
        dev = dev[:, :M]
    sel.set_propensities(dev)
    out = sel.select(K)
    sel.sync()
    return [t.cpu().numpy() for t in out]


def _check(host, out, s0=0, epoch=0, M=None):
    idx, tau, trials = out
    a = host if M is None else np.ascontiguousarray(host[:, :M])
    K = a.shape[0]
    ref = oracle.it_select(a, K, seed=SEED, epoch=epoch, s0=s0, nthreads=8)
    mism = np.nonzero(idx != ref)[0]
    assert mism.size == 0, f"{mism.size} idx mismatches, first rows {mism[:5]}: gpu {idx[mism[:5]]} oracle {ref[mism[:5]]}"
    live = a.max(axis=1) > 0
    np.testing.assert_array_equal(trials.view(np.uint32), live.astype(np.uint32))
    tref = oracle.ar_select(a, K, seed=SEED, epoch=epoch, s0=s0, max_trials=1, nthreads=8)["tau_ref"]
    fin = np.isfinite(tref)
    assert np.array_equal(np.isinf(tau), np.isinf(tref))
    rel = np.abs(tau[fin].astype(np.float64) - tref[fin]) / tref[fin]
    assert rel.size == 0 or rel.max() <= TAU_RTOL


def _wide_rows(K, M, gen_seed=7):
    """Rows spanning 2^-40 .. 2^40: their binary64 partial sums round (sequential fallback)."""
    rng = np.random.default_rng(gen_seed)
    a = (2.0 ** rng.uniform(-40, 40, (K, M))).astype(np.float32)
    a[rng.random((K, M)) < 0.4] = 0.0
    return a


@pytest.mark.parametrize("rule", ["it", "it_scan"])
def test_it_rows_yeast(rule):
    M, K = synth.YEAST_M, 3001
    host = synth.rows(synth.yeast_rates(M), synth.GEN_SEED, 40, K)
    out = _run(host, rule, s0=40, epoch=3)
    _check(host, out, s0=40, epoch=3)


@pytest.mark.parametrize("rule", ["it", "it_scan"])
@pytest.mark.parametrize("M", [1, 2, 31, 32, 33, 63, 64, 65, 100, 511, 1029, 4099])
def test_it_rows_shapes(rule, M):
    """Every M mod 32 around the block and chunk edges; yeast-like and wide rows mixed."""
    K = 700
    host = synth.rows(synth.yeast_rates(M), synth.GEN_SEED, 0, K)
    host[1::3] = _wide_rows(K, M)[1::3]
    host[5] = 0.0                                   # all-zero row: idx -1, trials 0, tau +inf
    out = _run(host, rule, s0=9, epoch=1)
    _check(host, out, s0=9, epoch=1)
    assert out[0][5] == -1 and out[2][5] == 0 and np.isinf(out[1][5])


@pytest.mark.parametrize("rule", ["it", "it_scan"])
def test_it_rows_sequential_fallback_differs_from_exact_sum(rule):
    """Rows built so that the sequential binary64 sums round: one huge value first, then many
    tiny ones that each vanish in the running sum.  The exact prefix would cross earlier or
    later than the sequential one; the GPU must follow the oracle's sequential rounding."""
    M, K = 257, 2000
    rng = np.random.default_rng(11)
    host = np.zeros((K, M), np.float32)
    host[:, 0] = np.float32(2.0 ** 30)
    host[:, 1:] = (1.0 + rng.random((K, M - 1))).astype(np.float32) * np.float32(2.0 ** -25)
    host[:, -1] = np.float32(2.0 ** 30)             # the second half of the mass at the end
    out = _run(host, rule)
    _check(host, out)
    assert set(np.unique(out[0])) <= {0, M - 1}


@pytest.mark.parametrize("rule", ["it", "it_scan"])
def test_it_rows_pitch_and_invalid(rule):
    from paper_1404_0027_b200 import GpuarError
    M, ld, K = 1029, 1040, 999
    host = np.zeros((K, ld), np.float32)
    host[:, :M] = synth.rows(synth.yeast_rates(M), synth.GEN_SEED, 0, K)
    host[:, M:] = np.nan                            # padding is never read
    out = _run(host, rule, ld=M)
    _check(host, out, M=M)
    bad = synth.rows(synth.yeast_rates(M), synth.GEN_SEED, 0, 64)
    bad[7, 100] = np.nan
    bad[9, 3] = -1.0
    from paper_1404_0027_b200 import Selector
    sel = Selector(M, 64, SEED)
    sel.set_rule(rule)
    sel.set_propensities(torch.from_numpy(bad).cuda())
    idx, tau, trials = sel.select(64)
    with pytest.raises(GpuarError):
        sel.sync()
    idx, tau, trials = idx.cpu().numpy(), tau.cpu().numpy(), trials.cpu().numpy()
    assert idx[7] == -1 and idx[9] == -1 and trials[7] == 0 and np.isnan(tau[7])
    ok = np.ones(64, bool)
    ok[[7, 9]] = False
    np.testing.assert_array_equal(idx[ok], oracle.it_select(bad, 64, seed=SEED, nthreads=8)[ok])


def test_it_rows_geometry_invariant(monkeypatch):
    """Outputs depend only on (row, seed, epoch, s_g): other warp counts, ring depths and
    row-block sizes give the same bytes."""
    M, K = 1029, 5000
    host = synth.rows(synth.yeast_rates(M), synth.GEN_SEED, 0, K)
    base = _run(host, "it")
    for env in ({"GPUAR_ROWS_WARPS": "16"}, {"GPUAR_ROWS_STAGES": "1"}, {"GPUAR_ROWS_LOG2_BLOCK": "0"},
                {"GPUAR_ROWS_LOG2_BLOCK": "5", "GPUAR_NO_PDL": "1"}):
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        for rule in ("it", "it_scan"):
            out = _run(host, rule)
            for a, b in zip(base, out):
                np.testing.assert_array_equal(a.view(np.uint32), b.view(np.uint32))
        for k in env:
            monkeypatch.delenv(k)


def test_it_rows_law():
    """Per-row inverse transform samples alpha_j / alpha_0."""
    a = synth.hand([1, 2, 3, 4])
    K = 100_000
    host = np.tile(a, (K, 1))
    idx = _run(host, "it")[0]
    h = np.bincount(idx, minlength=4)
    assert oracle.chi2_pvalue(h, oracle.exact_law(a))[1] > 0.001


@pytest.mark.slow
def test_it_rows_c4_full_size_sampled():
    """Both IT forms at c4's full size (K = 2^20, M = 1029, generated in HBM by libsynth), as
    bench.py's it_comparison runs them; oracle on sampled rows (first and last 2048, every
    997th); every row's pick must be an enabled reaction."""
    import synth.gpu as sg
    from paper_1404_0027_b200 import Selector
    M, K = synth.YEAST_M, 1 << 20
    rates = synth.yeast_rates(M)
    mat = torch.empty((K, M), dtype=torch.float32, device="cuda")
    sg.fill_rows(mat, torch.from_numpy(rates).cuda(), synth.GEN_SEED, 0)
    rows = np.unique(np.concatenate([np.arange(2048), np.arange(K - 2048, K), np.arange(0, K, 997)]))
    splits = np.nonzero(np.diff(rows) != 1)[0] + 1
    refs = {}
    for run in np.split(rows, splits):
        h = synth.rows(rates, synth.GEN_SEED, int(run[0]), run.size)
        refs[int(run[0])] = (run, oracle.it_select(h, run.size, seed=SEED, epoch=2, s0=int(run[0]), nthreads=8))
    for rule in ("it", "it_scan"):
        sel = Selector(M, K, SEED)
        sel.set_rule(rule)
        sel.epoch = 2
        sel.set_propensities(mat)
        idx, tau, trials = sel.select(K)
        sel.sync()
        gi = idx.cpu().numpy()
        for run, ref in refs.values():
            np.testing.assert_array_equal(gi[run], ref)
        assert (gi >= 0).all() and (trials.cpu().numpy() == 1).all()
        picked = mat.gather(1, idx.long().unsqueeze(1)).squeeze(1)
        assert bool((picked > 0).all())


@pytest.mark.parametrize("rule", ["it", "it_scan", "argmin"])
def test_select_host_rules_on_rows(rule):
    """gpuar_select_host (the e2e path: chunked H2D, select, D2H on three streams) with the
    non-classic rules on a matrix spanning three 64 MB host chunks: identical to the device
    path and (IT) to the oracle."""
    from paper_1404_0027_b200 import Selector
    M, K = 1029, 40_000
    host = synth.rows(synth.yeast_rates(M), synth.GEN_SEED, 0, K)
    sel = Selector(M, K, SEED)
    sel.set_rule(rule, 1.0)
    sel.set_selection_offset(77)
    hi, ht, htr = sel.select_host(torch.from_numpy(host).pin_memory())
    sel.epoch = 0
    sel.set_propensities(torch.from_numpy(host).cuda())
    di, dt, dtr = sel.select(K)
    sel.sync()
    assert torch.equal(hi, di.cpu()) and torch.equal(htr, dtr.cpu())
    assert torch.equal(ht.view(torch.int32), dt.cpu().view(torch.int32))
    if rule != "argmin":
        np.testing.assert_array_equal(hi.numpy(), oracle.it_select(host, K, seed=SEED, s0=77, nthreads=8))


@pytest.mark.parametrize("rule", ["it", "it_scan"])
def test_it_rows_hand_worked_sequential_rounding(rule):
    """The oracle pin of tests/test_oracle_pins.py on the GPU: alpha = (1, 2^-54, 2^-54, 1)
    has binary64 prefix sums (1, 1, 1, 2), so the inverse transform can only pick 0 or 3;
    exact prefix sums would pick 1 for u2 just above 1/2."""
    K = 4096
    host = np.tile(np.array([1.0, 2.0 ** -54, 2.0 ** -54, 1.0], np.float32), (K, 1))
    idx = _run(host, rule)[0]
    assert set(np.unique(idx)) == {0, 3}
    np.testing.assert_array_equal(idx, oracle.it_select(host, K, seed=SEED, nthreads=8))


def test_it_shared_hand_worked_sequential_rounding():
    """Same vector as a shared vector: the IT prefix kernel's sequential path (its partial
    sums round) must give C = (1, 1, 1, 2)."""
    from paper_1404_0027_b200 import Selector
    a = np.array([1.0, 2.0 ** -54, 2.0 ** -54, 1.0], np.float32)
    K = 4096
    sel = Selector(4, K, SEED)
    sel.set_rule("it")
    sel.set_propensities(torch.from_numpy(a).cuda())
    idx = sel.select(K)[0].cpu().numpy()
    sel.sync()
    assert set(np.unique(idx)) == {0, 3}
    np.testing.assert_array_equal(idx, oracle.it_select(a, K, seed=SEED, nthreads=8))
