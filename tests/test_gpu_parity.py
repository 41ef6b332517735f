"""GPU parity: libgpuar (through its C ABI via the thin binding) against the CPU oracle on
the same seeded inputs.  idx and trials bit-exact; tau within 1e-6 relative of the
oracle's binary64 tau_ref (north_star tolerance); per-row alpha_0 within 1e-6.
"""
import math

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

SEED = synth.SELECT_SEED
TAU_RTOL = 1e-6


def _sel(M, K, seed=SEED):
    from paper_1404_0027_b200 import Selector
    return Selector(M, K, seed)


def _check(gpu, ref, rows=None):
    idx, tau, trials = (t.cpu().numpy() for t in gpu)
    ridx, rtr = ref["idx"], ref["trials"]
    sl = slice(None) if rows is None else rows
    mism = np.nonzero(idx[sl] != ridx)[0]
    assert mism.size == 0, f"{mism.size} idx mismatches, first at {mism[:5]}: gpu {idx[sl][mism[:5]]} oracle {ridx[mism[:5]]}"
    np.testing.assert_array_equal(trials[sl].view(np.uint32), rtr)
    tref = ref["tau_ref"]
    g = tau[sl].astype(np.float64)
    fin = np.isfinite(tref)
    assert np.array_equal(np.isinf(g), np.isinf(tref)) and np.array_equal(np.isnan(g), np.isnan(tref))
    rel = np.abs(g[fin] - tref[fin]) / tref[fin]
    assert rel.size == 0 or rel.max() <= TAU_RTOL, rel.max()


def _shared_case(alpha, K, epoch=0, s0=0, max_trials=None, seed=SEED):
    a = np.asarray(alpha, np.float32)
    sel = _sel(a.size, K, seed)
    if max_trials:
        sel.set_max_trials(max_trials)
    sel.set_selection_offset(s0)
    sel.epoch = epoch
    sel.set_propensities(torch.from_numpy(a).cuda())
    out = sel.select(K)
    sel.sync()
    ref = oracle.ar_select(a, K, seed=seed, epoch=epoch, s0=s0, max_trials=max_trials or (1 << 20), nthreads=8)
    return sel, out, ref


# ---------------------------------------------------------------- shared vector

def test_c1_hand_1234_full():
    sel, out, ref = _shared_case([1, 2, 3, 4], 10_000)
    _check(out, ref)
    amax, a0, p = sel.stats()
    assert (amax, a0) == (4.0, 10.0) and abs(p - 0.625) < 1e-7
    # chi-square against the exact law on the GPU's own outputs
    h = np.bincount(out[0].cpu().numpy(), minlength=4)
    assert oracle.chi2_pvalue(h, oracle.exact_law([1, 2, 3, 4]))[1] > 0.01


@pytest.mark.parametrize("alpha", [[2, 1], [0, 5, 1], [3, 3, 3], [7.5]])
def test_small_vectors(alpha):
    _, out, ref = _shared_case(alpha, 4099)
    _check(out, ref)


def test_golden_file_values_on_gpu():
    _, out, _ = _shared_case([1, 2, 3, 4], 8, seed=14040027)
    assert out[0].cpu().tolist() == [2, 1, 3, 1, 3, 2, 2, 3]
    assert out[2].cpu().tolist() == [1, 1, 1, 1, 1, 2, 2, 2]


def test_c2_yeast_like_full():
    sel, out, ref = _shared_case(synth.yeast_like(), 65536)
    assert sel.path == "smem_thresholds"
    _check(out, ref)
    _, a0, _ = sel.stats()
    assert abs(a0 - ref["a0"][0]) <= 1e-12 * a0


@pytest.mark.parametrize("kind", ["uniform", "exponential", "pareto"])
@pytest.mark.parametrize("M", [1000, 10_000, 100_000])
def test_c3_distributions(kind, M):
    a = synth.distribution(kind, M)
    K = 1 << 14 if not (kind == "pareto" and M == 100_000) else 1 << 12
    sel, out, ref = _shared_case(a, K)
    assert sel.path == ("smem_thresholds" if M <= 50_000 else "smem_bracket16")
    _check(out, ref)
    # acceptance rate vs a0/(M amax) within 4 sigma (north_star invariant)
    p = oracle.acceptance_rate(a)
    t = out[2].cpu().numpy().astype(np.float64)
    assert abs(t.mean() - 1 / p) < 4 * math.sqrt((1 - p) / K) / p + 1e-9


def test_group_max_path_pareto_1e6():
    a = synth.pareto(1_000_000)
    sel, out, ref = _shared_case(a, 256)
    assert sel.path == "smem_group_max"
    _check(out, ref)


def test_group_max_path_uniform():
    a = synth.uniform(600_000)
    sel, out, ref = _shared_case(a, 20_000)
    assert sel.path == "smem_group_max"
    _check(out, ref)


def test_bracket16_boundaries():
    # path 2 (16-bit threshold brackets B_j = min(T_j >> 8, 65535)): alpha_max = 2 (a power of
    # two, so u * alpha_max is exact) and alpha_j = n 2^-15 give T_j = 256 n exactly, i.e.
    # brackets on their boundaries; alpha_j = alpha_max saturates B_j (T_j = 2^24); plus
    # bf16-grid values, values just below them, and zeros
    rng = np.random.default_rng(3)
    M = 70_000
    n = rng.integers(1, 65536, size=M).astype(np.float64)
    a = (n * 2.0 ** -15).astype(np.float32)
    a[::5] = 2.0
    grid = rng.integers(0x3F000000, 0x3FFFFFFF, size=M, dtype=np.uint32)
    grid[::2] &= 0xFFFF0000                     # exactly representable in bf16
    grid[1::2] |= 0x0000FFFF                    # just below the next bf16
    sel_grid = np.arange(M) % 7 == 3
    a[sel_grid] = grid[sel_grid].view(np.float32)
    a[::11] = 0.0
    assert a.max() == 2.0
    sel, out, ref = _shared_case(a, 40_000)
    assert sel.path == "smem_bracket16"
    _check(out, ref)


def test_group_bounds_on_boundaries():
    # path 3 (per-group bounds G = min(ceil(max T_j / 256), 65535)): T_j = 256 n exactly
    # (alpha_max = 2, alpha_j = n 2^-15), saturated groups (alpha_j = alpha_max) and zeros
    rng = np.random.default_rng(5)
    M = 600_000
    a = (rng.integers(1, 65536, size=M).astype(np.float64) * 2.0 ** -15).astype(np.float32)
    a[::997] = 2.0
    a[rng.random(M) < 0.3] = 0.0
    sel, out, ref = _shared_case(a, 20_000)
    assert sel.path == "smem_group_max"
    _check(out, ref)


def test_degenerate_and_single_nonzero():
    _, out, ref = _shared_case([0, 0, 0, 0, 0], 1000)
    _check(out, ref)
    a = np.zeros(300, np.float32)
    a[123] = 2.5
    _, out, ref = _shared_case(a, 3000)
    _check(out, ref)


def test_invalid_vector_sticky_error():
    from paper_1404_0027_b200 import GpuarError
    sel = _sel(4, 64)
    sel.set_propensities(torch.tensor([1.0, -1.0, 2.0, 3.0], device="cuda"))
    idx, tau, trials = sel.select(64)
    with pytest.raises(GpuarError) as e:
        sel.sync()
    assert e.value.status == -5
    sel.sync()                                   # cleared after being reported
    assert (idx.cpu() == -1).all() and torch.isnan(tau.cpu()).all()


@pytest.mark.parametrize("mt", [1, 2, 3, 7])
def test_max_trials_rejected_path(mt):
    _, out, ref = _shared_case(synth.yeast_like(), 5000, max_trials=mt)
    _check(out, ref)
    assert (out[0].cpu() == -1).any()


@pytest.mark.parametrize("mt", [1, 2, 3, 4, 5, 7, 1 << 20])
def test_lane_teams_two_calls_per_round_caps(mt):
    # one lane per selection with two Philox calls per round (p <= 1/4): max_trials caps
    # that end inside the round's first or second call, on either word
    a = synth.exponential(1000)
    sel, out, ref = _shared_case(a, 1 << 18, max_trials=mt, epoch=5, s0=12345)
    assert sel.last_team == 1
    _check(out, ref)


@pytest.mark.parametrize("mt", [300, 1001, 1 << 20])
def test_long_selections_few_per_warp(mt):
    # whole-warp teams with few selections per warp and ~E = 844 trials each (many rounds
    # per selection, the launch's tail made of long selections), including selections
    # rejected at a max_trials cap that is not a multiple of a round's 64 trials
    a = synth.pareto(100_000)
    sel, out, ref = _shared_case(a, 3000, max_trials=mt, epoch=2, s0=99)
    assert sel.last_team == 32
    _check(out, ref)
    if mt < 2000:
        assert (out[0].cpu() == -1).any()


def test_epochs_offsets_and_replay():
    a = synth.exponential(1000)
    sel = _sel(a.size, 5000)
    sel.set_propensities(torch.from_numpy(a).cuda())
    first = [t.clone() for t in sel.select(5000)]
    second = [t.clone() for t in sel.select(5000)]
    assert sel.epoch == 2
    assert not torch.equal(first[0], second[0])
    sel.epoch = 0
    again = sel.select(5000)
    for x, y in zip(first, again):
        assert torch.equal(x, y)
    # sharding: two halves at offsets equal the whole
    sel.epoch = 1
    sel.set_selection_offset(0)
    lo = [t.clone() for t in sel.select(2500)]
    sel.epoch = 1
    sel.set_selection_offset(2500)
    hi = sel.select(2500)
    for x, y, w in zip(lo, hi, second):
        assert torch.equal(torch.cat([x, y]), w)
    sel.sync()
    _check(second, oracle.ar_select(a, 5000, seed=SEED, epoch=1, nthreads=8))


@pytest.mark.parametrize("scale_exp", [-110, -125, 60])
def test_extreme_scales_thresholds(scale_exp):
    # alpha_max below 2^-102 (products of u and alpha_max underflow into subnormals) and
    # large (2^60: tau stays a normal binary32): the integer acceptance thresholds must reproduce
    # the oracle's fl32(u * alpha_max) < alpha_j decisions bit for bit
    a = (synth.yeast_like() * np.float32(2.0 ** scale_exp)).astype(np.float32)
    assert np.isfinite(a).all() and a.max() > 0
    _, out, ref = _shared_case(a, 20_000)
    _check(out, ref)


def test_thresholds_on_grid_values():
    # exact powers of two, values one ulp apart and alpha_j == alpha_max on path 1
    a = np.array([1.0, np.nextafter(np.float32(1.0), np.float32(0)), 0.5, 0.25 + 2 ** -25, 2 ** -24, 2 ** -25,
                  0.0, 1.0, 0.75, np.float32(1) - np.float32(2 ** -24)], dtype=np.float32)
    _, out, ref = _shared_case(a, 50_000)
    _check(out, ref)


def test_top_of_selection_and_epoch_range():
    # selection indices up to 2^32 - 1 and the largest epoch: counter words 1 and 2 at their
    # maxima, on the shared-vector and the matrix paths
    K = 5000
    s0 = (1 << 32) - K
    a = synth.yeast_like()
    _, out, ref = _shared_case(a, K, epoch=0xFFFFFFFF, s0=s0)
    _check(out, ref)
    _, out, ref, _ = _rows_case(1029, K, k0=s0, epoch=0xFFFFFFFF)
    _check(out, ref)


@pytest.mark.slow
def test_huge_shared_vector_group_path():
    # M = 2^26 (268 MB vector): 1024-reaction groups in the shared-memory prefilter
    M = 1 << 26
    a = synth.uniform(M)
    sel, out, ref = _shared_case(a, 4096)
    assert sel.path == "smem_group_max"
    _check(out, ref)


def test_last_team_reports_the_device_choice():
    sel = _sel(1029, 65536)
    assert sel.last_team == 0                       # no shared-vector select yet
    sel.set_propensities(torch.from_numpy(synth.yeast_like()).cuda())
    sel.select(65536)
    g = sel.last_team
    assert g in (1, 2, 4, 8, 16, 32)
    sel2 = _sel(1000, 1 << 20)
    sel2.set_propensities(torch.from_numpy(synth.uniform(1000)).cuda())
    sel2.select(1 << 20)
    assert sel2.last_team == 1                      # p ~ 0.5, many selections: one lane each


def test_power_of_two_scaling_gpu():
    a = synth.yeast_like()
    _, base, _ = _shared_case(a, 20_000)
    _, scaled, _ = _shared_case(a * np.float32(2.0**-40), 20_000)
    assert torch.equal(base[0], scaled[0]) and torch.equal(base[2], scaled[2])
    assert torch.equal(scaled[1], base[1] * 2.0**40)


# ---------------------------------------------------------------- per-realization rows

def _rows_case(M, K, ld=None, k0=0, epoch=0, max_trials=None, rates=None, mutate=None):
    rates = synth.yeast_rates(M) if rates is None else rates
    host = synth.rows(rates, synth.GEN_SEED, k0, K, ld=ld)
    if mutate:
        mutate(host)
    sel = _sel(M, K)
    if max_trials:
        sel.set_max_trials(max_trials)
    sel.set_selection_offset(k0)
    sel.epoch = epoch
    dev = torch.from_numpy(host).cuda()
    view = dev[:, :M] if ld else dev
    sel.set_propensities(view)
    assert sel.path == "rows"
    out = sel.select(K)
    amax, a0 = sel.row_stats()
    ref = oracle.ar_select(host, K, seed=SEED, epoch=epoch, s0=k0, M=M,
                           max_trials=max_trials or (1 << 20), nthreads=8)
    return sel, out, ref, (amax, a0)


@pytest.mark.parametrize("M,K", [(1029, 4096), (1029, 1000), (1, 100), (2, 333), (3, 257), (5, 64),
                                 (255, 1111), (256, 512), (257, 300), (4096, 200), (7000, 64)])
def test_rows_parity(M, K):
    sel, out, ref, (amax, a0) = _rows_case(M, K)
    sel.sync()
    _check(out, ref)
    np.testing.assert_array_equal(amax.cpu().numpy(), ref["amax"])
    d = a0.cpu().numpy()
    np.testing.assert_allclose(d, ref["a0"], rtol=1e-6)


@pytest.mark.parametrize("warps,stages,log2_block", [(24, 2, 0), (24, 2, 5), (16, 4, 3), (20, 1, 1), (32, 1, 2)])
def test_rows_pipeline_shapes(monkeypatch, warps, stages, log2_block):
    # other ring depths, warp counts and row-block sizes of the matrix kernel (the per-warp
    # row count, the 32-bit walk and the block flush) against the oracle, with a ragged K
    monkeypatch.setenv("GPUAR_ROWS_WARPS", str(warps))
    monkeypatch.setenv("GPUAR_ROWS_STAGES", str(stages))
    monkeypatch.setenv("GPUAR_ROWS_LOG2_BLOCK", str(log2_block))
    for M, K in [(1029, 30_001), (37, 4099)]:
        sel, out, ref, (amax, a0) = _rows_case(M, K, k0=12_345, epoch=3)
        sel.sync()
        _check(out, ref)
        np.testing.assert_array_equal(amax.cpu().numpy(), ref["amax"])


def test_rows_too_wide_for_the_ring_is_refused():
    from paper_1404_0027_b200 import GpuarError
    M, K = 60_000, 4
    sel = _sel(M, K)
    with pytest.raises(GpuarError) as e:
        sel.set_propensities(torch.ones((K, M), device="cuda"))
    assert e.value.status == -1


def test_rows_padded_pitch_and_offset():
    sel, out, ref, _ = _rows_case(1029, 999, ld=1036, k0=12345, epoch=5)
    _check(out, ref)


def test_rows_invalid_and_zero_rows():
    from paper_1404_0027_b200 import GpuarError

    def mutate(h):
        h[3, :] = 0.0
        h[10, 7] = np.float32(-1.0)
        h[11, 8] = np.nan
    sel, out, ref, _ = _rows_case(1029, 64, mutate=mutate)
    with pytest.raises(GpuarError):
        sel.sync()
    _check(out, ref)


def test_rows_max_trials():
    sel, out, ref, _ = _rows_case(1029, 2000, max_trials=33)
    _check(out, ref)


@pytest.mark.slow
def test_c4_full_size_sampled():
    """c4 at its full size (K = 2^20, M = 1029, generated in HBM by libsynth), in the
    launch configuration bench.py times; oracle on sampled rows: the first and last 4096
    and every 997th."""
    import synth.gpu as sg
    from paper_1404_0027_b200 import Selector
    M, K = synth.YEAST_M, 1 << 20
    rates = synth.yeast_rates(M)
    d_rates = torch.from_numpy(rates).cuda()
    mat = torch.empty((K, M), dtype=torch.float32, device="cuda")
    sg.fill_rows(mat, d_rates, synth.GEN_SEED, 0)
    sel = Selector(M, K, SEED)
    sel.set_propensities(mat)
    idx, tau, trials = sel.select(K)
    sel.sync()
    rows = np.unique(np.concatenate([np.arange(4096), np.arange(K - 4096, K), np.arange(0, K, 997)]))
    # check the generator agrees on the sampled rows, then run the oracle on host rows
    host = np.concatenate([synth.rows(rates, synth.GEN_SEED, int(r), 1) for r in rows[:64]])
    np.testing.assert_array_equal(mat[torch.from_numpy(rows[:64]).cuda()].cpu().numpy(), host)
    gi, gt, gtr = idx.cpu().numpy(), tau.cpu().numpy(), trials.cpu().numpy().view(np.uint32)
    for start in range(0, rows.size, 4096):
        rr = rows[start:start + 4096]
        # contiguous runs: oracle per run
        splits = np.nonzero(np.diff(rr) != 1)[0] + 1
        for run in np.split(rr, splits):
            h = synth.rows(rates, synth.GEN_SEED, int(run[0]), run.size)
            ref = oracle.ar_select(h, run.size, seed=SEED, s0=int(run[0]), nthreads=8)
            np.testing.assert_array_equal(gi[run], ref["idx"])
            np.testing.assert_array_equal(gtr[run], ref["trials"])
            fin = np.isfinite(ref["tau_ref"])
            rel = np.abs(gt[run][fin] - ref["tau_ref"][fin]) / ref["tau_ref"][fin]
            assert rel.max() <= TAU_RTOL
    # properties at every row: trials >= 1, chosen reaction enabled
    assert (gtr >= 1).all() and (gi >= 0).all()
    chosen = mat[torch.arange(K, device="cuda"), idx.long()]
    assert (chosen > 0).all()


# ---------------------------------------------------------------- host path, helpers

def test_select_host_matches_device_rows():
    from paper_1404_0027_b200 import Selector
    M, K = 1029, 20_000
    host = torch.from_numpy(synth.rows(synth.yeast_rates(M), synth.GEN_SEED, 0, K)).pin_memory()
    sel = Selector(M, K, SEED)
    hi, ht, htr = sel.select_host(host)
    sel.epoch = 0
    sel.set_propensities(host.cuda())
    di, dt, dtr = sel.select(K)
    assert torch.equal(hi, di.cpu()) and torch.equal(ht, dt.cpu()) and torch.equal(htr, dtr.cpu())


def test_select_host_shared_vector():
    from paper_1404_0027_b200 import Selector
    a = synth.yeast_like()
    sel = Selector(a.size, 30_000, SEED)
    hi, ht, htr = sel.select_host(torch.from_numpy(a).pin_memory(), K=30_000)
    ref = oracle.ar_select(a, 30_000, seed=SEED, nthreads=8)
    _check((hi, ht, htr), ref)


def test_histogram_kernel():
    a = synth.yeast_like()
    sel, out, ref = _shared_case(a, 65536, max_trials=64)
    hist, totals = sel.histogram(out[0], out[2])
    h, ts = oracle.histogram(ref["idx"], ref["trials"], a.size)
    np.testing.assert_array_equal(hist.cpu().numpy(), h.astype(np.int64))
    assert totals[0].item() == ts and totals[1].item() == h[-1]


def test_synth_gpu_rows_match_numpy():
    import synth.gpu as sg
    rates = synth.yeast_rates()
    out = torch.empty((300, 1032), dtype=torch.float32, device="cuda")
    sg.fill_rows(out, torch.from_numpy(rates).cuda(), 99, 777)
    np.testing.assert_array_equal(out.cpu().numpy(), synth.rows(rates, 99, 777, 300, ld=1032))


def test_bench_philox_runs():
    sel = _sel(4, 4)
    sink = torch.zeros(1024, dtype=torch.int32, device="cuda")
    sel.bench_philox(1024, 8, sink)
    sel.sync()
    assert sink.abs().sum().item() > 0


# ---------------------------------------------------------------- the paper's printed rule (NEXT-1)

def _argmin_case(alpha, K, w=1.0, epoch=0, s0=0):
    a = np.asarray(alpha, np.float32)
    sel = _sel(a.shape[-1], K)
    sel.set_rule("argmin", w)
    sel.set_selection_offset(s0)
    sel.epoch = epoch
    sel.set_propensities(torch.from_numpy(a).cuda())
    out = sel.select(K)
    sel.sync()
    ref = oracle.argmin_select(a, K, seed=SEED, w=w, epoch=epoch, s0=s0, nthreads=8)
    return out, ref


@pytest.mark.parametrize("M", [4, 5, 64, 256, 1024, 1029])
@pytest.mark.parametrize("w", [1.0, 2.0])
def test_argmin_shared_gaussian(M, w):
    a = synth.discrete_gaussian(M) if M > 5 else np.arange(1, M + 1, dtype=np.float32)
    out, ref = _argmin_case(a, 20_000, w=w, epoch=3, s0=777)
    np.testing.assert_array_equal(out[0].cpu().numpy(), ref["idx"])
    assert (out[2].cpu().numpy() == M).all()
    rel = np.abs(out[1].cpu().numpy() - ref["tau_ref"]) / ref["tau_ref"]
    assert rel.max() <= TAU_RTOL
    if w == 1.0:
        assert (out[0].cpu() >= 0).all()          # zero rejection at w = 1


def test_argmin_shared_law_gpu():
    a = np.asarray([1, 2, 3, 4], np.float32)
    out, _ = _argmin_case(a, 200_000)
    h = np.bincount(out[0].cpu().numpy(), minlength=4)
    assert oracle.chi2_pvalue(h, oracle.argmin_law(a))[1] > 0.001


def test_argmin_large_vector_global_path():
    a = synth.exponential(70_000)
    out, ref = _argmin_case(a, 300, w=1.5)
    np.testing.assert_array_equal(out[0].cpu().numpy(), ref["idx"])


def test_argmin_rows():
    M, K = 1029, 3000
    host = synth.rows(synth.yeast_rates(M), synth.GEN_SEED, 0, K)
    host[5, :] = 0.0
    for w in (1.0, 1.5):
        sel = _sel(M, K)
        sel.set_rule("argmin", w)
        sel.set_propensities(torch.from_numpy(host).cuda())
        idx, tau, trials = sel.select(K)
        sel.sync()
        ref = oracle.argmin_select(host, K, seed=SEED, w=w, nthreads=8)
        np.testing.assert_array_equal(idx.cpu().numpy(), ref["idx"])
        fin = np.isfinite(ref["tau_ref"])
        rel = np.abs(tau.cpu().numpy()[fin] - ref["tau_ref"][fin]) / ref["tau_ref"][fin]
        assert rel.max() <= TAU_RTOL


@pytest.mark.parametrize("M", [1, 2, 3, 4, 5, 31, 63, 64, 65, 95, 128, 130, 257, 1030, 1031, 1032, 4099])
def test_argmin_rows_shapes(M):
    """The row kernel's argmin branch at every M mod 4 and around the 32/64-call loop edges
    (pair loop, leftover calls, partial call), on rows where eligibility is rare (yeast-like
    enable mask: the division path is the exception) and common (discrete Gaussian: most
    reactions eligible), plus an all-zero row and a one-reaction row."""
    K = 700
    rng = np.random.default_rng(1000 + M)
    sparse = synth.rows(synth.yeast_rates(max(M, 2))[:M].copy(), synth.GEN_SEED, 0, K // 2)
    dense = np.tile(synth.discrete_gaussian(M) if M > 5 else np.arange(1, M + 1, dtype=np.float32),
                    (K - K // 2, 1))
    dense *= rng.uniform(0.5, 2.0, size=(dense.shape[0], 1)).astype(np.float32)
    host = np.ascontiguousarray(np.vstack([sparse, dense]).astype(np.float32))
    host[3, :] = 0.0
    host[4, :] = 0.0
    host[4, M // 2] = 3.0
    for w in (1.0, 1.7):
        sel = _sel(M, K)
        sel.set_rule("argmin", w)
        sel.set_propensities(torch.from_numpy(host).cuda())
        idx, tau, trials = sel.select(K)
        sel.sync()
        ref = oracle.argmin_select(host, K, seed=SEED, w=w, nthreads=8)
        np.testing.assert_array_equal(idx.cpu().numpy(), ref["idx"])
        assert idx[3].item() == -1
        # every draw of a row is consumed; an all-zero row draws nothing
        np.testing.assert_array_equal(trials.cpu().numpy(), np.where(host.any(axis=1), M, 0))


def test_set_rule_validation():
    from paper_1404_0027_b200 import GpuarError
    sel = _sel(4, 4)
    with pytest.raises(GpuarError):
        sel.set_rule("classic", 2.0)
    with pytest.raises(GpuarError):
        sel.set_rule("argmin", 0.5)


# ---------------------------------------------------------------- inverse transform (NEXT-3)

def _wide_vector(M, gen_seed=5):
    """2^-40 .. 2^40 with zeros: binary64 partial sums round (the prefix kernel's sequential path)."""
    rng = np.random.default_rng(gen_seed)
    a = (2.0 ** rng.uniform(-40, 40, M)).astype(np.float32)
    a[rng.random(M) < 0.3] = 0.0
    return a


@pytest.mark.parametrize("kind,M", [("hand", 4), ("yeast", 1029), ("exponential", 10_000), ("pareto", 100_000),
                                    ("uniform", 100_000), ("wide", 5_000), ("wide", 1023), ("pareto", 1_000_000)])
def test_it_shared_bit_exact(kind, M):
    """The prefix C (parallel when no partial sum rounds, else sequential, R24) is
    bit-identical to the oracle's sequential sums: the selected indices agree exactly."""
    a = synth.hand([1, 2, 3, 4]) if kind == "hand" else _wide_vector(M) if kind == "wide" else synth.distribution(kind, M)
    K = 50_000 if M <= 100_000 else 3_000
    sel = _sel(a.size, K)
    sel.set_rule("it")
    sel.set_selection_offset(11)
    sel.epoch = 4
    sel.set_propensities(torch.from_numpy(a).cuda())
    idx, tau, trials = sel.select(K)
    sel.sync()
    ref = oracle.it_select(a, K, seed=SEED, epoch=4, s0=11, nthreads=8)
    np.testing.assert_array_equal(idx.cpu().numpy(), ref)
    tref = oracle.ar_select(a, K, seed=SEED, epoch=4, s0=11, max_trials=1, nthreads=8)["tau_ref"]
    assert (np.abs(tau.cpu().numpy() - tref) / tref).max() <= TAU_RTOL
    assert (trials.cpu() == 1).all()


def test_it_law_and_scan_refused_on_shared_vector():
    from paper_1404_0027_b200 import GpuarError
    a = synth.hand([1, 2, 3, 4])
    sel = _sel(4, 100_000)
    sel.set_rule("it")
    sel.set_propensities(torch.from_numpy(a).cuda())
    idx, _, _ = sel.select(100_000)
    h = np.bincount(idx.cpu().numpy(), minlength=4)
    assert oracle.chi2_pvalue(h, oracle.exact_law(a))[1] > 0.001
    sel2 = _sel(4, 8)
    sel2.set_rule("it_scan")        # the linear scan is a per-row (matrix) method
    sel2.set_propensities(torch.from_numpy(a).cuda())
    with pytest.raises(GpuarError):
        sel2.select(8)
    with pytest.raises(GpuarError):
        sel2.select_host(torch.from_numpy(a))


# ---------------------------------------------------------------- full-size shared-vector configs

def _sampled_rows(K):
    return np.unique(np.concatenate([np.arange(2048), np.arange(K - 2048, K), np.arange(0, K, 997)]))


def _check_sampled(a, K, rows, gi, gtr, gt, max_trials=1 << 20):
    splits = np.nonzero(np.diff(rows) != 1)[0] + 1
    for run in np.split(rows, splits):
        ref = oracle.ar_select(a, run.size, seed=SEED, s0=int(run[0]), max_trials=max_trials, nthreads=8)
        np.testing.assert_array_equal(gi[run], ref["idx"])
        np.testing.assert_array_equal(gtr[run], ref["trials"])
        rel = np.abs(gt[run] - ref["tau_ref"]) / ref["tau_ref"]
        assert rel.max() <= TAU_RTOL


@pytest.mark.slow
@pytest.mark.parametrize("kind,M", [("uniform", 10_000), ("exponential", 100_000), ("pareto", 10_000)])
def test_c3_full_size_sampled(kind, M):
    """c3 cells at the bench's K = 2^20 (same launch configuration), oracle on sampled selections."""
    a = synth.distribution(kind, M)
    K = 1 << 20
    sel = _sel(M, K)
    sel.set_propensities(torch.from_numpy(a).cuda())
    idx, tau, trials = sel.select(K)
    sel.sync()
    gi, gt, gtr = idx.cpu().numpy(), tau.cpu().numpy(), trials.cpu().numpy().view(np.uint32)
    _check_sampled(a, K, _sampled_rows(K), gi, gtr, gt)
    # every selection: a positive-propensity reaction, trials >= 1
    assert (gi >= 0).all() and (a[gi] > 0).all() and (gtr >= 1).all()
    p = oracle.acceptance_rate(a)
    assert abs(gtr.mean() - 1 / p) < 5 * math.sqrt((1 - p) / K) / p


@pytest.mark.slow
def test_c5_full_size_sampled():
    """c5 (M = 10^6 Pareto, group-max prefilter path) at the bench's K = 2^21 per GPU with the
    bench's max_trials = 2^24; oracle on a sampled subset (first/last 2048 + every 9973rd)."""
    a = synth.pareto(1_000_000)
    K = 1 << 21
    sel = _sel(a.size, K)
    sel.set_max_trials(1 << 24)
    sel.set_propensities(torch.from_numpy(a).cuda())
    assert sel.path == "smem_group_max"
    idx, tau, trials = sel.select(K)
    sel.sync()
    gi, gt, gtr = idx.cpu().numpy(), tau.cpu().numpy(), trials.cpu().numpy().view(np.uint32)
    rows = np.unique(np.concatenate([np.arange(256), np.arange(K - 256, K), np.arange(0, K, 9973)]))
    _check_sampled(a, K, rows, gi, gtr, gt, max_trials=1 << 24)
    assert (gi >= 0).all() and (a[gi] > 0).all()
    p = oracle.acceptance_rate(a)
    assert abs(gtr.astype(np.float64).mean() - 1 / p) < 5 * math.sqrt((1 - p) / K) / p


# ---------------------------------------------------------------- argument checking through the ABI

def test_abi_error_paths():
    from paper_1404_0027_b200 import GpuarError, Selector
    sel = Selector(8, 16, SEED)
    with pytest.raises(GpuarError) as e:
        sel.select(16)                                    # nothing registered
    assert e.value.status == -4
    with pytest.raises(GpuarError) as e:
        sel.stats()
    assert e.value.status == -4
    base = torch.zeros(16 * 8 + 4, device="cuda")
    with pytest.raises(GpuarError) as e:                  # matrix base not 16-byte aligned
        sel.set_propensities(base[1:1 + 16 * 8].view(16, 8))
    assert e.value.status == -1
    sel.set_propensities(torch.ones(8, device="cuda"))
    with pytest.raises(GpuarError):
        sel.select(17)                                    # K > capacity
    sel.set_selection_offset((1 << 32) - 8)
    with pytest.raises(GpuarError):
        sel.select(16)                                    # offset + K > 2^32
    with pytest.raises(GpuarError):
        sel.set_selection_offset(1 << 32)
    with pytest.raises(GpuarError):
        sel.set_max_trials(0)
    sel.set_selection_offset(0)
    idx, _, _ = sel.select(16)
    sel.sync()
    assert (idx.cpu() >= 0).all()
    m = Selector(8, 4, SEED)
    m.set_propensities(torch.ones((4, 8), device="cuda"))
    with pytest.raises(GpuarError):
        m.select(3)                                       # K != rows for a matrix
    with pytest.raises(GpuarError):
        m.stats()                                         # stats are for shared vectors


def test_stream_switch_keeps_handle_work_ordered():
    """Back-to-back selections issued on two different torch streams through one handle must
    not overlap (they share the work-stealing tickets): results equal the oracle's."""
    a = synth.exponential(1000)
    K = 200_000
    sel = _sel(a.size, K)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(s1):
        sel.set_propensities(torch.from_numpy(a).cuda())
        o1 = sel.select(K)
    with torch.cuda.stream(s2):
        o2 = sel.select(K)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(o1[0].cpu().numpy(), oracle.ar_select(a, K, seed=SEED, epoch=0, nthreads=8)["idx"])
    np.testing.assert_array_equal(o2[0].cpu().numpy(), oracle.ar_select(a, K, seed=SEED, epoch=1, nthreads=8)["idx"])
