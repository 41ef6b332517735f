"""gpuar_select_epochs: n consecutive selects in one call (one launch for a shared vector under
the classic rule) must be bit-identical to n gpuar_select calls -- every selection's draws
depend only on (seed, s_g, epoch) (R6, R12) -- and the first epoch to the oracle."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

SEED = synth.SELECT_SEED


def _vec(name):
    return {"uniform1k": lambda: synth.uniform(1000), "exp10k": lambda: synth.exponential(10_000),
            "pareto1k": lambda: synth.pareto(1000), "yeast": synth.yeast_like,
            "exp70k": lambda: synth.exponential(70_000), "pareto300k": lambda: synth.pareto(300_000),
            "hand": lambda: synth.hand([1, 2, 3, 4])}[name]()


def _compare(sel_a, sel_b, K, n, s0=0, epoch=0):
    """sel_a: one select_epochs call; sel_b: n select calls; both from the same epoch."""
    for s in (sel_a, sel_b):
        s.set_selection_offset(s0)
        s.epoch = epoch
    ia, ta, ra = sel_a.select_epochs(n, K)
    outs = [sel_b.select(K) for _ in range(n)]
    sel_a.sync()
    sel_b.sync()
    assert sel_a.epoch == sel_b.epoch == (epoch + n) & 0xFFFFFFFF
    ib = torch.stack([o[0] for o in outs])
    tb = torch.stack([o[1] for o in outs])
    rb = torch.stack([o[2] for o in outs])
    np.testing.assert_array_equal(ia.cpu().numpy(), ib.cpu().numpy())
    np.testing.assert_array_equal(ta.cpu().numpy().view(np.uint32), tb.cpu().numpy().view(np.uint32))
    np.testing.assert_array_equal(ra.cpu().numpy(), rb.cpu().numpy())
    return ia.cpu().numpy(), ra.cpu().numpy().view(np.uint32)


def _pair(a, K):
    from paper_1404_0027_b200 import Selector
    out = []
    for _ in range(2):
        s = Selector(a.size, K, SEED)
        s.set_propensities(torch.from_numpy(np.ascontiguousarray(a)).cuda())
        out.append(s)
    return out


@pytest.mark.parametrize("name", ["uniform1k", "exp10k", "pareto1k", "yeast", "exp70k", "pareto300k", "hand"])
@pytest.mark.parametrize("K,n", [(1, 7), (33, 64), (5000, 3), (20_000, 16)])
def test_epochs_equal_consecutive_selects(name, K, n):
    a = _vec(name)
    sa, sb = _pair(a, K)
    idx, tr = _compare(sa, sb, K, n, s0=123, epoch=5)
    if K * n <= 20_000:
        ref = oracle.ar_select(a, K, seed=SEED, epoch=5 + n - 1, s0=123, nthreads=8)   # the last epoch
        np.testing.assert_array_equal(idx[-1], ref["idx"])
        np.testing.assert_array_equal(tr[-1], ref["trials"])


@pytest.mark.parametrize("team", [1, 2, 4, 8, 16, 32])
def test_epochs_forced_teams(monkeypatch, team):
    monkeypatch.setenv("GPUAR_TEAM", str(team))
    for name in ("pareto1k", "uniform1k"):
        a = _vec(name)
        sa, sb = _pair(a, 3001)
        _compare(sa, sb, 3001, 5, s0=7, epoch=0xFFFFFFFE)   # the epoch counter wraps inside the launch


def test_epochs_other_rules_and_matrix():
    from paper_1404_0027_b200 import Selector
    a = synth.yeast_like()
    for rule, w in (("argmin", 1.5), ("it", 1.0)):
        sa, sb = _pair(a, 2000)
        for s in (sa, sb):
            s.set_rule(rule, w)
        _compare(sa, sb, 2000, 4)
    M, K = 1029, 1500
    host = torch.from_numpy(synth.rows(synth.yeast_rates(M), synth.GEN_SEED, 0, K)).cuda()
    sels = [Selector(M, K, SEED) for _ in range(2)]
    for s in sels:
        s.set_propensities(host)
    _compare(sels[0], sels[1], K, 3)


def test_epochs_errors():
    from paper_1404_0027_b200 import GpuarError, Selector
    a = torch.from_numpy(synth.yeast_like()).cuda()
    sel = Selector(a.numel(), 1 << 20, SEED)
    sel.set_propensities(a)
    with pytest.raises(GpuarError):
        sel.select_epochs(0, 10)
    # K * n >= 2^32 (the raw entry point returns before touching the output pointer)
    assert sel._lib.gpuar_select_epochs(sel._h, 1 << 20, 4096, 1, None, None) == -1
    sel.set_rule("it_scan")
    with pytest.raises(GpuarError):
        sel.select_epochs(2, 10)


def test_c2_multi_epoch_at_bench_config():
    """c2 (M = 1029 yeast-like, K = 65 536) as bench.py's multi_epoch record launches it: 256
    epochs in one launch; sampled epochs against the oracle, trials and tau included."""
    from paper_1404_0027_b200 import Selector
    a = synth.yeast_like()
    K, n = 65_536, 256
    sel = Selector(a.size, K, SEED)
    sel.set_propensities(torch.from_numpy(a).cuda())
    sel.epoch = 9
    idx, tau, tr = sel.select_epochs(n)
    sel.sync()
    idx, tau, tr = idx.cpu().numpy(), tau.cpu().numpy(), tr.cpu().numpy().view(np.uint32)
    for e in (0, 1, 128, 255):
        ref = oracle.ar_select(a, K, seed=SEED, epoch=9 + e, nthreads=8)
        np.testing.assert_array_equal(idx[e], ref["idx"])
        np.testing.assert_array_equal(tr[e], ref["trials"])
        assert (np.abs(tau[e] - ref["tau_ref"]) / ref["tau_ref"]).max() <= 1e-6


def test_epochs_with_rejections_and_invalid_vector():
    """max_trials small enough to reject (trials = max_trials, idx = -1 inside a multi-epoch
    launch), and an invalid vector: every item of every epoch -1 / NaN and the sticky error."""
    from paper_1404_0027_b200 import GpuarError, Selector
    a = synth.pareto(1000)
    sa, sb = _pair(a, 3000)
    for s in (sa, sb):
        s.set_max_trials(5)
    idx, tr = _compare(sa, sb, 3000, 6, s0=11, epoch=2)
    assert (idx == -1).any() and (tr[idx == -1] == 5).all()
    bad = synth.yeast_like().copy()
    bad[17] = np.nan
    sel = Selector(bad.size, 500, SEED)
    sel.set_propensities(torch.from_numpy(bad).cuda())
    i, t, r = sel.select_epochs(3, 500)
    with pytest.raises(GpuarError):
        sel.sync()
    assert (i.cpu() == -1).all() and torch.isnan(t.cpu()).all() and (r.cpu() == 0).all()
