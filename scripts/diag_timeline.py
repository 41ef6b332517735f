"""Diagnostic: where a shared-vector select call's time goes, from %globaltimer stamps.

Needs the instrumented build lib/exp_tl.so (nvcc ... -DGPUAR_TIMELINE, see kernels_select.cu),
selected with GPUAR_LIBRARY.  Runs n back-to-back selects (PDL on), then reads the stamps of
the last two launches and splits the last call, per SM, into: gap after the previous call's
CTA left the SM, pre-wait work, tau phase + CTA barrier, trial work until the SM's first warp
exits, the SM's own drain (first to last warp exit), and idle until the whole call ends.
  GPUAR_LIBRARY=paper_1404_0027_b200/lib/exp_tl.so python scripts/diag_timeline.py c2|c3u|c3e
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1404_0027_b200 import Selector, _abi  # noqa: E402

CFG = {"c2": ("yeast", 1029, 65536), "c3u": ("uniform", 10000, 1 << 20), "c3e": ("exponential", 10000, 1 << 20),
       "c3p": ("pareto", 1000, 1 << 20), "c1": ("hand", 4, 10000)}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    dist, M, K = CFG[name]
    if dist == "yeast":
        a = synth.yeast_like()
    elif dist == "hand":
        a = np.array([1, 2, 3, 4], np.float32)
    else:
        a = synth.distribution(dist, M)
    alpha = torch.from_numpy(a).cuda()
    sel = Selector(M, K, 7)
    sel.set_propensities(alpha)
    out = (torch.empty(K, dtype=torch.int32, device="cuda"), torch.empty(K, device="cuda"),
           torch.empty(K, dtype=torch.int32, device="cuda"))
    n = 30
    for _ in range(5):
        sel.select(out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        sel.select(out=out)
    e1.record()
    torch.cuda.synchronize()
    per_call = e0.elapsed_time(e1) / n * 1e3
    lib = _abi.load()
    kTlCta, kTlN = 4 * 1024, 4 * 1024 + 32 * 1024
    buf = np.zeros((2, kTlN), np.uint64)
    assert lib.gpuar_dbg_timeline(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes)) == 0
    last = (5 + n - 1) & 1  # epoch of the last call
    cur, prev = buf[last].astype(np.int64), buf[last ^ 1].astype(np.int64)
    ncta = int(np.count_nonzero(cur[0:4 * 1024:4]))
    wpc = 32  # warps per 1024-thread CTA
    def split(b):
        cta = b[:4 * ncta].reshape(ncta, 4)
        wexit = b[kTlCta:kTlCta + ncta * wpc].reshape(ncta, wpc)
        return cta, wexit
    c_cta, c_w = split(cur)
    p_cta, p_w = split(prev)
    t0 = p_w.max()  # end of the previous call
    sm_prev_exit = {}
    for i in range(ncta):
        sm_prev_exit[int(p_cta[i, 3])] = p_w[i].max()
    rows = []
    for i in range(ncta):
        sm = int(c_cta[i, 3])
        pe = sm_prev_exit.get(sm, t0)
        entry, wait, trial = c_cta[i, 0], c_cta[i, 1], c_cta[i, 2]
        first, lastw = c_w[i].min(), c_w[i].max()
        rows.append([entry - pe, wait - entry, trial - wait, first - trial, lastw - first, c_w.max() - lastw,
                     pe - t0])
    r = np.array(rows, np.float64) / 1e3
    call = (c_w.max() - t0) / 1e3
    labels = ["gap after prev CTA left SM", "entry -> past PDL wait", "tau phase + barrier", "trials to SM's 1st warp exit",
              "SM drain (1st -> last warp exit)", "SM idle until call ends", "(prev CTA exit - prev call end)"]
    print(f"{name}: M={M} K={K} per-call (events) {per_call:.2f} us; last call end-to-end {call:.2f} us; CTAs {ncta}")
    for j, l in enumerate(labels):
        print(f"  {l:36s} mean {r[:, j].mean():7.2f}  min {r[:, j].min():7.2f}  max {r[:, j].max():7.2f} us")
    wt = (c_w - c_cta[:, 2:3]).reshape(-1) / 1e3
    print("  warp exit after trials start, quantiles 0/10/50/90/99/100 %:",
          " ".join(f"{q:.2f}" for q in np.percentile(wt, [0, 10, 50, 90, 99, 100])))
    # work-stealing stripes (warp_global % 64): is the spread between stripes or within them?
    we = (c_w - t0).reshape(-1) / 1e3
    st = np.arange(we.size) % 64
    smax = np.array([we[st == k].max() for k in range(64)])
    smin = np.array([we[st == k].min() for k in range(64)])
    print("  stripe last-exit quantiles 0/50/100 %:", " ".join(f"{q:.2f}" for q in np.percentile(smax, [0, 50, 100])),
          "| within-stripe spread mean", f"{(smax - smin).mean():.2f}", "max", f"{(smax - smin).max():.2f}")
    # when each warp's pool ran dry (0: never asked, e.g. static chunks only) and its tail after
    dry = cur[kTlCta + 16384:kTlCta + 16384 + ncta * wpc].astype(np.int64)
    ok = dry > 0
    if ok.any():
        ex = c_w.reshape(-1)
        print("  pool dry (after prev call end) quantiles 0/10/50/90/100 %:",
              " ".join(f"{q:.2f}" for q in np.percentile((dry[ok] - t0) / 1e3, [0, 10, 50, 90, 100])))
        print("  warp tail (exit - dry) quantiles 0/10/50/90/100 %:",
              " ".join(f"{q:.2f}" for q in np.percentile((ex[ok] - dry[ok]) / 1e3, [0, 10, 50, 90, 100])))
    print(f"  team {sel.last_team}")


if __name__ == "__main__":
    main()
