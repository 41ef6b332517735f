"""NEXT-4: the paper's Table 1 and Fig. 2 protocol on
B200 through libgpuar.

For each propensity vector (discrete Gaussian M = 64, 256, 1024; the
yeast-like stand-in for the unpublished iron model, M = 1029), each K in {100, 1000,
10000, 50000, 62500} and each threshold T_w (w = 1, 2), select `n` = 10^7 reaction
indexes (ceil(n/K) epochs of K parallel realizations) `runs` times, and report the
WORST MSE between the normalised propensities and the observed frequencies
 plus the mean device time of the n selections (Fig. 2).  Both the
paper's printed argmin rule and the classic first-accept rule (the hot path) are run.

Measurement only (product path: Selector + gpuar_histogram); tests/test_table1.py compares
the numbers against the paper and the oracle's exact laws.

    python scripts/table1.py [--runs 10] [--n 10000000] [--out profiles/table1_r01.json]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1404_0027_b200 import Selector  # noqa: E402

KS = [100, 1000, 10000, 50000, 62500]
DISTS = {"gaussian64": lambda: synth.discrete_gaussian(64), "gaussian256": lambda: synth.discrete_gaussian(256),
         "gaussian1024": lambda: synth.discrete_gaussian(1024), "yeast1029": lambda: synth.yeast_like()}


def run_cell(alpha: torch.Tensor, K: int, rule: str, w: float, n: int, seed: int) -> dict:
    M = alpha.numel()
    sel = Selector(M, K, seed)
    sel.set_rule(rule, w)
    sel.set_propensities(alpha)
    out = (torch.empty(K, dtype=torch.int32, device="cuda"), torch.empty(K, dtype=torch.float32, device="cuda"),
           torch.empty(K, dtype=torch.int32, device="cuda"))
    hist = torch.zeros(M + 1, dtype=torch.int64, device="cuda")
    totals = torch.zeros(2, dtype=torch.int64, device="cuda")
    epochs = math.ceil(n / K)
    # pass 1: selections + validation histogram
    for _ in range(epochs):
        sel.select(K, out=out)
        sel.histogram(out[0], out[2], hist, totals)
    sel.sync()
    # pass 2: the same n selections (same epochs) timed alone with CUDA events
    sel.epoch = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(epochs):
        sel.select(K, out=out)
    e1.record()
    e1.synchronize()
    h = hist[:M].double().cpu().numpy()
    a = alpha.double().cpu().numpy()
    mse = float(np.mean((a / a.sum() - h / h.sum()) ** 2))
    res = {"mse": mse, "ms": e0.elapsed_time(e1), "selections": epochs * K,
           "rejected": int(totals[1].item()), "trials": int(totals[0].item())}
    sel.close()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--runs", type=int, default=10)
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--dists", default=",".join(DISTS))
    ap.add_argument("--ks", default=",".join(map(str, KS)))
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "table1_r01.json"))
    args = ap.parse_args()
    torch.cuda.set_device(0)
    rows = []
    t_start = time.time()
    for dname in args.dists.split(","):
        a = torch.from_numpy(np.ascontiguousarray(DISTS[dname]())).cuda()
        for K in map(int, args.ks.split(",")):
            for rule, w in (("argmin", 1.0), ("argmin", 2.0), ("classic", 1.0)):
                cells = [run_cell(a, K, rule, w, args.n, 1000 + r) for r in range(args.runs)]
                row = {"dist": dname, "M": a.numel(), "K": K, "rule": rule, "w": w,
                       "worst_mse": max(c["mse"] for c in cells), "mean_mse": float(np.mean([c["mse"] for c in cells])),
                       "mean_ms": float(np.mean([c["ms"] for c in cells])), "selections": cells[0]["selections"],
                       "rejected": sum(c["rejected"] for c in cells), "runs": args.runs}
                rows.append(row)
                print(json.dumps(row), flush=True)
    res = {"protocol": "PAPER.md:562-607 (Table 1), 648-679 (Fig. 2)", "n_per_run": args.n, "runs": args.runs,
           "device": torch.cuda.get_device_name(0), "wall_s": time.time() - t_start, "rows": rows}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
