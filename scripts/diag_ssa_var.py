"""s1 timing variance: per-launch CUDA-event times of gpuar_ssa_run, with and without the
nvidia-smi clock sampler running, over several fresh Selector instances."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_1404_0027_b200 import Selector

w = bench.CONFIGS["s1"]
dev = torch.device("cuda", 0)


def one(label, sampler, add=False):
    inp = bench.make_inputs(w, 0, dev)
    sel = Selector(w["M"], w["K"], 20140327, device=0)
    n = inp["net"]
    sel.set_network(n["reac"], n["rate"], n["didx"], n["dval"], inp["N"])
    X, t = inp["X"], inp["t"]
    steps = torch.zeros(w["K"], dtype=torch.int32, device=dev)
    for _ in range(5):
        sel.ssa_run(X, t, w["inner"], steps=steps)
    torch.cuda.synchronize()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(41)]
    ctx = bench.ClockSampler(0) if sampler else None
    if ctx:
        ctx.__enter__()
        ctx.wait_first()
    total = torch.zeros(w["K"], dtype=torch.int64, device=dev)
    evs[0].record()
    for i in range(40):
        sel.ssa_run(X, t, w["inner"], steps=steps)
        if add:
            total += steps
        evs[i + 1].record()
    torch.cuda.synchronize()
    if ctx:
        ctx.proc.terminate()
    ms = np.array([evs[i].elapsed_time(evs[i + 1]) for i in range(40)])
    print(f"{label} sampler={sampler} add={add}: total {ms.sum():.2f} ms, per launch min {ms.min():.3f} med {np.median(ms):.3f} max {ms.max():.3f}",
          " ".join(f"{x:.2f}" for x in ms[:40]), flush=True)


for r in range(2):
    one(f"run{r}", False)
    one(f"run{r}", True, add=True)
    one(f"run{r}", False, add=True)
