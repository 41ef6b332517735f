"""Diagnostic: host enqueue time vs device time per gpuar_select on a shared vector."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
from paper_1404_0027_b200 import Selector

M = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
dist = sys.argv[2] if len(sys.argv) > 2 else "uniform"
alpha = torch.from_numpy(synth.distribution(dist, M)).cuda()
for K in [1024, 16384, 65536, 262144, 1048576, 4194304]:
    sel = Selector(M, K, 7)
    sel.set_propensities(alpha)
    out = (torch.empty(K, dtype=torch.int32, device="cuda"), torch.empty(K, device="cuda"),
           torch.empty(K, dtype=torch.int32, device="cuda"))
    for _ in range(5):
        sel.select(out=out)
    torch.cuda.synchronize()
    n = 200
    t0 = time.perf_counter()
    for _ in range(n):
        sel.select(out=out)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        sel.select(out=out)
    e1.record()
    e1.synchronize()
    print(f"K={K:8d} host_enqueue_us={(t1 - t0) / n * 1e6:7.2f} wall_us={(t2 - t0) / n * 1e6:7.2f} "
          f"event_us={e0.elapsed_time(e1) / n * 1e3:8.2f}", flush=True)
    sel.close()
