"""Measure the Philox4x32-10 generate-and-fold microkernel (gpuar_bench_philox): calls/s at
full occupancy, the practical ALU ceiling the select kernels are compared against."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1404_0027_b200 import Selector  # noqa: E402


def main():
    sel = Selector(4, 4, 12345)
    n_threads = 148 * 2048 * 4
    calls = 256
    sink = torch.zeros(n_threads, dtype=torch.int32, device="cuda")
    for _ in range(3):
        sel.bench_philox(n_threads, calls, sink)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        sel.bench_philox(n_threads, calls, sink)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    rate = n_threads * calls / (ms * 1e-3)
    print(json.dumps({"kernel": "bench_philox", "threads": n_threads, "calls_per_thread": calls,
                      "ms": ms, "philox_calls_per_s": rate, "trials_per_s": 2 * rate}))


if __name__ == "__main__":
    main()
