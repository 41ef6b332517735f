"""Diagnostic: host-side cost of one gpuar_select call from Python, by component."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_1404_0027_b200 import Selector

def per_call(f, n=3000):
    for _ in range(100):
        f()
    t0 = time.perf_counter()
    for _ in range(n):
        f()
    return (time.perf_counter() - t0) / n * 1e6

K, M = 1024, 1000
alpha = torch.from_numpy(synth.distribution("uniform", M)).cuda()
sel = Selector(M, K, 7)
sel.set_propensities(alpha)
out = (torch.empty(K, dtype=torch.int32, device="cuda"), torch.empty(K, device="cuda"),
       torch.empty(K, dtype=torch.int32, device="cuda"))
dev = torch.device("cuda", 0)
e = ctypes.c_uint32()
lib, h = sel._lib, sel._h
p = [ctypes.c_void_p(t.data_ptr()) for t in out]
print("current_stream      %.2f us" % per_call(lambda: torch.cuda.current_stream(dev).cuda_stream))
print("ctypes get_epoch    %.2f us" % per_call(lambda: lib.gpuar_get_epoch(h, ctypes.byref(e))))
print("data_ptr x3         %.2f us" % per_call(lambda: [ctypes.c_void_p(t.data_ptr()) for t in out]))
print("raw gpuar_select    %.2f us" % per_call(lambda: lib.gpuar_select(h, K, p[0], p[1], p[2])))
torch.cuda.synchronize()
print("Selector.select     %.2f us" % per_call(lambda: sel.select(K, out=out)))
torch.cuda.synchronize()
print("empty kernel (torch) %.2f us" % per_call(lambda: out[0].zero_()))
torch.cuda.synchronize()
