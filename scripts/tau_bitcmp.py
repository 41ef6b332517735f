"""One-off check: dump idx/tau/trials of a few shared-vector selects (several a0 scales, both
kernels) with the library GPUAR_LIBRARY points at, so two builds can be compared byte for byte:
  GPUAR_LIBRARY=lib/exp_base.so python scripts/tau_bitcmp.py out_a.npz; python scripts/tau_bitcmp.py out_b.npz"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1404_0027_b200 import Selector  # noqa: E402

out = {}
for name, a in [("uniform", synth.uniform(10_000)), ("yeast", synth.yeast_like()), ("pareto", synth.pareto(1000))]:
    for e in (-125, -80, -40, 0, 40, 70):
        v = (a.astype(np.float64) * 2.0 ** e).astype(np.float32)
        for K in (50_000, 400_000):
            sel = Selector(v.size, K, 99)
            sel.set_propensities(torch.from_numpy(np.ascontiguousarray(v)).cuda())
            idx, tau, tr = sel.select(K)
            sel.sync()
            key = f"{name}_{e}_{K}"
            out[key + "_idx"] = idx.cpu().numpy()
            out[key + "_tau"] = tau.cpu().numpy()
            out[key + "_tr"] = tr.cpu().numpy()
np.savez(sys.argv[1], **out)
print("saved", len(out))
