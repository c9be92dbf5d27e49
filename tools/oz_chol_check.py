"""Factorisation with the trailing updates on the tcgen05 int8 pipe (digit
planes) against the DMMA factorisation: factor difference, loss, timings.

  N=8192 T=16 D=8 python tools/oz_chol_check.py           # parity + timing
  N=32768 T=64 D=128 EXPORT=0 python tools/oz_chol_check.py
"""
import os
import sys
import time

sys.path.insert(0, ".")
import numpy as np

import paper_2505_00136_b200 as gpb

n = int(os.environ.get("N", 8192))
d = int(os.environ.get("D", 8))
T = int(os.environ.get("T", 16))
planes = int(os.environ.get("PLANES", 8))
export = int(os.environ.get("EXPORT", 1))
reps = int(os.environ.get("REPS", 3))
train, test = gpb.make_msd_dataset(n, 256, d, seed=0)
rt = gpb.start_runtime()
flops = n**3 / 3 + n**2 / 2 + n / 6
out = {}
for label, p in (("dmma", 0), ("planes", planes)):
    model = gpb.GPModel(train, gpb.KernelParams(), T)
    model.digit_planes = p
    best = 1e30
    for it in range(reps):
        model.params = gpb.KernelParams()
        model.factorize()
        best = min(best, model.device_timings()["factor"])
    nll = model.compute_loss()
    L = model.cholesky() if export else None
    print(f"{label}: factor {best:.2f} ms = {flops / best / 1e9:.2f} TF/s, loss {nll!r}, "
          f"fallbacks {model.digit_plane_fallbacks()}", flush=True)
    out[label] = (L, nll)
    model.close()
if export:
    a, b = out["dmma"][0], out["planes"][0]
    print("rel fro (planes vs dmma):", np.linalg.norm(a - b) / np.linalg.norm(a))
print("loss rel diff:", abs(out["dmma"][1] - out["planes"][1]) / abs(out["dmma"][1]))
rt.stop()
