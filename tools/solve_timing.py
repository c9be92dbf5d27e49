"""Device time of the alpha/beta solves: one-launch dataflow kernel (solve_flow.cu)
vs the 4T-launch blocked solves (GPB_SOLVE_FLOW=0), per BASELINE config size."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2505_00136_b200 as gpb  # noqa: E402

rt = gpb.start_runtime()
for n, t in [(1024, 4), (8192, 32), (32768, 64), (65536, 128)]:
    train, _ = gpb.make_msd_dataset(n, 0, 8, seed=0)
    res = {}
    for flow in ("1", "0"):
        os.environ["GPB_SOLVE_FLOW"] = flow
        times = []
        lls = []
        for rep in range(3):
            m = gpb.GPModel(train, gpb.KernelParams(), t)
            lls.append(m.log_likelihood())
            times.append(m.device_timings()["solves"])
            m.close()
        res[flow] = (min(times), lls[0])
    bi = 512 if n >= 4096 else 256
    T = n // bi
    lower_bytes = 8.0 * bi * bi * T * (T + 1) / 2
    f, s = res["1"], res["0"]
    print(f"n={n}: one-launch {f[0]:.3f} ms ({2 * lower_bytes / f[0] / 1e6:.0f} GB/s of 2 factor reads), "
          f"multi-launch {s[0]:.3f} ms; nll rel diff {abs(f[1] - s[1]) / abs(s[1]):.1e}")
rt.stop()
