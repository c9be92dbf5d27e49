"""Per-rank compute time of the multi-GPU schedule, measured on one B200: each
rank of a P x Q grid runs its own factorisation schedule alone on the GPU with
every collective a no-op (gpb_dist_init_emulate), so the numbers are its
kernels' device time (smaller launches, its share of the tiles, its critical
path) without communication or waits on other ranks.  t_p >= max_r t_r, so
E(p) = t_1 / (p t_p) <= t_1 / (p max_r t_r): an upper bound from measurement.
Run: python tools/rank_emulation.py [config 3|4]"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_00136_b200 as gpb  # noqa: E402
from paper_2505_00136_b200 import _lib  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "3"
n, d, T = (65536, 8, 128) if cfg == "3" else (131072, 16, 256)
train, _ = gpb.make_msd_dataset(n, 0, d, seed=0)
rt = gpb.start_runtime()
lib = _lib.load()


def factor_ms(rank, world, p, q, grad=False):
    dc, m = ctypes.c_void_p(), ctypes.c_void_p()
    _lib.check(lib.gpb_dist_init_emulate(rt.handle, rank, world, p, q, ctypes.byref(dc)))
    _lib.check(lib.gpb_dist_model_create(dc, _lib.dptr(train.z), _lib.dptr(train.y), n, d, T, ctypes.byref(m)))
    flags = (ctypes.c_uint8 * 3)(1, 1, 1)
    best = None
    for it in range(2):
        _lib.check(lib.gpb_dist_set_params(m, 1.0, 1.0, 0.1 + 1e-3 * it, flags))
        try:
            _lib.check(lib.gpb_dist_factor(m))
        except gpb.errors.NotPositiveDefinite:
            pass  # meaningless data; the schedule ran to the end
        t = (ctypes.c_double * 8)()
        lib.gpb_dist_timings(m, t, 8)
        g = None
        if grad:
            out = (ctypes.c_double * 3)()
            lib.gpb_dist_loss_gradients(m, out)  # runs after the factor even if "not PD" (meaningless data)
            tg = (ctypes.c_double * 8)()
            lib.gpb_dist_timings(m, tg, 8)
            g = tg[4]
        best = (t[1], t[2], t[6], g) if best is None or t[1] < best[0] else best
    lib.gpb_dist_model_destroy(m)
    lib.gpb_dist_finalize(dc)
    return best


grad = len(sys.argv) > 2 and sys.argv[2] == "grad"
t1, s1, _, g1 = factor_ms(0, 1, 1, 1, grad)
print(f"config {cfg} (n={n}, T={T}): 1 GPU factor {t1:.1f} ms, solves {s1:.1f} ms"
      + (f", gradient {g1:.1f} ms" if grad else ""), flush=True)
for p, q in [(1, 2), (2, 2), (2, 4)]:
    w = p * q
    res = [factor_ms(r, w, p, q, grad) for r in range(w)]
    f = np.array([x[0] for x in res])
    line = (f"{p}x{q}: per-rank factor ms {np.round(f, 1).tolist()}; max {f.max():.1f} -> E <= "
            f"{t1 / (w * f.max()):.3f}; host enqueue {np.mean([x[2] for x in res]):.1f} us/step")
    if grad:
        gr = np.array([x[3] for x in res])
        line += f"; gradient per rank max {gr.max():.1f} ms -> E <= {g1 / (w * gr.max()):.3f}"
    print(line, flush=True)
rt.stop()
