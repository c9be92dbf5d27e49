"""Launch timeline of one factorisation (GPB_PROF_DUMP): every launch's class,
start / end (ms from the phase origin) and flops, and the idle gaps of the
GEMM class.  Usage: factor_timeline.py n tiles"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_00136_b200 as gpb  # noqa: E402
from paper_2505_00136_b200 import _lib  # noqa: E402

n, t = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (8192, 32)
dump = "/tmp/gpb_timeline.txt"
train, _ = gpb.make_msd_dataset(n, 0, 8, seed=0)
rt = gpb.start_runtime()
lib = _lib.load()
m = gpb.GPModel(train, gpb.KernelParams(), t)
m.compute_loss()
for rep in range(3):
    if os.path.exists(dump):
        os.remove(dump)
    m.params = gpb.KernelParams(1.0 + 0.01 * rep)
    lib.gpb_model_set_profiling(m._handle, 1)
    m.compute_loss()
    os.environ["GPB_PROF_DUMP"] = dump
    busy = (ctypes.c_double * 8)()
    lib.gpb_model_kernel_busy(m._handle, busy)
    os.environ.pop("GPB_PROF_DUMP")
    dt = m.device_timings()
names = {0: "GEMM", 1: "POTRF", 2: "SEK", 3: "SOLVE", 4: "OTHER", 5: "PLANES"}
rows = [tuple(float(x) for x in line.split()) for line in open(dump)]
rows.sort(key=lambda r: r[1])
print(f"n={n}: factor {dt['factor']:.3f} ms assembly {dt['assembly']:.3f} solves {dt['solves']:.3f}")
t0 = rows[0][1]
for c, a, b, f in rows:
    print(f"{names[int(c)]:6s} {a - t0:9.3f} {b - t0:9.3f} {1e3 * (b - a):8.1f} us {f / 1e9:8.2f} GF"
          + (f" {f / (b - a) / 1e9:6.1f} TF/s" if f > 0 and b > a else ""))
