"""How busy is the DMMA GEMM during the config-2 factorisation?  Device time of
the factor phase against the union of GEMM launch intervals inside it."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_00136_b200 as gpb  # noqa: E402
from paper_2505_00136_b200 import _lib  # noqa: E402

n, t = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (32768, 64)
d = int(sys.argv[3]) if len(sys.argv) > 3 else 8
train, _ = gpb.make_msd_dataset(n, 0, d, seed=0)
rt = gpb.start_runtime()
lib = _lib.load()
m = gpb.GPModel(train, gpb.KernelParams(), t)
m.compute_loss()
for rep in range(2):
    m.params = gpb.KernelParams(1.0 + 0.01 * rep)
    lib.gpb_model_set_profiling(m._handle, 1)
    m.compute_loss()
    busy, ms, fl = (ctypes.c_double * 8)(), (ctypes.c_double * 8)(), (ctypes.c_double * 8)()
    cnt = (ctypes.c_int64 * 8)()
    lib.gpb_model_kernel_busy(m._handle, busy)
    lib.gpb_model_kernel_stats(m._handle, ms, fl, cnt)
    dt = m.device_timings()
    print(f"n={n}: factor {dt['factor']:.2f} ms, assembly {dt['assembly']:.2f}; GEMM busy {busy[0]:.2f} ms "
          f"({cnt[0]} launches, summed {ms[0]:.2f} ms, {fl[0] / busy[0] / 1e9:.2f} TF/s executed over busy), "
          f"POTRF busy {busy[1]:.2f} ms ({cnt[1]}), solve {busy[3]:.2f}; digit-plane products busy "
          f"{busy[5]:.2f} ms ({cnt[5]} launches, summed {ms[5]:.2f} ms, "
          f"{fl[5] / max(busy[5], 1e-9) / 1e9:.2f} TF/s over busy), slicing/other busy {busy[4]:.2f} ms ({cnt[4]})",
          flush=True)
lib.gpb_model_set_profiling(m._handle, 0)
rt.stop()
