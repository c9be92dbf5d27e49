"""Gradient phase breakdown at config 1 (n = 8192): GEMM launches and rate."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_00136_b200 as gpb
from paper_2505_00136_b200 import _lib

n = int(os.environ.get("N", 8192))
train, _ = gpb.make_msd_dataset(n, 0, 8, seed=0)
rt = gpb.start_runtime()
lib = _lib.load()
model = gpb.GPModel(train, gpb.KernelParams(), 32)
model.loss_gradients()
for rep in range(2):
    lib.gpb_model_set_profiling(model._handle, 1)
    model.loss_gradients()
    ms, fl, cnt = (ctypes.c_double * 8)(), (ctypes.c_double * 8)(), (ctypes.c_int64 * 8)()
    lib.gpb_model_kernel_stats(model._handle, ms, fl, cnt)
    lib.gpb_model_set_profiling(model._handle, 0)
    print("gradient", round(model.device_timings()["gradient"], 2), "ms | gemm", round(ms[0], 2), "ms x", cnt[0],
          round(fl[0] / max(ms[0], 1e-9) / 1e9, 2), "TF/s | sek", round(ms[2], 2), "| solves", round(ms[3], 2), flush=True)
rt.stop()
