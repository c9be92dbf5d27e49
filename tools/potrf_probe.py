"""Per-kernel-class device times of one config-1 factorisation (gpb_model_set_profiling)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_00136_b200 as gpb
from paper_2505_00136_b200 import _lib

n = int(os.environ.get("N", 8192))
train, _ = gpb.make_msd_dataset(n, 0, 8, seed=0)
rt = gpb.start_runtime()
lib = _lib.load()
model = gpb.GPModel(train, gpb.KernelParams(), 32)
model.compute_loss()
for rep in range(2):
    model.params = gpb.KernelParams(1.0 + 0.01 * (rep + 1))
    lib.gpb_model_set_profiling(model._handle, 1)
    model.compute_loss()
    ms, fl, cnt = (ctypes.c_double * 8)(), (ctypes.c_double * 8)(), (ctypes.c_int64 * 8)()
    lib.gpb_model_kernel_stats(model._handle, ms, fl, cnt)
    lib.gpb_model_set_profiling(model._handle, 0)
    print("factor", round(model.device_timings()["factor"], 2), "ms | gemm", round(ms[0], 2), "ms x", cnt[0],
          "| potrf", round(ms[1], 2), "ms x", cnt[1], "->", round(ms[1] / max(cnt[1], 1) * 1e3, 1), "us each", flush=True)
rt.stop()
