"""Driver for an ncu capture of an in-situ prediction-sweep GEMM at config 2:
compute_loss (assembly + factorisation + solves) then predict_with_uncertainty
for 32768 test points.  With the default schedule the factorisation issues
GPB_FACTOR_GEMMS grouped-GEMM launches, then the sweep issues PRED_W, PRED_V
per row block: launch index FACTOR + 2 i is row block i's PRED_W."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes
import paper_2505_00136_b200 as gpb
from paper_2505_00136_b200 import _lib

train, test = gpb.make_msd_dataset(32768, 32768, 128, seed=0)
rt = gpb.start_runtime()
lib = _lib.load()
model = gpb.GPModel(train, gpb.KernelParams(), 64)
model.compute_loss()
lib.gpb_model_set_profiling(model._handle, 1)
model.predict_with_uncertainty(test)
ms, fl, cnt = (ctypes.c_double * 8)(), (ctypes.c_double * 8)(), (ctypes.c_int64 * 8)()
lib.gpb_model_kernel_stats(model._handle, ms, fl, cnt)
print("prediction GEMM launches", cnt[0], "device ms", round(ms[0], 1), "TF/s", round(fl[0] / ms[0] / 1e9, 2))
rt.stop()
