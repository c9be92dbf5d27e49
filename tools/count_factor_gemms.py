import os, sys, ctypes
sys.path.insert(0, '.')
import paper_2505_00136_b200 as gpb
from paper_2505_00136_b200 import _lib
train, _ = gpb.make_msd_dataset(32768, 0, 128, seed=0)
rt = gpb.start_runtime(); lib = _lib.load()
m = gpb.GPModel(train, gpb.KernelParams(), 64)
m.compute_loss(); m.params = gpb.KernelParams(1.01)
lib.gpb_model_set_profiling(m._handle, 1); m.compute_loss()
ms, fl, cnt = (ctypes.c_double * 8)(), (ctypes.c_double * 8)(), (ctypes.c_int64 * 8)()
lib.gpb_model_kernel_stats(m._handle, ms, fl, cnt); print("factor GEMM launches", cnt[0])
