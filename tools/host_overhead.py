"""Host-side overhead breakdown of small calls (config 0 shapes)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2505_00136_b200 as gpb
from paper_2505_00136_b200 import _lib

train, test = gpb.make_msd_dataset(1024, 1024, 8, seed=0)
rt = gpb.start_runtime()
lib = _lib.load()
def t(f):
    t0 = time.perf_counter(); r = f(); return 1e3 * (time.perf_counter() - t0), r
for rep in range(4):
    row = {}
    row["create"], h = t(lambda: (lambda hh: (_lib.check(lib.gpb_model_create(rt.handle, _lib.dptr(train.z), _lib.dptr(train.y), 1024, 8, 4, ctypes.byref(hh))), hh)[1])(ctypes.c_void_p()))
    flags = (ctypes.c_uint8 * 3)(1, 1, 1)
    row["set_params"], _ = t(lambda: lib.gpb_model_set_params(h, 1.0, 1.0, 0.1, flags))
    row["cholesky(no export)"], _ = t(lambda: lib.gpb_cholesky(h, None))
    L = np.empty((1024, 1024))
    row["cholesky(export, cached)"], _ = t(lambda: lib.gpb_cholesky(h, _lib.dptr(L)))
    ll = ctypes.c_double()
    row["loglik"], _ = t(lambda: lib.gpb_log_likelihood(h, ctypes.byref(ll)))
    mean, var = np.empty(1024), np.empty(1024)
    row["predict var (1st)"], _ = t(lambda: lib.gpb_predict(h, _lib.dptr(test.z), 1024, 8, _lib.dptr(mean), _lib.dptr(var), None))
    row["predict var (2nd)"], _ = t(lambda: lib.gpb_predict(h, _lib.dptr(test.z), 1024, 8, _lib.dptr(mean), _lib.dptr(var), None))
    row["refactor+predict"], _ = t(lambda: (lib.gpb_model_set_params(h, 1.1, 1.0, 0.1, flags), lib.gpb_predict(h, _lib.dptr(test.z), 1024, 8, _lib.dptr(mean), _lib.dptr(var), None)))
    row["destroy"], _ = t(lambda: lib.gpb_model_destroy(h))
    print({k: round(v, 3) for k, v in row.items()}, flush=True)
rt.stop()
