"""BASELINE config 0 (n = m = 1024, D = 8, 4 tiles of 256): cholesky + predict_with_uncertainty
through the public API, wall clock per call (host numpy in and out)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2505_00136_b200 as gpb

train, test = gpb.make_msd_dataset(1024, 1024, 8, seed=0)
rt = gpb.start_runtime()
for rep in range(5):
    t0 = time.perf_counter()
    model = gpb.GPModel(train, gpb.KernelParams(1.0, 1.0, 0.1), 4)
    L = model.cholesky()
    t1 = time.perf_counter()
    pv = model.predict_with_uncertainty(test)
    t2 = time.perf_counter()
    print(f"cholesky {1e3*(t1-t0):.2f} ms (incl. model creation, dense L export) | predict_with_uncertainty {1e3*(t2-t1):.2f} ms | device {model.device_timings()}", flush=True)
rt.stop()
