"""Host-side latency of the public API at small n (BASELINE configs 0 and 1):
wall clock per call against the device time of the same call."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_00136_b200 as gpb  # noqa: E402

for n, m, d, t in [(1024, 1024, 8, 4), (8192, 1024, 8, 32)]:
    train, test = gpb.make_msd_dataset(n, m, d, seed=0)
    rt = gpb.start_runtime()
    for rep in range(4):
        t0 = time.perf_counter()
        model = gpb.GPModel(train, gpb.KernelParams(1.0, 1.0, 0.1), t)
        t1 = time.perf_counter()
        nll = model.compute_loss()
        t2 = time.perf_counter()
        L = model.cholesky()
        t3 = time.perf_counter()
        pv = model.predict_with_uncertainty(test)
        t4 = time.perf_counter()
        g = model.loss_gradients()
        t5 = time.perf_counter()
        dt = model.device_timings()
        model.close()
        print(f"n={n}: create {1e3*(t1-t0):.3f} | compute_loss {1e3*(t2-t1):.3f} | dense L {1e3*(t3-t2):.3f} | "
              f"predict_var {1e3*(t4-t3):.3f} | grad {1e3*(t5-t4):.3f} ms ; device {dt}", flush=True)
    rt.stop()
