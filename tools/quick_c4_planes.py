"""BASELINE config 4 on ONE GPU (n = 131072, m = 8192, D = 16, T = 256; ops:
cholesky, compute_loss, predict_with_full_cov) with the long products on the
tcgen05 digit planes (default) and on the FP64 DMMA kernels: timings and the
difference between the two paths."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2505_00136_b200 as gpb

n, m, d, T = (int(os.environ.get(k, v)) for k, v in (("N", 131072), ("M", 8192), ("D", 16), ("T", 256)))
train, test = gpb.make_msd_dataset(n, m, d, seed=0)
rt = gpb.start_runtime()
res = {}
for planes in (8, 0):
    model = gpb.GPModel(train, gpb.KernelParams(1.0, 1.0, 0.1), T)
    model.digit_planes = planes
    t0 = time.time(); nll = model.compute_loss(); t1 = time.time()
    tm = model.device_timings()
    fc = model.predict_with_full_cov(test); t2 = time.time()
    tp = model.device_timings()
    res[planes] = (nll, fc.mean, np.diag(fc.full_covariance).copy(), fc.full_covariance)
    print(json.dumps(dict(planes=planes, nll=nll, loss_wall_s=round(t1 - t0, 2), factor_ms=round(tm["factor"], 1),
                          factor_tflops=round((n**3 / 3) / tm["factor"] / 1e9, 2), solves_ms=round(tm["solves"], 2),
                          predict_full_cov_wall_s=round(t2 - t1, 2), trsm_ms=round(tp["trsm_variance"], 1),
                          full_cov_ms=round(tp["full_cov"], 1), fallbacks=model.digit_plane_fallbacks())), flush=True)
    model.close()
    del model
a, b = res[8], res[0]
rel = lambda x, y: float(np.linalg.norm(x - y) / np.linalg.norm(y))
print(json.dumps(dict(nll_rel=abs(a[0] - b[0]) / abs(b[0]), mean_rel=rel(a[1], b[1]), var_rel=rel(a[2], b[2]),
                      cov_rel=rel(a[3], b[3]), cov_symmetric=bool(np.array_equal(a[3], a[3].T)))))
rt.stop()
