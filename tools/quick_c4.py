"""BASELINE config 4 on one GPU (n = 131072, m = 8192, D = 16, T = 256):
timings plus blocking invariance (internal tiles 512 vs 256)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2505_00136_b200 as gpb

n, m, d, T = 131072, 8192, 16, 256
t0 = time.time()
train, test = gpb.make_msd_dataset(n, m, d, seed=0)
print("generated in", round(time.time() - t0, 1), "s", flush=True)
rt = gpb.start_runtime()
res = {}
for tile in (512, 256):
    os.environ["GPB_TILE"] = str(tile)
    model = gpb.GPModel(train, gpb.KernelParams(1.0, 1.0, 0.1), T)
    t0 = time.time(); nll = model.compute_loss(); t1 = time.time()
    tm = model.device_timings()
    pv = model.predict_with_uncertainty(test); t2 = time.time()
    tp = model.device_timings()
    res[tile] = (nll, pv.mean, pv.variance)
    print(json.dumps(dict(tile=tile, nll=nll, loss_wall_s=round(t1 - t0, 2), factor_ms=round(tm["factor"], 1),
                          factor_tflops=round((n**3 / 3) / tm["factor"] / 1e9, 2), assembly_ms=round(tm["assembly"], 1),
                          predict_wall_s=round(t2 - t1, 2), trsm_ms=round(tp["trsm_variance"], 1),
                          cross_ms=round(tp["cross_mean"], 1), var_min=float(pv.variance.min()),
                          var_max=float(pv.variance.max()))), flush=True)
    model.close()
    del model
a, b = res[512], res[256]
rel = lambda x, y: float(np.linalg.norm(x - y) / np.linalg.norm(y))
print(json.dumps(dict(nll_rel=abs(a[0] - b[0]) / abs(b[0]), mean_rel=rel(a[1], b[1]), var_rel=rel(a[2], b[2]))))
rt.stop()
