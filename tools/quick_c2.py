import sys, time, os
sys.path.insert(0, '.')
import numpy as np
import paper_2505_00136_b200 as gpb
n = int(os.environ.get("N", 32768)); m = int(os.environ.get("M", 32768)); d = int(os.environ.get("D", 128)); T = int(os.environ.get("T", 64))
t0 = time.time()
train, test = gpb.make_msd_dataset(n, m, d, seed=0)
print("gen", time.time() - t0, flush=True)
rt = gpb.start_runtime()
model = gpb.GPModel(train, gpb.KernelParams(), T)
flops = n**3/3 + n**2/2 + n/6
for it in range(3):
    model.params = gpb.KernelParams()
    t0 = time.time(); model.factorize(); t1 = time.time()
    tm = model.device_timings()
    print(f"factor wall {t1-t0:.3f}s dev {tm['factor']:.1f} ms asm {tm['assembly']:.1f} ms -> {flops/tm['factor']/1e9:.2f} TF", flush=True)
t0 = time.time(); nll = model.compute_loss(); print("loss", nll, time.time()-t0, model.device_timings()['solves'], "ms solves", flush=True)
for it in range(2):
    t0 = time.time(); r = model.predict_with_uncertainty(test); t1 = time.time()
    tm = model.device_timings()
    print(f"predvar wall {t1-t0:.3f}s cross {tm['cross_mean']:.1f} ms trsm {tm['trsm_variance']:.1f} ms -> {m/(t1-t0):.0f} pts/s; var range {r.variance.min():.3g} {r.variance.max():.3g}", flush=True)
rt.stop()
