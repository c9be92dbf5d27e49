import sys, time
sys.path.insert(0, '.')
import paper_2505_00136_b200 as gpb
train, _ = gpb.make_msd_dataset(8192, 0, 8, seed=0)
rt = gpb.start_runtime()
for rep in range(2):
    model = gpb.GPModel(train, gpb.KernelParams(1.0, 1.0, 0.1), 32)
    t0 = time.time(); nll = model.compute_loss(); t1 = time.time()
    hist = model.optimize(gpb.AdamConfig(learning_rate=0.1, iterations=3)); t2 = time.time()
    print(f"loss {nll:.6f} {1e3*(t1-t0):.1f} ms; optimize(3) {1e3*(t2-t1):.1f} ms; hist {hist}; timings {model.device_timings()}", flush=True)
    t0 = time.time(); g = model.loss_gradients(); print("grad", g, 1e3*(time.time()-t0), "ms", model.device_timings()['gradient'])
rt.stop()
