"""Config 1 (n = 8192, D = 8): factor / solves / gradient device times per internal tile size."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_00136_b200 as gpb  # noqa: E402

train, _ = gpb.make_msd_dataset(8192, 0, 8, seed=0)
rt = gpb.start_runtime()
for rep in range(3):
    m = gpb.GPModel(train, gpb.KernelParams(1.0, 1.0, 0.1), 32)
    ll = m.compute_loss()
    g = m.loss_gradients()
    dt = m.device_timings()
    m.close()
print(f"GPB_TILE={os.environ.get('GPB_TILE', 'auto')} GPB_PANELS={os.environ.get('GPB_PANELS', 'auto')}: "
      f"factor {dt['factor']:.2f} ms solves {dt['solves']:.2f} gradient {dt['gradient']:.2f} nll {ll!r}", flush=True)
rt.stop()
