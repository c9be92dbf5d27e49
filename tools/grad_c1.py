"""Config 1 gradient (n = 8192): one loss_gradients call after the factor (ncu target)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_00136_b200 as gpb  # noqa: E402

train, _ = gpb.make_msd_dataset(8192, 0, 8, seed=0)
rt = gpb.start_runtime()
m = gpb.GPModel(train, gpb.KernelParams(1.0, 1.0, 0.1), 32)
m.compute_loss()
m.loss_gradients()
print(m.device_timings()["gradient"])
rt.stop()
