"""The reference itself (taskgp 0.1.0 from baseline/_ref) at the headline size:
BASELINE config 2 (n = 32768, D = 128, 64 tiles of 512), one compute of the
log-likelihood (assembly + tiled Cholesky + alpha solves) on all host cores --
the like-for-like CPU number for the bench's n = 16384 sample."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
import taskgp  # noqa: E402
from taskgp.model import GPModel  # noqa: E402

from paper_2505_00136_b200.data import make_msd_dataset  # noqa: E402

n, d, tiles = 32768, 128, 64
train, _ = make_msd_dataset(n, 0, d, seed=0)
workers = len(os.sched_getaffinity(0))
taskgp.start_runtime(taskgp.RuntimeConfig(worker_count=workers))
ds = taskgp.Dataset(train.z, train.y)
t0 = time.perf_counter()
ll = GPModel(ds, taskgp.KernelParams(1.0, 1.0, 0.1), tiles_per_dim=tiles).log_likelihood()
dt = time.perf_counter() - t0
taskgp.stop_runtime()
flops = n ** 3 / 3.0 + n ** 2 / 2.0 + n / 6.0
print(f"taskgp config 2 (n={n}, D={d}, {tiles} tiles, {workers} workers): log_likelihood {ll!r} in {dt:.1f} s "
      f"= {flops / dt / 1e12:.3f} TF/s (Cholesky flops, assembly + factor + solves)", flush=True)
