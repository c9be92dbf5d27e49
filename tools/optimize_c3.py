"""optimize(3) at config 3 size (n = 65536, D = 8, 128 tiles of 512): the
multi-GPU runtime's replica-free gradient at world size 1 (its own NCCL
communicators) against the single-GPU model; per-phase device times."""
import os
import sys
import time

import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_00136_b200 as gpb  # noqa: E402
from paper_2505_00136_b200.distributed import DistributedGP  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29541")
dist.init_process_group("gloo", rank=0, world_size=1)
rt = gpb.start_runtime(gpb.RuntimeConfig(device=0))
train, _ = gpb.make_msd_dataset(n, 0, 8, seed=0)
opt = gpb.AdamConfig(learning_rate=0.1, iterations=3)
m = DistributedGP(train, gpb.KernelParams(1.0, 1.0, 0.1), n // 512)
t0 = time.perf_counter()
loss0 = m.compute_loss()
t1 = time.perf_counter()
hist = m.optimize(opt)
t2 = time.perf_counter()
print(f"distributed (world 1): compute_loss {t1 - t0:.2f} s, optimize(3) {t2 - t1:.2f} s, history {hist}, "
      f"last gradient {m.timings['gradient_ms']:.0f} ms, factor {m.timings['factor_ms']:.0f} ms", flush=True)
m.close()
s = gpb.GPModel(train, gpb.KernelParams(1.0, 1.0, 0.1), n // 512)
t0 = time.perf_counter()
s.compute_loss()
t1 = time.perf_counter()
hs = s.optimize(opt)
t2 = time.perf_counter()
dt = s.device_timings()
print(f"single GPU: compute_loss {t1 - t0:.2f} s, optimize(3) {t2 - t1:.2f} s, history {hs}, "
      f"last gradient {dt['gradient']:.0f} ms, factor {dt['factor']:.0f} ms", flush=True)
rel = max(abs(a - b) / abs(b) for a, b in zip(hist, hs))
print(f"history max rel diff {rel:.2e}", flush=True)
s.close()
rt.stop()
dist.destroy_process_group()
