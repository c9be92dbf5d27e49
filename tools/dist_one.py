"""World-size-1 run of the multi-GPU runtime (library NCCL communicators) at a
given config against the single-GPU model: factor/solve/gradient times, host
enqueue per panel step, bitwise factor check (small n) and loss agreement."""
import os
import sys
import time

import numpy as np
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_00136_b200 as gpb  # noqa: E402
from paper_2505_00136_b200.distributed import DistributedGP  # noqa: E402

n, d, t = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
grad = len(sys.argv) > 4 and sys.argv[4] == "grad"
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533")
dist.init_process_group("gloo", rank=0, world_size=1)
rt = gpb.start_runtime(gpb.RuntimeConfig(device=0))
train, _ = gpb.make_msd_dataset(n, 0, d, seed=0)
m = DistributedGP(train, gpb.KernelParams(1.0, 1.0, 0.1), t)
for it in range(3):
    m.params = gpb.KernelParams(1.0, 1.0, 0.1)
    t0 = time.perf_counter()
    ll = m.log_likelihood()
    print(f"dist: ll={ll!r} wall={time.perf_counter() - t0:.3f}s timings={m.timings}", flush=True)
if grad:
    for it in range(2):
        g = m.loss_gradients()
        print(f"dist grad {g} {m.timings['gradient_ms']:.1f} ms", flush=True)
s = gpb.GPModel(train, gpb.KernelParams(1.0, 1.0, 0.1), t)
for it in range(2):
    s.params = gpb.KernelParams(1.0, 1.0, 0.1)
    lls = s.log_likelihood()
print(f"single: ll={lls!r} rel={abs(ll - lls) / abs(lls):.3e}", flush=True)
if grad:
    gs = s.loss_gradients()
    print(f"single grad {gs} rel={np.max(np.abs(np.array(g) - gs) / np.abs(gs)):.3e}", flush=True)
if n <= 16384:
    same = np.array_equal(m.cholesky(), s.cholesky())
    print(f"factor bitwise equal: {same}", flush=True)
m.close()
s.close()
rt.stop()
dist.destroy_process_group()
