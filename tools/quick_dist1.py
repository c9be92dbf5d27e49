"""DistributedGP on one rank (gloo, world 1): overhead of the multi-GPU schedule vs the fused single-GPU path."""
import os, sys, time
sys.path.insert(0, '.')
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29631")
import numpy as np, torch, torch.distributed as dist
dist.init_process_group(os.environ.get("BACKEND", "gloo"), rank=0, world_size=1, **({"device_id": __import__("torch").device("cuda", 0)} if os.environ.get("BACKEND") == "nccl" else {}))
import paper_2505_00136_b200 as gpb
from paper_2505_00136_b200.distributed import DistributedGP
n = int(os.environ.get("N", 32768)); d = int(os.environ.get("D", 128)); T = int(os.environ.get("T", 64)); m = int(os.environ.get("M", 4096))
train, test = gpb.make_msd_dataset(n, m, d, seed=0)
rt = gpb.start_runtime()
flops = n**3/3
for rep in range(int(os.environ.get("REPS", 3))):
    model = DistributedGP(train, gpb.KernelParams(), T)
    t0 = time.time(); ll = model.log_likelihood(); t1 = time.time()
    pv = model.predict_variance(test); t2 = time.time()
    print(f"rep {rep}: ll {ll:.6f} enqueue {model.timings['enqueue_ms']:.1f} ms factor {model.timings['factor_ms']:.1f} ms ({flops/model.timings['factor_ms']/1e9:.2f} TF) solve {model.timings['solve_ms']:.1f} ms wall {t1-t0:.2f}s predict {1e3*(t2-t1):.0f} ms", flush=True)
    model.close()
ref = gpb.GPModel(train, gpb.KernelParams(), T)
print("single-GPU ll", -ref.compute_loss(), ref.device_timings()['factor'], "ms")
rt.stop()
