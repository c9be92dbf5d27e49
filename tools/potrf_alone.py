"""Device time of the diagonal-tile POTRF/TRTRI kernel alone (no concurrent
GEMM): a random SPD b x b tile factored repeatedly through gpb_dev_potrf."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2505_00136_b200 as gpb
from paper_2505_00136_b200.distributed import DeviceTileOps

rt = gpb.start_runtime()
ops = DeviceTileOps(rt, 0)
for b in (128, 256, 512):
    rng = np.random.default_rng(0)
    x = rng.normal(size=(b, b))
    a = x @ x.T / b + np.eye(b)
    src = torch.from_numpy(a).cuda()
    tile, dinv = torch.empty_like(src), torch.empty_like(src)
    logd = torch.zeros(1, dtype=torch.float64, device="cuda")
    info = torch.full((1,), -1, dtype=torch.int32, device="cuda")
    lay = {"b": b, "pad_bp": b, "pad_b": b}
    times = []
    for rep in range(12):
        tile.copy_(src)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ops.potrf(tile, dinv, lay, 0, logd, info)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) * 1e3)
    L = np.linalg.cholesky(a)
    err = np.linalg.norm(np.tril(tile.cpu().numpy()) - L) / np.linalg.norm(L)
    print(f"b={b}: {np.median(times[2:]):.1f} us per tile (median of 10), rel err {err:.1e}, info {int(info.item())}",
          flush=True)
rt.stop()
