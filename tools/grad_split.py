"""Tile-column gradient split (distributed.py gradient_columns) timed on one GPU.

For each world size the column set of every rank is run through
gpb_loss_gradient_terms and timed with the library's device events; the
slowest rank's total is the modelled per-step gradient time on that many
GPUs (the only exchange is a 3-double all-gather).
"""
import ctypes, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2505_00136_b200 as gpb
from paper_2505_00136_b200 import _lib
from paper_2505_00136_b200.distributed import gradient_columns

rt = gpb.start_runtime()
lib = _lib.load()
res = []
for n, d, t in [(8192, 8, 32), (32768, 8, 64)]:
    train, _ = gpb.make_msd_dataset(n, 0, d, seed=0)
    model = gpb.GPModel(train, gpb.KernelParams(), t)
    model.loss_gradients(); g = np.array(model.loss_gradients())
    t_whole = model.device_timings()["gradient"]
    lay = _lib.layout(n, t)
    for world in (1, 2, 4, 8):
        per_rank = []
        tot = np.zeros(3)
        for cols in gradient_columns(lay["T"], world):
            out = (ctypes.c_double * 3)()
            arr = (ctypes.c_int * len(cols))(*cols)
            _lib.check(lib.gpb_loss_gradient_terms(model._handle, arr, len(cols), out))
            per_rank.append(model.device_timings()["gradient"])
            tot += np.array(out[:3])
        row = dict(n=n, T=lay["T"], b=lay["b"], world=world, single_gpu_ms=round(t_whole, 2),
                   max_rank_ms=round(max(per_rank), 2), sum_ms=round(sum(per_rank), 2),
                   modelled_eff=round(t_whole / (world * max(per_rank)), 3))
        print(json.dumps(row), flush=True)
        res.append(row)
rt.stop()
