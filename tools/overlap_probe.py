"""Do SEK assembly (FP64 FMA pipe) and the DMMA GEMM overlap when run
concurrently on two streams?  Times each alone and both together."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_00136_b200 as gpb  # noqa: E402
from paper_2505_00136_b200 import _lib  # noqa: E402

rt = gpb.start_runtime()
lib = _lib.load()
b, d = 512, 128
ntile = 512  # assembly: 512 tiles of 512 x 512 (D = 128)
z = torch.randn(64 * b, d, dtype=torch.float64, device="cuda")
tiles = torch.empty(ntile, b, b, dtype=torch.float64, device="cuda")
desc = (_lib.TileDesc * ntile)(*[_lib.TileDesc(i % 64, (i * 7) % 64 if (i * 7) % 64 <= i % 64 else 0,
                                               tiles[i].data_ptr()) for i in range(ntile)])
# GEMM: 512 output tiles, K = 2048 (a trailing update of 4 panels)
A = torch.randn(4, 64, b, b, dtype=torch.float64, device="cuda")
C = torch.randn(512, b, b, dtype=torch.float64, device="cuda")
jobs = (_lib.GemmJob * 512)(*[_lib.GemmJob(A[0, i % 64].data_ptr(), A[0, (i * 3) % 64].data_ptr(), C[i].data_ptr(),
                                           C[i].data_ptr(), 4 * b, 0) for i in range(512)])
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def asm(s):
    _lib.check(lib.gpb_dev_assemble(rt.handle, ctypes.c_void_p(s.cuda_stream), ctypes.c_void_p(z.data_ptr()), d, b,
                                    1 << 30, 1 << 30, 1.0, 1.0, 0.1, 1, desc, ntile))


def gem(s):
    _lib.check(lib.gpb_dev_gemm_tiled(rt.handle, ctypes.c_void_p(s.cuda_stream), jobs, 512, b, b, b, b, 1, 1, b,
                                      64 * b * b, -1.0, 1.0))


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


for rep in range(3):
    ta = timed(lambda: (asm(s1), s1.synchronize()))
    tg = timed(lambda: (gem(s1), s1.synchronize()))
    tb = timed(lambda: (asm(s1), gem(s2), s1.synchronize(), s2.synchronize()))
    print(f"assembly {ta:.2f} ms, gemm {tg:.2f} ms, both concurrently {tb:.2f} ms (sum {ta + tg:.2f})", flush=True)
rt.stop()
