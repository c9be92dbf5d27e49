"""Driver for an ncu capture of the digit-plane product inside the config-2
factorisation (compute_loss: assembly + factorisation + solves).  The
trailing updates launch ozaki_gemm2_kernel twice per update (groups 4..7, then
0..3); capture e.g. launches 2 and 3 (the first full-size UPD of a 4-panel
group):
  ncu --set full --clock-control none --import-source on -k regex:ozaki_gemm2 \
      --launch-skip 2 --launch-count 2 -o gpurun_out/planes python tools/ncu_planes.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_00136_b200 as gpb

n = int(os.environ.get("N", 32768))
train, _ = gpb.make_msd_dataset(n, 0, int(os.environ.get("D", 128)), seed=0)
rt = gpb.start_runtime()
model = gpb.GPModel(train, gpb.KernelParams(), n // 512)
print("loss", model.compute_loss(), model.device_timings())
rt.stop()
