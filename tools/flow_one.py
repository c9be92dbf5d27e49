"""One factorisation + one-launch alpha solve at n = 32768 (ncu target for solve_flow_kernel)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_00136_b200 as gpb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
rt = gpb.start_runtime()
tr, _ = gpb.make_msd_dataset(n, 0, 8, seed=0)
m = gpb.GPModel(tr, gpb.KernelParams(), n // 512)
print(m.log_likelihood(), m.device_timings()["solves"])
rt.stop()
