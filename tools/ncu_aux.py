"""Driver for ncu captures of the non-GEMM kernels at config-2 shapes:
SEK assembly (assemble_lower_kernel), cross-covariance + fused mean partials
(cross_kernel) and the prediction finalize (pred_finalize_kernel)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_00136_b200 as gpb

n, m, d, T = 32768, int(os.environ.get("M", 8192)), 128, 64
train, test = gpb.make_msd_dataset(n, m, d, seed=0)
rt = gpb.start_runtime()
model = gpb.GPModel(train, gpb.KernelParams(), T)
print("loss", model.compute_loss())
pv = model.predict_with_uncertainty(test)
print("var range", pv.variance.min(), pv.variance.max())
rt.stop()
