import numpy as np, sys, os
sys.path.insert(0, '.')
import paper_2505_00136_b200 as gpb
from oracle.tiled_gp import OracleGP, dense_k
rng = np.random.default_rng(2)
z=rng.normal(size=(32,3)); y=rng.normal(size=32)
rt = gpb.start_runtime()
ps = [gpb.KernelParams(1.0, 1.0, 0.1), gpb.KernelParams(1.5, 0.7, 0.3)]
a = gpb.GPModel(gpb.Dataset(z,y), ps[0], 4)
a.factorize(); a.cholesky(); a.log_likelihood()
os.environ["GPB_DEBUG_ASSEMBLY_ONLY"] = "1"
a.params = ps[1]
K = a.cholesky()
Kd = np.tril(dense_k(z, 1.5, 0.7, 0.3))
print("K err", np.abs(np.tril(K) - Kd).max())
print(np.round(K[:6,:6],4)); print(np.round(Kd[:6,:6],4))
b = gpb.GPModel(gpb.Dataset(z,y), ps[1], 4)
Kb = b.cholesky()
print("fresh K err", np.abs(np.tril(Kb) - Kd).max())
rt.stop()
