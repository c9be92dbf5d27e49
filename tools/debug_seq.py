import numpy as np, sys, os
sys.path.insert(0, '.')
import paper_2505_00136_b200 as gpb
from oracle.tiled_gp import OracleGP
rng = np.random.default_rng(2)
z=rng.normal(size=(32,3)); y=rng.normal(size=32)
rt = gpb.start_runtime()
ps = [gpb.KernelParams(1.0, 1.0, 0.1), gpb.KernelParams(1.5, 0.7, 0.3)]
a = gpb.GPModel(gpb.Dataset(z,y), ps[0], 4)
a.factorize(); a.cholesky(); a.log_likelihood()
a.params = ps[1]
a.factorize()
L = a.cholesky()
print("err", np.abs(L - OracleGP(z,y,4,1.5,0.7,0.3).factor_dense()).max())
rt.stop()
