"""The reference's own acceptance corpus on the GPU path (through the C ABI).

Fixtures were produced by running the reference (tests/golden/make_golden.py):

* the oracle-equivalence grid of pkg/tests/test_acceptance.py:35-78,
  (n, m, T) in {16, 64, 256} x {16, 64} x {1, 4, 8}: every output against
  taskgp's own output for that tiling (factor <= 1e-10 relative Frobenius,
  the rest <= 1e-9 relative, BASELINE.json north_star) and against the
  reference's dense checker (pkg/tests/oracles.py) within the reference
  test's 1e-8 max-abs bound;
* determinism across tilings (test_acceptance.py:135-169): tilings 1, 2, 4, 8,
  16 agree within 1e-10 and match the reference's tilings 1 and 4;
* variance consistency (test_acceptance.py:106-132): full-covariance
  diagonal == variance-only output within 1e-12;
* scaled BASELINE config-3 / config-4 shapes at the benchmark tile size
  (b = 512, T = 16);
* full factors by relative Frobenius against the live oracle at BASELINE
  configs 0 and 1;
* the variance clamp (model.py:488-496, test_model.py:165-172) on device
  results: round-off negatives become 0, genuine negatives raise.
"""

import ctypes

import numpy as np
import pytest

import paper_2505_00136_b200 as gpb
from conftest import load_golden
from oracle.tiled_gp import OracleGP, ThreadedCholesky, rel_fro
from paper_2505_00136_b200.errors import NumericalConsistencyError

pytestmark = pytest.mark.gpu

L_TOL = 1e-10  # Cholesky factor, relative Frobenius
TOL = 1e-9     # loss, gradients, mean, variance, covariance (norm-wise relative)


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den else 1.0))


def instance(seed, n, m, d=4):
    """pkg/tests/test_acceptance.py:28-32 inputs."""
    r = np.random.default_rng(seed)
    return (gpb.Dataset(z=r.normal(size=(n, d)), y=r.normal(size=n)),
            gpb.Dataset(z=r.normal(size=(m, d)), y=np.zeros(m)))


@pytest.mark.parametrize("n", [16, 64, 256])
@pytest.mark.parametrize("m", [16, 64])
def test_acceptance_grid(runtime, n, m):
    g = load_golden("accept_grid")
    key = f"n{n}_m{m}"
    train, test = instance(n * 1000 + m, n, m)
    np.testing.assert_array_equal([train.z.sum(), train.y.sum(), test.z.sum()], g[key + "_zsum"])
    worst_dense = 0.0
    for t in (1, 4, 8):
        k = f"{key}_t{t}"
        model = gpb.GPModel(train, gpb.KernelParams(), tiles_per_dim=t)
        L = model.cholesky()
        full = model.predict_with_full_cov(test)
        var = model.predict_variance(test)
        ll = model.log_likelihood()
        assert rel(L, g[k + "_L"]) <= L_TOL
        assert rel(full.mean, g[k + "_mean"]) <= TOL
        assert rel(full.full_covariance, g[k + "_cov"]) <= TOL
        assert rel(var.variance, g[k + "_var"]) <= TOL
        assert abs(ll - float(g[k + "_ll"])) <= TOL * abs(float(g[k + "_ll"]))
        assert rel(model.loss_gradients(), g[k + "_grads"]) <= TOL
        worst_dense = max(worst_dense,
                          np.abs(L - g[key + "_dense_L"]).max(),
                          np.abs(full.mean - g[key + "_dense_mean"]).max(),
                          np.abs(full.full_covariance - g[key + "_dense_cov"]).max(),
                          np.abs(var.variance - np.diag(g[key + "_dense_cov"])).max(),
                          abs(ll - float(g[key + "_dense_ll"])))
    assert worst_dense <= 1e-8  # test_acceptance.py:76


def test_determinism_across_tilings(runtime):
    g = load_golden("determinism")
    train, test = instance(2024, 64, 16)
    np.testing.assert_array_equal([train.z.sum(), train.y.sum(), test.z.sum()], g["zsum"])
    params = gpb.KernelParams(lengthscale=0.9, noise_variance=0.15)
    outs = {}
    for t in (1, 2, 4, 8, 16):
        model = gpb.GPModel(train, params, tiles_per_dim=t)
        full = model.predict_with_full_cov(test)
        outs[t] = (full.mean, full.full_covariance, model.predict_variance(test).variance,
                   model.log_likelihood())
    base = outs[1]
    worst = max(max(np.abs(o[0] - base[0]).max(), np.abs(o[1] - base[1]).max(),
                    np.abs(o[2] - base[2]).max(), abs(o[3] - base[3])) for o in outs.values())
    assert worst <= 1e-10
    for t in (1, 4):
        assert rel(outs[t][0], g[f"t{t}_mean"]) <= TOL
        assert rel(outs[t][1], g[f"t{t}_cov"]) <= TOL
        assert rel(outs[t][2], g[f"t{t}_var"]) <= TOL
        assert abs(outs[t][3] - float(g[f"t{t}_ll"])) <= TOL * abs(float(g[f"t{t}_ll"]))


def test_variance_consistency(runtime):
    worst = 0.0
    for seed in range(10):
        r = np.random.default_rng(seed)
        n = int(r.choice([16, 32, 64]))
        train, test = instance(seed, n, 16)
        params = gpb.KernelParams(lengthscale=float(r.uniform(0.5, 2.0)),
                                  noise_variance=float(r.uniform(0.01, 0.5)))
        model = gpb.GPModel(train, params, tiles_per_dim=4)
        full = model.predict_with_full_cov(test)
        var = model.predict_variance(test)
        worst = max(worst, np.abs(np.diag(full.full_covariance) - var.variance).max())
    assert worst <= 1e-12


def _check_summary(prefix, a, g, tol):
    scale = float(g[prefix + "_fro"])
    assert abs(np.linalg.norm(a) - scale) <= tol * scale
    assert rel(np.diagonal(a), g[prefix + "_diag"]) <= tol
    assert rel(a.sum(axis=0), g[prefix + "_colsum"]) <= tol
    assert rel(a[g[prefix + "_sr"], g[prefix + "_sc"]], g[prefix + "_sv"]) <= tol


@pytest.mark.parametrize("name,m,d", [("c3s", 0, 8), ("c4s", 512, 16)])
def test_scaled_large_configs(runtime, name, m, d):
    """Config 3 / config 4 shapes at b = 512, T = 16, run by the reference."""
    g = load_golden(name)
    train, test = gpb.make_msd_dataset(8192, m, d, seed=0)
    np.testing.assert_array_equal(train.z[:16], g["z_head"])
    model = gpb.GPModel(train, gpb.KernelParams(1.0, 1.0, 0.1), 16)
    _check_summary("L", model.cholesky(), g, L_TOL)
    assert abs(model.compute_loss() + float(g["loglik"])) <= TOL * abs(float(g["loglik"]))
    assert rel(model.loss_gradients(), g["grads"]) <= TOL
    if m:
        pv = model.predict_with_uncertainty(test)
        assert rel(pv.mean, g["mean"]) <= TOL
        assert rel(pv.variance, g["var"]) <= TOL
        _check_summary("cov", model.predict_with_full_cov(test).full_covariance, g, TOL)


@pytest.mark.parametrize("n,m,t", [(1024, 1024, 4), (8192, 0, 32)])
def test_full_factor_against_live_oracle(runtime, n, m, t):
    """BASELINE configs 0 and 1: the whole factor by relative Frobenius (not
    checksums) against the oracle run on the same inputs, plus the loss."""
    import os

    train, _ = gpb.make_msd_dataset(n, m, 8, seed=0)
    model = gpb.GPModel(train, gpb.KernelParams(1.0, 1.0, 0.1), t)
    L = model.cholesky()
    workers = max(1, len(os.sched_getaffinity(0)))
    o = OracleGP(train.z, train.y, t, cholesky=ThreadedCholesky(workers), assembly_workers=workers)
    err = rel_fro(L, o.factor_dense())
    print(f"n={n}: L relative Frobenius {err:.2e}")
    assert err <= L_TOL
    assert abs(model.compute_loss() + o.log_likelihood()) <= TOL * abs(o.log_likelihood())


def _raw_device_variance(model, test):
    """Unclamped device variances (gpb_predict_device skips the clamp)."""
    import torch

    from paper_2505_00136_b200 import _lib

    zt = torch.from_numpy(np.ascontiguousarray(test.z)).cuda()
    mean = torch.empty(test.n, dtype=torch.float64, device="cuda")
    var = torch.empty(test.n, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    h = model._bind()
    _lib.check(_lib.load().gpb_predict_device(h, ctypes.c_void_p(zt.data_ptr()), test.n, test.d,
                                              ctypes.c_void_p(mean.data_ptr()),
                                              ctypes.c_void_p(var.data_ptr())))
    return var.cpu().numpy()


def test_variance_clamp_round_off(runtime):
    """Noise-free model predicting at its own training points: the exact
    variance is 0, the computed one is +-round-off; the public path returns
    the clamped values (model.py:488-496)."""
    z = (np.arange(512, dtype=np.float64) * 3.0).reshape(-1, 1)
    train = gpb.Dataset(z=z, y=np.sin(z[:, 0]))
    model = gpb.GPModel(train, gpb.KernelParams(noise_variance=0.0), tiles_per_dim=4)
    test = gpb.Dataset(z=z, y=np.zeros(512))
    raw = _raw_device_variance(model, test)
    assert raw.min() >= -1e-9 and raw.min() < 0.0  # round-off negatives exist
    got = model.predict_variance(test).variance
    np.testing.assert_array_equal(got, np.where(raw < 0.0, 0.0, raw))
    fc = model.predict_with_full_cov(gpb.Dataset(z=z[:64], y=np.zeros(64))).full_covariance
    assert np.all(np.diagonal(fc) >= 0.0)


def test_variance_clamp_raises_on_genuine_negative(runtime):
    """With a huge vertical scale the round-off of nu - ||v||^2 exceeds the
    1e-9 allowance: the public path raises NumericalConsistencyError, as the
    reference's _clamp_variances does for such values."""
    z = (np.arange(512, dtype=np.float64) * 3.0).reshape(-1, 1)
    train = gpb.Dataset(z=z, y=np.sin(z[:, 0]))
    model = gpb.GPModel(train, gpb.KernelParams(vertical_scale=1e12, noise_variance=0.0), 4)
    test = gpb.Dataset(z=z, y=np.zeros(512))
    raw = _raw_device_variance(model, test)
    assert raw.min() < -1e-9
    with pytest.raises(NumericalConsistencyError):
        model.predict_variance(test)
