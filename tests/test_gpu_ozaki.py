"""GPU parity of the tcgen05 digit-plane products (csrc/ozaki.cu).

The long-k products of the prediction sweep (taskgp tiled.py:263-298) run on
the int8 tensor pipe from signed 7-bit digit planes of L and V.  With 8
planes every kept term is exact, so the results must meet the same bars as
the FP64 DMMA path: predictive mean / variance / full covariance <= 1e-9
relative against the CPU oracle (BASELINE.json north_star), and agree with
the DMMA path itself far below that.
"""

import numpy as np
import pytest

import paper_2505_00136_b200 as gpb
from oracle.tiled_gp import OracleGP, rel_fro

pytestmark = pytest.mark.gpu

TOL = 1e-9


def _model(n, m, d, tiles, planes, seed=0, params=(1.0, 1.0, 0.1)):
    train, test = gpb.make_msd_dataset(n, m, d, seed=seed)
    model = gpb.GPModel(train, gpb.KernelParams(*params), tiles_per_dim=tiles)
    model.digit_planes = planes
    return model, train, test


@pytest.mark.parametrize("n,m,d,tiles", [(4096, 1024, 8, 8), (2560, 384, 4, 10), (6144, 1000, 8, 12)])
def test_eight_planes_match_oracle_and_dmma(runtime, n, m, d, tiles):
    model, train, test = _model(n, m, d, tiles, 8)
    assert model.digit_planes == 8
    res = model.predict_with_uncertainty(test)
    assert model.digit_plane_fallbacks() == 0
    ref = OracleGP(train.z, train.y, tiles)
    mean_o, var_o = ref.predict_variance(test.z)
    assert rel_fro(res.mean, mean_o) <= TOL
    assert rel_fro(res.variance, var_o) <= TOL
    model.digit_planes = 0
    dm = model.predict_with_uncertainty(test)
    assert rel_fro(res.mean, dm.mean) <= 1e-12
    assert rel_fro(res.variance, dm.variance) <= 1e-11


def test_products_really_run_on_the_int8_pipe(runtime):
    """The digit-plane launches are counted: more launches than the DMMA sweep
    (one slicing launch per block row), and switching them off restores it."""
    model, train, test = _model(4096, 256, 8, 8, 8)
    model.predict_with_uncertainty(test)
    a = model.launch_count()
    model.predict_with_uncertainty(test)
    with_planes = model.launch_count() - a
    model.digit_planes = 0
    b = model.launch_count()
    model.predict_with_uncertainty(test)
    without = model.launch_count() - b
    assert with_planes > without


def test_full_covariance_with_planes(runtime):
    model, train, test = _model(4096, 256, 8, 8, 8, seed=3)
    fc = model.predict_with_full_cov(test)
    ref = OracleGP(train.z, train.y, 8)
    cov_o = ref.predict_full_cov(test.z)[1]
    model.digit_planes = 0
    fd = model.predict_with_full_cov(test)
    assert rel_fro(fc.full_covariance, fd.full_covariance) <= 1e-11
    assert rel_fro(fc.full_covariance, cov_o) <= TOL


@pytest.mark.parametrize("planes,tol", [(7, 1e-9), (6, 1e-7)])
def test_fewer_planes_degrade_gracefully(runtime, planes, tol):
    model, train, test = _model(4096, 512, 8, 8, planes)
    res = model.predict_with_uncertainty(test)
    model.digit_planes = 0
    dm = model.predict_with_uncertainty(test)
    assert rel_fro(res.mean, dm.mean) <= tol
    assert rel_fro(res.variance, dm.variance) <= tol


def test_bitwise_reproducible(runtime):
    model, train, test = _model(4096, 512, 8, 8, 8)
    a = model.predict_with_uncertainty(test)
    b = model.predict_with_uncertainty(test)
    assert np.array_equal(a.mean, b.mean) and np.array_equal(a.variance, b.variance)


def test_other_kernel_parameters(runtime):
    """Scales follow the hyper-parameters: a large vertical scale and a small noise."""
    model, train, test = _model(4096, 512, 8, 8, 8, params=(0.7, 5.0, 0.02))
    res = model.predict_with_uncertainty(test)
    assert model.digit_plane_fallbacks() == 0
    model.digit_planes = 0
    dm = model.predict_with_uncertainty(test)
    assert rel_fro(res.mean, dm.mean) <= 1e-11
    assert rel_fro(res.variance, dm.variance) <= 1e-10


def test_plane_count_validation(runtime):
    model, _, _ = _model(256, 16, 4, 2, 0)
    with pytest.raises(gpb.errors.InvalidConfig):
        model.digit_planes = 3
    with pytest.raises(gpb.errors.InvalidConfig):
        model.digit_planes = 9


# ---- the factorisation's trailing updates on the int8 pipe ------------------
# taskgp tiled.py:187-204 (SYRK/GEMM updates).  With 512-wide internal tiles a
# group of two panels gives K = 1024, the shortest update that takes the
# digit-plane path; north-star bars: factor <= 1e-10 relative Frobenius, loss
# and gradients <= 1e-9 relative.


def _train_model(n, d, tiles, planes, seed=0, params=(1.0, 1.0, 0.1)):
    train, _ = gpb.make_msd_dataset(n, 0, d, seed=seed)
    model = gpb.GPModel(train, gpb.KernelParams(*params), tiles_per_dim=tiles)
    if planes is not None:
        model.digit_planes = planes
    return model, train


def test_planes_are_the_default(runtime):
    model, _ = _train_model(256, 4, 2, None)
    model.log_likelihood()
    assert model.digit_planes == 8


@pytest.mark.parametrize("n,d,tiles", [(8192, 8, 16), (6144, 4, 12), (8192, 8, 32)])
def test_factor_with_planes_matches_oracle_and_dmma(runtime, n, d, tiles):
    model, train = _train_model(n, d, tiles, 8)
    before = model.launch_count()
    L = model.cholesky()
    with_planes = model.launch_count() - before
    assert model.digit_plane_fallbacks() == 0
    nll = model.compute_loss()
    ref = OracleGP(train.z, train.y, tiles)
    assert rel_fro(L, ref.factor_dense()) <= 1e-10
    assert abs(nll + ref.log_likelihood()) <= 1e-9 * abs(ref.log_likelihood())
    model.digit_planes = 0
    model.params = gpb.KernelParams(1.0, 1.0, 0.1)  # drop the cached factor
    before = model.launch_count()
    Ld = model.cholesky()
    assert model.launch_count() - before < with_planes  # slicing + two window launches per update
    assert rel_fro(L, Ld) <= 1e-11


def test_gradients_and_adam_with_planes(runtime):
    """Config-1 shape: loss gradients and three Adam steps from a digit-plane factor."""
    model, train = _train_model(8192, 8, 32, 8)
    g = np.array(model.loss_gradients())
    hist = model.optimize(gpb.AdamConfig(learning_rate=0.1, iterations=3))
    dm, _ = _train_model(8192, 8, 32, 0)
    gd = np.array(dm.loss_gradients())
    hd = dm.optimize(gpb.AdamConfig(learning_rate=0.1, iterations=3))
    assert np.max(np.abs(g - gd) / np.abs(gd)) <= 1e-9
    assert np.max(np.abs(np.array(hist) - np.array(hd)) / np.abs(np.array(hd))) <= 1e-9
    ref = OracleGP(train.z, train.y, 32)
    go = np.array(ref.loss_gradients())
    assert np.max(np.abs(g - go) / np.abs(go)) <= 1e-9


def test_factor_with_planes_bitwise_reproducible(runtime):
    model, _ = _train_model(8192, 8, 16, 8)
    a = model.cholesky()
    model.params = gpb.KernelParams(1.0, 1.0, 0.1)
    b = model.cholesky()
    assert np.array_equal(a, b)


def test_not_positive_definite_with_planes(runtime):
    """Duplicate inputs and zero noise: the digit-plane factorisation must still
    report NotPositiveDefinite (the DMMA repeat names the pivot)."""
    rng = np.random.default_rng(5)
    z = rng.normal(size=(8192, 4))
    z[5000] = z[100]
    model = gpb.GPModel(gpb.Dataset(z=z, y=rng.normal(size=8192)),
                        gpb.KernelParams(1.0, 1.0, 0.0), tiles_per_dim=16)
    model.digit_planes = 8
    with pytest.raises(gpb.errors.NotPositiveDefinite):
        model.cholesky()
    model.params = gpb.KernelParams(1.0, 1.0, 0.1)
    assert np.isfinite(model.log_likelihood())


def test_other_parameters_factor(runtime):
    model, train = _train_model(8192, 8, 16, 8, params=(0.7, 5.0, 0.02))
    L = model.cholesky()
    assert model.digit_plane_fallbacks() == 0
    ref = OracleGP(train.z, train.y, 16, l=0.7, nu=5.0, s2=0.02)
    model.digit_planes = 0
    model.params = gpb.KernelParams(0.7, 5.0, 0.02)
    Ld = model.cholesky()
    assert rel_fro(L, Ld) <= 1e-10
    assert rel_fro(L, ref.factor_dense()) <= 1e-10


@pytest.mark.parametrize("n,m,d,tiles", [(5000, 333, 5, 10), (4608, 130, 3, 9), (7000, 77, 6, 7)])
def test_ragged_sizes_with_planes(runtime, n, m, d, tiles):
    """User tiles that are no multiple of 128 (padded once at the end with decoupled
    identity rows, |L| = 1 there) and odd test counts: factor, loss, mean, variance and
    full covariance from the digit planes against the oracle."""
    train, test = gpb.make_msd_dataset(n, m, d, seed=11)
    model = gpb.GPModel(train, gpb.KernelParams(0.9, 1.3, 0.07), tiles_per_dim=tiles)
    assert model.digit_planes == 8
    L = model.cholesky()
    nll = model.compute_loss()
    fc = model.predict_with_full_cov(test)
    pv = model.predict_with_uncertainty(test)
    assert model.digit_plane_fallbacks() == 0
    ref = OracleGP(train.z, train.y, tiles, l=0.9, nu=1.3, s2=0.07)
    assert rel_fro(L, ref.factor_dense()) <= 1e-10
    assert abs(nll + ref.log_likelihood()) <= 1e-9 * abs(ref.log_likelihood())
    mean_o, cov_o = ref.predict_full_cov(test.z)
    _, var_o = ref.predict_variance(test.z)
    assert rel_fro(fc.mean, mean_o) <= TOL and rel_fro(fc.full_covariance, cov_o) <= TOL
    assert rel_fro(pv.variance, var_o) <= TOL
    assert np.array_equal(fc.full_covariance, fc.full_covariance.T)


def test_toggling_planes_keeps_results_within_contract(runtime):
    """digit_planes can be switched on a live model: a changed panel grouping drops the
    cached factor, and both settings meet the oracle bars."""
    model, train = _train_model(24576, 8, 48, 8)  # 48 internal tiles: 8-panel groups with planes, 4 without
    a = model.compute_loss()
    model.digit_planes = 0
    b = model.compute_loss()
    model.digit_planes = 8
    c = model.compute_loss()
    assert a == c  # bitwise reproducible after the round trip
    assert abs(a - b) <= 1e-10 * abs(b)


def test_planes_are_optional_when_memory_is_short(runtime, monkeypatch):
    """The plane buffers are an optimisation: when they cannot be allocated the
    same calls run on the FP64 DMMA kernels (bitwise the digit_planes = 0 results)."""
    train, test = gpb.make_msd_dataset(4096, 300, 6, seed=2)
    monkeypatch.setenv("GPB_PLANES_ALLOC_FAIL", "1")
    a = gpb.GPModel(train, gpb.KernelParams(1.0, 1.0, 0.1), tiles_per_dim=8)
    assert a.digit_planes == 8
    ra = a.predict_with_full_cov(test)
    la = a.compute_loss()
    monkeypatch.delenv("GPB_PLANES_ALLOC_FAIL")
    b = gpb.GPModel(train, gpb.KernelParams(1.0, 1.0, 0.1), tiles_per_dim=8)
    b.digit_planes = 0
    rb = b.predict_with_full_cov(test)
    assert la == b.compute_loss()
    assert np.array_equal(ra.mean, rb.mean) and np.array_equal(ra.full_covariance, rb.full_covariance)


def test_gradient_planes_across_k_segments(runtime):
    """n = 36864 (72 tiles of 512): the K^-1 = X^T X products are deeper than one int32-exact
    segment (32768), so the first columns run in two k segments; against the FP64 DMMA path."""
    model, _ = _train_model(36864, 8, 72, 8)
    g = np.array(model.loss_gradients())
    assert model.digit_plane_fallbacks() == 0
    model.digit_planes = 0
    gd = np.array(model.loss_gradients())
    assert np.max(np.abs(g - gd) / np.abs(gd)) <= 1e-10


def test_gradient_with_tiny_noise_keeps_fp64(runtime):
    """noise below 1e-6: no useful bound on L^-1, the K^-1 product stays on the FP64 kernels
    (same launches as with the planes off)."""
    train, _ = gpb.make_msd_dataset(4096, 0, 6, seed=4)
    a = gpb.GPModel(train, gpb.KernelParams(1.0, 1.0, 1e-7), tiles_per_dim=8)
    b = gpb.GPModel(train, gpb.KernelParams(1.0, 1.0, 1e-7), tiles_per_dim=8)
    b.digit_planes = 0
    ga, gb = np.array(a.loss_gradients()), np.array(b.loss_gradients())
    assert np.max(np.abs(ga - gb) / np.abs(gb)) <= 1e-7  # conditioning 1e7: the factors differ at 1e-13
