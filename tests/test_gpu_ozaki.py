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
