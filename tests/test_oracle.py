"""Pin the CPU oracle against the reference's own outputs (tests/golden/*.npz).

The fixtures were produced by running the reference ``taskgp`` GPModel in
the build container (tests/golden/make_golden.py).  The oracle restates the
same tile algorithm with the same numpy operations in the same order, so
agreement is expected to the last bit; the asserted bound is 1e-13 relative.
"""

import numpy as np
import pytest

from conftest import load_golden
from oracle.tiled_gp import OracleGP, dense_k, rel_fro, tiled_cholesky, assemble_covariance, to_dense_lower
from paper_2505_00136_b200.data import make_msd_dataset


@pytest.fixture(autouse=True)
def _one_blas_thread():
    """The reference pins BLAS to one thread per worker (runtime.py:180-181);
    doing the same makes every dgemm reduce in the reference's order."""
    from threadpoolctl import threadpool_limits

    with threadpool_limits(1):
        yield

RAND = ["rand_n16_m16_t4", "rand_n64_m16_t4", "rand_n64_m64_t8", "rand_n256_m64_t4",
        "rand_n48_m12_t4", "rand_n16_m7_t4"]


@pytest.mark.parametrize("name", RAND)
def test_oracle_matches_reference_small(name):
    g = load_golden(name)
    t = int(g["t"])
    o = OracleGP(g["z"], g["y"], t)
    assert np.array_equal(o.factor_dense(), g["L"]) or rel_fro(o.factor_dense(), g["L"]) < 1e-13
    assert o.log_likelihood() == pytest.approx(float(g["loglik"]), rel=1e-13)
    mean, var = o.predict_variance(g["zt"])
    np.testing.assert_allclose(mean, g["mean"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(var, g["var"], rtol=1e-12, atol=1e-14)
    if "cov" in g:
        _, cov = o.predict_full_cov(g["zt"])
        np.testing.assert_allclose(cov, g["cov"], rtol=1e-12, atol=1e-14)
    if "grads" in g:
        np.testing.assert_allclose(o.loss_gradients(), g["grads"], rtol=1e-12, atol=1e-15)
    if "adam_history" in g:
        hist = o.optimize(lr=0.1, iterations=len(g["adam_history"]))
        np.testing.assert_allclose(hist, g["adam_history"], rtol=1e-12)
        np.testing.assert_allclose([o.l, o.nu, o.s2], g["adam_params"], rtol=1e-12)


def _check_summary(prefix, a, g, rtol):
    np.testing.assert_allclose(np.diagonal(a), g[prefix + "_diag"], rtol=rtol, atol=1e-15)
    np.testing.assert_allclose(a.sum(axis=0), g[prefix + "_colsum"], rtol=rtol, atol=1e-12)
    np.testing.assert_allclose(a[g[prefix + "_sr"], g[prefix + "_sc"]], g[prefix + "_sv"],
                               rtol=rtol, atol=1e-15)
    assert float(np.linalg.norm(a)) == pytest.approx(float(g[prefix + "_fro"]), rel=rtol)


@pytest.mark.parametrize("name,n,m,d,seed", [("c0", 1024, 1024, 8, 0), ("c2s", 2048, 512, 128, 0),
                                             ("d8b512", 4096, 512, 8, 1)])
def test_oracle_matches_reference_configs(name, n, m, d, seed):
    g = load_golden(name)
    train, test = make_msd_dataset(n, m, d, seed=seed)
    # the BASELINE generator is pinned by the reference-run fixture too
    np.testing.assert_array_equal(train.z[:16], g["z_head"])
    np.testing.assert_array_equal(train.y[:16], g["y_head"])
    np.testing.assert_array_equal(test.z[:16], g["zt_head"])
    o = OracleGP(train.z, train.y, int(g["t"]))
    _check_summary("L", o.factor_dense(), g, 1e-12)
    assert o.log_likelihood() == pytest.approx(float(g["loglik"]), rel=1e-13)
    mean, var = o.predict_variance(test.z)
    np.testing.assert_allclose(mean, g["mean"], rtol=1e-11, atol=1e-14)
    np.testing.assert_allclose(var, g["var"], rtol=1e-11, atol=1e-14)
    if "grads" in g:
        np.testing.assert_allclose(o.loss_gradients(), g["grads"], rtol=1e-11)


def test_oracle_c1_loglik():
    g = load_golden("c1")
    train, _ = make_msd_dataset(8192, 0, 8, seed=0)
    np.testing.assert_array_equal(train.z[:16], g["z_head"])
    o = OracleGP(train.z, train.y, 32)
    assert o.log_likelihood() == pytest.approx(float(g["loglik"]), rel=1e-12)


def test_oracle_tiling_invariance_and_dense_check(rng):
    """covariance.py's exact tiling invariance and a dense Cholesky cross-check."""
    z = rng.normal(size=(64, 3))
    dense = [to_dense_lower(assemble_covariance(z, 1.0, 1.0, 0.1, t), t, True) for t in (1, 2, 4, 8)]
    for a in dense[1:]:
        np.testing.assert_array_equal(a, dense[0])
    L = to_dense_lower(tiled_cholesky(assemble_covariance(z, 1.0, 1.0, 0.1, 4), 4), 4, False)
    np.testing.assert_allclose(L, np.linalg.cholesky(dense_k(z, 1.0, 1.0, 0.1)), atol=1e-12)


def test_oracle_known_answers():
    """Reference known answers (test_model.py:176-190)."""
    o = OracleGP(np.zeros((1, 1)), np.zeros(1), 1, nu=0.5, s2=0.5)
    assert o.log_likelihood() == pytest.approx(-0.9189385332046727, abs=1e-15)
    o = OracleGP(np.zeros((1, 1)), np.ones(1), 1, nu=0.5, s2=0.5)
    assert o.log_likelihood() == pytest.approx(-1.4189385332046727, abs=1e-15)


def acceptance_instance(seed, n, m, d=4):
    """pkg/tests/test_acceptance.py:28-32 inputs."""
    r = np.random.default_rng(seed)
    return r.normal(size=(n, d)), r.normal(size=n), r.normal(size=(m, d))


@pytest.mark.parametrize("n", [16, 64, 256])
@pytest.mark.parametrize("m", [16, 64])
def test_oracle_matches_reference_acceptance_grid(n, m):
    """The reference's oracle-equivalence grid (test_acceptance.py:35-78): the
    oracle reproduces taskgp's outputs for every tiling, and those agree with
    the reference's dense checker within the reference test's 1e-8."""
    g = load_golden("accept_grid")
    key = f"n{n}_m{m}"
    z, y, zt = acceptance_instance(n * 1000 + m, n, m)
    np.testing.assert_array_equal([z.sum(), y.sum(), zt.sum()], g[key + "_zsum"])
    for t in (1, 4, 8):
        k = f"{key}_t{t}"
        o = OracleGP(z, y, t)
        assert rel_fro(o.factor_dense(), g[k + "_L"]) < 1e-13
        mean, var = o.predict_variance(zt)
        _, cov = o.predict_full_cov(zt)
        np.testing.assert_allclose(mean, g[k + "_mean"], rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(var, g[k + "_var"], rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(cov, g[k + "_cov"], rtol=1e-12, atol=1e-14)
        assert o.log_likelihood() == pytest.approx(float(g[k + "_ll"]), rel=1e-13)
        np.testing.assert_allclose(o.loss_gradients(), g[k + "_grads"], rtol=1e-11, atol=1e-15)
        worst = max(np.abs(g[k + "_L"] - g[key + "_dense_L"]).max(),
                    np.abs(g[k + "_mean"] - g[key + "_dense_mean"]).max(),
                    np.abs(g[k + "_cov"] - g[key + "_dense_cov"]).max(),
                    abs(float(g[k + "_ll"]) - float(g[key + "_dense_ll"])))
        assert worst <= 1e-8


@pytest.mark.parametrize("name,m,d", [("c3s", 0, 8), ("c4s", 512, 16)])
def test_oracle_matches_reference_scaled_large(name, m, d):
    """Scaled config-3 / config-4 shapes (b = 512, T = 16) run by the reference."""
    g = load_golden(name)
    train, test = make_msd_dataset(8192, m, d, seed=0)
    np.testing.assert_array_equal(train.z[:16], g["z_head"])
    o = OracleGP(train.z, train.y, 16)
    _check_summary("L", o.factor_dense(), g, 1e-12)
    assert o.log_likelihood() == pytest.approx(float(g["loglik"]), rel=1e-13)
    if m:
        np.testing.assert_array_equal(test.z[:16], g["zt_head"])
        mean, var = o.predict_variance(test.z)
        np.testing.assert_allclose(mean, g["mean"], rtol=1e-11, atol=1e-14)
        np.testing.assert_allclose(var, g["var"], rtol=1e-11, atol=1e-14)


def test_oracle_clamp_matches_reference():
    """_clamp_variances known answers (test_model.py:165-172)."""
    from oracle.tiled_gp import clamp_variances

    np.testing.assert_array_equal(clamp_variances(np.array([1.0, -1e-10, 0.0])), [1.0, 0.0, 0.0])
    with pytest.raises(ArithmeticError):
        clamp_variances(np.array([0.5, -1e-6]))
