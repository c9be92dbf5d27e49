"""GPU parity: the sm_100a path (through the C ABI) against the reference.

Tolerances (BASELINE.json north_star): Cholesky factor <= 1e-10 relative
Frobenius; loss, gradients, predictive mean and variance <= 1e-9 relative
(norm-wise).  References are the golden
fixtures produced by the reference implementation (tests/golden) and the
CPU oracle (oracle/tiled_gp.py) on the same seeded inputs.
"""

import numpy as np
import pytest

import paper_2505_00136_b200 as gpb
from conftest import load_golden
from oracle.tiled_gp import OracleGP, dense_k, rel_fro
from paper_2505_00136_b200.errors import (
    DimensionMismatch,
    NotPositiveDefinite,
    NotRunning,
)

pytestmark = pytest.mark.gpu

L_TOL = 1e-10
TOL = 1e-9


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den else 1.0))


def ds(z, y=None):
    z = np.asarray(z, dtype=np.float64)
    return gpb.Dataset(z=z, y=np.zeros(z.shape[0]) if y is None else y)


RAND = ["rand_n16_m16_t4", "rand_n64_m16_t4", "rand_n64_m64_t8", "rand_n256_m64_t4",
        "rand_n48_m12_t4", "rand_n16_m7_t4"]


@pytest.mark.parametrize("name", RAND)
def test_reference_corpus_instances(runtime, name):
    """Reference-run fixtures of the test-suite shapes (test_acceptance.py:35-78)."""
    g = load_golden(name)
    model = gpb.GPModel(ds(g["z"], g["y"]), gpb.KernelParams(1.0, 1.0, 0.1), int(g["t"]))
    assert rel(model.cholesky(), g["L"]) <= L_TOL
    assert abs(model.log_likelihood() - g["loglik"]) <= TOL * abs(g["loglik"])
    pv = model.predict_with_uncertainty(ds(g["zt"]))
    assert rel(pv.mean, g["mean"]) <= TOL
    assert rel(pv.variance, g["var"]) <= TOL
    fc = model.predict_with_full_cov(ds(g["zt"]))
    assert rel(fc.full_covariance, g["cov"]) <= TOL
    assert rel(model.loss_gradients(), g["grads"]) <= TOL
    if "adam_history" in g:
        hist = model.optimize(gpb.AdamConfig(learning_rate=0.1, iterations=len(g["adam_history"])))
        assert rel(hist, g["adam_history"]) <= TOL
        p = model.params
        assert rel([p.lengthscale, p.vertical_scale, p.noise_variance], g["adam_params"]) <= TOL


def _check_summary(prefix, a, g, tol):
    scale = float(g[prefix + "_fro"])
    assert abs(np.linalg.norm(a) - scale) <= tol * scale
    assert rel(np.diagonal(a), g[prefix + "_diag"]) <= tol
    assert rel(a.sum(axis=0), g[prefix + "_colsum"]) <= tol
    assert rel(a[g[prefix + "_sr"], g[prefix + "_sc"]], g[prefix + "_sv"]) <= tol


@pytest.mark.parametrize("name,n,m,d,seed", [("c0", 1024, 1024, 8, 0), ("c2s", 2048, 512, 128, 0),
                                             ("d8b512", 4096, 512, 8, 1)])
def test_baseline_configs(runtime, name, n, m, d, seed):
    """BASELINE config 0 (and scaled config 2 shapes) against the reference run."""
    g = load_golden(name)
    train, test = gpb.make_msd_dataset(n, m, d, seed=seed)
    model = gpb.GPModel(train, gpb.KernelParams(1.0, 1.0, 0.1), int(g["t"]))
    _check_summary("L", model.cholesky(), g, L_TOL)
    assert abs(model.compute_loss() + g["loglik"]) <= TOL * abs(g["loglik"])
    pv = model.predict_with_uncertainty(test)
    assert rel(pv.mean, g["mean"]) <= TOL
    assert rel(pv.variance, g["var"]) <= TOL
    if "cov_fro" in g:
        _check_summary("cov", model.predict_with_full_cov(test).full_covariance, g, TOL)
    if "grads" in g:
        assert rel(model.loss_gradients(), g["grads"]) <= TOL


def test_config1_training(runtime):
    """BASELINE config 1: compute_loss + 3 Adam iterations (reference-run fixture)."""
    g = load_golden("c1")
    train, _ = gpb.make_msd_dataset(8192, 0, 8, seed=0)
    model = gpb.GPModel(train, gpb.KernelParams(1.0, 1.0, 0.1), 32)
    assert abs(model.compute_loss() + g["loglik"]) <= TOL * abs(g["loglik"])
    assert rel(model.loss_gradients(), g["grads"]) <= TOL
    hist = model.optimize(gpb.AdamConfig(learning_rate=0.1, iterations=3))
    assert rel(hist, g["adam_history"]) <= TOL
    p = model.params
    assert rel([p.lengthscale, p.vertical_scale, p.noise_variance], g["adam_params"]) <= TOL


@pytest.mark.parametrize("n,m,t,d", [(200, 37, 4, 3), (1000, 130, 8, 5), (768, 300, 3, 2),
                                     (130, 1, 1, 1), (1, 3, 1, 2), (640, 96, 5, 16)])
def test_ragged_tiles_against_oracle(runtime, n, m, t, d):
    """Tile sizes that are not multiples of the kernel block (padding path)."""
    rng = np.random.default_rng(n * 7 + m)
    z, y, zt = rng.normal(size=(n, d)), rng.normal(size=n), rng.normal(size=(m, d))
    model = gpb.GPModel(ds(z, y), gpb.KernelParams(1.3, 0.8, 0.2), t)
    o = OracleGP(z, y, t, 1.3, 0.8, 0.2)
    assert rel(model.cholesky(), o.factor_dense()) <= L_TOL
    assert abs(model.log_likelihood() - o.log_likelihood()) <= TOL * abs(o.log_likelihood())
    mean, var = o.predict_variance(zt)
    pv = model.predict_variance(ds(zt))
    assert rel(pv.mean, mean) <= TOL
    assert rel(pv.variance, var) <= TOL
    _, cov = o.predict_full_cov(zt)
    assert rel(model.predict_with_full_cov(ds(zt)).full_covariance, cov) <= TOL
    assert rel(model.loss_gradients(), o.loss_gradients()) <= TOL


def test_prediction_chunking(runtime, monkeypatch):
    """Test points beyond the device-memory budget are processed in chunks;
    every column's arithmetic is unchanged, so results are bitwise equal."""
    from paper_2505_00136_b200.errors import DeviceError

    rng = np.random.default_rng(77)
    z, y, zt = rng.normal(size=(600, 3)), rng.normal(size=600), rng.normal(size=(700, 3))
    model = gpb.GPModel(ds(z, y), tiles_per_dim=3)
    ref = model.predict_variance(ds(zt))
    monkeypatch.setenv("GPB_PRED_CHUNK", "128")
    got = model.predict_variance(ds(zt))
    assert np.array_equal(got.mean, ref.mean) and np.array_equal(got.variance, ref.variance)
    with pytest.raises(DeviceError, match="full posterior covariance"):
        model.predict_with_full_cov(ds(zt))


def test_determinism_bitwise(runtime):
    """Fixed reduction orders: repeated runs are bitwise identical
    (the reference's determinism check, test_tiled.py:99-111)."""
    train, test = gpb.make_msd_dataset(2048, 512, 8, seed=3)
    outs = []
    for _ in range(2):
        model = gpb.GPModel(train, gpb.KernelParams(), 4)
        pv = model.predict_variance(test)
        outs.append((model.cholesky(), pv.mean, pv.variance, model.log_likelihood(),
                     model.loss_gradients()))
    for a, b in zip(*outs):
        assert np.array_equal(np.asarray(a), np.asarray(b))


def test_tiling_invariance(runtime, rng):
    """test_acceptance.py:135-169 / test_gradients.py:65-75 on the GPU path."""
    z, y, zt = rng.normal(size=(512, 3)), rng.normal(size=512), rng.normal(size=(64, 3))
    res = []
    for t in (1, 2, 4, 8):
        model = gpb.GPModel(ds(z, y), tiles_per_dim=t)
        pv = model.predict_variance(ds(zt))
        res.append((pv.mean, pv.variance, model.log_likelihood(), model.loss_gradients()))
    for r in res[1:]:
        for a, b in zip(r, res[0]):
            np.testing.assert_allclose(a, b, rtol=1e-10, atol=1e-10)


class TestModelBehaviour:
    """Reference test_model.py behaviours on the GPU path."""

    def test_known_answers(self, runtime):
        kp = gpb.KernelParams(vertical_scale=0.5, noise_variance=0.5)
        m0 = gpb.GPModel(gpb.Dataset(z=np.zeros((1, 1)), y=np.zeros(1)), kp)
        assert m0.log_likelihood() == pytest.approx(-0.9189385332046727, abs=1e-15)
        m1 = gpb.GPModel(gpb.Dataset(z=np.zeros((1, 1)), y=np.ones(1)), kp)
        assert m1.log_likelihood() == pytest.approx(-1.4189385332046727, abs=1e-15)

    def test_zero_observations_give_zero_mean(self, runtime, rng):
        train = gpb.Dataset(z=rng.normal(size=(16, 2)), y=np.zeros(16))
        result = gpb.GPModel(train, tiles_per_dim=4).predict(ds(rng.normal(size=(4, 2))))
        np.testing.assert_array_equal(result.mean, np.zeros(4))
        assert result.variance is None and result.full_covariance is None

    def test_interpolates_noise_free_data(self, runtime):
        z = np.arange(8.0).reshape(-1, 1) * 3.0
        model = gpb.GPModel(gpb.Dataset(z=z, y=np.sin(z[:, 0])), gpb.KernelParams(noise_variance=0.0))
        assert model.predict(ds(z[2:3])).mean[0] == pytest.approx(np.sin(6.0), abs=1e-8)

    def test_dense_oracle(self, runtime, rng):
        z, y, zt = rng.normal(size=(64, 3)), rng.normal(size=64), rng.normal(size=(32, 3))
        k = dense_k(z, 1.0, 1.0, 0.1)
        ks = np.exp(-((zt[:, None] - z[None]) ** 2).sum(-1) / 2)
        model = gpb.GPModel(ds(z, y), tiles_per_dim=4)
        np.testing.assert_allclose(model.predict(ds(zt)).mean, ks @ np.linalg.solve(k, y), atol=1e-8)

    def test_feature_mismatch(self, runtime, rng):
        model = gpb.GPModel(gpb.Dataset(z=rng.normal(size=(8, 2)), y=np.zeros(8)))
        with pytest.raises(DimensionMismatch):
            model.predict(ds(rng.normal(size=(4, 3))))

    def test_not_pd_then_recovers(self, runtime):
        """test_model.py:89-94 and :233-243: failure raises and clears the cache."""
        z = np.ones((4, 2))
        model = gpb.GPModel(gpb.Dataset(z=z, y=np.ones(4)), gpb.KernelParams(noise_variance=0.0))
        with pytest.raises(NotPositiveDefinite):
            model.log_likelihood()
        with pytest.raises(NotPositiveDefinite):
            model.predict(ds(z[:1]))
        model.params = gpb.KernelParams(noise_variance=0.5)
        assert np.isfinite(model.log_likelihood())

    def test_full_cov_symmetric_and_matches_variance(self, runtime, rng):
        z, y, zt = rng.normal(size=(48, 3)), rng.normal(size=48), rng.normal(size=(12, 3))
        model = gpb.GPModel(ds(z, y), tiles_per_dim=4)
        full = model.predict_with_full_cov(ds(zt))
        var = model.predict_variance(ds(zt))
        np.testing.assert_array_equal(full.full_covariance, full.full_covariance.T)
        np.testing.assert_allclose(var.variance, np.diag(full.full_covariance), atol=1e-12)
        np.testing.assert_array_equal(var.mean, full.mean)

    def test_far_points_recover_prior(self, runtime, rng):
        train = gpb.Dataset(z=rng.normal(size=(8, 1)), y=rng.normal(size=8))
        test = ds(200.0 + rng.normal(size=(3, 1)))
        result = gpb.GPModel(train, gpb.KernelParams(vertical_scale=1.7)).predict_with_full_cov(test)
        prior = 1.7 * np.exp(-((test.z[:, None] - test.z[None]) ** 2).sum(-1) / 2)
        np.testing.assert_allclose(result.full_covariance, prior, atol=1e-12)
        v = gpb.GPModel(train, gpb.KernelParams(vertical_scale=2.5)).predict_variance(ds([[500.0]]))
        assert v.variance[0] == pytest.approx(2.5, abs=1e-12)

    def test_cache_invalidation(self, runtime, rng):
        z, y, zt = rng.normal(size=(16, 3)), rng.normal(size=16), rng.normal(size=(4, 3))
        model = gpb.GPModel(ds(z, y), tiles_per_dim=2)
        first = model.predict(ds(zt)).mean
        model.params = gpb.KernelParams(lengthscale=0.3)
        assert not np.array_equal(first, model.predict(ds(zt)).mean)
        second = model.predict(ds(zt)).mean
        model.train = gpb.Dataset(z=z, y=y + 1.0)
        assert not np.array_equal(second, model.predict(ds(zt)).mean)

    def test_runtime_lifecycle(self, runtime, rng):
        from paper_2505_00136_b200.errors import AlreadyRunning

        with pytest.raises(AlreadyRunning):
            gpb.start_runtime()
        model = gpb.GPModel(gpb.Dataset(z=rng.normal(size=(8, 2)), y=np.zeros(8)))
        model.log_likelihood()
        runtime.stop()
        with pytest.raises(NotRunning):
            model.log_likelihood()
        rt2 = gpb.start_runtime()
        try:
            assert np.isfinite(model.log_likelihood())  # rebinds to the new runtime
        finally:
            rt2.stop()


class TestGradientsAndAdam:
    @staticmethod
    def fd(model, h=1e-5):
        from dataclasses import replace

        base, g = model.params, np.empty(3)
        for i, name in enumerate(("lengthscale", "vertical_scale", "noise_variance")):
            theta = getattr(base, name)
            model.params = replace(base, **{name: float(np.exp(np.log(theta) + h))})
            hi = -model.log_likelihood()
            model.params = replace(base, **{name: float(np.exp(np.log(theta) - h))})
            lo = -model.log_likelihood()
            g[i] = (hi - lo) / (2 * h) / theta
        model.params = base
        return g

    @pytest.mark.parametrize("seed", range(3))
    def test_finite_differences(self, runtime, seed):
        rng = np.random.default_rng(seed)
        model = gpb.GPModel(ds(rng.normal(size=(32, 3)), rng.normal(size=32)),
                            gpb.KernelParams(*rng.uniform([0.5, 0.5, 0.05], [2.0, 2.0, 0.5])), 4)
        analytic = np.array(model.loss_gradients())
        numeric = self.fd(model)
        assert np.max(np.abs(analytic - numeric) / np.maximum(np.abs(numeric), 1e-12)) < 1e-5

    def test_flags(self, runtime, rng):
        train = ds(rng.normal(size=(16, 3)), rng.normal(size=16))
        assert gpb.GPModel(train, gpb.KernelParams(trainable=(False,) * 3)).loss_gradients() == (0.0, 0.0, 0.0)
        g = gpb.GPModel(train, gpb.KernelParams(trainable=(True, False, False)), 2).loss_gradients()
        assert g[0] != 0.0 and g[1] == 0.0 and g[2] == 0.0

    def test_noise_gradient_identity(self, runtime, rng):
        z, y = rng.normal(size=(24, 3)), rng.normal(size=24)
        k = dense_k(z, 1.0, 1.0, 0.1)
        alpha = np.linalg.solve(k, y)
        expected = 0.5 * (np.trace(np.linalg.inv(k)) - alpha @ alpha)
        assert gpb.GPModel(ds(z, y), tiles_per_dim=4).loss_gradients()[2] == pytest.approx(expected, rel=1e-9)

    @pytest.mark.parametrize("n,t,world", [(600, 6, 2), (1024, 4, 3), (2048, 4, 1)])
    def test_column_panel_terms(self, runtime, n, t, world):
        """gpb_loss_gradient_terms (the multi-GPU split of the gradient):
        summed over every rank's tile columns it reproduces loss_gradients and the oracle."""
        import ctypes

        from paper_2505_00136_b200 import _lib

        def gradient_columns(tiles, world):  # snake-order split of the tile columns
            out = [[] for _ in range(world)]
            for j in range(tiles):
                r, lap = j % world, (j // world) % 2
                out[world - 1 - r if lap else r].append(j)
            return out

        rng = np.random.default_rng(n + t)
        z, y = rng.normal(size=(n, 3)), rng.normal(size=n)
        model = gpb.GPModel(ds(z, y), gpb.KernelParams(1.2, 0.9, 0.15), t)
        whole = np.array(model.loss_gradients())
        lay = _lib.layout(n, t)
        lib, tot = _lib.load(), np.zeros(3)
        for cols in gradient_columns(lay["T"], world):
            if cols:
                out = (ctypes.c_double * 3)()
                arr = (ctypes.c_int * len(cols))(*cols)
                _lib.check(lib.gpb_loss_gradient_terms(model._handle, arr, len(cols), out))
                tot += np.array(out[:3])
        p = model.params
        alpha = np.linalg.solve(dense_k(z, 1.2, 0.9, 0.15), y)
        split = np.array([0.5 * p.vertical_scale / p.lengthscale ** 3 * tot[0], 0.5 * tot[1],
                          0.5 * (tot[2] - alpha @ alpha)])
        assert rel(split, whole) <= 1e-11
        assert rel(split, OracleGP(z, y, t, 1.2, 0.9, 0.15).loss_gradients()) <= TOL
        with pytest.raises(gpb.errors.InvalidConfig):
            bad = (ctypes.c_int * 2)(1, 0)  # not increasing
            _lib.check(lib.gpb_loss_gradient_terms(model._handle, bad, 2, (ctypes.c_double * 3)()))

    def test_adam_semantics(self, runtime, rng):
        train = ds(rng.normal(size=(16, 3)), rng.normal(size=16))
        kp = gpb.KernelParams()
        model = gpb.GPModel(train, kp, 2)
        before = np.log([kp.lengthscale, kp.vertical_scale, kp.noise_variance])
        model.optimize(gpb.AdamConfig(learning_rate=0.05, iterations=1))
        p = model.params
        d = np.abs(np.log([p.lengthscale, p.vertical_scale, p.noise_variance]) - before)
        assert np.all(d >= 0.99 * 0.05) and np.all(d <= 0.05 + 1e-12)
        split = gpb.GPModel(train, kp, 2)
        split.optimize(gpb.AdamConfig(iterations=1))
        split.optimize(gpb.AdamConfig(iterations=1))
        joint = gpb.GPModel(train, kp, 2)
        joint.optimize(gpb.AdamConfig(iterations=2))
        assert split.params.lengthscale == pytest.approx(joint.params.lengthscale, rel=1e-12)
        fixed = gpb.GPModel(train, gpb.KernelParams(1.5, 1.0, 0.3, (False, True, False)), 2)
        fixed.optimize(gpb.AdamConfig(iterations=3))
        assert fixed.params.lengthscale == 1.5 and fixed.params.noise_variance == 0.3

    def test_adam_state_survives_rebind(self, runtime, rng):
        """Moments and step count persist across close() and a runtime restart
        (model.py:446-448): optimize(1) + close() + optimize(1) == optimize(2)."""
        train = ds(rng.normal(size=(32, 3)), rng.normal(size=32))
        joint = gpb.GPModel(train, gpb.KernelParams(), 4)
        h_joint = joint.optimize(gpb.AdamConfig(iterations=2))
        split = gpb.GPModel(train, gpb.KernelParams(), 4)
        h1 = split.optimize(gpb.AdamConfig(iterations=1))
        split.close()
        runtime.stop()
        rt2 = gpb.start_runtime()
        try:
            h2 = split.optimize(gpb.AdamConfig(iterations=1))
        finally:
            rt2.stop()
        assert h1 + h2 == h_joint
        assert split.params == joint.params

    def test_failure_reports_iteration(self, runtime):
        kp = gpb.KernelParams(noise_variance=0.0, trainable=(False, False, False))
        model = gpb.GPModel(gpb.Dataset(z=np.ones((4, 2)), y=np.ones(4)), kp)
        with pytest.raises(NotPositiveDefinite, match="iteration 1"):
            model.optimize(gpb.AdamConfig(iterations=3))


class TestTilePlugin:
    """tiles.py:132-164 contract on the GPU tile kernels (test_tiles.py answers)."""

    def test_potrf(self, runtime):
        out = gpb.B200TileKernels.potrf(np.array([[4.0, 2.0], [2.0, 3.0]]))
        np.testing.assert_allclose(out, [[2.0, 0.0], [1.0, np.sqrt(2.0)]], atol=1e-15)
        with pytest.raises(NotPositiveDefinite):
            gpb.B200TileKernels.potrf(np.array([[1.0, 2.0], [2.0, 1.0]]))
        a = np.random.default_rng(0).normal(size=(300, 300))
        a = a @ a.T + 300 * np.eye(300)
        assert rel(gpb.B200TileKernels.potrf(a), np.linalg.cholesky(a)) <= 1e-13

    @pytest.mark.parametrize("b,k", [(256, 5), (256, 40), (512, 33), (512, 300), (512, 511)])
    def test_potrf_failure_deep_in_the_tile(self, runtime, b, k):
        """A non-positive pivot in any panel of the tile kernel -- including the
        panels the chain factors ahead, inside the previous panel's barrier
        window -- raises NotPositiveDefinite naming that pivot, like LAPACK's
        info (tiles.py:29-33)."""
        rng = np.random.default_rng(k)
        x = rng.normal(size=(b, b)) / np.sqrt(b)
        a = x @ x.T + np.eye(b)
        a[k, :] = a[:, k] = 0.0
        a[k, k] = -1.0
        with pytest.raises(NotPositiveDefinite, match=f"index {k}\\b"):
            gpb.B200TileKernels.potrf(a)
        a[k, k] = 2.0  # now positive definite again
        assert rel(gpb.B200TileKernels.potrf(a), np.linalg.cholesky(a)) <= 1e-13

    def test_trsm_syrk_gemm(self, runtime):
        rng = np.random.default_rng(1)
        a = rng.normal(size=(200, 200))
        l = np.linalg.cholesky(a @ a.T + 200 * np.eye(200))
        b = rng.normal(size=(150, 200))
        x = gpb.B200TileKernels.trsm(l, b)
        assert rel(x @ l.T, b) <= 1e-13
        c = rng.normal(size=(200, 200))
        assert rel(gpb.B200TileKernels.syrk(a, c), c - a @ a.T) <= 1e-13
        bb = rng.normal(size=(170, 200))
        c2 = rng.normal(size=(200, 170))
        assert rel(gpb.B200TileKernels.gemm(a, bb, c2), c2 - a @ bb.T) <= 1e-13
        np.testing.assert_allclose(
            gpb.B200TileKernels.trsm(np.array([[2.0, 0.0], [1.0, 1.0]]), np.array([[4.0, 3.0]])),
            [[2.0, 1.0]], atol=1e-15)


_GEMM_PATH_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[2])
import paper_2505_00136_b200 as gpb
train, test = gpb.make_msd_dataset(4096, 1024, 8, seed=5)
rt = gpb.start_runtime()
model = gpb.GPModel(train, gpb.KernelParams(), 8)
L = model.cholesky()
pv = model.predict_variance(test)
np.savez(sys.argv[1], L=L, mean=pv.mean, var=pv.variance, grads=np.array(model.loss_gradients()))
rt.stop()
"""


def test_tma_gemm_matches_cpasync_gemm(tmp_path):
    """The TMA-fed GEMM (gemm_tma.cu) consumes k in the order of the paired
    cp.async kernel (gemm.cu): the factorisation (K-major x K-major products
    only) is bitwise identical between the two, and prediction / gradients
    agree to round-off.  GPB_GEMM_TMA=0 forces the cp.async kernel."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for mode in ("3", "0"):
        path = str(tmp_path / f"m{mode}.npz")
        env = dict(os.environ, GPB_GEMM_TMA=mode, GPB_GEMM_CFG="99")
        subprocess.run([sys.executable, "-c", _GEMM_PATH_SCRIPT, path, root], env=env, check=True,
                       timeout=600)
        out[mode] = np.load(path)
    a, b = out["3"], out["0"]
    assert np.array_equal(a["L"], b["L"])
    assert rel(a["mean"], b["mean"]) <= 1e-12
    assert rel(a["var"], b["var"]) <= 1e-12
    assert rel(a["grads"], b["grads"]) <= 1e-12


def test_device_gemm_views_and_fallback(runtime, rng):
    """gpb_dev_gemm_tiled (the multi-GPU schedule's GEMM) builds TMA views from
    the job pointers when every job's block sits inside one row of an
    ld-wide view of one buffer, and falls back to the cp.async kernel when the
    operands come from unrelated allocations at arbitrary offsets; both must
    give C - A B^T (K-major x K-major, tiled-k walk over two panel tiles)."""
    import ctypes

    import torch

    from paper_2505_00136_b200 import _lib

    def gemm(jobs, b, alpha, beta):  # (a, b, cin, cout, k, lower); a / b are (2, b, b) panel stacks
        arr = (_lib.GemmJob * len(jobs))(*[_lib.GemmJob(a.data_ptr(), bb.data_ptr(), ci.data_ptr(), co.data_ptr(),
                                                        k, int(lo)) for a, bb, ci, co, k, lo in jobs])
        stride = jobs[0][0].stride(0)
        _lib.check(_lib.load().gpb_dev_gemm_tiled(runtime.handle, None, arr, len(jobs), b, b, b, b, 1, 1, b,
                                                  stride, alpha, beta))

    b = 128
    a_h = rng.normal(size=(3, 2, b, b))  # 3 row tiles x 2 panels
    c_h = rng.normal(size=(3, b, b))
    want = np.stack([c_h[i] - np.concatenate(a_h[i], axis=1) @ np.concatenate(a_h[0], axis=1).T
                     for i in range(3)])
    # (1) one allocation: panel buffer (2, 3, b, b), walked with a stride of 3 tiles
    pan = torch.from_numpy(np.ascontiguousarray(a_h.transpose(1, 0, 2, 3))).cuda()
    c1 = torch.from_numpy(c_h.copy()).cuda()
    gemm([(pan[:, i], pan[:, 0], c1[i], c1[i], 2 * b, False) for i in range(3)], b, -1.0, 1.0)
    # (2) separate allocations, each padded by an odd number of doubles
    pads = [torch.zeros(2 * 3 * b * b + 8 * k + 2, dtype=torch.float64, device="cuda") for k in range(3)]
    tiles = []
    for i in range(3):
        view = pads[i][2 + 8 * i:].view(-1)[: 2 * b * b].view(2, b, b)
        view.copy_(torch.from_numpy(a_h[i]))
        tiles.append(view)
    c2 = torch.from_numpy(c_h.copy()).cuda()
    gemm([(tiles[i], tiles[0], c2[i], c2[i], 2 * b, False) for i in range(3)], b, -1.0, 1.0)
    torch.cuda.synchronize()
    for got in (c1, c2):
        assert rel(got.cpu().numpy(), want) <= 1e-14


@pytest.mark.parametrize("n,t,d", [(1024, 4, 8), (4096, 8, 8), (3000, 6, 3), (8192, 32, 8), (20000, 40, 5)])
def test_one_launch_solves_match_multi_launch(runtime, monkeypatch, n, t, d):
    """The cooperative one-launch alpha/beta solves (solve_flow.cu) against the
    4T-launch blocked solves (solve.cu) and the oracle: same loss and mean to
    round-off, bitwise reproducible run to run."""
    rng = np.random.default_rng(n + t)
    z, y, zt = rng.normal(size=(n, d)), rng.normal(size=n), rng.normal(size=(64, d))
    out = {}
    for flow in ("1", "0", "1"):
        monkeypatch.setenv("GPB_SOLVE_FLOW", flow)
        model = gpb.GPModel(ds(z, y), gpb.KernelParams(1.1, 0.9, 0.2), t)
        res = (model.log_likelihood(), model.predict(ds(zt)).mean)
        if flow in out:
            assert res[0] == out[flow][0] and np.array_equal(res[1], out[flow][1])
        out[flow] = res
    assert abs(out["1"][0] - out["0"][0]) <= 1e-12 * abs(out["0"][0])
    assert rel(out["1"][1], out["0"][1]) <= 1e-11
    if n <= 4096:
        o = OracleGP(z, y, t, 1.1, 0.9, 0.2)
        assert abs(out["1"][0] - o.log_likelihood()) <= TOL * abs(o.log_likelihood())
        assert rel(out["1"][1], o.predict(zt)) <= TOL


@pytest.mark.parametrize("n_train,n_test,d,seed", [(1024, 1024, 8, 0), (8192, 0, 8, 3), (131072, 8192, 16, 0)])
def test_device_generator_matches_host(runtime, n_train, n_test, d, seed):
    """gpb_msd_series_device: the trajectory and the lag
    embedding computed on the GPU are bitwise the host generator's arrays (up
    to config 4's 139264 samples), and a model built from them gives the same
    loss as one built from the host arrays."""
    train, test = gpb.make_msd_dataset(n_train, n_test, d, seed=seed)
    zt, yt, zs, ys = gpb.make_msd_dataset_device(n_train, n_test, d, seed=seed)
    assert np.array_equal(zt.cpu().numpy(), train.z) and np.array_equal(yt.cpu().numpy(), train.y)
    if n_test:
        assert np.array_equal(zs.cpu().numpy(), test.z) and np.array_equal(ys.cpu().numpy(), test.y)
    if n_train <= 8192:
        ll_host = gpb.GPModel(train, tiles_per_dim=8).log_likelihood()
        ll_dev = gpb.GPModel(gpb.Dataset(zt.cpu().numpy(), yt.cpu().numpy()), tiles_per_dim=8).log_likelihood()
        assert ll_host == ll_dev
