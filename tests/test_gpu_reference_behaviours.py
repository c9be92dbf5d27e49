"""The reference test suite's behavioural checks that are not already in
test_gpu_parity.py / test_gpu_corpus.py, re-expressed on the GPU class
(taskgp pkg/tests run against the B200 backend).

Each test names the reference test it follows; instances are drawn like the
reference's (standard-normal features, the CPU oracle as the dense answer).
"""

import numpy as np
import pytest

import paper_2505_00136_b200 as gpb
from oracle.tiled_gp import OracleGP, rel_fro

pytestmark = pytest.mark.gpu


def ds(z, y=None):
    z = np.asarray(z, dtype=np.float64)
    return gpb.Dataset(z, np.zeros(len(z)) if y is None else y)


def instance(rng, n, m=0, d=3):
    z, y = rng.normal(size=(n, d)), rng.normal(size=n)
    zt = rng.normal(size=(m, d)) if m else None
    kp = gpb.KernelParams(lengthscale=float(rng.uniform(0.7, 1.6)), vertical_scale=float(rng.uniform(0.6, 1.4)),
                          noise_variance=float(rng.uniform(0.05, 0.3)))
    return ds(z, y), zt, kp


def test_odd_test_count(runtime, rng):
    """test_model.py TestPredict.test_odd_test_count_works: 7 test points, 4 tiles."""
    train, _, kp = instance(rng, 16)
    zt = rng.normal(size=(7, 3))
    got = gpb.GPModel(train, kp, tiles_per_dim=4).predict(ds(zt)).mean
    o = OracleGP(train.z, train.y, 4, kp.lengthscale, kp.vertical_scale, kp.noise_variance)
    np.testing.assert_allclose(got, o.predict(zt), atol=1e-8)


def test_variances_non_negative_on_random_instances(runtime, rng):
    """test_model.py TestPredictUncertainty.test_variances_non_negative_on_random_instances."""
    for _ in range(20):
        train, zt, kp = instance(rng, 16, 8)
        res = gpb.GPModel(train, kp, tiles_per_dim=2).predict_variance(ds(zt))
        assert np.all(res.variance >= 0.0)


def test_posterior_contraction(runtime):
    """test_model.py test_posterior_contraction: a noise-free observation at the
    test point shrinks its variance."""
    for seed in range(5):
        local = np.random.default_rng(seed)
        z = local.uniform(-3, 3, size=(9, 1))
        y = np.sin(z[:, 0])
        kp = gpb.KernelParams(noise_variance=1e-8)
        zt = np.array([[0.37]])
        before = gpb.GPModel(ds(z, y), kp).predict_variance(ds(zt)).variance[0]
        after = gpb.GPModel(ds(np.vstack([z, zt]), np.append(y, np.sin(0.37))), kp).predict_variance(ds(zt))
        assert after.variance[0] <= before + 1e-12


def test_train_setter_checks_tiling(runtime, rng):
    """test_model.py TestCaching.test_train_setter_checks_tiling."""
    train, _, kp = instance(rng, 16)
    model = gpb.GPModel(train, kp, tiles_per_dim=4)
    with pytest.raises(gpb.errors.TilingError):
        model.train = ds(rng.normal(size=(6, 3)))


def test_repeated_predict_reuses_factor(runtime, rng):
    """test_model.py TestCaching.test_repeated_predict_reuses_factor: the second
    predict on unchanged parameters launches fewer kernels (no refactor)."""
    train, zt, kp = instance(rng, 32, 8)
    model = gpb.GPModel(train, kp, tiles_per_dim=4)
    model.predict(ds(zt))
    first = model.launch_count()
    model.predict(ds(zt))
    second = model.launch_count() - first
    assert second < first


def test_loss_decreases_on_smooth_data(runtime):
    """test_model.py TestOptimize.test_loss_decreases_on_smooth_data: 50 Adam
    steps on a lag-embedded sine."""
    x = np.linspace(0.0, 6.0, 72)
    data = gpb.lag_embed(np.sin(x), gpb.LagSpec(4))
    model = gpb.GPModel(data, gpb.KernelParams(lengthscale=2.5, vertical_scale=0.5, noise_variance=0.5),
                        tiles_per_dim=4)
    hist = model.optimize(gpb.AdamConfig(iterations=50))
    assert len(hist) == 50 and hist[-1] < hist[0]


def test_first_step_magnitude(runtime, rng):
    """test_model.py test_first_step_magnitude: bias correction makes the first
    log-space step about the learning rate."""
    train, _, kp = instance(rng, 16)
    model = gpb.GPModel(train, kp, tiles_per_dim=2)
    lr = 0.05
    before = np.log([kp.lengthscale, kp.vertical_scale, kp.noise_variance])
    model.optimize(gpb.AdamConfig(learning_rate=lr, iterations=1))
    p = model.params
    deltas = np.abs(np.log([p.lengthscale, p.vertical_scale, p.noise_variance]) - before)
    assert np.all(deltas >= 0.99 * lr) and np.all(deltas <= lr + 1e-12)


def test_parameters_stay_positive(runtime, rng):
    """test_model.py test_parameters_stay_positive."""
    train, _, _ = instance(rng, 16)
    model = gpb.GPModel(train, gpb.KernelParams(lengthscale=0.05, vertical_scale=0.05, noise_variance=1e-6),
                        tiles_per_dim=2)
    model.optimize(gpb.AdamConfig(iterations=25))
    p = model.params
    assert p.lengthscale > 0 and p.vertical_scale > 0 and p.noise_variance >= 1e-12


def test_non_trainable_parameters_fixed(runtime, rng):
    """test_model.py test_non_trainable_parameters_fixed."""
    train, _, _ = instance(rng, 16)
    kp = gpb.KernelParams(lengthscale=1.5, noise_variance=0.3, trainable=(False, True, False))
    model = gpb.GPModel(train, kp, tiles_per_dim=2)
    model.optimize(gpb.AdamConfig(iterations=5))
    assert model.params.lengthscale == 1.5 and model.params.noise_variance == 0.3
    assert model.params.vertical_scale != 1.0


def test_moments_persist_across_calls(runtime, rng):
    """test_model.py test_moments_persist_across_calls: two 1-step calls continue
    the same Adam trajectory."""
    train, _, kp = instance(rng, 16)
    split = gpb.GPModel(train, kp, tiles_per_dim=2)
    split.optimize(gpb.AdamConfig(iterations=1))
    split.optimize(gpb.AdamConfig(iterations=1))
    joint = gpb.GPModel(train, kp, tiles_per_dim=2)
    joint.optimize(gpb.AdamConfig(iterations=2))
    assert split.params.lengthscale == pytest.approx(joint.params.lengthscale, rel=1e-12)


def _fd_gradients(train, kp, tiles, h=1e-6):
    """Central differences of the negative log-likelihood in (l, nu, s2)."""
    theta = np.array([kp.lengthscale, kp.vertical_scale, kp.noise_variance])
    out = np.zeros(3)
    for k in range(3):
        vals = []
        for sgn in (1.0, -1.0):
            t = theta.copy()
            t[k] += sgn * h * t[k]
            vals.append(gpb.GPModel(train, gpb.KernelParams(*t), tiles_per_dim=tiles).compute_loss())
        out[k] = (vals[0] - vals[1]) / (2 * h * theta[k])
    return out


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_gradients_random_models(runtime, seed):
    """test_gradients.py test_random_models: analytic vs finite differences."""
    rng = np.random.default_rng(100 + seed)
    train, _, kp = instance(rng, 24, d=2)
    analytic = np.array(gpb.GPModel(train, kp, tiles_per_dim=2).loss_gradients())
    numeric = _fd_gradients(train, kp, 2)
    assert np.max(np.abs(analytic - numeric) / np.maximum(np.abs(numeric), 1e-12)) < 1e-5


def test_gradients_short_lengthscale_regime(runtime):
    """test_gradients.py test_short_lengthscale_regime: nearly diagonal K."""
    rng = np.random.default_rng(99)
    train = ds(rng.normal(size=(24, 2)), rng.normal(size=24))
    kp = gpb.KernelParams(lengthscale=0.15, noise_variance=0.2)
    analytic = np.array(gpb.GPModel(train, kp, tiles_per_dim=2).loss_gradients())
    np.testing.assert_allclose(analytic, _fd_gradients(train, kp, 2), rtol=1e-5)


def test_gradients_tile_invariant(runtime):
    """test_gradients.py test_gradients_tile_invariant."""
    rng = np.random.default_rng(5)
    train = ds(rng.normal(size=(16, 2)), rng.normal(size=16))
    g = [np.array(gpb.GPModel(train, tiles_per_dim=t).loss_gradients()) for t in (1, 2, 4)]
    np.testing.assert_allclose(g[0], g[1], atol=1e-10)
    np.testing.assert_allclose(g[0], g[2], atol=1e-10)


def test_random_models_against_oracle(runtime):
    """test_acceptance.py test_oracle_equivalence in spirit: loss, gradients and
    predictions of random models against the oracle at 1e-9."""
    for seed in range(4):
        rng = np.random.default_rng(700 + seed)
        train, zt, kp = instance(rng, 96, 24, d=4)
        model = gpb.GPModel(train, kp, tiles_per_dim=4)
        o = OracleGP(train.z, train.y, 4, kp.lengthscale, kp.vertical_scale, kp.noise_variance)
        assert abs(model.log_likelihood() - o.log_likelihood()) <= 1e-9 * abs(o.log_likelihood())
        assert rel_fro(np.array(model.loss_gradients()), np.array(o.loss_gradients())) <= 1e-9
        mean_o, var_o = o.predict_variance(zt)
        res = model.predict_variance(ds(zt))
        assert rel_fro(res.mean, mean_o) <= 1e-9 and rel_fro(res.variance, var_o) <= 1e-9
