"""CPU-only checks: the C-ABI library loads and exports the header's symbols,
and the host-side mirror of the reference interface validates like it does."""

import os
import re

import numpy as np
import pytest

import paper_2505_00136_b200 as gpb
from paper_2505_00136_b200 import _lib
from paper_2505_00136_b200.errors import (
    DimensionMismatch,
    InvalidConfig,
    NotRunning,
    TilingError,
)
from conftest import ROOT, load_golden


def header_symbols():
    text = open(os.path.join(ROOT, "include", "gpb200.h")).read()
    return sorted(set(re.findall(r"\b(gpb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()  # loading needs no GPU (static cudart, lazy init)
    syms = header_symbols()
    assert len(syms) >= 24
    for name in syms:
        assert hasattr(lib, name), name
    # and the binding declares exactly those
    assert set(syms) == set(_lib.SIGNATURES)


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_abi_version():
    assert _lib.load().gpb_abi_version() == 1


def test_generator_pinned_by_reference_fixture():
    g = load_golden("c0")
    tr, te = gpb.make_msd_dataset(1024, 1024, 8, seed=0)
    np.testing.assert_array_equal(tr.z[:16], g["z_head"])
    assert float(tr.z.sum()) == float(g["z_sum"])
    assert float(tr.y.sum()) == float(g["y_sum"])
    assert float(te.z.sum()) == float(g["zt_sum"])
    # zero padding of the first lags, continuation into the test rows
    assert np.all(tr.z[0, 1:] == 0.0)
    np.testing.assert_array_equal(te.z[0, 1:], tr.z[-1, :-1])


class TestValidation:
    def test_kernel_params(self):
        for kw in ({"lengthscale": 0.0}, {"vertical_scale": -1.0}, {"noise_variance": -1e-3},
                   {"trainable": (True, True)}):
            with pytest.raises(InvalidConfig):
                gpb.KernelParams(**kw)

    @pytest.mark.parametrize("kw", [{"learning_rate": 0.0}, {"beta1": 1.0}, {"beta2": -0.1},
                                    {"epsilon": 0.0}, {"iterations": 0}])
    def test_adam_config(self, kw):
        with pytest.raises(InvalidConfig):
            gpb.AdamConfig(**kw)

    def test_dataset(self):
        with pytest.raises(DimensionMismatch):
            gpb.Dataset(z=np.zeros(3), y=np.zeros(3))
        with pytest.raises(DimensionMismatch):
            gpb.Dataset(z=np.zeros((3, 2)), y=np.zeros(2))
        with pytest.raises(InvalidConfig):
            gpb.Dataset(z=np.full((2, 1), np.nan), y=np.zeros(2))

    def test_tiling(self, rng):
        train = gpb.Dataset(z=rng.normal(size=(10, 2)), y=np.zeros(10))
        with pytest.raises(TilingError):
            gpb.GPModel(train, tiles_per_dim=3)
        with pytest.raises(TilingError):
            gpb.GPModel(train, tiles_per_dim=0)
        model = gpb.GPModel(train, tiles_per_dim=5)
        with pytest.raises(TilingError):
            model.train = gpb.Dataset(z=rng.normal(size=(6, 2)), y=np.zeros(6))

    def test_defaults(self, rng):
        model = gpb.GPModel(gpb.Dataset(z=rng.normal(size=(8, 2)), y=np.zeros(8)))
        assert model.tiles_per_dim == 1
        assert model.params == gpb.KernelParams()

    def test_calls_require_runtime(self, rng):
        """test_model.py:43-47: every heavy call needs a live runtime."""
        train = gpb.Dataset(z=rng.normal(size=(8, 2)), y=np.zeros(8))
        model = gpb.GPModel(train)
        for call in (lambda: model.predict(train), model.log_likelihood, model.cholesky,
                     model.loss_gradients):
            with pytest.raises(NotRunning):
                call()
        with pytest.raises(NotRunning):
            gpb.stop_runtime()

    def test_runtime_config(self, monkeypatch):
        monkeypatch.setenv("TASKGP_WORKERS", "3")
        assert gpb.RuntimeConfig().resolved_worker_count() == 3
        monkeypatch.setenv("TASKGP_WORKERS", "x")
        with pytest.raises(InvalidConfig):
            gpb.RuntimeConfig().resolved_worker_count()
        with pytest.raises(InvalidConfig):
            gpb.RuntimeConfig(worker_count=0).resolved_worker_count()
        monkeypatch.setenv("GPB_DEVICE", "2")
        assert gpb.RuntimeConfig().resolved_device() == 2
        assert gpb.RuntimeConfig(device=1).resolved_device() == 1

    def test_gprat_constructor_builds_lag_features(self):
        u = np.arange(1.0, 9.0)
        model = gpb.GP(u, np.zeros(8), n_tiles=2, n_tile_size=4, n_regressors=3)
        np.testing.assert_array_equal(model.train.z[:3], [[1, 0, 0], [2, 1, 0], [3, 2, 1]])
        with pytest.raises(TilingError):
            gpb.GP(u, np.zeros(8), n_tiles=3, n_tile_size=2, n_regressors=3)


def test_status_mapping():
    from paper_2505_00136_b200 import errors

    assert _lib._STATUS[6] is errors.NotPositiveDefinite
    assert _lib._STATUS[8] is errors.NumericalConsistencyError
    assert _lib._STATUS[4] is errors.TilingError
    assert _lib._STATUS[3] is errors.NotRunning


def test_product_path_does_not_import_oracle():
    """The product package must never route through the CPU oracle."""
    pkg = os.path.join(ROOT, "paper_2505_00136_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "oracle" not in re.sub(r"#.*|\"\"\"[\s\S]*?\"\"\"", "", src), fn


class TestVarianceClamp:
    """test_model.py:165-172 on the library's clamp (gpb_clamp_variances, the
    host routine gpb_predict applies to every variance it returns)."""

    def test_round_off_clamped_to_zero(self):
        from paper_2505_00136_b200.model import _clamp_variances

        out = _clamp_variances(np.array([1.0, -1e-10, 0.0]))
        np.testing.assert_array_equal(out, np.array([1.0, 0.0, 0.0]))

    def test_genuinely_negative_raises(self):
        from paper_2505_00136_b200.errors import NumericalConsistencyError
        from paper_2505_00136_b200.model import _clamp_variances

        with pytest.raises(NumericalConsistencyError):
            _clamp_variances(np.array([0.5, -1e-6]))

    def test_boundary_and_input_untouched(self):
        from paper_2505_00136_b200.model import _clamp_variances

        v = np.array([-1e-9, -0.0, 2.0])
        np.testing.assert_array_equal(_clamp_variances(v), [0.0, 0.0, 2.0])
        assert v[0] == -1e-9  # the caller's array is not modified
