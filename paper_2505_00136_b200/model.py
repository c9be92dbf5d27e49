"""GP regression model: the drop-in for ``taskgp.GPModel`` (model.py:91-485).

Every heavy call goes through the C ABI (``include/gpb200.h``) into the
sm_100a kernels; there is no host fallback.  Names, argument meaning,
return types, caching and error behaviour follow the reference:

* ``GPModel(train, params=None, tiles_per_dim=1)`` (model.py:111-131),
  ``TilingError`` unless ``tiles_per_dim`` divides n;
* ``train`` / ``params`` setters invalidate the cached factor
  (model.py:135-165);
* ``predict``, ``predict_variance``, ``predict_with_full_cov`` return a
  ``PredictionResult`` (model.py:77-88, 221-314);
* ``log_likelihood`` returns +log L (model.py:316-339),
  ``loss_gradients`` dNLL/d(l, nu, sigma^2) (model.py:341-435),
  ``optimize(AdamConfig)`` the NLL history (model.py:437-485);
* any failure invalidates cached state (``_guarded``, model.py:210-217).

GPRat-style aliases from BASELINE.json's ``north_star``: ``cholesky()``,
``compute_loss()`` (= -log_likelihood),
``predict_with_uncertainty()`` (= predict_variance), and the ``GP``
constructor taking the raw training series plus ``n_regressors``.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, replace

import numpy as np

from . import _lib
from .covariance import KernelParams
from .data import Dataset, lag_features
from .errors import DimensionMismatch, InvalidConfig, TaskGPError, TilingError
from .runtime import require_runtime


@dataclass(frozen=True)
class AdamConfig:
    """Adam settings (model.py:38-74), validated identically."""

    learning_rate: float = 0.1
    beta1: float = 0.9
    beta2: float = 0.999
    epsilon: float = 1e-8
    iterations: int = 100

    def __post_init__(self) -> None:
        if not self.learning_rate > 0:
            raise InvalidConfig(f"learning_rate must be positive, got {self.learning_rate}")
        for name, beta in (("beta1", self.beta1), ("beta2", self.beta2)):
            if not 0.0 <= beta < 1.0:
                raise InvalidConfig(f"{name} must lie in [0, 1), got {beta}")
        if not self.epsilon > 0:
            raise InvalidConfig(f"epsilon must be positive, got {self.epsilon}")
        if self.iterations < 1:
            raise InvalidConfig(f"iterations must be at least 1, got {self.iterations}")


@dataclass(frozen=True)
class PredictionResult:
    """Predicted mean plus optional uncertainty (model.py:77-88)."""

    mean: np.ndarray
    variance: np.ndarray | None = None
    full_covariance: np.ndarray | None = None


def _clamp_variances(variance: np.ndarray) -> np.ndarray:
    """Round-off negatives in [-1e-9, 0) become 0; anything below raises
    ``NumericalConsistencyError`` (model.py:488-496).  Runs the library's
    clamp (``gpb_clamp_variances``, the one ``gpb_predict`` applies) on a copy."""
    out = np.array(variance, dtype=np.float64, copy=True, order="C").reshape(-1)
    _lib.check(_lib.load().gpb_clamp_variances(_lib.dptr(out), out.shape[0]))
    return out.reshape(np.shape(variance))


def _as_dataset(data) -> Dataset:
    if isinstance(data, Dataset):
        return data
    return Dataset(z=np.asarray(data.z), y=np.asarray(data.y))


class GPModel:
    """Squared-exponential GP regression over a fixed training set.

    Not safe for concurrent calls on the same instance (model.py:104-108);
    distinct models may be used concurrently.
    """

    def __init__(self, train, params: KernelParams | None = None, tiles_per_dim: int = 1):
        train = _as_dataset(train)
        if tiles_per_dim < 1 or train.n % tiles_per_dim != 0:
            raise TilingError(
                f"tiles_per_dim={tiles_per_dim} must divide the {train.n} training points"
            )
        self._train = train
        self._params = params if params is not None else KernelParams()
        self._tiles_per_dim = int(tiles_per_dim)
        self._handle = None  # ctypes.c_void_p of the bound gpb_model
        self._runtime = None
        # Adam moments and step count (model.py:446-448 keeps them on the
        # model across optimize calls): read back from the C model after every
        # optimize and restored into a re-created handle (close(), runtime restart)
        self._adam = (np.zeros(3), np.zeros(3), 0)
        self._pending_train = False
        self._digit_planes = None  # None: the library default (GPB_OZAKI)

    # -- attribute management (model.py:135-165) ---------------------------
    @property
    def train(self) -> Dataset:
        return self._train

    @train.setter
    def train(self, value) -> None:
        value = _as_dataset(value)
        if value.n % self._tiles_per_dim != 0:
            raise TilingError(
                f"tiles_per_dim={self._tiles_per_dim} must divide the {value.n} training points"
            )
        self._train = value
        if self._handle is not None:
            self._pending_train = True

    @property
    def params(self) -> KernelParams:
        return self._params

    @params.setter
    def params(self, value: KernelParams) -> None:
        self._params = value
        if self._handle is not None:
            self._push_params()

    @property
    def tiles_per_dim(self) -> int:
        return self._tiles_per_dim

    # -- binding to the C model --------------------------------------------
    def _push_params(self) -> None:
        p = self._params
        flags = (ctypes.c_uint8 * 3)(*[1 if t else 0 for t in p.trainable])
        _lib.check(_lib.load().gpb_model_set_params(
            self._handle, float(p.lengthscale), float(p.vertical_scale),
            float(p.noise_variance), flags))

    def _bind(self):
        """The live gpb_model handle (created on first use under the runtime)."""
        rt = require_runtime()
        lib = _lib.load()
        if self._handle is not None and self._runtime is not rt:
            lib.gpb_model_destroy(self._handle)
            self._handle = None
        if self._handle is None:
            z, y = self._train.z, self._train.y
            h = ctypes.c_void_p()
            _lib.check(lib.gpb_model_create(rt.handle, _lib.dptr(z), _lib.dptr(y), z.shape[0],
                                            z.shape[1], self._tiles_per_dim, ctypes.byref(h)))
            self._handle = h
            self._runtime = rt
            self._pending_train = False
            self._push_params()
            m1, m2, step = self._adam
            _lib.check(lib.gpb_model_set_adam(h, _lib.dptr(m1), _lib.dptr(m2), step))
            if self._digit_planes is not None:
                _lib.check(lib.gpb_model_set_ozaki(h, self._digit_planes))
        elif self._pending_train:
            z, y = self._train.z, self._train.y
            _lib.check(lib.gpb_model_set_train(self._handle, _lib.dptr(z), _lib.dptr(y),
                                               z.shape[0], z.shape[1]))
            self._pending_train = False
        return self._handle

    def _guarded(self, fn):
        handle = self._bind()
        try:
            return fn(_lib.load(), handle)
        except TaskGPError:
            # model.py:210-217: a failure must not leave a poisoned cache
            if self._handle is not None:
                self._push_params()
            raise

    def close(self) -> None:
        """Release the model's device buffers now (they are re-created on the next call)."""
        h, self._handle = self._handle, None
        if h is not None:
            _lib.load().gpb_model_destroy(h)

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None:
            try:
                _lib.load().gpb_model_destroy(h)
            except Exception:
                pass

    def _check_test(self, test) -> Dataset:
        test = _as_dataset(test)
        if test.d != self._train.d:
            raise DimensionMismatch(
                f"test has {test.d} features, model was trained with {self._train.d}"
            )
        return test

    # -- public API ---------------------------------------------------------
    def _predict(self, test, var: bool, cov: bool):
        test = self._check_test(test)
        m = test.n
        mean = np.empty(m)
        v = np.empty(m) if var else None
        c = np.empty((m, m)) if cov else None

        def call(lib, h):
            _lib.check(lib.gpb_predict(h, _lib.dptr(test.z), m, test.d, _lib.dptr(mean),
                                       _lib.dptr(v), _lib.dptr(c)))

        self._guarded(call)
        return mean, v, c

    def predict(self, test) -> PredictionResult:
        """Posterior mean at the test points (model.py:221-240)."""
        mean, _, _ = self._predict(test, False, False)
        return PredictionResult(mean=mean)

    def predict_variance(self, test) -> PredictionResult:
        """Posterior mean and per-point variances (model.py:280-314)."""
        mean, var, _ = self._predict(test, True, False)
        return PredictionResult(mean=mean, variance=var)

    def predict_with_full_cov(self, test) -> PredictionResult:
        """Posterior mean and full posterior covariance (model.py:242-278)."""
        mean, _, cov = self._predict(test, False, True)
        return PredictionResult(mean=mean, full_covariance=cov)

    def log_likelihood(self) -> float:
        """Log marginal likelihood of the training observations (model.py:316-339)."""
        out = ctypes.c_double()
        self._guarded(lambda lib, h: _lib.check(lib.gpb_log_likelihood(h, ctypes.byref(out))))
        return float(out.value)

    def loss_gradients(self) -> tuple[float, float, float]:
        """dNLL/d(lengthscale, vertical_scale, noise_variance) (model.py:341-435)."""
        tr = self._params.trainable
        if not (tr[0] or tr[1] or tr[2]):
            return (0.0, 0.0, 0.0)
        out = (ctypes.c_double * 3)()
        self._guarded(lambda lib, h: _lib.check(lib.gpb_loss_gradients(h, out)))
        return (float(out[0]), float(out[1]), float(out[2]))

    def optimize(self, opt: AdamConfig | None = None) -> list[float]:
        """Adam on the log-parameters; returns the NLL after each step (model.py:437-485)."""
        opt = opt if opt is not None else AdamConfig()
        hist = np.zeros(opt.iterations)

        def call(lib, h):
            status = lib.gpb_optimize(h, opt.learning_rate, opt.beta1, opt.beta2, opt.epsilon,
                                      opt.iterations, _lib.dptr(hist))
            # parameters and Adam state advanced on the device side even on failure
            got = (ctypes.c_double * 3)()
            lib.gpb_model_get_params(h, got)
            self._params = replace(self._params, lengthscale=float(got[0]),
                                   vertical_scale=float(got[1]), noise_variance=float(got[2]))
            m1, m2, step = np.zeros(3), np.zeros(3), ctypes.c_int64()
            lib.gpb_model_get_adam(h, _lib.dptr(m1), _lib.dptr(m2), ctypes.byref(step))
            self._adam = (m1, m2, int(step.value))
            _lib.check(status)

        self._guarded(call)
        return [float(x) for x in hist]

    # -- GPRat-style aliases (BASELINE.json north_star) ---------
    def cholesky(self) -> np.ndarray:
        """Dense lower Cholesky factor of K (the reference's _ensure_factor)."""
        n = self._train.n
        out = np.empty((n, n))
        self._guarded(lambda lib, h: _lib.check(lib.gpb_cholesky(h, _lib.dptr(out))))
        return out

    def factorize(self) -> None:
        """Assemble and factor K on the device without exporting the factor."""
        self._guarded(lambda lib, h: _lib.check(lib.gpb_cholesky(h, None)))

    def compute_loss(self) -> float:
        """Negative log marginal likelihood (GPRat ``compute_loss``)."""
        return -self.log_likelihood()

    def predict_with_uncertainty(self, test) -> PredictionResult:
        """GPRat name of :meth:`predict_variance`."""
        return self.predict_variance(test)

    # -- instrumentation ----------------------------------------------------
    def device_timings(self) -> dict:
        """Per-phase device times (ms, CUDA events) of the latest calls."""
        out = (ctypes.c_double * 8)()
        if self._handle is None:
            return {}
        _lib.load().gpb_model_timings(self._handle, out, 8)
        names = ("assembly", "factor", "solves", "cross_mean", "trsm_variance", "gradient",
                 "full_cov")
        return {k: float(out[i]) for i, k in enumerate(names)}

    # -- tcgen05 digit-plane products (csrc/ozaki.cuh) ----------------------
    @property
    def digit_planes(self) -> int:
        """Planes per operand of the tcgen05 int8 products that carry the long
        FP64 contractions (trailing updates, prediction sweep, full covariance);
        8 by default (env ``GPB_OZAKI``), 0: every product on the FP64 DMMA kernels."""
        if self._handle is None:
            if self._digit_planes is not None:
                return self._digit_planes
            env = os.environ.get("GPB_OZAKI")
            return 8 if env is None else (0 if int(env) <= 0 else min(8, max(4, int(env))))
        out = ctypes.c_int()
        _lib.check(_lib.load().gpb_model_get_ozaki(self._handle, ctypes.byref(out), None))
        return int(out.value)

    @digit_planes.setter
    def digit_planes(self, planes: int) -> None:
        planes = int(planes)
        if planes != 0 and not 4 <= planes <= 8:
            raise InvalidConfig("digit_planes must be 0 (off) or 4..8")
        self._digit_planes = planes
        if self._handle is not None:
            _lib.check(_lib.load().gpb_model_set_ozaki(self._handle, planes))

    def digit_plane_fallbacks(self) -> int:
        if self._handle is None:
            return 0
        out = ctypes.c_int64()
        _lib.check(_lib.load().gpb_model_get_ozaki(self._handle, None, ctypes.byref(out)))
        return int(out.value)

    def launch_count(self) -> int:
        if self._handle is None:
            return 0
        out = ctypes.c_int64()
        _lib.load().gpb_model_launch_count(self._handle, ctypes.byref(out))
        return int(out.value)


class GP(GPModel):
    """GPRat-style constructor (``gprat.GP``) over a raw input series.

    ``GP(train_in, train_out, n_tiles, n_tile_size, n_regressors,
    kernel_params=[l, nu, sigma2], trainable=[True, True, True])``: the
    features of sample t are the lagged inputs (u_t, ..., u_{t-R+1}),
    zero-padded (BASELINE.json data generator), and ``n_tiles * n_tile_size``
    must equal the number of samples.
    """

    def __init__(self, train_in, train_out, n_tiles: int, n_tile_size: int, n_regressors: int,
                 kernel_params=(1.0, 1.0, 0.1), trainable=(True, True, True)):
        u = np.asarray(train_in, dtype=np.float64)
        y = np.asarray(train_out, dtype=np.float64)
        if u.ndim != 1 or y.shape != u.shape:
            raise DimensionMismatch("train_in and train_out must be equal-length vectors")
        if n_tiles * n_tile_size != u.shape[0]:
            raise TilingError(
                f"n_tiles * n_tile_size = {n_tiles * n_tile_size} != {u.shape[0]} samples"
            )
        self.n_regressors = int(n_regressors)
        params = KernelParams(*[float(x) for x in kernel_params], trainable=tuple(trainable))
        super().__init__(Dataset(z=lag_features(u, self.n_regressors), y=y), params, n_tiles)

    def features(self, test_in) -> Dataset:
        u = np.asarray(test_in, dtype=np.float64)
        return Dataset(z=lag_features(u, self.n_regressors), y=np.zeros(u.shape[0]))
