"""Training/test containers and the BASELINE.json synthetic generator.

``Dataset`` mirrors the reference container (``pkg/src/taskgp/data.py:18-45``):
an N x D float64 feature matrix ``z`` (one row per sample) and an N-vector
``y``, validated and made C-contiguous.

``make_msd_dataset`` is the generator BASELINE.json prescribes for every
config (it is NOT the reference's RK4/Duffing generator, see SURVEY.md D2;
parity does not depend on it because both paths consume identical arrays).
Conventions are pinned in SURVEY.md Appendix A:

1. ``rng = default_rng(seed)``; draw ``u ~ U[-1, 1]`` (N values) first,
   then ``noise ~ N(0, 0.1^2)`` (N values), N = n_train + n_test.
2. Mass-spring-damper m=1, c=0.5, k=1, semi-implicit Euler, dt=0.01, x0=v0=0:
   ``v += dt * (u_t - c v - k x) / m``; ``x += dt * v``; position_t = x.
3. ``y_t = position_t + noise_t``.
4. Feature row t = (u_t, u_{t-1}, ..., u_{t-n_reg+1}), u_{<0} = 0.
5. Train = rows [0, n_train), test = rows [n_train, N) (a continuation).

The reference's lag embedding and dataset CSV format (``LagSpec`` /
``lag_embed`` / ``save_csv`` / ``load_csv``) are
provided with the same observable behaviour -- pinned by files the reference
wrote, tests/golden/ref_dataset* -- so reference-produced series and files
load unchanged.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import DimensionMismatch, InvalidConfig, ParseError


@dataclass(frozen=True)
class Dataset:
    """Feature matrix z (one row per sample) and observation vector y.

    Same validation contract as ``taskgp.Dataset`` (data.py:25-37).
    """

    z: np.ndarray
    y: np.ndarray

    def __post_init__(self) -> None:
        z = np.ascontiguousarray(self.z, dtype=np.float64)
        y = np.ascontiguousarray(self.y, dtype=np.float64)
        if z.ndim != 2 or z.shape[1] < 1:
            raise DimensionMismatch(f"z must be N x D with D >= 1, got shape {z.shape}")
        if y.ndim != 1 or y.shape[0] != z.shape[0]:
            raise DimensionMismatch(
                f"y must have one entry per row of z, got {y.shape} vs {z.shape}"
            )
        if not (np.isfinite(z).all() and np.isfinite(y).all()):
            raise InvalidConfig("dataset entries must be finite")
        object.__setattr__(self, "z", z)
        object.__setattr__(self, "y", y)

    @property
    def n(self) -> int:
        return self.z.shape[0]

    @property
    def d(self) -> int:
        return self.z.shape[1]


def msd_series(n: int, seed: int, dt: float = 0.01, mass: float = 1.0,
               damping: float = 0.5, stiffness: float = 1.0):
    """Forcing u, noisy position y of the BASELINE mass-spring-damper."""
    rng = np.random.default_rng(seed)
    u = rng.uniform(-1.0, 1.0, size=n)
    noise = rng.normal(0.0, 0.1, size=n)
    pos = np.empty(n)
    x = 0.0
    v = 0.0
    for t in range(n):
        v = v + dt * (u[t] - damping * v - stiffness * x) / mass
        x = x + dt * v
        pos[t] = x
    return u, pos + noise


def lag_features(u: np.ndarray, n_reg: int) -> np.ndarray:
    """Row t = (u_t, u_{t-1}, ..., u_{t-n_reg+1}), zero before the start."""
    n = u.shape[0]
    z = np.zeros((n, n_reg))
    for lag in range(n_reg):
        z[lag:, lag] = u[: n - lag]
    return z


def make_msd_dataset(n_train: int, n_test: int, n_reg: int, seed: int = 0):
    """(train, test) Datasets from one BASELINE.json trajectory."""
    if n_train < 1 or n_test < 0 or n_reg < 1:
        raise InvalidConfig("need n_train >= 1, n_test >= 0, n_reg >= 1")
    u, y = msd_series(n_train + n_test, seed)
    z = lag_features(u, n_reg)
    train = Dataset(z=z[:n_train], y=y[:n_train])
    test = Dataset(z=z[n_train:], y=y[n_train:]) if n_test else None
    return train, test


def make_msd_dataset_device(n_train: int, n_test: int, n_reg: int, seed: int = 0, device: int | None = None):
    """make_msd_dataset with the trajectory and the lag embedding computed on
    the GPU (gpb_msd_series_device; bitwise the host arrays): returns torch
    tensors (z_train, y_train, z_test, y_test) in device memory -- only the
    2 N random draws cross PCIe.  Needs a running runtime."""
    import ctypes

    import torch

    from . import _lib
    from .runtime import require_runtime

    if n_train < 1 or n_test < 0 or n_reg < 1:
        raise InvalidConfig("need n_train >= 1, n_test >= 0, n_reg >= 1")
    rt = require_runtime()
    dev = torch.device("cuda", rt.device if device is None else device)
    n = n_train + n_test
    rng = np.random.default_rng(seed)  # the draws of msd_series, in its order
    u = torch.from_numpy(rng.uniform(-1.0, 1.0, size=n)).to(dev)
    noise = torch.from_numpy(rng.normal(0.0, 0.1, size=n)).to(dev)
    z = torch.empty((n, n_reg), dtype=torch.float64, device=dev)
    y = torch.empty(n, dtype=torch.float64, device=dev)
    torch.cuda.synchronize(dev)  # the library works on its own stream
    _lib.check(_lib.load().gpb_msd_series_device(rt.handle, ctypes.c_void_p(u.data_ptr()),
                                                 ctypes.c_void_p(noise.data_ptr()), n, n_reg, 0.01, 1.0, 0.5,
                                                 1.0, ctypes.c_void_p(z.data_ptr()), ctypes.c_void_p(y.data_ptr())))
    return z[:n_train], y[:n_train], z[n_train:], y[n_train:]


@dataclass(frozen=True)
class LagSpec:
    """How many past samples form one feature row."""

    num_regressors: int

    def __post_init__(self) -> None:
        if self.num_regressors < 1:
            raise InvalidConfig(f"num_regressors must be >= 1, got {self.num_regressors}")


def lag_embed(series, spec: LagSpec) -> Dataset:
    """Sliding windows of D + 1 samples over a series: the window's last
    sample is the target, the D before it (most recent first) the features,
    so a series of length L gives L - D rows (the reference's lag embedding,
    taskgp data.py:144-161, whose fixtures tests/golden/ref_dataset* pin it)."""
    x = np.asarray(series, dtype=np.float64)
    d = spec.num_regressors
    if x.ndim != 1 or x.size <= d:
        raise DimensionMismatch(f"need a 1-D series longer than {d} samples, got shape {x.shape}")
    win = np.lib.stride_tricks.sliding_window_view(x, d + 1)
    return Dataset(z=win[:, d - 1::-1], y=win[:, d])


def save_csv(data: Dataset, path: str, header: bool = False) -> None:
    """Feature columns then y per line, every value as its shortest exact
    repr, optionally under a ``z0,...,y`` header (loss-free round trip)."""
    table = np.column_stack([data.z, data.y]).tolist()
    lines = [",".join(map(repr, row)) for row in table]
    if header:
        lines.insert(0, ",".join([f"z{j}" for j in range(data.d)] + ["y"]))
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("".join(line + "\n" for line in lines))


def load_csv(path: str, header: bool = False) -> Dataset:
    """Inverse of save_csv (the last column is y).  ``ParseError`` carries the
    1-based line of the first ragged row or unparsable number, or of an empty file."""
    with open(path, "r", encoding="utf-8") as fh:
        numbered = [(k + 1, t.strip()) for k, t in enumerate(fh.read().splitlines())]
    body = [(k, t) for k, t in numbered[1 if header else 0:] if t]
    if not body:
        raise ParseError("no data rows", 1)
    split = [(k, t.split(",")) for k, t in body]
    width = len(split[0][1])
    if width < 2:
        raise ParseError("need at least one feature column and y", split[0][0])
    values = []
    for k, cells in split:
        if len(cells) != width:
            raise ParseError(f"expected {width} columns, got {len(cells)}", k)
        try:
            values.append(list(map(float, cells)))
        except ValueError as exc:
            raise ParseError(str(exc), k) from exc
    table = np.array(values)
    return Dataset(z=table[:, :-1], y=table[:, -1])
