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

The reference's own lag embedding (``LagSpec``/``lag_embed``, data.py:131-161:
rows t >= D only, the D preceding samples most recent first) and its CSV
round trip (``save_csv``/``load_csv``, data.py:164-201) are provided with the
same semantics so reference-produced files and series load unchanged.
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


@dataclass(frozen=True)
class LagSpec:
    """Number of lagged samples used as features (data.py:131-141)."""

    num_regressors: int

    def __post_init__(self) -> None:
        if self.num_regressors < 1:
            raise InvalidConfig(f"num_regressors must be >= 1, got {self.num_regressors}")


def lag_embed(series, spec: LagSpec) -> Dataset:
    """Regression dataset of lagged windows of a series (data.py:144-161):
    row t holds the D samples preceding sample t + D, most recent first, and
    y[t] is that sample; a series of length L gives L - D rows."""
    series = np.asarray(series, dtype=np.float64)
    d = spec.num_regressors
    if series.ndim != 1 or series.shape[0] <= d:
        raise DimensionMismatch(f"need a 1-D series longer than {d} samples, got shape {series.shape}")
    n = series.shape[0] - d
    z = np.empty((n, d))
    for j in range(d):
        z[:, j] = series[d - 1 - j: d - 1 - j + n]
    return Dataset(z=z, y=series[d:].copy())


def save_csv(data: Dataset, path: str, header: bool = False) -> None:
    """One row per sample, feature columns then y, floats via repr (loss-free)."""
    with open(path, "w", encoding="utf-8") as fh:
        if header:
            fh.write(",".join([f"z{j}" for j in range(data.d)] + ["y"]) + "\n")
        for row, target in zip(data.z, data.y):
            fh.write(",".join(repr(float(v)) for v in row) + f",{float(target)!r}\n")


def load_csv(path: str, header: bool = False) -> Dataset:
    """Read a file written by save_csv; the last column is y.  ParseError
    (with the line number) on ragged rows, bad numbers or an empty file."""
    rows: list[list[float]] = []
    width = None
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, line in enumerate(fh, start=1):
            if lineno == 1 and header:
                continue
            line = line.strip()
            if not line:
                continue
            cols = line.split(",")
            if width is None:
                width = len(cols)
                if width < 2:
                    raise ParseError("need at least one feature column and y", lineno)
            elif len(cols) != width:
                raise ParseError(f"expected {width} columns, got {len(cols)}", lineno)
            try:
                rows.append([float(c) for c in cols])
            except ValueError as exc:
                raise ParseError(str(exc), lineno) from exc
    if not rows:
        raise ParseError("no data rows", 1)
    arr = np.array(rows)
    return Dataset(z=arr[:, :-1], y=arr[:, -1])
