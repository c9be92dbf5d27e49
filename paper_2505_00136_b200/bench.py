"""Sweep harness speaking the reference's record format.

The CSV file format, the bootstrap statistic and the summary text are the
interface: records written here load in taskgp's harness and vice versa, and
``tests/test_records.py`` checks that against files the reference wrote
(``tests/golden/ref_*``).  The format, restated from those files and from
taskgp bench.py's docstrings:

* one header line with the 13 field names of ``BenchRecord`` in order, then
  one line per record, fields joined by ``,``;
* integers in decimal, floats via ``repr`` (shortest loss-free form, ``nan``
  for failed cells), the raw repetition times joined by ``;``, the error text
  last (newlines flattened to spaces, empty when the cell succeeded) -- being
  the last field it may itself contain commas;
* the 95 % percentile-bootstrap half width of the mean: 1000 resamples drawn
  with ``numpy.random.default_rng(seed).integers`` as one (1000, n) index
  matrix, percentiles 2.5 / 97.5 of the resampled means;
* the summary: a title line, then per tiling the worker-count speedups and per
  worker count the tiling speedups, each against the slowest cell of its
  group, then one FAILED line per failed cell.

Execution is the B200 path: a cell binds the device runtime, runs warm-up
calls, then times each repetition as one blocking public-API call (host numpy
in, host numpy out: assembly, factorisation and copies are inside the timed
call, as for a library user).  ``worker_count`` keeps its validation and is
recorded, but sizes no host pool.  Data come from the BASELINE generator.
"""

from __future__ import annotations

import itertools
import math
import time
from dataclasses import dataclass, fields

import numpy as np

from .covariance import KernelParams
from .data import Dataset, make_msd_dataset
from .errors import InvalidConfig, ParseError, TaskGPError, TilingError
from .model import AdamConfig, GPModel
from .runtime import RuntimeConfig, start_runtime, stop_runtime

OPERATIONS = ("optimize", "predict", "predict_full_cov", "predict_var")
OPTIMIZE_ITERATIONS = 3  # fixed Adam steps per optimisation cell


def _pow2(v: int) -> bool:
    return v >= 1 and v & (v - 1) == 0


@dataclass(frozen=True)
class ExperimentSpec:
    """An operation crossed with worker counts and tilings."""

    operation: str = "predict"
    n_train: int = 256
    n_test: int = 256
    regressors: int = 8
    tiles_per_dim: tuple[int, ...] = (1,)
    worker_count: tuple[int, ...] = (1,)
    repetitions: int = 5
    warmup: int = 1
    output_path: str | None = None
    seed: int = 0

    def __post_init__(self) -> None:
        problems = [
            (self.operation not in OPERATIONS,
             f"operation must be one of {OPERATIONS}, got {self.operation!r}"),
            (not _pow2(self.n_train), f"n_train must be a power of two, got {self.n_train}"),
            (not _pow2(self.n_test), f"n_test must be a power of two, got {self.n_test}"),
            (self.regressors < 1, f"regressors must be >= 1, got {self.regressors}"),
            (self.repetitions < 1, f"repetitions must be >= 1, got {self.repetitions}"),
            (self.warmup < 0, f"warmup must be >= 0, got {self.warmup}"),
            (not self.tiles_per_dim or not self.worker_count,
             "tiles_per_dim and worker_count must be non-empty"),
        ]
        for bad, message in problems:
            if bad:
                raise InvalidConfig(message)
        bad_tiles = [t for t in self.tiles_per_dim if t < 1 or self.n_train % t]
        if bad_tiles:
            raise TilingError(f"tiles_per_dim={bad_tiles[0]} does not divide n_train={self.n_train}")
        bad_workers = [w for w in self.worker_count if w < 1]
        if bad_workers:
            raise InvalidConfig(f"worker_count entries must be >= 1, got {bad_workers[0]}")


@dataclass(frozen=True)
class BenchRecord:
    """Timing result of one sweep cell (field order = CSV column order)."""

    operation: str
    n_train: int
    n_test: int
    regressors: int
    tiles_per_dim: int
    worker_count: int
    repetitions: int
    warmup: int
    seed: int
    mean_s: float
    ci_half_width_s: float
    raw_times_s: tuple[float, ...]
    error: str | None = None


# ---- text codecs of the CSV columns, keyed by field type --------------------------
def _enc_times(ts) -> str:
    return ";".join(map(repr, ts))


def _dec_times(text: str) -> tuple[float, ...]:
    return tuple(float(tok) for tok in text.split(";") if tok)


def _enc_error(err) -> str:
    return "" if err is None else err.replace("\n", " ")


_CODECS = {
    "str": (str, str),
    "int": (str, int),
    "float": (repr, float),
    "tuple[float, ...]": (_enc_times, _dec_times),
    "str | None": (_enc_error, lambda text: text or None),
}
_SCHEMA = [(f.name,) + _CODECS[f.type] for f in fields(BenchRecord)]
_HEADER = ",".join(name for name, _, _ in _SCHEMA)


def emit_csv(records: list[BenchRecord], path: str) -> None:
    """Write the header and one line per record."""
    if not records:
        raise InvalidConfig("no records to write")
    body = [_HEADER] + [",".join(enc(getattr(rec, name)) for name, enc, _ in _SCHEMA) for rec in records]
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("\n".join(body) + "\n")


def load_records(path: str) -> list[BenchRecord]:
    """Parse a record file; ``ParseError`` names the failing line."""
    with open(path, "r", encoding="utf-8") as fh:
        lines = fh.read().split("\n")
    if lines[0].strip() != _HEADER:
        raise ParseError(f"unexpected header {lines[0].strip()!r}", 1)
    out = []
    width = len(_SCHEMA)
    for number, text in enumerate(lines[1:], start=2):
        if not text:
            continue
        cells = text.split(",", width - 1)  # the trailing error text may contain commas
        if len(cells) != width:
            raise ParseError(f"expected {width} columns, got {len(cells)}", number)
        try:
            values = {name: dec(cell) for (name, _, dec), cell in zip(_SCHEMA, cells)}
        except ValueError as exc:
            raise ParseError(str(exc), number) from exc
        out.append(BenchRecord(**values))
    return out


def bootstrap_half_width(times, seed: int = 0, resamples: int = 1000) -> float:
    """Half width of the 95 % percentile-bootstrap interval of the mean."""
    sample = np.asarray(times, dtype=np.float64).ravel()
    if not sample.size:
        raise InvalidConfig("need at least one sample")
    draws = np.random.default_rng(seed).integers(0, sample.size, size=(resamples, sample.size))
    boot_means = np.take(sample, draws).mean(axis=1)
    q_lo, q_hi = np.percentile(boot_means, [2.5, 97.5])
    return float(0.5 * (q_hi - q_lo))


# ---- execution ----------------------------------------------------------------------
def make_benchmark_data(n_train: int, n_test: int, regressors: int, seed: int) -> tuple[Dataset, Dataset]:
    """Train/test split of one BASELINE trajectory (identical arrays per seed)."""
    return make_msd_dataset(n_train, n_test, regressors, seed=seed)


_CALLS = {
    "optimize": lambda m, test: m.optimize(AdamConfig(iterations=OPTIMIZE_ITERATIONS)),
    "predict": lambda m, test: m.predict(test),
    "predict_full_cov": lambda m, test: m.predict_with_full_cov(test),
    "predict_var": lambda m, test: m.predict_variance(test),
}


def _run_operation(op: str, train: Dataset, test: Dataset, tiles: int) -> None:
    """One library-user call: a fresh model, then the operation."""
    _CALLS[op](GPModel(train, KernelParams(), tiles_per_dim=tiles), test)


def _time_cell(spec: ExperimentSpec, train, test, tiles: int) -> list[float]:
    for _ in range(spec.warmup):
        _run_operation(spec.operation, train, test, tiles)
    laps = []
    for _ in range(spec.repetitions):
        start = time.perf_counter()
        _run_operation(spec.operation, train, test, tiles)
        laps.append(time.perf_counter() - start)
    return laps


def run_experiment(spec: ExperimentSpec, device: int | None = None) -> list[BenchRecord]:
    """Every (worker count, tiling) cell under its own runtime; a failing cell
    becomes an error record and the sweep goes on."""
    train, test = make_benchmark_data(spec.n_train, spec.n_test, spec.regressors, spec.seed)
    shared = {k: getattr(spec, k) for k in ("operation", "n_train", "n_test", "regressors",
                                            "repetitions", "warmup", "seed")}
    records = []
    for workers, tiles in itertools.product(spec.worker_count, spec.tiles_per_dim):
        cell = dict(shared, tiles_per_dim=tiles, worker_count=workers)
        start_runtime(RuntimeConfig(worker_count=workers, device=device))
        try:
            laps = _time_cell(spec, train, test, tiles)
            stats = dict(mean_s=float(np.mean(laps)),
                         ci_half_width_s=bootstrap_half_width(laps, seed=spec.seed),
                         raw_times_s=tuple(laps))
        except TaskGPError as exc:
            stats = dict(mean_s=math.nan, ci_half_width_s=math.nan, raw_times_s=(),
                         error=f"{type(exc).__name__}: {exc}")
        finally:
            stop_runtime()
        records.append(BenchRecord(**cell, **stats))
    if spec.output_path:
        emit_csv(records, spec.output_path)
    return records


# ---- summary text ------------------------------------------------------------------
def _speedups(records, group_by: str, vary: str, title: str) -> list[str]:
    groups: dict[int, list[BenchRecord]] = {}
    for rec in records:
        groups.setdefault(getattr(rec, group_by), []).append(rec)
    label = {"worker_count": "workers", "tiles_per_dim": "tiles"}
    text = []
    for key in sorted(groups):
        members = sorted(groups[key], key=lambda r: getattr(r, vary))
        slowest = max(r.mean_s for r in members)
        text.append(f"{label[group_by]}={key}: {title} speedup vs slowest")
        text += [f"  {label[vary]}={getattr(r, vary)}: {r.mean_s:.4f}s (+-{r.ci_half_width_s:.4f}) "
                 f"speedup {slowest / r.mean_s:.2f}" for r in members]
    return text


def summarize(records: list[BenchRecord]) -> str:
    """Self-relative speedup tables over worker counts and tilings."""
    if not records:
        raise InvalidConfig("no records to summarize")
    ops = sorted({r.operation for r in records})
    sizes = sorted({r.n_train for r in records})
    if len(ops) != 1 or len(sizes) != 1:
        raise InvalidConfig(f"records mix operations {ops} or sizes {sizes}")
    good = [r for r in records if r.error is None]
    head = records[0]
    text = [f"operation={head.operation} n_train={head.n_train} n_test={head.n_test}"]
    text += _speedups(good, "tiles_per_dim", "worker_count", "parallel")
    text += _speedups(good, "worker_count", "tiles_per_dim", "tiling")
    text += [f"FAILED workers={r.worker_count} tiles={r.tiles_per_dim}: {r.error}"
             for r in records if r.error is not None]
    return "\n".join(text)
