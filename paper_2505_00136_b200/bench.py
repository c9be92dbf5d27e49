"""Timing sweeps with the reference's record format (taskgp bench.py:79-301).

One format for the CPU and GPU tables: the same
``ExperimentSpec`` validation, ``BenchRecord`` fields, percentile-bootstrap
half width, loss-free CSV round trip and ``summarize`` text as the reference
harness, so records written here load with ``taskgp.bench.load_records`` and
vice versa.

Differences, all on the execution side:

* a cell runs on the B200 runtime (``start_runtime`` binds the device);
  ``worker_count`` keeps the reference's validation and is recorded in the
  CSV, but the device path has no host worker pool to size;
* every timed call is one blocking public-API call (``GPModel`` methods
  return host numpy arrays), so the wall-clock repetition times include
  assembly, factorisation and the device-to-host copies, like the
  reference's timing of a library user's call (bench.py:1-9);
* data come from the BASELINE generator (``make_msd_dataset``), which stands
  in for the reference's RK4 trajectory; a fixed seed gives
  identical arrays on every call.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, fields

import numpy as np

from .covariance import KernelParams
from .data import Dataset, make_msd_dataset
from .errors import InvalidConfig, ParseError, TaskGPError, TilingError
from .model import AdamConfig, GPModel
from .runtime import RuntimeConfig, start_runtime, stop_runtime

OPERATIONS = ("optimize", "predict", "predict_full_cov", "predict_var")

# bench.py:25-27: fixed Adam step count so optimisation cells scale with the
# per-iteration cost, not with convergence
OPTIMIZE_ITERATIONS = 3


def _is_power_of_two(n: int) -> bool:
    return n > 0 and (n & (n - 1)) == 0


@dataclass(frozen=True)
class ExperimentSpec:
    """One sweep: an operation crossed with worker counts and tilings
    (validation as bench.py:34-76)."""

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
        if self.operation not in OPERATIONS:
            raise InvalidConfig(f"operation must be one of {OPERATIONS}, got {self.operation!r}")
        for name in ("n_train", "n_test"):
            value = getattr(self, name)
            if not _is_power_of_two(value):
                raise InvalidConfig(f"{name} must be a power of two, got {value}")
        if self.regressors < 1:
            raise InvalidConfig(f"regressors must be >= 1, got {self.regressors}")
        if self.repetitions < 1:
            raise InvalidConfig(f"repetitions must be >= 1, got {self.repetitions}")
        if self.warmup < 0:
            raise InvalidConfig(f"warmup must be >= 0, got {self.warmup}")
        if not self.tiles_per_dim or not self.worker_count:
            raise InvalidConfig("tiles_per_dim and worker_count must be non-empty")
        for t in self.tiles_per_dim:
            if t < 1 or self.n_train % t != 0:
                raise TilingError(f"tiles_per_dim={t} does not divide n_train={self.n_train}")
        for w in self.worker_count:
            if w < 1:
                raise InvalidConfig(f"worker_count entries must be >= 1, got {w}")


@dataclass(frozen=True)
class BenchRecord:
    """Timing result of one sweep cell (field order = CSV column order, bench.py:79-96)."""

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


def make_benchmark_data(n_train: int, n_test: int, regressors: int, seed: int) -> tuple[Dataset, Dataset]:
    """Deterministic train/test split of one simulated trajectory (bench.py:99-108)."""
    return make_msd_dataset(n_train, n_test, regressors, seed=seed)


def _run_operation(op: str, train: Dataset, test: Dataset, tiles: int) -> None:
    """One library-user call per repetition (bench.py:111-120)."""
    model = GPModel(train, KernelParams(), tiles_per_dim=tiles)
    if op == "optimize":
        model.optimize(AdamConfig(iterations=OPTIMIZE_ITERATIONS))
    elif op == "predict":
        model.predict(test)
    elif op == "predict_full_cov":
        model.predict_with_full_cov(test)
    else:
        model.predict_variance(test)


def bootstrap_half_width(times, seed: int = 0, resamples: int = 1000) -> float:
    """Half width of the 95% percentile bootstrap interval of the mean
    (bench.py:123-134: same resampling stream for the same seed)."""
    times = np.asarray(times, dtype=np.float64)
    if times.size == 0:
        raise InvalidConfig("need at least one sample")
    rng = np.random.default_rng(seed)
    idx = rng.integers(0, times.size, size=(resamples, times.size))
    means = times[idx].mean(axis=1)
    lo, hi = np.percentile(means, [2.5, 97.5])
    return float((hi - lo) / 2.0)


def run_experiment(spec: ExperimentSpec, device: int | None = None) -> list[BenchRecord]:
    """Run the sweep; a failing cell becomes an error record (bench.py:137-186).
    The runtime is started per cell and stopped afterwards."""
    train, test = make_benchmark_data(spec.n_train, spec.n_test, spec.regressors, spec.seed)
    records = []
    for workers in spec.worker_count:
        for tiles in spec.tiles_per_dim:
            common = dict(operation=spec.operation, n_train=spec.n_train, n_test=spec.n_test,
                          regressors=spec.regressors, tiles_per_dim=tiles, worker_count=workers,
                          repetitions=spec.repetitions, warmup=spec.warmup, seed=spec.seed)
            start_runtime(RuntimeConfig(worker_count=workers, device=device))
            try:
                for _ in range(spec.warmup):
                    _run_operation(spec.operation, train, test, tiles)
                raw = []
                for _ in range(spec.repetitions):
                    began = time.perf_counter()
                    _run_operation(spec.operation, train, test, tiles)
                    raw.append(time.perf_counter() - began)
            except TaskGPError as exc:
                records.append(BenchRecord(**common, mean_s=float("nan"), ci_half_width_s=float("nan"),
                                           raw_times_s=(), error=f"{type(exc).__name__}: {exc}"))
                continue
            finally:
                stop_runtime()
            records.append(BenchRecord(**common, mean_s=float(np.mean(raw)),
                                       ci_half_width_s=bootstrap_half_width(raw, seed=spec.seed),
                                       raw_times_s=tuple(raw)))
    if spec.output_path:
        emit_csv(records, spec.output_path)
    return records


# -- CSV round trip (bench.py:189-258) -------------------------------------------

_COLUMNS = [f.name for f in fields(BenchRecord)]


def _row(rec: BenchRecord) -> list[str]:
    return [rec.operation, str(rec.n_train), str(rec.n_test), str(rec.regressors),
            str(rec.tiles_per_dim), str(rec.worker_count), str(rec.repetitions), str(rec.warmup),
            str(rec.seed), repr(rec.mean_s), repr(rec.ci_half_width_s),
            ";".join(repr(t) for t in rec.raw_times_s),
            rec.error.replace("\n", " ") if rec.error is not None else ""]


def emit_csv(records: list[BenchRecord], path: str) -> None:
    """Header plus one row per record; floats written with repr (loss-free)."""
    if not records:
        raise InvalidConfig("no records to write")
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(",".join(_COLUMNS) + "\n")
        for rec in records:
            fh.write(",".join(_row(rec)) + "\n")


def load_records(path: str) -> list[BenchRecord]:
    """Read back a CSV written by emit_csv (or by the reference's harness)."""
    records = []
    with open(path, "r", encoding="utf-8") as fh:
        header = fh.readline().strip()
        if header.split(",") != _COLUMNS:
            raise ParseError(f"unexpected header {header!r}", 1)
        for lineno, line in enumerate(fh, start=2):
            line = line.rstrip("\n")
            if not line:
                continue
            parts = line.split(",", maxsplit=len(_COLUMNS) - 1)  # the error text may hold commas
            if len(parts) != len(_COLUMNS):
                raise ParseError(f"expected {len(_COLUMNS)} columns, got {len(parts)}", lineno)
            try:
                records.append(BenchRecord(
                    operation=parts[0], n_train=int(parts[1]), n_test=int(parts[2]),
                    regressors=int(parts[3]), tiles_per_dim=int(parts[4]),
                    worker_count=int(parts[5]), repetitions=int(parts[6]), warmup=int(parts[7]),
                    seed=int(parts[8]), mean_s=float(parts[9]), ci_half_width_s=float(parts[10]),
                    raw_times_s=tuple(float(t) for t in parts[11].split(";") if t),
                    error=parts[12] or None))
            except ValueError as exc:
                raise ParseError(str(exc), lineno) from exc
    return records


def summarize(records: list[BenchRecord]) -> str:
    """Self-relative speedup tables over worker counts and tilings (bench.py:261-301)."""
    if not records:
        raise InvalidConfig("no records to summarize")
    ops = {r.operation for r in records}
    sizes = {r.n_train for r in records}
    if len(ops) > 1 or len(sizes) > 1:
        raise InvalidConfig(f"records mix operations {sorted(ops)} or sizes {sorted(sizes)}")
    ok = [r for r in records if r.error is None]
    lines = [f"operation={records[0].operation} n_train={records[0].n_train} n_test={records[0].n_test}"]
    by_tiles: dict[int, list[BenchRecord]] = {}
    by_workers: dict[int, list[BenchRecord]] = {}
    for rec in ok:
        by_tiles.setdefault(rec.tiles_per_dim, []).append(rec)
        by_workers.setdefault(rec.worker_count, []).append(rec)
    for tiles, group in sorted(by_tiles.items()):
        slowest = max(r.mean_s for r in group)
        lines.append(f"tiles={tiles}: parallel speedup vs slowest")
        for rec in sorted(group, key=lambda r: r.worker_count):
            lines.append(f"  workers={rec.worker_count}: {rec.mean_s:.4f}s "
                         f"(+-{rec.ci_half_width_s:.4f}) speedup {slowest / rec.mean_s:.2f}")
    for workers, group in sorted(by_workers.items()):
        slowest = max(r.mean_s for r in group)
        lines.append(f"workers={workers}: tiling speedup vs slowest")
        for rec in sorted(group, key=lambda r: r.tiles_per_dim):
            lines.append(f"  tiles={rec.tiles_per_dim}: {rec.mean_s:.4f}s "
                         f"(+-{rec.ci_half_width_s:.4f}) speedup {slowest / rec.mean_s:.2f}")
    for rec in records:
        if rec.error is not None:
            lines.append(f"FAILED workers={rec.worker_count} tiles={rec.tiles_per_dim}: {rec.error}")
    return "\n".join(lines)
