"""Golden fixtures for the record/CSV layer, written by the REFERENCE.

Run in the build container only (needs ``/root/reference``):

    python tests/golden/make_golden_records.py

Imports ``taskgp`` from ``/root/reference/pkg/src`` and writes
  ref_records.csv    taskgp.bench.emit_csv of a fixed record list
  ref_summary.txt    taskgp.bench.summarize of the same records
  ref_bootstrap.json taskgp.bench.bootstrap_half_width of fixed samples
  ref_dataset.csv    taskgp.data.save_csv(lag_embed(series, LagSpec(3)), header=True)
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from taskgp import bench, data  # noqa: E402


def records():
    base = dict(operation="predict_var", n_train=64, n_test=32, regressors=4, tiles_per_dim=1,
                worker_count=1, repetitions=3, warmup=1, seed=5, mean_s=1.0,
                ci_half_width_s=0.1, raw_times_s=(0.9, 1.0, 1.1))
    out = []
    for w, t, m in [(1, 1, 2.5), (2, 1, 1.3), (4, 1, 0.7), (1, 4, 1.9), (2, 4, 0.95),
                    (4, 4, 0.123456789012345678)]:
        out.append(bench.BenchRecord(**dict(base, worker_count=w, tiles_per_dim=t, mean_s=m,
                                            raw_times_s=(m * 0.9, m, m * 1.1))))
    out.append(bench.BenchRecord(**dict(base, worker_count=8, tiles_per_dim=4, mean_s=float("nan"),
                                        ci_half_width_s=float("nan"), raw_times_s=(),
                                        error="TaskGPError: cell exploded, twice")))
    return out


if __name__ == "__main__":
    recs = records()
    bench.emit_csv(recs, os.path.join(HERE, "ref_records.csv"))
    with open(os.path.join(HERE, "ref_summary.txt"), "w") as fh:
        fh.write(bench.summarize(recs) + "\n")
    samples = {"five": [1.0, 1.5, 2.0, 0.5, 1.2], "equal": [2.0, 2.0, 2.0, 2.0],
               "one": [3.25], "ramp": list(np.linspace(0.1, 2.0, 17))}
    out = {k: {str(seed): bench.bootstrap_half_width(v, seed=seed) for seed in (0, 3, 11)}
           for k, v in samples.items()}
    with open(os.path.join(HERE, "ref_bootstrap.json"), "w") as fh:
        json.dump({"samples": samples, "half_width": out}, fh, indent=1)
    series = np.sin(np.arange(40) * 0.37) + 0.01 * np.arange(40)
    data.save_csv(data.lag_embed(series, data.LagSpec(3)), os.path.join(HERE, "ref_dataset.csv"),
                  header=True)
    np.save(os.path.join(HERE, "ref_dataset_series.npy"), series)
    print("wrote record fixtures")
