"""Record/CSV layer and dataset IO against fixtures written by the reference
(tests/golden/make_golden_records.py), plus the sweep harness on the GPU.

Mirrors pkg/tests/test_bench.py and the CSV / lag-embedding cases of
pkg/tests/test_data.py.
"""

import json
import math
import os

import numpy as np
import pytest

import paper_2505_00136_b200 as gpb
from paper_2505_00136_b200 import bench
from paper_2505_00136_b200.bench import (
    BenchRecord,
    ExperimentSpec,
    bootstrap_half_width,
    emit_csv,
    load_records,
    run_experiment,
    summarize,
)
from paper_2505_00136_b200.errors import InvalidConfig, ParseError, TaskGPError, TilingError

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def record(**overrides):
    base = dict(operation="predict", n_train=64, n_test=64, regressors=4, tiles_per_dim=1,
                worker_count=1, repetitions=2, warmup=0, seed=0, mean_s=1.0,
                ci_half_width_s=0.1, raw_times_s=(0.9, 1.1))
    base.update(overrides)
    return BenchRecord(**base)


def same(a, b):
    """Record equality with NaN == NaN (failed cells carry NaN timings)."""
    for x, y in zip(a.__dict__.values(), b.__dict__.values()):
        if isinstance(x, float) and math.isnan(x):
            assert isinstance(y, float) and math.isnan(y)
        else:
            assert x == y


class TestAgainstReferenceFixtures:
    def test_reference_csv_loads_and_rewrites_byte_identical(self, tmp_path):
        src = os.path.join(GOLDEN, "ref_records.csv")
        recs = load_records(src)
        assert len(recs) == 7 and recs[-1].error == "TaskGPError: cell exploded, twice"
        out = tmp_path / "again.csv"
        emit_csv(recs, str(out))
        assert out.read_bytes() == open(src, "rb").read()

    def test_summary_text_identical(self):
        recs = load_records(os.path.join(GOLDEN, "ref_records.csv"))
        assert summarize(recs) + "\n" == open(os.path.join(GOLDEN, "ref_summary.txt")).read()

    def test_bootstrap_identical(self):
        ref = json.load(open(os.path.join(GOLDEN, "ref_bootstrap.json")))
        for name, samples in ref["samples"].items():
            for seed, width in ref["half_width"][name].items():
                assert bootstrap_half_width(samples, seed=int(seed)) == width

    def test_dataset_csv_and_lag_embed(self, tmp_path):
        series = np.load(os.path.join(GOLDEN, "ref_dataset_series.npy"))
        ds = gpb.lag_embed(series, gpb.LagSpec(3))
        path = tmp_path / "d.csv"
        gpb.save_csv(ds, str(path), header=True)
        assert path.read_bytes() == open(os.path.join(GOLDEN, "ref_dataset.csv"), "rb").read()
        back = gpb.load_csv(os.path.join(GOLDEN, "ref_dataset.csv"), header=True)
        np.testing.assert_array_equal(back.z, ds.z)
        np.testing.assert_array_equal(back.y, ds.y)


class TestDatasetIO:
    """pkg/tests/test_data.py lag-embedding and CSV cases."""

    def test_lag_embed_known_answer(self):
        ds = gpb.lag_embed([1.0, 2.0, 3.0, 4.0], gpb.LagSpec(2))
        np.testing.assert_array_equal(ds.z, [[2.0, 1.0], [3.0, 2.0]])
        np.testing.assert_array_equal(ds.y, [3.0, 4.0])

    def test_lag_embed_rejects_short_series(self):
        from paper_2505_00136_b200.errors import DimensionMismatch

        with pytest.raises(DimensionMismatch):
            gpb.lag_embed([1.0, 2.0], gpb.LagSpec(2))
        with pytest.raises(InvalidConfig):
            gpb.LagSpec(0)

    @pytest.mark.parametrize("text,line", [("1.0,2.0\n3.0\n", 2), ("1.0,abc\n", 1), ("", 1), ("1.0\n", 1)])
    def test_malformed_files(self, tmp_path, text, line):
        path = tmp_path / "bad.csv"
        path.write_text(text)
        with pytest.raises(ParseError) as info:
            gpb.load_csv(str(path))
        assert info.value.line == line


class TestSpecAndRecords:
    def test_spec_validation(self):
        assert ExperimentSpec().operation == "predict"
        with pytest.raises(InvalidConfig):
            ExperimentSpec(operation="train")
        for n in (0, 3, 100):
            with pytest.raises(InvalidConfig):
                ExperimentSpec(n_train=n)
        with pytest.raises(TilingError):
            ExperimentSpec(n_train=64, tiles_per_dim=(1, 3))
        with pytest.raises(InvalidConfig):
            ExperimentSpec(repetitions=0)
        with pytest.raises(InvalidConfig):
            ExperimentSpec(worker_count=(0,))

    def test_round_trip_and_errors(self, tmp_path):
        path = str(tmp_path / "b.csv")
        original = [record(), record(tiles_per_dim=4, mean_s=0.123456789012345678),
                    record(error="TaskGPError: cell exploded", raw_times_s=())]
        emit_csv(original, path)
        assert load_records(path) == original
        with pytest.raises(InvalidConfig):
            emit_csv([], path)
        (tmp_path / "h.csv").write_text("operation,n_train\n")
        with pytest.raises(ParseError):
            load_records(str(tmp_path / "h.csv"))

    def test_summarize_rules(self):
        assert "speedup 1.00" in summarize([record()])
        text = summarize([record(worker_count=1, mean_s=10.0), record(worker_count=4, mean_s=5.0)])
        assert "workers=4: 5.0000s" in text and "speedup 2.00" in text
        with pytest.raises(InvalidConfig):
            summarize([record(n_train=64), record(n_train=128)])
        text = summarize([record(), record(worker_count=2, error="boom")])
        assert "FAILED" in text and "boom" in text

    def test_failed_cell_recorded_not_raised(self, monkeypatch):
        """bench.py:164-175 semantics, without a device (the runtime calls are stubbed)."""
        calls = []

        def flaky(op, train, test, tiles):
            calls.append(tiles)
            if tiles == 2:
                raise TaskGPError("synthetic failure")

        monkeypatch.setattr(bench, "_run_operation", flaky)
        monkeypatch.setattr(bench, "start_runtime", lambda cfg: None)
        monkeypatch.setattr(bench, "stop_runtime", lambda: None)
        recs = run_experiment(ExperimentSpec(n_train=16, n_test=16, regressors=2,
                                             tiles_per_dim=(1, 2), repetitions=2))
        assert recs[0].error is None and len(recs[0].raw_times_s) == 2
        assert "synthetic failure" in recs[1].error and recs[1].raw_times_s == ()
        same(recs[1], recs[1])

    def test_deterministic_data_per_seed(self):
        a, _ = bench.make_benchmark_data(16, 8, 2, seed=7)
        b, _ = bench.make_benchmark_data(16, 8, 2, seed=7)
        np.testing.assert_array_equal(a.z, b.z)


@pytest.mark.gpu
class TestSweepOnDevice:
    def test_record_count_and_raw_times(self, tmp_path):
        spec = ExperimentSpec(operation="predict", n_train=16, n_test=16, regressors=2,
                              tiles_per_dim=(1, 2), worker_count=(1, 2), repetitions=3, warmup=1,
                              output_path=str(tmp_path / "sweep.csv"))
        recs = run_experiment(spec)
        assert len(recs) == 4
        for rec in recs:
            assert rec.error is None and len(rec.raw_times_s) == 3
            assert rec.mean_s == pytest.approx(np.mean(rec.raw_times_s))
            assert rec.ci_half_width_s >= 0.0
        assert gpb.current_runtime() is None
        assert load_records(spec.output_path) == recs

    @pytest.mark.parametrize("op", ["optimize", "predict_var", "predict_full_cov"])
    def test_all_operations_run(self, op):
        recs = run_experiment(ExperimentSpec(operation=op, n_train=16, n_test=16, regressors=2,
                                             repetitions=1))
        assert recs[0].error is None
