#!/usr/bin/env python
"""Benchmark of the B200 tiled-GP hot path (BASELINE.json metric).

Metric: "tiled Cholesky FP64 TFLOP/s (n=32768) and predict+variance test
points/s" on BASELINE config 2 (n_train = n_test = 32768, 128 regressors,
64 tiles of 512), synthetic data from the BASELINE.json generator.

One step = one pass of the hot path over the config-2 inputs already
resident in HBM: assemble K (SEK tiles) -> tiled Cholesky -> alpha solves +
loss -> predict_with_uncertainty for all 32768 test points.  ``value`` is the
Cholesky rate (LAPACK flop count n^3/3 + n^2/2 + n/6 over the factorisation's
device time, K resident in HBM); ``predict_variance`` the
test points/s of the prediction phase; both measured with CUDA events on the
library's own stream.  ``e2e`` repeats the metric through the public API
with host buffers (H2D of z, y, zt and D2H of the loss, mean and variance
inside the timed region).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun): strong scaling of BASELINE config 3 (n = 65536, the same n
at every N; GPB_BENCH_CONFIG=4: config 4, n = 131072) factored 2D
block-cyclic by the library's multi-GPU runtime (csrc/dist.cu: its own NCCL
world / row / column communicators, schedule replayed from resident job
tables); value = total n^3/3 flops over the slowest rank's factorisation
time.  The N = 1 line carries the 1-GPU time of that workload
("strong_scaling_base") for E(p) = t_1 / (p t_p), and every rank of the
8-GPU 2 x 4 grid emulated alone on the GPU (no-op collectives: a measured
upper bound on E(8); then with every collective charged a modelled NVLink
transfer time).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tiled Cholesky FP64 TFLOP/s (n=32768) and predict+variance test points/s"
CFG = {"n": 32768, "m": 32768, "d": 128, "tiles": 64}
if os.environ.get("GPB_BENCH_SMALL"):  # plumbing checks only (tests); never a bench number
    CFG = {"n": 4096, "m": 1024, "d": 8, "tiles": 8}
WORKLOAD = ("config 2: n_train=32768, n_test=32768, n_regressors=128, 64 tiles of 512, FP64; "
            "step = SEK assembly + tiled Cholesky + alpha solves + loss + predict_with_uncertainty")
DATA = "synthetic: BASELINE.json mass-spring-damper generator, seed 0 (stands in for the paper's MSD data)"


def workload_config(world: int) -> dict:
    """The `config` object of the bench line (both arms print the same one)."""
    if world == 1:
        return {"workload": WORKLOAD, "l2": "inputs larger than L2 (lower K tiles 4.36 GB, "
                "cross-covariance 8.6 GB per step)", "parallelism": "single GPU"}
    c = strong_cfg()
    p, q = _grid(world)
    return {"workload": f"config 3 strong scaling: n_train={c['n']}, n_regressors={c['d']}, {c['tiles']} tiles "
                        "of 512, FP64; step = SEK assembly + tiled Cholesky + alpha solve + loss "
                        "(same n at every GPU count)",
            "l2": "inputs larger than L2 (lower K tiles 17.3 GB)",
            "parallelism": f"2D block-cyclic {p}x{q} tile grid, NCCL panel broadcasts on row/column communicators"}


def _grid(world: int):
    p = int(math.isqrt(world))
    while world % p:
        p -= 1
    return p, world // p


def strong_cfg() -> dict:
    """BASELINE config 3 (GPB_BENCH_CONFIG=4: config 4's n = 131072, D = 16, T = 256)."""
    if os.environ.get("GPB_BENCH_SMALL"):
        return {"n": 4096, "d": 8, "tiles": 8}
    if os.environ.get("GPB_BENCH_CONFIG") == "4":
        return {"n": 131072, "m": 8192, "d": 16, "tiles": 256}
    return {"n": 65536, "d": 8, "tiles": 128}


def chol_flops(n: int) -> float:
    return n ** 3 / 3.0 + n ** 2 / 2.0 + n / 6.0


def pred_flops_per_point(n: int, d: int) -> float:
    # n^2 (triangular solve) + 2n (mean) + 2n (sum of squares) + n(3D+2) (SEK)
    return n * n + 4.0 * n + n * (3.0 * d + 2.0)


# ---------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(self.device), "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[5:9]):
                if flag.lower().startswith("active"):
                    reasons.add(name)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def _ncu_traffic(name="r02_gemm_traffic.json"):
    """DRAM bytes per launch of a kernel from its committed ncu --set full
    capture (profiles/<name>), or None."""
    path = os.path.join(ROOT, "profiles", name)
    try:
        with open(path) as f:
            return json.load(f)["traffic_bytes_per_launch"]
    except (OSError, KeyError, ValueError):
        return None


def _measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


# ---------------------------------------------------------------- CPU side
# The CPU arm runs the reference itself when it is importable: taskgp 0.1.0
# installed into baseline/_ref (pip install --target, git-ignored, travels to
# the GPU box), through its public API with the protocol of BASELINE.md 3 /
# start_runtime(RuntimeConfig(worker_count = all host cores))
# (BLAS pinned to one thread per worker by the runtime, runtime.py:180-181) and
# a fresh GPModel per repetition whose log_likelihood() assembles K, factors it
# and runs the alpha solves -- the same work as the GPU arm's e2e
# compute_loss().  Without it, the oracle port (oracle/tiled_gp.py, the same
# tile algorithm: threaded assembly + ThreadedCholesky + blocked solves) runs.
#
# Sample: config 2 halved -- n = 16384, D = 128, 32 tiles of 512 (config 2's
# tile size and feature count).  A full config-2 step takes ~2 min of taskgp
# on the GPU box's 16 cores, so K + W of them do not fit the bench's few
# minutes; the GPU arm reports its own rate on this same sample
# ("e2e_at_cpu_sample") for the like-for-like ratio.
CPU_SAMPLE = {"n": 16384, "d": 128, "tiles": 32}   # N = 1: config 2 halved
CPU_SAMPLE_STRONG = {"n": 16384, "d": 8, "tiles": 32}  # N > 1: config 3 quartered
if os.environ.get("GPB_BENCH_SMALL"):
    CPU_SAMPLE = CPU_SAMPLE_STRONG = {"n": 2048, "d": 8, "tiles": 4}


def _taskgp():
    """The reference package from baseline/_ref, or None."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "taskgp")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    try:
        import taskgp
        from taskgp.model import GPModel  # noqa: F401
    except Exception:
        return None
    return taskgp


class CpuArm:
    """One step = assemble + factor + alpha solves of the CPU sample, the
    reference's own code path when available."""

    def __init__(self, sample=None):
        from paper_2505_00136_b200.data import make_msd_dataset

        c = sample or CPU_SAMPLE
        self.n, self.d, self.tiles = c["n"], c["d"], c["tiles"]
        self.train, _ = make_msd_dataset(self.n, 0, self.d, seed=0)
        self.workers = len(os.sched_getaffinity(0))
        self.tg = _taskgp()
        self.kind = "reference" if self.tg else "port"
        if self.tg:
            self.tg.start_runtime(self.tg.RuntimeConfig(worker_count=self.workers))
            self.ds = self.tg.Dataset(self.train.z, self.train.y)

    def step(self) -> float:
        t0 = time.perf_counter()
        if self.tg:
            from taskgp.model import GPModel

            GPModel(self.ds, self.tg.KernelParams(1.0, 1.0, 0.1), tiles_per_dim=self.tiles).log_likelihood()
        else:
            from oracle.tiled_gp import OracleGP, ThreadedCholesky

            OracleGP(self.train.z, self.train.y, self.tiles, cholesky=ThreadedCholesky(self.workers),
                     assembly_workers=self.workers).log_likelihood()
        return time.perf_counter() - t0

    def close(self):
        if self.tg:
            self.tg.stop_runtime()

    def describe(self, seconds: float) -> str:
        who = ("taskgp 0.1.0 (the reference, baseline/_ref) GPModel(train, KernelParams(1, 1, 0.1), "
               f"tiles_per_dim={self.tiles}).log_likelihood() under start_runtime(worker_count={self.workers})"
               if self.tg else
               f"oracle port of taskgp (threaded assembly + ThreadedCholesky + blocked solves, {self.workers} "
               "workers x 1 BLAS thread)")
        return (f"{who}: SEK assembly + tiled Cholesky + alpha solves at n={self.n}, D={self.d}, "
                f"{self.tiles} tiles of {self.n // self.tiles}, {seconds:.1f} s per step; "
                "flops counted as n^3/3 + n^2/2 + n/6")


def run_reference(args, rank: int):
    if rank != 0:
        return
    arm = CpuArm(CPU_SAMPLE if args.gpus == 1 else CPU_SAMPLE_STRONG)
    try:
        times = []
        for it in range(args.warmup + args.steps):
            dt = arm.step()
            if it >= args.warmup:
                times.append(dt)
    finally:
        arm.close()
    tf = len(times) * chol_flops(arm.n) / sum(times) / 1e12
    sample = arm.describe(sum(times) / len(times))
    line = {"metric": METRIC, "value": tf, "unit": "TFLOP/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
            "higher_is_better": True, "scaling": "strong" if args.gpus > 1 else "weak", "vs_baseline": None,
            "dtype": "f64", "data": DATA, "config": workload_config(args.gpus), "impl": "reference",
            "sample": sample,
            "cpu_baseline": {"value": tf, "unit": "TFLOP/s", "cores": arm.workers, "kind": arm.kind,
                             "sample": sample},
            "e2e": {"value": tf, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline_block():
    """One bounded step of the CPU arm (rank 0, N = 1)."""
    arm = CpuArm()
    try:
        dt = arm.step()
    finally:
        arm.close()
    return {"value": chol_flops(arm.n) / dt / 1e12, "unit": "TFLOP/s", "cores": arm.workers,
            "kind": arm.kind, "sample": arm.describe(dt)}


# ---------------------------------------------------------------- GPU side
def roofline_block(planes, pairs, planes_tf, planes_tf_exec, gemm_tf, gemm_tf_exec, fp64_peak, kcnt, kbusy, kms,
                   total_ms, chol_tf, clk=None, int8_probe=None):
    """`roofline` of the bench line for the step's dominant kernel."""
    dmma = {"kernel": "dgemm_tma_kernel (TMA-fed DMMA.8x8x4)", "achieved": gemm_tf, "peak": fp64_peak,
            "unit": "TFLOP/s", "frac": gemm_tf / fp64_peak if fp64_peak else None,
            "achieved_executed_flops": gemm_tf_exec, "launches": int(kcnt[0]), "busy_ms": kbusy[0],
            "summed_launch_ms": kms[0], "share_of_step": kbusy[0] / total_ms if total_ms else None,
            "peak_source": "in-run FP64 DMMA probe (MEASURED_PEAKS.json has no FP64 entry)"}
    basis = ("algorithmic flops n^3/3 + n^2 m per step, split between the two tensor-kernel classes in "
             "proportion to their executed flops, over each class's busy time: the union of its launch "
             "intervals on both streams (CUDA events around every launch), so overlapping launches count once")
    if not planes or not kbusy[5]:
        dmma.update({"bound": "tensor", "traffic": _ncu_traffic(), "achieved_basis": basis,
                     "traffic_source": "profiles/r02_gemm_traffic.json (ncu --set full of the prediction-sweep "
                                       "GEMM; not measured in this run)",
                     "cholesky_frac_of_peak": chol_tf / fp64_peak if fp64_peak else None})
        return dmma
    mp = _measured_peaks()
    # MEASURED_PEAKS.json has no int8 figure, so (as for FP64) the denominator is an in-run probe:
    # tcgen05.mma kind::i8 128 x 128 x 32 issued back to back from shared memory on every SM, no
    # global traffic, best of three ~80 ms bursts.  Twice the measured cuBLAS bf16 rate (the int8
    # pipe's nominal ratio) is reported beside it.
    at_max = bool(clk and clk.get("sm_mhz") and clk.get("sm_max_mhz") and clk["sm_mhz"] >= 0.95 * clk["sm_max_mhz"])
    key = "bf16_tflops" if at_max and mp.get("bf16_tflops") else "bf16_tflops_sustained"
    bf16 = mp.get(key) or mp.get("bf16_tflops")
    if int8_probe:
        peak, src = int8_probe, ("in-run int8 tcgen05 probe (MEASURED_PEAKS.json has no int8 entry): 128 x 128 x 32 MMAs "
                                 "back to back from shared memory on every SM, best of three ~80 ms bursts")
    elif bf16:
        peak, src = 2.0 * bf16, f"of measured: 2 x MEASURED_PEAKS.json {key}"
    else:
        peak, src = 4500.0, "of nominal: dense int8 peak of B200"
    achieved = planes_tf * pairs
    return {"bound": "tensor",
            "kernel": "ozaki_gemm_kernel (tcgen05.mma kind::i8 on signed 7-bit digit planes, TMEM accumulators)",
            "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak, "frac_of_nominal_int8_dense": achieved / 4500.0,
            "frac_of_2x_measured_bf16": achieved / (2.0 * bf16) if bf16 else None,
            "two_x_measured_bf16": {"key": key, "value": 2.0 * bf16} if bf16 else None,
            "achieved_basis": f"int8 operations per second: {pairs} digit-pair products ({planes} planes per "
                              "operand) per algorithmic FP64 multiply-add; " + basis,
            "peak_source": src,
            "fp64_equivalent_tflops": planes_tf, "fp64_equivalent_executed_tflops": planes_tf_exec,
            "fp64_dmma_peak": fp64_peak,
            "fp64_equivalent_over_dmma_peak": planes_tf / fp64_peak if fp64_peak else None,
            "traffic": _ncu_traffic("r02_planes_traffic.json"),
            "traffic_source": "dram__bytes_read.sum + dram__bytes_write.sum per launch of the digit-plane "
                              "product from the committed ncu --set full capture "
                              "(profiles/r02_planes_traffic.json), not measured in this run",
            "launches": int(kcnt[5]), "busy_ms": kbusy[5], "summed_launch_ms": kms[5],
            "share_of_step": kbusy[5] / total_ms if total_ms else None,
            "cholesky_fp64_equivalent_over_dmma_peak": chol_tf / fp64_peak if fp64_peak else None,
            "dmma_class": dmma}


def run_ours(args, rank: int, world: int, local_rank: int):
    import numpy as np
    import torch

    import paper_2505_00136_b200 as gpb
    from paper_2505_00136_b200 import _lib

    dist = None
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    torch.cuda.set_device(local_rank)
    lib = _lib.load()
    n, m, d, tiles = CFG["n"], CFG["m"], CFG["d"], CFG["tiles"]
    train, test = gpb.make_msd_dataset(n, m, d, seed=0)
    rt = gpb.start_runtime(gpb.RuntimeConfig(device=local_rank))
    peak = ctypes.c_double()
    _lib.check(lib.gpb_fp64_peak_probe(rt.handle, 1.0, ctypes.byref(peak)))
    peak_i8 = ctypes.c_double()
    _lib.check(lib.gpb_int8_peak_probe(rt.handle, 0.25, ctypes.byref(peak_i8)))

    # inputs resident in HBM (torch tensors are buffers only)
    z_dev = torch.from_numpy(train.z).cuda()
    y_dev = torch.from_numpy(train.y).cuda()
    zt_dev = torch.from_numpy(test.z).cuda()
    mean_dev = torch.empty(m, dtype=torch.float64, device="cuda")
    var_dev = torch.empty(m, dtype=torch.float64, device="cuda")
    h = ctypes.c_void_p()
    _lib.check(lib.gpb_model_create_device(rt.handle, ctypes.c_void_p(z_dev.data_ptr()),
                                           ctypes.c_void_p(y_dev.data_ptr()), n, d, tiles,
                                           ctypes.byref(h)))
    sptr = ctypes.c_void_p()
    lib.gpb_model_stream(h, ctypes.byref(sptr))
    stream = torch.cuda.ExternalStream(sptr.value)
    flags = (ctypes.c_uint8 * 3)(1, 1, 1)
    ll = ctypes.c_double()

    def step():
        _lib.check(lib.gpb_model_set_params(h, 1.0, 1.0, 0.1, flags))  # invalidates the factor
        _lib.check(lib.gpb_cholesky(h, None))
        _lib.check(lib.gpb_log_likelihood(h, ctypes.byref(ll)))
        _lib.check(lib.gpb_predict_device(h, ctypes.c_void_p(zt_dev.data_ptr()), m, d,
                                          ctypes.c_void_p(mean_dev.data_ptr()),
                                          ctypes.c_void_p(var_dev.data_ptr())))

    for _ in range(args.warmup):
        step()
    tm = (ctypes.c_double * 8)()
    lc0, lc1 = ctypes.c_int64(), ctypes.c_int64()
    phase = np.zeros(8)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local_rank)
    clocks.start()
    _lib.check(lib.gpb_model_set_profiling(h, 1))
    lib.gpb_model_launch_count(h, ctypes.byref(lc0))
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
        lib.gpb_model_timings(h, tm, 8)
        phase += np.array(tm[:])
    ev1.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    lib.gpb_model_launch_count(h, ctypes.byref(lc1))
    kms, kfl, kcnt = (ctypes.c_double * 8)(), (ctypes.c_double * 8)(), (ctypes.c_int64 * 8)()
    kbusy = (ctypes.c_double * 8)()
    lib.gpb_model_kernel_stats(h, kms, kfl, kcnt)
    lib.gpb_model_kernel_busy(h, kbusy)
    lib.gpb_model_set_profiling(h, 0)
    total_ms = ev0.elapsed_time(ev1)
    factor_ms, pred_ms = phase[1], phase[3] + phase[4]
    if dist:
        t = torch.tensor([total_ms, factor_ms, pred_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, factor_ms, pred_ms = t.tolist()
    K = args.steps
    value = world * K * chol_flops(n) / (factor_ms * 1e-3) / 1e12
    pts = world * K * m / (pred_ms * 1e-3)
    # roofline.achieved from ALGORITHMIC flops: the step's GEMM work is the
    # Cholesky trailing updates and panel solves (n^3/3) plus the prediction
    # triangular solve (n^2 m); POTRF/TRTRI tiles (2 b^3/3 each, <0.1%) are
    # not GEMM work.  Time base: the GEMM class's BUSY time, i.e. the length
    # of the union of its launch intervals over both streams (CUDA events
    # around every launch on its stream), so overlapping launches of the
    # critical and main streams are not double-counted.  The executed count
    # (with the lower-triangular waste of 128-blocks) is reported beside it.
    gemm_alg = K * (n ** 3 / 3.0 + float(n) * n * m)
    # Two tensor-kernel classes share that work: the tcgen05 int8 digit-plane
    # products (class 5: trailing updates with K >= 1024 and prediction rows
    # with K >= 2048) and the FP64 DMMA GEMM (class 0: everything shorter).
    # The algorithmic flops are split between them in proportion to the
    # executed flops each class reports.
    planes_h = ctypes.c_int()
    lib.gpb_model_get_ozaki(h, ctypes.byref(planes_h), None)
    planes = int(planes_h.value)
    pairs = planes * (planes + 1) // 2
    exec_total = kfl[0] + kfl[5]
    alg_dmma = gemm_alg * kfl[0] / exec_total if exec_total else 0.0
    alg_planes = gemm_alg * kfl[5] / exec_total if exec_total else 0.0
    gemm_tf = alg_dmma / (kbusy[0] * 1e-3) / 1e12 if kbusy[0] else 0.0
    gemm_tf_exec = kfl[0] / (kbusy[0] * 1e-3) / 1e12 if kbusy[0] else 0.0
    planes_tf = alg_planes / (kbusy[5] * 1e-3) / 1e12 if kbusy[5] else 0.0
    planes_tf_exec = kfl[5] / (kbusy[5] * 1e-3) / 1e12 if kbusy[5] else 0.0
    main_stats = {"kms": list(kms), "kbusy": list(kbusy), "kcnt": list(kcnt)}

    # ---- the same step with every product on the FP64 DMMA kernels (planes off)
    dmma_only = None
    if planes and world == 1 and not args.no_dmma_only:
        _lib.check(lib.gpb_model_set_ozaki(h, 0))
        step()
        k2 = max(2, min(3, K))
        ph2 = np.zeros(8)
        _lib.check(lib.gpb_model_set_profiling(h, 1))
        for _ in range(k2):
            step()
            lib.gpb_model_timings(h, tm, 8)
            ph2 += np.array(tm[:])
        torch.cuda.synchronize()
        lib.gpb_model_kernel_stats(h, kms, kfl, kcnt)
        lib.gpb_model_kernel_busy(h, kbusy)
        lib.gpb_model_set_profiling(h, 0)
        d_tf = k2 * chol_flops(n) / (ph2[1] * 1e-3) / 1e12
        d_gemm = k2 * (n ** 3 / 3.0 + float(n) * n * m) / (kbusy[0] * 1e-3) / 1e12 if kbusy[0] else 0.0
        dmma_only = {
            "note": "GPB_OZAKI=0 / digit_planes = 0: the same step with every product on the FP64 tensor "
                    "pipe (DMMA.8x8x4), the path BASELINE.json's north_star names",
            "steps": k2, "value": d_tf, "unit": "TFLOP/s",
            "cholesky_frac_of_fp64_peak": d_tf / peak.value if peak.value else None,
            "predict_variance_points_per_s": k2 * m / ((ph2[3] + ph2[4]) * 1e-3),
            "phases_ms_per_step": {k: float(ph2[i] / k2) for i, k in enumerate(
                ("assembly", "factor", "solves", "cross_mean", "trsm_variance"))},
            "gemm_roofline": {"achieved": d_gemm, "peak": peak.value, "unit": "TFLOP/s",
                              "frac": d_gemm / peak.value if peak.value else None,
                              "basis": "algorithmic flops n^3/3 + n^2 m over the DMMA GEMM busy time",
                              "traffic": _ncu_traffic(),
                              "traffic_source": "profiles/r02_gemm_traffic.json (ncu --set full, prediction-sweep "
                                                "GEMM; not measured in this run)"}}
        _lib.check(lib.gpb_model_set_ozaki(h, planes))
    kms, kbusy, kcnt = main_stats["kms"], main_stats["kbusy"], main_stats["kcnt"]

    # ---- the same sizes on a DENSE covariance (D = 8).  Config 2's 128-feature K is nearly
    # diagonal, so most digits of its planes are zero and the int8 pipe draws
    # less power; on dense operands the chip touches its power cap and the digit-plane phases
    # run slower (the FP64 DMMA path does not care).  Reported beside the headline for context.
    dense = None
    if planes and world == 1 and not args.no_dense_check:
        d8 = 8
        tr8, te8 = gpb.make_msd_dataset(n, m, d8, seed=0)
        z8, y8, zt8 = (torch.from_numpy(a).cuda() for a in (tr8.z, tr8.y, te8.z))
        h8 = ctypes.c_void_p()
        _lib.check(lib.gpb_model_create_device(rt.handle, ctypes.c_void_p(z8.data_ptr()), ctypes.c_void_p(y8.data_ptr()),
                                               n, d8, tiles, ctypes.byref(h8)))
        ph8 = np.zeros(8)
        reps8 = 2
        for it in range(1 + reps8):
            _lib.check(lib.gpb_model_set_params(h8, 1.0, 1.0, 0.1, flags))
            _lib.check(lib.gpb_cholesky(h8, None))
            _lib.check(lib.gpb_log_likelihood(h8, ctypes.byref(ll)))
            _lib.check(lib.gpb_predict_device(h8, ctypes.c_void_p(zt8.data_ptr()), m, d8,
                                              ctypes.c_void_p(mean_dev.data_ptr()), ctypes.c_void_p(var_dev.data_ptr())))
            lib.gpb_model_timings(h8, tm, 8)
            if it >= 1:
                ph8 += np.array(tm[:])
        lib.gpb_model_destroy(h8)
        dense = {"workload": f"n_train = n_test = {n}, n_regressors = {d8}, {tiles} tiles: dense K (config 2's sizes)",
                 "steps": reps8, "cholesky_tflops": reps8 * chol_flops(n) / (ph8[1] * 1e-3) / 1e12,
                 "predict_variance_points_per_s": reps8 * m / ((ph8[3] + ph8[4]) * 1e-3),
                 "factor_ms": float(ph8[1] / reps8), "trsm_variance_ms": float(ph8[4] / reps8),
                 "note": "data-dependent power: with dense digit planes the SM clock dips under sw_power_cap during "
                         "the int8 products (profiles/r02_planes_dense_clocks.txt)"}

    # ---- e2e: public API, host buffers, copies inside the timed region
    # inputs live in pinned host memory (the API's H2D copies read them there)
    def pinned(a):
        t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
        t.numpy()[...] = a
        return t.numpy()

    train_h = gpb.Dataset(pinned(train.z), pinned(train.y))
    test_h = gpb.Dataset(pinned(test.z), pinned(test.y))

    def e2e_reps(tr, te, t, reps):
        chol, pred = [], []
        for _ in range(reps):
            t0 = time.perf_counter()
            model = gpb.GPModel(tr, gpb.KernelParams(1.0, 1.0, 0.1), t)
            model.compute_loss()  # H2D z, y; assemble; factor; solves; D2H loss terms
            t1 = time.perf_counter()
            if te is not None:
                model.predict_with_uncertainty(te)  # H2D zt; predict; D2H mean + var
            t2 = time.perf_counter()
            chol.append(t1 - t0)
            pred.append(t2 - t1)
            model.close()
        return chol, pred

    e2e_chol, e2e_pred = e2e_reps(train_h, test_h, tiles, K) if rank == 0 else ([], [])
    # the GPU arm on the CPU arm's sample (like-for-like ratio at the same n)
    same = None
    if rank == 0 and world == 1:
        cs = CPU_SAMPLE
        tr_s, _ = gpb.make_msd_dataset(cs["n"], 0, cs["d"], seed=0)
        tr_s = gpb.Dataset(pinned(tr_s.z), pinned(tr_s.y))
        e2e_reps(tr_s, None, cs["tiles"], 2)  # warm-up of that shape
        sc, _ = e2e_reps(tr_s, None, cs["tiles"], K)
        same = {"n": cs["n"], "d": cs["d"], "tiles": cs["tiles"], "unit": "TFLOP/s",
                "value": chol_flops(cs["n"]) / statistics.median(sc) / 1e12,
                "api": "GPModel(train).compute_loss(), host numpy in pinned memory (assembly + factor + "
                       "solves + copies), median of K reps"}
    lib.gpb_model_destroy(h)
    base = None
    if not args.no_strong_base:
        base = strong_base(args)
    rt.stop()
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": total_ms / K, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": DATA,
        "config": workload_config(1),
        "predict_variance": {"value": pts, "unit": "test points/s",
                             "tflops": pts * pred_flops_per_point(n, d) / 1e12},
        "phases_ms_per_step": {k: float(phase[i] / K) for i, k in enumerate(
            ("assembly", "factor", "solves", "cross_mean", "trsm_variance"))},
        # the Cholesky rate also with assembly included, and
        # predict+variance also cold (assembly + factor + solves + prediction)
        "cholesky_with_assembly_tflops": world * K * chol_flops(n) / (float(phase[0] + phase[1]) * 1e-3) / 1e12
        if world == 1 else None,
        "predict_variance_cold_points_per_s": world * K * m / (float(sum(phase[:5])) * 1e-3)
        if world == 1 else None,
        "e2e": {"value": chol_flops(n) / statistics.median(e2e_chol) / 1e12 if e2e_chol else None,
                "unit": "TFLOP/s",
                "predict_variance_points_per_s": m / statistics.median(e2e_pred) if e2e_pred else None,
                "h2d_bytes_per_step": 8 * (n * d + n + m * d), "d2h_bytes_per_step": 8 * (2 + 2 * m),
                "api": "GPModel(train).compute_loss() then predict_with_uncertainty(test), host numpy "
                       "arrays in pinned memory, median of K reps"},
        "e2e_at_cpu_sample": same,
        "roofline": roofline_block(planes, pairs, planes_tf, planes_tf_exec, gemm_tf, gemm_tf_exec, peak.value,
                                   kcnt, kbusy, kms, total_ms, value / world, clk, peak_i8.value),
        "dmma_only": dmma_only,
        "dense_k_check": dense,
        "digit_planes": planes,
        "arithmetic": ("FP64 inputs, outputs and accumulation across updates; long contractions (trailing updates, "
                       "prediction sweep) as exact int32 sums of int8 digit-plane products on tcgen05 "
                       f"({planes} signed 7-bit planes per operand, dropped tail < 2^-53 of the operand scales), "
                       "everything else FP64 (DMMA / DFMA); parity with the FP64 oracle is tested at the bench "
                       "sizes (factor <= 1e-10, loss / mean / variance <= 1e-9)") if planes else
                      "FP64 throughout (DMMA / DFMA)",
        "kernel_classes_ms": {"gemm_dmma": kms[0], "digit_plane_products": kms[5], "potrf_trtri": kms[1],
                              "sek": kms[2], "solves": kms[3], "slicing_other": kms[4]},
        "clocks": clk,
        "gpu_launches": int(lc1.value - lc0.value),
        "strong_scaling_base": base,
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_block()
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def run_distributed(args, rank: int, world: int, local_rank: int):
    """N > 1: strong scaling -- BASELINE config 3 (n = 65536, D = 8, 128 tiles
    of 512; GPB_BENCH_CONFIG=4: config 4's n = 131072, D = 16, 256 tiles) at
    every N, factored 2D block-cyclic over the P x Q grid by the library's
    multi-GPU runtime (its own NCCL communicators: world, process rows,
    process columns).  One step = SEK assembly + tiled Cholesky + beta / alpha
    solves + loss (config 4 also predict_with_full_cov of its 8192 test points).
    value = the n^3/3 Cholesky flops over the slowest rank's factorisation
    device time (CUDA events on the library's stream, K resident in HBM);
    e2e = the same metric through the public API from host numpy
    (DistributedGP(train).log_likelihood(), wall clock, max over ranks)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2505_00136_b200 as gpb
    from paper_2505_00136_b200.distributed import DistComm, DistributedGP, process_grid

    device = int(os.environ.get("GPB_FORCE_DEVICE", local_rank))
    torch.cuda.set_device(device)
    os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator lines (nranks) on stderr
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    # torch.distributed only bootstraps (the NCCL unique id); the data path is the library's
    dist.init_process_group(os.environ.get("GPB_DIST_BACKEND", "gloo"))
    cfg = strong_cfg()
    n, d, tiles = cfg["n"], cfg["d"], cfg["tiles"]
    m = cfg.get("m", 0)
    train, test = gpb.make_msd_dataset(n, m, d, seed=0)
    rt = gpb.start_runtime(gpb.RuntimeConfig(device=device))
    import ctypes

    from paper_2505_00136_b200 import _lib

    peak = ctypes.c_double()
    _lib.check(_lib.load().gpb_fp64_peak_probe(rt.handle, 1.0, ctypes.byref(peak)))
    comm = DistComm(rt)
    params = gpb.KernelParams(1.0, 1.0, 0.1)
    # device-resident inputs: the model keeps z, y on the GPU; each step re-assembles K
    model = DistributedGP(train, params, tiles, comm=comm)
    rows = []
    clocks = ClockSampler(device)
    for it in range(args.warmup + args.steps):
        if it == args.warmup:
            dist.barrier()
            torch.cuda.synchronize()
            clocks.start()
        model.params = params  # invalidates the factor
        model.log_likelihood()
        t = model.timings
        pred_ms = 0.0
        if m:
            model.predict_with_full_cov(test)
            pred_ms = model.timings["predict_ms"]
        if it >= args.warmup:
            rows.append([t["factor_ms"], t["solve_ms"], pred_ms, t["enqueue_us_per_step"], t["collectives"]])
    torch.cuda.synchronize()
    dist.barrier()
    clk = clocks.stop()
    launches = model.launch_count()
    model.close()
    # e2e through the public API: host numpy in, loss out (construction included)
    walls = []
    for it in range(1 + args.steps):
        dist.barrier()
        t0 = time.perf_counter()
        mm = DistributedGP(train, params, tiles, comm=comm)
        mm.log_likelihood()
        if m:
            mm.predict_with_full_cov(test)
        walls.append(time.perf_counter() - t0)
        mm.close()
    K = args.steps
    a = np.array(rows).sum(axis=0)
    tt = torch.tensor([a[0], a[1], a[2], sum(walls[1:]), a[3] / K], dtype=torch.float64)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    factor_ms, solve_ms, pred_ms, wall, enq = tt.tolist()
    lt = torch.tensor([launches], dtype=torch.float64)
    dist.all_reduce(lt, op=dist.ReduceOp.SUM)
    comm.close()
    if rank == 0:
        p, q = process_grid(world)
        value = K * chol_flops(n) / (factor_ms * 1e-3) / 1e12
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": (factor_ms + solve_ms + pred_ms) / K, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": DATA,
            "config": workload_config(world),
            "phases_ms_per_step": {"factor": factor_ms / K, "solves": solve_ms / K, "full_cov": pred_ms / K},
            "host_enqueue_us_per_panel_step": enq, "collectives_per_factorisation": float(a[4] / K),
            "e2e": {"value": K * chol_flops(n) / wall / 1e12, "unit": "TFLOP/s",
                    "h2d_bytes_per_step": 8 * world * (n * d + n + m * d),
                    "d2h_bytes_per_step": 8 * world * (1 + m * m),
                    "api": "DistributedGP(train).log_likelihood()" + (" then predict_with_full_cov(test)" if m else "")
                           + ", host numpy on every rank, wall clock max over ranks"},
            "gpu_launches": int(lt.item()),
            "clocks": clk,
            "roofline": {"bound": "tensor", "kernel": "tiled Cholesky per GPU (dgemm_tma_kernel dominated)",
                         "achieved": value / world, "peak": peak.value, "unit": "TFLOP/s",
                         "frac": value / world / peak.value if peak.value else None, "traffic": None,
                         "peak_source": "in-run FP64 DMMA probe (MEASURED_PEAKS.json has no FP64 entry)"},
        }
        print(json.dumps(line), flush=True)
    rt.stop()
    dist.destroy_process_group()


EMU_LINK = "12,450"  # modelled NCCL collective over NVLink 5: latency us, GB/s


def strong_base(args):
    """The 1-GPU time of the strong-scaling workload (config 3; same library,
    single-GPU path, bitwise the same factor as the 1x1 grid): t_1 of
    E(p) = t_1 / (p t_p)."""
    import ctypes

    import torch

    import paper_2505_00136_b200 as gpb
    from paper_2505_00136_b200 import _lib

    lib = _lib.load()
    c = strong_cfg()
    train, _ = gpb.make_msd_dataset(c["n"], 0, c["d"], seed=0)
    z = torch.from_numpy(train.z).cuda()
    y = torch.from_numpy(train.y).cuda()
    h = ctypes.c_void_p()
    rt = gpb.current_runtime()
    _lib.check(lib.gpb_model_create_device(rt.handle, ctypes.c_void_p(z.data_ptr()), ctypes.c_void_p(y.data_ptr()),
                                           c["n"], c["d"], c["tiles"], ctypes.byref(h)))
    flags = (ctypes.c_uint8 * 3)(1, 1, 1)
    ll = ctypes.c_double()
    tm = (ctypes.c_double * 8)()
    fac, sol, fac_dmma = [], [], []
    try:
        # t_1 on the library default (digit planes for the long products, as the multi-GPU
        # executor uses for 512-wide tiles); the FP64 DMMA-only time beside it
        for it in range(3):
            _lib.check(lib.gpb_model_set_params(h, 1.0, 1.0, 0.1, flags))
            _lib.check(lib.gpb_log_likelihood(h, ctypes.byref(ll)))
            lib.gpb_model_timings(h, tm, 8)
            if it >= 1:
                fac.append(tm[1])
                sol.append(tm[2])
        planes_h = ctypes.c_int()
        lib.gpb_model_get_ozaki(h, ctypes.byref(planes_h), None)
        if planes_h.value:
            _lib.check(lib.gpb_model_set_ozaki(h, 0))
            for it in range(2):
                _lib.check(lib.gpb_model_set_params(h, 1.0, 1.0, 0.1, flags))
                _lib.check(lib.gpb_log_likelihood(h, ctypes.byref(ll)))
                lib.gpb_model_timings(h, tm, 8)
                if it >= 1:
                    fac_dmma.append(tm[1])
    finally:
        lib.gpb_model_destroy(h)
    f, s_ = statistics.median(fac), statistics.median(sol)
    # every rank of the 8-GPU 2 x 4 grid emulated alone on this GPU (no-op
    # collectives, gpb_dist_init_emulate): its own kernels' device time, so
    # t_8 >= max over ranks and E(8) <= t_1 / (8 max) from measurement.  A
    # second pass makes every collective occupy its stream for a modelled
    # NVLink transfer (GPB_EMU_LINK: latency + bytes / bandwidth) so the
    # schedule's exposure of communication is measured too.
    def emulate(link):
        if link:
            os.environ["GPB_EMU_LINK"] = link
        else:
            os.environ.pop("GPB_EMU_LINK", None)
        per_rank = []
        for r in range(8):
            dc, dm = ctypes.c_void_p(), ctypes.c_void_p()
            _lib.check(lib.gpb_dist_init_emulate(rt.handle, r, 8, 2, 4, ctypes.byref(dc)))
            _lib.check(lib.gpb_dist_model_create(dc, _lib.dptr(train.z), _lib.dptr(train.y), c["n"], c["d"],
                                                 c["tiles"], ctypes.byref(dm)))
            best = None
            for it in range(2):
                _lib.check(lib.gpb_dist_set_params(dm, 1.0, 1.0, 0.1 + 1e-3 * it, flags))
                try:
                    _lib.check(lib.gpb_dist_factor(dm))
                except gpb.errors.NotPositiveDefinite:
                    pass  # the data is meaningless without the exchanges; the schedule ran to the end
                lib.gpb_dist_timings(dm, tm, 8)
                best = tm[1] if best is None else min(best, tm[1])
            lib.gpb_dist_model_destroy(dm)
            lib.gpb_dist_finalize(dc)
            per_rank.append(round(best, 2))
        os.environ.pop("GPB_EMU_LINK", None)
        return per_rank

    per_rank = emulate(None)
    per_rank_link = emulate(EMU_LINK)
    return {"workload": f"config 3 on 1 GPU: n={c['n']}, D={c['d']}, {c['tiles']} tiles", "factor_ms": f,
            "solves_ms": s_, "tflops": chol_flops(c["n"]) / (f * 1e-3) / 1e12,
            "note": "t_1 of the strong-scaling efficiency E(p) = t_1 / (p t_p) (1 warm-up + 2 timed): the "
                    "single-GPU path at its default (long products on the digit planes, 8-panel groups, "
                    "left-looking in-group updates), which is also the multi-GPU executor's schedule for "
                    "512-wide tiles",
            "factor_ms_dmma_only": fac_dmma[0] if fac_dmma else None,
            "tflops_dmma_only": chol_flops(c["n"]) / (fac_dmma[0] * 1e-3) / 1e12 if fac_dmma else None,
            "emulated_2x4_factor_ms_per_rank": per_rank,
            "emulated_2x4_efficiency_upper_bound": f / (8 * max(per_rank)),
            "emulated_2x4_link_factor_ms_per_rank": per_rank_link,
            "emulated_2x4_link_efficiency": f / (8 * max(per_rank_link)),
            "emulation": "each rank of the 2 x 4 grid run alone on this GPU (its kernels' device time, "
                         "no cross-rank waits): with no-op collectives E(8) <= t_1 / (8 max_r t_r) -- a bound "
                         "above 1 says that t_1 itself is not purely throughput-bound (the single-GPU critical "
                         "path shows in it), not that 8 GPUs would scale super-linearly; "
                         f"the 'link' pass charges every collective {EMU_LINK.split(',')[0]} us + "
                         f"bytes / {EMU_LINK.split(',')[1]} GB/s on its stream (modelled NVLink transfer)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-strong-base", action="store_true")
    ap.add_argument("--no-dmma-only", action="store_true", help="skip the extra pass with digit planes off")
    ap.add_argument("--no-dense-check", action="store_true", help="skip the dense-covariance pass (D = 8)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: at least 3 warm-up steps
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", args.gpus))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if world > 1:
        run_distributed(args, rank, world, local_rank)
        return
    run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
