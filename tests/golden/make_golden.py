"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container only (it needs ``/root/reference``):

    python tests/golden/make_golden.py

It imports ``taskgp`` 0.1.0 from ``/root/reference/pkg/src`` and runs its
public ``GPModel`` API (model.py:91-485) on seeded inputs, writing compact
``.npz`` fixtures next to this script.  Large matrices are stored as
checksums (diagonal, column sums, Frobenius norm, seeded entry samples) so
the fixtures stay small; small cases store them whole.

Cases (BASELINE.json configs + the reference test corpus shapes):
  c0        config 0: n=m=1024, D=8, T=4 (b=256), BASELINE generator seed 0
  c1        config 1: n=8192, D=8, T=32 (b=256): loss, gradients, 3 Adam steps
  c2s       config 2 scaled: n=2048, m=512, D=128, T=4 (b=512)
  d8b512    n=4096, m=512, D=8, T=8 (b=512): non-degenerate K at the c2 tile size
  rand_*    random-normal instances as in pkg/tests/test_acceptance.py:28-32
  c3s       config 3 scaled: n=8192, D=8, T=16 (b=512): factor, loss, gradients
  c4s       config 4 scaled: n=8192, m=512, D=16, T=16 (b=512): + full covariance
  accept_grid   test_acceptance.py:35-78 grid (n, m, T) in {16,64,256}x{16,64}x{1,4,8}
                with the reference's dense-oracle values (pkg/tests/oracles.py)
  determinism   test_acceptance.py:135-169 instance, tilings 1 and 4

``python tests/golden/make_golden.py accept_grid determinism large`` regenerates
only the named groups.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import taskgp  # noqa: E402  (the reference)
from taskgp.model import AdamConfig, GPModel  # noqa: E402

from paper_2505_00136_b200.data import make_msd_dataset  # noqa: E402

SAMPLES = 4096


def sample_idx(n_rows, n_cols, seed, lower=False):
    rng = np.random.default_rng(seed)
    r = rng.integers(0, n_rows, SAMPLES)
    c = rng.integers(0, n_cols, SAMPLES)
    if lower:
        r, c = np.maximum(r, c), np.minimum(r, c)
    return r, c


def summarize(prefix, a, out, lower=False, seed=7):
    out[prefix + "_diag"] = np.diagonal(a).copy()
    out[prefix + "_colsum"] = a.sum(axis=0)
    out[prefix + "_fro"] = np.array(np.linalg.norm(a))
    r, c = sample_idx(a.shape[0], a.shape[1], seed, lower)
    out[prefix + "_sr"] = r
    out[prefix + "_sc"] = c
    out[prefix + "_sv"] = a[r, c]


def factor(model):
    return taskgp.run_as_root(lambda: model._ensure_factor().to_dense())


def run_case(name, train, test, t, full_store, do_full_cov=True, do_grad=True,
             adam_iters=0):
    out = {"t": np.array(t)}
    tic = time.perf_counter()
    if full_store:
        out["z"], out["y"] = train.z, train.y
        if test is not None:
            out["zt"] = test.z
    else:  # pin the generator instead of storing inputs
        out["z_head"], out["y_head"] = train.z[:16].copy(), train.y[:16].copy()
        out["z_sum"], out["y_sum"] = np.array(train.z.sum()), np.array(train.y.sum())
        if test is not None:
            out["zt_head"], out["zt_sum"] = test.z[:16].copy(), np.array(test.z.sum())
    model = GPModel(train, taskgp.KernelParams(1.0, 1.0, 0.1), tiles_per_dim=t)
    L = factor(model)
    if full_store:
        out["L"] = L
    else:
        summarize("L", L, out, lower=True)
    out["loglik"] = np.array(model.log_likelihood())
    if test is not None:
        pv = model.predict_variance(test)
        out["mean"], out["var"] = pv.mean, pv.variance
        if do_full_cov:
            fc = model.predict_with_full_cov(test)
            if full_store:
                out["cov"] = fc.full_covariance
            else:
                summarize("cov", fc.full_covariance, out)
    if do_grad:
        out["grads"] = np.array(model.loss_gradients())
    if adam_iters:
        hist = model.optimize(AdamConfig(learning_rate=0.1, iterations=adam_iters))
        out["adam_history"] = np.array(hist)
        p = model.params
        out["adam_params"] = np.array([p.lengthscale, p.vertical_scale, p.noise_variance])
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(f"{name}: {time.perf_counter() - tic:.1f}s  loglik={float(out['loglik']):.15g}")


def _instance(seed, n, m, d=4):
    """pkg/tests/test_acceptance.py:28-32 instance shapes."""
    rng = np.random.default_rng(seed)
    train = taskgp.Dataset(z=rng.normal(size=(n, d)), y=rng.normal(size=n))
    test = taskgp.Dataset(z=rng.normal(size=(m, d)), y=np.zeros(m))
    return train, test


def acceptance_grid():
    """The reference's oracle-equivalence grid (test_acceptance.py:35-78):
    (n, m, T) in {16, 64, 256} x {16, 64} x {1, 4, 8}, reference outputs per
    tiling plus the dense-oracle values the reference test compares them to
    (pkg/tests/oracles.py DenseGP)."""
    sys.path.insert(0, "/root/reference/pkg/tests")
    import oracles  # the reference's dense checker

    out = {}
    tic = time.perf_counter()
    for n in (16, 64, 256):
        for m in (16, 64):
            train, test = _instance(n * 1000 + m, n, m)
            key = f"n{n}_m{m}"
            out[key + "_zsum"] = np.array([train.z.sum(), train.y.sum(), test.z.sum()])
            o = oracles.DenseGP(train.z, train.y, 1.0, 1.0, 0.1)
            out[key + "_dense_L"] = np.linalg.cholesky(o.k_train)
            out[key + "_dense_mean"] = o.predict_mean(test.z)
            out[key + "_dense_cov"] = o.posterior_cov(test.z)
            out[key + "_dense_ll"] = np.array(o.log_likelihood())
            for t in (1, 4, 8):
                k = f"{key}_t{t}"
                model = GPModel(train, taskgp.KernelParams(), tiles_per_dim=t)
                out[k + "_L"] = factor(model)
                full = model.predict_with_full_cov(test)
                var = model.predict_variance(test)
                out[k + "_mean"] = full.mean
                out[k + "_cov"] = full.full_covariance
                out[k + "_var"] = var.variance
                out[k + "_ll"] = np.array(model.log_likelihood())
                out[k + "_grads"] = np.array(model.loss_gradients())
    np.savez_compressed(os.path.join(HERE, "accept_grid.npz"), **out)
    print(f"accept_grid: {time.perf_counter() - tic:.1f}s")


def determinism():
    """test_acceptance.py:135-169: one instance, tilings 1 and 4, reference
    outputs (the GPU test adds more tilings and compares them all)."""
    train, test = _instance(2024, 64, 16)
    out = {"zsum": np.array([train.z.sum(), train.y.sum(), test.z.sum()])}
    for t in (1, 4):
        model = GPModel(train, taskgp.KernelParams(lengthscale=0.9, noise_variance=0.15), tiles_per_dim=t)
        full = model.predict_with_full_cov(test)
        out[f"t{t}_mean"] = full.mean
        out[f"t{t}_cov"] = full.full_covariance
        out[f"t{t}_var"] = model.predict_variance(test).variance
        out[f"t{t}_ll"] = np.array(model.log_likelihood())
    np.savez_compressed(os.path.join(HERE, "determinism.npz"), **out)
    print("determinism: done")


def scaled_large_configs():
    """Scaled shapes of BASELINE configs 3 and 4 at the benchmark tile size
    (b = 512, T = 16): c3s n = 8192, D = 8 (cholesky + alpha solve + loss,
    gradients); c4s n = 8192, m = 512 (config 4's m / n = 1/16), D = 16 with
    full covariance and gradients."""
    tr, _ = make_msd_dataset(8192, 0, 8, seed=0)
    run_case("c3s", taskgp.Dataset(tr.z, tr.y), None, 16, full_store=False)
    tr, te = make_msd_dataset(8192, 512, 16, seed=0)
    run_case("c4s", taskgp.Dataset(tr.z, tr.y), taskgp.Dataset(te.z, te.y), 16, full_store=False)


def main():
    taskgp.start_runtime(taskgp.RuntimeConfig(worker_count=os.cpu_count()))
    try:
        only = sys.argv[1:]
        if only:
            for name in only:
                {"accept_grid": acceptance_grid, "determinism": determinism,
                 "large": scaled_large_configs}[name]()
            return
        acceptance_grid()
        determinism()
        scaled_large_configs()
        # reference-corpus random instances (test_acceptance.py:28-32 shapes)
        for n, m, t in ((16, 16, 4), (64, 16, 4), (64, 64, 8), (256, 64, 4), (48, 12, 4)):
            rng = np.random.default_rng(n * 1000 + m)
            train = taskgp.Dataset(z=rng.normal(size=(n, 4)), y=rng.normal(size=n))
            test = taskgp.Dataset(z=rng.normal(size=(m, 4)), y=np.zeros(m))
            run_case(f"rand_n{n}_m{m}_t{t}", train, test, t, full_store=True, adam_iters=3)
        # odd test count (gcd tiling fallback, model.py:193-195)
        rng = np.random.default_rng(4242)
        train = taskgp.Dataset(z=rng.normal(size=(16, 3)), y=rng.normal(size=16))
        test = taskgp.Dataset(z=rng.normal(size=(7, 3)), y=np.zeros(7))
        run_case("rand_n16_m7_t4", train, test, 4, full_store=True)

        tr, te = make_msd_dataset(1024, 1024, 8, seed=0)
        run_case("c0", taskgp.Dataset(tr.z, tr.y), taskgp.Dataset(te.z, te.y), 4,
                 full_store=False, adam_iters=0)
        tr, te = make_msd_dataset(2048, 512, 128, seed=0)
        run_case("c2s", taskgp.Dataset(tr.z, tr.y), taskgp.Dataset(te.z, te.y), 4,
                 full_store=False, do_grad=False)
        tr, te = make_msd_dataset(4096, 512, 8, seed=1)
        run_case("d8b512", taskgp.Dataset(tr.z, tr.y), taskgp.Dataset(te.z, te.y), 8,
                 full_store=False, do_full_cov=False)
        tr, _ = make_msd_dataset(8192, 0, 8, seed=0)
        run_case("c1", taskgp.Dataset(tr.z, tr.y), None, 32, full_store=False,
                 adam_iters=3)
    finally:
        taskgp.stop_runtime()


if __name__ == "__main__":
    main()
