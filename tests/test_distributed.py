"""Multi-rank schedule of the 2D block-cyclic tiled GP (distributed.py).

CPU: world_size 2, 3 and 4 under gloo with the host tile-ops test double,
checked against the CPU oracle.  GPU: two ranks sharing cuda:0 under gloo run
the real sm_100a kernels through the device-level C ABI (collectives are
host-mediated, so the ranks never spin on each other's kernels).
"""

import os
import socket
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case(kind):
    rng = np.random.default_rng(11)
    if kind == "padded":  # b = 100: n padded once to 640 (5 x 5 grid of 128)
        n, t, d, m = 600, 6, 3, 37
    else:  # b = 128, no padding (GPB_TILE=128 forces an 8 x 8 grid)
        n, t, d, m = 1024, 8, 4, 50
    return (rng.normal(size=(n, d)), rng.normal(size=n), rng.normal(size=(m, d)), t)


def _worker(rank, world, port, kind, device, out_q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), GPB_TILE="128")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _body(rank, world, kind, device, out_q)
    except BaseException as exc:  # report instead of leaving the parent waiting
        import traceback

        out_q.put((rank, "error", traceback.format_exc(), None, None))
        raise
    finally:
        dist.destroy_process_group()


def _body(rank, world, kind, device, out_q):
    if True:
        import paper_2505_00136_b200 as gpb
        from paper_2505_00136_b200.distributed import DistributedGP

        z, y, zt, t = _case(kind)
        rt = None
        if device:
            rt = gpb.start_runtime(gpb.RuntimeConfig(device=0))
            ops = None
        else:
            from dist_host_ops import HostTileOps

            ops = HostTileOps()
        model = DistributedGP(gpb.Dataset(z, y), gpb.KernelParams(1.1, 0.9, 0.2), t, ops=ops)
        ll = model.log_likelihood()
        pv = model.predict_variance(gpb.Dataset(zt, np.zeros(len(zt))))
        L = model.cholesky()
        fc = model.predict_with_full_cov(gpb.Dataset(zt, np.zeros(len(zt))))
        grads = model.loss_gradients()
        hist = model.optimize(gpb.AdamConfig(learning_rate=0.1, iterations=2))
        model.close()
        if rt is not None:
            rt.stop()
        out_q.put((rank, ll, pv.mean, pv.variance,
                   (L if rank == 0 else None, grads, hist, fc.mean, fc.full_covariance)))


def _run(world, kind, device=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, device, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    errors = [r[2] for r in res if isinstance(r[1], str)]
    assert not errors, errors[0]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(res, key=lambda r: r[0])


def _check(res, kind):
    from oracle.tiled_gp import OracleGP, rel_fro

    z, y, zt, t = _case(kind)
    o = OracleGP(z, y, t, 1.1, 0.9, 0.2)
    mean_o, var_o = o.predict_variance(zt)
    ll_o = o.log_likelihood()
    L_o = o.factor_dense()
    grads_o = o.loss_gradients()
    _, cov_o = o.predict_full_cov(zt)
    hist_o = o.optimize(lr=0.1, iterations=2)  # changes o's parameters: last
    for rank, ll, mean, var, (L, grads, hist, fc_mean, cov) in res:  # every rank: full result
        assert abs(ll - ll_o) <= 1e-9 * abs(ll_o)
        assert rel_fro(mean, mean_o) <= 1e-9
        assert rel_fro(var, var_o) <= 1e-9
        assert rel_fro(np.array(grads), np.array(grads_o)) <= 1e-9
        assert rel_fro(np.array(hist), np.array(hist_o)) <= 1e-9
        assert rel_fro(fc_mean, mean_o) <= 1e-9
        assert rel_fro(cov, cov_o) <= 1e-9 and np.array_equal(cov, cov.T)
        if L is not None:
            assert rel_fro(L, L_o) <= 1e-10


@pytest.mark.parametrize("world,kind", [(2, "padded"), (3, "dense"), (4, "padded")])
def test_block_cyclic_schedule_cpu(world, kind):
    _check(_run(world, kind), kind)


def test_process_grid_and_ownership():
    from paper_2505_00136_b200.distributed import BlockCyclic, process_grid

    assert process_grid(8) == (2, 4) and process_grid(4) == (2, 2) and process_grid(2) == (1, 2)
    assert process_grid(1) == (1, 1) and process_grid(6) == (2, 3)
    cyc = BlockCyclic(7, 2, 4)
    owners = [cyc.owner(i, j) for i in range(7) for j in range(i + 1)]
    assert sorted(set(owners)) == list(range(8))
    assert sum(len(cyc.owned(r)) for r in range(8)) == 28
    assert cyc.panel_rows(2, 1) == [3, 5]


def test_gradient_columns_partition():
    from paper_2505_00136_b200.distributed import gradient_columns

    for T, world in [(1, 1), (6, 2), (64, 8), (256, 8), (7, 3), (3, 4)]:
        parts = gradient_columns(T, world)
        assert len(parts) == world and parts == gradient_columns(T, world)
        assert sorted(c for p in parts for c in p) == list(range(T))  # each column once
        assert all(p == sorted(p) for p in parts)
        if T >= 4 * world:  # snake order balances sum (T - J)^2 within a few percent
            cost = [sum((T - j) ** 2 for j in p) for p in parts]
            assert max(cost) <= 1.1 * sum(cost) / world


@pytest.mark.gpu
def test_two_ranks_one_gpu_device_kernels():
    _check(_run(2, "padded", device=True), "padded")


@pytest.mark.gpu
@pytest.mark.parametrize("panels", ["2", "3"])
def test_four_ranks_2x2_grid_one_gpu_device_kernels(monkeypatch, panels):
    """P = 2 process rows: panel slots i // P, per-row broadcasts and the
    tiled-k trailing update addresses on the real kernels; 3-panel groups
    leave a partial last group (T = 8)."""
    monkeypatch.setenv("GPB_DIST_PANELS", panels)
    _check(_run(4, "dense", device=True), "dense")


@pytest.mark.gpu
@pytest.mark.parametrize("world,kind", [(2, "padded"), (4, "dense")])
def test_p2p_panel_exchange_one_gpu(monkeypatch, world, kind):
    """Transport "p2p": the TRSM epilogue stores the panel tiles into the peer
    ranks' panel buffers (CUDA IPC mappings), readiness and buffer reuse are
    ordered by stream-written flags -- no broadcast of the panel.  Ranks share
    cuda:0 here; every wait is a stream memory operation, not a spinning
    kernel, so no rank's kernel waits on another's."""
    monkeypatch.setenv("GPB_DIST_TRANSPORT", "p2p")
    _check(_run(world, kind, device=True), kind)


@pytest.mark.gpu
@pytest.mark.parametrize("transport", ["nccl", "p2p"])
def test_bench_distributed_branch_two_ranks_one_gpu(transport):
    """bench.py's N>1 path end to end (torchrun, 2 ranks on cuda:0, gloo
    collectives; the panel exchange by broadcasts or by the fused p2p path)."""
    import json
    import subprocess

    env = dict(os.environ, GPB_DIST_BACKEND="gloo", GPB_FORCE_DEVICE="0", GPB_BENCH_SMALL="1",
               GPB_DIST_TRANSPORT=transport)
    out = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
         "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
         os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "3"],
        capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "weak" and line["value"] > 0
    assert line["e2e"]["value"] > 0 and line["gpu_launches"] > 0


def _nccl_one_rank(port, out_q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        import torch

        import paper_2505_00136_b200 as gpb
        from paper_2505_00136_b200.distributed import DistributedGP

        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
        rt = gpb.start_runtime(gpb.RuntimeConfig(device=0))
        train, test = gpb.make_msd_dataset(4096, 512, 8, seed=5)
        model = DistributedGP(train, gpb.KernelParams(1.1, 0.9, 0.2), 8)
        ll = model.log_likelihood()
        pv = model.predict_variance(test)
        fc = model.predict_with_full_cov(test)
        grads = model.loss_gradients()
        model.close()
        ref = gpb.GPModel(train, gpb.KernelParams(1.1, 0.9, 0.2), 8)
        rpv = ref.predict_variance(test)
        out_q.put((ll, ref.log_likelihood(), pv.mean, rpv.mean, pv.variance, rpv.variance,
                   np.diagonal(fc.full_covariance), grads, ref.loss_gradients()))
        rt.stop()
        dist.destroy_process_group()
    except BaseException:
        import traceback

        out_q.put(traceback.format_exc())
        raise


@pytest.mark.gpu
def test_nccl_backend_one_rank_matches_single_gpu():
    """The collectives through NCCL (world size 1: every call is a real NCCL
    collective on the library's streams) against the fused single-GPU model."""
    from oracle.tiled_gp import rel_fro

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_one_rank, args=(_free_port(), q))
    p.start()
    res = q.get(timeout=300)
    p.join(timeout=60)
    assert not isinstance(res, str), res
    ll, rll, mean, rmean, var, rvar, fdiag, grads, rgrads = res
    assert abs(ll - rll) <= 1e-10 * abs(rll)
    assert rel_fro(mean, rmean) <= 1e-9 and rel_fro(var, rvar) <= 1e-10
    assert rel_fro(fdiag, rvar) <= 1e-10
    assert rel_fro(np.array(grads), np.array(rgrads)) <= 1e-10
