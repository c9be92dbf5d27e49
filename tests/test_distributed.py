"""Multi-GPU tiled GP: the library's 2D block-cyclic schedule (dist_plan.cu)
and its device executor (dist.cu, the DistributedGP shim).

CPU: the schedule IR of every rank of 1x1, 1x2, 2x1, 1x3 and 2x2 grids is
replayed by the numpy interpreter (tests/dist_interp.py) under gloo and
checked against the CPU oracle: factor, log-likelihood, replica-free
gradient.  GPU: ranks sharing cuda:0 run the real executor with host-staged
collectives over gloo (the ranks never wait on each other's kernels); a
world-size-1 run goes through the library's own NCCL communicators.  The
block-cyclic factor must equal the single-GPU factor bit for bit (same GEMMs
with the same K split on every tile).
"""

import os
import socket
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PARAMS = (1.1, 0.9, 0.2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case(kind):
    rng = np.random.default_rng(11)
    if kind == "tiny":  # 2 x 2 tile grid: on a 2 x 2 process grid rank 1 owns no tile
        n, t, d, m = 256, 2, 3, 9
    elif kind == "grid8":  # 12 x 12 tile grid for the 2 x 4 grid of an 8-GPU box (n padded 1500 -> 1536)
        n, t, d, m = 1500, 12, 4, 20
    elif kind == "planes512":  # 512-wide tiles (6 x 6 grid): the trailing updates run on the digit planes
        n, t, d, m = 3072, 6, 4, 40
    elif kind == "padded":  # b = 100: n padded once to 640 (5 x 5 grid of 128)
        n, t, d, m = 600, 6, 3, 37
    else:  # b = 128, no padding (GPB_TILE=128 forces an 8 x 8 grid)
        n, t, d, m = 1024, 8, 4, 50
    return (rng.normal(size=(n, d)), rng.normal(size=n), rng.normal(size=(m, d)), t)


def _spawn(target, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_entry, args=(target, r, world, port, args, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    errs = [r[1] for r in res if r[0] == "error"]
    assert not errs, errs[0]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return [r[1] for r in sorted(res, key=lambda r: r[2])]


def _entry(target, rank, world, port, args, out_q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), GPB_TILE="128")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out_q.put(("ok", globals()[target](rank, world, *args), rank))
    except BaseException:  # report instead of leaving the parent waiting
        import traceback

        out_q.put(("error", traceback.format_exc(), rank))
        raise
    finally:
        dist.destroy_process_group()


# ---- CPU: the schedule IR under the numpy interpreter ---------------------------------
def _interp_rank(rank, world, grid, kind, exchange=0):
    from dist_interp import HostColl, Interp

    z, y, _, t = _case(kind)
    p, q = grid
    coll = HostColl(rank, world, p, q)
    it = Interp(rank, world, p, q, z, y, t, PARAMS, coll, exchange)
    it.run(0)
    it.finish()
    assert it.info < 0
    it.run(1)
    it.run(2)
    tiles = [None] * world
    dist.all_gather_object(tiles, it.owned_tiles())
    m = it.meta
    vec = it.buf[4]
    return {"ll": it.log_likelihood(), "grads": it.gradients(), "tiles": tiles if rank == 0 else None,
            "bi": it.bi, "np": it.np_, "alpha": vec[m["ALPHA"]:m["ALPHA"] + it.np_].copy(), "calls": coll.calls}


@pytest.mark.parametrize("world,grid,kind,exchange", [
    (1, (1, 1), "dense", 0), (2, (1, 2), "padded", 0), (2, (2, 1), "dense", 0), (3, (1, 3), "padded", 0),
    (4, (2, 2), "dense", 0), (4, (2, 2), "padded", 0),
    (2, (1, 2), "dense", 1), (2, (2, 1), "padded", 1), (4, (2, 2), "dense", 1), (3, (1, 3), "padded", 1),
    (4, (2, 2), "tiny", 0), (4, (2, 2), "tiny", 1), (8, (2, 4), "grid8", 0), (8, (2, 4), "grid8", 1),
    (4, (2, 2), "planes512", 1)])
def test_schedule_ir_against_oracle_cpu(world, grid, kind, exchange):
    """Every rank's operation lists (factor, solves, gradient) replayed on CPU
    with gloo collectives reproduce the oracle; every rank ends with the same
    replicated alpha, log-likelihood and gradient.  exchange 1: the panel
    tiles travel as the TRSM's mirror stores into the readers' panel buffers
    (one message per destination, applied at the reader's ready-flag wait)."""
    from oracle.tiled_gp import OracleGP, rel_fro

    res = _spawn("_interp_rank", world, grid, kind, exchange)
    z, y, _, t = _case(kind)
    n = len(y)
    o = OracleGP(z, y, t, *PARAMS)
    ll_o, g_o, L_o = o.log_likelihood(), np.array(o.loss_gradients()), o.factor_dense()
    bi, np_ = res[0]["bi"], res[0]["np"]
    L = np.zeros((np_, np_))
    for owned in res[0]["tiles"]:
        for (i, j), tile in owned.items():
            L[i * bi:(i + 1) * bi, j * bi:(j + 1) * bi] = tile
    assert rel_fro(np.tril(L)[:n, :n], L_o) <= 1e-10
    for r in res:
        assert abs(r["ll"] - ll_o) <= 1e-9 * abs(ll_o)
        assert rel_fro(np.array(r["grads"]), g_o) <= 1e-9
        assert np.array_equal(r["alpha"], res[0]["alpha"])
        if world > 1:
            assert r["calls"] > 0


def test_plan_structure_and_ownership():
    """Host-only checks of the schedule: ownership covers the grid once, the
    buffers hold what the plan addresses, every collective of a group is issued
    by all its members in the same order and with the same size."""
    from paper_2505_00136_b200 import _lib
    from paper_2505_00136_b200.distributed import BlockCyclic, process_grid

    assert process_grid(8) == (2, 4) and process_grid(4) == (2, 2) and process_grid(2) == (1, 2)
    assert process_grid(1) == (1, 1) and process_grid(6) == (2, 3)
    for world, (p, q), n, t in [(8, (2, 4), 8192, 16), (4, (2, 2), 3000, 6), (6, (2, 3), 4096, 8),
                                 (2, (1, 2), 1024, 4), (3, (3, 1), 2048, 4)]:
        cyc = BlockCyclic(_lib.layout(n, t)["T"], p, q)
        owned = [cyc.owned(r) for r in range(world)]
        assert sorted(ij for o in owned for ij in o) == sorted((i, j) for i in range(cyc.T) for j in range(i + 1))
        for phase, exchange in [(0, 0), (1, 0), (2, 0), (0, 1)]:
            seqs, sig, wai = {}, {}, {}
            for r in range(world):
                ops, jobs, bufsz, meta = _lib.dist_plan(r, world, p, q, n, t, phase, exchange)
                for o in ops:  # peer-memory flags: every wait has exactly one matching signal
                    if o["kind"] == 16:
                        sig.setdefault((r, int(o["i"]), int(o["j"]), int(o["count"])), 0)
                        sig[(r, int(o["i"]), int(o["j"]), int(o["count"]))] += 1
                    if o["kind"] == 17:
                        wai.setdefault((int(o["i"]), r, int(o["j"]), int(o["count"])), 0)
                        wai[(int(o["i"]), r, int(o["j"]), int(o["count"]))] += 1
                assert meta["nown"] == len(owned[r])
                for o in ops:  # every buffer reference inside its buffer
                    if o["kind"] in (7, 8, 9, 12):
                        b = _lib.BUFFERS[o["buf"][0]]
                        assert 0 <= o["off"][0] and o["off"][0] + o["count"] <= bufsz[b]
                mirror = np.zeros(len(jobs), bool)  # MIRROR jobs address the destination rank's buffers
                for o in ops:
                    if o["kind"] == 15:
                        mirror[o["job0"]:o["job0"] + o["njobs"]] = True
                for jb, mir in zip(jobs, mirror):
                    sizes = _lib.dist_plan(int(jb["i"]), world, p, q, n, t, phase, exchange)[2] if mir else bufsz
                    for s in range(4):
                        if jb["buf"][s] >= 0:
                            assert 0 <= jb["off"][s] < sizes[_lib.BUFFERS[jb["buf"][s]]]
                mp_, mq = divmod(r, q)
                for o in ops:
                    if o["kind"] in (7, 8, 9):
                        g = int(o["group"])
                        key = (g, 0 if g == 0 else (mp_ if g == 1 else mq))
                        seqs.setdefault(key, {})
                        seqs[key].setdefault(r, []).append((int(o["kind"]), int(o["root"]), int(o["count"])))
            assert all(sig.get(k, 0) == 1 for k in wai), f"unmatched flag waits (phase {phase})"
            assert all(k in wai or k[2] == 1 for k in sig), f"ready signals nobody waits for (phase {phase})"
            for key, per_rank in seqs.items():
                members = {0: range(world), 1: [key[1] * q + qq for qq in range(q)],
                           2: [pp * q + key[1] for pp in range(p)]}[key[0]]
                got = [per_rank.get(r, []) for r in members]
                assert all(g == got[0] for g in got), f"group {key} phase {phase}: mismatched collectives"


# ---- GPU: the device executor --------------------------------------------------------------
def _device_rank(rank, world, grid, kind, transport, exchange="collective"):
    import paper_2505_00136_b200 as gpb
    from paper_2505_00136_b200.distributed import DistributedGP

    z, y, zt, t = _case(kind)
    rt = gpb.start_runtime(gpb.RuntimeConfig(device=0))
    try:
        model = DistributedGP(gpb.Dataset(z, y), gpb.KernelParams(*PARAMS), t, grid=grid, transport=transport,
                              exchange=exchange)
        ll = model.log_likelihood()
        pv = model.predict_variance(gpb.Dataset(zt, np.zeros(len(zt))))
        L = model.cholesky()
        fc = model.predict_with_full_cov(gpb.Dataset(zt, np.zeros(len(zt))))
        grads = model.loss_gradients()
        hist = model.optimize(gpb.AdamConfig(learning_rate=0.1, iterations=2))
        launches = model.launch_count()
        model.close()
        single = None
        if rank == 0:  # the single-GPU model on the same inputs
            ref = gpb.GPModel(gpb.Dataset(z, y), gpb.KernelParams(*PARAMS), t)
            ref.digit_planes = 0  # the multi-GPU executor runs every product on the FP64 DMMA kernels
            single = ref.cholesky()
            ref.close()
        return {"ll": ll, "mean": pv.mean, "var": pv.variance, "L": L if rank == 0 else None, "single": single,
                "fc_mean": fc.mean, "cov": fc.full_covariance, "grads": grads, "hist": hist, "launches": launches}
    finally:
        rt.stop()


def _check_device(res, kind):
    from oracle.tiled_gp import OracleGP, rel_fro

    z, y, zt, t = _case(kind)
    o = OracleGP(z, y, t, *PARAMS)
    mean_o, var_o = o.predict_variance(zt)
    ll_o, L_o, grads_o = o.log_likelihood(), o.factor_dense(), o.loss_gradients()
    _, cov_o = o.predict_full_cov(zt)
    hist_o = o.optimize(lr=0.1, iterations=2)  # changes o's parameters: last
    if kind == "planes512":  # int8 digit planes in the executor: same contract, not the same bits
        assert rel_fro(res[0]["L"], res[0]["single"]) <= 1e-11
    else:
        assert np.array_equal(res[0]["L"], res[0]["single"]), "block-cyclic factor differs from the single-GPU one"
    assert rel_fro(res[0]["L"], L_o) <= 1e-10
    for r in res:  # every rank: the full result
        assert abs(r["ll"] - ll_o) <= 1e-9 * abs(ll_o)
        assert rel_fro(r["mean"], mean_o) <= 1e-9 and rel_fro(r["var"], var_o) <= 1e-9
        assert rel_fro(np.array(r["grads"]), np.array(grads_o)) <= 1e-9
        assert rel_fro(np.array(r["hist"]), np.array(hist_o)) <= 1e-9
        assert rel_fro(r["fc_mean"], mean_o) <= 1e-9
        assert rel_fro(r["cov"], cov_o) <= 1e-9 and np.array_equal(r["cov"], r["cov"].T)
        assert r["launches"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("world,grid,kind", [(2, (1, 2), "padded"), (2, (2, 1), "dense"), (4, (2, 2), "dense"),
                                             (3, (1, 3), "padded"), (4, (2, 2), "tiny")])
def test_device_executor_host_collectives_one_gpu(world, grid, kind):
    _check_device(_spawn("_device_rank", world, grid, kind, "host"), kind)


@pytest.mark.gpu
@pytest.mark.parametrize("world,grid,kind", [(2, (1, 2), "padded"), (4, (2, 2), "dense"), (2, (2, 1), "dense")])
def test_device_executor_peer_memory_exchange_one_gpu(world, grid, kind):
    """Exchange "p2p": the TRSM's epilogue stores every panel tile into the
    row / column panels of the ranks that read it (CUDA IPC mappings), ready and
    free flags written and awaited in stream order (cuStreamWrite/WaitValue64:
    no kernel waits on another rank's kernel).  The factor stays bitwise the
    single-GPU one."""
    _check_device(_spawn("_device_rank", world, grid, kind, "host", "p2p"), kind)


@pytest.mark.gpu
@pytest.mark.parametrize("world,grid,exchange", [(2, (1, 2), "collective"), (2, (2, 1), "p2p"), (4, (2, 2), "p2p"),
                                                 (4, (2, 2), "collective")])
def test_device_executor_digit_planes_one_gpu(world, grid, exchange):
    """512-wide tiles: every rank slices the row / column panels it received into digit
    planes (SLICE ops) and runs NEXT / UPD on the tcgen05 int8 pipe (GEMM ops with flag 1);
    factor, loss, predictions, gradients and Adam history against the oracle."""
    _check_device(_spawn("_device_rank", world, grid, "planes512", "host", exchange), "planes512")


def _not_pd_rank(rank, world, grid):
    import paper_2505_00136_b200 as gpb
    from paper_2505_00136_b200.distributed import DistributedGP

    rng = np.random.default_rng(3)
    z = rng.normal(size=(512, 2))
    z[1] = z[0]  # duplicate point, no noise: the second pivot is exactly 1 - 1 = 0 (rank 0's tile)
    rt = gpb.start_runtime(gpb.RuntimeConfig(device=0))
    try:
        model = DistributedGP(gpb.Dataset(z, rng.normal(size=512)), gpb.KernelParams(1.0, 1.0, 0.0), 4, grid=grid,
                              transport="host")
        try:
            model.log_likelihood()
            raised = None
        except gpb.errors.NotPositiveDefinite as exc:
            raised = str(exc)
        model.params = gpb.KernelParams(1.0, 1.0, 0.1)  # the cache was invalidated: a valid refactor works
        ll = model.log_likelihood()
        model.close()
        return raised, ll
    finally:
        rt.stop()


@pytest.mark.gpu
def test_device_executor_not_positive_definite_on_every_rank():
    """A failing pivot on one rank is reported as NotPositiveDefinite on every
    rank (smallest failing index over the ranks, model.py:210-217), and the
    model recovers after a parameter change."""
    from oracle.tiled_gp import OracleGP

    res = _spawn("_not_pd_rank", 2, (1, 2))
    assert all(r[0] is not None and "non-positive pivot" in r[0] for r in res)
    assert res[0][0] == res[1][0]
    rng = np.random.default_rng(3)
    z = rng.normal(size=(512, 2))
    z[1] = z[0]
    ll_o = OracleGP(z, rng.normal(size=512), 4, 1.0, 1.0, 0.1).log_likelihood()
    assert all(abs(r[1] - ll_o) <= 1e-9 * abs(ll_o) for r in res)


@pytest.mark.gpu
def test_device_executor_nccl_one_rank():
    """World size 1 through the library's own NCCL communicators (world, row and
    column splits created in C++): factor bitwise the single-GPU one."""
    _check_device(_spawn("_device_rank", 1, (1, 1), "dense", "nccl"), "dense")


@pytest.mark.gpu
def test_bench_distributed_branch_two_ranks_one_gpu():
    """bench.py's N>1 path end to end (torchrun, 2 ranks on cuda:0, host-staged
    gloo collectives), strong-scaling line."""
    import json
    import subprocess

    env = dict(os.environ, GPB_DIST_TRANSPORT="host", GPB_FORCE_DEVICE="0", GPB_BENCH_SMALL="1")
    out = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
         "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
         os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "3"],
        capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong" and line["value"] > 0
    assert line["e2e"]["value"] > 0 and line["gpu_launches"] > 0
