"""Multi-GPU tiled GP: 2D block-cyclic Cholesky and test-point-sharded prediction.

SURVEY.md §8(e).  One process per GPU (torchrun), ranks arranged in a P x Q
process grid (8 -> 2x4, 4 -> 2x2, 2 -> 1x2).  Lower tile (i, j) of K/L lives
on rank (i mod P) * Q + (j mod Q).  Per step k of the right-looking tiled
Cholesky (taskgp tiled.py:168-204):

1. the owner of (k, k) runs POTRF/TRTRI on it and broadcasts L_kk^-1;
2. the ranks of process column k mod Q solve their panel tiles (i, k) with
   one grouped DMMA launch (X_i = L_ik L_kk^-T) into per-process-row panel
   buffers;
3. each process row's share of the panel is broadcast (P broadcasts of
   packed tiles) -- the panel exchange of the north star;
4. every rank applies the trailing update to the tiles it owns (one grouped
   DMMA launch with K = b).

The alpha solve (tiled.py:215-260) runs right-looking over tile columns:
each rank accumulates L_ij beta_j (resp. L_ji^T alpha_j) over the tiles it
owns; the partial vectors of segment i are all-gathered and summed in rank
order (deterministic), then L_ii^-1 gives beta_i.  Log-determinant partials
are gathered the same way.

Gradients (model.py:341-435) are split by tile columns of K^-1: each rank
forms K^-1[:, J] = L^-T (L^-1 E_J) for the columns assigned to it
(``gradient_columns``) from its copy of the factor and runs the fused trace
pass over them; the three partial sums are all-gathered and added in rank
order.  Columns are independent, so this needs no other exchange.

Prediction is sharded over test points (no collective during the solve):
every rank gathers the full lower factor into a local single-GPU model
(owned tiles broadcast rank by rank), predicts its slice of the test points
and the slices are all-gathered.

All collectives go through torch.distributed (NCCL on GPUs, gloo on CPU);
all arithmetic through a tile-ops backend: ``DeviceTileOps`` runs the
library's sm_100a kernels through the device-level C ABI on CUDA tensors
used as buffers.  Tests drive the same schedule with a host test double.
"""

from __future__ import annotations

import contextlib
import ctypes
import math
import os
import time

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .covariance import KernelParams
from .data import Dataset
from .errors import DimensionMismatch, NotPositiveDefinite, NumericalConsistencyError, TilingError

_HALF_LOG_2PI = 0.5 * math.log(2.0 * math.pi)
_VARIANCE_SLACK = 1e-9


def process_grid(world: int) -> tuple[int, int]:
    """P x Q with P <= Q as square as possible (2D block-cyclic grid)."""
    p = int(math.isqrt(world))
    while world % p:
        p -= 1
    return p, world // p


class BlockCyclic:
    """Owner map of the lower tile grid."""

    def __init__(self, tiles: int, p: int, q: int):
        self.T, self.P, self.Q = tiles, p, q

    def owner(self, i: int, j: int) -> int:
        return (i % self.P) * self.Q + (j % self.Q)

    def owned(self, rank: int) -> list[tuple[int, int]]:
        return [(i, j) for i in range(self.T) for j in range(i + 1) if self.owner(i, j) == rank]

    def panel_rows(self, k: int, p: int) -> list[int]:
        """Panel tiles i > k held by process row p at step k (in order)."""
        return [i for i in range(k + 1, self.T) if i % self.P == p]


def gradient_columns(tiles: int, world: int) -> list[list[int]]:
    """Deterministic assignment of the internal tile columns of K^-1 to ranks
    for the distributed gradient.  Column J costs ~2 (T - J)^2 tile GEMMs
    (forward and backward solve below row block J), so columns are dealt in
    snake order (0..p-1, p-1..0, ...) which balances the sums of squares."""
    out: list[list[int]] = [[] for _ in range(world)]
    for j in range(tiles):
        r, lap = j % world, (j // world) % 2
        out[world - 1 - r if lap else r].append(j)
    return out


class DeviceTileOps:
    """Tile operations on CUDA tensors via the device-level C ABI (gpb_dev_*)."""

    def __init__(self, runtime, device: int):
        self.rt = runtime
        self.device = torch.device("cuda", device)
        self.lib = _lib.load()
        self.launches = 0  # kernels launched through gpb_dev_* (one per call)

    # buffers --------------------------------------------------------------
    def zeros(self, *shape, dtype=torch.float64):
        return torch.zeros(*shape, dtype=dtype, device=self.device)

    def from_numpy(self, a):
        return torch.from_numpy(np.ascontiguousarray(a)).to(self.device)

    def to_numpy(self, t):
        return t.detach().cpu().numpy()

    def _s(self):
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    @staticmethod
    def _p(t):
        return ctypes.c_void_p(t.data_ptr()) if t is not None else None

    # kernels --------------------------------------------------------------
    def pad(self, src, n_p: int, d: int, lay: dict):
        out = self.zeros(n_p, d) if d else self.zeros(n_p)
        self.launches += 1
        _lib.check(self.lib.gpb_dev_pad(self.rt.handle, self._s(), self._p(src), n_p, d,
                                        lay["pad_bp"], lay["pad_b"], self._p(out)))
        return out

    def assemble(self, zp, d, lay, params: KernelParams, add_noise, tiles):
        if not tiles:
            return
        arr = (_lib.TileDesc * len(tiles))(*[_lib.TileDesc(i, j, t.data_ptr()) for i, j, t in tiles])
        self.launches += 1
        _lib.check(self.lib.gpb_dev_assemble(
            self.rt.handle, self._s(), self._p(zp), d, lay["b"], lay["pad_bp"], lay["pad_b"],
            params.lengthscale, params.vertical_scale, params.noise_variance, int(add_noise),
            arr, len(tiles)))

    def potrf(self, tile, dinv, lay, tile_off, logdiag_slot, info):
        self.launches += 1
        _lib.check(self.lib.gpb_dev_potrf(self.rt.handle, self._s(), self._p(tile), self._p(dinv),
                                          lay["b"], tile_off, lay["pad_bp"], lay["pad_b"],
                                          self._p(logdiag_slot), self._p(info)))

    def gemm(self, jobs, b, alpha, beta):
        """jobs: (a, b_op, cin, cout, k, lower), NT product on b x b tiles.
        a / b_op may be (G, b, b) stacks of panel tiles (one panel buffer
        slot per panel, a fixed stride apart): a tiled-k walk with K = G b."""
        if not jobs:
            return
        arr = (_lib.GemmJob * len(jobs))(*[
            _lib.GemmJob(a.data_ptr(), bb.data_ptr(), ci.data_ptr() if ci is not None else None,
                         co.data_ptr(), k, int(lo)) for a, bb, ci, co, k, lo in jobs])
        strides = {a.stride(0) for a, bb, *_ in jobs if a.dim() == 3} | \
                  {bb.stride(0) for a, bb, *_ in jobs if bb.dim() == 3}
        if strides:
            assert len(strides) == 1, "one panel stride per launch"
            self.launches += 1
            _lib.check(self.lib.gpb_dev_gemm_tiled(self.rt.handle, self._s(), arr, len(jobs), b, b, b,
                                                   b, 1, 1, b, strides.pop(), alpha, beta))
        else:
            self.launches += 1
            _lib.check(self.lib.gpb_dev_gemm(self.rt.handle, self._s(), arr, len(jobs), b, b, b, b,
                                             1, 1, alpha, beta))

    _JOB_DTYPE = np.dtype([("a", "<u8"), ("b", "<u8"), ("cin", "<u8"), ("cout", "<u8"),
                           ("k", "<i4"), ("lower", "<i4")])  # gpb_gemm_job

    def gemm_addr(self, a_addr, b_addr, c_addr, lower, k, b, alpha, beta, kstride=0):
        """Vectorised job table (device addresses as int64 arrays): the
        trailing update of one step at large T without per-tile Python work.
        kstride > 0: operands walk K in b-deep tiles kstride doubles apart."""
        n = len(c_addr)
        if n == 0:
            return
        tab = np.empty(n, dtype=self._JOB_DTYPE)
        tab["a"], tab["b"], tab["cin"], tab["cout"] = a_addr, b_addr, c_addr, c_addr
        tab["k"], tab["lower"] = k, lower
        assert tab.dtype.itemsize == ctypes.sizeof(_lib.GemmJob)
        self.launches += 1
        _lib.check(self.lib.gpb_dev_gemm_tiled(self.rt.handle, self._s(), tab.ctypes.data, n, b, b, b,
                                               b, 1, 1, b if kstride else 0, kstride, alpha, beta))

    def gemv(self, jobs, b, trans, alpha, accumulate):
        if not jobs:
            return
        arr = (_lib.GemvJob * len(jobs))(*[_lib.GemvJob(a.data_ptr(), x.data_ptr(), y.data_ptr())
                                           for a, x, y in jobs])
        self.launches += 1
        _lib.check(self.lib.gpb_dev_gemv(self.rt.handle, self._s(), arr, len(jobs), b, int(trans),
                                         alpha, int(accumulate)))

    def copy(self, pairs):
        if not pairs:
            return
        nbytes = pairs[0][0].numel() * 8
        arr = (_lib.CopyJob * len(pairs))(*[_lib.CopyJob(s.data_ptr(), d.data_ptr()) for s, d in pairs])
        self.launches += 1
        _lib.check(self.lib.gpb_dev_copy(self.rt.handle, self._s(), arr, len(pairs), nbytes))

    # peer memory / stream-ordered flags (transport "p2p") ------------------------
    def ipc_alloc(self, nbytes: int):
        ptr = ctypes.c_void_p()
        handle = ctypes.create_string_buffer(64)
        _lib.check(self.lib.gpb_dev_ipc_alloc(self.rt.handle, nbytes, ctypes.byref(ptr), handle))
        return ptr.value, handle.raw

    def ipc_open(self, handle: bytes) -> int:
        ptr = ctypes.c_void_p()
        _lib.check(self.lib.gpb_dev_ipc_open(self.rt.handle, handle, ctypes.byref(ptr)))
        return ptr.value

    def ipc_close(self, ptr: int):
        _lib.check(self.lib.gpb_dev_ipc_close(self.rt.handle, ctypes.c_void_p(ptr)))

    def free(self, ptr: int):
        _lib.check(self.lib.gpb_dev_free(self.rt.handle, ctypes.c_void_p(ptr)))

    def alias(self, ptr: int, shape):
        return _alias(ptr, shape, self.device)

    def signal(self, addr: int, value: int):
        _lib.check(self.lib.gpb_dev_signal(self.rt.handle, self._s(), ctypes.c_void_p(addr), value))

    def wait(self, addr: int, value: int):
        _lib.check(self.lib.gpb_dev_wait(self.rt.handle, self._s(), ctypes.c_void_p(addr), value))

    def gemm_mirror(self, jobs, b, alpha, beta, mirrors):
        """gemm() whose job j also stores its output at the addresses
        mirrors[j] (a list of ints, one per peer, 0 = skip)."""
        if not jobs:
            return
        arr = (_lib.GemmJob * len(jobs))(*[
            _lib.GemmJob(a.data_ptr(), bb.data_ptr(), ci.data_ptr() if ci is not None else None,
                         co.data_ptr(), k, int(lo)) for a, bb, ci, co, k, lo in jobs])
        nm = max(1, max(len(m) for m in mirrors))
        tab = (ctypes.c_void_p * (len(jobs) * nm))(
            *[m[r] if r < len(m) and m[r] else None for m in mirrors for r in range(nm)])
        self.launches += 1
        _lib.check(self.lib.gpb_dev_gemm_mirror(self.rt.handle, self._s(), arr, len(jobs), b, b, b, b, 1, 1,
                                                0, 0, alpha, beta, tab, nm))

    def copy_addr(self, src_addr, dst_addr, nbytes: int):
        """Batched device copies from address arrays (gpb_dev_copy)."""
        n = len(src_addr)
        if n == 0:
            return
        tab = np.empty(n, dtype=[("src", "<u8"), ("dst", "<u8")])
        tab["src"], tab["dst"] = src_addr, dst_addr
        self.launches += 1
        _lib.check(self.lib.gpb_dev_copy(self.rt.handle, self._s(), tab.ctypes.data, n, nbytes))

    def combine(self, base, parts, out):
        self.launches += 1
        _lib.check(self.lib.gpb_dev_combine(self.rt.handle, self._s(), self._p(base), self._p(parts),
                                            parts.shape[0], base.numel(), self._p(out)))

    # replica for sharded prediction ------------------------------------------
    def make_replica(self, train: Dataset, params: KernelParams, tiles_per_dim: int):
        return _DeviceReplica(self, train, params, tiles_per_dim)


class _DeviceReplica:
    """A local single-GPU model whose factor buffers receive the gathered L."""

    def __init__(self, ops: DeviceTileOps, train: Dataset, params: KernelParams, tiles_per_dim: int):
        self.ops = ops
        lib = ops.lib
        self.z = ops.from_numpy(train.z)
        self.y = ops.from_numpy(train.y)
        h = ctypes.c_void_p()
        _lib.check(lib.gpb_model_create_device(ops.rt.handle, ctypes.c_void_p(self.z.data_ptr()),
                                               ctypes.c_void_p(self.y.data_ptr()), train.n, train.d,
                                               tiles_per_dim, ctypes.byref(h)))
        self.h = h
        self.n, self.tiles_per_dim = train.n, tiles_per_dim
        flags = (ctypes.c_uint8 * 3)(*[1 if t else 0 for t in params.trainable])
        _lib.check(lib.gpb_model_set_params(h, params.lengthscale, params.vertical_scale,
                                            params.noise_variance, flags))
        ptrs = [ctypes.c_void_p() for _ in range(5)]
        _lib.check(lib.gpb_model_factor_buffers(h, *[ctypes.byref(p) for p in ptrs]))
        self.ptr = dict(zip(("tiles", "dinv", "logdiag", "beta", "alpha"), [p.value for p in ptrs]))

    def tile_view(self, index: int, b: int):
        """A tensor aliasing packed tile `index` of the model's factor buffer."""
        return _alias(self.ptr["tiles"] + index * b * b * 8, (b, b), self.ops.device)

    def dinv_view(self, k: int, b: int):
        return _alias(self.ptr["dinv"] + k * b * b * 8, (b, b), self.ops.device)

    def vec_view(self, name: str, n: int):
        return _alias(self.ptr[name], (n,), self.ops.device)

    def export_lower(self, n: int) -> np.ndarray:
        return _export(self, n)

    def loss_gradients(self):
        out = (ctypes.c_double * 3)()
        _lib.check(self.ops.lib.gpb_loss_gradients(self.h, out))
        return (float(out[0]), float(out[1]), float(out[2]))

    def gradient_terms(self, cols: list[int]) -> np.ndarray:
        """Trace partials of the K^-1 tile columns `cols` (gpb_loss_gradient_terms),
        in groups whose (n - J0 b) x (len b) panel fits in device memory."""
        lay = _lib.layout(self.n, self.tiles_per_dim)
        free, _ = torch.cuda.mem_get_info(self.ops.device)
        acc = np.zeros(3)
        rest = sorted(cols)
        while rest:
            per_col = 8.0 * (lay["T"] - rest[0]) * lay["b"] * lay["b"]
            take = max(1, min(len(rest), int(0.4 * free // max(per_col, 1.0))))
            group, rest = rest[:take], rest[take:]
            arr = (ctypes.c_int * len(group))(*group)
            out = (ctypes.c_double * 3)()
            _lib.check(self.ops.lib.gpb_loss_gradient_terms(self.h, arr, len(group), out))
            acc += np.array(out[:3])
        return acc

    def _order(self):
        """The model's entry points run on the library's own stream: work queued
        on torch's current stream (buffer fills, uploads) must finish first."""
        torch.cuda.current_stream(self.ops.device).synchronize()

    def publish(self):
        torch.cuda.current_stream(self.ops.device).synchronize()
        _lib.check(self.ops.lib.gpb_model_mark_factored(self.h))

    def predict(self, zt: np.ndarray, want_var: bool):
        m = zt.shape[0]
        if m == 0:
            return np.zeros(0), (np.zeros(0) if want_var else None)
        ztd = self.ops.from_numpy(zt)
        mean = torch.empty(m, dtype=torch.float64, device=self.ops.device)
        var = torch.empty(m, dtype=torch.float64, device=self.ops.device) if want_var else None
        self._order()
        _lib.check(self.ops.lib.gpb_predict_device(
            self.h, ctypes.c_void_p(ztd.data_ptr()), m, zt.shape[1],
            ctypes.c_void_p(mean.data_ptr()), ctypes.c_void_p(var.data_ptr()) if want_var else None))
        return mean, var

    def solve_cross(self, zt: np.ndarray, ldv: int):
        """(mean, V) of a shard of test points: V = L^-1 K*^T, n_p x ldv on the device."""
        lay = _lib.layout(self.n, self.tiles_per_dim)
        v = self.ops.zeros(lay["np"], ldv)
        m = zt.shape[0]
        mean = self.ops.zeros(max(1, m))
        if m:
            ztd = self.ops.from_numpy(zt)
            self._order()
            _lib.check(self.ops.lib.gpb_predict_solve_device(
                self.h, ctypes.c_void_p(ztd.data_ptr()), m, zt.shape[1], ctypes.c_void_p(mean.data_ptr()),
                ctypes.c_void_p(v.data_ptr()), ldv))
        return mean[:m], v

    def cov_block(self, za: np.ndarray, va, zb: np.ndarray, vb, rows, col0: int):
        """rows[:ma, col0:col0+mb] = K**(za, zb) - Va^T Vb (gpb_cov_block_device)."""
        zad, zbd = self.ops.from_numpy(za), self.ops.from_numpy(zb)
        ldo = rows.shape[1]
        self._order()
        _lib.check(self.ops.lib.gpb_cov_block_device(
            self.h, ctypes.c_void_p(zad.data_ptr()), za.shape[0], ctypes.c_void_p(va.data_ptr()),
            va.shape[1], ctypes.c_void_p(zbd.data_ptr()), zb.shape[0], ctypes.c_void_p(vb.data_ptr()),
            vb.shape[1], ctypes.c_void_p(rows.data_ptr() + col0 * 8), ldo))

    def close(self):
        if self.h is not None:
            self.ops.lib.gpb_model_destroy(self.h)
            self.h = None


def _alias(ptr: int, shape, device):
    """Wrap raw device memory owned by the library as a tensor (no copy)."""
    class _Holder:
        __cuda_array_interface__ = {
            "shape": tuple(shape), "typestr": "<f8", "data": (ptr, False), "version": 3,
            "strides": None,
        }
    return torch.as_tensor(_Holder(), device=device)


class DistributedGP:
    """The GPModel contract over a torch.distributed group (one rank per GPU).

    Collective: every rank must call every method with the same arguments.
    Results are returned on every rank.
    """

    def __init__(self, train, params: KernelParams | None = None, tiles_per_dim: int = 1,
                 ops=None, group=None, grid: tuple[int, int] | None = None):
        train = train if isinstance(train, Dataset) else Dataset(np.asarray(train.z), np.asarray(train.y))
        if tiles_per_dim < 1 or train.n % tiles_per_dim != 0:
            raise TilingError(f"tiles_per_dim={tiles_per_dim} must divide the {train.n} training points")
        self.train = train
        self.params = params if params is not None else KernelParams()
        self.tiles_per_dim = tiles_per_dim
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.P, self.Q = grid or process_grid(self.world)
        if self.P * self.Q != self.world:
            raise ValueError(f"process grid {self.P}x{self.Q} does not match {self.world} ranks")
        if ops is None:
            from .runtime import require_runtime

            rt = require_runtime()
            ops = DeviceTileOps(rt, rt.device)
        self.ops = ops
        self.lay = _lib.layout(train.n, tiles_per_dim)
        self.b, self.T, self.np_ = self.lay["b"], self.lay["T"], self.lay["np"]
        self.cyc = BlockCyclic(self.T, self.P, self.Q)
        self.owned = self.cyc.owned(self.rank)
        self.slot = {ij: s for s, ij in enumerate(self.owned)}
        self._factored = False
        self._replica = None
        self.timings = {}
        # panel exchange: "nccl" (broadcasts) or "p2p" (the TRSM epilogue stores
        # into peer ranks' panel buffers over CUDA IPC, stream-ordered flags)
        self.transport = os.environ.get("GPB_DIST_TRANSPORT", "nccl")
        self._p2p = None
        self._epoch = 0

    # -- collectives (src/dst are global ranks of the group) --------------------
    def _bcast(self, t, src):
        dist.broadcast(t, src=dist.get_global_rank(self.group, src) if self.group else src,
                       group=self.group)

    def _allgather(self, t):
        out = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(out, t.contiguous(), group=self.group)
        return torch.stack(out)

    # -- device timing (CUDA events on the launching stream) -----------------------
    def _event(self):
        if getattr(self.ops, "device", None) is None or self.ops.device.type != "cuda":
            return None
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(torch.cuda.current_stream(self.ops.device))
        return ev

    @staticmethod
    def _elapsed(a, b):
        if a is None or b is None:
            return None
        b.synchronize()
        return a.elapsed_time(b)

    # -- factorisation ---------------------------------------------------------
    def _factor(self):
        """2D block-cyclic tiled Cholesky with panel groups (tiled.py:168-204).

        Panels are factored in groups of G (GPB_DIST_PANELS, default 2) as on
        one GPU: per panel k of group s, on the high-priority critical stream,
        POTRF(k) on its owner, the L_kk^-1 broadcast, the panel TRSM on the
        ranks of process column k mod Q, the per-process-row panel broadcasts
        and the in-group update of the group's later columns (K = b); then
        NEXT(s): the next group's columns updated with all G panels (K = G b).
        The main stream applies UPD(s), the rest of the trailing update, with
        K = G b: each operand walks the G panel tiles of its row, which sit a
        fixed stride apart in the group's panel buffer (tile (i, k) in slot
        i // P of process row i mod P), so C tiles are read and written once
        per group.  Panel buffers alternate between two sets across groups.
        """
        if self._factored:
            return
        ops, b, T, lay = self.ops, self.b, self.T, self.lay
        P, Q = self.P, self.Q
        d = self.train.d
        G = max(1, int(os.environ.get("GPB_DIST_PANELS", "2")))
        self.zp = ops.pad(ops.from_numpy(self.train.z), self.np_, d, lay)
        self.yp = ops.pad(ops.from_numpy(self.train.y), self.np_, 0, lay)
        self.L = ops.zeros(max(1, len(self.owned)), b, b)
        self.dinv = ops.zeros(T, b, b)
        self.logdiag = ops.zeros(T)
        info = ops.zeros(1, dtype=torch.int32) - 1
        ops.assemble(self.zp, d, lay, self.params, True,
                     [(i, j, self.L[s]) for s, (i, j) in enumerate(self.owned)])
        rows_per = -(-T // P)
        # panel buffers: [set][process row] -> (G, rows_per, b, b), one
        # allocation so every panel tile sits a whole number of tiles from
        # the others (the GEMM's TMA view of the launch's operands needs that)
        cuda = getattr(ops, "device", None) is not None and ops.device.type == "cuda"
        p2p = cuda and self.transport == "p2p" and self.world > 1
        if p2p:
            pall, flag_base, peer_base = self._p2p_buffers((2, P, G, rows_per, b, b))
            self._epoch += 1
            epoch = self._epoch << 24  # flag values grow across factorisations
        else:
            pall = ops.zeros(2, P, G, rows_per, b, b)
        panels = [[pall[h, p] for p in range(P)] for h in range(2)]
        my_p, my_q = divmod(self.rank, Q)

        # flags of rank r: ready[src] at slot src, free[src] at slot world + src
        def peer_flag(r, slot):
            return peer_base[r] + pall.numel() * 8 + slot * 8

        def my_flag(slot):
            return flag_base + slot * 8
        by_col = {}
        for s_, (i, j) in enumerate(self.owned):
            by_col.setdefault(j, []).append((s_, i))
        main = torch.cuda.current_stream(ops.device) if cuda else None
        crit = torch.cuda.Stream(device=ops.device, priority=-1) if cuda else None
        on_crit = (lambda: torch.cuda.stream(crit)) if cuda else contextlib.nullcontext
        ev_upd = {}
        vector_upd = hasattr(ops, "gemm_addr")
        if vector_upd:
            own_i = np.array([i for i, _ in self.owned], dtype=np.int64)
            own_j = np.array([j for _, j in self.owned], dtype=np.int64)
            tile_bytes = b * b * 8
            c_addr = self.L.data_ptr() + np.arange(len(self.owned), dtype=np.int64) * tile_bytes
            pbase = [np.array([panels[h][p].data_ptr() for p in range(P)], dtype=np.int64)
                     for h in range(2)]
        if cuda:
            crit.wait_stream(main)  # assembly
        t0 = self._event()
        h0 = time.perf_counter()
        starts = list(range(0, T, G))
        for s, k0 in enumerate(starts):
            k1 = min(T, k0 + G) - 1
            gs = k1 - k0 + 1
            buf = panels[s % 2]

            def stack(i, g_hi):  # panel tiles (i, k0 .. k0+g_hi-1) as a (g_hi, b, b) stack
                return buf[i % P][:g_hi, i // P]

            with on_crit():
                for k in range(k0, k1 + 1):
                    g = k - k0
                    own = self.cyc.owner(k, k)
                    if self.rank == own:
                        ops.potrf(self.L[self.slot[k, k]], self.dinv[k], lay, k * b,
                                  self.logdiag[k:k + 1], info)
                    self._bcast(self.dinv[k], own)
                    if k + 1 == T:
                        break
                    if p2p and g == 0 and s >= 2:
                        # panel set s % 2 is free once every rank has applied group s - 2
                        for r in range(self.world):
                            if r != self.rank:
                                ops.wait(my_flag(self.world + r), epoch + s - 1)
                    if my_q == k % Q and vector_upd and not p2p:
                        # panel TRSM and its copy back into L from address tables
                        sel = (own_j == k) & (own_i > k)
                        ii = own_i[sel]
                        pan = pbase[s % 2][my_p] + (g * rows_per + ii // P) * tile_bytes
                        dk = np.full(len(ii), self.dinv[k].data_ptr(), dtype=np.int64)
                        ops.gemm_addr(c_addr[sel], dk, pan, np.zeros(len(ii), dtype=np.int32), b, b, 1.0, 0.0,
                                      kstride=0)
                        ops.copy_addr(pan, c_addr[sel], tile_bytes)
                    elif my_q == k % Q:  # this rank holds panel tiles of column k
                        mine = self.cyc.panel_rows(k, my_p)
                        jobs = [(self.L[self.slot[i, k]], self.dinv[k], None, buf[my_p][g, i // P], b, False)
                                for i in mine]
                        if p2p:
                            # fused TRSM + panel exchange: the epilogue also stores
                            # tile i into the panel buffer of every peer that
                            # reads it -- process row i mod P (its tiles (i, j))
                            # and process column i mod Q (its tiles (r, i)) --
                            # 1/P + 1/Q of the panel per rank instead of all of it
                            def dest(i, r):
                                return r != self.rank and (r // Q == i % P or r % Q == i % Q)

                            ops.gemm_mirror(jobs, b, 1.0, 0.0, [
                                [peer_base[r] + buf[my_p][g, i // P].data_ptr() - pall.data_ptr()
                                 if dest(i, r) else 0 for r in range(self.world)] for i in mine])
                            for r in range(self.world):
                                if r != self.rank:
                                    ops.signal(peer_flag(r, self.rank), epoch + k + 1)
                        else:
                            ops.gemm(jobs, b, 1.0, 0.0)
                        ops.copy([(buf[my_p][g, i // P], self.L[self.slot[i, k]]) for i in mine])
                    for p in range(P):
                        rows = self.cyc.panel_rows(k, p)
                        src = p * Q + k % Q
                        if not rows:
                            continue
                        if p2p:
                            if src != self.rank:
                                ops.wait(my_flag(src), epoch + k + 1)
                        else:
                            self._bcast(buf[p][g, rows[0] // P: rows[-1] // P + 1], src)
                    # in-group: the group's later columns get panel k (K = b)
                    if vector_upd:  # job tables from address arithmetic (no per-tile Python work)
                        sel = (own_j > k) & (own_j <= k1)
                        ii, jj = own_i[sel], own_j[sel]
                        base = pbase[s % 2]
                        addr_g = lambda x: base[x % P] + (g * rows_per + x // P) * tile_bytes  # noqa: E731
                        ops.gemm_addr(addr_g(ii), addr_g(jj), c_addr[sel], (ii == jj).astype(np.int32), b, b,
                                      -1.0, 1.0, kstride=0)
                    else:
                        ops.gemm([(buf[i % P][g, i // P], buf[j % P][g, j // P], self.L[s_], self.L[s_], b,
                                   i == j) for j in range(k + 1, k1 + 1) for s_, i in by_col.get(j, [])],
                                 b, -1.0, 1.0)
                if k1 + 1 < T:
                    # NEXT(s): the next group's columns get all gs panels (K = gs b);
                    # UPD(s-1) covered them too
                    if cuda and s >= 1:
                        crit.wait_event(ev_upd[s - 1])
                    nxt_hi = min(T, k1 + 1 + G)
                    if vector_upd:
                        sel = (own_j > k1) & (own_j < nxt_hi)
                        ii, jj = own_i[sel], own_j[sel]
                        base = pbase[s % 2]
                        addr0 = lambda x: base[x % P] + (x // P) * tile_bytes  # noqa: E731
                        ops.gemm_addr(addr0(ii), addr0(jj), c_addr[sel], (ii == jj).astype(np.int32), gs * b, b,
                                      -1.0, 1.0, kstride=rows_per * b * b)
                    else:
                        ops.gemm([(stack(i, gs), stack(j, gs), self.L[s_], self.L[s_], gs * b, i == j)
                                  for j in range(k1 + 1, nxt_hi) for s_, i in by_col.get(j, [])],
                                 b, -1.0, 1.0)
                if cuda:
                    ev_panel = torch.cuda.Event()
                    ev_panel.record(crit)
            if k1 + 1 >= T:
                break
            # UPD(s) on the main stream: owned tiles (i, j), j beyond the next group
            if cuda:
                main.wait_event(ev_panel)
            j_lo = k1 + 1 + G
            if vector_upd:  # job table built with numpy (large T)
                sel = own_j >= j_lo
                ii, jj = own_i[sel], own_j[sel]
                base = pbase[s % 2]
                addr = lambda x: base[x % P] + (x // P) * tile_bytes  # noqa: E731
                ops.gemm_addr(addr(ii), addr(jj), c_addr[sel], (ii == jj).astype(np.int32), gs * b, b,
                              -1.0, 1.0, kstride=rows_per * b * b)
            else:
                ops.gemm([(stack(i, gs), stack(j, gs), self.L[s_], self.L[s_], gs * b, i == j)
                          for j in range(j_lo, T) for s_, i in by_col.get(j, [])], b, -1.0, 1.0)
            if p2p:  # this rank is done reading panel set s % 2
                for r in range(self.world):
                    if r != self.rank:
                        ops.signal(peer_flag(r, self.world + self.rank), epoch + s + 1)
            if cuda:
                ev_upd[s] = torch.cuda.Event()
                ev_upd[s].record(main)
        if cuda:
            main.wait_stream(crit)
        h1 = time.perf_counter()  # host time to enqueue the schedule
        t1 = self._event()
        infos = self._allgather(info).view(-1).cpu().numpy()
        bad = [int(v) for v in infos if v >= 0]
        if bad:
            raise NotPositiveDefinite(
                f"Matrix is not positive definite (non-positive pivot at index {min(bad)})")
        t2 = self._event()
        self._solve()
        t3 = self._event()
        self.timings = {"factor_ms": self._elapsed(t0, t1), "solve_ms": self._elapsed(t2, t3),
                        "enqueue_ms": 1e3 * (h1 - h0)}
        self._factored = True

    def _p2p_buffers(self, shape):
        """This rank's IPC-shared panel buffer (plus 2 x world flag words after
        it) and every peer's mapping of theirs; allocated once per instance."""
        numel = int(np.prod(shape))
        if self._p2p is None or self._p2p["shape"] != shape:
            self._p2p_release()
            ops = self.ops
            ptr, handle = ops.ipc_alloc(numel * 8 + 2 * self.world * 8)
            handles = [None] * self.world
            dist.all_gather_object(handles, handle, group=self.group)
            peers = [ptr if r == self.rank else ops.ipc_open(handles[r]) for r in range(self.world)]
            self._p2p = {"shape": shape, "ptr": ptr, "peers": peers,
                         "pall": ops.alias(ptr, shape)}
        p = self._p2p
        return p["pall"], p["ptr"] + numel * 8, p["peers"]

    def _p2p_release(self):
        if self._p2p is None:
            return
        torch.cuda.synchronize(self.ops.device)
        dist.barrier(group=self.group)  # no peer still writes into our buffer
        for r, q in enumerate(self._p2p["peers"]):
            if r != self.rank:
                self.ops.ipc_close(q)
        dist.barrier(group=self.group)  # every mapping closed before the free
        self.ops.free(self._p2p["ptr"])
        self._p2p = None

    def _solve(self):
        ops, b, T = self.ops, self.b, self.T
        self.beta = ops.zeros(self.np_)
        self.alpha = ops.zeros(self.np_)
        acc = ops.zeros(self.np_)
        tmp = ops.zeros(b)
        seg = lambda i: slice(i * b, (i + 1) * b)  # noqa: E731
        col = {}
        for (i, j) in self.owned:
            col.setdefault(j, []).append(i)
        for i in range(T):  # beta = L^-1 y
            parts = self._allgather(acc[seg(i)])
            ops.combine(self.yp[seg(i)], parts, tmp)
            ops.gemv([(self.dinv[i], tmp, self.beta[seg(i)])], b, False, 1.0, False)
            ops.gemv([(self.L[self.slot[r, i]], self.beta[seg(i)], acc[seg(r)])
                      for r in col.get(i, []) if r > i], b, False, 1.0, True)
        acc.zero_()
        row = {}
        for (i, j) in self.owned:
            row.setdefault(i, []).append(j)
        for i in reversed(range(T)):  # alpha = L^-T beta
            parts = self._allgather(acc[seg(i)])
            ops.combine(self.beta[seg(i)], parts, tmp)
            ops.gemv([(self.dinv[i], tmp, self.alpha[seg(i)])], b, True, 1.0, False)
            ops.gemv([(self.L[self.slot[i, q]], self.alpha[seg(i)], acc[seg(q)])
                      for q in row.get(i, []) if q < i], b, True, 1.0, True)
        parts = self._allgather(self.logdiag).cpu().numpy()
        self.logdiag_total = parts.sum(axis=0)  # one owner per tile: exact

    # -- replica of the full factor for sharded prediction ---------------------------
    def _ensure_replica(self):
        self._factor()
        if self._replica is not None:
            return self._replica
        ops, b = self.ops, self.b
        rep = ops.make_replica(self.train, self.params, self.tiles_per_dim)
        cap = max(len(self.cyc.owned(r)) for r in range(self.world))
        stage = ops.zeros(max(1, cap), b, b)
        for r in range(self.world):
            tiles_r = self.cyc.owned(r)
            if not tiles_r:
                continue
            if r == self.rank:
                stage[:len(tiles_r)].copy_(self.L[:len(tiles_r)])
            self._bcast(stage[:len(tiles_r)], r)
            ops.copy([(stage[s], rep.tile_view(i * (i + 1) // 2 + j, b))
                      for s, (i, j) in enumerate(tiles_r)])
        rep.vec_view("beta", self.np_).copy_(self.beta)
        rep.vec_view("alpha", self.np_).copy_(self.alpha)
        rep.vec_view("logdiag", self.T).copy_(torch.as_tensor(self.logdiag_total).to(self.beta.device))
        ops.copy([(self.dinv[k], rep.dinv_view(k, b)) for k in range(self.T)])
        rep.publish()
        self._replica = rep
        return rep

    # -- public API (model.py names) ---------------------------------------------
    def log_likelihood(self) -> float:
        self._factor()
        beta = self.ops.to_numpy(self.beta)
        half_log_det = float(sum(float(v) for v in self.logdiag_total))
        return -half_log_det - 0.5 * float(beta @ beta) - self.train.n * _HALF_LOG_2PI

    def compute_loss(self) -> float:
        return -self.log_likelihood()

    def cholesky(self) -> np.ndarray:
        """Dense lower factor, gathered on every rank (small problems only)."""
        return self._ensure_replica().export_lower(self.train.n)

    def _shard(self, m: int) -> slice:
        per = -(-m // self.world)
        return slice(min(m, self.rank * per), min(m, (self.rank + 1) * per))

    def _predict(self, test, want_var: bool):
        test = test if isinstance(test, Dataset) else Dataset(np.asarray(test.z), np.asarray(test.y))
        if test.d != self.train.d:
            raise DimensionMismatch(f"test has {test.d} features, model was trained with {self.train.d}")
        rep = self._ensure_replica()
        m = test.n
        sh = self._shard(m)
        t0 = self._event()
        per = -(-m // self.world)
        mean, var = rep.predict(test.z[sh], want_var)
        out_m = self.ops.zeros(per)
        out_m[: sh.stop - sh.start] = torch.as_tensor(mean).to(out_m.device) if len(mean) else 0
        gm = self._allgather(out_m).cpu().numpy().reshape(-1)[:m]
        gv = None
        if want_var:
            out_v = self.ops.zeros(per)
            out_v[: sh.stop - sh.start] = torch.as_tensor(var).to(out_v.device) if len(var) else 0
            gv = self._allgather(out_v).cpu().numpy().reshape(-1)[:m]
            bad = gv < -_VARIANCE_SLACK
            if np.any(bad):
                raise NumericalConsistencyError(
                    f"variance {float(gv[bad].min()):g} is below the round-off allowance "
                    f"-{_VARIANCE_SLACK:g}")
            gv = np.where(gv < 0.0, 0.0, gv)
        self.timings["predict_ms"] = self._elapsed(t0, self._event())
        return gm, gv

    def predict(self, test):
        from .model import PredictionResult

        mean, _ = self._predict(test, False)
        return PredictionResult(mean=mean)

    def predict_variance(self, test):
        from .model import PredictionResult

        mean, var = self._predict(test, True)
        return PredictionResult(mean=mean, variance=var)

    predict_with_uncertainty = predict_variance

    def predict_with_full_cov(self, test):
        """Mean and full posterior covariance, sharded over test points
        (option (i)): rank a solves V_a = L^-1 K*(shard a)^T,
        the V blocks are all-gathered, rank a forms its block row
        Sigma[a, :] = K**(a, :) - V_a^T V (one DMMA GEMM per column block) and
        the block rows are all-gathered.  Diagonal clamped as model.py:488-496."""
        from .model import PredictionResult

        test = test if isinstance(test, Dataset) else Dataset(np.asarray(test.z), np.asarray(test.y))
        if test.d != self.train.d:
            raise DimensionMismatch(f"test has {test.d} features, model was trained with {self.train.d}")
        rep = self._ensure_replica()
        m = test.n
        per = -(-m // self.world)
        ldv = max(128, -(-per // 128) * 128)
        sh = self._shard(m)
        t0 = self._event()
        mean_a, va = rep.solve_cross(test.z[sh], ldv)
        vall = self._allgather(va)
        rows = self.ops.zeros(per, m)
        for r in range(self.world):
            lo, hi = min(m, r * per), min(m, (r + 1) * per)
            if sh.stop > sh.start and hi > lo:
                rep.cov_block(test.z[sh], va, test.z[lo:hi], vall[r], rows, lo)
        out_m = self.ops.zeros(per)
        out_m[: sh.stop - sh.start] = mean_a
        gm = self._allgather(out_m).cpu().numpy().reshape(-1)[:m]
        cov = self._allgather(rows).cpu().numpy().reshape(-1, m)[:m]
        diag = np.diagonal(cov).copy()
        bad = diag < -_VARIANCE_SLACK
        if np.any(bad):
            raise NumericalConsistencyError(
                f"variance {float(diag[bad].min()):g} is below the round-off allowance "
                f"-{_VARIANCE_SLACK:g}")
        np.fill_diagonal(cov, np.where(diag < 0.0, 0.0, diag))
        self.timings["full_cov_ms"] = self._elapsed(t0, self._event())
        return PredictionResult(mean=gm, full_covariance=cov)

    # -- training (model.py:341-485) ----------------------------------------------
    def loss_gradients(self) -> tuple[float, float, float]:
        """dNLL/d(l, nu, sigma^2) (model.py:341-435), split over ranks by
        tile columns of K^-1 (``gradient_columns``): each rank sums the trace
        terms of its columns, the partials are all-gathered and added in rank
        order, so every rank returns the same values."""
        tr = self.params.trainable
        if not (tr[0] or tr[1] or tr[2]):
            return (0.0, 0.0, 0.0)
        rep = self._ensure_replica()
        t0 = self._event()
        mine = gradient_columns(self.T, self.world)[self.rank]
        acc = rep.gradient_terms(mine) if mine else np.zeros(3)
        parts = self._allgather(self.ops.from_numpy(acc)).cpu().numpy()
        tot = np.zeros(3)
        for r in range(self.world):  # fixed rank order
            tot += parts[r]
        alpha = self.ops.to_numpy(self.alpha)
        p = self.params
        gl = 0.5 * (p.vertical_scale / p.lengthscale ** 3) * tot[0] if tr[0] else 0.0
        gv = 0.5 * tot[1] if tr[1] else 0.0
        gn = 0.5 * (tot[2] - float(alpha @ alpha)) if tr[2] else 0.0
        self.timings["gradient_ms"] = self._elapsed(t0, self._event())
        return (float(gl), float(gv), float(gn))

    def _set_params(self, params: KernelParams) -> None:
        self.params = params
        self._close_replica()
        self._factored = False

    def optimize(self, opt=None) -> list[float]:
        """Adam on the log-parameters (model.py:437-485); every iteration
        re-factors K distributed.  Moments persist across calls."""
        from dataclasses import replace

        from .model import AdamConfig

        opt = opt if opt is not None else AdamConfig()
        if not hasattr(self, "_adam"):
            self._adam = [np.zeros(3), np.zeros(3), 0]
        m_, v_, _ = self._adam
        history = []
        for _ in range(opt.iterations):
            self._adam[2] += 1
            step_no = self._adam[2]
            try:
                grads = np.array(self.loss_gradients())
                p = self.params
                theta = np.array([p.lengthscale, p.vertical_scale, p.noise_variance])
                g = grads * theta
                m_[:] = opt.beta1 * m_ + (1 - opt.beta1) * g
                v_[:] = opt.beta2 * v_ + (1 - opt.beta2) * g * g
                m_hat = m_ / (1 - opt.beta1 ** step_no)
                v_hat = v_ / (1 - opt.beta2 ** step_no)
                step = opt.learning_rate * m_hat / (np.sqrt(v_hat) + opt.epsilon)
                mask = np.array(p.trainable, dtype=bool)
                u = np.where(mask, np.log(np.maximum(theta, 1e-300)) - step, 0.0)
                theta = np.where(mask, np.exp(u), theta)
                if mask[2]:
                    theta[2] = max(theta[2], 1e-12)
                self._set_params(replace(p, lengthscale=float(theta[0]),
                                         vertical_scale=float(theta[1]),
                                         noise_variance=float(theta[2])))
                history.append(-self.log_likelihood())
            except NotPositiveDefinite as exc:
                raise NotPositiveDefinite(f"iteration {step_no}: {exc}") from exc
        return history

    def launch_count(self) -> int:
        """Kernels this instance launched: the device-level ABI calls of the
        schedule plus the replica model's own launches (prediction, gradient)."""
        n = getattr(self.ops, "launches", 0)
        rep = self._replica
        if rep is not None and getattr(rep, "h", None) is not None:
            c = ctypes.c_int64()
            self.ops.lib.gpb_model_launch_count(rep.h, ctypes.byref(c))
            n += int(c.value)
        return n

    def _close_replica(self):
        if self._replica is not None:
            self._replica.close()
            self._replica = None

    def close(self):
        """Release the replica and the peer buffers (collective with p2p)."""
        self._close_replica()
        self._p2p_release()


def _export(rep, n: int) -> np.ndarray:
    out = np.empty((n, n))
    _lib.check(rep.ops.lib.gpb_cholesky(rep.h, _lib.dptr(out)))
    return out
