"""Multi-GPU tiled GP: the GPModel contract over ranks (one process per GPU).

A thin shim over the library's multi-GPU runtime (``gpb_dist_*`` in
include/gpb200.h, csrc/dist.cu + csrc/dist_plan.cu): the ranks form a P x Q
process grid (8 -> 2x4, 4 -> 2x2, 2 -> 1x2), lower tile (i, j) of K / L lives
on rank (i mod P) Q + (j mod Q), and the library schedules the 2D
block-cyclic tiled Cholesky (panel broadcasts on its own NCCL row / column
communicators, lookahead on a high-priority stream), the beta / alpha solves
(partial sums reduced onto the diagonal owners, segments broadcast along the
process rows / columns), the replica-free gradient (distributed TRTRI + LAUUM
on the block-cyclic tiles, trace pass per rank, an all-reduce of three
partial sums) and prediction sharded over test points.  Python only creates
the communicator bootstrap and maps results onto the reference's types
(taskgp model.py:91-485).

Panel exchange: "collective" (default; broadcasts on the row / column
communicators) or "p2p" -- the panel TRSM's epilogue stores each solved tile
straight into the panel buffers of the ranks that read it (CUDA IPC mappings,
NVLink stores), ordered by stream-written flags; a rank then receives only
the tiles its trailing update reads and no SM waits on a collective.

Transports: "nccl" (default) -- rank 0 makes an NCCL unique id, the ranks
exchange it over the torch.distributed group (any backend; the data path never
touches torch), the library creates and splits its communicators.  "host" --
the library calls back into Python for host-staged collectives over
torch.distributed (gloo): used by the tests to run several ranks, each with
its own device executor, on CPU collectives.
"""

from __future__ import annotations

import ctypes
import math
import os

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .covariance import KernelParams
from .data import Dataset
from .errors import DimensionMismatch, TilingError


def process_grid(world: int) -> tuple[int, int]:
    """P x Q with P <= Q as square as possible (2D block-cyclic grid)."""
    p = int(math.isqrt(world))
    while world % p:
        p -= 1
    return p, world // p


class BlockCyclic:
    """Owner map of the lower tile grid (the library's, dist_plan.cu)."""

    def __init__(self, tiles: int, p: int, q: int):
        self.T, self.P, self.Q = tiles, p, q

    def owner(self, i: int, j: int) -> int:
        return (i % self.P) * self.Q + (j % self.Q)

    def owned(self, rank: int) -> list[tuple[int, int]]:
        return [(i, j) for i in range(self.T) for j in range(i + 1) if self.owner(i, j) == rank]


class _HostCollectives:
    """gpb_host_coll over torch.distributed (CPU tensors aliasing the library's
    pinned staging buffer).  Groups: 0 world, 1 this rank's process row, 2 its
    process column; roots are ranks within the group."""

    def __init__(self, rank: int, p: int, q: int):
        self.rank, self.P, self.Q = rank, p, q
        # every rank creates every group, in the same order (torch.distributed rule)
        self.rows = [dist.new_group([pp * q + qq for qq in range(q)]) for pp in range(p)]
        self.cols = [dist.new_group([pp * q + qq for pp in range(p)]) for qq in range(q)]
        self.fns = (_lib.BCAST_FN(self._bcast), _lib.REDUCE_FN(self._reduce), _lib.ALLREDUCE_FN(self._allreduce))
        self.struct = _lib.HostColl(self.fns[0], self.fns[1], self.fns[2], None)

    def _group(self, g):
        mp, mq = divmod(self.rank, self.Q)
        if g == 0:
            return None, lambda r: r
        if g == 1:
            return self.rows[mp], lambda r: mp * self.Q + r
        return self.cols[mq], lambda r: r * self.Q + mq

    @staticmethod
    def _doubles(ptr, count):
        return torch.from_numpy(np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(ctypes.c_double)),
                                                      shape=(count,)))

    def _bcast(self, user, g, buf, nbytes, root):
        try:
            grp, glob = self._group(g)
            dist.broadcast(self._doubles(buf, nbytes // 8), src=glob(root), group=grp)
            return 0
        except Exception:  # noqa: BLE001 -- reported to the library as a failed collective
            return 1

    def _reduce(self, user, g, buf, count, root):
        try:
            grp, glob = self._group(g)
            dist.reduce(self._doubles(buf, count), dst=glob(root), op=dist.ReduceOp.SUM, group=grp)
            return 0
        except Exception:  # noqa: BLE001
            return 1

    def _allreduce(self, user, g, buf, count):
        try:
            grp, _ = self._group(g)
            dist.all_reduce(self._doubles(buf, count), op=dist.ReduceOp.SUM, group=grp)
            return 0
        except Exception:  # noqa: BLE001
            return 1


class DistComm:
    """A gpb_dist handle: this rank's place in the P x Q grid and the
    library's communicators.  Collective: every rank constructs it."""

    def __init__(self, runtime=None, grid: tuple[int, int] | None = None, transport: str | None = None,
                 exchange: str | None = None):
        if runtime is None:
            from .runtime import require_runtime

            runtime = require_runtime()
        self.runtime = runtime
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.P, self.Q = grid or process_grid(self.world)
        if self.P * self.Q != self.world:
            raise ValueError(f"process grid {self.P}x{self.Q} does not match {self.world} ranks")
        self.transport = transport or os.environ.get("GPB_DIST_TRANSPORT", "nccl")
        lib = _lib.load()
        h = ctypes.c_void_p()
        if self.transport == "nccl":
            uid = ctypes.create_string_buffer(_lib.NCCL_ID_BYTES)
            if self.rank == 0:
                _lib.check(lib.gpb_nccl_unique_id(uid))
            box = [uid.raw]
            dist.broadcast_object_list(box, src=0)
            uid = ctypes.create_string_buffer(box[0], _lib.NCCL_ID_BYTES)
            _lib.check(lib.gpb_dist_init(runtime.handle, self.rank, self.world, self.P, self.Q, uid,
                                         ctypes.byref(h)))
        elif self.transport == "host":
            self._coll = _HostCollectives(self.rank, self.P, self.Q)
            _lib.check(lib.gpb_dist_init_host(runtime.handle, self.rank, self.world, self.P, self.Q,
                                              ctypes.byref(self._coll.struct), ctypes.byref(h)))
        else:
            raise ValueError(f"unknown transport {self.transport!r} (nccl or host)")
        self.handle = h
        # panel exchange of the factorisation: "collective" (row / column broadcasts)
        # or "p2p" (TRSM epilogue stores into the readers' panel buffers over CUDA IPC)
        self.exchange = exchange or os.environ.get("GPB_DIST_EXCHANGE", "collective")
        if self.exchange not in ("collective", "p2p"):
            raise ValueError(f"unknown exchange {self.exchange!r} (collective or p2p)")
        _lib.check(lib.gpb_dist_set_exchange(h, 1 if self.exchange == "p2p" else 0))

    def close(self):
        if self.handle:
            _lib.load().gpb_dist_finalize(self.handle)
            self.handle = None


class DistributedGP:
    """The GPModel contract over the ranks of the default torch.distributed
    group.  Collective: every rank calls every method with the same
    arguments; results are returned on every rank.

    ``comm``: a DistComm to share between models (default: one per model).
    """

    def __init__(self, train, params: KernelParams | None = None, tiles_per_dim: int = 1,
                 comm: DistComm | None = None, grid: tuple[int, int] | None = None,
                 transport: str | None = None, exchange: str | None = None):
        train = train if isinstance(train, Dataset) else Dataset(np.asarray(train.z), np.asarray(train.y))
        if tiles_per_dim < 1 or train.n % tiles_per_dim != 0:
            raise TilingError(f"tiles_per_dim={tiles_per_dim} must divide the {train.n} training points")
        self.train = train
        self.tiles_per_dim = tiles_per_dim
        self._own_comm = comm is None
        self.comm = comm or DistComm(grid=grid, transport=transport, exchange=exchange)
        self.rank, self.world = self.comm.rank, self.comm.world
        self.P, self.Q = self.comm.P, self.comm.Q
        self._lib = _lib.load()
        h = ctypes.c_void_p()
        _lib.check(self._lib.gpb_dist_model_create(self.comm.handle, _lib.dptr(train.z), _lib.dptr(train.y),
                                                   train.n, train.d, tiles_per_dim, ctypes.byref(h)))
        self._h = h
        self.params = params if params is not None else KernelParams()
        self.timings = {}

    # -- parameters (model.py:149-156) -----------------------------------------
    @property
    def params(self) -> KernelParams:
        return self._params

    @params.setter
    def params(self, params: KernelParams) -> None:
        flags = (ctypes.c_uint8 * 3)(*[1 if t else 0 for t in params.trainable])
        _lib.check(self._lib.gpb_dist_set_params(self._h, params.lengthscale, params.vertical_scale,
                                                 params.noise_variance, flags))
        self._params = params

    def _sync_params(self):
        from dataclasses import replace

        out = (ctypes.c_double * 3)()
        _lib.check(self._lib.gpb_dist_get_params(self._h, out))
        self._params = replace(self._params, lengthscale=out[0], vertical_scale=out[1], noise_variance=out[2])

    def _collect_timings(self):
        t = (ctypes.c_double * 8)()
        self._lib.gpb_dist_timings(self._h, t, 8)
        self.timings = {"factor_ms": t[1], "solve_ms": t[2], "predict_ms": t[3], "gradient_ms": t[4],
                        "replica_ms": t[5], "enqueue_us_per_step": t[6], "collectives": t[7]}

    # -- public API (model.py names) ---------------------------------------------
    def factor(self) -> None:
        """Assemble + factor + solves (cached until the parameters change)."""
        _lib.check(self._lib.gpb_dist_factor(self._h))
        self._collect_timings()

    def log_likelihood(self) -> float:
        out = ctypes.c_double()
        _lib.check(self._lib.gpb_dist_log_likelihood(self._h, ctypes.byref(out)))
        self._collect_timings()
        return float(out.value)

    def compute_loss(self) -> float:
        return -self.log_likelihood()

    def cholesky(self) -> np.ndarray:
        """Dense lower factor on every rank (through the replica; small problems)."""
        n = self.train.n
        out = np.empty((n, n))
        _lib.check(self._lib.gpb_dist_cholesky(self._h, _lib.dptr(out)))
        return out

    def _test(self, test):
        test = test if isinstance(test, Dataset) else Dataset(np.asarray(test.z), np.asarray(test.y))
        if test.d != self.train.d:
            raise DimensionMismatch(f"test has {test.d} features, model was trained with {self.train.d}")
        return test

    def _predict(self, test, var: bool, cov: bool):
        from .model import PredictionResult

        test = self._test(test)
        m = test.n
        mean = np.empty(m)
        v = np.empty(m) if var else None
        c = np.empty((m, m)) if cov else None
        _lib.check(self._lib.gpb_dist_predict(self._h, _lib.dptr(test.z), m, test.d, _lib.dptr(mean),
                                              _lib.dptr(v), _lib.dptr(c)))
        self._collect_timings()
        return PredictionResult(mean=mean, variance=v, full_covariance=c)

    def predict(self, test):
        return self._predict(test, False, False)

    def predict_variance(self, test):
        return self._predict(test, True, False)

    predict_with_uncertainty = predict_variance

    def predict_with_full_cov(self, test):
        return self._predict(test, False, True)

    def loss_gradients(self) -> tuple[float, float, float]:
        out = (ctypes.c_double * 3)()
        _lib.check(self._lib.gpb_dist_loss_gradients(self._h, out))
        self._collect_timings()
        return (float(out[0]), float(out[1]), float(out[2]))

    def optimize(self, opt=None) -> list[float]:
        """Adam on the log-parameters (model.py:437-485); moments persist across calls."""
        from .model import AdamConfig

        opt = opt if opt is not None else AdamConfig()
        hist = np.zeros(opt.iterations)
        try:
            _lib.check(self._lib.gpb_dist_optimize(self._h, opt.learning_rate, opt.beta1, opt.beta2, opt.epsilon,
                                                   opt.iterations, _lib.dptr(hist)))
        finally:
            self._sync_params()
            self._collect_timings()
        return [float(v) for v in hist]

    def launch_count(self) -> int:
        c = ctypes.c_int64()
        self._lib.gpb_dist_launch_count(self._h, ctypes.byref(c))
        return int(c.value)

    def close(self):
        """Release the model (collective with the peer-memory exchange)."""
        if self._h:
            self._lib.gpb_dist_model_destroy(self._h)
            self._h = None
        if self._own_comm and self.comm is not None:
            self.comm.close()
            self.comm = None

    def __del__(self):
        # with the peer-memory exchange, destroying a model is collective (no peer
        # may still store into its panels): that needs an explicit close() on every
        # rank, never a garbage-collection point that differs between ranks
        if self.comm is not None and getattr(self.comm, "exchange", "collective") == "p2p":
            return
        try:
            self.close()
        except Exception:  # noqa: BLE001 -- interpreter shutdown
            pass
