"""Tile-kernel plugin for the reference registry (taskgp tiles.py:98-117).

``B200TileKernels`` exposes the four factorisation kernels with the
reference backend contract (tiles.py:11-12, 23-46): read-only float64
tiles in, fresh arrays out, ``potrf`` raises ``NotPositiveDefinite``.
Each call runs the sm_100a tile kernels through the C ABI
(``gpb_tile_*``).  With the reference installed a user can do::

    taskgp.tiles.register_tile_backend("b200", B200TileKernels)
    taskgp.set_tile_backend("b200")

and the reference's own ``tiled_cholesky`` runs its tile tasks on the GPU.
This is a parity harness, not the performance path (one PCIe round trip
per tile); the fused path is ``GPModel``.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .errors import DimensionMismatch, NotPositiveDefinite
from .runtime import require_runtime


def _tile(a) -> np.ndarray:
    arr = np.ascontiguousarray(a, dtype=np.float64)
    if arr.ndim != 2:
        raise DimensionMismatch(f"tile must be 2-D, got shape {arr.shape}")
    return arr


class B200TileKernels:
    name = "b200"

    @staticmethod
    def potrf(a) -> np.ndarray:
        a = _tile(a)
        if a.shape[0] != a.shape[1]:
            raise DimensionMismatch(f"potrf needs a square tile, got {a.shape}")
        out = np.empty_like(a)
        rt = require_runtime()
        status = _lib.load().gpb_tile_potrf(rt.handle, _lib.dptr(a), a.shape[0], _lib.dptr(out))
        if status == 6:
            raise NotPositiveDefinite(_lib.load().gpb_last_error().decode())
        _lib.check(status)
        return out

    @staticmethod
    def trsm(l, b) -> np.ndarray:
        """X with X @ l.T == b (tiles.py:36-38)."""
        l, b = _tile(l), _tile(b)
        if l.shape[0] != l.shape[1] or b.shape[1] != l.shape[0]:
            raise DimensionMismatch(f"trsm shapes incompatible: {l.shape} vs {b.shape}")
        out = np.empty_like(b)
        rt = require_runtime()
        _lib.check(_lib.load().gpb_tile_trsm(rt.handle, _lib.dptr(l), _lib.dptr(b), b.shape[0],
                                             l.shape[0], _lib.dptr(out)))
        return out

    @staticmethod
    def syrk(a, c) -> np.ndarray:
        """c - a @ a.T (tiles.py:41-42)."""
        a, c = _tile(a), _tile(c)
        if c.shape[0] != c.shape[1] or a.shape[0] != c.shape[0]:
            raise DimensionMismatch(f"syrk shapes incompatible: {a.shape} vs {c.shape}")
        out = np.empty_like(c)
        rt = require_runtime()
        _lib.check(_lib.load().gpb_tile_syrk(rt.handle, _lib.dptr(a), _lib.dptr(c), a.shape[0],
                                             a.shape[1], _lib.dptr(out)))
        return out

    @staticmethod
    def gemm(a, b, c) -> np.ndarray:
        """c - a @ b.T (tiles.py:45-46)."""
        a, b, c = _tile(a), _tile(b), _tile(c)
        if a.shape[1] != b.shape[1] or c.shape != (a.shape[0], b.shape[0]):
            raise DimensionMismatch(f"gemm shapes incompatible: {a.shape}, {b.shape}, {c.shape}")
        out = np.empty_like(c)
        rt = require_runtime()
        _lib.check(_lib.load().gpb_tile_gemm(rt.handle, _lib.dptr(a), _lib.dptr(b), _lib.dptr(c),
                                             a.shape[0], b.shape[0], a.shape[1], _lib.dptr(out)))
        return out
