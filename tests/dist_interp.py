"""CPU interpreter of the multi-GPU schedule IR (gpb_dist_plan, include/gpb200.h).

TEST INFRASTRUCTURE ONLY.  The library's schedule generator (dist_plan.cu)
emits, per rank, the ordered operation list that its device executor
(dist.cu) runs on the GPU.  This module replays the same lists on numpy
buffers with torch.distributed (gloo) collectives, so the 2D block-cyclic
distribution -- ownership, panel and X-row exchanges, the distributed solves
and the replica-free gradient -- is checked against the oracle on CPU with
several ranks.  Operation semantics follow the kernels they stand for:

  GEMM  cout = alpha a b^T + beta cin per job, operands K-major (element
        (m, k) at off + (k // ktile) kstride + m ld + k % ktile) or M/N-major
        (at off + k ld + m); `lower` skips 128-blocks above the block diagonal
  POTRF lower Cholesky of the tile in place + its inverse, log-diagonal sum,
        first failing pivot
  GEMV  y (+)= alpha op(A) x on b x b tiles;  COMBINE out = base - part
  TRACE the gradient trace pass (sek.cu trace_kernel) over K^-1 tiles
"""

from __future__ import annotations

import math

import numpy as np
import torch
import torch.distributed as dist

from paper_2505_00136_b200 import _lib

BLK = 128
WORLD, ROWG, COLG = 0, 1, 2


class HostColl:
    """gloo process groups of the P x Q grid (every rank builds all of them in
    the same order, as torch.distributed requires)."""

    def __init__(self, rank: int, world: int, p: int, q: int):
        self.rank, self.world, self.P, self.Q = rank, world, p, q
        self.rows = [dist.new_group([pp * q + qq for qq in range(q)]) for pp in range(p)]
        self.cols = [dist.new_group([pp * q + qq for pp in range(p)]) for qq in range(q)]
        self.calls = 0

    def _group(self, g):
        mp, mq = divmod(self.rank, self.Q)
        if g == WORLD:
            return None, lambda r: r
        if g == ROWG:
            return self.rows[mp], lambda r: mp * self.Q + r
        return self.cols[mq], lambda r: r * self.Q + mq

    def bcast(self, g, arr, root):
        grp, glob = self._group(g)
        self.calls += 1
        dist.broadcast(torch.from_numpy(arr), src=glob(root), group=grp)

    def reduce(self, g, arr, root):
        grp, glob = self._group(g)
        self.calls += 1
        dist.reduce(torch.from_numpy(arr), dst=glob(root), op=dist.ReduceOp.SUM, group=grp)

    def allreduce(self, g, arr):
        grp, _ = self._group(g)
        self.calls += 1
        dist.all_reduce(torch.from_numpy(arr), op=dist.ReduceOp.SUM, group=grp)


class Interp:
    """One rank's buffers and the replay of its phases."""

    def __init__(self, rank, world, p, q, z, y, tiles, params, coll, exchange=0):
        self.rank, self.world, self.P, self.Q = rank, world, p, q
        self.n, self.d = z.shape
        self.tiles = tiles
        self.l, self.nu, self.s2 = params
        self.coll = coll
        self.plans = [_lib.dist_plan(rank, world, p, q, self.n, tiles, ph, exchange) for ph in range(3)]
        self._last_gemm = []  # (buf, off, ld, values, mask) of the latest GEMM's jobs
        self._sends = []
        _, _, bufsz, meta = self.plans[0]
        self.meta = meta
        self.bi, self.Ti, self.np_ = meta["bi"], meta["Ti"], meta["np"]
        lay = _lib.layout(self.n, tiles)
        self.pad_bp, self.pad_b = lay["pad_bp"], lay["pad_b"]
        self.buf = [np.zeros(max(1, bufsz[name])) for name in _lib.BUFFERS]
        pos = np.arange(self.np_)
        self.real = (pos % self.pad_bp) < self.pad_b
        orig = (pos // self.pad_bp) * self.pad_b + pos % self.pad_bp
        self.zp = np.zeros((self.np_, self.d))
        self.zp[self.real] = z[orig[self.real]]
        vec = self.buf[4]
        vec[meta["Y"] + np.flatnonzero(self.real)] = y[orig[self.real]]
        self.info = -1

    # ---- helpers -------------------------------------------------------------
    def _sek(self, i, j):
        bi = self.bi
        a, c = self.zp[i * bi:(i + 1) * bi], self.zp[j * bi:(j + 1) * bi]
        d2 = np.zeros((bi, bi))
        for f in range(self.d):  # direct differences in fixed feature order (covariance.py:65-76)
            diff = a[:, f][:, None] - c[:, f][None, :]
            d2 += diff * diff
        e = np.exp(d2 * (-1.0 / (2.0 * self.l * self.l)))
        rr = self.real[i * bi:(i + 1) * bi][:, None] & self.real[j * bi:(j + 1) * bi][None, :]
        return d2, e, rr

    def _operand(self, b, off, rows, k, ld, kmaj, ktile, kstride):
        r = np.arange(rows)[:, None]
        kk = np.arange(k)[None, :]
        if kmaj:
            kt = ktile if ktile > 0 else 1 << 40
            idx = off + (kk // kt) * kstride + r * ld + kk % kt
        else:
            idx = off + kk * ld + r
        return self.buf[b][idx]

    def _mat(self, b, off, rows, cols, ld):
        return self.buf[b][off + np.arange(rows)[:, None] * ld + np.arange(cols)[None, :]]

    def _set(self, b, off, ld, val, mask=None):
        rows, cols = val.shape
        idx = off + np.arange(rows)[:, None] * ld + np.arange(cols)[None, :]
        if mask is None:
            self.buf[b][idx] = val
        else:
            self.buf[b][idx[mask]] = val[mask]

    # ---- ops -----------------------------------------------------------------
    def run(self, phase):
        ops, jobs, _, meta = self.plans[phase]
        for o in ops:
            kind = _lib.OPS[int(o["kind"])]
            getattr(self, "op_" + kind.lower())(o, jobs[o["job0"]:o["job0"] + o["njobs"]])

    def op_zero(self, o, jobs):
        self.buf[o["buf"][0]][o["off"][0]:o["off"][0] + o["count"]] = 0.0

    def op_record(self, o, jobs):
        pass

    op_wait = op_record

    def op_assemble(self, o, jobs):
        bi = self.bi
        for jb in jobs:
            i, j = int(jb["i"]), int(jb["j"])
            d2, e, rr = self._sek(i, j)
            k = self.nu * e
            gi = i * bi + np.arange(bi)[:, None]
            gj = j * bi + np.arange(bi)[None, :]
            diag = gi == gj
            k = np.where(rr, k + (self.s2 if o["flag"] else 0.0) * diag, diag.astype(float))
            self._set(jb["buf"][3], jb["off"][3], bi, k)

    def op_potrf(self, o, jobs):
        bi, k = self.bi, int(o["i"])
        if self.info >= 0:
            return
        a = self._mat(o["buf"][0], o["off"][0], bi, bi, bi)
        a = np.tril(a) + np.tril(a, -1).T
        try:
            lo = np.linalg.cholesky(a)
        except np.linalg.LinAlgError:
            self.info = k * bi
            return
        self._set(o["buf"][0], o["off"][0], bi, lo)
        self._set(o["buf"][1], o["off"][1], bi, np.linalg.inv(lo))
        dg = np.diagonal(lo)
        self.buf[4][self.meta["LOGDIAG"] + k] = float(np.sum(np.log(dg[self.real[k * bi:(k + 1) * bi]])))

    def op_gemm(self, o, jobs):
        M, N = int(o["mblk"]) * BLK, int(o["nblk"]) * BLK
        outs = []
        for jb in jobs:
            K = int(jb["k"])
            a = self._operand(jb["buf"][0], jb["off"][0], M, K, o["lda"], o["ak"], o["a_ktile"], o["a_kstride"])
            b = self._operand(jb["buf"][1], jb["off"][1], N, K, o["ldb"], o["bk"], o["b_ktile"], o["b_kstride"])
            r = o["alpha"] * (a @ b.T)
            if jb["buf"][2] >= 0 and o["beta"] != 0.0:
                r = r + o["beta"] * self._mat(jb["buf"][2], jb["off"][2], M, N, o["ldc"])
            mask = None
            if jb["lower"]:
                mask = (np.arange(M)[:, None] // BLK) >= (np.arange(N)[None, :] // BLK)
            outs.append((jb["buf"][3], jb["off"][3], r, mask))
        for b, off, r, mask in outs:  # jobs of one launch are independent
            self._set(b, off, o["ldc"], r, mask)
        self._last_gemm = [(int(o["ldc"]), r, mask) for _, _, r, mask in outs]

    # peer-memory exchange: a MIRROR's stores into another rank's buffers travel
    # as one gloo message per destination, applied at that rank's WAITFLAG on
    # this rank's "ready" flag (the flag orders them the same way on the GPU)
    def op_mirror(self, o, jobs):
        per = {}
        for jb in jobs:
            ld, r, mask = self._last_gemm[int(jb["k"])]
            dst, b, off = int(jb["i"]), int(jb["buf"][3]), int(jb["off"][3])
            if dst == self.rank:
                self._set(b, off, ld, r, mask)
            else:
                per.setdefault(dst, []).append((b, off, ld, r, mask))
        for dst, entries in per.items():
            head = [len(entries)]
            data = []
            for b, off, ld, r, mask in entries:
                m = np.ones(r.shape, bool) if mask is None else mask
                head += [b, off, ld, r.shape[0], r.shape[1]]
                data.append(np.where(m, r, np.nan).ravel())
            h = torch.tensor(head, dtype=torch.int64)
            d = torch.from_numpy(np.concatenate(data))
            self._sends += [dist.isend(torch.tensor([len(head)], dtype=torch.int64), dst), dist.isend(h, dst),
                            dist.isend(d, dst)]

    def op_signal(self, o, jobs):
        pass

    def op_slice(self, o, jobs):
        pass  # digit planes are an executor detail: a flagged GEMM is the same product

    def op_waitflag(self, o, jobs):
        if int(o["j"]) != 0:  # "free" flags: buffer reuse cannot race here (messages are copies)
            return
        src = int(o["i"])
        n = torch.zeros(1, dtype=torch.int64)
        dist.recv(n, src)
        h = torch.zeros(int(n.item()), dtype=torch.int64)
        dist.recv(h, src)
        head = h.tolist()
        sizes = [head[1 + 5 * e + 3] * head[1 + 5 * e + 4] for e in range(head[0])]
        d = torch.zeros(sum(sizes), dtype=torch.float64)
        dist.recv(d, src)
        vals, at = d.numpy(), 0
        for e in range(head[0]):
            b, off, ld, rows, cols = head[1 + 5 * e:6 + 5 * e]
            r = vals[at:at + rows * cols].reshape(rows, cols)
            at += rows * cols
            self._set(b, off, ld, r, ~np.isnan(r))

    def finish(self):
        for w in self._sends:
            w.wait()
        self._sends = []

    def op_copy(self, o, jobs):
        c = int(o["count"])
        vals = [self.buf[jb["buf"][0]][jb["off"][0]:jb["off"][0] + c].copy() for jb in jobs]
        for jb, v in zip(jobs, vals):
            self.buf[jb["buf"][3]][jb["off"][3]:jb["off"][3] + c] = v

    def op_gemv(self, o, jobs):
        bi = self.bi
        for jb in jobs:
            a = self._mat(jb["buf"][0], jb["off"][0], bi, bi, bi)
            x = self.buf[jb["buf"][1]][jb["off"][1]:jb["off"][1] + bi]
            yv = o["alpha"] * ((a.T if o["flag"] else a) @ x)
            dst = self.buf[jb["buf"][3]]
            sl = slice(jb["off"][3], jb["off"][3] + bi)
            dst[sl] = dst[sl] + yv if o["beta"] != 0.0 else yv

    def op_combine(self, o, jobs):
        c = int(o["count"])
        base = self.buf[o["buf"][0]][o["off"][0]:o["off"][0] + c]
        part = self.buf[o["buf"][1]][o["off"][1]:o["off"][1] + c]
        self.buf[o["buf"][2]][o["off"][2]:o["off"][2] + c] = base - part

    def _view(self, o):
        return self.buf[o["buf"][0]][o["off"][0]:o["off"][0] + o["count"]]

    def op_bcast(self, o, jobs):
        v = self._view(o)
        t = np.ascontiguousarray(v)
        self.coll.bcast(int(o["group"]), t, int(o["root"]))
        v[:] = t

    def op_reduce(self, o, jobs):
        v = self._view(o)
        t = np.ascontiguousarray(v)
        self.coll.reduce(int(o["group"]), t, int(o["root"]))
        v[:] = t

    def op_allreduce(self, o, jobs):
        v = self._view(o)
        t = np.ascontiguousarray(v)
        self.coll.allreduce(int(o["group"]), t)
        v[:] = t

    def op_solve_flow(self, o, jobs):
        from scipy.linalg import solve_triangular

        lo = self.dense_factor_local()
        vec, m = self.buf[4], self.meta
        y = vec[m["Y"]:m["Y"] + self.np_]
        beta = solve_triangular(lo, y, lower=True)
        vec[m["BETA"]:m["BETA"] + self.np_] = beta
        vec[m["ALPHA"]:m["ALPHA"] + self.np_] = solve_triangular(lo, beta, lower=True, trans="T")

    def op_trace(self, o, jobs):
        bi, m = self.bi, self.meta
        alpha = self.buf[4][m["ALPHA"]:m["ALPHA"] + self.np_]
        sl = sv = st = 0.0
        for jb in jobs:
            i, j = int(jb["i"]), int(jb["j"])
            kinv = self._mat(jb["buf"][0], jb["off"][0], bi, bi, bi)
            d2, e, rr = self._sek(i, j)
            w = np.where(rr, 2.0, 0.0)
            if i == j:  # diagonal tiles: 64-blocks below the diagonal twice, on it once
                rb = np.arange(bi)[:, None] // 64
                cb = np.arange(bi)[None, :] // 64
                w = np.where(rb > cb, w, np.where(rb == cb, 0.5 * w, 0.0))
                st += float(np.sum(np.diagonal(kinv)[self.real[i * bi:(i + 1) * bi]]))
            g = kinv - np.outer(alpha[i * bi:(i + 1) * bi], alpha[j * bi:(j + 1) * bi])
            sl += float(np.sum(w * g * e * d2))
            sv += float(np.sum(w * g * e))
        self.buf[o["buf"][2]][o["off"][2]:o["off"][2] + 3] = (sl, sv, st)

    # ---- results -----------------------------------------------------------------
    def dense_factor_local(self):
        """Dense factor from this rank's tiles (world 1: all of them)."""
        ops, jobs, _, meta = self.plans[0]
        bi, Ti = self.bi, self.Ti
        lo = np.zeros((self.np_, self.np_))
        s = 0
        for i in range(Ti):
            for j in range(i + 1):
                if (i % self.P) * self.Q + (j % self.Q) == self.rank:
                    lo[i * bi:(i + 1) * bi, j * bi:(j + 1) * bi] = self.buf[0][s * bi * bi:(s + 1) * bi * bi].reshape(bi, bi)
                    s += 1
        return np.tril(lo)

    def owned_tiles(self):
        bi, out, s = self.bi, {}, 0
        for i in range(self.Ti):
            for j in range(i + 1):
                if (i % self.P) * self.Q + (j % self.Q) == self.rank:
                    out[(i, j)] = self.buf[0][s * bi * bi:(s + 1) * bi * bi].reshape(bi, bi).copy()
                    s += 1
        return out

    def log_likelihood(self):
        m, vec = self.meta, self.buf[4]
        beta = vec[m["BETA"]:m["BETA"] + self.np_]
        half_log_det = math.fsum(vec[m["LOGDIAG"]:m["LOGDIAG"] + self.Ti])
        return -half_log_det - 0.5 * float(beta @ beta) - self.n * 0.5 * math.log(2.0 * math.pi)

    def gradients(self):
        m, vec = self.meta, self.buf[4]
        red = vec[m["RED"]:m["RED"] + 3]
        alpha = vec[m["ALPHA"]:m["ALPHA"] + self.np_]
        return (0.5 * self.nu / self.l ** 3 * red[0], 0.5 * red[1], 0.5 * (red[2] - float(alpha @ alpha)))
