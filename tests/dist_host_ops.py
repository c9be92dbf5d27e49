"""Host (numpy) test double of DeviceTileOps for CPU tests of the multi-rank
schedule in paper_2505_00136_b200/distributed.py.

TEST INFRASTRUCTURE ONLY: it lets the 2D block-cyclic schedule, the panel
broadcasts and the distributed solves run under gloo on CPU, so the
distribution logic is checked without GPUs.  Tile arithmetic here is plain
numpy (the GPU path runs the sm_100a kernels through the C ABI instead).
"""

import numpy as np
import torch


class HostTileOps:
    device = torch.device("cpu")

    def zeros(self, *shape, dtype=torch.float64):
        return torch.zeros(*shape, dtype=dtype)

    def from_numpy(self, a):
        return torch.from_numpy(np.array(a, dtype=np.float64))

    def to_numpy(self, t):
        return t.numpy()

    @staticmethod
    def _valid(P, lay):
        return (P % lay["pad_bp"]) < lay["pad_b"]

    @staticmethod
    def _orig(P, lay):
        return (P // lay["pad_bp"]) * lay["pad_b"] + P % lay["pad_bp"]

    def pad(self, src, n_p, d, lay):
        s = src.numpy()
        out = np.zeros((n_p, d)) if d else np.zeros(n_p)
        for P in range(n_p):
            if self._valid(P, lay):
                out[P] = s[self._orig(P, lay)]
        return torch.from_numpy(out)

    def assemble(self, zp, d, lay, params, add_noise, tiles):
        z = zp.numpy()
        b = lay["b"]
        for i, j, t in tiles:
            a, c = z[i * b:(i + 1) * b], z[j * b:(j + 1) * b]
            d2 = ((a[:, None, :] - c[None, :, :]) ** 2).sum(-1)
            k = params.vertical_scale * np.exp(d2 * (-1.0 / (2.0 * params.lengthscale ** 2)))
            P = i * b + np.arange(b)[:, None]
            Q = j * b + np.arange(b)[None, :]
            valid = self._valid(P, lay) & self._valid(Q, lay)
            k = np.where(valid, k + (add_noise and params.noise_variance) * (P == Q),
                         (P == Q).astype(np.float64))
            t.copy_(torch.from_numpy(k))

    def potrf(self, tile, dinv, lay, tile_off, logdiag_slot, info):
        if int(info[0]) >= 0:
            return
        a = np.tril(tile.numpy())
        a = a + np.tril(a, -1).T
        try:
            lo = np.linalg.cholesky(a)
        except np.linalg.LinAlgError:
            for j in range(a.shape[0]):  # first failing pivot (textbook recurrence)
                lo = np.linalg.cholesky(a[: j + 1, : j + 1]) if j else None
            info[0] = self._orig(tile_off, lay)
            return
        tile.copy_(torch.from_numpy(lo))
        dinv.copy_(torch.from_numpy(np.linalg.inv(lo)))
        diag = np.diagonal(lo)
        valid = [self._valid(tile_off + r, lay) for r in range(len(diag))]
        logdiag_slot[0] = float(np.sum(np.log(diag[valid])))

    @staticmethod
    def _k_operand(t):
        """(G, b, b) stacks of panel tiles are one b x G b operand (tiled-k walk)."""
        x = t.numpy()
        return np.concatenate(list(x), axis=1) if x.ndim == 3 else x

    def gemm(self, jobs, b, alpha, beta):
        for a, bb, cin, cout, k, lower in jobs:
            acc = alpha * (self._k_operand(a)[:, :k] @ self._k_operand(bb)[:, :k].T)
            if beta != 0.0:
                acc = acc + beta * cin.numpy()
            cout.copy_(torch.from_numpy(acc))

    def gemv(self, jobs, b, trans, alpha, accumulate):
        for a, x, y in jobs:
            m = a.numpy().T if trans else a.numpy()
            v = alpha * (m @ x.numpy())
            y.copy_(torch.from_numpy(y.numpy() + v if accumulate else v))

    def copy(self, pairs):
        for s, d in pairs:
            d.copy_(s)

    def combine(self, base, parts, out):
        s = base.numpy().copy()
        for p in range(parts.shape[0]):
            s -= parts[p].numpy()
        out.copy_(torch.from_numpy(s))

    def make_replica(self, train, params, tiles_per_dim):
        return HostReplica(self, train, params, tiles_per_dim)


class HostReplica:
    """Full factor gathered on one rank; dense numpy prediction from it."""

    def __init__(self, ops, train, params, tiles_per_dim):
        from paper_2505_00136_b200 import _lib

        self.ops, self.train, self.params = ops, train, params
        self.lay = _lib.layout(train.n, tiles_per_dim)
        b, T = self.lay["b"], self.lay["T"]
        self.tiles = torch.zeros(T * (T + 1) // 2, b, b, dtype=torch.float64)
        self.dinv = torch.zeros(T, b, b, dtype=torch.float64)
        f64 = torch.float64
        self.vecs = {"beta": torch.zeros(self.lay["np"], dtype=f64), "alpha": torch.zeros(self.lay["np"], dtype=f64),
                     "logdiag": torch.zeros(T, dtype=f64)}

    def tile_view(self, index, b):
        return self.tiles[index]

    def dinv_view(self, k, b):
        return self.dinv[k]

    def vec_view(self, name, n):
        return self.vecs[name][:n]

    def publish(self):
        pass

    def _dense(self):
        b, T, n_p = self.lay["b"], self.lay["T"], self.lay["np"]
        full = np.zeros((n_p, n_p))
        for i in range(T):
            for j in range(i + 1):
                full[i * b:(i + 1) * b, j * b:(j + 1) * b] = self.tiles[i * (i + 1) // 2 + j].numpy()
        real = [P for P in range(n_p) if self.ops._valid(P, self.lay)]
        return full[np.ix_(real, real)], np.array(real)

    def export_lower(self, n):
        return np.tril(self._dense()[0])

    def predict(self, zt, want_var):
        lo, real = self._dense()
        z, p = self.train.z, self.params
        d2 = ((zt[:, None, :] - z[None, :, :]) ** 2).sum(-1)
        ks = p.vertical_scale * np.exp(d2 * (-1.0 / (2.0 * p.lengthscale ** 2)))
        alpha = self.vecs["alpha"].numpy()[real]
        mean = ks @ alpha
        var = None
        if want_var:
            v = np.linalg.solve(lo, ks.T)
            var = p.vertical_scale - (v * v).sum(0)
        return mean, var

    def _cross(self, zt):
        z, p = self.train.z, self.params
        d2 = ((zt[:, None, :] - z[None, :, :]) ** 2).sum(-1)
        return p.vertical_scale * np.exp(d2 * (-1.0 / (2.0 * p.lengthscale ** 2)))

    def solve_cross(self, zt, ldv):
        lo, real = self._dense()
        v = np.zeros((self.lay["np"], ldv))
        mean = np.zeros(zt.shape[0])
        if zt.shape[0]:
            ks = self._cross(zt)
            v[real, : zt.shape[0]] = np.linalg.solve(lo, ks.T)
            mean = ks @ self.vecs["alpha"].numpy()[real]
        return torch.from_numpy(mean), torch.from_numpy(v)

    def cov_block(self, za, va, zb, vb, rows, col0):
        p = self.params
        d2 = ((za[:, None, :] - zb[None, :, :]) ** 2).sum(-1)
        prior = p.vertical_scale * np.exp(d2 * (-1.0 / (2.0 * p.lengthscale ** 2)))
        blk = prior - va.numpy()[:, : za.shape[0]].T @ vb.numpy()[:, : zb.shape[0]]
        rows[: za.shape[0], col0:col0 + zb.shape[0]] = torch.from_numpy(blk)

    def gradient_terms(self, cols):
        """Numpy restatement of gpb_loss_gradient_terms over padded positions."""
        b, n_p = self.lay["b"], self.lay["np"]
        lo, real = self._dense()
        z, p = self.train.z, self.params
        d2 = ((z[:, None, :] - z[None, :, :]) ** 2).sum(-1)
        e = np.exp(d2 * (-1.0 / (2.0 * p.lengthscale ** 2)))
        linv = np.linalg.inv(lo)
        kinv = linv.T @ linv
        alpha = self.vecs["alpha"].numpy()[real]
        w = kinv - np.outer(alpha, alpha)
        full = lambda a: self._embed(a, real, n_p)  # noqa: E731
        ml, mv, kd = full(w * e * d2), full(w * e), full(np.diag(np.diag(kinv)))
        out = np.zeros(3)
        for jj in cols:
            for i in range(jj, self.lay["T"]):
                blk = (slice(i * b, (i + 1) * b), slice(jj * b, (jj + 1) * b))
                wt = 1.0 if i == jj else 2.0
                out += [wt * ml[blk].sum(), wt * mv[blk].sum(), kd[blk].sum()]
        return out

    @staticmethod
    def _embed(a, real, n_p):
        out = np.zeros((n_p, n_p))
        out[np.ix_(real, real)] = a
        return out

    def close(self):
        pass
