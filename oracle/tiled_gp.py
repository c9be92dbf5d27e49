"""CPU oracle: a numpy restatement of the reference tiled-GP algorithm.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2505_00136_b200`` imports this
module; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
baseline / ``--impl reference`` leg use it, and only as the checker (or as the
timed stand-in for the reference CPU implementation, which cannot travel to
the GPU box because ``/root/reference`` is absent there).

Every function restates the reference algorithm of ``taskgp`` 0.1.0
(``/root/reference/pkg/src/taskgp``) with the same numpy/scipy tile
operations in the same per-tile order, so results agree with the reference
to the last bit on the same inputs (pinned by ``tests/test_oracle.py``
against ``tests/golden/*.npz``, which ``tests/golden/make_golden.py``
produced by running the reference itself in the build container).

Storage: a lower tile grid ``dict[(i, j)] -> ndarray`` (i >= j), tiles
row-major, like ``TiledMatrix`` (tiled.py:44-80).  The task runtime
(runtime.py) only orders tile operations; each tile's update sequence is
fixed by the algorithm, so a sequential restatement yields the same values.
``ThreadedCholesky`` adds the runtime's parallelism back (BSP per step, one
BLAS thread per worker like runtime.py:180-181) for the CPU baseline.
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np
from scipy.linalg import solve_triangular

_CHUNK = 256  # covariance.py:23
_VARIANCE_SLACK = 1e-9  # model.py:33
_HALF_LOG_2PI = 0.5 * math.log(2.0 * math.pi)  # model.py:35


class OracleNotPD(ArithmeticError):
    pass


# -- covariance (covariance.py) ----------------------------------------------

def sq_dists(a, b):
    """Direct-difference squared distances, 256-row chunks (covariance.py:65-73)."""
    out = np.empty((a.shape[0], b.shape[0]))
    for s in range(0, a.shape[0], _CHUNK):
        e = min(s + _CHUNK, a.shape[0])
        diff = a[s:e, None, :] - b[None, :, :]
        np.square(diff, out=diff)
        np.sum(diff, axis=2, out=out[s:e])
    return out


def kernel_block(a, b, l, nu):
    """nu * exp(-d2 / (2 l^2)) (covariance.py:76-82)."""
    d2 = sq_dists(a, b)
    d2 *= -1.0 / (2.0 * l ** 2)
    np.exp(d2, out=d2)
    d2 *= nu
    return d2


def row_blocks(z, t):
    ts = z.shape[0] // t
    return [z[i * ts:(i + 1) * ts] for i in range(t)]


def assemble_covariance(z, l, nu, s2, t, include_noise=True):
    """Lower tile grid of K (covariance.py:118-164)."""
    blocks = row_blocks(z, t)
    noise = s2 if include_noise else 0.0
    grid = {}
    for i in range(t):
        for j in range(i + 1):
            tile = kernel_block(blocks[i], blocks[j], l, nu)
            if i == j and noise:
                tile[np.diag_indices_from(tile)] += noise
            grid[i, j] = tile
    return grid


def assemble_covariance_threaded(z, l, nu, s2, t, workers, include_noise=True):
    """assemble_covariance with the independent tiles built by W threads (numpy
    releases the GIL inside the ufunc loops); every tile is computed by the
    same kernel_block call, so the grid is bitwise identical."""
    blocks = row_blocks(z, t)
    noise = s2 if include_noise else 0.0
    pairs = [(i, j) for i in range(t) for j in range(i + 1)]

    def one(ij):
        i, j = ij
        tile = kernel_block(blocks[i], blocks[j], l, nu)
        if i == j and noise:
            tile[np.diag_indices_from(tile)] += noise
        return tile

    with ThreadPoolExecutor(workers) as ex:
        return dict(zip(pairs, ex.map(one, pairs)))


def assemble_cross(zt, z, l, nu, row_tiles, col_tiles):
    """Test-by-train K* tiles (covariance.py:167-193)."""
    rows, cols = row_blocks(zt, row_tiles), row_blocks(z, col_tiles)
    return {(i, j): kernel_block(rows[i], cols[j], l, nu)
            for i in range(row_tiles) for j in range(col_tiles)}


def assemble_dk_lengthscale(z, l, nu, t):
    """dK/dl = nu/l^3 * e * d2 (covariance.py:196-207)."""
    scale = nu / l ** 3
    blocks = row_blocks(z, t)
    grid = {}
    for i in range(t):
        for j in range(i + 1):
            d2 = sq_dists(blocks[i], blocks[j])
            e = np.exp(d2 * (-1.0 / (2.0 * l ** 2)))
            grid[i, j] = scale * e * d2
    return grid


def assemble_dk_vertical(z, l, t):
    """dK/dnu = e (covariance.py:210-220)."""
    blocks = row_blocks(z, t)
    grid = {}
    for i in range(t):
        for j in range(i + 1):
            d2 = sq_dists(blocks[i], blocks[j])
            d2 *= -1.0 / (2.0 * l ** 2)
            grid[i, j] = np.exp(d2)
    return grid


# -- tile kernels (tiles.py:23-46, 170-217) ----------------------------------

def potrf(a):
    try:
        return np.linalg.cholesky(a)  # tiles.py:29-33
    except np.linalg.LinAlgError as exc:
        raise OracleNotPD(str(exc)) from exc


def trsm(l, b):
    return solve_triangular(l, b.T, lower=True, check_finite=False).T  # tiles.py:36-38


def syrk(a, c):
    return c - a @ a.T  # tiles.py:41-42


def gemm(a, b, c):
    return c - a @ b.T  # tiles.py:45-46


# -- tiled algorithms (tiled.py) ---------------------------------------------

def tiled_cholesky(grid, t):
    """Right-looking tile Cholesky (tiled.py:168-204)."""
    g = dict(grid)
    for k in range(t):
        g[k, k] = potrf(g[k, k])
        for i in range(k + 1, t):
            g[i, k] = trsm(g[k, k], g[i, k])
        for i in range(k + 1, t):
            g[i, i] = syrk(g[i, k], g[i, i])
            for j in range(k + 1, i):
                g[i, j] = gemm(g[i, k], g[j, k], g[i, j])
    return g


class ThreadedCholesky:
    """The same tile DAG run by W worker threads (CPU-baseline executor).

    Step-synchronous restatement of runtime.py's work-stealing pool: every
    tile op of one phase (TRSM column, then SYRK/GEMM trailing tiles) is an
    independent task; BLAS is pinned to one thread per worker exactly like
    runtime.py:180-181, so parallelism comes from tiles, as in the reference.
    """

    def __init__(self, workers):
        self.workers = workers

    def __call__(self, grid, t):
        from threadpoolctl import threadpool_limits

        g = dict(grid)
        with threadpool_limits(1), ThreadPoolExecutor(self.workers) as ex:
            for k in range(t):
                g[k, k] = potrf(g[k, k])
                lkk = g[k, k]
                rows = list(range(k + 1, t))
                for i, x in zip(rows, ex.map(lambda i: trsm(lkk, g[i, k]), rows)):
                    g[i, k] = x
                pairs = [(i, j) for i in rows for j in range(k + 1, i + 1)]

                def upd(ij):
                    i, j = ij
                    if i == j:
                        return syrk(g[i, k], g[i, i])
                    return gemm(g[i, k], g[j, k], g[i, j])

                for ij, x in zip(pairs, ex.map(upd, pairs)):
                    g[ij] = x
        return g

    def forward_solve_matrix(self, lg, cross, t, row_tiles):
        """Column tiles of V = L^-1 K*^T are independent: one task each."""
        from threadpoolctl import threadpool_limits

        def one(c):
            return forward_solve_matrix_col(lg, cross, t, c)

        v = {}
        with threadpool_limits(1), ThreadPoolExecutor(self.workers) as ex:
            for c, col in zip(range(row_tiles), ex.map(one, range(row_tiles))):
                for i in range(t):
                    v[i, c] = col[i]
        return v


def forward_solve(lg, b, t):
    """l @ x == b, blocked (tiled.py:215-237)."""
    x = []
    for i in range(t):
        acc = b[i]
        for j in range(i):
            acc = acc - lg[i, j] @ x[j]  # tiles.py:196-197
        x.append(solve_triangular(lg[i, i], acc, lower=True, check_finite=False))
    return x


def backward_solve(lg, b, t):
    """l.T @ x == b, blocked (tiled.py:240-260)."""
    x = {}
    for i in reversed(range(t)):
        acc = b[i]
        for j in range(i + 1, t):
            acc = acc - lg[j, i].T @ x[j]  # tiles.py:200-201
        x[i] = solve_triangular(lg[i, i], acc, trans="T", lower=True, check_finite=False)
    return [x[i] for i in range(t)]


def forward_solve_matrix_col(lg, cross, t, c):
    """One column tile c of V = L^-1 B^T (tiled.py:277-295)."""
    col = []
    for i in range(t):
        acc = cross[c, i].T.copy()
        for j in range(i):
            acc = acc - lg[i, j] @ col[j]  # tiles.py:204-205
        col.append(solve_triangular(lg[i, i], acc, lower=True, check_finite=False))
    return col


def forward_solve_matrix(lg, cross, t, row_tiles):
    v = {}
    for c in range(row_tiles):
        col = forward_solve_matrix_col(lg, cross, t, c)
        for i in range(t):
            v[i, c] = col[i]
    return v


def gemv(cross, x, row_tiles, col_tiles):
    """mean = K* alpha (tiled.py:301-324)."""
    out = []
    for r in range(row_tiles):
        acc = cross[r, 0] @ x[0]
        for c in range(1, col_tiles):
            acc = acc + cross[r, c] @ x[c]
        out.append(acc)
    return out


def to_dense_lower(g, t, symmetric):
    """TiledMatrix.to_dense (tiled.py:70-80)."""
    ts = g[0, 0].shape[0]
    out = np.zeros((t * ts, t * ts))
    for i in range(t):
        for j in range(i + 1):
            out[i * ts:(i + 1) * ts, j * ts:(j + 1) * ts] = g[i, j]
            if symmetric and i != j:
                out[j * ts:(j + 1) * ts, i * ts:(i + 1) * ts] = g[i, j].T
    return out


def clamp_variances(var):
    """model.py:488-496; returns (clamped, worst) with worst < -slack flagged."""
    bad = var < -_VARIANCE_SLACK
    if np.any(bad):
        raise ArithmeticError(f"variance {float(var[bad].min()):g} below -{_VARIANCE_SLACK:g}")
    return np.where(var < 0.0, 0.0, var)


# -- model (model.py) --------------------------------------------------------

class OracleGP:
    """The reference GPModel's numerics (model.py:91-485) on numpy tiles."""

    def __init__(self, z, y, t, l=1.0, nu=1.0, s2=0.1, trainable=(True, True, True),
                 cholesky=tiled_cholesky, assembly_workers=1):
        self.z = np.ascontiguousarray(z, dtype=np.float64)
        self.y = np.ascontiguousarray(y, dtype=np.float64)
        self.t = t
        self.l, self.nu, self.s2 = float(l), float(nu), float(s2)
        self.trainable = tuple(trainable)
        self._chol = cholesky
        self._workers = assembly_workers
        self.adam_m = np.zeros(3)
        self.adam_v = np.zeros(3)
        self.adam_step = 0
        self._invalidate()

    def _invalidate(self):
        self.factor = None
        self.beta = None
        self.alpha = None

    def set_params(self, l, nu, s2):
        self.l, self.nu, self.s2 = float(l), float(nu), float(s2)
        self._invalidate()

    def ensure_factor(self):  # model.py:169-177
        if self.factor is None:
            if self._workers > 1:
                k = assemble_covariance_threaded(self.z, self.l, self.nu, self.s2, self.t, self._workers)
            else:
                k = assemble_covariance(self.z, self.l, self.nu, self.s2, self.t)
            self.factor = self._chol(k, self.t)
            del k
            self.beta = self.alpha = None
        return self.factor

    def ensure_weights(self):  # model.py:179-186
        if self.alpha is None:
            lg = self.ensure_factor()
            ys = row_blocks(self.y, self.t)
            self.beta = forward_solve(lg, ys, self.t)
            self.alpha = backward_solve(lg, self.beta, self.t)
        return self.alpha

    def factor_dense(self):
        return to_dense_lower(self.ensure_factor(), self.t, symmetric=False)

    def log_likelihood(self):  # model.py:316-339
        self.ensure_weights()
        half_log_det = sum(float(np.sum(np.log(np.diagonal(self.factor[i, i]))))
                           for i in range(self.t))
        fit = sum(float(s @ s) for s in self.beta)
        return -half_log_det - 0.5 * fit - self.z.shape[0] * _HALF_LOG_2PI

    def _cross_and_mean(self, zt):  # model.py:188-208
        rt = math.gcd(self.t, zt.shape[0])
        cross = assemble_cross(zt, self.z, self.l, self.nu, rt, self.t)
        mean = gemv(cross, self.ensure_weights(), rt, self.t)
        return rt, cross, mean

    def predict(self, zt):
        _, _, mean = self._cross_and_mean(zt)
        return np.concatenate(mean)

    def predict_variance(self, zt, solver=None):  # model.py:280-314
        rt, cross, mean = self._cross_and_mean(zt)
        fsm = solver or forward_solve_matrix
        v = fsm(self.factor, cross, self.t, rt)
        segs = []
        for i in range(rt):
            acc = np.einsum("ij,ij->j", v[0, i], v[0, i])  # tiles.py:216-217
            for c in range(1, self.t):
                acc = acc + np.einsum("ij,ij->j", v[c, i], v[c, i])
            segs.append(self.nu - acc)
        return np.concatenate(mean), clamp_variances(np.concatenate(segs))

    def predict_full_cov(self, zt):  # model.py:242-278
        rt, cross, mean = self._cross_and_mean(zt)
        v = forward_solve_matrix(self.factor, cross, self.t, rt)
        prior = assemble_covariance(zt, self.l, self.nu, self.s2, rt, include_noise=False)
        grid = {}
        for i in range(rt):
            for j in range(i + 1):
                acc = prior[i, j]
                for c in range(self.t):
                    acc = acc - v[c, i].T @ v[c, j]  # tiles.py:208-209
                grid[i, j] = acc
        sigma = to_dense_lower(grid, rt, symmetric=True)
        diag = clamp_variances(np.diagonal(sigma).copy())
        np.fill_diagonal(sigma, diag)
        return np.concatenate(mean), sigma

    def loss_gradients(self):  # model.py:341-435
        tl, tv, tn = self.trainable
        if not (tl or tv or tn):
            return (0.0, 0.0, 0.0)
        alpha = self.ensure_weights()
        lg, t, n = self.factor, self.t, self.z.shape[0]
        ts = n // t
        eye, zero = np.eye(ts), np.zeros((ts, ts))
        ident = {(i, j): (eye if i == j else zero) for i in range(t) for j in range(t)}
        x = forward_solve_matrix(lg, ident, t, t)
        kinv = {}
        for r in range(t):
            for c in range(r + 1):
                acc = None
                for i in range(max(r, c), t):
                    if acc is None:
                        acc = x[i, r].T @ x[i, c]
                    else:
                        acc = acc + x[i, r].T @ x[i, c]  # tiles.py:212-213
                kinv[r, c] = acc

        def quadratic_terms(dk):
            parts = []
            for r in range(t):
                for c in range(r + 1):
                    w = 1.0 if r == c else 2.0
                    parts.append(w * float(np.sum(kinv[r, c] * dk[r, c])))
                    parts.append(-w * float(alpha[r] @ dk[r, c] @ alpha[c]))
            return 0.5 * sum(parts)

        gl = gv = gn = 0.0
        if tl:
            gl = quadratic_terms(assemble_dk_lengthscale(self.z, self.l, self.nu, t))
        if tv:
            gv = quadratic_terms(assemble_dk_vertical(self.z, self.l, t))
        if tn:
            trace = sum(float(np.sum(x[i, c] ** 2)) for i in range(t) for c in range(t))
            fit = sum(float(s @ s) for s in alpha)
            gn = 0.5 * (trace - fit)
        return (gl, gv, gn)

    def optimize(self, lr=0.1, beta1=0.9, beta2=0.999, eps=1e-8, iterations=100):
        """Adam on log-parameters (model.py:437-485)."""
        history = []
        for _ in range(iterations):
            self.adam_step += 1
            grads = np.array(self.loss_gradients())
            theta = np.array([self.l, self.nu, self.s2])
            g = grads * theta
            self.adam_m = beta1 * self.adam_m + (1 - beta1) * g
            self.adam_v = beta2 * self.adam_v + (1 - beta2) * g * g
            m_hat = self.adam_m / (1 - beta1 ** self.adam_step)
            v_hat = self.adam_v / (1 - beta2 ** self.adam_step)
            step = lr * m_hat / (np.sqrt(v_hat) + eps)
            mask = np.array(self.trainable, dtype=bool)
            u = np.where(mask, np.log(np.maximum(theta, 1e-300)) - step, 0.0)
            theta = np.where(mask, np.exp(u), theta)
            if mask[2]:
                theta[2] = max(theta[2], 1e-12)
            self.set_params(float(theta[0]), float(theta[1]), float(theta[2]))
            history.append(-self.log_likelihood())
        return history


# -- independent dense checks (pkg/tests/oracles.py:11-78 restated) ----------

def dense_k(z, l, nu, s2):
    d2 = ((z[:, None, :] - z[None, :, :]) ** 2).sum(-1)
    return nu * np.exp(-d2 / (2.0 * l ** 2)) + s2 * np.eye(z.shape[0])


def rel_fro(a, b):
    """||a - b||_F / ||b||_F."""
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den else 1.0))
