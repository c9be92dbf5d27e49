// Blocked vector solves, deterministic reductions and layout helpers.
//
// Forward/backward substitution (taskgp tiled.py:215-260 with tiles.py
// solve_lower_vec / solve_lower_t_vec / matvec_sub / matvec_t_sub :170-201)
// run right-looking over tile columns: the diagonal solve is a product with
// the inverted diagonal tile, the off-diagonal work a GEMV over the column
// (forward) or row (backward) panel.  Both are HBM/latency bound: each reads
// the lower factor exactly once.  All reductions use a fixed order (warp
// butterflies and sequential partial sums), never floating-point atomics,
// so results are bitwise reproducible run to run.
#include "kernels.cuh"

namespace gpb {

namespace {

__global__ void __launch_bounds__(256) fwd_diag_kernel(const double* dinv, const double* yhat,
                                                       double* beta, int bi) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * 8 + warp;
  if (r >= bi) return;
  const double* row = dinv + static_cast<int64_t>(r) * bi;
  double s = 0.0;
  for (int c = lane; c <= r; c += 32) s += row[c] * yhat[c];
  s = warp_sum(s);
  if (lane == 0) beta[r] = s;
}

__global__ void __launch_bounds__(256) fwd_update_kernel(const double* ltiles, int i, int bi,
                                                         const double* beta_i, double* yhat) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t gr = static_cast<int64_t>(blockIdx.x) * 8 + warp;  // row within tile rows > i
  const int r = i + 1 + static_cast<int>(gr / bi);
  const int row = static_cast<int>(gr % bi);
  const double* L = ltiles + tri_rm(r, i) * bi * bi + static_cast<int64_t>(row) * bi;
  double s = 0.0;
  for (int c = lane; c < bi; c += 32) s += L[c] * beta_i[c];
  s = warp_sum(s);
  if (lane == 0) yhat[static_cast<int64_t>(r) * bi + row] -= s;
}

// out[c] (+)= sign * sum_r M[r][c] v[r] for 32 columns per CTA; 8 warps split r.
__global__ void __launch_bounds__(256) colgemv_kernel(const double* M, int64_t tile_stride, int bi,
                                                      const double* v, double* out, int accumulate) {
  __shared__ double part[8][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cpt = bi / 32;  // column groups per tile
  const int q = blockIdx.x / cpt;
  const int c = (blockIdx.x % cpt) * 32 + lane;
  const double* T = M + static_cast<int64_t>(q) * tile_stride;
  double s = 0.0;
  for (int r = warp; r < bi; r += 8) s += T[static_cast<int64_t>(r) * bi + c] * v[r];
  part[warp][lane] = s;
  __syncthreads();
  if (warp == 0) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += part[w][lane];
    double* o = out + static_cast<int64_t>(q) * bi + c;
    if (accumulate) *o -= t; else *o = t;
  }
}

__global__ void __launch_bounds__(1024) reduce_kernel(const double* x, int64_t n, int square,
                                                      const double* logdiag, int T, double* out) {
  __shared__ double red[1024];
  const int tid = threadIdx.x;
  double s = 0.0;
  for (int64_t k = tid; k < n; k += 1024) s += square ? x[k] * x[k] : x[k];
  red[tid] = s;
  __syncthreads();
  for (int w = 512; w > 0; w >>= 1) {
    if (tid < w) red[tid] += red[tid + w];
    __syncthreads();
  }
  if (tid == 0) {
    if (logdiag) {
      double l = 0.0;
      for (int k = 0; k < T; ++k) l += logdiag[k];
      out[0] = l;
      out[1] = red[0];
    } else {
      out[0] = red[0];
    }
  }
}

__global__ void pred_finalize_kernel(const double* mpart, int64_t nmrb, const double* sq,
                                     int64_t nsrb, int64_t ld, int64_t mc, double nu, double* mean,
                                     double* var) {
  const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= mc) return;
  if (mean) {
    double s = 0.0;
    for (int64_t r = 0; r < nmrb; ++r) s += mpart[r * ld + c];
    mean[c] = s;
  }
  if (var) {
    double s = 0.0;
    for (int64_t r = 0; r < nsrb; ++r) s += sq[r * ld + c];
    var[c] = nu - s;
  }
}

__global__ void symmetrize_kernel(double* S, int64_t mp, int64_t m) {
  __shared__ double tile[32][33];
  const int64_t bx = blockIdx.x, by = blockIdx.y;  // source block (row by, col bx) in the lower part
  if (bx > by) return;
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int k = ty; k < 32; k += 8) {
    const int64_t r = by * 32 + k, c = bx * 32 + tx;
    tile[k][tx] = (r < m && c < m) ? S[r * mp + c] : 0.0;
  }
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {
    const int64_t r = bx * 32 + k, c = by * 32 + tx;  // destination (upper) entry (r, c), c > r
    if (r < m && c < m && c > r) S[r * mp + c] = tile[tx][k];
  }
}

__global__ void pad_vector_kernel(const double* src, double* dst, int64_t np_, PadMap pm) {
  const int64_t P = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (P >= np_) return;
  dst[P] = pm.valid(P) ? src[(P / pm.bp_user) * pm.b_user + P % pm.bp_user] : 0.0;
}

__global__ void pad_rows_kernel(const double* src, double* dst, int64_t np_, int d, PadMap pm) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= np_ * d) return;
  const int64_t P = e / d;
  const int k = static_cast<int>(e % d);
  dst[e] = pm.valid(P) ? src[((P / pm.bp_user) * pm.b_user + P % pm.bp_user) * d + k] : 0.0;
}

__global__ void export_lower_kernel(const double* tiles, int bi, int64_t n, int64_t row0,
                                    int64_t rows, PadMap pm, double* out) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= rows * n) return;
  const int64_t r = row0 + e / n, c = e % n;
  const int64_t P = (r / pm.b_user) * pm.bp_user + r % pm.b_user;
  const int64_t Q = (c / pm.b_user) * pm.bp_user + c % pm.b_user;
  const int64_t ti = P / bi, tj = Q / bi;
  out[e] = (tj > ti) ? 0.0 : tiles[tri_rm(ti, tj) * bi * bi + (P % bi) * bi + (Q % bi)];
}

__global__ void copy_panel_kernel(double* ltiles, const double* scratch, int k, int bi) {
  const int64_t per = static_cast<int64_t>(bi) * bi / 2;
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t q = e / per, w = e % per;
  const double2* src = reinterpret_cast<const double2*>(scratch + q * bi * bi);
  double2* dst = reinterpret_cast<double2*>(ltiles + tri_rm(k + 1 + q, k) * bi * bi);
  dst[w] = src[w];
}

__global__ void __launch_bounds__(256) gemv_n_jobs_kernel(const GemvJob* jobs, int bi, double alpha,
                                                          int accumulate) {
  const int per = bi / 8;
  const GemvJob jb = jobs[blockIdx.x / per];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = (blockIdx.x % per) * 8 + warp;
  const double* row = jb.a + static_cast<int64_t>(r) * bi;
  double s = 0.0;
  for (int c = lane; c < bi; c += 32) s += row[c] * jb.x[c];
  s = warp_sum(s);
  if (lane == 0) jb.y[r] = (accumulate ? jb.y[r] : 0.0) + alpha * s;
}

__global__ void __launch_bounds__(256) gemv_t_jobs_kernel(const GemvJob* jobs, int bi, double alpha,
                                                          int accumulate) {
  __shared__ double part[8][32];
  const int per = bi / 32;
  const GemvJob jb = jobs[blockIdx.x / per];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = (blockIdx.x % per) * 32 + lane;
  double s = 0.0;
  for (int r = warp; r < bi; r += 8) s += jb.a[static_cast<int64_t>(r) * bi + c] * jb.x[r];
  part[warp][lane] = s;
  __syncthreads();
  if (warp == 0) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += part[w][lane];
    jb.y[c] = (accumulate ? jb.y[c] : 0.0) + alpha * t;
  }
}

__global__ void combine_kernel(const double* base, const double* parts, int64_t nparts, int64_t len,
                               double* out) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= len) return;
  double s = base[e];
  for (int64_t p = 0; p < nparts; ++p) s -= parts[p * len + e];
  out[e] = s;
}

}  // namespace

cudaError_t launch_gemv_jobs(const GemvJob* jobs, int64_t njobs, int bi, int trans, double alpha,
                             int accumulate, cudaStream_t s) {
  if (njobs <= 0) return cudaSuccess;
  if (trans)
    gemv_t_jobs_kernel<<<static_cast<unsigned>(njobs * (bi / 32)), 256, 0, s>>>(jobs, bi, alpha,
                                                                                 accumulate);
  else
    gemv_n_jobs_kernel<<<static_cast<unsigned>(njobs * (bi / 8)), 256, 0, s>>>(jobs, bi, alpha,
                                                                                accumulate);
  return cudaGetLastError();
}

cudaError_t launch_combine(const double* base, const double* parts, int64_t nparts, int64_t len,
                           double* out, cudaStream_t s) {
  if (len <= 0) return cudaSuccess;
  combine_kernel<<<static_cast<unsigned>((len + 255) / 256), 256, 0, s>>>(base, parts, nparts, len, out);
  return cudaGetLastError();
}

cudaError_t launch_fwd_diag(const double* dinv, const double* yhat, double* beta, int bi,
                            cudaStream_t s) {
  fwd_diag_kernel<<<bi / 8, 256, 0, s>>>(dinv, yhat, beta, bi);
  return cudaGetLastError();
}

cudaError_t launch_fwd_update(const double* ltiles, int T, int i, int bi, const double* beta_i,
                              double* yhat, cudaStream_t s) {
  const int64_t rows = static_cast<int64_t>(T - i - 1) * bi;
  if (rows <= 0) return cudaSuccess;
  fwd_update_kernel<<<static_cast<unsigned>(rows / 8), 256, 0, s>>>(ltiles, i, bi, beta_i, yhat);
  return cudaGetLastError();
}

cudaError_t launch_bwd_diag(const double* dinv, const double* bhat, double* alpha, int bi,
                            cudaStream_t s) {
  colgemv_kernel<<<bi / 32, 256, 0, s>>>(dinv, 0, bi, bhat, alpha, 0);
  return cudaGetLastError();
}

cudaError_t launch_bwd_update(const double* ltiles, int i, int bi, const double* alpha_i,
                              double* bhat, cudaStream_t s) {
  if (i <= 0) return cudaSuccess;
  const double* row_panel = ltiles + h_tri_rm(i, 0) * bi * bi;
  colgemv_kernel<<<static_cast<unsigned>(i * (bi / 32)), 256, 0, s>>>(
      row_panel, static_cast<int64_t>(bi) * bi, bi, alpha_i, bhat, 1);
  return cudaGetLastError();
}

cudaError_t launch_loss_terms(const double* logdiag, int T, const double* x, int64_t n,
                              double* out, cudaStream_t s) {
  reduce_kernel<<<1, 1024, 0, s>>>(x, n, 1, logdiag, T, out);
  return cudaGetLastError();
}

cudaError_t launch_reduce(const double* part, int64_t n, double* out, cudaStream_t s) {
  reduce_kernel<<<1, 1024, 0, s>>>(part, n, 0, nullptr, 0, out);
  return cudaGetLastError();
}

cudaError_t launch_pred_finalize(const double* mpart, int64_t nmrb, const double* sq,
                                 int64_t nsrb, int64_t ld, int64_t mc, double nu, double* mean,
                                 double* var, cudaStream_t s) {
  const unsigned blocks = static_cast<unsigned>((mc + 255) / 256);
  pred_finalize_kernel<<<blocks, 256, 0, s>>>(mpart, nmrb, sq, nsrb, ld, mc, nu, mean, var);
  return cudaGetLastError();
}

cudaError_t launch_symmetrize(double* S, int64_t mp, int64_t m, cudaStream_t s) {
  dim3 grid(static_cast<unsigned>((m + 31) / 32), static_cast<unsigned>((m + 31) / 32));
  symmetrize_kernel<<<grid, dim3(32, 8), 0, s>>>(S, mp, m);
  return cudaGetLastError();
}

cudaError_t launch_pad_vector(const double* src, double* dst, int64_t np_, PadMap pm,
                              cudaStream_t s) {
  pad_vector_kernel<<<static_cast<unsigned>((np_ + 255) / 256), 256, 0, s>>>(src, dst, np_, pm);
  return cudaGetLastError();
}

cudaError_t launch_pad_rows(const double* src, double* dst, int64_t np_, int d, PadMap pm,
                            cudaStream_t s) {
  const int64_t n = np_ * d;
  pad_rows_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(src, dst, np_, d, pm);
  return cudaGetLastError();
}

cudaError_t launch_export_lower(const double* tiles, int bi, int64_t n, int64_t row0, int64_t rows,
                                PadMap pm, double* out, cudaStream_t s) {
  const int64_t e = rows * n;
  if (e <= 0) return cudaSuccess;
  export_lower_kernel<<<static_cast<unsigned>((e + 255) / 256), 256, 0, s>>>(tiles, bi, n, row0, rows,
                                                                              pm, out);
  return cudaGetLastError();
}

namespace {
__global__ void set_diag_kernel(double* G, int64_t ld, int64_t count) {
  const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c < count) G[c * ld + c] = 1.0;
}
}  // namespace

cudaError_t launch_set_diag(double* G, int64_t ld, int64_t count, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  set_diag_kernel<<<static_cast<unsigned>((count + 255) / 256), 256, 0, s>>>(G, ld, count);
  return cudaGetLastError();
}

cudaError_t launch_copy_panel(double* ltiles, const double* scratch, int T, int k, int bi,
                              cudaStream_t s) {
  const int64_t e = static_cast<int64_t>(T - k - 1) * bi * bi / 2;
  if (e <= 0) return cudaSuccess;
  copy_panel_kernel<<<static_cast<unsigned>(e / 256), 256, 0, s>>>(ltiles, scratch, k, bi);
  return cudaGetLastError();
}

}  // namespace gpb
