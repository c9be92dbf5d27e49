// Squared-exponential (SEK) tile kernels.
//
// Replaces taskgp covariance.py: _sq_dists/_kernel_block (:65-82),
// assemble_covariance (:118-164), assemble_cross_covariance (:167-193) and
// the dK/dtheta assemblies (:196-230), which here are never materialised:
// the gradient trace pass regenerates e and d^2 on the fly.
//
// Every entry uses direct differences summed over the features in a fixed
// order, so an entry depends only on its two rows: assembled matrices are
// exactly symmetric and exactly tiling-invariant (the reference's own
// invariants, test_covariance.py:77-98).
//
// CTA = 64 x 64 entries, 256 threads, thread (tx, ty) owns rows ty + 16 ii and
// cols tx + 16 jj so that shared-memory reads broadcast / stay conflict-free
// and each half-warp stores 128 contiguous bytes.
#include "kernels.cuh"

namespace gpb {

namespace {

constexpr int SB = kSekBlock;  // entries per CTA side
// staging row pitch: the transposing stores sa[dd][r] of 32 consecutive
// features would all hit one bank with a pitch of 64 doubles
constexpr int SBP = SB + 1;
constexpr int DC = 32;  // feature chunk
constexpr int R = SB / 16;  // entries per thread per dimension
constexpr int ST = 256;  // threads

struct Frag {
  double v[R][R];
};

// d2[ii][jj] for rows ra0 + ty + 16 ii of za (ld d) and rows rb0 + tx + 16 jj of zb.
GPB_DEVINL void sq_dists_blk(Frag& d2, const double* za, int64_t ra0, const double* zb, int64_t rb0,
                            int d, double (*sa)[SBP], double (*sb)[SBP], int tx, int ty, int tid) {
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < R; ++j) d2.v[i][j] = 0.0;
  for (int d0 = 0; d0 < d; d0 += DC) {
    const int dn = min(DC, d - d0);
    __syncthreads();
    for (int e = tid; e < SB * DC; e += ST) {
      const int r = e / DC, dd = e % DC;
      if (dd < dn) {
        sa[dd][r] = za[(ra0 + r) * d + d0 + dd];
        sb[dd][r] = zb[(rb0 + r) * d + d0 + dd];
      }
    }
    __syncthreads();
    for (int dd = 0; dd < dn; ++dd) {
      double a[R], b[R];
#pragma unroll
      for (int i = 0; i < R; ++i) a[i] = sa[dd][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < R; ++j) b[j] = sb[dd][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < R; ++i)
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const double df = a[i] - b[j];
          d2.v[i][j] = fma(df, df, d2.v[i][j]);
        }
    }
  }
}

GPB_DEVINL double sek(double d2, const SekParams& sp) {
  // covariance.py:79-81 order: d2 *= -1/(2 l^2); exp; *= nu
  return exp(d2 * sp.neg_half_inv_l2) * sp.vertical;
}

// fixed-order block reduction of one double per thread (ST threads)
GPB_DEVINL double block_sum(double v, double* red, int tid) {
  __syncthreads();
  red[tid] = v;
  __syncthreads();
#pragma unroll
  for (int s = ST / 2; s > 0; s >>= 1) {
    if (tid < s) red[tid] += red[tid + s];
    __syncthreads();
  }
  return red[0];
}

// one 64x64 block (rb, cb) of tile (ti, tj), written to `tile`
GPB_DEVINL void assemble_block(double* tile, int ti, int tj, int rb, int cb, const double* zp,
                               int d, int bi, PadMap pm, SekParams sp, int add_noise,
                               double (*sa)[SBP], double (*sb)[SBP]) {
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t P0 = static_cast<int64_t>(ti) * bi + rb * SB;
  const int64_t Q0 = static_cast<int64_t>(tj) * bi + cb * SB;
  Frag d2;
  sq_dists_blk(d2, zp, P0, zp, Q0, d, sa, sb, tx, ty, tid);
  double* out = tile + static_cast<int64_t>(rb * SB) * bi + cb * SB;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int64_t P = P0 + ty + 16 * i;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const int64_t Q = Q0 + tx + 16 * j;
      double v;
      if (pm.valid(P) && pm.valid(Q)) {
        v = sek(d2.v[i][j], sp);
        if (add_noise && P == Q) v += sp.noise;
      } else {
        v = (P == Q) ? 1.0 : 0.0;  // decoupled identity padding
      }
      out[static_cast<int64_t>(ty + 16 * i) * bi + tx + 16 * j] = v;
    }
  }
}

__global__ void __launch_bounds__(ST) assemble_lower_kernel(double* tiles, const int2* tile_ij,
                                                            int64_t t0, const double* zp, int d,
                                                            int bi, PadMap pm, SekParams sp,
                                                            int add_noise) {
  __shared__ double sa[DC][SBP], sb[DC][SBP];
  const int nbs = bi / SB;
  const int64_t t = t0 + blockIdx.x / (nbs * nbs);
  const int blk = blockIdx.x % (nbs * nbs);
  const int2 ij = tile_ij[t];
  assemble_block(tiles + t * bi * bi, ij.x, ij.y, blk / nbs, blk % nbs, zp, d, bi, pm, sp,
                 add_noise, sa, sb);
}

// tiles given as (i, j, destination) descriptors (external schedulers)
__global__ void __launch_bounds__(ST) assemble_desc_kernel(const TileDesc* desc, const double* zp,
                                                           int d, int bi, PadMap pm, SekParams sp,
                                                           int add_noise) {
  __shared__ double sa[DC][SBP], sb[DC][SBP];
  const int nbs = bi / SB;
  const TileDesc td = desc[blockIdx.x / (nbs * nbs)];
  const int blk = blockIdx.x % (nbs * nbs);
  assemble_block(td.ptr, td.i, td.j, blk / nbs, blk % nbs, zp, d, bi, pm, sp, add_noise, sa, sb);
}

__global__ void __launch_bounds__(ST) cross_kernel(double* B, int64_t ldb, double* mpart,
                                                   const double* alpha, const double* zp,
                                                   const double* zt, int64_t mc, int d,
                                                   PadMap pm, SekParams sp) {
  __shared__ double sa[DC][SBP], sb[DC][SBP];
  __shared__ double red[16][SB];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t P0 = static_cast<int64_t>(blockIdx.x) * SB;  // training rows
  const int64_t C0 = static_cast<int64_t>(blockIdx.y) * SB;  // test columns
  // clamp test rows for loading (rows >= mc are masked below)
  const int64_t c_load0 = C0;
  Frag d2;
  // zt rows beyond mc: read a valid row instead (masked) by using min()
  {
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
      for (int j = 0; j < R; ++j) d2.v[i][j] = 0.0;
    for (int d0 = 0; d0 < d; d0 += DC) {
      const int dn = min(DC, d - d0);
      __syncthreads();
      for (int e = tid; e < SB * DC; e += ST) {
        const int r = e / DC, dd = e % DC;
        if (dd < dn) {
          sa[dd][r] = zp[(P0 + r) * d + d0 + dd];
          const int64_t cr = min(c_load0 + r, mc - 1);
          sb[dd][r] = zt[cr * d + d0 + dd];
        }
      }
      __syncthreads();
      for (int dd = 0; dd < dn; ++dd) {
        double a[R], b[R];
#pragma unroll
        for (int i = 0; i < R; ++i) a[i] = sa[dd][ty + 16 * i];
#pragma unroll
        for (int j = 0; j < R; ++j) b[j] = sb[dd][tx + 16 * j];
#pragma unroll
        for (int i = 0; i < R; ++i)
#pragma unroll
          for (int j = 0; j < R; ++j) {
            const double df = a[i] - b[j];
            d2.v[i][j] = fma(df, df, d2.v[i][j]);
          }
      }
    }
  }
  double msum[R] = {};
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int64_t P = P0 + ty + 16 * i;
    const bool pv = pm.valid(P);
    const double a = alpha ? alpha[P] : 0.0;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const int64_t c = C0 + tx + 16 * j;
      const double v = (pv && c < mc) ? sek(d2.v[i][j], sp) : 0.0;
      B[P * ldb + c] = v;
      msum[j] += v * a;
    }
  }
  if (mpart) {
#pragma unroll
    for (int j = 0; j < R; ++j) red[ty][tx + 16 * j] = msum[j];
    __syncthreads();
    if (tid < SB) {
      double s = 0.0;
#pragma unroll
      for (int r = 0; r < 16; ++r) s += red[r][tid];
      mpart[static_cast<int64_t>(blockIdx.x) * ldb + C0 + tid] = s;
    }
  }
}

// S (ld lds) = nu exp(-|za_r - zb_c|^2 / 2l^2) for r < ma, c < mb, else 0
__global__ void __launch_bounds__(ST) prior_kernel(double* S, int64_t lds, const double* za,
                                                   int64_t ma, const double* zb, int64_t mb, int d,
                                                   SekParams sp) {
  __shared__ double sa[DC][SBP], sb[DC][SBP];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t R0 = static_cast<int64_t>(blockIdx.x) * SB;
  const int64_t C0 = static_cast<int64_t>(blockIdx.y) * SB;
  Frag d2;
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < R; ++j) d2.v[i][j] = 0.0;
  for (int d0 = 0; d0 < d; d0 += DC) {
    const int dn = min(DC, d - d0);
    __syncthreads();
    for (int e = tid; e < SB * DC; e += ST) {
      const int r = e / DC, dd = e % DC;
      if (dd < dn) {
        sa[dd][r] = za[min(R0 + r, ma - 1) * d + d0 + dd];
        sb[dd][r] = zb[min(C0 + r, mb - 1) * d + d0 + dd];
      }
    }
    __syncthreads();
    for (int dd = 0; dd < dn; ++dd) {
      double a[R], b[R];
#pragma unroll
      for (int i = 0; i < R; ++i) a[i] = sa[dd][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < R; ++j) b[j] = sb[dd][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < R; ++i)
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const double df = a[i] - b[j];
          d2.v[i][j] = fma(df, df, d2.v[i][j]);
        }
    }
  }
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int64_t r = R0 + ty + 16 * i;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const int64_t c = C0 + tx + 16 * j;
      S[r * lds + c] = (r < ma && c < mb) ? sek(d2.v[i][j], sp) : 0.0;
    }
  }
}

__global__ void __launch_bounds__(ST) trace_kernel(const double* kinv, const int2* tile_ij,
                                                   const double* zp, const double* alpha, int d,
                                                   int bi, PadMap pm, SekParams sp, TraceTiles tt,
                                                   double* part_l, double* part_v, double* part_t) {
  __shared__ double sa[DC][SBP], sb[DC][SBP];
  __shared__ double red[ST];
  const int nbs = bi / SB;
  const int64_t t = blockIdx.x / (nbs * nbs);
  const int blk = blockIdx.x % (nbs * nbs);
  const int rb = blk / nbs, cb = blk % nbs;
  const int2 ij = tile_ij[t];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  // K^-1 and dK/dtheta are symmetric: in a diagonal tile only the blocks on
  // and below the diagonal are read (strictly lower ones twice), so the
  // K^-1 producer may leave the strictly upper blocks of diagonal tiles unset
  if (ij.x == ij.y && rb < cb) {
    if (tid == 0) {
      part_l[blockIdx.x] = 0.0;
      part_v[blockIdx.x] = 0.0;
      if (part_t) part_t[blockIdx.x] = 0.0;
    }
    return;
  }
  const int64_t P0 = static_cast<int64_t>(ij.x) * bi + rb * SB;
  const int64_t Q0 = static_cast<int64_t>(ij.y) * bi + cb * SB;
  Frag d2;
  sq_dists_blk(d2, zp, P0, zp, Q0, d, sa, sb, tx, ty, tid);
  // packed tiles (ld == 0): tile t at kinv + t * bi^2; dense column panel
  // (ld > 0): row P at kinv + (P - row0 * bi) * ld, columns from slot[t] * bi
  // (or Q - col0 * bi)
  const int64_t ldk = tt.ld > 0 ? tt.ld : bi;
  const int64_t pc = tt.slot ? static_cast<int64_t>(tt.slot[t]) * bi + cb * SB
                             : Q0 - static_cast<int64_t>(tt.col0) * bi;
  const double* kt = tt.ld > 0 ? kinv + (P0 - static_cast<int64_t>(tt.row0) * bi) * tt.ld + pc
                               : kinv + t * bi * bi + static_cast<int64_t>(rb * SB) * bi + cb * SB;
  double sl = 0.0, sv = 0.0, st = 0.0;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int64_t P = P0 + ty + 16 * i;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const int64_t Q = Q0 + tx + 16 * j;
      if (pm.valid(P) && pm.valid(Q)) {
        const double e = exp(d2.v[i][j] * sp.neg_half_inv_l2);
        const double kv = kt[static_cast<int64_t>(ty + 16 * i) * ldk + tx + 16 * j];
        const double coef = kv - alpha[P] * alpha[Q];
        sl += coef * e * d2.v[i][j];
        sv += coef * e;
        if (P == Q) st += kv;
      }
    }
  }
  const double w = (ij.x == ij.y && rb == cb) ? 1.0 : 2.0;
  const double tl = block_sum(sl, red, tid);
  const double tv = block_sum(sv, red, tid);
  const double ts = part_t ? block_sum(st, red, tid) : 0.0;
  if (tid == 0) {
    part_l[blockIdx.x] = w * tl;
    part_v[blockIdx.x] = w * tv;
    if (part_t) part_t[blockIdx.x] = ts;
  }
}

__global__ void __launch_bounds__(ST) tiles_sumsq_kernel(const double* x, const int2* tile_ij,
                                                         int bi, PadMap pm, double* part) {
  __shared__ double red[ST];
  const int nbs = bi / SB;
  const int64_t t = blockIdx.x / (nbs * nbs);
  const int blk = blockIdx.x % (nbs * nbs);
  const int rb = blk / nbs, cb = blk % nbs;
  const int2 ij = tile_ij[t];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t P0 = static_cast<int64_t>(ij.x) * bi + rb * SB;
  const int64_t Q0 = static_cast<int64_t>(ij.y) * bi + cb * SB;
  const double* xt = x + t * bi * bi + static_cast<int64_t>(rb * SB) * bi + cb * SB;
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < R; ++j) {
      if (pm.valid(P0 + ty + 16 * i) && pm.valid(Q0 + tx + 16 * j)) {
        const double v = xt[static_cast<int64_t>(ty + 16 * i) * bi + tx + 16 * j];
        s += v * v;
      }
    }
  const double tot = block_sum(s, red, tid);
  if (tid == 0) part[blockIdx.x] = tot;
}

}  // namespace

cudaError_t launch_assemble_lower(double* tiles, const int2* tile_ij, int64_t t0, int64_t t1,
                                  const double* zp, int d, int bi, PadMap pm, SekParams sp,
                                  bool add_noise, cudaStream_t s) {
  const int64_t nbs = bi / SB;
  const int64_t blocks = (t1 - t0) * nbs * nbs;
  if (blocks <= 0) return cudaSuccess;
  assemble_lower_kernel<<<static_cast<unsigned>(blocks), ST, 0, s>>>(tiles, tile_ij, t0, zp, d, bi,
                                                                     pm, sp, add_noise ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_assemble_desc(const TileDesc* desc, int64_t ntiles, const double* zp, int d,
                                 int bi, PadMap pm, SekParams sp, bool add_noise, cudaStream_t s) {
  const int64_t nbs = bi / SB;
  if (ntiles <= 0) return cudaSuccess;
  assemble_desc_kernel<<<static_cast<unsigned>(ntiles * nbs * nbs), ST, 0, s>>>(desc, zp, d, bi, pm, sp,
                                                                               add_noise ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_cross(double* B, int64_t ldb, double* mpart, const double* alpha,
                         const double* zp, int64_t np_, const double* zt, int64_t mc,
                         int64_t mcp, int d, PadMap pm, SekParams sp, cudaStream_t s) {
  dim3 grid(static_cast<unsigned>(np_ / SB), static_cast<unsigned>(mcp / SB));
  cross_kernel<<<grid, ST, 0, s>>>(B, ldb, mpart, alpha, zp, zt, mc, d, pm, sp);
  return cudaGetLastError();
}

cudaError_t launch_prior(double* S, int64_t mp, const double* zt, int64_t m, int d, SekParams sp,
                         cudaStream_t s) {
  return launch_prior2(S, mp, mp, mp, zt, m, zt, m, d, sp, s);
}

cudaError_t launch_prior2(double* S, int64_t lds, int64_t mpa, int64_t mpb, const double* za,
                          int64_t ma, const double* zb, int64_t mb, int d, SekParams sp,
                          cudaStream_t s) {
  if (mpa <= 0 || mpb <= 0) return cudaSuccess;
  dim3 grid(static_cast<unsigned>(mpa / SB), static_cast<unsigned>(mpb / SB));
  prior_kernel<<<grid, ST, 0, s>>>(S, lds, za, ma, zb, mb, d, sp);
  return cudaGetLastError();
}

cudaError_t launch_trace(const double* kinv, const int2* tile_ij, int64_t ntiles, TraceTiles tt,
                         const double* zp, const double* alpha, int d, int bi, PadMap pm,
                         SekParams sp, double* part_l, double* part_v, double* part_t,
                         cudaStream_t s) {
  const int64_t nbs = bi / SB;
  if (ntiles <= 0) return cudaSuccess;
  trace_kernel<<<static_cast<unsigned>(ntiles * nbs * nbs), ST, 0, s>>>(
      kinv, tile_ij, zp, alpha, d, bi, pm, sp, tt, part_l, part_v, part_t);
  return cudaGetLastError();
}

cudaError_t launch_tiles_sumsq(const double* x, const int2* tile_ij_cm, int64_t ntiles, int bi,
                               PadMap pm, double* part, cudaStream_t s) {
  const int64_t nbs = bi / SB;
  tiles_sumsq_kernel<<<static_cast<unsigned>(ntiles * nbs * nbs), ST, 0, s>>>(x, tile_ij_cm, bi, pm,
                                                                              part);
  return cudaGetLastError();
}

}  // namespace gpb
