// Launch interfaces of the non-GEMM kernels (potrf.cu, sek.cu, solve.cu).
#pragma once
#include "common.cuh"

namespace gpb {

// Index map of the padded internal layout: padded position P is real iff
// P % bp_user < b_user; its original index is (P / bp_user) * b_user + P % bp_user.
struct PadMap {
  int bp_user;
  int b_user;
  GPB_DEVINL bool valid(int64_t P) const { return (P % bp_user) < b_user; }
};

struct PotrfArgs {
  double* tile;     // bi x bi, in place -> L_kk (upper zeroed)
  double* dinv;     // bi x bi output: L_kk^-1
  double* logdiag;  // [T] per-tile sum of log L_jj over real pivots
  int* info;        // -1, or first failing original pivot index
  int bi;
  int tile_index;
  int tile_off;     // padded global position of the tile's first row
  int bp_user, b_user;
  int trtri_only;   // 1: tile already holds L; only form dinv = L^-1
  long long* prof;  // optional per-phase cycle counters (GPB_POTRF_PROF), else null
  int tiles;        // diagonal tiles of the factorisation (cluster-size hint), 0 if unknown
  int remaining;    // diagonal tiles from this one to the end (cluster-size hint), 0 if unknown
};
cudaError_t launch_potrf(const PotrfArgs& a, cudaStream_t s);
cudaError_t potrf_init_attributes();

// ---- squared-exponential tiles (sek.cu) -----------------------------------
// Entries per CTA side of the SEK kernels (tile sizes are multiples of it);
// the gradient trace pass writes one partial per kSekBlock^2 block and the
// cross kernel one mean partial per kSekBlock training rows.
constexpr int kSekBlock = 64;
struct SekParams {
  double lengthscale, vertical, noise;
  double neg_half_inv_l2;  // -1 / (2 l^2)   (covariance.py:79)
};

// Lower tiles [t0, t1) of the packed row-major tile grid (tile list entries
// are (i, j) pairs).  Noise goes on the global diagonal when add_noise.
cudaError_t launch_assemble_lower(double* tiles, const int2* tile_ij, int64_t t0, int64_t t1,
                                  const double* zp, int d, int bi, PadMap pm, SekParams sp,
                                  bool add_noise, cudaStream_t s);

// Tile descriptor for external schedulers: tile (i, j) of the padded grid,
// written/read at `ptr` (bi x bi row-major).  Same layout as gpb_tile_desc.
struct TileDesc {
  int i, j;
  double* ptr;
};
cudaError_t launch_assemble_desc(const TileDesc* desc, int64_t ntiles, const double* zp, int d,
                                 int bi, PadMap pm, SekParams sp, bool add_noise, cudaStream_t s);

// Batched tile GEMV: y_q (+)= alpha * op(A_q) x_q, one (A, x, y) triple per job; every
// job's y is written by one CTA group, so outputs must be distinct within a launch.
struct GemvJob {
  const double* a;
  const double* x;
  double* y;
};
cudaError_t launch_gemv_jobs(const GemvJob* jobs, int64_t njobs, int bi, int trans, double alpha,
                             int accumulate, cudaStream_t s);
// out[e] = base[e] - sum_{p = 0..nparts-1} parts[p * len + e]   (fixed order)
cudaError_t launch_combine(const double* base, const double* parts, int64_t nparts, int64_t len,
                           double* out, cudaStream_t s);

// B = K*^T for one chunk of test points: rows = padded training positions
// (np rows), cols = mcp (mc real).  Fused mean partials over 64-row blocks:
// mpart[rb][c] = sum_{rows in rb} B[r][c] * alpha[r].
cudaError_t launch_cross(double* B, int64_t ldb, double* mpart, const double* alpha,
                         const double* zp, int64_t np_, const double* zt, int64_t mc,
                         int64_t mcp, int d, PadMap pm, SekParams sp, cudaStream_t s);

// Dense prior K** (mp x mp, row-major) of the test chunk, noise-free.
cudaError_t launch_prior(double* S, int64_t mp, const double* zt, int64_t m, int d, SekParams sp,
                         cudaStream_t s);
// Cross prior K**(za, zb): S (mpa x mpb, ld lds; multiples of kSekBlock), zero
// outside the ma x mb real block.
cudaError_t launch_prior2(double* S, int64_t lds, int64_t mpa, int64_t mpb, const double* za,
                          int64_t ma, const double* zb, int64_t mb, int d, SekParams sp,
                          cudaStream_t s);

// Gradient trace pass over lower tiles of K^-1, one partial per kSekBlock^2 block:
// part_l = w * sum (Kinv - alpha alpha^T) e d2,  part_v = w * sum (Kinv - ..) e,
// part_t (optional) = sum of the real diagonal entries of Kinv (w = 2 off the diagonal).
// Tile t = tile_ij[t] is read from packed tiles (ld == 0: kinv + t * bi^2, column-major
// tile order) or from a dense row-major panel (ld > 0) whose row 0 is global
// position row0 * bi; tile t's columns start at panel column slot[t] * bi (slot
// non-null) or at (j - col0) * bi.
struct TraceTiles {
  int64_t ld;
  int row0, col0;
  const int* slot;
};
cudaError_t launch_trace(const double* kinv, const int2* tile_ij, int64_t ntiles, TraceTiles tt,
                         const double* zp, const double* alpha, int d, int bi, PadMap pm,
                         SekParams sp, double* part_l, double* part_v, double* part_t,
                         cudaStream_t s);
// part[blk] = sum of squares of the real entries of lower tiles (column-major order).
cudaError_t launch_tiles_sumsq(const double* x, const int2* tile_ij_cm, int64_t ntiles, int bi,
                               PadMap pm, double* part, cudaStream_t s);

// ---- solves and reductions (solve.cu) -------------------------------------
cudaError_t launch_fwd_diag(const double* dinv, const double* yhat, double* beta, int bi,
                            cudaStream_t s);
cudaError_t launch_fwd_update(const double* ltiles, int T, int i, int bi, const double* beta_i,
                              double* yhat, cudaStream_t s);
cudaError_t launch_bwd_diag(const double* dinv, const double* bhat, double* alpha, int bi,
                            cudaStream_t s);
cudaError_t launch_bwd_update(const double* ltiles, int i, int bi, const double* alpha_i,
                              double* bhat, cudaStream_t s);
// Both vector solves in one cooperative launch (solve_flow.cu): beta = L^-1 y,
// alpha = L^-T beta with per-block-row counters (flags: 4T ints, zeroed here;
// xr: n_p doubles of exchange).  R = slice height from solve_flow_slice_rows
// (0: the grid cannot be co-resident).  *launched = false: nothing was
// launched and the caller must run the multi-launch solves.
int solve_flow_slice_rows(int64_t np_, int bi);
size_t solve_flow_scratch_bytes(int T, int bi);  // per-model scratch of launch_solve_flow
cudaError_t launch_solve_flow(const double* L, const double* dinv, const double* y, double* beta,
                              double* alpha, double* xr, void* scratch, int T, int bi, int R,
                              cudaStream_t s, bool* launched);
// out[0] = sum_k logdiag[k] (sequential k), out[1] = sum x^2 (fixed order)
cudaError_t launch_loss_terms(const double* logdiag, int T, const double* x, int64_t n,
                              double* out, cudaStream_t s);
// out[i] = fixed-order sum of part[0..n)  (one output per call, slot i)
cudaError_t launch_reduce(const double* part, int64_t n, double* out, cudaStream_t s);
// mean[c] = sum_rb mpart[rb][c];  var[c] = nu - sum_rb sq[rb][c]  (either may be null)
cudaError_t launch_pred_finalize(const double* mpart, int64_t nmrb, const double* sq,
                                 int64_t nsrb, int64_t ld, int64_t mc, double nu, double* mean,
                                 double* var, cudaStream_t s);
// S[c][r] = S[r][c] for c > r (mirror the lower triangle)
cudaError_t launch_symmetrize(double* S, int64_t mp, int64_t m, cudaStream_t s);
// scatter padded vector -> dense, gather dense -> padded
cudaError_t launch_pad_vector(const double* src, double* dst, int64_t np_, PadMap pm, cudaStream_t s);
cudaError_t launch_pad_rows(const double* src, double* dst, int64_t np_, int d, PadMap pm,
                            cudaStream_t s);
// dense lower factor export, rows [row0, row0 + rows) of the n x n factor
// (user indices): out[r - row0][c] from packed tiles
cudaError_t launch_export_lower(const double* tiles, int bi, int64_t n, int64_t row0, int64_t rows,
                                PadMap pm, double* out, cudaStream_t s);
// G[c * ld + c] = 1 for c < count (identity right-hand side of a column panel)
cudaError_t launch_set_diag(double* G, int64_t ld, int64_t count, cudaStream_t s);
// copy the solved panel (scratch tiles q = 0..T-k-2) back to tiles (k+1+q, k)
cudaError_t launch_copy_panel(double* ltiles, const double* scratch, int T, int k, int bi,
                              cudaStream_t s);

}  // namespace gpb
