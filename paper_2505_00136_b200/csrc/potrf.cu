// Diagonal-tile factorisation: POTRF + TRTRI of one bi x bi tile by one
// thread-block cluster (GPB_POTRF_CLUSTER CTAs, default 8, on as many SMs).
//
// Replaces taskgp tile_potrf (tiles.py:132-137 -> np.linalg.cholesky,
// tiles.py:29-33) and provides the inverted diagonal tile that turns every
// triangular solve of the hot path (panel TRSM tiles.py:140-146, vector
// solves tiles.py:170-180, panel solves tiles.py:182-185) into DMMA products.
//
// Blocked Cholesky with 32-column panels.  Per panel p, two phases:
//   B (CTA 0 warp 0) factor the 32x32 diagonal block -- the serial pivot
//                   chain in registers, each new column broadcast through
//                   shared memory;
//     (CTA 0 warp 1) invert it by a column sweep one pivot behind the chain;
//     (other warps) panel p-1's rank-32 update of every 32-block below the
//                   diagonal block (right-looking) and the TRTRI of Dinv
//                   (finalise block row p-1, accumulate term p-2);
//   C (all warps)   solve the rows below the diagonal block (x Li^T); the
//                   warp of row block p+1 also applies panel p to the next
//                   diagonal block, so B(p+1) can start at once;
// so the DMMA work of the update and of TRTRI runs while the pivot chain
// advances.  The warp jobs of every phase are dealt over all warps of the
// cluster and the phases are separated by cluster barriers (release/acquire
// at cluster scope orders the global-memory tile between the SMs), so the
// lookahead DMMA work is spread over CL SMs while CTA 0's warp 0 runs the
// pivot chain.  Epilogue: Sigma log L_jj over real (non-padding) pivots and a
// LAPACK-style info word holding the first failing original pivot index.
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace gpb {

namespace {

constexpr int PT = 256;  // threads
constexpr int NW = PT / 32;
constexpr int NB = 32;   // panel width
constexpr int SLD = NB + 1;

// acc[i][j][e] <-> C[8i+g][8j+2t+e] of a 32x32 warp tile.
GPB_DEVINL void zero_acc(double (&acc)[4][4][2]) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
}

// Operands come straight from L2 (the tile is produced inside this kernel),
// so the warp GEMMs fetch the fragments of a 16-deep k chunk (32 loads per
// lane) one chunk ahead of the DMMAs that consume them.
GPB_DEVINL void load_chunk(double (&a)[4][4], double (&b)[4][4], const double* A, int64_t lda,
                           const double* B, int64_t ldb, int k, int g, int t) {
#pragma unroll
  for (int s = 0; s < 4; ++s)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      a[s][i] = A[(8 * i + g) * lda + k + 4 * s + t];
      b[s][i] = B[(8 * i + g) * ldb + k + 4 * s + t];
    }
}

GPB_DEVINL void load_chunk_nn(double (&a)[4][4], double (&b)[4][4], const double* A, int64_t lda,
                              const double* B, int64_t ldb, int k, int g, int t) {
#pragma unroll
  for (int s = 0; s < 4; ++s)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      a[s][i] = A[(8 * i + g) * lda + k + 4 * s + t];
      b[s][i] = B[(k + 4 * s + t) * ldb + 8 * i + g];
    }
}

GPB_DEVINL void mma_chunk(double (&acc)[4][4][2], const double (&a)[4][4], const double (&b)[4][4]) {
#pragma unroll
  for (int s = 0; s < 4; ++s)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[s][i], b[s][j]);
}

// acc += A(32 x K) * B(32 x K)^T, both k-contiguous, K a multiple of 32.
GPB_DEVINL void warp_nt(double (&acc)[4][4][2], const double* A, int64_t lda, const double* B,
                        int64_t ldb, int K, int g, int t) {
  double a0[4][4], b0[4][4], a1[4][4], b1[4][4];
  if (K <= 0) return;
  load_chunk(a0, b0, A, lda, B, ldb, 0, g, t);
  for (int k = 0; k < K; k += 32) {
    load_chunk(a1, b1, A, lda, B, ldb, k + 16, g, t);
    mma_chunk(acc, a0, b0);
    if (k + 32 < K) load_chunk(a0, b0, A, lda, B, ldb, k + 32, g, t);
    mma_chunk(acc, a1, b1);
  }
}

// acc += A(32 x K) * B(K x 32), A k-contiguous, B row-major (n contiguous).
GPB_DEVINL void warp_nn(double (&acc)[4][4][2], const double* A, int64_t lda, const double* B,
                        int64_t ldb, int K, int g, int t) {
  double a0[4][4], b0[4][4], a1[4][4], b1[4][4];
  if (K <= 0) return;
  load_chunk_nn(a0, b0, A, lda, B, ldb, 0, g, t);
  for (int k = 0; k < K; k += 32) {
    load_chunk_nn(a1, b1, A, lda, B, ldb, k + 16, g, t);
    mma_chunk(acc, a0, b0);
    if (k + 32 < K) load_chunk_nn(a0, b0, A, lda, B, ldb, k + 32, g, t);
    mma_chunk(acc, a1, b1);
  }
}

// C[32x32 at c, ldc] -= acc  (or = acc when assign)
GPB_DEVINL void store_acc(double* c, int64_t ldc, const double (&acc)[4][4][2], int g, int t,
                          bool assign, double scale) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double* p = c + static_cast<int64_t>(8 * i + g) * ldc + 8 * j + 2 * t;
      if (assign) {
        p[0] = scale * acc[i][j][0];
        p[1] = scale * acc[i][j][1];
      } else {
        p[0] -= acc[i][j][0];
        p[1] -= acc[i][j][1];
      }
    }
}


// Right-looking TRTRI of the tile, X = L^-1 by 32-blocks:
//   X_IJ = -X_II sum_{K=J}^{I-1} L_IK X_KJ.
// Block (I, J) of D accumulates -sum L_IK X_KJ one K per panel (term K in
// phase C(K+1) for row K+1 and in B(K+2) for the rows below, once row K of X
// is final), and row I is finalised in phase B(I+1) as X_II * D_IJ: every
// job has K = 32, so no single warp carries a long dependency chain.
GPB_DEVINL void trtri_acc(const double* T, double* D, int bi, int I, int J, int K, int g, int t) {
  double acc[4][4][2];
  zero_acc(acc);
  warp_nn(acc, T + static_cast<int64_t>(I) * NB * bi + K * NB, bi,
          D + static_cast<int64_t>(K) * NB * bi + J * NB, bi, NB, g, t);
  // first term assigns (D_IJ = -acc), later terms subtract
  store_acc(D + static_cast<int64_t>(I) * NB * bi + J * NB, bi, acc, g, t, K == J, -1.0);
}

GPB_DEVINL void trtri_fin(double* D, int bi, int I, int J, int g, int t) {
  double acc[4][4][2];
  zero_acc(acc);
  warp_nn(acc, D + static_cast<int64_t>(I) * NB * bi + I * NB, bi,
          D + static_cast<int64_t>(I) * NB * bi + J * NB, bi, NB, g, t);
  __syncwarp();  // every lane has read D_IJ before it is overwritten
  store_acc(D + static_cast<int64_t>(I) * NB * bi + J * NB, bi, acc, g, t, true, 1.0);
  __syncwarp();
}

// 8-row fragments of the K = 32 block jobs: a 32x32 job is split into four
// independent row fragments (acc[j][e] <-> C[g][8j+2t+e]) dealt to warps on
// different SMSPs, since one warp's DMMAs are issue-bound on its SMSP.  All
// 40 operand loads of a lane are issued before the DMMAs.
GPB_DEVINL void frag_mma(double (&acc)[4][2], const double (&a)[8], const double (&b)[8][4]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll
  for (int s = 0; s < 8; ++s)
#pragma unroll
    for (int j = 0; j < 4; ++j) dmma884(acc[j][0], acc[j][1], a[s], b[s][j]);
}

// acc = A(8 x 32) * B(32 x 32)^T, both k-contiguous
GPB_DEVINL void frag_nt(double (&acc)[4][2], const double* A, int64_t lda, const double* B, int64_t ldb,
                        int g, int t) {
  double a[8], b[8][4];
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    a[s] = A[g * lda + 4 * s + t];
#pragma unroll
    for (int j = 0; j < 4; ++j) b[s][j] = B[(8 * j + g) * ldb + 4 * s + t];
  }
  frag_mma(acc, a, b);
}

// acc = A(8 x 32) * B(32 x 32), A k-contiguous, B row-major (n contiguous)
GPB_DEVINL void frag_nn(double (&acc)[4][2], const double* A, int64_t lda, const double* B, int64_t ldb,
                        int g, int t) {
  double a[8], b[8][4];
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    a[s] = A[g * lda + 4 * s + t];
#pragma unroll
    for (int j = 0; j < 4; ++j) b[s][j] = B[(4 * s + t) * ldb + 8 * j + g];
  }
  frag_mma(acc, a, b);
}

// C[8x32 at c, ldc] -= acc  (or = scale * acc when assign)
GPB_DEVINL void store_frag(double* c, int64_t ldc, const double (&acc)[4][2], int g, int t, bool assign,
                           double scale) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    double* q = c + static_cast<int64_t>(g) * ldc + 8 * j + 2 * t;
    if (assign) {
      q[0] = scale * acc[j][0];
      q[1] = scale * acc[j][1];
    } else {
      q[0] -= acc[j][0];
      q[1] -= acc[j][1];
    }
  }
}

// row fragment f of trtri_acc: D_IJ (-)= T_IK D_KJ (the first term, K == J, assigns)
GPB_DEVINL void trtri_acc_frag(const double* T, double* D, int bi, int I, int J, int K, int f, int g,
                               int t) {
  double acc[4][2];
  const int64_t r = static_cast<int64_t>(I) * NB + 8 * f;
  frag_nn(acc, T + r * bi + K * NB, bi, D + static_cast<int64_t>(K) * NB * bi + J * NB, bi, g, t);
  store_frag(D + r * bi + J * NB, bi, acc, g, t, K == J, -1.0);
}

// the cluster's warps except CTA 0's warps 0..3, numbered so that
// consecutive indices sit on different CTAs first, then on different SMSPs
GPB_DEVINL int c_worker(int cta, int ncta, int lw) {
  return cta + ncta * lw - min(4, lw + (cta > 0 ? 1 : 0));
}

// all threads of the cluster (a plain launch is a cluster of one CTA)
GPB_DEVINL void cluster_barrier(bool clustered) {
  if (clustered)
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::
                     : "memory");
  else
    __syncthreads();
}

}  // namespace

__global__ void __launch_bounds__(PT, 1) potrf_tile_kernel(PotrfArgs a) {
  extern __shared__ double sm[];
  double* Ld = sm;                 // [64][33] factor block (rows 32..63: padding)
  double* rdg = Ld + 2 * NB * SLD;  // [32] 1 / l_jj of the current panel
  __shared__ volatile int prog_s;  // pivots of the chain published so far
  volatile int* prog = &prog_s;
  // every CTA reads info before the first cluster barrier; only CTA 0
  // writes it, and only after that barrier
  if (*a.info >= 0) return;  // an earlier tile already failed
  const int bi = a.bi;
  double* T = a.tile;
  double* D = a.dinv;
  const int P = bi / NB;
  const int tid = threadIdx.x, lane = tid & 31;
  const int cta = blockIdx.x, ncta = gridDim.x;
  const bool clustered = ncta > 1;
  const bool lead = cta == 0;
  const int lw = tid >> 5;                 // warp index within the CTA
  const int warp = cta * NW + lw;          // warp index within the cluster
  const int GW = ncta * NW;                // warps in the cluster
  const int g = lane >> 2, t = lane & 3;
  const bool factor = !a.trtri_only;
  double logsum = 0.0;  // meaningful in lane 0 of warp 0
  if (tid == 0) *prog = 0;
  cluster_barrier(clustered);
  long long t_last = clock64(), t_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  // per-phase cycles of thread 0 of CTA 0 (slots 0-7) and of CTA 1 (8-15)
#define PROF_MARK(i)                                   \
  if (a.prof && tid == 0 && cta < 2) {                 \
    const long long now_ = clock64();                  \
    t_acc[i] += now_ - t_last;                         \
    t_last = now_;                                     \
  }

  long long t_phase = 0;  // profiling: start of phase B of this panel
  for (int p = 0; p < P; ++p) {
    const int c0 = p * NB;
    PROF_MARK(0)
    if (a.prof && lane == 0) t_phase = clock64();
    if (!(lead && lw < 2)) {
      // B, job warps (CTAs 1.. when clustered, else warps 2..7), dealt
      // round-robin: panel p-1's rank-32 contribution to every 32-block
      // (rb, cb), p <= cb <= rb, below the diagonal block (right-looking;
      // the diagonal block (p, p) got it in C(p-1)), the finalisation of
      // block row p-1 of the inverse, and the TRTRI term K = p-2 of rows I >= p
      const int m = P - p;  // block rows p .. P-1; (p, p) excluded
      const int pre = (factor && p > 0) ? m * (m + 1) / 2 - 1 : 0;
      const int inv = (p >= 2) ? p - 1 : 0;  // blocks J = 0..p-2 of row I = p-1
      const int accn = (p >= 2) ? (P - p) * (p - 1) : 0;  // term K = p-2 of rows I >= p
      // clustered: CTA 0 keeps only the pivot chain so its SMSPs are not
      // shared with DMMA warps; the other CTAs' warps take the jobs
      // consecutive jobs go to different CTAs first, then to different warps
      // (SMSPs) of a CTA: a K = 32 job is DMMA-issue bound on its SMSP
      const int w0 = clustered ? (lead ? -1 : (cta - 1) + (ncta - 1) * lw) : warp - 2;
      const int nwk = clustered ? GW - NW : NW - 2;
      // whole 32x32 jobs here (row fragments would repeat the B operand's
      // loads four times: this phase is load-bound, measured slower)
      for (int q = (w0 >= 0 ? w0 : pre + inv + accn); q < pre + inv + accn; q += nwk) {
        if (q < pre) {
          const int qq = q + 1;  // skip (p, p)
          int rr = static_cast<int>((sqrtf(8.0f * qq + 1.0f) - 1.0f) * 0.5f);
          while (rr * (rr + 1) / 2 > qq) --rr;
          while ((rr + 1) * (rr + 2) / 2 <= qq) ++rr;
          const int rb = p + rr, cb = p + (qq - rr * (rr + 1) / 2);
          double acc[4][4][2];
          zero_acc(acc);
          warp_nt(acc, T + static_cast<int64_t>(rb) * NB * bi + c0 - NB, bi,
                  T + static_cast<int64_t>(cb) * NB * bi + c0 - NB, bi, NB, g, t);
          store_acc(T + static_cast<int64_t>(rb) * NB * bi + cb * NB, bi, acc, g, t, false, 1.0);
        } else if (q < pre + inv) {
          trtri_fin(D, bi, p - 1, q - pre, g, t);
        } else {
          const int w = q - pre - inv;
          trtri_acc(T, D, bi, p + w / (p - 1), w % (p - 1), p - 2, g, t);
        }
      }
      PROF_MARK(5)
      if (a.prof && lane == 0 && lw == 0) atomicAdd(reinterpret_cast<unsigned long long*>(a.prof + 16 + cta),
                                                    static_cast<unsigned long long>(clock64() - t_phase));
    } else if (lead && lw == 0) {
      // B, chain: lane i keeps row i of the diagonal block in registers,
      // shifted so that register 0 always holds the current pivot column
      // (short code: the pivot loop is not unrolled; LAPACK dpotf2 order).
      // After pivot j, row j of L is complete: publish it to the inverse warp.
      const int base = p * NB;
      double r[NB];
#pragma unroll
      for (int c = 0; c < NB; ++c) r[c] = T[static_cast<int64_t>(c0 + lane) * bi + c0 + c];
      int fail = -1;
      double my_l = 1.0;
      if (factor) {
        // Blocked by sub-panels of SP = 8 columns: a pivot updates only the
        // columns of its own sub-panel; at the end of a sub-panel one rank-8
        // update (the same FMAs in the same order, so results are unchanged)
        // brings the later columns up to date, and the registers shift by 8.
        // Entries of lanes above the current row are updated too (they lie in
        // the upper triangle, are never read again, and lcol = 0 leaves them
        // unchanged for lanes < j), which drops the per-entry predicate.
        // Software-pipelined: the next pivot column is updated first, its
        // pivot fetched and its rsqrt started, and only then the other
        // columns, so the rsqrt latency hides behind those FMAs; progress is
        // published every two pivots.
        constexpr int SP = 8;
        double piv = __shfl_sync(0xffffffffu, r[0], 0);
        double rinv = rsqrt(piv);
#pragma unroll 1
        for (int j0 = 0; j0 < NB; j0 += SP) {
          double lc[SP];
#pragma unroll
          for (int t = 0; t < SP; ++t) {  // register t holds column j = j0 + t
            const int j = j0 + t;
            if (fail < 0 && !(piv > 0.0)) fail = j;
            const double lcol = (lane == j) ? piv * rinv : (lane > j ? r[t] * rinv : 0.0);
            lc[t] = lcol;
            if (lane == j) {
              my_l = lcol;
              rdg[j] = rinv;
            }
            Ld[lane * SLD + j] = lcol;
            __syncwarp();
            if ((t & 1) && lane == 0) {
              __threadfence_block();
              *prog = base + j + 1;
            }
            if (t + 1 < SP) {
              // lrow[c * SLD] = l_(j0 + c), j from shared memory (one address
              // per load)
              const double* lrow = Ld + j0 * SLD + j;
              r[t + 1] = fma(-lcol, lrow[(t + 1) * SLD], r[t + 1]);
              piv = __shfl_sync(0xffffffffu, r[t + 1], j + 1);
              rinv = rsqrt(piv);
#pragma unroll
              for (int c = t + 2; c < SP; ++c) r[c] = fma(-lcol, lrow[c * SLD], r[c]);
            }
          }
          if (j0 + SP < NB) {
            // rank-SP update of the later columns; rows past the panel read
            // the padding rows of Ld and only feed registers past the panel
            const double* lb = Ld + j0 * SLD + j0;  // lb[c * SLD + t] = l_(j0 + c), (j0 + t)
#pragma unroll
            for (int t = 0; t < SP; ++t) r[SP] = fma(-lc[t], lb[SP * SLD + t], r[SP]);
            piv = __shfl_sync(0xffffffffu, r[SP], j0 + SP);
            rinv = rsqrt(piv);
#pragma unroll
            for (int c = SP + 1; c < NB; ++c)
#pragma unroll
              for (int t = 0; t < SP; ++t) r[c] = fma(-lc[t], lb[c * SLD + t], r[c]);
#pragma unroll
            for (int c = 0; c < NB - SP; ++c) r[c] = r[c + SP];
          }
        }
        const int pos = a.tile_off + c0 + lane;  // padded global position
        const bool real = (pos % a.bp_user < a.b_user) && (fail < 0 || lane < fail);
        const double lsum = warp_sum(real ? log(my_l) : 0.0);
        if (lane == 0) logsum += lsum;
        PROF_MARK(5)
        __syncwarp();
        for (int c = lane + 1; c < NB; ++c) Ld[lane * SLD + c] = 0.0;  // strictly upper
        __syncwarp();
        if (fail >= 0) {
          if (lane == 0) {
            const int fp = a.tile_off + c0 + fail;
            *reinterpret_cast<volatile int*>(a.info) = (fp / a.bp_user) * a.b_user + fp % a.bp_user;
          }
        } else {
#pragma unroll 4
          for (int c = 0; c < NB; ++c) T[static_cast<int64_t>(c0 + lane) * bi + c0 + c] = Ld[lane * SLD + c];
        }
      } else {  // trtri-only: the tile already holds L
#pragma unroll
        for (int c = 0; c < NB; ++c) Ld[lane * SLD + c] = (c <= lane) ? r[c] : 0.0;
        __syncwarp();
        rdg[lane] = 1.0 / Ld[lane * SLD + lane];
        __syncwarp();
        if (lane == 0) {
          __threadfence_block();
          *prog = base + NB;
        }
      }
      PROF_MARK(6)
    } else if (lead && lw == 1) {
      // B, inverse of the diagonal block by a column sweep that trails the
      // chain by one pivot: lane k holds column k of Li = L^-1 in registers
      // (forward substitution of e_k), and step j needs only column j of L,
      // published by the chain right after pivot j:
      //   x_j *= 1 / l_jj;   x_i -= l_ij x_j  (i > j, independent FMAs)
      const int base = p * NB;
      double x[NB];
#pragma unroll
      for (int i = 0; i < NB; ++i) x[i] = (i == lane) ? 1.0 : 0.0;
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        while (*prog < base + j + 1) {
        }
        __threadfence_block();
        x[j] *= rdg[j];
#pragma unroll
        for (int i = j + 1; i < NB; ++i) x[i] = fma(-Ld[i * SLD + j], x[j], x[i]);
      }
#pragma unroll
      for (int i = 0; i < NB; ++i) D[static_cast<int64_t>(c0 + i) * bi + c0 + lane] = x[i];
      if (a.prof && lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(a.prof + 32),
                                         static_cast<unsigned long long>(clock64() - t_phase));
    }
    cluster_barrier(clustered);
    PROF_MARK(1)
    if (*reinterpret_cast<volatile int*>(a.info) >= 0) return;  // set by CTA 0 above
    // C: below-diagonal panel rows, L[r][c0:c0+32] = T[r][c0:c0+32] * Li^T
    // (Li read back from the diagonal block of D, written by CTA 0); the warp
    // of row block p+1 then applies panel p to the next diagonal block
    // (p+1, p+1), which is all the chain of B(p+1) needs.  Also the TRTRI
    // term K = p-1 of row I = p, which B(p+1) finalises.
    {
      const int nt = factor ? P - p - 1 : 0;
      const int na = p >= 1 ? p : 0;  // J = 0..p-1
      // The critical path, block row p+1 (which B(p+1) needs first), runs on
      // CTA 0's warps 0..3, one 8-row fragment each: X = T * Li^T, then, after
      // a named barrier of the four warps, (p+1, p+1) -= X X^T.  Every other
      // row block and TRTRI term is split into row fragments dealt to the
      // remaining warps (c_worker).
      const double* Li = D + static_cast<int64_t>(c0) * bi + c0;
      if (lead && lw < 4) {
        if (nt > 0) {
          double* blk = T + static_cast<int64_t>(p + 1) * NB * bi + c0;
          double* mine = blk + static_cast<int64_t>(8 * lw) * bi;
          double acc[4][2];
          frag_nt(acc, mine, bi, Li, bi, g, t);
          __syncwarp();
          store_frag(mine, bi, acc, g, t, true, 1.0);
          __threadfence_block();
          asm volatile("bar.sync 1, 128;\n" ::: "memory");
          frag_nt(acc, mine, bi, blk, bi, g, t);
          store_frag(mine + NB, bi, acc, g, t, false, 1.0);
        }
      } else {
        const int nw = GW - 4;
        const int nrow = nt > 0 ? 4 * (nt - 1) : 0;
        const int nsub = nrow + 4 * na;
        for (int q = c_worker(cta, ncta, lw); q < nsub; q += nw) {
          const int f = q % 4;
          if (q < nrow) {
            double* mine = T + (static_cast<int64_t>(p + 2 + q / 4) * NB + 8 * f) * bi + c0;
            double acc[4][2];
            frag_nt(acc, mine, bi, Li, bi, g, t);
            __syncwarp();
            store_frag(mine, bi, acc, g, t, true, 1.0);
          } else {
            trtri_acc_frag(T, D, bi, p, (q - nrow) / 4, p - 1, f, g, t);
          }
        }
      }
    }
    PROF_MARK(7)
    cluster_barrier(clustered);
    PROF_MARK(2)
  }
  // last block row of the inverse (its last term came in C(P-1)): X_II * D_IJ
  for (int J = warp; J < P - 1; J += GW) trtri_fin(D, bi, P - 1, J, g, t);
  PROF_MARK(3)
  // zero strictly-upper 32-blocks of L and Dinv (lower-triangular results)
  for (int r = warp; r < bi; r += GW) {
    const int c_begin = (r / NB + 1) * NB;
    for (int c = c_begin + 2 * lane; c < bi; c += 64) {
      const int64_t idx = static_cast<int64_t>(r) * bi + c;
      if (factor) *reinterpret_cast<double2*>(T + idx) = make_double2(0.0, 0.0);
      *reinterpret_cast<double2*>(D + idx) = make_double2(0.0, 0.0);
    }
  }
  PROF_MARK(4)
  if (a.prof && tid == 0 && cta < 2)
    for (int i = 0; i < 8; ++i) a.prof[8 * cta + i] += t_acc[i];
  if (tid == 0 && lead && a.logdiag) a.logdiag[a.tile_index] = logsum;
#undef PROF_MARK
}

size_t potrf_smem_bytes() { return sizeof(double) * (2 * NB * SLD + NB); }

static int g_cluster = -1;

// CTAs per diagonal tile: GPB_POTRF_CLUSTER (1 = single CTA, 2, 4, 8 or 16),
// else 16 where POTRF is on the critical path -- factorisations of fewer
// than 48 diagonal tiles (config 1 factor 8.8 -> 8.2 ms) and the last 8 tiles
// of larger ones -- and 8 otherwise (hidden behind the trailing update,
// where 16 latency-bound SMs would cost GEMM time)
static int potrf_cluster(int tiles, int remaining) {
  if (g_cluster < 0) {
    const char* e = getenv("GPB_POTRF_CLUSTER");
    const int c = e ? atoi(e) : 0;
    g_cluster = (c == 1 || c == 2 || c == 4 || c == 8 || c == 16) ? c : 0;
  }
  if (g_cluster > 0) return g_cluster;
  return ((tiles > 0 && tiles < 48) || (remaining > 0 && remaining <= 8)) ? 16 : 8;
}

cudaError_t launch_potrf(const PotrfArgs& a, cudaStream_t s) {
  const int cl = potrf_cluster(a.tiles, a.remaining);
  if (cl == 1) {
    potrf_tile_kernel<<<1, PT, potrf_smem_bytes(), s>>>(a);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(cl);
  cfg.blockDim = dim3(PT);
  cfg.dynamicSmemBytes = potrf_smem_bytes();
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, potrf_tile_kernel, a);
}

cudaError_t potrf_init_attributes() {
  cudaError_t e = cudaFuncSetAttribute(potrf_tile_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(potrf_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(potrf_smem_bytes()));
}

}  // namespace gpb
