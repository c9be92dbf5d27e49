// Diagonal-tile factorisation: POTRF + TRTRI of one bi x bi tile by one
// thread-block cluster (GPB_POTRF_CLUSTER CTAs, default 8, on as many SMs).
//
// Replaces taskgp tile_potrf (tiles.py:132-137 -> np.linalg.cholesky,
// tiles.py:29-33) and provides the inverted diagonal tile that turns every
// triangular solve of the hot path (panel TRSM tiles.py:140-146, vector
// solves tiles.py:170-180, panel solves tiles.py:182-185) into DMMA products.
//
// Blocked Cholesky with 32-column panels, two phases per panel separated by
// cluster barriers (release/acquire at cluster scope orders the tile in
// global memory between the SMs):
//   B(p)  CTA 0 warp 0: pivot chain of the 32x32 diagonal block in registers;
//         CTA 0 warp 1: its inverse by a column sweep one pivot behind;
//         other CTAs: panel p-1's rank-32 update of every trailing 32-block
//         (right-looking) and the TRTRI of Dinv; CTA 0 warps 2..5: panel
//         p-1 applied to blocks (p+1, p) and (p+1, p+1), kept in shared
//         memory;
//   C(p)  CTA 0 warps 2..5: block row p+1 solved (x Li^T) and applied to
//         (p+1, p+1) in shared memory -- all the next chain needs; other
//         CTAs: the other rows and TRTRI terms, as 8-row fragments.
// Lookahead: once the critical warps are done (named barrier), the chain and
// inverse warps arrive at the C(p) barrier and run panel p+1 before waiting
// on it, so the rest of C(p), the next B jobs and both barriers overlap the
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

}  // namespace

__global__ void __launch_bounds__(PT, 1) potrf_tile_kernel(PotrfArgs a) {
  extern __shared__ double sm[];
  double* Ld = sm;                 // [64][33] factor block (rows 32..63: padding)
  double* rdg = Ld + 2 * NB * SLD;  // [32] 1 / l_jj of the current panel
  // CTA 0's critical path through shared memory ([32][33] each): Ls = Li of
  // the current panel (from the inverse warp), Ts = block (p+1, p) and
  // Dd = block (p+1, p+1) as updated by the critical warps, Xs = L(p+1, p)
  double* Ls = rdg + NB;
  double* Ts = Ls + NB * SLD;
  double* Dd = Ts + NB * SLD;
  double* Xs = Dd + NB * SLD;
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
  const int cta = blockIdx.x, ncta = gridDim.x;  // a cluster of >= 2 CTAs
  const bool lead = cta == 0;
  const int lw = tid >> 5;                 // warp index within the CTA
  const int warp = cta * NW + lw;          // warp index within the cluster
  const int GW = ncta * NW;                // warps in the cluster
  const int g = lane >> 2, t = lane & 3;
  const bool factor = !a.trtri_only;
  // CTA 0: warp 0 runs the pivot chain, warp 1 the diagonal-block inverse,
  // warps 2..5 (one per SMSP; the chain and inverse warps are idle while they
  // work) the critical block row; the other CTAs' warps take every other job
  const bool chain_w = lead && lw == 0, inv_w = lead && lw == 1;
  const int crit = (lead && lw >= 2 && lw < 6) ? lw - 2 : -1;
  const int wj = lead ? -1 : (cta - 1) + (ncta - 1) * lw;  // job-warp index, CTAs first
  const int nwj = GW - NW;
  double logsum = 0.0;  // meaningful in lane 0 of warp 0
  if (tid == 0) *prog = 0;
  long long t_last = clock64(), t_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  // per-phase cycles of thread 0 of CTA 0 (slots 0-7) and of CTA 1 (8-15)
#define PROF_MARK(i)                                   \
  if (a.prof && tid == 0 && cta < 2) {                 \
    const long long now_ = clock64();                  \
    t_acc[i] += now_ - t_last;                         \
    t_last = now_;                                     \
  }
  auto arrive = [] { asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory"); };
  auto wait = [] { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory"); };

  // B-phase pivot chain of diagonal block p (CTA 0 warp 0): lane i keeps row
  // i of the block in registers, shifted so that register 0 always holds the
  // current pivot column (LAPACK dpotf2 order); each new column of L is
  // published to the inverse warp through Ld and the progress counter.
  auto chain = [&](int p) {
    const int c0 = p * NB;
      const int base = p * NB;
      double r[NB];
#pragma unroll
      for (int c = 0; c < NB; ++c)  // panel 0 from the tile, later ones as the critical warps left them
        r[c] = (p == 0 || !factor) ? T[static_cast<int64_t>(c0 + lane) * bi + c0 + c] : Dd[lane * SLD + c];
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
        // Pivots go in pairs (j, j+1): from A_jj, A_j+1,j and A_j+1,j+1 (three
        // shuffles) l_jj, l_j+1,j and l_j+1,j+1 follow in registers, every lane
        // forms both of its column entries, and one shared-memory exchange
        // serves both pivots -- the same operations in the same order as
        // pivoting one column at a time, so the factor is unchanged.
        double av = __shfl_sync(0xffffffffu, r[0], 0);
        double bv = __shfl_sync(0xffffffffu, r[0], 1);
        double cv = __shfl_sync(0xffffffffu, r[1], 1);
#pragma unroll 1
        for (int j0 = 0; j0 < NB; j0 += SP) {
          double lc[SP];
#pragma unroll
          for (int t = 0; t < SP; t += 2) {  // registers t, t+1 hold columns j, j+1
            const int j = j0 + t;
            if (fail < 0 && !(av > 0.0)) fail = j;
            const double rinv0 = rsqrt(av);
            const double l10 = bv * rinv0;
            const double sv = fma(-l10, l10, cv);
            if (fail < 0 && !(sv > 0.0)) fail = j + 1;
            const double rinv1 = rsqrt(sv);
            const double lcol0 = (lane == j) ? av * rinv0 : (lane > j ? r[t] * rinv0 : 0.0);
            const double u = fma(-lcol0, l10, r[t + 1]);
            const double lcol1 = (lane == j + 1) ? sv * rinv1 : (lane > j + 1 ? u * rinv1 : 0.0);
            lc[t] = lcol0;
            lc[t + 1] = lcol1;
            if (lane == j) {
              my_l = lcol0;
              rdg[j] = rinv0;
            }
            if (lane == j + 1) {
              my_l = lcol1;
              rdg[j + 1] = rinv1;
            }
            Ld[lane * SLD + j] = lcol0;
            Ld[lane * SLD + j + 1] = lcol1;
            __syncwarp();
            if (t == SP - 2 && lane == 0) {  // progress once per sub-panel (a fence costs ~90 cycles)
              asm volatile("fence.acq_rel.cta;\n" ::: "memory");
              *prog = base + j + 2;
            }
            if (t + 2 < SP) {
              // l0[c * SLD] = l_(j0 + c), j and l1[c * SLD] = l_(j0 + c), j+1 from
              // shared memory (one address per load); the next pair's columns first
              const double* l0 = Ld + j0 * SLD + j;
              const double* l1 = l0 + 1;
#pragma unroll
              for (int c = t + 2; c < t + 4; ++c) {
                r[c] = fma(-lcol0, l0[c * SLD], r[c]);
                r[c] = fma(-lcol1, l1[c * SLD], r[c]);
              }
              av = __shfl_sync(0xffffffffu, r[t + 2], j + 2);
              bv = __shfl_sync(0xffffffffu, r[t + 2], j + 3);
              cv = __shfl_sync(0xffffffffu, r[t + 3], j + 3);
#pragma unroll
              for (int c = t + 4; c < SP; ++c) {
                r[c] = fma(-lcol0, l0[c * SLD], r[c]);
                r[c] = fma(-lcol1, l1[c * SLD], r[c]);
              }
            }
          }
          if (j0 + SP < NB) {
            // rank-SP update of the later columns; rows past the panel read
            // the padding rows of Ld and only feed registers past the panel
            const double* lb = Ld + j0 * SLD + j0;  // lb[c * SLD + t] = l_(j0 + c), (j0 + t)
#pragma unroll
            for (int c = SP; c < SP + 2; ++c)
#pragma unroll
              for (int t = 0; t < SP; ++t) r[c] = fma(-lc[t], lb[c * SLD + t], r[c]);
            av = __shfl_sync(0xffffffffu, r[SP], j0 + SP);
            bv = __shfl_sync(0xffffffffu, r[SP], j0 + SP + 1);
            cv = __shfl_sync(0xffffffffu, r[SP + 1], j0 + SP + 1);
#pragma unroll
            for (int c = SP + 2; c < NB; ++c)
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
  };
  // inverse of diagonal block p by a column sweep one pivot behind the chain
  // (CTA 0 warp 1): lane k holds column k of Li = L^-1 in registers (forward
  // substitution of e_k); step j needs only column j of L:
  //   x_j *= 1 / l_jj;   x_i -= l_ij x_j  (i > j, independent FMAs)
  auto inverse = [&](int p) {
    const int c0 = p * NB;
      const int base = p * NB;
      double x[NB];
#pragma unroll
      for (int i = 0; i < NB; ++i) x[i] = (i == lane) ? 1.0 : 0.0;
      int avail = 0;  // columns of this panel published so far
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        if (j >= avail) {  // the chain publishes every 8 pivots: one fence per batch
          int v;
          while ((v = *prog) < base + j + 1) {
          }
          asm volatile("fence.acq_rel.cta;\n" ::: "memory");
          avail = v - base;
        }
        x[j] *= rdg[j];
#pragma unroll
        for (int i = j + 1; i < NB; ++i) x[i] = fma(-Ld[i * SLD + j], x[j], x[i]);
      }
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        D[static_cast<int64_t>(c0 + i) * bi + c0 + lane] = x[i];
        Ls[i * SLD + lane] = x[i];
      }
  };

  // Per panel p two phases separated by cluster barriers X_B(p), X_C(p):
  //   B(p): chain(p) and inverse(p) (done one phase early, see below); the
  //         job warps apply panel p-1's rank-32 update to every trailing
  //         32-block except (p, p), (p+1, p), (p+1, p+1), finalise block row
  //         p-1 of Dinv and add the TRTRI term K = p-2; the critical warps
  //         apply panel p-1 to (p+1, p) and (p+1, p+1).
  //   C(p): the critical warps solve block row p+1 (X = T(p+1,p) Li(p)^T, one
  //         8-row fragment each) and apply it to (p+1, p+1) -- all the next
  //         chain needs; the job warps solve the other rows and add the TRTRI
  //         term K = p-1 of row p.
  // Lookahead: the chain and inverse warps only wait for the critical warps
  // (named barrier 2), arrive at X_C(p) and run chain(p+1) / inverse(p+1)
  // before waiting for X_C(p), so the rest of C(p) and both barrier
  // latencies overlap the next pivot chain.
  arrive();
  wait();
  if (chain_w) chain(0);
  if (inv_w) inverse(0);
  for (int p = 0; p < P; ++p) {
    const int c0 = p * NB;
    const bool next = factor && p + 1 < P;  // block row p+1 exists: critical work in C(p)
    PROF_MARK(0)
    if (wj >= 0) {
      const int m = P - p;  // block rows p .. P-1
      const int skip = next ? 3 : 1;  // (p, p), and (p+1, p), (p+1, p+1) to the critical warps
      const int pre = (factor && p > 0) ? m * (m + 1) / 2 - skip : 0;
      const int inv = (p >= 2) ? p - 1 : 0;  // blocks J = 0..p-2 of row I = p-1
      const int accn = (p >= 2) ? (P - p) * (p - 1) : 0;  // term K = p-2 of rows I >= p
      for (int q = wj; q < pre + inv + accn; q += nwj) {
        if (q < pre) {
          const int qq = q + skip;
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
    } else if (crit >= 0 && next) {
      // blocks (p+1, p) and (p+1, p+1) into Ts / Dd, with panel p-1 applied
      // (row fragment `crit`; they stay in shared memory for C(p))
      const int64_t row = static_cast<int64_t>(p + 1) * NB + 8 * crit;
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        const int cb = p + h;
        double* sdst = (h ? Dd : Ts) + 8 * crit * SLD;
        const double* src = T + row * bi + cb * NB;
        double acc[4][2];
        if (p > 0)
          frag_nt(acc, T + row * bi + c0 - NB, bi, T + static_cast<int64_t>(cb) * NB * bi + c0 - NB, bi, g, t);
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int col = 8 * j + 2 * t + e;
            sdst[g * SLD + col] = src[static_cast<int64_t>(g) * bi + col] - (p > 0 ? acc[j][e] : 0.0);
          }
      }
    }
    arrive();  // X_B(p)
    wait();
    PROF_MARK(1)
    if (*reinterpret_cast<volatile int*>(a.info) >= 0) return;  // set by the chain
    const double* Li = D + static_cast<int64_t>(c0) * bi + c0;
    if (chain_w || inv_w) {
      if (next) asm volatile("bar.sync 2, 192;\n" ::: "memory");  // (p+1, p+1) is final
      arrive();  // X_C(p)
      if (p + 1 < P) {
        if (chain_w) chain(p + 1);
        else inverse(p + 1);
      }
      wait();
    } else {
      if (crit >= 0) {
        if (next) {
          // X = Ts Ls^T (row fragment `crit`) -> L(p+1, p) in T and in Xs
          double* mine = T + (static_cast<int64_t>(p + 1) * NB + 8 * crit) * bi + c0;
          double acc[4][2];
          __syncwarp();
          frag_nt(acc, Ts + 8 * crit * SLD, SLD, Ls, SLD, g, t);
          store_frag(mine, bi, acc, g, t, true, 1.0);
          store_frag(Xs + 8 * crit * SLD, SLD, acc, g, t, true, 1.0);
          asm volatile("bar.sync 1, 128;\n" ::: "memory");  // the four fragments of X
          // Dd -= X X^T: the next chain's input, left in shared memory
          frag_nt(acc, Xs + 8 * crit * SLD, SLD, Xs, SLD, g, t);
          store_frag(Dd + 8 * crit * SLD, SLD, acc, g, t, false, 1.0);
          __threadfence_block();
          asm volatile("bar.arrive 2, 192;\n" ::: "memory");
        }
      } else if (wj >= 0) {
        const int nt = factor ? P - p - 1 : 0;
        const int na = p >= 1 ? p : 0;  // J = 0..p-1
        const int nrow = nt > 1 ? 4 * (nt - 1) : 0;  // rows p+2 .. P-1, 4 fragments each
        const int nsub = nrow + 4 * na;
        for (int q = wj; q < nsub; q += nwj) {
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
      PROF_MARK(7)
      arrive();  // X_C(p)
      wait();
    }
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

size_t potrf_smem_bytes() { return sizeof(double) * (6 * NB * SLD + NB); }

static int g_cluster = -1;

// CTAs per diagonal tile: GPB_POTRF_CLUSTER (2, 4, 8 or 16),
// else 16 where POTRF is on the critical path -- factorisations of fewer
// than 48 diagonal tiles (config 1 factor 8.8 -> 8.2 ms), the first two and
// the last 8 tiles of larger ones -- and 8 otherwise (hidden behind the trailing update,
// where 16 latency-bound SMs would cost GEMM time)
static int potrf_cluster(int tiles, int remaining) {
  if (g_cluster < 0) {
    const char* e = getenv("GPB_POTRF_CLUSTER");
    const int c = e ? atoi(e) : 0;
    g_cluster = (c == 2 || c == 4 || c == 8 || c == 16) ? c : 0;
  }
  if (g_cluster > 0) return g_cluster;
  const bool edge = remaining > 0 && (remaining <= 8 || remaining >= tiles - 1);  // exposed first/last tiles
  return ((tiles > 0 && tiles < 48) || edge) ? 16 : 8;
}

cudaError_t launch_potrf(const PotrfArgs& a, cudaStream_t s) {
  const int cl = potrf_cluster(a.tiles, a.remaining);
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
