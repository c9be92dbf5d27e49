// Diagonal-tile factorisation: POTRF + TRTRI of one bi x bi tile in one CTA.
//
// Replaces taskgp tile_potrf (tiles.py:132-137 -> np.linalg.cholesky,
// tiles.py:29-33) and provides the inverted diagonal tile that turns every
// triangular solve of the hot path (panel TRSM tiles.py:140-146, vector
// solves tiles.py:170-180, panel solves tiles.py:182-185) into DMMA products.
//
// Blocked left-looking Cholesky with 32-column panels; the panel update and
// the below-diagonal solve run on the FP64 tensor pipe (DMMA.8x8x4) warp by
// warp; the 32x32 diagonal block is factored and inverted in shared memory
// by one warp.  TRTRI then forms Dinv = L^-1 block row by block row.
// Epilogue: Sigma log L_jj over real (non-padding) pivots and a LAPACK-style
// info word holding the first failing global pivot.
#include "common.cuh"
#include "kernels.cuh"

namespace gpb {

namespace {

constexpr int PT = 256;  // threads
constexpr int NB = 32;   // panel width
constexpr int SLD = NB + 1;

// acc[i][j][e] <-> C[8i+g][8j+2t+e] of a 32x32 warp tile.
GPB_DEVINL void zero_acc(double (&acc)[4][4][2]) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
}

// acc += A(32 x K) * B(32 x K)^T, both k-contiguous, K a multiple of 32.
// Operands come straight from L2 (the tile is produced inside this kernel),
// so the loop is latency-bound: fragments for a 16-deep k chunk (32 loads per
// lane) are fetched one chunk ahead of the DMMAs that consume them.
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

GPB_DEVINL void mma_chunk(double (&acc)[4][4][2], const double (&a)[4][4], const double (&b)[4][4]) {
#pragma unroll
  for (int s = 0; s < 4; ++s)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[s][i], b[s][j]);
}

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

// acc += A(32 x K) * B(K x 32), A k-contiguous, B row-major (n contiguous);
// same one-chunk-ahead fragment prefetch as warp_nt.
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

}  // namespace

__global__ void __launch_bounds__(PT, 1) potrf_tile_kernel(PotrfArgs a) {
  extern __shared__ double sm[];
  double* Ld = sm;                 // [32][33] factor block
  double* Li = Ld + NB * SLD;      // [32][33] its inverse
  double* S = Li + NB * SLD;       // [8][32][33] per-warp scratch
  __shared__ int s_fail;

  if (*a.info >= 0) return;  // an earlier tile already failed
  const int bi = a.bi;
  double* T = a.tile;
  double* D = a.dinv;
  const int P = bi / NB;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  if (tid == 0) s_fail = -1;
  double logsum = 0.0;  // meaningful in lane 0 of warp 0
  __syncthreads();
  long long t_last = clock64(), t_acc[5] = {0, 0, 0, 0, 0};
#define PROF_MARK(i) if (a.prof && tid == 0) { const long long now_ = clock64(); t_acc[i] += now_ - t_last; t_last = now_; }

  for (int p = 0; p < P; ++p) {
    const int c0 = p * NB;
    // (1) left-looking panel update, last contribution only:
    //     T[r][c0:c0+32] -= L[r][c0-32:c0] L[c0:c0+32][c0-32:c0]^T
    //     (panels 0..p-2 were applied in step p-1 while warp 0 factored)
    if (p > 0 && !a.trtri_only) {
      for (int rb = p + warp; rb < P; rb += PT / 32) {
        double acc[4][4][2];
        zero_acc(acc);
        warp_nt(acc, T + static_cast<int64_t>(rb) * NB * bi + c0 - NB, bi,
                T + static_cast<int64_t>(c0) * bi + c0 - NB, bi, NB, g, t);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            double* c = T + static_cast<int64_t>(rb * NB + 8 * i + g) * bi + c0 + 8 * j + 2 * t;
            c[0] -= acc[i][j][0];
            c[1] -= acc[i][j][1];
          }
      }
    }
    __syncthreads();
    PROF_MARK(0)
    // (2') lookahead inside the tile: warps 1..7 apply panels 0..p-1 to panel
    //      p+1 while warp 0 factors the diagonal block of panel p
    if (warp > 0 && p > 0 && p + 1 < P && !a.trtri_only) {
      const int c1 = c0 + NB;
      for (int rb = p + warp; rb < P; rb += PT / 32 - 1) {
        double acc[4][4][2];
        zero_acc(acc);
        warp_nt(acc, T + static_cast<int64_t>(rb) * NB * bi, bi, T + static_cast<int64_t>(c1) * bi,
                bi, c0, g, t);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            double* c = T + static_cast<int64_t>(rb * NB + 8 * i + g) * bi + c1 + 8 * j + 2 * t;
            c[0] -= acc[i][j][0];
            c[1] -= acc[i][j][1];
          }
      }
    }
    // (2) factor + invert the 32x32 diagonal block (one warp)
    if (warp == 0) {
      // lane i keeps row i of the block in registers; the right-looking
      // unblocked factorisation (LAPACK dpotf2 order: scale by 1/l_jj, then
      // rank-1 update) exchanges column j through warp shuffles.
      double r[NB];
#pragma unroll
      for (int c = 0; c < NB; ++c) r[c] = T[static_cast<int64_t>(c0 + lane) * bi + c0 + c];
      int fail = -1;
      double my_rinv = 0.0;  // lane j: 1 / l_jj
      if (!a.trtri_only) {
        // critical chain per pivot: shuffle -> rsqrt -> scale -> shuffle -> fma
        // (no divide, no log inside the chain)
        double my_l = 1.0;
#pragma unroll
        for (int j = 0; j < NB; ++j) {
          const double piv = __shfl_sync(0xffffffffu, r[j], j);
          if (fail < 0 && !(piv > 0.0)) fail = j;
          const double rinv = rsqrt(piv);
          const double ljj = piv * rinv;
          if (lane == j) {
            r[j] = ljj;
            my_l = ljj;
            my_rinv = rinv;
          } else if (lane > j) {
            r[j] *= rinv;
          }
#pragma unroll
          for (int c = 0; c < NB; ++c) {
            if (c > j) {
              const double lcj = __shfl_sync(0xffffffffu, r[j], c);
              if (lane >= c) r[c] = fma(-r[j], lcj, r[c]);
            }
          }
        }
        // log-determinant partial: every lane its own pivot, fixed-order butterfly
        const int pos = a.tile_off + c0 + lane;  // padded global position
        const bool real = (pos % a.bp_user < a.b_user) && (fail < 0 || lane < fail);
        const double lsum = warp_sum(real ? log(my_l) : 0.0);
        if (lane == 0) logsum += lsum;
      } else {
        my_rinv = 1.0 / r[lane];  // trtri-only: lane's diagonal entry of L
      }
#pragma unroll
      for (int c = 0; c < NB; ++c) Ld[lane * SLD + c] = (c <= lane) ? r[c] : 0.0;
      Li[lane * SLD + lane] = my_rinv;  // diagonal reciprocals for the inverse
      __syncwarp();
      if (fail >= 0) {
        if (lane == 0) {
          const int pos = a.tile_off + c0 + fail;
          s_fail = (pos / a.bp_user) * a.b_user + pos % a.bp_user;
        }
      } else {
        // lane j forms column j of the inverse by forward substitution; the
        // rows of L are shared-memory broadcasts, the column stays in registers
        // (four interleaved partial sums keep the dependent FMA chain short)
        double x[NB], dinv[NB];
#pragma unroll
        for (int i = 0; i < NB; ++i) dinv[i] = Li[i * SLD + i];
        __syncwarp();
#pragma unroll
        for (int i = 0; i < NB; ++i) {
          double s0 = (i == lane) ? 1.0 : 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
          for (int k = 0; k < NB; ++k) {
            if (k < i) {
              const double t_ = -Ld[i * SLD + k] * x[k];
              if ((k & 3) == 0) s0 += t_;
              else if ((k & 3) == 1) s1 += t_;
              else if ((k & 3) == 2) s2 += t_;
              else s3 += t_;
            }
          }
          x[i] = ((s0 + s1) + (s2 + s3)) * dinv[i];
        }
#pragma unroll
        for (int i = 0; i < NB; ++i) Li[i * SLD + lane] = x[i];
        __syncwarp();
        for (int c = 0; c < NB; ++c) {
          const int64_t o = static_cast<int64_t>(c0 + lane) * bi + c0 + c;
          if (!a.trtri_only) T[o] = c <= lane ? Ld[lane * SLD + c] : 0.0;
          D[o] = Li[lane * SLD + c];
        }
      }
    }
    __syncthreads();
    PROF_MARK(1)
    if (s_fail >= 0) break;
    // (3) below-diagonal panel: L[r][c0:c0+32] = T[r][c0:c0+32] * Li^T
    for (int rb = p + 1 + warp; rb < (a.trtri_only ? 0 : P); rb += PT / 32) {
      double acc[4][4][2];
      zero_acc(acc);
      double* blk = T + static_cast<int64_t>(rb) * NB * bi + c0;
      warp_nt(acc, blk, bi, Li, SLD, NB, g, t);
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          double* c = blk + static_cast<int64_t>(8 * i + g) * bi + 8 * j + 2 * t;
          c[0] = acc[i][j][0];
          c[1] = acc[i][j][1];
        }
    }
    __syncthreads();
    PROF_MARK(2)
  }
  if (s_fail >= 0) {
    if (tid == 0) *a.info = s_fail;
    return;
  }
  // zero strictly-upper 32-blocks of L and Dinv (lower-triangular results)
  for (int r = warp; r < bi; r += PT / 32) {
    const int c_begin = (r / NB + 1) * NB;  // first column of the strictly-upper blocks
    for (int c = c_begin + 2 * lane; c < bi; c += 64) {
      const int64_t idx = static_cast<int64_t>(r) * bi + c;
      if (!a.trtri_only) *reinterpret_cast<double2*>(T + idx) = make_double2(0.0, 0.0);
      *reinterpret_cast<double2*>(D + idx) = make_double2(0.0, 0.0);
    }
  }
  __syncthreads();
    PROF_MARK(3)
  // TRTRI: D[I][J] = -D[I][I] * sum_{K=J}^{I-1} L[I][K] D[K][J]
  double* Sw = S + warp * NB * SLD;
  for (int I = 1; I < P; ++I) {
    for (int J = warp; J < I; J += PT / 32) {
      double acc[4][4][2];
      zero_acc(acc);
      warp_nn(acc, T + static_cast<int64_t>(I) * NB * bi + J * NB, bi,
              D + static_cast<int64_t>(J) * NB * bi + J * NB, bi, (I - J) * NB, g, t);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          Sw[(8 * i + g) * SLD + 8 * j + 2 * t] = acc[i][j][0];
          Sw[(8 * i + g) * SLD + 8 * j + 2 * t + 1] = acc[i][j][1];
        }
      __syncwarp();
      zero_acc(acc);
      warp_nn(acc, D + static_cast<int64_t>(I) * NB * bi + I * NB, bi, Sw, SLD, NB, g, t);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          double* c = D + static_cast<int64_t>(I * NB + 8 * i + g) * bi + J * NB + 8 * j + 2 * t;
          c[0] = -acc[i][j][0];
          c[1] = -acc[i][j][1];
        }
      __syncwarp();
    }
    __syncthreads();
  }
  PROF_MARK(4)
  if (a.prof && tid == 0) for (int i = 0; i < 5; ++i) a.prof[i] += t_acc[i];
  if (tid == 0 && a.logdiag) a.logdiag[a.tile_index] = logsum;
}

size_t potrf_smem_bytes() { return sizeof(double) * (2 * NB * SLD + (PT / 32) * NB * SLD); }

cudaError_t launch_potrf(const PotrfArgs& a, cudaStream_t s) {
  potrf_tile_kernel<<<1, PT, potrf_smem_bytes(), s>>>(a);
  return cudaGetLastError();
}

cudaError_t potrf_init_attributes() {
  return cudaFuncSetAttribute(potrf_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(potrf_smem_bytes()));
}

}  // namespace gpb
