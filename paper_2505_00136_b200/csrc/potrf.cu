// Diagonal-tile factorisation: POTRF + TRTRI of one bi x bi tile by one
// thread-block cluster (GPB_POTRF_CLUSTER CTAs, default 8, on as many SMs).
//
// Replaces taskgp tile_potrf (tiles.py:132-137 -> np.linalg.cholesky,
// tiles.py:29-33) and provides the inverted diagonal tile that turns every
// triangular solve of the hot path (panel TRSM tiles.py:140-146, vector
// solves tiles.py:170-180, panel solves tiles.py:182-185) into DMMA products.
//
// Blocked left-looking Cholesky with 32-column panels.  Per panel p:
//   A (all warps)   last contribution (panel p-1) to panel p, DMMA warp tiles
//   B (warp 0)      factor + invert the 32x32 diagonal block -- the serial
//                   pivot chain, kept in registers / shuffles
//     (warps 1..7)  concurrently: contributions of panels 0..p-1 to panel p+1
//                   (in-tile lookahead) and block row p-1 of the inverse
//                   Dinv = L^-1 (TRTRI interleaved with the factorisation)
//   C (all warps)   solve the rows below the diagonal block (x Li^T)
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

// One TRTRI job: D[I][J] = -D[I][I] * sum_{K=J}^{I-1} L[I][K] D[K][J]  (32-blocks)
GPB_DEVINL void trtri_job(double* T, double* D, int bi, int I, int J, double* Sw, int g, int t) {
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
  store_acc(D + static_cast<int64_t>(I) * NB * bi + J * NB, bi, acc, g, t, true, -1.0);
  __syncwarp();
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
  double* Ld = sm;                 // [32][33] factor block
  double* Li = Ld + NB * SLD;      // [32][33] its inverse
  double* S = Li + NB * SLD;       // [8][32][33] per-warp scratch
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
  const int warp = cta * NW + (tid >> 5);  // warp index within the cluster
  const int GW = ncta * NW;                // warps in the cluster
  const int g = lane >> 2, t = lane & 3;
  const bool factor = !a.trtri_only;
  double* Sw = S + (tid >> 5) * NB * SLD;
  double logsum = 0.0;  // meaningful in lane 0 of warp 0
  cluster_barrier(clustered);
  long long t_last = clock64(), t_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#define PROF_MARK(i)                                   \
  if (a.prof && tid == 0) {                            \
    const long long now_ = clock64();                  \
    t_acc[i] += now_ - t_last;                         \
    t_last = now_;                                     \
  }

  for (int p = 0; p < P; ++p) {
    const int c0 = p * NB;
    // A: last contribution (panel p-1) to panel p, rows >= c0
    if (p > 0 && factor) {
      for (int rb = p + warp; rb < P; rb += GW) {
        double acc[4][4][2];
        zero_acc(acc);
        warp_nt(acc, T + static_cast<int64_t>(rb) * NB * bi + c0 - NB, bi,
                T + static_cast<int64_t>(c0) * bi + c0 - NB, bi, NB, g, t);
        store_acc(T + static_cast<int64_t>(rb) * NB * bi + c0, bi, acc, g, t, false, 1.0);
      }
    }
    cluster_barrier(clustered);
    PROF_MARK(0)
    if (warp > 0) {
      // B, warps 1..7: lookahead update of panel p+1 (panels 0..p-1) and
      // block row p-1 of the inverse, dealt round-robin
      const int pre = (factor && p > 0 && p + 1 < P) ? P - p - 1 : 0;
      const int inv = (p >= 2) ? p - 1 : 0;  // jobs J = 0..p-2 of row I = p-1
      // clustered: CTA 0 keeps only the pivot chain so its SMSPs are not
      // shared with DMMA warps; the other CTAs' warps take the jobs
      const int w0 = clustered ? warp - NW : warp - 1;
      const int nwk = clustered ? GW - NW : NW - 1;
      for (int q = (w0 >= 0 ? w0 : pre + inv); q < pre + inv; q += nwk) {
        if (q < pre) {
          const int rb = p + 1 + q, c1 = c0 + NB;
          double acc[4][4][2];
          zero_acc(acc);
          warp_nt(acc, T + static_cast<int64_t>(rb) * NB * bi, bi,
                  T + static_cast<int64_t>(c1) * bi, bi, c0, g, t);
          store_acc(T + static_cast<int64_t>(rb) * NB * bi + c1, bi, acc, g, t, false, 1.0);
        } else {
          trtri_job(T, D, bi, p - 1, q - pre, Sw, g, t);
        }
      }
    } else if (lead) {
      // B, warp 0: lane i keeps row i of the diagonal block in registers,
      // shifted so that register 0 always holds the current pivot column
      // (short code: the pivot loop is not unrolled; LAPACK dpotf2 order)
      double r[NB];
#pragma unroll
      for (int c = 0; c < NB; ++c) r[c] = T[static_cast<int64_t>(c0 + lane) * bi + c0 + c];
      int fail = -1;
      double my_l = 1.0, my_rinv = 0.0;
      if (factor) {
#pragma unroll 1
        for (int j = 0; j < NB; ++j) {
          const double piv = __shfl_sync(0xffffffffu, r[0], j);
          if (fail < 0 && !(piv > 0.0)) fail = j;
          const double rinv = rsqrt(piv);
          const double lcol = (lane == j) ? piv * rinv : (lane > j ? r[0] * rinv : 0.0);
          if (lane == j) {
            my_l = lcol;
            my_rinv = rinv;
          }
          Ld[lane * SLD + j] = lcol;
#pragma unroll
          for (int c = 1; c < NB; ++c) {
            const double lcj = __shfl_sync(0xffffffffu, lcol, (j + c) & (NB - 1));
            if (lane >= j + c) r[c] = fma(-lcol, lcj, r[c]);
          }
#pragma unroll
          for (int c = 0; c < NB - 1; ++c) r[c] = r[c + 1];
        }
        const int pos = a.tile_off + c0 + lane;  // padded global position
        const bool real = (pos % a.bp_user < a.b_user) && (fail < 0 || lane < fail);
        const double lsum = warp_sum(real ? log(my_l) : 0.0);
        if (lane == 0) logsum += lsum;
        PROF_MARK(5)
      } else {  // trtri-only: the tile already holds L
#pragma unroll
        for (int c = 0; c < NB; ++c) Ld[lane * SLD + c] = (c <= lane) ? r[c] : 0.0;
        my_rinv = 1.0 / Ld[lane * SLD + lane];
      }
      if (factor) {
        __syncwarp();
        for (int c = lane + 1; c < NB; ++c) Ld[lane * SLD + c] = 0.0;  // strictly upper
      }
      Li[lane * SLD + lane] = my_rinv;
      __syncwarp();
      if (fail >= 0) {
        if (lane == 0) {
          const int pos = a.tile_off + c0 + fail;
          *reinterpret_cast<volatile int*>(a.info) = (pos / a.bp_user) * a.b_user + pos % a.bp_user;
        }
      } else {
        // lane j forms column j of the inverse by forward substitution (rows
        // of L broadcast from shared memory, the column in shared memory)
#pragma unroll 1
        for (int i = 0; i < NB; ++i) {
          double s0 = (i == lane) ? 1.0 : 0.0, s1 = 0.0;
          int k = 0;
          for (; k + 1 < i; k += 2) {
            s0 = fma(-Ld[i * SLD + k], Li[k * SLD + lane], s0);
            s1 = fma(-Ld[i * SLD + k + 1], Li[(k + 1) * SLD + lane], s1);
          }
          if (k < i) s0 = fma(-Ld[i * SLD + k], Li[k * SLD + lane], s0);
          const double di = Li[i * SLD + i];
          __syncwarp();
          if (i != lane) Li[i * SLD + lane] = (i < lane) ? 0.0 : (s0 + s1) * di;
          __syncwarp();
        }
        PROF_MARK(6)
        for (int c = 0; c < NB; ++c) {
          const int64_t o = static_cast<int64_t>(c0 + lane) * bi + c0 + c;
          if (factor) T[o] = Ld[lane * SLD + c];
          D[o] = Li[lane * SLD + c];
        }
        PROF_MARK(7)
      }
    }
    cluster_barrier(clustered);
    PROF_MARK(1)
    if (*reinterpret_cast<volatile int*>(a.info) >= 0) return;  // set by CTA 0 above
    // C: below-diagonal panel rows, L[r][c0:c0+32] = T[r][c0:c0+32] * Li^T
    // (Li read back from the diagonal block of D, written by CTA 0)
    for (int rb = p + 1 + warp; rb < (factor ? P : 0); rb += GW) {
      double acc[4][4][2];
      zero_acc(acc);
      double* blk = T + static_cast<int64_t>(rb) * NB * bi + c0;
      warp_nt(acc, blk, bi, D + static_cast<int64_t>(c0) * bi + c0, bi, NB, g, t);
      __syncwarp();
      store_acc(blk, bi, acc, g, t, true, 1.0);
    }
    cluster_barrier(clustered);
    PROF_MARK(2)
  }
  // last block row of the inverse (rows 1..P-2 were interleaved above)
  if (P >= 2)
    for (int J = warp; J < P - 1; J += GW) trtri_job(T, D, bi, P - 1, J, Sw, g, t);
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
  if (a.prof && tid == 0 && lead)
    for (int i = 0; i < 8; ++i) a.prof[i] += t_acc[i];
  if (tid == 0 && lead && a.logdiag) a.logdiag[a.tile_index] = logsum;
#undef PROF_MARK
}

size_t potrf_smem_bytes() { return sizeof(double) * (2 * NB * SLD + NW * NB * SLD); }

static int g_cluster = 0;

// CTAs per diagonal tile (GPB_POTRF_CLUSTER: 1 = single CTA, up to 8)
static int potrf_cluster() {
  if (g_cluster == 0) {
    const char* e = getenv("GPB_POTRF_CLUSTER");
    int c = e ? atoi(e) : 8;
    g_cluster = (c == 1 || c == 2 || c == 4 || c == 8) ? c : 8;
  }
  return g_cluster;
}

cudaError_t launch_potrf(const PotrfArgs& a, cudaStream_t s) {
  const int cl = potrf_cluster();
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
  return cudaFuncSetAttribute(potrf_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(potrf_smem_bytes()));
}

}  // namespace gpb
