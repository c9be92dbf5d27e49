// Grouped DMMA GEMM kernel: 128x128x16 CTA tile, 8 warps (2 x 4, 64x32 per
// warp, 32 DMMA.8x8x4 per k4 step), 4-stage cp.async shared-memory pipeline.
//
// Shared-memory layouts are padded so both DMMA fragment loads and the
// 16-byte cp.async stores are bank-conflict free:
//   K-MAJOR stage  [128][16 + 4] doubles  (row stride 160 B)
//   MN-MAJOR stage [16][128 + 4] doubles  (row stride 1056 B)
// For 8-byte LDS a warp is served in two 16-lane phases; within a phase the
// lanes (g = 0..3, t = 0..3) hit banks 8g + 2t (K-major) or 8t + 2g (MN-major).
#include "gemm.cuh"

namespace gpb {

template <bool KMAJ, int ROWS>
struct StageLayout {
  static constexpr int kLd = KMAJ ? (GBK + 4) : (ROWS + 4);
  static constexpr int kElems = KMAJ ? ROWS * (GBK + 4) : GBK * (ROWS + 4);
};

// Streams one operand's BK-deep k chunks into shared memory.  Per-thread
// source/destination offsets are fixed for the whole k loop; moving to the
// next chunk is a pointer bump (plus a jump of `kstride` when a tiled-k walk
// crosses into the next tile), so the mainloop carries no 64-bit division.
template <bool KMAJ, int ROWS>
struct StageLoader {
  using L = StageLayout<KMAJ, ROWS>;
  static constexpr int kIters = ROWS * GBK / 2 / GTHREADS;  // 16-byte chunks per thread
  const double* cur;  // start of the current k chunk (row0 applied)
  int64_t off0, step;  // thread's first source offset and per-iteration stride
  int soff0;           // thread's first smem offset
  int kin, ktile;
  int64_t kstride;
  int64_t kbump;       // pointer advance per chunk inside a tile

  GPB_DEVINL void init(const double* base, int64_t ld, int64_t kt, int64_t ks, int row0, int tid) {
    ktile = static_cast<int>(kt < (int64_t(1) << 30) ? kt : (int64_t(1) << 30));
    kstride = ks;
    kin = 0;
    if (KMAJ) {
      cur = base + static_cast<int64_t>(row0) * ld;
      const int r = tid >> 3, kc = tid & 7;
      off0 = r * ld + kc * 2;
      step = (GTHREADS / 8) * ld;
      soff0 = r * L::kLd + kc * 2;
      kbump = GBK;
    } else {
      constexpr int kChunksPerRow = ROWS / 2;
      cur = base + row0;
      const int k = tid / kChunksPerRow, mc = tid % kChunksPerRow;
      off0 = k * ld + mc * 2;
      step = (GTHREADS / kChunksPerRow) * ld;
      soff0 = k * L::kLd + mc * 2;
      kbump = GBK * ld;
    }
  }
  GPB_DEVINL void load(double* s) {
    constexpr int sstep = KMAJ ? (GTHREADS / 8) * L::kLd : (GTHREADS / (ROWS / 2)) * L::kLd;
    const double* src = cur + off0;
#pragma unroll
    for (int it = 0; it < kIters; ++it) cp_async16(s + soff0 + it * sstep, src + it * step);
    kin += GBK;
    if (kin >= ktile) {  // next tile of a tiled-k walk
      cur += kstride - static_cast<int64_t>(ktile / GBK - 1) * kbump;
      kin = 0;
    } else {
      cur += kbump;
    }
  }
};

template <bool KMAJ, int ROWS>
GPB_DEVINL double frag(const double* s, int row, int k) {
  using L = StageLayout<KMAJ, ROWS>;
  return KMAJ ? s[row * L::kLd + k] : s[k * L::kLd + row];
}

template <bool AK, bool BK, int EPI>
__global__ void __launch_bounds__(GTHREADS, 1) dgemm_grouped_kernel(const GemmParams p) {
  using LA = StageLayout<AK, GBM>;
  using LB = StageLayout<BK, GBN>;
  extern __shared__ __align__(16) double smem[];
  double* sA = smem;
  double* sB = smem + GSTAGES * LA::kElems;

  const int per_job = p.mblk * p.nblk;
  const int job_id = blockIdx.x / per_job;
  const int local = blockIdx.x - job_id * per_job;
  const int mb = local / p.nblk;
  const int nb = local - mb * p.nblk;
  const GemmJob job = p.jobs[job_id];
  if (job.lower && nb > mb) return;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 2, wn = warp & 3;
  const int g = lane >> 2, t = lane & 3;

  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int nk = job.K / GBK;
  const int arow0 = mb * GBM, brow0 = nb * GBN;
  StageLoader<AK, GBM> la;
  StageLoader<BK, GBN> lb;
  la.init(job.A, p.lda, p.a_ktile, p.a_kstride, arow0, tid);
  lb.init(job.B, p.ldb, p.b_ktile, p.b_kstride, brow0, tid);
#pragma unroll
  for (int s = 0; s < GSTAGES - 1; ++s) {
    if (s < nk) {
      la.load(sA + s * LA::kElems);
      lb.load(sB + s * LB::kElems);
    }
    cp_async_commit();
  }
  for (int kc = 0; kc < nk; ++kc) {
    cp_async_wait<GSTAGES - 2>();
    __syncthreads();
    const int nx = kc + GSTAGES - 1;
    if (nx < nk) {
      const int st = nx % GSTAGES;
      la.load(sA + st * LA::kElems);
      lb.load(sB + st * LB::kElems);
    }
    cp_async_commit();
    const double* a_s = sA + (kc % GSTAGES) * LA::kElems;
    const double* b_s = sB + (kc % GSTAGES) * LB::kElems;
#pragma unroll
    for (int k4 = 0; k4 < GBK; k4 += 4) {
      double af[8], bf[4];
#pragma unroll
      for (int i = 0; i < 8; ++i) af[i] = frag<AK, GBM>(a_s, wm * 64 + i * 8 + g, k4 + t);
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = frag<BK, GBN>(b_s, wn * 32 + j * 8 + g, k4 + t);
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  // ---- epilogue: Cout = alpha * acc + beta * Cin ----
  const int64_t ldc = p.ldc;
  const double alpha = p.alpha, beta = p.beta;
  double colsq[4][2];
#pragma unroll
  for (int j = 0; j < 4; ++j) colsq[j][0] = colsq[j][1] = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t row = arow0 + wm * 64 + i * 8 + g;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t col = brow0 + wn * 32 + j * 8 + 2 * t;
      double2 v;
      v.x = alpha * acc[i][j][0];
      v.y = alpha * acc[i][j][1];
      if (beta != 0.0) {
        const double2 c = *reinterpret_cast<const double2*>(job.Cin + row * ldc + col);
        v.x += beta * c.x;
        v.y += beta * c.y;
      }
      *reinterpret_cast<double2*>(job.Cout + row * ldc + col) = v;
      if (EPI == EPI_SUMSQ) {
        colsq[j][0] += v.x * v.x;
        colsq[j][1] += v.y * v.y;
      }
    }
  }
  if (EPI == EPI_SUMSQ) {
    // reduce over g (lanes t, t+4, ..., t+28), then over the two warp rows
    __syncthreads();  // pipeline smem is free now
    double* red = smem;  // [2][128]
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double v = colsq[j][e];
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        if (g == 0) red[wm * GBN + wn * 32 + j * 8 + 2 * t + e] = v;
      }
    __syncthreads();
    if (tid < GBN) job.aux[static_cast<int64_t>(mb) * p.aux_ld + brow0 + tid] = red[tid] + red[GBN + tid];
  }
}

template <bool AK, bool BK, int EPI>
static size_t smem_bytes() {
  return sizeof(double) * GSTAGES * (StageLayout<AK, GBM>::kElems + StageLayout<BK, GBN>::kElems);
}

template <bool AK, bool BK, int EPI>
static cudaError_t set_attr() {
  return cudaFuncSetAttribute(dgemm_grouped_kernel<AK, BK, EPI>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(smem_bytes<AK, BK, EPI>()));
}

cudaError_t gemm_init_attributes() {
  cudaError_t e;
#define GPB_SET(a, b, c) if ((e = set_attr<a, b, c>()) != cudaSuccess) return e;
  GPB_SET(true, true, EPI_AXPBY)
  GPB_SET(true, false, EPI_AXPBY)
  GPB_SET(true, false, EPI_SUMSQ)
  GPB_SET(false, false, EPI_AXPBY)
  GPB_SET(true, true, EPI_SUMSQ)
  GPB_SET(false, false, EPI_SUMSQ)
  GPB_SET(false, true, EPI_AXPBY)
#undef GPB_SET
  return cudaSuccess;
}

template <bool AK, bool BK, int EPI>
static cudaError_t launch(const GemmParams& p, cudaStream_t s) {
  const long long blocks = static_cast<long long>(p.njobs) * p.mblk * p.nblk;
  if (blocks == 0) return cudaSuccess;
  dgemm_grouped_kernel<AK, BK, EPI>
      <<<static_cast<unsigned>(blocks), GTHREADS, smem_bytes<AK, BK, EPI>(), s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_gemm(const GemmParams& p, bool a_kmajor, bool b_kmajor, int epi,
                        cudaStream_t s) {
  if (epi == EPI_AXPBY) {
    if (a_kmajor && b_kmajor) return launch<true, true, EPI_AXPBY>(p, s);
    if (a_kmajor && !b_kmajor) return launch<true, false, EPI_AXPBY>(p, s);
    if (!a_kmajor && !b_kmajor) return launch<false, false, EPI_AXPBY>(p, s);
    return launch<false, true, EPI_AXPBY>(p, s);
  }
  if (a_kmajor && b_kmajor) return launch<true, true, EPI_SUMSQ>(p, s);
  if (a_kmajor && !b_kmajor) return launch<true, false, EPI_SUMSQ>(p, s);
  if (!a_kmajor && !b_kmajor) return launch<false, false, EPI_SUMSQ>(p, s);
  return cudaErrorInvalidValue;
}

}  // namespace gpb
