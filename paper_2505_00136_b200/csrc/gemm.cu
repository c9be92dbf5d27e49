// Grouped DMMA GEMM kernel: 128x128 CTA tile, DMMA.8x8x4 warp tiles fed from
// a multi-stage cp.async shared-memory pipeline.
//
// The warp layout (WM x WN warps), k depth per stage (BK) and stage count are
// template parameters (GemmCfg); launch_gemm selects the configuration that
// measured fastest on B200 (profiles/r01_gemm_configs.txt), GPB_GEMM_CFG overrides it;
// launches whose operands have tensor-map views run the TMA kernel instead
// (gemm_tma.cu).
//
// Shared-memory layouts are padded so both DMMA fragment loads and the
// 16-byte cp.async stores are bank-conflict free:
//   K-MAJOR stage  [128][BK + 4] doubles
//   MN-MAJOR stage [BK][128 + 4] doubles
// For 8-byte LDS a warp is served in two 16-lane phases; within a phase the
// lanes (g = 0..3, t = 0..3) hit banks 8g + 2t (K-major: (BK+4)*2 = 8 mod 32)
// or 8t + 2g (MN-major: 132*2 = 8 mod 32).
#include <cstdlib>

#include "gemm.cuh"

namespace gpb {

// BN < 128 splits each logical 128x128 block over 128/BN CTAs, which lets
// two CTAs share an SM (one's barrier or epilogue overlaps the other's DMMA).
template <int WM_, int WN_, int BK_, int STAGES_, int BN_ = 128, int MINB_ = 1, bool PAIR_ = false>
struct GemmCfg {
  static constexpr int WM = WM_, WN = WN_, BK = BK_, STAGES = STAGES_;
  // PAIR: each lane loads the k values of two consecutive k-steps with one
  // 16-byte LDS from K-major stages (k-steps 2q / 2q+1 take k = 8q + 2t / +1)
  static constexpr bool PAIR = PAIR_;
  static constexpr int BN = BN_, CPB = GBN / BN_, MINB = MINB_;
  static constexpr int THREADS = WM * WN * 32;
  static constexpr int FM = GBM / WM / 8;  // 8-row fragments per warp
  static constexpr int FN = BN / WN / 8;   // 8-col fragments per warp
};

template <class C, bool KMAJ, int ROWS>
struct StageLayout {
  // K-major pitch: BK + 4 keeps 8-byte fragment loads conflict-free; the
  // 16-byte loads of PAIR need BK + 8 (2 * pitch = 16 mod 32 banks)
  static constexpr int kLd = KMAJ ? (C::BK + (C::PAIR ? 8 : 4)) : (ROWS + 4);
  static constexpr int kElems = KMAJ ? ROWS * kLd : C::BK * (ROWS + 4);
};

// Streams one operand's BK-deep k chunks into shared memory.  Per-thread
// source/destination offsets are fixed for the whole k loop; moving to the
// next chunk is a pointer bump (plus a jump of `kstride` when a tiled-k walk
// crosses into the next tile), so the mainloop carries no 64-bit division.
template <class C, bool KMAJ, int ROWS>
struct StageLoader {
  using L = StageLayout<C, KMAJ, ROWS>;
  static constexpr int kChunksPerRow = KMAJ ? C::BK / 2 : ROWS / 2;  // 16-byte chunks
  static constexpr int kRowsPerIter = C::THREADS / kChunksPerRow;
  static constexpr int kIters = ROWS * C::BK / 2 / C::THREADS;
  static_assert(kIters >= 1, "tile too small for the thread count");
  const double* cur;  // start of the current k chunk (row0 applied)
  int64_t off0, step;
  int soff0;
  int kin, ktile;
  int64_t kstride, kbump;

  GPB_DEVINL void init(const double* base, int64_t ld, int64_t kt, int64_t ks, int row0, int tid) {
    ktile = static_cast<int>(kt < (int64_t(1) << 30) ? kt : (int64_t(1) << 30));
    kstride = ks;
    kin = 0;
    const int r = tid / kChunksPerRow, c = tid % kChunksPerRow;
    if (KMAJ) {
      cur = base + static_cast<int64_t>(row0) * ld;
      off0 = r * ld + c * 2;
      step = kRowsPerIter * ld;
      soff0 = r * L::kLd + c * 2;
      kbump = C::BK;
    } else {
      cur = base + row0;
      off0 = r * ld + c * 2;
      step = kRowsPerIter * ld;
      soff0 = r * L::kLd + c * 2;
      kbump = C::BK * ld;
    }
  }
  GPB_DEVINL void load(double* s) {
    const double* src = cur + off0;
#pragma unroll
    for (int it = 0; it < kIters; ++it) cp_async16(s + soff0 + it * kRowsPerIter * L::kLd, src + it * step);
    kin += C::BK;
    if (kin >= ktile) {  // next tile of a tiled-k walk
      cur += kstride - static_cast<int64_t>(ktile / C::BK - 1) * kbump;
      kin = 0;
    } else {
      cur += kbump;
    }
  }
};

template <class C, bool KMAJ, int ROWS>
GPB_DEVINL double frag(const double* s, int row, int k) {
  using L = StageLayout<C, KMAJ, ROWS>;
  return KMAJ ? s[row * L::kLd + k] : s[k * L::kLd + row];
}

// values at k and k + 1 of one row (K-major: one 16-byte load)
template <class C, bool KMAJ, int ROWS>
GPB_DEVINL double2 frag2(const double* s, int row, int k) {
  using L = StageLayout<C, KMAJ, ROWS>;
  if constexpr (KMAJ) return *reinterpret_cast<const double2*>(s + row * L::kLd + k);
  return make_double2(s[k * L::kLd + row], s[(k + 1) * L::kLd + row]);
}

template <class C, bool AK, bool BK, int EPI>
__global__ void __launch_bounds__(C::THREADS, C::MINB) dgemm_grouped_kernel(const GemmParams p) {
  using LA = StageLayout<C, AK, GBM>;
  using LB = StageLayout<C, BK, C::BN>;
  constexpr int FM = C::FM, FN = C::FN;
  extern __shared__ __align__(16) double smem[];
  double* sA = smem;
  double* sB = smem + C::STAGES * LA::kElems;

  const int per_job = p.mblk * p.nblk;
  const int lblock = blockIdx.x / C::CPB;  // logical 128x128 block
  const int half = blockIdx.x - lblock * C::CPB;
  const int job_id = lblock / per_job;
  const int local = lblock - job_id * per_job;
  // row blocks fastest: the CTAs that share a B column block (the big operand
  // of the prediction sweep) are resident together and hit it in L2
  const int nb = local / p.mblk;
  const int mb = local - nb * p.mblk;
  const GemmJob job = p.jobs[job_id];
  if (job.lower && nb > mb) return;
  if (job.nlim > 0 && nb >= job.nlim) return;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wm = warp / C::WN, wn = warp % C::WN;
  const int g = lane >> 2, t = lane & 3;

  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int nk = job.K / C::BK;
  const int arow0 = mb * GBM, brow0 = nb * GBN + half * C::BN;
  if (p.beta != 0.0 && nk > 0) {
    // warm L2 with this CTA's C block so the epilogue's read-modify-write
    // does not wait on HBM (128 rows x BN doubles = 128 * BN / 16 lines)
    constexpr int kLinesPerRow = C::BN * 8 / 128;
    for (int l = tid; l < GBM * kLinesPerRow; l += C::THREADS) {
      const double* a = job.Cin + static_cast<int64_t>(arow0 + l / kLinesPerRow) * p.ldc + brow0 +
                        (l % kLinesPerRow) * 16;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
    }
  }
  StageLoader<C, AK, GBM> la;
  StageLoader<C, BK, C::BN> lb;
  la.init(job.A, p.lda, p.a_ktile, p.a_kstride, arow0, tid);
  lb.init(job.B, p.ldb, p.b_ktile, p.b_kstride, brow0, tid);
#pragma unroll
  for (int s = 0; s < C::STAGES - 1; ++s) {
    if (s < nk) {
      la.load(sA + s * LA::kElems);
      lb.load(sB + s * LB::kElems);
    }
    cp_async_commit();
  }
  const int am0 = wm * (GBM / C::WM) + g, bn0 = wn * (C::BN / C::WN) + g;
  for (int kc = 0; kc < nk; ++kc) {
    cp_async_wait<C::STAGES - 2>();
    __syncthreads();
    const int nx = kc + C::STAGES - 1;
    if (nx < nk) {
      const int st = nx % C::STAGES;
      la.load(sA + st * LA::kElems);
      lb.load(sB + st * LB::kElems);
    }
    cp_async_commit();
    const double* a_s = sA + (kc % C::STAGES) * LA::kElems;
    const double* b_s = sB + (kc % C::STAGES) * LB::kElems;
    if constexpr (C::PAIR) {
#pragma unroll
      for (int k8 = 0; k8 < C::BK; k8 += 8) {
        double2 av[FM], bv[FN];
#pragma unroll
        for (int i = 0; i < FM; ++i) av[i] = frag2<C, AK, GBM>(a_s, am0 + i * 8, k8 + 2 * t);
#pragma unroll
        for (int j = 0; j < FN; ++j) bv[j] = frag2<C, BK, C::BN>(b_s, bn0 + j * 8, k8 + 2 * t);
#pragma unroll
        for (int i = 0; i < FM; ++i)
#pragma unroll
          for (int j = 0; j < FN; ++j) dmma884(acc[i][j][0], acc[i][j][1], av[i].x, bv[j].x);
#pragma unroll
        for (int i = 0; i < FM; ++i)
#pragma unroll
          for (int j = 0; j < FN; ++j) dmma884(acc[i][j][0], acc[i][j][1], av[i].y, bv[j].y);
      }
    } else {
#pragma unroll
      for (int k4 = 0; k4 < C::BK; k4 += 4) {
        double af[FM], bf[FN];
#pragma unroll
        for (int i = 0; i < FM; ++i) af[i] = frag<C, AK, GBM>(a_s, am0 + i * 8, k4 + t);
#pragma unroll
        for (int j = 0; j < FN; ++j) bf[j] = frag<C, BK, C::BN>(b_s, bn0 + j * 8, k4 + t);
#pragma unroll
        for (int i = 0; i < FM; ++i)
#pragma unroll
          for (int j = 0; j < FN; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
    }
  }
  cp_async_wait<0>();

  // ---- epilogue: Cout = alpha * acc + beta * Cin ----
  const int64_t ldc = p.ldc;
  const double alpha = p.alpha, beta = p.beta;
  double colsq[FN][2];
#pragma unroll
  for (int j = 0; j < FN; ++j) colsq[j][0] = colsq[j][1] = 0.0;
#pragma unroll
  for (int i = 0; i < FM; ++i) {
    const int64_t row = arow0 + am0 + i * 8;
#pragma unroll
    for (int j = 0; j < FN; ++j) {
      const int64_t col = brow0 + wn * (C::BN / C::WN) + j * 8 + 2 * t;
      double2 v;
      v.x = alpha * acc[i][j][0];
      v.y = alpha * acc[i][j][1];
      if (beta != 0.0) {
        const double2 c = *reinterpret_cast<const double2*>(job.Cin + row * ldc + col);
        v.x += beta * c.x;
        v.y += beta * c.y;
      }
      *reinterpret_cast<double2*>(job.Cout + row * ldc + col) = v;
      if (EPI == EPI_MIRROR) {
        store_mirrors(p, job_id, row * ldc + col, v.x);
        store_mirrors(p, job_id, row * ldc + col + 1, v.y);
      }
      if (EPI == EPI_SUMSQ) {
        colsq[j][0] += v.x * v.x;
        colsq[j][1] += v.y * v.y;
      }
    }
  }
  if (EPI == EPI_SUMSQ) {
    // reduce over g (lanes t, t+4, ..., t+28), then over the WM warp rows in order
    __syncthreads();  // pipeline smem is free now
    double* red = smem;  // [WM][BN]
#pragma unroll
    for (int j = 0; j < FN; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double v = colsq[j][e];
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        if (g == 0) red[wm * C::BN + wn * (C::BN / C::WN) + j * 8 + 2 * t + e] = v;
      }
    __syncthreads();
    if (tid < C::BN) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < C::WM; ++w) s += red[w * C::BN + tid];
      job.aux[static_cast<int64_t>(mb) * p.aux_ld + brow0 + tid] = s;
    }
  }
}

template <class C, bool AK, bool BK>
static size_t smem_bytes() {
  return sizeof(double) * C::STAGES *
         (StageLayout<C, AK, GBM>::kElems + StageLayout<C, BK, C::BN>::kElems);
}

template <class C, bool AK, bool BK, int EPI>
static cudaError_t set_attr() {
  return cudaFuncSetAttribute(dgemm_grouped_kernel<C, AK, BK, EPI>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(smem_bytes<C, AK, BK>()));
}

template <class C, bool AK, bool BK, int EPI>
static cudaError_t launch(const GemmParams& p, cudaStream_t s) {
  const long long blocks = static_cast<long long>(p.njobs) * p.mblk * p.nblk * C::CPB;
  if (blocks == 0) return cudaSuccess;
  dgemm_grouped_kernel<C, AK, BK, EPI>
      <<<static_cast<unsigned>(blocks), C::THREADS, smem_bytes<C, AK, BK>(), s>>>(p);
  return cudaGetLastError();
}

template <class C>
static cudaError_t init_cfg() {
  cudaError_t e;
#define GPB_SET(a, b, c) if ((e = set_attr<C, a, b, c>()) != cudaSuccess) return e;
  GPB_SET(true, true, EPI_AXPBY)
  GPB_SET(true, false, EPI_AXPBY)
  GPB_SET(true, false, EPI_SUMSQ)
  GPB_SET(false, false, EPI_AXPBY)
  GPB_SET(true, true, EPI_SUMSQ)
  GPB_SET(false, false, EPI_SUMSQ)
  GPB_SET(false, true, EPI_AXPBY)
  GPB_SET(true, true, EPI_MIRROR)
#undef GPB_SET
  return cudaSuccess;
}

template <class C>
static cudaError_t dispatch(const GemmParams& p, bool ak, bool bk, int epi, cudaStream_t s) {
  if (epi == EPI_MIRROR) {
    if (ak && bk) return launch<C, true, true, EPI_MIRROR>(p, s);
    return cudaErrorInvalidValue;
  }
  if (epi == EPI_AXPBY) {
    if (ak && bk) return launch<C, true, true, EPI_AXPBY>(p, s);
    if (ak && !bk) return launch<C, true, false, EPI_AXPBY>(p, s);
    if (!ak && !bk) return launch<C, false, false, EPI_AXPBY>(p, s);
    return launch<C, false, true, EPI_AXPBY>(p, s);
  }
  if (ak && bk) return launch<C, true, true, EPI_SUMSQ>(p, s);
  if (ak && !bk) return launch<C, true, false, EPI_SUMSQ>(p, s);
  if (!ak && !bk) return launch<C, false, false, EPI_SUMSQ>(p, s);
  return cudaErrorInvalidValue;
}

using Cfg0 = GemmCfg<2, 4, 16, 4>;  // 8 warps, 64x32 warp tiles, BK 16
using Cfg1 = GemmCfg<4, 4, 16, 4>;  // 16 warps, 32x32 warp tiles, BK 16
using Cfg2 = GemmCfg<2, 4, 32, 3>;  // 8 warps, BK 32
using Cfg3 = GemmCfg<4, 4, 32, 3>;  // 16 warps, BK 32
using Cfg4 = GemmCfg<4, 2, 16, 3, 64, 2>;  // 128x64 CTAs, 8 warps (32x32), 2 CTAs/SM
using Cfg5 = GemmCfg<2, 2, 16, 3, 64, 2>;  // 128x64 CTAs, 4 warps (64x32), 2 CTAs/SM
using Cfg6 = GemmCfg<2, 4, 16, 5>;         // 8 warps, 5 stages
using Cfg7 = GemmCfg<4, 2, 32, 2, 64, 2>;  // 128x64, 8 warps, BK 32, 2 stages, 2 CTAs/SM
using Cfg8 = GemmCfg<4, 2, 16, 3, 64, 2, true>;  // Cfg4 with paired k loads
using Cfg9 = GemmCfg<2, 2, 16, 3, 64, 2, true>;  // Cfg5 with paired k loads

static int g_cfg = -1;

// Default (tools/gemm_bench.cu, profiles/r01_gemm_configs.txt): two
// co-resident 128x64 CTAs per SM with paired 16-byte k loads -- 4 warps of
// 64x32 when K is long (>= 4096: the prediction sweep, +2.6% over unpaired),
// else 8 warps of 32x32 when both operands are K-major (the Cholesky update),
// else the unpaired 8-warp kernel.  GPB_GEMM_CFG forces one.
static void resolve_cfg() {
  if (g_cfg < 0) {
    const char* e = getenv("GPB_GEMM_CFG");
    g_cfg = e ? atoi(e) : 99;
    if (g_cfg < 0 || (g_cfg > 9 && g_cfg != 99)) g_cfg = 99;
  }
}

static int gemm_cfg(const GemmParams& p, bool ak, bool bk) {
  resolve_cfg();
  if (g_cfg != 99) return g_cfg;
  if (p.max_k >= 4096) return 9;
  return (ak && bk) ? 8 : 4;
}

void gemm_force_config(int cfg) { g_cfg = cfg; }

cudaError_t gemm_init_attributes() {
  cudaError_t e;
  if ((e = init_cfg<Cfg0>()) != cudaSuccess) return e;
  if ((e = init_cfg<Cfg1>()) != cudaSuccess) return e;
  if ((e = init_cfg<Cfg2>()) != cudaSuccess) return e;
  if ((e = init_cfg<Cfg4>()) != cudaSuccess) return e;
  if ((e = init_cfg<Cfg5>()) != cudaSuccess) return e;
  if ((e = init_cfg<Cfg6>()) != cudaSuccess) return e;
  if ((e = init_cfg<Cfg7>()) != cudaSuccess) return e;
  if ((e = init_cfg<Cfg8>()) != cudaSuccess) return e;
  if ((e = init_cfg<Cfg9>()) != cudaSuccess) return e;
  return init_cfg<Cfg3>();
}

cudaError_t launch_gemm(const GemmParams& p, bool a_kmajor, bool b_kmajor, int epi,
                        cudaStream_t s) {
  resolve_cfg();
  if (g_cfg == 99) {  // forced cp.async configurations bypass TMA
    bool used = false;
    const cudaError_t e = launch_gemm_tma(p, a_kmajor, b_kmajor, epi, s, &used);
    if (used || e != cudaSuccess) return e;
  }
  switch (gemm_cfg(p, a_kmajor, b_kmajor)) {
    case 1: return dispatch<Cfg1>(p, a_kmajor, b_kmajor, epi, s);
    case 2: return dispatch<Cfg2>(p, a_kmajor, b_kmajor, epi, s);
    case 3: return dispatch<Cfg3>(p, a_kmajor, b_kmajor, epi, s);
    case 4: return dispatch<Cfg4>(p, a_kmajor, b_kmajor, epi, s);
    case 5: return dispatch<Cfg5>(p, a_kmajor, b_kmajor, epi, s);
    case 6: return dispatch<Cfg6>(p, a_kmajor, b_kmajor, epi, s);
    case 7: return dispatch<Cfg7>(p, a_kmajor, b_kmajor, epi, s);
    case 8: return dispatch<Cfg8>(p, a_kmajor, b_kmajor, epi, s);
    case 9: return dispatch<Cfg9>(p, a_kmajor, b_kmajor, epi, s);
    default: return dispatch<Cfg0>(p, a_kmajor, b_kmajor, epi, s);
  }
}

}  // namespace gpb
