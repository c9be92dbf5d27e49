// Grouped DMMA GEMM fed by TMA: one elected thread streams 128-byte-swizzled
// k stages into shared memory with cp.async.bulk.tensor behind "full"
// mbarriers; every warp runs DMMA.8x8x4 with no CTA-wide barrier in the
// mainloop.  Same job semantics as dgemm_grouped_kernel (gemm.cuh):
//
//   Cout[job] = alpha * A[job] * B[job]^T + beta * Cin[job]
//
// Each operand is described by one 2-D tensor map per launch over the buffer
// its jobs live in (base, ld, rows): a job's pointer becomes a coordinate
// (row, column) of that view, and the tiled-k walk of a packed tile panel is
// a row jump of kstride / ld per k tile.  TMA therefore needs the caller to
// name the operand buffers (GemmParams::a_base / b_base); launch_gemm falls
// back to the cp.async kernel when they are absent.
//
// Shared-memory layouts (SWIZZLE_128B: the 16-byte chunk c of 128-byte row r
// is stored at chunk c ^ (r & 7)):
//   K-MAJOR stage   [rows][16 k]          one 128-byte row per matrix row
//   MN-MAJOR stage  [rows/16][16 k][16 m] one box per 16 m values
// Fragment reads are conflict-free 16-byte LDS (load_frags):
//   K-MAJOR: each lane fetches k = 8q + 2t, 8q + 2t + 1 at once (chunk 4q + t).
//   A quarter warp holds fragment rows g = 2h, 2h + 1; lane g reads matrix row
//   perm8(g) = (g >> 1) + 4 (g & 1) of its 8-row group, so the two rows' XOR
//   factors differ in bit 2 and the 8 lanes cover all 8 chunks.
//   MN-MAJOR: a lane fetches m = 2g, 2g + 1 of one k row, which feed two
//   fragments (2p: m = 16p + 2g, 2p + 1: m = 16p + 2g + 1); k rows 8q + 2t
//   (+1) put the four t of a quarter warp on XOR factors 2t (+1).
// The epilogue maps accumulators back through the same permutations
// (frag_row).  k is consumed in the order of the paired cp.async kernel, so
// K-major x K-major results are bitwise identical to it.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "gemm.cuh"

namespace gpb {
namespace {

constexpr int TBK = 16;          // k per stage: one 128-byte swizzle atom of doubles
constexpr int kAtom = 128 * 8;   // bytes of an 8-row swizzle pattern

GPB_DEVINL uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

GPB_DEVINL void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(count) : "memory");
}
GPB_DEVINL void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT;\n"
      "}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
GPB_DEVINL void mbar_expect_tx_u32(uint32_t bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
               : "memory");
}
GPB_DEVINL void tma_load(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}

GPB_DEVINL int perm8(int g) { return (g >> 1) + ((g & 1) << 2); }

// One operand's k-stage producer state: the view coordinates of k = 0 and the
// tiled-k walk.  It lives in shared memory (written once by thread 0, read by
// whichever thread refills a stage), which keeps it out of every warp's
// register budget.
struct __align__(16) TmaWalk {
  int c_lo, c_hi;  // K-major: (column, row) of k = 0; MN-major: (m, k row)
  int ktile, kt_rows;
};

template <bool KMAJ>
GPB_DEVINL void walk_init(TmaWalk* w, const double* ptr, const TmaOperand& o, int row0) {
  const int64_t off = ptr - o.base;
  const int64_t r = off / o.ld, c = off - r * o.ld;
  w->c_lo = static_cast<int>(KMAJ ? c : c + row0);
  w->c_hi = static_cast<int>(KMAJ ? r + row0 : r);
  w->ktile = static_cast<int>(o.ktile);
  w->kt_rows = static_cast<int>(o.kt_rows);
}

// k stage kc (k = 16 kc) of one operand into the stage at shared address dst
template <bool KMAJ, int ROWS>
GPB_DEVINL void walk_issue(uint32_t walk, int kc, uint32_t dst, const CUtensorMap* map, uint32_t bar) {
  int4 w;
  asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
               : "r"(walk)
               : "memory");
  const int k = kc * TBK;
  const int kt = k / w.z, kin = k - kt * w.z;
  if (KMAJ) {
    tma_load(dst, map, bar, w.x + kin, w.y + kt * w.w);
  } else {
#pragma unroll
    for (int h = 0; h < ROWS / 16; ++h) tma_load(dst + h * 2048, map, bar, w.x + 16 * h, w.y + kin + kt * w.w);
  }
}

// Fragments of one k step pair (k = 8q + 2t and 8q + 2t + 1) for F 8-row
// fragments starting at stage row `base` (a multiple of 16).
//   K-MAJOR: fragment f, lane g holds row base + 8 f + perm8(g); one 16-byte
//   LDS gives both k values.
//   MN-MAJOR: fragments 2p and 2p + 1 share one 16-wide box: lane g holds
//   m = 16 p + 2 g (fragment 2p) and 16 p + 2 g + 1 (fragment 2p + 1), so one
//   16-byte LDS at k row k0 feeds both fragments.  The chunk g ^ (k0 & 7) of
//   k rows 8q + 2t (+1) spreads a quarter warp over all 8 chunks.
template <bool KMAJ, int F>
GPB_DEVINL void load_frags(const double* s, int base, int g, int q, int t, double2 (&v)[F]) {
  if constexpr (KMAJ) {
    const int pg = perm8(g);
    const double* p = s + (base + pg) * TBK + 2 * ((4 * q + t) ^ pg);
#pragma unroll
    for (int f = 0; f < F; ++f) v[f] = *reinterpret_cast<const double2*>(p + f * 8 * TBK);
  } else {
    const int k0 = 8 * q + 2 * t;
    const double* p0 = s + (base >> 4) * 256 + k0 * 16 + ((g ^ (2 * t)) << 1);
    const double* p1 = s + (base >> 4) * 256 + (k0 + 1) * 16 + ((g ^ (2 * t + 1)) << 1);
#pragma unroll
    for (int f = 0; f < F / 2; ++f) {
      const double2 x0 = *reinterpret_cast<const double2*>(p0 + f * 256);
      const double2 x1 = *reinterpret_cast<const double2*>(p1 + f * 256);
      v[2 * f] = make_double2(x0.x, x1.x);
      v[2 * f + 1] = make_double2(x0.y, x1.y);
    }
  }
}

// stage row of accumulator row g of fragment f (relative to the warp's base)
template <bool KMAJ>
GPB_DEVINL int frag_row(int f, int g) {
  return KMAJ ? f * 8 + perm8(g) : (f >> 1) * 16 + 2 * g + (f & 1);
}

template <int WM, int WN, int STAGES, int BN, int MINB>
struct TmaCfg {
  static constexpr int CW = WM * WN;
  static constexpr int THREADS = CW * 32;
  static constexpr int FM = GBM / WM / 8, FN = BN / WN / 8, CPB = GBN / BN;
  static constexpr int A_BYTES = GBM * TBK * 8, B_BYTES = BN * TBK * 8;
  // byte offsets from the 1024-aligned base: A stages, B stages, "full"
  // barriers, per-stage release counters, the two TmaWalk records
  static constexpr int B_OFF = STAGES * A_BYTES, FULL_OFF = STAGES * (A_BYTES + B_BYTES);
  static constexpr int REL_OFF = FULL_OFF + 8 * STAGES, WALK_OFF = (REL_OFF + 4 * STAGES + 15) / 16 * 16;
  static constexpr size_t SMEM = size_t(WALK_OFF) + 2 * sizeof(TmaWalk) + kAtom;
  static constexpr int kMinB = MINB, kStages = STAGES, kWM = WM, kWN = WN, kBN = BN;
};

template <class C, bool AK, bool BKM, int EPI>
__global__ void __launch_bounds__(C::THREADS, C::kMinB)
    dgemm_tma_kernel(const GemmParams p, const __grid_constant__ CUtensorMap map_a,
                     const __grid_constant__ CUtensorMap map_b, const TmaOperand oa, const TmaOperand ob) {
  constexpr int FM = C::FM, FN = C::FN, BN = C::kBN, STAGES = C::kStages;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // 1024-byte aligned stage base, derived from smem_raw so loads stay LDS
  unsigned char* base = smem_raw + ((kAtom - (su32(smem_raw) & (kAtom - 1))) & (kAtom - 1));
  const double* sA = reinterpret_cast<const double*>(base);
  const double* sB = reinterpret_cast<const double*>(base + C::B_OFF);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + C::FULL_OFF);
  unsigned* released = reinterpret_cast<unsigned*>(base + C::REL_OFF);  // warps done with a stage
  const uint32_t sb = su32(base);
  // stage `st` gets k chunk kc of both operands (one "full" phase)
  auto fill = [&](int st, int kc) {
    const uint32_t bar = sb + C::FULL_OFF + 8 * st;
    mbar_expect_tx_u32(bar, C::A_BYTES + C::B_BYTES);
    walk_issue<AK, GBM>(sb + C::WALK_OFF, kc, sb + st * C::A_BYTES, &map_a, bar);
    walk_issue<BKM, C::kBN>(sb + C::WALK_OFF + 16, kc, sb + C::B_OFF + st * C::B_BYTES, &map_b, bar);
  };

  const int per_job = p.mblk * p.nblk;
  const int lblock = blockIdx.x / C::CPB;
  const int half = blockIdx.x - lblock * C::CPB;
  const int job_id = lblock / per_job;
  const int local = lblock - job_id * per_job;
  const int nb = local / p.mblk;
  const int mb = local - nb * p.mblk;
  const GemmJob job = p.jobs[job_id];
  if (job.lower && nb > mb) return;
  if (job.nlim > 0 && nb >= job.nlim) return;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int nk = job.K / TBK;
  const int arow0 = mb * GBM, brow0 = nb * GBN + half * BN;

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      released[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  const int wm = warp / C::kWN, wn = warp % C::kWN;
  const int g = lane >> 2, t = lane & 3;
  if (p.beta != 0.0 && nk > 0) {
    constexpr int kLinesPerRow = BN * 8 / 128;
    for (int l = tid; l < GBM * kLinesPerRow; l += C::THREADS) {
      const double* a = job.Cin + static_cast<int64_t>(arow0 + l / kLinesPerRow) * p.ldc + brow0 +
                        (l % kLinesPerRow) * 16;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
    }
  }
  // no dedicated producer warp: thread 0 fills every stage up front, and the
  // last warp to release a stage refills it at once (a shared counter per
  // stage), so nobody waits for a free stage, no warp-wide role split costs
  // registers and no CTA barrier sits in the mainloop
  if (tid == 0 && nk > 0) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
    TmaWalk* w = reinterpret_cast<TmaWalk*>(base + C::WALK_OFF);
    walk_init<AK>(w, job.A, oa, arow0);
    walk_init<BKM>(w + 1, job.B, ob, brow0);
    for (int kc = 0; kc < STAGES && kc < nk; ++kc) fill(kc, kc);
  }
  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int am0 = wm * (GBM / C::kWM), bn0 = wn * (BN / C::kWN);
  for (int kc = 0; kc < nk; ++kc) {
    const int st = kc % STAGES;
    mbar_wait(&full[st], (kc / STAGES) & 1);
    const double* a_s = sA + st * (C::A_BYTES / 8);
    const double* b_s = sB + st * (C::B_BYTES / 8);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      double2 av[FM], bv[FN];
      load_frags<AK, FM>(a_s, am0, g, q, t, av);
      load_frags<BKM, FN>(b_s, bn0, g, q, t, bv);
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) dmma884(acc[i][j][0], acc[i][j][1], av[i].x, bv[j].x);
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) dmma884(acc[i][j][0], acc[i][j][1], av[i].y, bv[j].y);
    }
    __syncwarp();
    if (lane == 0 && kc + STAGES < nk) {
      unsigned prev;
      asm volatile("atom.shared.acq_rel.cta.add.u32 %0, [%1], 1;\n"
                   : "=r"(prev)
                   : "r"(su32(&released[st]))
                   : "memory");
      if (prev % C::CW == C::CW - 1) {  // every warp's reads of the stage are done
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        fill(st, kc + STAGES);
      }
    }
  }
  {
    // ---- epilogue: Cout = alpha * acc + beta * Cin ----
    // accumulator (g, t, e) of fragments (i, j) is C[frag_row<AK>(i, g)]
    // [frag_row<BKM>(j, 2t + e)] (DMMA: lane (g, t) holds D[g][2t + e])
    const int64_t ldc = p.ldc;
    const double alpha = p.alpha, beta = p.beta;
    double colsq[FN][2];
#pragma unroll
    for (int j = 0; j < FN; ++j) colsq[j][0] = colsq[j][1] = 0.0;
#pragma unroll
    for (int i = 0; i < FM; ++i) {
      const int64_t off = (arow0 + am0 + frag_row<AK>(i, g)) * ldc + brow0 + bn0;
      double v[FN][2];
#pragma unroll
      for (int j = 0; j < FN; ++j) v[j][0] = alpha * acc[i][j][0], v[j][1] = alpha * acc[i][j][1];
      // all of the row's Cin loads are issued before any store (Cin may alias Cout)
      if (beta != 0.0) {
        double c[FN][2];
        const double* ci = job.Cin + off;
#pragma unroll
        for (int j = 0; j < FN; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            if constexpr (BKM) {
              c[j][e] = ci[frag_row<true>(j, 2 * t + e)];
            } else if ((j & 1) == 0) {  // fragments 2p, 2p + 1: adjacent columns
              const double2 x = *reinterpret_cast<const double2*>(ci + frag_row<false>(j, 2 * t + e));
              c[j][e] = x.x;
              c[j + 1][e] = x.y;
            }
          }
#pragma unroll
        for (int j = 0; j < FN; ++j) v[j][0] += beta * c[j][0], v[j][1] += beta * c[j][1];
      }
      double* co = job.Cout + off;
#pragma unroll
      for (int j = 0; j < FN; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          if constexpr (BKM) {
            co[frag_row<true>(j, 2 * t + e)] = v[j][e];
          } else if ((j & 1) == 0) {
            *reinterpret_cast<double2*>(co + frag_row<false>(j, 2 * t + e)) = make_double2(v[j][e], v[j + 1][e]);
          }
          if (EPI == EPI_SUMSQ) colsq[j][e] += v[j][e] * v[j][e];
        }
      if (EPI == EPI_MIRROR) {
#pragma unroll
        for (int j = 0; j < FN; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) store_mirrors(p, job_id, off + frag_row<BKM>(j, 2 * t + e), v[j][e]);
      }
    }
    if (EPI == EPI_SUMSQ) {
      double* red = reinterpret_cast<double*>(base);  // [WM][BN], pipeline smem is free
      __syncthreads();
#pragma unroll
      for (int j = 0; j < FN; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          double v = colsq[j][e];
          v += __shfl_xor_sync(0xffffffffu, v, 4);
          v += __shfl_xor_sync(0xffffffffu, v, 8);
          v += __shfl_xor_sync(0xffffffffu, v, 16);
          const int col = bn0 + frag_row<BKM>(j, 2 * t + e);
          if (g == 0) red[wm * BN + col] = v;
        }
      __syncthreads();
      if (tid < BN) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < C::kWM; ++w) s += red[w * BN + tid];
        job.aux[static_cast<int64_t>(mb) * p.aux_ld + brow0 + tid] = s;
      }
    }
  }
}

// ---- host side ----------------------------------------------------------------

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

struct MapKey {
  const void* base;
  int64_t ld, rows;
  int box0, box1;
  bool operator==(const MapKey& o) const {
    return base == o.base && ld == o.ld && rows == o.rows && box0 == o.box0 && box1 == o.box1;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    size_t h = reinterpret_cast<size_t>(k.base);
    h = h * 1000003u ^ static_cast<size_t>(k.ld);
    h = h * 1000003u ^ static_cast<size_t>(k.rows);
    h = h * 1000003u ^ static_cast<size_t>(k.box0 * 4096 + k.box1);
    return h;
  }
};

// 2-D view (ld doubles per row, `rows` rows) of the buffer at `base`, cached
bool tensor_map(const double* base, int64_t ld, int64_t rows, int box0, int box1, CUtensorMap* out) {
  static std::mutex mu;
  static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
  const MapKey key{base, ld, rows, box0, box1};
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return true;
  }
  auto fn = encode_fn();
  if (!fn) return false;
  CUtensorMap m;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(ld), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 8};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(box0), static_cast<cuuint32_t>(box1)};
  const cuuint32_t estr[2] = {1, 1};
  if (fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  if (cache.size() > 4096) cache.clear();
  cache.emplace(key, m);
  *out = m;
  return true;
}

// operand view for TMA, or false when this launch cannot use it
bool operand(const double* base, int64_t extent, int64_t ld, int64_t ktile, int64_t kstride, bool kmaj,
             int rows, CUtensorMap* map, TmaOperand* o) {
  if (!base || extent <= 0 || ld <= 0 || (ld & 1) || (reinterpret_cast<uintptr_t>(base) & 15)) return false;
  if (ld * 8 >= (int64_t(1) << 40)) return false;
  const bool tiled = ktile < (int64_t(1) << 30);
  if (tiled && (ktile % TBK || kstride % ld)) return false;
  const int64_t nrows = (extent + ld - 1) / ld;
  if (nrows >= (int64_t(1) << 31) || ld >= (int64_t(1) << 31)) return false;
  if (!tensor_map(base, ld, nrows, 16, kmaj ? rows : 16, map)) return false;
  o->base = base;
  o->ld = ld;
  o->ktile = tiled ? ktile : (int64_t(1) << 30);
  o->kt_rows = tiled ? kstride / ld : 0;
  return true;
}

template <class C, bool AK, bool BKM, int EPI>
cudaError_t tma_launch(const GemmParams& p, const CUtensorMap& ma, const CUtensorMap& mb, const TmaOperand& oa,
                       const TmaOperand& ob, cudaStream_t s) {
  static bool attr = [] {
    return cudaFuncSetAttribute(dgemm_tma_kernel<C, AK, BKM, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(C::SMEM)) == cudaSuccess;
  }();
  if (!attr) return cudaErrorInvalidConfiguration;
  const long long blocks = static_cast<long long>(p.njobs) * p.mblk * p.nblk * C::CPB;
  if (blocks == 0) return cudaSuccess;
  dgemm_tma_kernel<C, AK, BKM, EPI><<<static_cast<unsigned>(blocks), C::THREADS, C::SMEM, s>>>(p, ma, mb, oa, ob);
  return cudaGetLastError();
}

template <class C>
cudaError_t tma_dispatch(const GemmParams& p, bool ak, bool bk, int epi, const CUtensorMap& ma,
                         const CUtensorMap& mb, const TmaOperand& oa, const TmaOperand& ob, cudaStream_t s) {
#define GPB_TMA(a, b, e) \
  if (ak == a && bk == b && epi == e) return tma_launch<C, a, b, e>(p, ma, mb, oa, ob, s);
  GPB_TMA(true, true, EPI_AXPBY)
  GPB_TMA(true, false, EPI_AXPBY)
  GPB_TMA(false, false, EPI_AXPBY)
  GPB_TMA(false, true, EPI_AXPBY)
  GPB_TMA(true, true, EPI_SUMSQ)
  GPB_TMA(true, false, EPI_SUMSQ)
  GPB_TMA(false, false, EPI_SUMSQ)
  GPB_TMA(true, true, EPI_MIRROR)
#undef GPB_TMA
  return cudaErrorInvalidValue;
}

using Tma4 = TmaCfg<2, 2, 4, 64, 2>;  // 4 consumer warps of 64x32, 128x64 CTAs, 2 CTAs/SM
using Tma8 = TmaCfg<4, 2, 4, 64, 2>;  // 8 consumer warps of 32x32

}  // namespace

int g_tma_mode = -1;  // -1: GPB_GEMM_TMA (default on), 0 off, 1 four warps, 2 eight warps

cudaError_t launch_gemm_tma(const GemmParams& p, bool ak, bool bk, int epi, cudaStream_t s, bool* used) {
  *used = false;
  if (g_tma_mode < 0) {
    const char* e = getenv("GPB_GEMM_TMA");
    g_tma_mode = e ? atoi(e) : 3;
  }
  if (g_tma_mode == 0) return cudaSuccess;
  CUtensorMap ma, mb;
  TmaOperand oa{}, ob{};
  if (!operand(p.a_base, p.a_extent, p.lda, p.a_ktile, p.a_kstride, ak, GBM, &ma, &oa)) return cudaSuccess;
  if (!operand(p.b_base, p.b_extent, p.ldb, p.b_ktile, p.b_kstride, bk, Tma8::kBN, &mb, &ob)) return cudaSuccess;
  *used = true;
  // mode 3 (automatic, profiles/r01_gemm_tma_sweep.txt): eight 32x32 warps
  // for short K (the Cholesky update, TRSM and in-group updates), four 64x32
  // warps from K = 4096 (the prediction sweep, the inverse)
  const bool four = g_tma_mode == 1 || (g_tma_mode == 3 && p.max_k >= 4096);
  return four ? tma_dispatch<Tma4>(p, ak, bk, epi, ma, mb, oa, ob, s)
              : tma_dispatch<Tma8>(p, ak, bk, epi, ma, mb, oa, ob, s);
}

void gemm_force_tma(int mode) { g_tma_mode = mode; }

}  // namespace gpb
