// tcgen05 (kind::i8, TMEM accumulators) digit-plane product; see ozaki.cuh.
//
// Kernel shape.  One CTA per 128 x 128 output block, six warps:
//   warp 0   producer: per 32-byte k chunk ONE bulk copy (cp.async.bulk) per
//            operand brings the P planes the launch needs (P x 4 KB, already in
//            the MMA's shared-memory layout) into a ring of 3-4 stages behind
//            "full" mbarriers; it also owns the TMEM allocation;
//   warp 1   MMA issuer: one thread issues, per chunk, every digit pair (p, q),
//            p + q = g, of the launch's group window as tcgen05.mma M = 128,
//            N = 128, K = 32 into the int32 accumulator of group g; a
//            tcgen05.commit frees the stage;
//   warps 2-5 epilogue: after the last commit each thread owns one output row
//            (TMEM lane), reads its 128 columns of every group with tcgen05.ld,
//            combines the groups in FP64 (Horner in 2^-7, least significant
//            group first) and writes Cout = beta Cin + alpha sum.
// TMEM holds four 128-column accumulators, so the S digit groups are computed
// in two launches of up to four groups each, least significant first: launch
// one loads all S planes and adds groups [S-4, S) to C, launch two loads
// planes 0 .. S-5 only and adds groups [0, S-4).
//
// How the shape was arrived at (one B200, 8 planes, M = 512, N = 32768,
// K = 16384, FP64-equivalent rate):
//   128 x 64 blocks, 8 accumulators of 64 columns, 64-byte TMA boxes: 78 TF/s --
//     6 KB of shared-memory operand reads per 32-cycle MMA (fetch bound);
//   128 x 128 blocks in two group windows, 32-byte TMA boxes: 82 TF/s -- ncu: L2
//     tag pipeline 73% busy (one request per 32-byte box row), tensor pipe
//     66% / 43% active in the two windows; 2 x 2 clusters with multicast loads
//     of the shared rows: 73 TF/s (the L2 already merges neighbouring CTAs'
//     requests; the cluster only adds lock-step);
//   boxed planes + bulk copies (this file): 99 TF/s; with the coalesced epilogue 100 TF/s
//     (3.6 int8 POP/s) and 33k -> 10k cycles of epilogue per block;
//   CTA pairs on top of that (cta_group::2, M = 256: each CTA holds half of the B rows,
//     CTA 1 relays "stage full" to CTA 0, commits multicast to both): 91 TF/s, config 2
//     factor 155 vs 139 ms, prediction sweep 383 vs 343 ms -- slower, dropped.
#include "ozaki.cuh"

#include <cmath>
#include <cstdlib>

namespace gpb {
namespace {

constexpr int kThreads = 192;

GPB_DEVINL uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

GPB_DEVINL void mbar_init(uint32_t bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
GPB_DEVINL void mbar_wait(uint32_t bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "OZ_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra OZ_WAIT;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
GPB_DEVINL void mbar_expect_tx(uint32_t bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
// contiguous global -> shared copy, bytes counted on the mbarrier
GPB_DEVINL void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
GPB_DEVINL void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
GPB_DEVINL void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
// arrives on the mbarrier once every tcgen05.mma issued so far by this thread has completed
GPB_DEVINL void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar)
               : "memory");
}
// D[tmem] (+)= A[smem desc] * B[smem desc]^T, int8 x int8 -> int32
GPB_DEVINL void tc_mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
GPB_DEVINL void tc_ld8(uint32_t taddr, int (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr)
               : "memory");
}
GPB_DEVINL void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

// K-major operand box, 32-byte rows, SWIZZLE_32B (8-row atoms of 256 bytes):
// start address >> 4 | LBO 1 | SBO 256 >> 4 | descriptor version 1 | layout type 6
GPB_DEVINL uint64_t smem_desc32(uint32_t addr) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFFu) | (1ull << 16) | (16ull << 32) | (1ull << 46) | (6ull << 61);
}
// byte offset of (row, byte) inside a box: SWIZZLE_32B exchanges the two 16-byte
// halves of rows 4..7 of every 8-row atom (address bit 4 ^= bit 7)
GPB_DEVINL int box_offset(int row, int byte) {
  const int o = row * kOzakiBK + byte;
  return o ^ (((o >> 7) & 1) << 4);
}

// as many stages as fit in ~200 KB (a stage: P planes of both operands, 8 KB per plane):
// 3 for the 8-plane window, 6 for the 4-plane one -- its chunks hold only 10 MMAs (640
// cycles), and 4 stages did not cover the L2-miss latency (tensor pipe 66% active)
__host__ __device__ constexpr int stages_for(int P) { return 25 / P > 8 ? 8 : 25 / P; }
// epilogue staging in the stage memory: 128 rows of 64 doubles, pitch 65 (conflict-free row-per-lane stores)
constexpr int kEpiPitch = 65;
constexpr size_t kEpiBytes = size_t(kOzakiBM) * kEpiPitch * sizeof(double);
constexpr size_t smem_bytes(int P) {
  return (size_t(stages_for(P)) * P * 2 * kOzakiBox > kEpiBytes ? size_t(stages_for(P)) * P * 2 * kOzakiBox : kEpiBytes) +
         1024 + 256;
}

struct OperandArgs {
  const int8_t* planes;
  long long tile_stride, rb_stride, chunk_stride;
  int chunks_per_tile;
};

struct OzakiArgs {
  OperandArgs a, b;
  long long a_off, b_off;
  int kchunks, mtiles, blocks_per_job, plane_bytes;  // plane_bytes: slices * 4096, a chunk's boxes
  const OzakiJob* jobs;
  double alpha, beta;
  const double* Cin;
  double* Cout;
  long long ldc_in, ldc_out;
};

template <int G0, int NG>
__global__ void __launch_bounds__(kThreads, 1) ozaki_gemm_kernel(const OzakiArgs p) {
  constexpr int P = G0 + NG;  // planes of each operand the groups [G0, P) need
  constexpr int NST = stages_for(P);
  constexpr int kOperandBytes = P * kOzakiBox;
  constexpr int kStageBytes = 2 * kOperandBytes;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (su32(smem_raw) + 1023u) & ~1023u;
  // full[NST], empty[NST], accfull, tmem slot: behind the stages (and the epilogue's staging tile)
  const uint32_t bars = base + (NST * kStageBytes > static_cast<int>(kEpiBytes) ? NST * kStageBytes : static_cast<int>(kEpiBytes));
  const uint32_t full0 = bars, empty0 = bars + 8 * NST, accfull = bars + 16 * NST, slot = accfull + 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int r = blockIdx.x, job = 0;
  if (p.jobs) {  // grouped: blocks_per_job consecutive CTAs per job
    job = blockIdx.x / p.blocks_per_job;
    r = blockIdx.x - job * p.blocks_per_job;
  }
  const int mt = r % p.mtiles, nt = r / p.mtiles;
  long long a_off = p.a_off, b_off = p.b_off;
  const double* Cin = p.Cin;
  double* Cout = p.Cout;
  int kchunks = p.kchunks;
  if (p.jobs) {
    const OzakiJob j = p.jobs[job];
    if (j.lower && nt > mt) return;
    a_off += j.a_off;
    b_off += j.b_off;
    Cout = j.C;
    Cin = p.beta != 0.0 ? j.C : nullptr;
    if (j.kchunks > 0) kchunks = j.kchunks;
  }

  if (warp == 1 && lane == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    mbar_init(accfull, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(slot) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tmem;
  asm volatile("ld.shared.u32 %0, [%1];\n" : "=r"(tmem) : "r"(slot) : "memory");

  if (warp == 0) {
    if (lane == 0) {
      const int8_t* asrc = p.a.planes + a_off + mt * p.a.rb_stride;
      const int8_t* bsrc = p.b.planes + b_off + nt * p.b.rb_stride;
      int st = 0, ph = 0, ac = 0, bc = 0;  // chunk inside the current tile of A / B
      for (int c = 0; c < kchunks; ++c) {
        mbar_wait(empty0 + 8 * st, ph ^ 1);
        const uint32_t fb = full0 + 8 * st;
        mbar_expect_tx(fb, kStageBytes);
        const uint32_t sa = base + st * kStageBytes;
        bulk_load(sa, asrc + static_cast<long long>(ac) * p.a.chunk_stride, kOperandBytes, fb);
        bulk_load(sa + kOperandBytes, bsrc + static_cast<long long>(bc) * p.b.chunk_stride, kOperandBytes, fb);
        if (++ac == p.a.chunks_per_tile) ac = 0, asrc += p.a.tile_stride;
        if (++bc == p.b.chunks_per_tile) bc = 0, bsrc += p.b.tile_stride;
        if (++st == NST) st = 0, ph ^= 1;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // s32 accumulate, signed 8-bit A and B, both K-major, N = 128, M = 128
      constexpr uint32_t idesc =
          (2u << 4) | (1u << 7) | (1u << 10) | ((kOzakiBN >> 3) << 17) | ((kOzakiBM >> 4) << 24);
      int st = 0, ph = 0;
      for (int c = 0; c < kchunks; ++c) {
        mbar_wait(full0 + 8 * st, ph);
        tc_fence_after();
        const uint32_t sa = base + st * kStageBytes, sb = sa + kOperandBytes;
#pragma unroll
        for (int g = G0; g < P; ++g) {
#pragma unroll
          for (int q = 0; q <= g; ++q)
            tc_mma_i8(tmem + (g - G0) * kOzakiBN, smem_desc32(sa + q * kOzakiBox),
                      smem_desc32(sb + (g - q) * kOzakiBox), idesc, (c | q) != 0);
        }
        tc_commit(empty0 + 8 * st);
        if (++st == NST) st = 0, ph ^= 1;
      }
      tc_commit(accfull);
    }
  } else {
    // Epilogue.  A thread owns one accumulator row (TMEM lane), but rows of C are
    // ldc doubles apart: row-per-thread global accesses would be 32 scattered
    // 16-byte pieces per instruction and one exposed memory latency per 8 columns
    // (ncu: 33k of a K = 512 block's 60k cycles).  So the warp first pulls its 32
    // rows of C towards L2 while the MMAs run, then, per half of the columns,
    // combines the groups into the (by then free) stage memory and updates C
    // from there with whole-row coalesced accesses, 16 rows in flight.
    const int quarter = warp & 3;
    const int row0 = mt * kOzakiBM + quarter * 32;  // first of the warp's rows of the job's C
    double* cout = Cout + static_cast<long long>(row0) * p.ldc_out + static_cast<long long>(nt) * kOzakiBN;
    const double* cin = Cin ? Cin + static_cast<long long>(row0) * p.ldc_in + static_cast<long long>(nt) * kOzakiBN
                            : nullptr;
    if (cin) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {  // 32 rows x 8 lines of 128 bytes
        const int line = i * 32 + lane;
        asm volatile("prefetch.global.L2 [%0];\n" ::"l"(cin + static_cast<long long>(line >> 3) * p.ldc_in +
                                                          (line & 7) * 16));
      }
    }
    mbar_wait(accfull, 0);
    tc_fence_after();
    const uint32_t taddr = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
    double* tile = reinterpret_cast<double*>(smem_raw + (base - su32(smem_raw))) + quarter * 32 * kEpiPitch;
#pragma unroll 1
    for (int half = 0; half < 2; ++half) {
      double* mine = tile + lane * kEpiPitch;
#pragma unroll 1
      for (int c8 = 0; c8 < 64; c8 += 8) {
        int v[NG][8];
#pragma unroll
        for (int g = 0; g < NG; ++g) tc_ld8(taddr + g * kOzakiBN + half * 64 + c8, v[g]);
        tc_wait_ld();
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          double acc = static_cast<double>(v[NG - 1][j]);
#pragma unroll
          for (int g = NG - 2; g >= 0; --g) acc = fma(acc, 0.0078125, static_cast<double>(v[g][j]));
          mine[c8 + j] = p.alpha * acc;
        }
      }
      __syncwarp();
#pragma unroll 1
      for (int r0 = 0; r0 < 32; r0 += 16) {
        double x0[16], x1[16];
        if (cin) {
#pragma unroll
          for (int r = 0; r < 16; ++r) {
            const double* src = cin + static_cast<long long>(r0 + r) * p.ldc_in + half * 64;
            x0[r] = src[lane];
            x1[r] = src[lane + 32];
          }
        }
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const double* t = tile + (r0 + r) * kEpiPitch;
          double* dst = cout + static_cast<long long>(r0 + r) * p.ldc_out + half * 64;
          dst[lane] = cin ? fma(p.beta, x0[r], t[lane]) : t[lane];
          dst[lane + 32] = cin ? fma(p.beta, x1[r], t[lane + 32]) : t[lane + 32];
        }
      }
      __syncwarp();
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
  }
}

// digits of f (|f| <= 127/128 in units of the scale): exact; the first digit lies in
// [-127, 127], the later ones in [-64, 64]
constexpr double kMaxFraction = 127.0 / 128.0;
template <int MAXS>
GPB_DEVINL void digits(double f, int slices, int (&d)[MAXS]) {
#pragma unroll
  for (int p = 0; p < MAXS; ++p) {
    if (p < slices) {
      f *= 128.0;
      const double r = rint(f);
      f -= r;
      d[p] = static_cast<int>(r);
    } else {
      d[p] = 0;
    }
  }
}

// One work item = 8 consecutive k of one row: item w of a box covers row w / 4,
// bytes 8 (w % 4) .., so a warp reads 8 rows x 256 B and writes 256 contiguous
// bytes per plane.
__global__ void __launch_bounds__(256)
    ozaki_slice_tiles_kernel(const double* __restrict__ src, long long items, int tr, int tc, double inv_scale,
                             int8_t* __restrict__ planes, int slices, int* flag) {
  const long long w = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (w >= items) return;
  const int in_box = static_cast<int>(w & 511), row = in_box >> 2, k8 = in_box & 3;
  const long long box = w >> 9;  // ((tile * (tr / 128) + rb) * (tc / 32) + kc)
  const int kcs = tc / kOzakiBK, rbs = tr / kOzakiBM;
  const int kc = static_cast<int>(box % kcs);
  const long long trb = box / kcs;
  const int rb = static_cast<int>(trb % rbs);
  const long long tile = trb / rbs;
  const double* s = src + tile * tr * tc + static_cast<long long>(rb * kOzakiBM + row) * tc + kc * kOzakiBK + k8 * 8;
  unsigned lo[kOzakiMaxSlices], hi[kOzakiMaxSlices];
#pragma unroll
  for (int p = 0; p < kOzakiMaxSlices; ++p) lo[p] = hi[p] = 0;
  bool over = false;
#pragma unroll
  for (int j = 0; j < 8; j += 2) {
    const double2 x = *reinterpret_cast<const double2*>(s + j);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double f = (h ? x.y : x.x) * inv_scale;
      if (!(fabs(f) <= kMaxFraction)) {
        over = true;
        f = f > 0.0 ? kMaxFraction : -kMaxFraction;
      }
      int d[kOzakiMaxSlices];
      digits(f, slices, d);
      const int jj = j + h;
#pragma unroll
      for (int p = 0; p < kOzakiMaxSlices; ++p) {
        const unsigned b = static_cast<unsigned>(d[p]) & 0xFFu;
        if (jj < 4) lo[p] |= b << (8 * jj);
        else hi[p] |= b << (8 * (jj - 4));
      }
    }
  }
  if (over) *flag = 1;
  int8_t* dst = planes + box * slices * kOzakiBox + box_offset(row, k8 * 8);
  for (int p = 0; p < slices; ++p) *reinterpret_cast<uint2*>(dst + p * kOzakiBox) = make_uint2(lo[p], hi[p]);
}

// 64 (k) x 64 (columns) block per CTA; thread (tx = column, ty) packs the
// digits of 4 consecutive k into one word per plane, staged in shared memory
// so that the stores run along the box rows (one 32-byte row per column)
__global__ void __launch_bounds__(256)
    ozaki_slice_t_kernel(const double* __restrict__ src, long long ld, double inv_scale, int8_t* __restrict__ planes,
                         long long rb_boxes, long long kc_boxes, long long k0, int slices, int* flag,
                         const OzakiSliceJob* __restrict__ jobs) {
  __shared__ unsigned stage[kOzakiMaxSlices][64][17];
  if (jobs) {  // batched: one job per blockIdx.z
    const OzakiSliceJob j = jobs[blockIdx.z];
    src = j.src;
    planes = j.planes;
    k0 = j.k0;
  }
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
  const long long c0 = static_cast<long long>(blockIdx.x) * 64;
  const long long kb = static_cast<long long>(blockIdx.y) * 64;
  bool over = false;
#pragma unroll
  for (int kg = ty; kg < 16; kg += 4) {
    unsigned w[kOzakiMaxSlices];
#pragma unroll
    for (int p = 0; p < kOzakiMaxSlices; ++p) w[p] = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double f = src[(kb + kg * 4 + j) * ld + c0 + tx] * inv_scale;
      if (!(fabs(f) <= kMaxFraction)) {
        over = true;
        f = f > 0.0 ? kMaxFraction : -kMaxFraction;
      }
      int d[kOzakiMaxSlices];
      digits(f, slices, d);
#pragma unroll
      for (int p = 0; p < kOzakiMaxSlices; ++p) w[p] |= (static_cast<unsigned>(d[p]) & 0xFFu) << (8 * j);
    }
#pragma unroll
    for (int p = 0; p < kOzakiMaxSlices; ++p) stage[p][tx][kg] = w[p];
  }
  if (over) *flag = 1;
  __syncthreads();
  // two k chunks of 32 bytes; per chunk and plane 64 box rows of 8 words: thread t
  // writes word t & 7 of rows t >> 3 and (t >> 3) + 32
  const int wi = threadIdx.x & 7, cr = threadIdx.x >> 3;
  const long long rb = c0 / kOzakiBM;
  const int row0 = static_cast<int>(c0 % kOzakiBM);
  for (int kc2 = 0; kc2 < 2; ++kc2) {
    int8_t* box = planes + (rb * rb_boxes + ((k0 + kb) / kOzakiBK + kc2) * kc_boxes) * slices * kOzakiBox;
    for (int p = 0; p < slices; ++p) {
#pragma unroll
      for (int c = cr; c < 64; c += 32)
        *reinterpret_cast<unsigned*>(box + p * kOzakiBox + box_offset(row0 + c, wi * 4)) = stage[p][c][kc2 * 8 + wi];
    }
  }
}

template <int G0, int NG>
cudaError_t launch_w(const OzakiArgs& a, int blocks, cudaStream_t st) {
  ozaki_gemm_kernel<G0, NG><<<blocks, kThreads, smem_bytes(G0 + NG), st>>>(a);
  return cudaGetLastError();
}

// groups [g0, g0 + ng)
cudaError_t launch_window(int g0, int ng, const OzakiArgs& a, int blocks, cudaStream_t st) {
  if (g0 == 0) {
    switch (ng) {
      case 1: return launch_w<0, 1>(a, blocks, st);
      case 2: return launch_w<0, 2>(a, blocks, st);
      case 3: return launch_w<0, 3>(a, blocks, st);
      case 4: return launch_w<0, 4>(a, blocks, st);
    }
  } else if (ng == 4) {
    switch (g0) {
      case 1: return launch_w<1, 4>(a, blocks, st);
      case 2: return launch_w<2, 4>(a, blocks, st);
      case 3: return launch_w<3, 4>(a, blocks, st);
      case 4: return launch_w<4, 4>(a, blocks, st);
    }
  }
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t ozaki_init_attributes() {
  cudaError_t e;
#define GPB_OZ_ATTR(G0, NG)                                                                                \
  if ((e = cudaFuncSetAttribute(ozaki_gemm_kernel<G0, NG>, cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                                static_cast<int>(smem_bytes(G0 + NG)))) != cudaSuccess)                   \
    return e;
  GPB_OZ_ATTR(0, 1) GPB_OZ_ATTR(0, 2) GPB_OZ_ATTR(0, 3) GPB_OZ_ATTR(0, 4)
  GPB_OZ_ATTR(1, 4) GPB_OZ_ATTR(2, 4) GPB_OZ_ATTR(3, 4) GPB_OZ_ATTR(4, 4)
#undef GPB_OZ_ATTR
  return cudaSuccess;
}

cudaError_t launch_ozaki_slice_tiles(const double* src, int64_t ntiles, int tr, int tc, double scale,
                                     int8_t* planes, int slices, int* flag, cudaStream_t st) {
  if (ntiles <= 0) return cudaSuccess;
  if (slices < 1 || slices > kOzakiMaxSlices || tr % kOzakiBM || tc % kOzakiBK) return cudaErrorInvalidValue;
  const long long items = static_cast<long long>(ntiles) * tr * tc / 8;
  ozaki_slice_tiles_kernel<<<static_cast<unsigned>((items + 255) / 256), 256, 0, st>>>(src, items, tr, tc, 1.0 / scale,
                                                                                     planes, slices, flag);
  return cudaGetLastError();
}

cudaError_t launch_ozaki_slice_t(const double* src, int64_t rows, int64_t cols, int64_t ld, double scale,
                                 int8_t* planes, int64_t rb_boxes, int64_t kc_boxes, int64_t k0, int slices,
                                 int* flag, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  if (slices < 1 || slices > kOzakiMaxSlices || (rows & 63) || (cols & 127) || (k0 & 63))
    return cudaErrorInvalidValue;
  dim3 grid(static_cast<unsigned>(cols / 64), static_cast<unsigned>(rows / 64));
  if (rows / 64 > 65535) return cudaErrorInvalidValue;
  ozaki_slice_t_kernel<<<grid, 256, 0, st>>>(src, ld, 1.0 / scale, planes, rb_boxes, kc_boxes, k0, slices, flag,
                                             nullptr);
  return cudaGetLastError();
}

cudaError_t launch_ozaki_slice_t_batch(const OzakiSliceJob* jobs, int njobs, int64_t rows, int64_t cols, int64_t ld,
                                       double scale, int64_t rb_boxes, int64_t kc_boxes, int slices, int* flag,
                                       cudaStream_t st) {
  if (njobs <= 0) return cudaSuccess;
  if (slices < 1 || slices > kOzakiMaxSlices || (rows & 63) || (cols & 127) || njobs > 65535 || rows / 64 > 65535)
    return cudaErrorInvalidValue;
  dim3 grid(static_cast<unsigned>(cols / 64), static_cast<unsigned>(rows / 64), static_cast<unsigned>(njobs));
  ozaki_slice_t_kernel<<<grid, 256, 0, st>>>(nullptr, ld, 1.0 / scale, nullptr, rb_boxes, kc_boxes, 0, slices, flag, jobs);
  return cudaGetLastError();
}

cudaError_t launch_ozaki_gemm(const OzakiGemm& g, cudaStream_t st) {
  if (g.M % kOzakiBM || g.N % kOzakiBN || g.K % kOzakiBK || g.K <= 0 || g.K > kOzakiMaxK || g.slices < 4 ||
      g.slices > kOzakiMaxSlices)
    return cudaErrorInvalidValue;
  if (g.jobs && g.njobs <= 0) return cudaErrorInvalidValue;
  OzakiArgs a;
  const long long boxes = static_cast<long long>(g.slices) * kOzakiBox;
  a.a = {g.a.planes, g.a.tile_stride, g.a.rb_stride, g.a.chunk_stride ? g.a.chunk_stride : boxes, g.a.chunks_per_tile};
  a.b = {g.b.planes, g.b.tile_stride, g.b.rb_stride, g.b.chunk_stride ? g.b.chunk_stride : boxes, g.b.chunks_per_tile};
  a.a_off = g.a_off;
  a.b_off = g.b_off;
  a.jobs = g.jobs;
  a.mtiles = g.M / kOzakiBM;
  a.blocks_per_job = a.mtiles * (g.N / kOzakiBN);
  a.kchunks = g.K / kOzakiBK;
  a.plane_bytes = g.slices * kOzakiBox;
  a.beta = g.beta;
  a.Cin = g.beta != 0.0 ? g.Cin : nullptr;
  a.Cout = g.Cout;
  a.ldc_in = g.ldc_in;
  a.ldc_out = g.ldc_out;
  const int blocks = a.blocks_per_job * (g.jobs ? g.njobs : 1);
  // the first group's weight is 2^-14; least significant groups first, then
  // groups [0, S - 4) on top of the result
  const double unit = g.alpha * (1.0 / 16384.0);
  const int g0 = g.slices - 4;
  a.alpha = std::ldexp(unit, -7 * g0);
  cudaError_t e = launch_window(g0, 4, a, blocks, st);
  if (e == cudaSuccess && g0 > 0) {
    a.alpha = unit;
    a.beta = 1.0;
    a.Cin = g.Cout;
    a.ldc_in = g.ldc_out;
    e = launch_window(0, g0, a, blocks, st);
  }
  return e;
}

}  // namespace gpb
