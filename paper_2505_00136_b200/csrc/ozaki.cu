// tcgen05 (kind::i8, TMEM accumulators) digit-plane product; see ozaki.cuh.
//
// Kernel shape.  One CTA per 128 x 64 output block, six warps:
//   warp 0   TMA producer: per 64-deep k chunk, the S digit planes of the A
//            rows (128 x 64 B each) and of the B rows (64 x 64 B each) into one
//            of two shared-memory stages (cp.async.bulk.tensor, SWIZZLE_64B)
//            behind a "full" mbarrier; it also owns the TMEM allocation;
//   warp 1   MMA issuer: one thread issues, per chunk, the S(S+1)/2 digit
//            pairs (p, q), p + q = g, as tcgen05.mma M=128 N=64 K=32 (two per
//            pair) into the int32 accumulator of group g -- S accumulators of
//            64 TMEM columns live side by side for the whole k loop, so every
//            plane box loaded once is used against up to S others (the reuse
//            that keeps L2 -> shared-memory traffic at 1/4 of a plain int8
//            GEMM's with this block shape); tcgen05.commit frees the stage;
//   warps 2-5 epilogue: after the last commit each thread owns one output row
//            (TMEM lane), reads its 64 columns of every group with tcgen05.ld,
//            combines the groups in FP64 (Horner in 2^-7, least significant
//            group first) and writes Cout = beta Cin + alpha sum.
#include "ozaki.cuh"

#include <cudaTypedefs.h>

#include <cmath>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

namespace gpb {
namespace {

constexpr int kABox = kOzakiBM * kOzakiBK;  // 8 KB
constexpr int kBBox = kOzakiBN * kOzakiBK;  // 4 KB
constexpr int kStages = 2;
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
GPB_DEVINL void tma_load(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
// the same box written at the same shared-memory offset of every CTA in cta_mask, each
// destination's own mbarrier (same offset) receiving the bytes
GPB_DEVINL void tma_load_mc(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1, uint16_t cta_mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], "
      "[%1, {%2, %3}], [%4], %5;\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar), "h"(cta_mask)
      : "memory");
}
GPB_DEVINL void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
GPB_DEVINL uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
GPB_DEVINL void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
GPB_DEVINL void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
// arrives on the mbarrier once every tcgen05.mma issued so far by this thread has completed
GPB_DEVINL void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar)
               : "memory");
}
// ... arriving on the mbarrier at the same offset of every CTA in cta_mask
GPB_DEVINL void tc_commit_mc(uint32_t bar, uint16_t cta_mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(bar),
      "h"(cta_mask)
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

// K-major operand box, 64-byte rows, SWIZZLE_64B (8-row atoms of 512 bytes):
// start address >> 4 | LBO 1 | SBO 512 >> 4 | descriptor version 1 | layout type 4
GPB_DEVINL uint64_t smem_desc(uint32_t addr) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFFu) | (1ull << 16) | (32ull << 32) | (1ull << 46) | (4ull << 61);
}

struct OzakiArgs {
  int a_row0, a_rows, a_ktile, a_kt_rows;
  int b_row0, b_rows, b_col0, b_ktile, b_kt_rows;
  int kchunks, mtiles, blocks_per_job;
  const OzakiJob* jobs;
  double alpha, beta;
  const double* Cin;
  double* Cout;
  long long ldc_in, ldc_out;
};

template <int S>
__global__ void __launch_bounds__(kThreads, 1)
    ozaki_gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                      const OzakiArgs p) {
  extern __shared__ uint8_t smem_raw[];
  constexpr int kStageBytes = S * (kABox + kBBox);
  const uint32_t base = (su32(smem_raw) + 1023u) & ~1023u;
  const uint32_t bars = base + kStages * kStageBytes;  // full[2], empty[2], accfull, tmem slot
  const uint32_t full0 = bars, empty0 = bars + 16, accfull = bars + 32, slot = bars + 40;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int mt = blockIdx.x % p.mtiles, nt = blockIdx.x / p.mtiles;
  int a_row0 = p.a_row0, b_row0 = p.b_row0;
  const double* Cin = p.Cin;
  double* Cout = p.Cout;
  if (p.jobs) {  // grouped: blocks_per_job consecutive CTAs per job
    const int job = blockIdx.x / p.blocks_per_job, r = blockIdx.x - job * p.blocks_per_job;
    mt = r % p.mtiles;
    nt = r / p.mtiles;
    const OzakiJob j = p.jobs[job];
    if (j.lower && nt * kOzakiBN >= (mt + 1) * kOzakiBM) return;
    a_row0 = j.a_row0;
    b_row0 = j.b_row0;
    Cin = Cout = j.C;
  }

  if (warp == 1 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
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
      for (int c = 0; c < p.kchunks; ++c) {
        const int st = c & 1;
        mbar_wait(empty0 + 8 * st, ((c >> 1) & 1) ^ 1);
        const uint32_t fb = full0 + 8 * st;
        mbar_expect_tx(fb, kStageBytes);
        const int kb = c * kOzakiBK;
        const int ax = kb % p.a_ktile;
        const int ay = a_row0 + mt * kOzakiBM + (kb / p.a_ktile) * p.a_kt_rows;
        const uint32_t sa = base + st * kStageBytes;
#pragma unroll
        for (int q = 0; q < S; ++q) tma_load(sa + q * kABox, &map_a, fb, ax, ay + q * p.a_rows);
        const uint32_t sb = sa + S * kABox;
        const int bx = p.b_col0 + (p.b_ktile ? kb % p.b_ktile : kb);
        const int by = b_row0 + nt * kOzakiBN + (p.b_ktile ? (kb / p.b_ktile) * p.b_kt_rows : 0);
#pragma unroll
        for (int q = 0; q < S; ++q) tma_load(sb + q * kBBox, &map_b, fb, bx, by + q * p.b_rows);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // s32 accumulate, signed 8-bit A and B, both K-major, N = 64, M = 128
      constexpr uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((kOzakiBN >> 3) << 17) | ((kOzakiBM >> 4) << 24);
      for (int c = 0; c < p.kchunks; ++c) {
        const int st = c & 1;
        mbar_wait(full0 + 8 * st, (c >> 1) & 1);
        tc_fence_after();
        const uint32_t sa = base + st * kStageBytes, sb = sa + S * kABox;
#pragma unroll
        for (int g = 0; g < S; ++g) {
#pragma unroll
          for (int q = 0; q <= g; ++q) {
            const uint64_t ad = smem_desc(sa + q * kABox), bd = smem_desc(sb + (g - q) * kBBox);
#pragma unroll
            for (int kk = 0; kk < kOzakiBK / 32; ++kk)
              tc_mma_i8(tmem + g * kOzakiBN, ad + 2 * kk, bd + 2 * kk, idesc, (c | q | kk) != 0);
          }
        }
        tc_commit(empty0 + 8 * st);
      }
      tc_commit(accfull);
    }
  } else {
    const int quarter = warp & 3;
    const int row = mt * kOzakiBM + quarter * 32 + lane;  // row of the job's C
    mbar_wait(accfull, 0);
    tc_fence_after();
    const uint32_t taddr = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
    double* out = Cout + static_cast<long long>(row) * p.ldc_out + static_cast<long long>(nt) * kOzakiBN;
    const double* in = Cin ? Cin + static_cast<long long>(row) * p.ldc_in + static_cast<long long>(nt) * kOzakiBN
                           : nullptr;
#pragma unroll 1
    for (int c8 = 0; c8 < kOzakiBN; c8 += 8) {
      int v[S][8];
#pragma unroll
      for (int g = 0; g < S; ++g) tc_ld8(taddr + g * kOzakiBN + c8, v[g]);
      tc_wait_ld();
      double r[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        double acc = static_cast<double>(v[S - 1][j]);
#pragma unroll
        for (int g = S - 2; g >= 0; --g) acc = fma(acc, 0.0078125, static_cast<double>(v[g][j]));
        r[j] = p.alpha * acc;
      }
      if (in) {
#pragma unroll
        for (int j = 0; j < 8; j += 2) {
          const double2 ci = *reinterpret_cast<const double2*>(in + c8 + j);
          r[j] = fma(p.beta, ci.x, r[j]);
          r[j + 1] = fma(p.beta, ci.y, r[j + 1]);
        }
      }
#pragma unroll
      for (int j = 0; j < 8; j += 2) *reinterpret_cast<double2*>(out + c8 + j) = make_double2(r[j], r[j + 1]);
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
  }
}


// ---- second kernel shape: 128 x 128 blocks, a window of digit groups per launch --
// One tcgen05.mma of 128 x 64 x 32 reads 4 KB of A and 2 KB of B from shared
// memory for 32 cycles of tensor work: 192 B/cycle, above what shared memory
// delivers, so the 128 x 64 kernel above is operand-fetch bound (59% of the
// int8 issue rate).  With N = 128 an MMA reads 8 KB for 64 cycles.  TMEM then
// holds 4 accumulators of 128 columns, so the groups are computed in two
// launches of up to four groups each, least significant first: launch one
// loads all the planes and adds groups [G0, G0 + 4) to C, launch two loads
// planes 0 .. 3 only and adds groups [0, G0).  K is walked in 32-byte chunks
// (SWIZZLE_32B boxes of 128 rows) through a ring of 3-4 stages.
constexpr int kBN2 = 128, kBK2 = 32;
constexpr int kBox2 = 128 * kBK2;  // 4 KB per plane box, A and B alike

// K-major operand box, 32-byte rows, SWIZZLE_32B (8-row atoms of 256 bytes)
GPB_DEVINL uint64_t smem_desc32(uint32_t addr) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFFu) | (1ull << 16) | (16ull << 32) | (1ull << 46) | (6ull << 61);
}

__host__ __device__ constexpr int stages2(int P) { return P >= 7 ? 3 : 4; }
constexpr size_t smem_bytes2(int P) { return size_t(stages2(P)) * P * 2 * kBox2 + 1024 + 128; }

//
// MC: clusters of 2 x 2 blocks.  The products are bound by L2 -> shared-memory
// traffic (ncu: L2 throughput 73%, tensor pipe 66% / 43% active in the two
// windows), and the four blocks of a cluster share their A rows pairwise along
// n and their B rows pairwise along m: every CTA loads half of its A planes and
// half of its B planes and multicasts each box to the neighbour that needs it
// too, which halves the traffic.  A stage of a CTA is written by itself and its
// two neighbours, so its `empty` barrier collects the tcgen05.commit of all
// three (each CTA commits to itself and to both neighbours).
template <int G0, int NG, bool MC>
__global__ void __launch_bounds__(kThreads, 1)
    ozaki_gemm2_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                       const OzakiArgs p) {
  constexpr int P = G0 + NG;  // planes of each operand the groups [G0, P) need
  constexpr int NST = stages2(P);
  constexpr int kStageBytes = P * 2 * kBox2;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (su32(smem_raw) + 1023u) & ~1023u;
  const uint32_t bars = base + NST * kStageBytes;  // full[NST], empty[NST], accfull, tmem slot
  const uint32_t full0 = bars, empty0 = bars + 8 * NST, accfull = bars + 16 * NST, slot = accfull + 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int mt, nt, job = 0;
  uint32_t rank = 0;
  if (MC) {  // 4 consecutive CTAs = one 2 x 2 region of blocks; regions walk m first
    rank = cluster_rank();
    const int region = blockIdx.x >> 2, per_job = p.blocks_per_job >> 2, rm = p.mtiles >> 1;
    int r = region;
    if (p.jobs) {
      job = region / per_job;
      r = region - job * per_job;
    }
    mt = 2 * (r % rm) + (rank & 1);
    nt = 2 * (r / rm) + (rank >> 1);
  } else {
    int r = blockIdx.x;
    if (p.jobs) {  // grouped: blocks_per_job consecutive CTAs per job
      job = blockIdx.x / p.blocks_per_job;
      r = blockIdx.x - job * p.blocks_per_job;
    }
    mt = r % p.mtiles;
    nt = r / p.mtiles;
  }
  int a_row0 = p.a_row0, b_row0 = p.b_row0;
  const double* Cin = p.Cin;
  double* Cout = p.Cout;
  if (p.jobs) {
    const OzakiJob j = p.jobs[job];
    // lower jobs skip what lies above the diagonal: blocks, or whole regions (the
    // one upper block of a diagonal region is computed; it is never read)
    if (j.lower && (MC ? (nt >> 1) > (mt >> 1) : nt > mt)) return;
    a_row0 = j.a_row0;
    b_row0 = j.b_row0;
    Cin = Cout = j.C;
  }

  if (warp == 1 && lane == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, MC ? 3 : 1);
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
  if (MC) cluster_sync_all();  // every CTA's barriers exist before a neighbour signals them
  uint32_t tmem;
  asm volatile("ld.shared.u32 %0, [%1];\n" : "=r"(tmem) : "r"(slot) : "memory");
  // neighbours: rank ^ 2 shares the A rows (same mt), rank ^ 1 the B rows (same nt)
  const uint16_t mask_a = static_cast<uint16_t>((1u << rank) | (1u << (rank ^ 2)));
  const uint16_t mask_b = static_cast<uint16_t>((1u << rank) | (1u << (rank ^ 1)));

  if (warp == 0) {
    if (lane == 0) {
      int st = 0, ph = 0;
      // this CTA's share of the planes: the first half of A when it is the left block of
      // its pair, the first half of B when it is the upper one
      const int qa0 = MC ? ((rank >> 1) ? P / 2 : 0) : 0, qa1 = MC ? ((rank >> 1) ? P : P / 2) : P;
      const int qb0 = MC ? ((rank & 1) ? P / 2 : 0) : 0, qb1 = MC ? ((rank & 1) ? P : P / 2) : P;
      for (int c = 0; c < p.kchunks; ++c) {
        mbar_wait(empty0 + 8 * st, ph ^ 1);
        const uint32_t fb = full0 + 8 * st;
        mbar_expect_tx(fb, kStageBytes);
        const int kb = c * kBK2;
        const int ax = kb % p.a_ktile;
        const int ay = a_row0 + mt * kOzakiBM + (kb / p.a_ktile) * p.a_kt_rows;
        const uint32_t sa = base + st * kStageBytes;
        const uint32_t sb = sa + P * kBox2;
        const int bx = p.b_col0 + (p.b_ktile ? kb % p.b_ktile : kb);
        const int by = b_row0 + nt * kBN2 + (p.b_ktile ? (kb / p.b_ktile) * p.b_kt_rows : 0);
        if (MC) {
          for (int q = qa0; q < qa1; ++q) tma_load_mc(sa + q * kBox2, &map_a, fb, ax, ay + q * p.a_rows, mask_a);
          for (int q = qb0; q < qb1; ++q) tma_load_mc(sb + q * kBox2, &map_b, fb, bx, by + q * p.b_rows, mask_b);
        } else {
#pragma unroll
          for (int q = 0; q < P; ++q) tma_load(sa + q * kBox2, &map_a, fb, ax, ay + q * p.a_rows);
#pragma unroll
          for (int q = 0; q < P; ++q) tma_load(sb + q * kBox2, &map_b, fb, bx, by + q * p.b_rows);
        }
        if (++st == NST) st = 0, ph ^= 1;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // s32 accumulate, signed 8-bit A and B, both K-major, N = 128, M = 128
      constexpr uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((kBN2 >> 3) << 17) | ((kOzakiBM >> 4) << 24);
      int st = 0, ph = 0;
      for (int c = 0; c < p.kchunks; ++c) {
        mbar_wait(full0 + 8 * st, ph);
        tc_fence_after();
        const uint32_t sa = base + st * kStageBytes, sb = sa + P * kBox2;
#pragma unroll
        for (int g = G0; g < P; ++g) {
#pragma unroll
          for (int q = 0; q <= g; ++q)
            tc_mma_i8(tmem + (g - G0) * kBN2, smem_desc32(sa + q * kBox2), smem_desc32(sb + (g - q) * kBox2), idesc,
                      (c | q) != 0);
        }
        if (MC) tc_commit_mc(empty0 + 8 * st, mask_a | mask_b);
        else tc_commit(empty0 + 8 * st);
        if (++st == NST) st = 0, ph ^= 1;
      }
      tc_commit(accfull);
    }
  } else {
    const int quarter = warp & 3;
    const int row = mt * kOzakiBM + quarter * 32 + lane;  // row of the job's C
    mbar_wait(accfull, 0);
    tc_fence_after();
    const uint32_t taddr = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
    double* out = Cout + static_cast<long long>(row) * p.ldc_out + static_cast<long long>(nt) * kBN2;
    const double* in = Cin ? Cin + static_cast<long long>(row) * p.ldc_in + static_cast<long long>(nt) * kBN2
                           : nullptr;
#pragma unroll 1
    for (int c8 = 0; c8 < kBN2; c8 += 8) {
      int v[NG][8];
#pragma unroll
      for (int g = 0; g < NG; ++g) tc_ld8(taddr + g * kBN2 + c8, v[g]);
      tc_wait_ld();
      double r[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        double acc = static_cast<double>(v[NG - 1][j]);
#pragma unroll
        for (int g = NG - 2; g >= 0; --g) acc = fma(acc, 0.0078125, static_cast<double>(v[g][j]));
        r[j] = p.alpha * acc;
      }
      if (in) {
#pragma unroll
        for (int j = 0; j < 8; j += 2) {
          const double2 ci = *reinterpret_cast<const double2*>(in + c8 + j);
          r[j] = fma(p.beta, ci.x, r[j]);
          r[j + 1] = fma(p.beta, ci.y, r[j + 1]);
        }
      }
#pragma unroll
      for (int j = 0; j < 8; j += 2) *reinterpret_cast<double2*>(out + c8 + j) = make_double2(r[j], r[j + 1]);
    }
    tc_fence_before();
  }
  __syncthreads();
  if (MC) cluster_sync_all();  // no neighbour commit may arrive after this CTA is gone
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
  }
}

// digits of f (|f| <= 1/2 in units of the scale): exact
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

__global__ void __launch_bounds__(256)
    ozaki_slice_kernel(const double* __restrict__ src, long long count, double inv_scale, int8_t* __restrict__ planes,
                       long long plane_stride, int slices, int* flag) {
  const long long e0 = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) * 8;
  if (e0 >= count) return;
  unsigned lo[kOzakiMaxSlices], hi[kOzakiMaxSlices];
#pragma unroll
  for (int p = 0; p < kOzakiMaxSlices; ++p) lo[p] = hi[p] = 0;
  bool over = false;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    double f = (e0 + j < count ? src[e0 + j] : 0.0) * inv_scale;
    if (!(fabs(f) <= 0.5)) {
      over = true;
      f = f > 0.0 ? 0.5 : -0.5;
    }
    int d[kOzakiMaxSlices];
    digits(f, slices, d);
#pragma unroll
    for (int p = 0; p < kOzakiMaxSlices; ++p) {
      const unsigned b = static_cast<unsigned>(d[p]) & 0xFFu;
      if (j < 4) lo[p] |= b << (8 * j);
      else hi[p] |= b << (8 * (j - 4));
    }
  }
  if (over) *flag = 1;
  for (int p = 0; p < slices; ++p)
    *reinterpret_cast<uint2*>(planes + p * plane_stride + e0) = make_uint2(lo[p], hi[p]);
}

// 64 (k) x 64 (columns) block per CTA; thread (tx = column, ty) packs the
// digits of 4 consecutive k into one word per plane, staged in shared memory
// so that the stores run along k
__global__ void __launch_bounds__(256)
    ozaki_slice_t_kernel(const double* __restrict__ src, long long ld, double inv_scale, int8_t* __restrict__ planes,
                         long long plane_stride, long long out_ld, long long k0, int slices, int* flag) {
  __shared__ unsigned stage[kOzakiMaxSlices][64][17];
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
  const long long c0 = static_cast<long long>(blockIdx.x) * 64;
  const int kb = blockIdx.y * 64;
  bool over = false;
#pragma unroll
  for (int kg = ty; kg < 16; kg += 4) {
    unsigned w[kOzakiMaxSlices];
#pragma unroll
    for (int p = 0; p < kOzakiMaxSlices; ++p) w[p] = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double f = src[(kb + kg * 4 + j) * ld + c0 + tx] * inv_scale;
      if (!(fabs(f) <= 0.5)) {
        over = true;
        f = f > 0.0 ? 0.5 : -0.5;
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
  // 16 words per column row: thread t writes word t & 15 of columns t >> 4, + 16, ...
  const int wi = threadIdx.x & 15, cr = threadIdx.x >> 4;
  for (int p = 0; p < slices; ++p) {
#pragma unroll
    for (int c = cr; c < 64; c += 16) {
      unsigned* dst = reinterpret_cast<unsigned*>(planes + p * plane_stride + (c0 + c) * out_ld + k0 + kb);
      dst[wi] = stage[p][c][wi];
    }
  }
}

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
  int64_t pitch, rows;
  int box_rows, box_cols;
  bool operator==(const MapKey& o) const {
    return base == o.base && pitch == o.pitch && rows == o.rows && box_rows == o.box_rows &&
           box_cols == o.box_cols;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    size_t h = reinterpret_cast<size_t>(k.base);
    h = h * 1000003u ^ static_cast<size_t>(k.pitch);
    h = h * 1000003u ^ static_cast<size_t>(k.rows);
    return h * 1000003u ^ static_cast<size_t>(k.box_rows * 131 + k.box_cols);
  }
};

// byte view (pitch bytes per row, `rows` rows), boxes of box_cols (64 or 32) bytes x box_rows,
// swizzled over the box width
bool byte_map(const int8_t* base, int64_t pitch, int64_t rows, int box_rows, int box_cols, CUtensorMap* out) {
  static std::mutex mu;
  static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
  const MapKey key{base, pitch, rows, box_rows, box_cols};
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return true;
  }
  auto fn = encode_fn();
  if (!fn) return false;
  CUtensorMap m;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(pitch), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(pitch)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  if (fn(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(base), dims, strides, box, estr,
         CU_TENSOR_MAP_INTERLEAVE_NONE, box_cols == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_64B,
         CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  if (cache.size() > 1024) cache.clear();
  cache.emplace(key, m);
  *out = m;
  return true;
}

size_t smem_bytes(int S) { return size_t(kStages) * S * (kABox + kBBox) + 1024 + 64; }

template <int S>
cudaError_t launch_s(const CUtensorMap& ma, const CUtensorMap& mb, const OzakiArgs& a, int blocks, cudaStream_t st) {
  ozaki_gemm_kernel<S><<<blocks, kThreads, smem_bytes(S), st>>>(ma, mb, a);
  return cudaGetLastError();
}

template <int G0, int NG>
cudaError_t launch_w(const CUtensorMap& ma, const CUtensorMap& mb, const OzakiArgs& a, int blocks, bool mc,
                     cudaStream_t st) {
  if (!mc) {
    ozaki_gemm2_kernel<G0, NG, false><<<blocks, kThreads, smem_bytes2(G0 + NG), st>>>(ma, mb, a);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(blocks));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem_bytes2(G0 + NG);
  cfg.stream = st;
  cudaLaunchAttribute attr{};
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = 4;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, ozaki_gemm2_kernel<G0, NG, true>, ma, mb, a);
}

// groups [g0, g0 + ng) of the 128 x 128 kernel; mc: 2 x 2 clusters with multicast loads
cudaError_t launch_window(int g0, int ng, const CUtensorMap& ma, const CUtensorMap& mb, const OzakiArgs& a,
                          int blocks, bool mc, cudaStream_t st) {
  if (g0 == 0) {
    switch (ng) {
      case 1: return launch_w<0, 1>(ma, mb, a, blocks, mc, st);
      case 2: return launch_w<0, 2>(ma, mb, a, blocks, mc, st);
      case 3: return launch_w<0, 3>(ma, mb, a, blocks, mc, st);
      case 4: return launch_w<0, 4>(ma, mb, a, blocks, mc, st);
    }
  } else if (ng == 4) {
    switch (g0) {
      case 1: return launch_w<1, 4>(ma, mb, a, blocks, mc, st);
      case 2: return launch_w<2, 4>(ma, mb, a, blocks, mc, st);
      case 3: return launch_w<3, 4>(ma, mb, a, blocks, mc, st);
      case 4: return launch_w<4, 4>(ma, mb, a, blocks, mc, st);
    }
  }
  return cudaErrorInvalidValue;
}

// GPB_OZAKI_CLUSTER=0: no clusters (every CTA loads all of its planes)
bool use_clusters() {
  static const bool v = [] {
    const char* e = getenv("GPB_OZAKI_CLUSTER");
    return e ? atoi(e) != 0 : true;
  }();
  return v;
}

// GPB_OZAKI_KERNEL=1: the 128 x 64 single-launch kernel for every product
int kernel_shape() {
  static const int v = [] {
    const char* e = getenv("GPB_OZAKI_KERNEL");
    return e ? atoi(e) : 2;
  }();
  return v;
}

}  // namespace

cudaError_t ozaki_init_attributes() {
  cudaError_t e;
#define GPB_OZ_ATTR2(G0, NG)                                                                                    \
  if ((e = cudaFuncSetAttribute(ozaki_gemm2_kernel<G0, NG, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                static_cast<int>(smem_bytes2(G0 + NG)))) != cudaSuccess)                       \
    return e;                                                                                                   \
  if ((e = cudaFuncSetAttribute(ozaki_gemm2_kernel<G0, NG, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                                static_cast<int>(smem_bytes2(G0 + NG)))) != cudaSuccess)                       \
    return e;
  GPB_OZ_ATTR2(0, 1) GPB_OZ_ATTR2(0, 2) GPB_OZ_ATTR2(0, 3) GPB_OZ_ATTR2(0, 4)
  GPB_OZ_ATTR2(1, 4) GPB_OZ_ATTR2(2, 4) GPB_OZ_ATTR2(3, 4) GPB_OZ_ATTR2(4, 4)
#undef GPB_OZ_ATTR2
#define GPB_OZ_ATTR(S)                                                                              \
  if ((e = cudaFuncSetAttribute(ozaki_gemm_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                static_cast<int>(smem_bytes(S)))) != cudaSuccess)                  \
    return e;
  GPB_OZ_ATTR(4) GPB_OZ_ATTR(5) GPB_OZ_ATTR(6) GPB_OZ_ATTR(7) GPB_OZ_ATTR(8)
#undef GPB_OZ_ATTR
  return cudaSuccess;
}

cudaError_t launch_ozaki_slice(const double* src, int64_t count, double scale, int8_t* planes,
                               int64_t plane_stride, int slices, int* flag, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  if (slices < 1 || slices > kOzakiMaxSlices || (count & 7) || (plane_stride & 7)) return cudaErrorInvalidValue;
  const int64_t threads = (count + 7) / 8;
  ozaki_slice_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, st>>>(src, count, 1.0 / scale, planes,
                                                                                  plane_stride, slices, flag);
  return cudaGetLastError();
}

cudaError_t launch_ozaki_slice_t(const double* src, int rows, int64_t cols, int64_t ld, double scale,
                                 int8_t* planes, int64_t plane_stride, int64_t out_ld, int64_t k0,
                                 int slices, int* flag, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  if (slices < 1 || slices > kOzakiMaxSlices || (rows & 63) || (cols & 63) || (out_ld & 3) || (k0 & 63))
    return cudaErrorInvalidValue;
  dim3 grid(static_cast<unsigned>(cols / 64), static_cast<unsigned>(rows / 64));
  ozaki_slice_t_kernel<<<grid, 256, 0, st>>>(src, ld, 1.0 / scale, planes, plane_stride, out_ld, k0, slices, flag);
  return cudaGetLastError();
}

cudaError_t launch_ozaki_gemm(const OzakiGemm& g, cudaStream_t st, bool* used) {
  *used = false;
  if (g.M % kOzakiBM || g.N % kOzakiBN || g.K % kOzakiBK || g.K <= 0 || g.K > kOzakiMaxK || g.slices < 4 ||
      g.slices > kOzakiMaxSlices)
    return cudaErrorInvalidValue;
  if (g.jobs && (g.njobs <= 0 || g.beta == 0.0)) return cudaErrorInvalidValue;
  const bool wide = kernel_shape() == 2 && g.N % kBN2 == 0;
  CUtensorMap ma, mb;
  if (!byte_map(g.a_planes, g.a_pitch, g.a_rows * g.slices, kOzakiBM, wide ? kBK2 : kOzakiBK, &ma) ||
      !byte_map(g.b_planes, g.b_pitch, g.b_rows * g.slices, wide ? kBN2 : kOzakiBN, wide ? kBK2 : kOzakiBK, &mb))
    return cudaSuccess;
  OzakiArgs a;
  a.a_row0 = static_cast<int>(g.a_row0);
  a.a_rows = static_cast<int>(g.a_rows);
  a.a_ktile = g.a_ktile;
  a.a_kt_rows = g.a_kt_rows;
  a.b_row0 = static_cast<int>(g.b_row0);
  a.b_rows = static_cast<int>(g.b_rows);
  a.b_col0 = static_cast<int>(g.b_col0);
  a.b_ktile = g.b_ktile;
  a.b_kt_rows = g.b_kt_rows;
  a.jobs = g.jobs;
  a.blocks_per_job = (g.M / kOzakiBM) * (g.N / kOzakiBN);
  a.kchunks = g.K / kOzakiBK;
  a.mtiles = g.M / kOzakiBM;
  a.alpha = g.alpha * (1.0 / 16384.0);  // the first group's weight 2^-14
  a.beta = g.beta;
  a.Cin = g.beta != 0.0 ? g.Cin : nullptr;
  a.Cout = g.Cout;
  a.ldc_in = g.ldc_in;
  a.ldc_out = g.ldc_out;
  if (wide) {
    // least significant groups first, then groups [0, S - 4) on top of the result
    a.blocks_per_job = (g.M / kOzakiBM) * (g.N / kBN2);
    a.kchunks = g.K / kBK2;
    const int blocks = a.blocks_per_job * (g.jobs ? g.njobs : 1);
    const int g0 = g.slices - 4;
    const double unit = a.alpha;
    const bool mc = use_clusters() && (g.M / kOzakiBM) % 2 == 0 && (g.N / kBN2) % 2 == 0;
    a.alpha = std::ldexp(unit, -7 * g0);
    cudaError_t e = launch_window(g0, 4, ma, mb, a, blocks, mc, st);
    if (e == cudaSuccess && g0 > 0) {
      a.alpha = unit;
      a.beta = 1.0;
      a.Cin = g.Cout;
      a.ldc_in = g.ldc_out;
      e = launch_window(0, g0, ma, mb, a, blocks, mc, st);
    }
    *used = e == cudaSuccess;
    return e;
  }
  const int blocks = (g.M / kOzakiBM) * (g.N / kOzakiBN) * (g.jobs ? g.njobs : 1);
  cudaError_t e = cudaSuccess;
  switch (g.slices) {
    case 4: e = launch_s<4>(ma, mb, a, blocks, st); break;
    case 5: e = launch_s<5>(ma, mb, a, blocks, st); break;
    case 6: e = launch_s<6>(ma, mb, a, blocks, st); break;
    case 7: e = launch_s<7>(ma, mb, a, blocks, st); break;
    default: e = launch_s<8>(ma, mb, a, blocks, st); break;
  }
  *used = e == cudaSuccess;
  return e;
}

}  // namespace gpb
