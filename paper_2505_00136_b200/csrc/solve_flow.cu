// One-launch dataflow triangular solves: beta = L^-1 y, alpha = L^-T beta.
//
// Replaces the 4T serial launches of the blocked vector solves (taskgp
// tiled.py:215-260: tiled_forward_solve / tiled_backward_solve over
// solve_lower_vec, solve_lower_t_vec, matvec_sub, matvec_t_sub, tiles.py:170-201)
// with ONE cooperative launch in which every CTA owns one slice of R rows of
// the padded system and the slices synchronise through per-block-row counters
// in global memory (acquire/release), not grid barriers:
//
// forward, slice s (block row i, rows [i*bi + q*R, +R)):
//   r    = y - sum_{j<i} L(i,j)[rows, :] beta_j        (j ascending; waits on beta_j)
//   publish r's slice; wait until all bi/R slices of block row i have
//   beta_i[rows] = Dinv_i[rows, :] r                   (Dinv_i = L_ii^-1, lower)
// backward, slice s' (block row i' = T-1-i, same R columns of it):
//   t    = beta - sum_{j>i'} L(j,i')[:, cols]^T alpha_j (j descending; waits on alpha_j)
//   publish t's slice; wait for the block row;
//   alpha_i'[cols] = Dinv_i'[:, cols]^T t
//
// Each CTA runs its forward slice, then the backward slice mirrored across the
// grid, so the CTAs that finish their forward rows first own the first
// backward block rows.  The lower factor is read exactly twice (once per
// solve), which is the HBM bound of this phase.  Every sum has a fixed order
// (per-lane column chunks, warp butterflies, warps in index order, tiles in j
// order), so results are bitwise reproducible.  All slices must be resident at
// once (cooperative launch); launch_solve_flow reports when they are not and
// the caller keeps the multi-launch path.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kernels.cuh"

namespace gpb {

namespace {

constexpr int FT = 128;  // threads per CTA (4 warps)
// bytes of factor tiles the active slices may hold in L2 through look-ahead
// prefetches at once (of 126 MB): only the late, latency-bound phase uses them
constexpr int64_t kL2Window = int64_t(48) << 20;
constexpr int FW = FT / 32;

GPB_DEVINL int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// thread 0 polls (relaxed loads: no L1 invalidation per poll), then one
// gpu-scope fence orders the CTA's later loads after the observed count
// (they read L2 through ld.cg, so no stale L1 lines are involved)
GPB_DEVINL void wait_count(const int* flag, int want, bool hot = false) {
  if (threadIdx.x == 0) {
    int ns = 32;
    while (ld_relaxed(flag) < want) {
      if (!hot) {
        __nanosleep(ns);
        ns = ns < 256 ? 2 * ns : 256;
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// bulk L2 prefetch of a contiguous range (16-byte multiple; thread 0 issues)
GPB_DEVINL void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}

// L2 prefetch of `rows` rows of `width` doubles at stride ld (one 128-byte line per
// thread per step: the column slices of the backward solve)
GPB_DEVINL void prefetch_rows(const double* p, int rows, int width, int64_t ld) {
  const int lines = (width * 8 + 127) / 128;
  for (int e = threadIdx.x; e < rows * lines; e += blockDim.x) {
    const char* a = reinterpret_cast<const char*>(p + static_cast<int64_t>(e / lines) * ld) + 128 * (e % lines);
    asm volatile("prefetch.global.L2 [%0];\n" ::"l"(a));
  }
}

// L1 prefetch of this warp's part of a slice (rows of `width` doubles at stride ld):
// the critical tile is read by one CTA per row slice with at most ~8 loads in
// flight per lane (register cap of the co-resident grid), so from L2 its dot
// costs ~8 us per block row; staged in L1 while the CTA waits for beta it is
// read at L1 latency (the bulk loads are evict-first and do not displace it)
GPB_DEVINL void prefetch_rows_l1(const double* p, int rows, int width, int64_t ld, int lane) {
  const int lines = (width * 8 + 127) / 128;
  for (int e = lane; e < rows * lines; e += 32) {
    const char* q = reinterpret_cast<const char*>(p + static_cast<int64_t>(e / lines) * ld) + 128 * (e % lines);
    asm volatile("prefetch.global.L1 [%0];\n" ::"l"(q));
  }
}

// publish this CTA's stores: every thread's writes are fenced before the count
GPB_DEVINL void signal_count(int* flag) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd(flag, 1);
}

struct FlowArgs {
  const double* L;     // packed row-major lower tiles
  const double* dinv;  // T inverse diagonal tiles
  const double* y;     // padded right-hand side (n_p)
  double* beta;        // n_p
  double* alpha;       // n_p
  double* xr;          // n_p exchange buffer (r of the forward, t of the backward)
  int* flags;          // 4T counters + T*S helper counters, zero on entry
  double* part;        // helper partials of the critical tiles: [2][T][4][bi] (forward, backward)
  int T, bi, R;
  unsigned long long* prof;  // optional: 4T globaltimer stamps (GPB_SOLVE_PROF)
  int pf;                    // steps ahead the critical tile is staged in L2 (GPB_FLOW_PREFETCH, default 2)
  int l1;                    // stage the critical tile slices in L1 (GPB_FLOW_L1, default 1)
  int help;                  // helper quarters of the critical tiles (GPB_FLOW_HELP, default 1)
};

GPB_DEVINL unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// 8 per-lane partial sums (rows 0..7 of a group) -> the total of row
// 4*b4 + 2*b3 + b2 (bits of the lane index) in every lane: three halving
// exchanges then two full butterflies -- 9 shuffles instead of 8 x 5, in a
// fixed order (IEEE addition is commutative, so partner lanes agree bitwise)
GPB_DEVINL double reduce8(const double (&p)[8], int lane) {
  const bool h4 = lane & 16, h3 = lane & 8, h2 = lane & 4;
  double q4[4], q2[2];
#pragma unroll
  for (int k = 0; k < 4; ++k)
    q4[k] = (h4 ? p[k + 4] : p[k]) + __shfl_xor_sync(0xffffffffu, h4 ? p[k] : p[k + 4], 16);
#pragma unroll
  for (int k = 0; k < 2; ++k)
    q2[k] = (h3 ? q4[k + 2] : q4[k]) + __shfl_xor_sync(0xffffffffu, h3 ? q4[k] : q4[k + 2], 8);
  double q = (h2 ? q2[1] : q2[0]) + __shfl_xor_sync(0xffffffffu, h2 ? q2[0] : q2[1], 4);
  q += __shfl_xor_sync(0xffffffffu, q, 2);
  q += __shfl_xor_sync(0xffffffffu, q, 1);
  return q;
}
GPB_DEVINL int reduce8_row(int lane) { return ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1); }

// p[k] += M[row k][lane's columns] . v  for the 8 rows of a group (row-major
// M, ld = bi); diag: M is lower triangular, only columns <= row are read
// kL1: the rows were staged in L1 (critical tile): plain cached loads; otherwise
// streaming (evict-first) loads.  All 8 loads of a chunk are issued before its
// FMAs (the compiler would otherwise interleave them and keep ~3 in flight).
template <bool kDiag, bool kL1 = false>
GPB_DEVINL void rows8_dot(const double* M, int bi, int row0, const double2* v, int nchunk, int lane,
                          double (&p)[8]) {
#pragma unroll 2
  for (int c = 0; c < nchunk; ++c) {
    const int col = 2 * (lane + 32 * c);
    if (kDiag && col > row0 + 7) continue;
    double2 x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double2* r = reinterpret_cast<const double2*>(M + static_cast<int64_t>(row0 + k) * bi) + lane + 32 * c;
      if (!kDiag || col <= row0 + k)
        x[k] = kL1 ? __ldca(r) : (kDiag ? __ldcg(r) : __ldcs(r));
      else
        x[k] = make_double2(0.0, 0.0);
    }
    asm volatile("" ::: "memory");
    const double2 vc = v[lane + 32 * c];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      p[k] = fma(x[k].x, vc.x, p[k]);
      p[k] = fma(x[k].y, vc.y, p[k]);  // upper entries of Dinv are zero
    }
  }
}

// forward slice: rows [q R, q R + R) of block row i; each warp owns R / FW
// rows in groups of 8 (lane l accumulates row 8g + reduce8_row(l) of group g)
template <int R>
__device__ void forward_slice(const FlowArgs& a, int i, int q, double2* vs) {
  const int bi = a.bi, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int RW = R / FW;  // rows per warp
  constexpr int G = RW / 8;   // groups of 8 rows
  static_assert(RW % 8 == 0, "rows per warp must be a multiple of 8");
  const int64_t bi2 = static_cast<int64_t>(bi) * bi;
  const int rbase = q * R + warp * RW;  // first row of this warp inside block row i
  const int nchunk = bi / 64;           // double2 chunks per lane per row
  int* r_done = a.flags;
  int* b_done = a.flags + a.T;
  const int S = bi / R;
  int* p_done = a.flags + 4 * a.T;  // [T][S]: helper quarters delivered for (block row, slice)
  const int QC = bi / 4;            // columns of a quarter of the critical tile
  double acc[G];
#pragma unroll
  for (int g = 0; g < G; ++g) acc[g] = 0.0;
  // Helpers: quarter h = 1..3 of the critical tile (i, i-1) of block row i (its
  // columns [h QC, (h+1) QC)) is computed by slice q of block row i + h, which
  // waits for beta_{i-1} anyway for its own tile (i + h, i - 1): the dot on the
  // critical path shrinks to a quarter, spread over four CTAs
  const int nhelp = a.help ? min(3, a.T - 1 - i) : 0;  // helpers row i gets
  double crit[G], tail[G];  // own quarter 0; own quarters nhelp+1..3 (no helper below the last rows)
#pragma unroll
  for (int g = 0; g < G; ++g) crit[g] = tail[g] = 0.0;
  for (int j = 0; j < i; ++j) {
    if (j == i - a.pf && threadIdx.x == 0)
      prefetch_l2(a.L + tri_rm(i, i - 1) * bi2 + static_cast<int64_t>(q) * R * bi, sizeof(double) * R * bi);
    if (j == i - 1 && threadIdx.x == 0) {
      // the critical path of the solve runs through this slice from here on:
      // stage its last tile and its rows of Dinv_i in L2 while beta_{i-1} is
      // being produced, so they do not queue behind the bulk streaming reads
      prefetch_l2(a.L + tri_rm(i, j) * bi2 + static_cast<int64_t>(q) * R * bi, sizeof(double) * R * bi);
      prefetch_l2(a.dinv + static_cast<int64_t>(i) * bi2 + static_cast<int64_t>(q) * R * bi,
                  sizeof(double) * R * bi);
    }
    else if (threadIdx.x == 0 && int64_t(a.T - 1 - j) * bi2 * 8 <= kL2Window)
      // late phase (few block rows left): stream this band through L2 ahead of
      // the loads, so the slice's rate is not bounded by its own load depth
      prefetch_l2(a.L + tri_rm(i, j) * bi2 + static_cast<int64_t>(q) * R * bi, sizeof(double) * R * bi);
    if (j == i - 1 && a.l1) {  // this warp's rows of the critical tile and of Dinv_i into L1
      prefetch_rows_l1(a.L + tri_rm(i, j) * bi2 + static_cast<int64_t>(rbase) * bi, RW, bi, bi, lane);
      prefetch_rows_l1(a.dinv + static_cast<int64_t>(i) * bi2 + static_cast<int64_t>(rbase) * bi, RW, bi, bi, lane);
    }
    wait_count(b_done + j, S, j == i - 1);  // (its __syncthreads also retires the previous vs)
    if (a.prof && j == i - 1 && q == 0 && threadIdx.x == 0) a.prof[4 * a.T + i] = gtimer();
    const double* tile = a.L + tri_rm(i, j) * bi2;
    const double2* bj = reinterpret_cast<const double2*>(a.beta + static_cast<int64_t>(j) * bi);
    for (int e = threadIdx.x; e < bi / 2; e += FT) vs[e] = __ldcg(bj + e);
    __syncthreads();
    if (a.prof && j == i - 1 && q == 0 && threadIdx.x == 0) a.prof[6 * a.T + i] = gtimer();
    const int hh = i - 1 - j;  // this slice helps block row j + 1 with quarter hh
    if (a.help && hh >= 1 && hh <= 3) {
      const double* ct = a.L + tri_rm(j + 1, j) * bi2 + hh * QC;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        double p[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        rows8_dot<false>(ct, bi, rbase + 8 * g, vs + hh * (QC / 2), QC / 64, lane, p);
        const double out = reduce8(p, lane);
        if ((lane & 3) == 0)
          a.part[(static_cast<int64_t>(j + 1) * 4 + hh) * bi + rbase + 8 * g + reduce8_row(lane)] = out;
      }
      signal_count(p_done + (j + 1) * S + q);
    }
    if (j == i - 1 && a.help) {  // own critical tile: quarter 0 and the quarters without a helper
#pragma unroll
      for (int g = 0; g < G; ++g) {
        double p[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        rows8_dot<false, true>(tile, bi, rbase + 8 * g, vs, QC / 64, lane, p);
        crit[g] = reduce8(p, lane);
        if (nhelp < 3) {
          double pt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
          rows8_dot<false, true>(tile + (nhelp + 1) * QC, bi, rbase + 8 * g, vs + (nhelp + 1) * (QC / 2),
                                 (3 - nhelp) * QC / 64, lane, pt);
          tail[g] = reduce8(pt, lane);
        }
      }
      continue;
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      double p[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      if (j == i - 1 && a.l1)
        rows8_dot<false, true>(tile, bi, rbase + 8 * g, vs, nchunk, lane, p);
      else
        rows8_dot<false>(tile, bi, rbase + 8 * g, vs, nchunk, lane, p);
      acc[g] += reduce8(p, lane);
    }
    if (a.prof && j == i - 1 && q == 0 && threadIdx.x == 0) a.prof[7 * a.T + i] = gtimer();
  }
  const int64_t g0 = static_cast<int64_t>(i) * bi;
  if (i == 0 && threadIdx.x == 0)
    prefetch_l2(a.dinv + static_cast<int64_t>(q) * R * bi, sizeof(double) * R * bi);
  const int mine = reduce8_row(lane);
  if (a.help && i >= 1) {  // the critical tile's quarters, in a fixed order
    if (nhelp > 0) wait_count(p_done + i * S + q, nhelp, true);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      double t = crit[g];
      for (int h = 1; h <= 3; ++h)
        t += h <= nhelp ? __ldcg(a.part + (static_cast<int64_t>(i) * 4 + h) * bi + rbase + 8 * g + mine)
                        : (h == nhelp + 1 ? tail[g] : 0.0);
      acc[g] += t;
    }
  }
  if ((lane & 3) == 0) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int64_t r = g0 + rbase + 8 * g + mine;
      a.xr[r] = a.y[r] - acc[g];
    }
  }
  signal_count(r_done + i);
  if (a.prof && q == 0 && threadIdx.x == 0) a.prof[i] = gtimer();
  wait_count(r_done + i, S, true);
  if (a.prof && q == 0 && threadIdx.x == 0) a.prof[5 * a.T + i] = gtimer();
  // beta_i[rows] = Dinv_i[rows, 0..row] r_i   (lower triangular)
  const double* D = a.dinv + static_cast<int64_t>(i) * bi2;
  const double2* rv = reinterpret_cast<const double2*>(a.xr + g0);
  for (int e = threadIdx.x; e < bi / 2; e += FT) vs[e] = __ldcg(rv + e);
  __syncthreads();
#pragma unroll
  for (int g = 0; g < G; ++g) {
    double p[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    rows8_dot<true, true>(D, bi, rbase + 8 * g, vs, nchunk, lane, p);
    const double out = reduce8(p, lane);
    if ((lane & 3) == 0) a.beta[g0 + rbase + 8 * g + mine] = out;
  }
  signal_count(b_done + i);
  if (a.prof && q == 0 && threadIdx.x == 0) a.prof[a.T + i] = gtimer();
}

// out[cols] += sum over `rows` rows r of M[r][cols] w[r] (ld = bi): lanes own
// CPL adjacent columns (double2 loads), RPI rows per warp instruction; the
// row weights come from w through warp shuffles (32 rows per load)
// kMode: 0 L2 (ldcg), 1 streaming (ldcs), 2 staged in L1 (ldca)
template <int R, int kMode>
GPB_DEVINL void cols_dot(const double* M, int bi, int r_first, int rows, const double* w, int col0,
                         int lane, double (&acc)[R / 32 > 2 ? R / 32 : 2]) {
  constexpr int CPL = R / 32 > 2 ? R / 32 : 2;  // columns per lane
  constexpr int LPR = R / CPL;                  // lanes per row
  constexpr int RPI = 32 / LPR;                 // rows per instruction
  const int sub = lane / LPR;                   // which of the RPI rows
  const int cl = lane % LPR;
  for (int rb = 0; rb < rows; rb += 32) {
    const double wv = __ldcg(w + rb + lane);
#pragma unroll 16
    for (int k = 0; k < 32 / RPI; ++k) {
      const int rr = RPI * k + sub;
      const double wk = __shfl_sync(0xffffffffu, wv, rr);
      const double* row = M + static_cast<int64_t>(r_first + rb + rr) * bi + col0 + cl * CPL;
#pragma unroll
      for (int c = 0; c < CPL; c += 2) {
        const double2* rp = reinterpret_cast<const double2*>(row + c);
        const double2 x = kMode == 1 ? __ldcs(rp) : kMode == 2 ? __ldca(rp) : __ldcg(rp);
        acc[c] = fma(x.x, wk, acc[c]);
        acc[c + 1] = fma(x.y, wk, acc[c + 1]);
      }
    }
  }
}

// fixed-order sum of the warps' column partials: lanes of the same columns
// (RPI > 1) first, then warps in index order; warp 0 gets the totals
template <int R>
GPB_DEVINL void cols_reduce(double (&acc)[R / 32 > 2 ? R / 32 : 2], double* red, int lane, int warp) {
  constexpr int CPL = R / 32 > 2 ? R / 32 : 2;
  constexpr int LPR = R / CPL;
#pragma unroll
  for (int o = LPR; o < 32; o <<= 1)
#pragma unroll
    for (int c = 0; c < CPL; ++c) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
  if (lane < LPR)
#pragma unroll
    for (int c = 0; c < CPL; ++c) red[warp * R + lane * CPL + c] = acc[c];
  __syncthreads();
  if (warp == 0 && lane < LPR)
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      double s = 0.0;
      for (int w = 0; w < FW; ++w) s += red[w * R + lane * CPL + c];
      acc[c] = s;
    }
}

// backward slice: columns [q R, q R + R) of block row i; warps split the bi
// rows of each tile
template <int R>
__device__ void backward_slice(const FlowArgs& a, int i, int q, double* red) {
  const int bi = a.bi, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int CPL = R / 32 > 2 ? R / 32 : 2;
  constexpr int LPR = R / CPL;
  const int64_t bi2 = static_cast<int64_t>(bi) * bi;
  const int col0 = q * R;
  const int rows_w = bi / FW;  // rows of each tile per warp
  const int r0 = warp * rows_w;
  int* t_done = a.flags + 2 * a.T;
  int* a_done = a.flags + 3 * a.T;
  const int S = bi / R;
  int* pb_done = a.flags + 4 * a.T + a.T * S;  // [T][S] helper quarters (backward)
  double* partb = a.part + 4 * static_cast<int64_t>(a.T) * bi;
  const int QR = bi / 4;  // rows of a quarter of the critical column slice
  // Helpers, as in the forward: rows quarter h = 1..3 of the critical column
  // slice of tile (i + 1, i) is computed by slice q of block row i - h, which
  // waits for alpha_{i+1} anyway; its four warps split the quarter's rows
  const int nhelp = a.help ? min(3, i) : 0;
  double acc[CPL], crit[CPL], tail[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) acc[c] = crit[c] = tail[c] = 0.0;
  wait_count(a.flags + a.T + i, S);  // beta_i complete (and r_i no longer read)
  for (int j = a.T - 1; j > i; --j) {
    if (j == i + 1) {  // critical from here on: stage the column slices in L2
      prefetch_rows(a.L + tri_rm(j, i) * bi2 + col0, bi, R, bi);
      prefetch_rows(a.dinv + static_cast<int64_t>(i) * bi2 + col0, bi, R, bi);
    } else if (int64_t(j) * bi2 * 8 <= kL2Window) {  // late phase, as in the forward
      prefetch_rows(a.L + tri_rm(j, i) * bi2 + col0, bi, R, bi);
    }
    wait_count(a_done + j, S, j == i + 1);
    const int hh = j - 1 - i;  // this slice helps block row j - 1 with quarter hh
    if (a.help && hh >= 1 && hh <= 3) {
      double hacc[CPL];
#pragma unroll
      for (int c = 0; c < CPL; ++c) hacc[c] = 0.0;
      const int rq = hh * QR + warp * (QR / FW);
      cols_dot<R, 1>(a.L + tri_rm(j, j - 1) * bi2, bi, rq, QR / FW, a.alpha + static_cast<int64_t>(j) * bi + rq, col0,
                     lane, hacc);
      __syncthreads();  // red is reused
      cols_reduce<R>(hacc, red, lane, warp);
      if (warp == 0 && lane < LPR)
#pragma unroll
        for (int c = 0; c < CPL; ++c)
          partb[(static_cast<int64_t>(j - 1) * 4 + hh) * bi + col0 + lane * CPL + c] = hacc[c];
      signal_count(pb_done + (j - 1) * S + q);
    }
    if (j == i + 1 && a.help) {  // own critical slice: rows quarter 0 and the quarters without a helper
      const int rq = warp * (QR / FW);
      cols_dot<R, 1>(a.L + tri_rm(j, i) * bi2, bi, rq, QR / FW, a.alpha + static_cast<int64_t>(j) * bi + rq, col0,
                     lane, crit);
      if (nhelp < 3) {
        const int nt = (3 - nhelp) * QR / FW, rt = (nhelp + 1) * QR + warp * nt;
        cols_dot<R, 1>(a.L + tri_rm(j, i) * bi2, bi, rt, nt, a.alpha + static_cast<int64_t>(j) * bi + rt, col0,
                       lane, tail);
      }
      continue;
    }
    cols_dot<R, 1>(a.L + tri_rm(j, i) * bi2, bi, r0, rows_w, a.alpha + static_cast<int64_t>(j) * bi + r0,
                      col0, lane, acc);
  }
  if (i == a.T - 1) prefetch_rows(a.dinv + static_cast<int64_t>(i) * bi2 + col0, bi, R, bi);
  const int64_t g0 = static_cast<int64_t>(i) * bi;
  __syncthreads();  // red is reused
  cols_reduce<R>(acc, red, lane, warp);
  if (a.help && i + 1 < a.T) {  // the critical slice's quarters, in a fixed order
    __syncthreads();
    cols_reduce<R>(crit, red, lane, warp);
    __syncthreads();
    cols_reduce<R>(tail, red, lane, warp);
    if (nhelp > 0) wait_count(pb_done + i * S + q, nhelp, true);
    if (warp == 0 && lane < LPR)
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        double t = crit[c];
        for (int h = 1; h <= 3; ++h)
          t += h <= nhelp ? __ldcg(partb + (static_cast<int64_t>(i) * 4 + h) * bi + col0 + lane * CPL + c)
                          : (h == nhelp + 1 ? tail[c] : 0.0);
        acc[c] += t;
      }
  }
  if (warp == 0 && lane < LPR)
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const int64_t e = g0 + col0 + lane * CPL + c;
      a.xr[e] = __ldcg(a.beta + e) - acc[c];
    }
  signal_count(t_done + i);
  if (a.prof && q == 0 && threadIdx.x == 0) a.prof[2 * a.T + i] = gtimer();
  wait_count(t_done + i, S, true);
  // alpha_i[cols] = sum_{r >= first col} Dinv_i[r][cols] t[r]  (Dinv_i lower)
#pragma unroll
  for (int c = 0; c < CPL; ++c) acc[c] = 0.0;
  const int lo = max(r0, col0 & ~31);  // rows above the slice's first column are zero
  if (lo < r0 + rows_w)
    cols_dot<R, 0>(a.dinv + static_cast<int64_t>(i) * bi2, bi, lo, r0 + rows_w - lo, a.xr + g0 + lo, col0, lane,
                   acc);
  __syncthreads();  // red is reused
  cols_reduce<R>(acc, red, lane, warp);
  if (warp == 0 && lane < LPR)
#pragma unroll
    for (int c = 0; c < CPL; ++c) a.alpha[g0 + col0 + lane * CPL + c] = acc[c];
  signal_count(a_done + i);
  if (a.prof && q == 0 && threadIdx.x == 0) a.prof[3 * a.T + i] = gtimer();
}

template <int R>
__global__ void __launch_bounds__(FT, 7) solve_flow_kernel(FlowArgs a) {
  __shared__ double red[FW * R];
  __shared__ double2 vs[256];  // beta_j / r_i of the forward (bi <= 512)
  const int S = a.bi / R;
  const int s = blockIdx.x;
  forward_slice<R>(a, s / S, s % S, vs);
  const int sb = gridDim.x - 1 - s;  // mirrored: early finishers start the backward
  backward_slice<R>(a, a.T - 1 - sb / S, sb % S, red);
}

template <int R>
cudaError_t launch_r(const FlowArgs& a, int nslices, cudaStream_t s, bool* launched) {
  int per_sm = 0, dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, solve_flow_kernel<R>, FT, 0);
  if (e != cudaSuccess) return e;
  if (nslices > per_sm * sms) return cudaSuccess;  // not co-resident: caller falls back
  FlowArgs args = a;
  void* params[] = {&args};
  e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(solve_flow_kernel<R>),
                                  dim3(static_cast<unsigned>(nslices)), dim3(FT), params, 0, s);
  if (e == cudaSuccess) *launched = true;
  return e;
}

}  // namespace

int solve_flow_slice_rows(int64_t np_, int bi) {
  // smallest slice height whose grid fits on the chip at the kernel's occupancy
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  for (int R : {32, 64, 128}) {
    if (bi % R) continue;
    int per_sm = 0;
    cudaError_t e = cudaSuccess;
    if (R == 32) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, solve_flow_kernel<32>, FT, 0);
    if (R == 64) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, solve_flow_kernel<64>, FT, 0);
    if (R == 128) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, solve_flow_kernel<128>, FT, 0);
    if (e != cudaSuccess) return 0;
    if (np_ / R <= static_cast<int64_t>(per_sm) * sms) return R;
  }
  return 0;
}

size_t solve_flow_scratch_bytes(int T, int bi) {
  // helper partials [2][T][4][bi] doubles, then 4T + 2 T (bi / 32) counters (the largest slice count)
  return sizeof(double) * 8 * size_t(T) * bi + sizeof(int) * (4 * size_t(T) + 2 * size_t(T) * (bi / 32));
}

cudaError_t launch_solve_flow(const double* L, const double* dinv, const double* y, double* beta,
                              double* alpha, double* xr, void* scratch, int T, int bi, int R,
                              cudaStream_t s, bool* launched) {
  double* part = static_cast<double*>(scratch);
  int* flags = reinterpret_cast<int*>(part + 8 * size_t(T) * bi);
  *launched = false;
  if (R == 0 || bi % R != 0 || bi % 64 != 0 || bi > 512) return cudaSuccess;
  static unsigned long long* prof = nullptr;
  static int prof_T = 0;
  if (getenv("GPB_SOLVE_PROF") && prof_T != T) {
    if (prof) cudaFree(prof);
    cudaMalloc(&prof, sizeof(unsigned long long) * 8 * T);
    cudaMemset(prof, 0, sizeof(unsigned long long) * 8 * T);
    prof_T = T;
  }
  const char* pfe = getenv("GPB_FLOW_PREFETCH");
  const char* l1e = getenv("GPB_FLOW_L1");
  // helpers split the critical tiles in quarters of bi / 4 = 128 columns / rows,
  // i.e. 32 rows per warp (the 32-row chunks of cols_dot): bi = 512 only
  const char* hle = getenv("GPB_FLOW_HELP");
  FlowArgs a{L, dinv, y, beta, alpha, xr, flags, part, T, bi, R, getenv("GPB_SOLVE_PROF") ? prof : nullptr,
             pfe ? atoi(pfe) : 2, l1e ? atoi(l1e) : 1, bi == 512 ? (hle ? atoi(hle) : 1) : 0};
  cudaError_t e = cudaMemsetAsync(flags, 0, sizeof(int) * (4 * T + 2 * T * (bi / R)), s);
  if (e != cudaSuccess) return e;
  const int nslices = T * (bi / R);
  switch (R) {
    case 32: e = launch_r<32>(a, nslices, s, launched); break;
    case 64: e = launch_r<64>(a, nslices, s, launched); break;
    case 128: e = launch_r<128>(a, nslices, s, launched); break;
    default: break;
  }
  if (a.prof && *launched) {  // per block row: r published, beta published, t published, alpha published
    std::vector<unsigned long long> h(8 * T);
    cudaStreamSynchronize(s);
    cudaMemcpy(h.data(), a.prof, sizeof(unsigned long long) * 8 * T, cudaMemcpyDeviceToHost);
    const unsigned long long t0 = h[0];
    auto at = [&](unsigned long long v) { return v ? (double(v) - double(t0)) * 1e-3 : -1.0; };
    for (int i = 0; i < T; ++i)
      fprintf(stderr,
              "flow row %3d: seen beta_{i-1} %8.1f loaded %8.1f dot %8.1f r %8.1f all r %8.1f beta %8.1f | t %8.1f "
              "alpha %8.1f us\n",
              i, at(h[4 * T + i]), at(h[6 * T + i]), at(h[7 * T + i]), at(h[i]), at(h[5 * T + i]), at(h[T + i]),
              at(h[2 * T + i]), at(h[3 * T + i]));
  }
  return e;
}

}  // namespace gpb
