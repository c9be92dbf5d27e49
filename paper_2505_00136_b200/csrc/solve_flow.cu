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
#include "kernels.cuh"

namespace gpb {

namespace {

constexpr int FT = 128;  // threads per CTA (4 warps)
constexpr int FW = FT / 32;

GPB_DEVINL int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

GPB_DEVINL void wait_count(const int* flag, int want) {
  if (threadIdx.x == 0) {
    int ns = 32;
    while (ld_acquire(flag) < want) {
      __nanosleep(ns);
      ns = ns < 512 ? 2 * ns : 512;
    }
  }
  __syncthreads();
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
  int* flags;          // 4T counters, zero on entry
  int T, bi, R;
};

// forward slice: rows [row0, row0 + R) of block row i, R / FW rows per warp
template <int R>
__device__ void forward_slice(const FlowArgs& a, int i, int q) {
  const int bi = a.bi, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int RW = R / FW;  // rows per warp (<= 32: lane `k` owns row k of the warp)
  const int64_t bi2 = static_cast<int64_t>(bi) * bi;
  const int rbase = q * R + warp * RW;  // first row of this warp inside block row i
  double acc = 0.0;                     // sum for row rbase + lane (lane < RW)
  const int nchunk = bi / 64;           // double2 chunks per lane per row
  int* r_done = a.flags;
  int* b_done = a.flags + a.T;
  const int S = bi / R;
  for (int j = 0; j < i; ++j) {
    wait_count(b_done + j, S);
    const double* tile = a.L + tri_rm(i, j) * bi2;
    const double2* bj = reinterpret_cast<const double2*>(a.beta + static_cast<int64_t>(j) * bi);
    double2 bv[8];
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (c < nchunk) bv[c] = __ldcg(bj + lane + 32 * c);
#pragma unroll 2
    for (int k = 0; k < RW; ++k) {
      const double2* row = reinterpret_cast<const double2*>(tile + static_cast<int64_t>(rbase + k) * bi);
      double p = 0.0;
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c < nchunk) {
          const double2 v = __ldcs(row + lane + 32 * c);
          p = fma(v.x, bv[c].x, p);
          p = fma(v.y, bv[c].y, p);
        }
      p = warp_sum(p);
      if (lane == k) acc += p;
    }
  }
  const int64_t g0 = static_cast<int64_t>(i) * bi;
  if (lane < RW) a.xr[g0 + rbase + lane] = a.y[g0 + rbase + lane] - acc;
  signal_count(r_done + i);
  wait_count(r_done + i, S);
  // beta_i[rows] = Dinv_i[rows, 0..row] r_i   (lower triangular)
  const double* D = a.dinv + static_cast<int64_t>(i) * bi2;
  const double2* rv = reinterpret_cast<const double2*>(a.xr + g0);
  double2 r2[8];
#pragma unroll
  for (int c = 0; c < 8; ++c)
    if (c < nchunk) r2[c] = __ldcg(rv + lane + 32 * c);
  double out = 0.0;
  for (int k = 0; k < RW; ++k) {
    const int r = rbase + k;
    const double2* row = reinterpret_cast<const double2*>(D + static_cast<int64_t>(r) * bi);
    double p = 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int col = 2 * (lane + 32 * c);
      if (c < nchunk && col <= r) {
        const double2 v = __ldcg(row + lane + 32 * c);
        p = fma(v.x, r2[c].x, p);
        p = fma(v.y, r2[c].y, p);  // v.y = 0 above the diagonal
      }
    }
    p = warp_sum(p);
    if (lane == k) out = p;
  }
  if (lane < RW) a.beta[g0 + rbase + lane] = out;
  signal_count(b_done + i);
}

// backward slice: columns [col0, col0 + R) of block row i; lanes own R/32
// adjacent columns, warps split the bi rows of each tile
template <int R>
__device__ void backward_slice(const FlowArgs& a, int i, int q, double* red) {
  const int bi = a.bi, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int CL = R / 32;  // columns per lane
  const int64_t bi2 = static_cast<int64_t>(bi) * bi;
  const int col0 = q * R + lane * CL;
  const int rows_w = bi / FW;  // rows of each tile per warp
  const int r0 = warp * rows_w;
  int* t_done = a.flags + 2 * a.T;
  int* a_done = a.flags + 3 * a.T;
  const int S = bi / R;
  double acc[CL];
#pragma unroll
  for (int c = 0; c < CL; ++c) acc[c] = 0.0;
  wait_count(a.flags + a.T + i, S);  // beta_i complete (and r_i no longer read)
  for (int j = a.T - 1; j > i; --j) {
    wait_count(a_done + j, S);
    const double* tile = a.L + tri_rm(j, i) * bi2;
    const double* aj = a.alpha + static_cast<int64_t>(j) * bi + r0;
    for (int rb = 0; rb < rows_w; rb += 32) {
      const double av = __ldcg(aj + rb + lane);
#pragma unroll 16
      for (int k = 0; k < 32; ++k) {
        const double w = __shfl_sync(0xffffffffu, av, k);
        const double* row = tile + static_cast<int64_t>(r0 + rb + k) * bi + col0;
        if constexpr (CL == 1) {
          acc[0] = fma(__ldcs(row), w, acc[0]);
        } else {
#pragma unroll
          for (int c = 0; c < CL; c += 2) {
            const double2 v = __ldcs(reinterpret_cast<const double2*>(row + c));
            acc[c] = fma(v.x, w, acc[c]);
            acc[c + 1] = fma(v.y, w, acc[c + 1]);
          }
        }
      }
    }
  }
  // fixed-order cross-warp sum: t = beta - sum_w acc_w
  const int64_t g0 = static_cast<int64_t>(i) * bi;
#pragma unroll
  for (int c = 0; c < CL; ++c) red[warp * R + lane * CL + c] = acc[c];
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int c = 0; c < CL; ++c) {
      double s = 0.0;
      for (int w = 0; w < FW; ++w) s += red[w * R + lane * CL + c];
      a.xr[g0 + col0 + c] = __ldcg(a.beta + g0 + col0 + c) - s;
    }
  }
  signal_count(t_done + i);
  wait_count(t_done + i, S);
  // alpha_i[cols] = sum_{r >= col} Dinv_i[r][cols] t[r]
  const double* D = a.dinv + static_cast<int64_t>(i) * bi2;
  const double* tv = a.xr + g0 + r0;
#pragma unroll
  for (int c = 0; c < CL; ++c) acc[c] = 0.0;
  const int first = q * R;  // rows above the slice's first column are zero in Dinv
  for (int rb = 0; rb < rows_w; rb += 32) {
    if (r0 + rb + 31 < first) continue;
    const double tval = __ldcg(tv + rb + lane);
#pragma unroll 8
    for (int k = 0; k < 32; ++k) {
      const double w = __shfl_sync(0xffffffffu, tval, k);
      const double* row = D + static_cast<int64_t>(r0 + rb + k) * bi + col0;
      if constexpr (CL == 1) {
        acc[0] = fma(__ldcg(row), w, acc[0]);
      } else {
#pragma unroll
        for (int c = 0; c < CL; c += 2) {
          const double2 v = __ldcg(reinterpret_cast<const double2*>(row + c));
          acc[c] = fma(v.x, w, acc[c]);
          acc[c + 1] = fma(v.y, w, acc[c + 1]);
        }
      }
    }
  }
  __syncthreads();  // red is reused
#pragma unroll
  for (int c = 0; c < CL; ++c) red[warp * R + lane * CL + c] = acc[c];
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int c = 0; c < CL; ++c) {
      double s = 0.0;
      for (int w = 0; w < FW; ++w) s += red[w * R + lane * CL + c];
      a.alpha[g0 + col0 + c] = s;
    }
  }
  signal_count(a_done + i);
}

template <int R>
__global__ void __launch_bounds__(FT, 7) solve_flow_kernel(FlowArgs a) {
  __shared__ double red[FW * R];
  const int S = a.bi / R;
  const int s = blockIdx.x;
  forward_slice<R>(a, s / S, s % S);
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

cudaError_t launch_solve_flow(const double* L, const double* dinv, const double* y, double* beta,
                              double* alpha, double* xr, int* flags, int T, int bi, int R,
                              cudaStream_t s, bool* launched) {
  *launched = false;
  if (R == 0 || bi % R != 0 || bi % 64 != 0 || bi > 512) return cudaSuccess;
  FlowArgs a{L, dinv, y, beta, alpha, xr, flags, T, bi, R};
  cudaError_t e = cudaMemsetAsync(flags, 0, sizeof(int) * 4 * T, s);
  if (e != cudaSuccess) return e;
  const int nslices = T * (bi / R);
  switch (R) {
    case 32: return launch_r<32>(a, nslices, s, launched);
    case 64: return launch_r<64>(a, nslices, s, launched);
    case 128: return launch_r<128>(a, nslices, s, launched);
    default: return cudaSuccess;
  }
}

}  // namespace gpb
