// Shared device helpers for the B200 tiled-GP kernels (sm_100a, FP64).
//
// Storage conventions:
//  * The user's tiling (n = T * b, taskgp tiled.py:34-41) is kept; each b x b
//    tile is padded to bp = roundup(b, 128) rows/cols.  Padded indices are
//    "decoupled identity" rows (K[p,p] = 1, zero coupling), so the Cholesky
//    factor, solves and inverses of the real part are unchanged.
//  * Lower tile grids are packed in ROW-MAJOR TILE ORDER: tile (i, j), i >= j,
//    at index i(i+1)/2 + j, each tile bp x bp row-major.  A tile row panel
//    (i, 0..i) is therefore contiguous.  The inverse factor X = L^-1 uses
//    COLUMN-MAJOR tile order (tiles (j..T-1, j) contiguous) so its column
//    panels are plain row-major matrices with ld = bp.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define GPB_DEVINL __device__ __forceinline__

namespace gpb {

constexpr int kTileAlign = 128;  // bp and padded test chunks are multiples of this

GPB_DEVINL int64_t tri_rm(int64_t i, int64_t j) { return i * (i + 1) / 2 + j; }
// column-major packed lower index (tiles (j..T-1, j) contiguous)
GPB_DEVINL int64_t tri_cm(int64_t i, int64_t j, int64_t T) {
  return j * T - j * (j - 1) / 2 + (i - j);
}
inline int64_t h_tri_rm(int64_t i, int64_t j) { return i * (i + 1) / 2 + j; }
inline int64_t h_tri_cm(int64_t i, int64_t j, int64_t T) {
  return j * T - j * (j - 1) / 2 + (i - j);
}

// D = A(8x4, row) * B(4x8, col) + D on the FP64 tensor pipe (SASS DMMA.8x8x4).
// Lane l holds a = A[l/4][l%4], b = B[l%4][l/4], d = D[l/4][2(l%4) + {0,1}].
GPB_DEVINL void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

GPB_DEVINL void cp_async16(void* smem, const void* gmem) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
GPB_DEVINL void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
GPB_DEVINL void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

GPB_DEVINL double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace gpb
