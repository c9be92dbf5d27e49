// FP64 products on the 5th-generation tensor cores (tcgen05.mma kind::i8,
// accumulators in TMEM): the long-K prediction product
//
//   W = Cin - L[i, 0..i) V[0..i)            (taskgp tiled.py:263-298)
//
// computed from signed 7-bit digit planes of its operands (Ozaki splitting
// with a fixed-point scale per operand buffer):
//
//   x = sx * sum_{p=1..S} d_p(x) 2^(-7p) + r,   d_p in [-64, 64],  |r| <= sx 2^(-7S-1)
//   sum_k a_k b_k ~= sa sb sum_{t=2..S+1} 2^(-7t) G_t,
//   G_t = sum_{p+q=t} sum_k d_p(a_k) d_q(b_k)   (exact int32 sums on the int8 pipe)
//
// The digit extraction is exact (power-of-two scalings, round-to-nearest and
// the subtraction of the rounded value), the int32 group sums are exact for
// K <= kOzakiMaxK, and the groups are combined once, in FP64, least
// significant first.  The only errors are the dropped remainder r of each
// operand and the dropped digit pairs p+q > S+1: both below 2^(-7S+3) relative to
// sa sb per term (S = 8: 2^-53).  No FP64 tcgen05 kind exists on sm_100a, so this is
// how the path reaches the tcgen05 pipe at all; the DMMA kernels stay the
// default and the reference for parity (GPB_OZAKI=1 / gpb_model_set_ozaki
// opt in).
#pragma once
#include <cuda.h>

#include "common.cuh"

namespace gpb {

constexpr int kOzakiMaxSlices = 8;
constexpr int kOzakiBM = 128, kOzakiBN = 64, kOzakiBK = 64;
// |G_t| <= S * K * 64 * 64 < 2^31
constexpr int64_t kOzakiMaxK = 32768;

// Digit planes of a contiguous array, same element order as the source:
// plane p (0-based) of element e at planes[p * plane_stride + e].
// *flag is set to 1 when an element exceeds scale / 2 (digits saturate).
cudaError_t launch_ozaki_slice(const double* src, int64_t count, double scale, int8_t* planes,
                               int64_t plane_stride, int slices, int* flag, cudaStream_t st);

// Digit planes of a (rows x cols, row-major, ld) block, TRANSPOSED: plane p of
// element (k, c) at planes[p * plane_stride + c * out_ld + k0 + k]  (the
// K-major B operand of the product: one row per column c, k contiguous).
// rows must be a multiple of 64, cols a multiple of 64.
cudaError_t launch_ozaki_slice_t(const double* src, int rows, int64_t cols, int64_t ld, double scale,
                                 int8_t* planes, int64_t plane_stride, int64_t out_ld, int64_t k0,
                                 int slices, int* flag, cudaStream_t st);

struct OzakiJob {
  int a_row0, b_row0;
  double* C;
  int lower, pad;
};

struct OzakiGemm {
  // A planes: 2-D byte view (a_pitch bytes per row, a_rows rows per plane,
  // planes stacked along rows); the M x K operand starts at row a_row0,
  // column 0, and k walks a_ktile bytes per tile, a_kt_rows rows down per tile
  const int8_t* a_planes;
  int64_t a_pitch, a_rows, a_row0;
  int a_ktile, a_kt_rows;
  // B planes: N x K rows starting at row b_row0, column b_col0; plain walk
  // along the row when b_ktile == 0, else tiled like A
  const int8_t* b_planes;
  int64_t b_pitch, b_rows, b_row0, b_col0;
  int b_ktile = 0, b_kt_rows = 0;
  int M, N, K;     // multiples of 128 / 64 / 64; K <= kOzakiMaxK
  int slices;
  double alpha;    // Cout = beta * Cin + alpha * sa sb * sum (caller folds sa sb in)
  double beta;
  const double* Cin;
  double* Cout;
  int64_t ldc_in, ldc_out;
  // grouped form (the factorisation's trailing update, tiled.py:187-204): njobs
  // independent M x N products sharing the plane buffers, job j reading A rows
  // from jobs[j].a_row0, B rows from jobs[j].b_row0 (a_row0 / b_row0 above are
  // ignored) and updating C in place: C = beta C + alpha sum, ldc_in = ldc_out.
  // A `lower` job skips the 128 x 64 blocks above the diagonal 128-block.
  const OzakiJob* jobs = nullptr;  // device array
  int njobs = 0;
};

// false (nothing launched) when the driver entry point for tensor maps is missing
cudaError_t launch_ozaki_gemm(const OzakiGemm& g, cudaStream_t st, bool* used);
cudaError_t ozaki_init_attributes();

}  // namespace gpb
