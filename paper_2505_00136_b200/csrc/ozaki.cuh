// FP64 products on the 5th-generation tensor cores (tcgen05.mma kind::i8,
// accumulators in TMEM): the long-K products of the path,
//
//   W = Cin - L[i, 0..i) V[0..i)          prediction sweep   (taskgp tiled.py:263-298)
//   L(i,j) -= [X]_i [X]_j^T               trailing updates   (taskgp tiled.py:187-204)
//
// computed from signed 7-bit digit planes of their operands (Ozaki splitting
// with a fixed-point scale per operand buffer):
//
//   x = sx * sum_{p=1..S} d_p(x) 2^(-7p) + r,   |x| <= sx 127/128,  |r| <= sx 2^(-7S-1),
//       d_1 in [-127, 127], d_p in [-64, 64] for p > 1
//   sum_k a_k b_k ~= sa sb sum_{t=2..S+1} 2^(-7t) G_t,
//   G_t = sum_{p+q=t} sum_k d_p(a_k) d_q(b_k)   (exact int32 sums on the int8 pipe)
//
// The digit extraction of x / sx is exact (round-to-nearest and the
// subtraction of the rounded value; the division by the scale itself rounds
// once, 2^-53 relative, unless sx is a power of two), the int32 group sums are exact for
// K <= kOzakiMaxK, and the groups are combined in FP64, least significant
// first.  The only errors are the dropped remainder r of each operand and the
// dropped digit pairs p+q > S+1: both below 2^(-7S+3) relative to sa sb per
// term (S = 8: 2^-53).  No FP64 tcgen05 kind exists on sm_100a, so this is how
// the path reaches the tcgen05 pipe at all; the FP64 DMMA kernels remain for
// the short products and behind GPB_OZAKI=0 / gpb_model_set_ozaki(m, 0).
//
// Plane layout ("boxed").  An operand is a matrix of rows x K int8 digits per
// plane, rows in blocks of 128, k in chunks of 32.  The S planes of one (row
// block, k chunk) are S consecutive 4 KB boxes, each box the shared-memory
// image the MMA reads (128 rows of 32 bytes, SWIZZLE_32B), so a CTA fetches
// the planes of a chunk with ONE contiguous bulk copy per operand.  (Planes
// kept in the operand's own row-major order and fetched as 128 x 32-byte TMA
// boxes issue one L2 request per 32-byte row: ncu showed the L2 tag pipeline
// at 73% with the tensor pipe 43-66% active.)  Operands are tiled: tile t
// (tr rows x tc columns of k) occupies tr * tc * S bytes, its boxes ordered
// [row block][k chunk][plane]; a k walk visits tc / 32 chunks of a tile, then
// jumps tile_stride bytes to the next tile.
#pragma once
#include <cuda.h>

#include "common.cuh"

namespace gpb {

constexpr int kOzakiMaxSlices = 8;
constexpr int kOzakiBM = 128, kOzakiBN = 128, kOzakiBK = 32;
constexpr int kOzakiBox = kOzakiBM * kOzakiBK;  // bytes
// |G_t| <= K (2 * 127 * 64 + 6 * 64 * 64) < 2^31 (at most two pairs of a group hold a first digit)
constexpr int64_t kOzakiMaxK = 32768;

// Digit planes of `ntiles` consecutive row-major tiles of tr x tc doubles
// (tr a multiple of 128, tc of 32) into the boxed layout at `planes` (tile t
// at planes + t * tr * tc * slices).  *flag is set to 1 when an element
// exceeds scale * 127 / 128 (digits saturate).
cudaError_t launch_ozaki_slice_tiles(const double* src, int64_t ntiles, int tr, int tc, double scale,
                                     int8_t* planes, int slices, int* flag, cudaStream_t st);

// Digit planes of a (rows x cols, row-major, ld) block of doubles TRANSPOSED:
// operand row = source column c, k = k0 + source row.  One tile spans the
// whole K range: box of (c / 128, k / 32) at planes + ((c / 128) * rb_boxes +
// (k / 32) * kc_boxes) * slices * 4096 -- row-block major (rb_boxes = chunks
// of the whole K, kc_boxes = 1: the prediction's V^T) or chunk major (rb_boxes
// = 1, kc_boxes = row blocks: operands of different K with one rb_stride, the
// gradient's X panels).  rows and k0 multiples of 64, cols of 128.
cudaError_t launch_ozaki_slice_t(const double* src, int64_t rows, int64_t cols, int64_t ld, double scale,
                                 int8_t* planes, int64_t rb_boxes, int64_t kc_boxes, int64_t k0, int slices,
                                 int* flag, cudaStream_t st);

// fixed-point scale of an operand bounded by `bound`: digits cover |x| <= scale * 127 / 128;
// the margin absorbs round-off in entries that reach the bound
inline double ozaki_plane_scale(double bound) { return bound * (128.0 / 127.0) * (1.0 + 1e-9); }

// Batched form of launch_ozaki_slice_t: job t slices the rows x cols block at jobs[t].src into
// jobs[t].planes at k offset jobs[t].k0 (same rows, cols, ld and box strides for every job).
struct OzakiSliceJob {
  const double* src;
  int8_t* planes;
  int64_t k0;
};
cudaError_t launch_ozaki_slice_t_batch(const OzakiSliceJob* jobs, int njobs, int64_t rows, int64_t cols, int64_t ld,
                                       double scale, int64_t rb_boxes, int64_t kc_boxes, int slices, int* flag,
                                       cudaStream_t st);

struct OzakiOperand {
  const int8_t* planes;
  int64_t tile_stride;  // bytes from a tile to the next one along k
  int chunks_per_tile;  // tc / 32
  int64_t rb_stride;    // bytes from a row block to the next one inside a tile: chunks_per_tile * slices * 4096
  int64_t chunk_stride = 0;  // bytes from a k chunk to the next one inside a tile (0: slices * 4096)
};

struct OzakiJob {
  int64_t a_off, b_off;  // byte offsets of the job's first row block at k = 0 (added to the launch's)
  double* C;
  int lower;
  int kchunks;  // this job's depth in chunks of 32 (0: the launch's K)
};

struct OzakiGemm {
  OzakiOperand a, b;     // A: M rows, B: N rows, both K-major
  int64_t a_off, b_off;  // byte offsets of row block 0 at k = 0 (with jobs: a common offset, e.g. a k segment)
  int M, N, K;           // multiples of 128 / 128 / 32; K <= kOzakiMaxK
  int slices;
  double alpha;  // Cout = beta * Cin + alpha * sum (the caller folds the scales sa sb into alpha)
  double beta;
  const double* Cin;
  double* Cout;
  int64_t ldc_in, ldc_out;
  // grouped form (the factorisation's trailing updates): njobs independent
  // M x N products sharing the operand descriptions, job j reading its rows
  // from jobs[j].a_off / b_off and writing C = beta C + alpha sum in place
  // (ldc_in = ldc_out).  A `lower` job skips the blocks above the diagonal.
  const OzakiJob* jobs = nullptr;  // device array
  int njobs = 0;
};

cudaError_t launch_ozaki_gemm(const OzakiGemm& g, cudaStream_t st);
cudaError_t ozaki_init_attributes();

}  // namespace gpb
