// Grouped FP64 tensor-core GEMM (DMMA.8x8x4) for the tiled-GP hot path.
//
// One launch executes a list of independent tile jobs ("grouped GEMM"): the
// Cholesky trailing update of one step (taskgp tiles.py:41-46 SYRK/GEMM over
// every trailing tile), the panel TRSM as a product with the inverted
// diagonal tile, the prediction TRSM sweeps (tiled.py:263-298), the inverse
// factor (model.py:358-361), K^-1 = X^T X (model.py:362-380) and the full
// posterior covariance (model.py:258-269).
//
//   Cout[job] = alpha * A[job] * B[job]^T + beta * Cin[job]
//
// A is M x K, B is N x K (so the product is "NT"); each operand is either
// K-MAJOR (k contiguous: element (m,k) at base[m*ld + k]) or MN-MAJOR (m
// contiguous: element (m,k) at base[k*ld + m]).  Either operand may be
// "tiled in k": k runs through consecutive ktile-deep tiles kstride apart
// (K-MAJOR: element (m,k) at base[(k/ktile)*kstride + m*ld + k%ktile]), which
// walks a row (or, transposed, a column) panel of packed tiles without a copy.
#pragma once
#include "common.cuh"

namespace gpb {

// CTA tile is GBM x GBN; every job's K must be a multiple of GBK (the
// deepest k stage any kernel configuration uses).
constexpr int GBM = 128, GBN = 128, GBK = 32;

// EPI_MIRROR: EPI_AXPBY plus the mirror stores of GemmParams (K-major A and B)
enum GemmEpi : int { EPI_AXPBY = 0, EPI_SUMSQ = 1, EPI_MIRROR = 2 };

struct __align__(16) GemmJob {
  const double* A;
  const double* B;
  const double* Cin;   // may alias Cout (in-place update) or be null if beta == 0
  double* Cout;
  double* aux;         // EPI_SUMSQ: base of this job's partial rows
  int K;               // multiple of GBK, may be 0
  int lower;           // 1: skip blocks above the block diagonal (diagonal tiles)
  int nlim;            // > 0: only the first nlim 128-column blocks of this job
  int pad_;
};

struct GemmParams {
  const GemmJob* jobs;
  int njobs;
  int mblk, nblk;            // BM x BN blocks per job
  int64_t lda, ldb, ldc;
  int64_t a_ktile, a_kstride;  // K-MAJOR tiled-k walk (ktile = 1<<30 for plain)
  int64_t b_ktile, b_kstride;
  double alpha, beta;
  int64_t aux_ld;            // EPI_SUMSQ: stride between 128-row partial rows
  int64_t max_k;             // largest job K (kernel-configuration hint), 0 if unknown
  // TMA path (gemm_tma.cu): the buffers every job's A / B pointer lies in and
  // their extents in doubles from those bases; null = cp.async kernel only
  const double* a_base;
  int64_t a_extent;
  const double* b_base;
  int64_t b_extent;
  // mirror stores (the fused panel exchange of the multi-GPU schedule): every
  // output element of job j is also stored at mirror[j * nmirror + r] + the
  // same offset from Cout, for the non-null entries r < nmirror -- peer
  // ranks' buffers mapped through CUDA IPC, written over NVLink
  double* const* mirror;
  int nmirror;
};

// mirror stores of one output element (offset `idx` from the job's Cout)
GPB_DEVINL void store_mirrors(const GemmParams& p, int job_id, int64_t idx, double v) {
  for (int r = 0; r < p.nmirror; ++r) {
    double* m = p.mirror[static_cast<int64_t>(job_id) * p.nmirror + r];
    if (m) m[idx] = v;
  }
}

// one operand of the TMA kernel: a job pointer p maps to row (p - base) / ld,
// column (p - base) % ld of the tensor map; a tiled-k walk advances kt_rows
// rows per ktile-deep k tile
struct TmaOperand {
  const double* base;
  int64_t ld, ktile, kt_rows;
};

// Host launcher (gemm.cu).  a_kmajor / b_kmajor choose operand layouts.
cudaError_t launch_gemm(const GemmParams& p, bool a_kmajor, bool b_kmajor, int epi,
                        cudaStream_t stream);
cudaError_t gemm_init_attributes();
// TMA-fed kernel; *used = false when the launch does not qualify (no operand
// bases, unaligned views, GPB_GEMM_TMA=0) and nothing was launched
cudaError_t launch_gemm_tma(const GemmParams& p, bool a_kmajor, bool b_kmajor, int epi,
                            cudaStream_t stream, bool* used);
// tools only: 0 off, 1 four consumer warps, 2 eight, 3 automatic
void gemm_force_tma(int mode);
// tools only: force a kernel configuration (-1: GPB_GEMM_CFG / automatic)
void gemm_force_config(int cfg);

}  // namespace gpb
