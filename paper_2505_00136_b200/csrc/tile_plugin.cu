// Tile-kernel plugin entry points (secondary boundary).
//
// The reference lets a vendor backend replace its four factorisation
// kernels through register_tile_backend / set_tile_backend (taskgp
// tiles.py:98-117; contract tiles.py:132-164): potrf(a), trsm(l, b) solving
// X l^T = b, syrk(a, c) = c - a a^T, gemm(a, b, c) = c - a b^T on read-only
// float64 tiles, returning fresh arrays.  These entry points run each call on
// the same sm_100a kernels as the fused path (POTRF/TRTRI tile kernel and the
// grouped DMMA GEMM) so the reference's own tiled_cholesky can be driven by
// the GPU tile by tile.  Tiles of any size are padded to a multiple of 128
// with decoupled identity (potrf, trsm) or zeros (products).
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "gemm.cuh"
#include "gpb200.h"
#include "kernels.cuh"

using namespace gpb;

struct gpb_ctx;
extern "C" gpb_ctx* gpb_current(void);

namespace {

int64_t rup(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

struct Scratch {
  std::mutex mu;
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t n) {
    if (n <= bytes && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, n);
    if (e == cudaSuccess) bytes = n;
    return e;
  }
};
Scratch g_scratch;

// copy a (rows x cols, ld cols) into a zero-padded rp x cp buffer; optional identity padding
void pad_host(const double* a, int64_t rows, int64_t cols, int64_t rp, int64_t cp, bool ident,
              std::vector<double>& out) {
  out.assign(rp * cp, 0.0);
  for (int64_t r = 0; r < rows; ++r) std::memcpy(&out[r * cp], a + r * cols, sizeof(double) * cols);
  if (ident)
    for (int64_t r = rows; r < std::min(rp, cp); ++r) out[r * cp + r] = 1.0;
}

}  // namespace

extern "C" int gpb_plugin_fail(int code, const char* msg);

#define PL_TRY(x)                                                        \
  do {                                                                   \
    cudaError_t e_ = (x);                                                \
    if (e_ != cudaSuccess) return gpb_plugin_fail(GPB_CUDA, cudaGetErrorString(e_)); \
  } while (0)

namespace {

int run_gemm_nt(const double* a, const double* b, const double* c, int64_t m, int64_t n, int64_t k,
                double* out) {
  // out = c - a b^T  with a: m x k, b: n x k, c: m x n
  const int64_t mp = rup(m, GBM), np = rup(n, GBN), kp = rup(std::max<int64_t>(k, 1), GBK);
  std::vector<double> ha, hb, hc;
  pad_host(a, m, k, mp, kp, false, ha);
  pad_host(b, n, k, np, kp, false, hb);
  pad_host(c, m, n, mp, np, false, hc);
  std::lock_guard<std::mutex> lk(g_scratch.mu);
  const size_t need = sizeof(double) * (mp * kp + np * kp + mp * np) + sizeof(GemmJob);
  PL_TRY(g_scratch.ensure(need));
  double* da = static_cast<double*>(g_scratch.p);
  double* db = da + mp * kp;
  double* dc = db + np * kp;
  GemmJob* dj = reinterpret_cast<GemmJob*>(dc + mp * np);
  PL_TRY(cudaMemcpy(da, ha.data(), sizeof(double) * ha.size(), cudaMemcpyHostToDevice));
  PL_TRY(cudaMemcpy(db, hb.data(), sizeof(double) * hb.size(), cudaMemcpyHostToDevice));
  PL_TRY(cudaMemcpy(dc, hc.data(), sizeof(double) * hc.size(), cudaMemcpyHostToDevice));
  GemmJob j{};
  j.A = da;
  j.B = db;
  j.Cin = j.Cout = dc;
  j.K = static_cast<int>(kp);
  PL_TRY(cudaMemcpy(dj, &j, sizeof(j), cudaMemcpyHostToDevice));
  GemmParams p{};
  p.jobs = dj;
  p.njobs = 1;
  p.mblk = static_cast<int>(mp / GBM);
  p.nblk = static_cast<int>(np / GBN);
  p.lda = kp;
  p.ldb = kp;
  p.ldc = np;
  p.a_ktile = p.b_ktile = int64_t(1) << 40;
  p.a_base = da;
  p.a_extent = mp * kp;
  p.b_base = db;
  p.b_extent = np * kp;
  p.alpha = -1.0;
  p.beta = 1.0;
  PL_TRY(launch_gemm(p, true, true, EPI_AXPBY, 0));
  PL_TRY(cudaDeviceSynchronize());
  for (int64_t r = 0; r < m; ++r)
    PL_TRY(cudaMemcpy(out + r * n, dc + r * np, sizeof(double) * n, cudaMemcpyDeviceToHost));
  return GPB_OK;
}

}  // namespace

extern "C" {

int gpb_tile_potrf(gpb_ctx* ctx, const double* a, int64_t b, double* out) {
  if (!ctx || ctx != gpb_current()) return gpb_plugin_fail(GPB_NOT_RUNNING, "runtime is not running");
  if (b < 1) return gpb_plugin_fail(GPB_DIM, "potrf needs a non-empty square tile");
  const int64_t bp = rup(b, 128);
  std::vector<double> h;
  pad_host(a, b, b, bp, bp, true, h);
  std::lock_guard<std::mutex> lk(g_scratch.mu);
  PL_TRY(g_scratch.ensure(sizeof(double) * 2 * bp * bp + 64));
  double* dt = static_cast<double*>(g_scratch.p);
  double* dd = dt + bp * bp;
  int* info = reinterpret_cast<int*>(dd + bp * bp);
  PL_TRY(cudaMemcpy(dt, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice));
  PL_TRY(cudaMemset(info, 0xff, sizeof(int)));
  PotrfArgs pa{};
  pa.tile = dt;
  pa.dinv = dd;
  pa.logdiag = nullptr;
  pa.info = info;
  pa.bi = static_cast<int>(bp);
  pa.tile_off = 0;
  pa.bp_user = static_cast<int>(bp);
  pa.b_user = static_cast<int>(b);
  pa.trtri_only = 0;
  PL_TRY(launch_potrf(pa, 0));
  PL_TRY(cudaDeviceSynchronize());
  int hinfo = -1;
  PL_TRY(cudaMemcpy(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost));
  if (hinfo >= 0) {
    std::string msg = "Matrix is not positive definite (pivot at index " + std::to_string(hinfo) + ")";
    return gpb_plugin_fail(GPB_NOT_PD, msg.c_str());
  }
  for (int64_t r = 0; r < b; ++r)
    PL_TRY(cudaMemcpy(out + r * b, dt + r * bp, sizeof(double) * b, cudaMemcpyDeviceToHost));
  return GPB_OK;
}

int gpb_tile_trsm(gpb_ctx* ctx, const double* l, const double* b_in, int64_t rows, int64_t b,
                  double* out) {
  if (!ctx || ctx != gpb_current()) return gpb_plugin_fail(GPB_NOT_RUNNING, "runtime is not running");
  for (int64_t i = 0; i < b; ++i)
    if (l[i * b + i] == 0.0)
      return gpb_plugin_fail(GPB_SINGULAR, "triangular factor has a zero diagonal entry");
  const int64_t bp = rup(b, 128);
  std::vector<double> hl;
  pad_host(l, b, b, bp, bp, true, hl);
  // Dinv = l^-1 via the TRTRI-only mode of the tile kernel
  std::vector<double> dinv(bp * bp);
  {
    std::lock_guard<std::mutex> lk(g_scratch.mu);
    PL_TRY(g_scratch.ensure(sizeof(double) * 2 * bp * bp + 64));
    double* dt = static_cast<double*>(g_scratch.p);
    double* dd = dt + bp * bp;
    int* info = reinterpret_cast<int*>(dd + bp * bp);
    PL_TRY(cudaMemcpy(dt, hl.data(), sizeof(double) * hl.size(), cudaMemcpyHostToDevice));
    PL_TRY(cudaMemset(info, 0xff, sizeof(int)));
    PotrfArgs pa{};
    pa.tile = dt;
    pa.dinv = dd;
    pa.info = info;
    pa.bi = static_cast<int>(bp);
    pa.bp_user = static_cast<int>(bp);
    pa.b_user = static_cast<int>(b);
    pa.trtri_only = 1;
    PL_TRY(launch_potrf(pa, 0));
    PL_TRY(cudaDeviceSynchronize());
    PL_TRY(cudaMemcpy(dinv.data(), dd, sizeof(double) * bp * bp, cudaMemcpyDeviceToHost));
  }
  // X = b_in Dinv^T  ==  0 - b_in (-Dinv)^T
  std::vector<double> negd(b * b), zero(rows * b, 0.0);
  for (int64_t r = 0; r < b; ++r)
    for (int64_t c = 0; c < b; ++c) negd[r * b + c] = -dinv[r * bp + c];
  return run_gemm_nt(b_in, negd.data(), zero.data(), rows, b, b, out);
}

int gpb_tile_syrk(gpb_ctx* ctx, const double* a, const double* c, int64_t b, int64_t k, double* out) {
  if (!ctx || ctx != gpb_current()) return gpb_plugin_fail(GPB_NOT_RUNNING, "runtime is not running");
  return run_gemm_nt(a, a, c, b, b, k, out);
}

int gpb_tile_gemm(gpb_ctx* ctx, const double* a, const double* bm, const double* c, int64_t m,
                  int64_t n, int64_t k, double* out) {
  if (!ctx || ctx != gpb_current()) return gpb_plugin_fail(GPB_NOT_RUNNING, "runtime is not running");
  return run_gemm_nt(a, bm, c, m, n, k, out);
}

}  // extern "C"
