// Host runtime + C ABI (include/gpb200.h) of the B200 tiled-GP hot path.
//
// This is the native replacement of the reference's model layer
// (taskgp model.py:91-485) and its task runtime (runtime.py): instead of
// a Python work-stealing DAG of per-tile tasks, each algorithmic step is one
// grouped launch on a CUDA stream, and whole phases run without host
// round-trips.  Plans (the per-step GEMM job lists) are built once per model
// shape and kept resident in HBM.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "gemm.cuh"
#include "ozaki.cuh"
#include "gpb200.h"
#include "kernels.cuh"
#include "plan_common.h"

using namespace gpb;

extern "C" void gpb_dev_release_ring(void);  // dev_api.cu

namespace {

thread_local std::string g_err;
std::mutex g_mu;
gpb_ctx* g_ctx = nullptr;
uint64_t g_gen = 0;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(x)                                                                 \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      return fail(e_ == cudaErrorMemoryAllocation ? GPB_NO_MEMORY : GPB_CUDA,       \
                  std::string(#x) + ": " + cudaGetErrorString(e_));                 \
    }                                                                               \
  } while (0)

#define GPB_TRY(x)                \
  do {                            \
    int s_ = (x);                 \
    if (s_ != GPB_OK) return s_;  \
  } while (0)

constexpr double kHalfLog2Pi = 0.91893853320467274178;  // 0.5 * log(2 pi), model.py:35
constexpr double kVarianceSlack = 1e-9;                  // model.py:33

// Device-memory cache shared by all models of the process: model creation and
// destruction (and plan resizes) reuse blocks instead of paying cudaMalloc /
// cudaFree (which synchronises the device) on every small call.  A block is
// handed out again only after a device synchronisation at release, so no
// pending kernel can still touch it, and only to an allocation on the GPU it
// lives on.  Cached blocks are returned to CUDA when an allocation fails and
// at gpb_finalize.
struct BlockCache {
  struct Block {
    void* p;
    int device;
  };
  std::mutex mu;
  std::multimap<size_t, Block> free_blocks;  // capacity -> block
  size_t cached = 0;

  cudaError_t alloc(size_t n, void** p, size_t* cap, int* device) {
    int dev = 0;
    cudaGetDevice(&dev);
    *device = dev;
    {
      std::lock_guard<std::mutex> lk(mu);
      const size_t limit = std::max(2 * n, n + (size_t(1) << 20));
      for (auto it = free_blocks.lower_bound(n); it != free_blocks.end() && it->first <= limit; ++it) {
        if (it->second.device != dev) continue;
        *p = it->second.p;
        *cap = it->first;
        cached -= it->first;
        free_blocks.erase(it);
        return cudaSuccess;
      }
    }
    cudaError_t e = cudaMalloc(p, n);
    if (e == cudaErrorMemoryAllocation) {
      cudaGetLastError();
      trim();
      e = cudaMalloc(p, n);
    }
    if (e == cudaSuccess) *cap = n;
    return e;
  }
  // keep: false when the owning runtime is gone (the block is freed, not cached)
  void release(void* p, size_t cap, int device, bool keep) {
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != device) cudaSetDevice(device);
    if (!keep) {
      cudaFree(p);
    } else {
      cudaDeviceSynchronize();
      std::lock_guard<std::mutex> lk(mu);
      free_blocks.emplace(cap, Block{p, device});
      cached += cap;
    }
    if (cur != device) cudaSetDevice(cur);
  }
  void trim() {
    std::lock_guard<std::mutex> lk(mu);
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto& kv : free_blocks) {
      cudaSetDevice(kv.second.device);
      cudaFree(kv.second.p);
    }
    cudaSetDevice(cur);
    free_blocks.clear();
    cached = 0;
  }
};
BlockCache g_cache;

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;  // capacity
  int device = 0;
  template <class T>
  T* as() const { return static_cast<T*>(p); }
  cudaError_t ensure(size_t nbytes) {
    if (nbytes <= bytes && p) return cudaSuccess;
    release();
    void* q = nullptr;
    size_t cap = 0;
    cudaError_t e = g_cache.alloc(std::max<size_t>(nbytes, 16), &q, &cap, &device);
    if (e == cudaSuccess) {
      p = q;
      bytes = cap;
    }
    return e;
  }
  void release(bool keep = true) {
    if (p) g_cache.release(p, bytes, device, keep);
    p = nullptr;
    bytes = 0;
  }
};

int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// Allocation of an OPTIONAL buffer (digit planes: the FP64 DMMA kernels compute the same
// products without them): false, with the CUDA error cleared, when the memory is not there.
bool ensure_optional(DevBuf& b, size_t nbytes) {
  if (getenv("GPB_PLANES_ALLOC_FAIL")) return false;  // tests: behave as if the memory were not there
  if (b.ensure(nbytes) == cudaSuccess) return true;
  cudaGetLastError();
  return false;
}

}  // namespace

struct gpb_ctx {
  int device = 0;
  uint64_t gen = 0;
  cudaStream_t stream = nullptr;
  std::mutex tile_mu;  // tile plugin calls share scratch
  // pinned staging of the dense factor export (two strips), allocated on first use
  std::mutex export_mu;
  char* pinned = nullptr;
  size_t pinned_bytes = 0;
  cudaEvent_t strip_ev[2] = {nullptr, nullptr};
};

// One group of panels of the factorisation plan (build_chol_plan): job ranges
// in the model's job array.
struct CholGroup {
  int k0, np;
  int64_t trsm_off[kMaxGroup], trsm_cnt[kMaxGroup], in_off[kMaxGroup], in_cnt[kMaxGroup];
  // left-looking in-group updates (digit-plane path): column k0 + g from the g panels before it
  int64_t ll_off[kMaxGroup], ll_cnt[kMaxGroup];
  double ll_fl[kMaxGroup];
  int64_t next_off, next_cnt, upd_off, upd_cnt;
  double trsm_fl[kMaxGroup], in_fl[kMaxGroup], next_fl, upd_fl;  // executed flops per launch
};

struct gpb_model {
  gpb_ctx* ctx = nullptr;
  uint64_t gen = 0;
  int64_t n = 0, d = 0, T = 0;
  int b = 0, bi = 0, Ti = 0;
  int64_t np_ = 0;
  PadMap pm{};
  double l = 1.0, nu = 1.0, s2 = 0.1;
  uint8_t trainable[3] = {1, 1, 1};
  cudaStream_t st = nullptr;    // main stream (trailing updates, solves, prediction)
  cudaStream_t crit = nullptr;  // high-priority stream: the factorisation's critical path
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  std::vector<cudaEvent_t> sync_ev;  // cross-stream dependencies (timing disabled)

  DevBuf zp, yp, L, Dinv, scratch, logdiag, info, yhat, beta, alpha, bhat, red, tile_rm, tile_cm,
      chol_jobs, flow_flags;
  int flow_R = -1;  // slice height of the one-launch solves (0: multi-launch path)
  int G = 2;  // panels per trailing-update group (GPB_PANELS)
  std::vector<CholGroup> groups;
  std::vector<double> chol_flops_exec;
  bool plan_ok = false, factor_ok = false, weights_ok = false;
  int64_t last_pivot = -1;

  // gradient
  DevBuf X, Kinv, part_l, part_v, part_x, inv_jobs;
  DevBuf gp_panel, gp_h, gp_jobs, gp_tiles;  // column-panel gradient terms (multi-GPU split)
  std::vector<int64_t> invx_off;            // F_k
  std::vector<int64_t> urow_off, urow_cnt;  // U_k on row k + 1 (the lookahead row)
  std::vector<int64_t> urest_off, urest_cnt;  // U_k on rows > k + 1
  std::vector<double> urow_fl, urest_fl;
  std::vector<cudaEvent_t> grad_ev;         // [k] X(k, .) final (crit), [Ti + k] U_k rows > k+1 (main)
  double kinv_fl = 0.0;
  int64_t kinv_off = 0, kinv_cnt = 0;
  bool inv_plan = false;

  // prediction
  DevBuf Bv, W, mpart, sq, pred_jobs, zt, mean, var, S, fc_jobs;
  int64_t pred_mcp = -1, fc_mcp = -1;

  // tcgen05 digit-plane products (ozaki.cuh): planes of the off-diagonal L
  // tiles (same packing as L) and of V^T (one row per test point)
  DevBuf Ls, Vs, ozflag;
  // ... and of the solved panels of the current group (same element order as
  // `scratch`), read by the trailing updates NEXT / UPD of the factorisation
  DevBuf Ps, oz_jobs, fc_oz_jobs, Xs, kinv_oz_jobs;  // Xs: planes of X = L^-1 (gradient)
  std::vector<int64_t> kinv_oz_off, kinv_oz_cnt;  // per k segment of kOzakiMaxK: job range
  int64_t oz_grad_min_n = 4096;                   // K^-1 = X^T X on the planes from this n
  // left-looking X = L^-1 on the planes (from oz_llx_min_tiles internal tiles): per row i and k
  // segment the product jobs, per row the tiles to slice into Xs
  DevBuf llx_jobs, llx_slices;
  std::vector<std::vector<int64_t>> llx_off, llx_cnt;
  std::vector<int64_t> llx_slice_off;
  std::vector<OzakiSliceJob> llx_slices_host;  // `planes` = byte offset into Xs until uploaded
  const void* llx_slices_base = nullptr;       // the Xs the uploaded table points into
  std::vector<double> llx_fl;
  int oz_llx_min_tiles = 16;
  bool grad_fp64_only = false;  // transient: repeat of a gradient whose digits saturated
  bool vs_ok = false;  // Vs holds the planes of every row block of the current V (Bv)
  int64_t oz_chol_min_k = 512;  // updates with a shorter K = np * bi stay on the DMMA kernel
  bool oz_chol = true;           // GPB_OZAKI_CHOL=0: digit planes for the prediction sweep only
  bool oz_chol_in = true;        // GPB_OZAKI_CHOL_IN=0: in-group updates (K = bi) stay on the DMMA kernel
  int64_t oz_chol_in_min_k = 512;
  int oz_slices = 8;   // planes per operand (GPB_OZAKI; 0: every product on the FP64 DMMA kernels)
  bool ls_ok = false;  // Ls holds the planes of the current factor
  double oz_sa = 0.0, oz_sb = 0.0;
  int64_t oz_min_k = 2048;  // shorter products stay on the DMMA kernels
  int64_t oz_fallbacks = 0;

  double adam_m[3] = {0, 0, 0}, adam_v[3] = {0, 0, 0};
  int64_t adam_step = 0;
  double timing[8] = {0};
  int64_t launches = 0;
  long long* potrf_prof = nullptr;

  // per-kernel-class profiling (CUDA events around each launch on st)
  struct ProfRec {
    int cls;
    double flops;
    cudaEvent_t a, b;
  };
  bool prof = false;
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> evpool;
  size_t evnext = 0;
  cudaEvent_t prof_ref = nullptr;  // time origin of the launch intervals (on st)
  double cls_ms[8] = {0}, cls_flops[8] = {0}, cls_busy[8] = {0};
  int64_t cls_n[8] = {0};
};

namespace {

int check_live(gpb_model* m) {
  if (!m) return fail(GPB_INVALID_CONFIG, "null model");
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_ctx || g_ctx != m->ctx || g_ctx->gen != m->gen)
    return fail(GPB_NOT_RUNNING, "the runtime this model was bound to is not running");
  return GPB_OK;
}

// Internal layout (dev_api.cu gpb_layout): the internal tile size is a free
// parameter (results are tiling-invariant to round-off,
// test_acceptance.py:135-169); when 128 does not divide the user tile, n is
// padded once at the end with decoupled identity rows.
// Panels per trailing-update group.  On the DMMA kernels: plan_common.h (shared
// with the multi-GPU schedule).  With the updates on the int8 pipe a longer
// K = G bi amortises the block prologue / epilogue of the digit-plane product
// and the in-group updates cost little there: 8 panels from 48 tiles (config
// 2: 168.5 -> 162.7 ms against G = 4), 4 from 16.
int choose_panels(const gpb_model* m) {
  const int g = chol_panels(m->Ti);
  if (getenv("GPB_PANELS") || m->oz_slices == 0 || !m->oz_chol) return g;
  return m->Ti >= 48 ? 8 : m->Ti >= 16 ? 4 : g;
}

int apply_layout(gpb_model* m) {
  int64_t lay[6];
  if (int s = gpb_layout(m->n, m->T, lay)) return s;
  m->bi = static_cast<int>(lay[0]);
  m->Ti = static_cast<int>(lay[1]);
  m->np_ = lay[2];
  m->pm.bp_user = static_cast<int>(lay[3]);
  m->pm.b_user = static_cast<int>(lay[4]);
  m->G = choose_panels(m);
  return GPB_OK;
}

GemmParams base_params(const GemmJob* jobs, int njobs, int mblk, int nblk, int64_t lda,
                       int64_t ldb, int64_t ldc, double alpha, double beta) {
  GemmParams p{};
  p.jobs = jobs;
  p.njobs = njobs;
  p.mblk = mblk;
  p.nblk = nblk;
  p.lda = lda;
  p.ldb = ldb;
  p.ldc = ldc;
  p.a_ktile = p.b_ktile = int64_t(1) << 40;
  p.a_kstride = p.b_kstride = 0;
  p.alpha = alpha;
  p.beta = beta;
  p.aux_ld = 0;
  return p;
}

// TMA operand views (gemm_tma.cu): the buffers every A / B pointer of the
// launch lies in; launches without them run the cp.async kernel
GemmParams views(GemmParams p, const void* a, size_t a_bytes, const void* b, size_t b_bytes) {
  p.a_base = static_cast<const double*>(a);
  p.a_extent = static_cast<int64_t>(a_bytes / sizeof(double));
  p.b_base = static_cast<const double*>(b);
  p.b_extent = static_cast<int64_t>(b_bytes / sizeof(double));
  return p;
}
GemmParams views(const GemmParams& p, const DevBuf& a, const DevBuf& b) {
  return views(p, a.p, a.bytes, b.p, b.bytes);
}

enum KernelClass { KC_GEMM = 0, KC_POTRF = 1, KC_SEK = 2, KC_SOLVE = 3, KC_OTHER = 4, KC_OZAKI = 5 };

cudaEvent_t prof_event(gpb_model* m) {
  if (m->evnext == m->evpool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    m->evpool.push_back(e);
  }
  return m->evpool[m->evnext++];
}

// Bracket one launch with events when profiling is on.
struct ProfScope {
  gpb_model* m;
  int cls;
  double flops;
  cudaStream_t s;
  cudaEvent_t a = nullptr;
  ProfScope(gpb_model* mm, int c, double f, cudaStream_t ss = nullptr)
      : m(mm), cls(c), flops(f), s(ss ? ss : mm->st) {
    if (m->prof) {
      a = prof_event(m);
      cudaEventRecord(a, s);
    }
  }
  ~ProfScope() {
    if (a) {
      cudaEvent_t b = prof_event(m);
      cudaEventRecord(b, s);
      m->recs.push_back({cls, flops, a, b});
    }
  }
};

// Sum of launch durations per kernel class, and the class's busy time: the
// length of the union of its launch intervals across the model's streams
// (launches on the critical and main streams overlap, so their durations do
// not add up to wall time).
int prof_collect(gpb_model* m) {
  if (m->recs.empty()) return GPB_OK;
  CUDA_TRY(cudaDeviceSynchronize());
  std::vector<std::pair<double, double>> iv[8];
  FILE* dump = getenv("GPB_PROF_DUMP") ? fopen(getenv("GPB_PROF_DUMP"), "a") : nullptr;
  for (auto& r : m->recs) {
    float ms = 0, t0 = 0, t1 = 0;
    cudaEventElapsedTime(&ms, r.a, r.b);
    m->cls_ms[r.cls] += ms;
    m->cls_flops[r.cls] += r.flops;
    m->cls_n[r.cls] += 1;
    if (m->prof_ref && cudaEventElapsedTime(&t0, m->prof_ref, r.a) == cudaSuccess &&
        cudaEventElapsedTime(&t1, m->prof_ref, r.b) == cudaSuccess)
      iv[r.cls].push_back({t0, t1});
    if (dump) fprintf(dump, "%d %.4f %.4f %.4g\n", r.cls, t0, t1, r.flops);
  }
  if (dump) fclose(dump);
  for (int c = 0; c < 8; ++c) {
    auto& v = iv[c];
    std::sort(v.begin(), v.end());
    double busy = 0.0, lo = 0.0, hi = -1.0;
    for (auto& x : v) {
      if (x.first > hi) {
        if (hi > lo) busy += hi - lo;
        lo = x.first;
        hi = x.second;
      } else {
        hi = std::max(hi, x.second);
      }
    }
    if (hi > lo) busy += hi - lo;
    m->cls_busy[c] += busy;
  }
  m->recs.clear();
  m->evnext = 0;
  return GPB_OK;
}

// executed flops of a grouped launch: 2 * 128 * 128 * K per computed block
double gemm_flops(int64_t blocks, int64_t K) { return 2.0 * GBM * GBN * double(blocks) * double(K); }

int gemm(gpb_model* m, const GemmParams& p, bool ak, bool bk, int epi, double flops,
         cudaStream_t s = nullptr) {
  if (p.njobs == 0) return GPB_OK;
  if (!s) s = m->st;
  ProfScope ps(m, KC_GEMM, flops, s);
  CUDA_TRY(launch_gemm(p, ak, bk, epi, s));
  ++m->launches;
  return GPB_OK;
}

int alloc_model_buffers(gpb_model* m) {
  const int64_t bi2 = int64_t(m->bi) * m->bi;
  const int64_t ntiles = int64_t(m->Ti) * (m->Ti + 1) / 2;
  CUDA_TRY(m->zp.ensure(sizeof(double) * m->np_ * m->d));
  CUDA_TRY(m->yp.ensure(sizeof(double) * m->np_));
  CUDA_TRY(m->L.ensure(sizeof(double) * ntiles * bi2));
  CUDA_TRY(m->Dinv.ensure(sizeof(double) * m->Ti * bi2));
  CUDA_TRY(m->scratch.ensure(sizeof(double) * 2 * m->G * std::max<int64_t>(1, m->Ti - 1) * bi2));
  CUDA_TRY(m->logdiag.ensure(sizeof(double) * m->Ti));
  CUDA_TRY(m->info.ensure(sizeof(int) * 4));
  for (DevBuf* v : {&m->yhat, &m->beta, &m->alpha, &m->bhat}) CUDA_TRY(v->ensure(sizeof(double) * m->np_));
  CUDA_TRY(m->red.ensure(sizeof(double) * 16));
  // tile tables
  std::vector<int2> rm(ntiles), cm(ntiles);
  for (int i = 0; i < m->Ti; ++i)
    for (int j = 0; j <= i; ++j) {
      rm[h_tri_rm(i, j)] = make_int2(i, j);
      cm[h_tri_cm(i, j, m->Ti)] = make_int2(i, j);
    }
  CUDA_TRY(m->tile_rm.ensure(sizeof(int2) * ntiles));
  CUDA_TRY(m->tile_cm.ensure(sizeof(int2) * ntiles));
  CUDA_TRY(cudaMemcpy(m->tile_rm.p, rm.data(), sizeof(int2) * ntiles, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(m->tile_cm.p, cm.data(), sizeof(int2) * ntiles, cudaMemcpyHostToDevice));
  return GPB_OK;
}

// Cholesky plan: panels are factored in groups of G (GPB_PANELS; default 6 for
// T >= 96 internal tiles, 4 for T >= 48, else 2)
// and the trailing matrix is updated once per group with K = G * bi, which
// halves the read-modify-write passes over C at G = 2.  For group s
// (panels k0 .. k0+G'-1), with the panels solved into scratch set s % 2:
//   TRSM(k):  X_i = L(i,k) Dinv_k^T, i > k                      (critical stream)
//   IN(k):    L(i,j) -= X_i X_j^T for k < j < k0+G', i >= j      (critical, K = bi)
//   NEXT(s):  L(i,j) -= [X]_i [X]_j^T for the next group's columns (critical, K = G' bi)
//   UPD(s):   L(i,j) -= [X]_i [X]_j^T for all later columns      (main stream, K = G' bi)
// [X]_i concatenates row i of the group's panels, walked in k without a copy.
// POTRF/TRSM/IN/NEXT of group s+1 overlap the big trailing update of group s.
int build_chol_plan(gpb_model* m) {
  const int Ti = m->Ti, G = m->G, bi = m->bi;
  const int64_t bi2 = int64_t(bi) * bi;
  const int64_t pstride = std::max(1, Ti - 1) * bi2;  // doubles between panel buffers
  double* L = m->L.as<double>();
  double* D = m->Dinv.as<double>();
  std::vector<GemmJob> jobs;
  std::vector<OzakiJob> ozjobs;  // same indices as `jobs`; meaningful for NEXT / UPD entries
  m->groups.clear();
  // plan_common.h; with the updates on the int8 pipe and a large grid: tail r / 4, full first
  // group (config 2: 147.5 -> 138.7 ms)
  const bool planes_grid = m->oz_slices > 0 && m->oz_chol && Ti >= 48;
  const std::vector<int> sizes = planes_grid ? chol_group_sizes(Ti, G, 4, 0) : chol_group_sizes(Ti, G);
  for (int k0 = 0, s = 0; k0 < Ti; k0 += sizes[s], ++s) {
    CholGroup grp{};
    grp.k0 = k0;
    grp.np = sizes[s];
    double* set = m->scratch.as<double>() + int64_t(s % 2) * G * pstride;
    auto panel_tile = [&](int g, int i) { return set + g * pstride + int64_t(i - (k0 + g) - 1) * bi2; };
    for (int g = 0; g < grp.np; ++g) {
      const int k = k0 + g;
      grp.trsm_off[g] = jobs.size();
      // Dinv_k is lower triangular: output column block c only needs k < (c+1)*128
      for (int i = k + 1; i < Ti; ++i)
        for (int c = 0; c < bi / GBN; ++c) {
          GemmJob j{};
          j.A = L + h_tri_rm(i, k) * bi2;
          j.B = D + int64_t(k) * bi2 + int64_t(c) * GBN * bi;
          j.Cout = panel_tile(g, i) + c * GBN;
          j.K = (c + 1) * GBN;
          jobs.push_back(j);
        }
      grp.trsm_cnt[g] = jobs.size() - grp.trsm_off[g];
      grp.in_off[g] = jobs.size();
      for (int jj = k + 1; jj < k0 + grp.np; ++jj)
        for (int i = jj; i < Ti; ++i) {
          GemmJob j{};
          j.A = panel_tile(g, i);
          j.B = panel_tile(g, jj);
          j.Cin = j.Cout = L + h_tri_rm(i, jj) * bi2;
          j.K = bi;
          j.lower = (i == jj);
          jobs.push_back(j);
          // the same update from the planes of panel g alone (K = bi: one tile)
          OzakiJob o{};
          const int64_t tile_b = bi2 * m->oz_slices, panel_b = int64_t(std::max(1, Ti - 1)) * tile_b;
          o.a_off = (int64_t(s % 2) * G + g) * panel_b + int64_t(i - k0 - 1) * tile_b;
          o.b_off = (int64_t(s % 2) * G + g) * panel_b + int64_t(jj - k0 - 1) * tile_b;
          o.C = j.Cout;
          o.lower = j.lower;
          ozjobs.resize(jobs.size());
          ozjobs.back() = o;
        }
      grp.in_cnt[g] = jobs.size() - grp.in_off[g];
    }
    // trailing updates with the whole group (tiled-k walk across the G panels)
    const int c_next = k0 + grp.np;
    const int c_upd = std::min(Ti, c_next + (s + 1 < static_cast<int>(sizes.size()) ? sizes[s + 1] : 0));
    // job order = launch order of the blocks.  With the planes, tiles go in 2 x 2 super-tiles
    // (GPB_UPD_RASTER) so that the CTAs running together share A and B panel rows in L2: the
    // first trailing update reads 21% less from DRAM (26.6 -> 21.3 and 15.0 -> 10.5 GB in the
    // two windows); its time does not change (it is not DRAM-bound), nor do the results.
    static const int raster_env = [] {
      const char* e = getenv("GPB_UPD_RASTER");
      return e ? std::max(1, atoi(e)) : 0;
    }();
    const int raster = raster_env ? raster_env : (m->oz_slices > 0 && m->oz_chol ? 2 : 1);
    auto add_upd = [&](int jlo, int jhi) {
      std::vector<std::pair<int, int>> order;
      for (int i = jlo; i < Ti; ++i)
        for (int jj = jlo; jj <= std::min(i, jhi - 1); ++jj) order.emplace_back(i, jj);
      if (raster > 1)
        std::stable_sort(order.begin(), order.end(), [raster](const std::pair<int, int>& a, const std::pair<int, int>& b) {
          const int ai = a.first / raster, aj = a.second / raster, bi_ = b.first / raster, bj = b.second / raster;
          return ai != bi_ ? ai < bi_ : aj < bj;
        });
      for (const auto& ij : order) {
        const int i = ij.first, jj = ij.second;
        {
          GemmJob j{};
          j.A = panel_tile(0, i);
          j.B = panel_tile(0, jj);
          j.Cin = j.Cout = L + h_tri_rm(i, jj) * bi2;
          j.K = grp.np * bi;
          j.lower = (i == jj);
          jobs.push_back(j);
          // byte offsets into the panel planes (ensure_factor): tile slot of panel 0 of the set
          OzakiJob o{};
          const int64_t tile_b = bi2 * m->oz_slices, panel_b = int64_t(std::max(1, Ti - 1)) * tile_b;
          o.a_off = int64_t(s % 2) * G * panel_b + int64_t(i - k0 - 1) * tile_b;
          o.b_off = int64_t(s % 2) * G * panel_b + int64_t(jj - k0 - 1) * tile_b;
          o.C = j.Cout;
          o.lower = j.lower;
          ozjobs.resize(jobs.size());
          ozjobs.back() = o;
        }
      }
    };
    // LL(g): L(i, k0+g) -= [X]_i [X]_{k0+g}^T over panels 0 .. g-1 of the group (K = g bi):
    // what the right-looking IN launches add up to for that column, in one product
    for (int g = 1; g < grp.np; ++g) {
      grp.ll_off[g] = jobs.size();
      const int k = k0 + g;
      for (int i = k; i < Ti; ++i) {
        GemmJob j{};
        j.A = panel_tile(0, i);
        j.B = panel_tile(0, k);
        j.Cin = j.Cout = L + h_tri_rm(i, k) * bi2;
        j.K = g * bi;
        j.lower = (i == k);
        jobs.push_back(j);
        OzakiJob o{};
        const int64_t tile_b = bi2 * m->oz_slices, panel_b = int64_t(std::max(1, Ti - 1)) * tile_b;
        o.a_off = int64_t(s % 2) * G * panel_b + int64_t(i - k0 - 1) * tile_b;
        o.b_off = int64_t(s % 2) * G * panel_b + int64_t(k - k0 - 1) * tile_b;
        o.C = j.Cout;
        o.lower = j.lower;
        ozjobs.resize(jobs.size());
        ozjobs.back() = o;
      }
      grp.ll_cnt[g] = jobs.size() - grp.ll_off[g];
    }
    grp.next_off = jobs.size();
    add_upd(c_next, c_upd);
    grp.next_cnt = jobs.size() - grp.next_off;
    grp.upd_off = jobs.size();
    add_upd(c_upd, Ti);
    grp.upd_cnt = jobs.size() - grp.upd_off;
    // executed flops of each launch (profiling): 2*128*128*K per computed block
    const int nb = bi / GBM;
    auto fl = [&](int64_t off, int64_t cnt, int blocks_per_job) {
      double f = 0.0;
      for (int64_t q = off; q < off + cnt; ++q)
        f += 2.0 * GBM * GBN * double(jobs[q].K) *
             (jobs[q].lower ? nb * (nb + 1) / 2 : blocks_per_job);
      return f;
    };
    for (int g = 0; g < grp.np; ++g) {
      grp.trsm_fl[g] = fl(grp.trsm_off[g], grp.trsm_cnt[g], nb);
      grp.in_fl[g] = fl(grp.in_off[g], grp.in_cnt[g], nb * nb);
      grp.ll_fl[g] = g ? fl(grp.ll_off[g], grp.ll_cnt[g], nb * nb) : 0.0;
    }
    grp.next_fl = fl(grp.next_off, grp.next_cnt, nb * nb);
    grp.upd_fl = fl(grp.upd_off, grp.upd_cnt, nb * nb);
    m->groups.push_back(grp);
  }
  CUDA_TRY(m->chol_jobs.ensure(sizeof(GemmJob) * std::max<size_t>(1, jobs.size())));
  if (!jobs.empty())
    CUDA_TRY(cudaMemcpy(m->chol_jobs.p, jobs.data(), sizeof(GemmJob) * jobs.size(),
                        cudaMemcpyHostToDevice));
  ozjobs.resize(jobs.size());
  CUDA_TRY(m->oz_jobs.ensure(sizeof(OzakiJob) * std::max<size_t>(1, ozjobs.size())));
  if (!ozjobs.empty())
    CUDA_TRY(cudaMemcpy(m->oz_jobs.p, ozjobs.data(), sizeof(OzakiJob) * ozjobs.size(),
                        cudaMemcpyHostToDevice));
  m->chol_flops_exec.assign(m->groups.size(), 0.0);
  // cross-stream events: per group "panels solved" and "trailing update done"
  const size_t ng = m->groups.size();
  while (m->sync_ev.size() < 2 * ng + 2) {
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    m->sync_ev.push_back(e);
  }
  m->plan_ok = true;
  return GPB_OK;
}

SekParams sek_params(const gpb_model* m) {
  SekParams sp;
  sp.lengthscale = m->l;
  sp.vertical = m->nu;
  sp.noise = m->s2;
  sp.neg_half_inv_l2 = -1.0 / (2.0 * (m->l * m->l));
  return sp;
}

int upload_train(gpb_model* m, const double* z, const double* y, bool device_ptrs) {
  // stage dense z, y on device, then scatter into the padded layout
  DevBuf zd, yd;
  const double* zsrc = z;
  const double* ysrc = y;
  if (!device_ptrs) {
    CUDA_TRY(zd.ensure(sizeof(double) * m->n * m->d));
    CUDA_TRY(yd.ensure(sizeof(double) * m->n));
    CUDA_TRY(cudaMemcpyAsync(zd.p, z, sizeof(double) * m->n * m->d, cudaMemcpyHostToDevice, m->st));
    CUDA_TRY(cudaMemcpyAsync(yd.p, y, sizeof(double) * m->n, cudaMemcpyHostToDevice, m->st));
    zsrc = zd.as<double>();
    ysrc = yd.as<double>();
  }
  CUDA_TRY(launch_pad_rows(zsrc, m->zp.as<double>(), m->np_, static_cast<int>(m->d), m->pm, m->st));
  CUDA_TRY(launch_pad_vector(ysrc, m->yp.as<double>(), m->np_, m->pm, m->st));
  m->launches += 2;
  CUDA_TRY(cudaStreamSynchronize(m->st));
  zd.release();
  yd.release();
  return GPB_OK;
}

void invalidate(gpb_model* m) {
  m->factor_ok = false;
  m->weights_ok = false;
  m->ls_ok = false;
}

struct PhaseTimer {
  gpb_model* m;
  int slot;
  PhaseTimer(gpb_model* mm, int s) : m(mm), slot(s) { cudaEventRecord(m->e0, m->st); }
  int stop() {
    cudaEventRecord(m->e1, m->st);
    CUDA_TRY(cudaEventSynchronize(m->e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, m->e0, m->e1);
    m->timing[slot] = ms;
    return GPB_OK;
  }
};

double plane_scale(double bound) { return ozaki_plane_scale(bound); }

// assemble + factor (model.py:169-177 _ensure_factor)
int ensure_factor(gpb_model* m) {
  if (m->factor_ok) return GPB_OK;
  if (!m->plan_ok) GPB_TRY(build_chol_plan(m));
  const int Ti = m->Ti, bi = m->bi;
  const int64_t bi2 = int64_t(bi) * bi;
  const int64_t ntiles = int64_t(Ti) * (Ti + 1) / 2;
  double* L = m->L.as<double>();
  double* D = m->Dinv.as<double>();
  {
    PhaseTimer pt(m, 0);
    ProfScope ps(m, KC_SEK, 0.0);
    CUDA_TRY(launch_assemble_lower(L, m->tile_rm.as<int2>(), 0, ntiles, m->zp.as<double>(),
                                   static_cast<int>(m->d), bi, m->pm, sek_params(m), true, m->st));
    ++m->launches;
    GPB_TRY(pt.stop());
  }
  PhaseTimer pt(m, 1);
  CUDA_TRY(cudaMemsetAsync(m->info.p, 0xff, sizeof(int), m->st));
  const GemmJob* jobs = m->chol_jobs.as<GemmJob>();
  const int nb = bi / GBM;
  const int ng = static_cast<int>(m->groups.size());
  const int64_t pstride = std::max(1, Ti - 1) * bi2;
  cudaEvent_t* ev_panel = m->sync_ev.data();       // [s]: panels of group s solved (crit)
  cudaEvent_t* ev_upd = m->sync_ev.data() + ng;    // [s]: UPD(s) done (main)
  // the critical stream starts after the assembly/memset on the main stream
  CUDA_TRY(cudaEventRecord(ev_upd[ng], m->st));
  CUDA_TRY(cudaStreamWaitEvent(m->crit, ev_upd[ng], 0));
  auto walk = [&](GemmParams p) {  // [X]_i: tiled-k walk across the group's panels
    p = views(p, m->scratch, m->scratch);
    p.a_ktile = p.b_ktile = bi;
    p.a_kstride = p.b_kstride = pstride - bi2;
    return p;
  };
  // Trailing updates on the tcgen05 int8 pipe (ozaki.cuh): the solved panels
  // are final entries of L, |L(i, j)| <= sqrt(K_ii) = sqrt(vertical + noise)
  // (1 on the decoupled padding rows), so one fixed-point scale covers them.
  bool oz = m->oz_slices > 0 && m->oz_chol;
  // panel planes (boxed layout, ozaki.cuh): per scratch set and panel g of the
  // group, Ti - 1 tile slots of bi x bi; slot t of panel g holds L(k0 + 1 + t, k0 + g)
  const int S = m->oz_slices;
  const int64_t tile_bytes = bi2 * S, panel_bytes = int64_t(std::max(1, Ti - 1)) * tile_bytes;
  if (oz) {
    bool any = false;
    for (const CholGroup& grp : m->groups)
      any = any || (int64_t(grp.np) * bi >= m->oz_chol_min_k && grp.next_cnt + grp.upd_cnt > 0);
    oz = any;
  }
  if (oz && !ensure_optional(m->Ps, size_t(2) * m->G * panel_bytes)) oz = false;  // no room: DMMA
  if (oz) {
    if (!m->ozflag.p) {
      CUDA_TRY(m->ozflag.ensure(sizeof(int)));
      CUDA_TRY(cudaMemsetAsync(m->ozflag.p, 0, sizeof(int), m->st));
    }
    m->oz_sa = plane_scale(std::max(1.0, std::sqrt(m->nu + m->s2)));
  }
  // L(i,j) -= [X]_i [X]_j^T for `cnt` plan jobs from `off`
  auto oz_update = [&](int K, int64_t off, int64_t cnt, double flops, cudaStream_t s) -> int {
    OzakiGemm g{};
    g.a = g.b = {m->Ps.as<int8_t>(), panel_bytes, bi / kOzakiBK, int64_t(bi / kOzakiBK) * S * kOzakiBox};
    g.M = g.N = bi;
    g.K = K;
    g.slices = S;
    g.alpha = -m->oz_sa * m->oz_sa;
    g.beta = 1.0;
    g.ldc_in = g.ldc_out = bi;
    g.jobs = m->oz_jobs.as<OzakiJob>() + off;
    g.njobs = static_cast<int>(cnt);
    ProfScope ps(m, KC_OZAKI, flops, s);
    CUDA_TRY(launch_ozaki_gemm(g, s));
    m->launches += S > 4 ? 2 : 1;
    return GPB_OK;
  };
  for (int s = 0; s < ng; ++s) {
    const CholGroup& grp = m->groups[s];
    double* set = m->scratch.as<double>() + int64_t(s % 2) * m->G * pstride;
    const bool oz_grp = oz && int64_t(grp.np) * bi >= m->oz_chol_min_k && grp.next_cnt + grp.upd_cnt > 0;
    // in-group updates (K = bi) from the planes too when the group has them and bi is long enough
    const bool oz_in = oz_grp && m->oz_chol_in && bi >= m->oz_chol_in_min_k;
    // the group's columns are complete once NEXT(s-1) (crit, in order) and UPD(s-2) are done
    if (s >= 2) CUDA_TRY(cudaStreamWaitEvent(m->crit, ev_upd[s - 2], 0));
    for (int g = 0; g < grp.np; ++g) {
      const int k = grp.k0 + g;
      // digit-plane path: column k brought up to date from the group's earlier panels in one
      // product (K = g bi) instead of g right-looking updates with K = bi
      if (oz_in && g > 0) GPB_TRY(oz_update(g * bi, grp.ll_off[g], grp.ll_cnt[g], grp.ll_fl[g], m->crit));
      PotrfArgs a{};
      a.tile = L + h_tri_rm(k, k) * bi2;
      a.dinv = D + int64_t(k) * bi2;
      a.logdiag = m->logdiag.as<double>();
      a.info = m->info.as<int>();
      a.bi = bi;
      a.tile_index = k;
      a.tile_off = k * bi;
      a.bp_user = m->pm.bp_user;
      a.b_user = m->pm.b_user;
      a.prof = m->potrf_prof;
      a.tiles = Ti;
      a.remaining = Ti - k;
      {
        ProfScope ps(m, KC_POTRF, 2.0 / 3.0 * double(bi) * bi * bi, m->crit);
        CUDA_TRY(launch_potrf(a, m->crit));
      }
      ++m->launches;
      GemmParams tp = views(base_params(jobs + grp.trsm_off[g], static_cast<int>(grp.trsm_cnt[g]), nb, 1,
                                        bi, bi, bi, 1.0, 0.0),
                            m->L, m->Dinv);
      GPB_TRY(gemm(m, tp, true, true, EPI_AXPBY, grp.trsm_fl[g], m->crit));
      if (oz_grp) {  // digit planes of the solved panel
        ProfScope ps(m, KC_OTHER, 0.0, m->crit);
        int8_t* dst = m->Ps.as<int8_t>() + (int64_t(s % 2) * m->G + g) * panel_bytes + int64_t(g) * tile_bytes;
        CUDA_TRY(launch_ozaki_slice_tiles(set + g * pstride, Ti - k - 1, bi, bi, m->oz_sa, dst, S,
                                          m->ozflag.as<int>(), m->crit));
        ++m->launches;
      }
      if (grp.in_cnt[g] > 0 && !oz_in) {
        GemmParams ip = views(base_params(jobs + grp.in_off[g], static_cast<int>(grp.in_cnt[g]), nb, nb, bi,
                                          bi, bi, -1.0, 1.0),
                              m->scratch, m->scratch);
        GPB_TRY(gemm(m, ip, true, true, EPI_AXPBY, grp.in_fl[g], m->crit));
      }
    }
    CUDA_TRY(cudaEventRecord(ev_panel[s], m->crit));
    // lookahead: the next group's columns need UPD(s-1), which covered them
    if (grp.next_cnt > 0) {
      if (s >= 1) CUDA_TRY(cudaStreamWaitEvent(m->crit, ev_upd[s - 1], 0));
      if (oz_grp) {
        GPB_TRY(oz_update(grp.np * bi, grp.next_off, grp.next_cnt, grp.next_fl, m->crit));
      } else {
        GemmParams np = walk(base_params(jobs + grp.next_off, static_cast<int>(grp.next_cnt), nb, nb,
                                         bi, bi, bi, -1.0, 1.0));
        GPB_TRY(gemm(m, np, true, true, EPI_AXPBY, grp.next_fl, m->crit));
      }
    }
    // main stream: copy the panels back and apply the rest of the trailing update
    CUDA_TRY(cudaStreamWaitEvent(m->st, ev_panel[s], 0));
    for (int g = 0; g < grp.np; ++g) {
      CUDA_TRY(launch_copy_panel(L, set + g * pstride, Ti, grp.k0 + g, bi, m->st));
      ++m->launches;
    }
    if (grp.upd_cnt > 0) {
      if (oz_grp) {
        GPB_TRY(oz_update(grp.np * bi, grp.upd_off, grp.upd_cnt, grp.upd_fl, m->st));
      } else {
        GemmParams up = walk(base_params(jobs + grp.upd_off, static_cast<int>(grp.upd_cnt), nb, nb,
                                         bi, bi, bi, -1.0, 1.0));
        GPB_TRY(gemm(m, up, true, true, EPI_AXPBY, grp.upd_fl));
      }
    }
    CUDA_TRY(cudaEventRecord(ev_upd[s], m->st));
  }
  if (m->potrf_prof) {  // GPB_POTRF_PROF: per-phase cycles of the tile kernel (potrf.cu PROF_MARK)
    long long h[16];
    cudaStreamSynchronize(m->crit);
    cudaMemcpy(h, m->potrf_prof, sizeof(h), cudaMemcpyDeviceToHost);
    fprintf(stderr,
            "potrf cycles, chain warp (CTA 0): B-barrier %lld, critical wait + chain %lld, C-barrier %lld, "
            "trtri %lld, zero %lld | job warp 0 of CTA 1: B-jobs %lld, B-barrier %lld, C-jobs %lld, "
            "C-barrier %lld\n",
            h[1], h[5], h[2], h[3], h[4], h[13], h[9], h[15], h[10]);
    cudaMemset(m->potrf_prof, 0, sizeof(h));
  }
  // join: the main stream waits for the critical stream's last work
  CUDA_TRY(cudaEventRecord(m->sync_ev[2 * ng + 1], m->crit));
  CUDA_TRY(cudaStreamWaitEvent(m->st, m->sync_ev[2 * ng + 1], 0));
  GPB_TRY(pt.stop());
  int info = -1;
  CUDA_TRY(cudaMemcpy(&info, m->info.p, sizeof(int), cudaMemcpyDeviceToHost));
  if (oz) {
    // a panel entry beyond the fixed-point scale saturated its digits (only
    // possible for a matrix that is not positive definite, or never): the
    // factorisation is repeated on the DMMA kernels, which also report the pivot
    int over = 0;
    CUDA_TRY(cudaMemcpy(&over, m->ozflag.p, sizeof(int), cudaMemcpyDeviceToHost));
    if (over) {
      CUDA_TRY(cudaMemset(m->ozflag.p, 0, sizeof(int)));
      ++m->oz_fallbacks;
      const bool keep = m->oz_chol;
      m->oz_chol = false;
      const int st = ensure_factor(m);
      m->oz_chol = keep;
      return st;
    }
  }
  if (info >= 0) {
    m->last_pivot = info;
    invalidate(m);
    char buf[160];
    snprintf(buf, sizeof(buf), "Matrix is not positive definite (non-positive pivot at index %d)",
             info);
    return fail(GPB_NOT_PD, buf);
  }
  m->last_pivot = -1;
  m->factor_ok = true;
  m->weights_ok = false;
  m->ls_ok = false;
  return GPB_OK;
}

// beta = L^-1 y, alpha = L^-T beta (model.py:179-186)
int ensure_weights(gpb_model* m) {
  GPB_TRY(ensure_factor(m));
  if (m->weights_ok) return GPB_OK;
  const int Ti = m->Ti, bi = m->bi;
  const int64_t bi2 = int64_t(bi) * bi;
  double* L = m->L.as<double>();
  double* D = m->Dinv.as<double>();
  double* yhat = m->yhat.as<double>();
  double* beta = m->beta.as<double>();
  double* alpha = m->alpha.as<double>();
  double* bhat = m->bhat.as<double>();
  PhaseTimer pt(m, 2);
  if (m->flow_R < 0) {
    const char* fe = getenv("GPB_SOLVE_FLOW");
    m->flow_R = (fe && atoi(fe) == 0) ? 0 : solve_flow_slice_rows(m->np_, bi);
  }
  if (m->flow_R > 0) {
    bool launched = false;
    CUDA_TRY(m->flow_flags.ensure(solve_flow_scratch_bytes(Ti, bi)));
    {
      ProfScope ps(m, KC_SOLVE, 0.0);
      CUDA_TRY(launch_solve_flow(L, D, m->yp.as<double>(), beta, alpha, yhat, m->flow_flags.p, Ti,
                                 bi, m->flow_R, m->st, &launched));
    }
    if (launched) {
      m->launches += 1;
      GPB_TRY(pt.stop());
      m->weights_ok = true;
      return GPB_OK;
    }
    m->flow_R = 0;
  }
  CUDA_TRY(cudaMemcpyAsync(yhat, m->yp.p, sizeof(double) * m->np_, cudaMemcpyDeviceToDevice, m->st));
  for (int i = 0; i < Ti; ++i) {
    CUDA_TRY(launch_fwd_diag(D + i * bi2, yhat + int64_t(i) * bi, beta + int64_t(i) * bi, bi, m->st));
    CUDA_TRY(launch_fwd_update(L, Ti, i, bi, beta + int64_t(i) * bi, yhat, m->st));
    m->launches += 2;
  }
  CUDA_TRY(cudaMemcpyAsync(bhat, beta, sizeof(double) * m->np_, cudaMemcpyDeviceToDevice, m->st));
  for (int i = Ti - 1; i >= 0; --i) {
    CUDA_TRY(launch_bwd_diag(D + i * bi2, bhat + int64_t(i) * bi, alpha + int64_t(i) * bi, bi, m->st));
    CUDA_TRY(launch_bwd_update(L, i, bi, alpha + int64_t(i) * bi, bhat, m->st));
    m->launches += 2;
  }
  GPB_TRY(pt.stop());
  m->weights_ok = true;
  return GPB_OK;
}

int log_likelihood(gpb_model* m, double* out) {
  GPB_TRY(ensure_weights(m));
  CUDA_TRY(launch_loss_terms(m->logdiag.as<double>(), m->Ti, m->beta.as<double>(), m->np_,
                             m->red.as<double>(), m->st));
  ++m->launches;
  double h[2];
  CUDA_TRY(cudaMemcpyAsync(h, m->red.p, sizeof(h), cudaMemcpyDeviceToHost, m->st));
  CUDA_TRY(cudaStreamSynchronize(m->st));
  // model.py:335-337
  *out = -h[0] - 0.5 * h[1] - double(m->n) * kHalfLog2Pi;
  return GPB_OK;
}

// ---- gradient (model.py:341-435) ------------------------------------------
int build_inv_plan(gpb_model* m) {
  const int Ti = m->Ti;
  const int64_t bi2 = int64_t(m->bi) * m->bi;
  const int64_t ntiles = int64_t(Ti) * (Ti + 1) / 2;
  CUDA_TRY(m->X.ensure(sizeof(double) * ntiles * bi2));
  CUDA_TRY(m->Kinv.ensure(sizeof(double) * ntiles * bi2));
  const int64_t nblk = ntiles * (m->bi / kSekBlock) * (m->bi / kSekBlock);
  CUDA_TRY(m->part_l.ensure(sizeof(double) * nblk));
  CUDA_TRY(m->part_v.ensure(sizeof(double) * nblk));
  CUDA_TRY(m->part_x.ensure(sizeof(double) * nblk));
  double* L = m->L.as<double>();
  double* D = m->Dinv.as<double>();
  double* X = m->X.as<double>();
  double* Kv = m->Kinv.as<double>();
  std::vector<GemmJob> jobs;
  // X = L^-1 right-looking, with the K^-1 buffer as the accumulator
  // A(i, j) = -sum_{m=j}^{i-1} L(i, m) X(m, j):
  //   F_k: X(k, j) = Dinv_k A(k, j), j < k (row block r needs k < (r+1)*128)
  //   U_k: A(i, j) -= L(i, k) X(k, j), i > k, j <= k, one job per 128-column
  //        block of the output (K = bi; for j = k, X(k, k) = Dinv_k is lower
  //        triangular, so column block cb needs only K = bi - cb*128)
  // U_k is split into the lookahead row i = k + 1 (critical stream, followed by
  // F_{k+1}) and the rows i > k + 1 (main stream), like the factorisation
  // (the left-looking form put a K = i*bi job next to K = bi ones in one
  // launch: at config 1 the long jobs left most SMs idle)
  m->invx_off.assign(Ti + 1, 0);
  m->urow_off.assign(Ti + 1, 0);
  m->urow_cnt.assign(Ti + 1, 0);
  m->urest_off.assign(Ti + 1, 0);
  m->urest_cnt.assign(Ti + 1, 0);
  m->urow_fl.assign(Ti + 1, 0.0);
  m->urest_fl.assign(Ti + 1, 0.0);
  const int nbk = m->bi / GBN;
  auto add_u = [&](int k, int i, double* fl) {
    for (int j = 0; j <= k; ++j)
      for (int cb = 0; cb < nbk; ++cb) {
        const int64_t o = int64_t(cb) * GBN;
        GemmJob g{};
        if (j < k) {
          g.A = L + h_tri_rm(i, k) * bi2;
          g.B = X + h_tri_cm(k, j, Ti) * bi2 + o;
          g.Cin = g.Cout = Kv + h_tri_cm(i, j, Ti) * bi2 + o;
          g.K = m->bi;
        } else {
          g.A = L + h_tri_rm(i, k) * bi2 + o;
          g.B = X + h_tri_cm(k, k, Ti) * bi2 + o * m->bi + o;
          g.Cin = g.Cout = Kv + h_tri_cm(i, k, Ti) * bi2 + o;
          g.K = m->bi - static_cast<int>(o);
        }
        jobs.push_back(g);
        *fl += 2.0 * GBM * GBN * double(g.K) * (m->bi / GBM);
      }
  };
  for (int k = 0; k < Ti; ++k) {
    m->invx_off[k] = jobs.size();
    for (int j = 0; j < k; ++j)
      for (int r = 0; r < m->bi / GBM; ++r) {
        GemmJob g{};
        g.A = D + int64_t(k) * bi2 + int64_t(r) * GBM * m->bi;
        g.B = Kv + h_tri_cm(k, j, Ti) * bi2;
        g.Cout = X + h_tri_cm(k, j, Ti) * bi2 + int64_t(r) * GBM * m->bi;
        g.K = (r + 1) * GBM;
        jobs.push_back(g);
      }
    m->urow_off[k] = jobs.size();
    if (k + 1 < Ti) add_u(k, k + 1, &m->urow_fl[k]);
    m->urow_cnt[k] = jobs.size() - m->urow_off[k];
    m->urest_off[k] = jobs.size();
    for (int i = k + 2; i < Ti; ++i) add_u(k, i, &m->urest_fl[k]);
    m->urest_cnt[k] = jobs.size() - m->urest_off[k];
  }
  while (m->grad_ev.size() < size_t(2 * Ti + 1)) {
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    m->grad_ev.push_back(e);
  }
  // K^-1(r, c) = sum_{k >= r} X(k, r)^T X(k, c), one job per 128-row block rb
  // of the output: X(r, r) is lower triangular, so the k sum starts at row
  // rb*128 of the column panel; diagonal tiles only need the column blocks up
  // to rb (symmetric: the trace pass reads their lower triangle only)
  m->kinv_off = jobs.size();
  m->kinv_fl = 0.0;
  for (int r = 0; r < Ti; ++r)  // longest K first
    for (int c = 0; c <= r; ++c)
      for (int rb = 0; rb < m->bi / GBM; ++rb) {
        const int64_t o = int64_t(rb) * GBM;
        GemmJob g{};
        g.A = X + h_tri_cm(r, r, Ti) * bi2 + o * m->bi + o;
        g.B = X + h_tri_cm(r, c, Ti) * bi2 + o * m->bi;
        g.Cout = Kv + h_tri_cm(r, c, Ti) * bi2 + o * m->bi;
        g.K = (Ti - r) * m->bi - static_cast<int>(o);
        g.nlim = (r == c) ? rb + 1 : 0;
        jobs.push_back(g);
        m->kinv_fl += 2.0 * GBM * GBN * double(g.K) * (g.nlim ? g.nlim : m->bi / GBN);
      }
  m->kinv_cnt = jobs.size() - m->kinv_off;
  // The same product on the digit planes (ozaki.cuh): the planes of column panel c of X are
  // sliced transposed (operand row = column of the panel, k = row), chunk major, so every
  // panel has the same row-block stride; job (r, c) reads panel r from k = 0 and panel c
  // from k = (r - c) bi, K = (Ti - r) bi, in segments of kOzakiMaxK (exact int32 sums).
  {
    const int S = std::max(m->oz_slices, 1);
    const int nrb = m->bi / kOzakiBM;
    const int64_t chunk_b = int64_t(nrb) * S * kOzakiBox;  // bytes per k chunk of a panel
    const int64_t seg_chunks = kOzakiMaxK / kOzakiBK;
    std::vector<OzakiJob> oj;
    m->kinv_oz_off.clear();
    m->kinv_oz_cnt.clear();
    for (int64_t seg = 0; seg * kOzakiMaxK < int64_t(Ti) * m->bi; ++seg) {
      m->kinv_oz_off.push_back(static_cast<int64_t>(oj.size()));
      for (int r = 0; r < Ti; ++r) {  // longest K first
        const int64_t chunks = int64_t(Ti - r) * m->bi / kOzakiBK - seg * seg_chunks;
        if (chunks <= 0) continue;
        for (int c = 0; c <= r; ++c) {
          OzakiJob o{};
          o.a_off = h_tri_cm(r, r, Ti) * bi2 * S + seg * seg_chunks * chunk_b;
          o.b_off = h_tri_cm(c, c, Ti) * bi2 * S + (int64_t(r - c) * m->bi / kOzakiBK + seg * seg_chunks) * chunk_b;
          o.C = Kv + h_tri_cm(r, c, Ti) * bi2;
          o.lower = r == c;
          o.kchunks = static_cast<int>(std::min(chunks, seg_chunks));
          oj.push_back(o);
        }
      }
      m->kinv_oz_cnt.push_back(static_cast<int64_t>(oj.size()) - m->kinv_oz_off.back());
    }
    CUDA_TRY(m->kinv_oz_jobs.ensure(sizeof(OzakiJob) * std::max<size_t>(1, oj.size())));
    if (!oj.empty())
      CUDA_TRY(cudaMemcpy(m->kinv_oz_jobs.p, oj.data(), sizeof(OzakiJob) * oj.size(), cudaMemcpyHostToDevice));
    // Left-looking X = L^-1 on the planes: A(i, j) = -sum_{m=j}^{i-1} L(i, m) X(m, j) for row i in one
    // product per k segment (K = (i - j) bi: the planes of L's row panel from tile j against the planes
    // of column panel j of X from k = 0), then F_i, then row i's tiles are sliced into the X planes.
    std::vector<OzakiJob> lj;
    std::vector<OzakiSliceJob> sj;
    m->llx_off.assign(Ti, {});
    m->llx_cnt.assign(Ti, {});
    m->llx_slice_off.assign(Ti + 1, 0);
    m->llx_fl.assign(Ti, 0.0);
    const int64_t seg_tiles = kOzakiMaxK / m->bi;
    for (int i = 0; i < Ti; ++i) {
      for (int64_t seg = 0; seg * kOzakiMaxK < int64_t(i) * m->bi; ++seg) {
        m->llx_off[i].push_back(static_cast<int64_t>(lj.size()));
        for (int j = 0; j < i; ++j) {
          const int64_t chunks = int64_t(i - j) * m->bi / kOzakiBK - seg * seg_chunks;
          if (chunks <= 0) continue;
          OzakiJob o{};
          o.a_off = (h_tri_rm(i, 0) + j + seg * seg_tiles) * bi2 * S;
          o.b_off = h_tri_cm(j, j, Ti) * bi2 * S + seg * seg_chunks * chunk_b;
          o.C = Kv + h_tri_cm(i, j, Ti) * bi2;
          o.kchunks = static_cast<int>(std::min(chunks, seg_chunks));
          lj.push_back(o);
          if (seg == 0) m->llx_fl[i] += 2.0 * double(bi2) * double(i - j) * m->bi;
        }
        m->llx_cnt[i].push_back(static_cast<int64_t>(lj.size()) - m->llx_off[i].back());
      }
      m->llx_slice_off[i] = static_cast<int64_t>(sj.size());
      for (int j = 0; j <= i; ++j)
        sj.push_back(OzakiSliceJob{X + h_tri_cm(i, j, Ti) * bi2, m->Xs.as<int8_t>(), int64_t(i - j) * m->bi});
    }
    m->llx_slice_off[Ti] = static_cast<int64_t>(sj.size());
    // the plane pointers are filled in at launch time (Xs is allocated there): keep the panel
    // offsets in `planes` for now
    for (int i = 0, t = 0; i < Ti; ++i)
      for (int j = 0; j <= i; ++j, ++t)
        sj[t].planes = reinterpret_cast<int8_t*>(static_cast<intptr_t>(h_tri_cm(j, j, Ti) * bi2 * S));
    CUDA_TRY(m->llx_jobs.ensure(sizeof(OzakiJob) * std::max<size_t>(1, lj.size())));
    if (!lj.empty())
      CUDA_TRY(cudaMemcpy(m->llx_jobs.p, lj.data(), sizeof(OzakiJob) * lj.size(), cudaMemcpyHostToDevice));
    m->llx_slices_host = sj;
  }
  CUDA_TRY(m->inv_jobs.ensure(sizeof(GemmJob) * jobs.size()));
  CUDA_TRY(cudaMemcpy(m->inv_jobs.p, jobs.data(), sizeof(GemmJob) * jobs.size(),
                      cudaMemcpyHostToDevice));
  m->inv_plan = true;
  return GPB_OK;
}

int ensure_l_planes(gpb_model* m);  // prediction section

int loss_gradients(gpb_model* m, double out[3]) {
  const bool tl = m->trainable[0], tv = m->trainable[1], tn = m->trainable[2];
  out[0] = out[1] = out[2] = 0.0;
  if (!(tl || tv || tn)) return GPB_OK;  // model.py:350-352
  GPB_TRY(ensure_weights(m));
  if (!m->inv_plan) GPB_TRY(build_inv_plan(m));
  const int Ti = m->Ti, bi = m->bi, nb = bi / GBM;
  const int64_t bi2 = int64_t(bi) * bi;
  const int64_t ntiles = int64_t(Ti) * (Ti + 1) / 2;
  double* X = m->X.as<double>();
  double* D = m->Dinv.as<double>();
  const GemmJob* jobs = m->inv_jobs.as<GemmJob>();
  PhaseTimer pt(m, 5);
  // The int8 pipe for the long products of the gradient when the planes are on: |X_ij| <= ||L^-1||_2
  // <= 1 / sqrt(noise) (K >= noise I; 1 on the decoupled padding rows) bounds X; tiny noise keeps
  // the FP64 kernels.  K^-1 = X^T X from n = oz_grad_min_n; X itself left-looking from
  // oz_llx_min_tiles tiles (below that its per-row products are too small for the kernel).
  bool planes = m->oz_slices > 0 && !m->grad_fp64_only && m->np_ >= m->oz_grad_min_n && m->s2 >= 1e-6;
  if (planes && !ensure_optional(m->Xs, size_t(m->oz_slices) * ntiles * bi2)) planes = false;
  bool llx = planes && Ti >= m->oz_llx_min_tiles;
  if (llx && !m->ls_ok && !ensure_optional(m->Ls, size_t(m->oz_slices) * ntiles * bi2)) llx = false;
  const int S = std::max(m->oz_slices, 1), nrb = bi / kOzakiBM;
  const double sx = plane_scale(std::max(1.0, 1.0 / std::sqrt(std::max(m->s2, 1e-300))));
  if (planes && !m->ozflag.p) {
    CUDA_TRY(m->ozflag.ensure(sizeof(int)));
    CUDA_TRY(cudaMemsetAsync(m->ozflag.p, 0, sizeof(int), m->st));
  }
  // X = L^-1 (tiled.py:263-298 with the identity RHS, model.py:358-361),
  // with a one-row lookahead on the critical stream (build_inv_plan)
  for (int i = 0; i < Ti; ++i)
    CUDA_TRY(cudaMemcpyAsync(X + h_tri_cm(i, i, Ti) * bi2, D + int64_t(i) * bi2,
                             sizeof(double) * bi2, cudaMemcpyDeviceToDevice, m->st));
  CUDA_TRY(cudaMemsetAsync(m->Kinv.p, 0, sizeof(double) * ntiles * bi2, m->st));
  if (llx) {
    GPB_TRY(ensure_l_planes(m));
    if (m->llx_slices_base != m->Xs.p) {  // slice-job table with this Xs
      std::vector<OzakiSliceJob> sj = m->llx_slices_host;
      for (auto& j : sj) j.planes = m->Xs.as<int8_t>() + reinterpret_cast<intptr_t>(j.planes);
      CUDA_TRY(m->llx_slices.ensure(sizeof(OzakiSliceJob) * std::max<size_t>(1, sj.size())));
      CUDA_TRY(cudaMemcpy(m->llx_slices.p, sj.data(), sizeof(OzakiSliceJob) * sj.size(), cudaMemcpyHostToDevice));
      m->llx_slices_base = m->Xs.p;
    }
    auto slice_row = [&](int i) -> int {
      ProfScope ps(m, KC_OTHER, 0.0);
      CUDA_TRY(launch_ozaki_slice_t_batch(m->llx_slices.as<OzakiSliceJob>() + m->llx_slice_off[i], i + 1, bi, bi, bi, sx,
                                          1, nrb, S, m->ozflag.as<int>(), m->st));
      ++m->launches;
      return GPB_OK;
    };
    GPB_TRY(slice_row(0));
    for (int i = 1; i < Ti; ++i) {
      for (size_t seg = 0; seg < m->llx_off[i].size(); ++seg) {
        OzakiGemm g{};
        g.a = {m->Ls.as<int8_t>(), bi2 * S, bi / kOzakiBK, int64_t(bi / kOzakiBK) * S * kOzakiBox};
        g.b = {m->Xs.as<int8_t>(), 0, int(1) << 30, int64_t(S) * kOzakiBox, int64_t(nrb) * S * kOzakiBox};
        g.M = g.N = bi;
        g.K = static_cast<int>(std::min<int64_t>(kOzakiMaxK, int64_t(i) * bi - int64_t(seg) * kOzakiMaxK));
        g.slices = S;
        g.alpha = -m->oz_sa * sx;
        g.beta = seg == 0 ? 0.0 : 1.0;
        g.ldc_in = g.ldc_out = bi;
        g.jobs = m->llx_jobs.as<OzakiJob>() + m->llx_off[i][seg];
        g.njobs = static_cast<int>(m->llx_cnt[i][seg]);
        ProfScope ps(m, KC_OZAKI, seg == 0 ? m->llx_fl[i] : 0.0);
        CUDA_TRY(launch_ozaki_gemm(g, m->st));
        m->launches += 2;
      }
      GemmParams f = views(base_params(jobs + m->invx_off[i], i * nb, 1, nb, bi, bi, bi, 1.0, 0.0), m->Dinv, m->Kinv);
      GPB_TRY(gemm(m, f, true, false, EPI_AXPBY, gemm_flops(int64_t(i) * nb, int64_t(GBM) * nb * (nb + 1) / 2)));
      GPB_TRY(slice_row(i));
    }
  } else {
  cudaEvent_t* ev_x = m->grad_ev.data();       // [k]: X(k, .) final
  cudaEvent_t* ev_u = m->grad_ev.data() + Ti;  // [k]: U_k applied to rows > k + 1
  CUDA_TRY(cudaEventRecord(ev_x[0], m->st));   // X(0, 0) = Dinv_0
  CUDA_TRY(cudaStreamWaitEvent(m->crit, ev_x[0], 0));
  auto ugemm = [&](int64_t off, int64_t cnt, double fl, cudaStream_t s) -> int {
    if (cnt == 0) return GPB_OK;
    GemmParams u = views(base_params(jobs + off, static_cast<int>(cnt), nb, 1, bi, bi, bi, -1.0, 1.0), m->L, m->X);
    u.max_k = bi;
    return gemm(m, u, true, false, EPI_AXPBY, fl, s);
  };
  for (int k = 0; k < Ti; ++k) {
    // main: the bulk of U_k (rows > k + 1) once row k of X is final
    CUDA_TRY(cudaStreamWaitEvent(m->st, ev_x[k], 0));
    GPB_TRY(ugemm(m->urest_off[k], m->urest_cnt[k], m->urest_fl[k], m->st));
    CUDA_TRY(cudaEventRecord(ev_u[k], m->st));
    if (k + 1 < Ti) {
      // critical: row k + 1 (it already has U_0 .. U_{k-1} from the main stream), then F_{k+1}
      if (k >= 1) CUDA_TRY(cudaStreamWaitEvent(m->crit, ev_u[k - 1], 0));
      GPB_TRY(ugemm(m->urow_off[k], m->urow_cnt[k], m->urow_fl[k], m->crit));
      GemmParams f = views(base_params(jobs + m->invx_off[k + 1], (k + 1) * nb, 1, nb, bi, bi, bi, 1.0, 0.0),
                           m->Dinv, m->Kinv);
      GPB_TRY(gemm(m, f, true, false, EPI_AXPBY, gemm_flops(int64_t(k + 1) * nb, int64_t(GBM) * nb * (nb + 1) / 2),
                   m->crit));
      CUDA_TRY(cudaEventRecord(ev_x[k + 1], m->crit));
    }
  }
  CUDA_TRY(cudaStreamWaitEvent(m->st, ev_x[Ti - 1], 0));
  }

  double* red = m->red.as<double>();
  const int64_t nblk = ntiles * (bi / kSekBlock) * (bi / kSekBlock);
  if (tl || tv) {
    // K^-1 = X^T X, lower tiles (model.py:362-380)
    // On the int8 pipe when the planes are on: |X_ij| <= ||L^-1||_2 <= 1 / sqrt(noise) (K >= noise I;
    // 1 on the decoupled padding rows) bounds the operand; tiny noise keeps the FP64 kernels.
    if (planes) {
      if (!llx) {  // (the left-looking X phase sliced its rows as it went)
        ProfScope ps(m, KC_OTHER, 0.0);
        for (int c = 0; c < Ti; ++c) {  // planes of column panel c of X, transposed
          const int64_t e0 = h_tri_cm(c, c, Ti) * bi2;
          CUDA_TRY(launch_ozaki_slice_t(X + e0, int64_t(Ti - c) * bi, bi, bi, sx, m->Xs.as<int8_t>() + e0 * S, 1,
                                        nrb, 0, S, m->ozflag.as<int>(), m->st));
          ++m->launches;
        }
      }
      for (size_t seg = 0; seg < m->kinv_oz_off.size(); ++seg) {
        OzakiGemm g{};
        g.a = g.b = {m->Xs.as<int8_t>(), 0, int(1) << 30, int64_t(S) * kOzakiBox, int64_t(nrb) * S * kOzakiBox};
        g.M = g.N = bi;
        g.K = static_cast<int>(std::min<int64_t>(kOzakiMaxK, int64_t(Ti) * bi - int64_t(seg) * kOzakiMaxK));
        g.slices = S;
        g.alpha = sx * sx;
        g.beta = seg == 0 ? 0.0 : 1.0;
        g.ldc_in = g.ldc_out = bi;
        g.jobs = m->kinv_oz_jobs.as<OzakiJob>() + m->kinv_oz_off[seg];
        g.njobs = static_cast<int>(m->kinv_oz_cnt[seg]);
        ProfScope ps(m, KC_OZAKI, seg == 0 ? m->kinv_fl : 0.0);
        CUDA_TRY(launch_ozaki_gemm(g, m->st));
        m->launches += 2;
      }
      int over = 0;
      CUDA_TRY(cudaMemcpyAsync(&over, m->ozflag.p, sizeof(int), cudaMemcpyDeviceToHost, m->st));
      CUDA_TRY(cudaStreamSynchronize(m->st));
      if (over) {  // an entry beyond the bound: repeat on the FP64 kernels
        CUDA_TRY(cudaMemsetAsync(m->ozflag.p, 0, sizeof(int), m->st));
        ++m->oz_fallbacks;
        planes = false;
        if (llx) {  // X itself came from saturated digits: the whole gradient again
          m->grad_fp64_only = true;
          const int st = loss_gradients(m, out);
          m->grad_fp64_only = false;
          return st;
        }
      }
    }
    if (!planes) {
      GemmParams kp = views(base_params(jobs + m->kinv_off, static_cast<int>(m->kinv_cnt), 1, nb, bi, bi,
                                        bi, 1.0, 0.0),
                            m->X, m->X);
      kp.max_k = int64_t(Ti) * bi;
      GPB_TRY(gemm(m, kp, false, false, EPI_AXPBY, m->kinv_fl));
    }
    // fused trace pass (model.py:382-414 with covariance.py:196-220 regenerated)
    CUDA_TRY(launch_trace(m->Kinv.as<double>(), m->tile_cm.as<int2>(), ntiles, TraceTiles{0, 0, 0, nullptr},
                          m->zp.as<double>(), m->alpha.as<double>(), static_cast<int>(m->d), bi,
                          m->pm, sek_params(m), m->part_l.as<double>(), m->part_v.as<double>(),
                          nullptr, m->st));
    CUDA_TRY(launch_reduce(m->part_l.as<double>(), nblk, red + 0, m->st));
    CUDA_TRY(launch_reduce(m->part_v.as<double>(), nblk, red + 1, m->st));
    m->launches += 3;
  }
  if (tn) {
    // ||L^-1||_F^2 and ||alpha||^2 (model.py:415-432)
    CUDA_TRY(launch_tiles_sumsq(X, m->tile_cm.as<int2>(), ntiles, bi, m->pm, m->part_x.as<double>(),
                                m->st));
    CUDA_TRY(launch_reduce(m->part_x.as<double>(), nblk, red + 2, m->st));
    CUDA_TRY(launch_loss_terms(nullptr, 0, m->alpha.as<double>(), m->np_, red + 4, m->st));
    m->launches += 3;
  }
  double hh[6] = {0, 0, 0, 0, 0, 0};
  CUDA_TRY(cudaMemcpyAsync(hh, red, sizeof(hh), cudaMemcpyDeviceToHost, m->st));
  CUDA_TRY(cudaStreamSynchronize(m->st));
  GPB_TRY(pt.stop());

  if (tl) out[0] = 0.5 * (m->nu / (m->l * m->l * m->l)) * hh[0];
  if (tv) out[1] = 0.5 * hh[1];
  if (tn) out[2] = 0.5 * (hh[2] - hh[4]);
  return GPB_OK;
}

// ---- gradient terms over a set of K^-1 tile columns (multi-GPU split) ------
// The single-GPU gradient forms X = L^-1 then K^-1 = X^T X, which needs all of X
// for every column of K^-1.  Split across ranks, each rank instead forms the
// tile columns J of K^-1 it is assigned, K^-1[:, J] = L^-T (L^-1 E_J), from the
// (replicated) factor, one panel slot per column:
//   forward  V = L^-1 E: row block i, slot J <= i:  H_J = E_iJ - L[i, J..i) V[J..i)_J
//            (one GEMM job per slot, K = (i - J) b: no work on the zero rows above J),
//            then V_i = Dinv_i H over the active slots;
//   backward W = L^-T V: row block i (descending), the slots with J <= i at once:
//            H = V_i - L[i+1.., i]^T W[i+1..]  (column i of L read from a
//            column-major-tile copy kept in X, K = (T - 1 - i) b),  W_i = Dinv_i^T H;
// then the fused trace pass over the slots' lower tiles (i >= J).  Columns are
// independent, so ranks need no exchange until the three partial sums are added.
// out = {sum w (K^-1 - a a^T) e d2, sum w (K^-1 - a a^T) e, sum of real diag K^-1}.
int grad_partial(gpb_model* m, const int* cols, int ncols, double out[3]) {
  const int Ti = m->Ti, bi = m->bi, nb = bi / GBM;
  if (ncols < 1 || !cols) return fail(GPB_INVALID_CONFIG, "empty tile column set");
  for (int s = 0; s < ncols; ++s)
    if (cols[s] < 0 || cols[s] >= Ti || (s > 0 && cols[s] <= cols[s - 1]))
      return fail(GPB_INVALID_CONFIG, "tile columns must be increasing and inside [0, " +
                                          std::to_string(Ti) + ")");
  GPB_TRY(ensure_weights(m));
  const int64_t bi2 = int64_t(bi) * bi;
  const int R0 = cols[0];
  const int64_t w = int64_t(ncols) * bi;          // panel width: one slot per column
  const int64_t rows = int64_t(Ti - R0) * bi;     // panel rows: global R0*bi ..
  if (m->gp_panel.ensure(sizeof(double) * rows * w) != cudaSuccess) {
    cudaGetLastError();
    return fail(GPB_NO_MEMORY, "gradient panel of " + std::to_string(rows) + " x " +
                                   std::to_string(w) + " does not fit; pass fewer tile columns");
  }
  CUDA_TRY(m->gp_h.ensure(sizeof(double) * bi * w));
  double* G = m->gp_panel.as<double>();
  double* H = m->gp_h.as<double>();
  double* L = m->L.as<double>();
  double* D = m->Dinv.as<double>();
  PhaseTimer pt(m, 5);
  auto active = [&](int i) {  // slots with column <= i (a prefix: cols ascending)
    return static_cast<int>(std::upper_bound(cols, cols + ncols, i) - cols);
  };
  const int nbt = bi / GBN;
  std::vector<GemmJob> jobs;
  std::vector<int64_t> fd_off, fu_off, bd_off, bu_off;
  for (int i = R0; i < Ti; ++i) {  // forward, right-looking
    const int a = active(i);
    fd_off.push_back(jobs.size());
    for (int r = 0; r < nb; ++r) {  // H = V_i = Dinv_i G_i  (lower: k < (r+1)*128)
      GemmJob v{};
      v.A = D + int64_t(i) * bi2 + int64_t(r) * GBM * bi;
      v.B = G + int64_t(i - R0) * bi * w;
      v.Cout = H + int64_t(r) * GBM * w;
      v.K = (r + 1) * GBM;
      jobs.push_back(v);
    }
    fu_off.push_back(jobs.size());
    for (int q = i + 1; q < Ti; ++q) {  // G_q -= L[q, i] V_i  (active slots only)
      GemmJob u{};
      u.A = L + h_tri_rm(q, i) * bi2;
      u.B = H;
      u.Cin = u.Cout = G + int64_t(q - R0) * bi * w;
      u.K = bi;
      u.nlim = a * nbt;
      jobs.push_back(u);
    }
  }
  for (int i = Ti - 1; i >= R0; --i) {  // backward, right-looking
    bd_off.push_back(jobs.size());
    for (int r = 0; r < nb; ++r) {  // H = W_i = Dinv_i^T G_i  (upper: k >= r*128)
      GemmJob h{};
      h.A = D + int64_t(i) * bi2 + int64_t(r) * GBM * bi + r * GBM;
      h.B = G + (int64_t(i - R0) * bi + r * GBM) * w;
      h.Cout = H + int64_t(r) * GBM * w;
      h.K = bi - r * GBM;
      jobs.push_back(h);
    }
    bu_off.push_back(jobs.size());
    for (int q = R0; q < i; ++q) {  // G_q -= L[i, q]^T W_i  (slots with column <= q)
      GemmJob u{};
      u.A = L + h_tri_rm(i, q) * bi2;
      u.B = H;
      u.Cin = u.Cout = G + int64_t(q - R0) * bi * w;
      u.K = bi;
      u.nlim = active(q) * nbt;
      jobs.push_back(u);
    }
  }
  std::vector<int2> tl;
  std::vector<int> slot;
  for (int s = 0; s < ncols; ++s)
    for (int i = cols[s]; i < Ti; ++i) {
      tl.push_back(make_int2(i, cols[s]));
      slot.push_back(s);
    }
  const int64_t ntl = static_cast<int64_t>(tl.size());
  const int64_t nblk = ntl * (bi / kSekBlock) * (bi / kSekBlock);
  CUDA_TRY(m->gp_jobs.ensure(sizeof(GemmJob) * jobs.size()));
  CUDA_TRY(m->gp_tiles.ensure((sizeof(int2) + sizeof(int)) * tl.size()));
  CUDA_TRY(m->part_l.ensure(sizeof(double) * nblk));
  CUDA_TRY(m->part_v.ensure(sizeof(double) * nblk));
  CUDA_TRY(m->part_x.ensure(sizeof(double) * nblk));
  int2* d_tl = m->gp_tiles.as<int2>();
  int* d_slot = reinterpret_cast<int*>(d_tl + ntl);
  CUDA_TRY(cudaMemcpyAsync(m->gp_jobs.p, jobs.data(), sizeof(GemmJob) * jobs.size(),
                           cudaMemcpyHostToDevice, m->st));
  CUDA_TRY(cudaMemcpyAsync(d_tl, tl.data(), sizeof(int2) * ntl, cudaMemcpyHostToDevice, m->st));
  CUDA_TRY(cudaMemcpyAsync(d_slot, slot.data(), sizeof(int) * ntl, cudaMemcpyHostToDevice, m->st));
  const GemmJob* dj = m->gp_jobs.as<GemmJob>();
  CUDA_TRY(cudaMemsetAsync(G, 0, sizeof(double) * rows * w, m->st));
  for (int s = 0; s < ncols; ++s)  // E: identity block of column cols[s] in slot s
    CUDA_TRY(launch_set_diag(G + int64_t(cols[s] - R0) * bi * w + int64_t(s) * bi, w, bi, m->st));
  m->launches += ncols;
  const size_t row_bytes = sizeof(double) * bi * w;
  for (int i = R0; i < Ti; ++i) {
    const int a = active(i);
    const int64_t k = i - R0;
    GemmParams v = views(base_params(dj + fd_off[k], nb, 1, a * nbt, bi, w, w, 1.0, 0.0), m->Dinv, m->gp_panel);
    GPB_TRY(gemm(m, v, true, false, EPI_AXPBY, gemm_flops(a * nbt, int64_t(GBM) * nb * (nb + 1) / 2)));
    CUDA_TRY(cudaMemcpyAsync(G + k * bi * w, H, row_bytes, cudaMemcpyDeviceToDevice, m->st));
    if (i + 1 < Ti) {
      GemmParams u = views(base_params(dj + fu_off[k], Ti - 1 - i, nb, a * nbt, bi, w, w, -1.0, 1.0), m->L,
                           m->gp_h);
      u.max_k = bi;
      GPB_TRY(gemm(m, u, true, false, EPI_AXPBY,
                   gemm_flops(int64_t(Ti - 1 - i) * nb * a * nbt, bi)));
    }
  }
  for (int i = Ti - 1; i >= R0; --i) {
    const int a = active(i);
    const int64_t s = Ti - 1 - i;
    GemmParams h = views(base_params(dj + bd_off[s], nb, 1, a * nbt, bi, w, w, 1.0, 0.0), m->Dinv, m->gp_panel);
    GPB_TRY(gemm(m, h, false, false, EPI_AXPBY, gemm_flops(a * nbt, int64_t(GBM) * nb * (nb + 1) / 2)));
    CUDA_TRY(cudaMemcpyAsync(G + int64_t(i - R0) * bi * w, H, row_bytes, cudaMemcpyDeviceToDevice,
                             m->st));
    if (i > R0) {
      int64_t blocks = 0;
      for (int q = R0; q < i; ++q) blocks += int64_t(nb) * active(q) * nbt;
      GemmParams u = views(base_params(dj + bu_off[s], i - R0, nb, a * nbt, bi, w, w, -1.0, 1.0), m->L, m->gp_h);
      u.max_k = bi;
      GPB_TRY(gemm(m, u, false, false, EPI_AXPBY, gemm_flops(blocks, bi)));
    }
  }
  double* red = m->red.as<double>();
  CUDA_TRY(launch_trace(G, d_tl, ntl, TraceTiles{w, R0, 0, d_slot}, m->zp.as<double>(),
                        m->alpha.as<double>(), static_cast<int>(m->d), bi, m->pm, sek_params(m),
                        m->part_l.as<double>(), m->part_v.as<double>(), m->part_x.as<double>(),
                        m->st));
  CUDA_TRY(launch_reduce(m->part_l.as<double>(), nblk, red + 0, m->st));
  CUDA_TRY(launch_reduce(m->part_v.as<double>(), nblk, red + 1, m->st));
  CUDA_TRY(launch_reduce(m->part_x.as<double>(), nblk, red + 2, m->st));
  m->launches += 4;
  double hh[3];
  CUDA_TRY(cudaMemcpyAsync(hh, red, sizeof(hh), cudaMemcpyDeviceToHost, m->st));
  CUDA_TRY(cudaStreamSynchronize(m->st));
  GPB_TRY(pt.stop());
  out[0] = hh[0];
  out[1] = hh[1];
  out[2] = hh[2];
  return GPB_OK;
}

// ---- prediction (model.py:221-314) ----------------------------------------
// Digit planes of the off-diagonal factor tiles.  |L(i, j)| <= sqrt(K_ii) =
// sqrt(vertical + noise) (1 on the decoupled padding rows), so one
// fixed-point scale covers the whole factor.
int ensure_l_planes(gpb_model* m) {
  if (m->ls_ok) return GPB_OK;
  const int64_t bi2 = int64_t(m->bi) * m->bi;
  const int64_t ntiles = int64_t(m->Ti) * (m->Ti + 1) / 2;
  CUDA_TRY(m->Ls.ensure(size_t(m->oz_slices) * ntiles * bi2));
  if (!m->ozflag.p) {
    CUDA_TRY(m->ozflag.ensure(sizeof(int)));
    CUDA_TRY(cudaMemsetAsync(m->ozflag.p, 0, sizeof(int), m->st));
  }
  m->oz_sa = plane_scale(std::max(1.0, std::sqrt(m->nu + m->s2)));
  ProfScope ps(m, KC_OTHER, 0.0);
  // tile t of the packed factor -> tile t of the boxed planes; one launch per
  // block row (its off-diagonal tiles are consecutive)
  for (int i = 1; i < m->Ti; ++i) {
    const int64_t t0 = h_tri_rm(i, 0);
    CUDA_TRY(launch_ozaki_slice_tiles(m->L.as<double>() + t0 * bi2, i, m->bi, m->bi, m->oz_sa,
                                      m->Ls.as<int8_t>() + t0 * bi2 * m->oz_slices, m->oz_slices,
                                      m->ozflag.as<int>(), m->st));
    ++m->launches;
  }
  m->ls_ok = true;
  return GPB_OK;
}

// W = B_i - L[i, 0..i) V[0..i) on the tcgen05 pipe, in k segments of at most
// kOzakiMaxK (int32 group sums stay exact)
int ozaki_pred_w(gpb_model* m, int i, int64_t mcp, bool* done) {
  *done = false;
  const int bi = m->bi;
  const int64_t bi2 = int64_t(bi) * bi;
  const int64_t K = int64_t(i) * bi;
  double* W = m->W.as<double>();
  const int S = m->oz_slices;
  const int64_t kchunks = m->np_ / kOzakiBK;
  for (int64_t k0 = 0; k0 < K; k0 += kOzakiMaxK) {
    OzakiGemm g{};
    g.a = {m->Ls.as<int8_t>(), bi2 * S, bi / kOzakiBK, int64_t(bi / kOzakiBK) * S * kOzakiBox};
    g.a_off = (h_tri_rm(i, 0) + k0 / bi) * bi2 * S;
    g.b = {m->Vs.as<int8_t>(), 0, static_cast<int>(kchunks), kchunks * S * kOzakiBox};
    g.b_off = (k0 / kOzakiBK) * S * kOzakiBox;
    g.M = bi;
    g.N = static_cast<int>(mcp);
    g.K = static_cast<int>(std::min<int64_t>(kOzakiMaxK, K - k0));
    g.slices = S;
    g.alpha = -m->oz_sa * m->oz_sb;
    g.beta = 1.0;
    g.Cin = k0 == 0 ? m->Bv.as<double>() + int64_t(i) * bi * mcp : W;
    g.Cout = W;
    g.ldc_in = g.ldc_out = mcp;
    {
      ProfScope ps(m, KC_OZAKI, 2.0 * double(bi) * double(mcp) * double(g.K));
      CUDA_TRY(launch_ozaki_gemm(g, m->st));
    }
    m->launches += S > 4 ? 2 : 1;
  }
  *done = true;
  return GPB_OK;
}

int build_pred_plan(gpb_model* m, int64_t mcp) {
  if (m->pred_mcp == mcp) return GPB_OK;
  const int Ti = m->Ti, bi = m->bi;
  const int64_t bi2 = int64_t(bi) * bi;
  CUDA_TRY(m->Bv.ensure(sizeof(double) * m->np_ * mcp));
  CUDA_TRY(m->W.ensure(sizeof(double) * int64_t(bi) * mcp));
  CUDA_TRY(m->mpart.ensure(sizeof(double) * (m->np_ / kSekBlock) * mcp));
  CUDA_TRY(m->sq.ensure(sizeof(double) * (m->np_ / GBM) * mcp));
  double* L = m->L.as<double>();
  double* D = m->Dinv.as<double>();
  double* Bv = m->Bv.as<double>();
  std::vector<GemmJob> jobs;
  for (int i = 0; i < Ti; ++i) {
    GemmJob w{};  // W = B_i - L[i, 0..i) V[0..i)
    w.A = L + h_tri_rm(i, 0) * bi2;
    w.B = Bv;
    w.Cin = Bv + int64_t(i) * bi * mcp;
    w.Cout = m->W.as<double>();
    w.K = i * bi;
    jobs.push_back(w);
    // V_i = Dinv_i W (+ column sums of squares); Dinv_i is lower triangular,
    // so output row block r only needs k < (r+1)*128: one job per row block
    for (int r = 0; r < bi / GBM; ++r) {
      GemmJob v{};
      v.A = D + int64_t(i) * bi2 + int64_t(r) * GBM * bi;
      v.B = m->W.as<double>();
      v.Cout = Bv + (int64_t(i) * bi + r * GBM) * mcp;
      v.aux = m->sq.as<double>() + (int64_t(i) * bi / GBM + r) * mcp;
      v.K = (r + 1) * GBM;
      jobs.push_back(v);
    }
  }
  CUDA_TRY(m->pred_jobs.ensure(sizeof(GemmJob) * jobs.size()));
  CUDA_TRY(cudaMemcpy(m->pred_jobs.p, jobs.data(), sizeof(GemmJob) * jobs.size(),
                      cudaMemcpyHostToDevice));
  m->pred_mcp = mcp;
  return GPB_OK;
}

// zt_dev: mt x d on device. Results (mean, var) left in m->mean / m->var (length mt).
// Test points processed per chunk: the chunk's K*^T / V buffer (n_p x chunk)
// must fit in device memory; GPB_PRED_CHUNK overrides (multiple of 128).
int64_t pred_chunk(gpb_model* m, int64_t mt) {
  const int64_t all = round_up(std::max<int64_t>(mt, 1), GBM);
  if (const char* e = getenv("GPB_PRED_CHUNK")) {
    const int64_t c = round_up(std::max<int64_t>(atoll(e), 1), GBM);
    return std::min(c, all);
  }
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  const double per_col = 8.0 * double(m->np_ + m->bi + m->np_ / kSekBlock + m->np_ / GBM + 4) +
                         double(m->oz_slices) * double(m->np_);
  // cached blocks are returned to CUDA if an allocation would otherwise fail
  double avail = double(free_b) + double(g_cache.cached) + double(m->Bv.bytes);
  if (m->oz_slices > 0 && int64_t(m->Ti - 1) * m->bi >= m->oz_min_k) {
    // the planes of L (allocated on the first sweep) come out of the same memory
    const double ls = double(m->oz_slices) * double(m->Ti) * (m->Ti + 1) / 2 * double(m->bi) * m->bi;
    if (double(m->Ls.bytes) < ls && avail - ls > 0.25 * avail) avail -= ls;
  }
  const double budget = std::min(48e9, 0.6 * avail);
  const int64_t c = std::max<int64_t>(GBM, int64_t(budget / per_col) / GBM * GBM);
  return std::min(c, all);
}

// one chunk of test points: results written to mean_out / var_out (device)
int predict_chunk(gpb_model* m, const double* zt_dev, int64_t mt, bool want_var, double* mean_out,
                  double* var_out, double* t_cross, double* t_trsm) {
  const int Ti = m->Ti, bi = m->bi;
  const int64_t mcp = round_up(std::max<int64_t>(mt, 1), GBM);
  GPB_TRY(build_pred_plan(m, mcp));
  double* Bv = m->Bv.as<double>();
  const SekParams sp = sek_params(m);
  {
    PhaseTimer pt(m, 3);
    ProfScope ps(m, KC_SEK, 0.0);
    CUDA_TRY(launch_cross(Bv, mcp, m->mpart.as<double>(), m->alpha.as<double>(), m->zp.as<double>(),
                          m->np_, zt_dev, mt, mcp, static_cast<int>(m->d), m->pm, sp, m->st));
    ++m->launches;
    GPB_TRY(pt.stop());
    *t_cross += m->timing[3];
  }
  if (want_var) {
    PhaseTimer pt(m, 4);
    const GemmJob* jobs = m->pred_jobs.as<GemmJob>();
    // tcgen05 digit-plane products for the long-k rows (ozaki.cuh); |V| <=
    // sqrt(k(x*, x*)) = sqrt(vertical) since k*^T K^-1 k* <= k**
    const bool oz_wanted = m->oz_slices > 0 && int64_t(Ti - 1) * bi >= m->oz_min_k;
    bool oz = oz_wanted;
    if (oz && !m->ls_ok) {  // planes of L and of V^T: optional, the DMMA sweep needs neither
      const int64_t ntiles = int64_t(Ti) * (Ti + 1) / 2;
      if (!ensure_optional(m->Ls, size_t(m->oz_slices) * ntiles * int64_t(bi) * bi)) oz = false;
    }
    if (oz && !ensure_optional(m->Vs, size_t(m->oz_slices) * mcp * m->np_)) oz = false;
    if (oz) {
      GPB_TRY(ensure_l_planes(m));
      m->oz_sb = plane_scale(std::sqrt(m->nu));
    }
    for (int i = 0; i < Ti; ++i) {
      bool done = false;
      if (oz && int64_t(i) * bi >= m->oz_min_k) GPB_TRY(ozaki_pred_w(m, i, mcp, &done));
      if (!done) {
        GemmParams w = views(base_params(jobs + int64_t(i) * (1 + bi / GBM), 1, bi / GBM,
                                         static_cast<int>(mcp / GBN), bi, mcp, mcp, -1.0, 1.0),
                             m->L, m->Bv);
        w.a_ktile = bi;
        w.a_kstride = int64_t(bi) * bi;
        w.max_k = int64_t(i) * bi;
        const int64_t blocks = int64_t(bi / GBM) * (mcp / GBN);
        GPB_TRY(gemm(m, w, true, false, EPI_AXPBY, gemm_flops(blocks, int64_t(i) * bi)));
      }
      const int nbr = bi / GBM;
      GemmParams v = views(base_params(jobs + int64_t(i) * (1 + nbr) + 1, nbr, 1,
                                       static_cast<int>(mcp / GBN), bi, mcp, mcp, 1.0, 0.0),
                           m->Dinv, m->W);
      v.aux_ld = mcp;
      GPB_TRY(gemm(m, v, true, false, EPI_SUMSQ,
                   gemm_flops(mcp / GBN, int64_t(GBM) * nbr * (nbr + 1) / 2)));
      if (oz) {  // planes of V_i^T for the rows below (and the full-covariance product)
        ProfScope ps(m, KC_OTHER, 0.0);
        CUDA_TRY(launch_ozaki_slice_t(Bv + int64_t(i) * bi * mcp, bi, mcp, mcp, m->oz_sb, m->Vs.as<int8_t>(),
                                      m->np_ / kOzakiBK, 1, int64_t(i) * bi, m->oz_slices, m->ozflag.as<int>(),
                                      m->st));
        ++m->launches;
      }
    }
    m->vs_ok = oz;
    GPB_TRY(pt.stop());
    *t_trsm += m->timing[4];
  }
  CUDA_TRY(launch_pred_finalize(m->mpart.as<double>(), m->np_ / kSekBlock, m->sq.as<double>(),
                                m->np_ / GBM, mcp, mt, m->nu, mean_out,
                                want_var ? var_out : nullptr, m->st));
  ++m->launches;
  return GPB_OK;
}

// zt_dev: mt x d on device; results (mean, var) left in m->mean / m->var.
// Test points are processed in chunks that fit in device memory;
// single_chunk (full covariance) requires all of V at once.
int predict_core(gpb_model* m, const double* zt_dev, int64_t mt, bool want_var,
                 bool single_chunk = false) {
  GPB_TRY(ensure_weights(m));
  const int64_t chunk = pred_chunk(m, mt);
  const int64_t all = round_up(std::max<int64_t>(mt, 1), GBM);
  if (single_chunk && chunk < all)
    return fail(GPB_NO_MEMORY, "the full posterior covariance of " + std::to_string(mt) +
                                   " test points needs V for all of them at once (" +
                                   std::to_string(8.0 * double(m->np_) * double(all) / 1e9) +
                                   " GB); predict in smaller batches");
  CUDA_TRY(m->mean.ensure(sizeof(double) * all));
  CUDA_TRY(m->var.ensure(sizeof(double) * all));
  double t_cross = 0.0, t_trsm = 0.0;
  for (int64_t c0 = 0; c0 < mt; c0 += chunk) {
    const int64_t mc = std::min(chunk, mt - c0);
    GPB_TRY(predict_chunk(m, zt_dev + c0 * m->d, mc, want_var, m->mean.as<double>() + c0,
                          m->var.as<double>() + c0, &t_cross, &t_trsm));
  }
  if (want_var && m->oz_slices > 0 && m->ozflag.p) {
    // an operand beyond its fixed-point scale saturates its digits: never
    // expected (the scales are mathematical bounds), but then the products
    // are repeated on the DMMA kernels
    int over = 0;
    CUDA_TRY(cudaMemcpyAsync(&over, m->ozflag.p, sizeof(int), cudaMemcpyDeviceToHost, m->st));
    CUDA_TRY(cudaStreamSynchronize(m->st));
    if (over) {
      CUDA_TRY(cudaMemsetAsync(m->ozflag.p, 0, sizeof(int), m->st));
      const int keep = m->oz_slices;
      m->oz_slices = 0;
      ++m->oz_fallbacks;
      int s = predict_core(m, zt_dev, mt, want_var, single_chunk);
      m->oz_slices = keep;
      return s;
    }
  }
  m->timing[3] = t_cross;
  m->timing[4] = t_trsm;
  return GPB_OK;
}

int full_cov(gpb_model* m, const double* zt_dev, int64_t mt, double* cov_host) {
  const int64_t mcp = m->pred_mcp;
  const int64_t nbk = mcp / GBM;
  CUDA_TRY(m->S.ensure(sizeof(double) * mcp * mcp));
  double* S = m->S.as<double>();
  double* Bv = m->Bv.as<double>();
  if (m->fc_mcp != mcp) {
    std::vector<GemmJob> jobs;
    for (int64_t r = 0; r < nbk; ++r)
      for (int64_t c = 0; c <= r; ++c) {
        GemmJob g{};
        g.A = Bv + r * GBM;
        g.B = Bv + c * GBM;
        g.Cin = g.Cout = S + r * GBM * mcp + c * GBM;
        g.K = static_cast<int>(m->np_);
        jobs.push_back(g);
      }
    CUDA_TRY(m->fc_jobs.ensure(sizeof(GemmJob) * jobs.size()));
    CUDA_TRY(cudaMemcpy(m->fc_jobs.p, jobs.data(), sizeof(GemmJob) * jobs.size(),
                        cudaMemcpyHostToDevice));
    // the same lower blocks for the digit-plane product: rows r and c of V^T's planes
    std::vector<OzakiJob> oj;
    // (offsets for 8 planes per operand; with fewer planes the DMMA product runs)
    const int64_t rb_stride = (m->np_ / kOzakiBK) * int64_t(kOzakiMaxSlices) * kOzakiBox;
    for (int64_t r = 0; r < nbk; ++r)
      for (int64_t c = 0; c <= r; ++c) {
        OzakiJob o{};
        o.a_off = r * rb_stride;
        o.b_off = c * rb_stride;
        o.C = S + r * GBM * mcp + c * GBM;
        oj.push_back(o);
      }
    CUDA_TRY(m->fc_oz_jobs.ensure(sizeof(OzakiJob) * oj.size()));
    CUDA_TRY(cudaMemcpy(m->fc_oz_jobs.p, oj.data(), sizeof(OzakiJob) * oj.size(), cudaMemcpyHostToDevice));
    m->fc_mcp = mcp;
  }
  PhaseTimer pt(m, 6);
  CUDA_TRY(launch_prior(S, mcp, zt_dev, mt, static_cast<int>(m->d), sek_params(m), m->st));
  ++m->launches;
  // Sigma = K** - V^T V (model.py:254-269), lower blocks
  if (m->oz_slices == kOzakiMaxSlices && m->vs_ok && m->np_ >= m->oz_min_k) {
    // V^T V from the planes of V^T the prediction sweep left in Vs (k in segments of kOzakiMaxK)
    const int64_t kchunks = m->np_ / kOzakiBK;
    for (int64_t k0 = 0; k0 < m->np_; k0 += kOzakiMaxK) {
      OzakiGemm g{};
      g.a = g.b = {m->Vs.as<int8_t>(), 0, static_cast<int>(kchunks), kchunks * m->oz_slices * kOzakiBox};
      g.a_off = g.b_off = (k0 / kOzakiBK) * m->oz_slices * kOzakiBox;
      g.M = g.N = GBM;
      g.K = static_cast<int>(std::min<int64_t>(kOzakiMaxK, m->np_ - k0));
      g.slices = m->oz_slices;
      g.alpha = -m->oz_sb * m->oz_sb;
      g.beta = 1.0;
      g.ldc_in = g.ldc_out = mcp;
      g.jobs = m->fc_oz_jobs.as<OzakiJob>();
      g.njobs = static_cast<int>(nbk * (nbk + 1) / 2);
      ProfScope ps(m, KC_OZAKI, gemm_flops(nbk * (nbk + 1) / 2, g.K));
      CUDA_TRY(launch_ozaki_gemm(g, m->st));
      m->launches += 2;
    }
  } else {
    GemmParams p = views(base_params(m->fc_jobs.as<GemmJob>(), static_cast<int>(nbk * (nbk + 1) / 2), 1, 1,
                                     mcp, mcp, mcp, -1.0, 1.0),
                         m->Bv, m->Bv);
    p.max_k = m->np_;
    GPB_TRY(gemm(m, p, false, false, EPI_AXPBY, gemm_flops(nbk * (nbk + 1) / 2, m->np_)));
  }
  CUDA_TRY(launch_symmetrize(S, mcp, mt, m->st));
  ++m->launches;
  GPB_TRY(pt.stop());
  CUDA_TRY(cudaMemcpy2DAsync(cov_host, sizeof(double) * mt, S, sizeof(double) * mcp,
                             sizeof(double) * mt, mt, cudaMemcpyDeviceToHost, m->st));
  CUDA_TRY(cudaStreamSynchronize(m->st));
  return GPB_OK;
}

int clamp_variances(double* v, int64_t n, int64_t stride) {
  // model.py:488-496
  double worst = 0.0;
  bool bad = false;
  for (int64_t i = 0; i < n; ++i) {
    const double x = v[i * stride];
    if (x < -kVarianceSlack) {
      if (!bad || x < worst) worst = x;
      bad = true;
    }
  }
  if (bad) {
    char buf[160];
    snprintf(buf, sizeof(buf), "variance %g is below the round-off allowance -%g", worst,
             kVarianceSlack);
    return fail(GPB_NUMERIC, buf);
  }
  for (int64_t i = 0; i < n; ++i)
    if (v[i * stride] < 0.0) v[i * stride] = 0.0;
  return GPB_OK;
}

int model_create(gpb_ctx* ctx, const double* z, const double* y, int64_t n, int64_t d, int64_t T,
                 bool device_ptrs, gpb_model** out) {
  if (!out) return fail(GPB_INVALID_CONFIG, "null output pointer");
  *out = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!ctx || ctx != g_ctx) return fail(GPB_NOT_RUNNING, "runtime is not running");
  }
  if (n < 1 || d < 1) return fail(GPB_DIM, "z must be N x D with N, D >= 1");
  if (T < 1 || n % T != 0) {
    return fail(GPB_TILING, "tiles_per_dim=" + std::to_string(T) + " must divide the " +
                                std::to_string(n) + " training points");
  }
  CUDA_TRY(cudaSetDevice(ctx->device));
  gpb_model* m = new gpb_model();
  m->ctx = ctx;
  m->gen = ctx->gen;
  m->n = n;
  m->d = d;
  m->T = T;
  m->b = static_cast<int>(n / T);
  if (const char* e = getenv("GPB_OZAKI")) {
    const int v = atoi(e);
    m->oz_slices = v <= 0 ? 0 : std::min(kOzakiMaxSlices, std::max(4, v));
  }
  if (const char* e = getenv("GPB_OZAKI_MIN_K")) m->oz_min_k = std::max<int64_t>(64, atoll(e));
  if (const char* e = getenv("GPB_OZAKI_CHOL")) m->oz_chol = atoi(e) != 0;
  if (const char* e = getenv("GPB_OZAKI_CHOL_IN")) m->oz_chol_in = atoi(e) != 0;
  if (const char* e = getenv("GPB_OZAKI_LLX_MIN_TILES")) m->oz_llx_min_tiles = std::max(2, atoi(e));
  if (const char* e = getenv("GPB_OZAKI_CHOL_MIN_K")) m->oz_chol_min_k = std::max<int64_t>(64, atoll(e));
  if (int s_l = apply_layout(m)) {
    delete m;
    return s_l;
  }
  int s = GPB_OK;
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  if (cudaStreamCreateWithPriority(&m->st, cudaStreamNonBlocking, prio_lo) != cudaSuccess ||
      cudaStreamCreateWithPriority(&m->crit, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
      cudaEventCreate(&m->e0) != cudaSuccess || cudaEventCreate(&m->e1) != cudaSuccess) {
    s = fail(GPB_CUDA, "stream/event creation failed");
  }
  if (s == GPB_OK) s = alloc_model_buffers(m);
  if (s == GPB_OK && getenv("GPB_POTRF_PROF")) {
    cudaMalloc(&m->potrf_prof, 16 * sizeof(long long));
    cudaMemset(m->potrf_prof, 0, 16 * sizeof(long long));
  }
  if (s == GPB_OK) s = upload_train(m, z, y, device_ptrs);
  if (s != GPB_OK) {
    gpb_model_destroy(m);
    return s;
  }
  *out = m;
  return GPB_OK;
}

void free_model(gpb_model* m, bool keep = true) {
  for (DevBuf* b : {&m->zp, &m->yp, &m->L, &m->Dinv, &m->scratch, &m->logdiag, &m->info, &m->yhat,
                    &m->beta, &m->alpha, &m->bhat, &m->red, &m->tile_rm, &m->tile_cm, &m->chol_jobs,
                    &m->flow_flags,
                    &m->X, &m->Kinv, &m->part_l, &m->part_v, &m->part_x, &m->inv_jobs,
                    &m->Bv, &m->W, &m->mpart, &m->sq, &m->pred_jobs, &m->zt, &m->mean, &m->var,
                    &m->S, &m->fc_jobs, &m->gp_panel, &m->gp_h, &m->gp_jobs, &m->gp_tiles,
                    &m->Ls, &m->Vs, &m->ozflag, &m->Ps, &m->oz_jobs, &m->fc_oz_jobs, &m->Xs, &m->kinv_oz_jobs, &m->llx_jobs, &m->llx_slices})
    b->release(keep);
}

}  // namespace

// =========================== C ABI ==========================================
extern "C" {

int gpb_abi_version(void) { return 1; }

// error sink for tile_plugin.cu (shares the thread-local message)
int gpb_plugin_fail(int code, const char* msg) { return fail(code, msg); }

const char* gpb_last_error(void) { return g_err.c_str(); }

int gpb_init(int device, gpb_ctx** out) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_ctx) return fail(GPB_ALREADY_RUNNING, "a runtime is already running in this process");
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(GPB_INVALID_CONFIG, "no such CUDA device");
  CUDA_TRY(cudaSetDevice(device));
  CUDA_TRY(gemm_init_attributes());
  CUDA_TRY(ozaki_init_attributes());
  CUDA_TRY(potrf_init_attributes());
  gpb_ctx* c = new gpb_ctx();
  c->device = device;
  c->gen = ++g_gen;
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    return fail(GPB_CUDA, "stream creation failed");
  }
  g_ctx = c;
  if (out) *out = c;
  return GPB_OK;
}

int gpb_finalize(gpb_ctx* ctx) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_ctx || (ctx && ctx != g_ctx)) return fail(GPB_NOT_RUNNING, "no runtime is running");
  cudaDeviceSynchronize();
  cudaStreamDestroy(g_ctx->stream);
  if (g_ctx->pinned) cudaFreeHost(g_ctx->pinned);
  for (cudaEvent_t e : g_ctx->strip_ev)
    if (e) cudaEventDestroy(e);
  delete g_ctx;
  g_ctx = nullptr;
  g_cache.trim();  // blocks still owned by live models stay with them
  gpb_dev_release_ring();
  return GPB_OK;
}

gpb_ctx* gpb_current(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  return g_ctx;
}

int gpb_model_create(gpb_ctx* ctx, const double* z, const double* y, int64_t n, int64_t d,
                     int64_t tiles_per_dim, gpb_model** out) {
  if (!z || !y) return fail(GPB_INVALID_CONFIG, "null input");
  return model_create(ctx, z, y, n, d, tiles_per_dim, false, out);
}

int gpb_model_create_device(gpb_ctx* ctx, const double* z_dev, const double* y_dev, int64_t n,
                            int64_t d, int64_t tiles_per_dim, gpb_model** out) {
  if (!z_dev || !y_dev) return fail(GPB_INVALID_CONFIG, "null input");
  return model_create(ctx, z_dev, y_dev, n, d, tiles_per_dim, true, out);
}

int gpb_model_destroy(gpb_model* m) {
  if (!m) return GPB_OK;
  bool live;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    live = g_ctx && g_ctx == m->ctx && g_ctx->gen == m->gen;
  }
  if (m->st) cudaStreamSynchronize(m->st);
  // a model of a finalized runtime frees its blocks: a later runtime may run
  // on another GPU and must not be handed this one's memory
  free_model(m, live);
  for (cudaEvent_t e : m->evpool) cudaEventDestroy(e);
  for (cudaEvent_t e : m->sync_ev) cudaEventDestroy(e);
  for (cudaEvent_t e : m->grad_ev) cudaEventDestroy(e);
  if (m->prof_ref) cudaEventDestroy(m->prof_ref);
  if (m->crit) cudaStreamDestroy(m->crit);
  if (m->e0) cudaEventDestroy(m->e0);
  if (m->e1) cudaEventDestroy(m->e1);
  if (m->st) cudaStreamDestroy(m->st);
  delete m;
  return GPB_OK;
}

int gpb_model_set_train(gpb_model* m, const double* z, const double* y, int64_t n, int64_t d) {
  GPB_TRY(check_live(m));
  if (n % m->T != 0)
    return fail(GPB_TILING, "tiles_per_dim=" + std::to_string(m->T) + " must divide the " +
                                std::to_string(n) + " training points");
  if (n < 1 || d < 1) return fail(GPB_DIM, "z must be N x D with N, D >= 1");
  free_model(m);
  m->plan_ok = m->inv_plan = false;
  m->pred_mcp = m->fc_mcp = -1;
  m->n = n;
  m->d = d;
  m->b = static_cast<int>(n / m->T);
  GPB_TRY(apply_layout(m));
  invalidate(m);
  GPB_TRY(alloc_model_buffers(m));
  return upload_train(m, z, y, false);
}

int gpb_model_set_params(gpb_model* m, double l, double nu, double s2, const uint8_t tr[3]) {
  if (!m) return fail(GPB_INVALID_CONFIG, "null model");
  if (!(l > 0)) return fail(GPB_INVALID_CONFIG, "lengthscale must be positive");
  if (!(nu > 0)) return fail(GPB_INVALID_CONFIG, "vertical_scale must be positive");
  if (!(s2 >= 0)) return fail(GPB_INVALID_CONFIG, "noise_variance must be non-negative");
  m->l = l;
  m->nu = nu;
  m->s2 = s2;
  if (tr) for (int i = 0; i < 3; ++i) m->trainable[i] = tr[i] ? 1 : 0;
  invalidate(m);
  return GPB_OK;
}

int gpb_model_get_params(gpb_model* m, double out[3]) {
  if (!m || !out) return fail(GPB_INVALID_CONFIG, "null argument");
  out[0] = m->l;
  out[1] = m->nu;
  out[2] = m->s2;
  return GPB_OK;
}

namespace {
// host copy of one strip, split over threads when large (the pageable user
// array is written at host memory speed instead of the driver's bounce path)
void host_copy(char* dst, const char* src, size_t bytes) {
  const size_t chunk = size_t(4) << 20;
  const int nt = static_cast<int>(std::min<size_t>(8, (bytes + chunk - 1) / chunk));
  if (nt <= 1) {
    memcpy(dst, src, bytes);
    return;
  }
  std::vector<std::thread> th;
  const size_t per = (bytes + nt - 1) / nt;
  for (int t = 0; t < nt; ++t) {
    const size_t lo = std::min(bytes, t * per), hi = std::min(bytes, lo + per);
    th.emplace_back([=] { memcpy(dst + lo, src + lo, hi - lo); });
  }
  for (auto& x : th) x.join();
}
}  // namespace

int gpb_cholesky(gpb_model* m, double* L_out) {
  GPB_TRY(check_live(m));
  GPB_TRY(ensure_factor(m));
  if (L_out) {
    // Dense export in strips of rows: export kernel -> device strip -> pinned
    // host strip (full PCIe rate) -> the caller's array (threaded memcpy),
    // double-buffered so the host copy of strip s overlaps the device work of
    // strip s + 1.  Bounded memory (2 x 32 MB device and pinned), so configs 3/4
    // export without an n x n temporary.
    gpb_ctx* ctx = m->ctx;
    std::lock_guard<std::mutex> lk(ctx->export_mu);
    const int64_t n = m->n;
    const size_t strip_cap = size_t(32) << 20;
    const int64_t rows = std::max<int64_t>(1, std::min<int64_t>(n, int64_t(strip_cap / (8 * n))));
    const size_t strip_bytes = sizeof(double) * rows * n;
    if (ctx->pinned_bytes < 2 * strip_bytes) {
      if (ctx->pinned) cudaFreeHost(ctx->pinned);
      ctx->pinned = nullptr;
      ctx->pinned_bytes = 0;
      CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&ctx->pinned), 2 * strip_bytes, cudaHostAllocDefault));
      ctx->pinned_bytes = 2 * strip_bytes;
    }
    for (cudaEvent_t& e : ctx->strip_ev)
      if (!e) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    DevBuf stage[2];
    CUDA_TRY(stage[0].ensure(strip_bytes));
    CUDA_TRY(stage[1].ensure(strip_bytes));
    const int64_t nstrips = (n + rows - 1) / rows;
    auto issue = [&](int64_t s) -> int {
      const int64_t r0 = s * rows, nr = std::min(rows, n - r0);
      double* buf = stage[s % 2].as<double>();
      CUDA_TRY(launch_export_lower(m->L.as<double>(), m->bi, n, r0, nr, m->pm, buf, m->st));
      ++m->launches;
      CUDA_TRY(cudaMemcpyAsync(ctx->pinned + (s % 2) * strip_bytes, buf, sizeof(double) * nr * n,
                               cudaMemcpyDeviceToHost, m->st));
      CUDA_TRY(cudaEventRecord(ctx->strip_ev[s % 2], m->st));
      return GPB_OK;
    };
    for (int64_t s = 0; s < std::min<int64_t>(2, nstrips); ++s) GPB_TRY(issue(s));
    for (int64_t s = 0; s < nstrips; ++s) {
      const int64_t r0 = s * rows, nr = std::min(rows, n - r0);
      CUDA_TRY(cudaEventSynchronize(ctx->strip_ev[s % 2]));
      host_copy(reinterpret_cast<char*>(L_out + r0 * n), ctx->pinned + (s % 2) * strip_bytes,
                sizeof(double) * nr * n);
      if (s + 2 < nstrips) GPB_TRY(issue(s + 2));  // this pinned slot is free again
    }
    CUDA_TRY(cudaStreamSynchronize(m->st));
    stage[0].release();
    stage[1].release();
  }
  return GPB_OK;
}

int gpb_last_pivot(gpb_model* m, int64_t* pivot) {
  if (!m || !pivot) return fail(GPB_INVALID_CONFIG, "null argument");
  *pivot = m->last_pivot;
  return GPB_OK;
}

int gpb_log_likelihood(gpb_model* m, double* out) {
  GPB_TRY(check_live(m));
  return log_likelihood(m, out);
}

int gpb_loss_gradients(gpb_model* m, double out[3]) {
  GPB_TRY(check_live(m));
  return loss_gradients(m, out);
}

int gpb_loss_gradient_terms(gpb_model* m, const int* cols, int64_t ncols, double out[3]) {
  GPB_TRY(check_live(m));
  if (!out) return fail(GPB_INVALID_CONFIG, "null output");
  if (ncols > (int64_t(1) << 30)) return fail(GPB_INVALID_CONFIG, "too many tile columns");
  return grad_partial(m, cols, static_cast<int>(ncols), out);
}

int gpb_optimize(gpb_model* m, double lr, double b1, double b2, double eps, int64_t iters,
                 double* history) {
  GPB_TRY(check_live(m));
  // AdamConfig validation (model.py:61-74)
  if (!(lr > 0)) return fail(GPB_INVALID_CONFIG, "learning_rate must be positive");
  if (!(b1 >= 0 && b1 < 1)) return fail(GPB_INVALID_CONFIG, "beta1 must lie in [0, 1)");
  if (!(b2 >= 0 && b2 < 1)) return fail(GPB_INVALID_CONFIG, "beta2 must lie in [0, 1)");
  if (!(eps > 0)) return fail(GPB_INVALID_CONFIG, "epsilon must be positive");
  if (iters < 1) return fail(GPB_INVALID_CONFIG, "iterations must be at least 1");
  for (int64_t it = 0; it < iters; ++it) {
    m->adam_step += 1;
    double grads[3];
    int s = loss_gradients(m, grads);
    double theta[3] = {m->l, m->nu, m->s2};
    if (s == GPB_OK) {
      // model.py:462-479, same operation order
      double step[3];
      for (int i = 0; i < 3; ++i) {
        const double g = grads[i] * theta[i];
        m->adam_m[i] = b1 * m->adam_m[i] + (1 - b1) * g;
        m->adam_v[i] = b2 * m->adam_v[i] + (1 - b2) * g * g;
        const double mh = m->adam_m[i] / (1 - std::pow(b1, double(m->adam_step)));
        const double vh = m->adam_v[i] / (1 - std::pow(b2, double(m->adam_step)));
        step[i] = lr * mh / (std::sqrt(vh) + eps);
      }
      for (int i = 0; i < 3; ++i) {
        if (m->trainable[i]) {
          const double u = std::log(std::max(theta[i], 1e-300)) - step[i];
          theta[i] = std::exp(u);
        }
      }
      if (m->trainable[2]) theta[2] = std::max(theta[2], 1e-12);
      m->l = theta[0];
      m->nu = theta[1];
      m->s2 = theta[2];
      invalidate(m);
      double ll = 0;
      s = log_likelihood(m, &ll);
      if (s == GPB_OK && history) history[it] = -ll;
    }
    if (s == GPB_NOT_PD) {
      g_err = "iteration " + std::to_string(m->adam_step) + ": " + g_err;
      return s;
    }
    if (s != GPB_OK) return s;
  }
  return GPB_OK;
}

int gpb_predict(gpb_model* m, const double* zt, int64_t mt, int64_t d, double* mean, double* var,
                double* cov) {
  GPB_TRY(check_live(m));
  if (d != m->d)
    return fail(GPB_DIM, "test has " + std::to_string(d) + " features, model was trained with " +
                             std::to_string(m->d));
  if (mt < 1) return fail(GPB_DIM, "need at least one test point");
  if (!mean || !zt) return fail(GPB_INVALID_CONFIG, "null argument");
  CUDA_TRY(m->zt.ensure(sizeof(double) * mt * d));
  CUDA_TRY(cudaMemcpyAsync(m->zt.p, zt, sizeof(double) * mt * d, cudaMemcpyHostToDevice, m->st));
  const bool want_var = var || cov;
  int s = predict_core(m, m->zt.as<double>(), mt, want_var, cov != nullptr);
  if (s != GPB_OK) {
    invalidate(m);
    return s;
  }
  CUDA_TRY(cudaMemcpyAsync(mean, m->mean.p, sizeof(double) * mt, cudaMemcpyDeviceToHost, m->st));
  if (var) CUDA_TRY(cudaMemcpyAsync(var, m->var.p, sizeof(double) * mt, cudaMemcpyDeviceToHost, m->st));
  CUDA_TRY(cudaStreamSynchronize(m->st));
  if (cov) {
    GPB_TRY(full_cov(m, m->zt.as<double>(), mt, cov));
    GPB_TRY(clamp_variances(cov, mt, mt + 1));
  }
  if (var) GPB_TRY(clamp_variances(var, mt, 1));
  return GPB_OK;
}

int gpb_predict_device(gpb_model* m, const double* zt_dev, int64_t mt, int64_t d, double* mean_dev,
                       double* var_dev) {
  GPB_TRY(check_live(m));
  if (d != m->d) return fail(GPB_DIM, "feature count mismatch");
  GPB_TRY(predict_core(m, zt_dev, mt, var_dev != nullptr));
  if (mean_dev)
    CUDA_TRY(cudaMemcpyAsync(mean_dev, m->mean.p, sizeof(double) * mt, cudaMemcpyDeviceToDevice, m->st));
  if (var_dev)
    CUDA_TRY(cudaMemcpyAsync(var_dev, m->var.p, sizeof(double) * mt, cudaMemcpyDeviceToDevice, m->st));
  CUDA_TRY(cudaStreamSynchronize(m->st));
  return GPB_OK;
}

int gpb_predict_solve_device(gpb_model* m, const double* zt_dev, int64_t mt, int64_t d,
                             double* mean_dev, double* V_dev, int64_t ldv) {
  GPB_TRY(check_live(m));
  if (d != m->d) return fail(GPB_DIM, "feature count mismatch");
  if (mt < 0 || ldv < mt || !V_dev) return fail(GPB_INVALID_CONFIG, "V buffer must be n_p x ldv, ldv >= m");
  if (mt == 0) return GPB_OK;
  GPB_TRY(predict_core(m, zt_dev, mt, true, /*single_chunk=*/true));
  if (mean_dev)
    CUDA_TRY(cudaMemcpyAsync(mean_dev, m->mean.p, sizeof(double) * mt, cudaMemcpyDeviceToDevice, m->st));
  CUDA_TRY(cudaMemcpy2DAsync(V_dev, sizeof(double) * ldv, m->Bv.p, sizeof(double) * m->pred_mcp,
                             sizeof(double) * mt, m->np_, cudaMemcpyDeviceToDevice, m->st));
  CUDA_TRY(cudaStreamSynchronize(m->st));
  return GPB_OK;
}

int gpb_cov_block_device(gpb_model* m, const double* za, int64_t ma, const double* Va, int64_t ldva,
                         const double* zb, int64_t mb, const double* Vb, int64_t ldvb, double* out,
                         int64_t ldo) {
  GPB_TRY(check_live(m));
  const int64_t mpa = round_up(std::max<int64_t>(ma, 1), GBM);
  const int64_t mpb = round_up(std::max<int64_t>(mb, 1), GBM);
  if (ma < 0 || mb < 0 || ldva < mpa || ldvb < mpb || ldo < mb)
    return fail(GPB_INVALID_CONFIG, "V blocks need ld >= m rounded up to 128, out ld >= mb");
  if (ma == 0 || mb == 0) return GPB_OK;
  GPB_TRY(ensure_weights(m));
  CUDA_TRY(m->S.ensure(sizeof(double) * mpa * mpb));
  double* S = m->S.as<double>();
  PhaseTimer pt(m, 6);
  CUDA_TRY(launch_prior2(S, mpb, mpa, mpb, za, ma, zb, mb, static_cast<int>(m->d), sek_params(m),
                         m->st));
  ++m->launches;
  // Sigma_ab = K**(a, b) - Va^T Vb  (model.py:254-269 for one block)
  GemmJob g{};
  g.A = Va;
  g.B = Vb;
  g.Cin = g.Cout = S;
  g.K = static_cast<int>(m->np_);
  CUDA_TRY(m->gp_jobs.ensure(sizeof(GemmJob)));
  CUDA_TRY(cudaMemcpyAsync(m->gp_jobs.p, &g, sizeof(g), cudaMemcpyHostToDevice, m->st));
  GemmParams p = views(base_params(m->gp_jobs.as<GemmJob>(), 1, static_cast<int>(mpa / GBM),
                                   static_cast<int>(mpb / GBN), ldva, ldvb, mpb, -1.0, 1.0),
                       Va, sizeof(double) * m->np_ * ldva, Vb, sizeof(double) * m->np_ * ldvb);
  p.max_k = m->np_;
  GPB_TRY(gemm(m, p, false, false, EPI_AXPBY, gemm_flops((mpa / GBM) * (mpb / GBN), m->np_)));
  CUDA_TRY(cudaMemcpy2DAsync(out, sizeof(double) * ldo, S, sizeof(double) * mpb, sizeof(double) * mb,
                             ma, cudaMemcpyDeviceToDevice, m->st));
  CUDA_TRY(cudaStreamSynchronize(m->st));
  return pt.stop();
}

int gpb_model_adopt_factor(gpb_model* m, const double* tiles, const double* dinv,
                           const double* logdiag, const double* beta, const double* alpha) {
  GPB_TRY(check_live(m));
  if (!tiles || !dinv || !logdiag || !beta || !alpha) return fail(GPB_INVALID_CONFIG, "null argument");
  const int64_t bi2 = int64_t(m->bi) * m->bi;
  const int64_t ntiles = int64_t(m->Ti) * (m->Ti + 1) / 2;
  CUDA_TRY(cudaMemcpyAsync(m->L.p, tiles, sizeof(double) * ntiles * bi2, cudaMemcpyDeviceToDevice, m->st));
  CUDA_TRY(cudaMemcpyAsync(m->Dinv.p, dinv, sizeof(double) * m->Ti * bi2, cudaMemcpyDeviceToDevice, m->st));
  CUDA_TRY(cudaMemcpyAsync(m->logdiag.p, logdiag, sizeof(double) * m->Ti, cudaMemcpyDeviceToDevice, m->st));
  CUDA_TRY(cudaMemcpyAsync(m->beta.p, beta, sizeof(double) * m->np_, cudaMemcpyDeviceToDevice, m->st));
  CUDA_TRY(cudaMemcpyAsync(m->alpha.p, alpha, sizeof(double) * m->np_, cudaMemcpyDeviceToDevice, m->st));
  CUDA_TRY(cudaStreamSynchronize(m->st));
  m->factor_ok = true;
  m->weights_ok = true;
  m->ls_ok = false;
  m->last_pivot = -1;
  return GPB_OK;
}

int gpb_model_factor_buffers(gpb_model* m, double** tiles, double** dinv, double** logdiag,
                             double** beta, double** alpha) {
  GPB_TRY(check_live(m));
  if (tiles) *tiles = m->L.as<double>();
  if (dinv) *dinv = m->Dinv.as<double>();
  if (logdiag) *logdiag = m->logdiag.as<double>();
  if (beta) *beta = m->beta.as<double>();
  if (alpha) *alpha = m->alpha.as<double>();
  return GPB_OK;
}

int gpb_model_mark_factored(gpb_model* m) {
  GPB_TRY(check_live(m));
  CUDA_TRY(cudaDeviceSynchronize());
  m->factor_ok = true;
  m->weights_ok = true;
  m->ls_ok = false;
  m->last_pivot = -1;
  return GPB_OK;
}

int gpb_clamp_variances(double* v, int64_t n) {
  if (n < 0 || (n > 0 && !v)) return fail(GPB_INVALID_CONFIG, "null argument");
  return clamp_variances(v, n, 1);
}

int gpb_model_get_adam(gpb_model* m, double moment1[3], double moment2[3], int64_t* step) {
  if (!m || !moment1 || !moment2 || !step) return fail(GPB_INVALID_CONFIG, "null argument");
  for (int i = 0; i < 3; ++i) {
    moment1[i] = m->adam_m[i];
    moment2[i] = m->adam_v[i];
  }
  *step = m->adam_step;
  return GPB_OK;
}

int gpb_model_set_adam(gpb_model* m, const double moment1[3], const double moment2[3], int64_t step) {
  if (!m || !moment1 || !moment2 || step < 0) return fail(GPB_INVALID_CONFIG, "invalid Adam state");
  for (int i = 0; i < 3; ++i) {
    m->adam_m[i] = moment1[i];
    m->adam_v[i] = moment2[i];
  }
  m->adam_step = step;
  return GPB_OK;
}

int gpb_model_timings(gpb_model* m, double* ms_out, int n) {
  if (!m || !ms_out) return fail(GPB_INVALID_CONFIG, "null argument");
  for (int i = 0; i < n && i < 8; ++i) ms_out[i] = m->timing[i];
  return GPB_OK;
}

int gpb_model_stream(gpb_model* m, void** stream) {
  if (!m || !stream) return fail(GPB_INVALID_CONFIG, "null argument");
  *stream = static_cast<void*>(m->st);
  return GPB_OK;
}

int gpb_model_set_profiling(gpb_model* m, int on) {
  if (!m) return fail(GPB_INVALID_CONFIG, "null model");
  GPB_TRY(prof_collect(m));
  m->prof = on != 0;
  for (int i = 0; i < 8; ++i) {
    m->cls_ms[i] = m->cls_flops[i] = m->cls_busy[i] = 0.0;
    m->cls_n[i] = 0;
  }
  if (m->prof) {
    if (!m->prof_ref) CUDA_TRY(cudaEventCreate(&m->prof_ref));
    CUDA_TRY(cudaEventRecord(m->prof_ref, m->st));
  }
  return GPB_OK;
}

int gpb_model_kernel_stats(gpb_model* m, double ms[8], double flops[8], int64_t count[8]) {
  if (!m) return fail(GPB_INVALID_CONFIG, "null model");
  GPB_TRY(prof_collect(m));
  for (int i = 0; i < 8; ++i) {
    if (ms) ms[i] = m->cls_ms[i];
    if (flops) flops[i] = m->cls_flops[i];
    if (count) count[i] = m->cls_n[i];
  }
  return GPB_OK;
}

int gpb_model_kernel_busy(gpb_model* m, double busy_ms[8]) {
  if (!m || !busy_ms) return fail(GPB_INVALID_CONFIG, "null argument");
  GPB_TRY(prof_collect(m));
  for (int i = 0; i < 8; ++i) busy_ms[i] = m->cls_busy[i];
  return GPB_OK;
}

int gpb_model_set_ozaki(gpb_model* m, int slices) {
  GPB_TRY(check_live(m));
  if (slices != 0 && (slices < 4 || slices > kOzakiMaxSlices))
    return fail(GPB_INVALID_CONFIG, "digit planes: 0 (off) or 4..8");
  if (slices != m->oz_slices) {
    // plane offsets depend on the count, the panel grouping on whether planes are in use:
    // a different grouping is a different (round-off level) factor, so the cached one goes
    m->ls_ok = m->plan_ok = m->vs_ok = m->inv_plan = false;
    m->oz_slices = slices;
    const int g = choose_panels(m);
    if (g != m->G) {
      m->G = g;
      invalidate(m);
      const int64_t bi2 = int64_t(m->bi) * m->bi;
      CUDA_TRY(m->scratch.ensure(sizeof(double) * 2 * m->G * std::max<int64_t>(1, m->Ti - 1) * bi2));
    }
  }
  m->oz_slices = slices;
  return GPB_OK;
}

int gpb_model_get_ozaki(gpb_model* m, int* slices, int64_t* fallbacks) {
  GPB_TRY(check_live(m));
  if (slices) *slices = m->oz_slices;
  if (fallbacks) *fallbacks = m->oz_fallbacks;
  return GPB_OK;
}

int gpb_model_launch_count(gpb_model* m, int64_t* out) {
  if (!m || !out) return fail(GPB_INVALID_CONFIG, "null argument");
  *out = m->launches;
  return GPB_OK;
}

}  // extern "C"
