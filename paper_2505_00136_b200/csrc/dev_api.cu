// Device-level tile operations for external schedulers (C ABI, gpb200.h).
//
// The multi-GPU driver (paper_2505_00136_b200/distributed.py) keeps each
// rank's 2D block-cyclic share of the tile grid in its own device buffers and
// schedules the right-looking tiled Cholesky (taskgp tiled.py:168-204) and the
// blocked solves (tiled.py:215-260) step by step, exchanging panels with
// torch.distributed collectives.  These entry points run the same sm_100a
// kernels as the single-GPU path on caller-provided device memory and stream:
// SEK tile assembly, POTRF/TRTRI of a diagonal tile, grouped DMMA GEMM,
// batched tile GEMV and a fixed-order partial-sum combine.
#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include <cuda.h>

#include "gemm.cuh"
#include "gpb200.h"
#include "kernels.cuh"

using namespace gpb;

extern "C" int gpb_plugin_fail(int code, const char* msg);

namespace {

// Ring of device memory for per-call descriptor tables (copied in stream order).
// Tables are staged through a pinned host mirror of the ring, so the
// host-to-device copy is truly asynchronous (a pageable source could make the
// driver wait for the stream and stall the host-side scheduler).
struct DescRing {
  std::mutex mu;
  char* base = nullptr;  // device ring
  char* host = nullptr;  // pinned mirror
  size_t cap = 0, head = 0;
  void release() {
    if (base) cudaFree(base);
    if (host) cudaFreeHost(host);
    base = host = nullptr;
    cap = 0;
  }
  void* stage(const void* src, size_t bytes, cudaStream_t s, cudaError_t* err) {
    std::lock_guard<std::mutex> lk(mu);
    const size_t n = bytes;
    bytes = (bytes + 255) & ~size_t(255);
    if (!base || bytes > cap) {
      if (base) cudaDeviceSynchronize();
      release();
      const size_t want = std::max<size_t>(bytes, size_t(64) << 20);
      *err = cudaMalloc(&base, want);
      if (*err == cudaSuccess) *err = cudaMallocHost(&host, want);
      if (*err != cudaSuccess) {
        release();
        return nullptr;
      }
      cap = want;
      head = 0;
    }
    if (head + bytes > cap) {  // wrap: earlier tables may still be in flight
      cudaDeviceSynchronize();
      head = 0;
    }
    void* dst = base + head;
    std::memcpy(host + head, src, n);
    *err = cudaMemcpyAsync(dst, host + head, n, cudaMemcpyHostToDevice, s);
    head += bytes;
    return dst;
  }
};
DescRing g_ring;

#define DEV_TRY(x)                                                                       \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess) return gpb_plugin_fail(GPB_CUDA, cudaGetErrorString(e_));     \
  } while (0)

int check_ctx(gpb_ctx* ctx) {
  if (!ctx || ctx != gpb_current()) return gpb_plugin_fail(GPB_NOT_RUNNING, "runtime is not running");
  return GPB_OK;
}

SekParams make_sek(double l, double nu, double s2) {
  SekParams sp;
  sp.lengthscale = l;
  sp.vertical = nu;
  sp.noise = s2;
  sp.neg_half_inv_l2 = -1.0 / (2.0 * (l * l));
  return sp;
}

__global__ void copy_jobs_kernel(const gpb_copy_job* jobs, int64_t words16) {
  const gpb_copy_job jb = jobs[blockIdx.y];
  const double2* src = reinterpret_cast<const double2*>(jb.src);
  double2* dst = reinterpret_cast<double2*>(jb.dst);
  for (int64_t w = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; w < words16;
       w += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[w] = src[w];
}

}  // namespace

extern "C" {

// gpb_finalize: the ring belongs to the runtime's GPU
void gpb_dev_release_ring(void) {
  std::lock_guard<std::mutex> lk(g_ring.mu);
  g_ring.release();
  g_ring.head = 0;
}

int gpb_dev_copy(gpb_ctx* ctx, void* stream, const gpb_copy_job* jobs, int64_t njobs, int64_t bytes) {
  if (int s = check_ctx(ctx)) return s;
  if (njobs <= 0 || bytes <= 0) return GPB_OK;
  if (bytes % 16) return gpb_plugin_fail(GPB_DIM, "copy size must be a multiple of 16 bytes");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaSuccess;
  const void* dj = g_ring.stage(jobs, sizeof(gpb_copy_job) * njobs, st, &e);
  DEV_TRY(e);
  for (int64_t q0 = 0; q0 < njobs; q0 += 65535) {  // gridDim.y limit
    const int64_t nq = std::min<int64_t>(65535, njobs - q0);
    dim3 grid(static_cast<unsigned>(std::min<int64_t>(64, (bytes / 16 + 255) / 256)),
              static_cast<unsigned>(nq));
    copy_jobs_kernel<<<grid, 256, 0, st>>>(static_cast<const gpb_copy_job*>(dj) + q0, bytes / 16);
    DEV_TRY(cudaGetLastError());
  }
  return GPB_OK;
}

int gpb_layout(int64_t n, int64_t tiles_per_dim, int64_t out[6]) {
  if (!out) return gpb_plugin_fail(GPB_INVALID_CONFIG, "null output");
  if (tiles_per_dim < 1 || n < 1 || n % tiles_per_dim != 0)
    return gpb_plugin_fail(GPB_TILING, "tiles_per_dim must divide n");
  const int64_t b = n / tiles_per_dim;
  // Results are tiling-invariant to round-off, so the internal tile size is
  // free: 512 from n = 4096 up, else 256 (128 for n <= 128), or GPB_TILE.
  // When 128 divides the user tile the internal tile must divide n;
  // otherwise n is padded once, at the end, with decoupled identity rows
  // (not per user tile: tiny user tiles would inflate the problem).
  const char* env = getenv("GPB_TILE");
  const int64_t want = env ? atoll(env) : (n >= 4096 ? 512 : n > 128 ? 256 : 128);
  const bool dense = (b % kTileAlign == 0);
  int64_t bi = 0;
  for (int64_t c : {want, int64_t(512), int64_t(256), int64_t(128)})
    if (c > 0 && c % kTileAlign == 0 && (!dense || n % c == 0)) {
      bi = c;
      break;
    }
  const int64_t np_ = dense ? n : (n + bi - 1) / bi * bi;
  out[0] = bi;                                        // internal tile size
  out[1] = np_ / bi;                                  // internal tiles per dimension
  out[2] = np_;                                       // padded order
  out[3] = std::min<int64_t>(np_, int64_t(1) << 30);  // PadMap.bp_user: one block
  out[4] = dense ? out[3] : n;                        // PadMap.b_user: real rows P < n
  out[5] = b;                                         // user tile size
  return GPB_OK;
}

int gpb_dev_pad(gpb_ctx* ctx, void* stream, const double* src, int64_t np_, int64_t d,
                int64_t bp_user, int64_t b_user, double* dst) {
  if (int s = check_ctx(ctx)) return s;
  PadMap pm{static_cast<int>(bp_user), static_cast<int>(b_user)};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DEV_TRY(d == 0 ? launch_pad_vector(src, dst, np_, pm, st)
                 : launch_pad_rows(src, dst, np_, static_cast<int>(d), pm, st));
  return GPB_OK;
}

int gpb_dev_assemble(gpb_ctx* ctx, void* stream, const double* zp, int64_t d, int64_t b,
                     int64_t bp_user, int64_t b_user, double l, double nu, double s2,
                     int add_noise, const gpb_tile_desc* tiles, int64_t ntiles) {
  if (int s = check_ctx(ctx)) return s;
  if (ntiles <= 0) return GPB_OK;
  static_assert(sizeof(gpb_tile_desc) == sizeof(TileDesc), "descriptor layout");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaSuccess;
  const void* dd = g_ring.stage(tiles, sizeof(TileDesc) * ntiles, st, &e);
  DEV_TRY(e);
  PadMap pm{static_cast<int>(bp_user), static_cast<int>(b_user)};
  DEV_TRY(launch_assemble_desc(static_cast<const TileDesc*>(dd), ntiles, zp, static_cast<int>(d),
                               static_cast<int>(b), pm, make_sek(l, nu, s2), add_noise != 0, st));
  return GPB_OK;
}

int gpb_dev_potrf(gpb_ctx* ctx, void* stream, double* tile, double* dinv, int64_t b,
                  int64_t tile_off, int64_t bp_user, int64_t b_user, double* logdiag_out,
                  int* info_dev) {
  if (int s = check_ctx(ctx)) return s;
  PotrfArgs a{};
  a.tile = tile;
  a.dinv = dinv;
  a.logdiag = logdiag_out;
  a.info = info_dev;
  a.bi = static_cast<int>(b);
  a.tile_index = 0;
  a.tile_off = static_cast<int>(tile_off);
  a.bp_user = static_cast<int>(bp_user);
  a.b_user = static_cast<int>(b_user);
  DEV_TRY(launch_potrf(a, static_cast<cudaStream_t>(stream)));
  return GPB_OK;
}

int gpb_dev_gemm_tiled(gpb_ctx* ctx, void* stream, const gpb_gemm_job* jobs, int64_t njobs,
                       int64_t b, int64_t lda, int64_t ldb, int64_t ldc, int a_kmajor, int b_kmajor,
                       int64_t ktile, int64_t kstride, double alpha, double beta) {
  return gpb_dev_gemm_mirror(ctx, stream, jobs, njobs, b, lda, ldb, ldc, a_kmajor, b_kmajor, ktile,
                             kstride, alpha, beta, nullptr, 0);
}

int gpb_dev_gemm_mirror(gpb_ctx* ctx, void* stream, const gpb_gemm_job* jobs, int64_t njobs,
                        int64_t b, int64_t lda, int64_t ldb, int64_t ldc, int a_kmajor, int b_kmajor,
                        int64_t ktile, int64_t kstride, double alpha, double beta,
                        double* const* mirrors, int64_t nmirror) {
  if (int s = check_ctx(ctx)) return s;
  if (nmirror < 0 || (nmirror > 0 && !mirrors)) return gpb_plugin_fail(GPB_INVALID_CONFIG, "bad mirror table");
  if (njobs <= 0) return GPB_OK;
  if (b % GBM) return gpb_plugin_fail(GPB_DIM, "tile size must be a multiple of 128");
  std::vector<GemmJob> gj(njobs);
  int64_t maxk = 0;
  for (int64_t q = 0; q < njobs; ++q) {
    GemmJob g{};
    g.A = jobs[q].a;
    g.B = jobs[q].b;
    g.Cin = jobs[q].cin;
    g.Cout = jobs[q].cout;
    g.K = jobs[q].k;
    g.lower = jobs[q].lower;
    if (g.K % GBK) return gpb_plugin_fail(GPB_DIM, "K must be a multiple of 32");
    maxk = std::max<int64_t>(maxk, g.K);
    gj[q] = g;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaSuccess;
  const void* dj = g_ring.stage(gj.data(), sizeof(GemmJob) * njobs, st, &e);
  DEV_TRY(e);
  GemmParams p{};
  p.jobs = static_cast<const GemmJob*>(dj);
  p.njobs = static_cast<int>(njobs);
  p.mblk = p.nblk = static_cast<int>(b / GBM);
  p.lda = lda;
  p.ldb = ldb;
  p.ldc = ldc;
  if (ktile > 0) {
    if (!a_kmajor || !b_kmajor || ktile % GBK)
      return gpb_plugin_fail(GPB_DIM, "tiled-k walks need K-major operands and ktile % 32 == 0");
    p.a_ktile = p.b_ktile = ktile;
    p.a_kstride = p.b_kstride = kstride;
  } else {
    p.a_ktile = p.b_ktile = int64_t(1) << 40;
  }
  p.alpha = alpha;
  p.beta = beta;
  p.max_k = maxk;
  if (nmirror > 0) {
    const void* dm = g_ring.stage(mirrors, sizeof(double*) * njobs * nmirror, st, &e);
    DEV_TRY(e);
    p.mirror = static_cast<double* const*>(dm);
    p.nmirror = static_cast<int>(nmirror);
  }
  // TMA views: the operands' jobs come from arbitrary (torch) allocations, so
  // the view starts at the lowest pointer and is used only if every job's
  // block sits inside one row of the ld-wide view
  auto view = [&](bool a_side, const double** base, int64_t* extent) {
    const bool km = a_side ? a_kmajor != 0 : b_kmajor != 0;
    const int64_t ld = a_side ? lda : ldb, rows = GBM;  // rows of one block (GBM == GBN)
    const int64_t kt = a_side ? p.a_ktile : p.b_ktile, ks = a_side ? p.a_kstride : p.b_kstride;
    const double* lo = nullptr;
    for (const GemmJob& g : gj) {
      const double* q = a_side ? g.A : g.B;
      if (g.K > 0 && (!lo || q < lo)) lo = q;
    }
    if (!lo || ld <= 0) return;
    int64_t hi = 0;
    for (const GemmJob& g : gj) {
      if (g.K <= 0) continue;
      const int64_t off = (a_side ? g.A : g.B) - lo;
      const int64_t col = off % ld;
      const bool tiled = kt < (int64_t(1) << 30);
      const int64_t kspan = tiled ? std::min<int64_t>(g.K, kt) : g.K;
      const int64_t mspan = (a_side ? p.mblk : p.nblk) * rows;
      if (km ? col + kspan > ld : col + mspan > ld) return;
      const int64_t span = km ? (mspan * ld + (tiled ? (g.K / kt) * ks : 0)) : ((g.K + 1) * ld);
      hi = std::max(hi, off + span);
    }
    *base = lo;
    *extent = hi;
  };
  view(true, &p.a_base, &p.a_extent);
  view(false, &p.b_base, &p.b_extent);
  if (p.nmirror > 0 && !(a_kmajor && b_kmajor))
    return gpb_plugin_fail(GPB_INVALID_CONFIG, "mirror stores need K-major operands");
  DEV_TRY(launch_gemm(p, a_kmajor != 0, b_kmajor != 0, p.nmirror > 0 ? EPI_MIRROR : EPI_AXPBY, st));
  return GPB_OK;
}

int gpb_dev_gemm(gpb_ctx* ctx, void* stream, const gpb_gemm_job* jobs, int64_t njobs, int64_t b,
                 int64_t lda, int64_t ldb, int64_t ldc, int a_kmajor, int b_kmajor, double alpha,
                 double beta) {
  return gpb_dev_gemm_tiled(ctx, stream, jobs, njobs, b, lda, ldb, ldc, a_kmajor, b_kmajor, 0, 0,
                            alpha, beta);
}

int gpb_dev_gemv(gpb_ctx* ctx, void* stream, const gpb_gemv_job* jobs, int64_t njobs, int64_t b,
                 int trans, double alpha, int accumulate) {
  if (int s = check_ctx(ctx)) return s;
  if (njobs <= 0) return GPB_OK;
  static_assert(sizeof(gpb_gemv_job) == sizeof(GemvJob), "gemv job layout");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaSuccess;
  const void* dj = g_ring.stage(jobs, sizeof(GemvJob) * njobs, st, &e);
  DEV_TRY(e);
  DEV_TRY(launch_gemv_jobs(static_cast<const GemvJob*>(dj), njobs, static_cast<int>(b), trans,
                           alpha, accumulate, st));
  return GPB_OK;
}

int gpb_dev_combine(gpb_ctx* ctx, void* stream, const double* base, const double* parts,
                    int64_t nparts, int64_t len, double* out) {
  if (int s = check_ctx(ctx)) return s;
  DEV_TRY(launch_combine(base, parts, nparts, len, out, static_cast<cudaStream_t>(stream)));
  return GPB_OK;
}

// ---- peer memory for the fused panel exchange (distributed.py, transport "p2p")

int gpb_dev_ipc_alloc(gpb_ctx* ctx, int64_t bytes, void** ptr, void* handle) {
  if (int s = check_ctx(ctx)) return s;
  if (bytes <= 0 || !ptr || !handle) return gpb_plugin_fail(GPB_INVALID_CONFIG, "bad IPC allocation");
  void* p = nullptr;
  DEV_TRY(cudaMalloc(&p, static_cast<size_t>(bytes)));
  DEV_TRY(cudaMemset(p, 0, static_cast<size_t>(bytes)));
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) {
    cudaFree(p);
    DEV_TRY(e);
  }
  static_assert(sizeof(h) == GPB_IPC_HANDLE_BYTES, "IPC handle size");
  memcpy(handle, &h, sizeof(h));
  *ptr = p;
  return GPB_OK;
}

int gpb_dev_ipc_open(gpb_ctx* ctx, const void* handle, void** ptr) {
  if (int s = check_ctx(ctx)) return s;
  if (!handle || !ptr) return gpb_plugin_fail(GPB_INVALID_CONFIG, "bad IPC handle");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  DEV_TRY(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return GPB_OK;
}

int gpb_dev_ipc_close(gpb_ctx* ctx, void* ptr) {
  if (int s = check_ctx(ctx)) return s;
  if (ptr) DEV_TRY(cudaIpcCloseMemHandle(ptr));
  return GPB_OK;
}

int gpb_dev_free(gpb_ctx* ctx, void* ptr) {
  if (int s = check_ctx(ctx)) return s;
  if (ptr) DEV_TRY(cudaFree(ptr));
  return GPB_OK;
}

}  // extern "C"

namespace {
using StreamWrite64 = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
using StreamWait64 = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
template <class F>
F driver_fn(const char* name) {
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPointByVersion(name, &f, 12000, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(f);
}
}  // namespace

extern "C" {

// *flag = value in stream order, after a memory fence covering the stream's
// earlier work (flag may live in a peer rank's memory)
int gpb_dev_signal(gpb_ctx* ctx, void* stream, uint64_t* flag, uint64_t value) {
  if (int s = check_ctx(ctx)) return s;
  static StreamWrite64 fn = driver_fn<StreamWrite64>("cuStreamWriteValue64");
  if (!fn) return gpb_plugin_fail(GPB_CUDA, "cuStreamWriteValue64 unavailable");
  if (fn(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(flag), value, 0) != CUDA_SUCCESS)
    return gpb_plugin_fail(GPB_CUDA, "cuStreamWriteValue64 failed");
  return GPB_OK;
}

// later work on the stream waits until *flag >= value (no SM is occupied)
int gpb_dev_wait(gpb_ctx* ctx, void* stream, const uint64_t* flag, uint64_t value) {
  if (int s = check_ctx(ctx)) return s;
  static StreamWait64 fn = driver_fn<StreamWait64>("cuStreamWaitValue64");
  if (!fn) return gpb_plugin_fail(GPB_CUDA, "cuStreamWaitValue64 unavailable");
  static const unsigned flags = [] {
    int dev = 0, can = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&can, cudaDevAttrCanFlushRemoteWrites, dev);
    return can ? static_cast<unsigned>(CU_STREAM_WAIT_VALUE_FLUSH) : 0u;
  }();
  if (fn(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(flag), value,
         CU_STREAM_WAIT_VALUE_GEQ | flags) != CUDA_SUCCESS)
    return gpb_plugin_fail(GPB_CUDA, "cuStreamWaitValue64 failed");
  return GPB_OK;
}

}  // extern "C"
