// Multi-GPU runtime of the tiled GP (C ABI gpb_dist_*, include/gpb200.h).
//
// One process per GPU.  gpb_dist_init creates the library's own NCCL
// communicators (world from the caller's unique id, then ncclCommSplit into
// the process-row and process-column communicators); gpb_dist_init_host
// swaps them for caller-supplied host-staged collectives.  A model keeps only
// its rank's tiles of the 2D block-cyclic grid and runs the per-rank schedule
// of dist_plan.cu: the operation list of each phase is built once per model
// shape, its job tables are resolved to device pointers and uploaded once, and
// a call replays the list -- kernel launches on the main and critical
// streams, collectives on the row / column / world communicators -- with no
// per-step host logic beyond the launch itself.
//
// Replaces the reference's task runtime and model layer across GPUs
// (taskgp runtime.py:369-403, tiled.py:168-324, model.py:169-485).
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "dist_plan.h"
#include "ozaki.cuh"
#include "gemm.cuh"
#include "gpb200.h"
#include "kernels.cuh"

using namespace gpb;

extern "C" int gpb_plugin_fail(int code, const char* msg);

namespace {

int fail(int code, const std::string& msg) { return gpb_plugin_fail(code, msg.c_str()); }

#define DCUDA(x)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess)                                                                \
      return fail(e_ == cudaErrorMemoryAllocation ? GPB_NO_MEMORY : GPB_CUDA,             \
                  std::string(#x) + ": " + cudaGetErrorString(e_));                       \
  } while (0)
#define DTRY(x)                  \
  do {                           \
    int s_ = (x);                \
    if (s_ != GPB_OK) return s_; \
  } while (0)

constexpr double kHalfLog2Pi = 0.91893853320467274178;  // model.py:35

// ---- NCCL, loaded at run time ----------------------------------------------
// The few declarations used here (nccl.h 2.18+ ABI; ncclComm_t is opaque).
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[GPB_NCCL_ID_BYTES];
} ncclUniqueId;
typedef int ncclResult_t;  // 0 = ncclSuccess
constexpr int kNcclFloat64 = 8, kNcclSum = 0;

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, void*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Reduce)(const void*, void*, size_t, int, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  std::string err;
  bool load() {
    if (h) return true;
    const char* env = getenv("GPB_NCCL_LIB");
    for (const char* name : {env, "libnccl.so.2", "libnccl.so"}) {
      if (!name) continue;
      h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) {
      err = "cannot load NCCL (set GPB_NCCL_LIB): ";
      err += dlerror();
      return false;
    }
#define GPB_SYM(f)                                                                  \
  f = reinterpret_cast<decltype(f)>(dlsym(h, "nccl" #f));                           \
  if (!f) {                                                                         \
    err = "NCCL lacks nccl" #f;                                                     \
    return false;                                                                   \
  }
    GPB_SYM(GetUniqueId)
    GPB_SYM(CommInitRank)
    GPB_SYM(CommSplit)
    GPB_SYM(CommDestroy)
    GPB_SYM(Broadcast)
    GPB_SYM(Reduce)
    GPB_SYM(AllReduce)
    GPB_SYM(GroupStart)
    GPB_SYM(GroupEnd)
    GPB_SYM(GetErrorString)
#undef GPB_SYM
    return true;
  }
};
NcclApi g_nccl;

// ---- collectives -------------------------------------------------------------
struct Transport {
  virtual ~Transport() {}
  virtual int bcast(int group, double* buf, int64_t count, int root, cudaStream_t s) = 0;
  virtual int reduce(int group, double* buf, int64_t count, int root, cudaStream_t s) = 0;
  virtual int allreduce(int group, double* buf, int64_t count, cudaStream_t s) = 0;
  int64_t calls = 0;
};

struct NcclTransport : Transport {
  ncclComm_t comm[3] = {nullptr, nullptr, nullptr};
  ~NcclTransport() override {
    for (int g = 2; g >= 0; --g)
      if (comm[g]) g_nccl.CommDestroy(comm[g]);
  }
  int check(ncclResult_t r, const char* what) {
    if (r == 0) return GPB_OK;
    return fail(GPB_NCCL, std::string(what) + ": " + g_nccl.GetErrorString(r));
  }
  int bcast(int group, double* buf, int64_t count, int root, cudaStream_t s) override {
    ++calls;
    return check(g_nccl.Broadcast(buf, buf, size_t(count), kNcclFloat64, root, comm[group], s), "ncclBroadcast");
  }
  int reduce(int group, double* buf, int64_t count, int root, cudaStream_t s) override {
    ++calls;
    return check(g_nccl.Reduce(buf, buf, size_t(count), kNcclFloat64, kNcclSum, root, comm[group], s),
                 "ncclReduce");
  }
  int allreduce(int group, double* buf, int64_t count, cudaStream_t s) override {
    ++calls;
    return check(g_nccl.AllReduce(buf, buf, size_t(count), kNcclFloat64, kNcclSum, comm[group], s),
                 "ncclAllReduce");
  }
};

// host-staged collectives supplied by the caller: the stream is drained, the
// buffer copied to pinned host memory, the callback runs, the result is copied back
struct HostTransport : Transport {
  gpb_host_coll cb{};
  double* host = nullptr;
  int64_t cap = 0;
  ~HostTransport() override {
    if (host) cudaFreeHost(host);
  }
  int stage(const double* dev, int64_t count, cudaStream_t s) {
    if (count > cap) {
      if (host) cudaFreeHost(host);
      host = nullptr;
      cap = 0;
      DCUDA(cudaMallocHost(&host, sizeof(double) * count));
      cap = count;
    }
    DCUDA(cudaStreamSynchronize(s));
    DCUDA(cudaMemcpy(host, dev, sizeof(double) * count, cudaMemcpyDeviceToHost));
    return GPB_OK;
  }
  int unstage(double* dev, int64_t count) {
    DCUDA(cudaMemcpy(dev, host, sizeof(double) * count, cudaMemcpyHostToDevice));
    return GPB_OK;
  }
  int bcast(int group, double* buf, int64_t count, int root, cudaStream_t s) override {
    ++calls;
    DTRY(stage(buf, count, s));
    if (cb.bcast(cb.user, group, host, count * 8, root) != 0) return fail(GPB_NCCL, "host broadcast failed");
    return unstage(buf, count);
  }
  int reduce(int group, double* buf, int64_t count, int root, cudaStream_t s) override {
    ++calls;
    DTRY(stage(buf, count, s));
    if (cb.reduce_sum(cb.user, group, host, count, root) != 0) return fail(GPB_NCCL, "host reduce failed");
    return unstage(buf, count);
  }
  int allreduce(int group, double* buf, int64_t count, cudaStream_t s) override {
    ++calls;
    DTRY(stage(buf, count, s));
    if (cb.allreduce_sum(cb.user, group, host, count) != 0) return fail(GPB_NCCL, "host all-reduce failed");
    return unstage(buf, count);
  }
};

// stream-ordered delay of `ns` nanoseconds (one thread polls the global timer)
__global__ void delay_kernel(unsigned long long ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  do {
    __nanosleep(200);
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

// No data exchange at all: one rank's schedule run alone on a GPU to time its
// own kernels (gpb_dist_init_emulate).  Results are meaningless.  With
// GPB_EMU_LINK="latency_us,GB/s" every collective instead occupies its stream for
// latency + bytes / bandwidth (a modelled NVLink transfer, no data moved).
struct NullTransport : Transport {
  double lat_ns = 0.0, gbs = 0.0;
  NullTransport() {
    if (const char* e = getenv("GPB_EMU_LINK")) {
      double lat = 0.0, bw = 0.0;
      if (sscanf(e, "%lf,%lf", &lat, &bw) == 2 && bw > 0.0) {
        lat_ns = lat * 1e3;
        gbs = bw;
      }
    }
  }
  int wait(int64_t bytes, cudaStream_t s) {
    ++calls;
    if (gbs <= 0.0) return GPB_OK;
    delay_kernel<<<1, 1, 0, s>>>(static_cast<unsigned long long>(lat_ns + double(bytes) / gbs));
    DCUDA(cudaGetLastError());
    return GPB_OK;
  }
  int bcast(int, double*, int64_t count, int, cudaStream_t s) override { return wait(count * 8, s); }
  int reduce(int, double*, int64_t count, int, cudaStream_t s) override { return wait(count * 8, s); }
  int allreduce(int, double*, int64_t count, cudaStream_t s) override { return wait(2 * count * 8, s); }
};

struct CopyJob {
  const double* src;
  double* dst;
};

__global__ void dist_copy_kernel(const CopyJob* jobs, int64_t words16) {
  const CopyJob jb = jobs[blockIdx.y];
  const double2* src = reinterpret_cast<const double2*>(jb.src);
  double2* dst = reinterpret_cast<double2*>(jb.dst);
  for (int64_t w = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; w < words16;
       w += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[w] = src[w];
}

__global__ void dist_copy_small_kernel(const CopyJob* jobs, int64_t count) {  // odd sizes
  const CopyJob jb = jobs[blockIdx.y];
  for (int64_t w = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; w < count;
       w += static_cast<int64_t>(gridDim.x) * blockDim.x)
    jb.dst[w] = jb.src[w];
}

// A phase's operation list with its job tables resolved and resident in HBM.
struct Phase {
  std::vector<gpb_op> ops;
  std::vector<int64_t> table;  // per op: byte offset of its device table, or -1
  std::vector<int64_t> mirror; // per GEMM op: byte offset of its mirror-store table, or -1
  std::vector<int> nmirror;    // ... and its stores per job
  void* dev = nullptr;
  size_t bytes = 0;
  std::vector<int64_t> oz_table;  // per op: offset of the OzakiJob table of a flagged GEMM (-1: none)
  std::vector<int> oz_k;          // ... and its depth K
  int64_t launches_per_run = 0;
  ~Phase() {
    if (dev) cudaFree(dev);
  }
};

}  // namespace

struct gpb_dist {
  gpb_ctx* ctx = nullptr;
  int rank = 0, world = 1, P = 1, Q = 1;
  int exchange = 0;  // gpb_dist_set_exchange: 0 collectives, 1 peer memory
  int models = 0;    // live models (finalize refuses while any remains)
  Transport* tr = nullptr;
};

struct gpb_dmodel {
  gpb_dist* dc = nullptr;
  DistLayout L;
  int64_t n = 0, d = 0, T = 0;
  PadMap pm{};
  double l = 1.0, nu = 1.0, s2 = 0.1;
  uint8_t trainable[3] = {1, 1, 1};
  cudaStream_t st = nullptr, crit = nullptr;
  std::vector<cudaEvent_t> ev;
  cudaEvent_t t0 = nullptr, t1 = nullptr, ta = nullptr;  // ta: end of the assembly (phase 0)
  double* buf[GPB_NBUF] = {nullptr};
  double *z = nullptr, *y = nullptr, *zp = nullptr;  // replicated training data (z, y as given; zp padded)
  int* info = nullptr;
  double* parts = nullptr;  // trace partials
  double* red = nullptr;    // small reductions (loss terms)
  int* flow_flags = nullptr;
  double* flow_x = nullptr;
  Phase ph[3];
  bool planned[3] = {false, false, false};
  bool factor_ok = false;
  int64_t last_pivot = -1;
  double timing[8] = {0};
  int64_t launches = 0;
  double adam_m[3] = {0, 0, 0}, adam_v[3] = {0, 0, 0};
  int64_t adam_step = 0;
  gpb_model* rep = nullptr;  // local replica of the factor for sharded prediction
  bool rep_ok = false;
  // peer-memory panel exchange (L.p2p): this rank's flag words (ready[src] at
  // src, free[src] at world + src) and every peer's row panel, column panel and
  // flags mapped through CUDA IPC
  // digit planes of the row / column panels (L.planes > 0; boxed layout, tile t of the panel
  // buffer at t * bi2 * planes bytes) and the saturation flag of the slicing kernels
  int8_t* planes[GPB_NBUF] = {nullptr};
  int* ozflag = nullptr;
  uint64_t* flags = nullptr;
  std::vector<void*> peer_row, peer_col, peer_flags;
  bool p2p_ready = false;
  uint64_t epoch = 0;
};

namespace {

SekParams sek(const gpb_dmodel* m) {
  SekParams sp;
  sp.lengthscale = m->l;
  sp.vertical = m->nu;
  sp.noise = m->s2;
  sp.neg_half_inv_l2 = -1.0 / (2.0 * (m->l * m->l));
  return sp;
}

double* ref(gpb_dmodel* m, int b, int64_t off) { return b < 0 ? nullptr : m->buf[b] + off; }

int ensure_buffers(gpb_dmodel* m, std::initializer_list<int> ids) {
  for (int b : ids) {
    if (m->buf[b] || m->L.bufsz[b] == 0) continue;
    DCUDA(cudaMalloc(&m->buf[b], sizeof(double) * m->L.bufsz[b]));
    DCUDA(cudaMemset(m->buf[b], 0, sizeof(double) * m->L.bufsz[b]));
  }
  return GPB_OK;
}

// Build the op list of a phase and upload its resolved job tables.
int build_phase(gpb_dmodel* m, int phase) {
  if (m->planned[phase]) return GPB_OK;
  Phase& P = m->ph[phase];
  std::vector<gpb_op_job> jobs;
  P.ops.clear();
  dist_plan(m->L, phase, &P.ops, &jobs);
  std::vector<char> host;
  auto align = [&]() { host.resize((host.size() + 15) & ~size_t(15)); };
  P.table.assign(P.ops.size(), -1);
  P.mirror.assign(P.ops.size(), -1);
  P.nmirror.assign(P.ops.size(), 0);
  P.oz_table.assign(P.ops.size(), -1);
  P.oz_k.assign(P.ops.size(), 0);
  P.launches_per_run = 0;
  for (size_t q = 0; q < P.ops.size(); ++q) {
    const gpb_op& o = P.ops[q];
    const gpb_op_job* J = jobs.data() + o.job0;
    auto put = [&](const void* p, size_t n) {
      const size_t at = host.size();
      host.resize(at + n);
      memcpy(host.data() + at, p, n);
    };
    switch (o.kind) {
      case GPB_OP_MIRROR: {  // extra output stores of the preceding GEMM (peer panel buffers)
        if (q == 0 || P.ops[q - 1].kind != GPB_OP_GEMM || !m->p2p_ready)
          return fail(GPB_INVALID_CONFIG, "mirror stores without a preceding GEMM or peer mappings");
        const int64_t ng = P.ops[q - 1].njobs;
        std::vector<int> per(ng, 0);
        for (int64_t t = 0; t < o.njobs; ++t) ++per[J[t].k];
        const int nm = *std::max_element(per.begin(), per.end());
        std::vector<double*> tab(ng * nm, nullptr);
        std::fill(per.begin(), per.end(), 0);
        for (int64_t t = 0; t < o.njobs; ++t) {
          const int r = J[t].i, b = J[t].buf[3];
          if (b != GPB_BUF_ROW && b != GPB_BUF_COL) return fail(GPB_INVALID_CONFIG, "mirror outside the panels");
          char* base = r == m->L.rank ? reinterpret_cast<char*>(m->buf[b])
                                      : static_cast<char*>(b == GPB_BUF_ROW ? m->peer_row[r] : m->peer_col[r]);
          tab[J[t].k * nm + per[J[t].k]++] = reinterpret_cast<double*>(base) + J[t].off[3];
        }
        align();
        P.mirror[q - 1] = static_cast<int64_t>(host.size());
        P.nmirror[q - 1] = nm;
        put(tab.data(), sizeof(double*) * tab.size());
        break;
      }
      case GPB_OP_GEMM: {
        align();
        P.table[q] = static_cast<int64_t>(host.size());
        // TMA operand views: the buffer every A (B) of the launch lies in, or -1
        int ba = J[0].buf[0], bb = J[0].buf[1];
        for (int64_t t = 1; t < o.njobs; ++t) {
          if (J[t].buf[0] != ba) ba = -1;
          if (J[t].buf[1] != bb) bb = -1;
        }
        P.ops[q].buf[0] = ba;
        P.ops[q].buf[1] = bb;
        for (int64_t t = 0; t < o.njobs; ++t) {
          GemmJob g{};
          g.A = ref(m, J[t].buf[0], J[t].off[0]);
          g.B = ref(m, J[t].buf[1], J[t].off[1]);
          g.Cin = ref(m, J[t].buf[2], J[t].off[2]);
          g.Cout = ref(m, J[t].buf[3], J[t].off[3]);
          g.K = J[t].k;
          g.lower = J[t].lower;
          put(&g, sizeof(g));
        }
        if (o.flag && m->L.planes > 0 && (ba == GPB_BUF_ROW || ba == GPB_BUF_COL) &&
            (bb == GPB_BUF_ROW || bb == GPB_BUF_COL)) {
          // the same jobs for the digit-plane product: byte offsets into the panels' planes
          align();
          P.oz_table[q] = static_cast<int64_t>(host.size());
          P.oz_k[q] = J[0].k;
          for (int64_t t = 0; t < o.njobs; ++t) {
            OzakiJob z{};
            z.a_off = J[t].off[0] * m->L.planes;
            z.b_off = J[t].off[1] * m->L.planes;
            z.C = ref(m, J[t].buf[3], J[t].off[3]);
            z.lower = J[t].lower;
            put(&z, sizeof(z));
          }
          ++P.launches_per_run;  // two group windows
        }
        ++P.launches_per_run;
        break;
      }
      case GPB_OP_SLICE:
        ++P.launches_per_run;
        break;
      case GPB_OP_COPY: {
        align();
        P.table[q] = static_cast<int64_t>(host.size());
        for (int64_t t = 0; t < o.njobs; ++t) {
          CopyJob c{ref(m, J[t].buf[0], J[t].off[0]), ref(m, J[t].buf[3], J[t].off[3])};
          put(&c, sizeof(c));
        }
        ++P.launches_per_run;
        break;
      }
      case GPB_OP_GEMV: {
        align();
        P.table[q] = static_cast<int64_t>(host.size());
        for (int64_t t = 0; t < o.njobs; ++t) {
          GemvJob v{ref(m, J[t].buf[0], J[t].off[0]), ref(m, J[t].buf[1], J[t].off[1]),
                    ref(m, J[t].buf[3], J[t].off[3])};
          put(&v, sizeof(v));
        }
        ++P.launches_per_run;
        break;
      }
      case GPB_OP_ASSEMBLE: {
        align();
        P.table[q] = static_cast<int64_t>(host.size());
        for (int64_t t = 0; t < o.njobs; ++t) {
          TileDesc d{J[t].i, J[t].j, ref(m, J[t].buf[3], J[t].off[3])};
          put(&d, sizeof(d));
        }
        ++P.launches_per_run;
        break;
      }
      case GPB_OP_TRACE: {
        align();
        P.table[q] = static_cast<int64_t>(host.size());
        for (int64_t t = 0; t < o.njobs; ++t) {
          int2 ij = make_int2(J[t].i, J[t].j);
          put(&ij, sizeof(ij));
        }
        P.launches_per_run += 4;
        break;
      }
      case GPB_OP_POTRF:
      case GPB_OP_COMBINE:
      case GPB_OP_SOLVE_FLOW:
        ++P.launches_per_run;
        break;
      default:
        break;
    }
  }
  if (P.dev) cudaFree(P.dev);
  P.dev = nullptr;
  P.bytes = std::max<size_t>(host.size(), 16);
  DCUDA(cudaMalloc(&P.dev, P.bytes));
  if (!host.empty()) DCUDA(cudaMemcpy(P.dev, host.data(), host.size(), cudaMemcpyHostToDevice));
  m->planned[phase] = true;
  return GPB_OK;
}

int launch_copies(const CopyJob* jobs, int64_t njobs, int64_t count, cudaStream_t s) {
  for (int64_t q0 = 0; q0 < njobs; q0 += 65535) {
    const int64_t nq = std::min<int64_t>(65535, njobs - q0);
    if (count % 2 == 0) {
      dim3 grid(static_cast<unsigned>(std::min<int64_t>(64, (count / 2 + 255) / 256)), static_cast<unsigned>(nq));
      dist_copy_kernel<<<grid, 256, 0, s>>>(jobs + q0, count / 2);
    } else {
      dim3 grid(static_cast<unsigned>(std::min<int64_t>(64, (count + 255) / 256)), static_cast<unsigned>(nq));
      dist_copy_small_kernel<<<grid, 256, 0, s>>>(jobs + q0, count);
    }
    DCUDA(cudaGetLastError());
  }
  return GPB_OK;
}

// Replay one phase.
int run_phase(gpb_dmodel* m, int phase, double* enqueue_us = nullptr) {
  Phase& P = m->ph[phase];
  const DistLayout& L = m->L;
  const char* dev = static_cast<const char*>(P.dev);
  const auto h0 = std::chrono::steady_clock::now();
  if (phase == 0) DCUDA(cudaEventRecord(m->ta, m->st));  // re-recorded after the assembly
  for (size_t q = 0; q < P.ops.size(); ++q) {
    const gpb_op& o = P.ops[q];
    cudaStream_t s = o.stream ? m->crit : m->st;
    const void* tab = P.table[q] >= 0 ? dev + P.table[q] : nullptr;
    switch (o.kind) {
      case GPB_OP_ZERO:
        DCUDA(cudaMemsetAsync(ref(m, o.buf[0], o.off[0]), 0, sizeof(double) * o.count, s));
        break;
      case GPB_OP_RECORD:
        DCUDA(cudaEventRecord(m->ev[o.i], s));
        break;
      case GPB_OP_WAIT:
        DCUDA(cudaStreamWaitEvent(s, m->ev[o.i], 0));
        break;
      case GPB_OP_ASSEMBLE:
        DCUDA(launch_assemble_desc(static_cast<const TileDesc*>(tab), o.njobs, m->zp, static_cast<int>(m->d),
                                   L.bi, m->pm, sek(m), o.flag != 0, s));
        ++m->launches;
        if (phase == 0) DCUDA(cudaEventRecord(m->ta, s));
        break;
      case GPB_OP_POTRF: {
        PotrfArgs a{};
        a.tile = ref(m, o.buf[0], o.off[0]);
        a.dinv = ref(m, o.buf[1], o.off[1]);
        a.logdiag = m->buf[GPB_BUF_VEC] + L.vec[V_LOGDIAG];
        a.info = m->info;
        a.bi = L.bi;
        a.tile_index = o.i;
        a.tile_off = o.i * L.bi;
        a.bp_user = m->pm.bp_user;
        a.b_user = m->pm.b_user;
        a.tiles = L.Ti;  // the same cluster-size hints as the single-GPU plan
        a.remaining = L.Ti - o.i;
        DCUDA(launch_potrf(a, s));
        ++m->launches;
        break;
      }
      case GPB_OP_SLICE: {
        const double scale = ozaki_plane_scale(std::max(1.0, std::sqrt(m->nu + m->s2)));
        DCUDA(launch_ozaki_slice_tiles(ref(m, o.buf[0], o.off[0]), o.count, L.bi, L.bi, scale,
                                       m->planes[o.buf[0]] + o.off[0] * L.planes, L.planes, m->ozflag, s));
        ++m->launches;
        break;
      }
      case GPB_OP_GEMM: {
        if (P.oz_table[q] >= 0) {
          // L(i,j) -= [X]_i [X]_j^T from the digit planes of the row and column panels
          const double scale = ozaki_plane_scale(std::max(1.0, std::sqrt(m->nu + m->s2)));
          const int kc = L.bi / kOzakiBK;
          OzakiGemm g{};
          g.a = {m->planes[o.buf[0]], o.a_kstride * L.planes, kc, int64_t(kc) * L.planes * kOzakiBox};
          g.b = {m->planes[o.buf[1]], o.b_kstride * L.planes, kc, int64_t(kc) * L.planes * kOzakiBox};
          g.M = g.N = L.bi;
          g.K = P.oz_k[q];
          g.slices = L.planes;
          g.alpha = o.alpha * scale * scale;
          g.beta = o.beta;
          g.ldc_in = g.ldc_out = o.ldc;
          g.jobs = reinterpret_cast<const OzakiJob*>(dev + P.oz_table[q]);
          g.njobs = static_cast<int>(o.njobs);
          DCUDA(launch_ozaki_gemm(g, s));
          m->launches += L.planes > 4 ? 2 : 1;
          break;
        }
        GemmParams p{};
        p.jobs = static_cast<const GemmJob*>(tab);
        p.njobs = static_cast<int>(o.njobs);
        p.mblk = o.mblk;
        p.nblk = o.nblk;
        p.lda = o.lda;
        p.ldb = o.ldb;
        p.ldc = o.ldc;
        p.a_ktile = o.a_ktile > 0 ? o.a_ktile : int64_t(1) << 40;
        p.a_kstride = o.a_kstride;
        p.b_ktile = o.b_ktile > 0 ? o.b_ktile : int64_t(1) << 40;
        p.b_kstride = o.b_kstride;
        p.alpha = o.alpha;
        p.beta = o.beta;
        // TMA views: the buffers every A / B of the launch lies in (build_phase)
        const int ba = o.buf[0], bb = o.buf[1];
        p.a_base = ba >= 0 ? m->buf[ba] : nullptr;
        p.a_extent = ba >= 0 ? L.bufsz[ba] : 0;
        p.b_base = bb >= 0 ? m->buf[bb] : nullptr;
        p.b_extent = bb >= 0 ? L.bufsz[bb] : 0;
        int epi = EPI_AXPBY;
        if (P.mirror[q] >= 0) {  // fused panel exchange: stores into the peers' panels
          p.mirror = reinterpret_cast<double* const*>(dev + P.mirror[q]);
          p.nmirror = P.nmirror[q];
          epi = EPI_MIRROR;
        }
        DCUDA(launch_gemm(p, o.ak != 0, o.bk != 0, epi, s));
        ++m->launches;
        break;
      }
      case GPB_OP_MIRROR:  // merged into the preceding GEMM launch
        break;
      case GPB_OP_SIGNAL: {
        uint64_t* f = static_cast<uint64_t*>(m->peer_flags[o.i]) + int64_t(o.j) * L.world + L.rank;
        DTRY(gpb_dev_signal(m->dc->ctx, s, f, (m->epoch << 24) + static_cast<uint64_t>(o.count)));
        break;
      }
      case GPB_OP_WAITFLAG: {
        const uint64_t* f = m->flags + int64_t(o.j) * L.world + o.i;
        DTRY(gpb_dev_wait(m->dc->ctx, s, f, (m->epoch << 24) + static_cast<uint64_t>(o.count)));
        break;
      }
      case GPB_OP_COPY:
        DTRY(launch_copies(static_cast<const CopyJob*>(tab), o.njobs, o.count, s));
        ++m->launches;
        break;
      case GPB_OP_GEMV:
        DCUDA(launch_gemv_jobs(static_cast<const GemvJob*>(tab), o.njobs, L.bi, o.flag, o.alpha,
                               o.beta != 0.0 ? 1 : 0, s));
        ++m->launches;
        break;
      case GPB_OP_COMBINE:
        DCUDA(launch_combine(ref(m, o.buf[0], o.off[0]), ref(m, o.buf[1], o.off[1]), 1, o.count,
                             ref(m, o.buf[2], o.off[2]), s));
        ++m->launches;
        break;
      case GPB_OP_BCAST:
        DTRY(m->dc->tr->bcast(o.group, ref(m, o.buf[0], o.off[0]), o.count, o.root, s));
        break;
      case GPB_OP_REDUCE:
        DTRY(m->dc->tr->reduce(o.group, ref(m, o.buf[0], o.off[0]), o.count, o.root, s));
        break;
      case GPB_OP_ALLREDUCE:
        DTRY(m->dc->tr->allreduce(o.group, ref(m, o.buf[0], o.off[0]), o.count, s));
        break;
      case GPB_OP_SOLVE_FLOW: {
        double* vec = m->buf[GPB_BUF_VEC];
        const double* Lt = m->buf[GPB_BUF_L];
        const double* D = m->buf[GPB_BUF_DINV];
        double* beta = vec + L.vec[V_BETA];
        double* alpha = vec + L.vec[V_ALPHA];
        bool launched = false;
        const int R = solve_flow_slice_rows(L.np_, L.bi);
        if (R > 0)
          DCUDA(launch_solve_flow(Lt, D, vec + L.vec[V_Y], beta, alpha, m->flow_x, m->flow_flags, L.Ti, L.bi, R,
                                  s, &launched));
        if (launched) {
          ++m->launches;
          break;
        }
        // multi-launch fallback (one rank holds the packed row-major factor)
        const int64_t bi2 = L.bi2;
        double* yhat = m->flow_x;
        double* bhat = vec + L.vec[V_ACC];
        DCUDA(cudaMemcpyAsync(yhat, vec + L.vec[V_Y], sizeof(double) * L.np_, cudaMemcpyDeviceToDevice, s));
        for (int i = 0; i < L.Ti; ++i) {
          DCUDA(launch_fwd_diag(D + i * bi2, yhat + int64_t(i) * L.bi, beta + int64_t(i) * L.bi, L.bi, s));
          DCUDA(launch_fwd_update(Lt, L.Ti, i, L.bi, beta + int64_t(i) * L.bi, yhat, s));
        }
        DCUDA(cudaMemcpyAsync(bhat, beta, sizeof(double) * L.np_, cudaMemcpyDeviceToDevice, s));
        for (int i = L.Ti - 1; i >= 0; --i) {
          DCUDA(launch_bwd_diag(D + i * bi2, bhat + int64_t(i) * L.bi, alpha + int64_t(i) * L.bi, L.bi, s));
          DCUDA(launch_bwd_update(Lt, i, L.bi, alpha + int64_t(i) * L.bi, bhat, s));
        }
        m->launches += 4 * L.Ti;
        break;
      }
      case GPB_OP_TRACE: {
        const int64_t nblk = o.njobs * (L.bi / kSekBlock) * (L.bi / kSekBlock);
        double* pl = m->parts;
        double* pv = pl + nblk;
        double* pt = pv + nblk;
        double* out = ref(m, o.buf[2], o.off[2]);
        DCUDA(launch_trace(m->buf[GPB_BUF_KINV], static_cast<const int2*>(tab), o.njobs, TraceTiles{0, 0, 0, nullptr},
                           m->zp, m->buf[GPB_BUF_VEC] + L.vec[V_ALPHA], static_cast<int>(m->d), L.bi, m->pm,
                           sek(m), pl, pv, pt, s));
        DCUDA(launch_reduce(pl, nblk, out + 0, s));
        DCUDA(launch_reduce(pv, nblk, out + 1, s));
        DCUDA(launch_reduce(pt, nblk, out + 2, s));
        m->launches += 4;
        break;
      }
      default:
        return fail(GPB_INVALID_CONFIG, "unknown schedule operation " + std::to_string(o.kind));
    }
  }
  if (enqueue_us)
    *enqueue_us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - h0).count();
  return GPB_OK;
}

int check_model(gpb_dmodel* m) {
  if (!m || !m->dc) return fail(GPB_INVALID_CONFIG, "null model");
  if (gpb_current() != m->dc->ctx) return fail(GPB_NOT_RUNNING, "the runtime this model was bound to is not running");
  return GPB_OK;
}

float elapsed(gpb_dmodel* m) {
  float ms = 0;
  cudaEventElapsedTime(&ms, m->t0, m->t1);
  return ms;
}

// Peer-memory exchange: export this rank's panel buffers and flag words
// (CUDA IPC), broadcast the handles rank by rank, map every peer's.
int setup_p2p(gpb_dmodel* m) {
  if (m->p2p_ready) return GPB_OK;
  const DistLayout& L = m->L;
  const int W = L.world;
  DCUDA(cudaMalloc(&m->flags, sizeof(uint64_t) * 2 * W));
  DCUDA(cudaMemset(m->flags, 0, sizeof(uint64_t) * 2 * W));
  constexpr int kH = sizeof(cudaIpcMemHandle_t);  // 64 bytes = 8 doubles
  static_assert(kH % 8 == 0, "IPC handle size");
  constexpr int kSlot = 3 * kH / 8;                // doubles per rank: row, column, flags
  std::vector<cudaIpcMemHandle_t> mine(3);
  memset(mine.data(), 0, sizeof(cudaIpcMemHandle_t) * 3);
  DCUDA(cudaIpcGetMemHandle(&mine[0], m->buf[GPB_BUF_ROW]));
  if (m->buf[GPB_BUF_COL]) DCUDA(cudaIpcGetMemHandle(&mine[1], m->buf[GPB_BUF_COL]));
  DCUDA(cudaIpcGetMemHandle(&mine[2], m->flags));
  double* dh = nullptr;
  DCUDA(cudaMalloc(&dh, sizeof(double) * kSlot * W));
  std::vector<double> all(size_t(kSlot) * W, 0.0);
  memcpy(all.data() + size_t(kSlot) * L.rank, mine.data(), 3 * kH);
  DCUDA(cudaMemcpy(dh, all.data(), sizeof(double) * all.size(), cudaMemcpyHostToDevice));
  int s = GPB_OK;
  for (int r = 0; r < W && s == GPB_OK; ++r) s = m->dc->tr->bcast(0, dh + size_t(kSlot) * r, kSlot, r, m->st);
  if (s == GPB_OK && cudaStreamSynchronize(m->st) == cudaSuccess)
    cudaMemcpy(all.data(), dh, sizeof(double) * all.size(), cudaMemcpyDeviceToHost);
  cudaFree(dh);
  DTRY(s);
  m->peer_row.assign(W, nullptr);
  m->peer_col.assign(W, nullptr);
  m->peer_flags.assign(W, nullptr);
  for (int r = 0; r < W; ++r) {
    if (r == L.rank) {
      m->peer_row[r] = m->buf[GPB_BUF_ROW];
      m->peer_col[r] = m->buf[GPB_BUF_COL];
      m->peer_flags[r] = m->flags;
      continue;
    }
    cudaIpcMemHandle_t h[3];
    memcpy(h, all.data() + size_t(kSlot) * r, 3 * kH);
    DCUDA(cudaIpcOpenMemHandle(&m->peer_row[r], h[0], cudaIpcMemLazyEnablePeerAccess));
    if (L.P > 1) DCUDA(cudaIpcOpenMemHandle(&m->peer_col[r], h[1], cudaIpcMemLazyEnablePeerAccess));
    DCUDA(cudaIpcOpenMemHandle(&m->peer_flags[r], h[2], cudaIpcMemLazyEnablePeerAccess));
  }
  m->p2p_ready = true;
  return GPB_OK;
}

// collective: no peer may still store into this rank's panels when they are freed
void teardown_p2p(gpb_dmodel* m) {
  if (!m->p2p_ready) return;
  cudaDeviceSynchronize();
  m->dc->tr->allreduce(0, m->red, 1, m->st);  // every rank has drained its streams
  cudaStreamSynchronize(m->st);
  for (int r = 0; r < m->L.world; ++r) {
    if (r == m->L.rank) continue;
    for (void* p : {m->peer_row[r], m->peer_col[r], m->peer_flags[r]})
      if (p) cudaIpcCloseMemHandle(p);
  }
  m->dc->tr->allreduce(0, m->red, 1, m->st);  // every mapping closed before the owners free
  cudaStreamSynchronize(m->st);
  m->p2p_ready = false;
}

// assemble + factor + solves (model.py:169-186 _ensure_factor / _ensure_weights)
int ensure_factor(gpb_dmodel* m) {
  if (m->factor_ok) return GPB_OK;
  const DistLayout& L = m->L;
  if (L.p2p) DTRY(setup_p2p(m));
  ++m->epoch;  // flag values grow across factorisations: nothing is reset
  DTRY(build_phase(m, 0));
  DTRY(build_phase(m, 1));
  m->rep_ok = false;
  const int64_t calls0 = m->dc->tr->calls;
  DCUDA(cudaMemsetAsync(m->info, 0xff, sizeof(int), m->st));
  DCUDA(cudaEventRecord(m->t0, m->st));
  double enq = 0.0;
  DTRY(run_phase(m, 0, &enq));
  DCUDA(cudaEventRecord(m->t1, m->st));
  DCUDA(cudaEventSynchronize(m->t1));
  {  // [0] assembly, [1] factorisation (K resident in HBM to the factor complete)
    float a = 0, f = 0;
    cudaEventElapsedTime(&a, m->t0, m->ta);
    cudaEventElapsedTime(&f, m->ta, m->t1);
    m->timing[0] = a;
    m->timing[1] = f;
  }
  m->timing[6] = enq / std::max(1, L.Ti);
  // smallest failing pivot over the ranks (each rank's value in its own slot)
  int info = -1;
  DCUDA(cudaMemcpy(&info, m->info, sizeof(int), cudaMemcpyDeviceToHost));
  double* red = m->red;
  std::vector<double> v(L.world, -1.0);
  if (L.world > 1) {
    std::vector<double> mine(L.world, 0.0);
    mine[L.rank] = double(info) + 2.0;  // > 0 marks this rank's slot
    DCUDA(cudaMemcpy(red, mine.data(), sizeof(double) * L.world, cudaMemcpyHostToDevice));
    DTRY(m->dc->tr->allreduce(0, red, L.world, m->st));
    DCUDA(cudaMemcpyAsync(mine.data(), red, sizeof(double) * L.world, cudaMemcpyDeviceToHost, m->st));
    DCUDA(cudaStreamSynchronize(m->st));
    for (int r = 0; r < L.world; ++r) v[r] = mine[r] - 2.0;
  } else {
    v[0] = info;
  }
  int64_t piv = -1;
  for (double x : v)
    if (x >= 0 && (piv < 0 || int64_t(x) < piv)) piv = int64_t(x);
  if (piv >= 0) {
    m->last_pivot = piv;
    return fail(GPB_NOT_PD, "Matrix is not positive definite (non-positive pivot at index " + std::to_string(piv) + ")");
  }
  m->last_pivot = -1;
  DCUDA(cudaEventRecord(m->t0, m->st));
  DTRY(run_phase(m, 1));
  DCUDA(cudaEventRecord(m->t1, m->st));
  DCUDA(cudaEventSynchronize(m->t1));
  m->timing[2] = elapsed(m);
  m->timing[7] = double(m->dc->tr->calls - calls0);
  m->factor_ok = true;
  return GPB_OK;
}

int log_likelihood(gpb_dmodel* m, double* out) {
  DTRY(ensure_factor(m));
  const DistLayout& L = m->L;
  double* vec = m->buf[GPB_BUF_VEC];
  // every rank holds the replicated log-diagonal sums and beta: the same
  // fixed-order reductions as one GPU (model.py:316-339)
  DCUDA(launch_loss_terms(vec + L.vec[V_LOGDIAG], L.Ti, vec + L.vec[V_BETA], L.np_, m->red, m->st));
  ++m->launches;
  double h[2];
  DCUDA(cudaMemcpyAsync(h, m->red, sizeof(h), cudaMemcpyDeviceToHost, m->st));
  DCUDA(cudaStreamSynchronize(m->st));
  *out = -h[0] - 0.5 * h[1] - double(m->n) * kHalfLog2Pi;
  return GPB_OK;
}

int loss_gradients(gpb_dmodel* m, double out[3]) {
  const bool tl = m->trainable[0], tv = m->trainable[1], tn = m->trainable[2];
  out[0] = out[1] = out[2] = 0.0;
  if (!(tl || tv || tn)) return GPB_OK;  // model.py:350-352
  DTRY(ensure_factor(m));
  DTRY(ensure_buffers(m, {GPB_BUF_X, GPB_BUF_KINV, GPB_BUF_XCOL, GPB_BUF_XROW, GPB_BUF_LCOL}));
  if (!m->parts) {
    const int64_t nblk = std::max(1, m->L.nown()) * (m->L.bi / kSekBlock) * (m->L.bi / kSekBlock);
    DCUDA(cudaMalloc(&m->parts, sizeof(double) * 3 * nblk));
  }
  DTRY(build_phase(m, 2));
  const DistLayout& L = m->L;
  double* vec = m->buf[GPB_BUF_VEC];
  DCUDA(cudaEventRecord(m->t0, m->st));
  if (L.nown() == 0) DCUDA(cudaMemsetAsync(vec + L.vec[V_RED], 0, sizeof(double) * 3, m->st));
  DTRY(run_phase(m, 2));
  DCUDA(launch_loss_terms(nullptr, 0, vec + L.vec[V_ALPHA], L.np_, m->red, m->st));
  ++m->launches;
  DCUDA(cudaEventRecord(m->t1, m->st));
  double hh[3], aa[1];
  DCUDA(cudaMemcpyAsync(hh, vec + L.vec[V_RED], sizeof(hh), cudaMemcpyDeviceToHost, m->st));
  DCUDA(cudaMemcpyAsync(aa, m->red, sizeof(aa), cudaMemcpyDeviceToHost, m->st));
  DCUDA(cudaStreamSynchronize(m->st));
  m->timing[4] = elapsed(m);
  // model.py:382-432: dNLL/dl = nu / (2 l^3) sum, dNLL/dnu = sum / 2,
  // dNLL/ds2 = (tr K^-1 - |alpha|^2) / 2
  if (tl) out[0] = 0.5 * (m->nu / (m->l * m->l * m->l)) * hh[0];
  if (tv) out[1] = 0.5 * hh[1];
  if (tn) out[2] = 0.5 * (hh[2] - aa[0]);  // loss_terms without a log-diagonal: out[0] = sum x^2
  return GPB_OK;
}

// the factor gathered into a local single-GPU model (owned tiles broadcast rank by rank)
int ensure_replica(gpb_dmodel* m) {
  DTRY(ensure_factor(m));
  if (m->rep_ok) return GPB_OK;
  const DistLayout& L = m->L;
  if (!m->rep) DTRY(gpb_model_create_device(m->dc->ctx, m->z, m->y, m->n, m->d, m->T, &m->rep));
  DTRY(gpb_model_set_params(m->rep, m->l, m->nu, m->s2, m->trainable));
  double *tiles = nullptr, *dinv = nullptr, *logdiag = nullptr, *beta = nullptr, *alpha = nullptr;
  DTRY(gpb_model_factor_buffers(m->rep, &tiles, &dinv, &logdiag, &beta, &alpha));
  const int64_t bi2 = L.bi2;
  DCUDA(cudaEventRecord(m->t0, m->st));
  if (L.world == 1) {  // owned order is the packed row-major order
    DCUDA(cudaMemcpyAsync(tiles, m->buf[GPB_BUF_L], sizeof(double) * L.nown() * bi2, cudaMemcpyDeviceToDevice, m->st));
  } else {
    int cap = 0;
    std::vector<DistLayout> lays(L.world);
    for (int r = 0; r < L.world; ++r) {
      DTRY(dist_layout(r, L.world, L.P, L.Q, m->n, m->T, &lays[r], nullptr));
      cap = std::max(cap, lays[r].nown());
    }
    double* stage = nullptr;
    DCUDA(cudaMalloc(&stage, sizeof(double) * std::max(1, cap) * bi2));
    CopyJob* dj = nullptr;
    DCUDA(cudaMalloc(&dj, sizeof(CopyJob) * std::max(1, cap)));
    std::vector<CopyJob> cj;
    int s = GPB_OK;
    for (int r = 0; r < L.world && s == GPB_OK; ++r) {
      const DistLayout& R = lays[r];
      if (R.nown() == 0) continue;
      double* src = r == L.rank ? m->buf[GPB_BUF_L] : stage;
      s = m->dc->tr->bcast(0, src, int64_t(R.nown()) * bi2, r, m->st);
      if (s != GPB_OK) break;
      cj.clear();
      for (int t = 0; t < R.nown(); ++t)
        cj.push_back({src + t * bi2, tiles + h_tri_rm(R.own_i[t], R.own_j[t]) * bi2});
      cudaMemcpyAsync(dj, cj.data(), sizeof(CopyJob) * cj.size(), cudaMemcpyHostToDevice, m->st);
      s = launch_copies(dj, static_cast<int64_t>(cj.size()), bi2, m->st);
      ++m->launches;
      cudaStreamSynchronize(m->st);  // stage and dj are reused by the next rank
    }
    cudaFree(stage);
    cudaFree(dj);
    DTRY(s);
  }
  double* vec = m->buf[GPB_BUF_VEC];
  DCUDA(cudaMemcpyAsync(dinv, m->buf[GPB_BUF_DINV], sizeof(double) * L.Ti * bi2, cudaMemcpyDeviceToDevice, m->st));
  DCUDA(cudaMemcpyAsync(logdiag, vec + L.vec[V_LOGDIAG], sizeof(double) * L.Ti, cudaMemcpyDeviceToDevice, m->st));
  DCUDA(cudaMemcpyAsync(beta, vec + L.vec[V_BETA], sizeof(double) * L.np_, cudaMemcpyDeviceToDevice, m->st));
  DCUDA(cudaMemcpyAsync(alpha, vec + L.vec[V_ALPHA], sizeof(double) * L.np_, cudaMemcpyDeviceToDevice, m->st));
  DCUDA(cudaEventRecord(m->t1, m->st));
  DCUDA(cudaStreamSynchronize(m->st));
  m->timing[5] = elapsed(m);
  DTRY(gpb_model_mark_factored(m->rep));
  m->rep_ok = true;
  return GPB_OK;
}

void release(gpb_dmodel* m) {
  if (m->rep) gpb_model_destroy(m->rep);
  m->rep = nullptr;
  for (double*& b : m->buf)
    if (b) {
      cudaFree(b);
      b = nullptr;
    }
  for (int8_t*& b : m->planes)
    if (b) {
      cudaFree(b);
      b = nullptr;
    }
  if (m->ozflag) cudaFree(m->ozflag);
  m->ozflag = nullptr;
  for (void* p : {static_cast<void*>(m->z), static_cast<void*>(m->y), static_cast<void*>(m->zp),
                  static_cast<void*>(m->info), static_cast<void*>(m->parts), static_cast<void*>(m->red),
                  static_cast<void*>(m->flow_flags), static_cast<void*>(m->flow_x), static_cast<void*>(m->flags)})
    if (p) cudaFree(p);
  for (cudaEvent_t e : m->ev) cudaEventDestroy(e);
  if (m->t0) cudaEventDestroy(m->t0);
  if (m->t1) cudaEventDestroy(m->t1);
  if (m->ta) cudaEventDestroy(m->ta);
  if (m->crit) cudaStreamDestroy(m->crit);
  if (m->st) cudaStreamDestroy(m->st);
}

}  // namespace

extern "C" {

int gpb_nccl_unique_id(void* id_out) {
  if (!id_out) return fail(GPB_INVALID_CONFIG, "null output");
  if (!g_nccl.load()) return fail(GPB_NCCL, g_nccl.err);
  ncclUniqueId id;
  if (ncclResult_t r = g_nccl.GetUniqueId(&id)) return fail(GPB_NCCL, g_nccl.GetErrorString(r));
  memcpy(id_out, &id, sizeof(id));
  return GPB_OK;
}

static int dist_common(gpb_ctx* ctx, int rank, int world, int P, int Q, gpb_dist** out) {
  if (!out) return fail(GPB_INVALID_CONFIG, "null output");
  *out = nullptr;
  if (!ctx || ctx != gpb_current()) return fail(GPB_NOT_RUNNING, "runtime is not running");
  if (world < 1 || P < 1 || Q < 1 || P * Q != world || rank < 0 || rank >= world)
    return fail(GPB_INVALID_CONFIG, "process grid " + std::to_string(P) + " x " + std::to_string(Q) +
                                        " does not match " + std::to_string(world) + " ranks");
  return GPB_OK;
}

int gpb_dist_init(gpb_ctx* ctx, int rank, int world, int P, int Q, const void* nccl_id, gpb_dist** out) {
  DTRY(dist_common(ctx, rank, world, P, Q, out));
  if (!nccl_id) return fail(GPB_INVALID_CONFIG, "null NCCL unique id");
  if (!g_nccl.load()) return fail(GPB_NCCL, g_nccl.err);
  NcclTransport* t = new NcclTransport();
  ncclUniqueId id;
  memcpy(&id, nccl_id, sizeof(id));
  ncclResult_t r = g_nccl.CommInitRank(&t->comm[0], world, id, rank);
  // process-row communicator (ranks ordered by q) and process-column one (ordered by p)
  if (r == 0) r = g_nccl.CommSplit(t->comm[0], rank / Q, rank % Q, &t->comm[1], nullptr);
  if (r == 0) r = g_nccl.CommSplit(t->comm[0], world + rank % Q, rank / Q, &t->comm[2], nullptr);
  if (r != 0) {
    std::string msg = std::string("NCCL communicator setup: ") + g_nccl.GetErrorString(r);
    delete t;
    return fail(GPB_NCCL, msg);
  }
  gpb_dist* dc = new gpb_dist();
  dc->ctx = ctx;
  dc->rank = rank;
  dc->world = world;
  dc->P = P;
  dc->Q = Q;
  dc->tr = t;
  *out = dc;
  return GPB_OK;
}

int gpb_dist_init_host(gpb_ctx* ctx, int rank, int world, int P, int Q, const gpb_host_coll* coll,
                       gpb_dist** out) {
  DTRY(dist_common(ctx, rank, world, P, Q, out));
  if (!coll || !coll->bcast || !coll->reduce_sum || !coll->allreduce_sum)
    return fail(GPB_INVALID_CONFIG, "host collectives need bcast, reduce_sum and allreduce_sum");
  HostTransport* t = new HostTransport();
  t->cb = *coll;
  gpb_dist* dc = new gpb_dist();
  dc->ctx = ctx;
  dc->rank = rank;
  dc->world = world;
  dc->P = P;
  dc->Q = Q;
  dc->tr = t;
  *out = dc;
  return GPB_OK;
}

int gpb_dist_init_emulate(gpb_ctx* ctx, int rank, int world, int P, int Q, gpb_dist** out) {
  DTRY(dist_common(ctx, rank, world, P, Q, out));
  gpb_dist* dc = new gpb_dist();
  dc->ctx = ctx;
  dc->rank = rank;
  dc->world = world;
  dc->P = P;
  dc->Q = Q;
  dc->tr = new NullTransport();
  *out = dc;
  return GPB_OK;
}

int gpb_dist_set_exchange(gpb_dist* dc, int mode) {
  if (!dc) return fail(GPB_INVALID_CONFIG, "null runtime");
  if (mode != 0 && mode != 1) return fail(GPB_INVALID_CONFIG, "exchange must be 0 (collectives) or 1 (peer memory)");
  dc->exchange = mode;
  return GPB_OK;
}

int gpb_dist_finalize(gpb_dist* dc) {
  if (!dc) return GPB_OK;
  if (dc->models > 0)
    return fail(GPB_INVALID_CONFIG, std::to_string(dc->models) + " model(s) still use this runtime: destroy them first");
  cudaDeviceSynchronize();
  delete dc->tr;
  delete dc;
  return GPB_OK;
}

int gpb_dist_model_create(gpb_dist* dc, const double* z, const double* y, int64_t n, int64_t d,
                          int64_t tiles_per_dim, gpb_dmodel** out) {
  if (!out) return fail(GPB_INVALID_CONFIG, "null output");
  *out = nullptr;
  if (!dc || dc->ctx != gpb_current()) return fail(GPB_NOT_RUNNING, "runtime is not running");
  if (!z || !y) return fail(GPB_INVALID_CONFIG, "null input");
  if (n < 1 || d < 1) return fail(GPB_DIM, "z must be N x D with N, D >= 1");
  gpb_dmodel* m = new gpb_dmodel();
  m->dc = dc;
  std::string err;
  if (int s = dist_layout(dc->rank, dc->world, dc->P, dc->Q, n, tiles_per_dim, &m->L, &err, dc->exchange)) {
    delete m;
    return fail(s, err);
  }
  const DistLayout& L = m->L;
  m->n = n;
  m->d = d;
  m->T = tiles_per_dim;
  m->pm.bp_user = L.bp_user;
  m->pm.b_user = L.b_user;
  int s = GPB_OK;
  auto step = [&](int r) {
    if (s == GPB_OK) s = r;
  };
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  if (cudaStreamCreateWithPriority(&m->st, cudaStreamNonBlocking, lo) != cudaSuccess ||
      cudaStreamCreateWithPriority(&m->crit, cudaStreamNonBlocking, hi) != cudaSuccess ||
      cudaEventCreate(&m->t0) != cudaSuccess || cudaEventCreate(&m->t1) != cudaSuccess ||
      cudaEventCreate(&m->ta) != cudaSuccess)
    step(fail(GPB_CUDA, "stream/event creation failed"));
  for (int e = 0; e < L.nevents && s == GPB_OK; ++e) {
    cudaEvent_t ev;
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess)
      step(fail(GPB_CUDA, "event creation failed"));
    else
      m->ev.push_back(ev);
  }
  auto dalloc = [&](void** p, size_t bytes) {
    if (s != GPB_OK) return;
    cudaError_t e = cudaMalloc(p, std::max<size_t>(bytes, 16));
    if (e != cudaSuccess) {
      cudaGetLastError();
      step(fail(e == cudaErrorMemoryAllocation ? GPB_NO_MEMORY : GPB_CUDA,
                std::string("device allocation: ") + cudaGetErrorString(e)));
    }
  };
  dalloc(reinterpret_cast<void**>(&m->z), sizeof(double) * n * d);
  dalloc(reinterpret_cast<void**>(&m->y), sizeof(double) * n);
  dalloc(reinterpret_cast<void**>(&m->zp), sizeof(double) * L.np_ * d);
  dalloc(reinterpret_cast<void**>(&m->info), sizeof(int) * 4);
  dalloc(reinterpret_cast<void**>(&m->red), sizeof(double) * std::max(16, L.world));
  dalloc(reinterpret_cast<void**>(&m->flow_flags), solve_flow_scratch_bytes(L.Ti, L.bi));
  dalloc(reinterpret_cast<void**>(&m->flow_x), sizeof(double) * L.np_);
  if (s == GPB_OK) step(ensure_buffers(m, {GPB_BUF_L, GPB_BUF_DINV, GPB_BUF_ROW, GPB_BUF_COL, GPB_BUF_VEC}));
  if (L.planes > 0) {  // planes of the panel buffers, one byte per entry and plane
    for (int b : {GPB_BUF_ROW, GPB_BUF_COL})
      if (L.bufsz[b] > 0) dalloc(reinterpret_cast<void**>(&m->planes[b]), size_t(L.bufsz[b]) * L.planes);
    dalloc(reinterpret_cast<void**>(&m->ozflag), sizeof(int));
    if (s == GPB_OK && cudaMemset(m->ozflag, 0, sizeof(int)) != cudaSuccess) step(fail(GPB_CUDA, "memset failed"));
  }
  if (s == GPB_OK) {
    cudaMemcpyAsync(m->z, z, sizeof(double) * n * d, cudaMemcpyHostToDevice, m->st);
    cudaMemcpyAsync(m->y, y, sizeof(double) * n, cudaMemcpyHostToDevice, m->st);
    if (launch_pad_rows(m->z, m->zp, L.np_, static_cast<int>(d), m->pm, m->st) != cudaSuccess ||
        launch_pad_vector(m->y, m->buf[GPB_BUF_VEC] + L.vec[V_Y], L.np_, m->pm, m->st) != cudaSuccess)
      step(fail(GPB_CUDA, "padding the training data failed"));
    m->launches += 2;
    if (s == GPB_OK && cudaStreamSynchronize(m->st) != cudaSuccess) step(fail(GPB_CUDA, "upload failed"));
  }
  if (s != GPB_OK) {
    release(m);
    delete m;
    return s;
  }
  ++dc->models;
  *out = m;
  return GPB_OK;
}

int gpb_dist_model_destroy(gpb_dmodel* m) {
  if (!m) return GPB_OK;
  --m->dc->models;
  if (m->st) cudaStreamSynchronize(m->st);
  if (m->crit) cudaStreamSynchronize(m->crit);
  teardown_p2p(m);
  release(m);
  delete m;
  return GPB_OK;
}

int gpb_dist_set_params(gpb_dmodel* m, double l, double nu, double s2, const uint8_t trainable[3]) {
  DTRY(check_model(m));
  // covariance.py:50-62
  if (!(l > 0)) return fail(GPB_INVALID_CONFIG, "lengthscale must be positive");
  if (!(nu > 0)) return fail(GPB_INVALID_CONFIG, "vertical_scale must be positive");
  if (!(s2 >= 0)) return fail(GPB_INVALID_CONFIG, "noise_variance must be non-negative");
  m->l = l;
  m->nu = nu;
  m->s2 = s2;
  if (trainable)
    for (int i = 0; i < 3; ++i) m->trainable[i] = trainable[i] ? 1 : 0;
  m->factor_ok = false;
  m->rep_ok = false;
  return GPB_OK;
}

int gpb_dist_get_params(gpb_dmodel* m, double out[3]) {
  if (!m || !out) return fail(GPB_INVALID_CONFIG, "null argument");
  out[0] = m->l;
  out[1] = m->nu;
  out[2] = m->s2;
  return GPB_OK;
}

int gpb_dist_factor(gpb_dmodel* m) {
  DTRY(check_model(m));
  return ensure_factor(m);
}

int gpb_dist_last_pivot(gpb_dmodel* m, int64_t* pivot) {
  if (!m || !pivot) return fail(GPB_INVALID_CONFIG, "null argument");
  *pivot = m->last_pivot;
  return GPB_OK;
}

int gpb_dist_log_likelihood(gpb_dmodel* m, double* out) {
  DTRY(check_model(m));
  if (!out) return fail(GPB_INVALID_CONFIG, "null output");
  return log_likelihood(m, out);
}

int gpb_dist_loss_gradients(gpb_dmodel* m, double out[3]) {
  DTRY(check_model(m));
  if (!out) return fail(GPB_INVALID_CONFIG, "null output");
  return loss_gradients(m, out);
}

int gpb_dist_optimize(gpb_dmodel* m, double lr, double b1, double b2, double eps, int64_t iters,
                      double* history) {
  DTRY(check_model(m));
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
    if (s == GPB_OK) {
      // model.py:462-479, same operation order as gpb_optimize
      double theta[3] = {m->l, m->nu, m->s2}, step[3];
      for (int i = 0; i < 3; ++i) {
        const double g = grads[i] * theta[i];
        m->adam_m[i] = b1 * m->adam_m[i] + (1 - b1) * g;
        m->adam_v[i] = b2 * m->adam_v[i] + (1 - b2) * g * g;
        const double mh = m->adam_m[i] / (1 - std::pow(b1, double(m->adam_step)));
        const double vh = m->adam_v[i] / (1 - std::pow(b2, double(m->adam_step)));
        step[i] = lr * mh / (std::sqrt(vh) + eps);
      }
      for (int i = 0; i < 3; ++i)
        if (m->trainable[i]) theta[i] = std::exp(std::log(std::max(theta[i], 1e-300)) - step[i]);
      if (m->trainable[2]) theta[2] = std::max(theta[2], 1e-12);
      m->l = theta[0];
      m->nu = theta[1];
      m->s2 = theta[2];
      m->factor_ok = false;
      m->rep_ok = false;
      double ll = 0;
      s = log_likelihood(m, &ll);
      if (s == GPB_OK && history) history[it] = -ll;
    }
    if (s == GPB_NOT_PD) {
      std::string msg = "iteration " + std::to_string(m->adam_step) + ": " + gpb_last_error();
      return fail(s, msg);
    }
    if (s != GPB_OK) return s;
  }
  return GPB_OK;
}

int gpb_dist_predict(gpb_dmodel* m, const double* zt, int64_t mt, int64_t d, double* mean, double* var,
                     double* cov) {
  DTRY(check_model(m));
  if (d != m->d)
    return fail(GPB_DIM, "test has " + std::to_string(d) + " features, model was trained with " +
                             std::to_string(m->d));
  if (mt < 1) return fail(GPB_DIM, "need at least one test point");
  if (!zt || !mean) return fail(GPB_INVALID_CONFIG, "null argument");
  DTRY(ensure_replica(m));
  const DistLayout& L = m->L;
  const int W = L.world, r = L.rank;
  const int64_t per = (mt + W - 1) / W;
  auto lo = [&](int q) { return std::min<int64_t>(mt, q * per); };
  auto hi = [&](int q) { return std::min<int64_t>(mt, (q + 1) * per); };
  const int64_t ms = hi(r) - lo(r);
  double *ztd = nullptr, *res = nullptr;
  DCUDA(cudaMalloc(&ztd, sizeof(double) * mt * d));
  DCUDA(cudaMalloc(&res, sizeof(double) * 2 * W * per));
  int s = GPB_OK;
  auto ok = [&](cudaError_t e) {
    if (s == GPB_OK && e != cudaSuccess) s = fail(GPB_CUDA, cudaGetErrorString(e));
  };
  ok(cudaMemcpy(ztd, zt, sizeof(double) * mt * d, cudaMemcpyHostToDevice));
  ok(cudaMemset(res, 0, sizeof(double) * 2 * W * per));
  DCUDA(cudaEventRecord(m->t0, m->st));
  const bool want_var = var || cov;
  // this rank's shard of the test points (no collective during the solve)
  if (s == GPB_OK && ms > 0)
    s = gpb_predict_device(m->rep, ztd + lo(r) * d, ms, d, res + r * per, want_var ? res + (W + r) * per : nullptr);
  // each slot is written by one rank only, zeros elsewhere: the sum is exact
  if (s == GPB_OK && W > 1) s = m->dc->tr->allreduce(0, res, 2 * W * per, m->st);
  if (s == GPB_OK) {
    ok(cudaMemcpyAsync(mean, res, sizeof(double) * mt, cudaMemcpyDeviceToHost, m->st));
    if (var) ok(cudaMemcpyAsync(var, res + W * per, sizeof(double) * mt, cudaMemcpyDeviceToHost, m->st));
    ok(cudaStreamSynchronize(m->st));
  }
  if (s == GPB_OK && cov) {
    // SURVEY.md 8(e) option (i): V_a = L^-1 K*(shard a)^T per rank, V gathered,
    // block row a of Sigma = K**(a, :) - V_a^T V, block rows gathered
    const int64_t ldv = std::max<int64_t>(128, (per + 127) / 128 * 128);
    double *vall = nullptr, *rows = nullptr, *meanv = nullptr;
    ok(cudaMalloc(&vall, sizeof(double) * W * L.np_ * ldv));
    ok(cudaMalloc(&rows, sizeof(double) * W * per * mt));
    ok(cudaMalloc(&meanv, sizeof(double) * std::max<int64_t>(1, per)));
    if (s == GPB_OK) ok(cudaMemset(vall, 0, sizeof(double) * W * L.np_ * ldv));
    if (s == GPB_OK && ms > 0)
      s = gpb_predict_solve_device(m->rep, ztd + lo(r) * d, ms, d, meanv, vall + r * L.np_ * ldv, ldv);
    for (int q = 0; q < W && s == GPB_OK && W > 1; ++q)
      if (hi(q) > lo(q)) s = m->dc->tr->bcast(0, vall + q * L.np_ * ldv, L.np_ * ldv, q, m->st);
    if (s == GPB_OK) ok(cudaStreamSynchronize(m->st));
    for (int q = 0; q < W && s == GPB_OK && ms > 0; ++q)
      if (hi(q) > lo(q))
        s = gpb_cov_block_device(m->rep, ztd + lo(r) * d, ms, vall + r * L.np_ * ldv, ldv, ztd + lo(q) * d,
                                 hi(q) - lo(q), vall + q * L.np_ * ldv, ldv, rows + r * per * mt + lo(q), mt);
    for (int q = 0; q < W && s == GPB_OK && W > 1; ++q)
      if (hi(q) > lo(q)) s = m->dc->tr->bcast(0, rows + q * per * mt, (hi(q) - lo(q)) * mt, q, m->st);
    if (s == GPB_OK) {
      ok(cudaMemcpyAsync(cov, rows, sizeof(double) * mt * mt, cudaMemcpyDeviceToHost, m->st));
      ok(cudaStreamSynchronize(m->st));
    }
    cudaFree(vall);
    cudaFree(rows);
    cudaFree(meanv);
  }
  DCUDA(cudaEventRecord(m->t1, m->st));
  DCUDA(cudaEventSynchronize(m->t1));
  m->timing[3] = elapsed(m);
  cudaFree(ztd);
  cudaFree(res);
  DTRY(s);
  // _clamp_variances (model.py:488-496)
  if (cov) {
    std::vector<double> diag(mt);
    for (int64_t i = 0; i < mt; ++i) diag[i] = cov[i * mt + i];
    DTRY(gpb_clamp_variances(diag.data(), mt));
    for (int64_t i = 0; i < mt; ++i) cov[i * mt + i] = diag[i];
  }
  if (var) DTRY(gpb_clamp_variances(var, mt));
  return GPB_OK;
}

int gpb_dist_cholesky(gpb_dmodel* m, double* L_out) {
  DTRY(check_model(m));
  DTRY(ensure_replica(m));
  return gpb_cholesky(m->rep, L_out);
}

int gpb_dist_timings(gpb_dmodel* m, double* ms_out, int n) {
  if (!m || !ms_out) return fail(GPB_INVALID_CONFIG, "null argument");
  for (int i = 0; i < n && i < 8; ++i) ms_out[i] = m->timing[i];
  return GPB_OK;
}

int gpb_dist_launch_count(gpb_dmodel* m, int64_t* out) {
  if (!m || !out) return fail(GPB_INVALID_CONFIG, "null argument");
  int64_t rl = 0;
  if (m->rep) gpb_model_launch_count(m->rep, &rl);
  *out = m->launches + rl;
  return GPB_OK;
}

}  // extern "C"
