// FP64 tensor-pipe peak probe: the roofline denominator for the DMMA kernels.
//
// MEASURED_PEAKS.json carries HBM and bf16 figures only, so the FP64 peak is
// measured in-run on the same GPU: every warp issues independent
// DMMA.8x8x4 chains from registers (no memory traffic), 2 CTAs x 8 warps per SM.
#include <algorithm>

#include "common.cuh"
#include "gpb200.h"

namespace {

constexpr int kChains = 8;

__global__ void __launch_bounds__(256) dmma_probe_kernel(double* sink, int iters) {
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[kChains][2];
#pragma unroll
  for (int i = 0; i < kChains; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) gpb::dmma884(c[i][0], c[i][1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) s += c[i][0] + c[i][1];
  if (s == 1234.5) sink[threadIdx.x] = s;
}

// int8 tcgen05 peak probe: the roofline denominator for the digit-plane product.  One CTA
// per SM issues tcgen05.mma kind::i8 (M = 128, N = 128, K = 32, the product's shape) back to
// back from two shared-memory tiles of pseudo-random digits into four TMEM accumulators --
// no global traffic at all, so the rate is what the tensor pipe and its shared-memory
// operand fetch can do (MEASURED_PEAKS.json has no int8 figure).
constexpr int kI8Box = 128 * 32;

GPB_DEVINL uint32_t p_su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
GPB_DEVINL uint64_t p_desc32(uint32_t addr) {  // K-major, 32-byte rows, SWIZZLE_32B (ozaki.cu)
  return static_cast<uint64_t>((addr >> 4) & 0x3FFFu) | (1ull << 16) | (16ull << 32) | (1ull << 46) | (6ull << 61);
}

__global__ void __launch_bounds__(128, 1) i8_probe_kernel(int rounds) {
  __shared__ __align__(1024) int8_t tiles[2 * kI8Box];
  __shared__ __align__(8) unsigned long long bar;
  __shared__ uint32_t slot;
  unsigned x = 0x9E3779B9u * (threadIdx.x + 1) + blockIdx.x;
  for (int i = threadIdx.x; i < 2 * kI8Box; i += blockDim.x) {
    x = x * 1664525u + 1013904223u;
    tiles[i] = static_cast<int8_t>(static_cast<int>(x >> 24) % 65);  // digits in [-64, 64]
  }
  const uint32_t b = p_su32(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(b) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(p_su32(&slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // the tiles, for the tensor core's reads
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
    const uint64_t ad = p_desc32(p_su32(tiles)), bd = p_desc32(p_su32(tiles) + kI8Box);
    // issued without waiting in between (the MMA queue back-pressures the thread); one commit at the end
    for (int r = 0; r < rounds; ++r) {
#pragma unroll 8
      for (int i = 0; i < 64; ++i)
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + (i & 3) * 128),
            "l"(ad), "l"(bd), "r"(idesc), "r"(r | (i >> 2))
            : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(b) : "memory");
    asm volatile(
        "{\n.reg .pred P1;\nI8P_WAIT:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra I8P_WAIT;\n}\n" ::"r"(b),
        "r"(0)
        : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
  }
}

}  // namespace

extern "C" int gpb_plugin_fail(int code, const char* msg);

extern "C" int gpb_int8_peak_probe(gpb_ctx* ctx, double seconds, double* tops) {
  if (!ctx || !tops) return gpb_plugin_fail(GPB_INVALID_CONFIG, "null argument");
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double ops_per_round = 64.0 * 2.0 * 128 * 128 * 32 * double(sms);
  int rounds = 256;
  i8_probe_kernel<<<sms, 128>>>(8);
  float ms = 0;
  cudaEventRecord(e0);
  i8_probe_kernel<<<sms, 128>>>(rounds);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  if (ms > 0) rounds = static_cast<int>(rounds * (seconds * 1e3 / 3.0) / ms) + 1;
  double best = 0.0;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    i8_probe_kernel<<<sms, 128>>>(rounds);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    best = std::max(best, ops_per_round * rounds / (ms * 1e-3) / 1e12);
  }
  cudaError_t err = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (err != cudaSuccess) return gpb_plugin_fail(GPB_CUDA, cudaGetErrorString(err));
  *tops = best;
  return GPB_OK;
}

extern "C" int gpb_fp64_peak_probe(gpb_ctx* ctx, double seconds, double* tflops) {
  if (!ctx || !tflops) return gpb_plugin_fail(GPB_INVALID_CONFIG, "null argument");
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* sink = nullptr;
  if (cudaMalloc(&sink, 256 * sizeof(double)) != cudaSuccess)
    return gpb_plugin_fail(GPB_NO_MEMORY, "probe allocation failed");
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = 2 * sms, threads = 256;
  const double flops_per_iter = 2.0 * 8 * 8 * 4 * kChains * (threads / 32) * double(blocks);
  int iters = 20000;
  dmma_probe_kernel<<<blocks, threads>>>(sink, 100);
  float ms = 0;
  // calibrate to ~`seconds` of sustained issue, then keep the best of 3
  cudaEventRecord(e0);
  dmma_probe_kernel<<<blocks, threads>>>(sink, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  if (ms > 0) iters = static_cast<int>(iters * (seconds * 1e3 / 3.0) / ms) + 1;
  double best = 0.0;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    dmma_probe_kernel<<<blocks, threads>>>(sink, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    best = std::max(best, flops_per_iter * iters / (ms * 1e-3) / 1e12);
  }
  cudaError_t err = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  if (err != cudaSuccess) return gpb_plugin_fail(GPB_CUDA, cudaGetErrorString(err));
  *tflops = best;
  return GPB_OK;
}
