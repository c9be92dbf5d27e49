// Microbenchmark of the DMMA GEMM inner loop on B200: where does the 20% go?
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
// MODE 0: operands in registers (fixed).  1: LDS fragments each k4.  2: + __syncthreads every 4 k4.
template <int MODE, int FM, int FN>
__global__ void inner(double* out, int iters) {
  __shared__ double s[2][128 * 20];
  for (int i = threadIdx.x; i < 2 * 128 * 20; i += blockDim.x) (&s[0][0])[i] = 1.0 + i * 1e-9;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  const int wm = warp / (128 / (FN * 8)) , wn = warp % (128 / (FN * 8));
  double acc[FM][FN][2];
  for (int i = 0; i < FM; ++i) for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0;
  double af[FM], bf[FN];
  for (int i = 0; i < FM; ++i) af[i] = 1.0 + i; for (int j = 0; j < FN; ++j) bf[j] = 1.0 - j * 1e-3;
  for (int it = 0; it < iters; ++it) {
    for (int k4 = 0; k4 < 16; k4 += 4) {
      if (MODE >= 1) {
#pragma unroll
        for (int i = 0; i < FM; ++i) af[i] = s[0][(wm * FM * 8 + i * 8 + g) * 20 + k4 + t];
#pragma unroll
        for (int j = 0; j < FN; ++j) bf[j] = s[1][(wn * FN * 8 + j * 8 + g) * 20 + k4 + t];
      }
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    if (MODE >= 2) __syncthreads();
  }
  double sum = 0;
  for (int i = 0; i < FM; ++i) for (int j = 0; j < FN; ++j) sum += acc[i][j][0] + acc[i][j][1];
  if (sum == 1.2345) out[threadIdx.x] = sum;
}
template <class K> void run(const char* name, K k, int threads, int fm, int fn) {
  double* d; cudaMalloc(&d, 4096 * 8);
  int iters = 20000;
  k<<<148, threads>>>(d, 10); cudaDeviceSynchronize();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e30;
  for (int r = 0; r < 3; ++r) { cudaEventRecord(a); k<<<148, threads>>>(d, iters); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms; }
  double flops = 2.0 * 8 * 8 * 4 * fm * fn * 4.0 * iters * (threads / 32) * 148;
  printf("%-40s %6.2f TF/s  (%s)\n", name, flops / (best * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run("8w 64x32 regs", inner<0, 8, 4>, 256, 8, 4);
  run("8w 64x32 lds", inner<1, 8, 4>, 256, 8, 4);
  run("8w 64x32 lds+bar", inner<2, 8, 4>, 256, 8, 4);
  run("16w 32x32 regs", inner<0, 4, 4>, 512, 4, 4);
  run("16w 32x32 lds", inner<1, 4, 4>, 512, 4, 4);
  run("16w 32x32 lds+bar", inner<2, 4, 4>, 512, 4, 4);
  run("8w 32x64 lds", inner<1, 4, 8>, 256, 4, 8);
  run("4w 64x64 lds", inner<1, 8, 8>, 128, 8, 8);
  return 0;
}
