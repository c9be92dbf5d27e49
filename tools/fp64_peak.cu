// FP64 peak probe for B200 (sm_100a): DMMA (mma.sync f64) vs DFMA.
// Measures sustained FP64 throughput to use as the roofline denominator.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dmma_m8n8k4(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int CHAINS>
__global__ void dmma_m16n8k16(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + (threadIdx.x + i) * 1e-9;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - (threadIdx.x + i) * 1e-9;
  double c[CHAINS][4];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-12, b = 0.999999;
  double c[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <class K>
double run(K kern, int blocks, int threads, int iters, double flops_per_warp_iter, int reps, double* d) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(d, 10);
  cudaDeviceSynchronize();
  double best = 0;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double tf = flops_per_warp_iter * (double)blocks * (threads / 32) * iters / (ms * 1e-3) / 1e12;
    if (tf > best) best = tf;
  }
  return best;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  printf("device %s sms=%d\n", p.name, p.multiProcessorCount);
  double* d; CK(cudaMalloc(&d, 1 << 20));
  int sms = p.multiProcessorCount;
  for (int wpb : {4, 8, 16}) {
    for (int bps : {1, 2}) {
      double t1 = run(dmma_m8n8k4<8>, sms * bps, wpb * 32, 20000, 8 * 8 * 4 * 2 * 8, 3, d);
      double t2 = run(dmma_m16n8k16<4>, sms * bps, wpb * 32, 5000, 16 * 8 * 16 * 2 * 4, 3, d);
      double t3 = run(dfma_loop<16>, sms * bps, wpb * 32, 20000, 32 * 2 * 16, 3, d);
      printf("warps/blk=%2d blk/sm=%d  DMMA m8n8k4 %.2f TF  DMMA m16n8k16 %.2f TF  DFMA %.2f TF\n", wpb, bps, t1, t2, t3);
    }
  }
  // sustained: ~4 s of DMMA
  double ts = run(dmma_m8n8k4<8>, sms * 2, 8 * 32, 400000, 8 * 8 * 4 * 2 * 8, 2, d);
  printf("sustained DMMA m8n8k4 (long run) %.2f TF\n", ts);
  double tsf = run(dfma_loop<16>, sms * 2, 8 * 32, 400000, 32 * 2 * 16, 2, d);
  printf("sustained DFMA (long run) %.2f TF\n", tsf);
  return 0;
}
