#include <cstdio>
__global__ void k(double* out, long long* cyc, double seed) {
  __shared__ double sm[64];
  const int lane = threadIdx.x;
  double x = seed + lane * 1e-3;
  long long t0, t1;
  const int N = 1000;
  // DFMA dependent chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = fma(x, 0.999, 1e-3);
  t1 = clock64(); cyc[0] = (t1 - t0) / N;
  // rsqrt dependent chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = rsqrt(x) + 0.5;
  t1 = clock64(); cyc[1] = (t1 - t0) / N;
  // shfl dependent chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31) + 1e-9;
  t1 = clock64(); cyc[2] = (t1 - t0) / N;
  // STS -> syncwarp -> LDS round trip
  t0 = clock64();
  for (int i = 0; i < N; ++i) { sm[lane] = x; __syncwarp(); x = sm[(lane + 1) & 31] + 1e-9; __syncwarp(); }
  t1 = clock64(); cyc[3] = (t1 - t0) / N;
  // MEMBAR.CTA + volatile store (lane 0) inside the loop
  volatile int* pr = reinterpret_cast<volatile int*>(sm + 40);
  t0 = clock64();
  for (int i = 0; i < N; ++i) { sm[lane] = x; __syncwarp(); if (lane == 0) { __threadfence_block(); *pr = i; } x = sm[(lane + 1) & 31] + 1e-9; __syncwarp(); }
  t1 = clock64(); cyc[4] = (t1 - t0) / N;
  // DMUL chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = x * 1.0000001;
  t1 = clock64(); cyc[5] = (t1 - t0) / N;
  out[lane] = x;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 64);
  k<<<1, 32>>>(o, c, 1.5); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, c, 1.5);
  long long h[8]; cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
  printf("DFMA dep %lld | rsqrt(double)+add dep %lld | shfl+add %lld | STS/sync/LDS+add %lld | +membar %lld | DMUL dep %lld cycles\n", h[0], h[1], h[2], h[3], h[4], h[5]);
  return 0;
}
