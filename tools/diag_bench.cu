// Microbenchmark: cycles of one warp factoring + inverting a 32x32 SPD block.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NB = 32, SLD = 33;

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// variant 0: registers + shuffles, fully unrolled (current potrf.cu)
__device__ void diag_regs(const double* A, double* Lout, double* Linv, double* Ld, double* Li) {
  const int lane = threadIdx.x & 31;
  double r[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c) r[c] = A[lane * NB + c];
  double my_l = 1.0, my_rinv = 0.0;
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    const double piv = __shfl_sync(0xffffffffu, r[j], j);
    const double rinv = rsqrt(piv);
    const double ljj = piv * rinv;
    if (lane == j) { r[j] = ljj; my_l = ljj; my_rinv = rinv; }
    else if (lane > j) r[j] *= rinv;
#pragma unroll
    for (int c = 0; c < NB; ++c)
      if (c > j) {
        const double lcj = __shfl_sync(0xffffffffu, r[j], c);
        if (lane >= c) r[c] = fma(-r[j], lcj, r[c]);
      }
  }
#pragma unroll
  for (int c = 0; c < NB; ++c) Ld[lane * SLD + c] = (c <= lane) ? r[c] : 0.0;
  Li[lane * SLD + lane] = my_rinv;
  __syncwarp();
  double x[NB];
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    double s0 = (i == lane) ? 1.0 : 0.0, s1 = 0, s2 = 0, s3 = 0;
#pragma unroll
    for (int k = 0; k < NB; ++k)
      if (k < i) {
        const double t = -Ld[i * SLD + k] * x[k];
        if ((k & 3) == 0) s0 += t; else if ((k & 3) == 1) s1 += t; else if ((k & 3) == 2) s2 += t; else s3 += t;
      }
    x[i] = ((s0 + s1) + (s2 + s3)) * Li[i * SLD + i];
  }
#pragma unroll
  for (int i = 0; i < NB; ++i) Linv[i * NB + lane] = x[i];
  Lout[lane] = my_l;
}

// variant 1: shared memory, rolled loops
__device__ void diag_smem(const double* A, double* Lout, double* Linv, double* Ld, double* Li) {
  const int lane = threadIdx.x & 31;
  for (int c = 0; c < NB; ++c) Ld[lane * SLD + c] = A[lane * NB + c];
  __syncwarp();
  for (int j = 0; j < NB; ++j) {
    const double piv = Ld[j * SLD + j];
    const double rinv = rsqrt(piv);
    __syncwarp();
    if (lane > j) Ld[lane * SLD + j] *= rinv;
    if (lane == j) { Ld[j * SLD + j] = piv * rinv; Li[j * SLD + j] = rinv; }
    __syncwarp();
    if (lane > j) {
      const double lij = Ld[lane * SLD + j];
      for (int c = j + 1; c <= lane; ++c) Ld[lane * SLD + c] -= lij * Ld[c * SLD + j];
    }
    __syncwarp();
  }
  // inverse: lane = column
  for (int r = 0; r < NB; ++r) {
    if (r < lane) Li[r * SLD + lane] = 0.0;
  }
  for (int r = lane + 1; r < NB; ++r) {
    double s = 0.0;
    for (int k = lane; k < r; ++k) s += Ld[r * SLD + k] * Li[k * SLD + lane];
    Li[r * SLD + lane] = -s * Li[r * SLD + r];
  }
  __syncwarp();
  for (int c = 0; c < NB; ++c) Linv[lane * NB + c] = Li[lane * SLD + c];
  Lout[lane] = Ld[lane * SLD + lane];
}

// variant 2: shifted registers (small code: pivot loop rolled), smem inverse
__device__ void diag_shift(const double* A, double* Lout, double* Linv, double* Ld, double* Li) {
  const int lane = threadIdx.x & 31;
  double r[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c) r[c] = A[lane * NB + c];
  double my_rinv = 0.0;
#pragma unroll 1
  for (int j = 0; j < NB; ++j) {
    const double piv = __shfl_sync(0xffffffffu, r[0], j);
    const double rinv = rsqrt(piv);
    const double lcol = (lane == j) ? piv * rinv : (lane > j ? r[0] * rinv : 0.0);
    if (lane == j) my_rinv = rinv;
    Ld[lane * SLD + j] = lcol;
#pragma unroll
    for (int c = 1; c < NB; ++c) {
      const double lcj = __shfl_sync(0xffffffffu, lcol, (j + c) & 31);
      if (lane >= j + c) r[c] = fma(-lcol, lcj, r[c]);
    }
#pragma unroll
    for (int c = 0; c < NB - 1; ++c) r[c] = r[c + 1];
  }
  Li[lane * SLD + lane] = my_rinv;
  __syncwarp();
  // column `lane` of the inverse: forward substitution, rolled over rows
#pragma unroll 1
  for (int i = 0; i < NB; ++i) {
    double s0 = (i == lane) ? 1.0 : 0.0, s1 = 0.0;
    int k = 0;
    for (; k + 1 < i; k += 2) {
      s0 = fma(-Ld[i * SLD + k], Li[k * SLD + lane], s0);
      s1 = fma(-Ld[i * SLD + k + 1], Li[(k + 1) * SLD + lane], s1);
    }
    if (k < i) s0 = fma(-Ld[i * SLD + k], Li[k * SLD + lane], s0);
    const double di = Li[i * SLD + i];
    __syncwarp();
    if (i != lane) Li[i * SLD + lane] = (i < lane) ? 0.0 : (s0 + s1) * di;
    else Li[i * SLD + lane] = di;
    __syncwarp();
  }
  for (int c = 0; c < NB; ++c) Linv[lane * NB + c] = Li[lane * SLD + c];
  Lout[lane] = Ld[lane * SLD + lane];
}

// variant 3: shared memory, uniform trip counts (predicated), unrolled by 4;
// inverse: rolled forward substitution with the column in shared memory
__device__ void diag_smem2(const double* A, double* Lout, double* Linv, double* Ld, double* Li) {
  const int lane = threadIdx.x & 31;
  for (int c = 0; c < NB; ++c) Ld[lane * SLD + c] = A[lane * NB + c];
  __syncwarp();
  double my_rinv = 0.0;
#pragma unroll 1
  for (int j = 0; j < NB; ++j) {
    const double piv = Ld[j * SLD + j];
    const double rinv = rsqrt(piv);
    const double lij = (lane > j) ? Ld[lane * SLD + j] * rinv : (lane == j ? piv * rinv : 0.0);
    if (lane == j) my_rinv = rinv;
    __syncwarp();
    if (lane >= j) Ld[lane * SLD + j] = lij;
    __syncwarp();
#pragma unroll 4
    for (int c = j + 1; c < NB; ++c) {
      const double lcj = Ld[c * SLD + j];
      if (lane >= c) Ld[lane * SLD + c] = fma(-lij, lcj, Ld[lane * SLD + c]);
    }
    __syncwarp();
  }
  Li[lane * SLD + lane] = my_rinv;
  __syncwarp();
#pragma unroll 1
  for (int i = 0; i < NB; ++i) {
    double s0 = (i == lane) ? 1.0 : 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int k = 0;
#pragma unroll 1
    for (; k + 3 < i; k += 4) {
      s0 = fma(-Ld[i * SLD + k], Li[k * SLD + lane], s0);
      s1 = fma(-Ld[i * SLD + k + 1], Li[(k + 1) * SLD + lane], s1);
      s2 = fma(-Ld[i * SLD + k + 2], Li[(k + 2) * SLD + lane], s2);
      s3 = fma(-Ld[i * SLD + k + 3], Li[(k + 3) * SLD + lane], s3);
    }
    for (; k < i; ++k) s0 = fma(-Ld[i * SLD + k], Li[k * SLD + lane], s0);
    const double di = Li[i * SLD + i];
    __syncwarp();
    if (i != lane) Li[i * SLD + lane] = (i < lane) ? 0.0 : ((s0 + s1) + (s2 + s3)) * di;
    __syncwarp();
  }
  for (int c = 0; c < NB; ++c) Linv[lane * NB + c] = Li[lane * SLD + c];
  Lout[lane] = Ld[lane * SLD + lane];
}

template <int V>
__global__ void bench(const double* A, double* Lout, double* Linv, long long* cyc, int reps) {
  __shared__ double Ld[NB * SLD], Li[NB * SLD];
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (V == 0) diag_regs(A, Lout, Linv, Ld, Li);
    else if (V == 1) diag_smem(A, Lout, Linv, Ld, Li);
    else if (V == 2) diag_shift(A, Lout, Linv, Ld, Li);
    else diag_smem2(A, Lout, Linv, Ld, Li);
    __syncwarp();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = (t1 - t0) / reps;
}

int main() {
  double h[NB * NB];
  for (int i = 0; i < NB; ++i)
    for (int j = 0; j < NB; ++j) h[i * NB + j] = (i == j ? NB : 0) + 1.0 / (1 + i + j);
  double *A, *L, *Li;
  long long* c;
  cudaMalloc(&A, sizeof h); cudaMalloc(&L, 256 * 8); cudaMalloc(&Li, sizeof h); cudaMalloc(&c, 8);
  cudaMemcpy(A, h, sizeof h, cudaMemcpyHostToDevice);
  long long cyc;
  bench<0><<<1, 32>>>(A, L, Li, c, 100); cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
  printf("regs+shuffle unrolled: %lld cycles per 32x32 factor+inverse\n", cyc);
  bench<1><<<1, 32>>>(A, L, Li, c, 100); cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
  printf("smem rolled:           %lld cycles\n", cyc);
  double ref[NB * NB], got[NB * NB], lref[32], lgot[32];
  bench<0><<<1, 32>>>(A, L, Li, c, 1);
  cudaMemcpy(ref, Li, sizeof ref, cudaMemcpyDeviceToHost);
  cudaMemcpy(lref, L, sizeof lref, cudaMemcpyDeviceToHost);
  bench<2><<<1, 32>>>(A, L, Li, c, 100); cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
  printf("shifted regs rolled:   %lld cycles\n", cyc);
  cudaMemcpy(got, Li, sizeof got, cudaMemcpyDeviceToHost);
  cudaMemcpy(lgot, L, sizeof lgot, cudaMemcpyDeviceToHost);
  double e = 0, el = 0;
  for (int i = 0; i < NB * NB; ++i) e = fmax(e, fabs(got[i] - ref[i]));
  for (int i = 0; i < NB; ++i) el = fmax(el, fabs(lgot[i] - lref[i]));
  printf("max |Linv diff| %.3e  max |diag L diff| %.3e\n", e, el);
  bench<3><<<1, 32>>>(A, L, Li, c, 100); cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
  printf("smem uniform unroll4:  %lld cycles\n", cyc);
  cudaMemcpy(got, Li, sizeof got, cudaMemcpyDeviceToHost);
  cudaMemcpy(lgot, L, sizeof lgot, cudaMemcpyDeviceToHost);
  e = 0; el = 0;
  for (int i = 0; i < NB * NB; ++i) e = fmax(e, fabs(got[i] - ref[i]));
  for (int i = 0; i < NB; ++i) el = fmax(el, fabs(lgot[i] - lref[i]));
  printf("max |Linv diff| %.3e  max |diag L diff| %.3e\n", e, el);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
