// Standalone check and timing of the tcgen05 digit-plane product (csrc/ozaki.cu)
// against a plain FP64 kernel on the same inputs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_2505_00136_b200/csrc \
//        -o tools/ozaki_probe tools/ozaki_probe.cu paper_2505_00136_b200/csrc/ozaki.cu -lcuda
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ozaki.cuh"

using namespace gpb;

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                        \
    }                                                                                 \
  } while (0)

// C = beta Cin + alpha A B^T; A: M x K tiled (tile t of width kt: rows M, ld kt), B: K x N row-major (k rows)
__global__ void ref_kernel(const double* A, int kt, const double* B, long long ldb, const double* Cin, double* C,
                           long long ldc, int M, int N, int K, double alpha, double beta) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x, m = blockIdx.y;
  if (n >= N) return;
  double acc = 0.0;
  for (int k = 0; k < K; ++k) {
    const double a = A[(long long)(k / kt) * M * kt + (long long)m * kt + k % kt];
    acc = fma(a, B[(long long)k * ldb + n], acc);
  }
  C[(long long)m * ldc + n] = beta * Cin[(long long)m * ldc + n] + alpha * acc;
}

static double urand(unsigned long long& s) {
  s = s * 6364136223846793005ull + 1442695040888963407ull;
  return ((s >> 11) * (1.0 / 9007199254740992.0)) * 2.0 - 1.0;
}

int run_case(int M, int N, int K, int kt, int S, bool time_only, int reps) {
  // A: K/kt tiles of M x kt (the packed row-panel layout with M = bi = kt in the library)
  const size_t na = size_t(M) * K, nb = size_t(K) * N, nc = size_t(M) * N;
  double *A, *B, *C, *Cin, *Cref;
  int8_t *Ap, *Bp;
  int* flag;
  CK(cudaMalloc(&A, na * 8));
  CK(cudaMalloc(&B, nb * 8));
  CK(cudaMalloc(&C, nc * 8));
  CK(cudaMalloc(&Cin, nc * 8));
  CK(cudaMalloc(&Cref, nc * 8));
  CK(cudaMalloc(&Ap, na * S));
  CK(cudaMalloc(&Bp, nb * S));
  CK(cudaMalloc(&flag, 4));
  CK(cudaMemset(flag, 0, 4));
  {
    std::vector<double> h(std::max(std::max(na, nb), nc));
    unsigned long long s = 12345;
    // wide dynamic range: magnitudes from 1 down to 1e-6
    for (size_t i = 0; i < na; ++i) h[i] = urand(s) * std::pow(10.0, -6.0 * std::fabs(urand(s)));
    CK(cudaMemcpy(A, h.data(), na * 8, cudaMemcpyHostToDevice));
    for (size_t i = 0; i < nb; ++i) h[i] = 0.9 * urand(s) * std::pow(10.0, -6.0 * std::fabs(urand(s)));
    CK(cudaMemcpy(B, h.data(), nb * 8, cudaMemcpyHostToDevice));
    for (size_t i = 0; i < nc; ++i) h[i] = urand(s);
    CK(cudaMemcpy(Cin, h.data(), nc * 8, cudaMemcpyHostToDevice));
  }
  const double sa = 2.0, sb = 2.0;
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, st));
  CK(launch_ozaki_slice_tiles(A, K / kt, M, kt, sa, Ap, S, flag, st));
  CK(cudaEventRecord(e1, st));
  CK(cudaStreamSynchronize(st));
  float ms_sa;
  cudaEventElapsedTime(&ms_sa, e0, e1);
  CK(cudaEventRecord(e0, st));
  // B (K x N) -> planes [N][K]
  CK(launch_ozaki_slice_t(B, K, N, N, sb, Bp, K / 32, 1, 0, S, flag, st));
  CK(cudaEventRecord(e1, st));
  CK(cudaStreamSynchronize(st));
  float ms_sb;
  cudaEventElapsedTime(&ms_sb, e0, e1);
  OzakiGemm g{};
  g.a = {Ap, (long long)M * kt * S, kt / 32, (long long)(kt / 32) * S * 4096};
  g.b = {Bp, 0, K / 32, (long long)(K / 32) * S * 4096};
  g.a_off = g.b_off = 0;
  g.M = M;
  g.N = N;
  g.K = K;
  g.slices = S;
  g.alpha = -sa * sb;
  g.beta = 1.0;
  g.Cin = Cin;
  g.Cout = C;
  g.ldc_in = g.ldc_out = N;
  CK(launch_ozaki_gemm(g, st));
  CK(cudaStreamSynchronize(st));
  CK(cudaEventRecord(e0, st));
  for (int r = 0; r < reps; ++r) CK(launch_ozaki_gemm(g, st));
  CK(cudaEventRecord(e1, st));
  CK(cudaStreamSynchronize(st));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  const double flops = 2.0 * M * N * double(K);
  const double pairs = S * (S + 1) / 2.0;
  printf("M=%d N=%d K=%d kt=%d S=%d: %.3f ms = %.1f TF/s FP64-equivalent (int8 %.0f TOPS); slice A %.3f ms, slice B^T %.3f ms\n",
         M, N, K, kt, S, ms, flops / ms * 1e-9, flops * pairs / ms * 1e-9, ms_sa, ms_sb);
  int hflag = 0;
  CK(cudaMemcpy(&hflag, flag, 4, cudaMemcpyDeviceToHost));
  int bad = hflag;
  if (!time_only) {
    dim3 grid((N + 127) / 128, M);
    ref_kernel<<<grid, 128, 0, st>>>(A, kt, B, N, Cin, Cref, N, M, N, K, -1.0, 1.0);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    std::vector<double> h(nc), hr(nc);
    CK(cudaMemcpy(h.data(), C, nc * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hr.data(), Cref, nc * 8, cudaMemcpyDeviceToHost));
    double maxerr = 0.0, fro = 0.0, fro_r = 0.0;
    size_t worst = 0;
    for (size_t i = 0; i < nc; ++i) {
      const double d = std::fabs(h[i] - hr[i]);
      if (!(d <= maxerr)) {
        maxerr = d;
        worst = i;
      }
      fro += d * d;
      fro_r += hr[i] * hr[i];
    }
    printf("   flag=%d max abs err %.3e at (%zu, %zu): %.17g vs %.17g; rel fro %.3e\n", hflag, maxerr, worst / N,
           worst % N, h[worst], hr[worst], std::sqrt(fro / fro_r));
    const double tol = 4.0 * std::pow(2.0, -7.0 * S + 9);  // S = 8: 1.4e-14
    if (!(std::sqrt(fro / fro_r) < tol)) bad = 1;
  }
  cudaFree(A); cudaFree(B); cudaFree(C); cudaFree(Cin); cudaFree(Cref); cudaFree(Ap); cudaFree(Bp); cudaFree(flag);
  return bad;
}

int main(int argc, char** argv) {
  CK(ozaki_init_attributes());
  int bad = 0;
  // correctness: tiled A walk (kt = M = 512) and a plain walk, every plane count
  bad |= run_case(128, 128, 64, 64, 8, false, 1);
  bad |= run_case(128, 128, 256, 256, 5, false, 1);
  bad |= run_case(256, 384, 1024, 256, 4, false, 1);
  bad |= run_case(512, 1024, 2048, 512, 8, false, 1);
  bad |= run_case(512, 1024, 2048, 512, 7, false, 1);
  bad |= run_case(512, 1024, 2048, 512, 6, false, 1);
  bad |= run_case(256, 512, 4096, 4096, 8, false, 1);
  bad |= run_case(512, 512, 32768, 512, 8, false, 1);
  if (argc > 2) {  // long run of one shape (clock / power sampling)
    run_case(512, 32768, 16384, 512, 8, true, atoi(argv[2]));
  } else if (argc > 1) {
    // timing at the prediction sweep's shapes
    for (int S = 6; S <= 8; ++S) {
      run_case(512, 32768, 4096, 512, S, true, 3);
      run_case(512, 32768, 16384, 512, S, true, 2);
    }
  }
  printf(bad ? "FAILED\n" : "OK\n");
  return bad;
}
