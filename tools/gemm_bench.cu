// Standalone timing of the grouped DMMA GEMM (csrc/gemm.cu) on synthetic
// device buffers: isolates kernel efficiency from the factorisation schedule.
//   nvcc ... -o tools/gemm_bench tools/gemm_bench.cu paper_2505_00136_b200/csrc/gemm.cu
#include <cmath>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "gemm.cuh"

using namespace gpb;

static void fill(double* d, size_t n) {
  std::vector<double> h(n);
  for (size_t i = 0; i < n; ++i) h[i] = ((i * 2654435761u) % 1000) * 1e-3 - 0.5;
  cudaMemcpy(d, h.data(), n * sizeof(double), cudaMemcpyHostToDevice);
}

struct Case {
  const char* name;
  int ntiles;   // independent 512x512 output tiles
  int K;
  bool ak, bk;
  double beta;
};

int main(int argc, char** argv) {
  gemm_init_attributes();
  const int bi = 512;
  const size_t bi2 = size_t(bi) * bi;
  Case cases[] = {
      {"update K=512 (chol), 2016 tiles", 2016, 512, true, true, 1.0},
      {"update K=1024, 1008 tiles", 1008, 1024, true, true, 1.0},
      {"long K=16384 KK, 64 tiles", 64, 16384, true, true, 0.0},
      {"long K=16384 K-MN (pred W), 64 tiles", 64, 16384, true, false, 1.0},
      {"update K=2048 (chol G=4), 504 tiles", 504, 2048, true, true, 1.0},
      {"K=2048 K-MN (pred W, early rows), 256 tiles", 256, 2048, true, false, 1.0},
      {"K=4096 K-MN (pred W), 128 tiles", 128, 4096, true, false, 1.0},
  };
  double *A, *B, *C;
  size_t maxa = 0;
  for (auto& c : cases) maxa = std::max(maxa, size_t(c.ntiles) * bi * c.K);
  // A: per tile a 512 x K panel; B shared panel of 512 x K; C: per tile 512x512
  cudaMalloc(&A, std::min(maxa, size_t(1) << 28) * sizeof(double));
  cudaMalloc(&B, size_t(bi) * 16384 * sizeof(double) * 2);
  cudaMalloc(&C, size_t(2016) * bi2 * sizeof(double));
  fill(A, std::min(maxa, size_t(1) << 28));
  fill(B, size_t(bi) * 16384 * 2);
  fill(C, size_t(2016) * bi2);
  GemmJob* dj;
  cudaMalloc(&dj, 2016 * sizeof(GemmJob));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (auto& c : cases) {
    std::vector<GemmJob> jobs(c.ntiles);
    const size_t apanel = size_t(bi) * c.K;
    const size_t amax = std::min(maxa, size_t(1) << 28);
    for (int t = 0; t < c.ntiles; ++t) {
      GemmJob j{};
      j.A = A + ((size_t(t) * apanel) % (amax - apanel)) / c.K * c.K;  // whole rows (TMA view)
      j.B = B;
      j.Cin = j.Cout = C + size_t(t) * bi2;
      j.K = c.K;
      jobs[t] = j;
    }
    cudaMemcpy(dj, jobs.data(), jobs.size() * sizeof(GemmJob), cudaMemcpyHostToDevice);
    GemmParams p{};
    p.jobs = dj;
    p.njobs = c.ntiles;
    p.mblk = p.nblk = bi / GBM;
    p.lda = c.K;
    p.ldb = c.bk ? c.K : bi;
    p.ldc = bi;
    p.a_ktile = p.b_ktile = int64_t(1) << 40;
    p.alpha = -1.0;
    p.beta = c.beta;
    p.max_k = c.K;  // the library's automatic configuration choice uses it
    p.a_base = A;
    p.a_extent = static_cast<int64_t>(amax);
    p.b_base = B;
    p.b_extent = int64_t(bi) * 16384 * 2;
    launch_gemm(p, c.ak, c.bk, EPI_AXPBY, 0);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      launch_gemm(p, c.ak, c.bk, EPI_AXPBY, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = std::min(best, ms);
    }
    const double flops = 2.0 * bi * bi * double(c.K) * c.ntiles;
    // bitwise fingerprint of one launch from a fixed C, and the largest
    // difference to the default configuration (cfg 4) relative to max |C|
    fill(C, size_t(c.ntiles) * bi2);
    launch_gemm(p, c.ak, c.bk, EPI_AXPBY, 0);
    std::vector<double> h(size_t(c.ntiles) * bi2), r(h.size());
    cudaMemcpy(h.data(), C, h.size() * 8, cudaMemcpyDeviceToHost);
    unsigned long long fp = 1469598103934665603ull;
    for (double v : h) {
      unsigned long long u;
      memcpy(&u, &v, 8);
      fp = (fp ^ u) * 1099511628211ull;
    }
    fill(C, size_t(c.ntiles) * bi2);
    gemm_force_config(4);
    launch_gemm(p, c.ak, c.bk, EPI_AXPBY, 0);
    gemm_force_config(-1);
    cudaMemcpy(r.data(), C, r.size() * 8, cudaMemcpyDeviceToHost);
    double dmax = 0.0, cmax = 0.0;
    for (size_t q = 0; q < h.size(); ++q) {
      dmax = std::max(dmax, std::fabs(h[q] - r[q]));
      cmax = std::max(cmax, std::fabs(r[q]));
    }
    printf("%-42s %8.3f ms  %6.2f TF/s  %s  fp=%016llx  vs cfg4 %.1e\n", c.name, best,
           flops / (best * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()), fp, dmax / cmax);
  }
  return 0;
}
