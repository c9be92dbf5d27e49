// BASELINE.json input generator on the device: the
// mass-spring-damper trajectory and its lag embedding, written straight into
// device buffers for large n (config 4: 139264 samples) so the training and
// test features need not cross PCIe.
//
// The forcing u and the observation noise are drawn on the host with
// numpy's default_rng (the pinned convention) and
// uploaded; the recurrence (A.2) is inherently sequential and runs in one
// thread with every operation explicitly rounded in the order Python
// evaluates  v = v + dt * (u_t - c v - k x) / m;  x = x + dt v  -- no FMA
// contraction -- so the series is bitwise the host generator's
// (data.py msd_series).  The lag embedding (A.4) is a parallel gather.
#include "gpb200.h"
#include "kernels.cuh"

extern "C" int gpb_plugin_fail(int code, const char* msg);

namespace {

__global__ void msd_kernel(const double* u, const double* noise, int64_t n, double dt, double mass,
                           double damping, double stiffness, double* y) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  double x = 0.0, v = 0.0;
  for (int64_t t = 0; t < n; ++t) {
    const double a = __dmul_rn(damping, v);
    const double b = __dsub_rn(u[t], a);
    const double c = __dmul_rn(stiffness, x);
    const double e = __dmul_rn(dt, __dsub_rn(b, c));
    v = __dadd_rn(v, __ddiv_rn(e, mass));
    x = __dadd_rn(x, __dmul_rn(dt, v));
    y[t] = __dadd_rn(x, noise[t]);
  }
}

// z[t][l] = u[t - l] (0 before the start), rows [0, n)
__global__ void lag_kernel(const double* u, int64_t n, int d, double* z) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n * d) return;
  const int64_t t = e / d;
  const int l = static_cast<int>(e % d);
  z[e] = t >= l ? u[t - l] : 0.0;
}

}  // namespace

extern "C" int gpb_msd_series_device(gpb_ctx* ctx, const double* u_dev, const double* noise_dev, int64_t n,
                                     int64_t n_reg, double dt, double mass, double damping, double stiffness,
                                     double* z_dev, double* y_dev) {
  if (!ctx || ctx != gpb_current()) return gpb_plugin_fail(GPB_NOT_RUNNING, "runtime is not running");
  if (n < 1 || n_reg < 1 || !u_dev || !noise_dev || !z_dev || !y_dev)
    return gpb_plugin_fail(GPB_INVALID_CONFIG, "need n >= 1, n_reg >= 1 and device buffers");
  if (!(mass != 0.0)) return gpb_plugin_fail(GPB_INVALID_CONFIG, "mass must be non-zero");
  msd_kernel<<<1, 32>>>(u_dev, noise_dev, n, dt, mass, damping, stiffness, y_dev);
  const int64_t total = n * n_reg;
  lag_kernel<<<static_cast<unsigned>((total + 255) / 256), 256>>>(u_dev, n, static_cast<int>(n_reg), z_dev);
  const cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return gpb_plugin_fail(GPB_CUDA, cudaGetErrorString(e));
  return GPB_OK;
}
