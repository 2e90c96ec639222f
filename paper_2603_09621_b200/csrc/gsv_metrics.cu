// gsv_metrics.cu -- PSNR and full-3D SSIM on the device (metrics.py:35-77).
//
//   sqdiff_kernel   per-block f64 sums of (x - y)^2 (fixed tree), then
//                   sum_kernel-style fixed-order final sum: PSNR's MSE
//   ssim_pass_kernel  one axis of the separable 11-tap window over the five
//                   local-moment channels {a, b, a^2, b^2, ab}, zero-filled
//                   borders (scipy.ndimage.correlate1d mode="constant"); the
//                   first pass forms the channels from the inputs
//   ssim_map_kernel the last axis fused with mu/var/cov (divided by the
//                   window's coverage, the correlation of an all-ones
//                   volume), the SSIM map and per-block sums
// f64 throughout, like the reference; volumes are linear x-fastest.
#include "gsv_common.cuh"

namespace gsv {
namespace {

constexpr int kTaps = 11;
constexpr int kHalf = 5;
constexpr int kMetricThreads = 256;

struct Window {
  double w[kTaps];
};

__device__ __forceinline__ double load_any(const void* p, int f64, int64_t i) {
  return f64 ? reinterpret_cast<const double*>(p)[i]
             : (double)reinterpret_cast<const float*>(p)[i];
}

__device__ __forceinline__ double block_sum_d(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kMetricThreads / 32; ++w) t += sh[w];
  return t;  // valid in thread 0
}

__global__ void __launch_bounds__(kMetricThreads)
sqdiff_kernel(const void* __restrict__ x, int xf64, const void* __restrict__ y, int yf64,
              int64_t v, double* __restrict__ part) {
  __shared__ double sh[kMetricThreads / 32];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)kMetricThreads + threadIdx.x; i < v;
       i += (int64_t)gridDim.x * kMetricThreads) {
    const double d = load_any(x, xf64, i) - load_any(y, yf64, i);
    acc += d * d;
  }
  const double t = block_sum_d(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

__global__ void __launch_bounds__(1024) final_sum_kernel(const double* __restrict__ part, int n,
                                                          double* __restrict__ out) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += 1024) acc += part[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 32; ++w) t += sh[w];
    *out = t;
  }
}

// One separable pass along `axis` (0 = x, 1 = y, 2 = z) of the five moment
// channels.  FIRST: the channels are formed from the inputs (a = x, b = y).
// Channel c of voxel i lives at ch[c * v + i].
template <bool FIRST>
__global__ void __launch_bounds__(kMetricThreads)
ssim_pass_kernel(const void* __restrict__ x, int xf64, const void* __restrict__ y, int yf64,
                 const double* __restrict__ in, double* __restrict__ out, int nx, int ny,
                 int nz, int axis, Window win) {
  const int64_t v = (int64_t)nx * ny * nz;
  const int64_t i = blockIdx.x * (int64_t)kMetricThreads + threadIdx.x;
  if (i >= v) return;
  const int ix = (int)(i % nx);
  const int64_t r = i / nx;
  const int iy = (int)(r % ny), iz = (int)(r / ny);
  const int n = axis == 0 ? nx : axis == 1 ? ny : nz;
  const int c = axis == 0 ? ix : axis == 1 ? iy : iz;
  const int64_t st = axis == 0 ? 1 : axis == 1 ? (int64_t)nx : (int64_t)nx * ny;
  double s[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int t = 0; t < kTaps; ++t) {
    const int cc = c + t - kHalf;
    if (cc < 0 || cc >= n) continue;             // zero fill outside the volume
    const int64_t j = i + (int64_t)(t - kHalf) * st;
    const double w = win.w[t];
    if (FIRST) {
      const double a = load_any(x, xf64, j), b = load_any(y, yf64, j);
      s[0] += w * a;
      s[1] += w * b;
      s[2] += w * (a * a);
      s[3] += w * (b * b);
      s[4] += w * (a * b);
    } else {
#pragma unroll
      for (int k = 0; k < 5; ++k) s[k] += w * __ldg(in + k * v + j);
    }
  }
#pragma unroll
  for (int k = 0; k < 5; ++k) out[k * v + i] = s[k];
}

// Coverage of the zero-filled window at coordinate c of an axis of length n:
// the 1D correlation of ones (the reference's local_mean(ones), one axis).
__device__ __forceinline__ double coverage(int c, int n, const Window& win) {
  double s = 0.0;
#pragma unroll
  for (int t = 0; t < kTaps; ++t) {
    const int cc = c + t - kHalf;
    if (cc >= 0 && cc < n) s += win.w[t] * 1.0;
  }
  return s;
}

// Last pass (along z) fused with the SSIM map (metrics.py:69-77) and
// per-block sums of the map.
__global__ void __launch_bounds__(kMetricThreads)
ssim_map_kernel(const double* __restrict__ in, int nx, int ny, int nz, Window win,
                double* __restrict__ part) {
  __shared__ double sh[kMetricThreads / 32];
  const int64_t v = (int64_t)nx * ny * nz;
  const int64_t i = blockIdx.x * (int64_t)kMetricThreads + threadIdx.x;
  double val = 0.0;
  if (i < v) {
    const int ix = (int)(i % nx);
    const int64_t r = i / nx;
    const int iy = (int)(r % ny), iz = (int)(r / ny);
    const int64_t st = (int64_t)nx * ny;
    double s[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int t = 0; t < kTaps; ++t) {
      const int cc = iz + t - kHalf;
      if (cc < 0 || cc >= nz) continue;
      const int64_t j = i + (int64_t)(t - kHalf) * st;
#pragma unroll
      for (int k = 0; k < 5; ++k) s[k] += win.w[t] * __ldg(in + k * v + j);
    }
    // local_mean(ones): the product of the three axes' coverages, evaluated
    // in the reference's pass order (x, then y, then z)
    const double cx = coverage(ix, nx, win);
    double cy = 0.0, cz = 0.0;
#pragma unroll
    for (int t = 0; t < kTaps; ++t) {
      const int yy = iy + t - kHalf;
      if (yy >= 0 && yy < ny) cy += win.w[t] * cx;
    }
#pragma unroll
    for (int t = 0; t < kTaps; ++t) {
      const int zz = iz + t - kHalf;
      if (zz >= 0 && zz < nz) cz += win.w[t] * cy;
    }
    const double norm = cz;
    const double mu_a = s[0] / norm, mu_b = s[1] / norm;
    const double var_a = s[2] / norm - mu_a * mu_a;
    const double var_b = s[3] / norm - mu_b * mu_b;
    const double cov = s[4] / norm - mu_a * mu_b;
    const double c1 = 0.0001, c2 = 0.0009;        // (0.01 * 1)^2, (0.03 * 1)^2
    const double num = (2.0 * mu_a * mu_b + c1) * (2.0 * cov + c2);
    const double den = (mu_a * mu_a + mu_b * mu_b + c1) * (var_a + var_b + c2);
    val = num / den;
  }
  const double t = block_sum_d(val, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

}  // namespace
}  // namespace gsv

using namespace gsv;

extern "C" {

int gsv_sq_diff_sum(const void* x, int x_f64, const void* y, int y_f64, int64_t v,
                    double* partials, double* out, void* stream) {
  GSV_REQUIRE(x && y && partials && out, "null pointer argument");
  GSV_REQUIRE(v >= 1, "volume must have at least one voxel");
  cudaStream_t s = as_stream(stream);
  const int blocks = gsv_metric_blocks(v);
  sqdiff_kernel<<<blocks, kMetricThreads, 0, s>>>(x, x_f64, y, y_f64, v, partials);
  GSV_CHECK_LAUNCH("sqdiff_kernel");
  final_sum_kernel<<<1, 1024, 0, s>>>(partials, blocks, out);
  GSV_CHECK_LAUNCH("final_sum_kernel");
  return GSV_OK;
}

int gsv_metric_blocks(int64_t v) {
  int64_t b = (v + 4 * kMetricThreads - 1) / (4 * kMetricThreads);
  if (b < 1) b = 1;
  if (b > 4 * 148 * 8) b = 4 * 148 * 8;
  return (int)b;
}

int gsv_ssim3d_workspace(const gsv_grid* grid, size_t* bytes) {
  GSV_REQUIRE(grid && bytes, "null pointer argument");
  const int64_t v = (int64_t)grid->nx * grid->ny * grid->nz;
  const int64_t blocks = (v + kMetricThreads - 1) / kMetricThreads;
  *bytes = (size_t)(10 * v + blocks) * sizeof(double);
  return GSV_OK;
}

int gsv_ssim3d(const void* x, int x_f64, const void* y, int y_f64, const gsv_grid* grid,
               const double* window11, void* workspace, size_t workspace_bytes, double* out,
               void* stream) {
  GSV_REQUIRE(x && y && grid && window11 && workspace && out, "null pointer argument");
  GSV_REQUIRE(grid->nx >= kTaps && grid->ny >= kTaps && grid->nz >= kTaps,
              "volume too small for SSIM window: dims (%d, %d, %d), need >= %d per axis",
              grid->nx, grid->ny, grid->nz, kTaps);
  size_t need = 0;
  gsv_ssim3d_workspace(grid, &need);
  GSV_REQUIRE(workspace_bytes >= need, "ssim workspace too small: %zu < %zu", workspace_bytes,
              need);
  cudaStream_t s = as_stream(stream);
  Window win;
  for (int t = 0; t < kTaps; ++t) win.w[t] = window11[t];
  const int64_t v = (int64_t)grid->nx * grid->ny * grid->nz;
  double* ch0 = reinterpret_cast<double*>(workspace);
  double* ch1 = ch0 + 5 * v;
  double* part = ch1 + 5 * v;
  const unsigned blocks = (unsigned)((v + kMetricThreads - 1) / kMetricThreads);
  ssim_pass_kernel<true><<<blocks, kMetricThreads, 0, s>>>(x, x_f64, y, y_f64, nullptr, ch0,
                                                          grid->nx, grid->ny, grid->nz, 0, win);
  GSV_CHECK_LAUNCH("ssim_pass_kernel");
  ssim_pass_kernel<false><<<blocks, kMetricThreads, 0, s>>>(x, x_f64, y, y_f64, ch0, ch1,
                                                           grid->nx, grid->ny, grid->nz, 1, win);
  GSV_CHECK_LAUNCH("ssim_pass_kernel");
  ssim_map_kernel<<<blocks, kMetricThreads, 0, s>>>(ch1, grid->nx, grid->ny, grid->nz, win,
                                                    part);
  GSV_CHECK_LAUNCH("ssim_map_kernel");
  final_sum_kernel<<<1, 1024, 0, s>>>(part, (int)blocks, out);
  GSV_CHECK_LAUNCH("final_sum_kernel");
  return GSV_OK;
}

}  // extern "C"
