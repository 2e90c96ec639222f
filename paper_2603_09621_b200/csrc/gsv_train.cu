// gsv_train.cu -- merge, chain rule, loss, Adam, quaternion renormalisation.
//
//   merge_kernel      per-Gaussian sum of its pair partials in ascending brick
//                     order (_merge_pairs_kernel, raster.py:412-451)
//   chain_kernel      G6 -> d log_scales, d quaternion (ambient), sigmoid
//                     chains (raster.py:524-549, _rotation_jacobians 454-467)
//   loss_kernel       loss_and_grad (optimize.py:91-103)
//   adam_kernel       step_optimizer (optimize.py:127-148), numpy operand order
//   normalize_kernel  GaussianField.normalize_rotations (field.py:100-102)
// f64 throughout; reductions are fixed-order (bit-reproducible).
#include "gsv_common.cuh"

namespace gsv {
namespace {

template <typename T>
__global__ void __launch_bounds__(256)
merge_kernel(const T* __restrict__ partials, const int64_t* __restrict__ gstart, int64_t n,
             double* __restrict__ gsum) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double acc[11];
#pragma unroll
  for (int a = 0; a < 11; ++a) acc[a] = 0.0;
  const int64_t e0 = gstart[i], e1 = gstart[i + 1];
  for (int64_t e = e0; e < e1; ++e) {
    const T* p = partials + 12 * e;
#pragma unroll
    for (int a = 0; a < 11; ++a) acc[a] += (double)p[a];
  }
  double* o = gsum + 12 * i;
#pragma unroll
  for (int a = 0; a < 11; ++a) o[a] = acc[a];
  o[11] = 0.0;
}

// dR/dq_j of the rotation formula, raster.py:454-467 (row-major 3x3 each).
__device__ __forceinline__ void rotation_jacobians(const double* q, double J[4][9]) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  const double j0[9] = {0, -z, y, z, 0, -x, -y, x, 0};
  const double j1[9] = {0, y, z, y, -2 * x, -w, z, w, -2 * x};
  const double j2[9] = {-2 * y, x, w, x, 0, z, -w, z, -2 * y};
  const double j3[9] = {-2 * z, -w, x, w, -2 * z, y, x, y, 0};
#pragma unroll
  for (int a = 0; a < 9; ++a) {
    J[0][a] = 2 * j0[a];
    J[1][a] = 2 * j1[a];
    J[2][a] = 2 * j2[a];
    J[3][a] = 2 * j3[a];
  }
}

__global__ void __launch_bounds__(128)
chain_kernel(const double* __restrict__ gsum, const double* __restrict__ ls,
             const double* __restrict__ rot, const double* __restrict__ ra,
             const double* __restrict__ rr, int64_t n, int relax_enabled,
             double* __restrict__ g_amp, double* __restrict__ g_rel, double* __restrict__ g_pos,
             double* __restrict__ g_ls, double* __restrict__ g_rot) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* s = gsum + 12 * i;
  double G[9];
  G[0] = s[5]; G[4] = s[6]; G[8] = s[7];
  G[1] = G[3] = s[8];
  G[2] = G[6] = s[9];
  G[5] = G[7] = s[10];
  const double* q = rot + 4 * i;
  double R[9];
  rotation_f64(q, R);
  const double iv[3] = {exp(-2.0 * ls[3 * i]), exp(-2.0 * ls[3 * i + 1]), exp(-2.0 * ls[3 * i + 2])};
  // d ls_k = -2 inv_var_k (R^T G R)_kk
#pragma unroll
  for (int kk = 0; kk < 3; ++kk) {
    double t = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) t += R[3 * a + kk] * G[3 * a + b] * R[3 * b + kk];
    g_ls[3 * i + kk] = -2.0 * iv[kk] * t;
  }
  // d q_j = 2 tr(G dR_j D R^T): pmat[a][c] = sum_m J[a][m] iv[m] R[c][m]
  double J[4][9];
  rotation_jacobians(q, J);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    double t = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double pm = 0.0;  // pmat[c][a]
#pragma unroll
        for (int m = 0; m < 3; ++m) pm += J[j][3 * c + m] * iv[m] * R[3 * a + m];
        t += G[3 * a + c] * pm;
      }
    g_rot[4 * i + j] = 2.0 * t;
  }
  g_pos[3 * i + 0] = s[2];
  g_pos[3 * i + 1] = s[3];
  g_pos[3 * i + 2] = s[4];
  const double A = expit_f64(ra[i]);
  g_amp[i] = s[0] * A * (1.0 - A);
  if (relax_enabled) {
    const double r = expit_f64(rr[i]);
    g_rel[i] = s[1] * r * (1.0 - r);
  } else {
    g_rel[i] = 0.0;
  }
}

constexpr int kLossThreads = 256;

template <typename TP, typename TT>
__global__ void __launch_bounds__(kLossThreads)
loss_kernel(const TP* __restrict__ pred, const TT* __restrict__ target, int64_t v, int kind,
            double* __restrict__ grad, double* __restrict__ part) {
  __shared__ double sh[kLossThreads / 32];
  const int64_t per = (v + gridDim.x - 1) / gridDim.x;
  const int64_t lo = per * blockIdx.x, hi = min(v, lo + per);
  const double inv_v = 1.0 / (double)v;
  double acc = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += kLossThreads) {
    const double d = (double)pred[i] - (double)target[i];
    if (kind == 0) {
      acc += fabs(d);
      grad[i] = (d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0)) / (double)v;
    } else {
      acc += d * d;
      grad[i] = 2.0 * d / (double)v;
    }
  }
  (void)inv_v;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kLossThreads / 32; ++w) t += sh[w];
    part[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(1024) sum_kernel(const double* __restrict__ x, int64_t n,
                                                   double* __restrict__ out) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += 1024) acc += x[i];
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

__global__ void __launch_bounds__(256)
adam_kernel(double* __restrict__ p, double* __restrict__ m, double* __restrict__ v,
            const double* __restrict__ g, int64_t count, double lr, double b1, double b2,
            double eps, double bc1, double bc2) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= count) return;
  const double gi = g[i];
  const double mi = add(mul(m[i], b1), mul(sub(1.0, b1), gi));
  const double vi = add(mul(v[i], b2), mul(mul(sub(1.0, b2), gi), gi));
  m[i] = mi;
  v[i] = vi;
  const double step = __ddiv_rn(mul(lr, __ddiv_rn(mi, bc1)), add(sqrt(__ddiv_rn(vi, bc2)), eps));
  p[i] = sub(p[i], step);
}

__global__ void __launch_bounds__(256) normalize_kernel(double* __restrict__ q, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double* qi = q + 4 * i;
  const double nrm =
      sqrt(add(add(add(mul(qi[0], qi[0]), mul(qi[1], qi[1])), mul(qi[2], qi[2])), mul(qi[3], qi[3])));
#pragma unroll
  for (int a = 0; a < 4; ++a) qi[a] = __ddiv_rn(qi[a], nrm);
}

}  // namespace
}  // namespace gsv

using namespace gsv;

extern "C" {

int gsv_merge(const void* partials, const int64_t* gstart, int64_t n, int precision,
              double* gsum, void* stream) {
  GSV_REQUIRE(precision == 0 || precision == 1, "precision must be 0 (f32) or 1 (f64)");
  if (n <= 0) return GSV_OK;
  const unsigned blocks = (unsigned)((n + 255) / 256);
  if (precision == 0)
    merge_kernel<float><<<blocks, 256, 0, as_stream(stream)>>>((const float*)partials, gstart,
                                                               n, gsum);
  else
    merge_kernel<double><<<blocks, 256, 0, as_stream(stream)>>>((const double*)partials,
                                                                gstart, n, gsum);
  GSV_CHECK_LAUNCH("merge_kernel");
  return GSV_OK;
}

int gsv_chain_rule(const double* gsum, const double* log_scales, const double* rotations,
                   const double* raw_amplitude, const double* raw_relax, int64_t n,
                   int relax_enabled, double* g_raw_amplitude, double* g_raw_relax,
                   double* g_positions, double* g_log_scales, double* g_rotations,
                   void* stream) {
  if (n <= 0) return GSV_OK;
  chain_kernel<<<(unsigned)((n + 127) / 128), 128, 0, as_stream(stream)>>>(
      gsum, log_scales, rotations, raw_amplitude, raw_relax, n, relax_enabled, g_raw_amplitude,
      g_raw_relax, g_positions, g_log_scales, g_rotations);
  GSV_CHECK_LAUNCH("chain_kernel");
  return GSV_OK;
}

int gsv_loss_blocks(int64_t v) {
  int64_t b = (v + 4095) / 4096;
  if (b < 1) b = 1;
  if (b > 1184) b = 1184;  // 8 x 148 SMs
  return (int)b;
}

int gsv_loss(const void* pred, int pred_f64, const void* target, int target_f64, int64_t v,
             int loss_kind, double* grad, double* loss_part, void* stream) {
  GSV_REQUIRE(v >= 1, "volume must have at least one voxel");
  GSV_REQUIRE(loss_kind == 0 || loss_kind == 1, "loss_kind must be 0 (l1) or 1 (l2)");
  const unsigned blocks = (unsigned)gsv_loss_blocks(v);
  cudaStream_t s = as_stream(stream);
  if (!pred_f64 && !target_f64)
    loss_kernel<float, float><<<blocks, kLossThreads, 0, s>>>(
        (const float*)pred, (const float*)target, v, loss_kind, grad, loss_part);
  else if (!pred_f64 && target_f64)
    loss_kernel<float, double><<<blocks, kLossThreads, 0, s>>>(
        (const float*)pred, (const double*)target, v, loss_kind, grad, loss_part);
  else if (pred_f64 && !target_f64)
    loss_kernel<double, float><<<blocks, kLossThreads, 0, s>>>(
        (const double*)pred, (const float*)target, v, loss_kind, grad, loss_part);
  else
    loss_kernel<double, double><<<blocks, kLossThreads, 0, s>>>(
        (const double*)pred, (const double*)target, v, loss_kind, grad, loss_part);
  GSV_CHECK_LAUNCH("loss_kernel");
  return GSV_OK;
}

int gsv_sum(const double* x, int64_t n, double* out, void* stream) {
  sum_kernel<<<1, 1024, 0, as_stream(stream)>>>(x, n, out);
  GSV_CHECK_LAUNCH("sum_kernel");
  return GSV_OK;
}

int gsv_adam(double* p, double* m, double* v, const double* g, int64_t count, double lr,
             double beta1, double beta2, double eps, double bc1, double bc2, void* stream) {
  if (count <= 0) return GSV_OK;
  adam_kernel<<<(unsigned)((count + 255) / 256), 256, 0, as_stream(stream)>>>(
      p, m, v, g, count, lr, beta1, beta2, eps, bc1, bc2);
  GSV_CHECK_LAUNCH("adam_kernel");
  return GSV_OK;
}

int gsv_normalize_rotations(double* rotations, int64_t n, void* stream) {
  if (n <= 0) return GSV_OK;
  normalize_kernel<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(rotations, n);
  GSV_CHECK_LAUNCH("normalize_kernel");
  return GSV_OK;
}

}  // extern "C"
