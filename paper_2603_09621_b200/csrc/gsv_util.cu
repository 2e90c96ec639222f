// gsv_util.cu -- the per-Gaussian geometry helpers of the reference API on
// the device (f64): rotation_matrices (field.py:141-154), field_sigma_inv
// (render.py:67-71) and the scalar weight (render.py:74-81).
#include "gsv_common.cuh"

namespace gsv {
namespace {

__global__ void __launch_bounds__(256)
rotation_kernel(const double* __restrict__ q, int64_t n, double* __restrict__ R) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double r[9];
  rotation_f64(q + 4 * i, r);     // the stored quaternion, verbatim (no normalisation)
#pragma unroll
  for (int a = 0; a < 9; ++a) R[9 * i + a] = r[a];
}

// Sigma^-1 = R diag(exp(-2 ls)) R^T, summed over b in order like
// einsum("nab,nb,ncb->nac").
__device__ __forceinline__ void sigma_inv_one(const double* ls, const double* q, double out[9]) {
  double r[9];
  rotation_f64(q, r);
  const double iv[3] = {exp(mul(-2.0, ls[0])), exp(mul(-2.0, ls[1])), exp(mul(-2.0, ls[2]))};
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double t = 0.0;
#pragma unroll
      for (int b = 0; b < 3; ++b) t = add(t, mul(mul(r[3 * a + b], iv[b]), r[3 * c + b]));
      out[3 * a + c] = t;
    }
}

__global__ void __launch_bounds__(256)
sigma_inv_kernel(const double* __restrict__ ls, const double* __restrict__ q, int64_t n,
                 double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s[9];
  sigma_inv_one(ls + 3 * i, q + 4 * i, s);
#pragma unroll
  for (int a = 0; a < 9; ++a) out[9 * i + a] = s[a];
}

// weight(f, i, p): d2 = (delta @ Sigma^-1) @ delta, 0 beyond the cutoff,
// else exp(-d2/2) * r (r = sigmoid(raw_relax_i), or 1 when relax is off).
__global__ void weight_kernel(const double* __restrict__ pos, const double* __restrict__ ls,
                              const double* __restrict__ q, const double* __restrict__ rr,
                              int64_t i, int relax_enabled, double px, double py, double pz,
                              double cutoff2, double* __restrict__ out) {
  double s[9];
  sigma_inv_one(ls + 3 * i, q + 4 * i, s);
  const double d[3] = {sub(px, pos[3 * i]), sub(py, pos[3 * i + 1]), sub(pz, pos[3 * i + 2])};
  double d2 = 0.0;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double v = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a) v = add(v, mul(d[a], s[3 * a + c]));
    d2 = add(d2, mul(v, d[c]));
  }
  if (d2 > cutoff2) {
    *out = 0.0;
    return;
  }
  const double r = relax_enabled ? expit_f64(rr[i]) : 1.0;
  *out = mul(exp(mul(-0.5, d2)), r);
}

}  // namespace
}  // namespace gsv

using namespace gsv;

extern "C" {

int gsv_rotation_matrices(const double* rotations, int64_t n, double* R, void* stream) {
  GSV_REQUIRE(n >= 0 && (n == 0 || (rotations && R)), "bad arguments");
  if (n == 0) return GSV_OK;
  rotation_kernel<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(rotations, n, R);
  GSV_CHECK_LAUNCH("rotation_kernel");
  return GSV_OK;
}

int gsv_sigma_inv(const double* log_scales, const double* rotations, int64_t n, double* out,
                  void* stream) {
  GSV_REQUIRE(n >= 0 && (n == 0 || (log_scales && rotations && out)), "bad arguments");
  if (n == 0) return GSV_OK;
  sigma_inv_kernel<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(log_scales,
                                                                              rotations, n, out);
  GSV_CHECK_LAUNCH("sigma_inv_kernel");
  return GSV_OK;
}

int gsv_weight(const double* positions, const double* log_scales, const double* rotations,
               const double* raw_relax, int64_t n, int64_t i, int relax_enabled, double px,
               double py, double pz, double cutoff_sigma, double* out, void* stream) {
  GSV_REQUIRE(i >= 0 && i < n, "gaussian index %lld out of range [0, %lld)", (long long)i,
              (long long)n);
  GSV_REQUIRE(positions && log_scales && rotations && raw_relax && out, "null pointer argument");
  weight_kernel<<<1, 1, 0, as_stream(stream)>>>(positions, log_scales, rotations, raw_relax, i,
                                               relax_enabled, px, py, pz,
                                               cutoff_sigma * cutoff_sigma, out);
  GSV_CHECK_LAUNCH("weight_kernel");
  return GSV_OK;
}

}  // extern "C"
