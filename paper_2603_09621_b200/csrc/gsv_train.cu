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
#include "gsv_prep.cuh"

#include <cstdlib>

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

// Chain rule of one Gaussian from its merged partials s[0..10]
// (raster.py:524-549): G = sym(G6); d ls_k = -2 e^{-2 ls_k} (R^T G R)_kk;
// d q_j = 2 tr(G dR_j D R^T); sigmoid chains.  out[12] in field order:
// positions(3), log_scales(3), rotations(4), raw_amplitude, raw_relax.
#ifndef GSV_CHAIN_NOINLINE
#define GSV_CHAIN_NOINLINE 0
#endif
#if GSV_CHAIN_NOINLINE
__device__ __noinline__
#else
__device__ __forceinline__
#endif
void chain_one(const double* s, const double* ls, const double* q,
                                          double ra, double rr, int relax_enabled,
                                          double out[12]) {
  double G[9];
  G[0] = s[5]; G[4] = s[6]; G[8] = s[7];
  G[1] = G[3] = s[8];
  G[2] = G[6] = s[9];
  G[5] = G[7] = s[10];
  double R[9];
  rotation_f64(q, R);
  const double iv[3] = {exp(-2.0 * ls[0]), exp(-2.0 * ls[1]), exp(-2.0 * ls[2])};
#pragma unroll
  for (int kk = 0; kk < 3; ++kk) {
    double t = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) t += R[3 * a + kk] * G[3 * a + b] * R[3 * b + kk];
    out[3 + kk] = -2.0 * iv[kk] * t;
  }
  // d q_j = 2 sum_{a,c,m} G[a][c] dR_j[c][m] e^{-2 ls_m} R[a][m] = 2 <dR_j, K>
  // with K = G P, P[a][m] = e^{-2 ls_m} R[a][m] (G symmetric).
  double K[9];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      double t = 0.0;
#pragma unroll
      for (int a = 0; a < 3; ++a) t += G[3 * a + c] * (iv[m] * R[3 * a + m]);
      K[3 * c + m] = t;
    }
  double J[4][9];
  rotation_jacobians(q, J);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    double t = 0.0;
#pragma unroll
    for (int a = 0; a < 9; ++a) t += J[j][a] * K[a];
    out[6 + j] = 2.0 * t;
  }
  out[0] = s[2];
  out[1] = s[3];
  out[2] = s[4];
  const double A = expit_f64(ra);
  out[10] = s[0] * A * (1.0 - A);
  if (relax_enabled) {
    const double r = expit_f64(rr);
    out[11] = s[1] * r * (1.0 - r);
  } else {
    out[11] = 0.0;
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
  double o[12];
  chain_one(gsum + 12 * i, ls + 3 * i, rot + 4 * i, ra[i], rr[i], relax_enabled, o);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    g_pos[3 * i + a] = o[a];
    g_ls[3 * i + a] = o[3 + a];
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) g_rot[4 * i + a] = o[6 + a];
  g_amp[i] = o[10];
  g_rel[i] = o[11];
}

// Adam on one element, numpy operand order of step_optimizer
// (optimize.py:141-147): m*b1 + (1-b1) g; v*b2 + ((1-b2) g) g;
// p -= (lr (m/bc1)) / (sqrt(v/bc2) + eps).
#ifndef GSV_ADAM_NOINLINE
#define GSV_ADAM_NOINLINE 1     // one out-of-line Adam body: less code, update 0.376 -> 0.363 ms
#endif
#if GSV_ADAM_NOINLINE
__device__ __noinline__
#else
__device__ __forceinline__
#endif
double adam_one(double p, double& m, double& v, double g, double lr,
                                           double b1, double b2, double eps, double bc1,
                                           double bc2) {
  m = add(mul(m, b1), mul(sub(1.0, b1), g));
  v = add(mul(v, b2), mul(mul(sub(1.0, b2), g), g));
  return sub(p, __ddiv_rn(mul(lr, __ddiv_rn(m, bc1)), add(sqrt(__ddiv_rn(v, bc2)), eps)));
}

// Optimizer tail, kernel 1 of 2: per Gaussian, merge its pair partials in
// ascending brick order (raster.py:412-451) [or read the all-reduced sums],
// then the chain rule (raster.py:524-549) -> packed f64 gradients (N,12) in
// field order.  Kept apart from Adam so each kernel stays lean: this one is
// latency/compute bound, the Adam pass is a pure HBM stream.
template <typename T>
__global__ void __launch_bounds__(128)
merge_chain_kernel(const T* __restrict__ partials, const int64_t* __restrict__ gstart,
                   const double* __restrict__ gsum, int64_t n, const double* __restrict__ ls,
                   const double* __restrict__ rot, const double* __restrict__ ra,
                   const double* __restrict__ rr, int relax_en, double* __restrict__ g12) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s[11];
  if (gsum != nullptr) {
#pragma unroll
    for (int a = 0; a < 11; ++a) s[a] = gsum[12 * i + a];
  } else {
#pragma unroll
    for (int a = 0; a < 11; ++a) s[a] = 0.0;
    const int64_t e1 = gstart[i + 1];
#pragma unroll 2
    for (int64_t e = gstart[i]; e < e1; ++e) {
      const T* p = partials + 12 * e;
#pragma unroll
      for (int a = 0; a < 11; ++a) s[a] += (double)p[a];
    }
  }
  double g[12];
  chain_one(s, ls + 3 * i, rot + 4 * i, ra[i], rr[i], relax_en, g);
  double2* o = reinterpret_cast<double2*>(g12 + 12 * i);
#pragma unroll
  for (int a = 0; a < 6; ++a) o[a] = make_double2(g[2 * a], g[2 * a + 1]);
}

struct MomentPtrs {
  double* p[10];
  __device__ double* operator[](int k) const { return p[k]; }
};

// Optimizer tail, kernel 2 of 2: Adam on every enabled group from the packed
// gradients (optimize.py:127-148, numpy operand order) + quaternion
// renormalisation (field.py:100-102).  A streaming pass: coalesced f64
// loads/stores, small live state, high occupancy.
__global__ void __launch_bounds__(256)
adam12_kernel(const double* __restrict__ g12, int64_t n, double* __restrict__ pos,
              double* __restrict__ ls, double* __restrict__ rot, double* __restrict__ ra,
              double* __restrict__ rr, MomentPtrs mv, int amp_en, int relax_en,
              gsv_adam_hparams h) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* g = g12 + 12 * i;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double m = mv[0][3 * i + a], v = mv[5][3 * i + a];
    pos[3 * i + a] = adam_one(pos[3 * i + a], m, v, g[a], h.lr[0], h.b1, h.b2, h.eps, h.bc1, h.bc2);
    mv[0][3 * i + a] = m; mv[5][3 * i + a] = v;
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double m = mv[1][3 * i + a], v = mv[6][3 * i + a];
    ls[3 * i + a] = adam_one(ls[3 * i + a], m, v, g[3 + a], h.lr[1], h.b1, h.b2, h.eps, h.bc1, h.bc2);
    mv[1][3 * i + a] = m; mv[6][3 * i + a] = v;
  }
  double q[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    double m = mv[2][4 * i + a], v = mv[7][4 * i + a];
    q[a] = adam_one(rot[4 * i + a], m, v, g[6 + a], h.lr[2], h.b1, h.b2, h.eps, h.bc1, h.bc2);
    mv[2][4 * i + a] = m; mv[7][4 * i + a] = v;
  }
  const double nrm = sqrt(add(add(add(mul(q[0], q[0]), mul(q[1], q[1])), mul(q[2], q[2])),
                              mul(q[3], q[3])));
#pragma unroll
  for (int a = 0; a < 4; ++a) rot[4 * i + a] = __ddiv_rn(q[a], nrm);
  if (amp_en) {
    double m = mv[3][i], v = mv[8][i];
    ra[i] = adam_one(ra[i], m, v, g[10], h.lr[3], h.b1, h.b2, h.eps, h.bc1, h.bc2);
    mv[3][i] = m; mv[8][i] = v;
  }
  if (relax_en) {
    double m = mv[4][i], v = mv[9][i];
    rr[i] = adam_one(rr[i], m, v, g[11], h.lr[4], h.b1, h.b2, h.eps, h.bc1, h.bc2);
    mv[4][i] = m; mv[9][i] = v;
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

// Optimizer tail in one pass (the default): a CTA owns 128 consecutive
// Gaussians, whose pair partials are one contiguous range in gid-major
// emission order.  The range is staged through shared memory with coalesced
// float4 loads (in 512-pair sub-chunks); each thread sums its own segment in
// ascending brick order (raster.py:412-451), then applies the chain rule
// (raster.py:524-549), Adam on every enabled group (optimize.py:127-148) and
// the quaternion renormalisation (field.py:100-102) in place.
// Graph-replayed steps: the gate (overflow | non-finite loss) and the step
// counter live on the device; bc holds 1 - beta^t for t = 1, 2, ... computed
// on the host exactly as the reference does (Python float pow).
struct StepDev {
  const int32_t* gate;
  const double* bc;
  const int64_t* t;
};

__global__ void gate_kernel(const double* __restrict__ loss_sum,
                            const int32_t* __restrict__ overflow, int32_t* __restrict__ gate,
                            double* __restrict__ result) {
  const double l = *loss_sum;
  const int ovf = *overflow != 0;
  const int bad = !isfinite(l);
  *gate = ovf | bad;
  result[0] = l;
  result[1] = (double)(ovf | (bad << 1));
}

__global__ void advance_kernel(int64_t* __restrict__ t, const int32_t* __restrict__ gate) {
  if (*gate == 0) *t += 1;
}

__global__ void advance_publish_kernel(int64_t* __restrict__ t, const int32_t* __restrict__ gate,
                                       const double* __restrict__ result, double* ring,
                                       int64_t* __restrict__ counter, int slots) {
  if (*gate == 0) *t += 1;
  const int64_t k = *counter;
  double* dst = ring + 2 * (k % slots);
  dst[0] = result[0];
  dst[1] = result[1];
  *counter = k + 1;
}

// Sharded graph step: the one all_reduce carries the merged partials (f32,
// N x 12; column 11 is free), this rank's loss in [0][11] and its capacity
// overflow flag in [1][11].
__global__ void shard_pack_kernel(const double* __restrict__ gsum, int64_t n12,
                                  const double* __restrict__ loss_sum,
                                  const int32_t* __restrict__ overflow, float* __restrict__ red) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n12) return;
  float v = (float)gsum[i];
  if (i == 11) v = (float)*loss_sum;
  if (i == 23) v = *overflow != 0 ? 1.f : 0.f;
  red[i] = v;
}

__global__ void shard_unpack_kernel(const float* __restrict__ red, int64_t n12,
                                    double* __restrict__ gsum, double* __restrict__ loss_sum,
                                    int32_t* __restrict__ overflow) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n12) return;
  const float v = red[i];
  if (i == 11) {
    *loss_sum = (double)v;
    gsum[i] = 0.0;
  } else if (i == 23) {
    *overflow = v > 0.f ? 1 : 0;
    gsum[i] = 0.0;
  } else {
    gsum[i] = (double)v;
  }
}

// Bulk L2 prefetch of a contiguous range (TMA unit; a hint, no registers or
// shared memory): the address is rounded down and the size to 16 B.
__device__ __forceinline__ void prefetch_l2(const void* p, int64_t bytes) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const uintptr_t a16 = a & ~(uintptr_t)15;
  int64_t nb = (bytes + (int64_t)(a - a16)) & ~(int64_t)15;
  if (nb > (1 << 20)) nb = 1 << 20;
  if (nb > 0)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a16), "r"((unsigned)nb)
                 : "memory");
}

constexpr int kTailThreads = 128;
constexpr int kTailSub = 512;   // pairs per smem sub-chunk (24 KB)

// PREP (graph step): also write the next step's records, pair count and
// brick box from the updated parameters (preprocess_one), replacing the
// binning pass's separate preprocess of the whole field.
template <bool PREP>
__global__ void __launch_bounds__(kTailThreads, PREP ? 5 : 6)
tail_kernel(const float* __restrict__ partials, const int64_t* __restrict__ gstart,
            const double* __restrict__ gsum, int64_t n, double* __restrict__ pos,
            double* __restrict__ ls, double* __restrict__ rot, double* __restrict__ ra,
            double* __restrict__ rr, MomentPtrs mv, int amp_en, int relax_en,
            const gsv_adam_hparams h, StepDev sd, PrepArgs pa) {
  __shared__ float4 sp[kTailSub * 3];
  if (sd.gate != nullptr && *sd.gate != 0) return;   // overflow / non-finite loss: no update
  const int64_t i0 = blockIdx.x * (int64_t)kTailThreads;
  const int64_t i = i0 + threadIdx.x;
  const bool valid = i < n;
  // Pull this CTA's parameter and moment runs (and its partial segment) into
  // L2 now, so Adam's loads after the merge + chain rule hit L2.
  if (threadIdx.x < 11) {
    const int64_t cnt = min((int64_t)kTailThreads, n - i0);
    const int k = threadIdx.x;
    if (k < 10) {
      const int grp = k % 5;                       // pos, ls, rot, amp, rel
      const int w = grp < 2 ? 3 : (grp == 2 ? 4 : 1);
      const double* mom = nullptr;
#pragma unroll
      for (int j = 0; j < 10; ++j)                 // static indices: no local copy
        if (j == k) mom = mv.p[j];
      prefetch_l2(mom + w * i0, 8 * w * cnt);
      if (k < 5) {
        const double* prm = grp == 0 ? pos : grp == 1 ? ls : grp == 2 ? rot : grp == 3 ? ra : rr;
        prefetch_l2(prm + w * i0, 8 * w * cnt);
      }
    } else if (gsum == nullptr) {
      const int64_t e_lo = gstart[i0], e_hi = gstart[i0 + cnt];
      prefetch_l2(partials + 12 * e_lo, 48 * (e_hi - e_lo));
    }
  }
  double s[11];
#pragma unroll
  for (int a = 0; a < 11; ++a) s[a] = 0.0;
  if (gsum != nullptr) {
    if (valid) {
#pragma unroll
      for (int a = 0; a < 11; ++a) s[a] = gsum[12 * i + a];
    }
  } else {
    const int64_t iend = min(n, i0 + kTailThreads);
    const int64_t e_lo = gstart[i0], e_hi = gstart[iend];
    const int64_t my0 = valid ? gstart[i] : 0, my1 = valid ? gstart[i + 1] : 0;
    const float4* src = reinterpret_cast<const float4*>(partials);
    for (int64_t c0 = e_lo; c0 < e_hi; c0 += kTailSub) {
      const int cnt = (int)min((int64_t)kTailSub, e_hi - c0);
      __syncthreads();
      for (int q = threadIdx.x; q < 3 * cnt; q += kTailThreads) sp[q] = __ldg(src + 3 * c0 + q);
      __syncthreads();
      const int64_t a0 = max(my0, c0), a1 = min(my1, c0 + cnt);
      for (int64_t e = a0; e < a1; ++e) {
        const float4* pp = sp + 3 * (e - c0);
        const float4 x = pp[0], y = pp[1], z = pp[2];
        s[0] += (double)x.x; s[1] += (double)x.y; s[2] += (double)x.z; s[3] += (double)x.w;
        s[4] += (double)y.x; s[5] += (double)y.y; s[6] += (double)y.z; s[7] += (double)y.w;
        s[8] += (double)z.x; s[9] += (double)z.y; s[10] += (double)z.z;
      }
    }
  }
  if (!valid) return;
  double g[12];
  chain_one(s, ls + 3 * i, rot + 4 * i, ra[i], rr[i], relax_en, g);
  // bias corrections: from the device table at the device step counter
  // (graph replays) or the launch parameters
  double bc1 = h.bc1, bc2 = h.bc2;
  if (sd.bc != nullptr) {
    const int64_t t = *sd.t;
    bc1 = sd.bc[2 * t];
    bc2 = sd.bc[2 * t + 1];
  }
  double pn[3], ln[3], qn[4];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double m = mv[0][3 * i + a], v = mv[5][3 * i + a];
    pn[a] = adam_one(pos[3 * i + a], m, v, g[a], h.lr[0], h.b1, h.b2, h.eps, bc1, bc2);
    pos[3 * i + a] = pn[a];
    mv[0][3 * i + a] = m; mv[5][3 * i + a] = v;
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double m = mv[1][3 * i + a], v = mv[6][3 * i + a];
    ln[a] = adam_one(ls[3 * i + a], m, v, g[3 + a], h.lr[1], h.b1, h.b2, h.eps, bc1, bc2);
    ls[3 * i + a] = ln[a];
    mv[1][3 * i + a] = m; mv[6][3 * i + a] = v;
  }
  double q[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    double m = mv[2][4 * i + a], v = mv[7][4 * i + a];
    q[a] = adam_one(rot[4 * i + a], m, v, g[6 + a], h.lr[2], h.b1, h.b2, h.eps, bc1, bc2);
    mv[2][4 * i + a] = m; mv[7][4 * i + a] = v;
  }
  const double nrm = sqrt(add(add(add(mul(q[0], q[0]), mul(q[1], q[1])), mul(q[2], q[2])),
                              mul(q[3], q[3])));
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    qn[a] = __ddiv_rn(q[a], nrm);
    rot[4 * i + a] = qn[a];
  }
  double ran = ra[i], rrn = rr[i];
  if (amp_en) {
    double m = mv[3][i], v = mv[8][i];
    ran = adam_one(ran, m, v, g[10], h.lr[3], h.b1, h.b2, h.eps, bc1, bc2);
    ra[i] = ran;
    mv[3][i] = m; mv[8][i] = v;
  }
  if (relax_en) {
    double m = mv[4][i], v = mv[9][i];
    rrn = adam_one(rrn, m, v, g[11], h.lr[4], h.b1, h.b2, h.eps, bc1, bc2);
    rr[i] = rrn;
    mv[4][i] = m; mv[9][i] = v;
  }
  if (PREP) preprocess_one(i, pn, ln, qn, ran, rrn, pa);
}

// ---------------------------------------------------------------- TMA tail
// The same one-pass tail with its memory traffic on the bulk-copy (TMA)
// engine: a CTA's 128 Gaussians own contiguous runs of every parameter and
// moment array (15 runs, 36 KB) and one contiguous range of pair partials.
// One thread issues 1-D bulk copies global -> shared for all of them at
// once, signalled on mbarriers: the parameter/moment runs land while the
// merge walks the partials (double-buffered 128-pair chunks).  Adam and the
// renormalisation then run out of shared memory and the updated runs go back
// with bulk stores.  No per-thread strided f64 loads waiting on L2/HBM one
// dependent round trip after another (the old tail's long-scoreboard stalls).
// The last, partial CTA and misaligned caller pointers take a generic path
// into the same shared layout.
namespace tma {
__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(su32(bar)), "r"(phase)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(su32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void store_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// wait until the committed bulk stores have READ shared memory (the CTA may
// then exit; the global writes complete asynchronously, as in CUTLASS's
// TMA-store epilogues)
__device__ __forceinline__ void store_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
}  // namespace tma

#ifndef GSV_TMA_CHUNK
#define GSV_TMA_CHUNK 64
#endif
constexpr int kTmaChunk = GSV_TMA_CHUNK;       // pairs per staging buffer (48 B each)
// shared layout (doubles): per array family (params, m, v) the runs
// pos(3T) ls(3T) rot(4T) ra(T) rr(T), T = kTailThreads
__host__ __device__ constexpr int run_w(int g) { return g < 2 ? 3 : (g == 2 ? 4 : 1); }
template <int NT>
__host__ __device__ constexpr int run_off(int g) {
  return NT * (g == 0 ? 0 : g == 1 ? 3 : g == 2 ? 6 : g == 3 ? 10 : 11);
}
#ifndef GSV_TMA_THREADS
#define GSV_TMA_THREADS 64
#endif
constexpr int kTmaThreads = GSV_TMA_THREADS;   // Gaussians (= threads) per CTA
template <int NT>
constexpr size_t tma_smem() {
  return 3 * 12 * NT * sizeof(double) + 2 * kTmaChunk * 48 + 4 * sizeof(uint64_t);
}

#ifndef GSV_TMA_WARPS_PER_SM
#define GSV_TMA_WARPS_PER_SM 24
#endif
template <int NT>
__global__ void __launch_bounds__(NT, GSV_TMA_WARPS_PER_SM * 32 / NT)
tail_tma_kernel(const float* __restrict__ partials, const int64_t* __restrict__ gstart,
                const double* __restrict__ gsum, int64_t n, double* __restrict__ pos,
                double* __restrict__ ls, double* __restrict__ rot, double* __restrict__ ra,
                double* __restrict__ rr, MomentPtrs mv, int amp_en, int relax_en,
                const gsv_adam_hparams h, StepDev sd, int aligned) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* sprm = reinterpret_cast<double*>(smem_raw);
  double* sm = sprm + 12 * NT;
  double* sv = sm + 12 * NT;
  float4* spart = reinterpret_cast<float4*>(sv + 12 * NT);            // [2][kTmaChunk * 3]
  uint64_t* bar = reinterpret_cast<uint64_t*>(spart + 2 * 3 * kTmaChunk);
  if (sd.gate != nullptr && *sd.gate != 0) return;   // overflow / non-finite loss: no update
  const int tid = threadIdx.x;
  const int64_t i0 = blockIdx.x * (int64_t)NT;
  const int cnt = (int)min((int64_t)NT, n - i0);
  const int64_t i = i0 + tid;
  const bool valid = tid < cnt;
  const bool tma = aligned && cnt == NT;
  double* const gprm[5] = {pos, ls, rot, ra, rr};
  const bool en[5] = {true, true, true, amp_en != 0, relax_en != 0};
  const bool merge = gsum == nullptr;
  const int64_t e_lo = merge ? gstart[i0] : 0, e_hi = merge ? gstart[i0 + cnt] : 0;
  const int nch = (int)((e_hi - e_lo + kTmaChunk - 1) / kTmaChunk);
  const float4* src = reinterpret_cast<const float4*>(partials);

  auto chunk_pairs = [&](int c) {
    return (int)min((int64_t)kTmaChunk, e_hi - (e_lo + (int64_t)c * kTmaChunk));
  };
  auto issue_chunk = [&](int c) {   // thread 0, TMA path
    const int np = chunk_pairs(c);
    uint64_t* b = bar + 1 + (c & 1);
    tma::expect_tx(b, (uint32_t)(48 * np));
    tma::g2s(spart + (c & 1) * 3 * kTmaChunk, src + 3 * (e_lo + (int64_t)c * kTmaChunk),
             (uint32_t)(48 * np), b);
  };

  if (tma) {
    if (tid == 0) {
#pragma unroll
      for (int k = 0; k < 3; ++k) tma::mbar_init(bar + k);
      tma::fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) {
      uint32_t bytes = 0;
#pragma unroll
      for (int g = 0; g < 5; ++g) {
        const uint32_t b = (uint32_t)(8 * run_w(g) * NT);
        bytes += b;
        if (mv[g] != nullptr) bytes += b;
        if (mv[g + 5] != nullptr) bytes += b;
      }
      tma::expect_tx(bar, bytes);
#pragma unroll
      for (int g = 0; g < 5; ++g) {
        const uint32_t b = (uint32_t)(8 * run_w(g) * NT);
        const int64_t off = run_w(g) * i0;
        tma::g2s(sprm + run_off<NT>(g), gprm[g] + off, b, bar);
        if (mv[g] != nullptr) tma::g2s(sm + run_off<NT>(g), mv[g] + off, b, bar);
        if (mv[g + 5] != nullptr) tma::g2s(sv + run_off<NT>(g), mv[g + 5] + off, b, bar);
      }
      if (merge) {
        if (nch > 0) issue_chunk(0);
        if (nch > 1) issue_chunk(1);
      }
    }
  } else {
    // generic path: the same shared layout filled by plain loads
#pragma unroll
    for (int g = 0; g < 5; ++g) {
      const int w = run_w(g);
      const int64_t off = w * i0;
      for (int q = tid; q < w * cnt; q += NT) {
        sprm[run_off<NT>(g) + q] = gprm[g][off + q];
        if (mv[g] != nullptr) sm[run_off<NT>(g) + q] = mv[g][off + q];
        if (mv[g + 5] != nullptr) sv[run_off<NT>(g) + q] = mv[g + 5][off + q];
      }
    }
  }

  // ---- merge this thread's pair partials in ascending brick order
  double s[11];
#pragma unroll
  for (int a = 0; a < 11; ++a) s[a] = 0.0;
  if (!merge) {
    if (valid) {
#pragma unroll
      for (int a = 0; a < 11; ++a) s[a] = gsum[12 * i + a];
    }
  } else {
    const int64_t my0 = valid ? gstart[i] : 0, my1 = valid ? gstart[i + 1] : 0;
    for (int c = 0; c < nch; ++c) {
      const int64_t c0 = e_lo + (int64_t)c * kTmaChunk;
      const int np = chunk_pairs(c);
      const float4* buf = spart + (tma ? (c & 1) * 3 * kTmaChunk : 0);
      if (tma) {
        tma::wait(bar + 1 + (c & 1), (uint32_t)((c >> 1) & 1));
      } else {
        __syncthreads();
        for (int q = tid; q < 3 * np; q += NT) spart[q] = __ldg(src + 3 * c0 + q);
        __syncthreads();
      }
      const int64_t a0 = max(my0, c0), a1 = min(my1, c0 + np);
      GSV_DCHECK(np >= 0 && np <= kTmaChunk && (a0 >= a1 || (a0 >= c0 && a1 <= c0 + np)));
      for (int64_t e = a0; e < a1; ++e) {
        const float4* pp = buf + 3 * (e - c0);
        const float4 x = pp[0], y = pp[1], z = pp[2];
        s[0] += (double)x.x; s[1] += (double)x.y; s[2] += (double)x.z; s[3] += (double)x.w;
        s[4] += (double)y.x; s[5] += (double)y.y; s[6] += (double)y.z; s[7] += (double)y.w;
        s[8] += (double)z.x; s[9] += (double)z.y; s[10] += (double)z.z;
      }
      if (tma) {
        __syncthreads();                       // buffer (c & 1) free again
        if (tid == 0 && c + 2 < nch) issue_chunk(c + 2);
      }
    }
  }
  if (tma) tma::wait(bar, 0);                  // parameter and moment runs
  else __syncthreads();

  if (valid) {
    double* P[5];
    double* M[5];
    double* V[5];
#pragma unroll
    for (int g = 0; g < 5; ++g) {
      P[g] = sprm + run_off<NT>(g) + run_w(g) * tid;
      M[g] = sm + run_off<NT>(g) + run_w(g) * tid;
      V[g] = sv + run_off<NT>(g) + run_w(g) * tid;
    }
    double g[12];
    chain_one(s, P[1], P[2], P[3][0], P[4][0], relax_en, g);
    double bc1 = h.bc1, bc2 = h.bc2;
    if (sd.bc != nullptr) {
      const int64_t t = *sd.t;
      bc1 = sd.bc[2 * t];
      bc2 = sd.bc[2 * t + 1];
    }
#pragma unroll
    for (int a = 0; a < 3; ++a)
      P[0][a] = adam_one(P[0][a], M[0][a], V[0][a], g[a], h.lr[0], h.b1, h.b2, h.eps, bc1, bc2);
#pragma unroll
    for (int a = 0; a < 3; ++a)
      P[1][a] = adam_one(P[1][a], M[1][a], V[1][a], g[3 + a], h.lr[1], h.b1, h.b2, h.eps, bc1,
                         bc2);
    double q[4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
      q[a] = adam_one(P[2][a], M[2][a], V[2][a], g[6 + a], h.lr[2], h.b1, h.b2, h.eps, bc1, bc2);
    const double nrm = sqrt(add(add(add(mul(q[0], q[0]), mul(q[1], q[1])), mul(q[2], q[2])),
                                mul(q[3], q[3])));
#pragma unroll
    for (int a = 0; a < 4; ++a) P[2][a] = __ddiv_rn(q[a], nrm);
    if (amp_en)
      P[3][0] = adam_one(P[3][0], M[3][0], V[3][0], g[10], h.lr[3], h.b1, h.b2, h.eps, bc1, bc2);
    if (relax_en)
      P[4][0] = adam_one(P[4][0], M[4][0], V[4][0], g[11], h.lr[4], h.b1, h.b2, h.eps, bc1, bc2);
  }

  // ---- write the updated runs back (enabled groups only)
  if (tma) {
    tma::fence_async_smem();
    __syncthreads();
    if (tid == 0) {
#pragma unroll
      for (int g = 0; g < 5; ++g) {
        if (!en[g]) continue;
        const uint32_t b = (uint32_t)(8 * run_w(g) * NT);
        const int64_t off = run_w(g) * i0;
        tma::s2g(gprm[g] + off, sprm + run_off<NT>(g), b);
        if (mv[g] != nullptr) tma::s2g(mv[g] + off, sm + run_off<NT>(g), b);
        if (mv[g + 5] != nullptr) tma::s2g(mv[g + 5] + off, sv + run_off<NT>(g), b);
      }
      tma::store_commit();
    }
  } else {
    __syncthreads();
#pragma unroll
    for (int g = 0; g < 5; ++g) {
      if (!en[g]) continue;
      const int w = run_w(g);
      const int64_t off = w * i0;
      for (int q = tid; q < w * cnt; q += NT) {
        gprm[g][off + q] = sprm[run_off<NT>(g) + q];
        if (mv[g] != nullptr) mv[g][off + q] = sm[run_off<NT>(g) + q];
        if (mv[g + 5] != nullptr) mv[g + 5][off + q] = sv[run_off<NT>(g) + q];
      }
    }
  }
  if (tma && tid == 0) tma::store_wait_read();
}

}  // namespace
}  // namespace gsv

using namespace gsv;

namespace {
// TMA tail (default for the tail without PREP) or the per-thread-load tail
// (GSV_TAIL_V1=1, for A/B runs).
bool use_tma_tail() {
  static const bool v = [] {
    const char* e = getenv("GSV_TAIL_V1");
    return !(e != nullptr && e[0] == '1');
  }();
  return v;
}

bool aligned16(const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

int launch_tail_tma(cudaStream_t s, const float* partials,
                    const int64_t* gstart, const double* gsum, int64_t n, double* pos,
                    double* ls, double* rot, double* ra, double* rr, const MomentPtrs& mv,
                    int amp_en, int relax_en, const gsv_adam_hparams& h, const StepDev& sd) {
  constexpr size_t smem = tma_smem<kTmaThreads>();
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tail_tma_kernel<kTmaThreads>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_status(e, "tail_tma_kernel smem attribute");
    attr = true;
  }
  int ok = aligned16(partials) && aligned16(pos) && aligned16(ls) && aligned16(rot) &&
           aligned16(ra) && aligned16(rr);
  for (int k = 0; k < 10; ++k) ok = ok && aligned16(mv.p[k]);
  const unsigned blocks = (unsigned)((n + kTmaThreads - 1) / kTmaThreads);
  tail_tma_kernel<kTmaThreads><<<blocks, kTmaThreads, smem, s>>>(
      partials, gstart, gsum, n, pos, ls, rot, ra, rr, mv, amp_en, relax_en, h, sd, ok);
  GSV_CHECK_LAUNCH("tail_tma_kernel");
  return GSV_OK;
}
}  // namespace

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

int gsv_fused_update(const void* partials, const int64_t* gstart, const double* gsum,
                     int64_t n, int precision, double* positions, double* log_scales,
                     double* rotations, double* raw_amplitude, double* raw_relax,
                     double* const* moments, int amplitude_enabled, int relax_enabled,
                     const gsv_adam_hparams* hp, double* grad_scratch, void* stream) {
  GSV_REQUIRE(hp != nullptr && moments != nullptr, "null hparams/moments");
  GSV_REQUIRE(gsum != nullptr || (partials != nullptr && gstart != nullptr),
              "need gsum or partials+gstart");
  if (n <= 0) return GSV_OK;
  cudaStream_t s = as_stream(stream);
  MomentPtrs mv;
  for (int k = 0; k < 10; ++k) mv.p[k] = moments[k];
  if (precision == 0 && grad_scratch == nullptr) {
    // one pass: staged merge + chain rule + Adam + renorm
    if (use_tma_tail())
      return launch_tail_tma(s,
                                    (const float*)partials, gstart, gsum, n, positions,
                                    log_scales, rotations, raw_amplitude, raw_relax, mv,
                                    amplitude_enabled, relax_enabled, *hp,
                                    StepDev{nullptr, nullptr, nullptr});
    tail_kernel<false><<<(unsigned)((n + kTailThreads - 1) / kTailThreads), kTailThreads, 0, s>>>(
        (const float*)partials, gstart, gsum, n, positions, log_scales, rotations,
        raw_amplitude, raw_relax, mv, amplitude_enabled, relax_enabled, *hp,
        StepDev{nullptr, nullptr, nullptr}, PrepArgs{});
    GSV_CHECK_LAUNCH("tail_kernel");
    return GSV_OK;
  }
  GSV_REQUIRE(grad_scratch != nullptr, "the f64 tail needs grad_scratch (N,12) double");
  const unsigned b128 = (unsigned)((n + 127) / 128), b256 = (unsigned)((n + 255) / 256);
  if (precision == 0)
    merge_chain_kernel<float><<<b128, 128, 0, s>>>((const float*)partials, gstart, gsum, n,
                                                   log_scales, rotations, raw_amplitude,
                                                   raw_relax, relax_enabled, grad_scratch);
  else
    merge_chain_kernel<double><<<b128, 128, 0, s>>>((const double*)partials, gstart, gsum, n,
                                                    log_scales, rotations, raw_amplitude,
                                                    raw_relax, relax_enabled, grad_scratch);
  GSV_CHECK_LAUNCH("merge_chain_kernel");
  adam12_kernel<<<b256, 256, 0, s>>>(grad_scratch, n, positions, log_scales, rotations,
                                     raw_amplitude, raw_relax, mv, amplitude_enabled,
                                     relax_enabled, *hp);
  GSV_CHECK_LAUNCH("adam12_kernel");
  return GSV_OK;
}

int gsv_step_gate(const double* loss_sum, const int32_t* overflow, int32_t* gate,
                  double* result, void* stream) {
  GSV_REQUIRE(loss_sum && overflow && gate && result, "null pointer argument");
  gate_kernel<<<1, 1, 0, as_stream(stream)>>>(loss_sum, overflow, gate, result);
  GSV_CHECK_LAUNCH("gate_kernel");
  return GSV_OK;
}

int gsv_shard_pack(const double* gsum, int64_t n, const double* loss_sum, const int32_t* overflow,
                   float* red, void* stream) {
  GSV_REQUIRE(gsum && loss_sum && overflow && red, "null pointer argument");
  GSV_REQUIRE(n >= 2, "the sharded reduce buffer needs N >= 2 Gaussians");
  const int64_t n12 = 12 * n;
  shard_pack_kernel<<<(unsigned)((n12 + 255) / 256), 256, 0, as_stream(stream)>>>(
      gsum, n12, loss_sum, overflow, red);
  GSV_CHECK_LAUNCH("shard_pack_kernel");
  return GSV_OK;
}

int gsv_shard_unpack(const float* red, int64_t n, double* gsum, double* loss_sum,
                     int32_t* overflow, void* stream) {
  GSV_REQUIRE(gsum && loss_sum && overflow && red, "null pointer argument");
  GSV_REQUIRE(n >= 2, "the sharded reduce buffer needs N >= 2 Gaussians");
  const int64_t n12 = 12 * n;
  shard_unpack_kernel<<<(unsigned)((n12 + 255) / 256), 256, 0, as_stream(stream)>>>(
      red, n12, gsum, loss_sum, overflow);
  GSV_CHECK_LAUNCH("shard_unpack_kernel");
  return GSV_OK;
}

int gsv_fused_update_device(const float* partials, const int64_t* gstart, const double* gsum,
                            int64_t n,
                            double* positions, double* log_scales, double* rotations,
                            double* raw_amplitude, double* raw_relax, double* const* moments,
                            int amplitude_enabled, int relax_enabled,
                            const gsv_adam_hparams* hp, const double* bias_corrections,
                            const int64_t* step, const int32_t* gate, const gsv_grid* grid,
                            const gsv_bricks* bricks, double cutoff_sigma,
                            gsv_record32* rec32, int32_t* counts, int32_t* box, void* stream) {
  GSV_REQUIRE(hp && moments && bias_corrections && step && gate, "null pointer argument");
  GSV_REQUIRE(gsum != nullptr || (partials && gstart), "need gsum or partials + gstart");
  GSV_REQUIRE(rec32 == nullptr || (grid && bricks && counts && box && cutoff_sigma > 0),
              "records need grid, bricks, counts, box and a positive cutoff");
  if (n <= 0) return GSV_OK;
  cudaStream_t s = as_stream(stream);
  MomentPtrs mv;
  for (int k = 0; k < 10; ++k) mv.p[k] = moments[k];
  const unsigned blocks = (unsigned)((n + kTailThreads - 1) / kTailThreads);
  const StepDev sd{gate, bias_corrections, step};
  if (rec32 != nullptr) {
    if (int st = validate_grid_bricks(grid, bricks)) return st;
    const PrepArgs pa{*grid, *bricks, cutoff_sigma, isinf(cutoff_sigma) ? 1 : 0, relax_enabled,
                      rec32, nullptr, counts, box};
    // PREP stays on the L2-prefetch tail: measured faster there (0.49 vs
    // 0.55 ms at config 3), its f64 preprocessing wants the warps that the
    // TMA tail's shared staging takes away.
    tail_kernel<true><<<blocks, kTailThreads, 0, s>>>(
        partials, gstart, gsum, n, positions, log_scales, rotations, raw_amplitude,
        raw_relax, mv, amplitude_enabled, relax_enabled, *hp, sd, pa);
  } else {
    if (use_tma_tail())
      return launch_tail_tma(s, partials, gstart, gsum, n, positions, log_scales,
                                    rotations, raw_amplitude, raw_relax, mv, amplitude_enabled,
                                    relax_enabled, *hp, sd);
    tail_kernel<false><<<blocks, kTailThreads, 0, s>>>(
        partials, gstart, gsum, n, positions, log_scales, rotations, raw_amplitude,
        raw_relax, mv, amplitude_enabled, relax_enabled, *hp, sd, PrepArgs{});
  }
  GSV_CHECK_LAUNCH("tail_kernel");
  return GSV_OK;
}

int gsv_step_advance(int64_t* step, const int32_t* gate, void* stream) {
  GSV_REQUIRE(step && gate, "null pointer argument");
  advance_kernel<<<1, 1, 0, as_stream(stream)>>>(step, gate);
  GSV_CHECK_LAUNCH("advance_kernel");
  return GSV_OK;
}

int gsv_step_advance_publish(int64_t* step, const int32_t* gate, const double* result,
                             double* ring, int64_t* counter, int slots, void* stream) {
  GSV_REQUIRE(step && gate && result && ring && counter, "null pointer argument");
  GSV_REQUIRE(slots >= 1, "slots must be >= 1");
  advance_publish_kernel<<<1, 1, 0, as_stream(stream)>>>(step, gate, result, ring, counter,
                                                         slots);
  GSV_CHECK_LAUNCH("advance_publish_kernel");
  return GSV_OK;
}

int gsv_normalize_rotations(double* rotations, int64_t n, void* stream) {
  if (n <= 0) return GSV_OK;
  normalize_kernel<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(rotations, n);
  GSV_CHECK_LAUNCH("normalize_kernel");
  return GSV_OK;
}

}  // extern "C"
