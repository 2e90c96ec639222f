// gsv_setup.cu -- one-time setup of a fit on the device:
// phantom rasterization and blur (phantom.py:52-75), trilinear resampling
// (volume.py:126-154) and init_from_volume (field.py:212-234).
//
// resample: the reference's numpy operation order, every product and sum an
// explicit round-to-nearest f64 op, so the result is bit-identical to
// resample_trilinear (also the host restatement in volume.py).
// init: positions, log_scales, rotations and raw_relax are bit-identical to
// the reference; raw_amplitude = logit(clip(I, 1e-4, 1 - 1e-4)) uses the
// device log/log1p in xsf's formula, within a few ulp of scipy's (glibc).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include "gsv_common.cuh"

namespace gsv {
namespace {

__device__ __forceinline__ double load_vox(const void* p, int f64, int64_t i) {
  return f64 ? static_cast<const double*>(p)[i] : (double)static_cast<const float*>(p)[i];
}

// Per target coordinate along one axis: i0, i1 and the fraction, exactly as
// resample_trilinear: world = o + i * s; u = (world - so) / ss, clipped to
// [0, n - 1]; i0 = clip(floor(u), 0, max(n - 2, 0)); i1 = min(i0 + 1, n - 1).
__device__ __forceinline__ void axis_coord(int i, double o, double s, double so, double ss,
                                           int n, int& i0, int& i1, double& fr) {
  const double world = add(o, mul((double)i, s));
  double u = __ddiv_rn(sub(world, so), ss);
  u = fmin(fmax(u, 0.0), (double)(n - 1));
  int a = (int)floor(u);
  a = max(0, min(a, max(n - 2, 0)));
  i0 = a;
  i1 = min(a + 1, n - 1);
  fr = sub(u, (double)a);
}

__global__ void __launch_bounds__(256)
resample_kernel(const void* __restrict__ src, int f64, gsv_grid sg, void* __restrict__ out,
                gsv_grid dg) {
  const int64_t nv = (int64_t)dg.nx * dg.ny * dg.nz;
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= nv) return;
  const int x = (int)(v % dg.nx), y = (int)((v / dg.nx) % dg.ny), z = (int)(v / ((int64_t)dg.nx * dg.ny));
  int lx, hx, ly, hy, lz, hz;
  double fx, fy, fz;
  axis_coord(x, dg.ox, dg.sx, sg.ox, sg.sx, sg.nx, lx, hx, fx);
  axis_coord(y, dg.oy, dg.sy, sg.oy, sg.sy, sg.ny, ly, hy, fy);
  axis_coord(z, dg.oz, dg.sz, sg.oz, sg.sz, sg.nz, lz, hz, fz);
  const int cx[2] = {lx, hx}, cy[2] = {ly, hy}, cz[2] = {lz, hz};
  const double wx[2] = {sub(1.0, fx), fx}, wy[2] = {sub(1.0, fy), fy},
               wz[2] = {sub(1.0, fz), fz};
  double acc = 0.0;
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const double w = mul(mul(wx[a], wy[b]), wz[c]);
        const int64_t si = cx[a] + (int64_t)sg.nx * (cy[b] + (int64_t)sg.ny * cz[c]);
        acc = add(acc, mul(w, load_vox(src, f64, si)));
      }
  if (f64)
    static_cast<double*>(out)[v] = acc;
  else
    static_cast<float*>(out)[v] = __double2float_rn(acc);
}

// init: mask in numpy's argwhere order (C order over [ix, iy, iz]: ix slowest)
struct InitMask {
  const void* data;
  int f64;
  int nx, ny, nz;
  double thr;
  __device__ __forceinline__ int64_t lin(int64_t c) const {   // C-order index -> x-fastest
    const int64_t iz = c % nz, iy = (c / nz) % ny, ix = c / ((int64_t)nz * ny);
    return ix + (int64_t)nx * (iy + (int64_t)ny * iz);
  }
  __device__ __forceinline__ int operator()(int64_t c) const {
    return load_vox(data, f64, lin(c)) >= thr ? 1 : 0;
  }
};

// the mask over nv + 1 elements (the one past the end reads 0): the
// exclusive scan's last entry is then N
struct InitGuard {
  InitMask m;
  int64_t nv;
  __device__ __forceinline__ int operator()(int64_t c) const { return c < nv ? m(c) : 0; }
};
using InitIt = thrust::transform_iterator<InitGuard, thrust::counting_iterator<int64_t>, int>;

__global__ void __launch_bounds__(256)
init_fill_kernel(InitMask m, const int64_t* __restrict__ slot, gsv_grid g, double ls0,
                 double ls1, double ls2, double raw_relax, double* __restrict__ pos,
                 double* __restrict__ ls, double* __restrict__ rot, double* __restrict__ ra,
                 double* __restrict__ rr) {
  const int64_t nv = (int64_t)g.nx * g.ny * g.nz;
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= nv || !m(c)) return;
  const int64_t i = slot[c];
  const int64_t iz = c % g.nz, iy = (c / g.nz) % g.ny, ix = c / ((int64_t)g.nz * g.ny);
  // positions = origin + vox * spacing (numpy: mul, then add)
  pos[3 * i] = add(g.ox, mul((double)ix, g.sx));
  pos[3 * i + 1] = add(g.oy, mul((double)iy, g.sy));
  pos[3 * i + 2] = add(g.oz, mul((double)iz, g.sz));
  ls[3 * i] = ls0;
  ls[3 * i + 1] = ls1;
  ls[3 * i + 2] = ls2;
  rot[4 * i] = 1.0;
  rot[4 * i + 1] = 0.0;
  rot[4 * i + 2] = 0.0;
  rot[4 * i + 3] = 0.0;
  const double x = fmin(fmax(load_vox(m.data, m.f64, m.lin(c)), 1e-4), 1.0 - 1e-4);
  double lg;
  if (x < 0.3 || x > 0.65) {
    lg = log(__ddiv_rn(x, sub(1.0, x)));
  } else {
    const double s = sub(mul(2.0, x), 1.0);
    lg = sub(log1p(s), log1p(-s));
  }
  ra[i] = lg;
  rr[i] = raw_relax;
}

// LR-consistency loss (north_star (c); no reference counterpart): the LR
// prediction is the mean of each LR voxel's fx*fy*fz HR voxels of the HR
// render; loss and dL/dI per LR voxel as loss_and_grad (optimize.py:91-103);
// dL/dI_HR = dL/dI_LR / (fx fy fz) for each HR voxel of the block, written
// as the backward's {alpha = dL/dI / W, I}.  One thread per LR voxel; the
// mean is summed in x-fastest order in f64; per-CTA loss partials (fixed
// tree) for a deterministic total.
constexpr int kPoolThreads = 256;
__global__ void __launch_bounds__(kPoolThreads)
pool_loss_kernel(const float* __restrict__ I, const float* __restrict__ W,
                 const void* __restrict__ target, int target_f64, gsv_grid hr, gsv_grid lr,
                 int fx, int fy, int fz, int kind, double eps_w, float2* __restrict__ ab,
                 double* __restrict__ part) {
  __shared__ double sh[kPoolThreads / 32];
  const int64_t nl = (int64_t)lr.nx * lr.ny * lr.nz;
  const int64_t v = blockIdx.x * (int64_t)kPoolThreads + threadIdx.x;
  double acc = 0.0;
  if (v < nl) {
    const int x = (int)(v % lr.nx), y = (int)((v / lr.nx) % lr.ny),
              z = (int)(v / ((int64_t)lr.nx * lr.ny));
    const double inv_n = 1.0 / (double)(fx * fy * fz);
    double sum = 0.0;
    for (int c = 0; c < fz; ++c)
      for (int b = 0; b < fy; ++b)
        for (int a = 0; a < fx; ++a) {
          const int64_t h = (int64_t)(x * fx + a) +
                            (int64_t)hr.nx * ((y * fy + b) + (int64_t)hr.ny * (z * fz + c));
          sum += (double)I[h];
        }
    const double d = sum * inv_n - load_vox(target, target_f64, v);
    double dl;
    if (kind == 0) {
      acc = fabs(d);
      dl = (d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0)) / (double)nl;
    } else {
      acc = d * d;
      dl = 2.0 * d / (double)nl;
    }
    const double dh = dl * inv_n;
    for (int c = 0; c < fz; ++c)
      for (int b = 0; b < fy; ++b)
        for (int a = 0; a < fx; ++a) {
          const int64_t h = (int64_t)(x * fx + a) +
                            (int64_t)hr.nx * ((y * fy + b) + (int64_t)hr.ny * (z * fz + c));
          const double w = (double)W[h];
          const float alpha = (w >= eps_w && dh != 0.0) ? (float)(dh / w) : 0.f;
          ab[h] = make_float2(alpha, I[h]);
        }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kPoolThreads / 32; ++w) t += sh[w];
    part[blockIdx.x] = t;
  }
}

// ---- phantom (phantom.py:52-75).  Voxel (i, j, k) at axis_coords (origin +
// index * spacing); d2 = ((x - c) / a)^2 summed x, y, z left to right, each
// op rounded as numpy does; max over the primitives in order.  The volume is
// x-fastest linear (Volume.linear()).  Ellipsoids: intensity where d2 <= 1.
// Gaussian mixture: intensity * exp(-0.5 d2) (the device exp, within an ulp
// of numpy's).
__global__ void __launch_bounds__(256)
phantom_kernel(gsv_grid g, int kind, int np_, const double* __restrict__ prims,
               double* __restrict__ out) {
  const int64_t nv = (int64_t)g.nx * g.ny * g.nz;
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= nv) return;
  const int x = (int)(v % g.nx), y = (int)((v / g.nx) % g.ny),
            z = (int)(v / ((int64_t)g.nx * g.ny));
  const double px = add(g.ox, mul((double)x, g.sx)), py = add(g.oy, mul((double)y, g.sy)),
               pz = add(g.oz, mul((double)z, g.sz));
  double acc = 0.0;
  for (int q = 0; q < np_; ++q) {
    const double* pr = prims + 7 * q;   // cx cy cz ax ay az intensity
    const double tx = __ddiv_rn(sub(px, pr[0]), pr[3]);
    const double ty = __ddiv_rn(sub(py, pr[1]), pr[4]);
    const double tz = __ddiv_rn(sub(pz, pr[2]), pr[5]);
    const double d2 = add(add(mul(tx, tx), mul(ty, ty)), mul(tz, tz));
    const double val = kind == 0 ? (d2 <= 1.0 ? pr[6] : 0.0) : mul(pr[6], exp(mul(-0.5, d2)));
    acc = fmax(acc, val);
  }
  out[v] = acc;
}

// One axis of ndimage.gaussian_filter (scipy's symmetric correlate1d, mode
// "reflect"): o = x[c] w[r] + sum_{j = -r .. -1} (x[c + j] + x[c - j]) w[r + j]
// in that order, indices reflected about the half-sample edges.
__device__ __forceinline__ int reflect_index(int i, int n) {
  const int p = 2 * n;
  int m = i % p;
  if (m < 0) m += p;
  return m < n ? m : p - 1 - m;
}

__global__ void __launch_bounds__(256)
blur_axis_kernel(const double* __restrict__ in, double* __restrict__ out, int nx, int ny, int nz,
                 int axis, int radius, const double* __restrict__ w) {
  const int64_t nv = (int64_t)nx * ny * nz;
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= nv) return;
  const int x = (int)(v % nx), y = (int)((v / nx) % ny), z = (int)(v / ((int64_t)nx * ny));
  const int n = axis == 0 ? nx : (axis == 1 ? ny : nz);
  const int c = axis == 0 ? x : (axis == 1 ? y : z);
  const int64_t stride = axis == 0 ? 1 : (axis == 1 ? (int64_t)nx : (int64_t)nx * ny);
  const int64_t base = v - (int64_t)c * stride;
  double o = mul(in[v], w[radius]);
  for (int j = -radius; j < 0; ++j) {
    const double a = in[base + (int64_t)reflect_index(c + j, n) * stride];
    const double b = in[base + (int64_t)reflect_index(c - j, n) * stride];
    o = add(o, mul(add(a, b), w[radius + j]));
  }
  out[v] = o;
}

__global__ void __launch_bounds__(256)
clip_f32_kernel(const double* __restrict__ in, float* __restrict__ out, int64_t nv) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v < nv) out[v] = (float)fmin(fmax(in[v], 0.0), 1.0);
}

}  // namespace
}  // namespace gsv

using namespace gsv;

extern "C" {

int gsv_resample_trilinear(const void* src, int src_f64, const gsv_grid* src_grid, void* out,
                           const gsv_grid* dst_grid, void* stream) {
  GSV_REQUIRE(src_grid && dst_grid, "grids required");
  GSV_REQUIRE(src_grid->nx >= 1 && src_grid->ny >= 1 && src_grid->nz >= 1 && dst_grid->nx >= 1 &&
                  dst_grid->ny >= 1 && dst_grid->nz >= 1,
              "grid dims must be >= 1");
  GSV_REQUIRE(src_f64 == 0 || src_f64 == 1, "src_f64 must be 0 or 1");
  const int64_t nv = (int64_t)dst_grid->nx * dst_grid->ny * dst_grid->nz;
  resample_kernel<<<(unsigned)((nv + 255) / 256), 256, 0, as_stream(stream)>>>(
      src, src_f64, *src_grid, out, *dst_grid);
  GSV_CHECK_LAUNCH("resample_kernel");
  return GSV_OK;
}

int gsv_pool_loss_blocks(const gsv_grid* lr_grid) {
  const int64_t nl = (int64_t)lr_grid->nx * lr_grid->ny * lr_grid->nz;
  return (int)((nl + kPoolThreads - 1) / kPoolThreads);
}

int gsv_pool_loss(const float* I, const float* W, const void* target, int target_dtype,
                  const gsv_grid* hr_grid, const gsv_grid* lr_grid, int fx, int fy, int fz,
                  int loss_kind, double eps_w, float* ab, double* loss_part, void* stream) {
  GSV_REQUIRE(hr_grid && lr_grid, "grids required");
  GSV_REQUIRE(fx >= 1 && fy >= 1 && fz >= 1, "factors must be >= 1");
  GSV_REQUIRE(hr_grid->nx == lr_grid->nx * fx && hr_grid->ny == lr_grid->ny * fy &&
                  hr_grid->nz == lr_grid->nz * fz,
              "HR dims must be the LR dims times the factors");
  GSV_REQUIRE(loss_kind == 0 || loss_kind == 1, "loss_kind must be 0 (l1) or 1 (l2)");
  GSV_REQUIRE(target_dtype == 0 || target_dtype == 1, "target_dtype must be 0 or 1");
  pool_loss_kernel<<<(unsigned)gsv_pool_loss_blocks(lr_grid), kPoolThreads, 0,
                     as_stream(stream)>>>(I, W, target, target_dtype, *hr_grid, *lr_grid, fx, fy,
                                          fz, loss_kind, eps_w, (float2*)ab, loss_part);
  GSV_CHECK_LAUNCH("pool_loss_kernel");
  return GSV_OK;
}

int gsv_init_workspace(const gsv_grid* grid, size_t* bytes) {
  GSV_REQUIRE(grid && bytes, "grid and bytes required");
  const int64_t nv = (int64_t)grid->nx * grid->ny * grid->nz;
  InitIt in(thrust::counting_iterator<int64_t>(0),
            InitGuard{InitMask{nullptr, 0, grid->nx, grid->ny, grid->nz, 0.0}, nv});
  size_t b = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, b, in, (int64_t*)nullptr, nv + 1);
  if (e != cudaSuccess) return cuda_status(e, "init workspace");
  *bytes = b;
  return GSV_OK;
}

int gsv_init_count(const void* data, int data_f64, const gsv_grid* grid, double threshold,
                   int64_t* slot, void* workspace, size_t workspace_bytes, void* stream) {
  GSV_REQUIRE(grid && grid->nx >= 1 && grid->ny >= 1 && grid->nz >= 1, "bad grid");
  GSV_REQUIRE(data_f64 == 0 || data_f64 == 1, "data_f64 must be 0 or 1");
  const int64_t nv = (int64_t)grid->nx * grid->ny * grid->nz;
  InitIt in(thrust::counting_iterator<int64_t>(0),
            InitGuard{InitMask{data, data_f64, grid->nx, grid->ny, grid->nz, threshold}, nv});
  size_t b = workspace_bytes;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(workspace, b, in, slot, nv + 1,
                                                as_stream(stream));
  if (e != cudaSuccess) return cuda_status(e, "init count");
  return GSV_OK;
}

int gsv_init_fill(const void* data, int data_f64, const gsv_grid* grid, double threshold,
                  const int64_t* slot, const double* log_scales3, double raw_relax,
                  double* positions, double* log_scales, double* rotations,
                  double* raw_amplitude, double* raw_relax_out, void* stream) {
  GSV_REQUIRE(grid && grid->nx >= 1 && grid->ny >= 1 && grid->nz >= 1, "bad grid");
  GSV_REQUIRE(log_scales3 != nullptr, "log_scales3 (host) required");
  const int64_t nv = (int64_t)grid->nx * grid->ny * grid->nz;
  InitMask m{data, data_f64, grid->nx, grid->ny, grid->nz, threshold};
  init_fill_kernel<<<(unsigned)((nv + 255) / 256), 256, 0, as_stream(stream)>>>(
      m, slot, *grid, log_scales3[0], log_scales3[1], log_scales3[2], raw_relax, positions,
      log_scales, rotations, raw_amplitude, raw_relax_out);
  GSV_CHECK_LAUNCH("init_fill_kernel");
  return GSV_OK;
}

int gsv_phantom(const gsv_grid* grid, int kind, int nprims, const double* prims, int radius,
                const double* weights, double* scratch, float* out, void* stream) {
  GSV_REQUIRE(grid && out && scratch, "null pointer argument");
  GSV_REQUIRE(grid->nx >= 1 && grid->ny >= 1 && grid->nz >= 1, "grid dims must be >= 1");
  GSV_REQUIRE(kind == 0 || kind == 1, "kind must be 0 (ellipsoids) or 1 (gaussian mixture)");
  GSV_REQUIRE(nprims >= 0 && (nprims == 0 || prims != nullptr), "bad primitive list");
  GSV_REQUIRE(radius >= 0 && (radius == 0 || weights != nullptr), "bad blur weights");
  cudaStream_t s = as_stream(stream);
  const int64_t nv = (int64_t)grid->nx * grid->ny * grid->nz;
  const unsigned blocks = (unsigned)((nv + 255) / 256);
  double* a = scratch;
  double* b = scratch + nv;
  phantom_kernel<<<blocks, 256, 0, s>>>(*grid, kind, nprims, prims, a);
  GSV_CHECK_LAUNCH("phantom_kernel");
  if (radius > 0) {
    for (int axis = 0; axis < 3; ++axis) {
      blur_axis_kernel<<<blocks, 256, 0, s>>>(a, b, grid->nx, grid->ny, grid->nz, axis, radius,
                                              weights);
      GSV_CHECK_LAUNCH("blur_axis_kernel");
      double* t = a;
      a = b;
      b = t;
    }
  }
  clip_f32_kernel<<<blocks, 256, 0, s>>>(a, out, nv);
  GSV_CHECK_LAUNCH("clip_f32_kernel");
  return GSV_OK;
}

}  // extern "C"
