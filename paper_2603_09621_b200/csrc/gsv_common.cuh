// gsv_common.cuh -- shared device helpers for the B200 brick rasterizer.
//
// The f64 helpers reproduce the reference's numpy/numba arithmetic bit for
// bit where the reference's decisions depend on it (binning bounds,
// truncation test): every multiply and add is an explicit round-to-nearest
// intrinsic, so nvcc can never contract them into an FMA (numba 0.65 / numpy
// emit no FMA contraction, SURVEY.md §0 finding 1).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/gsv.h"

namespace gsv {

// ----------------------------------------------------------------- errors
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* what);

#define GSV_CHECK_LAUNCH(what)                                   \
  do {                                                           \
    cudaError_t _e = cudaGetLastError();                         \
    if (_e != cudaSuccess) return ::gsv::cuda_status(_e, what);  \
  } while (0)

#define GSV_REQUIRE(cond, ...)            \
  do {                                    \
    if (!(cond)) {                        \
      ::gsv::set_error(__VA_ARGS__);      \
      return GSV_ERR_ARG;                 \
    }                                     \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Device-side bounds checks for the debug variant (compute-sanitizer is not
// available on the GPU pool): `python -m paper_2603_09621_b200.build
// --variant dcheck -D GSV_DEBUG_CHECKS=1`, loaded with GSV_LIB; a failed check
// traps the kernel (the launch returns an error).  Compiled out otherwise.
#if defined(GSV_DEBUG_CHECKS) && GSV_DEBUG_CHECKS
#define GSV_DCHECK(cond)  \
  do {                    \
    if (!(cond)) __trap(); \
  } while (0)
#else
#define GSV_DCHECK(cond) \
  do {                   \
  } while (0)
#endif

// ------------------------------------------------------- unfused f64 math
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

// Rotation matrix of the stored (not renormalised) quaternion, numpy operand
// order of field.rotation_matrices (field.py:141-154):
//   R00 = 1 - 2*(y*y + z*z), R01 = 2*(x*y - w*z), ...
__device__ __forceinline__ void rotation_f64(const double* q, double R[9]) {
  const double w = q[0], x = q[1], y = q[2], z = q[3];
  const double xx = mul(x, x), yy = mul(y, y), zz = mul(z, z);
  const double xy = mul(x, y), xz = mul(x, z), yz = mul(y, z);
  const double wx = mul(w, x), wy = mul(w, y), wz = mul(w, z);
  R[0] = sub(1.0, mul(2.0, add(yy, zz)));
  R[1] = mul(2.0, sub(xy, wz));
  R[2] = mul(2.0, add(xz, wy));
  R[3] = mul(2.0, add(xy, wz));
  R[4] = sub(1.0, mul(2.0, add(xx, zz)));
  R[5] = mul(2.0, sub(yz, wx));
  R[6] = mul(2.0, sub(xz, wy));
  R[7] = mul(2.0, add(yz, wx));
  R[8] = sub(1.0, mul(2.0, add(xx, yy)));
}

// Whitening factor L = diag(exp(-ls)) R^T, i.e. L[a][b] = exp(-ls_a) R[b][a]
// (_whitening_factors, raster.py:233-237).
__device__ __forceinline__ void whitening_f64(const double* ls, const double* q,
                                              double L[9]) {
  double R[9];
  rotation_f64(q, R);
  const double i0 = exp(-ls[0]), i1 = exp(-ls[1]), i2 = exp(-ls[2]);
  L[0] = mul(i0, R[0]); L[1] = mul(i0, R[3]); L[2] = mul(i0, R[6]);
  L[3] = mul(i1, R[1]); L[4] = mul(i1, R[4]); L[5] = mul(i1, R[7]);
  L[6] = mul(i2, R[2]); L[7] = mul(i2, R[5]); L[8] = mul(i2, R[8]);
}

// Exact f64 truncation decision of the reference forward/backward kernels
// (raster.py:265-279): px = ox + ix*sx; dx = px - mx; v = L dx (left to
// right); d2 = v0*v0 + v1*v1 + v2*v2; live iff d2 <= cutoff2.
__device__ __forceinline__ double ref_d2(const double L[9], double mx, double my,
                                         double mz, int ix, int iy, int iz,
                                         const gsv_grid& g) {
  const double dx = sub(add(g.ox, mul((double)ix, g.sx)), mx);
  const double dy = sub(add(g.oy, mul((double)iy, g.sy)), my);
  const double dz = sub(add(g.oz, mul((double)iz, g.sz)), mz);
  const double v0 = add(add(mul(L[0], dx), mul(L[1], dy)), mul(L[2], dz));
  const double v1 = add(add(mul(L[3], dx), mul(L[4], dy)), mul(L[5], dz));
  const double v2 = add(add(mul(L[6], dx), mul(L[7], dy)), mul(L[8], dz));
  return add(add(mul(v0, v0), mul(v1, v1)), mul(v2, v2));
}

// scipy.special.expit in f64.
__device__ __forceinline__ double expit_f64(double x) {
  return 1.0 / (1.0 + exp(-x));
}

// Brick coordinates of a global brick id (raster.py:247-250).
struct BrickXYZ {
  int bx, by, bz;
};
__device__ __forceinline__ BrickXYZ brick_xyz(int b, const gsv_bricks& k) {
  BrickXYZ r;
  r.bx = b % k.bgx;
  const int rem = b / k.bgx;
  r.by = rem % k.bgy;
  r.bz = rem / k.bgy;
  return r;
}

// Unpack the per-Gaussian slab-clipped brick box written by preprocess.
// k0 = box-order index (x-fastest within the box) of the first brick inside
// the slab's id range; the slab's bricks of the box are box-order
// [k0, k0 + counts[i]) (box order and brick-id order are both lexicographic
// in (z, y, x), so an id range meets a box in one contiguous run).
struct GBox {
  int blo_x, blo_y, blo_z, nb_x, nb_y, nb_z, k0;
};
__device__ __forceinline__ GBox unpack_box(const int32_t* box, int64_t i) {
  const int4 b = reinterpret_cast<const int4*>(box)[i];
  GBox r;
  r.blo_x = b.x & 0xFFFF;
  r.blo_y = (b.x >> 16) & 0xFFFF;
  r.blo_z = b.y & 0xFFFF;
  r.nb_x = (b.y >> 16) & 0xFFFF;
  r.nb_y = b.z & 0xFFFF;
  r.nb_z = (b.z >> 16) & 0xFFFF;
  r.k0 = b.w;
  return r;
}
// Slot of brick (bx, by, bz) in the Gaussian's run of pair slots (the order
// binning emitted them: box order from k0), or -1 if binning emitted none.
__device__ __forceinline__ int64_t box_slot(const GBox& gb, int bx, int by, int bz) {
  const int rx = bx - gb.blo_x, ry = by - gb.blo_y, rz = bz - gb.blo_z;
  if (rx < 0 || rx >= gb.nb_x || ry < 0 || ry >= gb.nb_y || rz < 0 || rz >= gb.nb_z) return -1;
  const int64_t k = rx + (int64_t)gb.nb_x * (ry + (int64_t)gb.nb_y * rz) - gb.k0;
  return k >= 0 ? k : -1;
}

__host__ __device__ inline int64_t slab_bricks(const gsv_bricks& k) {
  return (int64_t)k.b1 - k.b0;
}
__host__ __device__ inline int64_t slab_first(const gsv_bricks& k) {
  return k.b0;
}

int validate_grid_bricks(const gsv_grid* g, const gsv_bricks* k);

}  // namespace gsv
