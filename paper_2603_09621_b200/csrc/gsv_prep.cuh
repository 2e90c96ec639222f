// gsv_prep.cuh -- per-Gaussian preprocessing shared by the binning pass
// (gsv_bin.cu: preprocess_kernel) and the graph step's fused optimizer tail
// (gsv_train.cu: tail_kernel<PREP>), which writes the next step's records
// straight from the updated parameters.
//
// Replaces _whitening_factors (raster.py:233-237), the sigmoid activations
// (field.py:86-94) and the AABB part of build_brick_index (raster.py:160-198).
// Every f64 operation that feeds a binning decision is an explicit _rn
// intrinsic (or a libm call / exact scaling), so the result does not depend
// on the translation unit's contraction flags.
#pragma once

#include "gsv_common.cuh"

namespace gsv {

// numpy float64 -> int64 cast on x86-64 (cvttsd2si / vcvttpd2qq): truncation,
// with NaN and out-of-range values mapping to INT64_MIN.
__device__ __forceinline__ int64_t np_to_int64(double x) {
  if (!(x > -9.2233720368547758e18 && x < 9.2233720368547758e18)) return INT64_MIN;
  return (int64_t)x;
}

__device__ __forceinline__ int64_t clip64(int64_t v, int64_t lo, int64_t hi) {
  return v < lo ? lo : (v > hi ? hi : v);
}

struct PrepArgs {
  gsv_grid g;
  gsv_bricks k;
  double cutoff;
  int dense;           // cutoff = inf: every Gaussian in every brick
  int relax_enabled;
  gsv_record32* rec32;
  gsv_record64* rec64;  // optional (f64 engine)
  int32_t* counts;
  int32_t* box;
  // optional change tracking (incremental binning, gsv_bin_incremental): a
  // Gaussian whose pair count or box differs from what counts / box held
  // before this pass is appended as (gid, old box, old count)
  int32_t* chg_count;
  int32_t* chg_gid;
  int32_t* chg_old;      // 4 ints per entry (the old box record)
  int32_t* chg_oldcnt;
  int chg_cap;
};

// Number of bricks of the box (origin blo, extent nb) whose brick id is < b;
// the box's bricks in x-fastest order have increasing ids.  Brick ids fit in
// int32 (validate_grid_bricks).
__device__ __forceinline__ int box_rank(int b, const int64_t blo[3], const int nb[3], int bgx,
                                        int plane) {
  const int z = b / plane, rem = b - z * plane;
  const int y = rem / bgx, x = rem - y * bgx;
  const int dz = z - (int)blo[2], dy = y - (int)blo[1], dx = x - (int)blo[0];
  if (dz < 0) return 0;
  if (dz >= nb[2]) return nb[0] * nb[1] * nb[2];
  int r = nb[0] * nb[1] * dz;
  if (dy < 0) return r;
  if (dy >= nb[1]) return r + nb[0] * nb[1];
  r += nb[0] * dy;
  return r + (dx < 0 ? 0 : (dx >= nb[0] ? nb[0] : dx));
}

// Records, pair count and slab-clipped brick box of Gaussian i from its
// (position, log-scales, unit quaternion, raw amplitude, raw relax).
__device__ __forceinline__ void preprocess_one(int64_t i, const double p[3], const double l[3],
                                               const double q[4], double ra, double rr,
                                               const PrepArgs& pa) {
  double R[9];
  rotation_f64(q, R);
  const double inv_s[3] = {exp(-l[0]), exp(-l[1]), exp(-l[2])};
  double L[9];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) L[3 * a + b] = mul(inv_s[a], R[3 * b + a]);
  const double A = expit_f64(ra);
  const double r = pa.relax_enabled ? expit_f64(rr) : 1.0;

  // Marginal variance Sigma_kk = einsum("nkm,nm->nk", R*R, exp(2 ls)); numpy
  // 2.3 reduces the length-3 axis as (p0 + p2) + p1 (SURVEY.md §0 finding 2).
  const double var[3] = {exp(mul(2.0, l[0])), exp(mul(2.0, l[1])), exp(mul(2.0, l[2]))};
  double half[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double p0 = mul(mul(R[3 * a + 0], R[3 * a + 0]), var[0]);
    const double p1 = mul(mul(R[3 * a + 1], R[3 * a + 1]), var[1]);
    const double p2 = mul(mul(R[3 * a + 2], R[3 * a + 2]), var[2]);
    const double skk = add(add(p0, p2), p1);
    half[a] = pa.dense ? __longlong_as_double(0x7ff0000000000000ULL) : mul(pa.cutoff, sqrt(skk));
  }

  gsv_record32 o;
#pragma unroll
  for (int a = 0; a < 9; ++a) o.l[a] = (float)L[a];
  o.amp = (float)A;
  o.relax = (float)r;
#pragma unroll
  for (int a = 0; a < 3; ++a) o.half[a] = (float)half[a];
  // 1/sigma_max^2 = lambda_min(L^T L): d2 >= |p - mu|^2 / sigma_max^2, the
  // forward's sphere-vs-tile culling bound.
  o.inv_smax2 = (float)exp(-2.0 * fmax(l[0], fmax(l[1], l[2])));
  o._pad = 0.f;
  {
    float4* dst = reinterpret_cast<float4*>(pa.rec32 + i);
    const float4* src = reinterpret_cast<const float4*>(&o);
#pragma unroll
    for (int a = 0; a < 4; ++a) dst[a] = src[a];
  }
  if (pa.rec64) {
    gsv_record64 d;
#pragma unroll
    for (int a = 0; a < 9; ++a) d.l[a] = L[a];
    d.amp = A;
    d.relax = r;
    d._pad = 0.0;
    pa.rec64[i] = d;
  }

  // ---- brick box (raster.py:160-198), clipped to the slab below.
  const gsv_grid& g = pa.g;
  const gsv_bricks& k = pa.k;
  const int dims[3] = {g.nx, g.ny, g.nz};
  const int bd[3] = {k.bdx, k.bdy, k.bdz};
  const int bg[3] = {k.bgx, k.bgy, k.bgz};
  int64_t blo[3], bhi[3];
  bool inside = true;
  if (pa.dense) {
    // cutoff = inf: every Gaussian in every brick (raster.py:166-171).
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      blo[a] = 0;
      bhi[a] = bg[a] - 1;
    }
  } else {
    const double org[3] = {g.ox, g.oy, g.oz};
    const double spc[3] = {g.sx, g.sy, g.sz};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      // a power-of-two spacing divides exactly as a product with its
      // (exact) reciprocal: two f64 multiplies instead of two divisions
      const bool pow2 = (__double_as_longlong(spc[a]) & 0x000FFFFFFFFFFFFFLL) == 0 &&
                        spc[a] >= 0x1p-1000 && spc[a] <= 0x1p1000;
      double glo, ghi;
      if (pow2) {
        const double inv = __drcp_rn(spc[a]);
        glo = mul(sub(sub(p[a], half[a]), org[a]), inv);
        ghi = mul(sub(add(p[a], half[a]), org[a]), inv);
      } else {
        glo = __ddiv_rn(sub(sub(p[a], half[a]), org[a]), spc[a]);
        ghi = __ddiv_rn(sub(add(p[a], half[a]), org[a]), spc[a]);
      }
      int64_t vlo = np_to_int64(ceil(sub(glo, 0.5)));
      int64_t vhi = np_to_int64(floor(add(ghi, 0.5)));
      vlo = clip64(vlo, 0, dims[a] - 1);
      vhi = clip64(vhi, 0, dims[a] - 1);
      inside = inside && (ghi >= -0.5) && (glo <= (double)dims[a] - 0.5);
      blo[a] = vlo / bd[a];
      bhi[a] = vhi / bd[a];
    }
  }
  // Slab clip: the slab owns brick ids [b0, b1).  First the
  // box is clipped to the brick layers the range touches; then, since box
  // order and id order are both lexicographic in (z, y, x), the slab's bricks
  // of the box are the box-order run [k0, k1) with k = #box bricks of id < b.
  const int plane = bg[0] * bg[1];
  int cnt = 0, k0 = 0;
  int nb[3] = {0, 0, 0};
  if (k.b1 > k.b0) {
    const bool whole = k.b0 == 0 && k.b1 == plane * bg[2];
    if (!whole) {
      const int zlo = k.b0 / plane, zhi = (k.b1 - 1) / plane;
      if (blo[2] < zlo) blo[2] = zlo;
      if (bhi[2] > zhi) bhi[2] = zhi;
    }
    if (inside && bhi[2] >= blo[2]) {
#pragma unroll
      for (int a = 0; a < 3; ++a) nb[a] = (int)(bhi[a] - blo[a] + 1);
      if (whole) {
        cnt = nb[0] * nb[1] * nb[2];
      } else {
        k0 = box_rank(k.b0, blo, nb, bg[0], plane);
        cnt = box_rank(k.b1, blo, nb, bg[0], plane) - k0;
      }
    }
  }
  if (cnt == 0) nb[0] = nb[1] = nb[2] = 0;
  int4 bx;
  bx.x = (int)(blo[0] & 0xFFFF) | ((int)(blo[1] & 0xFFFF) << 16);
  bx.y = (int)(blo[2] & 0xFFFF) | ((nb[0] & 0xFFFF) << 16);
  bx.z = (nb[1] & 0xFFFF) | ((nb[2] & 0xFFFF) << 16);
  bx.w = k0;
  if (pa.chg_count != nullptr) {
    const int oc = pa.counts[i];
    const int4 ob = reinterpret_cast<const int4*>(pa.box)[i];
    if (oc != cnt ||
        (cnt > 0 && (ob.x != bx.x || ob.y != bx.y || ob.z != bx.z || ob.w != bx.w))) {
      const int e = atomicAdd(pa.chg_count, 1);
      if (e < pa.chg_cap) {
        pa.chg_gid[e] = (int32_t)i;
        reinterpret_cast<int4*>(pa.chg_old)[e] = ob;
        pa.chg_oldcnt[e] = oc;
      }
    }
  }
  pa.counts[i] = cnt;
  reinterpret_cast<int4*>(pa.box)[i] = bx;
}

}  // namespace gsv
