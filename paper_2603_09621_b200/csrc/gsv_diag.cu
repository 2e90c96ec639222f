// gsv_diag.cu -- roofline instrumentation for bench.py (include/gsv_diag.h).
#include "gsv_common.cuh"
#include "../../include/gsv_diag.h"

namespace gsv {
namespace {

// Live pair-voxel census, same decision logic as forward32_kernel's culling
// and d2 test (f32 with the f64 guard band).
__global__ void __launch_bounds__(256)
count_live_kernel(const double* __restrict__ pos, const gsv_record32* __restrict__ rec,
                  const double* __restrict__ ls, const double* __restrict__ rot,
                  const int64_t* __restrict__ starts, const int32_t* __restrict__ gids,
                  gsv_grid g, gsv_bricks k, float cut2, double cut2d,
                  unsigned long long* counters) {
  const int lb = blockIdx.x;
  const int b = (int)slab_first(k) + lb;
  const BrickXYZ c = brick_xyz(b, k);
  const int x0 = c.bx * k.bdx, y0 = c.by * k.bdy, z0 = c.bz * k.bdz;
  const int ex = min(k.bdx, g.nx - x0), ey = min(k.bdy, g.ny - y0), ez = min(k.bdz, g.nz - z0);
  const double px = g.ox + (double)x0 * g.sx, py = g.oy + (double)y0 * g.sy,
               pz = g.oz + (double)z0 * g.sz;
  unsigned long long live = 0, evals = 0, tiled = 0;
  const int nv = ex * ey * ez;
  // warp tiles of the forward's default layout (8x8x4 bricks, VPL 4): warp w
  // owns y in [4w, 4w + 4); its tile box is the bounding box of its voxels
  const bool tiles8 = k.bdx == 8 && k.bdy == 8 && k.bdz == 4;
  const float isx = (float)(1.0 / g.sx), isy = (float)(1.0 / g.sy), isz = (float)(1.0 / g.sz);
  const float fsx = (float)g.sx, fsy = (float)g.sy, fsz = (float)g.sz;
  for (int64_t j = starts[lb] + threadIdx.x; j < starts[lb + 1]; j += blockDim.x) {
    const int gid = gids[j];
    const gsv_record32 r = rec[gid];
    const double* m = pos + 3 * (int64_t)gid;
    const float c0 = (float)(px - m[0]), c1 = (float)(py - m[1]), c2 = (float)(pz - m[2]);
    evals += nv;
    if (tiles8) {
      // the forward's staging tests: 3-sigma box, then the sphere bound
      const float cxv = -c0 * isx, cyv = -c1 * isy, czv = -c2 * isz;
      const float hxv = fmaf(r.half[0], isx, 1e-3f), hyv = fmaf(r.half[1], isy, 1e-3f),
                  hzv = fmaf(r.half[2], isz, 1e-3f);
      for (int w = 0; w < 2; ++w) {
        const int yl = 4 * w, yh = min(4 * w + 3, ey - 1);
        if (yl > yh) continue;
        const float fxl = 0.f, fxh = (float)(ex - 1), fyl = (float)yl, fyh = (float)yh,
                    fzl = 0.f, fzh = (float)(ez - 1);
        bool hit = cxv + hxv >= fxl && cxv - hxv <= fxh && cyv + hyv >= fyl &&
                   cyv - hyv <= fyh && czv + hzv >= fzl && czv - hzv <= fzh;
        if (hit && !isinf(cut2)) {
          const float ddx = fmaxf(fmaxf(fxl - cxv, cxv - fxh), 0.f) * fsx;
          const float ddy = fmaxf(fmaxf(fyl - cyv, cyv - fyh), 0.f) * fsy;
          const float ddz = fmaxf(fmaxf(fzl - czv, czv - fzh), 0.f) * fsz;
          hit = fmaf(ddx, ddx, fmaf(ddy, ddy, ddz * ddz)) * r.inv_smax2 <= cut2 * 1.0001f + 1e-6f;
        }
        tiled += hit ? 128ull : 0ull;              // 32 lanes x 4 voxels per hit
      }
    }
    for (int z = 0; z < ez; ++z)
      for (int y = 0; y < ey; ++y)
        for (int x = 0; x < ex; ++x) {
          const float dx = fmaf((float)x, (float)g.sx, c0);
          const float dy = fmaf((float)y, (float)g.sy, c1);
          const float dz = fmaf((float)z, (float)g.sz, c2);
          const float v0 = fmaf(r.l[0], dx, fmaf(r.l[1], dy, r.l[2] * dz));
          const float v1 = fmaf(r.l[3], dx, fmaf(r.l[4], dy, r.l[5] * dz));
          const float v2 = fmaf(r.l[6], dx, fmaf(r.l[7], dy, r.l[8] * dz));
          const float d2 = fmaf(v0, v0, fmaf(v1, v1, v2 * v2));
          bool is_live = d2 <= cut2;
          if (fabsf(d2 - cut2) <= 1e-3f * cut2) {
            double L[9];
            whitening_f64(ls + 3 * (int64_t)gid, rot + 4 * (int64_t)gid, L);
            is_live = ref_d2(L, m[0], m[1], m[2], x0 + x, y0 + y, z0 + z, g) <= cut2d;
          }
          live += is_live ? 1ull : 0ull;
        }
  }
  atomicAdd(&counters[0], live);
  atomicAdd(&counters[1], evals);
  atomicAdd(&counters[2], tiled);
}

// Slots the grouped-column forward (forward32c_kernel) evaluates: per
// 32-entry round, the staged hits' footprint rectangles (the forward's exact
// f32 staging tests), groups of consecutive equal rectangles, their columns
// dealt 32 at a time; a chunk runs max(group size) iterations of 32 lanes x
// 4 voxels.  One warp per brick, the forward's own round structure.
__global__ void __launch_bounds__(32)
count_grouped_kernel(const double* __restrict__ pos, const gsv_record32* __restrict__ rec,
                     const int64_t* __restrict__ starts, const int32_t* __restrict__ gids,
                     gsv_grid g, gsv_bricks k, float cut2, unsigned long long* counters) {
  const int lb = blockIdx.x;
  const int b = (int)slab_first(k) + lb;
  const BrickXYZ c = brick_xyz(b, k);
  const int x0 = c.bx * k.bdx, y0 = c.by * k.bdy, z0 = c.bz * k.bdz;
  const int ex = min(k.bdx, g.nx - x0), ey = min(k.bdy, g.ny - y0), ez = min(k.bdz, g.nz - z0);
  const double px = g.ox + (double)x0 * g.sx, py = g.oy + (double)y0 * g.sy,
               pz = g.oz + (double)z0 * g.sz;
  const float isx = (float)(1.0 / g.sx), isy = (float)(1.0 / g.sy), isz = (float)(1.0 / g.sz);
  const float fsx = (float)g.sx, fsy = (float)g.sy, fsz = (float)g.sz;
  const float ftxh = (float)(ex - 1), ftyh = (float)(ey - 1), ftzh = (float)(ez - 1);
  const int lane = threadIdx.x;
  const unsigned full = 0xffffffffu, lt = (1u << lane) - 1u;
  unsigned long long slots = 0;
  for (int64_t base = starts[lb]; base < starts[lb + 1]; base += 32) {
    const int64_t j = base + lane;
    bool hit = false;
    uint32_t rw = 0u;
    if (j < starts[lb + 1]) {
      const int gid = gids[j];
      const gsv_record32 r = rec[gid];
      const double* m = pos + 3 * (int64_t)gid;
      const float mx = (float)(m[0] - px), my = (float)(m[1] - py), mz = (float)(m[2] - pz);
      const float cxv = mx * isx, cyv = my * isy, czv = mz * isz;
      const float hxv = fmaf(r.half[0], isx, 1e-3f), hyv = fmaf(r.half[1], isy, 1e-3f),
                  hzv = fmaf(r.half[2], isz, 1e-3f);
      const float ax0 = fmaxf(ceilf(cxv - hxv), 0.f), ax1 = fminf(floorf(cxv + hxv), ftxh);
      const float ay0 = fmaxf(ceilf(cyv - hyv), 0.f), ay1 = fminf(floorf(cyv + hyv), ftyh);
      const float az0 = fmaxf(ceilf(czv - hzv), 0.f), az1 = fminf(floorf(czv + hzv), ftzh);
      hit = ax0 <= ax1 && ay0 <= ay1 && az0 <= az1;
      if (hit && !isinf(cut2)) {
        const float ddx = fmaxf(fmaxf(ax0 - cxv, cxv - ax1), 0.f) * fsx;
        const float ddy = fmaxf(fmaxf(ay0 - cyv, cyv - ay1), 0.f) * fsy;
        const float ddz = fmaxf(fmaxf(az0 - czv, czv - az1), 0.f) * fsz;
        hit = fmaf(ddx, ddx, fmaf(ddy, ddy, ddz * ddz)) * r.inv_smax2 <= cut2 * 1.0001f + 1e-6f;
      }
      if (hit)
        rw = (uint32_t)ax0 | (uint32_t)ay0 << 3 | (uint32_t)ax1 << 6 | (uint32_t)ay1 << 9;
    }
    // compacted hits in lane order; a group starts where the rectangle changes
    const unsigned hm = __ballot_sync(full, hit);
    const int nh = __popc(hm);
    // the previous hit's rectangle: shuffle from the lane holding hit r-1
    const int r = __popc(hm & lt);
    int src = 0;   // lane of the previous hit
    {
      const unsigned before = hm & lt;
      src = before ? 31 - __clz(before) : lane;
    }
    const uint32_t prev = __shfl_sync(full, rw, src);
    const bool gs = hit && (r == 0 || prev != rw);
    const unsigned gm = __ballot_sync(full, gs);
    // group of each hit lane; sizes and areas per group, in lane order
    const int gi = hit ? __popc(gm & (lt | (1u << lane))) - 1 : -1;
    const int wx = (int)((rw >> 6) & 7u) - (int)(rw & 7u) + 1;
    const int wy = (int)((rw >> 9) & 7u) - (int)((rw >> 3) & 7u) + 1;
    const int ng = __popc(gm);
    int gsize = 0, garea = 0;
    for (int q = 0; q < ng; ++q) {
      const int cnt = __popc(__ballot_sync(full, gi == q));
      const unsigned who = __ballot_sync(full, gs && gi == q);
      const int a = __shfl_sync(full, wx * wy, __ffs(who) - 1);
      if (lane == q) { gsize = cnt; garea = a; }
    }
    int incl = garea;
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(full, incl, o);
      if (lane >= o) incl += n;
    }
    const int gpre = incl - garea;
    const int T = __shfl_sync(full, incl, 31);
    for (int c0 = 0; c0 < T; c0 += 32) {
      const bool meets = lane < ng && gpre < c0 + 32 && gpre + garea > c0;
      const int kmax = __reduce_max_sync(full, meets ? gsize : 0);
      slots += 128ull * (unsigned long long)kmax;
    }
    (void)nh;
  }
  if (lane == 0) atomicAdd(&counters[3], slots);
}

__global__ void __launch_bounds__(256) fma_probe_kernel(int iters, float* out) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-7f + i;
  const float m = 0.999999f, s = 1e-7f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], m, s);
  }
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) t += a[i];
  if (t == 12345.678f) out[0] = t;  // keep the chains live
}

}  // namespace
}  // namespace gsv

using namespace gsv;

extern "C" {

int gsv_diag_count_live(const double* positions, const gsv_record32* rec32,
                        const double* log_scales, const double* rotations,
                        const int64_t* starts, const int32_t* gids, const gsv_grid* grid,
                        const gsv_bricks* bricks, double cutoff_sigma,
                        unsigned long long* counters, void* stream) {
  if (int s = validate_grid_bricks(grid, bricks)) return s;
  const int64_t nb = slab_bricks(*bricks);
  if (nb == 0) return GSV_OK;
  const double cut2d = cutoff_sigma * cutoff_sigma;
  count_live_kernel<<<(unsigned)nb, 256, 0, as_stream(stream)>>>(
      positions, rec32, log_scales, rotations, starts, gids, *grid, *bricks, (float)cut2d,
      cut2d, counters);
  GSV_CHECK_LAUNCH("count_live_kernel");
  if (bricks->bdx == 8 && bricks->bdy == 8 && bricks->bdz == 4) {
    count_grouped_kernel<<<(unsigned)nb, 32, 0, as_stream(stream)>>>(
        positions, rec32, starts, gids, *grid, *bricks, (float)cut2d, counters);
    GSV_CHECK_LAUNCH("count_grouped_kernel");
  }
  return GSV_OK;
}

int gsv_diag_fma_probe(int blocks, int iters, float* out, void* stream) {
  fma_probe_kernel<<<blocks, 256, 0, as_stream(stream)>>>(iters, out);
  GSV_CHECK_LAUNCH("fma_probe_kernel");
  return GSV_OK;
}

}  // extern "C"
