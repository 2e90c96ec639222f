// gsv_render.cu -- forward render and backward pair pass, one CTA per brick.
//
// forward  (raster.py:240-293): each CTA owns one brick's voxels, walks the
//          brick's Gaussian list in chunks staged in shared memory, and
//          accumulates S = sum A w, W = sum w in registers in list order (no
//          depth sort, no atomics: bit-reproducible).  The epilogue
//          normalises I = S/W and optionally fuses the L1/L2 loss
//          (optimize.py:91-103), emitting the backward's per-voxel inputs.
// backward (raster.py:322-409): one thread per (brick, Gaussian) pair walks
//          the pair's exact 3-sigma sub-box of the brick and keeps the 11
//          partial sums in registers; one 48-byte store per pair at the
//          pair's gid-major emission slot, so the merge is a contiguous
//          segmented reduction in ascending brick order (raster.py:512-522).
//
// f32 engine: per-pair math in fp32 with the voxel offset taken relative to
// the brick origin (computed in f64), so |delta| stays small; the truncation
// test d2 <= cutoff^2 is re-decided in f64 with the reference's exact
// operation order inside a guard band around the cutoff (SURVEY.md §7 hard
// part 2), so both engines agree on which pairs are live.
// f64 engine: the reference arithmetic in double (precision="f64").
#include <cfloat>
#include <cstdlib>
#include <type_traits>

#include "gsv_common.cuh"

namespace gsv {
namespace {

constexpr int kBwdThreads = 256;
#ifndef GSV_BWDM_THREADS
#define GSV_BWDM_THREADS 256     // masked backward CTA size (measurement builds may change it)
#endif
#ifndef GSV_BWDM_WARPS
#define GSV_BWDM_WARPS 24        // warps per SM it is built for
#endif
constexpr int kBwdMThreads = GSV_BWDM_THREADS;
constexpr int kBwdSmemVoxels = 2048; // brick voxels staged in smem by the backward
// f32 truncation guard band.  Each v component is u + x e_x + y e_y + z e_z
// with |terms| <= umax, so |dv| <= ~8 ulp(umax) ~ 4.8e-7 umax (f32 rounding of
// p_b0 - mu, of L, of u and of three FMAs); near the cutoff
// |d(d2)| <= 2 sqrt(3) cutoff |dv| + 3 ulp(d2) ~ 1.7e-6 cutoff umax + 2e-7 d2.
// The band is ~6x that; inside it the f64 reference decision is recomputed.
constexpr float kGuardRel = 2e-6f;   // x cutoff^2
constexpr float kGuardMag = 1e-5f;   // x umax x cutoff
constexpr unsigned kFull = 0xffffffffu;

// Shared-memory record of one staged pair (f32 forward), 64 bytes: four
// broadcast LDS.128 per (pair, warp-tile) evaluation.  The exponent
// q = -(1/2) log2(e) d2 + log2(r) is a quadratic in the lane's voxel offset
// (X, Y, Z) from the warp tile's centre, so w = A-free weight = 2^q needs 9
// FMAs (+4 for the second voxel) and one EX2 per voxel.
struct __align__(16) Pair32 {
  float4 a;  // k0 kx ky kz
  float4 b;  // kxx kyy kzz kxy
  float4 c;  // kxz kyz amp t_live    q >= t_live: live for sure
  float4 d;  // t_band gid - -        t_band <= q < t_live: re-decide in f64
};

struct BrickGeom {
  int x0, y0, z0;     // first voxel (global)
  int ex, ey, ez;     // voxels of this brick inside the grid
  double px, py, pz;  // world centre of the first voxel
};

__device__ __forceinline__ BrickGeom brick_geom(int b, const gsv_grid& g,
                                                const gsv_bricks& k) {
  const BrickXYZ c = brick_xyz(b, k);
  BrickGeom r;
  r.x0 = c.bx * k.bdx;
  r.y0 = c.by * k.bdy;
  r.z0 = c.bz * k.bdz;
  r.ex = min(k.bdx, g.nx - r.x0);
  r.ey = min(k.bdy, g.ny - r.y0);
  r.ez = min(k.bdz, g.nz - r.z0);
  r.px = g.ox + (double)r.x0 * g.sx;
  r.py = g.oy + (double)r.y0 * g.sy;
  r.pz = g.oz + (double)r.z0 * g.sz;
  return r;
}

// Brick-local voxel range [lo, hi] that can hold live voxels of a Gaussian
// with world centre offset c = mu - p_b0 and half extent h (3-sigma AABB,
// widened by 1e-3 voxel so rounding can never drop a live voxel).
__device__ __forceinline__ void sub_range(double c, double h, double s, int n,
                                          int& lo, int& hi) {
  const double ctr = c / s, hv = h / s;
  double a = ceil(ctr - hv - 1e-3), b = floor(ctr + hv + 1e-3);
  a = fmax(a, 0.0);
  b = fmin(b, (double)(n - 1));
  if (!(a <= b)) {
    lo = 1;
    hi = 0;
    return;
  }
  lo = (int)a;
  hi = (int)b;
}


// Exact f64 truncation decision of one (Gaussian, voxel) -- the rare
// guard-band path -- with the f64 whitening factor from rec64 when the caller
// built it (f64 engine), else recomputed from the field (f32 engine).
struct ExactSrc {
  const double* pos;
  const double* ls;
  const double* rot;
  const gsv_record64* rec64;
};

__device__ __noinline__ bool exact_live(int gid, int gx, int gy, int gz, const ExactSrc& x,
                                        const gsv_grid& g, double cutoff2) {
  double Lw[9];
  const double* L;
  if (x.rec64 != nullptr) {
    L = x.rec64[gid].l;
  } else {
    whitening_f64(x.ls + 3 * (int64_t)gid, x.rot + 4 * (int64_t)gid, Lw);
    L = Lw;
  }
  const double* m = x.pos + 3 * (int64_t)gid;
  return ref_d2(L, m[0], m[1], m[2], gx, gy, gz, g) <= cutoff2;
}

// One target voxel as double: the fused loss subtracts in f64 like
// loss_and_grad (optimize.py:97), from a float32 or float64 target.
__device__ __forceinline__ double target_value(const void* t, int f64, int64_t lin) {
  return f64 ? __ldg(static_cast<const double*>(t) + lin)
             : (double)__ldg(static_cast<const float*>(t) + lin);
}

// Deterministic block reduction of one double (fixed tree).
template <int THREADS>
__device__ double block_sum(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < THREADS / 32; ++w) t += sh[w];
  return t;  // valid in thread 0
}

// Live-mask layouts: VPL voxels per lane, one warp tile of 32 lanes; the
// units of a brick (column heads) must fit one CTA pass.
__host__ __device__ inline int64_t mask_units(const gsv_bricks& k, int vpl) {
  return (int64_t)k.bdx * k.bdy * ((k.bdz + vpl - 1) / vpl);
}
inline int mask_vpl_auto(const gsv_bricks& k) {
  return (k.bdz % 4 == 0 && mask_units(k, 4) <= 64) ? 4 : 2;
}
// (live masks: mask_units == 128 / vpl * 2, i.e. exactly 4 planes of words)

// --------------------------------------------------------------- forward f32
// Thread -> voxel ownership.  A "unit" is a column pair of voxels (x, y, z0)
// and (x, y, z0+1).  When the brick dims are multiples of 4 the 32 units of a
// warp form one compact 4x4x4 voxel tile, so a Gaussian's 3-sigma box touches
// as few warp tiles as possible; otherwise units are enumerated x-fastest.
__device__ __forceinline__ void unit_voxel(int u, const gsv_bricks& k, bool tiled, int& x,
                                           int& y, int& z0) {
  if (tiled) {
    const int t = u >> 5, l = u & 31;
    const int tgx = k.bdx >> 2, tgy = k.bdy >> 2;
    x = ((t % tgx) << 2) + (l & 3);
    y = (((t / tgx) % tgy) << 2) + ((l >> 2) & 3);
    z0 = ((t / (tgx * tgy)) << 2) + ((l >> 4) << 1);
  } else {
    x = u % k.bdx;
    y = (u / k.bdx) % k.bdy;
    z0 = (u / (k.bdx * k.bdy)) << 1;
  }
}

#ifndef GSV_FWD_PREFETCH
#define GSV_FWD_PREFETCH 1      // LR forward: 0 off, 1 L1 (-0.5%), 2 L2 (measurement builds)
#endif
__device__ __forceinline__ void prefetch_line(const void* p) {
#if GSV_FWD_PREFETCH == 1
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
#elif GSV_FWD_PREFETCH == 2
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
#endif
}

__device__ __forceinline__ float ex2_approx(float q) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(q));
  return r;
}


// One CTA per brick.  Each lane owns a z-column of VPL voxels; a warp's 32
// lanes form one voxel tile (VPL = 2: 4x4x4 tiles, 4 warps per 8x8x4 brick --
// small Gaussians, the LR train grid; VPL = 4: 8x4x4 tiles, 2 warps per brick
// -- Gaussians spanning several bricks, HR renders).  Warps walk the brick's
// list independently -- no CTA barrier in the pair loop: per round of 32 list
// entries every lane stages one pair, tests its 3-sigma box against the
// warp's tile, and the hits are compacted (ballot rank) into warp-private smem
// records, then evaluated in list order (deterministic, no atomics).  The
// exponent q = -(1/2) log2(e) d2 + log2(r) is a quadratic in the lane's voxel
// offset from the tile centre: 9 FMAs for the first voxel of the column, 2
// FADDs (second differences) for each further one, one EX2 per voxel.
// Staging is repeated per warp (L1-resident loads): cheaper than the barrier
// stalls of shared staging, where every warp waits for the slowest tile.
template <int VPL>
__device__ __forceinline__ void unit_voxel_v(int u, const gsv_bricks& k, int& x, int& y,
                                             int& z0) {
  const bool tiled = VPL == 2 && ((k.bdx | k.bdy | k.bdz) & 3) == 0;
  if (tiled) {
    const int t = u >> 5, l = u & 31;
    const int tgx = k.bdx >> 2, tgy = k.bdy >> 2;
    x = ((t % tgx) << 2) + (l & 3);
    y = (((t / tgx) % tgy) << 2) + ((l >> 2) & 3);
    z0 = ((t / (tgx * tgy)) << 2) + ((l >> 4) << 1);
  } else {
    x = u % k.bdx;
    y = (u / k.bdx) % k.bdy;
    z0 = (u / (k.bdx * k.bdy)) * VPL;
  }
}

// One hit's VPL live words into its shared slot (16-byte store at VPL 4).
template <int VPL>
__device__ __forceinline__ void store_mask_words(uint2* dst, const unsigned* w) {
  if constexpr (VPL == 4) {
    *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
  } else {
#pragma unroll
    for (int kk = 0; kk < VPL / 2; ++kk) dst[kk] = make_uint2(w[2 * kk], w[2 * kk + 1]);
  }
}

#ifndef GSV_FWD_OCC
#define GSV_FWD_OCC 640
#endif
// SPLIT: one 32-thread CTA per warp tile of a brick with exactly two tiles
// (VPL 4, e.g. 8x8x4): no CTA waits for its slower tile, the scheduler refills
// the SM as soon as a tile is done.  The brick's loss partial then gets two
// atomic adds onto a zeroed slot -- order-independent, so still deterministic.
template <int VPL, int THREADS, bool MASKS, bool SPLIT = false>
__global__ void __launch_bounds__(THREADS, GSV_FWD_OCC / THREADS)
forward32_kernel(const double* __restrict__ pos, const __grid_constant__ ExactSrc xsrc,
                 const gsv_record32* __restrict__ rec,
                 const int64_t* __restrict__ starts, const int32_t* __restrict__ gids,
                 const __grid_constant__ gsv_grid g, gsv_bricks k, float cut2, double cut2d,
                 double eps_w,
                 float* __restrict__ S, float* __restrict__ W, float* __restrict__ I,
                 const void* __restrict__ target, int target_f64, int loss_kind, double vox_count,
                 float2* __restrict__ ab, double* __restrict__ loss_part,
                 uint2* __restrict__ live_masks) {
  __shared__ Pair32 sp[THREADS];       // 32 slots per warp
  // live bits of this round's hits: per warp and hit VPL words (VPL/2 uint2)
  __shared__ __align__(16) uint2 smask[MASKS ? THREADS * VPL / 2 : 1];
  __shared__ __align__(16) uint2 sxmask[MASKS ? THREADS * VPL / 2 : 1];   // guard-band additions
  __shared__ double red[THREADS / 32];
  static_assert(!SPLIT || THREADS == 32, "split tiles run one warp per CTA");
  const int lb = SPLIT ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;   // slab-local brick
  const int b = (int)slab_first(k) + lb;                   // global brick id
  const BrickGeom bg = brick_geom(b, g, k);
  const int64_t lbeg = starts[lb], lend = starts[lb + 1];
  // tid / warp: the thread's place in the brick's tiling; swarp: its warp's
  // slot in this CTA's shared memory
  const int warp = SPLIT ? (int)(blockIdx.x & 1) : (int)(threadIdx.x >> 5);
  const int tid = (int)threadIdx.x + (SPLIT ? (warp << 5) : 0), lane = threadIdx.x & 31;
  const int swarp = SPLIT ? 0 : warp;
  Pair32* wsp = sp + (swarp << 5);
  const int units = k.bdx * k.bdy * ((k.bdz + VPL - 1) / VPL);
  const float fsx = (float)g.sx, fsy = (float)g.sy, fsz = (float)g.sz;
  const float isx = (float)(1.0 / g.sx), isy = (float)(1.0 / g.sy), isz = (float)(1.0 / g.sz);
  // masks: VPL 2, one pass over the brick's voxel units (4 warp tiles)
  // masks (host-checked: units <= THREADS): per pair VPL words per warp,
  // planes [warp * VPL/2 + k][pair] of uint2 {word 2k, word 2k+1}
  constexpr bool want_masks = MASKS;
  double lsum = 0.0;

  for (int ubase = 0; ubase < units; ubase += SPLIT ? units : THREADS) {
    const int u = ubase + tid;
    int lx = 0, ly = 0, lz = 0;
    if (u < units) unit_voxel_v<VPL>(u, k, lx, ly, lz);
    bool own[VPL];
    int zmax = -(1 << 20);
#pragma unroll
    for (int h = 0; h < VPL; ++h) {
      own[h] = u < units && lx < bg.ex && ly < bg.ey && lz + h < bg.ez && lz + h < k.bdz;
      if (own[h]) zmax = lz + h;
    }
    // This warp's tile box (brick-local voxel coords) from its owned voxels.
    int txl = own[0] ? lx : 1 << 20, txh = own[0] ? lx : -(1 << 20);
    int tyl = own[0] ? ly : 1 << 20, tyh = own[0] ? ly : -(1 << 20);
    int tzl = own[0] ? lz : 1 << 20, tzh = zmax;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      txl = min(txl, __shfl_xor_sync(kFull, txl, o));
      txh = max(txh, __shfl_xor_sync(kFull, txh, o));
      tyl = min(tyl, __shfl_xor_sync(kFull, tyl, o));
      tyh = max(tyh, __shfl_xor_sync(kFull, tyh, o));
      tzl = min(tzl, __shfl_xor_sync(kFull, tzl, o));
      tzh = max(tzh, __shfl_xor_sync(kFull, tzh, o));
    }
    const float ftxl = (float)txl, ftxh = (float)txh, ftyl = (float)tyl, ftyh = (float)tyh,
                ftzl = (float)tzl, ftzh = (float)tzh;
    // Tile centre and this lane's voxel offsets from it (exact halves in f32).
    const float ctx = 0.5f * (ftxl + ftxh), cty = 0.5f * (ftyl + ftyh), ctz = 0.5f * (ftzl + ftzh);
    const float ext_x = fmaxf(0.5f * (ftxh - ftxl), 0.f), ext_y = fmaxf(0.5f * (ftyh - ftyl), 0.f),
                ext_z = fmaxf(0.5f * (ftzh - ftzl), 0.f);
    // A voxel the lane does not own gets NaN offsets: every q is NaN, so it is
    // never live and never enters a mask (no per-hit ownership predicates).
    const float qnan = __int_as_float(0x7fc00000);
    const float mX = own[0] ? (float)lx - ctx : qnan, mY = (float)ly - cty, mZ = (float)lz - ctz;
    const float mZ1 = (VPL == 2 && !own[1]) ? qnan : mZ + 1.f;
    const int gx = bg.x0 + lx, gy = bg.y0 + ly, gz = bg.z0 + lz;
    unsigned ownb[VPL];
#pragma unroll
    for (int h = 0; h < VPL; ++h) ownb[h] = __ballot_sync(kFull, own[h]);
    float accS[VPL], accW[VPL];
#pragma unroll
    for (int h = 0; h < VPL; ++h) accS[h] = accW[h] = 0.f;

    int gid_next = (lbeg + lane < lend) ? __ldg(gids + lbeg + lane) : -1;
    int gid_next2 = (lbeg + 32 + lane < lend) ? __ldg(gids + lbeg + 32 + lane) : -1;
    for (int64_t base = lbeg; base < lend; base += 32) {
      const int gid = gid_next;
      gid_next = gid_next2;
      gid_next2 = (base + 64 + lane < lend) ? __ldg(gids + base + 64 + lane) : -1;
#if GSV_FWD_PREFETCH
      // next round's record and position lines, in flight during this round
      if (gid_next >= 0) {
        prefetch_line(rec + gid_next);
        prefetch_line(pos + 3 * (int64_t)gid_next);
      }
#endif
      bool hit = false;
      Pair32 p;
      if (gid >= 0) {
        const float4* r4 = reinterpret_cast<const float4*>(rec + gid);
        const float4 q0 = __ldg(r4), q1 = __ldg(r4 + 1), q2 = __ldg(r4 + 2), q3 = __ldg(r4 + 3);
        const double* m = pos + 3 * (int64_t)gid;
        // mu - p_b0 in f64, then f32 (small: |mu - p_b0| ~ brick size + 3 sigma)
        const float mx = (float)(__ldg(m) - bg.px), my = (float)(__ldg(m + 1) - bg.py),
                    mz = (float)(__ldg(m + 2) - bg.pz);
        // 3-sigma box (voxel units, brick-local) vs this warp's tile, widened
        // by 1e-3 voxel so rounding can never drop a live voxel.
        const float cxv = mx * isx, cyv = my * isy, czv = mz * isz;
        const float hxv = fmaf(q2.w, isx, 1e-3f), hyv = fmaf(q3.x, isy, 1e-3f),
                    hzv = fmaf(q3.y, isz, 1e-3f);
        hit = cxv + hxv >= ftxl && cxv - hxv <= ftxh && cyv + hyv >= ftyl &&
              cyv - hyv <= ftyh && czv + hzv >= ftzl && czv - hzv <= ftzh;
        if (hit && !isinf(cut2)) {
          // Sphere-vs-tile: d2 >= |p - mu|^2 / sigma_max^2 over the tile's
          // voxel-centre box (world units); reject when even that bound
          // exceeds cutoff^2 (with a 1e-4 relative margin for rounding).
          const float ddx = fmaxf(fmaxf(ftxl - cxv, cxv - ftxh), 0.f) * fsx;
          const float ddy = fmaxf(fmaxf(ftyl - cyv, cyv - ftyh), 0.f) * fsy;
          const float ddz = fmaxf(fmaxf(ftzl - czv, czv - ftzh), 0.f) * fsz;
          const float dist2 = fmaf(ddx, ddx, fmaf(ddy, ddy, ddz * ddz));
          hit = dist2 * q3.z <= cut2 * 1.0001f + 1e-6f;
        }
        if (hit) {
          const float L[9] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w, q2.x};
          float u3[3], e[3][3], umax = 0.f;
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            u3[a] = -fmaf(L[3 * a + 0], mx, fmaf(L[3 * a + 1], my, L[3 * a + 2] * mz));
            e[0][a] = L[3 * a + 0] * fsx;
            e[1][a] = L[3 * a + 1] * fsy;
            e[2][a] = L[3 * a + 2] * fsz;
            umax = fmaxf(umax, fabsf(u3[a]) + fabsf(e[0][a]) * k.bdx +
                                   fabsf(e[1][a]) * k.bdy + fabsf(e[2][a]) * k.bdz);
          }
          // v at the tile centre, then the quadratic's coefficients (scaled by s)
          float uc[3];
#pragma unroll
          for (int a = 0; a < 3; ++a)
            uc[a] = fmaf(ctz, e[2][a], fmaf(cty, e[1][a], fmaf(ctx, e[0][a], u3[a])));
          const float sc = -0.72134752044448170f;   // -(1/2) log2(e)
          const float lr2 = __log2f(q2.z);
          const float d00 = fmaf(uc[0], uc[0], fmaf(uc[1], uc[1], uc[2] * uc[2]));
          p.a.x = fmaf(sc, d00, lr2);
          p.a.y = 2.f * sc * fmaf(uc[0], e[0][0], fmaf(uc[1], e[0][1], uc[2] * e[0][2]));
          p.a.z = 2.f * sc * fmaf(uc[0], e[1][0], fmaf(uc[1], e[1][1], uc[2] * e[1][2]));
          p.a.w = 2.f * sc * fmaf(uc[0], e[2][0], fmaf(uc[1], e[2][1], uc[2] * e[2][2]));
          p.b.x = sc * fmaf(e[0][0], e[0][0], fmaf(e[0][1], e[0][1], e[0][2] * e[0][2]));
          p.b.y = sc * fmaf(e[1][0], e[1][0], fmaf(e[1][1], e[1][1], e[1][2] * e[1][2]));
          p.b.z = sc * fmaf(e[2][0], e[2][0], fmaf(e[2][1], e[2][1], e[2][2] * e[2][2]));
          p.b.w = 2.f * sc * fmaf(e[0][0], e[1][0], fmaf(e[0][1], e[1][1], e[0][2] * e[1][2]));
          p.c.x = 2.f * sc * fmaf(e[0][0], e[2][0], fmaf(e[0][1], e[2][1], e[0][2] * e[2][2]));
          p.c.y = 2.f * sc * fmaf(e[1][0], e[2][0], fmaf(e[1][1], e[2][1], e[1][2] * e[2][2]));
          p.c.z = q2.y;
          // Guard band in q units: the direct-v bound (kGuard*, scaled by |s|)
          // plus the rounding of the expanded quadratic and its VPL-1 finite
          // differences (~7e-7 of the sum of its term magnitudes), x3.5.
          const float qmag = fabsf(p.a.x) + ext_x * fabsf(p.a.y) + ext_y * fabsf(p.a.z) +
                             ext_z * fabsf(p.a.w) + ext_x * ext_x * fabsf(p.b.x) +
                             ext_y * ext_y * fabsf(p.b.y) + ext_z * ext_z * fabsf(p.b.z) +
                             ext_x * ext_y * fabsf(p.b.w) + ext_x * ext_z * fabsf(p.c.x) +
                             ext_y * ext_z * fabsf(p.c.y);
          const float guard = isinf(cut2) ? 0.f
                              : 0.72134752f * (kGuardRel * cut2 + kGuardMag * umax * sqrtf(cut2)) +
                                    2.5e-6f * qmag;
          const float qcut = isinf(cut2) ? -INFINITY : fmaf(sc, cut2, lr2);
          p.c.w = qcut + guard;          // live for sure above
          p.d = make_float4(qcut - guard, __int_as_float(gid), __int_as_float(lane), 0.f);
        }
      }
      // Compact this round's hits into consecutive slots (ballot rank), so the
      // evaluation loop below is a plain counter over broadcast smem records.
      const unsigned ball = __ballot_sync(kFull, hit);
      const int rank = __popc(ball & ((1u << lane) - 1u));
      if (hit) wsp[rank] = p;
      __syncwarp();
      const int nh = __popc(ball);
      if (want_masks) {                 // guard-band live bits of this round's hits
#pragma unroll
        for (int kk = 0; kk < VPL / 2; ++kk)
          sxmask[((swarp << 5) + lane) * (VPL / 2) + kk] = make_uint2(0u, 0u);
        __syncwarp();
      }
      for (int jj = 0; jj < nh; ++jj) {
        const float4 pa = wsp[jj].a, pb = wsp[jj].b, pc = wsp[jj].c;
        const float2 pd = *reinterpret_cast<const float2*>(&wsp[jj].d);   // qlo, gid
        // q(X,Y,Z) of the column's first voxel in nested form -- only the
        // lane's three offsets stay live across hits -- then differences in z
        float q[VPL];
        const float t1 = fmaf(pb.x, mX, fmaf(pb.w, mY, fmaf(pc.x, mZ, pa.y)));
        const float t2 = fmaf(pb.y, mY, fmaf(pc.y, mZ, pa.z));
        const float t3 = fmaf(pb.z, mZ, pa.w);
        q[0] = fmaf(mX, t1, fmaf(mY, t2, fmaf(mZ, t3, pa.x)));
        float dq = fmaf(pc.y, mY, fmaf(pc.x, mX, fmaf(pb.z, mZ1, t3)));
        const float d2q = 2.f * pb.z;
#pragma unroll
        for (int h = 1; h < VPL; ++h) {
          q[h] = q[h - 1] + dq;
          dq += d2q;
        }
        // Live for sure: q >= qhi -- accumulated first, branch-free.  Then
        // the guard band [qlo, qhi): the exact f64 decision (the reference's
        // truncation test; rare, warp-voted) adds those voxels' contributions
        // and records their mask bits.  A voxel is live or in the band, never
        // both, so its per-voxel order of additions is the list order either
        // way.  The band compare reuses the live predicate (NaN -- a voxel
        // the lane does not own -- is neither live nor in the band).
        bool live[VPL];
#pragma unroll
        for (int h = 0; h < VPL; ++h) {
          live[h] = q[h] >= pc.w;
          const float w = ex2_approx(q[h]);
          if (live[h]) {
            accS[h] = fmaf(pc.z, w, accS[h]);
            accW[h] += w;
          }
        }
        if (want_masks) {
          unsigned mw[VPL];
#pragma unroll
          for (int h = 0; h < VPL; ++h) mw[h] = __ballot_sync(kFull, live[h]);
          // warp-uniform values: every lane stores the same words (no predicate)
          store_mask_words<VPL>(smask + ((swarp << 5) + jj) * (VPL / 2), mw);
        }
        bool inband[VPL], band = false;
#pragma unroll
        for (int h = 0; h < VPL; ++h) {
          inband[h] = !live[h] && q[h] >= pd.x;
          band |= inband[h];
        }
        if (__any_sync(kFull, band)) {
          const int gidj = __float_as_int(pd.y);
          bool xl[VPL];
#pragma unroll
          for (int h = 0; h < VPL; ++h) {
            xl[h] = inband[h] && exact_live(gidj, gx, gy, gz + h, xsrc, g, cut2d);
            if (xl[h]) {
              const float w = ex2_approx(q[h]);
              accS[h] = fmaf(pc.z, w, accS[h]);
              accW[h] += w;
            }
          }
          if (want_masks) {
            unsigned xw[VPL];
#pragma unroll
            for (int h = 0; h < VPL; ++h) xw[h] = __ballot_sync(kFull, xl[h]);
            store_mask_words<VPL>(sxmask + ((swarp << 5) + jj) * (VPL / 2), xw);
          }
        }
      }
      // live-voxel masks for the backward, plane [warp][pair]: one coalesced
      // 256-byte store per warp and round (pairs missing the tile get zeros)
      if (want_masks) {
        __syncwarp();
        uint2 mm[VPL / 2];
#pragma unroll
        for (int kk = 0; kk < VPL / 2; ++kk) mm[kk] = make_uint2(0u, 0u);
        if (hit) {
          const int slot = ((swarp << 5) + rank) * (VPL / 2);
          if constexpr (VPL == 4) {
            const uint4 a = *reinterpret_cast<const uint4*>(smask + slot);
            const uint4 x = *reinterpret_cast<const uint4*>(sxmask + slot);
            mm[0] = make_uint2(a.x | x.x, a.y | x.y);
            mm[1] = make_uint2(a.z | x.z, a.w | x.w);
          } else {
#pragma unroll
            for (int kk = 0; kk < VPL / 2; ++kk) {
              const uint2 a = smask[slot + kk], x = sxmask[slot + kk];
              mm[kk] = make_uint2(a.x | x.x, a.y | x.y);
            }
          }
        }
#pragma unroll
        for (int kk = 0; kk < VPL / 2; ++kk) {
          mm[kk].x &= ownb[2 * kk];      // voxels outside the grid never enter a mask
          mm[kk].y &= ownb[2 * kk + 1];
        }
        // pair-major: the pair's 4 planes are 32 contiguous bytes
        if (gid >= 0) {
          uint2* dst = live_masks + 4 * (base + lane) + warp * (VPL / 2);
          if constexpr (VPL == 4) {
            *reinterpret_cast<uint4*>(dst) = make_uint4(mm[0].x, mm[0].y, mm[1].x, mm[1].y);
          } else {
#pragma unroll
            for (int kk = 0; kk < VPL / 2; ++kk) dst[kk] = mm[kk];
          }
        }
      }
      __syncwarp();
    }
    // Epilogue: normalise, store, fused loss (optimize.py:91-103).
#pragma unroll
    for (int h = 0; h < VPL; ++h) {
      if (!own[h]) continue;
      const int64_t lin = (int64_t)gx + (int64_t)g.nx * (gy + (int64_t)g.ny * (gz + h));
      const bool cov = (double)accW[h] >= eps_w;
      const float iv = cov ? __fdiv_rn(accS[h], accW[h]) : 0.f;
      S[lin] = accS[h];
      W[lin] = accW[h];
      I[lin] = iv;
      if (target) {
        const double d = (double)iv - target_value(target, target_f64, lin);
        double dl;
        if (loss_kind == 0) {
          lsum += fabs(d);
          dl = (d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0)) / vox_count;
        } else {
          lsum += d * d;
          dl = 2.0 * d / vox_count;
        }
        const float alpha = (cov && dl != 0.0) ? (float)(dl / (double)accW[h]) : 0.f;
        ab[lin] = make_float2(alpha, iv);
      }
    }
  }
  if (target) {
    if (SPLIT) {
      double t = lsum;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(kFull, t, o);
      if (lane == 0) atomicAdd(loss_part + lb, t);   // 2 adds onto 0: order-independent
    } else {
      const double t = block_sum<THREADS>(lsum, red);
      if (threadIdx.x == 0) loss_part[lb] = t;
    }
  }
}

// Shared-memory accesses by 32-bit shared address: the base is formed once,
// outside the loops (plain array indexing let ptxas rematerialise the
// generic->shared window base, an S2UR with its latency, in every iteration).
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(p);
  asm volatile("" : "+r"(a));   // opaque: keep it in a register
  return a;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ float2 lds_f2(uint32_t a) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ uint4 lds_u4(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_u4(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
// ------------------------------------------- forward f32, one warp per brick
// Renders with large Gaussians (pairs >= 8 N: nearly every pair hits both
// 8x4x4 tiles of a brick): one 32-thread CTA per 8x8x4 brick, lane l owns
// the columns (x, y) = (l & 7, l >> 3) and (x, y + 4), all 4 z.  A pair is
// staged and its quadratic built once per brick; column B's start value and
// z-step follow from column A's in 5 FMAs.  No live masks (renders only).
// Render form (no live masks): kept as its own function -- sharing the
// masked template measurably changed the render kernel's scheduling (+1.5%).
// hits_a: the 32-bit shared address of the compacted hits (an opaque base,
// formed once: list B's `wsp + 32` otherwise made ptxas re-derive the shared
// window base with an S2UR in every iteration)
__device__ __forceinline__ void eval_column_hits_plain(uint32_t hits_a, int nh,
                                                       float mX, float mY, float mZ, float mZ1,
                                                       int gx, int gy, int gz,
                                                       const ExactSrc& xsrc, const gsv_grid& g,
                                                       double cut2d, float* aS, float* aW) {
  constexpr int Z = 4;
  for (int jj = 0; jj < nh; ++jj) {
    const uint32_t ja = hits_a + (uint32_t)jj * (uint32_t)sizeof(Pair32);
    const float4 pa = lds_f4(ja), pb = lds_f4(ja + 16), pc = lds_f4(ja + 32);
    const float2 pd = lds_f2(ja + 48);   // qlo, gid
    float q[Z];
    const float t1 = fmaf(pb.x, mX, fmaf(pb.w, mY, fmaf(pc.x, mZ, pa.y)));
    const float t2 = fmaf(pb.y, mY, fmaf(pc.y, mZ, pa.z));
    const float t3 = fmaf(pb.z, mZ, pa.w);
    q[0] = fmaf(mX, t1, fmaf(mY, t2, fmaf(mZ, t3, pa.x)));
    float dq = fmaf(pc.y, mY, fmaf(pc.x, mX, fmaf(pb.z, mZ1, t3)));
    const float d2q = 2.f * pb.z;
#pragma unroll
    for (int h = 1; h < Z; ++h) {
      q[h] = q[h - 1] + dq;
      dq += d2q;
    }
    bool live[Z], band = false;
#pragma unroll
    for (int h = 0; h < Z; ++h) {
      live[h] = q[h] >= pc.w;
      const float w = ex2_approx(q[h]);
      if (live[h]) {
        aS[h] = fmaf(pc.z, w, aS[h]);
        aW[h] += w;
      }
    }
#pragma unroll
    for (int h = 0; h < Z; ++h) band |= !live[h] && q[h] >= pd.x;
    if (__any_sync(kFull, band)) {
      const int gidj = __float_as_int(pd.y);
#pragma unroll
      for (int h = 0; h < Z; ++h)
        if (!live[h] && q[h] >= pd.x && exact_live(gidj, gx, gy, gz + h, xsrc, g, cut2d)) {
          const float w = ex2_approx(q[h]);
          aS[h] = fmaf(pc.z, w, aS[h]);
          aW[h] += w;
        }
    }
  }
}

// Evaluate one column (4 voxels in z) of a lane against a compacted hit list
// (the two-list whole-brick forward): q in nested form at the column's first
// voxel, then second differences; live accumulation, then the guard band.
template <bool MASKS>
__device__ __forceinline__ void eval_column_hits(uint32_t hits_a, int nh,
                                                 float mX, float mY, float mZ, float mZ1,
                                                 int gx, int gy, int gz, const ExactSrc& xsrc,
                                                 const gsv_grid& g, double cut2d,
                                                 float* aS, float* aW, uint32_t smw_a) {
  constexpr int Z = 4;
  for (int jj = 0; jj < nh; ++jj) {
    const uint32_t ja = hits_a + (uint32_t)jj * (uint32_t)sizeof(Pair32);
    const float4 pa = lds_f4(ja), pb = lds_f4(ja + 16), pc = lds_f4(ja + 32);
    const float2 pd = lds_f2(ja + 48);   // qlo, gid
    float q[Z];
    const float t1 = fmaf(pb.x, mX, fmaf(pb.w, mY, fmaf(pc.x, mZ, pa.y)));
    const float t2 = fmaf(pb.y, mY, fmaf(pc.y, mZ, pa.z));
    const float t3 = fmaf(pb.z, mZ, pa.w);
    q[0] = fmaf(mX, t1, fmaf(mY, t2, fmaf(mZ, t3, pa.x)));
    float dq = fmaf(pc.y, mY, fmaf(pc.x, mX, fmaf(pb.z, mZ1, t3)));
    const float d2q = 2.f * pb.z;
#pragma unroll
    for (int h = 1; h < Z; ++h) {
      q[h] = q[h - 1] + dq;
      dq += d2q;
    }
    bool live[Z], band = false;
#pragma unroll
    for (int h = 0; h < Z; ++h) {
      live[h] = q[h] >= pc.w;
      const float w = ex2_approx(q[h]);
      if (live[h]) {
        aS[h] = fmaf(pc.z, w, aS[h]);
        aW[h] += w;
      }
    }
    if constexpr (MASKS)   // the column's live words of this hit (warp-uniform stores)
      sts_u4(smw_a + 16u * (uint32_t)jj,
             make_uint4(__ballot_sync(kFull, live[0]), __ballot_sync(kFull, live[1]),
                        __ballot_sync(kFull, live[2]), __ballot_sync(kFull, live[3])));
#pragma unroll
    for (int h = 0; h < Z; ++h) band |= !live[h] && q[h] >= pd.x;
    if (__any_sync(kFull, band)) {
      const int gidj = __float_as_int(pd.y);
      if constexpr (MASKS) {
        bool xl[Z];
#pragma unroll
        for (int h = 0; h < Z; ++h) {
          xl[h] = !live[h] && q[h] >= pd.x && exact_live(gidj, gx, gy, gz + h, xsrc, g, cut2d);
          if (xl[h]) {
            const float w = ex2_approx(q[h]);
            aS[h] = fmaf(pc.z, w, aS[h]);
            aW[h] += w;
          }
        }
        const uint4 x = make_uint4(__ballot_sync(kFull, xl[0]), __ballot_sync(kFull, xl[1]),
                                   __ballot_sync(kFull, xl[2]), __ballot_sync(kFull, xl[3]));
        const uint4 a = lds_u4(smw_a + 16u * (uint32_t)jj);
        __syncwarp();
        sts_u4(smw_a + 16u * (uint32_t)jj,
               make_uint4(a.x | x.x, a.y | x.y, a.z | x.z, a.w | x.w));
      } else {
#pragma unroll
        for (int h = 0; h < Z; ++h)
          if (!live[h] && q[h] >= pd.x && exact_live(gidj, gx, gy, gz + h, xsrc, g, cut2d)) {
            const float w = ex2_approx(q[h]);
            aS[h] = fmaf(pc.z, w, aS[h]);
            aW[h] += w;
          }
      }
    }
  }
}

// TWO: per 32-pair round, the hits are compacted into one list per y-half of
// the brick (each half's own box and sphere cull) and each list is evaluated
// for that half's column only -- a pair that reaches one half costs half.
// MASKS (two-list form, the train step): the pair's live-voxel words in the
// backward's VPL-4 pair-major layout -- column A (y < 4) is tile 0, column B
// tile 1, word = 4 tile + z, bit = lane -- one 32-byte store per pair.
#ifndef GSV_WHOLE_MINB
#define GSV_WHOLE_MINB 16       // CTAs (warps) per SM the whole-brick kernel is built for
#endif
template <bool TWO, bool MASKS = false>
__global__ void __launch_bounds__(32, GSV_WHOLE_MINB)
forward32w_kernel(const double* __restrict__ pos, const __grid_constant__ ExactSrc xsrc,
                  const gsv_record32* __restrict__ rec,
                  const int64_t* __restrict__ starts, const int32_t* __restrict__ gids,
                  const __grid_constant__ gsv_grid g, gsv_bricks k, float cut2, double cut2d,
                  double eps_w,
                  float* __restrict__ S, float* __restrict__ W, float* __restrict__ I,
                  const void* __restrict__ target, int target_f64, int loss_kind, double vox_count,
                  float2* __restrict__ ab, double* __restrict__ loss_part,
                  uint2* __restrict__ live_masks = nullptr) {
  static_assert(!MASKS || TWO, "live masks need the two-list form");
  constexpr int Z = 4;
  __shared__ Pair32 wsp[TWO ? 64 : 32];
  __shared__ uint4 smw[MASKS ? 64 : 1];      // per hit slot: its column's 4 live words
  const int lb = blockIdx.x;
  const int b = (int)slab_first(k) + lb;
  const BrickGeom bg = brick_geom(b, g, k);
  const int64_t lbeg = starts[lb], lend = starts[lb + 1];
  const int lane = threadIdx.x;
  const float fsx = (float)g.sx, fsy = (float)g.sy, fsz = (float)g.sz;
  const float isx = (float)(1.0 / g.sx), isy = (float)(1.0 / g.sy), isz = (float)(1.0 / g.sz);
  const int lx = lane & 7, lyA = lane >> 3, lyB = lyA + 4;
  // the brick's owned voxel box and centre (brick-local voxel coordinates)
  const float ftxh = (float)(bg.ex - 1), ftyh = (float)(bg.ey - 1), ftzh = (float)(bg.ez - 1);
  const float ftxl = 0.f, ftyl = 0.f, ftzl = 0.f;
  const float ctx = 0.5f * ftxh, cty = 0.5f * ftyh, ctz = 0.5f * ftzh;
  const float ext_x = ctx, ext_y = cty, ext_z = ctz;
  const float mX = (float)lx - ctx, mY = (float)lyA - cty, mZ = -ctz, mZ1 = mZ + 1.f;
  const float twoY4 = fmaf(2.f, mY, 4.f);      // column B = column A + 4 in y
  const float mYB = mY + 4.f;
  const uint32_t wsp_a = smem_addr(wsp);
  const int gx = bg.x0 + lx, gyA = bg.y0 + lyA, gyB = bg.y0 + lyB, gz = bg.z0;
  unsigned ownA[Z], ownB[Z];                   // voxels inside the grid (mask words)
  if constexpr (MASKS) {
#pragma unroll
    for (int h = 0; h < Z; ++h) {
      ownA[h] = __ballot_sync(kFull, lx < bg.ex && lyA < bg.ey && h < bg.ez);
      ownB[h] = __ballot_sync(kFull, lx < bg.ex && lyB < bg.ey && h < bg.ez);
    }
  }
  float aS[2][Z], aW[2][Z];
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int h = 0; h < Z; ++h) aS[c][h] = aW[c][h] = 0.f;
  double lsum = 0.0;

  int gid_next = (lbeg + lane < lend) ? __ldg(gids + lbeg + lane) : -1;
  for (int64_t base = lbeg; base < lend; base += 32) {
    const int gid = gid_next;
    gid_next = (base + 32 + lane < lend) ? __ldg(gids + base + 32 + lane) : -1;
    bool hit = false, hitA = false, hitB = false;
    Pair32 p;
    if (gid >= 0) {
      const float4* r4 = reinterpret_cast<const float4*>(rec + gid);
      const float4 q0 = __ldg(r4), q1 = __ldg(r4 + 1), q2 = __ldg(r4 + 2), q3 = __ldg(r4 + 3);
      const double* m = pos + 3 * (int64_t)gid;
      const float mx = (float)(__ldg(m) - bg.px), my = (float)(__ldg(m + 1) - bg.py),
                  mz = (float)(__ldg(m + 2) - bg.pz);
      const float cxv = mx * isx, cyv = my * isy, czv = mz * isz;
      const float hxv = fmaf(q2.w, isx, 1e-3f), hyv = fmaf(q3.x, isy, 1e-3f),
                  hzv = fmaf(q3.y, isz, 1e-3f);
      hit = cxv + hxv >= ftxl && cxv - hxv <= ftxh && cyv + hyv >= ftyl &&
            cyv - hyv <= ftyh && czv + hzv >= ftzl && czv - hzv <= ftzh;
      if (TWO && hit) {                        // y-half boxes: [0, 3] and [4, ey - 1]
        hitA = cyv - hyv <= fminf(3.f, ftyh);
        hitB = ftyh >= 4.f && cyv + hyv >= 4.f;
      }
      if (hit && !isinf(cut2)) {
        const float ddx = fmaxf(fmaxf(ftxl - cxv, cxv - ftxh), 0.f) * fsx;
        const float ddy = fmaxf(fmaxf(ftyl - cyv, cyv - ftyh), 0.f) * fsy;
        const float ddz = fmaxf(fmaxf(ftzl - czv, czv - ftzh), 0.f) * fsz;
        const float dist2 = fmaf(ddx, ddx, fmaf(ddy, ddy, ddz * ddz));
        const float lim = cut2 * 1.0001f + 1e-6f;
        hit = dist2 * q3.z <= lim;
        if (TWO) {
          const float ddyA = fmaxf(fmaxf(-cyv, cyv - fminf(3.f, ftyh)), 0.f) * fsy;
          const float ddyB = fmaxf(fmaxf(4.f - cyv, cyv - ftyh), 0.f) * fsy;
          const float xz = fmaf(ddx, ddx, ddz * ddz);
          hitA = hitA && fmaf(ddyA, ddyA, xz) * q3.z <= lim;
          hitB = hitB && fmaf(ddyB, ddyB, xz) * q3.z <= lim;
        }
      }
      if (TWO) {
        hitA = hitA && hit;
        hitB = hitB && hit;
        hit = hitA || hitB;
      }
      if (hit) {
        const float L[9] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w, q2.x};
        float u3[3], e[3][3], umax = 0.f;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          u3[a] = -fmaf(L[3 * a + 0], mx, fmaf(L[3 * a + 1], my, L[3 * a + 2] * mz));
          e[0][a] = L[3 * a + 0] * fsx;
          e[1][a] = L[3 * a + 1] * fsy;
          e[2][a] = L[3 * a + 2] * fsz;
          umax = fmaxf(umax, fabsf(u3[a]) + fabsf(e[0][a]) * k.bdx +
                                 fabsf(e[1][a]) * k.bdy + fabsf(e[2][a]) * k.bdz);
        }
        float uc[3];
#pragma unroll
        for (int a = 0; a < 3; ++a)
          uc[a] = fmaf(ctz, e[2][a], fmaf(cty, e[1][a], fmaf(ctx, e[0][a], u3[a])));
        const float sc = -0.72134752044448170f;   // -(1/2) log2(e)
        const float lr2 = __log2f(q2.z);
        const float d00 = fmaf(uc[0], uc[0], fmaf(uc[1], uc[1], uc[2] * uc[2]));
        p.a.x = fmaf(sc, d00, lr2);
        p.a.y = 2.f * sc * fmaf(uc[0], e[0][0], fmaf(uc[1], e[0][1], uc[2] * e[0][2]));
        p.a.z = 2.f * sc * fmaf(uc[0], e[1][0], fmaf(uc[1], e[1][1], uc[2] * e[1][2]));
        p.a.w = 2.f * sc * fmaf(uc[0], e[2][0], fmaf(uc[1], e[2][1], uc[2] * e[2][2]));
        p.b.x = sc * fmaf(e[0][0], e[0][0], fmaf(e[0][1], e[0][1], e[0][2] * e[0][2]));
        p.b.y = sc * fmaf(e[1][0], e[1][0], fmaf(e[1][1], e[1][1], e[1][2] * e[1][2]));
        p.b.z = sc * fmaf(e[2][0], e[2][0], fmaf(e[2][1], e[2][1], e[2][2] * e[2][2]));
        p.b.w = 2.f * sc * fmaf(e[0][0], e[1][0], fmaf(e[0][1], e[1][1], e[0][2] * e[1][2]));
        p.c.x = 2.f * sc * fmaf(e[0][0], e[2][0], fmaf(e[0][1], e[2][1], e[0][2] * e[2][2]));
        p.c.y = 2.f * sc * fmaf(e[1][0], e[2][0], fmaf(e[1][1], e[2][1], e[1][2] * e[2][2]));
        p.c.z = q2.y;
        const float qmag = fabsf(p.a.x) + ext_x * fabsf(p.a.y) + ext_y * fabsf(p.a.z) +
                           ext_z * fabsf(p.a.w) + ext_x * ext_x * fabsf(p.b.x) +
                           ext_y * ext_y * fabsf(p.b.y) + ext_z * ext_z * fabsf(p.b.z) +
                           ext_x * ext_y * fabsf(p.b.w) + ext_x * ext_z * fabsf(p.c.x) +
                           ext_y * ext_z * fabsf(p.c.y);
        const float guard = isinf(cut2) ? 0.f
                            : 0.72134752f * (kGuardRel * cut2 + kGuardMag * umax * sqrtf(cut2)) +
                                  2.5e-6f * qmag;
        const float qcut = isinf(cut2) ? -INFINITY : fmaf(sc, cut2, lr2);
        p.c.w = qcut + guard;
        p.d = make_float4(qcut - guard, __int_as_float(gid), 0.f, 0.f);
      }
    }
    if (TWO) {
      const unsigned lt = (1u << lane) - 1u;
      const unsigned ballA = __ballot_sync(kFull, hitA), ballB = __ballot_sync(kFull, hitB);
      if (hitA) wsp[__popc(ballA & lt)] = p;
      if (hitB) wsp[32 + __popc(ballB & lt)] = p;
      __syncwarp();
      if constexpr (MASKS) {
        eval_column_hits<true>(wsp_a, __popc(ballA), mX, mY, mZ, mZ1, gx, gyA, gz, xsrc, g,
                               cut2d, aS[0], aW[0], smem_addr(smw));
        eval_column_hits<true>(wsp_a + 32u * (uint32_t)sizeof(Pair32), __popc(ballB), mX, mYB,
                               mZ, mZ1, gx, gyB, gz, xsrc, g, cut2d, aS[1], aW[1],
                               smem_addr(smw) + 32u * 16u);
      } else {
        eval_column_hits_plain(wsp_a, __popc(ballA), mX, mY, mZ, mZ1, gx, gyA, gz, xsrc, g, cut2d,
                               aS[0], aW[0]);
        eval_column_hits_plain(wsp_a + 32u * (uint32_t)sizeof(Pair32), __popc(ballB), mX, mYB,
                               mZ, mZ1, gx, gyB, gz, xsrc,
                               g, cut2d, aS[1], aW[1]);
      }
      __syncwarp();
      if (MASKS && gid >= 0) {
        const uint4 zero = make_uint4(0u, 0u, 0u, 0u);
        uint4 wa = hitA ? smw[__popc(ballA & lt)] : zero;
        uint4 wb = hitB ? smw[32 + __popc(ballB & lt)] : zero;
        wa = make_uint4(wa.x & ownA[0], wa.y & ownA[1], wa.z & ownA[2], wa.w & ownA[3]);
        wb = make_uint4(wb.x & ownB[0], wb.y & ownB[1], wb.z & ownB[2], wb.w & ownB[3]);
        uint4* dst = reinterpret_cast<uint4*>(live_masks + 4 * (base + lane));
        dst[0] = wa;
        dst[1] = wb;
      }
      __syncwarp();
      continue;
    }
    const unsigned ball = __ballot_sync(kFull, hit);
    if (hit) wsp[__popc(ball & ((1u << lane) - 1u))] = p;
    __syncwarp();
    const int nh = __popc(ball);
    for (int jj = 0; jj < nh; ++jj) {
      const float4 pa = wsp[jj].a, pb = wsp[jj].b, pc = wsp[jj].c;
      const float2 pd = *reinterpret_cast<const float2*>(&wsp[jj].d);   // qlo, gid
      float q[2][Z];
      const float t1 = fmaf(pb.x, mX, fmaf(pb.w, mY, fmaf(pc.x, mZ, pa.y)));
      const float t2 = fmaf(pb.y, mY, fmaf(pc.y, mZ, pa.z));
      const float t3 = fmaf(pb.z, mZ, pa.w);
      q[0][0] = fmaf(mX, t1, fmaf(mY, t2, fmaf(mZ, t3, pa.x)));
      // column B (y + 4): q += 4 (a_z + b_w X + c_y Z + b_y (2Y + 4)); dq += 4 c_y
      q[1][0] = fmaf(4.f, fmaf(pb.y, twoY4, fmaf(pc.y, mZ, fmaf(pb.w, mX, pa.z))), q[0][0]);
      float dqA = fmaf(pc.y, mY, fmaf(pc.x, mX, fmaf(pb.z, mZ1, t3)));
      float dqB = fmaf(4.f, pc.y, dqA);
      const float d2q = 2.f * pb.z;
#pragma unroll
      for (int h = 1; h < Z; ++h) {
        q[0][h] = q[0][h - 1] + dqA;
        q[1][h] = q[1][h - 1] + dqB;
        dqA += d2q;
        dqB += d2q;
      }
      bool live[2][Z];
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int h = 0; h < Z; ++h) {
          live[c][h] = q[c][h] >= pc.w;
          const float w = ex2_approx(q[c][h]);
          if (live[c][h]) {
            aS[c][h] = fmaf(pc.z, w, aS[c][h]);
            aW[c][h] += w;
          }
        }
      bool band = false;
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int h = 0; h < Z; ++h) band |= !live[c][h] && q[c][h] >= pd.x;
      if (__any_sync(kFull, band)) {
        const int gidj = __float_as_int(pd.y);
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int h = 0; h < Z; ++h)
            if (!live[c][h] && q[c][h] >= pd.x &&
                exact_live(gidj, gx, c ? gyB : gyA, gz + h, xsrc, g, cut2d)) {
              const float w = ex2_approx(q[c][h]);
              aS[c][h] = fmaf(pc.z, w, aS[c][h]);
              aW[c][h] += w;
            }
      }
    }
    __syncwarp();
  }
  // Epilogue: normalise, store, fused loss (optimize.py:91-103).
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int h = 0; h < Z; ++h) {
      const int ly = c ? lyB : lyA;
      if (!(lx < bg.ex && ly < bg.ey && h < bg.ez)) continue;
      const int64_t lin = (int64_t)gx + (int64_t)g.nx * ((bg.y0 + ly) + (int64_t)g.ny * (gz + h));
      const bool cov = (double)aW[c][h] >= eps_w;
      const float iv = cov ? __fdiv_rn(aS[c][h], aW[c][h]) : 0.f;
      S[lin] = aS[c][h];
      W[lin] = aW[c][h];
      I[lin] = iv;
      if (target) {
        const double d = (double)iv - target_value(target, target_f64, lin);
        double dl;
        if (loss_kind == 0) {
          lsum += fabs(d);
          dl = (d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0)) / vox_count;
        } else {
          lsum += d * d;
          dl = 2.0 * d / vox_count;
        }
        const float alpha = (cov && dl != 0.0) ? (float)(dl / (double)aW[c][h]) : 0.f;
        ab[lin] = make_float2(alpha, iv);
      }
    }
  if (target) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lsum += __shfl_down_sync(kFull, lsum, o);
    if (lane == 0) loss_part[lb] = lsum;
  }
}

// ------------------------------------ forward f32, grouped columns (LR grids)
// One warp per 8x8x4 brick, like forward32w_kernel, but the voxel tile a warp
// evaluates adapts to the pairs.  Per 32-entry round every staged pair's
// footprint inside the brick -- its 3-sigma AABB clipped to the brick's owned
// voxels: a rectangle of columns (x, y) and a z range -- is computed.
// Consecutive hits (list order) with the same rectangle form a group: at LR a
// brick's list runs through each (ix, iy) of its neighbourhood in z, so a
// group is typically the ~8 Gaussians of one z-run, whose rectangles
// coincide.  The groups' rectangles are laid end to end and dealt to the
// lanes 32 columns at a time (a "chunk"); each lane walks its group's pairs
// in list order and accumulates its column's 4 voxels in registers, exactly
// the fixed-ownership kernels' per-hit evaluation (nested quadratic at the
// column top, second differences in z, f64 guard band) -- but only over
// columns some pair of the group reaches.  At config 3 this evaluates ~2.5x
// fewer (pair, column) slots than the two-list whole-brick kernel.
// The group's sum then goes into the brick's shared S and W, one group after
// another in list order (a group's columns are distinct, so its lanes never
// conflict).  Per voxel: S = ((S_prev + (c1 + c2 + ...)) + ...) -- a fixed,
// list-determined association: bit-reproducible across runs and list
// shuffles (canonical lists), equal to the sequential sum up to f32 rounding.
// MASKS: the live-voxel masks of the train step's backward, per pair 8
// words, word y (brick row), bit 4x + z -- one shared atomic OR per lane and
// evaluated (pair, column).
#ifndef GSV_COLS_MINB
#define GSV_COLS_MINB 16        // CTAs (warps) per SM the grouped kernel is built for
#endif
__device__ __forceinline__ void red_or_shared(uint32_t a, uint32_t v) {
  asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(v));
}
__device__ __forceinline__ uint32_t rect_word(int x0, int y0, int x1, int y1) {
  return (uint32_t)x0 | (uint32_t)y0 << 3 | (uint32_t)x1 << 6 | (uint32_t)y1 << 9;
}

template <bool MASKS>
__global__ void __launch_bounds__(32, GSV_COLS_MINB)
forward32c_kernel(const double* __restrict__ pos, const __grid_constant__ ExactSrc xsrc,
                  const gsv_record32* __restrict__ rec,
                  const int64_t* __restrict__ starts, const int32_t* __restrict__ gids,
                  const __grid_constant__ gsv_grid g, gsv_bricks k, float cut2, double cut2d,
                  double eps_w,
                  float* __restrict__ S, float* __restrict__ W, float* __restrict__ I,
                  const void* __restrict__ target, int target_f64, int loss_kind,
                  double vox_count, float2* __restrict__ ab, double* __restrict__ loss_part,
                  uint4* __restrict__ live_masks) {
  constexpr int Z = 4;
  __shared__ Pair32 sp[32];                   // the round's hits, compacted (list order)
  __shared__ uint32_t srect[32];              // hit -> rect_word
  __shared__ int sgs[33];                     // group -> first hit
  __shared__ float4 sS4[64], sW4[64];         // S, W of column x + 8 y, z = .x .. .w
  __shared__ uint32_t smk[MASKS ? 32 * 8 : 1];
  const int lb = blockIdx.x;
  const int b = (int)slab_first(k) + lb;
  const BrickGeom bg = brick_geom(b, g, k);
  const int64_t lbeg = starts[lb], lend = starts[lb + 1];
  const int lane = threadIdx.x;
  const unsigned lt = (1u << lane) - 1u;
  const float fsx = (float)g.sx, fsy = (float)g.sy, fsz = (float)g.sz;
  const float isx = (float)(1.0 / g.sx), isy = (float)(1.0 / g.sy), isz = (float)(1.0 / g.sz);
  // the brick's owned voxel box and centre (brick-local voxel coordinates):
  // the same quadratic origin as forward32w_kernel
  const float ftxh = (float)(bg.ex - 1), ftyh = (float)(bg.ey - 1), ftzh = (float)(bg.ez - 1);
  const float ctx = 0.5f * ftxh, cty = 0.5f * ftyh, ctz = 0.5f * ftzh;
  const float ext_x = ctx, ext_y = cty, ext_z = ctz;
  const float mZ = -ctz, mZ1 = mZ + 1.f;
  sS4[lane] = sS4[lane + 32] = sW4[lane] = sW4[lane + 32] = make_float4(0.f, 0.f, 0.f, 0.f);
  if constexpr (MASKS) {
#pragma unroll
    for (int i = 0; i < 8; ++i) smk[lane + 32 * i] = 0u;
  }
  __syncwarp();
  const uint32_t sp_a = smem_addr(sp);
  const uint32_t smk_a = smem_addr(smk);

  int gid_next = (lbeg + lane < lend) ? __ldg(gids + lbeg + lane) : -1;
  int gid_next2 = (lbeg + 32 + lane < lend) ? __ldg(gids + lbeg + 32 + lane) : -1;
  for (int64_t base = lbeg; base < lend; base += 32) {
    const int gid = gid_next;
    gid_next = gid_next2;
    gid_next2 = (base + 64 + lane < lend) ? __ldg(gids + base + 64 + lane) : -1;
    if (gid_next >= 0) {   // next round's record and position lines, in flight now
      prefetch_line(rec + gid_next);
      prefetch_line(pos + 3 * (int64_t)gid_next);
    }
    bool hit = false;
    Pair32 p;
    uint32_t rw = 0u;
    if (gid >= 0) {
      const float4* r4 = reinterpret_cast<const float4*>(rec + gid);
      const float4 q0 = __ldg(r4), q1 = __ldg(r4 + 1), q2 = __ldg(r4 + 2), q3 = __ldg(r4 + 3);
      const double* m = pos + 3 * (int64_t)gid;
      const float mx = (float)(__ldg(m) - bg.px), my = (float)(__ldg(m + 1) - bg.py),
                  mz = (float)(__ldg(m + 2) - bg.pz);
      const float cxv = mx * isx, cyv = my * isy, czv = mz * isz;
      const float hxv = fmaf(q2.w, isx, 1e-3f), hyv = fmaf(q3.x, isy, 1e-3f),
                  hzv = fmaf(q3.y, isz, 1e-3f);
      // footprint: the integer voxels of the (widened) 3-sigma box, clipped
      // to the owned voxels -- every live voxel lies in it
      const float ax0 = fmaxf(ceilf(cxv - hxv), 0.f), ax1 = fminf(floorf(cxv + hxv), ftxh);
      const float ay0 = fmaxf(ceilf(cyv - hyv), 0.f), ay1 = fminf(floorf(cyv + hyv), ftyh);
      const float az0 = fmaxf(ceilf(czv - hzv), 0.f), az1 = fminf(floorf(czv + hzv), ftzh);
      hit = ax0 <= ax1 && ay0 <= ay1 && az0 <= az1;
      if (hit && !isinf(cut2)) {
        // sphere bound |p - mu|^2 / sigma_max^2 <= cut^2 against the footprint box
        const float ddx = fmaxf(fmaxf(ax0 - cxv, cxv - ax1), 0.f) * fsx;
        const float ddy = fmaxf(fmaxf(ay0 - cyv, cyv - ay1), 0.f) * fsy;
        const float ddz = fmaxf(fmaxf(az0 - czv, czv - az1), 0.f) * fsz;
        const float dist2 = fmaf(ddx, ddx, fmaf(ddy, ddy, ddz * ddz));
        hit = dist2 * q3.z <= cut2 * 1.0001f + 1e-6f;
      }
      if (hit) {
        rw = rect_word((int)ax0, (int)ay0, (int)ax1, (int)ay1);
        const float L[9] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w, q2.x};
        float u3[3], e[3][3], umax = 0.f;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          u3[a] = -fmaf(L[3 * a + 0], mx, fmaf(L[3 * a + 1], my, L[3 * a + 2] * mz));
          e[0][a] = L[3 * a + 0] * fsx;
          e[1][a] = L[3 * a + 1] * fsy;
          e[2][a] = L[3 * a + 2] * fsz;
          umax = fmaxf(umax, fabsf(u3[a]) + fabsf(e[0][a]) * k.bdx +
                                 fabsf(e[1][a]) * k.bdy + fabsf(e[2][a]) * k.bdz);
        }
        float uc[3];
#pragma unroll
        for (int a = 0; a < 3; ++a)
          uc[a] = fmaf(ctz, e[2][a], fmaf(cty, e[1][a], fmaf(ctx, e[0][a], u3[a])));
        const float sc = -0.72134752044448170f;   // -(1/2) log2(e)
        const float lr2 = __log2f(q2.z);
        const float d00 = fmaf(uc[0], uc[0], fmaf(uc[1], uc[1], uc[2] * uc[2]));
        p.a.x = fmaf(sc, d00, lr2);
        p.a.y = 2.f * sc * fmaf(uc[0], e[0][0], fmaf(uc[1], e[0][1], uc[2] * e[0][2]));
        p.a.z = 2.f * sc * fmaf(uc[0], e[1][0], fmaf(uc[1], e[1][1], uc[2] * e[1][2]));
        p.a.w = 2.f * sc * fmaf(uc[0], e[2][0], fmaf(uc[1], e[2][1], uc[2] * e[2][2]));
        p.b.x = sc * fmaf(e[0][0], e[0][0], fmaf(e[0][1], e[0][1], e[0][2] * e[0][2]));
        p.b.y = sc * fmaf(e[1][0], e[1][0], fmaf(e[1][1], e[1][1], e[1][2] * e[1][2]));
        p.b.z = sc * fmaf(e[2][0], e[2][0], fmaf(e[2][1], e[2][1], e[2][2] * e[2][2]));
        p.b.w = 2.f * sc * fmaf(e[0][0], e[1][0], fmaf(e[0][1], e[1][1], e[0][2] * e[1][2]));
        p.c.x = 2.f * sc * fmaf(e[0][0], e[2][0], fmaf(e[0][1], e[2][1], e[0][2] * e[2][2]));
        p.c.y = 2.f * sc * fmaf(e[1][0], e[2][0], fmaf(e[1][1], e[2][1], e[1][2] * e[2][2]));
        p.c.z = q2.y;
        const float qmag = fabsf(p.a.x) + ext_x * fabsf(p.a.y) + ext_y * fabsf(p.a.z) +
                           ext_z * fabsf(p.a.w) + ext_x * ext_x * fabsf(p.b.x) +
                           ext_y * ext_y * fabsf(p.b.y) + ext_z * ext_z * fabsf(p.b.z) +
                           ext_x * ext_y * fabsf(p.b.w) + ext_x * ext_z * fabsf(p.c.x) +
                           ext_y * ext_z * fabsf(p.c.y);
        const float guard = isinf(cut2) ? 0.f
                            : 0.72134752f * (kGuardRel * cut2 + kGuardMag * umax * sqrtf(cut2)) +
                                  2.5e-6f * qmag;
        const float qcut = isinf(cut2) ? -INFINITY : fmaf(sc, cut2, lr2);
        p.c.w = qcut + guard;
        p.d = make_float4(qcut - guard, __int_as_float(gid), 0.f, 0.f);
      }
    }
    // ---- the round's hits, compacted in list order, and their groups
    const unsigned hitmask = __ballot_sync(kFull, hit);
    const int nh = __popc(hitmask);
    const int r = __popc(hitmask & lt);
    if (hit) {
      sp[r] = p;
      srect[r] = rw;
    }
    __syncwarp();
    // hit r (lane r) starts a group unless its rectangle equals hit r-1's
    const uint32_t myrect = lane < nh ? srect[lane] : 0u;
    const bool gstart_ = lane < nh && (lane == 0 || srect[lane - 1] != myrect);
    const unsigned gmask = __ballot_sync(kFull, gstart_);
    const int ng = __popc(gmask);
    if (gstart_) sgs[__popc(gmask & lt)] = lane;
    if (lane == 0) sgs[ng] = nh;
    __syncwarp();
    // lane gg describes group gg: first hit, size, column area, column prefix
    const int gfirst = lane < ng ? sgs[lane] : nh;
    const int gsize = lane < ng ? sgs[lane + 1] - gfirst : 0;
    uint32_t grect = lane < ng ? srect[gfirst] : 0u;
    const int gwx = (int)((grect >> 6) & 7u) - (int)(grect & 7u) + 1;
    // ceil(512 / wx) in bits 12-21: column k of the rectangle is row
    // (k * magic) >> 9 exactly for k < 64, wx <= 8 (no division per chunk)
    grect |= ((512u + (uint32_t)gwx - 1u) / (uint32_t)gwx) << 12;
    const int gwy = (int)((grect >> 9) & 7u) - (int)((grect >> 3) & 7u) + 1;
    const int garea = lane < ng ? gwx * gwy : 0;
    int incl = garea;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += n;
    }
    const int gpre = incl - garea;
    const int T = __shfl_sync(kFull, incl, 31);
    for (int c0 = 0; c0 < T; c0 += 32) {
      const int s = c0 + lane;
      const bool valid = s < T;
      // the group owning column slot s
      const int cnt0 = __popc(__ballot_sync(kFull, lane < ng && gpre <= c0));
      const unsigned sb = __reduce_or_sync(kFull, (lane < ng && gpre > c0 && gpre < c0 + 32)
                                                      ? 1u << (gpre - c0) : 0u);
      const int myg = valid ? cnt0 - 1 + __popc(sb & ((2u << lane) - 1u)) : cnt0 - 1;
      const int glast = __shfl_sync(kFull, myg, min(31, T - 1 - c0));
      const int gf = cnt0 - 1;
      const int h0 = __shfl_sync(kFull, gfirst, myg);
      const int hk_all = __shfl_sync(kFull, gsize, myg);   // every lane shuffles
      const int hk = valid ? hk_all : 0;
      const int kk = s - __shfl_sync(kFull, gpre, myg);
      const uint32_t rc = __shfl_sync(kFull, grect, myg);
      const int wx = (int)((rc >> 6) & 7u) - (int)(rc & 7u) + 1;
      const int dy = (int)(((uint32_t)kk * ((rc >> 12) & 1023u)) >> 9);
      const int x = (int)(rc & 7u) + kk - dy * wx;
      const int y = (int)((rc >> 3) & 7u) + dy;
      const float mX = (float)x - ctx, mY = (float)y - cty;
      const int kmax = __reduce_max_sync(kFull, hk);
      float aS[Z], aW[Z];
#pragma unroll
      for (int h = 0; h < Z; ++h) aS[h] = aW[h] = 0.f;
      bool any = false;
      // The pair loop: inactive lanes get infinite thresholds, the
      // live tests drive predicated accumulation directly, the rare guard
      // band adds its voxels in the same iteration (so per voxel the pairs
      // stay in list order); full-depth bricks skip the owned-z tests.
      auto walk = [&](auto fullz) {
        for (int t = 0; t < kmax; ++t) {
          const bool act0 = t < hk;
          GSV_DCHECK(!act0 || (h0 + t >= 0 && h0 + t < nh && x >= 0 && x < bg.ex && y >= 0 &&
                               y < bg.ey));
          const uint32_t ja = sp_a + (uint32_t)(act0 ? h0 + t : h0) * (uint32_t)sizeof(Pair32);
          const float4 pa = lds_f4(ja), pb = lds_f4(ja + 16), pc = lds_f4(ja + 32);
          const float4 p4 = lds_f4(ja + 48);   // qlo, gid
          float q[Z];
          const float t1 = fmaf(pb.x, mX, fmaf(pb.w, mY, fmaf(pc.x, mZ, pa.y)));
          const float t2 = fmaf(pb.y, mY, fmaf(pc.y, mZ, pa.z));
          const float t3 = fmaf(pb.z, mZ, pa.w);
          q[0] = fmaf(mX, t1, fmaf(mY, t2, fmaf(mZ, t3, pa.x)));
          float dq = fmaf(pc.y, mY, fmaf(pc.x, mX, fmaf(pb.z, mZ1, t3)));
          const float d2q = 2.f * pb.z;
#pragma unroll
          for (int h = 1; h < Z; ++h) {
            q[h] = q[h - 1] + dq;
            dq += d2q;
          }
          const float tl = act0 ? pc.w : INFINITY, tb = act0 ? p4.x : INFINITY;
          bool lv[Z], band = false;
          uint32_t lm = 0u;
#pragma unroll
          for (int h = 0; h < Z; ++h) {
            bool ownz = true;
            if constexpr (!decltype(fullz)::value) ownz = h < bg.ez;
            lv[h] = ownz && q[h] >= tl;
            const float w = ex2_approx(q[h]);
            if (lv[h]) {
              aS[h] = fmaf(pc.z, w, aS[h]);
              aW[h] += w;
            }
            lm |= (uint32_t)lv[h] << h;
            band |= ownz && !lv[h] && q[h] >= tb;
          }
          if (__any_sync(kFull, band)) {
            const int gidj = __float_as_int(p4.y);
#pragma unroll
            for (int h = 0; h < Z; ++h)
              if (!lv[h] && q[h] >= tb && h < bg.ez &&
                  exact_live(gidj, bg.x0 + x, bg.y0 + y, bg.z0 + h, xsrc, g, cut2d)) {
                const float w = ex2_approx(q[h]);
                aS[h] = fmaf(pc.z, w, aS[h]);
                aW[h] += w;
                lm |= 1u << h;
              }
          }
          any |= lm != 0u;
          if constexpr (MASKS) {
            if (lm) red_or_shared(smk_a + 4u * (uint32_t)(8 * (h0 + t) + y), lm << (4 * x));
          }
        }
      };
      if (bg.ez == Z)
        walk(std::integral_constant<bool, true>());
      else
        walk(std::integral_constant<bool, false>());
      // the groups' sums into the brick's S and W, one group after another
      const int col = x + 8 * y;
      GSV_DCHECK(!valid || (col >= 0 && col < 64 && myg >= 0 && myg < ng && kk >= 0));
      for (int gg = gf; gg <= glast; ++gg) {
        if (valid && myg == gg && any) {
          float4 sv = sS4[col], wv = sW4[col];
          sv.x += aS[0]; sv.y += aS[1]; sv.z += aS[2]; sv.w += aS[3];
          wv.x += aW[0]; wv.y += aW[1]; wv.z += aW[2]; wv.w += aW[3];
          sS4[col] = sv;
          sW4[col] = wv;
        }
        __syncwarp();
      }
    }
    if constexpr (MASKS) {
      // each entry's 32-byte mask record (zero for pairs without a footprint)
      __syncwarp();
      if (gid >= 0) {
        uint4 m0 = make_uint4(0u, 0u, 0u, 0u), m1 = m0;
        if (hit) {
          const uint4* src = reinterpret_cast<const uint4*>(smk + 8 * r);
          m0 = src[0];
          m1 = src[1];
        }
        GSV_DCHECK(base + lane < lend && (!hit || r < nh));
        uint4* dst = live_masks + 2 * (base + lane);
        dst[0] = m0;
        dst[1] = m1;
      }
      __syncwarp();
      reinterpret_cast<uint4*>(smk)[2 * lane] = make_uint4(0u, 0u, 0u, 0u);
      reinterpret_cast<uint4*>(smk)[2 * lane + 1] = make_uint4(0u, 0u, 0u, 0u);
    }
    __syncwarp();
  }
  // Epilogue: normalise, store, fused loss (optimize.py:91-103).
  double lsum = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int v = lane + 32 * i;
    const int x = v & 7, y = (v >> 3) & 7, z = v >> 6;
    if (!(x < bg.ex && y < bg.ey && z < bg.ez)) continue;
    const float2 sw = make_float2(reinterpret_cast<const float*>(sS4)[4 * (v & 63) + z],
                                  reinterpret_cast<const float*>(sW4)[4 * (v & 63) + z]);
    const int64_t lin = (int64_t)(bg.x0 + x) +
                        (int64_t)g.nx * ((bg.y0 + y) + (int64_t)g.ny * (bg.z0 + z));
    GSV_DCHECK(lin >= 0 && lin < (int64_t)g.nx * g.ny * g.nz);
    const bool cov = (double)sw.y >= eps_w;
    const float iv = cov ? __fdiv_rn(sw.x, sw.y) : 0.f;
    S[lin] = sw.x;
    W[lin] = sw.y;
    I[lin] = iv;
    if (target) {
      const double d = (double)iv - target_value(target, target_f64, lin);
      double dl;
      if (loss_kind == 0) {
        lsum += fabs(d);
        dl = (d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0)) / vox_count;
      } else {
        lsum += d * d;
        dl = 2.0 * d / vox_count;
      }
      const float alpha = (cov && dl != 0.0) ? (float)(dl / (double)sw.y) : 0.f;
      ab[lin] = make_float2(alpha, iv);
    }
  }
  if (target) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lsum += __shfl_down_sync(kFull, lsum, o);
    if (lane == 0) loss_part[lb] = lsum;
  }
}

// ------------------------------------------ the forward's loss epilogue, alone
// For a graph step whose target arrives over PCIe during binning and the
// forward (gsv_loss_bricks): exactly the epilogue of forward32c_kernel
// (order 0: voxel v = lane + 32 i) or of forward32w_kernel (order 1: lane's
// column A then column B, z inside), one warp per 8x8x4 brick, so the loss
// partials and {alpha, I} are bit-identical to the fused forward's.
__global__ void __launch_bounds__(32)
loss_bricks_kernel(const __grid_constant__ gsv_grid g, gsv_bricks k, double eps_w,
                   const float* __restrict__ W, const float* __restrict__ I,
                   const void* __restrict__ target, int target_f64, int loss_kind,
                   double vox_count, int order, float2* __restrict__ ab,
                   double* __restrict__ loss_part) {
  const int lb = blockIdx.x;
  const int b = (int)slab_first(k) + lb;
  const BrickGeom bg = brick_geom(b, g, k);
  const int lane = threadIdx.x;
  double lsum = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int x, y, z;
    if (order == 0) {
      const int v = lane + 32 * i;
      x = v & 7;
      y = (v >> 3) & 7;
      z = v >> 6;
    } else {
      x = lane & 7;
      y = (lane >> 3) + 4 * (i >> 2);
      z = i & 3;
    }
    if (!(x < bg.ex && y < bg.ey && z < bg.ez)) continue;
    const int64_t lin = (int64_t)(bg.x0 + x) +
                        (int64_t)g.nx * ((bg.y0 + y) + (int64_t)g.ny * (bg.z0 + z));
    const float wv = W[lin], iv = I[lin];
    const bool cov = (double)wv >= eps_w;
    const double d = (double)iv - target_value(target, target_f64, lin);
    double dl;
    if (loss_kind == 0) {
      lsum += fabs(d);
      dl = (d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0)) / vox_count;
    } else {
      lsum += d * d;
      dl = 2.0 * d / vox_count;
    }
    const float alpha = (cov && dl != 0.0) ? (float)(dl / (double)wv) : 0.f;
    ab[lin] = make_float2(alpha, iv);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lsum += __shfl_down_sync(kFull, lsum, o);
  if (lane == 0) loss_part[lb] = lsum;
}

// --------------------------------------------------------------- forward f64
struct __align__(16) Pair64 {
  double l[9];
  double mx, my, mz;
  double amp, relax;
  int box0, box1;
  double _pad;
};

__global__ void __launch_bounds__(128)
forward64_kernel(const double* __restrict__ pos, const gsv_record64* __restrict__ rec,
                 const double* __restrict__ half_src, const int64_t* __restrict__ starts,
                 const int32_t* __restrict__ gids, gsv_grid g, gsv_bricks k, double cut2,
                 double eps_w, double* __restrict__ S, double* __restrict__ W,
                 double* __restrict__ I, const void* __restrict__ target, int target_f64, int loss_kind,
                 double vox_count, double2* __restrict__ ab, double* __restrict__ loss_part,
                 const gsv_record32* __restrict__ rec32) {
  constexpr int T = 128;
  __shared__ Pair64 sp[T];
  __shared__ double red[T / 32];
  (void)half_src;
  const int lb = blockIdx.x;
  const int b = (int)slab_first(k) + lb;
  const BrickGeom bg = brick_geom(b, g, k);
  const int64_t lbeg = starts[lb], lend = starts[lb + 1];
  const int nvb = k.bdx * k.bdy * k.bdz;
  const int tid = threadIdx.x;
  double lsum = 0.0;
  for (int vbase = 0; vbase < nvb; vbase += T) {
    const int vl = vbase + tid;
    const int lx = vl % k.bdx, ly = (vl / k.bdx) % k.bdy, lz = vl / (k.bdx * k.bdy);
    const bool own = vl < nvb && lx < bg.ex && ly < bg.ey && lz < bg.ez;
    const int ix = bg.x0 + lx, iy = bg.y0 + ly, iz = bg.z0 + lz;
    const double px = add(g.ox, mul((double)ix, g.sx));
    const double py = add(g.oy, mul((double)iy, g.sy));
    const double pz = add(g.oz, mul((double)iz, g.sz));
    double accS = 0.0, accW = 0.0;
    for (int64_t cb = lbeg; cb < lend; cb += T) {
      const int cnt = (int)min((int64_t)T, lend - cb);
      __syncthreads();
      if (tid < cnt) {
        const int gid = gids[cb + tid];
        const gsv_record64 r = rec[gid];
        const gsv_record32 r32 = rec32[gid];
        Pair64 p;
#pragma unroll
        for (int a = 0; a < 9; ++a) p.l[a] = r.l[a];
        const double* m = pos + 3 * (int64_t)gid;
        p.mx = m[0]; p.my = m[1]; p.mz = m[2];
        p.amp = r.amp;
        p.relax = r.relax;
        int xl, xh, yl, yh, zl, zh;
        sub_range(p.mx - bg.px, (double)r32.half[0], g.sx, bg.ex, xl, xh);
        sub_range(p.my - bg.py, (double)r32.half[1], g.sy, bg.ey, yl, yh);
        sub_range(p.mz - bg.pz, (double)r32.half[2], g.sz, bg.ez, zl, zh);
        if (xl > xh || yl > yh || zl > zh) {
          xl = 255; xh = 0;
        }
        p.box0 = (xl & 255) | ((xh & 255) << 8) | ((yl & 255) << 16) | ((yh & 255) << 24);
        p.box1 = (zl & 255) | ((zh & 255) << 8);
        p._pad = 0.0;
        sp[tid] = p;
      }
      __syncthreads();
      if (own) {
        for (int j = 0; j < cnt; ++j) {
          const Pair64& p = sp[j];
          const int b0 = p.box0, b1 = p.box1;
          if (lx < (b0 & 255) || lx > ((b0 >> 8) & 255) || ly < ((b0 >> 16) & 255) ||
              ly > ((b0 >> 24) & 255) || lz < (b1 & 255) || lz > ((b1 >> 8) & 255))
            continue;
          const double dx = sub(px, p.mx), dy = sub(py, p.my), dz = sub(pz, p.mz);
          const double v0 = add(add(mul(p.l[0], dx), mul(p.l[1], dy)), mul(p.l[2], dz));
          const double v1 = add(add(mul(p.l[3], dx), mul(p.l[4], dy)), mul(p.l[5], dz));
          const double v2 = add(add(mul(p.l[6], dx), mul(p.l[7], dy)), mul(p.l[8], dz));
          const double d2 = add(add(mul(v0, v0), mul(v1, v1)), mul(v2, v2));
          if (d2 <= cut2) {
            const double w = mul(exp(mul(-0.5, d2)), p.relax);
            accS = add(accS, mul(p.amp, w));
            accW = add(accW, w);
          }
        }
      }
    }
    if (own) {
      const int64_t lin = (int64_t)ix + (int64_t)g.nx * (iy + (int64_t)g.ny * iz);
      const bool cov = accW >= eps_w;
      const double iv = cov ? __ddiv_rn(accS, accW) : 0.0;
      S[lin] = accS;
      W[lin] = accW;
      I[lin] = iv;
      if (target) {
        const double d = iv - target_value(target, target_f64, lin);
        double dl;
        if (loss_kind == 0) {
          lsum += fabs(d);
          dl = (d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0)) / vox_count;
        } else {
          lsum += d * d;
          dl = 2.0 * d / vox_count;
        }
        const double alpha = (cov && dl != 0.0) ? dl / accW : 0.0;
        ab[lin] = make_double2(alpha, iv);
      }
    }
  }
  if (target) {
    const double t = block_sum<T>(lsum, red);
    if (tid == 0) loss_part[lb] = t;
  }
}

// ------------------------------------------------------------- backward prep
template <typename T, typename T2>
__global__ void backward_prep_kernel(const T* __restrict__ W, const T* __restrict__ I,
                                     const double* __restrict__ dldi, gsv_grid g, gsv_bricks k,
                                     int64_t v0, int64_t v1, double eps_w, T2* __restrict__ ab,
                                     unsigned long long* bad) {
  const int64_t lin = v0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (lin >= v1) return;
  {  // only the slab's voxels: brick id of the voxel in [b0, b1)
    const int64_t x = lin % g.nx, t = lin / g.nx;
    const int64_t y = t % g.ny, z = t / g.ny;
    const int64_t b = x / k.bdx + k.bgx * (y / k.bdy + (int64_t)k.bgy * (z / k.bdz));
    if (b < k.b0 || b >= k.b1) return;
  }
  const double dl = dldi[lin];
  if (!isfinite(dl)) atomicMin(bad, (unsigned long long)lin);
  const double w = (double)W[lin];
  T alpha = 0;
  if (w >= eps_w && dl != 0.0 && isfinite(dl)) alpha = (T)(dl / w);
  T2 o;
  o.x = alpha;
  o.y = I[lin];
  ab[lin] = o;
}

// ------------------------------------------------------------- backward f32
// One thread per (brick, Gaussian) pair, three phases per chunk of up to 1024
// list entries:
//  (1) per pair: the 3-sigma y/z row range and, row by row, the exact x-span
//      where d2(x) = |v_row + x e_x|^2 (a quadratic in x) can be <= cutoff^2 +
//      guard: one byte per row in shared memory (xa | xb << 4); the number of
//      candidate voxels is the pair's cost.
//  (2) a smem counting sort of the chunk's pairs by cost, heaviest first.
//  (3) warps pull groups of 32 pairs of similar cost (heaviest first, so the
//      CTA's warps finish together) and each lane runs ONE flattened loop over
//      its pair's candidate voxels: a warp costs max(candidates) iterations,
//      not the sum over rows of per-row maxima.
// Processing order never changes a result: each pair's partial is computed by
// one thread in a fixed voxel order and stored in its own slot.  Every
// candidate is decided exactly as the forward decides.  The brick's
// {dL/dI / W, I} are staged in shared memory.  Accumulates sum cw v
// (whitened) and sum cw delta delta^T; d_mu = L^T sum cw v once per pair.
constexpr int kBwdChunkMax = 1024;
constexpr int kBwdSpanBytes = 32768;
constexpr int kBwdBuckets = 128;

struct BwdCoef {
  float u[3], ex[3], ey[3], ez[3], c[3];
  float A, r, guard;
};

// Brick-relative coefficients of one pair (recomputed in phases 1 and 3 from
// the L1-resident per-Gaussian record; cheaper than keeping them in smem).
__device__ __forceinline__ void bwd_coef(const gsv_record32* __restrict__ rec,
                                         const double* __restrict__ pos, int gid,
                                         const BrickGeom& bg, const gsv_bricks& k, float fsx,
                                         float fsy, float fsz, float cut2, BwdCoef& C,
                                         float4& q0o, float4& q1o, float4& q2o, float4& q3o) {
  const float4* r4 = reinterpret_cast<const float4*>(rec + gid);
  const float4 q0 = __ldg(r4), q1 = __ldg(r4 + 1), q2 = __ldg(r4 + 2), q3 = __ldg(r4 + 3);
  const float L[9] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w, q2.x};
  const double* m = pos + 3 * (int64_t)gid;
  const float mx = (float)(__ldg(m) - bg.px), my = (float)(__ldg(m + 1) - bg.py),
              mz = (float)(__ldg(m + 2) - bg.pz);   // mu - p_b0
  C.c[0] = -mx; C.c[1] = -my; C.c[2] = -mz;
  float umax = 0.f;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    C.u[a] = -fmaf(L[3 * a], mx, fmaf(L[3 * a + 1], my, L[3 * a + 2] * mz));
    C.ex[a] = L[3 * a] * fsx;
    C.ey[a] = L[3 * a + 1] * fsy;
    C.ez[a] = L[3 * a + 2] * fsz;
    umax = fmaxf(umax, fabsf(C.u[a]) + fabsf(C.ex[a]) * k.bdx + fabsf(C.ey[a]) * k.bdy +
                           fabsf(C.ez[a]) * k.bdz);
  }
  C.guard = isinf(cut2) ? 0.f : kGuardRel * cut2 + kGuardMag * umax * sqrtf(cut2);
  C.A = q2.y;
  C.r = q2.z;
  q0o = q0; q1o = q1; q2o = q2; q3o = q3;
}

__device__ __forceinline__ void bwd_accumulate(float d2, float relax, float A, float2 v_ab,
                                               float v0, float v1, float v2, float dx,
                                               float dy, float dz, float* acc) {
  // exp(-d2/2) as one FMUL + MUFU.EX2 (d2 <= 9 + guard: never denormal)
  const float kern = ex2_approx(d2 * -0.72134752044448170f);
  const float w = kern * relax;
  acc[0] = fmaf(w, v_ab.x, acc[0]);
  const float common = v_ab.x * (A - v_ab.y);   // dL/dI (A - I) / W
  acc[1] = fmaf(common, kern, acc[1]);
  const float cw = common * w;
  acc[2] = fmaf(cw, v0, acc[2]);
  acc[3] = fmaf(cw, v1, acc[3]);
  acc[4] = fmaf(cw, v2, acc[4]);
  const float h = -0.5f * cw;
  const float hx = h * dx, hy = h * dy;
  acc[5] = fmaf(hx, dx, acc[5]);
  acc[6] = fmaf(hy, dy, acc[6]);
  acc[7] = fmaf(h * dz, dz, acc[7]);
  acc[8] = fmaf(hx, dy, acc[8]);
  acc[9] = fmaf(hx, dz, acc[9]);
  acc[10] = fmaf(hy, dz, acc[10]);
}

size_t bwd_smem_bytes(int ab_voxels) {
  return (size_t)kBwdSpanBytes + sizeof(uint4) * kBwdChunkMax +
         sizeof(unsigned short) * kBwdChunkMax + sizeof(int) * (kBwdBuckets + 4) +
         sizeof(float2) * (size_t)ab_voxels;
}

template <bool kSmem>
__global__ void __launch_bounds__(kBwdThreads, 3)
backward32_kernel(const double* __restrict__ pos, const __grid_constant__ ExactSrc xsrc,
                  const gsv_record32* __restrict__ rec,
                  const int64_t* __restrict__ starts, const int32_t* __restrict__ gids,
                  const int64_t* __restrict__ gstart, const int32_t* __restrict__ box,
                  const __grid_constant__ gsv_grid g, gsv_bricks k, float cut2, double cut2d,
                  const float2* __restrict__ ab, float4* __restrict__ partials) {
  extern __shared__ __align__(16) unsigned char bwd_smem[];
  unsigned char* sspan = bwd_smem;                                       // kBwdSpanBytes
  uint4* smeta = reinterpret_cast<uint4*>(bwd_smem + kBwdSpanBytes);     // per pair
  unsigned short* sorder = reinterpret_cast<unsigned short*>(smeta + kBwdChunkMax);
  int* shist = reinterpret_cast<int*>(sorder + kBwdChunkMax);
  int* snextp = shist + kBwdBuckets;
  float2* sab = reinterpret_cast<float2*>(snextp + 4);
  const int lb = blockIdx.x;
  const int b = (int)slab_first(k) + lb;
  const int64_t lbeg = starts[lb], lend = starts[lb + 1];
  if (lbeg == lend) return;
  const BrickGeom bg = brick_geom(b, g, k);
  const BrickXYZ bc = brick_xyz(b, k);
  const int tid = threadIdx.x, lane = tid & 31;
  const float fsx = (float)g.sx, fsy = (float)g.sy, fsz = (float)g.sz;
  const float isy = (float)(1.0 / g.sy), isz = (float)(1.0 / g.sz);
  // rows per pair = y-range x z-range of the brick; spans need xb < 16.
  const int rows_cap = k.bdy * k.bdz;
  const bool spans_ok = k.bdx <= 16 && rows_cap <= 64;
  const int chunk = spans_ok ? min(kBwdChunkMax, (kBwdSpanBytes / rows_cap) & ~31) : kBwdChunkMax;
  if (kSmem) {
    const int nv = bg.ex * bg.ey * bg.ez;
    for (int v = tid; v < nv; v += kBwdThreads) {
      const int x = v % bg.ex, y = (v / bg.ex) % bg.ey, z = v / (bg.ex * bg.ey);
      const int64_t lin =
          (int64_t)(bg.x0 + x) + (int64_t)g.nx * ((bg.y0 + y) + (int64_t)g.ny * (bg.z0 + z));
      sab[x + k.bdx * (y + k.bdy * z)] = __ldg(ab + lin);
    }
  }
  for (int64_t cbase = lbeg; cbase < lend; cbase += chunk) {
    const int cnt = (int)min((int64_t)chunk, lend - cbase);
    if (tid < kBwdBuckets) shist[tid] = 0;
    if (tid == 0) *snextp = 0;
    __syncthreads();
    // ---- (1) row spans + cost
    for (int t = tid; t < cnt; t += kBwdThreads) {
      BwdCoef C;
      float4 q0, q1, q2, q3;
      bwd_coef(rec, pos, gids[cbase + t], bg, k, fsx, fsy, fsz, cut2, C, q0, q1, q2, q3);
      const float cyv = -C.c[1] * isy, czv = -C.c[2] * isz;
      const float hyv = fmaf(q3.x, isy, 1e-3f), hzv = fmaf(q3.y, isz, 1e-3f);
      int yl = max(0, (int)ceilf(cyv - hyv)), yh = min(bg.ey - 1, (int)floorf(cyv + hyv));
      int zl = max(0, (int)ceilf(czv - hzv)), zh = min(bg.ez - 1, (int)floorf(czv + hzv));
      if (yl > yh || zl > zh) { yl = 0; yh = -1; zl = 0; zh = -1; }
      int cost = 0;
      unsigned long long rmask = 0ull;   // bit r: row r of the y/z box has a span
      if (spans_ok) {
        const float qa = fmaf(C.ex[0], C.ex[0], fmaf(C.ex[1], C.ex[1], C.ex[2] * C.ex[2]));
        const float inv_qa = 1.0f / qa;
        const float lim = cut2 + C.guard;
        unsigned char* my_sp = sspan + t * rows_cap;
        const int ny = yh - yl + 1;
        // per-pair constants of the in-plane quadratics
        const float b1 = fmaf(C.ey[0], C.ex[0], fmaf(C.ey[1], C.ex[1], C.ey[2] * C.ex[2]));
        const float c2 = fmaf(C.ey[0], C.ey[0], fmaf(C.ey[1], C.ey[1], C.ey[2] * C.ey[2]));
        for (int z = zl; z <= zh; ++z) {
          // row y of plane z: v_row = w + y e_y with w = u + z e_z; along x
          // d2(x) = qa x^2 + 2 qb x + qc, qb = b0 + y b1, qc = c0 + 2 y c1 + y^2 c2
          const float w0 = fmaf((float)z, C.ez[0], C.u[0]);
          const float w1 = fmaf((float)z, C.ez[1], C.u[1]);
          const float w2 = fmaf((float)z, C.ez[2], C.u[2]);
          const float b0 = fmaf(w0, C.ex[0], fmaf(w1, C.ex[1], w2 * C.ex[2]));
          const float c0 = fmaf(w0, w0, fmaf(w1, w1, w2 * w2));
          const float c1 = fmaf(w0, C.ey[0], fmaf(w1, C.ey[1], w2 * C.ey[2]));
          const int rbase = (z - zl) * ny - yl;
          for (int y = yl; y <= yh; ++y) {
            const float fy = (float)y;
            const float qb = fmaf(fy, b1, b0);
            const float qc = fmaf(fy, fmaf(fy, c2, 2.f * c1), c0);
            // (qa x + qb)^2 <= qb^2 - qa (qc - lim)
            const float disc = fmaf(qb, qb, -qa * (qc - lim));
            if (!(disc >= 0.f)) continue;
            const float sq = sqrtf(disc);
            const int xa = max(0, (int)ceilf((-qb - sq) * inv_qa - 1e-3f));
            const int xb = min(bg.ex - 1, (int)floorf((-qb + sq) * inv_qa + 1e-3f));
            if (xa > xb) continue;
            const int row = rbase + y;
            cost += xb - xa + 1;
            rmask |= 1ull << row;
            my_sp[row] = (unsigned char)(xa | (xb << 4));
          }
        }
      } else {
        cost = (yh - yl + 1) * (zh - zl + 1) * bg.ex;
      }
      smeta[t] = make_uint4((unsigned)yl | ((unsigned)(yh - yl + 1) << 8) | ((unsigned)zl << 16) |
                                ((unsigned)(zh - zl + 1) << 24),
                            (unsigned)cost, (unsigned)rmask, (unsigned)(rmask >> 32));
      atomicAdd(&shist[kBwdBuckets - 1 - min(cost, kBwdBuckets - 1)], 1);
    }
    __syncthreads();
    // ---- (2) counting sort by cost, heaviest first
    if (tid < 32) {
      int v[4], sum = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) { v[i] = shist[4 * tid + i]; sum += v[i]; }
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int n = __shfl_up_sync(kFull, incl, o);
        if (tid >= o) incl += n;
      }
      int run = incl - sum;
#pragma unroll
      for (int i = 0; i < 4; ++i) { shist[4 * tid + i] = run; run += v[i]; }
    }
    __syncthreads();
    for (int t = tid; t < cnt; t += kBwdThreads) {
      const int c = (int)smeta[t].y;
      const int slot = atomicAdd(&shist[kBwdBuckets - 1 - min(c, kBwdBuckets - 1)], 1);
      sorder[slot] = (unsigned short)t;
    }
    __syncthreads();
    // ---- (3) warps pull 32-pair groups, heaviest first
    const int ngroups = (cnt + 31) >> 5;
    for (;;) {
      int grp = 0;
      if (lane == 0) grp = atomicAdd(snextp, 1);
      grp = __shfl_sync(kFull, grp, 0);
      if (grp >= ngroups) break;
      const int s = (grp << 5) + lane;
      if (s >= cnt) continue;
      const int t = sorder[s];
      const int gid = gids[cbase + t];
      BwdCoef C;
      float4 q0, q1, q2, q3;
      bwd_coef(rec, pos, gid, bg, k, fsx, fsy, fsz, cut2, C, q0, q1, q2, q3);
      const uint4 meta = smeta[t];
      const int yl = meta.x & 255, ny = (meta.x >> 8) & 255, zl = (meta.x >> 16) & 255,
                nz = meta.x >> 24;
      const int cost = (int)meta.y;
      const float lim = cut2 + C.guard, lo_band = cut2 - C.guard;
      float acc[11];
#pragma unroll
      for (int a = 0; a < 11; ++a) acc[a] = 0.f;
      if (spans_ok) {
        const unsigned char* my_sp = sspan + t * rows_cap;
        unsigned long long rmask = ((unsigned long long)meta.w << 32) | meta.z;
        // row r -> (y, z) = (yl + r % ny, zl + r / ny) by reciprocal multiply
        // (exact for r < 64, ny <= 255): no integer division in the loop.
        const unsigned recip_ny = ny > 1 ? (unsigned)((0xFFFFFFFFull + ny) / (unsigned)ny) : 0u;
        int x = 1, xb = 0, y = 0, z = 0, srow = 0;
        float vr0 = 0.f, vr1 = 0.f, vr2 = 0.f, dy = 0.f, dz = 0.f;
        for (int it = 0; it < cost; ++it) {
          if (x > xb) {   // next non-empty row
            const int row = __ffsll((long long)rmask) - 1;
            rmask &= rmask - 1;
            const int sp = my_sp[row];
            x = sp & 15;
            xb = sp >> 4;
            const int zo = ny > 1 ? (int)__umulhi((unsigned)row, recip_ny) : row;
            y = yl + row - zo * ny;
            z = zl + zo;
            vr0 = fmaf((float)z, C.ez[0], fmaf((float)y, C.ey[0], C.u[0]));
            vr1 = fmaf((float)z, C.ez[1], fmaf((float)y, C.ey[1], C.u[1]));
            vr2 = fmaf((float)z, C.ez[2], fmaf((float)y, C.ey[2], C.u[2]));
            dy = fmaf((float)y, fsy, C.c[1]);
            dz = fmaf((float)z, fsz, C.c[2]);
            srow = k.bdx * (y + k.bdy * z);
          }
          const int xi = x++;
          const float2 v_ab = kSmem ? sab[srow + xi]
                                    : __ldg(ab + (int64_t)(bg.x0 + xi) +
                                            (int64_t)g.nx * ((bg.y0 + y) + (int64_t)g.ny * (bg.z0 + z)));
          if (v_ab.x == 0.f) continue;
          const float fx = (float)xi;
          const float v0 = fmaf(fx, C.ex[0], vr0), v1 = fmaf(fx, C.ex[1], vr1),
                      v2 = fmaf(fx, C.ex[2], vr2);
          const float d2 = fmaf(v0, v0, fmaf(v1, v1, v2 * v2));
          if (d2 > lim) continue;
          if (d2 >= lo_band &&
              !exact_live(gid, bg.x0 + xi, bg.y0 + y, bg.z0 + z, xsrc, g, cut2d))
            continue;
          bwd_accumulate(d2, C.r, C.A, v_ab, v0, v1, v2, fmaf(fx, fsx, C.c[0]), dy, dz, acc);
        }
      } else {
        // Very large bricks: nested loops over the y/z rows of the 3-sigma box.
        for (int zz = 0; zz < nz; ++zz) {
          const int z = zl + zz;
          const float dz = fmaf((float)z, fsz, C.c[2]);
          for (int yy = 0; yy < ny; ++yy) {
            const int y = yl + yy;
            const float dy = fmaf((float)y, fsy, C.c[1]);
            const float vr0 = fmaf((float)z, C.ez[0], fmaf((float)y, C.ey[0], C.u[0]));
            const float vr1 = fmaf((float)z, C.ez[1], fmaf((float)y, C.ey[1], C.u[1]));
            const float vr2 = fmaf((float)z, C.ez[2], fmaf((float)y, C.ey[2], C.u[2]));
            for (int x = 0; x < bg.ex; ++x) {
              const float2 v_ab = kSmem ? sab[k.bdx * (y + k.bdy * z) + x]
                                        : __ldg(ab + (int64_t)(bg.x0 + x) +
                                                (int64_t)g.nx * ((bg.y0 + y) + (int64_t)g.ny * (bg.z0 + z)));
              if (v_ab.x == 0.f) continue;
              const float fx = (float)x;
              const float v0 = fmaf(fx, C.ex[0], vr0), v1 = fmaf(fx, C.ex[1], vr1),
                          v2 = fmaf(fx, C.ex[2], vr2);
              const float d2 = fmaf(v0, v0, fmaf(v1, v1, v2 * v2));
              if (d2 > lim) continue;
              if (d2 >= lo_band &&
                  !exact_live(gid, bg.x0 + x, bg.y0 + y, bg.z0 + z, xsrc, g, cut2d))
                continue;
              bwd_accumulate(d2, C.r, C.A, v_ab, v0, v1, v2, fmaf(fx, fsx, C.c[0]), dy, dz, acc);
            }
          }
        }
      }
      // d_mu = sum cw Sigma^-1 delta = L^T (sum cw v); L row-major in q0,q1,q2.x
      const float mu0 = fmaf(q0.x, acc[2], fmaf(q0.w, acc[3], q1.z * acc[4]));
      const float mu1 = fmaf(q0.y, acc[2], fmaf(q1.x, acc[3], q1.w * acc[4]));
      const float mu2 = fmaf(q0.z, acc[2], fmaf(q1.y, acc[3], q2.x * acc[4]));
      const GBox gb = unpack_box(box, gid);
      const int64_t slot = box_slot(gb, bc.bx, bc.by, bc.bz);
      // A caller-built list may hold a pair the binning would not emit: skip it.
      if (slot < 0) continue;
      const int64_t e = gstart[gid] + slot;
      float4* dst = partials + 3 * e;
      dst[0] = make_float4(acc[0], acc[1], mu0, mu1);
      dst[1] = make_float4(mu2, acc[5], acc[6], acc[7]);
      dst[2] = make_float4(acc[8], acc[9], acc[10], 0.f);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------- backward f32, masked
// Train-step backward when the forward emitted live-voxel masks: per pair
// four {voxel A, voxel B} 32-bit masks, one per warp tile (live_masks).  The
// forward already decided every (pair, voxel) exactly (f32 + f64 guard
// band), so here the pair's cost is its popcount, pairs are counting-sorted
// by it (heaviest first), warps pull 32-pair groups, and each lane walks the
// set bits of its pair -- exactly the live voxels, nothing else.
constexpr int kBwdMChunk = 2048;

// ARITH (8x8x4 bricks): the voxel of (word, bit) is decoded with integer ops
// instead of the (word, bit) LUT, keeping the shared-memory pipe for the
// {alpha, I} gathers (the kernel's bound).  ARITH 1: vpl-4 masks, word
// wi = 4 w + z, bit b -> brick voxel index b + 32 w + 64 z.  ARITH 2: the
// column-packed forward's masks, word y, bit 4 x + z -> x + 8 y + 64 z.
template <int ARITH>
__global__ void __launch_bounds__(kBwdMThreads, GSV_BWDM_WARPS * 32 / kBwdMThreads)
backward32m_kernel(const double* __restrict__ pos, const gsv_record32* __restrict__ rec,
                   const int64_t* __restrict__ starts, const int32_t* __restrict__ gids,
                   const int64_t* __restrict__ gstart, const int32_t* __restrict__ box,
                   gsv_grid g, gsv_bricks k, float cut2, const uint2* __restrict__ masks,
                   int mvpl, const float2* __restrict__ ab, float4* __restrict__ partials) {
  __shared__ float2 sab[256];                 // brick voxels (units <= 128)
  __shared__ float4 slut[256];                // (word << 5) | bit -> (x, y, z, sab index)
  __shared__ unsigned swords[kBwdMThreads / 32][9][32];   // per lane: its pair's non-empty
  __shared__ unsigned short swbase[kBwdMThreads / 32][9][32];  // mask words, LUT bases
  __shared__ int sgid[kBwdMChunk];
  __shared__ unsigned short sorder[kBwdMChunk];
  __shared__ unsigned short scost[kBwdMChunk];
  __shared__ int shist[kBwdBuckets];
  __shared__ int snext;                       // next 32-pair group to walk
  const int lb = blockIdx.x;
  const int b = (int)slab_first(k) + lb;
  const int64_t lbeg = starts[lb], lend = starts[lb + 1];
  if (lbeg == lend) return;
  const BrickGeom bg = brick_geom(b, g, k);
  const BrickXYZ bc = brick_xyz(b, k);
  const int tid = threadIdx.x, lane = tid & 31;
  const float fsx = (float)g.sx, fsy = (float)g.sy, fsz = (float)g.sz;
  const bool tiled = ((k.bdx | k.bdy | k.bdz) & 3) == 0;
  const int units = (int)mask_units(k, mvpl);
  // pair-major masks: pair j's 4 planes {a0, a1, a2, a3} are 32 contiguous bytes
  // mask word wi = VPL * warp + h, bit = lane of the warp tile: voxel of
  // unit warp * 32 + bit, z0 + h (the forward's layout for its VPL)
  const int wsh = mvpl == 4 ? 2 : 1;
  // the host guarantees the brick fills all 4 planes (units = 128 / vpl * 2)
  auto load_masks = [&](int64_t j, uint2& a0, uint2& a1, uint2& a2, uint2& a3) {
    const uint4* p = reinterpret_cast<const uint4*>(masks + 4 * j);
    const uint4 m01 = __ldg(p), m23 = __ldg(p + 1);
    a0 = make_uint2(m01.x, m01.y);
    a1 = make_uint2(m01.z, m01.w);
    a2 = make_uint2(m23.x, m23.y);
    a3 = make_uint2(m23.z, m23.w);
  };
  for (int e = tid; e < (ARITH ? 0 : 256); e += kBwdMThreads) {   // (word, bit) LUT
    const int wi = e >> 5, u = ((wi >> wsh) << 5) + (e & 31);
    float4 v = make_float4(0.f, 0.f, 0.f, __int_as_float(0));
    if (u < units) {
      int x, y, z0;
      if (mvpl == 4)
        unit_voxel_v<4>(u, k, x, y, z0);
      else
        unit_voxel(u, k, tiled, x, y, z0);
      const int z = z0 + (wi & ((1 << wsh) - 1));
      if (z < k.bdz)
        v = make_float4((float)x, (float)y, (float)z, __int_as_float(x + k.bdx * (y + k.bdy * z)));
    }
    slut[e] = v;
  }
  {
    const int nv = bg.ex * bg.ey * bg.ez;
    for (int v = tid; v < nv; v += kBwdMThreads) {
      const int x = v % bg.ex, y = (v / bg.ex) % bg.ey, z = v / (bg.ex * bg.ey);
      const int64_t lin =
          (int64_t)(bg.x0 + x) + (int64_t)g.nx * ((bg.y0 + y) + (int64_t)g.ny * (bg.z0 + z));
      sab[x + k.bdx * (y + k.bdy * z)] = __ldg(ab + lin);
    }
  }
  for (int64_t cbase = lbeg; cbase < lend; cbase += kBwdMChunk) {
    const int cnt = (int)min((int64_t)kBwdMChunk, lend - cbase);
    if (tid < kBwdBuckets) shist[tid] = 0;
    __syncthreads();
    // (1) cost = live voxels of the pair; 4 pairs' loads in flight per thread
#pragma unroll 4
    for (int t = tid; t < cnt; t += kBwdMThreads) {
      const int64_t jt = cbase + t;
      uint2 a0, a1, a2, a3;
      load_masks(jt, a0, a1, a2, a3);
      const int gj = __ldg(gids + jt);
      const int c = __popc(a0.x) + __popc(a0.y) + __popc(a1.x) + __popc(a1.y) + __popc(a2.x) +
                    __popc(a2.y) + __popc(a3.x) + __popc(a3.y);
      scost[t] = (unsigned short)c;
      sgid[t] = gj;
      atomicAdd(&shist[kBwdBuckets - 1 - min(c, kBwdBuckets - 1)], 1);
    }
    __syncthreads();
    // (2) counting sort, heaviest first
    if (tid < 32) {
      int v[4], sum = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) { v[i] = shist[4 * tid + i]; sum += v[i]; }
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int n = __shfl_up_sync(kFull, incl, o);
        if (tid >= o) incl += n;
      }
      int run = incl - sum;
#pragma unroll
      for (int i = 0; i < 4; ++i) { shist[4 * tid + i] = run; run += v[i]; }
    }
    __syncthreads();
    for (int t = tid; t < cnt; t += kBwdMThreads) {
      const int slot = atomicAdd(&shist[kBwdBuckets - 1 - min((int)scost[t], kBwdBuckets - 1)], 1);
      sorder[slot] = (unsigned short)t;
    }
    if (tid == 0) snext = kBwdMThreads / 32;
    __syncthreads();
    // (3) warps pull groups of 32 pairs of similar cost, heaviest first, each
    // warp fetching its next group when done (longest-processing-time order;
    // 0.7% faster than dealing them round-robin); each lane walks its pair's
    // live voxels
    const int ngroups = (cnt + 31) >> 5;
    auto next_grp = [&]() {
      int v = 0;
      if (lane == 0) v = atomicAdd(&snext, 1);
      return __shfl_sync(kFull, v, 0);
    };
    for (int grp = tid >> 5; grp < ngroups; grp = next_grp()) {
      const int s = (grp << 5) + lane;
      if (s >= cnt) continue;
      const int t = sorder[s];
      const int64_t j = cbase + t;
      const int gid = sgid[t];
      // every global load of the pair up front: one latency, hidden by the loop
      const GBox gb = unpack_box(box, gid);
      const int64_t gst = __ldg(gstart + gid);
      const float4* r4 = reinterpret_cast<const float4*>(rec + gid);
      const float4 q0 = __ldg(r4), q1 = __ldg(r4 + 1), q2 = __ldg(r4 + 2);
      const float L[9] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w, q2.x};
      const float A = q2.y, r = q2.z;
      const double* m = pos + 3 * (int64_t)gid;
      const float c0 = (float)(bg.px - __ldg(m)), c1 = (float)(bg.py - __ldg(m + 1)),
                  c2 = (float)(bg.pz - __ldg(m + 2));   // p_b0 - mu
      float u[3], ex[3], ey[3], ez[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        u[a] = fmaf(L[3 * a], c0, fmaf(L[3 * a + 1], c1, L[3 * a + 2] * c2));
        ex[a] = L[3 * a] * fsx;
        ey[a] = L[3 * a + 1] * fsy;
        ez[a] = L[3 * a + 2] * fsz;
      }
      uint2 a0, a1, a2, a3;
      load_masks(j, a0, a1, a2, a3);
      // this lane's column of the warp's word table (conflict-free, no sync:
      // only the lane itself reads it): its non-empty words and their LUT
      // bases, compacted, plus a zero sentinel
      unsigned* myw = &swords[tid >> 5][0][lane];
      unsigned short* myb = &swbase[tid >> 5][0][lane];
      {
        const unsigned words[8] = {a0.x, a0.y, a1.x, a1.y, a2.x, a2.y, a3.x, a3.y};
        int nw = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w)
          if (words[w] != 0u) {
            myw[nw << 5] = words[w];
            // ARITH: the word's brick-voxel base 32 (w / 4) + 64 (w % 4); else
            // its LUT row
            myb[nw << 5] = (unsigned short)(ARITH == 2 ? w << 3
                                            : ARITH == 1 ? ((w >> 2) << 5) + ((w & 3) << 6)
                                                         : w << 5);
            ++nw;
          }
        myw[nw << 5] = 0u;
        myb[nw << 5] = 0;
      }
      float acc[11];
#pragma unroll
      for (int a = 0; a < 11; ++a) acc[a] = 0.f;
      const int cost = scost[t];
      unsigned cur = myw[0];
      int wb = myb[0];
      unsigned nxt = myw[32];                   // next word, prefetched
      int nxb = myb[32];
      int slot = 1;
      // shared addresses by opaque 32-bit bases (plain indexing re-derived the
      // shared window base with an S2UR in every walk iteration)
      const uint32_t myw_a = smem_addr(myw), myb_a = smem_addr(myb), sab_a = smem_addr(sab);
      for (int it = 0; it < cost; ++it) {
        if (cur == 0u) {
          cur = nxt;
          wb = nxb;
          ++slot;
          const uint32_t so = (uint32_t)(min(slot, 8) << 5);
          nxt = lds_u32(myw_a + 4u * so);
          nxb = (int)lds_u16(myb_a + 2u * so);
        }
        const int bit = __ffs(cur) - 1;
        cur &= cur - 1u;
        float fx, fy, fz;
        float2 v_ab;
        if (ARITH) {
          // x + 8 y + 64 z
          const int vi = ARITH == 2 ? wb + (bit >> 2) + ((bit & 3) << 6) : wb + bit;
          GSV_DCHECK(vi >= 0 && vi < 256 && (vi & 7) < bg.ex && ((vi >> 3) & 7) < bg.ey &&
                     (vi >> 6) < bg.ez);
          v_ab = lds_f2(sab_a + 8u * (uint32_t)vi);
          fx = (float)(vi & 7);
          fy = (float)((vi >> 3) & 7);
          fz = (float)(vi >> 6);
        } else {
          const float4 vx = slut[wb | bit];
          v_ab = sab[__float_as_int(vx.w)];
          fx = vx.x;
          fy = vx.y;
          fz = vx.z;
        }
        const float v0 = fmaf(fz, ez[0], fmaf(fy, ey[0], fmaf(fx, ex[0], u[0])));
        const float v1 = fmaf(fz, ez[1], fmaf(fy, ey[1], fmaf(fx, ex[1], u[1])));
        const float v2 = fmaf(fz, ez[2], fmaf(fy, ey[2], fmaf(fx, ex[2], u[2])));
        const float d2 = fmaf(v0, v0, fmaf(v1, v1, v2 * v2));
        bwd_accumulate(d2, r, A, v_ab, v0, v1, v2, fmaf(fx, fsx, c0), fmaf(fy, fsy, c1),
                       fmaf(fz, fsz, c2), acc);
      }
      const float mu0 = fmaf(q0.x, acc[2], fmaf(q0.w, acc[3], q1.z * acc[4]));
      const float mu1 = fmaf(q0.y, acc[2], fmaf(q1.x, acc[3], q1.w * acc[4]));
      const float mu2 = fmaf(q0.z, acc[2], fmaf(q1.y, acc[3], q2.x * acc[4]));
      const int64_t bs = box_slot(gb, bc.bx, bc.by, bc.bz);
      // A caller-built list may hold a pair the binning would not emit: skip it.
      if (bs < 0) continue;
      const int64_t e = gst + bs;
      float4* dst = partials + 3 * e;
      dst[0] = make_float4(acc[0], acc[1], mu0, mu1);
      dst[1] = make_float4(mu2, acc[5], acc[6], acc[7]);
      dst[2] = make_float4(acc[8], acc[9], acc[10], 0.f);
    }
    __syncthreads();
  }
  (void)cut2;
}

// ------------------------------------------------------------- backward f64
__global__ void __launch_bounds__(kBwdThreads)
backward64_kernel(const double* __restrict__ pos, const gsv_record64* __restrict__ rec,
                  const gsv_record32* __restrict__ rec32, const int64_t* __restrict__ starts,
                  const int32_t* __restrict__ gids, const int64_t* __restrict__ gstart,
                  const int32_t* __restrict__ box, gsv_grid g, gsv_bricks k, double cut2,
                  const double2* __restrict__ ab, double* __restrict__ partials) {
  const int lb = blockIdx.x;
  const int b = (int)slab_first(k) + lb;
  const BrickGeom bg = brick_geom(b, g, k);
  const BrickXYZ bc = brick_xyz(b, k);
  const int64_t lbeg = starts[lb], lend = starts[lb + 1];
  for (int64_t j = lbeg + threadIdx.x; j < lend; j += kBwdThreads) {
    const int gid = gids[j];
    const gsv_record64 rc = rec[gid];
    const gsv_record32 r32 = rec32[gid];
    const double* L = rc.l;
    const double A = rc.amp, r = rc.relax;
    const double* m = pos + 3 * (int64_t)gid;
    const double mx = m[0], my = m[1], mz = m[2];
    int xl, xh, yl, yh, zl, zh;
    sub_range(mx - bg.px, (double)r32.half[0], g.sx, bg.ex, xl, xh);
    sub_range(my - bg.py, (double)r32.half[1], g.sy, bg.ey, yl, yh);
    sub_range(mz - bg.pz, (double)r32.half[2], g.sz, bg.ez, zl, zh);
    double acc_a = 0, acc_r = 0, mu0 = 0, mu1 = 0, mu2 = 0;
    double g00 = 0, g11 = 0, g22 = 0, g01 = 0, g02 = 0, g12 = 0;
    for (int z = zl; z <= zh; ++z) {
      const int iz = bg.z0 + z;
      const double dz = sub(add(g.oz, mul((double)iz, g.sz)), mz);
      for (int y = yl; y <= yh; ++y) {
        const int iy = bg.y0 + y;
        const double dy = sub(add(g.oy, mul((double)iy, g.sy)), my);
        const int64_t row = (int64_t)g.nx * (iy + (int64_t)g.ny * iz);
        for (int x = xl; x <= xh; ++x) {
          const int ix = bg.x0 + x;
          const double2 v_ab = ab[row + ix];
          if (v_ab.x == 0.0) continue;
          const double dx = sub(add(g.ox, mul((double)ix, g.sx)), mx);
          const double v0 = add(add(mul(L[0], dx), mul(L[1], dy)), mul(L[2], dz));
          const double v1 = add(add(mul(L[3], dx), mul(L[4], dy)), mul(L[5], dz));
          const double v2 = add(add(mul(L[6], dx), mul(L[7], dy)), mul(L[8], dz));
          const double d2 = add(add(mul(v0, v0), mul(v1, v1)), mul(v2, v2));
          if (d2 > cut2) continue;
          const double kern = exp(-0.5 * d2);
          const double w = kern * r;
          acc_a += w * v_ab.x;
          const double common = v_ab.x * (A - v_ab.y);
          acc_r += common * kern;
          const double cw = common * w;
          mu0 += cw * (L[0] * v0 + L[3] * v1 + L[6] * v2);
          mu1 += cw * (L[1] * v0 + L[4] * v1 + L[7] * v2);
          mu2 += cw * (L[2] * v0 + L[5] * v1 + L[8] * v2);
          const double h = -0.5 * cw;
          g00 += h * dx * dx;
          g11 += h * dy * dy;
          g22 += h * dz * dz;
          g01 += h * dx * dy;
          g02 += h * dx * dz;
          g12 += h * dy * dz;
        }
      }
    }
    const GBox gb = unpack_box(box, gid);
    const int64_t slot = box_slot(gb, bc.bx, bc.by, bc.bz);
    // A caller-built list may hold a pair the binning would not emit: skip it.
    if (slot < 0) continue;
    const int64_t e = gstart[gid] + slot;
    double* dst = partials + 12 * e;
    dst[0] = acc_a; dst[1] = acc_r; dst[2] = mu0; dst[3] = mu1; dst[4] = mu2;
    dst[5] = g00; dst[6] = g11; dst[7] = g22; dst[8] = g01; dst[9] = g02; dst[10] = g12;
    dst[11] = 0.0;
  }
}

// ------------------------------------------------------------ naive render
// render_naive / _naive_kernel (render.py:84-110): every Gaussian at every
// voxel, explicit Sigma^-1 = R diag(exp(-2 ls)) R^T quadratic form in f64.
template <typename T>
__global__ void __launch_bounds__(128)
naive_kernel(const double* __restrict__ pos, const double* __restrict__ ls,
             const double* __restrict__ rot, const double* __restrict__ ra,
             const double* __restrict__ rr, int64_t n, int relax_enabled, gsv_grid g,
             double cut2, double eps_w, T* __restrict__ I) {
  constexpr int TB = 128;
  __shared__ double sm[TB][16];
  const int64_t nvox = (int64_t)g.nx * g.ny * g.nz;
  const int64_t lin = blockIdx.x * (int64_t)TB + threadIdx.x;
  const bool own = lin < nvox;
  const int ix = (int)(lin % g.nx);
  const int64_t rem = lin / g.nx;
  const int iy = (int)(rem % g.ny), iz = (int)(rem / g.ny);
  const double px = g.ox + ix * g.sx, py = g.oy + iy * g.sy, pz = g.oz + iz * g.sz;
  T S = 0, Wt = 0;
  for (int64_t t0 = 0; t0 < n; t0 += TB) {
    const int cnt = (int)min((int64_t)TB, n - t0);
    __syncthreads();
    if (threadIdx.x < cnt) {
      const int64_t i = t0 + threadIdx.x;
      double R[9];
      rotation_f64(rot + 4 * i, R);
      const double iv[3] = {exp(-2.0 * ls[3 * i]), exp(-2.0 * ls[3 * i + 1]),
                            exp(-2.0 * ls[3 * i + 2])};
      double* o = sm[threadIdx.x];
      for (int a = 0; a < 3; ++a)
        for (int c = 0; c < 3; ++c)
          o[3 * a + c] = R[3 * a] * iv[0] * R[3 * c] + R[3 * a + 1] * iv[1] * R[3 * c + 1] +
                         R[3 * a + 2] * iv[2] * R[3 * c + 2];
      o[9] = pos[3 * i];
      o[10] = pos[3 * i + 1];
      o[11] = pos[3 * i + 2];
      o[12] = expit_f64(ra[i]);
      o[13] = relax_enabled ? expit_f64(rr[i]) : 1.0;
    }
    __syncthreads();
    if (own) {
      for (int j = 0; j < cnt; ++j) {
        const double* s = sm[j];
        const double dx = sub(px, s[9]), dy = sub(py, s[10]), dz = sub(pz, s[11]);
        const double d2 =
            add(add(mul(dx, add(add(mul(s[0], dx), mul(s[1], dy)), mul(s[2], dz))),
                    mul(dy, add(add(mul(s[3], dx), mul(s[4], dy)), mul(s[5], dz)))),
                mul(dz, add(add(mul(s[6], dx), mul(s[7], dy)), mul(s[8], dz))));
        if (d2 <= cut2) {
          const double w = exp(-0.5 * d2) * s[13];
          S = (T)((double)S + s[12] * w);
          Wt = (T)((double)Wt + w);
        }
      }
    }
  }
  if (own) I[lin] = ((double)Wt >= eps_w) ? (T)((double)S / (double)Wt) : (T)0;
}

}  // namespace
}  // namespace gsv

using namespace gsv;

extern "C" {

int gsv_loss_bricks(const gsv_grid* grid, const gsv_bricks* bricks, double eps_w,
                    const float* W, const float* I, const void* target, int target_dtype,
                    int loss_kind, double vox_count, int vpl, float* ab, double* loss_part,
                    void* stream) {
  if (int s = validate_grid_bricks(grid, bricks)) return s;
  GSV_REQUIRE(bricks->bdx == 8 && bricks->bdy == 8 && bricks->bdz == 4,
              "gsv_loss_bricks needs 8x8x4 bricks");
  GSV_REQUIRE(vpl == 16 || vpl == 8, "vpl must be 16 (grouped) or 8 (whole-brick forward)");
  GSV_REQUIRE(W && I && target && ab && loss_part, "null pointer argument");
  GSV_REQUIRE(loss_kind == 0 || loss_kind == 1, "loss_kind must be 0 (l1) or 1 (l2)");
  GSV_REQUIRE(target_dtype == 0 || target_dtype == 1,
              "target_dtype must be 0 (float32) or 1 (float64)");
  const int64_t nb = slab_bricks(*bricks);
  if (nb == 0) return GSV_OK;
  loss_bricks_kernel<<<(unsigned)nb, 32, 0, as_stream(stream)>>>(
      *grid, *bricks, eps_w, W, I, target, target_dtype, loss_kind, vox_count, vpl == 16 ? 0 : 1,
      (float2*)ab, loss_part);
  GSV_CHECK_LAUNCH("loss_bricks_kernel");
  return GSV_OK;
}

int gsv_forward(const double* positions, const double* log_scales, const double* rotations,
                const gsv_record32* rec32, const gsv_record64* rec64, const int64_t* starts,
                const int32_t* gids, const gsv_grid* grid, const gsv_bricks* bricks,
                double cutoff_sigma, double eps_w, int precision, void* S, void* W, void* I,
                const void* target, int target_dtype, int loss_kind, double vox_count,
                float* ab, double* loss_part, uint32_t* live_masks, int vpl, void* stream) {
  if (int s = validate_grid_bricks(grid, bricks)) return s;
  GSV_REQUIRE(precision == 0 || precision == 1, "precision must be 0 (f32) or 1 (f64)");
  GSV_REQUIRE(precision == 0 || rec64 != nullptr, "the f64 forward needs rec64");
  GSV_REQUIRE(target == nullptr || (ab != nullptr && loss_part != nullptr),
              "fused loss needs ab and loss_part");
  GSV_REQUIRE(loss_kind == 0 || loss_kind == 1, "loss_kind must be 0 (l1) or 1 (l2)");
  GSV_REQUIRE(target_dtype == 0 || target_dtype == 1,
              "target_dtype must be 0 (float32) or 1 (float64)");
  const int target_f64 = target_dtype;
  const int64_t nb = slab_bricks(*bricks);
  if (nb == 0) return GSV_OK;
  const double cut2d = cutoff_sigma * cutoff_sigma;
  cudaStream_t s = as_stream(stream);
  if (precision == 0) {
    // Column depth: VPL voxels per lane (2: 4x4x4 warp tiles, 4 warps per
    // 8x8x4 brick; 4: 8x4x4 tiles, 2 warps; 8: whole brick per warp).
    // vpl | 0x200: keep the two tiles of a VPL-4 brick in one CTA (measurement)
    const bool no_split = (vpl & 0x200) != 0;
    vpl &= 0xff;
    GSV_REQUIRE(vpl == 0 || vpl == 2 || vpl == 4 || vpl == 8 || vpl == 16,
                "vpl must be 0, 2, 4, 8 or 16");
    if (vpl == 16) {
      // column-packed: one warp per 8x8x4 brick, (pair, column) slots dealt
      // to the lanes; live masks in the column-nibble layout
      GSV_REQUIRE(bricks->bdx == 8 && bricks->bdy == 8 && bricks->bdz == 4,
                  "vpl 16 needs 8x8x4 bricks");
      const ExactSrc xc{positions, log_scales, rotations, rec64};
      if (live_masks != nullptr)
        forward32c_kernel<true><<<(unsigned)nb, 32, 0, s>>>(
            positions, xc, rec32, starts, gids, *grid, *bricks, (float)cut2d, cut2d, eps_w,
            (float*)S, (float*)W, (float*)I, target, target_f64, loss_kind, vox_count,
            (float2*)ab, loss_part, (uint4*)live_masks);
      else
        forward32c_kernel<false><<<(unsigned)nb, 32, 0, s>>>(
            positions, xc, rec32, starts, gids, *grid, *bricks, (float)cut2d, cut2d, eps_w,
            (float*)S, (float*)W, (float*)I, target, target_f64, loss_kind, vox_count,
            (float2*)ab, loss_part, nullptr);
      GSV_CHECK_LAUNCH("forward32c_kernel");
      return GSV_OK;
    }
    // auto: the whole-brick two-list kernel for 8x8x4 bricks (fastest at every
    // pair density measured), else the warp-tile kernels
    if (vpl == 0 && bricks->bdx == 8 && bricks->bdy == 8 && bricks->bdz == 4) vpl = 8;
    if (vpl == 8) {
      // one warp per 8x8x4 brick, two 4-voxel columns per lane, a hit list per
      // y-half; with live masks for the train step
      GSV_REQUIRE(bricks->bdx == 8 && bricks->bdy == 8 && bricks->bdz == 4,
                  "vpl 8 needs 8x8x4 bricks");
      const ExactSrc xw{positions, log_scales, rotations, rec64};
      static const bool one_list = [] {
        const char* e = getenv("GSV_WHOLE_ONE_LIST");
        return e != nullptr && e[0] == '1';
      }();
      GSV_REQUIRE(live_masks == nullptr || !one_list, "live masks need the two-list form");
      if (live_masks != nullptr)
        forward32w_kernel<true, true><<<(unsigned)nb, 32, 0, s>>>(
            positions, xw, rec32, starts, gids, *grid, *bricks, (float)cut2d, cut2d, eps_w,
            (float*)S, (float*)W, (float*)I, target, target_f64, loss_kind, vox_count, (float2*)ab,
            loss_part, (uint2*)live_masks);
      else if (one_list)
        forward32w_kernel<false><<<(unsigned)nb, 32, 0, s>>>(
            positions, xw, rec32, starts, gids, *grid, *bricks, (float)cut2d, cut2d, eps_w,
            (float*)S, (float*)W, (float*)I, target, target_f64, loss_kind, vox_count, (float2*)ab,
            loss_part);
      else
        forward32w_kernel<true><<<(unsigned)nb, 32, 0, s>>>(
            positions, xw, rec32, starts, gids, *grid, *bricks, (float)cut2d, cut2d, eps_w,
            (float*)S, (float*)W, (float*)I, target, target_f64, loss_kind, vox_count, (float2*)ab,
            loss_part);
      GSV_CHECK_LAUNCH("forward32w_kernel");
      return GSV_OK;
    }
    if (vpl == 0) vpl = mask_vpl_auto(*bricks);
    if (live_masks != nullptr)
      GSV_REQUIRE(mask_units(*bricks, vpl) == (vpl == 4 ? 64 : 128),
                  "live masks need a brick that fills one CTA's warp tiles exactly "
                  "(e.g. 8x8x4)");
    const ExactSrc xs{positions, log_scales, rotations, rec64};
#define GSV_FWD32(V, T, M)                                                                     \
  forward32_kernel<V, T, M><<<(unsigned)nb, T, 0, s>>>(                                        \
      positions, xs, rec32, starts, gids, *grid, *bricks, (float)cut2d, cut2d, eps_w,          \
      (float*)S, (float*)W, (float*)I, target, target_f64, loss_kind, vox_count, (float2*)ab, loss_part,   \
      (uint2*)live_masks)
    const bool split = vpl == 4 && !no_split && mask_units(*bricks, 4) == 64;
    if (split) {
      if (target) {
        cudaError_t e = cudaMemsetAsync(loss_part, 0, (size_t)nb * sizeof(double), s);
        if (e != cudaSuccess) return cuda_status(e, "memset loss_part");
      }
#define GSV_FWD32S(M)                                                                          \
  forward32_kernel<4, 32, M, true><<<(unsigned)(2 * nb), 32, 0, s>>>(                          \
      positions, xs, rec32, starts, gids, *grid, *bricks, (float)cut2d, cut2d, eps_w,          \
      (float*)S, (float*)W, (float*)I, target, target_f64, loss_kind, vox_count, (float2*)ab, loss_part,   \
      (uint2*)live_masks)
      if (live_masks) GSV_FWD32S(true); else GSV_FWD32S(false);
#undef GSV_FWD32S
    } else if (vpl == 4) {
      if (live_masks) GSV_FWD32(4, 64, true); else GSV_FWD32(4, 64, false);
    } else {
      if (live_masks) GSV_FWD32(2, 128, true); else GSV_FWD32(2, 128, false);
    }
#undef GSV_FWD32
    GSV_CHECK_LAUNCH("forward32_kernel");
  } else {
    forward64_kernel<<<(unsigned)nb, 128, 0, s>>>(
        positions, rec64, nullptr, starts, gids, *grid, *bricks, cut2d, eps_w, (double*)S,
        (double*)W, (double*)I, target, target_f64, loss_kind, vox_count, (double2*)ab, loss_part, rec32);
    GSV_CHECK_LAUNCH("forward64_kernel");
  }
  return GSV_OK;
}

int gsv_backward_prep(const void* W, const void* I, const double* dldi, const gsv_grid* grid,
                      const gsv_bricks* bricks, double eps_w, int precision, void* ab,
                      int64_t* bad, void* stream) {
  if (int s = validate_grid_bricks(grid, bricks)) return s;
  GSV_REQUIRE(precision == 0 || precision == 1, "precision must be 0 (f32) or 1 (f64)");
  cudaStream_t s = as_stream(stream);
  cudaError_t e = cudaMemsetAsync(bad, 0x7F, sizeof(int64_t), s);
  if (e != cudaSuccess) return cuda_status(e, "memset bad");
  if (bricks->b1 <= bricks->b0) return GSV_OK;
  // The voxel planes of the brick layers the slab touches; the kernel keeps
  // only the voxels of the slab's bricks.
  const int64_t plane = (int64_t)grid->nx * grid->ny;
  const int64_t bplane = (int64_t)bricks->bgx * bricks->bgy;
  const int64_t v0 = plane * ((bricks->b0 / bplane) * bricks->bdz);
  const int64_t zend = ((bricks->b1 - 1) / bplane + 1) * bricks->bdz;
  const int64_t v1 = plane * (zend < grid->nz ? zend : (int64_t)grid->nz);
  if (v1 <= v0) return GSV_OK;
  const unsigned blocks = (unsigned)((v1 - v0 + 255) / 256);
  if (precision == 0)
    backward_prep_kernel<float, float2><<<blocks, 256, 0, s>>>(
        (const float*)W, (const float*)I, dldi, *grid, *bricks, v0, v1, eps_w, (float2*)ab,
        (unsigned long long*)bad);
  else
    backward_prep_kernel<double, double2><<<blocks, 256, 0, s>>>(
        (const double*)W, (const double*)I, dldi, *grid, *bricks, v0, v1, eps_w, (double2*)ab,
        (unsigned long long*)bad);
  GSV_CHECK_LAUNCH("backward_prep_kernel");
  return GSV_OK;
}

int gsv_backward(const double* positions, const double* log_scales, const double* rotations,
                 const gsv_record32* rec32, const gsv_record64* rec64, const int64_t* starts,
                 const int32_t* gids, const int64_t* gstart, const int32_t* box,
                 const gsv_grid* grid, const gsv_bricks* bricks, double cutoff_sigma,
                 int precision, const void* ab, const uint32_t* live_masks, int mask_vpl,
                 void* partials, void* stream) {
  if (int s = validate_grid_bricks(grid, bricks)) return s;
  GSV_REQUIRE(precision == 0 || precision == 1, "precision must be 0 (f32) or 1 (f64)");
  GSV_REQUIRE(precision == 0 || rec64 != nullptr, "the f64 backward needs rec64");
  const int64_t nb = slab_bricks(*bricks);
  if (nb == 0) return GSV_OK;
  const double cut2d = cutoff_sigma * cutoff_sigma;
  cudaStream_t s = as_stream(stream);
  if (precision == 0 && live_masks != nullptr) {
    if (mask_vpl == 0) mask_vpl = mask_vpl_auto(*bricks);
    const bool b884 = bricks->bdx == 8 && bricks->bdy == 8 && bricks->bdz == 4;
    GSV_REQUIRE(mask_vpl == 2 || mask_vpl == 4 || mask_vpl == 16,
                "mask_vpl must be 0, 2, 4 or 16");
    GSV_REQUIRE(mask_vpl != 16 || b884, "mask_vpl 16 (column-packed masks) needs 8x8x4 bricks");
    GSV_REQUIRE(mask_vpl == 16 || mask_units(*bricks, mask_vpl) == (mask_vpl == 4 ? 64 : 128),
                "live masks need a brick that fills one CTA's warp tiles exactly "
                "(e.g. 8x8x4)");
#define GSV_BWDM(A)                                                                            \
  backward32m_kernel<A><<<(unsigned)nb, kBwdMThreads, 0, s>>>(                                  \
      positions, rec32, starts, gids, gstart, box, *grid, *bricks, (float)cut2d,               \
      (const uint2*)live_masks, mask_vpl, (const float2*)ab, (float4*)partials)
    if (mask_vpl == 16)
      GSV_BWDM(2);
    else if (mask_vpl == 4 && b884)
      GSV_BWDM(1);
    else
      GSV_BWDM(0);
#undef GSV_BWDM
    GSV_CHECK_LAUNCH("backward32m_kernel");
  } else if (precision == 0) {
    const int64_t bvox = (int64_t)bricks->bdx * bricks->bdy * bricks->bdz;
    const bool smem = bvox <= kBwdSmemVoxels;
    const size_t shm = bwd_smem_bytes(smem ? (int)bvox : 0);
    static bool attr_set[2] = {false, false};
    if (!attr_set[smem]) {
      const int maxb = (int)bwd_smem_bytes(smem ? kBwdSmemVoxels : 0);
      cudaError_t e = smem ? cudaFuncSetAttribute(backward32_kernel<true>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, maxb)
                           : cudaFuncSetAttribute(backward32_kernel<false>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize, maxb);
      if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(backward32)");
      attr_set[smem] = true;
    }
    if (smem)
      backward32_kernel<true><<<(unsigned)nb, kBwdThreads, shm, s>>>(
          positions, ExactSrc{positions, log_scales, rotations, rec64}, rec32, starts, gids, gstart, box, *grid, *bricks,
          (float)cut2d, cut2d, (const float2*)ab, (float4*)partials);
    else
      backward32_kernel<false><<<(unsigned)nb, kBwdThreads, shm, s>>>(
          positions, ExactSrc{positions, log_scales, rotations, rec64}, rec32, starts, gids, gstart, box, *grid, *bricks,
          (float)cut2d, cut2d, (const float2*)ab, (float4*)partials);
    GSV_CHECK_LAUNCH("backward32_kernel");
  } else {
    backward64_kernel<<<(unsigned)nb, kBwdThreads, 0, s>>>(
        positions, rec64, rec32, starts, gids, gstart, box, *grid, *bricks, cut2d,
        (const double2*)ab, (double*)partials);
    GSV_CHECK_LAUNCH("backward64_kernel");
  }
  return GSV_OK;
}

int gsv_render_naive(const double* positions, const double* log_scales,
                     const double* rotations, const double* raw_amplitude,
                     const double* raw_relax, int64_t n, int relax_enabled,
                     const gsv_grid* grid, double cutoff_sigma, double eps_w, int precision,
                     void* I, void* stream) {
  GSV_REQUIRE(grid && grid->nx >= 1 && grid->ny >= 1 && grid->nz >= 1, "bad grid");
  GSV_REQUIRE(precision == 0 || precision == 1, "precision must be 0 (f32) or 1 (f64)");
  const int64_t nvox = (int64_t)grid->nx * grid->ny * grid->nz;
  const double cut2 = cutoff_sigma * cutoff_sigma;
  const unsigned blocks = (unsigned)((nvox + 127) / 128);
  cudaStream_t s = as_stream(stream);
  if (precision == 0)
    naive_kernel<float><<<blocks, 128, 0, s>>>(positions, log_scales, rotations,
                                                raw_amplitude, raw_relax, n, relax_enabled,
                                                *grid, cut2, eps_w, (float*)I);
  else
    naive_kernel<double><<<blocks, 128, 0, s>>>(positions, log_scales, rotations,
                                                 raw_amplitude, raw_relax, n, relax_enabled,
                                                 *grid, cut2, eps_w, (double*)I);
  GSV_CHECK_LAUNCH("naive_kernel");
  return GSV_OK;
}

}  // extern "C"
