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

#include "gsv_common.cuh"

namespace gsv {
namespace {

constexpr int kFwdThreads = 128;     // 4 warps; each warp owns one voxel tile
constexpr int kBwdThreads = 256;
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
// broadcast LDS.128 per (pair, warp-tile) evaluation.
struct __align__(16) Pair32 {
  float4 a;  // u0 u1 u2 amp      u = L (p_b0 - mu): v at the brick's first voxel
  float4 b;  // ex0 ex1 ex2 relax e_x = sx L[:,0]: v step per voxel along x
  float4 c;  // ey0 ey1 ey2 guard
  float4 d;  // ez0 ez1 ez2 gid
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

// sub_range with precomputed 1/s (no f64 division on the staging path).
__device__ __forceinline__ void sub_range_inv(double c, double h, double inv_s, int n, int& lo,
                                              int& hi) {
  const double ctr = c * inv_s, hv = h * inv_s;
  double a = ceil(ctr - hv - 1e-3), b = floor(ctr + hv + 1e-3);
  a = fmax(a, 0.0);
  b = fmin(b, (double)(n - 1));
  if (!(a <= b)) {
    lo = 1 << 20;
    hi = -1;
    return;
  }
  lo = (int)a;
  hi = (int)b;
}

// Exact f64 truncation decision of one (Gaussian, voxel) -- the rare
// guard-band path -- from the f64 whitening factor written by preprocess.
__device__ __noinline__ bool exact_live(int gid, int gx, int gy, int gz,
                                        const double* __restrict__ pos,
                                        const gsv_record64* __restrict__ rec64,
                                        const gsv_grid& g, double cutoff2) {
  const double* L = rec64[gid].l;
  const double* m = pos + 3 * (int64_t)gid;
  return ref_d2(L, m[0], m[1], m[2], gx, gy, gz, g) <= cutoff2;
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

__device__ __forceinline__ void live_accumulate(float d2, float amp, float relax, float guard,
                                                float cut2, double cut2d, int gid, int gx,
                                                int gy, int gz, const double* pos,
                                                const gsv_record64* rec64,
                                                const gsv_grid& g, float& S, float& W) {
  if (d2 > cut2 + guard) return;
  if (d2 >= cut2 - guard && !exact_live(gid, gx, gy, gz, pos, rec64, g, cut2d)) return;
  const float w = __expf(-0.5f * d2) * relax;
  S = fmaf(amp, w, S);
  W += w;
}

// One CTA per brick, 4 warps, each owning one voxel tile (2 voxels per lane).
// Warps walk the brick's list independently -- no CTA barrier in the pair
// loop: per round of 32 list entries every lane stages one pair into the
// warp's private smem slots and tests its 3-sigma box against the warp's
// tile; a ballot leaves only the pairs that reach the tile, evaluated in list
// order (deterministic accumulation, no atomics).  Staging is repeated per
// warp (4x, L1-resident loads) -- cheaper than the barrier stalls of shared
// staging, where every warp waits for the slowest tile each chunk.
__global__ void __launch_bounds__(kFwdThreads)
forward32_kernel(const double* __restrict__ pos, const gsv_record32* __restrict__ rec,
                 const gsv_record64* __restrict__ rec64,
                 const int64_t* __restrict__ starts, const int32_t* __restrict__ gids,
                 gsv_grid g, gsv_bricks k, float cut2, double cut2d, double eps_w,
                 float* __restrict__ S, float* __restrict__ W, float* __restrict__ I,
                 const float* __restrict__ target, int loss_kind, double vox_count,
                 float2* __restrict__ ab, double* __restrict__ loss_part) {
  __shared__ Pair32 sp[kFwdThreads];   // 32 slots per warp
  __shared__ double red[kFwdThreads / 32];
  const int lb = blockIdx.x;                               // slab-local brick
  const int b = (int)slab_first(k) + lb;                   // global brick id
  const BrickGeom bg = brick_geom(b, g, k);
  const int64_t lbeg = starts[lb], lend = starts[lb + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  Pair32* wsp = sp + (warp << 5);
  const bool tiled = ((k.bdx | k.bdy | k.bdz) & 3) == 0;
  const int units = k.bdx * k.bdy * ((k.bdz + 1) >> 1);
  const float fsx = (float)g.sx, fsy = (float)g.sy, fsz = (float)g.sz;
  const float isx = (float)(1.0 / g.sx), isy = (float)(1.0 / g.sy), isz = (float)(1.0 / g.sz);
  double lsum = 0.0;

  for (int ubase = 0; ubase < units; ubase += kFwdThreads) {
    const int u = ubase + tid;
    int lx = 0, ly = 0, lz = 0;
    if (u < units) unit_voxel(u, k, tiled, lx, ly, lz);
    const bool ownA = u < units && lx < bg.ex && ly < bg.ey && lz < bg.ez;
    const bool ownB = ownA && lz + 1 < bg.ez && lz + 1 < k.bdz;
    // This warp's tile box (brick-local voxel coords) from its owned voxels.
    int txl = ownA ? lx : 1 << 20, txh = ownA ? lx : -(1 << 20);
    int tyl = ownA ? ly : 1 << 20, tyh = ownA ? ly : -(1 << 20);
    int tzl = ownA ? lz : 1 << 20, tzh = ownB ? lz + 1 : (ownA ? lz : -(1 << 20));
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
    const float fx = (float)lx, fy = (float)ly, fz = (float)lz;
    const int gx = bg.x0 + lx, gy = bg.y0 + ly, gz = bg.z0 + lz;
    float accSA = 0.f, accWA = 0.f, accSB = 0.f, accWB = 0.f;

    for (int64_t base = lbeg; base < lend; base += 32) {
      const int64_t j = base + lane;
      bool hit = false;
      if (j < lend) {
        const int gid = gids[j];
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
          const float guard = kGuardRel * cut2 + kGuardMag * umax * sqrtf(cut2);
          Pair32 p;
          p.a = make_float4(u3[0], u3[1], u3[2], q2.y);
          p.b = make_float4(e[0][0], e[0][1], e[0][2], q2.z);
          p.c = make_float4(e[1][0], e[1][1], e[1][2], guard);
          p.d = make_float4(e[2][0], e[2][1], e[2][2], __int_as_float(gid));
          wsp[lane] = p;
        }
      }
      unsigned ball = __ballot_sync(kFull, hit);
      __syncwarp();
      while (ball) {
        const int jj = __ffs(ball) - 1;
        ball &= ball - 1;
        const float4 pa = wsp[jj].a, pb = wsp[jj].b, pc = wsp[jj].c, pd = wsp[jj].d;
        const float v0 = fmaf(fz, pd.x, fmaf(fy, pc.x, fmaf(fx, pb.x, pa.x)));
        const float v1 = fmaf(fz, pd.y, fmaf(fy, pc.y, fmaf(fx, pb.y, pa.y)));
        const float v2 = fmaf(fz, pd.z, fmaf(fy, pc.z, fmaf(fx, pb.z, pa.z)));
        const float d2a = fmaf(v0, v0, fmaf(v1, v1, v2 * v2));
        const float w0 = v0 + pd.x, w1 = v1 + pd.y, w2 = v2 + pd.z;  // voxel z0+1
        const float d2b = fmaf(w0, w0, fmaf(w1, w1, w2 * w2));
        const int gid = __float_as_int(pd.w);
        live_accumulate(d2a, pa.w, pb.w, pc.w, cut2, cut2d, gid, gx, gy, gz, pos, rec64, g,
                        accSA, accWA);
        live_accumulate(d2b, pa.w, pb.w, pc.w, cut2, cut2d, gid, gx, gy, gz + 1, pos, rec64,
                        g, accSB, accWB);
      }
      __syncwarp();
    }
    // Epilogue: normalise, store, fused loss (optimize.py:91-103).
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const bool own = h == 0 ? ownA : ownB;
      if (!own) continue;
      const float accS = h == 0 ? accSA : accSB, accW = h == 0 ? accWA : accWB;
      const int64_t lin = (int64_t)gx + (int64_t)g.nx * (gy + (int64_t)g.ny * (gz + h));
      const bool cov = (double)accW >= eps_w;
      const float iv = cov ? __fdiv_rn(accS, accW) : 0.f;
      S[lin] = accS;
      W[lin] = accW;
      I[lin] = iv;
      if (target) {
        const double d = (double)iv - (double)target[lin];
        double dl;
        if (loss_kind == 0) {
          lsum += fabs(d);
          dl = (d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0)) / vox_count;
        } else {
          lsum += d * d;
          dl = 2.0 * d / vox_count;
        }
        const float alpha = (cov && dl != 0.0) ? (float)(dl / (double)accW) : 0.f;
        ab[lin] = make_float2(alpha, iv);
      }
    }
  }
  if (target) {
    const double t = block_sum<kFwdThreads>(lsum, red);
    if (tid == 0) loss_part[lb] = t;
  }
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
                 double* __restrict__ I, const float* __restrict__ target, int loss_kind,
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
        const double d = iv - (double)target[lin];
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
                                     const double* __restrict__ dldi, gsv_grid g,
                                     int64_t v0, int64_t v1, double eps_w, T2* __restrict__ ab,
                                     unsigned long long* bad) {
  const int64_t lin = v0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (lin >= v1) return;
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
// One thread per (brick, Gaussian) pair.  Three phases per chunk of up to 256
// list entries:
//  (1) per pair: brick-relative coefficients and, row by row, the exact x-span
//      where d2(x) = |v_row + x e_x|^2 (a quadratic) can be <= cutoff^2 +
//      guard; the spans go to shared memory, the candidate-voxel count is the
//      pair's cost.
//  (2) a smem counting sort of the pairs by cost, heaviest first.
//  (3) warps pull groups of 32 pairs of similar cost (dynamic, heaviest
//      first) and every lane runs ONE flattened loop over its pair's candidate
//      voxels, so a warp costs max(candidates) iterations rather than the sum
//      over rows of the per-row maxima.
// Order of processing never changes a result: each pair's partial is computed
// by one thread in a fixed voxel order and written to its own slot.  Every
// candidate is still decided exactly as the forward decides.  The brick's
// {dL/dI / W, I} are staged in shared memory.  Accumulates sum cw v
// (whitened) and sum cw delta delta^T; d_mu = L^T sum cw v once per pair.
constexpr int kBwdChunk = 256;      // pairs per chunk (one per thread)
constexpr int kBwdRows = 24;        // span slots per pair (LR/HR bricks need <= 20)
constexpr int kBwdBuckets = 128;

struct BwdPair;
size_t bwd_smem_bytes(int ab_voxels);

struct __align__(16) BwdPair {
  float u[3], ex[3], ey[3], ez[3];
  float c[3];          // p_b0 - mu
  float guard;
  int gid;
  int nspan;           // stored spans; -1 = overflow (rows > kBwdRows)
  int cost;            // candidate voxels
};

__device__ __forceinline__ void bwd_accumulate(float d2, float kernw_r, float A, float2 v_ab,
                                               float v0, float v1, float v2, float dx,
                                               float dy, float dz, float& acc_a,
                                               float& acc_r, float& s0, float& s1,
                                               float& s2, float& g00, float& g11,
                                               float& g22, float& g01, float& g02,
                                               float& g12) {
  const float kern = __expf(-0.5f * d2);
  const float w = kern * kernw_r;
  acc_a = fmaf(w, v_ab.x, acc_a);
  const float common = v_ab.x * (A - v_ab.y);   // dL/dI (A - I) / W
  acc_r = fmaf(common, kern, acc_r);
  const float cw = common * w;
  s0 = fmaf(cw, v0, s0);
  s1 = fmaf(cw, v1, s1);
  s2 = fmaf(cw, v2, s2);
  const float h = -0.5f * cw;
  const float hx = h * dx, hy = h * dy;
  g00 = fmaf(hx, dx, g00);
  g11 = fmaf(hy, dy, g11);
  g22 = fmaf(h * dz, dz, g22);
  g01 = fmaf(hx, dy, g01);
  g02 = fmaf(hx, dz, g02);
  g12 = fmaf(hy, dz, g12);
}

size_t bwd_smem_bytes(int ab_voxels) {
  return sizeof(BwdPair) * kBwdChunk + sizeof(unsigned) * kBwdChunk * kBwdRows +
         sizeof(unsigned short) * kBwdChunk + sizeof(int) * (kBwdBuckets + 4) +
         sizeof(float2) * (size_t)ab_voxels;
}

template <bool kSmem>
__global__ void __launch_bounds__(kBwdThreads, 3)
backward32_kernel(const double* __restrict__ pos, const gsv_record32* __restrict__ rec,
                  const gsv_record64* __restrict__ rec64,
                  const int64_t* __restrict__ starts, const int32_t* __restrict__ gids,
                  const int64_t* __restrict__ gstart, const int32_t* __restrict__ box,
                  gsv_grid g, gsv_bricks k, float cut2, double cut2d,
                  const float2* __restrict__ ab, float4* __restrict__ partials) {
  extern __shared__ __align__(16) unsigned char bwd_smem[];
  BwdPair* spair = reinterpret_cast<BwdPair*>(bwd_smem);
  unsigned* sspan = reinterpret_cast<unsigned*>(spair + kBwdChunk);  // y|z<<8|xa<<16|xb<<24
  unsigned short* sorder = reinterpret_cast<unsigned short*>(sspan + kBwdChunk * kBwdRows);
  int* shist = reinterpret_cast<int*>(sorder + kBwdChunk);
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
  const float isx = (float)(1.0 / g.sx), isy = (float)(1.0 / g.sy), isz = (float)(1.0 / g.sz);
  const float lo_cut = cut2;
  if (kSmem) {
    const int nv = bg.ex * bg.ey * bg.ez;
    for (int v = tid; v < nv; v += kBwdThreads) {
      const int x = v % bg.ex, y = (v / bg.ex) % bg.ey, z = v / (bg.ex * bg.ey);
      const int64_t lin =
          (int64_t)(bg.x0 + x) + (int64_t)g.nx * ((bg.y0 + y) + (int64_t)g.ny * (bg.z0 + z));
      sab[x + k.bdx * (y + k.bdy * z)] = __ldg(ab + lin);
    }
  }
  for (int64_t cbase = lbeg; cbase < lend; cbase += kBwdChunk) {
    const int cnt = (int)min((int64_t)kBwdChunk, lend - cbase);
    if (tid < kBwdBuckets) shist[tid] = 0;
    if (tid == 0) *snextp = 0;
    __syncthreads();
    // ---- (1) coefficients + exact row spans
    if (tid < cnt) {
      BwdPair P;
      const int gid = gids[cbase + tid];
      const float4* r4 = reinterpret_cast<const float4*>(rec + gid);
      const float4 q0 = __ldg(r4), q1 = __ldg(r4 + 1), q2 = __ldg(r4 + 2), q3 = __ldg(r4 + 3);
      const float L[9] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w, q2.x};
      const double* m = pos + 3 * (int64_t)gid;
      const float mx = (float)(__ldg(m) - bg.px), my = (float)(__ldg(m + 1) - bg.py),
                  mz = (float)(__ldg(m + 2) - bg.pz);   // mu - p_b0
      P.c[0] = -mx; P.c[1] = -my; P.c[2] = -mz;
      float umax = 0.f;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        P.u[a] = -fmaf(L[3 * a], mx, fmaf(L[3 * a + 1], my, L[3 * a + 2] * mz));
        P.ex[a] = L[3 * a] * fsx;
        P.ey[a] = L[3 * a + 1] * fsy;
        P.ez[a] = L[3 * a + 2] * fsz;
        umax = fmaxf(umax, fabsf(P.u[a]) + fabsf(P.ex[a]) * k.bdx + fabsf(P.ey[a]) * k.bdy +
                               fabsf(P.ez[a]) * k.bdz);
      }
      P.guard = kGuardRel * cut2 + kGuardMag * umax * sqrtf(cut2);
      P.gid = gid;
      // 3-sigma voxel box (brick-local), widened by 1e-3 voxel.
      const float cyv = my * isy, czv = mz * isz;
      const float hyv = fmaf(q3.x, isy, 1e-3f), hzv = fmaf(q3.y, isz, 1e-3f);
      const int yl = max(0, (int)ceilf(cyv - hyv)), yh = min(bg.ey - 1, (int)floorf(cyv + hyv));
      const int zl = max(0, (int)ceilf(czv - hzv)), zh = min(bg.ez - 1, (int)floorf(czv + hzv));
      const float qa = fmaf(P.ex[0], P.ex[0], fmaf(P.ex[1], P.ex[1], P.ex[2] * P.ex[2]));
      const float inv_qa = 1.0f / qa;
      const float lim = cut2 + P.guard;
      int ns = 0, cost = 0;
      unsigned* my_sp = sspan + tid * kBwdRows;
      for (int z = zl; z <= zh; ++z) {
        for (int y = yl; y <= yh; ++y) {
          const float vr0 = fmaf((float)z, P.ez[0], fmaf((float)y, P.ey[0], P.u[0]));
          const float vr1 = fmaf((float)z, P.ez[1], fmaf((float)y, P.ey[1], P.u[1]));
          const float vr2 = fmaf((float)z, P.ez[2], fmaf((float)y, P.ey[2], P.u[2]));
          const float qb = fmaf(vr0, P.ex[0], fmaf(vr1, P.ex[1], vr2 * P.ex[2]));
          const float qc = fmaf(vr0, vr0, fmaf(vr1, vr1, vr2 * vr2));
          // (qa x + qb)^2 <= qb^2 - qa (qc - lim)
          const float disc = fmaf(qb, qb, -qa * (qc - lim));
          if (!(disc >= 0.f)) continue;
          const float sq = sqrtf(disc);
          const int xa = max(0, (int)ceilf((-qb - sq) * inv_qa - 1e-3f));
          const int xb = min(bg.ex - 1, (int)floorf((-qb + sq) * inv_qa + 1e-3f));
          if (xa > xb) continue;
          if (ns < kBwdRows) my_sp[ns] = (unsigned)y | ((unsigned)z << 8) |
                                         ((unsigned)xa << 16) | ((unsigned)xb << 24);
          ++ns;
          cost += xb - xa + 1;
        }
      }
      P.nspan = ns <= kBwdRows ? ns : -1;
      P.cost = cost;
      spair[tid] = P;
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
    if (tid < cnt) {
      const int slot = atomicAdd(&shist[kBwdBuckets - 1 - min(spair[tid].cost, kBwdBuckets - 1)], 1);
      sorder[slot] = (unsigned short)tid;
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
      const BwdPair& P = spair[t];
      const int gid = P.gid;
      const float4* r4 = reinterpret_cast<const float4*>(rec + gid);
      const float4 q0 = __ldg(r4), q1 = __ldg(r4 + 1), q2 = __ldg(r4 + 2);
      const float A = q2.y, r = q2.z;
      const float ex0 = P.ex[0], ex1 = P.ex[1], ex2 = P.ex[2];
      const float c0 = P.c[0], c1 = P.c[1], c2 = P.c[2];
      const float lim = cut2 + P.guard, lo_band = lo_cut - P.guard;
      float acc_a = 0.f, acc_r = 0.f, s0 = 0.f, s1 = 0.f, s2 = 0.f;
      float g00 = 0.f, g11 = 0.f, g22 = 0.f, g01 = 0.f, g02 = 0.f, g12 = 0.f;
      if (P.nspan >= 0) {
        // Flattened loop over the candidate voxels of all spans.
        const unsigned* my_sp = sspan + t * kBwdRows;
        int si = 0, x = 0, xb = -1, y = 0, z = 0, srow = 0;
        float vr0 = 0.f, vr1 = 0.f, vr2 = 0.f, dy = 0.f, dz = 0.f;
        for (int it = 0; it < P.cost; ++it) {
          if (x > xb) {   // next span
            const unsigned sp = my_sp[si++];
            y = sp & 255; z = (sp >> 8) & 255; x = (sp >> 16) & 255; xb = sp >> 24;
            vr0 = fmaf((float)z, P.ez[0], fmaf((float)y, P.ey[0], P.u[0]));
            vr1 = fmaf((float)z, P.ez[1], fmaf((float)y, P.ey[1], P.u[1]));
            vr2 = fmaf((float)z, P.ez[2], fmaf((float)y, P.ey[2], P.u[2]));
            dy = fmaf((float)y, fsy, c1);
            dz = fmaf((float)z, fsz, c2);
            srow = k.bdx * (y + k.bdy * z);
          }
          const float2 v_ab = kSmem ? sab[srow + x]
                                    : __ldg(ab + (int64_t)(bg.x0 + x) +
                                            (int64_t)g.nx * ((bg.y0 + y) + (int64_t)g.ny * (bg.z0 + z)));
          const float fx = (float)x;
          ++x;
          if (v_ab.x == 0.f) continue;
          const float v0 = fmaf(fx, ex0, vr0), v1 = fmaf(fx, ex1, vr1), v2 = fmaf(fx, ex2, vr2);
          const float d2 = fmaf(v0, v0, fmaf(v1, v1, v2 * v2));
          if (d2 > lim) continue;
          if (d2 >= lo_band &&
              !exact_live(gid, bg.x0 + (int)fx, bg.y0 + y, bg.z0 + z, pos, rec64, g, cut2d))
            continue;
          bwd_accumulate(d2, r, A, v_ab, v0, v1, v2, fmaf(fx, fsx, c0), dy, dz, acc_a, acc_r, s0,
                         s1, s2, g00, g11, g22, g01, g02, g12);
        }
      } else {
        // More candidate rows than span slots (very large bricks): nested loops.
        const float cyv = -c1 * isy, czv = -c2 * isz;
        const float4 q3 = __ldg(r4 + 3);
        const float hyv = fmaf(q3.x, isy, 1e-3f), hzv = fmaf(q3.y, isz, 1e-3f);
        const int yl = max(0, (int)ceilf(cyv - hyv)), yh = min(bg.ey - 1, (int)floorf(cyv + hyv));
        const int zl = max(0, (int)ceilf(czv - hzv)), zh = min(bg.ez - 1, (int)floorf(czv + hzv));
        for (int z = zl; z <= zh; ++z) {
          const float dz = fmaf((float)z, fsz, c2);
          for (int y = yl; y <= yh; ++y) {
            const float dy = fmaf((float)y, fsy, c1);
            const float vr0 = fmaf((float)z, P.ez[0], fmaf((float)y, P.ey[0], P.u[0]));
            const float vr1 = fmaf((float)z, P.ez[1], fmaf((float)y, P.ey[1], P.u[1]));
            const float vr2 = fmaf((float)z, P.ez[2], fmaf((float)y, P.ey[2], P.u[2]));
            for (int x = 0; x < bg.ex; ++x) {
              const float2 v_ab = kSmem ? sab[k.bdx * (y + k.bdy * z) + x]
                                        : __ldg(ab + (int64_t)(bg.x0 + x) +
                                                (int64_t)g.nx * ((bg.y0 + y) + (int64_t)g.ny * (bg.z0 + z)));
              if (v_ab.x == 0.f) continue;
              const float fx = (float)x;
              const float v0 = fmaf(fx, ex0, vr0), v1 = fmaf(fx, ex1, vr1), v2 = fmaf(fx, ex2, vr2);
              const float d2 = fmaf(v0, v0, fmaf(v1, v1, v2 * v2));
              if (d2 > lim) continue;
              if (d2 >= lo_band &&
                  !exact_live(gid, bg.x0 + x, bg.y0 + y, bg.z0 + z, pos, rec64, g, cut2d))
                continue;
              bwd_accumulate(d2, r, A, v_ab, v0, v1, v2, fmaf(fx, fsx, c0), dy, dz, acc_a, acc_r,
                             s0, s1, s2, g00, g11, g22, g01, g02, g12);
            }
          }
        }
      }
      // d_mu = sum cw Sigma^-1 delta = L^T (sum cw v); L row-major in q0,q1,q2.x
      const float mu0 = fmaf(q0.x, s0, fmaf(q0.w, s1, q1.z * s2));
      const float mu1 = fmaf(q0.y, s0, fmaf(q1.x, s1, q1.w * s2));
      const float mu2b = fmaf(q0.z, s0, fmaf(q1.y, s1, q2.x * s2));
      const GBox gb = unpack_box(box, gid);
      const int rx = bc.bx - gb.blo_x, ry = bc.by - gb.blo_y, rz = bc.bz - gb.blo_z;
      // A caller-built list may hold a pair the binning would not emit: skip it.
      if (rx < 0 || rx >= gb.nb_x || ry < 0 || ry >= gb.nb_y || rz < 0 || rz >= gb.nb_z) continue;
      const int64_t e = gstart[gid] + rx + (int64_t)gb.nb_x * (ry + (int64_t)gb.nb_y * rz);
      float4* dst = partials + 3 * e;
      dst[0] = make_float4(acc_a, acc_r, mu0, mu1);
      dst[1] = make_float4(mu2b, g00, g11, g22);
      dst[2] = make_float4(g01, g02, g12, 0.f);
    }
    __syncthreads();
  }
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
    const int rx = bc.bx - gb.blo_x, ry = bc.by - gb.blo_y, rz = bc.bz - gb.blo_z;
    // A caller-built list may hold a pair the binning would not emit: skip it.
    if (rx < 0 || rx >= gb.nb_x || ry < 0 || ry >= gb.nb_y || rz < 0 || rz >= gb.nb_z) continue;
    const int64_t e = gstart[gid] + rx + (int64_t)gb.nb_x * (ry + (int64_t)gb.nb_y * rz);
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

int gsv_forward(const double* positions, const gsv_record32* rec32, const gsv_record64* rec64,
                const int64_t* starts,
                const int32_t* gids, const gsv_grid* grid, const gsv_bricks* bricks,
                double cutoff_sigma, double eps_w, int precision, void* S, void* W, void* I,
                const float* target, int loss_kind, double vox_count, float* ab,
                double* loss_part, void* stream) {
  if (int s = validate_grid_bricks(grid, bricks)) return s;
  GSV_REQUIRE(precision == 0 || precision == 1, "precision must be 0 (f32) or 1 (f64)");
  GSV_REQUIRE(rec64 != nullptr, "forward needs rec64 (f64 whitening factors)");
  GSV_REQUIRE(target == nullptr || (ab != nullptr && loss_part != nullptr),
              "fused loss needs ab and loss_part");
  GSV_REQUIRE(loss_kind == 0 || loss_kind == 1, "loss_kind must be 0 (l1) or 1 (l2)");
  const int64_t nb = slab_bricks(*bricks);
  if (nb == 0) return GSV_OK;
  const double cut2d = cutoff_sigma * cutoff_sigma;
  cudaStream_t s = as_stream(stream);
  if (precision == 0) {
    forward32_kernel<<<(unsigned)nb, kFwdThreads, 0, s>>>(
        positions, rec32, rec64, starts, gids, *grid, *bricks, (float)cut2d,
        cut2d, eps_w, (float*)S, (float*)W, (float*)I, target, loss_kind, vox_count,
        (float2*)ab, loss_part);
    GSV_CHECK_LAUNCH("forward32_kernel");
  } else {
    forward64_kernel<<<(unsigned)nb, 128, 0, s>>>(
        positions, rec64, nullptr, starts, gids, *grid, *bricks, cut2d, eps_w, (double*)S,
        (double*)W, (double*)I, target, loss_kind, vox_count, (double2*)ab, loss_part, rec32);
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
  // The slab's voxels: whole z-layers [bz0*bdz, min(bz1*bdz, nz)).
  const int64_t plane = (int64_t)grid->nx * grid->ny;
  const int64_t v0 = plane * ((int64_t)bricks->bz0 * bricks->bdz);
  const int64_t zend = (int64_t)bricks->bz1 * bricks->bdz;
  const int64_t v1 = plane * (zend < grid->nz ? zend : (int64_t)grid->nz);
  if (v1 <= v0) return GSV_OK;
  const unsigned blocks = (unsigned)((v1 - v0 + 255) / 256);
  if (precision == 0)
    backward_prep_kernel<float, float2><<<blocks, 256, 0, s>>>(
        (const float*)W, (const float*)I, dldi, *grid, v0, v1, eps_w, (float2*)ab,
        (unsigned long long*)bad);
  else
    backward_prep_kernel<double, double2><<<blocks, 256, 0, s>>>(
        (const double*)W, (const double*)I, dldi, *grid, v0, v1, eps_w, (double2*)ab,
        (unsigned long long*)bad);
  GSV_CHECK_LAUNCH("backward_prep_kernel");
  return GSV_OK;
}

int gsv_backward(const double* positions, const gsv_record32* rec32, const gsv_record64* rec64,
                 const int64_t* starts,
                 const int32_t* gids, const int64_t* gstart, const int32_t* box,
                 const gsv_grid* grid, const gsv_bricks* bricks, double cutoff_sigma,
                 int precision, const void* ab, void* partials, void* stream) {
  if (int s = validate_grid_bricks(grid, bricks)) return s;
  GSV_REQUIRE(precision == 0 || precision == 1, "precision must be 0 (f32) or 1 (f64)");
  GSV_REQUIRE(rec64 != nullptr, "backward needs rec64 (f64 whitening factors)");
  const int64_t nb = slab_bricks(*bricks);
  if (nb == 0) return GSV_OK;
  const double cut2d = cutoff_sigma * cutoff_sigma;
  cudaStream_t s = as_stream(stream);
  if (precision == 0) {
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
          positions, rec32, rec64, starts, gids, gstart, box, *grid, *bricks,
          (float)cut2d, cut2d, (const float2*)ab, (float4*)partials);
    else
      backward32_kernel<false><<<(unsigned)nb, kBwdThreads, shm, s>>>(
          positions, rec32, rec64, starts, gids, gstart, box, *grid, *bricks,
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
