// gsv_bin.cu -- fused per-Gaussian preprocessing and brick binning.
//
// Replaces build_brick_index (raster.py:148-217), _whitening_factors
// (raster.py:233-237) and the sigmoid activations (field.py:86-94).
//
//   preprocess_kernel   one thread per Gaussian, f64 AABB in the reference's
//                       exact operation order -> per-Gaussian pair count and
//                       brick box; fp32 (and optionally fp64) record for the
//                       pair kernels.
//   cub ExclusiveSum    counts -> gstart (gid-major emission offsets)
//   emit_warp_kernel    (slab-local brick id, gid) in gid-major order, each
//                       Gaussian's bricks x-fastest (raster.py:200-209);
//                       warp-cooperative, coalesced stores
//   cub SortPairs       stable LSD radix sort on the brick id, only
//                       ceil(log2 B) key bits -> lists ascending in gid
//   starts_search_kernel CSR starts by binary search in the sorted keys
//                       (raster.py:213-215)
//
// This translation unit is compiled with -fmad=false in addition to using
// the explicit _rn intrinsics, so no f64 expression that feeds a binning
// decision can be contracted.
#include <cub/cub.cuh>
#include <thrust/iterator/transform_iterator.h>

#include "gsv_prep.cuh"

namespace gsv {
namespace {

#ifndef GSV_PREP_MINB
#define GSV_PREP_MINB 4          // 256-thread CTAs per SM the preprocess is built for
#endif
__global__ void __launch_bounds__(256, GSV_PREP_MINB)
preprocess_kernel(const double* __restrict__ pos, const double* __restrict__ ls,
                  const double* __restrict__ rot, const double* __restrict__ ra,
                  const double* __restrict__ rr, int64_t n, PrepArgs pa) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double q[4], l[3], p[3];
#pragma unroll
  for (int a = 0; a < 4; ++a) q[a] = rot[4 * i + a];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    l[a] = ls[3 * i + a];
    p[a] = pos[3 * i + a];
  }
  preprocess_one(i, p, l, q, ra[i], rr[i], pa);
}

struct ToI64 {
  __host__ __device__ __forceinline__ int64_t operator()(int32_t v) const { return (int64_t)v; }
};

__global__ void scan_tail_kernel(const int32_t* counts, int64_t n, int64_t* gstart) {
  gstart[n] = n > 0 ? gstart[n - 1] + (int64_t)counts[n - 1] : 0;
}

// Warp-cooperative emission through shared memory: a warp owns 32
// consecutive Gaussians, prefix-sums their pair counts with shuffles, and
// fills its output range window by window (kEmitWin slots): each lane writes
// its own Gaussian's bricks of the window into shared memory, walking the box
// x-fastest with incremental counters (raster.py:200-209; one division per
// lane and window, none per pair), then the warp copies the window out with
// coalesced stores.
constexpr int kEmitWin = 512;

template <typename K>
__global__ void __launch_bounds__(256)
emit_warp_kernel(const int32_t* __restrict__ counts, const int32_t* __restrict__ box,
                 const int64_t* __restrict__ gstart, int64_t n, gsv_bricks k,
                 K* __restrict__ keys, int32_t* __restrict__ vals, int64_t cap) {
  __shared__ int2 swin[8][kEmitWin];          // per warp: (key, gid) of one window
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t g0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~(int64_t)31;
  if (g0 >= n) return;                       // warp-uniform
  const int64_t g = g0 + lane;
  int c = 0, nbx = 1, nby = 1, kb = 0, k0 = 0;
  if (g < n) {
    c = counts[g];
    if (c > 0) {
      const GBox b = unpack_box(box, g);
      nbx = b.nb_x;
      nby = b.nb_y;
      k0 = b.k0;                            // the slab's run starts k0 into the box
      kb = b.blo_x + k.bgx * (b.blo_y + k.bgy * b.blo_z) - k.b0;   // slab-local id
    }
  }
  int incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  const int off = incl - c;
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  const int64_t base = gstart[g0];
  const int bxy = k.bgx * k.bgy;
  int2* win = swin[warp];
  for (int w0 = 0; w0 < total; w0 += kEmitWin) {
    // this lane's pairs inside [w0, w0 + kEmitWin)
    const int r0 = max(0, w0 - off), r1 = min(c, w0 + kEmitWin - off);
    if (r0 < r1) {
      int rx = (r0 + k0) % nbx;
      const int t = (r0 + k0) / nbx;
      int ry = t % nby, rz = t / nby;
      int key = kb + rx + k.bgx * ry + bxy * rz;
      const int gid = (int)g;
      for (int r = r0; r < r1; ++r) {
        win[off + r - w0] = make_int2(key, gid);
        ++key;
        if (++rx == nbx) {                   // next row, then next layer
          rx = 0;
          key += k.bgx - nbx;
          if (++ry == nby) {
            ry = 0;
            key += bxy - k.bgx * nby;
          }
        }
      }
    }
    __syncwarp();
    const int cnt = min(kEmitWin, total - w0);
    for (int q = lane; q < cnt; q += 32) {
      const int64_t o = base + w0 + q;
      if (o < cap) {
        const int2 e = win[q];
        keys[o] = (K)e.x;
        vals[o] = e.y;
      }
    }
    __syncwarp();
  }
}

// starts[b] = lower_bound(keys, b) for b < B (one thread per brick, binary
// search over the sorted keys); starts[B] = P (capacity mode: the device
// count, which cuts off the padding); all zero on overflow.
template <typename K>
__global__ void starts_search_kernel(const K* __restrict__ keys, int64_t p, int32_t nb,
                                     int64_t* __restrict__ starts,
                                     const int32_t* __restrict__ overflow,
                                     const int64_t* __restrict__ p_true) {
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b > nb) return;
  if (overflow != nullptr && *overflow != 0) {
    starts[b] = 0;
    return;
  }
  if (b == nb) {
    starts[b] = p_true != nullptr ? *p_true : p;
    return;
  }
  int64_t lo = 0, hi = p;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int32_t)__ldg(keys + mid) < (int32_t)b) lo = mid + 1; else hi = mid;
  }
  starts[b] = lo;
}

// Capacity mode: the pair count P = gstart[n] stays on the device.  Slots
// [P, cap) get the last brick id nb - 1 (the stable sort keeps them behind
// that brick's real pairs, and starts[nb] = P cuts them off), so keys stay
// within ceil(log2 nb) bits; overflow = P > cap (or the caller's dry-run
// flag) empties every list.
template <typename K>
__global__ void pad_kernel(const int64_t* __restrict__ gstart, int64_t n, int64_t cap,
                           int32_t nb, const int32_t* __restrict__ dry,
                           K* __restrict__ keys, int32_t* __restrict__ vals,
                           int32_t* __restrict__ overflow) {
  const int64_t p = gstart[n];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = p + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < cap; j += stride) {
    keys[j] = (K)(nb - 1);
    vals[j] = 0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0)
    *overflow = (p > cap || (dry != nullptr && *dry != 0)) ? 1 : 0;
}

__global__ void unsorted_kernel(const int64_t* __restrict__ starts,
                                const int32_t* __restrict__ gids, int32_t nb,
                                int32_t* flag) {
  const int32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  for (int64_t j = starts[b] + 1; j < starts[b + 1]; ++j)
    if (gids[j] <= gids[j - 1]) {
      *flag = 1;
      return;
    }
}

// ------------------------------------------------- incremental binning
// Between two fit() iterations only a few Gaussians change their brick box
// (~100 of 2.1 M per step at config 3; up to ~2000 in iterations 20-60), so
// the graph step keeps last step's lists and edits them.  The preprocess pass
// records every Gaussian whose box or pair count changed (PrepArgs change
// tracking).  incr_ops_kernel turns those into (brick, gid, remove | insert)
// edits -- the bricks of the old box run not in the new one and vice versa --
// appended to a flat array while per-brick counters count each brick's
// edits and its length change; the new lengths and the edit counts are
// scanned together (one packed int64 scan) into the new CSR starts and the
// per-brick edit offsets; the edits are scattered into per-brick segments
// (the counters return to zero on the way); one warp per brick then copies
// its list (no edits) or sorts its few edits by gid and merges the survivors
// and the insertions in gid order into the output buffers.  The result
// equals a full rebuild (each list is the ascending gids of the Gaussians
// whose box run contains the brick); any capacity excess (changed Gaussians,
// edits, pairs) or a pair count that differs from the counts' scan raises
// the overflow flag and the caller rebuilds.
constexpr int kOpsCap = 16384;      // edits per step

// Is slab-local brick `key` in the box run (box record, count) of a Gaussian?
__device__ __forceinline__ bool run_contains(const GBox& gb, int cnt, int key,
                                             const gsv_bricks& k) {
  if (cnt <= 0) return false;
  const int bgl = key + k.b0;
  const int plane = k.bgx * k.bgy;
  const int bz = bgl / plane, rem = bgl - bz * plane;
  const int by = rem / k.bgx, bx = rem - by * k.bgx;
  const int rx = bx - gb.blo_x, ry = by - gb.blo_y, rz = bz - gb.blo_z;
  if (rx < 0 || rx >= gb.nb_x || ry < 0 || ry >= gb.nb_y || rz < 0 || rz >= gb.nb_z)
    return false;
  const int r = rx + gb.nb_x * (ry + gb.nb_y * rz) - gb.k0;
  return r >= 0 && r < cnt;
}

// Per-brick scratch of the incremental pass (int32 words, B = slab bricks;
// 8 (B + 1) words, zero when first used): [0, B+1) edit counters, [B+1,
// 2B+2) length changes (both back to zero after every clean call), then
// int64 [B+1] packed (length << 24 | edits), int64 [B+1] its exclusive
// scan, int32 [B+1] the edit offsets, and one poison word: set by any
// overflow (not a dry run), it makes every later call overflow -- the
// counters may be dirty -- until the caller rebuilds with fresh scratch.
struct IncrScratch {
  int32_t* bcnt;
  int32_t* bdelta;
  int64_t* packed;
  int64_t* scanned;
  int32_t* opbeg;
  int32_t* poison;
  __host__ __device__ IncrScratch(int32_t* w, int64_t nb)
      : bcnt(w), bdelta(w + (nb + 1)), packed(reinterpret_cast<int64_t*>(w + 2 * (nb + 1))),
        scanned(reinterpret_cast<int64_t*>(w + 4 * (nb + 1))), opbeg(w + 6 * (nb + 1)),
        poison(w + 7 * (nb + 1)) {}
};

// slab-local brick of entry r (box order from k0) of a box run
__device__ __forceinline__ int run_brick(const GBox& b, int r, const gsv_bricks& k) {
  const int t = b.k0 + r;
  const int rx = t % b.nb_x, u = t / b.nb_x;
  const int ry = u % b.nb_y, rz = u / b.nb_y;
  return (b.blo_x + rx) + k.bgx * ((b.blo_y + ry) + k.bgy * (b.blo_z + rz)) - k.b0;
}

// edit key: brick << 32 | gid << 1 | insert.  One warp per changed Gaussian:
// the lanes take the bricks of its old and new box runs, keep those not in
// the other run, and the warp reserves its edits with one atomic.
__global__ void __launch_bounds__(128)
incr_ops_kernel(const int32_t* __restrict__ counts, const int32_t* __restrict__ box,
                gsv_bricks k, const int32_t* __restrict__ chg_count,
                const int32_t* __restrict__ chg_gid, const int32_t* __restrict__ chg_old,
                const int32_t* __restrict__ chg_oldcnt, int chg_cap,
                const int32_t* __restrict__ dry, unsigned long long* __restrict__ raw,
                int32_t* __restrict__ nraw, int32_t* __restrict__ bcnt,
                int32_t* __restrict__ bdelta) {
  const int nc = *chg_count;
  if (nc > chg_cap || (dry != nullptr && *dry != 0)) return;
  const int lane = threadIdx.x & 31;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < nc; e += nwarps) {
    const int gid = chg_gid[e];
    const GBox ob = unpack_box(chg_old, e), nbx = unpack_box(box, gid);
    const int oc = chg_oldcnt[e], ncnt = counts[gid];
    const int rounds = (max(oc, ncnt) + 31) >> 5;
    for (int q = 0; q < rounds; ++q) {
      const int r = 32 * q + lane;
      int krm = -1, kin = -1;
      if (r < oc) {
        const int key = run_brick(ob, r, k);
        if (!run_contains(nbx, ncnt, key, k)) krm = key;
      }
      if (r < ncnt) {
        const int key = run_brick(nbx, r, k);
        if (!run_contains(ob, oc, key, k)) kin = key;
      }
      const int m = (krm >= 0) + (kin >= 0);
      int incl = m;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const int tot = __shfl_sync(0xffffffffu, incl, 31);
      if (tot == 0) continue;
      int base = 0;
      if (lane == 0) base = atomicAdd(nraw, tot);   // past kOpsCap: overflow, seen in *nraw
      int j = __shfl_sync(0xffffffffu, base, 0) + incl - m;
      if (krm >= 0) {
        if (j < kOpsCap) {
          raw[j] = ((unsigned long long)(unsigned)krm << 32) | ((unsigned)gid << 1);
          atomicAdd(bcnt + krm, 1);
          atomicAdd(bdelta + krm, -1);
        }
        ++j;
      }
      if (kin >= 0 && j < kOpsCap) {
        raw[j] = ((unsigned long long)(unsigned)kin << 32) | ((unsigned)gid << 1) | 1u;
        atomicAdd(bcnt + kin, 1);
        atomicAdd(bdelta + kin, 1);
      }
    }
  }
}

// packed[b] = new length << 24 | edits of brick b; thread nb also decides the
// step's first overflow conditions
__global__ void __launch_bounds__(256)
incr_len_kernel(const int64_t* __restrict__ starts, int32_t nb, const int32_t* __restrict__ bcnt,
                const int32_t* __restrict__ bdelta, int64_t* __restrict__ packed,
                const int32_t* __restrict__ chg_count, int chg_cap,
                const int32_t* __restrict__ nraw, const int32_t* __restrict__ dry,
                const int32_t* __restrict__ poison, int32_t* __restrict__ overflow) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b > nb) return;
  if (b == nb) {
    packed[b] = 0;
    *overflow = (*chg_count > chg_cap || *nraw > kOpsCap || (dry != nullptr && *dry != 0) ||
                 *poison != 0) ? 1 : 0;
    return;
  }
  const int64_t len = (starts[b + 1] - starts[b]) + bdelta[b];
  packed[b] = (len << 24) | (int64_t)bcnt[b];
}

// split the scan: new starts and edit offsets; the edited lists must hold
// exactly the pairs the counts give (gstart[n]) and fit the capacity
__global__ void __launch_bounds__(256)
incr_split_kernel(const int64_t* __restrict__ scanned, int32_t nb,
                  int64_t* __restrict__ starts_out, int32_t* __restrict__ opbeg,
                  const int64_t* __restrict__ gstart, int64_t n, int64_t cap,
                  int32_t* __restrict__ overflow) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b > nb) return;
  const int64_t v = scanned[b];
  starts_out[b] = v >> 24;
  opbeg[b] = (int32_t)(v & 0xFFFFFF);
  if (b == nb) {
    const int64_t p = v >> 24;
    if (p > cap || p != gstart[n]) *overflow = 1;
  }
}

// the edits into their bricks' segments; the counters return to zero
__global__ void __launch_bounds__(256)
incr_scatter_kernel(const unsigned long long* __restrict__ raw, const int32_t* __restrict__ nraw,
                    const int32_t* __restrict__ opbeg, int32_t* __restrict__ bcnt,
                    int32_t* __restrict__ bdelta, unsigned long long* __restrict__ ops,
                    const int32_t* __restrict__ overflow) {
  if (*overflow != 0) return;
  const int n = *nraw;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const unsigned long long o = raw[i];
    const int key = (int)(o >> 32);
    const int slot = atomicSub(bcnt + key, 1) - 1;
    ops[opbeg[key] + slot] = o;
    bdelta[key] = 0;                          // read by incr_len_kernel already
  }
}

// one warp per brick: copy, or merge the surviving and inserted gids.  A
// brick's edits (at most kMergeSeg; gids are distinct within a brick) are
// ranked by gid into shared memory with the exclusive prefix count of
// insertions, so each old entry finds the edits before it by binary search:
// new index = old index - removals before + insertions before.  Longer edit
// segments take a linear path (order-independent counts).
constexpr int kMergeSeg = 256;

__global__ void __launch_bounds__(256)
incr_merge_kernel(const int64_t* __restrict__ starts, const int32_t* __restrict__ gids,
                  const int64_t* __restrict__ starts_out, int32_t* __restrict__ gids_out,
                  int32_t nb, const unsigned long long* __restrict__ ops,
                  const int32_t* __restrict__ opbeg, const int32_t* __restrict__ overflow) {
  __shared__ unsigned sg[8][kMergeSeg];      // edit gid << 1 | insert, sorted
  __shared__ int spre[8][kMergeSeg + 1];     // insertions before edit q
  const int warp = threadIdx.x >> 5;
  const int b = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (b >= nb || *overflow != 0) return;
  const int64_t os = starts[b], oe = starts[b + 1], ns = starts_out[b];
  const int len = (int)(oe - os);
  const int p0 = opbeg[b], p1 = opbeg[b + 1];
  if (p0 == p1) {
    for (int i = lane; i < len; i += 32) gids_out[ns + i] = gids[os + i];
    return;
  }
  const int seg = p1 - p0;
  if (seg <= kMergeSeg) {
    unsigned* eg = sg[warp];
    int* ep = spre[warp];
    // rank each edit by gid (distinct within the brick) into its sorted slot
    for (int q = lane; q < seg; q += 32) {
      const unsigned v = (unsigned)ops[p0 + q];
      int r = 0;
      for (int u = 0; u < seg; ++u) r += (unsigned)ops[p0 + u] < v;
      eg[r] = v;
    }
    __syncwarp();
    int run = 0;
    for (int q0 = 0; q0 < seg; q0 += 32) {
      const int q = q0 + lane;
      const int ins = (q < seg) ? (int)(eg[q] & 1u) : 0;
      int incl = ins;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      if (q < seg) ep[q] = run + incl - ins;
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) ep[seg] = run;
    __syncwarp();
    // surviving entries, four loads in flight per lane
    for (int i0 = 0; i0 < len; i0 += 128) {
      int gv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + 32 * u + lane;
        gv[u] = i < len ? gids[os + i] : 0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + 32 * u + lane;
        if (i >= len) break;
        const int g = gv[u];
        int lo = 0, hi = seg;                    // first edit with gid >= g
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if ((int)(eg[mid] >> 1) < g) lo = mid + 1; else hi = mid;
        }
        const bool removed = lo < seg && (int)(eg[lo] >> 1) == g && !(eg[lo] & 1u);
        const int in_lt = ep[lo], rm_lt = lo - in_lt;
        if (!removed) gids_out[ns + i - rm_lt + in_lt] = g;
      }
    }
    // inserted entries
    for (int q = lane; q < seg; q += 32) {
      const unsigned v = eg[q];
      if (!(v & 1u)) continue;
      const int h = (int)(v >> 1);
      int lo = 0, hi = len;                      // old entries < h
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (gids[os + mid] < h) lo = mid + 1; else hi = mid;
      }
      const int in_lt = ep[q], rm_lt = q - in_lt;
      gids_out[ns + lo - rm_lt + in_lt] = h;
    }
    return;
  }
  // long edit segments: linear counts
  for (int i = lane; i < len; i += 32) {
    const int g = gids[os + i];
    int rm_lt = 0, in_lt = 0;
    bool removed = false;
    for (int p = p0; p < p1; ++p) {
      const unsigned long long o = ops[p];
      const int og = (int)((unsigned)o >> 1);
      const bool ins = o & 1ull;
      if (og < g) {
        if (ins) ++in_lt; else ++rm_lt;
      } else if (og == g && !ins) {
        removed = true;
      }
    }
    if (!removed) gids_out[ns + i - rm_lt + in_lt] = g;
  }
  for (int p = p0 + lane; p < p1; p += 32) {
    const unsigned long long o = ops[p];
    if (!(o & 1ull)) continue;
    const int h = (int)((unsigned)o >> 1);
    int lo = 0, hi = len;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (gids[os + mid] < h) lo = mid + 1; else hi = mid;
    }
    int rm_lt = 0, in_lt = 0;
    for (int q = p0; q < p1; ++q) {
      const unsigned long long u = ops[q];
      const int ug = (int)((unsigned)u >> 1);
      if (ug < h) {
        if (u & 1ull) ++in_lt; else ++rm_lt;
      }
    }
    gids_out[ns + lo - rm_lt + in_lt] = h;
  }
}

// overflow: empty lists downstream; otherwise (copy_back) the output becomes
// next step's input -- a caller that alternates the two buffers skips the
// copy.  Resets the edit and change counters for the next call (kept after
// an overflow, so steps already queued behind this one overflow too until
// the caller rebuilds).
__global__ void __launch_bounds__(256)
incr_commit_kernel(int64_t* __restrict__ starts, int32_t* __restrict__ gids,
                   int64_t* __restrict__ starts_out, const int32_t* __restrict__ gids_out,
                   int32_t nb, const int32_t* __restrict__ overflow, int copy_back,
                   int32_t* __restrict__ nraw, int32_t* __restrict__ chg_count,
                   const int32_t* __restrict__ dry, int32_t* __restrict__ poison) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (*overflow != 0) {
    for (int64_t i = i0; i <= nb; i += stride) starts_out[i] = 0;
    if (i0 == 0 && !(dry != nullptr && *dry != 0)) *poison = 1;
    return;
  }
  if (i0 == 0) {
    *nraw = 0;
    *chg_count = 0;
  }
  if (!copy_back) return;
  for (int64_t i = i0; i <= nb; i += stride) starts[i] = starts_out[i];
  const int64_t p = starts_out[nb];
  const int64_t p4 = p >> 2;
  const int4* src = reinterpret_cast<const int4*>(gids_out);
  int4* dst = reinterpret_cast<int4*>(gids);
  for (int64_t i = i0; i < p4; i += stride) dst[i] = src[i];
  for (int64_t i = 4 * p4 + i0; i < p; i += stride) gids[i] = gids_out[i];
}

// Slabs of at most 65536 bricks sort 16-bit keys: a quarter less traffic
// per radix pass (the key buffers, allocated for int32, are used at half width).
inline bool keys16(int64_t nb) { return nb <= 65536; }

template <typename K>
cudaError_t sort_pairs(void* ws, size_t& bytes, const int32_t* keys_in, int32_t* keys_out,
                       const int32_t* vals_in, int32_t* vals_out, int count, int bits,
                       cudaStream_t s) {
  return cub::DeviceRadixSort::SortPairs(ws, bytes, reinterpret_cast<const K*>(keys_in),
                                         reinterpret_cast<K*>(keys_out), vals_in, vals_out,
                                         count, 0, bits, s);
}

int key_bits(int64_t nb) {
  int bits = 1;
  while (((int64_t)1 << bits) < nb) ++bits;   // keys are brick ids 0 .. nb-1
  return bits;
}

}  // namespace
}  // namespace gsv

using namespace gsv;

extern "C" {

int gsv_preprocess(const double* positions, const double* log_scales,
                   const double* rotations, const double* raw_amplitude,
                   const double* raw_relax, int64_t n, int relax_enabled,
                   double cutoff_sigma, const gsv_grid* grid,
                   const gsv_bricks* bricks, gsv_record32* rec32,
                   gsv_record64* rec64, int32_t* counts, int32_t* box,
                   void* stream) {
  if (int s = validate_grid_bricks(grid, bricks)) return s;
  GSV_REQUIRE(n >= 0, "n must be >= 0");
  GSV_REQUIRE(cutoff_sigma > 0, "cutoff_sigma must be positive");
  GSV_REQUIRE(n == 0 || (positions && log_scales && rotations && raw_amplitude &&
                         raw_relax && rec32 && counts && box),
              "null pointer argument");
  if (n == 0) return GSV_OK;
  const int dense = isinf(cutoff_sigma) ? 1 : 0;
  const int threads = 256;
  const int64_t blocks = (n + threads - 1) / threads;
  const PrepArgs pa{*grid, *bricks, cutoff_sigma, dense, relax_enabled, rec32, rec64, counts,
                    box};
  preprocess_kernel<<<(unsigned)blocks, threads, 0, as_stream(stream)>>>(
      positions, log_scales, rotations, raw_amplitude, raw_relax, n, pa);
  GSV_CHECK_LAUNCH("preprocess_kernel");
  return GSV_OK;
}

int gsv_bin_workspace(int64_t n, int64_t max_pairs, int32_t nbricks, size_t* bytes) {
  GSV_REQUIRE(bytes != nullptr, "bytes must not be NULL");
  GSV_REQUIRE(max_pairs < (int64_t)INT32_MAX, "pair count %lld exceeds int32",
              (long long)max_pairs);
  size_t scan_bytes = 0, sort_bytes = 0;
  thrust::transform_iterator<ToI64, const int32_t*, int64_t> it(nullptr, ToI64());
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, it, (int64_t*)nullptr,
                                                (int)(n > 0 ? n : 1));
  if (e != cudaSuccess) return cuda_status(e, "DeviceScan sizing");
  {
    const int cnt = (int)(max_pairs > 0 ? max_pairs : 1);
    e = keys16(nbricks)
            ? sort_pairs<uint16_t>(nullptr, sort_bytes, nullptr, nullptr, nullptr, nullptr, cnt,
                                   key_bits(nbricks), nullptr)
            : sort_pairs<int32_t>(nullptr, sort_bytes, nullptr, nullptr, nullptr, nullptr, cnt,
                                  key_bits(nbricks), nullptr);
  }
  if (e != cudaSuccess) return cuda_status(e, "DeviceRadixSort sizing");
  *bytes = (scan_bytes > sort_bytes ? scan_bytes : sort_bytes) + 256;
  return GSV_OK;
}

int gsv_bin_scan(const int32_t* counts, int64_t n, int64_t* gstart, void* workspace,
                 size_t workspace_bytes, void* stream) {
  GSV_REQUIRE(n >= 0 && n < (int64_t)INT32_MAX, "n out of range");
  cudaStream_t s = as_stream(stream);
  if (n == 0) {
    cudaError_t e = cudaMemsetAsync(gstart, 0, sizeof(int64_t), s);
    if (e != cudaSuccess) return cuda_status(e, "memset gstart");
    return GSV_OK;
  }
  thrust::transform_iterator<ToI64, const int32_t*, int64_t> it(counts, ToI64());
  size_t bytes = workspace_bytes;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(workspace, bytes, it, gstart, (int)n, s);
  if (e != cudaSuccess) return cuda_status(e, "DeviceScan::ExclusiveSum");
  scan_tail_kernel<<<1, 1, 0, s>>>(counts, n, gstart);
  GSV_CHECK_LAUNCH("scan_tail_kernel");
  return GSV_OK;
}

int gsv_bin_fill(const int32_t* counts, const int32_t* box, const int64_t* gstart,
                 int64_t n, int64_t pairs, const gsv_bricks* bricks, int32_t* keys_tmp,
                 int32_t* vals_tmp, int32_t* keys_out, int32_t* gids_out,
                 int64_t* starts_out, void* workspace, size_t workspace_bytes,
                 void* stream) {
  GSV_REQUIRE(bricks != nullptr, "bricks must not be NULL");
  GSV_REQUIRE(pairs >= 0 && pairs < (int64_t)INT32_MAX, "pair count %lld exceeds int32",
              (long long)pairs);
  cudaStream_t s = as_stream(stream);
  const int64_t nb = slab_bricks(*bricks);
  const bool k16 = keys16(nb);
  if (pairs > 0) {
    if (k16)
      emit_warp_kernel<uint16_t><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(
          counts, box, gstart, n, *bricks, reinterpret_cast<uint16_t*>(keys_tmp), vals_tmp,
          INT64_MAX);
    else
      emit_warp_kernel<int32_t><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(
          counts, box, gstart, n, *bricks, keys_tmp, vals_tmp, INT64_MAX);
    GSV_CHECK_LAUNCH("emit_warp_kernel");
    size_t bytes = workspace_bytes;
    cudaError_t e = k16 ? sort_pairs<uint16_t>(workspace, bytes, keys_tmp, keys_out, vals_tmp,
                                               gids_out, (int)pairs, key_bits(nb), s)
                        : sort_pairs<int32_t>(workspace, bytes, keys_tmp, keys_out, vals_tmp,
                                              gids_out, (int)pairs, key_bits(nb), s);
    if (e != cudaSuccess) return cuda_status(e, "DeviceRadixSort::SortPairs");
  }
  if (k16)
    starts_search_kernel<uint16_t><<<(unsigned)((nb + 1 + 255) / 256), 256, 0, s>>>(
        reinterpret_cast<const uint16_t*>(keys_out), pairs, (int32_t)nb, starts_out, nullptr,
        nullptr);
  else
    starts_search_kernel<int32_t><<<(unsigned)((nb + 1 + 255) / 256), 256, 0, s>>>(
        keys_out, pairs, (int32_t)nb, starts_out, nullptr, nullptr);
  GSV_CHECK_LAUNCH("starts_search_kernel");
  return GSV_OK;
}

int gsv_bin_fill_capacity(const int32_t* counts, const int32_t* box, const int64_t* gstart,
                          int64_t n, int64_t capacity, const gsv_bricks* bricks,
                          int32_t* keys_tmp, int32_t* vals_tmp, int32_t* keys_out,
                          int32_t* gids_out, int64_t* starts_out, const int32_t* dry,
                          int32_t* overflow, void* workspace, size_t workspace_bytes,
                          void* stream) {
  GSV_REQUIRE(bricks != nullptr && overflow != nullptr, "null bricks/overflow");
  GSV_REQUIRE(capacity >= 1 && capacity < (int64_t)INT32_MAX, "capacity %lld out of range",
              (long long)capacity);
  cudaStream_t s = as_stream(stream);
  const int64_t nb = slab_bricks(*bricks);
  const bool k16 = keys16(nb);
  uint16_t* kt16 = reinterpret_cast<uint16_t*>(keys_tmp);
  if (n > 0) {
    if (k16)
      emit_warp_kernel<uint16_t><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(
          counts, box, gstart, n, *bricks, kt16, vals_tmp, capacity);
    else
      emit_warp_kernel<int32_t><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(
          counts, box, gstart, n, *bricks, keys_tmp, vals_tmp, capacity);
    GSV_CHECK_LAUNCH("emit_warp_kernel");
  }
  if (k16)
    pad_kernel<uint16_t><<<592, 256, 0, s>>>(gstart, n, capacity, (int32_t)nb, dry, kt16,
                                             vals_tmp, overflow);
  else
    pad_kernel<int32_t><<<592, 256, 0, s>>>(gstart, n, capacity, (int32_t)nb, dry, keys_tmp,
                                            vals_tmp, overflow);
  GSV_CHECK_LAUNCH("pad_kernel");
  size_t bytes = workspace_bytes;
  cudaError_t e = k16 ? sort_pairs<uint16_t>(workspace, bytes, keys_tmp, keys_out, vals_tmp,
                                             gids_out, (int)capacity, key_bits(nb), s)
                      : sort_pairs<int32_t>(workspace, bytes, keys_tmp, keys_out, vals_tmp,
                                            gids_out, (int)capacity, key_bits(nb), s);
  if (e != cudaSuccess) return cuda_status(e, "DeviceRadixSort::SortPairs");
  if (k16)
    starts_search_kernel<uint16_t><<<(unsigned)((nb + 1 + 255) / 256), 256, 0, s>>>(
        reinterpret_cast<const uint16_t*>(keys_out), capacity, (int32_t)nb, starts_out,
        overflow, gstart + n);
  else
    starts_search_kernel<int32_t><<<(unsigned)((nb + 1 + 255) / 256), 256, 0, s>>>(
        keys_out, capacity, (int32_t)nb, starts_out, overflow, gstart + n);
  GSV_CHECK_LAUNCH("starts_search_kernel");
  return GSV_OK;
}

int gsv_lists_unsorted(const int64_t* starts, const int32_t* gids, int32_t nbricks,
                       int64_t pairs, int32_t* flag, void* stream) {
  (void)pairs;
  cudaStream_t s = as_stream(stream);
  cudaError_t e = cudaMemsetAsync(flag, 0, sizeof(int32_t), s);
  if (e != cudaSuccess) return cuda_status(e, "memset flag");
  if (nbricks <= 0) return GSV_OK;
  unsorted_kernel<<<(nbricks + 255) / 256, 256, 0, s>>>(starts, gids, nbricks, flag);
  GSV_CHECK_LAUNCH("unsorted_kernel");
  return GSV_OK;
}

int gsv_canonicalize_workspace(int64_t pairs, int32_t nbricks, size_t* bytes) {
  GSV_REQUIRE(bytes != nullptr, "bytes must not be NULL");
  size_t b = 0;
  cudaError_t e = cub::DeviceSegmentedSort::SortKeys(
      nullptr, b, (const int32_t*)nullptr, (int32_t*)nullptr, (int)(pairs > 0 ? pairs : 1),
      nbricks > 0 ? nbricks : 1, (const int64_t*)nullptr, (const int64_t*)nullptr);
  if (e != cudaSuccess) return cuda_status(e, "DeviceSegmentedSort sizing");
  *bytes = b + 256;
  return GSV_OK;
}

int gsv_canonicalize(const int64_t* starts, const int32_t* gids_in, int32_t* gids_out,
                     int32_t nbricks, int64_t pairs, void* workspace,
                     size_t workspace_bytes, void* stream) {
  GSV_REQUIRE(pairs >= 0 && pairs < (int64_t)INT32_MAX, "pair count exceeds int32");
  if (pairs == 0 || nbricks == 0) return GSV_OK;
  size_t bytes = workspace_bytes;
  cudaError_t e = cub::DeviceSegmentedSort::SortKeys(workspace, bytes, gids_in, gids_out,
                                                     (int)pairs, nbricks, starts, starts + 1,
                                                     as_stream(stream));
  if (e != cudaSuccess) return cuda_status(e, "DeviceSegmentedSort::SortKeys");
  return GSV_OK;
}

int gsv_preprocess_track(const double* positions, const double* log_scales,
                         const double* rotations, const double* raw_amplitude,
                         const double* raw_relax, int64_t n, int relax_enabled,
                         double cutoff_sigma, const gsv_grid* grid, const gsv_bricks* bricks,
                         gsv_record32* rec32, int32_t* counts, int32_t* box,
                         int32_t* chg_count, int32_t* chg_gid, int32_t* chg_old,
                         int32_t* chg_oldcnt, int chg_cap, void* stream) {
  if (int s = validate_grid_bricks(grid, bricks)) return s;
  GSV_REQUIRE(n >= 0, "n must be >= 0");
  GSV_REQUIRE(cutoff_sigma > 0, "cutoff_sigma must be positive");
  GSV_REQUIRE(chg_count && chg_gid && chg_old && chg_oldcnt && chg_cap >= 0,
              "null change-tracking buffer");
  GSV_REQUIRE(n == 0 || (positions && log_scales && rotations && raw_amplitude &&
                         raw_relax && rec32 && counts && box),
              "null pointer argument");
  if (n == 0) return GSV_OK;
  const int dense = isinf(cutoff_sigma) ? 1 : 0;
  const int threads = 256;
  const int64_t blocks = (n + threads - 1) / threads;
  const PrepArgs pa{*grid, *bricks, cutoff_sigma, dense, relax_enabled, rec32, nullptr, counts,
                    box, chg_count, chg_gid, chg_old, chg_oldcnt, chg_cap};
  preprocess_kernel<<<(unsigned)blocks, threads, 0, as_stream(stream)>>>(
      positions, log_scales, rotations, raw_amplitude, raw_relax, n, pa);
  GSV_CHECK_LAUNCH("preprocess_kernel");
  return GSV_OK;
}

int gsv_bin_incremental_workspace(int32_t nbricks, size_t* bytes) {
  GSV_REQUIRE(bytes != nullptr, "bytes must not be NULL");
  size_t scan_bytes = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (const int64_t*)nullptr,
                                                (int64_t*)nullptr, (int)nbricks + 1);
  if (e != cudaSuccess) return cuda_status(e, "DeviceScan sizing");
  *bytes = scan_bytes + 256;
  return GSV_OK;
}

int gsv_bin_incremental(const int32_t* counts, const int32_t* box, const int64_t* gstart,
                        int64_t n, int64_t capacity,
                        const gsv_bricks* bricks, int32_t* chg_count, const int32_t* chg_gid,
                        const int32_t* chg_old, const int32_t* chg_oldcnt, int chg_cap,
                        int64_t* starts, int32_t* gids, int64_t* starts_out, int32_t* gids_out,
                        unsigned long long* ops, int32_t* nops, int32_t* lens,
                        const int32_t* dry, int32_t* overflow, int copy_back,
                        void* workspace, size_t workspace_bytes, void* stream) {
  GSV_REQUIRE(bricks && counts && box && gstart && chg_count && chg_gid && chg_old && chg_oldcnt &&
                  starts && gids && starts_out && gids_out && ops && nops && lens && overflow,
              "null pointer argument");
  GSV_REQUIRE(capacity >= 1 && capacity < (int64_t)INT32_MAX, "capacity %lld out of range",
              (long long)capacity);
  GSV_REQUIRE((reinterpret_cast<uintptr_t>(lens) & 7) == 0, "lens must be 8-byte aligned");
  cudaStream_t s = as_stream(stream);
  const int64_t nb = slab_bricks(*bricks);
  const IncrScratch w(lens, nb);
  unsigned long long* raw = ops;
  unsigned long long* sorted = ops + kOpsCap;
  const unsigned gb = (unsigned)((nb + 1 + 255) / 256);
  // one warp per changed Gaussian (chg_cap warps: idle ones exit at once)
  incr_ops_kernel<<<(unsigned)((chg_cap + 3) / 4), 128, 0, s>>>(counts, box, *bricks, chg_count,
                                                                chg_gid, chg_old,
                                     chg_oldcnt, chg_cap, dry, raw, nops, w.bcnt, w.bdelta);
  GSV_CHECK_LAUNCH("incr_ops_kernel");
  incr_len_kernel<<<gb, 256, 0, s>>>(starts, (int32_t)nb, w.bcnt, w.bdelta, w.packed, chg_count,
                                     chg_cap, nops, dry, w.poison, overflow);
  GSV_CHECK_LAUNCH("incr_len_kernel");
  size_t bytes = workspace_bytes;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(workspace, bytes, w.packed, w.scanned,
                                                (int)nb + 1, s);
  if (e != cudaSuccess) return cuda_status(e, "DeviceScan::ExclusiveSum");
  incr_split_kernel<<<gb, 256, 0, s>>>(w.scanned, (int32_t)nb, starts_out, w.opbeg, gstart, n,
                                       capacity, overflow);
  GSV_CHECK_LAUNCH("incr_split_kernel");
  incr_scatter_kernel<<<16, 256, 0, s>>>(raw, nops, w.opbeg, w.bcnt, w.bdelta, sorted, overflow);
  GSV_CHECK_LAUNCH("incr_scatter_kernel");
  if (nb > 0) {
    incr_merge_kernel<<<(unsigned)((nb * 32 + 255) / 256), 256, 0, s>>>(
        starts, gids, starts_out, gids_out, (int32_t)nb, sorted, w.opbeg, overflow);
    GSV_CHECK_LAUNCH("incr_merge_kernel");
  }
  // without the copy only the overflow case and the counter reset have work
  incr_commit_kernel<<<copy_back ? 1184 : 32, 256, 0, s>>>(
      starts, gids, starts_out, gids_out, (int32_t)nb, overflow, copy_back, nops, chg_count, dry,
      w.poison);
  GSV_CHECK_LAUNCH("incr_commit_kernel");
  return GSV_OK;
}

}  // extern "C"
