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

__global__ void __launch_bounds__(256, 4)
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

}  // extern "C"
