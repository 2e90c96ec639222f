/*
 * gsv.h -- C ABI of the B200 brick rasterizer (libgsv_b200.so).
 *
 * Drop-in boundary for the hot path of the reference package `gsvol`
 * (arxiv/paper_2603_09621).  The reference has no native FFI: its kernels are
 * numba @njit functions that take flat positional SoA arrays, scalars and
 * caller-allocated outputs (SURVEY.md §8b "Kernel-level ABI").  Every entry
 * point below replaces one of those call sites; the cited file:line is the
 * reference code whose semantics it reproduces (paths relative to
 * /root/reference/pkg/src/gsvol/).
 *
 * Conventions
 *  - All array pointers are DEVICE pointers (cudaMalloc / torch CUDA storage),
 *    except where a parameter says "host".  The library never allocates device
 *    memory: outputs and workspaces belong to the caller (raster.py:305-307,
 *    494-497, 517-520 -- the reference wrapper allocates every output too).
 *  - `stream` is a cudaStream_t passed as void*; every call only enqueues work
 *    on it (no device synchronisation) unless documented otherwise.
 *  - Field arrays are float64, C-contiguous, in GaussianField's SoA layout
 *    (field.py:33-70): positions (N,3), log_scales (N,3), rotations (N,4) with
 *    the quaternion scalar-first (w,x,y,z), raw_amplitude (N), raw_relax (N).
 *  - Volumes are linear, x-fastest: lin = ix + nx*(iy + ny*iz)
 *    (volume.py:100-102, raster.py:271).
 *  - Brick b covers voxels [bx*bdx, ...) with b = bx + bgx*(by + bgy*bz)
 *    (raster.py:209, 247-256).
 *  - Return value: GSV_OK (0) or a gsv_status code; gsv_last_error() returns
 *    a thread-local message for the last failure.
 */
#ifndef GSV_B200_H
#define GSV_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ABI history: 2 -- graph step, metrics, geometry helpers; 3 -- gsv_bricks
 * carries a brick-id range [b0, b1) instead of whole z-layers [bz0, bz1),
 * and the box record's 4th word holds k0 (see gsv_preprocess); 4 -- live
 * masks are pair-major (P x 4 uint2, see gsv_forward); 5 -- gsv_forward takes
 * the fused loss's target as float32 or float64 (target_dtype), vpl 16 (the
 * grouped-column forward, its column-nibble masks = gsv_backward mask_vpl
 * 16), and the device setup entry points (resample, init); 6 -- adds
 * gsv_step_advance_publish (the graph step's result into a pinned ring) and
 * incremental binning (gsv_preprocess_track, gsv_bin_incremental). */
#define GSV_ABI_VERSION 6

typedef enum {
  GSV_OK = 0,
  GSV_ERR_ARG = 1,      /* invalid argument (shape, null pointer, range) */
  GSV_ERR_CUDA = 2,     /* a CUDA runtime call failed */
  GSV_ERR_CAPACITY = 3, /* a count exceeds what the caller allocated / int32 */
} gsv_status;

/* Cell-centred sampling lattice; origin is the centre of voxel (0,0,0)
 * (volume.py:16-41 GridSpec). */
typedef struct {
  int32_t nx, ny, nz;
  int32_t _pad;
  double ox, oy, oz;
  double sx, sy, sz;
} gsv_grid;

/* Brick decomposition (raster.py:152-156) plus the slab this call owns: the
 * contiguous brick-id range [b0, b1) (bricks numbered x-fastest,
 * raster.py:209).  A whole-grid call uses b0 = 0, b1 = bgx*bgy*bgz.  Any
 * contiguous range is an exact slice of the global index, so
 * slabs may cut a brick layer anywhere: whole z-layers are the special case
 * b0, b1 multiples of bgx*bgy. */
typedef struct {
  int32_t bdx, bdy, bdz;
  int32_t bgx, bgy, bgz;
  int32_t b0, b1;
} gsv_bricks;

/* Per-Gaussian fp32 record consumed by the pair kernels (64 bytes). */
typedef struct {
  float l[9];      /* whitening factor L = diag(exp(-ls)) R^T, row-major     */
  float amp;       /* A = sigmoid(raw_amplitude)                            */
  float relax;     /* r = sigmoid(raw_relax), or 1 when relax is disabled    */
  float half[3];   /* cutoff*sqrt(Sigma_kk): world-axis half extents        */
  float inv_smax2; /* 1/sigma_max^2 = smallest eigenvalue of L^T L          */
  float _pad;
} gsv_record32;

/* Per-Gaussian fp64 record for the f64 engine (precision="f64"). */
typedef struct {
  double l[9];
  double amp;
  double relax;
  double _pad;
} gsv_record64;

int gsv_abi_version(void);
const char* gsv_last_error(void);
/* Number of SMs of the current device (host query, for grid sizing). */
int gsv_device_sm_count(void);

/* ------------------------------------------------------------------------
 * Preprocess + bin count: one fused per-Gaussian kernel.
 * Replaces field.rotation_matrices (field.py:141-154), _whitening_factors
 * (raster.py:233-237), activated_amplitude / activated_relax
 * (field.py:86-94) and the per-Gaussian AABB part of build_brick_index
 * (raster.py:175-198), computed in f64 with the reference's unfused operation
 * order (numpy einsum "nkm,nm->nk" sums (p0+p2)+p1).
 *   rec32  (N)   : gsv_record32, always written
 *   rec64  (N)   : gsv_record64, written when non-NULL (required by the f64
 *                  engine; the f32 engine recomputes the f64 factor from
 *                  log_scales/rotations in its rare guard-band path)
 *   counts (N)   : pairs Gaussian i emits inside the slab (0 if outside)
 *   box    (N,4) : int32 {blo_x | blo_y<<16, blo_z | nb_x<<16, nb_y | nb_z<<16, k0}
 *                  brick box of Gaussian i clipped to the slab's brick layers;
 *                  k0 = box-order (x-fastest) index of its first brick inside
 *                  [b0, b1): the slab's bricks of the box are the box-order
 *                  run [k0, k0 + counts[i]) (box order and brick-id order are
 *                  both lexicographic in (z, y, x)).
 * cutoff_sigma may be +inf (dense lists, raster.py:166-171).
 * ------------------------------------------------------------------------ */
int gsv_preprocess(const double* positions, const double* log_scales,
                   const double* rotations, const double* raw_amplitude,
                   const double* raw_relax, int64_t n, int relax_enabled,
                   double cutoff_sigma, const gsv_grid* grid,
                   const gsv_bricks* bricks, gsv_record32* rec32,
                   gsv_record64* rec64, int32_t* counts, int32_t* box,
                   void* stream);

/* Workspace bytes needed by gsv_bin_scan / gsv_bin_fill (CUB temp storage).*/
int gsv_bin_workspace(int64_t n, int64_t max_pairs, int32_t nbricks,
                      size_t* bytes);

/* Exclusive scan of counts -> gstart (N+1, int64).  gstart[N] = P.  The
 * caller reads gstart[N] (one 8-byte D2H) to size the pair buffers. */
int gsv_bin_scan(const int32_t* counts, int64_t n, int64_t* gstart,
                 void* workspace, size_t workspace_bytes, void* stream);

/* Emit (brick, gid) pairs in gid-major order (raster.py:200-209), stable
 * radix sort by brick id (raster.py:211-216; LSD radix sort is stable so
 * each brick's list is ascending in gid), CSR starts for the slab's bricks.
 *   keys_tmp, vals_tmp, keys_out : int32 (P) scratch
 *   gids_out : int32 (P), starts_out : int64 (nbricks_slab + 1). */
int gsv_bin_fill(const int32_t* counts, const int32_t* box,
                 const int64_t* gstart, int64_t n, int64_t pairs,
                 const gsv_bricks* bricks, int32_t* keys_tmp,
                 int32_t* vals_tmp, int32_t* keys_out, int32_t* gids_out,
                 int64_t* starts_out, void* workspace, size_t workspace_bytes,
                 void* stream);

/* Capacity mode of gsv_bin_fill for host-sync-free (CUDA-graph) steps: the
 * pair count P = gstart[N] is never read by the host.  Pairs fill slots
 * [0, P) as in gsv_bin_fill, slots [P, capacity) get the last brick id
 * (the stable sort keeps them behind that brick's pairs; starts[nbricks] = P
 * cuts them off), and the sort always covers `capacity` slots.  *overflow (device int32) = P > capacity, or *dry != 0
 * (dry may be NULL); on overflow every list is emptied (starts = 0) so the
 * downstream kernels do no work and the caller re-bins with more capacity.
 * Buffers as gsv_bin_fill, sized by capacity; workspace from
 * gsv_bin_workspace(n, capacity, nbricks). */
int gsv_bin_fill_capacity(const int32_t* counts, const int32_t* box,
                          const int64_t* gstart, int64_t n, int64_t capacity,
                          const gsv_bricks* bricks, int32_t* keys_tmp,
                          int32_t* vals_tmp, int32_t* keys_out, int32_t* gids_out,
                          int64_t* starts_out, const int32_t* dry, int32_t* overflow,
                          void* workspace, size_t workspace_bytes, void* stream);

/* Incremental binning for consecutive fit() iterations (CUDA-graph
 * capturable).  gsv_preprocess_track is gsv_preprocess (f32 records only)
 * that also appends every Gaussian whose pair count or box record differs
 * from the values counts / box held before the call: chg_gid[e], chg_old[4 e
 * .. 4 e + 3] (the old box record), chg_oldcnt[e], e = atomicAdd(chg_count);
 * entries beyond chg_cap are dropped (the count still grows).
 * gsv_bin_incremental turns the recorded changes into per-brick edits and
 * rebuilds the lists (starts, gids: the lists of the OLD boxes, capacity
 * entries) for the current counts / box: starts_out (nbricks_slab + 1) and
 * gids_out are the new lists, copied back into starts / gids for the next
 * call when copy_back != 0 (otherwise the caller swaps the two buffer pairs
 * for the next call); *chg_count is reset.  The result equals gsv_bin_fill for the current
 * boxes (each list ascending in gid).  *overflow = more than chg_cap changes,
 * more than 16384 edits, more than capacity pairs, edited lists whose pair
 * count differs from gstart[n] (gsv_bin_scan of counts), or *dry != 0 -- then
 * starts_out is all zero (empty lists downstream) and starts / gids are left
 * as they were (after an excess of changes or edits *chg_count is left above
 * chg_cap, so later calls overflow too); the caller rebuilds from scratch.
 * Scratch: ops (2 x 16384 uint64), nops (1 int32, zero before the first
 * call), lens (8 (nbricks_slab + 1) int32, 8-byte aligned, zero before the
 * first call; after an overflow the scratch is poisoned and every later call
 * overflows until it is zeroed again); workspace from gsv_bin_incremental_workspace(nbricks_slab). */
int gsv_preprocess_track(const double* positions, const double* log_scales,
                         const double* rotations, const double* raw_amplitude,
                         const double* raw_relax, int64_t n, int relax_enabled,
                         double cutoff_sigma, const gsv_grid* grid, const gsv_bricks* bricks,
                         gsv_record32* rec32, int32_t* counts, int32_t* box,
                         int32_t* chg_count, int32_t* chg_gid, int32_t* chg_old,
                         int32_t* chg_oldcnt, int chg_cap, void* stream);
int gsv_bin_incremental_workspace(int32_t nbricks, size_t* bytes);
int gsv_bin_incremental(const int32_t* counts, const int32_t* box, const int64_t* gstart,
                        int64_t n, int64_t capacity,
                        const gsv_bricks* bricks, int32_t* chg_count, const int32_t* chg_gid,
                        const int32_t* chg_old, const int32_t* chg_oldcnt, int chg_cap,
                        int64_t* starts, int32_t* gids, int64_t* starts_out, int32_t* gids_out,
                        unsigned long long* ops, int32_t* nops, int32_t* lens,
                        const int32_t* dry, int32_t* overflow, int copy_back,
                        void* workspace, size_t workspace_bytes, void* stream);

/* Canonical-order check and repair for caller-supplied lists
 * (BrickIndex.lists_sorted / canonicalized, raster.py:91-112).
 * gsv_lists_unsorted writes 1 to *flag (device int32) if any brick list is
 * not strictly ascending.  gsv_canonicalize sorts every list ascending. */
int gsv_lists_unsorted(const int64_t* starts, const int32_t* gids,
                       int32_t nbricks, int64_t pairs, int32_t* flag,
                       void* stream);
int gsv_canonicalize_workspace(int64_t pairs, int32_t nbricks, size_t* bytes);
int gsv_canonicalize(const int64_t* starts, const int32_t* gids_in,
                     int32_t* gids_out, int32_t nbricks, int64_t pairs,
                     void* workspace, size_t workspace_bytes, void* stream);

/* The fused loss epilogue of the 8x8x4 f32 forward as its own pass, for a
 * step whose target is still in flight over PCIe while the forward runs
 * (gsv_forward with target NULL, then this): from the forward's W and I,
 * writes ab = {dL/dI / W, I} and loss_part (one per brick of the slab) with
 * the same voxel order per brick as the forward kernel selected by vpl (16:
 * grouped, 8: whole brick), so both are bit-identical to the fused forward's.
 * Also added in ABI 6. */
int gsv_loss_bricks(const gsv_grid* grid, const gsv_bricks* bricks, double eps_w,
                    const float* W, const float* I, const void* target, int target_dtype,
                    int loss_kind, double vox_count, int vpl, float* ab, double* loss_part,
                    void* stream);

/* ------------------------------------------------------------------------
 * Forward render, CTA per brick.  Replaces _forward_kernel
 * (raster.py:240-293).  precision 0 = f32 (S/W/I float32; truncation decided
 * exactly in f64 inside a guard band), 1 = f64 (S/W/I float64, rec64 needed).
 * The slab's voxels only are written.  If target != NULL the L1/L2 loss of
 * optimize.loss_and_grad (optimize.py:91-103) is fused into the epilogue:
 *   ab (V,2) float : {alpha, I} with alpha = dL/dI / W (0 where W < eps_w or
 *                    dL/dI == 0), the backward's per-voxel inputs;
 *   loss_part (nbricks_slab) double : per-brick sum |I-T| (l1) or (I-T)^2.
 * target_dtype: 0 = target is float32 (V), 1 = float64 (V); the difference
 * I - T is taken in float64 either way, as optimize.py:97 does with the
 * target volume's own dtype.
 * loss_kind: 0 = l1, 1 = l2.  vox_count = global voxel count V, so
 * dL/dI = sign(I-T)/V (l1) or 2(I-T)/V (l2) exactly as optimize.py:99-102.
 * vpl: the f32 kernel: 2 (4x4x4 warp tiles when the brick dims are
 * multiples of 4, 4 warps per 8x8x4 brick), 4 (columns of 4 in z: 8x4x4
 * tiles, 2 warps), 8 (8x8x4 bricks only: one warp per brick, two columns
 * per lane, one hit list per y-half), 16 (8x8x4 bricks only: grouped
 * columns -- consecutive pairs with the same footprint rectangle form a
 * group, whose columns are dealt to the lanes; fastest at LR densities; the
 * Python API uses it when pairs <= 8 x the Gaussians reaching the index), or
 * 0 = auto (8 for 8x8x4 bricks, else 4 when bdz % 4 == 0 and the brick has
 * <= 64 columns, else 2).  S, W, I are bit-identical for a given vpl; across
 * vpl 8 and 16 they agree to f32 rounding (different association).
 * live_masks (optional, f32): P x 4 uint2 (pair-major: a pair's 8 words are
 * 32 contiguous bytes), the forward's exact truncation decisions, consumed by
 * gsv_backward so it walks only live voxels.  Word w of a pair (uint2 w/2,
 * .x/.y = w%2) holds, for vpl 2/4/8, the live bits of warp tile w/v at
 * depth w%v, bit = lane (v = 4 for vpl 8, whose masks use the VPL-4
 * layout); for vpl 16, brick row y = w, bit 4x + z.  Pass gsv_backward the
 * matching mask_vpl (4 for vpl 8, 16 for vpl 16).  Requires a brick that
 * fills the CTA's warp tiles exactly (vpl 2: 128 columns of 2; vpl 4: 64 of
 * 4 -- e.g. 8x8x4).
 * ------------------------------------------------------------------------ */
int gsv_forward(const double* positions, const double* log_scales,
                const double* rotations, const gsv_record32* rec32,
                const gsv_record64* rec64, const int64_t* starts,
                const int32_t* gids, const gsv_grid* grid,
                const gsv_bricks* bricks, double cutoff_sigma, double eps_w,
                int precision, void* S, void* W, void* I,
                const void* target, int target_dtype, int loss_kind,
                double vox_count, float* ab, double* loss_part,
                uint32_t* live_masks, int vpl, void* stream);

/* Per-voxel backward inputs from (W, I, dL/dI) for the unfused API path
 * (raster.py:484-508).  dldi is float64 (V).  Writes ab (V,2) = {dL/dI / W, I}
 * in the precision's type and *bad (device int64) = first non-finite voxel index or
 * -1.  Slab voxels only (the voxels of bricks [b0, b1)). */
int gsv_backward_prep(const void* W, const void* I, const double* dldi,
                      const gsv_grid* grid, const gsv_bricks* bricks,
                      double eps_w, int precision, void* ab, int64_t* bad,
                      void* stream);

/* Backward pair pass, per-pair partial gradients.  Replaces _backward_kernel
 * (raster.py:322-409).  Writes for every pair of the slab its 11 partials
 * {d_amp, d_relax, d_mu[3], G6[6]} (G6 = g00,g11,g22,g01,g02,g12) into
 * partials[(e)*12 ...] where e is the pair's gid-major emission index
 * gstart[gid] + rank of the brick in the Gaussian's box -- i.e. the order
 * the reference merges in (raster.py:512-516: stable argsort by gid keeps
 * ascending brick order).  partials: float (f32) or double (f64), (P,12).
 * live_masks: the masks gsv_forward wrote for the same index (f32 only), or
 * NULL to find live voxels from exact per-row spans; mask_vpl: the masks'
 * layout -- 2 or 4 (warp tiles; 4 also for gsv_forward vpl 8), 16 (the
 * grouped forward's row/column-nibble layout), or 0 = mask_units' auto rule
 * for the warp-tile kernels. */
int gsv_backward(const double* positions, const double* log_scales,
                 const double* rotations, const gsv_record32* rec32,
                 const gsv_record64* rec64, const int64_t* starts,
                 const int32_t* gids, const int64_t* gstart,
                 const int32_t* box, const gsv_grid* grid,
                 const gsv_bricks* bricks, double cutoff_sigma,
                 int precision, const void* ab, const uint32_t* live_masks,
                 int mask_vpl, void* partials, void* stream);

/* Deterministic per-Gaussian merge of pair partials in ascending brick order
 * (_merge_pairs_kernel, raster.py:412-451).  gsum (N,12) double. */
int gsv_merge(const void* partials, const int64_t* gstart, int64_t n,
              int precision, double* gsum, void* stream);

/* Chain rule to raw-parameter gradients (raster.py:524-549,
 * _rotation_jacobians 454-467).  Outputs f64 arrays in GradientBuffer layout
 * (raster.py:128-145). */
int gsv_chain_rule(const double* gsum, const double* log_scales,
                   const double* rotations, const double* raw_amplitude,
                   const double* raw_relax, int64_t n, int relax_enabled,
                   double* g_raw_amplitude, double* g_raw_relax,
                   double* g_positions, double* g_log_scales,
                   double* g_rotations, void* stream);

/* loss_and_grad (optimize.py:91-103).  pred/target float32 or float64 (V)
 * per pred_f64/target_f64; grad float64 (V); loss_part (nblocks) double where
 * nblocks = gsv_loss_blocks(V).  The caller sums loss_part (gsv_sum) and
 * divides by V. */
int gsv_loss_blocks(int64_t v);
int gsv_loss(const void* pred, int pred_f64, const void* target,
             int target_f64, int64_t v, int loss_kind, double* grad,
             double* loss_part, void* stream);

/* Deterministic sum of a double array into *out (single-CTA tree). */
int gsv_sum(const double* x, int64_t n, double* out, void* stream);

/* One Adam step on one parameter group (step_optimizer, optimize.py:127-148):
 * m = b1*m + (1-b1)*g; v = b2*v + ((1-b2)*g)*g;
 * p -= lr*(m/bc1) / (sqrt(v/bc2) + eps), unfused f64 like numpy. */
int gsv_adam(double* p, double* m, double* v, const double* g, int64_t count,
             double lr, double beta1, double beta2, double eps, double bc1,
             double bc2, void* stream);

/* Adam hyper-parameters of one step: per-group learning rates in field order
 * positions, log_scales, rotations, raw_amplitude, raw_relax
 * (FitConfig.resolved_lrs, optimize.py:62-74) and the bias corrections
 * bc1 = 1 - b1^t, bc2 = 1 - b2^t computed by the caller (optimize.py:131-132). */
typedef struct {
  double lr[5];
  double b1, b2, eps, bc1, bc2;
} gsv_adam_hparams;

/* The optimizer tail of one fit() iteration fused into one pass over the
 * per-Gaussian state: merge of the pair partials in ascending brick order
 * (or, when gsum != NULL, the already all-reduced sums (N,12) double), chain
 * rule (raster.py:524-549), Adam on every enabled group (optimize.py:127-148)
 * and quaternion renormalisation (field.py:100-102).  Same arithmetic as
 * gsv_merge + gsv_chain_rule + gsv_adam + gsv_normalize_rotations.
 * moments: host array of 10 device pointers {m_pos, m_ls, m_rot, m_amp,
 * m_rel, v_pos, v_ls, v_rot, v_amp, v_rel} (AdamState.m / .v).
 * grad_scratch: NULL for the one-pass f32 kernel (default); else an (N,12)
 * double workspace for the two-kernel path (merge+chain, then streaming
 * Adam), required for precision 1. */
int gsv_fused_update(const void* partials, const int64_t* gstart, const double* gsum,
                     int64_t n, int precision, double* positions, double* log_scales,
                     double* rotations, double* raw_amplitude, double* raw_relax,
                     double* const* moments, int amplitude_enabled, int relax_enabled,
                     const gsv_adam_hparams* hp, double* grad_scratch, void* stream);

/* Device-side control of a graph-replayed fit() iteration (optimize.py:177-197
 * with loss read before the update, as the reference: a non-finite loss
 * raises before step_optimizer).
 * gsv_step_gate: gate = overflow | !isfinite(*loss_sum); result[0] = loss
 * sum, result[1] = overflow | nonfinite << 1 (the step's 16-byte D2H).
 * gsv_fused_update_device: the one-pass f32 tail of gsv_fused_update, but a
 * no-op when *gate != 0, with bc1 = bias_corrections[2 t], bc2 =
 * bias_corrections[2 t + 1] for t = *step (the number of completed steps;
 * the table holds 1 - beta^(t+1) computed on the host like the reference).
 * With rec32 != NULL it also writes, from the updated parameters, the next
 * step's gsv_preprocess outputs (rec32, counts, box for grid/bricks/cutoff),
 * so the next step's binning starts at gsv_bin_scan; when gated it writes
 * nothing (the parameters, hence the records, are unchanged).
 * gsv_step_advance: *step += 1 unless *gate. */
int gsv_step_gate(const double* loss_sum, const int32_t* overflow, int32_t* gate,
                  double* result, void* stream);
int gsv_fused_update_device(const float* partials, const int64_t* gstart, const double* gsum,
                            int64_t n,
                            double* positions, double* log_scales, double* rotations,
                            double* raw_amplitude, double* raw_relax, double* const* moments,
                            int amplitude_enabled, int relax_enabled,
                            const gsv_adam_hparams* hp, const double* bias_corrections,
                            const int64_t* step, const int32_t* gate, const gsv_grid* grid,
                            const gsv_bricks* bricks, double cutoff_sigma,
                            gsv_record32* rec32, int32_t* counts, int32_t* box, void* stream);
int gsv_step_advance(int64_t* step, const int32_t* gate, void* stream);
/* gsv_step_advance, then the step's 16-byte result straight into slot
 * (*counter % slots) of a ring in pinned host memory (ring: 2 * slots
 * doubles, host-allocated page-locked, device-accessible under UVA) and
 * *counter += 1 -- the replayed graph's last node, so no separate D2H copy
 * sits between consecutive replays. */
int gsv_step_advance_publish(int64_t* step, const int32_t* gate, const double* result,
                             double* ring, int64_t* counter, int slots, void* stream);

/* Sharded graph step: the one all_reduce buffer red (N x 12
 * float) = the merged per-Gaussian partials gsum (gsv_merge, N x 12 double)
 * with this rank's loss sum in red[11] and its capacity overflow flag in
 * red[23]; after the all_reduce, gsv_shard_unpack restores gsum (double, the
 * two slots zeroed), the global loss sum and the global overflow flag (any
 * rank).  gsv_fused_update_device then takes gsum instead of partials. */
int gsv_shard_pack(const double* gsum, int64_t n, const double* loss_sum,
                   const int32_t* overflow, float* red, void* stream);
int gsv_shard_unpack(const float* red, int64_t n, double* gsum, double* loss_sum,
                     int32_t* overflow, void* stream);

/* q /= |q| per Gaussian (GaussianField.normalize_rotations, field.py:100). */
int gsv_normalize_rotations(double* rotations, int64_t n, void* stream);

/* ------------------------------------------------------------------------
 * Quality metrics (metrics.py:35-77), f64 like the reference.  x, y: V
 * values, float32 (x_f64 = 0) or float64 (1), linear x-fastest.
 * gsv_sq_diff_sum: *out = sum (x - y)^2 (PSNR's MSE numerator) in a fixed
 *   reduction order; partials: gsv_metric_blocks(V) doubles of scratch.
 * gsv_ssim3d: *out = sum over voxels of the local SSIM map (divide by V for
 *   ssim3d): the 11-tap window (window11: a HOST array of 11 doubles, built
 *   exactly as metrics.py:45-49) applied separably along x, y, z, zero fill,
 *   local moments divided by the window's coverage; needs nx, ny, nz >= 11.
 *   workspace: gsv_ssim3d_workspace bytes.
 * ------------------------------------------------------------------------ */
int gsv_metric_blocks(int64_t v);
int gsv_sq_diff_sum(const void* x, int x_f64, const void* y, int y_f64, int64_t v,
                    double* partials, double* out, void* stream);
int gsv_ssim3d_workspace(const gsv_grid* grid, size_t* bytes);
int gsv_ssim3d(const void* x, int x_f64, const void* y, int y_f64, const gsv_grid* grid,
               const double* window11, void* workspace, size_t workspace_bytes,
               double* out, void* stream);

/* Per-Gaussian geometry helpers of the reference API, f64 on the device:
 * gsv_rotation_matrices: R (N,3,3) from the stored quaternions, verbatim
 *   (field.py:141-154).
 * gsv_sigma_inv: Sigma^-1 = R diag(exp(-2 ls)) R^T (N,3,3) (render.py:67-71).
 * gsv_weight: *out = weight of Gaussian i at world point p, 0 beyond the
 *   cutoff (render.py:74-81). */
int gsv_rotation_matrices(const double* rotations, int64_t n, double* R, void* stream);
int gsv_sigma_inv(const double* log_scales, const double* rotations, int64_t n, double* out,
                  void* stream);
int gsv_weight(const double* positions, const double* log_scales, const double* rotations,
               const double* raw_relax, int64_t n, int64_t i, int relax_enabled, double px,
               double py, double pz, double cutoff_sigma, double* out, void* stream);

/* Brute-force O(N*V) render (render_naive / _naive_kernel, render.py:84-127)
 * on the device, Sigma^-1 quadratic form, f64 math.  precision selects the
 * accumulator / output type. */
int gsv_render_naive(const double* positions, const double* log_scales,
                     const double* rotations, const double* raw_amplitude,
                     const double* raw_relax, int64_t n, int relax_enabled,
                     const gsv_grid* grid, double cutoff_sigma, double eps_w,
                     int precision, void* I, void* stream);

/* ------------------------------------------------------------------------
 * Setup of a fit on the device.
 *
 * gsv_resample_trilinear: resample_trilinear (volume.py:126-154): samples
 * src (float32 or float64, x-fastest) at the voxel centres of dst_grid with
 * clamp-to-edge, f64 accumulation in the reference's operation order, the
 * result in the source dtype -- bit-identical to the reference.
 *
 * init_from_volume (field.py:212-234) in three calls:
 *   gsv_init_workspace(grid, &bytes)          CUB scratch size;
 *   gsv_init_count(data, f64, grid, thr, slot, ws, bytes, stream)
 *       slot (V+1, int64, device): exclusive scan of the mask data >= thr in
 *       numpy argwhere order (C order over [ix, iy, iz]); slot[V] = N (read
 *       it to size the field);
 *   gsv_init_fill(data, f64, grid, thr, slot, log_scales3 (host, 3 doubles:
 *       log(scale_factor * spacing) as numpy computes it), raw_relax
 *       (logit(relax_init)), positions (N,3), log_scales (N,3),
 *       rotations (N,4), raw_amplitude (N), raw_relax_out (N), stream).
 * positions, log_scales, rotations and raw_relax are bit-identical to the
 * reference; raw_amplitude = logit(clip(I, 1e-4, 1 - 1e-4)) is within a few
 * ulp (device log/log1p in xsf's formula; scipy uses glibc's).
 * ------------------------------------------------------------------------ */
/* LR-consistency loss (the north_star's HR-render-then-downsample training
 * mode; no reference counterpart, not part of the parity claims): the LR
 * prediction is the mean of each LR voxel's fx*fy*fz HR voxels of an HR
 * render I (HR dims = LR dims x factors, HR voxels nested in LR voxels);
 * per LR voxel the L1/L2 loss of optimize.py:91-103 against target (float32
 * or float64); dL/dI_HR = dL/dI_LR / (fx fy fz), written as the backward's
 * ab (HR, float2 {dL/dI / W, I}); loss_part: gsv_pool_loss_blocks(lr_grid)
 * doubles (sum them with gsv_sum). */
int gsv_pool_loss_blocks(const gsv_grid* lr_grid);
int gsv_pool_loss(const float* I, const float* W, const void* target, int target_dtype,
                  const gsv_grid* hr_grid, const gsv_grid* lr_grid, int fx, int fy, int fz,
                  int loss_kind, double eps_w, float* ab, double* loss_part, void* stream);
/* gsv_phantom: generate_phantom (phantom.py:52-75) on the device.  prims:
 * nprims x 7 doubles {cx, cy, cz, a_x, a_y, a_z, intensity} (semi-axes for
 * kind 0 = ellipsoids, sigmas for kind 1 = gaussian mixture), rasterized at
 * the voxel centres origin + index * spacing with the max at overlaps; then,
 * if radius > 0, ndimage.gaussian_filter with the 2 radius + 1 weights
 * (scipy's _gaussian_kernel1d, computed by the caller) along x, y, z with
 * scipy's symmetric-correlation order and "reflect" edges; clipped to [0, 1]
 * and written as float32, x-fastest linear.  Ellipsoids are bit-identical
 * to the reference; the mixture's exp is the device's (within an ulp).
 * scratch: 2 V doubles.  Added in ABI 6. */
int gsv_phantom(const gsv_grid* grid, int kind, int nprims, const double* prims, int radius,
                const double* weights, double* scratch, float* out, void* stream);
int gsv_resample_trilinear(const void* src, int src_f64, const gsv_grid* src_grid,
                           void* out, const gsv_grid* dst_grid, void* stream);
int gsv_init_workspace(const gsv_grid* grid, size_t* bytes);
int gsv_init_count(const void* data, int data_f64, const gsv_grid* grid,
                   double threshold, int64_t* slot, void* workspace,
                   size_t workspace_bytes, void* stream);
int gsv_init_fill(const void* data, int data_f64, const gsv_grid* grid,
                  double threshold, const int64_t* slot, const double* log_scales3,
                  double raw_relax, double* positions, double* log_scales,
                  double* rotations, double* raw_amplitude, double* raw_relax_out,
                  void* stream);

#ifdef __cplusplus
}
#endif

#endif /* GSV_B200_H */
