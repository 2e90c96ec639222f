/*
 * gsv_diag.h -- measurement entry points of libgsv_b200.so (not part of the
 * reference-facing boundary in gsv.h; used by bench.py for the roofline).
 */
#ifndef GSV_B200_DIAG_H
#define GSV_B200_DIAG_H

#include <stdint.h>

#include "gsv.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Exact number of live pair-voxels (d^2 <= cutoff^2, decided exactly as the
 * f32 forward decides them) of an index: the roofline work unit of
 * SURVEY.md §8d.  Also counts every (pair, voxel) of the brick (E_brick) and,
 * for 8x8x4 bricks, the (pair, voxel) slots the f32 forward evaluates: 128 per
 * pair x warp-tile hit under its staging tests (E_tile), and the slots the
 * grouped-column forward (gsv_forward vpl 16) evaluates: 128 per chunk
 * iteration, a chunk running max(group size) iterations (E_group).
 * counters: device uint64[4] = {E_live, E_brick, E_tile, E_group},
 * accumulated. */
int gsv_diag_count_live(const double* positions, const gsv_record32* rec32,
                        const double* log_scales, const double* rotations,
                        const int64_t* starts, const int32_t* gids,
                        const gsv_grid* grid, const gsv_bricks* bricks,
                        double cutoff_sigma, unsigned long long* counters,
                        void* stream);

/* FP32 FMA throughput probe: blocks x 256 threads, each running `iters`
 * iterations of 16 independent FFMA chains (2 FLOP each).  Time it with
 * events; flops = blocks * 256 * iters * 16 * 2.  out: device float sink. */
int gsv_diag_fma_probe(int blocks, int iters, float* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* GSV_B200_DIAG_H */
