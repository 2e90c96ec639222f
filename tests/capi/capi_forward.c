/*
 * capi_forward.c -- the C ABI of include/gsv.h driven from plain C: no
 * Python, no torch.  Reads a field and a grid from a little binary file,
 * bins it (gsv_preprocess -> gsv_bin_scan -> gsv_bin_fill), renders it
 * (gsv_forward, f32 engine) and writes starts, gids and I to an output file,
 * which tests/test_gpu_capi.py compares with the Python API's results.
 *
 * Input  (little endian): int32 nx, ny, nz; float64 origin[3], spacing[3],
 *        cutoff; int32 bdx, bdy, bdz; int64 n; then float64 positions[3n],
 *        log_scales[3n], rotations[4n], raw_amplitude[n], raw_relax[n]; int32 relax.
 * Output: int64 pairs, nbricks; int64 starts[nbricks + 1]; int32 gids[pairs];
 *        float32 I[nx ny nz]; int32 incremental_ok.
 *
 * Then the incremental entry points: every Gaussian moves by +0.37 spacing in
 * x; gsv_preprocess_track records the ones whose boxes changed, gsv_bin_scan
 * recounts, gsv_bin_incremental edits the lists, and the result is compared
 * with a full gsv_bin_fill of the moved field (incremental_ok = 1 if equal).
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "gsv.h"

#define CK(x)                                                                            \
  do {                                                                                   \
    int st_ = (x);                                                                       \
    if (st_ != 0) {                                                                      \
      fprintf(stderr, "%s failed (%d): %s\n", #x, st_, gsv_last_error());               \
      return 2;                                                                          \
    }                                                                                    \
  } while (0)
#define CU(x)                                                                            \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess) {                                                             \
      fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));                           \
      return 3;                                                                          \
    }                                                                                    \
  } while (0)

static void* dev_copy(const void* h, size_t bytes) {
  void* d = NULL;
  if (cudaMalloc(&d, bytes ? bytes : 16) != cudaSuccess) return NULL;
  if (h != NULL && bytes) {
    if (cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice) != cudaSuccess) return NULL;
  }
  return d;
}

static int read_all(FILE* f, void* p, size_t bytes) { return fread(p, 1, bytes, f) == bytes; }

int main(int argc, char** argv) {
  if (argc != 3) {
    fprintf(stderr, "usage: %s input.bin output.bin\n", argv[0]);
    return 1;
  }
  if (gsv_abi_version() != GSV_ABI_VERSION) {
    fprintf(stderr, "ABI mismatch: library %d, header %d\n", gsv_abi_version(), GSV_ABI_VERSION);
    return 1;
  }
  FILE* in = fopen(argv[1], "rb");
  if (!in) return 1;
  int32_t dims[3], bd[3], relax = 0;
  double org[3], spc[3], cutoff;
  int64_t n;
  if (!read_all(in, dims, 12) || !read_all(in, org, 24) || !read_all(in, spc, 24) ||
      !read_all(in, &cutoff, 8) || !read_all(in, bd, 12) || !read_all(in, &n, 8))
    return 1;
  double* h = (double*)malloc((size_t)(12 * n + 1) * sizeof(double));
  if (!read_all(in, h, (size_t)(12 * n) * sizeof(double)) || !read_all(in, &relax, 4)) return 1;
  fclose(in);

  gsv_grid g = {dims[0], dims[1], dims[2], 0, org[0], org[1], org[2], spc[0], spc[1], spc[2]};
  gsv_bricks k;
  k.bdx = bd[0];
  k.bdy = bd[1];
  k.bdz = bd[2];
  k.bgx = (dims[0] + bd[0] - 1) / bd[0];
  k.bgy = (dims[1] + bd[1] - 1) / bd[1];
  k.bgz = (dims[2] + bd[2] - 1) / bd[2];
  const int32_t nb = k.bgx * k.bgy * k.bgz;
  k.b0 = 0; /* the whole grid: brick ids [0, nb) */
  k.b1 = nb;
  const int64_t nv = (int64_t)dims[0] * dims[1] * dims[2];

  double* pos = (double*)dev_copy(h, (size_t)(3 * n) * 8);
  double* ls = (double*)dev_copy(h + 3 * n, (size_t)(3 * n) * 8);
  double* rot = (double*)dev_copy(h + 6 * n, (size_t)(4 * n) * 8);
  double* ra = (double*)dev_copy(h + 10 * n, (size_t)n * 8);
  double* rr = (double*)dev_copy(h + 11 * n, (size_t)n * 8);
  gsv_record32* rec32 = (gsv_record32*)dev_copy(NULL, (size_t)n * sizeof(gsv_record32));
  int32_t* counts = (int32_t*)dev_copy(NULL, (size_t)n * 4);
  int32_t* box = (int32_t*)dev_copy(NULL, (size_t)n * 16);
  int64_t* gstart = (int64_t*)dev_copy(NULL, (size_t)(n + 1) * 8);

  CK(gsv_preprocess(pos, ls, rot, ra, rr, n, relax, cutoff, &g, &k, rec32, NULL, counts, box,
                    NULL));
  size_t ws_bytes = 0;
  CK(gsv_bin_workspace(n, 1, nb, &ws_bytes));
  void* ws = dev_copy(NULL, ws_bytes);
  CK(gsv_bin_scan(counts, n, gstart, ws, ws_bytes, NULL));
  int64_t pairs = 0;
  CU(cudaMemcpy(&pairs, gstart + n, 8, cudaMemcpyDeviceToHost));   /* the one host read */

  CU(cudaFree(ws));
  CK(gsv_bin_workspace(n, pairs > 0 ? pairs : 1, nb, &ws_bytes));
  ws = dev_copy(NULL, ws_bytes);
  const size_t pb = (size_t)(pairs > 0 ? pairs : 1) * 4;
  int32_t* keys_tmp = (int32_t*)dev_copy(NULL, pb);
  int32_t* vals_tmp = (int32_t*)dev_copy(NULL, pb);
  int32_t* keys_out = (int32_t*)dev_copy(NULL, pb);
  int32_t* gids = (int32_t*)dev_copy(NULL, pb);
  int64_t* starts = (int64_t*)dev_copy(NULL, (size_t)(nb + 1) * 8);
  CK(gsv_bin_fill(counts, box, gstart, n, pairs, &k, keys_tmp, vals_tmp, keys_out, gids, starts,
                  ws, ws_bytes, NULL));

  float* S = (float*)dev_copy(NULL, (size_t)nv * 4);
  float* W = (float*)dev_copy(NULL, (size_t)nv * 4);
  float* I = (float*)dev_copy(NULL, (size_t)nv * 4);
  /* the Python API's kernel choice (raster._forward_vpl_arg): the grouped
   * forward (vpl 16) for 8x8x4 bricks at <= 8 pairs per Gaussian, else auto */
  const int b884 = bd[0] == 8 && bd[1] == 8 && bd[2] == 4;
  const int vpl = (b884 && pairs <= 8 * n) ? 16 : 0;
  CK(gsv_forward(pos, ls, rot, rec32, NULL, starts, gids, &g, &k, cutoff, 1e-8, 0, S, W, I, NULL,
                 0, 0, (double)nv, NULL, NULL, NULL, vpl, NULL));
  CU(cudaDeviceSynchronize());

  int64_t* h_starts = (int64_t*)malloc((size_t)(nb + 1) * 8);
  int32_t* h_gids = (int32_t*)malloc(pb);
  float* h_I = (float*)malloc((size_t)nv * 4);
  CU(cudaMemcpy(h_starts, starts, (size_t)(nb + 1) * 8, cudaMemcpyDeviceToHost));
  if (pairs > 0) CU(cudaMemcpy(h_gids, gids, (size_t)pairs * 4, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(h_I, I, (size_t)nv * 4, cudaMemcpyDeviceToHost));

  /* ---- incremental binning after a move */
  int32_t incremental_ok = 0;
  {
    for (int64_t i = 0; i < n; ++i) h[3 * i] += 0.37 * spc[0];
    CU(cudaMemcpy(pos, h, (size_t)(3 * n) * 8, cudaMemcpyHostToDevice));
    const int chg_cap = (int)(n > 0 ? n : 1);
    int32_t* chg_count = (int32_t*)dev_copy(NULL, 4);
    CU(cudaMemset(chg_count, 0, 4));
    int32_t* chg_gid = (int32_t*)dev_copy(NULL, (size_t)chg_cap * 4);
    int32_t* chg_old = (int32_t*)dev_copy(NULL, (size_t)chg_cap * 16);
    int32_t* chg_oldcnt = (int32_t*)dev_copy(NULL, (size_t)chg_cap * 4);
    CK(gsv_preprocess_track(pos, ls, rot, ra, rr, n, relax, cutoff, &g, &k, rec32, counts, box,
                            chg_count, chg_gid, chg_old, chg_oldcnt, chg_cap, NULL));
    CU(cudaFree(ws));
    CK(gsv_bin_workspace(n, 1, nb, &ws_bytes));
    ws = dev_copy(NULL, ws_bytes);
    CK(gsv_bin_scan(counts, n, gstart, ws, ws_bytes, NULL));
    int64_t pairs2 = 0;
    CU(cudaMemcpy(&pairs2, gstart + n, 8, cudaMemcpyDeviceToHost));
    const int64_t cap = (pairs2 > pairs ? pairs2 : pairs) + 64;
    int32_t* gids_a = (int32_t*)dev_copy(NULL, (size_t)cap * 4);
    if (pairs > 0) CU(cudaMemcpy(gids_a, gids, (size_t)pairs * 4, cudaMemcpyDeviceToDevice));
    int64_t* starts_out = (int64_t*)dev_copy(NULL, (size_t)(nb + 1) * 8);
    int32_t* gids_out = (int32_t*)dev_copy(NULL, (size_t)cap * 4);
    unsigned long long* ops = (unsigned long long*)dev_copy(NULL, (size_t)2 * 16384 * 8);
    int32_t* nops = (int32_t*)dev_copy(NULL, 4);
    int32_t* lens = (int32_t*)dev_copy(NULL, (size_t)8 * (nb + 1) * 4);
    int32_t* flags = (int32_t*)dev_copy(NULL, 8);          /* dry, overflow */
    CU(cudaMemset(nops, 0, 4));
    CU(cudaMemset(lens, 0, (size_t)8 * (nb + 1) * 4));
    CU(cudaMemset(flags, 0, 8));
    size_t iws = 0;
    CK(gsv_bin_incremental_workspace(nb, &iws));
    void* ws2 = dev_copy(NULL, iws);
    CK(gsv_bin_incremental(counts, box, gstart, n, cap, &k, chg_count, chg_gid, chg_old,
                           chg_oldcnt, chg_cap, starts, gids_a, starts_out, gids_out, ops, nops,
                           lens, flags, flags + 1, 1, ws2, iws, NULL));
    /* the full build of the moved field */
    CU(cudaFree(ws));
    CK(gsv_bin_workspace(n, pairs2 > 0 ? pairs2 : 1, nb, &ws_bytes));
    ws = dev_copy(NULL, ws_bytes);
    const size_t pb2 = (size_t)(pairs2 > 0 ? pairs2 : 1) * 4;
    int32_t* kt = (int32_t*)dev_copy(NULL, pb2);
    int32_t* vt = (int32_t*)dev_copy(NULL, pb2);
    int32_t* ko = (int32_t*)dev_copy(NULL, pb2);
    int32_t* gf = (int32_t*)dev_copy(NULL, pb2);
    int64_t* sf = (int64_t*)dev_copy(NULL, (size_t)(nb + 1) * 8);
    CK(gsv_bin_fill(counts, box, gstart, n, pairs2, &k, kt, vt, ko, gf, sf, ws, ws_bytes, NULL));
    CU(cudaDeviceSynchronize());
    int32_t h_flags[2];
    CU(cudaMemcpy(h_flags, flags, 8, cudaMemcpyDeviceToHost));
    int64_t* h_si = (int64_t*)malloc((size_t)(nb + 1) * 8);
    int64_t* h_sf = (int64_t*)malloc((size_t)(nb + 1) * 8);
    int32_t* h_gi = (int32_t*)malloc(pb2);
    int32_t* h_gf = (int32_t*)malloc(pb2);
    CU(cudaMemcpy(h_si, starts, (size_t)(nb + 1) * 8, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(h_sf, sf, (size_t)(nb + 1) * 8, cudaMemcpyDeviceToHost));
    if (pairs2 > 0) {
      CU(cudaMemcpy(h_gi, gids_a, (size_t)pairs2 * 4, cudaMemcpyDeviceToHost));
      CU(cudaMemcpy(h_gf, gf, (size_t)pairs2 * 4, cudaMemcpyDeviceToHost));
    }
    incremental_ok = h_flags[1] == 0;
    for (int64_t b = 0; b <= nb && incremental_ok; ++b) incremental_ok = h_si[b] == h_sf[b];
    for (int64_t j = 0; j < pairs2 && incremental_ok; ++j) incremental_ok = h_gi[j] == h_gf[j];
    printf("capi_forward: incremental pairs %lld -> %lld, equal to a full build: %d\n",
           (long long)pairs, (long long)pairs2, incremental_ok);
  }

  FILE* out = fopen(argv[2], "wb");
  if (!out) return 1;
  const int64_t nb64 = nb;
  fwrite(&pairs, 8, 1, out);
  fwrite(&nb64, 8, 1, out);
  fwrite(h_starts, 8, (size_t)(nb + 1), out);
  if (pairs > 0) fwrite(h_gids, 4, (size_t)pairs, out);
  fwrite(h_I, 4, (size_t)nv, out);
  fwrite(&incremental_ok, 4, 1, out);
  fclose(out);
  printf("capi_forward: pairs=%lld bricks=%d voxels=%lld\n", (long long)pairs, nb,
         (long long)nv);
  return 0;
}
