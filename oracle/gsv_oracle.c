/*
 * gsv_oracle.c -- CPU restatement of the reference rasterizer's loops.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the CUDA path and
 * the "port" CPU baseline timed by bench.py; it is never linked into or
 * called by the product (paper_2603_09621_b200/).  Only tests/, the smoke()
 * check in __graft_entry__.py and bench.py's cpu_baseline leg use it.
 *
 * Each function restates one numba kernel of /root/reference/pkg/src/gsvol
 * line for line, in f64 with no FMA contraction (compiled with
 * -ffp-contract=off, like numba 0.65 which emits no contraction) and the
 * same accumulation order.  OpenMP over bricks / Gaussians mirrors prange.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Pair expansion + stable sort by brick id of build_brick_index
 * (raster.py:189-216).  Inputs are the per-Gaussian brick boxes computed by
 * the numpy restatement (blo (N,3), nb (N,3), inside (N)); the stable argsort
 * by brick id of the gid-major emission equals a counting sort that visits
 * Gaussians in ascending gid.  starts (B+1) out; gids (P) out. */
void oracle_bin_pairs(int64_t n, const int64_t* blo, const int64_t* nb, const uint8_t* inside,
                      int64_t bgx, int64_t bgy, int64_t bgz, int64_t* starts, int64_t* gids) {
  const int64_t nbricks = bgx * bgy * bgz;
  int64_t* cnt = (int64_t*)calloc((size_t)nbricks + 1, sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) {
    if (!inside[i]) continue;
    for (int64_t z = 0; z < nb[3 * i + 2]; ++z)
      for (int64_t y = 0; y < nb[3 * i + 1]; ++y)
        for (int64_t x = 0; x < nb[3 * i + 0]; ++x) {
          const int64_t b = (blo[3 * i] + x) + bgx * ((blo[3 * i + 1] + y) + bgy * (blo[3 * i + 2] + z));
          cnt[b + 1]++;
        }
  }
  starts[0] = 0;
  for (int64_t b = 0; b < nbricks; ++b) starts[b + 1] = starts[b] + cnt[b + 1];
  for (int64_t b = 0; b < nbricks; ++b) cnt[b] = starts[b];
  for (int64_t i = 0; i < n; ++i) {
    if (!inside[i]) continue;
    for (int64_t z = 0; z < nb[3 * i + 2]; ++z)
      for (int64_t y = 0; y < nb[3 * i + 1]; ++y)
        for (int64_t x = 0; x < nb[3 * i + 0]; ++x) {
          const int64_t b = (blo[3 * i] + x) + bgx * ((blo[3 * i + 1] + y) + bgy * (blo[3 * i + 2] + z));
          gids[cnt[b]++] = i;
        }
  }
  free(cnt);
}

/* _forward_kernel (raster.py:240-293).  acc_f32 selects float32 S/W/I
 * (each add done in f64 and rounded on store, like numba's f32 arrays). */
void oracle_forward(const double* positions, const double* lfac, const double* amp,
                    const double* relax, const int64_t* starts, const int64_t* gids,
                    int64_t bgx, int64_t bgy, int64_t bgz, int64_t bdx, int64_t bdy, int64_t bdz,
                    int64_t nx, int64_t ny, int64_t nz, double ox, double oy, double oz,
                    double sx, double sy, double sz, double cutoff2, double eps_w, int acc_f32,
                    void* Sv, void* Wv, void* Iv) {
  const int64_t nbricks = bgx * bgy * bgz;
  float* S32 = (float*)Sv; float* W32 = (float*)Wv; float* I32 = (float*)Iv;
  double* S64 = (double*)Sv; double* W64 = (double*)Wv; double* I64 = (double*)Iv;
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t b = 0; b < nbricks; ++b) {
    const int64_t bx = b % bgx, rem = b / bgx, by = rem % bgy, bz = rem / bgy;
    const int64_t x0 = bx * bdx, y0 = by * bdy, z0 = bz * bdz;
    const int64_t x1 = x0 + bdx < nx ? x0 + bdx : nx;
    const int64_t y1 = y0 + bdy < ny ? y0 + bdy : ny;
    const int64_t z1 = z0 + bdz < nz ? z0 + bdz : nz;
    for (int64_t j = starts[b]; j < starts[b + 1]; ++j) {
      const int64_t i = gids[j];
      const double mx = positions[3 * i], my = positions[3 * i + 1], mz = positions[3 * i + 2];
      const double* l = lfac + 9 * i;
      const double ai = amp[i], ri = relax[i];
      for (int64_t iz = z0; iz < z1; ++iz) {
        const double pz = oz + iz * sz, dz = pz - mz;
        for (int64_t iy = y0; iy < y1; ++iy) {
          const double py = oy + iy * sy, dy = py - my;
          const int64_t base = nx * (iy + ny * iz);
          for (int64_t ix = x0; ix < x1; ++ix) {
            const double px = ox + ix * sx, dx = px - mx;
            const double v0 = l[0] * dx + l[1] * dy + l[2] * dz;
            const double v1 = l[3] * dx + l[4] * dy + l[5] * dz;
            const double v2 = l[6] * dx + l[7] * dy + l[8] * dz;
            const double d2 = v0 * v0 + v1 * v1 + v2 * v2;
            if (d2 <= cutoff2) {
              const double w = exp(-0.5 * d2) * ri;
              const int64_t lin = base + ix;
              if (acc_f32) {
                S32[lin] = (float)((double)S32[lin] + ai * w);
                W32[lin] = (float)((double)W32[lin] + w);
              } else {
                S64[lin] += ai * w;
                W64[lin] += w;
              }
            }
          }
        }
      }
    }
    for (int64_t iz = z0; iz < z1; ++iz)
      for (int64_t iy = y0; iy < y1; ++iy) {
        const int64_t base = nx * (iy + ny * iz);
        for (int64_t ix = x0; ix < x1; ++ix) {
          const int64_t lin = base + ix;
          if (acc_f32)
            I32[lin] = ((double)W32[lin] >= eps_w) ? S32[lin] / W32[lin] : 0.0f;
          else
            I64[lin] = (W64[lin] >= eps_w) ? S64[lin] / W64[lin] : 0.0;
        }
      }
  }
}

/* _backward_kernel (raster.py:322-409).  W/I are float32 or float64 per
 * acc_f32; dLdI f64; pg (P,11) f64 out: amp, rel, mu[3], cov[6]. */
void oracle_backward(const double* positions, const double* lfac, const double* amp,
                     const double* relax, const int64_t* starts, const int64_t* gids,
                     int64_t bgx, int64_t bgy, int64_t bgz, int64_t bdx, int64_t bdy, int64_t bdz,
                     int64_t nx, int64_t ny, int64_t nz, double ox, double oy, double oz,
                     double sx, double sy, double sz, double cutoff2, double eps_w, int acc_f32,
                     const void* Wv, const void* Iv, const double* dLdI, double* pg) {
  const int64_t nbricks = bgx * bgy * bgz;
  const float* W32 = (const float*)Wv; const float* I32 = (const float*)Iv;
  const double* W64 = (const double*)Wv; const double* I64 = (const double*)Iv;
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t b = 0; b < nbricks; ++b) {
    const int64_t bx = b % bgx, rem = b / bgx, by = rem % bgy, bz = rem / bgy;
    const int64_t x0 = bx * bdx, y0 = by * bdy, z0 = bz * bdz;
    const int64_t x1 = x0 + bdx < nx ? x0 + bdx : nx;
    const int64_t y1 = y0 + bdy < ny ? y0 + bdy : ny;
    const int64_t z1 = z0 + bdz < nz ? z0 + bdz : nz;
    for (int64_t j = starts[b]; j < starts[b + 1]; ++j) {
      const int64_t i = gids[j];
      const double mx = positions[3 * i], my = positions[3 * i + 1], mz = positions[3 * i + 2];
      const double* l = lfac + 9 * i;
      const double ai = amp[i], ri = relax[i];
      double acc_a = 0, acc_r = 0, mu0 = 0, mu1 = 0, mu2 = 0;
      double g00 = 0, g11 = 0, g22 = 0, g01 = 0, g02 = 0, g12 = 0;
      for (int64_t iz = z0; iz < z1; ++iz) {
        const double pz = oz + iz * sz, dz = pz - mz;
        for (int64_t iy = y0; iy < y1; ++iy) {
          const double py = oy + iy * sy, dy = py - my;
          const int64_t base = nx * (iy + ny * iz);
          for (int64_t ix = x0; ix < x1; ++ix) {
            const int64_t lin = base + ix;
            const double wp = acc_f32 ? (double)W32[lin] : W64[lin];
            if (wp < eps_w) continue;
            const double dl = dLdI[lin];
            if (dl == 0.0) continue;
            const double px = ox + ix * sx, dx = px - mx;
            const double v0 = l[0] * dx + l[1] * dy + l[2] * dz;
            const double v1 = l[3] * dx + l[4] * dy + l[5] * dz;
            const double v2 = l[6] * dx + l[7] * dy + l[8] * dz;
            const double d2 = v0 * v0 + v1 * v1 + v2 * v2;
            if (d2 > cutoff2) continue;
            const double kern = exp(-0.5 * d2);
            const double w = kern * ri;
            acc_a += dl * w / wp;
            const double il = acc_f32 ? (double)I32[lin] : I64[lin];
            const double common = dl * (ai - il) / wp;
            acc_r += common * kern;
            const double cw = common * w;
            mu0 += cw * (l[0] * v0 + l[3] * v1 + l[6] * v2);
            mu1 += cw * (l[1] * v0 + l[4] * v1 + l[7] * v2);
            mu2 += cw * (l[2] * v0 + l[5] * v1 + l[8] * v2);
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
      double* o = pg + 11 * j;
      o[0] = acc_a; o[1] = acc_r; o[2] = mu0; o[3] = mu1; o[4] = mu2;
      o[5] = g00; o[6] = g11; o[7] = g22; o[8] = g01; o[9] = g02; o[10] = g12;
    }
  }
}

/* _merge_pairs_kernel (raster.py:412-451): out (N,11) f64, each Gaussian's
 * pair partials summed in porder (ascending brick) order. */
void oracle_merge(int64_t n, const int64_t* gstarts, const int64_t* porder, const double* pg,
                  double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double acc[11] = {0};
    for (int64_t t = gstarts[i]; t < gstarts[i + 1]; ++t) {
      const double* p = pg + 11 * porder[t];
      for (int a = 0; a < 11; ++a) acc[a] += p[a];
    }
    for (int a = 0; a < 11; ++a) out[11 * i + a] = acc[a];
  }
}

int oracle_abi_version(void) { return 1; }

/* Chain rule of backward (raster.py:524-549, _rotation_jacobians 454-467) in
 * C for the CPU-baseline leg: same formulas as the numpy einsums (summation
 * order differs at the 1e-16 level).  sums (N,11) -> grads. */
void oracle_chain_rule(int64_t n, const double* sums, const double* ls, const double* q,
                       const double* ra, const double* rr, int relax_enabled,
                       double* g_amp, double* g_rel, double* g_pos, double* g_ls,
                       double* g_rot) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    const double* s = sums + 11 * i;
    double G[9] = {s[5], s[8], s[9], s[8], s[6], s[10], s[9], s[10], s[7]};
    const double w = q[4 * i], x = q[4 * i + 1], y = q[4 * i + 2], z = q[4 * i + 3];
    const double R[9] = {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                         2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                         2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)};
    const double iv[3] = {exp(-2.0 * ls[3 * i]), exp(-2.0 * ls[3 * i + 1]),
                          exp(-2.0 * ls[3 * i + 2])};
    for (int k = 0; k < 3; ++k) {
      double t = 0.0;
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) t += R[3 * a + k] * G[3 * a + b] * R[3 * b + k];
      g_ls[3 * i + k] = -2.0 * iv[k] * t;
    }
    const double J[4][9] = {
        {0, -2 * z, 2 * y, 2 * z, 0, -2 * x, -2 * y, 2 * x, 0},
        {0, 2 * y, 2 * z, 2 * y, -4 * x, -2 * w, 2 * z, 2 * w, -4 * x},
        {-4 * y, 2 * x, 2 * w, 2 * x, 0, 2 * z, -2 * w, 2 * z, -4 * y},
        {-4 * z, -2 * w, 2 * x, 2 * w, -4 * z, 2 * y, 2 * x, 2 * y, 0}};
    for (int j = 0; j < 4; ++j) {
      double t = 0.0;
      for (int a = 0; a < 3; ++a)
        for (int c = 0; c < 3; ++c) {
          double pm = 0.0;
          for (int m = 0; m < 3; ++m) pm += J[j][3 * c + m] * iv[m] * R[3 * a + m];
          t += G[3 * a + c] * pm;
        }
      g_rot[4 * i + j] = 2.0 * t;
    }
    g_pos[3 * i] = s[2];
    g_pos[3 * i + 1] = s[3];
    g_pos[3 * i + 2] = s[4];
    const double A = 1.0 / (1.0 + exp(-ra[i]));
    g_amp[i] = s[0] * A * (1.0 - A);
    if (relax_enabled) {
      const double r = 1.0 / (1.0 + exp(-rr[i]));
      g_rel[i] = s[1] * r * (1.0 - r);
    } else {
      g_rel[i] = 0.0;
    }
  }
}

/* One Adam step on one group (optimize.py:139-147), numpy operand order. */
void oracle_adam(int64_t count, double* p, double* m, double* v, const double* g, double lr,
                 double b1, double b2, double eps, double bc1, double bc2) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < count; ++i) {
    m[i] = m[i] * b1 + (1.0 - b1) * g[i];
    v[i] = v[i] * b2 + ((1.0 - b2) * g[i]) * g[i];
    p[i] -= lr * (m[i] / bc1) / (sqrt(v[i] / bc2) + eps);
  }
}

/* q /= |q| (field.py:100-102). */
void oracle_normalize(int64_t n, double* q) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double* r = q + 4 * i;
    const double nrm = sqrt(((r[0] * r[0] + r[1] * r[1]) + r[2] * r[2]) + r[3] * r[3]);
    for (int a = 0; a < 4; ++a) r[a] /= nrm;
  }
}

/* Per-Gaussian gstarts + porder of the merge (raster.py:514-516) by a
 * counting sort on gid (stable => ascending brick order within a gid). */
void oracle_merge_order(int64_t n, int64_t p, const int64_t* gids, int64_t* gstarts,
                        int64_t* porder) {
  memset(gstarts, 0, sizeof(int64_t) * (size_t)(n + 1));
  for (int64_t j = 0; j < p; ++j) gstarts[gids[j] + 1]++;
  for (int64_t i = 0; i < n; ++i) gstarts[i + 1] += gstarts[i];
  int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) cur[i] = gstarts[i];
  for (int64_t j = 0; j < p; ++j) porder[cur[gids[j]]++] = j;
  free(cur);
}
