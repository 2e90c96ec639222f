// gsv_capi.cu -- error channel, version and device queries of the C ABI.
#include <cstdarg>
#include <cstdio>

#include "gsv_common.cuh"

namespace gsv {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char* what) {
  set_error("%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
  return GSV_ERR_CUDA;
}

int validate_grid_bricks(const gsv_grid* g, const gsv_bricks* k) {
  GSV_REQUIRE(g != nullptr && k != nullptr, "grid/bricks must not be NULL");
  GSV_REQUIRE(g->nx >= 1 && g->ny >= 1 && g->nz >= 1,
              "grid dims must be >= 1, got (%d,%d,%d)", g->nx, g->ny, g->nz);
  GSV_REQUIRE(k->bdx >= 1 && k->bdy >= 1 && k->bdz >= 1,
              "brick_dims must be positive, got (%d,%d,%d)", k->bdx, k->bdy, k->bdz);
  GSV_REQUIRE(k->bdx <= 255 && k->bdy <= 255 && k->bdz <= 255,
              "brick_dims above 255 per axis are not supported, got (%d,%d,%d)",
              k->bdx, k->bdy, k->bdz);
  GSV_REQUIRE(k->bgx == (g->nx + k->bdx - 1) / k->bdx &&
                  k->bgy == (g->ny + k->bdy - 1) / k->bdy &&
                  k->bgz == (g->nz + k->bdz - 1) / k->bdz,
              "brick grid does not match ceil(dims / brick_dims)");
  GSV_REQUIRE(k->bgx <= 65535 && k->bgy <= 65535 && k->bgz <= 65535,
              "brick grid above 65535 per axis is not supported");
  GSV_REQUIRE((int64_t)k->bgx * k->bgy * k->bgz < (int64_t)INT32_MAX,
              "too many bricks");
  GSV_REQUIRE(0 <= k->b0 && k->b0 <= k->b1 && k->b1 <= k->bgx * k->bgy * k->bgz,
              "slab [%d,%d) outside brick ids [0,%d)", k->b0, k->b1, k->bgx * k->bgy * k->bgz);
  return GSV_OK;
}

}  // namespace gsv

extern "C" {

int gsv_abi_version(void) { return GSV_ABI_VERSION; }

const char* gsv_last_error(void) { return gsv::g_err; }

int gsv_device_sm_count(void) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return -1;
  return sms;
}

}  // extern "C"
