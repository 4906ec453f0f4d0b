// capi.cu — error reporting and version for the C ABI (include/packkv_b200.h).
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>

#include "pkv_common.cuh"

static thread_local char g_last_error[512] = "";
static thread_local int g_last_path = PKV_PATH_NONE;

void pkv_note_path(int path) { g_last_path = path; }

bool pkv_pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("PKV_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

void pkv_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

int pkv_cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return PKV_OK;
  pkv_set_error("%s: %s", what, cudaGetErrorString(e));
  return PKV_E_CUDA;
}

extern "C" const char* pkv_last_error(void) { return g_last_error; }

extern "C" int pkv_version(void) { return PKV_ABI_VERSION; }

extern "C" int pkv_last_path(void) { return g_last_path; }
