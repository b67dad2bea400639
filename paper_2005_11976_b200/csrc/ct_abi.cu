// ct_abi.cu -- C-ABI identity and error state (include/cyltomo_b200.h).
#include "ct_common.cuh"

namespace ctabi {

thread_local char g_err[512] = "";

int set_err(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(g_err, sizeof g_err, "%s: %s", what, cudaGetErrorString(e));
    return CT_ERR_CUDA;
  }
  return CT_OK;
}

}  // namespace ctabi

extern "C" {

int ct_abi_version(void) { return CT_ABI_VERSION; }
const char* ct_last_error(void) { return ctabi::g_err; }
const char* ct_arch(void) { return "sm_100a"; }

}  // extern "C"
