// C-ABI plumbing: thread-local last error, version, device query.
#include "common.cuh"

#include <cstdio>

namespace corr2d {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) return CORR2D_OK;
  std::string msg = std::string(what) + ": " + cudaGetErrorString(e);
  if (e == cudaErrorMemoryAllocation) return fail(CORR2D_ERR_OOM, msg);
  return fail(CORR2D_ERR_CUDA, msg);
}

}  // namespace corr2d

using namespace corr2d;

extern "C" const char* corr2d_last_error(void) { return g_last_error.c_str(); }

extern "C" int corr2d_abi_version(void) { return CORR2D_ABI_VERSION; }

extern "C" int corr2d_device_info(int device, int* sms, int* cc_major, int* cc_minor) {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    cudaGetLastError();
    return fail(CORR2D_ERR_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
  }
  if (device < 0 || device >= count) return fail(CORR2D_ERR_DATA, "device index out of range");
  if (sms) cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, device);
  if (cc_major) cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, device);
  if (cc_minor) cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, device);
  return CORR2D_OK;
}
