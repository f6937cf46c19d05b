// placeholder -- replaced by the tcgen05 kernel
#include "common.cuh"
using namespace corr2d;
extern "C" int corr2d_contract_bf16x3(
    const void*, const void*, const void*, int64_t, int64_t, int64_t,
    int, int, int, int, int, int,
    float*, float*, int64_t, unsigned long long*, void*) {
  return fail(CORR2D_ERR_UNSUPPORTED, "not built yet");
}
