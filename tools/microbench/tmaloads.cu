// L2 -> SMEM operand-load throughput for the bf16x3 contraction's access pattern:
// 148 persistent CTAs stream 64 KB stages (4 boxes of 16 KB) from a 64 MB packed
// operand array that stays L2-resident, with no compute.  Variants compare the
// current 3D tensor box {32 slots, 128 rows, 2 planes} (64-B row segments) with
// wider boxes and with contiguous pre-tiled 1D bulk copies.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("{\"err\": \"%s line %d\"}\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int STAGES = 3, STAGE = 65536;
constexpr int ROWS = 32768, LD = 768;  // bf16 slots per row, 2 planes

__global__ void __launch_bounds__(64, 1) loads(const __grid_constant__ CUtensorMap map, const uint8_t* flat, int mode,
                                               int iters) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (su32(sm_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar[STAGES];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < STAGES; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  uint32_t phase[STAGES] = {0, 0, 0};
  uint32_t seed = blockIdx.x * 2654435761u;
  for (int it = 0; it < iters + STAGES; ++it) {
    const int s = it % STAGES;
    if (it >= STAGES) {  // wait for this stage's previous fill
      asm volatile("{\n\t.reg .pred P;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W;\n\t}\n"
                   ::"r"(su32(&bar[s])), "r"(phase[s]) : "memory");
      phase[s] ^= 1;
    }
    if (it >= iters) continue;
    seed = seed * 1664525u + 1013904223u;
    const int rb = (seed >> 8) % (ROWS / 128), kb = (seed >> 20) % 8;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(&bar[s])), "r"(STAGE) : "memory");
    uint8_t* dst = sm + s * STAGE;
    if (mode == 0) {  // 3D box {32, 128, 2}: 4 boxes of 16 KB
      for (int b = 0; b < 4; ++b)
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
                     ::"r"(su32(dst + b * 16384)), "l"(reinterpret_cast<uint64_t>(&map)), "r"(b * 192 + kb * 32 % 192),
                       "r"((rb * 128 + b * 128 * 37) % ROWS), "r"(0), "r"(su32(&bar[s])) : "memory");
    } else if (mode == 1) {  // 3D box {64, 128, 2}: 2 boxes of 32 KB
      for (int b = 0; b < 2; ++b)
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
                     ::"r"(su32(dst + b * 32768)), "l"(reinterpret_cast<uint64_t>(&map)), "r"(b * 384 + (kb % 4) * 64),
                       "r"((rb * 128 + b * 128 * 37) % ROWS), "r"(0), "r"(su32(&bar[s])) : "memory");
    } else {  // contiguous pre-tiled chunks: 4 x 16 KB 1D bulk copies
      const size_t total = (size_t)ROWS * LD * 2 * 2;
      for (int b = 0; b < 4; ++b) {
        const size_t off = (((size_t)(rb * 4 + b) * 8 + kb) * 16384) % total;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                     ::"r"(su32(dst + b * 16384)), "l"(flat + off), "r"(16384), "r"(su32(&bar[s])) : "memory");
      }
    }
  }
}

int main() {
  uint8_t* buf;
  const size_t bytes = (size_t)ROWS * LD * 2 * 2;
  CK(cudaMalloc(&buf, bytes));
  CK(cudaMemset(buf, 1, bytes));
  void* ptr = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q));
  auto enc = reinterpret_cast<CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                           const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                           CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill)>(ptr);
  const int smem = STAGES * STAGE + 1024;
  CK(cudaFuncSetAttribute(loads, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  printf("{");
  const int iters = 4000;
  for (int mode = 0; mode < 3; ++mode)
    for (int promo = 0; promo < 2; ++promo) {
      CUtensorMap map;
      cuuint64_t dims[3] = {LD, ROWS, 2};
      cuuint64_t str[2] = {LD * 2, (cuuint64_t)ROWS * LD * 2};
      cuuint32_t box[3] = {mode == 1 ? 64u : 32u, 128, 2}, es[3] = {1, 1, 1};
      auto sw = mode == 1 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
      auto pr = promo ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE;
      if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, pr,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        printf("\"enc_fail_%d\": 0, ", mode);
        continue;
      }
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      loads<<<148, 64, smem>>>(map, buf, mode, iters);
      cudaEventRecord(a);
      for (int r = 0; r < 5; ++r) loads<<<148, 64, smem>>>(map, buf, mode, iters);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      ms /= 5;
      printf("\"mode%d_promo%d\": {\"ms\": %.3f, \"GBs\": %.0f}, ", mode, promo, ms, 148.0 * iters * STAGE / ms / 1e6);
    }
  printf("\"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
