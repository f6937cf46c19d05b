// Store-pattern microbenchmark for the homo contraction epilogue: 148 persistent
// CTAs write the upper-triangle 128x128 tiles of two 32768^2 fp32 planes plus their
// mirrors with TMA tensor stores of a given box shape, in the kernel's grouped
// raster order, with no compute.  Answers: how fast does the memory system accept
// this write pattern as a function of the box shape (row-segment length)?
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int INFLIGHT>
__global__ void __launch_bounds__(128, 1) tile_store(const __grid_constant__ CUtensorMap m0, const __grid_constant__ CUtensorMap m1,
                                                     const int2* tiles, int ntiles, int bw, int bh, int mirror) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 1.0f;
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncthreads();
  if (lane != 0) return;
  const int bx = 128 / bw, by = 128 / bh, nb = bx * by;
  int k = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int2 ij = tiles[t];
    const bool mir = mirror && ij.x != ij.y;
    for (int pl = 0; pl < 2; ++pl) {
      const CUtensorMap* m = pl ? &m1 : &m0;
      for (int b = warp; b < nb; b += 4) {
        const int r = ij.x * 128 + (b / bx) * bh, c = ij.y * 128 + (b % bx) * bw;
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n"
                     ::"l"(reinterpret_cast<uint64_t>(m)), "r"(c), "r"(r), "r"(su32(sm)) : "memory");
        if (mir) {
          const int r2 = ij.y * 128 + (b / bx) * bh, c2 = ij.x * 128 + (b % bx) * bw;
          asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n"
                       ::"l"(reinterpret_cast<uint64_t>(m)), "r"(c2), "r"(r2), "r"(su32(sm)) : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(INFLIGHT) : "memory");
        ++k;
      }
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

int main() {
  const long long n = 32768;
  float *p0, *p1;
  CK(cudaMalloc(&p0, n * n * 4));
  CK(cudaMalloc(&p1, n * n * 4));
  const int T = n / 128, G = 16;
  std::vector<int2> tiles;
  for (int i0 = 0; i0 < T; i0 += G)
    for (int j = i0; j < T; ++j)
      for (int i = i0; i < i0 + G && i < T; ++i)
        if (j >= i) tiles.push_back(make_int2(i, j));
  int2* dt;
  CK(cudaMalloc(&dt, tiles.size() * sizeof(int2)));
  CK(cudaMemcpy(dt, tiles.data(), tiles.size() * sizeof(int2), cudaMemcpyHostToDevice));
  void* ptr = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q));
  auto enc = reinterpret_cast<CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                           const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                           CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill)>(ptr);
  int shapes[][2] = {{32, 32}, {64, 32}, {128, 32}, {128, 8}, {128, 16}, {32, 128}, {16, 32}};
  cudaFuncSetAttribute(tile_store<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 17408);
  cudaFuncSetAttribute(tile_store<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 17408);
  printf("{");
  for (int mirror = 1; mirror >= 0; --mirror)
    for (auto& s : shapes)
      for (int infl : {1, 4}) {
        const int bw = s[0], bh = s[1];
        CUtensorMap m0, m1;
        cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)n};
        cuuint64_t str[1] = {(cuuint64_t)n * 4};
        cuuint32_t box[2] = {(cuuint32_t)bw, (cuuint32_t)bh}, es[2] = {1, 1};
        auto sw = bw == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE;
        if (enc(&m0, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, p0, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS ||
            enc(&m1, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, p1, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
          printf("\"enc_fail_%dx%d\": 0, ", bw, bh);
          continue;
        }
        auto k = infl == 1 ? tile_store<1> : tile_store<4>;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int w = 0; w < 2; ++w) k<<<148, 128, 17408>>>(m0, m1, dt, (int)tiles.size(), bw, bh, mirror);
        cudaEventRecord(a);
        const int reps = 5;
        for (int w = 0; w < reps; ++w) k<<<148, 128, 17408>>>(m0, m1, dt, (int)tiles.size(), bw, bh, mirror);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= reps;
        double bytes = 0;
        for (auto& t : tiles) bytes += 2.0 * 128 * 128 * 4 * ((mirror && t.x != t.y) ? 2 : 1);
        printf("\"%s_%dx%d_if%d\": {\"ms\": %.3f, \"GBs\": %.0f}, ", mirror ? "mir" : "dir", bw, bh, infl, ms,
               bytes / ms / 1e6);
        fflush(stdout);
      }
  printf("\"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
