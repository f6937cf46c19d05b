// Per-SM output-tile write rate of three ways to move a staged 64 x 64 fp64
// tile pair (phi, psi: 64 KB) from shared memory to HBM, 1 CTA per SM, each
// CTA writing `tiles` tiles back to back (the small-m path's epilogue):
//   0: 128 one-row bulk copies (cp.async.bulk, 512 B each) per tile
//   1: 8 TMA tensor stores per tile (64-row x 16-column fp64 boxes, SWIZZLE_128B)
//   2: plain 16-byte st.global.cs by all 128 threads, from the staging
//   3: as 1, with two staging slots (a slot is restaged once the store two
//      tiles back has read it: cp.async.bulk.wait_group.read 1)
// Ring of independent output buffers > 4 x L2, CUDA events around each launch.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include <algorithm>

struct P { double* phi; double* psi; long long ld; int tiles; int T2; int mode; };

__global__ void __launch_bounds__(128, 1) k(const __grid_constant__ CUtensorMap mphi, const __grid_constant__ CUtensorMap mpsi, P p) {
  extern __shared__ __align__(1024) double sm[];
  double* Cphi = sm;            // mode 0/2: [64][66]; mode 1: 4 boxes of [64][16] swizzled
  double* Cpsi = sm + 64 * 66;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 2 * 64 * 66; i += 128) sm[i] = 1.0 + i;
  for (int t = 0; t < p.tiles; ++t) {
    const long long b = (long long)blockIdx.x * p.tiles + t;
    const int I = (int)(b / p.T2), J = (int)(b % p.T2);
    if (p.mode == 3) {
      if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
      Cphi = sm + (t & 1) * 8192;
    } else if (warp == 0) {
      asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    }
    __syncthreads();
    for (int i = tid; i < 64 * 32; i += 128) {   // "stage": touch every 16 B
      reinterpret_cast<double2*>(Cphi)[i] = make_double2(t, i);
      reinterpret_cast<double2*>(Cpsi)[i] = make_double2(i, t);
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (p.mode == 0) {
      if (warp == 0) {
        for (int r = lane; r < 64; r += 32) {
          double* d0 = p.phi + (long long)(I * 64 + r) * p.ld + J * 64;
          double* d1 = p.psi + (d0 - p.phi);
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 512;\n" ::"l"(d0), "r"((unsigned)__cvta_generic_to_shared(Cphi + r * 66)) : "memory");
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 512;\n" ::"l"(d1), "r"((unsigned)__cvta_generic_to_shared(Cpsi + r * 66)) : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      }
    } else if (p.mode == 1 || p.mode == 3) {
      if (tid == 0) {
        for (int q = 0; q < 4; ++q) {
          asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n"
                       ::"l"(&mphi), "r"(J * 64 + 16 * q), "r"(I * 64), "r"((unsigned)__cvta_generic_to_shared(Cphi + q * 1024)) : "memory");
          asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n"
                       ::"l"(&mpsi), "r"(J * 64 + 16 * q), "r"(I * 64), "r"((unsigned)__cvta_generic_to_shared(Cphi + 4096 + q * 1024)) : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      }
    } else {
      for (int i = tid; i < 64 * 32; i += 128) {
        const int r = i >> 5, c = (i & 31) * 2;
        __stcs(reinterpret_cast<double2*>(p.phi + (long long)(I * 64 + r) * p.ld + J * 64 + c), *reinterpret_cast<double2*>(Cphi + r * 66 + c));
        __stcs(reinterpret_cast<double2*>(p.psi + (long long)(I * 64 + r) * p.ld + J * 64 + c), *reinterpret_cast<double2*>(Cpsi + r * 66 + c));
      }
    }
  }
  if (tid == 0 || warp == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int R = 8;   // ring of output pairs
  const int tiles_per = 6, T2 = 24;
  const long long tiles = (long long)sms * tiles_per;
  const int T1 = (int)((tiles + T2 - 1) / T2);
  const long long rows = 64LL * T1, cols = 64LL * T2;
  std::vector<double*> ph(R), ps(R);
  std::vector<CUtensorMap> mp(R), mq(R);
  for (int r = 0; r < R; ++r) {
    cudaMalloc(&ph[r], rows * cols * 8); cudaMalloc(&ps[r], rows * cols * 8);
    for (int w = 0; w < 2; ++w) {
      cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
      cuuint64_t str[1] = {(cuuint64_t)cols * 8};
      cuuint32_t box[2] = {16, 64}, es[2] = {1, 1};
      enc(w ? &mq[r] : &mp[r], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, w ? ps[r] : ph[r], dims, str, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
  }
  const size_t smem = 2 * 65536;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* names[4] = {"bulk rows (128 x 512 B)", "TMA tensor boxes (8 x 8 KB)", "st.global.cs v2",
                          "TMA boxes, 2 staging slots"};
  for (int tp : {1, 6}) {
    for (int mode = 0; mode < 4; ++mode) {
      std::vector<float> v;
      for (int it = 0; it < 60; ++it) {
        const int r = it % R;
        P p{ph[r], ps[r], cols, tp, T2, mode};
        cudaEventRecord(a);
        k<<<sms, 128, smem>>>(mp[r], mq[r], p);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (it >= 10) v.push_back(ms * 1e3f);
      }
      std::sort(v.begin(), v.end());
      const double bytes = (double)sms * tp * 65536.0;
      printf("tiles/CTA %d  %-30s median %7.2f us  (%.0f GB/s, %.1f GB/s per SM)\n", tp, names[mode], v[v.size() / 2],
             bytes / v[v.size() / 2] / 1e3, bytes / sms / v[v.size() / 2] / 1e3);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
