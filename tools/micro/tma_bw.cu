// Microbenchmark: per-SM copy throughput of TMA tensor boxes (64-B / 128-B rows)
// vs 1-D bulk copies, global (L2-resident) -> shared, 148 CTAs.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(su(b)), "r"(ph) : "memory");
}
__global__ void __launch_bounds__(32, 1) k(const __grid_constant__ CUtensorMap m, const float* g, int mode, int iters, int bytes, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar[4];
  unsigned char* base = sm + ((1024u - (su(sm) & 1023u)) & 1023u);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bar[i])), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  if (threadIdx.x != 0) return;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int s = it & 3;
    if (it >= 4) wait(&bar[s], ((it >> 2) - 1) & 1);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[s])), "r"(bytes) : "memory");
    unsigned char* dst = base + s * 48 * 1024;
    const int row = (blockIdx.x * 7 + it) % 64;
    if (mode == 2) {
      const float* src = g + size_t(row) * 128 * 16 * 3;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(dst)), "l"(src), "r"(bytes), "r"(su(&bar[s])) : "memory");
    } else {
      // box = (C, 128 px, rows): C = 16 (64-B rows) or 32 (128-B rows)
      asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(su(dst)), "l"(reinterpret_cast<uint64_t>(&m)), "r"(0), "r"(0), "r"(row), "r"(0), "r"(su(&bar[s])) : "memory");
    }
  }
  for (int s = 0; s < 4; ++s) wait(&bar[(iters + s) & 3], (((iters + s) >> 2) - 1) & 1);
  out[blockIdx.x] = clock64() - t0;
}
int main() {
  float* g; cudaMalloc(&g, 64 << 20);
  cudaMemset(g, 0, 64 << 20);
  long long* d; cudaMalloc(&d, 148 * 8);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int mode = 0; mode < 3; ++mode)
    for (int rows : {1, 3}) {
      const int C = mode == 1 ? 32 : 16;
      CUtensorMap m;
      const cuuint64_t dims[4] = {cuuint64_t(C), 128, 256, 1};
      const cuuint64_t strides[3] = {cuuint64_t(C) * 4, 128ull * C * 4, 256ull * 128 * C * 4};
      const cuuint32_t box[4] = {cuuint32_t(C), 128, cuuint32_t(rows), 1};
      const cuuint32_t es[4] = {1, 1, 1, 1};
      CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, g, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       C == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      const int bytes = C * 4 * 128 * rows;
      const int iters = 400;
      long long h[148];
      for (int rep = 0; rep < 2; ++rep) {
        k<<<148, 32, 200 * 1024>>>(m, g, mode, iters, bytes, d);
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      }
      long long mx = 0; for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
      const char* nm[3] = {"TMA 64B rows", "TMA 128B rows", "bulk 1-D"};
      printf("%-14s box %5d B: %7.1f cyc/copy, %6.1f B/clk/SM  (enc %d, %s)\n", nm[mode], bytes, double(mx) / iters,
             double(bytes) * iters / mx, int(r), cudaGetErrorString(cudaGetLastError()));
    }
}
