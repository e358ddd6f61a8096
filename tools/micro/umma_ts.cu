// Microbenchmark: tcgen05.mma kind::tf32 with A in TMEM (TS) vs A in smem (SS), M=128.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint32_t blo, uint32_t bhi, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\t.reg .b64 db;\n\tsetp.ne.b32 p, %5, 0;\n\tmov.b64 db, {%2, %3};\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], db, %4, p;\n\t}" ::"r"(d), "r"(a), "r"(blo), "r"(bhi), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint32_t alo, uint32_t ahi, uint32_t blo, uint32_t bhi, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\t.reg .b64 da, db;\n\tsetp.ne.b32 p, %6, 0;\n\tmov.b64 da, {%1, %2};\n\tmov.b64 db, {%3, %4};\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], da, db, %5, p;\n\t}" ::"r"(d), "r"(alo), "r"(ahi), "r"(blo), "r"(bhi), "r"(id), "r"(acc));
}
__global__ void __launch_bounds__(128, 1) k(int n, int mode, int iters, long long* out, int aoff) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  unsigned char* base = sm + ((1024u - (su(sm) & 1023u)) & 1023u);
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(base)[i] = 1.0f;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x == 0) {
    const uint32_t tm = slot;
    const uint32_t idN = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    const uint32_t id2N = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t((2 * n) >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    const uint32_t hi16 = (512u >> 4) | (1u << 14) | (4u << 29);
    const uint32_t alo = (su(base) >> 4) | (1u << 16), blo = (su(base + 64 * 1024) >> 4) | (1u << 16);
    const uint32_t ta = tm + aoff;
    long long t0 = clock64();
    for (int i = 0; i < iters; i += 8) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (mode == 0) {         // TS, same N chain
          mma_ts(tm, ta + 8 * u, blo + 2 * (u & 1), hi16, idN, i + u);
          mma_ts(tm, ta + 64 + 8 * u, blo + 2 * (u & 1), hi16, idN, 1);
        } else if (mode == 1) {  // TS, ncat pair (2N, N)
          mma_ts(tm, ta + 8 * u, blo + 2 * (u & 1), hi16, id2N, i + u);
          mma_ts(tm, ta + 64 + 8 * u, blo + 2 * (u & 1), hi16, idN, 1);
        } else {                 // SS, ncat pair
          mma_ss(tm, alo + 2 * (u & 1) + 512 * (u >> 1), hi16, blo + 2 * (u & 1), hi16, id2N, i + u);
          mma_ss(tm, alo + 1024 + 2 * (u & 1), hi16, blo + 2 * (u & 1), hi16, idN, 1);
        }
      }
    }
    long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&bar)) : "memory");
    asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(su(&bar)), "r"(0) : "memory");
    long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(512));
}
int main() {
  long long* d; cudaMalloc(&d, 16);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  const char* names[3] = {"TS same-N", "TS ncat", "SS ncat"};
  for (int aoff : {256})
  for (int mode = 0; mode < 3; ++mode)
    for (int n : {16, 48, 64, 128}) {
      const int iters = 512;
      long long h[2];
      for (int rep = 0; rep < 2; ++rep) {
        k<<<148, 128, 140 * 1024>>>(n, mode, iters, d, aoff);
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      }
      printf("aoff=%3d %-10s N=%3d: issue %6.1f cyc/mma, complete %6.1f cyc/mma  %s\n", aoff, names[mode], n, double(h[0]) / iters,
             double(h[1]) / iters, cudaGetErrorString(cudaGetLastError()));
    }
}
