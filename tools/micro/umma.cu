// Microbenchmark: tcgen05.mma kind::tf32 issue cost (SS mode, M=128) vs N and
// the number of independent accumulators the chain is spread over.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc(uint32_t a, int rowb) {
  uint64_t d = uint64_t((a & 0x3FFFF) >> 4) | (uint64_t(1) << 16) | (uint64_t((8 * rowb) >> 4) << 32) | (uint64_t(1) << 46);
  return d | (uint64_t(rowb == 128 ? 2 : 4) << 61);
}
__global__ void __launch_bounds__(128, 1) k(int n, int nacc, int iters, int rowb, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t slot;
  unsigned char* base = sm + ((1024u - (su(sm) & 1023u)) & 1023u);
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(base)[i] = 1.0f;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bar)), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&bar2)), "r"(1));
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
    const uint32_t id = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    const uint32_t a = su(base), b = su(base + 64 * 1024);
    long long t0 = clock64();
    const uint64_t da0 = desc(a, rowb), db0 = desc(b, rowb);
    const uint32_t id2 = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t((2 * n) >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    const uint64_t dal0 = desc(a + 32768, rowb);
    if (nacc == 1) {  // same-N chain: A*Wh, A*Wl, Al*Wh
      for (int i = 0; i < iters; i += 6) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm), "l"(da0 + 2 * u), "l"(db0 + 2 * u), "r"(id), "r"(i + u));
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm), "l"(da0 + 2 * u), "l"(db0 + 64 + 2 * u), "r"(id), "r"(1));
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm), "l"(dal0 + 2 * u), "l"(db0 + 2 * u), "r"(id), "r"(1));
        }
      }
    } else {  // ncat chain: A*[Wh;Wl] (2N), Al*Wh (N), commit every nacc*4 MMAs
      for (int i = 0; i < iters; i += 4) {
        if (nacc == 3) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (nacc == 2) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&bar2)) : "memory");
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm), "l"(da0 + 2 * u), "l"(db0 + 2 * u), "r"(id2), "r"(i + u));
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm), "l"(dal0 + 2 * u), "l"(db0 + 2 * u), "r"(id), "r"(1));
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
  for (int grid : {1, 2, 148})
  for (int rowb : {64})
    for (int n : {16, 128})
      for (int nacc : {1, 2, 3}) {
        if (n * nacc > 512) continue;
        const int iters = 480;
        long long h[2];
        for (int rep = 0; rep < 2; ++rep) {
          k<<<grid, 128, 140 * 1024>>>(n, nacc, iters, rowb, d);
          cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        }
        printf("grid=%3d rowb=%3d N=%3d nacc=%d: issue %6.1f cyc/mma, complete %6.1f cyc/mma (floor %5.1f)  %s\n", grid, rowb, n, nacc,
               double(h[0]) / iters, double(h[1]) / iters, 128.0 * n / 256, cudaGetErrorString(cudaGetLastError()));
      }
}
