// Measured dense TF32 tensor peak of this GPU: tcgen05.mma.cta_group::1.kind::tf32,
// A and B from shared memory (SS), M = 128, N = 256, K = 8 per instruction,
// fp32 accumulators in TMEM (two 256-column accumulators alternated).  One CTA
// per SM issues `iters` MMAs back to back from one elected thread; the whole
// grid is timed with CUDA events (2 * 128 * 256 * 8 flops per MMA).  The
// operands are constant (re-read from smem every MMA), so this is the
// issue-rate ceiling of the tensor pipe for kind::tf32 -- the denominator used
// for the U-Net convolutions' "% of tensor peak".
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tf32_peak tf32_peak.cu && ./tf32_peak
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
// K-major, no swizzle: 8-row x 16-byte core matrices; LBO (K direction) 128 B, SBO (M/N) 8 rows x 16 B... as used by
// the repo's conv kernels (rowb = 128: 128 B per row segment, SWIZZLE_128B)
__device__ __forceinline__ uint64_t desc128(uint32_t a) {
  return uint64_t((a & 0x3FFFF) >> 4) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) | (uint64_t(1) << 46) |
         (uint64_t(2) << 61);
}

__global__ void __launch_bounds__(128, 1) k_peak(int iters, int n, unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  unsigned char* base = sm + ((1024u - (su(sm) & 1023u)) & 1023u);
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(base)[i] = 1.0f / 1024;
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
    // instruction descriptor: D fp32 (bit 4), A/B tf32 (2 at 7, 2 at 10), K-major, N >> 3 at 17, M >> 4 at 24
    const uint32_t id = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    const uint64_t da = desc128(su(base)), db = desc128(su(base + 32 * 1024));
    for (int i = 0; i < iters; i += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t d = tm + (u & 1) * 256;  // two accumulators
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
            "l"(da + 2 * (u >> 1)), "l"(db + 2 * (u >> 1)), "r"(id), "r"(i + u > 1 ? 1 : 0));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&bar)) : "memory");
    asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
                     su(&bar)),
                 "r"(0)
                 : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x < 32) {
    uint32_t r0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r0) : "r"(slot));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (threadIdx.x == 0) atomicAdd(sink, r0);
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(512));
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  const int smem = 170 * 1024;
  cudaFuncSetAttribute(k_peak, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("{\"sms\": %d, \"runs\": [", sms);
  bool first = true;
  for (int n : {128, 256}) {
    const int iters = 1 << 16;
    k_peak<<<sms, 128, smem>>>(1024, n, sink);  // warm-up
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      k_peak<<<sms, 128, smem>>>(iters, n, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double flops = double(sms) * iters * 2.0 * 128 * n * 8;
    printf("%s{\"M\": 128, \"N\": %d, \"K\": 8, \"iters_per_sm\": %d, \"ms\": %.4f, \"tflops\": %.1f, \"err\": \"%s\"}",
           first ? "" : ", ", n, iters, best, flops / (best * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    first = false;
  }
  printf("]}\n");
  return 0;
}
