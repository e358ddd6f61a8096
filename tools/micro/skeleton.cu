// Microbenchmark: cost of the tcgen05 conv kernel's pipeline skeleton (no data).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(su(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(b)) : "memory"); }
template <int MODE>
__global__ void __launch_bounds__(320, 1) k(int iters, int stages) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t full[8], cvt[8], empty[8];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&cvt[s])), "r"(128));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&empty[s])), "r"(1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (MODE >= 1 && warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su(&slot)), "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  if (MODE >= 2) {
    int s = 0; uint32_t ph = 0;
    if (warp == 0 && lane == 0) {
      for (int it = 0; it < iters; ++it) {
        if (it >= stages) wait(&empty[s], ph ^ 1);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[s])), "r"(0) : "memory");
        if (++s == stages) { s = 0; ph ^= 1; }
      }
    } else if (warp == 1 && lane == 0) {
      for (int it = 0; it < iters; ++it) {
        wait(&cvt[s], ph);
        if (MODE >= 3) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&empty[s])) : "memory");
        else arrive(&empty[s]);
        if (++s == stages) { s = 0; ph ^= 1; }
      }
    } else if (warp >= 2 && warp < 6) {
      for (int it = 0; it < iters; ++it) {
        wait(&full[s], ph);
        if (MODE >= 4) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        arrive(&cvt[s]);
        if (++s == stages) { s = 0; ph ^= 1; }
      }
    }
  }
  __syncthreads();
  if (MODE >= 1 && warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(32));
}
template <int M>
void run(const char* name, int iters, int stages, size_t smem) {
  cudaFuncSetAttribute(k<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 5; ++i) k<M><<<148, 320, smem>>>(iters, stages);
  cudaEventRecord(a);
  for (int i = 0; i < 100; ++i) k<M><<<148, 320, smem>>>(iters, stages);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("%-28s iters=%4d stages=%d smem=%6zu: %7.2f us/launch  err=%s\n", name, iters, stages, smem, ms * 10, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  for (size_t smem : {size_t(0), size_t(200 * 1024)}) {
    run<0>("empty", 0, 4, smem);
    run<1>("tmem alloc", 0, 4, smem);
    for (int it : {36, 360}) {
      run<2>("ring (arrive)", it, 4, smem);
      run<3>("ring (tcgen05.commit)", it, 4, smem);
      run<4>("ring (+proxy fence)", it, 4, smem);
    }
  }
}
