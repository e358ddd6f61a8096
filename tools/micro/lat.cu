// Dependent-chain latency of a few ALU ops on the B200 (cycles per op).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a, float fa, int n) {
  double x = a, y = a * 0.5;
  float f = fa;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) x = fma(x, y, 0.25);
  }
  t1 = clock64();
  cyc[0] = t1 - t0;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) x = x + y;
  }
  t1 = clock64();
  cyc[1] = t1 - t0;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) f = fmaf(f, fa, 0.25f);
  }
  t1 = clock64();
  cyc[2] = t1 - t0;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) x = double(float(x)) + 1.0;  // F2F.F32.F64 + F2F.F64.F32 + DADD
  }
  t1 = clock64();
  cyc[3] = t1 - t0;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1.0;
  }
  t1 = clock64();
  cyc[4] = t1 - t0;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) x = rsqrt(x) + 1.0;
  }
  t1 = clock64();
  cyc[5] = t1 - t0;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) f = __shfl_xor_sync(0xffffffffu, f, 1) + 1.f;
  }
  t1 = clock64();
  cyc[6] = t1 - t0;
  out[threadIdx.x] = x + f;
}
int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 32 * 8);
  cudaMallocManaged(&c, 8 * 8);
  const int n = 64;
  k<<<1, 32>>>(o, c, 1.0000001, 1.0000001f, n);
  cudaDeviceSynchronize();
  k<<<1, 32>>>(o, c, 1.0000001, 1.0000001f, n);
  cudaDeviceSynchronize();
  const char* names[] = {"DFMA", "DADD", "FFMA", "F2F+F2F+DADD", "SHFL(f64 as 2)+DADD", "rsqrt(f64)+DADD", "SHFL+FADD"};
  for (int i = 0; i < 7; ++i) printf("%-22s %.1f cyc/op\n", names[i], double(c[i]) / (16.0 * n));
  return 0;
}
