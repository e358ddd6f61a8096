// Device helpers: complex64 arithmetic, fp64 block reductions.
#pragma once
#include <cuda_runtime.h>

namespace hb {

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
// a + s*b
__device__ __forceinline__ float2 caxpy(float2 a, float s, float2 b) {
  return make_float2(fmaf(s, b.x, a.x), fmaf(s, b.y, a.y));
}
__device__ __forceinline__ float2 crcp(float2 d) {
  const float s = 1.0f / fmaf(d.x, d.x, d.y * d.y);
  return make_float2(d.x * s, -d.y * s);
}

// Packed complex64 arithmetic on the sm_100 paired-fp32 pipe (FADD2 / FMUL2 /
// FFMA2: one instruction per complex add, two per complex multiply; ptxas folds
// the broadcasts, swizzles and per-lane negation into operand modifiers).
// Rounding is identical to the scalar helpers above (same fma association).
__device__ __forceinline__ unsigned long long pk2(float2 a) { return *reinterpret_cast<unsigned long long*>(&a); }
__device__ __forceinline__ float2 upk2(unsigned long long a) { return *reinterpret_cast<float2*>(&a); }
__device__ __forceinline__ float2 padd(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a)), "l"(pk2(b)));
  return upk2(r);
}
__device__ __forceinline__ float2 psub(float2 a, float2 b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a)), "l"(pk2(b)));
  return upk2(r);
}
__device__ __forceinline__ float2 pmulv(float2 a, float2 b) {  // element-wise
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a)), "l"(pk2(b)));
  return upk2(r);
}
__device__ __forceinline__ float2 pfmav(float2 a, float2 b, float2 c) {  // element-wise a*b + c
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk2(a)), "l"(pk2(b)), "l"(pk2(c)));
  return upk2(r);
}
__device__ __forceinline__ float2 pscale(float2 a, float s) { return pmulv(a, make_float2(s, s)); }
// a + s*b
__device__ __forceinline__ float2 paxpy(float2 a, float s, float2 b) { return pfmav(make_float2(s, s), b, a); }
// complex a*b (same roundings as cmul)
__device__ __forceinline__ float2 pmul(float2 a, float2 b) {
  float2 t = pmulv(make_float2(a.y, a.y), make_float2(b.y, b.x));
  t.x = -t.x;
  return pfmav(make_float2(a.x, a.x), b, t);
}

__device__ __forceinline__ double2 dadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
// conj(a) * b in fp64
__device__ __forceinline__ double2 dconjmul(float2 a, float2 b) {
  const double ax = a.x, ay = a.y, bx = b.x, by = b.y;
  return make_double2(fma(ax, bx, ay * by), fma(ax, by, -ay * bx));
}
__device__ __forceinline__ double dnorm2(float2 a) {
  const double ax = a.x, ay = a.y;
  return fma(ax, ax, ay * ay);
}
__device__ __forceinline__ float2 ld(const float2* p, size_t i) { return __ldg(p + i); }

// programmatic dependent launch (launch_pdl): block until the previous kernel's
// writes are visible.  No early launch_dependents: resident-but-waiting CTAs of
// the next kernel (the coarse solve takes a whole SM) would starve the other
// column groups' work (measured: early trigger 7.6k, wait-only 9.2k, off 9.0k
// c0 solves/s with 3 groups).
__device__ __forceinline__ void pdl_enter() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double2 warp_sum2(double2 v) {
  v.x = warp_sum(v.x);
  v.y = warp_sum(v.y);
  return v;
}

// 5-point stencil of u at (ix, iy) with zero padding: d*u - inv_h2*(sum of neighbours)
__device__ __forceinline__ float2 stencil_at(const float2* __restrict__ u, int nx, int ny, int ix, int iy,
                                             float2 d, float inv_h2, float s) {
  const size_t i = size_t(iy) * nx + ix;
  float2 nb = make_float2(0.f, 0.f);
  if (ix > 0) nb = cadd(nb, ld(u, i - 1));
  if (ix + 1 < nx) nb = cadd(nb, ld(u, i + 1));
  if (iy > 0) nb = cadd(nb, ld(u, i - nx));
  if (iy + 1 < ny) nb = cadd(nb, ld(u, i + nx));
  const float2 c = ld(u, i);
  float2 y = cmul(d, c);
  y.x = fmaf(-inv_h2, nb.x, y.x);
  y.y = fmaf(-inv_h2, nb.y, y.y);
  return cscale(y, s);
}

// same at storage index p of a row-slab field (u indexed by storage position;
// the rows above / below the slab are its ghost rows), bounds on global (ix, iy)
__device__ __forceinline__ float2 stencil_at_p(const float2* __restrict__ u, size_t p, int nx, int ny, int ix, int iy,
                                               float2 d, float inv_h2) {
  float2 nb = make_float2(0.f, 0.f);
  if (ix > 0) nb = cadd(nb, ld(u, p - 1));
  if (ix + 1 < nx) nb = cadd(nb, ld(u, p + 1));
  if (iy > 0) nb = cadd(nb, ld(u, p - nx));
  if (iy + 1 < ny) nb = cadd(nb, ld(u, p + nx));
  const float2 c = ld(u, p);
  float2 y = cmul(d, c);
  y.x = fmaf(-inv_h2, nb.x, y.x);
  y.y = fmaf(-inv_h2, nb.y, y.y);
  return y;
}

}  // namespace hb
