// Training of the paper's U-Net on the device:
// traindet::run_batch (inc/training.hpp:121-147) -- the train-mode forward of
// build_unet / build_encoder (inc/unet.hpp:139-257), the MSE loss, the reverse
// sweep of the Tape rules (inc/autodiff.hpp:121-480) -- and bias-corrected
// ADAM (inc/adam.hpp:25-58), driven by the reference's epoch loops train() and
// retrain() (inc/training.hpp:152-298).
//
// The tape is a static op list built once per (batch, H, W, mode) from the same
// registry the inference path uses (hb_paper.h), so parameter names, creation
// order and trainable flags are the reference's.  Layout NCHW fp32 like the
// reference's Tensor4, all activations and gradients in one device arena each,
// all parameters / gradients / ADAM moments in flat device buffers in registry
// order.  Kernels:
//   conv forward          direct, thread = 1 output pixel x 8 output channels
//   transposed conv       gather form of the exact adjoint (same kernel layout)
//   conv input gradient   = transposed conv of dy with the conv's kernel; the
//                           transposed conv's input gradient = conv of dz
//   kernel gradient       one CTA per (channel pair), thread-strided pixels,
//                           per-tap fp32 partials, fp64 block reduction
//   batch norm            fp64 channel statistics (two passes, as the
//                           reference), normalise; backward fp64 channel sums;
//                           every channel reduction is split over (channel,
//                           slice) CTAs and folded in a fixed order
//   ELU / add / concat / MSE / ADAM   elementwise (ADAM in fp64 arithmetic)
// The reductions the reference carries in double (batch-norm statistics, bias
// and loss sums, ADAM) are double here; convolution sums are fp32 in both
// (the reference's Eigen / sgemm products), in a different order.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "hb_common.cuh"
#include "hb_host.h"
#include "hb_internal.h"
#include "hb_paper.h"

namespace hb {

namespace {

constexpr int TB = 256;  // threads per CTA of the elementwise / pixel kernels
constexpr int CO = 8;    // output channels per thread (conv forward kernels)

inline int nblk(size_t n) { return int(std::min<size_t>((n + TB - 1) / TB, size_t(1) << 20)); }

// ------------------------------------------------------------------ kernels
// y[b,co,oy,ox] = bias[co] + sum_{ci,ky,kx} x[b,ci,oy*s+ky-p,ox*s+kx-p] K[co,ci,ky,kx]
// (conv2d, inc/autodiff.hpp:121-150: zero padding p = (k-1)/2, cross-correlation)
constexpr int PX = 4;  // output pixels per thread along x (forward convolutions)

template <int K, int S, int CO>
__global__ void __launch_bounds__(TB) k_conv_fwd(const float* __restrict__ x, int cin, int H, int W,
                                                 const float* __restrict__ Kw, const float* __restrict__ bias, int cout,
                                                 int Ho, int Wo, float* __restrict__ y) {
  const int gx = (Wo + PX - 1) / PX;
  const int gid = blockIdx.x * TB + threadIdx.x;
  const int co0 = blockIdx.y * CO, b = blockIdx.z;
  if (gid >= Ho * gx) return;
  constexpr int P = (K - 1) / 2, KK = K * K;
  const int oy = gid / gx, ox0 = (gid % gx) * PX;
  float acc[PX][CO];
#pragma unroll
  for (int q = 0; q < PX; ++q)
#pragma unroll
    for (int j = 0; j < CO; ++j) acc[q][j] = 0.f;
  int cj[CO];
#pragma unroll
  for (int j = 0; j < CO; ++j) cj[j] = min(co0 + j, cout - 1);
  for (int ci = 0; ci < cin; ++ci) {
    const float* xp = x + (size_t(b) * cin + ci) * H * W;
#pragma unroll
    for (int ky = 0; ky < K; ++ky) {
      const int iy = oy * S + ky - P;
      if (iy < 0 || iy >= H) continue;
#pragma unroll
      for (int kx = 0; kx < K; ++kx) {
        float xv[PX];
#pragma unroll
        for (int q = 0; q < PX; ++q) {
          const int ix = (ox0 + q) * S + kx - P;
          xv[q] = (ix >= 0 && ix < W) ? __ldg(xp + size_t(iy) * W + ix) : 0.f;
        }
#pragma unroll
        for (int j = 0; j < CO; ++j) {
          const float wv = __ldg(Kw + (size_t(cj[j]) * cin + ci) * KK + ky * K + kx);
#pragma unroll
          for (int q = 0; q < PX; ++q) acc[q][j] = fmaf(xv[q], wv, acc[q][j]);
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < CO; ++j) {
    const int co = co0 + j;
    if (co >= cout) continue;
    const float bv = bias ? __ldg(bias + co) : 0.f;
#pragma unroll
    for (int q = 0; q < PX; ++q)
      if (ox0 + q < Wo) y[(size_t(b) * cout + co) * Ho * Wo + size_t(oy) * Wo + ox0 + q] = acc[q][j] + bv;
  }
}

// output channels per thread: the layer's count rounded up to 2 / 4, else 8
template <int K, int S>
void conv_co(cudaStream_t st, dim3 g, const float* x, int cin, int H, int W, const float* Kw, const float* bias,
             int cout, int Ho, int Wo, float* y) {
  if (cout <= 2) {
    g.y = unsigned((cout + 1) / 2);
    k_conv_fwd<K, S, 2><<<g, TB, 0, st>>>(x, cin, H, W, Kw, bias, cout, Ho, Wo, y);
  } else if (cout <= 4) {
    g.y = 1;
    k_conv_fwd<K, S, 4><<<g, TB, 0, st>>>(x, cin, H, W, Kw, bias, cout, Ho, Wo, y);
  } else {  // 16 channels per thread measured slower (registers)
    g.y = unsigned((cout + 7) / 8);
    k_conv_fwd<K, S, 8><<<g, TB, 0, st>>>(x, cin, H, W, Kw, bias, cout, Ho, Wo, y);
  }
}
void launch_conv(cudaStream_t st, dim3 g, const float* x, int cin, int H, int W, const float* Kw, const float* bias,
                 int cout, int k, int s, int Ho, int Wo, float* y) {
  g.x = unsigned((Ho * ((Wo + PX - 1) / PX) + TB - 1) / TB);  // one thread per PX output pixels
  if (k == 5 && s == 2)
    conv_co<5, 2>(st, g, x, cin, H, W, Kw, bias, cout, Ho, Wo, y);
  else if (k == 3 && s == 1)
    conv_co<3, 1>(st, g, x, cin, H, W, Kw, bias, cout, Ho, Wo, y);
  else if (k == 5 && s == 1)
    conv_co<5, 1>(st, g, x, cin, H, W, Kw, bias, cout, Ho, Wo, y);
  else if (k == 3 && s == 2)
    conv_co<3, 2>(st, g, x, cin, H, W, Kw, bias, cout, Ho, Wo, y);
  else if (k == 1 && s == 1)
    conv_co<1, 1>(st, g, x, cin, H, W, Kw, bias, cout, Ho, Wo, y);
  else if (k == 1 && s == 2)
    conv_co<1, 2>(st, g, x, cin, H, W, Kw, bias, cout, Ho, Wo, y);
  else
    throw HbError{HB_ERR_ARG, "training supports 1x1, 3x3 and 5x5 kernels with stride 1 or 2"};
}

// z[b,cb,Y,X] += bias[cb] + sum_{ca, ky, kx: Y = y*s+ky-p, X = x*s+kx-p} u[b,ca,y,x] K[ca,cb,ky,kx]
// (conv2d_transpose, inc/autodiff.hpp:155-211: the exact adjoint of conv2d).
// Gather form with the kernel size and stride as template arguments: for
// stride 2 only the taps of the output pixel's parity class reach it
// (ky = (Y + p) mod 2, +2, ...), so a 5x5 tap loop visits 4-9 taps, not 25.
template <int K, int S, int CO>
__global__ void __launch_bounds__(TB) k_convT_fwd(const float* __restrict__ u, int ca, int h, int w,
                                                  const float* __restrict__ Kw, const float* __restrict__ bias, int cb,
                                                  int H, int W, float* __restrict__ z) {
  // thread = PX output pixels X = xb + S*q (one parity class) of one row
  constexpr int SPAN = S * PX;
  const int gx = ((W + SPAN - 1) / SPAN) * S;
  const int gid = blockIdx.x * TB + threadIdx.x;
  const int c0 = blockIdx.y * CO, b = blockIdx.z;
  if (gid >= H * gx) return;
  constexpr int P = (K - 1) / 2, KK = K * K;
  const int Y = gid / gx, g = gid % gx;
  const int xb = (g / S) * SPAN + (g % S);
  const int ky0 = S == 2 ? (Y + P) & 1 : 0, kx0 = S == 2 ? (xb + P) & 1 : 0;
  float acc[PX][CO];
#pragma unroll
  for (int q = 0; q < PX; ++q)
#pragma unroll
    for (int j = 0; j < CO; ++j) acc[q][j] = 0.f;
  int cj[CO];
#pragma unroll
  for (int j = 0; j < CO; ++j) cj[j] = min(c0 + j, cb - 1);
  for (int a = 0; a < ca; ++a) {
    const float* up = u + (size_t(b) * ca + a) * h * w;
    const float* ka = Kw + size_t(a) * cb * KK;
    for (int ky = ky0; ky < K; ky += S) {
      const int ty = Y + P - ky;
      if (ty < 0 || ty / S >= h) continue;
      const int y = ty / S;  // exact: ty is a multiple of S
      for (int kx = kx0; kx < K; kx += S) {
        float uv[PX];
#pragma unroll
        for (int q = 0; q < PX; ++q) {
          const int tx = xb + S * q + P - kx;  // multiple of S; input column tx / S = (xb + P - kx) / S + q
          uv[q] = (tx >= 0 && tx / S < w && xb + S * q < W) ? __ldg(up + size_t(y) * w + tx / S) : 0.f;
        }
        const int t = ky * K + kx;
#pragma unroll
        for (int j = 0; j < CO; ++j) {
          const float wv = __ldg(ka + size_t(cj[j]) * KK + t);
#pragma unroll
          for (int q = 0; q < PX; ++q) acc[q][j] = fmaf(uv[q], wv, acc[q][j]);
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < CO; ++j) {
    const int c = c0 + j;
    if (c >= cb) continue;
    const float bv = bias ? __ldg(bias + c) : 0.f;
#pragma unroll
    for (int q = 0; q < PX; ++q) {
      const int X = xb + S * q;
      if (X < W) z[(size_t(b) * cb + c) * H * W + size_t(Y) * W + X] += acc[q][j] + bv;
    }
  }
}

template <int K, int S>
void convT_co(cudaStream_t st, dim3 g, const float* u, int ca, int h, int w, const float* Kw, const float* bias, int cb,
              int H, int W, float* z) {
  if (cb <= 2) {
    g.y = 1;
    k_convT_fwd<K, S, 2><<<g, TB, 0, st>>>(u, ca, h, w, Kw, bias, cb, H, W, z);
  } else if (cb <= 4) {
    g.y = 1;
    k_convT_fwd<K, S, 4><<<g, TB, 0, st>>>(u, ca, h, w, Kw, bias, cb, H, W, z);
  } else {
    g.y = unsigned((cb + 7) / 8);
    k_convT_fwd<K, S, 8><<<g, TB, 0, st>>>(u, ca, h, w, Kw, bias, cb, H, W, z);
  }
}
void launch_convT(cudaStream_t st, dim3 g, const float* u, int ca, int h, int w, const float* Kw, const float* bias,
                  int cb, int k, int s, int H, int W, float* z) {
  g.x = unsigned((H * ((W + s * PX - 1) / (s * PX)) * s + TB - 1) / TB);  // one thread per PX pixels of a parity class
  if (k == 5 && s == 2)
    convT_co<5, 2>(st, g, u, ca, h, w, Kw, bias, cb, H, W, z);
  else if (k == 3 && s == 1)
    convT_co<3, 1>(st, g, u, ca, h, w, Kw, bias, cb, H, W, z);
  else if (k == 5 && s == 1)
    convT_co<5, 1>(st, g, u, ca, h, w, Kw, bias, cb, H, W, z);
  else if (k == 3 && s == 2)
    convT_co<3, 2>(st, g, u, ca, h, w, Kw, bias, cb, H, W, z);
  else if (k == 1 && s == 1)
    convT_co<1, 1>(st, g, u, ca, h, w, Kw, bias, cb, H, W, z);
  else if (k == 1 && s == 2)
    convT_co<1, 2>(st, g, u, ca, h, w, Kw, bias, cb, H, W, z);
  else
    throw HbError{HB_ERR_ARG, "training supports 1x1, 3x3 and 5x5 kernels with stride 1 or 2"};
}

// dK[a,c,ky,kx] += sum_{b,y,x} A[b,a,y,x] X[b,c,y*s+ky-p,x*s+kx-p]
// conv2d: A = dy (cout), X = x (cin); conv2d_transpose: A = u (x channels), X = dz
template <int K, int S>
__global__ void __launch_bounds__(TB) k_wgrad(int nb, const float* __restrict__ A, int na, int h, int w,
                                              const float* __restrict__ X, int nc, int H, int W,
                                              float* __restrict__ dK) {
  const int a = blockIdx.x / nc, c = blockIdx.x % nc;
  constexpr int P = (K - 1) / 2, KK = K * K;
  float acc[KK];
#pragma unroll
  for (int t = 0; t < KK; ++t) acc[t] = 0.f;
  const int hw = h * w;
  const size_t total = size_t(nb) * hw;
  for (size_t i = threadIdx.x; i < total; i += TB) {
    const int b = int(i / hw), q = int(i % hw);
    const int y = q / w, x = q % w;
    const float av = __ldg(A + (size_t(b) * na + a) * hw + q);
    const float* xp = X + (size_t(b) * nc + c) * H * W;
#pragma unroll
    for (int ky = 0; ky < K; ++ky) {
      const int iy = y * S + ky - P;
      if (iy < 0 || iy >= H) continue;
#pragma unroll
      for (int kx = 0; kx < K; ++kx) {
        const int ix = x * S + kx - P;
        if (ix >= 0 && ix < W) acc[ky * K + kx] = fmaf(av, __ldg(xp + size_t(iy) * W + ix), acc[ky * K + kx]);
      }
    }
  }
  __shared__ double red[TB / 32];
#pragma unroll 1
  for (int t = 0; t < KK; ++t) {
    double v = acc[t];
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s2 = 0;
      for (int r = 0; r < TB / 32; ++r) s2 += red[r];
      dK[(size_t(a) * nc + c) * KK + t] += float(s2);
    }
    __syncthreads();
  }
}

// Kernel gradient, blocked: a CTA owns one X channel c, AB A channels and one
// pixel slice; per pixel the K*K shifted X taps are loaded once and reused for
// the AB channels (AB*K*K FMAs per K*K + AB loads, the per-pair kernel above
// does one load per FMA).  Per-CTA fp64 partials go to ws[slice][a][c][t];
// k_wgrad_fold sums the slices in order (deterministic).
template <int K, int S, int AB>
__global__ void __launch_bounds__(TB) k_wgrad_blk(int nb, const float* __restrict__ A, int na, int h, int w,
                                                  const float* __restrict__ X, int nc, int H, int W,
                                                  double* __restrict__ ws) {
  const int c = blockIdx.x % nc, a0 = (blockIdx.x / nc) * AB;
  constexpr int P = (K - 1) / 2, KK = K * K;
  const int hw = h * w;
  const size_t total = size_t(nb) * hw, per = (total + gridDim.y - 1) / gridDim.y;
  const size_t lo = blockIdx.y * per, hi = min(total, lo + per);
  float acc[AB][KK];
#pragma unroll
  for (int u = 0; u < AB; ++u)
#pragma unroll
    for (int t = 0; t < KK; ++t) acc[u][t] = 0.f;
  int ac[AB];
#pragma unroll
  for (int u = 0; u < AB; ++u) ac[u] = min(a0 + u, na - 1);
  for (size_t i = lo + threadIdx.x; i < hi; i += TB) {
    const int b = int(i / hw), q = int(i % hw);
    const int y = q / w, x = q % w;
    float av[AB];
#pragma unroll
    for (int u = 0; u < AB; ++u) av[u] = __ldg(A + (size_t(b) * na + ac[u]) * hw + q);
    const float* xp = X + (size_t(b) * nc + c) * H * W;
#pragma unroll
    for (int ky = 0; ky < K; ++ky) {
      const int iy = y * S + ky - P;
      const bool oky = iy >= 0 && iy < H;
#pragma unroll
      for (int kx = 0; kx < K; ++kx) {
        const int ix = x * S + kx - P;
        const float xv = (oky && ix >= 0 && ix < W) ? __ldg(xp + size_t(iy) * W + ix) : 0.f;
#pragma unroll
        for (int u = 0; u < AB; ++u) acc[u][ky * K + kx] = fmaf(av[u], xv, acc[u][ky * K + kx]);
      }
    }
  }
  __shared__ double red[TB / 32][AB * KK];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
#pragma unroll
  for (int u = 0; u < AB; ++u)
#pragma unroll
    for (int t = 0; t < KK; ++t) {
      const double v = warp_sum(double(acc[u][t]));
      if (lane == 0) red[wp][u * KK + t] = v;
    }
  __syncthreads();
  const size_t slab = size_t(na) * nc * KK;
  for (int e = threadIdx.x; e < AB * KK; e += TB) {
    const int u = e / KK, t = e % KK;
    if (a0 + u >= na) continue;
    double s2 = 0;
    for (int r = 0; r < TB / 32; ++r) s2 += red[r][e];
    ws[blockIdx.y * slab + (size_t(a0 + u) * nc + c) * KK + t] = s2;
  }
}
__global__ void k_wgrad_fold(size_t n, int slices, const double* __restrict__ ws, float* dK) {
  for (size_t i = blockIdx.x * size_t(TB) + threadIdx.x; i < n; i += size_t(gridDim.x) * TB) {
    double s2 = 0;
    for (int j = 0; j < slices; ++j) s2 += ws[size_t(j) * n + i];
    dK[i] += float(s2);
  }
}

template <int K, int S, int AB>
void wgrad_blk(cudaStream_t st, int nsm, DBuf<double>& wsb, int nb, const float* A, int na, int h, int w,
               const float* X, int nc, int H, int W, float* dK) {
  const int groups = nc * ((na + AB - 1) / AB);
  const size_t pix = size_t(nb) * h * w;
  const int slices = int(std::max<size_t>(1, std::min<size_t>((size_t(2) * nsm + groups - 1) / groups, pix / 4096)));
  const size_t n = size_t(na) * nc * K * K;
  wsb.ensure(n * size_t(slices));
  k_wgrad_blk<K, S, AB><<<dim3(groups, slices), TB, 0, st>>>(nb, A, na, h, w, X, nc, H, W, wsb.p);
  k_wgrad_fold<<<nblk(n), TB, 0, st>>>(n, slices, wsb.p, dK);
}

void launch_wgrad(cudaStream_t st, int grid, int nb, const float* A, int na, int h, int w, const float* X, int nc,
                  int H, int W, int k, int s, float* dK, int nsm = 0, DBuf<double>* wsb = nullptr) {
  if (wsb && k == 3 && s == 1) return wgrad_blk<3, 1, 8>(st, nsm, *wsb, nb, A, na, h, w, X, nc, H, W, dK);
  if (wsb && k == 5 && s == 2) return wgrad_blk<5, 2, 2>(st, nsm, *wsb, nb, A, na, h, w, X, nc, H, W, dK);
  if (k == 5 && s == 2)
    k_wgrad<5, 2><<<grid, TB, 0, st>>>(nb, A, na, h, w, X, nc, H, W, dK);
  else if (k == 3 && s == 1)
    k_wgrad<3, 1><<<grid, TB, 0, st>>>(nb, A, na, h, w, X, nc, H, W, dK);
  else if (k == 5 && s == 1)
    k_wgrad<5, 1><<<grid, TB, 0, st>>>(nb, A, na, h, w, X, nc, H, W, dK);
  else if (k == 3 && s == 2)
    k_wgrad<3, 2><<<grid, TB, 0, st>>>(nb, A, na, h, w, X, nc, H, W, dK);
  else if (k == 1 && s == 1)
    k_wgrad<1, 1><<<grid, TB, 0, st>>>(nb, A, na, h, w, X, nc, H, W, dK);
  else if (k == 1 && s == 2)
    k_wgrad<1, 2><<<grid, TB, 0, st>>>(nb, A, na, h, w, X, nc, H, W, dK);
  else
    throw HbError{HB_ERR_ARG, "training supports 1x1, 3x3 and 5x5 kernels with stride 1 or 2"};
}

__device__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0;
  for (int i = 0; i < TB / 32; ++i) t += red[i];
  __syncthreads();
  return t;
}

// y = (x - mu) * is * g + be
__global__ void k_bn_apply(size_t n, int C, int plane, const float* __restrict__ x, const float2* __restrict__ st,
                           const float* __restrict__ g, const float* __restrict__ be, float* __restrict__ y) {
  for (size_t i = blockIdx.x * size_t(TB) + threadIdx.x; i < n; i += size_t(gridDim.x) * TB) {
    const int c = int((i / plane) % C);
    const float2 m = st[c];
    y[i] = (x[i] - m.x) * m.y * g[c] + be[c];
  }
}


// ---- split channel reductions: grid (C, S), CTA (c, j) sums slice j of the
// channel's nb * plane elements into part[c * S + j] (fp64, fixed order), a
// finishing kernel adds the S partials in order (deterministic)
enum { RED_SUM = 0, RED_SQDEV = 1, RED_BNBWD = 2 };
template <int MODE>
__global__ void __launch_bounds__(TB) k_chpart(int nb, int C, int plane, const float* __restrict__ x,
                                               const float* __restrict__ go, const double* __restrict__ mean,
                                               const float2* __restrict__ st, double2* part) {
  const int c = blockIdx.x, S = gridDim.y, j = blockIdx.y;
  const size_t n = size_t(nb) * plane, per = (n + S - 1) / S, lo = j * per, hi = min(n, lo + per);
  __shared__ double red[TB / 32];
  double a = 0, b = 0;
  const double mu64 = MODE == RED_SQDEV ? mean[c] : 0.0;
  const float mu = MODE == RED_BNBWD ? st[c].x : 0.f, is = MODE == RED_BNBWD ? st[c].y : 0.f;
  for (size_t i = lo + threadIdx.x; i < hi; i += TB) {
    const size_t o = ((i / plane) * C + c) * plane + i % plane;
    if (MODE == RED_SUM) {
      a += x[o];
    } else if (MODE == RED_SQDEV) {
      const double d = x[o] - mu64;
      a += d * d;
    } else {
      const double gp = go[o];
      a += gp;
      b += gp * (x[o] - mu) * is;
    }
  }
  a = block_sum(a, red);
  if (MODE == RED_BNBWD) b = block_sum(b, red);
  if (threadIdx.x == 0) part[size_t(c) * S + j] = make_double2(a, b);
}
__device__ __forceinline__ double2 fold(const double2* part, int c, int S) {
  double2 t = make_double2(0, 0);
  for (int j = 0; j < S; ++j) {
    t.x += part[size_t(c) * S + j].x;
    t.y += part[size_t(c) * S + j].y;
  }
  return t;
}
// mean[c] = sum / cnt
__global__ void k_fin_mean(int C, int S, double cnt, const double2* part, double* mean) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < C) mean[c] = fold(part, c, S).x / cnt;
}
// var, running buffers, (mean_f, inv_std_f)
__global__ void k_fin_var(int C, int S, double cnt, const double2* part, const double* mean, float eps, float momentum,
                          float* rmean, float* rvar, float* count, float2* st) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const double var = fold(part, c, S).x / cnt;
  rmean[c] = momentum * rmean[c] + (1.0f - momentum) * float(mean[c]);
  rvar[c] = momentum * rvar[c] + (1.0f - momentum) * float(var);
  if (c == 0) count[0] += 1.0f;
  st[c] = make_float2(float(mean[c]), float(1.0 / sqrt(var + double(eps))));
}
__global__ void k_bn_eval_stats(int C, float eps, const float* rmean, const float* rvar, float2* st) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < C) st[c] = make_float2(float(double(rmean[c])), float(1.0 / sqrt(double(rvar[c]) + double(eps))));
}
// bias gradients: out[c] += float(sum)
__global__ void k_fin_sum(int C, int S, const double2* part, float* out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < C) out[c] += float(fold(part, c, S).x);
}
// batch norm backward: scale / offset gradients and the (sum dy, sum dy xhat) / cnt pairs
__global__ void k_fin_bnbwd(int C, int S, double cnt, const double2* part, float* dscale, float* doffset,
                            double2* coef) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const double2 t = fold(part, c, S);
  if (dscale) dscale[c] += float(t.y);
  if (doffset) doffset[c] += float(t.x);
  coef[c] = make_double2(t.x / cnt, t.y / cnt);
}
__global__ void k_bn_dx(size_t n, int C, int plane, const float* __restrict__ x, const float* __restrict__ go,
                        const float2* __restrict__ st, const float* __restrict__ g, const double2* __restrict__ coef,
                        int train, float* dx) {
  for (size_t i = blockIdx.x * size_t(TB) + threadIdx.x; i < n; i += size_t(gridDim.x) * TB) {
    const int c = int((i / plane) % C);
    const float mu = st[c].x, is = st[c].y, gc = g[c];
    if (train) {
      const double xhat = double(x[i] - mu) * is;
      dx[i] += float(double(gc) * is * (go[i] - coef[c].x - xhat * coef[c].y));
    } else {
      dx[i] += gc * is * go[i];
    }
  }
}
// mse: partial sums of (p - t)^2 over slices, then loss = float(sum / nb); gp += 2/nb (p - t)
__global__ void __launch_bounds__(TB) k_sqdiff_part(size_t n, const float* __restrict__ p, const float* __restrict__ t,
                                                    double* part) {
  const size_t per = (n + gridDim.x - 1) / gridDim.x, lo = blockIdx.x * per, hi = min(n, lo + per);
  __shared__ double red[TB / 32];
  double s = 0;
  for (size_t i = lo + threadIdx.x; i < hi; i += TB) {
    const double d = double(p[i]) - t[i];
    s += d * d;
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}
__global__ void k_fin_mse(int S, int nb, const double* part, double* loss) {
  double s = 0;
  for (int j = 0; j < S; ++j) s += part[j];
  *loss = double(float(s / nb));
}
__global__ void k_mse_grad(size_t n, int nb, const float* __restrict__ p, const float* __restrict__ t, float* gp) {
  const float scale = 2.0f * 1.0f / float(nb);
  for (size_t i = blockIdx.x * size_t(TB) + threadIdx.x; i < n; i += size_t(gridDim.x) * TB) gp[i] += scale * (p[i] - t[i]);
}

__global__ void k_elu(size_t n, const float* __restrict__ x, float* __restrict__ y) {
  for (size_t i = blockIdx.x * size_t(TB) + threadIdx.x; i < n; i += size_t(gridDim.x) * TB) {
    const float t = x[i];
    y[i] = t >= 0.0f ? t : expm1f(t);
  }
}
__global__ void k_elu_bwd(size_t n, const float* __restrict__ x, const float* __restrict__ y,
                          const float* __restrict__ go, float* gx) {
  for (size_t i = blockIdx.x * size_t(TB) + threadIdx.x; i < n; i += size_t(gridDim.x) * TB)
    gx[i] += go[i] * (x[i] >= 0.0f ? 1.0f : y[i] + 1.0f);
}
__global__ void k_add(size_t n, const float* __restrict__ a, const float* __restrict__ b, float* __restrict__ y) {
  for (size_t i = blockIdx.x * size_t(TB) + threadIdx.x; i < n; i += size_t(gridDim.x) * TB) y[i] = a[i] + b[i];
}
__global__ void k_acc(size_t n, const float* __restrict__ g, float* d) {
  for (size_t i = blockIdx.x * size_t(TB) + threadIdx.x; i < n; i += size_t(gridDim.x) * TB) d[i] += g[i];
}
// channel concatenation [a | b] per batch slab; bsl = 0 broadcasts b over the batch
__global__ void k_concat(int nb, size_t sa, size_t sb, const float* __restrict__ a, const float* __restrict__ b,
                         size_t bsl, float* __restrict__ y) {
  const size_t so = sa + sb, n = size_t(nb) * so;
  for (size_t i = blockIdx.x * size_t(TB) + threadIdx.x; i < n; i += size_t(gridDim.x) * TB) {
    const size_t bi = i / so, q = i % so;
    y[i] = q < sa ? a[bi * sa + q] : b[bi * bsl + q - sa];
  }
}
__global__ void k_concat_bwd(int nb, size_t sa, size_t sb, const float* __restrict__ go, float* ga, float* gb) {
  const size_t so = sa + sb, n = size_t(nb) * so;
  for (size_t i = blockIdx.x * size_t(TB) + threadIdx.x; i < n; i += size_t(gridDim.x) * TB) {
    const size_t bi = i / so, q = i % so;
    if (q < sa) {
      if (ga) ga[bi * sa + q] += go[i];
    } else if (gb) {
      gb[bi * sb + q - sa] += go[i];
    }
  }
}
// non-finite count over a buffer
__global__ void k_nonfinite(size_t n, const float* __restrict__ g, int* bad) {
  int any = 0;
  for (size_t i = blockIdx.x * size_t(TB) + threadIdx.x; i < n; i += size_t(gridDim.x) * TB) any |= !isfinite(g[i]);
  if (__syncthreads_or(any) && threadIdx.x == 0) atomicAdd(bad, 1);
}
// ADAM (inc/adam.hpp:38-55), fp64 arithmetic, fp32 state
__global__ void k_adam(size_t n, const float* __restrict__ g, float* m, float* v, float* w, double lr, double b1,
                       double b2, double bc1, double bc2, double eps) {
  for (size_t i = blockIdx.x * size_t(TB) + threadIdx.x; i < n; i += size_t(gridDim.x) * TB) {
    const double gi = g[i];
    m[i] = float(b1 * m[i] + (1.0 - b1) * gi);
    v[i] = float(b2 * v[i] + (1.0 - b2) * gi * gi);
    const double mh = m[i] / bc1, vh = v[i] / bc2;
    w[i] -= float(lr * mh / (sqrt(vh) + eps));
  }
}

// ------------------------------------------------------------------ the tape
struct Ten {
  int n, c, h, w;
  size_t off;    // value offset in the arena
  bool grad;     // carries a gradient (not a leaf)
  size_t size() const { return size_t(n) * c * h * w; }
};

enum OpK { OP_CONV, OP_CONVT, OP_BN, OP_ELU, OP_ADD, OP_CONCAT };

struct Op {
  OpK kind;
  int a = -1, b = -1, y = -1;  // tensor ids
  int pk = -1, pb = -1;        // kernel / bias parameter (registry index)
  int k = 0, s = 1;
  int pbn = -1;                // batch norm: registry index of ".scale" (offset, rmean, rvar, count follow)
  bool train = true;
  size_t st = 0;               // batch norm: offset of its (mean, inv_std) pairs in the stats buffer
  bool bcast_b = false;        // concat: b is batch-1, broadcast
};

}  // namespace

struct TrainState {
  // flat parameter store (registry order) and per-parameter offsets
  std::vector<size_t> poff;
  size_t ptotal = 0;
  std::vector<char> trainable;
  DBuf<float> dparam, dgrad, adam_m, adam_v, snapshot;
  bool params_on_device = false;
  unsigned long long gen = ~0ull;  // PaperState::host_gen of the uploaded parameters
  long long adam_step = 0, adam_skipped = 0;
  bool adam_init = false;
  // tape
  int key_B = -1, key_H = -1, key_W = -1, key_mode = -1;
  std::vector<Ten> tens;
  std::vector<Op> ops;
  int t_input = -1, t_kappa = -1, t_target = -1, t_out = -1;
  std::vector<int> t_feats;  // frozen feature leaves (encoder_solver retrain)
  size_t arena = 0, nstats = 0;
  DBuf<float> vals, grads, tmp;
  DBuf<float2> stats;
  DBuf<double> dloss, dmean, wsw;
  DBuf<double2> dpart, dcoef;
  DBuf<int> dbad;
  // frozen encoder features (batch 1) for retrain
  std::vector<std::vector<float>> frozen;  // per level, NCHW [1][C][H>>l][W>>l]
  std::vector<std::array<int, 3>> frozen_dims;
};

namespace {


bool ends_with(const std::string& s, const char* t) {
  const size_t n = std::strlen(t);
  return s.size() >= n && s.compare(s.size() - n, n, t) == 0;
}
bool is_buffer(const std::string& n) { return ends_with(n, ".rmean") || ends_with(n, ".rvar") || ends_with(n, ".count"); }

TrainState& tstate(Context& c) {
  if (!c.train) c.train = std::make_shared<TrainState>();
  return *c.train;
}

// parameters to the device (flat, registry order); trainable flags default to
// the reference's (every kernel / bias / scale / offset; buffers are not)
void ensure_params(Context& c) {
  PaperState& P = paper_state(c);
  TrainState& T = tstate(c);
  if (!P.active) throw HbError{HB_ERR_STATE, "paper net not set (hb_set_paper_net)"};
  if (T.params_on_device && T.gen == P.host_gen && T.poff.size() == P.params.size()) return;
  T.poff.assign(P.params.size(), 0);
  T.trainable.assign(P.params.size(), 0);
  size_t o = 0;
  for (size_t i = 0; i < P.params.size(); ++i) {
    T.poff[i] = o;
    o += (P.params[i].size() + 3) & ~size_t(3);
    T.trainable[i] = !is_buffer(P.params[i].name);
  }
  T.ptotal = o;
  T.dparam.ensure(o);
  T.dgrad.ensure(o);
  std::vector<float> h(o, 0.f);
  for (size_t i = 0; i < P.params.size(); ++i)
    std::copy(P.params[i].v.begin(), P.params[i].v.end(), h.begin() + long(T.poff[i]));
  HB_CUDA(cudaMemcpyAsync(T.dparam.p, h.data(), o * sizeof(float), cudaMemcpyHostToDevice, c.stream));
  HB_CUDA(cudaStreamSynchronize(c.stream));
  T.params_on_device = true;
  T.gen = P.host_gen;
  T.adam_init = false;
  T.adam_step = 0;
  T.key_B = -1;
}

// device parameters back to the host registry (inference path re-uploads)
void params_to_host(Context& c) {
  PaperState& P = paper_state(c);
  TrainState& T = tstate(c);
  if (!T.params_on_device) return;
  std::vector<float> h(T.ptotal);
  // on the library stream: it does not synchronise with the legacy default stream
  HB_CUDA(cudaMemcpyAsync(h.data(), T.dparam.p, T.ptotal * sizeof(float), cudaMemcpyDeviceToHost, c.stream));
  HB_CUDA(cudaStreamSynchronize(c.stream));
  for (size_t i = 0; i < P.params.size(); ++i)
    std::copy(h.begin() + long(T.poff[i]), h.begin() + long(T.poff[i] + P.params[i].size()), P.params[i].v.begin());
  P.dirty = true;
  P.feat_gen = ~0ull;
}

struct Builder {
  const PaperState& P;
  TrainState& T;
  bool train;
  int pidx(const std::string& n) const {
    auto it = P.index.find(n);
    if (it == P.index.end()) throw HbError{HB_ERR_STATE, "paper net has no parameter " + n};
    return int(it->second);
  }
  int ten(int n, int c, int h, int w, bool grad) {
    T.tens.push_back(Ten{n, c, h, w, 0, grad});
    return int(T.tens.size()) - 1;
  }
  int conv(int x, const std::string& kn, const std::string& bn, int stride) {
    const Ten& X = T.tens[size_t(x)];
    const PParam& K = P.params[size_t(pidx(kn))];
    const int k = K.d[2];
    if (k > 5) throw HbError{HB_ERR_ARG, "training supports kernels up to 5x5"};
    if (K.d[1] != X.c) throw HbError{HB_ERR_STATE, "conv kernel in-channels mismatch at " + kn};
    const int p = (k - 1) / 2;
    const int ho = (X.h + 2 * p - k) / stride + 1, wo = (X.w + 2 * p - k) / stride + 1;
    Op o{OP_CONV};
    o.a = x;
    o.pk = pidx(kn);
    o.pb = pidx(bn);
    o.k = k;
    o.s = stride;
    o.y = ten(X.n, K.d[0], ho, wo, true);
    T.ops.push_back(o);
    return o.y;
  }
  int convT(int x, const std::string& kn, const std::string& bn, int stride) {
    const Ten& X = T.tens[size_t(x)];
    const PParam& K = P.params[size_t(pidx(kn))];
    if (K.d[0] != X.c) throw HbError{HB_ERR_STATE, "deconv kernel in-channels mismatch at " + kn};
    if (K.d[2] > 5) throw HbError{HB_ERR_ARG, "training supports kernels up to 5x5"};
    Op o{OP_CONVT};
    o.a = x;
    o.pk = pidx(kn);
    o.pb = pidx(bn);
    o.k = K.d[2];
    o.s = stride;
    o.y = ten(X.n, K.d[1], X.h * stride, X.w * stride, true);
    T.ops.push_back(o);
    return o.y;
  }
  int bn(int x, const std::string& name) {
    const Ten& X = T.tens[size_t(x)];
    Op o{OP_BN};
    o.a = x;
    o.pbn = pidx(name + ".scale");
    o.train = train;
    o.st = T.nstats;
    T.nstats += size_t(X.c);
    o.y = ten(X.n, X.c, X.h, X.w, true);
    T.ops.push_back(o);
    return o.y;
  }
  int elu(int x) {
    const Ten& X = T.tens[size_t(x)];
    Op o{OP_ELU};
    o.a = x;
    o.y = ten(X.n, X.c, X.h, X.w, true);
    T.ops.push_back(o);
    return o.y;
  }
  int add(int a, int b) {
    const Ten& A = T.tens[size_t(a)];
    Op o{OP_ADD};
    o.a = a;
    o.b = b;
    o.y = ten(A.n, A.c, A.h, A.w, true);
    T.ops.push_back(o);
    return o.y;
  }
  int concat(int a, int b) {
    const Ten A = T.tens[size_t(a)], Bt = T.tens[size_t(b)];
    Op o{OP_CONCAT};
    o.a = a;
    o.b = b;
    o.bcast_b = Bt.n == 1 && A.n > 1;
    o.y = ten(A.n, A.c + Bt.c, A.h, A.w, true);
    T.ops.push_back(o);
    return o.y;
  }
  // x <- elu(BN2(x + K2 elu(BN1(K1 x))))  (netdet::resnet_block, inc/unet.hpp:147-160)
  int resnet(const std::string& n, int x) {
    int t = conv(x, n + ".k1", n + ".b1", 1);
    t = elu(bn(t, n + ".bn1"));
    t = conv(t, n + ".k2", n + ".b2", 1);
    return elu(bn(add(x, t), n + ".bn2"));
  }
  // build_encoder (inc/unet.hpp:231-257)
  std::vector<int> encoder(int kap) {
    const hb_unet_cfg& c = P.cfg;
    std::vector<int> f;
    int x = elu(bn(conv(kap, "enc.entry.k", "enc.entry.b", 1), "enc.entry.bn"));
    f.push_back(x);
    for (int l = 0; l < c.levels; ++l) {
      const std::string d = "enc.down" + std::to_string(l);
      x = elu(bn(conv(x, d + ".k", d + ".b", 2), d + ".bn"));
      for (int r = 0; r < c.resnet_per_level; ++r) x = resnet("enc.res" + std::to_string(l + 1) + "_" + std::to_string(r), x);
      f.push_back(x);
    }
    return f;
  }
  // build_unet (inc/unet.hpp:165-226)
  int unet(int input, const std::string& pre, const std::vector<int>& feats) {
    const hb_unet_cfg& c = P.cfg;
    const bool es = !feats.empty();
    std::vector<int> skips(size_t(c.levels));
    skips[0] = input;
    int x = input;
    for (int l = 0; l < c.levels; ++l) {
      if (es) x = concat(x, feats[size_t(l)]);
      const std::string d = pre + "down" + std::to_string(l);
      x = elu(bn(conv(x, d + ".k", d + ".b", 2), d + ".bn"));
      if (l < c.levels - 1) {
        for (int r = 0; r < c.resnet_per_level; ++r) x = resnet(pre + "res" + std::to_string(l + 1) + "_" + std::to_string(r), x);
        skips[size_t(l) + 1] = x;
      }
    }
    for (int r = 0; r < c.bottleneck_resnets; ++r) x = resnet(pre + "bot" + std::to_string(r), x);
    for (int s = c.levels; s >= 1; --s) {
      const int t = s - 1;
      if (es) x = concat(x, feats[size_t(s)]);
      x = elu(x);
      const std::string u = pre + "up" + std::to_string(t);
      x = bn(convT(x, u + ".k", u + ".b", 2), u + ".bn");
      x = concat(x, skips[size_t(t)]);
    }
    return conv(x, pre + "out.k", pre + "out.b", 1);
  }
};

// mode: 0 standalone, 1 encoder_solver joint, 2 encoder_solver with frozen
// features, 3 the encoder alone in eval mode (frozen features)
void build_tape(Context& c, int B, int H, int W, int mode, bool train) {
  PaperState& P = paper_state(c);
  TrainState& T = tstate(c);
  const int key_mode = mode * 2 + (train ? 1 : 0);
  if (T.key_B == B && T.key_H == H && T.key_W == W && T.key_mode == key_mode) return;
  if (H % (1 << P.cfg.levels) || W % (1 << P.cfg.levels))
    throw HbError{HB_ERR_ARG, "input dims must be divisible by 2^levels"};
  T.tens.clear();
  T.ops.clear();
  T.t_feats.clear();
  T.nstats = 0;
  Builder bd{P, T, train};
  if (mode == 3) {
    T.t_kappa = bd.ten(1, 1, H, W, false);
    T.t_feats = bd.encoder(T.t_kappa);
    T.t_input = T.t_target = T.t_out = -1;
  } else {
    T.t_input = bd.ten(B, 4, H, W, false);
    T.t_target = bd.ten(B, 2, H, W, false);
    T.t_kappa = -1;
    std::vector<int> feats;
    if (mode == 1) {
      T.t_kappa = bd.ten(B, 1, H, W, false);
      feats = bd.encoder(T.t_kappa);
    } else if (mode == 2) {
      if (T.frozen.size() != size_t(P.cfg.levels) + 1) throw HbError{HB_ERR_STATE, "no frozen encoder features"};
      for (size_t l = 0; l < T.frozen.size(); ++l)
        feats.push_back(bd.ten(1, T.frozen_dims[l][0u], T.frozen_dims[l][1u], T.frozen_dims[l][2u], false));
      T.t_feats = feats;
    }
    T.t_out = bd.unet(T.t_input, mode == 0 ? "unet." : "sol.", feats);
  }
  size_t o = 0;
  for (auto& t : T.tens) {
    t.off = o;
    o += (t.size() + 3) & ~size_t(3);
  }
  T.arena = o;
  T.vals.ensure(o);
  T.grads.ensure(o);
  T.stats.ensure(std::max<size_t>(1, T.nstats));
  T.dloss.ensure(1);
  T.dbad.ensure(1);
  T.key_B = B;
  T.key_H = H;
  T.key_W = W;
  T.key_mode = key_mode;
}

float* V(TrainState& T, int t) { return T.vals.p + T.tens[size_t(t)].off; }
float* G(TrainState& T, int t) { return T.tens[size_t(t)].grad ? T.grads.p + T.tens[size_t(t)].off : nullptr; }
float* PV(TrainState& T, int i) { return T.dparam.p + T.poff[size_t(i)]; }
float* PG(TrainState& T, int i) { return T.trainable[size_t(i)] ? T.dgrad.p + T.poff[size_t(i)] : nullptr; }
int egrid(size_t n) { return nblk(n); }

// slices per channel so that C * S CTAs fill the GPU (>= 2048 elements per slice)
int split_s(const Context& c, int C, size_t per_channel) {
  const size_t want = (size_t(4) * c.num_sms + size_t(C) - 1) / size_t(C);
  const size_t cap = std::max<size_t>(1, per_channel / 2048);
  return int(std::max<size_t>(1, std::min<size_t>({want, cap, size_t(256)})));
}
void ensure_red(TrainState& T, size_t parts, size_t C) {
  T.dpart.ensure(std::max<size_t>(parts, 1024));
  T.dmean.ensure(std::max<size_t>(C, 1024));
  T.dcoef.ensure(std::max<size_t>(C, 1024));
}
// bias gradient: out[c] += sum over (batch, plane) of g
void chsum(Context& c, TrainState& T, int nb, int C, int plane, const float* g, float* out) {
  const int S = split_s(c, C, size_t(nb) * plane);
  ensure_red(T, size_t(C) * S, size_t(C));
  k_chpart<RED_SUM><<<dim3(C, S), TB, 0, c.stream>>>(nb, C, plane, g, nullptr, nullptr, nullptr, T.dpart.p);
  k_fin_sum<<<(C + 127) / 128, 128, 0, c.stream>>>(C, S, T.dpart.p, out);
}
// batch norm statistics (inc/autodiff.hpp:228-262).  train: biased batch mean /
// variance in fp64 (two passes, as the reference), running buffers folded with
// momentum 0.9, update count bumped; eval: the running buffers.
void bn_forward_stats(Context& c, TrainState& T, const Op& o, const Ten& A) {
  const int C = A.c, plane = A.h * A.w;
  float2* st = T.stats.p + o.st;
  if (!o.train) {
    k_bn_eval_stats<<<(C + 127) / 128, 128, 0, c.stream>>>(C, 1e-5f, PV(T, o.pbn + 2), PV(T, o.pbn + 3), st);
    return;
  }
  const int S = split_s(c, C, size_t(A.n) * plane);
  ensure_red(T, size_t(C) * S, size_t(C));
  const double cnt = double(A.n) * plane;
  k_chpart<RED_SUM><<<dim3(C, S), TB, 0, c.stream>>>(A.n, C, plane, V(T, o.a), nullptr, nullptr, nullptr, T.dpart.p);
  k_fin_mean<<<(C + 127) / 128, 128, 0, c.stream>>>(C, S, cnt, T.dpart.p, T.dmean.p);
  k_chpart<RED_SQDEV><<<dim3(C, S), TB, 0, c.stream>>>(A.n, C, plane, V(T, o.a), nullptr, T.dmean.p, nullptr, T.dpart.p);
  k_fin_var<<<(C + 127) / 128, 128, 0, c.stream>>>(C, S, cnt, T.dpart.p, T.dmean.p, 1e-5f, 0.9f, PV(T, o.pbn + 2),
                                                   PV(T, o.pbn + 3), PV(T, o.pbn + 4), st);
}
// batch norm backward (inc/autodiff.hpp:281-318): fp64 channel sums of dy and
// dy * xhat -> scale / offset gradients, then dx (train: through the batch
// statistics; eval: g * is * dy)
void bn_backward(Context& c, TrainState& T, const Op& o, const Ten& A, const float* gy) {
  const int C = A.c, plane = A.h * A.w;
  const float2* st = T.stats.p + o.st;
  const int S = split_s(c, C, size_t(A.n) * plane);
  ensure_red(T, size_t(C) * S, size_t(C));
  const double cnt = double(A.n) * plane;
  k_chpart<RED_BNBWD><<<dim3(C, S), TB, 0, c.stream>>>(A.n, C, plane, V(T, o.a), gy, nullptr, st, T.dpart.p);
  k_fin_bnbwd<<<(C + 127) / 128, 128, 0, c.stream>>>(C, S, cnt, T.dpart.p, PG(T, o.pbn), PG(T, o.pbn + 1), T.dcoef.p);
  if (float* dx = G(T, o.a))
    k_bn_dx<<<egrid(A.size()), TB, 0, c.stream>>>(A.size(), C, plane, V(T, o.a), gy, st, PV(T, o.pbn), T.dcoef.p,
                                                  o.train ? 1 : 0, dx);
}

void run_forward(Context& c) {
  TrainState& T = tstate(c);
  cudaStream_t st = c.stream;
  for (const Op& o : T.ops) {
    const Ten& A = T.tens[size_t(o.a)];
    const Ten& Y = T.tens[size_t(o.y)];
    switch (o.kind) {
      case OP_CONV: {
        const dim3 g((Y.h * Y.w + TB - 1) / TB, (Y.c + CO - 1) / CO, Y.n);
        launch_conv(st, g, V(T, o.a), A.c, A.h, A.w, PV(T, o.pk), PV(T, o.pb), Y.c, o.k, o.s, Y.h, Y.w, V(T, o.y));
        break;
      }
      case OP_CONVT: {
        HB_CUDA(cudaMemsetAsync(V(T, o.y), 0, Y.size() * sizeof(float), st));
        const dim3 g((Y.h * Y.w + TB - 1) / TB, (Y.c + CO - 1) / CO, Y.n);
        launch_convT(st, g, V(T, o.a), A.c, A.h, A.w, PV(T, o.pk), PV(T, o.pb), Y.c, o.k, o.s, Y.h, Y.w, V(T, o.y));
        break;
      }
      case OP_BN: {
        const int plane = A.h * A.w;
        bn_forward_stats(c, T, o, A);
        k_bn_apply<<<egrid(A.size()), TB, 0, st>>>(A.size(), A.c, plane, V(T, o.a), T.stats.p + o.st, PV(T, o.pbn),
                                                   PV(T, o.pbn + 1), V(T, o.y));
        break;
      }
      case OP_ELU:
        k_elu<<<egrid(A.size()), TB, 0, st>>>(A.size(), V(T, o.a), V(T, o.y));
        break;
      case OP_ADD:
        k_add<<<egrid(A.size()), TB, 0, st>>>(A.size(), V(T, o.a), V(T, o.b), V(T, o.y));
        break;
      case OP_CONCAT: {
        const Ten& Bt = T.tens[size_t(o.b)];
        const size_t sa = size_t(A.c) * A.h * A.w, sb = size_t(Bt.c) * Bt.h * Bt.w;
        k_concat<<<egrid(Y.size()), TB, 0, st>>>(A.n, sa, sb, V(T, o.a), V(T, o.b), o.bcast_b ? 0 : sb, V(T, o.y));
        break;
      }
    }
    HB_CUDA(cudaGetLastError());
  }
}

void run_backward(Context& c) {
  TrainState& T = tstate(c);
  cudaStream_t st = c.stream;
  for (auto it = T.ops.rbegin(); it != T.ops.rend(); ++it) {
    const Op& o = *it;
    const Ten& A = T.tens[size_t(o.a)];
    const Ten& Y = T.tens[size_t(o.y)];
    const float* gy = G(T, o.y);
    switch (o.kind) {
      case OP_CONV: {
        if (float* dk = PG(T, o.pk)) {
          launch_wgrad(st, Y.c * A.c, Y.n, gy, Y.c, Y.h, Y.w, V(T, o.a), A.c, A.h, A.w, o.k, o.s, dk, c.num_sms,
                       c.opt_wgrad_blk ? &T.wsw : nullptr);
        }
        if (float* db = PG(T, o.pb)) chsum(c, T, Y.n, Y.c, Y.h * Y.w, gy, db);
        if (float* dx = G(T, o.a)) {  // dx += conv^T(dy; K)
          const dim3 g((A.h * A.w + TB - 1) / TB, (A.c + CO - 1) / CO, A.n);
          launch_convT(st, g, gy, Y.c, Y.h, Y.w, PV(T, o.pk), nullptr, A.c, o.k, o.s, A.h, A.w, dx);
        }
        break;
      }
      case OP_CONVT: {
        // dK[a, c] += sum u[a] dz[c] (shifted); du += conv(dz; K viewed as (a, c))
        if (float* dk = PG(T, o.pk)) {
          launch_wgrad(st, A.c * Y.c, A.n, V(T, o.a), A.c, A.h, A.w, gy, Y.c, Y.h, Y.w, o.k, o.s, dk, c.num_sms,
                       c.opt_wgrad_blk ? &T.wsw : nullptr);
        }
        if (float* db = PG(T, o.pb)) chsum(c, T, Y.n, Y.c, Y.h * Y.w, gy, db);
        if (float* dx = G(T, o.a)) {
          // the conv kernel writes its output: run it into scratch, then accumulate
          T.tmp.ensure(A.size());
          float* tmp = T.tmp.p;
          const dim3 g((A.h * A.w + TB - 1) / TB, (A.c + CO - 1) / CO, A.n);
          launch_conv(st, g, gy, Y.c, Y.h, Y.w, PV(T, o.pk), nullptr, A.c, o.k, o.s, A.h, A.w, tmp);
          k_acc<<<egrid(A.size()), TB, 0, st>>>(A.size(), tmp, dx);
        }
        break;
      }
      case OP_BN:
        bn_backward(c, T, o, A, gy);
        break;
      case OP_ELU:
        if (float* gx = G(T, o.a)) k_elu_bwd<<<egrid(A.size()), TB, 0, st>>>(A.size(), V(T, o.a), V(T, o.y), gy, gx);
        break;
      case OP_ADD:
        if (float* ga = G(T, o.a)) k_acc<<<egrid(A.size()), TB, 0, st>>>(A.size(), gy, ga);
        if (float* gb = G(T, o.b)) k_acc<<<egrid(A.size()), TB, 0, st>>>(A.size(), gy, gb);
        break;
      case OP_CONCAT: {
        const Ten& Bt = T.tens[size_t(o.b)];
        float* ga = G(T, o.a);
        float* gb = o.bcast_b ? nullptr : G(T, o.b);
        if (ga || gb)
          k_concat_bwd<<<egrid(Y.size()), TB, 0, st>>>(A.n, size_t(A.c) * A.h * A.w, size_t(Bt.c) * Bt.h * Bt.w, gy, ga,
                                                       gb);
        break;
      }
    }
    HB_CUDA(cudaGetLastError());
  }
}

// run_batch (inc/training.hpp:121-147) on host NCHW inputs; returns the loss
double run_batch(Context& c, int B, int H, int W, const float* input, const float* kappa, const float* target,
                 bool train, bool with_grad, float* out_host) {
  PaperState& P = paper_state(c);
  TrainState& T = tstate(c);
  ensure_params(c);
  const int mode = P.variant == 0 ? 0 : (T.frozen.empty() ? 1 : 2);
  build_tape(c, B, H, W, mode, train);
  cudaStream_t st = c.stream;
  HB_CUDA(cudaMemcpyAsync(V(T, T.t_input), input, sizeof(float) * size_t(B) * 4 * H * W, cudaMemcpyHostToDevice, st));
  HB_CUDA(cudaMemcpyAsync(V(T, T.t_target), target, sizeof(float) * size_t(B) * 2 * H * W, cudaMemcpyHostToDevice, st));
  if (mode == 1) {
    if (!kappa) throw HbError{HB_ERR_ARG, "encoder_solver training needs the kappa^2 batch"};
    HB_CUDA(cudaMemcpyAsync(V(T, T.t_kappa), kappa, sizeof(float) * size_t(B) * H * W, cudaMemcpyHostToDevice, st));
  }
  if (mode == 2)
    for (size_t l = 0; l < T.frozen.size(); ++l)
      HB_CUDA(cudaMemcpyAsync(V(T, T.t_feats[l]), T.frozen[l].data(), sizeof(float) * T.frozen[l].size(),
                              cudaMemcpyHostToDevice, st));
  run_forward(c);
  const Ten& O = T.tens[size_t(T.t_out)];
  if (with_grad) {
    HB_CUDA(cudaMemsetAsync(T.grads.p, 0, sizeof(float) * T.arena, st));
    HB_CUDA(cudaMemsetAsync(T.dgrad.p, 0, sizeof(float) * T.ptotal, st));
  }
  {  // mse_loss (inc/autodiff.hpp:448-470)
    const int S = int(std::min<size_t>(size_t(4) * c.num_sms, std::max<size_t>(1, O.size() / 2048)));
    ensure_red(T, size_t(S), 1);
    double* part = reinterpret_cast<double*>(T.dpart.p);
    k_sqdiff_part<<<S, TB, 0, st>>>(O.size(), V(T, T.t_out), V(T, T.t_target), part);
    k_fin_mse<<<1, 1, 0, st>>>(S, O.n, part, T.dloss.p);
    if (with_grad) k_mse_grad<<<egrid(O.size()), TB, 0, st>>>(O.size(), O.n, V(T, T.t_out), V(T, T.t_target), G(T, T.t_out));
  }
  HB_CUDA(cudaGetLastError());
  if (with_grad) run_backward(c);
  double loss = 0;
  HB_CUDA(cudaMemcpyAsync(&loss, T.dloss.p, sizeof(double), cudaMemcpyDeviceToHost, st));
  if (out_host) HB_CUDA(cudaMemcpyAsync(out_host, V(T, T.t_out), sizeof(float) * O.size(), cudaMemcpyDeviceToHost, st));
  HB_CUDA(cudaStreamSynchronize(st));
  return loss;
}

// adam_step (inc/adam.hpp:25-58) over the trainable parameters; false = skipped
bool adam_step(Context& c, double lr) {
  PaperState& P = paper_state(c);
  TrainState& T = tstate(c);
  cudaStream_t st = c.stream;
  if (!T.adam_init) {
    T.adam_m.ensure(T.ptotal);
    T.adam_v.ensure(T.ptotal);
    HB_CUDA(cudaMemsetAsync(T.adam_m.p, 0, sizeof(float) * T.ptotal, st));
    HB_CUDA(cudaMemsetAsync(T.adam_v.p, 0, sizeof(float) * T.ptotal, st));
    T.adam_init = true;
    T.adam_step = 0;
  }
  HB_CUDA(cudaMemsetAsync(T.dbad.p, 0, sizeof(int), st));
  for (size_t i = 0; i < P.params.size(); ++i)
    if (T.trainable[i])
      k_nonfinite<<<egrid(P.params[i].size()), TB, 0, st>>>(P.params[i].size(), PG(T, int(i)), T.dbad.p);
  int bad = 0;
  HB_CUDA(cudaMemcpyAsync(&bad, T.dbad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  HB_CUDA(cudaStreamSynchronize(st));
  if (bad) {
    ++T.adam_skipped;
    return false;
  }
  T.adam_step += 1;
  const double b1 = 0.9, b2 = 0.999, eps = 1e-8;
  const double bc1 = 1.0 - std::pow(b1, double(T.adam_step)), bc2 = 1.0 - std::pow(b2, double(T.adam_step));
  for (size_t i = 0; i < P.params.size(); ++i) {
    if (!T.trainable[i]) continue;
    const size_t n = P.params[i].size(), o = T.poff[i];
    k_adam<<<egrid(n), TB, 0, st>>>(n, T.dgrad.p + o, T.adam_m.p + o, T.adam_v.p + o, T.dparam.p + o, lr, b1, b2, bc1,
                                    bc2, eps);
  }
  HB_CUDA(cudaGetLastError());
  return true;
}

void snapshot(Context& c) {
  TrainState& T = tstate(c);
  T.snapshot.ensure(T.ptotal);
  HB_CUDA(cudaMemcpyAsync(T.snapshot.p, T.dparam.p, sizeof(float) * T.ptotal, cudaMemcpyDeviceToDevice, c.stream));
}
void restore(Context& c) {
  TrainState& T = tstate(c);
  HB_CUDA(cudaMemcpyAsync(T.dparam.p, T.snapshot.p, sizeof(float) * T.ptotal, cudaMemcpyDeviceToDevice, c.stream));
}

// per-sample relative error (traindet::accumulate_rel_errors)
void acc_rel(const std::vector<float>& out, const float* target, int B, size_t slab, double& sum, size_t& count) {
  for (int b = 0; b < B; ++b) {
    double num = 0, den = 0;
    for (size_t i = 0; i < slab; ++i) {
      const double d = double(out[size_t(b) * slab + i]) - target[size_t(b) * slab + i];
      num += d * d;
      den += double(target[size_t(b) * slab + i]) * target[size_t(b) * slab + i];
    }
    sum += std::sqrt(num) / (std::sqrt(den) + 1e-30);
    ++count;
  }
}

// in-memory dataset (Dataset of TrainingSamples, inc/datagen.hpp:179-183,330-339)
struct DS {
  int H, W;
  const float* r_hat;   // [N][2][H][W]
  const float* e_true;  // [N][2][H][W]
  const int* model;     // [N]
  const double* kappa2; // [M][H][W] (row-major y, x)
  const double* gamma;
};

// traindet::assemble_batch (inc/training.hpp:61-87)
void assemble(const DS& ds, const std::vector<int>& idx, size_t lo, size_t hi, std::vector<float>& in,
              std::vector<float>& tg, std::vector<float>& kp) {
  const int B = int(hi - lo), H = ds.H, W = ds.W;
  const size_t pl = size_t(H) * W;
  in.assign(size_t(B) * 4 * pl, 0.f);
  tg.assign(size_t(B) * 2 * pl, 0.f);
  kp.assign(size_t(B) * pl, 0.f);
  for (int b = 0; b < B; ++b) {
    const int s = idx[lo + size_t(b)];
    const int m = ds.model[s];
    const float* r = ds.r_hat + size_t(s) * 2 * pl;
    const float* e = ds.e_true + size_t(s) * 2 * pl;
    for (size_t q = 0; q < pl; ++q) {
      in[(size_t(b) * 4 + 0) * pl + q] = r[q];
      in[(size_t(b) * 4 + 1) * pl + q] = r[pl + q];
      in[(size_t(b) * 4 + 2) * pl + q] = float(ds.kappa2[size_t(m) * pl + q]);
      in[(size_t(b) * 4 + 3) * pl + q] = float(ds.gamma[size_t(m) * pl + q]);
      tg[(size_t(b) * 2 + 0) * pl + q] = e[q];
      tg[(size_t(b) * 2 + 1) * pl + q] = e[pl + q];
      kp[size_t(b) * pl + q] = float(ds.kappa2[size_t(m) * pl + q]);
    }
  }
}

// schedule_at (inc/training.hpp:22-39)
std::pair<double, int> schedule_at(int epoch, const hb_train_cfg& cfg) {
  int drops = 0;
  double anchor = cfg.t0, gap = cfg.t0 / 2.0;
  while (epoch > anchor) {
    ++drops;
    anchor += std::max(1.0, std::round(gap));
    gap /= 2.0;
  }
  double lr = cfg.lr0;
  long long batch = cfg.batch0;
  for (int i = 0; i < drops; ++i) {
    lr /= 10.0;
    if (batch < (1 << 20)) batch *= 2;
  }
  return {lr, int(batch)};
}

struct Hist {
  double* out;  // [cap][4]: train rel error, val rel error, lr, batch
  int cap, n = 0;
  void push(double tr, double va, double lr, int batch) {
    if (n < cap && out) {
      out[n * 4 + 0] = tr;
      out[n * 4 + 1] = va;
      out[n * 4 + 2] = lr;
      out[n * 4 + 3] = batch;
    }
    ++n;
  }
};

void set_trainable_prefix(Context& c, const std::string& prefix, bool on) {
  PaperState& P = paper_state(c);
  TrainState& T = tstate(c);
  ensure_params(c);
  for (size_t i = 0; i < P.params.size(); ++i)
    if (P.params[i].name.compare(0, prefix.size(), prefix) == 0 && !is_buffer(P.params[i].name))
      T.trainable[i] = on ? 1 : 0;
}

// encoder_forward in eval mode (inc/unet.hpp:276-283) -> frozen features
void freeze_features(Context& c, const std::vector<float>& kappa, int H, int W) {
  TrainState& T = tstate(c);
  PaperState& P = paper_state(c);
  ensure_params(c);
  T.frozen.clear();
  build_tape(c, 1, H, W, 3, false);
  HB_CUDA(cudaMemcpyAsync(V(T, T.t_kappa), kappa.data(), sizeof(float) * kappa.size(), cudaMemcpyHostToDevice,
                          c.stream));
  run_forward(c);
  std::vector<std::vector<float>> f;
  std::vector<std::array<int, 3>> dims;
  for (int t : T.t_feats) {
    const Ten& F = T.tens[size_t(t)];
    std::vector<float> h(F.size());
    HB_CUDA(cudaMemcpyAsync(h.data(), V(T, t), sizeof(float) * F.size(), cudaMemcpyDeviceToHost, c.stream));
    f.push_back(std::move(h));
    dims.push_back({F.c, F.h, F.w});
  }
  HB_CUDA(cudaStreamSynchronize(c.stream));
  T.frozen = std::move(f);
  T.frozen_dims = std::move(dims);
  T.key_B = -1;
  (void)P;
}

// train() (inc/training.hpp:152-227)
int train_loop(Context& c, const hb_train_cfg& cfg, const DS& ds, int N, Hist& hist, int* aborted) {
  TrainState& T = tstate(c);
  ensure_params(c);
  Rng rng(cfg.seed);
  std::vector<int> order(static_cast<size_t>(N));
  std::iota(order.begin(), order.end(), 0);
  for (size_t i = order.size(); i > 1; --i) std::swap(order[i - 1], order[size_t(rng.uniform_int(0, int64_t(i) - 1))]);
  const size_t val_count = size_t(double(order.size()) * cfg.val_fraction);
  std::vector<int> val_idx(order.begin(), order.begin() + long(val_count));
  std::vector<int> train_idx(order.begin() + long(val_count), order.end());
  if (train_idx.empty()) throw HbError{HB_ERR_ARG, "no training samples after split"};
  T.adam_init = false;
  bool have_good = false;
  std::vector<float> in, tg, kp, out;
  const size_t slab = size_t(2) * ds.H * ds.W;
  *aborted = 0;
  for (int epoch = 1; epoch <= cfg.epochs; ++epoch) {
    auto [lr, batch] = schedule_at(epoch, cfg);
    batch = std::min<int>(batch, int(train_idx.size()));
    for (size_t i = train_idx.size(); i > 1; --i)
      std::swap(train_idx[i - 1], train_idx[size_t(rng.uniform_int(0, int64_t(i) - 1))]);
    double rel_sum = 0;
    size_t rel_count = 0;
    bool finite = true;
    for (size_t lo = 0; lo < train_idx.size(); lo += size_t(batch)) {
      const size_t hi = std::min(lo + size_t(batch), train_idx.size());
      assemble(ds, train_idx, lo, hi, in, tg, kp);
      out.resize(size_t(hi - lo) * slab);
      const double loss = run_batch(c, int(hi - lo), ds.H, ds.W, in.data(), kp.data(), tg.data(), true, true, out.data());
      if (!std::isfinite(loss)) {
        finite = false;
        break;
      }
      adam_step(c, lr);
      acc_rel(out, tg.data(), int(hi - lo), slab, rel_sum, rel_count);
    }
    if (!finite) {
      *aborted = 1;
      if (have_good) restore(c);
      break;
    }
    double val_sum = 0;
    size_t val_n = 0;
    for (size_t lo = 0; lo < val_idx.size(); lo += size_t(batch)) {
      const size_t hi = std::min(lo + size_t(batch), val_idx.size());
      assemble(ds, val_idx, lo, hi, in, tg, kp);
      out.resize(size_t(hi - lo) * slab);
      run_batch(c, int(hi - lo), ds.H, ds.W, in.data(), kp.data(), tg.data(), false, false, out.data());
      acc_rel(out, tg.data(), int(hi - lo), slab, val_sum, val_n);
    }
    hist.push(rel_count ? rel_sum / double(rel_count) : 0.0, val_n ? val_sum / double(val_n) : 0.0, lr, batch);
    snapshot(c);
    have_good = true;
  }
  params_to_host(c);
  return hist.n;
}

// retrain() (inc/training.hpp:229-298): n_pairs fresh samples of the context's
// problem (gen_sample_pair seeds seed * 6151 + i, on the device hierarchy),
// lr0 / 10, batch min(20, n), no schedule, no validation; encoder_solver: the
// encoder frozen and evaluated once
int retrain_loop(Context& c, int n_pairs, int epochs, const hb_train_cfg& base, uint64_t seed, Hist& hist,
                 int* aborted) {
  TrainState& T = tstate(c);
  PaperState& P = paper_state(c);
  *aborted = 0;
  if (epochs == 0 || n_pairs == 0) return 0;
  ensure_params(c);
  const int H = c.ny, W = c.nx;
  const size_t pl = size_t(H) * W;
  std::vector<uint64_t> seeds(static_cast<size_t>(n_pairs));
  for (int i = 0; i < n_pairs; ++i) seeds[size_t(i)] = seed * 6151ULL + uint64_t(i);
  std::vector<double> r(size_t(n_pairs) * pl * 2), e(size_t(n_pairs) * pl * 2);
  const int rc = hb_gen_sample_pairs(reinterpret_cast<hb_ctx*>(&c), n_pairs, seeds.data(), -1, 10, r.data(), e.data(), nullptr);
  if (rc != HB_OK) throw HbError{rc, c.err};
  // quantize_sample (inc/datagen.hpp:290-305): r_hat = float(h^2 r), e_true = float(e)
  const double h2 = c.h * c.h;
  std::vector<float> rh(size_t(n_pairs) * 2 * pl), et(size_t(n_pairs) * 2 * pl);
  for (int s = 0; s < n_pairs; ++s)
    for (size_t q = 0; q < pl; ++q) {
      const double* rq = r.data() + (size_t(s) * pl + q) * 2;
      const double* eq = e.data() + (size_t(s) * pl + q) * 2;
      rh[(size_t(s) * 2 + 0) * pl + q] = float(h2 * rq[0]);
      rh[(size_t(s) * 2 + 1) * pl + q] = float(h2 * rq[1]);
      et[(size_t(s) * 2 + 0) * pl + q] = float(eq[0]);
      et[(size_t(s) * 2 + 1) * pl + q] = float(eq[1]);
    }
  std::vector<int> model(static_cast<size_t>(n_pairs), 0);
  DS ds{H, W, rh.data(), et.data(), model.data(), c.k2.data(), c.gam.data()};
  const bool es = base.encoder_solver != 0;
  if (es) {
    std::vector<float> kap(pl);
    for (size_t q = 0; q < pl; ++q) kap[q] = float(c.k2[q]);
    freeze_features(c, kap, H, W);
    set_trainable_prefix(c, "enc.", false);
  }
  Rng rng(seed);
  std::vector<int> idx(static_cast<size_t>(n_pairs));
  std::iota(idx.begin(), idx.end(), 0);
  const double lr = base.lr0 / 10.0;
  const int batch = std::min<int>(20, n_pairs);
  T.adam_init = false;
  snapshot(c);
  std::vector<float> in, tg, kp, out;
  const size_t slab = 2 * pl;
  for (int epoch = 1; epoch <= epochs; ++epoch) {
    for (size_t i = idx.size(); i > 1; --i) std::swap(idx[i - 1], idx[size_t(rng.uniform_int(0, int64_t(i) - 1))]);
    double rel_sum = 0;
    size_t rel_count = 0;
    bool finite = true;
    for (size_t lo = 0; lo < idx.size(); lo += size_t(batch)) {
      const size_t hi = std::min(lo + size_t(batch), idx.size());
      assemble(ds, idx, lo, hi, in, tg, kp);
      out.resize(size_t(hi - lo) * slab);
      const double loss = run_batch(c, int(hi - lo), H, W, in.data(), kp.data(), tg.data(), true, true, out.data());
      if (!std::isfinite(loss)) {
        finite = false;
        break;
      }
      adam_step(c, lr);
      acc_rel(out, tg.data(), int(hi - lo), slab, rel_sum, rel_count);
    }
    if (!finite) {
      *aborted = 1;
      restore(c);
      break;
    }
    hist.push(rel_count ? rel_sum / double(rel_count) : 0.0, 0.0, lr, batch);
    snapshot(c);
  }
  if (es) {
    set_trainable_prefix(c, "enc.", true);
    T.frozen.clear();
    T.key_B = -1;
  }
  params_to_host(c);
  (void)P;
  return hist.n;
}

}  // namespace

}  // namespace hb

// ===================================================================== C ABI
using namespace hb;
struct hb_ctx : hb::Context {};

#define HB_API_BEGIN \
  if (!ctx) return HB_ERR_ARG; \
  try {
#define HB_API_END                  \
  return HB_OK;                     \
  }                                 \
  catch (const HbError& e) {        \
    ctx->err = e.msg;               \
    return e.code;                  \
  }                                 \
  catch (const std::exception& e) { \
    ctx->err = e.what();            \
    return HB_ERR_ARG;              \
  }

extern "C" {

int hb_paper_train_batch(hb_ctx* ctx, int batch, int H, int W, const float* input, const float* kappa,
                         const float* target, int train_mode, int with_grad, int step, double lr, double* loss,
                         float* out) {
  HB_API_BEGIN
  if (batch < 1 || H < 1 || W < 1 || !input || !target) throw HbError{HB_ERR_ARG, "bad batch"};
  if (step && !with_grad) throw HbError{HB_ERR_ARG, "an ADAM step needs gradients"};
  const double l = run_batch(*ctx, batch, H, W, input, kappa, target, train_mode != 0, with_grad != 0, out);
  if (loss) *loss = l;
  if (step) adam_step(*ctx, lr);
  params_to_host(*ctx);
  HB_API_END
}

int64_t hb_paper_trainable_count(hb_ctx* ctx) {
  if (!ctx || !ctx->paper) return 0;
  try {
    ensure_params(*ctx);
  } catch (...) {
    return 0;
  }
  int64_t n = 0;
  for (size_t i = 0; i < ctx->paper->params.size(); ++i)
    if (ctx->train->trainable[i]) n += int64_t(ctx->paper->params[i].size());
  return n;
}

int hb_paper_grads(hb_ctx* ctx, int64_t count, float* grads) {
  HB_API_BEGIN
  ensure_params(*ctx);
  PaperState& P = paper_state(*ctx);
  TrainState& T = tstate(*ctx);
  if (count != hb_paper_trainable_count(ctx) || !grads) throw HbError{HB_ERR_ARG, "gradient count mismatch"};
  std::vector<float> h(T.ptotal);
  HB_CUDA(cudaMemcpyAsync(h.data(), T.dgrad.p, sizeof(float) * T.ptotal, cudaMemcpyDeviceToHost, ctx->stream));
  HB_CUDA(cudaStreamSynchronize(ctx->stream));
  size_t o = 0;
  for (size_t i = 0; i < P.params.size(); ++i)
    if (T.trainable[i]) {
      std::copy(h.begin() + long(T.poff[i]), h.begin() + long(T.poff[i] + P.params[i].size()), grads + o);
      o += P.params[i].size();
    }
  HB_API_END
}

int hb_paper_set_trainable_prefix(hb_ctx* ctx, const char* prefix, int trainable) {
  HB_API_BEGIN
  if (!prefix) throw HbError{HB_ERR_ARG, "null prefix"};
  set_trainable_prefix(*ctx, prefix, trainable != 0);
  HB_API_END
}

int hb_paper_adam_reset(hb_ctx* ctx) {
  HB_API_BEGIN
  tstate(*ctx).adam_init = false;
  HB_API_END
}

int hb_paper_train(hb_ctx* ctx, const hb_train_cfg* cfg, int count, int H, int W, const float* r_hat,
                   const float* e_true, const int* model_id, int models, const double* kappa2, const double* gamma,
                   double* hist, int hist_cap, int* epochs_run, int* aborted) {
  HB_API_BEGIN
  if (!cfg || count < 1 || !r_hat || !e_true || !model_id || models < 1 || !kappa2 || !gamma)
    throw HbError{HB_ERR_ARG, "bad dataset"};
  for (int s = 0; s < count; ++s)
    if (model_id[s] < 0 || model_id[s] >= models) throw HbError{HB_ERR_ARG, "model id out of range"};
  PaperState& P = paper_state(*ctx);
  if ((cfg->encoder_solver != 0) != (P.variant == 1)) throw HbError{HB_ERR_ARG, "encoder_solver does not match the net"};
  tstate(*ctx).frozen.clear();
  DS ds{H, W, r_hat, e_true, model_id, kappa2, gamma};
  Hist h{hist, hist_cap};
  int ab = 0;
  train_loop(*ctx, *cfg, ds, count, h, &ab);
  if (epochs_run) *epochs_run = h.n;
  if (aborted) *aborted = ab;
  HB_API_END
}

int hb_paper_retrain(hb_ctx* ctx, int n_pairs, int epochs, const hb_train_cfg* base, uint64_t seed, double* hist,
                     int hist_cap, int* epochs_run, int* aborted) {
  HB_API_BEGIN
  if (!base || n_pairs < 0 || epochs < 0) throw HbError{HB_ERR_ARG, "bad retrain arguments"};
  if (!ctx->has_hier) throw HbError{HB_ERR_STATE, "hierarchy not built (hb_build_hierarchy)"};
  PaperState& P = paper_state(*ctx);
  if ((base->encoder_solver != 0) != (P.variant == 1)) throw HbError{HB_ERR_ARG, "encoder_solver does not match the net"};
  Hist h{hist, hist_cap};
  int ab = 0;
  retrain_loop(*ctx, n_pairs, epochs, *base, seed, h, &ab);
  if (epochs_run) *epochs_run = h.n;
  if (aborted) *aborted = ab;
  HB_API_END
}

}  // extern "C"
