// Fused V-cycle legs for nu1 = nu2 = 1 (the configuration of every BASELINE
// config; other (nu1, nu2) use the unfused kernels in hb_mg.cu).
//
// down leg, level l (inc/multigrid.hpp:110-112 + inc/stencil.hpp:69-92,119-140):
//     v  = e0 + w D^-1 (f - M e0)      (or w D^-1 f from a zero iterate)
//     fc = R_o (f - M v)
//   one CTA per coarse tile: f, D (and e0) staged in shared memory with a 2-
//   (3-) node fine halo; v and r never touch HBM.  Traffic per fine node:
//   read f + D (+ e0) = 16 (24) B, write fc = 2 B.
// up leg, level l (inc/multigrid.hpp:116-118 + inc/stencil.hpp:146-165):
//     v  = v_pre + P_o vc   (v_pre recomputed from f, D, e0 as in the down leg)
//     z  = v + w D^-1 (f - M v)
//   one CTA per fine tile with a 1- (2-) node halo; traffic per fine node:
//   read f + D (+ e0) + vc/4 = 18 (26) B, write z = 8 B.
#include "hb_common.cuh"
#include "hb_internal.h"

namespace hb {

namespace {

__device__ __forceinline__ bool in_dom(int x, int y, int nx, int ny) { return x >= 0 && x < nx && y >= 0 && y < ny; }

template <int CX, int CY, bool E0>
__global__ void __launch_bounds__(CX* CY) k_down_fused(LevelView L, float damping, int offset, const int* act,
                                                      const float2* __restrict__ f, const float* fscale,
                                                      const float2* __restrict__ e0, float2* __restrict__ fc) {
  constexpr int RW = 2 * CX + 1, RH = 2 * CY + 1;  // residual region
  constexpr int VW = RW + 2, VH = RH + 2;          // smoothed-iterate region
  constexpr int EW = VW + 2, EH = VH + 2;          // initial-guess region
  constexpr int NT = CX * CY;
  const int b = blockIdx.z;
  if (act && !act[b]) return;
  __shared__ float2 sf[VH][VW], sd[VH][VW], sw[VH][VW], sv[VH][VW];
  __shared__ float2 se_r[(EW * EH > RW * RH) ? EW * EH : RW * RH];  // e0 tile, then residual tile
  const int nx = L.nx, ny = L.ny;
  const size_t N = size_t(nx) * ny;
  const int cx0 = blockIdx.x * CX, cy0 = blockIdx.y * CY;
  const int xr0 = 2 * cx0 + offset - 1, yr0 = 2 * cy0 + offset - 1;
  const int xv0 = xr0 - 1, yv0 = yr0 - 1;
  const float2* fb = f + b * N;
  const float s = fscale ? fscale[b] : 1.0f;
  const int t = threadIdx.y * CX + threadIdx.x;
  for (int i = t; i < VW * VH; i += NT) {
    const int ly = i / VW, lx = i % VW;
    const int gx = xv0 + lx, gy = yv0 + ly;
    float2 fv = make_float2(0.f, 0.f), dv = make_float2(1.f, 0.f), wv = make_float2(0.f, 0.f);
    if (in_dom(gx, gy, nx, ny)) {
      const size_t g = size_t(gy) * nx + gx;
      fv = cscale(ld(fb, g), s);
      dv = ld(L.dM, g);
      wv = ld(L.wdi, g);
    }
    sf[ly][lx] = fv;
    sd[ly][lx] = dv;
    sw[ly][lx] = wv;
  }
  if (E0) {
    const float2* eb = e0 + b * N;
    for (int i = t; i < EW * EH; i += NT) {
      const int ly = i / EW, lx = i % EW;
      const int gx = xv0 - 1 + lx, gy = yv0 - 1 + ly;
      se_r[i] = in_dom(gx, gy, nx, ny) ? ld(eb, size_t(gy) * nx + gx) : make_float2(0.f, 0.f);
    }
  }
  __syncthreads();
  const float ih2 = L.inv_h2;
  for (int i = t; i < VW * VH; i += NT) {
    const int ly = i / VW, lx = i % VW;
    float2 v = make_float2(0.f, 0.f);
    if (in_dom(xv0 + lx, yv0 + ly, nx, ny)) {
      const float2 d = sd[ly][lx];
      if (E0) {
        const int ex = lx + 1, ey = ly + 1;
        const float2 c = se_r[ey * EW + ex];
        float2 nb = cadd(cadd(se_r[ey * EW + ex - 1], se_r[ey * EW + ex + 1]),
                         cadd(se_r[(ey - 1) * EW + ex], se_r[(ey + 1) * EW + ex]));
        float2 me = cmul(d, c);
        me.x = fmaf(-ih2, nb.x, me.x);
        me.y = fmaf(-ih2, nb.y, me.y);
        v = cadd(c, cmul(csub(sf[ly][lx], me), sw[ly][lx]));
      } else {
        v = cmul(sf[ly][lx], sw[ly][lx]);
      }
    }
    sv[ly][lx] = v;
  }
  __syncthreads();
  for (int i = t; i < RW * RH; i += NT) {
    const int ly = i / RW, lx = i % RW;
    float2 r = make_float2(0.f, 0.f);
    if (in_dom(xr0 + lx, yr0 + ly, nx, ny)) {
      const int vx = lx + 1, vy = ly + 1;
      const float2 nb = cadd(cadd(sv[vy][vx - 1], sv[vy][vx + 1]), cadd(sv[vy - 1][vx], sv[vy + 1][vx]));
      float2 mv = cmul(sd[vy][vx], sv[vy][vx]);
      mv.x = fmaf(-ih2, nb.x, mv.x);
      mv.y = fmaf(-ih2, nb.y, mv.y);
      r = csub(sf[vy][vx], mv);
    }
    se_r[i] = r;
  }
  __syncthreads();
  const int cnx = nx / 2, cny = ny / 2;
  const int jx = cx0 + threadIdx.x, jy = cy0 + threadIdx.y;
  if (jx >= cnx || jy >= cny) return;
  const int lx = 2 * threadIdx.x + 1, ly = 2 * threadIdx.y + 1;  // centre 2j+o in residual coordinates
  float2 acc = cscale(se_r[ly * RW + lx], 0.25f);
  acc = caxpy(acc, 0.125f, cadd(cadd(se_r[ly * RW + lx - 1], se_r[ly * RW + lx + 1]),
                                cadd(se_r[(ly - 1) * RW + lx], se_r[(ly + 1) * RW + lx])));
  acc = caxpy(acc, 0.0625f, cadd(cadd(se_r[(ly - 1) * RW + lx - 1], se_r[(ly - 1) * RW + lx + 1]),
                                 cadd(se_r[(ly + 1) * RW + lx - 1], se_r[(ly + 1) * RW + lx + 1])));
  fc[size_t(b) * cnx * cny + size_t(jy) * cnx + jx] = acc;
}

// floor division for possibly negative numerators
__device__ __forceinline__ int fdiv2(int a) { return a >= 0 ? a / 2 : -((-a + 1) / 2); }

template <int TX, int TY, bool E0>
__global__ void __launch_bounds__(TX* TY) k_up_fused(LevelView L, float damping, int offset, int cnx, int cny,
                                                    const int* act, const float2* __restrict__ f, const float* fscale,
                                                    const float2* __restrict__ e0, const float2* __restrict__ vc,
                                                    float2* __restrict__ z) {
  constexpr int VW = TX + 2, VH = TY + 2;
  constexpr int EW = VW + 2, EH = VH + 2;
  constexpr int CW = TX / 2 + 3, CH = TY / 2 + 3;
  constexpr int NT = TX * TY;
  const int b = blockIdx.z;
  if (act && !act[b]) return;
  __shared__ float2 sf[VH][VW], sd[VH][VW], sw[VH][VW], sv[VH][VW];
  __shared__ float2 se[E0 ? EH : 1][E0 ? EW : 1];
  __shared__ float2 sc[CH][CW];
  const int nx = L.nx, ny = L.ny;
  const size_t N = size_t(nx) * ny;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int xv0 = x0 - 1, yv0 = y0 - 1;
  const int jx0 = fdiv2(xv0 - offset - 1), jy0 = fdiv2(yv0 - offset - 1);
  const float2* fb = f + b * N;
  const float s = fscale ? fscale[b] : 1.0f;
  const int t = threadIdx.y * TX + threadIdx.x;
  for (int i = t; i < VW * VH; i += NT) {
    const int ly = i / VW, lx = i % VW;
    const int gx = xv0 + lx, gy = yv0 + ly;
    float2 fv = make_float2(0.f, 0.f), dv = make_float2(1.f, 0.f), wv = make_float2(0.f, 0.f);
    if (in_dom(gx, gy, nx, ny)) {
      const size_t g = size_t(gy) * nx + gx;
      fv = cscale(ld(fb, g), s);
      dv = ld(L.dM, g);
      wv = ld(L.wdi, g);
    }
    sf[ly][lx] = fv;
    sd[ly][lx] = dv;
    sw[ly][lx] = wv;
  }
  if (E0) {
    const float2* eb = e0 + b * N;
    for (int i = t; i < EW * EH; i += NT) {
      const int ly = i / EW, lx = i % EW;
      const int gx = xv0 - 1 + lx, gy = yv0 - 1 + ly;
      se[ly][lx] = in_dom(gx, gy, nx, ny) ? ld(eb, size_t(gy) * nx + gx) : make_float2(0.f, 0.f);
    }
  }
  const float2* cb = vc + size_t(b) * cnx * cny;
  for (int i = t; i < CW * CH; i += NT) {
    const int ly = i / CW, lx = i % CW;
    const int gx = jx0 + lx, gy = jy0 + ly;
    sc[ly][lx] = in_dom(gx, gy, cnx, cny) ? ld(cb, size_t(gy) * cnx + gx) : make_float2(0.f, 0.f);
  }
  __syncthreads();
  const float ih2 = L.inv_h2;
  for (int i = t; i < VW * VH; i += NT) {
    const int ly = i / VW, lx = i % VW;
    const int gx = xv0 + lx, gy = yv0 + ly;
    float2 v = make_float2(0.f, 0.f);
    if (in_dom(gx, gy, nx, ny)) {
      const float2 d = sd[ly][lx];
      if (E0) {
        const int ex = lx + 1, ey = ly + 1;
        const float2 c = se[ey][ex];
        const float2 nb = cadd(cadd(se[ey][ex - 1], se[ey][ex + 1]), cadd(se[ey - 1][ex], se[ey + 1][ex]));
        float2 me = cmul(d, c);
        me.x = fmaf(-ih2, nb.x, me.x);
        me.y = fmaf(-ih2, nb.y, me.y);
        v = cadd(c, cmul(csub(sf[ly][lx], me), sw[ly][lx]));
      } else {
        v = cmul(sf[ly][lx], sw[ly][lx]);
      }
      // + P_o vc: per axis, (g - o) even -> j = (g-o)/2 weight 1; odd -> j = (g-o+-1)/2 weight 1/2
      const int tx = gx - offset, ty = gy - offset;
      const int ax = fdiv2(tx) - jx0, ay = fdiv2(ty) - jy0;
      float2 p;
      if ((tx & 1) == 0) {
        if ((ty & 1) == 0)
          p = sc[ay][ax];
        else
          p = cscale(cadd(sc[ay][ax], sc[ay + 1][ax]), 0.5f);
      } else {
        if ((ty & 1) == 0)
          p = cscale(cadd(sc[ay][ax], sc[ay][ax + 1]), 0.5f);
        else
          p = cscale(cadd(cadd(sc[ay][ax], sc[ay][ax + 1]), cadd(sc[ay + 1][ax], sc[ay + 1][ax + 1])), 0.25f);
      }
      v = cadd(v, p);
    }
    sv[ly][lx] = v;
  }
  __syncthreads();
  float2* zb = z + b * N;
  for (int i = t; i < TX * TY; i += NT) {
    const int ly = i / TX + 1, lx = i % TX + 1;
    const int gx = xv0 + lx, gy = yv0 + ly;
    if (gx >= nx || gy >= ny) continue;
    const float2 d = sd[ly][lx];
    const float2 nb = cadd(cadd(sv[ly][lx - 1], sv[ly][lx + 1]), cadd(sv[ly - 1][lx], sv[ly + 1][lx]));
    float2 mv = cmul(d, sv[ly][lx]);
    mv.x = fmaf(-ih2, nb.x, mv.x);
    mv.y = fmaf(-ih2, nb.y, mv.y);
    zb[size_t(gy) * nx + gx] = cadd(sv[ly][lx], cmul(csub(sf[ly][lx], mv), sw[ly][lx]));
  }
}

}  // namespace

struct FScope {
  Context& c;
  int cls, tok;
  double bytes;
  FScope(Context& c_, int cls_, double bytes_) : c(c_), cls(cls_), tok(prof_begin(c_, cls_)), bytes(bytes_) {}
  ~FScope() { prof_end(c, cls, tok, bytes, 0); }
};

void launch_down_fused(Context& c, const LevelView& L, float damping, int offset, int B, const int* act,
                       const float2* f, const float* fscale, const float2* e0, float2* fc) {
  const int cnx = L.nx / 2, cny = L.ny / 2;
  FScope fs(c, PC_DOWN, double(B) * L.nx * L.ny * ((e0 ? 16.0 : 8.0) + 2.0) + double(L.nx) * L.ny * 16.0);  // f (+e0) in, fc out; D, wD^-1
  const size_t big = size_t(cnx) * cny * B;
  if (big >= size_t(2) * 148 * 256) {
    const dim3 grid((cnx + 31) / 32, (cny + 3) / 4, B);
    if (e0)
      k_down_fused<32, 4, true><<<grid, dim3(32, 4), 0, c.stream>>>(L, damping, offset, act, f, fscale, e0, fc);
    else
      k_down_fused<32, 4, false><<<grid, dim3(32, 4), 0, c.stream>>>(L, damping, offset, act, f, fscale, e0, fc);
  } else {
    const dim3 grid((cnx + 15) / 16, (cny + 7) / 8, B);
    if (e0)
      k_down_fused<16, 8, true><<<grid, dim3(16, 8), 0, c.stream>>>(L, damping, offset, act, f, fscale, e0, fc);
    else
      k_down_fused<16, 8, false><<<grid, dim3(16, 8), 0, c.stream>>>(L, damping, offset, act, f, fscale, e0, fc);
  }
  HB_CUDA(cudaGetLastError());
}

void launch_up_fused(Context& c, const LevelView& L, float damping, int offset, int cnx, int cny, int B,
                     const int* act, const float2* f, const float* fscale, const float2* e0, const float2* vc,
                     float2* z) {
  FScope fs(c, PC_UP, double(B) * L.nx * L.ny * ((e0 ? 16.0 : 8.0) + 2.0 + 8.0) + double(L.nx) * L.ny * 16.0);  // f (+e0), vc in; z out; D, wD^-1
  const size_t big = size_t(L.nx) * L.ny * B;
  if (big >= size_t(2) * 148 * 512) {
    const dim3 grid((L.nx + 63) / 64, (L.ny + 7) / 8, B);
    if (e0)
      k_up_fused<64, 8, true><<<grid, dim3(64, 8), 0, c.stream>>>(L, damping, offset, cnx, cny, act, f, fscale, e0,
                                                                   vc, z);
    else
      k_up_fused<64, 8, false><<<grid, dim3(64, 8), 0, c.stream>>>(L, damping, offset, cnx, cny, act, f, fscale, e0,
                                                                    vc, z);
  } else {
    const dim3 grid((L.nx + 31) / 32, (L.ny + 7) / 8, B);
    if (e0)
      k_up_fused<32, 8, true><<<grid, dim3(32, 8), 0, c.stream>>>(L, damping, offset, cnx, cny, act, f, fscale, e0,
                                                                   vc, z);
    else
      k_up_fused<32, 8, false><<<grid, dim3(32, 8), 0, c.stream>>>(L, damping, offset, cnx, cny, act, f, fscale, e0,
                                                                    vc, z);
  }
  HB_CUDA(cudaGetLastError());
}

}  // namespace hb
