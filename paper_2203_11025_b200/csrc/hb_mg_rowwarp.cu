// Full-row V-cycle legs for the narrow grids of many-column batches (c0's
// 128^2 and 64^2 levels): one warp owns a WHOLE row, NPL = nx / 32 adjacent
// fine columns per lane (NPL = 4 at 128^2, 2 at 64^2), and marches down a
// chunk of rows with the 3-row stencil window in registers.
//
// Same math as the strip legs (hb_mg_stream.cu / hb_mg_staged.cu; inc/
// multigrid.hpp:108-119 with inc/stencil.hpp:44-165, zero initial guess,
// nu1 = nu2 = 1):
//   down:  v = w D^-1 f ;  r = f - M v ;  fc = R_o r
//   up:    v = w D^-1 f + P_o vc ;  z = v + w D^-1 (f - M v)
// The strip legs give each warp 30 coarse columns plus two halo lanes, so a
// 128-wide row takes three warps with 26 of 96 lanes idle or redundant and a
// 64-wide row two warps with half the lanes idle; here the grid boundary is
// the row boundary (zero padding), every lane emits, and the per-row
// bookkeeping (address math, masks, prefetch) is shared by NPL nodes instead
// of 2.  Fine rows are prefetched two rows ahead in registers (float4 loads,
// two nodes each); horizontal neighbours across lanes come from shuffles
// (lane 0 / 31 see the zero padding).
#include "hb_common.cuh"
#include "hb_internal.h"

namespace hb {

namespace {

constexpr int RW_WARPS = 4;  // warps per CTA (independent row chunks)
#ifndef HB_ROW_MINB
#define HB_ROW_MINB 1
#endif

__device__ __forceinline__ float2 wfrom_d(float2 d, float damping) {  // damping / d (fast reciprocal)
  const float m = fmaf(d.x, d.x, d.y * d.y);
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(m));
  const float s = m > 0.f ? r * damping : 0.f;
  return make_float2(d.x * s, -d.y * s);
}
// neighbour values across lanes, zero beyond the row ends
__device__ __forceinline__ float2 from_left(float2 v, int lane) {
  const float2 u = make_float2(__shfl_up_sync(0xffffffffu, v.x, 1), __shfl_up_sync(0xffffffffu, v.y, 1));
  return lane == 0 ? make_float2(0.f, 0.f) : u;
}
__device__ __forceinline__ float2 from_right(float2 v, int lane) {
  const float2 u = make_float2(__shfl_down_sync(0xffffffffu, v.x, 1), __shfl_down_sync(0xffffffffu, v.y, 1));
  return lane == 31 ? make_float2(0.f, 0.f) : u;
}

template <int NPL>
struct FRow {  // one fine row at this lane's NPL columns (f scaled and zero outside the grid)
  float2 f[NPL], d[NPL];
  float m;  // 1 inside the grid, 0 for the padding rows
};

template <int NPL>
__device__ __forceinline__ void load_frow(const float2* fb, const float2* dM, int nx, int ny, int y, int lane, float s,
                                          FRow<NPL>& r) {
  const bool ok = y >= 0 && y < ny;
  const int o = (ok ? y : 0) * nx + NPL * lane;
  r.m = ok ? 1.f : 0.f;
  const float sm = ok ? s : 0.f;
#pragma unroll
  for (int k = 0; k < NPL; k += 2) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(fb + o + k));
    const float4 dd = __ldg(reinterpret_cast<const float4*>(dM + o + k));
    r.f[k] = make_float2(a.x * sm, a.y * sm);
    r.f[k + 1] = make_float2(a.z * sm, a.w * sm);
    r.d[k] = make_float2(dd.x, dd.y);
    r.d[k + 1] = make_float2(dd.z, dd.w);
  }
}

// r = f - M v at one row (v rows above / here / below), masked to the grid
template <int NPL>
__device__ __forceinline__ void residual_row(const FRow<NPL>& u, const float2 (&vm)[NPL], const float2 (&vc)[NPL],
                                             const float2 (&vp)[NPL], float ih2, int lane, float2 (&r)[NPL]) {
  const float2 left = from_left(vc[NPL - 1], lane), right = from_right(vc[0], lane);
#pragma unroll
  for (int k = 0; k < NPL; ++k) {
    const float2 l = k > 0 ? vc[k - 1] : left, rt = k + 1 < NPL ? vc[k + 1] : right;
    const float2 nb = cadd(cadd(vm[k], vp[k]), cadd(l, rt));
    float2 mv = cmul(u.d[k], vc[k]);
    mv.x = fmaf(-ih2, nb.x, mv.x);
    mv.y = fmaf(-ih2, nb.y, mv.y);
    r[k] = cscale(csub(u.f[k], mv), u.m);
  }
}

// down leg: grid (ceil(coarse row chunks / RW_WARPS), B), block 32 x RW_WARPS;
// warp = coarse rows [jy0, jy0 + rpc) of one column, all cnx = 16 NPL coarse columns
template <int NPL, int O>
__global__ void __launch_bounds__(32 * RW_WARPS, HB_ROW_MINB) k_down_row(LevelView L, float damping, int rpc,
                                                            const int* act, const float2* __restrict__ f,
                                                            const float* fscale, float2* __restrict__ fc) {
  constexpr int NC = NPL / 2;  // coarse columns per lane
  constexpr int offset = O;    // restriction / prolongation offset = level % 2
  pdl_enter();
  const int b = blockIdx.y;
  if (act && !act[b]) return;
  const int lane = threadIdx.x, nx = L.nx, ny = L.ny, cnx = nx / 2, cny = ny / 2;
  const int jy0 = (blockIdx.x * RW_WARPS + threadIdx.y) * rpc;
  if (jy0 >= cny) return;
  const int jy1 = min(cny, jy0 + rpc);
  const float2* fb = f + size_t(b) * nx * ny;
  const float s = fscale ? fscale[b] : 1.0f;
  const float ih2 = L.inv_h2;
  const int yb = 2 * jy0 + offset - 1;          // first residual row
  const int yend = 2 * (jy1 - 1) + offset + 1;  // last residual row
  FRow<NPL> rc, rp1;
  float2 vm[NPL], vc[NPL];
  load_frow<NPL>(fb, L.dM, nx, ny, yb - 1, lane, s, rc);
#pragma unroll
  for (int k = 0; k < NPL; ++k) vm[k] = cmul(rc.f[k], wfrom_d(rc.d[k], damping));
  load_frow<NPL>(fb, L.dM, nx, ny, yb, lane, s, rc);
  load_frow<NPL>(fb, L.dM, nx, ny, yb + 1, lane, s, rp1);
#pragma unroll
  for (int k = 0; k < NPL; ++k) vc[k] = cmul(rc.f[k], wfrom_d(rc.d[k], damping));
  float2 hm2[NC], hm1[NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) hm2[i] = hm1[i] = make_float2(0.f, 0.f);
  float2* fcb = fc + size_t(b) * cnx * cny;
  for (int y = yb; y <= yend; ++y) {
    FRow<NPL> rp2;
    load_frow<NPL>(fb, L.dM, nx, ny, y + 2, lane, s, rp2);  // in flight during this row
    float2 vp[NPL], r[NPL];
#pragma unroll
    for (int k = 0; k < NPL; ++k) vp[k] = cmul(rp1.f[k], wfrom_d(rp1.d[k], damping));
    residual_row<NPL>(rc, vm, vc, vp, ih2, lane, r);
    // horizontal full weighting at the centres 2j + o: (r(c-1) + 2 r(c) + r(c+1)) / 4
    float2 h[NC];
    if constexpr (O == 0) {
      const float2 rl = from_left(r[NPL - 1], lane);
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        const int k = 2 * i;
        h[i] = caxpy(cscale(r[k], 0.5f), 0.25f, cadd(k > 0 ? r[k - 1] : rl, r[k + 1]));
      }
    } else {
      const float2 rr = from_right(r[0], lane);
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        const int k = 2 * i + 1;
        h[i] = caxpy(cscale(r[k], 0.5f), 0.25f, cadd(r[k - 1], k + 1 < NPL ? r[k + 1] : rr));
      }
    }
    const int t = y - offset - 1;  // y = 2 jy + o + 1 closes coarse row jy
    if (t >= 2 * jy0 && (t & 1) == 0) {
      float2 o[NC];
#pragma unroll
      for (int i = 0; i < NC; ++i) o[i] = caxpy(cscale(hm1[i], 0.5f), 0.25f, cadd(hm2[i], h[i]));
      float2* dst = fcb + size_t(t >> 1) * cnx + NC * lane;
      if constexpr (NC == 2)
        *reinterpret_cast<float4*>(dst) = make_float4(o[0].x, o[0].y, o[1].x, o[1].y);
      else
        *dst = o[0];
    }
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      hm2[i] = hm1[i];
      hm1[i] = h[i];
    }
#pragma unroll
    for (int k = 0; k < NPL; ++k) {
      vm[k] = vc[k];
      vc[k] = vp[k];
    }
    rc = rp1;
    rp1 = rp2;
  }
}

template <int NPL>
struct URow {  // one fine row for the up leg: f, D and the vertically interpolated coarse correction
  FRow<NPL> u;
  float2 q[NPL / 2];  // at this lane's coarse columns NC lane .. NC lane + NC - 1
};

template <int NPL>
__device__ __forceinline__ void load_urow(const float2* fb, const float2* dM, const float2* cb, int nx, int ny,
                                          int cnx, int cny, int offset, int y, int lane, float s, URow<NPL>& r) {
  constexpr int NC = NPL / 2;
  load_frow<NPL>(fb, dM, nx, ny, y, lane, s, r.u);
  // vertical prolongation: t = y - o even -> coarse row t/2; odd -> mean of rows (t-1)/2, (t+1)/2
  const int t = y - offset;
  const int ja = t >> 1, jb = (t & 1) ? ja + 1 : ja;
  float wa = (t & 1) ? 0.5f : 1.f, wb = (t & 1) ? 0.5f : 0.f;
  if (ja < 0 || ja >= cny) wa = 0.f;
  if (jb < 0 || jb >= cny) wb = 0.f;
  wa *= r.u.m;  // padding rows carry no correction (v = 0 there)
  wb *= r.u.m;
  const float2* pa = cb + size_t(min(max(ja, 0), cny - 1)) * cnx + NC * lane;
  const float2* pb = cb + size_t(min(max(jb, 0), cny - 1)) * cnx + NC * lane;
  if constexpr (NC == 2) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(pa)), c = __ldg(reinterpret_cast<const float4*>(pb));
    r.q[0] = make_float2(wa * a.x + wb * c.x, wa * a.y + wb * c.y);
    r.q[1] = make_float2(wa * a.z + wb * c.z, wa * a.w + wb * c.w);
  } else {
    const float2 a = __ldg(pa), c = __ldg(pb);
    r.q[0] = make_float2(wa * a.x + wb * c.x, wa * a.y + wb * c.y);
  }
}

// v = w D^-1 f + P_o vc at one row (horizontal prolongation of the row's q)
template <int NPL, int O>
__device__ __forceinline__ void up_v(const URow<NPL>& r, float damping, int lane, float2 (&v)[NPL]) {
  constexpr int NC = NPL / 2;
  const float2 qprev = from_left(r.q[NC - 1], lane), qnext = from_right(r.q[0], lane);
#pragma unroll
  for (int k = 0; k < NPL; ++k) {
    // fine column NPL lane + k: t = k - o (relative to coarse column NC lane, doubled)
    const int t = k - O;  // compile time: no dynamic register-array indexing
    float2 p;
    if ((t & 1) == 0) {
      p = r.q[t >> 1];
    } else {
      const int ia = (t - 1) >> 1, ib = (t + 1) >> 1;
      const float2 a = ia < 0 ? qprev : r.q[ia], c = ib >= NC ? qnext : r.q[ib];
      p = cscale(cadd(a, c), 0.5f);
    }
    v[k] = cadd(cmul(r.u.f[k], wfrom_d(r.u.d[k], damping)), p);
  }
}

// up leg: grid (ceil(fine row chunks / RW_WARPS), B); warp = fine rows [y0, y0 + rpc) of one column
template <int NPL, int O>
__global__ void __launch_bounds__(32 * RW_WARPS, HB_ROW_MINB) k_up_row(LevelView L, float damping, int rpc,
                                                          const int* act, const float2* __restrict__ f,
                                                          const float* fscale, const float2* __restrict__ vcoarse,
                                                          float2* __restrict__ z) {
  constexpr int offset = O;
  pdl_enter();
  const int b = blockIdx.y;
  if (act && !act[b]) return;
  const int lane = threadIdx.x, nx = L.nx, ny = L.ny, cnx = nx / 2, cny = ny / 2;
  const int y0 = (blockIdx.x * RW_WARPS + threadIdx.y) * rpc;
  if (y0 >= ny) return;
  const int y1 = min(ny, y0 + rpc);
  const float2* fb = f + size_t(b) * nx * ny;
  const float2* cb = vcoarse + size_t(b) * cnx * cny;
  const float s = fscale ? fscale[b] : 1.0f;
  const float ih2 = L.inv_h2;
  URow<NPL> rc, rp1;
  float2 vm[NPL], vc[NPL];
  load_urow<NPL>(fb, L.dM, cb, nx, ny, cnx, cny, offset, y0 - 1, lane, s, rc);
  up_v<NPL, O>(rc, damping, lane, vm);
  load_urow<NPL>(fb, L.dM, cb, nx, ny, cnx, cny, offset, y0, lane, s, rc);
  load_urow<NPL>(fb, L.dM, cb, nx, ny, cnx, cny, offset, y0 + 1, lane, s, rp1);
  up_v<NPL, O>(rc, damping, lane, vc);
  float2* zb = z + size_t(b) * nx * ny;
  for (int y = y0; y < y1; ++y) {
    URow<NPL> rp2;
    load_urow<NPL>(fb, L.dM, cb, nx, ny, cnx, cny, offset, y + 2, lane, s, rp2);
    float2 vp[NPL], r[NPL];
    up_v<NPL, O>(rp1, damping, lane, vp);
    residual_row<NPL>(rc.u, vm, vc, vp, ih2, lane, r);  // f - M v (this row is inside the grid)
    float2 o[NPL];
#pragma unroll
    for (int k = 0; k < NPL; ++k) o[k] = cadd(vc[k], cmul(r[k], wfrom_d(rc.u.d[k], damping)));
    float2* dst = zb + size_t(y) * nx + NPL * lane;
#pragma unroll
    for (int k = 0; k < NPL; k += 2)
      *reinterpret_cast<float4*>(dst + k) = make_float4(o[k].x, o[k].y, o[k + 1].x, o[k + 1].y);
#pragma unroll
    for (int k = 0; k < NPL; ++k) {
      vm[k] = vc[k];
      vc[k] = vp[k];
    }
    rc = rp1;
    rp1 = rp2;
  }
}

bool row_legs_fit(const Context& c, const LevelView& L) {
  return c.opt_row_legs && (L.nx == 64 || L.nx == 128) && L.ny % 2 == 0 && L.w.row0 == 0 && L.w.rows == L.ny &&
         L.w.lo == 0 && L.w.hi == L.ny;
}

// rows per warp: halve from `start` while the launch would have fewer than 2 warps per SM slot
int row_rpc(const Context& c, int rows, int B, int start, int min_rpc) {
  int rpc = start;
  while (rpc > min_rpc && size_t((rows + rpc - 1) / rpc) * B < size_t(2) * c.num_sms * RW_WARPS) rpc /= 2;
  return rpc;
}

}  // namespace

bool launch_down_row(Context& c, const LevelView& L, float damping, int offset, int B, const int* act,
                     const float2* f, const float* fscale, float2* fc) {
  if (!row_legs_fit(c, L)) return false;
  const int cny = L.ny / 2;
  const int rpc = row_rpc(c, cny, B, 8, 4);
  const dim3 grid(((cny + rpc - 1) / rpc + RW_WARPS - 1) / RW_WARPS, B);
  auto k = L.nx == 128 ? (offset ? k_down_row<4, 1> : k_down_row<4, 0>) : (offset ? k_down_row<2, 1> : k_down_row<2, 0>);
  launch_pdl(c, k, grid, dim3(32, RW_WARPS), 0, L, damping, rpc, act, f, fscale, fc);
  HB_CUDA(cudaGetLastError());
  return true;
}

bool launch_up_row(Context& c, const LevelView& L, float damping, int offset, int B, const int* act, const float2* f,
                   const float* fscale, const float2* vc, float2* z) {
  if (!row_legs_fit(c, L)) return false;
  const int rpc = row_rpc(c, L.ny, B, 16, 8);
  const dim3 grid(((L.ny + rpc - 1) / rpc + RW_WARPS - 1) / RW_WARPS, B);
  auto k = L.nx == 128 ? (offset ? k_up_row<4, 1> : k_up_row<4, 0>) : (offset ? k_up_row<2, 1> : k_up_row<2, 0>);
  launch_pdl(c, k, grid, dim3(32, RW_WARPS), 0, L, damping, rpc, act, f, fscale, vc, z);
  HB_CUDA(cudaGetLastError());
  return true;
}

}  // namespace hb
