// Row-streaming V-cycle legs (zero initial guess, nu1 = nu2 = 1): the M_V /
// coarse-net path of every FGMRES inner step.  Same math as hb_mg_fused.cu
// (inc/multigrid.hpp:108-119 with inc/stencil.hpp:44-165) but organised for
// bandwidth: a warp owns a strip of 32 coarse columns (= 64 fine columns, each
// lane two adjacent fine columns 2jx+o, 2jx+o+1) and marches down a chunk of
// rows keeping the 3-row stencil window in registers; horizontal neighbours
// come from warp shuffles, so there is no shared memory and no CTA barrier.
// Lanes 0 and 31 are halo lanes (their neighbours live in other warps); each
// warp emits 30 coarse columns.  Loads are float4 (two fine nodes per lane).
//
//   down:  v = wD^-1 f ; r = f - M v ; fc(jy, jx) = sum_k W_k r(2j+o+k)
//   up:    v = wD^-1 f + P_o vc ; z = v + wD^-1 (f - M v)
#include <cstdlib>

#include "hb_common.cuh"
#include "hb_internal.h"

namespace hb {

namespace {

// row chunks per launch: halve the rows per warp while fewer than rpc_fill() x SMs x warps-per-CTA
// warps would run (HB_RPC_FILL overrides; experiments)
inline int rpc_fill() {
  static const int v = getenv("HB_RPC_FILL") ? atoi(getenv("HB_RPC_FILL")) : 2;
  return v;
}

constexpr int SW_OUT = 30;  // coarse columns emitted per warp
constexpr int WARPS = 4;    // warps per CTA (independent row chunks)

// damping / d (0 for the zero padding outside the grid), fast reciprocal
__device__ __forceinline__ float2 wfrom(float2 d, float damping) {
  const float m = fmaf(d.x, d.x, d.y * d.y);
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(m));  // 1 ulp; one MUFU op instead of the IEEE sequence
  const float s = m > 0.f ? r * damping : 0.f;
  return make_float2(d.x * s, -d.y * s);
}

struct Pair {
  float2 a, b;  // fine columns c0 = 2jx+o, c1 = c0+1
};

__device__ __forceinline__ Pair ld_pair(const float2* row, int c0, int nx) {
  // c0 may be -1..nx; c0 even-aligned iff o == 0
  Pair p;
  p.a = (c0 >= 0 && c0 < nx) ? __ldg(row + c0) : make_float2(0.f, 0.f);
  p.b = (c0 + 1 >= 0 && c0 + 1 < nx) ? __ldg(row + c0 + 1) : make_float2(0.f, 0.f);
  return p;
}
// the lane's two columns (c0, c0 + 1); EVEN: c0 even, so both lie inside or
// both outside the grid (nx even) and one aligned float4 load fetches them
template <bool EVEN>
__device__ __forceinline__ Pair ldp(const float2* row, int c0, int nx) {
  if (EVEN) {
    const float4 q = __ldg(reinterpret_cast<const float4*>(row + min(max(c0, 0), nx - 2)));
    const bool ok = c0 >= 0 && c0 < nx;
    Pair p;
    p.a = ok ? make_float2(q.x, q.y) : make_float2(0.f, 0.f);
    p.b = ok ? make_float2(q.z, q.w) : make_float2(0.f, 0.f);
    return p;
  }
  return ld_pair(row, c0, nx);
}
// unmasked variant at clamped columns (ca, cb = ca + 1 when EVEN)
template <bool EVEN>
__device__ __forceinline__ void ld2(const float2* row, int ca, int cb, float2& a, float2& b) {
  if (EVEN) {
    const float4 q = __ldg(reinterpret_cast<const float4*>(row + ca));
    a = make_float2(q.x, q.y);
    b = make_float2(q.z, q.w);
  } else {
    a = __ldg(row + ca);
    b = __ldg(row + cb);
  }
}
__device__ __forceinline__ float2 shfl_up2(float2 v) {
  return make_float2(__shfl_up_sync(0xffffffffu, v.x, 1), __shfl_up_sync(0xffffffffu, v.y, 1));
}
__device__ __forceinline__ float2 shfl_down2(float2 v) {
  return make_float2(__shfl_down_sync(0xffffffffu, v.x, 1), __shfl_down_sync(0xffffffffu, v.y, 1));
}
// M v at (c0, c1) of one row: d v - ih2 (up + down + left + right)
__device__ __forceinline__ Pair apply_M(const Pair& d, const Pair& vm, const Pair& v, const Pair& vp, float ih2) {
  const float2 left = shfl_up2(v.b);    // column c0 - 1 (lane - 1's c1)
  const float2 right = shfl_down2(v.a); // column c1 + 1 (lane + 1's c0)
  Pair o;
  float2 nb = cadd(cadd(vm.a, vp.a), cadd(left, v.b));
  o.a = cmul(d.a, v.a);
  o.a.x = fmaf(-ih2, nb.x, o.a.x);
  o.a.y = fmaf(-ih2, nb.y, o.a.y);
  nb = cadd(cadd(vm.b, vp.b), cadd(v.a, right));
  o.b = cmul(d.b, v.b);
  o.b.x = fmaf(-ih2, nb.x, o.b.x);
  o.b.y = fmaf(-ih2, nb.y, o.b.y);
  return o;
}

// down leg: grid (ceil(cnx / 30), ceil(row chunks / WARPS), B), block 32 x WARPS
template <bool WD>  // WD: Jacobi factor w = damping / d formed from d in registers (no wdi stream)
__global__ void __launch_bounds__(32 * WARPS) k_down_stream(LevelView L, float damping, int offset, int rows_per_chunk,
                                                            const int* act, const float2* __restrict__ f,
                                                            const float* fscale, float2* __restrict__ fc) {
  pdl_enter();
  const int b = blockIdx.z;
  if (act && !act[b]) return;
  const int lane = threadIdx.x, nx = L.nx, ny = L.ny, cnx = nx / 2, cny = ny / 2;
  const int jx = blockIdx.x * SW_OUT - 1 + lane;  // lane 0 / 31: halo
  const int c0 = 2 * jx + offset;
  const int jy0 = (blockIdx.y * WARPS + threadIdx.y) * rows_per_chunk;
  if (jy0 >= cny) return;
  const int jy1 = min(cny, jy0 + rows_per_chunk);
  const size_t N = size_t(nx) * ny;
  const float2* fb = f + b * N;
  const float s = fscale ? fscale[b] : 1.0f;
  const float ih2 = L.inv_h2;
  const bool colok_a = c0 >= 0 && c0 < nx, colok_b = c0 + 1 >= 0 && c0 + 1 < nx;
  // raw row data (f, wD^-1, D), zero outside the domain; prefetched two rows ahead
  struct Raw {
    Pair f, w, d;
  };
  auto load_raw = [&](int y) {
    Raw r;
    if (y < 0 || y >= ny) {
      r.f.a = r.f.b = r.w.a = r.w.b = r.d.a = r.d.b = make_float2(0.f, 0.f);
      return r;
    }
    const size_t o = size_t(y) * nx;
    r.f = ld_pair(fb + o, c0, nx);
    r.d = ld_pair(L.dM + o, c0, nx);
    if (WD) {
      r.w.a = wfrom(r.d.a, damping);
      r.w.b = wfrom(r.d.b, damping);
    } else {
      r.w = ld_pair(L.wdi + o, c0, nx);
    }
    return r;
  };
  auto vrow = [&](const Raw& r) {
    Pair v;
    v.a = cmul(cscale(r.f.a, s), r.w.a);
    v.b = cmul(cscale(r.f.b, s), r.w.b);
    return v;
  };
  // fine rows y from 2 jy0 + o - 1 to 2 (jy1 - 1) + o + 1; v needed one row beyond
  int y = 2 * jy0 + offset - 1;
  Raw r_c = load_raw(y), r_p1 = load_raw(y + 1), r_p2 = load_raw(y + 2);
  Pair v_m = vrow(load_raw(y - 1)), v_c = vrow(r_c);
  float2 h_m2 = make_float2(0.f, 0.f), h_m1 = make_float2(0.f, 0.f);
  const int yend = 2 * (jy1 - 1) + offset + 1;
  for (; y <= yend; ++y) {
    const Raw r_p3 = load_raw(y + 3);  // in flight during this row
    const Pair v_p = vrow(r_p1);
    float2 h = make_float2(0.f, 0.f);
    const Pair mv = apply_M(r_c.d, v_m, v_c, v_p, ih2);
    if (y >= 0 && y < ny) {
      Pair r;
      r.a = colok_a ? csub(cscale(r_c.f.a, s), mv.a) : make_float2(0.f, 0.f);
      r.b = colok_b ? csub(cscale(r_c.f.b, s), mv.b) : make_float2(0.f, 0.f);
      const float2 rl = shfl_up2(r.b);  // r at c0 - 1
      h = caxpy(cscale(r.a, 0.5f), 0.25f, cadd(rl, r.b));
    } else {
      (void)shfl_up2(v_c.b);  // keep the shuffles convergent
    }
    // y = 2 jy + o + 1 closes coarse row jy
    const int t = y - offset - 1;
    if (t >= 2 * jy0 && ((t & 1) == 0)) {
      const int jy = t >> 1;
      if (lane >= 1 && lane <= SW_OUT && jx < cnx && jy < jy1) {
        const float2 v = caxpy(cscale(h_m1, 0.5f), 0.25f, cadd(h_m2, h));
        fc[size_t(b) * cnx * cny + size_t(jy) * cnx + jx] = v;
      }
    }
    h_m2 = h_m1;
    h_m1 = h;
    v_m = v_c;
    v_c = v_p;
    r_c = r_p1;
    r_p1 = r_p2;
    r_p2 = r_p3;
  }
}

// up leg: grid (ceil(cnx / 30), ceil(row chunks / WARPS), B); each warp produces
// fine rows [y0, y1) for its 60 fine columns
template <bool WD, bool SLAB, bool EVEN>  // SLAB: honour row windows (whole grid: compile-time identity); EVEN: offset 0
__global__ void __launch_bounds__(32 * WARPS) k_up_stream(LevelView L, float damping, int offset, int cnx, int cny,
                                                          RowWin cw, int rows_per_chunk, const int* act,
                                                          const float2* __restrict__ f, const float* fscale,
                                                          const float2* __restrict__ vc, float2* __restrict__ z) {
  pdl_enter();
  const int b = blockIdx.z;
  if (act && !act[b]) return;
  const int lane = threadIdx.x, nx = L.nx, ny = L.ny;
  const int jx = blockIdx.x * SW_OUT - 1 + lane;
  const int c0 = 2 * jx + offset;
  // fine rows [L.w.lo, L.w.hi) are emitted; storage rows are global - L.w.row0;
  // loads outside the storage window (and the domain) read zero
  const int row0 = SLAB ? L.w.row0 : 0, rows = SLAB ? L.w.rows : ny;
  const int wlo = SLAB ? L.w.lo : 0, whi = SLAB ? L.w.hi : ny;
  const int y0 = wlo + (blockIdx.y * WARPS + threadIdx.y) * rows_per_chunk;
  if (y0 >= whi) return;
  const int y1 = min(whi, y0 + rows_per_chunk);
  const int ylo = SLAB ? max(0, row0) : 0, yhi = SLAB ? min(ny, row0 + rows) : ny;
  const int crow0 = SLAB ? cw.row0 : 0, crows = SLAB ? cw.rows : cny;
  const int clo = SLAB ? max(0, crow0) : 0, chi = SLAB ? min(cny, crow0 + crows) : cny;
  const size_t N = size_t(nx) * rows;
  const float2* fb = f + b * N - size_t(row0) * nx;  // indexed by global row
  const float2* cb = vc + size_t(b) * cnx * crows - ptrdiff_t(crow0) * cnx;
  const float s = fscale ? fscale[b] : 1.0f;
  const float ih2 = L.inv_h2;
  const bool colok_a = c0 >= 0 && c0 < nx, colok_b = c0 + 1 >= 0 && c0 + 1 < nx;
  // raw fine-row data (f, wD^-1, D) and the two coarse values this lane needs for
  // fine row y (coarse rows (y-o)/2 or floor/ceil), prefetched two rows ahead
  struct Raw {
    Pair f, w, d;
    float2 c0v, c1v;  // vc at this lane's coarse column, rows jlo / jhi
    int even;         // (y - o) even: one coarse row
  };
  auto cload = [&](int jy) {
    return (jy >= clo && jy < chi && jx >= 0 && jx < cnx) ? __ldg(cb + ptrdiff_t(jy) * cnx + jx) : make_float2(0.f, 0.f);
  };
  auto load_raw = [&](int y) {
    Raw r;
    r.even = 1;
    if (y < ylo || y >= yhi) {
      r.f.a = r.f.b = r.w.a = r.w.b = r.d.a = r.d.b = make_float2(0.f, 0.f);
      r.c0v = r.c1v = make_float2(0.f, 0.f);
      return r;
    }
    const ptrdiff_t o = ptrdiff_t(y) * nx, oc = ptrdiff_t(y - row0) * nx;
    r.f = ldp<EVEN>(fb + o, c0, nx);
    r.d = ldp<EVEN>(L.dM + oc, c0, nx);
    if (WD) {
      r.w.a = wfrom(r.d.a, damping);
      r.w.b = wfrom(r.d.b, damping);
    } else {
      r.w = ldp<EVEN>(L.wdi + oc, c0, nx);
    }
    const int t = y - offset;
    if ((t & 1) == 0) {
      r.c0v = cload(t >> 1);
      r.c1v = make_float2(0.f, 0.f);
    } else {
      const int jlo = (t - 1) >> 1;  // t >= -1
      r.c0v = cload(t < 0 ? -1 : jlo);
      r.c1v = cload(jlo + 1);
      r.even = 0;
    }
    return r;
  };
  // v(y) = wD^-1 f + P vc  (horizontal prolongation via one shuffle of the coarse value)
  auto vrow = [&](const Raw& r) {
    const float2 cur = r.even ? r.c0v : cscale(cadd(r.c0v, r.c1v), 0.5f);  // vertical prolongation
    const float2 nxt = shfl_down2(cur);                                   // coarse column jx + 1
    Pair v;
    v.a = colok_a ? cadd(cmul(cscale(r.f.a, s), r.w.a), cur) : make_float2(0.f, 0.f);
    v.b = colok_b ? cadd(cmul(cscale(r.f.b, s), r.w.b), cscale(cadd(cur, nxt), 0.5f)) : make_float2(0.f, 0.f);
    return v;
  };
  Raw r_c = load_raw(y0), r_p1 = load_raw(y0 + 1), r_p2 = load_raw(y0 + 2);
  Pair v_m = vrow(load_raw(y0 - 1)), v_c = vrow(r_c);
  float2* zb = z + b * N - size_t(row0) * nx;
  for (int y = y0; y < y1; ++y) {
    const Raw r_p3 = load_raw(y + 3);
    const Pair v_p = vrow(r_p1);
    const ptrdiff_t o = ptrdiff_t(y) * nx;
    const Pair mv = apply_M(r_c.d, v_m, v_c, v_p, ih2);
    const float2 fa = cscale(r_c.f.a, s), fb2 = cscale(r_c.f.b, s);
    if (lane >= 1 && lane <= SW_OUT) {
      const float2 za = cadd(v_c.a, cmul(csub(fa, mv.a), r_c.w.a));
      const float2 zb2 = cadd(v_c.b, cmul(csub(fb2, mv.b), r_c.w.b));
      if (colok_a && colok_b && ((c0 & 1) == 0)) {
        *reinterpret_cast<float4*>(zb + o + c0) = make_float4(za.x, za.y, zb2.x, zb2.y);
      } else {
        if (colok_a) zb[o + c0] = za;
        if (colok_b) zb[o + c0 + 1] = zb2;
      }
    } else if (lane == 0 && jx == -1 && colok_b) {
      // offset 1: fine column 0 is the second column of coarse column -1; it only
      // needs this lane's own first column and lane 1's, so the halo lane emits it
      zb[o + c0 + 1] = cadd(v_c.b, cmul(csub(fb2, mv.b), r_c.w.b));
    }
    v_m = v_c;
    v_c = v_p;
    r_c = r_p1;
    r_p1 = r_p2;
    r_p2 = r_p3;
  }
}

// Lean down leg: same geometry and arithmetic as k_down_stream, written
// branch-free for the issue-bound regime -- column and row validity become
// 0/1 masks folded into the column scale (loads hit clamped, always-valid
// addresses), shuffles are unconditional, row offsets are 32-bit, and the
// 3-row window rotates through registers in a 2x-unrolled loop.
struct RowIn {
  float2 fa, fb, wa, wb, da, db;  // f (scaled, masked), wD^-1, D at the lane's two fine columns
};

template <bool WD, bool EVEN>  // WD: w = damping / d from d in registers (no wdi stream: 8 B/node less)
__global__ void __launch_bounds__(32 * WARPS) k_down_lean(LevelView L, RowWin cw, float damping, int offset, int rows_per_chunk,
                                                          const int* act, const float2* __restrict__ f,
                                                          const float* fscale, float2* __restrict__ fc) {
  pdl_enter();
  const int b = blockIdx.z;
  if (act && !act[b]) return;
  const int lane = threadIdx.x, nx = L.nx, ny = L.ny, cnx = nx / 2;
  const int jx = blockIdx.x * SW_OUT - 1 + lane;  // lane 0 / 31: halo
  const int c0 = 2 * jx + offset;
  // coarse rows [cw.lo, cw.hi) are emitted into the coarse storage window cw;
  // fine rows are loaded from the storage window L.w (zero outside it)
  const int jy0 = cw.lo + (blockIdx.y * WARPS + threadIdx.y) * rows_per_chunk;
  if (jy0 >= cw.hi) return;
  const int jy1 = min(cw.hi, jy0 + rows_per_chunk);
  const int ylo = max(0, L.w.row0), yhi = min(ny, L.w.row0 + L.w.rows);
  const float2* fb = f + size_t(b) * nx * L.w.rows;
  const float s = fscale ? fscale[b] : 1.0f;
  const float ih2 = L.inv_h2;
  const int ca = EVEN ? min(max(c0, 0), nx - 2) : min(max(c0, 0), nx - 1);
  const int cb = EVEN ? ca + 1 : min(max(c0 + 1, 0), nx - 1);
  const float sa = (c0 >= 0 && c0 < nx) ? s : 0.f, sb = (c0 + 1 >= 0 && c0 + 1 < nx) ? s : 0.f;
  const float ma = sa != 0.f ? 1.f : 0.f, mb = sb != 0.f ? 1.f : 0.f;
  auto load = [&](int y) {
    const bool ok = y >= ylo && y < yhi;
    const int o = ((ok ? y : ylo) - L.w.row0) * nx;
    const float rm = ok ? 1.f : 0.f;
    RowIn r;
    ld2<EVEN>(fb + o, ca, cb, r.fa, r.fb);
    r.fa = cscale(r.fa, sa * rm);
    r.fb = cscale(r.fb, sb * rm);
    ld2<EVEN>(L.dM + o, ca, cb, r.da, r.db);
    if (WD) {
      r.wa = wfrom(r.da, damping);
      r.wb = wfrom(r.db, damping);
    } else {
      ld2<EVEN>(L.wdi + o, ca, cb, r.wa, r.wb);
    }
    return r;
  };
  const int yb = 2 * jy0 + offset - 1;
  const int yend = 2 * (jy1 - 1) + offset + 1;
  RowIn r_c = load(yb), r_p1 = load(yb + 1), r_p2 = load(yb + 2);
  RowIn r_m = load(yb - 1);
  float2 vma = cmul(r_m.fa, r_m.wa), vmb = cmul(r_m.fb, r_m.wb);
  float2 vca = cmul(r_c.fa, r_c.wa), vcb = cmul(r_c.fb, r_c.wb);
  float2 h_m2 = make_float2(0.f, 0.f), h_m1 = h_m2;
  const bool emit_col = lane >= 1 && lane <= SW_OUT && jx < cnx;
  float2* fcb = fc + size_t(b) * cnx * cw.rows - ptrdiff_t(cw.row0) * cnx;
#pragma unroll 2
  for (int y = yb; y <= yend; ++y) {
    const RowIn r_p3 = load(y + 3);  // in flight during this row
    const float2 vpa = cmul(r_p1.fa, r_p1.wa), vpb = cmul(r_p1.fb, r_p1.wb);
    const float2 left = shfl_up2(vcb), right = shfl_down2(vca);
    float2 nb = cadd(cadd(vma, vpa), cadd(left, vcb));
    float2 mva = cmul(r_c.da, vca);
    mva.x = fmaf(-ih2, nb.x, mva.x);
    mva.y = fmaf(-ih2, nb.y, mva.y);
    nb = cadd(cadd(vmb, vpb), cadd(vca, right));
    float2 mvb = cmul(r_c.db, vcb);
    mvb.x = fmaf(-ih2, nb.x, mvb.x);
    mvb.y = fmaf(-ih2, nb.y, mvb.y);
    const float rowm = (y >= 0 && y < ny) ? 1.f : 0.f;
    const float2 ra = cscale(csub(r_c.fa, mva), ma * rowm), rb = cscale(csub(r_c.fb, mvb), mb * rowm);
    const float2 rl = shfl_up2(rb);  // r at c0 - 1
    const float2 h = caxpy(cscale(ra, 0.5f), 0.25f, cadd(rl, rb));
    // y = 2 jy + o + 1 closes coarse row jy
    const int t = y - offset - 1;
    if (t >= 2 * jy0 && ((t & 1) == 0) && emit_col)
      fcb[ptrdiff_t(t >> 1) * cnx + jx] = caxpy(cscale(h_m1, 0.5f), 0.25f, cadd(h_m2, h));
    h_m2 = h_m1;
    h_m1 = h;
    vma = vca;
    vmb = vcb;
    vca = vpa;
    vcb = vpb;
    r_c = r_p1;
    r_p1 = r_p2;
    r_p2 = r_p3;
  }
}

// ---------------------------------------------------------------------------
// Row-streaming legs from a non-zero initial guess e0 (M_VU's level 0,
// inc/precond.hpp:151-158 -> cycle_at with x0 = e0): the pre-smoothed iterate
//   v = e0 + wD^-1 (f - M e0)
// needs the stencil twice, so the register window is one row deeper and the
// warp's left halo two lanes wide on the down leg (v at column c0-1 needs e0 at
// c0-2).  Same geometry otherwise: lane = two fine columns, horizontal
// neighbours by shuffles, no shared memory.  Traffic per fine node: down f, e0,
// D (+wD^-1) in, fc/4 out; up f, e0, D (+wD^-1), vc/4 in, z out.
constexpr int SWE_DOWN = 29;  // coarse columns emitted per warp (lanes 2..30)

struct RowE {
  float2 fa, fb, ea, eb, da, db, wa, wb;  // f (scaled, masked), e0 (masked), D, wD^-1
  float ma, mb;                           // node masks (column and row inside the domain)
};

template <bool WD, bool EVEN>
__device__ __forceinline__ RowE load_rowe(const LevelView& L, const float2* fb, const float2* eb, int y, int ca, int cb,
                                          float sa, float sb, float ma, float mb, float damping) {
  const bool ok = y >= 0 && y < L.ny;
  const int o = (ok ? y : 0) * L.nx;
  const float rm = ok ? 1.f : 0.f;
  RowE r;
  r.ma = ma * rm;
  r.mb = mb * rm;
  ld2<EVEN>(fb + o, ca, cb, r.fa, r.fb);
  r.fa = cscale(r.fa, sa * rm);
  r.fb = cscale(r.fb, sb * rm);
  ld2<EVEN>(eb + o, ca, cb, r.ea, r.eb);
  r.ea = cscale(r.ea, r.ma);
  r.eb = cscale(r.eb, r.mb);
  ld2<EVEN>(L.dM + o, ca, cb, r.da, r.db);
  if (WD) {
    r.wa = wfrom(r.da, damping);
    r.wb = wfrom(r.db, damping);
  } else {
    ld2<EVEN>(L.wdi + o, ca, cb, r.wa, r.wb);
  }
  return r;
}

// v = e0 + wD^-1 (f - M e0) on one row (masked to the domain)
__device__ __forceinline__ Pair smooth_e0(const RowE& um, const RowE& u, const RowE& up, float ih2) {
  const float2 left = shfl_up2(u.eb), right = shfl_down2(u.ea);
  Pair v;
  float2 nb = cadd(cadd(um.ea, up.ea), cadd(left, u.eb));
  float2 me = cmul(u.da, u.ea);
  me.x = fmaf(-ih2, nb.x, me.x);
  me.y = fmaf(-ih2, nb.y, me.y);
  v.a = cscale(cadd(u.ea, cmul(csub(u.fa, me), u.wa)), u.ma);
  nb = cadd(cadd(um.eb, up.eb), cadd(u.ea, right));
  me = cmul(u.db, u.eb);
  me.x = fmaf(-ih2, nb.x, me.x);
  me.y = fmaf(-ih2, nb.y, me.y);
  v.b = cscale(cadd(u.eb, cmul(csub(u.fb, me), u.wb)), u.mb);
  return v;
}

// down leg from e0: grid (ceil(cnx / 29), ceil(row chunks / WARPS), B)
template <bool WD, bool EVEN>
__global__ void __launch_bounds__(32 * WARPS) k_down_e0(LevelView L, float damping, int offset, int rows_per_chunk,
                                                        const int* act, const float2* __restrict__ f, const float* fscale,
                                                        const float2* __restrict__ e0, float2* __restrict__ fc) {
  pdl_enter();
  const int b = blockIdx.z;
  if (act && !act[b]) return;
  const int lane = threadIdx.x, nx = L.nx, ny = L.ny, cnx = nx / 2, cny = ny / 2;
  const int jx = blockIdx.x * SWE_DOWN - 2 + lane;  // lanes 0, 1 and 31: halo
  const int c0 = 2 * jx + offset;
  const int jy0 = (blockIdx.y * WARPS + threadIdx.y) * rows_per_chunk;
  if (jy0 >= cny) return;
  const int jy1 = min(cny, jy0 + rows_per_chunk);
  const size_t N = size_t(nx) * ny;
  const float2* fb = f + size_t(b) * N;
  const float2* eb = e0 + size_t(b) * N;
  const float s = fscale ? fscale[b] : 1.0f;
  const float ih2 = L.inv_h2;
  const int ca = EVEN ? min(max(c0, 0), nx - 2) : min(max(c0, 0), nx - 1);
  const int cb = EVEN ? ca + 1 : min(max(c0 + 1, 0), nx - 1);
  const float ma = (c0 >= 0 && c0 < nx) ? 1.f : 0.f, mb = (c0 + 1 >= 0 && c0 + 1 < nx) ? 1.f : 0.f;
  auto load = [&](int y) { return load_rowe<WD, EVEN>(L, fb, eb, y, ca, cb, s * ma, s * mb, ma, mb, damping); };
  const int yb = 2 * jy0 + offset - 1;  // first residual row
  const int yend = 2 * (jy1 - 1) + offset + 1;
  RowE R_m = load(yb - 1), R_c = load(yb), R_p1 = load(yb + 1), R_p2 = load(yb + 2);
  Pair v_m, v_c;
  {
    const RowE R_m2 = load(yb - 2);
    v_m = smooth_e0(R_m2, R_m, R_c, ih2);
    v_c = smooth_e0(R_m, R_c, R_p1, ih2);
  }
  float2 h_m2 = make_float2(0.f, 0.f), h_m1 = h_m2;
  const bool emit_col = lane >= 2 && lane <= SWE_DOWN + 1 && jx < cnx;
  float2* fcb = fc + size_t(b) * cnx * cny;
  for (int y = yb; y <= yend; ++y) {
    const RowE R_p3 = load(y + 3);  // in flight during this row
    const Pair v_p = smooth_e0(R_c, R_p1, R_p2, ih2);
    const float2 left = shfl_up2(v_c.b), right = shfl_down2(v_c.a);
    float2 nb = cadd(cadd(v_m.a, v_p.a), cadd(left, v_c.b));
    float2 mva = cmul(R_c.da, v_c.a);
    mva.x = fmaf(-ih2, nb.x, mva.x);
    mva.y = fmaf(-ih2, nb.y, mva.y);
    nb = cadd(cadd(v_m.b, v_p.b), cadd(v_c.a, right));
    float2 mvb = cmul(R_c.db, v_c.b);
    mvb.x = fmaf(-ih2, nb.x, mvb.x);
    mvb.y = fmaf(-ih2, nb.y, mvb.y);
    const float2 ra = cscale(csub(R_c.fa, mva), R_c.ma), rb = cscale(csub(R_c.fb, mvb), R_c.mb);
    const float2 rl = shfl_up2(rb);  // r at c0 - 1
    const float2 h = caxpy(cscale(ra, 0.5f), 0.25f, cadd(rl, rb));
    const int t = y - offset - 1;  // y = 2 jy + o + 1 closes coarse row jy
    if (t >= 2 * jy0 && ((t & 1) == 0) && emit_col)
      fcb[ptrdiff_t(t >> 1) * cnx + jx] = caxpy(cscale(h_m1, 0.5f), 0.25f, cadd(h_m2, h));
    h_m2 = h_m1;
    h_m1 = h;
    v_m = v_c;
    v_c = v_p;
    R_m = R_c;
    R_c = R_p1;
    R_p1 = R_p2;
    R_p2 = R_p3;
  }
}

// up leg from e0: grid (ceil(cnx / 30), ceil(row chunks / WARPS), B)
template <bool WD, bool EVEN>
__global__ void __launch_bounds__(32 * WARPS) k_up_e0(LevelView L, float damping, int offset, int cnx, int cny,
                                                      int rows_per_chunk, const int* act, const float2* __restrict__ f,
                                                      const float* fscale, const float2* __restrict__ e0,
                                                      const float2* __restrict__ vc, float2* __restrict__ z) {
  pdl_enter();
  const int b = blockIdx.z;
  if (act && !act[b]) return;
  const int lane = threadIdx.x, nx = L.nx, ny = L.ny;
  const int jx = blockIdx.x * SW_OUT - 1 + lane;  // lanes 0 and 31: halo
  const int c0 = 2 * jx + offset;
  const int y0 = (blockIdx.y * WARPS + threadIdx.y) * rows_per_chunk;
  if (y0 >= ny) return;
  const int y1 = min(ny, y0 + rows_per_chunk);
  const size_t N = size_t(nx) * ny;
  const float2* fb = f + size_t(b) * N;
  const float2* eb = e0 + size_t(b) * N;
  const float2* cbp = vc + size_t(b) * cnx * cny;
  const float s = fscale ? fscale[b] : 1.0f;
  const float ih2 = L.inv_h2;
  const int ca = EVEN ? min(max(c0, 0), nx - 2) : min(max(c0, 0), nx - 1);
  const int cb = EVEN ? ca + 1 : min(max(c0 + 1, 0), nx - 1);
  const float ma = (c0 >= 0 && c0 < nx) ? 1.f : 0.f, mb = (c0 + 1 >= 0 && c0 + 1 < nx) ? 1.f : 0.f;
  const int jxc = min(max(jx, 0), cnx - 1);
  const float mc = (jx >= 0 && jx < cnx) ? 1.f : 0.f;
  struct Raw {
    RowE u;
    float2 p;  // vertical prolongation of vc at this lane's coarse column
  };
  auto cval = [&](int jy) {
    const bool ok = jy >= 0 && jy < cny;
    return cscale(__ldg(cbp + (ok ? jy : 0) * cnx + jxc), ok ? mc : 0.f);
  };
  auto load = [&](int y) {
    Raw r;
    r.u = load_rowe<WD, EVEN>(L, fb, eb, y, ca, cb, s * ma, s * mb, ma, mb, damping);
    const int t = y - offset;
    if ((t & 1) == 0) {
      r.p = cval(t >> 1);
    } else {
      const int jlo = (t - 1) >> 1;  // t >= -1
      r.p = cscale(cadd(cval(jlo), cval(jlo + 1)), 0.5f);
    }
    return r;
  };
  // v(y) = smoothed e0 + P vc (horizontal prolongation via one shuffle)
  auto vrow = [&](const RowE& um, const Raw& r, const RowE& up) {
    Pair v = smooth_e0(um, r.u, up, ih2);
    const float2 nxt = shfl_down2(r.p);  // coarse column jx + 1
    v.a = cadd(v.a, cscale(r.p, r.u.ma));
    v.b = cadd(v.b, cscale(cscale(cadd(r.p, nxt), 0.5f), r.u.mb));
    return v;
  };
  Raw R_m = load(y0 - 1), R_c = load(y0), R_p1 = load(y0 + 1), R_p2 = load(y0 + 2);
  Pair v_m, v_c;
  {
    const Raw R_m2 = load(y0 - 2);
    v_m = vrow(R_m2.u, R_m, R_c.u);
    v_c = vrow(R_m.u, R_c, R_p1.u);
  }
  float2* zb = z + size_t(b) * N;
  const bool emit = lane >= 1 && lane <= SW_OUT;
  for (int y = y0; y < y1; ++y) {
    const Raw R_p3 = load(y + 3);
    const Pair v_p = vrow(R_c.u, R_p1, R_p2.u);
    const Pair mv = apply_M(Pair{R_c.u.da, R_c.u.db}, v_m, v_c, v_p, ih2);
    const ptrdiff_t o = ptrdiff_t(y) * nx;
    const float2 za = cadd(v_c.a, cmul(csub(R_c.u.fa, mv.a), R_c.u.wa));
    const float2 zb2 = cadd(v_c.b, cmul(csub(R_c.u.fb, mv.b), R_c.u.wb));
    if (emit) {
      if (ma != 0.f && mb != 0.f && ((c0 & 1) == 0)) {
        *reinterpret_cast<float4*>(zb + o + c0) = make_float4(za.x, za.y, zb2.x, zb2.y);
      } else {
        if (ma != 0.f) zb[o + c0] = za;
        if (mb != 0.f) zb[o + c0 + 1] = zb2;
      }
    } else if (lane == 0 && jx == -1 && mb != 0.f) {
      zb[o + c0 + 1] = zb2;  // offset 1: fine column 0 belongs to coarse column -1
    }
    v_m = v_c;
    v_c = v_p;
    R_m = R_c;
    R_c = R_p1;
    R_p1 = R_p2;
    R_p2 = R_p3;
  }
}

}  // namespace

// Jacobi factor source for the legs: read the stored wD^-1 (L2-resident working
// sets, where the legs are issue-bound and one more load is cheaper than a
// reciprocal) or form it from D in registers (HBM-bound working sets: the
// legs then move the algorithmic 18 / 26 B per fine node).  Decided on the
// global level size, so row slabs take the same path as the whole grid.
// HBM-streaming regime: >= 1M nodes per launch (c2-c4 fine levels; c0 and c1
// launches are 0.4-0.8M nodes of L2-resident, latency-bound work)
static bool hbm_bound(const Context& c, const LevelView& L, int B) {
  (void)c;
  return double(L.nx) * L.ny * B >= double(1 << 20);
}
static bool legs_wd(const Context& c, const LevelView& L, int B) {
  return c.opt_legs_wd == 2 ? hbm_bound(c, L, B) : c.opt_legs_wd != 0;
}
// cp.async-staged legs (hb_mg_staged.cu) where the working set streams from
// HBM; the register-prefetch kernels are faster on L2-resident levels (c0)
static bool legs_staged(const Context& c, const LevelView& L, int B) {
  return c.opt_staged_legs == 2 ? hbm_bound(c, L, B) : c.opt_staged_legs != 0;
}

void launch_down_stream(Context& c, const LevelView& L, const RowWin& cw, float damping, int offset, int B,
                        const int* act, const float2* f, const float* fscale, const float2* e0, float2* fc,
                        float2* vpre) {
  const int cnx = L.nx / 2, cny = cw.hi - cw.lo;  // coarse rows emitted
  // only the lean kernel honours row windows (row slabs)
  const bool slab = L.w.rows != L.ny || cw.rows != L.ny / 2 || cw.lo != 0;
  const bool staged = legs_staged(c, L, B);
  if (e0 && slab && !staged)
    throw HbError{HB_ERR_ARG, "register-prefetch legs from an initial guess run on whole grids only"};
  const int tok = prof_begin(c, PC_DOWN);
  // rows per warp: enough warps to fill the machine, >= 4 coarse rows to amortise the halo
  static const int env_d = getenv("HB_RPC_DOWN") ? atoi(getenv("HB_RPC_DOWN")) : 0;
  int rpc = 8;
  while (rpc > 4 && size_t((cnx + SW_OUT - 1) / SW_OUT) * ((cny + rpc - 1) / rpc) * B < size_t(rpc_fill()) * c.num_sms * WARPS)
    rpc /= 2;
  if (env_d) rpc = env_d;
  const int chunks = (cny + rpc - 1) / rpc;
  const bool wd = legs_wd(c, L, B), even = (offset & 1) == 0;
  if (!e0 && !slab && launch_down_row(c, L, damping, offset, B, act, f, fscale, fc)) {
    // full-row warps (hb_mg_rowwarp.cu: 64 / 128-wide levels)
  } else if (staged) {
    launch_down_staged(c, L, cw, damping, offset, B, act, f, fscale, e0, wd, fc, vpre);
  } else if (e0) {
    const dim3 grid((cnx + SWE_DOWN - 1) / SWE_DOWN, (chunks + WARPS - 1) / WARPS, B);
    auto k = wd ? (even ? k_down_e0<true, true> : k_down_e0<true, false>)
                : (even ? k_down_e0<false, true> : k_down_e0<false, false>);
    launch_pdl(c, k, grid, dim3(32, WARPS), 0, L, damping, offset, rpc, act, f, fscale, e0, fc);
  } else {
    const dim3 grid((cnx + SW_OUT - 1) / SW_OUT, (chunks + WARPS - 1) / WARPS, B);
    if (c.opt_lean_legs || slab) {
      auto k = wd ? (even ? k_down_lean<true, true> : k_down_lean<true, false>)
                  : (even ? k_down_lean<false, true> : k_down_lean<false, false>);
      launch_pdl(c, k, grid, dim3(32, WARPS), 0, L, cw, damping, offset, rpc, act, f, fscale, fc);
    } else {
      launch_pdl(c, wd ? k_down_stream<true> : k_down_stream<false>, grid, dim3(32, WARPS), 0, L, damping, offset, rpc,
                 act, f, fscale, fc);
    }
  }
  const double rows = 2.0 * cny;  // fine rows behind the emitted coarse rows
  // algorithmic bytes: coefficients count 8 B/node (D, c64) whichever
  // variant runs -- the stored-wD^-1 kernels read 8 more, which is overhead, not work
  prof_end(c, PC_DOWN, tok, double(B) * L.nx * rows * (e0 ? 18.0 : 10.0) + double(L.nx) * rows * 8.0, 0);
  HB_CUDA(cudaGetLastError());
}

void launch_up_stream(Context& c, const LevelView& L, float damping, int offset, int cnx, int cny, const RowWin& cw,
                      int B, const int* act, const float2* f, const float* fscale, const float2* e0, const float2* vc,
                      float2* z, const float2* vpre) {
  const int tok = prof_begin(c, PC_UP);
  static const int env_u = getenv("HB_RPC_UP") ? atoi(getenv("HB_RPC_UP")) : 0;
  const int nrows = L.w.hi - L.w.lo;
  int rpc = 16;
  while (rpc > 8 && size_t((cnx + SW_OUT - 1) / SW_OUT) * ((nrows + rpc - 1) / rpc) * B < size_t(rpc_fill()) * c.num_sms * WARPS)
    rpc /= 2;
  if (env_u) rpc = env_u;
  const int chunks = (nrows + rpc - 1) / rpc;
  const dim3 grid((cnx + SW_OUT - 1) / SW_OUT, (chunks + WARPS - 1) / WARPS, B);
  const bool slab = L.w.rows != L.ny || L.w.lo != 0 || L.w.hi != L.ny || cw.rows != cny || cw.row0 != 0;
  const bool wd = legs_wd(c, L, B), even = (offset & 1) == 0;
  if (!e0 && !slab && launch_up_row(c, L, damping, offset, B, act, f, fscale, vc, z)) {
    // full-row warps (hb_mg_rowwarp.cu: 64 / 128-wide levels)
  } else if (legs_staged(c, L, B)) {
    launch_up_staged(c, L, damping, offset, cnx, cny, cw, B, act, f, fscale, e0, vc, wd, z, vpre);
  } else if (e0 && slab) {
    throw HbError{HB_ERR_ARG, "register-prefetch legs from an initial guess run on whole grids only"};
  } else if (e0) {
    auto k = wd ? (even ? k_up_e0<true, true> : k_up_e0<true, false>)
                : (even ? k_up_e0<false, true> : k_up_e0<false, false>);
    launch_pdl(c, k, grid, dim3(32, WARPS), 0, L, damping, offset, cnx, cny, rpc, act, f, fscale, e0, vc, z);
  } else {
    decltype(&k_up_stream<true, true, true>) k;
    if (slab)
      k = wd ? (even ? k_up_stream<true, true, true> : k_up_stream<true, true, false>)
             : (even ? k_up_stream<false, true, true> : k_up_stream<false, true, false>);
    else
      k = wd ? (even ? k_up_stream<true, false, true> : k_up_stream<true, false, false>)
             : (even ? k_up_stream<false, false, true> : k_up_stream<false, false, false>);
    launch_pdl(c, k, grid, dim3(32, WARPS), 0, L, damping, offset, cnx, cny, cw, rpc, act, f, fscale, vc, z);
  }
  prof_end(c, PC_UP, tok, double(B) * L.nx * nrows * (e0 ? 26.0 : 18.0) + double(L.nx) * nrows * 8.0, 0);
  HB_CUDA(cudaGetLastError());
}

}  // namespace hb
