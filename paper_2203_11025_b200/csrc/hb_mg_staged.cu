// Row-streaming V-cycle legs with asynchronous shared-memory staging.
//
// Same geometry and arithmetic as hb_mg_stream.cu (a warp owns a strip of
// coarse columns, each lane two adjacent fine columns, and marches down a
// chunk of rows with the stencil window in registers; horizontal neighbours by
// shuffles), but the input rows no longer come through registers: each warp
// keeps a ring of NS row stages in shared memory, filled by cp.async (16-byte
// LDGSTS per lane, zero-filled outside the grid / the storage window), so NS
// rows per warp are in flight while the warp computes.  The register-prefetch
// kernels keep ~1 row in flight and were latency-bound at ~28% warp occupancy
// (ncu, c4 4096^2: 60% of DRAM peak on the down leg); the ring decouples the
// bytes in flight from the register budget.
//
//   down:  v = wD^-1 f             (E0: v = e0 + wD^-1 (f - M e0))
//          fc = R_o (f - M v)
//   up:    v = (as down) + P_o vc
//          z = v + wD^-1 (f - M v)
// (inc/multigrid.hpp:108-119 with inc/stencil.hpp:44-165; offset o = level % 2.)
//
// Stage layout (per warp, per row): NA fine arrays (f, D, [wD^-1], [e0]) of 68
// float2 (33 16-byte chunks from the warp's aligned base column; 68 keeps
// 16-byte alignment), and for the up leg 2 x 32 coarse values (the one or two
// coarse rows prolongation needs for that fine row).
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

constexpr int GW = 4;      // warps per CTA
constexpr int ROWF = 68;   // float2 per staged fine row

__device__ __forceinline__ void cp16(float2* dst, const float2* src, bool ok) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(src), "r"(ok ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp8(float2* dst, const float2* src, bool ok) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(src), "r"(ok ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// A fine row of one array is staged as 33 16-byte chunks from the warp's even
// base column B0: lane L copies columns B0 + 2L, B0 + 2L + 1 (B0 and nx even, so
// a chunk is inside or outside the grid as a whole); for odd offsets lane 0
// also copies the 33rd chunk (Ring::stage).

// the lane's two columns from a staged row (element 2L + o)
template <bool EVEN>
__device__ __forceinline__ void read_pair(const float2* st, int lane, float2& a, float2& b) {
  if (EVEN) {
    const float4 q = *reinterpret_cast<const float4*>(st + 2 * lane);
    a = make_float2(q.x, q.y);
    b = make_float2(q.z, q.w);
  } else {
    a = st[2 * lane + 1];
    b = st[2 * lane + 2];
  }
}

__device__ __forceinline__ float2 shfl_up2(float2 v) {
  return make_float2(__shfl_up_sync(0xffffffffu, v.x, 1), __shfl_up_sync(0xffffffffu, v.y, 1));
}
__device__ __forceinline__ float2 shfl_down2(float2 v) {
  return make_float2(__shfl_down_sync(0xffffffffu, v.x, 1), __shfl_down_sync(0xffffffffu, v.y, 1));
}
// damping / d (0 where d == 0: zero-filled padding)
__device__ __forceinline__ float2 wfrom(float2 d, float damping) {
  const float m = fmaf(d.x, d.x, d.y * d.y);
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(m));
  const float s = m > 0.f ? r * damping : 0.f;
  return pmulv(d, make_float2(s, -s));
}

struct Node2 {
  float2 fa, fb, da, db, wa, wb, ea, eb;  // f (scaled, masked), D, wD^-1, e0 at the lane's two columns
  float ma, mb;                           // node masks (column and row inside the grid / window)
  float2 p;                               // vertical prolongation of vc at this lane's coarse column (up leg)
};
struct Pair2 {
  float2 a, b;
};

template <bool E0, bool WD>
struct Arrays {
  static constexpr int NA = 2 + (WD ? 0 : 1) + (E0 ? 1 : 0);
  static constexpr int W = 2, E = WD ? 2 : 3;  // stage slots of wD^-1 and e0
};

// M u at the lane's two columns of one row: d u - ih2 (up + down + left + right)
__device__ __forceinline__ Pair2 apply_M2(float2 da, float2 db, const Pair2& um, const Pair2& u, const Pair2& up,
                                          float ih2) {
  const float2 left = shfl_up2(u.b), right = shfl_down2(u.a);
  Pair2 o;
  float2 nb = padd(padd(um.a, up.a), padd(left, u.b));
  o.a = paxpy(pmul(da, u.a), -ih2, nb);
  nb = padd(padd(um.b, up.b), padd(u.a, right));
  o.b = paxpy(pmul(db, u.b), -ih2, nb);
  return o;
}

// pre-smoothed iterate of one row: wD^-1 f, or e0 + wD^-1 (f - M e0)
template <bool E0>
__device__ __forceinline__ Pair2 presmooth(const Node2& um, const Node2& u, const Node2& up, float ih2) {
  Pair2 v;
  if (E0) {
    const Pair2 me = apply_M2(u.da, u.db, Pair2{um.ea, um.eb}, Pair2{u.ea, u.eb}, Pair2{up.ea, up.eb}, ih2);
    v.a = padd(u.ea, pmul(psub(u.fa, me.a), u.wa));  // zero outside: e0 = wD^-1 = 0 there (zero-filled)
    v.b = padd(u.eb, pmul(psub(u.fb, me.b), u.wb));
  } else {
    v.a = pmul(u.fa, u.wa);
    v.b = pmul(u.fb, u.wb);
  }
  return v;
}

// Per-warp row ring: rows first, first+1, ... are consumed in order; NS rows
// are in flight.  Row k lives in stage k % NS; after a row is read into
// registers its stage is refilled with row k + NS (zero-filled, without
// traffic, past the last row the warp needs).
template <bool E0, bool WD, bool EVEN, bool UP, int NS>
struct Ring {
  using A = Arrays<E0, WD>;
  static constexpr int STG = A::NA * ROWF + (UP ? 64 : 0);  // float2 per stage
  float2* ring;
  const float2* fb;   // f of this column, indexed by storage row
  const float2* eb;   // e0
  const float2* cb;   // vc of this column, indexed by global coarse row (UP)
  const float2* dM;
  const float2* wdi;
  int first, last, k, lane, B0, nx, ylo, yhi, row0, offset, jx, cnx, clo, chi;
  float sa, sb, ma, mb, damping;

  int cA, cB;      // clamped column of the lane's chunk (and lane 0's 33rd chunk)
  bool okA, okB, jok;
  const float2* cbase;  // vc at (coarse row clo, the lane's clamped coarse column)
  __device__ __forceinline__ void stage(float2* dst, const float2* base, int o, bool rok) {
    cp16(dst + 2 * lane, base + (o + cA), rok && okA);
    if (!EVEN && lane == 0) cp16(dst + 64, base + (o + cB), rok && okB);
  }
  __device__ __forceinline__ void issue(int kk) {
    const int y = first + kk;
    const bool ok = y >= ylo && y < yhi && y <= last;
    const int o = ((ok ? y : ylo) - row0) * nx;
    float2* st = ring + (kk & (NS - 1)) * STG;
    stage(st, fb, o, ok);
    stage(st + ROWF, dM, o, ok);
    if (!WD) stage(st + A::W * ROWF, wdi, o, ok);
    if (E0) stage(st + A::E * ROWF, eb, o, ok);
    if (UP) {
      // coarse rows of fine row y: t = y - o even -> t/2; odd -> (t-1)/2, (t+1)/2
      float2* sc = st + A::NA * ROWF;
      const int t = y - offset;
      const int j0 = t >> 1;  // floor: t even -> t/2, odd -> (t-1)/2
      const bool ok0 = ok && jok && unsigned(j0 - clo) < unsigned(chi - clo);
      const bool ok1 = ok && jok && (t & 1) && unsigned(j0 + 1 - clo) < unsigned(chi - clo);
      const int oc = (j0 - clo) * cnx;
      cp8(sc + lane, cbase + (ok0 ? oc : 0), ok0);
      cp8(sc + 32 + lane, cbase + (ok1 ? oc + cnx : 0), ok1);
    }
    cp_commit();
  }
  __device__ __forceinline__ void start() {
    k = 0;
    const int a = B0 + 2 * lane, b2 = B0 + 64;
    okA = a >= 0 && a < nx;
    okB = b2 < nx;
    cA = okA ? a : 0;
    cB = okB ? b2 : 0;
    if (UP) {
      jok = jx >= 0 && jx < cnx;
      cbase = cb + ptrdiff_t(clo) * cnx + (jok ? jx : 0);
    }
#pragma unroll
    for (int i = 0; i < NS; ++i) issue(i);
  }
  __device__ __forceinline__ Node2 next() {
    cp_wait<NS - 1>();
    __syncwarp();
    const float2* st = ring + (k & (NS - 1)) * STG;
    const int y = first + k;
    const float rm = (y >= ylo && y < yhi) ? 1.f : 0.f;
    Node2 n;
    n.ma = ma * rm;
    n.mb = mb * rm;
    read_pair<EVEN>(st, lane, n.fa, n.fb);  // zero outside the grid / window
    n.fa = pscale(n.fa, sa);
    n.fb = pscale(n.fb, sb);
    read_pair<EVEN>(st + ROWF, lane, n.da, n.db);
    if (WD) {
      n.wa = wfrom(n.da, damping);
      n.wb = wfrom(n.db, damping);
    } else {
      read_pair<EVEN>(st + A::W * ROWF, lane, n.wa, n.wb);
    }
    if (E0) read_pair<EVEN>(st + A::E * ROWF, lane, n.ea, n.eb);
    if (UP) {
      const float2* sc = st + A::NA * ROWF;
      const float2 c0v = sc[lane];
      n.p = ((y - offset) & 1) ? pscale(padd(c0v, sc[32 + lane]), 0.5f) : c0v;
    }
    __syncwarp();
    issue(k + NS);
    ++k;
    return n;
  }
  __device__ __forceinline__ void finish() { cp_wait<0>(); }
};

template <bool E0>
__host__ __device__ constexpr int down_halo() { return E0 ? 2 : 1; }  // left halo lanes (v at c0 - 1 needs e0 at c0 - 2)
template <bool E0>
__host__ __device__ constexpr int down_out() { return E0 ? 29 : 30; }  // coarse columns emitted per warp

// down leg: grid (ceil(cnx / SWOUT), ceil(row chunks / GW), B), block 32 x GW,
// dynamic smem GW * NS * STG * 8
template <bool E0, bool WD, bool EVEN, int NS>
__global__ void __launch_bounds__(32 * GW) k_down_staged(LevelView L, RowWin cw, float damping, int offset, int rpc,
                                                         const int* act, const float2* __restrict__ f,
                                                         const float* fscale, const float2* __restrict__ e0,
                                                         float2* __restrict__ fc, float2* __restrict__ vpre) {
  extern __shared__ float4 smem4[];
  constexpr int H = down_halo<E0>(), SWOUT = down_out<E0>();
  using R = Ring<E0, WD, EVEN, false, NS>;
  pdl_enter();
  const int b = blockIdx.z;
  if (act && !act[b]) return;
  const int lane = threadIdx.x, nx = L.nx, ny = L.ny, cnx = nx / 2;
  const int jy0 = cw.lo + (blockIdx.y * GW + threadIdx.y) * rpc;
  if (jy0 >= cw.hi) return;
  const int jy1 = min(cw.hi, jy0 + rpc);
  const int jx = blockIdx.x * SWOUT - H + lane;
  const int c0 = 2 * jx + offset;
  const float s = fscale ? fscale[b] : 1.0f;
  const float ih2 = L.inv_h2;
  R rg;
  rg.ring = reinterpret_cast<float2*>(smem4) + threadIdx.y * NS * R::STG;
  const size_t bstride = size_t(nx) * L.w.rows;
  rg.fb = f + b * bstride;
  rg.eb = E0 ? e0 + b * bstride : nullptr;
  rg.cb = nullptr;
  rg.dM = L.dM;
  rg.wdi = L.wdi;
  const int yb = 2 * jy0 + offset - 1;          // first residual row
  const int yend = 2 * (jy1 - 1) + offset + 1;  // last residual row
  rg.first = yb - 1 - (E0 ? 1 : 0);
  rg.last = yend + 1 + (E0 ? 1 : 0);
  rg.lane = lane;
  rg.B0 = 2 * (blockIdx.x * SWOUT - H);
  rg.nx = nx;
  rg.ylo = max(0, L.w.row0);
  rg.yhi = min(ny, L.w.row0 + L.w.rows);
  rg.row0 = L.w.row0;
  rg.offset = offset;
  rg.jx = jx;
  rg.cnx = cnx;
  rg.clo = rg.chi = 0;
  rg.ma = (c0 >= 0 && c0 < nx) ? 1.f : 0.f;
  rg.mb = (c0 + 1 >= 0 && c0 + 1 < nx) ? 1.f : 0.f;
  rg.sa = s * rg.ma;
  rg.sb = s * rg.mb;
  rg.damping = damping;
  rg.start();
  Node2 n_m, n_c, n_p;  // rows y - 1, y, y + 1 (E0: for the pre-smoothing stencil)
  Pair2 v_m, v_c;
  if (E0) {
    const Node2 n_m2 = rg.next();
    n_m = rg.next();
    n_c = rg.next();
    v_m = presmooth<true>(n_m2, n_m, n_c, ih2);
    n_p = rg.next();
    v_c = presmooth<true>(n_m, n_c, n_p, ih2);
  } else {
    n_m = rg.next();
    n_c = rg.next();
    v_m = presmooth<false>(n_m, n_m, n_m, ih2);
    v_c = presmooth<false>(n_c, n_c, n_c, ih2);
  }
  float2 h_m2 = make_float2(0.f, 0.f), h_m1 = h_m2;
  const bool emit_col = lane >= H && lane < H + SWOUT && jx < cnx;
  float2* fcb = fc + size_t(b) * cnx * cw.rows - ptrdiff_t(cw.row0) * cnx;
  for (int y = yb; y <= yend; ++y) {
    Pair2 v_p;
    if (E0) {
      const Node2 n_p2 = rg.next();  // row y + 2
      v_p = presmooth<true>(n_c, n_p, n_p2, ih2);
      n_m = n_c;
      n_c = n_p;
      n_p = n_p2;
    } else {
      n_p = rg.next();  // row y + 1
      v_p = presmooth<false>(n_p, n_p, n_p, ih2);
      n_m = n_c;
      n_c = n_p;
    }
    // residual at row y: n_m now holds row y (both variants)
    const Node2& u = n_m;
    if (E0 && EVEN && vpre && emit_col && y >= 2 * jy0 + offset && y < 2 * jy1 + offset)  // v_pre for the up leg
      *reinterpret_cast<float4*>(vpre + b * bstride + ptrdiff_t(y - L.w.row0) * nx + c0) =
          make_float4(v_c.a.x, v_c.a.y, v_c.b.x, v_c.b.y);
    const Pair2 mv = apply_M2(u.da, u.db, v_m, v_c, v_p, ih2);
    const float2 ra = pscale(psub(u.fa, mv.a), u.ma), rb = pscale(psub(u.fb, mv.b), u.mb);
    const float2 rl = shfl_up2(rb);  // r at c0 - 1
    const float2 h = paxpy(pscale(ra, 0.5f), 0.25f, padd(rl, rb));
    const int t = y - offset - 1;  // y = 2 jy + o + 1 closes coarse row jy
    if (t >= 2 * jy0 && ((t & 1) == 0) && emit_col)
      fcb[ptrdiff_t(t >> 1) * cnx + jx] = paxpy(pscale(h_m1, 0.5f), 0.25f, padd(h_m2, h));
    h_m2 = h_m1;
    h_m1 = h;
    v_m = v_c;
    v_c = v_p;
  }
  rg.finish();
}

// up leg: grid (ceil(cnx / 30), ceil(row chunks / GW), B); each warp produces
// fine rows [y0, y1) of its 60 fine columns
template <bool E0, bool WD, bool EVEN, int NS, bool VP = false>  // VP: read the down leg's v_pre instead of e0
__global__ void __launch_bounds__(32 * GW) k_up_staged(LevelView L, float damping, int offset, int cnx, int cny,
                                                       RowWin cw, int rpc, const int* act, const float2* __restrict__ f,
                                                       const float* fscale, const float2* __restrict__ e0,
                                                       const float2* __restrict__ vc, float2* __restrict__ z) {
  extern __shared__ float4 smem4[];
  constexpr int SWOUT = 30;
  using R = Ring<E0, WD, EVEN, true, NS>;
  pdl_enter();
  const int b = blockIdx.z;
  if (act && !act[b]) return;
  const int lane = threadIdx.x, nx = L.nx, ny = L.ny;
  const int y0 = L.w.lo + (blockIdx.y * GW + threadIdx.y) * rpc;
  if (y0 >= L.w.hi) return;
  const int y1 = min(L.w.hi, y0 + rpc);
  const int jx = blockIdx.x * SWOUT - 1 + lane;
  const int c0 = 2 * jx + offset;
  const float s = fscale ? fscale[b] : 1.0f;
  const float ih2 = L.inv_h2;
  R rg;
  rg.ring = reinterpret_cast<float2*>(smem4) + threadIdx.y * NS * R::STG;
  const size_t bstride = size_t(nx) * L.w.rows;
  rg.fb = f + b * bstride;
  rg.eb = E0 ? e0 + b * bstride : nullptr;
  rg.cb = vc + size_t(b) * cnx * cw.rows - ptrdiff_t(cw.row0) * cnx;
  rg.dM = L.dM;
  rg.wdi = L.wdi;
  constexpr bool DEEP = E0 && !VP;  // the pre-smoothing stencil needs e0 one row beyond
  rg.first = y0 - 1 - (DEEP ? 1 : 0);
  rg.last = y1 + (DEEP ? 1 : 0);
  rg.lane = lane;
  rg.B0 = 2 * (blockIdx.x * SWOUT - 1);
  rg.nx = nx;
  rg.ylo = max(0, L.w.row0);
  rg.yhi = min(ny, L.w.row0 + L.w.rows);
  rg.row0 = L.w.row0;
  rg.offset = offset;
  rg.jx = jx;
  rg.cnx = cnx;
  rg.clo = max(0, cw.row0);
  rg.chi = min(cny, cw.row0 + cw.rows);
  rg.ma = (c0 >= 0 && c0 < nx) ? 1.f : 0.f;
  rg.mb = (c0 + 1 >= 0 && c0 + 1 < nx) ? 1.f : 0.f;
  rg.sa = s * rg.ma;
  rg.sb = s * rg.mb;
  rg.damping = damping;
  rg.start();
  // v(y) = pre-smoothed + P vc (horizontal prolongation via one shuffle of the coarse value)
  auto vrow = [&](const Node2& um, const Node2& u, const Node2& up) {
    Pair2 v;
    if (VP) {
      v.a = u.ea;  // v_pre (zero outside the grid: zero-filled)
      v.b = u.eb;
    } else {
      v = presmooth<E0>(um, u, up, ih2);
    }
    const float2 nxt = shfl_down2(u.p);  // coarse column jx + 1
    v.a = padd(v.a, pscale(u.p, u.ma));
    v.b = padd(v.b, pscale(pscale(padd(u.p, nxt), 0.5f), u.mb));
    return v;
  };
  Node2 n_m, n_c, n_p;
  Pair2 v_m, v_c;
  if (DEEP) {
    const Node2 n_m2 = rg.next();
    n_m = rg.next();
    n_c = rg.next();
    v_m = vrow(n_m2, n_m, n_c);
    n_p = rg.next();
    v_c = vrow(n_m, n_c, n_p);
  } else {
    n_m = rg.next();
    n_c = rg.next();
    v_m = vrow(n_m, n_m, n_m);
    v_c = vrow(n_c, n_c, n_c);
  }
  float2* zb = z + b * bstride - size_t(L.w.row0) * nx;
  const bool emit = lane >= 1 && lane <= SWOUT;
  for (int y = y0; y < y1; ++y) {
    Pair2 v_p;
    if (DEEP) {
      const Node2 n_p2 = rg.next();
      v_p = vrow(n_c, n_p, n_p2);
      n_m = n_c;
      n_c = n_p;
      n_p = n_p2;
    } else {
      n_p = rg.next();
      v_p = vrow(n_p, n_p, n_p);
      n_m = n_c;
      n_c = n_p;
    }
    const Node2& u = n_m;  // row y
    const Pair2 mv = apply_M2(u.da, u.db, v_m, v_c, v_p, ih2);
    const ptrdiff_t o = ptrdiff_t(y) * nx;
    const float2 za = padd(v_c.a, pmul(psub(u.fa, mv.a), u.wa));
    const float2 zb2 = padd(v_c.b, pmul(psub(u.fb, mv.b), u.wb));
    if (emit) {
      if (rg.ma != 0.f && rg.mb != 0.f && EVEN) {
        *reinterpret_cast<float4*>(zb + o + c0) = make_float4(za.x, za.y, zb2.x, zb2.y);
      } else {
        if (rg.ma != 0.f) zb[o + c0] = za;
        if (rg.mb != 0.f) zb[o + c0 + 1] = zb2;
      }
    } else if (lane == 0 && jx == -1 && rg.mb != 0.f) {
      zb[o + c0 + 1] = zb2;  // offset 1: fine column 0 belongs to coarse column -1
    }
    v_m = v_c;
    v_c = v_p;
  }
  rg.finish();
}

template <typename K>
void set_smem(K k, size_t bytes) {
  HB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
}

constexpr int NSTAGE = 4;

template <bool E0, bool WD, bool EVEN>
void down_one(Context& c, dim3 grid, const LevelView& L, const RowWin& cw, float damping, int offset, int rpc,
              const int* act, const float2* f, const float* fscale, const float2* e0, float2* fc, float2* vpre) {
  auto k = k_down_staged<E0, WD, EVEN, NSTAGE>;
  const size_t smem = size_t(GW) * NSTAGE * Ring<E0, WD, EVEN, false, NSTAGE>::STG * sizeof(float2);
  static bool once = (set_smem(k, smem), true);
  (void)once;
  launch_pdl(c, k, grid, dim3(32, GW), smem, L, cw, damping, offset, rpc, act, f, fscale, e0, fc, vpre);
}
template <bool E0, bool WD, bool EVEN, bool VP = false>
void up_one(Context& c, dim3 grid, const LevelView& L, float damping, int offset, int cnx, int cny, const RowWin& cw,
            int rpc, const int* act, const float2* f, const float* fscale, const float2* e0, const float2* vc,
            float2* z) {
  auto k = k_up_staged<E0, WD, EVEN, NSTAGE, VP>;
  const size_t smem = size_t(GW) * NSTAGE * Ring<E0, WD, EVEN, true, NSTAGE>::STG * sizeof(float2);
  static bool once = (set_smem(k, smem), true);
  (void)once;
  launch_pdl(c, k, grid, dim3(32, GW), smem, L, damping, offset, cnx, cny, cw, rpc, act, f, fscale, e0, vc, z);
}

}  // namespace

void launch_down_staged(Context& c, const LevelView& L, const RowWin& cw, float damping, int offset, int B,
                        const int* act, const float2* f, const float* fscale, const float2* e0, bool wd, float2* fc,
                        float2* vpre) {
  if (vpre && (!e0 || (offset & 1))) vpre = nullptr;  // v_pre is stored for the level-0 legs from e0 only
  const int cnx = L.nx / 2, cny = cw.hi - cw.lo;
  const int swout = e0 ? down_out<true>() : down_out<false>();
  static const int env_d = getenv("HB_RPC_DOWN") ? atoi(getenv("HB_RPC_DOWN")) : 0;
  int rpc = 8;
  while (rpc > 4 && size_t((cnx + swout - 1) / swout) * ((cny + rpc - 1) / rpc) * B < size_t(rpc_fill()) * c.num_sms * GW)
    rpc /= 2;
  if (env_d) rpc = env_d;
  const int chunks = (cny + rpc - 1) / rpc;
  const dim3 grid((cnx + swout - 1) / swout, (chunks + GW - 1) / GW, B);
  const bool even = (offset & 1) == 0;
  if (e0) {
    if (wd)
      even ? down_one<true, true, true>(c, grid, L, cw, damping, offset, rpc, act, f, fscale, e0, fc, vpre)
           : down_one<true, true, false>(c, grid, L, cw, damping, offset, rpc, act, f, fscale, e0, fc, vpre);
    else
      even ? down_one<true, false, true>(c, grid, L, cw, damping, offset, rpc, act, f, fscale, e0, fc, vpre)
           : down_one<true, false, false>(c, grid, L, cw, damping, offset, rpc, act, f, fscale, e0, fc, vpre);
  } else {
    if (wd)
      even ? down_one<false, true, true>(c, grid, L, cw, damping, offset, rpc, act, f, fscale, e0, fc, vpre)
           : down_one<false, true, false>(c, grid, L, cw, damping, offset, rpc, act, f, fscale, e0, fc, vpre);
    else
      even ? down_one<false, false, true>(c, grid, L, cw, damping, offset, rpc, act, f, fscale, e0, fc, vpre)
           : down_one<false, false, false>(c, grid, L, cw, damping, offset, rpc, act, f, fscale, e0, fc, vpre);
  }
}

void launch_up_staged(Context& c, const LevelView& L, float damping, int offset, int cnx, int cny, const RowWin& cw,
                      int B, const int* act, const float2* f, const float* fscale, const float2* e0, const float2* vc,
                      bool wd, float2* z, const float2* vpre) {
  static const int env_u = getenv("HB_RPC_UP") ? atoi(getenv("HB_RPC_UP")) : 0;
  const int nrows = L.w.hi - L.w.lo;
  int rpc = 16;
  while (rpc > 8 && size_t((cnx + 29) / 30) * ((nrows + rpc - 1) / rpc) * B < size_t(rpc_fill()) * c.num_sms * GW) rpc /= 2;
  if (env_u) rpc = env_u;
  const int chunks = (nrows + rpc - 1) / rpc;
  const dim3 grid((cnx + 29) / 30, (chunks + GW - 1) / GW, B);
  const bool even = (offset & 1) == 0;
  if (e0 && vpre && even) {  // v_pre from the down leg: no pre-smoothing stencil here
    if (wd)
      up_one<true, true, true, true>(c, grid, L, damping, offset, cnx, cny, cw, rpc, act, f, fscale, vpre, vc, z);
    else
      up_one<true, false, true, true>(c, grid, L, damping, offset, cnx, cny, cw, rpc, act, f, fscale, vpre, vc, z);
  } else if (e0) {
    if (wd)
      even ? up_one<true, true, true>(c, grid, L, damping, offset, cnx, cny, cw, rpc, act, f, fscale, e0, vc, z)
           : up_one<true, true, false>(c, grid, L, damping, offset, cnx, cny, cw, rpc, act, f, fscale, e0, vc, z);
    else
      even ? up_one<true, false, true>(c, grid, L, damping, offset, cnx, cny, cw, rpc, act, f, fscale, e0, vc, z)
           : up_one<true, false, false>(c, grid, L, damping, offset, cnx, cny, cw, rpc, act, f, fscale, e0, vc, z);
  } else {
    if (wd)
      even ? up_one<false, true, true>(c, grid, L, damping, offset, cnx, cny, cw, rpc, act, f, fscale, e0, vc, z)
           : up_one<false, true, false>(c, grid, L, damping, offset, cnx, cny, cw, rpc, act, f, fscale, e0, vc, z);
    else
      even ? up_one<false, false, true>(c, grid, L, damping, offset, cnx, cny, cw, rpc, act, f, fscale, e0, vc, z)
           : up_one<false, false, false>(c, grid, L, damping, offset, cnx, cny, cw, rpc, act, f, fscale, e0, vc, z);
  }
}

}  // namespace hb
