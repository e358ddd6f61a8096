// CTA-resident coarsest-grid GMRES(k) for coarse grids of <= 2048 nodes
// (32x32 at c0): same contract as k_coarse_gmres in hb_mg.cu
// (coarse_solve_with_op, inc/multigrid.hpp:45-61: non-flexible GMRES(k),
// M = D^-1, x0 = 0, fixed budget, happy breakdown).  One 256-thread CTA per
// column; each thread owns NPT nodes; the Krylov basis and z live in shared
// memory (k+1 vectors, <= 200 KB), nothing touches global memory between
// the load of f and the store of x.  Per Arnoldi step
// the 2j+1 inner products (MGS via the Gram recurrence) are reduced with one
// warp reduce-scatter butterfly (62 shuffles for 32 complex slots) instead of
// 5 shuffles per value.
#include <cstdio>
#include <cstdlib>

#include "hb_coarse_common.cuh"

#ifndef HB_CREG_MINB
#define HB_CREG_MINB 2  // resident CTAs per SM asked of k_coarse_reg: 2 (<= 128 registers; ~0.5 KB of spills,
                        // measured 3% faster at c0 x 444 than one CTA at 228 registers)
#endif

namespace hb {

__device__ long long* g_coarse_trace = nullptr;

namespace {

// Per Arnoldi step j (two CTA barriers):
//   w_raw = M D^-1 Vraw_j          (neighbours of Vraw_j read from shared memory)
//   partials: <Vraw_i, w_raw> (i <= j), <Vraw_j, Vraw_k> (k < j), |Vraw_j|^2  -> one butterfly
//   ---- barrier ----
//   every warp folds the 8 warp partials for all slots (redundantly, no serial
//   section): s_j = 1/||Vraw_j||, h_ij = s_i s_j <Vraw_i, w_raw>, MGS Gram
//   correction h_ij -= sum_{k<i} h_kj^(cgs) G_ik (first order; G = O(eps32)),
//   Vraw_{j+1} = w_raw - sum_i (h_ij s_i / s_j) Vraw_i
//   ---- barrier ----
// so the subdiagonal H_{j+1,j} = s_j / s_{j+1} is known one step later.  The
// budget is fixed (tol 1e-300), so the Givens QR of the (k+1) x k Hessenberg
// runs once at the end, followed by back-substitution and x = D^-1 sum y_i V_i
// (krylov.hpp:119-137 non-flexible finalize).
template <int NT, int NPT, int MAXK>
__global__ void __launch_bounds__(NT, 1) k_coarse_small(LevelView L, int m, const int* act,
                                                         const float2* __restrict__ f, float2* __restrict__ x) {
  pdl_enter();
  const int b = blockIdx.x;
  if (act && !act[b]) return;
  extern __shared__ float2 dyn[];  // Vraw_0..Vraw_m [m+1][N], then D^-1 [N]
  __shared__ SmallSmem S;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int nx = L.nx, ny = L.ny, N = nx * ny;
  const float ih2 = L.inv_h2;
  float2* sV = dyn;
  float2* sDi = dyn + size_t(m + 1) * N;
  float2 d[NPT];
  int px[NPT], py[NPT];
  bool ok[NPT];
#pragma unroll
  for (int q = 0; q < NPT; ++q) {
    const int p = t + q * NT;
    ok[q] = p < N;
    px[q] = ok[q] ? p % nx : 0;
    py[q] = ok[q] ? p / nx : 0;
    d[q] = ok[q] ? ld(L.dM, p) : make_float2(1.f, 0.f);
    if (ok[q]) {
      sV[p] = ld(f + size_t(b) * N, p);
      sDi[p] = crcp(d[q]);
    }
  }
  __syncthreads();
  int k = m;
  double hn_prev = 0.0;
#pragma unroll 1
  for (int j = 0; j <= m; ++j) {
    const float2* Vj = sV + size_t(j) * N;
    float2 w[NPT], vj[NPT];
    float v[32];
#pragma unroll
    for (int s2 = 0; s2 < 32; ++s2) v[s2] = 0.f;
    float nrm_part = 0.f;
#pragma unroll
    for (int q = 0; q < NPT; ++q) {
      const int p = t + q * NT;
      w[q] = vj[q] = make_float2(0.f, 0.f);
      if (!ok[q]) continue;
      vj[q] = Vj[p];
      nrm_part = fmaf(vj[q].x, vj[q].x, fmaf(vj[q].y, vj[q].y, nrm_part));
      if (j == m) continue;
      float2 nb = make_float2(0.f, 0.f);
      if (px[q] > 0) nb = cadd(nb, cmul(Vj[p - 1], sDi[p - 1]));
      if (px[q] + 1 < nx) nb = cadd(nb, cmul(Vj[p + 1], sDi[p + 1]));
      if (py[q] > 0) nb = cadd(nb, cmul(Vj[p - nx], sDi[p - nx]));
      if (py[q] + 1 < ny) nb = cadd(nb, cmul(Vj[p + nx], sDi[p + nx]));
      float2 yv = cmul(d[q], cmul(vj[q], sDi[p]));
      yv.x = fmaf(-ih2, nb.x, yv.x);
      yv.y = fmaf(-ih2, nb.y, yv.y);
      w[q] = yv;
    }
    // dots <Vraw_i, w_raw>, i <= j  (floats 2i, 2i+1)
    if (j < m) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if (i > j) break;
        const float2* Vi = sV + size_t(i) * N;
#pragma unroll
        for (int q = 0; q < NPT; ++q) {
          if (!ok[q]) continue;
          const float2 a = Vi[t + q * NT], c = w[q];
          v[2 * i] = fmaf(a.x, c.x, fmaf(a.y, c.y, v[2 * i]));
          v[2 * i + 1] = fmaf(a.x, c.y, fmaf(-a.y, c.x, v[2 * i + 1]));
        }
      }
    }
    warp_reduce_scatter32(v);
    S.part[warp][lane] = v[0];
#pragma unroll
    for (int s2 = 0; s2 < 32; ++s2) v[s2] = 0.f;
    // Gram <Vraw_j, Vraw_k>, k < j (floats 2k, 2k+1), ||Vraw_j||^2 (float 30)
    v[30] = nrm_part;
    if (j < m) {
#pragma unroll
      for (int i = 0; i < 15; ++i) {
        if (i >= j) break;
        const float2* Vi = sV + size_t(i) * N;
#pragma unroll
        for (int q = 0; q < NPT; ++q) {
          if (!ok[q]) continue;
          const float2 a = Vi[t + q * NT], e = vj[q];
          v[2 * i] = fmaf(e.x, a.x, fmaf(e.y, a.y, v[2 * i]));
          v[2 * i + 1] = fmaf(e.x, a.y, fmaf(-e.y, a.x, v[2 * i + 1]));
        }
      }
    }
    warp_reduce_scatter32(v);
    S.part[warp][32 + lane] = v[0];
    __syncthreads();
    // fold (every warp, lane l <-> complex slot l: 0..15 dots, 16..30 Gram, 31 norm)
    double2 val = make_double2(0.0, 0.0);
    {
      const int f0 = lane < 16 ? 2 * lane : 32 + 2 * (lane - 16);
#pragma unroll 4
      for (int w2 = 0; w2 < NT / 32; ++w2) {
        val.x += S.part[w2][f0];
        val.y += S.part[w2][f0 + 1];
      }
    }
    const double nrm = sqrt(__shfl_sync(0xffffffffu, val.x, 31));  // ||Vraw_j|| (float 62 = slot 31 re)
    if (j == 0) {
      if (t == 0) S.beta0 = nrm;
      if (nrm == 0.0) {  // zero rhs -> zero correction
        k = 0;
        break;
      }
    } else {
      const double hn = hn_prev * nrm;  // true H_{j, j-1} = s_{j-1} ||Vraw_j||
      if (t == 0) S.H[j - 1][j] = make_double2(hn, 0.0);
      if (hn <= 1e-14 * S.beta0) {  // happy breakdown (krylov.hpp:240)
        k = j;
        break;
      }
    }
    const double sj = 1.0 / nrm;
    if (t == 0) S.scale[j] = sj;
    if (j == m) break;
    hn_prev = sj;
    // h_i (lane i <= j): s_i s_j <Vraw_i, w_raw>; Gram row j: s_j s_k <Vraw_j, Vraw_k>
    const double si = (lane < j) ? S.scale[lane] : sj;
    double2 hcgs = make_double2(0.0, 0.0);
    if (lane <= j) hcgs = zscale(val, si * sj);
    double2 gjk = make_double2(0.0, 0.0);
    {
      const double2 e = make_double2(__shfl_sync(0xffffffffu, val.x, (16 + lane) & 31),
                                     __shfl_sync(0xffffffffu, val.y, (16 + lane) & 31));
      if (lane < j) gjk = zscale(e, sj * S.scale[lane]);
    }
    // first-order MGS correction: h_i -= sum_{k<i} hcgs_k G_ik
    double2 h = hcgs;
    for (int kk = 0; kk < j; ++kk) {
      const double2 hk = make_double2(__shfl_sync(0xffffffffu, hcgs.x, kk), __shfl_sync(0xffffffffu, hcgs.y, kk));
      const double2 gjkk = make_double2(__shfl_sync(0xffffffffu, gjk.x, kk), __shfl_sync(0xffffffffu, gjk.y, kk));
      if (lane <= j && kk < lane) {
        const double2 Gik = (lane == j) ? gjkk : S.G[lane][kk];
        h = zsub(h, zmul(hk, Gik));
      }
    }
    if (warp == 0) {
      if (lane <= j) S.H[j][lane] = h;
      if (lane < j) S.G[j][lane] = gjk;
    }
    // raw update coefficients c_i = h_i s_i / s_j
    const double2 cc = zscale(h, si / sj);
    float2 cf = make_float2(float(cc.x), float(cc.y));
    float2 vn[NPT];
#pragma unroll
    for (int q = 0; q < NPT; ++q) vn[q] = w[q];
    for (int i = 0; i <= j; ++i) {
      const float2 ci = make_float2(__shfl_sync(0xffffffffu, cf.x, i), __shfl_sync(0xffffffffu, cf.y, i));
      const float2* Vi = sV + size_t(i) * N;
#pragma unroll
      for (int q = 0; q < NPT; ++q)
        if (ok[q]) vn[q] = csub(vn[q], cmul(ci, Vi[t + q * NT]));
    }
    float2* Vn = sV + size_t(j + 1) * N;
#pragma unroll
    for (int q = 0; q < NPT; ++q)
      if (ok[q]) Vn[t + q * NT] = vn[q];
    __syncthreads();
  }
  if (k == 0) {
#pragma unroll
    for (int q = 0; q < NPT; ++q)
      if (ok[q]) x[size_t(b) * N + t + q * NT] = make_float2(0.f, 0.f);
    return;
  }
  __syncthreads();
  if (t == 0) {
    // Givens QR of the (k+1) x k Hessenberg (inc/krylov.hpp:221-232) + back-substitution (:119-126)
    double* cs = S.cs;
    double2* sn = S.sn;
    double2* g = S.g;
    for (int i = 0; i <= k; ++i) g[i] = make_double2(0.0, 0.0);
    g[0] = make_double2(S.beta0, 0.0);
    for (int j = 0; j < k; ++j) {
      double2* hj = S.H[j];
      for (int i = 0; i < j; ++i) {
        const double2 t1 = dadd(zscale(hj[i], cs[i]), zmul(sn[i], hj[i + 1]));
        hj[i + 1] = dadd(zscale(zmul(zconj(sn[i]), hj[i]), -1.0), zscale(hj[i + 1], cs[i]));
        hj[i] = t1;
      }
      const double2 a = hj[j];
      const double hn = hj[j + 1].x;
      // make_givens (krylov.hpp:49-64) with reciprocal square roots instead of
      // hypot + divisions: c = |a|/rho, s = a hn / (rho |a|)
      const double a2 = a.x * a.x + a.y * a.y;
      if (a2 + hn * hn == 0.0) {
        cs[j] = 1.0;
        sn[j] = make_double2(0.0, 0.0);
      } else if (a2 == 0.0) {
        cs[j] = 0.0;
        sn[j] = make_double2(1.0, 0.0);
      } else {
        const double ia = rsqrt(a2), ir = rsqrt(a2 + hn * hn);
        cs[j] = a2 * ia * ir;
        sn[j] = zscale(a, hn * ia * ir);
      }
      hj[j] = dadd(zscale(hj[j], cs[j]), zmul(sn[j], hj[j + 1]));
      hj[j + 1] = make_double2(0.0, 0.0);
      g[j + 1] = zscale(zmul(zconj(sn[j]), g[j]), -1.0);
      g[j] = zscale(g[j], cs[j]);
    }
    for (int i = k - 1; i >= 0; --i) {
      double2 sum = g[i];
      for (int l = i + 1; l < k; ++l) sum = zsub(sum, zmul(S.H[l][i], S.y[l]));
      const double2 d = S.H[i][i];
      const double inv = 1.0 / (d.x * d.x + d.y * d.y);
      S.y[i] = zscale(zmul(sum, zconj(d)), inv);
    }
    for (int i = 0; i < k; ++i) {
      const double2 c = zscale(S.y[i], S.scale[i]);
      S.coef[i] = make_float2(float(c.x), float(c.y));
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NPT; ++q) {
    if (!ok[q]) continue;
    const int p = t + q * NT;
    float2 u = make_float2(0.f, 0.f);
    for (int i = 0; i < k; ++i) u = cadd(u, cmul(S.coef[i], sV[size_t(i) * N + p]));
    x[size_t(b) * N + p] = cmul(u, sDi[p]);
  }
}

// Register-resident variant (N <= NT*NPT, m <= MAXK): each thread keeps its
// NPT nodes of every basis vector in registers, so the inner products, the
// Gram row and the basis update read no shared memory; only u_j = D^-1 V_j
// goes through a zero-bordered smem tile for the stencil's neighbours (four
// independent loads per node, no bounds branches).  Same arithmetic and
// summation order as k_coarse_small (the MGS correction is fed from per-warp
// smem broadcasts instead of double-precision shuffles).
template <int NT, int NPT, int MAXK>
__global__ void __launch_bounds__(NT, HB_CREG_MINB) k_coarse_reg(LevelView L, int m, const int* act,
                                                       const float2* __restrict__ f, float2* __restrict__ x) {
  pdl_enter();
  const int b = blockIdx.x;
  if (act && !act[b]) return;
  long long* const tr = (b == 0 && threadIdx.x == 0) ? g_coarse_trace : nullptr;  // HB_COARSE_TRACE
  extern __shared__ float2 sU2[];  // 2 x (nx+2) x (ny+2) zero-bordered u_j = D^-1 V_j (double-buffered by j)
  __shared__ SmallSmem S;
  __shared__ double2 sHc[MAXK + 1], sGj[MAXK + 1];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int nx = L.nx, ny = L.ny, N = nx * ny, px2 = nx + 2;
  const float ih2 = L.inv_h2;
  float2 V[MAXK + 1][NPT];
  float2 d[NPT], di[NPT];
  int ui[NPT];  // this node's index in the bordered tile
  bool ok[NPT];
  const int tile = (nx + 2) * (ny + 2);
  for (int i = t; i < 2 * tile; i += NT) sU2[i] = make_float2(0.f, 0.f);
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NPT; ++q) {
    const int p = t + q * NT;
    ok[q] = p < N;
    const int xq = ok[q] ? p % nx : 0, yq = ok[q] ? p / nx : 0;
    ui[q] = (yq + 1) * px2 + xq + 1;
    d[q] = ok[q] ? ld(L.dM, p) : make_float2(1.f, 0.f);
    di[q] = crcp(d[q]);
    V[0][q] = ok[q] ? ld(f + size_t(b) * N, p) : make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 1; i <= MAXK; ++i) V[i][q] = make_float2(0.f, 0.f);
    if (ok[q]) sU2[ui[q]] = cmul(V[0][q], di[q]);
  }
  __syncthreads();
  int k = m;
  double hn_prev = 0.0;
  float2 vj[NPT];  // V_j, carried from the previous step (no register-array select)
#pragma unroll
  for (int q = 0; q < NPT; ++q) vj[q] = V[0][q];
#pragma unroll 1
  for (int j = 0; j <= m; ++j) {
    if (tr && j < 16) tr[j * 8 + 0] = clock64();
    const float2* sU = sU2 + (j & 1) * tile;
    float2 w[NPT];
#pragma unroll
    for (int q = 0; q < NPT; ++q) {
      w[q] = make_float2(0.f, 0.f);
      if (j == m || !ok[q]) continue;
      // neighbours (zero border = out of range), same summation order as k_coarse_small
      const float2 ul = sU[ui[q] - 1], ur = sU[ui[q] + 1], uu = sU[ui[q] - px2], ud = sU[ui[q] + px2];
      const float2 nb = cadd(cadd(cadd(ul, ur), uu), ud);
      float2 yv = cmul(d[q], cmul(vj[q], di[q]));
      yv.x = fmaf(-ih2, nb.x, yv.x);
      yv.y = fmaf(-ih2, nb.y, yv.y);
      w[q] = yv;
    }
    // slots: <V_i, w> at (2i, 2i+1); Gram <V_j, V_i> (i <= j, i == j: |V_j|^2)
    // mirrored at (31-2i re, 30-2i im).  Both fit one 32-slot butterfly while
    // 4j + 4 <= 32; later steps use a second butterfly for the Gram row.
    const bool one = j <= 7 || j == m;  // (j == m: no <V_i, w> slots)
    float v[32];
#pragma unroll
    for (int s2 = 0; s2 < 32; ++s2) v[s2] = 0.f;
    if (j < m) {
#pragma unroll
      for (int i = 0; i <= MAXK; ++i) {
        if (i > j) break;
#pragma unroll
        for (int q = 0; q < NPT; ++q) {
          const float2 a = V[i][q], c = w[q];
          v[2 * i] = fmaf(a.x, c.x, fmaf(a.y, c.y, v[2 * i]));
          v[2 * i + 1] = fmaf(a.x, c.y, fmaf(-a.y, c.x, v[2 * i + 1]));
        }
      }
    }
    if (tr && j < 16) tr[j * 8 + 1] = clock64();
    if (!one) {
      warp_reduce_scatter32(v);
      S.part[warp][lane] = v[0];
#pragma unroll
      for (int s2 = 0; s2 < 32; ++s2) v[s2] = 0.f;
    }
#pragma unroll
    for (int i = 0; i <= MAXK; ++i) {
      if (i > j) break;
#pragma unroll
      for (int q = 0; q < NPT; ++q) {
        const float2 a = V[i][q], e = vj[q];
        v[31 - 2 * i] = fmaf(e.x, a.x, fmaf(e.y, a.y, v[31 - 2 * i]));
        v[30 - 2 * i] = fmaf(e.x, a.y, fmaf(-e.y, a.x, v[30 - 2 * i]));
      }
    }
    warp_reduce_scatter32(v);
    if (tr && j < 16) tr[j * 8 + 2] = clock64();
    S.part[warp][(one ? 0 : 32) + lane] = v[0];
    __syncthreads();
    if (tr && j < 16) tr[j * 8 + 3] = clock64();
    // scalar phase on warp 0 only (the fp64 work and its smem reads are not
    // repeated by every warp); results go through smem behind one barrier
    if (warp == 0)
      coarse_scalar_phase<NT / 32, MAXK>(S, sHc, sGj, j, m, one, hn_prev, lane);
    else if (warp == NT / 32 - 1 && j >= 1)  // idle during the scalar phase: Givens of column j-1
      coarse_givens_col<NT / 32>(S, j, one, lane);
    __syncthreads();
    if (S.stop) {
      k = S.k;
      break;
    }
    float2 vn[NPT];
#pragma unroll
    for (int q = 0; q < NPT; ++q) vn[q] = w[q];
#pragma unroll
    for (int i = 0; i <= MAXK; ++i) {
      if (i > j) break;
      const float2 ci = S.coef[i];
#pragma unroll
      for (int q = 0; q < NPT; ++q) vn[q] = csub(vn[q], cmul(ci, V[i][q]));
    }
    if (tr && j < 16) tr[j * 8 + 5] = clock64();
#pragma unroll
    for (int q = 0; q < NPT; ++q) {
      if (!ok[q]) vn[q] = make_float2(0.f, 0.f);
      vj[q] = vn[q];
    }
#pragma unroll
    for (int q = 0; q < NPT; ++q)
#pragma unroll
      for (int i = 1; i <= MAXK; ++i)
        if (i == j + 1) V[i][q] = vn[q];
    // u_{j+1} into the other tile (its last readers, step j-1, passed barrier 1 of step j)
    float2* sUn = sU2 + ((j + 1) & 1) * tile;
#pragma unroll
    for (int q = 0; q < NPT; ++q)
      if (ok[q]) sUn[ui[q]] = cmul(vn[q], di[q]);
    __syncthreads();
    if (tr && j < 16) tr[j * 8 + 6] = clock64();
  }
  if (k == 0) {
#pragma unroll
    for (int q = 0; q < NPT; ++q)
      if (ok[q]) x[size_t(b) * N + t + q * NT] = make_float2(0.f, 0.f);
    return;
  }
  __syncthreads();
  if (tr) tr[11 * 8 + 0] = clock64();
  if (warp == 0) coarse_backsub_warp<MAXK>(S, k, lane);
  if (t == 0) {
    if (tr) tr[11 * 8 + 1] = clock64();
  }
  __syncthreads();
  if (tr) tr[11 * 8 + 3] = clock64();
  float2 cf[MAXK];
#pragma unroll
  for (int i = 0; i < MAXK; ++i) cf[i] = S.coef[i];
#pragma unroll
  for (int q = 0; q < NPT; ++q) {
    float2 u = make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < MAXK; ++i) u = cadd(u, cmul(cf[i], V[i][q]));
    if (ok[q]) x[size_t(b) * N + t + q * NT] = cmul(u, di[q]);
  }
  if (tr) tr[11 * 8 + 2] = clock64();
}

}  // namespace

bool launch_coarse_small(Context& c, const LevelView& L, int iters, int B, const int* act, const float2* f,
                         float2* x) {
  const int N = L.nx * L.ny;
  if (iters > 15 || N > 8 * 256) return false;
  const size_t smem = sizeof(float2) * size_t(N) * (iters + 2);
  if (smem > 200 * 1024) return false;
  static int attr_set = 0;  // per-device bitmask
  if (!(attr_set & (1 << c.device))) {
    const int mx = 200 * 1024;
    HB_CUDA(cudaFuncSetAttribute(k_coarse_small<256, 1, 15>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    HB_CUDA(cudaFuncSetAttribute(k_coarse_small<256, 2, 15>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    HB_CUDA(cudaFuncSetAttribute(k_coarse_small<256, 4, 15>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    HB_CUDA(cudaFuncSetAttribute(k_coarse_small<256, 8, 15>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    attr_set |= 1 << c.device;
  }
  const int tok = prof_begin(c, PC_COARSE);
  static bool reg_attr = false;
  if (c.opt_coarse_reg && iters <= 10 && N <= 1024) {  // basis in registers (c0: 32^2)
    if (!reg_attr) {
      HB_CUDA(cudaFuncSetAttribute(k_coarse_reg<256, 4, 10>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
      reg_attr = true;
    }
    const size_t su = 2 * sizeof(float2) * size_t(L.nx + 2) * (L.ny + 2);
    launch_pdl(c, k_coarse_reg<256, 4, 10>, dim3(B), dim3(256), su, L, iters, act, f, x);
  } else if (N <= 256) {
    launch_pdl(c, k_coarse_small<256, 1, 15>, dim3(B), dim3(256), smem, L, iters, act, f, x);
  } else if (N <= 512) {
    launch_pdl(c, k_coarse_small<256, 2, 15>, dim3(B), dim3(256), smem, L, iters, act, f, x);
  } else if (N <= 1024) {
    launch_pdl(c, k_coarse_small<256, 4, 15>, dim3(B), dim3(256), smem, L, iters, act, f, x);
  } else {
    launch_pdl(c, k_coarse_small<256, 8, 15>, dim3(B), dim3(256), smem, L, iters, act, f, x);
  }
  prof_end(c, PC_COARSE, tok, double(B) * N * 16.0 + double(N) * 8.0, 0);  // f in, x out; diag
  HB_CUDA(cudaGetLastError());
  static const bool trace = getenv("HB_COARSE_TRACE") != nullptr;
  static long long* dtr = nullptr;
  static int ntr = 0;
  if (trace && ntr < 3) {
    if (!dtr) {
      HB_CUDA(cudaMalloc(&dtr, 16 * 8 * sizeof(long long)));
      HB_CUDA(cudaMemcpyToSymbol(g_coarse_trace, &dtr, sizeof(dtr)));
    }
    long long h[128];
    HB_CUDA(cudaStreamSynchronize(c.stream));
    HB_CUDA(cudaMemcpy(h, dtr, sizeof(h), cudaMemcpyDeviceToHost));
    if (++ntr == 3) {
      fprintf(stderr, "coarse trace (cycles from step start): start acc bfly bar1 scalar update bar2\n");
      for (int j = 0; j <= iters && j < 16; ++j)
        fprintf(stderr, "  j=%2d %6lld %6lld %6lld %6lld %6lld %6lld %6lld\n", j, 0ll, h[j * 8 + 1] - h[j * 8],
                h[j * 8 + 2] - h[j * 8], h[j * 8 + 3] - h[j * 8], h[j * 8 + 4] - h[j * 8], h[j * 8 + 5] - h[j * 8],
                h[j * 8 + 6] - h[j * 8]);
      fprintf(stderr, "  total %lld, least squares %lld, barrier %lld, x %lld (cycles)\n", h[88 + 2] - h[0],
              h[89] - h[88], h[91] - h[89], h[90] - h[91]);

    }
  }
  return true;
}

}  // namespace hb
