// Device-resident restarted flexible GMRES over a block of independent
// columns: the hot loop of block_fgmres (inc/krylov.hpp:83-267) with all
// per-column control (Arnoldi, Givens, convergence, freezing, restarts) on the
// GPU, so the host only replays one CUDA graph per restart cycle.
//
// Basis layout: V [m+1][B][N] and Z [m][B][N] complex64 (slot-major so a
// preconditioner apply on V_j is one contiguous batch).  V_i is stored
// unnormalised with a per-column fp64 scale s_i (V_i = s_i * Vraw_i).
// Solution x and rhs b are complex128; the restart residual b - A x is formed
// in fp64.  Reductions accumulate in fp64; per-CTA
// partials are folded by the last CTA of each column (atomic ticket), which
// also runs the scalar recurrences:
//   MGS  h_ij = <V_i, w> - sum_{k<i} h_kj <V_i, V_k>   (one pass over V, Gram-corrected)
//   Givens with real c, complex s (inc/krylov.hpp:49-64,221-232)
//   stop on |g_{j+1}|/beta0 <= tol, happy breakdown hnorm <= 1e-14 beta0,
//   iters >= max_iters; history: [0] = ||b - A x0||, then |g_{j+1}|.
#include "hb_common.cuh"
#include "hb_internal.h"

#include <algorithm>
#include <mutex>

namespace hb {

struct ColState {
  double beta0;
  int iters, k, hist_len;
  int frozen, converged, breakdown, active;
  int max_it;  // per-column iteration limit (0: the solve's max_iters)
  double cs[kMaxRestart];
  double2 sn[kMaxRestart];
  double2 g[kMaxRestart + 1];
  double2 H[kMaxRestart][kMaxRestart + 1];
  double2 G[kMaxRestart][kMaxRestart];
  double2 hc[kMaxRestart + 1];
  double2 coef[kMaxRestart + 1];
  double scale[kMaxRestart + 1];
};

namespace {

constexpr int KT = 256;           // threads per CTA
constexpr int KNPT = 4;           // nodes per thread per tile
constexpr int KTILE = KT * KNPT;  // nodes per tile
constexpr int KMAXV = 2 * kMaxRestart + 1;

__device__ __forceinline__ double2 zmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 zconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 zsub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 zscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 zdiv(double2 a, double2 b) {
  if (fabs(b.x) >= fabs(b.y)) {
    const double r = b.y / b.x, den = b.x + b.y * r;
    return make_double2((a.x + a.y * r) / den, (a.y - a.x * r) / den);
  }
  const double r = b.x / b.y, den = b.x * r + b.y;
  return make_double2((a.x * r + a.y) / den, (a.y * r - a.x) / den);
}

struct FineView {
  int nx, ny;           // global grid
  double inv_h2;
  const double2* dA64;  // fp64 diagonal of A^h (restart residual)
  const float2* dA;     // fp32 diagonal (A z per inner step)
  RowWin w;             // storage window: vectors are [B][w.rows][nx]; nodes of rows [w.lo, w.hi) are owned
  const float2* dI = nullptr;  // coarse GMRES: D^-1 (the dots kernel applies A D^-1 s_j to Vraw_j itself)
  __device__ __forceinline__ size_t ns() const { return size_t(nx) * w.rows; }         // batch stride
  __device__ __forceinline__ size_t nown() const { return size_t(nx) * (w.hi - w.lo); }  // owned nodes
  __device__ __forceinline__ size_t off() const { return size_t(nx) * (w.lo - w.row0); } // first owned node
};

// Row-slab mode (gsum != nullptr): the per-column fold of the CTA partials is
// written to gsum[b][KMAXV] and the kernel stops there; the caller sums gsum
// over all slabs (NCCL allreduce or the in-process group sum) and launches the
// *_finish kernel, which runs the scalar recurrence on the global sums.  Every
// slab receives the same bits, so the replicated Hessenberg / Givens / flags
// stay identical across slabs.

// Fold the per-CTA partials of column b in its last CTA with every warp at
// once: warp w takes values w, w + 8, ...; lane l sums CTAs l, l + 32, ... in
// order (L2 loads, independent), then a fixed xor butterfly -- deterministic.
// (A serial loop of nblk dependent L2 round trips per value cost ~150 us at
// the end of every Krylov launch at c4, where one column has 592 CTAs.)
__device__ __forceinline__ void fold_parts2(const double2* part, int b, int nblk, int nv, double2* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int t = warp; t < nv; t += KT / 32) {
    double2 s = make_double2(0.0, 0.0);
    for (int q = lane; q < nblk; q += 32) {
      const double2 v = __ldcg(part + (size_t(b) * nblk + q) * KMAXV + t);
      s.x += v.x;
      s.y += v.y;
    }
    s = warp_sum2(s);
    if (lane == 0) out[t] = s;
  }
}
// the same for one double per CTA (part[b][nblk]); warp 0 only, result in lane 0 (all lanes)
__device__ __forceinline__ double fold_parts1(const double* part, int b, int nblk) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int q = lane; q < nblk; q += 32) s += __ldcg(part + size_t(b) * nblk + q);
  return warp_sum(s);
}

// last CTA of column b? (classic threadfence + ticket pattern; resets the ticket)
__device__ bool last_cta(unsigned* ticket, int b, int nblk) {
  __shared__ bool is_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(&ticket[b], 1u);
    is_last = (t == unsigned(nblk - 1));
    if (is_last) ticket[b] = 0;
  }
  __syncthreads();
  return is_last;
}

// r = b - A x (fp64), V0raw = r, ||r||^2 -> restart logic (inc/krylov.hpp:143-188)
__device__ void restart_scalar(ColState& S, int b, double t, double* hist, int hist_cap, double rel_tol,
                               int max_iters, int* act, float* scale_out, int* count);

__global__ void __launch_bounds__(KT) k_restart(FineView F, int B, ColState* st, const double2* __restrict__ bvec,
                                                const double2* __restrict__ x, float2* __restrict__ V0,
                                                double* part, unsigned* ticket, double* hist, int hist_cap,
                                                double rel_tol, int max_iters, int* act, float* scale_out,
                                                int* count, double2* gsum) {
  pdl_enter();
  const int b = blockIdx.y;
  ColState& S = st[b];
  if (S.frozen) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      S.k = 0;
      act[b] = 0;
    }
    return;
  }
  const size_t N = F.ns(), NO = F.nown(), OFF = F.off();
  const double2* xb = x + b * N + OFF;
  const double2* bb = bvec + b * N + OFF;
  const double2* dA64 = F.dA64 + OFF;
  float2* v0 = V0 + b * N + OFF;
  double acc = 0.0;
  for (size_t base = size_t(blockIdx.x) * KTILE; base < NO; base += size_t(gridDim.x) * KTILE) {
#pragma unroll
    for (int q = 0; q < KNPT; ++q) {
      const size_t p = base + q * KT + threadIdx.x;
      if (p >= NO) break;
      const int ix = int(p % F.nx), iy = F.w.lo + int(p / F.nx);  // global row
      double2 nb = make_double2(0.0, 0.0);
      if (ix > 0) nb = dadd(nb, xb[p - 1]);
      if (ix + 1 < F.nx) nb = dadd(nb, xb[p + 1]);
      if (iy > 0) nb = dadd(nb, xb[p - F.nx]);
      if (iy + 1 < F.ny) nb = dadd(nb, xb[p + F.nx]);
      const double2 ax = zsub(zmul(dA64[p], xb[p]), zscale(nb, F.inv_h2));
      const double2 r = zsub(bb[p], ax);
      v0[p] = make_float2(float(r.x), float(r.y));
      acc += r.x * r.x + r.y * r.y;
    }
  }
  acc = warp_sum(acc);
  __shared__ double wp[KT / 32];
  if ((threadIdx.x & 31) == 0) wp[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < KT / 32; ++w) t += wp[w];
    part[size_t(b) * gridDim.x + blockIdx.x] = t;
  }
  if (!last_cta(ticket, b, gridDim.x)) return;
  if (threadIdx.x >= 32) return;
  const double t = fold_parts1(part, b, gridDim.x);
  if (threadIdx.x != 0) return;
  if (gsum) {
    gsum[size_t(b) * KMAXV] = make_double2(t, 0.0);
    return;
  }
  restart_scalar(S, b, t, hist, hist_cap, rel_tol, max_iters, act, scale_out, count);
}

__global__ void k_restart_finish(int B, ColState* st, const double2* gsum, double* hist, int hist_cap,
                                 double rel_tol, int max_iters, int* act, float* scale_out, int* count) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B || st[b].frozen) return;
  restart_scalar(st[b], b, gsum[size_t(b) * KMAXV].x, hist, hist_cap, rel_tol, max_iters, act, scale_out, count);
}

// restart logic on the squared global residual norm t (inc/krylov.hpp:143-188)
__device__ void restart_scalar(ColState& S, int b, double t, double* hist, int hist_cap, double rel_tol,
                               int max_iters, int* act, float* scale_out, int* count) {
  const double beta = sqrt(t);
  S.k = 0;
  S.active = 0;
  if (S.hist_len == 0) {
    S.beta0 = beta;
    if (hist_cap > 0) hist[size_t(b) * hist_cap] = beta;
    S.hist_len = 1;
    if (beta == 0.0) {
      S.frozen = 1;
      S.converged = 1;
    }
  }
  if (!S.frozen) {
    if (beta / S.beta0 <= rel_tol) {
      S.frozen = 1;
      S.converged = 1;
    } else if (S.iters >= (S.max_it > 0 ? S.max_it : max_iters)) {
      S.frozen = 1;
    } else {
      for (int i = 0; i <= kMaxRestart; ++i) S.g[i] = make_double2(0.0, 0.0);
      S.g[0] = make_double2(beta, 0.0);
      S.scale[0] = 1.0 / beta;
      S.active = 1;
    }
  }
  act[b] = S.active;
  scale_out[b] = float(S.scale[0]);
  if (!S.frozen) atomicAdd(count, 1);
}

// warp reduce-scatter of NF floats (NF % 32 == 0): on return lane l holds the
// warp sums of floats [l*NF/32, (l+1)*NF/32) in v[0 .. NF/32)
template <int NF>
__device__ __forceinline__ void warp_reduce_scatter(float (&v)[NF]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int stage = 0; stage < 5; ++stage) {
    const int half = (NF / 2) >> stage;
    const int mask = 16 >> stage;
    const bool upper = (lane & mask) != 0;
#pragma unroll
    for (int k = 0; k < NF / 2; ++k) {
      if (k < half) {
        const float send = upper ? v[k] : v[k + half];
        const float keep = upper ? v[k + half] : v[k];
        v[k] = keep + __shfl_xor_sync(0xffffffffu, send, mask);
      }
    }
  }
}

// CTA sum of per-thread fp32 accumulators acc[0 .. nf) (nf <= NA, runtime):
// transposed through shared memory sred[NA][KT] (dynamic), each warp folds
// slots w, w + 8, ... over the CTA's threads in fp64; out[s] (shared, fp64)
template <int NA>
__device__ __forceinline__ void cta_reduce_acc(const float (&acc)[NA], int nf, float* sred, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int s = 0; s < NA; ++s)
    if (s < nf) sred[s * KT + threadIdx.x] = acc[s];
  __syncthreads();
  for (int s = warp; s < nf; s += KT / 32) {
    double v = 0.0;
#pragma unroll
    for (int k = 0; k < KT / 32; ++k) v += double(sred[s * KT + k * 32 + lane]);
    v = warp_sum(v);
    if (lane == 0) out[s] = v;
  }
  __syncthreads();
}

// w = A Z_j and the partial dots <Vraw_i, w> (i <= j).  (The Gram row
// <Vraw_j, Vraw_k>, k < j, of the Gram-corrected MGS is formed by k_update one
// step earlier, while V_j is still in registers.)  Each thread keeps 2(JM+1)
// fp32 accumulators (JM = the largest j of the instantiation, j <= JM) over
// all of its nodes -- a grid-strided loop, every basis load of a node issued
// before its FMAs -- and the CTA reduces once at the end: one warp
// reduce-scatter of NF floats, warps folded in fp64, CTA partials folded in
// fp64 by the last CTA of the column, which forms the MGS coefficients.
__device__ void adots_scalar(ColState& S, int j, const double2* red);

template <int JM, bool WIDE>
// up to JM = 9 (c0's FGMRES(10)): <= 64 registers, 4 CTAs per SM (measured 2% on the c0 step);
// the 20-32-vector instantiations would spill there
__global__ void __launch_bounds__(KT, (JM <= 9 ? 4 : 1)) k_adots(FineView F, int B, int j, ColState* st, const int* act,
                                              const float2* __restrict__ Z, float2* __restrict__ W,
                                              const float2* __restrict__ V, double2* part, unsigned* ticket,
                                              double2* gsum) {
  constexpr int NF = 2 * (JM + 1);
  pdl_enter();
  const int b = blockIdx.y;
  if (!act[b]) return;
  const size_t NS = F.ns(), N = F.nown(), OFF = F.off();
  const size_t BN = size_t(B) * NS;
  const float2* zb = Z + b * NS + OFF;
  float2* wb = W + b * NS + OFF;
  const float2* dA = F.dA + OFF;
  const float2* Vb = V + OFF + b * NS;
  const float inv_h2 = float(F.inv_h2);
  const float2* dI = F.dI ? F.dI + OFF : nullptr;
  const float sj = dI ? float(st[b].scale[j]) : 1.f;
  float acc[NF];
#pragma unroll
  for (int s = 0; s < NF; ++s) acc[s] = 0.f;
  // U nodes per thread per iteration, all their loads issued before the first
  // store (the compiler may not hoist loads above a possibly aliasing store):
  // few basis vectors leave registers for more nodes in flight.  WIDE: many
  // nodes per thread (large grids); short loops (c0) keep U = 1
  constexpr int U = !WIDE ? 1 : JM <= 1 ? 4 : JM <= 3 ? 2 : 1;
  const size_t stride = size_t(gridDim.x) * KT;
  const unsigned nxu = unsigned(F.nx);
  const bool pow2 = (nxu & (nxu - 1)) == 0 && N <= 0xffffffffull;
  const int nx_sh = 31 - __clz(nxu);
  for (size_t p0 = size_t(blockIdx.x) * KT + threadIdx.x; p0 < N; p0 += stride * U) {
    float2 a[U][JM + 1], w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t p = p0 + u * stride;
      const bool ok = p < N;
#pragma unroll
      for (int i = 0; i <= JM; ++i) a[u][i] = (ok && i <= j) ? ld(Vb + size_t(i) * BN, p) : make_float2(0.f, 0.f);
      w[u] = make_float2(0.f, 0.f);
      if (!ok) continue;
      // global row (ghost rows hold the neighbours); power-of-two widths (every BASELINE grid) by mask / shift
      const int ix = pow2 ? int(unsigned(p) & (nxu - 1)) : int(p % F.nx);
      const int iy = F.w.lo + (pow2 ? int(unsigned(p) >> nx_sh) : int(p / F.nx));
      if (dI) {  // w = A D^-1 (s_j Vraw_j), zb = Vraw_j (coarse GMRES, inc/multigrid.hpp:52-55)
        float2 nb = make_float2(0.f, 0.f);
        if (ix > 0) nb = cadd(nb, cmul(ld(zb, p - 1), ld(dI, p - 1)));
        if (ix + 1 < F.nx) nb = cadd(nb, cmul(ld(zb, p + 1), ld(dI, p + 1)));
        if (iy > 0) nb = cadd(nb, cmul(ld(zb, p - F.nx), ld(dI, p - F.nx)));
        if (iy + 1 < F.ny) nb = cadd(nb, cmul(ld(zb, p + F.nx), ld(dI, p + F.nx)));
        float2 y = cmul(ld(dA, p), cmul(ld(zb, p), ld(dI, p)));
        y.x = fmaf(-inv_h2, nb.x, y.x);
        y.y = fmaf(-inv_h2, nb.y, y.y);
        w[u] = cscale(y, sj);
      } else {
        w[u] = stencil_at_p(zb, p, F.nx, F.ny, ix, iy, ld(dA, p), inv_h2);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t p = p0 + u * stride;
      if (p < N) wb[p] = w[u];
#pragma unroll
      for (int i = 0; i <= JM; ++i) {
        acc[2 * i] = fmaf(a[u][i].x, w[u].x, fmaf(a[u][i].y, w[u].y, acc[2 * i]));
        acc[2 * i + 1] = fmaf(a[u][i].x, w[u].y, fmaf(-a[u][i].y, w[u].x, acc[2 * i + 1]));
      }
    }
  }
  extern __shared__ float sred[];  // [2 (JM + 1)][KT]
  __shared__ double2 red[KMAXV];
  const int nv = j + 1;
  cta_reduce_acc(acc, 2 * nv, sred, reinterpret_cast<double*>(red));
  for (int t = threadIdx.x; t < nv; t += KT) part[(size_t(b) * gridDim.x + blockIdx.x) * KMAXV + t] = red[t];
  if (!last_cta(ticket, b, gridDim.x)) return;
  fold_parts2(part, b, gridDim.x, nv, red);
  __syncthreads();
  if (gsum) {
    for (int t = threadIdx.x; t < nv; t += KT) gsum[size_t(b) * KMAXV + t] = red[t];
    return;
  }
  adots_scalar(st[b], j, red);
}

__global__ void k_adots_finish(int j, ColState* st, const int* act, const double2* gsum) {
  const int b = blockIdx.x;
  if (!act[b]) return;
  __shared__ double2 red[KMAXV];
  for (int t = threadIdx.x; t <= j; t += blockDim.x) red[t] = gsum[size_t(b) * KMAXV + t];
  __syncthreads();
  adots_scalar(st[b], j, red);
}

// MGS coefficients from the global sums red[0..j] = <Vraw_i, w> and the Gram
// rows S.G[i][k] = s_i s_k <Vraw_i, Vraw_k> (k < i <= j; row j written by the
// previous step's k_update).  Called by a whole CTA; red in shared memory.
__device__ void adots_scalar(ColState& S, int j, const double2* red) {
  const int lane = threadIdx.x & 31;
  // stage the Gram rows this step needs, then warp 0 forms the MGS coefficients
  // with lanes in parallel: h_i = s_i <Vraw_i, w> - sum_{k<i} h_k^(cgs) G_ik
  // (first-order Gram correction; G = O(eps32) off the diagonal)
  __shared__ double2 sG[kMaxRestart][kMaxRestart];
  __shared__ double ssc[kMaxRestart + 1];
  for (int t = threadIdx.x; t <= j; t += blockDim.x) ssc[t] = S.scale[t];
  for (int t = threadIdx.x; t < (j + 1) * (j + 1); t += blockDim.x) {
    const int i = t / (j + 1), kk = t % (j + 1);
    if (kk < i) sG[i][kk] = S.G[i][kk];
  }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const double si = lane <= j ? ssc[lane] : 0.0;
  const double2 zero = make_double2(0.0, 0.0);
  const double2 hcgs = lane <= j ? zscale(red[lane], si) : zero;
  double2 h = hcgs;
  for (int kk = 0; kk < j; ++kk) {
    const double2 hk = make_double2(__shfl_sync(0xffffffffu, hcgs.x, kk), __shfl_sync(0xffffffffu, hcgs.y, kk));
    if (lane <= j && kk < lane) h = zsub(h, zmul(hk, sG[lane][kk]));
  }
  if (lane <= j) {
    S.hc[lane] = h;
    S.coef[lane] = zscale(h, si);
  }
}

// V_{j+1}raw = w - sum_i coef_i Vraw_i ; hnorm ; Givens + convergence
// (inc/krylov.hpp:219-254); also the Gram row <Vraw_{j+1}, Vraw_i> (i <= j) for
// the next step's MGS coefficients while V_{j+1} and the V_i are in registers.
// gram: global sums of the Gram row (j+1 entries) or nullptr
__device__ void update_scalar(ColState& S, int b, int j, int m, double t, const double2* gram, int* act, double* hist,
                              int hist_cap, double rel_tol, int max_iters, float* scale_out);

template <int JM, bool WIDE>
__global__ void __launch_bounds__(KT) k_update(FineView F, int B, int j, int m, ColState* st, int* act,
                                               const float2* __restrict__ W, float2* __restrict__ V, double2* part,
                                               unsigned* ticket, double* hist, int hist_cap, double rel_tol,
                                               int max_iters, float* scale_out, double2* gsum) {
  constexpr int NF = 2 * (JM + 1);
  pdl_enter();
  const int b = blockIdx.y;
  if (!act[b]) return;
  ColState& S = st[b];
  const size_t NS = F.ns(), N = F.nown(), OFF = F.off();
  const size_t BN = size_t(B) * NS;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ float2 cf[kMaxRestart + 4];
  for (int i = threadIdx.x; i < kMaxRestart + 4; i += KT)
    cf[i] = i <= j ? make_float2(float(S.coef[i].x), float(S.coef[i].y)) : make_float2(0.f, 0.f);
  __syncthreads();
  const float2* wb = W + OFF + b * NS;
  const float2* Vb = V + OFF + b * NS;
  float2* Vn = V + OFF + size_t(j + 1) * BN + b * NS;
  // need the next Gram row only if the cycle can continue past step j + 1
  const bool gram = j + 1 < m;
  float acc[NF];
#pragma unroll
  for (int s2 = 0; s2 < NF; ++s2) acc[s2] = 0.f;
  double nrm = 0.0;
  constexpr int U = !WIDE ? 1 : JM <= 1 ? 4 : JM <= 3 ? 2 : 1;  // nodes in flight per thread (see k_adots)
  const size_t stride = size_t(gridDim.x) * KT;
  for (size_t p0 = size_t(blockIdx.x) * KT + threadIdx.x; p0 < N; p0 += stride * U) {
    float2 a[U][JM + 1], t[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t p = p0 + u * stride;
      const bool ok = p < N;
#pragma unroll
      for (int i = 0; i <= JM; ++i) a[u][i] = (ok && i <= j) ? ld(Vb + size_t(i) * BN, p) : make_float2(0.f, 0.f);
      t[u] = ok ? ld(wb, p) : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t p = p0 + u * stride;
#pragma unroll
      for (int i = 0; i <= JM; ++i) t[u] = csub(t[u], cmul(cf[i], a[u][i]));  // cf beyond j: zero
      if (p < N) Vn[p] = t[u];
      nrm += dnorm2(t[u]);
      if (gram) {
#pragma unroll
        for (int i = 0; i <= JM; ++i) {  // conj(V_{j+1}) V_i
          acc[2 * i] = fmaf(t[u].x, a[u][i].x, fmaf(t[u].y, a[u][i].y, acc[2 * i]));
          acc[2 * i + 1] = fmaf(t[u].x, a[u][i].y, fmaf(-t[u].y, a[u][i].x, acc[2 * i + 1]));
        }
      }
    }
  }
  nrm = warp_sum(nrm);
  __shared__ double wp[KT / 32];
  if (lane == 0) wp[warp] = nrm;
  extern __shared__ float sred[];  // [2 (JM + 1)][KT]
  __shared__ double2 red[KMAXV];
  const int ng = gram ? j + 1 : 0;
  cta_reduce_acc(acc, 2 * ng, sred, reinterpret_cast<double*>(red));  // (its barriers publish wp)
  double2* myp = part + (size_t(b) * gridDim.x + blockIdx.x) * KMAXV;
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w2 = 0; w2 < KT / 32; ++w2) t += wp[w2];
    myp[0] = make_double2(t, 0.0);
  }
  for (int t = threadIdx.x; t < ng; t += KT) myp[1 + t] = red[t];
  if (!last_cta(ticket, b, gridDim.x)) return;
  fold_parts2(part, b, gridDim.x, ng + 1, red);
  __syncthreads();
  if (gsum) {
    for (int t = threadIdx.x; t <= ng; t += KT) gsum[size_t(b) * KMAXV + t] = red[t];
    return;
  }
  if (threadIdx.x >= 32) return;
  update_scalar(S, b, j, m, red[0].x, gram ? red + 1 : nullptr, act, hist, hist_cap, rel_tol, max_iters, scale_out);
}

__global__ void k_update_finish(int j, int m, ColState* st, int* act, const double2* gsum, double* hist,
                                int hist_cap, double rel_tol, int max_iters, float* scale_out) {
  const int b = blockIdx.x;
  if (!act[b]) return;
  const double2* g = gsum + size_t(b) * KMAXV;
  update_scalar(st[b], b, j, m, g[0].x, j + 1 < m ? g + 1 : nullptr, act, hist, hist_cap, rel_tol, max_iters,
                scale_out);
}

// Givens + convergence on the global squared norm t of V_{j+1}raw (one warp)
__device__ void update_scalar(ColState& S, int b, int j, int m, double t, const double2* gram, int* act, double* hist,
                              int hist_cap, double rel_tol, int max_iters, float* scale_out) {
  const int lane = threadIdx.x & 31;
  const double hnorm = sqrt(t);
  __shared__ double2 hcol[kMaxRestart + 1], ssn[kMaxRestart];
  __shared__ double scs[kMaxRestart];
  if (lane <= j) hcol[lane] = S.hc[lane];
  if (lane < j) {
    scs[lane] = S.cs[lane];
    ssn[lane] = S.sn[lane];
  }
  __syncwarp();
  if (lane == 0) {
    double2* hj = hcol;
    hj[j + 1] = make_double2(hnorm, 0.0);
    for (int i = 0; i < j; ++i) {  // previous rotations (inc/krylov.hpp:221-225)
      const double2 t1 = dadd(zscale(hj[i], scs[i]), zmul(ssn[i], hj[i + 1]));
      hj[i + 1] = dadd(zscale(zmul(zconj(ssn[i]), hj[i]), -1.0), zscale(hj[i + 1], scs[i]));
      hj[i] = t1;
    }
    double c;
    double2 sn;
    {  // make_givens (inc/krylov.hpp:49-64)
      const double2 a = hj[j];
      const double aa = hypot(a.x, a.y), rho = hypot(aa, hnorm);
      if (rho == 0.0) {
        c = 1.0;
        sn = make_double2(0.0, 0.0);
      } else if (aa == 0.0) {
        c = 0.0;
        sn = make_double2(1.0, 0.0);
      } else {
        c = aa / rho;
        sn = zscale(a, hnorm / (rho * aa));
      }
    }
    S.cs[j] = c;
    S.sn[j] = sn;
    hj[j] = dadd(zscale(hj[j], c), zmul(sn, hj[j + 1]));
    hj[j + 1] = make_double2(0.0, 0.0);
    const double2 gj = S.g[j];
    const double2 gj1 = zscale(zmul(zconj(sn), gj), -1.0);
    S.g[j + 1] = gj1;
    S.g[j] = zscale(gj, c);
    S.k = j + 1;
    const int iters = S.iters + 1;
    S.iters = iters;
    const double est = hypot(gj1.x, gj1.y);
    const int hl = S.hist_len;
    if (hl < hist_cap) hist[size_t(b) * hist_cap + hl] = est;
    S.hist_len = hl + 1;
    const double beta0 = S.beta0;
    const bool happy = hnorm <= 1e-14 * beta0;
    if (happy) S.breakdown = 1;
    int active = 1;
    double snext = 0.0;
    if (est / beta0 <= rel_tol || happy) {
      S.converged = 1;
      S.frozen = 1;
      active = 0;
    } else if (iters >= (S.max_it > 0 ? S.max_it : max_iters)) {
      S.frozen = 1;
      active = 0;
    } else if (j + 1 < m) {
      snext = 1.0 / hnorm;
      S.scale[j + 1] = snext;
    } else {
      active = 0;  // cycle end; finalize folds the correction
    }
    S.active = active;
    act[b] = active;
    scale_out[b] = float(active ? snext : 0.0);
  }
  __syncwarp();
  if (lane <= j + 1) S.H[j][lane] = hcol[lane];
  // next step's Gram row G[j+1][i] = s_{j+1} s_i <Vraw_{j+1}, Vraw_i>
  if (gram && S.active && lane <= j) S.G[j + 1][lane] = zscale(gram[lane], S.scale[j + 1] * S.scale[lane]);
}

// y = R^-1 g (back-substitution, inc/krylov.hpp:119-126) into shared y[0..k):
// stage R (upper k x k of the rotated Hessenberg) and g, then warp 0 runs a
// column-sweep back-substitution with lanes in parallel (whole CTA calls)
__device__ void solve_small(const ColState& S, int k, double2 (*sH)[kMaxRestart], double2* y) {
  for (int t = threadIdx.x; t < k * k; t += blockDim.x) {
    const int col = t / k, row = t % k;
    if (row <= col) sH[col][row] = S.H[col][row];
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    double2 g = lane < k ? S.g[lane] : make_double2(0.0, 0.0);
    for (int i = k - 1; i >= 0; --i) {
      double2 yi = make_double2(0.0, 0.0);
      if (lane == i) {
        yi = zdiv(g, sH[i][i]);
        y[i] = yi;
      }
      yi = make_double2(__shfl_sync(0xffffffffu, yi.x, i), __shfl_sync(0xffffffffu, yi.y, i));
      if (lane < i) g = zsub(g, zmul(sH[i][lane], yi));
    }
  }
  __syncthreads();
}

// standard (non-flexible) right-preconditioned GMRES finalize, first half
// (inc/krylov.hpp:127-136): u = sum_i y_i V_i (V_i = s_i Vraw_i) into u (c64);
// fin[b] = 1 for columns with k > 0 -- the caller applies M to u on those and
// adds the result to x (k_add_to_x)
__global__ void __launch_bounds__(KT) k_finalize_v(FineView F, int B, ColState* st, const float2* __restrict__ V,
                                                   float2* __restrict__ u, int* fin) {
  pdl_enter();
  const int b = blockIdx.y;
  const ColState& S = st[b];
  const int k = S.k;
  if (blockIdx.x == 0 && threadIdx.x == 0) fin[b] = k > 0;
  if (k == 0) return;
  __shared__ double2 sH[kMaxRestart][kMaxRestart];  // sH[col][row]
  __shared__ double2 y[kMaxRestart];
  solve_small(S, k, sH, y);
  if (threadIdx.x < k) y[threadIdx.x] = make_double2(y[threadIdx.x].x * S.scale[threadIdx.x],
                                                     y[threadIdx.x].y * S.scale[threadIdx.x]);
  __syncthreads();
  const size_t NS = F.ns(), N = F.nown(), OFF = F.off();
  const size_t BN = size_t(B) * NS;
  for (size_t p = size_t(blockIdx.x) * KT + threadIdx.x; p < N; p += size_t(gridDim.x) * KT) {
    double2 acc = make_double2(0.0, 0.0);
    for (int i = 0; i < k; ++i) {
      const float2 v = ld(V + size_t(i) * BN + b * NS + OFF, p);
      acc.x += y[i].x * double(v.x) - y[i].y * double(v.y);
      acc.y += y[i].x * double(v.y) + y[i].y * double(v.x);
    }
    u[b * NS + OFF + p] = make_float2(float(acc.x), float(acc.y));
  }
}

// x += z on the columns finalised this cycle (second half of the non-flexible finalize)
__global__ void __launch_bounds__(KT) k_add_to_x(FineView F, const int* fin, const float2* __restrict__ z,
                                                 double2* __restrict__ x) {
  pdl_enter();
  const int b = blockIdx.y;
  if (!fin[b]) return;
  const size_t NS = F.ns(), N = F.nown(), OFF = F.off();
  for (size_t p = size_t(blockIdx.x) * KT + threadIdx.x; p < N; p += size_t(gridDim.x) * KT) {
    const float2 v = ld(z + b * NS + OFF, p);
    double2 a = x[b * NS + OFF + p];
    a.x += double(v.x);
    a.y += double(v.y);
    x[b * NS + OFF + p] = a;
  }
}

// y = R^-1 g (back-substitution, inc/krylov.hpp:119-126); x += sum_i y_i Z_i
// KM: the largest k of the instantiation; all k basis loads of a node are
// issued before its fp64 FMAs (the rolled loop serialised one load round trip
// per Z_i: 43% of HBM at c0)
template <int KM>
__global__ void __launch_bounds__(KT) k_finalize(FineView F, int B, ColState* st, const float2* __restrict__ Z,
                                                 double2* __restrict__ x) {
  pdl_enter();
  const int b = blockIdx.y;
  const ColState& S = st[b];
  const int k = S.k;
  if (k == 0) return;
  __shared__ double2 sH[kMaxRestart][kMaxRestart];  // sH[col][row]
  __shared__ double2 y[kMaxRestart];
  solve_small(S, k, sH, y);
  const size_t NS = F.ns(), N = F.nown(), OFF = F.off();
  const size_t BN = size_t(B) * NS;
  const float2* zb = Z + b * NS + OFF;
  for (size_t p = size_t(blockIdx.x) * KT + threadIdx.x; p < N; p += size_t(gridDim.x) * KT) {
    float2 z[KM];
#pragma unroll
    for (int i = 0; i < KM; ++i) z[i] = i < k ? ld(zb + size_t(i) * BN, p) : make_float2(0.f, 0.f);
    double2 acc = x[b * NS + OFF + p];
#pragma unroll
    for (int i = 0; i < KM; ++i) {
      if (i >= k) break;
      acc.x += y[i].x * double(z[i].x) - y[i].y * double(z[i].y);
      acc.y += y[i].x * double(z[i].y) + y[i].y * double(z[i].x);
    }
    x[b * NS + OFF + p] = acc;
  }
}

// coarse GMRES restart from x0 = 0: V_0raw = f (c64), ||f||^2 -> restart logic
__global__ void __launch_bounds__(KT) k_coarse_restart(FineView F, int B, ColState* st, const float2* __restrict__ f,
                                                       float2* __restrict__ V0, double* part, unsigned* ticket,
                                                       double* hist, int hist_cap, int max_iters, int* act,
                                                       float* scale_out, int* count) {
  pdl_enter();
  const int b = blockIdx.y;
  ColState& S = st[b];
  const size_t N = F.nown();
  double acc = 0.0;
  for (size_t p = size_t(blockIdx.x) * KT + threadIdx.x; p < N; p += size_t(gridDim.x) * KT) {
    const float2 v = ld(f + b * N, p);
    V0[b * N + p] = v;
    acc += dnorm2(v);
  }
  acc = warp_sum(acc);
  __shared__ double wp[KT / 32];
  if ((threadIdx.x & 31) == 0) wp[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < KT / 32; ++w) t += wp[w];
    part[size_t(b) * gridDim.x + blockIdx.x] = t;
  }
  if (!last_cta(ticket, b, gridDim.x)) return;
  if (threadIdx.x >= 32) return;
  const double t = fold_parts1(part, b, gridDim.x);
  if (threadIdx.x != 0) return;
  restart_scalar(S, b, t, hist, hist_cap, 1e-300, max_iters, act, scale_out, count);
}

// coarse GMRES finalize: y = R^-1 g; x = D^-1 (sum_i y_i s_i Vraw_i) into the
// c64 output (x0 = 0; inc/krylov.hpp:119-136, M = D^-1)
__global__ void __launch_bounds__(KT) k_coarse_finalize(FineView F, int B, ColState* st, const float2* __restrict__ V,
                                                        float2* __restrict__ x) {
  pdl_enter();
  const int b = blockIdx.y;
  const ColState& S = st[b];
  const int k = S.k;
  const size_t N = F.nown();
  if (k == 0) {
    for (size_t p = size_t(blockIdx.x) * KT + threadIdx.x; p < N; p += size_t(gridDim.x) * KT)
      x[b * N + p] = make_float2(0.f, 0.f);
    return;
  }
  __shared__ double2 sH[kMaxRestart][kMaxRestart];
  __shared__ double2 y[kMaxRestart];
  __shared__ float2 c[kMaxRestart];
  solve_small(S, k, sH, y);
  if (threadIdx.x < k)
    c[threadIdx.x] = make_float2(float(y[threadIdx.x].x * S.scale[threadIdx.x]),
                                 float(y[threadIdx.x].y * S.scale[threadIdx.x]));
  __syncthreads();
  const size_t BN = size_t(B) * N;
  for (size_t p = size_t(blockIdx.x) * KT + threadIdx.x; p < N; p += size_t(gridDim.x) * KT) {
    float2 u = make_float2(0.f, 0.f);
    for (int i = 0; i < k; ++i) u = cadd(u, cmul(c[i], ld(V + size_t(i) * BN + b * N, p)));
    x[b * N + p] = cmul(u, ld(F.dI, p));
  }
}

__global__ void k_init_state(ColState* st, int B, const int* limits) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  ColState& S = st[b];
  S.beta0 = 0.0;
  S.iters = S.k = S.hist_len = 0;
  S.frozen = S.converged = S.breakdown = S.active = 0;
  S.max_it = limits ? limits[b] : 0;
}

FineView fine_view(Context& c) {
  Level& L = *c.levels[0];
  return FineView{L.nx, L.ny, 1.0 / (L.h * L.h), L.dA64.p, L.dA.p, L.win()};
}

// CTAs per column of the basis-streaming kernels (k_adots, k_update): ~4 CTAs
// per SM over the whole batch, each thread covering >= 4 nodes (the per-CTA
// reduction is amortised over the rest of a CTA's nodes)
int nblk_basis(Context& c, size_t N, int B) {
  const size_t want = (N + size_t(KT) * 4 - 1) / (size_t(KT) * 4);
  const size_t cap = std::max<size_t>(1, size_t(4) * c.num_sms / std::max(1, B));
  return int(std::max<size_t>(1, std::min(want, cap)));
}

int nblk_for(Context& c, size_t N, int B) {
  const size_t tiles = (N + KTILE - 1) / KTILE;
  const int cap = std::max(1, 4 * c.num_sms / std::max(1, B));
  return int(std::max<size_t>(1, std::min<size_t>(tiles, size_t(cap))));
}

}  // namespace

struct KScope {
  Context& c;
  int cls, tok;
  double bytes;
  KScope(Context& c_, int cls_, double bytes_ = 0) : c(c_), cls(cls_), tok(prof_begin(c_, cls_)), bytes(bytes_) {}
  ~KScope() { prof_end(c, cls, tok, bytes, 0); }
};

void krylov_alloc(Context& c, int B, int m, int hist_cap, const int* limits) {
  if (m < 1 || m > kMaxRestart) throw HbError{HB_ERR_ARG, "restart must be in [1, 32]"};
  const size_t N = c.levels[0]->N();
  c.kstate.ensure(size_t(B) * sizeof(ColState));
  c.kV.ensure(size_t(m + 1) * B * N);
  c.kZ.ensure(size_t(m) * B * N);
  c.kW.ensure(size_t(B) * N);
  const int nb = std::max(nblk_for(c, N, B), nblk_basis(c, N, B));
  c.kpart.ensure(size_t(B) * nb * KMAXV);
  c.khist.ensure(size_t(B) * std::max(1, hist_cap));
  c.kact.ensure(B);
  c.kscale.ensure(B);
  c.kcount.ensure(1);
  if (c.kticket.n < size_t(B)) {
    c.kticket.ensure(B);
    HB_CUDA(cudaMemsetAsync(c.kticket.p, 0, sizeof(unsigned) * B, c.stream));
  }
  HB_CUDA(cudaMemsetAsync(c.kticket.p, 0, sizeof(unsigned) * B, c.stream));
  k_init_state<<<(B + 127) / 128, 128, 0, c.stream>>>(reinterpret_cast<ColState*>(c.kstate.p), B, limits);
  HB_CUDA(cudaGetLastError());
  c.k_B = B;
  c.k_m = m;
  c.k_hist = hist_cap;
}

// owned nodes of the fine level (whole grid, or this slab's rows)
static size_t owned_nodes(Context& c) {
  const Level& L = *c.levels[0];
  return size_t(L.nx) * (L.hi - L.lo);
}

void launch_fg_restart(Context& c, int B, const double2* b, const double2* x, float2* V0, int hist_cap,
                       double rel_tol, int max_iters, double2* gsum) {
  const size_t N = owned_nodes(c);
  const int nb = nblk_for(c, N, B);
  KScope ks(c, PC_KRYLOV_RESTART, double(B) * N * 40.0 + double(N) * 16.0);  // b, x (c128) in; V0 (c64) out; dA64
  HB_CUDA(cudaMemsetAsync(c.kcount.p, 0, sizeof(int), c.stream));
  launch_pdl(c, k_restart, dim3(nb, B), dim3(KT), 0, fine_view(c), B, reinterpret_cast<ColState*>(c.kstate.p), b, x, V0,
                                               reinterpret_cast<double*>(c.kpart.p), c.kticket.p, c.khist.p,
                                               hist_cap, rel_tol, max_iters, c.kact.p, c.kscale.p, c.kcount.p, gsum);
  HB_CUDA(cudaGetLastError());
}

// the basis-streaming kernels are instantiated for JM = 1, 3, ..., 15, 19, 23, 31
// (the largest j they accept: 2 (JM + 1) fp32 accumulators and JM + 1 basis
// values per thread; odd steps keep the unused registers few)
#define HB_JM_CASE(JMV, KERN, wide, grid, sm, ...)                                   \
  (wide ? launch_jm(c, KERN<JMV, true>, grid, sm, __VA_ARGS__) : launch_jm(c, KERN<JMV, false>, grid, sm, __VA_ARGS__))
#define HB_JM_DISPATCH(j, KERN, wide, grid, ...)                                    \
  do {                                                                              \
    const int jm_ = (j) <= 15 ? ((j) | 1) : (j) <= 19 ? 19 : (j) <= 23 ? 23 : 31;    \
    const size_t sm_ = size_t(2) * (jm_ + 1) * KT * sizeof(float);                  \
    switch (jm_) {                                                                  \
      case 1: HB_JM_CASE(1, KERN, wide, grid, sm_, __VA_ARGS__); break;             \
      case 3: HB_JM_CASE(3, KERN, wide, grid, sm_, __VA_ARGS__); break;             \
      case 5: HB_JM_CASE(5, KERN, wide, grid, sm_, __VA_ARGS__); break;             \
      case 7: HB_JM_CASE(7, KERN, wide, grid, sm_, __VA_ARGS__); break;             \
      case 9: HB_JM_CASE(9, KERN, wide, grid, sm_, __VA_ARGS__); break;             \
      case 11: HB_JM_CASE(11, KERN, wide, grid, sm_, __VA_ARGS__); break;           \
      case 13: HB_JM_CASE(13, KERN, wide, grid, sm_, __VA_ARGS__); break;           \
      case 15: HB_JM_CASE(15, KERN, wide, grid, sm_, __VA_ARGS__); break;           \
      case 19: HB_JM_CASE(19, KERN, wide, grid, sm_, __VA_ARGS__); break;           \
      case 23: HB_JM_CASE(23, KERN, wide, grid, sm_, __VA_ARGS__); break;           \
      default: HB_JM_CASE(31, KERN, wide, grid, sm_, __VA_ARGS__); break;           \
    }                                                                               \
  } while (0)

// PDL launch with dynamic shared memory; opts in once per kernel (static +
// dynamic shared memory may exceed the 48 KB default: adots_scalar stages 16 KB)
// The grid is capped at one full wave: nblk_basis aims at 4 CTAs per SM, but
// an instantiation whose registers allow only 3 would otherwise run 1.33
// waves, the last third of the CTAs at a third of the occupancy (ncu, c0:
// k_adots<5> at 68 registers, 592 CTAs).  The kernels grid-stride over the
// column's nodes and size their partials by gridDim.x, so any nb works.
template <typename... KArgs, typename... Args>
static void launch_jm(Context& c, void (*k)(KArgs...), dim3 grid, size_t smem, Args&&... args) {
  static std::vector<std::pair<const void*, int>> occ;  // (per process; attributes are per function)
  static std::mutex mu;  // column groups launch from several host threads
  int per_sm = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    for (const auto& e : occ)
      if (e.first == reinterpret_cast<const void*>(k)) per_sm = e.second;
    if (!per_sm) {
      HB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      HB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, KT, smem));
      per_sm = std::max(1, per_sm);
      occ.emplace_back(reinterpret_cast<const void*>(k), per_sm);
    }
  }
  if (c.opt_basis_wave && grid.x > 1) {
    const unsigned cap = std::max(1u, unsigned(per_sm * c.num_sms) / std::max(1u, grid.y));
    grid.x = std::min(grid.x, cap);
  }
  launch_pdl(c, k, grid, dim3(KT), smem, std::forward<Args>(args)...);
}

void launch_adots(Context& c, const FineView& F, int B, int j, ColState* st, const int* act, const float2* Zj, float2* w,
                  const float2* V, double2* part, unsigned* ticket, double2* gsum) {
  const size_t N = size_t(F.nx) * (F.w.hi - F.w.lo);
  const int nb = nblk_basis(c, N, B);
  const bool wide = N >= size_t(nb) * KT * 32;  // >= 32 nodes per thread
  HB_JM_DISPATCH(j, k_adots, wide, dim3(nb, B), F, B, j, st, act, Zj, w, V, part, ticket, gsum);
  HB_CUDA(cudaGetLastError());
}
void launch_update(Context& c, const FineView& F, int B, int j, int m, ColState* st, int* act, const float2* w, float2* V,
                   double2* part, unsigned* ticket, double* hist, int hist_cap, double rel_tol, int max_iters,
                   float* scale, double2* gsum) {
  const size_t N = size_t(F.nx) * (F.w.hi - F.w.lo);
  const int nb = nblk_basis(c, N, B);
  const bool wide = N >= size_t(nb) * KT * 32;  // >= 32 nodes per thread
  HB_JM_DISPATCH(j, k_update, wide, dim3(nb, B), F, B, j, m, st, act, w, V, part, ticket, hist, hist_cap, rel_tol,
                 max_iters, scale, gsum);
  HB_CUDA(cudaGetLastError());
}

void launch_fg_adots(Context& c, int B, int j, const float2* Zj, float2* w, const float2* V, double2* gsum) {
  const size_t N = owned_nodes(c);
  KScope ks(c, PC_KRYLOV_DOTS, double(B) * N * (8.0 * (j + 2) + 8.0) + double(N) * 8.0);  // Z_j, V_0..V_j in; w out; dA
  launch_adots(c, fine_view(c), B, j, reinterpret_cast<ColState*>(c.kstate.p), c.kact.p, Zj, w, V, c.kpart.p,
               c.kticket.p, gsum);
}

void launch_fg_update(Context& c, int B, int j, int m, const float2* w, float2* V, int hist_cap, double rel_tol,
                      int max_iters, double2* gsum) {
  const size_t N = owned_nodes(c);
  KScope ks(c, PC_KRYLOV_UPDATE, double(B) * N * (8.0 * (j + 1) + 16.0));  // w, V_0..V_j in; V_{j+1} out
  launch_update(c, fine_view(c), B, j, m, reinterpret_cast<ColState*>(c.kstate.p), c.kact.p, w, V, c.kpart.p,
                c.kticket.p, c.khist.p, hist_cap, rel_tol, max_iters, c.kscale.p, gsum);
}

// non-flexible finalize (inc/krylov.hpp:127-136): u = V y -> caller applies M -> x += M u
void launch_fg_finalize_v(Context& c, int B, const float2* V, float2* u, int* fin) {
  const size_t N = owned_nodes(c);
  const int nb = std::max(1, std::min<int>(int((N + KT - 1) / KT), 4 * c.num_sms / std::max(1, B)));
  KScope ks(c, PC_KRYLOV_FINAL, double(B) * N * (8.0 + 8.0 * c.k_m));  // V_0..V_{k-1} in, u out
  launch_pdl(c, k_finalize_v, dim3(nb, B), dim3(KT), 0, fine_view(c), B, reinterpret_cast<ColState*>(c.kstate.p), V,
             u, fin);
  HB_CUDA(cudaGetLastError());
}
void launch_fg_add_to_x(Context& c, int B, const int* fin, const float2* z, double2* x) {
  const size_t N = owned_nodes(c);
  const int nb = std::max(1, std::min<int>(int((N + KT - 1) / KT), 4 * c.num_sms / std::max(1, B)));
  KScope ks(c, PC_KRYLOV_FINAL, double(B) * N * 40.0);  // z (c64) in, x (c128) in + out
  launch_pdl(c, k_add_to_x, dim3(nb, B), dim3(KT), 0, fine_view(c), fin, z, x);
  HB_CUDA(cudaGetLastError());
}

// scalar halves of the split (row-slab) reductions, on the slab-summed gsum
void launch_fg_restart_finish(Context& c, int B, const double2* gsum, int hist_cap, double rel_tol, int max_iters) {
  c.launches++;
  k_restart_finish<<<(B + 31) / 32, 32, 0, c.stream>>>(B, reinterpret_cast<ColState*>(c.kstate.p), gsum, c.khist.p,
                                                      hist_cap, rel_tol, max_iters, c.kact.p, c.kscale.p, c.kcount.p);
  HB_CUDA(cudaGetLastError());
}
void launch_fg_adots_finish(Context& c, int B, int j, const double2* gsum) {
  c.launches++;
  k_adots_finish<<<B, 64, 0, c.stream>>>(j, reinterpret_cast<ColState*>(c.kstate.p), c.kact.p, gsum);
  HB_CUDA(cudaGetLastError());
}
void launch_fg_update_finish(Context& c, int B, int j, int m, const double2* gsum, int hist_cap, double rel_tol,
                             int max_iters) {
  c.launches++;
  k_update_finish<<<B, 32, 0, c.stream>>>(j, m, reinterpret_cast<ColState*>(c.kstate.p), c.kact.p, gsum, c.khist.p,
                                          hist_cap, rel_tol, max_iters, c.kscale.p);
  HB_CUDA(cudaGetLastError());
}

void launch_fg_finalize(Context& c, int B, int m, const float2* Z, double2* x) {
  const size_t N = owned_nodes(c);
  const int nb = std::max(1, std::min<int>(int((N + KT - 1) / KT), 4 * c.num_sms / std::max(1, B)));
  KScope ks(c, PC_KRYLOV_FINAL, double(B) * N * (32.0 + 8.0 * m));  // x (c128) in+out, Z_0..Z_{k-1} in (upper bound k = m)
  auto* st = reinterpret_cast<ColState*>(c.kstate.p);
  if (m <= 10)
    launch_pdl(c, k_finalize<10>, dim3(nb, B), dim3(KT), 0, fine_view(c), B, st, Z, x);
  else if (m <= 20)
    launch_pdl(c, k_finalize<20>, dim3(nb, B), dim3(KT), 0, fine_view(c), B, st, Z, x);
  else
    launch_pdl(c, k_finalize<kMaxRestart>, dim3(nb, B), dim3(KT), 0, fine_view(c), B, st, Z, x);
  HB_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// Coarsest-level GMRES(k) with D^-1 (coarse_solve_with_op, inc/multigrid.hpp:
// 45-61) on the same multi-CTA Krylov kernels as the fine level, for coarse
// grids too large for one CTA per column (c2: 128^2, c3: 256^2): right
// preconditioning with Z_j = D^-1 V_j is FGMRES with a fixed diagonal
// preconditioner, x0 = 0, tol 1e-300 (fixed budget), happy breakdown as
// krylov.hpp:240.  Operator = the level's shifted M^H (fp64 diagonal for the
// restart residual).  One state set per half-batch stream (slot).

void coarse_krylov_solve(Context& c, const Level& L, int iters, int B, int slot, const float2* f, float2* x) {
  if (iters < 1 || iters > kMaxRestart) throw HbError{HB_ERR_ARG, "coarse GMRES iterations out of range"};
  if (!L.dMi.p) throw HbError{HB_ERR_STATE, "coarsest level lacks D^-1"};
  Context::KrylovBufs& K = c.kcoarse[slot & 1];
  const size_t N = L.N();
  const int m = iters, cap = iters + 2;
  K.state.ensure(size_t(B) * sizeof(ColState));
  K.V.ensure(size_t(m + 1) * B * N);
  K.W.ensure(size_t(B) * N);
  const int nbk = std::max(nblk_for(c, N, B), nblk_basis(c, N, B));
  K.part.ensure(size_t(B) * nbk * KMAXV);
  K.hist.ensure(size_t(B) * cap);
  K.act.ensure(B);
  K.scale.ensure(B);
  K.count.ensure(1);
  if (K.ticket.n < size_t(B)) {
    K.ticket.ensure(B);
    HB_CUDA(cudaMemsetAsync(K.ticket.p, 0, sizeof(unsigned) * B, c.stream));
  }
  FineView F{L.nx, L.ny, 1.0 / (L.h * L.h), L.dM64.p, L.dM.p, L.win()};
  F.dI = L.dMi.p;
  ColState* st = reinterpret_cast<ColState*>(K.state.p);
  const int tok = prof_begin(c, PC_COARSE);
  c.launches += 2 + 2 * m;  // prof_begin counted one of the 3 + 2m kernels below
  k_init_state<<<(B + 127) / 128, 128, 0, c.stream>>>(st, B, nullptr);
  const int nb = nblk_for(c, N, B);
  launch_pdl(c, k_coarse_restart, dim3(nb, B), dim3(KT), 0, F, B, st, f, K.V.p, reinterpret_cast<double*>(K.part.p),
             K.ticket.p, K.hist.p, cap, m, K.act.p, K.scale.p, K.count.p);
  const size_t BN = size_t(B) * N;
  for (int j = 0; j < m; ++j) {
    // w = A D^-1 (s_j Vraw_j) inside the dots kernel (no Z vectors: right
    // preconditioning by a fixed diagonal, non-flexible as inc/multigrid.hpp:50)
    launch_adots(c, F, B, j, st, K.act.p, K.V.p + size_t(j) * BN, K.W.p, K.V.p, K.part.p, K.ticket.p, nullptr);
    launch_update(c, F, B, j, m, st, K.act.p, K.W.p, K.V.p, K.part.p, K.ticket.p, K.hist.p, cap, 1e-300, m, K.scale.p,
                  nullptr);
  }
  const int nf = std::max(1, std::min<int>(int((N + KT - 1) / KT), 4 * c.num_sms / std::max(1, B)));
  launch_pdl(c, k_coarse_finalize, dim3(nf, B), dim3(KT), 0, F, B, st, K.V.p, x);
  // algorithmic bytes: f in, x out (c64) -- the Krylov traffic of the coarse
  // level is accounted like the fine level's (Arnoldi over m steps)
  prof_end(c, PC_COARSE, tok, double(B) * N * 16.0 + double(N) * 8.0, 0);
  HB_CUDA(cudaGetLastError());
}

// report readback helpers (host side of hb_fgmres)
void krylov_report(Context& c, int B, double* hist, int hist_stride, int* hist_len, int* iters, uint8_t* conv,
                   uint8_t* brk) {
  std::vector<ColState> hs(B);
  HB_CUDA(cudaMemcpyAsync(hs.data(), c.kstate.p, sizeof(ColState) * B, cudaMemcpyDeviceToHost, c.stream));
  std::vector<double> hh;
  if (hist && c.k_hist > 0) {
    hh.resize(size_t(B) * c.k_hist);
    HB_CUDA(cudaMemcpyAsync(hh.data(), c.khist.p, sizeof(double) * hh.size(), cudaMemcpyDeviceToHost, c.stream));
  }
  HB_CUDA(cudaStreamSynchronize(c.stream));
  for (int b = 0; b < B; ++b) {
    if (hist_len) hist_len[b] = hs[b].hist_len;
    if (iters) iters[b] = hs[b].iters;
    if (conv) conv[b] = uint8_t(hs[b].converged);
    if (brk) brk[b] = uint8_t(hs[b].breakdown);
    if (hist)
      for (int i = 0; i < std::min(hist_stride, std::min(hs[b].hist_len, c.k_hist)); ++i)
        hist[size_t(b) * hist_stride + i] = hh[size_t(b) * c.k_hist + i];
  }
}

}  // namespace hb
