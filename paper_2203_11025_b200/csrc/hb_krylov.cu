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

// sum a per-warp smem partial table [8][nv] into out[nv] (threads < nv)
__device__ void cta_fold(double2 (*part)[KMAXV], int nv, double2* out) {
  __syncthreads();
  for (int t = threadIdx.x; t < nv; t += KT) {
    double2 s = make_double2(0.0, 0.0);
    for (int w = 0; w < KT / 32; ++w) s = dadd(s, part[w][t]);
    out[t] = s;
  }
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
  if (threadIdx.x != 0) return;
  double t = 0.0;
  for (unsigned q = 0; q < gridDim.x; ++q) t += ((volatile double*)part)[size_t(b) * gridDim.x + q];
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

// w = A Z_j ; partial <Vraw_i, w> (i <= j) and <Vraw_j, Vraw_k> (k < j).
// Basis vectors are streamed in groups of 4 (all 4*KNPT loads in flight
// before use); each group's 4 dot + 4 Gram products are summed in fp32 over
// the thread's nodes and reduced across the warp by one 16-float butterfly,
// the warp partial accumulates in shared memory; warps and CTAs fold in fp64;
// the last CTA of the column forms the MGS coefficients.
__device__ void adots_scalar(ColState& S, int j, const double2* red);

template <int NT, int NPT>  // NPT: nodes per thread per tile (more nodes per butterfly)
__global__ void __launch_bounds__(NT) k_adots(FineView F, int B, int j, ColState* st, const int* act,
                                              const float2* __restrict__ Z, float2* __restrict__ W,
                                              const float2* __restrict__ V, double2* part, unsigned* ticket,
                                              double2* gsum) {
  pdl_enter();
  const int b = blockIdx.y;
  if (!act[b]) return;
  const size_t NS = F.ns(), N = F.nown(), OFF = F.off();
  const size_t BN = size_t(B) * NS;
  const float2* zb = Z + b * NS + OFF;
  float2* wb = W + b * NS + OFF;
  const float2* dA = F.dA + OFF;
  V += OFF;
  const float2* Vj = V + size_t(j) * BN + b * NS;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nv = 2 * j + 1;
  const float inv_h2 = float(F.inv_h2);
  // wpart[warp][float]: dots of basis i at floats 2i, 2i+1; Gram k at 2*kMaxRestart + 2k
  __shared__ float wpart[NT / 32][4 * kMaxRestart + 8];
  for (int t = threadIdx.x; t < (NT / 32) * (4 * kMaxRestart + 8); t += NT) (&wpart[0][0])[t] = 0.f;
  __syncthreads();
  constexpr int TILE = NT * NPT;
  for (size_t base = size_t(blockIdx.x) * TILE; base < N; base += size_t(gridDim.x) * TILE) {
    float2 w[NPT], vj[NPT];
    bool ok[NPT];
#pragma unroll
    for (int q = 0; q < NPT; ++q) {
      const size_t p = base + q * NT + threadIdx.x;
      ok[q] = p < N;
      if (ok[q]) {
        const int ix = int(p % F.nx), iy = F.w.lo + int(p / F.nx);  // global row (ghost rows hold the neighbours)
        w[q] = stencil_at_p(zb, p, F.nx, F.ny, ix, iy, ld(dA, p), inv_h2);
        wb[p] = w[q];
        vj[q] = ld(Vj, p);
      } else {
        w[q] = vj[q] = make_float2(0.f, 0.f);
      }
    }
    for (int i0 = 0; i0 <= j; i0 += 4) {
      float2 a[4][NPT];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float2* Vi = V + size_t(i0 + u) * BN + b * NS;
#pragma unroll
        for (int q = 0; q < NPT; ++q)
          a[u][q] = (ok[q] && i0 + u <= j) ? ld(Vi, base + q * NT + threadIdx.x) : make_float2(0.f, 0.f);
      }
      float v[16];  // [0..7] dots of i0..i0+3, [8..15] Gram
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float dr = 0.f, di = 0.f, gr = 0.f, gi = 0.f;
#pragma unroll
        for (int q = 0; q < NPT; ++q) {
          const float2 ai = a[u][q], c = w[q], e = vj[q];
          dr = fmaf(ai.x, c.x, fmaf(ai.y, c.y, dr));
          di = fmaf(ai.x, c.y, fmaf(-ai.y, c.x, di));
          gr = fmaf(e.x, ai.x, fmaf(e.y, ai.y, gr));
          gi = fmaf(e.x, ai.y, fmaf(-e.y, ai.x, gi));
        }
        v[2 * u] = dr;
        v[2 * u + 1] = di;
        v[8 + 2 * u] = gr;
        v[8 + 2 * u + 1] = gi;
      }
      // 16-float reduce-scatter: 4 halving stages, then a pairwise allreduce
#pragma unroll
      for (int stage = 0; stage < 4; ++stage) {
        const int half = 8 >> stage, mask = 16 >> stage;
        const bool upper = (lane & mask) != 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (k < half) {
            const float send = upper ? v[k] : v[k + half];
            const float keep = upper ? v[k + half] : v[k];
            v[k] = keep + __shfl_xor_sync(0xffffffffu, send, mask);
          }
        }
      }
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
      if ((lane & 1) == 0) {
        const int fidx = lane >> 1;  // float index in the group's 16
        const int u = (fidx & 7) >> 1, comp = fidx & 1;
        const int i = i0 + u;
        if (fidx < 8) {
          if (i <= j) wpart[warp][2 * i + comp] += v[0];
        } else {
          if (i < j) wpart[warp][2 * kMaxRestart + 2 * i + comp] += v[0];
        }
      }
    }
  }
  __syncthreads();
  constexpr int HS = kMaxRestart;
  // fold warps in fp64: slot s <- floats 2s, 2s+1 (dots s <= j at s, Gram k < j at HS + k)
  __shared__ double2 red[KMAXV];
  for (int t = threadIdx.x; t < nv; t += NT) {
    const int slot = t <= j ? t : HS + (t - j - 1);
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll 4
    for (int w2 = 0; w2 < NT / 32; ++w2) {
      acc.x += wpart[w2][2 * slot];
      acc.y += wpart[w2][2 * slot + 1];
    }
    red[t] = acc;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < nv; t += NT) part[(size_t(b) * gridDim.x + blockIdx.x) * KMAXV + t] = red[t];
  if (!last_cta(ticket, b, gridDim.x)) return;
  for (int t = threadIdx.x; t < nv; t += NT) {
    double2 s = make_double2(0.0, 0.0);
    for (unsigned q = 0; q < gridDim.x; ++q) {
      const volatile double2* pp = part + (size_t(b) * gridDim.x + q) * KMAXV + t;
      s.x += pp->x;
      s.y += pp->y;
    }
    red[t] = s;
    if (gsum) gsum[size_t(b) * KMAXV + t] = s;
  }
  if (gsum) return;
  adots_scalar(st[b], j, red);
}

__global__ void k_adots_finish(int j, ColState* st, const int* act, const double2* gsum) {
  const int b = blockIdx.x;
  if (!act[b]) return;
  __shared__ double2 red[KMAXV];
  for (int t = threadIdx.x; t < 2 * j + 1; t += blockDim.x) red[t] = gsum[size_t(b) * KMAXV + t];
  adots_scalar(st[b], j, red);
}

// MGS coefficients from the global sums red[0..j] = <Vraw_i, w>, red[j+1..2j] =
// <Vraw_j, Vraw_k> (called by a whole CTA; red in shared memory)
__device__ void adots_scalar(ColState& S, int j, const double2* red) {
  const int lane = threadIdx.x & 31;
  // stage the Gram rows this step needs, then warp 0 forms the MGS coefficients
  // with lanes in parallel: h_i = s_i <Vraw_i, w> - sum_{k<i} h_k^(cgs) G_ik
  // (first-order Gram correction; G = O(eps32) off the diagonal)
  __shared__ double2 sG[kMaxRestart][kMaxRestart];
  __shared__ double ssc[kMaxRestart + 1];
  for (int t = threadIdx.x; t <= j; t += blockDim.x) ssc[t] = S.scale[t];
  for (int t = threadIdx.x; t < j * j; t += blockDim.x) {
    const int i = t / j, kk = t % j;
    if (kk < i) sG[i][kk] = S.G[i][kk];
  }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const double sj = ssc[j];
  const double si = lane <= j ? ssc[lane] : 0.0;
  const double2 zero = make_double2(0.0, 0.0);
  const double2 hcgs = lane <= j ? zscale(red[lane], si) : zero;
  const double2 gjk = lane < j ? zscale(red[j + 1 + lane], sj * si) : zero;
  if (lane < j) S.G[j][lane] = gjk;
  double2 h = hcgs;
  for (int kk = 0; kk < j; ++kk) {
    const double2 hk = make_double2(__shfl_sync(0xffffffffu, hcgs.x, kk), __shfl_sync(0xffffffffu, hcgs.y, kk));
    const double2 gk = make_double2(__shfl_sync(0xffffffffu, gjk.x, kk), __shfl_sync(0xffffffffu, gjk.y, kk));
    if (lane <= j && kk < lane) h = zsub(h, zmul(hk, lane == j ? gk : sG[lane][kk]));
  }
  if (lane <= j) {
    S.hc[lane] = h;
    S.coef[lane] = zscale(h, si);
  }
}

// V_{j+1}raw = w - sum_i coef_i Vraw_i ; hnorm ; Givens + convergence (inc/krylov.hpp:219-254)
__device__ void update_scalar(ColState& S, int b, int j, int m, double t, int* act, double* hist, int hist_cap,
                              double rel_tol, int max_iters, float* scale_out);

__global__ void __launch_bounds__(KT) k_update(FineView F, int B, int j, int m, ColState* st, int* act,
                                               const float2* __restrict__ W, float2* __restrict__ V, double* part,
                                               unsigned* ticket, double* hist, int hist_cap, double rel_tol,
                                               int max_iters, float* scale_out, double2* gsum) {
  pdl_enter();
  const int b = blockIdx.y;
  if (!act[b]) return;
  ColState& S = st[b];
  const size_t NS = F.ns(), N = F.nown(), OFF = F.off();
  const size_t BN = size_t(B) * NS;
  W += OFF;
  V += OFF;
  __shared__ float2 cf[kMaxRestart + 4];
  for (int i = threadIdx.x; i <= j; i += KT) cf[i] = make_float2(float(S.coef[i].x), float(S.coef[i].y));
  __syncthreads();
  const float2* wb = W + b * NS;
  float2* Vn = V + size_t(j + 1) * BN + b * NS;
  double acc = 0.0;
  for (size_t base = size_t(blockIdx.x) * KTILE; base < N; base += size_t(gridDim.x) * KTILE) {
    float2 t[KNPT];
    bool ok[KNPT];
#pragma unroll
    for (int q = 0; q < KNPT; ++q) {
      const size_t p = base + q * KT + threadIdx.x;
      ok[q] = p < N;
      t[q] = ok[q] ? ld(wb, p) : make_float2(0.f, 0.f);
    }
    for (int i0 = 0; i0 <= j; i0 += 4) {
      float2 a[4][KNPT];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float2* Vi = V + size_t(i0 + u) * BN + b * NS;
#pragma unroll
        for (int q = 0; q < KNPT; ++q)
          a[u][q] = (ok[q] && i0 + u <= j) ? ld(Vi, base + q * KT + threadIdx.x) : make_float2(0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float2 c = (i0 + u <= j) ? cf[i0 + u] : make_float2(0.f, 0.f);
#pragma unroll
        for (int q = 0; q < KNPT; ++q) t[q] = csub(t[q], cmul(c, a[u][q]));
      }
    }
#pragma unroll
    for (int q = 0; q < KNPT; ++q)
      if (ok[q]) {
        Vn[base + q * KT + threadIdx.x] = t[q];
        acc += dnorm2(t[q]);
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
  const int lane = threadIdx.x;
  // warp 0: fold the partial norms, stage rotation state in shared memory
  double t = 0.0;
  for (unsigned q = lane; q < gridDim.x; q += 32) t += ((volatile double*)part)[size_t(b) * gridDim.x + q];
  t = warp_sum(t);
  if (gsum) {
    if (lane == 0) gsum[size_t(b) * KMAXV] = make_double2(t, 0.0);
    return;
  }
  update_scalar(S, b, j, m, t, act, hist, hist_cap, rel_tol, max_iters, scale_out);
}

__global__ void k_update_finish(int j, int m, ColState* st, int* act, const double2* gsum, double* hist,
                                int hist_cap, double rel_tol, int max_iters, float* scale_out) {
  const int b = blockIdx.x;
  if (!act[b]) return;
  update_scalar(st[b], b, j, m, gsum[size_t(b) * KMAXV].x, act, hist, hist_cap, rel_tol, max_iters, scale_out);
}

// Givens + convergence on the global squared norm t of V_{j+1}raw (one warp)
__device__ void update_scalar(ColState& S, int b, int j, int m, double t, int* act, double* hist, int hist_cap,
                              double rel_tol, int max_iters, float* scale_out) {
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
  for (size_t p = size_t(blockIdx.x) * KT + threadIdx.x; p < N; p += size_t(gridDim.x) * KT) {
    double2 acc = x[b * NS + OFF + p];
    for (int i = 0; i < k; ++i) {
      const float2 z = ld(Z + size_t(i) * BN + b * NS + OFF, p);
      acc.x += y[i].x * double(z.x) - y[i].y * double(z.y);
      acc.y += y[i].x * double(z.y) + y[i].y * double(z.x);
    }
    x[b * NS + OFF + p] = acc;
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

// one tile per CTA for small columns (latency), capped for huge columns so the
// last-CTA fold stays short
int nblk_adots(Context& c, size_t N, int B, int tile) {
  const size_t tiles = (N + tile - 1) / tile;
  const size_t cap = std::max<size_t>(16, size_t(4) * c.num_sms / std::max(1, B));
  return int(std::max<size_t>(1, std::min(tiles, cap)));
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
  const int nb = std::max(nblk_for(c, N, B), nblk_adots(c, N, B, 256 * KNPT));
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

void launch_fg_adots(Context& c, int B, int j, const float2* Zj, float2* w, const float2* V, double2* gsum) {
  const size_t N = owned_nodes(c);
  KScope ks(c, PC_KRYLOV_DOTS, double(B) * N * (8.0 * (j + 2) + 8.0) + double(N) * 8.0);  // Z_j, V_0..V_j in; w out; dA
  // same tile as krylov_alloc sized kpart for (nblk_adots(..., 256 * KNPT))
  const int nb = nblk_adots(c, N, B, 256 * KNPT);
  launch_pdl(c, k_adots<256, KNPT>, dim3(nb, B), dim3(256), 0, fine_view(c), B, j,
             reinterpret_cast<ColState*>(c.kstate.p), c.kact.p, Zj, w, V, c.kpart.p, c.kticket.p, gsum);
  HB_CUDA(cudaGetLastError());
}

void launch_fg_update(Context& c, int B, int j, int m, const float2* w, float2* V, int hist_cap, double rel_tol,
                      int max_iters, double2* gsum) {
  const size_t N = owned_nodes(c);
  const int nb = nblk_for(c, N, B);
  KScope ks(c, PC_KRYLOV_UPDATE, double(B) * N * (8.0 * (j + 1) + 16.0));  // w, V_0..V_j in; V_{j+1} out
  launch_pdl(c, k_update, dim3(nb, B), dim3(KT), 0, fine_view(c), B, j, m, reinterpret_cast<ColState*>(c.kstate.p),
                                              c.kact.p, w, V, reinterpret_cast<double*>(c.kpart.p), c.kticket.p,
                                              c.khist.p, hist_cap, rel_tol, max_iters, c.kscale.p, gsum);
  HB_CUDA(cudaGetLastError());
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
  (void)m;
  const size_t N = owned_nodes(c);
  const int nb = std::max(1, std::min<int>(int((N + KT - 1) / KT), 4 * c.num_sms / std::max(1, B)));
  KScope ks(c, PC_KRYLOV_FINAL, double(B) * N * (32.0 + 8.0 * m));  // x (c128) in+out, Z_0..Z_{k-1} in (upper bound k = m)
  launch_pdl(c, k_finalize, dim3(nb, B), dim3(KT), 0, fine_view(c), B, reinterpret_cast<ColState*>(c.kstate.p), Z, x);
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
namespace {
__global__ void k_c64_to_c128(size_t n, const float2* __restrict__ a, double2* __restrict__ b) {
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    b[i] = make_double2(a[i].x, a[i].y);
}
__global__ void k_c128_to_c64(size_t n, const double2* __restrict__ a, float2* __restrict__ b) {
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    b[i] = make_float2(float(a[i].x), float(a[i].y));
}
// Z = D^-1 (s_b V)  (the diagonal "preconditioner" of the coarse GMRES)
__global__ void k_diag_precond(int N, const int* act, const float2* __restrict__ V, const float* scale,
                               const float2* __restrict__ d, float2* __restrict__ Z) {
  const int b = blockIdx.y;
  if (act && !act[b]) return;
  const float s = scale[b];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x)
    Z[size_t(b) * N + i] = cmul(cscale(V[size_t(b) * N + i], s), crcp(__ldg(d + i)));
}
}  // namespace

void coarse_krylov_solve(Context& c, const Level& L, int iters, int B, int slot, const float2* f, float2* x) {
  if (iters < 1 || iters > kMaxRestart) throw HbError{HB_ERR_ARG, "coarse GMRES iterations out of range"};
  if (!L.dM64.p) throw HbError{HB_ERR_STATE, "coarsest level lacks the fp64 M diagonal"};
  Context::KrylovBufs& K = c.kcoarse[slot & 1];
  const size_t N = L.N();
  const int m = iters, cap = iters + 2;
  K.state.ensure(size_t(B) * sizeof(ColState));
  K.V.ensure(size_t(m + 1) * B * N);
  K.Z.ensure(size_t(m) * B * N);
  K.W.ensure(size_t(B) * N);
  K.b.ensure(size_t(B) * N);
  K.x.ensure(size_t(B) * N);
  const int nbk = std::max(nblk_for(c, N, B), nblk_adots(c, N, B, 256 * KNPT));
  K.part.ensure(size_t(B) * nbk * KMAXV);
  K.hist.ensure(size_t(B) * cap);
  K.act.ensure(B);
  K.scale.ensure(B);
  K.count.ensure(1);
  if (K.ticket.n < size_t(B)) {
    K.ticket.ensure(B);
    HB_CUDA(cudaMemsetAsync(K.ticket.p, 0, sizeof(unsigned) * B, c.stream));
  }
  const FineView F{L.nx, L.ny, 1.0 / (L.h * L.h), L.dM64.p, L.dM.p, L.win()};
  ColState* st = reinterpret_cast<ColState*>(K.state.p);
  const size_t BN = size_t(B) * N;
  const int g1 = int(std::min<size_t>((BN + 255) / 256, size_t(c.num_sms) * 8));
  const int tok = prof_begin(c, PC_COARSE);
  c.launches += 4 + 3 * m;  // prof_begin counted one of the 5 + 3m kernels below
  k_init_state<<<(B + 127) / 128, 128, 0, c.stream>>>(st, B, nullptr);
  k_c64_to_c128<<<g1, 256, 0, c.stream>>>(BN, f, K.b.p);
  HB_CUDA(cudaMemsetAsync(K.x.p, 0, sizeof(double2) * BN, c.stream));
  HB_CUDA(cudaMemsetAsync(K.count.p, 0, sizeof(int), c.stream));
  const int nb = nblk_for(c, N, B);
  const double tol = 1e-300;
  launch_pdl(c, k_restart, dim3(nb, B), dim3(KT), 0, F, B, st, K.b.p, K.x.p, K.V.p, reinterpret_cast<double*>(K.part.p),
                                               K.ticket.p, K.hist.p, cap, tol, m, K.act.p, K.scale.p, K.count.p,
                                               (double2*)nullptr);
  const int na = nblk_adots(c, N, B, 256 * KNPT);
  const dim3 gz(unsigned(std::max<size_t>(1, std::min<size_t>((N + 255) / 256, size_t(4) * c.num_sms / B))), B);
  for (int j = 0; j < m; ++j) {
    float2* Vj = K.V.p + size_t(j) * BN;
    float2* Zj = K.Z.p + size_t(j) * BN;
    k_diag_precond<<<gz, 256, 0, c.stream>>>(int(N), K.act.p, Vj, K.scale.p, L.dM.p, Zj);
    launch_pdl(c, k_adots<256, KNPT>, dim3(na, B), dim3(256), 0, F, B, j, st, K.act.p, Zj, K.W.p, K.V.p, K.part.p, K.ticket.p,
               (double2*)nullptr);
    launch_pdl(c, k_update, dim3(nb, B), dim3(KT), 0, F, B, j, m, st, K.act.p, K.W.p, K.V.p,
                                                reinterpret_cast<double*>(K.part.p), K.ticket.p, K.hist.p, cap, tol,
                                                m, K.scale.p, (double2*)nullptr);
  }
  const int nf = std::max(1, std::min<int>(int((N + KT - 1) / KT), 4 * c.num_sms / std::max(1, B)));
  launch_pdl(c, k_finalize, dim3(nf, B), dim3(KT), 0, F, B, st, K.Z.p, K.x.p);
  k_c128_to_c64<<<g1, 256, 0, c.stream>>>(BN, K.x.p, x);
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
