// Multigrid kernels for sm_100a: 5-point complex Helmholtz / shifted-Laplacian
// stencil (inc/stencil.hpp:44-60), damped Jacobi (:78-92), residual + full-
// weighting restriction with offset (:69-75,119-140), bilinear prolongation
// with offset (:146-165), and the coarsest-level GMRES(k) with D^-1
// (inc/multigrid.hpp:45-61) as one CTA-resident kernel per right-hand side.
//
// Layout: complex64 (float2) fields, row-major [batch][ny][nx]; one thread per
// node, 32x8 CTAs, blockIdx.z = column.  Coefficients (the diagonal d = 4/h^2 +
// mass term) are per level, shared by all columns.
#include "hb_common.cuh"
#include "hb_internal.h"

namespace hb {

namespace {

constexpr int TBX = 32, TBY = 8;

__device__ __forceinline__ bool col_active(const int* act, int b) { return act == nullptr || act[b] != 0; }
__device__ __forceinline__ float col_scale(const float* s, int b) { return s ? s[b] : 1.0f; }

__global__ void __launch_bounds__(TBX* TBY) k_apply(LevelView L, int which, const int* act, const float2* __restrict__ u,
                                                   float2* __restrict__ y, const float* uscale) {
  const int b = blockIdx.z;
  if (!col_active(act, b)) return;
  const int ix = blockIdx.x * TBX + threadIdx.x, iy = blockIdx.y * TBY + threadIdx.y;
  if (ix >= L.nx || iy >= L.ny) return;
  const size_t N = size_t(L.nx) * L.ny, i = size_t(iy) * L.nx + ix;
  const float2* d = which ? L.dM : L.dA;
  y[b * N + i] = stencil_at(u + b * N, L.nx, L.ny, ix, iy, ld(d, i), L.inv_h2, col_scale(uscale, b));
}

// v = damping * f / d   (one Jacobi sweep from a zero iterate)
__global__ void __launch_bounds__(TBX* TBY) k_jacobi_zero(LevelView L, float damping, const int* act,
                                                         const float2* __restrict__ f, const float* fscale,
                                                         float2* __restrict__ v) {
  const int b = blockIdx.z;
  if (!col_active(act, b)) return;
  const int ix = blockIdx.x * TBX + threadIdx.x, iy = blockIdx.y * TBY + threadIdx.y;
  if (ix >= L.nx || iy >= L.ny) return;
  const size_t N = size_t(L.nx) * L.ny, i = size_t(iy) * L.nx + ix;
  const float2 fi = cscale(ld(f, b * N + i), col_scale(fscale, b));
  v[b * N + i] = cscale(cmul(fi, crcp(ld(L.dM, i))), damping);
}

// out = v + damping * (f - M v) / d
__global__ void __launch_bounds__(TBX* TBY) k_jacobi_sweep(LevelView L, float damping, const int* act,
                                                          const float2* __restrict__ v, const float2* __restrict__ f,
                                                          const float* fscale, float2* __restrict__ out) {
  const int b = blockIdx.z;
  if (!col_active(act, b)) return;
  const int ix = blockIdx.x * TBX + threadIdx.x, iy = blockIdx.y * TBY + threadIdx.y;
  if (ix >= L.nx || iy >= L.ny) return;
  const size_t N = size_t(L.nx) * L.ny, i = size_t(iy) * L.nx + ix;
  const float2 d = ld(L.dM, i);
  const float2 av = stencil_at(v + b * N, L.nx, L.ny, ix, iy, d, L.inv_h2, 1.0f);
  const float2 fi = cscale(ld(f, b * N + i), col_scale(fscale, b));
  const float2 corr = cmul(csub(fi, av), crcp(d));
  out[b * N + i] = caxpy(ld(v, b * N + i), damping, corr);
}

// out = s f - Op u, Op the 5-point operator with diagonal L.dM
__global__ void __launch_bounds__(TBX* TBY) k_residual(LevelView L, const int* act, const float2* __restrict__ u,
                                                      const float2* __restrict__ f, const float* fscale,
                                                      float2* __restrict__ out) {
  const int b = blockIdx.z;
  if (!col_active(act, b)) return;
  const int ix = blockIdx.x * TBX + threadIdx.x, iy = blockIdx.y * TBY + threadIdx.y;
  if (ix >= L.nx || iy >= L.ny) return;
  const size_t N = size_t(L.nx) * L.ny, i = size_t(iy) * L.nx + ix;
  const float2 au = stencil_at(u + b * N, L.nx, L.ny, ix, iy, ld(L.dM, i), L.inv_h2, 1.0f);
  out[b * N + i] = csub(cscale(ld(f, b * N + i), col_scale(fscale, b)), au);
}

// fc(j) = sum_k w_k (f - M v)(2j + o + k), w = [1 2 1]x[1 2 1]/16, out-of-range skipped
__global__ void __launch_bounds__(TBX* TBY) k_residual_restrict(LevelView L, int offset, const int* act,
                                                               const float2* __restrict__ v,
                                                               const float2* __restrict__ f, const float* fscale,
                                                               float2* __restrict__ fc) {
  const int b = blockIdx.z;
  if (!col_active(act, b)) return;
  const int cnx = L.nx / 2, cny = L.ny / 2;
  const int jx = blockIdx.x * TBX + threadIdx.x, jy = blockIdx.y * TBY + threadIdx.y;
  if (jx >= cnx || jy >= cny) return;
  const size_t N = size_t(L.nx) * L.ny;
  const float2* vb = v + b * N;
  const float2* fb = f + b * N;
  const float s = col_scale(fscale, b);
  float2 acc = make_float2(0.f, 0.f);
#pragma unroll
  for (int ky = -1; ky <= 1; ++ky) {
    const int iy = 2 * jy + offset + ky;
    if (iy < 0 || iy >= L.ny) continue;
#pragma unroll
    for (int kx = -1; kx <= 1; ++kx) {
      const int ix = 2 * jx + offset + kx;
      if (ix < 0 || ix >= L.nx) continue;
      const size_t i = size_t(iy) * L.nx + ix;
      const float2 r = csub(cscale(ld(fb, i), s), stencil_at(vb, L.nx, L.ny, ix, iy, ld(L.dM, i), L.inv_h2, 1.0f));
      const float w = float((kx == 0 ? 2 : 1) * (ky == 0 ? 2 : 1)) * (1.0f / 16.0f);
      acc = caxpy(acc, w, r);
    }
  }
  fc[size_t(b) * cnx * cny + size_t(jy) * cnx + jx] = acc;
}

// plain restriction of a field (test hook)
__global__ void k_restrict(int nx, int ny, int offset, const float2* __restrict__ fine, float2* __restrict__ coarse) {
  const int b = blockIdx.z;
  const int cnx = nx / 2, cny = ny / 2;
  const int jx = blockIdx.x * TBX + threadIdx.x, jy = blockIdx.y * TBY + threadIdx.y;
  if (jx >= cnx || jy >= cny) return;
  const float2* fb = fine + size_t(b) * nx * ny;
  float2 acc = make_float2(0.f, 0.f);
  for (int ky = -1; ky <= 1; ++ky) {
    const int iy = 2 * jy + offset + ky;
    if (iy < 0 || iy >= ny) continue;
    for (int kx = -1; kx <= 1; ++kx) {
      const int ix = 2 * jx + offset + kx;
      if (ix < 0 || ix >= nx) continue;
      const float w = float((kx == 0 ? 2 : 1) * (ky == 0 ? 2 : 1)) * (1.0f / 16.0f);
      acc = caxpy(acc, w, ld(fb, size_t(iy) * nx + ix));
    }
  }
  coarse[size_t(b) * cnx * cny + size_t(jy) * cnx + jx] = acc;
}

// v(i) += sum_j vc(j) * w(i - 2j - o), gathered: per axis, t = x - o - k even
// and 0 <= t/2 < cn contributes with 1-D weight {0.5, 1, 0.5}[k+1]
__device__ __forceinline__ int prolong_taps(int x, int o, int cn, int* j, float* w) {
  int n = 0;
  const int t0 = x - o;
  if ((t0 & 1) == 0) {
    const int jj = t0 >> 1;
    if (jj >= 0 && jj < cn) {
      j[n] = jj;
      w[n++] = 1.0f;
    }
  } else {
    const int ja = (t0 - 1) >> 1, jb = (t0 + 1) >> 1;  // k = +1, k = -1
    if (ja >= 0 && ja < cn) {
      j[n] = ja;
      w[n++] = 0.5f;
    }
    if (jb >= 0 && jb < cn) {
      j[n] = jb;
      w[n++] = 0.5f;
    }
  }
  return n;
}

__device__ __forceinline__ float2 prolong_at(const float2* __restrict__ vc, int cnx, int cny, int offset, int ix,
                                             int iy) {
  int jx[2], jy[2];
  float wx[2], wy[2];
  const int nxs = prolong_taps(ix, offset, cnx, jx, wx);
  const int nys = prolong_taps(iy, offset, cny, jy, wy);
  float2 acc = make_float2(0.f, 0.f);
  for (int a = 0; a < nys; ++a)
    for (int c = 0; c < nxs; ++c) acc = caxpy(acc, wx[c] * wy[a], ld(vc, size_t(jy[a]) * cnx + jx[c]));
  return acc;
}

__global__ void __launch_bounds__(TBX* TBY) k_prolong_add(int nx, int ny, int cnx, int cny, int offset,
                                                         const int* act, const float2* __restrict__ vc,
                                                         float2* __restrict__ v) {
  const int b = blockIdx.z;
  if (!col_active(act, b)) return;
  const int ix = blockIdx.x * TBX + threadIdx.x, iy = blockIdx.y * TBY + threadIdx.y;
  if (ix >= nx || iy >= ny) return;
  const size_t i = size_t(b) * nx * ny + size_t(iy) * nx + ix;
  v[i] = cadd(v[i], prolong_at(vc + size_t(b) * cnx * cny, cnx, cny, offset, ix, iy));
}

// ------------------------------------------------------------------------
// Coarsest-level GMRES(k): non-flexible, right-preconditioned with D^-1,
// x0 = 0, rel_tol 1e-300 (fixed budget; happy breakdown only), exactly the
// contract of coarse_solve_with_op (inc/multigrid.hpp:45-61) running through
// block_fgmres (inc/krylov.hpp:83-267, finalize :132-137).  One CTA per
// column; basis vectors in global scratch (L2-resident), kept unnormalised
// with per-vector scales s_i.  MGS coefficients are formed from one fused
// reduction pass via the Gram recurrence
//   h_ij = <V_i, w> - sum_{k<i} h_kj <V_i, V_k>     (= MGS in exact arithmetic)
// and ||w - sum h_ij V_i|| is then reduced directly.
constexpr int CG_THREADS = 1024;
constexpr int CG_WARPS = CG_THREADS / 32;
constexpr int CG_MAXV = 2 * kMaxCoarseIters + 1;

struct CoarseSmem {
  double2 part[CG_WARPS][CG_MAXV];
  double2 red[CG_MAXV];
  double2 H[kMaxCoarseIters][kMaxCoarseIters + 1];
  double2 G[kMaxCoarseIters][kMaxCoarseIters];  // G[i][k] = <V_i, V_k>, k < i
  double2 hc[kMaxCoarseIters + 1];              // MGS coefficients of the current column
  double2 sn[kMaxCoarseIters];
  double cs[kMaxCoarseIters];
  double2 g[kMaxCoarseIters + 1];
  double2 y[kMaxCoarseIters];
  double scale[kMaxCoarseIters + 1];
  float coef[kMaxCoarseIters + 1][2];
  double normpart[CG_WARPS];
  double beta0;
  int stop, k;
};

__device__ void cg_make_givens(double2 a, double b, double* c, double2* s) {
  const double aa = hypot(a.x, a.y);
  const double rho = hypot(aa, b);
  if (rho == 0.0) {
    *c = 1.0;
    *s = make_double2(0.0, 0.0);
  } else if (aa == 0.0) {
    *c = 0.0;
    *s = make_double2(1.0, 0.0);
  } else {
    *c = aa / rho;
    const double f = b / (rho * aa);
    *s = make_double2(a.x * f, a.y * f);
  }
}
__device__ __forceinline__ double2 zmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 zconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 zsub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 zscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 zdiv(double2 a, double2 b) {
  // Smith's algorithm (as __divdc3)
  if (fabs(b.x) >= fabs(b.y)) {
    const double r = b.y / b.x, den = b.x + b.y * r;
    return make_double2((a.x + a.y * r) / den, (a.y - a.x * r) / den);
  }
  const double r = b.x / b.y, den = b.x * r + b.y;
  return make_double2((a.x * r + a.y) / den, (a.y * r - a.x) / den);
}

__global__ void __launch_bounds__(CG_THREADS, 1) k_coarse_gmres(LevelView L, int m, const int* act,
                                                               const float2* __restrict__ f, float2* __restrict__ x,
                                                               float2* __restrict__ scratch) {
  const int b = blockIdx.x;
  if (!col_active(act, b)) return;
  __shared__ CoarseSmem S;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nx = L.nx, ny = L.ny;
  const size_t N = size_t(nx) * ny;
  const float2* fb = f + b * N;
  float2* Vb = scratch + size_t(b) * (m + 2) * N;  // V_1..V_m raw (V_0 raw = f), then z
  float2* zb = Vb + size_t(m + 1) * N;
  auto V = [&](int i) -> const float2* { return i == 0 ? fb : Vb + size_t(i) * N; };

  // beta = ||f||
  double acc = 0.0;
  for (size_t p = tid; p < N; p += CG_THREADS) acc += dnorm2(ld(fb, p));
  acc = warp_sum(acc);
  if (lane == 0) S.normpart[warp] = acc;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < CG_WARPS; ++w) t += S.normpart[w];
    const double beta = sqrt(t);
    S.beta0 = beta;
    S.stop = beta == 0.0;
    S.scale[0] = beta > 0.0 ? 1.0 / beta : 0.0;
    for (int i = 0; i <= m; ++i) S.g[i] = make_double2(0.0, 0.0);
    S.g[0] = make_double2(beta, 0.0);
    S.k = 0;
  }
  __syncthreads();
  if (S.stop) {
    for (size_t p = tid; p < N; p += CG_THREADS) x[b * N + p] = make_float2(0.f, 0.f);
    return;
  }
  for (int j = 0; j < m; ++j) {
    // z = D^-1 V_j
    const float sj = float(S.scale[j]);
    const float2* Vj = V(j);
    for (size_t p = tid; p < N; p += CG_THREADS) zb[p] = cmul(cscale(Vj[p], sj), crcp(ld(L.dM, p)));
    __syncthreads();
    // w = M z (stored in V_{j+1} raw slot), fused partial dots
    float2* w = Vb + size_t(j + 1) * N;
    for (size_t p = tid; p < N; p += CG_THREADS) {
      const int ix = int(p % nx), iy = int(p / nx);
      w[p] = stencil_at(zb, nx, ny, ix, iy, ld(L.dM, p), L.inv_h2, 1.0f);
    }
    // (each thread reads back only its own w entries: no barrier needed)
    const int nv = 2 * j + 1;
    for (int i = 0; i <= j; ++i) {
      const float2* Vi = V(i);
      double2 a = make_double2(0.0, 0.0);
      for (size_t p = tid; p < N; p += CG_THREADS) a = dadd(a, dconjmul(Vi[p], w[p]));
      a = warp_sum2(a);
      if (lane == 0) S.part[warp][i] = a;
    }
    for (int k = 0; k < j; ++k) {
      const float2* Vk = V(k);
      double2 a = make_double2(0.0, 0.0);
      for (size_t p = tid; p < N; p += CG_THREADS) a = dadd(a, dconjmul(Vj[p], Vk[p]));
      a = warp_sum2(a);
      if (lane == 0) S.part[warp][j + 1 + k] = a;
    }
    __syncthreads();
    if (tid < nv) {
      double2 t = make_double2(0.0, 0.0);
      for (int w2 = 0; w2 < CG_WARPS; ++w2) t = dadd(t, S.part[w2][tid]);
      S.red[tid] = t;
    }
    __syncthreads();
    if (tid == 0) {
      for (int k = 0; k < j; ++k) S.G[j][k] = zscale(S.red[j + 1 + k], S.scale[j] * S.scale[k]);
      for (int i = 0; i <= j; ++i) {
        double2 h = zscale(S.red[i], S.scale[i]);
        for (int k = 0; k < i; ++k) h = zsub(h, zmul(S.hc[k], S.G[i][k]));
        S.hc[i] = h;
        const double2 c = zscale(h, S.scale[i]);
        S.coef[i][0] = float(c.x);
        S.coef[i][1] = float(c.y);
      }
    }
    __syncthreads();
    // w <- w - sum_i h_ij V_i ; ||w||
    acc = 0.0;
    for (size_t p = tid; p < N; p += CG_THREADS) {
      float2 t = w[p];
      for (int i = 0; i <= j; ++i) {
        const float2 vi = V(i)[p];
        const float2 c = make_float2(S.coef[i][0], S.coef[i][1]);
        t = csub(t, cmul(c, vi));
      }
      w[p] = t;
      acc += dnorm2(t);
    }
    acc = warp_sum(acc);
    if (lane == 0) S.normpart[warp] = acc;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w2 = 0; w2 < CG_WARPS; ++w2) t += S.normpart[w2];
      const double hnorm = sqrt(t);
      double2* hj = S.H[j];
      for (int i = 0; i <= j; ++i) hj[i] = S.hc[i];
      hj[j + 1] = make_double2(hnorm, 0.0);
      for (int i = 0; i < j; ++i) {  // previous rotations (inc/krylov.hpp:221-225)
        const double2 t1 = dadd(zscale(hj[i], S.cs[i]), zmul(S.sn[i], hj[i + 1]));
        hj[i + 1] = dadd(zscale(zmul(zconj(S.sn[i]), hj[i]), -1.0), zscale(hj[i + 1], S.cs[i]));
        hj[i] = t1;
      }
      cg_make_givens(hj[j], hnorm, &S.cs[j], &S.sn[j]);
      hj[j] = dadd(zscale(hj[j], S.cs[j]), zmul(S.sn[j], hj[j + 1]));
      hj[j + 1] = make_double2(0.0, 0.0);
      S.g[j + 1] = zscale(zmul(zconj(S.sn[j]), S.g[j]), -1.0);
      S.g[j] = zscale(S.g[j], S.cs[j]);
      S.k = j + 1;
      const bool happy = hnorm <= 1e-14 * S.beta0;
      S.stop = happy || (j + 1 >= m);
      S.scale[j + 1] = hnorm > 0.0 ? 1.0 / hnorm : 0.0;
    }
    __syncthreads();
    if (S.stop) break;
  }
  // finalize: y = R^-1 g ; x = D^-1 (sum_i y_i V_i)
  if (tid == 0) {
    const int k = S.k;
    for (int i = k - 1; i >= 0; --i) {
      double2 sum = S.g[i];
      for (int l = i + 1; l < k; ++l) sum = zsub(sum, zmul(S.H[l][i], S.y[l]));
      S.y[i] = zdiv(sum, S.H[i][i]);
    }
    for (int i = 0; i < k; ++i) {
      const double2 c = zscale(S.y[i], S.scale[i]);
      S.coef[i][0] = float(c.x);
      S.coef[i][1] = float(c.y);
    }
  }
  __syncthreads();
  const int k = S.k;
  for (size_t p = tid; p < N; p += CG_THREADS) {
    float2 u = make_float2(0.f, 0.f);
    for (int i = 0; i < k; ++i) u = cadd(u, cmul(make_float2(S.coef[i][0], S.coef[i][1]), V(i)[p]));
    x[b * N + p] = cmul(u, crcp(ld(L.dM, p)));
  }
}

inline dim3 grid2(int nx, int ny, int B) { return dim3((nx + TBX - 1) / TBX, (ny + TBY - 1) / TBY, B); }

}  // namespace

struct ProfScope {
  Context& c;
  int cls, tok;
  double bytes, flops;
  ProfScope(Context& c_, int cls_, double bytes_ = 0, double flops_ = 0)
      : c(c_), cls(cls_), tok(prof_begin(c_, cls_)), bytes(bytes_), flops(flops_) {}
  ~ProfScope() { prof_end(c, cls, tok, bytes, flops); }
};

void launch_apply(Context& c, const LevelView& L, int which, int B, const int* act, const float2* u, float2* y,
                  const float* uscale) {
  ProfScope ps(c, PC_STENCIL, double(B) * L.nx * L.ny * 24.0);
  k_apply<<<grid2(L.nx, L.ny, B), dim3(TBX, TBY), 0, c.stream>>>(L, which, act, u, y, uscale);
  HB_CUDA(cudaGetLastError());
}

void launch_jacobi_zero(Context& c, const LevelView& L, float damping, int B, const int* act, const float2* f,
                        const float* fscale, float2* v) {
  ProfScope ps(c, PC_SMOOTH, double(B) * L.nx * L.ny * 24.0);
  k_jacobi_zero<<<grid2(L.nx, L.ny, B), dim3(TBX, TBY), 0, c.stream>>>(L, damping, act, f, fscale, v);
  HB_CUDA(cudaGetLastError());
}

void launch_residual(Context& c, const LevelView& L, int B, const int* act, const float2* u, const float2* f,
                     const float* fscale, float2* out) {
  ProfScope ps(c, PC_SMOOTH, double(B) * L.nx * L.ny * 24.0);
  k_residual<<<grid2(L.nx, L.ny, B), dim3(TBX, TBY), 0, c.stream>>>(L, act, u, f, fscale, out);
  HB_CUDA(cudaGetLastError());
}

void launch_jacobi_sweep(Context& c, const LevelView& L, float damping, int B, const int* act, const float2* v,
                         const float2* f, const float* fscale, float2* out) {
  ProfScope ps(c, PC_SMOOTH, double(B) * L.nx * L.ny * 32.0);
  k_jacobi_sweep<<<grid2(L.nx, L.ny, B), dim3(TBX, TBY), 0, c.stream>>>(L, damping, act, v, f, fscale, out);
  HB_CUDA(cudaGetLastError());
}

void launch_residual_restrict(Context& c, const LevelView& L, int offset, int B, const int* act, const float2* v,
                              const float2* f, const float* fscale, float2* fc) {
  ProfScope ps(c, PC_TRANSFER, double(B) * L.nx * L.ny * 26.0);
  k_residual_restrict<<<grid2(L.nx / 2, L.ny / 2, B), dim3(TBX, TBY), 0, c.stream>>>(L, offset, act, v, f, fscale,
                                                                                     fc);
  HB_CUDA(cudaGetLastError());
}

void launch_prolong_add(Context& c, const LevelView& Lf, int cnx, int cny, int offset, int B, const int* act,
                        const float2* vc, float2* v) {
  ProfScope ps(c, PC_TRANSFER, double(B) * Lf.nx * Lf.ny * 18.0);
  k_prolong_add<<<grid2(Lf.nx, Lf.ny, B), dim3(TBX, TBY), 0, c.stream>>>(Lf.nx, Lf.ny, cnx, cny, offset, act, vc, v);
  HB_CUDA(cudaGetLastError());
}

void launch_restrict_plain(Context& c, int nx, int ny, int offset, int B, const float2* fine, float2* coarse) {
  ProfScope ps(c, PC_TRANSFER);
  k_restrict<<<grid2(nx / 2, ny / 2, B), dim3(TBX, TBY), 0, c.stream>>>(nx, ny, offset, fine, coarse);
  HB_CUDA(cudaGetLastError());
}

// CoarseSolver::dense (inc/multigrid.hpp:84,95-104): x = (M^H)^-1 f with the
// inverse formed on the host (fp64 LU with partial pivoting, setup) and applied
// here as a dense fp64 matvec; one warp per row, lanes stride the columns
__global__ void __launch_bounds__(256) k_coarse_dense(int n, const int* act, const double2* __restrict__ inv,
                                                      const float2* __restrict__ f, float2* __restrict__ x) {
  const int b = blockIdx.y;
  if (act && !act[b]) return;
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= n) return;
  const double2* a = inv + size_t(row) * n;
  const float2* fb = f + size_t(b) * n;
  double re = 0.0, im = 0.0;
  for (int j = lane; j < n; j += 32) {
    const double2 m = a[j];
    const float2 v = fb[j];
    re += m.x * double(v.x) - m.y * double(v.y);
    im += m.x * double(v.y) + m.y * double(v.x);
  }
  for (int o = 16; o; o >>= 1) {
    re += __shfl_xor_sync(0xffffffffu, re, o);
    im += __shfl_xor_sync(0xffffffffu, im, o);
  }
  if (lane == 0) x[size_t(b) * n + row] = make_float2(float(re), float(im));
}

void launch_coarse_dense(Context& c, const Level& L, int B, const int* act, const float2* f, float2* x) {
  if (!L.dinv.p) throw HbError{HB_ERR_STATE, "dense coarse solver: inverse not built"};
  const int n = int(L.N());
  ProfScope ps(c, PC_COARSE, double(B) * n * 16.0 + double(n) * n * 16.0);
  k_coarse_dense<<<dim3((n + 7) / 8, B), 256, 0, c.stream>>>(n, act, L.dinv.p, f, x);
  HB_CUDA(cudaGetLastError());
}

void launch_coarse_gmres(Context& c, const LevelView& L, int iters, int B, const int* act, const float2* f,
                         float2* x, float2* scratch) {
  if (iters < 1 || iters > kMaxCoarseIters) throw HbError{HB_ERR_ARG, "coarse_iters must be in [1, 16]"};
  ProfScope ps(c, PC_COARSE);
  k_coarse_gmres<<<B, CG_THREADS, 0, c.stream>>>(L, iters, act, f, x, scratch);
  HB_CUDA(cudaGetLastError());
}

}  // namespace hb
