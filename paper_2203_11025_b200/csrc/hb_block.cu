// True block flexible GMRES (the reference's
// block_fgmres runs its columns as independent Arnoldi processes in lockstep,
// inc/krylov.hpp:78-82, and lists a true block method as a non-goal,
// SPEC.md:280; the paper's block-size study is PAPER.md:580).  All p
// right-hand sides share ONE block Krylov space:
//
//   restart:  R = B - A X (fp64),  R = V_0 S  (CholQR2)
//   step j:   Z_j = M V_j (the context's preconditioner, p columns at once),
//             W = A Z_j,
//             block CGS2:  H_{0..j, j} = V^H W,  W -= V H  (twice),
//             W = V_{j+1} H_{j+1, j}  (CholQR2: Gram, Cholesky, W R^-1, twice),
//             Givens QR of the new block column of the (m+1)p x mp block
//             Hessenberg (complex rotations, real cosine), the same rotations
//             on the p right-hand-side columns E = [S; 0];
//             per-column residual estimate = || E[(j+1)p : (j+2)p, c] ||
//   end:      Y = R^-1 E[0 : kp],  X += [Z_0 .. Z_{k-1}] Y  (fp64)
// stopping when every column's estimate is <= rel_tol * ||b_c|| (or on
// max_iters block steps, or when W loses rank: breakdown).  Vectors are c64,
// every inner product accumulates in fp64 across CTAs in a fixed order
// (deterministic), the small dense algebra runs in fp64 on one CTA.
#include <algorithm>
#include <cmath>
#include <vector>

#include "hb_common.cuh"
#include "hb_internal.h"

namespace hb {
namespace {

constexpr int BK_NT = 256;
constexpr int BK_MAXP = 16;  // block size
constexpr int BK_MAXM = 20;  // restart (block steps)
constexpr int BK_QT = 4, BK_PT = 8;

__device__ __forceinline__ double2 zmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 zconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 zsub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 zscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double zabs2(double2 a) { return a.x * a.x + a.y * a.y; }
__device__ __forceinline__ double2 zdiv(double2 a, double2 b) {
  const double d = zabs2(b);
  return make_double2((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
}

template <int NF>
__device__ __forceinline__ void warp_scatter(float (&v)[NF]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int stage = 0; stage < 5; ++stage) {
    const int half = (NF / 2) >> stage, mask = 16 >> stage;
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

// partial Gram of a node chunk: part[chunk][i][c] = sum conj(X_i) Y_c, i < q, c < p
// (X, Y: vectors of N nodes, consecutive with stride N)
__global__ void __launch_bounds__(BK_NT) k_bgram(int N, int q, int p, const float2* __restrict__ X,
                                                 const float2* __restrict__ Y, double2* __restrict__ part) {
  const int i0 = blockIdx.y * BK_QT, c0 = blockIdx.z * BK_PT;
  float acc[2 * BK_QT * BK_PT];
#pragma unroll
  for (int s = 0; s < 2 * BK_QT * BK_PT; ++s) acc[s] = 0.f;
  for (int n = blockIdx.x * BK_NT + threadIdx.x; n < N; n += gridDim.x * BK_NT) {
    float2 x[BK_QT], y[BK_PT];
#pragma unroll
    for (int u = 0; u < BK_QT; ++u) x[u] = i0 + u < q ? ld(X + size_t(i0 + u) * N, n) : make_float2(0.f, 0.f);
#pragma unroll
    for (int v = 0; v < BK_PT; ++v) y[v] = c0 + v < p ? ld(Y + size_t(c0 + v) * N, n) : make_float2(0.f, 0.f);
#pragma unroll
    for (int u = 0; u < BK_QT; ++u)
#pragma unroll
      for (int v = 0; v < BK_PT; ++v) {
        float* a = acc + 2 * (u * BK_PT + v);
        a[0] = fmaf(x[u].x, y[v].x, fmaf(x[u].y, y[v].y, a[0]));
        a[1] = fmaf(x[u].x, y[v].y, fmaf(-x[u].y, y[v].x, a[1]));
      }
  }
  warp_scatter<2 * BK_QT * BK_PT>(acc);  // lane l: floats 2l, 2l + 1 (one complex entry)
  __shared__ float wt[BK_NT / 32][64];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  wt[warp][2 * lane] = acc[0];
  wt[warp][2 * lane + 1] = acc[1];
  __syncthreads();
  if (threadIdx.x < BK_QT * BK_PT) {
    const int u = threadIdx.x / BK_PT, v = threadIdx.x % BK_PT;
    double2 s = make_double2(0.0, 0.0);
    for (int w = 0; w < BK_NT / 32; ++w) {
      s.x += wt[w][2 * threadIdx.x];
      s.y += wt[w][2 * threadIdx.x + 1];
    }
    if (i0 + u < q && c0 + v < p) part[(size_t(blockIdx.x) * q + i0 + u) * p + c0 + v] = s;
  }
}

// G[i][c] = sum over chunks (fixed order)
__global__ void k_bfold(int nchunk, int q, int p, const double2* __restrict__ part, double2* __restrict__ G) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= q * p) return;
  double2 s = make_double2(0.0, 0.0);
  for (int k = 0; k < nchunk; ++k) {
    const double2 v = part[size_t(k) * q * p + t];
    s.x += v.x;
    s.y += v.y;
  }
  G[t] = s;
}

// Y_c = beta Y_c + alpha sum_i C[i][c] X_i  (c < p; C fp64 -> fp32 in shared memory)
__global__ void __launch_bounds__(BK_NT) k_bupdate(int N, int q, int p, const float2* __restrict__ X,
                                                   const double2* __restrict__ C, float beta, float alpha, float2* Y) {
  extern __shared__ float2 sc[];  // [q][p]
  for (int t = threadIdx.x; t < q * p; t += BK_NT) sc[t] = make_float2(float(alpha * C[t].x), float(alpha * C[t].y));
  __syncthreads();
  for (int n = blockIdx.x * BK_NT + threadIdx.x; n < N; n += gridDim.x * BK_NT) {
    float2 y[BK_MAXP];
#pragma unroll
    for (int c = 0; c < BK_MAXP; ++c)
      y[c] = (c < p && beta != 0.f) ? cscale(Y[size_t(c) * N + n], beta) : make_float2(0.f, 0.f);
    for (int i = 0; i < q; ++i) {
      const float2 x = ld(X + size_t(i) * N, n);
#pragma unroll
      for (int c = 0; c < BK_MAXP; ++c)
        if (c < p) y[c] = cadd(y[c], cmul(sc[i * p + c], x));
    }
#pragma unroll
    for (int c = 0; c < BK_MAXP; ++c)
      if (c < p) Y[size_t(c) * N + n] = y[c];
  }
}

// X_c += sum_i C[i][c] Z_i in fp64 (the solution update)
__global__ void __launch_bounds__(BK_NT) k_bupdate64(int N, int q, int p, const float2* __restrict__ Z,
                                                     const double2* __restrict__ C, double2* X) {
  for (int n = blockIdx.x * BK_NT + threadIdx.x; n < N; n += gridDim.x * BK_NT) {
    double2 y[BK_MAXP];
#pragma unroll
    for (int c = 0; c < BK_MAXP; ++c) y[c] = c < p ? X[size_t(c) * N + n] : make_double2(0.0, 0.0);
    for (int i = 0; i < q; ++i) {
      const float2 z = ld(Z + size_t(i) * N, n);
      const double2 zd = make_double2(z.x, z.y);
#pragma unroll
      for (int c = 0; c < BK_MAXP; ++c)
        if (c < p) y[c] = dadd(y[c], zmul(C[i * p + c], zd));
    }
#pragma unroll
    for (int c = 0; c < BK_MAXP; ++c)
      if (c < p) X[size_t(c) * N + n] = y[c];
  }
}

// R = B - A X in fp64 (A = A^h of level 0), stored as c64
__global__ void k_bresidual(int nx, int ny, double inv_h2, const double2* __restrict__ dA, const double2* __restrict__ B,
                            const double2* __restrict__ X, float2* __restrict__ R) {
  const int b = blockIdx.y;
  const size_t N = size_t(nx) * ny;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < N; i += size_t(gridDim.x) * blockDim.x) {
    const int ix = int(i % nx), iy = int(i / nx);
    const double2* x = X + b * N;
    double2 nb = make_double2(0.0, 0.0);
    if (ix > 0) nb = dadd(nb, x[i - 1]);
    if (ix + 1 < nx) nb = dadd(nb, x[i + 1]);
    if (iy > 0) nb = dadd(nb, x[i - nx]);
    if (iy + 1 < ny) nb = dadd(nb, x[i + nx]);
    const double2 ax = zsub(zmul(dA[i], x[i]), zscale(nb, inv_h2));
    const double2 r = zsub(B[b * N + i], ax);
    R[b * N + i] = make_float2(float(r.x), float(r.y));
  }
}

// small dense state of one block solve (device, fp64)
struct BlockState {
  double2 H[(BK_MAXM + 1) * BK_MAXP][BK_MAXM * BK_MAXP];  // block Hessenberg, row-major [row][col]
  double2 E[(BK_MAXM + 1) * BK_MAXP][BK_MAXP];             // rotated right-hand sides
  double rc[BK_MAXM * BK_MAXP][BK_MAXP];                   // Givens cosines of column (jp + c), row pairs
  double2 rs[BK_MAXM * BK_MAXP][BK_MAXP];                  // Givens sines
  double2 Rt[BK_MAXP][BK_MAXP];                            // accumulated CholQR2 factor
  double2 Ri[BK_MAXP][BK_MAXP];                            // inverse of the last Cholesky factor
  double beta0[BK_MAXP];
  int k, stop, breakdown, converged;
};

// Cholesky of the p x p Gram G (Hermitian) into upper R (G = R^H R) and R^-1;
// Rt <- R Rt (first == 1: Rt <- R).  One thread.
__global__ void k_bchol(int p, const double2* __restrict__ G, BlockState* S, int first, double2* Rinv) {
  if (threadIdx.x != 0) return;
  double2 R[BK_MAXP][BK_MAXP];
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j) R[i][j] = make_double2(0.0, 0.0);
  double gmax = 0.0;
  for (int i = 0; i < p; ++i) gmax = fmax(gmax, G[i * p + i].x);
  if (!(gmax > 0.0)) {  // a zero block (b = 0): zero factor, zero basis
    for (int i = 0; i < p * p; ++i) Rinv[i] = make_double2(0.0, 0.0);
    for (int i = 0; i < p; ++i)
      for (int j = 0; j < p; ++j) S->Rt[i][j] = make_double2(0.0, 0.0);
    S->breakdown = 1;
    return;
  }
  for (int j = 0; j < p; ++j) {
    double d = G[j * p + j].x;
    for (int k = 0; k < j; ++k) d -= zabs2(R[k][j]);
    if (!(d > 1e-24 * gmax) || gmax <= 0.0) {  // rank loss: block breakdown
      S->breakdown = 1;
      d = fmax(d, 1e-300);
    }
    const double rjj = sqrt(d);
    R[j][j] = make_double2(rjj, 0.0);
    for (int i = j + 1; i < p; ++i) {
      double2 s = G[j * p + i];  // G[j][i] = <w_j, w_i>
      for (int k = 0; k < j; ++k) s = zsub(s, zmul(zconj(R[k][j]), R[k][i]));
      R[j][i] = zscale(s, 1.0 / rjj);
    }
  }
  // R^-1 (upper) by back-substitution, column by column
  double2 Ri[BK_MAXP][BK_MAXP];
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j) Ri[i][j] = make_double2(0.0, 0.0);
  for (int c = 0; c < p; ++c) {
    Ri[c][c] = make_double2(1.0 / R[c][c].x, 0.0);
    for (int i = c - 1; i >= 0; --i) {
      double2 s = make_double2(0.0, 0.0);
      for (int k = i + 1; k <= c; ++k) s = dadd(s, zmul(R[i][k], Ri[k][c]));
      Ri[i][c] = zscale(s, -1.0 / R[i][i].x);
    }
  }
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j) Rinv[i * p + j] = Ri[i][j];
  double2 T[BK_MAXP][BK_MAXP];
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j) {
      if (first) {
        T[i][j] = R[i][j];
      } else {
        double2 s = make_double2(0.0, 0.0);
        for (int k = 0; k < p; ++k) s = dadd(s, zmul(R[i][k], S->Rt[k][j]));
        T[i][j] = s;
      }
    }
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j) S->Rt[i][j] = T[i][j];
}

// restart: E = [Rt; 0], reset the Hessenberg; beta0 on the first restart; history
__global__ void k_brestart(int p, int m, BlockState* S, int first, double* hist, int hist_cap, int* hist_len) {
  const int c = threadIdx.x;
  for (int t = threadIdx.x; t < (m + 1) * p * p; t += blockDim.x) (&S->E[0][0])[(t / p) * BK_MAXP + t % p] = make_double2(0.0, 0.0);
  __syncthreads();
  if (c < p) {
    for (int i = 0; i < p; ++i) S->E[i][c] = S->Rt[i][c];
    double nr = 0.0;
    for (int i = 0; i < p; ++i) nr += zabs2(S->Rt[i][c]);
    nr = sqrt(nr);
    if (first) {
      S->beta0[c] = nr;
      hist[size_t(c) * hist_cap] = nr;
      hist_len[c] = 1;
    }
  }
  if (threadIdx.x == 0) {
    S->k = 0;
    S->stop = 0;
  }
}

// new block column j of H from the CGS2 coefficients (Hc1 + Hc2, (j+1)p x p) and
// the CholQR2 factor Rt; previous rotations, new rotations, E, estimates
__global__ void k_bstep(int p, int j, const double2* __restrict__ Hc1, const double2* __restrict__ Hc2, BlockState* S,
                        double rel_tol, int iters_done, int max_iters, double* hist, int hist_cap, int* hist_len,
                        int* status) {
  const int t = threadIdx.x;
  const int col = j * p + t;  // this thread's column of H
  if (t < p) {
    for (int i = 0; i < (j + 1) * p; ++i) S->H[i][col] = dadd(Hc1[i * p + t], Hc2[i * p + t]);
    for (int i = 0; i < p; ++i) S->H[(j + 1) * p + i][col] = S->Rt[i][t];
    // previous block columns' rotations, in order
    for (int cc = 0; cc < j * p; ++cc)
      for (int r = 0; r < p; ++r) {
        const int row = cc + p - r;  // rotation r of column cc acts on rows (row - 1, row)
        const double c = S->rc[cc][r];
        const double2 s = S->rs[cc][r];
        const double2 u = S->H[row - 1][col], v = S->H[row][col];
        S->H[row - 1][col] = dadd(zscale(u, c), zmul(s, v));
        S->H[row][col] = dadd(zscale(zmul(zconj(s), u), -1.0), zscale(v, c));
      }
  }
  __syncthreads();
  // rotations of this block's columns, one column at a time
  for (int c = 0; c < p; ++c) {
    const int cc = j * p + c;
    if (t == 0) {
      for (int r = 0; r < p; ++r) {  // zero rows cc + p .. cc + 1 bottom-up
        const int row = cc + p - r;
        const double2 a = S->H[row - 1][cc], b = S->H[row][cc];
        const double aa = sqrt(zabs2(a)), bb = sqrt(zabs2(b)), rho = hypot(aa, bb);
        double cs;
        double2 sn;
        if (rho == 0.0) {
          cs = 1.0;
          sn = make_double2(0.0, 0.0);
        } else if (aa == 0.0) {
          cs = 0.0;
          sn = zscale(zconj(b), 1.0 / bb);
        } else {
          cs = aa / rho;
          sn = zscale(zmul(a, zconj(b)), 1.0 / (aa * rho));
        }
        S->rc[cc][r] = cs;
        S->rs[cc][r] = sn;
        S->H[row - 1][cc] = dadd(zscale(a, cs), zmul(sn, b));
        S->H[row][cc] = make_double2(0.0, 0.0);
      }
    }
    __syncthreads();
    if (t > c && t < p) {  // later columns of this block
      for (int r = 0; r < p; ++r) {
        const int row = cc + p - r;
        const double cs = S->rc[cc][r];
        const double2 sn = S->rs[cc][r], u = S->H[row - 1][j * p + t], v = S->H[row][j * p + t];
        S->H[row - 1][j * p + t] = dadd(zscale(u, cs), zmul(sn, v));
        S->H[row][j * p + t] = dadd(zscale(zmul(zconj(sn), u), -1.0), zscale(v, cs));
      }
    }
    if (t < p) {  // right-hand side column t
      for (int r = 0; r < p; ++r) {
        const int row = cc + p - r;
        const double cs = S->rc[cc][r];
        const double2 sn = S->rs[cc][r], u = S->E[row - 1][t], v = S->E[row][t];
        S->E[row - 1][t] = dadd(zscale(u, cs), zmul(sn, v));
        S->E[row][t] = dadd(zscale(zmul(zconj(sn), u), -1.0), zscale(v, cs));
      }
    }
    __syncthreads();
  }
  // per-column residual estimates: the part of E below the triangular rows
  __shared__ int nconv;
  if (t == 0) nconv = 0;
  __syncthreads();
  if (t < p) {
    double e = 0.0;
    for (int i = 0; i < p; ++i) e += zabs2(S->E[(j + 1) * p + i][t]);
    e = sqrt(e);
    const int hl = hist_len[t];
    if (hl < hist_cap) hist[size_t(t) * hist_cap + hl] = e;
    hist_len[t] = hl + 1;
    if (e <= rel_tol * S->beta0[t]) atomicAdd(&nconv, 1);
  }
  __syncthreads();
  if (t == 0) {
    S->k = j + 1;
    const bool all = nconv == p;
    S->converged = all;
    const int st = all ? 1 : (S->breakdown ? 3 : (iters_done >= max_iters ? 2 : 0));
    S->stop = st != 0;
    *status = st;
  }
}

// Y = R^-1 E[0 : kp] (back-substitution on the rotated Hessenberg), one thread per column
__global__ void k_bsolve(int p, BlockState* S, double2* Y) {
  const int c = threadIdx.x;
  if (c >= p) return;
  const int n = S->k * p;
  for (int i = n - 1; i >= 0; --i) {
    double2 s = S->E[i][c];
    for (int l = i + 1; l < n; ++l) s = zsub(s, zmul(S->H[i][l], Y[l * p + c]));
    Y[i * p + c] = zdiv(s, S->H[i][i]);
  }
}

}  // namespace

struct BlockBufs {
  DBuf<float2> V, Z, W;
  DBuf<double2> part, G, Hc1, Hc2, Rinv, Y, X, Bd;
  DBuf<char> state;
  DBuf<double> hist;
  DBuf<int> hist_len, status;
};

// host driver (one sync per block step: the stop decision)
void block_fgmres_dev(Context& c, int kind, int p, int m, int max_iters, double rel_tol, const double2* dB,
                      double2* dX, double* hist_out, int hist_stride, int* hist_len_out, int* iters_out,
                      uint8_t* conv_out, uint8_t* brk_out) {
  if (p < 1 || p > BK_MAXP) throw HbError{HB_ERR_ARG, "block FGMRES: block size must be in [1, 16]"};
  if (m < 1 || m > BK_MAXM) throw HbError{HB_ERR_ARG, "block FGMRES: restart must be in [1, 20]"};
  if (!(rel_tol > 0.0 && rel_tol < 1.0)) throw HbError{HB_ERR_ARG, "rel_tol in (0,1)"};
  ensure_batch(c, p);
  Level& L0 = *c.levels[0];
  const int N = int(L0.N());
  static BlockBufs* bufs = nullptr;  // per process; contexts are used by one host thread each
  if (!bufs) bufs = new BlockBufs;
  BlockBufs& K = *bufs;
  const int q_max = (m + 1) * p;
  K.V.ensure(size_t(m + 1) * p * N);
  K.Z.ensure(size_t(m) * p * N);
  K.W.ensure(size_t(p) * N);
  const int nchunk = std::max(1, std::min(2 * c.num_sms, (N + BK_NT * 8 - 1) / (BK_NT * 8)));
  K.part.ensure(size_t(nchunk) * q_max * p);
  K.G.ensure(size_t(q_max) * p);
  K.Hc1.ensure(size_t(q_max) * p);
  K.Hc2.ensure(size_t(q_max) * p);
  K.Rinv.ensure(size_t(p) * p);
  K.Y.ensure(size_t(m * p) * p);
  K.state.ensure(sizeof(BlockState));
  const int cap = max_iters + 2;
  K.hist.ensure(size_t(p) * cap);
  K.hist_len.ensure(p);
  K.status.ensure(1);
  BlockState* S = reinterpret_cast<BlockState*>(K.state.p);
  HB_CUDA(cudaMemsetAsync(K.state.p, 0, sizeof(BlockState), c.stream));
  const LevelView LV = L0.view();
  auto gram = [&](const float2* X, int q, const float2* Y, double2* G) {
    const dim3 g(nchunk, (q + BK_QT - 1) / BK_QT, (p + BK_PT - 1) / BK_PT);
    k_bgram<<<g, BK_NT, 0, c.stream>>>(N, q, p, X, Y, K.part.p);
    k_bfold<<<(q * p + 255) / 256, 256, 0, c.stream>>>(nchunk, q, p, K.part.p, G);
    c.launches += 2;
  };
  auto update = [&](const float2* X, int q, const double2* C, float beta, float alpha, float2* Y) {
    const size_t smem = sizeof(float2) * size_t(q) * p;
    k_bupdate<<<std::min(4 * c.num_sms, (N + BK_NT - 1) / BK_NT), BK_NT, smem, c.stream>>>(N, q, p, X, C, beta, alpha,
                                                                                         Y);
    c.launches++;
  };
  static bool attr = false;
  if (!attr) {
    HB_CUDA(cudaFuncSetAttribute(k_bupdate, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    attr = true;
  }
  // CholQR2 of the p columns at Vp (in place, through the scratch W), the
  // factor accumulated in S->Rt (W_in = Vp_out Rt)
  auto cholqr2 = [&](float2* Vp) {
    for (int pass = 0; pass < 2; ++pass) {
      gram(Vp, p, Vp, K.G.p);
      k_bchol<<<1, 32, 0, c.stream>>>(p, K.G.p, S, pass == 0 ? 1 : 0, K.Rinv.p);
      update(Vp, p, K.Rinv.p, 0.f, 1.f, K.W.p);
      HB_CUDA(cudaMemcpyAsync(Vp, K.W.p, sizeof(float2) * size_t(p) * N, cudaMemcpyDeviceToDevice, c.stream));
      c.launches++;
    }
  };
  int iters = 0, st = 0;
  bool first = true;
  std::vector<int> hl(p);
  while (true) {
    // R = B - A X (fp64) into V_0, then V_0 S = R
    k_bresidual<<<dim3(std::max(1, std::min(2 * c.num_sms, (N + 255) / 256)), p), 256, 0, c.stream>>>(
        L0.nx, L0.ny, 1.0 / (L0.h * L0.h), L0.dA64.p, dB, dX, K.V.p);
    c.launches++;
    cholqr2(K.V.p);
    k_brestart<<<1, 64, 0, c.stream>>>(p, m, S, first ? 1 : 0, K.hist.p, cap, K.hist_len.p);
    c.launches++;
    if (first) {  // a zero right-hand-side block: X = X0 is the solution
      first = false;
      std::vector<double> b0(p);
      HB_CUDA(cudaMemcpyAsync(b0.data(), &S->beta0[0], sizeof(double) * p, cudaMemcpyDeviceToHost, c.stream));
      HB_CUDA(cudaStreamSynchronize(c.stream));
      if (*std::max_element(b0.begin(), b0.end()) == 0.0) {
        st = 1;
        break;
      }
    }
    int j = 0;
    for (; j < m; ++j) {
      float2* Vj = K.V.p + size_t(j) * p * N;
      float2* Zj = K.Z.p + size_t(j) * p * N;
      precond_apply_dev(c, kind, p, nullptr, Vj, nullptr, Zj);
      launch_apply(c, LV, 0, p, nullptr, Zj, K.W.p, nullptr);  // W = A Z_j
      // block CGS2 against V_0 .. V_j: W -= V (V^H W), twice
      const int q = (j + 1) * p;
      gram(K.V.p, q, K.W.p, K.Hc1.p);
      update(K.V.p, q, K.Hc1.p, 1.f, -1.f, K.W.p);
      gram(K.V.p, q, K.W.p, K.Hc2.p);
      update(K.V.p, q, K.Hc2.p, 1.f, -1.f, K.W.p);
      // W = V_{j+1} Rt
      float2* Vn = K.V.p + size_t(j + 1) * p * N;
      HB_CUDA(cudaMemcpyAsync(Vn, K.W.p, sizeof(float2) * size_t(p) * N, cudaMemcpyDeviceToDevice, c.stream));
      cholqr2(Vn);
      ++iters;
      k_bstep<<<1, 32, 0, c.stream>>>(p, j, K.Hc1.p, K.Hc2.p, S, rel_tol, iters, max_iters, K.hist.p, cap,
                                      K.hist_len.p, K.status.p);
      c.launches++;
      HB_CUDA(cudaMemcpyAsync(&st, K.status.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
      HB_CUDA(cudaStreamSynchronize(c.stream));
      if (st) break;
    }
    // X += Z Y
    if (j == 0 && st == 1 && iters == 0) break;
    k_bsolve<<<1, 32, 0, c.stream>>>(p, S, K.Y.p);
    const int kk = std::min(j + 1, m);
    k_bupdate64<<<std::min(4 * c.num_sms, (N + BK_NT - 1) / BK_NT), BK_NT, 0, c.stream>>>(N, kk * p, p, K.Z.p, K.Y.p,
                                                                                          dX);
    c.launches += 2;
    if (st) break;
  }
  // report
  std::vector<double> hh(size_t(p) * cap);
  HB_CUDA(cudaMemcpyAsync(hh.data(), K.hist.p, sizeof(double) * hh.size(), cudaMemcpyDeviceToHost, c.stream));
  HB_CUDA(cudaMemcpyAsync(hl.data(), K.hist_len.p, sizeof(int) * p, cudaMemcpyDeviceToHost, c.stream));
  BlockState hs;
  HB_CUDA(cudaMemcpyAsync(&hs.beta0, &S->beta0, sizeof(double) * BK_MAXP + 4 * sizeof(int), cudaMemcpyDeviceToHost,
                          c.stream));
  HB_CUDA(cudaStreamSynchronize(c.stream));
  for (int col = 0; col < p; ++col) {
    const int n = std::min(hl[col], cap);
    if (hist_len_out) hist_len_out[col] = n;
    if (iters_out) iters_out[col] = iters;
    if (conv_out) conv_out[col] = uint8_t(st == 1);
    if (brk_out) brk_out[col] = uint8_t(st == 3);
    if (hist_out)
      for (int i = 0; i < std::min(n, hist_stride); ++i) hist_out[size_t(col) * hist_stride + i] = hh[size_t(col) * cap + i];
  }
}

}  // namespace hb
