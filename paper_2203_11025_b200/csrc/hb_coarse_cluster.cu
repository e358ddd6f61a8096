// Coarsest-level GMRES(k) with D^-1 (coarse_solve_with_op, inc/multigrid.hpp:
// 45-61) for coarse grids too large for one CTA per column (c2: 128^2): ONE
// thread-block cluster per column, one launch per coarse solve, the whole
// Krylov basis ON CHIP.
//
// The column's rows are split over the CS CTAs of its cluster (contiguous row
// bands of <= 2048 nodes); each CTA keeps its band of V_0..V_k (c64,
// unnormalised, fp64 scales s_i) in shared memory (<= 176 KB), u_j = D^-1 V_j
// of the band (the stencil operand) and halo rows of u_j that its neighbours
// store into it (DSMEM).  Each Arnoldi step is two cluster-wide phases:
//   (A) w = M^H D^-1 (s_j Vraw_j) on the band (kept in registers); partial
//       <Vraw_i, w> (i <= j);
//   (B) Vraw_{j+1} = w - sum_i c_i Vraw_i into shared memory; partial
//       |Vraw_{j+1}|^2 and Gram row <Vraw_{j+1}, Vraw_i>; edge rows to the
//       neighbours' halos.
// A phase's per-thread fp32 partials go through one warp butterfly per warp;
// warp 0 folds the warps in fp64 and pushes the CTA's 32 slots into EVERY CTA
// of the cluster (DSMEM stores); one cluster barrier; warp 0 of every CTA
// folds the CS slots in rank order and runs the scalar recurrence (Gram-
// corrected MGS coefficients in phase A; norm, scale, next Gram row and the
// happy-breakdown test in phase B) redundantly and bit-identically, so no
// second barrier broadcasts results.  The Givens rotations and the back-
// substitution run once at the end (the budget is fixed: tol 1e-300, so the
// residual estimate steers nothing but the happy breakdown, which needs only
// |h_{j+1,j}|).  x = D^-1 (V y).  Same algorithm and fp64 scalar state as
// the single-CTA k_coarse_reg (hb_coarse_small.cu) and the multi-launch
// coarse_krylov_solve (hb_krylov.cu, still used above 32K coarse nodes: c3's
// 256^2): 2 cluster barriers per step instead of 3 kernel launches, and no
// basis traffic to L2 / HBM.
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>

#include "hb_common.cuh"
#include "hb_internal.h"

namespace cg = cooperative_groups;

namespace hb {
__device__ long long* g_cc_trace = nullptr;  // HB_CC_TRACE: per-phase clock64 stamps of CTA (0, 0)
namespace {

constexpr int CC_NT = 512;
constexpr int CC_MAXK = 10;   // coarse GMRES restart (VCycleConfig.coarse_iters <= 10)
constexpr int CC_MAXCS = 16;  // cluster size (non-portable above 8)
constexpr int CC_MAXNX = 256; // widest coarse grid (halo rows)

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
__device__ __forceinline__ double2 shfl2(double2 v, int l) {
  return make_double2(__shfl_sync(0xffffffffu, v.x, l), __shfl_sync(0xffffffffu, v.y, l));
}

struct CCState {                        // replicated in every CTA of the cluster
  double pA[CC_MAXCS][32];              // phase-A slots by source rank
  double pB[CC_MAXCS][32];              // phase-B (and restart) slots by source rank
  float wt[CC_NT / 32][32];             // per-warp butterfly results
  double2 H[CC_MAXK][CC_MAXK + 1];      // Hessenberg columns (unrotated until the end)
  double2 G[CC_MAXK + 1][CC_MAXK + 1];  // Gram rows s_i s_k <Vraw_i, Vraw_k>
  double scale[CC_MAXK + 1];
  float2 coef[CC_MAXK + 1];             // MGS coefficients c_i = h_i s_i; then y_i s_i
  double cs[CC_MAXK];                   // Givens rotations (applied one column behind)
  double2 sn[CC_MAXK], g[CC_MAXK + 1], y[CC_MAXK];
  double beta0;
  int stop, k;
};

// Givens rotation of Hessenberg column jj (inc/krylov.hpp:49-64,221-232): the
// previous rotations, then a new one; updates g.  One thread.
__device__ void givens_column(CCState& S, int jj) {
  double2* hj = S.H[jj];
  for (int i = 0; i < jj; ++i) {
    const double2 t1 = dadd(zscale(hj[i], S.cs[i]), zmul(S.sn[i], hj[i + 1]));
    hj[i + 1] = dadd(zscale(zmul(zconj(S.sn[i]), hj[i]), -1.0), zscale(hj[i + 1], S.cs[i]));
    hj[i] = t1;
  }
  const double2 a = hj[jj];
  const double hn = hj[jj + 1].x;
  const double aa = hypot(a.x, a.y), rho = hypot(aa, hn);
  double c;
  double2 s;
  if (rho == 0.0) {
    c = 1.0;
    s = make_double2(0.0, 0.0);
  } else if (aa == 0.0) {
    c = 0.0;
    s = make_double2(1.0, 0.0);
  } else {
    c = aa / rho;
    s = zscale(a, hn / (rho * aa));
  }
  S.cs[jj] = c;
  S.sn[jj] = s;
  hj[jj] = dadd(zscale(hj[jj], c), zmul(s, hj[jj + 1]));
  const double2 gj = S.g[jj];
  S.g[jj + 1] = zscale(zmul(zconj(s), gj), -1.0);
  S.g[jj] = zscale(gj, c);
}

// warp reduce-scatter of 32 floats: lane l ends with the warp sum of float l
__device__ __forceinline__ float warp_scatter32(float (&v)[32]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int stage = 0; stage < 5; ++stage) {
    const int half = 16 >> stage, mask = 16 >> stage;
    const bool upper = (lane & mask) != 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (k < half) {
        const float send = upper ? v[k] : v[k + half];
        const float keep = upper ? v[k + half] : v[k];
        v[k] = keep + __shfl_xor_sync(0xffffffffu, send, mask);
      }
    }
  }
  return v[0];
}

// phase end: CTA sum of the 32 per-thread slots (fp64 over warps), pushed into
// row `rank` of `dst` in every CTA of the cluster, cluster barrier; warp 0
// returns the cluster sum of slot `lane` (rank order: bit-identical in every
// CTA), other warps 0
__device__ __forceinline__ double cluster_sum32(cg::cluster_group& cl, CCState& S, double (*dst)[32], float (&v)[32],
                                                int rank, int CS) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  S.wt[warp][lane] = warp_scatter32(v);
  __syncthreads();
  if (warp == 0) {
    double t = 0.0;
#pragma unroll
    for (int w2 = 0; w2 < CC_NT / 32; ++w2) t += double(S.wt[w2][lane]);
    for (int r = 0; r < CS; ++r) cl.map_shared_rank(&dst[rank][lane], r)[0] = t;
  }
  cl.sync();  // barrier.cluster arrive.release / wait.acquire: orders the DSMEM stores
  double s = 0.0;
  if (warp == 0)
    for (int r = 0; r < CS; ++r) s += dst[r][lane];
  return s;
}

template <int NPT>
__global__ void __launch_bounds__(CC_NT, 1) k_coarse_cluster(LevelView L, int m, const int* act,
                                                             const float2* __restrict__ f, float2* __restrict__ x) {
  long long* const tr = (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) ? g_cc_trace : nullptr;
  if (tr) tr[120] = clock64();
  pdl_enter();
  cg::cluster_group cl = cg::this_cluster();
  const int CS = int(cl.num_blocks());
  const int rank = int(cl.block_rank());
  const int b = blockIdx.y;
  if (act && !act[b]) return;  // uniform across the cluster
  constexpr int NB = NPT * CC_NT;  // band capacity (one node per thread per q)
  extern __shared__ float2 dsm[];
  float2* const Vs = dsm;                      // [CC_MAXK + 1][NB] basis (raw, c64)
  float2* const U = Vs + (CC_MAXK + 1) * NB;  // [NB] u_j = D^-1 Vraw_j on the band (the stencil's operand)
  float2* const halo = U + NB;                 // [2][CC_MAXNX] u_j rows above (0) / below (1) the band
  __shared__ CCState S;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nx = L.nx, ny = L.ny;
  const int rows = ny / CS, r0 = rank * rows;
  const int n0 = r0 * nx, nb = rows * nx;  // band nodes (nb <= NB)
  const size_t N = size_t(nx) * ny;
  const float ih2 = L.inv_h2;
  const float2* fb = f + size_t(b) * N;
  // setup: own nodes' D^-1 and neighbour flags in registers; V_0 = f and u_0 = D^-1 f
  // on the band, u_0 on the halo rows (zero outside the grid)
  for (int t = threadIdx.x; t < 2 * nx; t += CC_NT) {
    const int side = t / nx, ix = t % nx, gy = side == 0 ? r0 - 1 : r0 + rows;
    const size_t gp = size_t(gy) * nx + ix;
    halo[side * CC_MAXNX + ix] = gy >= 0 && gy < ny ? cmul(ld(fb, gp), crcp(ld(L.dM, gp))) : make_float2(0.f, 0.f);
  }
  float2 di[NPT];
  int ixq[NPT], lyq[NPT];
  float v[32];
#pragma unroll
  for (int s = 0; s < 32; ++s) v[s] = 0.f;
#pragma unroll
  for (int q = 0; q < NPT; ++q) {
    const int t = threadIdx.x + q * CC_NT;
    ixq[q] = t % nx;
    lyq[q] = t / nx;
    di[q] = make_float2(0.f, 0.f);
    if (t < nb) {
      di[q] = crcp(ld(L.dM, n0 + t));
      const float2 a = ld(fb, n0 + t);
      Vs[t] = a;
      U[t] = cmul(a, di[q]);
      v[31] = fmaf(a.x, a.x, fmaf(a.y, a.y, v[31]));
    }
  }
  {
    const double t = cluster_sum32(cl, S, S.pB, v, rank, CS);
    if (warp == 0) {
      const double beta = sqrt(__shfl_sync(0xffffffffu, t, 31));
      if (lane == 0) {
        S.beta0 = beta;
        S.stop = beta == 0.0;
        S.k = 0;
        S.scale[0] = beta > 0.0 ? 1.0 / beta : 0.0;
        S.g[0] = make_double2(beta, 0.0);
      }
    }
    __syncthreads();
  }
#define CC_STAMP(k) \
  if (tr && j < 16) tr[j * 8 + (k)] = clock64();
  float2 w[NPT];
  if (tr) tr[121] = clock64();
  for (int j = 0; j < m && !S.stop; ++j) {
    CC_STAMP(0)
    // the previous column's Givens rotation runs on the last warp's lane 0 while
    // the other threads compute phase A (its results are first read at the end)
    if (j > 0 && threadIdx.x == CC_NT - 32) givens_column(S, j - 1);
    // ---- (A) w = M^H D^-1 (s_j Vraw_j); partial <Vraw_i, w> in slots 2i, 2i+1
    const float sj = float(S.scale[j]);
    const float2* Vj = Vs + j * NB;
#pragma unroll
    for (int s = 0; s < 32; ++s) v[s] = 0.f;
#pragma unroll
    for (int q = 0; q < NPT; ++q) {
      const int t = threadIdx.x + q * CC_NT;
      w[q] = make_float2(0.f, 0.f);
      if (t >= nb) continue;
      const int ix = ixq[q], ly = lyq[q];
      float2 nbs = make_float2(0.f, 0.f);
      if (ix > 0) nbs = cadd(nbs, U[t - 1]);
      if (ix + 1 < nx) nbs = cadd(nbs, U[t + 1]);
      nbs = cadd(nbs, ly > 0 ? U[t - nx] : halo[ix]);
      nbs = cadd(nbs, ly + 1 < rows ? U[t + nx] : halo[CC_MAXNX + ix]);
      float2 yv = Vj[t];  // D (D^-1 v) = v
      yv.x = fmaf(-ih2, nbs.x, yv.x);
      yv.y = fmaf(-ih2, nbs.y, yv.y);
      w[q] = cscale(yv, sj);
#pragma unroll
      for (int i = 0; i <= CC_MAXK; ++i) {
        if (i > j) break;
        const float2 a = Vs[i * NB + t];
        v[2 * i] = fmaf(a.x, w[q].x, fmaf(a.y, w[q].y, v[2 * i]));
        v[2 * i + 1] = fmaf(a.x, w[q].y, fmaf(-a.y, w[q].x, v[2 * i + 1]));
      }
    }
    CC_STAMP(1)
    {
      const double d = cluster_sum32(cl, S, S.pA, v, rank, CS);
      CC_STAMP(2)
      // MGS coefficients (Gram-corrected, as adots_scalar): h_i = s_i <Vraw_i, w> - sum_{k<i} hcgs_k G_ik
      if (warp == 0) {
        const double2 dot = make_double2(__shfl_sync(0xffffffffu, d, (2 * lane) & 31),
                                         __shfl_sync(0xffffffffu, d, (2 * lane + 1) & 31));
        const double si = lane <= j ? S.scale[lane] : 0.0;
        const double2 hcgs = lane <= j ? zscale(dot, si) : make_double2(0.0, 0.0);
        double2 h = hcgs;
        for (int kk = 0; kk < j; ++kk) {
          const double2 hk = shfl2(hcgs, kk);
          if (lane <= j && kk < lane) h = zsub(h, zmul(hk, S.G[lane][kk]));
        }
        if (lane <= j) {
          S.H[j][lane] = h;
          const double2 c = zscale(h, si);
          S.coef[lane] = make_float2(float(c.x), float(c.y));
        }
      }
      __syncthreads();
    }
    CC_STAMP(3)
    // ---- (B) Vraw_{j+1} = w - sum_i c_i Vraw_i; Gram row in slots 2i, 2i+1; |.|^2 in slot 31
    float2* Vn = Vs + (j + 1) * NB;
    const bool more = j + 1 < m;
#pragma unroll
    for (int s = 0; s < 32; ++s) v[s] = 0.f;
#pragma unroll
    for (int q = 0; q < NPT; ++q) {
      const int t = threadIdx.x + q * CC_NT;
      if (t >= nb) continue;
      float2 tv = w[q];
#pragma unroll
      for (int i = 0; i <= CC_MAXK; ++i) {
        if (i > j) break;
        tv = csub(tv, cmul(S.coef[i], Vs[i * NB + t]));
      }
      Vn[t] = tv;
      U[t] = cmul(tv, di[q]);
      v[31] = fmaf(tv.x, tv.x, fmaf(tv.y, tv.y, v[31]));
      if (more) {
#pragma unroll
        for (int i = 0; i <= CC_MAXK; ++i) {
          if (i > j) break;
          const float2 a = Vs[i * NB + t];
          v[2 * i] = fmaf(tv.x, a.x, fmaf(tv.y, a.y, v[2 * i]));
          v[2 * i + 1] = fmaf(tv.x, a.y, fmaf(-tv.y, a.x, v[2 * i + 1]));
        }
      }
    }
    CC_STAMP(4)
    // band edge rows of u_{j+1} into the neighbours' halos (read after the barrier below)
    if (more) {
      __syncthreads();  // U complete
      for (int t = threadIdx.x; t < 2 * nx; t += CC_NT) {
        const int side = t / nx, ix = t % nx;  // 0: first row -> upper neighbour's "below"; 1: last -> lower's "above"
        const int nbr = side == 0 ? rank - 1 : rank + 1;
        if (nbr < 0 || nbr >= CS) continue;
        float2* hn = cl.map_shared_rank(halo, nbr);
        hn[(side == 0 ? CC_MAXNX : 0) + ix] = U[(side == 0 ? 0 : (rows - 1) * nx) + ix];
      }
    }
    CC_STAMP(5)
    {
      const double g = cluster_sum32(cl, S, S.pB, v, rank, CS);
      CC_STAMP(6)
      if (warp == 0) {
        const double hnorm = sqrt(__shfl_sync(0xffffffffu, g, 31));
        const double2 gr = make_double2(__shfl_sync(0xffffffffu, g, (2 * lane) & 31),
                                        __shfl_sync(0xffffffffu, g, (2 * lane + 1) & 31));
        const bool happy = hnorm <= 1e-14 * S.beta0;  // inc/krylov.hpp:240-241
        if (lane == 0) {
          S.H[j][j + 1] = make_double2(hnorm, 0.0);
          S.k = j + 1;
          if (happy || !more) S.stop = 1;
        }
        if (!happy && more) {
          const double sn1 = 1.0 / hnorm;
          if (lane == 0) S.scale[j + 1] = sn1;
          if (lane <= j) S.G[j + 1][lane] = zscale(gr, sn1 * S.scale[lane]);
        }
      }
      __syncthreads();
    }
    CC_STAMP(7)
  }
#undef CC_STAMP
  // ---- the last column's Givens rotation, y = R^-1 g (column-sweep back-
  // substitution, inc/krylov.hpp:119-126, lanes in parallel); x = D^-1 (sum_i y_i s_i Vraw_i)
  const int k = S.k;
  if (tr) tr[122] = clock64();
  if (threadIdx.x == 0 && k > 0) givens_column(S, k - 1);
  __syncthreads();
  if (warp == 0 && k > 0) {
    double2 gl = lane < k ? S.g[lane] : make_double2(0.0, 0.0);
    for (int i = k - 1; i >= 0; --i) {
      double2 yi = make_double2(0.0, 0.0);
      if (lane == i) {
        yi = zdiv(gl, S.H[i][i]);
        S.coef[i] = make_float2(float(yi.x * S.scale[i]), float(yi.y * S.scale[i]));
      }
      yi = shfl2(yi, i);
      if (lane < i) gl = zsub(gl, zmul(S.H[i][lane], yi));
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NPT; ++q) {
    const int t = threadIdx.x + q * CC_NT;
    if (t >= nb) continue;
    float2 u = make_float2(0.f, 0.f);
    for (int i = 0; i < k; ++i) u = cadd(u, cmul(S.coef[i], Vs[i * NB + t]));
    x[size_t(b) * N + n0 + t] = cmul(u, di[q]);
  }
  if (tr) tr[123] = clock64();
  // no CTA may exit while another can still store into its shared memory
  cl.sync();
  if (tr) tr[124] = clock64();
}

template <int NPT>
constexpr size_t cc_smem() {
  return sizeof(float2) * ((CC_MAXK + 2) * NPT * CC_NT + 2 * CC_MAXNX);
}

template <int NPT>
void launch_cc(Context& c, int CS, int B, const LevelView& L, int m, const int* act, const float2* f, float2* x) {
  static int attr = -1;
  constexpr size_t smem = cc_smem<NPT>();
  if (attr != c.device) {
    HB_CUDA(cudaFuncSetAttribute(k_coarse_cluster<NPT>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    HB_CUDA(cudaFuncSetAttribute(k_coarse_cluster<NPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr = c.device;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CS, B);
  cfg.blockDim = dim3(CC_NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c.stream;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = c.opt_pdl ? 2 : 1;
  HB_CUDA(cudaLaunchKernelEx(&cfg, k_coarse_cluster<NPT>, L, m, act, f, x));
}

}  // namespace

// true if launched: coarse grids of 2K..32K nodes (<= 256 wide) with <= 10 GMRES iterations
bool launch_coarse_cluster(Context& c, const LevelView& L, int iters, int B, int slot, const int* act, const float2* f,
                           float2* x) {
  (void)slot;
  const int N = L.nx * L.ny;
  if (iters < 1 || iters > CC_MAXK || N <= 2048 || L.nx > CC_MAXNX) return false;
  // bands of <= 2048 nodes (the on-chip basis: 11 x 2048 x 8 B = 176 KB) and >=
  // 2 rows: the smallest such cluster (two 8-CTA clusters share a GPC; a
  // 16-CTA cluster takes a whole one)
  int CS = 0;
  for (int cs : {2, 4, 8, 16})
    if (L.ny % cs == 0 && L.ny / cs >= 2 && N / cs <= 4 * CC_NT) {
      CS = cs;
      break;
    }
  if (!CS) return false;
  const int tok = prof_begin(c, PC_COARSE);
  if (N / CS <= 2 * CC_NT)
    launch_cc<2>(c, CS, B, L, iters, act, f, x);
  else
    launch_cc<4>(c, CS, B, L, iters, act, f, x);
  prof_end(c, PC_COARSE, tok, double(B) * N * 16.0 + double(N) * 8.0, 0);  // f in, x out; diag
  HB_CUDA(cudaGetLastError());
  static const bool trace = getenv("HB_CC_TRACE") != nullptr;
  static long long* dtr = nullptr;
  static int ntr = 0;
  if (trace && ntr < 3) {
    if (!dtr) {
      HB_CUDA(cudaMalloc(&dtr, 16 * 8 * sizeof(long long)));
      HB_CUDA(cudaMemcpyToSymbol(g_cc_trace, &dtr, sizeof(dtr)));
    }
    long long h[128];
    HB_CUDA(cudaStreamSynchronize(c.stream));
    HB_CUDA(cudaMemcpy(h, dtr, sizeof(h), cudaMemcpyDeviceToHost));
    if (++ntr == 3) {
      fprintf(stderr, "cluster coarse trace (cycles from step start): A-compute A-sum MGS B-compute halo B-sum scalar\n");
      for (int j = 0; j < iters && j < 16; ++j)
        fprintf(stderr, "  j=%2d %6lld %6lld %6lld %6lld %6lld %6lld %6lld\n", j, h[j * 8 + 1] - h[j * 8],
                h[j * 8 + 2] - h[j * 8], h[j * 8 + 3] - h[j * 8], h[j * 8 + 4] - h[j * 8], h[j * 8 + 5] - h[j * 8],
                h[j * 8 + 6] - h[j * 8], h[j * 8 + 7] - h[j * 8]);
      fprintf(stderr, "  setup %lld, steps %lld, lsq+x %lld, exit sync %lld cycles\n", h[121] - h[120], h[122] - h[121],
              h[123] - h[122], h[124] - h[123]);
      int ncl = 0;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(CS, B);
      cfg.blockDim = dim3(CC_NT);
      cfg.dynamicSmemBytes = N / CS <= 2 * CC_NT ? cc_smem<2>() : cc_smem<4>();
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = CS;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaOccupancyMaxActiveClusters(&ncl, N / CS <= 2 * CC_NT ? (void*)k_coarse_cluster<2> : (void*)k_coarse_cluster<4>, &cfg);
      fprintf(stderr, "  cluster size %d, max active clusters %d\n", CS, ncl);
    }
  }
  return true;
}

}  // namespace hb
