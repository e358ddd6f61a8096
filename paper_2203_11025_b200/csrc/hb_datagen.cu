// Training-pair generation: gen_sample_pair
// (inc/datagen.hpp:191-219) for a batch of seeds on the device hot path.
//
//   x ~ CN(0, I) (Rng(seed)); b = A x; k = k_forced or uniform_int(1, k_max);
//   x~ = FGMRES(A, M_V, b, 0, restart 10, k iterations, tol 1e-6);
//   r = b - A x~; e = x - x~.
//
// The draws stay on the host (they define the pair; one Rng per seed, as the
// reference).  The reference draws each node as Complex(rng.normal(),
// rng.normal()): C++ leaves the argument order unspecified and the compiled
// reference (GCC) evaluates right to left, so the IMAGINARY part is drawn
// first -- pinned by the k = 0 golden pairs.  The draws run on all host
// threads (one Rng per seed, so the split changes nothing); the samples with
// k > 0 of a chunk are ONE device-resident batched FGMRES with a per-column
// iteration limit k (columns are independent Arnoldi processes); b = A x,
// r = b - A x~ and e = x - x~ are formed in fp64 on the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <numeric>
#include <thread>
#include <vector>

#include "hb_common.cuh"
#include "hb_host.h"
#include "hb_internal.h"

namespace hb {

void fgmres_dev_entry(Context& c, const hb_krylov_cfg* cfg, int kind, int B, const double2* dB, double2* dX,
                      const int* d_limits);

namespace {

// y = A u in fp64 (5-point stencil with the fp64 diagonal, zero padding), y = s*(f - A u) when f
__global__ void k_apply64(int nx, int ny, double inv_h2, const double2* __restrict__ dA, const double2* __restrict__ u,
                          const double2* __restrict__ f, double2* __restrict__ y) {
  const size_t N = size_t(nx) * ny;
  const int b = blockIdx.y;
  const double2* ub = u + b * N;
  for (size_t p = size_t(blockIdx.x) * blockDim.x + threadIdx.x; p < N; p += size_t(gridDim.x) * blockDim.x) {
    const int ix = int(p % nx), iy = int(p / nx);
    double2 nb = make_double2(0.0, 0.0);
    if (ix > 0) nb = dadd(nb, ub[p - 1]);
    if (ix + 1 < nx) nb = dadd(nb, ub[p + 1]);
    if (iy > 0) nb = dadd(nb, ub[p - nx]);
    if (iy + 1 < ny) nb = dadd(nb, ub[p + nx]);
    const double2 d = dA[p], v = ub[p];
    double2 a = make_double2(d.x * v.x - d.y * v.y - inv_h2 * nb.x, d.x * v.y + d.y * v.x - inv_h2 * nb.y);
    if (f) a = make_double2(f[b * N + p].x - a.x, f[b * N + p].y - a.y);
    y[b * N + p] = a;
  }
}
__global__ void k_sub64(size_t n, const double2* __restrict__ a, const double2* __restrict__ b, double2* __restrict__ y) {
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    y[i] = make_double2(a[i].x - b[i].x, a[i].y - b[i].y);
}

}  // namespace
}  // namespace hb

using namespace hb;
struct hb_ctx : hb::Context {};

#define HB_API_BEGIN \
  if (!ctx) return HB_ERR_ARG; \
  try {
#define HB_API_END                  \
  return HB_OK;                     \
  }                                 \
  catch (const HbError& e) {        \
    ctx->err = e.msg;               \
    return e.code;                  \
  }                                 \
  catch (const std::exception& e) { \
    ctx->err = e.what();            \
    return HB_ERR_ARG;              \
  }

extern "C" {

int hb_gen_sample_pairs(hb_ctx* ctx, int count, const uint64_t* seeds, int k_forced, int k_max, double* r_out,
                        double* e_out, int* k_used) {
  HB_API_BEGIN
  require_whole(*ctx);
  if (!ctx->has_hier) throw HbError{HB_ERR_STATE, "hierarchy not built (hb_build_hierarchy)"};
  if (count < 1 || !seeds || !r_out || !e_out) throw HbError{HB_ERR_ARG, "bad buffers / count"};
  if (k_forced < 0 && k_max < 1) throw HbError{HB_ERR_ARG, "k_max must be >= 1"};
  if (k_forced > 100000) throw HbError{HB_ERR_ARG, "k_forced too large"};
  Context& c = *ctx;
  const Level& L0 = *c.levels[0];
  const int nx = L0.nx, ny = L0.ny;
  const size_t N = size_t(nx) * ny;
  // host draws (inc/datagen.hpp:185-201), all host threads: per node
  // Complex(normal, normal) with the imaginary part drawn first
  std::vector<double2> xs(N * size_t(count));
  std::vector<int> ks(static_cast<size_t>(count));
  {
    const int T = std::max(1, std::min<int>(count, int(std::thread::hardware_concurrency())));
    auto work = [&](int t) {
      for (int s = t; s < count; s += T) {
        Rng rng(seeds[s]);
        double2* x = xs.data() + N * size_t(s);
        for (size_t i = 0; i < N; ++i) {
          const double im = rng.normal();
          const double re = rng.normal();
          x[i] = make_double2(re, im);
        }
        ks[size_t(s)] = k_forced >= 0 ? k_forced : int(rng.uniform_int(1, k_max));
      }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& h : th) h.join();
  }
  if (k_used)
    for (int s = 0; s < count; ++s) k_used[s] = ks[size_t(s)];
  // order: samples that need a solve first (stable), so each chunk's solve is a prefix
  std::vector<int> order(static_cast<size_t>(count));
  std::iota(order.begin(), order.end(), 0);
  std::stable_partition(order.begin(), order.end(), [&](int s) { return ks[size_t(s)] > 0; });
  constexpr int kChunk = 512;
  DBuf<double2> dx, db, dxt, dr;
  const double inv_h2 = 1.0 / (L0.h * L0.h);
  std::vector<double2> stage(N * size_t(std::min(count, kChunk)));
  std::vector<int> lim;
  for (int g0 = 0; g0 < count; g0 += kChunk) {
    const int B = std::min(kChunk, count - g0);
    const size_t n = N * size_t(B);
    dx.ensure(n);
    db.ensure(n);
    dxt.ensure(n);
    dr.ensure(n);
    lim.assign(size_t(B), 0);
    int nsolve = 0, kmax = 0;
    for (int j = 0; j < B; ++j) {
      const int s = order[size_t(g0 + j)];
      std::copy_n(xs.data() + N * size_t(s), N, stage.data() + N * size_t(j));
      lim[size_t(j)] = ks[size_t(s)];
      if (ks[size_t(s)] > 0) {
        nsolve = j + 1;
        kmax = std::max(kmax, ks[size_t(s)]);
      }
    }
    HB_CUDA(cudaMemcpyAsync(dx.p, stage.data(), n * sizeof(double2), cudaMemcpyHostToDevice, c.stream));
    const dim3 grid(unsigned(std::min<size_t>((N + 255) / 256, 1024)), unsigned(B));
    c.launches++;
    k_apply64<<<grid, 256, 0, c.stream>>>(nx, ny, inv_h2, L0.dA64.p, dx.p, nullptr, db.p);  // b = A x
    HB_CUDA(cudaGetLastError());
    HB_CUDA(cudaMemsetAsync(dxt.p, 0, n * sizeof(double2), c.stream));
    if (nsolve > 0) {  // FGMRES(A, M_V, b, 0; restart 10, k_j iterations, tol 1e-6) (inc/datagen.hpp:203-211)
      c.klimit.ensure(size_t(nsolve));
      HB_CUDA(cudaMemcpyAsync(c.klimit.p, lim.data(), sizeof(int) * size_t(nsolve), cudaMemcpyHostToDevice,
                              c.stream));
      hb_krylov_cfg kc{10, kmax, 1e-6, 1};
      fgmres_dev_entry(c, &kc, HB_PC_V, nsolve, db.p, dxt.p, c.klimit.p);
    }
    c.launches += 2;
    k_apply64<<<grid, 256, 0, c.stream>>>(nx, ny, inv_h2, L0.dA64.p, dxt.p, db.p, dr.p);  // r = b - A x~
    k_sub64<<<unsigned(std::min<size_t>((n + 255) / 256, 4096)), 256, 0, c.stream>>>(n, dx.p, dxt.p, db.p);  // e
    HB_CUDA(cudaGetLastError());
    for (int pass = 0; pass < 2; ++pass) {
      HB_CUDA(cudaMemcpyAsync(stage.data(), pass ? db.p : dr.p, n * sizeof(double2), cudaMemcpyDeviceToHost,
                              c.stream));
      HB_CUDA(cudaStreamSynchronize(c.stream));
      double2* dst = reinterpret_cast<double2*>(pass ? e_out : r_out);
      for (int j = 0; j < B; ++j)
        std::copy_n(stage.data() + N * size_t(j), N, dst + N * size_t(order[size_t(g0 + j)]));
    }
  }
  HB_API_END
}

}  // extern "C"
