// libhelmgpu host runtime + C ABI (include/helmgpu.h).
//
// The host owns: problem setup and fp64 coefficient coarsening (as
// coarsen_problem, inc/stencil.hpp:169-185, offset (l-1)%2 per
// inc/multigrid.hpp:80-81), the V-cycle schedule (cycle_at,
// inc/multigrid.hpp:108-119), the preconditioner plugins (inc/precond.hpp) and
// the FGMRES restart loop; every arithmetic step runs on the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <string>
#include <vector>

#include "hb_host.h"
#include "hb_internal.h"

namespace hb {

unsigned long long g_alloc_gen = 0;

void krylov_report(Context& c, int B, double* hist, int hist_stride, int* hist_len, int* iters, uint8_t* conv,
                   uint8_t* brk);

// ------------------------------------------------------------ profiling --
static const char* kProfNames[PC_COUNT] = {"stencil",        "smooth",         "vcycle_down",   "vcycle_up",
                                           "transfer",       "coarse_solve",   "krylov_adots",  "krylov_update",
                                           "krylov_restart", "krylov_finalize", "conv3x3",      "net_io"};

int prof_begin(Context& c, int cls) {
  (void)cls;
  c.launches++;
  if (!c.prof_on) return -1;
  cudaEvent_t a, b;
  if (c.ev_pool.size() >= 2) {
    a = c.ev_pool.back();
    c.ev_pool.pop_back();
    b = c.ev_pool.back();
    c.ev_pool.pop_back();
  } else {
    HB_CUDA(cudaEventCreate(&a));
    HB_CUDA(cudaEventCreate(&b));
  }
  HB_CUDA(cudaEventRecord(a, c.stream));
  c.ev_pending.push_back({cls, {a, b}});
  return int(c.ev_pending.size()) - 1;
}

void prof_collect(Context& c) {
  if (c.ev_pending.empty()) return;
  HB_CUDA(cudaStreamSynchronize(c.stream));
  std::vector<float> times(c.ev_pending.size());
  for (size_t i = 0; i < c.ev_pending.size(); ++i) {
    auto& e = c.ev_pending[i];
    float ms = 0.f;
    HB_CUDA(cudaEventElapsedTime(&ms, e.second.first, e.second.second));
    times[i] = ms;
    if (e.first >= 0) c.prof[size_t(e.first)].ms += ms;  // < 0: launch with no active column, not counted
    c.ev_pool.push_back(e.second.first);
    c.ev_pool.push_back(e.second.second);
  }
  for (auto& d : c.detail) {
    d.ms = d.token < times.size() ? times[d.token] : 0.0;
    c.detail_done.push_back(d);
  }
  c.detail.clear();
  c.ev_pending.clear();
}

void prof_end(Context& c, int cls, int token, double bytes, double flops) {
  if (token < 0) return;
  HB_CUDA(cudaEventRecord(c.ev_pending[size_t(token)].second.second, c.stream));
  if (c.prof_detail)
    c.detail.push_back(Context::DetailRec{c.prof_label.empty() ? c.prof[size_t(cls)].name : c.prof_label,
                                          size_t(token), 0.0, bytes, flops});
  c.prof_label.clear();
  Prof& p = c.prof[size_t(cls)];
  if (c.prof_scale <= 0.0) {  // every column frozen: the launch is a no-op, keep it out of the rates
    c.ev_pending[size_t(token)].first = -1;
    return;
  }
  p.launches += 1;
  p.bytes += bytes * c.prof_scale;
  p.flops += flops * c.prof_scale;
  if (c.ev_pending.size() > 8192) prof_collect(c);
}

// ------------------------------------------------------------- helpers --
static std::vector<float2> to_c64(const double* p, size_t n) {
  std::vector<float2> v(n);
  for (size_t i = 0; i < n; ++i) v[i] = make_float2(float(p[2 * i]), float(p[2 * i + 1]));
  return v;
}
static void from_c64(const std::vector<float2>& v, double* p) {
  for (size_t i = 0; i < v.size(); ++i) {
    p[2 * i] = v[i].x;
    p[2 * i + 1] = v[i].y;
  }
}

// CoarseSolver::dense setup: assemble M^H as assemble_dense does
// (inc/multigrid.hpp:24-42), invert it by Gauss-Jordan elimination with partial
// pivoting in fp64 (the reference factors it once with PartialPivLU, :84, and
// solves per call, :95-104), upload the inverse
static void build_dense_inverse(Level& L, double omega, double alpha, double beta) {
  const int nx = L.nx, ny = L.ny, n = nx * ny;
  if (n > 1024) throw HbError{HB_ERR_ARG, "dense coarse solver: coarsest grid larger than 32x32 nodes"};
  using cd = std::complex<double>;
  const double inv_h2 = 1.0 / (L.h * L.h);
  const cd sh(alpha, -beta);
  std::vector<cd> A(size_t(n) * n, cd(0.0)), I(size_t(n) * n, cd(0.0));
  for (int iy = 0; iy < ny; ++iy)
    for (int ix = 0; ix < nx; ++ix) {
      const size_t i = size_t(iy) * nx + ix;
      const cd damp(1.0, -L.gam[i]);
      A[i * n + i] = 4.0 * inv_h2 - omega * omega * L.k2[i] * sh * damp;
      if (ix > 0) A[i * n + i - 1] = -inv_h2;
      if (ix + 1 < nx) A[i * n + i + 1] = -inv_h2;
      if (iy > 0) A[i * n + i - nx] = -inv_h2;
      if (iy + 1 < ny) A[i * n + i + nx] = -inv_h2;
      I[i * n + i] = 1.0;
    }
  for (int k = 0; k < n; ++k) {
    int piv = k;
    for (int r = k + 1; r < n; ++r)
      if (std::abs(A[size_t(r) * n + k]) > std::abs(A[size_t(piv) * n + k])) piv = r;
    if (std::abs(A[size_t(piv) * n + k]) == 0.0) throw HbError{HB_ERR_NUMERIC, "dense coarse operator is singular"};
    if (piv != k)
      for (int j = 0; j < n; ++j) {
        std::swap(A[size_t(k) * n + j], A[size_t(piv) * n + j]);
        std::swap(I[size_t(k) * n + j], I[size_t(piv) * n + j]);
      }
    const cd d = 1.0 / A[size_t(k) * n + k];
    for (int j = 0; j < n; ++j) {
      A[size_t(k) * n + j] *= d;
      I[size_t(k) * n + j] *= d;
    }
    for (int r = 0; r < n; ++r) {
      if (r == k) continue;
      const cd f = A[size_t(r) * n + k];
      if (f == 0.0) continue;
      for (int j = 0; j < n; ++j) {
        A[size_t(r) * n + j] -= f * A[size_t(k) * n + j];
        I[size_t(r) * n + j] -= f * I[size_t(k) * n + j];
      }
    }
  }
  std::vector<double2> h(size_t(n) * n);
  for (size_t i = 0; i < h.size(); ++i) h[i] = make_double2(I[i].real(), I[i].imag());
  L.dinv.ensure(h.size());
  HB_CUDA(cudaMemcpy(L.dinv.p, h.data(), h.size() * sizeof(double2), cudaMemcpyHostToDevice));
}

static void require_hier(Context& c) {
  if (!c.has_hier) throw HbError{HB_ERR_STATE, "hierarchy not built (hb_build_hierarchy)"};
}

void require_whole(const Context& c) {
  if (c.slab) throw HbError{HB_ERR_STATE, "context holds a row slab: use the hb_*_slab entry points"};
}

void fill_level_device(Level& L, double omega, double alpha, double beta, double damping, bool fp64A,
                              bool fp64M) {
  // storage window [row0, row0 + rows) of the (global) level; rows outside the
  // domain are zero padding
  const size_t n = L.N();
  const double inv_h2 = 1.0 / (L.h * L.h);
  std::vector<float2> dm(n, make_float2(0.f, 0.f)), da(n, make_float2(0.f, 0.f)), wd(n, make_float2(0.f, 0.f));
  std::vector<double2> da64(fp64A ? n : 0, make_double2(0.0, 0.0)), dm64(fp64M ? n : 0, make_double2(0.0, 0.0));
  std::vector<float> kf(n, 0.f);
  const std::complex<double> sh(alpha, -beta), sh0(1.0, 0.0);
  for (size_t i = 0; i < n; ++i) {
    const int gy = L.row0 + int(i / size_t(L.nx));
    if (gy < 0 || gy >= L.ny) continue;
    const size_t gi = size_t(gy) * L.nx + i % size_t(L.nx);
    // inc/stencil.hpp:27-34: d = 4/h^2 - omega^2 kappa^2 (alpha - beta i)(1 - gamma i)
    const std::complex<double> damp(1.0, -L.gam[gi]);
    const std::complex<double> mM = -omega * omega * L.k2[gi] * sh * damp;
    const std::complex<double> mA = -omega * omega * L.k2[gi] * sh0 * damp;
    const std::complex<double> dMd = 4.0 * inv_h2 + mM, dAd = 4.0 * inv_h2 + mA;
    if (dMd == 0.0 || dAd == 0.0) throw HbError{HB_ERR_NUMERIC, "zero stencil diagonal"};
    dm[i] = make_float2(float(dMd.real()), float(dMd.imag()));
    const std::complex<double> w = damping / dMd;
    wd[i] = make_float2(float(w.real()), float(w.imag()));
    da[i] = make_float2(float(dAd.real()), float(dAd.imag()));
    if (fp64A) da64[i] = make_double2(dAd.real(), dAd.imag());
    if (fp64M) dm64[i] = make_double2(dMd.real(), dMd.imag());
    kf[i] = float(L.k2[gi]);
  }
  L.dM.ensure(n);
  L.dA.ensure(n);
  L.wdi.ensure(n);
  HB_CUDA(cudaMemcpy(L.wdi.p, wd.data(), n * sizeof(float2), cudaMemcpyHostToDevice));
  L.k2f.ensure(n);
  HB_CUDA(cudaMemcpy(L.dM.p, dm.data(), n * sizeof(float2), cudaMemcpyHostToDevice));
  HB_CUDA(cudaMemcpy(L.dA.p, da.data(), n * sizeof(float2), cudaMemcpyHostToDevice));
  HB_CUDA(cudaMemcpy(L.k2f.p, kf.data(), n * sizeof(float), cudaMemcpyHostToDevice));
  if (fp64A) {
    L.dA64.ensure(n);
    HB_CUDA(cudaMemcpy(L.dA64.p, da64.data(), n * sizeof(double2), cudaMemcpyHostToDevice));
  }
  if (fp64M) {
    L.dM64.ensure(n);
    HB_CUDA(cudaMemcpy(L.dM64.p, dm64.data(), n * sizeof(double2), cudaMemcpyHostToDevice));
    // D^-1 (c64) for the multi-CTA coarse GMRES: the fp32 reciprocal of the c64 diagonal (as crcp)
    std::vector<float2> dmi(n, make_float2(0.f, 0.f));
    for (size_t i = 0; i < n; ++i) {
      const float s = 1.0f / std::fma(dm[i].x, dm[i].x, dm[i].y * dm[i].y);
      dmi[i] = make_float2(dm[i].x * s, -dm[i].y * s);
    }
    L.dMi.ensure(n);
    HB_CUDA(cudaMemcpy(L.dMi.p, dmi.data(), n * sizeof(float2), cudaMemcpyHostToDevice));
  }
}

void ensure_batch(Context& c, int B) {
  require_hier(c);
  if (B <= c.batch_cap) return;
  for (auto& L : c.levels) {
    const size_t n = L->N() * size_t(B);
    L->f.ensure(n);
    L->v.ensure(n);
    L->t.ensure(n);
    L->x.ensure(n);
  }
  const Level& C = *c.levels.back();
  c.scratch_c64.ensure(size_t(B) * (kMaxCoarseIters + 2) * C.N());
  c.act_all.ensure(B);
  std::vector<int> ones(size_t(B), 1);
  HB_CUDA(cudaMemcpy(c.act_all.p, ones.data(), sizeof(int) * B, cudaMemcpyHostToDevice));
  c.batch_cap = B;
}

// ------------------------------------------------------------- V-cycle --
// cycle_at (inc/multigrid.hpp:108-119) on device buffers; level-0 input f may
// carry a per-column scale (FGMRES basis vectors are stored unnormalised).
void coarsest_solve(Context& c, int B, int c0, const int* act, const float2* f, float2* out) {
  Level& L = *c.levels.back();
  const LevelView V = L.view();
  float2* tbuf = L.t.p + size_t(c0) * L.N();
  switch (c.vc.coarse_solver) {
    case HB_COARSE_GMRES:
      if (c.opt_small_coarse && launch_coarse_small(c, V, c.vc.coarse_iters, B, act, f, out)) break;
      // one thread-block cluster per column, basis on chip (c2: 128^2)
      if (c.opt_coarse_cluster && launch_coarse_cluster(c, V, c.vc.coarse_iters, B, c0 != 0 ? 1 : 0, act, f, out))
        break;
      if (c.opt_coarse_krylov && L.N() > 2048 && c.vc.coarse_iters <= kMaxRestart) {  // multi-CTA Krylov kernels: fills the GPU at 128^2+
        coarse_krylov_solve(c, L, c.vc.coarse_iters, B, c0 != 0 ? 1 : 0, f, out);
        break;
      }
      launch_coarse_gmres(c, V, c.vc.coarse_iters, B, act, f, out,
                          c.scratch_c64.p + size_t(c0) * (kMaxCoarseIters + 2) * L.N());
      break;
    case HB_COARSE_JACOBI: {  // A3: iters damped sweeps from zero
      const float w = float(c.vc.damping);
      if (c.vc.coarse_iters <= 0) {
        HB_CUDA(cudaMemsetAsync(out, 0, sizeof(float2) * L.N() * B, c.stream));
        break;
      }
      float2* a = (c.vc.coarse_iters % 2 == 1) ? out : tbuf;
      float2* bb = (a == out) ? tbuf : out;
      launch_jacobi_zero(c, V, w, B, act, f, nullptr, a);
      for (int s = 1; s < c.vc.coarse_iters; ++s) {
        launch_jacobi_sweep(c, V, w, B, act, a, f, nullptr, bb);
        std::swap(a, bb);
      }
      break;
    }
    case HB_COARSE_DENSE:  // exact coarsest solve (inc/multigrid.hpp:84,95-104)
      launch_coarse_dense(c, L, B, act, f, out);
      break;
    case HB_COARSE_NET: {  // A4: U-Net on [H^2 Re f, H^2 Im f, kappa^2]
      if (c0 != 0) throw HbError{HB_ERR_STATE, "split V-cycle with a net coarse solver"};
      Net& n = c.nets[0];
      if (!n.set) throw HbError{HB_ERR_STATE, "coarse solver is the net but net slot 0 is not set"};
      const int H = L.ny, W = L.nx;
      const size_t np = size_t(B) * H * W;
      DBuf<float>& io = c.cn_io;  // staging: in (3 ch) + out (2 ch), NHWC
      io.ensure(np * 5);
      launch_pack_input(c, V, L.h * L.h, B, act, f, nullptr, io.p);
      net_forward_dev(c, 0, B, act, H, W, io.p, io.p + np * 3);
      launch_unpack_output(c, H * W, B, act, io.p + np * 3, out);
      break;
    }
    default:
      throw HbError{HB_ERR_ARG, "unknown coarse solver"};
  }
}

// c0: first column of this (sub-)batch within the level work buffers
static void vcycle_at(Context& c, int l, int B, int c0, const int* act, const float2* f, const float* fscale,
                      const float2* e0, float2* out) {
  const int nl = int(c.levels.size());
  if (l == nl - 1) {
    if (c.ev_at_coarse) {  // split V-cycle: release the second half-batch
      HB_CUDA(cudaEventRecord(c.ev_at_coarse, c.stream));
      c.ev_at_coarse = nullptr;
    }
    if (!(c.dbg_skip & 4)) coarsest_solve(c, B, c0, act, f, out);
    return;
  }
  Level& L = *c.levels[size_t(l)];
  Level& C = *c.levels[size_t(l + 1)];
  const LevelView V = L.view();
  const float w = float(c.vc.damping);
  const int offset = l % 2;
  const int nu1 = c.vc.nu1, nu2 = c.vc.nu2;
  float2* Cf = C.f.p + size_t(c0) * C.N();
  float2* Cx = C.x.p + size_t(c0) * C.N();
  if (c.opt_fused && nu1 == 1 && nu2 == 1) {
    // fused legs: v and r stay on chip (row-streaming kernels for a zero
    // initial guess, shared-memory tiles otherwise)
    const bool stream = c.opt_stream && (e0 == nullptr || c.opt_stream_e0) && L.nx >= 16;
    // staged legs from e0 (level 0): the down leg stores the pre-smoothed iterate
    // into the level's v buffer and the up leg reads it back instead of e0
    float2* vpre = (e0 && c.opt_vpre && L.rows == L.ny) ? L.v.p + size_t(c0) * L.N() : nullptr;
    const bool skip = c.dbg_skip & (l == 0 ? 1 : 2);
    if (skip) {
    } else if (stream)
      launch_down_stream(c, V, C.win(), w, offset, B, act, f, fscale, e0, Cf, vpre);
    else
      launch_down_fused(c, V, w, offset, B, act, f, fscale, e0, Cf);
    vcycle_at(c, l + 1, B, c0, act, Cf, nullptr, nullptr, Cx);
    if (skip) {
    } else if (stream)
      launch_up_stream(c, V, w, offset, C.nx, C.ny, C.win(), B, act, f, fscale, e0, Cx, out, vpre);
    else
      launch_up_fused(c, V, w, offset, C.nx, C.ny, B, act, f, fscale, e0, Cx, out);
    return;
  }
  float2* const Lv = L.v.p + size_t(c0) * L.N();
  float2* const Lt = L.t.p + size_t(c0) * L.N();
  float2* v = Lv;
  float2* t = Lt;
  // pre-smoothing (nu1 sweeps from e0 or zero)
  if (nu1 == 0) {
    if (e0)
      HB_CUDA(cudaMemcpyAsync(v, e0, sizeof(float2) * L.N() * B, cudaMemcpyDeviceToDevice, c.stream));
    else
      HB_CUDA(cudaMemsetAsync(v, 0, sizeof(float2) * L.N() * B, c.stream));
  } else {
    if (e0)
      launch_jacobi_sweep(c, V, w, B, act, e0, f, fscale, v);
    else
      launch_jacobi_zero(c, V, w, B, act, f, fscale, v);
    for (int s = 1; s < nu1; ++s) {
      launch_jacobi_sweep(c, V, w, B, act, v, f, fscale, t);
      std::swap(v, t);
    }
  }
  launch_residual_restrict(c, V, offset, B, act, v, f, fscale, Cf);
  vcycle_at(c, l + 1, B, c0, act, Cf, nullptr, nullptr, Cx);
  launch_prolong_add(c, V, C.nx, C.ny, offset, B, act, Cx, v);
  if (nu2 == 0) {
    HB_CUDA(cudaMemcpyAsync(out, v, sizeof(float2) * L.N() * B, cudaMemcpyDeviceToDevice, c.stream));
    return;
  }
  for (int s = 0; s < nu2; ++s) {
    float2* dst = (s == nu2 - 1) ? out : (v == Lv ? Lt : Lv);
    launch_jacobi_sweep(c, V, w, B, act, v, f, fscale, dst);
    v = dst;
  }
}

void vcycle(Context& c, int B, const int* act, const float2* f0, const float* fscale, const float2* e0, float2* z) {
  const bool split = c.opt_split && B >= 2 && c.vc.coarse_solver != HB_COARSE_NET && act != nullptr;
  if (!split) {
    vcycle_at(c, 0, B, 0, act, f0, fscale, e0, z);
    return;
  }
  // two half-batches on two streams (forked/joined with events; captured as
  // parallel graph branches): one half's latency-bound coarsest solve (one CTA
  // per column) overlaps the other half's bandwidth-bound fine-level legs
  // (Starting the second half only when the first reaches its coarsest level
  // -- staggering -- measured slower on B200; both halves start together.)
  const int Bh = B / 2;
  const size_t N0 = c.levels[0]->N();
  HB_CUDA(cudaEventRecord(c.ev_fork, c.stream));
  HB_CUDA(cudaStreamWaitEvent(c.stream2, c.ev_fork, 0));
  vcycle_at(c, 0, Bh, 0, act, f0, fscale, e0, z);
  cudaStream_t main = c.stream;
  c.stream = c.stream2;
  try {
    vcycle_at(c, 0, B - Bh, Bh, act + Bh, f0 + Bh * N0, fscale ? fscale + Bh : nullptr, e0 ? e0 + Bh * N0 : nullptr,
              z + Bh * N0);
  } catch (...) {
    c.stream = main;
    throw;
  }
  c.stream = main;
  HB_CUDA(cudaEventRecord(c.ev_join, c.stream2));
  HB_CUDA(cudaStreamWaitEvent(c.stream, c.ev_join, 0));
}

void precond_apply_dev(Context& c, int kind, int B, const int* act, const float2* r, const float* rscale,
                       float2* z) {
  if (kind == HB_PC_V) {
    vcycle(c, B, act, r, rscale, nullptr, z);
    return;
  }
  if (kind == HB_PC_JU) {
    // M_JU (inc/precond.hpp:112-130), damped Jacobi on A^h with omega = 0.8:
    // e1 = J_A(0, r); de = net(r - A e1) (fine-h packing, :74-83); z = J_A(e1 + de, r)
    const bool paper = paper_active(c);
    Net& n = c.nets[0];
    if (!n.set && !paper) throw HbError{HB_ERR_STATE, "M_JU needs net slot 0 or the paper net"};
    Level& L = *c.levels[0];
    LevelView VA = L.view();
    VA.dM = L.dA.p;  // Jacobi / residual on A^h, not the shifted M^h
    const size_t np = size_t(B) * L.N();
    if (paper) {  // the paper's network (inc/precond.hpp:112-130 with NetworkApplier, :57-98)
      DBuf<float2>& e1 = c.pc_e0;
      e1.ensure(np);
      c.pc_res.ensure(np);
      const float om = 0.8f;
      launch_jacobi_zero(c, VA, om, B, act, r, rscale, e1.p);
      launch_residual(c, VA, B, act, e1.p, r, rscale, c.pc_res.p);
      paper_infer(c, B, act, c.pc_res.p, nullptr, e1.p, e1.p);  // e2 = e1 + net(h^2 res)
      launch_jacobi_sweep(c, VA, om, B, act, e1.p, r, rscale, z);
      return;
    }
    DBuf<float>& io = c.pc_io;
    DBuf<float2>& e1 = c.pc_e0;
    io.ensure(np * 5 + np * 2);
    e1.ensure(np);
    float2* res = reinterpret_cast<float2*>(io.p + np * 5);
    const float om = 0.8f;
    launch_jacobi_zero(c, VA, om, B, act, r, rscale, e1.p);
    launch_residual(c, VA, B, act, e1.p, r, rscale, res);
    launch_pack_input(c, VA, L.h * L.h, B, act, res, nullptr, io.p);
    net_forward_dev(c, 0, B, act, L.ny, L.nx, io.p, io.p + np * 3);
    launch_unpack_add(c, int(L.N()), B, act, io.p + np * 3, e1.p, e1.p);  // e2 = e1 + de (in place)
    launch_jacobi_sweep(c, VA, om, B, act, e1.p, r, rscale, z);
    return;
  }
  if (kind != HB_PC_VU) throw HbError{HB_ERR_ARG, "unknown preconditioner kind"};
  // M_VU (inc/precond.hpp:151-158): e0 = net(h^2 r, kappa^2); z = cycle(e0, r)
  if (paper_active(c)) {  // UnetVCyclePreconditioner with the paper net (inc/precond.hpp:151-158)
    DBuf<float2>& e0 = c.pc_e0;
    e0.ensure(size_t(B) * c.levels[0]->N());
    paper_infer(c, B, act, r, rscale, nullptr, e0.p);
    vcycle(c, B, act, r, rscale, e0.p, z);
    return;
  }
  Net& n = c.nets[0];
  if (!n.set) throw HbError{HB_ERR_STATE, "M_VU needs net slot 0"};
  Level& L = *c.levels[0];
  const LevelView V = L.view();
  const size_t np = size_t(B) * L.N();
  DBuf<float>& io = c.pc_io;
  DBuf<float2>& e0 = c.pc_e0;
  io.ensure(np * 5);
  e0.ensure(np);
  launch_pack_input(c, V, L.h * L.h, B, act, r, rscale, io.p);
  net_forward_dev(c, 0, B, act, L.ny, L.nx, io.p, io.p + np * 3);
  launch_unpack_output(c, int(L.N()), B, act, io.p + np * 3, e0.p);
  vcycle(c, B, act, r, rscale, e0.p, z);
}

// ------------------------------------------------------------- FGMRES --
// name() / requires_flexible() of the reference plugins (inc/precond.hpp:14-27):
// network-based preconditioners are non-stationary (inc/precond.hpp:132,160)
static const char* precond_name(int kind) { return kind == HB_PC_VU ? "vu" : kind == HB_PC_JU ? "ju" : "v"; }
static bool requires_flexible(const Context& c, int kind) {
  return kind == HB_PC_VU || kind == HB_PC_JU || c.vc.coarse_solver == HB_COARSE_NET;
}

static void fgmres_dev(Context& c, const hb_krylov_cfg* cfg, int kind, int B, const double2* dB, double2* dX,
                       double* hist, int hist_stride, int* hist_len, int* iters, uint8_t* conv, uint8_t* brk,
                       const int* d_limits = nullptr) {
  require_hier(c);
  if (!cfg) throw HbError{HB_ERR_ARG, "null krylov config"};
  if (cfg->restart < 1) throw HbError{HB_ERR_ARG, "restart must be >= 1"};
  if (!(cfg->rel_tol > 0.0 && cfg->rel_tol < 1.0)) throw HbError{HB_ERR_ARG, "rel_tol in (0,1)"};
  // flexible = 0: standard right-preconditioned GMRES (inc/krylov.hpp:127-136) --
  // same Arnoldi, x += M (V y) at the end of each cycle; the preconditioner must be
  // stationary (check_flexible_contract, inc/precond.hpp:29-32)
  const bool flexible = cfg->flexible != 0;
  if (!flexible && requires_flexible(c, kind))
    throw HbError{HB_ERR_ARG, std::string("preconditioner ") + precond_name(kind) + " requires flexible = true"};
  if (B < 1) throw HbError{HB_ERR_ARG, "batch must be >= 1"};
  ensure_batch(c, B);
  const int m = cfg->restart;
  const int cap = std::max(1, cfg->max_iters + 2);
  krylov_alloc(c, B, m, cap, d_limits);
  const size_t N = c.levels[0]->N();
  const size_t BN = size_t(B) * N;
  if (!c.h_count) HB_CUDA(cudaMallocHost(&c.h_count, sizeof(int)));
  // profiling (eager) only: scale each launch's algorithmic bytes/flops by the
  // fraction of still-active columns -- frozen columns early-exit in every kernel
  std::vector<int> h_act;
  auto prof_active = [&]() {
    if (!c.prof_on) return;
    h_act.resize(size_t(B));
    HB_CUDA(cudaMemcpyAsync(h_act.data(), c.kact.p, sizeof(int) * size_t(B), cudaMemcpyDeviceToHost, c.stream));
    HB_CUDA(cudaStreamSynchronize(c.stream));
    int a = 0;
    for (int v : h_act) a += v != 0;
    c.prof_scale = double(a) / double(B);
  };
  auto cycle_body = [&]() {
    for (int j = 0; j < m; ++j) {
      prof_active();
      float2* Vj = c.kV.p + size_t(j) * BN;
      float2* Zj = c.kZ.p + size_t(j) * BN;
      precond_apply_dev(c, kind, B, c.kact.p, Vj, c.kscale.p, Zj);
      if (!(c.dbg_skip & 8)) launch_fg_adots(c, B, j, Zj, c.kW.p, c.kV.p);
      launch_fg_update(c, B, j, m, c.kW.p, c.kV.p, cap, cfg->rel_tol, cfg->max_iters);
    }
    prof_active();
    if (flexible) {
      if (!(c.dbg_skip & 16)) launch_fg_finalize(c, B, m, c.kZ.p, dX);
    } else {
      c.kfin.ensure(B);
      launch_fg_finalize_v(c, B, c.kV.p, c.kW.p, c.kfin.p);
      precond_apply_dev(c, kind, B, c.kfin.p, c.kW.p, nullptr, c.kZ.p);
      launch_fg_add_to_x(c, B, c.kfin.p, c.kZ.p, dX);
    }
    launch_fg_restart(c, B, dB, dX, c.kV.p, cap, cfg->rel_tol, cfg->max_iters);
    c.prof_scale = 1.0;
  };
  auto read_count = [&]() {
    HB_CUDA(cudaMemcpyAsync(c.h_count, c.kcount.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    HB_CUDA(cudaStreamSynchronize(c.stream));
    return *c.h_count;
  };
  launch_fg_restart(c, B, dB, dX, c.kV.p, cap, cfg->rel_tol, cfg->max_iters);
  if (read_count() == 0) {
    // nothing to do
  } else if (c.opt_graphs && !c.prof_on) {
    // one CUDA graph per restart cycle: m inner steps + finalize + next restart
    Context::GraphEntry* ge = nullptr;
    for (auto& g : c.graphs)
      if (g.gen == g_alloc_gen && g.kind == kind && g.B == B && g.m == m && g.cap == cap && g.flexible == flexible &&
          g.max_iters == cfg->max_iters && g.tol == cfg->rel_tol && g.dB == dB && g.dX == dX)
        ge = &g;
    bool more = true;
    if (!ge) {
      // first cycle of a new shape runs eagerly (lazy allocations happen here,
      // outside capture); the following cycles replay the captured graph
      cycle_body();
      more = read_count() > 0;
    }
    if (more && !ge) {
      cudaGraph_t graph;
      const int64_t l0 = c.launches;
      HB_CUDA(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
      try {
        cycle_body();
      } catch (...) {
        cudaStreamEndCapture(c.stream, &graph);
        throw;
      }
      HB_CUDA(cudaStreamEndCapture(c.stream, &graph));
      const int64_t per_cycle = c.launches - l0;  // captured, not yet executed
      c.launches = l0;
      cudaGraphExec_t exec;
      HB_CUDA(cudaGraphInstantiate(&exec, graph, 0));
      HB_CUDA(cudaGraphDestroy(graph));
      c.graphs.push_back(Context::GraphEntry{g_alloc_gen, kind, B, m, cap, cfg->max_iters, cfg->rel_tol, dB, dX,
                                             exec, per_cycle, flexible});
      ge = &c.graphs.back();
    }
    while (more) {
      HB_CUDA(cudaGraphLaunch(ge->exec, c.stream));
      c.launches += ge->launches;
      more = read_count() > 0;
    }
  } else {
    do {
      cycle_body();
    } while (read_count() > 0);
  }
  if (hist || hist_len || iters || conv || brk) krylov_report(c, B, hist, hist_stride, hist_len, iters, conv, brk);
}

void fgmres_dev_entry(Context& c, const hb_krylov_cfg* cfg, int kind, int B, const double2* dB, double2* dX,
                      const int* d_limits) {
  fgmres_dev(c, cfg, kind, B, dB, dX, nullptr, 0, nullptr, nullptr, nullptr, nullptr, d_limits);
}

}  // namespace hb

// ===================================================================== C ABI
using namespace hb;

struct hb_ctx : hb::Context {};

static std::string g_create_err;

#define HB_API_BEGIN \
  if (!ctx) return HB_ERR_ARG; \
  try {
#define HB_API_END                          \
  return HB_OK;                             \
  }                                         \
  catch (const HbError& e) {                \
    ctx->err = e.msg;                       \
    return e.code;                          \
  }                                         \
  catch (const std::exception& e) {         \
    ctx->err = e.what();                    \
    return HB_ERR_ARG;                      \
  }

extern "C" {

int hb_create(int device, hb_ctx** out) {
  if (!out) return HB_ERR_ARG;
  *out = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    g_create_err = std::string("no CUDA device: ") + cudaGetErrorString(e);
    return HB_ERR_CUDA;
  }
  if (device < 0 || device >= ndev) {
    g_create_err = "device index out of range";
    return HB_ERR_ARG;
  }
  cudaSetDevice(device);
  cudaDeviceProp prop{};
  cudaGetDeviceProperties(&prop, device);
  if (prop.major < 10) {
    g_create_err = "libhelmgpu is built for sm_100a (B200); found sm_" + std::to_string(prop.major) +
                   std::to_string(prop.minor);
    return HB_ERR_CUDA;
  }
  auto* c = new hb_ctx();
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  c->l2_bytes = size_t(prop.l2CacheSize);
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->stream2, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess) {
    g_create_err = "stream creation failed";
    delete c;
    return HB_ERR_CUDA;
  }
  c->prof.resize(PC_COUNT);
  for (int i = 0; i < PC_COUNT; ++i) c->prof[size_t(i)].name = kProfNames[i];
  *out = c;
  return HB_OK;
}

void hb_destroy(hb_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  for (auto& e : ctx->ev_pending) {
    cudaEventDestroy(e.second.first);
    cudaEventDestroy(e.second.second);
  }
  if (ctx->h_count) cudaFreeHost(ctx->h_count);
  for (auto& g : ctx->graphs) cudaGraphExecDestroy(g.exec);
  cudaStreamDestroy(ctx->stream_own ? ctx->stream_own : ctx->stream);
  cudaStreamDestroy(ctx->stream2);
  ctx->slab.reset();  // the last member of an in-process slab group releases the group stream
  cudaEventDestroy(ctx->ev_fork);
  cudaEventDestroy(ctx->ev_join);
  delete ctx;
}

const char* hb_last_error(const hb_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }
void* hb_stream(hb_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

int hb_synchronize(hb_ctx* ctx) {
  HB_API_BEGIN
  HB_CUDA(cudaStreamSynchronize(ctx->stream));
  HB_API_END
}

int hb_set_problem(hb_ctx* ctx, int nx, int ny, double h, double omega, const double* kappa2, const double* gamma,
                   double lo, double hi) {
  HB_API_BEGIN
  if (nx < 8 || ny < 8) throw HbError{HB_ERR_ARG, "grid must be at least 8x8"};
  if (!kappa2 || !gamma) throw HbError{HB_ERR_ARG, "null coefficient array"};
  if (!(lo < hi) || lo < 0.0) throw HbError{HB_ERR_ARG, "slowness range must satisfy 0 <= lo < hi"};
  if (omega < 0.0) throw HbError{HB_ERR_ARG, "omega must be nonnegative"};
  const size_t n = size_t(nx) * ny;
  double kmax = 0.0;
  for (size_t i = 0; i < n; ++i) {
    if (!(kappa2[i] >= lo - 1e-12 && kappa2[i] <= hi + 1e-12))
      throw HbError{HB_ERR_ARG, "slowness value outside declared range"};
    kmax = std::max(kmax, std::sqrt(kappa2[i]));
  }
  if (omega * kmax * h > 0.6284) throw HbError{HB_ERR_ARG, "discretization bound omega*kappa*h <= 0.628 violated"};
  ctx->nx = nx;
  ctx->ny = ny;
  ctx->h = h;
  ctx->omega = omega;
  ctx->klo = lo;
  ctx->khi = hi;
  ctx->k2.assign(kappa2, kappa2 + n);
  ctx->gam.assign(gamma, gamma + n);
  ctx->has_problem = true;
  ctx->has_hier = false;
  ctx->levels.clear();
  ctx->batch_cap = 0;
  ctx->ctx_valid = false;
  ctx->slab.reset();
  ++ctx->prob_gen;
  HB_API_END
}

int hb_build_hierarchy(hb_ctx* ctx, const hb_vcycle_cfg* cfg) {
  HB_API_BEGIN
  if (!ctx->has_problem) throw HbError{HB_ERR_STATE, "problem not set"};
  if (!cfg) throw HbError{HB_ERR_ARG, "null config"};
  if (cfg->levels < 2) throw HbError{HB_ERR_ARG, "levels must be >= 2"};
  if (cfg->nu1 + cfg->nu2 < 1 || cfg->nu1 < 0 || cfg->nu2 < 0) throw HbError{HB_ERR_ARG, "nu1 + nu2 must be >= 1"};
  if (!(cfg->damping > 0.0 && cfg->damping <= 1.0)) throw HbError{HB_ERR_ARG, "damping must be in (0,1]"};
  if (cfg->beta < 0.0) throw HbError{HB_ERR_ARG, "shift beta must be >= 0"};
  const int div = 1 << (cfg->levels - 1);
  if (ctx->nx % div || ctx->ny % div)
    throw HbError{HB_ERR_ARG, "grid does not support the configured level count"};
  if (cfg->coarse_solver == HB_COARSE_GMRES && (cfg->coarse_iters < 1 || cfg->coarse_iters > kMaxCoarseIters))
    throw HbError{HB_ERR_ARG, "coarse GMRES iterations must be in [1, 16]"};
  ctx->vc = *cfg;
  ctx->levels.clear();
  ctx->batch_cap = 0;
  auto L0 = std::make_unique<Level>();
  L0->nx = ctx->nx;
  L0->ny = ctx->ny;
  L0->h = ctx->h;
  L0->k2 = ctx->k2;
  L0->gam = ctx->gam;
  ctx->levels.push_back(std::move(L0));
  for (int l = 1; l < cfg->levels; ++l) {
    const Level& P = *ctx->levels.back();
    auto L = std::make_unique<Level>();
    L->nx = P.nx / 2;
    L->ny = P.ny / 2;
    L->h = P.h * 2.0;
    L->rows = L->hi = L->ny;  // whole grid (row slabs re-lay this in hb_slab.cu)
    L->k2.resize(L->N());
    L->gam.resize(L->N());
    const int off = (l - 1) % 2;
    restrict_real(P.k2.data(), P.nx, P.ny, off, L->k2.data());
    restrict_real(P.gam.data(), P.nx, P.ny, off, L->gam.data());
    for (double& x : L->k2) x = std::clamp(x, ctx->klo, ctx->khi);
    for (double& x : L->gam) x = std::max(x, 0.0);
    ctx->levels.push_back(std::move(L));
  }
  for (auto& L : ctx->levels) {
    L->row0 = L->lo = 0;
    L->rows = L->hi = L->ny;
  }
  ctx->slab.reset();
  for (size_t l = 0; l < ctx->levels.size(); ++l)
    fill_level_device(*ctx->levels[l], ctx->omega, cfg->alpha, cfg->beta, cfg->damping, l == 0,
                      l == int(ctx->levels.size()) - 1);
  if (cfg->coarse_solver == HB_COARSE_DENSE) build_dense_inverse(*ctx->levels.back(), ctx->omega, cfg->alpha, cfg->beta);
  ctx->has_hier = true;
  HB_API_END
}

int hb_level_info(hb_ctx* ctx, int level, int* nx, int* ny, double* h) {
  HB_API_BEGIN
  require_hier(*ctx);
  if (level < 0 || level >= int(ctx->levels.size())) throw HbError{HB_ERR_ARG, "level out of range"};
  const Level& L = *ctx->levels[size_t(level)];
  if (nx) *nx = L.nx;
  if (ny) *ny = L.ny;
  if (h) *h = L.h;
  HB_API_END
}

// ---- operator hooks (host c128 buffers, staged as c64) ----
static Level& level_at(hb_ctx* ctx, int level) {
  require_hier(*ctx);
  if (level < 0 || level >= int(ctx->levels.size())) throw HbError{HB_ERR_ARG, "level out of range"};
  return *ctx->levels[size_t(level)];
}

int hb_operator_apply(hb_ctx* ctx, int level, int shifted, int batch, const double* u, double* y) {
  HB_API_BEGIN
  require_whole(*ctx);
  Level& L = level_at(ctx, level);
  const size_t n = L.N() * size_t(batch);
  ctx->io_f.ensure(n);
  ctx->io_g.ensure(n);
  auto hu = to_c64(u, n);
  HB_CUDA(cudaMemcpyAsync(ctx->io_f.p, hu.data(), n * sizeof(float2), cudaMemcpyHostToDevice, ctx->stream));
  launch_apply(*ctx, L.view(), shifted ? 1 : 0, batch, nullptr, ctx->io_f.p, ctx->io_g.p, nullptr);
  HB_CUDA(cudaMemcpyAsync(hu.data(), ctx->io_g.p, n * sizeof(float2), cudaMemcpyDeviceToHost, ctx->stream));
  HB_CUDA(cudaStreamSynchronize(ctx->stream));
  from_c64(hu, y);
  HB_API_END
}

int hb_jacobi(hb_ctx* ctx, int level, int batch, double* v, const double* f, int iters) {
  HB_API_BEGIN
  require_whole(*ctx);
  Level& L = level_at(ctx, level);
  if (iters < 0) throw HbError{HB_ERR_ARG, "iters must be >= 0"};
  const size_t n = L.N() * size_t(batch);
  ctx->io_f.ensure(n);
  ctx->io_g.ensure(n);
  ctx->scratch_c64.ensure(n);
  auto hv = to_c64(v, n), hf = to_c64(f, n);
  HB_CUDA(cudaMemcpyAsync(ctx->io_f.p, hv.data(), n * sizeof(float2), cudaMemcpyHostToDevice, ctx->stream));
  HB_CUDA(cudaMemcpyAsync(ctx->io_g.p, hf.data(), n * sizeof(float2), cudaMemcpyHostToDevice, ctx->stream));
  float2* a = ctx->io_f.p;
  float2* b = ctx->scratch_c64.p;
  for (int s = 0; s < iters; ++s) {
    launch_jacobi_sweep(*ctx, L.view(), float(ctx->vc.damping), batch, nullptr, a, ctx->io_g.p, nullptr, b);
    std::swap(a, b);
  }
  HB_CUDA(cudaMemcpyAsync(hv.data(), a, n * sizeof(float2), cudaMemcpyDeviceToHost, ctx->stream));
  HB_CUDA(cudaStreamSynchronize(ctx->stream));
  from_c64(hv, v);
  HB_API_END
}

int hb_restrict(hb_ctx* ctx, int level, int batch, const double* fine, double* coarse) {
  HB_API_BEGIN
  require_whole(*ctx);
  Level& L = level_at(ctx, level);
  const size_t n = L.N() * size_t(batch), nc = n / 4;
  ctx->io_f.ensure(n);
  ctx->io_g.ensure(n);
  auto hf = to_c64(fine, n);
  HB_CUDA(cudaMemcpyAsync(ctx->io_f.p, hf.data(), n * sizeof(float2), cudaMemcpyHostToDevice, ctx->stream));
  launch_restrict_plain(*ctx, L.nx, L.ny, level % 2, batch, ctx->io_f.p, ctx->io_g.p);
  std::vector<float2> hc(nc);
  HB_CUDA(cudaMemcpyAsync(hc.data(), ctx->io_g.p, nc * sizeof(float2), cudaMemcpyDeviceToHost, ctx->stream));
  HB_CUDA(cudaStreamSynchronize(ctx->stream));
  from_c64(hc, coarse);
  HB_API_END
}

int hb_prolong(hb_ctx* ctx, int level, int batch, const double* coarse, double* fine) {
  HB_API_BEGIN
  require_whole(*ctx);
  Level& L = level_at(ctx, level);
  const size_t n = L.N() * size_t(batch), nc = n / 4;
  ctx->io_f.ensure(n);
  ctx->io_g.ensure(n);
  auto hc = to_c64(coarse, nc);
  HB_CUDA(cudaMemcpyAsync(ctx->io_f.p, hc.data(), nc * sizeof(float2), cudaMemcpyHostToDevice, ctx->stream));
  HB_CUDA(cudaMemsetAsync(ctx->io_g.p, 0, n * sizeof(float2), ctx->stream));
  launch_prolong_add(*ctx, L.view(), L.nx / 2, L.ny / 2, level % 2, batch, nullptr, ctx->io_f.p, ctx->io_g.p);
  std::vector<float2> hf(n);
  HB_CUDA(cudaMemcpyAsync(hf.data(), ctx->io_g.p, n * sizeof(float2), cudaMemcpyDeviceToHost, ctx->stream));
  HB_CUDA(cudaStreamSynchronize(ctx->stream));
  from_c64(hf, fine);
  HB_API_END
}

int hb_coarse_solve(hb_ctx* ctx, int batch, const double* f, double* x) {
  HB_API_BEGIN
  require_whole(*ctx);
  require_hier(*ctx);
  ensure_batch(*ctx, batch);
  Level& C = *ctx->levels.back();
  const size_t n = C.N() * size_t(batch);
  ctx->io_f.ensure(n);
  ctx->io_g.ensure(n);
  auto hf = to_c64(f, n);
  HB_CUDA(cudaMemcpyAsync(ctx->io_f.p, hf.data(), n * sizeof(float2), cudaMemcpyHostToDevice, ctx->stream));
  coarsest_solve(*ctx, batch, 0, ctx->act_all.p, ctx->io_f.p, ctx->io_g.p);
  HB_CUDA(cudaMemcpyAsync(hf.data(), ctx->io_g.p, n * sizeof(float2), cudaMemcpyDeviceToHost, ctx->stream));
  HB_CUDA(cudaStreamSynchronize(ctx->stream));
  from_c64(hf, x);
  HB_API_END
}

int hb_precond_apply(hb_ctx* ctx, int kind, int batch, const double* r, double* z) {
  HB_API_BEGIN
  require_whole(*ctx);
  require_hier(*ctx);
  if (batch < 1) throw HbError{HB_ERR_ARG, "batch must be >= 1"};
  ensure_batch(*ctx, batch);
  const size_t n = ctx->levels[0]->N() * size_t(batch);
  ctx->io_f.ensure(n);
  ctx->io_g.ensure(n);
  auto hr = to_c64(r, n);
  HB_CUDA(cudaMemcpyAsync(ctx->io_f.p, hr.data(), n * sizeof(float2), cudaMemcpyHostToDevice, ctx->stream));
  precond_apply_dev(*ctx, kind, batch, ctx->act_all.p, ctx->io_f.p, nullptr, ctx->io_g.p);
  HB_CUDA(cudaMemcpyAsync(hr.data(), ctx->io_g.p, n * sizeof(float2), cudaMemcpyDeviceToHost, ctx->stream));
  HB_CUDA(cudaStreamSynchronize(ctx->stream));
  from_c64(hr, z);
  HB_API_END
}

int hb_precond_apply_device(hb_ctx* ctx, int kind, int batch, const void* dr, void* dz) {
  HB_API_BEGIN
  require_whole(*ctx);
  require_hier(*ctx);
  if (batch < 1) throw HbError{HB_ERR_ARG, "batch must be >= 1"};
  if (!dr || !dz) throw HbError{HB_ERR_ARG, "null device buffer"};
  ensure_batch(*ctx, batch);
  precond_apply_dev(*ctx, kind, batch, ctx->act_all.p, static_cast<const float2*>(dr), nullptr,
                    static_cast<float2*>(dz));
  HB_CUDA(cudaGetLastError());
  HB_API_END
}

const char* hb_precond_name(int kind) { return precond_name(kind); }

int hb_precond_requires_flexible(hb_ctx* ctx, int kind) { return !ctx || requires_flexible(*ctx, kind) ? 1 : 0; }

int hb_fgmres(hb_ctx* ctx, const hb_krylov_cfg* cfg, int kind, int batch, const double* B, const double* X0,
              double* X, double* hist, int hist_stride, int* hist_len, int* iters, uint8_t* converged,
              uint8_t* breakdown) {
  HB_API_BEGIN
  require_whole(*ctx);
  require_hier(*ctx);
  if (!B || !X) throw HbError{HB_ERR_ARG, "null B or X"};
  const size_t n = ctx->levels[0]->N() * size_t(batch);
  ctx->kB.ensure(n);
  ctx->kX.ensure(n);
  HB_CUDA(cudaMemcpyAsync(ctx->kB.p, B, n * sizeof(double2), cudaMemcpyHostToDevice, ctx->stream));
  if (X0)
    HB_CUDA(cudaMemcpyAsync(ctx->kX.p, X0, n * sizeof(double2), cudaMemcpyHostToDevice, ctx->stream));
  else
    HB_CUDA(cudaMemsetAsync(ctx->kX.p, 0, n * sizeof(double2), ctx->stream));
  fgmres_dev(*ctx, cfg, kind, batch, ctx->kB.p, ctx->kX.p, hist, hist_stride, hist_len, iters, converged, breakdown);
  HB_CUDA(cudaMemcpyAsync(X, ctx->kX.p, n * sizeof(double2), cudaMemcpyDeviceToHost, ctx->stream));
  HB_CUDA(cudaStreamSynchronize(ctx->stream));
  HB_API_END
}

int hb_block_fgmres(hb_ctx* ctx, const hb_krylov_cfg* cfg, int kind, int batch, const double* B, const double* X0,
                    double* X, double* hist, int hist_stride, int* hist_len, int* iters, uint8_t* converged,
                    uint8_t* breakdown) {
  HB_API_BEGIN
  require_whole(*ctx);
  require_hier(*ctx);
  if (!cfg) throw HbError{HB_ERR_ARG, "null krylov config"};
  if (!cfg->flexible) throw HbError{HB_ERR_ARG, "block FGMRES is flexible (stores the preconditioned block)"};
  if (!B || !X) throw HbError{HB_ERR_ARG, "null B or X"};
  const size_t n = ctx->levels[0]->N() * size_t(batch);
  ctx->kB.ensure(n);
  ctx->kX.ensure(n);
  HB_CUDA(cudaMemcpyAsync(ctx->kB.p, B, n * sizeof(double2), cudaMemcpyHostToDevice, ctx->stream));
  if (X0)
    HB_CUDA(cudaMemcpyAsync(ctx->kX.p, X0, n * sizeof(double2), cudaMemcpyHostToDevice, ctx->stream));
  else
    HB_CUDA(cudaMemsetAsync(ctx->kX.p, 0, n * sizeof(double2), ctx->stream));
  block_fgmres_dev(*ctx, kind, batch, cfg->restart, cfg->max_iters, cfg->rel_tol, ctx->kB.p, ctx->kX.p, hist,
                   hist_stride, hist_len, iters, converged, breakdown);
  HB_CUDA(cudaMemcpyAsync(X, ctx->kX.p, n * sizeof(double2), cudaMemcpyDeviceToHost, ctx->stream));
  HB_CUDA(cudaStreamSynchronize(ctx->stream));
  HB_API_END
}

int hb_fgmres_device(hb_ctx* ctx, const hb_krylov_cfg* cfg, int kind, int batch, const void* dB, void* dX,
                     double* hist, int hist_stride, int* hist_len, int* iters, uint8_t* converged,
                     uint8_t* breakdown) {
  HB_API_BEGIN
  require_whole(*ctx);
  if (!dB || !dX) throw HbError{HB_ERR_ARG, "null device buffer"};
  fgmres_dev(*ctx, cfg, kind, batch, static_cast<const double2*>(dB), static_cast<double2*>(dX), hist, hist_stride,
             hist_len, iters, converged, breakdown);
  HB_API_END
}

// ---- setup helpers ----
void hb_rng_normals(uint64_t seed, int64_t n, double* out) {
  Rng r(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = r.normal();
}

int hb_absorbing_layer(int nx, int ny, int width, double gamma_max, double* out) {
  if (gamma_max < 0.0 || width < 0 || width > std::min(nx, ny) / 2 || !out) return HB_ERR_ARG;
  for (int iy = 0; iy < ny; ++iy)
    for (int ix = 0; ix < nx; ++ix) {
      const int d = std::min(std::min(ix, nx - 1 - ix), std::min(iy, ny - 1 - iy));
      double g = 0.0;
      if (width > 0 && d < width) {
        const double t = double(width - d) / double(width);
        g = gamma_max * t * t;
      }
      out[size_t(iy) * nx + ix] = g;
    }
  return HB_OK;
}

int hb_make_medium(int nx, int ny, uint64_t seed, double sigma, double vmin, double vmax, int n_interfaces,
                   uint64_t iface_seed, int iface_margin, double jmin, double jmax, double* kappa2) {
  if (nx < 1 || ny < 1 || !kappa2 || !(sigma > 0) || !(vmin < vmax)) return HB_ERR_ARG;
  const size_t n = size_t(nx) * ny;
  std::vector<double> f(n), c(n);
  Rng r(seed);
  for (auto& x : f) x = r.normal();
  gaussian_blur(f.data(), nx, ny, sigma, c.data());
  normalize_range(c, vmin, vmax);
  if (n_interfaces > 0) {
    Rng ir(iface_seed);
    for (int t = 0; t < n_interfaces; ++t) {
      const int row = int(ir.uniform_int(iface_margin, ny - iface_margin - 1));
      const double jump = jmin + (jmax - jmin) * ir.uniform();
      for (int iy = row; iy < ny; ++iy)
        for (int ix = 0; ix < nx; ++ix) c[size_t(iy) * nx + ix] += jump;
    }
    normalize_range(c, vmin, vmax);
  }
  for (size_t i = 0; i < n; ++i) kappa2[i] = 1.0 / (c[i] * c[i]);
  return HB_OK;
}

void hb_point_sources(uint64_t seed, int batch, int mode, int lo, int hi, int row, int* xs, int* ys) {
  Rng r(seed);
  for (int b = 0; b < batch; ++b) {
    if (mode == 0) {
      xs[b] = int(r.uniform_int(lo, hi));
      ys[b] = int(r.uniform_int(lo, hi));
    } else {
      xs[b] = int(r.uniform_int(lo, hi));
      ys[b] = row;
    }
  }
}

// ---- instrumentation ----
int hb_prof_enable(hb_ctx* ctx, int on) {
  HB_API_BEGIN
  if (!on) prof_collect(*ctx);
  ctx->prof_on = on != 0;
  HB_API_END
}
int hb_prof_reset(hb_ctx* ctx) {
  HB_API_BEGIN
  prof_collect(*ctx);
  for (auto& p : ctx->prof) {
    p.ms = 0;
    p.launches = 0;
    p.bytes = p.flops = 0;
  }
  ctx->launches = 0;
  HB_API_END
}
int hb_set_option(hb_ctx* ctx, const char* key, int64_t value) {
  HB_API_BEGIN
  if (!key) throw HbError{HB_ERR_ARG, "null option key"};
  const std::string k(key);
  // options change the captured kernel sequence: drop cached cycle graphs
  for (auto& g : ctx->graphs) cudaGraphExecDestroy(g.exec);
  ctx->graphs.clear();
  if (k == "fused_vcycle")
    ctx->opt_fused = value != 0;
  else if (k == "cuda_graphs")
    ctx->opt_graphs = value != 0;
  else if (k == "small_coarse")
    ctx->opt_small_coarse = value != 0;
  else if (k == "split_vcycle")
    ctx->opt_split = value != 0;
  else if (k == "tc_conv")
    ctx->opt_tc_conv = value != 0;
  else if (k == "conv_ksplit")
    ctx->opt_conv_ksplit = value != 0;
  else if (k == "tconv_par4")
    ctx->opt_tconv_par4 = value != 0;
  else if (k == "ctx_pre")
    ctx->opt_ctx_pre = value != 0;
  else if (k == "row_legs")
    ctx->opt_row_legs = value != 0;
  else if (k == "coarse_reg")
    ctx->opt_coarse_reg = value != 0;
  else if (k == "legs_wd")
    ctx->opt_legs_wd = int(value);
  else if (k == "pdl")
    ctx->opt_pdl = value != 0;
  else if (k == "basis_wave")
    ctx->opt_basis_wave = value != 0;
  else if (k == "coarse_krylov")
    ctx->opt_coarse_krylov = value != 0;
  else if (k == "coarse_cluster")
    ctx->opt_coarse_cluster = value != 0;
  else if (k == "lean_legs")
    ctx->opt_lean_legs = value != 0;
  else if (k == "conv_rows")
    ctx->opt_conv_rows = value != 0;
  else if (k == "stream_vcycle")
    ctx->opt_stream = value != 0;
  else if (k == "wgrad_blk")
    ctx->opt_wgrad_blk = value != 0;
  else if (k == "small_pw")
    ctx->opt_small_pw = value != 0;
  else if (k == "conv_cols")
    ctx->opt_conv_cols = value != 0;
  else if (k == "vpre")
    ctx->opt_vpre = value != 0;
  else if (k == "staged_legs")
    ctx->opt_staged_legs = int(value);
  else if (k == "debug_skip")
    ctx->dbg_skip = int(value);
  else if (k == "stream_e0")
    ctx->opt_stream_e0 = value != 0;
  else
    throw HbError{HB_ERR_ARG, "unknown option " + k};
  HB_API_END
}

int hb_prof_detail(hb_ctx* ctx, int on, char* buf, int cap) {
  HB_API_BEGIN
  prof_collect(*ctx);
  if (buf && cap > 0) {
    std::string s;
    for (const auto& d : ctx->detail_done)
      s += d.label + "," + std::to_string(d.ms * 1e3) + "," + std::to_string(d.bytes) + "," + std::to_string(d.flops) +
           "\n";
    const size_t n = std::min(s.size(), size_t(cap - 1));
    std::memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
  ctx->detail_done.clear();
  ctx->prof_detail = on != 0;
  HB_API_END
}

int hb_prof_count(hb_ctx* ctx) { return ctx ? int(ctx->prof.size()) : 0; }
const char* hb_prof_name(hb_ctx* ctx, int i) {
  return (ctx && i >= 0 && i < int(ctx->prof.size())) ? ctx->prof[size_t(i)].name.c_str() : "";
}
int hb_prof_get(hb_ctx* ctx, int i, double* total_ms, int64_t* launches, double* bytes, double* flops) {
  HB_API_BEGIN
  prof_collect(*ctx);
  if (i < 0 || i >= int(ctx->prof.size())) throw HbError{HB_ERR_ARG, "bad profile index"};
  const Prof& p = ctx->prof[size_t(i)];
  if (total_ms) *total_ms = p.ms;
  if (launches) *launches = p.launches;
  if (bytes) *bytes = p.bytes;
  if (flops) *flops = p.flops;
  HB_API_END
}
int64_t hb_launch_count(hb_ctx* ctx) { return ctx ? ctx->launches : 0; }

}  // extern "C"
