// helmgpu_helm.hpp -- drop-in adapters that put libhelmgpu (include/helmgpu.h)
// behind the reference's own C++ plugin and solver API
// (/root/reference/proj/include/helmbench, "inc/"):
//
//   helm::gpu::Context                 one hb_ctx (one GPU), RAII
//   helm::gpu::GpuSLVCycle             : helm::Preconditioner   (M_V, inc/precond.hpp:35-53;
//                                        with a net coarse solver: the SURVEY A4 coarse-net cycle)
//   helm::gpu::GpuUnetVCycle           : helm::Preconditioner   (M_VU, inc/precond.hpp:143-165)
//   helm::gpu::GpuJacobiUnet           : helm::Preconditioner   (M_JU, inc/precond.hpp:104-139)
//   helm::gpu::make_jacobi_unet / make_unet_vcycle
//                                      the reference constructors (problem / hierarchy, shared
//                                      NetworkWeights, UNetConfig, NetVariant) on the device with the
//                                      paper U-Net (inc/unet.hpp:113-257)
//   helm::gpu::block_fgmres(M, B, cfg) device-resident block_fgmres (inc/krylov.hpp:83-86)
//   helm::gpu::block_fgmres(apply_A, M, B, cfg) the reference signature (apply_A must be A^h)
//   helm::gpu::block_fgmres_shared_space(M, B, cfg) true block FGMRES (one block Krylov space)
//
// Error convention of the reference: contract violations throw
// std::invalid_argument, device / numeric failures std::runtime_error.
// Header-only; include after (or instead of) helmbench/precond.hpp.
#pragma once
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "helmbench/precond.hpp"
#include "helmgpu.h"

namespace helm {
namespace gpu {

inline void check(hb_ctx* c, int rc) {
  if (rc == HB_OK) return;
  const std::string msg = hb_last_error(c);
  if (rc == HB_ERR_ARG) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

class Context {
 public:
  explicit Context(int device = 0) {
    const int rc = hb_create(device, &c_);
    if (rc != HB_OK) throw std::runtime_error(std::string("hb_create: ") + hb_last_error(nullptr));
  }
  ~Context() { hb_destroy(c_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  hb_ctx* get() const { return c_; }

  // HelmholtzProblem (inc/grid.hpp:121-126) -> device; VCycleConfig (inc/multigrid.hpp:13-21)
  void set_problem(const HelmholtzProblem& p, const VCycleConfig& vc, int coarse_solver_override = -1) {
    check(c_, hb_set_problem(c_, p.grid.nx, p.grid.ny, p.grid.h, p.omega, p.kappa2.values.v.data(),
                             p.gamma.values.v.data(), p.kappa2.lo, p.kappa2.hi));
    const int coarse = coarse_solver_override >= 0                   ? coarse_solver_override
                       : vc.coarse_solver == CoarseSolver::dense ? HB_COARSE_DENSE
                                                                   : HB_COARSE_GMRES;
    hb_vcycle_cfg cfg{vc.levels, vc.nu1, vc.nu2, vc.damping, vc.shift.alpha, vc.shift.beta, coarse, vc.coarse_iters};
    check(c_, hb_build_hierarchy(c_, &cfg));
    nx_ = p.grid.nx;
    ny_ = p.grid.ny;
  }
  // classic U-Net in slot 0 (solver / coarse net) or 1 (encoder), He-normal from a seed
  void set_net(int slot, const hb_net_cfg& cfg, uint64_t he_seed) {
    check(c_, hb_set_net(c_, slot, &cfg));
    check(c_, hb_init_net_he(c_, slot, he_seed));
  }
  // the paper's U-Net (inc/unet.hpp:113-257) with the reference's own weights
  // registry: every parameter copied by name (dims checked); M_JU / M_VU then use it
  void set_paper_net(const UNetConfig& cfg, NetVariant variant, const NetworkWeights& w) {
    const hb_unet_cfg c{cfg.levels, cfg.base_channels, cfg.resnet_per_level, cfg.bottleneck_resnets,
                        cfg.updown_kernel, cfg.res_kernel};
    check(c_, hb_set_paper_net(c_, &c, variant == NetVariant::encoder_solver ? 1 : 0));
    for (std::size_t i = 0; i < w.size(); ++i) {
      const Param& p = w.at(i);
      if (p.name.rfind("adam.", 0) == 0) continue;
      check(c_, hb_paper_param(c_, p.name.c_str(), int64_t(p.value.v.size()), p.value.v.data(), nullptr));
    }
  }
  // UNW1 checkpoint written by save_checkpoint (inc/checkpoint.hpp:57-104)
  void load_checkpoint(const UNetConfig& cfg, NetVariant variant, const std::string& path) {
    const hb_unet_cfg c{cfg.levels, cfg.base_channels, cfg.resnet_per_level, cfg.bottleneck_resnets,
                        cfg.updown_kernel, cfg.res_kernel};
    check(c_, hb_set_paper_net(c_, &c, variant == NetVariant::encoder_solver ? 1 : 0));
    check(c_, hb_load_checkpoint(c_, path.c_str()));
  }
  int nx() const { return nx_; }
  int ny() const { return ny_; }

 private:
  hb_ctx* c_ = nullptr;
  int nx_ = 0, ny_ = 0;
};

namespace detail {
inline std::vector<double> pack(const std::vector<ComplexField>& r) {
  std::vector<double> out;
  out.reserve(r.size() * r[0].v.size() * 2);
  for (const auto& f : r)
    for (const auto& z : f.v) {
      out.push_back(z.real());
      out.push_back(z.imag());
    }
  return out;
}
inline std::vector<ComplexField> unpack(const std::vector<double>& buf, int nb, int nx, int ny) {
  std::vector<ComplexField> out;
  out.reserve(size_t(nb));
  const size_t n = size_t(nx) * ny;
  for (int b = 0; b < nb; ++b) {
    ComplexField f(nx, ny);
    for (size_t i = 0; i < n; ++i) f.v[i] = Complex(buf[2 * (b * n + i)], buf[2 * (b * n + i) + 1]);
    out.push_back(std::move(f));
  }
  return out;
}
}  // namespace detail

// Batched preconditioner plugin: the reference's Preconditioner interface,
// computed by the device (host buffers in and out per apply -- the parity
// path; block_fgmres below keeps everything resident).
class GpuPreconditioner : public Preconditioner {
 public:
  GpuPreconditioner(std::shared_ptr<Context> ctx, int kind) : ctx_(std::move(ctx)), kind_(kind) {}
  std::vector<ComplexField> apply(const std::vector<ComplexField>& r) override {
    if (r.empty()) return {};
    for (const auto& f : r)
      if (f.nx != ctx_->nx() || f.ny != ctx_->ny()) throw std::invalid_argument("field shape mismatch");
    const auto in = detail::pack(r);
    std::vector<double> out(in.size());
    check(ctx_->get(), hb_precond_apply(ctx_->get(), kind_, int(r.size()), in.data(), out.data()));
    return detail::unpack(out, int(r.size()), ctx_->nx(), ctx_->ny());
  }
  bool requires_flexible() const override { return hb_precond_requires_flexible(ctx_->get(), kind_) != 0; }
  std::string name() const override { return hb_precond_name(kind_); }
  int kind() const { return kind_; }
  Context& context() const { return *ctx_; }

 private:
  std::shared_ptr<Context> ctx_;
  int kind_;
};

class GpuSLVCycle : public GpuPreconditioner {
 public:
  explicit GpuSLVCycle(std::shared_ptr<Context> ctx) : GpuPreconditioner(std::move(ctx), HB_PC_V) {}
};

class GpuUnetVCycle : public GpuPreconditioner {
 public:
  explicit GpuUnetVCycle(std::shared_ptr<Context> ctx) : GpuPreconditioner(std::move(ctx), HB_PC_VU) {}
};

// drop-in for JacobiUnetPreconditioner (inc/precond.hpp:104-139), name() == "ju"
class GpuJacobiUnet : public GpuPreconditioner {
 public:
  explicit GpuJacobiUnet(std::shared_ptr<Context> ctx) : GpuPreconditioner(std::move(ctx), HB_PC_JU) {}
};

// JacobiUnetPreconditioner(problem, weights, cfg, variant) (inc/precond.hpp:106-110)
// and UnetVCyclePreconditioner(hier, weights, cfg, variant) (:145-149) on one
// device: same arguments, the network is the paper U-Net with those weights.
inline GpuJacobiUnet make_jacobi_unet(const HelmholtzProblem& problem, std::shared_ptr<NetworkWeights> weights,
                                      UNetConfig cfg, NetVariant variant, int device = 0) {
  auto ctx = std::make_shared<Context>(device);
  VCycleConfig vc;
  vc.levels = 2;  // M_JU runs on the fine grid only; the hierarchy is the minimal one
  ctx->set_problem(problem, vc);
  ctx->set_paper_net(cfg, variant, *weights);
  return GpuJacobiUnet(std::move(ctx));
}
inline GpuUnetVCycle make_unet_vcycle(const HelmholtzProblem& problem, const VCycleConfig& vc,
                                      std::shared_ptr<NetworkWeights> weights, UNetConfig cfg, NetVariant variant,
                                      int device = 0) {
  auto ctx = std::make_shared<Context>(device);
  ctx->set_problem(problem, vc);
  ctx->set_paper_net(cfg, variant, *weights);
  return GpuUnetVCycle(std::move(ctx));
}

// Device-resident block FGMRES with A = A^h of the context's problem and M =
// the plugin; same contract and SolveReport as inc/krylov.hpp:83-267.
// cfg.flexible = false runs standard right-preconditioned GMRES (x += M V y,
// inc/krylov.hpp:127-136) on the device; network preconditioners throw
// std::invalid_argument there, as check_flexible_contract does.
inline std::pair<std::vector<ComplexField>, SolveReport> block_fgmres(GpuPreconditioner& M,
                                                                      const std::vector<ComplexField>& B,
                                                                      const KrylovConfig& cfg,
                                                                      const std::vector<ComplexField>* X0 = nullptr) {
  check_flexible_contract(cfg, M);
  if (cfg.restart < 1) throw std::invalid_argument("restart must be >= 1");
  if (!(cfg.rel_tol > 0.0 && cfg.rel_tol < 1.0)) throw std::invalid_argument("rel_tol in (0,1)");
  Context& c = M.context();
  const int nb = int(B.size());
  if (nb == 0) return {{}, SolveReport{}};
  const auto b = detail::pack(B);
  std::vector<double> x0;
  if (X0) x0 = detail::pack(*X0);
  std::vector<double> x(b.size());
  const int cap = cfg.max_iters + 2;
  std::vector<double> hist(size_t(nb) * cap);
  std::vector<int> hl(nb), it(nb);
  std::vector<uint8_t> cv(nb), bk(nb);
  hb_krylov_cfg kc{cfg.restart, cfg.max_iters, cfg.rel_tol, cfg.flexible ? 1 : 0};
  check(c.get(), hb_fgmres(c.get(), &kc, M.kind(), nb, b.data(), X0 ? x0.data() : nullptr, x.data(), hist.data(),
                           cap, hl.data(), it.data(), cv.data(), bk.data()));
  SolveReport rep;
  rep.residual_history.resize(size_t(nb));
  for (int q = 0; q < nb; ++q)
    rep.residual_history[size_t(q)].assign(hist.begin() + size_t(q) * cap, hist.begin() + size_t(q) * cap + hl[size_t(q)]);
  rep.iterations.assign(it.begin(), it.end());
  rep.converged.assign(cv.begin(), cv.end());
  rep.breakdown.assign(bk.begin(), bk.end());
  return {detail::unpack(x, nb, c.nx(), c.ny()), std::move(rep)};
}

// True block FGMRES on the device (hb_block_fgmres): the
// columns of B (<= 16) share one block Krylov space; cfg.restart / max_iters
// count block steps; every column reports the same iteration count.
inline std::pair<std::vector<ComplexField>, SolveReport> block_fgmres_shared_space(
    GpuPreconditioner& M, const std::vector<ComplexField>& B, const KrylovConfig& cfg,
    const std::vector<ComplexField>* X0 = nullptr) {
  if (cfg.restart < 1) throw std::invalid_argument("restart must be >= 1");
  if (!(cfg.rel_tol > 0.0 && cfg.rel_tol < 1.0)) throw std::invalid_argument("rel_tol in (0,1)");
  Context& c = M.context();
  const int nb = int(B.size());
  if (nb == 0) return {{}, SolveReport{}};
  const auto b = detail::pack(B);
  std::vector<double> x0;
  if (X0) x0 = detail::pack(*X0);
  std::vector<double> x(b.size());
  const int cap = cfg.max_iters + 2;
  std::vector<double> hist(size_t(nb) * cap);
  std::vector<int> hl(nb), it(nb);
  std::vector<uint8_t> cv(nb), bk(nb);
  hb_krylov_cfg kc{cfg.restart, cfg.max_iters, cfg.rel_tol, 1};
  check(c.get(), hb_block_fgmres(c.get(), &kc, M.kind(), nb, b.data(), X0 ? x0.data() : nullptr, x.data(),
                                 hist.data(), cap, hl.data(), it.data(), cv.data(), bk.data()));
  SolveReport rep;
  rep.residual_history.resize(size_t(nb));
  for (int q = 0; q < nb; ++q)
    rep.residual_history[size_t(q)].assign(hist.begin() + size_t(q) * cap, hist.begin() + size_t(q) * cap + hl[size_t(q)]);
  rep.iterations.assign(it.begin(), it.end());
  rep.converged.assign(cv.begin(), cv.end());
  rep.breakdown.assign(bk.begin(), bk.end());
  return {detail::unpack(x, nb, c.nx(), c.ny()), std::move(rep)};
}

// The reference signature block_fgmres(apply_A, apply_M, B, cfg, X0)
// (inc/krylov.hpp:83-86) with M a device plugin.  The device solve applies
// A^h of M's context itself, so apply_A must BE that operator: it is probed
// once on a seeded random field against hb_operator_apply (relative L2
// difference <= 1e-5: the device applies it in complex64) and a different operator is rejected with std::invalid_argument
// (no host-callback Krylov path exists on the device).
inline std::pair<std::vector<ComplexField>, SolveReport> block_fgmres(const BatchedOp& apply_A,
                                                                      GpuPreconditioner& M,
                                                                      const std::vector<ComplexField>& B,
                                                                      const KrylovConfig& cfg,
                                                                      const std::vector<ComplexField>* X0 = nullptr) {
  Context& c = M.context();
  if (!B.empty()) {
    Rng rng(0x5eedULL);
    ComplexField u(c.nx(), c.ny());
    for (auto& z : u.v) z = Complex(rng.normal(), rng.normal());
    const auto host = apply_A(std::vector<ComplexField>{u});
    if (host.size() != 1 || host[0].nx != c.nx() || host[0].ny != c.ny())
      throw std::invalid_argument("apply_A returned a batch of the wrong shape");
    const auto in = detail::pack({u});
    std::vector<double> dev(in.size());
    check(c.get(), hb_operator_apply(c.get(), 0, 0, 1, in.data(), dev.data()));
    double num = 0.0, den = 0.0;
    for (std::size_t i = 0; i < host[0].v.size(); ++i) {
      const Complex d(dev[2 * i], dev[2 * i + 1]);
      num += std::norm(host[0].v[i] - d);
      den += std::norm(host[0].v[i]);
    }
    if (!(num <= 1e-10 * den))
      throw std::invalid_argument("apply_A is not the Helmholtz operator A^h of the preconditioner's problem");
  }
  return block_fgmres(M, B, cfg, X0);
}

}  // namespace gpu
}  // namespace helm
