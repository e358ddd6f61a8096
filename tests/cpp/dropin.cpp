// Drop-in check at the C++ plugin boundary (built against the UNMODIFIED
// reference headers; see tests/cpp/build.sh).  The GPU preconditioner is
// plugged into the reference's own block_fgmres through helm::Preconditioner,
// and the device-resident helm::gpu::block_fgmres is run beside the reference
// CPU solve on the same problem.
#include <cmath>
#include <cstdio>
#include <memory>

#include "helmbench/grid.hpp"
#include "helmbench/krylov.hpp"
#include "helmbench/multigrid.hpp"
#include "helmbench/precond.hpp"
#include "helmbench/rng.hpp"
#include "helmbench/unet.hpp"
#include "helmgpu_helm.hpp"

using namespace helm;

static double rel(const std::vector<ComplexField>& a, const std::vector<ComplexField>& b) {
  double num = 0, den = 0;
  for (size_t c = 0; c < a.size(); ++c)
    for (size_t i = 0; i < a[c].v.size(); ++i) {
      num += std::norm(a[c].v[i] - b[c].v[i]);
      den += std::norm(b[c].v[i]);
    }
  return std::sqrt(num / den);
}

int main() {
  const int n = 64;
  const double omega = 2 * M_PI * 1.5 * n / 10;
  auto grid = make_grid(n, n, 3);
  RealField k2(n, n);
  for (int iy = 0; iy < n; ++iy)
    for (int ix = 0; ix < n; ++ix) {  // smooth velocity in [1.5, 4] -> kappa^2 = 1/c^2
      const double x = double(ix) / n, y = double(iy) / n;
      const double c = 2.75 + 1.25 * std::sin(3.1 * x + 1.0) * std::cos(2.3 * y);
      k2.at(ix, iy) = 1.0 / (c * c);
    }
  auto prob = make_problem(grid, omega, make_slowness_squared(std::move(k2), 1.0 / 16, 1.0 / 2.25),
                           make_absorbing_layer(grid, 8, 2 * omega));
  VCycleConfig vc;  // 3 levels, V(1,1), damping 0.8, shift (1, 0.5), GMRES(10) coarsest
  auto hier = std::make_shared<MultigridHierarchy>(prob, vc);
  SLVCyclePreconditioner M_cpu(hier);
  StencilOperator A(prob, kHelmholtzShift);
  BatchedOp apply_A = [&A](const std::vector<ComplexField>& in) {
    std::vector<ComplexField> out;
    for (const auto& f : in) out.push_back(A.apply(f));
    return out;
  };
  std::vector<ComplexField> B;
  Rng rng(7);
  for (int c = 0; c < 2; ++c) {
    ComplexField f(n, n);
    for (auto& z : f.v) z = Complex(rng.normal(), rng.normal());
    B.push_back(std::move(f));
  }
  ComplexField pt(n, n);
  pt.at(n / 2, n / 2) = 1.0;
  B.push_back(pt);
  KrylovConfig cfg;
  cfg.restart = 10;
  cfg.max_iters = 300;

  auto [X_ref, rep_ref] = block_fgmres(apply_A, M_cpu.as_batched_op(), B, cfg);

  auto ctx = std::make_shared<gpu::Context>(0);
  ctx->set_problem(prob, vc);
  gpu::GpuSLVCycle M_gpu(ctx);
  // (1) GPU plugin inside the reference's CPU block_fgmres
  auto [X_mix, rep_mix] = block_fgmres(apply_A, M_gpu.as_batched_op(), B, cfg);
  // (2) device-resident solve behind the reference's signature
  auto [X_gpu, rep_gpu] = gpu::block_fgmres(M_gpu, B, cfg);
  // (3) single preconditioner apply parity
  const double pc_err = rel(M_gpu.apply(B), M_cpu.apply(B));

  bool ok = pc_err < 1e-4;
  std::printf("{\"pc_rel\": %.3e, \"cols\": [", pc_err);
  for (size_t c = 0; c < B.size(); ++c) {
    const int d1 = rep_mix.iterations[c] - rep_ref.iterations[c], d2 = rep_gpu.iterations[c] - rep_ref.iterations[c];
    ok = ok && std::abs(d1) <= 1 && std::abs(d2) <= 1 && rep_gpu.converged[c];
    std::printf("%s{\"ref\": %d, \"plugin\": %d, \"device\": %d}", c ? ", " : "", rep_ref.iterations[c],
                rep_mix.iterations[c], rep_gpu.iterations[c]);
  }
  const double xe = rel(X_gpu, X_ref), xm = rel(X_mix, X_ref);
  ok = ok && xe < 1e-4 && xm < 1e-4 && M_gpu.name() == M_cpu.name();

  // (4) the paper U-Net preconditioners from the reference's own weights
  // registry: the reference constructors vs the device drop-ins
  UNetConfig ucfg;  // 3 levels, base 16, 1 ResNet per level, 3 bottleneck ResNets, 5x5 / 3x3
  ucfg.bottleneck_resnets = 1;
  auto w = std::make_shared<NetworkWeights>(1234);
  {
    Tensor4 x(1, 4, n, n, 0.1f);
    unet_forward(*w, ucfg, x, true);  // creates the parameters (registry order), one running-stat update
  }
  mark_bn_initialized(*w);
  JacobiUnetPreconditioner ju_cpu(prob, w, ucfg, NetVariant::standalone);
  auto ju_gpu = gpu::make_jacobi_unet(prob, w, ucfg, NetVariant::standalone);
  UnetVCyclePreconditioner vu_cpu(hier, w, ucfg, NetVariant::standalone);
  auto vu_gpu = gpu::make_unet_vcycle(prob, vc, w, ucfg, NetVariant::standalone);
  const double ju_err = rel(ju_gpu.apply(B), ju_cpu.apply(B)), vu_err = rel(vu_gpu.apply(B), vu_cpu.apply(B));
  ok = ok && ju_err < 1e-4 && vu_err < 1e-4 && ju_gpu.name() == "ju" && vu_gpu.name() == "vu" &&
       ju_gpu.requires_flexible() && vu_gpu.requires_flexible();
  // (5) the reference signature with apply_A: the Helmholtz operator is accepted
  // (same solve as (2)), any other operator is rejected
  auto [X_a, rep_a] = gpu::block_fgmres(apply_A, M_gpu, B, cfg);
  ok = ok && rel(X_a, X_gpu) == 0.0;
  StencilOperator Ms(prob, kShiftedLaplacianShift);
  BatchedOp apply_wrong = [&Ms](const std::vector<ComplexField>& in) {
    std::vector<ComplexField> out;
    for (const auto& f : in) out.push_back(Ms.apply(f));
    return out;
  };
  bool rejected = false;
  try {
    gpu::block_fgmres(apply_wrong, M_gpu, B, cfg);
  } catch (const std::invalid_argument&) {
    rejected = true;
  }
  ok = ok && rejected;
  // (6) standard (non-flexible) GMRES with a stationary M: the dense coarsest
  // solve makes M_V exactly linear (tests/test_classic.cpp:442-467); the device
  // honours cfg.flexible = false and matches the reference's non-flexible solve
  VCycleConfig vd = vc;
  vd.coarse_solver = CoarseSolver::dense;
  auto hier_d = std::make_shared<MultigridHierarchy>(prob, vd);
  SLVCyclePreconditioner Md_cpu(hier_d);
  auto ctx_d = std::make_shared<gpu::Context>(0);
  ctx_d->set_problem(prob, vd);
  gpu::GpuSLVCycle Md_gpu(ctx_d);
  KrylovConfig cs = cfg;
  cs.flexible = false;
  auto [X_sr, rep_sr] = block_fgmres(apply_A, Md_cpu.as_batched_op(), B, cs);
  auto [X_sg, rep_sg] = gpu::block_fgmres(Md_gpu, B, cs);
  const double d_pc = rel(Md_gpu.apply(B), Md_cpu.apply(B)), d_x = rel(X_sg, X_sr);
  int d_it = 0;
  for (size_t c = 0; c < B.size(); ++c) d_it = std::max(d_it, std::abs(rep_sg.iterations[c] - rep_sr.iterations[c]));
  ok = ok && d_pc < 1e-4 && d_x < 1e-4 && d_it <= 1;
  bool nonflex_rejected = false;
  try {
    gpu::block_fgmres(vu_gpu, B, cs);
  } catch (const std::invalid_argument&) {
    nonflex_rejected = true;
  }
  ok = ok && nonflex_rejected;
  // (7) true block FGMRES: converged solutions of the same system
  auto [X_bk, rep_bk] = gpu::block_fgmres_shared_space(M_gpu, B, cfg);
  const double bk_rel = rel(X_bk, X_ref);
  ok = ok && bk_rel < 1e-4 && rep_bk.converged[0] && rep_bk.iterations[0] <= rep_ref.iterations[0];
  std::printf("], \"x_rel_device\": %.3e, \"x_rel_plugin\": %.3e, \"name\": \"%s\", \"ju_rel\": %.3e, "
              "\"vu_rel\": %.3e, \"apply_A_rejects_wrong_op\": %s, \"dense_pc_rel\": %.3e, "
              "\"nonflex_x_rel\": %.3e, \"nonflex_iter_diff\": %d, \"vu_nonflex_rejected\": %s, "
              "\"block_x_rel\": %.3e, \"block_iters\": %d, \"ok\": %s}\n",
              xe, xm, M_gpu.name().c_str(), ju_err, vu_err, rejected ? "true" : "false", d_pc, d_x, d_it,
              nonflex_rejected ? "true" : "false", bk_rel, rep_bk.iterations[0], ok ? "true" : "false");
  return ok ? 0 : 1;
}
