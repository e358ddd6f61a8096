// ref_capi.cpp -- C ABI over the UNMODIFIED reference headers
// (/root/reference/proj/include/helmbench, compiled in place; nothing copied).
// TEST INFRASTRUCTURE: built by oracle/build_ref.sh into oracle/_ref/ to pin the
// C restatement (oracle/helm_oracle.c) and to serve as the CPU reference arm of
// bench.py (--impl reference).  Entry points mirror oracle/helm_oracle.c.
//
// The BASELINE-config extensions are assembled here from
// reference primitives only: Tape::conv2d / Tape::concat (inc/autodiff.hpp:124,403),
// bilinear_resize (inc/datagen.hpp:19), StencilOperator::jacobi/residual,
// restrict_field/prolong_field (inc/stencil.hpp:69-165), MultigridHierarchy
// (inc/multigrid.hpp:70-125), block_fgmres (inc/krylov.hpp:83), Rng
// (inc/rng.hpp).  New forward-only ops (ReLU, 2x2 max-pool) are loops on Tensor4.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <memory>
#include <optional>
#include <thread>

#include "helmbench/bench.hpp"
#include "helmbench/checkpoint.hpp"
#include "helmbench/datagen.hpp"
#include "helmbench/grid.hpp"
#include "helmbench/krylov.hpp"
#include "helmbench/multigrid.hpp"
#include "helmbench/precond.hpp"
#include "helmbench/rng.hpp"
#include "helmbench/stencil.hpp"
#include "helmbench/tensor.hpp"
#include "helmbench/training.hpp"
#include "helmbench/unet.hpp"

extern "C" void openblas_set_num_threads(int);

using namespace helm;

#define HR_EXPORT extern "C" __attribute__((visibility("default")))

namespace {

ComplexField to_field(const double* p, int nx, int ny) {
  ComplexField f(nx, ny);
  std::memcpy(f.v.data(), p, sizeof(Complex) * f.v.size());
  return f;
}
void from_field(const ComplexField& f, double* p) { std::memcpy(p, f.v.data(), sizeof(Complex) * f.v.size()); }

HelmholtzProblem make_prob(int nx, int ny, double omega, const double* k2, const double* gam, double lo, double hi) {
  ProblemGrid g = make_grid(nx, ny, 1);
  RealField K(nx, ny), G(nx, ny);
  std::memcpy(K.v.data(), k2, sizeof(double) * K.v.size());
  std::memcpy(G.v.data(), gam, sizeof(double) * G.v.size());
  return make_problem(g, omega, make_slowness_squared(std::move(K), lo, hi), Attenuation{std::move(G)});
}

// ---------------- classic U-Net (oracle ext A5/A7) on the reference Tape ----
struct ClassicNet {
  int kind = 0, L = 0, base = 16, in_ch = 3, ctx_ch = 0;
  std::vector<std::unique_ptr<Param>> k, b;  // creation order
  int enc1[8], enc2[8], up[8], dec1[8], dec2[8], head = -1;
  int add(int cout, int cin) {
    auto pk = std::make_unique<Param>();
    pk->value = Tensor4(cout, cin, 3, 3);
    pk->trainable = false;
    auto pb = std::make_unique<Param>();
    pb->value = Tensor4(1, cout, 1, 1);
    pb->trainable = false;
    k.push_back(std::move(pk));
    b.push_back(std::move(pb));
    return int(k.size()) - 1;
  }
};

Tensor4 relu(Tensor4 t) {
  for (auto& x : t.v) x = x < 0.0f ? 0.0f : x;
  return t;
}
Tensor4 maxpool2(const Tensor4& a) {
  Tensor4 o(a.n, a.c, a.h / 2, a.w / 2);
  for (int n = 0; n < a.n; ++n)
    for (int c = 0; c < a.c; ++c)
      for (int y = 0; y < o.h; ++y)
        for (int x = 0; x < o.w; ++x)
          o.at(n, c, y, x) = std::max(std::max(a.at(n, c, 2 * y, 2 * x), a.at(n, c, 2 * y, 2 * x + 1)),
                                      std::max(a.at(n, c, 2 * y + 1, 2 * x), a.at(n, c, 2 * y + 1, 2 * x + 1)));
  return o;
}
// x2 bilinear with half-pixel centres / clamped edges = bilinear_resize per plane
Tensor4 upsample2(const Tensor4& a) {
  Tensor4 o(a.n, a.c, 2 * a.h, 2 * a.w);
  RealField src(a.w, a.h);
  for (int n = 0; n < a.n; ++n)
    for (int c = 0; c < a.c; ++c) {
      for (int y = 0; y < a.h; ++y)
        for (int x = 0; x < a.w; ++x) src.at(x, y) = a.at(n, c, y, x);
      RealField dst = bilinear_resize(src, 2 * a.w, 2 * a.h);
      for (int y = 0; y < o.h; ++y)
        for (int x = 0; x < o.w; ++x) o.at(n, c, y, x) = float(dst.at(x, y));
    }
  return o;
}

Tensor4 conv(Tape& tape, ClassicNet& net, int i, const Tensor4& x) {
  const int id = tape.leaf(x);
  return tape.value(tape.conv2d(id, *net.k[std::size_t(i)], net.b[std::size_t(i)].get(), 1));
}
Tensor4 cat(Tape& tape, const Tensor4& a, const Tensor4& b) {
  const Tensor4 bb = (b.n == a.n) ? b : tile_batch(b, a.n);
  return tape.value(tape.concat(tape.leaf(a), tape.leaf(bb)));
}

Tensor4 unet_fwd(ClassicNet& n, const Tensor4& in, const std::vector<Tensor4>* ctx) {
  Tape tape(false);
  std::vector<Tensor4> skip(std::size_t(n.L));
  Tensor4 x = in;
  for (int l = 0; l < n.L; ++l) {
    if (l > 0) x = maxpool2(x);
    if (ctx) x = cat(tape, x, (*ctx)[std::size_t(l)]);
    x = relu(conv(tape, n, n.enc1[l], x));
    x = relu(conv(tape, n, n.enc2[l], x));
    skip[std::size_t(l)] = x;
  }
  for (int l = n.L - 2; l >= 0; --l) {
    if (ctx) x = cat(tape, x, (*ctx)[std::size_t(l + 1)]);
    x = conv(tape, n, n.up[l], upsample2(x));
    x = cat(tape, x, skip[std::size_t(l)]);
    x = relu(conv(tape, n, n.dec1[l], x));
    x = relu(conv(tape, n, n.dec2[l], x));
  }
  return conv(tape, n, n.head, x);
}

std::vector<Tensor4> encoder_fwd(ClassicNet& e, const Tensor4& kappa) {
  Tape tape(false);
  std::vector<Tensor4> ctx;
  Tensor4 x = kappa;
  for (int l = 0; l < e.L; ++l) {
    if (l > 0) x = maxpool2(x);
    x = relu(conv(tape, e, e.enc1[l], x));
    x = relu(conv(tape, e, e.enc2[l], x));
    ctx.push_back(x);
  }
  return ctx;
}

// network applier: [H^2 Re f, H^2 Im f, kappa^2] -> complex (inc/precond.hpp:71-91 pattern)
ComplexField net_apply(ClassicNet& n, const ComplexField& f, const RealField& k2, double h,
                       const std::vector<Tensor4>* ctx) {
  const double h2 = h * h;
  Tensor4 in(1, 3, f.ny, f.nx);
  for (int y = 0; y < f.ny; ++y)
    for (int x = 0; x < f.nx; ++x) {
      in.at(0, 0, y, x) = float(h2 * f.at(x, y).real());
      in.at(0, 1, y, x) = float(h2 * f.at(x, y).imag());
      in.at(0, 2, y, x) = float(k2.at(x, y));
    }
  return complex_from_channels(unet_fwd(n, in, ctx), 0);
}

struct RefMG {
  HelmholtzProblem prob;
  VCycleConfig cfg;
  std::shared_ptr<MultigridHierarchy> hier;  // coarse GMRES / dense levels
  int coarse_kind = 0;                        // 0 gmres, 1 jacobi (A3), 2 net (A4)
  ClassicNet* coarse_net = nullptr;
};

// public-API restatement of MultigridHierarchy::cycle_at (inc/multigrid.hpp:108-119)
// with the coarsest solve replaced (A3 Jacobi / A4 net)
ComplexField cycle_ext(const RefMG& m, int level, ComplexField v, const ComplexField& f) {
  const MultigridHierarchy& H = *m.hier;
  const StencilOperator& op = H.op(level);
  if (level == H.levels() - 1) {
    if (m.coarse_kind == 1) return op.jacobi(ComplexField(f.nx, f.ny), f, m.cfg.damping, m.cfg.coarse_iters);
    return net_apply(*m.coarse_net, f, H.problem(level).kappa2.values, H.problem(level).grid.h, nullptr);
  }
  const int offset = level % 2;
  v = op.jacobi(std::move(v), f, m.cfg.damping, m.cfg.nu1);
  ComplexField r = op.residual(v, f);
  ComplexField fc = restrict_field(r, offset);
  ComplexField vc = cycle_ext(m, level + 1, ComplexField(fc.nx, fc.ny), fc);
  ComplexField corr = prolong_field(vc, offset);
  for (std::size_t i = 0; i < v.v.size(); ++i) v.v[i] += corr.v[i];
  return op.jacobi(std::move(v), f, m.cfg.damping, m.cfg.nu2);
}

ComplexField cycle(const RefMG& m, ComplexField v, const ComplexField& f) {
  if (m.coarse_kind == 0) return m.hier->cycle(std::move(v), f);
  return cycle_ext(m, 0, std::move(v), f);
}

struct RefPC : Preconditioner {
  RefMG* mg;
  int kind;  // 0 M_V / coarse-net cycle, 1 M_VU (A8)
  ClassicNet* net = nullptr;
  std::vector<Tensor4> ctx;
  bool has_ctx = false;
  std::vector<ComplexField> apply(const std::vector<ComplexField>& r) override {
    std::vector<ComplexField> out;
    for (const auto& col : r) {
      ComplexField v0(col.nx, col.ny);
      if (kind == 1)
        v0 = net_apply(*net, col, mg->prob.kappa2.values, mg->prob.grid.h, has_ctx ? &ctx : nullptr);
      out.push_back(cycle(*mg, std::move(v0), col));
    }
    return out;
  }
  bool requires_flexible() const override { return kind == 1 || mg->coarse_kind == 2; }
  std::string name() const override { return kind == 1 ? "vu" : "v"; }
};

thread_local std::string g_err;

}  // namespace

#define HR_TRY(...)                   \
  try {                               \
    __VA_ARGS__;                      \
    return 0;                         \
  } catch (const std::exception& e) { \
    g_err = e.what();                 \
    return -1;                        \
  }

HR_EXPORT const char* hr_last_error() { return g_err.c_str(); }

HR_EXPORT void hr_init() { openblas_set_num_threads(1); }

HR_EXPORT void hr_rng_normals(uint64_t seed, int64_t n, double* out) {
  Rng r(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = r.normal();
}
HR_EXPORT void hr_rng_u64(uint64_t seed, int64_t n, uint64_t* out) {
  Rng r(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = r.next_u64();
}

HR_EXPORT int hr_absorbing_layer(int nx, int ny, int width, double gmax, double* out) {
  HR_TRY({
    auto att = make_absorbing_layer(make_grid(nx, ny, 1), width, gmax);
    std::memcpy(out, att.values.v.data(), sizeof(double) * att.values.v.size());
  })
}

// synthetic_slowness (inc/datagen.hpp:94-119): the media of the reference's
// acceptance gates (tests/acceptance.cpp:62-67,184-186)
HR_EXPORT int hr_synthetic_slowness(uint64_t seed, int nx, int ny, double lo, double hi, double* out) {
  HR_TRY({
    auto s = synthetic_slowness(seed, make_grid(nx, ny, 1), SlownessRange{lo, hi});
    std::memcpy(out, s.values.v.data(), sizeof(double) * s.values.v.size());
  })
}
// random_rhs_block (inc/bench.hpp:83-90): count c128 fields [count][ny][nx]
HR_EXPORT int hr_random_rhs_block(int nx, int ny, int count, uint64_t seed, double* out) {
  HR_TRY({
    auto B = random_rhs_block(make_grid(nx, ny, 1), count, seed);
    for (int c = 0; c < count; ++c) from_field(B[size_t(c)], out + size_t(c) * 2 * nx * ny);
  })
}

HR_EXPORT int hr_restrict(int nx, int ny, int offset, int ncomp, const double* fine, double* coarse) {
  HR_TRY({
    if (ncomp == 1) {
      RealField f(nx, ny);
      std::memcpy(f.v.data(), fine, sizeof(double) * f.v.size());
      auto c = restrict_field(f, offset);
      std::memcpy(coarse, c.v.data(), sizeof(double) * c.v.size());
    } else {
      auto c = restrict_field(to_field(fine, nx, ny), offset);
      from_field(c, coarse);
    }
  })
}
HR_EXPORT int hr_prolong(int cnx, int cny, int offset, int ncomp, const double* coarse, double* fine) {
  HR_TRY({
    if (ncomp == 1) {
      RealField c(cnx, cny);
      std::memcpy(c.v.data(), coarse, sizeof(double) * c.v.size());
      auto f = prolong_field(c, offset);
      std::memcpy(fine, f.v.data(), sizeof(double) * f.v.size());
    } else {
      from_field(prolong_field(to_field(coarse, cnx, cny), offset), fine);
    }
  })
}

// ---- hierarchy
HR_EXPORT void* hr_mg_create(int nx, int ny, double omega, const double* k2, const double* gam, double lo, double hi,
                             int levels, int nu1, int nu2, double damping, double alpha, double beta, int coarse_kind,
                             int coarse_iters) {
  try {
    auto* m = new RefMG();
    m->prob = make_prob(nx, ny, omega, k2, gam, lo, hi);
    m->cfg.levels = levels;
    m->cfg.nu1 = nu1;
    m->cfg.nu2 = nu2;
    m->cfg.damping = damping;
    m->cfg.shift = Shift{alpha, beta};
    m->cfg.coarse_iters = coarse_iters;
    m->cfg.coarse_solver = coarse_kind == 3 ? CoarseSolver::dense : CoarseSolver::gmres;
    m->coarse_kind = coarse_kind == 3 ? 0 : coarse_kind;
    m->hier = std::make_shared<MultigridHierarchy>(m->prob, m->cfg);
    return m;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
HR_EXPORT void hr_mg_destroy(void* p) { delete static_cast<RefMG*>(p); }

HR_EXPORT void hr_mg_level_coef(void* p, int l, double* k2, double* gam, double* diagA, double* diagM) {
  auto* m = static_cast<RefMG*>(p);
  const auto& pr = m->hier->problem(l);
  const std::size_t n = pr.kappa2.values.v.size();
  if (k2) std::memcpy(k2, pr.kappa2.values.v.data(), n * sizeof(double));
  if (gam) std::memcpy(gam, pr.gamma.values.v.data(), n * sizeof(double));
  if (diagA) {
    StencilOperator A(pr, kHelmholtzShift);
    std::memcpy(diagA, A.diagonal().data(), n * sizeof(Complex));
  }
  if (diagM) std::memcpy(diagM, m->hier->op(l).diagonal().data(), n * sizeof(Complex));
}

HR_EXPORT int hr_apply(void* p, int l, int which, const double* u, double* y) {
  HR_TRY({
    auto* m = static_cast<RefMG*>(p);
    const auto& pr = m->hier->problem(l);
    StencilOperator A(pr, which ? m->cfg.shift : kHelmholtzShift);
    from_field(A.apply(to_field(u, pr.grid.nx, pr.grid.ny)), y);
  })
}
HR_EXPORT int hr_jacobi(void* p, int l, int which, double* v, const double* f, double damping, int iters) {
  HR_TRY({
    auto* m = static_cast<RefMG*>(p);
    const auto& pr = m->hier->problem(l);
    StencilOperator A(pr, which ? m->cfg.shift : kHelmholtzShift);
    const int nx = pr.grid.nx, ny = pr.grid.ny;
    from_field(A.jacobi(to_field(v, nx, ny), to_field(f, nx, ny), damping, iters), v);
  })
}
HR_EXPORT int hr_coarse_gmres(void* p, int l, const double* f, double* x) {
  HR_TRY({
    auto* m = static_cast<RefMG*>(p);
    const auto& pr = m->hier->problem(l);
    from_field(coarse_solve_with_op(m->hier->op(l), to_field(f, pr.grid.nx, pr.grid.ny), m->cfg), x);
  })
}

// ---- classic nets
HR_EXPORT void* hr_net_create(int kind, int L, int base, int in_ch, int ctx_ch) {
  auto* n = new ClassicNet();
  n->kind = kind;
  n->L = L;
  n->base = base;
  n->in_ch = in_ch;
  n->ctx_ch = ctx_ch;
  if (kind == 1) {
    for (int l = 0; l < L; ++l) {
      n->enc1[l] = n->add(base, l == 0 ? in_ch : base);
      n->enc2[l] = n->add(base, base);
    }
    return n;
  }
  for (int l = 0; l < L; ++l) {
    n->enc1[l] = n->add(base << l, (l == 0 ? in_ch : base << (l - 1)) + ctx_ch);
    n->enc2[l] = n->add(base << l, base << l);
  }
  for (int l = L - 2; l >= 0; --l) {
    n->up[l] = n->add(base << l, (base << (l + 1)) + ctx_ch);
    n->dec1[l] = n->add(base << l, 2 * (base << l));
    n->dec2[l] = n->add(base << l, base << l);
  }
  n->head = n->add(2, base);
  return n;
}
HR_EXPORT void hr_net_destroy(void* p) { delete static_cast<ClassicNet*>(p); }
HR_EXPORT int hr_net_nconv(void* p) { return int(static_cast<ClassicNet*>(p)->k.size()); }
HR_EXPORT float* hr_net_weight(void* p, int i) { return static_cast<ClassicNet*>(p)->k[std::size_t(i)]->value.v.data(); }
HR_EXPORT float* hr_net_bias(void* p, int i) { return static_cast<ClassicNet*>(p)->b[std::size_t(i)]->value.v.data(); }
// He-normal (A6) via fill_normal semantics (inc/tensor.hpp:51-53)
HR_EXPORT void hr_net_init_he(void* p, uint64_t seed) {
  auto* n = static_cast<ClassicNet*>(p);
  Rng rng(seed);
  for (std::size_t i = 0; i < n->k.size(); ++i) {
    auto& t = n->k[i]->value;
    fill_normal(t, rng, float(std::sqrt(2.0 / double(t.c * 9))));
    std::fill(n->b[i]->value.v.begin(), n->b[i]->value.v.end(), 0.0f);
  }
}
HR_EXPORT int hr_net_forward(void* p, int B, int H, int W, const float* in, const float* const* ctx, float* out) {
  HR_TRY({
    auto* n = static_cast<ClassicNet*>(p);
    Tensor4 x(B, n->in_ch, H, W);
    std::memcpy(x.v.data(), in, sizeof(float) * x.v.size());
    std::vector<Tensor4> cx;
    if (ctx)
      for (int l = 0; l < n->L; ++l) {
        Tensor4 t(1, n->ctx_ch, H >> l, W >> l);
        std::memcpy(t.v.data(), ctx[l], sizeof(float) * t.v.size());
        cx.push_back(std::move(t));
      }
    Tensor4 y = unet_fwd(*n, x, ctx ? &cx : nullptr);
    std::memcpy(out, y.v.data(), sizeof(float) * y.v.size());
  })
}
HR_EXPORT int hr_encoder_forward(void* p, int H, int W, const float* kappa, float** ctx) {
  HR_TRY({
    auto* e = static_cast<ClassicNet*>(p);
    Tensor4 k(1, 1, H, W);
    std::memcpy(k.v.data(), kappa, sizeof(float) * k.v.size());
    auto c = encoder_fwd(*e, k);
    for (int l = 0; l < e->L; ++l) std::memcpy(ctx[l], c[std::size_t(l)].v.data(), sizeof(float) * c[std::size_t(l)].v.size());
  })
}
// raw Tape::conv2d (3x3 or 5x5, stride 1 or 2) for the conv KATs
HR_EXPORT int hr_conv2d(int N, int cin, int cout, int H, int W, int k, int stride, const float* x, const float* w,
                        const float* b, float* y) {
  HR_TRY({
    Param K, Bp;
    K.value = Tensor4(cout, cin, k, k);
    std::memcpy(K.value.v.data(), w, sizeof(float) * K.value.v.size());
    Bp.value = Tensor4(1, cout, 1, 1);
    std::memcpy(Bp.value.v.data(), b, sizeof(float) * cout);
    K.trainable = Bp.trainable = false;
    Tape tape(false);
    Tensor4 xt(N, cin, H, W);
    std::memcpy(xt.v.data(), x, sizeof(float) * xt.v.size());
    const Tensor4& o = tape.value(tape.conv2d(tape.leaf(xt), K, &Bp, stride));
    std::memcpy(y, o.v.data(), sizeof(float) * o.v.size());
  })
}

// ---- preconditioners + solve
HR_EXPORT void hr_mg_set_coarse_net(void* mg, void* net) {
  auto* m = static_cast<RefMG*>(mg);
  m->coarse_net = static_cast<ClassicNet*>(net);
}

HR_EXPORT void* hr_pc_create(int kind, void* mg, void* net, void* enc) {
  auto* pc = new RefPC();
  pc->mg = static_cast<RefMG*>(mg);
  pc->kind = kind;
  pc->net = static_cast<ClassicNet*>(net);
  if (enc) {  // encoder runs once per medium (inc/precond.hpp:66-67)
    auto* e = static_cast<ClassicNet*>(enc);
    const auto& K = pc->mg->prob.kappa2.values;
    Tensor4 k(1, 1, K.ny, K.nx);
    for (int y = 0; y < K.ny; ++y)
      for (int x = 0; x < K.nx; ++x) k.at(0, 0, y, x) = float(K.at(x, y));
    pc->ctx = encoder_fwd(*e, k);
    pc->has_ctx = true;
  }
  return pc;
}
HR_EXPORT void hr_pc_destroy(void* p) { delete static_cast<RefPC*>(p); }
HR_EXPORT int hr_pc_apply(void* p, int B, const double* r, double* z) {
  HR_TRY({
    auto* pc = static_cast<RefPC*>(p);
    const int nx = pc->mg->prob.grid.nx, ny = pc->mg->prob.grid.ny;
    std::vector<ComplexField> R;
    for (int b = 0; b < B; ++b) R.push_back(to_field(r + std::size_t(b) * nx * ny * 2, nx, ny));
    auto Z = pc->apply(R);
    for (int b = 0; b < B; ++b) from_field(Z[std::size_t(b)], z + std::size_t(b) * nx * ny * 2);
  })
}

// block FGMRES through the reference's own entry point, exactly as
// run_preconditioner_test (inc/bench.hpp:93-110).  nthreads > 1 splits the
// columns into contiguous independent blocks (columns are independent,
// tests/test_classic.cpp:469-508), each with its own preconditioner object.
HR_EXPORT int hr_fgmres(void* p, int restart, int max_iters, double rel_tol, int flexible, int B, const double* b,
                        double* x, double* hist, int hist_cap, int* iters, int* conv, int* brk, int* hlen,
                        int nthreads, double* seconds) {
  HR_TRY({
    auto* pc0 = static_cast<RefPC*>(p);
    const int nx = pc0->mg->prob.grid.nx, ny = pc0->mg->prob.grid.ny;
    const std::size_t n2 = std::size_t(nx) * ny * 2;
    KrylovConfig cfg;
    cfg.restart = restart;
    cfg.max_iters = max_iters;
    cfg.rel_tol = rel_tol;
    cfg.flexible = flexible != 0;
    check_flexible_contract(cfg, *pc0);
    StencilOperator A(pc0->mg->prob, kHelmholtzShift);
    BatchedOp apply_A = [&A](const std::vector<ComplexField>& in) {
      std::vector<ComplexField> out;
      out.reserve(in.size());
      for (const auto& f : in) out.push_back(A.apply(f));
      return out;
    };
    const int T = std::max(1, std::min(nthreads, B));
    std::vector<std::string> errs;
    errs.resize(std::size_t(T));
    auto work = [&](int t) {
      try {
        const int c0 = B * t / T, c1 = B * (t + 1) / T;
        RefPC pc = *pc0;  // per-thread preconditioner object (same weights, shared ctx)
        std::vector<ComplexField> Bc;
        for (int c = c0; c < c1; ++c) Bc.push_back(to_field(b + std::size_t(c) * n2, nx, ny));
        auto [X, rep] = block_fgmres(apply_A, pc.as_batched_op(), Bc, cfg);
        for (int c = c0; c < c1; ++c) {
          const std::size_t q = std::size_t(c - c0);
          from_field(X[q], x + std::size_t(c) * n2);
          const auto& h = rep.residual_history[q];
          hlen[c] = int(h.size());
          for (int i = 0; i < std::min<int>(hist_cap, int(h.size())); ++i) hist[std::size_t(c) * hist_cap + i] = h[std::size_t(i)];
          iters[c] = rep.iterations[q];
          conv[c] = rep.converged[q] ? 1 : 0;
          brk[c] = rep.breakdown[q] ? 1 : 0;
        }
      } catch (const std::exception& e) {
        errs[std::size_t(t)] = e.what();
      }
    };
    const auto t0 = std::chrono::steady_clock::now();
    if (T == 1) {
      work(0);
    } else {
      std::vector<std::thread> th;
      for (int t = 0; t < T; ++t) th.emplace_back(work, t);
      for (auto& h : th) h.join();
    }
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    for (auto& e : errs)
      if (!e.empty()) throw std::runtime_error(e);
  })
}

// ---------------- paper U-Net on the reference's own builders ----
// NetworkWeights + build_unet / build_encoder (inc/unet.hpp:10-111,139-257), eval-mode
// forward through unet_forward / solver_forward (:261-295), UNW1 checkpoints
// (inc/checkpoint.hpp:51-104), JacobiUnetPreconditioner / UnetVCyclePreconditioner
// (inc/precond.hpp:104-165).  Parameters are materialised by one train-mode forward
// (creation order = the reference's), then the batch-norm buffers are set to seeded
// values (count = 1) so eval mode is meaningful on untrained weights.
namespace {
struct PaperNet {
  std::shared_ptr<NetworkWeights> w;
  UNetConfig cfg;
  NetVariant variant = NetVariant::standalone;
  std::optional<FeatureStack> feats;
  AdamState adam;                 // hr_paper_train_batch's ADAM state
  std::vector<Param*> trainable;
};
}  // namespace

HR_EXPORT void* hr_paper_create(int levels, int base, int rpl, int bot, int kud, int kres, int variant,
                                uint64_t seed) {
  try {
    auto* p = new PaperNet();
    p->w = std::make_shared<NetworkWeights>(seed);
    p->cfg.levels = levels;
    p->cfg.base_channels = base;
    p->cfg.resnet_per_level = rpl;
    p->cfg.bottleneck_resnets = bot;
    p->cfg.updown_kernel = kud;
    p->cfg.res_kernel = kres;
    p->variant = variant ? NetVariant::encoder_solver : NetVariant::standalone;
    const int n = 2 << levels;
    Tensor4 in(1, 4, n, n, 0.1f);
    if (p->variant == NetVariant::encoder_solver) {
      RealField k(n, n);
      for (auto& x : k.v) x = 0.3;
      const FeatureStack fs = encoder_forward(*p->w, p->cfg, k, true);  // NetworkApplier order: encoder first
      solver_forward(*p->w, p->cfg, in, fs, true);
    } else {
      unet_forward(*p->w, p->cfg, in, true);
    }
    Rng r(seed ^ 0x9e3779b97f4a7c15ULL);
    for (std::size_t i = 0; i < p->w->size(); ++i) {
      Param& q = p->w->at(i);
      auto ends = [&](const char* s) {
        const std::string t(s);
        return q.name.size() >= t.size() && q.name.compare(q.name.size() - t.size(), t.size(), t) == 0;
      };
      if (ends(".count")) q.value.v[0] = 1.0f;
      else if (ends(".rmean") || ends(".offset") || ends(".b") || ends(".b1") || ends(".b2"))
        for (auto& x : q.value.v) x = float(r.uniform(-0.2, 0.2));
      else if (ends(".rvar")) for (auto& x : q.value.v) x = float(r.uniform(0.5, 2.0));
      else if (ends(".scale")) for (auto& x : q.value.v) x = float(r.uniform(0.5, 1.5));
    }
    return p;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
HR_EXPORT void hr_paper_destroy(void* p) { delete static_cast<PaperNet*>(p); }
// zero every bias, batch-norm offset and running mean: the net becomes
// positively homogeneous up to ELU's curvature (well-conditioned FGMRES fixtures)
HR_EXPORT void hr_paper_zero_shifts(void* p) {
  auto* q = static_cast<PaperNet*>(p);
  for (std::size_t i = 0; i < q->w->size(); ++i) {
    Param& x = q->w->at(i);
    auto ends = [&](const char* s) {
      const std::string t(s);
      return x.name.size() >= t.size() && x.name.compare(x.name.size() - t.size(), t.size(), t) == 0;
    };
    if (ends(".b") || ends(".b1") || ends(".b2") || ends(".offset") || ends(".rmean"))
      std::fill(x.value.v.begin(), x.value.v.end(), 0.0f);
    if (ends("out.k"))  // damp the head: the untrained net becomes a small correction
      for (auto& v : x.value.v) v *= 0.01f;
    if (x.name == "unet.down0.k")  // drop the kappa^2 / gamma input channels: net(a r) = a net(r) up to ELU curvature
      for (int o = 0; o < x.value.n; ++o)
        for (int c = 2; c < 4; ++c)
          for (int t = 0; t < x.value.h * x.value.w; ++t)
            x.value.v[(std::size_t(o) * x.value.c + c) * x.value.h * x.value.w + t] = 0.0f;
  }
  q->feats.reset();
}
HR_EXPORT int hr_paper_save(void* p, const char* path, const char* digest) {
  HR_TRY(save_checkpoint(*static_cast<PaperNet*>(p)->w, path, digest))
}
HR_EXPORT int hr_paper_load(void* p, const char* path) {
  HR_TRY({
    auto* q = static_cast<PaperNet*>(p);
    q->w = std::make_shared<NetworkWeights>();
    load_checkpoint(path, *q->w);
    q->feats.reset();
  })
}
HR_EXPORT int hr_paper_encode(void* p, int nx, int ny, const double* kappa2) {
  HR_TRY({
    auto* q = static_cast<PaperNet*>(p);
    RealField k(nx, ny);
    std::memcpy(k.v.data(), kappa2, sizeof(double) * k.v.size());
    q->feats = encoder_forward(*q->w, q->cfg, k, false);
  })
}
// in: NCHW [B][4][H][W] -> out NCHW [B][2][H][W]
HR_EXPORT int hr_paper_forward(void* p, int B, int H, int W, const float* in, float* out) {
  HR_TRY({
    auto* q = static_cast<PaperNet*>(p);
    Tensor4 x(B, 4, H, W);
    std::memcpy(x.v.data(), in, sizeof(float) * x.v.size());
    Tensor4 y = q->variant == NetVariant::standalone ? unet_forward(*q->w, q->cfg, x, false)
                                                     : solver_forward(*q->w, q->cfg, x, q->feats.value(), false);
    std::memcpy(out, y.v.data(), sizeof(float) * y.v.size());
  })
}
// encoder feature level l -> NCHW [1][C][H>>l][W>>l]
HR_EXPORT int hr_paper_feature(void* p, int l, float* out) {
  HR_TRY({
    const auto& f = static_cast<PaperNet*>(p)->feats.value().f.at(std::size_t(l));
    std::memcpy(out, f.v.data(), sizeof(float) * f.v.size());
  })
}


// ---------------- training: traindet::run_batch + adam_step,
// train() and retrain() (inc/training.hpp:121-298) on the reference's own code
HR_EXPORT int64_t hr_paper_trainable_count(void* p) {
  auto* q = static_cast<PaperNet*>(p);
  int64_t n = 0;
  for (Param* x : q->w->trainable()) n += int64_t(x->value.size());
  return n;
}
// one run_batch (+ optional adam_step); grads: trainable gradients concatenated in registry order
HR_EXPORT int hr_paper_train_batch(void* p, int B, int H, int W, const float* input, const float* kappa,
                                   const float* target, int train_mode, int with_grad, int step, double lr,
                                   double* loss, float* out, float* grads) {
  HR_TRY({
    auto* q = static_cast<PaperNet*>(p);
    Tensor4 in(B, 4, H, W), tg(B, 2, H, W), kp(B, 1, H, W);
    std::memcpy(in.v.data(), input, sizeof(float) * in.v.size());
    std::memcpy(tg.v.data(), target, sizeof(float) * tg.v.size());
    if (kappa) std::memcpy(kp.v.data(), kappa, sizeof(float) * kp.v.size());
    q->w->zero_grads();
    auto res = traindet::run_batch(*q->w, q->cfg, q->variant == NetVariant::encoder_solver, in, kp, tg,
                                   train_mode != 0, with_grad != 0);
    if (loss) *loss = res.loss;
    if (out) std::memcpy(out, res.out.v.data(), sizeof(float) * res.out.v.size());
    if (grads) {
      std::size_t o = 0;
      for (Param* x : q->w->trainable()) {
        if (x->grad.size() == x->value.size())
          std::memcpy(grads + o, x->grad.v.data(), sizeof(float) * x->grad.v.size());
        else
          std::fill(grads + o, grads + o + x->value.size(), 0.0f);
        o += x->value.size();
      }
    }
    if (step) {
      if (q->trainable.empty()) q->trainable = q->w->trainable();
      adam_step(q->trainable, q->adam, lr);
    }
  })
}
static TrainConfig train_cfg(int epochs, double lr0, int batch0, int t0, double val_fraction, int es, uint64_t seed) {
  TrainConfig c;
  c.epochs = epochs;
  c.lr0 = lr0;
  c.batch0 = batch0;
  c.t0 = t0;
  c.val_fraction = val_fraction;
  c.encoder_solver = es != 0;
  c.seed = seed;
  return c;
}
static void put_hist(const TrainHistory& h, double* hist, int cap, int* n, int* aborted) {
  for (std::size_t i = 0; i < h.epochs.size() && int(i) < cap; ++i) {
    hist[i * 4 + 0] = h.epochs[i].mean_rel_error_train;
    hist[i * 4 + 1] = h.epochs[i].mean_rel_error_val;
    hist[i * 4 + 2] = h.epochs[i].lr;
    hist[i * 4 + 3] = h.epochs[i].batch;
  }
  *n = int(h.epochs.size());
  *aborted = h.aborted_non_finite ? 1 : 0;
}
// train() over an in-memory dataset: r_hat / e_true [count][2][H][W], kappa2 / gamma [models][H][W]
HR_EXPORT int hr_paper_train(void* p, int epochs, double lr0, int batch0, int t0, double val_fraction, int es,
                             uint64_t seed, int count, int H, int W, const float* r_hat, const float* e_true,
                             const int* model_id, int models, const double* kappa2, const double* gamma, double* hist,
                             int cap, int* n, int* aborted) {
  HR_TRY({
    auto* q = static_cast<PaperNet*>(p);
    Dataset ds;
    ds.spec.nx = W;
    ds.spec.ny = H;
    const std::size_t pl = std::size_t(H) * W;
    for (int m = 0; m < models; ++m) {
      HelmholtzProblem pr;
      pr.kappa2.values = RealField(W, H);
      pr.gamma.values = RealField(W, H);
      std::memcpy(pr.kappa2.values.v.data(), kappa2 + m * pl, sizeof(double) * pl);
      std::memcpy(pr.gamma.values.v.data(), gamma + m * pl, sizeof(double) * pl);
      ds.problems.push_back(pr);
      ds.model_refs.push_back("(in-memory)");
    }
    for (int s = 0; s < count; ++s) {
      TrainingSample t;
      t.model_id = model_id[s];
      t.r_hat = Tensor4(1, 2, H, W);
      t.e_true = Tensor4(1, 2, H, W);
      std::memcpy(t.r_hat.v.data(), r_hat + std::size_t(s) * 2 * pl, sizeof(float) * 2 * pl);
      std::memcpy(t.e_true.v.data(), e_true + std::size_t(s) * 2 * pl, sizeof(float) * 2 * pl);
      ds.samples.push_back(std::move(t));
    }
    const TrainHistory h = train(ds, *q->w, q->cfg, train_cfg(epochs, lr0, batch0, t0, val_fraction, es, seed));
    put_hist(h, hist, cap, n, aborted);
  })
}
// retrain() on the problem of a RefMG (its own default-VCycleConfig hierarchy, as the reference)
HR_EXPORT int hr_paper_retrain(void* p, void* mg, int n_pairs, int epochs, double lr0, int es, uint64_t seed,
                               double* hist, int cap, int* n, int* aborted) {
  HR_TRY({
    auto* q = static_cast<PaperNet*>(p);
    const auto* m = static_cast<RefMG*>(mg);
    const TrainHistory h = retrain(*q->w, q->cfg, m->prob, n_pairs, epochs, train_cfg(1, lr0, 20, 48, 0.1, es, 1), seed);
    put_hist(h, hist, cap, n, aborted);
  })
}

namespace {
struct PaperPC {
  std::unique_ptr<Preconditioner> pc;
  HelmholtzProblem prob;
};
}  // namespace

// kind 0: M_JU (JacobiUnetPreconditioner), 1: M_VU (UnetVCyclePreconditioner over mg's hierarchy)
HR_EXPORT void* hr_paper_pc_create(int kind, void* mg, void* net) {
  try {
    auto* m = static_cast<RefMG*>(mg);
    auto* q = static_cast<PaperNet*>(net);
    auto* p = new PaperPC();
    p->prob = m->prob;
    if (kind == 0)
      p->pc = std::make_unique<JacobiUnetPreconditioner>(p->prob, q->w, q->cfg, q->variant);
    else
      p->pc = std::make_unique<UnetVCyclePreconditioner>(m->hier, q->w, q->cfg, q->variant);
    return p;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
HR_EXPORT void hr_paper_pc_destroy(void* p) { delete static_cast<PaperPC*>(p); }
HR_EXPORT int hr_paper_pc_apply(void* p, int B, const double* r, double* z) {
  HR_TRY({
    auto* q = static_cast<PaperPC*>(p);
    const int nx = q->prob.grid.nx, ny = q->prob.grid.ny;
    std::vector<ComplexField> R;
    for (int b = 0; b < B; ++b) R.push_back(to_field(r + std::size_t(b) * nx * ny * 2, nx, ny));
    auto Z = q->pc->apply(R);
    for (int b = 0; b < B; ++b) from_field(Z[std::size_t(b)], z + std::size_t(b) * nx * ny * 2);
  })
}
// block_fgmres (inc/krylov.hpp:83) with the paper preconditioner, as run_preconditioner_test
HR_EXPORT int hr_paper_fgmres(void* p, int restart, int max_iters, double rel_tol, int B, const double* b, double* x,
                              double* hist, int hist_cap, int* iters, int* hlen) {
  HR_TRY({
    auto* q = static_cast<PaperPC*>(p);
    const int nx = q->prob.grid.nx, ny = q->prob.grid.ny;
    KrylovConfig cfg;
    cfg.restart = restart;
    cfg.max_iters = max_iters;
    cfg.rel_tol = rel_tol;
    cfg.flexible = true;
    StencilOperator A(q->prob, kHelmholtzShift);
    BatchedOp apply_A = [&A](const std::vector<ComplexField>& in) {
      std::vector<ComplexField> out;
      for (const auto& f : in) out.push_back(A.apply(f));
      return out;
    };
    std::vector<ComplexField> Bc;
    for (int c = 0; c < B; ++c) Bc.push_back(to_field(b + std::size_t(c) * nx * ny * 2, nx, ny));
    auto [X, rep] = block_fgmres(apply_A, q->pc->as_batched_op(), Bc, cfg);
    for (int c = 0; c < B; ++c) {
      from_field(X[std::size_t(c)], x + std::size_t(c) * nx * ny * 2);
      const auto& h = rep.residual_history[std::size_t(c)];
      hlen[c] = int(h.size());
      for (int i = 0; i < std::min<int>(hist_cap, int(h.size())); ++i) hist[std::size_t(c) * hist_cap + i] = h[std::size_t(i)];
      iters[c] = rep.iterations[std::size_t(c)];
    }
  })
}

// ---------------- training pairs: gen_sample_pair (inc/datagen.hpp:191-219)
HR_EXPORT int hr_gen_sample_pair(void* mg, uint64_t seed, int k_forced, int k_max, double* r, double* e) {
  HR_TRY({
    auto* m = static_cast<RefMG*>(mg);
    const SamplePair s = gen_sample_pair(m->prob, *m->hier, seed, k_forced, k_max);
    from_field(s.r, r);
    from_field(s.e, e);
  })
}

// ---------------- SLW1 fields (inc/field_io.hpp:46-76)
HR_EXPORT int hr_write_slw1(const char* path, int nx, int ny, const double* v) {
  HR_TRY({
    RealField f(nx, ny);
    std::memcpy(f.v.data(), v, sizeof(double) * f.v.size());
    write_slw1(std::string(path), f);
  })
}
HR_EXPORT int hr_read_slw1(const char* path, int* nx, int* ny, double* v) {
  HR_TRY({
    const RealField f = read_slw1(std::string(path));
    *nx = f.nx;
    *ny = f.ny;
    if (v) std::memcpy(v, f.v.data(), sizeof(double) * f.v.size());
  })
}
