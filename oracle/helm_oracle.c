/*
 * helm_oracle.c -- CPU restatement of the arXiv 2203.11025 reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in paper_2203_11025_b200/ links, loads or
 * calls this file.  It is imported by tests/, by __graft_entry__.smoke() as the
 * checker, and by bench.py's cpu_baseline leg.  It is never the thing measured
 * as the GPU product and never a fallback.
 *
 * Parity status: pinned.  Every primitive below is checked against the
 * reference headers compiled in place (oracle/build_ref.sh -> oracle/_ref/)
 * and against committed golden vectors generated from that build
 * (tests/golden/make_golden.py).  The BASELINE-config extensions (medium
 * generator, point sources, classic U-Net ops, He init, coarse-net cycle) are
 * "survey-added" rows A1..A8; they are pinned by the same
 * build (built there from reference primitives) plus hand KATs.
 *
 * Arithmetic mirrors the reference: complex128 fields, fp64 stencil, fp32 NCHW
 * network tensors.  Reference = /root/reference/proj/include/helmbench/ (inc/).
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

typedef double complex cplx;

#define HO_EXPORT __attribute__((visibility("default")))

/* ------------------------------------------------------------------ rng --
 * inc/rng.hpp:9-67: splitmix64 seed expansion, xoshiro256++, 53-bit uniform,
 * modulo uniform_int, Box-Muller normal with a cached spare. */
typedef struct {
  uint64_t s[4];
  double spare;
  int have_spare;
} ho_rng;

static inline uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

HO_EXPORT void ho_rng_init(ho_rng* r, uint64_t seed) {
  uint64_t z = seed;
  for (int i = 0; i < 4; ++i) {
    z += 0x9e3779b97f4a7c15ull;
    uint64_t x = z;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    r->s[i] = x ^ (x >> 31);
  }
  r->spare = 0.0;
  r->have_spare = 0;
}

HO_EXPORT uint64_t ho_rng_next(ho_rng* r) {
  uint64_t* s = r->s;
  const uint64_t result = rotl64(s[0] + s[3], 23) + s[0];
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl64(s[3], 45);
  return result;
}

HO_EXPORT double ho_rng_uniform(ho_rng* r) { return (double)(ho_rng_next(r) >> 11) * 0x1.0p-53; }

HO_EXPORT int64_t ho_rng_uniform_int(ho_rng* r, int64_t lo, int64_t hi) {
  return lo + (int64_t)(ho_rng_next(r) % (uint64_t)(hi - lo + 1));
}

HO_EXPORT double ho_rng_normal(ho_rng* r) {
  if (r->have_spare) {
    r->have_spare = 0;
    return r->spare;
  }
  double u1 = 0.0;
  while (u1 <= 0.0) u1 = ho_rng_uniform(r);
  const double u2 = ho_rng_uniform(r);
  const double rr = sqrt(-2.0 * log(u1));
  const double theta = 6.283185307179586476925286766559 * u2;
  r->spare = rr * sin(theta);
  r->have_spare = 1;
  return rr * cos(theta);
}

HO_EXPORT int ho_rng_sizeof(void) { return (int)sizeof(ho_rng); }

/* n normals from Rng(seed) (test helper; inc/rng.hpp:45) */
HO_EXPORT void ho_rng_normals(uint64_t seed, int64_t n, double* out) {
  ho_rng r;
  ho_rng_init(&r, seed);
  for (int64_t i = 0; i < n; ++i) out[i] = ho_rng_normal(&r);
}

/* seeded complex-normal field, (re, im) draw order: datagen.hpp:185-189 */
HO_EXPORT void ho_random_complex_normal(uint64_t seed, int64_t n, double* out) {
  ho_rng r;
  ho_rng_init(&r, seed);
  for (int64_t i = 0; i < n; ++i) {
    out[2 * i] = ho_rng_normal(&r);
    out[2 * i + 1] = ho_rng_normal(&r);
  }
}

/* ----------------------------------------------------------- grid / ABL --
 * inc/grid.hpp:101-119 quadratic ramp at min(dx, dy). */
HO_EXPORT int ho_absorbing_layer(int nx, int ny, int width, double gamma_max, double* out) {
  if (gamma_max < 0.0) return -1;
  const int mn = nx < ny ? nx : ny;
  if (width < 0 || width > mn / 2) return -1;
  for (int iy = 0; iy < ny; ++iy)
    for (int ix = 0; ix < nx; ++ix) {
      int dx = ix < nx - 1 - ix ? ix : nx - 1 - ix;
      int dy = iy < ny - 1 - iy ? iy : ny - 1 - iy;
      int d = dx < dy ? dx : dy;
      double g = 0.0;
      if (width > 0 && d < width) {
        const double t = (double)(width - d) / (double)width;
        g = gamma_max * t * t;
      }
      out[(size_t)iy * nx + ix] = g;
    }
  return 0;
}

/* inc/datagen.hpp:66-79 */
static void normalize_range(double* f, size_t n, double lo, double hi) {
  double mn = f[0], mx = f[0];
  for (size_t i = 0; i < n; ++i) {
    if (f[i] < mn) mn = f[i];
    if (f[i] > mx) mx = f[i];
  }
  if (mx - mn < 1e-300) {
    for (size_t i = 0; i < n; ++i) f[i] = hi;
    return;
  }
  const double scale = (hi - lo) / (mx - mn);
  for (size_t i = 0; i < n; ++i) f[i] = lo + (f[i] - mn) * scale;
}

static inline int clampi(int x, int lo, int hi) { return x < lo ? lo : (x > hi ? hi : x); }

/* Separable Gaussian with replicate padding: the inc/datagen.hpp:40-62
 * gaussian_blur5 pattern generalised to radius ceil(3 sigma). */
HO_EXPORT void ho_gaussian_blur(int nx, int ny, double sigma, const double* src, double* out) {
  const int R = (int)ceil(3.0 * sigma);
  double* w = (double*)malloc(sizeof(double) * (2 * R + 1));
  double sum = 0.0;
  for (int i = -R; i <= R; ++i) {
    w[i + R] = exp(-0.5 * i * i / (sigma * sigma));
    sum += w[i + R];
  }
  for (int i = 0; i <= 2 * R; ++i) w[i] /= sum;
  double* tmp = (double*)malloc(sizeof(double) * (size_t)nx * ny);
  for (int y = 0; y < ny; ++y)
    for (int x = 0; x < nx; ++x) {
      double acc = 0.0;
      for (int i = -R; i <= R; ++i) acc += w[i + R] * src[(size_t)y * nx + clampi(x + i, 0, nx - 1)];
      tmp[(size_t)y * nx + x] = acc;
    }
  for (int y = 0; y < ny; ++y)
    for (int x = 0; x < nx; ++x) {
      double acc = 0.0;
      for (int i = -R; i <= R; ++i) acc += w[i + R] * tmp[(size_t)clampi(y + i, 0, ny - 1) * nx + x];
      out[(size_t)y * nx + x] = acc;
    }
  free(tmp);
  free(w);
}

/* Oracle extension A1 (+D7): N(0,1) field from Rng(seed) in row-major draw
 * order -> Gaussian(sigma) -> min-max to velocity [vmin, vmax]; optionally
 * n_interfaces horizontal jumps (row = uniform_int(w, ny-w-1), jump =
 * uniform(jmin, jmax), added to all rows iy >= row) followed by a second
 * min-max; kappa^2 = 1/c^2 (inc/grid.hpp:72 declared range [1/vmax^2, 1/vmin^2]). */
HO_EXPORT void ho_make_medium(int nx, int ny, uint64_t seed, double sigma, double vmin, double vmax,
                              int n_interfaces, uint64_t iface_seed, int iface_margin, double jmin,
                              double jmax, double* kappa2) {
  const size_t n = (size_t)nx * ny;
  double* f = (double*)malloc(sizeof(double) * n);
  ho_rng r;
  ho_rng_init(&r, seed);
  for (size_t i = 0; i < n; ++i) f[i] = ho_rng_normal(&r);
  ho_gaussian_blur(nx, ny, sigma, f, kappa2);
  normalize_range(kappa2, n, vmin, vmax);
  if (n_interfaces > 0) {
    ho_rng ir;
    ho_rng_init(&ir, iface_seed);
    for (int t = 0; t < n_interfaces; ++t) {
      const int row = (int)ho_rng_uniform_int(&ir, iface_margin, ny - iface_margin - 1);
      const double jump = jmin + (jmax - jmin) * ho_rng_uniform(&ir);
      for (int iy = row; iy < ny; ++iy)
        for (int ix = 0; ix < nx; ++ix) kappa2[(size_t)iy * nx + ix] += jump;
    }
    normalize_range(kappa2, n, vmin, vmax);
  }
  for (size_t i = 0; i < n; ++i) kappa2[i] = 1.0 / (kappa2[i] * kappa2[i]);
  free(f);
}

/* Oracle extension A2: point-source positions.  mode 0: B sources at
 * (uniform_int(lo,hi), uniform_int(lo,hi)) in x,y draw order; mode 1: B
 * sources on row `row` at x = uniform_int(lo, hi). */
HO_EXPORT void ho_point_sources(uint64_t seed, int B, int mode, int lo, int hi, int row, int* xs, int* ys) {
  ho_rng r;
  ho_rng_init(&r, seed);
  for (int b = 0; b < B; ++b) {
    if (mode == 0) {
      xs[b] = (int)ho_rng_uniform_int(&r, lo, hi);
      ys[b] = (int)ho_rng_uniform_int(&r, lo, hi);
    } else {
      xs[b] = (int)ho_rng_uniform_int(&r, lo, hi);
      ys[b] = row;
    }
  }
}

/* ------------------------------------------------------------ operators --
 * inc/stencil.hpp:21-104 */
typedef struct {
  int nx, ny;
  double h, omega;
  double* k2;   /* kappa^2 */
  double* gam;  /* gamma */
  double lo, hi;
  cplx* diagA;  /* shift (1, 0)   -- inc/stencil.hpp:15 */
  cplx* diagM;  /* shift (alpha, beta) of the V-cycle */
} ho_level;

static void level_diag(ho_level* L, double alpha, double beta, cplx* out) {
  const double inv_h2 = 1.0 / (L->h * L->h);
  const cplx sh = alpha - beta * I; /* Complex sh(alpha, -beta)  stencil.hpp:26 */
  const size_t n = (size_t)L->nx * L->ny;
  for (size_t i = 0; i < n; ++i) {
    const cplx damp = 1.0 - L->gam[i] * I; /* stencil.hpp:29 */
    const double mr = -L->omega * L->omega * L->k2[i];
    const cplx m = (mr * sh) * damp;
    out[i] = 4.0 * inv_h2 + m;
  }
}

/* inc/stencil.hpp:44-60 */
static void stencil_apply(int nx, int ny, double h, const cplx* diag, const cplx* u, cplx* out) {
  const double inv_h2 = 1.0 / (h * h);
  for (int iy = 0; iy < ny; ++iy) {
    const size_t row = (size_t)iy * nx;
    for (int ix = 0; ix < nx; ++ix) {
      const size_t i = row + ix;
      cplx nbr = 0.0;
      if (ix > 0) nbr += u[i - 1];
      if (ix + 1 < nx) nbr += u[i + 1];
      if (iy > 0) nbr += u[i - nx];
      if (iy + 1 < ny) nbr += u[i + nx];
      out[i] = diag[i] * u[i] - inv_h2 * nbr;
    }
  }
}

/* inc/stencil.hpp:78-92: iters sweeps of v += damping (f - A v) / d */
static void jacobi(int nx, int ny, double h, const cplx* diag, cplx* v, const cplx* f, double damping,
                   int iters) {
  const size_t n = (size_t)nx * ny;
  cplx* av = (cplx*)malloc(sizeof(cplx) * n);
  for (int it = 0; it < iters; ++it) {
    stencil_apply(nx, ny, h, diag, v, av);
    for (size_t i = 0; i < n; ++i) v[i] += damping * (f[i] - av[i]) / diag[i];
  }
  free(av);
}

/* inc/stencil.hpp:119-140 (real or complex fields; ncomp = 1 or 2 doubles) */
static const double kT1D[3] = {1.0, 2.0, 1.0};

HO_EXPORT int ho_restrict(int nx, int ny, int offset, int ncomp, const double* fine, double* coarse) {
  if (nx % 2 || ny % 2 || (offset != 0 && offset != 1)) return -1;
  const int cnx = nx / 2, cny = ny / 2;
  for (int jy = 0; jy < cny; ++jy)
    for (int jx = 0; jx < cnx; ++jx) {
      double acc[2] = {0.0, 0.0};
      for (int ky = -1; ky <= 1; ++ky) {
        const int iy = 2 * jy + offset + ky;
        if (iy < 0 || iy >= ny) continue;
        for (int kx = -1; kx <= 1; ++kx) {
          const int ix = 2 * jx + offset + kx;
          if (ix < 0 || ix >= nx) continue;
          const double w = kT1D[ky + 1] * kT1D[kx + 1] / 16.0;
          for (int c = 0; c < ncomp; ++c) acc[c] += fine[((size_t)iy * nx + ix) * ncomp + c] * w;
        }
      }
      for (int c = 0; c < ncomp; ++c) coarse[((size_t)jy * cnx + jx) * ncomp + c] = acc[c];
    }
  return 0;
}

/* inc/stencil.hpp:146-165 (accumulates into a zeroed fine field) */
HO_EXPORT int ho_prolong(int cnx, int cny, int offset, int ncomp, const double* coarse, double* fine) {
  if (offset != 0 && offset != 1) return -1;
  const int fnx = 2 * cnx, fny = 2 * cny;
  memset(fine, 0, sizeof(double) * (size_t)fnx * fny * ncomp);
  for (int jy = 0; jy < cny; ++jy)
    for (int jx = 0; jx < cnx; ++jx) {
      const double* c = coarse + ((size_t)jy * cnx + jx) * ncomp;
      for (int ky = -1; ky <= 1; ++ky) {
        const int iy = 2 * jy + offset + ky;
        if (iy < 0 || iy >= fny) continue;
        for (int kx = -1; kx <= 1; ++kx) {
          const int ix = 2 * jx + offset + kx;
          if (ix < 0 || ix >= fnx) continue;
          const double w = kT1D[ky + 1] * kT1D[kx + 1] / 4.0;
          for (int q = 0; q < ncomp; ++q) fine[((size_t)iy * fnx + ix) * ncomp + q] += c[q] * w;
        }
      }
    }
  return 0;
}

/* --------------------------------------------------------------- U-Net --
 * Oracle extension A5/A6/A7 (classic U-Net).  NCHW fp32
 * tensors (inc/tensor.hpp:14-43), 3x3 cross-correlation with zero padding 1
 * (inc/autodiff.hpp:43-69,124-149), fp64 accumulation, bias added before the
 * fp32 store; ReLU; 2x2 max-pool; x2 bilinear upsample with half-pixel centres
 * and clamped edges (inc/datagen.hpp:19-37 semantics); channel concat
 * [a | b] (inc/autodiff.hpp:403-413). */
typedef struct {
  int cout, cin;
  float* w; /* (cout, cin, 3, 3) */
  float* b; /* cout */
} ho_conv;

#define HO_MAXL 8
typedef struct {
  int kind; /* 0 = solver U-Net, 1 = encoder */
  int L, base, in_ch, ctx_ch;
  int nconv;
  ho_conv conv[4 * HO_MAXL + 2];
  /* indices into conv[] */
  int enc1[HO_MAXL], enc2[HO_MAXL], up[HO_MAXL], dec1[HO_MAXL], dec2[HO_MAXL], head;
} ho_unet;

static int add_conv(ho_unet* n, int cout, int cin) {
  ho_conv* c = &n->conv[n->nconv];
  c->cout = cout;
  c->cin = cin;
  c->w = (float*)calloc((size_t)cout * cin * 9, sizeof(float));
  c->b = (float*)calloc((size_t)cout, sizeof(float));
  return n->nconv++;
}

/* Creation order (= init order = parameter order, cf. inc/unet.hpp:10-25):
 * solver: enc0.c1, enc0.c2, ..., enc{L-1}.c2, up{L-2}, dec{L-2}.c1, dec{L-2}.c2,
 *         ..., up0, dec0.c1, dec0.c2, head.   Each conv = kernel then bias.
 * encoder (kind 1): e0.c1 (1 -> base), e0.c2, e1.c1 (base -> base), ... */
HO_EXPORT ho_unet* ho_unet_create(int kind, int L, int base, int in_ch, int ctx_ch) {
  if (L < 1 || L > HO_MAXL) return NULL;
  ho_unet* n = (ho_unet*)calloc(1, sizeof(ho_unet));
  n->kind = kind;
  n->L = L;
  n->base = base;
  n->in_ch = in_ch;
  n->ctx_ch = ctx_ch;
  if (kind == 1) {
    for (int l = 0; l < L; ++l) {
      n->enc1[l] = add_conv(n, base, l == 0 ? in_ch : base);
      n->enc2[l] = add_conv(n, base, base);
    }
    n->head = -1;
    return n;
  }
  for (int l = 0; l < L; ++l) {
    const int c = base << l;
    const int cin = (l == 0 ? in_ch : (base << (l - 1))) + ctx_ch;
    n->enc1[l] = add_conv(n, c, cin);
    n->enc2[l] = add_conv(n, c, c);
  }
  for (int l = L - 2; l >= 0; --l) {
    const int c = base << l;
    n->up[l] = add_conv(n, c, (base << (l + 1)) + ctx_ch);
    n->dec1[l] = add_conv(n, c, 2 * c);
    n->dec2[l] = add_conv(n, c, c);
  }
  n->head = add_conv(n, 2, base);
  return n;
}

HO_EXPORT void ho_unet_destroy(ho_unet* n) {
  if (!n) return;
  for (int i = 0; i < n->nconv; ++i) {
    free(n->conv[i].w);
    free(n->conv[i].b);
  }
  free(n);
}

HO_EXPORT int ho_unet_nconv(const ho_unet* n) { return n->nconv; }
HO_EXPORT void ho_unet_conv_shape(const ho_unet* n, int i, int* cout, int* cin) {
  *cout = n->conv[i].cout;
  *cin = n->conv[i].cin;
}
HO_EXPORT float* ho_unet_conv_weight(ho_unet* n, int i) { return n->conv[i].w; }
HO_EXPORT float* ho_unet_conv_bias(ho_unet* n, int i) { return n->conv[i].b; }

/* A6: He-normal kernels, x = float(normal) * float(sqrt(2 / (cin*9)))
 * (inc/tensor.hpp:51-53 fill_normal), biases zero, creation order. */
HO_EXPORT void ho_unet_init_he(ho_unet* n, uint64_t seed) {
  ho_rng r;
  ho_rng_init(&r, seed);
  for (int i = 0; i < n->nconv; ++i) {
    ho_conv* c = &n->conv[i];
    const float sd = (float)sqrt(2.0 / (double)(c->cin * 9));
    const size_t cnt = (size_t)c->cout * c->cin * 9;
    for (size_t k = 0; k < cnt; ++k) c->w[k] = (float)ho_rng_normal(&r) * sd;
    memset(c->b, 0, sizeof(float) * c->cout);
  }
}

typedef struct {
  int n, c, h, w;
  float* v;
} ho_t4;

static ho_t4 t4_new(int n, int c, int h, int w) {
  ho_t4 t = {n, c, h, w, (float*)calloc((size_t)n * c * h * w, sizeof(float))};
  return t;
}
static void t4_free(ho_t4* t) {
  free(t->v);
  t->v = NULL;
}

/* 3x3, stride 1, pad 1; input = channel concat of (a | b) (b may be NULL) */
static ho_t4 conv3x3(const ho_t4* a, const ho_t4* b, const ho_conv* cv, int relu) {
  const int H = a->h, W = a->w, N = a->n;
  const int ca = a->c, cb = b ? b->c : 0;
  ho_t4 out = t4_new(N, cv->cout, H, W);
#pragma omp parallel for collapse(2) schedule(static) if (N * cv->cout > 1)
  for (int nb = 0; nb < N; ++nb)
    for (int co = 0; co < cv->cout; ++co) {
      double* ac = (double*)malloc(sizeof(double) * (size_t)H * W);
      for (size_t p = 0; p < (size_t)H * W; ++p) ac[p] = 0.0;
      for (int ci = 0; ci < ca + cb; ++ci) {
        const float* src = ci < ca ? a->v + ((size_t)nb * ca + ci) * H * W
                                   : b->v + ((size_t)(b->n == 1 ? 0 : nb) * cb + (ci - ca)) * H * W;
        const float* k = cv->w + ((size_t)co * cv->cin + ci) * 9;
        for (int ky = 0; ky < 3; ++ky)
          for (int kx = 0; kx < 3; ++kx) {
            const double wk = k[ky * 3 + kx];
            if (wk == 0.0) continue;
            for (int y = 0; y < H; ++y) {
              const int iy = y + ky - 1;
              if (iy < 0 || iy >= H) continue;
              const float* srow = src + (size_t)iy * W;
              double* arow = ac + (size_t)y * W;
              const int x0 = kx == 0 ? 1 : 0, x1 = kx == 2 ? W - 1 : W;
              for (int x = x0; x < x1; ++x) arow[x] += wk * srow[x + kx - 1];
            }
          }
      }
      float* dst = out.v + ((size_t)nb * cv->cout + co) * H * W;
      const double bias = cv->b[co];
      for (size_t p = 0; p < (size_t)H * W; ++p) {
        float v = (float)(ac[p] + bias);
        dst[p] = (relu && v < 0.0f) ? 0.0f : v;
      }
      free(ac);
    }
  return out;
}

static ho_t4 maxpool2(const ho_t4* a) {
  ho_t4 o = t4_new(a->n, a->c, a->h / 2, a->w / 2);
  for (int nc = 0; nc < a->n * a->c; ++nc)
    for (int y = 0; y < o.h; ++y)
      for (int x = 0; x < o.w; ++x) {
        const float* s = a->v + (size_t)nc * a->h * a->w;
        float m = s[(size_t)(2 * y) * a->w + 2 * x];
        float t;
        t = s[(size_t)(2 * y) * a->w + 2 * x + 1];
        if (t > m) m = t;
        t = s[(size_t)(2 * y + 1) * a->w + 2 * x];
        if (t > m) m = t;
        t = s[(size_t)(2 * y + 1) * a->w + 2 * x + 1];
        if (t > m) m = t;
        o.v[(size_t)nc * o.h * o.w + (size_t)y * o.w + x] = m;
      }
  return o;
}

/* bilinear x2: weights computed exactly as inc/datagen.hpp:19-37 with
 * src dims n, out dims 2n (double), value rounded to float */
static ho_t4 upsample2(const ho_t4* a) {
  ho_t4 o = t4_new(a->n, a->c, 2 * a->h, 2 * a->w);
  for (int nc = 0; nc < a->n * a->c; ++nc) {
    const float* s = a->v + (size_t)nc * a->h * a->w;
    float* d = o.v + (size_t)nc * o.h * o.w;
    for (int oy = 0; oy < o.h; ++oy) {
      const double sy = (oy + 0.5) * a->h / o.h - 0.5;
      const int y0 = clampi((int)floor(sy), 0, a->h - 1);
      const int y1 = y0 + 1 < a->h - 1 ? y0 + 1 : a->h - 1;
      double fy = sy - y0;
      fy = fy < 0.0 ? 0.0 : (fy > 1.0 ? 1.0 : fy);
      for (int ox = 0; ox < o.w; ++ox) {
        const double sx = (ox + 0.5) * a->w / o.w - 0.5;
        const int x0 = clampi((int)floor(sx), 0, a->w - 1);
        const int x1 = x0 + 1 < a->w - 1 ? x0 + 1 : a->w - 1;
        double fx = sx - x0;
        fx = fx < 0.0 ? 0.0 : (fx > 1.0 ? 1.0 : fx);
        const double v = (1 - fy) * ((1 - fx) * s[(size_t)y0 * a->w + x0] + fx * s[(size_t)y0 * a->w + x1]) +
                         fy * ((1 - fx) * s[(size_t)y1 * a->w + x0] + fx * s[(size_t)y1 * a->w + x1]);
        d[(size_t)oy * o.w + ox] = (float)v;
      }
    }
  }
  return o;
}

static ho_t4 concat(const ho_t4* a, const ho_t4* b) {
  ho_t4 o = t4_new(a->n, a->c + b->c, a->h, a->w);
  const size_t pa = (size_t)a->c * a->h * a->w, pb = (size_t)b->c * b->h * b->w;
  for (int i = 0; i < a->n; ++i) {
    memcpy(o.v + i * (pa + pb), a->v + i * pa, pa * sizeof(float));
    memcpy(o.v + i * (pa + pb) + pa, b->v + (b->n == 1 ? 0 : i * pb), pb * sizeof(float));
  }
  return o;
}

/* Test helpers for the single ops. */
HO_EXPORT void ho_op_conv3x3(int N, int cin, int cout, int H, int W, const float* x, const float* w,
                             const float* b, int relu, float* y) {
  ho_t4 a = {N, cin, H, W, (float*)x};
  ho_conv cv = {cout, cin, (float*)w, (float*)b};
  ho_t4 o = conv3x3(&a, NULL, &cv, relu);
  memcpy(y, o.v, sizeof(float) * (size_t)N * cout * H * W);
  t4_free(&o);
}
HO_EXPORT void ho_op_maxpool2(int N, int C, int H, int W, const float* x, float* y) {
  ho_t4 a = {N, C, H, W, (float*)x};
  ho_t4 o = maxpool2(&a);
  memcpy(y, o.v, sizeof(float) * (size_t)N * C * (H / 2) * (W / 2));
  t4_free(&o);
}
HO_EXPORT void ho_op_upsample2(int N, int C, int H, int W, const float* x, float* y) {
  ho_t4 a = {N, C, H, W, (float*)x};
  ho_t4 o = upsample2(&a);
  memcpy(y, o.v, sizeof(float) * (size_t)N * C * H * W * 4);
  t4_free(&o);
}

/* Encoder (A7, mirrors inc/unet.hpp:231-257 contraction path): level l
 * = [maxpool if l>0] -> relu(conv) -> relu(conv); ctx_l = level output.
 * kappa: (1, 1, H, W).  ctx[l]: (1, base, H>>l, W>>l), caller-allocated. */
HO_EXPORT void ho_encoder_forward(const ho_unet* e, int H, int W, const float* kappa, float** ctx) {
  ho_t4 x = t4_new(1, 1, H, W);
  memcpy(x.v, kappa, sizeof(float) * (size_t)H * W);
  for (int l = 0; l < e->L; ++l) {
    if (l > 0) {
      ho_t4 p = maxpool2(&x);
      t4_free(&x);
      x = p;
    }
    ho_t4 t = conv3x3(&x, NULL, &e->conv[e->enc1[l]], 1);
    t4_free(&x);
    x = conv3x3(&t, NULL, &e->conv[e->enc2[l]], 1);
    t4_free(&t);
    memcpy(ctx[l], x.v, sizeof(float) * (size_t)x.c * x.h * x.w);
  }
  t4_free(&x);
}

/* Solver U-Net forward (A5, with A7 context concat when ctx != NULL):
 *   encoder level l: [maxpool if l>0] [concat ctx_l] relu(conv) relu(conv) -> skip_l
 *   decoder level l = L-2..0: [concat ctx_{l+1}] upsample2 conv (no act)
 *                             concat skip_l, relu(conv), relu(conv)
 *   head: conv3x3 -> 2 channels, no activation (inc/unet.hpp:223-225). */
HO_EXPORT void ho_unet_forward(const ho_unet* n, int B, int H, int W, const float* in, float* const* ctx,
                               float* out) {
  const int L = n->L;
  ho_t4 skip[HO_MAXL];
  ho_t4 x = t4_new(B, n->in_ch, H, W);
  memcpy(x.v, in, sizeof(float) * (size_t)B * n->in_ch * H * W);
  for (int l = 0; l < L; ++l) {
    if (l > 0) {
      ho_t4 p = maxpool2(&x);
      t4_free(&x);
      x = p;
    }
    ho_t4 c;
    if (ctx) {
      ho_t4 cl = {1, n->ctx_ch, x.h, x.w, ctx[l]};
      c = conv3x3(&x, &cl, &n->conv[n->enc1[l]], 1);
    } else {
      c = conv3x3(&x, NULL, &n->conv[n->enc1[l]], 1);
    }
    t4_free(&x);
    x = conv3x3(&c, NULL, &n->conv[n->enc2[l]], 1);
    t4_free(&c);
    skip[l] = x;
    if (l < L - 1) {
      ho_t4 cp = t4_new(x.n, x.c, x.h, x.w);
      memcpy(cp.v, x.v, sizeof(float) * (size_t)x.n * x.c * x.h * x.w);
      x = cp;
    }
  }
  /* x aliases skip[L-1] now */
  for (int l = L - 2; l >= 0; --l) {
    ho_t4 u;
    if (ctx) {
      ho_t4 cl = {1, n->ctx_ch, x.h, x.w, ctx[l + 1]};
      ho_t4 xc = concat(&x, &cl);
      u = upsample2(&xc);
      t4_free(&xc);
    } else {
      u = upsample2(&x);
    }
    t4_free(&x);
    ho_t4 y = conv3x3(&u, NULL, &n->conv[n->up[l]], 0);
    t4_free(&u);
    ho_t4 t = conv3x3(&y, &skip[l], &n->conv[n->dec1[l]], 1);
    t4_free(&y);
    t4_free(&skip[l]);
    x = conv3x3(&t, NULL, &n->conv[n->dec2[l]], 1);
    t4_free(&t);
  }
  ho_t4 o = conv3x3(&x, NULL, &n->conv[n->head], 0);
  t4_free(&x);
  if (L == 1) { /* skip[0] aliased x */ }
  memcpy(out, o.v, sizeof(float) * (size_t)B * 2 * H * W);
  t4_free(&o);
}

/* ------------------------------------------------------------ multigrid --
 * inc/multigrid.hpp:13-21,45-61,70-125 */
enum { HO_COARSE_GMRES = 0, HO_COARSE_JACOBI = 1, HO_COARSE_NET = 2 };

typedef struct {
  int nlev;
  ho_level lev[12];
  int nu1, nu2;
  double damping, alpha, beta;
  int coarse_kind, coarse_iters;
  const ho_unet* coarse_net; /* A4 */
} ho_mg;

static void level_init(ho_level* L, int nx, int ny, double h, double omega, const double* k2, const double* g,
                       double lo, double hi, double alpha, double beta) {
  const size_t n = (size_t)nx * ny;
  L->nx = nx;
  L->ny = ny;
  L->h = h;
  L->omega = omega;
  L->lo = lo;
  L->hi = hi;
  L->k2 = (double*)malloc(sizeof(double) * n);
  L->gam = (double*)malloc(sizeof(double) * n);
  memcpy(L->k2, k2, sizeof(double) * n);
  memcpy(L->gam, g, sizeof(double) * n);
  L->diagA = (cplx*)malloc(sizeof(cplx) * n);
  L->diagM = (cplx*)malloc(sizeof(cplx) * n);
  level_diag(L, 1.0, 0.0, L->diagA);
  level_diag(L, alpha, beta, L->diagM);
}

/* levels: number of V-cycle levels (>= 1; 1 = fine level only, used for the
 * FGMRES operator).  Coefficient coarsening: inc/stencil.hpp:169-185 with the
 * offset (l-1)%2 of inc/multigrid.hpp:80-81. */
HO_EXPORT ho_mg* ho_mg_create(int nx, int ny, double h, double omega, const double* k2, const double* gam,
                              double lo, double hi, int levels, int nu1, int nu2, double damping, double alpha,
                              double beta, int coarse_kind, int coarse_iters) {
  if (levels < 1 || levels > 12) return NULL;
  ho_mg* mg = (ho_mg*)calloc(1, sizeof(ho_mg));
  mg->nlev = levels;
  mg->nu1 = nu1;
  mg->nu2 = nu2;
  mg->damping = damping;
  mg->alpha = alpha;
  mg->beta = beta;
  mg->coarse_kind = coarse_kind;
  mg->coarse_iters = coarse_iters;
  level_init(&mg->lev[0], nx, ny, h, omega, k2, gam, lo, hi, alpha, beta);
  for (int l = 1; l < levels; ++l) {
    ho_level* P = &mg->lev[l - 1];
    const int off = (l - 1) % 2;
    const int cnx = P->nx / 2, cny = P->ny / 2;
    double* ck = (double*)malloc(sizeof(double) * (size_t)cnx * cny);
    double* cg = (double*)malloc(sizeof(double) * (size_t)cnx * cny);
    ho_restrict(P->nx, P->ny, off, 1, P->k2, ck);
    ho_restrict(P->nx, P->ny, off, 1, P->gam, cg);
    for (size_t i = 0; i < (size_t)cnx * cny; ++i) {
      ck[i] = ck[i] < P->lo ? P->lo : (ck[i] > P->hi ? P->hi : ck[i]);
      cg[i] = cg[i] > 0.0 ? cg[i] : 0.0;
    }
    level_init(&mg->lev[l], cnx, cny, P->h * 2.0, omega, ck, cg, lo, hi, alpha, beta);
    free(ck);
    free(cg);
  }
  return mg;
}

HO_EXPORT void ho_mg_destroy(ho_mg* mg) {
  if (!mg) return;
  for (int l = 0; l < mg->nlev; ++l) {
    free(mg->lev[l].k2);
    free(mg->lev[l].gam);
    free(mg->lev[l].diagA);
    free(mg->lev[l].diagM);
  }
  free(mg);
}

HO_EXPORT void ho_mg_set_coarse_net(ho_mg* mg, const ho_unet* net) { mg->coarse_net = net; }

HO_EXPORT void ho_mg_level_info(const ho_mg* mg, int l, int* nx, int* ny, double* h) {
  *nx = mg->lev[l].nx;
  *ny = mg->lev[l].ny;
  *h = mg->lev[l].h;
}
HO_EXPORT void ho_mg_level_coef(const ho_mg* mg, int l, double* k2, double* gam, double* diagA, double* diagM) {
  const size_t n = (size_t)mg->lev[l].nx * mg->lev[l].ny;
  if (k2) memcpy(k2, mg->lev[l].k2, n * sizeof(double));
  if (gam) memcpy(gam, mg->lev[l].gam, n * sizeof(double));
  if (diagA) memcpy(diagA, mg->lev[l].diagA, n * sizeof(cplx));
  if (diagM) memcpy(diagM, mg->lev[l].diagM, n * sizeof(cplx));
}

/* operator helpers on level l; which = 0 -> A^h (shift (1,0)), 1 -> M^h */
HO_EXPORT void ho_apply(const ho_mg* mg, int l, int which, const double* u, double* y) {
  const ho_level* L = &mg->lev[l];
  stencil_apply(L->nx, L->ny, L->h, which ? L->diagM : L->diagA, (const cplx*)u, (cplx*)y);
}
HO_EXPORT void ho_jacobi(const ho_mg* mg, int l, int which, double* v, const double* f, double damping,
                         int iters) {
  const ho_level* L = &mg->lev[l];
  jacobi(L->nx, L->ny, L->h, which ? L->diagM : L->diagA, (cplx*)v, (const cplx*)f, damping, iters);
}

/* ---------------------------------------------------------------- FGMRES --
 * inc/krylov.hpp:83-267, one column (block columns are independent Arnoldi
 * processes; tests/test_classic.cpp:469-508 pins block == single). */
typedef void (*ho_op_fn)(void* ctx, const cplx* in, cplx* out);

typedef struct {
  int restart, max_iters, flexible;
  double rel_tol;
} ho_kcfg;

typedef struct {
  int iterations, converged, breakdown, hist_len;
} ho_krep;

/* make_givens: inc/krylov.hpp:49-64 */
static void make_givens(cplx a, double b, double* c, cplx* s) {
  const double aa = cabs(a);
  const double rho = hypot(aa, b);
  if (rho == 0.0) {
    *c = 1.0;
    *s = 0.0;
  } else if (aa == 0.0) {
    *c = 0.0;
    *s = 1.0;
  } else {
    *c = aa / rho;
    *s = a * b / (rho * aa);
  }
}

static double nrm2(const cplx* v, size_t n) {
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) s += creal(v[i]) * creal(v[i]) + cimag(v[i]) * cimag(v[i]);
  return sqrt(s);
}
static cplx cdot(const cplx* a, const cplx* b, size_t n) {
  cplx s = 0.0;
  for (size_t i = 0; i < n; ++i) s += conj(a[i]) * b[i];
  return s;
}

static void fgmres_column(ho_op_fn A, void* actx, ho_op_fn M, void* mctx, size_t n, const cplx* b, cplx* x,
                          const ho_kcfg* cfg, double* hist, int hist_cap, ho_krep* rep) {
  const int m = cfg->restart;
  cplx* V = (cplx*)malloc(sizeof(cplx) * n * (m + 1));
  cplx* Z = cfg->flexible ? (cplx*)malloc(sizeof(cplx) * n * m) : NULL;
  cplx* w = (cplx*)malloc(sizeof(cplx) * n);
  cplx* zt = (cplx*)malloc(sizeof(cplx) * n);
  cplx* H = (cplx*)calloc((size_t)m * (m + 1), sizeof(cplx)); /* H[j*(m+1)+i] */
  double* rc = (double*)malloc(sizeof(double) * m);
  cplx* rs = (cplx*)malloc(sizeof(cplx) * m);
  cplx* g = (cplx*)malloc(sizeof(cplx) * (m + 1));
  cplx* y = (cplx*)malloc(sizeof(cplx) * m);
  int iters = 0, hlen = 0;
  double beta0 = 0.0;
  rep->converged = 0;
  rep->breakdown = 0;
#define PUSH(v_)                            \
  do {                                      \
    if (hlen < hist_cap) hist[hlen] = (v_); \
    ++hlen;                                 \
  } while (0)
  int frozen = 0;
  while (!frozen) {
    /* restart: true residual (krylov.hpp:153-187) */
    A(actx, x, w);
    for (size_t p = 0; p < n; ++p) V[p] = b[p] - w[p];
    const double beta = nrm2(V, n);
    if (hlen == 0) {
      beta0 = beta;
      PUSH(beta);
      if (beta == 0.0) {
        rep->converged = 1;
        break;
      }
    }
    if (beta / beta0 <= cfg->rel_tol) {
      rep->converged = 1;
      break;
    }
    if (iters >= cfg->max_iters) break;
    for (int i = 0; i <= m; ++i) g[i] = 0.0;
    g[0] = beta;
    const double inv = 1.0 / beta;
    for (size_t p = 0; p < n; ++p) V[p] *= inv;
    int k = 0, done = 0;
    for (int j = 0; j < m; ++j) {
      cplx* Vj = V + (size_t)j * n;
      cplx* zj = cfg->flexible ? Z + (size_t)j * n : zt;
      M(mctx, Vj, zj);
      A(actx, zj, w);
      cplx* hj = H + (size_t)j * (m + 1);
      for (int i = 0; i < j + 2; ++i) hj[i] = 0.0;
      for (int i = 0; i <= j; ++i) { /* MGS krylov.hpp:214-218 */
        const cplx* Vi = V + (size_t)i * n;
        const cplx hij = cdot(Vi, w, n);
        hj[i] = hij;
        for (size_t p = 0; p < n; ++p) w[p] -= hij * Vi[p];
      }
      const double hnorm = nrm2(w, n);
      hj[j + 1] = hnorm;
      for (int i = 0; i < j; ++i) {
        const cplx t = rc[i] * hj[i] + rs[i] * hj[i + 1];
        hj[i + 1] = -conj(rs[i]) * hj[i] + rc[i] * hj[i + 1];
        hj[i] = t;
      }
      make_givens(hj[j], hnorm, &rc[j], &rs[j]);
      hj[j] = rc[j] * hj[j] + rs[j] * hj[j + 1];
      hj[j + 1] = 0.0;
      g[j + 1] = -conj(rs[j]) * g[j];
      g[j] = rc[j] * g[j];
      k = j + 1;
      iters += 1;
      const double est = cabs(g[j + 1]);
      PUSH(est);
      const int happy = hnorm <= 1e-14 * beta0;
      if (happy) rep->breakdown = 1;
      if (est / beta0 <= cfg->rel_tol || happy) {
        rep->converged = 1;
        frozen = 1;
        done = 1;
      } else if (iters >= cfg->max_iters) {
        frozen = 1;
        done = 1;
      } else if (k < m) {
        const double invn = 1.0 / hnorm;
        cplx* Vn = V + (size_t)(j + 1) * n;
        for (size_t p = 0; p < n; ++p) Vn[p] = w[p] * invn;
      }
      if (done) break;
    }
    /* finalize (krylov.hpp:119-140) */
    for (int i = k - 1; i >= 0; --i) {
      cplx sum = g[i];
      for (int l = i + 1; l < k; ++l) sum -= H[(size_t)l * (m + 1) + i] * y[l];
      y[i] = sum / H[(size_t)i * (m + 1) + i];
    }
    if (cfg->flexible) {
      for (int i = 0; i < k; ++i)
        for (size_t p = 0; p < n; ++p) x[p] += y[i] * Z[(size_t)i * n + p];
    } else if (k > 0) {
      for (size_t p = 0; p < n; ++p) zt[p] = 0.0;
      for (int i = 0; i < k; ++i)
        for (size_t p = 0; p < n; ++p) zt[p] += y[i] * V[(size_t)i * n + p];
      M(mctx, zt, w);
      for (size_t p = 0; p < n; ++p) x[p] += w[p];
    }
  }
#undef PUSH
  rep->iterations = iters;
  rep->hist_len = hlen;
  free(V);
  free(Z);
  free(w);
  free(zt);
  free(H);
  free(rc);
  free(rs);
  free(g);
  free(y);
}

/* ----------------------------------------------------- coarse + V-cycle -- */
typedef struct {
  const ho_level* L;
  int diag_which; /* 0 A, 1 M */
} op_ctx;

static void op_apply_cb(void* c, const cplx* in, cplx* out) {
  const op_ctx* o = (const op_ctx*)c;
  stencil_apply(o->L->nx, o->L->ny, o->L->h, o->diag_which ? o->L->diagM : o->L->diagA, in, out);
}
static void op_diaginv_cb(void* c, const cplx* in, cplx* out) {
  const op_ctx* o = (const op_ctx*)c;
  const size_t n = (size_t)o->L->nx * o->L->ny;
  const cplx* d = o->diag_which ? o->L->diagM : o->L->diagA;
  for (size_t i = 0; i < n; ++i) out[i] = in[i] / d[i];
}

/* inc/multigrid.hpp:45-61: GMRES(coarse_iters), non-flexible, M = D^-1,
 * x0 = 0, rel_tol 1e-300 (fixed budget). */
static void coarse_gmres(const ho_level* L, int iters, const cplx* f, cplx* x) {
  const size_t n = (size_t)L->nx * L->ny;
  op_ctx oc = {L, 1};
  ho_kcfg kc = {iters, iters, 0, 1e-300};
  ho_krep rep;
  double hist[1];
  for (size_t i = 0; i < n; ++i) x[i] = 0.0;
  fgmres_column(op_apply_cb, &oc, op_diaginv_cb, &oc, n, f, x, &kc, hist, 0, &rep);
}

/* A4: the coarse-net solve on [H^2 Re f, H^2 Im f, kappa^2_c] (H = coarse
 * mesh width; packing as inc/precond.hpp:74-83 with gamma dropped). */
static void coarse_net_solve(const ho_level* L, const ho_unet* net, const cplx* f, cplx* x) {
  const int nx = L->nx, ny = L->ny;
  const size_t n = (size_t)nx * ny;
  const double h2 = L->h * L->h;
  float* in = (float*)malloc(sizeof(float) * 3 * n);
  float* out = (float*)malloc(sizeof(float) * 2 * n);
  for (size_t i = 0; i < n; ++i) {
    in[i] = (float)(h2 * creal(f[i]));
    in[n + i] = (float)(h2 * cimag(f[i]));
    in[2 * n + i] = (float)L->k2[i];
  }
  ho_unet_forward(net, 1, ny, nx, in, NULL, out);
  for (size_t i = 0; i < n; ++i) x[i] = (double)out[i] + (double)out[n + i] * I;
  free(in);
  free(out);
}

/* inc/multigrid.hpp:108-119 */
static void cycle_at(const ho_mg* mg, int level, cplx* v, const cplx* f) {
  const ho_level* L = &mg->lev[level];
  const size_t n = (size_t)L->nx * L->ny;
  if (level == mg->nlev - 1) {
    if (mg->coarse_kind == HO_COARSE_GMRES) {
      coarse_gmres(L, mg->coarse_iters, f, v);
    } else if (mg->coarse_kind == HO_COARSE_JACOBI) { /* A3 */
      for (size_t i = 0; i < n; ++i) v[i] = 0.0;
      jacobi(L->nx, L->ny, L->h, L->diagM, v, f, mg->damping, mg->coarse_iters);
    } else {
      coarse_net_solve(L, mg->coarse_net, f, v);
    }
    return;
  }
  const int offset = level % 2;
  jacobi(L->nx, L->ny, L->h, L->diagM, v, f, mg->damping, mg->nu1);
  cplx* r = (cplx*)malloc(sizeof(cplx) * n);
  stencil_apply(L->nx, L->ny, L->h, L->diagM, v, r);
  for (size_t i = 0; i < n; ++i) r[i] = f[i] - r[i];
  const ho_level* C = &mg->lev[level + 1];
  const size_t nc = (size_t)C->nx * C->ny;
  cplx* fc = (cplx*)malloc(sizeof(cplx) * nc);
  cplx* vc = (cplx*)calloc(nc, sizeof(cplx));
  ho_restrict(L->nx, L->ny, offset, 2, (const double*)r, (double*)fc);
  cycle_at(mg, level + 1, vc, fc);
  ho_prolong(C->nx, C->ny, offset, 2, (const double*)vc, (double*)r); /* r reused as corr */
  for (size_t i = 0; i < n; ++i) v[i] += r[i];
  jacobi(L->nx, L->ny, L->h, L->diagM, v, f, mg->damping, mg->nu2);
  free(r);
  free(fc);
  free(vc);
}

/* cycle(v0, f): v0 may be NULL (zero guess); result in out. */
HO_EXPORT void ho_mg_cycle(const ho_mg* mg, const double* v0, const double* f, double* out) {
  const size_t n = (size_t)mg->lev[0].nx * mg->lev[0].ny;
  if (v0)
    memcpy(out, v0, sizeof(cplx) * n);
  else
    memset(out, 0, sizeof(cplx) * n);
  cycle_at(mg, 0, (cplx*)out, (const cplx*)f);
}

HO_EXPORT void ho_coarse_gmres(const ho_mg* mg, int l, int iters, const double* f, double* x) {
  coarse_gmres(&mg->lev[l], iters, (const cplx*)f, (cplx*)x);
}

/* ------------------------------------------------------- preconditioners --
 * inc/precond.hpp: M_V (:35-53), M_VU (:143-165, A8), M_JU (:104-139, with
 * the classic A5 net), coarse-net cycle (A4; it is M_V whose hierarchy has
 * coarse_kind NET). */
enum { HO_PC_V = 0, HO_PC_VU = 1, HO_PC_JU = 2 };

typedef struct {
  int kind;
  const ho_mg* mg;
  const ho_unet* net; /* M_VU solver net */
  float** ctx;        /* encoder context per level (encoder-solver), or NULL */
  float* k2f;         /* fine kappa^2 as float */
} ho_pc;

HO_EXPORT ho_pc* ho_pc_create(int kind, const ho_mg* mg, const ho_unet* net, const ho_unet* enc) {
  ho_pc* p = (ho_pc*)calloc(1, sizeof(ho_pc));
  p->kind = kind;
  p->mg = mg;
  p->net = net;
  const ho_level* L = &mg->lev[0];
  const size_t n = (size_t)L->nx * L->ny;
  p->k2f = (float*)malloc(sizeof(float) * n);
  for (size_t i = 0; i < n; ++i) p->k2f[i] = (float)L->k2[i];
  if (enc) { /* encoder runs once per medium, cached (inc/precond.hpp:66-67) */
    p->ctx = (float**)calloc(enc->L, sizeof(float*));
    for (int l = 0; l < enc->L; ++l)
      p->ctx[l] = (float*)malloc(sizeof(float) * (size_t)enc->base * (L->nx >> l) * (L->ny >> l));
    ho_encoder_forward(enc, L->ny, L->nx, p->k2f, p->ctx);
  }
  return p;
}

HO_EXPORT void ho_pc_destroy(ho_pc* p) {
  if (!p) return;
  if (p->ctx) {
    for (int l = 0; l < HO_MAXL && p->ctx[l]; ++l) free(p->ctx[l]);
    free(p->ctx);
  }
  free(p->k2f);
  free(p);
}

HO_EXPORT const float* ho_pc_ctx(const ho_pc* p, int l) { return p->ctx ? p->ctx[l] : NULL; }

/* e0 = net([h^2 Re r, h^2 Im r, kappa^2]) (inc/precond.hpp:71-91, gamma dropped) */
static void pc_net_guess(const ho_pc* p, const cplx* r, cplx* e0) {
  const ho_level* L = &p->mg->lev[0];
  const size_t n = (size_t)L->nx * L->ny;
  const double h2 = L->h * L->h;
  float* in = (float*)malloc(sizeof(float) * 3 * n);
  float* out = (float*)malloc(sizeof(float) * 2 * n);
  for (size_t i = 0; i < n; ++i) {
    in[i] = (float)(h2 * creal(r[i]));
    in[n + i] = (float)(h2 * cimag(r[i]));
    in[2 * n + i] = p->k2f[i];
  }
  ho_unet_forward(p->net, 1, L->ny, L->nx, in, p->ctx, out);
  for (size_t i = 0; i < n; ++i) e0[i] = (double)out[i] + (double)out[n + i] * I;
  free(in);
  free(out);
}

static void pc_apply_one(void* c, const cplx* r, cplx* z) {
  const ho_pc* p = (const ho_pc*)c;
  const ho_level* L0 = &p->mg->lev[0];
  const size_t n = (size_t)L0->nx * L0->ny;
  if (p->kind == HO_PC_JU) {
    /* inc/precond.hpp:112-130: e1 = J_A(0, r); de = net(r - A e1); z = J_A(e1 + de, r), omega = 0.8 */
    cplx* e1 = (cplx*)calloc(n, sizeof(cplx));
    cplx* res = (cplx*)malloc(sizeof(cplx) * n);
    cplx* de = (cplx*)malloc(sizeof(cplx) * n);
    jacobi(L0->nx, L0->ny, L0->h, L0->diagA, e1, r, 0.8, 1);
    stencil_apply(L0->nx, L0->ny, L0->h, L0->diagA, e1, res);
    for (size_t i = 0; i < n; ++i) res[i] = r[i] - res[i];
    pc_net_guess(p, res, de);
    for (size_t i = 0; i < n; ++i) z[i] = e1[i] + de[i];
    jacobi(L0->nx, L0->ny, L0->h, L0->diagA, z, r, 0.8, 1);
    free(e1);
    free(res);
    free(de);
    return;
  }
  if (p->kind == HO_PC_V) {
    memset(z, 0, sizeof(cplx) * n);
  } else {
    pc_net_guess(p, r, z);
  }
  cycle_at(p->mg, 0, z, r);
}

HO_EXPORT void ho_pc_apply(const ho_pc* p, int B, const double* r, double* z) {
  const size_t n = (size_t)p->mg->lev[0].nx * p->mg->lev[0].ny;
  for (int b = 0; b < B; ++b) pc_apply_one((void*)p, (const cplx*)r + b * n, (cplx*)z + b * n);
}

/* net-only test hook: e0 = net(h^2 r, kappa^2) */
HO_EXPORT void ho_pc_net_guess(const ho_pc* p, const double* r, double* e0) {
  pc_net_guess(p, (const cplx*)r, (cplx*)e0);
}

/* Block FGMRES with A = A^h on level 0 of mg and M = pc, columns in
 * parallel (nthreads; columns are independent, krylov.hpp:78-82).
 * hist: B x hist_cap; outputs per column: iterations, converged, breakdown,
 * hist_len.  x: B x n (initial guess in, solution out). */
HO_EXPORT void ho_fgmres(const ho_pc* pc, int restart, int max_iters, double rel_tol, int flexible, int B,
                         const double* b, double* x, double* hist, int hist_cap, int* iters, int* conv,
                         int* brk, int* hlen, int nthreads) {
  const ho_level* L = &pc->mg->lev[0];
  const size_t n = (size_t)L->nx * L->ny;
  ho_kcfg kc = {restart, max_iters, flexible, rel_tol};
  op_ctx oc = {L, 0};
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1) if (nthreads != 1)
#endif
  for (int c = 0; c < B; ++c) {
    ho_krep rep;
    fgmres_column(op_apply_cb, &oc, pc_apply_one, (void*)pc, n, (const cplx*)b + c * n, (cplx*)x + c * n,
                  &kc, hist + (size_t)c * hist_cap, hist_cap, &rep);
    iters[c] = rep.iterations;
    conv[c] = rep.converged;
    brk[c] = rep.breakdown;
    hlen[c] = rep.hist_len;
  }
  (void)nthreads;
}

/* inc/bench.hpp:22-38 convergence factor (T, rho) */
HO_EXPORT int ho_convergence_factor(const double* hist, int len, double target_drop, double* rho) {
  for (int t = 1; t < len; ++t) {
    const double ratio = hist[t] / hist[0];
    if (ratio <= 1.0 / target_drop) {
      *rho = pow(ratio, 1.0 / (double)t);
      return t;
    }
  }
  *rho = NAN;
  return -(len - 1);
}
