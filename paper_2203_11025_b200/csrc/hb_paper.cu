// The paper's U-Net: the network the reference trains
// and checkpoints (inc/unet.hpp:113-257), in eval mode, on the device --
// 5x5 stride-2 down-convolutions, ResNet blocks (3x3 conv, batch norm, ELU,
// residual add), 5x5 stride-2 transposed up-convolutions, skip concatenation,
// a 3x3 output head; optional encoder over kappa^2 whose feature maps are
// concatenated before every down- and up-convolution (encoder_solver).  The
// input is the reference's 4-channel (h^2 Re r, h^2 Im r, kappa^2, gamma) stack
// (inc/precond.hpp:74-90).  Parameters live in a registry with the reference's
// names and creation order (NetworkWeights, inc/unet.hpp:10-111), initialised
// by the same Rng draws or loaded from / saved to UNW1 checkpoints
// (inc/checkpoint.hpp:12-104) byte-compatibly.
//
// Device layout: NHWC fp32 (channel-concatenations are channel slices of one
// buffer).  Every convolution is one direct-convolution kernel (thread per
// output pixel, 16 output channels per pass, weights [tap][cin][cout] read as
// warp-uniform broadcasts) with the batch norm, bias, residual add and ELU
// fused into its epilogue and the up-path's ELU fused into its input loads.
#include <cuda_runtime.h>

#include <array>
#include <cmath>
#include <cstring>
#include <fstream>
#include <map>
#include <string>
#include <vector>

#include "hb_common.cuh"
#include "hb_host.h"
#include "hb_internal.h"
#include "hb_paper.h"

namespace hb {

namespace {

// ------------------------------------------------------------- layout --
// creation order of build_encoder / build_unet (inc/unet.hpp:139-257)
int solver_ch(const hb_unet_cfg& c, int l) { return c.base_channels << (l - 1); }
int up_out_ch(const hb_unet_cfg& c, int t) { return t >= 1 ? (c.base_channels << (t - 1)) : c.base_channels / 2; }
int enc_ch(const hb_unet_cfg& c, int l) { return l == 0 ? c.base_channels / 2 : (c.base_channels << (l - 1)); }

struct Layout {
  std::vector<std::pair<std::string, std::array<int, 4>>> p;
  void kernel(const std::string& n, int a, int b, int k) { p.push_back({n, {a, b, k, k}}); }
  void vec(const std::string& n, int c) { p.push_back({n, {1, c, 1, 1}}); }
  void bn(const std::string& n, int c) {
    vec(n + ".scale", c);
    vec(n + ".offset", c);
    vec(n + ".rmean", c);
    vec(n + ".rvar", c);
    p.push_back({n + ".count", {1, 1, 1, 1}});
  }
  void resnet(const std::string& n, int ch, int k) {
    kernel(n + ".k1", ch, ch, k);
    vec(n + ".b1", ch);
    bn(n + ".bn1", ch);
    kernel(n + ".k2", ch, ch, k);
    vec(n + ".b2", ch);
    bn(n + ".bn2", ch);
  }
};

Layout make_layout(const hb_unet_cfg& c, int variant, int in_ch) {
  Layout L;
  const bool es = variant == 1;
  if (es) {  // build_encoder (inc/unet.hpp:231-257), created first by NetworkApplier
    int cur = enc_ch(c, 0);
    L.kernel("enc.entry.k", cur, 1, c.res_kernel);
    L.vec("enc.entry.b", cur);
    L.bn("enc.entry.bn", cur);
    for (int l = 0; l < c.levels; ++l) {
      const int out = enc_ch(c, l + 1);
      const std::string d = "enc.down" + std::to_string(l);
      L.kernel(d + ".k", out, cur, c.updown_kernel);
      L.vec(d + ".b", out);
      L.bn(d + ".bn", out);
      cur = out;
      for (int r = 0; r < c.resnet_per_level; ++r)
        L.resnet("enc.res" + std::to_string(l + 1) + "_" + std::to_string(r), cur, c.res_kernel);
    }
  }
  const std::string pre = es ? "sol." : "unet.";
  int cur = in_ch;
  for (int l = 0; l < c.levels; ++l) {
    if (es) cur += enc_ch(c, l);
    const int out = solver_ch(c, l + 1);
    const std::string d = pre + "down" + std::to_string(l);
    L.kernel(d + ".k", out, cur, c.updown_kernel);
    L.vec(d + ".b", out);
    L.bn(d + ".bn", out);
    cur = out;
    if (l < c.levels - 1)
      for (int r = 0; r < c.resnet_per_level; ++r)
        L.resnet(pre + "res" + std::to_string(l + 1) + "_" + std::to_string(r), cur, c.res_kernel);
  }
  for (int r = 0; r < c.bottleneck_resnets; ++r) L.resnet(pre + "bot" + std::to_string(r), cur, c.res_kernel);
  for (int s = c.levels; s >= 1; --s) {
    const int t = s - 1;
    if (es) cur += enc_ch(c, s);
    const int out = up_out_ch(c, t);
    const std::string u = pre + "up" + std::to_string(t);
    L.kernel(u + ".k", cur, out, c.updown_kernel);  // transposed: (x channels, out channels, k, k)
    L.vec(u + ".b", out);
    L.bn(u + ".bn", out);
    cur = out + (t >= 1 ? solver_ch(c, t) : in_ch);
  }
  L.kernel(pre + "out.k", 2, cur, 3);
  L.vec(pre + "out.b", 2);
  return L;
}

bool ends_with(const std::string& s, const char* t) {
  const size_t n = std::strlen(t);
  return s.size() >= n && s.compare(s.size() - n, n, t) == 0;
}

// NetworkWeights init (inc/unet.hpp:13-33, tensor.hpp:55-57): kernels uniform
// +-1/sqrt(c_in k k) from one Rng in creation order; vectors constant
void init_params(PaperState& P, uint64_t seed) {
  Rng rng(seed);
  for (auto& q : P.params) {
    q.v.assign(q.size(), 0.f);
    const bool kern = q.d[2] > 1 || ends_with(q.name, ".k") || ends_with(q.name, ".k1") || ends_with(q.name, ".k2");
    if (kern) {
      const float bound = 1.0f / std::sqrt(float(q.d[1]) * q.d[2] * q.d[3]);
      for (auto& x : q.v) x = float(rng.uniform(double(-bound), double(bound)));
    } else if (ends_with(q.name, ".scale") || ends_with(q.name, ".rvar")) {
      for (auto& x : q.v) x = 1.0f;
    }
  }
}

void set_layout(PaperState& P, const hb_unet_cfg& c, int variant) {
  P.cfg = c;
  P.variant = variant;
  P.params.clear();
  P.index.clear();
  for (auto& e : make_layout(c, variant, 4).p) {
    PParam q;
    q.name = e.first;
    for (int i = 0; i < 4; ++i) q.d[i] = e.second[size_t(i)];
    P.index[q.name] = P.params.size();
    P.params.push_back(std::move(q));
  }
  P.dev.clear();
  P.dirty = true;
  ++P.host_gen;
  P.feat_gen = ~0ull;
}

PParam& param(PaperState& P, const std::string& n) {
  auto it = P.index.find(n);
  if (it == P.index.end()) throw HbError{HB_ERR_ARG, "paper net has no parameter " + n};
  return P.params[it->second];
}

// ---- device upload: weights repacked to [tap][cin][cout], bn buffers per channel
void upload_conv(PaperState& P, const std::string& kname, const std::string& bname, const std::string& bn,
                 bool transpose) {
  PParam& K = param(P, kname);
  PParam& Bq = param(P, bname);
  DevConv& D = P.dev[kname];
  const int a = K.d[0], b = K.d[1], k = K.d[2];
  D.k = k;
  D.transpose = transpose;
  D.cout = transpose ? b : a;
  D.cin = transpose ? a : b;
  std::vector<float> w(size_t(k) * k * D.cin * D.cout);
  for (int i = 0; i < a; ++i)
    for (int j = 0; j < b; ++j)
      for (int t = 0; t < k * k; ++t) {
        const float x = K.v[(size_t(i) * b + j) * k * k + t];
        const int co = transpose ? j : i, ci = transpose ? i : j;
        w[(size_t(t) * D.cin + ci) * D.cout + co] = x;
      }
  auto up = [](DBuf<float>& d, const std::vector<float>& h) {
    d.ensure(h.size());
    HB_CUDA(cudaMemcpy(d.p, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice));
  };
  up(D.w, w);
  up(D.bias, Bq.v);
  if ((D.cin == 12 || D.cin == 16 || D.cin == 20) && D.cout == 2 && k == 3 && !transpose) {  // output layer: k_conv_cols
    D.hw = w;
    D.hb = Bq.v;
  } else {
    D.hw.clear();
    D.hb.clear();
  }
  // tensor-core form (hb_conv_tc.cu): taps as input offsets (dy, dx) of the
  // output pixel's stride-s origin, weights packed [cout][tap][cin]
  D.tc.clear();
  // output channels padded to a multiple of 16 with zero weights (the up path's
  // base/2 = 8-channel layer); the epilogue stores only the real ones
  const int coutp = (D.cout + 15) / 16 * 16;
  if (D.cin % 16 == 0 && coutp <= 256 && k <= 5) {
    const int pad = (k - 1) / 2;
    auto padv = [&](const std::vector<float>& v, float fill) {
      std::vector<float> o(v);
      o.resize(size_t(coutp), fill);
      return o;
    };
    auto make = [&](const std::vector<std::pair<int, int>>& tk, const std::vector<std::pair<int, int>>& off, int py,
                    int px) {
      PaperTc T;
      T.cw.cout = coutp;
      T.cw.cin = D.cin;
      const int nt = int(tk.size());
      std::vector<float> packed(size_t(coutp) * nt * D.cin, 0.f);
      for (int co = 0; co < D.cout; ++co)
        for (int t = 0; t < nt; ++t)
          for (int ci = 0; ci < D.cin; ++ci)
            packed[(size_t(co) * nt + t) * D.cin + ci] = w[(size_t(tk[t].first * k + tk[t].second) * D.cin + ci) * D.cout + co];
      conv_tc_upload_packed(T.cw, packed);
      up(T.cw.db, padv(Bq.v, 0.f));
      int oy = 0, ox = 0;
      for (auto& o : off) {
        oy = std::min(oy, o.first);
        ox = std::min(ox, o.second);
      }
      T.geo = TcGeo{};
      T.geo.ntaps = nt;
      T.geo.oy = oy;
      T.geo.ox = ox;
      T.geo.py = py;
      T.geo.px = px;
      for (int t = 0; t < nt; ++t) {
        T.geo.ty[t] = off[t].first - oy;
        T.geo.tx[t] = off[t].second - ox;
      }
      D.tc.push_back(std::move(T));
    };
    if (!transpose) {  // conv2d (inc/autodiff.hpp:31-39): input (o s + ky - pad, o s + kx - pad)
      std::vector<std::pair<int, int>> tk, off;
      for (int ky = 0; ky < k; ++ky)
        for (int kx = 0; kx < k; ++kx) {
          tk.push_back({ky, kx});
          off.push_back({ky - pad, kx - pad});
        }
      make(tk, off, 0, 0);
    } else if (P.par4 && D.cin % 16 == 0 && 4 * coutp <= 128) {
      // conv2d_transpose, stride 2 (:190-215), all four output parity classes in ONE
      // implicit GEMM: output pixel 2o + p meets kernel taps k = p + pad - 2d at
      // input o + d, d in {-1, 0, 1}^2 -- a 3x3 neighbourhood shared by the classes;
      // N = 4 x coutp (class q = 2 py + px in channel block q, zero weights where a
      // class has no tap) and the epilogue scatters block q to (2o_y + py, 2o_x + px):
      // one launch of N = 64 MMAs instead of four launches of N = 16 (25 taps)
      PaperTc T;
      T.cw.cout = 4 * coutp;
      T.cw.cin = D.cin;
      std::vector<float> packed(size_t(4) * coutp * 9 * D.cin, 0.f);
      for (int q = 0; q < 4; ++q) {
        const int py = q >> 1, px = q & 1;
        for (int t = 0; t < 9; ++t) {
          const int dy = t / 3 - 1, dx = t % 3 - 1;
          const int ky = py + pad - 2 * dy, kx = px + pad - 2 * dx;
          if (ky < 0 || ky >= k || kx < 0 || kx >= k) continue;
          for (int co = 0; co < D.cout; ++co)
            for (int ci = 0; ci < D.cin; ++ci)
              packed[(size_t(q * coutp + co) * 9 + t) * D.cin + ci] = w[(size_t(ky * k + kx) * D.cin + ci) * D.cout + co];
        }
      }
      conv_tc_upload_packed(T.cw, packed);
      std::vector<float> b4;
      for (int q = 0; q < 4; ++q) {
        const std::vector<float> bq = padv(Bq.v, 0.f);
        b4.insert(b4.end(), bq.begin(), bq.end());
      }
      up(T.cw.db, b4);
      T.geo = TcGeo{};
      T.geo.ntaps = 9;
      T.geo.oy = T.geo.ox = -1;
      for (int t = 0; t < 9; ++t) {
        T.geo.ty[t] = t / 3;
        T.geo.tx[t] = t % 3;
      }
      T.geo.par4 = coutp;
      T.geo.par4_kk = k * k;
      D.tc.push_back(std::move(T));
    } else {  // conv2d_transpose, stride 2 (:190-215): output class (py, px) of pixel 2 o + p meets taps
      // k = p + pad (mod 2), input o + (p + pad - k) / 2
      for (int py = 0; py < 2; ++py)
        for (int px = 0; px < 2; ++px) {
          std::vector<std::pair<int, int>> tk, off;
          for (int ky = (py + pad) & 1; ky < k; ky += 2)
            for (int kx = (px + pad) & 1; kx < k; kx += 2) {
              tk.push_back({ky, kx});
              off.push_back({(py + pad - ky) / 2, (px + pad - kx) / 2});
            }
          make(tk, off, py, px);
        }
    }
  }
  D.bn = !bn.empty();
  if (D.bn) {
    if (param(P, bn + ".count").v[0] <= 0.0f)
      throw HbError{HB_ERR_NUMERIC, "batch_norm eval mode before any running-stat update (" + bn + ")"};
    const PParam& rv = param(P, bn + ".rvar");
    std::vector<float> is(size_t(D.cout));
    for (int ch = 0; ch < D.cout; ++ch) is[size_t(ch)] = float(1.0 / std::sqrt(double(rv.v[size_t(ch)]) + 1e-5));
    up(D.mu, param(P, bn + ".rmean").v);
    up(D.is, is);
    up(D.g, param(P, bn + ".scale").v);
    up(D.be, param(P, bn + ".offset").v);
    auto padv = [&](const std::vector<float>& v, float fill) {
      std::vector<float> o(v);
      o.resize(size_t(coutp), fill);
      return o;
    };
    for (PaperTc& T : D.tc) {
      const int rep = T.geo.par4 ? 4 : 1;  // one copy per parity-class channel block
      auto padr = [&](const std::vector<float>& v, float fill) {
        std::vector<float> o;
        for (int r = 0; r < rep; ++r) {
          const std::vector<float> b = padv(v, fill);
          o.insert(o.end(), b.begin(), b.end());
        }
        return o;
      };
      up(T.mu, padr(param(P, bn + ".rmean").v, 0.f));
      up(T.is, padr(is, 1.f));
      up(T.g, padr(param(P, bn + ".scale").v, 1.f));
      up(T.be, padr(param(P, bn + ".offset").v, 0.f));
    }
  }
}

void upload_all(PaperState& P) {
  const hb_unet_cfg& c = P.cfg;
  const bool es = P.variant == 1;
  auto res = [&](const std::string& n) {
    upload_conv(P, n + ".k1", n + ".b1", n + ".bn1", false);
    upload_conv(P, n + ".k2", n + ".b2", n + ".bn2", false);
  };
  if (es) {
    upload_conv(P, "enc.entry.k", "enc.entry.b", "enc.entry.bn", false);
    for (int l = 0; l < c.levels; ++l) {
      const std::string d = "enc.down" + std::to_string(l);
      upload_conv(P, d + ".k", d + ".b", d + ".bn", false);
      for (int r = 0; r < c.resnet_per_level; ++r) res("enc.res" + std::to_string(l + 1) + "_" + std::to_string(r));
    }
  }
  const std::string pre = es ? "sol." : "unet.";
  for (int l = 0; l < c.levels; ++l) {
    const std::string d = pre + "down" + std::to_string(l);
    upload_conv(P, d + ".k", d + ".b", d + ".bn", false);
    if (l < c.levels - 1)
      for (int r = 0; r < c.resnet_per_level; ++r) res(pre + "res" + std::to_string(l + 1) + "_" + std::to_string(r));
  }
  for (int r = 0; r < c.bottleneck_resnets; ++r) res(pre + "bot" + std::to_string(r));
  for (int t = 0; t < c.levels; ++t) {
    const std::string u = pre + "up" + std::to_string(t);
    upload_conv(P, u + ".k", u + ".b", u + ".bn", true);
  }
  upload_conv(P, pre + "out.k", pre + "out.b", "", false);
  P.dirty = false;
  ++g_alloc_gen;  // the output layer carries its weights as kernel parameters: drop captured graphs
}

// ------------------------------------------------------------- kernels --
__device__ __forceinline__ float elu(float t) { return t >= 0.0f ? t : expm1f(t); }

struct PConv {
  const float* x;
  int ldx, cin, Hin, Win;
  float* y;
  int ldy, cout, Ho, Wo;
  const float *w, *bias, *mu, *is, *g, *be, *res;
  int ldres;
  int k, stride, transpose, in_elu, act, B;
  int xbatch;  // 0: the input is one image shared by every batch item (encoder features)
};

// thread per output pixel, CO output channels per pass; cross-correlation with
// zero padding (k-1)/2 (inc/autodiff.hpp:36-69) or its exact adjoint for
// transpose (gather form of col2im, inc/autodiff.hpp:190-215)
template <int CO>
__global__ void __launch_bounds__(128) k_pconv(PConv a) {
  pdl_enter();
  const long long npix = (long long)a.B * a.Ho * a.Wo;
  const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= npix) return;
  const int b = int(p / ((long long)a.Ho * a.Wo));
  const int rem = int(p - (long long)b * a.Ho * a.Wo);
  const int oy = rem / a.Wo, ox = rem - oy * a.Wo;
  const int pad = (a.k - 1) / 2;
  const int bx = a.xbatch ? b : 0;
  for (int c0 = 0; c0 < a.cout; c0 += CO) {
    float acc[CO];
#pragma unroll
    for (int j = 0; j < CO; ++j) acc[j] = 0.f;
    const int nco = min(CO, a.cout - c0);
    for (int ky = 0; ky < a.k; ++ky) {
      int iy;
      if (!a.transpose) {
        iy = oy * a.stride + ky - pad;
      } else {
        iy = oy + pad - ky;
        if (a.stride == 2) {
          if (iy & 1) continue;
          iy >>= 1;
        }
      }
      if (iy < 0 || iy >= a.Hin) continue;
      for (int kx = 0; kx < a.k; ++kx) {
        int ix;
        if (!a.transpose) {
          ix = ox * a.stride + kx - pad;
        } else {
          ix = ox + pad - kx;
          if (a.stride == 2) {
            if (ix & 1) continue;
            ix >>= 1;
          }
        }
        if (ix < 0 || ix >= a.Win) continue;
        const float* xp = a.x + ((size_t(bx) * a.Hin + iy) * a.Win + ix) * a.ldx;
        const float* wp = a.w + (size_t(ky * a.k + kx) * a.cin) * a.cout + c0;
        for (int ci = 0; ci < a.cin; ++ci) {
          float v = __ldg(xp + ci);
          if (a.in_elu) v = elu(v);
          const float* wr = wp + size_t(ci) * a.cout;
          if (nco == CO) {
#pragma unroll
            for (int j = 0; j < CO; ++j) acc[j] = fmaf(v, __ldg(wr + j), acc[j]);
          } else {
            for (int j = 0; j < nco; ++j) acc[j] = fmaf(v, __ldg(wr + j), acc[j]);
          }
        }
      }
    }
    float* yp = a.y + size_t(p) * a.ldy + c0;
    const float* rp = a.res ? a.res + size_t(p) * a.ldres + c0 : nullptr;
#pragma unroll
    for (int j = 0; j < CO; ++j) {
      if (j >= nco) break;
      const int co = c0 + j;
      float t = acc[j] + a.bias[co];
      if (rp) t = rp[j] + t;  // tape.add(x, t) (inc/unet.hpp:158)
      if (a.mu) t = ((t - a.mu[co]) * a.is[co]) * a.g[co] + a.be[co];  // batch_norm eval (inc/autodiff.hpp:289-296)
      if (a.act) t = elu(t);
      yp[j] = t;
    }
  }
}

// Register-tiled variant: a CTA owns 128*P output pixels x CO output channels
// (CO = 16, or 4 for the narrow output layers); each thread P pixels (128
// apart: coalesced stores) x CO channels = CO*P accumulators.  Weights of a
// 16-input-channel chunk (all taps, CO outputs, zero-padded) are staged in
// shared memory and read as warp-uniform float4 broadcasts; inputs come from
// global (L1) as float4 over 4 channels.  At one pixel per thread (the small,
// latency-bound layers) the input loads of a whole tap row (up to 5 taps) are
// issued before its FMAs: one memory round trip per tap row, not per tap.
constexpr int PC_T = 128, PC_CI = 16, PC_KMAX = 5;
// Stride-2 transposed convolutions run per output parity class (blockIdx.z):
// class (py, px) only meets taps ky = py + pad (mod 2), kx = px + pad (mod 2),
// so no work is spent on the 3/4 of the taps that miss.
template <int P, bool VEC, int CO>  // VEC: cin % 4 == 0 and ldx % 4 == 0 (float4 input loads)
__global__ void __launch_bounds__(PC_T) k_pconv_tiled(PConv a) {
  // input loads batched ahead of their FMAs: KB taps of a row (registers allow it
  // at P = 1) x CB float4 channel groups (more measured slower: occupancy)
  constexpr int KB = P == 1 ? PC_KMAX : 1, CB = 1;
  pdl_enter();
  extern __shared__ float4 sw4[];  // [tap][ci_local][CO] as float4 x CO/4
  float* sw = reinterpret_cast<float*>(sw4);
  const int t = threadIdx.x;
  const int co0 = blockIdx.y * CO;
  const int nco = min(CO, a.cout - co0);
  const bool par = a.transpose && a.stride == 2;
  const int cls = blockIdx.z, py = cls >> 1, px = cls & 1;
  const int Hc = par ? (a.Ho - py + 1) / 2 : a.Ho, Wc = par ? (a.Wo - px + 1) / 2 : a.Wo;  // class grid
  const long long npix = (long long)a.B * Hc * Wc;
  const int pad = (a.k - 1) / 2, kk = a.k * a.k;
  const int ky0 = par ? ((py + pad) & 1) : 0, kx0 = par ? ((px + pad) & 1) : 0, kst = par ? 2 : 1;
  int pb[P], poy[P], pox[P];
  long long pout[P];
  bool pv[P];
#pragma unroll
  for (int q = 0; q < P; ++q) {
    const long long p = (long long)blockIdx.x * (PC_T * P) + q * PC_T + t;
    pv[q] = p < npix;
    const long long pp = pv[q] ? p : 0;
    pb[q] = int(pp / ((long long)Hc * Wc));
    const int rem = int(pp - (long long)pb[q] * Hc * Wc);
    poy[q] = rem / Wc;
    pox[q] = rem - poy[q] * Wc;
    if (par) {
      poy[q] = 2 * poy[q] + py;
      pox[q] = 2 * pox[q] + px;
    }
    pout[q] = ((long long)pb[q] * a.Ho + poy[q]) * a.Wo + pox[q];
    if (!a.xbatch) pb[q] = 0;
  }
  float acc[P][CO];
#pragma unroll
  for (int q = 0; q < P; ++q)
#pragma unroll
    for (int j = 0; j < CO; ++j) acc[q][j] = 0.f;
  for (int ci0 = 0; ci0 < a.cin; ci0 += PC_CI) {
    const int nci = min(PC_CI, a.cin - ci0);
    __syncthreads();
    for (int i = t; i < kk * PC_CI * CO; i += PC_T) {
      const int j = i % CO, cl = (i / CO) % PC_CI, tap = i / (CO * PC_CI);
      sw[i] = (j < nco && cl < nci) ? __ldg(a.w + (size_t(tap) * a.cin + ci0 + cl) * a.cout + co0 + j) : 0.f;
    }
    __syncthreads();
    for (int ky = ky0; ky < a.k; ky += kst)
      for (int i0 = 0; i0 < PC_KMAX; i0 += KB) {
        if (kx0 + i0 * kst >= a.k) break;
        // input offsets of KB taps of this row (element index; -1 = outside / other class)
        long long xo[KB][P];
#pragma unroll
        for (int i = 0; i < KB; ++i) {
          const int kx = kx0 + (i0 + i) * kst;
#pragma unroll
          for (int q = 0; q < P; ++q) {
            int iy, ix;
            bool ok = pv[q] && kx < a.k;
            if (!a.transpose) {
              iy = poy[q] * a.stride + ky - pad;
              ix = pox[q] * a.stride + kx - pad;
            } else {
              iy = poy[q] + pad - ky;
              ix = pox[q] + pad - kx;
              if (a.stride == 2) {
                ok = ok && !((iy | ix) & 1);
                iy >>= 1;
                ix >>= 1;
              }
            }
            ok = ok && iy >= 0 && iy < a.Hin && ix >= 0 && ix < a.Win;
            xo[i][q] = ok ? ((long long)(size_t(pb[q]) * a.Hin + iy) * a.Win + ix) * a.ldx + ci0 : -1;
          }
        }
        if (VEC) {
          for (int c0 = 0; c0 < nci; c0 += 4 * CB) {
            float4 xv[KB][CB][P];
#pragma unroll
            for (int i = 0; i < KB; ++i)
#pragma unroll
              for (int cb = 0; cb < CB; ++cb)
#pragma unroll
                for (int q = 0; q < P; ++q) {
                  const int c4 = c0 + 4 * cb;
                  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                  if (xo[i][q] >= 0 && c4 < nci) v = __ldg(reinterpret_cast<const float4*>(a.x + xo[i][q] + c4));
                  if (a.in_elu) v = make_float4(elu(v.x), elu(v.y), elu(v.z), elu(v.w));
                  xv[i][cb][q] = v;
                }
#pragma unroll
            for (int i = 0; i < KB; ++i) {
              const int kx = kx0 + (i0 + i) * kst;
              if (kx >= a.k) break;
              const float4* wt = sw4 + (size_t(ky * a.k + kx) * PC_CI) * (CO / 4);
#pragma unroll
              for (int cb = 0; cb < CB; ++cb) {
                const int c4 = c0 + 4 * cb;
                if (c4 >= nci) break;
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  const float4* wr = wt + (c4 + u) * (CO / 4);
                  float w[CO];
#pragma unroll
                  for (int j4 = 0; j4 < CO / 4; ++j4) {
                    const float4 v = wr[j4];
                    w[4 * j4] = v.x;
                    w[4 * j4 + 1] = v.y;
                    w[4 * j4 + 2] = v.z;
                    w[4 * j4 + 3] = v.w;
                  }
#pragma unroll
                  for (int q = 0; q < P; ++q) {
                    const float4 xq = xv[i][cb][q];
                    const float xs = u == 0 ? xq.x : u == 1 ? xq.y : u == 2 ? xq.z : xq.w;
#pragma unroll
                    for (int j = 0; j < CO; ++j) acc[q][j] = fmaf(xs, w[j], acc[q][j]);
                  }
                }
              }
            }
          }
        } else {
#pragma unroll
          for (int i = 0; i < KB; ++i) {
            const int kx = kx0 + (i0 + i) * kst;
            if (kx >= a.k) break;
            const float4* wt = sw4 + (size_t(ky * a.k + kx) * PC_CI) * (CO / 4);
            for (int cl = 0; cl < nci; ++cl) {
              const float4* wr = wt + cl * (CO / 4);
              float w[CO];
#pragma unroll
              for (int j4 = 0; j4 < CO / 4; ++j4) {
                const float4 v = wr[j4];
                w[4 * j4] = v.x;
                w[4 * j4 + 1] = v.y;
                w[4 * j4 + 2] = v.z;
                w[4 * j4 + 3] = v.w;
              }
#pragma unroll
              for (int q = 0; q < P; ++q) {
                float xs = xo[i][q] >= 0 ? __ldg(a.x + xo[i][q] + cl) : 0.f;
                if (a.in_elu) xs = elu(xs);
#pragma unroll
                for (int j = 0; j < CO; ++j) acc[q][j] = fmaf(xs, w[j], acc[q][j]);
              }
            }
          }
        }
      }
  }
  // epilogue: bias, residual, batch norm (eval), ELU
#pragma unroll
  for (int q = 0; q < P; ++q) {
    if (!pv[q]) continue;
    const long long p = pout[q];
    float* yp = a.y + size_t(p) * a.ldy + co0;
    const float* rp = a.res ? a.res + size_t(p) * a.ldres + co0 : nullptr;
#pragma unroll
    for (int j = 0; j < CO; ++j) {
      if (j >= nco) break;
      const int co = co0 + j;
      float v = acc[q][j] + a.bias[co];
      if (rp) v = rp[j] + v;
      if (a.mu) v = ((v - a.mu[co]) * a.is[co]) * a.g[co] + a.be[co];
      if (a.act) v = elu(v);
      yp[j] = v;
    }
  }
}

// dst[pix][off + c] = src[pix (mod plane if bcast)][c]
__global__ void k_copy_ch(long long npix, int plane, int bcast, int C, const float* __restrict__ src, int lds,
                          float* __restrict__ dst, int ldd) {
  pdl_enter();
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npix * C) return;
  const long long p = i / C;
  const int c = int(i - p * C);
  const long long ps = bcast ? p % plane : p;
  dst[p * ldd + c] = src[ps * lds + c];
}

// (h^2 Re r, h^2 Im r, kappa^2, gamma) NHWC (inc/precond.hpp:74-90)
__global__ void k_pack4(int N, float h2, const int* act, const float2* __restrict__ r, const float* rscale,
                        const float* __restrict__ k2, const float* __restrict__ gam, float* __restrict__ x) {
  pdl_enter();
  const int b = blockIdx.y;
  if (act && !act[b]) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const float s = (rscale ? rscale[b] : 1.0f) * h2;
  const float2 v = r[size_t(b) * N + i];
  reinterpret_cast<float4*>(x)[size_t(b) * N + i] = make_float4(v.x * s, v.y * s, k2[i], gam[i]);
}

// ------------------------------------------------------------ executor --
struct TView {
  float* p;
  int H, W, C, ld;  // NHWC, ld = floats per pixel
  TView slice(int off, int c) const { return TView{p + off, H, W, c, ld}; }
};

struct Exec {
  Context& c;
  PaperState& P;
  int B;
  bool plan;
  size_t top = 0;
  float* base = nullptr;
  Exec(Context& c_, PaperState& P_, int B_, bool plan_, float* base_) : c(c_), P(P_), B(B_), plan(plan_), base(base_) {}

  TView alloc(int H, int W, int C, int nb) {
    const size_t n = (size_t(nb) * H * W * C + 31) & ~size_t(31);
    TView t{plan ? nullptr : base + top, H, W, C, C};
    top += n;
    return t;
  }
  void conv(const TView& x, const std::string& kname, const TView& y, int stride, bool in_elu, bool act,
            const TView* res, bool xbatch = true, int nb = -1) {
    if (plan) return;
    const DevConv& D = P.dev.at(kname);
    if (D.cin != x.C || D.cout != y.C) throw HbError{HB_ERR_STATE, "paper net channel mismatch at " + kname};
    PConv a{};
    a.x = x.p;
    a.ldx = x.ld;
    a.cin = x.C;
    a.Hin = x.H;
    a.Win = x.W;
    a.y = y.p;
    a.ldy = y.ld;
    a.cout = y.C;
    a.Ho = y.H;
    a.Wo = y.W;
    a.w = D.w.p;
    a.bias = D.bias.p;
    if (D.bn) {
      a.mu = D.mu.p;
      a.is = D.is.p;
      a.g = D.g.p;
      a.be = D.be.p;
    }
    a.res = res ? res->p : nullptr;
    a.ldres = res ? res->ld : 0;
    a.k = D.k;
    a.stride = stride;
    a.transpose = D.transpose;
    a.in_elu = in_elu;
    a.act = act;
    a.B = nb < 0 ? B : nb;
    a.xbatch = xbatch;
    const long long npix = (long long)a.B * a.Ho * a.Wo;
    // the 16 -> 2 output layer: column strips with parameter-space weights
    if (!D.hw.empty() && stride == 1 && !D.bn && !res && !in_elu && !act && xbatch && x.ld == D.cin && y.ld == 2) {
      if (c.prof_detail) c.prof_label = kname;
      if (launch_head_cols(c, D.cin, a.B, y.H, y.W, x.p, D.hw.data(), D.hb.data(), y.p)) return;
    }
    // tensor cores (3xTF32 implicit GEMM, hb_conv_tc.cu) where the layer's
    // channels and dense input allow; the register-tiled SIMT kernel otherwise
    if (!D.tc.empty() && xbatch && x.ld == x.C && (!res || res->ld == y.C) && y.ld % 4 == 0 && c.opt_tc_conv &&
        (!D.transpose || stride == 2)) {
      bool ok = true;
      for (const PaperTc& T : D.tc) {
        TcConv t{};
        t.cw = &T.cw;
        t.B = a.B;
        t.Hin = x.H;
        t.Win = x.W;
        t.H = D.transpose ? x.H : y.H;  // tile grid: the output (class) grid
        t.W = D.transpose ? x.W : y.W;
        t.a = x.p;
        t.ca = x.C;
        t.geo = T.geo;
        t.geo.s = D.transpose ? 1 : stride;
        t.geo.os = D.transpose ? 2 : 1;
        t.geo.Ho = y.H;
        t.geo.Wo = y.W;
        t.geo.ldo = y.ld;
        t.epi = TcEpi{res ? res->p : nullptr, res ? res->ld : 0, D.bn ? T.mu.p : nullptr, T.is.p, T.g.p, T.be.p,
                      act ? 2 : 0, in_elu ? 1 : 0, D.cout};
        t.out = y.p;
        if (c.prof_detail) c.prof_label = kname;
        if (!launch_conv_tc_gen(c, t)) {
          ok = false;
          break;
        }
      }
      if (ok) return;  // (a refused class falls through: the SIMT kernel below rewrites every class)
    }
    const int tok = prof_begin(c, PC_CONV);
    {
      const bool par = a.transpose && a.stride == 2;
      const long long cpix = par ? (npix + 3) / 4 : npix;  // pixels per parity class
      const int CO = a.cout <= 4 ? 4 : 16;  // narrow output layers (the net's 2-channel head)
      const int coblk = (a.cout + CO - 1) / CO;
      // 4 pixels per thread when that still gives >= 2 CTAs per SM, else 1; 1 for
      // few input channels (latency-bound: one pixel with batched tap-row loads
      // beat four at the 4-channel first layer, 151 -> 118 us at batch 128)
      const bool big = a.cin > 4 && (cpix + PC_T * 4 - 1) / (PC_T * 4) * coblk * (par ? 4 : 1) >= 2 * c.num_sms;
      const int P = big ? 4 : 1;
      const dim3 grid(unsigned((cpix + PC_T * P - 1) / (PC_T * P)), unsigned(coblk), par ? 4u : 1u);
      const size_t smem = size_t(D.k) * D.k * PC_CI * CO * sizeof(float);
      const bool vec = a.cin % 4 == 0 && a.ldx % 4 == 0;
      static bool attr = false;
      if (!attr) {
        const int mx = 100 * 1024;
        for (auto k : {k_pconv_tiled<4, true, 16>, k_pconv_tiled<4, false, 16>, k_pconv_tiled<1, true, 16>,
                       k_pconv_tiled<1, false, 16>, k_pconv_tiled<4, true, 4>, k_pconv_tiled<4, false, 4>,
                       k_pconv_tiled<1, true, 4>, k_pconv_tiled<1, false, 4>})
          HB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
        attr = true;
      }
      void (*kern)(PConv) =
          CO == 4 ? (P == 4 ? (vec ? k_pconv_tiled<4, true, 4> : k_pconv_tiled<4, false, 4>)
                            : (vec ? k_pconv_tiled<1, true, 4> : k_pconv_tiled<1, false, 4>))
                  : (P == 4 ? (vec ? k_pconv_tiled<4, true, 16> : k_pconv_tiled<4, false, 16>)
                            : (vec ? k_pconv_tiled<1, true, 16> : k_pconv_tiled<1, false, 16>));
      if (smem > 100 * 1024 || D.k > PC_KMAX)
        launch_pdl(c, k_pconv<16>, dim3(unsigned((npix + 127) / 128)), dim3(128), 0, a);
      else
        launch_pdl(c, kern, dim3(grid), dim3(PC_T), smem, a);
    }
    HB_CUDA(cudaGetLastError());
    const double taps = D.transpose && stride == 2 ? double(D.k) * D.k / 4.0 : double(D.k) * D.k;
    if (c.prof_detail) c.prof_label = kname;
    prof_end(c, PC_CONV, tok, 0, 2.0 * npix * taps * D.cin * D.cout);
  }
  void copy(const TView& src, const TView& dst, bool bcast) {
    if (plan) return;
    const long long npix = (long long)B * dst.H * dst.W;
    const long long n = npix * src.C;
    c.launches++;
    launch_pdl(c, k_copy_ch, dim3(unsigned((n + 255) / 256)), dim3(256), 0, npix, dst.H * dst.W, bcast ? 1 : 0, src.C, src.p,
                                                               src.ld, dst.p, dst.ld);
    HB_CUDA(cudaGetLastError());
  }
  // x <- elu(BN2(x + K2 elu(BN1(K1 x))))  (inc/unet.hpp:150-162)
  TView resnet(const TView& x, const std::string& n, int nb) {
    TView t = alloc(x.H, x.W, x.C, nb), u = alloc(x.H, x.W, x.C, nb);
    conv(x, n + ".k1", t, 1, false, true, nullptr, true, nb);
    conv(t, n + ".k2", u, 1, false, true, &x, true, nb);
    return u;
  }
};

// encoder features (inc/unet.hpp:231-257) over kappa^2 (batch 1)
void run_encoder(Exec& E, const float* k2f, int H, int W, std::vector<TView>& feats) {
  const hb_unet_cfg& c = E.P.cfg;
  TView kin{const_cast<float*>(k2f), H, W, 1, 1};
  TView x = E.alloc(H, W, enc_ch(c, 0), 1);
  E.conv(kin, "enc.entry.k", x, 1, false, true, nullptr, true, 1);
  feats.push_back(x);
  for (int l = 0; l < c.levels; ++l) {
    TView y = E.alloc(H >> (l + 1), W >> (l + 1), enc_ch(c, l + 1), 1);
    E.conv(x, "enc.down" + std::to_string(l) + ".k", y, 2, false, true, nullptr, true, 1);
    x = y;
    for (int r = 0; r < c.resnet_per_level; ++r)
      x = E.resnet(x, "enc.res" + std::to_string(l + 1) + "_" + std::to_string(r), 1);
    feats.push_back(x);
  }
}

// build_unet (inc/unet.hpp:171-226): in NHWC [B][H][W][4] -> out NHWC [B][H][W][2]
void run_solver(Exec& E, const TView& in, const std::vector<TView>& feats, const TView& out) {
  const hb_unet_cfg& c = E.P.cfg;
  const bool es = E.P.variant == 1;
  const std::string pre = es ? "sol." : "unet.";
  std::vector<TView> skips(size_t(c.levels));
  skips[0] = in;
  TView x = in;
  auto cat_feat = [&](const TView& a, int l) {  // tape.concat(x, features[l])
    const TView& f = feats[size_t(l)];
    TView t = E.alloc(a.H, a.W, a.C + f.C, E.B);
    E.copy(a, t.slice(0, a.C), false);
    E.copy(f, t.slice(a.C, f.C), true);
    return t;
  };
  for (int l = 0; l < c.levels; ++l) {
    if (es) x = cat_feat(x, l);
    TView y = E.alloc(x.H / 2, x.W / 2, solver_ch(c, l + 1), E.B);
    E.conv(x, pre + "down" + std::to_string(l) + ".k", y, 2, false, true, nullptr);
    x = y;
    if (l < c.levels - 1) {
      for (int r = 0; r < c.resnet_per_level; ++r)
        x = E.resnet(x, pre + "res" + std::to_string(l + 1) + "_" + std::to_string(r), E.B);
      skips[size_t(l) + 1] = x;
    }
  }
  for (int r = 0; r < c.bottleneck_resnets; ++r) x = E.resnet(x, pre + "bot" + std::to_string(r), E.B);
  for (int s = c.levels; s >= 1; --s) {
    const int t = s - 1;
    if (es) x = cat_feat(x, s);
    const int oc = up_out_ch(c, t);
    const TView& sk = skips[size_t(t)];
    TView y = E.alloc(x.H * 2, x.W * 2, oc + sk.C, E.B);  // [up | skip] (tape.concat, :221)
    E.conv(x, pre + "up" + std::to_string(t) + ".k", y.slice(0, oc), 2, /*in_elu=*/true, /*act=*/false, nullptr);
    E.copy(sk, y.slice(oc, sk.C), false);
    x = y;
  }
  E.conv(x, pre + "out.k", out, 1, false, false, nullptr);
}

PaperState& state(Context& c) {
  if (!c.paper) c.paper = std::make_shared<PaperState>();
  return *c.paper;
}

void ensure_coef(Context& c, PaperState& P) {
  if (P.coef_gen == c.prob_gen) return;
  const size_t n = c.k2.size();
  std::vector<float> k(n), g(n);
  for (size_t i = 0; i < n; ++i) {
    k[i] = float(c.k2[i]);
    g[i] = float(c.gam[i]);
  }
  P.k2f.ensure(n);
  P.gamf.ensure(n);
  HB_CUDA(cudaMemcpy(P.k2f.p, k.data(), n * sizeof(float), cudaMemcpyHostToDevice));
  HB_CUDA(cudaMemcpy(P.gamf.p, g.data(), n * sizeof(float), cudaMemcpyHostToDevice));
  P.coef_gen = c.prob_gen;
  P.feat_gen = ~0ull;
}

// forward of the paper net on device NHWC buffers (in 4ch, out 2ch)
void paper_forward_dev(Context& c, int B, int H, int W, const float* in, float* out) {
  PaperState& P = state(c);
  if (!P.active) throw HbError{HB_ERR_STATE, "paper net not set (hb_set_paper_net)"};
  const int q = 1 << P.cfg.levels;
  if (H % q || W % q) throw HbError{HB_ERR_ARG, "input dims must be divisible by 2^levels"};
  if (P.par4 != c.opt_tconv_par4) {
    P.par4 = c.opt_tconv_par4;
    P.dirty = true;
  }
  if (P.dirty) upload_all(P);
  const bool es = P.variant == 1;
  std::vector<TView> feats;
  if (es) {
    if (!c.has_problem || c.nx != W || c.ny != H)
      throw HbError{HB_ERR_STATE, "encoder_solver needs the problem's kappa^2 at the input size"};
    ensure_coef(c, P);
    // features: persistent buffers, recomputed when the problem or weights change
    Exec plan(c, P, 1, true, nullptr);
    std::vector<TView> fp;
    run_encoder(plan, P.k2f.p, H, W, fp);
    if (P.feat_gen != c.prob_gen || P.feat.size() != fp.size()) {
      P.feat.clear();
      P.feat.resize(fp.size());
      DBuf<float> tmp;
      tmp.ensure(plan.top);
      Exec run(c, P, 1, false, tmp.p);
      std::vector<TView> fr;
      run_encoder(run, P.k2f.p, H, W, fr);
      for (size_t l = 0; l < fr.size(); ++l) {
        const size_t n = size_t(fr[l].H) * fr[l].W * fr[l].C;
        P.feat[l].ensure(n);
        HB_CUDA(cudaMemcpyAsync(P.feat[l].p, fr[l].p, n * sizeof(float), cudaMemcpyDeviceToDevice, c.stream));
      }
      HB_CUDA(cudaStreamSynchronize(c.stream));
      P.feat_gen = c.prob_gen;
    }
    for (size_t l = 0; l < fp.size(); ++l) feats.push_back(TView{P.feat[l].p, fp[l].H, fp[l].W, fp[l].C, fp[l].C});
  }
  const TView tin{const_cast<float*>(in), H, W, 4, 4}, tout{out, H, W, 2, 2};
  Exec plan(c, P, B, true, nullptr);
  run_solver(plan, tin, feats, tout);
  P.arena.ensure(plan.top);
  Exec run(c, P, B, false, P.arena.p);
  run_solver(run, tin, feats, tout);
}

}  // namespace

PaperState& paper_state(Context& c) { return state(c); }
bool paper_active(const Context& c) { return c.paper && c.paper->active; }
void paper_deactivate(Context& c) {
  if (c.paper) c.paper->active = false;
}

// e = net(h^2 r s, kappa^2, gamma) [+ base]  (NetworkApplier::infer_error, inc/precond.hpp:70-90)
void paper_infer(Context& c, int B, const int* act, const float2* r, const float* rscale, const float2* base,
                 float2* e) {
  PaperState& P = state(c);
  ensure_coef(c, P);
  const Level& L = *c.levels[0];
  const int N = int(L.N());
  const size_t np = size_t(B) * N;
  P.io.ensure(np * 6);
  {
    const int tok = prof_begin(c, PC_NETIO);
    launch_pdl(c, k_pack4, dim3((N + 255) / 256, B), dim3(256), 0, N, float(L.h * L.h), act, r, rscale, P.k2f.p, P.gamf.p,
                                                            P.io.p);
    HB_CUDA(cudaGetLastError());
    prof_end(c, PC_NETIO, tok, double(np) * (8 + 16) + double(N) * 8, 0);
  }
  paper_forward_dev(c, B, L.ny, L.nx, P.io.p, P.io.p + np * 4);
  if (base)
    launch_unpack_add(c, N, B, act, P.io.p + np * 4, base, e);
  else
    launch_unpack_output(c, N, B, act, P.io.p + np * 4, e);
}

}  // namespace hb

// ===================================================================== C ABI
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

namespace {
uint32_t get_u32(std::istream& is) {
  unsigned char b[4];
  is.read(reinterpret_cast<char*>(b), 4);
  return uint32_t(b[0]) | uint32_t(b[1]) << 8 | uint32_t(b[2]) << 16 | uint32_t(b[3]) << 24;
}
void put_u32(std::ostream& os, uint32_t v) {
  const unsigned char b[4] = {uint8_t(v), uint8_t(v >> 8), uint8_t(v >> 16), uint8_t(v >> 24)};
  os.write(reinterpret_cast<const char*>(b), 4);
}
}  // namespace

extern "C" {

int hb_set_paper_net(hb_ctx* ctx, const hb_unet_cfg* cfg, int variant) {
  HB_API_BEGIN
  if (!cfg || cfg->levels < 1 || cfg->levels > 8 || cfg->base_channels < 2 || cfg->base_channels % 2 ||
      cfg->resnet_per_level < 0 || cfg->bottleneck_resnets < 0 || cfg->updown_kernel < 1 || cfg->updown_kernel % 2 == 0 ||
      cfg->res_kernel < 1 || cfg->res_kernel % 2 == 0)
    throw HbError{HB_ERR_ARG, "bad UNetConfig"};
  if (variant != 0 && variant != 1) throw HbError{HB_ERR_ARG, "variant: 0 standalone, 1 encoder_solver"};
  PaperState& P = state(*ctx);
  set_layout(P, *cfg, variant);
  init_params(P, 0x5eedULL);  // NetworkWeights default seed (inc/unet.hpp:13)
  P.active = true;
  HB_API_END
}

int hb_paper_init(hb_ctx* ctx, uint64_t seed) {
  HB_API_BEGIN
  PaperState& P = state(*ctx);
  if (!P.active) throw HbError{HB_ERR_STATE, "paper net not set"};
  init_params(P, seed);
  P.dirty = true;
  ++P.host_gen;
  P.feat_gen = ~0ull;
  HB_API_END
}

int hb_paper_param_count(hb_ctx* ctx) { return ctx && ctx->paper ? int(ctx->paper->params.size()) : 0; }

int hb_paper_param_info(hb_ctx* ctx, int i, char* name, int cap, int* dims) {
  HB_API_BEGIN
  PaperState& P = state(*ctx);
  if (i < 0 || i >= int(P.params.size())) throw HbError{HB_ERR_ARG, "parameter index out of range"};
  const PParam& q = P.params[size_t(i)];
  if (name && cap > 0) {
    const size_t n = std::min(q.name.size(), size_t(cap - 1));
    std::memcpy(name, q.name.data(), n);
    name[n] = 0;
  }
  if (dims)
    for (int k = 0; k < 4; ++k) dims[k] = q.d[k];
  HB_API_END
}

int hb_paper_param(hb_ctx* ctx, const char* name, int64_t count, const float* in, float* out) {
  HB_API_BEGIN
  if (!name) throw HbError{HB_ERR_ARG, "null name"};
  PaperState& P = state(*ctx);
  PParam& q = param(P, name);
  if (count != int64_t(q.v.size()))
    throw HbError{HB_ERR_ARG, "parameter " + std::string(name) + " dims changed"};
  if (out) std::memcpy(out, q.v.data(), q.v.size() * sizeof(float));
  if (in) {
    std::memcpy(q.v.data(), in, q.v.size() * sizeof(float));
    P.dirty = true;
  ++P.host_gen;
    P.feat_gen = ~0ull;
  }
  HB_API_END
}

// UNW1 (inc/checkpoint.hpp:12-104): records by name into the registry (adam.* skipped)
int hb_load_checkpoint(hb_ctx* ctx, const char* path) {
  HB_API_BEGIN
  PaperState& P = state(*ctx);
  if (!P.active) throw HbError{HB_ERR_STATE, "set the paper net (hb_set_paper_net) before loading weights"};
  std::ifstream is(path ? path : "", std::ios::binary);
  if (!is) throw HbError{HB_ERR_ARG, std::string("cannot open checkpoint: ") + (path ? path : "")};
  char magic[4];
  is.read(magic, 4);
  if (!is || std::memcmp(magic, "UNW1", 4) != 0) throw HbError{HB_ERR_NUMERIC, "bad checkpoint magic"};
  if (get_u32(is) != 1) throw HbError{HB_ERR_NUMERIC, "unsupported checkpoint version"};
  const uint32_t dl = get_u32(is);
  if (dl > 4096) throw HbError{HB_ERR_NUMERIC, "bad checkpoint digest"};
  is.ignore(dl);
  const uint32_t count = get_u32(is);
  std::vector<bool> seen(P.params.size(), false);
  for (uint32_t r = 0; r < count; ++r) {
    const uint32_t nl = get_u32(is);
    if (nl > 4096) throw HbError{HB_ERR_NUMERIC, "checkpoint record name too long"};
    std::string name(nl, '\0');
    is.read(name.data(), nl);
    const int dtype = is.get(), rank = is.get();
    if (dtype != 0 || rank != 4) throw HbError{HB_ERR_NUMERIC, "unsupported checkpoint record"};
    int d[4];
    for (int k = 0; k < 4; ++k) d[k] = int(get_u32(is));
    const size_t n = size_t(d[0]) * d[1] * d[2] * d[3];
    if (d[0] <= 0 || d[1] <= 0 || d[2] <= 0 || d[3] <= 0 || n > (size_t(1) << 28))
      throw HbError{HB_ERR_NUMERIC, "bad checkpoint record dims"};
    std::vector<float> v(n);
    is.read(reinterpret_cast<char*>(v.data()), std::streamsize(n * 4));  // f32 LE (x86)
    if (!is) throw HbError{HB_ERR_NUMERIC, "truncated checkpoint"};
    if (name.rfind("adam.", 0) == 0) continue;
    auto it = P.index.find(name);
    if (it == P.index.end()) throw HbError{HB_ERR_ARG, "checkpoint parameter " + name + " not in this UNetConfig"};
    PParam& q = P.params[it->second];
    if (std::memcmp(q.d, d, sizeof d) != 0) throw HbError{HB_ERR_ARG, "parameter " + name + " dims changed"};
    q.v = std::move(v);
    seen[it->second] = true;
  }
  P.dirty = true;
  ++P.host_gen;
  P.feat_gen = ~0ull;
  HB_API_END
}

int hb_save_checkpoint(hb_ctx* ctx, const char* path, const char* digest) {
  HB_API_BEGIN
  PaperState& P = state(*ctx);
  if (!P.active) throw HbError{HB_ERR_STATE, "paper net not set"};
  std::ofstream os(path ? path : "", std::ios::binary);
  if (!os) throw HbError{HB_ERR_ARG, "cannot write checkpoint"};
  const std::string dg = digest ? digest : "";
  os.write("UNW1", 4);
  put_u32(os, 1);
  put_u32(os, uint32_t(dg.size()));
  os.write(dg.data(), std::streamsize(dg.size()));
  put_u32(os, uint32_t(P.params.size()));
  for (const auto& q : P.params) {
    put_u32(os, uint32_t(q.name.size()));
    os.write(q.name.data(), std::streamsize(q.name.size()));
    os.put(char(0));
    os.put(char(4));
    for (int k = 0; k < 4; ++k) put_u32(os, uint32_t(q.d[k]));
    os.write(reinterpret_cast<const char*>(q.v.data()), std::streamsize(q.v.size() * 4));
  }
  if (!os) throw HbError{HB_ERR_ARG, "checkpoint write failed"};
  HB_API_END
}

// in: NCHW [B][4][H][W] fp32 host -> out NCHW [B][2][H][W] (unet_forward / solver_forward, eval)
int hb_paper_forward(hb_ctx* ctx, int batch, int H, int W, const float* in, float* out) {
  HB_API_BEGIN
  if (!in || !out || batch < 1) throw HbError{HB_ERR_ARG, "bad buffers"};
  const size_t px = size_t(batch) * H * W;
  std::vector<float> a(px * 4), y(px * 2);
  for (int b = 0; b < batch; ++b)
    for (int c = 0; c < 4; ++c)
      for (size_t i = 0; i < size_t(H) * W; ++i) a[(size_t(b) * H * W + i) * 4 + c] = in[(size_t(b) * 4 + c) * H * W + i];
  DBuf<float> d;
  d.ensure(px * 6);
  HB_CUDA(cudaMemcpyAsync(d.p, a.data(), px * 4 * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
  paper_forward_dev(*ctx, batch, H, W, d.p, d.p + px * 4);
  HB_CUDA(cudaMemcpyAsync(y.data(), d.p + px * 4, px * 2 * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
  HB_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int b = 0; b < batch; ++b)
    for (int c = 0; c < 2; ++c)
      for (size_t i = 0; i < size_t(H) * W; ++i) out[(size_t(b) * 2 + c) * H * W + i] = y[(size_t(b) * H * W + i) * 2 + c];
  HB_API_END
}

}  // extern "C"
