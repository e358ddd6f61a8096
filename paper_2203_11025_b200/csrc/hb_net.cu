// Classic U-Net / encoder forward on sm_100a.
//
// Activations are NHWC fp32 so a 3x3 convolution is an implicit GEMM with
// M = pixels, N = C_out, K = 9*C_in (taps outer, channels inner).  Channel
// concatenation [a | b] (inc/autodiff.hpp:403) is never materialised: the
// conv reads K from two sources.  The encoder context maps are broadcast over
// the batch (tile_batch, inc/tensor.hpp:81) by a zero batch stride.
//
// Conv kernel (this file): CTA tile 128 pixels x 32 output channels, K in
// chunks of 8 input channels x 9 taps staged in shared memory, 4x4 register
// micro-tile, fp32 FFMA with fused bias + ReLU.
#include <cmath>
#include <cstring>
#include <vector>

#include "hb_common.cuh"
#include "hb_host.h"
#include "hb_internal.h"

namespace hb {

namespace {

constexpr int CT_H = 8, CT_W = 16, CT_CO = 32, CT_CI = 8;
constexpr int PH = CT_H + 2, PW = CT_W + 2;

struct ConvArgs {
  int B, H, W;
  const float* a;  // NHWC, ca channels
  long long sa;    // batch stride of a (elements)
  int ca;
  const float* b;  // NHWC, cb channels (may be null)
  long long sb;    // batch stride of b (0 = broadcast)
  int cb;
  const float* w;  // packed [(tap*cin + ci)][cout]
  const float* bias;
  int cout;
  int relu;
  float* out;  // NHWC cout
  const int* act;
  const float* pre = nullptr;  // per-pixel [H][W][cout] term replacing the bias, batch-broadcast (k_conv_small_pw)
};

__global__ void __launch_bounds__(256) k_conv3x3(ConvArgs p) {
  pdl_enter();
  const int bz = blockIdx.z;
  if (p.act && !p.act[bz]) return;
  __shared__ float patch[PH * PW][CT_CI + 1];
  __shared__ __align__(16) float wts[9][CT_CI][CT_CO];
  const int tilesW = (p.W + CT_W - 1) / CT_W;
  const int y0 = (blockIdx.x / tilesW) * CT_H, x0 = (blockIdx.x % tilesW) * CT_W;
  const int co0 = blockIdx.y * CT_CO;
  const int t = threadIdx.x;
  const int cg = t % (CT_CO / 4), pg = t / (CT_CO / 4);
  const int prow = pg / (CT_W / 4), pcol = (pg % (CT_W / 4)) * 4;
  const int cin = p.ca + p.cb;
  float acc[4][4];
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int r = 0; r < 4; ++r) acc[q][r] = 0.f;
  const float* A = p.a + bz * p.sa;
  const float* Bsrc = p.b ? p.b + bz * p.sb : nullptr;
  for (int ci0 = 0; ci0 < cin; ci0 += CT_CI) {
    for (int idx = t; idx < PH * PW * CT_CI; idx += 256) {
      const int c = idx % CT_CI, pix = idx / CT_CI;
      const int gy = y0 + pix / PW - 1, gx = x0 + pix % PW - 1;
      const int ci = ci0 + c;
      float v = 0.f;
      if (gy >= 0 && gy < p.H && gx >= 0 && gx < p.W && ci < cin) {
        const size_t px = size_t(gy) * p.W + gx;
        v = ci < p.ca ? __ldg(A + px * p.ca + ci) : __ldg(Bsrc + px * p.cb + (ci - p.ca));
      }
      patch[pix][c] = v;
    }
    for (int idx = t; idx < 9 * CT_CI * CT_CO; idx += 256) {
      const int col = idx % CT_CO, rest = idx / CT_CO;
      const int cl = rest % CT_CI, tap = rest / CT_CI;
      const int ci = ci0 + cl, co = co0 + col;
      wts[tap][cl][col] = (ci < cin && co < p.cout) ? __ldg(p.w + (size_t(tap) * cin + ci) * p.cout + co) : 0.f;
    }
    __syncthreads();
#pragma unroll 2
    for (int c = 0; c < CT_CI; ++c) {
#pragma unroll
      for (int ky = 0; ky < 3; ++ky)
#pragma unroll
        for (int kx = 0; kx < 3; ++kx) {
          const float4 w4 = *reinterpret_cast<const float4*>(&wts[ky * 3 + kx][c][cg * 4]);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float v = patch[(prow + ky) * PW + pcol + q + kx][c];
            acc[q][0] = fmaf(v, w4.x, acc[q][0]);
            acc[q][1] = fmaf(v, w4.y, acc[q][1]);
            acc[q][2] = fmaf(v, w4.z, acc[q][2]);
            acc[q][3] = fmaf(v, w4.w, acc[q][3]);
          }
        }
    }
    __syncthreads();
  }
  const int y = y0 + prow;
  if (y >= p.H) return;
  float* O = p.out + size_t(bz) * p.H * p.W * p.cout;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int x = x0 + pcol + q;
    if (x >= p.W) continue;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int co = co0 + cg * 4 + r;
      if (co >= p.cout) continue;
      float v = acc[q][r] + __ldg(p.bias + co);
      if (p.relu) v = fmaxf(v, 0.f);
      O[(size_t(y) * p.W + x) * p.cout + co] = v;
    }
  }
}

// Narrow convolutions the tensor-core path does not take -- the 3-channel input
// layer (3 [+ ctx] -> 16) and the 16 -> 2 head.  A 32 x 8 output tile per
// CTA, CS_PX consecutive pixels x COUT outputs per thread (broadcast float4
// weight loads); the (8+2) x (32+2) x Cin input tile and all
// weights sit in shared memory (pixel stride Cin|1 words).
constexpr int CS_TW = 32, CS_TH = 8, CS_PX = 1, CS_NT = CS_TW * CS_TH / CS_PX;

template <int COUT>
__global__ void __launch_bounds__(CS_NT) k_conv_small(ConvArgs p) {
  pdl_enter();
  extern __shared__ __align__(16) float cs_sm[];
  const int bz = blockIdx.z;
  if (p.act && !p.act[bz]) return;
  const int cin = p.ca + p.cb, cp = cin | 1;
  float* wts = cs_sm;                                  // [9][cin][COUT]
  float* tile = cs_sm + ((9 * cin * COUT + 3) & ~3);   // [(TH+2)(TW+2)][cp]
  const int tilesW = (p.W + CS_TW - 1) / CS_TW;
  const int y0 = (blockIdx.x / tilesW) * CS_TH, x0 = (blockIdx.x % tilesW) * CS_TW;
  const int t = threadIdx.x;
  for (int i = t; i < 9 * cin * COUT; i += CS_NT) wts[i] = __ldg(p.w + i);
  const float* A = p.a + bz * p.sa;
  const float* Bsrc = p.b ? p.b + bz * p.sb : nullptr;
  const int npix = (CS_TH + 2) * (CS_TW + 2);
  // thread per halo-tile pixel: its Cin channels are contiguous (float4 when
  // possible); no per-element index division
  for (int pix = t; pix < npix; pix += CS_NT) {
    const int gy = y0 + pix / (CS_TW + 2) - 1, gx = x0 + pix % (CS_TW + 2) - 1;
    float* dst = tile + pix * cp;
    if (gy >= 0 && gy < p.H && gx >= 0 && gx < p.W) {
      const size_t px = size_t(gy) * p.W + gx;
      const float* sa = A + px * p.ca;
      if ((p.ca & 3) == 0) {
        for (int c = 0; c < p.ca; c += 4) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(sa + c));
          dst[c] = v.x;
          dst[c + 1] = v.y;
          dst[c + 2] = v.z;
          dst[c + 3] = v.w;
        }
      } else {
        for (int c = 0; c < p.ca; ++c) dst[c] = __ldg(sa + c);
      }
      if (p.cb) {
        const float* sb = Bsrc + px * p.cb;
        for (int c = 0; c < p.cb; ++c) dst[p.ca + c] = __ldg(sb + c);
      }
    } else {
      for (int c = 0; c < cin; ++c) dst[c] = 0.f;
    }
  }
  __syncthreads();
  const int ty = t / (CS_TW / CS_PX), tx = (t % (CS_TW / CS_PX)) * CS_PX;
  float acc[CS_PX][COUT];
#pragma unroll
  for (int q = 0; q < CS_PX; ++q)
#pragma unroll
    for (int co = 0; co < COUT; ++co) acc[q][co] = 0.f;
  for (int ky = 0; ky < 3; ++ky) {
    const float* rp = tile + ((ty + ky) * (CS_TW + 2) + tx) * cp;
    for (int ci = 0; ci < cin; ++ci) {
      float v[CS_PX + 2];
#pragma unroll
      for (int j = 0; j < CS_PX + 2; ++j) v[j] = rp[j * cp + ci];
#pragma unroll
      for (int kx = 0; kx < 3; ++kx) {
        const float* wp = wts + ((ky * 3 + kx) * cin + ci) * COUT;
        if constexpr (COUT % 4 == 0) {
#pragma unroll
          for (int c4 = 0; c4 < COUT; c4 += 4) {
            const float4 w = *reinterpret_cast<const float4*>(wp + c4);
#pragma unroll
            for (int q = 0; q < CS_PX; ++q) {
              acc[q][c4] = fmaf(v[q + kx], w.x, acc[q][c4]);
              acc[q][c4 + 1] = fmaf(v[q + kx], w.y, acc[q][c4 + 1]);
              acc[q][c4 + 2] = fmaf(v[q + kx], w.z, acc[q][c4 + 2]);
              acc[q][c4 + 3] = fmaf(v[q + kx], w.w, acc[q][c4 + 3]);
            }
          }
        } else {
#pragma unroll
          for (int co = 0; co < COUT; ++co) {
            const float w = wp[co];
#pragma unroll
            for (int q = 0; q < CS_PX; ++q) acc[q][co] = fmaf(v[q + kx], w, acc[q][co]);
          }
        }
      }
    }
  }
  const int y = y0 + ty;
  if (y >= p.H) return;
#pragma unroll
  for (int q = 0; q < CS_PX; ++q) {
    const int x = x0 + tx + q;
    if (x >= p.W) continue;
    float* O = p.out + ((size_t(bz) * p.H + y) * p.W + x) * COUT;
    float r[COUT];
#pragma unroll
    for (int co = 0; co < COUT; ++co) {
      r[co] = acc[q][co] + __ldg(p.bias + co);
      if (p.relu) r[co] = fmaxf(r[co], 0.f);
    }
    if constexpr (COUT % 4 == 0) {
#pragma unroll
      for (int co = 0; co < COUT; co += 4)
        *reinterpret_cast<float4*>(O + co) = make_float4(r[co], r[co + 1], r[co + 2], r[co + 3]);
    } else {
#pragma unroll
      for (int co = 0; co < COUT; ++co) O[co] = r[co];
    }
  }
}

// The same narrow convolution with the weights and bias passed by value in
// the kernel parameter space (up to 32 KB on sm_70+): fully unrolled over
// (ky, ci, kx, co), every weight is a compile-time constant-bank operand of its
// FFMA, so the inner loop issues no weight loads (the smem-weight kernel above
// spends ~2 LDS per FFMA and ran at 11-19 TFLOP/s).  Weight changes bump
// g_alloc_gen (net_upload), which drops captured graphs holding old values.
template <int CIN, int COUT>
struct SmallW {
  float w[9 * CIN * COUT];  // [(ky*3 + kx)][ci][co]
  float b[COUT];
};

template <int CIN, int COUT>
__global__ void __launch_bounds__(CS_NT) k_conv_small_pw(ConvArgs p, const __grid_constant__ SmallW<CIN, COUT> wt) {
  pdl_enter();
  extern __shared__ __align__(16) float cs_sm[];
  const int bz = blockIdx.z;
  if (p.act && !p.act[bz]) return;
  constexpr int cp = CIN | 1;
  float* tile = cs_sm;  // [(TH+2)(TW+2)][cp]
  const int tilesW = (p.W + CS_TW - 1) / CS_TW;
  const int y0 = (blockIdx.x / tilesW) * CS_TH, x0 = (blockIdx.x % tilesW) * CS_TW;
  const int t = threadIdx.x;
  const float* A = p.a + bz * p.sa;
  const float* Bsrc = p.b ? p.b + bz * p.sb : nullptr;
  constexpr int npix = (CS_TH + 2) * (CS_TW + 2);
  for (int pix = t; pix < npix; pix += CS_NT) {
    const int gy = y0 + pix / (CS_TW + 2) - 1, gx = x0 + pix % (CS_TW + 2) - 1;
    float* dst = tile + pix * cp;
    if (gy >= 0 && gy < p.H && gx >= 0 && gx < p.W) {
      const size_t px = size_t(gy) * p.W + gx;
      const float* sa = A + px * p.ca;
      if ((p.ca & 3) == 0) {
        for (int c = 0; c < p.ca; c += 4) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(sa + c));
          dst[c] = v.x;
          dst[c + 1] = v.y;
          dst[c + 2] = v.z;
          dst[c + 3] = v.w;
        }
      } else {
        for (int c = 0; c < p.ca; ++c) dst[c] = __ldg(sa + c);
      }
      if (p.cb) {
        const float* sb = Bsrc + px * p.cb;
        for (int c = 0; c < p.cb; ++c) dst[p.ca + c] = __ldg(sb + c);
      }
    } else {
#pragma unroll
      for (int c = 0; c < CIN; ++c) dst[c] = 0.f;
    }
  }
  __syncthreads();
  const int ty = t / CS_TW, tx = t % CS_TW;
  float acc[COUT];
  if (p.pre) {  // batch-broadcast per-pixel term (the context channels' share, bias included)
    const int yq = min(y0 + ty, p.H - 1), xq = min(x0 + tx, p.W - 1);
    const float* pp = p.pre + (size_t(yq) * p.W + xq) * COUT;
    if constexpr (COUT % 4 == 0) {
#pragma unroll
      for (int co = 0; co < COUT; co += 4) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(pp + co));
        acc[co] = v.x;
        acc[co + 1] = v.y;
        acc[co + 2] = v.z;
        acc[co + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int co = 0; co < COUT; ++co) acc[co] = __ldg(pp + co);
    }
  } else {
#pragma unroll
    for (int co = 0; co < COUT; ++co) acc[co] = wt.b[co];
  }
#pragma unroll
  for (int ky = 0; ky < 3; ++ky) {
    const float* rp = tile + ((ty + ky) * (CS_TW + 2) + tx) * cp;
#pragma unroll
    for (int ci = 0; ci < CIN; ++ci) {
      const float v0 = rp[ci], v1 = rp[cp + ci], v2 = rp[2 * cp + ci];
#pragma unroll
      for (int co = 0; co < COUT; ++co) {
        acc[co] = fmaf(v0, wt.w[((ky * 3 + 0) * CIN + ci) * COUT + co], acc[co]);
        acc[co] = fmaf(v1, wt.w[((ky * 3 + 1) * CIN + ci) * COUT + co], acc[co]);
        acc[co] = fmaf(v2, wt.w[((ky * 3 + 2) * CIN + ci) * COUT + co], acc[co]);
      }
    }
  }
  const int y = y0 + ty, x = x0 + tx;
  if (y >= p.H || x >= p.W) return;
  float* O = p.out + ((size_t(bz) * p.H + y) * p.W + x) * COUT;
  float r[COUT];
#pragma unroll
  for (int co = 0; co < COUT; ++co) r[co] = p.relu ? fmaxf(acc[co], 0.f) : acc[co];
  if constexpr (COUT % 4 == 0) {
#pragma unroll
    for (int co = 0; co < COUT; co += 4)
      *reinterpret_cast<float4*>(O + co) = make_float4(r[co], r[co + 1], r[co + 2], r[co + 3]);
  } else {
#pragma unroll
    for (int co = 0; co < COUT; ++co) O[co] = r[co];
  }
}

template <int CIN, int COUT>
bool conv_small_pw(Context& c, const ConvW& cw, const ConvArgs& p, dim3 g) {
  if (cw.cin != CIN || cw.cout != COUT) return false;
  SmallW<CIN, COUT> wt;
  for (int co = 0; co < COUT; ++co) {
    wt.b[co] = cw.b[size_t(co)];
    for (int ci = 0; ci < CIN; ++ci)
      for (int tap = 0; tap < 9; ++tap) wt.w[(tap * CIN + ci) * COUT + co] = cw.w[(size_t(co) * CIN + ci) * 9 + tap];
  }
  const size_t smem = size_t(CS_TH + 2) * (CS_TW + 2) * size_t(CIN | 1) * sizeof(float);
  launch_pdl(c, k_conv_small_pw<CIN, COUT>, dim3(g), dim3(CS_NT), smem, p, wt);
  return true;
}

// Narrow-output head (Cin % 4 == 0 -> COUT <= 2, e.g. the U-Net's 16 -> 2):
// one thread per output column, CC_R output rows slid down the column.  Input
// rows stream through a CC_NS-slot shared-memory ring filled by coalesced
// 16-byte cp.async (zero-filled outside the grid), pixel stride Cin + 4 words so
// the per-thread float4 reads of 3 neighbouring pixels are conflict-free.  Each
// input row is read once and feeds up to 3 output rows; no per-element halo
// logic.  (Reading the rows straight from global memory instead spread every
// 16-byte load over 32 L1 sectors and ran L1-bound.)  The accumulation order per
// output (ky, ci, kx) is the tiled kernel's, so both give identical bits.
constexpr int CC_NS = 4, CC_TW = 128;  // CC_R (rows per strip): 16, or 4 for grids that would not fill the SMs

__device__ __forceinline__ void cc_cp16(float* dst, const float* src, bool ok) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(src), "r"(ok ? 16 : 0) : "memory");
}

template <int CIN, int COUT, int CC_R>
__global__ void __launch_bounds__(CC_TW) k_conv_cols(ConvArgs p, const __grid_constant__ SmallW<CIN, COUT> wt) {
  static_assert(CIN % 4 == 0, "float4 rows");
  constexpr int PS = CIN + 4, SEG = CC_TW + 2, NCH = SEG * (CIN / 4);
  extern __shared__ __align__(16) float cc_sm[];  // [CC_NS][SEG][PS]
  pdl_enter();
  const int bz = blockIdx.z;
  if (p.act && !p.act[bz]) return;
  const int t = threadIdx.x, x0 = blockIdx.x * CC_TW, y0 = blockIdx.y * CC_R;
  const float* A = p.a + bz * p.sa;
  auto issue = [&](int r) {  // input row y0 + r - 1 -> slot r % CC_NS
    const int y = y0 + r - 1;
    const bool rok = r < CC_R + 2 && y >= 0 && y < p.H;
    float* slot = cc_sm + (r % CC_NS) * SEG * PS;
    for (int i = t; i < NCH; i += CC_TW) {
      const int px = i / (CIN / 4), c4 = i % (CIN / 4), x = x0 - 1 + px;
      const bool ok = rok && x >= 0 && x < p.W;
      cc_cp16(slot + px * PS + 4 * c4, ok ? A + (size_t(y) * p.W + x) * CIN + 4 * c4 : A, ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  float acc[CC_R][COUT];
#pragma unroll
  for (int o = 0; o < CC_R; ++o)
#pragma unroll
    for (int co = 0; co < COUT; ++co) acc[o][co] = wt.b[co];
#pragma unroll
  for (int r = 0; r < CC_NS - 1; ++r) issue(r);
#pragma unroll
  for (int r = 0; r < CC_R + 2; ++r) {
    asm volatile("cp.async.wait_group %0;" ::"n"(CC_NS - 2) : "memory");
    __syncthreads();  // row r visible to all; slot (r - 1) % CC_NS released by all
    issue(r + CC_NS - 1);
    const float* rp = cc_sm + (r % CC_NS) * SEG * PS + t * PS;
#pragma unroll
    for (int c4 = 0; c4 < CIN / 4; ++c4) {
      float4 v[3];
#pragma unroll
      for (int kx = 0; kx < 3; ++kx) v[kx] = *reinterpret_cast<const float4*>(rp + kx * PS + 4 * c4);
#pragma unroll
      for (int ky = 0; ky < 3; ++ky) {
        const int o = r - ky;  // input row y0 + r - 1 is tap ky of output row y0 + o
        if (o < 0 || o >= CC_R) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int ci = 4 * c4 + j;
#pragma unroll
          for (int co = 0; co < COUT; ++co) {
            const float a0 = j == 0 ? v[0].x : j == 1 ? v[0].y : j == 2 ? v[0].z : v[0].w;
            const float a1 = j == 0 ? v[1].x : j == 1 ? v[1].y : j == 2 ? v[1].z : v[1].w;
            const float a2 = j == 0 ? v[2].x : j == 1 ? v[2].y : j == 2 ? v[2].z : v[2].w;
            acc[o][co] = fmaf(a0, wt.w[((ky * 3 + 0) * CIN + ci) * COUT + co], acc[o][co]);
            acc[o][co] = fmaf(a1, wt.w[((ky * 3 + 1) * CIN + ci) * COUT + co], acc[o][co]);
            acc[o][co] = fmaf(a2, wt.w[((ky * 3 + 2) * CIN + ci) * COUT + co], acc[o][co]);
          }
        }
      }
    }
  }
  const int x = x0 + t;
  if (x >= p.W) return;
#pragma unroll
  for (int o = 0; o < CC_R; ++o) {
    const int y = y0 + o;
    if (y >= p.H) break;
    float* O = p.out + ((size_t(bz) * p.H + y) * p.W + x) * COUT;
    float r[COUT];
#pragma unroll
    for (int co = 0; co < COUT; ++co) r[co] = p.relu ? fmaxf(acc[o][co], 0.f) : acc[o][co];
    if constexpr (COUT == 2) {
      *reinterpret_cast<float2*>(O) = make_float2(r[0], r[1]);
    } else {
#pragma unroll
      for (int co = 0; co < COUT; ++co) O[co] = r[co];
    }
  }
}

template <int CIN, int COUT>
void conv_cols_launch(Context& c, const ConvArgs& p, const SmallW<CIN, COUT>& wt);

template <int CIN, int COUT>
bool conv_cols(Context& c, const ConvW& cw, const ConvArgs& p) {
  if (cw.cin != CIN || cw.cout != COUT || p.ca != CIN || p.cb != 0) return false;
  SmallW<CIN, COUT> wt;
  for (int co = 0; co < COUT; ++co) {
    wt.b[co] = cw.b[size_t(co)];
    for (int ci = 0; ci < CIN; ++ci)
      for (int tap = 0; tap < 9; ++tap) wt.w[(tap * CIN + ci) * COUT + co] = cw.w[(size_t(co) * CIN + ci) * 9 + tap];
  }
  conv_cols_launch(c, p, wt);
  return true;
}

template <int CIN, int COUT>
void conv_cols_launch(Context& c, const ConvArgs& p, const SmallW<CIN, COUT>& wt) {
  constexpr size_t smem = size_t(CC_NS) * (CC_TW + 2) * (CIN + 4) * sizeof(float);
  static bool attr = false;
  if (!attr) {
    HB_CUDA(cudaFuncSetAttribute(k_conv_cols<CIN, COUT, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    HB_CUDA(cudaFuncSetAttribute(k_conv_cols<CIN, COUT, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    attr = true;
  }
  const int strips = (p.W + CC_TW - 1) / CC_TW;
  if (strips * ((p.H + 15) / 16) * p.B >= 2 * c.num_sms)
    launch_pdl(c, k_conv_cols<CIN, COUT, 16>, dim3(strips, (p.H + 15) / 16, p.B), dim3(CC_TW), smem, p, wt);
  else  // small grids (c4's 512^2 coarse U-Net at B = 1): shorter strips, more CTAs
    launch_pdl(c, k_conv_cols<CIN, COUT, 4>, dim3(strips, (p.H + 3) / 4, p.B), dim3(CC_TW), smem, p, wt);
}

// 2x2 max-pool / x2 bilinear upsample, NHWC, 4 channels per thread (C % 4 == 0);
// one CTA per output row (grid (rows, B)), threads stride along the row
__global__ void __launch_bounds__(256) k_maxpool2_v4(int H, int W, int C4, const float4* __restrict__ in,
                                                     float4* __restrict__ out, const int* act) {
  pdl_enter();
  const int b = blockIdx.y, oy = blockIdx.x;
  if (act && !act[b]) return;
  const int Wo = W / 2, n = Wo * C4;
  const float4* s0 = in + (size_t(b) * H + 2 * oy) * W * C4;
  const float4* s1 = s0 + size_t(W) * C4;
  float4* o = out + (size_t(b) * (H / 2) + oy) * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int ox = i / C4, c = i - ox * C4;
    const int k = 2 * ox * C4 + c;
    const float4 a0 = __ldg(s0 + k), a1 = __ldg(s0 + k + C4), a2 = __ldg(s1 + k), a3 = __ldg(s1 + k + C4);
    float4 m;
    m.x = fmaxf(fmaxf(a0.x, a1.x), fmaxf(a2.x, a3.x));
    m.y = fmaxf(fmaxf(a0.y, a1.y), fmaxf(a2.y, a3.y));
    m.z = fmaxf(fmaxf(a0.z, a1.z), fmaxf(a2.z, a3.z));
    m.w = fmaxf(fmaxf(a0.w, a1.w), fmaxf(a2.w, a3.w));
    o[i] = m;
  }
}

__global__ void k_maxpool2(int B, int H, int W, int C, const float* __restrict__ in, float* __restrict__ out,
                           const int* act) {
  pdl_enter();
  const int Ho = H / 2, Wo = W / 2;
  const size_t total = size_t(Ho) * Wo * C;
  const int b = blockIdx.y;
  if (act && !act[b]) return;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += size_t(gridDim.x) * blockDim.x) {
    const int c = int(i % C);
    const size_t px = i / C;
    const int x = int(px % Wo), y = int(px / Wo);
    const float* s = in + size_t(b) * H * W * C;
    const float a0 = s[(size_t(2 * y) * W + 2 * x) * C + c], a1 = s[(size_t(2 * y) * W + 2 * x + 1) * C + c];
    const float a2 = s[(size_t(2 * y + 1) * W + 2 * x) * C + c], a3 = s[(size_t(2 * y + 1) * W + 2 * x + 1) * C + c];
    out[size_t(b) * Ho * Wo * C + i] = fmaxf(fmaxf(a0, a1), fmaxf(a2, a3));
  }
}

// x2 bilinear, half-pixel centres, clamped edges (inc/datagen.hpp:19-37 weights)
__device__ __forceinline__ void up_taps(int o, int n, int* i0, int* i1, float* f) {
  const float s = (o + 0.5f) * 0.5f - 0.5f;
  int a = int(floorf(s));
  a = a < 0 ? 0 : (a > n - 1 ? n - 1 : a);
  *i0 = a;
  *i1 = a + 1 < n - 1 ? a + 1 : n - 1;
  float fr = s - float(a);
  *f = fr < 0.f ? 0.f : (fr > 1.f ? 1.f : fr);
}

__global__ void k_upsample2(int B, int H, int W, int C, const float* __restrict__ in, long long sin_,
                            float* __restrict__ out, const int* act) {
  pdl_enter();
  const int Ho = 2 * H, Wo = 2 * W;
  const size_t total = size_t(Ho) * Wo * C;
  const int b = blockIdx.y;
  if (act && !act[b]) return;
  const float* s = in + b * sin_;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += size_t(gridDim.x) * blockDim.x) {
    const int c = int(i % C);
    const size_t px = i / C;
    const int ox = int(px % Wo), oy = int(px / Wo);
    int y0, y1, x0, x1;
    float fy, fx;
    up_taps(oy, H, &y0, &y1, &fy);
    up_taps(ox, W, &x0, &x1, &fx);
    const float v00 = s[(size_t(y0) * W + x0) * C + c], v01 = s[(size_t(y0) * W + x1) * C + c];
    const float v10 = s[(size_t(y1) * W + x0) * C + c], v11 = s[(size_t(y1) * W + x1) * C + c];
    out[size_t(b) * total + i] = (1.f - fy) * ((1.f - fx) * v00 + fx * v01) + fy * ((1.f - fx) * v10 + fx * v11);
  }
}

__global__ void __launch_bounds__(256) k_upsample2_v4(int H, int W, int C4, const float4* __restrict__ in,
                                                      long long sin4, float4* __restrict__ out, const int* act) {
  pdl_enter();
  const int b = blockIdx.y, oy = blockIdx.x;
  if (act && !act[b]) return;
  const int Wo = 2 * W, n = Wo * C4;
  int y0, y1, x0, x1;
  float fy, fx;
  up_taps(oy, H, &y0, &y1, &fy);
  const float4* s = in + b * sin4;
  const float4* r0 = s + size_t(y0) * W * C4;
  const float4* r1 = s + size_t(y1) * W * C4;
  float4* o = out + (size_t(b) * 2 * H + oy) * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int ox = i / C4, c = i - ox * C4;
    up_taps(ox, W, &x0, &x1, &fx);
    const float4 v00 = __ldg(r0 + x0 * C4 + c), v01 = __ldg(r0 + x1 * C4 + c);
    const float4 v10 = __ldg(r1 + x0 * C4 + c), v11 = __ldg(r1 + x1 * C4 + c);
    auto lerp2 = [&](float a, float bq, float cq, float d) {
      return (1.f - fy) * ((1.f - fx) * a + fx * bq) + fy * ((1.f - fx) * cq + fx * d);
    };
    o[i] = make_float4(lerp2(v00.x, v01.x, v10.x, v11.x), lerp2(v00.y, v01.y, v10.y, v11.y),
                       lerp2(v00.z, v01.z, v10.z, v11.z), lerp2(v00.w, v01.w, v10.w, v11.w));
  }
}

// [h^2 Re r, h^2 Im r, kappa^2] NHWC (inc/precond.hpp:74-83, gamma dropped)
__global__ void k_pack(int N, float h2, const int* act, const float2* __restrict__ r, const float* rscale,
                       const float* __restrict__ k2, float* __restrict__ x) {
  pdl_enter();
  const int b = blockIdx.y;
  if (act && !act[b]) return;
  const float s = h2 * (rscale ? rscale[b] : 1.0f);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    const float2 v = r[size_t(b) * N + i];
    float* o = x + (size_t(b) * N + i) * 3;
    o[0] = s * v.x;
    o[1] = s * v.y;
    o[2] = k2[i];
  }
}

__global__ void k_unpack(int N, const int* act, const float* __restrict__ y, float2* __restrict__ e) {
  pdl_enter();
  const int b = blockIdx.y;
  if (act && !act[b]) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    const float* s = y + (size_t(b) * N + i) * 2;
    e[size_t(b) * N + i] = make_float2(s[0], s[1]);
  }
}

__global__ void k_unpack_add(int N, const int* act, const float* __restrict__ y, const float2* base, float2* e) {
  pdl_enter();
  const int b = blockIdx.y;
  if (act && !act[b]) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    const float* s = y + (size_t(b) * N + i) * 2;
    const float2 o = base[size_t(b) * N + i];
    e[size_t(b) * N + i] = make_float2(o.x + s[0], o.y + s[1]);
  }
}

__global__ void k_nhwc_to_nchw(int B, int C, int HW, const float* __restrict__ in, float* __restrict__ out) {
  const size_t total = size_t(B) * C * HW;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += size_t(gridDim.x) * blockDim.x) {
    const int p = int(i % HW);
    const size_t bc = i / HW;
    const int c = int(bc % C), b = int(bc / C);
    out[i] = in[(size_t(b) * HW + p) * C + c];
  }
}
__global__ void k_nchw_to_nhwc(int B, int C, int HW, const float* __restrict__ in, float* __restrict__ out) {
  const size_t total = size_t(B) * C * HW;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += size_t(gridDim.x) * blockDim.x) {
    const int c = int(i % C);
    const size_t bp = i / C;
    const int p = int(bp % HW), b = int(bp / HW);
    out[i] = in[(size_t(b) * C + c) * HW + p];
  }
}

int grid1(size_t work, int cap = 4096) { return int(std::max<size_t>(1, std::min<size_t>((work + 255) / 256, cap))); }

}  // namespace


struct NScope {
  Context& c;
  int cls, tok;
  double bytes, flops;
  NScope(Context& c_, int cls_, double bytes_ = 0, double flops_ = 0)
      : c(c_), cls(cls_), tok(prof_begin(c_, cls_)), bytes(bytes_), flops(flops_) {}
  ~NScope() { prof_end(c, cls, tok, bytes, flops); }
};

template <int CIN>
static void head_cols(Context& c, int B, int H, int W, const float* x, const float* w, const float* b, float* y) {
  SmallW<CIN, 2> wt;
  for (int i = 0; i < 9 * CIN * 2; ++i) wt.w[i] = w[i];  // [tap][ci][co], as SmallW
  wt.b[0] = b[0];
  wt.b[1] = b[1];
  ConvArgs p{B, H, W, x, (long long)H * W * CIN, CIN, nullptr, 0, 0, nullptr, nullptr, 2, 0, y, nullptr};
  NScope ns(c, PC_CONV, double(B) * H * W * 4.0 * (CIN + 2), 2.0 * B * H * W * 9.0 * CIN * 2);
  conv_cols_launch(c, p, wt);
  HB_CUDA(cudaGetLastError());
}

bool launch_head_cols(Context& c, int cin, int B, int H, int W, const float* x, const float* w, const float* b,
                      float* y) {
  if (!c.opt_small_pw || !c.opt_conv_cols) return false;
  switch (cin) {
    case 12: head_cols<12>(c, B, H, W, x, w, b, y); return true;
    case 16: head_cols<16>(c, B, H, W, x, w, b, y); return true;
    case 20: head_cols<20>(c, B, H, W, x, w, b, y); return true;
    default: return false;
  }
}

// ---------------------------------------------------------------- launchers
static void conv(Context& c, const ConvW& cw, int B, const int* act, int H, int W, const float* a, long long sa,
                 int ca, const float* b, long long sb, int cb, int relu, float* out) {
  if (ca + cb != cw.cin) throw HbError{HB_ERR_ARG, "conv input channels mismatch"};
  if (launch_conv_rows(c, cw, B, act, H, W, a, ca, b, cb, b != nullptr && sb == 0, relu, out)) return;
  if (launch_conv_tc(c, cw, B, act, H, W, a, ca, b, cb, b != nullptr && sb == 0, relu, out)) return;
  ConvArgs p{B, H, W, a, sa, ca, b, sb, cb, cw.dw.p, cw.db.p, cw.cout, relu, out, act};
  const int cin = ca + cb;
  if ((cw.cout == 16 || cw.cout == 2) && cin <= 40) {
    const size_t smem =
        (size_t(CS_TH + 2) * (CS_TW + 2) * size_t(cin | 1) + ((size_t(9) * cin * cw.cout + 3) & ~size_t(3))) * sizeof(float);
    const dim3 g(((W + CS_TW - 1) / CS_TW) * ((H + CS_TH - 1) / CS_TH), 1, B);
    NScope ns(c, PC_CONV, double(B) * H * W * 4.0 * (cw.cin + cw.cout), 2.0 * B * H * W * 9.0 * cw.cin * cw.cout);
    if (c.prof_detail)
      c.prof_label = "conv_small " + std::to_string(B) + "x" + std::to_string(H) + "x" + std::to_string(W) + " " +
                     std::to_string(ca) + "+" + std::to_string(cb) + "->" + std::to_string(cw.cout);
    static bool attr = false;
    if (!attr) {
      HB_CUDA(cudaFuncSetAttribute(k_conv_small<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      HB_CUDA(cudaFuncSetAttribute(k_conv_small<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      attr = true;
    }
    const bool pw = c.opt_small_pw && ((c.opt_conv_cols && (conv_cols<16, 2>(c, cw, p) || conv_cols<8, 2>(c, cw, p))) ||
                                       conv_small_pw<3, 16>(c, cw, p, g) || conv_small_pw<19, 16>(c, cw, p, g) ||
                                       conv_small_pw<1, 16>(c, cw, p, g) || conv_small_pw<16, 2>(c, cw, p, g) ||
                                       conv_small_pw<8, 2>(c, cw, p, g));
    if (pw) {
    } else if (cw.cout == 16) {
      launch_pdl(c, k_conv_small<16>, dim3(g), dim3(CS_NT), smem, p);
    } else {
      launch_pdl(c, k_conv_small<2>, dim3(g), dim3(CS_NT), smem, p);
    }
    HB_CUDA(cudaGetLastError());
    return;
  }
  const dim3 grid(((W + CT_W - 1) / CT_W) * ((H + CT_H - 1) / CT_H), (cw.cout + CT_CO - 1) / CT_CO, B);
  NScope ns(c, PC_CONV, double(B) * H * W * 4.0 * (cw.cin + cw.cout), 2.0 * B * H * W * 9.0 * cw.cin * cw.cout);
  if (c.prof_detail)
    c.prof_label = "conv_simt " + std::to_string(B) + "x" + std::to_string(H) + "x" + std::to_string(W) + " " +
                   std::to_string(ca) + "+" + std::to_string(cb) + "->" + std::to_string(cw.cout);
  launch_pdl(c, k_conv3x3, dim3(grid), dim3(256), 0, p);
  HB_CUDA(cudaGetLastError());
}

static void maxpool(Context& c, int B, const int* act, int H, int W, int C, const float* in, float* out) {
  NScope ns(c, PC_NETIO);
  if (C % 4 == 0) {
    const int n = (W / 2) * (C / 4);
    launch_pdl(c, k_maxpool2_v4, dim3(H / 2, B), dim3(n >= 256 ? 256 : ((n + 31) / 32) * 32), 0,
        H, W, C / 4, reinterpret_cast<const float4*>(in), reinterpret_cast<float4*>(out), act);
    HB_CUDA(cudaGetLastError());
    return;
  }
  launch_pdl(c, k_maxpool2, dim3(grid1(size_t(H / 2) * (W / 2) * C), B), dim3(256), 0, B, H, W, C, in, out, act);
  HB_CUDA(cudaGetLastError());
}

static void upsample(Context& c, int B, const int* act, int H, int W, int C, const float* in, long long sin_,
                     float* out) {
  NScope ns(c, PC_NETIO);
  if (C % 4 == 0 && sin_ % 4 == 0) {
    const int n = 2 * W * (C / 4);
    launch_pdl(c, k_upsample2_v4, dim3(2 * H, B), dim3(n >= 256 ? 256 : ((n + 31) / 32) * 32), 0,
        H, W, C / 4, reinterpret_cast<const float4*>(in), sin_ / 4, reinterpret_cast<float4*>(out), act);
    HB_CUDA(cudaGetLastError());
    return;
  }
  launch_pdl(c, k_upsample2, dim3(grid1(size_t(4) * H * W * C), B), dim3(256), 0, B, H, W, C, in, sin_, out, act);
  HB_CUDA(cudaGetLastError());
}

void launch_pack_input(Context& c, const LevelView& L, double h2, int B, const int* act, const float2* r,
                       const float* rscale, float* x) {
  NScope ns(c, PC_NETIO);
  const int N = L.nx * L.ny;
  launch_pdl(c, k_pack, dim3(grid1(N), B), dim3(256), 0, N, float(h2), act, r, rscale, L.k2f, x);
  HB_CUDA(cudaGetLastError());
}

void launch_unpack_add(Context& c, int N, int B, const int* act, const float* y, const float2* base, float2* e) {
  NScope ns(c, PC_NETIO);
  launch_pdl(c, k_unpack_add, dim3(grid1(N), B), dim3(256), 0, N, act, y, base, e);
  HB_CUDA(cudaGetLastError());
}

void launch_unpack_output(Context& c, int N, int B, const int* act, const float* y, float2* e) {
  NScope ns(c, PC_NETIO);
  launch_pdl(c, k_unpack, dim3(grid1(N), B), dim3(256), 0, N, act, y, e);
  HB_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------ net topology
static void build_topology(Net& n) {
  const hb_net_cfg& g = n.cfg;
  n.convs.clear();
  auto add = [&](int cout, int cin) {
    ConvW w;
    w.cout = cout;
    w.cin = cin;
    w.w.assign(size_t(cout) * cin * 9, 0.f);
    w.b.assign(size_t(cout), 0.f);
    n.convs.push_back(std::move(w));
    return int(n.convs.size()) - 1;
  };
  if (g.kind == HB_NET_ENCODER) {
    for (int l = 0; l < g.levels; ++l) {
      n.enc1[l] = add(g.base, l == 0 ? g.in_ch : g.base);
      n.enc2[l] = add(g.base, g.base);
    }
    n.head = -1;
  } else {
    for (int l = 0; l < g.levels; ++l) {
      n.enc1[l] = add(g.base << l, (l == 0 ? g.in_ch : g.base << (l - 1)) + g.ctx_ch);
      n.enc2[l] = add(g.base << l, g.base << l);
    }
    for (int l = g.levels - 2; l >= 0; --l) {
      n.up[l] = add(g.base << l, (g.base << (l + 1)) + g.ctx_ch);
      n.dec1[l] = add(g.base << l, 2 * (g.base << l));
      n.dec2[l] = add(g.base << l, g.base << l);
    }
    n.head = add(2, g.base);
  }
  n.dirty = true;
}

void net_upload(Context& c, int slot) {
  Net& n = c.nets[slot];
  if (!n.dirty) return;
  std::vector<ConvW*> up;
  for (auto& cw : n.convs) up.push_back(&cw);
  n.pre_split = false;
  if (n.cfg.kind == HB_NET_SOLVER && n.cfg.ctx_ch > 0 && n.cfg.in_ch == 3 && n.cfg.ctx_ch == 16 && n.cfg.base == 16) {
    // split the input layer's [x | ctx] weights: pre_ctx (16 -> 16, bias) and pre_x (3 -> 16, no bias)
    const ConvW& full = n.convs[size_t(n.enc1[0])];
    const int ci0 = n.cfg.in_ch, cc = n.cfg.ctx_ch, co = full.cout;
    n.pre_ctx.cin = cc;
    n.pre_x.cin = ci0;
    n.pre_ctx.cout = n.pre_x.cout = co;
    n.pre_ctx.w.assign(size_t(co) * cc * 9, 0.f);
    n.pre_x.w.assign(size_t(co) * ci0 * 9, 0.f);
    for (int o = 0; o < co; ++o)
      for (int ci = 0; ci < full.cin; ++ci)
        for (int t = 0; t < 9; ++t) {
          const float v = full.w[(size_t(o) * full.cin + ci) * 9 + t];
          if (ci < ci0)
            n.pre_x.w[(size_t(o) * ci0 + ci) * 9 + t] = v;
          else
            n.pre_ctx.w[(size_t(o) * cc + (ci - ci0)) * 9 + t] = v;
        }
    n.pre_ctx.b = full.b;
    n.pre_x.b.assign(size_t(co), 0.f);
    up.push_back(&n.pre_ctx);
    up.push_back(&n.pre_x);
    n.pre_split = true;
  }
  // the other context-concat convs (first conv of levels >= 1, the up-convs)
  // whose x part runs on the tensor cores: [x | ctx] weights -> x part (no bias) +
  // context part (bias); the forward computes the context share once (B = 1)
  n.split_of.assign(n.convs.size(), -1);
  n.split_ctx.clear();
  n.split_x.clear();
  if (n.cfg.kind == HB_NET_SOLVER && n.cfg.ctx_ch > 0 && n.cfg.ctx_ch % 16 == 0) {
    std::vector<int> cands;
    for (int l = 1; l < n.cfg.levels; ++l) cands.push_back(n.enc1[l]);
    for (int l = 0; l + 1 < n.cfg.levels; ++l) cands.push_back(n.up[l]);
    for (int idx : cands) {
      const ConvW& full = n.convs[size_t(idx)];
      const int cc = n.cfg.ctx_ch, cx = full.cin - cc, co = full.cout;
      if (co % 16 || co > 256 || cx % 16 || cx <= 0) continue;  // x part must run on k_conv_rows / k_conv_tc
      ConvW xc, cp;
      xc.cin = cx;
      cp.cin = cc;
      xc.cout = cp.cout = co;
      xc.w.assign(size_t(co) * cx * 9, 0.f);
      cp.w.assign(size_t(co) * cc * 9, 0.f);
      for (int o = 0; o < co; ++o)
        for (int ci = 0; ci < full.cin; ++ci)
          for (int t = 0; t < 9; ++t) {
            const float v = full.w[(size_t(o) * full.cin + ci) * 9 + t];
            if (ci < cx)
              xc.w[(size_t(o) * cx + ci) * 9 + t] = v;
            else
              cp.w[(size_t(o) * cc + (ci - cx)) * 9 + t] = v;
          }
      cp.b = full.b;
      xc.b.assign(size_t(co), 0.f);
      n.split_of[size_t(idx)] = int(n.split_x.size());
      n.split_x.push_back(std::move(xc));
      n.split_ctx.push_back(std::move(cp));
    }
    for (auto& w : n.split_x) up.push_back(&w);
    for (auto& w : n.split_ctx) up.push_back(&w);
  }
  ++n.upload_gen;
  n.pre_buf = std::vector<DBuf<float>>(n.split_x.size() + 1);
  n.pre_ok.assign(n.split_x.size() + 1, 0);
  for (ConvW* cwp : up) {
    ConvW& cw = *cwp;
    std::vector<float> pk(size_t(9) * cw.cin * cw.cout);
    for (int co = 0; co < cw.cout; ++co)
      for (int ci = 0; ci < cw.cin; ++ci)
        for (int tap = 0; tap < 9; ++tap)
          pk[(size_t(tap) * cw.cin + ci) * cw.cout + co] = cw.w[(size_t(co) * cw.cin + ci) * 9 + tap];
    cw.dw.ensure(pk.size());
    cw.db.ensure(cw.b.size());
    HB_CUDA(cudaMemcpy(cw.dw.p, pk.data(), pk.size() * sizeof(float), cudaMemcpyHostToDevice));
    HB_CUDA(cudaMemcpy(cw.db.p, cw.b.data(), cw.b.size() * sizeof(float), cudaMemcpyHostToDevice));
    conv_tc_prepare(cw);
    conv_rows_prepare(cw);
  }
  ++g_alloc_gen;  // the narrow convolutions carry their weights as kernel parameters: drop captured graphs
  n.dirty = false;
  if (slot == 1) c.ctx_valid = false;
}

// per-forward activation buffers, keyed by shape
struct NetBuffers {
  int B = 0, H = 0, W = 0, slot = -1;
  std::vector<DBuf<float>> skip, tmp, pool, up, u;
};
static thread_local NetBuffers g_nb[2];

static NetBuffers& buffers(Context& c, int slot, int B, int H, int W) {
  NetBuffers& nb = g_nb[slot];
  const Net& n = c.nets[slot];
  const int L = n.cfg.levels;
  if (nb.B >= B && nb.H == H && nb.W == W && nb.slot == slot && int(nb.skip.size()) == L) return nb;
  nb.skip = std::vector<DBuf<float>>(size_t(L));
  nb.tmp = std::vector<DBuf<float>>(size_t(L));
  nb.pool = std::vector<DBuf<float>>(size_t(L));
  nb.up = std::vector<DBuf<float>>(size_t(L));
  nb.u = std::vector<DBuf<float>>(size_t(L));
  for (int l = 0; l < L; ++l) {
    const size_t px = size_t(B) * (H >> l) * (W >> l);
    const int cl = n.cfg.kind == HB_NET_ENCODER ? n.cfg.base : (n.cfg.base << l);
    nb.skip[size_t(l)].ensure(px * cl);
    nb.tmp[size_t(l)].ensure(px * cl);
    if (l > 0) nb.pool[size_t(l)].ensure(px * (n.cfg.kind == HB_NET_ENCODER ? n.cfg.base : (n.cfg.base << (l - 1))));
    if (l < L - 1 && n.cfg.kind == HB_NET_SOLVER) {
      nb.up[size_t(l)].ensure(px * (n.cfg.base << (l + 1)));
      nb.u[size_t(l)].ensure(px * cl);
    }
  }
  nb.B = B;
  nb.H = H;
  nb.W = W;
  nb.slot = slot;
  return nb;
}

// solver U-Net (A5, + A7 context concat); x NHWC in_ch -> y NHWC 2
// a context-concat conv as x part (per column, k_conv_rows) + context share
// (batch-broadcast ctx, once); false if the layer is not split / not eligible
static bool conv_split(Context& c, Net& n, NetBuffers& nb, int idx, int B, const int* act, int H, int W,
                       const float* x, int cx, const float* ctxp, int relu, float* out) {
  if (!c.opt_ctx_pre || idx < 0 || size_t(idx) >= n.split_of.size() || n.split_of[size_t(idx)] < 0 || !ctxp)
    return false;
  const int si = n.split_of[size_t(idx)];
  const ConvW& xc = n.split_x[size_t(si)];
  const ConvW& cp = n.split_ctx[size_t(si)];
  if (xc.cin != cx) return false;
  DBuf<float>& pre = n.pre_buf[size_t(si)];
  if (!n.pre_ok[size_t(si)]) {  // the context share: once per (weights, context maps)
    pre.ensure(size_t(H) * W * cp.cout);
    conv(c, cp, 1, nullptr, H, W, ctxp, 0, cp.cin, nullptr, 0, 0, 0, pre.p);
    n.pre_ok[size_t(si)] = 1;
  }
  return launch_conv_rows(c, xc, B, act, H, W, x, cx, nullptr, 0, false, relu, out, pre.p) ||
         launch_conv_tc(c, xc, B, act, H, W, x, cx, nullptr, 0, false, relu, out, pre.p);
}

// the per-column part of the split input layer: 3 -> 16 narrow conv whose
// accumulators start from the batch-broadcast context share pre (bias included)
static void conv_pre(Context& c, const ConvW& cw, int B, const int* act, int H, int W, const float* a, long long sa,
                     int ca, const float* pre, int relu, float* out) {
  ConvArgs p{B, H, W, a, sa, ca, nullptr, 0, 0, cw.dw.p, cw.db.p, cw.cout, relu, out, act};
  p.pre = pre;
  const dim3 g(((W + CS_TW - 1) / CS_TW) * ((H + CS_TH - 1) / CS_TH), 1, B);
  NScope ns(c, PC_CONV, double(B) * H * W * 4.0 * (cw.cin + 2 * cw.cout), 2.0 * B * H * W * 9.0 * cw.cin * cw.cout);
  if (c.prof_detail)
    c.prof_label = "conv_small(pre) " + std::to_string(B) + "x" + std::to_string(H) + "x" + std::to_string(W) + " " +
                   std::to_string(ca) + "->" + std::to_string(cw.cout);
  if (!conv_small_pw<3, 16>(c, cw, p, g)) throw HbError{HB_ERR_STATE, "split input layer: no 3 -> 16 kernel"};
  HB_CUDA(cudaGetLastError());
}

void net_forward_dev(Context& c, int slot, int B, const int* act, int H, int W, const float* x, float* y) {
  Net& n = c.nets[slot];
  if (!n.set || n.cfg.kind != HB_NET_SOLVER) throw HbError{HB_ERR_STATE, "solver net not set"};
  const int L = n.cfg.levels;
  if (H % (1 << (L - 1)) || W % (1 << (L - 1))) throw HbError{HB_ERR_ARG, "input dims must be divisible by 2^(L-1)"};
  const bool es = n.cfg.ctx_ch > 0;
  if (es && !c.ctx_valid) throw HbError{HB_ERR_STATE, "encoder-solver net needs hb_encode first"};
  net_upload(c, slot);
  NetBuffers& nb = buffers(c, slot, B, H, W);
  if (es) {  // cached context shares: valid for these weights, context maps and dims
    const unsigned long long key = (c.ctx_gen << 40) ^ (n.upload_gen << 28) ^ (unsigned long long)(H) << 14 ^ W;
    if (key != n.pre_key) {
      n.pre_key = key;
      n.pre_ok.assign(n.pre_ok.size(), 0);
    }
  }
  const float* cur = x;
  int curc = n.cfg.in_ch;
  for (int l = 0; l < L; ++l) {
    const int Hl = H >> l, Wl = W >> l, cl = n.cfg.base << l;
    if (l > 0) {
      maxpool(c, B, act, Hl * 2, Wl * 2, curc, cur, nb.pool[size_t(l)].p);
      cur = nb.pool[size_t(l)].p;
    }
    const float* ctxp = es ? c.ctx_maps[size_t(2 * l)].p : nullptr;
    if (l == 0 && es && n.pre_split && c.opt_small_pw && c.opt_ctx_pre) {
      // conv(concat(x, ctx)) = conv_x(x) + conv_ctx(ctx): the context maps are the
      // same for every column, so their share (with the bias) is computed once
      // (B = 1) and the per-column kernel convolves only the 3 input channels
      DBuf<float>& pre = n.pre_buf.back();
      if (!n.pre_ok.back()) {
        pre.ensure(size_t(Hl) * Wl * n.pre_ctx.cout);
        conv(c, n.pre_ctx, 1, nullptr, Hl, Wl, ctxp, 0, n.cfg.ctx_ch, nullptr, 0, 0, 0, pre.p);
        n.pre_ok.back() = 1;
      }
      conv_pre(c, n.pre_x, B, act, Hl, Wl, cur, (long long)Hl * Wl * curc, curc, pre.p, 1, nb.tmp[size_t(l)].p);
    } else if (!(es && conv_split(c, n, nb, n.enc1[l], B, act, Hl, Wl, cur, curc, ctxp, 1, nb.tmp[size_t(l)].p))) {
      conv(c, n.convs[size_t(n.enc1[l])], B, act, Hl, Wl, cur, (long long)Hl * Wl * curc, curc, ctxp, 0,
           es ? n.cfg.ctx_ch : 0, 1, nb.tmp[size_t(l)].p);
    }
    conv(c, n.convs[size_t(n.enc2[l])], B, act, Hl, Wl, nb.tmp[size_t(l)].p, (long long)Hl * Wl * cl, cl, nullptr, 0,
         0, 1, nb.skip[size_t(l)].p);
    cur = nb.skip[size_t(l)].p;
    curc = cl;
  }
  for (int l = L - 2; l >= 0; --l) {
    const int Hl = H >> l, Wl = W >> l, cl = n.cfg.base << l;
    // concat(x, ctx_{l+1}) then upsample == [upsample(x) | upsample(ctx_{l+1})]; the latter is cached
    upsample(c, B, act, Hl / 2, Wl / 2, curc, cur, (long long)(Hl / 2) * (Wl / 2) * curc, nb.up[size_t(l)].p);
    const float* cup = es ? c.ctx_maps[size_t(2 * (l + 1) + 1)].p : nullptr;
    if (!(es && conv_split(c, n, nb, n.up[l], B, act, Hl, Wl, nb.up[size_t(l)].p, curc, cup, 0, nb.u[size_t(l)].p)))
      conv(c, n.convs[size_t(n.up[l])], B, act, Hl, Wl, nb.up[size_t(l)].p, (long long)Hl * Wl * curc, curc, cup, 0,
           es ? n.cfg.ctx_ch : 0, 0, nb.u[size_t(l)].p);
    conv(c, n.convs[size_t(n.dec1[l])], B, act, Hl, Wl, nb.u[size_t(l)].p, (long long)Hl * Wl * cl, cl,
         nb.skip[size_t(l)].p, (long long)Hl * Wl * cl, cl, 1, nb.tmp[size_t(l)].p);
    conv(c, n.convs[size_t(n.dec2[l])], B, act, Hl, Wl, nb.tmp[size_t(l)].p, (long long)Hl * Wl * cl, cl, nullptr, 0,
         0, 1, nb.skip[size_t(l)].p);
    cur = nb.skip[size_t(l)].p;
    curc = cl;
  }
  conv(c, n.convs[size_t(n.head)], B, act, H, W, cur, (long long)H * W * curc, curc, nullptr, 0, 0, 0, y);
}

// encoder over kappa^2 (once per medium): ctx_maps[2l] = ctx_l (NHWC base ch at
// level l), ctx_maps[2l+1] = upsample(ctx_l) at level l-1 (for the up-convs)
void encoder_forward_dev(Context& c, int H, int W, const float* k2f) {
  Net& e = c.nets[1];
  if (!e.set || e.cfg.kind != HB_NET_ENCODER) throw HbError{HB_ERR_STATE, "encoder net (slot 1) not set"};
  net_upload(c, 1);
  const int L = e.cfg.levels, C = e.cfg.base;
  NetBuffers& nb = buffers(c, 1, 1, H, W);
  c.ctx_maps = std::vector<DBuf<float>>(size_t(2 * L));
  const float* cur = k2f;  // NHWC with 1 channel == plain [H][W]
  int curc = 1;
  for (int l = 0; l < L; ++l) {
    const int Hl = H >> l, Wl = W >> l;
    if (l > 0) {
      maxpool(c, 1, nullptr, Hl * 2, Wl * 2, curc, cur, nb.pool[size_t(l)].p);
      cur = nb.pool[size_t(l)].p;
    }
    conv(c, e.convs[size_t(e.enc1[l])], 1, nullptr, Hl, Wl, cur, 0, curc, nullptr, 0, 0, 1, nb.tmp[size_t(l)].p);
    c.ctx_maps[size_t(2 * l)].ensure(size_t(Hl) * Wl * C);
    conv(c, e.convs[size_t(e.enc2[l])], 1, nullptr, Hl, Wl, nb.tmp[size_t(l)].p, 0, C, nullptr, 0, 0, 1,
         c.ctx_maps[size_t(2 * l)].p);
    cur = c.ctx_maps[size_t(2 * l)].p;
    curc = C;
    if (l > 0) {
      c.ctx_maps[size_t(2 * l + 1)].ensure(size_t(4) * Hl * Wl * C);
      upsample(c, 1, nullptr, Hl, Wl, C, cur, 0, c.ctx_maps[size_t(2 * l + 1)].p);
    }
  }
  c.ctx_valid = true;
  ++c.ctx_gen;
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

static Net& net_slot(hb_ctx* ctx, int slot) {
  if (slot < 0 || slot > 1) throw HbError{HB_ERR_ARG, "net slot must be 0 or 1"};
  return ctx->nets[slot];
}

extern "C" {

int hb_set_net(hb_ctx* ctx, int slot, const hb_net_cfg* cfg) {
  HB_API_BEGIN
  Net& n = net_slot(ctx, slot);
  if (!cfg || cfg->levels < 1 || cfg->levels > 8 || cfg->base < 1 || cfg->in_ch < 1 || cfg->ctx_ch < 0)
    throw HbError{HB_ERR_ARG, "bad net config"};
  if (cfg->kind != HB_NET_SOLVER && cfg->kind != HB_NET_ENCODER) throw HbError{HB_ERR_ARG, "bad net kind"};
  n.cfg = *cfg;
  build_topology(n);
  n.set = true;
  if (slot == 0) paper_deactivate(*ctx);  // the classic net becomes slot 0's network
  if (slot == 1) ctx->ctx_valid = false;
  HB_API_END
}

int hb_net_num_convs(hb_ctx* ctx, int slot) {
  if (!ctx || slot < 0 || slot > 1) return HB_ERR_ARG;
  return int(ctx->nets[slot].convs.size());
}

int hb_net_conv_shape(hb_ctx* ctx, int slot, int index, int* cout, int* cin) {
  HB_API_BEGIN
  Net& n = net_slot(ctx, slot);
  if (index < 0 || index >= int(n.convs.size())) throw HbError{HB_ERR_ARG, "conv index out of range"};
  if (cout) *cout = n.convs[size_t(index)].cout;
  if (cin) *cin = n.convs[size_t(index)].cin;
  HB_API_END
}

int hb_load_conv(hb_ctx* ctx, int slot, int index, const float* w, const float* b) {
  HB_API_BEGIN
  Net& n = net_slot(ctx, slot);
  if (index < 0 || index >= int(n.convs.size())) throw HbError{HB_ERR_ARG, "conv index out of range"};
  ConvW& cw = n.convs[size_t(index)];
  if (w) std::memcpy(cw.w.data(), w, cw.w.size() * sizeof(float));
  if (b) std::memcpy(cw.b.data(), b, cw.b.size() * sizeof(float));
  n.dirty = true;
  if (slot == 1) ctx->ctx_valid = false;
  HB_API_END
}

int hb_get_conv(hb_ctx* ctx, int slot, int index, float* w, float* b) {
  HB_API_BEGIN
  Net& n = net_slot(ctx, slot);
  if (index < 0 || index >= int(n.convs.size())) throw HbError{HB_ERR_ARG, "conv index out of range"};
  const ConvW& cw = n.convs[size_t(index)];
  if (w) std::memcpy(w, cw.w.data(), cw.w.size() * sizeof(float));
  if (b) std::memcpy(b, cw.b.data(), cw.b.size() * sizeof(float));
  HB_API_END
}

int hb_init_net_he(hb_ctx* ctx, int slot, uint64_t seed) {
  HB_API_BEGIN
  Net& n = net_slot(ctx, slot);
  if (!n.set) throw HbError{HB_ERR_STATE, "net not set"};
  Rng r(seed);
  for (auto& cw : n.convs) {
    const float sd = float(std::sqrt(2.0 / double(cw.cin * 9)));
    for (auto& x : cw.w) x = float(r.normal()) * sd;  // fill_normal (inc/tensor.hpp:51-53)
    std::fill(cw.b.begin(), cw.b.end(), 0.f);
  }
  n.dirty = true;
  if (slot == 1) ctx->ctx_valid = false;
  HB_API_END
}

int hb_net_forward(hb_ctx* ctx, int batch, int H, int W, const float* in, float* out) {
  HB_API_BEGIN
  Net& n = net_slot(ctx, 0);
  if (!n.set) throw HbError{HB_ERR_STATE, "net slot 0 not set"};
  const int cin = n.cfg.in_ch;
  const size_t px = size_t(batch) * H * W;
  DBuf<float> a, b2, y, y2;
  a.ensure(px * cin);
  b2.ensure(px * cin);
  y.ensure(px * 2);
  y2.ensure(px * 2);
  HB_CUDA(cudaMemcpyAsync(a.p, in, px * cin * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
  k_nchw_to_nhwc<<<grid1(px * cin), 256, 0, ctx->stream>>>(batch, cin, H * W, a.p, b2.p);
  net_forward_dev(*ctx, 0, batch, nullptr, H, W, b2.p, y.p);
  k_nhwc_to_nchw<<<grid1(px * 2), 256, 0, ctx->stream>>>(batch, 2, H * W, y.p, y2.p);
  HB_CUDA(cudaMemcpyAsync(out, y2.p, px * 2 * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
  HB_CUDA(cudaStreamSynchronize(ctx->stream));
  HB_API_END
}

int hb_encode(hb_ctx* ctx) {
  HB_API_BEGIN
  if (!ctx->has_hier) throw HbError{HB_ERR_STATE, "hierarchy not built"};
  require_whole(*ctx);
  const Level& L = *ctx->levels[0];
  encoder_forward_dev(*ctx, L.ny, L.nx, L.k2f.p);
  HB_CUDA(cudaStreamSynchronize(ctx->stream));
  HB_API_END
}

int hb_get_context(hb_ctx* ctx, int level, float* out) {
  HB_API_BEGIN
  if (!ctx->ctx_valid) throw HbError{HB_ERR_STATE, "no encoder context (hb_encode)"};
  const Net& e = ctx->nets[1];
  if (level < 0 || level >= e.cfg.levels) throw HbError{HB_ERR_ARG, "level out of range"};
  const Level& L = *ctx->levels[0];
  const int Hl = L.ny >> level, Wl = L.nx >> level, C = e.cfg.base;
  DBuf<float> t;
  t.ensure(size_t(Hl) * Wl * C);
  k_nhwc_to_nchw<<<grid1(size_t(Hl) * Wl * C), 256, 0, ctx->stream>>>(1, C, Hl * Wl, ctx->ctx_maps[size_t(2 * level)].p,
                                                                      t.p);
  HB_CUDA(cudaMemcpyAsync(out, t.p, size_t(Hl) * Wl * C * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
  HB_CUDA(cudaStreamSynchronize(ctx->stream));
  HB_API_END
}

}  // extern "C"
