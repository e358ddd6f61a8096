// Row-streaming tensor-core 3x3 convolution for the 16-output-channel layers
// of the U-Nets (the top resolution level: 16 -> 16, 16+16 -> 16, 32 -> 16),
// where the per-tap implicit GEMM of hb_conv_tc.cu is bound by the count of
// N = 16/32 MMAs (~55 cycles each on B200 whatever N <= 64).
//
// The three vertical taps ky are batched into N instead of K: the A operand
// is one INPUT row x (one kx shift), B stacks the weights of ky = 0, 1, 2,
//   D_r[x, (ky, co)] = sum_ci X[r, x + kx - 1, ci] W[co, ci, ky, kx]   (N = 3*16)
// and output row y is assembled in the epilogue from three row accumulators,
//   out[y, x, co] = sum_ky D_{y+ky-1}[x, (ky, co)] + bias,
// so an input row is loaded and split into tf32 hi/lo once instead of three
// times, at 12-18 MMAs per 16-channel chunk instead of 36 per output tile.
// 3xTF32 (A = A_hi + A_lo, W = W_hi + W_lo, A_lo W_lo dropped) in two layouts:
//  * one CTA per SM (512 TMEM columns; layers whose weights need > ~75 KB of
//    shared memory): split accumulators, D[:, 0:96] += A_hi [W_hi | W_lo],
//    D[:, 48:96] += A_lo W_hi (two MMAs of N = 96 / 48 per k-step), a 3-4 row
//    D ring of 96 columns, two 16-channel chunks per step;
//  * two CTAs per SM (256 TMEM columns each; the 16-output-channel layers):
//    ONE 48-column accumulator per row, D += A_hi W_hi + A_hi W_lo + A_lo W_hi
//    (three N = 48 MMAs per k-step), a 3-row ring and one A slot.  Each CTA's
//    row pipeline (TMA -> A build -> MMA -> epilogue) is latency-bound --
//    per-role clock64 traces showed the stages handing over at ~1840 cycles
//    per input row with the tensor pipe ~30% busy -- so two independent
//    pipelines per SM raise throughput (16 -> 16 at 512^2 x 16: 228 -> 180 us).
//
// Persistent CTAs, warps: w0 TMA producer (input rows, a 16-channel (130 px)
// box per chunk, out-of-range pixels read zeros = the padding) | w1 MMA issuer
// | 8 (one CTA) or 4 (two CTAs) A-build warps (smem row -> TMEM hi/lo, three
// kx shifts) | 4 epilogue warps.  Work item = (image, 128-column strip, block
// of rb output rows); it streams rb + 2 input rows.  Row accumulators live in
// a TMEM ring; a D slot is released once the last output row using it is out.
#include "hb_common.cuh"
#include "hb_internal.h"
#include "hb_tc_ptx.cuh"

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

namespace hb {

namespace {

using namespace tcx;

// NCTA resident CTAs per SM: 1 -> 14 warps (8 A-build warps), 512 TMEM columns;
// 2 -> 10 warps (4 A-build warps), 256 TMEM columns each: two independent row
// pipelines share the SM's tensor pipe (the layer is latency-bound per CTA)
template <int NCTA>
struct CrShape {
  static constexpr int NAB = NCTA == 1 ? 8 : 4;  // A-build warps
  static constexpr int THREADS = 32 * (2 + NAB + 4);
  static constexpr int TMEM = NCTA == 1 ? 512 : 256;
  // one CTA: split accumulators [main 48 | correction 48] per row (two MMAs of N = 96 / 48 per k-step);
  // two CTAs: ONE 48-column accumulator per row (three N = 48 MMAs) so a 3-row ring + an A slot fit 256 columns
  static constexpr bool SPLIT = NCTA == 1;
  static constexpr int DW = SPLIT ? 96 : 48;
};
constexpr int CR_RBUF = 4;              // input rows in flight (smem ring)
constexpr int CR_BOX = 9216;            // one 16-channel row box: 130 px x 64 B = 8320 B, 1024-aligned
constexpr int CR_WBLK = 96 * 64;        // one (chunk, kx) weight block: 96 rows x 16 ch fp32
constexpr int CR_MAXRING = 6;

struct CrParams {
  int B, H, W, relu;
  int ldo;               // output pixel stride (floats): the layer's cout (a launch may cover one 16-channel slice)
  int ca, cb, b_is_ctx;  // source channels (multiples of 16)
  int nch;               // (ca + cb) / 16 input chunks
  int nslice;            // cout / 16 output slices (one work item each)
  int gch;               // chunks per step (input row group), 1 or 2
  int rb;                // output rows per work item
  int ring, na;          // D ring depth, A slots
  int rbuf;              // input-row smem buffers (<= CR_RBUF)
  const float* wrow;     // [nslice][nch][3 kx][96 rows][16 ci] packed, SW64-swizzled
  const float* bias;
  const float* pre;  // optional per-pixel [H][W][ldo] term replacing the bias, batch-broadcast (context share)
  float* out;
  const int* act;
};

template <int NCTA>
__global__ void __launch_bounds__(CrShape<NCTA>::THREADS, NCTA)
    k_conv_rows(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, CrParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ uint64_t bar_rfull[CR_RBUF], bar_rempty[CR_RBUF];
  __shared__ uint64_t bar_afull[2], bar_aempty[2];
  __shared__ uint64_t bar_dfull[CR_MAXRING], bar_dempty[CR_MAXRING], bar_w;
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int nch = p.nch, ring = p.ring, na = p.na, gch = p.gch, nrb = p.rbuf;
  const int ngrp = (nch + gch - 1) / gch;  // steps per input row
  const int nca = p.ca / 16;
  const int rowbuf = gch * CR_BOX;
  unsigned char* wsm = base + nrb * rowbuf;
  const int strips = p.W / 128, rblocks = (p.H + p.rb - 1) / p.rb;
  const int nitems = p.nslice * p.B * strips * rblocks;
  const int aw = gch * 3 * 32;   // TMEM columns of one A slot: (chunk, kx) x [hi 16 | lo 16]
  constexpr int DW = CrShape<NCTA>::DW;
  const int a0 = ring * DW;      // first A-slot column (D ring first)
  if (threadIdx.x == 0) {
    for (int i = 0; i < CR_RBUF; ++i) {
      mbar_init(&bar_rfull[i], 1);
      mbar_init(&bar_rempty[i], 32 * CrShape<NCTA>::NAB);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar_afull[i], 32 * CrShape<NCTA>::NAB);
      mbar_init(&bar_aempty[i], 1);
    }
    for (int i = 0; i < CR_MAXRING; ++i) {
      mbar_init(&bar_dfull[i], 1);
      mbar_init(&bar_dempty[i], 128);
    }
    mbar_init(&bar_w, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                 "r"(CrShape<NCTA>::TMEM));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_slot;

  // item -> output slice sl, image b, strip x0, output rows [y0, y1); rows fastest
  int sl = 0;
  auto decode = [&](int item, int& b, int& x0, int& y0, int& y1) {
    const int rbk = item % rblocks;
    int rest = item / rblocks;
    x0 = (rest % strips) * 128;
    rest /= strips;
    b = rest % p.B;
    sl = rest / p.B;
    y0 = rbk * p.rb;
    y1 = min(p.H, y0 + p.rb);
  };

  if (warp != 0) pdl_enter();  // the producer waits after issuing the weights
  if (warp == 0) {
    // ---------------- producer: weights once, then one row box per chunk and input row
    mbar_expect_tx_elect(&bar_w, uint32_t(p.nslice * nch * 3 * CR_WBLK));
    bulk_load_elect(wsm, p.wrow, uint32_t(p.nslice * nch * 3 * CR_WBLK), &bar_w);
    pdl_enter();  // PDL: the weights above are constant; rows / act / outputs only after the predecessor
    int s = 0;
    for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
      int b, x0, y0, y1;
      decode(item, b, x0, y0, y1);
      if (p.act && !p.act[b]) continue;
      const int bb = p.b_is_ctx ? 0 : b;
      for (int r = y0 - 1; r <= y1; ++r)
        for (int g = 0; g < ngrp; ++g, ++s) {
          const int rb_ = s % nrb;
          if (s >= nrb) mbar_wait(&bar_rempty[rb_], ((s / nrb) - 1) & 1);
          const bool valid = r >= 0 && r < p.H;
          const int c0 = g * gch, c1 = min(nch, c0 + gch);
          mbar_expect_tx_elect(&bar_rfull[rb_], valid ? uint32_t((c1 - c0) * 130 * 64) : 0u);
          if (valid) {
            for (int ch = c0; ch < c1; ++ch) {
              unsigned char* dst = base + rb_ * rowbuf + (ch - c0) * CR_BOX;
              if (ch < nca)
                tma_load_4d_elect(dst, &mapA, &bar_rfull[rb_], ch * 16, x0 - 1, r, b);
              else
                tma_load_4d_elect(dst, &mapB, &bar_rfull[rb_], (ch - nca) * 16, x0 - 1, r, bb);
            }
          }
        }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (whole warp, elected lane issues)
    const uint32_t id96 = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(96 >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    const uint32_t id48 = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(48 >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    const uint32_t hi16 = (512u >> 4) | (1u << 14) | (4u << 29);  // 64-B rows, SWIZZLE_64B
    const uint32_t tbase = __shfl_sync(0xffffffffu, tmem_base, 0);
    const uint32_t wlo0 = __shfl_sync(0xffffffffu, (smem_u32(wsm) >> 4) | (1u << 16), 0);
    mbar_wait(&bar_w, 0);
    int s = 0, rs = 0;  // step, input-row step (D slot index)
    for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
      int b, x0, y0, y1;
      decode(item, b, x0, y0, y1);
      if (p.act && !p.act[b]) continue;
      for (int r = y0 - 1; r <= y1; ++r, ++rs) {
        const int ds = rs % ring;
        if (rs >= ring) mbar_wait(&bar_dempty[ds], ((rs / ring) - 1) & 1);  // epilogue released this slot
        const uint32_t d = tbase + uint32_t(ds * DW);
        uint32_t first = 0;
        for (int g = 0; g < ngrp; ++g, ++s) {
          const int as = s % na;
          mbar_wait(&bar_afull[as], (s / na) & 1);
          tc_fence_after();
          if (r >= 0 && r < p.H) {
            const int c0 = g * gch, c1 = min(nch, c0 + gch);
            for (int u = 0; u < (c1 - c0) * 3; ++u) {
              const int ch = c0 + u / 3, kx = u - 3 * (u / 3);
              const uint32_t lw = wlo0 + uint32_t(((sl * nch + ch) * 3 + kx) * (CR_WBLK >> 4));
              const uint32_t ta = tbase + uint32_t(a0 + as * aw + u * 32);
#pragma unroll
              for (int kk = 0; kk < 2; ++kk) {
                if (CrShape<NCTA>::SPLIT) {
                  umma_ts(d, ta + 8 * kk, lw + 2 * kk, hi16, id96, first);            // A_hi [W_hi | W_lo]
                  umma_ts(d + 48, ta + 16 + 8 * kk, lw + 2 * kk, hi16, id48, 1u);   // A_lo W_hi -> correction
                } else {
                  umma_ts(d, ta + 8 * kk, lw + 2 * kk, hi16, id48, first);                // A_hi W_hi
                  umma_ts(d, ta + 8 * kk, lw + 2 * kk + (48 * 64 >> 4), hi16, id48, 1u);  // A_hi W_lo (rows 48..95)
                  umma_ts(d, ta + 16 + 8 * kk, lw + 2 * kk, hi16, id48, 1u);             // A_lo W_hi
                }
                first = 1;
              }
            }
          }
          umma_commit_elect(&bar_aempty[as]);
        }
        umma_commit_elect(&bar_dfull[ds]);
      }
    }
  } else if (warp < 2 + CrShape<NCTA>::NAB) {
    // ---------------- A build: input row (3 kx shifts x chunks) -> TMEM [hi | lo]
    constexpr int NG = CrShape<NCTA>::NAB / 4;  // A-build groups (4 warps = the TMEM lane quarters)
    const int q = warp & 3, half = (warp - 2) >> 2;
    const int pix = 32 * q + lane;
    int s = 0;
    for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
      int b, x0, y0, y1;
      decode(item, b, x0, y0, y1);
      if (p.act && !p.act[b]) continue;
      for (int r = y0 - 1; r <= y1; ++r)
       for (int g = 0; g < ngrp; ++g, ++s) {
        const int rb_ = s % nrb, as = s % na;
        mbar_wait(&bar_rfull[rb_], (s / nrb) & 1);
        if (s >= na) mbar_wait(&bar_aempty[as], ((s / na) - 1) & 1);
        tc_fence_after();
        if (r >= 0 && r < p.H) {
          const uint32_t ta = tmem_base + (uint32_t(32 * q) << 16) + uint32_t(a0 + as * aw);
          const int nu = (min(nch, (g + 1) * gch) - g * gch) * 3;
          for (int u = half; u < nu; u += NG) {
            const int ch = u / 3, kx = u - 3 * ch;  // chunk within this step's group
            const int hp = pix + kx;  // halo pixel (the box starts at x0 - 1)
            const unsigned char* row = base + rb_ * rowbuf + ch * CR_BOX + hp * 64;
            const int f = (hp >> 1) & 3;  // SWIZZLE_64B: 16-B chunk c of row hp sits at c ^ f
            uint32_t vh[16], vl[16];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const float4 x = *reinterpret_cast<const float4*>(row + ((c ^ f) << 4));
              const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const uint32_t hb = __float_as_uint(xs[e]) & 0xffffe000u;
                vh[4 * c + e] = hb;
                vl[4 * c + e] = __float_as_uint(xs[e] - __uint_as_float(hb));
              }
            }
            tmem_st16(ta + uint32_t(u * 32), vh);
            tmem_st16(ta + uint32_t(u * 32 + 16), vl);
          }
        }
        mbar_arrive(&bar_rempty[rb_]);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        mbar_arrive(&bar_afull[as]);
      }
    }
  } else {
    // ---------------- epilogue: out[y] = bias + sum_ky D_{y+ky-1}[ky] (main + correction)
    const int q = warp & 3;
    const int pix = 32 * q + lane;
    const uint32_t trow = tmem_base + (uint32_t(32 * q) << 16);
    const int cout = p.ldo;
    int sb = 0;  // step of the item's first input row
    for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
      int b, x0, y0, y1;
      decode(item, b, x0, y0, y1);
      if (p.act && !p.act[b]) continue;
      const int nst = (y1 - y0) + 2;
      for (int y = y0; y < y1; ++y) {
        const int j = y - y0;
        const int sn = sb + j + 2;  // input row y + 1: its commit implies rows y - 1, y
        mbar_wait(&bar_dfull[sn % ring], (sn / ring) & 1);
        tc_fence_after();
        float o[16];
        if (p.pre) {  // the batch-broadcast context share of a split encoder-solver layer (bias included)
          const float4* pp = reinterpret_cast<const float4*>(p.pre + (size_t(y) * p.W + x0 + pix) * cout + sl * 16);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float4 v = __ldg(pp + i);
            o[4 * i] = v.x;
            o[4 * i + 1] = v.y;
            o[4 * i + 2] = v.z;
            o[4 * i + 3] = v.w;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] = __ldg(p.bias + sl * 16 + i);
        }
        if (CrShape<NCTA>::SPLIT) {
#pragma unroll
          for (int ky = 0; ky < 3; ++ky) {
            const int rr = y + ky - 1;
            if (rr < 0 || rr >= p.H) continue;  // zero padding row: no accumulator
            const uint32_t dcol = uint32_t(((sb + j + ky) % ring) * DW + ky * 16);
            uint32_t v[16], u[16];
            tmem_ld16(trow + dcol, v);
            tmem_ld16(trow + dcol + 48, u);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int i = 0; i < 16; ++i) o[i] += __uint_as_float(v[i]) + __uint_as_float(u[i]);
          }
        } else {
          uint32_t v[3][16];
#pragma unroll
          for (int ky = 0; ky < 3; ++ky) {
            const int rr = y + ky - 1;
            if (rr < 0 || rr >= p.H) {  // zero padding row: no accumulator
#pragma unroll
              for (int i = 0; i < 16; ++i) v[ky][i] = 0u;
              continue;
            }
            tmem_ld16(trow + uint32_t(((sb + j + ky) % ring) * DW + ky * 16), v[ky]);
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int i = 0; i < 16; ++i)
            o[i] += __uint_as_float(v[0][i]) + __uint_as_float(v[1][i]) + __uint_as_float(v[2][i]);
        }
        if (p.relu) {
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] = fmaxf(o[i], 0.f);
        }
        float* dst = p.out + ((size_t(b) * p.H + y) * p.W + x0 + pix) * cout + sl * 16;
#pragma unroll
        for (int i = 0; i < 16; i += 4)
          *reinterpret_cast<float4*>(dst + i) = make_float4(o[i], o[i + 1], o[i + 2], o[i + 3]);
        tc_fence_before();
        mbar_arrive(&bar_dempty[(sb + j) % ring]);  // input row y - 1 has no later consumer
      }
      tc_fence_before();
      mbar_arrive(&bar_dempty[(sb + nst - 2) % ring]);  // rows y1 - 1 and y1
      mbar_arrive(&bar_dempty[(sb + nst - 1) % ring]);
      sb += nst;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(CrShape<NCTA>::TMEM));
  }
}

}  // namespace

// pack [Cout=16][Cin][3][3] into per-(chunk, kx) blocks of 96 rows x 16 ci:
// rows (part, ky, co), part 0 = W_hi, 1 = W_lo (tf32 round-to-nearest split),
// stored pre-swizzled (SWIZZLE_64B) so a linear bulk copy lands in UMMA layout
void conv_rows_prepare(ConvW& cw) {
  if (cw.cout % 16 || cw.cout > 32 || cw.cin % 16 || cw.cin > 128) return;
  const int nch = cw.cin / 16, nsl = cw.cout / 16;
  std::vector<float> pk(size_t(nsl) * nch * 3 * 96 * 16, 0.f);
  auto tf32 = [](float x) {
    uint32_t u;
    std::memcpy(&u, &x, 4);
    if ((u & 0x7f800000u) != 0x7f800000u) u = (u + 0x1000u) & 0xffffe000u;
    float r;
    std::memcpy(&r, &u, 4);
    return r;
  };
  for (int sl = 0; sl < nsl; ++sl)
  for (int ch = 0; ch < nch; ++ch)
    for (int kx = 0; kx < 3; ++kx)
      for (int part = 0; part < 2; ++part)
        for (int ky = 0; ky < 3; ++ky)
          for (int co = 0; co < 16; ++co)
            for (int k = 0; k < 16; ++k) {
              const int ci = ch * 16 + k;
              const float w = cw.w[(size_t(sl * 16 + co) * cw.cin + ci) * 9 + ky * 3 + kx];
              const float h = tf32(w);
              const float v = part == 0 ? h : tf32(w - h);
              const int row = part * 48 + ky * 16 + co;
              const size_t blk = size_t((sl * nch + ch) * 3 + kx) * 96 * 16;
              const int pos = ((k >> 2) ^ ((row >> 1) & 3)) * 4 + (k & 3);  // SW64 within the 512-B atom
              pk[blk + size_t(row) * 16 + size_t(pos)] = v;
            }
  cw.dwrow.ensure(pk.size());
  HB_CUDA(cudaMemcpy(cw.dwrow.p, pk.data(), pk.size() * 4, cudaMemcpyHostToDevice));
}

bool launch_conv_rows(Context& c, const ConvW& cw, int B, const int* act, int H, int W, const float* a, int ca,
                      const float* bsrc, int cb, bool b_ctx, int relu, float* out, const float* pre) {
  if (!c.opt_conv_rows || !c.opt_tc_conv) return false;
  if (cw.cout % 16 || cw.cout > 32 || !cw.dwrow.p || W % 128 || ca % 16 || cb % 16 || ca + cb != cw.cin ||
      cw.cin > 128)
    return false;
  CrParams p{};
  p.B = B;
  p.H = H;
  p.W = W;
  p.relu = relu;
  p.ca = ca;
  p.cb = cb;
  p.b_is_ctx = b_ctx ? 1 : 0;
  p.nch = cw.cin / 16;
  p.ldo = cw.cout;
  const size_t wslice = size_t(p.nch) * 3 * CR_WBLK;  // weights of one 16-channel output slice
  const int nsl_all = cw.cout / 16;
  // all output slices in one launch when their weights fit beside the row ring;
  // else (wide inputs, e.g. c3's 64 + 16 context -> 32) one launch per slice,
  // each holding only its slice's weights
  const bool per_slice = size_t(2) * CR_BOX * 2 + wslice * nsl_all + 1024 > 200 * 1024;
  p.nslice = per_slice ? 1 : nsl_all;
  const size_t wbytes = wslice * p.nslice;
  // two CTAs per SM when both fit the shared memory (112 KB each): 256 TMEM
  // columns each -> single accumulators, one chunk per step, one A slot, a
  // 3-row D ring; else one CTA with split accumulators (HB_CR_NCTA: force)
  static const int env_n = getenv("HB_CR_NCTA") ? atoi(getenv("HB_CR_NCTA")) : 0;
  const bool two = env_n ? env_n == 2 : (size_t(3) * CR_BOX + wbytes + 1024 <= 112 * 1024);
  if (two) {
    p.gch = 1;
    p.na = 1;
    p.ring = 3;
  } else {
    p.gch = p.nch == 1 ? 1 : 2;
    p.ring = p.gch == 1 ? 4 : 3;
    p.na = (p.ring * 96 + 2 * p.gch * 96 <= 512) ? 2 : 1;
  }
  const int strips = W / 128;
  // rows per work item: enough items for ~2 per SM, each >= 4 rows (halo: 2 extra input rows)
  p.rb = std::max(4, std::min(32, (p.nslice * B * strips * H) / std::max(1, (two ? 4 : 2) * c.num_sms)));
  p.act = act;
  const CUtensorMap mA = act_map(a, B, H, W, ca, 16, 130, 1);
  const CUtensorMap mB = cb ? act_map(bsrc, b_ctx ? 1 : B, H, W, cb, 16, 130, 1) : mA;
  const size_t cap = two ? 112 * 1024 : 200 * 1024;
  p.rbuf = CR_RBUF;
  while (p.rbuf > 2 && size_t(p.rbuf) * p.gch * CR_BOX + wbytes + 1024 > cap) --p.rbuf;
  const size_t smem = size_t(p.rbuf) * p.gch * CR_BOX + wbytes + 1024;
  if (smem > cap) return false;
  static int attr_dev = -1;
  if (attr_dev != c.device) {
    HB_CUDA(cudaFuncSetAttribute(k_conv_rows<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    HB_CUDA(cudaFuncSetAttribute(k_conv_rows<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024));
    attr_dev = c.device;
  }
  const int items = p.nslice * B * strips * ((H + p.rb - 1) / p.rb);
  const int grid = std::min(items, (two ? 2 : 1) * c.num_sms);
  const int tok = prof_begin(c, PC_CONV);
  if (c.prof_detail)
    c.prof_label = "conv_rows " + std::to_string(B) + "x" + std::to_string(H) + "x" + std::to_string(W) + " " +
                   std::to_string(ca) + "+" + std::to_string(cb) + "->" + std::to_string(cw.cout);
  for (int s = 0; s < (per_slice ? nsl_all : 1); ++s) {
    p.wrow = cw.dwrow.p + size_t(s) * wslice / sizeof(float);
    p.bias = cw.db.p + 16 * s;
    p.out = out + 16 * s;
    p.pre = pre ? pre + 16 * s : nullptr;
    if (two)
      launch_pdl(c, k_conv_rows<2>, dim3(grid), dim3(CrShape<2>::THREADS), smem, mA, mB, p);
    else
      launch_pdl(c, k_conv_rows<1>, dim3(grid), dim3(CrShape<1>::THREADS), smem, mA, mB, p);
  }
  prof_end(c, PC_CONV, tok, double(B) * H * W * 4.0 * (cw.cin + cw.cout), 2.0 * B * H * W * 9.0 * cw.cin * cw.cout);
  HB_CUDA(cudaGetLastError());
  return true;
}

}  // namespace hb
