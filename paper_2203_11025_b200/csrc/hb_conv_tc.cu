// 3x3 convolution (stride 1, zero padding 1, fused bias + ReLU) as an
// implicit GEMM on the 5th-generation tensor cores: tcgen05.mma kind::tf32
// with TMEM accumulators and TMA-staged operands -- the U-Net's dense
// contraction (inc/autodiff.hpp:124-149).
//
//   D[128 pixels x Cout] += A[128 x K] * W[Cout x K]^T,  K = 9 * Cin ordered (tap, ci)
//
// fp32-grade accuracy with 3xTF32: every operand is split x = x_hi + x_lo
// (x_hi a tf32 value, x_lo = x - x_hi) and D accumulates A_hi W_hi + A_hi W_lo
// + A_lo W_hi.  Weights are split once on the host (round-to-nearest);
// activations are split in shared memory right after their TMA load
// (truncation mask, exact residual).
//
// Persistent CTA per SM, 10 warps (see k_conv_tc).  An M tile of 128 pixels
// is a (bh x bw) pixel box of one image (bw = min(W, 128)), loaded per tap by a 4-D TMA box
// (channels, bw, bh, 1) whose out-of-range taps read zeros (= the padding).
// Channel concatenation [a | b] is two TMA sources inside the K loop.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "hb_common.cuh"
#include "hb_internal.h"
#include "hb_tc_ptx.cuh"

namespace hb {

namespace {

using namespace tcx;

constexpr int TC_THREADS = 448;  // 14 warps, see k_conv_tc
constexpr int TC_MAX_STAGES = 8;
constexpr int TC_M = 128;

struct TcSources {
  int ca, cb;         // channels of source a, b (b may be 0)
  int kca, kcb;       // K chunk (16 | 32) per source
  int b_is_ctx;       // source b is a batch-broadcast 3-D map (encoder context)
};

struct TcParams {
  int B, H, W, cout, relu;
  int ntile, nsplit;  // output channels per work item (N of the MMA), output-channel blocks per pixel tile
  int ksplit;         // K splits per (tile, block): > 1 writes raw partial sums to ws (bias/ReLU in the reduce)
  int sps;            // stages per K split (every split non-empty)
  float* ws;          // [ksplit][B*H*W][cout] partial sums
  int bw, bh;         // pixel box of one M tile
  TcSources s;
  const float* bias;
  float* out;
  const int* act;
  long long* trace;  // debug: per-stage role timestamps of CTA 0 (HB_CONV_TRACE), else null
  TcGeo geo;
  TcEpi epi;
};

// pipeline geometry chosen on the host (see launch_conv_tc)
struct TcLayout {
  int kcmax;      // widest channel chunk (16 | 32)
  int nchunk;     // channel chunks over both sources
  int CG;         // channel chunks per halo group
  int nhbuf;      // halo group buffers (1 | 2)
  int box_bytes;  // smem bytes per halo box (one channel chunk), 1024-aligned
  int G;          // K entries per MMA stage (= per TMEM A slot); stages never straddle a group
  int stages;     // weight ring depth (streamed weights)
  int nslots;     // TMEM A-slot ring depth
  int nacc;       // accumulator buffers (1 | 2)
  int wres;       // all weights resident in smem (loaded once per CTA)
};

// Persistent CTA (one per SM), 14 warps:
//   w0 TMA producer | w1 MMA issuer | w2..w9 A build (smem halo -> TMEM) | w10..w13 epilogue.
//
// An M tile is a bh x bw box of 128 output pixels of one image.  Its input is
// loaded ONCE per channel chunk as a TMA box of (bh+2) x (bw+2) pixels at
// (y0-1, x0-1): out-of-range rows/columns read zeros, which is the conv
// padding, and the 9 taps are 9 shifted views of that halo tile (an implicit
// GEMM that does not re-read the input per tap).  Channel chunks are grouped
// so a group's halo boxes fit a smem buffer (double-buffered when they fit).
//
// K is ordered (group, tap, chunk of the group); one K entry = one tap x kc
// input channels.  The A-build warps own TMEM lanes 32*(warp%4).. (= tile
// pixels): each thread reads its shifted halo pixel's kc channels (swizzled
// rows, conflict-free), splits x = hi + lo (hi = x with the 13 low mantissa
// bits cleared, lo = x - hi, exact) and stores both into a TMEM slot.  The MMA
// thread issues kind::tf32 MMAs with A read from TMEM and B = [W_hi ; W_lo]
// (2N rows) from smem, accumulating
//   D[:, 0:2N]  += A_hi [W_hi | W_lo]      D[:, N:2N] += A_lo W_hi
// so the small 3xTF32 terms sum apart from A_hi W_hi (the epilogue adds the
// halves).  Weights are resident in smem for small layers, else streamed per
// stage.  Accumulators are double-buffered in TMEM where the slot ring leaves
// room, so tile t's epilogue (TMEM -> bias, ReLU -> NHWC) overlaps tile t+1.
// All schedules are tabulated in shared memory once per CTA: the producer and
// MMA loops are serial, and integer division there costs more than a
// 16-channel chunk's data movement.
__device__ __forceinline__ float elu_f(float t) { return t >= 0.0f ? t : expm1f(t); }
// y = act(BN(t [+ res])) for output channel co (t includes the bias)
__device__ __forceinline__ float tc_epilogue(const TcEpi& e, int co, float t, const float* res) {
  if (res) t = *res + t;  // tape.add(x, t) (inc/unet.hpp:158)
  if (e.mu) t = ((t - __ldg(e.mu + co)) * __ldg(e.is + co)) * __ldg(e.g + co) + __ldg(e.be + co);
  return e.act == 1 ? fmaxf(t, 0.f) : e.act == 2 ? elu_f(t) : t;
}

constexpr int TC_MAX_CHUNKS = 320;  // K entries per tile (taps x channel chunks)
constexpr int TC_MAX_SLOTS = 8;
constexpr int TC_DYN_SMEM = 216 * 1024;  // + ~8 KB of static tables/barriers <= 227 KB

// GEN: general geometry / epilogue (paper net); false: the classic 3x3 stride-1
// bias (+ ReLU) layer with compile-time tap arithmetic and the plain epilogue
template <int KC, bool GEN>  // KC: uniform chunk width (16 | 32), or 0 = mixed-width sources
__global__ void __launch_bounds__(TC_THREADS, 1)
    k_conv_tc(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
              const __grid_constant__ CUtensorMap mapWh32, const __grid_constant__ CUtensorMap mapWl32,
              const __grid_constant__ CUtensorMap mapWh16, const __grid_constant__ CUtensorMap mapWl16, TcParams p,
              TcLayout lay, int dbg) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ uint64_t bar_full[TC_MAX_STAGES], bar_empty[TC_MAX_STAGES];  // weight ring
  __shared__ uint64_t bar_hfull[2], bar_hempty[2];                         // halo group buffers
  __shared__ uint64_t bar_afull[TC_MAX_SLOTS], bar_aempty[TC_MAX_SLOTS];   // TMEM A slots
  __shared__ uint64_t bar_tfull[2], bar_tempty[2], bar_w;
  __shared__ uint32_t tmem_slot;
  __shared__ int4 sched[TC_MAX_CHUNKS];  // per K entry: {chunk-in-group | ty << 8 | tx << 16, chunk, kglob, kc}
  __shared__ int2 stg[TC_MAX_CHUNKS];    // per stage: {kb0 | kb1 << 16, group | last stage of group << 16}
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (p.trace && blockIdx.x == 0 && threadIdx.x == 0) p.trace[240] = clock64();
  const int N = p.ntile;  // output channels of this CTA's work items; p.cout = row stride of out
  const int G = lay.G, kcmax = KC ? KC : lay.kcmax, nslots = lay.nslots, stages = lay.stages;
  const int CG = lay.CG, nhbuf = lay.nhbuf, nchunk = lay.nchunk;
  const int accw = 2 * N;                // TMEM columns per accumulator buffer [main | correction]
  const int slot_cols = G * 2 * kcmax;   // TMEM columns per A slot: G x [hi | lo]
  const int slot0 = lay.nacc * accw;     // first A-slot column
  const int tiles_x = p.W / p.bw, tiles_y = p.H / p.bh;
  const int ntiles = p.B * tiles_x * tiles_y * p.nsplit * p.ksplit;
  const int hw = p.geo.boxw;             // halo tile row pitch (pixels)
  const int NT = p.geo.ntaps, cs = p.geo.s;
  // 1024-align by offset (not by integer cast) so the compiler keeps the shared address space
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int w_bytes = 2 * N * kcmax * 4;  // one K entry of [W_hi ; W_lo]
  const bool wres = lay.wres != 0;
  const int hbuf_bytes = CG * lay.box_bytes;
  unsigned char* wbase = base + nhbuf * hbuf_bytes;  // resident weights (entry kb) or the weight ring
  const int wstage_bytes = G * w_bytes;
  const int nca = p.s.ca / p.s.kca;
  const int cin = p.s.ca + p.s.cb;
  const int ngrp = (nchunk + CG - 1) / CG;
  const int spg = (NT * CG + G - 1) / G;  // stages of a full group
  const int cg_last = nchunk - (ngrp - 1) * CG;
  const int nst = (ngrp - 1) * spg + (NT * cg_last + G - 1) / G;
  const int nk = NT * nchunk;
  for (int kb = threadIdx.x; kb < nk; kb += blockDim.x) {
    const int g = kb / (NT * CG), r = kb - g * NT * CG;
    const int cgn = min(CG, nchunk - g * CG);
    const int tap = r / cgn, j = r - tap * cgn;
    const int ch = g * CG + j;
    const bool srcb = ch >= nca;
    const int kc = srcb ? p.s.kcb : p.s.kca;
    const int cglob = srcb ? p.s.ca + (ch - nca) * kc : ch * kc;
    // x: chunk-in-group | tap's halo-box offsets (ty << 8, tx << 16)
    sched[kb] = make_int4(j | (p.geo.ty[tap] << 8) | (p.geo.tx[tap] << 16), ch, tap * cin + cglob, kc);
  }
  for (int st = threadIdx.x; st < nst; st += blockDim.x) {
    const int g = min(st / spg, ngrp - 1), ls = st - g * spg;
    const int cgn = min(CG, nchunk - g * CG);
    const int gend = NT * g * CG + NT * cgn;
    const int kb0 = NT * g * CG + ls * G, kb1 = min(kb0 + G, gend);
    stg[st] = make_int2(kb0 | (kb1 << 16), g | ((kb1 == gend ? 1 : 0) << 16));
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&bar_full[s], 1);
      mbar_init(&bar_empty[s], 1);
    }
    for (int h = 0; h < 2; ++h) {
      mbar_init(&bar_hfull[h], 1);
      mbar_init(&bar_hempty[h], 256);
    }
    for (int j = 0; j < nslots; ++j) {
      mbar_init(&bar_afull[j], 256);
      mbar_init(&bar_aempty[j], 1);
    }
    mbar_init(&bar_w, 1);
    for (int a = 0; a < 2; ++a) {
      mbar_init(&bar_tfull[a], 1);
      mbar_init(&bar_tempty[a], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_slot;
  if (p.trace && blockIdx.x == 0 && threadIdx.x == 0) p.trace[241] = clock64();

  // work item -> (image, pixel box, output-channel block n0, K split: stages [s0, s1))
  int n0 = 0, ks = 0, s0 = 0, s1 = 0;
  const int sps = p.ksplit > 1 ? p.sps : nst;
  auto tile_coords = [&](int item, int& b, int& y0, int& x0) {
    ks = item % p.ksplit;
    s0 = ks * sps;
    s1 = min(nst, s0 + sps);
    item /= p.ksplit;
    n0 = (item % p.nsplit) * N;
    const int tile = item / p.nsplit;
    b = tile / (tiles_x * tiles_y);
    y0 = ((tile / tiles_x) % tiles_y) * p.bh;
    x0 = (tile % tiles_x) * p.bw;
  };

  if (warp != 0) pdl_enter();  // the producer waits after issuing its resident weights
  if (warp == 0) {
    // ---------------- producer (whole warp, elected lane issues)
    int s = 0, it = 0, hb = 0, hit = 0;
    uint32_t ph = 0, hph = 0;
    if (wres) {  // the whole [W_hi ; W_lo] schedule, once
      uint32_t wb = 0;
      for (int kb = 0; kb < nk; ++kb) wb += uint32_t(2 * N * sched[kb].w * 4);
      mbar_expect_tx_elect(&bar_w, (dbg & 8) ? 0u : wb);
      for (int kb = 0; kb < nk && !(dbg & 8); ++kb) {
        const int4 e = sched[kb];
        const int kc = KC ? KC : e.w;
        unsigned char* w = wbase + kb * w_bytes;
        tma_load_2d_elect(w, kc == 32 ? &mapWh32 : &mapWh16, &bar_w, e.z, 0);
        tma_load_2d_elect(w + N * kc * 4, kc == 32 ? &mapWl32 : &mapWl16, &bar_w, e.z, 0);
      }
    }
    pdl_enter();  // PDL: weights above are constant; activations / act / outputs only after the predecessor
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      int b, y0, x0;
      tile_coords(tile, b, y0, x0);
      if (p.act && !p.act[b]) continue;
      const int bb = p.s.b_is_ctx ? 0 : b;
      for (int st = s0; st < s1; ++st) {
        const int2 sg2 = stg[st];
        const int4 sg = make_int4(sg2.x & 0xffff, sg2.x >> 16, sg2.y & 0xffff, sg2.y >> 16);
        if (sg.x == NT * sg.z * CG || st == s0) {  // first stage of a group (in this split): its halo boxes
          if (hit >= nhbuf) mbar_wait(&bar_hempty[hb], hph ^ 1);
          const int c0 = sg.z * CG, c1 = min(nchunk, c0 + CG);
          uint32_t bytes = 0;
          for (int ch = c0; ch < c1; ++ch) bytes += uint32_t((ch >= nca ? p.s.kcb : p.s.kca) * 4 * hw * p.geo.boxh);
          if (p.trace && blockIdx.x == 0 && lane == 0 && it < 64) p.trace[it * 4 + 0] = clock64();
          mbar_expect_tx_elect(&bar_hfull[hb], (dbg & 8) ? 0u : bytes);
          for (int ch = c0; ch < c1 && !(dbg & 8); ++ch) {
            unsigned char* dst = base + hb * hbuf_bytes + (ch - c0) * lay.box_bytes;
            if (ch < nca)
              tma_load_4d_elect(dst, &mapA, &bar_hfull[hb], ch * p.s.kca, x0 * cs + p.geo.ox, y0 * cs + p.geo.oy, b);
            else
              tma_load_4d_elect(dst, &mapB, &bar_hfull[hb], (ch - nca) * p.s.kcb, x0 * cs + p.geo.ox, y0 * cs + p.geo.oy,
                                bb);
          }
          if (++hb == nhbuf) {
            hb = 0;
            hph ^= 1;
          }
          ++hit;
        }
        if (!wres) {  // this stage's weights
          if (it >= stages) mbar_wait(&bar_empty[s], ph ^ 1);
          uint32_t wb = 0;
          for (int kb = sg.x; kb < sg.y; ++kb) wb += uint32_t(2 * N * sched[kb].w * 4);
          mbar_expect_tx_elect(&bar_full[s], (dbg & 8) ? 0u : wb);
          for (int kb = sg.x; kb < sg.y && !(dbg & 8); ++kb) {
            const int4 e = sched[kb];
            const int kc = KC ? KC : e.w;
            unsigned char* w = wbase + s * wstage_bytes + (kb - sg.x) * w_bytes;
            tma_load_2d_elect(w, kc == 32 ? &mapWh32 : &mapWh16, &bar_full[s], e.z, n0);
            tma_load_2d_elect(w + N * kc * 4, kc == 32 ? &mapWl32 : &mapWl16, &bar_full[s], e.z, n0);
          }
          if (++s == stages) {
            s = 0;
            ph ^= 1;
          }
          ++it;
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (whole warp, elected lane issues)
    // B descriptors as (lo, hi) words: lo = start >> 4 | LBO, hi = SBO |
    // version | layout; entry and K-step offsets are 32-bit adds on lo (the
    // 14-bit start field never carries for smem < 256 KB)
    const uint32_t idN = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(TC_M >> 4) << 24);
    const uint32_t id2N = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t((2 * N) >> 3) << 17) | (uint32_t(TC_M >> 4) << 24);
    const uint32_t hi32 = (1024u >> 4) | (1u << 14) | (2u << 29);  // 128-B rows, SWIZZLE_128B
    const uint32_t hi16 = (512u >> 4) | (1u << 14) | (4u << 29);   // 64-B rows, SWIZZLE_64B
    // warp-uniform copies (shfl from lane 0 lets the compiler keep them in uniform registers)
    const uint32_t tbase = __shfl_sync(0xffffffff, tmem_base, 0);
    const uint32_t wlo0 = __shfl_sync(0xffffffff, (smem_u32(wbase) >> 4) | (1u << 16), 0);
    const uint32_t w16 = uint32_t(w_bytes) >> 4, ws16 = uint32_t(wstage_bytes) >> 4;
    if (wres) mbar_wait(&bar_w, 0);
    int s = 0, j = 0;
    uint32_t ph = 0, aph = 0;
    int tl = 0;  // local tile counter
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      int b, y0, x0;
      tile_coords(tile, b, y0, x0);
      if (p.act && !p.act[b]) continue;
      const int acc = lay.nacc == 2 ? (tl & 1) : 0;
      const uint32_t tmem_d = tbase + uint32_t(acc * accw);
      if (lay.nacc == 2) {
        if (tl >= 2) mbar_wait(&bar_tempty[acc], ((tl >> 1) - 1) & 1);  // epilogue drained this buffer
      } else if (tl >= 1) {
        mbar_wait(&bar_tempty[0], (tl - 1) & 1);
      }
      tc_fence_after();
      uint32_t first = 0;  // accumulate flag: 0 only for the tile's first MMA
      for (int st = s0; st < s1; ++st) {
        const int2 sg2 = stg[st];
        const int4 sg = make_int4(sg2.x & 0xffff, sg2.x >> 16, sg2.y & 0xffff, sg2.y >> 16);
        if (!wres) mbar_wait(&bar_full[s], ph);  // weights in smem
        mbar_wait(&bar_afull[j], aph);           // A hi/lo in TMEM
        tc_fence_after();
        if (p.trace && blockIdx.x == 0 && lane == 0 && tl * nst + st < 64) p.trace[(tl * nst + st) * 4 + 2] = clock64();
        uint32_t lW = wres ? wlo0 + uint32_t(sg.x) * w16 : wlo0 + uint32_t(s) * ws16;
        uint32_t ta = tbase + uint32_t(slot0 + j * slot_cols);
        for (int kb = sg.x; kb < sg.y; ++kb, lW += w16, ta += uint32_t(2 * kcmax)) {
          const int kc = KC ? KC : sched[kb].w;
          if (dbg & 1) continue;
          const uint32_t hi = kc == 32 ? hi32 : hi16;
          const uint32_t tal = ta + uint32_t(kc);
#pragma unroll
          for (int k = 0; k < kc / 8; ++k) {
            umma_ts(tmem_d, ta + 8 * k, lW + 2 * k, hi, id2N, first);
            umma_ts(tmem_d + uint32_t(N), tal + 8 * k, lW + 2 * k, hi, idN, 1u);
            first = 1;
          }
        }
        if (!wres) umma_commit_elect(&bar_empty[s]);  // weight stage free once these MMAs completed
        umma_commit_elect(&bar_aempty[j]);             // A slot free likewise
        if (!wres && ++s == stages) {
          s = 0;
          ph ^= 1;
        }
        if (++j == nslots) {
          j = 0;
          aph ^= 1;
        }
      }
      umma_commit_elect(&bar_tfull[acc]);
      ++tl;
    }
  } else if (warp < 10) {
    // ---------------- warps 2..9: A build, halo smem -> TMEM slot [hi | lo];
    // two warps per TMEM lane quarter, taking alternate entries of a stage
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;
    const int r = 32 * q + lane;  // tile pixel = TMEM lane
    const int yy = r / p.bw, xx = r - yy * p.bw;
    int j = 0, hb = 0, itc = 0;
    uint32_t aph = 0, hph = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      int b, y0, x0;
      tile_coords(tile, b, y0, x0);
      if (p.act && !p.act[b]) continue;
      for (int st = s0; st < s1; ++st, ++itc) {
        const int2 sg2 = stg[st];
        const int4 sg = make_int4(sg2.x & 0xffff, sg2.x >> 16, sg2.y & 0xffff, sg2.y >> 16);
        if (sg.x == NT * sg.z * CG || st == s0) {
          mbar_wait(&bar_hfull[hb], hph);
          if (GEN && p.epi.in_elu) {
            // ELU of the input once per halo element, in place, by all 8 A-build
            // warps (every tap reads each element; applying it per tap in the A build
            // cost 9 expm1 per element and made the A build the pipeline's bottleneck)
            float4* h4 = reinterpret_cast<float4*>(base + hb * hbuf_bytes);
            const int n4 = hbuf_bytes / 16;
            for (int i0 = threadIdx.x - 64; i0 < n4; i0 += 4 * 256) {  // 4 independent elements in flight
              float4 x[4];
#pragma unroll
              for (int u = 0; u < 4; ++u)
                if (i0 + u * 256 < n4) x[u] = h4[i0 + u * 256];
#pragma unroll
              for (int u = 0; u < 4; ++u)
                if (i0 + u * 256 < n4) h4[i0 + u * 256] = make_float4(elu_f(x[u].x), elu_f(x[u].y), elu_f(x[u].z), elu_f(x[u].w));
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // before the TMA refills this buffer
            asm volatile("bar.sync 1, 256;" ::: "memory");
          }
        }
        if (itc >= nslots) mbar_wait(&bar_aempty[j], aph ^ 1);
        tc_fence_after();
        if (p.trace && blockIdx.x == 0 && r == 0 && half == 0 && itc < 64) p.trace[itc * 4 + 1] = clock64();
        const unsigned char* hbuf = base + hb * hbuf_bytes;
        uint32_t ta = tmem_base + (uint32_t(32 * q) << 16) + uint32_t(slot0 + j * slot_cols);
        for (int kb = sg.x; kb < sg.y; ++kb, ta += uint32_t(2 * kcmax)) {
          if ((dbg & 2) || ((kb - sg.x) & 1) != half) continue;
          const int4 e = sched[kb];
          const int kc = KC ? KC : e.w;
          const int cj = e.x & 255, ty = (e.x >> 8) & 255, tx = (e.x >> 16) & 255;
          const int hp = GEN ? (yy * cs + ty) * hw + xx * cs + tx : (yy + ty) * hw + xx + tx;  // shifted halo pixel
          const unsigned char* row = hbuf + cj * lay.box_bytes + hp * (kc * 4);
          // swizzled 16-B chunk c of smem row hp sits at c ^ f(hp): SW128 f = hp & 7, SW64 f = (hp >> 1) & 3
          const int f = kc == 32 ? (hp & 7) : ((hp >> 1) & 3);
#pragma unroll
          for (int h = 0; h < kc / 16; ++h) {
            uint32_t vh[16], vl[16];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const float4 x = *reinterpret_cast<const float4*>(row + (((4 * h + c) ^ f) << 4));
              const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const uint32_t hbits = __float_as_uint(xs[u]) & 0xffffe000u;
                vh[4 * c + u] = hbits;
                vl[4 * c + u] = __float_as_uint(xs[u] - __uint_as_float(hbits));
              }
            }
            tmem_st16(ta + uint32_t(16 * h), vh);
            tmem_st16(ta + uint32_t(kc + 16 * h), vl);
          }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        mbar_arrive(&bar_afull[j]);
        if (sg.w || st == s1 - 1) {  // group (or split) done: its halo buffer may be refilled
          mbar_arrive(&bar_hempty[hb]);
          if (++hb == nhbuf) {
            hb = 0;
            hph ^= 1;
          }
        }
        if (p.trace && blockIdx.x == 0 && r == 0 && half == 0 && itc < 64) p.trace[itc * 4 + 3] = clock64();
        if (++j == nslots) {
          j = 0;
          aph ^= 1;
        }
      }
    }
  } else {
    // ---------------- warps 10..13: epilogue; warp owns TMEM lanes 32*(warp%4) .. +31 (= tile pixel rows)
    const int q = warp & 3;
    int tl = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      int b, y0, x0;
      tile_coords(tile, b, y0, x0);
      if (p.act && !p.act[b]) continue;
      const int acc = lay.nacc == 2 ? (tl & 1) : 0;
      const uint32_t uph = lay.nacc == 2 ? uint32_t((tl >> 1) & 1) : uint32_t(tl & 1);
      mbar_wait(&bar_tfull[acc], uph);
      tc_fence_after();
      const int row = 32 * q + lane;
      const int yy = row / p.bw, xx = row % p.bw;
      const size_t pix = (size_t(b) * p.H + (y0 + yy)) * p.W + (x0 + xx);
      const size_t opix = (size_t(b) * p.geo.Ho + (y0 + yy) * p.geo.os + p.geo.py) * p.geo.Wo +
                          (x0 + xx) * p.geo.os + p.geo.px;
      const bool part = p.ksplit > 1;  // raw partial sum; the epilogue runs after the K reduction
      float* orow = part ? p.ws + size_t(ks) * p.B * p.H * p.W * p.cout + pix * p.cout + n0
                         : p.out + opix * p.geo.ldo + n0;
      const float* rrow = p.epi.res ? p.epi.res + opix * p.epi.ldres + n0 : nullptr;
      const float* bias = p.bias + n0;
      const uint32_t trow = tmem_base + (uint32_t(32 * q) << 16) + uint32_t(acc * accw);
      for (int c0 = 0; c0 < ((dbg & 4) ? 0 : N); c0 += 16) {
        int cq = n0 + c0;  // output channel of the chunk (par4: within its parity block)
        if (GEN && p.geo.par4 && !part) {
          const int qb = (n0 + c0) / p.geo.par4;
          cq = (n0 + c0) - qb * p.geo.par4;
          const size_t op = (size_t(b) * p.geo.Ho + (y0 + yy) * 2 + (qb >> 1)) * p.geo.Wo + (x0 + xx) * 2 + (qb & 1);
          orow = p.out + op * p.geo.ldo + cq - c0;  // + c0 + i below
          rrow = p.epi.res ? p.epi.res + op * p.epi.ldres + cq - c0 : nullptr;
        }
        uint32_t v[16], u[16];
        tmem_ld16(trow + uint32_t(c0), v);
        tmem_ld16(trow + uint32_t(N + c0), u);
        float bz[16];  // bias, or the per-pixel context share (bias included) of a split layer
        if (p.epi.pre) {
          const float4* pp = reinterpret_cast<const float4*>(
              p.epi.pre + (opix - size_t(b) * p.geo.Ho * p.geo.Wo) * p.epi.ldpre + n0 + c0);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float4 w4 = __ldg(pp + i);
            bz[4 * i] = w4.x;
            bz[4 * i + 1] = w4.y;
            bz[4 * i + 2] = w4.z;
            bz[4 * i + 3] = w4.w;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) bz[i] = __ldg(bias + c0 + i);
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        float o[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float x = __uint_as_float(v[i]) + __uint_as_float(u[i]);
          if (GEN) {
            o[i] = part ? x : tc_epilogue(p.epi, n0 + c0 + i, x + bz[i], rrow ? rrow + c0 + i : nullptr);
          } else {
            const float y = x + bz[i];
            o[i] = part ? x : p.relu ? fmaxf(y, 0.f) : y;
          }
        }
        const int nvalid = GEN && p.epi.nco && !part ? p.epi.nco - cq : 16;  // padded output channels: not stored
#pragma unroll
        for (int i = 0; i < 16; i += 4)
          if (i < nvalid) *reinterpret_cast<float4*>(orow + c0 + i) = make_float4(o[i], o[i + 1], o[i + 2], o[i + 3]);
      }
      tc_fence_before();
      mbar_arrive(&bar_tempty[acc]);
      ++tl;
    }
  }
  if (p.trace && blockIdx.x == 0 && lane == 0 && warp >= 10) p.trace[242 + warp - 10] = clock64();
  tc_fence_before();
  __syncthreads();
  if (p.trace && blockIdx.x == 0 && threadIdx.x == 0) p.trace[246] = clock64();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512));
  }
}

// split-K reduction for the dense bias (+ ReLU) case: float4 over channels
__global__ void k_conv_ksum4(int ksplit, size_t n4, int cout4, size_t img4, const int* act,
                             const float4* __restrict__ ws, const float4* __restrict__ bias, int relu,
                             float4* __restrict__ out) {
  pdl_enter();
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += size_t(gridDim.x) * blockDim.x) {
    if (act && !act[i / img4]) continue;  // frozen column: its partials were not written
    float4 a = __ldg(bias + (i % cout4));
    for (int s = 0; s < ksplit; ++s) {
      const float4 v = __ldg(ws + size_t(s) * n4 + i);
      a.x += v.x;
      a.y += v.y;
      a.z += v.z;
      a.w += v.w;
    }
    if (relu) a = make_float4(fmaxf(a.x, 0.f), fmaxf(a.y, 0.f), fmaxf(a.z, 0.f), fmaxf(a.w, 0.f));
    out[i] = a;
  }
}

// split-K reduction: out = epilogue(bias + sum_s ws[s]) in fixed order
// (deterministic); ws is dense over the tile grid, out follows the geometry
__global__ void k_conv_ksum(int ksplit, int B, int H, int W, int cout, const int* act, const float* __restrict__ ws,
                            const float* __restrict__ bias, TcGeo geo, TcEpi epi, float* __restrict__ out) {
  pdl_enter();
  const size_t n = size_t(B) * H * W * cout;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    const size_t pix = i / cout;
    const int co = int(i - pix * cout);
    const int b = int(pix / (size_t(H) * W));
    if (act && !act[b]) continue;  // frozen column: its partials were not written
    const int rem = int(pix - size_t(b) * H * W), y = rem / W, x = rem - y * W;
    float a = __ldg(bias + co);
    for (int s = 0; s < ksplit; ++s) a += __ldg(ws + size_t(s) * n + i);
    int cq = co;
    size_t opix = (size_t(b) * geo.Ho + y * geo.os + geo.py) * geo.Wo + x * geo.os + geo.px;
    if (geo.par4) {  // the four parity classes of a transposed conv in one GEMM
      const int qb = co / geo.par4;
      cq = co - qb * geo.par4;
      opix = (size_t(b) * geo.Ho + y * 2 + (qb >> 1)) * geo.Wo + x * 2 + (qb & 1);
    }
    if (epi.nco && cq >= epi.nco) continue;  // padded output channel
    out[opix * geo.ldo + cq] = tc_epilogue(epi, co, a, epi.res ? epi.res + opix * epi.ldres + cq : nullptr);
  }
}

}  // namespace

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    HB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) throw HbError{HB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable"};
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// activation map: NHWC fp32 [B][H][W][C] as 4-D (C, W, H, B); box (kc, bw, bh, 1)
// (the conv loads halo tiles: bw, bh include the 1-pixel border)
CUtensorMap act_map(const float* ptr, int B, int H, int W, int C, int kc, int bw, int bh) {
  CUtensorMap m;
  const cuuint64_t dims[4] = {cuuint64_t(C), cuuint64_t(W), cuuint64_t(H), cuuint64_t(B)};
  const cuuint64_t strides[3] = {cuuint64_t(C) * 4, cuuint64_t(W) * C * 4, cuuint64_t(H) * W * C * 4};
  const cuuint32_t box[4] = {cuuint32_t(kc), cuuint32_t(bw), cuuint32_t(bh), 1};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  const CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(ptr), dims, strides, box,
                                  es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                  kc == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw HbError{HB_ERR_CUDA, "cuTensorMapEncodeTiled(act) failed " + std::to_string(int(r))};
  return m;
}

// weight map: [Cout][K] fp32 as 2-D (K, Cout); box (kc, rows)
CUtensorMap w_map(const float* ptr, int cout, int K, int kc, int rows) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {cuuint64_t(K), cuuint64_t(cout)};
  const cuuint64_t strides[1] = {cuuint64_t(K) * 4};
  const cuuint32_t box[2] = {cuuint32_t(kc), cuuint32_t(rows)};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides, box,
                                  es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                  kc == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw HbError{HB_ERR_CUDA, "cuTensorMapEncodeTiled(w) failed " + std::to_string(int(r))};
  return m;
}


// hi/lo split of the packed [Cout][9*Cin] weights (host, once per upload)
void conv_tc_prepare(ConvW& cw) {
  const int K = 9 * cw.cin;
  std::vector<float> packed(size_t(cw.cout) * K);
  for (int co = 0; co < cw.cout; ++co)
    for (int tap = 0; tap < 9; ++tap)
      for (int ci = 0; ci < cw.cin; ++ci)
        packed[size_t(co) * K + size_t(tap) * cw.cin + ci] = cw.w[(size_t(co) * cw.cin + ci) * 9 + tap];
  conv_tc_upload_packed(cw, packed);
}

static bool tc_ok_channels(int c) { return c > 0 && c % 16 == 0; }

// returns false when the shape is not supported by the tensor-core path
bool launch_conv_tc_gen(Context& c, const TcConv& t) {
  const ConvW& cw = *t.cw;
  const int B = t.B, H = t.H, W = t.W, ca = t.ca, cb = t.cb;
  const int NT = t.geo.ntaps;
  if (!c.opt_tc_conv) return false;
  if (NT < 1 || NT > TC_MAX_TAPS) return false;
  if (!tc_ok_channels(ca) || (cb && !tc_ok_channels(cb))) return false;
  if (cw.cout % 16 || cw.cout > 256 || cw.cout < 16 || !cw.dwh.p) return false;
  const int bw = W < TC_M ? W : TC_M;
  const int bh = TC_M / bw;
  if (W % bw || H % bh || bw * bh != TC_M || bw < 8) return false;
  int mty = 0, mtx = 0;
  for (int i = 0; i < NT; ++i) {
    mty = std::max(mty, t.geo.ty[i]);
    mtx = std::max(mtx, t.geo.tx[i]);
  }
  TcGeo geo = t.geo;
  geo.boxh = (bh - 1) * geo.s + mty + 1;
  geo.boxw = (bw - 1) * geo.s + mtx + 1;
  if (geo.boxh > 256 || geo.boxw > 256) return false;
  const int kca = ca % 32 == 0 ? 32 : 16, kcb = cb ? (cb % 32 == 0 ? 32 : 16) : 32;
  const int kcmax = (kca == 32 || (cb && kcb == 32)) ? 32 : 16;
  const int nchunk = ca / kca + (cb ? cb / kcb : 0);
  const int nk = NT * nchunk;
  if (nk > TC_MAX_CHUNKS) return false;
  // Cout > 128 is split into 128-channel work items so every layer uses the
  // split-accumulator form (correction terms summed apart, better accuracy)
  const int nsplit = cw.cout > 128 ? cw.cout / 128 : 1;
  const int ntile = cw.cout / nsplit;
  if (ntile * nsplit != cw.cout || ntile > 128) return false;

  TcLayout lay{};
  lay.kcmax = kcmax;
  lay.nchunk = nchunk;
  // TMEM (512 columns): accumulators [nacc x 2N] then A slots of G x [hi | lo] entries
  const int accw = 2 * ntile;
  lay.nacc = 2 * accw + 2 * (2 * 2 * kcmax) <= 512 ? 2 : 1;
  const int free_cols = 512 - lay.nacc * accw;
  if (free_cols < 2 * 2 * kcmax) return false;
  lay.G = std::max(1, std::min(9, free_cols / (3 * 2 * kcmax)));  // aim for ~3 slots in flight
  lay.nslots = std::min(TC_MAX_SLOTS, free_cols / (lay.G * 2 * kcmax));
  if (lay.nslots < 2) return false;
  // shared memory: halo group buffers, then resident weights or a weight ring
  const int budget = TC_DYN_SMEM - 1024;
  const int w_chunk = 2 * ntile * kcmax * 4;
  lay.wres = nsplit == 1 && nk * w_chunk <= 96 * 1024 ? 1 : 0;
  lay.stages = lay.wres ? 1 : 4;
  lay.box_bytes = ((kcmax * 4 * geo.boxw * geo.boxh) + 1023) & ~1023;
  auto wsmem = [&]() { return lay.wres ? nk * w_chunk : lay.stages * lay.G * w_chunk; };
  for (;;) {
    const int room = budget - wsmem();
    lay.CG = std::min(nchunk, room / (2 * lay.box_bytes));
    lay.nhbuf = 2;
    if (lay.CG < 1) {
      lay.CG = std::min(nchunk, room / lay.box_bytes);
      lay.nhbuf = 1;
    }
    if (lay.CG >= 1 || lay.wres || lay.stages == 2) break;
    --lay.stages;
  }
  if (lay.CG < 1) return false;
  const int ngrp = (nchunk + lay.CG - 1) / lay.CG;
  const int spg = (NT * lay.CG + lay.G - 1) / lay.G;
  if (ngrp * spg > TC_MAX_CHUNKS) return false;
  const size_t smem = size_t(lay.nhbuf) * lay.CG * lay.box_bytes + size_t(wsmem()) + 1024;

  const CUtensorMap mA = act_map(t.a, B, t.Hin, t.Win, ca, kca, geo.boxw, geo.boxh);
  const CUtensorMap mB = cb ? act_map(t.bsrc, t.b_ctx ? 1 : B, t.Hin, t.Win, cb, kcb, geo.boxw, geo.boxh) : mA;
  const int K = NT * cw.cin;
  const CUtensorMap wh32 = w_map(cw.dwh.p, cw.cout, K, 32, ntile), wl32 = w_map(cw.dwl.p, cw.cout, K, 32, ntile);
  const CUtensorMap wh16 = w_map(cw.dwh.p, cw.cout, K, 16, ntile), wl16 = w_map(cw.dwl.p, cw.cout, K, 16, ntile);
  // split K when the pixel tiles alone cannot fill the SMs (low-resolution levels)
  const int tiles0 = B * (H / bh) * (W / bw) * nsplit;
  const int nst = (ngrp - 1) * spg + (NT * (nchunk - (ngrp - 1) * lay.CG) + lay.G - 1) / lay.G;
  int ksplit = 1;
  if (c.opt_conv_ksplit && tiles0 * 2 <= c.num_sms && !t.epi.pre)  // (the reduce kernels add the bias, not pre)
    ksplit = std::max(1, std::min({nst, c.num_sms / tiles0, 8}));
  const int sps = (nst + ksplit - 1) / ksplit;
  ksplit = (nst + sps - 1) / sps;  // no empty split
  float* ws = nullptr;
  if (ksplit > 1) {
    c.conv_ws.ensure(size_t(ksplit) * B * H * W * cw.cout);
    ws = c.conv_ws.p;
  }
  TcParams p{B,  H,  W,     cw.cout, t.epi.act == 1 ? 1 : 0, ntile,   nsplit, ksplit, sps, ws, bw, bh,
             TcSources{ca, cb, kca, kcb, t.b_ctx ? 1 : 0}, cw.db.p, t.out, t.act, nullptr, geo, t.epi};
  static const bool trace = getenv("HB_CONV_TRACE") != nullptr;
  static long long* dtrace = nullptr;
  if (trace) {
    if (!dtrace) HB_CUDA(cudaMalloc(&dtrace, 256 * sizeof(long long)));
    HB_CUDA(cudaMemsetAsync(dtrace, 0, 256 * sizeof(long long), c.stream));
    p.trace = dtrace;
  }
  // uniform chunk width as a template argument (fully unrolled issue loops);
  // mixed-width sources take the generic instantiation
  const bool uni = !cb || kca == kcb;
  const bool gen = geo.par4 || geo.s != 1 || geo.os != 1 || geo.ldo != cw.cout || t.epi.res || t.epi.mu || t.epi.act == 2 ||
                   t.epi.in_elu || t.epi.nco;
  void (*kern)(CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, TcParams, TcLayout, int) =
      gen ? (!uni ? k_conv_tc<0, true> : kcmax == 32 ? k_conv_tc<32, true> : k_conv_tc<16, true>)
          : (!uni ? k_conv_tc<0, false> : kcmax == 32 ? k_conv_tc<32, false> : k_conv_tc<16, false>);
  static int attr_dev = -1;
  if (attr_dev != c.device) {
    for (auto k : {k_conv_tc<0, true>, k_conv_tc<32, true>, k_conv_tc<16, true>, k_conv_tc<0, false>,
                   k_conv_tc<32, false>, k_conv_tc<16, false>})
      HB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_DYN_SMEM));
    attr_dev = c.device;
  }
  const int tiles = tiles0 * ksplit;
  const int grid = std::min(tiles, c.num_sms);
  const int tok = prof_begin(c, PC_CONV);
  if (c.prof_detail)
    c.prof_label = "conv_tc " + std::to_string(B) + "x" + std::to_string(H) + "x" + std::to_string(W) + " " +
                   std::to_string(ca) + "+" + std::to_string(cb) + "->" + std::to_string(cw.cout) + " taps " +
                   std::to_string(NT) + " s" + std::to_string(geo.s) + (geo.par4 ? " par4" : "");
  static const int dbg = getenv("HB_CONV_DEBUG") ? atoi(getenv("HB_CONV_DEBUG")) : 0;
  launch_pdl(c, kern, dim3(grid), dim3(TC_THREADS), smem, mA, mB, wh32, wl32, wh16, wl16, p, lay, dbg);
  if (ksplit > 1) {
    HB_CUDA(cudaGetLastError());
    const size_t n = size_t(B) * H * W * cw.cout;
    const bool dense = geo.os == 1 && geo.ldo == cw.cout && !t.epi.res && !t.epi.mu && t.epi.act != 2 && !t.epi.nco;
    if (dense) {
      const size_t n4 = n / 4;
      launch_pdl(c, k_conv_ksum4, dim3(unsigned(std::min<size_t>((n4 + 255) / 256, size_t(c.num_sms) * 8))), dim3(256),
                 0, ksplit, n4, cw.cout / 4, size_t(H) * W * cw.cout / 4, t.act, reinterpret_cast<const float4*>(ws),
                 reinterpret_cast<const float4*>(cw.db.p), int(t.epi.act == 1), reinterpret_cast<float4*>(t.out));
    } else {
      launch_pdl(c, k_conv_ksum, dim3(unsigned(std::min<size_t>((n + 255) / 256, size_t(c.num_sms) * 8))), dim3(256), 0,
                 ksplit, B, H, W, int(cw.cout), t.act, static_cast<const float*>(ws), static_cast<const float*>(cw.db.p),
                 geo, t.epi, t.out);
    }
  }
  // useful flops: a 4-class transposed conv counts its k^2 real taps and real output channels
  const double flops = geo.par4 ? 2.0 * B * H * W * double(geo.par4_kk) * cw.cin * (t.epi.nco ? t.epi.nco : geo.par4)
                                : 2.0 * B * H * W * double(NT) * cw.cin * cw.cout;
  prof_end(c, PC_CONV, tok, double(B) * H * W * 4.0 * (cw.cin + cw.cout), flops);
  HB_CUDA(cudaGetLastError());
  if (trace) {
    long long h[256];
    HB_CUDA(cudaStreamSynchronize(c.stream));
    HB_CUDA(cudaMemcpy(h, dtrace, sizeof(h), cudaMemcpyDeviceToHost));
    fprintf(stderr,
            "conv_tc %dx%dx%d %d+%d->%d G=%d slots=%d nacc=%d wres=%d stages=%d CG=%d nhbuf=%d box=%d ksplit=%d: it "
            "prod cvt_in mma cvt_out\n",
            B, H, W, ca, cb, cw.cout, lay.G, lay.nslots, lay.nacc, lay.wres, lay.stages, lay.CG, lay.nhbuf,
            lay.box_bytes, ksplit);
    const long long t0 = h[240];
    fprintf(stderr, "  setup %lld, epilogue done %lld %lld %lld %lld, exit %lld (cycles from entry)\n", h[241] - t0,
            h[242] - t0, h[243] - t0, h[244] - t0, h[245] - t0, h[246] - t0);
    for (int i = 0; i < 64 && (h[i * 4] || h[i * 4 + 2]); ++i)
      fprintf(stderr, "  %2d %7lld %7lld %7lld %7lld\n", i, h[i * 4] - t0, h[i * 4 + 1] - t0, h[i * 4 + 2] - t0,
              h[i * 4 + 3] - t0);
  }
  return true;
}

// the classic U-Net's 3x3 / stride 1 / pad 1 conv with bias + ReLU
bool launch_conv_tc(Context& c, const ConvW& cw, int B, const int* act, int H, int W, const float* a, int ca,
                    const float* bsrc, int cb, bool b_ctx, int relu, float* out, const float* pre) {
  TcConv t{};
  t.cw = &cw;
  t.B = B;
  t.Hin = t.H = H;
  t.Win = t.W = W;
  t.a = a;
  t.ca = ca;
  t.bsrc = bsrc;
  t.cb = cb;
  t.b_ctx = b_ctx;
  t.out = out;
  t.act = act;
  t.geo = conv_geo_3x3(H, W, cw.cout);
  t.epi = TcEpi{nullptr, 0, nullptr, nullptr, nullptr, nullptr, relu ? 1 : 0, 0, 0};
  t.epi.pre = pre;  // the batch-broadcast context share of a split encoder-solver layer (bias included)
  t.epi.ldpre = cw.cout;
  return launch_conv_tc_gen(c, t);
}

// stride-1, pad-1 3x3 geometry on an H x W grid, dense output (ldo = cout)
TcGeo conv_geo_3x3(int H, int W, int cout) {
  TcGeo g{};
  g.ntaps = 9;
  g.s = 1;
  g.oy = g.ox = -1;
  g.os = 1;
  g.Ho = H;
  g.Wo = W;
  g.ldo = cout;
  for (int tap = 0; tap < 9; ++tap) {
    g.ty[tap] = tap / 3;
    g.tx[tap] = tap % 3;
  }
  return g;
}

// hi/lo split (3xTF32) of packed [Cout][K] weights, K = ntaps * Cin ordered
// (tap, ci), uploaded to cw.dwh / cw.dwl (host, once per upload)
void conv_tc_upload_packed(ConvW& cw, const std::vector<float>& packed) {
  auto tf32 = [](float x) {  // round to nearest, ties away (cvt.rna.tf32.f32)
    uint32_t u;
    std::memcpy(&u, &x, 4);
    if ((u & 0x7f800000u) != 0x7f800000u) u = (u + 0x1000u) & 0xffffe000u;
    float r;
    std::memcpy(&r, &u, 4);
    return r;
  };
  std::vector<float> hi(packed.size()), lo(packed.size());
  for (size_t i = 0; i < packed.size(); ++i) {
    hi[i] = tf32(packed[i]);
    lo[i] = tf32(packed[i] - hi[i]);
  }
  cw.dwh.ensure(hi.size());
  cw.dwl.ensure(lo.size());
  HB_CUDA(cudaMemcpy(cw.dwh.p, hi.data(), hi.size() * 4, cudaMemcpyHostToDevice));
  HB_CUDA(cudaMemcpy(cw.dwl.p, lo.data(), lo.size() * 4, cudaMemcpyHostToDevice));
}

}  // namespace hb
