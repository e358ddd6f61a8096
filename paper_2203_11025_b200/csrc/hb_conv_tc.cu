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
#include <cstdlib>
#include <cstring>
#include <vector>

#include "hb_common.cuh"
#include "hb_internal.h"

namespace hb {

namespace {

constexpr int TC_THREADS = 320;
constexpr int TC_MAX_STAGES = 8;
constexpr int TC_M = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// UMMA shared-memory descriptor, K-major, SWIZZLE_128B (2) or SWIZZLE_64B (4):
// start >> 4 [0,14), LBO [16,30) (unused for swizzled K-major), SBO = 8 rows *
// row bytes >> 4 [32,46), version 1 [46,48), layout [61,64)
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, int row_bytes) {
  uint64_t d = 0;
  d |= uint64_t((saddr & 0x3FFFF) >> 4);
  d |= uint64_t(1) << 16;
  d |= uint64_t((8 * row_bytes) >> 4) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(row_bytes == 128 ? 2 : 4) << 61;
  return d;
}
__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

struct TcSources {
  int ca, cb;         // channels of source a, b (b may be 0)
  int kca, kcb;       // K chunk (16 | 32) per source
  int b_is_ctx;       // source b is a batch-broadcast 3-D map (encoder context)
};

struct TcParams {
  int B, H, W, cout, relu;
  int bw, bh;         // pixel box of one M tile
  TcSources s;
  const float* bias;
  float* out;
  const int* act;
};

// Persistent CTA (one per SM), 10 warps:
//   w0 TMA producer | w1 MMA issuer | w2..w5 split A in smem | w6..w9 epilogue.
// The smem ring runs continuously across the CTA's M tiles; the accumulator is
// double-buffered in TMEM (2 x N columns), so tile t's epilogue (TMEM -> bias,
// ReLU -> NHWC) overlaps tile t+1's MMAs.
__global__ void __launch_bounds__(TC_THREADS, 1)
    k_conv_tc(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
              const __grid_constant__ CUtensorMap mapWh32, const __grid_constant__ CUtensorMap mapWl32,
              const __grid_constant__ CUtensorMap mapWh16, const __grid_constant__ CUtensorMap mapWl16, TcParams p,
              int stages, int kcmax, int G, int dbg) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ uint64_t bar_full[TC_MAX_STAGES], bar_cvt[TC_MAX_STAGES], bar_empty[TC_MAX_STAGES];
  __shared__ uint64_t bar_tfull[2], bar_tempty[2];
  __shared__ uint32_t tmem_slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int N = p.cout;
  const int tiles_x = p.W / p.bw, tiles_y = p.H / p.bh;
  const int ntiles = p.B * tiles_x * tiles_y;
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // a stage holds G consecutive K chunks: A[G], A_lo[G], W_hi[G], W_lo[G]
  const int a_bytes = TC_M * kcmax * 4, w_bytes = N * kcmax * 4;
  const int stage_bytes = G * (2 * a_bytes + 2 * w_bytes);
  auto sA = [&](int s, int g) { return base + s * stage_bytes + g * a_bytes; };
  auto sAl = [&](int s, int g) { return base + s * stage_bytes + (G + g) * a_bytes; };
  auto sWh = [&](int s, int g) { return base + s * stage_bytes + 2 * G * a_bytes + g * w_bytes; };
  auto sWl = [&](int s, int g) { return base + s * stage_bytes + 2 * G * a_bytes + (G + g) * w_bytes; };
  const int cin = p.s.ca + p.s.cb;
  const int nchunk_a = p.s.ca / p.s.kca, nchunk_b = p.s.cb ? p.s.cb / p.s.kcb : 0;
  const int per_tap = nchunk_a + nchunk_b;
  const int nk = 9 * per_tap;
  const int nst = (nk + G - 1) / G;  // stage iterations per tile
  uint32_t ncols = 32;
  while (ncols < uint32_t(2 * N)) ncols <<= 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&bar_full[s], 1);
      mbar_init(&bar_cvt[s], 128);
      mbar_init(&bar_empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&bar_tfull[a], 1);
      mbar_init(&bar_tempty[a], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tmem_slot;

  auto tile_coords = [&](int tile, int& b, int& y0, int& x0) {
    b = tile / (tiles_x * tiles_y);
    y0 = ((tile / tiles_x) % tiles_y) * p.bh;
    x0 = (tile % tiles_x) * p.bw;
  };

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int s = 0;
      uint32_t ph = 0;
      int it = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        int b, y0, x0;
        tile_coords(tile, b, y0, x0);
        const bool skip = p.act && !p.act[b];
        if (skip) continue;
        for (int st = 0; st < nst; ++st, ++it) {
          if (it >= stages) mbar_wait(&bar_empty[s], ph ^ 1);
          const int k0 = st * G, k1 = min(nk, k0 + G);
          uint32_t bytes = 0;
          for (int kb = k0; kb < k1; ++kb) {
            const int r = kb % per_tap;
            const int kc = (r >= nchunk_a) ? p.s.kcb : p.s.kca;
            bytes += uint32_t(TC_M * kc * 4 + 2 * N * kc * 4);
          }
          if (dbg & 8) bytes = 0;
          mbar_expect_tx(&bar_full[s], bytes);
          for (int kb = k0; kb < k1; ++kb) {
            const int g = kb - k0;
            const int tap = kb / per_tap, r = kb % per_tap;
            const bool srcb = r >= nchunk_a;
            const int kc = srcb ? p.s.kcb : p.s.kca;
            const int ci0 = srcb ? (r - nchunk_a) * kc : r * kc;
            const int kglob = tap * cin + (srcb ? p.s.ca : 0) + ci0;
            const int ky = tap / 3, kx = tap % 3;
            if (dbg & 8) continue;
            if (!srcb)
              tma_load_4d(sA(s, g), &mapA, &bar_full[s], ci0, x0 + kx - 1, y0 + ky - 1, b);
            else
              tma_load_4d(sA(s, g), &mapB, &bar_full[s], ci0, x0 + kx - 1, y0 + ky - 1, p.s.b_is_ctx ? 0 : b);
            tma_load_2d(sWh(s, g), kc == 32 ? &mapWh32 : &mapWh16, &bar_full[s], kglob, 0);
            tma_load_2d(sWl(s, g), kc == 32 ? &mapWl32 : &mapWl16, &bar_full[s], kglob, 0);
          }
          if (++s == stages) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(TC_M >> 4) << 24);
      int s = 0;
      uint32_t ph = 0;
      int tl = 0;  // local tile counter (accumulator buffer = tl & 1)
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        int b, y0, x0;
        tile_coords(tile, b, y0, x0);
        if (p.act && !p.act[b]) continue;
        const int acc = tl & 1;
        const uint32_t tmem_d = tmem_base + uint32_t(acc * N);
        if (tl >= 2) mbar_wait(&bar_tempty[acc], ((tl >> 1) - 1) & 1);  // epilogue drained this buffer
        tc_fence_after();
        for (int st = 0; st < nst; ++st) {
          mbar_wait(&bar_cvt[s], ph);
          tc_fence_after();
          const int k0 = st * G, k1 = min(nk, k0 + G);
          for (int kb = k0; kb < k1; ++kb) {
            const int g = kb - k0;
            const int r = kb % per_tap;
            const int kc = (r >= nchunk_a) ? p.s.kcb : p.s.kca;
            const int rowb = kc * 4;
            const uint32_t a = smem_u32(sA(s, g)), al = smem_u32(sAl(s, g));
            const uint32_t wh = smem_u32(sWh(s, g)), wl = smem_u32(sWl(s, g));
            for (int k = 0; k < ((dbg & 1) ? 0 : kc / 8); ++k) {
              const uint32_t off = k * 32;
              const uint64_t dA = umma_desc(a + off, rowb), dAl = umma_desc(al + off, rowb);
              const uint64_t dWh = umma_desc(wh + off, rowb), dWl = umma_desc(wl + off, rowb);
              umma_tf32(tmem_d, dA, dWh, idesc, (kb | k) ? 1u : 0u);
              umma_tf32(tmem_d, dA, dWl, idesc, 1u);
              umma_tf32(tmem_d, dAl, dWh, idesc, 1u);
            }
          }
          umma_commit(&bar_empty[s]);
          if (++s == stages) {
            s = 0;
            ph ^= 1;
          }
        }
        umma_commit(&bar_tfull[acc]);
        ++tl;
      }
    }
  } else if (warp < 6) {
    // ---------------- warps 2..5: split each A stage into tf32 hi / lo in place
    const int ct = threadIdx.x - 64;
    int s = 0;
    uint32_t ph = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      int b, y0, x0;
      tile_coords(tile, b, y0, x0);
      if (p.act && !p.act[b]) continue;
      for (int st = 0; st < nst; ++st) {
        mbar_wait(&bar_full[s], ph);
        const int k0 = st * G, k1 = min(nk, k0 + G);
        for (int kb = k0; kb < k1; ++kb) {
          const int g = kb - k0;
          const int r = kb % per_tap;
          const int kc = (r >= nchunk_a) ? p.s.kcb : p.s.kca;
          float4* a4 = reinterpret_cast<float4*>(sA(s, g));
          float4* l4 = reinterpret_cast<float4*>(sAl(s, g));
          const int n4 = (dbg & 2) ? 0 : TC_M * kc / 4;
          // hi = x with the 13 low mantissa bits cleared (a tf32 value), lo = x - hi
          // (exact in fp32; the MMA reads its top 10 mantissa bits) -- integer
          // mask + one FADD per element, no cvt (conversion-pipe bound otherwise)
          for (int i = ct; i < n4; i += 128) {
            const float4 x = a4[i];
            float4 hi, lo;
            hi.x = __uint_as_float(__float_as_uint(x.x) & 0xffffe000u);
            hi.y = __uint_as_float(__float_as_uint(x.y) & 0xffffe000u);
            hi.z = __uint_as_float(__float_as_uint(x.z) & 0xffffe000u);
            hi.w = __uint_as_float(__float_as_uint(x.w) & 0xffffe000u);
            lo.x = x.x - hi.x;
            lo.y = x.y - hi.y;
            lo.z = x.z - hi.z;
            lo.w = x.w - hi.w;
            a4[i] = hi;
            l4[i] = lo;
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor-core reads
        mbar_arrive(&bar_cvt[s]);
        if (++s == stages) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else {
    // ---------------- warps 6..9: epilogue; warp owns TMEM lanes 32*(warp%4) .. +31 (= tile pixel rows)
    const int q = warp & 3;
    int tl = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      int b, y0, x0;
      tile_coords(tile, b, y0, x0);
      if (p.act && !p.act[b]) continue;
      const int acc = tl & 1;
      mbar_wait(&bar_tfull[acc], (tl >> 1) & 1);
      tc_fence_after();
      const int row = 32 * q + lane;
      const int yy = row / p.bw, xx = row % p.bw;
      float* orow = p.out + ((size_t(b) * p.H + (y0 + yy)) * p.W + (x0 + xx)) * N;
      for (int c0 = 0; c0 < ((dbg & 4) ? 0 : N); c0 += 16) {
        uint32_t v[16];
        const uint32_t taddr = tmem_base + (uint32_t(32 * q) << 16) + uint32_t(acc * N + c0);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        float o[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float x = __uint_as_float(v[i]) + __ldg(p.bias + c0 + i);
          o[i] = p.relu ? fmaxf(x, 0.f) : x;
        }
#pragma unroll
        for (int i = 0; i < 16; i += 4)
          *reinterpret_cast<float4*>(orow + c0 + i) = make_float4(o[i], o[i + 1], o[i + 2], o[i + 3]);
      }
      tc_fence_before();
      mbar_arrive(&bar_tempty[acc]);
      ++tl;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(ncols));
  }
}

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

// weight map: [Cout][K] fp32 as 2-D (K, Cout); box (kc, Cout)
CUtensorMap w_map(const float* ptr, int cout, int K, int kc) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {cuuint64_t(K), cuuint64_t(cout)};
  const cuuint64_t strides[1] = {cuuint64_t(K) * 4};
  const cuuint32_t box[2] = {cuuint32_t(kc), cuuint32_t(cout)};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides, box,
                                  es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                  kc == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw HbError{HB_ERR_CUDA, "cuTensorMapEncodeTiled(w) failed " + std::to_string(int(r))};
  return m;
}

}  // namespace

// hi/lo split of the packed [Cout][9*Cin] weights (host, once per upload)
void conv_tc_prepare(ConvW& cw) {
  const int K = 9 * cw.cin;
  std::vector<float> hi(size_t(cw.cout) * K), lo(size_t(cw.cout) * K);
  auto tf32 = [](float x) {  // round to nearest, ties away (cvt.rna.tf32.f32)
    uint32_t u;
    std::memcpy(&u, &x, 4);
    if ((u & 0x7f800000u) != 0x7f800000u) u = (u + 0x1000u) & 0xffffe000u;
    float r;
    std::memcpy(&r, &u, 4);
    return r;
  };
  for (int co = 0; co < cw.cout; ++co)
    for (int tap = 0; tap < 9; ++tap)
      for (int ci = 0; ci < cw.cin; ++ci) {
        const float w = cw.w[(size_t(co) * cw.cin + ci) * 9 + tap];
        const float h = tf32(w);
        hi[size_t(co) * K + size_t(tap) * cw.cin + ci] = h;
        lo[size_t(co) * K + size_t(tap) * cw.cin + ci] = tf32(w - h);
      }
  cw.dwh.ensure(hi.size());
  cw.dwl.ensure(lo.size());
  HB_CUDA(cudaMemcpy(cw.dwh.p, hi.data(), hi.size() * 4, cudaMemcpyHostToDevice));
  HB_CUDA(cudaMemcpy(cw.dwl.p, lo.data(), lo.size() * 4, cudaMemcpyHostToDevice));
}

static bool tc_ok_channels(int c) { return c > 0 && c % 16 == 0; }

// returns false when the shape is not supported by the tensor-core path
bool launch_conv_tc(Context& c, const ConvW& cw, int B, const int* act, int H, int W, const float* a, int ca,
                    const float* bsrc, int cb, bool b_ctx, int relu, float* out) {
  if (!c.opt_tc_conv) return false;
  if (!tc_ok_channels(ca) || (cb && !tc_ok_channels(cb))) return false;
  if (cw.cout % 16 || cw.cout > 256 || cw.cout < 16) return false;
  const int bw = W < TC_M ? W : TC_M;
  const int bh = TC_M / bw;
  if (W % bw || H % bh || bw * bh != TC_M || !cw.dwh.p) return false;
  const int kca = ca % 32 == 0 ? 32 : 16, kcb = cb ? (cb % 32 == 0 ? 32 : 16) : 32;
  const CUtensorMap mA = act_map(a, B, H, W, ca, kca, bw, bh);
  const CUtensorMap mB = cb ? act_map(bsrc, b_ctx ? 1 : B, H, W, cb, kcb, bw, bh) : mA;
  const int K = 9 * cw.cin;
  const CUtensorMap wh32 = w_map(cw.dwh.p, cw.cout, K, 32), wl32 = w_map(cw.dwl.p, cw.cout, K, 32);
  const CUtensorMap wh16 = w_map(cw.dwh.p, cw.cout, K, 16), wl16 = w_map(cw.dwl.p, cw.cout, K, 16);
  TcParams p{B, H, W, cw.cout, relu, bw, bh, TcSources{ca, cb, kca, kcb, b_ctx ? 1 : 0}, cw.db.p, out, act};
  const int kcmax = (kca == 32 || (cb && kcb == 32)) ? 32 : 16;
  const int chunk_bytes = 2 * TC_M * kcmax * 4 + 2 * cw.cout * kcmax * 4;
  // group K chunks per stage so a stage moves >= ~48 KB (latency-bound otherwise)
  static const int g_env = getenv("HB_CONV_G") ? atoi(getenv("HB_CONV_G")) : 0;
  const int G = g_env > 0 ? g_env : std::max(1, std::min(9, (48 * 1024) / chunk_bytes));
  const int stage_bytes = G * chunk_bytes;
  int stages = TC_MAX_STAGES;
  while (stages > 2 && stages * stage_bytes + 1024 > 220 * 1024) --stages;
  const size_t smem = size_t(stages) * stage_bytes + 1024;
  static int attr_dev = -1;
  if (attr_dev != c.device) {
    HB_CUDA(cudaFuncSetAttribute(k_conv_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    attr_dev = c.device;
  }
  const int tiles = B * (H / bh) * (W / bw);
  const int grid = std::min(tiles, c.num_sms);
  const int tok = prof_begin(c, PC_CONV);
  if (c.prof_detail)
    c.prof_label = "conv_tc " + std::to_string(B) + "x" + std::to_string(H) + "x" + std::to_string(W) + " " +
                   std::to_string(ca) + "+" + std::to_string(cb) + "->" + std::to_string(cw.cout);
  static const int dbg = getenv("HB_CONV_DEBUG") ? atoi(getenv("HB_CONV_DEBUG")) : 0;
  k_conv_tc<<<grid, TC_THREADS, smem, c.stream>>>(mA, mB, wh32, wl32, wh16, wl16, p, stages, kcmax, G, dbg);
  prof_end(c, PC_CONV, tok, double(B) * H * W * 4.0 * (cw.cin + cw.cout),
           2.0 * B * H * W * 9.0 * cw.cin * cw.cout);
  HB_CUDA(cudaGetLastError());
  return true;
}

}  // namespace hb
