// Internal declarations shared by the libhelmgpu translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "../../include/helmgpu.h"

namespace hb {

constexpr int kMaxRestart = 32;  // FGMRES restart cap (device column state)
constexpr int kMaxCoarseIters = 16;

struct HbError {
  int code;
  std::string msg;
};

#define HB_CUDA(x)                                                                                     \
  do {                                                                                                 \
    cudaError_t e_ = (x);                                                                              \
    if (e_ != cudaSuccess)                                                                             \
      throw ::hb::HbError{HB_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)};              \
  } while (0)

// bumped on every device (re)allocation: captured CUDA graphs are keyed on it
extern unsigned long long g_alloc_gen;

// device buffer (RAII)
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) {
    o.p = nullptr;
    o.n = 0;
  }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      n = o.n;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
  ~DBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void ensure(size_t count) {
    if (count <= n) return;
    release();
    HB_CUDA(cudaMalloc(&p, sizeof(T) * (count ? count : 1)));
    n = count;
    ++g_alloc_gen;
  }
};

// Row window of one level's storage (all rows are GLOBAL row indices).  A
// whole-grid level is {0, ny, 0, ny}; a row slab of a distributed grid stores
// rows [row0, row0 + rows) = its owned rows [lo, hi) plus ghost rows, and rows
// outside [0, ny) of the storage are zero-padding (outside the domain).
struct RowWin {
  int row0, rows;  // storage origin and row count (batch stride = nx * rows)
  int lo, hi;      // rows this slab owns (computed / emitted)
};

// device view of one multigrid level (passed by value to kernels)
struct LevelView {
  int nx, ny;        // GLOBAL grid size
  float inv_h2;
  const float2* dM;  // diagonal of the shifted operator M^h (c64)
  const float2* dA;  // diagonal of A^h (c64)
  const float* k2f;  // kappa^2 (fp32)
  const float2* wdi; // damping / diag(M^h) (c64), the Jacobi update factor
  RowWin w;          // storage window; only the row-streaming legs and the Krylov kernels honour a slab window
};

struct Level {
  int nx = 0, ny = 0;  // global size
  int row0 = 0, rows = 0, lo = 0, hi = 0;  // storage window (RowWin); whole grid: 0, ny, 0, ny
  double h = 0;
  std::vector<double> k2, gam;  // host fp64 coefficients (inc/stencil.hpp:169-185 coarsening)
  DBuf<float2> dM, dA, wdi;
  DBuf<double2> dA64;  // level 0: fp64 diagonal of A^h for the restart residual
  DBuf<double2> dM64;  // coarsest level: fp64 diagonal of M^H (multi-CTA coarse GMRES restart)
  DBuf<double2> dinv;  // coarsest level, CoarseSolver::dense: (M^H)^-1 row-major fp64
  DBuf<float2> dMi;    // coarsest level: D^-1 of M^H (c64), the coarse GMRES right preconditioner
  DBuf<float> k2f;
  // V-cycle work buffers [B][N]
  DBuf<float2> f, v, t, x;
  LevelView view() const {
    return LevelView{nx, ny, float(1.0 / (h * h)), dM.p, dA.p, k2f.p, wdi.p, win()};
  }
  RowWin win() const { return RowWin{row0, rows, lo, hi}; }
  size_t N() const { return size_t(nx) * rows; }  // storage nodes per column
};

struct ConvW {
  int cout = 0, cin = 0;
  std::vector<float> w, b;  // host OIHW + bias
  DBuf<float> dw;           // device packed weights [9*cin][cout] (k-major rows), SIMT path
  DBuf<float> db;
  DBuf<float> dwh, dwl;     // tensor-core path: [cout][9*cin] tf32 hi / lo split
  DBuf<float> dwrow;        // row-streaming path (Cout = 16): packed (chunk, kx) blocks, hb_conv_rows.cu
};

struct Net {
  hb_net_cfg cfg{};
  bool set = false;
  std::vector<ConvW> convs;
  int enc1[8], enc2[8], up[8], dec1[8], dec2[8], head = -1;
  bool dirty = true;
  // encoder-solver input layer split (hb_net.cu, net_forward_dev): the context
  // channels are batch-broadcast, so their share of conv(concat(x, ctx)) is
  // computed once per forward (pre_ctx, with the bias) and added per column to
  // the in_ch-channel conv of x (pre_x)
  ConvW pre_ctx, pre_x;
  bool pre_split = false;
  // the same split for the other context-concat convs whose x part runs on
  // k_conv_rows (Cout <= 32): conv index -> (context part, x part)
  std::vector<int> split_of;
  std::vector<ConvW> split_ctx, split_x;
  // the context shares depend only on the weights and the context maps (fixed
  // during a solve): cached per split layer (index split_x.size() = the input
  // layer), recomputed when the key (encode / upload generations, H, W) changes
  std::vector<DBuf<float>> pre_buf;
  std::vector<char> pre_ok;
  unsigned long long pre_key = ~0ull, upload_gen = 0;
};

struct Prof {
  std::string name;
  double ms = 0;
  int64_t launches = 0;
  double bytes = 0, flops = 0;
};

struct Context;
struct SlabState;  // row-slab decomposition of one grid (hb_slab.cu)
struct PaperState;  // the paper's U-Net (hb_paper.cu)
struct TrainState;  // its training state (hb_train.cu)

// ---- multigrid / operator launchers (hb_mg.cu)
void launch_apply(Context& c, const LevelView& L, int which, int B, const int* act, const float2* u, float2* y,
                  const float* uscale);
void launch_jacobi_zero(Context& c, const LevelView& L, float damping, int B, const int* act, const float2* f,
                        const float* fscale, float2* v);
void launch_jacobi_sweep(Context& c, const LevelView& L, float damping, int B, const int* act, const float2* v,
                         const float2* f, const float* fscale, float2* out);
void launch_residual_restrict(Context& c, const LevelView& L, int offset, int B, const int* act, const float2* v,
                              const float2* f, const float* fscale, float2* fc);
void launch_prolong_add(Context& c, const LevelView& Lf, int cnx, int cny, int offset, int B, const int* act,
                        const float2* vc, float2* v);
void launch_restrict_plain(Context& c, int nx, int ny, int offset, int B, const float2* fine, float2* coarse);
void launch_coarse_dense(Context& c, const Level& L, int B, const int* act, const float2* f, float2* x);
// coarsest GMRES with one thread-block cluster per column (hb_coarse_cluster.cu); false if not applicable
bool launch_coarse_cluster(Context& c, const LevelView& L, int iters, int B, int slot, const int* act, const float2* f,
                           float2* x);
void launch_coarse_gmres(Context& c, const LevelView& L, int iters, int B, const int* act, const float2* f,
                         float2* x, float2* scratch);
// coarsest GMRES(iters) with D^-1 on the multi-CTA Krylov kernels (hb_krylov.cu), large coarse grids
void coarse_krylov_solve(Context& c, const Level& L, int iters, int B, int slot, const float2* f, float2* x);
// register-resident variant for <= 1024-node coarse grids, iters <= 10 (hb_coarse_small.cu); false if not applicable
// full-row-warp V-cycle legs for 64 / 128-wide whole-grid levels (hb_mg_rowwarp.cu); false: not applicable
bool launch_down_row(Context& c, const LevelView& L, float damping, int offset, int B, const int* act,
                     const float2* f, const float* fscale, float2* fc);
bool launch_up_row(Context& c, const LevelView& L, float damping, int offset, int B, const int* act, const float2* f,
                   const float* fscale, const float2* vc, float2* z);
bool launch_coarse_small(Context& c, const LevelView& L, int iters, int B, const int* act, const float2* f,
                         float2* x);
// fused down/up legs (nu1 = nu2 = 1)
void launch_down_fused(Context& c, const LevelView& L, float damping, int offset, int B, const int* act,
                       const float2* f, const float* fscale, const float2* e0, float2* fc);
void launch_up_fused(Context& c, const LevelView& L, float damping, int offset, int cnx, int cny, int B,
                     const int* act, const float2* f, const float* fscale, const float2* e0, const float2* vc,
                     float2* z);
// tensor-core conv (hb_conv_tc.cu, hb_conv_rows.cu)
void conv_tc_prepare(ConvW& cw);
// generalised tensor-core convolution (hb_conv_tc.cu): any tap set (<= 25),
// input stride 1 | 2, output scatter / channel slice, fused bias [+ residual]
// [+ BN eval] [+ ReLU | ELU] epilogue, optional ELU on the inputs
constexpr int TC_MAX_TAPS = 25;  // up to a 5x5 kernel

// Geometry of one implicit-GEMM launch.  Output tile grid [H][W] (tiles of bh
// x bw pixels); tap t of output pixel (y, x) reads the input pixel at
// (y * s + oy + ty[t], x * s + ox + tx[t]) -- inside the tile's halo box of
// boxh x boxw pixels whose origin is (y0 * s + oy, x0 * s + ox).  Tile-grid
// pixel (y, x) is stored at output pixel (y * os + py, x * os + px) of [Ho][Wo]
// with a row stride of ldo floats (a parity class of a stride-2 transposed
// convolution: os = 2; a channel slice of a concatenation: ldo > cout).
struct TcGeo {
  int ntaps, s, oy, ox, boxh, boxw;
  int os, py, px, Ho, Wo, ldo;
  int ty[TC_MAX_TAPS], tx[TC_MAX_TAPS];
  // par4 > 0: the four output parity classes of a stride-2 transposed conv in one
  // GEMM -- output channel block q = c / par4 (par4 channels each) is stored at
  // output pixel (2y + (q >> 1), 2x + (q & 1)), channel c % par4 (os must be 2)
  int par4 = 0;
  int par4_kk = 0;  // par4: kernel taps k^2 of the transposed conv (useful flops: zero-weight taps not counted)
};
// epilogue: y = act(BN(x + bias [+ res])), BN in eval form ((t - mu) is) g + be
// (inc/autodiff.hpp:289-296); act 0 none, 1 ReLU, 2 ELU; in_elu: ELU applied to
// the input values as they are loaded (the paper net's up path)
struct TcEpi {
  const float* res;
  int ldres;
  const float *mu, *is, *g, *be;
  int act, in_elu;
  int nco;  // output channels actually stored (< cout when cout was padded to a multiple of 16); 0: all
  const float* pre = nullptr;  // batch-broadcast per-pixel term [Ho][Wo][ldpre] replacing the bias (context share)
  int ldpre = 0;
};

// one launch: weights cw (dwh / dwl [cout][ntaps * cin], db bias), input a
// [B][Hin][Win][ca] (+ b [.][Hin][Win][cb], batch-broadcast when b_ctx), output
// tile grid H x W
struct TcConv {
  const ConvW* cw;
  int B, Hin, Win, H, W;
  const float *a, *bsrc;
  int ca, cb;
  bool b_ctx;
  TcGeo geo;
  TcEpi epi;
  float* out;
  const int* act;
};
bool launch_conv_tc_gen(Context& c, const TcConv& t);
TcGeo conv_geo_3x3(int H, int W, int cout);
void conv_tc_upload_packed(ConvW& cw, const std::vector<float>& packed);
void conv_rows_prepare(ConvW& cw);
bool launch_conv_rows(Context& c, const ConvW& cw, int B, const int* act, int H, int W, const float* a, int ca,
                      const float* bsrc, int cb, bool b_ctx, int relu, float* out,
                      const float* pre = nullptr);
// cin (12 | 16 | 20) -> 2 3x3 head (zero padding 1, bias, no activation) as
// column strips (k_conv_cols, hb_net.cu); w host [9][cin][2], b host [2]
bool launch_head_cols(Context& c, int cin, int B, int H, int W, const float* x, const float* w, const float* b,
                      float* y);
bool launch_conv_tc(Context& c, const ConvW& cw, int B, const int* act, int H, int W, const float* a, int ca,
                    const float* bsrc, int cb, bool b_ctx, int relu, float* out, const float* pre = nullptr);
// row-streaming legs, zero initial guess (hb_mg_stream.cu)
// cw: storage window of the coarse field (down: emitted rows [cw.lo, cw.hi); up: vc)
void launch_down_stream(Context& c, const LevelView& L, const RowWin& cw, float damping, int offset, int B,
                        const int* act, const float2* f, const float* fscale, const float2* e0, float2* fc,
                        float2* vpre = nullptr);
void launch_up_stream(Context& c, const LevelView& L, float damping, int offset, int cnx, int cny, const RowWin& cw,
                      int B, const int* act, const float2* f, const float* fscale, const float2* e0, const float2* vc,
                      float2* z, const float2* vpre = nullptr);
// cp.async-staged variants (hb_mg_staged.cu), same contracts; wd: form wD^-1 from D
void launch_down_staged(Context& c, const LevelView& L, const RowWin& cw, float damping, int offset, int B,
                        const int* act, const float2* f, const float* fscale, const float2* e0, bool wd, float2* fc,
                        float2* vpre = nullptr);
void launch_up_staged(Context& c, const LevelView& L, float damping, int offset, int cnx, int cny, const RowWin& cw,
                      int B, const int* act, const float2* f, const float* fscale, const float2* e0, const float2* vc,
                      bool wd, float2* z, const float2* vpre = nullptr);
// network pack / unpack (hb_net.cu)
void launch_pack_input(Context& c, const LevelView& L, double h2, int B, const int* act, const float2* r,
                       const float* rscale, float* x /*NHWC, 3 ch*/);
void launch_unpack_output(Context& c, int N, int B, const int* act, const float* y /*NHWC 2ch*/, float2* e);
// e = base + y (NHWC 2ch -> c64); base may alias e
void launch_unpack_add(Context& c, int N, int B, const int* act, const float* y, const float2* base, float2* e);
// out = s f - Op u  (Op = the level operator whose diagonal is L.dM), hb_mg.cu
void launch_residual(Context& c, const LevelView& L, int B, const int* act, const float2* u, const float2* f,
                     const float* fscale, float2* out);

// ---- Krylov (hb_krylov.cu)
struct ColState;
// limits: optional DEVICE array of per-column iteration limits (0 = max_iters)
void krylov_alloc(Context& c, int B, int m, int hist_cap, const int* limits = nullptr);
// gsum != nullptr: row-slab split mode (fold the slab's partial sums into
// gsum[B][kMaxDots] and stop; the *_finish launchers run the scalar part on the
// slab-summed gsum)
constexpr int kMaxDots = 2 * kMaxRestart + 1;
void launch_fg_restart(Context& c, int B, const double2* b, const double2* x, float2* V0, int hist_cap,
                       double rel_tol, int max_iters, double2* gsum = nullptr);
void launch_fg_adots(Context& c, int B, int j, const float2* Zj, float2* w, const float2* V, double2* gsum = nullptr);
void launch_fg_update(Context& c, int B, int j, int m, const float2* w, float2* V, int hist_cap, double rel_tol,
                      int max_iters, double2* gsum = nullptr);
void launch_fg_restart_finish(Context& c, int B, const double2* gsum, int hist_cap, double rel_tol, int max_iters);
void launch_fg_adots_finish(Context& c, int B, int j, const double2* gsum);
void launch_fg_update_finish(Context& c, int B, int j, int m, const double2* gsum, int hist_cap, double rel_tol,
                             int max_iters);
void launch_fg_finalize(Context& c, int B, int m, const float2* Z, double2* x);
// non-flexible (standard right-preconditioned) GMRES: u = V y, fin[b] = k > 0; then x += z
void launch_fg_finalize_v(Context& c, int B, const float2* V, float2* u, int* fin);
void launch_fg_add_to_x(Context& c, int B, const int* fin, const float2* z, double2* x);
// true block FGMRES (hb_block.cu): p <= 16 right-hand sides in one block Krylov space
void block_fgmres_dev(Context& c, int kind, int p, int m, int max_iters, double rel_tol, const double2* dB,
                      double2* dX, double* hist_out, int hist_stride, int* hist_len_out, int* iters_out,
                      uint8_t* conv_out, uint8_t* brk_out);
void krylov_report(Context& c, int B, double* hist, int hist_stride, int* hist_len, int* iters, uint8_t* conv,
                   uint8_t* brk);

// ---- profiling / launch accounting
int prof_begin(Context& c, int cls);
void prof_end(Context& c, int cls, int token, double bytes, double flops);

enum ProfClass {
  PC_STENCIL = 0,
  PC_SMOOTH,
  PC_DOWN,
  PC_UP,
  PC_TRANSFER,
  PC_COARSE,
  PC_KRYLOV_DOTS,
  PC_KRYLOV_UPDATE,
  PC_KRYLOV_RESTART,
  PC_KRYLOV_FINAL,
  PC_CONV,
  PC_NETIO,
  PC_COUNT
};

struct Context {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t stream_own = nullptr;  // the context's own stream while an in-process slab group lends it one
  cudaStream_t stream2 = nullptr;  // second branch for split V-cycles
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_at_coarse = nullptr;  // recorded when a V-cycle reaches its coarsest level
  int num_sms = 148;
  size_t l2_bytes = size_t(126) << 20;
  std::string err;
  // problem
  bool has_problem = false;
  int nx = 0, ny = 0;
  double h = 0, omega = 0, klo = 0, khi = 0;
  std::vector<double> k2, gam;
  // hierarchy
  bool has_hier = false;
  hb_vcycle_cfg vc{};
  std::vector<std::unique_ptr<Level>> levels;
  int batch_cap = 0;
  // nets: slot 0 solver, slot 1 encoder
  Net nets[2];
  // generic scratch
  DBuf<float2> scratch_c64;
  DBuf<double2> io_a, io_b;  // c128 staging
  DBuf<float2> io_f, io_g;   // c64 staging
  DBuf<int> act_all;         // all-ones activity flags
  // Krylov
  DBuf<char> kstate;         // ColState[B]
  DBuf<double2> kpart;       // per-CTA partials
  DBuf<int> kfin;            // non-flexible finalize: columns with k > 0
  DBuf<double> khist;        // [B][hist_cap]
  DBuf<int> kact;            // per-column: active in the current inner step
  DBuf<int> klimit;          // per-column iteration limits (training-pair generation)
  DBuf<float> kscale;        // per-column: scale of the current V_j
  DBuf<unsigned> kticket;    // per-column last-CTA counters
  DBuf<int> kcount;          // number of unfrozen columns (host-visible after restart)
  DBuf<float2> kV, kZ, kW;   // [B][m+1][N], [B][m][N], [B][N]
  DBuf<double2> kX, kB;      // c128 solution / rhs when called with host buffers
  struct KrylovBufs {        // coarsest-level GMRES on the Krylov kernels, one set per half-batch stream
    DBuf<char> state;
    DBuf<double2> part;
    DBuf<double> hist;
    DBuf<int> act, count;
    DBuf<float> scale;
    DBuf<unsigned> ticket;
    DBuf<float2> V, Z, W;
    DBuf<double2> b, x;
  } kcoarse[2];
  int k_B = 0, k_m = 0, k_hist = 0;
  int* h_count = nullptr;    // pinned
  // preconditioner staging (context-owned so captured graphs see stable pointers)
  DBuf<float> pc_io, cn_io;
  DBuf<float2> pc_e0, pc_res;
  // options
  double prof_scale = 1.0;  // active-column fraction while profiling (eager) FGMRES steps
  bool opt_fused = true, opt_graphs = true, opt_small_coarse = true, opt_split = true, opt_tc_conv = true, opt_stream = true, opt_conv_ksplit = true,
       opt_coarse_reg = true, opt_row_legs = true, opt_ctx_pre = true, opt_tconv_par4 = true,
       opt_conv_rows = true, opt_lean_legs = true, opt_coarse_krylov = true, opt_coarse_cluster = true, opt_basis_wave = true, opt_pdl = true, opt_stream_e0 = true, opt_vpre = true, opt_wgrad_blk = true, opt_small_pw = true, opt_conv_cols = true;
  int dbg_skip = 0;  // diagnostics only (tools/debug/c0_marginal.py): skip kernel classes, results invalid
  int opt_staged_legs = 2;  // cp.async-staged legs: 0 off, 1 on, 2 by working-set size
  int opt_legs_wd = 2;  // Jacobi factor in the legs: 0 stored wD^-1, 1 from D, 2 by working-set size
  // captured FGMRES cycle graphs
  struct GraphEntry {
    unsigned long long gen;
    int kind, B, m, cap, max_iters;
    double tol;
    const void *dB, *dX;
    cudaGraphExec_t exec;
    int64_t launches;
    bool flexible;
  };
  std::vector<GraphEntry> graphs;
  // net activations
  DBuf<float> net_act;       // arena
  DBuf<float> conv_ws;       // split-K partial sums of the tensor-core conv
  std::vector<DBuf<float>> ctx_maps;  // encoder context per level (NHWC)
  bool ctx_valid = false;
  // profiling
  bool prof_on = false;
  std::vector<Prof> prof;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_pending;
  // per-launch detail (label set by the launcher just before prof_end)
  bool prof_detail = false;
  std::string prof_label;
  struct DetailRec {
    std::string label;
    size_t token;
    double ms, bytes, flops;
  };
  std::vector<DetailRec> detail, detail_done;
  int64_t launches = 0;
  // row-slab decomposition (null: whole grid)
  std::shared_ptr<SlabState> slab;
  // the paper's U-Net (inc/unet.hpp:139-257); when active it is the network of M_JU / M_VU
  std::shared_ptr<PaperState> paper;
  std::shared_ptr<TrainState> train;  // device parameters, tape and ADAM moments while training
  unsigned long long prob_gen = 0;  // bumped by hb_set_problem
  unsigned long long ctx_gen = 0;   // bumped by every encoder forward (new context maps)
};

// Launch with programmatic dependent launch (PDL, sm_90+): the kernel may be
// scheduled while its stream predecessor drains, hiding the launch gap of the
// latency-bound FGMRES chain.  Every kernel launched this way calls
// pdl_wait() (hb_common.cuh) before it touches memory its predecessor writes.
template <typename... KArgs, typename... Args>
inline void launch_pdl(Context& c, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c.stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = c.opt_pdl ? 1 : 0;
  HB_CUDA(cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...));
}

void ensure_batch(Context& c, int B);
// coarsest-level solve on a whole-grid coarsest level (hb_api.cu)
void coarsest_solve(Context& c, int B, int c0, const int* act, const float2* f, float2* out);
void fill_level_device(Level& L, double omega, double alpha, double beta, double damping, bool fp64A, bool fp64M);
void require_whole(const Context& c);  // throws for a row-slab context on whole-grid entry points
// V-cycle driver (hb_api.cu)
void vcycle(Context& c, int B, const int* act, const float2* f0, const float* fscale, const float2* e0, float2* z);
void precond_apply_dev(Context& c, int kind, int B, const int* act, const float2* r, const float* rscale,
                       float2* z);
// network forward on device (hb_net.cu): x NHWC [B][H][W][in_ch] -> y NHWC [B][H][W][2]
void net_forward_dev(Context& c, int slot, int B, const int* act, int H, int W, const float* x, float* y);
void encoder_forward_dev(Context& c, int H, int W, const float* k2f);
void net_upload(Context& c, int slot);
// paper U-Net (hb_paper.cu): e = net(h^2 s r, kappa^2, gamma) [+ base]
bool paper_active(const Context& c);
void paper_deactivate(Context& c);
void paper_infer(Context& c, int B, const int* act, const float2* r, const float* rscale, const float2* base,
                 float2* e);

}  // namespace hb
