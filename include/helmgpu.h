/*
 * helmgpu.h -- C ABI of the B200-native (sm_100a) hot path of arXiv 2203.11025:
 * flexible GMRES on the heterogeneous 2-D Helmholtz operator, preconditioned by
 * a shifted-Laplacian multigrid V-cycle combined with a U-Net (coarse solver or
 * deflation guess), optionally with an encoder network.
 *
 * Plain C, plain pointers and sizes.  Host buffers are caller-owned, device
 * buffers are library-owned.  One hb_ctx per GPU, used by one host thread.
 * Every call returns 0 on success, or a negative status with the message in
 * hb_last_error(ctx).  Complex fields are interleaved (re, im) doubles
 * (std::complex<double>, inc/grid.hpp:11), row-major iy*nx+ix
 * (inc/grid.hpp:22-36); batches are contiguous [batch][ny][nx].
 *
 * Reference interfaces each entry point replaces (inc/ =
 * /root/reference/proj/include/helmbench/):
 *   hb_set_problem      make_problem / HelmholtzProblem        inc/grid.hpp:121-141
 *   hb_build_hierarchy  MultigridHierarchy(problem, VCycleConfig) inc/multigrid.hpp:13-21,72-86
 *   hb_operator_apply   StencilOperator::apply                 inc/stencil.hpp:44-60
 *   hb_jacobi           StencilOperator::jacobi                inc/stencil.hpp:78-92
 *   hb_restrict/prolong restrict_field / prolong_field         inc/stencil.hpp:119-165
 *   hb_set_net / hb_load_conv / hb_init_net_he
 *                       NetworkWeights + build_unet/build_encoder (classic U-Net)
 *                                                              inc/unet.hpp:10-33,171-257
 *   hb_net_forward      unet_forward / solver_forward          inc/unet.hpp:261-295
 *   hb_precond_apply    Preconditioner::apply (M_V / coarse-net cycle / M_VU)
 *                                                              inc/precond.hpp:14-27,35-53,143-165
 *   hb_fgmres           block_fgmres (device-resident)         inc/krylov.hpp:83-267
 */
#ifndef HELMGPU_H_
#define HELMGPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

typedef struct hb_ctx hb_ctx;

#define HB_OK 0
#define HB_ERR_ARG (-1)     /* std::invalid_argument in the reference */
#define HB_ERR_CUDA (-2)    /* device / runtime failure */
#define HB_ERR_STATE (-3)   /* call order (e.g. no problem set) */
#define HB_ERR_NUMERIC (-4) /* std::runtime_error (zero diagonal, ...) */

/* ---- context ---------------------------------------------------------- */
int hb_create(int device, hb_ctx** out);
void hb_destroy(hb_ctx* ctx);
const char* hb_last_error(const hb_ctx* ctx); /* ctx may be NULL: last create error */
/* cudaStream_t the library launches on (for event timing by the caller) */
void* hb_stream(hb_ctx* ctx);
int hb_synchronize(hb_ctx* ctx);

/* ---- problem + hierarchy ------------------------------------------------ */
/* kappa2, gamma: nx*ny doubles; enforces the reference's contracts
 * (inc/grid.hpp:72-78,128-141): kappa2 in [lo, hi], omega*sqrt(max kappa2)*h <= 0.6284. */
int hb_set_problem(hb_ctx* ctx, int nx, int ny, double h, double omega, const double* kappa2,
                   const double* gamma, double kappa_lo, double kappa_hi);

#define HB_COARSE_GMRES 0  /* GMRES(coarse_iters) with D^-1, inc/multigrid.hpp:45-61 */
#define HB_COARSE_JACOBI 1 /* coarse_iters damped-Jacobi sweeps */
#define HB_COARSE_NET 2    /* U-Net in net slot 0 as coarsest solver */
#define HB_COARSE_DENSE 3  /* exact solve, CoarseSolver::dense (inc/multigrid.hpp:84,95-104); coarsest <= 1024 nodes */

typedef struct hb_vcycle_cfg {
  int levels;          /* >= 2 (inc/multigrid.hpp:73) */
  int nu1, nu2;        /* pre/post damped-Jacobi sweeps */
  double damping;      /* 0.8 */
  double alpha, beta;  /* shift (1, 0.5) */
  int coarse_solver;   /* HB_COARSE_* */
  int coarse_iters;    /* GMRES restart / Jacobi sweeps */
} hb_vcycle_cfg;

int hb_build_hierarchy(hb_ctx* ctx, const hb_vcycle_cfg* cfg);
/* level geometry after coarsening (inc/stencil.hpp:169-185) */
int hb_level_info(hb_ctx* ctx, int level, int* nx, int* ny, double* h);

/* ---- networks (classic U-Net) ------------------------ */
#define HB_NET_SOLVER 0
#define HB_NET_ENCODER 1
typedef struct hb_net_cfg {
  int kind;    /* HB_NET_SOLVER or HB_NET_ENCODER */
  int levels;  /* resolution levels L */
  int base;    /* channels at level 0 (16) */
  int in_ch;   /* 3 for the solver (h^2 Re r, h^2 Im r, kappa^2), 1 for the encoder */
  int ctx_ch;  /* encoder context channels concatenated per level (0 = standalone) */
} hb_net_cfg;
/* slot 0: solver / coarse net, slot 1: encoder */
int hb_set_net(hb_ctx* ctx, int slot, const hb_net_cfg* cfg);
int hb_net_num_convs(hb_ctx* ctx, int slot);
int hb_net_conv_shape(hb_ctx* ctx, int slot, int index, int* cout, int* cin);
/* weights (cout, cin, 3, 3) OIHW fp32 + bias (cout) in creation order */
int hb_load_conv(hb_ctx* ctx, int slot, int index, const float* w, const float* b);
/* He-normal init from Rng(seed) in creation order (inc/tensor.hpp:51-53) */
int hb_init_net_he(hb_ctx* ctx, int slot, uint64_t seed);
int hb_get_conv(hb_ctx* ctx, int slot, int index, float* w, float* b);
/* forward on host NCHW buffers: in (B, in_ch, H, W) -> out (B, 2, H, W);
 * ctx maps from the encoder are used when the solver net has ctx_ch > 0 and
 * hb_encode has been run.  Test hook (unet_forward, inc/unet.hpp:261). */
int hb_net_forward(hb_ctx* ctx, int batch, int H, int W, const float* in, float* out);
/* encoder over the fine kappa^2 (run once per medium, cached on device). */
int hb_encode(hb_ctx* ctx);
int hb_get_context(hb_ctx* ctx, int level, float* out); /* (base, H>>l, W>>l) */

/* ---- operators (parity hooks, host c128 buffers) ------------------------ */
int hb_operator_apply(hb_ctx* ctx, int level, int shifted, int batch, const double* u, double* y);
int hb_jacobi(hb_ctx* ctx, int level, int batch, double* v, const double* f, int iters);
int hb_restrict(hb_ctx* ctx, int level, int batch, const double* fine, double* coarse);
int hb_prolong(hb_ctx* ctx, int level, int batch, const double* coarse, double* fine);
int hb_coarse_solve(hb_ctx* ctx, int batch, const double* f, double* x);

/* ---- preconditioners ----------------------------------------------------- */
#define HB_PC_V 0  /* SL V-cycle from zero (M_V; with HB_COARSE_NET = coarse-net cycle) */
#define HB_PC_VU 1 /* e0 = net(h^2 r, kappa^2) then V-cycle from e0 (M_VU) */
#define HB_PC_JU 2 /* e1 = J_A(0, r); z = J_A(e1 + net(h^2 (r - A e1), kappa^2), r)  (M_JU,
                      inc/precond.hpp:104-139, JacobiUnetPreconditioner::apply with the A5 net) */
int hb_precond_apply(hb_ctx* ctx, int kind, int batch, const double* r, double* z);
/* Same on device buffers: r, z are complex64 (interleaved float pairs)
 * [batch][ny][nx] in device memory; enqueued on hb_stream(ctx), no host
 * synchronisation (callers keeping their fields in HBM, e.g. a device-side
 * outer Krylov loop).  r and z must not overlap. */
int hb_precond_apply_device(hb_ctx* ctx, int kind, int batch, const void* r, void* z);
/* name() and requires_flexible() of the reference plugin (inc/precond.hpp:14-27) */
const char* hb_precond_name(int kind);
int hb_precond_requires_flexible(hb_ctx* ctx, int kind);

/* ---- FGMRES -------------------------------------------------------------- */
typedef struct hb_krylov_cfg {
  int restart;    /* m */
  int max_iters;  /* preconditioner applications per column */
  double rel_tol; /* in (0, 1) */
  int flexible;   /* 1: flexible GMRES (x += Z y); 0: standard right-preconditioned GMRES
                     (x += M (V y), inc/krylov.hpp:127-136), stationary preconditioners only
                     (HB_ERR_ARG otherwise, check_flexible_contract, inc/precond.hpp:29-32) */
} hb_krylov_cfg;

/* Solve A X = B for `batch` independent columns (block_fgmres semantics).
 * B, X0 (may be NULL), X: host c128 [batch][ny][nx].  hist: [batch][hist_stride]
 * absolute residual history (entry 0 = ||b - A x0||, then |g_{j+1}|);
 * hist_len/iters per column; converged/breakdown flags per column. */
int hb_fgmres(hb_ctx* ctx, const hb_krylov_cfg* cfg, int kind, int batch, const double* B, const double* X0,
              double* X, double* hist, int hist_stride, int* hist_len, int* iters, uint8_t* converged,
              uint8_t* breakdown);
/* True block FGMRES (a non-goal of the reference,
 * SPEC.md:280, its block-size study PAPER.md:580): the batch (<= 16 columns)
 * shares ONE block Krylov space -- block CGS2 orthogonalisation, CholQR2 of
 * each new block, Givens QR of the block Hessenberg; cfg->restart = block
 * steps per cycle (<= 20), cfg->max_iters = block steps in total (every
 * column reports the same count), stop when every column's residual
 * estimate is <= rel_tol ||b_c||; breakdown = the new block lost rank.
 * Arguments as hb_fgmres (flexible must be 1). */
int hb_block_fgmres(hb_ctx* ctx, const hb_krylov_cfg* cfg, int kind, int batch, const double* B, const double* X0,
                    double* X, double* hist, int hist_stride, int* hist_len, int* iters, uint8_t* converged,
                    uint8_t* breakdown);
/* Same, with B and X as DEVICE c128 buffers (inputs resident in HBM); the
 * report arrays are host buffers and may be NULL. */
int hb_fgmres_device(hb_ctx* ctx, const hb_krylov_cfg* cfg, int kind, int batch, const void* dB, void* dX,
                     double* hist, int hist_stride, int* hist_len, int* iters, uint8_t* converged,
                     uint8_t* breakdown);

/* ---- the paper's U-Net ------------------------------
 * UNetConfig (inc/unet.hpp:113-120) and the network built by build_unet /
 * build_encoder (inc/unet.hpp:139-257): 5x5 stride-2 down convs + batch norm +
 * ELU, ResNet blocks, transposed 5x5 stride-2 up convs, 4 input channels
 * (h^2 Re r, h^2 Im r, kappa^2, gamma; inc/precond.hpp:74-90), eval mode.
 * Once set, it is the network of M_JU and M_VU (JacobiUnetPreconditioner /
 * UnetVCyclePreconditioner with NetworkApplier, inc/precond.hpp:57-165);
 * hb_set_net(slot 0) switches back to the classic net. */
typedef struct hb_unet_cfg {
  int levels;             /* downsamplings */
  int base_channels;      /* even */
  int resnet_per_level;
  int bottleneck_resnets;
  int updown_kernel;      /* odd (5) */
  int res_kernel;         /* odd (3) */
} hb_unet_cfg;
/* variant 0: standalone ("unet." names), 1: encoder_solver ("enc." + "sol.");
 * parameters are created in the reference's registry order and initialised as
 * NetworkWeights() (seed 0x5eed) */
int hb_set_paper_net(hb_ctx* ctx, const hb_unet_cfg* cfg, int variant);
/* NetworkWeights(seed) initialisation (inc/unet.hpp:13-33) */
int hb_paper_init(hb_ctx* ctx, uint64_t seed);
int hb_paper_param_count(hb_ctx* ctx);
/* name (NUL-terminated, cap bytes) and dims (n, c, h, w) of parameter i */
int hb_paper_param_info(hb_ctx* ctx, int i, char* name, int cap, int* dims);
/* in != NULL: set the parameter's values; out != NULL: read them; count =
 * the caller's element count, which must equal the parameter's (n*c*h*w) */
int hb_paper_param(hb_ctx* ctx, const char* name, int64_t count, const float* in, float* out);
/* UNW1 checkpoints (load_checkpoint / save_checkpoint, inc/checkpoint.hpp:51-104) */
int hb_load_checkpoint(hb_ctx* ctx, const char* path);
int hb_save_checkpoint(hb_ctx* ctx, const char* path, const char* digest);
/* unet_forward / solver_forward (inc/unet.hpp:261-295), eval mode:
 * in NCHW [batch][4][H][W] -> out NCHW [batch][2][H][W] (host fp32) */
int hb_paper_forward(hb_ctx* ctx, int batch, int H, int W, const float* in, float* out);

/* ---- SLW1 raw fields (write_slw1 / read_slw1, inc/field_io.hpp:46-76) ------
 * "SLW1", u32 nx, u32 ny (LE), nx*ny f32 LE row-major; host only.  read with
 * values == NULL reports the dims.  Errors: HB_ERR_ARG (cannot open),
 * HB_ERR_NUMERIC (bad magic / dims / truncated). */
int hb_write_slw1(const char* path, int nx, int ny, const double* values);
int hb_read_slw1(const char* path, int* nx, int* ny, double* values);

/* ---- training pairs ----------------------------------
 * gen_sample_pair (inc/datagen.hpp:191-219) for `count` seeds: x ~ CN(0, I)
 * from Rng(seed), b = A x, k = k_forced (>= 0) or uniform_int(1, k_max),
 * x~ = FGMRES(A, M_V, b, 0; restart 10, k iterations, tol 1e-6), r = b - A x~,
 * e = x - x~.  r_out, e_out: host c128 [count][ny][nx]; k_used may be NULL.
 * Samples are grouped by k into batched device solves. */
int hb_gen_sample_pairs(hb_ctx* ctx, int count, const uint64_t* seeds, int k_forced, int k_max, double* r_out,
                        double* e_out, int* k_used);

/* ---- training -----------------------------------------
 * The paper net's training on the device: traindet::run_batch (train-mode
 * forward of build_unet / build_encoder, MSE loss, reverse sweep of the Tape
 * rules; inc/training.hpp:121-147, inc/autodiff.hpp:121-480) and adam_step
 * (inc/adam.hpp:25-58).  Trainable parameters are the reference's (kernels,
 * biases, batch-norm scale / offset); running buffers update in train mode.
 * TrainConfig (inc/training.hpp:12-20): */
typedef struct hb_train_cfg {
  int epochs;           /* 40 */
  double lr0;           /* 1e-4 */
  int batch0;           /* 20 */
  int t0;               /* 48 */
  double val_fraction;  /* 0.1 */
  int encoder_solver;   /* must match the net's variant */
  uint64_t seed;        /* 1 */
} hb_train_cfg;
/* One run_batch on host NCHW fp32 input [batch][4][H][W], kappa [batch][1][H][W]
 * (encoder_solver only; else NULL), target [batch][2][H][W]: train_mode (batch
 * statistics) or eval, gradients (zeroed first, as zero_grads) when with_grad,
 * then one ADAM step at lr when step (Adam moments persist across calls until
 * hb_paper_adam_reset).  loss: the MSE; out (may be NULL): the net output. */
int hb_paper_train_batch(hb_ctx* ctx, int batch, int H, int W, const float* input, const float* kappa,
                         const float* target, int train_mode, int with_grad, int step, double lr, double* loss,
                         float* out);
/* trainable element count, and the last batch's trainable gradients concatenated in registry order */
int64_t hb_paper_trainable_count(hb_ctx* ctx);
int hb_paper_grads(hb_ctx* ctx, int64_t count, float* grads);
/* NetworkWeights::set_trainable_prefix (inc/unet.hpp:78-86) */
int hb_paper_set_trainable_prefix(hb_ctx* ctx, const char* prefix, int trainable);
int hb_paper_adam_reset(hb_ctx* ctx);
/* train() (inc/training.hpp:152-227) over an in-memory Dataset: count samples
 * r_hat / e_true [count][2][H][W] fp32 (quantize_sample form), model_id[count]
 * into models problems' kappa2 / gamma [models][H][W] fp64 (row-major y, x).
 * hist [hist_cap][4] per epoch: mean train rel error, mean val rel error, lr,
 * batch.  aborted: a non-finite loss stopped training (weights restored to the
 * last finite epoch). */
int hb_paper_train(hb_ctx* ctx, const hb_train_cfg* cfg, int count, int H, int W, const float* r_hat,
                   const float* e_true, const int* model_id, int models, const double* kappa2, const double* gamma,
                   double* hist, int hist_cap, int* epochs_run, int* aborted);
/* retrain() (inc/training.hpp:229-298) on the context's problem: n_pairs
 * gen_sample_pair samples (seeds seed*6151+i, on the context's hierarchy),
 * lr0/10, batch min(20, n_pairs); encoder_solver freezes the encoder. */
int hb_paper_retrain(hb_ctx* ctx, int n_pairs, int epochs, const hb_train_cfg* base, uint64_t seed, double* hist,
                     int hist_cap, int* epochs_run, int* aborted);

/* ---- row slabs: one large grid over several GPUs --
 * The reference solves one grid in one process (block_fgmres,
 * inc/krylov.hpp:83-267; cycle_at, inc/multigrid.hpp:108-119); these entry
 * points run the same FGMRES + M_V on a grid split into row slabs, slab r owning
 * level-0 rows [a_r, a_{r+1}) (multiples of 2^(levels-1)).  Every level but the
 * coarsest keeps 2 ghost rows per side (halo exchange), the coarsest is
 * all-gathered and solved replicated, the Arnoldi sums are allreduced in fp64.
 * Call after hb_set_problem + hb_build_hierarchy (nu1 = nu2 = 1) with the WHOLE
 * problem on every slab; afterwards the context only serves the *_slab calls.
 * Host buffers hold the rows the calling process supplies (hb_slab_rows):
 * [batch][row_end - row_begin][nx] c128. */
#define HB_NCCL_ID_BYTES 128
/* slab `slab` of `nslabs` for an ny-row grid with `levels` levels (host only) */
int hb_slab_partition(int ny, int levels, int nslabs, int slab, int* row_begin, int* row_end);
/* ncclGetUniqueId of the process's NCCL (libnccl.so.2, loaded on first use) */
int hb_nccl_unique_id(unsigned char* id);
/* one slab per process (one GPU per rank): NCCL halos / allreduce / gathers */
int hb_slab_init_nccl(hb_ctx* ctx, int rank, int nranks, const unsigned char* id);
/* nslabs contexts of one process on one device as slabs 0..nslabs-1 (they
 * share one stream; halos are device copies); drive the group through ctxs[0] */
int hb_slab_init_local(hb_ctx** ctxs, int nslabs);
/* rows [row_begin, row_end) whose data this process supplies / receives */
int hb_slab_rows(hb_ctx* ctx, int* row_begin, int* row_end);
/* Preconditioner::apply (M_V only) on slabs; r, z: host c128 rows of this process */
int hb_precond_apply_slab(hb_ctx* ctx, int kind, int batch, const double* r, double* z);
/* block_fgmres on slabs (M_V); B, X0 (may be NULL), X: host c128 rows of this process;
 * the report arrays as hb_fgmres (identical on every slab) */
int hb_fgmres_slab(hb_ctx* ctx, const hb_krylov_cfg* cfg, int kind, int batch, const double* B, const double* X0,
                   double* X, double* hist, int hist_stride, int* hist_len, int* iters, uint8_t* converged,
                   uint8_t* breakdown);

/* ---- setup helpers (host restatements of the reference RNG / generators) -- */
/* Rng (inc/rng.hpp:9-67): n normals from Rng(seed) */
void hb_rng_normals(uint64_t seed, int64_t n, double* out);
/* absorbing layer (inc/grid.hpp:101-119) */
int hb_absorbing_layer(int nx, int ny, int width, double gamma_max, double* out);
/* medium generator SURVEY A1 (+D7 interfaces) -> kappa^2 */
int hb_make_medium(int nx, int ny, uint64_t seed, double sigma, double vmin, double vmax, int n_interfaces,
                   uint64_t iface_seed, int iface_margin, double jmin, double jmax, double* kappa2);
/* point sources SURVEY A2 (mode 0: uniform (x, y) in [lo, hi]^2, mode 1: on `row`) */
void hb_point_sources(uint64_t seed, int batch, int mode, int lo, int hi, int row, int* xs, int* ys);

/* ---- options ------------------------------------------------------------ */
/* "fused_vcycle" (1): fused down/up V-cycle legs for nu1 = nu2 = 1
 * "cuda_graphs"  (1): replay each FGMRES restart cycle as one CUDA graph
 * "small_coarse" (1): register-resident coarsest GMRES for <= 1024-node grids */
int hb_set_option(hb_ctx* ctx, const char* key, int64_t value);

/* ---- instrumentation ------------------------------------------------------ */
/* per-kernel-class device time (CUDA events on the library stream), for the
 * roofline numerator/denominator in bench.py.  classes: see hb_prof_name. */
int hb_prof_enable(hb_ctx* ctx, int on);
int hb_prof_reset(hb_ctx* ctx);
int hb_prof_count(hb_ctx* ctx);
const char* hb_prof_name(hb_ctx* ctx, int i);
int hb_prof_get(hb_ctx* ctx, int i, double* total_ms, int64_t* launches, double* bytes, double* flops);
/* per-launch detail: turn on/off; dumps (and clears) the records collected so far
 * as "label,us,bytes,flops" lines into buf */
int hb_prof_detail(hb_ctx* ctx, int on, char* buf, int cap);
/* number of library kernel launches since the last reset */
int64_t hb_launch_count(hb_ctx* ctx);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* HELMGPU_H_ */
