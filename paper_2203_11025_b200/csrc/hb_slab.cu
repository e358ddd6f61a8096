// Row-slab decomposition of one large grid (one
// 4096^2 right-hand side spread over the GPUs of a node).
//
// Slab r owns level-0 rows [a_r, a_{r+1}) (boundaries multiples of 2^(L-1), so
// every level l owns [a_r >> l, a_{r+1} >> l)).  Each non-coarsest level is
// stored as the owned rows plus G = 2 ghost rows above and below; the coarsest
// level is stored whole on every slab and its solve (GMRES(10), Jacobi or the
// U-Net) is replicated, after an all-gather of the coarse right-hand side --
// the "gathered coarse solve" option of 8(e), chosen because the coarse grid is
// 1/64 of the fine one at c4 and the replicated net needs no conv halos.
//
// Communication per FGMRES inner step (the reference's single-process
// block_fgmres, inc/krylov.hpp:190-254, has none):
//   halo(V_j, 2 rows) -> down legs, halo(f_l) per level -> gather(f_coarse)
//   -> coarse solve -> halo(x_l) per level, up legs -> halo(Z_j) ->
//   adots partial -> allreduce -> MGS coefficients -> update partial ->
//   allreduce -> Givens / convergence.
// The two allreduces carry fp64 per-column sums; every slab receives the same
// bits, so the replicated Hessenberg, Givens and convergence flags agree.
//
// Transports: NCCL (one slab per process, dlopen'ed libnccl.so.2: ncclSend /
// ncclRecv halos, ncclAllReduce, ncclBroadcast gathers, all on the library
// stream, so a restart cycle is one captured CUDA graph), or an in-process
// group (several slabs of one process on one device and one stream: halos are
// device copies between the slabs' buffers, the allreduce a summing kernel).
// The in-process group runs the decomposed algorithm on one GPU with nothing
// waiting on anything else; it is how the slab path is tested on one B200.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "hb_internal.h"

namespace hb {

constexpr int kGhost = 2;
constexpr int kMaxLocalSlabs = 16;

// ------------------------------------------------------------------ NCCL --
struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    // the process may already hold an NCCL (torch's): dlopen by soname reuses it
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.err = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return a;
    }
#define HB_SYM(name, field)                                                  \
  a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, name));             \
  if (!a.field) {                                                            \
    a.err = std::string("libnccl lacks ") + name;                            \
    return a;                                                                \
  }
    HB_SYM("ncclGetUniqueId", GetUniqueId)
    HB_SYM("ncclCommInitRank", CommInitRank)
    HB_SYM("ncclCommDestroy", CommDestroy)
    HB_SYM("ncclAllReduce", AllReduce)
    HB_SYM("ncclBroadcast", Broadcast)
    HB_SYM("ncclSend", Send)
    HB_SYM("ncclRecv", Recv)
    HB_SYM("ncclGroupStart", GroupStart)
    HB_SYM("ncclGroupEnd", GroupEnd)
    HB_SYM("ncclGetErrorString", GetErrorString)
#undef HB_SYM
    a.ok = true;
    return a;
  }();
  if (!api.ok) throw HbError{HB_ERR_STATE, api.err};
  return api;
}

#define HB_NCCL(x)                                                                               \
  do {                                                                                           \
    ncclResult_t r_ = (x);                                                                       \
    if (r_ != ncclSuccess)                                                                       \
      throw ::hb::HbError{HB_ERR_CUDA, std::string(#x) + ": " + nccl().GetErrorString(r_)};      \
  } while (0)

// --------------------------------------------------------------- state --
struct SlabGroup {  // in-process slabs sharing one device and one stream
  std::vector<Context*> members;  // rank order
  cudaStream_t stream = nullptr;
  ~SlabGroup() {
    if (stream) cudaStreamDestroy(stream);
  }
};

struct SlabState {
  int rank = 0, nranks = 1;
  std::vector<int> bounds;  // level-0 row boundaries, nranks + 1
  ncclComm_t comm = nullptr;
  std::shared_ptr<SlabGroup> group;  // in-process transport (null: NCCL)
  DBuf<double2> gsum;                // [B][kMaxDots] per-column sums of the split reductions
  ~SlabState() {
    if (comm) nccl().CommDestroy(comm);
  }
};

// boundaries: multiples of q = 2^(levels-1), as even as the grid allows
static std::vector<int> partition(int ny, int levels, int nslabs) {
  const int q = 1 << (levels - 1);
  if (nslabs < 1) throw HbError{HB_ERR_ARG, "nslabs must be >= 1"};
  if (ny % q) throw HbError{HB_ERR_ARG, "grid rows not divisible by 2^(levels-1)"};
  const int units = ny / q;
  // every slab-stored level (0 .. levels-2) needs >= kGhost owned rows per slab
  const int min_units = std::max(1, (kGhost * (1 << std::max(0, levels - 2)) + q - 1) / q);
  if (units < nslabs * min_units) throw HbError{HB_ERR_ARG, "too many slabs for this grid / level count"};
  std::vector<int> b(size_t(nslabs) + 1);
  for (int r = 0; r <= nslabs; ++r) b[size_t(r)] = int((int64_t(r) * units) / nslabs) * q;
  for (int r = 0; r < nslabs; ++r)
    if ((b[size_t(r) + 1] - b[size_t(r)]) / q < min_units) throw HbError{HB_ERR_ARG, "slab too thin"};
  return b;
}

// re-lay the context's hierarchy as slab `rank` of `bounds`
static void apply_slab(Context& c, int rank, const std::vector<int>& bounds) {
  if (!c.has_hier) throw HbError{HB_ERR_STATE, "hierarchy not built (hb_build_hierarchy)"};
  if (c.vc.nu1 != 1 || c.vc.nu2 != 1) throw HbError{HB_ERR_ARG, "row slabs run the fused legs: nu1 = nu2 = 1"};
  const int nl = int(c.levels.size());
  for (int l = 0; l < nl; ++l) {
    Level& L = *c.levels[size_t(l)];
    const int lo = bounds[size_t(rank)] >> l, hi = bounds[size_t(rank) + 1] >> l;
    L.lo = lo;
    L.hi = hi;
    if (l < nl - 1) {
      L.row0 = lo - kGhost;
      L.rows = hi - lo + 2 * kGhost;
    } else {  // coarsest: stored whole, solved replicated
      L.row0 = 0;
      L.rows = L.ny;
    }
    for (auto* d : {&L.dM, &L.dA, &L.wdi, &L.f, &L.v, &L.t, &L.x}) d->release();
    L.k2f.release();
    L.dA64.release();
    L.dM64.release();
    fill_level_device(L, c.omega, c.vc.alpha, c.vc.beta, c.vc.damping, l == 0, l == nl - 1);
  }
  c.batch_cap = 0;
  for (auto& g : c.graphs) cudaGraphExecDestroy(g.exec);
  c.graphs.clear();
  c.kV.release();
  c.kZ.release();
  c.kW.release();
  c.kX.release();
  c.kB.release();
  ++g_alloc_gen;
}

// contexts this process drives (rank order) and the stream they share
static std::vector<Context*> members(Context& c) {
  if (!c.slab) throw HbError{HB_ERR_STATE, "not a slab context (hb_slab_init_*)"};
  if (c.slab->group) {
    if (c.slab->rank != 0) throw HbError{HB_ERR_ARG, "drive an in-process slab group through its slab 0"};
    return c.slab->group->members;
  }
  return {&c};
}

// ----------------------------------------------------------- transport --
// a per-slab device field: base pointer of column 0 (storage row 0), element size
using FieldFn = void* (*)(Context&, int level, int j);

struct PtrList {
  double* p[kMaxLocalSlabs];
  int n;
};
__global__ void k_group_sum(PtrList L, int count) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < L.n; ++r) s += L.p[r][i];
    for (int r = 0; r < L.n; ++r) L.p[r][i] = s;
  }
}

static void* rowptr(Context& c, int l, void* base, size_t esz, int grow) {
  const Level& L = *c.levels[size_t(l)];
  return static_cast<char*>(base) + (size_t(grow - L.row0) * L.nx) * esz;
}

// fill the kGhost ghost rows above and below every slab's owned rows of a
// level-l field (B columns) from the neighbouring slabs' owned rows
static void halo(std::vector<Context*>& S, int l, int B, size_t esz, FieldFn fld, int j) {
  SlabState& st = *S[0]->slab;
  const Level& L0 = *S[0]->levels[size_t(l)];
  const size_t width = size_t(kGhost) * L0.nx * esz;
  if (st.group) {
    const int R = int(S.size());
    for (int r = 0; r < R; ++r) {
      Context& c = *S[size_t(r)];
      const Level& L = *c.levels[size_t(l)];
      void* base = fld(c, l, j);
      const size_t dp = L.N() * esz;
      if (r > 0) {  // top ghosts <- slab r-1's last owned rows
        Context& n = *S[size_t(r) - 1];
        const Level& Ln = *n.levels[size_t(l)];
        HB_CUDA(cudaMemcpy2DAsync(rowptr(c, l, base, esz, L.lo - kGhost), dp,
                                  rowptr(n, l, fld(n, l, j), esz, Ln.hi - kGhost), Ln.N() * esz, width, size_t(B),
                                  cudaMemcpyDeviceToDevice, c.stream));
      }
      if (r + 1 < R) {  // bottom ghosts <- slab r+1's first owned rows
        Context& n = *S[size_t(r) + 1];
        const Level& Ln = *n.levels[size_t(l)];
        HB_CUDA(cudaMemcpy2DAsync(rowptr(c, l, base, esz, L.hi), dp, rowptr(n, l, fld(n, l, j), esz, Ln.lo),
                                  Ln.N() * esz, width, size_t(B), cudaMemcpyDeviceToDevice, c.stream));
      }
    }
    return;
  }
  Context& c = *S[0];
  const Level& L = *c.levels[size_t(l)];
  void* base = fld(c, l, j);
  const size_t cnt = width / 4, cs = L.N() * esz;
  auto& N = nccl();
  HB_NCCL(N.GroupStart());
  for (int b = 0; b < B; ++b) {
    char* col = static_cast<char*>(base) + size_t(b) * cs;
    if (st.rank > 0) {
      HB_NCCL(N.Send(rowptr(c, l, col, esz, L.lo), cnt, ncclFloat32, st.rank - 1, st.comm, c.stream));
      HB_NCCL(N.Recv(rowptr(c, l, col, esz, L.lo - kGhost), cnt, ncclFloat32, st.rank - 1, st.comm, c.stream));
    }
    if (st.rank + 1 < st.nranks) {
      HB_NCCL(N.Send(rowptr(c, l, col, esz, L.hi - kGhost), cnt, ncclFloat32, st.rank + 1, st.comm, c.stream));
      HB_NCCL(N.Recv(rowptr(c, l, col, esz, L.hi), cnt, ncclFloat32, st.rank + 1, st.comm, c.stream));
    }
  }
  HB_NCCL(N.GroupEnd());
}

// whole coarsest-level field (B columns) on every slab from the owned rows
// (to0: in-process group, assemble it on slab 0 only -- see slab_vcycle)
static void gather_coarse(std::vector<Context*>& S, int B, FieldFn fld, bool to0 = false) {
  SlabState& st = *S[0]->slab;
  const int l = int(S[0]->levels.size()) - 1;
  const Level& C = *S[0]->levels[size_t(l)];
  const size_t esz = sizeof(float2), cs = C.N() * esz;
  if (st.group) {
    const int R = int(S.size());
    for (int r = 0; r < R; ++r) {
      Context& src = *S[size_t(r)];
      const Level& Ls = *src.levels[size_t(l)];
      const size_t width = size_t(Ls.hi - Ls.lo) * Ls.nx * esz;
      for (int t = 0; t < R; ++t) {
        if (t == r || (to0 && t != 0)) continue;
        Context& dst = *S[size_t(t)];
        HB_CUDA(cudaMemcpy2DAsync(rowptr(dst, l, fld(dst, l, 0), esz, Ls.lo), cs,
                                  rowptr(src, l, fld(src, l, 0), esz, Ls.lo), cs, width, size_t(B),
                                  cudaMemcpyDeviceToDevice, dst.stream));
      }
    }
    return;
  }
  Context& c = *S[0];
  auto& N = nccl();
  HB_NCCL(N.GroupStart());
  for (int r = 0; r < st.nranks; ++r) {
    const int lo = st.bounds[size_t(r)] >> l, hi = st.bounds[size_t(r) + 1] >> l;
    const size_t cnt = size_t(hi - lo) * C.nx * 2;  // floats
    for (int b = 0; b < B; ++b) {
      void* p = rowptr(c, l, static_cast<char*>(fld(c, l, 0)) + size_t(b) * cs, esz, lo);
      HB_NCCL(N.Broadcast(p, p, cnt, ncclFloat32, r, st.comm, c.stream));
    }
  }
  HB_NCCL(N.GroupEnd());
}

// sum every slab's gsum[B][kMaxDots] (fp64) and hand every slab the result
static void allreduce_gsum(std::vector<Context*>& S, int B) {
  SlabState& st = *S[0]->slab;
  const size_t count = size_t(B) * kMaxDots * 2;
  if (st.group) {
    PtrList pl{};
    pl.n = int(S.size());
    for (int r = 0; r < pl.n; ++r) pl.p[r] = reinterpret_cast<double*>(S[size_t(r)]->slab->gsum.p);
    S[0]->launches++;
    k_group_sum<<<int(std::min<size_t>(64, (count + 255) / 256)), 256, 0, S[0]->stream>>>(pl, int(count));
    HB_CUDA(cudaGetLastError());
    return;
  }
  Context& c = *S[0];
  HB_NCCL(nccl().AllReduce(st.gsum.p, st.gsum.p, count, ncclFloat64, ncclSum, st.comm, c.stream));
}

// ------------------------------------------------------------- V-cycle --
static void* f_level(Context& c, int l, int) { return c.levels[size_t(l)]->f.p; }
static void* x_level(Context& c, int l, int) { return c.levels[size_t(l)]->x.p; }

// M_V on slabs: cycle_at (inc/multigrid.hpp:108-119) with nu1 = nu2 = 1, zero
// initial guess, fused row-streaming legs; per-slab level-0 input f0 (with
// ghosts valid), column scales fs, output z (owned rows written)
static void slab_vcycle(std::vector<Context*>& S, int B, const std::vector<const int*>& act,
                        const std::vector<const float2*>& f0, const std::vector<const float*>& fs,
                        const std::vector<float2*>& z) {
  const int nl = int(S[0]->levels.size());
  const float w = float(S[0]->vc.damping);
  for (int l = 0; l < nl - 1; ++l) {
    for (size_t s = 0; s < S.size(); ++s) {
      Context& c = *S[s];
      Level& L = *c.levels[size_t(l)];
      Level& C = *c.levels[size_t(l) + 1];
      launch_down_stream(c, L.view(), C.win(), w, l % 2, B, act[s], l == 0 ? f0[s] : L.f.p, l == 0 ? fs[s] : nullptr,
                         nullptr, C.f.p);
    }
    if (l + 1 < nl - 1)
      halo(S, l + 1, B, sizeof(float2), f_level, 0);
    else
      gather_coarse(S, B, f_level, S[0]->slab->group != nullptr);
  }
  if (S[0]->slab->group != nullptr) {
    // in-process group (all slabs on one device and stream): the replicated
    // coarsest solve -- identical inputs, deterministic kernels, identical bits
    // on every slab -- runs once on slab 0 and its solution is copied to the
    // others (with one GPU per slab every rank solves it concurrently instead)
    Context& c0 = *S[0];
    Level& C0 = *c0.levels.back();
    coarsest_solve(c0, B, 0, act[0], C0.f.p, C0.x.p);
    for (size_t s = 1; s < S.size(); ++s)
      HB_CUDA(cudaMemcpyAsync(S[s]->levels.back()->x.p, C0.x.p, sizeof(float2) * C0.N() * size_t(B),
                              cudaMemcpyDeviceToDevice, c0.stream));
  } else {
    for (size_t s = 0; s < S.size(); ++s) {
      Context& c = *S[s];
      Level& C = *c.levels.back();
      coarsest_solve(c, B, 0, act[s], C.f.p, C.x.p);
    }
  }
  for (int l = nl - 2; l >= 0; --l) {
    if (l + 1 < nl - 1) halo(S, l + 1, B, sizeof(float2), x_level, 0);
    for (size_t s = 0; s < S.size(); ++s) {
      Context& c = *S[s];
      Level& L = *c.levels[size_t(l)];
      Level& C = *c.levels[size_t(l) + 1];
      launch_up_stream(c, L.view(), w, l % 2, C.nx, C.ny, C.win(), B, act[s], l == 0 ? f0[s] : L.f.p,
                       l == 0 ? fs[s] : nullptr, nullptr, C.x.p, l == 0 ? z[s] : L.x.p);
    }
  }
}

// ------------------------------------------------------------- FGMRES --
static void* kv_slot(Context& c, int, int j) { return c.kV.p + size_t(j) * c.k_B * c.levels[0]->N(); }
static void* kz_slot(Context& c, int, int j) { return c.kZ.p + size_t(j) * c.k_B * c.levels[0]->N(); }
static void* kx_field(Context& c, int, int) { return c.kX.p; }

static void slab_fgmres(std::vector<Context*>& S, const hb_krylov_cfg* cfg, int kind, int B) {
  if (!cfg) throw HbError{HB_ERR_ARG, "null krylov config"};
  if (cfg->restart < 1) throw HbError{HB_ERR_ARG, "restart must be >= 1"};
  if (!(cfg->rel_tol > 0.0 && cfg->rel_tol < 1.0)) throw HbError{HB_ERR_ARG, "rel_tol in (0,1)"};
  if (!cfg->flexible) throw HbError{HB_ERR_ARG, "the device FGMRES stores Z: flexible must be 1"};
  if (kind != HB_PC_V) throw HbError{HB_ERR_ARG, "row slabs run the SL V-cycle preconditioner (M_V)"};
  const int m = cfg->restart;
  const int cap = std::max(1, cfg->max_iters + 2);
  const double tol = cfg->rel_tol;
  const int maxit = cfg->max_iters;
  for (Context* c : S) {
    krylov_alloc(*c, B, m, cap);
    c->slab->gsum.ensure(size_t(B) * kMaxDots);
  }
  Context& lead = *S[0];
  const size_t R = S.size();
  auto gs = [&](size_t s) { return S[s]->slab->gsum.p; };
  auto restart = [&]() {
    halo(S, 0, B, sizeof(double2), kx_field, 0);
    for (size_t s = 0; s < R; ++s)
      launch_fg_restart(*S[s], B, S[s]->kB.p, S[s]->kX.p, S[s]->kV.p, cap, tol, maxit, gs(s));
    allreduce_gsum(S, B);
    for (size_t s = 0; s < R; ++s) launch_fg_restart_finish(*S[s], B, gs(s), cap, tol, maxit);
  };
  std::vector<const int*> act(R);
  std::vector<const float*> fs(R);
  std::vector<const float2*> f0(R);
  std::vector<float2*> z(R);
  for (size_t s = 0; s < R; ++s) {
    act[s] = S[s]->kact.p;
    fs[s] = S[s]->kscale.p;
  }
  auto cycle_body = [&]() {
    for (int j = 0; j < m; ++j) {
      halo(S, 0, B, sizeof(float2), kv_slot, j);
      for (size_t s = 0; s < R; ++s) {
        f0[s] = static_cast<const float2*>(kv_slot(*S[s], 0, j));
        z[s] = static_cast<float2*>(kz_slot(*S[s], 0, j));
      }
      slab_vcycle(S, B, act, f0, fs, z);
      halo(S, 0, B, sizeof(float2), kz_slot, j);
      for (size_t s = 0; s < R; ++s) launch_fg_adots(*S[s], B, j, z[s], S[s]->kW.p, S[s]->kV.p, gs(s));
      allreduce_gsum(S, B);
      for (size_t s = 0; s < R; ++s) launch_fg_adots_finish(*S[s], B, j, gs(s));
      for (size_t s = 0; s < R; ++s) launch_fg_update(*S[s], B, j, m, S[s]->kW.p, S[s]->kV.p, cap, tol, maxit, gs(s));
      allreduce_gsum(S, B);
      for (size_t s = 0; s < R; ++s) launch_fg_update_finish(*S[s], B, j, m, gs(s), cap, tol, maxit);
    }
    for (size_t s = 0; s < R; ++s) launch_fg_finalize(*S[s], B, m, S[s]->kZ.p, S[s]->kX.p);
    restart();
  };
  if (!lead.h_count) HB_CUDA(cudaMallocHost(&lead.h_count, sizeof(int)));
  auto read_count = [&]() {
    HB_CUDA(cudaMemcpyAsync(lead.h_count, lead.kcount.p, sizeof(int), cudaMemcpyDeviceToHost, lead.stream));
    HB_CUDA(cudaStreamSynchronize(lead.stream));
    return *lead.h_count;
  };
  restart();
  if (read_count() == 0) return;
  if (!lead.opt_graphs) {
    do cycle_body();
    while (read_count() > 0);
    return;
  }
  // first cycle eager (lazy allocations), then one captured graph per cycle
  cycle_body();
  if (read_count() == 0) return;
  Context::GraphEntry* ge = nullptr;
  const int gkind = 100 + kind;
  for (auto& g : lead.graphs)
    if (g.gen == g_alloc_gen && g.kind == gkind && g.B == B && g.m == m && g.cap == cap && g.max_iters == maxit &&
        g.tol == tol && g.dB == lead.kB.p && g.dX == lead.kX.p)
      ge = &g;
  if (!ge) {
    std::vector<int64_t> l0(R);
    for (size_t s = 0; s < R; ++s) l0[s] = S[s]->launches;
    cudaGraph_t graph;
    HB_CUDA(cudaStreamBeginCapture(lead.stream, cudaStreamCaptureModeThreadLocal));
    try {
      cycle_body();
    } catch (...) {
      cudaStreamEndCapture(lead.stream, &graph);
      throw;
    }
    HB_CUDA(cudaStreamEndCapture(lead.stream, &graph));
    int64_t per_cycle = 0;
    for (size_t s = 0; s < R; ++s) {
      per_cycle += S[s]->launches - l0[s];
      S[s]->launches = l0[s];
    }
    cudaGraphExec_t exec;
    HB_CUDA(cudaGraphInstantiate(&exec, graph, 0));
    HB_CUDA(cudaGraphDestroy(graph));
    lead.graphs.push_back(Context::GraphEntry{g_alloc_gen, gkind, B, m, cap, maxit, tol, lead.kB.p, lead.kX.p, exec,
                                              per_cycle});
    ge = &lead.graphs.back();
  }
  do {
    HB_CUDA(cudaGraphLaunch(ge->exec, lead.stream));
    lead.launches += ge->launches;
  } while (read_count() > 0);
}

// host rows [lo, hi) of the calling process (B columns of prow rows starting
// at global row plo) <-> the slab storage of every member
static void scatter_rows(std::vector<Context*>& S, int B, const double* host, int plo, int prows, bool x) {
  for (Context* cp : S) {
    Context& c = *cp;
    const Level& L = *c.levels[0];
    double2* dst = x ? c.kX.p : c.kB.p;
    HB_CUDA(cudaMemsetAsync(dst, 0, sizeof(double2) * L.N() * B, c.stream));
    if (!host) continue;
    HB_CUDA(cudaMemcpy2DAsync(dst + size_t(L.lo - L.row0) * L.nx, L.N() * sizeof(double2),
                              host + 2 * size_t(L.lo - plo) * L.nx, size_t(prows) * L.nx * sizeof(double2),
                              size_t(L.hi - L.lo) * L.nx * sizeof(double2), size_t(B), cudaMemcpyHostToDevice,
                              c.stream));
  }
}
static void gather_rows(std::vector<Context*>& S, int B, double* host, int plo, int prows) {
  for (Context* cp : S) {
    Context& c = *cp;
    const Level& L = *c.levels[0];
    HB_CUDA(cudaMemcpy2DAsync(host + 2 * size_t(L.lo - plo) * L.nx, size_t(prows) * L.nx * sizeof(double2),
                              c.kX.p + size_t(L.lo - L.row0) * L.nx, L.N() * sizeof(double2),
                              size_t(L.hi - L.lo) * L.nx * sizeof(double2), size_t(B), cudaMemcpyDeviceToHost,
                              c.stream));
  }
}

static void proc_rows(Context& c, int* lo, int* hi) {
  const SlabState& st = *c.slab;
  if (st.group) {
    *lo = 0;
    *hi = st.bounds.back();
  } else {
    *lo = st.bounds[size_t(st.rank)];
    *hi = st.bounds[size_t(st.rank) + 1];
  }
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

extern "C" {

int hb_slab_partition(int ny, int levels, int nslabs, int slab, int* row_begin, int* row_end) {
  try {
    if (levels < 2 || slab < 0 || slab >= nslabs) return HB_ERR_ARG;
    const auto b = partition(ny, levels, nslabs);
    if (row_begin) *row_begin = b[size_t(slab)];
    if (row_end) *row_end = b[size_t(slab) + 1];
    return HB_OK;
  } catch (const HbError& e) {
    return e.code;
  }
}

int hb_nccl_unique_id(unsigned char* id) {
  if (!id) return HB_ERR_ARG;
  try {
    ncclUniqueId u;
    HB_NCCL(nccl().GetUniqueId(&u));
    static_assert(sizeof(u.internal) == HB_NCCL_ID_BYTES, "ncclUniqueId size");
    std::memcpy(id, u.internal, HB_NCCL_ID_BYTES);
    return HB_OK;
  } catch (const HbError& e) {
    return e.code;
  }
}

int hb_slab_init_nccl(hb_ctx* ctx, int rank, int nranks, const unsigned char* id) {
  HB_API_BEGIN
  if (!id || nranks < 1 || rank < 0 || rank >= nranks) throw HbError{HB_ERR_ARG, "bad rank / nranks / id"};
  auto st = std::make_shared<SlabState>();
  st->rank = rank;
  st->nranks = nranks;
  st->bounds = partition(ctx->ny, ctx->vc.levels, nranks);
  ncclUniqueId u;
  std::memcpy(u.internal, id, HB_NCCL_ID_BYTES);
  HB_CUDA(cudaSetDevice(ctx->device));
  HB_NCCL(nccl().CommInitRank(&st->comm, nranks, u, rank));
  apply_slab(*ctx, rank, st->bounds);
  ctx->slab = st;
  HB_API_END
}

int hb_slab_init_local(hb_ctx** ctxs, int nslabs) {
  if (!ctxs || nslabs < 1 || nslabs > kMaxLocalSlabs) return HB_ERR_ARG;
  hb_ctx* ctx = ctxs[0];
  HB_API_BEGIN
  for (int r = 0; r < nslabs; ++r) {
    hb_ctx* c = ctxs[r];
    if (!c || !c->has_hier) throw HbError{HB_ERR_STATE, "every slab context needs the problem and hierarchy"};
    if (c->device != ctx->device || c->nx != ctx->nx || c->ny != ctx->ny || c->vc.levels != ctx->vc.levels ||
        c->vc.coarse_solver != ctx->vc.coarse_solver)
      throw HbError{HB_ERR_ARG, "slab contexts must share device, grid and hierarchy"};
  }
  const auto bounds = partition(ctx->ny, ctx->vc.levels, nslabs);
  auto grp = std::make_shared<SlabGroup>();
  HB_CUDA(cudaSetDevice(ctx->device));
  HB_CUDA(cudaStreamCreateWithFlags(&grp->stream, cudaStreamNonBlocking));
  for (int r = 0; r < nslabs; ++r) {
    hb_ctx* c = ctxs[r];
    HB_CUDA(cudaStreamSynchronize(c->stream));
    apply_slab(*c, r, bounds);
    auto st = std::make_shared<SlabState>();
    st->rank = r;
    st->nranks = nslabs;
    st->bounds = bounds;
    st->group = grp;
    if (!c->stream_own) c->stream_own = c->stream;
    c->stream = grp->stream;
    c->slab = st;
    grp->members.push_back(c);
  }
  HB_API_END
}

int hb_slab_rows(hb_ctx* ctx, int* row_begin, int* row_end) {
  HB_API_BEGIN
  if (!ctx->slab) throw HbError{HB_ERR_STATE, "not a slab context"};
  int lo, hi;
  proc_rows(*ctx, &lo, &hi);
  if (row_begin) *row_begin = lo;
  if (row_end) *row_end = hi;
  HB_API_END
}

int hb_precond_apply_slab(hb_ctx* ctx, int kind, int batch, const double* r, double* z) {
  HB_API_BEGIN
  if (kind != HB_PC_V) throw HbError{HB_ERR_ARG, "row slabs run the SL V-cycle preconditioner (M_V)"};
  if (!r || !z || batch < 1) throw HbError{HB_ERR_ARG, "bad buffers / batch"};
  auto S = members(*ctx);
  int plo, phi;
  proc_rows(*ctx, &plo, &phi);
  const int prows = phi - plo;
  const size_t R = S.size();
  std::vector<const int*> act(R);
  std::vector<const float*> fs(R, nullptr);
  std::vector<const float2*> f0(R);
  std::vector<float2*> zz(R);
  std::vector<std::vector<float2>> h(R);
  for (size_t s = 0; s < R; ++s) {
    Context& c = *S[s];
    ensure_batch(c, batch);
    const Level& L = *c.levels[0];
    c.io_f.ensure(L.N() * batch);
    c.io_g.ensure(L.N() * batch);
    // c128 host rows -> c64 storage (ghosts filled by the halo below)
    h[s].assign(L.N() * batch, make_float2(0.f, 0.f));
    for (int b = 0; b < batch; ++b)
      for (int y = L.lo; y < L.hi; ++y)
        for (int x = 0; x < L.nx; ++x) {
          const double* p = r + 2 * ((size_t(b) * prows + (y - plo)) * L.nx + x);
          h[s][(size_t(b) * L.rows + (y - L.row0)) * L.nx + x] = make_float2(float(p[0]), float(p[1]));
        }
    HB_CUDA(cudaMemcpyAsync(c.io_f.p, h[s].data(), h[s].size() * sizeof(float2), cudaMemcpyHostToDevice, c.stream));
    act[s] = c.act_all.p;
    f0[s] = c.io_f.p;
    zz[s] = c.io_g.p;
  }
  halo(S, 0, batch, sizeof(float2), [](Context& c, int, int) -> void* { return c.io_f.p; }, 0);
  slab_vcycle(S, batch, act, f0, fs, zz);
  for (size_t s = 0; s < R; ++s) {
    Context& c = *S[s];
    HB_CUDA(cudaMemcpyAsync(h[s].data(), c.io_g.p, h[s].size() * sizeof(float2), cudaMemcpyDeviceToHost, c.stream));
    HB_CUDA(cudaStreamSynchronize(c.stream));
    const Level& L = *c.levels[0];
    for (int b = 0; b < batch; ++b)
      for (int y = L.lo; y < L.hi; ++y)
        for (int x = 0; x < L.nx; ++x) {
          const float2 v = h[s][(size_t(b) * L.rows + (y - L.row0)) * L.nx + x];
          double* p = z + 2 * ((size_t(b) * prows + (y - plo)) * L.nx + x);
          p[0] = v.x;
          p[1] = v.y;
        }
  }
  HB_API_END
}

int hb_fgmres_slab(hb_ctx* ctx, const hb_krylov_cfg* cfg, int kind, int batch, const double* B, const double* X0,
                   double* X, double* hist, int hist_stride, int* hist_len, int* iters, uint8_t* converged,
                   uint8_t* breakdown) {
  HB_API_BEGIN
  if (!B || !X || batch < 1) throw HbError{HB_ERR_ARG, "bad buffers / batch"};
  auto S = members(*ctx);
  int plo, phi;
  proc_rows(*ctx, &plo, &phi);
  for (Context* c : S) {
    ensure_batch(*c, batch);
    const size_t n = c->levels[0]->N() * size_t(batch);
    c->kB.ensure(n);
    c->kX.ensure(n);
  }
  scatter_rows(S, batch, B, plo, phi - plo, false);
  scatter_rows(S, batch, X0, plo, phi - plo, true);
  slab_fgmres(S, cfg, kind, batch);
  gather_rows(S, batch, X, plo, phi - plo);
  HB_CUDA(cudaStreamSynchronize(S[0]->stream));
  if (hist || hist_len || iters || converged || breakdown)
    krylov_report(*S[0], batch, hist, hist_stride, hist_len, iters, converged, breakdown);
  HB_API_END
}

}  // extern "C"
