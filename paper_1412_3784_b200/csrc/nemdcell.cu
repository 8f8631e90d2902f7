// nemdcell.cu -- C-ABI (include/nemdcell.h) over the sm_100a kernels in
// kernels.cuh.  Host side: context, buffers, geometry (geom.hpp), launch
// sequencing on the caller's stream, pointer-kind handling, deterministic
// reductions and error reporting.  No torch types, no exceptions across the ABI.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/nemdcell.h"
#include "geom.hpp"
#include "kernels.cuh"

using namespace nc;

struct nc_ctx {
  nc_config cfg;
  // peer-memory data plane (nc_ipc_*): buffers this context exported, peer buffers it mapped, and the
  // interprocess events it created or opened
  std::vector<void*> ipc_own, ipc_open;
  std::vector<cudaEvent_t> ipc_ev;
  cudaStream_t stream = nullptr;
  std::string err;
  int64_t launches = 0;

  // geometry / flow
  bool have_box = false, have_flow = false, have_state = false, have_cells = false, have_eval = false;
  Geom g;
  double A[9] = {0};
  Policy pol;
  double t = 0.0;

  // capacity
  int64_t cap = 0, max_cells = 0, max_blocks = 0, max_layers = 0;

  // resident state (sorted by (cell, gid)), double-buffered q/p/gid
  void *st_q[2] = {nullptr, nullptr}, *st_p[2] = {nullptr, nullptr}, *st_F = nullptr;
  uint32_t* st_gid[2] = {nullptr, nullptr};
  int cur = 0;
  int64_t n_state = 0;

  // user-call scratch
  void *wq = nullptr;     // wrapped positions, input order (T4)
  void *sq = nullptr;     // sorted positions (T4)
  uint32_t* sgid = nullptr;
  void *sF = nullptr;     // sorted forces (T4)
  void *io_a = nullptr, *io_b = nullptr;  // n x 3 device staging for host pointers

  // shared transient
  double4* u = nullptr;   // sorted cell-local rotated coords, fp64 (w = sorted index)
  float4* u32 = nullptr;  // the same in fp32 (w = the cell column, exact): the filter's staging source
  uint32_t *nh = nullptr, *key = nullptr, *slot = nullptr;
  uint4* srec = nullptr;  // bucket records (source index, gid, cell key) of the counting sort
  uint32_t *counts = nullptr, *cs = nullptr, *bsum = nullptr, *tot = nullptr;
  // slab (multi-GPU) scratch
  uint32_t *gin = nullptr, *sidx = nullptr, *pbcnt = nullptr, *pboff = nullptr, *ptot = nullptr;
  uint8_t* cls = nullptr;
  double *bpart = nullptr, *lpart = nullptr, *part_tot = nullptr, *part_acc = nullptr;
  unsigned int* rcount = nullptr;  // k_reduce's last-block counter (kept at 0 between launches)
  // digest
  uint32_t* dcnt = nullptr;
  uint64_t *dhs = nullptr, *dhx = nullptr;
  unsigned long long* hist = nullptr;

  // last build bookkeeping
  int64_t n_last = 0;
  bool last_resident = false;     // last build used the resident state
  const uint32_t* last_in_gid = nullptr;  // gid of input order (nullptr = identity)
  int last_cpb = 0, last_bpl = 0;
  // SLLOD: the closing half kick of the last step is deferred (leapfrog-style) into the next
  // step's kick-drift kernel, or applied by k_kick when the resident state is read
  // pipelined host-buffer evaluations (nc_compute_forces_async): copy streams, double-buffered
  // device staging, events ordering copy-in -> evaluation -> copy-out per buffer
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  void* ain[2] = {nullptr, nullptr};
  void* aout[2] = {nullptr, nullptr};
  cudaEvent_t ev_in_ready[2] = {}, ev_in_free[2] = {}, ev_out_ready[2] = {}, ev_out_free[2] = {};
  bool ab_used[2] = {false, false};
  int ab = 0;
  bool async_eval = false;  // an evaluation was enqueued by the async call and not yet synced
  // a slab evaluation between nc_slab_forces_begin and nc_slab_forces_end
  int64_t slab_n_own = 0, slab_n1 = 0, slab_n2 = 0, slab_b_own = 0;
  int slab_klo = 0, slab_khi = 0;
  bool slab_open = false;
  void* fuser = nullptr;  // user-order force output of the evaluation in flight (the pair kernel writes it)
  // the previous user evaluation's sorted order (build_user pre-gathers the next input through it)
  uint32_t *perm = nullptr, *pgid = nullptr;
  void* pq = nullptr;
  int64_t perm_n = -1;
  // host-synchronization-free slab step (csrc/slab_dc.cuh): device counters and host-side bookkeeping
  uint32_t* sd = nullptr;
  int64_t sd_ncap = 0, sd_hcap = 0, sd_H = 0, sd_n_hint = 0;
  int sd_pre = 0;
  bool sd_open = false;
  int seg_nw = 2;  // warps per block of the sparse-cell kernel (seg_cells)
  bool kick_pending = false;
  bool count_tiers = false;  // nc_profile mode 2: k_pairs counts its fp32-tier interactions
  K3Kick pend{};
  int pair_kernel = NC_PK_AUTO;   // nc_set_pair_kernel
  int pair_kernel_used = 0;
  double occ_hint = -1.0;         // slab path: particles per cell of the own layers (auto kernel choice)
  double host_tot[NPART];
  bool tot_valid = false;
  int dbg_drop = 0;               // nc_debug negative control
  PairOut po{nullptr, nullptr, 0};  // nc_get_pairs: pair-list output of the next digest evaluation

  // slab data plane over NCCL (nccl_slab.cuh): communicator, its stream, scratch
  void* comm = nullptr;
  int comm_rank = 0, comm_nranks = 1;
  cudaStream_t s_comm = nullptr;
  cudaEvent_t ev_comm_in = nullptr, ev_comm_out = nullptr;
  int64_t* comm_cnt = nullptr;
  void* comm_gather = nullptr;
  size_t comm_gather_bytes = 0;
  bool comm_pending = false;

  // live kernel timing (nc_profile)
  bool prof = false;
  bool prof_pairs_only = false;
  int64_t counts_clean = 0;  // counts[0, counts_clean) known to be zero (cleared by the step's scatter)
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> prof_ev;
  std::vector<cudaEvent_t> ev_pool;
  cudaEvent_t prof_start = nullptr;
};

static thread_local std::string g_create_err;

namespace {

size_t tsize(const nc_ctx* c) { return c->cfg.prec == NC_F32 ? sizeof(float) : sizeof(double); }
size_t v4size(const nc_ctx* c) { return 4 * tsize(c); }

nc_status fail(nc_ctx* c, nc_status st, const std::string& msg) {
  if (c) c->err = msg; else g_create_err = msg;
  return st;
}

nc_status cuda_check(nc_ctx* c, cudaError_t e, const char* what) {
  if (e == cudaSuccess) return NC_OK;
  return fail(c, NC_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(expr)                                                   \
  do {                                                             \
    nc_status _s = cuda_check(ctx, (expr), #expr);                 \
    if (_s != NC_OK) return _s;                                    \
  } while (0)

#define LAUNCHED()                                                     \
  do {                                                                 \
    ctx->launches++;                                                   \
    nc_status _s = cuda_check(ctx, cudaGetLastError(), "kernel launch"); \
    if (_s != NC_OK) return _s;                                        \
  } while (0)

cudaEvent_t pool_event(nc_ctx* ctx) {
  if (!ctx->ev_pool.empty()) {
    cudaEvent_t e = ctx->ev_pool.back();
    ctx->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// RAII-free helpers: mark the start / end of one kernel launch of kind k
// (k: the kernel about to be timed; in pairs-only mode (nc_profile bit 4) only K3 gets events, so the
// instrumentation of a timed region is two events per evaluation)
inline void prof_begin(nc_ctx* ctx, int k = -1) {
  if (!ctx->prof || (ctx->prof_pairs_only && k != NC_K_PAIRS)) return;
  ctx->prof_start = pool_event(ctx);
  cudaEventRecord(ctx->prof_start, ctx->stream);
}
inline void prof_end(nc_ctx* ctx, int k) {
  if (!ctx->prof || (ctx->prof_pairs_only && k != NC_K_PAIRS)) return;
  cudaEvent_t e = pool_event(ctx);
  cudaEventRecord(e, ctx->stream);
  ctx->prof_ev.push_back({k, {ctx->prof_start, e}});
}

inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

// Launch with programmatic stream serialization (PDL, kernels.cuh PDL_ENTRY): the next grid is set up
// while this one drains.  NC_PDL=0 turns it off (A/B).  Every argument is passed explicitly.
inline bool pdl_on() {
  static const bool on = [] { const char* e = getenv("NC_PDL"); return !(e && e[0] == '0'); }();
  return on;
}
template <typename... P, typename... A>
inline cudaError_t launch_pdl(void (*k)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, A&&... a) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_on() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, std::forward<A>(a)...);
}

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) { cudaGetLastError(); return false; }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// NC_DEFER_KICK=0 launches k_kick at the end of every step (A/B runs)
bool defer_kick() {
  static const bool on = [] {
    const char* e = getenv("NC_DEFER_KICK");
    return !(e && e[0] == '0');
  }();
  return on;
}

// Cells per k_pairs block (one warp): more cells amortize the block prologue/epilogue (C4 DO: 4 / 8 /
// 16 cells -> 32.6 / 31.9 / 31.7 ms), fewer keep small grids busy (C0: 1 cell 0.089 ms vs 4 cells
// 0.315 ms; C2: 0.163 vs 0.178 ms).  The largest power of two <= K3_CELLS_MAX that still leaves
// K3_MIN_BLOCKS blocks (~32 waves of resident warps).  It depends on the global grid only, so
// every rank of a slab decomposition groups the same cells (bitwise-equal partial sums).
constexpr int64_t K3_MIN_BLOCKS = 75776;
// NC_F64 on grids below K3_F64_SPLIT_CELLS cells (fewer than ~4 waves of one-warp blocks): each cell's
// i-batches of 8 are spread over K3_F64_SPLIT blocks (a function of the global grid only: P-invariant)
constexpr int64_t K3_F64_SPLIT_CELLS = 8192;
#ifndef NC_F64_SPLIT
#define NC_F64_SPLIT 4
#endif
constexpr int K3_F64_SPLIT = NC_F64_SPLIT;
int cells_per_block(const Geom& g) {
  int cpb = K3_CELLS;
  while (cpb * 2 <= K3_CELLS_MAX && g.ncells / (cpb * 2) >= K3_MIN_BLOCKS) cpb *= 2;
  return cpb;
}

// Cells per segment of the sparse-cell kernel, 0 = use the warp-per-cell kernel.  Mean occupancy
// below 4 particles per cell (WCA at rho = 0.8442: ~1.3) selects segments of ~48 particles (two
// warps); nc_set_pair_kernel forces either kernel, NC_SEG=0 / NC_SEG=1 likewise (A/B runs).
int seg_cells(nc_ctx* ctx, const Geom& g) {
  static int env_mode = [] {
    const char* e = getenv("NC_SEG");
    return e ? (e[0] == '1' ? 1 : 0) : -1;
  }();
  int mode = ctx->pair_kernel == NC_PK_SEGMENT ? 1 : env_mode;
  if (mode == 0) return 0;
  const double occ = ctx->occ_hint >= 0.0 ? ctx->occ_hint
                                          : (double)ctx->n_last / (double)std::max<int64_t>(g.ncells, 1);
  if (mode < 0 && occ >= 4.0) return 0;
  // a fixed segment length (not occupancy-derived): block partials group the same cells on every
  // rank of a slab decomposition, so U and W stay bitwise independent of the rank count (P7).
  // 4 warps per block (96-cell segments) when that still leaves >= ~8 waves of blocks (large grids:
  // C3 0.728 vs 0.771 ms), else 2 (48 cells; C1 0.028 vs 0.037 ms) -- from the global grid only.
  const int64_t rows = (int64_t)g.dims[1] * g.dims[2];
  int NW = 2;
  if ((int64_t)((g.dims[0] + SgCfg<4>::GMAX - 1) / SgCfg<4>::GMAX) * rows >= 4736) NW = 4;
  int G = std::min(NW == 4 ? SgCfg<4>::GMAX : SgCfg<2>::GMAX, g.dims[0]);
  int64_t blocks = (int64_t)((g.dims[0] + G - 1) / G) * rows;
  if (blocks > ctx->max_blocks) return 0;
  ctx->seg_nw = NW;
  return G;
}

// Pair kernel for this grid: 0 = warp per cell (k_pairs), 1 = row segments (k_pairs_seg), 2 = one
// thread per particle (k_pairs_sparse; k_pairs_sparse64 in NC_F64), 3 = row windows (k_pairs_rows).
// AUTO below 4 particles per cell: the particle-per-thread kernel from 2^18 particles on and on grids
// below 65,536 cells (sparse_lpp: 2-8 threads per particle there), the row-segment kernel otherwise
// (DESIGN.md sections 5 and 7).
int sparse_kind(nc_ctx* ctx, const Geom& g) {
  if (ctx->cfg.prec != NC_F32) {  // NC_F64: the warp-per-cell kernel or k_pairs_sparse64
    if (ctx->pair_kernel == NC_PK_SPARSE) return 2;
    if (ctx->pair_kernel != NC_PK_AUTO) return 0;
    // sparse cells (C1 in fp64: pair kernel 0.106 -> 0.027 ms, DO) get one thread per particle
    const double occ64 = ctx->occ_hint >= 0.0 ? ctx->occ_hint
                                              : (double)ctx->n_last / (double)std::max<int64_t>(g.ncells, 1);
    return occ64 < 4.0 ? 2 : 0;
  }
  if (ctx->pair_kernel == NC_PK_CELL) return 0;
  if (ctx->pair_kernel == NC_PK_SEGMENT) return 1;
  if (ctx->pair_kernel == NC_PK_SPARSE) return 2;
  if (ctx->pair_kernel == NC_PK_ROWS) return 3;
  static int env_mode = [] {
    const char* e = getenv("NC_SEG");
    return e ? (e[0] == '1' ? 1 : 0) : -1;
  }();
  const double occ = ctx->occ_hint >= 0.0 ? ctx->occ_hint
                                          : (double)ctx->n_last / (double)std::max<int64_t>(g.ncells, 1);
  if (env_mode == 0 || occ >= 4.0) return 0;
  // thread-per-particle wins once the grid fills the GPU (C3 DO 0.68 vs 0.72 ms, DS 0.67 vs 0.86 ms);
  // below 65,536 cells the particle-per-thread kernel with 2-8 threads per particle beats the row-segment
  // kernel (C1: 36.9 vs 40.8 us per DO step; the paper's E2 system: 24.0 vs 29.0 us)
  if (g.ncells < SP_LPP2_CELLS) return 2;  // with 2 / 4 / 8 threads per particle (sparse_lpp)
  return ctx->n_last >= (1 << 18) ? 2 : 1;
}

// Threads per particle of k_pairs_sparse: 8 below 2,048 cells, 4 below 8,192, 2 below 65,536 (the
// kernel's chain per warp, not the GPU's throughput, bounds such grids: C1 36.9 vs 42.0 us per step with
// one thread, C3's 1.7M cells 0.72 vs 0.52 ms the other way), else 1.  NC_SP_LPP=1/2/4/8 forces one.  A function of the
// grid only, so slab ranks and one device agree.
int sparse_lpp(nc_ctx* ctx, const Geom& g) {
  (void)ctx;
  static int env = [] { const char* e = getenv("NC_SP_LPP"); return e ? atoi(e) : 0; }();
  if (env == 1 || env == 2 || env == 4 || env == 8) return env;
  if (g.ncells < SP_LPP_CELLS / 4) return 8;  // E2 (1,331 cells)
  if (g.ncells < SP_LPP_CELLS) return 4;
  return g.ncells < SP_LPP2_CELLS ? 2 : 1;    // C1 (24,389 cells): 2 threads per particle
}

nc_status apply_box(nc_ctx* ctx, const double* L) {
  Geom g;
  int st = make_geom(g, L, (int)ctx->cfg.variant, ctx->cfg.rc);
  if (st == GEOM_BAD_BOX) return fail(ctx, NC_E_BOX, "box matrix has det <= 0 or a non-finite entry");
  if (st == GEOM_DEGENERATE)
    return fail(ctx, NC_E_DEGENERATE,
                "degenerate cell grid (DS needs c_k >= 3; DO needs l1,l2 >= 4 and l3 >= 3): dims " +
                    std::to_string(g.dims[0]) + "x" + std::to_string(g.dims[1]) + "x" + std::to_string(g.dims[2]));
  if (g.ncells > ctx->max_cells)
    return fail(ctx, NC_E_OOM, "cell count " + std::to_string(g.ncells) + " exceeds max_cells " +
                                   std::to_string(ctx->max_cells));
  int cpb = cells_per_block(g);
  int64_t bpl = (((int64_t)g.dims[0] * g.dims[1]) + cpb - 1) / cpb;
  if (bpl * g.dims[2] > ctx->max_blocks || g.dims[2] > ctx->max_layers)
    return fail(ctx, NC_E_OOM, "block/layer partial buffers too small for this grid");
  g.eps = ctx->cfg.eps;
  g.sig2 = ctx->cfg.sigma * ctx->cfg.sigma;
  g.ushift = ctx->cfg.u_shift;
  // fp32 superset band: the dot-form filter's cancellation error (<~ 1e-5 sigma^2) stays far inside it
  double tau = ctx->cfg.prec == NC_F32 ? 1e-4 : 1e-10;
  g.band_lo = g.rc2 * (1.0 - tau);
  g.band_hi = g.rc2 * (1.0 + tau);
  // two-tier evaluation: fp32 force math only where the LJ force is small
  // (r >= 1.2 sigma: |f| <= 2.4 eps/sigma), fp64 for closer pairs
  // r_split = 1.2 sigma: the fp32 far tier's position rounding costs <= ~3e-5 eps/sigma per pair above it
  // (NC_RSPLIT: an experiment override, in units of sigma)
  static const double rsplit_env = [] { const char* e = getenv("NC_RSPLIT"); return e ? atof(e) : 1.2; }();
  g.rsplit2 = rsplit_env * rsplit_env * g.sig2;
  g.f_split2 = (float)g.rsplit2;
  g.f_lo = (float)g.band_lo;
  g.f_hi = (float)g.band_hi;
  g.f_sig2 = (float)g.sig2;
  g.f_c48 = (float)(48.0 * g.eps);
  g.f_m24 = (float)(-24.0 * g.eps);
  // fp32 staging frame: centred on the cell (DS: u = R (lambda - a/c) spans R [0, 1/c); DO: [0, w)),
  // R_i = the largest |u - cc| over the cell (half its longest diagonal)
  double Ri = 0.0;
  if (g.variant == 0) {
    const double h0 = 0.5 * g.cinv[0], h1 = 0.5 * g.cinv[1], h2 = 0.5 * g.cinv[2];
    g.cc[0] = g.R[0] * h0 + g.R[1] * h1 + g.R[2] * h2;
    g.cc[1] = g.R[4] * h1 + g.R[5] * h2;
    g.cc[2] = g.R[8] * h2;
    for (int sx = -1; sx <= 1; sx += 2)
      for (int sy = -1; sy <= 1; sy += 2) {
        const double x = g.R[0] * sx * h0 + g.R[1] * sy * h1 + g.R[2] * h2, y = g.R[4] * sy * h1 + g.R[5] * h2,
                     z = g.R[8] * h2;
        Ri = std::max(Ri, std::sqrt(x * x + y * y + z * z));
      }
  } else {
    for (int k = 0; k < 3; ++k) g.cc[k] = 0.5 * g.w[k];
    Ri = std::sqrt(g.cc[0] * g.cc[0] + g.cc[1] * g.cc[1] + g.cc[2] * g.cc[2]);
  }
  for (int k = 0; k < 3; ++k) g.f_cc[k] = (float)g.cc[k];
  Ri *= 1.0 + 1e-6;  // clamped keys (R14) may leave a particle ~1 ulp outside its cell
  // tensor-core filter bound (kernels.cuh, mma_filter): tf32 operands (x, y, z truncated to 10
  // mantissa bits, |v|^2 rounded) give |r~^2 - r^2| <= 2^-10 4.01 |u_i| |v_j| + 2^-11 |v_j|^2, with
  // |u_i| <= R_i and |v_j| <= R_i + r_c inside the cutoff; plus 1e-4 r_c^2 for the fp32 accumulation
  // and the two-part row constant
  const double vmax = Ri + ctx->cfg.rc;
  g.f_hmma = (float)(g.rc2 + std::ldexp(4.01 * Ri * vmax, -10) + std::ldexp(vmax * vmax, -11) + 1e-4 * g.rc2);
  g.dbg_drop = ctx->dbg_drop;
  ctx->g = g;
  ctx->have_box = true;
  return NC_OK;
}

// exclusive scan of m counts into out[0..m] (out[m] = total); one launch for small m
nc_status launch_scan_raw(nc_ctx* ctx, const uint32_t* in, int64_t m, uint32_t* out) {
  cudaStream_t s = ctx->stream;
  if (m <= SCAN_SMALL) {
    launch_pdl(k_scan_small, dim3(1), dim3(SCAN_SMALL_T), 0, s, in, m, out);
    LAUNCHED();
  } else {
    const int64_t nb = (m + SCAN_TILE - 1) / SCAN_TILE;
    launch_pdl(k_scan_reduce, dim3((unsigned)nb), dim3(SCAN_T), 0, s, in, m, ctx->bsum);
    LAUNCHED();
    launch_pdl(k_scan_bsums, dim3(1), dim3(1024), 0, s, ctx->bsum, nb, ctx->tot);
    LAUNCHED();
    launch_pdl(k_scan_apply, dim3((unsigned)nb), dim3(SCAN_T), 0, s, in, m, (const uint32_t*)ctx->bsum, out,
               (const uint32_t*)ctx->tot);
    LAUNCHED();
  }
  return NC_OK;
}
nc_status launch_scan(nc_ctx* ctx, const uint32_t* in, int64_t m, uint32_t* out) {
  prof_begin(ctx);
  nc_status st = launch_scan_raw(ctx, in, m, out);
  if (st) return st;
  prof_end(ctx, NC_K_SCAN);
  return NC_OK;
}

template <typename T>
nc_status launch_build(nc_ctx* ctx, const T* qin, int stride, typename V4<T>::t* qwrap, int64_t n,
                       const uint32_t* gid_in, const typename V4<T>::t* p_in, typename V4<T>::t* q_out,
                       typename V4<T>::t* p_out, uint32_t* gid_out) {
  cudaStream_t s = ctx->stream;
  const Geom& g = ctx->g;
  int64_t C = g.ncells;
  CK(cudaMemsetAsync(ctx->counts, 0, sizeof(uint32_t) * (C + 1), s));
  ctx->counts_clean = 0;  // this build leaves the histogram filled
  if (n > 0) {
    prof_begin(ctx);
    launch_pdl(k_wrap_key<T>, dim3(nblk(n, 256)), dim3(256), 0, s, n, qin, stride, qwrap, ctx->key, ctx->slot,
               ctx->counts, g);
    LAUNCHED();
    prof_end(ctx, NC_K_WRAPKEY);
  }
  {
    nc_status sst = launch_scan(ctx, ctx->counts, C, ctx->cs);
    if (sst) return sst;
  }
  if (n > 0) {
    prof_begin(ctx);
    launch_pdl(k_scatter, dim3(nblk(n, 256)), dim3(256), 0, s, n, (const uint32_t*)ctx->key,
               (const uint32_t*)ctx->slot, (const uint32_t*)ctx->cs, gid_in, ctx->srec, (int64_t)0,
               (const uint32_t*)nullptr, (uint32_t*)nullptr, (int64_t)0);
    LAUNCHED();
    prof_end(ctx, NC_K_SCATTER);
    prof_begin(ctx);
    launch_pdl(k_rank_gather<T>, dim3(nblk(n, 256)), dim3(256), 0, s, n, (const uint4*)ctx->srec,
               (const uint32_t*)ctx->cs, (const typename V4<T>::t*)qwrap, p_in, q_out, p_out, gid_out, ctx->u, ctx->u32,
               ctx->nh, g, (uint32_t*)nullptr, (int64_t)0, (const uint32_t*)nullptr);
    LAUNCHED();
    prof_end(ctx, NC_K_RANKGATHER);
  }
  ctx->n_last = n;
  ctx->last_in_gid = gid_in;
  ctx->have_cells = true;
  return NC_OK;
}

template <typename T, bool DIGEST>
nc_status launch_pairs(nc_ctx* ctx, const typename V4<T>::t* qs, const uint32_t* gid, typename V4<T>::t* F,
                       int layer0 = 0, int nlay = -1, int part_layer0 = -1, bool reduce = true) {
  // part_layer0: the layer whose block partials start bpart (default layer0); a slab evaluation
  // launches its layers in two parts and reduces once (reduce = false for the parts)
  cudaStream_t s = ctx->stream;
  const Geom& g = ctx->g;
  if (part_layer0 < 0) part_layer0 = layer0;
  if (nlay < 0) nlay = g.dims[2];
  int cpb = cells_per_block(g);
  int bpl = (int)((((int64_t)g.dims[0] * g.dims[1]) + cpb - 1) / cpb);
  if (sizeof(T) == 8 && g.ncells < K3_F64_SPLIT_CELLS) {  // NC_F64 on a small grid: 4 blocks per cell
    cpb = -K3_F64_SPLIT;
    bpl = (int)((int64_t)g.dims[0] * g.dims[1] * K3_F64_SPLIT);
  }
  int nblocks = bpl * nlay;
  size_t smem = sizeof(K3Smem<T>);
  (void)nblocks;
  const PairOut po = DIGEST ? ctx->po : PairOut{nullptr, nullptr, 0, ctx->fuser};
  prof_begin(ctx, NC_K_PAIRS);
  double* bp = nullptr;  // set once bpl is final (below)
  if constexpr (sizeof(T) == 4) {
    const int Gseg = sparse_kind(ctx, g) == 1 ? seg_cells(ctx, g) : 0;
    if (sparse_kind(ctx, g) == 3) {  // sparse cells: one warp per cell row, staged neighbour rows (k3_rows.cuh)
      bpl = (g.dims[1] + RW_NW - 1) / RW_NW;  // a function of the grid only (P-invariant)
      nblocks = bpl * nlay;
      bp = ctx->bpart + (int64_t)(layer0 - part_layer0) * bpl * NPART;
      ctx->pair_kernel_used = NC_PK_ROWS;
      launch_pdl(k_pairs_rows<DIGEST>, dim3(nblocks), dim3(32 * RW_NW), sizeof(RwSmem), s, (const double4*)ctx->u,
                 (const float4*)ctx->u32, (const uint32_t*)ctx->cs, (const float4*)qs, (const uint32_t*)ctx->nh, gid,
                 (float4*)F, bp, ctx->dcnt, ctx->dhs, ctx->dhx, g, bpl, layer0, po);
    } else if (sparse_kind(ctx, g) == 2) {  // sparse cells: one thread per particle (k3_sparse.cuh)
      // small systems: four threads per particle (more warps, a quarter of the rows each)
      const int lpp = sparse_lpp(ctx, g);
      const int cpb = SP_CPB / lpp;
      bpl = (int)(((int64_t)g.dims[0] * g.dims[1] + cpb - 1) / cpb);  // a function of the grid only (P-invariant)
      nblocks = bpl * nlay;
      bp = ctx->bpart + (int64_t)(layer0 - part_layer0) * bpl * NPART;
      ctx->pair_kernel_used = NC_PK_SPARSE;
      if (lpp == 2)
        launch_pdl(k_pairs_sparse<DIGEST, 2>, dim3(nblocks), dim3(SP_NT), sizeof(SpSmem), s, (const double4*)ctx->u,
                   (const float4*)ctx->u32, (const uint32_t*)ctx->cs, (const uint4*)ctx->srec, (const float4*)qs,
                   (const uint32_t*)ctx->nh, gid, (float4*)F, bp, ctx->dcnt, ctx->dhs, ctx->dhx, g, bpl, layer0, po);
      else if (lpp == 8)
        launch_pdl(k_pairs_sparse<DIGEST, 8>, dim3(nblocks), dim3(SP_NT), sizeof(SpSmem), s, (const double4*)ctx->u,
                   (const float4*)ctx->u32, (const uint32_t*)ctx->cs, (const uint4*)ctx->srec, (const float4*)qs,
                   (const uint32_t*)ctx->nh, gid, (float4*)F, bp, ctx->dcnt, ctx->dhs, ctx->dhx, g, bpl, layer0, po);
      else if (lpp == 4)
        launch_pdl(k_pairs_sparse<DIGEST, 4>, dim3(nblocks), dim3(SP_NT), sizeof(SpSmem), s, (const double4*)ctx->u,
                   (const float4*)ctx->u32, (const uint32_t*)ctx->cs, (const uint4*)ctx->srec, (const float4*)qs,
                   (const uint32_t*)ctx->nh, gid, (float4*)F, bp, ctx->dcnt, ctx->dhs, ctx->dhx, g, bpl, layer0, po);
      else
        launch_pdl(k_pairs_sparse<DIGEST, 1>, dim3(nblocks), dim3(SP_NT), sizeof(SpSmem), s, (const double4*)ctx->u,
                   (const float4*)ctx->u32, (const uint32_t*)ctx->cs, (const uint4*)ctx->srec, (const float4*)qs,
                   (const uint32_t*)ctx->nh, gid, (float4*)F, bp, ctx->dcnt, ctx->dhs, ctx->dhx, g, bpl, layer0, po);
    } else if (Gseg > 0) {  // sparse cells: one warp per row segment of Gseg cells (k3_seg.cuh)
      const int nseg = (g.dims[0] + Gseg - 1) / Gseg;
      const int bpl_s = nseg * g.dims[1];
      const size_t smem_s = ctx->seg_nw == 4 ? sizeof(SgSmem<4>) : sizeof(SgSmem<2>);
      bpl = bpl_s;
      nblocks = bpl * nlay;
      bp = ctx->bpart + (int64_t)(layer0 - part_layer0) * bpl * NPART;
      ctx->pair_kernel_used = NC_PK_SEGMENT;
      if (ctx->seg_nw == 4)
        launch_pdl(k_pairs_seg<DIGEST, 4>, dim3(nblocks), dim3(SgCfg<4>::NT), smem_s, s, (const double4*)ctx->u,
                   (const float4*)ctx->u32, (const uint32_t*)ctx->cs, (const float4*)qs, (const uint32_t*)ctx->nh, gid,
                   (float4*)F, bp, ctx->dcnt, ctx->dhs, ctx->dhx, g, Gseg, nseg, bpl, layer0, po);
      else
        launch_pdl(k_pairs_seg<DIGEST, 2>, dim3(nblocks), dim3(SgCfg<2>::NT), smem_s, s, (const double4*)ctx->u,
                   (const float4*)ctx->u32, (const uint32_t*)ctx->cs, (const float4*)qs, (const uint32_t*)ctx->nh, gid,
                   (float4*)F, bp, ctx->dcnt, ctx->dhs, ctx->dhx, g, Gseg, nseg, bpl, layer0, po);
    } else {
      ctx->pair_kernel_used = NC_PK_CELL;
      bp = ctx->bpart + (int64_t)(layer0 - part_layer0) * bpl * NPART;
      if (!DIGEST && ctx->count_tiers)
        launch_pdl(k_pairs<T, DIGEST, true>, dim3(nblocks), dim3(32), smem, s, (const double4*)ctx->u,
                   (const float4*)ctx->u32, (const uint32_t*)ctx->cs, qs, (const uint32_t*)ctx->nh, gid, F, bp,
                   ctx->dcnt, ctx->dhs, ctx->dhx, g, cpb, bpl, layer0, po);
      else
        launch_pdl(k_pairs<T, DIGEST, false>, dim3(nblocks), dim3(32), smem, s, (const double4*)ctx->u,
                   (const float4*)ctx->u32, (const uint32_t*)ctx->cs, qs, (const uint32_t*)ctx->nh, gid, F, bp,
                   ctx->dcnt, ctx->dhs, ctx->dhx, g, cpb, bpl, layer0, po);
    }
  } else if (sparse_kind(ctx, g) == 2) {  // NC_F64 sparse cells: one thread per particle (k3_sparse64.cuh)
    const int lpp = sparse_lpp(ctx, g) >= 2 ? 2 : 1;  // two threads per particle on small grids
    const int cpb64 = SP_CPB / lpp;
    bpl = (int)(((int64_t)g.dims[0] * g.dims[1] + cpb64 - 1) / cpb64);  // a function of the grid only
    nblocks = bpl * nlay;
    bp = ctx->bpart + (int64_t)(layer0 - part_layer0) * bpl * NPART;
    ctx->pair_kernel_used = NC_PK_SPARSE;
    if (lpp == 2)
      launch_pdl(k_pairs_sparse64<DIGEST, 2>, dim3(nblocks), dim3(SP_NT), sizeof(Sp64Smem), s, (const uint32_t*)ctx->cs,
                 (const uint4*)ctx->srec, (const double4*)qs, (const uint32_t*)ctx->nh, gid, (double4*)F, bp,
                 ctx->dcnt, ctx->dhs, ctx->dhx, g, bpl, layer0, po);
    else
      launch_pdl(k_pairs_sparse64<DIGEST, 1>, dim3(nblocks), dim3(SP_NT), sizeof(Sp64Smem), s, (const uint32_t*)ctx->cs,
                 (const uint4*)ctx->srec, (const double4*)qs, (const uint32_t*)ctx->nh, gid, (double4*)F, bp,
                 ctx->dcnt, ctx->dhs, ctx->dhx, g, bpl, layer0, po);
  } else {
    ctx->pair_kernel_used = NC_PK_CELL;
    bp = ctx->bpart + (int64_t)(layer0 - part_layer0) * bpl * NPART;
    launch_pdl(k_pairs<T, DIGEST, false>, dim3(nblocks), dim3(32), smem, s, (const double4*)ctx->u,
               (const float4*)ctx->u32, (const uint32_t*)ctx->cs, qs, (const uint32_t*)ctx->nh, gid, F, bp, ctx->dcnt,
               ctx->dhs, ctx->dhx, g, cpb, bpl, layer0, po);
  }
  LAUNCHED();
  prof_end(ctx, NC_K_PAIRS);
  ctx->last_cpb = cpb;
  ctx->last_bpl = bpl;
  if (reduce) {
    const int nl = layer0 + nlay - part_layer0;  // every layer whose partials start at bpart
    prof_begin(ctx);
    launch_pdl(k_reduce, dim3(nl), dim3(K3R_T), 0, s, (const double*)ctx->bpart, bpl, nl, ctx->lpart, ctx->part_tot,
               ctx->part_acc, ctx->rcount);
    LAUNCHED();
    prof_end(ctx, NC_K_REDUCE);
  }
  ctx->last_bpl = bpl;
  ctx->tot_valid = false;
  ctx->have_eval = true;
  return NC_OK;
}

nc_status fetch_totals(nc_ctx* ctx) {
  if (ctx->tot_valid) return NC_OK;
  CK(cudaMemcpyAsync(ctx->host_tot, ctx->part_tot, sizeof(double) * NPART, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->tot_valid = true;
  return NC_OK;
}

// U and the lab-frame virial W = Q W_rot Q^T (W = (xx,yy,zz,xy,xz,yz))
void totals_to_UW(const nc_ctx* ctx, double* U, double* W) {
  const double* t = ctx->host_tot;
  if (U) *U = t[0];
  if (W && ctx->cfg.prec == NC_F64) {  // fp64 mode accumulates in the lab frame
    for (int k = 0; k < 6; ++k) W[k] = t[1 + k];
  } else if (W) {  // fp32 mode: rotated frame, W = Q W_rot Q^T
    double Wr[9] = {t[1], t[4], t[5], t[4], t[2], t[6], t[5], t[6], t[3]};
    const double* Q = ctx->g.Q;
    double X[9], Y[9];
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) X[3 * r + c] = Q[3 * r] * Wr[c] + Q[3 * r + 1] * Wr[3 + c] + Q[3 * r + 2] * Wr[6 + c];
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) Y[3 * r + c] = X[3 * r] * Q[3 * c] + X[3 * r + 1] * Q[3 * c + 1] + X[3 * r + 2] * Q[3 * c + 2];
    W[0] = Y[0]; W[1] = Y[4]; W[2] = Y[8]; W[3] = Y[1]; W[4] = Y[2]; W[5] = Y[5];
  }
}

nc_status check_finite(nc_ctx* ctx) {
  nc_status st = fetch_totals(ctx);
  if (st) return st;
  if (ctx->host_tot[NPART - 1] >= K3_OVERFLOW)
    return fail(ctx, NC_E_OOM, "a neighborhood holds more particles than the pair kernel can stage (cell kernel: " +
                                   std::to_string(K3_CAP) + " per cell; sparse-cell kernel: one neighborhood per "
                                   "segment union): too dense for this cutoff / kernel");
  bool ok = ctx->host_tot[NPART - 1] == 0.0;
  for (int k = 0; k < 7; ++k) ok = ok && std::isfinite(ctx->host_tot[k]);
  if (!ok) return fail(ctx, NC_E_NONFINITE, "non-finite force, energy or virial");
  return NC_OK;
}

// copy a caller n x 3 array to device staging if it is host memory
nc_status stage_in(nc_ctx* ctx, const void* src, void* dev_buf, int64_t n, const void** out) {
  if (is_device_ptr(src)) { *out = src; return NC_OK; }
  CK(cudaMemcpyAsync(dev_buf, src, 3 * tsize(ctx) * n, cudaMemcpyHostToDevice, ctx->stream));
  *out = dev_buf;
  return NC_OK;
}

template <typename T>
nc_status build_user(nc_ctx* ctx, const void* q, int64_t n) {
  const void* qd = nullptr;
  nc_status st = stage_in(ctx, q, ctx->io_a, n, &qd);
  if (st) return st;
  // A caller's particles keep their order from call to call (and move little): the previous call's
  // sorted order (sorted slot -> caller index) pre-gathers this call's positions, so the counting sort
  // sees an almost sorted input (coalesced scatter and gathers instead of random ones).  Only the
  // ORDER of the input changes -- the gids are the caller's indices, the (cell, gid) sort and every
  // result are exactly those without it.
  const T* src = (const T*)qd;
  const uint32_t* gsrc = nullptr;
  if (n > 0 && ctx->perm_n == n) {
    prof_begin(ctx);
    k_pregather<T><<<nblk(n, 256), 256, 0, ctx->stream>>>(n, (const T*)qd, ctx->perm, (T*)ctx->pq, ctx->pgid);
    LAUNCHED();
    prof_end(ctx, NC_K_OTHER);
    src = (const T*)ctx->pq;
    gsrc = ctx->pgid;
  }
  st = launch_build<T>(ctx, src, 3, (typename V4<T>::t*)ctx->wq, n, gsrc, nullptr, (typename V4<T>::t*)ctx->sq,
                       nullptr, ctx->sgid);
  if (st) return st;
  if (n > 0) {  // this call's sorted order (the sorted gids ARE caller indices) for the next call
    if (!ctx->perm) {
      CK(cudaMalloc(&ctx->perm, sizeof(uint32_t) * (size_t)ctx->cap));
      CK(cudaMalloc(&ctx->pgid, sizeof(uint32_t) * (size_t)ctx->cap));
      CK(cudaMalloc(&ctx->pq, 3 * sizeof(T) * (size_t)ctx->cap));
    }
    CK(cudaMemcpyAsync(ctx->perm, ctx->sgid, sizeof(uint32_t) * (size_t)n, cudaMemcpyDeviceToDevice, ctx->stream));
    ctx->perm_n = n;
  }
  ctx->last_resident = false;
  return NC_OK;
}

template <typename T>
nc_status unsort_out(nc_ctx* ctx, const void* src4, const uint32_t* gid, int64_t n, void* dst) {
  bool dev = is_device_ptr(dst);
  T* d = dev ? (T*)dst : (T*)ctx->io_b;
  if (n > 0) {
    prof_begin(ctx);
    k_unsort3<T><<<nblk(n, 256), 256, 0, ctx->stream>>>(n, (const typename V4<T>::t*)src4, gid, d);
    LAUNCHED();
    prof_end(ctx, NC_K_OTHER);
  }
  if (!dev) {
    CK(cudaMemcpyAsync(dst, ctx->io_b, 3 * sizeof(T) * n, cudaMemcpyDeviceToHost, ctx->stream));
  }
  return NC_OK;
}

template <typename T>
nc_status compute_user(nc_ctx* ctx, const void* q, int64_t n, void* F, double* U, double* W) {
  nc_status st = build_user<T>(ctx, q, n);
  if (st) return st;
  // the pair kernel writes F straight into the user order (device F, or the io_b staging buffer)
  const bool dev = F && is_device_ptr(F);
  ctx->fuser = F ? (dev ? F : ctx->io_b) : nullptr;
  st = launch_pairs<T, false>(ctx, (const typename V4<T>::t*)ctx->sq, ctx->sgid, (typename V4<T>::t*)ctx->sF);
  ctx->fuser = nullptr;
  if (st) return st;
  if (F && !dev && n > 0)
    CK(cudaMemcpyAsync(F, ctx->io_b, 3 * sizeof(T) * (size_t)n, cudaMemcpyDeviceToHost, ctx->stream));
  st = check_finite(ctx);  // synchronizes the stream
  if (st) return st;
  totals_to_UW(ctx, U, W);
  return NC_OK;
}

// Pipelined evaluation on host buffers: H2D on s_h2d, evaluation on the context stream, D2H on
// s_d2h, buffer b alternating, so the copies of one call overlap the evaluation of its neighbours.
template <typename T>
nc_status compute_async_t(nc_ctx* ctx, const void* q, int64_t n, void* F) {
  const size_t bytes = 3 * sizeof(T) * (size_t)n;
  if (!ctx->s_h2d) {
    CK(cudaStreamCreateWithFlags(&ctx->s_h2d, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&ctx->s_d2h, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
      CK(cudaMalloc(&ctx->ain[b], 3 * sizeof(T) * (size_t)ctx->cap));
      CK(cudaMalloc(&ctx->aout[b], 3 * sizeof(T) * (size_t)ctx->cap));
      CK(cudaEventCreateWithFlags(&ctx->ev_in_ready[b], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ctx->ev_in_free[b], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ctx->ev_out_ready[b], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ctx->ev_out_free[b], cudaEventDisableTiming));
    }
  }
  const int b = ctx->ab;
  ctx->ab ^= 1;
  cudaStream_t s = ctx->stream;
  // copy in (after the evaluation that last read this buffer)
  if (ctx->ab_used[b]) CK(cudaStreamWaitEvent(ctx->s_h2d, ctx->ev_in_free[b], 0));
  if (n > 0) CK(cudaMemcpyAsync(ctx->ain[b], q, bytes, cudaMemcpyHostToDevice, ctx->s_h2d));
  CK(cudaEventRecord(ctx->ev_in_ready[b], ctx->s_h2d));
  // evaluate (device pointers: no staging through io_a / io_b)
  CK(cudaStreamWaitEvent(s, ctx->ev_in_ready[b], 0));
  if (ctx->ab_used[b]) CK(cudaStreamWaitEvent(s, ctx->ev_out_free[b], 0));
  nc_status st = build_user<T>(ctx, ctx->ain[b], n);
  if (st) return st;
  CK(cudaEventRecord(ctx->ev_in_free[b], s));
  ctx->fuser = F ? ctx->aout[b] : nullptr;  // the pair kernel writes F in the user order
  st = launch_pairs<T, false>(ctx, (const typename V4<T>::t*)ctx->sq, ctx->sgid, (typename V4<T>::t*)ctx->sF);
  ctx->fuser = nullptr;
  if (st) return st;
  CK(cudaEventRecord(ctx->ev_out_ready[b], s));
  // copy out
  CK(cudaStreamWaitEvent(ctx->s_d2h, ctx->ev_out_ready[b], 0));
  if (F && n > 0) CK(cudaMemcpyAsync(F, ctx->aout[b], bytes, cudaMemcpyDeviceToHost, ctx->s_d2h));
  CK(cudaEventRecord(ctx->ev_out_free[b], ctx->s_d2h));
  ctx->ab_used[b] = true;
  ctx->async_eval = true;
  return NC_OK;
}

template <typename T>
nc_status set_state_t(nc_ctx* ctx, const void* q, const void* p, const int64_t* gid, int64_t n) {
  cudaStream_t s = ctx->stream;
  const void* qd = nullptr;
  const void* pd = nullptr;
  nc_status st = stage_in(ctx, q, ctx->io_a, n, &qd);
  if (st) return st;
  // pack into the current state buffers (input order), gid
  int c = ctx->cur;
  if (n > 0) {
    prof_begin(ctx);
    k_pack4<T><<<nblk(n, 256), 256, 0, s>>>(n, (const T*)qd, (typename V4<T>::t*)ctx->st_q[c]);
    LAUNCHED();
    prof_end(ctx, NC_K_OTHER);
  }
  if (p) {
    st = stage_in(ctx, p, ctx->io_b, n, &pd);
    if (st) return st;
    if (n > 0) {
      prof_begin(ctx);
      k_pack4<T><<<nblk(n, 256), 256, 0, s>>>(n, (const T*)pd, (typename V4<T>::t*)ctx->st_p[c]);
      LAUNCHED();
      prof_end(ctx, NC_K_OTHER);
    }
  } else {
    CK(cudaMemsetAsync(ctx->st_p[c], 0, v4size(ctx) * n, s));
  }
  std::vector<uint32_t> hg(n);
  for (int64_t i = 0; i < n; ++i) hg[i] = gid ? (uint32_t)gid[i] : (uint32_t)i;
  CK(cudaMemcpyAsync(ctx->st_gid[c], hg.data(), sizeof(uint32_t) * n, cudaMemcpyHostToDevice, s));
  // build from the packed state (stride 4), in place wrap, gather into the other buffers
  int o = 1 - c;
  st = launch_build<T>(ctx, (const T*)ctx->st_q[c], 4, (typename V4<T>::t*)ctx->st_q[c], n, ctx->st_gid[c],
                       (const typename V4<T>::t*)ctx->st_p[c], (typename V4<T>::t*)ctx->st_q[o],
                       (typename V4<T>::t*)ctx->st_p[o], ctx->st_gid[o]);
  if (st) return st;
  CK(cudaStreamSynchronize(s));  // hg lifetime
  ctx->cur = o;
  ctx->n_state = n;
  ctx->last_resident = true;
  st = launch_pairs<T, false>(ctx, (const typename V4<T>::t*)ctx->st_q[o], ctx->st_gid[o],
                              (typename V4<T>::t*)ctx->st_F);
  if (st) return st;
  st = check_finite(ctx);
  if (st) return st;
  ctx->have_state = true;
  return NC_OK;
}

template <typename T>
nc_status step_t(nc_ctx* ctx, double dt, int nsteps, double* U, double* W) {
  cudaStream_t s = ctx->stream;
  int64_t n = ctx->n_state;
  SllodParams sp;
  expm3(ctx->A, -0.5 * dt, sp.Em);
  expm3(ctx->A, dt, sp.Ed);
  expm3(ctx->A, 0.5 * dt, sp.Eh);
  sp.dt = dt;
  sp.inv_m = 1.0 / ctx->cfg.mass;
  for (int k = 0; k < nsteps; ++k) {
    // new box at t + dt (remapped) before the drift+wrap kernel
    double Lnew[9];
    box_advance(ctx->pol, ctx->A, ctx->t + dt, Lnew);
    nc_status st = apply_box(ctx, Lnew);
    if (st) return st;
    ctx->t += dt;
    int c = ctx->cur, o = 1 - c;
    const Geom& g = ctx->g;
    // the counts are zeroed by the previous step's scatter (below, up to its grid's C + 1); the first step
    // of a call, and a step whose grid grew, clear them here
    if (g.ncells + 1 > ctx->counts_clean)
      CK(cudaMemsetAsync(ctx->counts, 0, sizeof(uint32_t) * (g.ncells + 1), s));
    ctx->counts_clean = 0;  // (kick-drift-key fills it; the scatter below clears it again)
    if (n > 0) {
      prof_begin(ctx);
      launch_pdl(k_kick_drift_key<T>, dim3(nblk(n, 256)), dim3(256), 0, s, n, (typename V4<T>::t*)ctx->st_q[c],
                 (typename V4<T>::t*)ctx->st_p[c], (const typename V4<T>::t*)ctx->st_F, sp, g, ctx->key, ctx->slot,
                 ctx->counts, ctx->kick_pending ? 1 : 0, ctx->pend);
      LAUNCHED();
      ctx->kick_pending = false;
      prof_end(ctx, NC_K_WRAPKEY);
    }
    int64_t C = g.ncells;
    {
      nc_status sst = launch_scan(ctx, ctx->counts, C, ctx->cs);
      if (sst) return sst;
    }
    if (n > 0) {
      prof_begin(ctx);
      launch_pdl(k_scatter, dim3(nblk(n, 256)), dim3(256), 0, s, n, (const uint32_t*)ctx->key,
                 (const uint32_t*)ctx->slot, (const uint32_t*)ctx->cs, (const uint32_t*)ctx->st_gid[c], ctx->srec,
                 (int64_t)0, (const uint32_t*)nullptr, ctx->counts, C + 1);
      ctx->counts_clean = C + 1;
      LAUNCHED();
      prof_end(ctx, NC_K_SCATTER);
      prof_begin(ctx);
      launch_pdl(k_rank_gather<T>, dim3(nblk(n, 256)), dim3(256), 0, s, n, (const uint4*)ctx->srec,
                 (const uint32_t*)ctx->cs, (const typename V4<T>::t*)ctx->st_q[c],
                 (const typename V4<T>::t*)ctx->st_p[c], (typename V4<T>::t*)ctx->st_q[o],
                 (typename V4<T>::t*)ctx->st_p[o], ctx->st_gid[o], ctx->u, ctx->u32, ctx->nh, g, (uint32_t*)nullptr,
                 (int64_t)0, (const uint32_t*)nullptr);
      LAUNCHED();
      prof_end(ctx, NC_K_RANKGATHER);
    }
    ctx->cur = o;
    ctx->n_last = n;
    ctx->last_in_gid = ctx->st_gid[c];
    ctx->last_resident = true;
    ctx->have_cells = true;
    st = launch_pairs<T, false>(ctx, (const typename V4<T>::t*)ctx->st_q[o], ctx->st_gid[o],
                                (typename V4<T>::t*)ctx->st_F);
    if (st) return st;
    // closing half kick p <- E(-dt/2) p + dt/2 F: deferred into the next step's kick-drift pass
    // (same arithmetic; k_kick applies it instead when the state is read, see materialize_kick)
    if (n > 0 && defer_kick()) {
      for (int e = 0; e < 9; ++e) ctx->pend.Em[e] = sp.Em[e];
      ctx->pend.hd = 0.5 * dt;
      ctx->kick_pending = true;
    } else if (n > 0) {
      prof_begin(ctx);
      k_kick<T><<<nblk(n, 256), 256, 0, s>>>(n, (typename V4<T>::t*)ctx->st_p[o], (const typename V4<T>::t*)ctx->st_F, sp);
      LAUNCHED();
      prof_end(ctx, NC_K_KICK);
    }
  }
  if (U || W) {
    nc_status st = check_finite(ctx);
    if (st) return st;
    totals_to_UW(ctx, U, W);
  }
  return NC_OK;
}

// Apply a deferred closing half kick to the resident momenta (k_kick with the deferring step's
// E(-dt/2) and dt/2; bitwise what the fused path computes).
template <typename T>
nc_status materialize_kick_t(nc_ctx* ctx) {
  if (!ctx->kick_pending) return NC_OK;
  const int64_t n = ctx->n_state;
  SllodParams sp{};
  for (int e = 0; e < 9; ++e) sp.Em[e] = ctx->pend.Em[e];
  sp.dt = 2.0 * ctx->pend.hd;
  ctx->kick_pending = false;
  if (n > 0) {
    prof_begin(ctx);
    k_kick<T><<<nblk(n, 256), 256, 0, ctx->stream>>>(n, (typename V4<T>::t*)ctx->st_p[ctx->cur],
                                                      (const typename V4<T>::t*)ctx->st_F, sp);
    LAUNCHED();
    prof_end(ctx, NC_K_KICK);
  }
  return NC_OK;
}
nc_status materialize_kick(nc_ctx* ctx) {
  return ctx->cfg.prec == NC_F32 ? materialize_kick_t<float>(ctx) : materialize_kick_t<double>(ctx);
}

template <typename T>
nc_status digest_t(nc_ctx* ctx, uint32_t* cnt, uint64_t* hsum, uint64_t* hxor) {
  const void* qs = ctx->last_resident ? ctx->st_q[ctx->cur] : ctx->sq;
  const uint32_t* gid = ctx->last_resident ? ctx->st_gid[ctx->cur] : ctx->sgid;
  nc_status st = launch_pairs<T, true>(ctx, (const typename V4<T>::t*)qs, gid, (typename V4<T>::t*)ctx->sF);
  if (st) return st;
  int64_t n = ctx->n_last;
  std::vector<uint32_t> c(n), gg(n);
  std::vector<uint64_t> a(n), b(n);
  CK(cudaMemcpyAsync(c.data(), ctx->dcnt, 4 * n, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(a.data(), ctx->dhs, 8 * n, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(b.data(), ctx->dhx, 8 * n, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(gg.data(), gid, 4 * n, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  for (int64_t s = 0; s < n; ++s) {
    if (cnt) cnt[gg[s]] = c[s];
    if (hsum) hsum[gg[s]] = a[s];
    if (hxor) hxor[gg[s]] = b[s];
  }
  return NC_OK;
}

// Full pair list of the last built cells: one digest evaluation with the pair output enabled, then
// a host sort by (gid_i, gid_j, n1, n2, n3).
template <typename T>
nc_status pairs_t(nc_ctx* ctx, int64_t cap, int32_t* ijn, int64_t* npairs) {
  int32_t* dev = nullptr;
  unsigned long long* dn = nullptr;
  const int64_t dcap = std::max<int64_t>(cap, 1);
  CK(cudaMalloc(&dev, sizeof(int32_t) * 5 * (size_t)dcap));
  CK(cudaMalloc(&dn, sizeof(unsigned long long)));
  CK(cudaMemsetAsync(dn, 0, sizeof(unsigned long long), ctx->stream));
  ctx->po = PairOut{dev, dn, (long long)cap};
  nc_status st = digest_t<T>(ctx, nullptr, nullptr, nullptr);
  ctx->po = PairOut{nullptr, nullptr, 0};
  unsigned long long total = 0;
  std::vector<int32_t> h;
  if (st == NC_OK) {
    cudaMemcpy(&total, dn, sizeof total, cudaMemcpyDeviceToHost);
    const int64_t m = std::min<int64_t>((int64_t)total, cap);
    h.resize(5 * (size_t)m);
    if (m > 0) cudaMemcpy(h.data(), dev, sizeof(int32_t) * 5 * (size_t)m, cudaMemcpyDeviceToHost);
  }
  cudaFree(dev);
  cudaFree(dn);
  if (st) return st;
  CK(cudaGetLastError());
  *npairs = (int64_t)total;
  if ((int64_t)total > cap) return fail(ctx, NC_E_OOM, "pair list longer than cap (npairs holds the count)");
  std::vector<int64_t> order(total);
  for (int64_t k = 0; k < (int64_t)total; ++k) order[k] = k;
  std::sort(order.begin(), order.end(), [&](int64_t x, int64_t y) {
    for (int f = 0; f < 5; ++f)
      if (h[5 * x + f] != h[5 * y + f]) return h[5 * x + f] < h[5 * y + f];
    return false;
  });
  for (int64_t k = 0; k < (int64_t)total; ++k)
    for (int f = 0; f < 5; ++f) ijn[5 * k + f] = h[5 * order[k] + f];
  return NC_OK;
}

// ---------------------------------------------------------------- slab helpers
nc_status sllod_params(nc_ctx* ctx, double dt, SllodParams& sp) {
  expm3(ctx->A, -0.5 * dt, sp.Em);
  expm3(ctx->A, dt, sp.Ed);
  expm3(ctx->A, 0.5 * dt, sp.Eh);
  sp.dt = dt;
  sp.inv_m = 1.0 / ctx->cfg.mass;
  return NC_OK;
}

// deterministic class partition of n particles; returns class totals on the host
template <typename T>
nc_status partition(nc_ctx* ctx, int64_t n, const T* q, const T* p, const uint32_t* gid, T* q0, T* p0, uint32_t* g0,
                    typename V4<T>::t* r1, typename V4<T>::t* r2, int words, uint32_t tot_out[4]) {
  cudaStream_t s = ctx->stream;
  int64_t nb = (n + PART_T - 1) / PART_T;
  if (n > 0) {
    prof_begin(ctx);
    k_class_count<<<(unsigned)nb, PART_T, 0, s>>>(n, nb, ctx->cls, ctx->pbcnt);
    LAUNCHED();
    const int64_t m = 4 * nb;
    nc_status sst = launch_scan_raw(ctx, ctx->pbcnt, m, ctx->pboff);
    if (sst) return sst;
    k_class_totals<<<1, 32, 0, s>>>(ctx->pboff, nb, ctx->ptot);
    LAUNCHED();
    k_class_scatter<T><<<(unsigned)nb, PART_T, 0, s>>>(n, ctx->cls, ctx->pboff, q, p, gid, q0, p0, g0, r1, r2, words);
    LAUNCHED();
    prof_end(ctx, NC_K_OTHER);
    CK(cudaMemcpyAsync(tot_out, ctx->ptot, 16, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  } else {
    tot_out[0] = tot_out[1] = tot_out[2] = tot_out[3] = 0;
  }
  return NC_OK;
}

// Slab force evaluation in two phases so the halo exchange can overlap the interior work:
//  begin: own particles -> cells (their bucket positions after the halo particles that precede them
//         in cell order, whose COUNT is known from the count exchange), K3 on the interior own layers
//         (klo+1 .. khi-2), whose stencils touch own layers only;
//  end:   halo particles -> cells (a full rescan reproduces the own cells' starts), K3 on the two
//         boundary layers, one fixed-order reduction over all own layers, forces unsorted.
// Results are bitwise those of the one-phase evaluation (the same cells, orders and partials).
template <typename T>
nc_status slab_begin_t(nc_ctx* ctx, const T* q, const uint32_t* gid, int64_t n_own, int64_t n1, int64_t n2, int klo,
                       int khi) {
  cudaStream_t s = ctx->stream;
  const Geom& g = ctx->g;
  const int64_t n = n_own + n1 + n2;
  if (n > ctx->cap) return fail(ctx, NC_E_OOM, "own + halo particles exceed capacity");
  const int64_t C = g.ncells, per_layer = (int64_t)g.dims[0] * g.dims[1];
  const int l3 = g.dims[2];
  CK(cudaMemsetAsync(ctx->counts, 0, sizeof(uint32_t) * (C + 1), s));
  ctx->counts_clean = 0;  // this build leaves the histogram filled
  typename V4<T>::t* wq = (typename V4<T>::t*)ctx->wq;
  prof_begin(ctx);
  if (n_own > 0)
    k_wrap_key_src<T><<<nblk(n_own, 256), 256, 0, s>>>(n_own, q, 3, gid, 0, wq, ctx->gin, ctx->key, ctx->slot,
                                                      ctx->counts, g);
  LAUNCHED();
  prof_end(ctx, NC_K_WRAPKEY);
  {
    nc_status sst = launch_scan(ctx, ctx->counts, C, ctx->cs);
    if (sst) return sst;
  }
  // halo particles in cells before the own cells: the lower halo layer when it precedes klo (not
  // on the periodic seam), the upper one when it wraps to layer 0
  const int L_lo = (klo - 1 + l3) % l3, L_hi = khi % l3;
  const int64_t b_own = (L_lo < klo ? n1 : 0) + (L_hi < klo ? n2 : 0);
  if (b_own > 0) {
    const int64_t c0 = (int64_t)klo * per_layer;
    k_add_range<<<nblk(C + 1 - c0, 256), 256, 0, s>>>(ctx->cs, c0, C + 1, (uint32_t)b_own);
    LAUNCHED();
  }
  if (n_own > 0) {
    prof_begin(ctx);
    k_scatter<<<nblk(n_own, 256), 256, 0, s>>>(n_own, ctx->key, ctx->slot, ctx->cs, ctx->gin, ctx->srec);
    LAUNCHED();
    prof_end(ctx, NC_K_SCATTER);
    prof_begin(ctx);
    k_rank_gather<T><<<nblk(n_own, 256), 256, 0, s>>>(n_own, ctx->srec, ctx->cs, wq, nullptr,
                                                      (typename V4<T>::t*)ctx->sq, nullptr, ctx->sgid, ctx->u,
                                                      ctx->u32, ctx->nh, g, ctx->sidx, b_own);
    LAUNCHED();
    prof_end(ctx, NC_K_RANKGATHER);
  }
  ctx->slab_n_own = n_own;
  ctx->slab_n1 = n1;
  ctx->slab_n2 = n2;
  ctx->slab_b_own = b_own;
  ctx->slab_klo = klo;
  ctx->slab_khi = khi;
  ctx->slab_open = true;
  ctx->occ_hint = (double)n_own / ((double)per_layer * (double)(khi - klo));
  if (khi - klo > 2) {  // interior layers: their stencils see own cells only
    nc_status st = launch_pairs<T, false>(ctx, (const typename V4<T>::t*)ctx->sq, ctx->sgid,
                                          (typename V4<T>::t*)ctx->sF, klo + 1, khi - klo - 2, klo, false);
    if (st) return st;
  }
  return NC_OK;
}

template <typename T>
nc_status slab_end_t(nc_ctx* ctx, const void* h1, const void* h2, T* F, double* parts) {
  cudaStream_t s = ctx->stream;
  const Geom& g = ctx->g;
  const int64_t n_own = ctx->slab_n_own, n1 = ctx->slab_n1, n2 = ctx->slab_n2, b_own = ctx->slab_b_own;
  const int klo = ctx->slab_klo, khi = ctx->slab_khi;
  const int64_t n = n_own + n1 + n2, C = g.ncells;
  ctx->slab_open = false;
  typename V4<T>::t* wq = (typename V4<T>::t*)ctx->wq;
  prof_begin(ctx);
  if (n1 > 0)
    k_wrap_key_src<T><<<nblk(n1, 256), 256, 0, s>>>(n1, (const T*)h1, 4, nullptr, n_own, wq, ctx->gin, ctx->key,
                                                    ctx->slot, ctx->counts, g);
  if (n2 > 0)
    k_wrap_key_src<T><<<nblk(n2, 256), 256, 0, s>>>(n2, (const T*)h2, 4, nullptr, n_own + n1, wq, ctx->gin,
                                                    ctx->key, ctx->slot, ctx->counts, g);
  LAUNCHED();
  prof_end(ctx, NC_K_WRAPKEY);
  {  // all counts now: the own cells' starts come out as in begin (b_own halo particles before them)
    nc_status sst = launch_scan(ctx, ctx->counts, C, ctx->cs);
    if (sst) return sst;
  }
  if (n1 + n2 > 0) {
    prof_begin(ctx);
    k_scatter<<<nblk(n1 + n2, 256), 256, 0, s>>>(n1 + n2, ctx->key, ctx->slot, ctx->cs, ctx->gin, ctx->srec, n_own);
    LAUNCHED();
    prof_end(ctx, NC_K_SCATTER);
    // the halo buckets: [0, b_own) and [b_own + n_own, n)
    prof_begin(ctx);
    if (b_own > 0)
      k_rank_gather<T><<<nblk(b_own, 256), 256, 0, s>>>(b_own, ctx->srec, ctx->cs, wq, nullptr,
                                                        (typename V4<T>::t*)ctx->sq, nullptr, ctx->sgid, ctx->u,
                                                        ctx->u32, ctx->nh, g, ctx->sidx, 0);
    const int64_t rest = n - (b_own + n_own);
    if (rest > 0)
      k_rank_gather<T><<<nblk(rest, 256), 256, 0, s>>>(rest, ctx->srec, ctx->cs, wq, nullptr,
                                                       (typename V4<T>::t*)ctx->sq, nullptr, ctx->sgid, ctx->u,
                                                       ctx->u32, ctx->nh, g, ctx->sidx, b_own + n_own);
    LAUNCHED();
    prof_end(ctx, NC_K_RANKGATHER);
  }
  ctx->n_last = n;
  ctx->last_in_gid = ctx->gin;
  ctx->last_resident = false;
  ctx->have_cells = true;
  // boundary layers, then one reduction over all own layers
  nc_status st = launch_pairs<T, false>(ctx, (const typename V4<T>::t*)ctx->sq, ctx->sgid, (typename V4<T>::t*)ctx->sF,
                                        klo, 1, klo, khi - klo == 1);
  if (st) return st;
  if (khi - klo > 1) {
    st = launch_pairs<T, false>(ctx, (const typename V4<T>::t*)ctx->sq, ctx->sgid, (typename V4<T>::t*)ctx->sF,
                                khi - 1, 1, klo, true);
    if (st) return st;
  }
  if (n > 0 && F) {
    prof_begin(ctx);
    k_unsort_idx<T><<<nblk(n, 256), 256, 0, s>>>(n, (const typename V4<T>::t*)ctx->sF, ctx->sidx, n_own, F);
    LAUNCHED();
    prof_end(ctx, NC_K_OTHER);
  }
  if (parts) {
    CK(cudaMemcpyAsync(parts, ctx->lpart, sizeof(double) * NPART * (size_t)(khi - klo), cudaMemcpyDeviceToHost, s));
  }
  CK(cudaStreamSynchronize(s));
  return NC_OK;
}

template <typename T>
nc_status slab_forces_t(nc_ctx* ctx, const T* q, const uint32_t* gid, int64_t n_own, const void* h1, int64_t n1,
                        const void* h2, int64_t n2, int klo, int khi, T* F, double* parts) {
  nc_status st = slab_begin_t<T>(ctx, q, gid, n_own, n1, n2, klo, khi);
  if (st) return st;
  return slab_end_t<T>(ctx, h1, h2, F, parts);
}
}  // namespace

// ============================================================================ C-ABI

extern "C" {

const char* nc_version(void) { return "nemdcell 0.1 (sm_100a)"; }

const char* nc_last_error(const nc_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }

int64_t nc_launch_count(const nc_ctx* ctx) { return ctx ? ctx->launches : 0; }

nc_status nc_set_pair_kernel(nc_ctx* ctx, int which) {
  if (!ctx) return fail(ctx, NC_E_ARG, "null ctx");
  if (which != NC_PK_AUTO && which != NC_PK_CELL && which != NC_PK_SEGMENT && which != NC_PK_SPARSE &&
      which != NC_PK_ROWS)
    return fail(ctx, NC_E_ARG, "pair kernel must be NC_PK_AUTO, NC_PK_CELL, NC_PK_SEGMENT, NC_PK_SPARSE or NC_PK_ROWS");
  if ((which == NC_PK_SEGMENT || which == NC_PK_ROWS) && ctx->cfg.prec != NC_F32)
    return fail(ctx, NC_E_ARG, "the segment and row-window pair kernels are NC_F32 only");
  ctx->pair_kernel = which;
  return NC_OK;
}

int nc_pair_kernel_used(const nc_ctx* ctx) { return ctx ? ctx->pair_kernel_used : 0; }

nc_status nc_profile(nc_ctx* ctx, int enable) {
  if (!ctx) return fail(ctx, NC_E_ARG, "null ctx");
  CK(cudaStreamSynchronize(ctx->stream));  // recorded events may still be pending
  for (auto& p : ctx->prof_ev) {
    ctx->ev_pool.push_back(p.second.first);
    ctx->ev_pool.push_back(p.second.second);
  }
  ctx->prof_ev.clear();  // every event now lives in exactly one list (destroyed once)
  if (enable) {
    CK(cudaMemsetAsync(ctx->part_acc, 0, sizeof(double) * (NPART + 1), ctx->stream));
  }
  ctx->prof = enable != 0;
  ctx->count_tiers = (enable & 2) != 0;
  ctx->prof_pairs_only = (enable & 4) != 0;
  if (enable) ctx->prof_ev.reserve(4096);
  return NC_OK;
}

nc_status nc_profile_read(nc_ctx* ctx, double ms[8], int64_t counts[8]) {
  if (!ctx || !ms || !counts) return fail(ctx, NC_E_ARG, "null argument");
  CK(cudaStreamSynchronize(ctx->stream));
  for (int k = 0; k < NC_K_COUNT; ++k) { ms[k] = 0.0; counts[k] = 0; }
  for (auto& p : ctx->prof_ev) {
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, p.second.first, p.second.second));
    ms[p.first] += t;
    counts[p.first]++;
  }
  return NC_OK;
}

nc_status nc_create(const nc_config* cfg, nc_ctx** out) {
  if (!out) return fail(nullptr, NC_E_ARG, "out is NULL");
  *out = nullptr;
  if (!cfg) return fail(nullptr, NC_E_ARG, "cfg is NULL");
  if (cfg->variant != NC_DS && cfg->variant != NC_DO) return fail(nullptr, NC_E_ARG, "bad variant");
  if (cfg->prec != NC_F32 && cfg->prec != NC_F64) return fail(nullptr, NC_E_ARG, "bad precision");
  if (!(cfg->rc > 0) || !(cfg->sigma > 0) || !(cfg->mass > 0) || !std::isfinite(cfg->eps))
    return fail(nullptr, NC_E_ARG, "rc, sigma and mass must be positive");
  if (cfg->capacity < 0 || cfg->capacity > (int64_t)0xFFFFFFF0LL)
    return fail(nullptr, NC_E_ARG, "capacity out of range (< 2^32 particles)");
  nc_ctx* ctx = new nc_ctx();
  ctx->cfg = *cfg;
  ctx->stream = (cudaStream_t)cfg->stream;
  cudaError_t e = cudaSetDevice(cfg->device);
  if (e != cudaSuccess) {
    delete ctx;
    return fail(nullptr, NC_E_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  }
  int64_t N = std::max<int64_t>(cfg->capacity, 1);
  ctx->cap = N;
  ctx->max_cells = cfg->max_cells > 0 ? cfg->max_cells : 2 * N + 4096;
  ctx->max_layers = 1 << 16;
  // blocks = sum over layers of ceil(l1 l2 / cpb) <= C/cpb + layers, and cells_per_block keeps C/cpb
  // below 2 K3_MIN_BLOCKS unless cpb = K3_CELLS_MAX
  ctx->max_blocks = std::max<int64_t>(2 * K3_MIN_BLOCKS, ctx->max_cells / K3_CELLS_MAX) + ctx->max_layers + 16;
  size_t v4 = v4size(ctx), ts = tsize(ctx);
  int64_t C1 = ctx->max_cells + 1;
  const size_t N_ = (size_t)N;
  struct A { void** p; size_t bytes; } allocs[] = {
      {&ctx->st_q[0], v4 * N_}, {&ctx->st_q[1], v4 * N_}, {&ctx->st_p[0], v4 * N_}, {&ctx->st_p[1], v4 * N_},
      {(void**)&ctx->st_gid[0], 4 * N_}, {(void**)&ctx->st_gid[1], 4 * N_}, {&ctx->st_F, v4 * N_},
      {&ctx->wq, v4 * N_}, {&ctx->sq, v4 * N_}, {(void**)&ctx->sgid, 4 * N_}, {&ctx->sF, v4 * N_},
      {&ctx->io_a, 3 * ts * N_}, {&ctx->io_b, 3 * ts * N_}, {(void**)&ctx->u, sizeof(double4) * N_}, {(void**)&ctx->u32, sizeof(float4) * N_},
      {(void**)&ctx->nh, 4 * N_}, {(void**)&ctx->key, 4 * N_}, {(void**)&ctx->slot, 4 * N_},
      {(void**)&ctx->srec, sizeof(uint4) * N_},
      {(void**)&ctx->counts, 4 * (size_t)C1}, {(void**)&ctx->cs, 4 * (size_t)C1},
      {(void**)&ctx->bsum, 4 * (size_t)(C1 / SCAN_TILE + 2)}, {(void**)&ctx->tot, 16},
      {(void**)&ctx->bpart, sizeof(double) * NPART * (size_t)ctx->max_blocks},
      {(void**)&ctx->lpart, sizeof(double) * NPART * (size_t)ctx->max_layers},
      {(void**)&ctx->part_tot, sizeof(double) * NPART}, {(void**)&ctx->part_acc, sizeof(double) * (NPART + 1)},
      {(void**)&ctx->rcount, 16},
      {(void**)&ctx->dcnt, 4 * N_}, {(void**)&ctx->dhs, 8 * N_}, {(void**)&ctx->dhx, 8 * N_},
      {(void**)&ctx->hist, 8 * 64},
      {(void**)&ctx->gin, 4 * N_}, {(void**)&ctx->sidx, 4 * N_}, {(void**)&ctx->cls, N_},
      {(void**)&ctx->pbcnt, 16 * (N_ / PART_T + 2)}, {(void**)&ctx->pboff, 16 * (N_ / PART_T + 2) + 4},
      {(void**)&ctx->ptot, 16},
      {(void**)&ctx->sd, 4 * 16},
  };
  for (auto& a : allocs) {
    e = cudaMalloc(a.p, a.bytes);
    if (e != cudaSuccess) {
      std::string m = std::string("cudaMalloc: ") + cudaGetErrorString(e);
      cudaGetLastError();
      nc_destroy(ctx);
      return fail(nullptr, e == cudaErrorMemoryAllocation ? NC_E_OOM : NC_E_CUDA, m);
    }
  }
  e = cudaMemset(ctx->part_acc, 0, sizeof(double) * (NPART + 1));
  if (e == cudaSuccess) e = cudaMemset(ctx->rcount, 0, 16);
  if (e != cudaSuccess) {
    nc_destroy(ctx);
    return fail(nullptr, NC_E_CUDA, std::string("cudaMemset: ") + cudaGetErrorString(e));
  }
  ctx->pol.kind = 0;
  // kernel attributes once per context (the launch paths set nothing)
  {
    struct KA { const void* f; size_t smem; } ka[] = {
        {(const void*)k_pairs<float, false>, sizeof(K3Smem<float>)},
        {(const void*)k_pairs<float, false, true>, sizeof(K3Smem<float>)},
        {(const void*)k_pairs<float, true>, sizeof(K3Smem<float>)},
        {(const void*)k_pairs<double, false>, sizeof(K3Smem<double>)},
        {(const void*)k_pairs<double, true>, sizeof(K3Smem<double>)},
        {(const void*)k_pairs_seg<false, 2>, sizeof(SgSmem<2>)},
        {(const void*)k_pairs_seg<true, 2>, sizeof(SgSmem<2>)},
        {(const void*)k_pairs_seg<false, 4>, sizeof(SgSmem<4>)},
        {(const void*)k_pairs_seg<true, 4>, sizeof(SgSmem<4>)},
        {(const void*)k_pairs_sparse<false>, sizeof(SpSmem)},
        {(const void*)k_pairs_sparse<true>, sizeof(SpSmem)},
        {(const void*)k_pairs_sparse<false, 4>, sizeof(SpSmem)},
        {(const void*)k_pairs_sparse<true, 4>, sizeof(SpSmem)},
        {(const void*)k_pairs_sparse<false, 2>, sizeof(SpSmem)},
        {(const void*)k_pairs_sparse<true, 2>, sizeof(SpSmem)},
        {(const void*)k_pairs_sparse<false, 8>, sizeof(SpSmem)},
        {(const void*)k_pairs_sparse<true, 8>, sizeof(SpSmem)},
        {(const void*)k_pairs_sparse64<false, 1>, sizeof(Sp64Smem)},
        {(const void*)k_pairs_sparse64<true, 1>, sizeof(Sp64Smem)},
        {(const void*)k_pairs_sparse64<false, 2>, sizeof(Sp64Smem)},
        {(const void*)k_pairs_sparse64<true, 2>, sizeof(Sp64Smem)},
        {(const void*)k_pairs_rows<false>, sizeof(RwSmem)},
        {(const void*)k_pairs_rows<true>, sizeof(RwSmem)}};
    for (const KA& a : ka) {
      cudaError_t e = cudaFuncSetAttribute(a.f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)a.smem);
      if (e != cudaSuccess) {
        nc_destroy(ctx);
        return fail(nullptr, NC_E_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
      }
    }
  }
  *out = ctx;
  return NC_OK;
}

void nc_comm_release(nc_ctx* ctx);  // nccl_slab.cuh

void nc_destroy(nc_ctx* ctx) {
  if (!ctx) return;
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  void* ps[] = {ctx->st_q[0], ctx->st_q[1], ctx->st_p[0], ctx->st_p[1], ctx->st_gid[0], ctx->st_gid[1], ctx->st_F,
                ctx->wq, ctx->sq, ctx->sgid, ctx->sF, ctx->io_a, ctx->io_b, ctx->u, ctx->u32, ctx->nh, ctx->key, ctx->slot,
                ctx->srec, ctx->counts, ctx->cs, ctx->bsum, ctx->tot, ctx->bpart, ctx->lpart,
                ctx->part_tot, ctx->part_acc, ctx->rcount, ctx->dcnt, ctx->dhs, ctx->dhx, ctx->hist,
                ctx->gin, ctx->sidx, ctx->cls, ctx->pbcnt, ctx->pboff, ctx->ptot, ctx->sd,
                ctx->perm, ctx->pgid, ctx->pq};
  for (void* p : ps)
    if (p) cudaFree(p);
  if (ctx->s_h2d) {
    cudaStreamSynchronize(ctx->s_h2d);
    cudaStreamSynchronize(ctx->s_d2h);
    for (int b = 0; b < 2; ++b) {
      cudaFree(ctx->ain[b]);
      cudaFree(ctx->aout[b]);
      cudaEventDestroy(ctx->ev_in_ready[b]);
      cudaEventDestroy(ctx->ev_in_free[b]);
      cudaEventDestroy(ctx->ev_out_ready[b]);
      cudaEventDestroy(ctx->ev_out_free[b]);
    }
    cudaStreamDestroy(ctx->s_h2d);
    cudaStreamDestroy(ctx->s_d2h);
  }
  for (auto& p : ctx->prof_ev) {
    cudaEventDestroy(p.second.first);
    cudaEventDestroy(p.second.second);
  }
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  for (void* p : ctx->ipc_open) cudaIpcCloseMemHandle(p);
  for (void* p : ctx->ipc_own) cudaFree(p);
  for (auto e : ctx->ipc_ev) cudaEventDestroy(e);
  nc_comm_release(ctx);
  delete ctx;
}

nc_status nc_set_box(nc_ctx* ctx, const double L[9]) {
  if (!ctx || !L) return fail(ctx, NC_E_ARG, "null argument");
  nc_status st = apply_box(ctx, L);
  if (st) return st;
  if (!ctx->have_flow) {
    ctx->pol.kind = 0;
    std::memcpy(ctx->pol.L0, L, sizeof(double) * 9);
    std::memset(ctx->A, 0, sizeof ctx->A);
    ctx->t = 0.0;
  }
  return NC_OK;
}

nc_status nc_set_flow(nc_ctx* ctx, const double A[9], const nc_remap* pol, double t) {
  if (!ctx || !A) return fail(ctx, NC_E_ARG, "null argument");
  double amax = 1.0, tr = A[0] + A[4] + A[8];
  for (int k = 0; k < 9; ++k) {
    if (!std::isfinite(A[k])) return fail(ctx, NC_E_FLOW, "non-finite flow matrix");
    amax = std::max(amax, std::fabs(A[k]));
  }
  if (std::fabs(tr) > 1e-12 * amax) return fail(ctx, NC_E_FLOW, "flow matrix A must be traceless (incompressible)");
  Policy p;
  std::memset(&p, 0, sizeof p);
  if (pol) {
    p.kind = (int)pol->kind;
    std::memcpy(p.L0, pol->L0, sizeof(double) * 9);
    p.tstar = pol->tstar;
    for (int k = 0; k < 3; ++k) { p.om1[k] = pol->omega1[k]; p.om2[k] = pol->omega2[k]; }
    p.beta[0] = pol->beta[0];
    p.beta[1] = pol->beta[1];
    p.eps = pol->eps;
    if (p.kind < 0 || p.kind > 4) return fail(ctx, NC_E_ARG, "bad remap kind");
    if (p.kind == 4) {  // R30: reduce e^{At} L0 once, then carry (Lr, tr)
      double E[9];
      expm3(A, t, E);
      matmul3(E, p.L0, p.Lr);
      lattice_reduce(p.Lr);
      p.tr = t;
    }
    if (p.kind == 2 && !(p.tstar > 0)) return fail(ctx, NC_E_ARG, "KR needs tstar > 0");
    if (p.kind == 1 && !(A[1] != 0.0)) return fail(ctx, NC_E_ARG, "LE needs a shear flow A[0][1] != 0");
  } else {
    if (!ctx->have_box) return fail(ctx, NC_E_STATE, "nc_set_flow without a policy needs nc_set_box first");
    p.kind = 0;
    std::memcpy(p.L0, ctx->g.L, sizeof(double) * 9);
  }
  double L[9];
  std::memcpy(ctx->A, A, sizeof(double) * 9);
  box_at(p, A, t, L);
  nc_status st = apply_box(ctx, L);
  if (st) return st;
  ctx->pol = p;
  ctx->t = t;
  ctx->have_flow = true;
  return NC_OK;
}

nc_status nc_build_cells(nc_ctx* ctx, const void* q, int64_t n) {
  if (!ctx || (!q && n > 0)) return fail(ctx, NC_E_ARG, "null argument");
  if (!ctx->have_box) return fail(ctx, NC_E_STATE, "nc_set_box first");
  if (n < 0 || n > ctx->cap) return fail(ctx, NC_E_OOM, "n exceeds capacity");
  nc_status st = ctx->cfg.prec == NC_F32 ? build_user<float>(ctx, q, n) : build_user<double>(ctx, q, n);
  if (st) return st;
  return cuda_check(ctx, cudaStreamSynchronize(ctx->stream), "build_cells");
}

nc_status nc_compute_forces(nc_ctx* ctx, const void* q, int64_t n, void* F, double* U, double W[6]) {
  if (!ctx || (!q && n > 0)) return fail(ctx, NC_E_ARG, "null argument");
  if (!ctx->have_box) return fail(ctx, NC_E_STATE, "nc_set_box first");
  if (n < 0 || n > ctx->cap) return fail(ctx, NC_E_OOM, "n exceeds capacity");
  return ctx->cfg.prec == NC_F32 ? compute_user<float>(ctx, q, n, F, U, W) : compute_user<double>(ctx, q, n, F, U, W);
}

nc_status nc_compute_forces_async(nc_ctx* ctx, const void* q, int64_t n, void* F) {
  if (!ctx || (!q && n > 0)) return fail(ctx, NC_E_ARG, "null argument");
  if (!ctx->have_box) return fail(ctx, NC_E_STATE, "nc_set_box first");
  if (n < 0 || n > ctx->cap) return fail(ctx, NC_E_OOM, "n exceeds capacity");
  if ((q && is_device_ptr(q)) || (F && is_device_ptr(F)))
    return fail(ctx, NC_E_ARG, "nc_compute_forces_async takes host buffers (device ones: nc_compute_forces)");
  return ctx->cfg.prec == NC_F32 ? compute_async_t<float>(ctx, q, n, F) : compute_async_t<double>(ctx, q, n, F);
}

nc_status nc_compute_sync(nc_ctx* ctx, double* U, double W[6]) {
  if (!ctx) return fail(ctx, NC_E_ARG, "null ctx");
  if (ctx->s_d2h) CK(cudaStreamSynchronize(ctx->s_d2h));
  if (!ctx->async_eval) return fail(ctx, NC_E_STATE, "no pending nc_compute_forces_async");
  ctx->async_eval = false;
  nc_status st = check_finite(ctx);  // synchronizes the context stream
  if (st) return st;
  totals_to_UW(ctx, U, W);
  return NC_OK;
}

nc_status nc_set_state(nc_ctx* ctx, const void* q, const void* p, const int64_t* gid, int64_t n) {
  if (!ctx || (!q && n > 0)) return fail(ctx, NC_E_ARG, "null argument");
  if (!ctx->have_box) return fail(ctx, NC_E_STATE, "nc_set_box or nc_set_flow first");
  if (n < 0 || n > ctx->cap) return fail(ctx, NC_E_OOM, "n exceeds capacity");
  if (gid) {  // must be a permutation of 0..n-1: outputs are indexed by gid (nc_get_state, digests)
    std::vector<uint8_t> seen((size_t)n, 0);
    for (int64_t i = 0; i < n; ++i) {
      if (gid[i] < 0 || gid[i] >= n) return fail(ctx, NC_E_ARG, "gid must be a permutation of 0..n-1 (out of range)");
      if (seen[(size_t)gid[i]]++) return fail(ctx, NC_E_ARG, "gid must be a permutation of 0..n-1 (duplicate)");
    }
  }
  ctx->kick_pending = false;  // the new state replaces the momenta the deferred kick belonged to
  return ctx->cfg.prec == NC_F32 ? set_state_t<float>(ctx, q, p, gid, n) : set_state_t<double>(ctx, q, p, gid, n);
}

nc_status nc_step_sllod(nc_ctx* ctx, double dt, int nsteps, double* U, double W[6]) {
  if (!ctx) return fail(ctx, NC_E_ARG, "null ctx");
  if (!ctx->have_state) return fail(ctx, NC_E_STATE, "nc_set_state first");
  if (!(dt > 0) || nsteps < 0) return fail(ctx, NC_E_ARG, "dt must be > 0 and nsteps >= 0");
  return ctx->cfg.prec == NC_F32 ? step_t<float>(ctx, dt, nsteps, U, W) : step_t<double>(ctx, dt, nsteps, U, W);
}

nc_status nc_get_state(nc_ctx* ctx, void* q, void* p, int64_t* gid, int64_t* n, double L[9], double* t) {
  if (!ctx) return fail(ctx, NC_E_ARG, "null ctx");
  if (!ctx->have_state) return fail(ctx, NC_E_STATE, "no resident state");
  {
    nc_status mst = materialize_kick(ctx);
    if (mst) return mst;
  }
  int64_t m = ctx->n_state;
  int c = ctx->cur;
  nc_status st;
  if (q) {
    st = ctx->cfg.prec == NC_F32 ? unsort_out<float>(ctx, ctx->st_q[c], ctx->st_gid[c], m, q)
                                 : unsort_out<double>(ctx, ctx->st_q[c], ctx->st_gid[c], m, q);
    if (st) return st;
    CK(cudaStreamSynchronize(ctx->stream));
  }
  if (p) {
    st = ctx->cfg.prec == NC_F32 ? unsort_out<float>(ctx, ctx->st_p[c], ctx->st_gid[c], m, p)
                                 : unsort_out<double>(ctx, ctx->st_p[c], ctx->st_gid[c], m, p);
    if (st) return st;
    CK(cudaStreamSynchronize(ctx->stream));
  }
  if (gid) {
    std::vector<uint32_t> g(m);
    CK(cudaMemcpyAsync(g.data(), ctx->st_gid[c], 4 * m, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    std::vector<uint32_t> s(g);
    std::sort(s.begin(), s.end());
    for (int64_t i = 0; i < m; ++i) gid[i] = s[i];
  }
  if (n) *n = m;
  if (L) std::memcpy(L, ctx->g.L, sizeof(double) * 9);
  if (t) *t = ctx->t;
  return NC_OK;
}

nc_status nc_get_cells(nc_ctx* ctx, int64_t* cell_of, int64_t* cell_start, int32_t dims[3], void* wrapped_q) {
  if (!ctx) return fail(ctx, NC_E_ARG, "null ctx");
  if (!ctx->have_cells) return fail(ctx, NC_E_STATE, "no cells built");
  int64_t n = ctx->n_last, C = ctx->g.ncells;
  cudaStream_t s = ctx->stream;
  std::vector<uint32_t> key(n), ig(n), cs(C + 1);
  CK(cudaMemcpyAsync(key.data(), ctx->key, 4 * n, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(cs.data(), ctx->cs, 4 * (C + 1), cudaMemcpyDeviceToHost, s));
  if (ctx->last_in_gid) CK(cudaMemcpyAsync(ig.data(), ctx->last_in_gid, 4 * n, cudaMemcpyDeviceToHost, s));
  std::vector<unsigned char> wq;
  size_t ts = tsize(ctx);
  const void* wsrc = ctx->last_resident ? ctx->st_q[1 - ctx->cur] : ctx->wq;
  if (wrapped_q) {
    wq.resize(4 * ts * n);
    CK(cudaMemcpyAsync(wq.data(), wsrc, 4 * ts * n, cudaMemcpyDeviceToHost, s));
  }
  CK(cudaStreamSynchronize(s));
  for (int64_t i = 0; i < n; ++i) {
    int64_t gi = ctx->last_in_gid ? (int64_t)ig[i] : i;
    if (cell_of) cell_of[gi] = key[i];
    if (wrapped_q)
      for (int k = 0; k < 3; ++k)
        std::memcpy((unsigned char*)wrapped_q + (3 * gi + k) * ts, wq.data() + (4 * i + k) * ts, ts);
  }
  if (cell_start)
    for (int64_t c = 0; c <= C; ++c) cell_start[c] = cs[c];
  if (dims)
    for (int k = 0; k < 3; ++k) dims[k] = ctx->g.dims[k];
  return NC_OK;
}

nc_status nc_get_pair_digest(nc_ctx* ctx, uint32_t* cnt, uint64_t* hsum, uint64_t* hxor) {
  if (!ctx) return fail(ctx, NC_E_ARG, "null ctx");
  if (!ctx->have_cells) return fail(ctx, NC_E_STATE, "no cells built");
  nc_status st = ctx->cfg.prec == NC_F32 ? digest_t<float>(ctx, cnt, hsum, hxor) : digest_t<double>(ctx, cnt, hsum, hxor);
  return st;
}

nc_status nc_get_pairs(nc_ctx* ctx, int64_t cap, int32_t* i_j_n, int64_t* npairs) {
  if (!ctx || !npairs || (cap > 0 && !i_j_n) || cap < 0) return fail(ctx, NC_E_ARG, "null argument or cap < 0");
  if (!ctx->have_cells) return fail(ctx, NC_E_STATE, "no cells built");
  return ctx->cfg.prec == NC_F32 ? pairs_t<float>(ctx, cap, i_j_n, npairs) : pairs_t<double>(ctx, cap, i_j_n, npairs);
}

nc_status nc_get_cell_gids(nc_ctx* ctx, int64_t* gid_sorted) {
  if (!ctx || !gid_sorted) return fail(ctx, NC_E_ARG, "null argument");
  if (!ctx->have_cells) return fail(ctx, NC_E_STATE, "no cells built");
  const int64_t n = ctx->n_last;
  const uint32_t* gid = ctx->last_resident ? ctx->st_gid[ctx->cur] : ctx->sgid;
  std::vector<uint32_t> g(n);
  CK(cudaMemcpyAsync(g.data(), gid, 4 * n, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  for (int64_t k = 0; k < n; ++k) gid_sorted[k] = g[k];
  return NC_OK;
}

nc_status nc_get_pair_counts(nc_ctx* ctx, uint32_t* cnt) {
  if (!ctx || !cnt) return fail(ctx, NC_E_ARG, "null argument");
  if (!ctx->have_eval) return fail(ctx, NC_E_STATE, "no evaluation yet");
  const int64_t n = ctx->n_last;
  const bool f32 = ctx->cfg.prec == NC_F32;
  const void* F = ctx->last_resident ? ctx->st_F : ctx->sF;
  const uint32_t* gid = ctx->last_resident ? ctx->st_gid[ctx->cur] : ctx->sgid;
  std::vector<unsigned char> f(v4size(ctx) * n);
  std::vector<uint32_t> g(n);
  CK(cudaMemcpyAsync(f.data(), F, f.size(), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(g.data(), gid, 4 * n, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  for (int64_t k = 0; k < n; ++k) {
    uint32_t c;
    if (f32) std::memcpy(&c, f.data() + 16 * k + 12, 4);
    else { double w; std::memcpy(&w, f.data() + 32 * k + 24, 8); c = (uint32_t)w; }
    cnt[g[k]] = c;
  }
  return NC_OK;
}

nc_status nc_debug(nc_ctx* ctx, int what, int value) {
  if (!ctx) return fail(ctx, NC_E_ARG, "null ctx");
  if (what != NC_DBG_DROP_ENTRIES || value < 0 || value > 1) return fail(ctx, NC_E_ARG, "bad debug option");
  ctx->dbg_drop = value;
  ctx->g.dbg_drop = value;
  return NC_OK;
}

nc_status nc_get_stats(nc_ctx* ctx, nc_stats* out) {
  if (!ctx || !out) return fail(ctx, NC_E_ARG, "null argument");
  if (!ctx->have_eval) return fail(ctx, NC_E_STATE, "no evaluation yet");
  nc_status st = fetch_totals(ctx);
  if (st) return st;
  std::memset(out, 0, sizeof *out);
  out->n = ctx->n_last;
  for (int k = 0; k < 3; ++k) out->dims[k] = ctx->g.dims[k];
  out->ncells = ctx->g.ncells;
  out->interactions = ctx->host_tot[7];
  out->candidates = ctx->host_tot[8];
  out->stencil_cells = ctx->host_tot[9];
  out->rechecks = ctx->host_tot[10];
  totals_to_UW(ctx, &out->U, out->W);
  double acc[NPART + 1];
  CK(cudaMemcpyAsync(acc, ctx->part_acc, sizeof acc, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  out->acc_evals = acc[NPART];
  out->acc_interactions = acc[7];
  out->acc_candidates = acc[8];
  out->interactions_fp32 = ctx->host_tot[11];
  out->acc_interactions_fp32 = acc[11];
  return NC_OK;
}

nc_status nc_get_stencil_histogram(nc_ctx* ctx, int64_t hist[64]) {
  if (!ctx || !hist) return fail(ctx, NC_E_ARG, "null argument");
  if (!ctx->have_box) return fail(ctx, NC_E_STATE, "nc_set_box first");
  CK(cudaMemsetAsync(ctx->hist, 0, 8 * 64, ctx->stream));
  prof_begin(ctx);
  k_stencil_hist<<<1184, 32, 0, ctx->stream>>>(ctx->g, ctx->hist);
  LAUNCHED();
  prof_end(ctx, NC_K_OTHER);
  unsigned long long h[64];
  CK(cudaMemcpyAsync(h, ctx->hist, 8 * 64, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  for (int k = 0; k < 64; ++k) hist[k] = (int64_t)h[k];
  return NC_OK;
}


// ============================================================================ slab (multi-GPU) C-ABI

nc_status nc_slab_layers(nc_ctx* ctx, int rank, int nranks, int32_t* klo, int32_t* khi, int32_t* l3) {
  if (!ctx || nranks < 1 || rank < 0 || rank >= nranks) return fail(ctx, NC_E_ARG, "bad rank / nranks");
  if (!ctx->have_box) return fail(ctx, NC_E_STATE, "nc_set_box or nc_set_flow first");
  const int L3 = ctx->g.dims[2];
  if (L3 < 2 * nranks) return fail(ctx, NC_E_DEGENERATE, "slab decomposition needs >= 2 cell layers per rank");
  if (klo) *klo = (int32_t)((int64_t)rank * L3 / nranks);
  if (khi) *khi = (int32_t)((int64_t)(rank + 1) * L3 / nranks);
  if (l3) *l3 = L3;
  return NC_OK;
}

nc_status nc_slab_kick_drift(nc_ctx* ctx, void* q, void* p, const void* F, int64_t n, double dt) {
  return nc_slab_kick_kick_drift(ctx, q, p, F, n, 0.0, dt);
}

nc_status nc_slab_kick_kick_drift(nc_ctx* ctx, void* q, void* p, const void* F, int64_t n, double dt_prev,
                                  double dt) {
  if (!ctx || (n > 0 && (!q || !p || !F))) return fail(ctx, NC_E_ARG, "null argument");
  if (!ctx->have_flow && !ctx->have_box) return fail(ctx, NC_E_STATE, "nc_set_flow first");
  if (!(dt > 0) || dt_prev < 0) return fail(ctx, NC_E_ARG, "dt must be > 0 and dt_prev >= 0");
  K3Kick pk{};
  if (dt_prev > 0) {
    SllodParams pp;
    sllod_params(ctx, dt_prev, pp);
    for (int e = 0; e < 9; ++e) pk.Em[e] = pp.Em[e];
    pk.hd = 0.5 * dt_prev;
  }
  const int pending = dt_prev > 0 ? 1 : 0;
  SllodParams sp;
  sllod_params(ctx, dt, sp);
  double Lnew[9];
  box_advance(ctx->pol, ctx->A, ctx->t + dt, Lnew);
  nc_status st = apply_box(ctx, Lnew);
  if (st) return st;
  ctx->t += dt;
  if (n > 0) {
    prof_begin(ctx);
    if (ctx->cfg.prec == NC_F32)
      k_kick_drift3<float><<<nblk(n, 256), 256, 0, ctx->stream>>>(n, (float*)q, (float*)p, (const float*)F, sp,
                                                                    pending, pk);
    else
      k_kick_drift3<double><<<nblk(n, 256), 256, 0, ctx->stream>>>(n, (double*)q, (double*)p, (const double*)F, sp,
                                                                     pending, pk);
    LAUNCHED();
    prof_end(ctx, NC_K_KICK);
  }
  return NC_OK;
}

nc_status nc_slab_migrate(nc_ctx* ctx, void* q, const void* p, const uint32_t* gid, int64_t n, int klo, int khi,
                          void* q_out, void* p_out, uint32_t* gid_out, void* send_lo, void* send_hi, int64_t cap,
                          int64_t counts[3]) {
  if (!ctx || !counts || (n > 0 && (!q || !p || !gid || !q_out || !p_out || !gid_out || !send_lo || !send_hi)))
    return fail(ctx, NC_E_ARG, "null argument");
  if (n > ctx->cap) return fail(ctx, NC_E_OOM, "n exceeds capacity");
  uint32_t tot[4] = {0, 0, 0, 0};
  nc_status st;
  if (n > 0) {
    prof_begin(ctx);
    if (ctx->cfg.prec == NC_F32)
      k_slab_classify<float><<<nblk(n, 256), 256, 0, ctx->stream>>>(n, (float*)q, ctx->g, klo, khi, 0, ctx->cls);
    else
      k_slab_classify<double><<<nblk(n, 256), 256, 0, ctx->stream>>>(n, (double*)q, ctx->g, klo, khi, 0, ctx->cls);
    LAUNCHED();
    prof_end(ctx, NC_K_WRAPKEY);
  }
  if (ctx->cfg.prec == NC_F32)
    st = partition<float>(ctx, n, (const float*)q, (const float*)p, gid, (float*)q_out, (float*)p_out, gid_out,
                          (float4*)send_lo, (float4*)send_hi, 2, tot);
  else
    st = partition<double>(ctx, n, (const double*)q, (const double*)p, gid, (double*)q_out, (double*)p_out, gid_out,
                           (double4*)send_lo, (double4*)send_hi, 2, tot);
  if (st) return st;
  if (tot[3]) return fail(ctx, NC_E_STATE, "a particle moved more than one cell layer past its slab in one step");
  if ((int64_t)tot[1] > cap || (int64_t)tot[2] > cap) return fail(ctx, NC_E_OOM, "migration buffer too small");
  counts[0] = tot[0]; counts[1] = tot[1]; counts[2] = tot[2];
  return NC_OK;
}

nc_status nc_slab_layer_of(nc_ctx* ctx, void* q, int64_t n, int32_t* layer) {
  if (!ctx || (n > 0 && (!q || !layer)) || n < 0) return fail(ctx, NC_E_ARG, "null argument");
  if (!ctx->have_box) return fail(ctx, NC_E_STATE, "nc_set_box or nc_set_flow first");
  if (n > 0) {
    prof_begin(ctx);
    if (ctx->cfg.prec == NC_F32)
      k_slab_classify<float><<<nblk(n, 256), 256, 0, ctx->stream>>>(n, (float*)q, ctx->g, 0, 0, 2, nullptr, layer);
    else
      k_slab_classify<double><<<nblk(n, 256), 256, 0, ctx->stream>>>(n, (double*)q, ctx->g, 0, 0, 2, nullptr, layer);
    LAUNCHED();
    prof_end(ctx, NC_K_WRAPKEY);
  }
  return NC_OK;
}

nc_status nc_slab_unpack(nc_ctx* ctx, const void* rec, int64_t n, void* q, void* p, uint32_t* gid) {
  if (!ctx || (n > 0 && (!rec || !q || !p || !gid))) return fail(ctx, NC_E_ARG, "null argument");
  if (n <= 0) return NC_OK;
  prof_begin(ctx);
  if (ctx->cfg.prec == NC_F32)
    k_records_unpack<float><<<nblk(n, 256), 256, 0, ctx->stream>>>(n, (const float4*)rec, (float*)q, (float*)p, gid);
  else
    k_records_unpack<double><<<nblk(n, 256), 256, 0, ctx->stream>>>(n, (const double4*)rec, (double*)q, (double*)p,
                                                                     gid);
  LAUNCHED();
  prof_end(ctx, NC_K_OTHER);
  return NC_OK;
}

nc_status nc_slab_halo(nc_ctx* ctx, void* q, const uint32_t* gid, int64_t n, int klo, int khi, void* halo_lo,
                       void* halo_hi, int64_t cap, int64_t counts[2]) {
  if (!ctx || !counts || (n > 0 && (!q || !gid || !halo_lo || !halo_hi))) return fail(ctx, NC_E_ARG, "null argument");
  if (khi - klo < 2) return fail(ctx, NC_E_DEGENERATE, "slab decomposition needs >= 2 cell layers per rank");
  uint32_t tot[4] = {0, 0, 0, 0};
  nc_status st;
  if (n > 0) {
    prof_begin(ctx);
    if (ctx->cfg.prec == NC_F32)
      k_slab_classify<float><<<nblk(n, 256), 256, 0, ctx->stream>>>(n, (float*)q, ctx->g, klo, khi, 1, ctx->cls);
    else
      k_slab_classify<double><<<nblk(n, 256), 256, 0, ctx->stream>>>(n, (double*)q, ctx->g, klo, khi, 1, ctx->cls);
    LAUNCHED();
    prof_end(ctx, NC_K_WRAPKEY);
  }
  if (ctx->cfg.prec == NC_F32)
    st = partition<float>(ctx, n, (const float*)q, nullptr, gid, nullptr, nullptr, nullptr, (float4*)halo_lo,
                          (float4*)halo_hi, 1, tot);
  else
    st = partition<double>(ctx, n, (const double*)q, nullptr, gid, nullptr, nullptr, nullptr, (double4*)halo_lo,
                           (double4*)halo_hi, 1, tot);
  if (st) return st;
  if ((int64_t)tot[1] > cap || (int64_t)tot[2] > cap) return fail(ctx, NC_E_OOM, "halo buffer too small");
  counts[0] = tot[1];
  counts[1] = tot[2];
  return NC_OK;
}

nc_status nc_slab_forces(nc_ctx* ctx, const void* q, const uint32_t* gid, int64_t n_own, const void* halo_from_lo,
                         int64_t n_lo, const void* halo_from_hi, int64_t n_hi, int klo, int khi, void* F,
                         double* layer_parts) {
  if (!ctx || (n_own > 0 && (!q || !gid))) return fail(ctx, NC_E_ARG, "null argument");
  if (!ctx->have_box) return fail(ctx, NC_E_STATE, "nc_set_box or nc_set_flow first");
  if (klo < 0 || khi > ctx->g.dims[2] || khi - klo < 1) return fail(ctx, NC_E_ARG, "bad layer range");
  ctx->occ_hint = (double)n_own / ((double)ctx->g.dims[0] * ctx->g.dims[1] * (double)(khi - klo));
  return ctx->cfg.prec == NC_F32
             ? slab_forces_t<float>(ctx, (const float*)q, gid, n_own, halo_from_lo, n_lo, halo_from_hi, n_hi, klo, khi,
                                    (float*)F, layer_parts)
             : slab_forces_t<double>(ctx, (const double*)q, gid, n_own, halo_from_lo, n_lo, halo_from_hi, n_hi, klo,
                                     khi, (double*)F, layer_parts);
}

nc_status nc_slab_forces_begin(nc_ctx* ctx, const void* q, const uint32_t* gid, int64_t n_own, int64_t n_lo,
                               int64_t n_hi, int klo, int khi) {
  if (!ctx || (n_own > 0 && (!q || !gid)) || n_lo < 0 || n_hi < 0) return fail(ctx, NC_E_ARG, "null argument");
  if (!ctx->have_box) return fail(ctx, NC_E_STATE, "nc_set_box or nc_set_flow first");
  if (klo < 0 || khi > ctx->g.dims[2] || khi - klo < 1) return fail(ctx, NC_E_ARG, "bad layer range");
  return ctx->cfg.prec == NC_F32 ? slab_begin_t<float>(ctx, (const float*)q, gid, n_own, n_lo, n_hi, klo, khi)
                                 : slab_begin_t<double>(ctx, (const double*)q, gid, n_own, n_lo, n_hi, klo, khi);
}

nc_status nc_slab_forces_end(nc_ctx* ctx, const void* halo_from_lo, const void* halo_from_hi, void* F,
                             double* layer_parts) {
  if (!ctx) return fail(ctx, NC_E_ARG, "null ctx");
  if (!ctx->slab_open) return fail(ctx, NC_E_STATE, "nc_slab_forces_begin first");
  if ((ctx->slab_n1 > 0 && !halo_from_lo) || (ctx->slab_n2 > 0 && !halo_from_hi))
    return fail(ctx, NC_E_ARG, "null argument");
  return ctx->cfg.prec == NC_F32 ? slab_end_t<float>(ctx, halo_from_lo, halo_from_hi, (float*)F, layer_parts)
                                 : slab_end_t<double>(ctx, halo_from_lo, halo_from_hi, (double*)F, layer_parts);
}

nc_status nc_slab_kick(nc_ctx* ctx, void* p, const void* F, int64_t n, double dt) {
  if (!ctx || (n > 0 && (!p || !F))) return fail(ctx, NC_E_ARG, "null argument");
  if (n <= 0) return NC_OK;
  SllodParams sp;
  sllod_params(ctx, dt, sp);
  prof_begin(ctx);
  if (ctx->cfg.prec == NC_F32)
    k_kick3<float><<<nblk(n, 256), 256, 0, ctx->stream>>>(n, (float*)p, (const float*)F, sp);
  else
    k_kick3<double><<<nblk(n, 256), 256, 0, ctx->stream>>>(n, (double*)p, (const double*)F, sp);
  LAUNCHED();
  prof_end(ctx, NC_K_KICK);
  return NC_OK;
}

nc_status nc_slab_reduce(nc_ctx* ctx, const double* parts, int nlayers, double* U, double W[6], double stats[4]) {
  if (!ctx || !parts || nlayers < 1) return fail(ctx, NC_E_ARG, "null argument");
  // the same fixed-order layer sum as k_reduce, then the same frame rotation as a single-device evaluation
  for (int c = 0; c < NPART; ++c) {
    double v = 0;
    for (int l = 0; l < nlayers; ++l) v += parts[(int64_t)l * NPART + c];
    ctx->host_tot[c] = v;
  }
  ctx->tot_valid = true;
  ctx->have_eval = true;
  if (ctx->host_tot[NPART - 1] >= K3_OVERFLOW)
    return fail(ctx, NC_E_OOM, "a neighborhood holds more particles than the pair kernel can stage (cell kernel: " +
                                   std::to_string(K3_CAP) + " per cell; sparse-cell kernel: one neighborhood per "
                                   "segment union): too dense for this cutoff / kernel");
  bool ok = ctx->host_tot[NPART - 1] == 0.0;
  for (int k = 0; k < 7; ++k) ok = ok && std::isfinite(ctx->host_tot[k]);
  totals_to_UW(ctx, U, W);
  if (stats) { stats[0] = ctx->host_tot[7]; stats[1] = ctx->host_tot[8]; stats[2] = ctx->host_tot[9]; stats[3] = ctx->host_tot[10]; }
  if (!ok) return fail(ctx, NC_E_NONFINITE, "non-finite force, energy or virial");
  return NC_OK;
}

}  // extern "C"

#include "nccl_slab.cuh"
#include "slab_dc.cuh"
#include "ipc_slab.cuh"

void nc_comm_release(nc_ctx* ctx) {
  if (!ctx->comm) return;
  if (ctx->s_comm) cudaStreamSynchronize(ctx->s_comm);
  nccl().CommDestroy((ncclComm_t)ctx->comm);
  ctx->comm = nullptr;
  if (ctx->s_comm) cudaStreamDestroy(ctx->s_comm);
  if (ctx->ev_comm_in) cudaEventDestroy(ctx->ev_comm_in);
  if (ctx->ev_comm_out) cudaEventDestroy(ctx->ev_comm_out);
  if (ctx->comm_cnt) cudaFree(ctx->comm_cnt);
  if (ctx->comm_gather) cudaFree(ctx->comm_gather);
}
