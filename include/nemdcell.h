/*
 * nemdcell.h -- C-ABI of the B200 (sm_100a) cell-list force path for
 * nonequilibrium MD in a periodic box that deforms with a homogeneous
 * linear flow, after arXiv 1412.3784 (Dobson, Fox, Saracino: "Cell list
 * algorithms for nonequilibrium molecular dynamics").
 *
 * Library: paper_1412_3784_b200/libnemdcell.so.  Every entry point is
 * extern "C", takes plain pointers and sizes, and returns an nc_status; no
 * call throws or aborts across the ABI.  nc_last_error() gives the text of
 * the last failure on a context.
 *
 * Citations: P:n = line n of the paper text; Eq. (k) numbered as
 * in DESIGN.md section 1; Rn = reading n in DESIGN.md section 3 (where the
 * paper is silent or ambiguous).
 *
 * Conventions shared by all calls
 *  - Box matrix L: double[9], ROW-major, whose COLUMNS are the box vectors
 *    v1, v2, v3 (Eq. 1).  det L > 0 is required.
 *  - Positions q, momenta p, forces F: n x 3 contiguous, row-major, element
 *    type float (NC_F32) or double (NC_F64) as chosen in nc_config.prec.
 *    Pointers may be DEVICE memory (e.g. torch CUDA tensors; used in place)
 *    or HOST memory (pageable or pinned; the library copies through its own
 *    device buffers on cfg.stream).  The kind is detected per pointer.
 *  - Arrays are in particle-id (gid) order at the ABI; internally the
 *    library keeps particles sorted by (cell, gid) (R27).
 *  - All GPU work is enqueued on cfg.stream (a cudaStream_t; NULL = the
 *    legacy default stream).  Calls that return host values synchronize that
 *    stream only.  One context per host thread; calls are not re-entrant.
 *  - Ownership: the caller owns every pointer it passes; the library owns
 *    all scratch and the resident particle state for the context lifetime.
 *  - Units: epsilon = sigma = m = 1 are the usual choice; any positive
 *    values are accepted.
 */
#ifndef NEMDCELL_H
#define NEMDCELL_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct nc_ctx nc_ctx;

/* The paper's two cell-list variants. */
typedef enum {
    NC_DS = 0, /* dynamic size: cells congruent to the box, c_k = floor(h_k/d_cut), 27 cells */
    NC_DO = 1  /* dynamic offset: QR-rotated rectangular cells, l_k = floor(r_kk/d_cut), 27/30/34/36 */
} nc_variant;

/* Storage and pair-arithmetic precision.  NC_F32 keeps fp32 positions,
 * filters candidates in fp32 (superset bound r^2 < r_c^2 (1 + 1e-4)),
 * evaluates pairs with r >= 1.2 sigma below the band in fp32 and closer
 * pairs and every candidate whose r^2 lies in the band around r_c^2 in fp64
 * from fp64 cell-local coordinates, the band ones by the canonical test, so
 * the pair SET is the canonical fp64 one (R16).
 * Forces, U and W are accumulated in fp64.  NC_F64 does everything in fp64. */
typedef enum { NC_F32 = 0, NC_F64 = 1 } nc_prec;

typedef enum {
    NC_OK = 0,
    NC_E_ARG = 1,        /* null pointer, n out of range, bad enum, unsupported pointer */
    NC_E_BOX = 2,        /* det L <= 0 or a non-finite entry */
    NC_E_DEGENERATE = 3, /* DS: some c_k < 3; DO: l1 < 4, l2 < 4 or l3 < 3 (R9).  No fallback. */
    NC_E_FLOW = 4,       /* |tr A| > 1e-12 max(1, max|A_ij|): flow not incompressible */
    NC_E_STATE = 5,      /* call order: no box / flow / state set yet */
    NC_E_CUDA = 6,       /* a CUDA runtime error (text in nc_last_error) */
    NC_E_NCCL = 7,       /* an NCCL call of the slab path failed (text in nc_last_error) */
    NC_E_OOM = 8,        /* n or the cell count exceeds what was allocated; a cell above the pair kernel's
                            staging capacity (448 particles); a pair list above its cap */
    NC_E_NONFINITE = 9   /* a non-finite force, energy or virial was produced */
} nc_status;

/* Lattice remapping policies. */
typedef enum {
    NC_REMAP_NONE = 0, /* L_t = e^{At} L0 (Eq. 5) */
    NC_REMAP_LE = 1,   /* Lees-Edwards: shear A = eps e1 e2^T, tilt kept in [-1/2,1/2) by M of Eq. (8) */
    NC_REMAP_KR = 2,   /* Kraynik-Reinelt planar: L~ = e^{A (t mod t*)} L0 with e^{At*}L0 = L0 M (Eq. 9) */
    NC_REMAP_GKR = 3,  /* generalized KR, diagonal A: L~ = exp(diag(f1 w1 + f2 w2)) L0 (Eq. 10; R23) */
    NC_REMAP_REDUCE = 4 /* any traceless A ("general three dimensional linear flows"): L_t = e^{A(t-t_r)} L_r,
                           re-based by greedy pairwise Lagrange reduction (a unimodular change of basis of the same
                           lattice) whenever a box vector can be shortened -- the LE reset for shear;
                           R30.  Only L0 is used.  Valid while the lattice itself keeps h_k >= 3 r_c. */
} nc_remap_kind;

typedef struct {
    nc_remap_kind kind;
    double L0[9];      /* reference basis at t = 0 (row-major, columns = box vectors) */
    double tstar;      /* KR: period t* (> 0) */
    double omega1[3];  /* GKR: log-eigenvalues of the first automorphism, in the axis order of L0 */
    double omega2[3];  /* GKR: log-eigenvalues of the second automorphism */
    double beta[2];    /* GKR: alpha_k(t) = beta_k * eps * t; f_k = alpha_k - floor(alpha_k + 1/2) */
    double eps;        /* GKR: rate scale eps of A = eps diag(a) */
} nc_remap;

typedef struct {
    nc_variant variant;
    nc_prec prec;
    double rc;         /* cutoff d_cut; the pair test is r^2 < rc^2 strictly (R10) */
    double eps, sigma; /* LJ 12-6 parameters (R11) */
    double u_shift;    /* energy shift: phi(r) = 4 eps((s/r)^12-(s/r)^6) - u_shift for r < rc.
                          LJ: u_shift = phi_LJ(rc); WCA (rc = 2^(1/6) sigma): u_shift = -eps */
    double mass;       /* particle mass m (SLLOD) */
    int device;        /* CUDA device ordinal */
    void *stream;      /* cudaStream_t for all work (NULL = default stream) */
    int64_t capacity;  /* maximum particle count; buffers are allocated once in nc_create */
    int64_t max_cells; /* maximum cell count over the run (0 = derive from capacity: 2*capacity + 4096) */
} nc_config;

/* Per-evaluation instrumentation (R28): from the last force evaluation. */
typedef struct {
    int64_t n;                 /* particles */
    int32_t dims[3];           /* grid: c (DS) or l (DO) */
    int64_t ncells;
    double candidates;         /* (i, j, image) triples distance-checked, self excluded */
    double interactions;       /* ordered pairs with r < rc (|P| in DESIGN.md) */
    double stencil_cells;      /* sum over cells of the neighborhood size (mean = / ncells) */
    double rechecks;           /* fp32 candidates re-decided in canonical fp64 (R16) */
    double U;                  /* total potential energy */
    double W[6];               /* configurational virial 1/2 sum fr d(x)d: xx,yy,zz,xy,xz,yz (R12) */
    double acc_evals;          /* force evaluations since the last nc_profile(ctx, 1) */
    double acc_interactions;   /* their summed interactions */
    double acc_candidates;     /* their summed candidates */
    double interactions_fp32;  /* of interactions: evaluated in the fp32 far tier (counted in nc_profile mode 3 only) */
    double acc_interactions_fp32; /* their summed fp32-tier interactions (roofline accounting) */
} nc_stats;

/* Create a context on cfg->device; allocates all buffers for cfg->capacity
 * particles.  *out receives the context (NULL on failure).  Errors: NC_E_ARG,
 * NC_E_CUDA, NC_E_OOM. */
nc_status nc_create(const nc_config *cfg, nc_ctx **out);

/* Free the context and all device memory it owns (synchronizes its stream). */
void nc_destroy(nc_ctx *ctx);

/* Set the box L_t.  Recomputes the host geometry: L^{-1},
 * heights h_k, DS counts c_k or the QR factor R,
 * counts l_k and widths.  Errors: NC_E_BOX,
 * NC_E_DEGENERATE, NC_E_OOM (more cells than max_cells). */
nc_status nc_set_box(nc_ctx *ctx, const double L[9]);

/* Set the flow matrix A (row-major) and the remap policy at time t;
 * also sets the box to the policy's L~_t.  pol may be NULL (NC_REMAP_NONE
 * with L0 = current box).  Errors: NC_E_FLOW, NC_E_ARG, NC_E_BOX,
 * NC_E_DEGENERATE. */
nc_status nc_set_flow(nc_ctx *ctx, const double A[9], const nc_remap *pol, double t);

/* Wrap q into the unit cell Omega (R14, R15), compute cell keys
 * and sort particles into cells by (cell, gid) (R27).
 * q: n x 3 positions (device or host), read only -- the wrapped copy is kept
 * internally and returned by nc_get_cells / nc_get_wrapped.  Errors:
 * NC_E_ARG, NC_E_STATE (no box), NC_E_OOM, NC_E_CUDA. */
nc_status nc_build_cells(nc_ctx *ctx, const void *q, int64_t n);

/* One force evaluation (implies nc_build_cells): pair set by the chosen
 * cell list, F_i = -sum fr d, U, W (R11, R12).
 * F: n x 3 output (device or host), gid order, lab frame.  U, W: host
 * outputs (may be NULL).  Synchronizes the stream.  Errors: as
 * nc_build_cells, plus NC_E_NONFINITE. */
nc_status nc_compute_forces(nc_ctx *ctx, const void *q, int64_t n, void *F, double *U, double W[6]);

/* Pipelined force evaluations on HOST buffers (pinned memory for the copies
 * to overlap): the H2D copy of q runs on a library copy stream, the
 * evaluation on cfg.stream, the D2H copy of F on a second copy stream, with
 * double-buffered device staging, and the call returns without waiting, so
 * the copies of consecutive calls overlap the neighbouring evaluations.
 * q and F (n x 3, host) must stay valid, and F unread, until
 * nc_compute_sync, which waits for every pending evaluation and returns U and
 * W (may be NULL) of the LAST one; a non-finite result of any earlier one is
 * not reported.  Errors: as nc_compute_forces, plus NC_E_ARG for device
 * pointers and NC_E_STATE for nc_compute_sync without a pending call. */
nc_status nc_compute_forces_async(nc_ctx *ctx, const void *q, int64_t n, void *F);
nc_status nc_compute_sync(nc_ctx *ctx, double *U, double W[6]);

/* Load the resident particle state: positions q and PECULIAR momenta p
 * (n x 3, device or host, R19), particle ids gid (int64, may be NULL for
 * 0..n-1; otherwise a permutation of 0..n-1, NC_E_ARG if not: outputs are indexed
 * by gid).  Computes the initial forces.  Errors: as nc_compute_forces. */
nc_status nc_set_state(nc_ctx *ctx, const void *q, const void *p, const int64_t *gid, int64_t n);

/* Advance the resident state by nsteps SLLOD velocity-Verlet steps of size
 * dt (R19): kick + flow factor, drift with e^{A dt}, box update and remap
 * (P:342, 349, 380, 428, 433), rewrap, cell rebuild, forces, flow
 * factor + kick.  U, W (host, may be NULL) receive the values after the
 * last step.  The closing half kick of the last step may be held back and
 * fused into the next call's first kick (same arithmetic, bit for bit);
 * nc_get_state applies it first, so the state a caller reads is always the
 * complete step.  Errors: NC_E_STATE, NC_E_DEGENERATE, NC_E_NONFINITE,
 * NC_E_CUDA. */
nc_status nc_step_sllod(nc_ctx *ctx, double dt, int nsteps, double *U, double W[6]);

/* Copy the resident state out in gid order: q, p (n x 3, device or host,
 * may be NULL), gid (int64 host, may be NULL), the box L (host double[9],
 * may be NULL) and time t (may be NULL).  *n receives the count. */
nc_status nc_get_state(nc_ctx *ctx, void *q, void *p, int64_t *gid, int64_t *n, double L[9], double *t);

/* Parity instrumentation from the last build: cell_of[gid] (int64 host, n),
 * cell_start (int64 host, ncells+1), dims (int32[3]) and the wrapped
 * positions in gid order (host, n x 3, storage precision).  Any may be NULL. */
nc_status nc_get_cells(nc_ctx *ctx, int64_t *cell_of, int64_t *cell_start, int32_t dims[3], void *wrapped_q);

/* Per-particle pair digests (gid order, host arrays of n): cnt_i = number
 * of partners, hsum_i = sum mix64(key), hxor_i = xor mix64(key) with
 * key = gid_j | (n1+8)<<32 | (n2+8)<<36 | (n3+8)<<40 and n the lattice image
 * of the canonical displacement d = (q_j + L n) - q_i.  Runs a separate
 * digest evaluation of the last built cells (not on the timed path). */
nc_status nc_get_pair_digest(nc_ctx *ctx, uint32_t *cnt, uint64_t *hsum, uint64_t *hxor);

/* Full pair set of the last built cells (small N only): a separate digest evaluation (the same
 * kernel, membership decisions and tier split as the timed one) that also lists every ordered
 * pair (i, j, n) of the pair set P as 5 int32 per pair --
 * gid_i, gid_j, n1, n2, n3, with n the lattice image of the canonical displacement
 * d = (q_j + L n) - q_i -- sorted ascending by (gid_i, gid_j, n1, n2, n3) into i_j_n (host,
 * 5 x cap int32).  *npairs receives the count.  Errors: NC_E_STATE (no cells), NC_E_ARG,
 * NC_E_OOM if the list is longer than cap (*npairs still holds the count), NC_E_CUDA. */
nc_status nc_get_pairs(nc_ctx *ctx, int64_t cap, int32_t *i_j_n, int64_t *npairs);

/* Cell contents of the last build (parity of the counting sort, R27): gid of every slot of the
 * cell-sorted order (host int64, n); cell c holds slots [cell_start[c], cell_start[c+1]) of
 * nc_get_cells, in ascending gid.  Errors: NC_E_STATE, NC_E_ARG. */
nc_status nc_get_cell_gids(nc_ctx *ctx, int64_t *gid_sorted);

/* Per-particle interaction counts written by the TIMED pair kernel of the last force evaluation
 * (nc_compute_forces / nc_set_state / nc_step_sllod; not a digest run): cnt[gid] (host uint32, n).
 * A digest or pair-list call is itself an evaluation: read the counts before it.  Errors:
 * NC_E_STATE (no evaluation), NC_E_ARG. */
nc_status nc_get_pair_counts(nc_ctx *ctx, uint32_t *cnt);

/* Test hooks.  NC_DBG_DROP_ENTRIES = 1 drops the LAST entry of every neighborhood (a truncated
 * stencil: the negative control that parity tests must catch); 0 restores the method.  Takes
 * effect at the next nc_set_box / step.  Errors: NC_E_ARG. */
enum { NC_DBG_DROP_ENTRIES = 1 };
nc_status nc_debug(nc_ctx *ctx, int what, int value);

/* Instrumentation of the last evaluation. */
nc_status nc_get_stats(nc_ctx *ctx, nc_stats *out);

/* Histogram of neighborhood sizes over all cells of the current box
 * (index = size, 64 entries, host int64).  Runs a small kernel. */
nc_status nc_get_stencil_histogram(nc_ctx *ctx, int64_t hist[64]);

/* Live per-kernel timing with CUDA events recorded on cfg.stream around
 * every launch of the path (enable = 1 starts a fresh accumulation, 0 stops;
 * enable = 3 also makes k_pairs count its fp32-tier interactions, reported in
 * nc_stats.interactions_fp32 -- a separate, ~1% slower instantiation; bit 4 (enable = 5) times the
 * pair kernel only: two events per evaluation, the least instrumentation inside a timed region).
 * nc_profile_read synchronizes the stream and returns, per kernel id
 * (NC_K_*), the summed device milliseconds and the launch counts. */
enum { NC_K_WRAPKEY = 0, NC_K_SCAN = 1, NC_K_SCATTER = 2, NC_K_RANKGATHER = 3, NC_K_PAIRS = 4, NC_K_REDUCE = 5,
       NC_K_KICK = 6, NC_K_OTHER = 7, NC_K_COUNT = 8 };
nc_status nc_profile(nc_ctx *ctx, int enable);
nc_status nc_profile_read(nc_ctx *ctx, double ms[8], int64_t counts[8]);

/* ---------------------------------------------------------------------------
 * Slab decomposition for several GPUs (one process per GPU).
 * The box is cut into slabs of whole cell layers along the third lattice
 * direction (lambda_3; DS layer floor(lambda_3 c_3), DO layer floor(z/w_3),
 * z = r_33 lambda_3 -- the same axis for both variants).  Each rank owns the
 * particles of its layers, receives one r_c-thick halo layer from each
 * neighbour rank, and computes full i-side forces for its own particles only
 * (no reverse force communication).  The host driver
 * (paper_1412_3784_b200/slab.py) moves the packed buffers between ranks.
 * All pointers are DEVICE memory.  Arrays q, p, F are n x 3 (storage type),
 * gid is uint32.  Records: migration = 2 four-vectors per particle
 * (q.xyz + gid, p.xyz + 0), halo = 1 four-vector (q.xyz + gid); gid is the
 * bit pattern (fp32) or the exact value (fp64) of the fourth component.
 * ------------------------------------------------------------------------- */

/* Layers [klo, khi) owned by rank of nranks for the current box (needs
 * l3 >= 2 nranks).  Errors: NC_E_STATE, NC_E_DEGENERATE, NC_E_ARG. */
nc_status nc_slab_layers(nc_ctx *ctx, int rank, int nranks, int32_t *klo, int32_t *khi, int32_t *l3);

/* SLLOD first half (R19) on n own particles in place, then advance the box
 * to t + dt with its remap.  Positions are wrapped by nc_slab_migrate. */
nc_status nc_slab_kick_drift(nc_ctx *ctx, void *q, void *p, const void *F, int64_t n, double dt);

/* As nc_slab_kick_drift, preceded in the same pass by the PREVIOUS step's
 * closing half kick p <- e^{-A dt_prev/2} p + dt_prev/2 F (what nc_slab_kick
 * would have done with the same F; bitwise the same arithmetic), so a run of
 * slab steps needs no separate kick pass.  dt_prev = 0: no pending kick.
 * Errors: as nc_slab_kick_drift, NC_E_ARG for dt_prev < 0. */
nc_status nc_slab_kick_kick_drift(nc_ctx *ctx, void *q, void *p, const void *F, int64_t n, double dt_prev,
                                  double dt);

/* Wrap q in place (R15), then split the n particles by layer: those still
 * in [klo, khi) go to q_out/p_out/gid_out (index order), those in layer
 * klo-1 / khi (mod l3) are packed as migration records into send_lo /
 * send_hi (capacity cap each).  counts = (stay, to_lo, to_hi).
 * NC_E_STATE if a particle moved further than one layer. */
nc_status nc_slab_migrate(nc_ctx *ctx, void *q, const void *p, const uint32_t *gid, int64_t n, int klo, int khi,
                          void *q_out, void *p_out, uint32_t *gid_out, void *send_lo, void *send_hi, int64_t cap,
                          int64_t counts[3]);

/* Wrap q in place (R15) and write each particle's cell layer (DS floor(lambda_3 c_3), DO floor(z/w_3))
 * to layer (int32, device): the ownership test after the layer count l3 changed (GKR boxes, DS under
 * general flows), when particles can be further than one layer from their slab and the host driver
 * repartitions instead of migrating. */
nc_status nc_slab_layer_of(nc_ctx *ctx, void *q, int64_t n, int32_t *layer);

/* Unpack n migration records into n x 3 q, p and gid (append arrivals). */
nc_status nc_slab_unpack(nc_ctx *ctx, const void *rec, int64_t n, void *q, void *p, uint32_t *gid);

/* Pack halo records of the own particles in layer klo (-> halo_lo, for rank
 * r-1) and in layer khi-1 (-> halo_hi, for rank r+1).  counts = (lo, hi). */
nc_status nc_slab_halo(nc_ctx *ctx, void *q, const uint32_t *gid, int64_t n, int klo, int khi, void *halo_lo,
                       void *halo_hi, int64_t cap, int64_t counts[2]);

/* Forces on the n_own own particles (output F in their input order) with the
 * halo records received from the lower and upper neighbour; K3 runs over the
 * own layers [klo, khi) only.  layer_parts (host, (khi-klo) x 13 doubles, may
 * be NULL) receives the per-layer partials (U, W0..W5, interactions,
 * candidates, stencil cells, rechecks, fp32-tier interactions, non-finite)
 * for nc_slab_reduce. */
nc_status nc_slab_forces(nc_ctx *ctx, const void *q, const uint32_t *gid, int64_t n_own, const void *halo_from_lo,
                         int64_t n_lo, const void *halo_from_hi, int64_t n_hi, int klo, int khi, void *F,
                         double *layer_parts);

/* nc_slab_forces in two calls, so the halo exchange can overlap work: begin
 * (with the halo COUNTS n_lo, n_hi already known) sorts the own particles
 * into their cells and runs K3 on the interior own layers klo+1 .. khi-2,
 * whose neighborhoods contain own cells only; end (with the halo records)
 * sorts the halo particles in, runs K3 on the two boundary layers, reduces
 * and writes F and layer_parts exactly as nc_slab_forces (bitwise).  Both are
 * enqueued on cfg.stream; end synchronizes it.  Errors: as nc_slab_forces;
 * NC_E_STATE for end without begin. */
nc_status nc_slab_forces_begin(nc_ctx *ctx, const void *q, const uint32_t *gid, int64_t n_own, int64_t n_lo,
                               int64_t n_hi, int klo, int khi);
nc_status nc_slab_forces_end(nc_ctx *ctx, const void *halo_from_lo, const void *halo_from_hi, void *F,
                             double *layer_parts);

/* SLLOD second half: p <- E(-dt/2) p + dt/2 F on n own particles. */
nc_status nc_slab_kick(nc_ctx *ctx, void *p, const void *F, int64_t n, double dt);

/* Fixed-order sum of all l3 layers' partials (global layer order, host) ->
 * U, W (lab frame) and stats = (interactions, candidates, stencil cells,
 * rechecks): bitwise the same as a single-device evaluation. */
nc_status nc_slab_reduce(nc_ctx *ctx, const double *parts, int nlayers, double *U, double W[6], double stats[4]);

/* ---- The slab data plane over NCCL: the library moves the halo, migration and
 * partial-sum bytes itself, ring neighbours r-1 / r+1, on its own communication stream.  NCCL is loaded
 * at run time (the copy already in the process, else torch's wheel, else the system one).  The host
 * only has to broadcast the 128-byte unique id of rank 0 (e.g. torch.distributed.broadcast).
 * Errors: NC_E_NCCL (library missing or an NCCL call failed; text in nc_last_error), NC_E_ARG,
 * NC_E_STATE (no communicator / no exchange in flight), NC_E_OOM (a count above the capacity). */

/* A fresh NCCL unique id (rank 0 calls it and broadcasts the 128 bytes). */
nc_status nc_nccl_unique_id(uint8_t id[128]);

/* Join the communicator of nranks ranks (this context = rank `rank`, on cfg.device). */
nc_status nc_slab_comm_init(nc_ctx *ctx, int rank, int nranks, const uint8_t id[128]);

/* One ring exchange of records (`words` four-vectors of the storage type each: 2 for migration records,
 * 1 for halo records; device buffers): send_lo (n_lo records) goes to rank r-1, send_hi (n_hi) to
 * rank r+1; recv_lo receives rank r-1's upper send, recv_hi rank r+1's lower send, counts[2] = (from
 * r-1, from r+1), each at most cap.  _start exchanges the counts (one host synchronization of the
 * communication stream) and leaves the payload in flight on the communication stream after the work
 * already queued on cfg.stream; _wait makes cfg.stream wait for it (so K3 on interior layers overlaps
 * the transfer).  nc_slab_exchange = _start + _wait.  Messages to one peer are matched in issue
 * order, which makes P = 1 (a self ring) and P = 2 pair up correctly. */
nc_status nc_slab_exchange_start(nc_ctx *ctx, const void *send_lo, int64_t n_lo, const void *send_hi, int64_t n_hi,
                                 void *recv_lo, void *recv_hi, int64_t cap, int words, int64_t counts[2]);
nc_status nc_slab_exchange_wait(nc_ctx *ctx);
nc_status nc_slab_exchange(nc_ctx *ctx, const void *send_lo, int64_t n_lo, const void *send_hi, int64_t n_hi,
                           void *recv_lo, void *recv_hi, int64_t cap, int words, int64_t counts[2]);

/* All-gather of the per-layer partials (host in / out): this rank's nloc rows of 13 doubles (as
 * nc_slab_forces writes them), padded to max_rows; out receives nranks x max_rows rows in rank order. */
nc_status nc_slab_allgather(nc_ctx *ctx, const double *local, int64_t nloc, int64_t max_rows, double *out);

/* ---- Host-synchronization-free slab step (csrc/slab_dc.cuh, the step above without
 * any device-to-host read).  The context keeps the rank's own-particle count in device memory
 * (nc_sd_load sets it); every call below launches over the CAPACITY ncap and reads that count on the
 * device.  Messages are fixed-capacity device buffers of (1 + cap) records: record 0 is a header whose
 * first 4 bytes hold the record count (uint32), records 1..cap the payload (migration: 2 T4 words per
 * record = q.xyz + gid, p.xyz; halo: 1 word = q.xyz + gid); whole buffers are exchanged, so no count
 * crosses to the host.  The own particles of a force evaluation are sorted to fixed slots [H, H + n),
 * H = hcap per halo layer that precedes the own layers in cell order, so the interior layers' pair kernel
 * runs before the halo arrives.  F, U, W, the per-layer partials and whole trajectories are bitwise
 * those of nc_slab_* (and of one device).  Overflow of a message (more records than its capacity) or of
 * the own capacity drops the excess and sets a device flag; nc_sd_status reads count and flags (the
 * only synchronizing call) and fails with NC_E_OOM (overflow) or NC_E_STATE (a particle moved more
 * than one layer past its slab).
 *   nc_sd_load        the own count (device word) after the caller filled q, p, gid (n x 3, n, device).
 *   nc_sd_kick_drift  nc_slab_kick_kick_drift over the device count (box advanced on the host).
 *   nc_sd_kick        closing half kick over the device count.
 *   nc_sd_migrate     nc_slab_migrate into two migration messages (stayers to q_out, p_out, gid_out).
 *   nc_sd_absorb      both received migration messages appended after the own particles.
 *   nc_sd_halo        the boundary layers' particles into two halo messages.
 *   nc_sd_exchange_start  whole-buffer exchange with r-1 / r+1 over NCCL (nc_slab_comm_init first) on the
 *                     communication stream after the work queued on cfg.stream; nc_slab_exchange_wait
 *                     makes cfg.stream wait for it.
 *   nc_sd_forces_begin  own particles into cells at fixed slots, K3 on the interior own layers
 *                     (requires the context capacity >= ncap + 2 hcap).
 *   nc_sd_forces_end  received halo messages into cells, K3 on the boundary layers, reduction, forces of
 *                     the own particles in their local order into F (n x 3); parts (nlayers x 13
 *                     doubles, host) or NULL -- only a non-NULL parts synchronizes. */
nc_status nc_sd_load(nc_ctx *ctx, int64_t n);
nc_status nc_sd_status(nc_ctx *ctx, int64_t *n_own, uint32_t *flags);
nc_status nc_sd_kick_drift(nc_ctx *ctx, void *q, void *p, const void *F, int64_t ncap, double dt_prev, double dt);
nc_status nc_sd_kick(nc_ctx *ctx, void *p, const void *F, int64_t ncap, double dt);
nc_status nc_sd_migrate(nc_ctx *ctx, void *q, const void *p, const uint32_t *gid, int64_t ncap, int klo, int khi,
                        void *q_out, void *p_out, uint32_t *gid_out, void *msg_lo, void *msg_hi, int64_t mcap);
nc_status nc_sd_absorb(nc_ctx *ctx, const void *msg_lo, const void *msg_hi, int64_t mcap, void *q, void *p,
                       uint32_t *gid, int64_t ncap);
nc_status nc_sd_halo(nc_ctx *ctx, void *q, const uint32_t *gid, int64_t ncap, int klo, int khi, void *msg_lo,
                     void *msg_hi, int64_t hcap);
nc_status nc_sd_exchange_start(nc_ctx *ctx, const void *send_lo, const void *send_hi, void *recv_lo, void *recv_hi,
                               int64_t cap, int words);
nc_status nc_sd_forces_begin(nc_ctx *ctx, const void *q, const uint32_t *gid, int64_t ncap, int64_t hcap, int klo,
                             int khi);
nc_status nc_sd_forces_end(nc_ctx *ctx, const void *msg_lo, const void *msg_hi, void *F, double *parts);
/* nc_sd_forces_end, and the own particles adopt their sorted (cell, gid) order: q_out (wrapped q), p_out
 * (p gathered from the caller's p), gid_out and F in that order (all n x 3 / n, device; q_out, p_out,
 * gid_out distinct from the inputs) -- the next step then reads spatially ordered arrays. */
nc_status nc_sd_forces_end_sorted(nc_ctx *ctx, const void *msg_lo, const void *msg_hi, const void *p, void *q_out,
                                  void *p_out, uint32_t *gid_out, void *F, double *parts);

/* Peer-memory data plane of the slab step (the halo of P:445's cell layers and the migration
 * of particles between slabs, written by the packing kernels STRAIGHT into the neighbour ranks' receive
 * buffers -- pack and transfer in one pass over NVLink peer memory, no send buffer, copy or collective):
 *  nc_ipc_alloc       a zeroed device buffer of `bytes` owned by ctx (freed by nc_destroy), and its
 *                     64-byte cudaIpcMemHandle for the neighbours; pass *dptr as the RECEIVE buffer of
 *                     nc_sd_absorb / nc_sd_forces_end(_sorted);
 *  nc_ipc_open        map a neighbour's buffer from its handle (unmapped by nc_destroy); pass *dptr as
 *                     the msg_lo / msg_hi argument of nc_sd_halo / nc_sd_migrate, which then write the
 *                     neighbour's receive buffer directly;
 *  nc_ipc_event       an interprocess event of ctx (64-byte handle), returned as an id;
 *  nc_ipc_event_open  a neighbour's event from its handle, returned as an id;
 *  nc_ipc_record      record event `id` after the work queued on cfg.stream;
 *  nc_ipc_wait        cfg.stream waits for the latest record of event `id` (a stream wait: no kernel
 *                     spins).  A wait binds to the record that precedes it on the host, so the caller
 *                     separates neighbours' records from its waits by a host barrier (slab.IpcTransport).
 * Errors: NC_E_ARG (null / bad id), NC_E_CUDA (IPC not available, e.g. no peer access). */
nc_status nc_ipc_alloc(nc_ctx *ctx, int64_t bytes, void **dptr, void *handle);
nc_status nc_ipc_open(nc_ctx *ctx, const void *handle, void **dptr);
nc_status nc_ipc_event(nc_ctx *ctx, void *handle, int *id);
nc_status nc_ipc_event_open(nc_ctx *ctx, const void *handle, int *id);
nc_status nc_ipc_record(nc_ctx *ctx, int id);
nc_status nc_ipc_wait(nc_ctx *ctx, int id);

/* Choice of the K3 pair kernel.  All evaluate the same neighborhoods, the
 * same candidates and the same pair set; they differ in how work maps to warps.  NC_F64 has two:
 * the warp-per-cell kernel and a particle-per-thread one (NC_PK_SPARSE, k_pairs_sparse64; AUTO
 * below 4 particles per cell), both with the canonical fp64 test on every candidate.  NC_F32:
 *  NC_PK_AUTO    (default) per cell when the mean occupancy is at least 4 particles per
 *                cell; below that (WCA at rho = 0.8442: ~1.3) per particle from 2^18
 *                particles on and on grids of fewer than 65,536 cells (there with two,
 *                four or eight threads per particle), per row segment otherwise;
 *  NC_PK_CELL    one warp per center cell (k_pairs);
 *  NC_PK_SEGMENT one 2-warp block per row segment of cells sharing one staged
 *                union of their neighborhoods (k_pairs_seg, round 1), fp64 pair forces;
 *  NC_PK_SPARSE  one thread per particle, 32 consecutive particles of a cell row per warp walking
 *                their exact stencils in lockstep through L1 (k_pairs_sparse), fp64 pair forces;
 *  NC_PK_ROWS    one warp per cell row, batches of 32 consecutive particles whose neighbour rows
 *                are staged once in shared memory (k_pairs_rows, round 2), fp64 pair forces
 *                bitwise those of NC_PK_SPARSE.
 * Errors: NC_E_ARG (bad value, or NC_PK_SEGMENT / NC_PK_ROWS on an NC_F64 context).
 * nc_pair_kernel_used returns the kernel of the last evaluation (1, 2, 3 or 4, 0 = none). */
typedef enum { NC_PK_AUTO = 0, NC_PK_CELL = 1, NC_PK_SEGMENT = 2, NC_PK_SPARSE = 3, NC_PK_ROWS = 4 } nc_pair_kernel;
nc_status nc_set_pair_kernel(nc_ctx *ctx, int which);
int nc_pair_kernel_used(const nc_ctx *ctx);

/* Number of kernel launches this context has issued so far. */
int64_t nc_launch_count(const nc_ctx *ctx);

/* Text of the last error on ctx (or of the last nc_create failure if ctx is NULL). */
const char *nc_last_error(const nc_ctx *ctx);

/* Library version string. */
const char *nc_version(void);

#ifdef __cplusplus
}
#endif
#endif /* NEMDCELL_H */
