// kernels.cuh -- sm_100a kernels of the cell-list force path (arXiv 1412.3784).
//
//   K1  k_wrap_key        : lambda = L^{-1} q (canonical fp64), wrap into Omega,
//                           DS / DO cell key, fused histogram (atomic slot)
//   K2  k_scan_*          : exclusive scan of the cell histogram -> cell_start
//       k_scatter         : particle -> (cell, arrival slot) bucket
//       k_rank_gather     : stable (cell, gid) order; gather q, p, gid and the
//                           cell-local rotated coordinates u (+ DO home shift)
//   K3  k_pairs           : warp-per-cell pair kernel: builds the 27 (DS) or
//                           27/30/34/36 (DO) neighborhood on the fly, stages
//                           the neighbor particles (image shift applied) in
//                           shared memory, filters r^2 < r_c^2 (1 + tau) two
//                           candidates at a time (LDS.64 + FADD2/FFMA2) into
//                           per-lane hit words, evaluates the hits in a packed
//                           fp32 far tier and an fp64 close tier, full i-side
//                           accumulation, no atomics
//       k_pairs_seg       : the same pair set for sparse cells (k3_seg.cuh)
//   K3r k_reduce          : deterministic fixed-order reduction of partials (one launch)
//   K4  k_kick_drift_key  : SLLOD half kick + flow factor + drift, fused with K1 (and with
//                           the previous step's deferred closing half kick)
//       k_kick            : SLLOD flow factor + half kick (when the state is read)
//
// Canonical fp64 arithmetic (reading R16): every operation that decides an
// integer (wrap, cell key, stencil rows/columns, pair membership in the
// re-check band) uses explicit round-to-nearest intrinsics (__dmul_rn,
// __dadd_rn, __ddiv_rn) in the association order of the definition, so no
// FMA contraction can change a decision.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "geom.hpp"

namespace nc {

// Programmatic dependent launch (sm_90+): the step's kernels are launched with programmatic stream
// serialization, so the next kernel's grid is set up while this one drains; every such kernel waits
// for its predecessor's completion (and memory) before its first dependent access, and lets its
// successor launch as soon as all its own blocks have started.  Without the launch attribute both are
// no-ops.
#define PDL_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")
#define PDL_LAUNCH() asm volatile("griddepcontrol.launch_dependents;" :::)
#define PDL_ENTRY() do { PDL_WAIT(); PDL_LAUNCH(); } while (0)
// bounds checks of shared-memory indices in the newer pair kernels (a debug build: -DNC_BOUNDS; a failed
// check traps the kernel, which the host reports as NC_E_CUDA)
#ifdef NC_BOUNDS
#define NC_CHECK(c) do { if (!(c)) __trap(); } while (0)
#else
#define NC_CHECK(c) do { } while (0)
#endif

template <typename T> struct V4;
template <> struct V4<float> { using t = float4; };
template <> struct V4<double> { using t = double4; };

// Arrival slot in cell c's bucket (counting sort): one atomic per group of lanes with the same
// cell (cells are sorted, so a warp covers 2-3 cells); slots only need to be distinct, the
// (cell, gid) rank of k_rank_gather fixes the final order.
__device__ __forceinline__ uint32_t arrival_slot(uint32_t* counts, uint32_t c) {
  const uint32_t act = __activemask();
  const uint32_t peers = __match_any_sync(act, c);
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(peers) - 1;
  uint32_t base = 0;
  if (lane == leader) base = atomicAdd(&counts[c], (uint32_t)__popc(peers));
  base = __shfl_sync(act, base, leader);
  return base + (uint32_t)__popc(peers & ((1u << lane) - 1u));
}

__device__ __forceinline__ float4 mk4(float x, float y, float z, float w) { return make_float4(x, y, z, w); }
__device__ __forceinline__ double4 mk4(double x, double y, double z, double w) { return make_double4(x, y, z, w); }

// index <-> 4th component (bit pattern for fp32, exact value for fp64)
__device__ __forceinline__ float idx_to_w(uint32_t i, float) { return __uint_as_float(i); }
__device__ __forceinline__ double idx_to_w(uint32_t i, double) { return (double)i; }
__device__ __forceinline__ uint32_t w_to_idx(float w) { return __float_as_uint(w); }
__device__ __forceinline__ uint32_t w_to_idx(double w) { return (uint32_t)w; }

__device__ __forceinline__ double round_to(double v, float) { return (double)__double2float_rn(v); }
__device__ __forceinline__ double round_to(double v, double) { return v; }

__device__ __forceinline__ int floordiv(int a, int b) {  // floor(a / b) for b > 0
  // neighbor offsets are small: compare-based fast paths avoid the integer-division sequence
  if (a >= 0 && a < b) return 0;
  if (a < 0 && a >= -b) return -1;
  if (a >= b && a < 2 * b) return 1;
  int q = a / b;
  if ((a % b) != 0 && ((a < 0) != (b < 0))) --q;
  return q;
}
__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// canonical lambda_k = (Li_k0 q0 + Li_k1 q1) + Li_k2 q2
__device__ __forceinline__ void frac_c(const Geom& g, double q0, double q1, double q2, double* lam) {
#pragma unroll
  for (int k = 0; k < 3; ++k)
    lam[k] = __dadd_rn(__dadd_rn(__dmul_rn(g.Li[3 * k], q0), __dmul_rn(g.Li[3 * k + 1], q1)),
                       __dmul_rn(g.Li[3 * k + 2], q2));
}

// canonical lattice shift s_a = (L_a0 n0 + L_a1 n1) + L_a2 n2
__device__ __forceinline__ double lshift_c(const Geom& g, int a, int n0, int n1, int n2) {
  return __dadd_rn(__dadd_rn(__dmul_rn(g.L[3 * a], (double)n0), __dmul_rn(g.L[3 * a + 1], (double)n1)),
                   __dmul_rn(g.L[3 * a + 2], (double)n2));
}

// Cell of one particle from its fractional coordinates (P:668-672
// with R1, R2, R14).  Returns the x-fastest cell id, the cell coordinates,
// the DO home shift nh = (-kx, -ky, 0) and the rotated rearranged point.
struct CellPos {
  int a[3];
  int nh0, nh1;
  double xr[3];  // DO: rearranged rotated point (x', y', z); DS: unused
};

__device__ __forceinline__ uint32_t cell_of(const Geom& g, const double* lam, CellPos& cp) {
  if (g.variant == 0) {
#pragma unroll
    for (int k = 0; k < 3; ++k) cp.a[k] = clampi((int)floor(__dmul_rn(lam[k], (double)g.dims[k])), 0, g.dims[k] - 1);
    cp.nh0 = cp.nh1 = 0;
  } else {
    double x = __dadd_rn(__dadd_rn(__dmul_rn(g.R[0], lam[0]), __dmul_rn(g.R[1], lam[1])), __dmul_rn(g.R[2], lam[2]));
    double y = __dadd_rn(__dmul_rn(g.R[4], lam[1]), __dmul_rn(g.R[5], lam[2]));
    double z = __dmul_rn(g.R[8], lam[2]);
    double ky = floor(__ddiv_rn(y, g.R[4]));
    double yp = __dsub_rn(y, __dmul_rn(ky, g.R[4]));
    double xpp = __dsub_rn(x, __dmul_rn(ky, g.R[1]));
    double kx = floor(__ddiv_rn(xpp, g.R[0]));
    double xp = __dsub_rn(xpp, __dmul_rn(kx, g.R[0]));
    cp.a[0] = clampi((int)floor(__ddiv_rn(xp, g.w[0])), 0, g.dims[0] - 1);
    cp.a[1] = clampi((int)floor(__ddiv_rn(yp, g.w[1])), 0, g.dims[1] - 1);
    cp.a[2] = clampi((int)floor(__ddiv_rn(z, g.w[2])), 0, g.dims[2] - 1);
    cp.nh0 = -(int)kx;
    cp.nh1 = -(int)ky;
    cp.xr[0] = xp;
    cp.xr[1] = yp;
    cp.xr[2] = z;
  }
  return (uint32_t)cp.a[0] + (uint32_t)g.dims[0] * ((uint32_t)cp.a[1] + (uint32_t)g.dims[1] * (uint32_t)cp.a[2]);
}

// Cell-local coordinates in the QR-rotated frame (not canonical: they only
// feed the fp32/fp64 distance filter and the forces).  DS: u = R(lambda - a/c);
// DO: u = (x' - a0 w0, y' - a1 w1, z - a2 w2).
__device__ __forceinline__ void local_u(const Geom& g, const double* lam, const CellPos& cp, double* u) {
  if (g.variant == 0) {
    double m0 = lam[0] - (double)cp.a[0] * g.cinv[0];
    double m1 = lam[1] - (double)cp.a[1] * g.cinv[1];
    double m2 = lam[2] - (double)cp.a[2] * g.cinv[2];
    u[0] = g.R[0] * m0 + g.R[1] * m1 + g.R[2] * m2;
    u[1] = g.R[4] * m1 + g.R[5] * m2;
    u[2] = g.R[8] * m2;
  } else {
    u[0] = cp.xr[0] - (double)cp.a[0] * g.w[0];
    u[1] = cp.xr[1] - (double)cp.a[1] * g.w[1];
    u[2] = cp.xr[2] - (double)cp.a[2] * g.w[2];
  }
}

__device__ __forceinline__ uint32_t pack_nh(int nh0, int nh1) {
  return ((uint32_t)(nh0 & 0xffff)) | ((uint32_t)(nh1 & 0xffff) << 16);
}
__device__ __forceinline__ int nh_x(uint32_t p) { return (int)(int16_t)(p & 0xffff); }
__device__ __forceinline__ int nh_y(uint32_t p) { return (int)(int16_t)(p >> 16); }

// ---------------------------------------------------------------------------
// K1: wrap + key + histogram.  qin: n x stride (stride 3 = caller layout,
// 4 = internal).  Stored (wrapped, rounded to T) positions go to qout.
// Wrap rule (R14, R15): if lambda outside [0,1)^3, q <- round_T(q - L floor(lambda))
// once; keys from the stored value, clamped.
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ uint32_t wrap_key_one(const Geom& g, double& q0, double& q1, double& q2) {
  double lam[3];
  frac_c(g, q0, q1, q2, lam);
  if (lam[0] < 0.0 || lam[0] >= 1.0 || lam[1] < 0.0 || lam[1] >= 1.0 || lam[2] < 0.0 || lam[2] >= 1.0) {
    int n0 = (int)floor(lam[0]), n1 = (int)floor(lam[1]), n2 = (int)floor(lam[2]);
    q0 = round_to(__dsub_rn(q0, lshift_c(g, 0, n0, n1, n2)), T());
    q1 = round_to(__dsub_rn(q1, lshift_c(g, 1, n0, n1, n2)), T());
    q2 = round_to(__dsub_rn(q2, lshift_c(g, 2, n0, n1, n2)), T());
    frac_c(g, q0, q1, q2, lam);
  }
  CellPos cp;
  return cell_of(g, lam, cp);
}

template <typename T>
__global__ void k_wrap_key(int64_t n, const T* __restrict__ qin, int stride, typename V4<T>::t* __restrict__ qout,
                           uint32_t* __restrict__ key, uint32_t* __restrict__ slot, uint32_t* __restrict__ counts,
                           const __grid_constant__ Geom g) {
  PDL_ENTRY();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double q0 = (double)qin[i * stride], q1 = (double)qin[i * stride + 1], q2 = (double)qin[i * stride + 2];
  uint32_t c = wrap_key_one<T>(g, q0, q1, q2);
  qout[i] = mk4((T)q0, (T)q1, (T)q2, (T)0);
  key[i] = c;
  slot[i] = arrival_slot(counts, c);
}

// ---------------------------------------------------------------------------
// K2: exclusive scan (3 phases, deterministic: integer counts).
// ---------------------------------------------------------------------------
constexpr int SCAN_T = 256, SCAN_E = 8, SCAN_TILE = SCAN_T * SCAN_E;

__global__ void k_scan_reduce(const uint32_t* __restrict__ in, int64_t m, uint32_t* __restrict__ bsum) {
  PDL_ENTRY();
  __shared__ uint32_t s[SCAN_T / 32];
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  uint32_t acc = 0;
  for (int k = 0; k < SCAN_E; ++k) {
    int64_t idx = base + (int64_t)k * SCAN_T + threadIdx.x;
    if (idx < m) acc += in[idx];
  }
  acc = __reduce_add_sync(0xffffffffu, acc);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < SCAN_T / 32; ++w) t += s[w];
    bsum[blockIdx.x] = t;
  }
}

// single block: exclusive scan of nb block sums in place; total to *tot
__global__ void k_scan_bsums(uint32_t* __restrict__ bsum, int64_t nb, uint32_t* __restrict__ tot) {
  PDL_ENTRY();
  __shared__ uint32_t carry_s;
  __shared__ uint32_t wsum[32];
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  for (int64_t base = 0; base < nb; base += blockDim.x) {
    int64_t idx = base + threadIdx.x;
    uint32_t v = idx < nb ? bsum[idx] : 0u;
    uint32_t x = v;
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    if (wid == 0) {
      uint32_t ws = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, ws, o);
        if (lane >= o) ws += y;
      }
      wsum[lane] = ws;
    }
    __syncthreads();
    uint32_t excl = carry_s + (wid > 0 ? wsum[wid - 1] : 0u) + x - v;
    if (idx < nb) bsum[idx] = excl;
    __syncthreads();
    if (threadIdx.x == 0) carry_s += wsum[(blockDim.x >> 5) - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) *tot = carry_s;
}

// out[i] = exclusive prefix of in; out[m] = total (out has m+1 entries)
__global__ void k_scan_apply(const uint32_t* __restrict__ in, int64_t m, const uint32_t* __restrict__ bsum,
                             uint32_t* __restrict__ out, const uint32_t* __restrict__ tot) {
  PDL_ENTRY();
  __shared__ uint32_t wsum[SCAN_T / 32];
  __shared__ uint32_t carry_s;
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry_s = bsum[blockIdx.x];
  __syncthreads();
  // each thread owns SCAN_E consecutive elements
  int64_t my0 = base + (int64_t)threadIdx.x * SCAN_E;
  uint32_t v[SCAN_E], s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_E; ++k) {
    v[k] = (my0 + k < m) ? in[my0 + k] : 0u;
    s += v[k];
  }
  uint32_t x = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < SCAN_T / 32; ++w) {
      uint32_t c = wsum[w];
      wsum[w] = t;
      t += c;
    }
  }
  __syncthreads();
  uint32_t run = carry_s + wsum[wid] + x - s;
#pragma unroll
  for (int k = 0; k < SCAN_E; ++k) {
    if (my0 + k < m) out[my0 + k] = run;
    run += v[k];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[m] = *tot;
}

// Small inputs (m <= SCAN_SMALL): the whole exclusive scan in one block, one launch instead of
// three (C1's 24k cells, C2's 20k, slab migration blocks, ...).  One SM does all of it, so it is bound by
// that SM's instruction issue: each thread scans its own run of R consecutive counts (R a multiple of 4,
// loaded / stored as 16-byte vectors, kept in registers), then one warp scan of the run totals and one of
// the warp totals.  out[m] = total.  (A shared-memory copy with strided runs was bound by bank conflicts,
// and a 32-wide shuffle scan per step by issue: ~10 us for C1's 24k cells either way.)
constexpr int SCAN_SMALL_T = 1024, SCAN_SMALL_R = 32, SCAN_SMALL = SCAN_SMALL_R * SCAN_SMALL_T;
__global__ void __launch_bounds__(SCAN_SMALL_T) k_scan_small(const uint32_t* __restrict__ in, int64_t m,
                                                             uint32_t* __restrict__ out) {
  PDL_ENTRY();
  __shared__ uint32_t wsum[SCAN_SMALL_T / 32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int mm = (int)m;
  const int R = ((mm + SCAN_SMALL_T - 1) / SCAN_SMALL_T + 3) & ~3;  // run length, a multiple of 4
  const int b0 = tid * R;
  uint32_t v[SCAN_SMALL_R];
#pragma unroll
  for (int q = 0; q < SCAN_SMALL_R / 4; ++q) {
    const int i = b0 + 4 * q;
    uint4 x = make_uint4(0u, 0u, 0u, 0u);
    if (4 * q < R) {
      if (i + 4 <= mm) {
        x = *reinterpret_cast<const uint4*>(in + i);
      } else {
        if (i < mm) x.x = in[i];
        if (i + 1 < mm) x.y = in[i + 1];
        if (i + 2 < mm) x.z = in[i + 2];
      }
    }
    v[4 * q] = x.x; v[4 * q + 1] = x.y; v[4 * q + 2] = x.z; v[4 * q + 3] = x.w;
  }
  uint32_t run = 0;
#pragma unroll
  for (int k = 0; k < SCAN_SMALL_R; ++k) {  // exclusive prefixes inside the run (zeros past R / m)
    const uint32_t c = v[k];
    v[k] = run;
    run += c;
  }
  uint32_t x = run;  // inclusive scan of the run totals: warp, then warp sums
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t w = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    wsum[lane] = w;  // inclusive over warps
  }
  __syncthreads();
  const uint32_t pre = (wid > 0 ? wsum[wid - 1] : 0u) + x - run;  // exclusive prefix of this run
#pragma unroll
  for (int q = 0; q < SCAN_SMALL_R / 4; ++q) {
    const int i = b0 + 4 * q;
    if (4 * q < R) {
      const uint4 y = make_uint4(pre + v[4 * q], pre + v[4 * q + 1], pre + v[4 * q + 2], pre + v[4 * q + 3]);
      if (i + 4 <= mm) {
        *reinterpret_cast<uint4*>(out + i) = y;
      } else {
        if (i < mm) out[i] = y.x;
        if (i + 1 < mm) out[i + 1] = y.y;
        if (i + 2 < mm) out[i + 2] = y.z;
      }
    }
  }
  if (tid == 0) out[m] = wsum[31];
}

// bucket each particle at (cell_start[key] + arrival slot); carry its gid
__global__ void k_scatter(int64_t n, const uint32_t* __restrict__ key, const uint32_t* __restrict__ slot,
                          const uint32_t* __restrict__ cs, const uint32_t* __restrict__ gid_in,
                          uint4* __restrict__ rec, int64_t i0 = 0, const uint32_t* __restrict__ dn = nullptr,
                          uint32_t* __restrict__ zero = nullptr, int64_t nzero = 0) {
  PDL_ENTRY();
  // zero: the cell counts, consumed by the scan before this kernel, cleared for the next step's
  // histogram (one memset fewer per step, so the step's launches chain without a break)
  if (zero)
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < nzero; c += (int64_t)gridDim.x * blockDim.x)
      zero[c] = 0u;
  // particles [i0, i0 + n) (a slab evaluation scatters its own and its halo particles separately).
  // One 16-byte record per particle (source index, gid, cell): a random-order input costs one sector
  // per particle, not three; k_rank_gather reads the records in bucket order (coalesced)
  // (dn: the count lives on the device -- the grid covers a capacity; host-synchronization-free slab step)
  if (dn) n = (int64_t)min((unsigned long long)n, (unsigned long long)*dn);
  int64_t i = i0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= i0 + n) return;
  const uint32_t c = key[i];
  const uint32_t pos = cs[c] + slot[i];
  rec[pos] = make_uint4((uint32_t)i, gid_in ? gid_in[i] : (uint32_t)i, c, 0u);
}

// cs[c] += b for c in [c0, c1): the own cells' starts after the halo particles that precede them
__global__ void k_add_range(uint32_t* __restrict__ cs, int64_t c0, int64_t c1, uint32_t b,
                            const uint32_t* __restrict__ db = nullptr) {
  if (db) b += *db;  // device-side part of the offset (host-synchronization-free slab step)
  const int64_t c = c0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c < c1) cs[c] += b;
}

#ifndef RG_MINB
#define RG_MINB 8  // 32 registers, full occupancy: 2.06 -> 1.53 ms on C4 (the gathers need warps in flight)
#endif
// Stable (cell, gid) order (R27): the destination of bucket entry s is
// cell_start + #{members with smaller gid}.  Gathers q (stored), p, gid and
// writes the cell-local rotated coordinates u (4th component = sorted index)
// and the packed DO home shift.
template <typename T>
__global__ void __launch_bounds__(256, RG_MINB)
k_rank_gather(int64_t n, const uint4* __restrict__ rec, const uint32_t* __restrict__ cs,
                              const typename V4<T>::t* __restrict__ qw, const typename V4<T>::t* __restrict__ p_in,
                              typename V4<T>::t* __restrict__ q_out, typename V4<T>::t* __restrict__ p_out,
                              uint32_t* __restrict__ gid_out, double4* __restrict__ u_out,
                              float4* __restrict__ u32_out, uint32_t* __restrict__ nh_out,
                              const __grid_constant__ Geom g, uint32_t* __restrict__ idx_out = nullptr,
                              int64_t s0 = 0, const uint32_t* __restrict__ drange = nullptr) {
  PDL_ENTRY();
  // bucket positions [s0, s0 + n) (a slab evaluation places own and halo particles in two phases);
  // drange: [drange[0], drange[1]) from the device (the grid covers a capacity)
  int64_t send = s0 + n;
  if (drange) { s0 = drange[0]; send = (int64_t)min((long long)drange[1], (long long)(s0 + n)); }
  int64_t s = s0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= send) return;
  const uint4 r = rec[s];
  const uint32_t i = r.x, gg = r.y, c = r.z;
  const typename V4<T>::t q = qw[i];  // gathers issued before the rank loop
  const uint32_t c0 = cs[c], c1 = cs[c + 1];
  uint32_t rank = 0;
  for (uint32_t t = c0; t < c1; ++t) rank += (rec[t].y < gg) ? 1u : 0u;
  uint32_t dst = c0 + rank;
  double lam[3];
  frac_c(g, (double)q.x, (double)q.y, (double)q.z, lam);
  CellPos cp;
  cell_of(g, lam, cp);
  double u[3];
  local_u(g, lam, cp, u);
  q_out[dst] = q;
  if (p_in) p_out[dst] = p_in[i];
  gid_out[dst] = gg;
  u_out[dst] = make_double4(u[0], u[1], u[2], (double)dst);
  u32_out[dst] = make_float4((float)u[0], (float)u[1], (float)u[2], (float)cp.a[0]);  // .w: cell column (exact)
  nh_out[dst] = pack_nh(cp.nh0, cp.nh1);
  if (idx_out) idx_out[dst] = i;
}

// ---------------------------------------------------------------------------
// K3: the pair kernel.
//
// Precision design: the candidate FILTER runs in the
// storage type T (fp32 in NC_F32 mode: ~85% of candidates are rejected there);
// every candidate that passes is re-evaluated from fp64 cell-local coordinates
// (error ~1e-16 |d|) and its force, energy and virial are computed and
// accumulated in fp64.  Membership is decided by the fp64 r^2, and inside a
// 1e-12 relative band around r_c^2 by the canonical fp64 test of R16.
// ---------------------------------------------------------------------------
#ifndef K3_PF_L2
#define K3_PF_L2 1  // L2 prefetch of the staged particles' fp64 coordinates (close tier): fluid -0.5%, lattice +0.4%
#endif
#ifndef NC_F64_SPLIT_B
#define NC_F64_SPLIT_B 8
#endif
constexpr int K3_F64_SPLIT_B = NC_F64_SPLIT_B;  // NC_F64 small grids: particles per i-batch when blocks share a cell
#ifndef K3_CAP_OVR
#define K3_CAP_OVR 448
#endif
constexpr int K3_CAP = K3_CAP_OVR;  // staged neighbor particles per warp per chunk
constexpr int K3_DUMMY = K3_CAP + 64;  // permanent far element (padding slot of the evaluation)
constexpr int K3_STAGE = K3_CAP + 66;  // fp64 mode: + up to S far sentinels so the filter needs no bounds checks
#ifndef K3_QCAP_OVR
#define K3_QCAP_OVR 48
#endif
#ifndef K3_MAXNREG
#define K3_MAXNREG 0  // nonzero: register cap for k_pairs instead of K3_MINB
#endif
#ifndef K3_MINB
#define K3_MINB 14
#endif
typedef uint16_t K3QT;  // queue entries: low 16 bits of shared addresses (see addr_from16)
#ifndef K3_STGR
#define K3_STGR 4  // staging: global loads in flight per lane
#endif
#ifndef K3_MW_OVR
#define K3_MW_OVR 15
#endif
constexpr int K3_MW = K3_MW_OVR;  // hit words per lane (static_assert in filter_chunk_f32: enough for one chunk)
#ifndef K3_CQ_OVR
#define K3_CQ_OVR 24
#endif
constexpr int K3_CQ = K3_CQ_OVR;  // close-tier queue entries per lane (mask mode); flushed when nearly full
constexpr uint32_t K3_QSTRIDE = 32u * sizeof(K3QT);  // bytes between consecutive entries of one lane
constexpr int K3_QCAP = K3_QCAP_OVR;     // per-lane queue of filter survivors (low 16 bits of shared addresses / staged indices)
#ifndef K3_UNROLL_OVR
#define K3_UNROLL_OVR 8
#endif
constexpr int K3_UNROLL = K3_UNROLL_OVR;  // filter steps per group (loads of a group issued together)
constexpr int K3_MAXE = 40;     // neighborhood entries (<= 36)
#ifndef K3_CELLS_OVR
#define K3_CELLS_OVR 1
#endif
constexpr int K3_CELLS = K3_CELLS_OVR;  // fewest cells per warp (= per block: one warp per block)
#ifndef K3_CELLS_MAX
#define K3_CELLS_MAX 16  // most cells per block (large layers; host cells_per_block)
#endif
constexpr int NPART = 13;       // U, W0..W5, interactions, candidates, stencil cells, rechecks, fp32-tier interactions, nonfinite
constexpr double K3_BAND64 = 1e-12;

// fp32 mode: staged x, y, z (image bracket applied, centred on the center cell) and |v|^2 as four
// arrays of stride K3_SSTR floats.  K3_SSTR = 8 (mod 32): the four words one mma B fragment takes
// (lane (g, t) reads component t of element 8k + g) fall in four disjoint bank octets.
constexpr int K3_SSTR = ((K3_CAP + 64 + 1 + 23) / 32) * 32 + 8;  // > K3_DUMMY, = 8 (mod 32): 520 for 448
constexpr int K3_HW = (K3_CAP + 127) / 128;  // hit words per (row, MMA stream): 16 column blocks each
static_assert(K3_SSTR % 32 == 8 && K3_SSTR > K3_DUMMY && 128 * K3_HW <= K3_DUMMY, "staging stride / padding");
template <typename T>
struct K3Stage64 {
  float sc[4][K3_SSTR];
};
template <>
struct K3Stage64<double> {  // fp64 mode: stage holds LAB positions; packed DO home shift of each j
  uint32_t nh[K3_STAGE];
};

template <typename T>
struct K3Smem {
  typename V4<T>::t stage[sizeof(T) == 8 ? K3_STAGE : 1];  // fp64 mode: staged lab positions, .w = sorted index
  K3Stage64<T> s64;
  K3QT queue[sizeof(T) == 4 ? K3_CQ : K3_QCAP][32];  // fp32: close-tier queue; fp64: survivor queue
  union {  // fp32: the entries' fp32 brackets while staging, then the hit words [row][MMA stream t][word w]
    float Bf[K3_MAXE][3];
    uint32_t hw[sizeof(T) == 4 ? 16 * 4 * K3_HW : 1];
  };
  uint8_t sent[K3_STAGE];
  uint32_t e_start[K3_MAXE], e_cnt[K3_MAXE], e_off[K3_MAXE];
  int8_t e_n[K3_MAXE][3];  // lattice image shift of the entry (|n_k| <= 2)
  int e_center;            // the entry of the center cell itself (build_entries)
  double e_B[K3_MAXE][3];
};

// Full (i, j, n) pair lists for nc_get_pairs (digest instantiations only; small N): one global
// atomic slot per ordered pair, the host sorts.
struct PairOut {
  int32_t* ijn;            // 5 x int32 per pair: gid_i, gid_j, n1, n2, n3
  unsigned long long* n;   // pairs found (may exceed cap: the host reports the count)
  long long cap;
  void* fu = nullptr;      // user-order forces (n x 3 of T, index = gid): the owner writes F there too,
                           // so an evaluation from user positions needs no separate unsort pass
};
// F of particle `me` (sorted) into the user-order output at its gid (scattered; overlapped with K3's work)
template <typename V>
__device__ __forceinline__ void store_user_F(const PairOut& po, const uint32_t* __restrict__ gid, uint32_t me,
                                             const V& f) {
  if (po.fu) {
    using T = decltype(f.x);
    T* d = (T*)po.fu + 3 * (size_t)gid[me];
    d[0] = f.x; d[1] = f.y; d[2] = f.z;
  }
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// Build the neighborhood of center cell (a0,a1,a2) into smem; returns the
// entry count (warp-uniform).  DS: 27 cells m = a + delta wrapped with
// n_k = floor(m_k/c_k); bracket B = R(delta/c).  DO: exact
// interval overlap (R3-R5), bracket
// B = ((col-a0) w0 + n1 e0 + n2 r12 + n3 r13, (m-a1) w1 + n2 e1 + n3 r23, dz w2 + n3 e2).
template <typename SM>
__device__ __forceinline__ int build_entries(const Geom& g, int a0, int a1, int a2, SM& sm, int lane) {
  const int l1 = g.dims[0], l2 = g.dims[1], l3 = g.dims[2];
  if (g.variant == 0) {
    if (lane < 27) {
      int d0 = lane % 3 - 1, d1 = (lane / 3) % 3 - 1, d2 = lane / 9 - 1;
      int m0 = a0 + d0, m1 = a1 + d1, m2 = a2 + d2;
      int n0 = floordiv(m0, l1), n1 = floordiv(m1, l2), n2 = floordiv(m2, l3);
      m0 -= n0 * l1; m1 -= n1 * l2; m2 -= n2 * l3;
      uint32_t cell = (uint32_t)m0 + (uint32_t)l1 * ((uint32_t)m1 + (uint32_t)l2 * (uint32_t)m2);
      sm.e_start[lane] = cell;  // the cell id until the counts pass replaces it
      sm.e_n[lane][0] = n0; sm.e_n[lane][1] = n1; sm.e_n[lane][2] = n2;
      double u0 = (double)d0 * g.cinv[0], u1 = (double)d1 * g.cinv[1], u2 = (double)d2 * g.cinv[2];
      sm.e_B[lane][0] = g.R[0] * u0 + g.R[1] * u1 + g.R[2] * u2;
      sm.e_B[lane][1] = g.R[4] * u1 + g.R[5] * u2;
      sm.e_B[lane][2] = g.R[8] * u2;
    }
    if (lane == 0) sm.e_center = 13;  // delta = (0, 0, 0)
    __syncwarp();
    return 27 - g.dbg_drop;  // dbg_drop > 0 only for the negative-control test (nc_debug)
  }
  // DO: lanes 0..11 = (layer dz, row index ri)
  int ncols = 0, c0 = 0, m = 0, n2 = 0, n3 = 0, kd = 0, jd = 0, dz = 0;
  if (lane < 12) {
    dz = lane / 4 - 1;
    int ri = lane % 4;
    int kk = a2 + dz;
    n3 = floordiv(kk, l3);
    kd = kk - n3 * l3;
    double oy = __dmul_rn((double)n3, g.d32);
    int m0 = (int)floor(__dsub_rn((double)(a1 - 1), oy));
    int m1 = (int)ceil(__dsub_rn((double)(a1 + 2), oy));
    if (ri < m1 - m0) {
      m = m0 + ri;
      n2 = floordiv(m, l2);
      jd = m - n2 * l2;
      double ox = __dadd_rn(__dmul_rn((double)n3, g.d31), __dmul_rn((double)n2, g.d21));
      c0 = (int)floor(__dsub_rn((double)(a0 - 1), ox));
      int c1 = (int)ceil(__dsub_rn((double)(a0 + 2), ox));
      ncols = c1 - c0;
    }
  }
  int x = ncols;
#pragma unroll
  for (int o = 1; o < 16; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  int total = __shfl_sync(0xffffffffu, x, 15);
  int off = x - ncols;
  // the center cell: layer dz = 0 (n3 = 0), its middle row m = a1 (n2 = 0, ri = 1, lane 5), middle column
  if (lane == 5) sm.e_center = off + 1;
  for (int t = 0; t < ncols; ++t) {
    int col = c0 + t;
    int n1 = floordiv(col, l1);
    int id = col - n1 * l1;
    int e = off + t;
    sm.e_start[e] = (uint32_t)id + (uint32_t)l1 * ((uint32_t)jd + (uint32_t)l2 * (uint32_t)kd);
    sm.e_n[e][0] = n1; sm.e_n[e][1] = n2; sm.e_n[e][2] = n3;
    sm.e_B[e][0] = (double)(col - a0) * g.w[0] + (double)n1 * g.e[0] + (double)n2 * g.R[1] + (double)n3 * g.R[2];
    sm.e_B[e][1] = (double)(m - a1) * g.w[1] + (double)n2 * g.e[1] + (double)n3 * g.R[5];
    sm.e_B[e][2] = (double)dz * g.w[2] + (double)n3 * g.e[2];
  }
  __syncwarp();
  return total - g.dbg_drop;
}

// Per-lane accumulators: F (lab frame in fp64 mode, rotated in fp32 mode),
// u = sum s6 (s6 - 1), w = sum fr d (x) d; U_i = 2 eps u - cnt u_shift / 2 and
// W_i = w / 2 are formed once at the end (exact algebra of R11/R12).
struct Acc {
  double fx, fy, fz, u, w0, w1, w2, w3, w4, w5;
  uint32_t cnt, nrc;
  uint64_t hs, hx;
};

// canonical fp64 membership test of the pair (i, j, n) (R16): only for the
// pairs whose fp64 r^2 lies within 1e-12 r_c^2 of the cutoff.
template <typename T>
__device__ __noinline__ bool canonical_in(const Geom& g, const typename V4<T>::t* qs, uint32_t i, uint32_t j, int n0,
                                          int n1, int n2) {
  typename V4<T>::t qi = qs[i];
  typename V4<T>::t qj = qs[j];
  double d0 = __dsub_rn(__dadd_rn((double)qj.x, lshift_c(g, 0, n0, n1, n2)), (double)qi.x);
  double d1 = __dsub_rn(__dadd_rn((double)qj.y, lshift_c(g, 1, n0, n1, n2)), (double)qi.y);
  double d2 = __dsub_rn(__dadd_rn((double)qj.z, lshift_c(g, 2, n0, n1, n2)), (double)qi.z);
  double r2 = __dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2));
  return r2 < g.rc2;
}

template <typename T>
struct PairCtx {
  double ux, uy, uz;   // i: fp32 mode = rotated cell-local fp64; fp64 mode = lab position
  T fx, fy, fz;        // i cell-local, filter precision (fp32 mode)
  float m2x, m2y, m2z, uu;  // fp32 filter: -2 u_i and |u_i|^2 (r^2 = (|v|^2 + |u|^2) + v.(-2u))
  uint32_t base_off;   // staging offset of the current chunk (sorted index of a staged element: see sidx_of)
  uint32_t my;         // i sorted index
  T hi;                // fp32 filter bound on r^2 (superset of the pair set)
  double lo64, hi64;   // band on the fp64 r^2 where the canonical test decides
  const typename V4<T>::t* qs;
  const uint32_t* nh;
  const uint32_t* gid;
  uint32_t nh_i;
  PairOut po;          // digest instantiations: optional full pair list
  uint32_t gi;         // gid of i (pair lists)
};

__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  double bb = __dsub_rn(s, a);
  e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}

// d_a = (q_j + L n) - q_i without intermediate rounding (error-free
// transformations; one final rounding): the fp64-mode force displacement.
__device__ __forceinline__ double exact_d(const Geom& g, int a, double qj, double qi, int n0, int n1, int n2) {
  double p0 = __dmul_rn(g.L[3 * a], (double)n0), p1 = __dmul_rn(g.L[3 * a + 1], (double)n1),
         p2 = __dmul_rn(g.L[3 * a + 2], (double)n2);
  double e0 = __fma_rn(g.L[3 * a], (double)n0, -p0), f1 = __fma_rn(g.L[3 * a + 1], (double)n1, -p1),
         f2 = __fma_rn(g.L[3 * a + 2], (double)n2, -p2);
  double s1, c1, s2, c2, s3, c3, s4, c4;
  two_sum(qj, -qi, s1, c1);
  two_sum(s1, p0, s2, c2);
  two_sum(s2, p1, s3, c3);
  two_sum(s3, p2, s4, c4);
  return s4 + (((c1 + c2) + (c3 + c4)) + ((e0 + f1) + f2));
}

// canonical membership r^2 of (i, j, n) (R16)
__device__ __forceinline__ double canonical_r2(const Geom& g, double qj0, double qj1, double qj2, double qi0,
                                               double qi1, double qi2, int n0, int n1, int n2) {
  double d0 = __dsub_rn(__dadd_rn(qj0, lshift_c(g, 0, n0, n1, n2)), qi0);
  double d1 = __dsub_rn(__dadd_rn(qj1, lshift_c(g, 1, n0, n1, n2)), qi1);
  double d2 = __dsub_rn(__dadd_rn(qj2, lshift_c(g, 2, n0, n1, n2)), qi2);
  return __dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2));
}

// image of staged element t relative to particle i: n_cross + nh_j - nh_i (DS: n_cross)
template <typename T>
__device__ __forceinline__ void image_of(const Geom& g, const K3Smem<T>& sm, uint32_t t, uint32_t nh_j, uint32_t nh_i,
                                         int& n0, int& n1, int& n2) {
  int e = sm.sent[t];
  n0 = sm.e_n[e][0]; n1 = sm.e_n[e][1]; n2 = sm.e_n[e][2];
  if (g.variant == 1) {
    n0 += nh_x(nh_j) - nh_x(nh_i);
    n1 += nh_y(nh_j) - nh_y(nh_i);
  }
}

__device__ __forceinline__ double rcp64(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  y = y * (2.0 - x * y);  // Newton: ~2^-23 -> 2^-46
  y = y * (2.0 - x * y);  //         -> full fp64
  return y;
}

// LJ 12-6 pair with energy shift (R11): fr = 24 eps s6 (2 s6 - 1) / r^2.
__device__ __forceinline__ void lj_accumulate(double sig2, double eps24, Acc& acc, double dx, double dy, double dz,
                                              double r2) {
  double ir2 = rcp64(r2);
  double s2 = sig2 * ir2;
  double s6 = s2 * s2 * s2;
  double fr = (eps24 * s6) * (2.0 * s6 - 1.0) * ir2;
  double tx = fr * dx, ty = fr * dy, tz = fr * dz;
  acc.fx -= tx; acc.fy -= ty; acc.fz -= tz;
  acc.u += s6 * s6 - s6;
  acc.w0 += tx * dx; acc.w1 += ty * dy; acc.w2 += tz * dz;
  acc.w3 += tx * dy; acc.w4 += tx * dz; acc.w5 += ty * dz;
  acc.cnt++;
}

template <bool DIGEST>
__device__ __forceinline__ void digest_add(Acc& acc, const uint32_t* gid, uint32_t j, int n0, int n1, int n2,
                                           const PairOut& po, uint32_t gi) {
  if (DIGEST) {
    uint64_t key = (uint64_t)gid[j] | ((uint64_t)(n0 + 8) << 32) | ((uint64_t)(n1 + 8) << 36) |
                   ((uint64_t)(n2 + 8) << 40);
    uint64_t h = mix64(key);
    acc.hs += h;
    acc.hx ^= h;
    if (po.ijn) {
      const unsigned long long k = atomicAdd(po.n, 1ull);
      if ((long long)k < po.cap) {
        int32_t* o = po.ijn + 5 * k;
        o[0] = (int32_t)gi; o[1] = (int32_t)gid[j]; o[2] = n0; o[3] = n1; o[4] = n2;
      }
    }
  }
}

// NC_F64: evaluate ONE queued survivor t of this lane.  The filter already
// applied the canonical membership test (R16); d is formed error-free in the lab
// frame.  (NC_F32 uses filter_chunk_f32 / eval_masks_f32x2 / eval_close_f64.)
template <typename T, bool DIGEST>
__device__ __forceinline__ void eval_one(const Geom& g, const PairCtx<T>& pc, const K3Smem<T>& sm, Acc& acc,
                                         uint32_t t, double sig2, double eps24) {
  static_assert(sizeof(T) == 8, "generic evaluation is the NC_F64 path");
  typename V4<T>::t v = sm.stage[t];
  uint32_t j = w_to_idx(v.w);
  int n0, n1, n2;
  image_of<T>(g, sm, t, sm.s64.nh[t], pc.nh_i, n0, n1, n2);
  double dx = exact_d(g, 0, v.x, pc.ux, n0, n1, n2);
  double dy = exact_d(g, 1, v.y, pc.uy, n0, n1, n2);
  double dz = exact_d(g, 2, v.z, pc.uz, n0, n1, n2);
  double r2 = dx * dx + dy * dy + dz * dz;
  lj_accumulate(sig2, eps24, acc, dx, dy, dz, r2);
  digest_add<DIGEST>(acc, pc.gid, j, n0, n1, n2, pc.po, pc.gi);
}

// Evaluate the queued filter survivors of every lane (warp-uniform loop, two
// independent entries per iteration for instruction-level parallelism).
template <typename T, bool DIGEST>
__device__ __forceinline__ void eval_queue(const Geom& g, const PairCtx<T>& pc, K3Smem<T>& sm, Acc& acc, int qlen,
                                           int lane) {
  int qmax = __reduce_max_sync(0xffffffffu, qlen);
  const double sig2 = g.sig2, eps24 = 24.0 * g.eps;
  for (int k = 0; k < qmax; k += 2) {
    if (k < qlen) eval_one<T, DIGEST>(g, pc, sm, acc, sm.queue[k][lane], sig2, eps24);
    if (k + 1 < qlen) eval_one<T, DIGEST>(g, pc, sm, acc, sm.queue[k + 1][lane], sig2, eps24);
  }
}

// NC_F64 filter step for staged element t: the canonical fp64 membership test (R16).
template <typename T>
__device__ __forceinline__ bool filter_one(const Geom& g, const PairCtx<T>& pc, const K3Smem<T>& sm, uint32_t t) {
  static_assert(sizeof(T) == 8, "generic filter is the NC_F64 path");
  typename V4<T>::t v = sm.stage[t];
  int n0, n1, n2;
  image_of<T>(g, sm, t, sm.s64.nh[t], pc.nh_i, n0, n1, n2);
  double r2 = canonical_r2(g, v.x, v.y, v.z, pc.ux, pc.uy, pc.uz, n0, n1, n2);
  return r2 < g.rc2 && w_to_idx(v.w) != pc.my;
}

__device__ __forceinline__ double shfl_comb(double x, int src, bool take) {
  double y = __shfl_sync(0xffffffffu, x, src);
  return take ? x + y : x;
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Far-away sentinel for padding the staged list (never passes the filter).
template <typename T> __device__ __forceinline__ typename V4<T>::t far4();
template <> __device__ __forceinline__ float4 far4<float>() {
  return make_float4(1e30f, 1e30f, 1e30f, __int_as_float(0x7f800000));  // |v|^2 = +inf
}
template <> __device__ __forceinline__ double4 far4<double>() { return make_double4(1e300, 1e300, 1e300, 0.0); }

// Filter stream s of the staged chunk: t = s, s+S, ... for `iters` steps
// (warp-uniform count; the S sentinels after the chunk make every access
// valid).  Survivors go to this lane's queue; the queue is evaluated when
// any lane could overflow.
template <typename T, bool DIGEST>
__device__ __forceinline__ void filter_chunk(const Geom& g, const PairCtx<T>& pc, K3Smem<T>& sm, Acc& acc, int s,
                                             int S, int iters, int lane) {
  uint32_t t = (uint32_t)s;
  int qlen = 0;
  int it = 0;
  const int main_iters = iters - iters % K3_UNROLL;
  for (; it < main_iters; it += K3_UNROLL) {
#pragma unroll
    for (int k = 0; k < K3_UNROLL; ++k) {
      bool hit = filter_one<T>(g, pc, sm, t);
      sm.queue[qlen][lane] = (K3QT)t;
      qlen += hit ? 1 : 0;
      t += (uint32_t)S;
    }
    if (__any_sync(0xffffffffu, qlen > K3_QCAP - K3_UNROLL)) {
      eval_queue<T, DIGEST>(g, pc, sm, acc, qlen, lane);
      qlen = 0;
    }
  }
  for (; it < iters; ++it) {
    bool hit = filter_one<T>(g, pc, sm, t);
    sm.queue[qlen][lane] = (K3QT)t;
    qlen += hit ? 1 : 0;
    t += (uint32_t)S;
  }
  eval_queue<T, DIGEST>(g, pc, sm, acc, qlen, lane);
}

// ---------------------------------------------------------------------------
// Hot path of NC_F32 (hand-scheduled): fp32 filter with shared-address queues
// (11 instructions per candidate: LDS.128, 6 FP, FSETP + predicated IADD,
// STS, pointer step) and a branch-light fp64 evaluation of two survivors per
// iteration.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds16(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return (uint32_t)v;
}
__device__ __forceinline__ void sts16(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((unsigned short)v) : "memory");
}
// full shared address of a staged element from the low 16 bits kept in a queue
// (the staged array spans < 64 KB, so one possible carry into bit 16)
// The CTA's shared window starts at (cluster rank << 24) + 0x400 on sm_100, so the whole
// K3Smem (< 16 KB) lies inside one 64 KB page and no carry into bit 16 can occur; k_pairs
// checks this once per block (flagged as non-finite, i.e. a loud failure, if it ever breaks).
__device__ __forceinline__ uint32_t addr_from16(uint32_t lo16, uint32_t stage0) {
  return (stage0 & 0xffff0000u) | lo16;
}
__device__ __forceinline__ void stsq(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((unsigned short)v) : "memory");
}
// shared address of a queued staged element
__device__ __forceinline__ uint32_t qaddr(K3QT e, uint32_t stage0) { return addr_from16(e, stage0); }

// fp32 staging is three float arrays (sx, sy, sz): a broadcast LDS.32 is one shared-memory
// wavefront, a 16-byte LDS.128 four (the filter is bound by the shared-memory pipe)
constexpr uint32_t K3_YOFF = 4u * K3_SSTR, K3_ZOFF = 8u * K3_SSTR;  // bytes from the x array to y, z
__device__ __forceinline__ float ldsf(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}

// packed fp32x2 arithmetic (sm_100: FADD2 / FMUL2 / FFMA2, round-to-nearest like the scalar ops)
__device__ __forceinline__ uint64_t pk2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk2(uint64_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

__device__ __forceinline__ uint32_t ldsu(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void stsu(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}


// Close tier: survivors with r < r_split (large forces), in the r_c band, or
// all survivors in digest mode -- fp64 from the fp64 staged coordinates,
// canonical membership inside the 1e-12 band.  Two per iteration.
// sorted particle index of staged element t (entry e = sent[t] of the current chunk)
__device__ __forceinline__ uint32_t sidx_of(const K3Smem<float>& sm, uint32_t t, uint32_t base_off) {
  const int e = sm.sent[t];
  return sm.e_start[e] + t - (sm.e_off[e] - base_off);
}

template <bool DIGEST>
__device__ __forceinline__ void eval_close_f64(const Geom& g, const PairCtx<float>& pc, K3Smem<float>& sm, Acc& acc,
                                               int qlen, int lane, uint32_t stage0, const double4* __restrict__ u64,
                                               K3QT (*queue)[32]) {
  // the two far lanes of a row (lanes 2r, 2r + 1: the same particle i, accumulators combined later
  // in fixed order) split their queued items evenly: lane 2r takes the first ceil(T/2) items of the
  // concatenation (its own queue, then its partner's), lane 2r + 1 the rest
  const int qp = __shfl_xor_sync(0xffffffffu, qlen, 1);
  const int odd = lane & 1, tot2 = qlen + qp, h0 = (tot2 + 1) >> 1;
  const int q0 = odd ? qp : qlen;          // the even lane's own count
  const int myn = odd ? tot2 - h0 : h0;    // items this lane evaluates
  const int gbase = odd ? h0 : 0;
  const int qmax = __reduce_max_sync(0xffffffffu, myn);
  const double sig2 = g.sig2, eps24 = 24.0 * g.eps;
  const uint32_t dummy = stage0 + 4u * K3_DUMMY;
  auto pair2 = [&](uint32_t ta, uint32_t tb, uint32_t ja, uint32_t jb, int ea, int eb, const double4& pa,
                   const double4& pb) {
    const double dxa = (pa.x + sm.e_B[ea][0]) - pc.ux, dya = (pa.y + sm.e_B[ea][1]) - pc.uy,
                 dza = (pa.z + sm.e_B[ea][2]) - pc.uz;
    const double dxb = (pb.x + sm.e_B[eb][0]) - pc.ux, dyb = (pb.y + sm.e_B[eb][1]) - pc.uy,
                 dzb = (pb.z + sm.e_B[eb][2]) - pc.uz;
    const double r2a = dxa * dxa + dya * dya + dza * dza;
    const double r2b = dxb * dxb + dyb * dyb + dzb * dzb;
    bool oka = (ja != pc.my) && (r2a < pc.hi64);
    bool okb = (jb != pc.my) && (r2b < pc.hi64);
    int na0 = 0, na1 = 0, na2 = 0, nb0 = 0, nb1 = 0, nb2 = 0;
    if (DIGEST || (oka && r2a >= pc.lo64) || (okb && r2b >= pc.lo64)) {  // rare: canonical band / digest
      if (oka) {
        image_of<float>(g, sm, ta, g.variant == 1 ? pc.nh[ja] : 0u, pc.nh_i, na0, na1, na2);
        if (r2a >= pc.lo64) { oka = canonical_in<float>(g, pc.qs, pc.my, ja, na0, na1, na2); acc.nrc++; }
      }
      if (okb) {
        image_of<float>(g, sm, tb, g.variant == 1 ? pc.nh[jb] : 0u, pc.nh_i, nb0, nb1, nb2);
        if (r2b >= pc.lo64) { okb = canonical_in<float>(g, pc.qs, pc.my, jb, nb0, nb1, nb2); acc.nrc++; }
      }
    }
    const double ira = rcp64(r2a), irb = rcp64(r2b);
    const double s2a = sig2 * ira, s2b = sig2 * irb;
    const double s6a = s2a * s2a * s2a, s6b = s2b * s2b * s2b;
    double fra = (eps24 * s6a) * (2.0 * s6a - 1.0) * ira;
    double frb = (eps24 * s6b) * (2.0 * s6b - 1.0) * irb;
    fra = oka ? fra : 0.0;
    frb = okb ? frb : 0.0;
    const double txa = fra * dxa, tya = fra * dya, tza = fra * dza;
    const double txb = frb * dxb, tyb = frb * dyb, tzb = frb * dzb;
    acc.fx -= txa + txb; acc.fy -= tya + tyb; acc.fz -= tza + tzb;
    acc.u += (oka ? s6a * s6a - s6a : 0.0) + (okb ? s6b * s6b - s6b : 0.0);
    acc.w0 += txa * dxa + txb * dxb; acc.w1 += tya * dya + tyb * dyb; acc.w2 += tza * dza + tzb * dzb;
    acc.w3 += txa * dya + txb * dyb; acc.w4 += txa * dza + txb * dzb; acc.w5 += tya * dza + tyb * dzb;
    acc.cnt += (oka ? 1u : 0u) + (okb ? 1u : 0u);
    if (DIGEST) {
      if (oka) digest_add<DIGEST>(acc, pc.gid, ja, na0, na1, na2, pc.po, pc.gi);
      if (okb) digest_add<DIGEST>(acc, pc.gid, jb, nb0, nb1, nb2, pc.po, pc.gi);
    }
  };
  // queue entry k of this lane -> staged index t, sorted index j (pc.my + dummy for none), entry e
  auto item = [&](int k, uint32_t& t, uint32_t& j, int& e) {
    const int gk = gbase + k;
    const int src = gk < q0 ? (lane & ~1) : (lane | 1), slot = gk < q0 ? gk : gk - q0;
    const uint32_t a = k < myn ? qaddr(queue[slot][src], stage0) : dummy;
    t = (a - stage0) >> 2;
    j = k < myn ? sidx_of(sm, t, pc.base_off) : pc.my;
    e = sm.sent[t];
  };
  for (int k = 0; k < qmax; k += 2) {
    uint32_t ta, tb, ja, jb;
    int ea, eb;
    item(k, ta, ja, ea); item(k + 1, tb, jb, eb);
    const double4 pa = u64[ja], pb = u64[jb];
    pair2(ta, tb, ja, jb, ea, eb, pa, pb);
  }
}

// (m << 1) | (v >> 31): one funnel shift
__device__ __forceinline__ uint32_t shl_in(uint32_t m, uint32_t v) {
  uint32_t r;
  asm("shf.l.clamp.b32 %0, %1, %2, 1;" : "=r"(r) : "r"(v), "r"(m));
  return r;
}

// ---------------------------------------------------------------------------
// NC_F32 candidate filter on the tensor cores (mma.sync m16n8k4, tf32 operands, fp32 accumulate).
//
// The distance check of a cell's particles i against its staged neighborhood j is a dense
// rank-3 contraction: r^2 = |u_i|^2 + |v_j|^2 - 2 u_i . v_j.  One mma.m16n8k4 takes 16 rows i x 8
// columns j with A row i = (-2u_i, 1), B column j = (v_j, |v_j|^2) and the fp32 accumulator input
// C = |u_i|^2 - h per row, so the SIGN of D is the superset test r~^2 < h.  tf32 keeps 10 mantissa bits (x, y, z truncated, |v|^2 rounded):
// |r~^2 - r^2| <= 2^-10 4.01 |u_i| |v_j| + 2^-11 |v_j|^2 + accumulation rounding, and with cell-centred
// coordinates |u_i| <= R_i (half the cell diagonal) and |v_j| <= R_i + r_c for any pair inside the
// cutoff, so h = r_c^2 + that bound (Geom::f_hmma, host) makes the hit set a SUPERSET of the pair
// set; every hit is re-decided exactly by the fp32 far tier / fp64 close tier (canonical inside the
// 1e-12 band), so the pair set is unchanged.  Lane (g = lane/4, t = lane%4) holds rows g, g+8
// (+16, +24) and columns 8k + 2t + {0, 1}: its hit bits for row r, "MMA stream" t, are packed
// into 32-bit words, bit 31 - (2k' + h) of word w <-> staged element 8 (16 w + k') + 2 t + h.
// ---------------------------------------------------------------------------
// C is a persistent register quad per row group (c[0] = c[1] = row g, c[2] = c[3] = row g + 8):
// distinct registers, so no accumulator copies are needed per mma
__device__ __forceinline__ void mma1684(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t b0, const float (&c)[4]) {
  asm("mma.sync.aligned.m16n8k4.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%7,%8,%9,%10};"
      : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
      : "r"(a0), "r"(a1), "r"(b0), "f"(c[0]), "f"(c[1]), "f"(c[2]), "f"(c[3]));
}

__device__ __forceinline__ float tf32_rna(float x) {  // round to the nearest tf32 (10 mantissa bits)
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// one column block: rows g, g+8 of lane (g, t), columns 8k + 2t + {0, 1}
__device__ __forceinline__ void mma_step(uint32_t b, uint32_t a0, uint32_t a1, const float (&c)[4], uint32_t& m0,
                                         uint32_t& m1) {
  float d[4];
  mma1684(d, a0, a1, b, c);
  m0 = shl_in(m0, __float_as_uint(d[0]));
  m0 = shl_in(m0, __float_as_uint(d[1]));
  m1 = shl_in(m1, __float_as_uint(d[2]));
  m1 = shl_in(m1, __float_as_uint(d[3]));
}

// 2-bit groups of a 16-bit value (group k = bits 15-2k, 14-2k) spread to bits 29-4k, 28-4k
__device__ __forceinline__ uint32_t spread2(uint32_t x) {
  x = (x | (x << 8)) & 0x00FF00FFu;
  x = (x | (x << 4)) & 0x0F0F0F0Fu;
  x = (x | (x << 2)) & 0x33333333u;
  return x;
}

// Filter W words (16 column blocks each; the staged chunk is padded to 128 W elements) into the hit
// words of the far-tier lanes (row, s), two per row: lane (row, s) takes MMA streams s and s + 2 of
// its row, interleaved in 2-bit groups (one shuffle with the partner lane t ^ 2, which holds the other
// stream of the same rows): word w2 at hw[(row 2 + s) 2W + w2], bit c = 2q + h <-> staged element
// 64 w2 + 4 q + 2 s + h -- a lane's words cover its elements in order with a uniform stride (pop_hit).
__device__ __forceinline__ void mma_filter(uint32_t stage0, uint32_t hw0, int W, uint32_t a0, uint32_t a1,
                                           const float (&c)[4], int lane) {
  const int g = lane >> 2, t = lane & 3;
  const uint32_t bb = stage0 + 4u * ((uint32_t)t * K3_SSTR + (uint32_t)g);  // component t of element 8k + g
  const bool lo = t < 2;  // lane t < 2 builds row g's words (streams t, t + 2), lane t >= 2 row g + 8's
  const uint32_t o0 = hw0 + 4u * (uint32_t)(((lo ? g : g + 8) * 2 + (t & 1)) * 2 * W);
#pragma unroll 1
  for (int w = 0; w < W; ++w) {
    uint32_t m0 = 0u, m1 = 0u;
    const uint32_t bw = bb + 512u * (uint32_t)w;
    uint32_t b[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) b[k] = ldsu(bw + 32u * k);  // all loads of the word first
#pragma unroll
    for (int k = 0; k < 16; ++k) mma_step(b[k], a0, a1, c, m0, m1);
    const uint32_t x = __shfl_xor_sync(0xffffffffu, lo ? m1 : m0, 2);
    const uint32_t ma = lo ? m0 : x, mb = lo ? x : m1;  // streams s = t & 1 and s + 2
    // stored bit-reversed (bit p = 31 - c): pop_hit takes the highest set bit p without a 31 - x
    stsu(o0 + 8u * (uint32_t)w, __brev((spread2(ma >> 16) << 2) | spread2(mb >> 16)));               // blocks 0-7
    stsu(o0 + 8u * (uint32_t)w + 4u, __brev((spread2(ma & 0xffffu) << 2) | spread2(mb & 0xffffu)));  // blocks 8-15
  }
}

// Hit cursor over one far lane's words (mma_filter's layout, stored bit-reversed): bit position c = 2q + h
// of the current word is the staged element at address wa + 16 q + 4 h = wa + 4 c + 8 (c >> 1); pop the
// highest hit and refill the word when it empties (predicated: next word +4 bytes, element base +64).
struct HitCur {
  uint32_t cur, wa, wq, wend;
};
__device__ __forceinline__ uint32_t pop_hit(HitCur& h, bool& valid) {
  // words are stored bit-reversed, so bit POSITION p is element index c = p: the highest set bit
  // (bfind, no 31 - x) is the element at wa + 4p + 8(p >> 1)
  valid = h.cur != 0;
  uint32_t p, m;
  asm("bfind.u32 %0, %1;" : "=r"(p) : "r"(h.cur));           // highest set bit (0xffffffff if none)
  asm("shl.b32 %0, %1, %2;" : "=r"(m) : "r"(1u), "r"(p));     // shifts >= 32 give 0: nothing to clear
  h.cur ^= m;
  const uint32_t pp = valid ? p : 0u;  // idle lanes read their word's first element: finite, masked
  const uint32_t a = h.wa + 4u * pp + 8u * (pp >> 1);
  if (h.cur == 0 && h.wq < h.wend) {
    h.cur = ldsu(h.wq);
    h.wq += 4u;
    h.wa += 256u;
  }
  return a;
}

// Far tier straight from the hit words, two hits per iteration on packed fp32x2 (FADD2/FMUL2/FFMA2)
// with packed partial sums folded into the fp64 Acc once per chunk.  Each hit is re-decided from the
// staged fp32 coordinates: r_split^2 <= r^2 < r_c^2 (1 - 1e-4) is a far pair (fp32 force math);
// everything else (r < r_split, the cutoff band, the MMA filter's margin beyond it) is compacted into
// the close queue, which is handed to the fp64 tier (canonical membership inside the 1e-12 band, no
// pair beyond r_c) whenever some lane's queue is nearly full, and at the end.  Digest mode keeps
// exactly this split (the timed kernel's membership decisions) and adds every far pair's key.
template <bool DIGEST>
__device__ __forceinline__ void eval_hits(const Geom& g, const PairCtx<float>& pc, K3Smem<float>& sm, Acc& acc,
                                          uint32_t& nfar, uint32_t wl0, int nwords, uint32_t wa0, int lane,
                                          uint32_t stage0, const double4* __restrict__ u64) {
  int nhit = 0, qits = 0;  // this lane's hits and empty words (an empty word costs one idle pop)
  for (int k = 0; k < nwords; ++k) {
    const int c = __popc(ldsu(wl0 + 4u * k));
    nhit += c;
    qits += c ? c : 1;
  }
  HitCur h;
  h.cur = ldsu(wl0);
  h.wa = wa0;
  h.wq = wl0 + 4u;
  h.wend = wl0 + 4u * (uint32_t)nwords;
  const int qmax = (__reduce_max_sync(0xffffffffu, qits) + 1) >> 1;  // two hits per iteration
  const float split2 = g.f_split2, lo32 = g.f_lo;
  const uint64_t nfx = pk2(-pc.fx, -pc.fx), nfy = pk2(-pc.fy, -pc.fy), nfz = pk2(-pc.fz, -pc.fz);
  const uint64_t SIG2 = pk2(g.f_sig2, g.f_sig2), C48 = pk2(g.f_c48, g.f_c48), M24 = pk2(g.f_m24, g.f_m24),
                 NEG1 = pk2(-1.0f, -1.0f);
  const uint32_t qc0 = smem_u32(&sm.queue[0][lane]), qclim = qc0 + K3_QSTRIDE * (K3_CQ - 8);
  uint32_t qc = qc0;
  int nclose_all = 0;
  uint64_t Fx = 0, Fy = 0, Fz = 0, Uq = 0, W0 = 0, W1 = 0, W2 = 0, W3 = 0, W4 = 0, W5 = 0;  // packed partial sums
  // far iterations until some lane's close queue nears capacity (checked every 4 iterations = 8 hits)
  // or the hits run out, then the fp64 tier on the queued items: one inlined copy of each tier
  int k = 0;
  while (true) {
    bool flush = false;
    for (; k < qmax; ++k) {
      bool va, vb;
      const uint32_t aa = pop_hit(h, va);
      const uint32_t ab = pop_hit(h, vb);
      const uint64_t DX = add2(pk2(ldsf(aa), ldsf(ab)), nfx), DY = add2(pk2(ldsf(aa + K3_YOFF), ldsf(ab + K3_YOFF)), nfy),
                     DZ = add2(pk2(ldsf(aa + K3_ZOFF), ldsf(ab + K3_ZOFF)), nfz);
      float r2a, r2b;
      upk2(fma2(DZ, DZ, fma2(DY, DY, mul2(DX, DX))), r2a, r2b);
      // far: r_split <= r and r^2 < r_c^2 (1 - 1e-4); everything else -- close pairs, the cutoff band and
      // the MMA margin beyond it (the fp64 tier rejects those) -- goes to the close queue
      const bool fa = r2a >= split2 && r2a < lo32, fb = r2b >= split2 && r2b < lo32;
      const bool qa = va && !fa, qb = vb && !fb;  // predicated stores: no wavefront otherwise
      NC_CHECK(!qa || qc < qc0 + K3_QSTRIDE * K3_CQ);
      if (qa) stsq(qc, aa);
      qc += qa ? K3_QSTRIDE : 0u;
      NC_CHECK(!qb || qc < qc0 + K3_QSTRIDE * K3_CQ);
      if (qb) stsq(qc, ab);
      qc += qb ? K3_QSTRIDE : 0u;
      float ia, ib;
      asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(ia) : "f"(r2a));
      asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(ib) : "f"(r2b));
      const uint64_t IR = pk2((va && fa) ? ia : 0.0f, (vb && fb) ? ib : 0.0f);  // one mask per pair
      const uint64_t S2 = mul2(SIG2, IR);
      const uint64_t S6 = mul2(mul2(S2, S2), S2);
      const uint64_t FR = mul2(mul2(fma2(C48, S6, M24), S6), IR);  // (48 eps s6 - 24 eps) s6 / r^2
      const uint64_t TX = mul2(FR, DX), TY = mul2(FR, DY), TZ = mul2(FR, DZ);
      Fx = add2(Fx, TX); Fy = add2(Fy, TY); Fz = add2(Fz, TZ);
      Uq = fma2(S6, add2(S6, NEG1), Uq);
      W0 = fma2(TX, DX, W0); W1 = fma2(TY, DY, W1); W2 = fma2(TZ, DZ, W2);
      W3 = fma2(TX, DY, W3); W4 = fma2(TX, DZ, W4); W5 = fma2(TY, DZ, W5);
      if (DIGEST) {  // far pairs' keys (the close tier adds its own)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          if (hh == 0 ? (va && fa) : (vb && fb)) {
            const uint32_t t = ((hh == 0 ? aa : ab) - stage0) >> 2;
            const uint32_t j = sidx_of(sm, t, pc.base_off);
            int n0, n1, n2;
            image_of<float>(g, sm, t, g.variant == 1 ? pc.nh[j] : 0u, pc.nh_i, n0, n1, n2);
            digest_add<DIGEST>(acc, pc.gid, j, n0, n1, n2, pc.po, pc.gi);
          }
        }
      }
      if ((k & 3) == 3 && __any_sync(0xffffffffu, qc > qclim)) {
        flush = true;
        ++k;
        break;
      }
    }
    __syncwarp();
    const int nclose = (int)((qc - qc0) / K3_QSTRIDE);
    nclose_all += nclose;
    eval_close_f64<DIGEST>(g, pc, sm, acc, nclose, lane, stage0, u64, sm.queue);
    __syncwarp();
    qc = qc0;
    if (!flush) break;
  }
  auto fold = [](uint64_t v) { float a, b; upk2(v, a, b); return (double)a + (double)b; };
  acc.fx -= fold(Fx); acc.fy -= fold(Fy); acc.fz -= fold(Fz); acc.u += fold(Uq);
  acc.w0 += fold(W0); acc.w1 += fold(W1); acc.w2 += fold(W2);
  acc.w3 += fold(W3); acc.w4 += fold(W4); acc.w5 += fold(W5);
  const int nf = nhit - nclose_all;  // every hit is far or went to the fp64 tier
  acc.cnt += (uint32_t)nf;
  nfar += (uint32_t)nf;  // this lane's fp32-tier count (roofline accounting)
}

__device__ __forceinline__ uint64_t lds64(uint32_t a) {
  uint64_t v;
  asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}

// Staging offsets of the entries of one chunk [e0, e1) of the neighborhood (<= K3_CAP elements);
// returns e1 (warp-uniform).  A single entry above K3_CAP (a cell of more than K3_CAP particles)
// returns e0: the caller flags it (NC_E_OOM on the host) and skips the entry.
template <typename SM>
__device__ __forceinline__ int chunk_end(const SM& sm, int e0, int nst, int lane) {
  const uint32_t base_off = sm.e_off[e0];
  int e1 = e0;
  for (int eb = e0; eb < nst; eb += 32) {
    const int e = eb + lane;
    const bool fits = e < nst && (sm.e_off[e] + sm.e_cnt[e] - base_off) <= (uint32_t)K3_CAP;
    const int nfit = __popc(__ballot_sync(0xffffffffu, fits));  // the fitting entries are a prefix
    e1 = eb + nfit;
    if (nfit < 32) break;
  }
  return e1;
}
constexpr double K3_OVERFLOW = 1048576.0;  // tNF marker of a cell above K3_CAP particles (host: NC_E_OOM)

// Stream combine of a lane group: rows are S consecutive lanes, fixed binary tree over s.
__device__ __forceinline__ void combine_streams(Acc& acc, int S, int s, bool act, int lane) {
  for (int o = 1; o < S; o <<= 1) {
    const bool take = act && ((s & (2 * o - 1)) == 0);
    const int src = lane ^ o;
    acc.fx = shfl_comb(acc.fx, src, take); acc.fy = shfl_comb(acc.fy, src, take);
    acc.fz = shfl_comb(acc.fz, src, take); acc.u = shfl_comb(acc.u, src, take);
    acc.w0 = shfl_comb(acc.w0, src, take); acc.w1 = shfl_comb(acc.w1, src, take);
    acc.w2 = shfl_comb(acc.w2, src, take); acc.w3 = shfl_comb(acc.w3, src, take);
    acc.w4 = shfl_comb(acc.w4, src, take); acc.w5 = shfl_comb(acc.w5, src, take);
    const uint32_t c2 = __shfl_sync(0xffffffffu, acc.cnt, src);
    const uint32_t r2c = __shfl_sync(0xffffffffu, acc.nrc, src);
    const uint64_t h1 = __shfl_sync(0xffffffffu, acc.hs, src);
    const uint64_t h2 = __shfl_sync(0xffffffffu, acc.hx, src);
    if (take) { acc.cnt += c2; acc.nrc += r2c; acc.hs += h1; acc.hx ^= h2; }
  }
}

// One warp per block; each warp handles K3_CELLS consecutive cells of one
// cell layer, so block partials are layer-aligned and their fixed-order sums
// are independent of timing (determinism).  grid = l3 * blocks_per_layer.
template <typename T, bool DIGEST, bool COUNT = false>
#if K3_MAXNREG
__global__ void __maxnreg__(K3_MAXNREG)
#else
__global__ void __launch_bounds__(32, K3_MINB)
#endif
k_pairs(const double4* __restrict__ u, const float4* __restrict__ u32, const uint32_t* __restrict__ cs,
        const typename V4<T>::t* __restrict__ qs, const uint32_t* __restrict__ nh, const uint32_t* __restrict__ gid,
        typename V4<T>::t* __restrict__ Fout, double* __restrict__ bpart, uint32_t* __restrict__ dcnt,
        uint64_t* __restrict__ dhs, uint64_t* __restrict__ dhx, const __grid_constant__ Geom g, int cpb, int bpl,
        int layer0, const PairOut po) {
  PDL_WAIT();  // (the successor is released at the end: PDL_LAUNCH below)
  extern __shared__ __align__(16) unsigned char smraw[];
  const int lane = threadIdx.x & 31;
  K3Smem<T>& sm = *reinterpret_cast<K3Smem<T>*>(smraw);

  const int l1 = g.dims[0], l2 = g.dims[1];
  const int layer = layer0 + (int)(blockIdx.x / bpl);  // global cell layer (slab mode: owned layers only)
  const int chunk = (int)blockIdx.x - (layer - layer0) * bpl;
  const int per_layer = l1 * l2;
  // cpb < 0 (NC_F64 on small grids): -cpb blocks share one cell, block `sub` taking its i-batches
  // sub, sub + nsplit, ... of K3_F64_SPLIT_B particles -- more warps in flight when the grid has few cells
  const int nsplit = cpb < 0 ? -cpb : 1, sub = cpb < 0 ? chunk % nsplit : 0;
  const int cbeg = cpb < 0 ? chunk / nsplit : chunk * cpb;
  const int cend = cpb < 0 ? cbeg + 1 : min(per_layer, cbeg + cpb);

  PairCtx<T> pc;
  pc.hi = (T)g.band_hi;
  pc.lo64 = g.rc2 * (1.0 - K3_BAND64);
  pc.hi64 = g.rc2 * (1.0 + K3_BAND64);
  pc.qs = qs;
  pc.nh = nh;
  pc.gid = gid;
  pc.po = po;
  pc.gi = 0u;

  double tU = 0, tW[6] = {0, 0, 0, 0, 0, 0}, tI = 0, tC = 0, tS = 0, tR = 0, tNF = 0;
  uint32_t tFu = 0;  // this lane's fp32-tier interactions (< 2^32 per lane)
  if constexpr (sizeof(T) == 4) {
    // 16-bit queue entries decode without a carry only if the block's shared memory sits in one 64 KB page
    if ((smem_u32(smraw) & 0xffffu) + (uint32_t)sizeof(K3Smem<T>) > 0x10000u) tNF += 1.0;
    if (lane == 0) {  // permanent far element used to pad the two-wide close evaluation (far bracket)
      sm.s64.sc[0][K3_DUMMY] = sm.s64.sc[1][K3_DUMMY] = sm.s64.sc[2][K3_DUMMY] = 1e30f;
      sm.sent[K3_DUMMY] = K3_MAXE - 1;
      sm.e_B[K3_MAXE - 1][0] = 1e150; sm.e_B[K3_MAXE - 1][1] = 1e150; sm.e_B[K3_MAXE - 1][2] = 1e150;
    }
    __syncwarp();
  }

  for (int cl = cbeg; cl < cend; ++cl) {
    const int a0 = cl % l1, a1 = cl / l1, a2 = layer;
    const uint32_t cid = (uint32_t)cl + (uint32_t)per_layer * (uint32_t)layer;
    const int nst = build_entries(g, a0, a1, a2, sm, lane);
    // entry sizes and staging offsets (exclusive scan over <= 36 entries)
    uint32_t tot = 0;
    for (int e0 = 0; e0 < nst; e0 += 32) {
      int e = e0 + lane;
      uint32_t cnt = 0, st = 0;
      if (e < nst) {
        uint32_t cell = sm.e_start[e];
        st = cs[cell];
        cnt = cs[cell + 1] - st;
      }
      uint32_t x = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      __syncwarp();
      if (e < nst) {
        sm.e_start[e] = st;
        sm.e_cnt[e] = cnt;
        sm.e_off[e] = tot + x - cnt;
      }
      tot += __shfl_sync(0xffffffffu, x, 31);
    }
    __syncwarp();
    if (sub == 0) tS += (double)nst;  // cell-level statistics once per cell
    const uint32_t ibase = cs[cid];
    const int ni = (int)(cs[cid + 1] - ibase);
    if (ni == 0) continue;
    if (sub == 0) tC += (double)ni * (double)tot - (double)ni;

    if constexpr (sizeof(T) == 4) {
      // ---------------- NC_F32: tensor-core filter, packed fp32 far tier, fp64 close tier
      const uint32_t stage0 = smem_u32(&sm.s64.sc[0][0]);
      const uint32_t hw0 = smem_u32(&sm.hw[0]);
      const int g8 = lane >> 2, t4 = lane & 3;
      int staged0 = -1, staged1 = -1;  // entries currently staged (reused by the next i-batch)
      for (int ib = 0; ib < ni; ib += 16) {
        const int nb = min(16, ni - ib);
        constexpr int S = 2;  // far-tier lanes per row (mma_filter's interleaved word layout)
        const int row = lane / S, s = lane % S;
        const bool act = row < nb;
        pc.my = ibase + ib + (act ? row : 0);
        const double4 ui = u[pc.my];  // fp64 i (close tier); consumed after staging: its latency overlaps
        pc.ux = ui.x; pc.uy = ui.y; pc.uz = ui.z;
        pc.nh_i = (g.variant == 1) ? nh[pc.my] : 0u;
        if (DIGEST) pc.gi = gid[pc.my];
        // MMA A fragments (rows g8, g8 + 8: component t4 of (-2 u, 1)), C = |u|^2 - h per row, and the
        // far lanes' fp32 i: from the staged center cell (set with the first chunk that holds it)
        uint32_t a0 = 0u, a1 = 0u;
        float c[4];
        bool have_a = false;
        Acc acc = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0u, 0u, 0ull, 0ull};

        int e0 = 0;
        while (e0 < nst) {
          const uint32_t base_off = sm.e_off[e0];
          const int e1 = chunk_end(sm, e0, nst, lane);
          if (e1 == e0) {  // one cell above K3_CAP particles: cannot stage it (host reports NC_E_OOM)
            tNF += (lane == 0 && ib == 0) ? K3_OVERFLOW : 0.0;
            e0 += 1;
            continue;
          }
          const uint32_t ctot = (e1 < nst ? sm.e_off[e1] : tot) - base_off;
          NC_CHECK(ctot <= (uint32_t)K3_CAP);
          const int W = (int)((ctot + 127) / 128);  // hit words: 16 column blocks of 8 elements each
          NC_CHECK(128 * W <= K3_DUMMY && 2 * W <= K3_MW);
          // (a vote: the compiler then knows the branch is warp-uniform and keeps the shuffles of the
          // rest of the kernel free of divergence handling)
          if (__any_sync(0xffffffffu, e0 != staged0 || e1 != staged1)) {
            // stage: element t <- particle e_start[e] + (t - e_off[e]) of entry e, plus the entry's image
            // bracket relative to the center cell's centre (coalesced over t); |v|^2 for the MMA filter
            for (int eb = e0; eb < e1; eb += 32) {
              const int e = eb + lane;
              if (e < e1) {
                const uint32_t dst = sm.e_off[e] - base_off, cnt = sm.e_cnt[e];
                for (uint32_t k = 0; k < cnt; ++k) sm.sent[dst + k] = (uint8_t)e;
                sm.Bf[e][0] = (float)(sm.e_B[e][0] - g.cc[0]);
                sm.Bf[e][1] = (float)(sm.e_B[e][1] - g.cc[1]);
                sm.Bf[e][2] = (float)(sm.e_B[e][2] - g.cc[2]);
              }
            }
            __syncwarp();
            for (uint32_t t0 = 0; t0 < ctot; t0 += 32 * K3_STGR) {
              uint32_t tt[K3_STGR], jj[K3_STGR];
              int ee[K3_STGR];
              float4 pp[K3_STGR];
#pragma unroll
              for (int r = 0; r < K3_STGR; ++r) {
                tt[r] = t0 + 32u * r + lane;
                const bool v = tt[r] < ctot;
                ee[r] = v ? sm.sent[tt[r]] : e0;
                jj[r] = sm.e_start[ee[r]] + tt[r] - (sm.e_off[ee[r]] - base_off);
                pp[r] = v ? u32[jj[r]] : make_float4(0.f, 0.f, 0.f, 0.f);
#if K3_PF_L2
                // the fp64 coordinates the close tier may gather later: start moving them into L2 now
                if (v) asm volatile("prefetch.global.L2 [%0];" ::"l"(u + jj[r]));
#endif
              }
#pragma unroll
              for (int r = 0; r < K3_STGR; ++r) {
                if (tt[r] < ctot) {
                  const float x = pp[r].x + sm.Bf[ee[r]][0], y = pp[r].y + sm.Bf[ee[r]][1],
                              z = pp[r].z + sm.Bf[ee[r]][2];
                  sm.s64.sc[0][tt[r]] = x;
                  sm.s64.sc[1][tt[r]] = y;
                  sm.s64.sc[2][tt[r]] = z;
                  sm.s64.sc[3][tt[r]] = tf32_rna(fmaf(z, z, fmaf(y, y, x * x)));
                }
              }
            }
            for (int t = (int)ctot + lane; t < 128 * W; t += 32) {  // pad to whole words: never a hit
              sm.s64.sc[0][t] = sm.s64.sc[1][t] = sm.s64.sc[2][t] = 0.0f;
              sm.s64.sc[3][t] = 1e30f;
            }
            staged0 = e0;
            staged1 = e1;
          }
          __syncwarp();
          if (!have_a) {
            const int ec = sm.e_center;
            // a vote: warp-uniform for the compiler (the shuffles after it need no divergence handling)
            const bool in_chunk = __any_sync(0xffffffffu, ec >= e0 && ec < e1);
            const uint32_t ci0 = in_chunk ? sm.e_off[ec] - base_off + (uint32_t)ib : 0u;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int r = g8 + 8 * q;
              uint32_t av = 0u;
              float cr = 1e30f;  // ghost rows: never a hit
              if (r < nb) {
                float x, y, z;
                if (in_chunk) {  // staged = u32 + (0 - cc) rounded: the same value as below
                  x = sm.s64.sc[0][ci0 + r]; y = sm.s64.sc[1][ci0 + r]; z = sm.s64.sc[2][ci0 + r];
                } else {
                  const float4 v = u32[ibase + ib + r];
                  x = v.x - g.f_cc[0]; y = v.y - g.f_cc[1]; z = v.z - g.f_cc[2];
                }
                const float comp = t4 == 0 ? x : (t4 == 1 ? y : z);
                av = __float_as_uint(t4 < 3 ? -2.0f * comp : 1.0f);
                cr = fmaf(z, z, fmaf(y, y, x * x)) - g.f_hmma;
              }
              if (q == 0) a0 = av; else a1 = av;
              c[2 * q] = cr;
              c[2 * q + 1] = cr;
            }
            if (in_chunk) {
              const uint32_t ti = ci0 + (uint32_t)(act ? row : 0);
              pc.fx = sm.s64.sc[0][ti]; pc.fy = sm.s64.sc[1][ti]; pc.fz = sm.s64.sc[2][ti];
            } else {
              pc.fx = (float)(ui.x - g.cc[0]); pc.fy = (float)(ui.y - g.cc[1]); pc.fz = (float)(ui.z - g.cc[2]);
            }
            have_a = true;
          }
          mma_filter(stage0, hw0, W, a0, a1, c, lane);
          __syncwarp();
          pc.base_off = base_off;
          const int nw = 2 * W;  // words per far lane
          eval_hits<DIGEST>(g, pc, sm, acc, tFu, hw0 + 4u * (uint32_t)((row * S + s) * nw), nw,
                            stage0 + 8u * (uint32_t)s, lane, stage0, u);
          __syncwarp();
          e0 = e1;
        }
        combine_streams(acc, S, s, act, lane);
        const bool owner = act && s == 0;
        // fold the factors of R11/R12: U_i = 2 eps sum s6(s6-1) - cnt u_shift / 2; W_i = sum fr d d / 2
        const double Ui = 2.0 * g.eps * acc.u - 0.5 * g.ushift * (double)acc.cnt;
        if (owner) {  // lab-frame force F = Q F_rot; .w = the particle's interaction count (parity)
          const double Fx = g.Q[0] * acc.fx + g.Q[1] * acc.fy + g.Q[2] * acc.fz;
          const double Fy = g.Q[3] * acc.fx + g.Q[4] * acc.fy + g.Q[5] * acc.fz;
          const double Fz = g.Q[6] * acc.fx + g.Q[7] * acc.fy + g.Q[8] * acc.fz;
          const typename V4<T>::t fv = mk4((T)Fx, (T)Fy, (T)Fz, idx_to_w(acc.cnt, T()));
          Fout[pc.my] = fv;
          store_user_F(pc.po, gid, pc.my, fv);
          if (DIGEST) { dcnt[pc.my] = acc.cnt; dhs[pc.my] = acc.hs; dhx[pc.my] = acc.hx; }
          tU += Ui;
          tW[0] += 0.5 * acc.w0; tW[1] += 0.5 * acc.w1; tW[2] += 0.5 * acc.w2;
          tW[3] += 0.5 * acc.w3; tW[4] += 0.5 * acc.w4; tW[5] += 0.5 * acc.w5;
          tI += (double)acc.cnt;
          tR += (double)acc.nrc;
        }
        const double fchk = owner ? acc.fx + acc.fy + acc.fz + Ui : 0.0;
        tNF += isfinite(fchk) ? 0.0 : 1.0;
      }
    } else {
      // ---------------- NC_F64: canonical fp64 filter on every candidate, error-free d
      const int fb = nsplit > 1 ? K3_F64_SPLIT_B : 32;  // particles per i-batch
      for (int ib = sub * fb; ib < ni; ib += nsplit * fb) {
        const int nb = min(fb, ni - ib);
        const int S = 32 / nb;               // streams over the j list
        const int il = lane % nb;
        const bool act = lane < S * nb;
        const int s = act ? lane / nb : 0;   // ghost lanes shadow stream 0 (no extra smem addresses)
        pc.my = ibase + ib + il;
        {
          typename V4<T>::t qi = qs[pc.my];
          pc.ux = act ? qi.x : -1e300; pc.uy = qi.y; pc.uz = qi.z;
        }
        pc.nh_i = (g.variant == 1) ? nh[pc.my] : 0u;
        if (DIGEST) pc.gi = gid[pc.my];
        Acc acc = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0u, 0u, 0ull, 0ull};
        int e0 = 0;
        while (e0 < nst) {
          const uint32_t base_off = sm.e_off[e0];
          const int e1 = chunk_end(sm, e0, nst, lane);
          if (e1 == e0) {
            tNF += (lane == 0) ? K3_OVERFLOW : 0.0;
            e0 += 1;
            continue;
          }
          const uint32_t ctot = (e1 < nst ? sm.e_off[e1] : tot) - base_off;
          for (int eb = e0; eb < e1; eb += 32) {
            int e = eb + lane;
            uint32_t cnt = 0, st = 0, dst = 0;
            if (e < e1) { cnt = sm.e_cnt[e]; st = sm.e_start[e]; dst = sm.e_off[e] - base_off; }
            uint32_t cmax = __reduce_max_sync(0xffffffffu, cnt);
            for (uint32_t k = 0; k < cmax; ++k) {
              if (k < cnt) {
                typename V4<T>::t v = qs[st + k];
                sm.stage[dst + k] = mk4(v.x, v.y, v.z, idx_to_w(st + k, T()));
                sm.s64.nh[dst + k] = g.variant == 1 ? nh[st + k] : 0u;
                sm.sent[dst + k] = (uint8_t)e;
              }
            }
          }
          for (int t = lane; t < S; t += 32) {  // far sentinels after the chunk (one per stream)
            sm.stage[ctot + t] = far4<T>();
            sm.s64.nh[ctot + t] = 0u;
            sm.sent[ctot + t] = 0;
          }
          __syncwarp();
          const int iters = (int)((ctot + S - 1) / S);
          pc.base_off = base_off;
          filter_chunk<T, DIGEST>(g, pc, sm, acc, s, S, iters, lane);
          __syncwarp();
          e0 = e1;
        }
        // combine the S streams of each i: fixed binary tree over s (log2 S shuffle steps)
        for (int o = 1; o < S; o <<= 1) {
          const int src_s = s + o;
          bool take = act && ((s & (2 * o - 1)) == 0) && (src_s < S);
          const int src = (lane + o * nb) & 31;
          acc.fx = shfl_comb(acc.fx, src, take); acc.fy = shfl_comb(acc.fy, src, take);
          acc.fz = shfl_comb(acc.fz, src, take); acc.u = shfl_comb(acc.u, src, take);
          acc.w0 = shfl_comb(acc.w0, src, take); acc.w1 = shfl_comb(acc.w1, src, take);
          acc.w2 = shfl_comb(acc.w2, src, take); acc.w3 = shfl_comb(acc.w3, src, take);
          acc.w4 = shfl_comb(acc.w4, src, take); acc.w5 = shfl_comb(acc.w5, src, take);
          uint32_t c2 = __shfl_sync(0xffffffffu, acc.cnt, src);
          uint32_t r2c = __shfl_sync(0xffffffffu, acc.nrc, src);
          if (take) { acc.cnt += c2; acc.nrc += r2c; }
          if (DIGEST) {
            uint64_t h1 = __shfl_sync(0xffffffffu, acc.hs, src);
            uint64_t h2 = __shfl_sync(0xffffffffu, acc.hx, src);
            if (take) { acc.hs += h1; acc.hx ^= h2; }
          }
        }
        const bool owner = (lane < nb);
        const double Ui = 2.0 * g.eps * acc.u - 0.5 * g.ushift * (double)acc.cnt;
        if (owner) {
          const typename V4<T>::t fv = mk4((T)acc.fx, (T)acc.fy, (T)acc.fz, idx_to_w(acc.cnt, T()));
          Fout[pc.my] = fv;
          store_user_F(pc.po, gid, pc.my, fv);
          if (DIGEST) { dcnt[pc.my] = acc.cnt; dhs[pc.my] = acc.hs; dhx[pc.my] = acc.hx; }
          tU += Ui;
          tW[0] += 0.5 * acc.w0; tW[1] += 0.5 * acc.w1; tW[2] += 0.5 * acc.w2;
          tW[3] += 0.5 * acc.w3; tW[4] += 0.5 * acc.w4; tW[5] += 0.5 * acc.w5;
          tI += (double)acc.cnt;
          tR += (double)acc.nrc;
        }
        const double fchk = owner ? acc.fx + acc.fy + acc.fz + Ui : 0.0;
        tNF += isfinite(fchk) ? 0.0 : 1.0;
      }
    }
  }
  tU = warp_sum_d(tU);
  tW[0] = warp_sum_d(tW[0]); tW[1] = warp_sum_d(tW[1]); tW[2] = warp_sum_d(tW[2]);
  tW[3] = warp_sum_d(tW[3]); tW[4] = warp_sum_d(tW[4]); tW[5] = warp_sum_d(tW[5]);
  tI = warp_sum_d(tI);
  tR = warp_sum_d(tR);
  // fp32-tier interactions only in the counting instantiation (nc_profile mode 3): the counter's
  // register costs the hot kernel ~1%
  const double tF = COUNT ? warp_sum_d((double)tFu) : 0.0;
  tNF = warp_sum_d(tNF);
  if (lane < NPART) {
    double v = 0;
    if (lane == 0) v = tU;
    else if (lane == 1) v = tW[0];
    else if (lane == 2) v = tW[1];
    else if (lane == 3) v = tW[2];
    else if (lane == 4) v = tW[3];
    else if (lane == 5) v = tW[4];
    else if (lane == 6) v = tW[5];
    else if (lane == 7) v = tI;
    else if (lane == 8) v = tC;
    else if (lane == 9) v = tS;
    else if (lane == 10) v = tR;
    else if (lane == 11) v = tF;
    else v = tNF;
    bpart[(int64_t)blockIdx.x * NPART + lane] = v;
  }
  PDL_LAUNCH();
}

// K3r: per-layer partials (one block per layer: each thread sums a fixed
// strided subset of the layer's block partials in order, then a fixed-shape
// tree), then the total in layer order.  Deterministic and layer-aligned, so
// identical for any assignment of layers to devices.
constexpr int K3R_T = 256;
// One launch: block l sums layer l's block partials (thread t takes blocks t, t+256, ... in order;
// a fixed warp-shuffle tree, then the 8 warp sums in order), all NPART components at once; the last
// block to finish (device-scope counter) sums the layers in layer order into tot and acc (acc[NPART]
// counts evaluations) and re-arms the counter.  Deterministic: no order depends on timing.
__global__ void __launch_bounds__(K3R_T) k_reduce(const double* __restrict__ bpart, int bpl, int nlayers,
                                                  double* __restrict__ lpart, double* __restrict__ tot,
                                                  double* __restrict__ acc, unsigned int* __restrict__ counter) {
  PDL_ENTRY();
  __shared__ double wred[K3R_T / 32][NPART];
  __shared__ bool last;
  const int layer = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const double* base = bpart + (int64_t)layer * bpl * NPART;
  double v[NPART];
#pragma unroll
  for (int c = 0; c < NPART; ++c) v[c] = 0.0;
  for (int b = tid; b < bpl; b += K3R_T)
#pragma unroll
    for (int c = 0; c < NPART; ++c) v[c] += base[(int64_t)b * NPART + c];
#pragma unroll
  for (int c = 0; c < NPART; ++c) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[c] += __shfl_xor_sync(0xffffffffu, v[c], o);
  }
  if (lane == 0)
#pragma unroll
    for (int c = 0; c < NPART; ++c) wred[wid][c] = v[c];
  __syncthreads();
  if (tid < NPART) {
    double s = 0.0;
    for (int w = 0; w < K3R_T / 32; ++w) s += wred[w][tid];
    lpart[(int64_t)layer * NPART + tid] = s;
    __threadfence();
  }
  __syncthreads();
  if (tid == 0) last = atomicAdd(counter, 1u) == (unsigned)(nlayers - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  // the layer sum in layer order (bitwise the host's nc_slab_reduce), the layer partials staged through
  // shared memory 64 layers at a time (all loads in flight, instead of one dependent L2 load per layer)
  __shared__ double lbuf[64][NPART];
  double s = 0.0;
  for (int l0 = 0; l0 < nlayers; l0 += 64) {
    const int nl = min(64, nlayers - l0);
    for (int k = tid; k < nl * NPART; k += K3R_T) lbuf[k / NPART][k % NPART] = __ldcg(&lpart[(int64_t)l0 * NPART + k]);
    __syncthreads();
    if (tid < NPART)
      for (int l = 0; l < nl; ++l) s += lbuf[l][tid];
    __syncthreads();
  }
  if (tid < NPART) {
    tot[tid] = s;
    acc[tid] += s;
  } else if (tid == NPART) {
    acc[NPART] += 1.0;
    *counter = 0u;
  }
}

// neighborhood-size histogram (instrumentation): one warp per block
__global__ void __launch_bounds__(32) k_stencil_hist(const __grid_constant__ Geom g, unsigned long long* __restrict__ hist) {
  __shared__ K3Smem<float> tab;
  __shared__ unsigned int h[64];
  int lane = threadIdx.x & 31;
  h[lane] = 0;
  h[lane + 32] = 0;
  __syncwarp();
  for (int64_t c = blockIdx.x; c < g.ncells; c += gridDim.x) {
    int a0 = (int)(c % g.dims[0]);
    int a1 = (int)((c / g.dims[0]) % g.dims[1]);
    int a2 = (int)(c / ((int64_t)g.dims[0] * g.dims[1]));
    int ne = build_entries(g, a0, a1, a2, tab, lane);
    if (lane == 0) h[ne]++;
    __syncwarp();
  }
  __syncwarp();
  for (int k = lane; k < 64; k += 32)
    if (h[k]) atomicAdd(&hist[k], (unsigned long long)h[k]);
}

// ---------------------------------------------------------------------------
// Scatter sorted-order vectors back to gid order (n x 3 caller layout),
// optionally rotating (not needed: forces are already lab frame).
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_unsort3(int64_t n, const typename V4<T>::t* __restrict__ src, const uint32_t* __restrict__ gid,
                          T* __restrict__ dst) {
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  typename V4<T>::t v = src[s];
  int64_t g = gid[s];
  dst[3 * g] = v.x;
  dst[3 * g + 1] = v.y;
  dst[3 * g + 2] = v.z;
}

template <typename T>
__global__ void k_pack4(int64_t n, const T* __restrict__ src, typename V4<T>::t* __restrict__ dst) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  dst[i] = mk4(src[3 * i], src[3 * i + 1], src[3 * i + 2], (T)0);
}

// ---------------------------------------------------------------------------
// K4: SLLOD (reading R19).  E(s) = e^{A s} as 3x3 matrices from the host.
// ---------------------------------------------------------------------------
struct SllodParams {
  double Em[9];   // e^{-A dt/2}
  double Ed[9];   // e^{A dt}
  double Eh[9];   // e^{A dt/2}
  double dt, inv_m;
};

__device__ __forceinline__ void mv3(const double* E, double x, double y, double z, double& ox, double& oy, double& oz) {
  ox = E[0] * x + E[1] * y + E[2] * z;
  oy = E[3] * x + E[4] * y + E[5] * z;
  oz = E[6] * x + E[7] * y + E[8] * z;
}

// A deferred closing half kick of a SLLOD step, p <- e^{-A dt/2} p + dt/2 F (what k_kick does)
struct K3Kick {
  double Em[9];  // e^{-A dt/2} of the step that deferred it
  double hd;     // its dt / 2
};

// p <- E(-dt/2)(p + dt/2 F); q <- E(dt) q + dt E(dt/2) p / m; then K1 on the
// new box (wrap + key + histogram), in place on q and p.
#ifndef KDK_MINB
#define KDK_MINB 8
#endif
template <typename T>
__global__ void __launch_bounds__(256, KDK_MINB) k_kick_drift_key(int64_t n, typename V4<T>::t* __restrict__ q, typename V4<T>::t* __restrict__ p,
                                 const typename V4<T>::t* __restrict__ F, SllodParams sp, const __grid_constant__ Geom g,
                                 uint32_t* __restrict__ key, uint32_t* __restrict__ slot, uint32_t* __restrict__ counts,
                                 int pending = 0, const K3Kick pk = K3Kick{}) {
  PDL_ENTRY();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  typename V4<T>::t qi = q[i], pi = p[i], fi = F[i];
  if (pending) {  // the previous step's closing half kick (k_kick's arithmetic, same F, same rounding)
    double ax, ay, az;
    mv3(pk.Em, (double)pi.x, (double)pi.y, (double)pi.z, ax, ay, az);
    pi = mk4((T)(ax + pk.hd * (double)fi.x), (T)(ay + pk.hd * (double)fi.y), (T)(az + pk.hd * (double)fi.z), (T)0);
  }
  double hd = 0.5 * sp.dt;
  double px = (double)pi.x + hd * (double)fi.x, py = (double)pi.y + hd * (double)fi.y,
         pz = (double)pi.z + hd * (double)fi.z;
  double ax, ay, az;
  mv3(sp.Em, px, py, pz, ax, ay, az);
  double hx, hy, hz;
  mv3(sp.Eh, ax, ay, az, hx, hy, hz);
  double qx, qy, qz;
  mv3(sp.Ed, (double)qi.x, (double)qi.y, (double)qi.z, qx, qy, qz);
  qx += sp.dt * hx * sp.inv_m;
  qy += sp.dt * hy * sp.inv_m;
  qz += sp.dt * hz * sp.inv_m;
  // stored precision first, then the canonical wrap/key of K1
  double q0 = (double)(T)qx, q1 = (double)(T)qy, q2 = (double)(T)qz;
  uint32_t c = wrap_key_one<T>(g, q0, q1, q2);
  q[i] = mk4((T)q0, (T)q1, (T)q2, (T)0);
  p[i] = mk4((T)ax, (T)ay, (T)az, (T)0);
  key[i] = c;
  slot[i] = arrival_slot(counts, c);
}

// p <- E(-dt/2) p + dt/2 F
template <typename T>
__global__ void k_kick(int64_t n, typename V4<T>::t* __restrict__ p, const typename V4<T>::t* __restrict__ F,
                       SllodParams sp) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  typename V4<T>::t pi = p[i], fi = F[i];
  double ax, ay, az;
  mv3(sp.Em, (double)pi.x, (double)pi.y, (double)pi.z, ax, ay, az);
  double hd = 0.5 * sp.dt;
  p[i] = mk4((T)(ax + hd * (double)fi.x), (T)(ay + hd * (double)fi.y), (T)(az + hd * (double)fi.z), (T)0);
}


// ---------------------------------------------------------------------------
// Slab decomposition primitives (multi-GPU).  Caller arrays are
// n x 3 (the ABI layout); records exchanged between ranks are T4 words:
// migration = 2 words (q.xyz + gid, p.xyz + 0), halo = 1 word (q.xyz + gid).
// The gid travels as the bit pattern (fp32) or the exact value (fp64) of .w.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_kick_drift3(int64_t n, T* __restrict__ q, T* __restrict__ p, const T* __restrict__ F, SllodParams sp,
                              int pending = 0, const K3Kick pk = K3Kick{}, const uint32_t* __restrict__ dn = nullptr) {
  if (dn) n = (int64_t)min((unsigned long long)n, (unsigned long long)*dn);
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double hd = 0.5 * sp.dt;
  double p0 = (double)p[3 * i], p1 = (double)p[3 * i + 1], p2 = (double)p[3 * i + 2];
  if (pending) {  // the previous step's closing half kick (k_kick3's arithmetic, same F, same rounding)
    double ax, ay, az;
    mv3(pk.Em, p0, p1, p2, ax, ay, az);
    p0 = (double)(T)(ax + pk.hd * (double)F[3 * i]);
    p1 = (double)(T)(ay + pk.hd * (double)F[3 * i + 1]);
    p2 = (double)(T)(az + pk.hd * (double)F[3 * i + 2]);
  }
  double px = p0 + hd * (double)F[3 * i], py = p1 + hd * (double)F[3 * i + 1], pz = p2 + hd * (double)F[3 * i + 2];
  double ax, ay, az, hx, hy, hz, qx, qy, qz;
  mv3(sp.Em, px, py, pz, ax, ay, az);
  mv3(sp.Eh, ax, ay, az, hx, hy, hz);
  mv3(sp.Ed, (double)q[3 * i], (double)q[3 * i + 1], (double)q[3 * i + 2], qx, qy, qz);
  q[3 * i] = (T)(qx + sp.dt * hx * sp.inv_m);
  q[3 * i + 1] = (T)(qy + sp.dt * hy * sp.inv_m);
  q[3 * i + 2] = (T)(qz + sp.dt * hz * sp.inv_m);
  p[3 * i] = (T)ax; p[3 * i + 1] = (T)ay; p[3 * i + 2] = (T)az;
}

template <typename T>
__global__ void k_kick3(int64_t n, T* __restrict__ p, const T* __restrict__ F, SllodParams sp,
                        const uint32_t* __restrict__ dn = nullptr) {
  if (dn) n = (int64_t)min((unsigned long long)n, (unsigned long long)*dn);
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double ax, ay, az;
  mv3(sp.Em, (double)p[3 * i], (double)p[3 * i + 1], (double)p[3 * i + 2], ax, ay, az);
  double hd = 0.5 * sp.dt;
  p[3 * i] = (T)(ax + hd * (double)F[3 * i]);
  p[3 * i + 1] = (T)(ay + hd * (double)F[3 * i + 1]);
  p[3 * i + 2] = (T)(az + hd * (double)F[3 * i + 2]);
}

// mode 0 (migration): wrap q in place (R15); class 0 = layer owned, 1 = layer klo-1 (to rank r-1),
//                     2 = layer khi (to rank r+1), 3 = further away (error).
// mode 1 (halo):      class 1 = layer klo (copy to r-1), 2 = layer khi-1 (copy to r+1), else 0.
// mode 2 (layers):    wrap q in place and write each particle's cell layer to layer_out.
template <typename T>
__global__ void k_slab_classify(int64_t n, T* __restrict__ q, const __grid_constant__ Geom g, int klo, int khi,
                                int mode, uint8_t* __restrict__ cls, int32_t* __restrict__ layer_out = nullptr,
                                const uint32_t* __restrict__ dn = nullptr) {
  if (dn) n = (int64_t)min((unsigned long long)n, (unsigned long long)*dn);
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double q0 = (double)q[3 * i], q1 = (double)q[3 * i + 1], q2 = (double)q[3 * i + 2];
  double lam[3];
  frac_c(g, q0, q1, q2, lam);
  if (lam[0] < 0.0 || lam[0] >= 1.0 || lam[1] < 0.0 || lam[1] >= 1.0 || lam[2] < 0.0 || lam[2] >= 1.0) {
    int n0 = (int)floor(lam[0]), n1 = (int)floor(lam[1]), n2 = (int)floor(lam[2]);
    q0 = round_to(__dsub_rn(q0, lshift_c(g, 0, n0, n1, n2)), T());
    q1 = round_to(__dsub_rn(q1, lshift_c(g, 1, n0, n1, n2)), T());
    q2 = round_to(__dsub_rn(q2, lshift_c(g, 2, n0, n1, n2)), T());
    q[3 * i] = (T)q0; q[3 * i + 1] = (T)q1; q[3 * i + 2] = (T)q2;
    frac_c(g, q0, q1, q2, lam);
  }
  CellPos cp;
  cell_of(g, lam, cp);
  const int k = cp.a[2], l3 = g.dims[2];
  if (mode == 2) {  // the layer itself (repartition after a change of l3)
    layer_out[i] = k;
    return;
  }
  uint8_t c;
  if (mode == 0) {
    if (k >= klo && k < khi) c = 0;
    else if (k == (klo - 1 + l3) % l3) c = 1;
    else if (k == khi % l3) c = 2;
    else c = 3;
  } else {
    c = (k == klo) ? 1 : (k == khi - 1 ? 2 : 0);
  }
  cls[i] = c;
}

constexpr int PART_T = 256;
// per-block counts of classes 0..3, CLASS-MAJOR (bcnt[c * nb + b]) so that one
// exclusive scan of the 4 nb entries gives every class's block offsets
__global__ void k_class_count(int64_t n, int64_t nb, const uint8_t* __restrict__ cls, uint32_t* __restrict__ bcnt,
                              const uint32_t* __restrict__ dn = nullptr) {
  if (dn) n = (int64_t)min((unsigned long long)n, (unsigned long long)*dn);
  __shared__ uint32_t c[4];
  if (threadIdx.x < 4) c[threadIdx.x] = 0;
  __syncthreads();
  int64_t i = (int64_t)blockIdx.x * PART_T + threadIdx.x;
  if (i < n) atomicAdd(&c[cls[i]], 1u);  // counts only: order-free
  __syncthreads();
  if (threadIdx.x < 4) bcnt[(int64_t)threadIdx.x * nb + blockIdx.x] = c[threadIdx.x];
}
// class totals from the scanned class-major counts (boff has 4 nb + 1 entries)
__global__ void k_class_totals(const uint32_t* __restrict__ boff, int64_t nb, uint32_t* __restrict__ tot) {
  int c = threadIdx.x;
  if (c < 4) tot[c] = boff[(c + 1) * nb] - boff[c * nb];
}
// stable partition by class (index order within each class): class 0 -> SoA outputs, classes 1, 2 ->
// records of `words` T4 words (2: q+gid, p; 1: q+gid)
template <typename T>
__global__ void k_class_scatter(int64_t n, const uint8_t* __restrict__ cls, const uint32_t* __restrict__ boff,
                                const T* __restrict__ q, const T* __restrict__ p, const uint32_t* __restrict__ gid,
                                T* __restrict__ q0, T* __restrict__ p0, uint32_t* __restrict__ g0,
                                typename V4<T>::t* __restrict__ r1, typename V4<T>::t* __restrict__ r2, int words,
                                const uint32_t* __restrict__ dn = nullptr, int64_t rcap = INT64_MAX) {
  // (dn: device count, the grid covers a capacity; rcap: records beyond a message's capacity are dropped
  // -- the totals flag the overflow)
  if (dn) n = (int64_t)min((unsigned long long)n, (unsigned long long)*dn);
  __shared__ uint32_t wsum[PART_T / 32][4];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int64_t i = (int64_t)blockIdx.x * PART_T + threadIdx.x;
  const int c = i < n ? cls[i] : 4;
  uint32_t rank_in_warp = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    unsigned b = __ballot_sync(0xffffffffu, c == k);
    if (c == k) rank_in_warp = __popc(b & ((1u << lane) - 1u));
    if (lane == 0) wsum[wid][k] = __popc(b);
  }
  __syncthreads();
  if (c >= 3) return;
  const int64_t nb = gridDim.x;
  uint32_t pos = boff[(int64_t)c * nb + blockIdx.x] - boff[(int64_t)c * nb] + rank_in_warp;
  for (int w = 0; w < wid; ++w) pos += wsum[w][c];
  const T x = q[3 * i], y = q[3 * i + 1], z = q[3 * i + 2];
  const uint32_t gg = gid[i];
  if (c == 0) {
    if (q0) {
      q0[3 * pos] = x; q0[3 * pos + 1] = y; q0[3 * pos + 2] = z;
      if (p0) { p0[3 * pos] = p[3 * i]; p0[3 * pos + 1] = p[3 * i + 1]; p0[3 * pos + 2] = p[3 * i + 2]; }
      g0[pos] = gg;
    }
    return;
  }
  if ((int64_t)pos >= rcap) return;
  typename V4<T>::t* r = (c == 1 ? r1 : r2) + (int64_t)pos * words;
  r[0] = mk4(x, y, z, idx_to_w(gg, T()));
  if (words == 2) r[1] = mk4(p[3 * i], p[3 * i + 1], p[3 * i + 2], (T)0);
}

template <typename T>
__global__ void k_records_unpack(int64_t n, const typename V4<T>::t* __restrict__ r, T* __restrict__ q,
                                 T* __restrict__ p, uint32_t* __restrict__ gid) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  typename V4<T>::t a = r[2 * i], b = r[2 * i + 1];
  q[3 * i] = a.x; q[3 * i + 1] = a.y; q[3 * i + 2] = a.z;
  p[3 * i] = b.x; p[3 * i + 1] = b.y; p[3 * i + 2] = b.z;
  gid[i] = w_to_idx(a.w);
}

// K1 over one source of the local system (own particles: n x 3 + gid array; halo records: T4 with gid in .w)
template <typename T>
__global__ void k_wrap_key_src(int64_t n, const T* __restrict__ qin, int stride, const uint32_t* __restrict__ gsrc,
                               int64_t off, typename V4<T>::t* __restrict__ qout, uint32_t* __restrict__ gout,
                               uint32_t* __restrict__ key, uint32_t* __restrict__ slot, uint32_t* __restrict__ counts,
                               const __grid_constant__ Geom g, const uint32_t* __restrict__ dn = nullptr) {
  if (dn) n = (int64_t)min((unsigned long long)n, (unsigned long long)*dn);
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double q0 = (double)qin[i * stride], q1 = (double)qin[i * stride + 1], q2 = (double)qin[i * stride + 2];
  uint32_t gg = gsrc ? gsrc[i] : w_to_idx(qin[i * stride + 3]);
  uint32_t c = wrap_key_one<T>(g, q0, q1, q2);
  qout[off + i] = mk4((T)q0, (T)q1, (T)q2, (T)0);
  gout[off + i] = gg;
  key[off + i] = c;
  slot[off + i] = arrival_slot(counts, c);
}

// positions of the caller's particles in a given order (build_user): slot s takes caller index perm[s]
template <typename T>
__global__ void k_pregather(int64_t n, const T* __restrict__ q, const uint32_t* __restrict__ perm, T* __restrict__ qo,
                            uint32_t* __restrict__ go) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const uint32_t i = perm[s];
  qo[3 * s] = q[3 * (int64_t)i]; qo[3 * s + 1] = q[3 * (int64_t)i + 1]; qo[3 * s + 2] = q[3 * (int64_t)i + 2];
  go[s] = i;
}

// F of the own particles back to their input order (sorted slot -> original local index)
template <typename T>
__global__ void k_unsort_idx(int64_t n, const typename V4<T>::t* __restrict__ src, const uint32_t* __restrict__ sidx,
                             int64_t n_own, T* __restrict__ dst, const uint32_t* __restrict__ drange = nullptr) {
  // drange: sorted slots [drange[0], drange[1]) (the own particles of a device-count slab step)
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (drange) {
    s += drange[0];
    if (s >= (int64_t)drange[1]) return;
    n_own = INT64_MAX;
  } else if (s >= n) {
    return;
  }
  uint32_t i = sidx[s];
  if ((int64_t)i >= n_own) return;
  typename V4<T>::t v = src[s];
  dst[3 * (int64_t)i] = v.x; dst[3 * (int64_t)i + 1] = v.y; dst[3 * (int64_t)i + 2] = v.z;
}

}  // namespace nc

#include "k3_seg.cuh"
#include "k3_sparse.cuh"
#include "k3_rows.cuh"
#include "k3_sparse64.cuh"
