// k3_sparse.cuh -- K3 for sparse cells (WCA at rho = 0.8442: ~1.3 particles per cell), NC_F32.
// Included at the end of kernels.cuh.
//
// One thread per particle i, the paper's loop literally: for each cell of
// i's neighborhood (27 DS / 27-36 DO by the exact interval rule, the same fp64 expressions as
// build_entries, so stencils and candidate counts are the oracle's bit for bit), each particle j of
// that cell, distance check.  The 32 lanes of a warp hold 32 CONSECUTIVE particles of the
// (cell, gid) order -- consecutive cells of one row -- and walk the stencil rows in lockstep: in row
// r, lane i scans the contiguous particle range of its 3-4 neighbour columns, and because the lanes'
// cells are consecutive, each warp-wide load touches a few consecutive 128-byte lines (coalesced,
// L1/L2-resident: no shared-memory staging, no per-segment setup).  Lattice images: the column
// shift of a wrapped column and the row's (n2, n3) shift, applied as a bracket in i's cell-local
// rotated frame (|d| stays ~ r_c: fp32 filter with the superset band), exactly as k_pairs' entries.
// Filter survivors are queued per lane (shared memory) and evaluated in fp64 from the fp64
// cell-local coordinates with the canonical R16 test inside the 1e-12 band (WCA pairs all lie below
// r_split: every interaction is fp64).  Full i-side accumulation, no atomics; block partials are a
// fixed-order sum over a fixed particle range of ONE layer (layer-aligned, P-invariant).
#pragma once

namespace nc {

#ifndef NC_SP_NT
#define NC_SP_NT 128
#endif
constexpr int SP_NT = NC_SP_NT;  // threads per block (one particle each per chunk)
constexpr int SP_QCAP = 16;   // per-thread hit queue (flushed when some lane could overflow)
#ifndef NC_SP_UNR
#define NC_SP_UNR 4
#endif
#ifndef NC_SP_MINB
#define NC_SP_MINB 4
#endif
constexpr int SP_UNR = NC_SP_UNR;
#ifndef NC_SP_LPP_CELLS
#define NC_SP_LPP_CELLS 8192  // grids below this many cells use 4 threads per particle (host sparse_lpp)
#endif
constexpr int64_t SP_LPP_CELLS = NC_SP_LPP_CELLS;
constexpr int64_t SP_LPP2_CELLS = 65536;  // grids below this many cells: 2 threads per particle (AUTO)
constexpr int SP_QD = SP_QCAP * SP_NT * 4;  // byte offset of qd from qj
constexpr int SP_CPB = 96 * SP_NT / 128;  // cells of a layer per block (~1.3 particles each: ~one pass of SP_NT)  // candidates per iteration (their loads in flight together)

struct SpSmem {
  uint32_t qj[SP_QCAP][SP_NT];  // sorted index of a queued j
  uint32_t qd[SP_QCAP][SP_NT];  // its neighbour cell: unwrapped column delta d0 + 32768 | stencil row << 16
  double part[SP_NT / 32][NPART];
  // per-thread accumulators (live only inside sp_eval: the registers go to the candidate loop)
  double acc[10][SP_NT];
  double tuw[7][SP_NT];   // per-thread block statistics U, W0..W5
  uint32_t cnt[SP_NT], nrc[SP_NT];
  uint64_t hs[SP_NT], hx[SP_NT];
  struct RowW {           // the a0-independent part of a stencil row (sp_row_inv), per warp and cell row
    double ox, bxr;       // DO x offset of the row (DS: 0); the row's part of the fp64 x bracket
    float byf, bzf;       // fp32 y, z brackets
    uint32_t base, meta;  // first cell id of the row; exists | d1 | n2 | n3 | d2 (sp_meta)
  } rw[SP_NT / 32][2][12];
};

// row ri of cell (a0, a1, a2)'s neighborhood: columns [c0, c1) (unwrapped), row image shifts and the
// row's unwrapped deltas.  Returns false if the row does not exist (DO: 3 of the 4 slots of a layer
// when the y offset is a multiple of the cell height; DS: ri >= 9).  The expressions are
// build_entries' (canonical fp64 for DO).
struct SpRow {
  int c0, c1;          // unwrapped columns
  int n2, n3, d1, d2;  // image shifts (y, z) and unwrapped row deltas (m - a1, kk - a2)
  uint32_t base;       // first cell id of the row: l1 (jd + l2 kd)
};
__device__ __forceinline__ bool sp_row(const Geom& g, int ri, int a0, int a1, int a2, SpRow& r) {
  const int l1 = g.dims[0], l2 = g.dims[1], l3 = g.dims[2];
  if (g.variant == 0) {
    if (ri >= 9) return false;
    const int d1 = ri % 3 - 1, d2 = ri / 3 - 1;
    const int m1 = a1 + d1, m2 = a2 + d2;
    const int n1 = floordiv(m1, l2), n2 = floordiv(m2, l3);
    r.c0 = a0 - 1;
    r.c1 = a0 + 2;
    r.n2 = n1;  // DS: the y and z lattice shifts of the row
    r.n3 = n2;
    r.d1 = d1;
    r.d2 = d2;
    r.base = (uint32_t)l1 * ((uint32_t)(m1 - n1 * l2) + (uint32_t)l2 * (uint32_t)(m2 - n2 * l3));
    return true;
  }
  const int dz = ri / 4 - 1, rr = ri % 4;
  const int kk = a2 + dz;
  const int n3 = floordiv(kk, l3);
  const int kd = kk - n3 * l3;
  const double oy = __dmul_rn((double)n3, g.d32);
  const int m0 = (int)floor(__dsub_rn((double)(a1 - 1), oy));
  const int m1 = (int)ceil(__dsub_rn((double)(a1 + 2), oy));
  if (rr >= m1 - m0) return false;
  const int m = m0 + rr;
  const int n2 = floordiv(m, l2);
  const int jd = m - n2 * l2;
  const double ox = __dadd_rn(__dmul_rn((double)n3, g.d31), __dmul_rn((double)n2, g.d21));
  r.c0 = (int)floor(__dsub_rn((double)(a0 - 1), ox));
  r.c1 = (int)ceil(__dsub_rn((double)(a0 + 2), ox));
  r.n2 = n2;
  r.n3 = n3;
  r.d1 = m - a1;
  r.d2 = dz;
  r.base = (uint32_t)l1 * ((uint32_t)jd + (uint32_t)l2 * (uint32_t)kd);
  return true;
}

// The part of row ri of the cells (*, a1, a2) that does not depend on the column a0 (lanes of a warp
// share it: 32 consecutive particles sit in one or two cell rows).  With it, sp_row's columns are
// c0 = floor(fl(a0 - 1 - ox)), c1 = ceil(fl(a0 + 2 - ox)) -- the same fp64 expressions (DS: ox = 0).
__device__ __forceinline__ uint32_t sp_meta(bool ex, int d1, int n2, int n3, int d2) {
  return (ex ? 1u : 0u) | ((uint32_t)(d1 + 32768) << 1) | ((uint32_t)(n2 + 8) << 17) | ((uint32_t)(n3 + 8) << 21) |
         ((uint32_t)(d2 + 2) << 25);
}
__device__ __forceinline__ void sp_row_inv(const Geom& g, int ri, int a1, int a2, SpSmem::RowW& w) {
  const int l1 = g.dims[0], l2 = g.dims[1], l3 = g.dims[2];
  if (g.variant == 0) {
    const int d1 = ri % 3 - 1, d2 = ri / 3 - 1;
    const int m1 = a1 + d1, m2 = a2 + d2;
    const int n1 = floordiv(m1, l2), n2 = floordiv(m2, l3);
    const double u1 = (double)d1 * g.cinv[1], u2 = (double)d2 * g.cinv[2];
    w.ox = 0.0;
    w.bxr = g.R[1] * u1 + g.R[2] * u2;
    w.byf = (float)(g.R[4] * u1 + g.R[5] * u2);
    w.bzf = (float)(g.R[8] * u2);
    w.base = (uint32_t)l1 * ((uint32_t)(m1 - n1 * l2) + (uint32_t)l2 * (uint32_t)(m2 - n2 * l3));
    w.meta = sp_meta(ri < 9, d1, n1, n2, d2);
    return;
  }
  const int dz = ri / 4 - 1, rr = ri % 4;
  const int kk = a2 + dz;
  const int n3 = floordiv(kk, l3);
  const int kd = kk - n3 * l3;
  const double oy = __dmul_rn((double)n3, g.d32);
  const int m0 = (int)floor(__dsub_rn((double)(a1 - 1), oy));
  const int m1 = (int)ceil(__dsub_rn((double)(a1 + 2), oy));
  const int m = m0 + rr;
  const int n2 = floordiv(m, l2);
  const int jd = m - n2 * l2;
  w.ox = __dadd_rn(__dmul_rn((double)n3, g.d31), __dmul_rn((double)n2, g.d21));
  w.bxr = (double)n2 * g.R[1] + (double)n3 * g.R[2];
  w.byf = (float)((double)(m - a1) * g.w[1] + (double)n2 * g.e[1] + (double)n3 * g.R[5]);
  w.bzf = (float)((double)dz * g.w[2] + (double)n3 * g.e[2]);
  w.base = (uint32_t)l1 * ((uint32_t)jd + (uint32_t)l2 * (uint32_t)kd);
  w.meta = sp_meta(rr < m1 - m0, m - a1, n2, n3, dz);
}

// A neighbour cell relative to i's cell: unwrapped deltas (d0 column, d1 row, d2 layer) and the
// lattice image n (DO: the column's x shift n1 and the row's n2, n3; DS: the x, y, z wraps).  The
// column / row deltas can be large in DO (the rows of the offset faces sit ~n2 d21 cells away): a
// queued hit carries d0 in 16 bits and its stencil row; the rest comes from the row data (sp_meta).
struct SpCell {
  int d0, d1, d2, n1, n2, n3;
};

// fp64 bracket of a neighbour cell relative to i's cell (build_entries' formulas): DS R (delta / c);
// DO (d0 w0 + n1 e0 + n2 r12 + n3 r13, d1 w1 + n2 e1 + n3 r23, d2 w2 + n3 e2)
__device__ __forceinline__ void sp_bracket(const Geom& g, const SpCell& c, double& bx, double& by, double& bz) {
  if (g.variant == 0) {
    const double u0 = (double)c.d0 * g.cinv[0], u1 = (double)c.d1 * g.cinv[1], u2 = (double)c.d2 * g.cinv[2];
    bx = g.R[0] * u0 + g.R[1] * u1 + g.R[2] * u2;
    by = g.R[4] * u1 + g.R[5] * u2;
    bz = g.R[8] * u2;
  } else {
    bx = (double)c.d0 * g.w[0] + (double)c.n1 * g.e[0] + (double)c.n2 * g.R[1] + (double)c.n3 * g.R[2];
    by = (double)c.d1 * g.w[1] + (double)c.n2 * g.e[1] + (double)c.n3 * g.R[5];
    bz = (double)c.d2 * g.w[2] + (double)c.n3 * g.e[2];
  }
}

// fp64 evaluation of this thread's queued candidates (two per iteration, loads first)
template <bool DIGEST>
__device__ __forceinline__ void sp_eval(const Geom& g, SpSmem& sm, const double4* __restrict__ u,
                                        const float4* __restrict__ qs, const uint32_t* __restrict__ nh,
                                        const uint32_t* __restrict__ gid, int nq, int tid, uint32_t me, uint32_t nh_i,
                                        double lo64, double hi64, const PairOut& po, uint32_t gi, int a0, int a1,
                                        int grp, int wid, int layer) {
  const int lane = tid & 31;
  const int qmax = __reduce_max_sync(0xffffffffu, nq);
  if (qmax == 0) return;
  const double4 ui = u[me];
  const double uix = ui.x, uiy = ui.y, uiz = ui.z;
  Acc acc;
  acc.fx = sm.acc[0][tid]; acc.fy = sm.acc[1][tid]; acc.fz = sm.acc[2][tid]; acc.u = sm.acc[3][tid];
  acc.w0 = sm.acc[4][tid]; acc.w1 = sm.acc[5][tid]; acc.w2 = sm.acc[6][tid];
  acc.w3 = sm.acc[7][tid]; acc.w4 = sm.acc[8][tid]; acc.w5 = sm.acc[9][tid];
  acc.cnt = sm.cnt[tid]; acc.nrc = sm.nrc[tid];
  if (DIGEST) { acc.hs = sm.hs[tid]; acc.hx = sm.hx[tid]; }
  const double sig2 = g.sig2, eps24 = 24.0 * g.eps;
  for (int k0 = 0; k0 < qmax; k0 += 2) {
    uint32_t jj[2];
    SpCell cc[2];
    bool ok0[2];
    double4 uj[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      ok0[h] = k0 + h < nq;
      jj[h] = ok0[h] ? sm.qj[k0 + h][tid] : me;
      // the queue code: unwrapped column delta d0 and the stencil row; the row's deltas and image
      // shifts from the warp's row data; the column's x image from the unwrapped column a0 + d0
      const uint32_t code = ok0[h] ? sm.qd[k0 + h][tid] : 32768u;
      const int ri = (int)(code >> 16);
      uint32_t meta;
      if (grp >= 0) meta = sm.rw[wid][grp][ri].meta;
      else { SpSmem::RowW w; sp_row_inv(g, ri, a1, layer, w); meta = w.meta; }
      cc[h].d0 = (int)(code & 0xffffu) - 32768;
      cc[h].d1 = (int)((meta >> 1) & 0xffffu) - 32768;
      cc[h].n2 = (int)((meta >> 17) & 15u) - 8;
      cc[h].n3 = (int)((meta >> 21) & 15u) - 8;
      cc[h].d2 = (int)((meta >> 25) & 3u) - 2;
      cc[h].n1 = floordiv(a0 + cc[h].d0, g.dims[0]);
      uj[h] = u[jj[h]];
    }
    (void)lane;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double bx, by, bz;
      sp_bracket(g, cc[h], bx, by, bz);
      const double dx = (uj[h].x + bx) - uix, dy = (uj[h].y + by) - uiy, dz = (uj[h].z + bz) - uiz;
      const double r2 = dx * dx + dy * dy + dz * dz;
      bool ok = ok0[h] && (jj[h] != me) && (r2 < hi64);
      int n0 = 0, n1 = 0, n2 = 0;
      // (a real branch: pairs inside the 1e-12 band are rare, the vote keeps the canonical test out of line)
      if ((DIGEST || __any_sync(0xffffffffu, ok && r2 >= lo64)) && ok && (DIGEST || r2 >= lo64)) {
        n0 = cc[h].n1;
        n1 = cc[h].n2;
        n2 = cc[h].n3;
        if (g.variant == 1) {
          const uint32_t nh_j = nh[jj[h]];
          n0 += nh_x(nh_j) - nh_x(nh_i);
          n1 += nh_y(nh_j) - nh_y(nh_i);
        }
        if (r2 >= lo64) {
          const float4 qi = qs[me], qj = qs[jj[h]];
          ok = canonical_r2(g, (double)qj.x, (double)qj.y, (double)qj.z, (double)qi.x, (double)qi.y, (double)qi.z, n0,
                            n1, n2) < g.rc2;
          acc.nrc++;
        }
      }
      const double ir = rcp64(r2);
      const double s2 = sig2 * ir;
      const double s6 = s2 * s2 * s2;
      double fr = (eps24 * s6) * (2.0 * s6 - 1.0) * ir;
      fr = ok ? fr : 0.0;
      const double tx = fr * dx, ty = fr * dy, tz = fr * dz;
      acc.fx -= tx; acc.fy -= ty; acc.fz -= tz;
      acc.u += ok ? s6 * s6 - s6 : 0.0;
      acc.w0 += tx * dx; acc.w1 += ty * dy; acc.w2 += tz * dz;
      acc.w3 += tx * dy; acc.w4 += tx * dz; acc.w5 += ty * dz;
      acc.cnt += ok ? 1u : 0u;
      if (DIGEST && ok) digest_add<DIGEST>(acc, gid, jj[h], n0, n1, n2, po, gi);
    }
  }
  sm.acc[0][tid] = acc.fx; sm.acc[1][tid] = acc.fy; sm.acc[2][tid] = acc.fz; sm.acc[3][tid] = acc.u;
  sm.acc[4][tid] = acc.w0; sm.acc[5][tid] = acc.w1; sm.acc[6][tid] = acc.w2;
  sm.acc[7][tid] = acc.w3; sm.acc[8][tid] = acc.w4; sm.acc[9][tid] = acc.w5;
  sm.cnt[tid] = acc.cnt; sm.nrc[tid] = acc.nrc;
  if (DIGEST) { sm.hs[tid] = acc.hs; sm.hx[tid] = acc.hx; }
  __syncwarp();
}

// grid = nlay layers x bpl blocks; block b of layer L takes the layer's particles
// [b SP_NT, (b+1) SP_NT) + k bpl SP_NT, k = 0, 1, ... (a fixed partition of the layer).  The cells of
// the layer are walked the same way for the stencil-size statistic (empty cells included).
template <bool DIGEST, int LPP = 1>
__global__ void __launch_bounds__(SP_NT, NC_SP_MINB)
k_pairs_sparse(const double4* __restrict__ u, const float4* __restrict__ u32, const uint32_t* __restrict__ cs,
               const uint4* __restrict__ rec, const float4* __restrict__ qs, const uint32_t* __restrict__ nh,
               const uint32_t* __restrict__ gid, float4* __restrict__ Fout, double* __restrict__ bpart,
               uint32_t* __restrict__ dcnt, uint64_t* __restrict__ dhs, uint64_t* __restrict__ dhx,
               const __grid_constant__ Geom g, int bpl, int layer0, const PairOut po) {
  PDL_WAIT();  // (the successor is released at the end)
  extern __shared__ __align__(16) unsigned char sp_raw[];
  SpSmem& sm = *reinterpret_cast<SpSmem*>(sp_raw);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int l1 = g.dims[0], l2 = g.dims[1];
  const int layer = layer0 + (int)(blockIdx.x / bpl);
  const int b = (int)blockIdx.x - (layer - layer0) * bpl;
  const uint32_t per_layer = (uint32_t)l1 * (uint32_t)l2;
  const uint32_t cell0 = per_layer * (uint32_t)layer;
  const uint32_t P0 = cs[cell0], P1 = cs[cell0 + per_layer];
  const double lo64 = g.rc2 * (1.0 - K3_BAND64), hi64 = g.rc2 * (1.0 + K3_BAND64);
  const float hi32 = (float)g.band_hi;
  const float w0x = (float)(g.variant == 0 ? g.R[0] * g.cinv[0] : g.w[0]);
  // block statistics: U and W per thread in shared memory (registers go to the candidate loop), counts
  // as integers
#pragma unroll
  for (int f = 0; f < 7; ++f) sm.tuw[f][tid] = 0.0;
  uint32_t tI = 0, tC = 0, tS = 0, tR = 0, tNF = 0;

  // stencil sizes of the layer's cells (empty ones included): the neighborhood-size statistic, from the
  // warp's shared row data (a row of cells (a0, a1) has ceil(fl(a0 + 2 - ox)) - floor(fl(a0 - 1 - ox))
  // columns, sp_row's expressions)
  for (uint32_t cb = (uint32_t)b * SP_NT; cb < per_layer; cb += (uint32_t)bpl * SP_NT) {
    const uint32_t c = cb + (uint32_t)tid;
    const bool cv = c < per_layer;
    const uint32_t cc = cv ? c : cb;
    const int a0 = (int)(cc % (uint32_t)l1), a1 = (int)(cc / (uint32_t)l1);
    const int a1A = __shfl_sync(0xffffffffu, a1, 0), a1B = __shfl_sync(0xffffffffu, a1, 31);
    __syncwarp();
    if ((lane & 15) < 12) sp_row_inv(g, lane & 15, lane < 16 ? a1A : a1B, layer, sm.rw[wid][lane >> 4][lane & 15]);
    __syncwarp();
    const int grp = a1 == a1A ? 0 : (a1 == a1B ? 1 : -1);
    // a row's width c1 - c0 does not depend on a0 unless ox lies within 2^-30 of an integer without being
    // one (then fl(a0 - 1 - ox) could round across it): 3 for an integral ox (DS: ox = 0), else 4; the
    // building lanes sum their group's widths (64 flags a row that needs the per-cell expressions)
    int wcode = 0;
    if ((lane & 15) < 12) {
      const SpSmem::RowW& wr = sm.rw[wid][lane >> 4][lane & 15];  // written by this lane above
      if (wr.meta & 1u) {
        const double f = wr.ox - floor(wr.ox);
        wcode = f == 0.0 ? 3 : (fmin(f, 1.0 - f) > 0x1p-30 ? 4 : 64);
      }
    }
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) wcode += __shfl_xor_sync(0xffffffffu, wcode, o);
    const int totA = __shfl_sync(0xffffffffu, wcode, 0), totB = __shfl_sync(0xffffffffu, wcode, 16);
    const int tot = grp == 0 ? totA : (grp == 1 ? totB : 64);
    int ns = tot;
    if (tot >= 64) {  // the per-cell expressions (sp_row's)
      ns = 0;
      for (int ri = 0; ri < 12; ++ri) {
        SpSmem::RowW w;
        if (grp >= 0) w = sm.rw[wid][grp][ri];
        else sp_row_inv(g, ri, a1, layer, w);
        if (w.meta & 1u)
          ns += (int)ceil(__dsub_rn((double)(a0 + 2), w.ox)) - (int)floor(__dsub_rn((double)(a0 - 1), w.ox));
      }
    }
    if (cv) tS += (uint32_t)(ns - g.dbg_drop);
  }

  // LPP > 1 (small systems: more warps, a shorter chain per warp): LPP consecutive threads share one
  // particle, thread `sub` walking the stencil rows sub, sub + LPP, ...; their partial sums are combined
  // in fixed order (sub 0 + 1 + ... ) by the owner (sub 0)
  constexpr int NPB = SP_NT / LPP;  // particles per block pass
  const int sub = LPP > 1 ? tid % LPP : 0;
  for (uint32_t base = P0 + (uint32_t)b * NPB; base < P1; base += (uint32_t)bpl * NPB) {
    const uint32_t i = base + (uint32_t)(LPP > 1 ? tid / LPP : tid);
    const bool act = i < P1;
    const uint32_t me = act ? i : P0;
    const uint32_t c = rec[me].z;  // the cell of sorted slot me (bucket records: same cell order)
    const int a0 = (int)(c % (uint32_t)l1), a1 = (int)((c / (uint32_t)l1) % (uint32_t)l2);
    const float4 ui32 = u32[me];
    const uint32_t nh_i = (g.variant == 1) ? nh[me] : 0u;
    const uint32_t gi = DIGEST ? gid[me] : 0u;
#pragma unroll
    for (int f = 0; f < 10; ++f) sm.acc[f][tid] = 0.0;
    sm.cnt[tid] = 0u; sm.nrc[tid] = 0u;
    if (DIGEST) { sm.hs[tid] = 0ull; sm.hx[tid] = 0ull; }
    int nq = 0;
    uint32_t ncand = 0;
    // the last neighborhood entry is dropped in the negative-control mode (nc_debug): the last
    // column of the last existing row
    int last_ri = 0;
    if (g.dbg_drop)
      for (int ri = 0; ri < 12; ++ri) {
        SpRow r;
        if (sp_row(g, ri, a0, a1, layer, r)) last_ri = ri;
      }
    // the a0-independent row data of the warp's (at most) two cell rows, built once by lanes 0-11 / 16-27;
    // a lane of a third cell row (tiny grids) builds its own
    __syncwarp();  // the previous particle batch's readers are done
    const int a1A = __shfl_sync(0xffffffffu, a1, 0), a1B = __shfl_sync(0xffffffffu, a1, 31);
    if ((lane & 15) < 12) sp_row_inv(g, lane & 15, lane < 16 ? a1A : a1B, layer, sm.rw[wid][lane >> 4][lane & 15]);
    __syncwarp();
    const int grp = a1 == a1A ? 0 : (a1 == a1B ? 1 : -1);
    // queue slot addresses of this thread: qj[k][tid] at qa0 + 4 SP_NT k, qd[k][tid] SP_QD bytes further
    const uint32_t qa0 = smem_u32(&sm.qj[0][tid]);
    uint32_t qa = qa0;
    for (int it = 0; it < (12 + LPP - 1) / LPP; ++it) {  // (the same trip count for every lane of the warp)
      const int rs = sub + it * LPP;  // this thread's stencil row (none past row 11 when LPP does not divide 12)
      const int ri = rs < 12 ? rs : 11;
      SpSmem::RowW w;
      if (grp >= 0) w = sm.rw[wid][grp][ri];
      else sp_row_inv(g, ri, a1, layer, w);
      const bool has = act && rs < 12 && (w.meta & 1u);
      if (!__any_sync(0xffffffffu, has)) continue;
      // columns [c0, c1) in <= 2 pieces of constant x shift n1 (the row wraps at most once:
      // c1 - c0 <= 4 <= l1) and the pieces' cell starts
      int c0 = (int)floor(__dsub_rn((double)(a0 - 1), w.ox));
      int c1 = (int)ceil(__dsub_rn((double)(a0 + 2), w.ox));
      if (!has) { c0 = c1 = a0; w.base = 0u; }
      if (has && g.dbg_drop && ri == last_ri) c1 -= 1;
      const int n1a = floordiv(c0, l1);
      const int cut = (n1a + 1) * l1;            // first column of the next x image
      const uint32_t pa0 = cs[w.base + (uint32_t)(c0 - n1a * l1)];
      const uint32_t pa1 = cs[w.base + (uint32_t)(min(c1, cut) - n1a * l1)];
      uint32_t pb0 = 0u, pb1 = 0u;
      if (c1 > cut) {
        pb0 = cs[w.base];
        pb1 = cs[w.base + (uint32_t)(c1 - cut)];
      }
      const uint32_t la = pa1 - pa0, lb = pb1 - pb0;
      ncand += la + lb;
      // fp32 brackets of the two pieces' first columns (fp64, rounded once; pinned in registers so the
      // compiler does not re-derive them per candidate); per element only (column - first) w0 is added
      float bxa, bxb;
      {
        double xa, xb;
        if (g.variant == 0) {
          xa = g.R[0] * ((double)(c0 - a0) * g.cinv[0]) + w.bxr;
          xb = g.R[0] * ((double)(cut - a0) * g.cinv[0]) + w.bxr;
        } else {
          xa = ((double)(c0 - a0) * g.w[0] + (double)n1a * g.e[0]) + w.bxr;
          xb = ((double)(cut - a0) * g.w[0] + (double)(n1a + 1) * g.e[0]) + w.bxr;
        }
        asm volatile("mov.b32 %0, %1;" : "=f"(bxa) : "f"((float)xa));
        asm volatile("mov.b32 %0, %1;" : "=f"(bxb) : "f"((float)xb));
      }
      const float byf = w.byf, bzf = w.bzf;
      const float firstaf = (float)(c0 - n1a * l1);  // piece a's first wrapped column (piece b: column 0)
      // queue code of a hit: its unwrapped column delta d0 = column + n1 l1 - a0 (16 bits) and the row
      const int ka = n1a * l1 - a0 + 32768 + (ri << 16), kb = ka + l1;
      const int lmax = (int)__reduce_max_sync(0xffffffffu, la + lb);
      for (int k0 = 0; k0 < lmax; k0 += SP_UNR) {
        if (__any_sync(0xffffffffu, nq > SP_QCAP - SP_UNR)) {
          sp_eval<DIGEST>(g, sm, u, qs, nh, gid, nq, tid, me, nh_i, lo64, hi64, po, gi, a0, a1, grp, wid, layer);
          nq = 0;
          qa = qa0;
        }
        float4 v[SP_UNR];
        uint32_t jv[SP_UNR];
#pragma unroll
        for (int h = 0; h < SP_UNR; ++h) {  // SP_UNR loads in flight before the first use
          const uint32_t k = (uint32_t)(k0 + h);
          jv[h] = k >= la ? pb0 + (k - la) : pa0 + k;
          v[h] = u32[k < la + lb ? jv[h] : me];
        }
#pragma unroll
        for (int h = 0; h < SP_UNR; ++h) {
          const uint32_t k = (uint32_t)(k0 + h);
          const bool inb = k >= la;
          const bool valid = k < la + lb;
          // j's cell column (wrapped; exact in .w) relative to its piece's first column, times w0
          const float bx = fmaf(v[h].w - (inb ? 0.0f : firstaf), w0x, inb ? bxb : bxa);
          const float dx = (v[h].x + bx) - ui32.x, dy = (v[h].y + byf) - ui32.y, dz = (v[h].z + bzf) - ui32.z;
          const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
          const bool hit = valid && jv[h] != me && r2 < hi32;
          if (hit) {
            stsu(qa, jv[h]);
            stsu(qa + SP_QD, (uint32_t)((int)v[h].w + (inb ? kb : ka)));
          }
          qa += hit ? 4u * SP_NT : 0u;
          nq += hit ? 1 : 0;
        }
      }
    }
    sp_eval<DIGEST>(g, sm, u, qs, nh, gid, nq, tid, me, nh_i, lo64, hi64, po, gi, a0, a1, grp, wid, layer);
    Acc acc;
    acc.fx = sm.acc[0][tid]; acc.fy = sm.acc[1][tid]; acc.fz = sm.acc[2][tid]; acc.u = sm.acc[3][tid];
    acc.w0 = sm.acc[4][tid]; acc.w1 = sm.acc[5][tid]; acc.w2 = sm.acc[6][tid];
    acc.w3 = sm.acc[7][tid]; acc.w4 = sm.acc[8][tid]; acc.w5 = sm.acc[9][tid];
    acc.cnt = sm.cnt[tid]; acc.nrc = sm.nrc[tid];
    if (DIGEST) { acc.hs = sm.hs[tid]; acc.hx = sm.hx[tid]; }
    if (LPP > 1) {  // the owner adds its siblings' partial sums in fixed order (sp_eval ended in __syncwarp)
      if (act && sub == 0) {
#pragma unroll
        for (int k = 1; k < LPP; ++k) {
          const int o = tid + k;
          NC_CHECK(o < SP_NT && (o >> 5) == (tid >> 5));
          acc.fx += sm.acc[0][o]; acc.fy += sm.acc[1][o]; acc.fz += sm.acc[2][o]; acc.u += sm.acc[3][o];
          acc.w0 += sm.acc[4][o]; acc.w1 += sm.acc[5][o]; acc.w2 += sm.acc[6][o];
          acc.w3 += sm.acc[7][o]; acc.w4 += sm.acc[8][o]; acc.w5 += sm.acc[9][o];
          acc.cnt += sm.cnt[o]; acc.nrc += sm.nrc[o];
          if (DIGEST) { acc.hs += sm.hs[o]; acc.hx ^= sm.hx[o]; }
        }
      }
      if (act) tC += ncand;  // every thread its own rows' candidates (the self pair subtracted below)
      __syncwarp();  // the siblings' sums are read before the next batch clears them
    }
    if (act && sub == 0) {
      const double Ui = 2.0 * g.eps * acc.u - 0.5 * g.ushift * (double)acc.cnt;
      const float4 fv = make_float4((float)(g.Q[0] * acc.fx + g.Q[1] * acc.fy + g.Q[2] * acc.fz),
                                    (float)(g.Q[3] * acc.fx + g.Q[4] * acc.fy + g.Q[5] * acc.fz),
                                    (float)(g.Q[6] * acc.fx + g.Q[7] * acc.fy + g.Q[8] * acc.fz),
                                    __uint_as_float(acc.cnt));
      Fout[me] = fv;
      store_user_F(po, gid, me, fv);
      if (DIGEST) { dcnt[me] = acc.cnt; dhs[me] = acc.hs; dhx[me] = acc.hx; }
      sm.tuw[0][tid] += Ui;
      sm.tuw[1][tid] += 0.5 * acc.w0; sm.tuw[2][tid] += 0.5 * acc.w1; sm.tuw[3][tid] += 0.5 * acc.w2;
      sm.tuw[4][tid] += 0.5 * acc.w3; sm.tuw[5][tid] += 0.5 * acc.w4; sm.tuw[6][tid] += 0.5 * acc.w5;
      tI += acc.cnt;
      tR += acc.nrc;
      tC += (LPP > 1 ? 0u : ncand) - 1u;
      tNF += isfinite(acc.fx + acc.fy + acc.fz + Ui) ? 0u : 1u;
    }
  }
  // warp sums of the 13 partials by a transposing butterfly (16 slots: each step halves the slots a
  // lane carries; 16 shuffles instead of 13 x 5); lane l ends with slot (l >> 1) & 15, fixed order
  double v[16] = {sm.tuw[0][tid], sm.tuw[1][tid], sm.tuw[2][tid], sm.tuw[3][tid], sm.tuw[4][tid], sm.tuw[5][tid],
                  sm.tuw[6][tid], (double)tI, (double)tC, (double)tS, (double)tR, 0.0, (double)tNF, 0.0, 0.0, 0.0};
  // (slot 11: the fp32-tier count -- every interaction of this kernel is evaluated in fp64)
#pragma unroll
  for (int o = 16, m = 8; o >= 2; o >>= 1, m >>= 1) {
    const bool hi = (lane & o) != 0;
#pragma unroll
    for (int k = 0; k < m; ++k) {
      const double keep = hi ? v[k + m] : v[k], send = hi ? v[k] : v[k + m];
      v[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
  static_assert(NPART == 13, "slot layout");
  if ((lane & 1) == 0 && (lane >> 1) < NPART) sm.part[wid][lane >> 1] = v[0];
  __syncthreads();
  if (tid < NPART) {  // fixed-order combine of the warps
    double sum = 0.0;
    for (int w = 0; w < SP_NT / 32; ++w) sum += sm.part[w][tid];
    bpart[(int64_t)blockIdx.x * NPART + tid] = sum;
  }
  PDL_LAUNCH();
}

}  // namespace nc
