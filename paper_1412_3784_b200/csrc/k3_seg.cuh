// k3_seg.cuh -- K3 for sparse cells (WCA: ~1.3 particles per cell), NC_F32.
// Included at the end of kernels.cuh.
//
// The warp-per-cell kernel (k_pairs) spends almost all of its time on the
// per-cell neighborhood setup when a cell holds ~1 particle.  Here one warp
// owns a SEGMENT of G consecutive cells of one row (same a1, a2) and builds
// the UNION of their neighborhoods once: the stencil rows of the segment
// (9 DS rows; up to 12 DO rows by the exact interval rule R4,
// P:673-687), each row's union column range, the neighbor particles staged
// in shared memory in the segment's frame (cell-local coordinates plus the
// column's image bracket).  Every lane owns one particle i of the segment and
// scans exactly its own cell's neighborhood -- the same 27 (DS) or 27/30/34/36
// (DO) cells as k_pairs, row by row, as contiguous sub-ranges of the staged
// union -- so the candidate set, the pair set and every count are those of
// the method.  Filter in fp32 (difference form), superset band as k_pairs;
// every survivor is evaluated in fp64 from the fp64 cell-local coordinates
// (WCA pairs all lie below r_split), membership inside the 1e-12 band by the
// canonical R16 test.  Full i-side accumulation, no atomics, layer-aligned
// deterministic block partials (one block = one segment).
#pragma once

namespace nc {

constexpr int SG_ROWS = 12;                 // stencil rows (DS 9, DO <= 12)
constexpr int SG_QCAP = 32;                 // per-lane hit queue
// NW warps per block share one staged union: 2 (segments of 48 cells) or 4 (96 cells, large grids)
template <int NW>
struct SgCfg {
  static constexpr int NT = 32 * NW;
  static constexpr int CAP = 384 * NW;          // staged union elements
  static constexpr int GMAX = 24 * NW;          // cells per segment
  static constexpr int MAXE = SG_ROWS * (GMAX + 4);  // union entries (row x column)
};

template <int NW>
struct SgSmem {
  float4 stage[SgCfg<NW>::CAP];                     // segment-frame x, y, z; w = sorted index bits
  uint32_t e_start[SgCfg<NW>::MAXE];                // first sorted particle of the entry's cell
  uint16_t e_off[SgCfg<NW>::MAXE + 1];              // staging offset of the entry
  uint16_t sent[SgCfg<NW>::CAP];                    // entry of each staged element
  uint8_t e_row[SgCfg<NW>::MAXE];
  uint8_t e_ci[SgCfg<NW>::MAXE];                    // column index inside the row's union range
  int8_t e_nx[SgCfg<NW>::MAXE];                     // x image shift floor(col / l1) of the entry's column
  uint16_t rg[SgCfg<NW>::GMAX][SG_ROWS][2];         // per cell and row: staged sub-range [st, en)
  uint16_t queue[NW][SG_QCAP][32];
  uint32_t wtot[NW][SG_ROWS];            // per-warp row totals (block scan)
  double part[NW][NPART];                // per-warp partials (fixed-order combine)
  uint32_t cst[SgCfg<NW>::GMAX];                    // first sorted particle of each segment cell
  uint16_t ct0[SgCfg<NW>::GMAX];                    // staged offset of each segment cell
  uint16_t nsz[SgCfg<NW>::GMAX];                    // neighborhood size (cells) of each segment cell
  // rows
  int r_lo[SG_ROWS], r_n[SG_ROWS], r_eb[SG_ROWS + 1], r_base[SG_ROWS];
  int r_ny[SG_ROWS], r_nz[SG_ROWS];         // image shifts of the row (DO n2, n3; DS n1, n2)
  double r_ox[SG_ROWS];                     // DO: row x offset in cell units (n3 d31 + n2 d21)
  double r_b[SG_ROWS][3];                   // row part of the bracket (fp64)
  float r_bf[SG_ROWS][3];
  int nrows, r0;                            // row count; the center row (dy = dz = 0)
};

// Stencil rows of the segment [A, A+G) in row (a1, a2): union column ranges, brackets,
// staged union, per-cell sub-ranges.  All SG_NT threads of the block call it.  Returns
// false (uniformly) if the union holds more than SG_CAP elements (caller shrinks G).
template <int NW>
__device__ bool sg_setup(const Geom& g, const uint32_t* __restrict__ cs, const float4* __restrict__ u32, int A, int G,
                         int a1, int a2, SgSmem<NW>& sm, int tid) {
  constexpr int SG_NT = SgCfg<NW>::NT, SG_CAP = SgCfg<NW>::CAP, SG_GMAX = SgCfg<NW>::GMAX,
                SG_MAXE = SgCfg<NW>::MAXE, SG_NW = NW;
  const int l1 = g.dims[0], l2 = g.dims[1], l3 = g.dims[2];
  const int lane = tid & 31, wid = tid >> 5;
  // ---- rows (warp 0)
  if (wid == 0) {
    bool valid = false;
    int lo = 0, n = 0, ny = 0, nz = 0, base = 0;
    double ox = 0.0, b0 = 0.0, b1 = 0.0, b2 = 0.0;
    bool center = false;
    if (g.variant == 0) {
      if (lane < 9) {
        const int d1 = lane % 3 - 1, d2 = lane / 3 - 1;
        int m1 = a1 + d1, m2 = a2 + d2;
        ny = floordiv(m1, l2);
        nz = floordiv(m2, l3);
        m1 -= ny * l2;
        m2 -= nz * l3;
        base = l1 * (m1 + l2 * m2);
        lo = A - 1;
        n = G + 2;
        const double v1 = (double)d1 * g.cinv[1], v2 = (double)d2 * g.cinv[2];
        b0 = g.R[1] * v1 + g.R[2] * v2;
        b1 = g.R[4] * v1 + g.R[5] * v2;
        b2 = g.R[8] * v2;
        valid = true;
        center = (d1 == 0 && d2 == 0);
      }
    } else {
      if (lane < 12) {
        const int dz = lane / 4 - 1, ri = lane % 4;
        const int kk = a2 + dz;
        const int n3 = floordiv(kk, l3);
        const int kd = kk - n3 * l3;
        const double oy = __dmul_rn((double)n3, g.d32);
        const int m0 = (int)floor(__dsub_rn((double)(a1 - 1), oy));
        const int m1 = (int)ceil(__dsub_rn((double)(a1 + 2), oy));
        if (ri < m1 - m0) {
          const int m = m0 + ri;
          const int n2 = floordiv(m, l2);
          const int jd = m - n2 * l2;
          ox = __dadd_rn(__dmul_rn((double)n3, g.d31), __dmul_rn((double)n2, g.d21));
          // union of [floor(a0 - 1 - ox), ceil(a0 + 2 - ox)) over a0 in [A, A+G) (build_entries' expressions)
          lo = (int)floor(__dsub_rn((double)(A - 1), ox));
          const int hi = (int)ceil(__dsub_rn((double)(A + G - 1 + 2), ox));
          n = hi - lo;
          ny = n2;
          nz = n3;
          base = l1 * (jd + l2 * kd);
          b0 = (double)n2 * g.R[1] + (double)n3 * g.R[2];
          b1 = (double)(m - a1) * g.w[1] + (double)n2 * g.e[1] + (double)n3 * g.R[5];
          b2 = (double)dz * g.w[2] + (double)n3 * g.e[2];
          valid = true;
          center = (dz == 0 && m == a1);
        }
      }
    }
    const unsigned vm = __ballot_sync(0xffffffffu, valid);
    const int ridx = __popc(vm & ((1u << lane) - 1u));
    const int ncols = valid ? n : 0;
    int x = ncols;
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (valid) {
      sm.r_lo[ridx] = lo; sm.r_n[ridx] = n; sm.r_eb[ridx] = x - ncols; sm.r_base[ridx] = base;
      sm.r_ny[ridx] = ny; sm.r_nz[ridx] = nz; sm.r_ox[ridx] = ox;
      sm.r_b[ridx][0] = b0; sm.r_b[ridx][1] = b1; sm.r_b[ridx][2] = b2;
      sm.r_bf[ridx][0] = (float)b0; sm.r_bf[ridx][1] = (float)b1; sm.r_bf[ridx][2] = (float)b2;
      if (center) sm.r0 = ridx;
    }
    const int nrows_w = __popc(vm);
    const int E_w = __shfl_sync(0xffffffffu, x, 15);
    if (lane == 0) { sm.nrows = nrows_w; sm.r_eb[nrows_w] = E_w; }
  }
  __syncthreads();
  const int nrows = sm.nrows;
  const int E = sm.r_eb[nrows];
  if (E > SG_MAXE) return false;
  // ---- entries (row, column), row-major: thread tid owns column tid of every row (a row spans at
  // most G + 4 <= SG_NT columns).  All cell-start loads first; then per-row warp scans and one
  // barrier give every entry's staging offset (entries numbered row by row, e = r_eb[r] + ci).
  static_assert(SG_GMAX + 4 <= SG_NT, "a union row must fit one column per thread");
  uint32_t est[SG_ROWS], ecn[SG_ROWS];
#pragma unroll
  for (int r = 0; r < SG_ROWS; ++r) {
    est[r] = 0u;
    ecn[r] = 0u;
    if (r < nrows && tid < sm.r_n[r]) {
      const int col = sm.r_lo[r] + tid;
      const int nx = floordiv(col, l1);
      const uint32_t cell = (uint32_t)sm.r_base[r] + (uint32_t)(col - nx * l1);
      sm.e_nx[sm.r_eb[r] + tid] = (int8_t)nx;
      est[r] = cs[cell];
      ecn[r] = cs[cell + 1];
      const int e = sm.r_eb[r] + tid;
      sm.e_row[e] = (uint8_t)r;
      sm.e_ci[e] = (uint8_t)tid;
    }
  }
  uint32_t incl[SG_ROWS];
#pragma unroll
  for (int r = 0; r < SG_ROWS; ++r) {
    uint32_t y = ecn[r] - est[r];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t z = __shfl_up_sync(0xffffffffu, y, o);
      if (lane >= o) y += z;
    }
    incl[r] = y;
    if (lane == 31) sm.wtot[wid][r] = y;
  }
  __syncthreads();
  uint32_t tot = 0;
#pragma unroll
  for (int r = 0; r < SG_ROWS; ++r) {
    if (r >= nrows) break;
    uint32_t before = tot, rowtot = 0;
#pragma unroll
    for (int w = 0; w < SG_NW; ++w) {
      const uint32_t v = sm.wtot[w][r];
      if (w < wid) before += v;
      rowtot += v;
    }
    if (tid < sm.r_n[r]) {
      const int e = sm.r_eb[r] + tid;
      sm.e_start[e] = est[r];
      sm.e_off[e] = (uint16_t)min(before + incl[r] - (ecn[r] - est[r]), 65535u);
    }
    tot += rowtot;
  }
  if (tid == 0) sm.e_off[E] = (uint16_t)min(tot, 65535u);
  __syncthreads();
  if (tot > (uint32_t)SG_CAP) return false;
  // ---- staged element -> entry, then the coalesced copy with the bracket in the segment frame
  for (int e = tid; e < E; e += SG_NT)
    for (uint32_t k = sm.e_off[e]; k < sm.e_off[e + 1]; ++k) sm.sent[k] = (uint16_t)e;
  __syncthreads();
  const float wx = g.variant == 0 ? (float)(g.R[0] * g.cinv[0]) : (float)g.w[0];
  const float ex = g.variant == 0 ? 0.0f : (float)g.e[0];
  for (uint32_t t0 = 0; t0 < tot; t0 += 4 * SG_NT) {
    uint32_t tt[4], jj[4];
    int ee[4];
    float4 pp[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      tt[r] = t0 + (uint32_t)(SG_NT * r + tid);
      const bool v = tt[r] < tot;
      ee[r] = v ? sm.sent[tt[r]] : 0;
      jj[r] = sm.e_start[ee[r]] + tt[r] - sm.e_off[ee[r]];
      pp[r] = v ? u32[jj[r]] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      if (tt[r] < tot) {
        const int row = sm.e_row[ee[r]];
        const int col = sm.r_lo[row] + sm.e_ci[ee[r]];
        const int nx = sm.e_nx[ee[r]];
        const float bx = (float)(col - A) * wx + (float)nx * ex + sm.r_bf[row][0];
        sm.stage[tt[r]] = make_float4(pp[r].x + bx, pp[r].y + sm.r_bf[row][1], pp[r].z + sm.r_bf[row][2],
                                      __uint_as_float(jj[r]));
      }
    }
  }
  // ---- per cell and row: the cell's own sub-range of the union row (exact stencil of k_pairs)
  if (tid < G) {
    const int a0 = A + tid;
    int ns = 0;
    for (int r = 0; r < nrows; ++r) {
      int c0, c1;
      if (g.variant == 0) {
        c0 = a0 - 1;
        c1 = a0 + 2;
      } else {
        c0 = (int)floor(__dsub_rn((double)(a0 - 1), sm.r_ox[r]));
        c1 = (int)ceil(__dsub_rn((double)(a0 + 2), sm.r_ox[r]));
      }
      if (r == nrows - 1) c1 -= g.dbg_drop;  // negative control (nc_debug): the last entry of build_entries
      ns += c1 - c0;
      const int eb = sm.r_eb[r] - sm.r_lo[r];
      sm.rg[tid][r][0] = sm.e_off[eb + c0];
      sm.rg[tid][r][1] = sm.e_off[eb + c1];
    }
    sm.nsz[tid] = (uint16_t)ns;
    const int ec = sm.r_eb[sm.r0] - sm.r_lo[sm.r0] + a0;
    sm.cst[tid] = sm.e_start[ec];
    sm.ct0[tid] = sm.e_off[ec];
  }
  __syncthreads();
  return true;
}

// fp64 evaluation of one lane's queued staged indices (four per iteration, global loads first).
template <bool DIGEST, int NW>
__device__ __forceinline__ void sg_eval(const Geom& g, const SgSmem<NW>& sm, const double4* __restrict__ u,
                                        const float4* __restrict__ qs, const uint32_t* __restrict__ nh,
                                        const uint32_t* __restrict__ gid, uint32_t qb, int nq, uint32_t me,
                                        uint32_t nh_i, int A, double uix, double uiy, double uiz, double wx64,
                                        double lo64, double hi64, Acc& acc, const PairOut& po, uint32_t gi) {
  const int qmax = __reduce_max_sync(0xffffffffu, nq);
  const double sig2 = g.sig2, eps24 = 24.0 * g.eps;
  for (int q0 = 0; q0 < qmax; q0 += 4) {
    uint32_t jj[4];
    int ee[4];
    bool ok0[4];
    double4 uj[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      ok0[h] = q0 + h < nq;
      const uint32_t tq = ok0[h] ? lds16(qb + 64u * (uint32_t)(q0 + h)) : 0u;
      jj[h] = ok0[h] ? __float_as_uint(sm.stage[tq].w) : me;
      ee[h] = sm.sent[tq];
      uj[h] = u[jj[h]];
    }
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const uint32_t j = jj[h];
      const int row = sm.e_row[ee[h]];
      const int col = sm.r_lo[row] + sm.e_ci[ee[h]];
      const int nx = sm.e_nx[ee[h]];
      const double bx = (double)(col - A) * wx64 + (g.variant == 1 ? (double)nx * g.e[0] : 0.0) + sm.r_b[row][0];
      const double dx = (uj[h].x + bx) - uix, dy = (uj[h].y + sm.r_b[row][1]) - uiy,
                   dz = (uj[h].z + sm.r_b[row][2]) - uiz;
      const double r2 = dx * dx + dy * dy + dz * dz;
      bool ok = ok0[h] && (j != me) && (r2 < hi64);
      int n0 = 0, n1 = 0, n2 = 0;
      if (ok && (DIGEST || r2 >= lo64)) {
        n0 = nx;
        n1 = sm.r_ny[row];
        n2 = sm.r_nz[row];
        if (g.variant == 1) {
          const uint32_t nh_j = nh[j];
          n0 += nh_x(nh_j) - nh_x(nh_i);
          n1 += nh_y(nh_j) - nh_y(nh_i);
        }
        if (r2 >= lo64) {
          const float4 qi = qs[me], qj = qs[j];
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
      if (DIGEST && ok) digest_add<DIGEST>(acc, gid, j, n0, n1, n2, po, gi);
    }
  }
  __syncwarp();
}

template <bool DIGEST, int NW>
__global__ void __launch_bounds__(32 * NW, 16 / NW)
k_pairs_seg(const double4* __restrict__ u, const float4* __restrict__ u32, const uint32_t* __restrict__ cs,
            const float4* __restrict__ qs, const uint32_t* __restrict__ nh, const uint32_t* __restrict__ gid,
            float4* __restrict__ Fout, double* __restrict__ bpart, uint32_t* __restrict__ dcnt,
            uint64_t* __restrict__ dhs, uint64_t* __restrict__ dhx, const __grid_constant__ Geom g, int G, int nseg,
            int bpl, int layer0, const PairOut po) {
  PDL_WAIT();  // (the successor is released at the end)
  extern __shared__ __align__(16) unsigned char smraw[];
  constexpr int SG_NT = SgCfg<NW>::NT, SG_CAP = SgCfg<NW>::CAP, SG_NW = NW;
  (void)SG_NT;
  SgSmem<NW>& sm = *reinterpret_cast<SgSmem<NW>*>(smraw);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int l1 = g.dims[0];
  const int layer = layer0 + (int)(blockIdx.x / bpl);
  const int rem = (int)blockIdx.x - (layer - layer0) * bpl;
  const int a1 = rem / nseg, a2 = layer;
  const int Abeg = (rem - a1 * nseg) * G;
  const int Aend = min(l1, Abeg + G);
  const double lo64 = g.rc2 * (1.0 - K3_BAND64), hi64 = g.rc2 * (1.0 + K3_BAND64);
  const float hi32 = (float)g.band_hi;
  const double wx64 = g.variant == 0 ? g.R[0] * g.cinv[0] : g.w[0];
  const uint32_t qb = smem_u32(&sm.queue[wid][0][lane]);
  const uint32_t stage0 = smem_u32(&sm.stage[0]);

  double tU = 0, tW[6] = {0, 0, 0, 0, 0, 0}, tI = 0, tC = 0, tS = 0, tR = 0, tNF = 0;

  int A = Abeg;
  while (A < Aend) {
    int Gs = Aend - A;
    while (!sg_setup<NW>(g, cs, u32, A, Gs, a1, a2, sm, tid)) {
      if (Gs == 1) { Gs = 0; break; }  // a single cell's neighborhood above SG_CAP: flagged below
      Gs = (Gs + 1) / 2;
    }
    if (Gs == 0) {  // cannot stage (cells of > ~20 particles): the host fails loudly (NC_E_OOM)
      tNF += (tid == 0) ? K3_OVERFLOW : 0.0;
      A += 1;
      continue;
    }
    const int nrows = sm.nrows;
    // neighborhood size of every cell (instrumentation: k_pairs' tS)
    if (tid < Gs) tS += (double)sm.nsz[tid];
    // particles of the segment: contiguous in the center row
    const int ecA = sm.r_eb[sm.r0] - sm.r_lo[sm.r0] + A;
    const uint32_t P0 = sm.e_start[ecA];
    const uint32_t P1 = sm.e_start[ecA + Gs - 1] + (uint32_t)(sm.e_off[ecA + Gs] - sm.e_off[ecA + Gs - 1]);
    // each warp takes a contiguous share of the segment's particles (balanced across the block)
    const uint32_t per = (P1 - P0 + SG_NW - 1) / SG_NW;
    const uint32_t W0 = min(P1, P0 + per * (uint32_t)wid), W1 = min(P1, W0 + per);
    for (uint32_t pb = W0; pb < W1; pb += 32u) {
      const uint32_t p = pb + (uint32_t)lane;
      const bool act = p < W1;
      // cell of p inside the segment
      int gc = 0;
      if (act) {
        int lo_ = 0, hi_ = Gs - 1;
        while (lo_ < hi_) {
          const int mid = (lo_ + hi_ + 1) >> 1;
          if (sm.cst[mid] <= p) lo_ = mid; else hi_ = mid - 1;
        }
        // skip empty cells that share the start
        gc = lo_;
      }
      const uint32_t ti = sm.ct0[gc] + (p - sm.cst[gc]);
      const float4 vi = sm.stage[act ? ti : 0];
      // i in the segment frame, fp64
      const uint32_t me = act ? p : 0u;
      const double4 ui = u[me];
      const double uix = ui.x + (double)(A + gc - A) * wx64, uiy = ui.y, uiz = ui.z;
      const uint32_t nh_i = (g.variant == 1 && act) ? nh[me] : 0u;
      const uint32_t gi = DIGEST ? gid[me] : 0u;
      // candidates of i: its cell's stencil minus itself
      int T = 0;
      if (act)
        for (int r = 0; r < nrows; ++r) T += sm.rg[gc][r][1] - sm.rg[gc][r][0];
      if (act) tC += (double)(T - 1);
      Acc acc = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0u, 0u, 0ull, 0ull};
      // filter: rows in order; every lane scans its own cell's contiguous sub-range of the row
      // (uniform trip count = the warp's longest sub-range, predicated per lane)
      int nq = 0;
      for (int r = 0; r < nrows; ++r) {
        const uint32_t st = act ? sm.rg[gc][r][0] : 0u, en = act ? sm.rg[gc][r][1] : 0u;
        const int len = (int)(en - st);
        const int lmax = __reduce_max_sync(0xffffffffu, len);
        for (int k0 = 0; k0 < lmax; k0 += 8) {
          if (__any_sync(0xffffffffu, nq > SG_QCAP - 8)) {  // room for 8 more hits in every queue
            sg_eval<DIGEST, NW>(g, sm, u, qs, nh, gid, qb, nq, me, nh_i, A, uix, uiy, uiz, wx64, lo64, hi64, acc, po, gi);
            nq = 0;
          }
          const int kend = min(lmax, k0 + 8);
          for (int k = k0; k < kend; ++k) {
            const uint32_t t = st + (uint32_t)k;
            const float4 v = lds128(stage0 + 16u * min(t, (uint32_t)(SG_CAP - 1)));
            const float dx = v.x - vi.x, dy = v.y - vi.y, dz = v.z - vi.z;
            const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
            const bool hit = (k < len) && (r2 < hi32) && (t != ti);
            sts16(qb + 64u * (uint32_t)nq, t);  // nq <= SG_QCAP - 1 here
            nq += hit ? 1 : 0;
          }
        }
      }
      sg_eval<DIGEST, NW>(g, sm, u, qs, nh, gid, qb, nq, me, nh_i, A, uix, uiy, uiz, wx64, lo64, hi64, acc, po, gi);
      const double fx = acc.fx, fy = acc.fy, fz = acc.fz, uu = acc.u;
      const double w0 = acc.w0, w1 = acc.w1, w2 = acc.w2, w3 = acc.w3, w4 = acc.w4, w5 = acc.w5;
      const uint32_t cnt = acc.cnt, nrc = acc.nrc;
      const uint64_t hs = acc.hs, hx = acc.hx;
      if (act) {
        const double Ui = 2.0 * g.eps * uu - 0.5 * g.ushift * (double)cnt;
        const float4 fv = make_float4((float)(g.Q[0] * fx + g.Q[1] * fy + g.Q[2] * fz),
                                      (float)(g.Q[3] * fx + g.Q[4] * fy + g.Q[5] * fz),
                                      (float)(g.Q[6] * fx + g.Q[7] * fy + g.Q[8] * fz), __uint_as_float(cnt));
        Fout[me] = fv;
        store_user_F(po, gid, me, fv);
        if (DIGEST) { dcnt[me] = cnt; dhs[me] = hs; dhx[me] = hx; }
        tU += Ui;
        tW[0] += 0.5 * w0; tW[1] += 0.5 * w1; tW[2] += 0.5 * w2;
        tW[3] += 0.5 * w3; tW[4] += 0.5 * w4; tW[5] += 0.5 * w5;
        tI += (double)cnt;
        tR += (double)nrc;
        tNF += isfinite(fx + fy + fz + Ui) ? 0.0 : 1.0;
      }
    }
    A += Gs;
    __syncthreads();  // the next sub-segment overwrites the staged union
  }
  tU = warp_sum_d(tU);
  tW[0] = warp_sum_d(tW[0]); tW[1] = warp_sum_d(tW[1]); tW[2] = warp_sum_d(tW[2]);
  tW[3] = warp_sum_d(tW[3]); tW[4] = warp_sum_d(tW[4]); tW[5] = warp_sum_d(tW[5]);
  tI = warp_sum_d(tI);
  tC = warp_sum_d(tC);
  tS = warp_sum_d(tS);
  tR = warp_sum_d(tR);
  tNF = warp_sum_d(tNF);
  if (lane < NPART) {
    double v = 0;
    if (lane == 0) v = tU;
    else if (lane <= 6) v = tW[lane - 1];
    else if (lane == 7) v = tI;
    else if (lane == 8) v = tC;
    else if (lane == 9) v = tS;
    else if (lane == 10) v = tR;
    else if (lane == 11) v = 0.0;  // every interaction of this kernel is evaluated in fp64
    else v = tNF;
    sm.part[wid][lane] = v;
  }
  __syncthreads();
  if (tid < NPART) {  // fixed-order combine of the warps
    double v = 0.0;
    for (int w = 0; w < SG_NW; ++w) v += sm.part[w][tid];
    bpart[(int64_t)blockIdx.x * NPART + tid] = v;
  }
  PDL_LAUNCH();
}

}  // namespace nc
