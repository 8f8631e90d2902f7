// k3_rows.cuh -- K3 for sparse cells (WCA at rho = 0.8442: ~1.3 particles per cell), NC_F32:
// one warp per CELL ROW, the row's particles in batches of 32 consecutive ones, each batch's
// neighbour rows staged once in shared memory.  Included at the end of kernels.cuh.
//
// The method's loop is unchanged: every particle i visits exactly the
// cells of its own neighborhood -- 27 (DS) or 27/30/34/36 (DO, exact interval rule) -- and checks
// every particle j in them.  What changes against k_pairs_sparse is where j comes from.  A batch of
// 32 consecutive particles of one cell row (a1, a2) spans ~25 cells along x; in each of the <= 12
// stencil rows (same dy, dz for the whole batch) the union of the lanes' column windows is ONE
// contiguous column interval [cl, ch) (two pieces when it wraps in x), i.e. one or two contiguous
// ranges of the (cell, gid)-sorted arrays.  Those ranges are copied once into shared memory in the
// batch's frame (cell-local coordinates + the row / column bracket relative to the corner of cell
// (A_ref, a1, a2), A_ref the batch's middle column), so the candidate loop is a shared-memory load and
// the fp32 distance test; lane i's own stencil cells in a row are a contiguous sub-range (window) of
// the staged row.  Survivors (superset band as everywhere) are evaluated in fp64 from the fp64
// cell-local coordinates with sp_bracket -- the same expressions, in the same candidate order, as
// k_pairs_sparse, so per-particle forces are bitwise those of that kernel -- with the canonical R16
// test inside the 1e-12 band.  Full i-side accumulation, no atomics.  Block partials: RW_NW
// consecutive cell rows of ONE layer (layer-aligned, a function of the grid only: P-invariant).
#pragma once

namespace nc {

#ifndef NC_RW_NW
#define NC_RW_NW 4
#endif
#ifndef NC_RW_CAP
#define NC_RW_CAP 512
#endif
#ifndef NC_RW_MINB
#define NC_RW_MINB 4
#endif
constexpr int RW_NW = NC_RW_NW;    // warps (cell rows) per block
constexpr int RW_CAP = NC_RW_CAP;  // staged elements per warp (a batch's rows are staged in groups that fit)
constexpr int RW_QCAP = 16;        // per-lane survivor queue
constexpr int RW_ROWS = 12;        // stencil rows (DS 9, DO <= 12)

struct RwWarp {
  float4 st[RW_CAP];              // batch frame x, y, z; w = sorted index bits
  uint32_t code[RW_CAP];          // unwrapped column - A_ref + 32768 | stencil row << 16
  uint16_t q[RW_QCAP][32];        // queued staged indices
  SpSmem::RowW rw[RW_ROWS];       // the a0-independent row data of this cell row (sp_row_inv)
  int S[RW_ROWS + 1];             // staged offset of each row of the batch (prefix over rows)
  int cut[RW_ROWS], nla[RW_ROWS];  // first unwrapped column of piece b; n1a l1 (column shift of piece a)
  uint32_t pa0[RW_ROWS], lena[RW_ROWS], pb0[RW_ROWS];  // piece a: sorted [pa0, pa0 + lena); piece b from pb0
  uint32_t win[RW_ROWS][32];      // each lane's window per row: staged start | length << 16
  float bxa[RW_ROWS], bxb[RW_ROWS];  // fp32 x bracket of the first column of piece a / b (batch frame)
  int cwa[RW_ROWS], n1a[RW_ROWS];    // wrapped first column of piece a; its x image n1
};
struct RwSmem {
  RwWarp w[RW_NW];
  double part[RW_NW][NPART];
};

// fp64 evaluation of one lane's queued staged indices (sp_eval's arithmetic, two per iteration)
template <bool DIGEST>
__device__ __forceinline__ void rw_eval(const Geom& g, const RwWarp& sm, const double4* __restrict__ u,
                                       const float4* __restrict__ qs, const uint32_t* __restrict__ nh,
                                       const uint32_t* __restrict__ gid, int nq, uint32_t qa0, uint32_t me,
                                       uint32_t nh_i, double uix, double uiy, double uiz, int a0, int Aref,
                                       double lo64, double hi64, Acc& acc, const PairOut& po, uint32_t gi) {
  const int qmax = __reduce_max_sync(0xffffffffu, nq);
  const double sig2 = g.sig2, eps24 = 24.0 * g.eps;
  for (int k0 = 0; k0 < qmax; k0 += 2) {
    uint32_t jj[2];
    SpCell cc[2];
    bool ok0[2];
    double4 uj[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      ok0[h] = k0 + h < nq;
      const uint32_t t = ok0[h] ? lds16(qa0 + 64u * (uint32_t)(k0 + h)) : 0u;
      jj[h] = ok0[h] ? __float_as_uint(sm.st[t].w) : me;
      const uint32_t code = ok0[h] ? sm.code[t] : (uint32_t)(32768 + a0 - Aref);
      const int ri = (int)((code >> 16) & 15u);
      const uint32_t meta = sm.rw[ri].meta;
      cc[h].d0 = (int)(code & 0xffffu) - 32768 + Aref - a0;
      cc[h].d1 = (int)((meta >> 1) & 0xffffu) - 32768;
      cc[h].n2 = (int)((meta >> 17) & 15u) - 8;
      cc[h].n3 = (int)((meta >> 21) & 15u) - 8;
      cc[h].d2 = (int)((meta >> 25) & 3u) - 2;
      cc[h].n1 = sm.n1a[ri] + (int)((code >> 20) & 1u);  // = floordiv(a0 + d0, l1): the piece's x image
      uj[h] = u[jj[h]];
    }
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
  __syncwarp();
}

// grid = nlay layers x bpl blocks, bpl = ceil(l2 / RW_NW); warp w of block b takes cell row
// a1 = b RW_NW + w of the layer (all its particles, batches of 32, and all its cells for the
// stencil-size statistic).
template <bool DIGEST>
__global__ void __launch_bounds__(32 * RW_NW, NC_RW_MINB)
k_pairs_rows(const double4* __restrict__ u, const float4* __restrict__ u32, const uint32_t* __restrict__ cs,
             const float4* __restrict__ qs, const uint32_t* __restrict__ nh, const uint32_t* __restrict__ gid,
             float4* __restrict__ Fout, double* __restrict__ bpart, uint32_t* __restrict__ dcnt,
             uint64_t* __restrict__ dhs, uint64_t* __restrict__ dhx, const __grid_constant__ Geom g, int bpl,
             int layer0, const PairOut po) {
  PDL_WAIT();  // (the successor is released at the end)
  extern __shared__ __align__(16) unsigned char rw_raw[];
  RwSmem& smb = *reinterpret_cast<RwSmem*>(rw_raw);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  RwWarp& sm = smb.w[wid];
  const int l1 = g.dims[0], l2 = g.dims[1];
  const int layer = layer0 + (int)(blockIdx.x / bpl);
  const int a1 = ((int)blockIdx.x - (layer - layer0) * bpl) * RW_NW + wid, a2 = layer;
  const double lo64 = g.rc2 * (1.0 - K3_BAND64), hi64 = g.rc2 * (1.0 + K3_BAND64);
  const float hi32 = (float)g.band_hi;
  const uint32_t st0 = smem_u32(&sm.st[0]);
  const uint32_t qa0 = smem_u32(&sm.q[0][lane]);

  double tU = 0, tW[6] = {0, 0, 0, 0, 0, 0}, tNF = 0;
  uint32_t tI = 0, tC = 0, tS = 0, tR = 0;

  if (a1 < l2) {  // (warp-uniform)
    if (lane < RW_ROWS) sp_row_inv(g, lane, a1, a2, sm.rw[lane]);
    __syncwarp();
    // the last existing row (its last column is dropped in the negative-control mode, nc_debug)
    int last_ri = 0;
#pragma unroll
    for (int r = 0; r < RW_ROWS; ++r)
      if (sm.rw[r].meta & 1u) last_ri = r;
    // stencil sizes of the row's cells (empty ones included): a row's width c1 - c0 is 3 for an integral
    // ox (DS: ox = 0), else 4, unless ox lies within 2^-30 of an integer (then per cell, sp_row's expressions)
    {
      int wcode = 0;
      if (lane < RW_ROWS && (sm.rw[lane].meta & 1u)) {
        const double ox = sm.rw[lane].ox, f = ox - floor(ox);
        wcode = f == 0.0 ? 3 : (fmin(f, 1.0 - f) > 0x1p-30 ? 4 : 64);
      }
      const int tot = (int)__reduce_add_sync(0xffffffffu, (uint32_t)wcode);
      if (tot < 64) {
        if (lane == 0) tS += (uint32_t)l1 * (uint32_t)(tot - g.dbg_drop);
      } else {
        for (int a0 = lane; a0 < l1; a0 += 32) {
          int ns = 0;
          for (int r = 0; r < RW_ROWS; ++r) {
            const SpSmem::RowW& w = sm.rw[r];
            if (w.meta & 1u)
              ns += (int)ceil(__dsub_rn((double)(a0 + 2), w.ox)) - (int)floor(__dsub_rn((double)(a0 - 1), w.ox));
          }
          tS += (uint32_t)(ns - g.dbg_drop);
        }
      }
    }
    const uint32_t rowc = (uint32_t)l1 * ((uint32_t)a1 + (uint32_t)l2 * (uint32_t)a2);
    const uint32_t R0 = cs[rowc], R1 = cs[rowc + (uint32_t)l1];
    const bool ds = g.variant == 0;
    const float w0x = (float)(ds ? g.R[0] * g.cinv[0] : g.w[0]);

    for (uint32_t pb = R0; pb < R1;) {
      int B = (int)min(32u, R1 - pb);
      uint32_t me = 0u;
      int a0 = 0, Aref = 0;
      bool act = false;
      bool overflow = false;
      // windows of every lane, the batch's union per row; halve the batch until every row's union fits
      // the staging buffer and stays inside one x period
      while (true) {
        act = lane < B;
        me = act ? pb + (uint32_t)lane : pb;
        a0 = (int)u32[me].w;  // the cell column (exact in .w)
        Aref = (__shfl_sync(0xffffffffu, a0, 0) + __shfl_sync(0xffffffffu, a0, B - 1)) >> 1;
        // the batch's union per row: a lane's columns [c0, c1) grow with its cell column a0, which is
        // non-decreasing over the lanes, so the union is [c0(first lane), c1(last lane))
        int mycl = 0, mych = 0;
        {
          const int aF = __shfl_sync(0xffffffffu, a0, 0), aL = __shfl_sync(0xffffffffu, a0, B - 1);
          if (lane < RW_ROWS) {
            const SpSmem::RowW& w = sm.rw[lane];
            mycl = (int)floor(__dsub_rn((double)(aF - 1), w.ox));
            mych = (int)ceil(__dsub_rn((double)(aL + 2), w.ox)) - (lane == last_ri ? g.dbg_drop : 0);
          }
        }
        // row lanes: pieces, their sorted ranges, the staged length
        int len = 0;
        bool fits = true;
        if (lane < RW_ROWS) {
          const SpSmem::RowW& w = sm.rw[lane];
          if ((w.meta & 1u) && mych > mycl) {
            const int n1a = floordiv(mycl, l1);
            const int cut = (n1a + 1) * l1;
            const int ea = min(mych, cut);
            const uint32_t pa0 = cs[w.base + (uint32_t)(mycl - n1a * l1)];
            const uint32_t pa1 = cs[w.base + (uint32_t)(ea - n1a * l1)];
            const uint32_t pb0 = cs[w.base];
            const uint32_t pb1 = mych > cut ? cs[w.base + (uint32_t)(mych - cut)] : pb0;
            len = (int)(pa1 - pa0 + pb1 - pb0);
            fits = (mych - mycl <= l1) && len <= RW_CAP;
            sm.cut[lane] = cut;
            sm.nla[lane] = n1a * l1;
            sm.n1a[lane] = n1a;
            sm.cwa[lane] = mycl - n1a * l1;
            // the row / column bracket of the pieces' first columns relative to the corner of cell
            // (Aref, a1, a2) in fp64 (build_entries' expressions), rounded once; per element only
            // (column - first) w0 is added in fp32 (k_pairs_sparse's staging arithmetic)
            double xa, xb;
            if (ds) {
              xa = g.R[0] * ((double)(mycl - Aref) * g.cinv[0]) + w.bxr;
              xb = g.R[0] * ((double)(cut - Aref) * g.cinv[0]) + w.bxr;
            } else {
              xa = ((double)(mycl - Aref) * g.w[0] + (double)n1a * g.e[0]) + w.bxr;
              xb = ((double)(cut - Aref) * g.w[0] + (double)(n1a + 1) * g.e[0]) + w.bxr;
            }
            sm.bxa[lane] = (float)xa;
            sm.bxb[lane] = (float)xb;
            sm.pa0[lane] = pa0;
            sm.lena[lane] = pa1 - pa0;
            sm.pb0[lane] = pb0;
          } else {
            sm.cut[lane] = 0x7fffffff;  // empty row: every window is empty
            sm.nla[lane] = 0;
            sm.n1a[lane] = 0;
            sm.cwa[lane] = 0;
            sm.bxa[lane] = sm.bxb[lane] = 0.0f;
            sm.pa0[lane] = 0u;
            sm.lena[lane] = 0u;
            sm.pb0[lane] = 0u;
          }
        }
        int x = len;  // exclusive scan over the 12 row lanes
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, x, o);
          if (lane >= o) x += y;
        }
        if (lane < RW_ROWS) sm.S[lane] = x - len;
        if (lane == RW_ROWS - 1) sm.S[RW_ROWS] = x;
        __syncwarp();
        if (__all_sync(0xffffffffu, fits)) {
          // this lane's window in every row: staged [S + idx(c0), S + idx(c1)), idx(c) = the staged
          // offset of column c's first particle (piece a: c < cut, piece b: c >= cut)
#pragma unroll
          for (int r = 0; r < RW_ROWS; ++r) {
            const SpSmem::RowW& w = sm.rw[r];
            uint32_t wv = 0u;
            if (act && (w.meta & 1u)) {
              const int cut = sm.cut[r], nla = sm.nla[r];
              const uint32_t pa0 = sm.pa0[r], lena = sm.lena[r], pb0 = sm.pb0[r];
              const int c0 = (int)floor(__dsub_rn((double)(a0 - 1), w.ox));
              const int c1 = (int)ceil(__dsub_rn((double)(a0 + 2), w.ox)) - (r == last_ri ? g.dbg_drop : 0);
              const uint32_t i0 = c0 < cut ? cs[w.base + (uint32_t)(c0 - nla)] - pa0
                                           : lena + cs[w.base + (uint32_t)(c0 - cut)] - pb0;
              const uint32_t i1 = c1 < cut ? cs[w.base + (uint32_t)(c1 - nla)] - pa0
                                           : lena + cs[w.base + (uint32_t)(c1 - cut)] - pb0;
              wv = ((uint32_t)sm.S[r] + i0) | ((i1 - i0) << 16);
            }
            sm.win[r][lane] = wv;
          }
          break;
        }
        __syncwarp();
        if (B == 1) { overflow = true; break; }  // one particle's neighbour row above RW_CAP
        B = (B + 1) >> 1;
      }
      if (overflow) {  // cannot stage (cells of > ~RW_CAP / 4 particles): the host fails loudly (NC_E_OOM)
        tNF += (lane == 0) ? K3_OVERFLOW : 0.0;
        pb += 1u;
        continue;
      }
      // i in the batch frame (corner of cell (Aref, a1, a2)): fp32 for the filter, fp64 cell-local for the
      // evaluation (sp_eval's frame)
      const float4 vi = u32[me];
      const double4 ui = u[me];
      const uint32_t nh_i = (g.variant == 1) ? nh[me] : 0u;
      const uint32_t gi = DIGEST ? gid[me] : 0u;
      const float xi = vi.x + (float)(ds ? g.R[0] * ((double)(a0 - Aref) * g.cinv[0]) : (double)(a0 - Aref) * g.w[0]);
      const float yi = vi.y, zi = vi.z;
      Acc acc = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0u, 0u, 0ull, 0ull};
      uint32_t ncand = 0;
      int nq = 0;
      // rows in groups that fit the staging buffer (normally all of them at once)
      int r0 = 0;
      while (r0 < RW_ROWS) {
        int r1 = RW_ROWS;
        if (sm.S[RW_ROWS] - sm.S[r0] > RW_CAP) {
          r1 = r0 + 1;
          while (r1 < RW_ROWS && sm.S[r1 + 1] - sm.S[r0] <= RW_CAP) ++r1;
        }
        const int gbase = sm.S[r0];
        // stage rows [r0, r1): element t of row r <- particle pa0 + t (piece a) / pb0 + t - lena (piece b),
        // x + the piece's bracket base + (column - first column) w0 in fp32; chunks of 32 elements of
        // RW_SR rows at a time (their global loads in flight together)
        constexpr int RW_SR = 6;
        int nmax = 0;
        for (int r = r0; r < r1; ++r) nmax = max(nmax, sm.S[r + 1] - sm.S[r]);
        for (int c = 0; c < nmax; c += 32) {
          for (int rb = r0; rb < r1; rb += RW_SR) {
            float4 v[RW_SR];
            uint32_t jv[RW_SR];
            bool ok[RW_SR];
#pragma unroll
            for (int h = 0; h < RW_SR; ++h) {
              const int r = min(rb + h, RW_ROWS - 1);
              const uint32_t t = (uint32_t)(c + lane);
              const uint32_t lena = sm.lena[r];
              ok[h] = rb + h < r1 && (int)t < sm.S[r + 1] - sm.S[r];
              jv[h] = t < lena ? sm.pa0[r] + t : sm.pb0[r] + (t - lena);
              v[h] = ok[h] ? u32[jv[h]] : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int h = 0; h < RW_SR; ++h) {
              if (ok[h]) {
                const int r = rb + h;
                const uint32_t t = (uint32_t)(c + lane);
                const bool inb = t >= sm.lena[r];
                const int colw = (int)v[h].w;  // wrapped column
                const float bx = fmaf((float)(colw - (inb ? 0 : sm.cwa[r])), w0x, inb ? sm.bxb[r] : sm.bxa[r]);
                const SpSmem::RowW& w = sm.rw[r];
                const int off = sm.S[r] - gbase + (int)t;
                NC_CHECK(off >= 0 && off < RW_CAP);
                sm.st[off] = make_float4(v[h].x + bx, v[h].y + w.byf, v[h].z + w.bzf, __uint_as_float(jv[h]));
                // unwrapped column - Aref (16 bits), stencil row, piece (its x image: n1a + inb)
                sm.code[off] = (uint32_t)(colw + (inb ? sm.cut[r] : sm.nla[r]) - Aref + 32768) | ((uint32_t)r << 16) |
                               (inb ? (1u << 20) : 0u);
              }
            }
          }
        }
        __syncwarp();
        // filter: rows in order, each lane over its own window (lockstep to the warp's longest window)
        for (int r = r0; r < r1; ++r) {
          const uint32_t wv = sm.win[r][lane];
          const int len = (int)(wv >> 16);
          const int s0 = (int)(wv & 0xffffu) - gbase;
          ncand += (uint32_t)len;
          const int lmax = __reduce_max_sync(0xffffffffu, len);
          for (int k = 0; k < lmax; k += 2) {
            if (__any_sync(0xffffffffu, nq > RW_QCAP - 2)) {
              rw_eval<DIGEST>(g, sm, u, qs, nh, gid, nq, qa0, me, nh_i, ui.x, ui.y, ui.z, a0, Aref, lo64, hi64, acc,
                              po, gi);
              nq = 0;
            }
            float4 v[2];
            int t[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              t[h] = k + h < len ? s0 + k + h : 0;
              NC_CHECK(t[h] >= 0 && t[h] < RW_CAP);
              v[h] = lds128(st0 + 16u * (uint32_t)t[h]);
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const float dx = v[h].x - xi, dy = v[h].y - yi, dz = v[h].z - zi;
              const float r2 = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
              const bool hit = (k + h < len) && (r2 < hi32) && (__float_as_uint(v[h].w) != me);
              NC_CHECK(nq < RW_QCAP);
              sts16(qa0 + 64u * (uint32_t)nq, (uint32_t)t[h]);  // nq <= RW_QCAP - 1 here
              nq += hit ? 1 : 0;
            }
          }
        }
        // the queue refers to the staged group: evaluate before restaging
        rw_eval<DIGEST>(g, sm, u, qs, nh, gid, nq, qa0, me, nh_i, ui.x, ui.y, ui.z, a0, Aref, lo64, hi64, acc, po,
                        gi);
        nq = 0;
        r0 = r1;
      }
      if (act) {
        const double Ui = 2.0 * g.eps * acc.u - 0.5 * g.ushift * (double)acc.cnt;
        const float4 fv = make_float4((float)(g.Q[0] * acc.fx + g.Q[1] * acc.fy + g.Q[2] * acc.fz),
                                      (float)(g.Q[3] * acc.fx + g.Q[4] * acc.fy + g.Q[5] * acc.fz),
                                      (float)(g.Q[6] * acc.fx + g.Q[7] * acc.fy + g.Q[8] * acc.fz),
                                      __uint_as_float(acc.cnt));
        Fout[me] = fv;
        store_user_F(po, gid, me, fv);
        if (DIGEST) { dcnt[me] = acc.cnt; dhs[me] = acc.hs; dhx[me] = acc.hx; }
        tU += Ui;
        tW[0] += 0.5 * acc.w0; tW[1] += 0.5 * acc.w1; tW[2] += 0.5 * acc.w2;
        tW[3] += 0.5 * acc.w3; tW[4] += 0.5 * acc.w4; tW[5] += 0.5 * acc.w5;
        tI += acc.cnt;
        tR += acc.nrc;
        tC += ncand - 1u;
        tNF += isfinite(acc.fx + acc.fy + acc.fz + Ui) ? 0.0 : 1.0;
      }
      pb += (uint32_t)B;
    }
  }
  // warp sums, then the warps of the block in fixed order
  double v[NPART] = {tU, tW[0], tW[1], tW[2], tW[3], tW[4], tW[5], (double)tI, (double)tC, (double)tS, (double)tR,
                     0.0, tNF};  // (slot 11: fp32-tier count -- every interaction here is fp64)
#pragma unroll
  for (int k = 0; k < NPART; ++k) v[k] = warp_sum_d(v[k]);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NPART; ++k) smb.part[wid][k] = v[k];
  }
  __syncthreads();
  if (tid < NPART) {
    double sum = 0.0;
    for (int w = 0; w < RW_NW; ++w) sum += smb.part[w][tid];
    bpart[(int64_t)blockIdx.x * NPART + tid] = sum;
  }
  PDL_LAUNCH();
}

}  // namespace nc
