// k3_sparse64.cuh -- K3 for sparse cells in NC_F64 (WCA at rho = 0.8442: ~1.3 particles per cell).
// Included at the end of kernels.cuh.
//
// The NC_F64 semantics of k_pairs (reading R16): every candidate is decided by the canonical fp64
// membership test r^2 = |(q_j + L n) - q_i|^2 < r_c^2 evaluated in the definition's association order
// (canonical_r2), and every pair's displacement is formed error-free in the lab frame (exact_d); only the
// work mapping differs.  The warp-per-cell kernel spends its time on per-cell set-up when a cell holds
// ~1.3 particles; here, as in k_pairs_sparse, one thread owns one particle i and walks its own stencil
// rows (sp_row: build_entries' fp64 expressions, so stencils and candidate counts are the oracle's bit
// for bit) in lockstep with the 31 other particles of its warp, reading the lab positions of each row's
// one or two contiguous particle ranges straight from global memory.  Survivors are queued per thread
// (sorted index and packed image) and evaluated in fp64 in batches.  Full i-side accumulation, no
// atomics; block partials over a fixed particle range of one layer (P-invariant).
#pragma once

namespace nc {

constexpr int SP64_QCAP = 16;  // per-thread survivor queue

struct Sp64Smem {
  uint32_t qj[SP64_QCAP][SP_NT];  // sorted index of a queued j
  uint32_t qn[SP64_QCAP][SP_NT];  // its image n, three int8 (n + 128)
  double part[SP_NT / 32][NPART];
};

__device__ __forceinline__ uint32_t pack_n3(int n0, int n1, int n2) {
  return (uint32_t)(n0 + 128) | ((uint32_t)(n1 + 128) << 8) | ((uint32_t)(n2 + 128) << 16);
}

// the queued survivors of this thread: error-free d in the lab frame, LJ with the energy shift (R11/R12)
template <bool DIGEST>
__device__ __forceinline__ void sp64_eval(const Geom& g, const Sp64Smem& sm, const double4* __restrict__ qs,
                                          const uint32_t* __restrict__ gid, int nq, int tid, const double4& qi,
                                          Acc& acc, const PairOut& po, uint32_t gi) {
  const int qmax = __reduce_max_sync(0xffffffffu, nq);
  const double sig2 = g.sig2, eps24 = 24.0 * g.eps;
  for (int k = 0; k < qmax; ++k) {
    if (k < nq) {
      const uint32_t j = sm.qj[k][tid], pn = sm.qn[k][tid];
      const int n0 = (int)(pn & 255u) - 128, n1 = (int)((pn >> 8) & 255u) - 128, n2 = (int)((pn >> 16) & 255u) - 128;
      const double4 qj = qs[j];
      const double dx = exact_d(g, 0, qj.x, qi.x, n0, n1, n2);
      const double dy = exact_d(g, 1, qj.y, qi.y, n0, n1, n2);
      const double dz = exact_d(g, 2, qj.z, qi.z, n0, n1, n2);
      const double r2 = dx * dx + dy * dy + dz * dz;
      lj_accumulate(sig2, eps24, acc, dx, dy, dz, r2);
      digest_add<DIGEST>(acc, gid, j, n0, n1, n2, po, gi);
    }
  }
  __syncwarp();
}

// grid = nlay layers x bpl blocks, bpl = ceil(l1 l2 / SP_CPB): block b of layer L takes the layer's
// particles [b SP_NT, (b+1) SP_NT) + k bpl SP_NT, k = 0, 1, ... and the layer's cells the same way
// for the stencil-size statistic (empty cells included).
template <bool DIGEST, int LPP = 1>
__global__ void __launch_bounds__(SP_NT, 4)
k_pairs_sparse64(const uint32_t* __restrict__ cs, const uint4* __restrict__ rec, const double4* __restrict__ qs,
                 const uint32_t* __restrict__ nh, const uint32_t* __restrict__ gid, double4* __restrict__ Fout,
                 double* __restrict__ bpart, uint32_t* __restrict__ dcnt, uint64_t* __restrict__ dhs,
                 uint64_t* __restrict__ dhx, const __grid_constant__ Geom g, int bpl, int layer0, const PairOut po) {
  PDL_WAIT();  // (the successor is released at the end)
  extern __shared__ __align__(16) unsigned char sp64_raw[];
  Sp64Smem& sm = *reinterpret_cast<Sp64Smem*>(sp64_raw);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int l1 = g.dims[0], l2 = g.dims[1];
  const int layer = layer0 + (int)(blockIdx.x / bpl);
  const int b = (int)blockIdx.x - (layer - layer0) * bpl;
  const uint32_t per_layer = (uint32_t)l1 * (uint32_t)l2;
  const uint32_t cell0 = per_layer * (uint32_t)layer;
  const uint32_t P0 = cs[cell0], P1 = cs[cell0 + per_layer];
  double tU = 0.0, tW[6] = {0, 0, 0, 0, 0, 0}, tNF = 0.0;
  uint32_t tI = 0, tC = 0, tS = 0;

  // stencil sizes of the layer's cells (sp_row's expressions, per cell)
  for (uint32_t c = (uint32_t)b * SP_NT + (uint32_t)tid; c < per_layer; c += (uint32_t)bpl * SP_NT) {
    const int a0 = (int)(c % (uint32_t)l1), a1 = (int)(c / (uint32_t)l1);
    int ns = 0;
    for (int ri = 0; ri < 12; ++ri) {
      SpRow r;
      if (sp_row(g, ri, a0, a1, layer, r)) ns += r.c1 - r.c0;
    }
    tS += (uint32_t)(ns - g.dbg_drop);
  }

  // LPP > 1 (small grids): LPP consecutive threads share one particle, thread `sub` walking the stencil
  // rows sub, sub + LPP, ...; the owner (sub 0) adds the others' sums in fixed order (shuffles)
  constexpr int NPB = SP_NT / LPP;
  const int sub = LPP > 1 ? tid % LPP : 0;
  for (uint32_t base = P0 + (uint32_t)b * NPB; base < P1; base += (uint32_t)bpl * NPB) {
    const uint32_t i = base + (uint32_t)(LPP > 1 ? tid / LPP : tid);
    const bool act = i < P1;
    const uint32_t me = act ? i : P0;
    const uint32_t c = rec[me].z;  // the cell of sorted slot me
    const int a0 = (int)(c % (uint32_t)l1), a1 = (int)((c / (uint32_t)l1) % (uint32_t)l2);
    const double4 qi = qs[me];
    const uint32_t nh_i = (g.variant == 1) ? nh[me] : 0u;
    const uint32_t gi = DIGEST ? gid[me] : 0u;
    Acc acc = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0u, 0u, 0ull, 0ull};
    int nq = 0;
    uint32_t ncand = 0;
    int last_ri = 0;  // the negative-control mode (nc_debug) drops the last column of the last row
    if (g.dbg_drop)
      for (int ri = 0; ri < 12; ++ri) {
        SpRow r;
        if (sp_row(g, ri, a0, a1, layer, r)) last_ri = ri;
      }
    for (int it = 0; it < (12 + LPP - 1) / LPP; ++it) {  // (the same trip count for every lane)
      const int ri = sub + it * LPP;
      SpRow r;
      const bool has = act && ri < 12 && sp_row(g, ri, a0, a1, layer, r);
      if (!__any_sync(0xffffffffu, has)) continue;
      if (!has) { r.c0 = r.c1 = a0; r.base = 0u; r.n2 = r.n3 = 0; }
      if (has && g.dbg_drop && ri == last_ri) r.c1 -= 1;
      // columns [c0, c1) in <= 2 pieces of constant x image (c1 - c0 <= 4 <= l1)
      const int n1a = floordiv(r.c0, l1);
      const int cut = (n1a + 1) * l1;
      const uint32_t pa0 = cs[r.base + (uint32_t)(r.c0 - n1a * l1)];
      const uint32_t pa1 = cs[r.base + (uint32_t)(min(r.c1, cut) - n1a * l1)];
      uint32_t pb0 = 0u, pb1 = 0u;
      if (r.c1 > cut) {
        pb0 = cs[r.base];
        pb1 = cs[r.base + (uint32_t)(r.c1 - cut)];
      }
      const uint32_t la = pa1 - pa0, lb = pb1 - pb0;
      ncand += la + lb;
      const int lmax = (int)__reduce_max_sync(0xffffffffu, la + lb);
      for (int k0 = 0; k0 < lmax; k0 += 2) {
        if (__any_sync(0xffffffffu, nq > SP64_QCAP - 2)) {
          sp64_eval<DIGEST>(g, sm, qs, gid, nq, tid, qi, acc, po, gi);
          nq = 0;
        }
        uint32_t jv[2];
        double4 qj[2];
        uint32_t nhj[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // both candidates' loads in flight
          const uint32_t k = (uint32_t)(k0 + h);
          jv[h] = k >= la ? pb0 + (k - la) : pa0 + k;
          const bool valid = k < la + lb;
          qj[h] = qs[valid ? jv[h] : me];
          nhj[h] = (g.variant == 1) ? nh[valid ? jv[h] : me] : 0u;
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t k = (uint32_t)(k0 + h);
          const bool valid = k < la + lb;
          int n0 = n1a + (k >= la ? 1 : 0), n1 = r.n2, n2 = r.n3;
          if (g.variant == 1) {  // DO: the home shifts of j and i (R5)
            n0 += nh_x(nhj[h]) - nh_x(nh_i);
            n1 += nh_y(nhj[h]) - nh_y(nh_i);
          }
          const double r2 = canonical_r2(g, qj[h].x, qj[h].y, qj[h].z, qi.x, qi.y, qi.z, n0, n1, n2);
          const bool hit = valid && jv[h] != me && r2 < g.rc2;
          NC_CHECK(nq < SP64_QCAP);
          sm.qj[nq][tid] = jv[h];  // (slot nq <= SP64_QCAP - 1 here)
          sm.qn[nq][tid] = pack_n3(n0, n1, n2);
          nq += hit ? 1 : 0;
        }
      }
    }
    sp64_eval<DIGEST>(g, sm, qs, gid, nq, tid, qi, acc, po, gi);
    if (LPP > 1) {
      if (act) tC += ncand;  // each thread its own rows' candidates (the self pair subtracted by the owner)
#pragma unroll
      for (int k = 1; k < LPP; ++k) {  // the owner adds sub 1, 2, ... in order
        const double fx = __shfl_down_sync(0xffffffffu, acc.fx, k), fy = __shfl_down_sync(0xffffffffu, acc.fy, k),
                     fz = __shfl_down_sync(0xffffffffu, acc.fz, k), uu = __shfl_down_sync(0xffffffffu, acc.u, k);
        const double w0 = __shfl_down_sync(0xffffffffu, acc.w0, k), w1 = __shfl_down_sync(0xffffffffu, acc.w1, k),
                     w2 = __shfl_down_sync(0xffffffffu, acc.w2, k), w3 = __shfl_down_sync(0xffffffffu, acc.w3, k),
                     w4 = __shfl_down_sync(0xffffffffu, acc.w4, k), w5 = __shfl_down_sync(0xffffffffu, acc.w5, k);
        const uint32_t cn = __shfl_down_sync(0xffffffffu, acc.cnt, k);
        const uint64_t h1 = __shfl_down_sync(0xffffffffu, acc.hs, k), h2 = __shfl_down_sync(0xffffffffu, acc.hx, k);
        if (sub == 0) {
          acc.fx += fx; acc.fy += fy; acc.fz += fz; acc.u += uu;
          acc.w0 += w0; acc.w1 += w1; acc.w2 += w2; acc.w3 += w3; acc.w4 += w4; acc.w5 += w5;
          acc.cnt += cn;
          if (DIGEST) { acc.hs += h1; acc.hx ^= h2; }
        }
      }
    }
    if (act && sub == 0) {
      const double Ui = 2.0 * g.eps * acc.u - 0.5 * g.ushift * (double)acc.cnt;
      const double4 fv = make_double4(acc.fx, acc.fy, acc.fz, (double)acc.cnt);  // lab frame
      Fout[me] = fv;
      store_user_F(po, gid, me, fv);
      if (DIGEST) { dcnt[me] = acc.cnt; dhs[me] = acc.hs; dhx[me] = acc.hx; }
      tU += Ui;
      tW[0] += 0.5 * acc.w0; tW[1] += 0.5 * acc.w1; tW[2] += 0.5 * acc.w2;
      tW[3] += 0.5 * acc.w3; tW[4] += 0.5 * acc.w4; tW[5] += 0.5 * acc.w5;
      tI += acc.cnt;
      tC += (LPP > 1 ? 0u : ncand) - 1u;
      tNF += isfinite(acc.fx + acc.fy + acc.fz + Ui) ? 0.0 : 1.0;
    }
  }
  // warp sums, then the block's warps in fixed order (slot 10: re-checks -- none, every candidate is
  // canonical; slot 11: fp32-tier interactions -- none)
  double v[NPART] = {tU, tW[0], tW[1], tW[2], tW[3], tW[4], tW[5], (double)tI, (double)tC, (double)tS, 0.0, 0.0, tNF};
#pragma unroll
  for (int k = 0; k < NPART; ++k) v[k] = warp_sum_d(v[k]);
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NPART; ++k) sm.part[wid][k] = v[k];
  }
  __syncthreads();
  if (tid < NPART) {
    double sum = 0.0;
    for (int w = 0; w < SP_NT / 32; ++w) sum += sm.part[w][tid];
    bpart[(int64_t)blockIdx.x * NPART + tid] = sum;
  }
  PDL_LAUNCH();
}

}  // namespace nc
