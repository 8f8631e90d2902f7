// k3_pairs.cuh -- K3 v4, the NC_F32 pair kernel with two particles per lane
// (included at the end of kernels.cuh).
//
// Same contract and the same per-cell structure as k_pairs<float, DIGEST>
// (kernels.cuh): one warp per block, K3_CELLS consecutive cells of one layer
// per warp, the neighborhood rebuilt from L_t (DS 27 cells P:445, DO
// 27/30/34/36 cells P:673-687, R4), neighbor particles staged in shared memory
// with the entry's image bracket, full i-side accumulation, no atomics,
// deterministic block partials.  What changes is the candidate filter (the
// "distance check first" of P:747):
//
//   every lane owns TWO particles (a, b) of the center cell and one stream s
//   of the staged list; one LDS.128 of a staged element serves both, and the
//   two dot-form tests r^2 - hi = (|v|^2 + (|u|^2 - hi)) - 2 u.v run as one
//   FADD2 + three FFMA2 with the element as the broadcast operand.  The
//   shared-memory pipe -- 83% busy in k_pairs, where every candidate costs one
//   LDS.128 (~4 wavefronts) -- does half the loads per candidate.  Hits go to
//   two per-lane queues (a and b) that are evaluated by k_pairs' own far/close
//   tiers (eval_pairs_f32, eval_close_f64) exactly as there.
#pragma once

namespace nc {

struct K4Smem : K3Smem<float> {
  K3QT queue_b[K3_QCAP][32];  // survivors of particle b (queue of K3Smem holds particle a)
};

// qa += K3_QSTRIDE if the sign bit of r is set (hit: r^2 - hi < 0)
__device__ __forceinline__ uint32_t bump_if_neg(uint32_t a, float r) {
  asm("{\n\t.reg .pred p;\n\tsetp.lt.s32 p, %1, 0;\n\t@p add.u32 %0, %0, %2;\n\t}"
      : "+r"(a)
      : "r"(__float_as_uint(r)), "n"(K3_QSTRIDE));
  return a;
}

__device__ __forceinline__ float2 bcast2(float x) { return make_float2(x, x); }

// Filter stream s of the staged chunk for the pair (a, b); survivors of each
// particle to its own queue; both queues evaluated when any could overflow.
template <bool DIGEST>
__device__ __forceinline__ void filter_chunk_v4(const Geom& g, const PairCtx<float>& pa, const PairCtx<float>& pb,
                                                bool hasb, K4Smem& sm, Acc& acc_a, Acc& acc_b, Acc32& a32_a,
                                                Acc32& a32_b, int s, int S, int iters, int lane,
                                                const double4* __restrict__ u64) {
  const uint32_t stage0 = smem_u32(&sm.stage[0]);
  const uint32_t qa0 = smem_u32(&sm.queue[0][lane]), qb0 = smem_u32(&sm.queue_b[0][lane]);
  const uint32_t qlim = K3_QSTRIDE * (K3_QCAP - K3_UNROLL);
  const uint32_t step = 16u * (uint32_t)S;
  const float inf32 = __int_as_float(0x7f800000);
  // packed (a, b) filter constants; a missing b never sets the sign bit
  const float2 cx = make_float2(pa.m2x, hasb ? pb.m2x : 0.0f), cy = make_float2(pa.m2y, hasb ? pb.m2y : 0.0f),
               cz = make_float2(pa.m2z, hasb ? pb.m2z : 0.0f);
  const float2 uuh = make_float2(pa.uu - pa.hi, hasb ? pb.uu - pb.hi : inf32);
  uint32_t sa = stage0 + 16u * (uint32_t)s;
  uint32_t qa = qa0, qb = qb0;
  int it = 0;
  const int main_iters = iters - iters % K3_UNROLL;
  for (;;) {
    bool full = false;
    while (it < main_iters) {
#pragma unroll
      for (int k = 0; k < K3_UNROLL; ++k) {
        const float4 v = lds128(sa);
        float2 r = __fadd2_rn(bcast2(v.w), uuh);
        r = __ffma2_rn(bcast2(v.x), cx, r);
        r = __ffma2_rn(bcast2(v.y), cy, r);
        r = __ffma2_rn(bcast2(v.z), cz, r);
        stsq(qa, sa);
        qa = bump_if_neg(qa, r.x);
        stsq(qb, sa);
        qb = bump_if_neg(qb, r.y);
        sa += step;
      }
      it += K3_UNROLL;
      if (__any_sync(0xffffffffu, (qa - qa0) > qlim || (qb - qb0) > qlim)) { full = true; break; }
    }
    if (!full) {
      for (; it < iters; ++it) {
        const float4 v = lds128(sa);
        float2 r = __fadd2_rn(bcast2(v.w), uuh);
        r = __ffma2_rn(bcast2(v.x), cx, r);
        r = __ffma2_rn(bcast2(v.y), cy, r);
        r = __ffma2_rn(bcast2(v.z), cz, r);
        stsq(qa, sa);
        qa = bump_if_neg(qa, r.x);
        stsq(qb, sa);
        qb = bump_if_neg(qb, r.y);
        sa += step;
      }
    }
    __syncwarp();
    eval_pairs_f32<DIGEST>(sm.queue, g, pa, sm, acc_a, a32_a, (int)((qa - qa0) / K3_QSTRIDE), lane, stage0, u64);
    eval_pairs_f32<DIGEST>(sm.queue_b, g, pb, sm, acc_b, a32_b, (int)((qb - qb0) / K3_QSTRIDE), lane, stage0, u64);
    qa = qa0;
    qb = qb0;
    if (it >= iters) break;
  }
}

__device__ __forceinline__ void combine_streams(Acc& acc, int S, int s, int NP, bool act, int lane) {
  for (int o = 1; o < S; o <<= 1) {
    const bool take = act && ((s & (2 * o - 1)) == 0) && (s + o < S);
    const int src = (lane + o * NP) & 31;
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

template <bool DIGEST>
__global__ void __launch_bounds__(32, K3_MINB)
k_pairs_v4(const double4* __restrict__ u, const float4* __restrict__ u32, const uint32_t* __restrict__ cs,
           const float4* __restrict__ qs, const uint32_t* __restrict__ nh, const uint32_t* __restrict__ gid,
           float4* __restrict__ Fout, double* __restrict__ bpart, uint32_t* __restrict__ dcnt,
           uint64_t* __restrict__ dhs, uint64_t* __restrict__ dhx, const __grid_constant__ Geom g, int cpb, int bpl,
           int layer0) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int lane = threadIdx.x & 31;
  K4Smem& sm = *reinterpret_cast<K4Smem*>(smraw);

  const int l1 = g.dims[0], l2 = g.dims[1];
  const int layer = layer0 + (int)(blockIdx.x / bpl);
  const int chunk = (int)blockIdx.x - (layer - layer0) * bpl;
  const int per_layer = l1 * l2;
  const int cbeg = chunk * cpb;
  const int cend = min(per_layer, cbeg + cpb);

  PairCtx<float> pa, pb;
  pa.hi = pb.hi = (float)g.band_hi;
  pa.lo64 = pb.lo64 = g.rc2 * (1.0 - K3_BAND64);
  pa.hi64 = pb.hi64 = g.rc2 * (1.0 + K3_BAND64);
  pa.qs = pb.qs = qs;
  pa.nh = pb.nh = nh;
  pa.gid = pb.gid = gid;

  double tU = 0, tW[6] = {0, 0, 0, 0, 0, 0}, tI = 0, tC = 0, tS = 0, tR = 0, tNF = 0;
  if (lane == 0) {  // permanent far element padding the evaluation (reads particle i + far bracket)
    sm.stage[K3_DUMMY] = far4<float>();
    sm.sent[K3_DUMMY] = K3_MAXE - 1;
    sm.e_B[K3_MAXE - 1][0] = 1e150; sm.e_B[K3_MAXE - 1][1] = 1e150; sm.e_B[K3_MAXE - 1][2] = 1e150;
  }
  __syncwarp();

  for (int cl = cbeg; cl < cend; ++cl) {
    const int a0 = cl % l1, a1 = cl / l1, a2 = layer;
    const uint32_t cid = (uint32_t)cl + (uint32_t)per_layer * (uint32_t)layer;
    const int nst = build_entries(g, a0, a1, a2, sm, lane);
    uint32_t tot = 0;
    for (int e0 = 0; e0 < nst; e0 += 32) {
      const int e = e0 + lane;
      uint32_t cnt = 0, st = 0;
      if (e < nst) {
        const uint32_t cell = sm.e_start[e];
        st = cs[cell];
        cnt = cs[cell + 1] - st;
      }
      uint32_t x = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
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
    tS += (double)nst;
    const uint32_t ibase = cs[cid];
    const int ni = (int)(cs[cid + 1] - ibase);
    if (ni == 0) continue;
    tC += (double)ni * (double)tot - (double)ni;

    for (int ib = 0; ib < ni; ib += 32) {
      const int nbat = min(32, ni - ib);
      const int NP = (nbat + 1) >> 1;      // particle pairs
      const int S = 32 / NP;               // streams over the staged list
      const int p = lane % NP;
      const bool act = lane < S * NP;
      const int s = act ? lane / NP : 0;   // ghost lanes shadow stream 0
      const bool hasb = act && (2 * p + 1 < nbat);
      pa.my = ibase + ib + 2 * p;
      pb.my = (2 * p + 1 < nbat) ? pa.my + 1 : pa.my;
      {
        const double4 ua = u[pa.my], ub = u[pb.my];
        const float4 fa = u32[pa.my], fb = u32[pb.my];
        const float inf32 = __int_as_float(0x7f800000);
        pa.ux = ua.x; pa.uy = ua.y; pa.uz = ua.z;
        pb.ux = ub.x; pb.uy = ub.y; pb.uz = ub.z;
        pa.fx = fa.x; pa.fy = fa.y; pa.fz = fa.z;
        pb.fx = fb.x; pb.fy = fb.y; pb.fz = fb.z;
        pa.m2x = act ? -2.0f * fa.x : 0.0f; pa.m2y = act ? -2.0f * fa.y : 0.0f; pa.m2z = act ? -2.0f * fa.z : 0.0f;
        pb.m2x = -2.0f * fb.x; pb.m2y = -2.0f * fb.y; pb.m2z = -2.0f * fb.z;
        pa.uu = act ? fmaf(fa.z, fa.z, fmaf(fa.y, fa.y, fa.x * fa.x)) : inf32;  // ghost lanes never hit
        pb.uu = fmaf(fb.z, fb.z, fmaf(fb.y, fb.y, fb.x * fb.x));
        pa.nh_i = (g.variant == 1) ? nh[pa.my] : 0u;
        pb.nh_i = (g.variant == 1) ? nh[pb.my] : 0u;
      }
      Acc acc_a = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0u, 0u, 0ull, 0ull};
      Acc acc_b = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0u, 0u, 0ull, 0ull};
      Acc32 a32_a = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0u};
      Acc32 a32_b = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0u};

      int e0 = 0;
      while (e0 < nst) {
        const uint32_t base_off = sm.e_off[e0];
        int e1 = e0;
        for (int eb = e0; eb < nst; eb += 32) {
          const int e = eb + lane;
          const bool fits = e < nst && (sm.e_off[e] + sm.e_cnt[e] - base_off) <= (uint32_t)K3_CAP;
          const int nfit = __popc(__ballot_sync(0xffffffffu, fits));  // the fitting entries are a prefix
          e1 = eb + nfit;
          if (nfit < 32) break;
        }
        if (e1 == e0) e1 = e0 + 1;  // unreachable: a cell holds fewer than K3_CAP particles
        const uint32_t ctot = (e1 < nst ? sm.e_off[e1] : tot) - base_off;
        for (int eb = e0; eb < e1; eb += 32) {
          const int e = eb + lane;
          if (e < e1) {
            const uint32_t dst = sm.e_off[e] - base_off, cnt = sm.e_cnt[e];
            for (uint32_t k = 0; k < cnt; ++k) sm.sent[dst + k] = (uint8_t)e;
            sm.s64.Bf[e][0] = (float)sm.e_B[e][0];
            sm.s64.Bf[e][1] = (float)sm.e_B[e][1];
            sm.s64.Bf[e][2] = (float)sm.e_B[e][2];
          }
        }
        __syncwarp();
        for (uint32_t t0 = 0; t0 < ctot; t0 += 128) {
          uint32_t tt[4], jj[4];
          int ee[4];
          float4 pp[4];
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            tt[r] = t0 + 32u * r + lane;
            const bool v = tt[r] < ctot;
            ee[r] = v ? sm.sent[tt[r]] : e0;
            jj[r] = sm.e_start[ee[r]] + tt[r] - (sm.e_off[ee[r]] - base_off);
            pp[r] = v ? u32[jj[r]] : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            if (tt[r] < ctot) {
              const float x = pp[r].x + sm.s64.Bf[ee[r]][0], y = pp[r].y + sm.s64.Bf[ee[r]][1],
                          z = pp[r].z + sm.s64.Bf[ee[r]][2];
              sm.stage[tt[r]] = make_float4(x, y, z, fmaf(z, z, fmaf(y, y, x * x)));  // .w = |v|^2
            }
          }
        }
        if (lane < S) {
          sm.stage[ctot + lane] = far4<float>();
          sm.sent[ctot + lane] = 0;
        }
        __syncwarp();
        const int iters = (int)((ctot + S - 1) / S);
        pa.base_off = pb.base_off = base_off;
        filter_chunk_v4<DIGEST>(g, pa, pb, hasb, sm, acc_a, acc_b, a32_a, a32_b, s, S, iters, lane, u);
        __syncwarp();
        e0 = e1;
      }
      fold32(acc_a, a32_a);
      fold32(acc_b, a32_b);
      combine_streams(acc_a, S, s, NP, act, lane);
      combine_streams(acc_b, S, s, NP, act, lane);
      const bool owner = act && s == 0;
      const double Ua = 2.0 * g.eps * acc_a.u - 0.5 * g.ushift * (double)acc_a.cnt;
      const double Ub = 2.0 * g.eps * acc_b.u - 0.5 * g.ushift * (double)acc_b.cnt;
      if (owner) {
        Fout[pa.my] = make_float4((float)(g.Q[0] * acc_a.fx + g.Q[1] * acc_a.fy + g.Q[2] * acc_a.fz),
                                  (float)(g.Q[3] * acc_a.fx + g.Q[4] * acc_a.fy + g.Q[5] * acc_a.fz),
                                  (float)(g.Q[6] * acc_a.fx + g.Q[7] * acc_a.fy + g.Q[8] * acc_a.fz), 0.0f);
        if (DIGEST) { dcnt[pa.my] = acc_a.cnt; dhs[pa.my] = acc_a.hs; dhx[pa.my] = acc_a.hx; }
        if (hasb) {
          Fout[pb.my] = make_float4((float)(g.Q[0] * acc_b.fx + g.Q[1] * acc_b.fy + g.Q[2] * acc_b.fz),
                                    (float)(g.Q[3] * acc_b.fx + g.Q[4] * acc_b.fy + g.Q[5] * acc_b.fz),
                                    (float)(g.Q[6] * acc_b.fx + g.Q[7] * acc_b.fy + g.Q[8] * acc_b.fz), 0.0f);
          if (DIGEST) { dcnt[pb.my] = acc_b.cnt; dhs[pb.my] = acc_b.hs; dhx[pb.my] = acc_b.hx; }
        }
      }
      const double fchk = owner ? acc_a.fx + acc_a.fy + acc_a.fz + Ua + acc_b.fx + acc_b.fy + acc_b.fz + Ub : 0.0;
      if (owner) {
        tU += Ua + Ub;
        tW[0] += 0.5 * (acc_a.w0 + acc_b.w0); tW[1] += 0.5 * (acc_a.w1 + acc_b.w1);
        tW[2] += 0.5 * (acc_a.w2 + acc_b.w2); tW[3] += 0.5 * (acc_a.w3 + acc_b.w3);
        tW[4] += 0.5 * (acc_a.w4 + acc_b.w4); tW[5] += 0.5 * (acc_a.w5 + acc_b.w5);
        tI += (double)(acc_a.cnt + acc_b.cnt);
        tR += (double)(acc_a.nrc + acc_b.nrc);
      }
      tNF += isfinite(fchk) ? 0.0 : 1.0;
    }
  }
  tU = warp_sum_d(tU);
  tW[0] = warp_sum_d(tW[0]); tW[1] = warp_sum_d(tW[1]); tW[2] = warp_sum_d(tW[2]);
  tW[3] = warp_sum_d(tW[3]); tW[4] = warp_sum_d(tW[4]); tW[5] = warp_sum_d(tW[5]);
  tI = warp_sum_d(tI);
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
    else v = tNF;
    bpart[(int64_t)blockIdx.x * NPART + lane] = v;
  }
}

}  // namespace nc
