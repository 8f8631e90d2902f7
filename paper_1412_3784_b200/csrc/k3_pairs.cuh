// k3_pairs.cuh -- K3 v3, the NC_F32 pair kernel (included at the end of kernels.cuh).
//
// Same contract as k_pairs<float, DIGEST> (kernels.cuh): one warp per block,
// K3_CELLS consecutive cells of one layer per warp, the neighborhood of each
// center cell rebuilt from L_t (DS 27 cells P:445, DO 27/30/34/36 cells
// P:673-687 by the exact interval rule R4), neighbor particles staged in shared
// memory with the entry's image bracket applied, full i-side accumulation, no
// atomics, deterministic block partials.  What changes is how the "distance
// check first" of P:747 and the force evaluation are executed on sm_100a:
//
//   pairs    every lane owns TWO particles i_a, i_b of the center cell and one
//            stream s of the staged neighbor list (t = s, s+S, ...);
//   filter   r^2 - hi for (i_a, j) and (i_b, j) in one packed pass,
//            (|v|^2 + (|u|^2 - hi)) - 2 u.v = FADD2 + 3 FFMA2 with the staged
//            j coordinate as the broadcast operand; j is queued (one STS.U16,
//            pointer bumped under a predicate) when either sign bit is set;
//   far      the queued j are evaluated against both i in packed fp32
//            (FFMA2/FMUL2: one instruction per component pair) for the pairs
//            with r_split <= r below the lower cutoff band;
//   close    pairs with r < r_split or inside the cutoff band (and every pair
//            in digest mode) are queued as (j, half) items and evaluated in
//            fp64 from the fp64 cell-local coordinates, with the canonical R16
//            membership test inside the 1e-12 band -- the precision design of
//            DESIGN.md section 5, unchanged.
#pragma once

#ifdef NC_V3_CHECK
#include <cstdio>
#define V3CHK(cond, fmt, ...) do { if (!(cond)) { printf("V3CHK %d " fmt "\n", __LINE__, __VA_ARGS__); } } while (0)
#else
#define V3CHK(cond, fmt, ...) do { } while (0)
#endif

namespace nc {

constexpr int V3_CAP = 448;                            // staged neighbor elements per chunk
constexpr int V3_MAXS = 8;                             // streams per pair (bounds the sentinel pad)
constexpr int V3_PAD = 8 * V3_MAXS;                    // the 8-unrolled filter reads < 8 S elements past the chunk
constexpr int V3_DUMMY = V3_CAP + V3_PAD;              // permanent far element (queue padding)
constexpr int V3_STAGE = V3_DUMMY + 1;
#ifndef V3_QCAP_OVR
#define V3_QCAP_OVR 64
#endif
#ifndef V3_SLICE_OVR
#define V3_SLICE_OVR 32
#endif
#ifndef V3_MINB
#define V3_MINB 16
#endif
constexpr int V3_QCAP = V3_QCAP_OVR;                   // per-lane queue of filter hits (staged indices)
constexpr int V3_SLICE = V3_SLICE_OVR;                 // far-tier entries per close-tier round
constexpr int V3_CQCAP = 2 * V3_SLICE;                 // close items per round (<= 2 per entry)

struct V3Lane {                      // per-lane fp64 state kept out of registers
  double ua[3], ub[3];               // fp64 cell-local coordinates of i_a, i_b
  double fa[3], fb[3];               // fp64 force sums (cell-local rotated frame)
  double u, w[6];                    // sum s6(s6-1), sum fr d d
};

struct V3Smem {
  float4 stage[V3_STAGE];            // x, y, z (bracket applied), w = |v|^2
  V3Lane ln[32];
  uint16_t queue[V3_QCAP][32];       // staged indices of this lane's filter hits
  uint16_t cq[V3_CQCAP][32];         // close items: staged index | half << 15
  uint8_t sent[V3_STAGE];            // entry of each staged element
  uint32_t e_start[K3_MAXE], e_cnt[K3_MAXE], e_off[K3_MAXE];
  int32_t e_n[K3_MAXE][3];
  double e_B[K3_MAXE][3];
  float Bf[K3_MAXE][3];
};

struct V3Pair {
  float2 cx, cy, cz, uuh;  // filter: -2 u and |u|^2 - hi for (a, b)
  float2 nx, ny, nz;       // far tier: -u (fp32 cell-local) for (a, b)
  uint32_t ia, ib;         // sorted indices (ib == ia for a missing b)
  uint32_t nha, nhb;       // packed DO home shifts
  uint32_t base_off;       // staging offset of the current chunk
};

// per-lane counters (the fp64 sums live in shared memory, V3Lane)
struct Acc3 {
  uint32_t cnt, nrc, cna, cnb;
  uint64_t hsa, hxa, hsb, hxb;
};

struct Acc3f {  // packed (a, b) fp32 sums of the far tier: +fr d, s6^2, s6, fr d d
  float2 fx, fy, fz, u12, u6, w0, w1, w2, w3, w4, w5;
  uint32_t cnt;
};

__device__ __forceinline__ void fold3(V3Lane& L, Acc3& A, Acc3f& a) {
  L.fa[0] -= a.fx.x; L.fa[1] -= a.fy.x; L.fa[2] -= a.fz.x;
  L.fb[0] -= a.fx.y; L.fb[1] -= a.fy.y; L.fb[2] -= a.fz.y;
  L.u += ((double)a.u12.x + (double)a.u12.y) - ((double)a.u6.x + (double)a.u6.y);
  L.w[0] += (double)a.w0.x + (double)a.w0.y; L.w[1] += (double)a.w1.x + (double)a.w1.y;
  L.w[2] += (double)a.w2.x + (double)a.w2.y; L.w[3] += (double)a.w3.x + (double)a.w3.y;
  L.w[4] += (double)a.w4.x + (double)a.w4.y; L.w[5] += (double)a.w5.x + (double)a.w5.y;
  A.cnt += a.cnt;
  const float2 z = make_float2(0.f, 0.f);
  a.fx = z; a.fy = z; a.fz = z; a.u12 = z; a.u6 = z;
  a.w0 = z; a.w1 = z; a.w2 = z; a.w3 = z; a.w4 = z; a.w5 = z;
  a.cnt = 0u;
}

__device__ __forceinline__ float2 bc2(float x) { return make_float2(x, x); }

__device__ __forceinline__ uint32_t lds16(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return (uint32_t)v;
}

// qa += 64 if (ra < 0 or rb < 0) as sign bits: LOP3 + ISETP + predicated IADD
__device__ __forceinline__ uint32_t bump_either(uint32_t qa, float2 r) {
  asm("{\n\t.reg .pred p;\n\t.reg .b32 x;\n\tor.b32 x, %1, %2;\n\tsetp.lt.s32 p, x, 0;\n\t@p add.u32 %0, %0, 64;\n\t}"
      : "+r"(qa)
      : "r"(__float_as_uint(r.x)), "r"(__float_as_uint(r.y)));
  return qa;
}

// One group of 8 filter steps for stream offset sa (bytes) and staged index t.
template <int S>
__device__ __forceinline__ void v3_filter8(const V3Pair& pc, uint32_t& sa, uint32_t& t, uint32_t& qa) {
  float4 v[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) v[u] = lds128(sa + 16u * S * u);
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    float2 r = __fadd2_rn(bc2(v[u].w), pc.uuh);
    r = __ffma2_rn(bc2(v[u].x), pc.cx, r);
    r = __ffma2_rn(bc2(v[u].y), pc.cy, r);
    r = __ffma2_rn(bc2(v[u].z), pc.cz, r);
    sts16(qa, t + (uint32_t)(S * u));
    qa = bump_either(qa, r);
  }
  sa += 128u * S;
  t += 8u * S;
}

__device__ __forceinline__ uint32_t v3_sidx(const V3Smem& sm, uint32_t t, uint32_t base_off) {
  const int e = sm.sent[t];
  return sm.e_start[e] + t - (sm.e_off[e] - base_off);
}

__device__ __forceinline__ void v3_image(const Geom& g, const V3Smem& sm, uint32_t t, uint32_t nh_j, uint32_t nh_i,
                                         int& n0, int& n1, int& n2) {
  const int e = sm.sent[t];
  n0 = sm.e_n[e][0]; n1 = sm.e_n[e][1]; n2 = sm.e_n[e][2];
  if (g.variant == 1) {
    n0 += nh_x(nh_j) - nh_x(nh_i);
    n1 += nh_y(nh_j) - nh_y(nh_i);
  }
}

__device__ __forceinline__ bool v3_canonical_in(const Geom& g, const float4* qs, uint32_t i, uint32_t j, int n0, int n1,
                                                int n2) {
  const float4 qi = qs[i], qj = qs[j];
  return canonical_r2(g, (double)qj.x, (double)qj.y, (double)qj.z, (double)qi.x, (double)qi.y, (double)qi.z, n0, n1,
                      n2) < g.rc2;
}

struct V3Env {  // per-launch constants and pointers of the evaluation
  uint32_t ntot;
  const float4* qs;
  const uint32_t* nh;
  const uint32_t* gid;
  const double4* u64;
  double lo64, hi64;
};

// fp64 tier: items cq[0..nq) = staged index | half << 15.  Two per iteration;
// padding reads the dummy element (far bracket) with j = i (rejected).
template <bool DIGEST>
__device__ __forceinline__ void v3_eval_close(const Geom& g, const V3Env& ev, const V3Pair& pc, V3Smem& sm, Acc3& A,
                                              int nq, int lane) {
  const int qmax = __reduce_max_sync(0xffffffffu, nq);
  if (qmax == 0) return;
  const double sig2 = g.sig2, eps24 = 24.0 * g.eps;
  V3Lane& L = sm.ln[lane];
  double fa0 = L.fa[0], fa1 = L.fa[1], fa2 = L.fa[2], fb0 = L.fb[0], fb1 = L.fb[1], fb2 = L.fb[2];
  double uu = L.u, w0 = L.w[0], w1 = L.w[1], w2 = L.w[2], w3 = L.w[3], w4 = L.w[4], w5 = L.w[5];
  for (int k = 0; k < qmax; k += 2) {
    double dx[2], dy[2], dz[2], r2[2];
    bool ok[2], hb[2];
    uint32_t jj[2], tt[2], ii[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const bool valid = k + h < nq;
      const uint32_t it = valid ? lds16(smem_u32(&sm.cq[0][0]) + 64u * (uint32_t)(k + h) + 2u * (uint32_t)lane)
                                : (uint32_t)V3_DUMMY;
      const uint32_t t = it & 0x7fffu;
      const bool b = (it >> 15) != 0;
      const uint32_t i = b ? pc.ib : pc.ia;
      const uint32_t j = valid ? v3_sidx(sm, t, pc.base_off) : i;
      const int e = sm.sent[t];
      V3CHK(t < V3_STAGE && e < K3_MAXE && k + h < V3_CQCAP, "close t=%u e=%d j=%u k=%d nq=%d", t, e, j, k + h, nq);
      V3CHK(j < ev.ntot, "close j=%u ntot=%u t=%u valid=%d", j, ev.ntot, t, (int)valid);
      const double4 p = ev.u64[j];
      const double* ui = b ? L.ub : L.ua;
      dx[h] = (p.x + sm.e_B[e][0]) - ui[0];
      dy[h] = (p.y + sm.e_B[e][1]) - ui[1];
      dz[h] = (p.z + sm.e_B[e][2]) - ui[2];
      r2[h] = dx[h] * dx[h] + dy[h] * dy[h] + dz[h] * dz[h];
      ok[h] = (j != i) && (r2[h] < ev.hi64);
      hb[h] = b;
      jj[h] = j;
      tt[h] = t;
      ii[h] = i;
    }
    int nn[2][3] = {{0, 0, 0}, {0, 0, 0}};
    if (DIGEST || (ok[0] && r2[0] >= ev.lo64) || (ok[1] && r2[1] >= ev.lo64)) {  // rare: canonical band / digest
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (ok[h]) {
          v3_image(g, sm, tt[h], g.variant == 1 ? ev.nh[jj[h]] : 0u, hb[h] ? pc.nhb : pc.nha, nn[h][0], nn[h][1],
                   nn[h][2]);
          if (r2[h] >= ev.lo64) {
            V3CHK(jj[h] < ev.ntot && ii[h] < ev.ntot, "canon i=%u j=%u", ii[h], jj[h]);
            ok[h] = v3_canonical_in(g, ev.qs, ii[h], jj[h], nn[h][0], nn[h][1], nn[h][2]);
            A.nrc++;
          }
        }
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const double ir = rcp64(r2[h]);
      const double s2 = sig2 * ir;
      const double s6 = s2 * s2 * s2;
      double fr = (eps24 * s6) * (2.0 * s6 - 1.0) * ir;
      fr = ok[h] ? fr : 0.0;
      const double tx = fr * dx[h], ty = fr * dy[h], tz = fr * dz[h];
      if (hb[h]) { fb0 -= tx; fb1 -= ty; fb2 -= tz; }
      else { fa0 -= tx; fa1 -= ty; fa2 -= tz; }
      uu += ok[h] ? s6 * s6 - s6 : 0.0;
      w0 += tx * dx[h]; w1 += ty * dy[h]; w2 += tz * dz[h];
      w3 += tx * dy[h]; w4 += tx * dz[h]; w5 += ty * dz[h];
      A.cnt += ok[h] ? 1u : 0u;
      if (DIGEST && ok[h]) {
        const uint64_t key = (uint64_t)ev.gid[jj[h]] | ((uint64_t)(nn[h][0] + 8) << 32) |
                             ((uint64_t)(nn[h][1] + 8) << 36) | ((uint64_t)(nn[h][2] + 8) << 40);
        const uint64_t hh = mix64(key);
        if (hb[h]) { A.hsb += hh; A.hxb ^= hh; A.cnb++; }
        else { A.hsa += hh; A.hxa ^= hh; A.cna++; }
      }
    }
  }
  L.fa[0] = fa0; L.fa[1] = fa1; L.fa[2] = fa2; L.fb[0] = fb0; L.fb[1] = fb1; L.fb[2] = fb2;
  L.u = uu; L.w[0] = w0; L.w[1] = w1; L.w[2] = w2; L.w[3] = w3; L.w[4] = w4; L.w[5] = w5;
}

// Evaluate this lane's queue[0..nq) against (a, b): far pairs in packed fp32,
// close / band pairs (all pairs in digest mode) as fp64 items, in slices.
template <bool DIGEST>
__device__ __forceinline__ void v3_eval(const Geom& g, const V3Env& ev, const V3Pair& pc, V3Smem& sm, Acc3& A,
                                        Acc3f& a, int nq, int lane) {
  const int qmax = __reduce_max_sync(0xffffffffu, nq);
  const float split2 = g.f_split2, lo32 = g.f_lo, hi32 = g.f_hi;
  const float2 sig2 = bc2(g.f_sig2), c48 = bc2(g.f_c48), m24 = bc2(g.f_m24);
  const uint32_t stage0 = smem_u32(&sm.stage[0]);
  const uint32_t cq0 = smem_u32(&sm.cq[0][lane]);
  const uint32_t qb = smem_u32(&sm.queue[0][lane]);
  for (int k0 = 0; k0 < qmax; k0 += V3_SLICE) {
    const int kend = min(qmax, k0 + V3_SLICE);
    uint32_t cqa = cq0;
#pragma unroll 2
    for (int k = k0; k < kend; ++k) {
      const uint32_t t = k < nq ? lds16(qb + 64u * (uint32_t)k) : (uint32_t)V3_DUMMY;
      V3CHK(t < V3_STAGE && k < V3_QCAP, "far t=%u k=%d nq=%d", t, k, nq);
      const float4 v = lds128(stage0 + 16u * t);
      const float2 dx = __fadd2_rn(bc2(v.x), pc.nx);
      const float2 dy = __fadd2_rn(bc2(v.y), pc.ny);
      const float2 dz = __fadd2_rn(bc2(v.z), pc.nz);
      float2 r2 = __fmul2_rn(dx, dx);
      r2 = __ffma2_rn(dy, dy, r2);
      r2 = __ffma2_rn(dz, dz, r2);
      bool far_a = false, far_b = false;
      if (!DIGEST) {
        far_a = r2.x >= split2 && r2.x < lo32;
        far_b = r2.y >= split2 && r2.y < lo32;
      }
      const bool close_a = !far_a && r2.x < hi32;  // the dummy and ghost b (r2 = inf) are neither
      const bool close_b = !far_b && r2.y < hi32;
      V3CHK(cqa + 128u <= cq0 + 64u * V3_CQCAP || !(close_a || close_b), "cq overflow k=%d k0=%d", k, k0);
      if (close_a) { sts16(cqa, t); cqa += 64u; }
      if (close_b) { sts16(cqa, t | 0x8000u); cqa += 64u; }
      if (!DIGEST) {
        float ira, irb;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(ira) : "f"(r2.x));
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(irb) : "f"(r2.y));
        const float2 ir = make_float2(far_a ? ira : 0.0f, far_b ? irb : 0.0f);  // masks s6, fr and u at once
        const float2 s2 = __fmul2_rn(sig2, ir);
        const float2 s6 = __fmul2_rn(__fmul2_rn(s2, s2), s2);
        const float2 fr = __fmul2_rn(__fmul2_rn(s6, __ffma2_rn(s6, c48, m24)), ir);
        const float2 tx = __fmul2_rn(fr, dx), ty = __fmul2_rn(fr, dy), tz = __fmul2_rn(fr, dz);
        a.fx = __fadd2_rn(a.fx, tx); a.fy = __fadd2_rn(a.fy, ty); a.fz = __fadd2_rn(a.fz, tz);
        a.u12 = __ffma2_rn(s6, s6, a.u12); a.u6 = __fadd2_rn(a.u6, s6);
        a.w0 = __ffma2_rn(tx, dx, a.w0); a.w1 = __ffma2_rn(ty, dy, a.w1); a.w2 = __ffma2_rn(tz, dz, a.w2);
        a.w3 = __ffma2_rn(tx, dy, a.w3); a.w4 = __ffma2_rn(tx, dz, a.w4); a.w5 = __ffma2_rn(ty, dz, a.w5);
        a.cnt += (far_a ? 1u : 0u) + (far_b ? 1u : 0u);
      }
    }
    __syncwarp();
    v3_eval_close<DIGEST>(g, ev, pc, sm, A, (int)((cqa - cq0) >> 6), lane);
    __syncwarp();
  }
}

// Filter groups of 8 from group k until some lane's queue is nearly full or K8
// is reached; returns the next group index.  Only this loop depends on S.
template <int S>
__device__ __forceinline__ int v3_filter_until_full(const V3Pair& pc, uint32_t& sa, uint32_t& t, uint32_t& qa,
                                                    uint32_t qlim, int k, int K8) {
  while (k < K8) {
    v3_filter8<S>(pc, sa, t, qa);
    k += 8;
    if (__any_sync(0xffffffffu, qa > qlim)) break;
  }
  return k;
}

__device__ __forceinline__ int v3_filter_dispatch(const V3Pair& pc, uint32_t& sa, uint32_t& t, uint32_t& qa,
                                                  uint32_t qlim, int k, int K8, int S) {
  switch (S) {
    case 1: return v3_filter_until_full<1>(pc, sa, t, qa, qlim, k, K8);
    case 2: return v3_filter_until_full<2>(pc, sa, t, qa, qlim, k, K8);
    case 3: return v3_filter_until_full<3>(pc, sa, t, qa, qlim, k, K8);
    case 4: return v3_filter_until_full<4>(pc, sa, t, qa, qlim, k, K8);
    case 5: return v3_filter_until_full<5>(pc, sa, t, qa, qlim, k, K8);
    case 6: return v3_filter_until_full<6>(pc, sa, t, qa, qlim, k, K8);
    case 7: return v3_filter_until_full<7>(pc, sa, t, qa, qlim, k, K8);
    default: return v3_filter_until_full<8>(pc, sa, t, qa, qlim, k, K8);
  }
}

// Filter + evaluate one staged chunk: rounds of (filter until a queue is nearly
// full, evaluate every lane's queue); one evaluation body for all S.
template <bool DIGEST>
__device__ __forceinline__ void v3_chunk(const Geom& g, const V3Env& ev, const V3Pair& pc, V3Smem& sm, Acc3& A,
                                         Acc3f& a, int s, int S, int K8, int lane) {
  uint32_t sa = smem_u32(&sm.stage[0]) + 16u * (uint32_t)s;
  uint32_t t = (uint32_t)s;
  const uint32_t q0 = smem_u32(&sm.queue[0][lane]);
  const uint32_t qlim = q0 + 64u * (V3_QCAP - 8);
  int k = 0;
  do {
    uint32_t qa = q0;
    k = v3_filter_dispatch(pc, sa, t, qa, qlim, k, K8, S);
    __syncwarp();
    V3CHK(qa <= q0 + 64u * V3_QCAP, "queue overflow n=%d k=%d K8=%d", (int)((qa - q0) >> 6), k, K8);
    v3_eval<DIGEST>(g, ev, pc, sm, A, a, (int)((qa - q0) >> 6), lane);
  } while (k < K8);
}

__device__ __forceinline__ uint64_t shfl_u64(uint64_t x, int src) {
  return ((uint64_t)__shfl_sync(0xffffffffu, (uint32_t)(x >> 32), src) << 32) |
         (uint64_t)__shfl_sync(0xffffffffu, (uint32_t)x, src);
}

template <bool DIGEST>
__global__ void __launch_bounds__(32, V3_MINB)
k_pairs_v3(const double4* __restrict__ u, const float4* __restrict__ u32, const uint32_t* __restrict__ cs,
           const float4* __restrict__ qs, const uint32_t* __restrict__ nh, const uint32_t* __restrict__ gid,
           float4* __restrict__ Fout, double* __restrict__ bpart, uint32_t* __restrict__ dcnt,
           uint64_t* __restrict__ dhs, uint64_t* __restrict__ dhx, const __grid_constant__ Geom g, int cpb, int bpl,
           int layer0) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int lane = threadIdx.x & 31;
  V3Smem& sm = *reinterpret_cast<V3Smem*>(smraw);

  const int l1 = g.dims[0], l2 = g.dims[1];
  const int layer = layer0 + (int)(blockIdx.x / bpl);
  const int chunk = (int)blockIdx.x - (layer - layer0) * bpl;
  const int per_layer = l1 * l2;
  const int cbeg = chunk * cpb;
  const int cend = min(per_layer, cbeg + cpb);

  V3Env ev;
  ev.qs = qs;
  ev.nh = nh;
  ev.gid = gid;
  ev.u64 = u;
  ev.ntot = cs[g.ncells];
  ev.lo64 = g.rc2 * (1.0 - K3_BAND64);
  V3Lane& LN = sm.ln[lane];
  ev.hi64 = g.rc2 * (1.0 + K3_BAND64);
  const float hi32 = (float)g.band_hi;
  const float inf32 = __int_as_float(0x7f800000);

  double tU = 0, tW[6] = {0, 0, 0, 0, 0, 0}, tI = 0, tC = 0, tS = 0, tR = 0, tNF = 0;
  if (lane == 0) {  // permanent far element: pads the evaluations (far bracket, j = i)
    sm.stage[V3_DUMMY] = far4<float>();
    sm.sent[V3_DUMMY] = K3_MAXE - 1;
    sm.e_B[K3_MAXE - 1][0] = 1e150; sm.e_B[K3_MAXE - 1][1] = 1e150; sm.e_B[K3_MAXE - 1][2] = 1e150;
  }
  __syncwarp();

  for (int cl = cbeg; cl < cend; ++cl) {
    const int a0 = cl % l1, a1 = cl / l1, a2 = layer;
    const uint32_t cid = (uint32_t)cl + (uint32_t)per_layer * (uint32_t)layer;
    const int nst = build_entries(g, a0, a1, a2, sm, lane);
    V3CHK(nst <= 36 && cid < g.ncells, "nst=%d cid=%u", nst, cid);
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

    for (int ib0 = 0; ib0 < ni; ib0 += 32) {
      const int nb = min(32, ni - ib0);
      const int NP = (nb + 1) >> 1;
      const int S = min(V3_MAXS, 32 / NP);
      const int p = lane % NP;
      const bool act = lane < S * NP;
      const int s = act ? lane / NP : 0;
      const bool hasb = 2 * p + 1 < nb;
      V3Pair pc;
      pc.ia = ibase + ib0 + 2 * p;
      pc.ib = hasb ? pc.ia + 1 : pc.ia;
      V3CHK(pc.ib < ev.ntot && pc.ia < ev.ntot, "pair ia=%u ib=%u ntot=%u ni=%d nb=%d p=%d", pc.ia, pc.ib, ev.ntot, ni, nb, p);
      {
        const double4 ua = u[pc.ia], ub = u[pc.ib];
        const float4 fa = u32[pc.ia];
        float4 fb = u32[pc.ib];
        LN.ua[0] = ua.x; LN.ua[1] = ua.y; LN.ua[2] = ua.z;
        LN.ub[0] = ub.x; LN.ub[1] = ub.y; LN.ub[2] = ub.z;
        if (!hasb) fb = make_float4(-1e30f, -1e30f, -1e30f, 0.f);  // ghost b: r^2 = inf against every element (staged sentinels sit at +1e30)
        pc.nx = make_float2(-fa.x, -fb.x);
        pc.ny = make_float2(-fa.y, -fb.y);
        pc.nz = make_float2(-fa.z, -fb.z);
        pc.cx = make_float2(act ? -2.0f * fa.x : 0.0f, (act && hasb) ? -2.0f * fb.x : 0.0f);
        pc.cy = make_float2(act ? -2.0f * fa.y : 0.0f, (act && hasb) ? -2.0f * fb.y : 0.0f);
        pc.cz = make_float2(act ? -2.0f * fa.z : 0.0f, (act && hasb) ? -2.0f * fb.z : 0.0f);
        // ghost lanes / ghost b: +inf never sets the sign bit
        pc.uuh = make_float2(act ? fmaf(fa.z, fa.z, fmaf(fa.y, fa.y, fa.x * fa.x)) - hi32 : inf32,
                             (act && hasb) ? fmaf(fb.z, fb.z, fmaf(fb.y, fb.y, fb.x * fb.x)) - hi32 : inf32);
        pc.nha = (g.variant == 1) ? nh[pc.ia] : 0u;
        pc.nhb = (g.variant == 1) ? nh[pc.ib] : 0u;
      }
      Acc3 A;
      for (int c = 0; c < 3; ++c) { LN.fa[c] = 0.0; LN.fb[c] = 0.0; }
      LN.u = 0.0;
      for (int c = 0; c < 6; ++c) LN.w[c] = 0.0;
      A.cnt = A.nrc = A.cna = A.cnb = 0u;
      A.hsa = A.hxa = A.hsb = A.hxb = 0ull;
      Acc3f a;
      {
        const float2 z = make_float2(0.f, 0.f);
        a.fx = z; a.fy = z; a.fz = z; a.u12 = z; a.u6 = z;
        a.w0 = z; a.w1 = z; a.w2 = z; a.w3 = z; a.w4 = z; a.w5 = z;
        a.cnt = 0u;
      }

      int e0 = 0;
      while (e0 < nst) {
        const uint32_t base_off = sm.e_off[e0];
        int e1 = e0;
        for (int eb = e0; eb < nst; eb += 32) {
          const int e = eb + lane;
          const bool fits = e < nst && (sm.e_off[e] + sm.e_cnt[e] - base_off) <= (uint32_t)V3_CAP;
          const int nfit = __popc(__ballot_sync(0xffffffffu, fits));  // the fitting entries are a prefix
          e1 = eb + nfit;
          if (nfit < 32) break;
        }
        if (e1 == e0) e1 = e0 + 1;  // unreachable: a cell holds fewer than V3_CAP particles
        const uint32_t ctot = (e1 < nst ? sm.e_off[e1] : tot) - base_off;
        // stage: entry id per element and fp32 brackets, then a flattened coalesced copy
        for (int eb = e0; eb < e1; eb += 32) {
          const int e = eb + lane;
          if (e < e1) {
            const uint32_t dst = sm.e_off[e] - base_off, cnt = sm.e_cnt[e];
            for (uint32_t k = 0; k < cnt; ++k) sm.sent[dst + k] = (uint8_t)e;
            sm.Bf[e][0] = (float)sm.e_B[e][0];
            sm.Bf[e][1] = (float)sm.e_B[e][1];
            sm.Bf[e][2] = (float)sm.e_B[e][2];
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
            V3CHK(!v || jj[r] < ev.ntot, "stage jj=%u t=%u e=%d", jj[r], tt[r], ee[r]);
            pp[r] = v ? u32[jj[r]] : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            if (tt[r] < ctot) {
              const float x = pp[r].x + sm.Bf[ee[r]][0], y = pp[r].y + sm.Bf[ee[r]][1], z = pp[r].z + sm.Bf[ee[r]][2];
              sm.stage[tt[r]] = make_float4(x, y, z, fmaf(z, z, fmaf(y, y, x * x)));
            }
          }
        }
        // far sentinels: the unrolled filter reads t < K8 S <= ctot + 8 S - 1
        const int K = (int)((ctot + S - 1) / S);
        const int K8 = (K + 7) & ~7;
        const int npad = K8 * S - (int)ctot;
        V3CHK(npad >= 0 && (int)ctot + npad <= V3_DUMMY && S >= 1 && S <= V3_MAXS, "pad ctot=%u npad=%d S=%d", ctot, npad, S);
        for (int q = lane; q < npad; q += 32) sm.stage[ctot + q] = far4<float>();
        __syncwarp();
        pc.base_off = base_off;
        v3_chunk<DIGEST>(g, ev, pc, sm, A, a, s, S, K8, lane);
        __syncwarp();
        e0 = e1;
      }
      fold3(LN, A, a);
      __syncwarp();
      double fax = LN.fa[0], fay = LN.fa[1], faz = LN.fa[2], fbx = LN.fb[0], fby = LN.fb[1], fbz = LN.fb[2];
      double uacc = LN.u, w0 = LN.w[0], w1 = LN.w[1], w2 = LN.w[2], w3 = LN.w[3], w4 = LN.w[4], w5 = LN.w[5];

      // combine the S streams of each pair: fixed binary tree over s (log2 S shuffle steps)
      for (int o = 1; o < S; o <<= 1) {
        const bool take = act && ((s & (2 * o - 1)) == 0) && (s + o < S);
        const int src = (lane + o * NP) & 31;
        fax = shfl_comb(fax, src, take); fay = shfl_comb(fay, src, take);
        faz = shfl_comb(faz, src, take); fbx = shfl_comb(fbx, src, take);
        fby = shfl_comb(fby, src, take); fbz = shfl_comb(fbz, src, take);
        uacc = shfl_comb(uacc, src, take);
        w0 = shfl_comb(w0, src, take); w1 = shfl_comb(w1, src, take);
        w2 = shfl_comb(w2, src, take); w3 = shfl_comb(w3, src, take);
        w4 = shfl_comb(w4, src, take); w5 = shfl_comb(w5, src, take);
        const uint32_t c2 = __shfl_sync(0xffffffffu, A.cnt, src);
        const uint32_t r2c = __shfl_sync(0xffffffffu, A.nrc, src);
        if (take) { A.cnt += c2; A.nrc += r2c; }
        if (DIGEST) {
          const uint32_t ca = __shfl_sync(0xffffffffu, A.cna, src), cb = __shfl_sync(0xffffffffu, A.cnb, src);
          const uint64_t h1 = shfl_u64(A.hsa, src), h2 = shfl_u64(A.hxa, src);
          const uint64_t h3 = shfl_u64(A.hsb, src), h4 = shfl_u64(A.hxb, src);
          if (take) { A.cna += ca; A.cnb += cb; A.hsa += h1; A.hxa ^= h2; A.hsb += h3; A.hxb ^= h4; }
        }
      }
      const bool owner = act && s == 0;
      // R11/R12 factors: U = 2 eps sum s6(s6-1) - cnt u_shift / 2; W = sum fr d d / 2
      const double Ul = 2.0 * g.eps * uacc - 0.5 * g.ushift * (double)A.cnt;
      if (owner) {
        Fout[pc.ia] = make_float4((float)(g.Q[0] * fax + g.Q[1] * fay + g.Q[2] * faz),
                                  (float)(g.Q[3] * fax + g.Q[4] * fay + g.Q[5] * faz),
                                  (float)(g.Q[6] * fax + g.Q[7] * fay + g.Q[8] * faz), 0.0f);
        if (hasb)
          Fout[pc.ib] = make_float4((float)(g.Q[0] * fbx + g.Q[1] * fby + g.Q[2] * fbz),
                                    (float)(g.Q[3] * fbx + g.Q[4] * fby + g.Q[5] * fbz),
                                    (float)(g.Q[6] * fbx + g.Q[7] * fby + g.Q[8] * fbz), 0.0f);
        if (DIGEST) {
          dcnt[pc.ia] = A.cna; dhs[pc.ia] = A.hsa; dhx[pc.ia] = A.hxa;
          if (hasb) { dcnt[pc.ib] = A.cnb; dhs[pc.ib] = A.hsb; dhx[pc.ib] = A.hxb; }
        }
      }
      const double fchk = owner ? fax + fay + faz + fbx + fby + fbz + Ul : 0.0;
      if (owner) {
        tU += Ul;
        tW[0] += 0.5 * w0; tW[1] += 0.5 * w1; tW[2] += 0.5 * w2;
        tW[3] += 0.5 * w3; tW[4] += 0.5 * w4; tW[5] += 0.5 * w5;
        tI += (double)A.cnt;
        tR += (double)A.nrc;
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
