// slab_dc.cuh -- the host-synchronization-free slab step.
// Included at the end of nemdcell.cu (after nccl_slab.cuh).
//
// The counts of the slab step (own particles, migration and halo records) never leave the device:
//  * the own count lives in the context's device word sd[SD_N]; every kernel over own particles is
//    launched over the rank's capacity and reads it (the `dn` arguments of kernels.cuh);
//  * a migration / halo message is a fixed-capacity buffer whose first record is a header carrying the
//    record count (uint32 at byte 0); NCCL moves the whole (1 + cap)-record buffer, so the sizes of the
//    sends and receives are known on the host without reading any count;
//  * the receivers read the headers on the device (unpack, K1 of the halo, the cell ranges);
//  * forces: the own particles are sorted to FIXED slots [H, H + n_own), H = hcap for each halo layer
//    that precedes the own layers in cell order (0, 1 or 2 of them), so the interior layers' pair kernel
//    runs before the halo counts are known; the halo particles preceding the own ones end at H
//    (right-aligned), the following ones start at H + n_own (device offsets).  Cell starts stay one
//    monotone exclusive scan (plus a device-side offset), so every K3 kernel runs unchanged and the
//    cell contents -- hence F, U, W and the per-layer partials -- are bitwise those of one device.
// Overflow of a message or of the own capacity sets a bit in sd[SD_FLAGS] (records are dropped, never
// written out of bounds); nc_sd_status reads count and flags -- the only host synchronization, taken
// when the caller wants it (e.g. once per run, or with the energies).

namespace nc {

enum : int {
  SD_N = 0,        // own particles
  SD_FLAGS = 1,    // 1: migration message overflow, 2: halo message overflow, 4: moved > 1 layer,
                   // 8: own capacity overflow
  SD_DB = 2,       // device part of the cell-start offset of the end phase (H - n_pre)
  SD_OWN0 = 3,     // sorted slots of the own particles [SD_OWN0, SD_OWN1)
  SD_OWN1 = 4,
  SD_PRE0 = 5,     // sorted slots of the halo particles preceding the own ones
  SD_PRE1 = 6,
  SD_POST0 = 7,    // ... and following them
  SD_POST1 = 8,
  SD_WORDS = 16
};
enum : uint32_t { SDF_MIG = 1u, SDF_HALO = 2u, SDF_FAR = 4u, SDF_OWN = 8u };

__device__ __forceinline__ uint32_t msg_count(const void* buf) { return *(const uint32_t*)buf; }

__global__ void k_sd_set(uint32_t* __restrict__ sd, uint32_t n) {
  if (threadIdx.x == 0) { sd[SD_N] = n; sd[SD_FLAGS] = 0u; }
}

// after a partition: class 0 stays (migration) and the record counts go into the message headers
// (clamped to the capacity, overflow flagged)
__global__ void k_sd_part_finish(const uint32_t* __restrict__ tot, uint32_t* __restrict__ sd, void* __restrict__ lo,
                                 void* __restrict__ hi, uint32_t cap, int migration) {
  if (threadIdx.x != 0) return;
  uint32_t f = 0u;
  if (tot[1] > cap || tot[2] > cap) f |= migration ? SDF_MIG : SDF_HALO;
  if (migration) {
    if (tot[3]) f |= SDF_FAR;
    sd[SD_N] = tot[0];
  }
  *(uint32_t*)lo = min(tot[1], cap);
  *(uint32_t*)hi = min(tot[2], cap);
  sd[SD_FLAGS] |= f;
}

// append the migration records of both messages after the own particles (lo first, then hi)
template <typename T>
__global__ void k_sd_unpack(const typename V4<T>::t* __restrict__ rlo, const typename V4<T>::t* __restrict__ rhi,
                            uint32_t cap, T* __restrict__ q, T* __restrict__ p, uint32_t* __restrict__ gid, int64_t ncap,
                            uint32_t* __restrict__ sd) {
  const int m = blockIdx.y;  // 0: from the lower neighbour, 1: from the upper one
  const typename V4<T>::t* r = m ? rhi : rlo;
  const uint32_t cnt = min(msg_count(r), cap);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cnt) return;
  const int64_t dst = (int64_t)sd[SD_N] + (m ? (int64_t)min(msg_count(rlo), cap) : 0) + i;
  if (dst >= ncap) {
    atomicOr(&sd[SD_FLAGS], SDF_OWN);
    return;
  }
  const typename V4<T>::t a = r[2 * (1 + i)], b = r[2 * (1 + i) + 1];  // record 0 is the header
  q[3 * dst] = a.x; q[3 * dst + 1] = a.y; q[3 * dst + 2] = a.z;
  p[3 * dst] = b.x; p[3 * dst + 1] = b.y; p[3 * dst + 2] = b.z;
  gid[dst] = w_to_idx(a.w);
}

template <typename T>
__global__ void k_sd_absorb_finish(const typename V4<T>::t* __restrict__ rlo, const typename V4<T>::t* __restrict__ rhi,
                                   uint32_t cap, int64_t ncap, uint32_t* __restrict__ sd) {
  if (threadIdx.x != 0) return;
  const int64_t n = (int64_t)sd[SD_N] + min(msg_count(rlo), cap) + min(msg_count(rhi), cap);
  sd[SD_N] = (uint32_t)min(n, ncap);
}

// sorted-slot ranges of the begin phase: own [H, H + n_own)
__global__ void k_sd_ranges_begin(uint32_t* __restrict__ sd, uint32_t H) {
  if (threadIdx.x != 0) return;
  sd[SD_OWN0] = H;
  sd[SD_OWN1] = H + sd[SD_N];
}

// the end phase: halo counts from the received headers; halo particles preceding the own ones end at H
template <typename T>
__global__ void k_sd_ranges_end(uint32_t* __restrict__ sd, const void* __restrict__ hlo, const void* __restrict__ hhi,
                                uint32_t cap, int lo_precedes, int hi_precedes, uint32_t H) {
  if (threadIdx.x != 0) return;
  const uint32_t n1 = min(msg_count(hlo), cap), n2 = min(msg_count(hhi), cap);
  const uint32_t pre = (lo_precedes ? n1 : 0u) + (hi_precedes ? n2 : 0u), post = n1 + n2 - pre;
  sd[SD_DB] = H - pre;  // added (mod 2^32) to the cell starts of the full scan
  sd[SD_PRE0] = H - pre;
  sd[SD_PRE1] = H;
  sd[SD_POST0] = H + sd[SD_N];
  sd[SD_POST1] = H + sd[SD_N] + post;
}

// the own particles adopt their sorted (cell, gid) order: slot k = s - H of the outputs takes sorted slot s
// (wrapped q, p gathered from the local order, gid, F) -- the next step's kernels then read spatially
// ordered arrays (the single-device path keeps its resident state sorted the same way)
template <typename T>
__global__ void k_sd_adopt(const uint32_t* __restrict__ sd, const typename V4<T>::t* __restrict__ sq,
                           const uint32_t* __restrict__ sgid, const typename V4<T>::t* __restrict__ sF,
                           const uint32_t* __restrict__ sidx, const T* __restrict__ p, T* __restrict__ q_out,
                           T* __restrict__ p_out, uint32_t* __restrict__ gid_out, T* __restrict__ F_out) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t s = (int64_t)sd[SD_OWN0] + k;
  if (s >= (int64_t)sd[SD_OWN1]) return;
  const uint32_t i = sidx[s];
  const typename V4<T>::t a = sq[s], f = sF[s];
  q_out[3 * k] = a.x; q_out[3 * k + 1] = a.y; q_out[3 * k + 2] = a.z;
  p_out[3 * k] = p[3 * (int64_t)i]; p_out[3 * k + 1] = p[3 * (int64_t)i + 1]; p_out[3 * k + 2] = p[3 * (int64_t)i + 2];
  gid_out[k] = sgid[s];
  F_out[3 * k] = f.x; F_out[3 * k + 1] = f.y; F_out[3 * k + 2] = f.z;
}

// deterministic class partition of the own particles with the count on the device (no host read):
// the grid covers ncap
template <typename T>
nc_status partition_sd(nc_ctx* ctx, int64_t ncap, const T* q, const T* p, const uint32_t* gid, T* q0, T* p0,
                       uint32_t* g0, typename V4<T>::t* r1, typename V4<T>::t* r2, int words, int64_t rcap) {
  cudaStream_t s = ctx->stream;
  const uint32_t* dn = ctx->sd + SD_N;
  const int64_t nb = (ncap + PART_T - 1) / PART_T;
  k_class_count<<<(unsigned)nb, PART_T, 0, s>>>(ncap, nb, ctx->cls, ctx->pbcnt, dn);
  LAUNCHED();
  nc_status sst = launch_scan_raw(ctx, ctx->pbcnt, 4 * nb, ctx->pboff);
  if (sst) return sst;
  k_class_totals<<<1, 32, 0, s>>>(ctx->pboff, nb, ctx->ptot);
  LAUNCHED();
  k_class_scatter<T><<<(unsigned)nb, PART_T, 0, s>>>(ncap, ctx->cls, ctx->pboff, q, p, gid, q0, p0, g0, r1, r2, words,
                                                     dn, rcap);
  LAUNCHED();
  return NC_OK;
}

template <typename T>
nc_status sd_forces_begin_t(nc_ctx* ctx, const T* q, const uint32_t* gid, int64_t ncap, int64_t hcap, int klo, int khi) {
  cudaStream_t s = ctx->stream;
  const Geom& g = ctx->g;
  if (ncap + 2 * hcap > ctx->cap) return fail(ctx, NC_E_OOM, "own + 2 halo capacities exceed the context capacity");
  const int64_t C = g.ncells, per_layer = (int64_t)g.dims[0] * g.dims[1];
  const int l3 = g.dims[2];
  const uint32_t* dn = ctx->sd + SD_N;
  CK(cudaMemsetAsync(ctx->counts, 0, sizeof(uint32_t) * (C + 1), s));
  ctx->counts_clean = 0;
  typename V4<T>::t* wq = (typename V4<T>::t*)ctx->wq;
  prof_begin(ctx);
  k_wrap_key_src<T><<<nblk(ncap, 256), 256, 0, s>>>(ncap, q, 3, gid, 0, wq, ctx->gin, ctx->key, ctx->slot, ctx->counts,
                                                   g, dn);
  LAUNCHED();
  prof_end(ctx, NC_K_WRAPKEY);
  {
    nc_status sst = launch_scan(ctx, ctx->counts, C, ctx->cs);
    if (sst) return sst;
  }
  // halo layers preceding the own cells in cell order: the lower one unless on the seam, the upper one
  // when it wraps to layer 0; each reserves hcap slots before the own particles
  const int L_lo = (klo - 1 + l3) % l3, L_hi = khi % l3;
  const int lo_pre = L_lo < klo ? 1 : 0, hi_pre = L_hi < klo ? 1 : 0;
  const int64_t H = (int64_t)(lo_pre + hi_pre) * hcap;
  if (H > 0) {
    const int64_t c0 = (int64_t)klo * per_layer;
    k_add_range<<<nblk(C + 1 - c0, 256), 256, 0, s>>>(ctx->cs, c0, C + 1, (uint32_t)H);
    LAUNCHED();
  }
  k_sd_ranges_begin<<<1, 32, 0, s>>>(ctx->sd, (uint32_t)H);
  LAUNCHED();
  prof_begin(ctx);
  k_scatter<<<nblk(ncap, 256), 256, 0, s>>>(ncap, ctx->key, ctx->slot, ctx->cs, ctx->gin, ctx->srec, 0, dn);
  LAUNCHED();
  prof_end(ctx, NC_K_SCATTER);
  prof_begin(ctx);
  k_rank_gather<T><<<nblk(ncap, 256), 256, 0, s>>>(ncap, ctx->srec, ctx->cs, wq, nullptr, (typename V4<T>::t*)ctx->sq,
                                                  nullptr, ctx->sgid, ctx->u, ctx->u32, ctx->nh, g, ctx->sidx, 0,
                                                  ctx->sd + SD_OWN0);
  LAUNCHED();
  prof_end(ctx, NC_K_RANKGATHER);
  ctx->sd_ncap = ncap;
  ctx->sd_hcap = hcap;
  ctx->sd_H = H;
  ctx->sd_pre = (lo_pre ? 1 : 0) | (hi_pre ? 2 : 0);
  ctx->slab_klo = klo;
  ctx->slab_khi = khi;
  ctx->sd_open = true;
  // the pair-kernel choice from host-side hints (the last known own count: never a device read)
  ctx->occ_hint = (double)ctx->sd_n_hint / ((double)per_layer * (double)(khi - klo));
  ctx->n_last = ctx->sd_n_hint;
  if (khi - klo > 2) {  // interior layers: their stencils see own cells only
    nc_status st = launch_pairs<T, false>(ctx, (const typename V4<T>::t*)ctx->sq, ctx->sgid,
                                          (typename V4<T>::t*)ctx->sF, klo + 1, khi - klo - 2, klo, false);
    if (st) return st;
  }
  return NC_OK;
}

template <typename T>
nc_status sd_forces_end_t(nc_ctx* ctx, const void* h1, const void* h2, T* F, double* parts, const T* p_in = nullptr,
                          T* q_out = nullptr, T* p_out = nullptr, uint32_t* gid_out = nullptr) {
  cudaStream_t s = ctx->stream;
  const Geom& g = ctx->g;
  const int64_t ncap = ctx->sd_ncap, hcap = ctx->sd_hcap, H = ctx->sd_H, C = g.ncells;
  const int klo = ctx->slab_klo, khi = ctx->slab_khi;
  ctx->sd_open = false;
  typename V4<T>::t* wq = (typename V4<T>::t*)ctx->wq;
  // halo records (1 word: q + gid) after the header record; local indices [ncap, ncap + 2 hcap)
  const T* q1 = (const T*)h1 + 4;
  const T* q2 = (const T*)h2 + 4;
  prof_begin(ctx);
  k_wrap_key_src<T><<<nblk(hcap, 256), 256, 0, s>>>(hcap, q1, 4, nullptr, ncap, wq, ctx->gin, ctx->key, ctx->slot,
                                                   ctx->counts, g, (const uint32_t*)h1);
  k_wrap_key_src<T><<<nblk(hcap, 256), 256, 0, s>>>(hcap, q2, 4, nullptr, ncap + hcap, wq, ctx->gin, ctx->key,
                                                   ctx->slot, ctx->counts, g, (const uint32_t*)h2);
  LAUNCHED();
  prof_end(ctx, NC_K_WRAPKEY);
  {  // all counts: the full scan, then + (H - n_pre) everywhere: the own cells' starts come out as in begin
    nc_status sst = launch_scan(ctx, ctx->counts, C, ctx->cs);
    if (sst) return sst;
  }
  k_sd_ranges_end<T><<<1, 32, 0, s>>>(ctx->sd, h1, h2, (uint32_t)hcap, ctx->sd_pre & 1, (ctx->sd_pre >> 1) & 1,
                                      (uint32_t)H);
  LAUNCHED();
  k_add_range<<<nblk(C + 1, 256), 256, 0, s>>>(ctx->cs, 0, C + 1, 0u, ctx->sd + SD_DB);
  LAUNCHED();
  prof_begin(ctx);
  k_scatter<<<nblk(hcap, 256), 256, 0, s>>>(hcap, ctx->key, ctx->slot, ctx->cs, ctx->gin, ctx->srec, ncap,
                                            (const uint32_t*)h1);
  k_scatter<<<nblk(hcap, 256), 256, 0, s>>>(hcap, ctx->key, ctx->slot, ctx->cs, ctx->gin, ctx->srec, ncap + hcap,
                                            (const uint32_t*)h2);
  LAUNCHED();
  prof_end(ctx, NC_K_SCATTER);
  prof_begin(ctx);
  k_rank_gather<T><<<nblk(2 * hcap, 256), 256, 0, s>>>(2 * hcap, ctx->srec, ctx->cs, wq, nullptr,
                                                      (typename V4<T>::t*)ctx->sq, nullptr, ctx->sgid, ctx->u,
                                                      ctx->u32, ctx->nh, g, ctx->sidx, 0, ctx->sd + SD_PRE0);
  k_rank_gather<T><<<nblk(2 * hcap, 256), 256, 0, s>>>(2 * hcap, ctx->srec, ctx->cs, wq, nullptr,
                                                      (typename V4<T>::t*)ctx->sq, nullptr, ctx->sgid, ctx->u,
                                                      ctx->u32, ctx->nh, g, ctx->sidx, 0, ctx->sd + SD_POST0);
  LAUNCHED();
  prof_end(ctx, NC_K_RANKGATHER);
  ctx->last_in_gid = ctx->gin;
  ctx->last_resident = false;
  ctx->have_cells = true;
  nc_status st = launch_pairs<T, false>(ctx, (const typename V4<T>::t*)ctx->sq, ctx->sgid, (typename V4<T>::t*)ctx->sF,
                                        klo, 1, klo, khi - klo == 1);
  if (st) return st;
  if (khi - klo > 1) {
    st = launch_pairs<T, false>(ctx, (const typename V4<T>::t*)ctx->sq, ctx->sgid, (typename V4<T>::t*)ctx->sF,
                                khi - 1, 1, klo, true);
    if (st) return st;
  }
  if (F && q_out) {  // adopt the sorted order (q, p, gid, F of the own particles)
    prof_begin(ctx);
    k_sd_adopt<T><<<nblk(ncap, 256), 256, 0, s>>>(ctx->sd, (const typename V4<T>::t*)ctx->sq, ctx->sgid,
                                                 (const typename V4<T>::t*)ctx->sF, ctx->sidx, p_in, q_out, p_out,
                                                 gid_out, F);
    LAUNCHED();
    prof_end(ctx, NC_K_OTHER);
  } else if (F) {
    prof_begin(ctx);
    k_unsort_idx<T><<<nblk(ncap, 256), 256, 0, s>>>(ncap, (const typename V4<T>::t*)ctx->sF, ctx->sidx, 0, F,
                                                   ctx->sd + SD_OWN0);
    LAUNCHED();
    prof_end(ctx, NC_K_OTHER);
  }
  if (parts) {  // the energies were asked for: the one synchronization of this evaluation
    CK(cudaMemcpyAsync(parts, ctx->lpart, sizeof(double) * NPART * (size_t)(khi - klo), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  return NC_OK;
}

}  // namespace nc

extern "C" {

nc_status nc_sd_load(nc_ctx* ctx, int64_t n) {
  if (!ctx || n < 0 || n > 0xffffffffLL) return fail(ctx, NC_E_ARG, "bad count");
  k_sd_set<<<1, 32, 0, ctx->stream>>>(ctx->sd, (uint32_t)n);
  LAUNCHED();
  ctx->sd_n_hint = n;
  return NC_OK;
}

nc_status nc_sd_status(nc_ctx* ctx, int64_t* n_own, uint32_t* flags) {
  if (!ctx) return fail(ctx, NC_E_ARG, "null ctx");
  uint32_t h[2];
  CK(cudaMemcpyAsync(h, ctx->sd, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (n_own) *n_own = h[SD_N];
  if (flags) *flags = h[SD_FLAGS];
  ctx->sd_n_hint = h[SD_N];
  if (h[SD_FLAGS] & SDF_FAR) return fail(ctx, NC_E_STATE, "a particle moved more than one cell layer past its slab");
  if (h[SD_FLAGS] & (SDF_MIG | SDF_HALO)) return fail(ctx, NC_E_OOM, "a migration or halo message overflowed");
  if (h[SD_FLAGS] & SDF_OWN) return fail(ctx, NC_E_OOM, "own particles exceed the capacity");
  return NC_OK;
}

nc_status nc_sd_kick_drift(nc_ctx* ctx, void* q, void* p, const void* F, int64_t ncap, double dt_prev, double dt) {
  if (!ctx || (ncap > 0 && (!q || !p || !F))) return fail(ctx, NC_E_ARG, "null argument");
  if (!ctx->have_flow && !ctx->have_box) return fail(ctx, NC_E_STATE, "nc_set_flow first");
  if (!(dt > 0) || dt_prev < 0) return fail(ctx, NC_E_ARG, "dt must be > 0 and dt_prev >= 0");
  K3Kick pk{};
  if (dt_prev > 0) {
    SllodParams pp;
    sllod_params(ctx, dt_prev, pp);
    for (int e = 0; e < 9; ++e) pk.Em[e] = pp.Em[e];
    pk.hd = 0.5 * dt_prev;
  }
  SllodParams sp;
  sllod_params(ctx, dt, sp);
  double Lnew[9];
  box_advance(ctx->pol, ctx->A, ctx->t + dt, Lnew);
  nc_status st = apply_box(ctx, Lnew);
  if (st) return st;
  ctx->t += dt;
  if (ncap > 0) {
    prof_begin(ctx);
    if (ctx->cfg.prec == NC_F32)
      k_kick_drift3<float><<<nblk(ncap, 256), 256, 0, ctx->stream>>>(ncap, (float*)q, (float*)p, (const float*)F, sp,
                                                                       dt_prev > 0 ? 1 : 0, pk, ctx->sd + SD_N);
    else
      k_kick_drift3<double><<<nblk(ncap, 256), 256, 0, ctx->stream>>>(ncap, (double*)q, (double*)p, (const double*)F,
                                                                        sp, dt_prev > 0 ? 1 : 0, pk, ctx->sd + SD_N);
    LAUNCHED();
    prof_end(ctx, NC_K_KICK);
  }
  return NC_OK;
}

nc_status nc_sd_kick(nc_ctx* ctx, void* p, const void* F, int64_t ncap, double dt) {
  if (!ctx || (ncap > 0 && (!p || !F))) return fail(ctx, NC_E_ARG, "null argument");
  SllodParams sp;
  sllod_params(ctx, dt, sp);
  if (ncap > 0) {
    prof_begin(ctx);
    if (ctx->cfg.prec == NC_F32)
      k_kick3<float><<<nblk(ncap, 256), 256, 0, ctx->stream>>>(ncap, (float*)p, (const float*)F, sp, ctx->sd + SD_N);
    else
      k_kick3<double><<<nblk(ncap, 256), 256, 0, ctx->stream>>>(ncap, (double*)p, (const double*)F, sp,
                                                                ctx->sd + SD_N);
    LAUNCHED();
    prof_end(ctx, NC_K_KICK);
  }
  return NC_OK;
}

// migration: wrap + classify the own particles, stayers to (q_out, p_out, gid_out), leavers as 2-word
// records into the two messages (header + mcap records each)
nc_status nc_sd_migrate(nc_ctx* ctx, void* q, const void* p, const uint32_t* gid, int64_t ncap, int klo, int khi,
                        void* q_out, void* p_out, uint32_t* gid_out, void* msg_lo, void* msg_hi, int64_t mcap) {
  if (!ctx || !q || !p || !gid || !q_out || !p_out || !gid_out || !msg_lo || !msg_hi || mcap < 1)
    return fail(ctx, NC_E_ARG, "null argument");
  if (ncap > ctx->cap) return fail(ctx, NC_E_OOM, "capacity exceeds the context's");
  const uint32_t* dn = ctx->sd + SD_N;
  prof_begin(ctx);
  if (ctx->cfg.prec == NC_F32)
    k_slab_classify<float><<<nblk(ncap, 256), 256, 0, ctx->stream>>>(ncap, (float*)q, ctx->g, klo, khi, 0, ctx->cls,
                                                                       nullptr, dn);
  else
    k_slab_classify<double><<<nblk(ncap, 256), 256, 0, ctx->stream>>>(ncap, (double*)q, ctx->g, klo, khi, 0, ctx->cls,
                                                                        nullptr, dn);
  LAUNCHED();
  nc_status st;
  if (ctx->cfg.prec == NC_F32)
    st = partition_sd<float>(ctx, ncap, (const float*)q, (const float*)p, gid, (float*)q_out, (float*)p_out, gid_out,
                             (float4*)msg_lo + 2, (float4*)msg_hi + 2, 2, mcap);
  else
    st = partition_sd<double>(ctx, ncap, (const double*)q, (const double*)p, gid, (double*)q_out, (double*)p_out,
                              gid_out, (double4*)msg_lo + 2, (double4*)msg_hi + 2, 2, mcap);
  if (st) return st;
  k_sd_part_finish<<<1, 32, 0, ctx->stream>>>(ctx->ptot, ctx->sd, msg_lo, msg_hi, (uint32_t)mcap, 1);
  LAUNCHED();
  prof_end(ctx, NC_K_OTHER);
  return NC_OK;
}

// arrivals: both messages' records appended after the own particles
nc_status nc_sd_absorb(nc_ctx* ctx, const void* msg_lo, const void* msg_hi, int64_t mcap, void* q, void* p,
                       uint32_t* gid, int64_t ncap) {
  if (!ctx || !msg_lo || !msg_hi || !q || !p || !gid || mcap < 1) return fail(ctx, NC_E_ARG, "null argument");
  prof_begin(ctx);
  const dim3 grid((unsigned)((mcap + 255) / 256), 2);
  if (ctx->cfg.prec == NC_F32) {
    k_sd_unpack<float><<<grid, 256, 0, ctx->stream>>>((const float4*)msg_lo, (const float4*)msg_hi, (uint32_t)mcap,
                                                     (float*)q, (float*)p, gid, ncap, ctx->sd);
    k_sd_absorb_finish<float><<<1, 32, 0, ctx->stream>>>((const float4*)msg_lo, (const float4*)msg_hi,
                                                         (uint32_t)mcap, ncap, ctx->sd);
  } else {
    k_sd_unpack<double><<<grid, 256, 0, ctx->stream>>>((const double4*)msg_lo, (const double4*)msg_hi,
                                                      (uint32_t)mcap, (double*)q, (double*)p, gid, ncap, ctx->sd);
    k_sd_absorb_finish<double><<<1, 32, 0, ctx->stream>>>((const double4*)msg_lo, (const double4*)msg_hi,
                                                          (uint32_t)mcap, ncap, ctx->sd);
  }
  LAUNCHED();
  prof_end(ctx, NC_K_OTHER);
  return NC_OK;
}

// halo: the own particles of the boundary layers as 1-word records (header + hcap records each)
nc_status nc_sd_halo(nc_ctx* ctx, void* q, const uint32_t* gid, int64_t ncap, int klo, int khi, void* msg_lo,
                     void* msg_hi, int64_t hcap) {
  if (!ctx || !q || !gid || !msg_lo || !msg_hi || hcap < 1) return fail(ctx, NC_E_ARG, "null argument");
  if (khi - klo < 2) return fail(ctx, NC_E_DEGENERATE, "slab decomposition needs >= 2 cell layers per rank");
  const uint32_t* dn = ctx->sd + SD_N;
  prof_begin(ctx);
  if (ctx->cfg.prec == NC_F32)
    k_slab_classify<float><<<nblk(ncap, 256), 256, 0, ctx->stream>>>(ncap, (float*)q, ctx->g, klo, khi, 1, ctx->cls,
                                                                       nullptr, dn);
  else
    k_slab_classify<double><<<nblk(ncap, 256), 256, 0, ctx->stream>>>(ncap, (double*)q, ctx->g, klo, khi, 1, ctx->cls,
                                                                        nullptr, dn);
  LAUNCHED();
  nc_status st;
  if (ctx->cfg.prec == NC_F32)
    st = partition_sd<float>(ctx, ncap, (const float*)q, nullptr, gid, nullptr, nullptr, nullptr, (float4*)msg_lo + 1,
                             (float4*)msg_hi + 1, 1, hcap);
  else
    st = partition_sd<double>(ctx, ncap, (const double*)q, nullptr, gid, nullptr, nullptr, nullptr,
                              (double4*)msg_lo + 1, (double4*)msg_hi + 1, 1, hcap);
  if (st) return st;
  k_sd_part_finish<<<1, 32, 0, ctx->stream>>>(ctx->ptot, ctx->sd, msg_lo, msg_hi, (uint32_t)hcap, 0);
  LAUNCHED();
  prof_end(ctx, NC_K_OTHER);
  return NC_OK;
}

// the fixed-size message exchange over NCCL (no count phase): (1 + cap) records of `words` T4 words each
// way, on the communication stream after the work queued on cfg.stream; nc_slab_exchange_wait joins it
nc_status nc_sd_exchange_start(nc_ctx* ctx, const void* send_lo, const void* send_hi, void* recv_lo, void* recv_hi,
                               int64_t cap, int words) {
  if (!ctx || !send_lo || !send_hi || !recv_lo || !recv_hi || cap < 1 || words < 1)
    return fail(ctx, NC_E_ARG, "bad argument");
  if (!ctx->comm) return fail(ctx, NC_E_STATE, "nc_slab_comm_init first");
  const size_t bytes = (size_t)(1 + cap) * (size_t)words * v4size(ctx);
  CK(cudaEventRecord(ctx->ev_comm_in, ctx->stream));
  CK(cudaStreamWaitEvent(ctx->s_comm, ctx->ev_comm_in, 0));
  nc_status st = ring_exchange(ctx, send_lo, bytes, send_hi, bytes, recv_lo, bytes, recv_hi, bytes, ctx->s_comm);
  if (st) return st;
  CK(cudaEventRecord(ctx->ev_comm_out, ctx->s_comm));
  ctx->comm_pending = true;
  return NC_OK;
}

nc_status nc_sd_forces_begin(nc_ctx* ctx, const void* q, const uint32_t* gid, int64_t ncap, int64_t hcap, int klo,
                             int khi) {
  if (!ctx || !q || !gid || ncap < 1 || hcap < 1) return fail(ctx, NC_E_ARG, "null argument");
  if (!ctx->have_box) return fail(ctx, NC_E_STATE, "nc_set_box or nc_set_flow first");
  if (khi - klo < 2) return fail(ctx, NC_E_DEGENERATE, "slab decomposition needs >= 2 cell layers per rank");
  return ctx->cfg.prec == NC_F32 ? sd_forces_begin_t<float>(ctx, (const float*)q, gid, ncap, hcap, klo, khi)
                                 : sd_forces_begin_t<double>(ctx, (const double*)q, gid, ncap, hcap, klo, khi);
}

nc_status nc_sd_forces_end(nc_ctx* ctx, const void* msg_lo, const void* msg_hi, void* F, double* parts) {
  if (!ctx || !msg_lo || !msg_hi) return fail(ctx, NC_E_ARG, "null argument");
  if (!ctx->sd_open) return fail(ctx, NC_E_STATE, "nc_sd_forces_begin first");
  return ctx->cfg.prec == NC_F32 ? sd_forces_end_t<float>(ctx, msg_lo, msg_hi, (float*)F, parts)
                                 : sd_forces_end_t<double>(ctx, msg_lo, msg_hi, (double*)F, parts);
}

nc_status nc_sd_forces_end_sorted(nc_ctx* ctx, const void* msg_lo, const void* msg_hi, const void* p, void* q_out,
                                  void* p_out, uint32_t* gid_out, void* F, double* parts) {
  if (!ctx || !msg_lo || !msg_hi || !p || !q_out || !p_out || !gid_out || !F)
    return fail(ctx, NC_E_ARG, "null argument");
  if (!ctx->sd_open) return fail(ctx, NC_E_STATE, "nc_sd_forces_begin first");
  return ctx->cfg.prec == NC_F32
             ? sd_forces_end_t<float>(ctx, msg_lo, msg_hi, (float*)F, parts, (const float*)p, (float*)q_out,
                                      (float*)p_out, gid_out)
             : sd_forces_end_t<double>(ctx, msg_lo, msg_hi, (double*)F, parts, (const double*)p, (double*)q_out,
                                       (double*)p_out, gid_out);
}

}  // extern "C"
