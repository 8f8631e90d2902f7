// nccl_slab.cuh -- the slab decomposition's data plane behind the C-ABI:
// NCCL point-to-point halo / migration exchange with the ring neighbours r-1, r+1 and the
// all-gather of the per-layer partials, on the library's own streams.  The host driver only
// broadcasts the 128-byte unique id (torch.distributed); every byte of the data plane moves here.
//
// NCCL is loaded at run time (dlopen; the copy torch already loaded if any, else torch's wheel, else
// the system one), so the library carries no link-time NCCL dependency and single-GPU use needs none.
// Included at the end of nemdcell.cu (needs the nc_ctx internals).
#pragma once
#include <dlfcn.h>
#include <nccl.h>

namespace {

struct NcclApi {
  bool tried = false, ok = false;
  std::string err;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  if (api.tried) return api;
  api.tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the copy already in the process (torch's)
  const char* env = getenv("NC_NCCL_LIB");
  if (!h && env) h = dlopen(env, RTLD_NOW);
  if (!h) {  // torch's wheel copy (this image's venv), else the loader's search path
    const char* cands[] = {"/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib/libnccl.so.2",
                           "libnccl.so.2", "libnccl.so"};
    for (const char* c : cands)
      if ((h = dlopen(c, RTLD_NOW))) break;
  }
  if (!h) {
    api.err = std::string("cannot load libnccl.so.2: ") + (dlerror() ? dlerror() : "");
    return api;
  }
  auto sym = [&](const char* n) { return dlsym(h, n); };
  api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
  api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
  api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
  api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
  api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
  api.Send = (decltype(api.Send))sym("ncclSend");
  api.Recv = (decltype(api.Recv))sym("ncclRecv");
  api.AllGather = (decltype(api.AllGather))sym("ncclAllGather");
  api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
  api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.GroupStart && api.GroupEnd && api.Send &&
           api.Recv && api.AllGather && api.GetErrorString;
  if (!api.ok) api.err = "libnccl.so.2 lacks an expected symbol";
  return api;
}

nc_status nccl_check(nc_ctx* ctx, ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return NC_OK;
  return fail(ctx, NC_E_NCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

#define NK(expr)                                          \
  do {                                                    \
    nc_status _s = nccl_check(ctx, (expr), #expr);        \
    if (_s != NC_OK) return _s;                           \
  } while (0)

// the ring exchange of one phase: to_lo -> rank r-1 (its from_hi), to_hi -> rank r+1 (its from_lo).
// Messages to one peer are matched in issue order on both sides: every rank sends to r-1 first,
// then to r+1, and receives from r+1 first, then from r-1 (so P = 1 and P = 2 pair up correctly).
nc_status ring_exchange(nc_ctx* ctx, const void* s_lo, size_t b_lo, const void* s_hi, size_t b_hi, void* r_lo,
                        size_t rb_lo, void* r_hi, size_t rb_hi, cudaStream_t s) {
  NcclApi& api = nccl();
  const int P = ctx->comm_nranks, r = ctx->comm_rank;
  const int lo = (r - 1 + P) % P, hi = (r + 1) % P;
  ncclComm_t comm = (ncclComm_t)ctx->comm;
  NK(api.GroupStart());
  NK(api.Send(s_lo, b_lo, ncclInt8, lo, comm, s));
  NK(api.Send(s_hi, b_hi, ncclInt8, hi, comm, s));
  NK(api.Recv(r_hi, rb_hi, ncclInt8, hi, comm, s));
  NK(api.Recv(r_lo, rb_lo, ncclInt8, lo, comm, s));
  NK(api.GroupEnd());
  return NC_OK;
}

}  // namespace

extern "C" {

nc_status nc_nccl_unique_id(uint8_t id[128]) {
  if (!id) return fail(nullptr, NC_E_ARG, "id is NULL");
  NcclApi& api = nccl();
  if (!api.ok) return fail(nullptr, NC_E_NCCL, api.err);
  ncclUniqueId u;
  ncclResult_t r = api.GetUniqueId(&u);
  if (r != ncclSuccess) return fail(nullptr, NC_E_NCCL, std::string("ncclGetUniqueId: ") + api.GetErrorString(r));
  static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(id, &u, 128);
  return NC_OK;
}

nc_status nc_slab_comm_init(nc_ctx* ctx, int rank, int nranks, const uint8_t id[128]) {
  if (!ctx || !id || nranks < 1 || rank < 0 || rank >= nranks) return fail(ctx, NC_E_ARG, "bad rank / nranks / id");
  if (ctx->comm) return fail(ctx, NC_E_STATE, "communicator already initialized");
  NcclApi& api = nccl();
  if (!api.ok) return fail(ctx, NC_E_NCCL, api.err);
  CK(cudaSetDevice(ctx->cfg.device));
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  ncclComm_t comm = nullptr;
  NK(api.CommInitRank(&comm, nranks, u, rank));
  ctx->comm = comm;
  ctx->comm_rank = rank;
  ctx->comm_nranks = nranks;
  CK(cudaStreamCreateWithFlags(&ctx->s_comm, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&ctx->ev_comm_in, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->ev_comm_out, cudaEventDisableTiming));
  CK(cudaMalloc(&ctx->comm_cnt, 4 * sizeof(int64_t)));
  const size_t gbytes = (size_t)nranks * (size_t)(ctx->max_layers / nranks + 2) * NPART * sizeof(double);
  CK(cudaMalloc(&ctx->comm_gather, 2 * gbytes));
  ctx->comm_gather_bytes = gbytes;
  return NC_OK;
}

// counts, then (start) the payload on the communication stream; counts[2] = records received from
// the lower / upper neighbour.  The payload reads the send buffers after the work already queued on
// cfg.stream (event), and nc_slab_exchange_wait makes cfg.stream wait for its completion.
nc_status nc_slab_exchange_start(nc_ctx* ctx, const void* send_lo, int64_t n_lo, const void* send_hi, int64_t n_hi,
                                 void* recv_lo, void* recv_hi, int64_t cap, int words, int64_t counts[2]) {
  if (!ctx || !counts || words < 1 || n_lo < 0 || n_hi < 0 || cap < 1) return fail(ctx, NC_E_ARG, "bad argument");
  if (!ctx->comm) return fail(ctx, NC_E_STATE, "nc_slab_comm_init first");
  if (n_lo > cap || n_hi > cap) return fail(ctx, NC_E_OOM, "send count above capacity");
  const size_t rec = (size_t)words * v4size(ctx);
  // phase 1: counts (device scratch: [0, 1] sent, [2, 3] received), on the communication stream
  int64_t hc[2] = {n_lo, n_hi};
  CK(cudaEventRecord(ctx->ev_comm_in, ctx->stream));
  CK(cudaStreamWaitEvent(ctx->s_comm, ctx->ev_comm_in, 0));
  CK(cudaMemcpyAsync(ctx->comm_cnt, hc, sizeof hc, cudaMemcpyHostToDevice, ctx->s_comm));
  nc_status st = ring_exchange(ctx, ctx->comm_cnt, sizeof(int64_t), ctx->comm_cnt + 1, sizeof(int64_t),
                               ctx->comm_cnt + 2, sizeof(int64_t), ctx->comm_cnt + 3, sizeof(int64_t), ctx->s_comm);
  if (st) return st;
  int64_t rc[2];
  CK(cudaMemcpyAsync(rc, ctx->comm_cnt + 2, sizeof rc, cudaMemcpyDeviceToHost, ctx->s_comm));
  CK(cudaStreamSynchronize(ctx->s_comm));
  if (rc[0] < 0 || rc[1] < 0 || rc[0] > cap || rc[1] > cap)
    return fail(ctx, NC_E_OOM, "received count above the receive capacity");
  counts[0] = rc[0];
  counts[1] = rc[1];
  // phase 2: payload (at least one record each way keeps every message non-empty)
  st = ring_exchange(ctx, send_lo, rec * (size_t)std::max<int64_t>(n_lo, 1), send_hi,
                     rec * (size_t)std::max<int64_t>(n_hi, 1), recv_lo, rec * (size_t)std::max<int64_t>(rc[0], 1),
                     recv_hi, rec * (size_t)std::max<int64_t>(rc[1], 1), ctx->s_comm);
  if (st) return st;
  CK(cudaEventRecord(ctx->ev_comm_out, ctx->s_comm));
  ctx->comm_pending = true;
  return NC_OK;
}

nc_status nc_slab_exchange_wait(nc_ctx* ctx) {
  if (!ctx) return fail(ctx, NC_E_ARG, "null ctx");
  if (!ctx->comm_pending) return fail(ctx, NC_E_STATE, "no exchange in flight");
  CK(cudaStreamWaitEvent(ctx->stream, ctx->ev_comm_out, 0));
  ctx->comm_pending = false;
  return NC_OK;
}

nc_status nc_slab_exchange(nc_ctx* ctx, const void* send_lo, int64_t n_lo, const void* send_hi, int64_t n_hi,
                           void* recv_lo, void* recv_hi, int64_t cap, int words, int64_t counts[2]) {
  nc_status st = nc_slab_exchange_start(ctx, send_lo, n_lo, send_hi, n_hi, recv_lo, recv_hi, cap, words, counts);
  if (st) return st;
  return nc_slab_exchange_wait(ctx);
}

// all-gather of every rank's per-layer partials (host in, host out): rank r contributes nloc rows of
// NPART doubles (nloc <= max_rows, padded), out receives nranks x max_rows rows in rank order.
nc_status nc_slab_allgather(nc_ctx* ctx, const double* local, int64_t nloc, int64_t max_rows, double* out) {
  if (!ctx || !out || (nloc > 0 && !local) || nloc < 0 || nloc > max_rows) return fail(ctx, NC_E_ARG, "bad argument");
  if (!ctx->comm) return fail(ctx, NC_E_STATE, "nc_slab_comm_init first");
  const size_t row = NPART * sizeof(double), per = (size_t)max_rows * row;
  if (per * (size_t)ctx->comm_nranks > ctx->comm_gather_bytes) return fail(ctx, NC_E_OOM, "too many rows per rank");
  NcclApi& api = nccl();
  double* dsend = (double*)ctx->comm_gather;
  double* drecv = (double*)((char*)ctx->comm_gather + ctx->comm_gather_bytes);
  CK(cudaMemsetAsync(dsend, 0, per, ctx->stream));
  if (nloc > 0) CK(cudaMemcpyAsync(dsend, local, (size_t)nloc * row, cudaMemcpyHostToDevice, ctx->stream));
  NK(api.AllGather(dsend, drecv, per / sizeof(double), ncclDouble, (ncclComm_t)ctx->comm, ctx->stream));
  CK(cudaMemcpyAsync(out, drecv, per * (size_t)ctx->comm_nranks, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return NC_OK;
}

}  // extern "C"
