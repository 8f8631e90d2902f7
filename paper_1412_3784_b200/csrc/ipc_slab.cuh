// ipc_slab.cuh -- the slab step's peer-memory data plane (included at the end of nemdcell.cu).
//
// The halo and migration messages of the host-synchronization-free slab step (slab_dc.cuh) are
// written by the packing kernels themselves straight into the receive buffers of the neighbour
// ranks: each rank exports its receive buffers (cudaIpcGetMemHandle) and maps its neighbours'
// (cudaIpcOpenMemHandle, peer access over NVLink between GPUs), so `nc_sd_halo` / `nc_sd_migrate`
// given the mapped pointers pack AND transfer in one pass, with no separate send buffer, copy or
// collective.  Ordering across processes uses interprocess events: a rank records "sent" after its
// packing kernels and "consumed" after the kernels that read the previous messages; its neighbours'
// streams wait on them (cudaStreamWaitEvent: no kernel ever spins on another rank).  Because such a
// wait binds to the event's most recent record at the time it is issued, the host driver separates the
// records from the waits with a host barrier (slab.IpcTransport).
#pragma once

// a zeroed device buffer owned by the context, exported for the neighbours (handle: 64 bytes)
nc_status nc_ipc_alloc(nc_ctx* ctx, int64_t bytes, void** dptr, void* handle) {
  if (!ctx || bytes < 1 || !dptr || !handle) return fail(ctx, NC_E_ARG, "bad argument");
  CK(cudaSetDevice(ctx->cfg.device));
  void* p = nullptr;
  CK(cudaMalloc(&p, (size_t)bytes));
  ctx->ipc_own.push_back(p);
  CK(cudaMemset(p, 0, (size_t)bytes));
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, p));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  std::memcpy(handle, &h, 64);
  *dptr = p;
  return NC_OK;
}

// map a neighbour's exported buffer into this context (unmapped by nc_destroy)
nc_status nc_ipc_open(nc_ctx* ctx, const void* handle, void** dptr) {
  if (!ctx || !handle || !dptr) return fail(ctx, NC_E_ARG, "bad argument");
  CK(cudaSetDevice(ctx->cfg.device));
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  void* p = nullptr;
  CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  ctx->ipc_open.push_back(p);
  *dptr = p;
  return NC_OK;
}

// an interprocess event of this context (handle: 64 bytes); returns its id
nc_status nc_ipc_event(nc_ctx* ctx, void* handle, int* id) {
  if (!ctx || !handle || !id) return fail(ctx, NC_E_ARG, "bad argument");
  CK(cudaSetDevice(ctx->cfg.device));
  cudaEvent_t e;
  CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming | cudaEventInterprocess));
  cudaIpcEventHandle_t h;
  CK(cudaIpcGetEventHandle(&h, e));
  static_assert(sizeof(h) == 64, "cudaIpcEventHandle_t is 64 bytes");
  std::memcpy(handle, &h, 64);
  ctx->ipc_ev.push_back(e);
  *id = (int)ctx->ipc_ev.size() - 1;
  return NC_OK;
}

// open a neighbour's interprocess event; returns its id
nc_status nc_ipc_event_open(nc_ctx* ctx, const void* handle, int* id) {
  if (!ctx || !handle || !id) return fail(ctx, NC_E_ARG, "bad argument");
  CK(cudaSetDevice(ctx->cfg.device));
  cudaIpcEventHandle_t h;
  std::memcpy(&h, handle, 64);
  cudaEvent_t e;
  CK(cudaIpcOpenEventHandle(&e, h));
  ctx->ipc_ev.push_back(e);
  *id = (int)ctx->ipc_ev.size() - 1;
  return NC_OK;
}

// record an event after the work queued on the context's stream / make the stream wait for one
nc_status nc_ipc_record(nc_ctx* ctx, int id) {
  if (!ctx || id < 0 || id >= (int)ctx->ipc_ev.size()) return fail(ctx, NC_E_ARG, "bad event id");
  CK(cudaEventRecord(ctx->ipc_ev[(size_t)id], ctx->stream));
  return NC_OK;
}

nc_status nc_ipc_wait(nc_ctx* ctx, int id) {
  if (!ctx || id < 0 || id >= (int)ctx->ipc_ev.size()) return fail(ctx, NC_E_ARG, "bad event id");
  CK(cudaStreamWaitEvent(ctx->stream, ctx->ipc_ev[(size_t)id], 0));
  return NC_OK;
}
