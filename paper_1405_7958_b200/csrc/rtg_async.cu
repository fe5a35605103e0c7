// rtg_process_tile_async / rtg_ticket_wait / rtg_ticket_query (include/rtg.h):
// the stage body on host buffers as a 3-phase pipeline.
//
// The reference models this pipeline only in virtual time: the GPU slot's
// next upload may start once the upload channel frees, overlapping the
// previous task's compute and download (wrm.cpp:385-415 prefetch_pipeline,
// sim.cpp:672-684).  Here each context owns kAsyncSlots slots of device
// buffers and three streams:
//   up_stream:   H2D RGB -> slot.rgb                     record slot.up
//   ctx->stream: wait slot.up, the stage (cached graph)  record slot.comp
//   down_stream: wait slot.comp, D2H mask / labels / hema / count / rows
//                                                        record slot.down
// so tile t+1 uploads while tile t computes and tile t-1 downloads.  A slot is
// reused only after its download event completed (host wait); a ticket
// retired that way keeps its result until the caller waits for it.
#include <cstring>
#include <string>

#include "common.cuh"

namespace rtg {
namespace {

int ensure_slots(rtg_ctx* ctx) {
  if (ctx->slots) return RTG_OK;
  AsyncSlot* s = new AsyncSlot[kAsyncSlots];
  ctx->slots = s;  // rtg_ctx_destroy releases whatever was allocated
  const size_t n = (size_t)ctx->max_px;
  for (int k = 0; k < kAsyncSlots; ++k) {
    RTG_CUDA(cudaMalloc((void**)&s[k].rgb, 3 * n));
    RTG_CUDA(cudaMalloc((void**)&s[k].mask, n));
    RTG_CUDA(cudaMalloc((void**)&s[k].labels, 4 * n));
    RTG_CUDA(cudaMalloc((void**)&s[k].hema, n));
    RTG_CUDA(cudaMalloc((void**)&s[k].feats,
                        sizeof(float) * RTG_MAX_FEATURE_COLUMNS * (size_t)ctx->max_objects));
    RTG_CUDA(cudaMalloc((void**)&s[k].d_n, sizeof(int32_t)));
    RTG_CUDA(cudaHostAlloc((void**)&s[k].h_n, sizeof(int32_t), cudaHostAllocPortable));
    RTG_CUDA(cudaEventCreateWithFlags(&s[k].up, cudaEventDisableTiming));
    RTG_CUDA(cudaEventCreateWithFlags(&s[k].comp, cudaEventDisableTiming));
    RTG_CUDA(cudaEventCreateWithFlags(&s[k].down, cudaEventDisableTiming));
  }
  RTG_CUDA(cudaStreamCreateWithFlags(&ctx->up_stream, cudaStreamNonBlocking));
  RTG_CUDA(cudaStreamCreateWithFlags(&ctx->down_stream, cudaStreamNonBlocking));
  return RTG_OK;
}

// Waits for the slot's download and records its ticket's result.
int retire(rtg_ctx* ctx, AsyncSlot& s) {
  RTG_CUDA(cudaEventSynchronize(s.down));
  ctx->retired.push_back({s.ticket, *s.h_n, s.max_rows});
  s.ticket = 0;
  return RTG_OK;
}

int result(rtg_ctx* ctx, int32_t n, int32_t max_rows, int32_t* n_objects) {
  if (n_objects) *n_objects = n;
  if (n > ctx->max_objects)
    return fail(RTG_ERR_OVERFLOW, "tile has " + std::to_string(n) +
                                      " objects, more than the context's max_objects " +
                                      std::to_string(ctx->max_objects));
  if (max_rows >= 0 && n > max_rows)
    return fail(RTG_ERR_OVERFLOW, "tile has " + std::to_string(n) + " objects; feature rows: " +
                                      std::to_string(max_rows));
  return RTG_OK;
}

}  // namespace

void release_slots(rtg_ctx* c) {
  if (!c->slots) return;
  if (c->up_stream) cudaStreamSynchronize(c->up_stream);
  if (c->down_stream) cudaStreamSynchronize(c->down_stream);
  for (int k = 0; k < kAsyncSlots; ++k) {
    AsyncSlot& s = c->slots[k];
    void* dev[] = {s.rgb, s.mask, s.labels, s.hema, s.feats, s.d_n};
    for (void* p : dev)
      if (p) cudaFree(p);
    if (s.h_n) cudaFreeHost(s.h_n);
    for (cudaEvent_t e : {s.up, s.comp, s.down})
      if (e) cudaEventDestroy(e);
  }
  delete[] c->slots;
  c->slots = nullptr;
  if (c->up_stream) cudaStreamDestroy(c->up_stream);
  if (c->down_stream) cudaStreamDestroy(c->down_stream);
  c->up_stream = c->down_stream = nullptr;
}

}  // namespace rtg

using namespace rtg;

extern "C" {

int rtg_process_tile_async(rtg_ctx* ctx, const uint8_t* rgb, int64_t h, int64_t w,
                           int64_t pitch_bytes, const rtg_params* params, uint8_t* mask_out,
                           int32_t* labels_out, uint8_t* hema_out, float* features_out,
                           int32_t max_rows, uint64_t* ticket) {
  RTG_TRY(check_ctx(ctx, h, w));
  RTG_TRY(check_params(params));
  if (!rgb || !ticket) return fail(RTG_ERR_INVALID_ARG, "null rgb or ticket");
  if (pitch_bytes < 3 * w) return fail(RTG_ERR_DIMENSION, "pitch_bytes < 3 * w");
  if (features_out && max_rows < 0) return fail(RTG_ERR_INVALID_ARG, "max_rows < 0");
  RTG_TRY(ensure_slots(ctx));
  // a free slot, else the oldest in flight (its result is kept for the caller)
  int pick = -1;
  for (int k = 0; k < kAsyncSlots; ++k) {
    const AsyncSlot& s = ctx->slots[k];
    if (s.ticket == 0) {
      pick = k;
      break;
    }
    if (pick < 0 || s.ticket < ctx->slots[pick].ticket) pick = k;
  }
  AsyncSlot& s = ctx->slots[pick];
  if (s.ticket != 0) RTG_TRY(retire(ctx, s));

  // phase 1: upload
  if (pitch_bytes == 3 * w)
    RTG_CUDA(cudaMemcpyAsync(s.rgb, rgb, (size_t)(3 * h * w), cudaMemcpyHostToDevice,
                             ctx->up_stream));
  else
    RTG_CUDA(cudaMemcpy2DAsync(s.rgb, (size_t)(3 * w), rgb, (size_t)pitch_bytes, (size_t)(3 * w),
                               (size_t)h, cudaMemcpyHostToDevice, ctx->up_stream));
  RTG_CUDA(cudaEventRecord(s.up, ctx->up_stream));
  // phase 2: the stage
  RTG_CUDA(cudaStreamWaitEvent(ctx->stream, s.up, 0));
  RTG_TRY(run_stage(ctx, s.rgb, h, w, 3 * w, params, s.mask, s.labels, s.hema, s.feats, s.d_n));
  RTG_CUDA(cudaEventRecord(s.comp, ctx->stream));
  // phase 3: download
  RTG_CUDA(cudaStreamWaitEvent(ctx->down_stream, s.comp, 0));
  const size_t px = (size_t)(h * w);
  RTG_CUDA(cudaMemcpyAsync(s.h_n, s.d_n, sizeof(int32_t), cudaMemcpyDeviceToHost,
                           ctx->down_stream));
  if (mask_out)
    RTG_CUDA(cudaMemcpyAsync(mask_out, s.mask, px, cudaMemcpyDeviceToHost, ctx->down_stream));
  if (labels_out)
    RTG_CUDA(cudaMemcpyAsync(labels_out, s.labels, 4 * px, cudaMemcpyDeviceToHost,
                             ctx->down_stream));
  if (hema_out)
    RTG_CUDA(cudaMemcpyAsync(hema_out, s.hema, px, cudaMemcpyDeviceToHost, ctx->down_stream));
  const int32_t rows = max_rows < ctx->max_objects ? max_rows : ctx->max_objects;
  if (features_out && rows > 0)
    RTG_TRY(rows_to_host(ctx, ctx->down_stream, s.feats, s.d_n, features_out, rows,
                         feature_cols(params)));
  RTG_CUDA(cudaEventRecord(s.down, ctx->down_stream));
  s.max_rows = features_out ? max_rows : -1;
  s.ticket = ctx->next_ticket++;
  *ticket = s.ticket;
  return RTG_OK;
}

int rtg_ticket_wait(rtg_ctx* ctx, uint64_t ticket, int32_t* n_objects) {
  if (!ctx) return fail(RTG_ERR_INVALID_ARG, "null rtg_ctx");
  RTG_CUDA(cudaSetDevice(ctx->device));
  for (size_t i = 0; i < ctx->retired.size(); ++i) {
    if (ctx->retired[i].ticket != ticket) continue;
    const rtg_ctx::Retired r = ctx->retired[i];
    ctx->retired.erase(ctx->retired.begin() + (std::ptrdiff_t)i);
    return result(ctx, r.n, r.max_rows, n_objects);
  }
  for (int k = 0; ctx->slots && k < kAsyncSlots; ++k) {
    AsyncSlot& s = ctx->slots[k];
    if (s.ticket != ticket || ticket == 0) continue;
    RTG_CUDA(cudaEventSynchronize(s.down));
    s.ticket = 0;
    return result(ctx, *s.h_n, s.max_rows, n_objects);
  }
  return fail(RTG_ERR_NOT_FOUND, "unknown or already-waited ticket " + std::to_string(ticket));
}

int rtg_ticket_query(rtg_ctx* ctx, uint64_t ticket, int* done) {
  if (!ctx || !done) return fail(RTG_ERR_INVALID_ARG, "null argument");
  RTG_CUDA(cudaSetDevice(ctx->device));
  for (const auto& r : ctx->retired)
    if (r.ticket == ticket) {
      *done = 1;
      return RTG_OK;
    }
  for (int k = 0; ctx->slots && k < kAsyncSlots; ++k) {
    const AsyncSlot& s = ctx->slots[k];
    if (s.ticket != ticket || ticket == 0) continue;
    const cudaError_t e = cudaEventQuery(s.down);
    if (e == cudaErrorNotReady) {
      *done = 0;
      return RTG_OK;
    }
    RTG_CUDA(e);
    *done = 1;
    return RTG_OK;
  }
  return fail(RTG_ERR_NOT_FOUND, "unknown or already-waited ticket " + std::to_string(ticket));
}

}  // extern "C"
