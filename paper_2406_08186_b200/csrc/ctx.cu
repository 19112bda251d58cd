// ctx.cu — engine lifecycle (init_engine / stop_engine, backend.py:291-314),
// error strings and the stream-ordered workspace.
#include <stdarg.h>
#include <stdlib.h>

#include "qwb_internal.cuh"

static thread_local std::string g_thread_error;

namespace qwb {

void set_error(qwb_ctx* ctx, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_thread_error = buf;
  if (ctx) ctx->last_error = buf;
}

int cuda_status(qwb_ctx* ctx, cudaError_t e, const char* what) {
  set_error(ctx, "CUDA error %s (%s) in %s", cudaGetErrorName(e), cudaGetErrorString(e), what);
  return e == cudaErrorMemoryAllocation ? QWB_E_OUT_OF_MEMORY : QWB_E_CUDA;
}

int begin(qwb_ctx* ctx) {
  if (!ctx) {
    set_error(nullptr, "null engine context");
    return QWB_E_NOT_ON_DEVICE;
  }
  if (ctx->stopped) {
    set_error(ctx, "engine has been stopped");
    return QWB_E_ENGINE_STOPPED;
  }
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_status(ctx, e, "cudaSetDevice");
  return QWB_OK;
}

int workspace(qwb_ctx* ctx, size_t bytes, cudaStream_t s, void** out) {
  if (ctx->ws && s != ctx->ws_stream) {
    // the previous user's stream may still run kernels on the workspace
    if (!ctx->ws_event) {
      cudaError_t e = cudaEventCreateWithFlags(&ctx->ws_event, cudaEventDisableTiming);
      if (e != cudaSuccess) return cuda_status(ctx, e, "cudaEventCreate(workspace)");
    }
    cudaError_t e = cudaEventRecord(ctx->ws_event, ctx->ws_stream);
    if (e == cudaSuccess) {
      e = cudaStreamWaitEvent(s, ctx->ws_event, 0);
    } else {
      // the previous stream is gone (destroyed by its owner): drain the device
      cudaGetLastError();
      e = cudaDeviceSynchronize();
    }
    if (e != cudaSuccess) return cuda_status(ctx, e, "workspace stream ordering");
  }
  ctx->ws_stream = s;
  bytes = (bytes + 255) & ~size_t(255);
  if (bytes < 256) bytes = 256;
  if (ctx->ws_bytes < bytes) {
    if (ctx->ws) {
      cudaError_t e = cudaFreeAsync(ctx->ws, s);
      if (e != cudaSuccess) return cuda_status(ctx, e, "cudaFreeAsync(workspace)");
      ctx->ws = nullptr;
      ctx->ws_bytes = 0;
    }
    size_t want = bytes + bytes / 4;
    cudaError_t e = cudaMallocAsync(&ctx->ws, want, s);
    if (e != cudaSuccess) return cuda_status(ctx, e, "cudaMallocAsync(workspace)");
    ctx->ws_bytes = want;
  }
  *out = ctx->ws;
  return QWB_OK;
}

}  // namespace qwb

extern "C" {

const char* qwb_version(void) { return "qwb200 0.1.0 (sm_100a)"; }

int qwb_device_count(int* count_host) {
  cudaError_t e = cudaGetDeviceCount(count_host);
  if (e != cudaSuccess) {
    *count_host = 0;
    return qwb::cuda_status(nullptr, e, "cudaGetDeviceCount");
  }
  return QWB_OK;
}

int qwb_init(int device, qwb_ctx** out) {
  if (!out) {
    qwb::set_error(nullptr, "qwb_init: null output pointer");
    return QWB_E_INVALID_ARGUMENT;
  }
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess) return qwb::cuda_status(nullptr, e, "cudaGetDeviceCount");
  if (device < 0 || device >= count) {
    qwb::set_error(nullptr, "device %d not available (%d CUDA devices)", device, count);
    return QWB_E_UNSUPPORTED;
  }
  cudaDeviceProp prop;
  e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) return qwb::cuda_status(nullptr, e, "cudaGetDeviceProperties");
  if (prop.major != 10) {
    qwb::set_error(nullptr, "device %d is sm_%d%d; libqwb200 is built for sm_100a only", device,
                   prop.major, prop.minor);
    return QWB_E_UNSUPPORTED;
  }
  qwb_ctx* c = new qwb_ctx();
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  c->stopped = false;
  c->ws = nullptr;
  c->ws_bytes = 0;
  c->ws_stream = nullptr;
  c->ws_event = nullptr;
  c->lat_sticky = nullptr;
  c->pinned = nullptr;
  c->comm = nullptr;
  c->nranks = 1;
  c->rank = 0;
  c->comm_stream = nullptr;
  c->ev_ready = nullptr;
  c->ev_done = nullptr;
  e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaMallocHost(&c->pinned, 4096);
  if (e != cudaSuccess) {
    delete c;
    return qwb::cuda_status(nullptr, e, "qwb_init");
  }
  *out = c;
  return QWB_OK;
}

int qwb_shutdown(qwb_ctx* ctx) {
  if (!ctx) {
    qwb::set_error(nullptr, "null engine context");
    return QWB_E_NOT_ON_DEVICE;
  }
  if (ctx->stopped) {
    qwb::set_error(ctx, "engine already stopped");
    return QWB_E_ALREADY_STOPPED;
  }
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  if (ctx->comm) qwb_comm_destroy(ctx);
  if (ctx->ws) cudaFree(ctx->ws);
  if (ctx->ws_event) cudaEventDestroy(ctx->ws_event);
  ctx->ws_event = nullptr;
  if (ctx->lat_sticky) cudaFree(ctx->lat_sticky);
  ctx->lat_sticky = nullptr;
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  ctx->ws = nullptr;
  ctx->pinned = nullptr;
  ctx->stopped = true;
  // the struct is intentionally kept (not freed) so that a second shutdown
  // reports AlreadyStopped instead of touching freed memory; it is 100 bytes.
  return QWB_OK;
}

const char* qwb_last_error(const qwb_ctx* ctx) {
  if (ctx && !ctx->last_error.empty()) return ctx->last_error.c_str();
  return g_thread_error.c_str();
}

}  // extern "C"
