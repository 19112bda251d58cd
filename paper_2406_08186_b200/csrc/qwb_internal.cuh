// qwb_internal.cuh — context, error plumbing and launch helpers shared by the
// libqwb200 translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <utility>
#include <string>

#include "../../include/qwb200.h"
#include "qwb_numerics.cuh"

struct qwb_ctx {
  int device;
  int num_sms;
  bool stopped;
  // stream-ordered scratch (grown on demand).  ws_stream: the stream of the
  // last call that used it; a call on another stream first waits for the
  // work queued there (ws_event), so neither reuse nor cudaFreeAsync on
  // growth can overlap an earlier kernel that still reads or writes it.
  void* ws;
  size_t ws_bytes;
  cudaStream_t ws_stream;
  cudaEvent_t ws_event;
  // device int: a lattice run met tiny amplitudes (lattice_tb.cu)
  int* lat_sticky;
  // pinned host staging for small readbacks
  void* pinned;
  std::string last_error;
  // multi-GPU (comm.cu): NCCL communicator, its stream and ordering events
  void* comm;
  int nranks, rank;
  cudaStream_t comm_stream;
  cudaEvent_t ev_ready, ev_done;
};

namespace qwb {

void set_error(qwb_ctx* ctx, const char* fmt, ...);
int cuda_status(qwb_ctx* ctx, cudaError_t e, const char* what);
inline int cuda_status_if(qwb_ctx* ctx, cudaError_t e, const char* what) {
  return e == cudaSuccess ? 0 : cuda_status(ctx, e, what);
}
// scratch of at least `bytes` (256-B aligned), stream-ordered
int workspace(qwb_ctx* ctx, size_t bytes, cudaStream_t s, void** out);
int begin(qwb_ctx* ctx);   // checks ctx alive and sets the device
// NCCL (comm.cu): grouped send/recv with each peer; float64 all-gather
int nccl_exchange(qwb_ctx* ctx, const void* send, void* const* recv, const int* peers, int npeers,
                  size_t count, cudaStream_t s);
int nccl_allgather_f64(qwb_ctx* ctx, const double* send, double* recv, size_t count, cudaStream_t s);
int nccl_sendrecv_list(qwb_ctx* ctx, const void* const* send, const size_t* send_count, void* const* recv,
                       const size_t* recv_count, const int* peers, int npeers, cudaStream_t s);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Programmatic dependent launch (PDL).  A kernel calls pdl_enter() before its
// first global read: it waits until the previous kernel in the stream has
// completed and its writes are visible, then lets the next kernel be scheduled
// so that kernel's launch latency hides behind this one.  Both instructions
// are no-ops for a launch without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
__device__ __forceinline__ void pdl_enter() {
  pdl_wait();
  pdl_trigger();
}

// integer environment switch (unset or empty: dflt)
inline int env_flag(const char* name, int dflt) {
  const char* e = getenv(name);
  return (e && *e) ? atoi(e) : dflt;
}

// launch `kernel` on `s`, with the PDL attribute when `pdl`
template <class... P, class... A>
cudaError_t launch_pdl(bool pdl, void (*kernel)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       A&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<A>(args)...);
}

inline unsigned blocks_for(int64_t n, int threads, int64_t cap = 1 << 30) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return static_cast<unsigned>(b);
}

}  // namespace qwb

#define QWB_BEGIN(ctx)                   \
  do {                                   \
    int _st = qwb::begin(ctx);           \
    if (_st != QWB_OK) return _st;       \
  } while (0)

#define QWB_CUDA(ctx, call)                                           \
  do {                                                                \
    cudaError_t _e = (call);                                          \
    if (_e != cudaSuccess) return qwb::cuda_status(ctx, _e, #call);   \
  } while (0)

#define QWB_LAUNCH_CHECK(ctx, what)                                   \
  do {                                                                \
    cudaError_t _e = cudaGetLastError();                              \
    if (_e != cudaSuccess) return qwb::cuda_status(ctx, _e, what);    \
  } while (0)

#define QWB_FAIL(ctx, code, ...)            \
  do {                                      \
    qwb::set_error(ctx, __VA_ARGS__);       \
    return (code);                          \
  } while (0)
