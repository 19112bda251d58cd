// comm.cu — multi-GPU slab stepping with an NCCL halo exchange.
//
// The reference has no distribution beyond an in-process row-block thread
// pool (backend.py:426-430); PAPER.md:499-501 lists multi-GPU as future work.
// Here a periodic nx x ny lattice is split into contiguous y-slabs, one per
// rank/GPU (lattice.cu "Slabs").  Per coined step:
//
//   compute stream:  [wait recv(t-1)] boundary rows (first, last) -> record ready
//   comm stream:     [wait ready] ncclGroupStart; send/recv 2 rows of nx
//                     complex128 to/from each y-neighbour; ncclGroupEnd -> record done
//   compute stream:  interior rows (overlaps the exchange)
//
// The exchanged rows are the step's outputs that belong to the neighbour
// (plane U of its last row, plane D of its first row); NCCL receives straight
// into this rank's planes and sends straight from its two extra rows, so there
// is no packing.  Volume: 2 x 16 x nx bytes per direction per step.
//
// NCCL is dlopen'ed (libnccl.so.2, or $QWB_NCCL_LIB) so the library has no
// link-time NCCL dependency and shares the NCCL that torch.distributed loaded.
#include <dlfcn.h>
#include <stdlib.h>
#include <string.h>

#include "qwb_lattice.cuh"

namespace {

typedef struct {
  char internal[128];
} NcclUid;
typedef void* NcclComm;
typedef int (*fn_get_uid)(NcclUid*);
typedef int (*fn_init_rank)(NcclComm*, int, NcclUid, int);
typedef int (*fn_destroy)(NcclComm);
typedef int (*fn_sendrecv)(void*, size_t, int, int, NcclComm, cudaStream_t);
typedef int (*fn_group)(void);
typedef const char* (*fn_errstr)(int);
typedef int (*fn_allgather)(const void*, void*, size_t, int, NcclComm, cudaStream_t);

constexpr int kNcclFloat64 = 8;

struct Nccl {
  void* h = nullptr;
  fn_get_uid get_uid = nullptr;
  fn_init_rank init_rank = nullptr;
  fn_destroy destroy = nullptr;
  fn_sendrecv send = nullptr;
  fn_sendrecv recv = nullptr;
  fn_group group_start = nullptr;
  fn_group group_end = nullptr;
  fn_errstr errstr = nullptr;
  fn_allgather allgather = nullptr;
};

Nccl g_nccl;

int load_nccl(qwb_ctx* ctx) {
  if (g_nccl.h) return QWB_OK;
  const char* path = getenv("QWB_NCCL_LIB");
  void* h = dlopen(path && *path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) QWB_FAIL(ctx, QWB_E_NCCL, "cannot load NCCL (%s): %s", path ? path : "libnccl.so.2", dlerror());
  Nccl n;
  n.h = h;
  n.get_uid = (fn_get_uid)dlsym(h, "ncclGetUniqueId");
  n.init_rank = (fn_init_rank)dlsym(h, "ncclCommInitRank");
  n.destroy = (fn_destroy)dlsym(h, "ncclCommDestroy");
  // ncclSend's buffer is const; the ABI is identical for our purposes
  n.send = (fn_sendrecv)dlsym(h, "ncclSend");
  n.recv = (fn_sendrecv)dlsym(h, "ncclRecv");
  n.group_start = (fn_group)dlsym(h, "ncclGroupStart");
  n.group_end = (fn_group)dlsym(h, "ncclGroupEnd");
  n.errstr = (fn_errstr)dlsym(h, "ncclGetErrorString");
  n.allgather = (fn_allgather)dlsym(h, "ncclAllGather");
  if (!n.get_uid || !n.init_rank || !n.destroy || !n.send || !n.recv || !n.group_start ||
      !n.group_end || !n.errstr || !n.allgather)
    QWB_FAIL(ctx, QWB_E_NCCL, "NCCL library lacks a required symbol");
  g_nccl = n;
  return QWB_OK;
}

#define QWB_NCCL(ctx, call)                                                             \
  do {                                                                                  \
    int _r = (call);                                                                    \
    if (_r != 0) QWB_FAIL(ctx, QWB_E_NCCL, "NCCL error %d (%s) in %s", _r,              \
                          g_nccl.errstr ? g_nccl.errstr(_r) : "?", #call);              \
  } while (0)

}  // namespace

namespace qwb {

// One grouped exchange: send `send` (count float64s) to every peer and receive
// each peer's buffer into recv[i], on stream s.
int nccl_exchange(qwb_ctx* ctx, const void* send, void* const* recv, const int* peers, int npeers,
                  size_t count, cudaStream_t s) {
  if (!ctx->comm) QWB_FAIL(ctx, QWB_E_NCCL, "qwb_comm_init has not been called");
  NcclComm comm = (NcclComm)ctx->comm;
  QWB_NCCL(ctx, g_nccl.group_start());
  for (int i = 0; i < npeers; ++i) {
    QWB_NCCL(ctx, g_nccl.send(const_cast<void*>(send), count, kNcclFloat64, peers[i], comm, s));
    QWB_NCCL(ctx, g_nccl.recv(recv[i], count, kNcclFloat64, peers[i], comm, s));
  }
  QWB_NCCL(ctx, g_nccl.group_end());
  return QWB_OK;
}

// One grouped exchange with per-peer buffers and counts (float64s).
int nccl_sendrecv_list(qwb_ctx* ctx, const void* const* send, const size_t* send_count, void* const* recv,
                       const size_t* recv_count, const int* peers, int npeers, cudaStream_t s) {
  if (!ctx->comm) QWB_FAIL(ctx, QWB_E_NCCL, "qwb_comm_init has not been called");
  NcclComm comm = (NcclComm)ctx->comm;
  QWB_NCCL(ctx, g_nccl.group_start());
  for (int i = 0; i < npeers; ++i) {
    if (send_count[i])
      QWB_NCCL(ctx, g_nccl.send(const_cast<void*>(send[i]), send_count[i], kNcclFloat64, peers[i], comm, s));
    if (recv_count[i]) QWB_NCCL(ctx, g_nccl.recv(recv[i], recv_count[i], kNcclFloat64, peers[i], comm, s));
  }
  QWB_NCCL(ctx, g_nccl.group_end());
  return QWB_OK;
}

// recv[r * count ...] = rank r's send (count float64s), on stream s
int nccl_allgather_f64(qwb_ctx* ctx, const double* send, double* recv, size_t count, cudaStream_t s) {
  if (!ctx->comm) QWB_FAIL(ctx, QWB_E_NCCL, "qwb_comm_init has not been called");
  QWB_NCCL(ctx, g_nccl.allgather(send, recv, count, kNcclFloat64, (NcclComm)ctx->comm, s));
  return QWB_OK;
}

}  // namespace qwb

extern "C" {

int qwb_comm_unique_id(void* id_out_host) {
  int st = load_nccl(nullptr);
  if (st) return st;
  NcclUid uid;
  int r = g_nccl.get_uid(&uid);
  if (r != 0) {
    qwb::set_error(nullptr, "ncclGetUniqueId failed: %d", r);
    return QWB_E_NCCL;
  }
  memcpy(id_out_host, &uid, sizeof(uid));
  return QWB_OK;
}

int qwb_comm_init(qwb_ctx* ctx, const void* id_host, int nranks, int rank) {
  QWB_BEGIN(ctx);
  if (ctx->comm) QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "communicator already initialised");
  if (nranks < 1 || rank < 0 || rank >= nranks)
    QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "bad rank %d of %d", rank, nranks);
  int st = load_nccl(ctx);
  if (st) return st;
  NcclUid uid;
  memcpy(&uid, id_host, sizeof(uid));
  NcclComm comm = nullptr;
  QWB_NCCL(ctx, g_nccl.init_rank(&comm, nranks, uid, rank));
  ctx->comm = comm;
  ctx->nranks = nranks;
  ctx->rank = rank;
  QWB_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking));
  QWB_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_ready, cudaEventDisableTiming));
  QWB_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_done, cudaEventDisableTiming));
  return QWB_OK;
}

int qwb_comm_destroy(qwb_ctx* ctx) {
  if (!ctx || !ctx->comm) return QWB_OK;
  cudaSetDevice(ctx->device);
  if (ctx->comm_stream) cudaStreamSynchronize(ctx->comm_stream);
  g_nccl.destroy((NcclComm)ctx->comm);
  ctx->comm = nullptr;
  if (ctx->comm_stream) cudaStreamDestroy(ctx->comm_stream);
  if (ctx->ev_ready) cudaEventDestroy(ctx->ev_ready);
  if (ctx->ev_done) cudaEventDestroy(ctx->ev_done);
  ctx->comm_stream = nullptr;
  ctx->ev_ready = ctx->ev_done = nullptr;
  ctx->nranks = 1;
  ctx->rank = 0;
  return QWB_OK;
}

// Run `steps` coined steps on this rank's slab, exchanging the two boundary
// rows with rank_below / rank_above each step.  Result in a (even steps) or
// b (odd), reported through *final_in_b_host.
int qwb_slab_run(qwb_ctx* ctx, int64_t nx, int64_t ny, int64_t y0, int64_t ny_local, int shift,
                 const uint32_t* marked_bits, qwb_z* a, qwb_z* b, int64_t steps, int rank_below,
                 int rank_above, int* final_in_b_host, void* stream) {
  QWB_BEGIN(ctx);
  qwb::Geom g;
  int st = qwb::lattice_slab_geom(ctx, nx, ny, y0, ny_local, &g);
  if (!st) st = qwb::lattice_check_shift(ctx, shift);
  if (st) return st;
  if (!ctx->comm) QWB_FAIL(ctx, QWB_E_NCCL, "qwb_comm_init has not been called");
  if (rank_below < 0 || rank_below >= ctx->nranks || rank_above < 0 || rank_above >= ctx->nranks)
    QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "neighbour ranks out of range");
  if (steps < 0) QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "steps must be >= 0");
  cudaStream_t s = qwb::as_stream(stream);
  cudaStream_t cs = ctx->comm_stream;
  NcclComm comm = (NcclComm)ctx->comm;
  const int64_t P = g.pstride;
  const size_t cnt = 2 * (size_t)nx;   // one row of complex128 as float64s
  // plane pushed across the lower / upper slab edge: flip-flop writes the
  // reverse arc (plane U below, plane D above), persistent keeps the direction
  const int64_t pd = shift == QWB_SHIFT_FLIPFLOP ? 3 : 0, pu = 3 - pd;
  const qwb::Rows edge = qwb::slab_rows(ny_local, 1);
  const qwb::Rows inner = qwb::slab_rows(ny_local, 2);
  qwb::TraceArgs tr{};
  double2* cur = reinterpret_cast<double2*>(a);
  double2* nxt = reinterpret_cast<double2*>(b);
  // the comm stream starts after everything already queued on s
  QWB_CUDA(ctx, cudaEventRecord(ctx->ev_done, s));
  for (int64_t k = 0; k < steps; ++k) {
    QWB_CUDA(ctx, cudaStreamWaitEvent(s, ctx->ev_done, 0));
    qwb::lattice_launch(shift, s, g, edge, cur, nxt, marked_bits, nullptr, 0, tr);
    QWB_CUDA(ctx, cudaEventRecord(ctx->ev_ready, s));
    QWB_CUDA(ctx, cudaStreamWaitEvent(cs, ctx->ev_ready, 0));
    double2* send_down = nxt + pd * P;                                 // extra row 0
    double2* recv_from_up = nxt + pd * P + (int64_t)ny_local * nx;     // last owned row
    double2* send_up = nxt + pu * P + (int64_t)(ny_local + 1) * nx;    // extra row ny_local+1
    double2* recv_from_down = nxt + pu * P + (int64_t)nx;              // first owned row
    QWB_NCCL(ctx, g_nccl.group_start());
    QWB_NCCL(ctx, g_nccl.send(send_down, cnt, kNcclFloat64, rank_below, comm, cs));
    QWB_NCCL(ctx, g_nccl.recv(recv_from_up, cnt, kNcclFloat64, rank_above, comm, cs));
    QWB_NCCL(ctx, g_nccl.send(send_up, cnt, kNcclFloat64, rank_above, comm, cs));
    QWB_NCCL(ctx, g_nccl.recv(recv_from_down, cnt, kNcclFloat64, rank_below, comm, cs));
    QWB_NCCL(ctx, g_nccl.group_end());
    QWB_CUDA(ctx, cudaEventRecord(ctx->ev_done, cs));
    qwb::lattice_launch(shift, s, g, inner, cur, nxt, marked_bits, nullptr, 0, tr);
    double2* t = cur;
    cur = nxt;
    nxt = t;
  }
  QWB_CUDA(ctx, cudaStreamWaitEvent(s, ctx->ev_done, 0));
  QWB_LAUNCH_CHECK(ctx, "lattice_step_kernel(slab run)");
  if (final_in_b_host) *final_in_b_host = (steps % 2) ? 1 : 0;
  return QWB_OK;
}

static __global__ void gather_z_kernel(int64_t n, const int64_t* __restrict__ idx, const double2* __restrict__ x,
                                double2* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = x[idx[i]];
}

// Halo exchange of a row-partitioned CSR operator (distributed.csr_partition).
// x_ext = [own entries (n_local) | halo]; for peer i: send x_ext[send_idx[
// send_off[i] .. send_off[i+1])] and receive recv_off[i+1] - recv_off[i]
// entries into x_ext[n_local + recv_off[i] ..].  send_buf: send_off[npeers]
// qwb_z of scratch.
int qwb_csr_halo_exchange(qwb_ctx* ctx, int64_t n_local, qwb_z* x_ext, const int64_t* send_idx,
                          const int64_t* send_off_host, const int64_t* recv_off_host, const int* peers_host,
                          int npeers, qwb_z* send_buf, void* stream) {
  QWB_BEGIN(ctx);
  if (npeers < 0 || npeers > 1024) QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "bad peer count %d", npeers);
  if (npeers == 0) return QWB_OK;
  cudaStream_t s = qwb::as_stream(stream);
  double2* xe = reinterpret_cast<double2*>(x_ext);
  double2* sb = reinterpret_cast<double2*>(send_buf);
  const int64_t nsend = send_off_host[npeers];
  if (nsend > 0) {
    gather_z_kernel<<<qwb::blocks_for(nsend, 256, (int64_t)ctx->num_sms * 8), 256, 0, s>>>(nsend, send_idx, xe, sb);
    QWB_LAUNCH_CHECK(ctx, "gather_z_kernel");
  }
  const void* sp[1024];
  void* rp[1024];
  size_t sc[1024], rc[1024];
  for (int i = 0; i < npeers; ++i) {
    sp[i] = sb + send_off_host[i];
    sc[i] = 2 * (size_t)(send_off_host[i + 1] - send_off_host[i]);
    rp[i] = xe + n_local + recv_off_host[i];
    rc[i] = 2 * (size_t)(recv_off_host[i + 1] - recv_off_host[i]);
  }
  return qwb::nccl_sendrecv_list(ctx, sp, sc, rp, rc, peers_host, npeers, s);
}

// Ghost-row exchange of slab state (the fused multi-GPU lattice path): every
// plane's first g owned rows go to the rank below's top ghost rows, the last
// g owned rows to the rank above's bottom ghost rows (g = ghost before a
// temporally blocked launch, 1 before a single pull step).
static int ghost_exchange_nccl(qwb_ctx* ctx, int64_t nx, int64_t nl, int64_t G, int g, double2* planes,
                               int below, int above, cudaStream_t s) {
  NcclComm comm = (NcclComm)ctx->comm;
  const int64_t P = nx * (nl + 2 * G);
  const size_t cnt = 2 * (size_t)(g * nx);
  QWB_NCCL(ctx, g_nccl.group_start());
  for (int p = 0; p < 4; ++p) {
    double2* pl = planes + p * P;
    QWB_NCCL(ctx, g_nccl.send(pl + G * nx, cnt, kNcclFloat64, below, comm, s));
    QWB_NCCL(ctx, g_nccl.recv(pl + (G + nl) * nx, cnt, kNcclFloat64, above, comm, s));
    QWB_NCCL(ctx, g_nccl.send(pl + (G + nl - g) * nx, cnt, kNcclFloat64, above, comm, s));
    QWB_NCCL(ctx, g_nccl.recv(pl + (G - g) * nx, cnt, kNcclFloat64, below, comm, s));
  }
  QWB_NCCL(ctx, g_nccl.group_end());
  return QWB_OK;
}

// `steps` coined steps on a ghost-row slab: temporally blocked launches of
// `ghost` steps each (ghost-row exchange before each), the remainder as
// single pull steps (one-row exchange before each).  Result in a or b.
//
// The exchange overlaps the first launch after it: that launch is split by
// tile rows into a middle band, whose regions read owned rows only, and two
// edge bands.  The NCCL group runs on the comm stream while the middle band
// runs on the caller's stream on all SMs but kSlabFreeSMs (so NCCL's kernels
// find SMs: nothing waits on anything inside a kernel, so even without free
// SMs the two only serialise); the edge bands follow after an event wait.
// QWB_SLAB_OVERLAP=0: exchange in stream order before the launch instead.
constexpr int kSlabFreeSMs = 8;

int qwb_slab_run_fused(qwb_ctx* ctx, int64_t nx, int64_t ny, int64_t y0, int64_t ny_local, int64_t ghost,
                       int shift, const uint32_t* marked_bits, const int64_t* marked_host, int64_t n_marked,
                       qwb_z* a, qwb_z* b, int64_t steps, int rank_below, int rank_above, int* final_in_b_host,
                       void* stream) {
  QWB_BEGIN(ctx);
  if (!ctx->comm) QWB_FAIL(ctx, QWB_E_NCCL, "qwb_comm_init has not been called");
  if (rank_below < 0 || rank_below >= ctx->nranks || rank_above < 0 || rank_above >= ctx->nranks)
    QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "neighbour ranks out of range");
  if (steps < 0) QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "steps must be >= 0");
  cudaStream_t s = qwb::as_stream(stream);
  cudaStream_t cs = ctx->comm_stream;
  double2* cur = reinterpret_cast<double2*>(a);
  double2* nxt = reinterpret_cast<double2*>(b);
  // G = mT: per exchange of g = jT rows (j = m, fewer at the end), j launches
  // over the owned rows extended by (j-1)T, ..., T, 0 rows each side; the last
  // < T steps as single pull steps (1-row exchange)
  const int T = qwb::kSlabDepth;
  if (qwb::lattice_slab_depth(T) != T || ghost < T || ghost % T)
    QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "ghost rows must be a multiple of the slab depth");
  if (n_marked > 0 && (!marked_bits || !marked_host))
    QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "marked vertices need both the bitmap and the host list");
  static const int overlap = qwb::env_flag("QWB_SLAB_OVERLAP", 1);
  int swaps = 0;
  auto swap = [&]() {
    double2* t = cur;
    cur = nxt;
    nxt = t;
    ++swaps;
  };
  // subnormal guard: the first launch after each exchange tests its tiles
  // (its regions hold every value that reaches an owned row before the next
  // exchange); a hit switches the rest of the run to numpy's arithmetic
  int* sticky = nullptr;
  {
    const int st = qwb::lattice_sticky(ctx, &sticky);
    if (st) return st;
    QWB_CUDA(ctx, cudaMemsetAsync(sticky, 0, sizeof(int), s));
  }
  auto geo_of = [&](int ext) {
    return qwb::TbGeo{(int)(ny_local + 2 * ghost), (int)ghost - ext, (int)ny_local + 2 * ext, (int)(y0 - ext), 0};
  };
  auto launch = [&](int nsteps, int ext, int check) -> int {
    int st;
    if (nsteps == 1) {
      st = qwb_slab_advance_local(ctx, nx, ny, y0, ny_local, ghost, shift, marked_bits, marked_host, n_marked,
                                  reinterpret_cast<qwb_z*>(cur), reinterpret_cast<qwb_z*>(nxt), 1, 0, stream);
    } else {
      st = qwb::lattice_tb_launch_geo(ctx, T, shift, s, (int)nx, (int)ny, geo_of(ext), cur, nxt, marked_bits,
                                      marked_host, n_marked, 0, 0, 0, check, sticky);
    }
    swap();
    return st;
  };
  // the T-step launch over owned rows + ext, as middle band (during the
  // exchange) and edge bands (after it); false: no middle band here
  auto overlapped = [&](int g, int ext, int* st) -> bool {
    const qwb::TbGeo geo = geo_of(ext);
    int tx, ty;
    const int oy = qwb::lattice_tb_tiles(T, (int)nx, geo.nown, &tx, &ty);
    // tile row r: local rows own0 + r oy + [-T, oy + T) must lie in the owned rows
    const int r_lo = (ext + T + oy - 1) / oy;
    const int r_hi_num = (int)ny_local + ext - T - oy;
    const int r_hi = r_hi_num >= 0 ? r_hi_num / oy : -1;
    if (!overlap || r_lo > r_hi || r_hi >= ty) return false;
    *st = QWB_OK;
    auto part = [&](int t0, int t1, int cap) -> int {
      if (t1 <= t0) return QWB_OK;
      return qwb::lattice_tb_launch_geo(ctx, T, shift, s, (int)nx, (int)ny, geo, cur, nxt, marked_bits, marked_host,
                                        n_marked, t0, t1, cap, 1, sticky);
    };
    cudaError_t e = cudaEventRecord(ctx->ev_ready, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, ctx->ev_ready, 0);
    if (e != cudaSuccess) {
      *st = qwb::cuda_status(ctx, e, "slab exchange ordering");
      return true;
    }
    *st = ghost_exchange_nccl(ctx, nx, ny_local, ghost, g, cur, rank_below, rank_above, cs);
    if (!*st) *st = qwb::cuda_status_if(ctx, cudaEventRecord(ctx->ev_done, cs), "cudaEventRecord");
    if (!*st) *st = part(r_lo * tx, (r_hi + 1) * tx, ctx->num_sms - kSlabFreeSMs);
    if (!*st) *st = qwb::cuda_status_if(ctx, cudaStreamWaitEvent(s, ctx->ev_done, 0), "cudaStreamWaitEvent");
    if (!*st) *st = part(0, r_lo * tx, 0);
    if (!*st) *st = part((r_hi + 1) * tx, tx * ty, 0);
    swap();
    return true;
  };
  for (int64_t k = 0; k < steps;) {
    int64_t g = (steps - k) / T * T;
    if (g > ghost) g = ghost;
    if (g == 0) g = 1;
    int st = QWB_OK;
    if (g == 1) {
      st = ghost_exchange_nccl(ctx, nx, ny_local, ghost, 1, cur, rank_below, rank_above, s);
      if (!st) st = launch(1, 0, 0);
    } else {
      int ext = (int)g - T;
      if (!overlapped((int)g, ext, &st)) {
        st = ghost_exchange_nccl(ctx, nx, ny_local, ghost, (int)g, cur, rank_below, rank_above, s);
        if (!st) st = launch(T, ext, 1);
      }
      for (ext -= T; ext >= 0 && !st; ext -= T) st = launch(T, ext, 0);
    }
    if (st) return st;
    k += g;
  }
  QWB_LAUNCH_CHECK(ctx, "slab launches");
  if (final_in_b_host) *final_in_b_host = swaps & 1;
  return QWB_OK;
}

// the same exchange for nslabs ghost-row slabs on ONE device (tests)
int qwb_slab_ghost_exchange_local(qwb_ctx* ctx, int64_t nx, int64_t ghost, int g, const int64_t* ny_local_host,
                                  qwb_z* const* planes_host, int nslabs, void* stream) {
  QWB_BEGIN(ctx);
  if (g < 1 || g > ghost) QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "exchange rows must be in 1..ghost");
  cudaStream_t s = qwb::as_stream(stream);
  const size_t bytes = 16 * (size_t)(g * nx);
  for (int i = 0; i < nslabs; ++i) {
    const int below = (i + nslabs - 1) % nslabs, above = (i + 1) % nslabs;
    const int64_t nl = ny_local_host[i], P = nx * (nl + 2 * ghost);
    const int64_t nlb = ny_local_host[below], Pb = nx * (nlb + 2 * ghost);
    const int64_t nla = ny_local_host[above], Pa = nx * (nla + 2 * ghost);
    double2* me = reinterpret_cast<double2*>(planes_host[i]);
    double2* bl = reinterpret_cast<double2*>(planes_host[below]);
    double2* ab = reinterpret_cast<double2*>(planes_host[above]);
    for (int p = 0; p < 4; ++p) {
      // my first g owned rows -> below's top ghost rows
      QWB_CUDA(ctx, cudaMemcpyAsync(bl + p * Pb + (ghost + nlb) * nx, me + p * P + ghost * nx, bytes,
                                    cudaMemcpyDeviceToDevice, s));
      // my last g owned rows -> above's bottom ghost rows
      QWB_CUDA(ctx, cudaMemcpyAsync(ab + p * Pa + (ghost - g) * nx, me + p * P + (ghost + nl - g) * nx, bytes,
                                    cudaMemcpyDeviceToDevice, s));
    }
  }
  return QWB_OK;
}

// Single-process emulation of the exchange for P slabs held on ONE device
// (tests): after qwb_slab_step(part=0) on every slab, move the two boundary
// rows of slab i into its neighbours exactly as qwb_slab_run's NCCL group
// does.  planes[i] are device pointers to the slabs' output buffers.
int qwb_slab_exchange_local(qwb_ctx* ctx, int64_t nx, int shift, const int64_t* ny_local_host,
                            qwb_z* const* planes_host, int nslabs, void* stream) {
  QWB_BEGIN(ctx);
  int st = qwb::lattice_check_shift(ctx, shift);
  if (st) return st;
  cudaStream_t s = qwb::as_stream(stream);
  const size_t bytes = 16 * (size_t)nx;
  const int64_t pd = shift == QWB_SHIFT_FLIPFLOP ? 3 : 0, pu = 3 - pd;
  for (int i = 0; i < nslabs; ++i) {
    const int below = (i + nslabs - 1) % nslabs, above = (i + 1) % nslabs;
    const int64_t nl = ny_local_host[i];
    const int64_t P = nx * (nl + 2);
    double2* me = reinterpret_cast<double2*>(planes_host[i]);
    // my extra row 0 -> below's last owned row (plane pd)
    const int64_t nlb = ny_local_host[below], Pb = nx * (nlb + 2);
    double2* bl = reinterpret_cast<double2*>(planes_host[below]);
    QWB_CUDA(ctx, cudaMemcpyAsync(bl + pd * Pb + nlb * nx, me + pd * P, bytes, cudaMemcpyDeviceToDevice, s));
    // my extra row ny_local+1 -> above's first owned row (plane pu)
    const int64_t nla = ny_local_host[above], Pa = nx * (nla + 2);
    double2* ab = reinterpret_cast<double2*>(planes_host[above]);
    QWB_CUDA(ctx, cudaMemcpyAsync(ab + pu * Pa + nx, me + pu * P + (nl + 1) * nx, bytes,
                                  cudaMemcpyDeviceToDevice, s));
  }
  return QWB_OK;
}

}  // extern "C"
