// lattice.cu — matrix-free coined Grover step on the periodic 2-D lattice.
//
// Replaces, for `grid(nx, ny, periodic=True)` with nx, ny >= 3, the CSR step
// `matvec_mul(U, psi)` of coined.simulate (coined.py:263-270, backend.py:394-404)
// with U = S C built by coined.evolution_operator (coined.py:230-238).
//
// State layout in HBM ("planes"): four direction planes [D, L, R, U], each a
// dense (rows x nx) complex128 array indexed by vertex (x, y), holding the
// amplitude of the arc leaving the vertex towards its down/left/right/up
// neighbour.  The reference's arc order (tail-major, heads ascending,
// graphs.py:178-194) is a per-vertex permutation of the same four values whose
// slot order depends on the vertex position class:
//     interior          D L R U
//     x in {0, nx-1}    D R L U
//     y == 0            L R U D   (R L U D on x edges)
//     y == ny-1         U D L R   (U D R L on x edges)
// qwb_lattice_to_planes / _from_planes convert exactly.
//
// Step (push form).  Vertex w reads its 4 amplitudes (4 coalesced 16-B loads),
// forms for every direction e the row value
//     O_e(w) = p0 + ((p1 + p2) + p3),  p_i = (i == slot(e) ? -0.5 : 0.5) * s_i
// with s_i the amplitudes in w's reference slot order (exactly numpy's
// reduceat over U's row), or O_e(w) = -psi_e(w) when w is
// marked (the -I oracle, coined.py:188-219), and stores it to
//     flip-flop : plane(-e)[w + e]     (row (w+e, w) of U)
//     persistent: plane(e)[w + e]      (row (w+e, w+2e) of U)
// i.e. 4 shifted-but-coalesced 16-B stores.  No shared memory and no halo
// reads: every byte of psi is read once and every byte of psi' written once,
// 32 B per arc per step — the HBM roofline of this operator.
//
// Slabs (multi-GPU).  A rank owns global rows [y0, y0 + ny_local) of an
// nx x ny torus, stored as local rows 1..ny_local of planes with one extra row
// on each side (local rows 0 and ny_local + 1).  Because the step is a push,
// a slab needs NO halo input: the only outputs it cannot produce are plane D
// of its first row and plane U of its last row, which the neighbours push into
// their own extra rows.  Exchanging those two nx-long rows per step (NCCL
// send/recv, comm.cu) completes the state.  Position classes use GLOBAL y, so
// every arc is computed by the same formula as on one GPU: sharded results are
// bitwise identical to the single-GPU run.
#include "qwb_lattice.cuh"

namespace {

using qwb::abs2_np;
using qwb::cadd;
using qwb::cmul_np;
using qwb::Geom;
using qwb::kMaxTrace;
using qwb::Rows;
using qwb::TraceArgs;

using qwb::order_slots;
using qwb::pick;
using qwb::scale_np;
using qwb::Slots;

// slot -> direction (D=0, L=1, R=2, U=3) for the conversions
__device__ __forceinline__ void slot_dirs(int x, int gy, int nx, int ny, int d[4]) {
  const bool xe = (x == 0) | (x == nx - 1);
  const int h0 = xe ? 2 : 1, h1 = xe ? 1 : 2;
  if (gy == 0) {
    d[0] = h0; d[1] = h1; d[2] = 3; d[3] = 0;
  } else if (gy == ny - 1) {
    d[0] = 3; d[1] = 0; d[2] = h0; d[3] = h1;
  } else {
    d[0] = 0; d[1] = h0; d[2] = h1; d[3] = 3;
  }
}

__device__ __forceinline__ int global_row(const Geom& g, int ly) {
  int gy = g.gy0 + ly;   // >= 0; a whole-torus slab's ghost rows can wrap twice
  while (gy >= g.ny) gy -= g.ny;
  return gy;
}

template <int SHIFT, bool MARKED, bool PROB, bool TRACE>
__global__ void __launch_bounds__(256)
lattice_step_kernel(Geom g, Rows rows, const double2* __restrict__ in, double2* __restrict__ out,
                    const uint32_t* __restrict__ bits, double* __restrict__ prob, int prob_row0,
                    TraceArgs tr) {
  qwb::pdl_enter();   // the previous step's output is this step's input
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= g.nx) return;
  const int64_t P = g.pstride;
  for (int r = blockIdx.y; r < rows.nrows; r += gridDim.y) {
    const int ly = rows.row0 + r * rows.rstep;
    const int gy = global_row(g, ly);
    const int64_t w = (int64_t)ly * g.nx + x;
    const double2 vD = __ldcs(in + w);
    const double2 vL = __ldcs(in + P + w);
    const double2 vR = __ldcs(in + 2 * P + w);
    const double2 vU = __ldcs(in + 3 * P + w);
    const Slots o = order_slots(x, gy, g.nx, g.ny, vD, vL, vR, vU);

    double2 oD, oL, oR, oU;
    bool marked = false;
    if (MARKED) {
      const int64_t wg = (int64_t)gy * g.nx + x;
      marked = (__ldg(bits + (wg >> 5)) >> (wg & 31)) & 1u;
    }
    qwb::vertex_outputs(o, marked, vD, vL, vR, vU, oD, oL, oR, oU);
    int ym = ly - 1, yp = ly + 1;
    if (g.wrap) {
      ym = (ly == 0) ? g.lrows - 1 : ym;
      yp = (ly == g.lrows - 1) ? 0 : yp;
    }
    const int xm = (x == 0) ? g.nx - 1 : x - 1;
    const int xp = (x == g.nx - 1) ? 0 : x + 1;
    const int64_t below = (int64_t)ym * g.nx + x, above = (int64_t)yp * g.nx + x;
    const int64_t left = (int64_t)ly * g.nx + xm, right = (int64_t)ly * g.nx + xp;
    if (SHIFT == QWB_SHIFT_FLIPFLOP) {
      __stcs(out + 3 * P + below, oD);   // arc (below -> w) points up
      __stcs(out + 2 * P + left, oL);    // arc (left  -> w) points right
      __stcs(out + 1 * P + right, oR);   // arc (right -> w) points left
      __stcs(out + 0 * P + above, oU);   // arc (above -> w) points down
    } else {
      __stcs(out + 0 * P + below, oD);
      __stcs(out + 1 * P + left, oL);
      __stcs(out + 2 * P + right, oR);
      __stcs(out + 3 * P + above, oU);
    }
    if (PROB || TRACE) {
      const double m0 = abs2_np(o.s0), m1 = abs2_np(o.s1), m2 = abs2_np(o.s2), m3 = abs2_np(o.s3);
      const double p = __dadd_rn(m0, __dadd_rn(__dadd_rn(m1, m2), m3));
      if (PROB) __stcs(prob + (int64_t)(ly - prob_row0) * g.nx + x, p);
      if (TRACE) {
        const int64_t wg = (int64_t)gy * g.nx + x;
#pragma unroll
        for (int j = 0; j < kMaxTrace; ++j)
          if (j < tr.n && tr.v[j] == wg) tr.out[j] = p;
      }
    }
  }
}

// arcs (reference order, owned rows only, contiguous) <-> planes
__global__ void to_planes_kernel(Geom g, int ly0, int nrows, const double2* __restrict__ arcs,
                                 double2* __restrict__ planes) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= g.nx) return;
  for (int r = blockIdx.y; r < nrows; r += gridDim.y) {
    const int ly = ly0 + r;
    const int64_t w = (int64_t)ly * g.nx + x;
    const int64_t a = (int64_t)r * g.nx + x;
    int d[4];
    slot_dirs(x, global_row(g, ly), g.nx, g.ny, d);
#pragma unroll
    for (int i = 0; i < 4; ++i) planes[d[i] * g.pstride + w] = arcs[4 * a + i];
  }
}

__global__ void from_planes_kernel(Geom g, int ly0, int nrows, const double2* __restrict__ planes,
                                   double2* __restrict__ arcs) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= g.nx) return;
  for (int r = blockIdx.y; r < nrows; r += gridDim.y) {
    const int ly = ly0 + r;
    const int64_t w = (int64_t)ly * g.nx + x;
    const int64_t a = (int64_t)r * g.nx + x;
    int d[4];
    slot_dirs(x, global_row(g, ly), g.nx, g.ny, d);
#pragma unroll
    for (int i = 0; i < 4; ++i) arcs[4 * a + i] = planes[d[i] * g.pstride + w];
  }
}

__global__ void lattice_prob_kernel(Geom g, int ly0, int nrows, const double2* __restrict__ planes,
                                    double* __restrict__ p) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= g.nx) return;
  const int64_t P = g.pstride;
  for (int r = blockIdx.y; r < nrows; r += gridDim.y) {
    const int ly = ly0 + r;
    const int64_t w = (int64_t)ly * g.nx + x;
    const Slots o = order_slots(x, global_row(g, ly), g.nx, g.ny, planes[w], planes[P + w],
                                planes[2 * P + w], planes[3 * P + w]);
    const double m0 = abs2_np(o.s0), m1 = abs2_np(o.s1), m2 = abs2_np(o.s2), m3 = abs2_np(o.s3);
    p[(int64_t)r * g.nx + x] = __dadd_rn(m0, __dadd_rn(__dadd_rn(m1, m2), m3));
  }
}

dim3 grid_for(int nx, int nrows) {
  const unsigned gx = (unsigned)((nx + 255) / 256);
  const unsigned gy = (unsigned)(nrows < 65535 ? (nrows > 0 ? nrows : 1) : 65535);
  return dim3(gx, gy, 1);
}

template <int SHIFT, bool MARKED, bool PROB, bool TRACE>
void launch_t(cudaStream_t s, const Geom& g, const Rows& r, const double2* in, double2* out,
              const uint32_t* bits, double* prob, int prob_row0, const TraceArgs& tr) {
  static const bool pdl = qwb::env_flag("QWB_STEP_PDL", 1) != 0;   // see qwb::launch_pdl
  qwb::launch_pdl(pdl, lattice_step_kernel<SHIFT, MARKED, PROB, TRACE>, grid_for(g.nx, r.nrows), 256, 0, s,
                  g, r, in, out, bits, prob, prob_row0, tr);
}

template <int SHIFT>
void launch_s(cudaStream_t s, const Geom& g, const Rows& r, const double2* in, double2* out,
              const uint32_t* bits, double* prob, int prob_row0, const TraceArgs& tr) {
  const bool m = bits != nullptr, p = prob != nullptr, t = tr.n > 0 && tr.out != nullptr;
  if (m) {
    if (p) {
      if (t) launch_t<SHIFT, true, true, true>(s, g, r, in, out, bits, prob, prob_row0, tr);
      else   launch_t<SHIFT, true, true, false>(s, g, r, in, out, bits, prob, prob_row0, tr);
    } else {
      if (t) launch_t<SHIFT, true, false, true>(s, g, r, in, out, bits, prob, prob_row0, tr);
      else   launch_t<SHIFT, true, false, false>(s, g, r, in, out, bits, prob, prob_row0, tr);
    }
  } else {
    if (p) {
      if (t) launch_t<SHIFT, false, true, true>(s, g, r, in, out, bits, prob, prob_row0, tr);
      else   launch_t<SHIFT, false, true, false>(s, g, r, in, out, bits, prob, prob_row0, tr);
    } else {
      if (t) launch_t<SHIFT, false, false, true>(s, g, r, in, out, bits, prob, prob_row0, tr);
      else   launch_t<SHIFT, false, false, false>(s, g, r, in, out, bits, prob, prob_row0, tr);
    }
  }
}

int check_dims(qwb_ctx* ctx, int64_t nx, int64_t ny) {
  if (nx < 3 || ny < 3)
    QWB_FAIL(ctx, QWB_E_UNSUPPORTED, "matrix-free lattice needs nx, ny >= 3 (got %lld x %lld)",
             (long long)nx, (long long)ny);
  if (nx > (1LL << 30) || ny > (1LL << 30) || nx * ny > (1LL << 34))
    QWB_FAIL(ctx, QWB_E_DIMENSION, "lattice %lld x %lld too large", (long long)nx, (long long)ny);
  return QWB_OK;
}

Geom single_geom(int64_t nx, int64_t ny) {
  Geom g;
  g.nx = (int)nx;
  g.ny = (int)ny;
  g.lrows = (int)ny;
  g.gy0 = 0;
  g.wrap = 1;
  g.pstride = nx * ny;
  return g;
}

}  // namespace

namespace qwb {

void lattice_launch(int shift, cudaStream_t s, const Geom& g, const Rows& r, const double2* in,
                    double2* out, const uint32_t* bits, double* prob, int prob_row0,
                    const TraceArgs& tr) {
  if (r.nrows <= 0) return;
  if (shift == QWB_SHIFT_FLIPFLOP)
    launch_s<QWB_SHIFT_FLIPFLOP>(s, g, r, in, out, bits, prob, prob_row0, tr);
  else
    launch_s<QWB_SHIFT_PERSISTENT>(s, g, r, in, out, bits, prob, prob_row0, tr);
}

int lattice_check_shift(qwb_ctx* ctx, int shift) {
  if (shift != QWB_SHIFT_FLIPFLOP && shift != QWB_SHIFT_PERSISTENT)
    QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "shift: unknown shift code %d", shift);
  return QWB_OK;
}

int lattice_slab_geom(qwb_ctx* ctx, int64_t nx, int64_t ny, int64_t y0, int64_t ny_local, Geom* g) {
  int st = check_dims(ctx, nx, ny);
  if (st) return st;
  if (ny_local < 2 || y0 < 0 || y0 + ny_local > ny)
    QWB_FAIL(ctx, QWB_E_DIMENSION, "slab rows [%lld, %lld) invalid for ny=%lld (need >= 2 rows)",
             (long long)y0, (long long)(y0 + ny_local), (long long)ny);
  g->nx = (int)nx;
  g->ny = (int)ny;
  g->lrows = (int)(ny_local + 2);
  g->gy0 = (int)((y0 - 1 + ny) % ny);
  g->wrap = 0;
  g->pstride = nx * (ny_local + 2);
  return QWB_OK;
}

// slab with G ghost rows each side: owned rows are local rows [G, G + ny_local)
int lattice_slab_geom_g(qwb_ctx* ctx, int64_t nx, int64_t ny, int64_t y0, int64_t ny_local, int64_t ghost,
                        Geom* g) {
  int st = check_dims(ctx, nx, ny);
  if (st) return st;
  if (ghost < 1 || ghost > 32) QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "ghost rows must be in 1..32");
  if (ny_local < ghost || ny_local < 2 || y0 < 0 || y0 + ny_local > ny)
    QWB_FAIL(ctx, QWB_E_DIMENSION, "slab rows [%lld, %lld) invalid for ny=%lld (need >= %lld rows)",
             (long long)y0, (long long)(y0 + ny_local), (long long)ny, (long long)(ghost > 2 ? ghost : 2));
  g->nx = (int)nx;
  g->ny = (int)ny;
  g->lrows = (int)(ny_local + 2 * ghost);
  g->gy0 = (int)(((y0 - ghost) % ny + ny) % ny);
  g->wrap = 0;
  g->pstride = nx * (ny_local + 2 * ghost);
  return QWB_OK;
}

Rows slab_rows(int64_t ny_local, int part) {
  const int nl = (int)ny_local;
  if (part == 1) return Rows{1, nl - 1, 2};
  if (part == 2) return Rows{2, 1, nl - 2};
  return Rows{1, 1, nl};
}

}  // namespace qwb

extern "C" {

int qwb_lattice_to_planes(qwb_ctx* ctx, int64_t nx, int64_t ny, const qwb_z* arcs, qwb_z* planes,
                          void* stream) {
  QWB_BEGIN(ctx);
  int st = check_dims(ctx, nx, ny);
  if (st) return st;
  const Geom g = single_geom(nx, ny);
  to_planes_kernel<<<grid_for(g.nx, g.ny), 256, 0, qwb::as_stream(stream)>>>(
      g, 0, g.ny, reinterpret_cast<const double2*>(arcs), reinterpret_cast<double2*>(planes));
  QWB_LAUNCH_CHECK(ctx, "to_planes_kernel");
  return QWB_OK;
}

int qwb_lattice_from_planes(qwb_ctx* ctx, int64_t nx, int64_t ny, const qwb_z* planes, qwb_z* arcs,
                            void* stream) {
  QWB_BEGIN(ctx);
  int st = check_dims(ctx, nx, ny);
  if (st) return st;
  const Geom g = single_geom(nx, ny);
  from_planes_kernel<<<grid_for(g.nx, g.ny), 256, 0, qwb::as_stream(stream)>>>(
      g, 0, g.ny, reinterpret_cast<const double2*>(planes), reinterpret_cast<double2*>(arcs));
  QWB_LAUNCH_CHECK(ctx, "from_planes_kernel");
  return QWB_OK;
}

int qwb_lattice_step(qwb_ctx* ctx, int64_t nx, int64_t ny, int shift, const uint32_t* marked_bits,
                     const qwb_z* in, qwb_z* out, double* prob_in, void* stream) {
  QWB_BEGIN(ctx);
  int st = check_dims(ctx, nx, ny);
  if (!st) st = qwb::lattice_check_shift(ctx, shift);
  if (st) return st;
  TraceArgs tr{};
  const Geom g = single_geom(nx, ny);
  const Rows r{0, 1, g.ny};
  qwb::lattice_launch(shift, qwb::as_stream(stream), g, r, reinterpret_cast<const double2*>(in),
                      reinterpret_cast<double2*>(out), marked_bits, prob_in, 0, tr);
  QWB_LAUNCH_CHECK(ctx, "lattice_step_kernel");
  return QWB_OK;
}

int qwb_lattice_run(qwb_ctx* ctx, int64_t nx, int64_t ny, int shift, const uint32_t* marked_bits,
                    const int64_t* marked_host, int64_t n_marked, qwb_z* a, qwb_z* b, int64_t steps,
                    const int64_t* trace_vertices_host, int n_trace, double* trace,
                    int* final_in_b_host, void* stream) {
  QWB_BEGIN(ctx);
  int st = check_dims(ctx, nx, ny);
  if (!st) st = qwb::lattice_check_shift(ctx, shift);
  if (st) return st;
  if (steps < 0) QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "steps must be >= 0");
  if (n_trace < 0 || n_trace > kMaxTrace)
    QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "at most %d trace vertices", kMaxTrace);
  TraceArgs tr{};
  tr.n = trace ? n_trace : 0;
  for (int j = 0; j < tr.n; ++j) {
    tr.v[j] = trace_vertices_host[j];
    if (tr.v[j] < 0 || tr.v[j] >= nx * ny)
      QWB_FAIL(ctx, QWB_E_MARKED_OUT_OF_RANGE, "trace vertex %lld out of range", (long long)tr.v[j]);
  }
  cudaStream_t s = qwb::as_stream(stream);
  const Geom g = single_geom(nx, ny);
  const Rows r{0, 1, g.ny};
  double2* cur = reinterpret_cast<double2*>(a);
  double2* nxt = reinterpret_cast<double2*>(b);
  int swaps = 0;
  int64_t k = 0;
  // T coined steps per HBM pass when no per-step trace is requested
  if (n_marked > 0 && (!marked_bits || !marked_host))
    QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "marked vertices need both the bitmap and the host list");
  const int depth = qwb::lattice_tb_depth(nx, ny, n_marked);
  // untraced runs: one persistent dataflow launch for all whole T-step blocks
  const int nflow = depth > 0 ? qwb::lattice_flow_blocks(nx, ny, depth, trace != nullptr, steps, ctx->num_sms) : 0;
  if (nflow > 0) {
    st = qwb::lattice_flow_launch(ctx, shift, s, (int)nx, (int)ny, cur, nxt, marked_bits, marked_host, n_marked,
                                  nflow);
  }
  if (nflow > 0 && st == -1) {   // no co-resident grid here: one launch per T steps
    st = QWB_OK;
  } else if (nflow > 0) {
    if (st) return st;
    k = (int64_t)nflow * 4;   // the flow kernel's depth (lattice_tb.cu kFlowT)
    if (nflow & 1) {
      double2* t = cur;
      cur = nxt;
      nxt = t;
    }
    swaps += nflow;
  }
  if (depth > 0 && steps - k >= 2) {
    // subnormal guard: the first launch and every kCheckEvery-th test the
    // tiles' inputs; a hit switches the rest of the run to numpy's arithmetic
    int* sticky = nullptr;
    st = qwb::lattice_sticky(ctx, &sticky);
    if (st) return st;
    QWB_CUDA(ctx, cudaMemsetAsync(sticky, 0, sizeof(int), s));
    int64_t i = 0;
    while (steps - k >= 2) {
      // whole T-step launches, then one shallower launch for a remainder >= 2
      const int d = steps - k >= depth ? depth : (int)(steps - k);
      st = qwb::lattice_tb_launch(ctx, d, shift, s, (int)nx, (int)ny, cur, nxt, marked_bits,
                                  marked_host, n_marked, trace_vertices_host, trace ? n_trace : 0,
                                  trace ? trace + k * n_trace : nullptr, i % qwb::kCheckEvery == 0 || d != depth,
                                  sticky);
      if (st) return st;
      double2* t = cur;
      cur = nxt;
      nxt = t;
      ++swaps;
      k += d;
      ++i;
    }
  }
  for (; k < steps; ++k) {
    tr.out = trace ? trace + k * n_trace : nullptr;
    qwb::lattice_launch(shift, s, g, r, cur, nxt, marked_bits, nullptr, 0, tr);
    double2* t = cur;
    cur = nxt;
    nxt = t;
    ++swaps;
  }
  QWB_LAUNCH_CHECK(ctx, "lattice kernels");
  if (final_in_b_host) *final_in_b_host = swaps & 1;
  return QWB_OK;
}

int qwb_lattice_probability(qwb_ctx* ctx, int64_t nx, int64_t ny, const qwb_z* planes, double* p,
                            void* stream) {
  QWB_BEGIN(ctx);
  int st = check_dims(ctx, nx, ny);
  if (st) return st;
  const Geom g = single_geom(nx, ny);
  lattice_prob_kernel<<<grid_for(g.nx, g.ny), 256, 0, qwb::as_stream(stream)>>>(
      g, 0, g.ny, reinterpret_cast<const double2*>(planes), p);
  QWB_LAUNCH_CHECK(ctx, "lattice_prob_kernel");
  return QWB_OK;
}

// ---- slabs (one rank's rows of a sharded torus) ----------------------------

int qwb_slab_to_planes(qwb_ctx* ctx, int64_t nx, int64_t ny, int64_t y0, int64_t ny_local,
                       const qwb_z* arcs, qwb_z* planes, void* stream) {
  QWB_BEGIN(ctx);
  Geom g;
  int st = qwb::lattice_slab_geom(ctx, nx, ny, y0, ny_local, &g);
  if (st) return st;
  to_planes_kernel<<<grid_for(g.nx, (int)ny_local), 256, 0, qwb::as_stream(stream)>>>(
      g, 1, (int)ny_local, reinterpret_cast<const double2*>(arcs), reinterpret_cast<double2*>(planes));
  QWB_LAUNCH_CHECK(ctx, "to_planes_kernel(slab)");
  return QWB_OK;
}

int qwb_slab_from_planes(qwb_ctx* ctx, int64_t nx, int64_t ny, int64_t y0, int64_t ny_local,
                         const qwb_z* planes, qwb_z* arcs, void* stream) {
  QWB_BEGIN(ctx);
  Geom g;
  int st = qwb::lattice_slab_geom(ctx, nx, ny, y0, ny_local, &g);
  if (st) return st;
  from_planes_kernel<<<grid_for(g.nx, (int)ny_local), 256, 0, qwb::as_stream(stream)>>>(
      g, 1, (int)ny_local, reinterpret_cast<const double2*>(planes), reinterpret_cast<double2*>(arcs));
  QWB_LAUNCH_CHECK(ctx, "from_planes_kernel(slab)");
  return QWB_OK;
}

int qwb_slab_probability(qwb_ctx* ctx, int64_t nx, int64_t ny, int64_t y0, int64_t ny_local,
                         const qwb_z* planes, double* p, void* stream) {
  QWB_BEGIN(ctx);
  Geom g;
  int st = qwb::lattice_slab_geom(ctx, nx, ny, y0, ny_local, &g);
  if (st) return st;
  lattice_prob_kernel<<<grid_for(g.nx, (int)ny_local), 256, 0, qwb::as_stream(stream)>>>(
      g, 1, (int)ny_local, reinterpret_cast<const double2*>(planes), p);
  QWB_LAUNCH_CHECK(ctx, "lattice_prob_kernel(slab)");
  return QWB_OK;
}

int qwb_slab_to_planes_g(qwb_ctx* ctx, int64_t nx, int64_t ny, int64_t y0, int64_t ny_local, int64_t ghost,
                         const qwb_z* arcs, qwb_z* planes, void* stream) {
  QWB_BEGIN(ctx);
  Geom g;
  int st = qwb::lattice_slab_geom_g(ctx, nx, ny, y0, ny_local, ghost, &g);
  if (st) return st;
  to_planes_kernel<<<grid_for(g.nx, (int)ny_local), 256, 0, qwb::as_stream(stream)>>>(
      g, (int)ghost, (int)ny_local, reinterpret_cast<const double2*>(arcs), reinterpret_cast<double2*>(planes));
  QWB_LAUNCH_CHECK(ctx, "to_planes_kernel(ghost slab)");
  return QWB_OK;
}

int qwb_slab_from_planes_g(qwb_ctx* ctx, int64_t nx, int64_t ny, int64_t y0, int64_t ny_local, int64_t ghost,
                           const qwb_z* planes, qwb_z* arcs, void* stream) {
  QWB_BEGIN(ctx);
  Geom g;
  int st = qwb::lattice_slab_geom_g(ctx, nx, ny, y0, ny_local, ghost, &g);
  if (st) return st;
  from_planes_kernel<<<grid_for(g.nx, (int)ny_local), 256, 0, qwb::as_stream(stream)>>>(
      g, (int)ghost, (int)ny_local, reinterpret_cast<const double2*>(planes), reinterpret_cast<double2*>(arcs));
  QWB_LAUNCH_CHECK(ctx, "from_planes_kernel(ghost slab)");
  return QWB_OK;
}

int qwb_slab_probability_g(qwb_ctx* ctx, int64_t nx, int64_t ny, int64_t y0, int64_t ny_local, int64_t ghost,
                           const qwb_z* planes, double* p, void* stream) {
  QWB_BEGIN(ctx);
  Geom g;
  int st = qwb::lattice_slab_geom_g(ctx, nx, ny, y0, ny_local, ghost, &g);
  if (st) return st;
  lattice_prob_kernel<<<grid_for(g.nx, (int)ny_local), 256, 0, qwb::as_stream(stream)>>>(
      g, (int)ghost, (int)ny_local, reinterpret_cast<const double2*>(planes), p);
  QWB_LAUNCH_CHECK(ctx, "lattice_prob_kernel(ghost slab)");
  return QWB_OK;
}

int qwb_slab_depth(int* depth_host) {
  if (depth_host) *depth_host = qwb::kSlabDepth;
  return QWB_OK;
}

int qwb_slab_ghost_rows(int64_t nx, int64_t ny, int64_t ny_local, int64_t n_marked, int* ghost_host) {
  // G = m T ghost rows (m temporally blocked launches per exchange), m = 4
  // (QWB_SLAB_GHOST_MULT, G <= 32) and G <= the thinnest slab; 0: not available
  // slabs run the T = kSlabDepth tile kernel whatever the torus default depth
  const int d = qwb::lattice_tb_depth(nx, ny, n_marked) > 0 ? qwb::lattice_slab_depth(qwb::kSlabDepth) : 0;
  int g = 0;
  if (d >= 2 && nx >= 64 && ny_local >= d) {
    const char* e = getenv("QWB_SLAB_GHOST_MULT");
    int m = (e && *e) ? atoi(e) : 4;
    if (m < 1) m = 1;
    if (m > 8) m = 8;
    if (m > ny_local / d) m = (int)(ny_local / d);
    if (m * d > 32) m = 32 / d;   // lattice_slab_geom_g: at most 32 ghost rows
    g = m * d;
  }
  if (ghost_host) *ghost_host = g;
  return QWB_OK;
}

// One launch on a ghost-row slab, no exchange.  nsteps == 1: one pull step
// (owned rows plus one ghost row each side pushed, so every owned output
// receives all four pushes).  nsteps == T (the slab depth): the temporally
// blocked kernel over the owned rows extended by ext rows each side (global
// rows [y0 - ext, y0 + ny_local + ext)); needs ghost - ext >= T valid ghost
// rows each side.  With G = mT, ext = (m-1)T, ..., T, 0 advance mT steps per
// exchange of mT rows.
int qwb_slab_advance_local(qwb_ctx* ctx, int64_t nx, int64_t ny, int64_t y0, int64_t ny_local, int64_t ghost,
                           int shift, const uint32_t* marked_bits, const int64_t* marked_host, int64_t n_marked,
                           const qwb_z* in, qwb_z* out, int nsteps, int ext, void* stream) {
  QWB_BEGIN(ctx);
  Geom g;
  int st = qwb::lattice_slab_geom_g(ctx, nx, ny, y0, ny_local, ghost, &g);
  if (!st) st = qwb::lattice_check_shift(ctx, shift);
  if (st) return st;
  if (ghost < 2) QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "ghost-row slabs need >= 2 ghost rows");
  if (n_marked > 0 && (!marked_bits || !marked_host))
    QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "marked vertices need both the bitmap and the host list");
  cudaStream_t s = qwb::as_stream(stream);
  const double2* x = reinterpret_cast<const double2*>(in);
  double2* y = reinterpret_cast<double2*>(out);
  if (nsteps == 1) {
    if (ext != 0) QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "pull steps cover the owned rows only (ext = 0)");
    TraceArgs tr{};
    qwb::lattice_launch(shift, s, g, Rows{(int)ghost - 1, 1, (int)ny_local + 2}, x, y, marked_bits, nullptr, 0, tr);
    QWB_LAUNCH_CHECK(ctx, "lattice_step_kernel(ghost slab)");
    return QWB_OK;
  }
  const int T = qwb::lattice_slab_depth(nsteps);
  if (T == 0 || nsteps != T) QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "nsteps must be 1 or the slab depth");
  if (ext < 0 || ghost - ext < T)
    QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "ext = %d leaves fewer than %d ghost rows", ext, T);
  const qwb::TbGeo geo{(int)(ny_local + 2 * ghost), (int)ghost - ext, (int)ny_local + 2 * ext, (int)y0 - ext, 0};
  st = qwb::lattice_tb_launch_geo(ctx, T, shift, s, (int)nx, (int)ny, geo, x, y, marked_bits, marked_host,
                                  n_marked, 0, 0);
  if (st) return st;
  QWB_LAUNCH_CHECK(ctx, "lattice_tb_kernel(ghost slab)");
  return QWB_OK;
}

int qwb_slab_step(qwb_ctx* ctx, int64_t nx, int64_t ny, int64_t y0, int64_t ny_local, int shift,
                  const uint32_t* marked_bits, const qwb_z* in, qwb_z* out, int part, void* stream) {
  QWB_BEGIN(ctx);
  Geom g;
  int st = qwb::lattice_slab_geom(ctx, nx, ny, y0, ny_local, &g);
  if (!st) st = qwb::lattice_check_shift(ctx, shift);
  if (st) return st;
  if (part < 0 || part > 2) QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "part must be 0, 1 or 2");
  TraceArgs tr{};
  qwb::lattice_launch(shift, qwb::as_stream(stream), g, qwb::slab_rows(ny_local, part),
                      reinterpret_cast<const double2*>(in), reinterpret_cast<double2*>(out),
                      marked_bits, nullptr, 0, tr);
  QWB_LAUNCH_CHECK(ctx, "lattice_step_kernel(slab)");
  return QWB_OK;
}

}  // extern "C"
