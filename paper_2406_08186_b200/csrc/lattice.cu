// lattice.cu — matrix-free coined Grover step on the periodic 2-D lattice.
//
// Replaces, for `grid(nx, ny, periodic=True)` with nx, ny >= 3, the CSR step
// `matvec_mul(U, psi)` of coined.simulate (coined.py:263-270, backend.py:394-404)
// with U = S C built by coined.evolution_operator (coined.py:230-238).
//
// State layout in HBM ("planes"): four direction planes [D, L, R, U], each a
// dense nx*ny complex128 array indexed by vertex id v = x + nx*y, holding the
// amplitude of the arc leaving v towards its down/left/right/up neighbour.  The
// reference's arc order (tail-major, heads ascending, graphs.py:178-194) is a
// per-vertex permutation of the same four values whose slot order depends on
// the vertex position class:
//     interior          D L R U
//     x in {0, nx-1}    D R L U
//     y == 0            L R U D   (R L U D on x edges)
//     y == ny-1         U D L R   (U D R L on x edges)
// qwb_lattice_to_planes / _from_planes convert exactly.
//
// Step (push form).  Vertex w reads its 4 amplitudes (4 coalesced 16-B loads),
// forms for every direction e the row value
//     O_e(w) = p0 + ((p1 + p2) + p3),  p_i = (i == slot(e) ? -0.5 : 0.5) * s_i
// with s_i the amplitudes in w's reference slot order (this is exactly
// numpy's reduceat over U's row), or O_e(w) = -psi_e(w) when w
// is marked (the -I oracle, coined.py:188-219), and stores it to
//     flip-flop : plane(-e)[w + e]     (row (w+e, w) of U)
//     persistent: plane(e)[w + e]      (row (w+e, w+2e) of U)
// i.e. 4 shifted-but-coalesced 16-B stores.  No shared memory and no halo:
// every byte of psi is read once and every byte of psi' written once, 32 B per
// arc per step — the HBM roofline of this operator.
#include "qwb_internal.cuh"

namespace {

using qwb::abs2_np;
using qwb::cadd;
using qwb::cmul_np;

constexpr int kMaxTrace = 8;
struct TraceArgs {
  int n;
  int64_t v[kMaxTrace];
  double* out;
};

// numpy product (c + 0i) * a
__device__ __forceinline__ double2 scale_np(double c, double2 a) {
  return cmul_np(make_double2(c, 0.0), a);
}

struct Slots {
  // amplitudes in reference slot order and the slot of each direction
  double2 s0, s1, s2, s3;
  int pD, pL, pR, pU;
};

__device__ __forceinline__ Slots order_slots(int x, int y, int nx, int ny, double2 vD, double2 vL,
                                             double2 vR, double2 vU) {
  Slots o;
  const bool xe = (x == 0) | (x == nx - 1);
  const double2 h0 = xe ? vR : vL;
  const double2 h1 = xe ? vL : vR;
  int ph0, ph1;
  if (y == 0) {
    o.s0 = h0; o.s1 = h1; o.s2 = vU; o.s3 = vD;
    ph0 = 0; ph1 = 1; o.pU = 2; o.pD = 3;
  } else if (y == ny - 1) {
    o.s0 = vU; o.s1 = vD; o.s2 = h0; o.s3 = h1;
    o.pU = 0; o.pD = 1; ph0 = 2; ph1 = 3;
  } else {
    o.s0 = vD; o.s1 = h0; o.s2 = h1; o.s3 = vU;
    o.pD = 0; ph0 = 1; ph1 = 2; o.pU = 3;
  }
  o.pL = xe ? ph1 : ph0;
  o.pR = xe ? ph0 : ph1;
  return o;
}

__device__ __forceinline__ double2 pick(int p, double2 a0, double2 a1, double2 a2, double2 a3) {
  double2 r = a0;
  r = (p == 1) ? a1 : r;
  r = (p == 2) ? a2 : r;
  r = (p == 3) ? a3 : r;
  return r;
}

// slot -> direction for the conversions
__device__ __forceinline__ void slot_dirs(int x, int y, int nx, int ny, int d[4]) {
  const bool xe = (x == 0) | (x == nx - 1);
  const int h0 = xe ? 2 : 1, h1 = xe ? 1 : 2;  // L=1, R=2
  if (y == 0) {
    d[0] = h0; d[1] = h1; d[2] = 3; d[3] = 0;
  } else if (y == ny - 1) {
    d[0] = 3; d[1] = 0; d[2] = h0; d[3] = h1;
  } else {
    d[0] = 0; d[1] = h0; d[2] = h1; d[3] = 3;
  }
}

template <int SHIFT, bool MARKED, bool PROB, bool TRACE>
__global__ void __launch_bounds__(256)
lattice_step_kernel(int nx, int ny, const double2* __restrict__ in, double2* __restrict__ out,
                    const uint32_t* __restrict__ bits, double* __restrict__ prob, TraceArgs tr) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= nx) return;
  const int64_t n = (int64_t)nx * ny;
  for (int y = blockIdx.y; y < ny; y += gridDim.y) {
    const int64_t w = (int64_t)y * nx + x;
    const double2 vD = __ldcs(in + w);
    const double2 vL = __ldcs(in + n + w);
    const double2 vR = __ldcs(in + 2 * n + w);
    const double2 vU = __ldcs(in + 3 * n + w);
    const Slots o = order_slots(x, y, nx, ny, vD, vL, vR, vU);

    double2 oD, oL, oR, oU;
    bool marked = false;
    if (MARKED) marked = (__ldg(bits + (w >> 5)) >> (w & 31)) & 1u;
    if (MARKED && marked) {
      oD = scale_np(-1.0, vD);
      oL = scale_np(-1.0, vL);
      oR = scale_np(-1.0, vR);
      oU = scale_np(-1.0, vU);
    } else {
      const double2 q0 = scale_np(0.5, o.s0), q1 = scale_np(0.5, o.s1);
      const double2 q2 = scale_np(0.5, o.s2), q3 = scale_np(0.5, o.s3);
      const double2 n0 = scale_np(-0.5, o.s0), n1 = scale_np(-0.5, o.s1);
      const double2 n2 = scale_np(-0.5, o.s2), n3 = scale_np(-0.5, o.s3);
      const double2 t12 = cadd(q1, q2);
      const double2 O0 = cadd(n0, cadd(t12, q3));
      const double2 O1 = cadd(q0, cadd(cadd(n1, q2), q3));
      const double2 O2 = cadd(q0, cadd(cadd(q1, n2), q3));
      const double2 O3 = cadd(q0, cadd(t12, n3));
      oD = pick(o.pD, O0, O1, O2, O3);
      oL = pick(o.pL, O0, O1, O2, O3);
      oR = pick(o.pR, O0, O1, O2, O3);
      oU = pick(o.pU, O0, O1, O2, O3);
    }
    const int ym = (y == 0) ? ny - 1 : y - 1;
    const int yp = (y == ny - 1) ? 0 : y + 1;
    const int xm = (x == 0) ? nx - 1 : x - 1;
    const int xp = (x == nx - 1) ? 0 : x + 1;
    const int64_t below = (int64_t)ym * nx + x, above = (int64_t)yp * nx + x;
    const int64_t left = (int64_t)y * nx + xm, right = (int64_t)y * nx + xp;
    if (SHIFT == QWB_SHIFT_FLIPFLOP) {
      __stcs(out + 3 * n + below, oD);   // arc (below -> w) points up
      __stcs(out + 2 * n + left, oL);    // arc (left  -> w) points right
      __stcs(out + 1 * n + right, oR);   // arc (right -> w) points left
      __stcs(out + 0 * n + above, oU);   // arc (above -> w) points down
    } else {
      __stcs(out + 0 * n + below, oD);
      __stcs(out + 1 * n + left, oL);
      __stcs(out + 2 * n + right, oR);
      __stcs(out + 3 * n + above, oU);
    }
    if (PROB || TRACE) {
      const double m0 = abs2_np(o.s0), m1 = abs2_np(o.s1), m2 = abs2_np(o.s2), m3 = abs2_np(o.s3);
      const double p = __dadd_rn(m0, __dadd_rn(__dadd_rn(m1, m2), m3));
      if (PROB) __stcs(prob + w, p);
      if (TRACE) {
#pragma unroll
        for (int j = 0; j < kMaxTrace; ++j)
          if (j < tr.n && tr.v[j] == w) tr.out[j] = p;
      }
    }
  }
}

__global__ void to_planes_kernel(int nx, int ny, const double2* __restrict__ arcs,
                                 double2* __restrict__ planes) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= nx) return;
  const int64_t n = (int64_t)nx * ny;
  for (int y = blockIdx.y; y < ny; y += gridDim.y) {
    const int64_t w = (int64_t)y * nx + x;
    int d[4];
    slot_dirs(x, y, nx, ny, d);
#pragma unroll
    for (int i = 0; i < 4; ++i) planes[d[i] * n + w] = arcs[4 * w + i];
  }
}

__global__ void from_planes_kernel(int nx, int ny, const double2* __restrict__ planes,
                                   double2* __restrict__ arcs) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= nx) return;
  const int64_t n = (int64_t)nx * ny;
  for (int y = blockIdx.y; y < ny; y += gridDim.y) {
    const int64_t w = (int64_t)y * nx + x;
    int d[4];
    slot_dirs(x, y, nx, ny, d);
#pragma unroll
    for (int i = 0; i < 4; ++i) arcs[4 * w + i] = planes[d[i] * n + w];
  }
}

__global__ void lattice_prob_kernel(int nx, int ny, const double2* __restrict__ planes,
                                    double* __restrict__ p) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= nx) return;
  const int64_t n = (int64_t)nx * ny;
  for (int y = blockIdx.y; y < ny; y += gridDim.y) {
    const int64_t w = (int64_t)y * nx + x;
    const Slots o = order_slots(x, y, nx, ny, planes[w], planes[n + w], planes[2 * n + w],
                                planes[3 * n + w]);
    const double m0 = abs2_np(o.s0), m1 = abs2_np(o.s1), m2 = abs2_np(o.s2), m3 = abs2_np(o.s3);
    p[w] = __dadd_rn(m0, __dadd_rn(__dadd_rn(m1, m2), m3));
  }
}

dim3 lattice_grid(int64_t nx, int64_t ny) {
  const unsigned gx = (unsigned)((nx + 255) / 256);
  const unsigned gy = (unsigned)(ny < 65535 ? ny : 65535);
  return dim3(gx, gy, 1);
}

int check_dims(qwb_ctx* ctx, int64_t nx, int64_t ny) {
  if (nx < 3 || ny < 3)
    QWB_FAIL(ctx, QWB_E_UNSUPPORTED, "matrix-free lattice needs nx, ny >= 3 (got %lld x %lld)",
             (long long)nx, (long long)ny);
  if (nx > (1LL << 30) || ny > (1LL << 30) || nx * ny > (1LL << 34))
    QWB_FAIL(ctx, QWB_E_DIMENSION, "lattice %lld x %lld too large", (long long)nx, (long long)ny);
  return QWB_OK;
}

template <int SHIFT, bool MARKED, bool PROB, bool TRACE>
void launch_step_t(dim3 g, cudaStream_t s, int nx, int ny, const double2* in, double2* out,
                   const uint32_t* bits, double* prob, const TraceArgs& tr) {
  lattice_step_kernel<SHIFT, MARKED, PROB, TRACE><<<g, 256, 0, s>>>(nx, ny, in, out, bits, prob, tr);
}

template <int SHIFT>
void launch_step_s(dim3 g, cudaStream_t s, int nx, int ny, const double2* in, double2* out,
                   const uint32_t* bits, double* prob, const TraceArgs& tr) {
  const bool m = bits != nullptr, p = prob != nullptr, t = tr.n > 0 && tr.out != nullptr;
  if (m) {
    if (p) {
      if (t) launch_step_t<SHIFT, true, true, true>(g, s, nx, ny, in, out, bits, prob, tr);
      else   launch_step_t<SHIFT, true, true, false>(g, s, nx, ny, in, out, bits, prob, tr);
    } else {
      if (t) launch_step_t<SHIFT, true, false, true>(g, s, nx, ny, in, out, bits, prob, tr);
      else   launch_step_t<SHIFT, true, false, false>(g, s, nx, ny, in, out, bits, prob, tr);
    }
  } else {
    if (p) {
      if (t) launch_step_t<SHIFT, false, true, true>(g, s, nx, ny, in, out, bits, prob, tr);
      else   launch_step_t<SHIFT, false, true, false>(g, s, nx, ny, in, out, bits, prob, tr);
    } else {
      if (t) launch_step_t<SHIFT, false, false, true>(g, s, nx, ny, in, out, bits, prob, tr);
      else   launch_step_t<SHIFT, false, false, false>(g, s, nx, ny, in, out, bits, prob, tr);
    }
  }
}

void launch_step(int shift, dim3 g, cudaStream_t s, int nx, int ny, const double2* in,
                 double2* out, const uint32_t* bits, double* prob, const TraceArgs& tr) {
  if (shift == QWB_SHIFT_FLIPFLOP)
    launch_step_s<QWB_SHIFT_FLIPFLOP>(g, s, nx, ny, in, out, bits, prob, tr);
  else
    launch_step_s<QWB_SHIFT_PERSISTENT>(g, s, nx, ny, in, out, bits, prob, tr);
}

}  // namespace

extern "C" {

int qwb_lattice_to_planes(qwb_ctx* ctx, int64_t nx, int64_t ny, const qwb_z* arcs, qwb_z* planes,
                          void* stream) {
  QWB_BEGIN(ctx);
  int st = check_dims(ctx, nx, ny);
  if (st) return st;
  to_planes_kernel<<<lattice_grid(nx, ny), 256, 0, qwb::as_stream(stream)>>>(
      (int)nx, (int)ny, reinterpret_cast<const double2*>(arcs), reinterpret_cast<double2*>(planes));
  QWB_LAUNCH_CHECK(ctx, "to_planes_kernel");
  return QWB_OK;
}

int qwb_lattice_from_planes(qwb_ctx* ctx, int64_t nx, int64_t ny, const qwb_z* planes, qwb_z* arcs,
                            void* stream) {
  QWB_BEGIN(ctx);
  int st = check_dims(ctx, nx, ny);
  if (st) return st;
  from_planes_kernel<<<lattice_grid(nx, ny), 256, 0, qwb::as_stream(stream)>>>(
      (int)nx, (int)ny, reinterpret_cast<const double2*>(planes), reinterpret_cast<double2*>(arcs));
  QWB_LAUNCH_CHECK(ctx, "from_planes_kernel");
  return QWB_OK;
}

int qwb_lattice_step(qwb_ctx* ctx, int64_t nx, int64_t ny, int shift, const uint32_t* marked_bits,
                     const qwb_z* in, qwb_z* out, double* prob_in, void* stream) {
  QWB_BEGIN(ctx);
  int st = check_dims(ctx, nx, ny);
  if (st) return st;
  if (shift != QWB_SHIFT_FLIPFLOP && shift != QWB_SHIFT_PERSISTENT)
    QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "shift: unknown shift code %d", shift);
  TraceArgs tr{};
  tr.n = 0;
  tr.out = nullptr;
  launch_step(shift, lattice_grid(nx, ny), qwb::as_stream(stream), (int)nx, (int)ny,
              reinterpret_cast<const double2*>(in), reinterpret_cast<double2*>(out), marked_bits,
              prob_in, tr);
  QWB_LAUNCH_CHECK(ctx, "lattice_step_kernel");
  return QWB_OK;
}

int qwb_lattice_run(qwb_ctx* ctx, int64_t nx, int64_t ny, int shift, const uint32_t* marked_bits,
                    qwb_z* a, qwb_z* b, int64_t steps, const int64_t* trace_vertices_host,
                    int n_trace, double* trace, int* final_in_b_host, void* stream) {
  QWB_BEGIN(ctx);
  int st = check_dims(ctx, nx, ny);
  if (st) return st;
  if (shift != QWB_SHIFT_FLIPFLOP && shift != QWB_SHIFT_PERSISTENT)
    QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "shift: unknown shift code %d", shift);
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
  const dim3 g = lattice_grid(nx, ny);
  double2* cur = reinterpret_cast<double2*>(a);
  double2* nxt = reinterpret_cast<double2*>(b);
  for (int64_t k = 0; k < steps; ++k) {
    tr.out = trace ? trace + k * n_trace : nullptr;
    launch_step(shift, g, s, (int)nx, (int)ny, cur, nxt, marked_bits, nullptr, tr);
    double2* t = cur;
    cur = nxt;
    nxt = t;
  }
  QWB_LAUNCH_CHECK(ctx, "lattice_step_kernel");
  if (final_in_b_host) *final_in_b_host = (steps % 2) ? 1 : 0;
  return QWB_OK;
}

int qwb_lattice_probability(qwb_ctx* ctx, int64_t nx, int64_t ny, const qwb_z* planes, double* p,
                            void* stream) {
  QWB_BEGIN(ctx);
  int st = check_dims(ctx, nx, ny);
  if (st) return st;
  lattice_prob_kernel<<<lattice_grid(nx, ny), 256, 0, qwb::as_stream(stream)>>>(
      (int)nx, (int)ny, reinterpret_cast<const double2*>(planes), p);
  QWB_LAUNCH_CHECK(ctx, "lattice_prob_kernel");
  return QWB_OK;
}

}  // extern "C"
