// qwb_lattice.cuh — lattice geometry shared by lattice.cu and comm.cu.
#pragma once
#include "qwb_internal.cuh"

namespace qwb {

constexpr int kMaxTrace = 8;
struct TraceArgs {
  int n;
  int64_t v[kMaxTrace];   // global vertex ids
  double* out;
};

// local-row geometry of a planes buffer
struct Geom {
  int nx;          // columns
  int ny;          // GLOBAL rows of the torus
  int lrows;       // rows stored (single GPU: ny; slab: ny_local + 2)
  int gy0;         // global row of local row 0, in [0, ny)
  int wrap;        // 1: single GPU, rows wrap inside the buffer; 0: slab with extra rows
  int64_t pstride; // plane stride = nx * lrows
};

// rows a launch covers: ly = row0 + i * rstep for i < nrows
struct Rows {
  int row0, rstep, nrows;
};

// numpy product (c + 0i) * a
__device__ __forceinline__ double2 scale_np(double c, double2 a) {
  return cmul_np(make_double2(c, 0.0), a);
}

struct Slots {
  double2 s0, s1, s2, s3;   // amplitudes in reference slot order
  int pD, pL, pR, pU;       // slot of each direction
};

// reference slot order of vertex (x, gy) on an nx x ny torus
__device__ __forceinline__ Slots order_slots(int x, int gy, int nx, int ny, double2 vD, double2 vL,
                                             double2 vR, double2 vU) {
  Slots o;
  const bool xe = (x == 0) | (x == nx - 1);
  const double2 h0 = xe ? vR : vL;
  const double2 h1 = xe ? vL : vR;
  int ph0, ph1;
  if (gy == 0) {
    o.s0 = h0; o.s1 = h1; o.s2 = vU; o.s3 = vD;
    ph0 = 0; ph1 = 1; o.pU = 2; o.pD = 3;
  } else if (gy == ny - 1) {
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

// The four row values of U that vertex w feeds (one per direction e):
// O_e = p0 + ((p1 + p2) + p3), p_i = (i == slot(e) ? -0.5 : 0.5) * s_i, numpy's
// reduceat over the row; -psi_e for a marked vertex.
__device__ __forceinline__ void vertex_outputs(const Slots& o, bool marked, double2 vD, double2 vL,
                                               double2 vR, double2 vU, double2& oD, double2& oL,
                                               double2& oR, double2& oU) {
  if (marked) {
    oD = scale_np(-1.0, vD);
    oL = scale_np(-1.0, vL);
    oR = scale_np(-1.0, vR);
    oU = scale_np(-1.0, vU);
    return;
  }
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

// ---- doubled-space forms (temporally blocked kernels) -----------------------
// numpy computes O = q0 + ((q1 + q2) + q3) with q_i = +-0.5 s_i.  When every
// product 0.5 s_i is exact, halving commutes with round-to-nearest, so
//     O = 0.5 * fl(+-s0 + fl(fl(+-s1 +- s2) +- s3))
// and the fused kernels iterate the doubled operator 2U with additions only
// (after t on-chip steps the state is 2^t psi_t exactly), scaling by 2^-T when
// they store.  Identical bits to numpy for every non-zero result; an exact
// zero may come out as -0.0 instead of +0.0 or vice versa (equal under ==,
// np.array_equal and every reduction).
//
// The products are exact unless a halving rounds in the subnormal range.  If
// every non-zero input component of a tile has |x| >= 2^-1016 (exponent field
// >= 7), all values are multiples of 2^(-1068-t) at level t (a sum of
// multiples of a power of two rounds to a multiple of it), so the halvings of
// levels t < 6 land on multiples of 2^-1074, i.e. are exact, and the doubled
// sums are numpy's bit for bit for any depth T <= 6.  A tile
// holding a smaller non-zero value (a localized start's light-cone front after
// ~1000 steps: |psi| = 2^-t) runs in EXACT mode instead: each step halves its
// inputs first (fl(0.5 s_i), numpy's products) and sums them in numpy's
// order, i.e. the numpy arithmetic itself, with a store scale of 1.
__device__ __forceinline__ double2 csub(double2 a, double2 b) {
  return make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y));
}
__device__ __forceinline__ double2 halve(double2 v) {
  return make_double2(__dmul_rn(v.x, 0.5), __dmul_rn(v.y, 0.5));
}

// min-accumulator of the tiny test: key(x) - 1 (unsigned) is below
// kTinyKey iff 0 < |x| < 2^-1016.  key = |x|'s high word with bit 0 set when
// the low word is non-zero (so key == 0 iff x == 0; bit 0 does not move the
// comparison with 7 << 20).
constexpr unsigned kTinyKey = (7u << 20) - 1u;
// Periodic form: a launch that finds no non-zero |x| < 2^-926 (exponent
// field >= 97) guarantees exact doubled-space steps for the next 96 steps
// (multiples of 2^(-978-t) at step t stay on the 2^-1074 grid for t < 96):
// 16 launches of T <= 6 steps until the next such check.
constexpr unsigned kTinyKeyPeriodic = (97u << 20) - 1u;
constexpr int kCheckEvery = 16;
__device__ __forceinline__ unsigned tiny_acc(unsigned m, double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  const unsigned hi = (unsigned)(b >> 32), lo = (unsigned)b;
  const unsigned key = (hi & 0x7fffffffu) | min(lo, 1u);
  return min(m, key - 1u);
}
__device__ __forceinline__ unsigned tiny_acc2(unsigned m, double2 v) { return tiny_acc(tiny_acc(m, v.x), v.y); }

__device__ __forceinline__ void vertex_outputs2_interior(double2 vD, double2 vL, double2 vR, double2 vU,
                                                         double2& oD, double2& oL, double2& oR,
                                                         double2& oU) {
  const double2 t = cadd(vL, vR);     // L + R
  const double2 w = csub(vR, vL);     // -L + R
  oD = csub(cadd(t, vU), vD);         // -D + ((L + R) + U)
  oL = cadd(vD, cadd(w, vU));         //  D + ((-L + R) + U)
  oR = cadd(vD, csub(vU, w));         //  D + ((L - R) + U)
  oU = cadd(vD, csub(t, vU));         //  D + ((L + R) - U)
}

// One vertex, doubled space (exact == false) or numpy's own per-step
// arithmetic (exact == true).  The slot order matters only on
// the rows y = 0 and y = ny - 1: on x = 0 / nx - 1 with interior y the order
// is D R L U, and swapping the two middle slots leaves every row sum
// p0 + ((p1 + p2) + p3) bitwise unchanged (IEEE addition commutes), so those
// vertices take the interior formula; a warp (one region row) branches
// uniformly.
__device__ __forceinline__ void vertex_outputs2(int gx, int gy, int nx, int ny, bool marked, bool exact,
                                                double2 vD, double2 vL, double2 vR, double2 vU, double2& oD,
                                                double2& oL, double2& oR, double2& oU) {
  if (marked) {   // numpy: -psi (exact); doubled space: 2 * (-psi)
    if (exact) {
      oD = make_double2(-vD.x, -vD.y);
      oL = make_double2(-vL.x, -vL.y);
      oR = make_double2(-vR.x, -vR.y);
      oU = make_double2(-vU.x, -vU.y);
    } else {
      oD = make_double2(-__dadd_rn(vD.x, vD.x), -__dadd_rn(vD.y, vD.y));
      oL = make_double2(-__dadd_rn(vL.x, vL.x), -__dadd_rn(vL.y, vL.y));
      oR = make_double2(-__dadd_rn(vR.x, vR.x), -__dadd_rn(vR.y, vR.y));
      oU = make_double2(-__dadd_rn(vU.x, vU.x), -__dadd_rn(vU.y, vU.y));
    }
    return;
  }
  if (exact) {
    vD = halve(vD);
    vL = halve(vL);
    vR = halve(vR);
    vU = halve(vU);
  }
  if ((gy > 0) & (gy < ny - 1)) {
    vertex_outputs2_interior(vD, vL, vR, vU, oD, oL, oR, oU);
    return;
  }
  const Slots o = order_slots(gx, gy, nx, ny, vD, vL, vR, vU);
  const double2 t12 = cadd(o.s1, o.s2);
  const double2 d21 = csub(o.s2, o.s1);
  const double2 O0 = csub(cadd(t12, o.s3), o.s0);
  const double2 O1 = cadd(o.s0, cadd(d21, o.s3));
  const double2 O2 = cadd(o.s0, csub(o.s3, d21));
  const double2 O3 = cadd(o.s0, csub(t12, o.s3));
  oD = pick(o.pD, O0, O1, O2, O3);
  oL = pick(o.pL, O0, O1, O2, O3);
  oR = pick(o.pR, O0, O1, O2, O3);
  oU = pick(o.pU, O0, O1, O2, O3);
}

void lattice_launch(int shift, cudaStream_t s, const Geom& g, const Rows& r, const double2* in,
                    double2* out, const uint32_t* bits, double* prob, int prob_row0,
                    const TraceArgs& tr);
int lattice_check_shift(qwb_ctx* ctx, int shift);
// temporally blocked torus steps (lattice_tb.cu).  TbGeo: the rows a launch
// owns inside a planes buffer of lrows rows (plane stride nx * lrows): local
// rows [own0, own0 + nown) = global rows [ybase, ybase + nown).  wrap = 1:
// the buffer is the whole torus (rows wrap inside it); wrap = 0: a slab with
// >= T ghost rows each side holding the neighbours' state (no wrap).
constexpr int kSlabDepth = 6;   // the slab (ghost-row) tile kernels are built for this depth
struct TbGeo {
  int lrows, own0, nown, ybase, wrap;
};
int lattice_tb_depth(int64_t nx, int64_t ny, int64_t n_marked);
int lattice_tb_owned_rows(int depth);   // owned rows per tile row of the tile kernel (0: n/a)
int lattice_slab_depth(int depth);      // ghost-row depth usable by slab runs (0: none)
// tiles [tile0, tile1) of the launch's tile grid (tile1 = 0: all tiles), on
// at most grid_cap SMs (0: all).  Subnormal guard: without a run flag every
// tile tests its input; with one (sticky), `check` launches test against the
// periodic threshold and the others follow the flag.
int lattice_tb_launch_geo(qwb_ctx* ctx, int depth, int shift, cudaStream_t s, int nx, int ny, const TbGeo& geo,
                          const double2* in, double2* out, const uint32_t* bits, const int64_t* marked_host,
                          int64_t n_marked, int tile0, int tile1, int grid_cap = 0, int check = 1,
                          int* sticky = nullptr);
// the tile grid of a launch over nown owned rows (row-major tiles); returns
// the owned rows per tile row
int lattice_tb_tiles(int depth, int nx, int nown, int* tiles_x, int* tiles_y);
// persistent dataflow run of nblocks x 4 steps on the torus (lattice_tb.cu):
// the number of blocks it would take for `steps` (0: not available)
int lattice_flow_blocks(int64_t nx, int64_t ny, int depth, bool traced, int64_t steps, int num_sms);
int lattice_flow_launch(qwb_ctx* ctx, int shift, cudaStream_t s, int nx, int ny, double2* a, double2* b,
                        const uint32_t* bits, const int64_t* marked_host, int64_t n_marked, int nblocks);
// check: 1 = test every tile's input for tiny amplitudes (threshold
// kTinyKeyPeriodic), redo such tiles exactly and raise *sticky; 0 = no test:
// all tiles exact if *sticky is raised, else doubled space.  A run checks its
// first launch and every kCheckEvery-th (qwb_lattice_run).
int lattice_tb_launch(qwb_ctx* ctx, int depth, int shift, cudaStream_t s, int nx, int ny,
                      const double2* in, double2* out, const uint32_t* bits,
                      const int64_t* marked_host, int64_t n_marked,
                      const int64_t* trace_vertices_host, int n_trace, double* trace, int check, int* sticky);
// the context's sticky flag (device int, allocated on first use)
int lattice_sticky(qwb_ctx* ctx, int** out);
int lattice_slab_geom(qwb_ctx* ctx, int64_t nx, int64_t ny, int64_t y0, int64_t ny_local, Geom* g);
int lattice_slab_geom_g(qwb_ctx* ctx, int64_t nx, int64_t ny, int64_t y0, int64_t ny_local, int64_t ghost,
                        Geom* g);
// part: 0 = all owned rows, 1 = first and last owned rows, 2 = interior owned rows
Rows slab_rows(int64_t ny_local, int part);

}  // namespace qwb
