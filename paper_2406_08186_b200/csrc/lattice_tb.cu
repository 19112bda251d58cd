// lattice_tb.cu — temporally blocked torus walk: T coined steps per HBM pass.
//
// The single-step kernel (lattice.cu) already moves exactly the 32 B per arc
// per step that one application of U needs, at ~96 % of the measured HBM copy
// bandwidth.  The only way past that roofline is to apply U several times per
// trip through HBM.  Each CTA owns a region of 32 x (BY*V) vertices; a thread
// owns V vertically adjacent vertices with their 4 direction amplitudes in
// registers:
//
//   * the region's state arrives in shared memory one tile ahead of its use,
//     so HBM reads overlap the arithmetic of the current tile: regions inside
//     the buffer with ONE tensor TMA (box [4 planes][BY*V rows][32]
//     complex128, completing on the stage's mbarrier), regions that wrap
//     around the torus with per-thread 16-B cp.async;
//   * T steps run on chip, in doubled space (qwb_lattice.cuh "doubled-space
//     forms": the operator 2U needs additions only — 20 FP64 adds per vertex
//     and step — and the state is scaled by 2^-T on the way out, so the result
//     has numpy's bits).  A tile whose input holds a non-zero amplitude below
//     2^-1016 (checked on the loaded registers) runs the same steps in EXACT
//     mode (numpy's halving first), which keeps the bits in the subnormal
//     range too.  Pushes to x +- 1 go through warp shuffles (a warp is one
//     region row of 32 columns), pushes between a thread's own V rows stay in
//     registers, and only the pushes across thread rows go through a
//     double-buffered shared-memory exchange (one barrier per step);
//   * values near the region edge go stale one ring per step, so after T steps
//     the inner (32 - 2T) x (BY*V - 2T) vertices are exact and are written.
//
// Two launch forms:
//   * lattice_tb_kernel — one launch per T steps over all tiles (persistent
//     CTAs, static tile order).  Used for traced search runs (the light-cone
//     trace kernel reads each launch's input) and for multi-GPU y-slabs with
//     ghost state rows (SLAB, TbGeo: owned rows only, no y-wrap; comm.cu).
//   * lattice_flow_kernel — ONE launch for a whole run of K x T steps on the
//     torus.  Work items (block k, tile) are taken in order from a global
//     counter; an item waits until the tiles whose owned cells its region
//     reads have finished block k - 1 (per-tile progress counters,
//     release / acquire), so block k + 1 starts on a tile while other tiles
//     still finish block k.  No launch gap, no pipeline refill and no tail per
//     T steps; the tile-row order rotates by half the torus every block so an
//     item's dependencies are ~half a block old.  Items depend only on earlier
//     items, so the schedule cannot deadlock whatever the CTA residency.
//
// Regions wrap around the torus (modular global coordinates): any nx, ny >= 3.
// Default tile: 16 warps x 4 rows (32 x 64 region), T = 4.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <string.h>

#include <cmath>

#include "qwb_lattice.cuh"

namespace {

using qwb::TbGeo;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void tb_mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void tb_mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tb_mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "TB_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra TB_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// progress counters of the flow kernel
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// after observing the counters with relaxed loads: acquire, then order the
// async proxy (TMA / bulk copies) after it
__device__ __forceinline__ void acquire_for_async() {
  asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
}

#ifdef QWB_EXP_TIMING
__device__ unsigned long long g_dbg[2][8];   // [kernel: 0 tile, 1 flow][slot]
// launch timeline (tools/r02_timeline.py): per launch and CTA, globaltimer at
// entry, after the grid-dependency wait, when the first tile's stage is ready,
// at exit
__device__ unsigned long long g_tl[64][160][4];
__device__ unsigned int g_ctas;
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long dbg_clock() { return clock64(); }
#define DBG_T(var) const unsigned long long var = dbg_clock()
#define DBG_ADD(k, slot, v) atomicAdd(&g_dbg[k][slot], (unsigned long long)(v))
#else
#define DBG_T(var)
#define DBG_ADD(k, slot, v)
#endif

__device__ __forceinline__ int wrapc(int v, int n) {
  v = v < 0 ? v + n : v;
  return v >= n ? v - n : v;
}

__device__ __forceinline__ double2 shfl_down2(double2 v) {
  return make_double2(__shfl_down_sync(0xffffffffu, v.x, 1), __shfl_down_sync(0xffffffffu, v.y, 1));
}
__device__ __forceinline__ double2 shfl_up2(double2 v) {
  return make_double2(__shfl_up_sync(0xffffffffu, v.x, 1), __shfl_up_sync(0xffffffffu, v.y, 1));
}

using qwb::kSlabDepth;

template <int BY, int V>
struct TbShape {
  static constexpr int RX = 32;            // region columns (= warp lanes)
  static constexpr int RY = BY * V;        // region rows
  static constexpr int NT = 32 * BY;       // threads
  static constexpr int REG = RX * RY;      // region vertices
  // stages of the next tiles' amplitudes: two (loads of two tiles in flight)
  // when they fit next to the exchange buffers, else one
  static constexpr int NSTAGE = ((8 * (size_t)REG + 4 * (size_t)NT) * sizeof(double2) + 64 <= 232448) ? 2 : 1;
  static constexpr size_t smem_bytes() {   // stages + exchange + two mbarriers + scheduling words
    return (4 * (size_t)REG * NSTAGE + 4 * (size_t)NT) * sizeof(double2) + 2 * sizeof(uint64_t) + kSchedBytes;
  }
  // flow kernel: 2 item words + 32 dependency pointers and block counts
  static constexpr size_t kSchedBytes = 16 + 32 * sizeof(void*) + 32 * sizeof(unsigned);
};

// p(v) per step for up to 8 traced vertices (search runs): out[t * n + k];
// x, y: the vertices' coordinates (host-computed, no division on the device)
struct TraceList {
  int n;
  int64_t v[8];
  int x[8], y[8];
  double* out;
};

struct MarkedList {   // up to 8 marked vertex ids; n < 0: more than 8 (use the bitmap)
  int n;
  int64_t v[8];
  int x[8], y[8];     // their coordinates (host-computed)
};

// Marked vertex `lane` of the list in registers (lanes 0..7; static indices:
// the list stays in the parameter space), so a tile's "does my region hold a
// marked vertex" test is one check per lane and a warp vote.
struct MarkLane {
  int x, y;
};
__device__ __forceinline__ MarkLane mark_lane(const MarkedList& mk, int lane) {
  MarkLane ml{-1, -1};
#pragma unroll
  for (int j = 0; j < 8; ++j)
    if (lane == j) ml = MarkLane{mk.x[j], mk.y[j]};
  return ml;
}

// p of a traced vertex from its level-t amplitudes a[0..3] (planes D, L, R,
// U; sc undoes the doubled-space scale): reference slot order, numpy |z|^2,
// row sum.
__device__ __forceinline__ double trace_p(int gx, int gy, int nx, int ny, double sc, const double2* a) {
  const auto un = [&](double2 z) { return make_double2(__dmul_rn(z.x, sc), __dmul_rn(z.y, sc)); };
  const qwb::Slots o = qwb::order_slots(gx, gy, nx, ny, un(a[0]), un(a[1]), un(a[2]), un(a[3]));
  const double m0 = qwb::abs2_np(o.s0), m1 = qwb::abs2_np(o.s1), m2 = qwb::abs2_np(o.s2), m3 = qwb::abs2_np(o.s3);
  return __dadd_rn(m0, __dadd_rn(__dadd_rn(m1, m2), m3));
}

// Light-cone trace.  The traced vertex's amplitudes at levels 0..T-1 of a
// T-step launch depend only on the (2T+1)^2 input vertices around it, so one
// CTA per traced vertex recomputes that patch with the tile kernel's own
// arithmetic (vertex_outputs2, the same pushes; exact mode when the patch
// holds a non-zero amplitude below 2^-1016) and writes p per level: numpy's
// values, at a few microseconds instead of a whole 32x64 tile.  Reads the
// launch's input, writes the trace only.  Patch vertices whose neighbours
// fall outside the patch go stale one ring per step; the centre stays exact
// for T steps.
template <int SHIFT, int T>
__global__ void __launch_bounds__(256)
lattice_trace_cone_kernel(int nx, int ny, const double2* __restrict__ in, const uint32_t* __restrict__ bits,
                          TraceList tr) {
  constexpr int P = 2 * T + 1;
  static_assert(P * P <= 256, "patch larger than the CTA");
  __shared__ double2 o[4][P * P];
  qwb::pdl_enter();
  const int k = blockIdx.x;
  if (k >= tr.n) return;
  const int i = threadIdx.x;
  const bool act = i < P * P;
  const int px = i % P, py = i / P;
  int cx = 0, cy = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j)   // static indices: tr stays in the param space
    if (j == k) {
      cx = tr.x[j];
      cy = tr.y[j];
    }
  const int gx = wrapc(cx - T + px, nx), gy = wrapc(cy - T + py, ny);
  const int64_t n = (int64_t)nx * ny, w = (int64_t)gy * nx + gx;
  double2 v[4] = {};
  bool mk = false;
  unsigned m = ~0u;
  if (act) {
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      v[p] = in[p * n + w];
      m = qwb::tiny_acc2(m, v[p]);
    }
    if (bits) mk = (__ldg(bits + (w >> 5)) >> (w & 31)) & 1u;
  }
  const bool exact = __syncthreads_or(m < qwb::kTinyKey);
  const bool centre = act && px == T && py == T;
#pragma unroll 1
  for (int t = 0; t < T; ++t) {
    if (centre) tr.out[t * tr.n + k] = trace_p(gx, gy, nx, ny, exact ? 1.0 : 1.0 / (double)(1 << t), v);
    if (act)
      qwb::vertex_outputs2(gx, gy, nx, ny, mk, exact, v[0], v[1], v[2], v[3], o[0][i], o[1][i], o[2][i], o[3][i]);
    __syncthreads();
    if (act) {
      const double2 fromRight = o[1][px + 1 < P ? i + 1 : i];   // O_L of (x+1, y)
      const double2 fromLeft = o[2][px > 0 ? i - 1 : i];        // O_R of (x-1, y)
      const double2 fromAbove = o[0][py + 1 < P ? i + P : i];   // O_D of (x, y+1)
      const double2 fromBelow = o[3][py > 0 ? i - P : i];       // O_U of (x, y-1)
      if (SHIFT == QWB_SHIFT_FLIPFLOP) {
        v[3] = fromAbove; v[0] = fromBelow; v[2] = fromRight; v[1] = fromLeft;
      } else {
        v[0] = fromAbove; v[3] = fromBelow; v[1] = fromRight; v[2] = fromLeft;
      }
    }
    __syncthreads();
  }
}

// T steps of a tile on chip (see the file comment).  INTERIOR: no row of the
// region is a torus edge row (y = 0, ny - 1) and no marked vertex lies in it:
// one formula for every vertex (x-edge vertices included, qwb_lattice.cuh),
// no per-vertex branch.  exact: numpy's per-step arithmetic (tiny inputs).
//
// The first step's barrier also ORs the threads' tiny-input flags (m, from
// stage_to_regs): the result says whether the doubled-space attempt is
// numpy's (false) or must be redone in EXACT mode (true; tile_run).
// after0() runs right after the first step's barrier (the flow kernel issues
// a wrapping next region's copies there).
struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};
template <int SHIFT, bool MARKED, int T, int BY, int V, bool INTERIOR, bool EXACT, class F>
__device__ __forceinline__ bool tile_steps(int nx, int ny, int gx, const int (&gy)[V], unsigned m, unsigned key,
                                           const uint32_t* __restrict__ bits, double2 (&vD)[V],
                                           double2 (&vL)[V], double2 (&vR)[V], double2 (&vU)[V],
                                           double2* xD, double2* xU, int tid, int ty, const F& after0) {
  bool tiny = false;
  bool mk[V];
#pragma unroll
  for (int j = 0; j < V; ++j) {
    mk[j] = false;
    if (MARKED && !INTERIOR) {
      const int64_t wg = (int64_t)gy[j] * nx + gx;
      mk[j] = (__ldg(bits + (wg >> 5)) >> (wg & 31)) & 1u;
    }
  }
#pragma unroll
  for (int t = 0; t < T; ++t) {
    double2 oD[V], oL[V], oR[V], oU[V];
#pragma unroll
    for (int j = 0; j < V; ++j) {
      if (INTERIOR) {
        if (EXACT) {
          vD[j] = qwb::halve(vD[j]);
          vL[j] = qwb::halve(vL[j]);
          vR[j] = qwb::halve(vR[j]);
          vU[j] = qwb::halve(vU[j]);
        }
        qwb::vertex_outputs2_interior(vD[j], vL[j], vR[j], vU[j], oD[j], oL[j], oR[j], oU[j]);
      } else {
        qwb::vertex_outputs2(gx, gy[j], nx, ny, mk[j], EXACT, vD[j], vL[j], vR[j], vU[j], oD[j], oL[j], oR[j],
                             oU[j]);
      }
    }
    const int b = (t & 1) * 32 * BY;
    xD[b + tid] = oD[0];
    xU[b + tid] = oU[V - 1];
    double2 fromRight[V], fromLeft[V];
#pragma unroll
    for (int j = 0; j < V; ++j) {
      fromRight[j] = shfl_down2(oL[j]);   // O_L of (x+1, y)
      fromLeft[j] = shfl_up2(oR[j]);      // O_R of (x-1, y)
    }
    if (!EXACT && t == 0)
      tiny = __syncthreads_or(m < key);
    else
      __syncthreads();
    if (t == 0) after0();
    double2 fromAbove[V], fromBelow[V];   // O_D of (x, y+1), O_U of (x, y-1)
#pragma unroll
    for (int j = 0; j < V - 1; ++j) fromAbove[j] = oD[j + 1];
    fromAbove[V - 1] = (ty < BY - 1) ? xD[b + tid + 32] : oD[V - 1];
#pragma unroll
    for (int j = 1; j < V; ++j) fromBelow[j] = oU[j - 1];
    fromBelow[0] = (ty > 0) ? xU[b + tid - 32] : oU[0];
#pragma unroll
    for (int j = 0; j < V; ++j) {
      if (SHIFT == QWB_SHIFT_FLIPFLOP) {
        vU[j] = fromAbove[j]; vD[j] = fromBelow[j]; vR[j] = fromRight[j]; vL[j] = fromLeft[j];
      } else {
        vD[j] = fromAbove[j]; vU[j] = fromBelow[j]; vL[j] = fromRight[j]; vR[j] = fromLeft[j];
      }
    }
  }
  return tiny;
}

// Region loads.  A region inside the buffer arrives with ONE tensor TMA
// issued by thread 0, completing on the stage's mbarrier; a region that wraps
// around the torus (or reaches past a slab buffer) with per-thread 16-B
// cp.async (all threads; rows outside a slab buffer are skipped: they are
// > T rows from every owned row, left stale), completing on the threads'
// cp.async group.  bx: global column of region column 0 (< 0 or past nx:
// wrap); by: local buffer row of region row 0.
template <class S>
__device__ __forceinline__ bool region_inside(int nx, int lrows, int bx, int by, bool use_tma) {
  return use_tma && bx >= 0 && bx + S::RX <= nx && by >= 0 && by + S::RY <= lrows;
}
template <class S>
__device__ __forceinline__ void tma_region(double2* stage, uint64_t* bar, const CUtensorMap* map, int bx, int by) {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // earlier LDS of this stage
  tb_mbar_expect_tx(bar, 4u * S::REG * (uint32_t)sizeof(double2));
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];\n" ::"r"(smem_u32(stage)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(2 * bx), "r"(by), "r"(0), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

template <class S, int V, bool SLAB>
__device__ __forceinline__ void cp_region(double2* stage, const double2* in, int nx, int ny, int lrows, int bx,
                                          int by, int tx, int ty) {
  const int64_t n = (int64_t)nx * lrows;   // plane stride
  const int gx = wrapc(bx + tx, nx);
#pragma unroll
  for (int j = 0; j < V; ++j) {
    const int ly = by + ty * V + j;
    if (SLAB && (ly < 0 || ly >= lrows)) continue;
    const int r = SLAB ? ly : wrapc(ly, ny);
    const int64_t w = (int64_t)r * nx + gx;
    const int li = (ty * V + j) * 32 + tx;
#pragma unroll
    for (int p = 0; p < 4; ++p) cp_async16(stage + p * S::REG + li, in + p * n + w);
  }
}

// Registers of a tile from its stage, with the tiny-amplitude test.
template <class S, int V>
__device__ __forceinline__ unsigned stage_to_regs(const double2* stage, int tx, int ty, double2 (&vD)[V],
                                                  double2 (&vL)[V], double2 (&vR)[V], double2 (&vU)[V],
                                                  bool check = true) {
  unsigned m = ~0u;
#pragma unroll
  for (int j = 0; j < V; ++j) {
    const int li = (ty * V + j) * 32 + tx;
    vD[j] = stage[li];
    vL[j] = stage[S::REG + li];
    vR[j] = stage[2 * S::REG + li];
    vU[j] = stage[3 * S::REG + li];
    if (!check) continue;
    m = qwb::tiny_acc2(m, vD[j]);
    m = qwb::tiny_acc2(m, vL[j]);
    m = qwb::tiny_acc2(m, vR[j]);
    m = qwb::tiny_acc2(m, vU[j]);
  }
  return m;
}

// The tile's T steps in numpy's own arithmetic (halve, then sum: the
// reference's bits in the subnormal range too), its region loaded from `in`
// (intact while the tile runs: a launch writes the other buffer, and a flow
// item's input region is not overwritten before the item is done), owned
// block stored.  Out of line: the rare path stays out of the hot kernel body
// (instruction-cache footprint).
template <int SHIFT, bool MARKED, int T, int BY, int V, bool SLAB>
__device__ __noinline__ void tile_exact(int nx, int ny, int64_t n, int lrows, int x0, int y0, int lyb, int rows_left,
                                        bool interior, const double2* __restrict__ in,
                                        const uint32_t* __restrict__ bits, double2* xD, double2* xU,
                                        double2* __restrict__ out) {
  using S = TbShape<BY, V>;
  constexpr int OX = S::RX - 2 * T, OY = S::RY - 2 * T;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
  const int gx = wrapc(x0 - T + tx, nx);
  int gy[V];
  double2 vD[V], vL[V], vR[V], vU[V];
#pragma unroll
  for (int j = 0; j < V; ++j) {
    gy[j] = wrapc(y0 - T + ty * V + j, ny);
    const int ly = lyb - T + ty * V + j;   // local buffer row
    const bool ok = !SLAB || (ly >= 0 && ly < lrows);
    const int64_t w = (int64_t)(SLAB ? (ok ? ly : 0) : wrapc(ly, ny)) * nx + gx;
    const double2 z = make_double2(0.0, 0.0);
    // L2 loads (.cg): in the persistent kernel an L1 line of this buffer can
    // be two blocks old; the region's current values were published to L2
    // before the item's dependencies were acquired
    vD[j] = ok ? __ldcg(in + w) : z;
    vL[j] = ok ? __ldcg(in + n + w) : z;
    vR[j] = ok ? __ldcg(in + 2 * n + w) : z;
    vU[j] = ok ? __ldcg(in + 3 * n + w) : z;
  }
  if (interior)
    tile_steps<SHIFT, false, T, BY, V, true, true>(nx, ny, gx, gy, 0u, 0u, bits, vD, vL, vR, vU, xD, xU, tid, ty,
                                                   NoHook{});
  else
    tile_steps<SHIFT, MARKED, T, BY, V, false, true>(nx, ny, gx, gy, 0u, 0u, bits, vD, vL, vR, vU, xD, xU, tid, ty,
                                                     NoHook{});
  const bool col_ok = tx >= T && tx < T + OX && x0 + tx - T < nx;
#pragma unroll
  for (int j = 0; j < V; ++j) {
    const int ly = ty * V + j;
    if (col_ok && ly >= T && ly < T + OY && ly - T < rows_left) {
      const int64_t w = (int64_t)(lyb - T + ly) * nx + gx;
      __stcs(out + w, vD[j]);
      __stcs(out + n + w, vL[j]);
      __stcs(out + 2 * n + w, vR[j]);
      __stcs(out + 3 * n + w, vU[j]);
    }
  }
}

// A tile whose region holds a marked vertex (rare: a few tiles per launch),
// doubled space, region reloaded from `in` (L2 loads, as tile_exact).  Out of
// line: inlined, the marked slot path changed the code of the whole MARKED
// kernel and every interior tile ran 6.5 % slower (4096^2: 94.5 vs 88.8
// us/step, profiles/r02_marked_variant.txt).  m: the threads' tiny-input flags
// from the stage, tested against key on the first step's barrier.
template <int SHIFT, int T, int BY, int V, bool SLAB>
__device__ __noinline__ bool tile_marked(int nx, int ny, int64_t n, int lrows, int x0, int y0, int lyb,
                                         int rows_left, unsigned m, unsigned key, const double2* __restrict__ in,
                                         const uint32_t* __restrict__ bits, double2* xD, double2* xU,
                                         double2* __restrict__ out, int* sticky) {
  using S = TbShape<BY, V>;
  constexpr int OX = S::RX - 2 * T, OY = S::RY - 2 * T;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
  const int gx = wrapc(x0 - T + tx, nx);
  int gy[V];
  double2 vD[V], vL[V], vR[V], vU[V];
#pragma unroll
  for (int j = 0; j < V; ++j) {
    gy[j] = wrapc(y0 - T + ty * V + j, ny);
    const int ly = lyb - T + ty * V + j;
    const bool ok = !SLAB || (ly >= 0 && ly < lrows);
    const int64_t w = (int64_t)(SLAB ? (ok ? ly : 0) : wrapc(ly, ny)) * nx + gx;
    const double2 z = make_double2(0.0, 0.0);
    vD[j] = ok ? __ldcg(in + w) : z;
    vL[j] = ok ? __ldcg(in + n + w) : z;
    vR[j] = ok ? __ldcg(in + 2 * n + w) : z;
    vU[j] = ok ? __ldcg(in + 3 * n + w) : z;
  }
  const bool tiny = tile_steps<SHIFT, true, T, BY, V, false, false>(nx, ny, gx, gy, m, key, bits, vD, vL, vR, vU,
                                                                   xD, xU, tid, ty, NoHook{});
  if (tiny) {
    if (sticky && tid == 0) atomicOr(sticky, 1);
    tile_exact<SHIFT, true, T, BY, V, SLAB>(nx, ny, n, lrows, x0, y0, lyb, rows_left, false, in, bits, xD, xU, out);
    return true;
  }
  constexpr double sc = 1.0 / (double)(1 << T);
  const bool col_ok = tx >= T && tx < T + OX && x0 + tx - T < nx;
#pragma unroll
  for (int j = 0; j < V; ++j) {
    const int ly = ty * V + j;
    if (col_ok && ly >= T && ly < T + OY && ly - T < rows_left) {
      const int64_t w = (int64_t)(lyb - T + ly) * nx + gx;
      __stcs(out + w, make_double2(__dmul_rn(vD[j].x, sc), __dmul_rn(vD[j].y, sc)));
      __stcs(out + n + w, make_double2(__dmul_rn(vL[j].x, sc), __dmul_rn(vL[j].y, sc)));
      __stcs(out + 2 * n + w, make_double2(__dmul_rn(vR[j].x, sc), __dmul_rn(vR[j].y, sc)));
      __stcs(out + 3 * n + w, make_double2(__dmul_rn(vU[j].x, sc), __dmul_rn(vU[j].y, sc)));
    }
  }
  return false;
}

// Steps + store of one tile whose registers are loaded.  (x0, y0): global
// column / unwrapped global row of its first owned vertex; lyb: local buffer
// row of that row; rows_left: owned rows from y0 to the end of the launch's
// owned range; m: the threads' tiny-input flags (stage_to_regs), tested
// against `key` (0: no test).  The steps run in doubled space; if any input
// amplitude of the region is tiny (rare: the front of a localized start after
// ~1000 steps) the tile is redone in numpy's arithmetic (tile_exact), as it is
// from the start when all_exact.  The test is off the critical path: its
// integer work interleaves with the first step, its reduction rides on that
// step's barrier.  Returns whether numpy's arithmetic was used.
template <int SHIFT, bool MARKED, int T, int BY, int V, bool SLAB, class F>
__device__ __forceinline__ bool tile_run(int nx, int ny, int64_t n, int lrows, int x0, int y0, int lyb,
                                         int rows_left, unsigned m, unsigned key, bool all_exact,
                                         const double2* __restrict__ in,
                                         const uint32_t* __restrict__ bits, const MarkedList& mk,
                                         double2 (&vD)[V], double2 (&vL)[V], double2 (&vR)[V], double2 (&vU)[V],
                                         double2* xD, double2* xU, double2* __restrict__ out, int tx, int ty,
                                         int tid, const F& after0, int* sticky = nullptr,
                                         MarkLane ml = MarkLane{-1, -1}) {
  using S = TbShape<BY, V>;
  constexpr int OX = S::RX - 2 * T, OY = S::RY - 2 * T;
  const int gx = wrapc(x0 - T + tx, nx);
  int gy[V];
#pragma unroll
  for (int j = 0; j < V; ++j) gy[j] = wrapc(y0 - T + ty * V + j, ny);
  // regions with no torus edge row and no marked vertex: one formula
  bool interior = y0 - T >= 1 && y0 - T + S::RY - 1 <= ny - 2;
  bool has_marked = false;   // the region holds a marked vertex: out-of-line path
  if (MARKED) {
    // lane k tests marked vertex k: offsets from the region's first column /
    // row modulo the torus (arguments within one period of [0, n): x0 in
    // [0, nx), y0 - T within a slab's ghost rows of [0, ny))
    const int dx = wrapc(ml.x - (x0 - T), nx), dy = wrapc(ml.y - (y0 - T), ny);
    has_marked = mk.n < 0 || __any_sync(0xffffffffu, tx < mk.n && dx < S::RX && dy < S::RY);
    interior &= !has_marked;
  }
  if (all_exact) {   // a run that met tiny amplitudes: numpy's arithmetic from the start
    __syncthreads();   // after0 reads what the flow kernel's polling warp decided just before
    after0();
    tile_exact<SHIFT, MARKED, T, BY, V, SLAB>(nx, ny, n, lrows, x0, y0, lyb, rows_left, interior, in, bits, xD, xU,
                                              out);
    return true;
  }
  if (MARKED && has_marked) {
    __syncthreads();   // as above
    after0();
    return tile_marked<SHIFT, T, BY, V, SLAB>(nx, ny, n, lrows, x0, y0, lyb, rows_left, m, key, in, bits, xD, xU,
                                              out, sticky);
  }
  const bool tiny =
      interior ? tile_steps<SHIFT, false, T, BY, V, true, false>(nx, ny, gx, gy, m, key, bits, vD, vL, vR, vU, xD,
                                                                 xU, tid, ty, after0)
               : tile_steps<SHIFT, false, T, BY, V, false, false>(nx, ny, gx, gy, m, key, bits, vD, vL, vR, vU, xD,
                                                                  xU, tid, ty, after0);
  if (tiny) {
    if (sticky && tid == 0) atomicOr(sticky, 1);
    tile_exact<SHIFT, MARKED, T, BY, V, SLAB>(nx, ny, n, lrows, x0, y0, lyb, rows_left, interior, in, bits, xD, xU,
                                              out);
    return true;
  }
  constexpr double sc = 1.0 / (double)(1 << T);   // undo the doubled-space steps (exact)
  const bool col_ok = tx >= T && tx < T + OX && x0 + tx - T < nx;
#pragma unroll
  for (int j = 0; j < V; ++j) {
    const int ly = ty * V + j;
    if (col_ok && ly >= T && ly < T + OY && ly - T < rows_left) {
      const int64_t w = (int64_t)(lyb - T + ly) * nx + gx;
      __stcs(out + w, make_double2(__dmul_rn(vD[j].x, sc), __dmul_rn(vD[j].y, sc)));
      __stcs(out + n + w, make_double2(__dmul_rn(vL[j].x, sc), __dmul_rn(vL[j].y, sc)));
      __stcs(out + 2 * n + w, make_double2(__dmul_rn(vR[j].x, sc), __dmul_rn(vR[j].y, sc)));
      __stcs(out + 3 * n + w, make_double2(__dmul_rn(vU[j].x, sc), __dmul_rn(vU[j].y, sc)));
    }
  }
  return false;
}

// ---------------------------------------------------------------------------
// One launch = T steps over tiles [tile0, ntiles).  SLAB: the buffer is a
// y-slab with ghost rows (geo), else the whole torus.
// ---------------------------------------------------------------------------
template <int SHIFT, bool MARKED, int T, int BY, int V, bool SLAB>
__global__ void __launch_bounds__(32 * BY, 1)
lattice_tb_kernel(int nx, int ny, TbGeo geo, const double2* __restrict__ in, double2* __restrict__ out,
                  const uint32_t* __restrict__ bits, MarkedList mk, int tiles_x, int ntiles, int tile0,
                  const __grid_constant__ CUtensorMap imap, int use_tma, unsigned key, int* sticky) {
#ifdef QWB_EXP_TIMING
  const unsigned long long tl0 = gtime();
#endif
  using S = TbShape<BY, V>;
  constexpr int OX = S::RX - 2 * T, OY = S::RY - 2 * T;   // exact (owned) block
  extern __shared__ __align__(128) double2 sm[];
  double2* stage0 = sm;                        // [NSTAGE][4][RY][RX] next tiles' amplitudes
  double2* xD = sm + 4 * S::REG * S::NSTAGE;   // [2][BY][32] O_D of each thread's lowest row
  double2* xU = xD + 2 * S::NT;                // [2][BY][32] O_U of each thread's highest row
  uint64_t* tbar = reinterpret_cast<uint64_t*>(xU + 2 * S::NT);   // [2] stage barriers
  const int tx = threadIdx.x, ty = threadIdx.y;
  const MarkLane ml = MARKED ? mark_lane(mk, tx) : MarkLane{-1, -1};
  const int tid = ty * 32 + tx;
  if (!SLAB) geo = TbGeo{ny, 0, ny, 0, 1};   // compile-time constants for the torus
  if (tid == 0) {
    tb_mbar_init(tbar, 1);
    tb_mbar_init(tbar + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int64_t n = (int64_t)nx * geo.lrows;   // plane stride of the buffers

  // tile coordinates advance by gridDim.x tiles per iteration: (gdiv, gmod)
  // rows / columns, carried without a division per tile
  const int gdiv = (int)gridDim.x / tiles_x, gmod = (int)gridDim.x % tiles_x;
  auto advance = [&](int& c, int& r) {
    c += gmod;
    r += gdiv;
    if (c >= tiles_x) {
      c -= tiles_x;
      ++r;
    }
  };
  auto inside = [&](int pc, int pr) {
    return region_inside<S>(nx, geo.lrows, pc * OX - T, geo.own0 + pr * OY - T, use_tma != 0);
  };
  // one cp.async group per issue (empty for a TMA stage) keeps the group
  // count per stage uniform
  auto issue = [&](int k, int pc, int pr) {
    double2* st = stage0 + (size_t)k * 4 * S::REG;
    if (inside(pc, pr)) {
      if (tid == 0) tma_region<S>(st, tbar + k, &imap, pc * OX - T, geo.own0 + pr * OY - T);
    } else {
      cp_region<S, V, SLAB>(st, in, nx, ny, geo.lrows, pc * OX - T, geo.own0 + pr * OY - T, tx, ty);
    }
    cp_commit();
  };

  // programmatic dependent launch: everything above overlaps the previous
  // launch's last tiles; its output (this launch's input) is visible after the
  // wait (a no-op when launched without the PDL attribute)
  qwb::pdl_wait();
#ifdef QWB_EXP_TIMING
  const unsigned long long tl1 = gtime();
  unsigned long long tl2 = 0;
  unsigned lid = 0;
  if (threadIdx.x == 0 && threadIdx.y == 0) lid = atomicAdd(&g_ctas, 1u) / gridDim.x;
#endif
  int tile = blockIdx.x + tile0;   // tile0 > 0: a launch over tiles [tile0, ntiles) only
  if (tile >= ntiles) return;
  // key != 0: test the tiles' inputs (and raise *sticky on a hit); key == 0:
  // no test, numpy's arithmetic throughout if an earlier check raised *sticky
  const bool check = key != 0;
  const bool all_exact = !check && sticky && *reinterpret_cast<volatile int*>(sticky) != 0;
  int tcol = tile % tiles_x, trow = tile / tiles_x;
  // (pcol, prow): the tile the next load fetches, NSTAGE - 1 tiles ahead of (tcol, trow)
  int pcol = tcol, prow = trow, ptile = tile;
  for (int k = 0; k < S::NSTAGE; ++k) {
    if (ptile < ntiles)
      issue(k, pcol, prow);
    else
      cp_commit();
    advance(pcol, prow);
    ptile += gridDim.x;
  }
  uint32_t ph = 0;   // bit k: parity of stage k's barrier
  for (int it = 0; tile < ntiles; tile += gridDim.x, ++it) {
    // last tile of this CTA: let the next launch's CTAs take the SMs that
    // finish first (they block in griddepcontrol.wait until this grid is done)
    if (tile + (int)gridDim.x >= ntiles) qwb::pdl_trigger();
    const int k = S::NSTAGE == 2 ? (it & 1) : 0;
    const int trow_now = trow, tcol_now = tcol;
    const int x0 = tcol * OX, y0 = geo.ybase + trow_now * OY, lyb = geo.own0 + trow_now * OY;
    advance(tcol, trow);
    double2 vD[V], vL[V], vR[V], vU[V];
    DBG_T(t_a);
    if (inside(tcol_now, trow_now)) {
      tb_mbar_wait(tbar + k, (ph >> k) & 1u);
      ph ^= 1u << k;
    } else {
      cp_wait<S::NSTAGE - 1>();   // this stage's group; the other stage's may fly
      __syncthreads();
    }
    DBG_T(t_b);
    const unsigned m = stage_to_regs<S, V>(stage0 + (size_t)k * 4 * S::REG, tx, ty, vD, vL, vR, vU, check);
#ifdef QWB_EXP_TIMING
    if (it == 0) tl2 = gtime();
#endif
    __syncthreads();   // stage k consumed
    DBG_T(t_c);
    if (ptile < ntiles)
      issue(k, pcol, prow);
    else
      cp_commit();
    advance(pcol, prow);
    ptile += gridDim.x;
    tile_run<SHIFT, MARKED, T, BY, V, SLAB>(nx, ny, n, geo.lrows, x0, y0, lyb, geo.nown - trow_now * OY, m, key,
                                            all_exact, in, bits, mk, vD, vL, vR, vU, xD, xU, out, tx, ty, tid,
                                            NoHook{}, sticky, ml);
#ifdef QWB_EXP_TIMING
    DBG_T(t_d);
    if (tid == 0) {
      DBG_ADD(0, 0, t_b - t_a);
      DBG_ADD(0, 1, t_c - t_b);
      DBG_ADD(0, 2, t_d - t_c);
      DBG_ADD(0, 3, 1);
    }
    if (tid == 32 * 7) DBG_ADD(0, 4, dbg_clock() - t_c);   // a storing warp
#endif
  }
#ifdef QWB_EXP_TIMING
  if (threadIdx.x == 0 && threadIdx.y == 0 && lid < 64 && blockIdx.x < 160) {
    g_tl[lid][blockIdx.x][0] = tl0;
    g_tl[lid][blockIdx.x][1] = tl1;
    g_tl[lid][blockIdx.x][2] = tl2;
    g_tl[lid][blockIdx.x][3] = gtime();
  }
#endif
}

// ---------------------------------------------------------------------------
// Flow kernel: nblocks x T steps on the torus in one launch (file comment).
//
// Items (block k, tile) are numbered k-major; CTA c takes items c, c + G,
// c + 2G, ... (G = gridDim.x CTAs, co-resident: cooperative launch).  An
// item waits for the progress counters of the 5 x 5 tiles around it (a
// superset of the tiles whose owned cells its region reads: only the last
// tile column / row can be narrower than T) to reach its block; every item
// depends only on items earlier in the numbering, and each CTA runs its
// items in order, so the earliest unfinished item can always proceed.
// ---------------------------------------------------------------------------
struct FlowArgs {
  double2* buf0;      // block k reads buf[k & 1], writes buf[(k + 1) & 1]
  double2* buf1;
  // [ntiles] per tile: blocks completed (bits 0..30) and, bit 31, the
  // subnormal flag of its last block (zeroed before the launch)
  unsigned* done;
  int nblocks;
  int rot;            // tile-row rotation per block
};

// position of a CTA's item in the (block, tile row, tile column) grid,
// advanced by G items without a division
struct FlowPos {
  int k, r, c, rk;    // block, unrotated tile row, tile column, (k * rot) mod tiles_y
};

template <int SHIFT, bool MARKED, int T, int BY, int V>
__global__ void __launch_bounds__(32 * BY, 1)
lattice_flow_kernel(int nx, int ny, FlowArgs fa, const uint32_t* __restrict__ bits, MarkedList mk, int tiles_x,
                    int tiles_y, const __grid_constant__ CUtensorMap imap0, const __grid_constant__ CUtensorMap imap1,
                    int use_tma) {
  using S = TbShape<BY, V>;
  static_assert(S::NSTAGE == 1, "the flow kernel is written for one stage");
  constexpr int OX = S::RX - 2 * T, OY = S::RY - 2 * T;
  extern __shared__ __align__(128) double2 sm[];
  double2* stage = sm;
  double2* xD = sm + 4 * S::REG;
  double2* xU = xD + 2 * S::NT;
  uint64_t* tbar = reinterpret_cast<uint64_t*>(xU + 2 * S::NT);
  // [0]: the next item's load state (0 / 1 TMA / 2 cp.async); [2 + (it & 1)]:
  // iteration it's item inherits the subnormal flag (from its dependencies)
  int* shw = reinterpret_cast<int*>(tbar + 2);
  const int tx = threadIdx.x, ty = threadIdx.y;
  const MarkLane ml = MARKED ? mark_lane(mk, tx) : MarkLane{-1, -1};
  const int tid = ty * 32 + tx;
  const int ntiles = tiles_x * tiles_y;
  const int64_t n = (int64_t)nx * ny;
  const int G = (int)gridDim.x;
  const int gdiv = G / tiles_x, gmod = G % tiles_x;
  auto adv = [&](FlowPos p) -> FlowPos {
    p.c += gmod;
    p.r += gdiv;
    if (p.c >= tiles_x) {
      p.c -= tiles_x;
      ++p.r;
    }
    if (p.r >= tiles_y) {
      p.r -= tiles_y;
      ++p.k;
      p.rk += fa.rot;
      if (p.rk >= tiles_y) p.rk -= tiles_y;
    }
    return p;
  };
  auto trow = [&](const FlowPos& p) { return p.r + p.rk >= tiles_y ? p.r + p.rk - tiles_y : p.r + p.rk; };
  // polling warp, lane i < 25: progress counter of dependency i of the item at p
  // (nullptr: none) and the count it must reach (= the item's block)
  const int ddr = tx / 5 - 2, ddc = tx % 5 - 2;
  auto dep_ptr = [&](const FlowPos& p) -> const unsigned* {
    if (p.k == 0 || p.k >= fa.nblocks || tx >= 25) return nullptr;
    const int rr = wrapc(trow(p) + ddr, tiles_y), cc = wrapc(p.c + ddc, tiles_x);
    return fa.done + rr * tiles_x + cc;
  };
  auto poll = [&](const FlowPos& p) -> unsigned {   // one relaxed read of the lane's dependency
    const unsigned* q = dep_ptr(p);
    return q ? ld_relaxed(q) : 0xffffffffu;
  };

  auto need_of = [&](const FlowPos& p) -> unsigned { return (unsigned)p.k; };
  constexpr unsigned kFlag = 0x80000000u;   // counter bit 31: the tile's block ran numpy's arithmetic
  auto done_ok = [&](unsigned v, unsigned need) { return (v & ~kFlag) >= need; };
  auto inside = [&](const FlowPos& p) {
    return region_inside<S>(nx, ny, p.c * OX - T, trow(p) * OY - T, use_tma != 0);
  };
  auto tma_item = [&](const FlowPos& p) {   // thread 0
    tma_region<S>(stage, tbar, (p.k & 1) ? &imap1 : &imap0, p.c * OX - T, trow(p) * OY - T);
  };
  auto cp_item = [&](const FlowPos& p) {   // all threads
    cp_region<S, V, false>(stage, (p.k & 1) ? fa.buf1 : fa.buf0, nx, ny, ny, p.c * OX - T, trow(p) * OY - T, tx, ty);
    cp_commit();
  };
  // Roles: the last warp (a halo-row warp: it stores nothing) polls the next
  // items' dependencies, acquires them and issues the TMA loads; thread 0
  // (the first, also store-free warp) publishes finished tiles.  Their fences
  // then wait for no outstanding stores or polls of their own.
  const bool pw = ty == BY - 1;       // polling warp
  const bool pw0 = pw && tx == 0;
  // all threads: wait until the item's dependencies are done, then load it
  // Subnormal guard: blocks k % kCheckEvery == 0 test their inputs; a tile
  // that ran numpy's arithmetic publishes bit 31 with its counter, and an item
  // of a later block inherits it from its dependencies (cone by cone), until
  // the next check block (qwb_lattice.cuh).  The polling warp records, with
  // the counters it observed, whether the item inherits the flag.
  auto note_flag = [&](const FlowPos& p, unsigned v, int slot) {
    // lanes without a dependency read 0xffffffff: not a flag
    const unsigned any = __ballot_sync(0xffffffffu, dep_ptr(p) != nullptr && (v & kFlag) != 0u);
    if (pw0) shw[2 + slot] = any != 0u;
  };
  auto blocking_load = [&](const FlowPos& p, int slot) {
    if (pw) {
      unsigned v;
      while (!__all_sync(0xffffffffu, done_ok(v = poll(p), need_of(p)))) __nanosleep(64);
      acquire_for_async();
      note_flag(p, v, slot);
    }
    __syncthreads();   // the other threads' loads are ordered after the polling warp's acquire
    if (inside(p)) {
      if (pw0) tma_item(p);
    } else {
      cp_item(p);
    }
  };
  // publish a finished tile: every thread's stores precede the caller's
  // barrier; thread 0 (no stores of its own) releases
  auto release = [&](int tile, unsigned value) {
    if (tid == 0) {
      asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
      asm volatile("st.relaxed.gpu.global.u32 [%0], %1;\n" ::"l"(fa.done + tile), "r"(value) : "memory");
    }
  };

  if (blockIdx.x >= ntiles) return;
  if (tid == 0) {
    tb_mbar_init(tbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  FlowPos cur{0, (int)blockIdx.x / tiles_x, (int)blockIdx.x % tiles_x, 0};
  blocking_load(cur, 0);
  int it = 0;
  // the polling warp reads the counters of the items one and two ahead in
  // advance, so the prefetch point rarely waits for an L2 round trip
  // the polling warp reads the counters of the next item in advance (at the
  // end of the previous item)
  unsigned v1 = pw ? poll(adv(cur)) : 0u, v2 = 0u;
  uint32_t ph = 0;
  int pend_tile = -1;   // finished tile whose counter is not yet published
  unsigned pend_val = 0;
  while (true) {
    const FlowPos nxt = adv(cur);
    const int tr = trow(cur);
    double2 vD[V], vL[V], vR[V], vU[V];
    DBG_T(t_a);
    if (inside(cur)) {
      tb_mbar_wait(tbar, ph);
      ph ^= 1u;
    } else {
      cp_wait<0>();
      __syncthreads();
    }
    DBG_T(t_b);
    // subnormal guard (qwb_lattice.cuh): blocks k % kCheckEvery == 0 test
    // their inputs, later blocks run exactly once a test in their cone hit
    const bool check = cur.k % qwb::kCheckEvery == 0;
    const unsigned m = stage_to_regs<S, V>(stage, tx, ty, vD, vL, vR, vU, check);
    __syncthreads();   // stage consumed
    DBG_T(t_c);
    const bool all_exact = !check && shw[2 + (it & 1)] != 0;
    const bool more = nxt.k < fa.nblocks;
    // the previous tile's counter: its stores precede the barrier above
    if (pend_tile >= 0) release(pend_tile, pend_val);
    // the next item's load now if its dependencies are done: TMA at once,
    // a wrapping region's cp.async after the first step (shw[0] = 2);
    // otherwise after this tile (shw[0] = 0: it may depend on this tile)
    if (pw && more) {
      unsigned v = v1;
      bool ok = __all_sync(0xffffffffu, done_ok(v, need_of(nxt)));
      if (!ok) ok = __all_sync(0xffffffffu, done_ok(v = poll(nxt), need_of(nxt)));   // one fresh poll
      if (ok) {
        acquire_for_async();
        note_flag(nxt, v, (it + 1) & 1);
      }
      const bool tma = inside(nxt);
      if (ok && tma && pw0) tma_item(nxt);
      if (pw0) shw[0] = ok ? (tma ? 1 : 2) : 0;
#ifdef QWB_EXP_TIMING
      if (pw0) {
        DBG_ADD(1, 5, ok ? 0 : 1);
        DBG_ADD(1, 6, dbg_clock() - t_c);
      }
#endif
    }
    const double2* in = (cur.k & 1) ? fa.buf1 : fa.buf0;
    double2* out = (cur.k & 1) ? fa.buf0 : fa.buf1;
    auto after0 = [&]() {
      if (more && shw[0] == 2) cp_item(nxt);
    };
    const bool exact_used =
        tile_run<SHIFT, MARKED, T, BY, V, false>(nx, ny, n, ny, cur.c * OX, tr * OY, tr * OY, ny - tr * OY, m,
                                                 check ? qwb::kTinyKeyPeriodic : 0u, all_exact, in, bits, mk, vD, vL,
                                                 vR, vU, xD, xU, out, tx, ty, tid, after0, nullptr, ml);
#ifdef QWB_EXP_TIMING
    DBG_T(t_d);
    if (tid == 0) {
      DBG_ADD(1, 0, t_b - t_a);
      DBG_ADD(1, 1, t_c - t_b);
      DBG_ADD(1, 2, t_d - t_c);
      DBG_ADD(1, 3, 1);
    }
    if (tid == 32 * 7) DBG_ADD(1, 4, dbg_clock() - t_c);
#endif
    // this tile's counter is published at the next prefetch point (after a
    // barrier that its stores precede), or here when the next item waits
    pend_tile = tr * tiles_x + cur.c;
    pend_val = ((unsigned)cur.k + 1) | (exact_used ? kFlag : 0u);
    if (!more) break;
    if (pw) v2 = poll(adv(nxt));
    if (shw[0] == 0) {
      __syncthreads();
      release(pend_tile, pend_val);
      pend_tile = -1;
      blocking_load(nxt, (it + 1) & 1);
    }
    cur = nxt;
    v1 = v2;
    ++it;
  }
  __syncthreads();
  if (pend_tile >= 0) release(pend_tile, pend_val);
}

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e && *e ? atoi(e) : dflt;
}

// tensor map of a planes buffer for the TMA tile loads: doubles
// [4][lrows][2 nx], box [4][RY][64] = one stage
template <class S>
bool encode_map(CUtensorMap* m, const double2* base, int nx, int lrows) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (e == cudaSuccess && fn) encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  if (!encode) return false;
  const cuuint64_t dims[3] = {2 * (cuuint64_t)nx, (cuuint64_t)lrows, 4};
  const cuuint64_t strides[2] = {2 * (cuuint64_t)nx * sizeof(double), (cuuint64_t)nx * lrows * sizeof(double2)};
  const cuuint32_t box[3] = {2 * (cuuint32_t)S::RX, (cuuint32_t)S::RY, 4};
  const cuuint32_t estr[3] = {1, 1, 1};
  return encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double2*>(base), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Encoded maps, keyed by (buffer, nx, lrows) per region shape: a run's
// ping-pong buffers are re-used launch after launch, so each is encoded once.
template <class S>
bool cached_map(CUtensorMap* m, const double2* base, int nx, int lrows) {
  struct Entry {
    const void* base;
    int nx, lrows;
    CUtensorMap map;
  };
  static Entry cache[8] = {};
  static int next = 0;
  static const bool use = env_int("QWB_LATTICE_TMA", 1) != 0;
  if (!use) return false;
  for (const Entry& e : cache)
    if (e.base == base && e.nx == nx && e.lrows == lrows) {
      *m = e.map;
      return true;
    }
  if (!encode_map<S>(m, base, nx, lrows)) return false;
  cache[next] = Entry{base, nx, lrows, *m};
  next = (next + 1) % 8;
  return true;
}

template <class K>
int configure(qwb_ctx* ctx, K kernel, size_t smem, bool* configured) {
  const int dev = ctx->device & 255;
  if (!configured[dev]) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return qwb::cuda_status(ctx, e, "cudaFuncSetAttribute(lattice_tb)");
    configured[dev] = true;
  }
  return QWB_OK;
}

template <int SHIFT, bool MARKED, int T, int BY, int V>
int launch_tb_t(qwb_ctx* ctx, cudaStream_t s, int nx, int ny, const TbGeo& geo, const double2* in,
                double2* out, const uint32_t* bits, const MarkedList& mk, const TraceList& tr, int tile0,
                int tile1, unsigned key, int* sticky, int grid_cap) {
  using Sh = TbShape<BY, V>;
  constexpr int OX = Sh::RX - 2 * T, OY = Sh::RY - 2 * T;
  const int tiles_x = (nx + OX - 1) / OX, tiles_y = (geo.nown + OY - 1) / OY;
  const int ntiles = tile1 > 0 ? tile1 : tiles_x * tiles_y;
  const size_t smem = Sh::smem_bytes();
  const int span = ntiles - tile0;
  if (span <= 0) return QWB_OK;
  const int cap = grid_cap > 0 && grid_cap < ctx->num_sms ? grid_cap : ctx->num_sms;
  const int grid = span < cap ? span : cap;
  CUtensorMap imap{};
  const int use_tma = cached_map<Sh>(&imap, in, nx, geo.lrows) ? 1 : 0;
  static const bool pdl = env_int("QWB_LATTICE_PDL", 1) != 0;   // see qwb::launch_pdl
  static bool conf_plain[256] = {}, conf_slab[256] = {};   // per instantiation, device
  if (!geo.wrap) {
    if constexpr (T == kSlabDepth && BY == 16 && V == 4) {
      if (tr.n > 0) QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "slab launches do not fuse traces");
      auto kernel = lattice_tb_kernel<SHIFT, MARKED, T, BY, V, true>;
      int st = configure(ctx, kernel, smem, conf_slab);
      if (st) return st;
      const cudaError_t e = qwb::launch_pdl(pdl, kernel, dim3(grid), dim3(32, BY), smem, s, nx, ny, geo, in, out,
                                            bits, mk, tiles_x, ntiles, tile0, imap, use_tma, key, sticky);
      if (e != cudaSuccess) return qwb::cuda_status(ctx, e, "cudaLaunchKernelEx(lattice_tb slab)");
      return QWB_OK;
    } else {
      QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "slab kernels exist for T = %d on 32x64 regions only", kSlabDepth);
    }
  }
  auto kernel = lattice_tb_kernel<SHIFT, MARKED, T, BY, V, false>;
  int st = configure(ctx, kernel, smem, conf_plain);
  if (st) return st;
  cudaError_t e = qwb::launch_pdl(pdl, kernel, dim3(grid), dim3(32, BY), smem, s, nx, ny, geo, in, out, bits, mk,
                                  tiles_x, ntiles, tile0, imap, use_tma, key, sticky);
  if (e != cudaSuccess) return qwb::cuda_status(ctx, e, "cudaLaunchKernelEx(lattice_tb)");
  if (tr.n == 0) return QWB_OK;
  // traced run: the light-cone kernel re-derives the traced vertices' levels
  // from this launch's (intact) input
  e = qwb::launch_pdl(pdl, lattice_trace_cone_kernel<SHIFT, T>, dim3(tr.n), dim3(256), 0, s, nx, ny, in,
                      MARKED ? bits : nullptr, tr);
  if (e != cudaSuccess) return qwb::cuda_status(ctx, e, "lattice_trace_cone_kernel");
  return QWB_OK;
}

template <int T, int BY, int V>
int launch_tb(qwb_ctx* ctx, int shift, cudaStream_t s, int nx, int ny, const TbGeo& g, const double2* in,
              double2* out, const uint32_t* bits, const MarkedList& mk, const TraceList& tr, int tile0, int tile1,
              unsigned key, int* sticky, int grid_cap) {
#define QWB_TB_GO(SH, MK) \
  launch_tb_t<SH, MK, T, BY, V>(ctx, s, nx, ny, g, in, out, bits, mk, tr, tile0, tile1, key, sticky, grid_cap)
  if (shift == QWB_SHIFT_FLIPFLOP) return bits ? QWB_TB_GO(QWB_SHIFT_FLIPFLOP, true) : QWB_TB_GO(QWB_SHIFT_FLIPFLOP, false);
  return bits ? QWB_TB_GO(QWB_SHIFT_PERSISTENT, true) : QWB_TB_GO(QWB_SHIFT_PERSISTENT, false);
#undef QWB_TB_GO
}

constexpr int kFlowT = 4, kFlowBY = 16, kFlowV = 4;

template <int SHIFT, bool MARKED>
int launch_flow_t(qwb_ctx* ctx, cudaStream_t s, int nx, int ny, double2* a, double2* b, const uint32_t* bits,
                  const MarkedList& mk, int nblocks) {
  using Sh = TbShape<kFlowBY, kFlowV>;
  constexpr int OX = Sh::RX - 2 * kFlowT, OY = Sh::RY - 2 * kFlowT;
  const int tiles_x = (nx + OX - 1) / OX, tiles_y = (ny + OY - 1) / OY;
  const int ntiles = tiles_x * tiles_y;
  void* ws;
  int st = qwb::workspace(ctx, (size_t)(ntiles + 1) * sizeof(unsigned), s, &ws);
  if (st) return st;
  QWB_CUDA(ctx, cudaMemsetAsync(ws, 0, (size_t)(ntiles + 1) * sizeof(unsigned), s));
  FlowArgs fa;
  fa.buf0 = a;
  fa.buf1 = b;
  fa.done = reinterpret_cast<unsigned*>(ws);
  fa.nblocks = nblocks;
  fa.rot = tiles_y / 2;
  CUtensorMap m0{}, m1{};
  const int use_tma = (cached_map<Sh>(&m0, a, nx, ny) && cached_map<Sh>(&m1, b, nx, ny)) ? 1 : 0;
  const size_t smem = Sh::smem_bytes();
  auto kernel = lattice_flow_kernel<SHIFT, MARKED, kFlowT, kFlowBY, kFlowV>;
  static bool conf[256] = {};
  st = configure(ctx, kernel, smem, conf);
  if (st) return st;
  // one CTA per SM, all co-resident (cooperative launch: the items of one
  // CTA wait on items of the others); -1: not possible here (caller falls
  // back to one launch per T steps)
  const int grid = ntiles < ctx->num_sms ? ntiles : ctx->num_sms;
  int per_sm = 0;
  QWB_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 32 * kFlowBY, smem));
  if (per_sm * ctx->num_sms < grid) return -1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(32, kFlowBY);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, nx, ny, fa, bits, mk, tiles_x, tiles_y, m0, m1, use_tma);
  if (e != cudaSuccess) return qwb::cuda_status(ctx, e, "cudaLaunchKernelEx(lattice_flow, cooperative)");
  return QWB_OK;
}

MarkedList marked_list(int nx, const int64_t* marked_host, int64_t n_marked) {
  MarkedList mk{};
  mk.n = n_marked <= 8 ? (int)n_marked : -1;
  for (int k = 0; k < mk.n; ++k) {
    mk.v[k] = marked_host[k];
    mk.x[k] = (int)(marked_host[k] % nx);
    mk.y[k] = (int)(marked_host[k] / nx);
  }
  return mk;
}

}  // namespace

namespace qwb {

// Steps per temporally blocked launch (0 = single-step kernel only).
// QWB_LATTICE_T overrides (0, 2..6); QWB_LATTICE_SHAPE the tile shape.
// Default 6: the tiles are HBM-bound at T = 4 (a tile costs its compulsory
// bytes' HBM time); at T = 6 each step moves 2/3 of the bytes for 30 % more
// on-chip adds, and the lower HBM power keeps the SM clock higher under the
// power cap (2048^2: 25.7 vs 27.9 us/step at 1920 vs 1770 MHz).
int lattice_tb_depth(int64_t nx, int64_t ny, int64_t n_marked) {
  (void)n_marked;
  static int depth = -1;
  if (depth < 0) {
    depth = env_int("QWB_LATTICE_T", 6);
    if (depth < 0 || depth == 1) depth = 6;
    if (depth > 6) depth = 6;
  }
  if (nx < 64 || ny < 64) return 0;   // tiny lattices: the single-step kernel is launch-bound anyway
  return depth;
}

static int shape_of(bool traced) {
  static int shape_env = env_int("QWB_LATTICE_SHAPE", 4);
  static int trace_shape = env_int("QWB_LATTICE_TRACE_SHAPE", 4);
  return traced ? trace_shape : shape_env;
}

static int tb_launch_impl(qwb_ctx* ctx, int depth, int shift, cudaStream_t s, int nx, int ny, const TbGeo& geo,
                          const double2* in, double2* out, const uint32_t* bits, const int64_t* marked_host,
                          int64_t n_marked, const int64_t* trace_vertices_host, int n_trace, double* trace,
                          int tile0, int tile1, unsigned key, int* sticky, int grid_cap = 0) {
  const int shape = shape_of(trace != nullptr);
  if (depth > 6) depth = 6;
  const MarkedList mk = marked_list(nx, marked_host, n_marked);
  TraceList tl{};
  tl.n = trace ? n_trace : 0;
  tl.out = trace;
  for (int k = 0; k < tl.n; ++k) {
    tl.v[k] = trace_vertices_host[k];
    tl.x[k] = (int)(trace_vertices_host[k] % nx);
    tl.y[k] = (int)(trace_vertices_host[k] / nx);
  }
  // shape 4 (default): 32x16 threads, 4 rows each (32x64 region); 3: 32x16
  // threads, 3 rows each (32x48 region, two load stages).  The 32x32 and
  // 24-warp 32x48 shapes measured slower and are not built.
#define QWB_TB_CASE(T_)                                                                                          \
  case T_:                                                                                                       \
    if (shape == 3)                                                                                            \
      return launch_tb<T_, 16, 3>(ctx, shift, s, nx, ny, geo, in, out, bits, mk, tl, tile0, tile1, key, sticky, \
                                  grid_cap);                                                                 \
    return launch_tb<T_, 16, 4>(ctx, shift, s, nx, ny, geo, in, out, bits, mk, tl, tile0, tile1, key, sticky,   \
                                grid_cap);
  switch (depth) {
    QWB_TB_CASE(2)
    QWB_TB_CASE(3)
    QWB_TB_CASE(4)
    QWB_TB_CASE(5)
    QWB_TB_CASE(6)
    default:
      QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "unsupported temporal block depth %d", depth);
  }
#undef QWB_TB_CASE
}

int lattice_tb_launch(qwb_ctx* ctx, int depth, int shift, cudaStream_t s, int nx, int ny,
                      const double2* in, double2* out, const uint32_t* bits,
                      const int64_t* marked_host, int64_t n_marked,
                      const int64_t* trace_vertices_host, int n_trace, double* trace, int check, int* sticky) {
  const TbGeo geo{ny, 0, ny, 0, 1};
  return tb_launch_impl(ctx, depth, shift, s, nx, ny, geo, in, out, bits, marked_host, n_marked,
                        trace_vertices_host, n_trace, trace, 0, 0, check ? kTinyKeyPeriodic : 0u, sticky);
}

int lattice_sticky(qwb_ctx* ctx, int** out) {
  if (!ctx->lat_sticky) {
    cudaError_t e = cudaMalloc(&ctx->lat_sticky, 256);
    if (e != cudaSuccess) return cuda_status(ctx, e, "cudaMalloc(lattice flag)");
  }
  *out = ctx->lat_sticky;
  return QWB_OK;
}

// The flow kernel (its own depth kFlowT) runs untraced torus runs of >= 2
// blocks when a block is 2 to 16 waves of tiles (num_sms CTAs) and the
// per-launch kernel at `depth` would leave more than 10 % of its last wave
// idle: there the per-launch kernel's fixed cost per launch (grid fill, tail,
// launch gap: ~11 us) dominates; on larger lattices the flow kernel's own
// per-item scheduling costs more (measured).
// QWB_LATTICE_FLOW=0: never, 2: always.
int lattice_flow_blocks(int64_t nx, int64_t ny, int depth, bool traced, int64_t steps, int num_sms) {
  static const int use = env_int("QWB_LATTICE_FLOW", 1);
  if (!use || traced || shape_of(false) != 4 || nx < 256 || ny < 256) return 0;
  using Sh = TbShape<kFlowBY, kFlowV>;
  constexpr int OX = Sh::RX - 2 * kFlowT, OY = Sh::RY - 2 * kFlowT;
  const int64_t ntiles = ((nx + OX - 1) / OX) * ((ny + OY - 1) / OY);
  if (use == 1) {
    if (ntiles < 2 * (int64_t)num_sms || ntiles >= 16 * (int64_t)num_sms) return 0;
    int tx, ty;
    lattice_tb_tiles(depth, (int)nx, (int)ny, &tx, &ty);
    const double waves = (double)tx * ty / num_sms;
    if (waves / std::ceil(waves) >= 0.9) return 0;
  }
  const int64_t nb = steps / kFlowT;
  return nb >= 2 ? (int)(nb < (1 << 24) ? nb : (1 << 24)) : 0;
}

int lattice_flow_launch(qwb_ctx* ctx, int shift, cudaStream_t s, int nx, int ny, double2* a, double2* b,
                        const uint32_t* bits, const int64_t* marked_host, int64_t n_marked, int nblocks) {
  const MarkedList mk = marked_list(nx, marked_host, n_marked);
  if (shift == QWB_SHIFT_FLIPFLOP)
    return bits ? launch_flow_t<QWB_SHIFT_FLIPFLOP, true>(ctx, s, nx, ny, a, b, bits, mk, nblocks)
                : launch_flow_t<QWB_SHIFT_FLIPFLOP, false>(ctx, s, nx, ny, a, b, bits, mk, nblocks);
  return bits ? launch_flow_t<QWB_SHIFT_PERSISTENT, true>(ctx, s, nx, ny, a, b, bits, mk, nblocks)
              : launch_flow_t<QWB_SHIFT_PERSISTENT, false>(ctx, s, nx, ny, a, b, bits, mk, nblocks);
}

int lattice_slab_depth(int depth) {   // the ghost-row depth a slab run can use (0: none)
  return (depth == kSlabDepth && env_int("QWB_LATTICE_SHAPE", 4) == 4) ? depth : 0;
}

int lattice_tb_owned_rows(int depth) {
  if (depth < 2) return 0;
  const int shape = env_int("QWB_LATTICE_SHAPE", 4);
  const int ry = shape == 3 ? 16 * 3 : 16 * 4;
  return ry - 2 * (depth > 6 ? 6 : depth);
}

int lattice_tb_launch_geo(qwb_ctx* ctx, int depth, int shift, cudaStream_t s, int nx, int ny, const TbGeo& geo,
                          const double2* in, double2* out, const uint32_t* bits, const int64_t* marked_host,
                          int64_t n_marked, int tile0, int tile1, int grid_cap, int check, int* sticky) {
  // no run flag: every launch tests its tiles (horizon: one launch);
  // with one: the run's first launch after each exchange tests (qwb_slab_run_fused)
  const unsigned key = sticky ? (check ? kTinyKeyPeriodic : 0u) : kTinyKey;
  return tb_launch_impl(ctx, depth, shift, s, nx, ny, geo, in, out, bits, marked_host, n_marked, nullptr, 0,
                        nullptr, tile0, tile1, key, sticky, grid_cap);
}

int lattice_tb_tiles(int depth, int nx, int nown, int* tiles_x, int* tiles_y) {
  const int shape = env_int("QWB_LATTICE_SHAPE", 4);
  const int ry = shape == 3 ? 16 * 3 : 16 * 4;
  const int d = depth > 6 ? 6 : depth;
  const int ox = 32 - 2 * d, oy = ry - 2 * d;
  *tiles_x = (nx + ox - 1) / ox;
  *tiles_y = (nown + oy - 1) / oy;
  return oy;
}

}  // namespace qwb

extern "C" int qwb_lattice_fused_depth(int64_t nx, int64_t ny, int64_t n_marked, int* depth_host,
                                       int* kind_host) {
  const int d = qwb::lattice_tb_depth(nx, ny, n_marked);
  if (depth_host) *depth_host = d;
  // 2: one flow launch per untraced run, 1: one tile launch per T steps
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaGetLastError();
  if (kind_host) *kind_host = (d > 0 && qwb::lattice_flow_blocks(nx, ny, d, false, 2 * d, sms)) ? 2 : 1;
  return QWB_OK;
}

#ifdef QWB_EXP_TIMING
extern "C" int qwb_exp_timeline(unsigned long long* out_host, int reset) {
  cudaMemcpyFromSymbol(out_host, g_tl, sizeof(g_tl));
  if (reset) {
    unsigned int z = 0;
    cudaMemcpyToSymbol(g_ctas, &z, sizeof(z));
  }
  return 0;
}
extern "C" int qwb_exp_dbg(unsigned long long* out_host, int reset) {
  cudaMemcpyFromSymbol(out_host, g_dbg, sizeof(g_dbg));
  if (reset) {
    unsigned long long z[2][8] = {};
    cudaMemcpyToSymbol(g_dbg, z, sizeof(z));
  }
  return 0;
}
#endif
