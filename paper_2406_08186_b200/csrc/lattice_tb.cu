// lattice_tb.cu — temporally blocked torus walk: T coined steps per HBM pass.
//
// The single-step kernel (lattice.cu) already moves exactly the 32 B per arc
// per step that one application of U needs, at ~96 % of the measured HBM copy
// bandwidth.  The only way past that roofline is to apply U several times per
// trip through HBM.  Each CTA owns a region of 32 x (BY*V) vertices; a thread
// owns V vertically adjacent vertices with their 4 direction amplitudes in
// registers:
//
//   * the region's state arrives in shared memory one or two tiles ahead of its
//     use, so HBM reads overlap the arithmetic of the current tile: regions
//     inside the buffer with ONE tensor TMA (box [4 planes][BY*V rows][32]
//     complex128, completion on a stage mbarrier), regions that wrap around
//     the torus with per-thread 16-B cp.async;
//   * T steps run on chip, in doubled space (qwb_lattice.cuh "doubled-space
//     forms": the operator 2U needs additions only — 20 FP64 adds per vertex
//     and step — and the state is scaled by 2^-T on the way out, so the result
//     has numpy's bits for every non-zero amplitude).  Pushes to x +- 1 go
//     through warp shuffles (a warp is one region row of 32 columns), pushes
//     between a thread's own V rows stay in registers, and only the pushes
//     across thread rows go through a double-buffered shared-memory exchange
//     (one barrier per step);
//   * values near the region edge go stale one ring per step, so after T steps
//     the inner (32 - 2T) x (BY*V - 2T) vertices are exact and are written.
//
// Regions wrap around the torus (modular global coordinates): any nx, ny >= 3.
// The same kernel runs on multi-GPU y-slabs with ghost state rows (SLAB,
// TbGeo): owned rows only, no y-wrap (comm.cu qwb_slab_run_fused).
// Default tile: 16 warps x 4 rows (32 x 64 region), T = 4.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <string.h>

#include "qwb_lattice.cuh"

namespace {

using qwb::TbGeo;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

__device__ __forceinline__ void tb_mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void tb_mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tb_mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "TB_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra TB_WAIT_%=;\n"
      "}\n" ::"r"((unsigned)__cvta_generic_to_shared(b)),
      "r"(parity)
      : "memory");
}

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
constexpr size_t kTraceRecBytes = 6 * 8 * 4 * sizeof(double2);   // [T <= 6][8 vertices][4 planes]

template <int BY, int V>
struct TbShape {
  static constexpr int RX = 32;            // region columns (= warp lanes)
  static constexpr int RY = BY * V;        // region rows
  static constexpr int NT = 32 * BY;       // threads
  static constexpr int REG = RX * RY;      // region vertices
  // stages of the next tiles' amplitudes: two (loads of two tiles in flight)
  // when they fit next to the exchange buffers, else one
  static constexpr int NSTAGE =
      ((8 * (size_t)REG + 4 * (size_t)NT) * sizeof(double2) + 16 + kTraceRecBytes <= 232448) ? 2 : 1;
  static constexpr size_t smem_bytes() {   // + two mbarriers for the TMA loads + the trace record
    return (4 * (size_t)REG * NSTAGE + 4 * (size_t)NT) * sizeof(double2) + 2 * sizeof(uint64_t) +
           kTraceRecBytes;
  }
};

// p(v) per step for up to 8 traced vertices (search runs): out[t * n + k];
// x, y: the vertices' coordinates (host-computed, no division on the device)
struct TraceList {
  int n;
  int64_t v[8];
  int x[8], y[8];
  double* out;
};

// p of a traced vertex from its level-t (doubled-space) amplitudes a[0..3]
// (planes D, L, R, U): unscale, reference slot order, numpy |z|^2, row sum.
__device__ __forceinline__ double trace_p(int gx, int gy, int nx, int ny, double sc, const double2* a) {
  const auto un = [&](double2 z) { return make_double2(__dmul_rn(z.x, sc), __dmul_rn(z.y, sc)); };
  const qwb::Slots o = qwb::order_slots(gx, gy, nx, ny, un(a[0]), un(a[1]), un(a[2]), un(a[3]));
  const double m0 = qwb::abs2_np(o.s0), m1 = qwb::abs2_np(o.s1), m2 = qwb::abs2_np(o.s2), m3 = qwb::abs2_np(o.s3);
  return __dadd_rn(m0, __dadd_rn(__dadd_rn(m1, m2), m3));
}

// Light-cone trace.  The traced vertex's amplitudes at levels 0..T-1 of a
// T-step launch depend only on the (2T+1)^2 input vertices around it, so one
// CTA per traced vertex recomputes that patch with the tile kernel's own
// arithmetic (vertex_outputs2 in doubled space, the same pushes) and writes p
// per level: bit-identical to the TRACE tile recompute, at a few microseconds
// instead of a whole 32x64 tile.  Reads the launch's input, writes the trace
// only.  Patch vertices whose neighbours fall outside the patch go stale one
// ring per step; the centre stays exact for T steps.
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
  if (act) {
#pragma unroll
    for (int p = 0; p < 4; ++p) v[p] = in[p * n + w];
    if (bits) mk = (__ldg(bits + (w >> 5)) >> (w & 31)) & 1u;
  }
  const bool centre = act && px == T && py == T;
#pragma unroll 1
  for (int t = 0; t < T; ++t) {
    if (centre) tr.out[t * tr.n + k] = trace_p(gx, gy, nx, ny, 1.0 / (double)(1 << t), v);
    if (act) qwb::vertex_outputs2(gx, gy, nx, ny, mk, v[0], v[1], v[2], v[3], o[0][i], o[1][i], o[2][i], o[3][i]);
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

// T steps of a tile on chip (see the file comment).  INTERIOR: every vertex of
// the region is an unmarked, untraced interior vertex (no slot permutation, no
// branches).  TRACE: record the level-t amplitudes of the traced vertices this
// tile owns (the exact inner block) in trbuf[t][k][4]; p is computed after
// the steps (no call and no extra registers in the step loop).
template <int SHIFT, bool MARKED, int T, int BY, int V, bool INTERIOR, bool TRACE>
__device__ __forceinline__ void tile_steps(int nx, int ny, int gx, const int (&gy)[V],
                                           const uint32_t* __restrict__ bits, double2 (&vD)[V],
                                           double2 (&vL)[V], double2 (&vR)[V], double2 (&vU)[V],
                                           double2* xD, double2* xU, int tid, int ty,
                                           const TraceList& tr, const bool (&own)[V], double2* trbuf) {
  bool mk[V];
#pragma unroll
  for (int j = 0; j < V; ++j) {
    mk[j] = false;
    if (MARKED) {
      const int64_t wg = (int64_t)gy[j] * nx + gx;
      mk[j] = (__ldg(bits + (wg >> 5)) >> (wg & 31)) & 1u;
    }
  }
#pragma unroll
  for (int t = 0; t < T; ++t) {
    if (TRACE) {
#pragma unroll
      for (int j = 0; j < V; ++j) {
        if (!own[j]) continue;
        const int64_t wg = (int64_t)gy[j] * nx + gx;
#pragma unroll
        for (int k = 0; k < 8; ++k) {   // static indices: tr stays in the param space
          if (k >= tr.n || tr.v[k] != wg) continue;
          double2* a = trbuf + (t * 8 + k) * 4;   // level t holds 2^t psi_t
          a[0] = vD[j];
          a[1] = vL[j];
          a[2] = vR[j];
          a[3] = vU[j];
        }
      }
    }
    double2 oD[V], oL[V], oR[V], oU[V];
#pragma unroll
    for (int j = 0; j < V; ++j) {
      if (INTERIOR)
        qwb::vertex_outputs2_interior(vD[j], vL[j], vR[j], vU[j], oD[j], oL[j], oR[j], oU[j]);
      else
        qwb::vertex_outputs2(gx, gy[j], nx, ny, mk[j], vD[j], vL[j], vR[j], vU[j], oD[j], oL[j],
                             oR[j], oU[j]);
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
    __syncthreads();
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
}

struct MarkedList {   // up to 8 marked vertex ids; n < 0: more than 8 (use the bitmap)
  int n;
  int64_t v[8];
  int x[8], y[8];     // their coordinates (host-computed)
};

// SLAB: the buffer is a y-slab with ghost rows (geo), else the whole torus
template <int SHIFT, bool MARKED, int T, int BY, int V, bool TRACE, bool SLAB>
__global__ void __launch_bounds__(32 * BY, 1)
lattice_tb_kernel(int nx, int ny, TbGeo geo, const double2* __restrict__ in, double2* __restrict__ out,
                  const uint32_t* __restrict__ bits, MarkedList mk, TraceList tr, int tiles_x,
                  int ntiles, int tile0, const __grid_constant__ CUtensorMap imap, int use_tma) {
  using S = TbShape<BY, V>;
  constexpr int OX = S::RX - 2 * T, OY = S::RY - 2 * T;   // exact (owned) block
  extern __shared__ double2 sm[];
  double2* stage0 = sm;                // [NSTAGE][4][RY][RX] next tiles' amplitudes
  double2* xD = sm + 4 * S::REG * S::NSTAGE;   // [2][BY][32] O_D of each thread's lowest row
  double2* xU = xD + 2 * S::NT;        // [2][BY][32] O_U of each thread's highest row
  uint64_t* tbar = reinterpret_cast<uint64_t*>(xU + 2 * S::NT);   // [2] TMA-load barriers
  double2* trbuf = reinterpret_cast<double2*>(tbar + 2);          // [T][8][4] traced amplitudes (TRACE)
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = ty * 32 + tx;
  if (!SLAB) geo = TbGeo{ny, 0, ny, 0, 1};   // compile-time constants for the torus
  // Tiles whose region lies inside the torus (no wrap) load all four planes
  // with ONE tensor TMA (box [4][RY][32] complex128) completing on a stage
  // mbarrier; regions that wrap use per-thread cp.async.
  const bool tma = use_tma;
  if (tma) {
    if (tid == 0) {
      tb_mbar_init(tbar, 1);
      tb_mbar_init(tbar + 1, 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
  }
  auto tma_ok = [&](int tcol, int trow) {   // the region lies inside the buffer (no wrap)
    const int bx = tcol * OX - T, by = geo.own0 + trow * OY - T;
    return tma && bx >= 0 && bx + S::RX <= nx && by >= 0 && by + S::RY <= geo.lrows;
  };
  auto tma_load = [&](double2* stage, uint64_t* bar, int tcol, int trow) {
    if (tid == 0) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // earlier LDS of this stage
      tb_mbar_expect_tx(bar, 4u * S::REG * (uint32_t)sizeof(double2));
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
          "[%5];\n" ::"r"((unsigned)__cvta_generic_to_shared(stage)),
          "l"(reinterpret_cast<uint64_t>(&imap)), "r"(2 * (tcol * OX - T)), "r"(geo.own0 + trow * OY - T), "r"(0),
          "r"((unsigned)__cvta_generic_to_shared(bar))
          : "memory");
    }
  };
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
  auto prefetch = [&](double2* stage, int tcol, int trow) {
    const int bx = tcol * OX - T + tx;
    const int by = geo.own0 + trow * OY - T + ty * V;   // local buffer row
    const int gx = wrapc(bx, nx);
#pragma unroll
    for (int j = 0; j < V; ++j) {
      // rows outside a slab buffer are > T rows from every owned row: left stale
      const int ly = by + j;
      if (SLAB && (ly < 0 || ly >= geo.lrows)) continue;
      const int r = SLAB ? ly : wrapc(ly, ny);
      const int64_t w = (int64_t)r * nx + gx;
      const int li = (ty * V + j) * 32 + tx;
#pragma unroll
      for (int p = 0; p < 4; ++p) cp_async16(stage + p * S::REG + li, in + p * n + w);
    }
  };

  // programmatic dependent launch: everything above overlaps the previous
  // launch's last tiles; its output (this launch's input) is visible after the
  // wait (a no-op when launched without the PDL attribute)
  qwb::pdl_wait();
  int tile = blockIdx.x + tile0;   // tile0 > 0: a launch over tiles [tile0, ntiles) only
  if (tile >= ntiles) return;
  int tcol = tile % tiles_x, trow = tile / tiles_x;
  // (pcol, prow): the tile the next prefetch loads, NSTAGE - 1 tiles ahead of (tcol, trow)
  int pcol = tcol, prow = trow, ptile = tile;
  // per stage: whether its pending load is a TMA (f) and that barrier's parity (ph)
  bool f0 = false, f1 = false;
  uint32_t ph0 = 0, ph1 = 0;
  for (int k = 0; k < S::NSTAGE; ++k) {
    if (ptile < ntiles) {
      double2* st = stage0 + (size_t)k * 4 * S::REG;
      if (tma_ok(pcol, prow)) {
        tma_load(st, tbar + k, pcol, prow);
        (k ? f1 : f0) = true;
      } else {
        prefetch(st, pcol, prow);
      }
    }
    cp_commit();
    advance(pcol, prow);
    ptile += gridDim.x;
  }
  for (int it = 0; tile < ntiles; tile += gridDim.x, ++it) {
    // last tile of this CTA: let the next launch's CTAs take the SMs that
    // finish first (they block in griddepcontrol.wait until this grid is done)
    if (tile + (int)gridDim.x >= ntiles) qwb::pdl_trigger();
    const int k = S::NSTAGE == 2 ? (it & 1) : 0;
    double2* stage = stage0 + (size_t)k * 4 * S::REG;
    // x0: global column of the tile's first owned column; y0: unwrapped
    // global row of its first owned row; lyb: its local buffer row
    const int trow_now = trow;
    const int x0 = tcol * OX, y0 = geo.ybase + trow_now * OY, lyb = geo.own0 + trow_now * OY;
    advance(tcol, trow);
    const int gx = wrapc(x0 - T + tx, nx);
    int gy[V];
    double2 vD[V], vL[V], vR[V], vU[V];
    if (S::NSTAGE == 2)
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");   // this tile's group; the next may fly
    else
      cp_wait_all();
    if (k ? f1 : f0) {   // this stage came by TMA: wait for its bytes
      tb_mbar_wait(tbar + k, k ? ph1 : ph0);
      if (k) ph1 ^= 1u; else ph0 ^= 1u;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < V; ++j) {
      gy[j] = wrapc(y0 - T + ty * V + j, ny);
      const int li = (ty * V + j) * 32 + tx;
      vD[j] = stage[li];
      vL[j] = stage[S::REG + li];
      vR[j] = stage[2 * S::REG + li];
      vU[j] = stage[3 * S::REG + li];
    }
    __syncthreads();
    if (k) f1 = false; else f0 = false;
    if (ptile < ntiles) {   // into the stage just consumed
      if (tma_ok(pcol, prow)) {
        tma_load(stage, tbar + k, pcol, prow);
        if (k) f1 = true; else f0 = true;
      } else {
        prefetch(stage, pcol, prow);
      }
    }
    cp_commit();
    advance(pcol, prow);
    ptile += gridDim.x;
    // regions that touch no torus edge and hold no marked or traced vertex run
    // a branch-free specialisation: every vertex is interior (slot order D L R U)
    auto in_region = [&](int mx, int my) {
      return mx >= x0 - T && mx < x0 - T + 32 && my >= y0 - T && my < y0 - T + S::RY;
    };
    bool interior = x0 - T >= 1 && x0 - T + 31 <= nx - 2 && y0 - T >= 1 &&
                    y0 - T + S::RY - 1 <= ny - 2;
    if (MARKED && interior) {
      if (mk.n < 0) {
        interior = false;   // too many marked vertices for the list: general path
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) interior &= (k >= mk.n) || !in_region(mk.x[k], mk.y[k]);
      }
    }
    if (TRACE)
#pragma unroll
      for (int k = 0; k < 8; ++k) interior &= (k >= tr.n) || !in_region(tr.x[k], tr.y[k]);
    const bool col_ok = tx >= T && tx < T + OX && x0 + tx - T < nx;
    bool own[V];
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int ly = ty * V + j;
      own[j] = col_ok && ly >= T && ly < T + OY && trow_now * OY + ly - T < geo.nown;
    }
    if (interior) {
      tile_steps<SHIFT, false, T, BY, V, true, false>(nx, ny, gx, gy, bits, vD, vL, vR, vU, xD, xU,
                                                      tid, ty, tr, own, trbuf);
    } else {
      tile_steps<SHIFT, MARKED, T, BY, V, false, TRACE>(nx, ny, gx, gy, bits, vD, vL, vR, vU, xD, xU,
                                                        tid, ty, tr, own, trbuf);
      if (TRACE) {   // p of the traced vertices this tile owns, every level
        __syncthreads();
        if (tid < T * 8) {
          const int t = tid >> 3, k = tid & 7;
          const int mx = tr.x[k < tr.n ? k : 0], my = tr.y[k < tr.n ? k : 0];
          const bool mine = k < tr.n && mx >= x0 && mx < x0 + OX && mx < nx && my >= y0 && my < y0 + OY &&
                            my - y0 + trow_now * OY < geo.nown;
          if (mine)
            tr.out[t * tr.n + k] = trace_p(mx, my, nx, ny, 1.0 / (double)(1 << t), trbuf + (t * 8 + k) * 4);
        }
      }
    }
    constexpr double kScale = 1.0 / (double)(1 << T);   // undo the doubled-space steps (exact)
#pragma unroll
    for (int j = 0; j < V; ++j) {
      if (own[j]) {
        const int64_t w = (int64_t)(lyb - T + ty * V + j) * nx + gx;
        __stcs(out + w, make_double2(__dmul_rn(vD[j].x, kScale), __dmul_rn(vD[j].y, kScale)));
        __stcs(out + n + w, make_double2(__dmul_rn(vL[j].x, kScale), __dmul_rn(vL[j].y, kScale)));
        __stcs(out + 2 * n + w, make_double2(__dmul_rn(vR[j].x, kScale), __dmul_rn(vR[j].y, kScale)));
        __stcs(out + 3 * n + w, make_double2(__dmul_rn(vU[j].x, kScale), __dmul_rn(vU[j].y, kScale)));
      }
    }
  }
  cp_wait_all();
}

int env_int(const char* name, int dflt);

template <int SHIFT, bool MARKED, int T, int BY, int V>
int launch_tb_t(qwb_ctx* ctx, cudaStream_t s, int nx, int ny, const TbGeo& geo, const double2* in,
                double2* out, const uint32_t* bits, const MarkedList& mk, const TraceList& tr) {
  using Sh = TbShape<BY, V>;
  constexpr int OX = Sh::RX - 2 * T, OY = Sh::RY - 2 * T;
  const int tiles_x = (nx + OX - 1) / OX, tiles_y = (geo.nown + OY - 1) / OY;
  const int ntiles = tiles_x * tiles_y;
  const size_t smem = Sh::smem_bytes();
  const int grid = ntiles < ctx->num_sms ? ntiles : ctx->num_sms;
  // tensor map of the input planes for the TMA tile loads: doubles
  // [4][lrows][2 nx] (lrows = ny on the torus, the slab's buffer rows), box
  // [4][RY][64] = one stage
  CUtensorMap imap{};
  static int use_tma_env = env_int("QWB_LATTICE_TMA", 1);
  int use_tma = 0;
  if (use_tma_env) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
      cudaDriverEntryPointQueryResult q;
      void* fn = nullptr;
      cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
      if (e == cudaSuccess && fn) encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    if (encode) {
      const cuuint64_t dims[3] = {2 * (cuuint64_t)nx, (cuuint64_t)geo.lrows, 4};
      const cuuint64_t strides[2] = {2 * (cuuint64_t)nx * sizeof(double),
                                     (cuuint64_t)nx * geo.lrows * sizeof(double2)};
      const cuuint32_t box[3] = {2 * (cuuint32_t)Sh::RX, (cuuint32_t)Sh::RY, 4};
      const cuuint32_t estr[3] = {1, 1, 1};
      use_tma = encode(&imap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double2*>(in), dims, strides, box,
                       estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
  }
  auto go = [&](auto kernel, bool* configured, int grid_ = 0, int tile0 = 0, int ntiles_ = 0) -> int {
    const int dev = ctx->device & 255;
    if (!configured[dev]) {
      cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return qwb::cuda_status(ctx, e, "cudaFuncSetAttribute(lattice_tb)");
      configured[dev] = true;
    }
    static const bool pdl = env_int("QWB_LATTICE_PDL", 1) != 0;   // see qwb::launch_pdl
    const cudaError_t e = qwb::launch_pdl(pdl, kernel, dim3(grid_ ? grid_ : grid), dim3(32, BY), smem, s, nx, ny,
                                          geo, in, out, bits, mk, tr, tiles_x, ntiles_ ? ntiles_ : ntiles, tile0,
                                          imap, use_tma);
    if (e != cudaSuccess) return qwb::cuda_status(ctx, e, "cudaLaunchKernelEx(lattice_tb)");
    return QWB_OK;
  };
  static bool conf_plain[256] = {}, conf_trace[256] = {}, conf_slab[256] = {};   // per instantiation, device
  if (!geo.wrap) {
    if constexpr (T == kSlabDepth && BY == 16 && V == 4) {
      if (tr.n > 0) QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "slab launches do not fuse traces");
      return go(lattice_tb_kernel<SHIFT, MARKED, T, BY, V, false, true>, conf_slab);
    } else {
      QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "slab kernels exist for T = %d on 32x64 regions only", kSlabDepth);
    }
  }
  // QWB_LATTICE_TRACE_SPLIT: 2 (default) light-cone trace kernel after the
  // plain launch, 1 TRACE tile recompute per traced tile, 0 trace fused into
  // the full launch (the last two measured slower: DESIGN.md §4)
  static int trace_split = env_int("QWB_LATTICE_TRACE_SPLIT", 2);
  if (tr.n > 0 && !trace_split) return go(lattice_tb_kernel<SHIFT, MARKED, T, BY, V, true, false>, conf_trace);
  int st = go(lattice_tb_kernel<SHIFT, MARKED, T, BY, V, false, false>, conf_plain);
  if (st || tr.n == 0) return st;
  if (trace_split == 2) {
    static const bool pdl = env_int("QWB_LATTICE_PDL", 1) != 0;
    const cudaError_t e = qwb::launch_pdl(pdl, lattice_trace_cone_kernel<SHIFT, T>, dim3(tr.n), dim3(256), 0, s,
                                          nx, ny, in, MARKED ? bits : nullptr, tr);
    if (e != cudaSuccess) return qwb::cuda_status(ctx, e, "lattice_trace_cone_kernel");
    return QWB_OK;
  }
  // Traced run: the plain launch above advanced every tile; the tiles that own
  // a traced vertex are then recomputed from the same input (still intact: the
  // output is the other buffer) by the TRACE instantiation, one CTA each, which
  // records the traced vertices' per-level p and stores the same owned values
  // again.  Keeps the trace's registers and checks out of the full launch.
  int done_tiles[8];
  int nd = 0;
  for (int k = 0; k < tr.n; ++k) {
    const int t = (tr.y[k] / OY) * tiles_x + tr.x[k] / OX;
    bool seen = false;
    for (int j = 0; j < nd; ++j) seen |= done_tiles[j] == t;
    if (seen) continue;
    done_tiles[nd++] = t;
    st = go(lattice_tb_kernel<SHIFT, MARKED, T, BY, V, true, false>, conf_trace, 1, t, t + 1);
    if (st) return st;
  }
  return QWB_OK;
}

template <int T, int BY, int V>
int launch_tb(qwb_ctx* ctx, int shift, cudaStream_t s, int nx, int ny, const TbGeo& g, const double2* in,
              double2* out, const uint32_t* bits, const MarkedList& mk, const TraceList& tr) {
  if (shift == QWB_SHIFT_FLIPFLOP) {
    return bits ? launch_tb_t<QWB_SHIFT_FLIPFLOP, true, T, BY, V>(ctx, s, nx, ny, g, in, out, bits, mk, tr)
                : launch_tb_t<QWB_SHIFT_FLIPFLOP, false, T, BY, V>(ctx, s, nx, ny, g, in, out, bits, mk, tr);
  }
  return bits ? launch_tb_t<QWB_SHIFT_PERSISTENT, true, T, BY, V>(ctx, s, nx, ny, g, in, out, bits, mk, tr)
              : launch_tb_t<QWB_SHIFT_PERSISTENT, false, T, BY, V>(ctx, s, nx, ny, g, in, out, bits, mk, tr);
}

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e && *e ? atoi(e) : dflt;
}

// ---------------------------------------------------------------------------
// Wavefront variant: one warp = one column strip of 32 lanes that streams
// along y.  Level t+1 of row r needs level t of rows r-1, r, r+1 only, so a
// warp keeps, for each level, the outputs of the last two rows in registers
// and completes one row per level per iteration (a skewed wavefront): no
// shared memory, no barriers, warps fully independent.  Pushes along x use
// shuffles; pushes along y are register moves.  Redundant work: 2T halo lanes
// of 32 and 2T warm-up rows per strip.
// ---------------------------------------------------------------------------
__device__ __forceinline__ bool in_list(const MarkedList& m, int64_t w) {
  bool r = false;
#pragma unroll
  for (int k = 0; k < 8; ++k) r |= (k < m.n) && (m.v[k] == w);
  return r;
}

__device__ __forceinline__ void ld4(const double2* __restrict__ in, int64_t n, int64_t w, double2& d,
                                    double2& l, double2& r, double2& u) {
  d = __ldcs(in + w);
  l = __ldcs(in + n + w);
  r = __ldcs(in + 2 * n + w);
  u = __ldcs(in + 3 * n + w);
}

template <int SHIFT, bool MARKED, int T>
__global__ void __launch_bounds__(128)
lattice_wf_kernel(int nx, int ny, const double2* __restrict__ in, double2* __restrict__ out,
                  MarkedList mk, int strips_x, int nstrips, int L) {
  constexpr int OX = 32 - 2 * T;
  const int lane = threadIdx.x & 31;
  const int strip = (int)((blockIdx.x * (unsigned)blockDim.x + threadIdx.x) >> 5);
  if (strip >= nstrips) return;
  const int x0 = (strip % strips_x) * OX, y0 = (strip / strips_x) * L;
  const int yend = min(y0 + L, ny);
  const int gx = wrapc(x0 - T + lane, nx);
  const bool col_out = lane >= T && lane < T + OX && x0 + lane - T < nx;
  const int64_t n = (int64_t)nx * ny;
  const int ys = y0 - T;
  const int rows = (yend - y0) + 2 * T;

  // per level t-1 (0..T-1): outputs of the previous row (L, R, U needed) and
  // the U output of the row before it
  double2 pOL[T], pOR[T], pOU[T], ppOU[T];
#pragma unroll
  for (int t = 0; t < T; ++t) {
    pOL[t] = pOR[t] = pOU[t] = ppOU[t] = make_double2(0.0, 0.0);
  }
  double2 nD, nL, nR, nU;
  ld4(in, n, (int64_t)wrapc(ys, ny) * nx + gx, nD, nL, nR, nU);
#pragma unroll 1
  for (int i = 0; i < rows; ++i) {
    double2 sD = nD, sL = nL, sR = nR, sU = nU;
    {
      const int nr = (i + 1 < rows) ? ys + i + 1 : ys + i;   // clamped prefetch, no branch
      ld4(in, n, (int64_t)wrapc(nr, ny) * nx + gx, nD, nL, nR, nU);
    }
    const int r = ys + i;
    int gy = wrapc(r, ny);
    double2 cD, cL, cR, cU;
    {
      const bool m = MARKED && in_list(mk, (int64_t)gy * nx + gx);
      qwb::vertex_outputs2(gx, gy, nx, ny, m, sD, sL, sR, sU, cD, cL, cR, cU);
    }
#pragma unroll
    for (int t = 1; t <= T; ++t) {   // level t holds 2^t psi_t (doubled-space steps)
      const double2 fromAbove = cD;                    // O_D of row r-t+1
      const double2 fromRight = shfl_down2(pOL[t - 1]);   // O_L of (x+1, r-t)
      const double2 fromLeft = shfl_up2(pOR[t - 1]);      // O_R of (x-1, r-t)
      const double2 fromBelow = ppOU[t - 1];           // O_U of row r-t-1
      ppOU[t - 1] = pOU[t - 1];
      pOL[t - 1] = cL;
      pOR[t - 1] = cR;
      pOU[t - 1] = cU;
      if (SHIFT == QWB_SHIFT_FLIPFLOP) {
        sU = fromAbove; sD = fromBelow; sR = fromRight; sL = fromLeft;
      } else {
        sD = fromAbove; sU = fromBelow; sL = fromRight; sR = fromLeft;
      }
      gy = gy == 0 ? ny - 1 : gy - 1;                  // row r - t
      if (t < T) {
        const bool m = MARKED && in_list(mk, (int64_t)gy * nx + gx);
        qwb::vertex_outputs2(gx, gy, nx, ny, m, sD, sL, sR, sU, cD, cL, cR, cU);
      } else if (i >= 2 * T && col_out) {
        constexpr double kScale = 1.0 / (double)(1 << T);
        const int64_t w = (int64_t)gy * nx + gx;
        __stcs(out + w, make_double2(__dmul_rn(sD.x, kScale), __dmul_rn(sD.y, kScale)));
        __stcs(out + n + w, make_double2(__dmul_rn(sL.x, kScale), __dmul_rn(sL.y, kScale)));
        __stcs(out + 2 * n + w, make_double2(__dmul_rn(sR.x, kScale), __dmul_rn(sR.y, kScale)));
        __stcs(out + 3 * n + w, make_double2(__dmul_rn(sU.x, kScale), __dmul_rn(sU.y, kScale)));
      }
    }
  }
}

template <int SHIFT, bool MARKED, int T>
int launch_wf_t(qwb_ctx* ctx, cudaStream_t s, int nx, int ny, const double2* in, double2* out,
                const MarkedList& mk) {
  constexpr int OX = 32 - 2 * T;
  const int strips_x = (nx + OX - 1) / OX;
  // strip length: long strips amortise the 2T warm-up rows, but keep >= ~16
  // warps per SM in flight
  int L = env_int("QWB_LATTICE_L", 0);
  if (L <= 0) {
    const long long want = (long long)ctx->num_sms * 16;
    L = 256;
    while (L > 32 && (long long)strips_x * ((ny + L - 1) / L) < want) L /= 2;
  }
  const int strips_y = (ny + L - 1) / L;
  const int nstrips = strips_x * strips_y;
  const int threads = 128;
  const int blocks = (nstrips * 32 + threads - 1) / threads;
  lattice_wf_kernel<SHIFT, MARKED, T><<<blocks, threads, 0, s>>>(nx, ny, in, out, mk, strips_x, nstrips, L);
  return QWB_OK;
}

template <int T>
int launch_wf(qwb_ctx* ctx, int shift, cudaStream_t s, int nx, int ny, const double2* in,
              double2* out, const MarkedList& mk) {
  const bool m = mk.n > 0;
  if (shift == QWB_SHIFT_FLIPFLOP)
    return m ? launch_wf_t<QWB_SHIFT_FLIPFLOP, true, T>(ctx, s, nx, ny, in, out, mk)
             : launch_wf_t<QWB_SHIFT_FLIPFLOP, false, T>(ctx, s, nx, ny, in, out, mk);
  return m ? launch_wf_t<QWB_SHIFT_PERSISTENT, true, T>(ctx, s, nx, ny, in, out, mk)
           : launch_wf_t<QWB_SHIFT_PERSISTENT, false, T>(ctx, s, nx, ny, in, out, mk);
}

}  // namespace

namespace qwb {

// Steps per temporally blocked launch (0 = single-step kernel only).
// QWB_LATTICE_T overrides (0, 2..8); QWB_LATTICE_KIND picks the CTA-tile
// variant (default) or, with "wf", the wavefront variant (opt-in A/B switch);
// QWB_LATTICE_SHAPE the tile shape.
int lattice_kind() {   // 1 = CTA tile (default), 0 = wavefront
  static int kind = -1;
  if (kind < 0) {
    const char* e = getenv("QWB_LATTICE_KIND");
    kind = (e && strcmp(e, "wf") == 0) ? 0 : 1;
  }
  return kind;
}

int lattice_tb_depth(int64_t nx, int64_t ny, int64_t n_marked) {
  static int depth = -1;
  if (depth < 0) {
    depth = env_int("QWB_LATTICE_T", 4);
    if (depth < 0 || depth > 8 || depth == 1) depth = 4;
  }
  if (nx < 64 || ny < 64) return 0;   // tiny lattices: the single-step kernel is launch-bound anyway
  if (lattice_kind() == 0 && n_marked > 8) return 0;   // wavefront takes marked as a short list
  if (lattice_kind() == 1 && depth > 6) return 6;
  return depth;
}

static int tb_launch_impl(qwb_ctx* ctx, int depth, int shift, cudaStream_t s, int nx, int ny, const TbGeo& geo,
                          const double2* in, double2* out, const uint32_t* bits, const int64_t* marked_host,
                          int64_t n_marked, const int64_t* trace_vertices_host, int n_trace, double* trace) {
  if (lattice_kind() == 0) {
    if (!geo.wrap) QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "the wavefront kernel does not run on slabs");
    if (trace) QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "the wavefront kernel does not fuse traces");
    MarkedList mk{};
    mk.n = (int)n_marked;
    for (int k = 0; k < mk.n; ++k) mk.v[k] = marked_host[k];
    switch (depth) {
      case 2: return launch_wf<2>(ctx, shift, s, nx, ny, in, out, mk);
      case 3: return launch_wf<3>(ctx, shift, s, nx, ny, in, out, mk);
      case 4: return launch_wf<4>(ctx, shift, s, nx, ny, in, out, mk);
      case 5: return launch_wf<5>(ctx, shift, s, nx, ny, in, out, mk);
      case 6: return launch_wf<6>(ctx, shift, s, nx, ny, in, out, mk);
      case 7: return launch_wf<7>(ctx, shift, s, nx, ny, in, out, mk);
      case 8: return launch_wf<8>(ctx, shift, s, nx, ny, in, out, mk);
      default: QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "unsupported temporal block depth %d", depth);
    }
  }
  static int shape_env = -1;
  if (shape_env < 0) shape_env = env_int("QWB_LATTICE_SHAPE", 4);
  static int trace_shape = env_int("QWB_LATTICE_TRACE_SHAPE", 4);
  const int shape = trace ? trace_shape : shape_env;
  if (depth > 6) depth = 6;
  MarkedList mk{};
  mk.n = n_marked <= 8 ? (int)n_marked : -1;
  for (int k = 0; k < mk.n; ++k) {
    mk.v[k] = marked_host[k];
    mk.x[k] = (int)(marked_host[k] % nx);
    mk.y[k] = (int)(marked_host[k] / nx);
  }
  TraceList tl{};
  tl.n = trace ? n_trace : 0;
  tl.out = trace;
  for (int k = 0; k < tl.n; ++k) {
    tl.v[k] = trace_vertices_host[k];
    tl.x[k] = (int)(trace_vertices_host[k] % nx);
    tl.y[k] = (int)(trace_vertices_host[k] / nx);
  }
  // shape 4 (default): 32x16 threads, 4 rows each (32x64 region); 3: 32x16
  // threads, 3 rows each (32x48 region; traced launches).  The 32x32 and
  // 24-warp 32x48 shapes measured slower and are not built.
#define QWB_TB_CASE(T_)                                                                        \
  case T_:                                                                                     \
    if (shape == 3) return launch_tb<T_, 16, 3>(ctx, shift, s, nx, ny, geo, in, out, bits, mk, tl); \
    return launch_tb<T_, 16, 4>(ctx, shift, s, nx, ny, geo, in, out, bits, mk, tl);
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
                      const int64_t* trace_vertices_host, int n_trace, double* trace) {
  const TbGeo geo{ny, 0, ny, 0, 1};
  return tb_launch_impl(ctx, depth, shift, s, nx, ny, geo, in, out, bits, marked_host, n_marked,
                        trace_vertices_host, n_trace, trace);
}

int lattice_slab_depth(int depth) {   // the ghost-row depth a slab run can use (0: none)
  return (lattice_kind() == 1 && depth == kSlabDepth && env_int("QWB_LATTICE_SHAPE", 4) == 4) ? depth : 0;
}

int lattice_tb_owned_rows(int depth) {
  if (lattice_kind() != 1 || depth < 2) return 0;
  const int shape = env_int("QWB_LATTICE_SHAPE", 4);
  const int ry = shape == 3 ? 16 * 3 : 16 * 4;
  return ry - 2 * (depth > 6 ? 6 : depth);
}

int lattice_tb_launch_geo(qwb_ctx* ctx, int depth, int shift, cudaStream_t s, int nx, int ny, const TbGeo& geo,
                          const double2* in, double2* out, const uint32_t* bits, const int64_t* marked_host,
                          int64_t n_marked) {
  return tb_launch_impl(ctx, depth, shift, s, nx, ny, geo, in, out, bits, marked_host, n_marked, nullptr, 0,
                        nullptr);
}

}  // namespace qwb

extern "C" int qwb_lattice_fused_depth(int64_t nx, int64_t ny, int64_t n_marked, int* depth_host,
                                       int* kind_host) {
  if (depth_host) *depth_host = qwb::lattice_tb_depth(nx, ny, n_marked);
  if (kind_host) *kind_host = qwb::lattice_kind();
  return QWB_OK;
}
