// lattice_tb.cu — temporally blocked torus walk: T coined steps per HBM pass.
//
// The single-step kernel (lattice.cu) already moves exactly the 32 B per arc
// per step that one application of U needs, and runs at ~96 % of the measured
// HBM copy bandwidth.  The only way past that roofline is to apply U several
// times per trip through HBM.  Each CTA owns a 32 x 32 region of vertices, one
// per thread, with the 4 direction amplitudes in registers:
//
//   * the region's state arrives by cp.async into shared memory (prefetched
//     one tile ahead, so HBM reads overlap the arithmetic of the current tile);
//   * T steps run on chip.  A step is the same per-vertex formula as the
//     single-step kernel (qwb::vertex_outputs — identical arithmetic, so the
//     result stays bitwise equal to the reference); the pushes to x +- 1 go
//     through warp shuffles (a warp is one region row), the pushes to y +- 1
//     through a double-buffered shared-memory exchange (one barrier per step);
//   * values near the region edge go stale one ring per step, so after T steps
//     the inner (32 - 2T)^2 vertices are exact and are written back.
//
// HBM traffic per T steps: 64 B x 32^2 read + 64 B x (32-2T)^2 written per
// tile, i.e. for T = 4 about 11 B per arc-step instead of 32.  Regions wrap
// around the torus (modular global coordinates), so any nx, ny >= 3 works.
#include "qwb_lattice.cuh"

namespace {

using qwb::order_slots;
using qwb::Slots;

constexpr int R = 32;          // region side; blockDim = (32, 32)
constexpr int RR = R * R;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

__device__ __forceinline__ int wrap(int v, int n) {
  v = v < 0 ? v + n : v;
  return v >= n ? v - n : v;
}

__device__ __forceinline__ double2 shfl_down2(double2 v) {
  return make_double2(__shfl_down_sync(0xffffffffu, v.x, 1), __shfl_down_sync(0xffffffffu, v.y, 1));
}
__device__ __forceinline__ double2 shfl_up2(double2 v) {
  return make_double2(__shfl_up_sync(0xffffffffu, v.x, 1), __shfl_up_sync(0xffffffffu, v.y, 1));
}

template <int SHIFT, bool MARKED, int T>
__global__ void __launch_bounds__(RR, 1)
lattice_tb_kernel(int nx, int ny, const double2* __restrict__ in, double2* __restrict__ out,
                  const uint32_t* __restrict__ bits, int tiles_x, int ntiles) {
  constexpr int O = R - 2 * T;   // owned (exact) side
  extern __shared__ double2 sm[];
  double2* stage = sm;            // [4][R][R] next tile's amplitudes
  double2* xD = sm + 4 * RR;      // [2][R][R] O_D exchange
  double2* xU = xD + 2 * RR;      // [2][R][R] O_U exchange
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int me = ty * R + tx;
  const int64_t n = (int64_t)nx * ny;

  int tile = blockIdx.x;
  if (tile >= ntiles) return;
  {
    const int gx = wrap((tile % tiles_x) * O - T + tx, nx);
    const int gy = wrap((tile / tiles_x) * O - T + ty, ny);
    const int64_t w = (int64_t)gy * nx + gx;
#pragma unroll
    for (int p = 0; p < 4; ++p) cp_async16(stage + p * RR + me, in + p * n + w);
    cp_commit();
  }
  for (; tile < ntiles; tile += gridDim.x) {
    const int x0 = (tile % tiles_x) * O, y0 = (tile / tiles_x) * O;
    const int gx = wrap(x0 - T + tx, nx);
    const int gy = wrap(y0 - T + ty, ny);
    cp_wait_all();
    __syncthreads();
    double2 vD = stage[me], vL = stage[RR + me], vR = stage[2 * RR + me], vU = stage[3 * RR + me];
    __syncthreads();
    const int nt = tile + gridDim.x;
    if (nt < ntiles) {
      const int ngx = wrap((nt % tiles_x) * O - T + tx, nx);
      const int ngy = wrap((nt / tiles_x) * O - T + ty, ny);
      const int64_t nw = (int64_t)ngy * nx + ngx;
#pragma unroll
      for (int p = 0; p < 4; ++p) cp_async16(stage + p * RR + me, in + p * n + nw);
    }
    cp_commit();
    bool marked = false;
    if (MARKED) {
      const int64_t wg = (int64_t)gy * nx + gx;
      marked = (__ldg(bits + (wg >> 5)) >> (wg & 31)) & 1u;
    }
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const Slots o = order_slots(gx, gy, nx, ny, vD, vL, vR, vU);
      double2 oD, oL, oR, oU;
      qwb::vertex_outputs(o, marked, vD, vL, vR, vU, oD, oL, oR, oU);
      const int b = (t & 1) * RR;
      xD[b + me] = oD;
      xU[b + me] = oU;
      const double2 fromRight = shfl_down2(oL);   // O_L of (x+1, y)
      const double2 fromLeft = shfl_up2(oR);      // O_R of (x-1, y)
      __syncthreads();
      const double2 fromAbove = (ty < R - 1) ? xD[b + me + R] : oD;   // O_D of (x, y+1)
      const double2 fromBelow = (ty > 0) ? xU[b + me - R] : oU;       // O_U of (x, y-1)
      if (SHIFT == QWB_SHIFT_FLIPFLOP) {
        vU = fromAbove; vD = fromBelow; vR = fromRight; vL = fromLeft;
      } else {
        vD = fromAbove; vU = fromBelow; vL = fromRight; vR = fromLeft;
      }
    }
    if (tx >= T && tx < T + O && ty >= T && ty < T + O && x0 + tx - T < nx && y0 + ty - T < ny) {
      const int64_t w = (int64_t)gy * nx + gx;
      __stcs(out + w, vD);
      __stcs(out + n + w, vL);
      __stcs(out + 2 * n + w, vR);
      __stcs(out + 3 * n + w, vU);
    }
  }
  cp_wait_all();
}

template <int SHIFT, bool MARKED, int T>
int launch_tb_t(qwb_ctx* ctx, cudaStream_t s, int nx, int ny, const double2* in, double2* out,
                const uint32_t* bits) {
  constexpr int O = R - 2 * T;
  const int tiles_x = (nx + O - 1) / O, tiles_y = (ny + O - 1) / O;
  const int ntiles = tiles_x * tiles_y;
  const size_t smem = (4 + 4) * RR * sizeof(double2);
  static bool configured[256] = {};   // per instantiation and device
  const int dev = ctx->device & 255;
  if (!configured[dev]) {
    cudaError_t e = cudaFuncSetAttribute(lattice_tb_kernel<SHIFT, MARKED, T>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return qwb::cuda_status(ctx, e, "cudaFuncSetAttribute(lattice_tb)");
    configured[dev] = true;
  }
  const int grid = ntiles < ctx->num_sms ? ntiles : ctx->num_sms;
  lattice_tb_kernel<SHIFT, MARKED, T><<<grid, dim3(R, R), smem, s>>>(nx, ny, in, out, bits, tiles_x, ntiles);
  return QWB_OK;
}

template <int T>
int launch_tb(qwb_ctx* ctx, int shift, cudaStream_t s, int nx, int ny, const double2* in, double2* out,
              const uint32_t* bits) {
  if (shift == QWB_SHIFT_FLIPFLOP) {
    return bits ? launch_tb_t<QWB_SHIFT_FLIPFLOP, true, T>(ctx, s, nx, ny, in, out, bits)
                : launch_tb_t<QWB_SHIFT_FLIPFLOP, false, T>(ctx, s, nx, ny, in, out, bits);
  }
  return bits ? launch_tb_t<QWB_SHIFT_PERSISTENT, true, T>(ctx, s, nx, ny, in, out, bits)
              : launch_tb_t<QWB_SHIFT_PERSISTENT, false, T>(ctx, s, nx, ny, in, out, bits);
}

}  // namespace

namespace qwb {

// steps per temporally blocked launch (0 = not available); 2, 4, 6 or 8
int lattice_tb_depth(int64_t nx, int64_t ny) {
  static int depth = -1;
  if (depth < 0) {
    const char* e = getenv("QWB_LATTICE_T");
    depth = e ? atoi(e) : 4;
    if (depth != 0 && depth != 2 && depth != 4 && depth != 6 && depth != 8) depth = 4;
  }
  if (nx < 64 || ny < 64) return 0;   // tiny lattices: the single-step kernel is launch-bound anyway
  return depth;
}

int lattice_tb_launch(qwb_ctx* ctx, int depth, int shift, cudaStream_t s, int nx, int ny,
                      const double2* in, double2* out, const uint32_t* bits) {
  switch (depth) {
    case 2: return launch_tb<2>(ctx, shift, s, nx, ny, in, out, bits);
    case 4: return launch_tb<4>(ctx, shift, s, nx, ny, in, out, bits);
    case 6: return launch_tb<6>(ctx, shift, s, nx, ny, in, out, bits);
    case 8: return launch_tb<8>(ctx, shift, s, nx, ny, in, out, bits);
    default: QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "unsupported temporal block depth %d", depth);
  }
}

}  // namespace qwb
