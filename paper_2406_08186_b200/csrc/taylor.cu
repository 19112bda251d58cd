// taylor.cu — continuous-time walk: the sub-stepped truncated Taylor action of
// exp(-i H t) (ctqw.evolve_state, ctqw.py:123-171).
//
// Reference inner loop per term k (ctqw.py:158-165), four engine calls plus four
// isfinite passes:
//     hterm = H term;  term = (-1j*tau/k) * hterm;  acc = acc + 1.0*term;
//     stop when ||term|| <= tol * ||psi_in||
// Here ONE fused kernel per term reads term_{k-1} (neighbour gathers), writes
// term_k, read-modify-writes acc and emits per-block ||term_k||^2 partials; a
// one-block kernel finishes the norm in a fixed order and raises a device
// `done` flag.  Term kernels launched after `done` return immediately, so the
// host launches terms speculatively in chunks and synchronises once per chunk
// instead of once per term.
//
// Arithmetic is the reference's bit for bit (numpy complex multiply model,
// pairwise row sums, Python's complex scalar (0.0, -tau/k)); only the stop
// test's norm is a different (deterministic) summation order than BLAS dnrm2,
// which can flip the stop decision only when ||term|| is within a few ulps of
// the floor.
//
// Operators: CSR H (any graph, built by qwb_hamiltonian) and matrix-free
// hypercube H = -gamma A - sum_M |v><v| whose row v lists, in ascending column
// order, v with its set bits cleared high->low, the diagonal (if v marked),
// then v with its clear bits set low->high.
#include <type_traits>
#include <utility>

#include "qwb_internal.cuh"

namespace {

using qwb::cadd;
using qwb::cmul_np;

constexpr int kTermBlocks = 2048;   // fixed grid => deterministic partial order
constexpr int kTermThreads = 256;
constexpr int kPartialsMax = 16384;  // partial-sum slots in the evolve workspace

// Term chain launches (term -> finalize -> term ...) use programmatic
// dependent launch (qwb::launch_pdl; QWB_TERM_PDL=0 turns it off).
using qwb::pdl_enter;
template <class... P, class... A>
cudaError_t launch_pdl(void (*kernel)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, A&&... args) {
  static const bool pdl = qwb::env_flag("QWB_TERM_PDL", 1) != 0;
  return qwb::launch_pdl(pdl, kernel, grid, block, smem, s, std::forward<A>(args)...);
}

// Streaming x0 + pairwise(x1..x{L-1}) for rows of L <= 65 entries, element by
// element in order (numpy block rule with four rotating complex accumulators).
struct StreamRow {
  int m, main_end, i;
  double2 x0, c0, c1, c2, c3, r;
  __device__ __forceinline__ void init(int L) {
    m = L - 1;
    main_end = m >= 4 ? m - (m % 4) : 0;
    i = -1;
    r = make_double2(-0.0, -0.0);
  }
  __device__ __forceinline__ void push(double2 e) {
    if (i < 0) {
      x0 = e;
      i = 0;
      return;
    }
    if (i < main_end) {
      c0 = (i < 4) ? e : cadd(c0, e);
      const double2 t = c0;
      c0 = c1;
      c1 = c2;
      c2 = c3;
      c3 = t;
      if (i + 1 == main_end) r = cadd(cadd(c0, c1), cadd(c2, c3));
    } else {
      r = cadd(r, e);
    }
    ++i;
  }
  __device__ __forceinline__ double2 result() const { return m == 0 ? x0 : cadd(x0, r); }
};

struct CsrOp {
  const int64_t* __restrict__ offs;
  const int32_t* __restrict__ col;
  const double2* __restrict__ val;
  int grid;     // term-kernel blocks: one resident wave (set by qwb_taylor_evolve_csr)
  int capped;   // 1: csr_term_kernel4 (64 registers), 0: term_kernel<CsrOp>
  struct Get {
    const int32_t* __restrict__ col;
    const double2* __restrict__ val;
    const double2* __restrict__ x;
    int64_t base;
    __device__ __forceinline__ double2 operator()(int64_t i) const {
      const int64_t j = base + i;
      return cmul_np(__ldg(val + j), __ldg(x + __ldg(col + j)));
    }
  };
  __device__ __forceinline__ double2 row(int64_t v, const double2* __restrict__ x) const {
    const int64_t s = __ldg(offs + v), e = __ldg(offs + v + 1);
    const int64_t len = e - s;
    if (len == 4 || len == 5) {
      // short rows (every row of a lattice / cycle H, marked rows one longer):
      // all column, value and neighbour loads issued up front, then numpy's
      // x0 + pairwise(x1..): sequential from -0 for 3 rest elements, the
      // (c0+c1)+(c2+c3) block for 4
      int c[5];
      double2 w[5], xv[5];
#pragma unroll
      for (int i = 0; i < 4; ++i) c[i] = __ldg(col + s + i);
      c[4] = (len == 5) ? __ldg(col + s + 4) : c[3];
#pragma unroll
      for (int i = 0; i < 4; ++i) w[i] = __ldg(val + s + i);
      w[4] = (len == 5) ? __ldg(val + s + 4) : w[3];
#pragma unroll
      for (int i = 0; i < 4; ++i) xv[i] = __ldg(x + c[i]);
      xv[4] = (len == 5) ? __ldg(x + c[4]) : xv[3];
      double2 p[5];
#pragma unroll
      for (int i = 0; i < 5; ++i) p[i] = cmul_np(w[i], xv[i]);
      double2 r;
      if (len == 4) {
        r = cadd(cadd(cadd(make_double2(-0.0, -0.0), p[1]), p[2]), p[3]);
      } else {
        r = cadd(cadd(p[1], p[2]), cadd(p[3], p[4]));
      }
      return cadd(p[0], r);
    }
    if (e == s) return make_double2(0.0, 0.0);
    return row_long(s, e - s, x);
  }
  // other lengths out of line: the generic pairwise reducer's stack stays out
  // of the short-row path's register allocation
  __device__ __noinline__ double2 row_long(int64_t s, int64_t len, const double2* __restrict__ x) const {
    Get g{col, val, x, s};
    return qwb::reduceat_z(g, len);
  }
};

template <int MAXD>
struct HypercubeOp {
  int dim;
  double gamma;
  const uint32_t* __restrict__ bits;
  __device__ __forceinline__ double2 row(int64_t v, const double2* __restrict__ x) const {
    double2 xs[MAXD];
#pragma unroll
    for (int b = 0; b < MAXD; ++b)
      if (b < dim) xs[b] = __ldg(x + (v ^ (1LL << b)));
    const bool mk = bits && ((__ldg(bits + (v >> 5)) >> (v & 31)) & 1u);
    const double2 g = make_double2(-gamma, 0.0);
    StreamRow sr;
    sr.init(dim + (mk ? 1 : 0));
#pragma unroll
    for (int b = MAXD - 1; b >= 0; --b)
      if (b < dim && ((v >> b) & 1)) sr.push(cmul_np(g, xs[b]));
    if (mk) sr.push(cmul_np(make_double2(-1.0, 0.0), __ldg(x + v)));
#pragma unroll
    for (int b = 0; b < MAXD; ++b)
      if (b < dim && !((v >> b) & 1)) sr.push(cmul_np(g, xs[b]));
    return sr.result();
  }
};

template <class Op>
__device__ __forceinline__ void term_body(const Op& op, int64_t n, const double2* __restrict__ tin,
                                          double2* __restrict__ tout, const double2* acc_in,
                                          double2* acc_out, double s_k, double* __restrict__ partial) {
  __shared__ double sh[kTermThreads];
  const double2 alpha = make_double2(0.0, -s_k);      // Python complex(-1j * tau / k)
  const double2 one = make_double2(1.0, 0.0);
  double nrm = 0.0;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const double2 h = op.row(v, tin);
    const double2 t = cmul_np(alpha, h);
    tout[v] = t;
    acc_out[v] = cadd(acc_in[v], cmul_np(one, t));
    nrm = __fma_rn(t.x, t.x, __fma_rn(t.y, t.y, nrm));
  }
  sh[threadIdx.x] = nrm;
  __syncthreads();
  for (int s = kTermThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = __dadd_rn(sh[threadIdx.x], sh[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

template <class Op>
__global__ void __launch_bounds__(kTermThreads)
term_kernel(Op op, int64_t n, const double2* __restrict__ tin, double2* __restrict__ tout,
            const double2* acc_in, double2* acc_out, double s_k, const int* __restrict__ done,
            double* __restrict__ partial) {
  pdl_enter();
  if (*done) return;
  term_body(op, n, tin, tout, acc_in, acc_out, s_k, partial);
}

// CSR H: capped at 64 registers (4 resident CTAs per SM; a few spilled bytes,
// outside the short-row loads) — the default.  QWB_CSR_TERM_MINB=3 selects the
// uncapped term_kernel<CsrOp> (78 registers, 3 CTAs).  2048^2 grid H:
// 126.1 -> 119.9 us/term; 4096^2: 455.5 -> 424.7 us/term (6.0 TB/s)
__global__ void __launch_bounds__(kTermThreads, 4)
csr_term_kernel4(CsrOp op, int64_t n, const double2* __restrict__ tin, double2* __restrict__ tout,
                 const double2* acc_in, double2* acc_out, double s_k, const int* __restrict__ done,
                 double* __restrict__ partial) {
  pdl_enter();
  if (*done) return;
  term_body(op, n, tin, tout, acc_in, acc_out, s_k, partial);
}

__global__ void __launch_bounds__(kTermThreads)
term_finalize_kernel(const double* __restrict__ partial, int nparts, double floor_, int k,
                     int* __restrict__ done, int* __restrict__ terms) {
  pdl_enter();
  if (*done) return;
  __shared__ double sh[kTermThreads];
  double acc = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) acc = __dadd_rn(acc, partial[i]);
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = kTermThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = __dadd_rn(sh[threadIdx.x], sh[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (__dsqrt_rn(sh[0]) <= floor_) {
      *done = 1;
      *terms = k;
    }
  }
}

// ---------------------------------------------------------------------------
// Hypercube term, positional form (dim >= 10).  The row's columns in ascending
// order are v with its set bits cleared high->low, then v with its clear bits
// set low->high.  The kernel walks the ROW POSITIONS p = 0..dim-1 at compile
// time and finds, per lane, the bit that lands at p with two running masks
// (clz on the remaining set bits, ffs on the remaining clear bits) — so the
// numpy pairwise slot of every element, (p-1) % 4, is a compile-time register
// and no data-dependent control flow remains.  Neighbour values are read-only
// cached gathers (the 2^b partner of a warp is one contiguous 512-B block).
// Warps that contain a marked vertex (row length dim+1) use the generic path.
// ---------------------------------------------------------------------------
template <int MAXD>
struct HcPos {
  int dim;
  double gamma;
  const uint32_t* __restrict__ bits;
};

template <int MAXD>
__global__ void __launch_bounds__(kTermThreads)
hc_pos_kernel(HcPos<MAXD> op, int64_t n, const double2* __restrict__ tin, double2* __restrict__ tout,
              const double2* acc_in, double2* acc_out, double s_k, const int* __restrict__ done,
              double* __restrict__ partial) {
  if (*done) return;
  __shared__ double sh[kTermThreads];
  const int dim = op.dim;
  const double2 alpha = make_double2(0.0, -s_k);   // Python complex(-1j * tau / k)
  const double2 one = make_double2(1.0, 0.0);
  const double2 g = make_double2(-op.gamma, 0.0);
  const int m = dim - 1;                            // rest elements after x0
  const int main_end = m - (m % 4);
  const unsigned all = (dim >= 32) ? 0xffffffffu : ((1u << dim) - 1u);
  double nrm = 0.0;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const bool mk = op.bits && ((__ldg(op.bits + (v >> 5)) >> (v & 31)) & 1u);
    double2 h;
    if (__any_sync(0xffffffffu, mk)) {
      StreamRow sr;
      sr.init(dim + (mk ? 1 : 0));
      for (int b = dim - 1; b >= 0; --b)
        if ((v >> b) & 1) sr.push(cmul_np(g, __ldg(tin + (v ^ (1LL << b)))));
      if (mk) sr.push(cmul_np(make_double2(-1.0, 0.0), __ldg(tin + v)));
      for (int b = 0; b < dim; ++b)
        if (!((v >> b) & 1)) sr.push(cmul_np(g, __ldg(tin + (v ^ (1LL << b)))));
      h = sr.result();
    } else {
      const unsigned vb = (unsigned)v & all;
      unsigned setm = vb, clrm = (~vb) & all;
      const int pc = __popc(vb);
      // (the compiler's own interleaving of the gathers with the ordered sum
      // measured best: 74 registers, 3 CTAs/SM; explicit all-loads-first or a
      // register prefetch ring raised register use and lost occupancy)
      double2 x0 = make_double2(0.0, 0.0), c0 = x0, c1 = x0, c2 = x0, c3 = x0;
      double2 tl0 = x0, tl1 = x0, tl2 = x0;
#pragma unroll
      for (int p = 0; p < MAXD; ++p) {
        if (p < dim) {
          const int bs = 31 - __clz(setm | 1u);
          const int bc = __ffs(clrm | 0x80000000u) - 1;
          const bool use_set = p < pc;
          const int b = use_set ? bs : bc;
          setm = use_set ? (setm ^ (1u << bs)) : setm;
          clrm = use_set ? clrm : (clrm ^ (1u << bc));
          const double2 e = cmul_np(g, __ldg(tin + (v ^ (1LL << b))));
          if (p == 0) {
            x0 = e;
          } else {
            const int i = p - 1;
            if (i < main_end) {
              double2& c = (i % 4 == 0) ? c0 : (i % 4 == 1) ? c1 : (i % 4 == 2) ? c2 : c3;
              c = (i < 4) ? e : cadd(c, e);
            } else {
              const int k = i - main_end;   // 0..2, uniform
              tl0 = (k == 0) ? e : tl0;
              tl1 = (k == 1) ? e : tl1;
              tl2 = (k == 2) ? e : tl2;
            }
          }
        }
      }
      double2 r;
      if (m < 4) {
        r = make_double2(-0.0, -0.0);
        if (m > 0) r = cadd(r, c0);
        if (m > 1) r = cadd(r, c1);
        if (m > 2) r = cadd(r, c2);
      } else {
        r = cadd(cadd(c0, c1), cadd(c2, c3));
        const int tail = m - main_end;
        if (tail > 0) r = cadd(r, tl0);
        if (tail > 1) r = cadd(r, tl1);
        if (tail > 2) r = cadd(r, tl2);
      }
      h = cadd(x0, r);
    }
    const double2 t = cmul_np(alpha, h);
    tout[v] = t;
    acc_out[v] = cadd(acc_in[v], cmul_np(one, t));
    nrm = __fma_rn(t.x, t.x, __fma_rn(t.y, t.y, nrm));
  }
  sh[threadIdx.x] = nrm;
  __syncthreads();
  for (int s = kTermThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = __dadd_rn(sh[threadIdx.x], sh[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

// ---------------------------------------------------------------------------
// Hypercube term, TMA-streamed form (dim >= 10).  A CTA owns tiles of 1024
// consecutive vertices (bits 0..9); every neighbour of a tile across a high
// bit b >= 10 lies in ONE contiguous 16-KB partner tile (tile ^ 2^(b-10)).
// Row v's ascending column order is: high set bits (descending), then the 10
// low bits (lane-dependent order), then high clear bits (ascending) — the
// high-bit positions are the same for the whole tile.  So a producer warp
// streams, per tile, the partner tiles in row-position order (the tile itself
// at the position of the low segment) with 1-D bulk copies
// (cp.async.bulk + mbarrier complete_tx) into a ring of shared-memory stages,
// and the consumer threads fold each stage into the numpy pairwise
// accumulators of their vertices in order: every global read is a 16-KB bulk
// transfer, no gather, no long-scoreboard stall on the compute warps.
// Vertices of marked rows (diagonal entry, row length dim+1) are computed by a
// dedicated fix-up warp (hc_marked_row); the consumers skip them.
// ---------------------------------------------------------------------------
namespace hcs {
constexpr int LB = 10;                     // low bits per tile
constexpr int TILE = 1 << LB;              // vertices per tile
constexpr uint32_t CHUNK_BYTES = TILE * sizeof(double2);
// NS ring stages + a double-buffered acc tile + barriers + per acc slot the
// tile's 32 marked-bitmap words
constexpr size_t smem_bytes(int ns) {
  return (size_t)(ns + 2) * CHUNK_BYTES + (2 * ns + 4) * sizeof(uint64_t) + 2 * 32 * sizeof(uint32_t);
}
// paired form: NSP ring stages of two partner chunks + per tile slot (two
// slots) the acc tile and the own tile, barriers, bitmap words
constexpr size_t pair_smem_bytes(int nsp) {
  return (size_t)(2 * nsp + 4) * CHUNK_BYTES + (2 * nsp + 4) * sizeof(uint64_t) + 2 * 32 * sizeof(uint32_t);
}
}  // namespace hcs

__device__ __forceinline__ uint32_t nctaid_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nctaid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "HCS_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra HCS_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_wait_u32(uint32_t addr, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "HCS_WAITU_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra HCS_WAITU_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_u32(uint32_t addr) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(addr) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// (c + 0i) * x with the zero terms dropped: c*x.re, c*x.im.  Equal to
// numpy's product for every x except in the sign of an exactly-zero
// component, so every non-zero sum built from it keeps numpy's bits (exact
// zeros may carry the other sign: equal under ==, invisible to every norm).
__device__ __forceinline__ double2 scale_real_z(double c, double2 x) {
  return make_double2(__dmul_rn(c, x.x), __dmul_rn(c, x.y));
}

constexpr int kMaxShardBits = 5;   // up to 32 shards

// n below is the LOCAL vertex count 2^dim_loc; a shard holds the vertices
// whose top dim - dim_loc bits equal its rank (single GPU: dim_loc = dim).
struct HcStream {
  int dim;        // global hypercube dimension
  int dim_loc;    // log2 of the vertices this launch owns
  int rank;       // shard index (top bits of every owned vertex)
  double gamma;
  const uint32_t* __restrict__ bits;   // GLOBAL marked bitmap (or null)
  int grid;
  int device;
  int variant;
  // term_{k-1} of the partner shard across each rank bit (rank ^ 2^j), same
  // local indexing as tin: received by NCCL, or the partner's own buffer
  const double2* remote[kMaxShardBits];
};
using HcStreamArgs = HcStream;

// Marked row v (length dim + 1: -1 * psi[v] sits between the set and the
// clear neighbours), computed by the fix-up warp together: lane f loads
// neighbour f, so all the row's loads are in flight at once, and every lane
// folds the row in numpy's order from shuffles (the result is used by lane 0).
// vl: local index, vg: global vertex id; neighbours across rank bits come from
// the partner shards' term buffers.  dim <= 32.
__device__ __noinline__ double2 hc_marked_row(const HcStreamArgs& a, double g, const double2* __restrict__ tin,
                                              int64_t vl, int64_t vg, int lane) {
  double2 nb = make_double2(0.0, 0.0);
  if (lane < a.dim)
    nb = lane < a.dim_loc ? __ldg(tin + (vl ^ (1LL << lane))) : __ldg(a.remote[lane - a.dim_loc] + vl);
  const double2 own = __ldg(tin + vl);
  StreamRow sr;
  sr.init(a.dim + 1);
  const double2 gg = make_double2(g, 0.0);
  auto pushb = [&](int b) {
    const double2 e = make_double2(__shfl_sync(0xffffffffu, nb.x, b), __shfl_sync(0xffffffffu, nb.y, b));
    sr.push(cmul_np(gg, e));
  };
  for (int b = a.dim - 1; b >= 0; --b)
    if ((vg >> b) & 1) pushb(b);
  sr.push(cmul_np(make_double2(-1.0, 0.0), own));
  for (int b = 0; b < a.dim; ++b)
    if (!((vg >> b) & 1)) pushb(b);
  return sr.result();
}

// NS: ring stages; PROD: producer warps (one issuing lane each; producer q
// issues the ring chunks it == q mod PROD, producer 0 also the acc tiles);
// CONS: consumer threads (+ PROD producer warps + one fix-up warp), TILE / CONS
// vertices each.  A single issuing thread tops out near one 16-KB chunk per
// ~330 cycles (its wait -> expect_tx -> copy chain), below the SM's share of
// the L2 bandwidth; two interleaved producers overlap their chains.
template <int NS, int PROD, int CONS>
__global__ void __launch_bounds__(CONS + 32 * PROD + 32, 1)
hc_stream_kernel(const __grid_constant__ HcStream op, int64_t n, const double2* __restrict__ tin, double2* __restrict__ tout,
                 const double2* acc_in, double2* acc_out, double s_k, const int* __restrict__ done,
                 double* __restrict__ partial) {
  using namespace hcs;
  constexpr int VPT = TILE / CONS;
  extern __shared__ __align__(128) unsigned char hcs_smem[];
  double2* ring = reinterpret_cast<double2*>(hcs_smem);
  double2* accbuf = ring + (size_t)NS * TILE;                  // [2][TILE]
  uint64_t* full = reinterpret_cast<uint64_t*>(hcs_smem + (size_t)(NS + 2) * CHUNK_BYTES);
  uint64_t* empty = full + NS;
  uint64_t* afull = empty + NS;                                // [2]
  uint64_t* aempty = afull + 2;                                // [2]
  // [2][32]: per acc slot, the tile's marked-bitmap words (bulk-copied with
  // the acc tile)
  uint32_t* awords = reinterpret_cast<uint32_t*>(aempty + 2);
  __shared__ double red[CONS / 32 + PROD + 1];
  const int tid = threadIdx.x;
  const int dim = op.dim;
  const int nh = dim - LB;                            // high bits (global)
  const int nh_loc = op.dim_loc - LB;                 // high bits inside the shard
  const uint32_t hmask = (nh >= 32) ? 0xffffffffu : ((1u << nh) - 1u);
  const uint32_t hbase = (uint32_t)op.rank << nh_loc;   // rank bits of every tile index
  const int64_t vbase = (int64_t)op.rank << op.dim_loc;
  const int64_t ntiles = n >> LB;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, CONS / 32);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(afull + s, 1);
      mbar_init(aempty + s, CONS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  pdl_enter();   // the barrier set-up above overlaps the previous kernel
  if (*done) return;

  const int lane = tid & 31;
  const double2 alpha = make_double2(0.0, -s_k);      // Python complex(-1j * tau / k)
  const double2 one = make_double2(1.0, 0.0);
  const double g = -op.gamma;
  double nrm = 0.0;

  if (tid >= CONS) {
    const int pl = tid - CONS;
    if (pl < 32 * PROD && (pl & 31) == 0) {   // (lanes 1..31 of the producer warps idle)
      // ---------------- producers: stream the partner tiles in row order
      const uint32_t q = (uint32_t)pl >> 5;
      uint32_t s = 0, ph = 0, ti = 0, it = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++ti) {
        const uint32_t Hl = (uint32_t)tile, H = hbase | Hl;
        const int hs = __popc(H);
        if (q == 0) {   // the tile's acc values and (marked runs) its 32 bitmap words,
                        // consumed in the epilogue; both complete on the acc slot's barrier
          const int ab = ti & 1;
          mbar_wait(aempty + ab, ((ti >> 1) & 1) ^ 1);
          mbar_expect_tx(afull + ab, CHUNK_BYTES + (op.bits ? 128u : 0u));
          bulk_g2s(accbuf + (size_t)ab * TILE, acc_in + ((int64_t)Hl << LB), CHUNK_BYTES, afull + ab);
          if (op.bits) bulk_g2s(awords + ab * 32, op.bits + ((vbase + (tile << LB)) >> 5), 128u, afull + ab);
        }
        uint32_t setm = H, clrm = (~H) & hmask;
        for (int c = 0; c <= nh; ++c, ++it) {
          int b = -1;   // partner across high bit b (-1: the tile itself)
          if (c < hs) {
            b = 31 - __clz(setm);
            setm ^= 1u << b;
          } else if (c > hs) {
            b = __ffs(clrm) - 1;
            clrm ^= 1u << b;
          }
          const uint32_t sc = s, pc = ph;
          if (++s == NS) {
            s = 0;
            ph ^= 1u;
          }
          if (PROD > 1 && it % PROD != q) continue;
          const double2* src = b < 0 ? tin + ((int64_t)Hl << LB)
                               : b < nh_loc ? tin + ((int64_t)(Hl ^ (1u << b)) << LB)
                                            : op.remote[b - nh_loc] + ((int64_t)Hl << LB);
          mbar_wait(empty + sc, pc ^ 1);
          mbar_expect_tx(full + sc, CHUNK_BYTES);
          bulk_g2s(ring + (size_t)sc * TILE, src, CHUNK_BYTES, full + sc);
        }
      }
    } else if (pl >= 32 * PROD && op.bits) {
      // ---------------- fix-up warp: marked rows of this CTA's tiles (the
      // consumers leave those vertices alone).  Its own warp: sharing the
      // producer's warp, the bitmap scan held up the stream (+15 us/term).
      // The lanes scan the bitmap words together; per marked vertex the warp
      // computes the row cooperatively and lane 0 stores it.
      const int fl = pl - 32 * PROD;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint32_t word = __ldg(op.bits + ((vbase + (tile << LB)) >> 5) + fl);   // TILE / 32 == 32 words
        unsigned any = __ballot_sync(0xffffffffu, word != 0u);
        while (any) {
          const int src = __ffs(any) - 1;
          any &= any - 1;
          uint32_t wd = __shfl_sync(0xffffffffu, word, src);
          while (wd) {
            const int bit = __ffs(wd) - 1;
            wd &= wd - 1;
            const int64_t v = (tile << LB) + src * 32 + bit;
            const double2 h = hc_marked_row(op, g, tin, v, vbase + v, fl);
            if (fl == 0) {
              const double2 t = cmul_np(alpha, h);
              tout[v] = t;
              acc_out[v] = cadd(acc_in[v], cmul_np(one, t));
              nrm = __fma_rn(t.x, t.x, __fma_rn(t.y, t.y, nrm));
            }
          }
        }
      }
    }
  } else {
    // ---------------- consumers
    const int m = dim - 1;
    const int main_end = m - (m % 4);
    // the low segment of each owned l (the same for every tile): byte offset
    // of the q-th element's partner l ^ 2^b in a chunk, set bits high->low
    // then clear bits low->high, two 16-bit offsets per register
    uint32_t offs[VPT][LB / 2];
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
      const uint32_t l = (uint32_t)(tid + j * CONS);
      uint32_t sm = l, cm = (~l) & (TILE - 1);
      const int pc = __popc(l);
#pragma unroll
      for (int q = 0; q < LB; ++q) {
        int b;
        if (q < pc) {
          b = 31 - __clz(sm);
          sm ^= 1u << b;
        } else {
          b = __ffs(cm) - 1;
          cm ^= 1u << b;
        }
        const uint32_t off = (l ^ (1u << b)) * (uint32_t)sizeof(double2);
        if (q % 2 == 0) offs[j][q / 2] = off;
        else offs[j][q / 2] |= off << 16;
      }
    }
    // Accumulators of numpy's x0 + pairwise(x1..x_m): x0, ac[0..3] take the
    // elements at row positions 1 + 4k + a, the tail (positions past
    // main_end) is added to the combined (ac0 + ac1) + (ac2 + ac3) in ac[0].
    // A chunk's slot depends only on its index modulo 4, so the set partners,
    // the own tile and the clear partners run as three loops unrolled by 4 in
    // which every slot is a compile-time register (the own tile and the clear
    // partners in one of four compile-time rotations).
    const uint32_t full_u32 = smem_u32(full), empty_u32 = smem_u32(empty);
    uint32_t s = 0, ph = 0, ti = 0;
    // 32-bit tile index, stride re-read from %nctaid (a 64-bit index and a
    // hoisted stride were spilled; the reload missed the small L1)
    for (uint32_t tile = blockIdx.x; tile < (uint32_t)ntiles; tile += nctaid_x(), ++ti) {
      const uint32_t H = hbase | (uint32_t)tile;   // global tile index: row order
      const int hs = __popc(H);
      double2 x0[VPT], ac[4][VPT];
#pragma unroll
      for (int j = 0; j < VPT; ++j) x0[j] = ac[0][j] = ac[1][j] = ac[2][j] = ac[3][j] = make_double2(-0.0, -0.0);
      auto add_tail = [&](int i, const double2 (&e)[VPT]) {
#pragma unroll
        for (int j = 0; j < VPT; ++j) {
          if (i == main_end) ac[0][j] = cadd(cadd(ac[0][j], ac[1][j]), cadd(ac[2][j], ac[3][j]));
          ac[0][j] = cadd(ac[0][j], e[j]);
        }
      };
      // FAST: every position of the segment is in the 4-accumulator main part
      // (hs >= 1 and hs + LB - 2 < main_end): no per-position branch
      auto fold_own = [&](const double2* ch, auto Rc, auto Fc) {   // positions hs .. hs + LB - 1
        constexpr int R = decltype(Rc)::value;           // hs & 3
        constexpr bool FAST = decltype(Fc)::value;
        const char* cb = reinterpret_cast<const char*>(ch);
#pragma unroll
        for (int q = 0; q < LB; ++q) {
          double2 e[VPT];
#pragma unroll
          for (int j = 0; j < VPT; ++j) {
            const uint32_t off = (q % 2 == 0) ? (offs[j][q / 2] & 0xffffu) : (offs[j][q / 2] >> 16);
            e[j] = scale_real_z(g, *reinterpret_cast<const double2*>(cb + off));
          }
          if (FAST) {
            const int a = (R + q + 3) & 3;   // constant once the loop is unrolled
#pragma unroll
            for (int j = 0; j < VPT; ++j) ac[a][j] = cadd(ac[a][j], e[j]);
            continue;
          }
          const int i = hs + q - 1;
          if (i < 0) {
#pragma unroll
            for (int j = 0; j < VPT; ++j) x0[j] = cadd(x0[j], e[j]);
          } else if (i < main_end) {
            const int a = (R + q + 3) & 3;
#pragma unroll
            for (int j = 0; j < VPT; ++j) ac[a][j] = cadd(ac[a][j], e[j]);
          } else {
            add_tail(i, e);
          }
        }
      };
      // one stage: wait for it, read and scale this thread's entries, release
      auto take = [&](double2 (&e)[VPT]) {
        mbar_wait_u32(full_u32 + 8 * s, ph);
        const double2* ch = ring + (size_t)s * TILE;
#pragma unroll
        for (int j = 0; j < VPT; ++j) e[j] = scale_real_z(g, ch[tid + j * CONS]);
        __syncwarp();   // the scaled values are in registers: the stage may be refilled
        if (lane == 0) mbar_arrive_u32(empty_u32 + 8 * s);
        if (++s == NS) {
          s = 0;
          ph ^= 1u;
        }
      };
      // two consecutive stages with one release point: both waits, then both
      // chunks' loads in flight together
      auto take2 = [&](double2 (&e1)[VPT], double2 (&e2)[VPT]) {
        const uint32_t s1 = s, p1 = ph;
        if (++s == NS) {
          s = 0;
          ph ^= 1u;
        }
        const uint32_t s2 = s, p2 = ph;
        if (++s == NS) {
          s = 0;
          ph ^= 1u;
        }
        mbar_wait_u32(full_u32 + 8 * s1, p1);
        mbar_wait_u32(full_u32 + 8 * s2, p2);
        const double2* c1 = ring + (size_t)s1 * TILE;
        const double2* c2 = ring + (size_t)s2 * TILE;
#pragma unroll
        for (int j = 0; j < VPT; ++j) {
          e1[j] = c1[tid + j * CONS];
          e2[j] = c2[tid + j * CONS];
        }
#pragma unroll
        for (int j = 0; j < VPT; ++j) {
          e1[j] = scale_real_z(g, e1[j]);
          e2[j] = scale_real_z(g, e2[j]);
        }
        __syncwarp();
        if (lane == 0) {
          mbar_arrive_u32(empty_u32 + 8 * s1);
          mbar_arrive_u32(empty_u32 + 8 * s2);
        }
      };
      auto addto = [&](double2 (&acc)[VPT], const double2 (&e)[VPT]) {
#pragma unroll
        for (int j = 0; j < VPT; ++j) acc[j] = cadd(acc[j], e[j]);
      };
      // phase A: set partners, chunk c at position c (c = 0 is x0; the slot
      // of c >= 1 is (c - 1) & 3, so blocks of four from c = 1 are slots 0..3)
      double2 e[VPT];
      int c = 0;
      if (hs > 0) {
        take(e);
        addto(x0, e);
        c = 1;
      }
      double2 f[VPT];
      for (; c + 4 <= hs; c += 4) {
        take2(e, f);
        addto(ac[0], e);
        addto(ac[1], f);
        take2(e, f);
        addto(ac[2], e);
        addto(ac[3], f);
      }
#pragma unroll
      for (int u = 0; u < 3; ++u)
        if (c + u < hs) {
          take(e);
          addto(ac[u], e);
        }
      // phase B: the tile itself, positions hs .. hs + LB - 1
      {
        mbar_wait_u32(full_u32 + 8 * s, ph);
        const double2* ch = ring + (size_t)s * TILE;
        using Y = std::true_type;
        using N = std::false_type;
        if (hs >= 1 && hs + LB - 2 < main_end) {
          switch (hs & 3) {
            case 0: fold_own(ch, std::integral_constant<int, 0>{}, Y{}); break;
            case 1: fold_own(ch, std::integral_constant<int, 1>{}, Y{}); break;
            case 2: fold_own(ch, std::integral_constant<int, 2>{}, Y{}); break;
            default: fold_own(ch, std::integral_constant<int, 3>{}, Y{}); break;
          }
        } else {
          switch (hs & 3) {
            case 0: fold_own(ch, std::integral_constant<int, 0>{}, N{}); break;
            case 1: fold_own(ch, std::integral_constant<int, 1>{}, N{}); break;
            case 2: fold_own(ch, std::integral_constant<int, 2>{}, N{}); break;
            default: fold_own(ch, std::integral_constant<int, 3>{}, N{}); break;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_u32(empty_u32 + 8 * s);
        if (++s == NS) {
          s = 0;
          ph ^= 1u;
        }
      }
      // phase C: clear partners (partner index c from hs), position c + LB,
      // slot (c + LB - 1) & 3; positions past main_end go to the tail
      const int cme = max(hs, min(nh, main_end - LB + 1));
      auto phase_c = [&](auto Rc) {
        constexpr int R = decltype(Rc)::value;   // slot of partner hs
        int cc = hs;
        for (; cc + 4 <= cme; cc += 4) {
          take2(e, f);
          addto(ac[R & 3], e);
          addto(ac[(R + 1) & 3], f);
          take2(e, f);
          addto(ac[(R + 2) & 3], e);
          addto(ac[(R + 3) & 3], f);
        }
#pragma unroll
        for (int u = 0; u < 3; ++u)
          if (cc + u < cme) {
            take(e);
            addto(ac[(R + u) & 3], e);
          }
      };
      switch ((hs + LB - 1) & 3) {
        case 0: phase_c(std::integral_constant<int, 0>{}); break;
        case 1: phase_c(std::integral_constant<int, 1>{}); break;
        case 2: phase_c(std::integral_constant<int, 2>{}); break;
        default: phase_c(std::integral_constant<int, 3>{}); break;
      }
      for (int cc = cme; cc < nh; ++cc) {
        take(e);
        add_tail(cc + LB - 1, e);
      }
      const int ab = ti & 1;
      mbar_wait(afull + ab, (ti >> 1) & 1);
      const double2* ach = accbuf + (size_t)ab * TILE;
#pragma unroll
      for (int j = 0; j < VPT; ++j) {
        const int64_t v = ((int64_t)tile << LB) + tid + j * CONS;   // local index
        const uint32_t mword = op.bits ? awords[ab * 32 + ((tid + j * CONS) >> 5)] : 0u;
        if ((mword >> (v & 31)) & 1u) continue;   // marked: the fix-up warp's
        const double2 r = (m == main_end) ? cadd(cadd(ac[0][j], ac[1][j]), cadd(ac[2][j], ac[3][j])) : ac[0][j];
        const double2 t = cmul_np(alpha, cadd(x0[j], r));
        tout[v] = t;
        __stcs(acc_out + v, cadd(ach[tid + j * CONS], cmul_np(one, t)));
        nrm = __fma_rn(t.x, t.x, __fma_rn(t.y, t.y, nrm));
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(aempty + ab);
    }
  }
  // deterministic block reduction: consumers + fix-up lanes, fixed order
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nrm = __dadd_rn(nrm, __shfl_xor_sync(0xffffffffu, nrm, o));
  if (lane == 0) red[tid >> 5] = nrm;
  __syncthreads();
  if (tid == 0) {
    double r = 0.0;
    for (int w = 0; w < CONS / 32 + PROD + 1; ++w) r = __dadd_rn(r, red[w]);
    partial[blockIdx.x] = r;
  }
}

// Paired form of the streamed hypercube term (nh = dim - LB even, e.g. the
// C4 dimension 22).  The own tile travels with the acc tile in a per-tile
// slot, so the ring carries exactly the nh partner tiles, TWO per stage behind
// one barrier pair: a consumer warp waits, reads and releases once per two
// partner tiles.  Partner k (row order: set bits high->low, then clear bits
// low->high) sits at row position k (k < hs) or k + LB (k >= hs), so its
// numpy accumulator slot is (k + 3) & 3 before the own tile and (k + LB - 1)
// & 3 after it: with partners taken four at a time from k = 0 every slot is
// a compile-time register, and only the group holding the own tile (k = hs)
// branches on hs & 3.
template <int NSP, int PROD, int CONS>
__global__ void __launch_bounds__(CONS + 32 * PROD + 32, 1)
hc_pair_kernel(const __grid_constant__ HcStream op, int64_t n, const double2* __restrict__ tin, double2* __restrict__ tout,
               const double2* acc_in, double2* acc_out, double s_k, const int* __restrict__ done,
               double* __restrict__ partial) {
  using namespace hcs;
  constexpr int VPT = TILE / CONS;
  static_assert(LB % 4 == 2, "slot rule below assumes (k + LB - 1) & 3 == (k + 1) & 3");
  extern __shared__ __align__(128) unsigned char hcs_smem[];
  double2* ring = reinterpret_cast<double2*>(hcs_smem);                // [NSP][2][TILE]
  double2* slotbuf = ring + (size_t)2 * NSP * TILE;                    // [2][acc, own][TILE]
  uint64_t* full = reinterpret_cast<uint64_t*>(hcs_smem + (size_t)(2 * NSP + 4) * CHUNK_BYTES);
  uint64_t* empty = full + NSP;
  uint64_t* afull = empty + NSP;                                       // [2]
  uint64_t* aempty = afull + 2;                                        // [2]
  uint32_t* awords = reinterpret_cast<uint32_t*>(aempty + 2);          // [2][32]
  __shared__ double red[CONS / 32 + PROD + 1];
  const int tid = threadIdx.x;
  const int dim = op.dim;
  const int nh = dim - LB;
  const int nh_loc = op.dim_loc - LB;
  const uint32_t hmask = (nh >= 32) ? 0xffffffffu : ((1u << nh) - 1u);
  const uint32_t hbase = (uint32_t)op.rank << nh_loc;
  const int64_t vbase = (int64_t)op.rank << op.dim_loc;
  const int64_t ntiles = n >> LB;
  if (tid == 0) {
    for (int s = 0; s < NSP; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, CONS / 32);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(afull + s, 1);
      mbar_init(aempty + s, CONS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  pdl_enter();
  if (*done) return;

  const int lane = tid & 31;
  const double2 alpha = make_double2(0.0, -s_k);
  const double2 one = make_double2(1.0, 0.0);
  const double g = -op.gamma;
  double nrm = 0.0;

  if (tid >= CONS) {
    const int pl = tid - CONS;
    if (pl < 32 * PROD && (pl & 31) == 0) {
      // ---------------- producers: partner pairs in row order; producer q
      // fills the pairs it == q mod PROD, producer 0 also the tile slots
      const uint32_t q = (uint32_t)pl >> 5;
      uint32_t s = 0, ph = 0, ti = 0, it = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++ti) {
        const uint32_t Hl = (uint32_t)tile, H = hbase | Hl;
        if (q == 0) {   // acc tile, own tile and (marked runs) the 32 bitmap words
          const int ab = ti & 1;
          double2* sb = slotbuf + (size_t)ab * 2 * TILE;
          mbar_wait(aempty + ab, ((ti >> 1) & 1) ^ 1);
          mbar_expect_tx(afull + ab, 2 * CHUNK_BYTES + (op.bits ? 128u : 0u));
          bulk_g2s(sb, acc_in + ((int64_t)Hl << LB), CHUNK_BYTES, afull + ab);
          bulk_g2s(sb + TILE, tin + ((int64_t)Hl << LB), CHUNK_BYTES, afull + ab);
          if (op.bits) bulk_g2s(awords + ab * 32, op.bits + ((vbase + (tile << LB)) >> 5), 128u, afull + ab);
        }
        uint32_t setm = H, clrm = (~H) & hmask;
        for (int c = 0; c < nh; c += 2, ++it) {
          const double2* src[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            int b;
            if (setm) {
              b = 31 - __clz(setm);
              setm ^= 1u << b;
            } else {
              b = __ffs(clrm) - 1;
              clrm ^= 1u << b;
            }
            src[h] = b < nh_loc ? tin + ((int64_t)(Hl ^ (1u << b)) << LB) : op.remote[b - nh_loc] + ((int64_t)Hl << LB);
          }
          const uint32_t sc = s, pc = ph;
          if (++s == NSP) {
            s = 0;
            ph ^= 1u;
          }
          if (PROD > 1 && it % PROD != q) continue;
          mbar_wait(empty + sc, pc ^ 1);
          mbar_expect_tx(full + sc, 2 * CHUNK_BYTES);
          bulk_g2s(ring + (size_t)sc * 2 * TILE, src[0], CHUNK_BYTES, full + sc);
          bulk_g2s(ring + (size_t)sc * 2 * TILE + TILE, src[1], CHUNK_BYTES, full + sc);
        }
      }
    } else if (pl >= 32 * PROD && op.bits) {
      // ---------------- fix-up warp (as in hc_stream_kernel)
      const int fl = pl - 32 * PROD;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const uint32_t word = __ldg(op.bits + ((vbase + (tile << LB)) >> 5) + fl);
        unsigned any = __ballot_sync(0xffffffffu, word != 0u);
        while (any) {
          const int src = __ffs(any) - 1;
          any &= any - 1;
          uint32_t wd = __shfl_sync(0xffffffffu, word, src);
          while (wd) {
            const int bit = __ffs(wd) - 1;
            wd &= wd - 1;
            const int64_t v = (tile << LB) + src * 32 + bit;
            const double2 h = hc_marked_row(op, g, tin, v, vbase + v, fl);
            if (fl == 0) {
              const double2 t = cmul_np(alpha, h);
              tout[v] = t;
              acc_out[v] = cadd(acc_in[v], cmul_np(one, t));
              nrm = __fma_rn(t.x, t.x, __fma_rn(t.y, t.y, nrm));
            }
          }
        }
      }
    }
  } else {
    // ---------------- consumers
    const int m = dim - 1;
    const int main_end = m - (m % 4);
    uint32_t offs[VPT][LB / 2];
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
      const uint32_t l = (uint32_t)(tid + j * CONS);
      uint32_t sm = l, cm = (~l) & (TILE - 1);
      const int pc = __popc(l);
#pragma unroll
      for (int qq = 0; qq < LB; ++qq) {
        int b;
        if (qq < pc) {
          b = 31 - __clz(sm);
          sm ^= 1u << b;
        } else {
          b = __ffs(cm) - 1;
          cm ^= 1u << b;
        }
        const uint32_t off = (l ^ (1u << b)) * (uint32_t)sizeof(double2);
        if (qq % 2 == 0) offs[j][qq / 2] = off;
        else offs[j][qq / 2] |= off << 16;
      }
    }
    const uint32_t full_u32 = smem_u32(full), empty_u32 = smem_u32(empty);
    // C-side partners k >= kt go to the tail (row positions past main_end)
    const int kt = main_end - LB + 1;
    uint32_t s = 0, ph = 0, ti = 0;
    for (uint32_t tile = blockIdx.x; tile < (uint32_t)ntiles; tile += nctaid_x(), ++ti) {
      const uint32_t H = hbase | (uint32_t)tile;
      const int hs = __popc(H);
      double2 x0[VPT], ac[4][VPT];
#pragma unroll
      for (int j = 0; j < VPT; ++j) x0[j] = ac[0][j] = ac[1][j] = ac[2][j] = ac[3][j] = make_double2(-0.0, -0.0);
      auto add_tail = [&](int i, const double2 (&e)[VPT]) {
#pragma unroll
        for (int j = 0; j < VPT; ++j) {
          if (i == main_end) ac[0][j] = cadd(cadd(ac[0][j], ac[1][j]), cadd(ac[2][j], ac[3][j]));
          ac[0][j] = cadd(ac[0][j], e[j]);
        }
      };
      auto addto = [&](double2 (&acc)[VPT], const double2 (&e)[VPT]) {
#pragma unroll
        for (int j = 0; j < VPT; ++j) acc[j] = cadd(acc[j], e[j]);
      };
      // the next pair of partner tiles (e: partner 2p, f: 2p + 1)
      auto take_pair = [&](double2 (&e)[VPT], double2 (&f)[VPT]) {
        mbar_wait_u32(full_u32 + 8 * s, ph);
        const double2* c = ring + (size_t)s * 2 * TILE;
#pragma unroll
        for (int j = 0; j < VPT; ++j) {
          e[j] = c[tid + j * CONS];
          f[j] = c[TILE + tid + j * CONS];
        }
#pragma unroll
        for (int j = 0; j < VPT; ++j) {
          e[j] = scale_real_z(g, e[j]);
          f[j] = scale_real_z(g, f[j]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_u32(empty_u32 + 8 * s);
        if (++s == NSP) {
          s = 0;
          ph ^= 1u;
        }
      };
      // partner k = k0 + J (k0 % 4 == 0) before the own tile: slot (J + 3) & 3,
      // partner 0 is x0 (J is a literal at every call: after inlining the slot
      // is a fixed register; a generic-lambda form crashes cudafe++ 12.9)
      auto add_a = [&](int k, int J, const double2 (&e)[VPT]) {
        if (J == 0 && k == 0)
          addto(x0, e);
        else
          addto(ac[(J + 3) & 3], e);
      };
      // after the own tile: slot (J + 1) & 3, or the tail
      auto add_c = [&](int k, int J, const double2 (&e)[VPT]) {
        if (k >= kt)
          add_tail(k + LB - 1, e);
        else
          addto(ac[(J + 1) & 3], e);
      };
      using I0 = std::integral_constant<int, 0>;
      using I1 = std::integral_constant<int, 1>;
      using I2 = std::integral_constant<int, 2>;
      using I3 = std::integral_constant<int, 3>;
      const int ab = ti & 1;
      const double2* sb = slotbuf + (size_t)ab * 2 * TILE;
      // the own tile, row positions hs .. hs + LB - 1 (after the slot arrived)
      const char* owncb = reinterpret_cast<const char*>(sb + TILE);
      auto fold = [&](auto Rc, auto Fc) {
        constexpr int R = decltype(Rc)::value;
        constexpr bool FAST = decltype(Fc)::value;
#pragma unroll
        for (int qq = 0; qq < LB; ++qq) {
          double2 e[VPT];
#pragma unroll
          for (int j = 0; j < VPT; ++j) {
            const uint32_t off = (qq % 2 == 0) ? (offs[j][qq / 2] & 0xffffu) : (offs[j][qq / 2] >> 16);
            e[j] = scale_real_z(g, *reinterpret_cast<const double2*>(owncb + off));
          }
          const int a = (R + qq + 3) & 3;
          if (FAST) {
            addto(ac[a], e);
            continue;
          }
          const int i = hs + qq - 1;
          if (i < 0)
            addto(x0, e);
          else if (i < main_end)
            addto(ac[a], e);
          else
            add_tail(i, e);
        }
      };
      auto own = [&]() {
        mbar_wait(afull + ab, (ti >> 1) & 1);
        if (hs >= 1 && hs + LB - 2 < main_end) {
          switch (hs & 3) {
            case 0: fold(I0{}, std::true_type{}); break;
            case 1: fold(I1{}, std::true_type{}); break;
            case 2: fold(I2{}, std::true_type{}); break;
            default: fold(I3{}, std::true_type{}); break;
          }
        } else {
          switch (hs & 3) {
            case 0: fold(I0{}, std::false_type{}); break;
            case 1: fold(I1{}, std::false_type{}); break;
            case 2: fold(I2{}, std::false_type{}); break;
            default: fold(I3{}, std::false_type{}); break;
          }
        }
      };
      double2 e[VPT], f[VPT];
      int k0 = 0;
      // groups of four partners wholly before the own tile
      for (; k0 + 4 <= hs; k0 += 4) {
        take_pair(e, f);
        add_a(k0, 0, e);
        add_a(k0, 1, f);
        take_pair(e, f);
        add_a(k0, 2, e);
        add_a(k0, 3, f);
      }
      // the group holding the own tile: partners k0 .. min(k0 + 4, nh) - 1,
      // the own tile after the first r = hs - k0 of them (one call site: the
      // pending second half of a pair waits in f)
      {
        const int r = hs - k0;   // 0..3
        const bool p0 = k0 < nh, p1 = k0 + 2 < nh;   // pairs present
        if (r >= 1) {
          take_pair(e, f);
          add_a(k0, 0, e);
        }
        if (r >= 2) add_a(k0, 1, f);
        if (r >= 3) {
          take_pair(e, f);
          add_a(k0, 2, e);
        }
        own();
        if (r == 1) add_c(k0 + 1, 1, f);
        if (r == 3) add_c(k0 + 3, 3, f);
        if (r == 0 && p0) {
          take_pair(e, f);
          add_c(k0, 0, e);
          add_c(k0 + 1, 1, f);
        }
        if (r <= 2 && p1) {
          take_pair(e, f);
          add_c(k0 + 2, 2, e);
          add_c(k0 + 3, 3, f);
        }
        k0 += 4;
      }
      // groups wholly after the own tile: first those clear of the tail
      for (; k0 + 4 <= kt && k0 + 4 <= nh; k0 += 4) {
        take_pair(e, f);
        addto(ac[1], e);
        addto(ac[2], f);
        take_pair(e, f);
        addto(ac[3], e);
        addto(ac[0], f);
      }
      for (; k0 < nh; k0 += 4) {
        take_pair(e, f);
        add_c(k0, 0, e);
        add_c(k0 + 1, 1, f);
        if (k0 + 2 < nh) {
          take_pair(e, f);
          add_c(k0 + 2, 2, e);
          add_c(k0 + 3, 3, f);
        }
      }
      const double2* ach = sb;
#pragma unroll
      for (int j = 0; j < VPT; ++j) {
        const int64_t v = ((int64_t)tile << LB) + tid + j * CONS;
        const uint32_t mword = op.bits ? awords[ab * 32 + ((tid + j * CONS) >> 5)] : 0u;
        if ((mword >> (v & 31)) & 1u) continue;   // marked: the fix-up warp's
        const double2 rr = (m == main_end) ? cadd(cadd(ac[0][j], ac[1][j]), cadd(ac[2][j], ac[3][j])) : ac[0][j];
        const double2 t = cmul_np(alpha, cadd(x0[j], rr));
        tout[v] = t;
        __stcs(acc_out + v, cadd(ach[tid + j * CONS], cmul_np(one, t)));
        nrm = __fma_rn(t.x, t.x, __fma_rn(t.y, t.y, nrm));
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(aempty + ab);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nrm = __dadd_rn(nrm, __shfl_xor_sync(0xffffffffu, nrm, o));
  if (lane == 0) red[tid >> 5] = nrm;
  __syncthreads();
  if (tid == 0) {
    double r = 0.0;
    for (int w = 0; w < CONS / 32 + PROD + 1; ++w) r = __dadd_rn(r, red[w]);
    partial[blockIdx.x] = r;
  }
}

// launch one term; returns the number of partials the kernel wrote
template <int NS, int PROD, int CONS>
void launch_stream(const HcStream& op, cudaStream_t s, int64_t n, const double2* tin, double2* tout,
                   const double2* ain, double2* acc, double s_k, const int* flags, double* partial) {
  static bool configured[256] = {};
  const int dev = op.device & 255;
  if (!configured[dev]) {
    cudaFuncSetAttribute(hc_stream_kernel<NS, PROD, CONS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)hcs::smem_bytes(NS));
    configured[dev] = true;
  }
  launch_pdl(hc_stream_kernel<NS, PROD, CONS>, op.grid, CONS + 32 * PROD + 32, hcs::smem_bytes(NS), s, op, n, tin, tout,
             ain, acc, s_k, flags, partial);
}

template <int NSP, int PROD, int CONS>
void launch_pair(const HcStream& op, cudaStream_t s, int64_t n, const double2* tin, double2* tout,
                 const double2* ain, double2* acc, double s_k, const int* flags, double* partial) {
  static bool configured[256] = {};
  const int dev = op.device & 255;
  if (!configured[dev]) {
    cudaFuncSetAttribute(hc_pair_kernel<NSP, PROD, CONS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)hcs::pair_smem_bytes(NSP));
    configured[dev] = true;
  }
  launch_pdl(hc_pair_kernel<NSP, PROD, CONS>, op.grid, CONS + 32 * PROD + 32, hcs::pair_smem_bytes(NSP), s, op, n,
             tin, tout, ain, acc, s_k, flags, partial);
}

int launch_term(const HcStream& op, cudaStream_t s, int64_t n, const double2* tin, double2* tout,
                const double2* ain, double2* acc, double s_k, const int* flags, double* partial) {
  // QWB_HC_STREAM = CONS/256 * 10000 + NS * 100 + PROD (tuning knob; dim 22,
  // us/term on one box: 21201 105.4, 21202 92.5, 21203 102.5 (96 registers,
  // spills), 21002 94.5; profiles/r02_hc_producers.txt)
  // paired form (variants < 1000: NSP * 10 + PROD) where the partner count is
  // even; dim 22 us/term on one box: 52 90.8, 51 91.3, 42 94.0 (21202 92.7);
  // L2 evict-first / evict-last hints with a persisting set-aside of 0 / 40 /
  // 64 / 90 MB: 91.2 / 91.0 / 95.3 / 103.3 (profiles/r02_hc_producers.txt)
  if (op.variant < 1000) {
    if ((op.dim - hcs::LB) % 2 != 0) {   // odd partner count: the single-chunk ring
      launch_stream<12, 2, 512>(op, s, n, tin, tout, ain, acc, s_k, flags, partial);
      return op.grid;
    }
    switch (op.variant) {
      case 51: launch_pair<5, 1, 512>(op, s, n, tin, tout, ain, acc, s_k, flags, partial); break;
      case 41: launch_pair<4, 1, 512>(op, s, n, tin, tout, ain, acc, s_k, flags, partial); break;
      case 42: launch_pair<4, 2, 512>(op, s, n, tin, tout, ain, acc, s_k, flags, partial); break;
      default: launch_pair<5, 2, 512>(op, s, n, tin, tout, ain, acc, s_k, flags, partial); break;
    }
    return op.grid;
  }
  switch (op.variant) {
    case 21001: launch_stream<10, 1, 512>(op, s, n, tin, tout, ain, acc, s_k, flags, partial); break;
    case 21002: launch_stream<10, 2, 512>(op, s, n, tin, tout, ain, acc, s_k, flags, partial); break;
    case 21201: launch_stream<12, 1, 512>(op, s, n, tin, tout, ain, acc, s_k, flags, partial); break;
    case 21203: launch_stream<12, 3, 512>(op, s, n, tin, tout, ain, acc, s_k, flags, partial); break;
    default: launch_stream<12, 2, 512>(op, s, n, tin, tout, ain, acc, s_k, flags, partial); break;
  }
  return op.grid;
}

template <int MAXD>
int launch_term(const HcPos<MAXD>& op, cudaStream_t s, int64_t n, const double2* tin, double2* tout,
                 const double2* ain, double2* acc, double s_k, const int* flags, double* partial) {
  hc_pos_kernel<MAXD><<<kTermBlocks, kTermThreads, 0, s>>>(op, n, tin, tout, ain, acc, s_k, flags, partial);
  return kTermBlocks;
}

template <class Op>
int launch_term(const Op& op, cudaStream_t s, int64_t n, const double2* tin, double2* tout,
                 const double2* ain, double2* acc, double s_k, const int* flags, double* partial) {
  term_kernel<Op><<<kTermBlocks, kTermThreads, 0, s>>>(op, n, tin, tout, ain, acc, s_k, flags, partial);
  return kTermBlocks;
}

// CSR term: a grid of exactly one resident wave (SMs x resident CTAs) — the
// grid-stride loop then has no partial last wave (2048 blocks were 4.6 waves:
// 140 -> 126 us/term on a 2048^2 grid H).  Deterministic for a given device.
int launch_term(const CsrOp& op, cudaStream_t s, int64_t n, const double2* tin, double2* tout,
                const double2* ain, double2* acc, double s_k, const int* flags, double* partial) {
  const int grid = op.grid;
  if (op.capped)
    launch_pdl(csr_term_kernel4, grid, kTermThreads, 0, s, op, n, tin, tout, ain, acc, s_k, flags, partial);
  else
    launch_pdl(term_kernel<CsrOp>, grid, kTermThreads, 0, s, op, n, tin, tout, ain, acc, s_k, flags, partial);
  return grid;
}


__global__ void apply_kernel_hc(HypercubeOp<32> op, int64_t n, const double2* __restrict__ x,
                                double2* __restrict__ y) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    y[v] = op.row(v, x);
}

template <class Op>
int evolve(qwb_ctx* ctx, const Op& op, int64_t n, double2* psi, double2* work, int64_t substeps,
           double tau, double floor_, int max_terms, int* terms_host, cudaStream_t s) {
  if (substeps < 1) QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "substeps must be >= 1");
  if (max_terms < 1) QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "max_terms must be >= 1");
  void* ws;
  int st = qwb::workspace(ctx, kPartialsMax * sizeof(double) + 256, s, &ws);
  if (st) return st;
  double* partial = reinterpret_cast<double*>(ws);
  int* flags = reinterpret_cast<int*>(reinterpret_cast<char*>(ws) + kPartialsMax * sizeof(double));
  int* pin = reinterpret_cast<int*>(ctx->pinned);
  // 4 distinct buffers: cur, acc, term ping-pong
  double2* bufs[4] = {psi, work, work + n, work + 2 * n};
  int cur = 0;
  int prev_terms = 8;
  for (int64_t sub = 0; sub < substeps; ++sub) {
    int others[3], j = 0;
    for (int b = 0; b < 4; ++b)
      if (b != cur) others[j++] = b;
    double2* acc = bufs[others[0]];
    double2* ta = bufs[others[1]];
    double2* tb = bufs[others[2]];
    QWB_CUDA(ctx, cudaMemsetAsync(flags, 0, 2 * sizeof(int), s));
    int launched = 0;
    int chunk = prev_terms + 1;
    bool done = false;
    while (!done) {
      if (launched >= max_terms) {
        QWB_FAIL(ctx, QWB_E_SERIES_NOT_CONVERGED,
                 "series did not reach the tolerance within %d terms per sub-step", max_terms);
      }
      const int upto = launched + chunk < max_terms ? launched + chunk : max_terms;
      for (int k = launched + 1; k <= upto; ++k) {
        const double2* tin = (k == 1) ? bufs[cur] : ((k % 2) ? tb : ta);
        double2* tout = (k % 2) ? ta : tb;
        const double2* ain = (k == 1) ? bufs[cur] : acc;
        const double s_k = tau / (double)k;
        const int nparts = launch_term(op, s, n, tin, tout, ain, acc, s_k, flags, partial);
        launch_pdl(term_finalize_kernel, 1, kTermThreads, 0, s, (const double*)partial, nparts, floor_, k,
                   flags, flags + 1);
      }
      QWB_LAUNCH_CHECK(ctx, "term kernels");
      launched = upto;
      QWB_CUDA(ctx, cudaMemcpyAsync(pin, flags, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
      QWB_CUDA(ctx, cudaStreamSynchronize(s));
      done = pin[0] != 0;
      chunk = 4;
    }
    prev_terms = pin[1];
    if (terms_host) terms_host[sub] = pin[1];
    cur = others[0];   // acc becomes the current state
  }
  if (bufs[cur] != psi)
    QWB_CUDA(ctx, cudaMemcpyAsync(psi, bufs[cur], n * sizeof(double2), cudaMemcpyDeviceToDevice, s));
  return QWB_OK;
}

// ---------------------------------------------------------------------------
// Sharded hypercube evolve.  2^S shards of 2^(dim-S) consecutive vertices
// (shard r = the vertices whose top S bits are r).  Per Taylor term every
// shard needs, for each rank bit j, the partner shard r ^ 2^j's whole term
// slice (same local index), so the term loop is:
//   exchange: NCCL grouped send/recv of term_{k-1} with the S partners
//             (emulation: the partner's buffer is read in place)
//   term:     hc_stream_kernel on the local slice, partner tiles across rank
//             bits streamed from the received slices
//   norm:     local partial sums -> one float64 per shard -> all-gather ->
//             every shard sums the 2^S values in rank order (identical stop
//             decision everywhere)
// Every vertex's row is computed with the single-GPU formula and order, so
// states are bitwise equal to one GPU; only the norm's summation tree differs.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kTermThreads)
term_local_sum_kernel(const double* __restrict__ partial, int nparts, const int* __restrict__ done,
                      double* __restrict__ out) {
  if (*done) return;
  __shared__ double sh[kTermThreads];
  double acc = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) acc = __dadd_rn(acc, partial[i]);
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = kTermThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = __dadd_rn(sh[threadIdx.x], sh[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

__global__ void term_global_finalize_kernel(const double* __restrict__ gsum, int nshards, double floor_, int k,
                                            int* __restrict__ done, int* __restrict__ terms) {
  if (*done || threadIdx.x != 0) return;
  double acc = 0.0;
  for (int i = 0; i < nshards; ++i) acc = __dadd_rn(acc, gsum[i]);
  if (__dsqrt_rn(acc) <= floor_) {
    *done = 1;
    *terms = k;
  }
}

struct ShardSet {
  int nlocal;                 // shards held by this process (1 with NCCL, 2^S emulated)
  int first_rank;             // rank of local shard 0
  bool nccl;
  double2* bufs[32][4];       // per local shard: psi, work, work + n, work + 2n
  double2* recv[kMaxShardBits];   // NCCL mode: received partner slices
};

int evolve_hc_sharded(qwb_ctx* ctx, const HcStream& base, int S, ShardSet& sh, int64_t substeps, double tau,
                      double floor_, int max_terms, int* terms_host, cudaStream_t s) {
  if (substeps < 1) QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "substeps must be >= 1");
  if (max_terms < 1) QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "max_terms must be >= 1");
  const int P = 1 << S;
  const int64_t nloc = 1LL << base.dim_loc;
  const int grid = base.grid;
  void* ws;
  const size_t part_bytes = (size_t)sh.nlocal * grid * sizeof(double);
  int st = qwb::workspace(ctx, part_bytes + P * sizeof(double) + 256, s, &ws);
  if (st) return st;
  double* partial = reinterpret_cast<double*>(ws);
  double* gsum = partial + (size_t)sh.nlocal * grid;
  int* flags = reinterpret_cast<int*>(gsum + P);
  int* pin = reinterpret_cast<int*>(ctx->pinned);
  int peers[kMaxShardBits];
  for (int j = 0; j < S; ++j) peers[j] = sh.first_rank ^ (1 << j);
  int cur = 0;
  int prev_terms = 8;
  for (int64_t sub = 0; sub < substeps; ++sub) {
    int others[3], jj = 0;
    for (int b = 0; b < 4; ++b)
      if (b != cur) others[jj++] = b;
    QWB_CUDA(ctx, cudaMemsetAsync(flags, 0, 2 * sizeof(int), s));
    int launched = 0;
    int chunk = prev_terms + 1;
    bool done = false;
    while (!done) {
      if (launched >= max_terms) {
        QWB_FAIL(ctx, QWB_E_SERIES_NOT_CONVERGED,
                 "series did not reach the tolerance within %d terms per sub-step", max_terms);
      }
      const int upto = launched + chunk < max_terms ? launched + chunk : max_terms;
      for (int k = launched + 1; k <= upto; ++k) {
        // buffer roles, identical on every shard
        const int i_tin = (k == 1) ? cur : ((k % 2) ? others[2] : others[1]);
        const int i_tout = (k % 2) ? others[1] : others[2];
        const int i_ain = (k == 1) ? cur : others[0];
        const int i_acc = others[0];
        const double s_k = tau / (double)k;
        if (sh.nccl) {
          void* rv[kMaxShardBits];
          for (int j = 0; j < S; ++j) rv[j] = sh.recv[j];
          st = qwb::nccl_exchange(ctx, sh.bufs[0][i_tin], rv, peers, S, 2 * (size_t)nloc, s);
          if (st) return st;
        }
        for (int i = 0; i < sh.nlocal; ++i) {
          HcStream op = base;
          op.rank = sh.first_rank + i;
          for (int j = 0; j < S; ++j)
            op.remote[j] = sh.nccl ? sh.recv[j] : sh.bufs[i ^ (1 << j)][i_tin];
          launch_term(op, s, nloc, sh.bufs[i][i_tin], sh.bufs[i][i_tout], sh.bufs[i][i_ain], sh.bufs[i][i_acc],
                      s_k, flags, partial + (size_t)i * grid);
          term_local_sum_kernel<<<1, kTermThreads, 0, s>>>(partial + (size_t)i * grid, grid, flags,
                                                           gsum + op.rank);
        }
        if (sh.nccl) {
          st = qwb::nccl_allgather_f64(ctx, gsum + sh.first_rank, gsum, 1, s);
          if (st) return st;
        }
        term_global_finalize_kernel<<<1, 32, 0, s>>>(gsum, P, floor_, k, flags, flags + 1);
      }
      QWB_LAUNCH_CHECK(ctx, "sharded term kernels");
      launched = upto;
      QWB_CUDA(ctx, cudaMemcpyAsync(pin, flags, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
      QWB_CUDA(ctx, cudaStreamSynchronize(s));
      done = pin[0] != 0;
      chunk = 4;
    }
    prev_terms = pin[1];
    if (terms_host) terms_host[sub] = pin[1];
    cur = others[0];
  }
  if (cur != 0)
    for (int i = 0; i < sh.nlocal; ++i)
      QWB_CUDA(ctx, cudaMemcpyAsync(sh.bufs[i][0], sh.bufs[i][cur], nloc * sizeof(double2),
                                    cudaMemcpyDeviceToDevice, s));
  return QWB_OK;
}

int hc_stream_base(qwb_ctx* ctx, int dim, int S, double gamma, const uint32_t* bits, HcStream* op) {
  if (dim < 1 || dim > 32) QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "hypercube dim must be in 1..32");
  if (S < 0 || S > kMaxShardBits) QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "log2_shards must be in 0..%d", kMaxShardBits);
  if (dim - S < hcs::LB)
    QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "shards of hypercube(%d) over 2^%d ranks hold < 2^%d vertices", dim, S,
             hcs::LB);
  static int variant = -1;
  if (variant < 0) {
    const char* e = getenv("QWB_HC_STREAM");
    variant = (e && *e) ? atoi(e) : 52;
  }
  const int64_t ntiles = 1LL << (dim - S - hcs::LB);
  *op = HcStream{};
  op->dim = dim;
  op->dim_loc = dim - S;
  op->gamma = gamma;
  op->bits = bits;
  op->grid = (int)(ntiles < ctx->num_sms ? ntiles : ctx->num_sms);
  op->device = ctx->device;
  op->variant = variant;
  return QWB_OK;
}

}  // namespace

extern "C" {

int qwb_taylor_evolve_hypercube_sharded(qwb_ctx* ctx, int dim, int log2_shards, double gamma,
                                        const uint32_t* marked_bits, qwb_z* psi, qwb_z* work, int64_t substeps,
                                        double tau, double floor, int max_terms, int* terms_host, void* stream) {
  QWB_BEGIN(ctx);
  HcStream base;
  int st = hc_stream_base(ctx, dim, log2_shards, gamma, marked_bits, &base);
  if (st) return st;
  if (!ctx->comm) QWB_FAIL(ctx, QWB_E_NCCL, "qwb_comm_init has not been called");
  if (ctx->nranks != (1 << log2_shards))
    QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "communicator has %d ranks, expected 2^%d", ctx->nranks, log2_shards);
  const int64_t nloc = 1LL << base.dim_loc;
  ShardSet sh{};
  sh.nlocal = 1;
  sh.first_rank = ctx->rank;
  sh.nccl = true;
  double2* w = reinterpret_cast<double2*>(work);
  sh.bufs[0][0] = reinterpret_cast<double2*>(psi);
  for (int b = 1; b < 4; ++b) sh.bufs[0][b] = w + (b - 1) * nloc;
  for (int j = 0; j < log2_shards; ++j) sh.recv[j] = w + (3 + j) * nloc;
  return evolve_hc_sharded(ctx, base, log2_shards, sh, substeps, tau, floor, max_terms, terms_host,
                           qwb::as_stream(stream));
}

int qwb_taylor_evolve_hypercube_shards_local(qwb_ctx* ctx, int dim, int log2_shards, double gamma,
                                             const uint32_t* marked_bits, qwb_z* const* psi_host,
                                             qwb_z* const* work_host, int64_t substeps, double tau, double floor,
                                             int max_terms, int* terms_host, void* stream) {
  QWB_BEGIN(ctx);
  HcStream base;
  int st = hc_stream_base(ctx, dim, log2_shards, gamma, marked_bits, &base);
  if (st) return st;
  const int64_t nloc = 1LL << base.dim_loc;
  ShardSet sh{};
  sh.nlocal = 1 << log2_shards;
  sh.first_rank = 0;
  sh.nccl = false;
  for (int i = 0; i < sh.nlocal; ++i) {
    double2* w = reinterpret_cast<double2*>(work_host[i]);
    sh.bufs[i][0] = reinterpret_cast<double2*>(psi_host[i]);
    for (int b = 1; b < 4; ++b) sh.bufs[i][b] = w + (b - 1) * nloc;
  }
  return evolve_hc_sharded(ctx, base, log2_shards, sh, substeps, tau, floor, max_terms, terms_host,
                           qwb::as_stream(stream));
}

int qwb_taylor_evolve_csr(qwb_ctx* ctx, int64_t n, const int64_t* row_offsets, const int32_t* col,
                          const qwb_z* val, qwb_z* psi, qwb_z* work, int64_t substeps, double tau,
                          double floor, int max_terms, int* terms_host, void* stream) {
  QWB_BEGIN(ctx);
  if (n < 1) QWB_FAIL(ctx, QWB_E_DIMENSION, "dimension must be positive");
  static int capped = -1;
  if (capped < 0) {
    const char* e = getenv("QWB_CSR_TERM_MINB");
    capped = (e && *e && atoi(e) == 3) ? 0 : 1;   // default: the 4-CTA kernel
  }
  int per_sm = 0;
  if (capped)
    QWB_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, csr_term_kernel4,
                                                                kTermThreads, 0));
  else
    QWB_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, term_kernel<CsrOp>,
                                                                kTermThreads, 0));
  int grid = (per_sm > 0 ? per_sm : 1) * ctx->num_sms;
  if (grid > kPartialsMax) grid = kPartialsMax;
  CsrOp op{row_offsets, col, reinterpret_cast<const double2*>(val), grid, capped};
  return evolve(ctx, op, n, reinterpret_cast<double2*>(psi), reinterpret_cast<double2*>(work),
                substeps, tau, floor, max_terms, terms_host, qwb::as_stream(stream));
}

int qwb_taylor_evolve_hypercube(qwb_ctx* ctx, int dim, double gamma, const uint32_t* marked_bits,
                                qwb_z* psi, qwb_z* work, int64_t substeps, double tau, double floor,
                                int max_terms, int* terms_host, void* stream) {
  QWB_BEGIN(ctx);
  if (dim < 1 || dim > 32) QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "hypercube dim must be in 1..32");
  const int64_t n = 1LL << dim;
  double2* p = reinterpret_cast<double2*>(psi);
  double2* w = reinterpret_cast<double2*>(work);
  cudaStream_t s = qwb::as_stream(stream);
  // QWB_HC_KERNEL: 3 = TMA-streamed tiles (default), 2 = positional gather,
  // 0 = generic gather (the slower designs, kept for A/B measurements)
  static int tiled = -1;
  if (tiled < 0) {
    const char* e = getenv("QWB_HC_KERNEL");
    tiled = (e && *e) ? atoi(e) : 3;
  }
  if (dim <= 8) {
    HypercubeOp<8> op{dim, gamma, marked_bits};
    return evolve(ctx, op, n, p, w, substeps, tau, floor, max_terms, terms_host, s);
  }
  if (tiled == 3 && dim >= hcs::LB) {
    HcStream op;
    int st = hc_stream_base(ctx, dim, 0, gamma, marked_bits, &op);
    if (st) return st;
    return evolve(ctx, op, n, p, w, substeps, tau, floor, max_terms, terms_host, s);
  }
  if (tiled == 2 && dim >= 10) {
    if (dim <= 16) {
      HcPos<16> op{dim, gamma, marked_bits};
      return evolve(ctx, op, n, p, w, substeps, tau, floor, max_terms, terms_host, s);
    }
    if (dim <= 24) {
      HcPos<24> op{dim, gamma, marked_bits};
      return evolve(ctx, op, n, p, w, substeps, tau, floor, max_terms, terms_host, s);
    }
    HcPos<31> op{dim, gamma, marked_bits};
    return evolve(ctx, op, n, p, w, substeps, tau, floor, max_terms, terms_host, s);
  }
  if (dim <= 16) {
    HypercubeOp<16> op{dim, gamma, marked_bits};
    return evolve(ctx, op, n, p, w, substeps, tau, floor, max_terms, terms_host, s);
  }
  if (dim <= 24) {
    HypercubeOp<24> op{dim, gamma, marked_bits};
    return evolve(ctx, op, n, p, w, substeps, tau, floor, max_terms, terms_host, s);
  }
  HypercubeOp<32> op{dim, gamma, marked_bits};
  return evolve(ctx, op, n, p, w, substeps, tau, floor, max_terms, terms_host, s);
}

int qwb_hypercube_apply(qwb_ctx* ctx, int dim, double gamma, const uint32_t* marked_bits,
                        const qwb_z* x, qwb_z* y, void* stream) {
  QWB_BEGIN(ctx);
  if (dim < 1 || dim > 32) QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "hypercube dim must be in 1..32");
  const int64_t n = 1LL << dim;
  HypercubeOp<32> op{dim, gamma, marked_bits};
  apply_kernel_hc<<<qwb::blocks_for(n, 256, (int64_t)ctx->num_sms * 16), 256, 0, qwb::as_stream(stream)>>>(
      op, n, reinterpret_cast<const double2*>(x), reinterpret_cast<double2*>(y));
  QWB_LAUNCH_CHECK(ctx, "apply_kernel_hc");
  return QWB_OK;
}

}  // extern "C"
