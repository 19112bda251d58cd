// builders.cu — device builders for the bit-exact integer structure.
//
//  * graph families: cycle / line / grid / hypercube adjacency CSR
//    (graphs.py:115-159; sorted heads, duplicates merged like the reference's
//    edge set, graphs.py:138-150)
//  * coined operator U = S C with the -I oracle (coined.py:164-238): the row of
//    U for arc r is the coin row of its source arc k = S^-1(r), i.e. the arc
//    span of k's tail t with value 2/d - [col == k] (exact zeros dropped,
//    coined.py:181), or the single entry -1 at k when t is marked
//    (coined.py:188-219).  Count -> exclusive scan -> fill, no sort needed
//    because a span is already in ascending column order (the reference gets
//    the same order from csr_from_triplets' key sort, backend.py:228-236).
//  * Hamiltonian H = -gamma A - sum_M |v><v| with the diagonal inserted at its
//    sorted position (ctqw.py:84-98) and ||H||_inf (ctqw.py:112-120).
#include <cub/cub.cuh>

#include "qwb_internal.cuh"

namespace {

// ---------------------------------------------------------------------------
// families
// ---------------------------------------------------------------------------
struct Family {
  int kind;
  int64_t p0, p1, p2;
  int64_t n;
};

__device__ __forceinline__ void sort4(int64_t c[4]) {
#define QWB_CSWAP(i, j)                    \
  if (c[j] < c[i]) {                       \
    int64_t t = c[i];                      \
    c[i] = c[j];                           \
    c[j] = t;                              \
  }
  QWB_CSWAP(0, 1) QWB_CSWAP(2, 3) QWB_CSWAP(0, 2) QWB_CSWAP(1, 3) QWB_CSWAP(1, 2)
#undef QWB_CSWAP
}

// neighbours of v, sorted ascending, deduplicated; returns count.  For the
// hypercube `out` must hold dim entries.
__device__ int family_neighbours(const Family& f, int64_t v, int64_t* out) {
  if (f.kind == QWB_FAMILY_CYCLE) {
    const int64_t n = f.p0;
    int64_t a = (v + n - 1) % n, b = (v + 1) % n;
    if (a > b) { int64_t t = a; a = b; b = t; }
    out[0] = a;
    if (b == a) return 1;
    out[1] = b;
    return 2;
  }
  if (f.kind == QWB_FAMILY_LINE) {
    const int64_t n = f.p0;
    int k = 0;
    if (v > 0) out[k++] = v - 1;
    if (v < n - 1) out[k++] = v + 1;
    return k;
  }
  if (f.kind == QWB_FAMILY_GRID) {
    const int64_t nx = f.p0, ny = f.p1;
    const bool periodic = f.p2 != 0;
    const int64_t x = v % nx, y = v / nx;
    int64_t c[4];
    if (periodic) {
      c[0] = (x + nx - 1) % nx + nx * y;
      c[1] = (x + 1) % nx + nx * y;
      c[2] = x + nx * ((y + ny - 1) % ny);
      c[3] = x + nx * ((y + 1) % ny);
    } else {
      c[0] = x > 0 ? v - 1 : -1;
      c[1] = x < nx - 1 ? v + 1 : -1;
      c[2] = y > 0 ? v - nx : -1;
      c[3] = y < ny - 1 ? v + nx : -1;
    }
    sort4(c);
    int k = 0;
    for (int i = 0; i < 4; ++i) {
      if (c[i] < 0) continue;
      if (k > 0 && out[k - 1] == c[i]) continue;
      out[k++] = c[i];
    }
    return k;
  }
  // hypercube: clear set bits high->low (v - 2^b ascending), then set clear
  // bits low->high (v + 2^b ascending)
  const int dim = (int)f.p0;
  int k = 0;
  for (int b = dim - 1; b >= 0; --b)
    if ((v >> b) & 1) out[k++] = v ^ (1LL << b);
  for (int b = 0; b < dim; ++b)
    if (!((v >> b) & 1)) out[k++] = v ^ (1LL << b);
  return k;
}

__global__ void family_count_kernel(Family f, int64_t* __restrict__ counts_plus1) {
  int64_t nb[64];
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < f.n;
       v += (int64_t)gridDim.x * blockDim.x) {
    counts_plus1[v + 1] = family_neighbours(f, v, nb);
    if (v == 0) counts_plus1[0] = 0;
  }
}

__global__ void family_fill_kernel(Family f, const int64_t* __restrict__ offs,
                                   int64_t* __restrict__ col) {
  int64_t nb[64];
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < f.n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int k = family_neighbours(f, v, nb);
    const int64_t s = offs[v];
    for (int i = 0; i < k; ++i) col[s + i] = nb[i];
  }
}

// inclusive scan of counts[1..n] in place -> offsets (counts[0] == 0)
int scan_offsets(qwb_ctx* ctx, int64_t* offs, int64_t n, cudaStream_t s, void* extra_ws,
                 size_t extra_bytes) {
  size_t temp = 0;
  QWB_CUDA(ctx, cub::DeviceScan::InclusiveSum(nullptr, temp, offs + 1, offs + 1, n, s));
  if (extra_ws && extra_bytes >= temp) {
    QWB_CUDA(ctx, cub::DeviceScan::InclusiveSum(extra_ws, temp, offs + 1, offs + 1, n, s));
    return QWB_OK;
  }
  void* ws;
  int st = qwb::workspace(ctx, temp, s, &ws);
  if (st) return st;
  QWB_CUDA(ctx, cub::DeviceScan::InclusiveSum(ws, temp, offs + 1, offs + 1, n, s));
  return QWB_OK;
}

int read_last(qwb_ctx* ctx, const int64_t* offs, int64_t n, int64_t* out, cudaStream_t s) {
  int64_t* pin = reinterpret_cast<int64_t*>(ctx->pinned);
  QWB_CUDA(ctx, cudaMemcpyAsync(pin, offs + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  QWB_CUDA(ctx, cudaStreamSynchronize(s));
  *out = *pin;
  return QWB_OK;
}

// ---------------------------------------------------------------------------
// coined operator
// ---------------------------------------------------------------------------
struct Graph {
  int64_t n;
  const int64_t* offs;
  const int64_t* col;
};

__global__ void tails_kernel(Graph g, int32_t* __restrict__ tails) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < g.n;
       v += (int64_t)gridDim.x * blockDim.x) {
    for (int64_t k = g.offs[v]; k < g.offs[v + 1]; ++k) tails[k] = (int32_t)v;
  }
}

// index of arc (v, w): offs[v] + lower_bound(col[offs[v]:offs[v+1]], w); -1 if absent
__device__ __forceinline__ int64_t arc_index(const Graph& g, int64_t v, int64_t w) {
  int64_t lo = g.offs[v], hi = g.offs[v + 1];
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (g.col[mid] < w) lo = mid + 1;
    else hi = mid;
  }
  return (lo < g.offs[v + 1] && g.col[lo] == w) ? lo : -1;
}

// persistent shift target of arc k = (v, w) (coined.py:104-146)
__device__ int64_t persistent_target(const Graph& g, const Family& f, int64_t v, int64_t w) {
  if (f.kind == QWB_FAMILY_CYCLE) {
    const int64_t n = f.p0;
    const int64_t d = ((w - v) % n + n) % n;
    return arc_index(g, w, (w + d) % n);
  }
  if (f.kind == QWB_FAMILY_LINE) {
    const int64_t d = w - v, nxt = w + d;
    if (nxt >= 0 && nxt < g.n) return arc_index(g, w, nxt);
    return arc_index(g, w, v);
  }
  const int64_t nx = f.p0, ny = f.p1;
  const int64_t vx = v % nx, vy = v / nx, wx = w % nx, wy = w / nx;
  const int64_t dx = ((wx - vx) % nx + nx) % nx, dy = ((wy - vy) % ny + ny) % ny;
  int64_t tx, ty;
  if (dy == 0) {
    const int64_t st = dx == 1 ? 1 : -1;
    tx = ((wx + st) % nx + nx) % nx;
    ty = wy;
  } else {
    const int64_t st = dy == 1 ? 1 : -1;
    tx = wx;
    ty = ((wy + st) % ny + ny) % ny;
  }
  return arc_index(g, w, tx + nx * ty);
}

// src[r] = k with S e_k = e_r.  Flip-flop is an involution: k = rev(r).
__global__ void flipflop_src_kernel(Graph g, const int32_t* __restrict__ tails,
                                    int64_t* __restrict__ src, int64_t n_arcs, int* bad) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_arcs;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = tails[r], w = g.col[r];
    const int64_t k = arc_index(g, w, v);
    if (k < 0) atomicOr(bad, 1);
    src[r] = k < 0 ? r : k;
  }
}

__global__ void persistent_src_kernel(Graph g, Family f, const int32_t* __restrict__ tails,
                                      int64_t* __restrict__ src, int64_t n_arcs, int* bad) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n_arcs;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = persistent_target(g, f, tails[k], g.col[k]);
    if (t < 0) {
      atomicOr(bad, 1);
      continue;
    }
    src[t] = k;
  }
}

__global__ void identity_src_kernel(int64_t* __restrict__ src, int64_t n_arcs) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_arcs;
       r += (int64_t)gridDim.x * blockDim.x)
    src[r] = r;
}

__device__ __forceinline__ bool is_marked(const uint32_t* bits, int64_t v) {
  return bits && ((bits[v >> 5] >> (v & 31)) & 1u);
}

__global__ void coined_count_kernel(Graph g, const int32_t* __restrict__ tails,
                                    const int64_t* __restrict__ src, const uint32_t* __restrict__ bits,
                                    int64_t n_arcs, int64_t* __restrict__ counts_plus1) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_arcs;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = tails[src[r]];
    const int64_t d = g.offs[t + 1] - g.offs[t];
    int64_t c;
    if (is_marked(bits, t)) c = 1;
    else c = (__dsub_rn(__ddiv_rn(2.0, (double)d), 1.0) == 0.0) ? d - 1 : d;
    counts_plus1[r + 1] = c;
    if (r == 0) counts_plus1[0] = 0;
  }
}

__global__ void coined_fill_kernel(Graph g, const int32_t* __restrict__ tails,
                                   const int64_t* __restrict__ src, const uint32_t* __restrict__ bits,
                                   int64_t n_arcs, const int64_t* __restrict__ uoffs,
                                   int32_t* __restrict__ ucol, double2* __restrict__ uval) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_arcs;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = src[r];
    const int64_t t = tails[k];
    int64_t o = uoffs[r];
    if (is_marked(bits, t)) {
      ucol[o] = (int32_t)k;
      uval[o] = make_double2(-1.0, 0.0);
      continue;
    }
    const int64_t base = g.offs[t], d = g.offs[t + 1] - base;
    const double off = __ddiv_rn(2.0, (double)d);
    const double dia = __dsub_rn(off, 1.0);
    for (int64_t j = 0; j < d; ++j) {
      const int64_t c = base + j;
      const double v = (c == k) ? dia : off;
      if (v == 0.0) continue;
      ucol[o] = (int32_t)c;
      uval[o] = make_double2(v, 0.0);
      ++o;
    }
  }
}

// ---------------------------------------------------------------------------
// Hamiltonian
// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t count_below(const int64_t* m, int64_t nm, int64_t v) {
  int64_t lo = 0, hi = nm;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (m[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void ham_fill_kernel(Graph g, double gamma, const int64_t* __restrict__ marked,
                                int64_t n_marked, int64_t* __restrict__ hoffs,
                                int32_t* __restrict__ hcol, double2* __restrict__ hval) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < g.n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t below = count_below(marked, n_marked, v);
    const bool mk = below < n_marked && marked[below] == v;
    int64_t o = g.offs[v] + below;
    hoffs[v] = o;
    if (v == g.n - 1) hoffs[g.n] = g.offs[g.n] + n_marked;
    bool placed = !mk;
    for (int64_t j = g.offs[v]; j < g.offs[v + 1]; ++j) {
      const int64_t c = g.col[j];
      if (!placed && c > v) {
        hcol[o] = (int32_t)v;
        hval[o] = make_double2(-1.0, 0.0);
        ++o;
        placed = true;
      }
      hcol[o] = (int32_t)c;
      hval[o] = make_double2(-gamma, 0.0);
      ++o;
    }
    if (!placed) {
      hcol[o] = (int32_t)v;
      hval[o] = make_double2(-1.0, 0.0);
    }
  }
}

struct AbsGet {
  const double2* __restrict__ val;
  int64_t base;
  __device__ __forceinline__ double operator()(int64_t i) const { return qwb::cabs_np(val[base + i]); }
};

__global__ void inf_norm_kernel(int64_t n_rows, const int64_t* __restrict__ offs,
                                const double2* __restrict__ val, unsigned long long* __restrict__ out) {
  double best = 0.0;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = offs[r], e = offs[r + 1];
    if (e == s) continue;
    AbsGet g{val, s};
    const double sum = qwb::reduceat_d(g, e - s);
    best = fmax(best, sum);
  }
  // non-negative doubles order like their bit patterns
  atomicMax(out, (unsigned long long)__double_as_longlong(best));
}

__global__ void marked_bitmap_kernel(const int64_t* __restrict__ marked, int64_t n_marked,
                                     int64_t n, uint32_t* __restrict__ bits, int* bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_marked) return;
  const int64_t v = marked[i];
  if (v < 0 || v >= n) {
    atomicOr(bad, 2);
    return;
  }
  atomicOr(bits + (v >> 5), 1u << (v & 31));
}

// bitmap into caller-provided memory; range errors are OR-ed into *dbad as 2
int launch_bitmap(qwb_ctx* ctx, int64_t n, const int64_t* marked, int64_t n_marked, uint32_t* bits,
                  int* dbad, cudaStream_t s) {
  QWB_CUDA(ctx, cudaMemsetAsync(bits, 0, ((n + 31) / 32) * sizeof(uint32_t), s));
  if (n_marked > 0) {
    marked_bitmap_kernel<<<qwb::blocks_for(n_marked, 256), 256, 0, s>>>(marked, n_marked, n, bits, dbad);
    QWB_LAUNCH_CHECK(ctx, "marked_bitmap_kernel");
  }
  return QWB_OK;
}

int check_family(qwb_ctx* ctx, int family, const int64_t* p, Family* f) {
  f->kind = family;
  f->p0 = p[0];
  f->p1 = f->p2 = 0;
  switch (family) {
    case QWB_FAMILY_CYCLE:
      if (p[0] < 3) QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "cycle requires n >= 3");
      f->n = p[0];
      break;
    case QWB_FAMILY_LINE:
      if (p[0] < 2) QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "line requires n >= 2");
      f->n = p[0];
      break;
    case QWB_FAMILY_GRID:
      f->p1 = p[1];
      f->p2 = p[2];
      if (p[0] < 2 || p[1] < 2) QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "grid requires nx, ny >= 2");
      f->n = p[0] * p[1];
      break;
    case QWB_FAMILY_HYPERCUBE:
      if (p[0] < 1 || p[0] > 40) QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "hypercube dim must be in 1..40");
      f->n = 1LL << p[0];
      break;
    default:
      QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "unknown graph family %d", family);
  }
  return QWB_OK;
}

}  // namespace

extern "C" {

int qwb_marked_bitmap(qwb_ctx* ctx, int64_t n, const int64_t* marked, int64_t n_marked,
                      uint32_t* bits, void* stream) {
  QWB_BEGIN(ctx);
  cudaStream_t s = qwb::as_stream(stream);
  void* ws;
  int st = qwb::workspace(ctx, sizeof(int), s, &ws);
  if (st) return st;
  int* dbad = reinterpret_cast<int*>(ws);
  QWB_CUDA(ctx, cudaMemsetAsync(dbad, 0, sizeof(int), s));
  st = launch_bitmap(ctx, n, marked, n_marked, bits, dbad, s);
  if (st) return st;
  int* pin = reinterpret_cast<int*>(ctx->pinned);
  QWB_CUDA(ctx, cudaMemcpyAsync(pin, dbad, sizeof(int), cudaMemcpyDeviceToHost, s));
  QWB_CUDA(ctx, cudaStreamSynchronize(s));
  if (*pin) QWB_FAIL(ctx, QWB_E_MARKED_OUT_OF_RANGE, "marked vertex not in 0..%lld", (long long)(n - 1));
  return QWB_OK;
}

int qwb_family_adjacency(qwb_ctx* ctx, int family, const int64_t* params_host, int64_t* row_offsets,
                         int64_t* col, int64_t* nnz_host, void* stream) {
  QWB_BEGIN(ctx);
  Family f;
  int st = check_family(ctx, family, params_host, &f);
  if (st) return st;
  cudaStream_t s = qwb::as_stream(stream);
  const unsigned grid = qwb::blocks_for(f.n, 256, (int64_t)ctx->num_sms * 32);
  if (col == nullptr) {
    family_count_kernel<<<grid, 256, 0, s>>>(f, row_offsets);
    QWB_LAUNCH_CHECK(ctx, "family_count_kernel");
    st = scan_offsets(ctx, row_offsets, f.n, s, nullptr, 0);
    if (st) return st;
    return read_last(ctx, row_offsets, f.n, nnz_host, s);
  }
  family_fill_kernel<<<grid, 256, 0, s>>>(f, row_offsets, col);
  QWB_LAUNCH_CHECK(ctx, "family_fill_kernel");
  if (nnz_host) {
    st = read_last(ctx, row_offsets, f.n, nnz_host, s);
    if (st) return st;
  }
  return QWB_OK;
}

int qwb_coined_operator(qwb_ctx* ctx, int64_t n, const int64_t* adj_offs, const int64_t* adj_col,
                        const int64_t* marked, int64_t n_marked, int shift, int family,
                        const int64_t* params_host, int64_t* u_row_offsets, int32_t* u_col,
                        qwb_z* u_val, int64_t* nnz_host, void* stream) {
  QWB_BEGIN(ctx);
  cudaStream_t s = qwb::as_stream(stream);
  if (n < 1) QWB_FAIL(ctx, QWB_E_DIMENSION, "graph must have at least one vertex");
  int64_t n_arcs;
  int st = read_last(ctx, adj_offs, n, &n_arcs, s);
  if (st) return st;
  if (n_arcs < 1) QWB_FAIL(ctx, QWB_E_DIMENSION, "graph has no arcs");
  if (n_arcs > 2147483647LL) QWB_FAIL(ctx, QWB_E_DIMENSION, "device CSR supports < 2^31 arcs");
  Family f{};
  if (shift == QWB_SHIFT_PERSISTENT) {
    if (family != QWB_FAMILY_CYCLE && family != QWB_FAMILY_LINE && family != QWB_FAMILY_GRID)
      QWB_FAIL(ctx, QWB_E_PERSISTENT_SHIFT, "persistent shift is undefined on this graph family");
    st = check_family(ctx, family, params_host, &f);
    if (st) return st;
    if (family == QWB_FAMILY_GRID && (f.p2 == 0))
      QWB_FAIL(ctx, QWB_E_PERSISTENT_SHIFT, "persistent shift requires a periodic grid");
    if (family == QWB_FAMILY_GRID && (f.p0 < 3 || f.p1 < 3))
      QWB_FAIL(ctx, QWB_E_PERSISTENT_SHIFT, "persistent shift on a periodic grid requires nx, ny >= 3");
  } else if (shift != QWB_SHIFT_FLIPFLOP && shift != QWB_SHIFT_NONE) {
    QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "shift: unknown shift code %d", shift);
  }
  // workspace: tails int32[n_arcs] | src int64[n_arcs] | bits u32[(n+31)/32] | flag
  const size_t tails_b = ((size_t)n_arcs * 4 + 255) & ~size_t(255);
  const size_t src_b = ((size_t)n_arcs * 8 + 255) & ~size_t(255);
  const size_t bits_b = (((size_t)(n + 31) / 32) * 4 + 255) & ~size_t(255);
  size_t scan_temp = 0;
  QWB_CUDA(ctx, cub::DeviceScan::InclusiveSum(nullptr, scan_temp, u_row_offsets + 1,
                                               u_row_offsets + 1, n_arcs, s));
  void* ws;
  st = qwb::workspace(ctx, tails_b + src_b + bits_b + 256 + scan_temp, s, &ws);
  if (st) return st;
  char* base = reinterpret_cast<char*>(ws);
  int32_t* tails = reinterpret_cast<int32_t*>(base);
  int64_t* src = reinterpret_cast<int64_t*>(base + tails_b);
  uint32_t* bits = reinterpret_cast<uint32_t*>(base + tails_b + src_b);
  int* dbad = reinterpret_cast<int*>(base + tails_b + src_b + bits_b);
  void* scan_ws = base + tails_b + src_b + bits_b + 256;
  Graph g{n, adj_offs, adj_col};
  const unsigned gv = qwb::blocks_for(n, 256, (int64_t)ctx->num_sms * 32);
  const unsigned ga = qwb::blocks_for(n_arcs, 256, (int64_t)ctx->num_sms * 32);
  QWB_CUDA(ctx, cudaMemsetAsync(dbad, 0, sizeof(int), s));
  tails_kernel<<<gv, 256, 0, s>>>(g, tails);
  const uint32_t* bitsp = nullptr;
  if (n_marked > 0) {
    st = launch_bitmap(ctx, n, marked, n_marked, bits, dbad, s);
    if (st) return st;
    bitsp = bits;
  }
  if (shift == QWB_SHIFT_FLIPFLOP) {
    flipflop_src_kernel<<<ga, 256, 0, s>>>(g, tails, src, n_arcs, dbad);
  } else if (shift == QWB_SHIFT_PERSISTENT) {
    persistent_src_kernel<<<ga, 256, 0, s>>>(g, f, tails, src, n_arcs, dbad);
  } else {
    identity_src_kernel<<<ga, 256, 0, s>>>(src, n_arcs);
  }
  QWB_LAUNCH_CHECK(ctx, "coined src kernels");
  int* pin = reinterpret_cast<int*>(ctx->pinned);
  QWB_CUDA(ctx, cudaMemcpyAsync(pin, dbad, sizeof(int), cudaMemcpyDeviceToHost, s));
  QWB_CUDA(ctx, cudaStreamSynchronize(s));
  if (*pin & 2) QWB_FAIL(ctx, QWB_E_MARKED_OUT_OF_RANGE, "marked vertex not in 0..%lld", (long long)(n - 1));
  if (*pin & 1) QWB_FAIL(ctx, QWB_E_DIMENSION, "adjacency is not a symmetric simple graph");
  if (u_col == nullptr) {
    coined_count_kernel<<<ga, 256, 0, s>>>(g, tails, src, bitsp, n_arcs, u_row_offsets);
    QWB_LAUNCH_CHECK(ctx, "coined_count_kernel");
    QWB_CUDA(ctx, cub::DeviceScan::InclusiveSum(scan_ws, scan_temp, u_row_offsets + 1,
                                                 u_row_offsets + 1, n_arcs, s));
    return read_last(ctx, u_row_offsets, n_arcs, nnz_host, s);
  }
  coined_fill_kernel<<<ga, 256, 0, s>>>(g, tails, src, bitsp, n_arcs, u_row_offsets, u_col,
                                        reinterpret_cast<double2*>(u_val));
  QWB_LAUNCH_CHECK(ctx, "coined_fill_kernel");
  // keep the workspace alive until the fill has consumed it
  QWB_CUDA(ctx, cudaStreamSynchronize(s));
  if (nnz_host) return read_last(ctx, u_row_offsets, n_arcs, nnz_host, s);
  return QWB_OK;
}

int qwb_shift_sources(qwb_ctx* ctx, int64_t n, const int64_t* adj_offs, const int64_t* adj_col,
                      int shift, int family, const int64_t* params_host, int64_t* src,
                      void* stream) {
  QWB_BEGIN(ctx);
  cudaStream_t s = qwb::as_stream(stream);
  int64_t n_arcs;
  int st = read_last(ctx, adj_offs, n, &n_arcs, s);
  if (st) return st;
  if (n_arcs < 1) return QWB_OK;
  Family f{};
  if (shift == QWB_SHIFT_PERSISTENT) {
    if (family != QWB_FAMILY_CYCLE && family != QWB_FAMILY_LINE && family != QWB_FAMILY_GRID)
      QWB_FAIL(ctx, QWB_E_PERSISTENT_SHIFT, "persistent shift is undefined on this graph family");
    st = check_family(ctx, family, params_host, &f);
    if (st) return st;
    if (family == QWB_FAMILY_GRID && (f.p2 == 0))
      QWB_FAIL(ctx, QWB_E_PERSISTENT_SHIFT, "persistent shift requires a periodic grid");
    if (family == QWB_FAMILY_GRID && (f.p0 < 3 || f.p1 < 3))
      QWB_FAIL(ctx, QWB_E_PERSISTENT_SHIFT, "persistent shift on a periodic grid requires nx, ny >= 3");
  } else if (shift != QWB_SHIFT_FLIPFLOP && shift != QWB_SHIFT_NONE) {
    QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "shift: unknown shift code %d", shift);
  }
  const size_t tails_b = ((size_t)n_arcs * 4 + 255) & ~size_t(255);
  void* ws;
  st = qwb::workspace(ctx, tails_b + 256, s, &ws);
  if (st) return st;
  int32_t* tails = reinterpret_cast<int32_t*>(ws);
  int* dbad = reinterpret_cast<int*>(reinterpret_cast<char*>(ws) + tails_b);
  Graph g{n, adj_offs, adj_col};
  const unsigned gv = qwb::blocks_for(n, 256, (int64_t)ctx->num_sms * 32);
  const unsigned ga = qwb::blocks_for(n_arcs, 256, (int64_t)ctx->num_sms * 32);
  QWB_CUDA(ctx, cudaMemsetAsync(dbad, 0, sizeof(int), s));
  tails_kernel<<<gv, 256, 0, s>>>(g, tails);
  if (shift == QWB_SHIFT_FLIPFLOP) flipflop_src_kernel<<<ga, 256, 0, s>>>(g, tails, src, n_arcs, dbad);
  else if (shift == QWB_SHIFT_PERSISTENT) persistent_src_kernel<<<ga, 256, 0, s>>>(g, f, tails, src, n_arcs, dbad);
  else identity_src_kernel<<<ga, 256, 0, s>>>(src, n_arcs);
  QWB_LAUNCH_CHECK(ctx, "shift source kernels");
  int* pin = reinterpret_cast<int*>(ctx->pinned);
  QWB_CUDA(ctx, cudaMemcpyAsync(pin, dbad, sizeof(int), cudaMemcpyDeviceToHost, s));
  QWB_CUDA(ctx, cudaStreamSynchronize(s));
  if (*pin) QWB_FAIL(ctx, QWB_E_DIMENSION, "adjacency is not a symmetric simple graph");
  return QWB_OK;
}

int qwb_hamiltonian(qwb_ctx* ctx, int64_t n, const int64_t* adj_offs, const int64_t* adj_col,
                    double gamma, const int64_t* marked, int64_t n_marked, int64_t* h_row_offsets,
                    int32_t* h_col, qwb_z* h_val, void* stream) {
  QWB_BEGIN(ctx);
  if (n < 1) QWB_FAIL(ctx, QWB_E_DIMENSION, "graph must have at least one vertex");
  if (!(gamma > 0)) QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "gamma must be positive");
  cudaStream_t s = qwb::as_stream(stream);
  Graph g{n, adj_offs, adj_col};
  ham_fill_kernel<<<qwb::blocks_for(n, 256, (int64_t)ctx->num_sms * 32), 256, 0, s>>>(
      g, gamma, marked, n_marked, h_row_offsets, h_col, reinterpret_cast<double2*>(h_val));
  QWB_LAUNCH_CHECK(ctx, "ham_fill_kernel");
  return QWB_OK;
}

int qwb_inf_norm(qwb_ctx* ctx, int64_t n_rows, const int64_t* row_offsets, const qwb_z* val,
                 double* result_host, void* stream) {
  QWB_BEGIN(ctx);
  cudaStream_t s = qwb::as_stream(stream);
  void* ws;
  int st = qwb::workspace(ctx, sizeof(unsigned long long), s, &ws);
  if (st) return st;
  unsigned long long* d = reinterpret_cast<unsigned long long*>(ws);
  QWB_CUDA(ctx, cudaMemsetAsync(d, 0, sizeof(unsigned long long), s));
  inf_norm_kernel<<<qwb::blocks_for(n_rows, 256, (int64_t)ctx->num_sms * 16), 256, 0, s>>>(
      n_rows, row_offsets, reinterpret_cast<const double2*>(val), d);
  QWB_LAUNCH_CHECK(ctx, "inf_norm_kernel");
  unsigned long long* pin = reinterpret_cast<unsigned long long*>(ctx->pinned);
  QWB_CUDA(ctx, cudaMemcpyAsync(pin, d, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  QWB_CUDA(ctx, cudaStreamSynchronize(s));
  unsigned long long bitsv = *pin;
  double r;
  memcpy(&r, &bitsv, sizeof(double));
  *result_host = r;
  return QWB_OK;
}

}  // extern "C"
