// spmv.cu — complex128 CSR SpMV and the repeated-SpMV step loop.
//
// Replaces backend._csr_rows / matvec_mul (backend.py:394-430) and the
// coined.simulate snapshot loop (coined.py:263-272) for operators that are not
// handled matrix-free (generic graphs, cycles, lines, open or thin grids).
//
// Arithmetic is the reference's, bit for bit: products with numpy's FMA
// complex multiply, row sums as x0 + pairwise(x1..) (qwb_numerics.cuh).  Each
// output row is reduced by exactly one thread in a fixed order, so results are
// run-to-run deterministic like the reference's engines (backend.py:10-13).
//
// Layout: row_offsets int64[n+1], col int32[nnz] (narrowed on upload),
// values double2[nnz].  Rows of up to 8 entries (every lattice/cycle/line U)
// take a fully unrolled register path; longer rows (hypercube H, hubs of
// generic graphs) use the generic pairwise reducer.
#include "qwb_internal.cuh"

namespace {

using qwb::cadd;
using qwb::cmul_np;

struct RowGet {
  const int32_t* __restrict__ col;
  const double2* __restrict__ val;
  const double2* __restrict__ x;
  int64_t base;
  __device__ __forceinline__ double2 operator()(int64_t i) const {
    const int64_t j = base + i;
    return cmul_np(__ldg(val + j), __ldg(x + __ldg(col + j)));
  }
};

struct SmemRowGet {
  const int32_t* __restrict__ col;
  const double2* __restrict__ val;
  const double2* x;   // shared memory
  int64_t base;
  __device__ __forceinline__ double2 operator()(int64_t i) const {
    const int64_t j = base + i;
    return cmul_np(__ldg(val + j), x[__ldg(col + j)]);
  }
};

template <class G>
__device__ __forceinline__ double2 row_value(const G& g, int64_t len) {
  if (len == 0) return make_double2(0.0, 0.0);
  // short rows: fully unrolled x0 + pairwise(x1..) with pairwise(<4) sequential
  if (len <= 4) {
    double2 x0 = g(0);
    if (len == 1) return x0;
    double2 r = make_double2(-0.0, -0.0);
    r = cadd(r, g(1));
    if (len > 2) r = cadd(r, g(2));
    if (len > 3) r = cadd(r, g(3));
    return cadd(x0, r);
  }
  return qwb::reduceat_z(g, len);
}

// two consecutive complex128 (32 B, 32-B aligned) in one 256-bit load.  The
// kernel takes this path only when the caller's val and x are 32-B aligned
// (`vec`, checked on the host: any pointer is legal at the C ABI)
__host__ __forceinline__ int vec_ok(const void* val, const void* x) {
  return (((uintptr_t)val | (uintptr_t)x) & 31) == 0;
}

__device__ __forceinline__ void ld2z(const double2* p, double2& a, double2& b) {
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
      : "=d"(a.x), "=d"(a.y), "=d"(b.x), "=d"(b.y)
      : "l"(p));
}

__global__ void __launch_bounds__(256)
spmv_kernel(int64_t n_rows, const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
            const double2* __restrict__ val, const double2* __restrict__ x,
            double2* __restrict__ y, int vec) {
  qwb::pdl_enter();   // x is the previous launch's y in the step loop
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = __ldg(rowptr + r), e = __ldg(rowptr + r + 1);
    if (vec && e - s == 4 && (s & 3) == 0) {
      // 4-entry row (every Grover row of a degree-4 head): one 128-bit column
      // load, two 256-bit value loads; the columns are the head's arc span, so
      // x usually comes in two 256-bit loads as well
      const int4 c = __ldg(reinterpret_cast<const int4*>(col + s));
      double2 v0, v1, v2, v3, x0, x1, x2, x3;
      ld2z(val + s, v0, v1);
      ld2z(val + s + 2, v2, v3);
      if (c.w == c.x + 3 && c.y == c.x + 1 && c.z == c.x + 2 && (c.x & 1) == 0) {
        ld2z(x + c.x, x0, x1);
        ld2z(x + c.x + 2, x2, x3);
      } else {
        x0 = __ldg(x + c.x);
        x1 = __ldg(x + c.y);
        x2 = __ldg(x + c.z);
        x3 = __ldg(x + c.w);
      }
      // x0 + ((x1 + x2) + x3), numpy's reduceat of a 4-entry row
      const double2 r1 = cadd(cadd(make_double2(-0.0, -0.0), cmul_np(v1, x1)), cmul_np(v2, x2));
      y[r] = cadd(cmul_np(v0, x0), cadd(r1, cmul_np(v3, x3)));
      continue;
    }
    RowGet g{col, val, x, s};
    y[r] = row_value(g, e - s);
  }
}

// Whole snapshot loop in one CTA with both state vectors in shared memory.
// For operators whose 2 * n_rows * 16 B fits (cycle(1024): 64 KB).
__global__ void __launch_bounds__(1024)
csr_run_smem_kernel(int64_t n_rows, const int64_t* __restrict__ rowptr,
                    const int32_t* __restrict__ col, const double2* __restrict__ val,
                    const double2* __restrict__ psi0, const int64_t* __restrict__ ks,
                    int64_t n_snap, double2* __restrict__ snaps) {
  extern __shared__ double2 sh[];
  double2* xa = sh;
  double2* xb = sh + n_rows;
  for (int64_t i = threadIdx.x; i < n_rows; i += blockDim.x) xa[i] = psi0[i];
  __syncthreads();
  int64_t cur = 0;
  for (int64_t j = 0; j < n_snap; ++j) {
    const int64_t target = ks[j];
    for (; cur < target; ++cur) {
      for (int64_t r = threadIdx.x; r < n_rows; r += blockDim.x) {
        const int64_t s = __ldg(rowptr + r), e = __ldg(rowptr + r + 1);
        SmemRowGet g{col, val, xa, s};
        xb[r] = row_value(g, e - s);
      }
      __syncthreads();
      double2* t = xa;
      xa = xb;
      xb = t;
    }
    for (int64_t i = threadIdx.x; i < n_rows; i += blockDim.x) snaps[j * n_rows + i] = xa[i];
  }
}

__global__ void narrow_cols_kernel(int64_t n_rows, int64_t n_cols, const int64_t* __restrict__ rowptr,
                                   const int64_t* __restrict__ col64, const double2* __restrict__ val,
                                   int64_t nnz, int32_t* __restrict__ col32, int* __restrict__ flags) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = rowptr[r], e = rowptr[r + 1];
    if (r == 0 && s != 0) atomicOr(flags, 1);
    if (r == n_rows - 1 && e != nnz) atomicOr(flags, 1);
    if (e < s || s < 0 || e > nnz) {
      atomicOr(flags, 2);
      continue;
    }
    int64_t prev = -1;
    for (int64_t j = s; j < e; ++j) {
      const int64_t c = col64[j];
      if (c < 0 || c >= n_cols) atomicOr(flags, 4);
      if (c <= prev) atomicOr(flags, 8);
      prev = c;
      const double2 v = val[j];
      if (!isfinite(v.x) || !isfinite(v.y)) atomicOr(flags, 16);
      col32[j] = (int32_t)c;
    }
  }
}

}  // namespace

extern "C" {

int qwb_csr_prepare(qwb_ctx* ctx, int64_t n_rows, int64_t n_cols, const int64_t* row_offsets,
                    const int64_t* col64, const qwb_z* val, int64_t nnz, int32_t* col32,
                    void* stream) {
  QWB_BEGIN(ctx);
  if (n_rows < 1 || n_cols < 1) QWB_FAIL(ctx, QWB_E_DIMENSION, "matrix dimensions must be positive");
  if (n_cols > 2147483647LL)
    QWB_FAIL(ctx, QWB_E_DIMENSION, "device CSR supports n_cols < 2^31 (got %lld)", (long long)n_cols);
  cudaStream_t s = qwb::as_stream(stream);
  void* ws;
  int st = qwb::workspace(ctx, sizeof(int), s, &ws);
  if (st) return st;
  int* dflags = reinterpret_cast<int*>(ws);
  QWB_CUDA(ctx, cudaMemsetAsync(dflags, 0, sizeof(int), s));
  narrow_cols_kernel<<<qwb::blocks_for(n_rows, 256, 148 * 64), 256, 0, s>>>(
      n_rows, n_cols, row_offsets, col64, reinterpret_cast<const double2*>(val), nnz, col32, dflags);
  QWB_LAUNCH_CHECK(ctx, "narrow_cols_kernel");
  int* flags = reinterpret_cast<int*>(ctx->pinned);
  QWB_CUDA(ctx, cudaMemcpyAsync(flags, dflags, sizeof(int), cudaMemcpyDeviceToHost, s));
  QWB_CUDA(ctx, cudaStreamSynchronize(s));
  const int f = *flags;
  if (f & 1) QWB_FAIL(ctx, QWB_E_DIMENSION, "row_offsets inconsistent with nnz");
  if (f & 2) QWB_FAIL(ctx, QWB_E_DIMENSION, "row_offsets must be non-decreasing");
  if (f & 4) QWB_FAIL(ctx, QWB_E_DIMENSION, "column index out of range");
  if (f & 8) QWB_FAIL(ctx, QWB_E_DIMENSION, "columns must be strictly increasing within rows");
  if (f & 16) QWB_FAIL(ctx, QWB_E_NONFINITE, "structure contains NaN or infinite entries");
  return QWB_OK;
}

int qwb_spmv(qwb_ctx* ctx, int64_t n_rows, const int64_t* row_offsets, const int32_t* col,
             const qwb_z* val, const qwb_z* x, qwb_z* y, void* stream) {
  QWB_BEGIN(ctx);
  if (n_rows < 1) QWB_FAIL(ctx, QWB_E_DIMENSION, "n_rows must be positive");
  static const bool pdl = qwb::env_flag("QWB_STEP_PDL", 1) != 0;   // see qwb::launch_pdl
  qwb::launch_pdl(pdl, spmv_kernel, qwb::blocks_for(n_rows, 256, (int64_t)ctx->num_sms * 64), 256, 0,
                  qwb::as_stream(stream), n_rows, row_offsets, col, reinterpret_cast<const double2*>(val),
                  reinterpret_cast<const double2*>(x), reinterpret_cast<double2*>(y), vec_ok(val, x));
  QWB_LAUNCH_CHECK(ctx, "spmv_kernel");
  return QWB_OK;
}

int qwb_csr_run(qwb_ctx* ctx, int64_t n_rows, const int64_t* row_offsets, const int32_t* col,
                const qwb_z* val, const qwb_z* psi0, const int64_t* k_host, int64_t n_snap,
                qwb_z* snaps, qwb_z* scratch, void* stream) {
  QWB_BEGIN(ctx);
  if (n_rows < 1) QWB_FAIL(ctx, QWB_E_DIMENSION, "n_rows must be positive");
  if (n_snap < 0) QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "n_snap must be >= 0");
  for (int64_t j = 0; j < n_snap; ++j)
    if (k_host[j] < 0 || (j > 0 && k_host[j] < k_host[j - 1]))
      QWB_FAIL(ctx, QWB_E_INVALID_ARGUMENT, "snapshot step counts must be non-decreasing and >= 0");
  if (n_snap == 0) return QWB_OK;
  cudaStream_t s = qwb::as_stream(stream);
  const double2* v = reinterpret_cast<const double2*>(val);
  double2* out = reinterpret_cast<double2*>(snaps);
  const size_t smem = 2 * (size_t)n_rows * sizeof(double2);
  if (smem <= 200 * 1024) {
    void* ws;
    int st = qwb::workspace(ctx, n_snap * sizeof(int64_t), s, &ws);
    if (st) return st;
    int64_t* dks = reinterpret_cast<int64_t*>(ws);
    QWB_CUDA(ctx, cudaMemcpyAsync(dks, k_host, n_snap * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    QWB_CUDA(ctx, cudaFuncSetAttribute(csr_run_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
    csr_run_smem_kernel<<<1, 1024, smem, s>>>(n_rows, row_offsets, col, v,
                                               reinterpret_cast<const double2*>(psi0), dks, n_snap,
                                               out);
    QWB_LAUNCH_CHECK(ctx, "csr_run_smem_kernel");
    // the pageable k_host copy above is synchronous w.r.t. the host; keep the
    // workspace alive until the kernel consumed it
    QWB_CUDA(ctx, cudaStreamSynchronize(s));
    return QWB_OK;
  }
  // scratch holds 2 n_rows + 1 entries: b starts at an even offset so both
  // ping-pong vectors keep the scratch's 32-B alignment
  double2* a = reinterpret_cast<double2*>(scratch);
  double2* b = a + ((n_rows + 1) & ~(int64_t)1);
  const int vec = vec_ok(val, a) && vec_ok(val, b);
  QWB_CUDA(ctx, cudaMemcpyAsync(a, psi0, n_rows * sizeof(double2), cudaMemcpyDeviceToDevice, s));
  const unsigned grid = qwb::blocks_for(n_rows, 256, (int64_t)ctx->num_sms * 64);
  static const bool pdl = qwb::env_flag("QWB_STEP_PDL", 1) != 0;   // see qwb::launch_pdl
  int64_t cur = 0;
  for (int64_t j = 0; j < n_snap; ++j) {
    for (; cur < k_host[j]; ++cur) {
      qwb::launch_pdl(pdl, spmv_kernel, grid, 256, 0, s, n_rows, row_offsets, col, v,
                      (const double2*)a, b, vec);
      double2* t = a;
      a = b;
      b = t;
    }
    QWB_CUDA(ctx, cudaMemcpyAsync(out + j * n_rows, a, n_rows * sizeof(double2),
                                  cudaMemcpyDeviceToDevice, s));
  }
  QWB_LAUNCH_CHECK(ctx, "spmv_kernel");
  return QWB_OK;
}

}  // extern "C"
