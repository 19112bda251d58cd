// reduce.cu — probability reducers and the BLAS-1 of the engine API.
//
//  * qwb_prob_arcs : coined.probability_distribution (coined.py:275-294)
//                    p[v] = reduceat(|psi|^2 over v's arc span), bitwise numpy
//  * qwb_prob_abs2 : ctqw.probability_distribution (ctqw.py:205-212)
//  * axpy / scale / dot / norm : backend.py:433-464 (numpy complex multiply
//    model for axpy/scale; dot/norm are deterministic two-pass tree sums, equal
//    to numpy's BLAS result within rounding)
//  * check_finite : backend._check_finite (backend.py:60-62)
#include "qwb_internal.cuh"

namespace {

using qwb::abs2_np;
using qwb::cadd;
using qwb::cmul_np;

constexpr int kRedBlocks = 1024;   // fixed => run-to-run (and GPU-to-GPU) deterministic
constexpr int kRedThreads = 256;

struct Abs2Get {
  const double2* __restrict__ psi;
  int64_t base;
  __device__ __forceinline__ double operator()(int64_t i) const { return abs2_np(psi[base + i]); }
};

__global__ void prob_arcs_kernel(int64_t n, const int64_t* __restrict__ offs,
                                 const double2* __restrict__ psi, double* __restrict__ p) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = offs[v], e = offs[v + 1];
    if (e == s) {
      p[v] = 0.0;
      continue;
    }
    Abs2Get g{psi, s};
    p[v] = qwb::reduceat_d(g, e - s);
  }
}

__global__ void prob_abs2_kernel(int64_t n, const double2* __restrict__ psi, double* __restrict__ p) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = abs2_np(psi[i]);
}

__global__ void axpy_kernel(int64_t n, double2 alpha, const double2* __restrict__ x,
                            const double2* __restrict__ y, double2* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = cadd(y[i], cmul_np(alpha, x[i]));
}

__global__ void scale_kernel(int64_t n, double2 alpha, const double2* __restrict__ x,
                             double2* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = cmul_np(alpha, x[i]);
}

template <class T>
__device__ __forceinline__ T block_sum(T v, T* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = sh[threadIdx.x] + sh[threadIdx.x + s];
    __syncthreads();
  }
  return sh[0];
}

struct D2 {
  double a, b;
  __device__ D2 operator+(const D2& o) const { return D2{__dadd_rn(a, o.a), __dadd_rn(b, o.b)}; }
};

// mode 0: dot conj(x).y -> (re, im); mode 1: norm^2 -> (sum re^2, sum im^2)
__global__ void __launch_bounds__(kRedThreads)
red_partial_kernel(int64_t n, const double2* __restrict__ x, const double2* __restrict__ y, int mode,
                   D2* __restrict__ partial) {
  __shared__ D2 sh[kRedThreads];
  D2 acc{0.0, 0.0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double2 a = x[i];
    if (mode == 0) {
      const double2 b = y[i];
      // conj(a) * b
      acc.a = __fma_rn(a.x, b.x, __fma_rn(a.y, b.y, acc.a));
      acc.b = __fma_rn(a.x, b.y, __fma_rn(-a.y, b.x, acc.b));
    } else {
      acc.a = __fma_rn(a.x, a.x, acc.a);
      acc.b = __fma_rn(a.y, a.y, acc.b);
    }
  }
  const D2 s = block_sum(acc, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

__global__ void __launch_bounds__(kRedThreads)
red_final_kernel(const D2* __restrict__ partial, int nparts, D2* __restrict__ out) {
  __shared__ D2 sh[kRedThreads];
  D2 acc{0.0, 0.0};
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) acc = acc + partial[i];
  const D2 s = block_sum(acc, sh);
  if (threadIdx.x == 0) *out = s;
}

__global__ void finite_kernel(int64_t n, const double* __restrict__ x, int* __restrict__ bad) {
  bool ok = true;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    ok &= isfinite(x[i]);
  if (!__all_sync(0xffffffffu, ok) && (threadIdx.x & 31) == 0) atomicOr(bad, 1);
}

int reduce2(qwb_ctx* ctx, int64_t n, const double2* x, const double2* y, int mode, D2* result,
            cudaStream_t s) {
  void* ws;
  int st = qwb::workspace(ctx, (kRedBlocks + 1) * sizeof(D2), s, &ws);
  if (st) return st;
  D2* part = reinterpret_cast<D2*>(ws);
  red_partial_kernel<<<kRedBlocks, kRedThreads, 0, s>>>(n, x, y, mode, part);
  red_final_kernel<<<1, kRedThreads, 0, s>>>(part, kRedBlocks, part + kRedBlocks);
  QWB_LAUNCH_CHECK(ctx, "reduce kernels");
  D2* pin = reinterpret_cast<D2*>(ctx->pinned);
  QWB_CUDA(ctx, cudaMemcpyAsync(pin, part + kRedBlocks, sizeof(D2), cudaMemcpyDeviceToHost, s));
  QWB_CUDA(ctx, cudaStreamSynchronize(s));
  *result = *pin;
  return QWB_OK;
}

}  // namespace

extern "C" {

int qwb_prob_arcs(qwb_ctx* ctx, int64_t n, const int64_t* tail_offsets, const qwb_z* psi, double* p,
                  void* stream) {
  QWB_BEGIN(ctx);
  prob_arcs_kernel<<<qwb::blocks_for(n, 256, (int64_t)ctx->num_sms * 32), 256, 0,
                     qwb::as_stream(stream)>>>(n, tail_offsets,
                                               reinterpret_cast<const double2*>(psi), p);
  QWB_LAUNCH_CHECK(ctx, "prob_arcs_kernel");
  return QWB_OK;
}

int qwb_prob_abs2(qwb_ctx* ctx, int64_t n, const qwb_z* psi, double* p, void* stream) {
  QWB_BEGIN(ctx);
  prob_abs2_kernel<<<qwb::blocks_for(n, 256, (int64_t)ctx->num_sms * 32), 256, 0,
                     qwb::as_stream(stream)>>>(n, reinterpret_cast<const double2*>(psi), p);
  QWB_LAUNCH_CHECK(ctx, "prob_abs2_kernel");
  return QWB_OK;
}

int qwb_axpy(qwb_ctx* ctx, int64_t n, qwb_z alpha, const qwb_z* x, const qwb_z* y, qwb_z* out,
             void* stream) {
  QWB_BEGIN(ctx);
  axpy_kernel<<<qwb::blocks_for(n, 256, (int64_t)ctx->num_sms * 32), 256, 0, qwb::as_stream(stream)>>>(
      n, make_double2(alpha.re, alpha.im), reinterpret_cast<const double2*>(x),
      reinterpret_cast<const double2*>(y), reinterpret_cast<double2*>(out));
  QWB_LAUNCH_CHECK(ctx, "axpy_kernel");
  return QWB_OK;
}

int qwb_scale(qwb_ctx* ctx, int64_t n, qwb_z alpha, const qwb_z* x, qwb_z* out, void* stream) {
  QWB_BEGIN(ctx);
  scale_kernel<<<qwb::blocks_for(n, 256, (int64_t)ctx->num_sms * 32), 256, 0, qwb::as_stream(stream)>>>(
      n, make_double2(alpha.re, alpha.im), reinterpret_cast<const double2*>(x),
      reinterpret_cast<double2*>(out));
  QWB_LAUNCH_CHECK(ctx, "scale_kernel");
  return QWB_OK;
}

int qwb_dot(qwb_ctx* ctx, int64_t n, const qwb_z* x, const qwb_z* y, qwb_z* result_host,
            void* stream) {
  QWB_BEGIN(ctx);
  D2 r;
  int st = reduce2(ctx, n, reinterpret_cast<const double2*>(x), reinterpret_cast<const double2*>(y), 0,
                   &r, qwb::as_stream(stream));
  if (st) return st;
  result_host->re = r.a;
  result_host->im = r.b;
  return QWB_OK;
}

int qwb_norm(qwb_ctx* ctx, int64_t n, const qwb_z* x, double* result_host, void* stream) {
  QWB_BEGIN(ctx);
  D2 r;
  int st = reduce2(ctx, n, reinterpret_cast<const double2*>(x), nullptr, 1, &r, qwb::as_stream(stream));
  if (st) return st;
  *result_host = sqrt(r.a + r.b);
  return QWB_OK;
}

int qwb_check_finite(qwb_ctx* ctx, int64_t n_doubles, const double* x, int* all_finite_host,
                     void* stream) {
  QWB_BEGIN(ctx);
  cudaStream_t s = qwb::as_stream(stream);
  void* ws;
  int st = qwb::workspace(ctx, sizeof(int), s, &ws);
  if (st) return st;
  int* d = reinterpret_cast<int*>(ws);
  QWB_CUDA(ctx, cudaMemsetAsync(d, 0, sizeof(int), s));
  if (n_doubles > 0) {
    finite_kernel<<<qwb::blocks_for(n_doubles, 256, (int64_t)ctx->num_sms * 16), 256, 0, s>>>(n_doubles, x, d);
    QWB_LAUNCH_CHECK(ctx, "finite_kernel");
  }
  int* pin = reinterpret_cast<int*>(ctx->pinned);
  QWB_CUDA(ctx, cudaMemcpyAsync(pin, d, sizeof(int), cudaMemcpyDeviceToHost, s));
  QWB_CUDA(ctx, cudaStreamSynchronize(s));
  *all_finite_host = *pin ? 0 : 1;
  return QWB_OK;
}

}  // extern "C"
