// Micro-benchmark: L2 -> SM bandwidth of 16-KB bulk copies (cp.async.bulk)
// into a ring of shared-memory stages, as hc_stream_kernel streams partner
// tiles.  Source: a 64 MB buffer (L2-resident after the warm-up), chunk k of
// CTA c = tile (c * 7919 + k * 104729) mod 4096.  Consumers: 16 warps that
// wait for a stage, read 2 x 16 B per lane per chunk and release it.
// usage: l2_stream <stage bytes / 16 KB: K> <stages> <chunks per CTA> <producers P> <buffer tiles (2^k)>
// K chunks share a stage and its barrier pair; producer thread p of the
// producer warp fills the stages s with s % P == p.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int CHUNK = 16384;
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint32_t b, uint32_t ph) {
  asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(b), "r"(ph) : "memory");
}
template <int K>
__global__ void __launch_bounds__(544, 1) k(const char* src, int ns, int nstage_loads, int np, double* out, uint32_t tmask) {
  extern __shared__ __align__(128) char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)ns * K * CHUNK);
  uint64_t* empty = full + ns;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < ns; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sa(full + s)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 16;\n" ::"r"(sa(empty + s)));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  double acc = 0;
  if (tid >= 512) {
    const int p = tid - 512;
    if (p < np) {
      uint32_t s = p, ph = 0;
      for (int c = p; c < nstage_loads; c += np) {
        wait(sa(empty + s), ph ^ 1);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sa(full + s)), "r"(K * CHUNK) : "memory");
#pragma unroll
        for (int q = 0; q < K; ++q) {
          const uint32_t tile = ((uint32_t)blockIdx.x * 7919u + (uint32_t)(c * K + q) * 104729u) & tmask;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(sa(sm + ((size_t)s * K + q) * CHUNK)),
                       "l"(src + (size_t)tile * CHUNK), "r"(CHUNK), "r"(sa(full + s)) : "memory");
        }
        s += np;
        if (s >= (uint32_t)ns) { s -= ns; ph ^= 1; }
      }
    }
  } else {
    uint32_t s = 0, ph = 0;
    for (int c = 0; c < nstage_loads; ++c) {
      wait(sa(full + s), ph);
#pragma unroll
      for (int q = 0; q < K; ++q) {
        const double2* ch = reinterpret_cast<const double2*>(sm + ((size_t)s * K + q) * CHUNK);
        const double2 a = ch[tid], b = ch[tid + 512];
        acc += a.x + b.y;
      }
      __syncwarp();
      if ((tid & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(sa(empty + s)) : "memory");
      if (++s == (uint32_t)ns) { s = 0; ph ^= 1; }
    }
  }
  if (acc == 12345.0) out[0] = acc;
}
template <int K>
void run(int ns, int nchunks, int np, uint32_t ntiles) {
  char* src; double* out;
  cudaMalloc(&src, (size_t)ntiles * CHUNK);
  cudaMemset(src, 0, (size_t)ntiles * CHUNK);
  cudaMalloc(&out, 8);
  const size_t smem = (size_t)ns * K * CHUNK + 2 * ns * 8;
  cudaFuncSetAttribute(k<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int loads = nchunks / K;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) k<K><<<sms, 544, smem>>>(src, ns, loads, np, out, ntiles - 1);
  cudaEventRecord(a);
  const int reps = 20;
  for (int i = 0; i < reps; ++i) k<K><<<sms, 544, smem>>>(src, ns, loads, np, out, ntiles - 1);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double bytes = (double)sms * loads * K * CHUNK;
  printf("buffer %u MB ", ntiles / 64);
  printf("K %d stages %d P %d chunks/CTA %d: %.1f us/launch, %.2f TB/s L2->SM (%s)\n", K, ns, np, loads * K,
         ms * 1e3 / reps, bytes * reps / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(src); cudaFree(out);
}
int main(int argc, char** argv) {
  const int K = argc > 1 ? atoi(argv[1]) : 1, ns = argc > 2 ? atoi(argv[2]) : 12;
  const int nchunks = argc > 3 ? atoi(argv[3]) : 388, np = argc > 4 ? atoi(argv[4]) : 1;
  const uint32_t ntiles = argc > 5 ? (uint32_t)atoi(argv[5]) : 4096u;   // power of two
  if (K == 2) run<2>(ns, nchunks, np, ntiles);
  else if (K == 3) run<3>(ns, nchunks, np, ntiles);
  else run<1>(ns, nchunks, np, ntiles);
  return 0;
}
