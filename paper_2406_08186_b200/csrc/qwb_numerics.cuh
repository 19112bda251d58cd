// qwb_numerics.cuh — the reference's numpy arithmetic, restated for sm_100a.
//
// The library is compiled with --fmad=false, so every FMA below is explicit and
// no other multiply-add is contracted.  These device functions reproduce,
// bit for bit, the numpy 2.x primitives the reference calls:
//
//  * complex multiply `values * x[cols]`       (backend.py:400)
//      numpy SIMD: re = fma(ar, br, -(ai*bi)), im = fma(ar, bi, ai*br)
//  * `np.add.reduceat` over a CSR row            (backend.py:403, coined.py:292,
//      ctqw.py:119): out = x0 + pairwise(x1..x{k-1}); numpy's pairwise sum
//      (complex: over interleaved re/im doubles; real: over doubles)
//  * `np.abs(z)` for complex128                  (coined.py:289, ctqw.py:115,211)
//      numpy SIMD cabs: larger * sqrt(fma(r, r, 1)), r = smaller / larger
//  * `**2` -> x * x
//
// tests/tests_support_pairwise.py holds the same model in pure Python and
// tests/test_oracle.py pins it against numpy.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace qwb {

struct z2 { double x, y; };

__device__ __forceinline__ double2 cmul_np(double2 a, double2 b) {
  double2 r;
  r.x = __fma_rn(a.x, b.x, -__dmul_rn(a.y, b.y));
  r.y = __fma_rn(a.x, b.y, __dmul_rn(a.y, b.x));
  return r;
}

__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}

// numpy SIMD complex absolute value (loops_unary_complex simd_cabsolute).
__device__ __forceinline__ double cabs_np(double2 z) {
  double re = fabs(z.x), im = fabs(z.y);
  double larger = fmax(re, im), smaller = fmin(re, im);
  if (isinf(larger)) return larger;           // inf component -> inf (nan excluded upstream)
  if (larger == 0.0) return 0.0;
  double r = __ddiv_rn(smaller, larger);
  return __dmul_rn(__dsqrt_rn(__fma_rn(r, r, 1.0)), larger);
}

__device__ __forceinline__ double abs2_np(double2 z) {
  double a = cabs_np(z);
  return __dmul_rn(a, a);
}

// ---------------------------------------------------------------------------
// Pairwise sums.  `get(i)` returns element i (0-based) of the sequence to sum.
// numpy's count n is in doubles; for complex n = 2 * (#elements).
// ---------------------------------------------------------------------------

// complex: elements [lo, lo+m) of get()
template <class G>
__device__ __forceinline__ double2 pw_block_z(const G& get, int64_t lo, int64_t m) {
  // m complex elements, m <= 64 (numpy n = 2m <= 128)
  if (m < 4) {
    double2 r = make_double2(-0.0, -0.0);
    for (int64_t i = 0; i < m; ++i) r = cadd(r, get(lo + i));
    return r;
  }
  double2 c0 = get(lo), c1 = get(lo + 1), c2 = get(lo + 2), c3 = get(lo + 3);
  int64_t main_end = m - (m % 4);
  int64_t i = 4;
  for (; i < main_end; i += 4) {
    c0 = cadd(c0, get(lo + i));
    c1 = cadd(c1, get(lo + i + 1));
    c2 = cadd(c2, get(lo + i + 2));
    c3 = cadd(c3, get(lo + i + 3));
  }
  double2 r = cadd(cadd(c0, c1), cadd(c2, c3));
  for (; i < m; ++i) r = cadd(r, get(lo + i));
  return r;
}

// general m: numpy splits n doubles at n2 = n/2 - (n/2) % 8; with n = 2m
// that is m2 = (m - m % 8) / 2 complex elements.
template <class G>
__device__ double2 pw_z(const G& get, int64_t lo, int64_t m) {
  if (m <= 64) return pw_block_z(get, lo, m);
  // explicit stack (depth <= 40 for any int64 length)
  int64_t st_lo[48], st_m[48];
  int st_state[48];
  double2 st_acc[48];
  int sp = 0;
  st_lo[0] = lo; st_m[0] = m; st_state[0] = 0;
  double2 ret = make_double2(0.0, 0.0);
  while (sp >= 0) {
    int64_t clo = st_lo[sp], cm = st_m[sp];
    if (cm <= 64) {
      ret = pw_block_z(get, clo, cm);
      --sp;
      continue;
    }
    int64_t m2 = (cm - (cm % 8)) / 2;
    if (st_state[sp] == 0) {
      st_state[sp] = 1;
      ++sp; st_lo[sp] = clo; st_m[sp] = m2; st_state[sp] = 0;
    } else if (st_state[sp] == 1) {
      st_acc[sp] = ret;
      st_state[sp] = 2;
      ++sp; st_lo[sp] = clo + m2; st_m[sp] = cm - m2; st_state[sp] = 0;
    } else {
      ret = cadd(st_acc[sp], ret);
      --sp;
    }
  }
  return ret;
}

// reduceat over one segment of length k >= 1: x0 + pairwise(x1..)
template <class G>
__device__ __forceinline__ double2 reduceat_z(const G& get, int64_t k) {
  double2 x0 = get(0);
  if (k == 1) return x0;
  double2 rest = pw_z(get, 1, k - 1);
  return cadd(x0, rest);
}

// real pairwise: m doubles
template <class G>
__device__ __forceinline__ double pw_block_d(const G& get, int64_t lo, int64_t m) {
  if (m < 8) {
    double r = -0.0;
    for (int64_t i = 0; i < m; ++i) r = __dadd_rn(r, get(lo + i));
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = get(lo + j);
  int64_t main_end = m - (m % 8);
  int64_t i = 8;
  for (; i < main_end; i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], get(lo + i + j));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < m; ++i) res = __dadd_rn(res, get(lo + i));
  return res;
}

template <class G>
__device__ double pw_d(const G& get, int64_t lo, int64_t m) {
  if (m <= 128) return pw_block_d(get, lo, m);
  int64_t st_lo[48], st_m[48];
  int st_state[48];
  double st_acc[48];
  int sp = 0;
  st_lo[0] = lo; st_m[0] = m; st_state[0] = 0;
  double ret = 0.0;
  while (sp >= 0) {
    int64_t clo = st_lo[sp], cm = st_m[sp];
    if (cm <= 128) {
      ret = pw_block_d(get, clo, cm);
      --sp;
      continue;
    }
    int64_t m2 = cm / 2;
    m2 -= m2 % 8;
    if (st_state[sp] == 0) {
      st_state[sp] = 1;
      ++sp; st_lo[sp] = clo; st_m[sp] = m2; st_state[sp] = 0;
    } else if (st_state[sp] == 1) {
      st_acc[sp] = ret;
      st_state[sp] = 2;
      ++sp; st_lo[sp] = clo + m2; st_m[sp] = cm - m2; st_state[sp] = 0;
    } else {
      ret = __dadd_rn(st_acc[sp], ret);
      --sp;
    }
  }
  return ret;
}

template <class G>
__device__ __forceinline__ double reduceat_d(const G& get, int64_t k) {
  double x0 = get(0);
  if (k == 1) return x0;
  return __dadd_rn(x0, pw_d(get, 1, k - 1));
}

}  // namespace qwb
