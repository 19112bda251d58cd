"""Pure-Python model of numpy's complex128 reduction and multiply.

This is the arithmetic contract the CUDA kernels implement
(`paper_2406_08186_b200/csrc/qwb_numerics.cuh`):

* `np.add.reduceat` on a segment x0..x{k-1} returns x0 + pairwise(x1..x{k-1}),
  numpy's blocked pairwise sum over the interleaved (re, im) doubles:
  fewer than 4 complex -> sequential from -0.0; up to 64 complex -> four
  complex accumulators combined as (c0 + c1) + (c2 + c3) then the tail
  sequentially; more -> recursive halving at a multiple of 4 complex.
* complex multiply a*b (numpy's FMA SIMD path):
  re = fma(ar, br, -(ai*bi)),  im = fma(ar, bi, ai*br).

Pure-Python loops: small inputs only.  Test infrastructure.
"""

from __future__ import annotations

from fractions import Fraction


def _pw(a, lo, n):
    if n < 8:
        rr = -0.0
        ri = -0.0
        for i in range(0, n, 2):
            rr += a[lo + i]
            ri += a[lo + i + 1]
        return rr, ri
    if n <= 128:
        r = list(a[lo:lo + 8])
        i = 8
        while i < n - (n % 8):
            for j in range(8):
                r[j] += a[lo + i + j]
            i += 8
        rr = (r[0] + r[2]) + (r[4] + r[6])
        ri = (r[1] + r[3]) + (r[5] + r[7])
        while i < n:
            rr += a[lo + i]
            ri += a[lo + i + 1]
            i += 2
        return rr, ri
    n2 = n // 2
    n2 -= n2 % 8
    r1 = _pw(a, lo, n2)
    r2 = _pw(a, lo + n2, n - n2)
    return r1[0] + r2[0], r1[1] + r2[1]


def pairwise_reduceat(x) -> complex:
    flat = []
    for z in list(x)[1:]:
        flat += [float(z.real), float(z.imag)]
    rr, ri = _pw(flat, 0, len(flat))
    x0 = complex(x[0])
    return complex(x0.real + rr, x0.imag + ri)


def _fma(a, b, c):
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def cmul_fma(a, b) -> complex:
    a = complex(a)
    b = complex(b)
    return complex(_fma(a.real, b.real, -(a.imag * b.imag)), _fma(a.real, b.imag, a.imag * b.real))


def cabs_np(z) -> float:
    """numpy's SIMD complex absolute value: larger * sqrt(fma(r, r, 1)), r = smaller / larger."""
    import math
    re, im = abs(float(complex(z).real)), abs(float(complex(z).imag))
    larger, smaller = max(re, im), min(re, im)
    if larger == 0.0:
        return 0.0
    r = smaller / larger
    return math.sqrt(_fma(r, r, 1.0)) * larger
