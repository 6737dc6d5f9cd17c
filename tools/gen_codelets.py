#!/usr/bin/env python3
"""Generate PACKED-FP32 register DFT codelets for the B200 FFT kernels.

Writes paper_2005_10445_b200/csrc/codelets.cuh: for every size R in SIZES and
both directions, a fully unrolled `dft<R, SIGN>(float2 (&x)[R])` computing
    X[k] = sum_j x[j] * exp(SIGN * 2*pi*i*j*k/R)      (unnormalised)
in place, in natural order.

Every complex value is one 64-bit register pair and every operation is one
sm_100a packed instruction (PTX add/sub/mul/fma .rn.f32x2 -> SASS FADD2 /
FMUL2 / FFMA2), so a complex add costs one issue slot instead of two.
Multiplications by +-1 and +-i are kept lazy (a quarter-turn count carried
with each value) and folded into the next add/sub, where the swap of the
real/imaginary halves is free (SASS operand selector .F32x2.LO_HI) and the
signs come from a constant pair; a general complex constant costs FMUL2 +
FFMA2.  Composite sizes use mixed-radix decimation in time (radix 4 first,
then 2, 3, 5, 7); odd primes use the symmetric (x_j +/- x_{R-j}) form;
constants are computed in double and rounded once to float.

This is the B200 replacement for the per-stage butterflies FFTW executes
inside fftwf_execute (reference proj/src/fft.cpp:51,62).
"""
import math
import os
import sys

SIZES = [2, 3, 4, 5, 6, 7, 8, 9, 10, 12, 14, 15, 16, 18, 20, 21, 24, 25, 27, 28, 30, 32, 35, 36]


def lit(v):
    s = repr(float(v))
    if "e" not in s and "." not in s:
        s += ".0"
    return s + "f"


def pair(a, b):
    return f"pk({lit(a)}, {lit(b)})"


class Em:
    def __init__(self):
        self.lines = []
        self.n = 0
        self.ops = 0

    def tmp(self, expr, op=True):
        self.n += 1
        name = f"v{self.n}"
        self.lines.append(f"    const c2 {name} = {expr};")
        if op:
            self.ops += 1
        return name


# A complex value: (var, q) meaning var * i^q, q in 0..3.
def rot(a, k):
    return (a[0], (a[1] + k) % 4)


def cneg(a):
    return rot(a, 2)


def cmul_i(a, s):
    return rot(a, 1 if s > 0 else 3)


def add_rel(e, x, y, q):
    """x + y * i^q for plain vars x, y (one instruction)."""
    if q == 0:
        return e.tmp(f"add2({x}, {y})")
    if q == 2:
        return e.tmp(f"sub2({x}, {y})")
    if q == 1:   # x + i y = (x.re - y.im, x.im + y.re)
        return e.tmp(f"fma2(swp({y}), {pair(-1.0, 1.0)}, {x})")
    return e.tmp(f"fma2(swp({y}), {pair(1.0, -1.0)}, {x})")   # x - i y


def cadd(e, a, b):
    # a + b = i^qa (A + B i^(qb - qa))
    return (add_rel(e, a[0], b[0], (b[1] - a[1]) % 4), a[1])


def csub(e, a, b):
    return cadd(e, a, cneg(b))


def cmul_c(e, a, c, s):
    """a * (c + i s) for a general constant (quarter turns folded in)."""
    z = complex(c, s) * (1j ** a[1])
    c, s = z.real, z.imag
    t = e.tmp(f"mul2({a[0]}, {pair(c, c)})")
    return (e.tmp(f"fma2(swp({a[0]}), {pair(-s, s)}, {t})"), 0)


def fma_real(e, acc, a, c):
    """acc + a * c for a real constant c (one instruction)."""
    if acc is None:
        return (e.tmp(f"mul2({a[0]}, {pair(c, c)})"), a[1])
    q = (a[1] - acc[1]) % 4
    if q == 0:
        v = e.tmp(f"fma2({a[0]}, {pair(c, c)}, {acc[0]})")
    elif q == 2:
        v = e.tmp(f"fma2({a[0]}, {pair(-c, -c)}, {acc[0]})")
    elif q == 1:   # i a c = (-a.im c, a.re c)
        v = e.tmp(f"fma2(swp({a[0]}), {pair(-c, c)}, {acc[0]})")
    else:
        v = e.tmp(f"fma2(swp({a[0]}), {pair(c, -c)}, {acc[0]})")
    return (v, acc[1])


def cmul_const(e, a, num, den, sign):
    """a * exp(sign*2*pi*i*num/den)."""
    num %= den
    if num == 0:
        return a
    if (4 * num) % den == 0:
        q = (4 * num) // den
        return rot(a, (q * sign) % 4)
    ang = 2.0 * math.pi * num / den
    return cmul_c(e, a, math.cos(ang), sign * math.sin(ang))


def prime_dft(e, xs, sign):
    r = len(xs)
    if r == 1:
        return xs
    if r == 2:
        return [cadd(e, xs[0], xs[1]), csub(e, xs[0], xs[1])]
    if r == 4:
        t0 = cadd(e, xs[0], xs[2])
        t1 = csub(e, xs[0], xs[2])
        t2 = cadd(e, xs[1], xs[3])
        t3 = cmul_i(csub(e, xs[1], xs[3]), sign)
        return [cadd(e, t0, t2), cadd(e, t1, t3), csub(e, t0, t2), csub(e, t1, t3)]
    h = (r - 1) // 2
    A = [cadd(e, xs[j], xs[r - j]) for j in range(1, h + 1)]
    B = [csub(e, xs[j], xs[r - j]) for j in range(1, h + 1)]
    x0 = xs[0]
    acc = x0
    for a in A:
        acc = cadd(e, acc, a)
    out = [None] * r
    out[0] = acc
    for k in range(1, h + 1):
        p = x0
        qv = None
        for j in range(1, h + 1):
            c = math.cos(2.0 * math.pi * j * k / r)
            s = math.sin(2.0 * math.pi * j * k / r)
            p = fma_real(e, p, A[j - 1], c)
            qv = fma_real(e, qv, B[j - 1], s)
        iq = cmul_i(qv, sign)
        out[k] = cadd(e, p, iq)
        out[r - k] = csub(e, p, iq)
    return out


def choose_radix(n):
    if n % 4 == 0 and n != 4:
        return 4
    for p in (2, 3, 5, 7):
        if n % p == 0 and n != p:
            return p
    return n


def dft(e, xs, sign):
    n = len(xs)
    if n in (1, 2, 3, 4, 5, 7):
        return prime_dft(e, xs, sign)
    r = choose_radix(n)
    m = n // r
    ys = [dft(e, xs[j::r], sign) for j in range(r)]
    out = [None] * n
    for k in range(m):
        col = [cmul_const(e, ys[j][k], j * k, n, sign) for j in range(r)]
        z = prime_dft(e, col, sign) if r in (2, 3, 4, 5, 7) else dft(e, col, sign)
        for q in range(r):
            out[k + m * q] = z[q]
    return out


def materialize(e, a):
    v, q = a
    if q == 0:
        return v
    if q == 2:
        return e.tmp(f"mul2({v}, {pair(-1.0, -1.0)})")
    if q == 1:
        return e.tmp(f"mul2(swp({v}), {pair(-1.0, 1.0)})")
    return e.tmp(f"mul2(swp({v}), {pair(1.0, -1.0)})")


def gen(n, sign):
    e = Em()
    xs = [(e.tmp(f"pk(x[{j}].x, x[{j}].y)", op=False), 0) for j in range(n)]
    out = dft(e, xs, sign)
    outs = [materialize(e, o) for o in out]
    body = list(e.lines)
    for k, v in enumerate(outs):
        body.append(f"    x[{k}] = up({v});")
    head = f"// {n}-point DFT, sign {sign:+d}: {e.ops} packed ops\n"
    head += f"template <> __device__ __forceinline__ void dft<{n}, {sign}>(float2 (&x)[{n}]) {{\n"
    return head + "\n".join(body) + "\n}\n", e.ops


HELPERS = r"""
// Packed f32x2 helpers: a c2 is one 64-bit register pair (lo = re, hi = im).
typedef unsigned long long c2;
__device__ __forceinline__ c2 pk(float lo, float hi) {
    c2 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ float2 up(c2 v) {
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
    return r;
}
__device__ __forceinline__ c2 swp(c2 v) {   // (re, im) -> (im, re): a free operand selector in SASS
    const float2 t = up(v);
    return pk(t.y, t.x);
}
__device__ __forceinline__ c2 add2(c2 a, c2 b) {
    c2 d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ c2 sub2(c2 a, c2 b) {
    c2 d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ c2 mul2(c2 a, c2 b) {
    c2 d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ c2 fma2(c2 a, c2 b, c2 c) {
    c2 d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
"""


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(
        os.path.dirname(__file__), "..", "paper_2005_10445_b200", "csrc", "codelets.cuh")
    parts = [
        "// GENERATED by tools/gen_codelets.py -- do not edit.\n"
        "// Straight-line packed-FP32 register DFT codelets (see the generator docstring).\n"
        "#pragma once\n#include <cuda_runtime.h>\n\n"
        "namespace tdg {\n" + HELPERS + "\n"
        "template <int R, int SIGN> __device__ __forceinline__ void dft(float2 (&x)[R]);\n\n"
        "template <> __device__ __forceinline__ void dft<1, -1>(float2 (&)[1]) {}\n"
        "template <> __device__ __forceinline__ void dft<1, 1>(float2 (&)[1]) {}\n\n"
    ]
    for n in SIZES:
        for sign in (-1, 1):
            code, ops = gen(n, sign)
            parts.append(code)
    parts.append("}  // namespace tdg\n")
    with open(out, "w") as f:
        f.write("\n".join(parts))
    print("wrote", out)


if __name__ == "__main__":
    main()
