#!/usr/bin/env python3
"""Generate straight-line register DFT codelets for the B200 FFT kernels.

Writes paper_2005_10445_b200/csrc/codelets.cuh: for every size R in SIZES and
both directions, a fully unrolled `dft<R, SIGN>(float2 (&x)[R])` computing
    X[k] = sum_j x[j] * exp(SIGN * 2*pi*i*j*k/R)      (unnormalised)
in place, in natural order.  Composite sizes use mixed-radix decimation in
time (radix 4 first, then 2, 3, 5, 7); odd primes use the symmetric
(x_j +/- x_{R-j}) form; twiddles are compile-time constants computed in
double and rounded once to float, with the trivial ones (1, -1, +-i,
(+-1 +-i)/sqrt2) special-cased so no multiply is spent on them.

This is the B200 replacement for the per-stage butterflies FFTW executes
inside fftwf_execute (reference proj/src/fft.cpp:51,62); the codelets run
entirely in registers, so a CTA-level FFT of length P*Q needs only one
shared-memory exchange.
"""
import math
import os
import sys

SIZES = [2, 3, 4, 5, 6, 7, 8, 9, 10, 12, 14, 15, 16, 18, 20, 21, 24, 25, 27, 28, 30, 32, 35, 36]


class Em:
    def __init__(self):
        self.lines = []
        self.n = 0

    def tmp(self, expr):
        self.n += 1
        name = f"v{self.n}"
        self.lines.append(f"    const float {name} = {expr};")
        return name


def lit(v):
    s = repr(float(v))
    if "e" not in s and "." not in s:
        s += ".0"
    return s + "f"


def neg(a):
    return a[1:] if a.startswith("-") else "-" + a


def add(e, a, b):
    if b.startswith("-"):
        return e.tmp(f"{a} - {b[1:]}")
    if a.startswith("-"):
        return e.tmp(f"{b} - {a[1:]}")
    return e.tmp(f"{a} + {b}")


def sub(e, a, b):
    return add(e, a, neg(b))


def cadd(e, a, b):
    return (add(e, a[0], b[0]), add(e, a[1], b[1]))


def csub(e, a, b):
    return (sub(e, a[0], b[0]), sub(e, a[1], b[1]))


def cneg(a):
    return (neg(a[0]), neg(a[1]))


def cmul_i(a, s):
    # multiply by s*i (s = +1 or -1): (re, im) -> (-s*im, s*re)
    return (neg(a[1]) if s > 0 else a[1], a[0] if s > 0 else neg(a[0]))


def cmul_const(e, a, num, den, sign):
    """a * exp(sign*2*pi*i*num/den)."""
    num %= den
    if num == 0:
        return a
    if (4 * num) % den == 0:
        q = (4 * num) // den  # quarter turns
        if q == 2:
            return cneg(a)
        return cmul_i(a, sign if q == 1 else -sign)
    if (8 * num) % den == 0:
        o = (8 * num) // den  # odd eighth turn: 1,3,5,7
        h = lit(math.sqrt(0.5))
        # exp(sign*i*pi*o/4) = (cx + i*sy)/sqrt2 with cx, sy in {+1, -1}
        cx = 1 if o in (1, 7) else -1
        sy = (1 if o in (1, 3) else -1) * sign
        re, im = a
        # (re + i im)(cx + i sy) = (cx re - sy im) + i (sy re + cx im)
        r_re = e.tmp(f"({sgn(cx, re)} {'-' if sy > 0 else '+'} {par(im)}) * {h}")
        r_im = e.tmp(f"({sgn(sy, re)} {'+' if cx > 0 else '-'} {par(im)}) * {h}")
        return (r_re, r_im)
    ang = 2.0 * math.pi * num / den
    c = math.cos(ang)
    s = sign * math.sin(ang)
    re, im = a
    r_re = e.tmp(f"{par(re)} * {lit(c)} - {par(im)} * {lit(s)}")
    r_im = e.tmp(f"{par(re)} * {lit(s)} + {par(im)} * {lit(c)}")
    return (r_re, r_im)


def sgn(s, x):
    return par(x) if s > 0 else f"-{par(x)}"


def par(x):
    return f"({x})" if x.startswith("-") else x


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
    # odd prime: symmetric form
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
        pre, pim = x0
        qre, qim = None, None
        for j in range(1, h + 1):
            c = math.cos(2.0 * math.pi * j * k / r)
            s = math.sin(2.0 * math.pi * j * k / r)
            a = A[j - 1]
            b = B[j - 1]
            pre = e.tmp(f"{par(pre)} + {par(a[0])} * {lit(c)}")
            pim = e.tmp(f"{par(pim)} + {par(a[1])} * {lit(c)}")
            if qre is None:
                qre = e.tmp(f"{par(b[0])} * {lit(s)}")
                qim = e.tmp(f"{par(b[1])} * {lit(s)}")
            else:
                qre = e.tmp(f"{qre} + {par(b[0])} * {lit(s)}")
                qim = e.tmp(f"{qim} + {par(b[1])} * {lit(s)}")
        iq = cmul_i((qre, qim), sign)  # sign*i*Q
        out[k] = cadd(e, (pre, pim), iq)
        out[r - k] = csub(e, (pre, pim), iq)
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


def gen(n, sign):
    e = Em()
    xs = []
    for j in range(n):
        xs.append((e.tmp(f"x[{j}].x"), e.tmp(f"x[{j}].y")))
    out = dft(e, xs, sign)
    body = list(e.lines)
    for k, (re, im) in enumerate(out):
        body.append(f"    x[{k}] = make_float2({re}, {im});")
    flops = sum(l.count("+") + l.count(" - ") + l.count("*") for l in e.lines)
    head = f"// {n}-point DFT, sign {sign:+d}: {len(e.lines) - 2 * n} scalar ops (~{flops} flops)\n"
    head += f"template <> __device__ __forceinline__ void dft<{n}, {sign}>(float2 (&x)[{n}]) {{\n"
    return head + "\n".join(body) + "\n}\n"


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(
        os.path.dirname(__file__), "..", "paper_2005_10445_b200", "csrc", "codelets.cuh")
    parts = [
        "// GENERATED by tools/gen_codelets.py -- do not edit.\n"
        "// Straight-line register DFT codelets (see the generator docstring).\n"
        "#pragma once\n#include <cuda_runtime.h>\n\n"
        "namespace tdg {\n\n"
        "template <int R, int SIGN> __device__ __forceinline__ void dft(float2 (&x)[R]);\n\n"
        "template <> __device__ __forceinline__ void dft<1, -1>(float2 (&)[1]) {}\n"
        "template <> __device__ __forceinline__ void dft<1, 1>(float2 (&)[1]) {}\n\n"
    ]
    for n in SIZES:
        for sign in (-1, 1):
            parts.append(gen(n, sign))
    parts.append("}  // namespace tdg\n")
    with open(out, "w") as f:
        f.write("\n".join(parts))
    print("wrote", out)


if __name__ == "__main__":
    main()
