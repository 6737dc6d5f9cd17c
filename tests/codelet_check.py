"""Execute the generated CUDA codelets (csrc/codelets.cuh, packed f32x2
form written by tools/gen_codelets.py) on the CPU by translating their
straight-line bodies to Python, and compare with a float64 DFT.

A packed value (64-bit register pair, lo = re, hi = im) is modelled as a
Python complex whose real/imag parts are the two lanes; the PTX f32x2 ops
act lane-wise."""
import re

import numpy as np

_HDR = re.compile(r"template <> __device__ __forceinline__ void dft<(\d+), (-?\d+)>\(float2 \(&x\)\[\d+\]\) \{\n(.*?)\n\}\n", re.S)


def _lanes(f):
    return lambda *a: complex(f(*[z.real for z in a]), f(*[z.imag for z in a]))


ENV = {
    "pk": lambda lo, hi: complex(lo, hi),
    "up": lambda v: v,
    "swp": lambda v: complex(v.imag, v.real),
    "add2": _lanes(lambda a, b: a + b),
    "sub2": _lanes(lambda a, b: a - b),
    "mul2": _lanes(lambda a, b: a * b),
    "fma2": _lanes(lambda a, b, c: a * b + c),
}


def parse_codelets(path):
    src = open(path).read()
    out = {}
    for m in _HDR.finditer(src):
        n, sign, body = int(m.group(1)), int(m.group(2)), m.group(3)
        py = []
        for line in body.splitlines():
            line = line.strip().rstrip(";")
            if line.startswith("const c2 "):
                line = line[len("const c2 "):]
            elif line.startswith("x[") and "= up(" in line:
                k = line[2:line.index("]")]
                line = f"out[{k}] = {line[line.index('=') + 1:].strip()}"
            line = re.sub(r"x\[(\d+)\]\.x", r"x[\1].real", line)
            line = re.sub(r"x\[(\d+)\]\.y", r"x[\1].imag", line)
            line = re.sub(r"(\d\.\d*(?:e[-+]?\d+)?)f\b", r"\1", line)
            py.append(line)
        out[(n, sign)] = "\n".join(py)
    return out


def run_codelet(code, x):
    env = dict(ENV, x=list(x), out=[0j] * len(x))
    exec(code, env)
    return np.array(env["out"])


def check_all(path, trials=3, seed=0):
    rng = np.random.default_rng(seed)
    worst = {}
    for (n, sign), code in parse_codelets(path).items():
        e = 0.0
        for _ in range(trials):
            x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
            got = run_codelet(code, x)
            k = np.arange(n)
            want = np.exp(sign * 2j * np.pi * np.outer(k, k) / n) @ x
            e = max(e, float(np.abs(got - want).max() / np.abs(want).max()))
        worst[(n, sign)] = e
    return worst
