"""Execute the generated CUDA codelets on the CPU by translating their
straight-line bodies to Python, and compare with a float64 DFT."""
import re

import numpy as np

_HDR = re.compile(r"template <> __device__ __forceinline__ void dft<(\d+), (-?\d+)>\(float2 \(&x\)\[\d+\]\) \{\n(.*?)\n\}\n", re.S)


def parse_codelets(path):
    src = open(path).read()
    out = {}
    for m in _HDR.finditer(src):
        n, sign, body = int(m.group(1)), int(m.group(2)), m.group(3)
        py = []
        for line in body.splitlines():
            line = line.strip()
            if line.startswith("const float "):
                line = line[len("const float "):].rstrip(";")
            elif line.startswith("x[") and "make_float2" in line:
                k = line[2:line.index("]")]
                args = line[line.index("make_float2(") + len("make_float2("):line.rindex(")")]
                a, b = [s.strip() for s in args.split(",")]
                line = f"out[{k}] = complex({a}, {b})"
            line = re.sub(r"x\[(\d+)\]\.x", r"x[\1].real", line)
            line = re.sub(r"x\[(\d+)\]\.y", r"x[\1].imag", line)
            line = re.sub(r"(\d\.\d*(?:e[-+]?\d+)?)f\b", r"\1", line)
            py.append(line)
        out[(n, sign)] = "\n".join(py)
    return out


def run_codelet(code, x):
    env = {"x": list(x), "out": [0j] * len(x), "complex": complex}
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
