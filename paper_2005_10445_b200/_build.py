"""In-tree build of the sm_100a shared library (libtagdsp_gpu.so).

nvcc cross-compiles for sm_100a without a GPU, so this runs in the CPU
container (the driver's build() check) and the resulting .so travels to the
GPU box with the repo snapshot."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libtagdsp_gpu.so")
SOURCES = ["tagdsp_gpu.cu", "records.cpp"]
# nlohmann/json (header-only, the version the oracle compiles the reference with)
NLOHMANN = os.environ.get("NLOHMANN", "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty")
DEPS = SOURCES + ["kernels.cuh", "codelets.cuh", "corr_v3.cuh", "tma.cuh", "peak.cuh", "generic.cuh"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, d) for d in DEPS] + [os.path.join(ROOT, "include", h)
                                                   for h in ("tagdsp_gpu.h", "tagdsp_gpu_types.h")]
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(force=False, verbose=False, defines=(), out=None):
    """Build the library (defines: extra -D flags of a layout variant, out:
    another path -- tools/ab_libs.sh A/B builds go to abtest/)."""
    target = out or LIB
    if not force and not defines and out is None and not stale():
        return LIB
    cmd = [_nvcc()] + NVCC_FLAGS + ["-D" + d for d in defines] + \
        ["-I" + os.path.join(ROOT, "include"), "-I" + CSRC, "-I" + NLOHMANN, "-o", target] + [os.path.join(CSRC, s) for s in SOURCES]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(HERE, "build.log") if out is None else target + ".log"
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stderr[-4000:])
        raise RuntimeError("nvcc failed building libtagdsp_gpu.so (see %s)" % log)
    if verbose:
        print("built", target)
    return target


if __name__ == "__main__":
    # python _build.py [--force] [-DNAME=V ...] [-o path]
    args = sys.argv[1:]
    defs = [a[2:] for a in args if a.startswith("-D")]
    out = args[args.index("-o") + 1] if "-o" in args else None
    build(force="--force" in args, verbose=True, defines=defs, out=out)
