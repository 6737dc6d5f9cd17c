#!/usr/bin/env python3
"""Wall time of GPU code preparation (tdg_codeset_prepare) vs roster size,
cold and warm, with the device kernel time of the same call."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2005_10445_b200 import capi  # noqa: E402
from paper_2005_10445_b200._abi import demod_config  # noqa: E402


def main():
    cfg = demod_config()
    rng = np.random.default_rng(3)
    ctx = capi.Context(0)
    for n in [8, 64, 256, 64, 8]:
        bits = rng.integers(0, 2, size=(n, cfg.mod.packet_bits), dtype=np.uint8)
        ctx.synchronize()
        ctx.kernel_time_reset()
        ctx.set_option("time_kernels", 1)
        t0 = time.perf_counter()
        cs = capi.CodeSet.prepare(ctx, cfg, bench.W, bits)
        ctx.synchronize()
        t1 = time.perf_counter()
        ctx.set_option("time_kernels", 0)
        kt = {k: ctx.kernel_time(k) for k in ("demod", "fwd_pass1", "fwd_pass2")}
        t2 = time.perf_counter()
        cs.close()
        t3 = time.perf_counter()
        print("n=%4d prepare %.1f ms  close %.1f ms  kernels %s" % (
            n, (t1 - t0) * 1e3, (t3 - t2) * 1e3, {k: "%d x %.2f ms" % (v[0], v[1]) for k, v in kt.items()}), flush=True)


if __name__ == "__main__":
    main()
