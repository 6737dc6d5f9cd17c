#!/usr/bin/env python3
"""Tuning sweep of the fused correlation kernel's options on the bench
workload (cfg2).  Device-timed detect() per option set; prints one line each.

  python tools/sweep.py "wave_pairs=2,ring=3,a_share_pct=67" "a_share_pct=60" ...
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2005_10445_b200 import capi  # noqa: E402
from paper_2005_10445_b200._abi import demod_config  # noqa: E402


def main():
    lib = capi.lib()
    cfg = demod_config()
    bits, iq, _, _ = bench.make_inputs(0, 1)
    ctx = capi.Context(0)
    cs = capi.CodeSet.prepare(ctx, cfg, bench.W, bits)
    win = capi.Windows(ctx, bench.W, bench.N_WIN, len(bench.BINS))
    iq_dev = torch.from_numpy(iq).to("cuda:0")
    bins = np.ascontiguousarray(bench.BINS)
    capi._check(lib.tdg_demodulate_device(ctx.handle, win._h, ctypes.byref(cfg), capi._ptr(bins), bins.size,
                                          ctypes.c_void_p(iq_dev.data_ptr()), iq.size // 2, 0, bench.ADV, bench.N_WIN))
    stream = torch.cuda.ExternalStream(ctx.stream(), device="cuda:0")
    n_units = bench.N_CODES * bench.N_WIN * len(bins)
    ref = None
    for spec in sys.argv[1:] or [""]:
        for kv in filter(None, spec.split(",")):
            k, v = kv.split("=")
            ctx.set_option(k, int(v))
        for _ in range(2):
            capi._check(lib.tdg_detect(ctx.handle, win._h, cs._h, 0.25, bench.FS, None, 0))
        ctx.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        e0.record(stream)
        for _ in range(reps):
            capi._check(lib.tdg_detect(ctx.handle, win._h, cs._h, 0.25, bench.FS, None, 0))
        e1.record(stream)
        ctx.synchronize()
        ms = e0.elapsed_time(e1) / reps
        out = (ctypes.c_char * (n_units * 64))()
        capi._check(lib.tdg_detect(ctx.handle, win._h, cs._h, 0.25, bench.FS, out, n_units))
        h = hash(bytes(out))
        same = "" if ref is None else (" same-detections" if h == ref else " DIFFERENT-detections")
        ref = h if ref is None else ref
        print("%-40s detect %.3f ms  %.0f corr/s%s" % (spec, ms, n_units / ms * 1e3, same), flush=True)


if __name__ == "__main__":
    main()
