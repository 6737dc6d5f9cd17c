#!/usr/bin/env python3
"""Latency breakdown of one small tracking batch (tdg_track_device): host wall
time per call, and (under ncu) the kernels one call launches."""
import ctypes
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2005_10445_b200 import capi  # noqa: E402
from paper_2005_10445_b200._abi import DETECTION_DTYPE, TRACK_TASK_DTYPE, demod_config  # noqa: E402


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    lib = capi.lib()
    cfg = demod_config()
    bits, iq, inj, _ = bench.make_inputs(0, 1)
    n = iq.size // 2
    ctx = capi.Context(0)
    cs = capi.CodeSet.prepare(ctx, cfg, 96000, bits)
    iq_dev = torch.from_numpy(iq).to("cuda:0")
    tasks = np.zeros(B, dtype=TRACK_TASK_DTYPE)
    tasks["start"] = [int(t * 8e6) - 16000 for _, t, _, _ in inj[:B]] + [100000] * max(0, B - len(inj))
    tasks["code_index"] = [c for c, _, _, _ in inj[:B]] + [0] * max(0, B - len(inj))
    out = np.zeros(B, dtype=DETECTION_DTYPE)

    def call():
        capi._check(lib.tdg_track_device(ctx.handle, ctypes.byref(cfg), ctypes.c_void_p(iq_dev.data_ptr()), n, 0,
                                         capi._ptr(tasks), B, cs._h, 0.25, capi._ptr(out)))
    st = torch.cuda.ExternalStream(ctx.stream())

    def measure(label):
        for _ in range(20):
            call()
        ts, gs = [], []
        for _ in range(50):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record(st)
            call()
            e1.record(st)
            ts.append(time.perf_counter() - t0)
            e1.synchronize()
            gs.append(e0.elapsed_time(e1) * 1e3)
        print("B=%d %-28s wall p50 %.1f us (min %.1f), stream span p50 %.1f us" %
              (B, label, np.median(ts) * 1e6, np.min(ts) * 1e6, np.median(gs)))

    measure("default")
    for key, val in [("track_graphs", 0), ("one_stream", 1), ("n_streams", 1)]:
        ctx.set_option(key, val)
        measure("%s=%d" % (key, val))
    ctx.set_option("track_graphs", 1)
    ctx.set_option("one_stream", 0)
    ctx.set_option("n_streams", 2)
    measure("default")
    ctx.set_option("time_kernels", 1)
    ctx.kernel_time_reset()
    for _ in range(50):
        call()
    for k in ["demod", "fwd_pass1", "fwd_pass2", "stats"]:
        n_, ms = ctx.kernel_time(k)
        if n_:
            print("  %-10s %.1f us/call" % (k, ms / 50 * 1e3))
    ctx.set_option("time_kernels", 0)
    torch.cuda.cudart().cudaProfilerStart()
    call()
    torch.cuda.cudart().cudaProfilerStop()


if __name__ == "__main__":
    main()
