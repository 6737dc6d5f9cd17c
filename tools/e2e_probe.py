#!/usr/bin/env python3
"""Where does the end-to-end step lose time against the device-resident one?
Times 20 steps (CUDA events on the context stream) of:
  device      tdg_demodulate_device + tdg_detect (bench.py `value`)
  ring_only   tdg_search_ring of a second pushed once (no per-step upload)
  ring_e2e    tdg_ring_push + tdg_search_ring every step (bench.py `e2e`)
  linear_h2d  tdg_search (pinned host -> device copy inside the call)
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
from paper_2005_10445_b200._abi import DETECTION_DTYPE, demod_config  # noqa: E402


def main():
    steps = 20
    lib = capi.lib()
    cfg = demod_config()
    bits, iq, _, _ = bench.make_inputs(0, 1)
    n = iq.size // 2
    ctx = capi.Context(0)
    cs = capi.CodeSet.prepare(ctx, cfg, bench.W, bits)
    win = capi.Windows(ctx, bench.W, bench.N_WIN, len(bench.BINS))
    iq_dev = torch.from_numpy(iq).to("cuda:0")
    iq_pin = torch.from_numpy(iq).pin_memory()
    n_units = len(bits) * bench.N_WIN * len(bench.BINS)
    out_pin = torch.empty(n_units * DETECTION_DTYPE.itemsize, dtype=torch.uint8).pin_memory()
    st = torch.cuda.ExternalStream(ctx.stream())
    bins = np.ascontiguousarray(bench.BINS)
    ring = capi.Ring(ctx, 3 * n)
    pos = [0]

    def device():
        capi._check(lib.tdg_demodulate_device(ctx.handle, win._h, ctypes.byref(cfg), capi._ptr(bins), bins.size,
                                              ctypes.c_void_p(iq_dev.data_ptr()), n, 0, bench.ADV, bench.N_WIN))
        capi._check(lib.tdg_detect(ctx.handle, win._h, cs._h, 0.25, bench.FS, None, 0))

    def search_ring(start):
        capi._check(lib.tdg_search_ring(ctx.handle, ring._h, ctypes.byref(cfg), capi._ptr(bins), bins.size, start,
                                        bench.W, bench.ADV, bench.N_WIN, cs._h, 0.25,
                                        ctypes.c_void_p(out_pin.data_ptr()), n_units, 0))

    def push(start):
        capi._check(lib.tdg_ring_push(ring._h, ctypes.c_void_p(iq_pin.data_ptr()), n, start, None))

    def ring_only():
        search_ring(pos[0] - n)

    def ring_e2e():
        push(pos[0])
        search_ring(pos[0])
        pos[0] += n

    def linear_h2d():
        capi._check(lib.tdg_search(ctx.handle, ctypes.byref(cfg), capi._ptr(bins), bins.size,
                                   ctypes.c_void_p(iq_pin.data_ptr()), n, 0, bench.W, bench.ADV, cs._h,
                                   0.25, ctypes.c_void_p(out_pin.data_ptr()), n_units, None))

    def timed(name, fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ctx.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(steps):
            fn()
        e1.record(st)
        e1.synchronize()
        ctx.synchronize()
        ms = e0.elapsed_time(e1) / steps
        print("%-11s %.3f ms/step  %.0f corr/s" % (name, ms, n_units / ms * 1e3), flush=True)

    timed("device", device)
    ring_e2e()
    timed("ring_only", ring_only)
    timed("ring_e2e", ring_e2e)
    timed("linear_h2d", linear_h2d)
    timed("device", device)


if __name__ == "__main__":
    main()
