#!/usr/bin/env python3
"""CTA residency of the correlation passes over one detect() of the bench
workload (option "cta_trace", tdg_cta_trace): per SM, how many pass-A /
pass-B CTAs are resident over time, and how much of the 3-CTA-per-SM capacity
the step leaves unused (launch ramps, tails, dependency gaps)."""
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
    for _ in range(3):
        capi._check(lib.tdg_detect(ctx.handle, win._h, cs._h, 0.25, bench.FS, None, 0))
    cap = 400000
    ctx.set_option("cta_trace", cap)
    capi._check(lib.tdg_detect(ctx.handle, win._h, cs._h, 0.25, bench.FS, None, 0))
    buf = np.zeros(3 * cap, dtype=np.uint64)
    n = ctypes.c_uint64()
    capi._check(lib.tdg_cta_trace(ctx.handle, capi._ptr(buf), cap, ctypes.byref(n)))
    rec = buf[:3 * min(n.value, cap)].reshape(-1, 3).astype(np.int64)
    sm, typ = rec[:, 0] >> 8, rec[:, 0] & 255
    t0, t1 = rec[:, 1], rec[:, 2]
    T0, T1 = t0.min(), t1.max()
    span = (T1 - T0) / 1e3
    nsm = int(sm.max()) + 1
    print("records %d (A %d, B %d), span %.1f us, SMs %d" % (len(rec), (typ == 0).sum(), (typ == 1).sum(), span, nsm))
    busy = (t1 - t0).astype(np.float64)
    print("mean CTA lifetime: A %.1f us, B %.1f us" % (busy[typ == 0].mean() / 1e3, busy[typ == 1].mean() / 1e3))
    # resident-CTA count per SM over time (1 us bins)
    nb = int(np.ceil(span)) + 1
    occ = np.zeros((nsm, nb, 2))
    for s_, ty, a, b in zip(sm, typ, (t0 - T0) / 1e3, (t1 - T0) / 1e3):
        ia, ib = int(a), int(b)
        occ[s_, ia:ib + 1, ty] += 1.0
    tot = occ.sum(axis=2)
    print("CTA-slot utilisation (of 3 per SM): %.1f %%" % (100.0 * tot.mean() / 3.0))
    hist = np.bincount(np.minimum(tot, 4).astype(int).ravel(), minlength=5) / tot.size
    print("time share with 0/1/2/3/4+ resident CTAs: " + " ".join("%.1f%%" % (100 * h) for h in hist))
    mixes = {}
    for a_ in range(4):
        for b_ in range(4):
            m = ((occ[..., 0] == a_) & (occ[..., 1] == b_)).mean()
            if m > 0.005:
                mixes["%dA+%dB" % (a_, b_)] = round(100 * m, 1)
    print("A/B mixes:", mixes)


if __name__ == "__main__":
    main()
