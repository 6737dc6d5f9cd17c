"""Quick device-side timing of the correlation engine at the cfg2 shape
(64 codes x 11 windows x 9 bins, W = 800,000).  Development probe only."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2005_10445_b200 import capi  # noqa: E402
from paper_2005_10445_b200._abi import demod_config  # noqa: E402
import ctypes  # noqa: E402

cfg = demod_config()
rng = np.random.default_rng(1)
n_codes = int(os.environ.get("NC", 64))
n_win = int(os.environ.get("NW", 11))
bins = np.arange(-400e3, 400e3 + 1, 100e3)
W, adv = 800000, 720000
total = (n_win - 1) * adv + W
bits = rng.integers(0, 2, size=(n_codes, 8192), dtype=np.uint8)
iq = (rng.standard_normal(2 * total) * 2000).astype(np.int16)
ctx = capi.Context(0)
for k, v in [x.split("=") for x in sys.argv[1:]]:
    ctx.set_option(k, int(v))
t = time.time()
cs = capi.CodeSet.prepare(ctx, cfg, W, bits)
print("prepare %.3f s, corr_len %d, n %d" % (time.time() - t, cs.info(0)["corr_len"], cs.info(0)["nonzero_len"]))
win = capi.Windows(ctx, W, n_win, len(bins))
lib = capi.lib()
iq_dev = None
import torch  # noqa: E402  (plumbing only: device buffer + events)
iq_t = torch.from_numpy(iq).cuda()
st = torch.cuda.ExternalStream(ctx.stream())
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def step():
    capi._check(lib.tdg_demodulate_device(ctx.handle, win._h, ctypes.byref(cfg), capi._ptr(bins), bins.size,
                                          ctypes.c_void_p(iq_t.data_ptr()), total, 0, adv, n_win))
    capi._check(lib.tdg_detect(ctx.handle, win._h, cs._h, 0.25, cfg.mod.sample_rate, None, 0))


for _ in range(2):
    step()
ctx.synchronize()
reps = 3
ev0.record(st)
for _ in range(reps):
    step()
ev1.record(st)
ctx.synchronize()
ms = ev0.elapsed_time(ev1) / reps
ncorr = n_codes * n_win * len(bins)
print("step %.3f ms  -> %.0f corr/s  (%d corr)" % (ms, ncorr / ms * 1e3, ncorr))
# demod alone
ev0.record(st)
for _ in range(reps):
    capi._check(lib.tdg_demodulate_device(ctx.handle, win._h, ctypes.byref(cfg), capi._ptr(bins), bins.size,
                                          ctypes.c_void_p(iq_t.data_ptr()), total, 0, adv, n_win))
ev1.record(st)
ctx.synchronize()
print("demod %.3f ms per step" % (ev0.elapsed_time(ev1) / reps))
