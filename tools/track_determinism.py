#!/usr/bin/env python3
"""Diagnostic: run one tracking batch repeatedly through the stream path and
the graph path and report any record that differs between runs."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import numpy as np  # noqa: E402

from paper_2005_10445_b200 import capi  # noqa: E402
from paper_2005_10445_b200._abi import demod_config  # noqa: E402
import refpy as ref  # noqa: E402


def main():
    cfg = demod_config()
    fs = cfg.mod.sample_rate
    W = 96000
    seeds = [2100 + i for i in range(4)]
    bits = np.stack([ref.gen_code(s, cfg) for s in seeds])
    inj = [(0, 0.0103, 1.0, 0.0), (2, 0.0412, 0.8, 0.0), (3, 0.0707, 1.0, 0.0)]
    iq = ref.generate_recording(cfg, seeds, 0.1, 10.0, 78, inj)
    st, co = [312900, 550027, 65850], [0, 1, 2]
    toas = [int(round(t * fs)) for _, t, _, _ in inj]
    rng = np.random.default_rng(5)
    batches = []
    for k in range(6):
        nb = 3 if k % 3 != 2 else 2
        starts = [int(toas[(k + i) % 3] - 16000 + rng.integers(-3000, 3000)) for i in range(nb)]
        codes = [int((k + i) % 4) for i in range(nb)]
        batches.append((starts, codes))
    with capi.Context(0) as ctx:
        cs = capi.CodeSet.prepare(ctx, cfg, W, bits)
        ctx.set_option("track_graphs", 0)
        want = [capi.track(ctx, cfg, iq, b[0], b[1], cs, 0.25) for b in batches]
        ctx.set_option("track_graphs", 1)
        for rep in range(3):
            for k, ((s_, c_), w) in enumerate(zip(batches, want)):
                got = capi.track(ctx, cfg, iq, s_, c_, cs, 0.25)
                print("rep %d batch %d %s" % (rep, k, "ok" if got.tobytes() == w.tobytes() else
                      "DIFF peaks %s vs %s" % (list(got["peak_index"]), list(w["peak_index"]))), flush=True)
            if rep == 0:
                try:
                    capi.track(ctx, cfg, iq, [10], [len(bits)], cs, 0.25)
                except capi.InvalidArgument:
                    print("bad batch rejected", flush=True)
    # first call on a fresh context against later calls (reads of memory
    # before its first write differ between the two)
    for trial in range(3):
        with capi.Context(0) as ctx:
            cs = capi.CodeSet.prepare(ctx, cfg, W, bits)
            ctx.set_option("track_graphs", 0)
            first = capi.track(ctx, cfg, iq, st, co, cs, 0.25)
            for b in batches:
                capi.track(ctx, cfg, iq, b[0], b[1], cs, 0.25)
            later = capi.track(ctx, cfg, iq, st, co, cs, 0.25)
            print("fresh-context trial %d: first %s later %s %s" % (
                trial, list(first["peak_index"]), list(later["peak_index"]),
                "same" if first.tobytes() == later.tobytes() else "DIFFERENT"), flush=True)
    with capi.Context(0) as ctx:
        cs = capi.CodeSet.prepare(ctx, cfg, W, bits)
        for graphs in (0, 1):
            ctx.set_option("track_graphs", graphs)
            outs = [capi.track(ctx, cfg, iq, st, co, cs, 0.25) for _ in range(40)]
            base = outs[0]
            for k, o in enumerate(outs):
                if o.tobytes() != base.tobytes():
                    for i in range(len(st)):
                        if o[i].tobytes() != base[i].tobytes():
                            print("graphs=%d run %d task %d: peak %d vs %d, score %.7g vs %.7g" %
                                  (graphs, k, i, o[i]["peak_index"], base[i]["peak_index"], o[i]["score"],
                                   base[i]["score"]))
            print("graphs=%d: %d distinct results over %d runs; peaks %s" %
                  (graphs, len({o.tobytes() for o in outs}), len(outs), [int(x) for x in base["peak_index"]]))


if __name__ == "__main__":
    main()
