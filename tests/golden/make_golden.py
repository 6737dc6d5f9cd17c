"""Regenerate the golden fixtures from the reference compiled in place
(oracle/_ref/libtagdsp_ref.so, built by `make -C oracle ref` from
/root/reference/proj/src).  Run here, where /root/reference exists; the
fixtures travel with the repo so the oracle stays pinned on the GPU box.

  desk_e2e.npz    desk-scale (1 Ms/s, 1024-bit) window at 10 dB: iq, d, u,
                  code bits, replicas, xc rows and the reference Detections
  lo_demod.npz    8 Ms/s window demodulated at lo_freq = 123 kHz
  golden.json     the reference test suites' inline known answers
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [os.path.join(ROOT, "oracle"), ROOT]
import refpy  # noqa: E402
from paper_2005_10445_b200._abi import DETECTION_DTYPE, demod_config, desk_config  # noqa: E402


def main():
    cfg = desk_config(1024)
    W = 1024 * 8 + 1000
    seeds = [100, 101, 102, 103]
    bits = np.stack([refpy.gen_code(s, cfg) for s in seeds])
    iq = refpy.channel_window(bits[0], cfg, 12.25, W, 55, snr_db=10.0)
    d, u = refpy.demodulate_window(iq, 0, cfg)
    s = refpy.Session()
    idx = [s.prepare_code(bits[i], cfg, W, "c%d" % i) for i in range(len(seeds))]
    reps = [s.code_replica(i) for i in idx]
    info = [s.code_info(i) for i in idx]
    xc = s.batch_xcorr(d, idx)
    det = s.detect(d, u, idx, 0.25, 0, cfg.mod.sample_rate)
    np.savez_compressed(os.path.join(HERE, "desk_e2e.npz"), iq=iq, d=d, u=u, bits=bits, xc=xc,
                        det=det.view(np.uint8), nonzero=np.array([x["nonzero_len"] for x in info]),
                        energy=np.array([x["energy"] for x in info], np.float32),
                        corr_len=np.array([x["corr_len"] for x in info]),
                        **{"rep%d" % i: r for i, r in enumerate(reps)})
    cfg8 = demod_config(lo_freq=123e3)
    iq8 = refpy.channel_window(refpy.gen_code(9, demod_config()), demod_config(), 500.5, 100000, 3, snr_db=5.0)
    d8, u8 = refpy.demodulate_window(iq8, 777, cfg8)
    np.savez_compressed(os.path.join(HERE, "lo_demod.npz"), iq=iq8, d=d8, u=u8, start=777, lo=123e3)
    g = {
        "gen_code_seed7_16bits": refpy.gen_code(7, demod_config(packet_bits=16)).tolist(),
        "hamming_seed42_43": int((refpy.gen_code(42, demod_config()) != refpy.gen_code(43, demod_config())).sum()),
        "pad_length": {str(n): refpy.pad_length(n) for n in (1, 1000, 101, 828, 161743, 865743)},
        "find_peak": [[[0.0, -5.0, 3.0], list(refpy.find_peak(np.array([0.0, -5.0, 3.0], np.float32)))],
                      [[2.0, 2.0], list(refpy.find_peak(np.array([2.0, 2.0], np.float32)))]],
        "interpolate_peak": [[[0.5, 1.0, 0.5], 1, refpy.interpolate_peak(np.array([0.5, 1.0, 0.5], np.float32), 1)],
                             [[1.0, 1.0, 1.0], 1, refpy.interpolate_peak(np.array([1.0, 1.0, 1.0], np.float32), 1)],
                             [[0.4, 1.0, 0.6], 1, refpy.interpolate_peak(np.array([0.4, 1.0, 0.6], np.float32), 1)]],
        "gaussian_seed5_first8": refpy.gaussian(5, 8).tolist(),
        "sources": "proj/tests/test_codegen.cpp:39-51, test_dsp.cpp:132-137, test_detector.cpp:153-181",
    }
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(g, f, indent=1)
    print("fixtures written")


if __name__ == "__main__":
    main()
