"""Parity on the headline configuration (BASELINE.json configs[1]: 64 tag codes
x 1 s of 8 Ms/s I/Q = 11 windows x the 9-bin lo_freq sweep) and on the
1024-code roster (configs[2]) -- the multi-wave, multi-stream correlation
pipeline with M-ring reuse that bench.py times -- against the reference
compiled in place (oracle/_ref).

Inputs come from the compiled reference's own generator
(generate_recording, proj/src/recording.cpp:177-219): 16 of the 64 codes
injected at known fractional arrival times, carrier offsets U(-200, 200) kHz
and SNRs {0, 5, 10, 20} dB over a 10 dB noise floor.  Both paths see the same
int16.  The B200 side runs the whole stream through tdg_search (every window x
bin x code in one call: 396 correlation waves over the six stream pairs, the M
ring reused 132 times) and through the device CircularBuffer path
(tdg_ring_push + tdg_search_ring, bench.py's e2e); the reference runs
demodulate_window + detect per (window, bin) (recording.cpp:277-286).

Compared: every record of windows {0, 5, 10} x 9 bins x 64 codes (1,728
detections), and window 3 x bin +100 kHz x all 1024 roster codes.  Peak
indices and accept/partial exact except near-ties, which are documented with
their margin on the reference's own xc; the worst |delta| per field is
reported.  TDG_PARITY_OUT=<dir> writes the report (parity_cfg2.md / .json)."""
import os

import numpy as np
import pytest

from parity import ParityReport, compare_detections
from paritycheck import RefSlots

pytestmark = pytest.mark.gpu

W = 800000
ADV = 720000
FS = 8.0e6
BINS = np.arange(-400e3, 400e3 + 1.0, 100e3)
CHECK_WINDOWS = (0, 5, 10)


def cfg2_scene(ref, n_codes=64, n_inject=16, seed=7):
    """The cfg2 scene from the compiled reference's generate_recording."""
    from paper_2005_10445_b200._abi import demod_config
    cfg = demod_config()
    seeds = [1000 + i for i in range(n_codes)]
    rng = np.random.default_rng(seed)
    snrs = [0.0, 5.0, 10.0, 20.0]
    inj = []
    for k in range(n_inject):
        t = float(rng.uniform(0.0, 1.0 - 0.0085))
        g = 10.0 ** ((snrs[k % 4] - 10.0) / 20.0)
        inj.append((k, t, g, float(rng.uniform(-200e3, 200e3))))
    iq = ref.generate_recording(cfg, seeds, 1.0, 10.0, seed, inj)
    bits = np.stack([ref.gen_code(s, cfg) for s in seeds])
    return cfg, bits, iq, inj


def _write_report(reports, extra):
    out = os.environ.get("TDG_PARITY_OUT")
    if not out:
        return
    os.makedirs(out, exist_ok=True)
    md = ["# Parity on the headline configuration (B200 vs oracle/_ref)", "", extra, ""]
    md += [r.markdown() for r in reports]
    with open(os.path.join(out, "parity_cfg2.md"), "a") as f:
        f.write("\n".join(md) + "\n")
    import json
    with open(os.path.join(out, "parity_cfg2.json"), "a") as f:
        for r in reports:
            f.write(json.dumps(r.summary(), default=str) + "\n")


@pytest.fixture(scope="module")
def scene(ref):
    return cfg2_scene(ref)


def test_cfg2_sweep_against_reference(gpu_ctx, ref, scene):
    from paper_2005_10445_b200 import capi
    cfg, bits, iq, inj = scene
    n = iq.size // 2
    n_win = (n - W) // ADV + 1
    assert n_win == 11
    cs = capi.CodeSet.prepare(gpu_ctx, cfg, W, bits)
    got = capi.search(gpu_ctx, cfg, BINS, iq, cs, W, ADV)
    assert got.size == n_win * BINS.size * len(bits)
    # the e2e path of bench.py: device CircularBuffer + tdg_search_ring, bitwise equal
    ring = capi.Ring(gpu_ctx, 3 * n)
    ring.push(iq, 0)
    got_ring = capi.search_ring(gpu_ctx, ring, cfg, BINS, 0, n_win, cs, ADV)
    assert got_ring.tobytes() == got.tobytes()
    got = got.reshape(n_win, BINS.size, len(bits))
    threads = os.cpu_count() or 1
    rs = RefSlots(ref, cfg, bits, iq, W)
    rs.prefetch(slots=[(wi * ADV, lo) for wi in CHECK_WINDOWS for lo in BINS], codes=range(len(bits)))
    rep = ParityReport("cfg2: windows %s x 9 bins x 64 codes (tdg_search, 396 waves)" % (CHECK_WINDOWS,))
    allbad = []
    for wi in CHECK_WINDOWS:
        s0 = wi * ADV
        _, want, _ = ref.search_bench_shared(iq[2 * s0:2 * (s0 + W)], s0, cfg, BINS, bits, W, ADV, 1, 0.25, threads,
                                             code_chunk=2)
        want = want.reshape(BINS.size, len(bits))
        for b in range(BINS.size):
            bad = rs.compare(got[wi, b], want[b], s0, BINS[b], FS, report=rep)
            allbad += [(wi, b) + tuple(x) for x in bad]
    # every injected packet of SNR >= 5 dB wholly inside a window is found at
    # its nearest bin with |ToA error| < 0.5 sample (harness.cpp:58-73's
    # gate); 0 dB packets are reported, not required (the reference misses
    # some of them too -- the records are compared above)
    found, found0, n0 = 0, 0, 0
    for ci, t, g, foff in inj:
        a = t * FS
        b = int(np.argmin(np.abs(BINS - foff)))
        snr = 10.0 + 20.0 * np.log10(g)
        for wi in range(n_win):
            s0 = wi * ADV
            if s0 <= a and a + 65536 + 256 <= s0 + W:
                r = got[wi, b, ci]
                hit = bool(r["accepted"]) and abs(float(r["toa_seconds"]) * FS - a) < 0.5
                if snr >= 5.0:
                    assert hit, (ci, t, foff, wi, float(r["score"]), float(r["toa_seconds"]) * FS, a)
                    found += 1
                else:
                    n0 += 1
                    found0 += int(hit)
    acc = got["accepted"]
    injected = {ci for ci, _, _, _ in inj}
    spurious = [(w, b, c) for w, b, c in zip(*np.nonzero(acc)) if int(c) not in injected]
    _write_report([rep], "Scene: compiled reference generate_recording, 64 codes gen_code(1000+i), 16 injected "
                         "(SNR 0/5/10/20 dB, offsets U(-200,200) kHz), noise 10 dB, seed 7.  B200: tdg_search over "
                         "the whole second (11 windows x 9 bins x 64 codes = 6,336 detections) and tdg_search_ring "
                         "(bitwise equal).  Injected packets (SNR >= 5 dB) found at their nearest bin with |ToA err| "
                         "< 0.5 sample: %d; 0 dB packets found: %d of %d; accepted detections of absent codes: %d."
                         % (found, found0, n0, len(spurious)))
    assert not spurious, spurious[:10]
    assert found >= 12
    assert not allbad, allbad[:20]
    assert rep.records == len(CHECK_WINDOWS) * BINS.size * len(bits)
    _assert_plain_tolerance(rep)


def test_roster_1024_against_reference(gpu_ctx, ref, scene):
    """configs[2] roster: 1024 codes (512 stored pairs = 256 code-pair groups,
    64 correlation waves, M ring reuse) on one window x one nonzero bin."""
    from paper_2005_10445_b200 import capi
    from paper_2005_10445_b200._abi import demod_config
    cfg, bits64, iq, inj = scene
    bits = np.concatenate([bits64, np.stack([ref.gen_code(1064 + i, cfg) for i in range(1024 - 64)])])
    wi, lo = 3, 100e3
    s0 = wi * ADV
    cs = capi.CodeSet.prepare(gpu_ctx, cfg, W, bits)
    win = capi.Windows(gpu_ctx, W, 1, 1)
    win.demodulate(cfg, [lo], iq[2 * s0:2 * (s0 + W)], s0, W, 1)
    got = capi.detect(gpu_ctx, win, cs, 0.25, FS)
    threads = os.cpu_count() or 1
    _, want, _ = ref.search_bench_shared(iq[2 * s0:2 * (s0 + W)], s0, demod_config(), [lo], bits, W, ADV, 1, 0.25,
                                         threads, code_chunk=4)
    want["bin"] = 0
    rs = RefSlots(ref, cfg, bits, iq, W)
    rs.prefetch(slots=[(s0, lo)], codes=range(len(bits)))
    rep = ParityReport("cfg3 roster: window 3 x bin +100 kHz x 1024 codes (64 waves, 256 code-pair groups)")
    bad = rs.compare(got, want, s0, lo, FS, report=rep)
    _write_report([rep], "")
    assert not bad, bad[:20]
    assert rep.records == 1024
    _assert_plain_tolerance(rep)


def _assert_plain_tolerance(rep):
    """SURVEY 8(c)'s plain bounds hold outright on every accepted record
    (the conditioning-aware bound of tests/parity.py is only needed for weak,
    rejected peaks): sub-sample offset / ToA within 1e-4 samples, peak value,
    w_c, q, p_c and score within 1e-4 relative."""
    m = rep.max_rel_accepted
    assert m["subsample_offset"] <= 1e-4 and m["toa_samples"] <= 1e-4, m
    for f in ("peak_value", "w_c", "q", "p_c", "score"):
        assert m[f] <= 1e-4, (f, m[f])
