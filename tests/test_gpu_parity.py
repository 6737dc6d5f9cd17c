"""GPU parity: the B200 path through the C-ABI against the reference compiled
in place (oracle/_ref) and brute-force oracles, on the reference's own test
cases (proj/tests/test_detector.cpp, acceptance.cpp) and the search shape."""
import numpy as np
import pytest

from parity import compare_detections, direct_xcorr, near_tie_margin

pytestmark = pytest.mark.gpu


def assert_d_conditioned(d, d_ref, u_ref, rel=1e-6):
    """|d - d_ref| <= rel * max(den) / den + 1e-6 with den = |u|/|d| = |f1|+|f0|
    (the discriminator's conditioning, proj/src/dsp.cpp:147-157), and at most
    1e-4 absolute wherever den >= 1e-2 * max(den)."""
    den = np.abs(u_ref).astype(np.float64) / np.maximum(np.abs(d_ref).astype(np.float64), 1e-30)
    den = np.where(np.abs(d_ref) > 0, den, 0.0)
    dm = den.max()
    err = np.abs(d.astype(np.float64) - d_ref)
    tol = rel * dm / np.maximum(den, 1e-30 * dm) + 1e-6
    assert (err <= tol).all(), (float(err.max()), int(np.argmax(err / tol)))
    good = den >= 1e-2 * dm
    assert err[good].max() <= 1e-4, float(err[good].max())


def _cs_from(capi, ctx, dcs, W, ref):
    n = max(len(x) for x in dcs)
    return capi.CodeSet.from_replicas(ctx, W, ref.pad_length(W + n), dcs, dcs)


def test_xcorr_matches_brute_force(gpu_ctx, ref):
    """test_detector.cpp:110-122: 20 random instances, |err| <= 1e-3 * energy."""
    from paper_2005_10445_b200 import capi
    worst = 0.0
    for trial in range(20):
        dc = ref.gaussian(100 + trial, 64)
        d = ref.gaussian(200 + trial, 4096)
        cs = _cs_from(capi, gpu_ctx, [dc], d.size, ref)
        w = capi.Windows(gpu_ctx, d.size)
        w.set_du(0, d, d)
        got = capi.batch_xcorr(gpu_ctx, w, 0, cs)[0]
        want = direct_xcorr(d, dc)
        e = cs.info(0)["energy"]
        worst = max(worst, float(np.abs(got - want).max() / e))
    assert worst <= 1e-4, worst


def test_batch_xcorr_matches_reference(gpu_ctx, ref):
    """batch_xcorr (detector.cpp:102-120) on 16 codes (odd/even pairing)."""
    from paper_2005_10445_b200 import capi
    W = 2048
    dcs = [ref.gaussian(8000 + i, 100) for i in range(15)]
    d = ref.gaussian(8999, W)
    cs = _cs_from(capi, gpu_ctx, dcs, W, ref)
    w = capi.Windows(gpu_ctx, W)
    w.set_du(0, d, d)
    got = capi.batch_xcorr(gpu_ctx, w, 0, cs)
    s = ref.Session()
    idx = [s.make_transformed(x, x, W, ref.pad_length(W + 100)) for x in dcs]
    want = s.batch_xcorr(d, idx)
    for i in range(len(dcs)):
        e = cs.info(i)["energy"]
        assert np.abs(got[i] - want[i]).max() <= 1e-5 * e


def test_autocorrelation_peak_is_energy(gpu_ctx, ref):
    """test_detector.cpp:89-99."""
    from paper_2005_10445_b200 import capi
    dc = ref.gaussian(5, 512)
    d = np.zeros(2048, np.float32)
    d[:512] = dc
    cs = _cs_from(capi, gpu_ctx, [dc], 2048, ref)
    w = capi.Windows(gpu_ctx, 2048)
    w.set_du(0, d, d)
    det = capi.detect(gpu_ctx, w, cs, 0.25, 1.0)[0]
    assert det["peak_index"] == 0
    assert abs(det["peak_value"] - cs.info(0)["energy"]) <= 1e-4 * cs.info(0)["energy"]


def test_demodulate_matches_reference_default_cfg(gpu_ctx, ref):
    """demodulate_window on a default-config search window, with LO bins."""
    from paper_2005_10445_b200 import capi
    from paper_2005_10445_b200._abi import demod_config
    cfg = demod_config()
    bits = ref.gen_code(1000, cfg)
    W = 200000
    iq = ref.channel_window(bits, cfg, 1000.25, W, 3, snr_db=10.0, freq_offset=50e3)
    bins = [0.0, 100e3, -100e3]
    win = capi.Windows(gpu_ctx, W, 1, len(bins))
    win.demodulate(cfg, bins, iq, stream_start=12345, advance=W, n_windows=1)
    for b, lo in enumerate(bins):
        c = demod_config(lo_freq=lo)
        d_ref, u_ref = ref.demodulate_window(iq, 12345, c)
        d, u = win.get_du(b)
        assert np.abs(u - u_ref).max() <= 1e-4 * np.abs(u_ref).max(), lo
        # d = u / (|f1| + |f0|): absolute fp32 errors e in |f| give
        # |dd| ~ 2e / (|f1| + |f0|), so near the causal start of the window
        # (0/0-like dust) d is ill-conditioned in BOTH implementations.
        assert_d_conditioned(d, d_ref, u_ref)


def test_prepare_code_matches_reference_desk(gpu_ctx, ref):
    """prepare_code support n, energy and replica (test_detector.cpp:70-87)."""
    from paper_2005_10445_b200 import capi
    from paper_2005_10445_b200._abi import desk_config
    cfg = desk_config(256)
    W = 2048 + 500
    bits = np.stack([ref.gen_code(s, cfg) for s in (1, 2, 3)])
    cs = capi.CodeSet.prepare(gpu_ctx, cfg, W, bits)
    s = ref.Session()
    for i in range(3):
        k = s.prepare_code(bits[i], cfg, W, "c%d" % i)
        want = s.code_info(k)
        got = cs.info(i)
        assert got["nonzero_len"] == want["nonzero_len"], (i, got, want)
        # north-star tolerance (1e-4 rel): sum d^2 includes the causal-start
        # samples whose d is 0/0-conditioned in both implementations
        assert abs(got["energy"] - want["energy"]) <= 1e-4 * want["energy"], (i, got, want)
        rg, rw = cs.replica(i), s.code_replica(k)
        # replica d = u / (|f1| + |f0|): compare where the denominator is
        # well conditioned (the causal filter start is 0/0-like dust)
        rep = ref.synth_replica(bits[i], cfg, W)
        d_ref, u_ref = ref.demodulate_signal(rep, 0, 0.0, cfg)
        n = want["nonzero_len"]
        assert np.array_equal(rw, d_ref[:n])
        assert_d_conditioned(rg, rw, u_ref[:n])


def test_end_to_end_desk_fractional_delay(gpu_ctx, ref):
    """test_detector.cpp:253-292 on the GPU, and parity with the reference."""
    from paper_2005_10445_b200 import capi
    from paper_2005_10445_b200._abi import desk_config
    cfg = desk_config(1024)
    P = 1024 * 8
    W = P + 1000
    bits = np.stack([ref.gen_code(s, cfg) for s in (100, 101, 102)])
    iq = ref.channel_window(bits[0], cfg, 12.25, W, 55)
    cs = capi.CodeSet.prepare(gpu_ctx, cfg, W, bits)
    win = capi.Windows(gpu_ctx, W)
    win.demodulate(cfg, [0.0], iq, 0, W, 1)
    dets = capi.detect(gpu_ctx, win, cs, 0.25, cfg.mod.sample_rate)
    assert dets[0]["accepted"] and dets[0]["score"] > 0.9
    assert abs(dets[0]["toa_seconds"] * cfg.mod.sample_rate - 12.25) <= 0.05
    assert not dets[1]["accepted"] and not dets[2]["accepted"]
    s = ref.Session()
    idx = [s.prepare_code(bits[i], cfg, W, "c%d" % i) for i in range(3)]
    d, u = ref.demodulate_window(iq, 0, cfg)
    want = s.detect(d, u, idx, 0.25, 0, cfg.mod.sample_rate)
    # the injected code: full parity end to end
    bad = compare_detections(dets[:1], want[:1], cfg.mod.sample_rate)
    assert not bad, bad
    # absent codes in this noise-free window correlate against the 0/0 dust
    # of d in the exactly-zero stretches, which is FFT-rounding dependent;
    # with the same d,u the whole detect() back half must agree.
    win.set_du(0, d, u, 0)
    dets2 = capi.detect(gpu_ctx, win, cs, 0.25, cfg.mod.sample_rate)
    bad = compare_detections(dets2, want, cfg.mod.sample_rate, xc_ref=s.batch_xcorr(d, idx))
    assert not bad, bad


def test_end_to_end_desk_noisy_all_codes(gpu_ctx, ref):
    """Same scene at 10 dB SNR: every code's Detection end to end."""
    from paper_2005_10445_b200 import capi
    from paper_2005_10445_b200._abi import desk_config
    cfg = desk_config(1024)
    W = 1024 * 8 + 1000
    bits = np.stack([ref.gen_code(s, cfg) for s in (100, 101, 102, 103, 104)])
    iq = ref.channel_window(bits[0], cfg, 12.25, W, 55, snr_db=10.0)
    cs = capi.CodeSet.prepare(gpu_ctx, cfg, W, bits)
    win = capi.Windows(gpu_ctx, W)
    win.demodulate(cfg, [0.0], iq, 0, W, 1)
    dets = capi.detect(gpu_ctx, win, cs, 0.25, cfg.mod.sample_rate)
    s = ref.Session()
    idx = [s.prepare_code(bits[i], cfg, W, "c%d" % i) for i in range(len(bits))]
    d, u = ref.demodulate_window(iq, 0, cfg)
    want = s.detect(d, u, idx, 0.25, 0, cfg.mod.sample_rate)
    xc = s.batch_xcorr(d, idx)

    def tie_ok(g, w):
        c = int(w["code_index"])
        return near_tie_margin(xc[c], int(w["peak_index"]), int(g["peak_index"])) < 1e-5

    bad = compare_detections(dets, want, cfg.mod.sample_rate, tie_ok=tie_ok, xc_ref=xc, eps=1e-5,
                             pc_ref=(u, {i: s.code_replica(idx[i]) for i in range(len(bits))}))
    assert not bad, bad


def test_detect_statistics_alignment_paths(gpu_ctx, ref):
    """detect() back half (statistics, parabola, score) on odd window lengths
    and several slots, so the statistics kernel sees every 16-byte phase of
    d[j-1] and u[j] (vector path), misaligned slots (scalar path), peaks near
    the window end (partial, edge lags) and peak index 0."""
    from paper_2005_10445_b200 import capi
    rng = np.random.default_rng(77)
    for W in (4099, 4096 + 1024):
        dcs = [ref.gaussian(9100 + i, n) for i, n in enumerate((100, 257, 1000, 1501, 2100))]
        cs = _cs_from(capi, gpu_ctx, dcs, W, ref)
        s = ref.Session()
        N = ref.pad_length(W + max(x.size for x in dcs))
        idx = [s.make_transformed(x, x, W, N) for x in dcs]
        n_slots = 4
        win = capi.Windows(gpu_ctx, W, n_slots)
        want, xcs, us = [], [], []
        for slot in range(n_slots):
            d = (0.05 * rng.standard_normal(W)).astype(np.float32)
            # code k at offset placed per slot: start of window, interior, and
            # across the end (partial statistics)
            for k, dc in enumerate(dcs):
                off = [0, 1 + 37 * slot + k, 1777 + 3 * slot + k, W - 60 - k][(slot + k) % 4]
                m = min(dc.size, W - off)
                d[off:off + m] += dc[:m]
            u = (0.5 * d + 0.01 * rng.standard_normal(W)).astype(np.float32)
            win.set_du(slot, d, u, 1000 * slot)
            want.extend(s.detect(d, u, idx, 0.25, 1000 * slot, 8.0e6))
            xcs.append(s.batch_xcorr(d, idx))
            us.append(u)
        got = capi.detect(gpu_ctx, win, cs, 0.25, 8.0e6)
        nc = len(dcs)
        for slot in range(n_slots):
            g = got[slot * nc:(slot + 1) * nc]
            w = want[slot * nc:(slot + 1) * nc]
            xc = xcs[slot]

            def tie_ok(a, b):
                c = int(b["code_index"])
                return near_tie_margin(xc[c], int(b["peak_index"]), int(a["peak_index"])) < 1e-5

            bad = compare_detections(g, w, 8.0e6, tie_ok=tie_ok, xc_ref=xc,
                                     pc_ref=(us[slot], {i: dcs[i] for i in range(nc)}))
            assert not bad, (W, slot, bad)


@pytest.mark.slow
def test_search_shape_parity(gpu_ctx, ref):
    """Default 8 Ms/s search shape (W = 800,000, N = 870,912): one injected
    code in noise plus absent codes, every Detection field vs the reference."""
    from paper_2005_10445_b200 import capi
    from paper_2005_10445_b200._abi import demod_config
    cfg = demod_config()
    W = 800000
    bits = np.stack([ref.gen_code(1000 + i, cfg) for i in range(5)])
    iq = ref.channel_window(bits[0], cfg, 1000.25, W, 1, snr_db=0.0)
    cs = capi.CodeSet.prepare(gpu_ctx, cfg, W, bits)
    # any N >= W + n - 1 gives the reference's lags; the B200 path picks the
    # cheapest supported split (1024 x 864 = 884,736 vs the reference's 870,912)
    assert cs.info(0)["corr_len"] >= W + cs.info(0)["nonzero_len"] - 1
    win = capi.Windows(gpu_ctx, W)
    win.demodulate(cfg, [0.0], iq, 0, W, 1)
    dets = capi.detect(gpu_ctx, win, cs, 0.25, cfg.mod.sample_rate)
    s = ref.Session()
    idx = [s.prepare_code(bits[i], cfg, W, "c%d" % i) for i in range(len(bits))]
    for i in range(len(bits)):
        assert cs.info(i)["nonzero_len"] == s.code_info(idx[i])["nonzero_len"]
    d, u = ref.demodulate_window(iq, 0, cfg)
    want = s.detect(d, u, idx, 0.25, 0, cfg.mod.sample_rate)
    assert want[0]["accepted"] and abs(want[0]["peak_index"] - 1000) <= 1
    xc = s.batch_xcorr(d, idx)

    def tie_ok(g, w):
        c = int(w["code_index"])
        return near_tie_margin(xc[c], int(w["peak_index"]), int(g["peak_index"])) < 1e-5

    bad = compare_detections(dets, want, cfg.mod.sample_rate, tie_ok=tie_ok, xc_ref=xc, eps=1e-5,
                             pc_ref=(u, {i: s.code_replica(idx[i]) for i in range(len(bits))}))
    assert not bad, bad


def test_detect_on_golden_fixture(gpu_ctx):
    """GPU detect() on the committed fixture's d,u against the reference's
    Detections stored in tests/golden/desk_e2e.npz (no oracle needed)."""
    import os

    from paper_2005_10445_b200 import capi
    from paper_2005_10445_b200._abi import DETECTION_DTYPE, desk_config
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "desk_e2e.npz"))
    cfg = desk_config(1024)
    W = z["d"].size
    cs = capi.CodeSet.prepare(gpu_ctx, cfg, W, z["bits"])
    for i in range(len(z["bits"])):
        assert cs.info(i)["nonzero_len"] == int(z["nonzero"][i])
    win = capi.Windows(gpu_ctx, W)
    win.set_du(0, z["d"], z["u"], 0)
    got = capi.detect(gpu_ctx, win, cs, 0.25, cfg.mod.sample_rate)
    want = z["det"].view(DETECTION_DTYPE)
    bad = compare_detections(got, want, cfg.mod.sample_rate, xc_ref=z["xc"], eps=1e-5)
    assert not bad, bad
    # end to end from the fixture's int16 window
    win.demodulate(cfg, [0.0], z["iq"], 0, W, 1)
    d, u = win.get_du(0)
    assert_d_conditioned(d, z["d"], z["u"])
    got2 = capi.detect(gpu_ctx, win, cs, 0.25, cfg.mod.sample_rate)
    bad = compare_detections(got2, want, cfg.mod.sample_rate, xc_ref=z["xc"], eps=1e-5)
    assert not bad, bad


def test_lo_demod_on_golden_fixture(gpu_ctx):
    import os

    from paper_2005_10445_b200 import capi
    from paper_2005_10445_b200._abi import demod_config
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "lo_demod.npz"))
    W = z["d"].size
    win = capi.Windows(gpu_ctx, W, 1, 1)
    win.demodulate(demod_config(), [float(z["lo"])], z["iq"], int(z["start"]), W, 1)
    d, u = win.get_du(0)
    assert np.abs(u - z["u"]).max() <= 1e-4 * np.abs(z["u"]).max()
    assert_d_conditioned(d, z["d"], z["u"])


def test_invalid_arguments_raise(gpu_ctx):
    """Reference preconditions surface as InvalidArgument (std::invalid_argument)."""
    from paper_2005_10445_b200 import capi
    from paper_2005_10445_b200._abi import desk_config
    cfg = desk_config(256)
    bits = np.zeros((1, 256), np.uint8)
    with pytest.raises(capi.InvalidArgument):
        capi.CodeSet.prepare(gpu_ctx, cfg, 1000, bits)            # window shorter than a packet
    dc = np.ones(64, np.float32)
    with pytest.raises(capi.InvalidArgument):
        capi.CodeSet.from_replicas(gpu_ctx, 512, 500, [dc])       # transform too short
    cs = capi.CodeSet.from_replicas(gpu_ctx, 512, 1024, [dc])
    w = capi.Windows(gpu_ctx, 600)
    with pytest.raises(capi.InvalidArgument):
        capi.detect(gpu_ctx, w, cs)                               # mixed window shapes
    with pytest.raises(capi.InvalidArgument):
        capi.demodulate_window(gpu_ctx, np.zeros(3, np.int16), 0, cfg)   # odd raw count
    # beyond one transform (1024 x 1024) the window is correlated in segments
    # (tests below); a support longer than half the largest transform is
    # rejected with a clear error, before any launch
    assert capi.corr_len(1 << 20, 2) == 0
    with pytest.raises(capi.GpuError, match="half of the largest transform"):
        capi.CodeSet.from_replicas(gpu_ctx, 1 << 21, (1 << 21) + 600000, [np.ones(600000, np.float32)])


def test_tracking_batch_parity(gpu_ctx, ref):
    """Tracking mode (BASELINE configs[3]; proj/src/recording.cpp:360-378 per
    scheduler Task): a batch of 12 ms windows [toa - 2 ms, toa + 10 ms) at the
    default 8 Ms/s, one code each, through tdg_track against the reference's
    demodulate_window + prepare_code(track_shape) + detect per task.  Covers
    injected codes (accepted), absent codes, odd/even code slots of a stored
    pair and overlapping windows."""
    from paper_2005_10445_b200 import capi
    from paper_2005_10445_b200._abi import demod_config
    cfg = demod_config()
    fs = cfg.mod.sample_rate
    W = 96000                     # (track_pre_s + track_post_s) * fs, scheduler.hpp:68-69
    pre = 16000
    seeds = [2000 + i for i in range(5)]
    bits = np.stack([ref.gen_code(s, cfg) for s in seeds])
    inj = [(0, 0.0103, 1.0, 0.0), (3, 0.0412, 0.8, 0.0), (1, 0.0707, 1.0, 0.0)]
    iq = ref.generate_recording(cfg, seeds, 0.1, 10.0, 77, inj)
    n = iq.size // 2
    toas = [int(round(t * fs)) for _, t, _, _ in inj]
    starts = [toas[0] - pre, toas[1] - pre, toas[2] - pre, toas[0] - pre, toas[1] - pre + 5000, 30000,
              toas[2] - 40000]
    codes = [0, 3, 1, 2, 3, 4, 1]  # tasks 3, 5: absent codes; task 4: shifted window; task 6: packet cut
                                   # by the window end (partial: detector.cpp:151-153,197)
    assert all(0 <= s0 and s0 + W <= n for s0 in starts)
    cs = capi.CodeSet.prepare(gpu_ctx, cfg, W, bits)
    dets = capi.track(gpu_ctx, cfg, iq, starts, codes, cs, 0.25)
    s = ref.Session()
    idx = [s.prepare_code(bits[i], cfg, W, "c%d" % i) for i in range(len(bits))]
    for i, (s0, c) in enumerate(zip(starts, codes)):
        d, u = ref.demodulate_window(iq[2 * s0:2 * (s0 + W)], s0, cfg)
        want = s.detect(d, u, [idx[c]], 0.25, s0, fs)
        xc = s.batch_xcorr(d, [idx[c]])
        want["code_index"] = c

        def tie_ok(g, w, xc=xc):
            return near_tie_margin(xc[0], int(w["peak_index"]), int(g["peak_index"])) < 1e-5

        bad = compare_detections(dets[i:i + 1], want, fs, tie_ok=tie_ok, xc_ref={c: xc[0]}, eps=1e-5,
                                 pc_ref=(u, {c: s.code_replica(idx[c])}))
        assert not bad, (i, bad)
        assert int(dets[i]["window_start"]) == s0 and int(dets[i]["code_index"]) == c
    assert dets[0]["accepted"] and dets[1]["accepted"] and dets[2]["accepted"]
    assert not dets[3]["accepted"] and not dets[5]["accepted"]
    assert dets[6]["partial"] and not dets[6]["accepted"]


def test_tracking_graph_replay_bitwise(ref):
    """Small tracking batches are replayed as CUDA graphs from the third call
    with the same shape (warm, capture, replay): every record must be bitwise
    equal to the stream path's, across changing tasks, interleaved batch
    sizes, a rejected batch and a code set rebuilt in between."""
    from paper_2005_10445_b200 import capi
    from paper_2005_10445_b200._abi import demod_config
    cfg = demod_config()
    fs = cfg.mod.sample_rate
    W = 96000
    seeds = [2100 + i for i in range(4)]
    bits = np.stack([ref.gen_code(s, cfg) for s in seeds])
    inj = [(0, 0.0103, 1.0, 0.0), (2, 0.0412, 0.8, 0.0), (3, 0.0707, 1.0, 0.0)]
    iq = ref.generate_recording(cfg, seeds, 0.1, 10.0, 78, inj)
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
        want = [capi.track(ctx, cfg, iq, st, co, cs, 0.25) for st, co in batches]
        ctx.set_option("track_graphs", 1)
        for rep in range(3):
            for (st, co), w in zip(batches, want):
                got = capi.track(ctx, cfg, iq, st, co, cs, 0.25)
                assert got.tobytes() == w.tobytes(), (rep, st, co)
            if rep == 0:
                with pytest.raises(capi.InvalidArgument):
                    capi.track(ctx, cfg, iq, [10], [len(bits)], cs, 0.25)
            if rep == 1:
                # a rebuilt code set moves buffers: graphs must not replay stale pointers
                cs.close()
                cs = capi.CodeSet.prepare(ctx, cfg, W, bits)
        assert want[0]["accepted"].any()


def test_tracking_multiwave_matches_single_tasks(ref):
    """A batch of 20 tracking tasks (three correlation waves over the four
    stream pairs) against the same tasks one at a time (single-wave path,
    CUDA-graph replays from the third): peak indices and flags exact, the
    statistics equal up to the summation order of the split dot products."""
    from paper_2005_10445_b200 import capi
    from paper_2005_10445_b200._abi import demod_config
    cfg = demod_config()
    fs = cfg.mod.sample_rate
    W = 96000
    seeds = [2200 + i for i in range(6)]
    bits = np.stack([ref.gen_code(s, cfg) for s in seeds])
    inj = [(0, 0.0103, 1.0, 0.0), (2, 0.0412, 0.8, 0.0), (5, 0.0707, 1.0, 0.0)]
    iq = ref.generate_recording(cfg, seeds, 0.1, 10.0, 79, inj)
    toas = [int(round(t * fs)) for _, t, _, _ in inj]
    rng = np.random.default_rng(11)
    starts = [int(toas[i % 3] - 16000 + rng.integers(-4000, 4000)) for i in range(20)]
    codes = [int(i % 6) for i in range(20)]
    with capi.Context(0) as ctx:
        cs = capi.CodeSet.prepare(ctx, cfg, W, bits)
        batch = capi.track(ctx, cfg, iq, starts, codes, cs, 0.25)
        singles = np.concatenate([capi.track(ctx, cfg, iq, [s0], [c], cs, 0.25) for s0, c in zip(starts, codes)])
    for f in ("code_index", "window_start", "peak_index", "accepted", "partial"):
        assert np.array_equal(batch[f], singles[f]), f
    for f in ("subsample_offset", "w_c", "q", "p_c", "score", "peak_value"):
        g, w = batch[f].astype(np.float64), singles[f].astype(np.float64)
        assert np.all(np.abs(g - w) <= 1e-5 * np.maximum(np.abs(w), 1e-3)), (f, float(np.max(np.abs(g - w))))
    assert batch["accepted"].sum() >= 3


def test_tracking_rejects_bad_tasks(gpu_ctx):
    from paper_2005_10445_b200 import capi
    from paper_2005_10445_b200._abi import desk_config
    cfg = desk_config(1024)
    W = 1024 * 8 + 500
    bits = np.random.default_rng(0).integers(0, 2, (2, 1024), dtype=np.uint8)
    cs = capi.CodeSet.prepare(gpu_ctx, cfg, W, bits)
    iq = np.zeros(2 * (W + 100), np.int16)
    with pytest.raises(capi.InvalidArgument):
        capi.track(gpu_ctx, cfg, iq, [200], [0], cs)          # window past the block
    with pytest.raises(capi.InvalidArgument):
        capi.track(gpu_ctx, cfg, iq, [0], [2], cs)            # code index out of range
    assert capi.track(gpu_ctx, cfg, iq, [], [], cs).size == 0


def _scene_two_codes(ref, cfg, bits, W, delays, seed):
    a = ref.channel_window(bits[0], cfg, delays[0], W, seed, snr_db=5.0).astype(np.int32)
    b = ref.channel_window(bits[1], cfg, delays[1], W, seed + 1, snr_db=5.0).astype(np.int32)
    return np.clip(a + b, -32767, 32767).astype(np.int16)


@pytest.mark.parametrize("W", [300000, 1200000])
def test_window_lengths_beyond_the_menu(gpu_ctx, ref, W):
    """Any W the reference's pad_length accepts (proj/src/fft.cpp:93-101,
    detector.hpp:19-21): W = 300,000 lies between the instantiated splits
    (padded up to the next one), W = 1,200,000 (150 ms at 8 Ms/s) needs
    W + n - 1 > 1024 x 1024 and runs as a segmented correlation -- segments of
    B = 2^20 - n + 1 lags, each from B + n - 1 samples, argmax keys merged over
    the global lag.  Code 1 sits across the segment boundary (its peak lag
    within a few samples of B), code 0 early; every Detection field is checked
    against the reference compiled in place, and batch_xcorr's full rows too."""
    from paper_2005_10445_b200 import capi
    from paper_2005_10445_b200._abi import demod_config
    cfg = demod_config()
    bits = np.stack([ref.gen_code(2000 + i, cfg) for i in range(4)])
    cs = capi.CodeSet.prepare(gpu_ctx, cfg, W, bits)
    n = max(cs.info(i)["nonzero_len"] for i in range(len(bits)))
    B = (1 << 20) - n + 1
    seg = W + n - 1 > (1 << 20)
    delays = (1000.25, (B - 3.5) if seg else W // 2 + 0.5)
    iq = _scene_two_codes(ref, cfg, bits, W, delays, 41)
    win = capi.Windows(gpu_ctx, W)
    win.demodulate(cfg, [0.0], iq, 0, W, 1)
    dets = capi.detect(gpu_ctx, win, cs, 0.25, cfg.mod.sample_rate)
    s = ref.Session()
    idx = [s.prepare_code(bits[i], cfg, W, "c%d" % i) for i in range(len(bits))]
    d, u = ref.demodulate_window(iq, 0, cfg)
    want = s.detect(d, u, idx, 0.25, 0, cfg.mod.sample_rate)
    assert want[0]["accepted"] and want[1]["accepted"]
    assert abs(int(want[1]["peak_index"]) - int(delays[1])) <= 2
    xc = s.batch_xcorr(d, idx)

    def tie_ok(g, w):
        c = int(w["code_index"])
        return near_tie_margin(xc[c], int(w["peak_index"]), int(g["peak_index"])) < 1e-5

    bad = compare_detections(dets, want, cfg.mod.sample_rate, tie_ok=tie_ok, xc_ref=xc, eps=1e-5,
                             pc_ref=(u, {i: s.code_replica(idx[i]) for i in range(len(bits))}))
    assert not bad, bad
    # full correlation rows, segment by segment, against the reference's
    win.set_du(0, d, u)
    got = capi.batch_xcorr(gpu_ctx, win, 0, cs)
    for i in range(len(bits)):
        e = cs.info(i)["energy"]
        assert np.abs(got[i] - xc[i]).max() <= 2e-5 * e, i


def test_cta_trace_diagnostics(gpu_ctx, ref):
    """Option cta_trace + tdg_cta_trace: every correlation-pass CTA of a
    detect records its SM and start/exit times (tools/cta_trace.py)."""
    import ctypes

    from paper_2005_10445_b200 import capi
    W = 2048
    dcs = [ref.gaussian(8100 + i, 100) for i in range(6)]
    d = ref.gaussian(8199, W)
    cs = _cs_from(capi, gpu_ctx, dcs, W, ref)
    w = capi.Windows(gpu_ctx, W)
    w.set_du(0, d, d)
    gpu_ctx.set_option("cta_trace", 4096)
    try:
        capi.detect(gpu_ctx, w, cs)
        buf = np.zeros(3 * 4096, dtype=np.uint64)
        n = ctypes.c_uint64()
        capi._check(capi.lib().tdg_cta_trace(gpu_ctx.handle, capi._ptr(buf), 4096, ctypes.byref(n)))
        rec = buf[:3 * n.value].reshape(-1, 3)
        assert n.value > 0
        assert set((rec[:, 0] & 255).tolist()) == {0, 1}          # both passes
        assert (rec[:, 2] >= rec[:, 1]).all() and (rec[:, 1] > 0).all()
        capi._check(capi.lib().tdg_cta_trace(gpu_ctx.handle, capi._ptr(buf), 4096, ctypes.byref(n)))
        assert n.value == 0                                         # read resets the count
    finally:
        gpu_ctx.set_option("cta_trace", 0)
