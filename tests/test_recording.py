"""Recording format (proj/src/recording.cpp:17-64) and the offline searching
pass over a recording (:258-289) on the B200 path.  CPU tests: file format
round trip and its error cases, the bench/synthetic code generator against the
compiled reference.  GPU tests: detect_recording against the reference's
per-window demodulate_window + detect, and byte-identical output on a rerun
(acceptance.cpp:412-437, criterion 9)."""
import numpy as np
import pytest

from parity import compare_detections


def test_recording_round_trip_and_errors(tmp_path):
    from paper_2005_10445_b200 import recording
    rng = np.random.default_rng(1)
    iq = rng.integers(-32768, 32767, 2 * 1000, dtype=np.int16)
    p = str(tmp_path / "rec.iq")
    recording.write_recording(p, iq, 1.0e6, start_time=4242, center_freq=150.1e6, creator="test")
    got, rate, start, cf, creator = recording.read_recording(p)
    assert np.array_equal(got, iq) and rate == 1.0e6 and start == 4242 and cf == 150.1e6 and creator == "test"
    with open(p, "ab") as f:                      # payload not whole I/Q pairs
        f.write(b"\x00\x00")
    with pytest.raises(RuntimeError, match="malformed"):
        recording.read_recording(p)
    q = str(tmp_path / "nosidecar.iq")
    iq.tofile(q)
    with pytest.raises(RuntimeError, match="missing sidecar"):
        recording.read_recording(q)
    recording.write_recording(q, iq, -1.0)
    with pytest.raises(RuntimeError, match="invalid sample_rate"):
        recording.read_recording(q)


def test_detection_json_line_format():
    from paper_2005_10445_b200 import recording
    from paper_2005_10445_b200._abi import DETECTION_DTYPE
    r = np.zeros(1, DETECTION_DTYPE)[0]
    r["toa_seconds"], r["peak_index"], r["subsample_offset"] = 0.125, 1000, np.float32(0.25)
    r["w_c"], r["q"], r["p_c"], r["score"], r["accepted"] = 3.5, 4.0, 1.0, np.float32(0.5), 1
    line = recording.detection_json_line(r, "t7")
    # nlohmann::json::dump(): keys sorted, no spaces
    assert line == ('{"accepted":true,"p_c":1.0,"partial":false,"peak_index":1000,"q":4.0,"score":0.5,'
                    '"subsample_offset":0.25,"tag_id":"t7","toa_seconds":0.125,"w_c":3.5}')


def test_recording_files_match_reference(ref, tmp_path):
    """write_recording / read_recording (proj/src/recording.cpp:23-64): files
    written by recording.py and by the compiled reference are byte-identical
    (payload and sidecar) and each side reads the other's."""
    from paper_2005_10445_b200 import recording
    rng = np.random.default_rng(8)
    for k, (n, rate, start, cf, creator) in enumerate([(1000, 8.0e6, 0, 0.0, ""), (3, 1.0e6, 4242, 150.1e6, "test"),
                                                       (7777, 2.5e5, -17, 1.5e8, "tagdsp generate")]):
        iq = rng.integers(-32768, 32767, 2 * n, dtype=np.int16)
        a, b = str(tmp_path / ("ours%d.iq" % k)), str(tmp_path / ("ref%d.iq" % k))
        recording.write_recording(a, iq, rate, start_time=start, center_freq=cf, creator=creator)
        ref.write_recording(b, iq, rate, start_time=start, center_freq=cf, creator=creator)
        assert open(a, "rb").read() == open(b, "rb").read()
        assert open(recording.sidecar_path(a)).read() == open(recording.sidecar_path(b)).read()
        got = recording.read_recording(b)
        assert np.array_equal(got[0], iq) and got[1:] == (rate, start, cf, creator)
        got = ref.read_recording(a, n)
        assert np.array_equal(got[0], iq) and got[1:] == (rate, start, cf, creator)
    bad = str(tmp_path / "bad.iq")
    recording.write_recording(bad, np.zeros(4, np.int16), 1.0e6)
    with open(bad, "ab") as f:
        f.write(b"\x00\x00")
    with pytest.raises(Exception):
        ref.read_recording(bad, 10)
    with pytest.raises(RuntimeError):
        recording.read_recording(bad)


def test_detection_json_line_matches_reference(ref):
    """detection_json_line (proj/src/recording.cpp:228-242): byte-identical to
    the compiled reference's nlohmann dump on random records."""
    from paper_2005_10445_b200 import recording
    from paper_2005_10445_b200._abi import DETECTION_DTYPE
    rng = np.random.default_rng(4)
    recs = np.zeros(300, DETECTION_DTYPE)
    recs["toa_seconds"] = rng.uniform(-1, 1e3, recs.size) * rng.choice([1, 1e-9, 1e9], recs.size)
    recs["peak_index"] = rng.integers(0, 1 << 40, recs.size)
    for f in ("subsample_offset", "w_c", "q", "p_c", "score"):
        recs[f] = (rng.standard_normal(recs.size) * rng.choice([1e-30, 1e-3, 1, 1e6, 1e30], recs.size))
    recs["subsample_offset"][:5] = [0.0, -0.0, 0.5, -0.5, 0.25]
    recs["accepted"] = rng.integers(0, 2, recs.size)
    recs["partial"] = rng.integers(0, 2, recs.size)
    for i, r in enumerate(recs):
        tag = "t%d" % i if i % 3 else "tag \"%d\" \u00e9" % i
        assert recording.detection_json_line(r, tag) == ref.detection_json_line(r, tag), i


def test_synth_gen_code_matches_reference(ref):
    from paper_2005_10445_b200 import synth
    from paper_2005_10445_b200._abi import demod_config
    cfg = demod_config()
    for seed in (0, 7, 1000, 123456789):
        assert np.array_equal(synth.gen_code(seed, 8192), ref.gen_code(seed, cfg))


@pytest.mark.gpu
def test_detect_recording_matches_reference_and_is_deterministic(gpu_ctx, ref, tmp_path):
    from paper_2005_10445_b200 import recording
    from paper_2005_10445_b200._abi import desk_config
    cfg = desk_config(1024)
    fs = cfg.mod.sample_rate
    seeds = [501, 502, 503]
    tags = [("a", seeds[0]), ("b", seeds[1]), ("c", seeds[2])]
    inj = [(0, 0.0031, 1.0, 0.0), (2, 0.0242, 0.8, 0.0), (1, 0.0405, 1.0, 0.0)]
    iq = ref.generate_recording(cfg, seeds, 0.06, 10.0, 11, inj)
    p = str(tmp_path / "scene.iq")
    recording.write_recording(p, iq, fs, start_time=1000)
    window_s, overlap_s = 0.02, 0.004
    recs, ids = recording.detect_recording(gpu_ctx, p, tags, window_s, overlap_s, cfg=cfg)
    W = int(window_s * fs + 0.5)
    adv = int((window_s - overlap_s) * fs + 0.5)
    n = iq.size // 2
    s = ref.Session()
    idx = [s.prepare_code(ref.gen_code(sd, cfg), cfg, W, t) for t, sd in tags]
    starts = list(range(0, n - W + 1, adv))
    assert len(recs) == len(starts) * len(tags)
    for k, st in enumerate(starts):
        d, u = ref.demodulate_window(iq[2 * st:2 * (st + W)], 1000 + st, cfg)
        want = s.detect(d, u, idx, 0.25, 1000 + st, fs)
        xc = s.batch_xcorr(d, idx)
        reps = {c: s.code_replica(idx[c]) for c in range(len(tags))}
        bad = compare_detections(recs[k * 3:(k + 1) * 3], want, fs, xc_ref=xc, eps=1e-5, pc_ref=(u, reps))
        assert not bad, (k, bad)
    assert sum(int(r["accepted"]) for r in recs) >= 3
    text1 = recording.detections_jsonl(recs, ids, all_candidates=True)
    recs2, _ = recording.detect_recording(gpu_ctx, p, tags, window_s, overlap_s, cfg=cfg)
    assert recording.detections_jsonl(recs2, ids, all_candidates=True) == text1
