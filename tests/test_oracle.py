"""CPU: the oracle restatement (oracle/tagdsp_oracle.c) pinned against the
reference's own known answers, the committed golden fixtures (generated from
the reference compiled in place, tests/golden/make_golden.py) and, when
present, the compiled reference itself (bitwise)."""
import json
import os

import numpy as np
import pytest

import oraclepy as O
from parity import direct_xcorr
from paper_2005_10445_b200._abi import DETECTION_DTYPE, demod_config, desk_config

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(G, "golden.json")) as f:
        return json.load(f)


def test_reference_known_answers(golden):
    """test_codegen.cpp:39-51, test_dsp.cpp:132-137, test_detector.cpp:153-181."""
    assert O.gen_code(7, 16).tolist() == golden["gen_code_seed7_16bits"]
    assert int((O.gen_code(42) != O.gen_code(43)).sum()) == golden["hamming_seed42_43"] == 4079
    for n, m in golden["pad_length"].items():
        assert O.pad_length(int(n)) == m
    assert O.pad_length(865743) == 870912 and O.pad_length(161743) == 162000
    for xs, (j, v) in golden["find_peak"]:
        assert O.find_peak(np.array(xs, np.float32)) == (j, v)
    for xs, j, d in golden["interpolate_peak"]:
        assert O.interpolate_peak(np.array(xs, np.float32), j) == d
    np.testing.assert_array_equal(O.gaussian(5, 8), np.array(golden["gaussian_seed5_first8"], np.float32))


def test_restatement_matches_fixture_bitwise():
    z = np.load(os.path.join(G, "desk_e2e.npz"))
    cfg = desk_config(1024)
    W = z["d"].size
    d, u = O.demodulate_window(z["iq"], 0, cfg)
    np.testing.assert_array_equal(d, z["d"])
    np.testing.assert_array_equal(u, z["u"])
    codes = [O.prepare_code(b, cfg, W) for b in z["bits"]]
    for i, c in enumerate(codes):
        assert c.nonzero_len == int(z["nonzero"][i])
        assert c.energy == z["energy"][i]
        np.testing.assert_array_equal(c.replica_d, z["rep%d" % i])
    np.testing.assert_array_equal(O.batch_xcorr(d, codes), z["xc"])
    det = O.detect(d, u, codes, 0.25, 0, cfg.mod.sample_rate)
    assert det.tobytes() == z["det"].view(DETECTION_DTYPE).tobytes()
    assert det[0]["accepted"] and abs(det[0]["toa_seconds"] * 1e6 - 12.25) <= 0.05


def test_restatement_lo_demod_fixture():
    z = np.load(os.path.join(G, "lo_demod.npz"))
    d, u = O.demodulate_window(z["iq"], int(z["start"]), demod_config(lo_freq=float(z["lo"])))
    np.testing.assert_array_equal(d, z["d"])
    np.testing.assert_array_equal(u, z["u"])


def test_xcorr_brute_force():
    """test_detector.cpp:110-122 and acceptance.cpp:119-135 on the oracle."""
    worst = 0.0
    rng = np.random.default_rng(4242)
    for trial in range(30):
        dn, cn = 64 + int(rng.integers(193)), 8 + int(rng.integers(25))
        g = O.gaussian(7000 + trial, cn + dn)
        dc, d = g[:cn], g[cn:]
        c = O.make_transformed(dc, dc, dn, O.pad_length(dn + cn))
        got = O.batch_xcorr(d, [c])[0]
        worst = max(worst, float(np.abs(got - direct_xcorr(d, dc)).max() / c.energy))
    assert worst <= 1e-4


def test_make_transformed_precondition():
    dc = O.gaussian(1, 64)
    with pytest.raises(ValueError):
        O.make_transformed(dc, dc, 512, 500)


def test_restatement_matches_compiled_reference(ref):
    """Bitwise against oracle/_ref on a fresh 8 Ms/s case (packet 512 bits)."""
    cfg = demod_config(packet_bits=512)
    W = 512 * 8 + 3000
    bits = [O.gen_code(s, 512) for s in (5, 6)]
    iq = ref.channel_window(bits[1], cfg, 333.4, W, 9, snr_db=3.0, freq_offset=20e3)
    d, u = O.demodulate_window(iq, 100, cfg)
    d2, u2 = ref.demodulate_window(iq, 100, cfg)
    np.testing.assert_array_equal(d, d2)
    np.testing.assert_array_equal(u, u2)
    codes = [O.prepare_code(b, cfg, W) for b in bits]
    s = ref.Session()
    idx = [s.prepare_code(b, cfg, W, "c%d" % i) for i, b in enumerate(bits)]
    a = O.detect(d, u, codes, 0.25, 100, cfg.mod.sample_rate)
    b = s.detect(d2, u2, idx, 0.25, 100, cfg.mod.sample_rate)
    assert a.tobytes() == b.tobytes()
    assert b[1]["accepted"]
