"""The drop-in boundary on the B200: the reference's own code
compiled UNMODIFIED against include/tagdsp_b200 + libtagdsp_b200.so
(integration/Makefile, built by __graft_entry__.build() where the reference
tree exists; the executables travel to the GPU box in build/dropin/).

* The reference's own test suites -- test_dsp, test_detector, test_codegen,
  test_scheduler, test_harness, test_formats (doctest) and acceptance.cpp's
  nine criteria -- running their detector / dsp / fft calls on the GPU.
* detect_recording (proj/src/recording.cpp:258-289, compiled from the
  reference) over the drop-in vs the reference CPU build on the same file:
  every Detection under the parity contract.
* simulate_recording (recording.cpp:291-389, the scheduler-driven searching +
  tracking loop) over the drop-in, and the batched variant (tracking tasks
  drained into one tdg_track_ring call, device CircularBuffer): event logs
  byte-identical to the reference CPU run.
* run_bench (harness.cpp:28-104) with its correctness gate on the GPU path."""
import json
import os
import subprocess

import numpy as np
import pytest

from paritycheck import ParityReport, RefSlots

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "dropin")
SUITES = ["test_dsp", "test_detector", "test_codegen", "test_scheduler", "test_harness", "test_formats", "acceptance"]


def _need(name):
    p = os.path.join(BIN, name)
    if not os.path.exists(p):
        pytest.skip("build/dropin/%s not built (make -C integration needs the reference tree)" % name)
    return p


@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_on_b200(suite, tmp_path):
    exe = _need(suite)
    r = subprocess.run([exe], cwd=str(tmp_path), capture_output=True, text=True, timeout=1200)
    tail = (r.stdout + r.stderr)[-3000:]
    out = os.environ.get("TDG_PARITY_OUT")
    if out:
        os.makedirs(out, exist_ok=True)
        with open(os.path.join(out, "dropin_suites.log"), "a") as f:
            f.write("== %s rc=%d\n%s\n" % (suite, r.returncode, tail))
    assert r.returncode == 0, tail


def _scene(ref, tmp_path, duration=3.0, n_tags=5):
    from paper_2005_10445_b200._abi import demod_config
    cfg = demod_config()
    seeds = [7000 + i for i in range(n_tags)]
    inj = [(0, 0.300, 1.0, 0.0), (0, 1.300, 1.0, 0.0), (0, 2.300, 1.0, 0.0),
           (2, 0.555, 0.7, 0.0), (2, 1.555, 0.7, 0.0), (2, 2.555, 0.7, 0.0),
           (4, 1.800, 1.0, 0.0)]
    iq = ref.generate_recording(cfg, seeds, duration, 10.0, 21, [x for x in inj if x[1] + 0.01 < duration])
    rec = str(tmp_path / "scene.iq")
    ref.write_recording(rec, iq, cfg.mod.sample_rate, creator="test_gpu_dropin")
    conf = str(tmp_path / "config.json")
    with open(conf, "w") as f:
        json.dump({"tags": [{"id": "t%d" % i, "seed": s, "period_s": 1.0} for i, s in enumerate(seeds)]}, f)
    bits = np.stack([ref.gen_code(s, cfg) for s in seeds])
    return cfg, bits, iq, rec, conf


def _records(path, ids, W, adv, n):
    from paper_2005_10445_b200._abi import DETECTION_DTYPE
    lines = [json.loads(x) for x in open(path)]
    out = np.zeros(len(lines), DETECTION_DTYPE)
    per = len(ids)
    for i, j in enumerate(lines):
        r = out[i]
        r["code_index"] = ids.index(j["tag_id"])
        r["window_start"] = (i // per) * adv
        for f in ("peak_index", "toa_seconds", "subsample_offset", "w_c", "q", "p_c", "score", "accepted",
                  "partial"):
            r[f] = j[f]
        r["peak_value"] = j["w_c"]
    return out


def test_detect_recording_dropin_vs_reference(ref, tmp_path):
    exe = _need("tagdsp_b200_run")
    cfg, bits, iq, rec, conf = _scene(ref, tmp_path, duration=2.0)
    got_p, want_p = str(tmp_path / "gpu.jsonl"), str(tmp_path / "ref.jsonl")
    r = subprocess.run([exe, "detect", rec, conf, got_p], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    ref.run_detect_recording(rec, conf, want_p)
    fs = cfg.mod.sample_rate
    W, adv, n = 800000, 720000, iq.size // 2
    ids = ["t%d" % i for i in range(len(bits))]
    got, want = _records(got_p, ids, W, adv, n), _records(want_p, ids, W, adv, n)
    assert got.size == want.size == ((n - W) // adv + 1) * len(ids)
    rs = RefSlots(ref, cfg, bits, iq, W)
    starts = sorted({int(s) for s in want["window_start"]})
    rs.prefetch(slots=[(s, 0.0) for s in starts], codes=range(len(bits)))
    rep = ParityReport("detect_recording through the drop-in (reference recording.cpp on the B200 path)")
    bad = []
    for s in starts:
        m = want["window_start"] == s
        bad += rs.compare(got[m], want[m], s, 0.0, fs, report=rep)
    assert not bad, bad[:10]
    assert int(want["accepted"].sum()) >= 3
    # lines of accepted detections: identical text up to float rounding -> same tags / peaks
    g_acc = [(j["tag_id"], j["peak_index"]) for j in map(json.loads, open(got_p)) if j["accepted"]]
    w_acc = [(j["tag_id"], j["peak_index"]) for j in map(json.loads, open(want_p)) if j["accepted"]]
    assert g_acc == w_acc


def test_simulate_dropin_and_batched_match_reference(ref, tmp_path):
    exe = _need("tagdsp_b200_run")
    cfg, bits, iq, rec, conf = _scene(ref, tmp_path, duration=3.0)
    ref_ev, seq_ev, bat_ev = (str(tmp_path / x) for x in ("ref.jsonl", "seq.jsonl", "bat.jsonl"))
    det_ref, miss_ref = ref.run_simulate(rec, conf, ref_ev, 0.1)
    r1 = subprocess.run([exe, "simulate", rec, conf, seq_ev, "0.1"], capture_output=True, text=True, timeout=900)
    assert r1.returncode == 0, r1.stderr
    r2 = subprocess.run([exe, "simulate-batched", rec, conf, bat_ev, "0.1"], capture_output=True, text=True,
                        timeout=900)
    assert r2.returncode == 0, r2.stderr
    s1, s2 = json.loads(r1.stdout.strip().splitlines()[-1]), json.loads(r2.stdout.strip().splitlines()[-1])
    ref_text = open(ref_ev).read()
    assert "track_detect" in ref_text and "promoted" in ref_text
    assert open(seq_ev).read() == ref_text
    assert open(bat_ev).read() == ref_text
    assert (s1["detections"], s1["misses"]) == (det_ref, miss_ref)
    assert (s2["detections"], s2["misses"]) == (det_ref, miss_ref)
    out = os.environ.get("TDG_PARITY_OUT")
    if out:
        os.makedirs(out, exist_ok=True)
        with open(os.path.join(out, "dropin_simulate.json"), "w") as f:
            json.dump({"reference": {"detections": det_ref, "misses": miss_ref,
                                     "events": ref_text.count("\n")}, "dropin": s1, "batched": s2}, f)


def test_run_bench_gate_on_b200():
    exe = _need("tagdsp_b200_run")
    r = subprocess.run([exe, "bench", "800000", "1", "2", "1", "8", "64"], capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stderr
    s = json.loads(r.stdout)
    assert s
