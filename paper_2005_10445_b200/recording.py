"""Recording I/O and the offline searching pass over a recording on the B200
path.

Mirrors the reference's file format and caller
(/root/reference/proj/src/recording.cpp):

  write_recording / read_recording   :23-64   little-endian int16 I/Q payload
                                              + "<payload>.meta.json" sidecar
  detection_json_line                :228-242 one JSON object per Detection
  detect_recording                   :258-289 every window of the recording
                                              (window_s, overlap_s) x roster

The search itself is one tdg_search call (all windows x codes); records come
back in the reference's order (window-major, roster order within a window).
"""
import json
import os

import numpy as np

from . import capi
from ._abi import demod_config


def sidecar_path(payload_path):
    """recording.cpp:17-21."""
    return str(payload_path) + ".meta.json"


def write_recording(payload_path, iq, sample_rate, start_time=0, center_freq=0.0, creator=""):
    """recording.cpp:23-39: raw int16 payload, JSON sidecar (indent 2)."""
    iq = np.ascontiguousarray(iq, dtype="<i2")
    with open(payload_path, "wb") as f:
        f.write(iq.tobytes())
    meta = {"sample_rate": float(sample_rate), "start_time": int(start_time), "center_freq": float(center_freq),
            "creator": creator}
    with open(sidecar_path(payload_path), "w") as f:
        f.write(json.dumps(meta, indent=2, sort_keys=True, ensure_ascii=False) + "\n")


def read_recording(payload_path):
    """recording.cpp:41-64 -> (iq int16 [2n], sample_rate, start_time, center_freq, creator).
    Raises like the reference on a payload that is not whole I/Q pairs, a
    missing sidecar or a non-positive sample rate."""
    if not os.path.exists(payload_path):
        raise RuntimeError("cannot read " + str(payload_path))
    nbytes = os.path.getsize(payload_path)
    if nbytes % 4:
        raise RuntimeError("malformed recording (payload not whole I/Q pairs): " + str(payload_path))
    iq = np.fromfile(payload_path, dtype="<i2").astype(np.int16)
    if not os.path.exists(sidecar_path(payload_path)):
        raise RuntimeError("missing sidecar " + sidecar_path(payload_path))
    with open(sidecar_path(payload_path)) as f:
        meta = json.load(f)
    rate = float(meta["sample_rate"])
    if rate <= 0.0:
        raise RuntimeError("invalid sample_rate in " + sidecar_path(payload_path))
    return iq, rate, int(meta["start_time"]), float(meta.get("center_freq", 0.0)), meta.get("creator", "")


def detection_json_line(rec, tag_id):
    """recording.cpp:228-242, through the library (the reference's own
    nlohmann dump: byte-identical number formatting and escaping)."""
    return capi.detection_json_line(rec, tag_id)


def detect_recording(ctx, payload_path, tags, window_s=0.100, overlap_s=0.010, threshold=0.25, cfg=None,
                     codes=None):
    """recording.cpp:258-289 on the GPU.  tags: list of (tag_id, seed) or of
    (tag_id, bits).  Returns (records, tag_ids): one Detection record per
    (window, tag), window-major like the reference's `all`."""
    iq, rate, start_time, _, _ = read_recording(payload_path)
    cfg = cfg or demod_config()
    cfg.mod.sample_rate = rate
    window = int(window_s * rate + 0.5)
    advance = int((window_s - overlap_s) * rate + 0.5)
    ids = [t[0] for t in tags]
    if codes is None:
        from .synth import gen_code
        bits = np.stack([np.asarray(t[1], np.uint8) if not np.isscalar(t[1]) else
                         gen_code(int(t[1]), int(cfg.mod.packet_bits)) for t in tags])
        codes = capi.CodeSet.prepare(ctx, cfg, window, bits)
    recs = capi.search(ctx, cfg, [cfg.lo_freq], iq, codes, window, advance, threshold, stream_start=start_time)
    return recs, ids


def detections_jsonl(records, tag_ids, all_candidates=False):
    """The `tagdsp detect` output (tagdsp_cli.cpp:76-86): accepted detections
    (or every candidate) as JSON lines."""
    n = len(tag_ids)
    return "".join(detection_json_line(r, tag_ids[i % n]) + "\n" for i, r in enumerate(records)
                   if all_candidates or r["accepted"])
