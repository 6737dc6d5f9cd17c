"""TEST INFRASTRUCTURE ONLY (oracle).  ctypes bindings for
oracle/_ref/libtagdsp_ref.so (the unmodified reference compiled in place, see
oracle/Makefile).  Only tests/, __graft_entry__.smoke() and bench.py's CPU
baseline / reference arm import this module."""
import ctypes
import os
import sys

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(_HERE))
from paper_2005_10445_b200._abi import DETECTION_DTYPE, DemodConfig, Modulation  # noqa: E402

REF_LIB = os.path.join(_HERE, "_ref", "libtagdsp_ref.so")
_P = ctypes.c_void_p
_U64 = ctypes.c_uint64
_I64 = ctypes.c_int64
_lib = None


def available():
    return os.path.exists(REF_LIB)


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(REF_LIB)
        sig = {
            "tdref_last_error": (ctypes.c_char_p, []),
            "tdref_pad_length": (_U64, [_U64]),
            "tdref_gen_code": (ctypes.c_int, [_U64, ctypes.POINTER(Modulation), _P]),
            "tdref_synth_replica": (ctypes.c_int, [_P, _U64, ctypes.POINTER(Modulation), _U64, _P]),
            "tdref_channel_window": (ctypes.c_int, [_P, _U64, ctypes.POINTER(Modulation), ctypes.c_double,
                                                    ctypes.c_double, ctypes.c_double, ctypes.c_double, _U64, _U64,
                                                    ctypes.c_float, _P]),
            "tdref_noise_window": (ctypes.c_int, [_U64, _U64, ctypes.c_float, _P]),
            "tdref_gaussian": (ctypes.c_int, [_U64, _U64, _P]),
            "tdref_generate_recording": (_I64, [ctypes.POINTER(DemodConfig), ctypes.c_float, _P, _U64,
                                                ctypes.c_double, ctypes.c_double, _U64, _P, _P, _P, _P, _U64, _P,
                                                _U64]),
            "tdref_demodulate_window": (ctypes.c_int, [_P, _U64, _I64, ctypes.POINTER(DemodConfig), _P, _P]),
            "tdref_demodulate_signal": (ctypes.c_int, [_P, _U64, _I64, ctypes.c_double,
                                                       ctypes.POINTER(DemodConfig), _P, _P]),
            "tdref_overlap_add": (ctypes.c_int, [_P, _U64, _P, _U64, _P]),
            "tdref_composed_filters": (ctypes.c_int, [ctypes.POINTER(DemodConfig), _P, _P]),
            "tdref_session_new": (_P, []),
            "tdref_session_free": (None, [_P]),
            "tdref_session_prepare_code": (_I64, [_P, _P, _U64, ctypes.POINTER(DemodConfig), _U64,
                                                  ctypes.c_char_p]),
            "tdref_session_make_transformed": (_I64, [_P, _P, _P, _U64, _U64, _U64]),
            "tdref_session_code_info": (ctypes.c_int, [_P, _I64, ctypes.POINTER(_U64),
                                                       ctypes.POINTER(ctypes.c_float),
                                                       ctypes.POINTER(ctypes.c_float), ctypes.POINTER(_U64)]),
            "tdref_session_code_replica": (ctypes.c_int, [_P, _I64, _P]),
            "tdref_session_code_spectrum": (ctypes.c_int, [_P, _I64, _P]),
            "tdref_session_batch_xcorr": (ctypes.c_int, [_P, _P, _U64, _P, _U64, _P]),
            "tdref_session_detect": (ctypes.c_int, [_P, _P, _P, _U64, _P, _U64, ctypes.c_float, _I64,
                                                    ctypes.c_double, ctypes.c_int32, _P]),
            "tdref_find_peak": (ctypes.c_int, [_P, _U64, ctypes.POINTER(_U64), ctypes.POINTER(ctypes.c_float)]),
            "tdref_interpolate_peak": (ctypes.c_float, [_P, _U64, _U64]),
            "tdref_search_bench": (ctypes.c_double, [_P, _U64, _I64, ctypes.POINTER(DemodConfig), _P, _U64, _P,
                                                     _U64, _U64, _U64, _U64, ctypes.c_float, ctypes.c_int,
                                                     ctypes.c_int, _P]),
            "tdref_search_bench_shared": (ctypes.c_double, [_P, _U64, _I64, ctypes.POINTER(DemodConfig), _P, _U64,
                                                            _P, _U64, _U64, _U64, _U64, ctypes.c_float, ctypes.c_int,
                                                            ctypes.c_int, _P, _P]),
            "tdref_run_detect_recording": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p]),
            "tdref_run_simulate": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_double,
                                                  ctypes.POINTER(_U64), ctypes.POINTER(_U64)]),
            "tdref_write_recording": (ctypes.c_int, [ctypes.c_char_p, _P, _U64, ctypes.c_double, _I64,
                                                     ctypes.c_double, ctypes.c_char_p]),
            "tdref_read_recording": (ctypes.c_int, [ctypes.c_char_p, _P, _U64, ctypes.POINTER(_U64),
                                                    ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_I64),
                                                    ctypes.POINTER(ctypes.c_double), ctypes.c_char_p, _U64]),
            "tdref_detection_json_line": (ctypes.c_int, [_P, ctypes.c_char_p, ctypes.c_char_p, _U64]),
            "tdref_ring_new": (_P, [_U64]),
            "tdref_ring_free": (None, [_P]),
            "tdref_ring_push": (ctypes.c_int, [_P, _P, _U64, _I64, ctypes.POINTER(_I64), ctypes.POINTER(_I64),
                                               ctypes.POINTER(ctypes.c_int32)]),
            "tdref_ring_read": (ctypes.c_int, [_P, _I64, _I64, _P, ctypes.POINTER(ctypes.c_int32)]),
            "tdref_ring_bounds": (None, [_P, ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
            "tdref_track_bench": (ctypes.c_double, [_P, _U64, _I64, ctypes.POINTER(DemodConfig), _P, _U64, _U64, _P,
                                                    _P, _U64, ctypes.c_float, _P]),
        }
        for k, (r, a) in sig.items():
            f = getattr(L, k)
            f.restype = r
            f.argtypes = a
        _lib = L
    return _lib


class RefError(RuntimeError):
    pass


def _ck(rc):
    if rc != 0:
        msg = lib().tdref_last_error().decode()
        if rc == 1:
            raise ValueError(msg)
        raise RefError(msg)


def _p(a):
    return ctypes.c_void_p(a.ctypes.data)


def pad_length(n):
    return int(lib().tdref_pad_length(n))


def gen_code(seed, cfg):
    out = np.empty(int(cfg.mod.packet_bits), dtype=np.uint8)
    _ck(lib().tdref_gen_code(seed, ctypes.byref(cfg.mod), _p(out)))
    return out


def synth_replica(bits, cfg, padded_len):
    bits = np.ascontiguousarray(bits, dtype=np.uint8)
    out = np.empty(2 * padded_len, dtype=np.float32)
    _ck(lib().tdref_synth_replica(_p(bits), bits.size, ctypes.byref(cfg.mod), padded_len, _p(out)))
    return out.view(np.complex64)


def channel_window(bits, cfg, delay, window_len, seed, snr_db=float("inf"), gain=1.0, freq_offset=0.0,
                   scale=8192.0):
    bits = np.ascontiguousarray(bits, dtype=np.uint8)
    out = np.empty(2 * window_len, dtype=np.int16)
    _ck(lib().tdref_channel_window(_p(bits), bits.size, ctypes.byref(cfg.mod), delay, snr_db, gain, freq_offset,
                                   window_len, seed, scale, _p(out)))
    return out


def noise_window(n, seed, scale):
    out = np.empty(2 * n, dtype=np.int16)
    _ck(lib().tdref_noise_window(n, seed, scale, _p(out)))
    return out


def gaussian(seed, n):
    out = np.empty(n, dtype=np.float32)
    _ck(lib().tdref_gaussian(seed, n, _p(out)))
    return out


def generate_recording(cfg, tag_seeds, duration_s, noise_snr_db, noise_seed, injections, quantize_scale=8192.0):
    """injections: list of (tag_index, time_s, gain, freq_offset)."""
    seeds = np.ascontiguousarray(tag_seeds, dtype=np.uint64)
    inj = list(injections)
    it = np.array([i[0] for i in inj], dtype=np.int32)
    tt = np.array([i[1] for i in inj], dtype=np.float64)
    gg = np.array([i[2] for i in inj], dtype=np.float64)
    ff = np.array([i[3] for i in inj], dtype=np.float64)
    total = int(duration_s * cfg.mod.sample_rate + 0.5)
    out = np.empty(2 * total, dtype=np.int16)
    n = lib().tdref_generate_recording(ctypes.byref(cfg), quantize_scale, _p(seeds), seeds.size, duration_s,
                                       noise_snr_db, noise_seed, _p(it) if len(inj) else None,
                                       _p(tt) if len(inj) else None, _p(gg) if len(inj) else None,
                                       _p(ff) if len(inj) else None, len(inj), _p(out), out.size)
    if n < 0:
        _ck(int(-n))
    return out[:2 * n]


def demodulate_window(iq, start, cfg):
    iq = np.ascontiguousarray(iq, dtype=np.int16)
    n = iq.size // 2
    d = np.empty(n, np.float32)
    u = np.empty(n, np.float32)
    _ck(lib().tdref_demodulate_window(_p(iq), n, start, ctypes.byref(cfg), _p(d), _p(u)))
    return d, u


def demodulate_signal(x, start, lo_freq, cfg):
    x = np.ascontiguousarray(x, dtype=np.complex64)
    d = np.empty(x.size, np.float32)
    u = np.empty(x.size, np.float32)
    _ck(lib().tdref_demodulate_signal(_p(x), x.size, start, lo_freq, ctypes.byref(cfg), _p(d), _p(u)))
    return d, u


def composed_filters(cfg):
    n = int(cfg.bandpass_taps) + int(round(cfg.mod.sample_rate / cfg.mod.bit_rate)) - 1
    h1 = np.empty(n, np.complex64)
    h0 = np.empty(n, np.complex64)
    _ck(lib().tdref_composed_filters(ctypes.byref(cfg), _p(h1), _p(h0)))
    return h1, h0


def find_peak(xc):
    xc = np.ascontiguousarray(xc, dtype=np.float32)
    j = _U64()
    v = ctypes.c_float()
    _ck(lib().tdref_find_peak(_p(xc), xc.size, ctypes.byref(j), ctypes.byref(v)))
    return j.value, v.value


def interpolate_peak(xc, j):
    xc = np.ascontiguousarray(xc, dtype=np.float32)
    return float(lib().tdref_interpolate_peak(_p(xc), xc.size, j))


class Session:
    """PlanCache + CodeCache of the reference (one per thread)."""

    def __init__(self):
        self.h = lib().tdref_session_new()

    def close(self):
        if self.h:
            lib().tdref_session_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def prepare_code(self, bits, cfg, window_len, tag_id="t"):
        bits = np.ascontiguousarray(bits, dtype=np.uint8)
        r = lib().tdref_session_prepare_code(self.h, _p(bits), bits.size, ctypes.byref(cfg), window_len,
                                             tag_id.encode())
        if r < 0:
            _ck(int(-r))
        return int(r)

    def make_transformed(self, replica_d, replica_u, window_len, corr_len):
        d = np.ascontiguousarray(replica_d, dtype=np.float32)
        u = None if replica_u is None else np.ascontiguousarray(replica_u, dtype=np.float32)
        r = lib().tdref_session_make_transformed(self.h, _p(d), _p(u) if u is not None else None, d.size,
                                                 window_len, corr_len)
        if r < 0:
            _ck(int(-r))
        return int(r)

    def code_info(self, idx):
        n = _U64()
        e = ctypes.c_float()
        a = ctypes.c_float()
        c = _U64()
        _ck(lib().tdref_session_code_info(self.h, idx, ctypes.byref(n), ctypes.byref(e), ctypes.byref(a),
                                          ctypes.byref(c)))
        return {"nonzero_len": n.value, "energy": e.value, "abs_sum": a.value, "corr_len": c.value}

    def code_replica(self, idx):
        out = np.empty(self.code_info(idx)["nonzero_len"], np.float32)
        _ck(lib().tdref_session_code_replica(self.h, idx, _p(out)))
        return out

    def code_spectrum(self, idx):
        out = np.empty(self.code_info(idx)["corr_len"], np.complex64)
        _ck(lib().tdref_session_code_spectrum(self.h, idx, _p(out)))
        return out

    def batch_xcorr(self, d, idx):
        d = np.ascontiguousarray(d, dtype=np.float32)
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        out = np.empty((idx.size, d.size), np.float32)
        _ck(lib().tdref_session_batch_xcorr(self.h, _p(d), d.size, _p(idx), idx.size, _p(out)))
        return out

    def detect(self, d, u, idx, threshold, window_start, sample_rate, bin_index=0):
        d = np.ascontiguousarray(d, dtype=np.float32)
        u = np.ascontiguousarray(u, dtype=np.float32)
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        out = np.zeros(idx.size, DETECTION_DTYPE)
        _ck(lib().tdref_session_detect(self.h, _p(d), _p(u), d.size, _p(idx), idx.size, threshold, window_start,
                                       sample_rate, bin_index, _p(out)))
        return out


def search_bench(iq, stream_start, cfg, lo_bins, bits, window_len, advance, n_windows, threshold, threads,
                 code_chunk=0):
    """Timed reference searching pass; returns (seconds, detections [w][b][c])."""
    iq = np.ascontiguousarray(iq, dtype=np.int16)
    bins = np.ascontiguousarray(lo_bins, dtype=np.float64)
    bits = np.ascontiguousarray(bits, dtype=np.uint8)
    n_codes = bits.shape[0]
    out = np.zeros(n_windows * bins.size * n_codes, DETECTION_DTYPE)
    t = lib().tdref_search_bench(_p(iq), iq.size // 2, stream_start, ctypes.byref(cfg), _p(bins), bins.size,
                                 _p(bits), n_codes, window_len, advance, n_windows, threshold, threads, code_chunk,
                                 _p(out))
    if t < 0:
        _ck(int(-t))
    return t, out


def search_bench_shared(iq, stream_start, cfg, lo_bins, bits, window_len, advance, n_windows, threshold, threads,
                        code_chunk=4):
    """The reference's own loop (one demodulate_window per (window, bin),
    shared by all codes) on `threads` host threads.  Returns (seconds,
    detections [w][b][c], stage thread-seconds {demod, correlation,
    peak_stats})."""
    iq = np.ascontiguousarray(iq, dtype=np.int16)
    bins = np.ascontiguousarray(lo_bins, dtype=np.float64)
    bits = np.ascontiguousarray(np.atleast_2d(bits), dtype=np.uint8)
    n_codes = bits.shape[0]
    out = np.zeros(n_windows * bins.size * n_codes, DETECTION_DTYPE)
    st = np.zeros(3, np.float64)
    t = lib().tdref_search_bench_shared(_p(iq), iq.size // 2, stream_start, ctypes.byref(cfg), _p(bins), bins.size,
                                        _p(bits), n_codes, window_len, advance, n_windows, threshold, threads,
                                        code_chunk, _p(out), _p(st))
    if t < 0:
        _ck(int(-t))
    return t, out, {"demod": float(st[0]), "correlation": float(st[1]), "peak_stats": float(st[2])}


def track_bench(iq, stream_start, cfg, bits, window_len, starts, code_idx, threshold):
    """Tracking tasks through the reference (single thread): (seconds, detections)."""
    iq = np.ascontiguousarray(iq, dtype=np.int16)
    bits = np.ascontiguousarray(np.atleast_2d(bits), dtype=np.uint8)
    st = np.ascontiguousarray(starts, dtype=np.int64)
    ci = np.ascontiguousarray(code_idx, dtype=np.uint64)
    out = np.zeros(st.size, DETECTION_DTYPE)
    t = lib().tdref_track_bench(_p(iq), iq.size // 2, stream_start, ctypes.byref(cfg), _p(bits), bits.shape[0],
                                window_len, _p(st), _p(ci), st.size, threshold, _p(out))
    if t < 0:
        _ck(int(-t))
    return t, out


def run_detect_recording(rec_path, cfg_path, out_path):
    """The reference's detect_recording over a recording file, JSON lines out."""
    _ck(lib().tdref_run_detect_recording(str(rec_path).encode(), str(cfg_path).encode(), str(out_path).encode()))


def run_simulate(rec_path, cfg_path, out_path, compute_ratio):
    """The reference's simulate_recording; event JSON lines out; returns (detections, misses)."""
    d, m = _U64(), _U64()
    _ck(lib().tdref_run_simulate(str(rec_path).encode(), str(cfg_path).encode(), str(out_path).encode(),
                                 float(compute_ratio), ctypes.byref(d), ctypes.byref(m)))
    return d.value, m.value


def write_recording(path, iq, sample_rate, start_time=0, center_freq=0.0, creator=""):
    iq = np.ascontiguousarray(iq, dtype=np.int16)
    _ck(lib().tdref_write_recording(str(path).encode(), _p(iq), iq.size // 2, float(sample_rate), int(start_time),
                                    float(center_freq), creator.encode()))


def read_recording(path, cap_complex):
    out = np.empty(2 * cap_complex, np.int16)
    n, rate, start, cf = _U64(), ctypes.c_double(), _I64(), ctypes.c_double()
    creator = ctypes.create_string_buffer(4096)
    _ck(lib().tdref_read_recording(str(path).encode(), _p(out), out.size, ctypes.byref(n), ctypes.byref(rate),
                                   ctypes.byref(start), ctypes.byref(cf), creator, 4096))
    return out[:2 * n.value], rate.value, start.value, cf.value, creator.value.decode()


def detection_json_line(rec, tag_id):
    r = np.ascontiguousarray(np.atleast_1d(rec).astype(DETECTION_DTYPE))
    buf = ctypes.create_string_buffer(4096)
    _ck(lib().tdref_detection_json_line(_p(r), tag_id.encode(), buf, 4096))
    return buf.value.decode()


class Ring:
    """The reference CircularBuffer (proj/src/scheduler.cpp:7-45)."""

    def __init__(self, capacity):
        self.h = lib().tdref_ring_new(int(capacity))

    def push(self, iq, start):
        iq = np.ascontiguousarray(iq, dtype=np.int16)
        b, e, g = _I64(), _I64(), ctypes.c_int32()
        _ck(lib().tdref_ring_push(self.h, _p(iq), iq.size // 2, int(start), ctypes.byref(b), ctypes.byref(e),
                                  ctypes.byref(g)))
        return b.value, e.value, bool(g.value)

    def read(self, start, end):
        out = np.empty(2 * max(0, int(end) - int(start)), np.int16)
        ok = ctypes.c_int32()
        _ck(lib().tdref_ring_read(self.h, int(start), int(end), _p(out), ctypes.byref(ok)))
        return out if ok.value else None

    def bounds(self):
        h, t = _I64(), _I64()
        lib().tdref_ring_bounds(self.h, ctypes.byref(h), ctypes.byref(t))
        return h.value, t.value

    def __del__(self):
        try:
            lib().tdref_ring_free(self.h)
        except Exception:
            pass
