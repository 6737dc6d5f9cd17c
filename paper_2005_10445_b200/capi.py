"""Python mirror of the reference tagdsp detector API over the B200 C-ABI.

Every call goes through libtagdsp_gpu.so (include/tagdsp_gpu.h); there is no
CPU fallback -- if the library is missing or no CUDA device is usable the
call raises.  Names and argument meaning follow the reference
(/root/reference/proj/include/tagdsp/{dsp,detector}.hpp):

  demodulate_window(ctx, iq, start, cfg)      dsp.hpp:70-71
  prepare_codes(ctx, cfg, window_len, bits)   detector.hpp:67-68 (batched)
  make_transformed(ctx, replicas, ...)        detector.hpp:60-62 (batched)
  batch_xcorr(ctx, windows, slot, codes, idx) detector.hpp:75-77
  detect(ctx, windows, codes, threshold, fs)  detector.hpp:103-106
  search(ctx, cfg, bins, iq, ...)             recording.cpp:258-289 (detect_recording)
  track(ctx, cfg, iq, tasks, codes)           recording.cpp:360-378 (tracking tasks, batched)
  Ring(ctx, capacity).push/read/bounds        scheduler.hpp:11-40 (CircularBuffer, device-resident)
  search_ring / track_ring                    the same passes reading windows from a Ring

Errors: TDG_EINVAL -> InvalidArgument (a ValueError, the reference's
std::invalid_argument), anything else -> GpuError (RuntimeError).
"""
import ctypes
import os

import numpy as np

from ._abi import (DETECTION_DTYPE, TRACK_TASK_DTYPE, DemodConfig, RingPushResult, demod_config,  # noqa: F401
                   desk_config)

_HERE = os.path.dirname(os.path.abspath(__file__))
# TDG_LIB_PATH: load another build of the same library (A/B timing of
# compile-time variants with tools/; still the CUDA path, never a fallback)
LIB_PATH = os.environ.get("TDG_LIB_PATH") or os.path.join(_HERE, "libtagdsp_gpu.so")

TDG_OK, TDG_EINVAL, TDG_ECUDA, TDG_ENOMEM, TDG_ERANGE, TDG_EINTERNAL = range(6)


class GpuError(RuntimeError):
    pass


class InvalidArgument(ValueError):
    pass


_lib = None

_P = ctypes.c_void_p
_U64 = ctypes.c_uint64
_I64 = ctypes.c_int64
_PROTOS = {
    "tdg_last_error": (ctypes.c_char_p, []),
    "tdg_version": (ctypes.c_char_p, []),
    "tdg_kernel_launches": (_U64, []),
    "tdg_ctx_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_P)]),
    "tdg_ctx_destroy": (None, [_P]),
    "tdg_ctx_synchronize": (ctypes.c_int, [_P]),
    "tdg_ctx_stream": (_P, [_P]),
    "tdg_pad_length": (_U64, [_U64]),
    "tdg_corr_len": (_U64, [_U64, _U64]),
    "tdg_codeset_prepare": (ctypes.c_int, [_P, ctypes.POINTER(DemodConfig), _U64, _P, _U64, ctypes.POINTER(_P)]),
    "tdg_codeset_from_replicas": (ctypes.c_int, [_P, _U64, _U64, _P, _P, _P, _U64, ctypes.POINTER(_P)]),
    "tdg_codeset_append": (ctypes.c_int, [_P, _P, ctypes.POINTER(DemodConfig), _P, _U64]),
    "tdg_codeset_destroy": (None, [_P]),
    "tdg_codeset_size": (_U64, [_P]),
    "tdg_codeset_info": (ctypes.c_int, [_P, _U64, ctypes.POINTER(_U64), ctypes.POINTER(ctypes.c_float),
                                        ctypes.POINTER(ctypes.c_float), ctypes.POINTER(_U64)]),
    "tdg_codeset_replica": (ctypes.c_int, [_P, _U64, _P]),
    "tdg_windows_create": (ctypes.c_int, [_P, _U64, _U64, _U64, ctypes.POINTER(_P)]),
    "tdg_windows_destroy": (None, [_P]),
    "tdg_demodulate": (ctypes.c_int, [_P, _P, ctypes.POINTER(DemodConfig), _P, _U64, _P, _U64, _I64, _U64, _U64]),
    "tdg_demodulate_device": (ctypes.c_int, [_P, _P, ctypes.POINTER(DemodConfig), _P, _U64, _P, _U64, _I64, _U64,
                                             _U64]),
    "tdg_windows_set_du": (ctypes.c_int, [_P, _P, _U64, _P, _P, _I64]),
    "tdg_windows_get_du": (ctypes.c_int, [_P, _P, _U64, _P, _P]),
    "tdg_windows_set_start": (ctypes.c_int, [_P, _P, _U64, _I64]),
    "tdg_detect": (ctypes.c_int, [_P, _P, _P, ctypes.c_float, ctypes.c_double, _P, _U64]),
    "tdg_detect_codes": (ctypes.c_int, [_P, _P, _P, _P, _U64, ctypes.c_float, ctypes.c_double, _P, _U64]),
    "tdg_batch_xcorr": (ctypes.c_int, [_P, _P, _U64, _P, _P, _U64, _P]),
    "tdg_search": (ctypes.c_int, [_P, ctypes.POINTER(DemodConfig), _P, _U64, _P, _U64, _I64, _U64, _U64, _P,
                                  ctypes.c_float, _P, _U64, ctypes.POINTER(_U64)]),
    "tdg_track": (ctypes.c_int, [_P, ctypes.POINTER(DemodConfig), _P, _U64, _I64, _P, _U64, _P, ctypes.c_float,
                                 _P]),
    "tdg_track_device": (ctypes.c_int, [_P, ctypes.POINTER(DemodConfig), _P, _U64, _I64, _P, _U64, _P,
                                        ctypes.c_float, _P]),
    "tdg_ring_create": (ctypes.c_int, [_P, _U64, ctypes.POINTER(_P)]),
    "tdg_ring_destroy": (None, [_P]),
    "tdg_ring_push": (ctypes.c_int, [_P, _P, _U64, _I64, ctypes.POINTER(RingPushResult)]),
    "tdg_ring_read": (ctypes.c_int, [_P, _I64, _I64, _P, ctypes.POINTER(ctypes.c_int)]),
    "tdg_ring_bounds": (ctypes.c_int, [_P, ctypes.POINTER(_I64), ctypes.POINTER(_I64), ctypes.POINTER(_U64)]),
    "tdg_search_ring": (ctypes.c_int, [_P, _P, ctypes.POINTER(DemodConfig), _P, _U64, _I64, _U64, _U64, _U64, _P,
                                       ctypes.c_float, _P, _U64, ctypes.c_int]),
    "tdg_track_ring": (ctypes.c_int, [_P, _P, ctypes.POINTER(DemodConfig), _P, _U64, _P, ctypes.c_float, _P,
                                      ctypes.c_int]),
    "tdg_set_option": (ctypes.c_int, [_P, ctypes.c_char_p, _I64]),
    "tdg_kernel_time": (ctypes.c_int, [_P, ctypes.c_char_p, ctypes.POINTER(_U64), ctypes.POINTER(ctypes.c_double)]),
    "tdg_kernel_time_reset": (ctypes.c_int, [_P]),
    "tdg_cta_trace": (ctypes.c_int, [_P, _P, _U64, ctypes.POINTER(_U64)]),
    "tdg_fft": (ctypes.c_int, [_P, _P, _P, _U64, ctypes.c_int]),
    "tdg_convert": (ctypes.c_int, [_P, _P, _U64, _P]),
    "tdg_mix": (ctypes.c_int, [_P, _P, _U64, ctypes.c_double, _I64, ctypes.c_double]),
    "tdg_convolve": (ctypes.c_int, [_P, _P, _U64, _P, _U64, _P]),
    "tdg_discriminate": (ctypes.c_int, [_P, _P, _P, _U64, ctypes.c_float, _P, _P]),
    "tdg_find_peak": (ctypes.c_int, [_P, _P, _U64, ctypes.POINTER(_U64), ctypes.POINTER(ctypes.c_float)]),
    "tdg_statistics": (ctypes.c_int, [_P, _P, _P, _U64, _P, _U64, _U64, ctypes.POINTER(ctypes.c_float),
                                      ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float),
                                      ctypes.POINTER(ctypes.c_int)]),
    "tdg_demodulate_signal": (ctypes.c_int, [_P, _P, ctypes.POINTER(DemodConfig), ctypes.c_double, _P, _U64, _I64]),
    "tdg_detect_timings": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
    "tdg_detection_json_line": (ctypes.c_int, [_P, ctypes.c_char_p, ctypes.c_char_p, _U64, ctypes.POINTER(_U64)]),
    "tdg_fp32_peak": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
}
EXPORTED_SYMBOLS = sorted(_PROTOS)


def lib():
    """Load libtagdsp_gpu.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise GpuError("libtagdsp_gpu.so not built (run __graft_entry__.build()); "
                           "there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _PROTOS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(rc):
    if rc != TDG_OK:
        msg = lib().tdg_last_error().decode(errors="replace")
        if rc == TDG_EINVAL:
            raise InvalidArgument(msg)
        raise GpuError("tagdsp_gpu error %d: %s" % (rc, msg))


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


def kernel_launches():
    return int(lib().tdg_kernel_launches())


def fp32_peak(device=0):
    """(FFMA, FFMA2) TFLOP/s measured on `device` at its current clock."""
    a, b = ctypes.c_double(), ctypes.c_double()
    _check(lib().tdg_fp32_peak(int(device), ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def pad_length(n):
    """pad_length (proj/src/fft.cpp:93-101)."""
    if n < 1:
        raise InvalidArgument("pad_length: n must be >= 1")
    return int(lib().tdg_pad_length(n))


def corr_len(window_len, nonzero_len):
    return int(lib().tdg_corr_len(window_len, nonzero_len))


class Context:
    """One CUDA device + stream + plan tables (the reference's PlanCache role)."""

    def __init__(self, device=0):
        h = ctypes.c_void_p()
        _check(lib().tdg_ctx_create(int(device), ctypes.byref(h)))
        self._h = h
        self.device = device

    @property
    def handle(self):
        return self._h

    def stream(self):
        return int(lib().tdg_ctx_stream(self._h) or 0)

    def synchronize(self):
        _check(lib().tdg_ctx_synchronize(self._h))

    def set_option(self, key, value):
        _check(lib().tdg_set_option(self._h, key.encode(), int(value)))

    def kernel_time(self, name):
        """(launch count, total device ms) of a kernel family (time_kernels=1)."""
        n = _U64()
        ms = ctypes.c_double()
        _check(lib().tdg_kernel_time(self._h, name.encode(), ctypes.byref(n), ctypes.byref(ms)))
        return n.value, ms.value

    def kernel_time_reset(self):
        _check(lib().tdg_kernel_time_reset(self._h))

    def close(self):
        if getattr(self, "_h", None):
            lib().tdg_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


class CodeSet:
    """Device-resident TransformedCodes for one window shape (CodeCache)."""

    def __init__(self, ctx, handle, window_len):
        self.ctx = ctx
        self._h = handle
        self.window_len = window_len

    @classmethod
    def prepare(cls, ctx, cfg, window_len, bits):
        """prepare_code (proj/src/detector.cpp:50-66) for every row of `bits`."""
        bits = np.ascontiguousarray(np.atleast_2d(bits), dtype=np.uint8)
        if bits.shape[1] != int(cfg.mod.packet_bits):
            raise InvalidArgument("bits rows must have packet_bits entries")
        h = ctypes.c_void_p()
        _check(lib().tdg_codeset_prepare(ctx.handle, ctypes.byref(cfg), int(window_len), _ptr(bits),
                                         bits.shape[0], ctypes.byref(h)))
        return cls(ctx, h, int(window_len))

    def append(self, cfg, bits):
        """prepare_code for more codes of the same configuration (appended)."""
        bits = np.ascontiguousarray(np.atleast_2d(bits), dtype=np.uint8)
        _check(lib().tdg_codeset_append(self.ctx.handle, self._h, ctypes.byref(cfg), _ptr(bits), bits.shape[0]))

    @classmethod
    def from_replicas(cls, ctx, window_len, corr_len, replicas_d, replicas_u=None):
        """make_transformed (proj/src/detector.cpp:11-48) for each replica."""
        ds = [np.ascontiguousarray(r, dtype=np.float32) for r in replicas_d]
        us = None if replicas_u is None else [np.ascontiguousarray(r, dtype=np.float32) for r in replicas_u]
        n = len(ds)
        lens = np.array([len(r) for r in ds], dtype=np.uint64)
        dp = (ctypes.c_void_p * n)(*[r.ctypes.data for r in ds])
        up = None if us is None else (ctypes.c_void_p * n)(*[r.ctypes.data for r in us])
        h = ctypes.c_void_p()
        _check(lib().tdg_codeset_from_replicas(ctx.handle, int(window_len), int(corr_len), ctypes.cast(dp, _P),
                                               ctypes.cast(up, _P) if up is not None else None, _ptr(lens), n,
                                               ctypes.byref(h)))
        return cls(ctx, h, int(window_len))

    def __len__(self):
        return int(lib().tdg_codeset_size(self._h))

    def info(self, i):
        n = _U64()
        e = ctypes.c_float()
        a = ctypes.c_float()
        c = _U64()
        _check(lib().tdg_codeset_info(self._h, int(i), ctypes.byref(n), ctypes.byref(e), ctypes.byref(a),
                                      ctypes.byref(c)))
        return {"nonzero_len": n.value, "energy": e.value, "abs_sum": a.value, "corr_len": c.value}

    def replica(self, i):
        n = self.info(i)["nonzero_len"]
        out = np.empty(n, dtype=np.float32)
        _check(lib().tdg_codeset_replica(self._h, int(i), _ptr(out)))
        return out

    def close(self):
        if getattr(self, "_h", None):
            lib().tdg_codeset_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Windows:
    """Device-resident demodulated windows: slot = window * n_bins + bin."""

    def __init__(self, ctx, window_len, n_windows=1, n_bins=1):
        h = ctypes.c_void_p()
        _check(lib().tdg_windows_create(ctx.handle, int(window_len), int(n_windows), int(n_bins), ctypes.byref(h)))
        self.ctx = ctx
        self._h = h
        self.window_len = int(window_len)
        self.n_windows = int(n_windows)
        self.n_bins = int(n_bins)

    @property
    def slots(self):
        return self.n_windows * self.n_bins

    def demodulate(self, cfg, lo_bins, iq, stream_start=0, advance=None, n_windows=None):
        """demodulate_window (proj/src/dsp.cpp:193-197) for windows x bins."""
        iq = np.ascontiguousarray(iq, dtype=np.int16)
        if iq.size % 2:
            raise InvalidArgument("convert: odd raw sample count")
        bins = np.ascontiguousarray(np.atleast_1d(lo_bins), dtype=np.float64)
        nw = self.n_windows if n_windows is None else int(n_windows)
        adv = self.window_len if advance is None else int(advance)
        _check(lib().tdg_demodulate(self.ctx.handle, self._h, ctypes.byref(cfg), _ptr(bins), bins.size, _ptr(iq),
                                    iq.size // 2, int(stream_start), adv, nw))

    def set_du(self, slot, d, u, window_start=0):
        d = np.ascontiguousarray(d, dtype=np.float32)
        u = np.ascontiguousarray(u, dtype=np.float32)
        if d.size != self.window_len or u.size != self.window_len:
            raise InvalidArgument("detect: d/u length must equal the window length")
        _check(lib().tdg_windows_set_du(self.ctx.handle, self._h, int(slot), _ptr(d), _ptr(u), int(window_start)))

    def get_du(self, slot):
        d = np.empty(self.window_len, dtype=np.float32)
        u = np.empty(self.window_len, dtype=np.float32)
        _check(lib().tdg_windows_get_du(self.ctx.handle, self._h, int(slot), _ptr(d), _ptr(u)))
        return d, u

    def close(self):
        if getattr(self, "_h", None):
            lib().tdg_windows_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def demodulate_window(ctx, iq, start, cfg):
    """demodulate_window(block, cfg) -> (d, u) for one block at cfg.lo_freq."""
    iq = np.ascontiguousarray(iq, dtype=np.int16)
    if iq.size % 2:
        raise InvalidArgument("convert: odd raw sample count")
    n = iq.size // 2
    if n == 0:
        return np.empty(0, np.float32), np.empty(0, np.float32)
    w = Windows(ctx, n, 1, 1)
    try:
        w.demodulate(cfg, [cfg.lo_freq], iq, start, n, 1)
        return w.get_du(0)
    finally:
        w.close()


def detect(ctx, windows, codes, threshold=0.25, sample_rate=8.0e6, idx=None):
    """detect() for every slot x code (or the codes `idx`, in that order)
    -> DETECTION_DTYPE records [slot][code]."""
    if idx is None:
        out = np.zeros(windows.slots * len(codes), dtype=DETECTION_DTYPE)
        _check(lib().tdg_detect(ctx.handle, windows._h, codes._h, float(threshold), float(sample_rate), _ptr(out),
                                out.size))
        return out
    idx = np.ascontiguousarray(np.atleast_1d(idx), dtype=np.int64)
    out = np.zeros(windows.slots * idx.size, dtype=DETECTION_DTYPE)
    _check(lib().tdg_detect_codes(ctx.handle, windows._h, codes._h, _ptr(idx), idx.size, float(threshold),
                                  float(sample_rate), _ptr(out), out.size))
    return out


def batch_xcorr(ctx, windows, slot, codes, idx=None):
    """batch_xcorr (proj/src/detector.cpp:102-120): xc[t], t < W, per code."""
    idx = np.arange(len(codes), dtype=np.int64) if idx is None else np.ascontiguousarray(idx, dtype=np.int64)
    out = np.empty((idx.size, windows.window_len), dtype=np.float32)
    _check(lib().tdg_batch_xcorr(ctx.handle, windows._h, int(slot), codes._h, _ptr(idx), idx.size, _ptr(out)))
    return out


def search(ctx, cfg, lo_bins, iq, codes, window_len, advance, threshold=0.25, stream_start=0, out=None):
    """Searching pass over a stream (detect_recording with an lo_freq sweep)."""
    iq = np.ascontiguousarray(iq, dtype=np.int16)
    bins = np.ascontiguousarray(np.atleast_1d(lo_bins), dtype=np.float64)
    n = iq.size // 2
    nw = (n - window_len) // advance + 1 if n >= window_len else 0
    total = nw * bins.size * len(codes)
    if out is None:
        out = np.zeros(total, dtype=DETECTION_DTYPE)
    n_out = _U64()
    _check(lib().tdg_search(ctx.handle, ctypes.byref(cfg), _ptr(bins), bins.size, _ptr(iq), n, int(stream_start),
                            int(window_len), int(advance), codes._h, float(threshold), _ptr(out), out.size,
                            ctypes.byref(n_out)))
    return out[:n_out.value]


def track(ctx, cfg, iq, starts, code_idx, codes, threshold=0.25, stream_start=0):
    """Tracking tasks (proj/src/recording.cpp:360-378, one scheduler Task of
    kind Tracking each): window [starts[i], starts[i] + codes.window_len)
    demodulated at cfg.lo_freq and detected against code code_idx[i].
    Returns DETECTION_DTYPE records, one per task."""
    iq = np.ascontiguousarray(iq, dtype=np.int16)
    tasks = np.zeros(len(starts), dtype=TRACK_TASK_DTYPE)
    tasks["start"] = starts
    tasks["code_index"] = code_idx
    out = np.zeros(tasks.size, dtype=DETECTION_DTYPE)
    _check(lib().tdg_track(ctx.handle, ctypes.byref(cfg), _ptr(iq), iq.size // 2, int(stream_start), _ptr(tasks),
                           tasks.size, codes._h, float(threshold), _ptr(out)))
    return out


class Ring:
    """Device-resident CircularBuffer (proj/include/tagdsp/scheduler.hpp:11-40):
    push(block, start) -> (evicted_begin, evicted_end, gap); read(start, end)
    -> int16 I/Q or None if any part was evicted / not yet received."""

    def __init__(self, ctx, capacity):
        self.ctx = ctx
        h = _P()
        _check(lib().tdg_ring_create(ctx.handle, int(capacity), ctypes.byref(h)))
        self._h = h
        self._keep = []   # host blocks whose asynchronous upload may still be in flight

    def push(self, iq, start):
        iq = np.ascontiguousarray(iq, dtype=np.int16)
        if iq.size % 2:
            raise InvalidArgument("convert: odd raw sample count")
        res = RingPushResult()
        self._keep = self._keep[-3:] + [iq]
        _check(lib().tdg_ring_push(self._h, _ptr(iq), iq.size // 2, int(start), ctypes.byref(res)))
        return res.evicted_begin, res.evicted_end, bool(res.gap)

    def read(self, start, end):
        out = np.empty(2 * max(0, int(end) - int(start)), dtype=np.int16)
        ok = ctypes.c_int()
        _check(lib().tdg_ring_read(self._h, int(start), int(end), _ptr(out), ctypes.byref(ok)))
        return out if ok.value else None

    def bounds(self):
        h, t, c = _I64(), _I64(), _U64()
        _check(lib().tdg_ring_bounds(self._h, ctypes.byref(h), ctypes.byref(t), ctypes.byref(c)))
        return h.value, t.value, c.value

    @property
    def head(self):
        return self.bounds()[0]

    @property
    def tail(self):
        return self.bounds()[1]

    def close(self):
        if getattr(self, "_h", None):
            lib().tdg_ring_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def search_ring(ctx, ring, cfg, lo_bins, first_start, n_windows, codes, advance, threshold=0.25):
    """Searching pass over windows [first_start + w*advance, + codes.window_len) held by `ring`."""
    bins = np.ascontiguousarray(np.atleast_1d(lo_bins), dtype=np.float64)
    out = np.zeros(int(n_windows) * bins.size * len(codes), dtype=DETECTION_DTYPE)
    _check(lib().tdg_search_ring(ctx.handle, ring._h, ctypes.byref(cfg), _ptr(bins), bins.size, int(first_start),
                                 codes.window_len, int(advance), int(n_windows), codes._h, float(threshold), _ptr(out),
                                 out.size, 1))
    return out


def track_ring(ctx, ring, cfg, starts, code_idx, codes, threshold=0.25):
    """Tracking tasks reading their windows from `ring` (see track())."""
    tasks = np.zeros(len(starts), dtype=TRACK_TASK_DTYPE)
    tasks["start"] = starts
    tasks["code_index"] = code_idx
    out = np.zeros(tasks.size, dtype=DETECTION_DTYPE)
    _check(lib().tdg_track_ring(ctx.handle, ring._h, ctypes.byref(cfg), _ptr(tasks), tasks.size, codes._h,
                                float(threshold), _ptr(out), 1))
    return out


# ---- span-level functions (reference free functions on host arrays) --------
def fft(ctx, x, inverse=False):
    """PlanCache::forward / inverse (proj/src/fft.cpp:46-67) on the GPU."""
    x = np.ascontiguousarray(x, dtype=np.complex64)
    out = np.empty_like(x)
    _check(lib().tdg_fft(ctx.handle, _ptr(x), _ptr(out), x.size, int(bool(inverse))))
    return out


def convert(ctx, iq):
    iq = np.ascontiguousarray(iq, dtype=np.int16)
    out = np.empty(iq.size // 2, np.complex64)
    _check(lib().tdg_convert(ctx.handle, _ptr(iq), iq.size, _ptr(out)))
    return out


def mix(ctx, x, lo_freq, start_index, sample_rate):
    x = np.array(x, dtype=np.complex64, copy=True)
    _check(lib().tdg_mix(ctx.handle, _ptr(x), x.size, float(lo_freq), int(start_index), float(sample_rate)))
    return x


def convolve(ctx, x, h):
    x = np.ascontiguousarray(x, dtype=np.complex64)
    h = np.ascontiguousarray(h, dtype=np.complex64)
    out = np.empty(max(0, x.size + h.size - 1) if x.size else 0, np.complex64)
    _check(lib().tdg_convolve(ctx.handle, _ptr(x), x.size, _ptr(h), h.size, _ptr(out)))
    return out


def discriminate(ctx, f1, f0, eps=1e-12):
    f1 = np.ascontiguousarray(f1, dtype=np.complex64)
    f0 = np.ascontiguousarray(f0, dtype=np.complex64)
    d = np.empty(f1.size, np.float32)
    u = np.empty(f1.size, np.float32)
    _check(lib().tdg_discriminate(ctx.handle, _ptr(f1), _ptr(f0), f1.size, float(eps), _ptr(d), _ptr(u)))
    return d, u


def find_peak(ctx, xc):
    xc = np.ascontiguousarray(xc, dtype=np.float32)
    j, v = _U64(), ctypes.c_float()
    _check(lib().tdg_find_peak(ctx.handle, _ptr(xc), xc.size, ctypes.byref(j), ctypes.byref(v)))
    return j.value, v.value


def statistics(ctx, d, u, dc, j):
    d = np.ascontiguousarray(d, dtype=np.float32)
    u = np.ascontiguousarray(u, dtype=np.float32)
    dc = np.ascontiguousarray(dc, dtype=np.float32)
    w, q, p, part = ctypes.c_float(), ctypes.c_float(), ctypes.c_float(), ctypes.c_int()
    _check(lib().tdg_statistics(ctx.handle, _ptr(d), _ptr(u), d.size, _ptr(dc), dc.size, int(j), ctypes.byref(w),
                                ctypes.byref(q), ctypes.byref(p), ctypes.byref(part)))
    return {"w_c": w.value, "q": q.value, "p_c": p.value, "partial": bool(part.value)}


def demodulate_signal(ctx, x, start_index, lo_freq, cfg):
    x = np.ascontiguousarray(x, dtype=np.complex64)
    w = Windows(ctx, x.size, 1, 1)
    try:
        _check(lib().tdg_demodulate_signal(ctx.handle, w._h, ctypes.byref(cfg), float(lo_freq), _ptr(x), x.size,
                                           int(start_index)))
        return w.get_du(0)
    finally:
        w.close()


def detection_json_line(rec, tag_id):
    """detection_json_line (proj/src/recording.cpp:228-242), byte-identical."""
    r = np.ascontiguousarray(np.atleast_1d(rec).astype(DETECTION_DTYPE))
    buf = ctypes.create_string_buffer(1024 + 8 * len(tag_id))
    n = _U64()
    _check(lib().tdg_detection_json_line(_ptr(r), tag_id.encode(), buf, len(buf), ctypes.byref(n)))
    return buf.raw[:n.value].decode()
