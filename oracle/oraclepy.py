"""TEST INFRASTRUCTURE ONLY (oracle).  ctypes bindings for oracle/liboracle.so,
the plain-C restatement of the reference path (oracle/tagdsp_oracle.c).
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg use it."""
import ctypes
import os
import sys

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(_HERE))
from paper_2005_10445_b200._abi import DETECTION_DTYPE, DemodConfig, Modulation  # noqa: E402

LIB = os.path.join(_HERE, "liboracle.so")
_P = ctypes.c_void_p
_U64 = ctypes.c_uint64
_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(LIB)
        sig = {
            "tdo_gaussian": (None, [_U64, _U64, _P]),
            "tdo_gen_code": (None, [_U64, _U64, _P]),
            "tdo_synth_replica": (None, [_P, _U64, ctypes.POINTER(Modulation), _U64, _P]),
            "tdo_pad_length": (_U64, [_U64]),
            "tdo_demodulate_signal": (ctypes.c_int, [_P, _U64, ctypes.c_int64, ctypes.c_double,
                                                     ctypes.POINTER(DemodConfig), _P, _P]),
            "tdo_demodulate_window": (ctypes.c_int, [_P, _U64, ctypes.c_int64, ctypes.POINTER(DemodConfig), _P, _P]),
            "tdo_make_transformed": (ctypes.c_int, [_P, _P, _U64, _U64, _U64, ctypes.POINTER(_U64),
                                                    ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float),
                                                    _P]),
            "tdo_prepare_code": (ctypes.c_int, [_P, ctypes.POINTER(DemodConfig), _U64, ctypes.POINTER(_U64),
                                                ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float), _P,
                                                _P, ctypes.POINTER(_U64)]),
            "tdo_batch_xcorr": (ctypes.c_int, [_P, _U64, _P, _P, _U64, _U64, _P]),
            "tdo_find_peak": (ctypes.c_int, [_P, _U64, ctypes.POINTER(_U64), ctypes.POINTER(ctypes.c_float)]),
            "tdo_interpolate_peak": (ctypes.c_float, [_P, _U64, _U64]),
            "tdo_detect": (ctypes.c_int, [_P, _P, _U64, _P, _P, _P, _P, _U64, _U64, ctypes.c_float, ctypes.c_int64,
                                          ctypes.c_double, ctypes.c_int32, _P]),
        }
        for k, (r, a) in sig.items():
            f = getattr(L, k)
            f.restype = r
            f.argtypes = a
        _lib = L
    return _lib


def _p(a):
    return ctypes.c_void_p(a.ctypes.data)


def gaussian(seed, n):
    out = np.empty(n, np.float32)
    lib().tdo_gaussian(seed, n, _p(out))
    return out


def gen_code(seed, packet_bits=8192):
    out = np.empty(packet_bits, np.uint8)
    lib().tdo_gen_code(seed, packet_bits, _p(out))
    return out


def synth_replica(bits, cfg, padded_len):
    bits = np.ascontiguousarray(bits, np.uint8)
    out = np.empty(2 * padded_len, np.float32)
    lib().tdo_synth_replica(_p(bits), bits.size, ctypes.byref(cfg.mod), padded_len, _p(out))
    return out.view(np.complex64)


def pad_length(n):
    return int(lib().tdo_pad_length(n))


def demodulate_window(iq, start, cfg):
    iq = np.ascontiguousarray(iq, np.int16)
    n = iq.size // 2
    d = np.empty(n, np.float32)
    u = np.empty(n, np.float32)
    lib().tdo_demodulate_window(_p(iq), n, start, ctypes.byref(cfg), _p(d), _p(u))
    return d, u


def demodulate_signal(x, start, lo, cfg):
    x = np.ascontiguousarray(x, np.complex64)
    d = np.empty(x.size, np.float32)
    u = np.empty(x.size, np.float32)
    lib().tdo_demodulate_signal(_p(x), x.size, start, lo, ctypes.byref(cfg), _p(d), _p(u))
    return d, u


class Code:
    def __init__(self, replica_d, nonzero_len, energy, abs_sum, spectrum, corr_len):
        self.replica_d = replica_d
        self.nonzero_len = nonzero_len
        self.energy = energy
        self.abs_sum = abs_sum
        self.spectrum = spectrum
        self.corr_len = corr_len


def make_transformed(replica_d, replica_u, window_len, corr_len):
    d = np.ascontiguousarray(replica_d, np.float32)
    u = None if replica_u is None else np.ascontiguousarray(replica_u, np.float32)
    n = _U64()
    e = ctypes.c_float()
    a = ctypes.c_float()
    spec = np.empty(corr_len, np.complex64)
    rc = lib().tdo_make_transformed(_p(d), _p(u) if u is not None else None, d.size, window_len, corr_len,
                                    ctypes.byref(n), ctypes.byref(e), ctypes.byref(a), _p(spec))
    if rc:
        raise ValueError("make_transformed: transform too short for linear correlation")
    return Code(d[:n.value].copy(), n.value, e.value, a.value, spec, corr_len)


def prepare_code(bits, cfg, window_len):
    bits = np.ascontiguousarray(bits, np.uint8)
    n = _U64()
    e = ctypes.c_float()
    a = ctypes.c_float()
    cl = _U64()
    spb = int(round(cfg.mod.sample_rate / cfg.mod.bit_rate))
    corr = pad_length(window_len + int(cfg.mod.packet_bits) * spb + int(cfg.bandpass_taps) + spb - 1)
    rd = np.empty(window_len, np.float32)
    spec = np.empty(corr, np.complex64)
    rc = lib().tdo_prepare_code(_p(bits), ctypes.byref(cfg), window_len, ctypes.byref(n), ctypes.byref(e),
                                ctypes.byref(a), _p(rd), _p(spec), ctypes.byref(cl))
    if rc:
        raise ValueError("prepare_code: window shorter than a packet")
    return Code(rd[:n.value].copy(), n.value, e.value, a.value, spec, cl.value)


def batch_xcorr(d, codes):
    d = np.ascontiguousarray(d, np.float32)
    N = codes[0].corr_len
    spectra = np.ascontiguousarray(np.stack([c.spectrum for c in codes]))
    nz = np.array([c.nonzero_len for c in codes], np.uint64)
    out = np.empty((len(codes), d.size), np.float32)
    if lib().tdo_batch_xcorr(_p(d), d.size, _p(spectra), _p(nz), len(codes), N, _p(out)):
        raise ValueError("batch_xcorr: window does not fit transform size")
    return out


def find_peak(xc):
    xc = np.ascontiguousarray(xc, np.float32)
    j = _U64()
    v = ctypes.c_float()
    if lib().tdo_find_peak(_p(xc), xc.size, ctypes.byref(j), ctypes.byref(v)):
        raise ValueError("find_peak: empty input")
    return j.value, v.value


def interpolate_peak(xc, j):
    xc = np.ascontiguousarray(xc, np.float32)
    return float(lib().tdo_interpolate_peak(_p(xc), xc.size, j))


def detect(d, u, codes, threshold, window_start, sample_rate, bin_index=0):
    d = np.ascontiguousarray(d, np.float32)
    u = np.ascontiguousarray(u, np.float32)
    N = codes[0].corr_len
    spectra = np.ascontiguousarray(np.stack([c.spectrum for c in codes]))
    reps = (ctypes.c_void_p * len(codes))(*[c.replica_d.ctypes.data for c in codes])
    nz = np.array([c.nonzero_len for c in codes], np.uint64)
    en = np.array([c.energy for c in codes], np.float32)
    out = np.zeros(len(codes), DETECTION_DTYPE)
    rc = lib().tdo_detect(_p(d), _p(u), d.size, _p(spectra), ctypes.cast(reps, _P), _p(nz), _p(en), len(codes), N,
                          threshold, window_start, sample_rate, bin_index, _p(out))
    if rc:
        raise ValueError("batch_xcorr: window does not fit transform size")
    return out
