"""ctypes mirror of the POD records in include/tagdsp_gpu_types.h.

Shared by the product bindings (capi.py) and the test-side oracle bindings
(oracle/refpy.py) so both produce identical numpy record arrays."""
import ctypes

import numpy as np


class Modulation(ctypes.Structure):
    """tagdsp::ModulationParams (proj/include/tagdsp/types.hpp:24-40)."""
    _fields_ = [("sample_rate", ctypes.c_double), ("bit_rate", ctypes.c_double),
                ("freq_one", ctypes.c_double), ("freq_zero", ctypes.c_double),
                ("packet_bits", ctypes.c_uint64)]


class DemodConfig(ctypes.Structure):
    """tagdsp::DemodConfig (proj/include/tagdsp/dsp.hpp:25-36)."""
    _fields_ = [("mod", Modulation), ("lo_freq", ctypes.c_double),
                ("bandpass_center", ctypes.c_double), ("bandpass_width", ctypes.c_double),
                ("bandpass_taps", ctypes.c_uint64), ("eps", ctypes.c_float),
                ("reserved", ctypes.c_uint32)]


def demod_config(sample_rate=8.0e6, bit_rate=1.0e6, freq_one=250.0e3, freq_zero=-250.0e3,
                 packet_bits=8192, lo_freq=0.0, bandpass_center=0.0, bandpass_width=1.5e6,
                 bandpass_taps=200, eps=1e-12):
    """DemodConfig with the reference defaults (types.hpp:24-30, dsp.hpp:25-36)."""
    return DemodConfig(Modulation(sample_rate, bit_rate, freq_one, freq_zero, packet_bits),
                       lo_freq, bandpass_center, bandpass_width, bandpass_taps, eps, 0)


def desk_config(packet_bits=8192):
    """The reference tests' scaled 'desk' modulation (test_detector.cpp:13-28,
    acceptance.cpp:52-61): 1 Ms/s, 125 kb/s, +-31.25 kHz, 187.5 kHz band."""
    return demod_config(sample_rate=1.0e6, bit_rate=125.0e3, freq_one=31.25e3,
                        freq_zero=-31.25e3, packet_bits=packet_bits, bandpass_width=187.5e3)


DETECTION_DTYPE = np.dtype({
    "names": ["code_index", "bin", "window_start", "peak_index", "toa_seconds",
              "subsample_offset", "peak_value", "w_c", "q", "p_c", "score", "accepted",
              "partial"],
    "formats": [np.int32, np.int32, np.int64, np.uint64, np.float64, np.float32, np.float32,
                np.float32, np.float32, np.float32, np.float32, np.uint8, np.uint8],
    "offsets": [0, 4, 8, 16, 24, 32, 36, 40, 44, 48, 52, 56, 57],
    "itemsize": 64,
})

assert ctypes.sizeof(DemodConfig) == 80


def samples_per_bit(cfg):
    spb = cfg.mod.sample_rate / cfg.mod.bit_rate
    n = int(spb + 0.5)
    if n < 1 or abs(spb - n) > 1e-9:
        raise ValueError("sample_rate / bit_rate must be a positive integer")
    return n


def packet_samples(cfg):
    return int(cfg.mod.packet_bits) * samples_per_bit(cfg)


def composed_filter_len(cfg):
    return int(cfg.bandpass_taps) + samples_per_bit(cfg) - 1


# tdg_track_task (include/tagdsp_gpu_types.h)
TRACK_TASK_DTYPE = np.dtype([("start", np.int64), ("code_index", np.uint64)])

# tdg_ring_push_result (include/tagdsp_gpu_types.h)
class RingPushResult(ctypes.Structure):
    """tagdsp::CircularBuffer::PushResult (proj/include/tagdsp/scheduler.hpp:18-24)."""
    _fields_ = [("evicted_begin", ctypes.c_int64), ("evicted_end", ctypes.c_int64), ("gap", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]
