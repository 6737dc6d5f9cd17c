"""Synthetic I/Q scenes for benchmarking (not part of the hot path).

A numpy restatement of the reference's scenario generator
(generate_recording, proj/src/recording.cpp:177-219, with gen_code and
synth_replica from proj/src/codegen.cpp:26-60 and the channel model of
apply_channel :84-124): tag packets injected at known fractional arrival
times, gains and carrier offsets, white Gaussian noise referenced to a
unit-amplitude packet, quantised to int16 (quantize :126-143).

The noise RNG is numpy's, not the reference's splitmix64 Box-Muller, so
streams are statistically but not bitwise equal to the reference's.  Parity
tests feed identical int16 produced by the compiled reference instead
(oracle/refpy.py); this module only makes bench workloads of the named shape.
"""
import numpy as np

MASK64 = (1 << 64) - 1


def splitmix64(state):
    state = (state + 0x9E3779B97F4A7C15) & MASK64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return state, z ^ (z >> 31)


def gen_code(seed, packet_bits=8192):
    """gen_code (proj/src/codegen.cpp:26-38): bit i = bit (i % 64) of word i//64."""
    bits = np.empty(packet_bits, dtype=np.uint8)
    state = seed & MASK64
    word = 0
    for i in range(packet_bits):
        if i % 64 == 0:
            state, word = splitmix64(state)
        bits[i] = (word >> (i % 64)) & 1
    return bits


def synth_replica(bits, sample_rate=8.0e6, bit_rate=1.0e6, freq_one=250.0e3, freq_zero=-250.0e3):
    """Continuous-phase FSK, unit amplitude (proj/src/codegen.cpp:40-60)."""
    spb = int(round(sample_rate / bit_rate))
    step = np.where(np.repeat(bits, spb) != 0, 2 * np.pi * freq_one / sample_rate,
                    2 * np.pi * freq_zero / sample_rate)
    phase = np.concatenate([[0.0], np.cumsum(step)[:-1]])
    return np.exp(1j * phase)


def fractional_shift(s, frac):
    """Band-limited delay by a linear phase ramp (codegen.cpp:66-80)."""
    n = len(s) + 64
    spec = np.fft.fft(np.concatenate([s, np.zeros(64)]))
    k = np.arange(n)
    kf = np.where(k <= n // 2, k, k - n)
    return np.fft.ifft(spec * np.exp(-2j * np.pi * kf * frac / n))


def scene(duration_s, injections, codes_bits, noise_snr_db=10.0, sample_rate=8.0e6, scale=8192.0, seed=1,
          **mod):
    """int16 interleaved I/Q stream of duration_s with packets injected.

    injections: list of (code_index, time_s, gain, freq_offset_hz).
    Returns (iq int16 [2*total], truth list of (code_index, arrival_sample))."""
    total = int(duration_s * sample_rate + 0.5)
    stream = np.zeros(total, dtype=np.complex128)
    truth = []
    for ci, t, gain, foff in injections:
        rep = synth_replica(codes_bits[ci], sample_rate=sample_rate, **mod)
        arrival = t * sample_rate
        base = int(np.floor(arrival))
        frac = arrival - base
        sh = fractional_shift(rep, frac) if frac > 1e-9 else np.concatenate([rep, np.zeros(64)])
        idx = base + np.arange(len(sh))
        ok = (idx >= 0) & (idx < total)
        ph = np.exp(2j * np.pi * foff * np.arange(len(sh)) / sample_rate)
        stream[idx[ok]] += (gain * sh * ph)[ok]
        truth.append((ci, arrival))
    rng = np.random.default_rng(seed)
    if np.isfinite(noise_snr_db):
        sigma = np.sqrt(10.0 ** (-noise_snr_db / 10.0) / 2.0)
        stream += sigma * (rng.standard_normal(total) + 1j * rng.standard_normal(total))
    iq = np.empty(2 * total, dtype=np.int16)
    iq[0::2] = np.clip(np.rint(scale * stream.real), -32768, 32767)
    iq[1::2] = np.clip(np.rint(scale * stream.imag), -32768, 32767)
    return iq, truth


def cfg2_scene(n_codes=64, code_seed0=1000, n_inject=16, duration_s=1.0, seed=7):
    """BASELINE.json configs[1]: codes gen_code(1000+i); n_inject of them at
    known fractional delays, offsets U(-200, 200) kHz and SNRs {0,5,10,20} dB
    (gain relative to the 10 dB noise floor); the rest absent."""
    rng = np.random.default_rng(seed)
    bits = np.stack([gen_code(code_seed0 + i) for i in range(n_codes)])
    inj = []
    snrs = [0.0, 5.0, 10.0, 20.0]
    for k in range(min(n_inject, n_codes)):
        t = rng.uniform(0.0, duration_s - 0.0085)
        g = 10.0 ** ((snrs[k % 4] - 10.0) / 20.0)
        inj.append((k, t, g, rng.uniform(-200e3, 200e3)))
    iq, truth = scene(duration_s, inj, bits, noise_snr_db=10.0, seed=seed)
    return bits, iq, inj, truth
