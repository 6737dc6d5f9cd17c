// Kernels behind the span-level entry points of the reference API that the
// drop-in (include/tagdsp_b200, libtagdsp_b200.so) exposes besides the
// batched path: PlanCache::forward/inverse of any {2,3,5,7}-smooth length
// (proj/src/fft.cpp:46-67), convert (dsp.cpp:9-16), mix (dsp.cpp:18-33), the
// spectral product of overlap_add_filter (dsp.cpp:77-104), demodulate
// (dsp.cpp:147-157) and find_peak (detector.cpp:122-134).  None of these is
// on the batched hot path (tdg_search / tdg_detect fuse them into k_demod and
// the correlation passes); they make every reference function callable on
// the GPU with the reference's argument meaning.
#pragma once
#include "kernels.cuh"

namespace tdg {

// One Stockham autosort stage of radix R over a length-n complex sequence
// (Govindaraju et al.'s formulation): element j < n/R takes in[j + r n/R],
// twiddles by w^{r (j mod ns)} with w = e^{sign 2 pi i / (ns R)}, an R-point
// DFT, and writes out[(j / ns) ns R + (j mod ns) + r ns].  ns is the product
// of the radices of the earlier stages.  Twiddles in double (sincospi).
template <int R, int SIGN>
__global__ void k_stockham(const float2* __restrict__ in, float2* __restrict__ out, uint32_t n, uint32_t ns,
                           float scale) {
    const uint32_t m = n / R;
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x) {
        const uint32_t k = j % ns;
        float2 v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = in[j + uint32_t(r) * m];
        if (ns > 1) {
#pragma unroll
            for (int r = 1; r < R; ++r) {
                double s, c;
                sincospi(double(SIGN) * 2.0 * double(uint64_t(r) * k) / double(uint64_t(ns) * R), &s, &c);
                v[r] = cmul(v[r], make_float2(float(c), float(s)));
            }
        }
        dft<R, SIGN>(v);
        const uint32_t base = (j / ns) * ns * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) out[base + uint32_t(r) * ns] = make_float2(v[r].x * scale, v[r].y * scale);
    }
}

// convert (dsp.cpp:9-16): interleaved int16 I,Q -> complex float
__global__ void k_convert(const short2* __restrict__ in, float2* __restrict__ out, uint64_t n) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const short2 s = in[i];
        out[i] = make_float2(float(s.x), float(s.y));
    }
}

// mix (dsp.cpp:18-33): x[i] *= exp(-2 pi i lo (start + i) / fs), the phase
// of every sample from the absolute index in double (the reference's
// renormalised rotator reaches the same values to ~1e-7)
__global__ void k_mix(float2* __restrict__ x, uint64_t n, double cyc_per_sample, int64_t start) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        double t = cyc_per_sample * double(start + int64_t(i));
        t -= floor(t);
        double s, c;
        sincospi(-2.0 * t, &s, &c);
        x[i] = cmul(x[i], make_float2(float(c), float(s)));
    }
}

// pointwise complex product a[k] *= b[k] (overlap_add_filter's spectral product)
__global__ void k_cmul_inplace(float2* __restrict__ a, const float2* __restrict__ b, uint64_t n) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        a[i] = cmul(a[i], b[i]);
}

// demodulate (dsp.cpp:147-157): u = |f1| - |f0|, d = u / max(|f1| + |f0|, eps)
__global__ void k_discriminate(const float2* __restrict__ f1, const float2* __restrict__ f0, uint64_t n, float eps,
                               float* __restrict__ d, float* __restrict__ u) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const float2 a = f1[i], b = f0[i];
        const float m1 = hypotf(a.x, a.y), m0 = hypotf(b.x, b.y);
        const float uu = m1 - m0;
        u[i] = uu;
        d[i] = uu / fmaxf(m1 + m0, eps);
    }
}

// find_peak (detector.cpp:122-134): first index of the largest |xc| via the
// packed (magnitude, ~index) key of the correlation passes
__global__ void k_argmax_abs(const float* __restrict__ x, uint64_t n, unsigned long long* __restrict__ key) {
    unsigned long long best = 0ull;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const unsigned long long k = peak_key(fabsf(x[i]), uint32_t(i));
        best = k > best ? k : best;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(0xffffffffu, best, o);
        best = y > best ? y : best;
    }
    if ((threadIdx.x & 31) == 0 && best) atomicMax(key, best);
}

}  // namespace tdg
