// FP32 issue-rate probe for bench.py's roofline denominator: the FP32 peak
// the correlation engine is bound by, MEASURED on the running GPU at its
// current clock instead of assumed (MEASURED_PEAKS.json has HBM and bf16
// only).  Two variants: scalar FFMA and packed FFMA2 (fma.rn.f32x2, what the
// FFT codelets use).  Eight independent accumulation chains per thread, 16
// warps per SM, so the fma pipe -- not latency -- is the limit.
#pragma once
#include "codelets.cuh"

namespace tdg {

__global__ void __launch_bounds__(512) k_peak_ffma(float* out, int iters) {
    float a[8];
    const float b = out[1], c = out[2];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = float(threadIdx.x + k);
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int k = 0; k < 8; ++k) a[k] = fmaf(a[k], b, c);
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 0.123f) out[0] = s;
}

__global__ void __launch_bounds__(512) k_peak_ffma2(float* out, int iters) {
    c2 a[8];
    const c2 b = pk(out[1], out[3]), c = pk(out[2], out[4]);
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = pk(float(threadIdx.x + k), float(k));
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int k = 0; k < 8; ++k) a[k] = fma2(a[k], b, c);
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const float2 v = up(a[k]);
        s += v.x + v.y;
    }
    if (s == 0.123f) out[0] = s;
}

}  // namespace tdg
