// Shared-memory wavefronts of the pass-A operand access patterns: 27 active
// lanes reading 27 consecutive float2 (monotone, reversed, PFA-mirrored
// (27 - a) % 27) at every start offset b*27 of a 32-row column.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* out, int iters) {
  __shared__ __align__(128) float2 s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = make_float2(i, 1);
  __syncthreads();
  const int a = threadIdx.x & 31;
  const int col = (threadIdx.x >> 5) * 896;
  int idx = MODE == 0 ? a : MODE == 1 ? 26 - a : MODE == 2 ? (a ? 27 - a : 0) : MODE == 3 ? ((a + 1) % 27) : a * 2;
  float acc = 0;
  if (a < 27) {
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int b = 0; b < 32; ++b) { float2 v = s[col + idx + 27 * b]; acc += v.x; }
      idx ^= 0;  // keep the pattern
      acc *= 0.999f;
    }
  }
  if (acc == 0.5f) out[0] = acc;
}
int main() {
  float* out; cudaMalloc(&out, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  void (*ks[])(float*, int) = {k<0>, k<1>, k<2>, k<3>};
  const char* names[] = {"monotone a", "reversed 26-a", "pfa mirror (27-a)%27", "rotated (a+1)%27"};
  for (int m = 0; m < 4; ++m) {
    ks[m]<<<sms * 4, 128>>>(out, 16);
    float ms; int it = 2048;
    cudaEventRecord(e0); ks[m]<<<sms * 4, 128>>>(out, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double lds = (double)sms * 4 * 4 * it * 32;
    printf("%-24s %.3f LDS.64/clk/SM  (%.1f B/clk/SM of 216-B requests)\n", names[m], lds / sms / (ms * 1e-3 * clk * 1e3),
           216.0 * lds / sms / (ms * 1e-3 * clk * 1e3));
  }
}
