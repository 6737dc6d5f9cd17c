// Microbenchmarks to ground the FFT-correlation design on B200:
// L2-resident read/write bandwidth, HBM bandwidth, FP32 issue rates, smem bandwidth.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1;}}while(0)

__global__ void rd(const float4* __restrict__ p, size_t n, int reps, float* out) {
  float4 acc = make_float4(0,0,0,0);
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      float4 v = __ldcg(p + i); acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w; }
  if (acc.x + acc.y + acc.z + acc.w == 1234.5f) out[0] = acc.x;
}
__global__ void cp(const float4* __restrict__ a, float4* __restrict__ b, size_t n, int reps) {
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
      __stcg(b + i, __ldcg(a + i));
}
__global__ void ffma(float* out, int iters) {
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0+4, a5=a0+5, a6=a0+6, a7=a0+7;
  float b = out[1], c = out[2];
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) { a0 = fmaf(a0, b, c); a1 = fmaf(a1, b, c); a2 = fmaf(a2, b, c); a3 = fmaf(a3, b, c);
      a4 = fmaf(a4, b, c); a5 = fmaf(a5, b, c); a6 = fmaf(a6, b, c); a7 = fmaf(a7, b, c); }
  }
  if (a0+a1+a2+a3+a4+a5+a6+a7 == 0.123f) out[0] = a0;
}
__global__ void fadd(float* out, int iters) {
  float a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0+4, a5=a0+5, a6=a0+6, a7=a0+7;
  float b = out[1];
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) { a0 += b; a1 -= b; a2 += b; a3 -= b; a4 += b; a5 -= b; a6 += b; a7 -= b;
      b = b * 1.0000001f; }
  }
  if (a0+a1+a2+a3+a4+a5+a6+a7 == 0.123f) out[0] = a0;
}
__global__ void fadd3(float* out, int iters) {   // adds with two distinct register sources
  float a[8], c[8];
  for (int k = 0; k < 8; ++k) { a[k] = threadIdx.x + k; c[k] = out[k+1]; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) { a[k] = a[k] + c[(k+1)&7]; c[k] = c[k] - a[(k+3)&7]; }
  }
  float s = 0; for (int k = 0; k < 8; ++k) s += a[k] + c[k];
  if (s == 0.123f) out[0] = s;
}
__global__ void smem(float* out, int iters) {
  __shared__ float2 s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = make_float2(i, i);
  __syncthreads();
  float2 acc = make_float2(0,0);
  int idx = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) { float2 v = s[(idx + k * 256) & 4095]; acc.x += v.x; acc.y += v.y; }
    idx += 33;
  }
  if (acc.x + acc.y == 0.5f) out[0] = acc.x;
}
int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  printf("dev %s SMs %d smemPerBlockOptin %zu L2 %d clock %d memclk %d busw %d\n", prop.name, prop.multiProcessorCount,
         prop.sharedMemPerBlockOptin, prop.l2CacheSize, prop.clockRate, prop.memoryClockRate, prop.memoryBusWidth);
  int sms = prop.multiProcessorCount;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float* out; CK(cudaMalloc(&out, 1024)); CK(cudaMemset(out, 0, 1024));
  size_t big = (size_t)2 << 30;
  float4 *a, *b; CK(cudaMalloc(&a, big)); CK(cudaMalloc(&b, big)); CK(cudaMemset(a, 0, big)); CK(cudaMemset(b, 0, big));
  float ms;
  for (size_t mb : {8, 16, 32, 48, 64, 96, 2048}) {
    size_t n = mb * (1 << 20) / 16; int reps = mb >= 1024 ? 3 : 200;
    rd<<<sms * 8, 512>>>(a, n, 1, out);
    cudaEventRecord(e0); rd<<<sms * 8, 512>>>(a, n, reps, out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("read  %5zu MB: %8.1f GB/s\n", mb, (double)n * 16 * reps / ms / 1e6);
    cp<<<sms * 8, 512>>>(a, b, n / 2, 1);
    cudaEventRecord(e0); cp<<<sms * 8, 512>>>(a, b, n / 2, reps); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("copy  %5zu MB (r+w): %8.1f GB/s\n", mb, (double)n * 16 * reps / ms / 1e6);
  }
  int it = 4096;
  ffma<<<sms * 4, 512>>>(out, 16);
  cudaEventRecord(e0); ffma<<<sms * 4, 512>>>(out, it); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1);
  double fl = (double)sms * 4 * 512 * it * 64;
  printf("ffma: %.1f TFLOP/s (fma=2)  %.1f Tinstr/s\n", 2 * fl / ms / 1e9, fl / ms / 1e9);
  cudaEventRecord(e0); fadd<<<sms * 4, 512>>>(out, it); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1);
  fl = (double)sms * 4 * 512 * it * 72;
  printf("fadd(+fmul): %.1f Tinstr/s\n", fl / ms / 1e9);
  cudaEventRecord(e0); fadd3<<<sms * 4, 512>>>(out, it); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1);
  fl = (double)sms * 4 * 512 * it * 16;
  printf("fadd 2-reg: %.1f Tinstr/s\n", fl / ms / 1e9);
  cudaEventRecord(e0); smem<<<sms * 4, 512>>>(out, it); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1);
  double by = (double)sms * 4 * 512 * it * 8 * 8;
  printf("smem LDS.64: %.1f TB/s  (%.1f B/clk/SM at %d MHz)\n", by / ms / 1e9, by / ms / 1e3 / sms / (prop.clockRate / 1e3) / 1e3 * 1e3 / 1e3, prop.clockRate/1000);
  return 0;
}
