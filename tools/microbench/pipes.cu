// Pipe-rate microbenchmark for the correlation engine's design: packed FP32
// (fma/mul/add .f32x2 -> FFMA2/FMUL2/FADD2) vs scalar issue rates per SM and
// how LDS.64 traffic interleaves with them.  Build: nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 -o tools/microbench/pipes tools/microbench/pipes.cu
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1;}}while(0)

__device__ __forceinline__ unsigned long long f2u(float2 v) {
  unsigned long long r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(v.x), "f"(v.y)); return r; }
__device__ __forceinline__ float2 u2f(unsigned long long r) {
  float2 v; asm("mov.b64 {%0,%1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r)); return v; }
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ unsigned long long add2(unsigned long long a, unsigned long long b) {
  unsigned long long d; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ unsigned long long mul2(unsigned long long a, unsigned long long b) {
  unsigned long long d; asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }

// ILP chains: K independent accumulators per thread
template <int K, int OP>
__global__ void kpk(float* out, int iters) {
  unsigned long long a[K];
  unsigned long long b = f2u(make_float2(out[1], out[2])), c = f2u(make_float2(out[3], out[4]));
#pragma unroll
  for (int k = 0; k < K; ++k) a[k] = f2u(make_float2(threadIdx.x + k, k));
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int k = 0; k < K; ++k) a[k] = OP == 0 ? fma2(a[k], b, c) : OP == 1 ? add2(a[k], b) : mul2(a[k], b);
  }
  float s = 0; for (int k = 0; k < K; ++k) { float2 v = u2f(a[k]); s += v.x + v.y; }
  if (s == 0.123f) out[0] = s;
}
template <int K>
__global__ void kscalar(float* out, int iters) {
  float a[K]; float b = out[1], c = out[2];
#pragma unroll
  for (int k = 0; k < K; ++k) a[k] = threadIdx.x + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int k = 0; k < K; ++k) a[k] = fmaf(a[k], b, c);
  }
  float s = 0; for (int k = 0; k < K; ++k) s += a[k];
  if (s == 0.123f) out[0] = s;
}
// FFMA2 chains mixed with LDS.64 (one LDS per NF packed FMAs)
template <int K, int NF>
__global__ void kmix(float* out, int iters) {
  __shared__ float2 s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = make_float2(i, i);
  __syncthreads();
  unsigned long long a[K];
  unsigned long long b = f2u(make_float2(out[1], out[2])), c = f2u(make_float2(out[3], out[4]));
#pragma unroll
  for (int k = 0; k < K; ++k) a[k] = f2u(make_float2(threadIdx.x + k, k));
  int idx = threadIdx.x;
  unsigned long long acc = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        a[k] = fma2(a[k], b, c);
        if ((r * K + k) % NF == 0) { float2 v = s[(idx + (r * K + k) * 32) & 4095]; acc = add2(acc, f2u(v)); }
      }
    }
    idx += 37;
  }
  float sum = 0; for (int k = 0; k < K; ++k) { float2 v = u2f(a[k]); sum += v.x + v.y; }
  float2 v = u2f(acc); sum += v.x;
  if (sum == 0.123f) out[0] = sum;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("dev %s SMs %d clock %d MHz\n", prop.name, sms, clk / 1000);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float* out; CK(cudaMalloc(&out, 1024)); CK(cudaMemset(out, 0, 1024));
  float ms; int it = 2048;
  auto run = [&](const char* name, void (*k)(float*, int), int threads, double instr_per_thread_iter) {
    for (int blocksPerSM : {1, 2, 4}) {
      int grid = sms * blocksPerSM;
      k<<<grid, threads>>>(out, 8);
      cudaEventRecord(e0); k<<<grid, threads>>>(out, it); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      double warp_instr = (double)grid * threads / 32 * it * instr_per_thread_iter;
      double per_sm_clk = warp_instr / sms / (ms * 1e-3 * clk * 1e3);
      printf("%-28s thr %4d x %d/SM: %.3f warp-instr/clk/SM (%.2f ms)\n", name, threads, blocksPerSM, per_sm_clk, ms);
    }
  };
  run("fma2 K=8", kpk<8, 0>, 128, 64);
  run("fma2 K=8", kpk<8, 0>, 256, 64);
  run("fma2 K=8", kpk<8, 0>, 512, 64);
  run("fma2 K=4", kpk<4, 0>, 512, 32);
  run("add2 K=8", kpk<8, 1>, 512, 64);
  run("mul2 K=8", kpk<8, 2>, 512, 64);
  run("ffma K=8", kscalar<8>, 512, 64);
  run("ffma K=8", kscalar<8>, 128, 64);
  run("mix fma2:lds 8:1 (fma2 cnt)", kmix<8, 8>, 256, 64);
  run("mix fma2:lds 4:1 (fma2 cnt)", kmix<8, 4>, 256, 64);
  run("mix fma2:lds 2:1 (fma2 cnt)", kmix<8, 2>, 256, 64);
  return 0;
}
