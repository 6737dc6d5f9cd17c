// FP32x2 / shared-memory interference microbenchmark: per loop iteration
// NL independent LDS.64 (or STS.64) issued up front, 64 FFMA2 on 8 independent
// chains, then the loaded values folded in with NL/8 FADD2 per 8 loads.
// Reports FP (FFMA2+FADD2) and smem instruction rates per SM per clock.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long f2u(float2 v) { unsigned long long r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(v.x), "f"(v.y)); return r; }
__device__ __forceinline__ float2 u2f(unsigned long long r) { float2 v; asm("mov.b64 {%0,%1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r)); return v; }
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b, unsigned long long c) { unsigned long long d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ unsigned long long add2(unsigned long long a, unsigned long long b) { unsigned long long d; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }

template <int NL, int MODE, int NF>   // MODE 0: LDS.64, 1: STS.64, 2: LDS.128, 3: STG.64, 4: LDG.64 (L2-resident)
__global__ void kmix(float* out, int iters, float2* g) {
  __shared__ __align__(16) float2 s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = make_float2(i, i);
  __syncthreads();
  unsigned long long a[8];
  unsigned long long b = f2u(make_float2(out[1], out[2])), c = f2u(make_float2(out[3], out[4]));
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = f2u(make_float2(threadIdx.x + k, k));
  unsigned long long acc = 0;
  int base = (threadIdx.x & 31) + (threadIdx.x >> 5) * 512;
  for (int i = 0; i < iters; ++i) {
    unsigned long long v[NL > 0 ? NL : 1];
    const int off = (i & 7) * 32;
    if (MODE == 0) {
#pragma unroll
      for (int l = 0; l < NL; ++l) v[l] = f2u(s[(base + off + l * 32 * 0 + (l & 31) * 32 * 1 ) & 4095]);
    } else if (MODE == 3) {
      float2* gp = g + (size_t(blockIdx.x) * blockDim.x + threadIdx.x);
#pragma unroll
      for (int l = 0; l < NL; ++l) gp[size_t((i * NL + l) & 63) * gridDim.x * blockDim.x] = u2f(a[l & 7]);
    } else if (MODE == 4) {
      const float2* gp = g + (size_t(blockIdx.x) * blockDim.x + threadIdx.x);
#pragma unroll
      for (int l = 0; l < NL; ++l) v[l] = f2u(__ldcg(gp + size_t((i * NL + l) & 63) * gridDim.x * blockDim.x));
    } else if (MODE == 1) {
#pragma unroll
      for (int l = 0; l < NL; ++l) s[(base + off + (l & 31) * 32) & 4095] = u2f(a[l & 7]);
    } else {
#pragma unroll
      for (int l = 0; l < NL; l += 2) { float4 q = reinterpret_cast<const float4*>(s)[((base + off + (l & 31) * 32) & 4095) / 2]; v[l] = f2u(make_float2(q.x, q.y)); v[l + 1] = f2u(make_float2(q.z, q.w)); }
    }
#pragma unroll
    for (int r = 0; r < NF / 8; ++r)
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = fma2(a[k], b, c);
    if (MODE != 1 && MODE != 3) {
#pragma unroll
      for (int l = 0; l < NL; ++l) acc = add2(acc, v[l]);
    }
  }
  float sum = 0; for (int k = 0; k < 8; ++k) { float2 v = u2f(a[k]); sum += v.x + v.y; }
  float2 v = u2f(acc); sum += v.x;
  if (sum == 0.123f) out[0] = sum;
}

int main() {
  cudaDeviceProp prop; cudaGetDeviceProperties(&prop, 0);
  int sms = prop.multiProcessorCount, clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float* out; cudaMalloc(&out, 1024); cudaMemset(out, 0, 1024);
  int it = 4096; float ms;
  float2* g; cudaMalloc(&g, size_t(64) * sms * 12 * 32 * 8);
  auto run = [&](const char* name, void (*k)(float*, int, float2*), int nl, int nf, int mode) {
    for (int warps : {4, 8, 12}) {
      int threads = 128, grid = sms * warps / 4;
      k<<<grid, threads>>>(out, 8, g);
      cudaEventRecord(e0); k<<<grid, threads>>>(out, it, g); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      double cyc = ms * 1e-3 * clk * 1e3;
      double wi = (double)grid * threads / 32 * it;   // warp-iterations
      double fp = wi * (nf + ((mode == 1 || mode == 3) ? 0 : nl)) / sms / cyc, sm = wi * (mode == 2 ? nl / 2 : nl) / sms / cyc;
      printf("%-22s warps/SM %2d: FP %.3f  smem-instr %.3f  /clk/SM\n", name, warps, fp, sm);
    }
  };
  run("fp only", kmix<0, 0, 64>, 0, 64, 0);
  run("lds.64 x8 / 64 fma2", kmix<8, 0, 64>, 8, 64, 0);
  run("lds.64 x16 / 64 fma2", kmix<16, 0, 64>, 16, 64, 0);
  run("lds.64 x32 / 64 fma2", kmix<32, 0, 64>, 32, 64, 0);
  run("lds.128 x16 / 64 fma2", kmix<16, 2, 64>, 16, 64, 2);
  run("lds.128 x32 / 64 fma2", kmix<32, 2, 64>, 32, 64, 2);
  run("stg.64 x8 / 64 fma2", kmix<8, 3, 64>, 8, 64, 3);
  run("stg.64 x16 / 64 fma2", kmix<16, 3, 64>, 16, 64, 3);
  run("stg.64 x32 / 64 fma2", kmix<32, 3, 64>, 32, 64, 3);
  run("ldg.64 x16 / 64 fma2", kmix<16, 4, 64>, 16, 64, 4);
  run("ldg.64 x32 / 64 fma2", kmix<32, 4, 64>, 32, 64, 4);
  run("sts.64 x8 / 64 fma2", kmix<8, 1, 64>, 8, 64, 1);
  run("sts.64 x16 / 64 fma2", kmix<16, 1, 64>, 16, 64, 1);
  run("sts.64 x32 / 64 fma2", kmix<32, 1, 64>, 32, 64, 1);
  return 0;
}
