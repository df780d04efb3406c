// Pipe throughput probes for the soft kernels: FFMA (3-reg), FFMA2 (packed
// f32x2), MUFU.RCP, and FFMA2 + RCP mixes.  Rates in lane-ops/s and per
// SM-clock.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ float rcp(float x) { float r; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }

__global__ void k_ffma(float* o, float a, float b, int n) {
  float c[8];
  for (int i = 0; i < 8; ++i) c[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(c[i]) : "f"(a), "f"(b));
  float s = 0; for (int i = 0; i < 8; ++i) s += c[i];
  if (s == 1.2345f) o[0] = s;
}
__global__ void k_ffma2(float* o, float a, float b, int n) {
  unsigned long long c[8];
  unsigned long long A, B;
  float2 fa = make_float2(a, a), fb = make_float2(b, b);
  A = *reinterpret_cast<unsigned long long*>(&fa); B = *reinterpret_cast<unsigned long long*>(&fb);
  for (int i = 0; i < 8; ++i) { float2 t = make_float2(threadIdx.x * 1e-3f + i, i); c[i] = *reinterpret_cast<unsigned long long*>(&t); }
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = ffma2(c[i], A, B);
  float s = 0; for (int i = 0; i < 8; ++i) { float2 t = *reinterpret_cast<float2*>(&c[i]); s += t.x + t.y; }
  if (s == 1.2345f) o[0] = s;
}
__global__ void k_rcp(float* o, float a, float b, int n) {
  float c[8];
  for (int i = 0; i < 8; ++i) c[i] = threadIdx.x * 1e-3f + i + 1.f;
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = rcp(c[i] + a);
  float s = 0; for (int i = 0; i < 8; ++i) s += c[i];
  if (s == 1.2345f) o[0] = s;
}
// 1 RCP + 2 FFMA2 (4 lane-FMAs) per "pair"
__global__ void k_mix(float* o, float a, float b, int n) {
  float c[8];
  unsigned long long d[4];
  unsigned long long A, B;
  float2 fa = make_float2(a, a), fb = make_float2(b, b);
  A = *reinterpret_cast<unsigned long long*>(&fa); B = *reinterpret_cast<unsigned long long*>(&fb);
  for (int i = 0; i < 8; ++i) c[i] = threadIdx.x * 1e-3f + i + 1.f;
  for (int i = 0; i < 4; ++i) { float2 t = make_float2(i, i); d[i] = *reinterpret_cast<unsigned long long*>(&t); }
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = rcp(c[i]);
#pragma unroll
    for (int i = 0; i < 4; ++i) { d[i] = ffma2(d[i], A, B); d[i] = ffma2(d[i], A, B); d[i] = ffma2(d[i], A, B); d[i] = ffma2(d[i], A, B); }
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += c[i];
  for (int i = 0; i < 4; ++i) { float2 t = *reinterpret_cast<float2*>(&d[i]); s += t.x + t.y; }
  if (s == 1.2345f) o[0] = s;
}


__global__ void k_lop3(float* o, float a, float b, int n) {
  unsigned c[8];
  unsigned m = __float_as_uint(a), q = __float_as_uint(b);
  for (int i = 0; i < 8; ++i) c[i] = threadIdx.x * 7 + i;
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(c[i]) : "r"(m), "r"(q));
  unsigned s = 0; for (int i = 0; i < 8; ++i) s += c[i];
  if (s == 12345u) o[0] = 1.f;
}
__global__ void k_prmt(float* o, float a, float b, int n) {
  unsigned c[8];
  unsigned m = __float_as_uint(a);
  for (int i = 0; i < 8; ++i) c[i] = threadIdx.x * 7 + i;
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("prmt.b32 %0, %0, %1, 0x1234;" : "+r"(c[i]) : "r"(m));
  unsigned s = 0; for (int i = 0; i < 8; ++i) s += c[i];
  if (s == 12345u) o[0] = 1.f;
}
__global__ void k_iadd(float* o, float a, float b, int n) {
  unsigned c[8];
  unsigned m = __float_as_uint(a);
  for (int i = 0; i < 8; ++i) c[i] = threadIdx.x * 7 + i;
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("sub.u32 %0, %1, %0;" : "+r"(c[i]) : "r"(m));
  unsigned s = 0; for (int i = 0; i < 8; ++i) s += c[i];
  if (s == 12345u) o[0] = 1.f;
}
__global__ void k_mix_alu_fma(float* o, float a, float b, int n) {
  unsigned c[8];
  unsigned m = __float_as_uint(a), q = __float_as_uint(b);
  for (int i = 0; i < 8; ++i) c[i] = threadIdx.x * 7 + i;
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(c[i]) : "r"(m), "r"(q));
      asm volatile("sub.u32 %0, %1, %0;" : "+r"(c[i + 4]) : "r"(m));
    }
  unsigned s = 0; for (int i = 0; i < 8; ++i) s += c[i];
  if (s == 12345u) o[0] = 1.f;
}

__global__ void k_imad(float* o, float a, float b, int n) {
  unsigned c[8];
  unsigned m = __float_as_uint(a), q = __float_as_uint(b);
  for (int i = 0; i < 8; ++i) c[i] = threadIdx.x * 7 + i;
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(c[i]) : "r"(m), "r"(q));
  unsigned s = 0; for (int i = 0; i < 8; ++i) s += c[i];
  if (s == 12345u) o[0] = 1.f;
}
__global__ void k_imadhi(float* o, float a, float b, int n) {
  unsigned c[8];
  unsigned m = __float_as_uint(a), q = __float_as_uint(b);
  for (int i = 0; i < 8; ++i) c[i] = threadIdx.x * 7 + i;
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(c[i]) : "r"(m), "r"(q));
  unsigned s = 0; for (int i = 0; i < 8; ++i) s += c[i];
  if (s == 12345u) o[0] = 1.f;
}
// 4 lop3 + 4 imad per iteration (8 ops)
__global__ void k_lop3_imad(float* o, float a, float b, int n) {
  unsigned c[8];
  unsigned m = __float_as_uint(a), q = __float_as_uint(b);
  for (int i = 0; i < 8; ++i) c[i] = threadIdx.x * 7 + i;
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(c[i]) : "r"(m), "r"(q));
      asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(c[i + 4]) : "r"(m), "r"(q));
    }
  unsigned s = 0; for (int i = 0; i < 8; ++i) s += c[i];
  if (s == 12345u) o[0] = 1.f;
}
// 4 lop3 + 4 ffma per iteration (8 ops)
__global__ void k_lop3_ffma(float* o, float a, float b, int n) {
  unsigned c[4];
  float f[4];
  unsigned m = __float_as_uint(a), q = __float_as_uint(b);
  for (int i = 0; i < 4; ++i) { c[i] = threadIdx.x * 7 + i; f[i] = threadIdx.x * 1e-3f + i; }
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(c[i]) : "r"(m), "r"(q));
      asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[i]) : "f"(a), "f"(b));
    }
  unsigned s = 0; for (int i = 0; i < 4; ++i) s += c[i] + __float_as_uint(f[i]);
  if (s == 12345u) o[0] = 1.f;
}
// 2 lop3 + 1 prmt + 1 imad (the compare mix)
__global__ void k_cmpmix(float* o, float a, float b, int n) {
  unsigned c[8];
  unsigned m = __float_as_uint(a), q = __float_as_uint(b);
  for (int i = 0; i < 8; ++i) c[i] = threadIdx.x * 7 + i;
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(c[i]) : "r"(m), "r"(q));
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(c[i + 2]) : "r"(m), "r"(q));
      asm volatile("prmt.b32 %0, %0, %1, 0x1234;" : "+r"(c[i + 4]) : "r"(m));
      asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(c[i + 6]) : "r"(m), "r"(q));
    }
  unsigned s = 0; for (int i = 0; i < 8; ++i) s += c[i];
  if (s == 12345u) o[0] = 1.f;
}

template <typename K>
int run(const char* name, K kern, double ops_per_iter_thread) {
  float* o; CK(cudaMalloc(&o, 4));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int blocks = sms * 8, threads = 256, n = 4096;
  kern<<<blocks, threads>>>(o, 1.0001f, 0.5f, 16);
  cudaEvent_t s, ev; cudaEventCreate(&s); cudaEventCreate(&ev);
  cudaEventRecord(s);
  kern<<<blocks, threads>>>(o, 1.0001f, 0.5f, n);
  CK(cudaGetLastError());
  cudaEventRecord(ev); CK(cudaEventSynchronize(ev));
  float ms; cudaEventElapsedTime(&ms, s, ev);
  double ops = (double)blocks * threads * n * ops_per_iter_thread;
  printf("%-8s %8.3f ms  %.3e lane-ops/s  %.1f per SM-clk (at %d MHz nominal)\n", name, ms, ops / (ms * 1e-3),
         ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  return 0;
}
int main() {
  run("ffma", k_ffma, 8);
  run("ffma2", k_ffma2, 16);    // lane-FMAs
  run("rcp", k_rcp, 8);
  run("rcp+fadd", k_rcp, 8);
  run("mix", k_mix, 8);         // pairs (8 rcp + 32 lane-fma)
  run("lop3", k_lop3, 8);
  run("prmt", k_prmt, 8);
  run("sub.u32", k_iadd, 8);
  run("lop3+sub", k_mix_alu_fma, 8);   // 4 lop3 + 4 sub per iteration
  run("imad", k_imad, 8);
  run("imad.hi", k_imadhi, 8);
  run("lop3+imad", k_lop3_imad, 8);
  run("lop3+ffma", k_lop3_ffma, 8);
  run("cmpmix", k_cmpmix, 8);          // 4 lop3 + 2 prmt + 2 imad
  return 0;
}
