// FP64 pipe rate on sm_100 (DADD / DFMA / DSETP+SEL), lane-ops per SM-clock.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dadd(double* o, double a, int n) {
  double c[8];
  for (int i = 0; i < 8; ++i) c[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(c[i]) : "d"(a));
  double s = 0; for (int i = 0; i < 8; ++i) s += c[i];
  if (s == 1.2345) o[0] = s;
}
__global__ void k_dfma(double* o, double a, int n) {
  double c[8];
  for (int i = 0; i < 8; ++i) c[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(c[i]) : "d"(a));
  double s = 0; for (int i = 0; i < 8; ++i) s += c[i];
  if (s == 1.2345) o[0] = s;
}
__global__ void k_dsetp(double* o, double a, int n) {
  unsigned acc[8];
  double c[8];
  for (int i = 0; i < 8; ++i) { c[i] = threadIdx.x * 1e-3 + i; acc[i] = 0; }
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      unsigned r;
      asm volatile("{.reg .pred p; setp.le.f64 p, %1, %2; selp.u32 %0, 1, 0, p;}" : "=r"(r) : "d"(c[i]), "d"(a));
      acc[i] += r;
    }
  unsigned s = 0; for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 12345u) o[0] = s;
}
int main() {
  double* o; cudaMalloc(&o, 8);
  int sms, clk; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0); cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  struct { const char* n; void (*f)(double*, double, int); } ks[] = {{"dadd", k_dadd}, {"dfma", k_dfma}, {"dsetp+selp+add", k_dsetp}};
  for (auto& k : ks) {
    k.f<<<sms * 8, 256>>>(o, 1.0000001, 16);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); k.f<<<sms * 8, 256>>>(o, 1.0000001, 2048); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = (double)sms * 8 * 256 * 2048 * 8;
    printf("%-16s %8.1f lane-ops/SM-clk\n", k.n, ops / (ms * 1e-3) / sms / (clk * 1e3));
  }
}
