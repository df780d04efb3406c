// Which sm_100 pipe runs DP4A / DP2A / FSETP / ISETP / SEL / VIMNMX: each op alone and
// mixed 1:1 with LOP3 (ALU) or IMAD (FMA-heavy).  If a mix issues at about
// the sum of the two rates, the op is on the other pipe.  Lane-ops per SM-clock.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define N_IT 4096
#define OP_LOP3(x) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x) : "r"(m), "r"(q));
#define OP_IMAD(x) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x) : "r"(m), "r"(q));
#define OP_DP4A(x) asm volatile("dp4a.s32.s32 %0, %0, %1, %2;" : "+r"(x) : "r"(m), "r"(q));
#define OP_DP2A(x) asm volatile("dp2a.lo.u32.u32 %0, %0, %1, %2;" : "+r"(x) : "r"(m), "r"(q));
#define OP_FSETP(x) asm volatile("{.reg .pred p; setp.gt.f32 p, %1, %2; selp.u32 %0, 1, 0, p;}" : "=r"(x) : "f"(__uint_as_float(x)), "f"(__uint_as_float(q)));
#define OP_VMIN(x) asm volatile("min.u16x2 %0, %0, %1;" : "+r"(x) : "r"(m));
#define OP_PRMT(x) asm volatile("prmt.b32 %0, %0, %1, 0x6521;" : "+r"(x) : "r"(m));
#define K(name, A, B) \
__global__ void name(unsigned* o, unsigned m, unsigned q, int n) { \
  unsigned c[8], d[8]; \
  for (int i = 0; i < 8; ++i) { c[i] = threadIdx.x * 7 + i; d[i] = threadIdx.x * 5 + i; } \
  for (int it = 0; it < n; ++it) { \
    _Pragma("unroll") for (int i = 0; i < 8; ++i) { A(c[i]) B(d[i]) } \
  } \
  unsigned s = 0; for (int i = 0; i < 8; ++i) s += c[i] + d[i]; \
  if (s == 12345u) o[0] = s; }
#define NOP(x)
K(k_lop3, OP_LOP3, OP_LOP3)
K(k_imad, OP_IMAD, OP_IMAD)
K(k_dp4a, OP_DP4A, OP_DP4A)
K(k_dp2a, OP_DP2A, OP_DP2A)
K(k_prmt, OP_PRMT, OP_PRMT)
K(k_vmin, OP_VMIN, OP_VMIN)
K(k_lop3_imad, OP_LOP3, OP_IMAD)
K(k_lop3_dp4a, OP_LOP3, OP_DP4A)
K(k_lop3_dp2a, OP_LOP3, OP_DP2A)
K(k_imad_dp4a, OP_IMAD, OP_DP4A)
K(k_lop3_prmt, OP_LOP3, OP_PRMT)
K(k_lop3_vmin, OP_LOP3, OP_VMIN)
K(k_imad_vmin, OP_IMAD, OP_VMIN)
int main() {
  unsigned* o; cudaMalloc(&o, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  struct { const char* n; void (*f)(unsigned*, unsigned, unsigned, int); } ks[] = {
    {"lop3", k_lop3}, {"imad", k_imad}, {"dp4a", k_dp4a}, {"dp2a", k_dp2a}, {"prmt", k_prmt}, {"vmin16x2", k_vmin},
    {"lop3+imad", k_lop3_imad}, {"lop3+dp4a", k_lop3_dp4a}, {"lop3+dp2a", k_lop3_dp2a}, {"imad+dp4a", k_imad_dp4a},
    {"lop3+prmt", k_lop3_prmt}, {"lop3+vmin", k_lop3_vmin}, {"imad+vmin", k_imad_vmin}};
  for (auto& k : ks) {
    k.f<<<sms * 8, 256>>>(o, 0x01020304u, 0x00010001u, 16);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k.f<<<sms * 8, 256>>>(o, 0x01020304u, 0x00010001u, N_IT);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = (double)sms * 8 * 256 * N_IT * 16;
    printf("%-12s %8.1f lane-ops/SM-clk (nominal clock %d MHz)\n", k.n, ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  }
  return 0;
}
