// Microbenchmarks that size the ECC kernels: smem atomics, MUFU, HBM streaming.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__device__ __forceinline__ uint32_t hash32(uint32_t x){x^=x>>16;x*=0x7feb352dU;x^=x>>15;x*=0x846ca68bU;x^=x>>16;return x;}

// per-warp histograms of NB bins; each thread does ITER atomics at pseudo-random bins
template<int NB, int PERWARP>
__global__ void atoms_kernel(int* out, int iters){
  extern __shared__ int h[];
  int nw = blockDim.x/32, w = threadIdx.x/32;
  int tot = PERWARP ? NB*nw : NB;
  for(int i=threadIdx.x;i<tot;i+=blockDim.x) h[i]=0;
  __syncthreads();
  int* hw = PERWARP ? h + w*NB : h;
  uint32_t s = hash32(blockIdx.x*blockDim.x+threadIdx.x);
  for(int i=0;i<iters;i++){
    s = s*1664525u+1013904223u;
    atomicAdd(&hw[(s>>16)&(NB-1)], (int)(s&3)-1);
  }
  __syncthreads();
  int acc=0; for(int i=threadIdx.x;i<tot;i+=blockDim.x) acc+=h[i];
  if(acc==12345) out[0]=acc;
}
__global__ void lcg_only(int* out, int iters){
  uint32_t s = hash32(blockIdx.x*blockDim.x+threadIdx.x); int acc=0;
  for(int i=0;i<iters;i++){ s = s*1664525u+1013904223u; acc += (s>>16)&1023; }
  if(acc==12345) out[0]=acc;
}
__global__ void mufu_rcp(float* out, int iters){
  float a = threadIdx.x*1e-3f+1.f, b=0.f, c=0.5f+blockIdx.x*1e-6f, d=0.f;
  for(int i=0;i<iters;i++){
    float r1,r2,r3,r4;
    asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(a));
    asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r2) : "f"(c));
    asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r3) : "f"(a+1.f));
    asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r4) : "f"(c+1.f));
    b += r1+r2; d += r3+r4; a += 1e-7f; c += 1e-7f;
  }
  if(b+d==12345.f) out[0]=b;
}
__global__ void stream_read(const float4* __restrict__ x, size_t n4, float* out){
  float acc=0.f;
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n4;i+=(size_t)gridDim.x*blockDim.x){
    float4 v = __ldg(x+i); acc += v.x+v.y+v.z+v.w;
  }
  if(acc==12345.f) out[0]=acc;
}
int main(){
  int* dout; CK(cudaMalloc(&dout, 64));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d clock %d kHz\n", sms, clk);
  float ms;
  int iters=4096;
  for(int threads: {256, 512}) {
    int blocks = sms*(2048/threads);
    double n = (double)blocks*threads*iters;
    lcg_only<<<blocks,threads>>>(dout,iters); cudaEventRecord(e0); lcg_only<<<blocks,threads>>>(dout,iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1); printf("lcg only   thr=%d: %.3f ms, %.1f G/s\n", threads, ms, n/ms/1e6);
    size_t sm1 = 1024*4*(threads/32);
    CK(cudaFuncSetAttribute(atoms_kernel<1024,1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000));
    atoms_kernel<1024,1><<<blocks,threads,sm1>>>(dout,iters); CK(cudaGetLastError());
    cudaEventRecord(e0); atoms_kernel<1024,1><<<blocks,threads,sm1>>>(dout,iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1); printf("atoms perwarp 1024 thr=%d: %.3f ms, %.1f G atom/s, %.3f atom/clk/SM\n", threads, ms, n/ms/1e6, n/ms/1e6/(sms*(clk/1e6)));
    atoms_kernel<1024,0><<<blocks,threads,4096>>>(dout,iters);
    cudaEventRecord(e0); atoms_kernel<1024,0><<<blocks,threads,4096>>>(dout,iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1); printf("atoms perCTA 1024 thr=%d: %.3f ms, %.1f G atom/s, %.3f atom/clk/SM\n", threads, ms, n/ms/1e6, n/ms/1e6/(sms*(clk/1e6)));
    atoms_kernel<256,0><<<blocks,threads,1024>>>(dout,iters);
    cudaEventRecord(e0); atoms_kernel<256,0><<<blocks,threads,1024>>>(dout,iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1); printf("atoms perCTA 256 thr=%d: %.3f ms, %.1f G atom/s, %.3f atom/clk/SM\n", threads, ms, n/ms/1e6, n/ms/1e6/(sms*(clk/1e6)));
  }
  {
    int blocks=sms*8, threads=256; double n=(double)blocks*threads*iters*4;
    mufu_rcp<<<blocks,threads>>>((float*)dout,iters);
    cudaEventRecord(e0); mufu_rcp<<<blocks,threads>>>((float*)dout,iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1); printf("mufu rcp: %.3f ms, %.1f G/s, %.2f /clk/SM\n", ms, n/ms/1e6, n/ms/1e6/(sms*(clk/1e6)));
  }
  {
    size_t bytes = (size_t)4<<30; float4* x; CK(cudaMalloc(&x, bytes)); cudaMemset(x, 0, bytes);
    for (int bpsm : {2,4,8,16}) {
      int blocks = sms*bpsm;
      stream_read<<<blocks,512>>>(x, bytes/16, (float*)dout);
      cudaEventRecord(e0); for(int r=0;r<5;r++) stream_read<<<blocks,512>>>(x, bytes/16, (float*)dout); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms,e0,e1); printf("stream read 4GiB blocks/SM=%d: %.3f ms, %.1f GB/s\n", bpsm, ms/5, bytes/(ms/5)/1e6);
    }
  }
  return 0;
}
