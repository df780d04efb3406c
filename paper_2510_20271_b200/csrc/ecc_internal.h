// ecc_internal.h -- error plumbing shared by the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>
#include "../../include/ecc_b200.h"

namespace ecc {
int set_error(int code, const char* msg);
int set_cuda_error(cudaError_t e, const char* what);
void clear_error();
inline int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_cuda_error(e, what);
  return ECC_OK;
}
// float32 fast path (ecc_fast3d.cu)
bool fast3d_eligible(const void* x, int64_t D, int64_t H, int64_t W, int64_t batch, int64_t nb);
int fast3d_launch(const float* x, int64_t D, int64_t H, int64_t W, int64_t batch, int64_t zb, int64_t ze,
                  const void* table, const ecc_binning* b, unsigned long long* hist, cudaStream_t stream);
// uint8 fast path (ecc_fast3d.cu): the value is the rank
bool fast3d_u8_eligible(const void* x, int64_t D, int64_t H, int64_t W, int64_t batch, int64_t nb);
int fast3d_u8_launch(const uint8_t* x, int64_t D, int64_t H, int64_t W, int64_t batch, int64_t zb, int64_t ze,
                     const void* table, const ecc_binning* b, unsigned long long* hist, cudaStream_t stream);
}  // namespace ecc
