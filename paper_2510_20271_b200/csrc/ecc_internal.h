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
}  // namespace ecc
