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
// nf: optional device flag set to 1 when a non-finite value is read; *nf_done
// tells whether the kernel chosen checked (else the caller runs a check pass)
int fast3d_launch(const float* x, int64_t D, int64_t H, int64_t W, int64_t batch, int64_t zb, int64_t ze,
                  const void* table, const ecc_binning* b, unsigned long long* hist, cudaStream_t stream,
                  int* nf, bool* nf_done);
// uint8 fast path (ecc_fast3d.cu): the value is the rank
bool fast3d_u8_eligible(const void* x, int64_t D, int64_t H, int64_t W, int64_t batch, int64_t nb);
int fast3d_u8_launch(const uint8_t* x, int64_t D, int64_t H, int64_t W, int64_t batch, int64_t zb, int64_t ze,
                     const void* table, const ecc_binning* b, unsigned long long* hist, cudaStream_t stream);
// Kernel-variant switches for A/B checks (tests, tools/).  Set through the C
// ABI (ecc_set_variant); read as relaxed atomics by the launchers -- no
// getenv on the launch path.  Defaults select the production kernels.
enum F3Mode { F3_DEFAULT = 0, F3_VALUE = 1, F3_BRANCH = 2, F3_CTA = 3, F3_RANK2 = 4, F3_NO2D = 5, F3_EDGE1 = 6,
              F3_DUMMY = 8, F3_STATIC = 9 };
int variant_f3();          // F3Mode
int variant_zunit();       // forced dynamic unit (planes), 0: automatic
bool variant_generic();    // route everything through the generic sweep
int variant_soft_t(bool bwd);   // thresholds per lane of the soft kernels (8 / 16 / 32)
bool variant_soft_band();       // windowed (band-sorted) soft kernels when the thresholds allow
int variant_soft_g();           // chunks per soft CTA, 0: automatic
bool variant_soft_prep_old();   // 3-D soft prepare: the per-voxel tile kernel instead of the row-word one
}  // namespace ecc
