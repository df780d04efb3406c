// ecc_fdcheck.cu -- device finite-difference harness for the soft ECC gradients
// (gradient_check, soft.py:260-359), SURVEY.md 8(f) rank 3.
//
// The reference's loss is separable in the pixels and in the thresholds:
//   L = sum_j up_j sum_p c_p sigma(lam (tau_j - f_p)),
// so the 4th-order central stencil it applies to the whole loss
// (soft.py:308-315) decomposes exactly into per-(pixel, threshold) stencils:
//   d/dX_p   : perturb f_p               (one pixel's terms change)
//   d/dtau_j : perturb tau_j             (one threshold's terms change)
//   d/du_a   : perturb every f_p by alpha pos_a(p) delta
//   d/dalpha : perturb every f_p by <u, pos_p> delta      (not in the reference)
// Everything here is float64 with exp(), independent of the fp32 factorised
// kernels it checks.  One thread per pixel loops over the thresholds; the
// threshold and direction sums are reduced per warp, then per block in
// shared memory, then with one global atomic per block.
#include <stdint.h>

#include "ecc_common.cuh"
#include "ecc_internal.h"

namespace ecc {

struct FdArgs {
  const double* field;     // effective field f_p, float64
  const int8_t* coeffs;    // c_p
  const double* taus;      // [nb]
  const double* up;        // upstream [nb]
  double* fd_values;       // [n]
  double* fd_tau;          // [nb]
  double* fd_dir;          // [ndim] direction components, then [ndim] = alpha
  int64_t n, nb;
  int64_t dims[3];
  int ndim;
  double lam, alpha, h;
  double u[3];
};

__device__ __forceinline__ double sig(double z) { return 1.0 / (1.0 + exp(-z)); }

// (-g(2e) + 8 g(e) - 8 g(-e) + g(-2e)) / 12 for g(e) = sigma(lam (z0 + e)), e in field units
__device__ __forceinline__ double stencil(double z0, double e, double lam) {
  return (-sig(lam * (z0 + 2.0 * e)) + 8.0 * sig(lam * (z0 + e)) - 8.0 * sig(lam * (z0 - e)) +
          sig(lam * (z0 - 2.0 * e))) / 12.0;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void soft_fd_kernel(FdArgs a) {
  extern __shared__ double s_acc[];   // [nb] tau, [4] directions + alpha
  for (int i = threadIdx.x; i < a.nb + 4; i += blockDim.x) s_acc[i] = 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool live = p < a.n && a.coeffs[p < a.n ? p : 0] != 0;
  double f = 0.0, cp = 0.0, pos[3] = {0.0, 0.0, 0.0}, step[4] = {0.0, 0.0, 0.0, 0.0};
  if (live) {
    f = a.field[p];
    cp = (double)a.coeffs[p];
    int64_t r = p;
    for (int k = a.ndim - 1; k >= 0; --k) {
      pos[k] = coord64(r % a.dims[k], a.dims[k]);
      r /= a.dims[k];
    }
    double dot = 0.0;
    for (int k = 0; k < a.ndim; ++k) {
      step[k] = a.alpha * pos[k];          // d f_p / d u_k
      dot += a.u[k] * pos[k];
    }
    step[3] = dot;                         // d f_p / d alpha
  }
  double fdv = 0.0;
  for (int64_t j = 0; j < a.nb; ++j) {     // warp-uniform trip count
    double dv = 0.0, dd[4] = {0.0, 0.0, 0.0, 0.0};
    if (live) {
      const double z0 = a.taus[j] - f;
      // pixel value: f -> f + delta, i.e. z0 -> z0 - delta
      dv = -stencil(z0, a.h, a.lam) / a.h;
      fdv += a.up[j] * cp * dv;
      for (int k = 0; k < 4; ++k)
        if ((k < a.ndim || k == 3) && step[k] != 0.0) dd[k] = -stencil(z0, step[k] * a.h, a.lam) / a.h;
    }
    // tau_j -> tau_j + delta is z0 -> z0 + delta: the negated pixel stencil
    const double t = warp_sum(live ? -a.up[j] * cp * dv : 0.0);
    if (lane == 0 && t != 0.0) atomicAdd(&s_acc[j], t);
    for (int k = 0; k < 4; ++k) {
      const double s = warp_sum(live ? a.up[j] * cp * dd[k] : 0.0);
      if (lane == 0 && s != 0.0) atomicAdd(&s_acc[a.nb + k], s);
    }
  }
  if (p < a.n) a.fd_values[p] = fdv;
  __syncthreads();
  for (int64_t i = threadIdx.x; i < a.nb; i += blockDim.x)
    if (s_acc[i] != 0.0) atomicAdd(&a.fd_tau[i], s_acc[i]);
  if (threadIdx.x < 4 && s_acc[a.nb + threadIdx.x] != 0.0) {
    const int k = threadIdx.x;
    const int slot = k == 3 ? a.ndim : k;
    if (k < a.ndim || k == 3) atomicAdd(&a.fd_dir[slot], s_acc[a.nb + k]);
  }
}

}  // namespace ecc

using namespace ecc;

extern "C" int ecc_soft_fd(const double* field, const int8_t* coeffs, int ndim, const int64_t* dims,
                           const double* taus, int64_t nbins, const double* upstream, double lam, double alpha,
                           const double* u_host, double step, double* fd_values, double* fd_tau, double* fd_dir,
                           void* stream) {
  clear_error();
  if (!field || !coeffs || !dims || !taus || !upstream || !u_host || !fd_values || !fd_tau || !fd_dir)
    return set_error(ECC_EINVAL, "null pointer argument");
  if (ndim != 2 && ndim != 3) return set_error(ECC_EINVAL, "ndim must be 2 or 3");
  if (nbins < 1 || nbins > 65536) return set_error(ECC_EINVAL, "nbins out of range");
  if (!(lam > 0.0) || !(step > 0.0)) return set_error(ECC_EINVAL, "lam and step must be positive");
  FdArgs a;
  a.field = field;
  a.coeffs = coeffs;
  a.taus = taus;
  a.up = upstream;
  a.fd_values = fd_values;
  a.fd_tau = fd_tau;
  a.fd_dir = fd_dir;
  a.ndim = ndim;
  a.n = 1;
  for (int k = 0; k < 3; ++k) {
    a.dims[k] = k < ndim ? dims[k] : 1;
    a.u[k] = k < ndim ? u_host[k] : 0.0;
  }
  for (int k = 0; k < ndim; ++k) {
    if (dims[k] < 1) return set_error(ECC_EINVAL, "extents must be positive");
    a.n *= dims[k];
  }
  a.nb = nbins;
  a.lam = lam;
  a.alpha = alpha;
  a.h = step;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(fd_tau, 0, sizeof(double) * nbins, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(fd_dir, 0, sizeof(double) * (ndim + 1), s);
  if (e != cudaSuccess) return set_cuda_error(e, "cudaMemsetAsync(fd)");
  const int threads = 256;
  const size_t smem = sizeof(double) * (nbins + 4);
  if (smem > 200 * 1024) return set_error(ECC_EINVAL, "too many thresholds for the fd harness");
  if (smem > 48 * 1024) {
    e = cudaFuncSetAttribute(soft_fd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(fd)");
  }
  const int64_t blocks = (a.n + threads - 1) / threads;
  soft_fd_kernel<<<(unsigned)blocks, threads, smem, s>>>(a);
  return check_launch("soft_fd_kernel");
}
