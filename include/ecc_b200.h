/*
 * ecc_b200.h -- C ABI of the B200 Euler Characteristic Curve engine
 * (libecc_b200.so, built from paper_2510_20271_b200/csrc/).
 *
 * The reference (ecckit 0.1.0, /root/reference/pkg/src/ecckit) is pure
 * Python and has no FFI; its hot path sits behind the Python functions
 * re-exported by ecckit/__init__.py:11-117.  Each entry point below replaces
 * the numpy kernel of one of those functions; the Python shim in
 * paper_2510_20271_b200/ keeps the reference's names, argument meaning and
 * exceptions and calls these through ctypes (INTEGRATION.md shows the
 * binding).
 *
 * Conventions
 *   - every array argument is a caller-owned DEVICE pointer unless the name
 *     ends in _host; nothing is allocated inside a launcher;
 *   - `stream` is a cudaStream_t (NULL = legacy default stream); launches are
 *     asynchronous on it;
 *   - grids are row-major, last axis fastest (grid.py:5-9); `dims` is a HOST
 *     array of `ndim` (2 or 3) extents; `batch` grids of that shape are
 *     stored back to back;
 *   - return 0 on success, a negative errno-style code on failure, with a
 *     thread-local message in ecc_last_error().
 */
#ifndef ECC_B200_H
#define ECC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ECC_OK 0
#define ECC_EINVAL (-22)   /* the reference raises ValueError here */
#define ECC_ECUDA (-5)     /* CUDA runtime / launch failure */

#define ECC_DTYPE_U8 0
#define ECC_DTYPE_F32 1
#define ECC_DTYPE_F64 2

#define ECC_MAX_BINS (1 << 20)

/* Binning parameters produced by ecc_threshold_table(). */
typedef struct {
  double t0;      /* first threshold, in the compare type's precision       */
  double inv_w;   /* (nbins-1)/(t_last-t0) or 0                              */
  int64_t nbins;  /* B                                                       */
  int32_t mode;   /* 0 affine guess + exact correction, 1 binary search      */
  int32_t max_correction; /* largest guess error seen at the breakpoints    */
  /* cell table of the float32 fast path: cell(x) = floor(sat(fma(x,
   * lut_scale, lut_bias)) * lut_cells), lut_cells a power of two; every
   * cell holds at most one threshold, so bin(x) = b[cell] + (x > t[cell])
   * exactly (verified for every float32 when the table is built). */
  float lut_scale;
  float lut_bias;
  int32_t lut_cells;
  int32_t lut_ok;
  /* 1: every threshold lies in the first or last 1/lut_edge_sub of its
   * cell (lut_edge_sub = 1024, else 256), and the table also holds the
   * boundary thresholds tE[cells + 1] and the rank -> bin map
   * rbin[cells + 2] after the cell table; the rank kernel then looks a
   * threshold up only for voxels in those edge sub-cells. */
  int32_t lut_edge;
  int32_t lut_edge_sub;
} ecc_binning;

/* Version string and thread-local description of the last failure. */
const char *ecc_version(void);
const char *ecc_last_error(void);

/* HOST.  Validates a threshold set exactly like ThresholdSet.__init__
 * (grid.py:129-139: non-empty, finite, strictly increasing) and writes the
 * device compare table into table_host (nbins+2 entries of float32 for
 * ECC_DTYPE_U8/F32 -- t32_j = the largest float32 <= tau_j -- or float64 for
 * ECC_DTYPE_F64, with -inf/+inf sentinels), followed for float32/uint8 by
 * the cell table of the fast path (8-byte aligned, lut_cells+1 entries of
 * {float t, int32 b}); size: ecc_threshold_table_bytes().
 * Replaces ThresholdSet._certify_affine / bin_indices (grid.py:147-180). */
int ecc_threshold_table(const double *taus_host, int64_t nbins, int dtype, void *table_host,
                        ecc_binning *binning_host);

/* Bytes of the table ecc_threshold_table writes (sentinel table + cell table). */
size_t ecc_threshold_table_bytes(int64_t nbins, int dtype);

/* Fused stencil + coefficient + bin + histogram sweep.
 * hist: int64 [batch][nbins+1], the last entry of each row is the overflow
 * bucket (HistogramBins.bins / .overflow, hard.py:75-86).  Zeroed here.
 * Replaces accumulate_histogram (hard.py:184-212) with FullSweep semantics. */
int ecc_histogram(const void *x, int dtype, int ndim, const int64_t *dims, int64_t batch, const void *table,
                  const ecc_binning *binning_host, int64_t *hist, void *stream);

/* As ecc_histogram, but only voxels in planes [plane_begin, plane_end) of
 * axis 0 are deposited; the planes outside act as halo (coefficients.py:
 * 141-152 _coefficient_rows); they must hold the neighbouring slab's real
 * values (at the volume's ends, pass a view without the halo plane instead).
 * This is the z-slab entry point of the multi-GPU path (one rank = one slab
 * plus a one-plane halo on each interior side).  3D only.
 * The histograms of any partition of the planes sum, bit for bit, to the
 * whole volume's (the all-reduce of the multi-GPU path).  A single range is a
 * partial sum in the kernel's vertex order: the float32 fast path orders
 * voxels by (threshold rank, index) rather than (value, index), so a cell
 * whose two highest vertices share a bin and straddle the range boundary may
 * be counted by the neighbouring range instead. */
int ecc_histogram_range(const void *x, int dtype, int ndim, const int64_t *dims, int64_t batch,
                        int64_t plane_begin, int64_t plane_end, const void *table,
                        const ecc_binning *binning_host, int64_t *hist, void *stream);

/* ecc_histogram_range plus the reference's finiteness rule (ScalarGrid,
 * grid.py:63-64) checked on the device: *nonfinite (device int32) is set to
 * 1 when any value read is NaN or +-Inf, else 0.  The float32 rank kernels
 * check while they sweep (no second pass over the volume); other paths run
 * a check pass.  plane_begin/plane_end as ecc_histogram_range (2D: 0, 1). */
int ecc_histogram_checked(const void *x, int dtype, int ndim, const int64_t *dims, int64_t batch,
                          int64_t plane_begin, int64_t plane_end, const void *table,
                          const ecc_binning *binning_host, int64_t *hist, int32_t *nonfinite, void *stream);

/* Inclusive prefix sum of bins[0..nbins) per batch item -> int64 curve
 * [batch][nbins] (compute_ecc, hard.py:226). */
int ecc_scan(const int64_t *hist, int64_t batch, int64_t nbins, int64_t *curve, void *stream);

/* Lower-star coefficients, int8 [batch][dims] (compute_coefficients,
 * coefficients.py:163-175). */
int ecc_coefficients(const void *x, int dtype, int ndim, const int64_t *dims, int64_t batch, int8_t *out,
                     void *stream);

/* Min / max / non-finite count of n values, as order-preserving uint64 keys
 * out3[0] (min), out3[1] (max), out3[2] (count of NaN/Inf); decode with
 * ecc_key_to_double().  Feeds uniform_thresholds (grid.py:183-196) and the
 * ScalarGrid finiteness check (grid.py:63-64). */
int ecc_minmax(const void *x, int dtype, int64_t n, uint64_t *out3, void *stream);
double ecc_key_to_double(uint64_t key);

/* Soft ECC (soft.py).  Parameters shared by forward and backward. */
typedef struct {
  double lam;          /* sharpness lambda > 0                                  */
  double alpha;        /* direction scale                                       */
  double u[3];         /* direction (first ndim used); any vector, not forced unit */
  double center;       /* m: taus and field are centred on m before fp32 math   */
  int32_t factorized;  /* 1: sigma = 1/(1 + a_j b_p), a_j = e^{-lam(tau_j-m_l)},
                          b_p = e^{lam(f_p-m_l)}, m_l the centre of the lane's
                          32-threshold block; 0: float64 exponent, ex2 + rcp   */
  int32_t pad;
} ecc_soft_params;

/* effective_field (soft.py:97-101): out = X + alpha * <u, pos> in float64
 * with the reference's rounding sequence.  u_host: ndim doubles (HOST). */
int ecc_effective_field(const void *x, int dtype, int ndim, const int64_t *dims, int64_t batch, double alpha,
                        const double *u_host, double *out, void *stream);

/* Workspace bytes for ecc_soft_forward/backward partials. */
size_t ecc_soft_workspace_bytes(int ndim, const int64_t *dims, int64_t batch, int64_t nbins);

/* Effective-field coefficients (the coefficients callers feed to soft_ecc:
 * compute_coefficients(effective_field(grid, alpha, u)), cli.py:201,
 * soft.py:292) computed from a float64 effective field built on the fly with
 * the reference's rounding sequence; also writes the centred field
 * f - m as float32 (field_c) and, when field_lo is not NULL, its float32
 * remainder (f - m) - field_c (needed by the direct mode below).
 * x: float32 or float64 grid. */
int ecc_soft_prepare(const void *x, int dtype, int ndim, const int64_t *dims, int64_t batch,
                     const ecc_soft_params *params_host, int8_t *coeffs, float *field_c, float *field_lo,
                     void *stream);

/* Forward: chi[batch][nbins] (float64) = sum_p c_p sigmoid(lam (tau_j - f_p))
 * (soft.py:154-196).  coeffs may be any int8 grid (e.g. the reference's).
 * taus: float64 [nbins] device.  workspace: ecc_soft_workspace_bytes.
 * factorized != 0: one MUFU.RCP per pair (per-lane centring, needs
 * lam*log2(e)*half-width of every 32-threshold block <= 40); otherwise the
 * direct mode forms each exponent in float64 (field_lo required). */
int ecc_soft_forward(const int8_t *coeffs, const float *field_c, const float *field_lo, int ndim,
                     const int64_t *dims, int64_t batch, const double *taus, int64_t nbins,
                     const ecc_soft_params *params_host, double *chi, void *workspace, void *stream);

/* Backward (soft.py:199-257 plus the alpha gradient):
 *   d_values[b][p] = -c_p w_p,  w_p = sum_j up[b][j] lam s(1-s)   (float32)
 *   d_tau[b][j]    = up[b][j] sum_p c_p lam s(1-s)                (float64)
 *   G[b][0..ndim)  = sum_p c_p w_p pos_p                          (float64)
 * from which d_u = -alpha G (then tangent-projected by the caller) and
 * d_alpha = -G.u.  upstream: float64 [batch][nbins]. */
int ecc_soft_backward(const int8_t *coeffs, const float *field_c, const float *field_lo, int ndim,
                      const int64_t *dims, int64_t batch, const double *taus, int64_t nbins,
                      const ecc_soft_params *params_host, const double *upstream, float *d_values, double *d_tau,
                      double *G, void *workspace, void *stream);

/* Sync-free variants for the autograd module (no device->host read per
 * call, so forward + backward can be captured in a CUDA graph or traced by
 * torch.compile): the parameters live in DEVICE memory.
 * ecc_soft_setup fills *params_dev from device tensors: center =
 * (min tau + max tau) / 2, factorized = lam log2(e) h <= 40 with h the
 * largest half-width of the 32-threshold blocks, lam, *alpha, u[0..ndim)
 * (taus, u, alpha: device float64).  The _d entry points take that device
 * struct instead of a host one; they launch both sigmoid modes and the one
 * the device flag does not select exits at once, so field_lo is required
 * (ecc_soft_prepare_d writes it only when the flag selects the direct mode). */
int ecc_soft_setup(const double *taus, int64_t nbins, const double *u, int ndim, const double *alpha, double lam,
                   ecc_soft_params *params_dev, void *stream);
int ecc_soft_prepare_d(const void *x, int dtype, int ndim, const int64_t *dims, int64_t batch,
                       const ecc_soft_params *params_dev, int8_t *coeffs, float *field_c, float *field_lo,
                       void *stream);
/* records (optional, ecc_soft_records_bytes; NULL: none): when the windowed
 * ("band") kernels run, the forward stores each warp's band-sorted non-zero
 * voxels there and the backward of the same inputs reads them instead of
 * compacting and sorting again (the kernels decide on the device; with the
 * full kernels the buffer is ignored).  16-byte aligned. */
size_t ecc_soft_records_bytes(int ndim, const int64_t *dims, int64_t batch);
int ecc_soft_forward_d(const int8_t *coeffs, const float *field_c, const float *field_lo, int ndim,
                       const int64_t *dims, int64_t batch, const double *taus, int64_t nbins,
                       const ecc_soft_params *params_dev, double *chi, void *workspace, void *records,
                       void *stream);
int ecc_soft_backward_d(const int8_t *coeffs, const float *field_c, const float *field_lo, int ndim,
                        const int64_t *dims, int64_t batch, const double *taus, int64_t nbins,
                        const ecc_soft_params *params_dev, const double *upstream, float *d_values, double *d_tau,
                        double *G, void *workspace, const void *records, void *stream);

/* Streaming a 3-D item in z-slabs (the host -> device copy overlapped with
 * the prepare and the forward; soft.py soft_ecc_fwd_host).  Same semantics as
 * ecc_soft_prepare_d / ecc_soft_forward_d restricted to part of the work:
 * ecc_soft_prepare_range_d writes the coefficients and fields of output
 * planes [plane_begin, plane_end) of a 3-D grid (reading the planes
 * plane_begin - 1 and plane_end as halos, which must be resident);
 * ecc_soft_units reports the forward's work split (chunks of 4096 voxels per
 * unit, units per item); ecc_soft_forward_range_d runs units [unit_begin,
 * unit_end) of items [item_begin, item_end) (their voxels must be prepared;
 * the buffers are the whole batch's) and, with finish != 0, reduces all
 * items' and units' partial rows into chi -- call it with finish once, after
 * every unit ran.  chunks_per_unit: 0 = the launcher's rule for the whole
 * batch (ecc_soft_units), else that many chunks per unit -- the same value
 * on every call of one pass (small item ranges fill the GPU with smaller
 * units).  Replaces the single-shot path of soft.py:154-196
 * (soft_ecc) for streamed inputs; the results are those of the single-shot
 * entry points. */
int ecc_soft_prepare_range_d(const void *x, int dtype, int ndim, const int64_t *dims, int64_t batch,
                             const ecc_soft_params *params_dev, int8_t *coeffs, float *field_c, float *field_lo,
                             int64_t plane_begin, int64_t plane_end, void *stream);
int ecc_soft_units(int ndim, const int64_t *dims, int64_t batch, int64_t *chunks_per_unit, int64_t *units);
int ecc_soft_forward_range_d(const int8_t *coeffs, const float *field_c, const float *field_lo, int ndim,
                             const int64_t *dims, int64_t batch, const double *taus, int64_t nbins,
                             const ecc_soft_params *params_dev, double *chi, void *workspace, void *records,
                             int64_t chunks_per_unit, int64_t item_begin, int64_t item_end, int64_t unit_begin,
                             int64_t unit_end, int finish, void *stream);
/* The backward of a unit range (upstream given up front, so a unit's
 * backward can follow its forward before the rest of the item arrived);
 * d_values of the range's voxels, the d_tau and G partial rows of its units,
 * reduced into d_tau and G on the call with finish.  Use a workspace apart
 * from the forward's while both are in flight (the partial rows share the
 * layout). */
int ecc_soft_backward_range_d(const int8_t *coeffs, const float *field_c, const float *field_lo, int ndim,
                              const int64_t *dims, int64_t batch, const double *taus, int64_t nbins,
                              const ecc_soft_params *params_dev, const double *upstream, float *d_values,
                              double *d_tau, double *G, void *workspace, const void *records,
                              int64_t chunks_per_unit, int64_t item_begin, int64_t item_end, int64_t unit_begin,
                              int64_t unit_end, int finish, void *stream);

/* Kernel-variant switch for A/B checks (tests, tools/): key "f3" with value
 * default | value | branch | cta | rank2 | no2d | edge1 | dummy | static,
 * "zunit" (forced dynamic unit in planes, "0" = automatic), "generic"
 * ("1": every grid through the generic sweep), "soft_fwd_t" / "soft_bwd_t"
 * (thresholds per soft lane: 8, 16, 32), "soft_band" ("0": the full soft
 * kernels even where the windowed ones apply), "soft_g" (chunks per soft
 * CTA, "0" = automatic), "soft_prep" ("1": the per-voxel tile prepare
 * instead of the row-word one).  Process-wide; the production kernels are
 * the defaults.  Returns 0 or ECC_EINVAL. */
int ecc_set_variant(const char *key, const char *value);

/* Finite-difference harness for gradient_check (soft.py:260-359), float64:
 * 4th-order central differences (soft.py:308-315) with step `step` of
 * L = sum_j up_j sum_p c_p sigmoid(lam (tau_j - f_p)), f the effective
 * field (float64, e.g. from ecc_effective_field), coefficients held fixed.
 * fd_values[n] = dL/dX_p, fd_tau[nbins] = dL/dtau_j, fd_dir[0..ndim) =
 * dL/du_a (free vector, unprojected), fd_dir[ndim] = dL/dalpha.  All
 * device pointers except u_host (ndim doubles, host). */
int ecc_soft_fd(const double *field, const int8_t *coeffs, int ndim, const int64_t *dims, const double *taus,
                int64_t nbins, const double *upstream, double lam, double alpha, const double *u_host, double step,
                double *fd_values, double *fd_tau, double *fd_dir, void *stream);

/* Counter-based synthetic float32 grid: out[i] = top-24-bits(splitmix64(
 * seed * K + start + i)) * 2^-24 (identical to the oracle's
 * generator so 2048^3 slabs are reproducible on both sides). */
int ecc_counter_grid(uint64_t seed, int64_t start, int64_t count, float *out, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* ECC_B200_H */
