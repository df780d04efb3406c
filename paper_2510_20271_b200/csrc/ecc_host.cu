// ecc_host.cu -- host-side pieces of the C ABI: errors, threshold tables,
// key decoding, and the counter-based synthetic generator kernel.
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <limits>
#include <vector>

#include "ecc_common.cuh"
#include "ecc_internal.h"

namespace ecc {
static thread_local char g_err[512] = "";

int set_error(int code, const char* msg) {
  snprintf(g_err, sizeof(g_err), "%s", msg);
  return code;
}
int set_cuda_error(cudaError_t e, const char* what) {
  snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
  return ECC_ECUDA;
}
void clear_error() { g_err[0] = 0; }

static std::atomic<int> g_f3{0}, g_zunit{0}, g_generic{0}, g_soft_fwd_t{16}, g_soft_bwd_t{16}, g_soft_band{1}, g_soft_g{0}, g_soft_prep{0};
int variant_f3() { return g_f3.load(std::memory_order_relaxed); }
int variant_zunit() { return g_zunit.load(std::memory_order_relaxed); }
bool variant_generic() { return g_generic.load(std::memory_order_relaxed) != 0; }
int variant_soft_t(bool bwd) { return (bwd ? g_soft_bwd_t : g_soft_fwd_t).load(std::memory_order_relaxed); }
bool variant_soft_band() { return g_soft_band.load(std::memory_order_relaxed) != 0; }
int variant_soft_g() { return g_soft_g.load(std::memory_order_relaxed); }
bool variant_soft_prep_old() { return g_soft_prep.load(std::memory_order_relaxed) != 0; }

// largest float32 <= t (round toward -inf), the t32 of DESIGN.md
static float round_down_f32(double t) {
  float f = (float)t;
  if ((double)f > t) f = std::nextafter(f, -std::numeric_limits<float>::infinity());
  return f;
}

template <typename V>
static int64_t true_bin(V x, const V* tab, int64_t nb) {
  // tab has sentinels: tab[j+1] = tau_j
  int64_t lo = 0, hi = nb;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (tab[mid + 1] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

template <typename V>
static int64_t guess_bin(V x, V t0, V inv_w, int64_t nb) {
  volatile V d = x - t0;  // volatile: no contraction, matches the device's two roundings
  V g = d * inv_w;
  if (g < V(0)) g = V(0);
  if (g > V(nb)) g = V(nb);
  return (int64_t)g;
}

template <typename V>
static void certify(const V* tab, int64_t nb, ecc_binning* b) {
  const V t0 = tab[1], tl = tab[nb];
  b->t0 = (double)t0;
  b->inv_w = 0.0;
  b->mode = 1;
  b->max_correction = -1;
  if (nb < 2) {
    b->mode = 0;  // guess 0 then correct: at most one step
    b->max_correction = 1;
    return;
  }
  if (!std::isfinite((double)t0) || !std::isfinite((double)tl) || !(tl > t0)) return;
  const V span = tl - t0;
  if (!std::isfinite((double)span)) return;
  const V inv_w = V(nb - 1) / span;
  if (!std::isfinite((double)inv_w) || !(inv_w > V(0))) return;
  int64_t worst = 0;
  for (int64_t j = 0; j < nb; ++j) {
    const V at = tab[j + 1];
    const V above = std::nextafter(at, std::numeric_limits<V>::infinity());
    const V probes[2] = {at, above};
    for (V x : probes) {
      int64_t t = true_bin<V>(x, tab, nb), gg = guess_bin<V>(x, t0, inv_w, nb);
      int64_t e = t > gg ? t - gg : gg - t;
      if (e > worst) worst = e;
    }
  }
  b->inv_w = (double)inv_w;
  b->max_correction = (int32_t)(worst > 0x7fffffff ? 0x7fffffff : worst);
  // a guess off by a few bins costs a few smem reads; beyond that binary
  // search is cheaper (grid.py:147-166 makes the same choice on the CPU)
  b->mode = worst <= 4 ? 0 : 1;
}

// ---- cell table of the float32 fast path (see ecc_binning in ecc_b200.h) ----
struct LutEntryH {
  float t;
  int32_t b;
};

// the device's cell computation, operation for operation:
//   g = sat(fma(x, scale, bias));  cell = floor(g * cells)   (cells = 2^k)
// (the device gets the floor from the mantissa of RZ(g + 1), exact for 2^k cells)
static int cell_of(float x, float scale, float bias, int cells) {
  float g = fmaf(x, scale, bias);
  if (!(g > 0.0f)) g = 0.0f;  // __saturatef: NaN -> 0
  if (g > 1.0f) g = 1.0f;
  return (int)floor((double)g * (double)cells);
}

static uint32_t fkey(float f) {
  uint32_t b;
  memcpy(&b, &f, 4);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
static float keyf(uint32_t k) {
  uint32_t b = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  float f;
  memcpy(&f, &b, 4);
  return f;
}

static int64_t bin32(float x, const float* t32, int64_t nb) {
  int64_t lo = 0, hi = nb;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (t32[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Build the cell table for thresholds t32 (non-decreasing); returns cells or 0.
// The cell grid maps [lo, hi] onto [0, 1]; by default lo/hi are the first and
// last thresholds.  aligned != 0 maps [t_0 - w, t_last] (w the mean spacing)
// instead, so that uniform thresholds fall on cell boundaries (cells == nb),
// which is what the edge tables below need.
// edge sub-cells per cell (ecc_fast3d.cu rank_edge / rank4): 1024 is tried
// first (fewer edge voxels), then 256
constexpr int EDGE_SUB_FINE = 1024, EDGE_SUB_COARSE = 256;
#ifndef ECC_EDGE_COARSE_ONLY
#define ECC_EDGE_COARSE_ONLY 0
#endif

static int build_lut(const float* t32, int64_t nb, int cells, float* scale_out, float* bias_out, LutEntryH* lut,
                     int aligned = 0) {
  if (nb < 2) return 0;
  float lo = t32[0];
  const float hi = t32[nb - 1];
  if (aligned) lo = (float)((double)t32[0] - ((double)hi - (double)t32[0]) / (double)(nb - 1));
  if (!std::isfinite(lo) || !std::isfinite(hi) || !(hi > lo)) return 0;
  volatile float span = hi - lo;
  if (!std::isfinite((float)span)) return 0;
  volatile float scale = 1.0f / span;
  if (!std::isfinite((float)scale) || !(scale > 0.0f)) return 0;
  volatile float bias = -(lo * scale);
  const uint32_t kmin = fkey(-std::numeric_limits<float>::max());
  const uint32_t kmax = fkey(std::numeric_limits<float>::max());
  // first key with cell >= k, for k = 0..cells+1
  std::vector<uint32_t> first((size_t)cells + 2);
  for (int k = 0; k <= cells + 1; ++k) {
    uint32_t a = kmin, b = kmax + 1;  // search in [a, b)
    while (a < b) {
      uint32_t mid = a + (b - a) / 2;
      if (cell_of(keyf(mid), scale, bias, cells) >= k) b = mid; else a = mid + 1;
    }
    first[k] = a;  // == kmax + 1 if no finite float reaches cell k
  }
  for (int k = 0; k <= cells; ++k) {
    if (first[k] >= first[k + 1]) {  // empty cell: never indexed
      lut[k].t = std::numeric_limits<float>::infinity();
      lut[k].b = (int32_t)nb;
      continue;
    }
    const float xlo = keyf(first[k]);
    const float xhi = keyf(first[k + 1] - 1);
    const int64_t b = bin32(xlo, t32, nb);
    if (bin32(xhi, t32, nb) > b + 1) return 0;  // two thresholds inside one cell
    lut[k].b = (int32_t)b;
    lut[k].t = b < nb ? t32[b] : std::numeric_limits<float>::infinity();
  }
  *scale_out = scale;
  *bias_out = bias;
  return cells;
}

// Edge tables for the float32 rank kernel (ecc_fast3d.cu).  Sub-cells are
// 1/256 of a cell, sub(x) = floor(sat(fma(x, scale, bias)) * 256 cells),
// computed by the device exactly as here.  When every threshold lies in the
// first or last sub-cell of a cell, a voxel needs its threshold only when it
// falls in such an edge sub-cell: rank(x) = idx + (x > tE[idx]) with
// idx = (sub(x) + 1) / 256 for edge sub-cells, and rank = cell + 1 otherwise.
// tE[b] is the threshold at boundary b (between cells b-1 and b), or the
// largest float below sub-cell 256 b when the boundary has none.  rank() is
// non-decreasing in x, so each rank's floats form one key interval, found by
// binary search; every interval is verified to lie in one bin (rbin[rank]).
// Returns 1 on success.
static int edge_rank(float x, float scale, float bias, int cells, const float* tE, int EDGE_SUB) {
  const int sidx = cell_of(x, scale, bias, cells * EDGE_SUB);
  const int k1 = sidx + 1;
  const int idx = k1 / EDGE_SUB;
  if ((k1 % EDGE_SUB) <= 1) return idx + (x > tE[idx] ? 1 : 0);
  return idx + 1;
}

static int build_edge(const float* t32, int64_t nb, int cells, float scale, float bias, float* tE,
                      int32_t* rbin, int EDGE_SUB) {
  const int nsub = cells * EDGE_SUB;
  if (cells + 2 >= 0x7FFF || nsub >= (1 << 23)) return 0;
  const uint32_t kmin = fkey(-std::numeric_limits<float>::max());
  const uint32_t kmax = fkey(std::numeric_limits<float>::max());
  auto first_key = [&](auto pred) {   // first finite key with pred(x) true (pred monotone)
    uint32_t a = kmin, b = kmax + 1;
    while (a < b) {
      const uint32_t mid = a + (b - a) / 2;
      if (pred(keyf(mid))) b = mid; else a = mid + 1;
    }
    return a;
  };
  std::vector<char> has((size_t)cells + 1, 0);
  for (int64_t j = 0; j < nb; ++j) {
    const float t = t32[j];
    const int sidx = cell_of(t, scale, bias, nsub);
    const int sub = sidx % EDGE_SUB;
    if (sub != 0 && sub != EDGE_SUB - 1) return 0;        // threshold inside a cell
    const int bnd = (sidx + 1) / EDGE_SUB;
    if (bnd > cells) return 0;
    if (has[bnd] && tE[bnd] != t) return 0;               // two thresholds at one boundary
    has[bnd] = 1;
    tE[bnd] = t;
  }
  for (int bnd = 0; bnd <= cells; ++bnd)
    if (!has[bnd]) {
      const uint32_t f = first_key([&](float x) { return cell_of(x, scale, bias, nsub) >= EDGE_SUB * bnd; });
      tE[bnd] = f > kmin ? keyf(f - 1) : -std::numeric_limits<float>::infinity();
    }
  // rank r holds keys [lo_r, lo_{r+1}); each nonempty interval must sit in one bin
  std::vector<uint32_t> lo((size_t)cells + 4);
  for (int r = 0; r <= cells + 3; ++r)
    lo[r] = first_key([&](float x) { return edge_rank(x, scale, bias, cells, tE, EDGE_SUB) >= r; });
  for (int r = 0; r <= cells + 1; ++r) {
    rbin[r] = 0;
    if (lo[r] >= lo[r + 1]) continue;
    const int64_t b0 = bin32(keyf(lo[r]), t32, nb), b1 = bin32(keyf(lo[r + 1] - 1), t32, nb);
    if (b0 != b1) return 0;
    rbin[r] = (int32_t)b0;
  }
  if (lo[cells + 2] <= kmax) return 0;   // no float may rank above cells + 1
  return 1;
}

__global__ void counter_grid_kernel(uint64_t seed, int64_t start, int64_t count, float* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = seed * 0xD1B54A32D192ED03ull + (uint64_t)(start + i);
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    out[i] = (float)(z >> 40) * (1.0f / 16777216.0f);
  }
}
}  // namespace ecc

using namespace ecc;

extern "C" const char* ecc_version(void) { return "ecc_b200 0.1.0 (sm_100a)"; }
extern "C" const char* ecc_last_error(void) { return g_err; }

extern "C" int ecc_set_variant(const char* key, const char* value) {
  clear_error();
  if (!key || !value) return set_error(ECC_EINVAL, "null pointer argument");
  if (!strcmp(key, "f3")) {
    static const struct { const char* n; int m; } names[] = {
        {"", F3_DEFAULT}, {"default", F3_DEFAULT}, {"value", F3_VALUE}, {"branch", F3_BRANCH}, {"cta", F3_CTA},
        {"rank2", F3_RANK2}, {"no2d", F3_NO2D}, {"edge1", F3_EDGE1}, {"dummy", F3_DUMMY}, {"static", F3_STATIC}};
    for (const auto& e : names)
      if (!strcmp(value, e.n)) {
        g_f3.store(e.m);
        return ECC_OK;
      }
    return set_error(ECC_EINVAL, "unknown f3 variant");
  }
  const int v = atoi(value);
  if (!strcmp(key, "zunit")) g_zunit.store(v > 0 ? v : 0);
  else if (!strcmp(key, "generic")) g_generic.store(v != 0);
  else if (!strcmp(key, "soft_fwd_t")) g_soft_fwd_t.store(v);
  else if (!strcmp(key, "soft_bwd_t")) g_soft_bwd_t.store(v);
  else if (!strcmp(key, "soft_band")) g_soft_band.store(v != 0);
  else if (!strcmp(key, "soft_g")) g_soft_g.store(v > 0 ? v : 0);
  else if (!strcmp(key, "soft_prep")) g_soft_prep.store(v != 0);
  else return set_error(ECC_EINVAL, "unknown variant key");
  return ECC_OK;
}

extern "C" double ecc_key_to_double(uint64_t k) {
  uint64_t b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
  double d;
  memcpy(&d, &b, sizeof d);
  return d;
}

extern "C" int ecc_threshold_table(const double* taus, int64_t nb, int dtype, void* table_host,
                                   ecc_binning* b) {
  clear_error();
  if (!taus || !table_host || !b) return set_error(ECC_EINVAL, "null pointer argument");
  if (nb < 1) return set_error(ECC_EINVAL, "threshold set must contain at least one value");
  if (nb > ECC_MAX_BINS) return set_error(ECC_EINVAL, "too many thresholds");
  for (int64_t j = 0; j < nb; ++j)
    if (!std::isfinite(taus[j])) return set_error(ECC_EINVAL, "thresholds must be finite");
  for (int64_t j = 1; j < nb; ++j)
    if (!(taus[j] > taus[j - 1])) return set_error(ECC_EINVAL, "thresholds must be strictly increasing");
  b->nbins = nb;
  b->lut_ok = 0;
  b->lut_edge = 0;
  b->lut_edge_sub = 0;
  b->lut_cells = 0;
  b->lut_scale = 0.0f;
  b->lut_bias = 0.0f;
  if (dtype == ECC_DTYPE_U8 || dtype == ECC_DTYPE_F32) {
    float* t = (float*)table_host;
    t[0] = -std::numeric_limits<float>::infinity();
    for (int64_t j = 0; j < nb; ++j) t[j + 1] = round_down_f32(taus[j]);
    t[nb + 1] = std::numeric_limits<float>::infinity();
    certify<float>(t, nb, b);
    LutEntryH* lut = reinterpret_cast<LutEntryH*>(t + ((nb + 2 + 1) & ~int64_t(1)));
    int64_t cells = 1;
    while (cells < nb) cells <<= 1;
    // every cell count tried here must stay within ecc_threshold_table_bytes'
    // cap (1 << 16 cells), which sized the caller's buffer
    if (cells == nb && nb >= 2 && cells <= (1 << 16)) {
      // power-of-two threshold count: try the boundary-aligned grid first
      float sc = 0.f, bi = 0.f;
      if (build_lut(t + 1, nb, (int)cells, &sc, &bi, lut, 1)) {
        float* tE = reinterpret_cast<float*>(lut + cells + 1);
        int32_t* rbin = reinterpret_cast<int32_t*>(tE + cells + 1);
        const int sub = (!ECC_EDGE_COARSE_ONLY && build_edge(t + 1, nb, (int)cells, sc, bi, tE, rbin, EDGE_SUB_FINE)) ? EDGE_SUB_FINE
                        : build_edge(t + 1, nb, (int)cells, sc, bi, tE, rbin, EDGE_SUB_COARSE) ? EDGE_SUB_COARSE
                                                                                             : 0;
        if (sub) {
          b->lut_ok = 1;
          b->lut_edge = 1;
          b->lut_edge_sub = sub;
          b->lut_cells = (int32_t)cells;
          b->lut_scale = sc;
          b->lut_bias = bi;
        }
      }
    }
    for (; cells <= 4 * nb && cells <= (1 << 16) && !b->lut_ok; cells <<= 1) {
      float sc = 0.f, bi = 0.f;
      if (build_lut(t + 1, nb, (int)cells, &sc, &bi, lut)) {
        b->lut_ok = 1;
        b->lut_cells = (int32_t)cells;
        b->lut_scale = sc;
        b->lut_bias = bi;
        float* tE = reinterpret_cast<float*>(lut + cells + 1);
        int32_t* rbin = reinterpret_cast<int32_t*>(tE + cells + 1);
        b->lut_edge_sub = build_edge(t + 1, nb, (int)cells, sc, bi, tE, rbin, EDGE_SUB_FINE) ? EDGE_SUB_FINE
                          : build_edge(t + 1, nb, (int)cells, sc, bi, tE, rbin, EDGE_SUB_COARSE) ? EDGE_SUB_COARSE
                                                                                               : 0;
        b->lut_edge = b->lut_edge_sub != 0;
      }
    }
  } else if (dtype == ECC_DTYPE_F64) {
    double* t = (double*)table_host;
    t[0] = -std::numeric_limits<double>::infinity();
    for (int64_t j = 0; j < nb; ++j) t[j + 1] = taus[j];
    t[nb + 1] = std::numeric_limits<double>::infinity();
    certify<double>(t, nb, b);
  } else {
    return set_error(ECC_EINVAL, "unsupported dtype");
  }
  return ECC_OK;
}

extern "C" int ecc_counter_grid(uint64_t seed, int64_t start, int64_t count, float* out, void* stream) {
  clear_error();
  if (!out) return set_error(ECC_EINVAL, "null pointer argument");
  if (count <= 0) return ECC_OK;
  int64_t blocks = (count + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  counter_grid_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(seed, start, count, out);
  return check_launch("counter_grid_kernel");
}

extern "C" size_t ecc_threshold_table_bytes(int64_t nb, int dtype) {
  if (nb < 1) return 0;
  if (dtype == ECC_DTYPE_F64) return sizeof(double) * (size_t)(nb + 2);
  int64_t cells = 1;
  while (cells < nb) cells <<= 1;
  cells *= 4;
  if (cells > (1 << 16)) cells = 1 << 16;
  // thresholds with sentinels, cell table, edge thresholds, rank -> bin
  return sizeof(float) * (size_t)((nb + 2 + 1) & ~int64_t(1)) + sizeof(LutEntryH) * (size_t)(cells + 1) +
         sizeof(float) * (size_t)(cells + 1) + sizeof(int32_t) * (size_t)(cells + 2);
}
