// ecc_discrete.cu -- discrete (exact, integer) ECC kernels for sm_100a.
//
//   K1/K2  ecc_sweep_kernel<Src, Sink>   stencil -> coefficient -> bin -> histogram
//   K3     ecc_scan_kernel               int64 prefix sum of the bins -> curve
//   K4     ecc_minmax_kernel             min/max (+ non-finite flag) for uniform_thresholds
//
// One streaming kernel sweeps every voxel once (hard.py:134-143's FullSweep
// per worker becomes a persistent CTA; hard.py:99-118's merge becomes one
// int64 atomic flush per CTA).  Compiled WITHOUT fast-math: FTZ would change
// subnormal comparisons (the reference's hypothesis test draws subnormals).
#include "ecc_common.cuh"
#include "ecc_internal.h"
#include <algorithm>
#include <map>
#include <mutex>
#include <type_traits>
#include <tuple>
#include <stdlib.h>

namespace ecc {

// ---------------------------------------------------------------------------
// Sources: produce the compared value of voxel (n, z, y, x) (in-bounds only).
// ---------------------------------------------------------------------------
template <typename T>
struct RawSrc;

// raw(lin) is the bare global load, make(raw, z, y, x) the value it stands
// for; the sweep issues raw loads one plane ahead and applies make() only
// when the plane is stored to shared memory, so the loads' latency overlaps
// the current plane's work.
template <>
struct RawSrc<uint8_t> {
  using V = float;
  using R = float;   // converted at load: nothing left for make()
  static constexpr bool kTransform = false;
  const uint8_t* __restrict__ x;
  __device__ __forceinline__ R raw(int64_t lin) const { return (float)x[lin]; }
  __device__ __forceinline__ V make(R r, int64_t, int64_t, int64_t) const { return r; }
  __device__ __forceinline__ V at(int64_t lin, int64_t, int64_t, int64_t) const { return (float)x[lin]; }
  __device__ __forceinline__ void init() {}
};
template <>
struct RawSrc<float> {
  using V = float;
  using R = float;
  static constexpr bool kTransform = false;
  const float* __restrict__ x;
  __device__ __forceinline__ R raw(int64_t lin) const { return x[lin]; }
  __device__ __forceinline__ V make(R r, int64_t, int64_t, int64_t) const { return r; }
  __device__ __forceinline__ V at(int64_t lin, int64_t, int64_t, int64_t) const { return x[lin]; }
  __device__ __forceinline__ void init() {}
};
template <>
struct RawSrc<double> {
  using V = double;
  using R = double;
  static constexpr bool kTransform = false;
  const double* __restrict__ x;
  __device__ __forceinline__ R raw(int64_t lin) const { return x[lin]; }
  __device__ __forceinline__ V make(R r, int64_t, int64_t, int64_t) const { return r; }
  __device__ __forceinline__ V at(int64_t lin, int64_t, int64_t, int64_t) const { return x[lin]; }
  __device__ __forceinline__ void init() {}
};


// Effective field f = X + alpha * <u, pos> in float64 with the reference's
// rounding sequence (soft.py:97-101, 147-151; numpy elementwise ops and
// OpenBLAS dgemv's fma order: 2D fma(p0,u0,p1*u1), 3D fma(p2,u2,fma(p0,u0,p1*u1))).
template <typename T>
struct EffSrc {
  using V = double;
  const T* __restrict__ x;
  double alpha, u0, u1, u2;
  int64_t D, H, W;
  int ndim;
  double sD, sH, sW;   // 2.0 / (d - 1) in float64 (host-computed like numpy), 0 when d == 1
  // device-resident soft parameters (ecc_soft_setup; sync-free module path):
  // alpha and u are read from there when the kernel starts
  const ecc_soft_params* pd = nullptr;
  __device__ __forceinline__ void init() {
    if (pd) {
      alpha = pd->alpha;
      u0 = pd->u[0];
      u1 = pd->u[1];
      u2 = pd->u[2];
    }
  }
  // pixel_coordinates (soft.py:79-94): idx * (2/(d-1)) - 1 with two roundings; 0 for d == 1
  __device__ __forceinline__ static double crd(int64_t idx, int64_t d, double s) {
    // extents are < 2^31 (checked by the launchers), so the int32 -> f64
    // conversion is exact and avoids the slow 64-bit integer conversion
    return d == 1 ? 0.0 : __dadd_rn(__dmul_rn((double)(int)idx, s), -1.0);
  }
  using R = T;
  static constexpr bool kTransform = true;
  __device__ __forceinline__ R raw(int64_t lin) const { return x[lin]; }
  __device__ __forceinline__ V make(R r, int64_t z, int64_t y, int64_t xx) const {
    double v = (double)r;
    if (alpha == 0.0) return v;
    double dot;
    if (ndim == 2) {
      double p0 = crd(y, H, sH), p1 = crd(xx, W, sW);
      dot = __fma_rn(p0, u0, __dmul_rn(p1, u1));
    } else {
      double p0 = crd(z, D, sD), p1 = crd(y, H, sH), p2 = crd(xx, W, sW);
      dot = __fma_rn(p2, u2, __fma_rn(p0, u0, __dmul_rn(p1, u1)));
    }
    return __dadd_rn(v, __dmul_rn(alpha, dot));
  }
  __device__ __forceinline__ V at(int64_t lin, int64_t z, int64_t y, int64_t xx) const {
    return make(x[lin], z, y, xx);
  }
};

static inline double coord_scale(int64_t d) { return d > 1 ? 2.0 / (double)(d - 1) : 0.0; }

// ---------------------------------------------------------------------------
// Sweep geometry
// ---------------------------------------------------------------------------
constexpr int TX = 32;            // tile width (x), one lane per column
constexpr int RY = 2;             // rows per thread
constexpr int WY = 8;             // warps per CTA
constexpr int TY = WY * RY;       // tile height (y) = 16
constexpr int NT = TX * WY;       // 256 threads
constexpr int PW = TX + 2;        // staged plane tile width  (1-voxel halo)
constexpr int PH = TY + 2;        // staged plane tile height
constexpr int PLANE = PW * PH;    // 612 values
constexpr int LPT = (PLANE + NT - 1) / NT;  // loads per thread per plane (3)
constexpr int NBUF = 4;           // ring: z-1, z, z+1 in use, z+2 being filled

struct Geom {
  int64_t D, H, W;       // per-item extents (2D grids use D = 1)
  int64_t zb, ze;        // planes [zb, ze) are deposited; planes outside are halo
  int64_t batch;
  int64_t tiles_x, tiles_y, zchunks, zc;  // zc = planes per work item
  int64_t items;         // batch * zchunks * tiles_y * tiles_x
};

// ---------------------------------------------------------------------------
// Sinks: consume (coefficient, value) of each in-bounds voxel.
// ---------------------------------------------------------------------------
template <typename V>
struct HistSink {
  // smem: histogram of nb+1 int32 (last = overflow) + threshold table (nb+2)
  const V* __restrict__ tab_g;     // device table with sentinels, nb+2 entries
  unsigned long long* __restrict__ hist;  // [batch][nb+1] int64 (two's complement)
  BinParams bp;
  int* s_hist;
  V* s_tab;
  int64_t cur_item_n;
  int64_t pending;   // voxels deposited since last flush (int32 overflow guard)
  // global mode (bin counts whose counters and table do not fit in shared
  // memory): the table is read through L1 and every voxel adds its c to the
  // int64 global histogram directly -- slower, but any bin count works
  int global_mode = 0;

  __device__ void init(unsigned char* smem) {
    const int nb = (int)bp.nb;
    cur_item_n = -1;
    pending = 0;
    if (global_mode) return;
    s_hist = reinterpret_cast<int*>(smem);
    size_t off = ((size_t)(nb + 1) * sizeof(int) + 15) & ~size_t(15);
    s_tab = reinterpret_cast<V*>(smem + off);
    for (int i = threadIdx.x; i <= nb; i += blockDim.x) s_hist[i] = 0;
    for (int i = threadIdx.x; i < nb + 2; i += blockDim.x) s_tab[i] = tab_g[i];
    cur_item_n = -1;
    pending = 0;
  }
  static size_t smem_bytes(int64_t nb) {
    return (((size_t)(nb + 1) * sizeof(int) + 15) & ~size_t(15)) + (size_t)(nb + 2) * sizeof(V);
  }
  // shared-memory budget of the counters + table; above it the global mode
  static constexpr size_t kSmemMax = 120 * 1024;
  __device__ void flush() {
    if (cur_item_n < 0 || global_mode) return;
    const int nb = (int)bp.nb;
    unsigned long long* h = hist + cur_item_n * (nb + 1);
    for (int i = threadIdx.x; i <= nb; i += blockDim.x) {
      int v = s_hist[i];
      if (v) {
        atomicAdd(h + i, (unsigned long long)(long long)v);
        s_hist[i] = 0;
      }
    }
  }
  // called by all threads at the start of a work item (after a barrier)
  __device__ void begin_item(int64_t n, int64_t voxels) {
    if (global_mode) {
      cur_item_n = n;
      return;
    }
    if (n != cur_item_n || pending + voxels > (int64_t(1) << 27)) {
      flush();
      __syncthreads();
      cur_item_n = n;
      pending = 0;
    }
    pending += voxels;
  }
  __device__ void end() { __syncthreads(); flush(); }
  __device__ __forceinline__ void put(int c, V value, int64_t, int64_t, int64_t, int64_t) {
    if (c != 0) {
      if (global_mode) {
        const int j = bin_of<V>(value, tab_g, (int)bp.nb, (V)bp.t0, (V)bp.inv_w, bp.mode);
        atomicAdd(hist + cur_item_n * (bp.nb + 1) + j, (unsigned long long)(long long)c);
      } else {
        const int j = bin_of<V>(value, s_tab, (int)bp.nb, (V)bp.t0, (V)bp.inv_w, bp.mode);
        atomicAdd(&s_hist[j], c);
      }
    }
  }
};

struct CoeffSink {
  int8_t* __restrict__ out;   // [batch][D][H][W]
  int64_t D, H, W;
  __device__ void init(unsigned char*) {}
  static size_t smem_bytes(int64_t) { return 0; }
  __device__ void begin_item(int64_t, int64_t) {}
  __device__ void end() {}
  template <typename V>
  __device__ __forceinline__ void put(int c, V, int64_t n, int64_t z, int64_t y, int64_t x) {
    out[((n * D + z) * H + y) * W + x] = (int8_t)c;
  }
};


// soft_prepare: coefficient of the effective field + centred fp32 field
struct SoftPrepSink {
  int8_t* __restrict__ coeffs;
  float* __restrict__ fc;
  float* __restrict__ fclo;   // optional: (f - m) - fc, for the float64-exponent direct mode
  double center;
  int64_t D, H, W;
  const ecc_soft_params* pd = nullptr;   // device-resident parameters: the centre is read there
  __device__ void init(unsigned char*) {
    if (pd) {
      center = pd->center;
      if (pd->factorized) fclo = nullptr;   // only the direct mode reads the remainders
    }
  }
  static size_t smem_bytes(int64_t) { return 0; }
  __device__ void begin_item(int64_t, int64_t) {}
  __device__ void end() {}
  template <typename V>
  __device__ __forceinline__ void put(int c, V value, int64_t n, int64_t z, int64_t y, int64_t x) {
    const int64_t i = ((n * D + z) * H + y) * W + x;
    coeffs[i] = (int8_t)c;
    const double d = (double)value - center;
    const float hi = (float)d;
    fc[i] = hi;
    if (fclo) fclo[i] = (float)(d - (double)hi);
  }
};

// ---------------------------------------------------------------------------
// The sweep kernel: persistent CTAs walk work items (n, z-chunk, tile_y,
// tile_x), x fastest so concurrently running CTAs share halo rows in L2.
// Each item stages planes of (TY+2) x (TX+2) values in a 4-deep smem ring
// (NaN outside the grid), keeps a rolling 3x(RY+2)x3 register window per
// thread and emits RY voxels per plane.
// ---------------------------------------------------------------------------
template <typename Src, typename Sink>
__global__ void __launch_bounds__(NT)
ecc_sweep_kernel(Src src, Sink sink, Geom g) {
  using V = typename Src::V;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* planes = reinterpret_cast<V*>(smem_raw);                       // [NBUF][PH][PW]
  unsigned char* sink_smem = smem_raw + sizeof(V) * NBUF * PLANE;
  sink.init(sink_smem);
  src.init();
  __syncthreads();

  const int tx = threadIdx.x & (TX - 1);
  const int wy = threadIdx.x >> 5;
  const V nanv = V(__int_as_float(0x7fffffff));

  for (int64_t item = blockIdx.x; item < g.items; item += gridDim.x) {
    int64_t r = item;
    const int64_t tile_x = r % g.tiles_x; r /= g.tiles_x;
    const int64_t tile_y = r % g.tiles_y; r /= g.tiles_y;
    const int64_t zchunk = r % g.zchunks; r /= g.zchunks;
    const int64_t n = r;
    const int64_t x0 = tile_x * TX, y0 = tile_y * TY;
    const int64_t zs = g.zb + zchunk * g.zc;
    const int64_t ze = min(zs + g.zc, g.ze);
    const int64_t item_base = n * g.D * g.H * g.W;
    sink.begin_item(n, (ze - zs) * TX * TY);

    // per-thread staging: raw loads (R) into registers, value transform +
    // shared-memory store later (see RawSrc)
    using R = typename Src::R;
    auto in_plane = [&](int64_t z, int k, int64_t& yy, int64_t& xx) -> bool {
      const int e = threadIdx.x + k * NT;
      if (e >= PLANE) return false;
      const int ry = e / PW, rx = e - ry * PW;
      yy = y0 - 1 + ry;
      xx = x0 - 1 + rx;
      return z >= 0 && z < g.D && yy >= 0 && yy < g.H && xx >= 0 && xx < g.W;
    };
    auto load_plane = [&](int64_t z, R (&buf)[LPT]) {
#pragma unroll
      for (int k = 0; k < LPT; ++k) {
        int64_t yy, xx;
        // sources without a transform load the final value (NaN out of grid)
        buf[k] = in_plane(z, k, yy, xx) ? src.raw(item_base + (z * g.H + yy) * g.W + xx)
                                        : (Src::kTransform ? R(0) : R(nanv));
      }
    };
    auto store_plane = [&](int64_t z, const R (&buf)[LPT]) {
      V* dst = planes + (int)((z + 4) & (NBUF - 1)) * PLANE;
#pragma unroll
      for (int k = 0; k < LPT; ++k) {
        const int e = threadIdx.x + k * NT;
        if (!Src::kTransform) {
          if (e < PLANE) dst[e] = buf[k];
        } else {
          int64_t yy, xx;
          const bool ok = in_plane(z, k, yy, xx);
          if (e < PLANE) dst[e] = ok ? src.make(buf[k], z, yy, xx) : nanv;
        }
      }
    };

    {
      R b0[LPT], b1[LPT], b2[LPT];
      load_plane(zs - 1, b0);
      load_plane(zs, b1);
      load_plane(zs + 1, b2);
      store_plane(zs - 1, b0);
      store_plane(zs, b1);
      store_plane(zs + 1, b2);
    }
    __syncthreads();

    // rolling window: win[plane][row][col], rows cover smem rows RY*wy .. RY*wy+RY+1
    V win[3][RY + 2][3];
#pragma unroll
    for (int pz = 0; pz < 2; ++pz) {
      const V* s = planes + (int)((zs - 1 + pz + 4) & (NBUF - 1)) * PLANE;
#pragma unroll
      for (int rr = 0; rr < RY + 2; ++rr)
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) win[pz + 1][rr][cc] = s[(RY * wy + rr) * PW + tx + cc];
    }

    for (int64_t z = zs; z < ze; ++z) {
      R nxt[LPT];
      const bool more = (z + 2 <= ze);   // plane z+2 is needed by step z+1
      if (more) load_plane(z + 2, nxt);
      // shift window and read plane z+1
      const V* s = planes + (int)((z + 1 + 4) & (NBUF - 1)) * PLANE;
#pragma unroll
      for (int rr = 0; rr < RY + 2; ++rr)
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) {
          win[0][rr][cc] = win[1][rr][cc];
          win[1][rr][cc] = win[2][rr][cc];
          win[2][rr][cc] = s[(RY * wy + rr) * PW + tx + cc];
        }
      const int64_t xg = x0 + tx;
#pragma unroll
      for (int ry = 0; ry < RY; ++ry) {
        const int64_t yg = y0 + RY * wy + ry;
        if (xg < g.W && yg < g.H) {
          V nb[3][3][3];
#pragma unroll
          for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b)
#pragma unroll
              for (int c = 0; c < 3; ++c) nb[a][b][c] = win[a][ry + b][c];
          const int c = coeff3<V>(nb);
          sink.put(c, nb[1][1][1], n, z, yg, xg);
        }
      }
      if (more) store_plane(z + 2, nxt);
      __syncthreads();
    }
  }
  sink.end();
}

// ---------------------------------------------------------------------------
// K3: inclusive prefix sum over nb bins per batch item (hard.py:226 cumsum).
// One CTA per item; blocked scan in int64.
// ---------------------------------------------------------------------------
__global__ void ecc_scan_kernel(const long long* __restrict__ hist, int64_t nb, long long* __restrict__ curve) {
  __shared__ long long s_part[1024];
  const int64_t n = blockIdx.x;
  const long long* h = hist + n * (nb + 1);
  long long* out = curve + n * nb;
  const int T = blockDim.x;
  const int64_t per = (nb + T - 1) / T;
  const int64_t b0 = threadIdx.x * per, b1 = min(b0 + per, nb);
  long long acc = 0;
  for (int64_t j = b0; j < b1; ++j) acc += h[j];
  s_part[threadIdx.x] = acc;
  __syncthreads();
  // Hillis-Steele over T partials
  for (int off = 1; off < T; off <<= 1) {
    long long v = threadIdx.x >= off ? s_part[threadIdx.x - off] : 0;
    __syncthreads();
    s_part[threadIdx.x] += v;
    __syncthreads();
  }
  long long run = threadIdx.x ? s_part[threadIdx.x - 1] : 0;
  for (int64_t j = b0; j < b1; ++j) {
    run += h[j];
    out[j] = run;
  }
}

// ---------------------------------------------------------------------------
// K4: min / max / non-finite count over n values (grid.py:192-193, 63-64).
// Results as order-preserving keys: out[0] = min key, out[1] = max key,
// out[2] = non-finite count.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void ecc_minmax_kernel(const T* __restrict__ x, int64_t n, unsigned long long* out) {
  unsigned long long mn = ~0ull, mx = 0ull, bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double v = (double)x[i];
    if (!isfinite(v)) { ++bad; continue; }
    unsigned long long k = f64_key(v);
    mn = k < mn ? k : mn;
    mx = k > mx ? k : mx;
  }
  for (int o = 16; o; o >>= 1) {
    unsigned long long a = __shfl_xor_sync(0xffffffffu, mn, o);
    unsigned long long b = __shfl_xor_sync(0xffffffffu, mx, o);
    unsigned long long c = __shfl_xor_sync(0xffffffffu, bad, o);
    mn = a < mn ? a : mn;
    mx = b > mx ? b : mx;
    bad += c;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(out + 0, mn);
    atomicMax(out + 1, mx);
    if (bad) atomicAdd(out + 2, bad);
  }
}

// float32 specialisation: 16-byte loads, float min/max, one key conversion per thread
__global__ void ecc_minmax_f32v_kernel(const float4* __restrict__ x4, int64_t n4, const float* __restrict__ tail,
                                       int ntail, unsigned long long* out) {
  float mn = INFINITY, mx = -INFINITY;
  unsigned long long bad = 0;
  auto take = [&](float v) {
    if (!(fabsf(v) <= 3.402823466e38f)) { ++bad; return; }
    mn = fminf(mn, v);
    mx = fmaxf(mx, v);
  };
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = __ldcs(x4 + i);
    take(v.x); take(v.y); take(v.z); take(v.w);
  }
  if (blockIdx.x == 0 && threadIdx.x < ntail) take(tail[threadIdx.x]);
  unsigned long long kmn = mn <= mx ? f64_key((double)mn) : ~0ull;
  unsigned long long kmx = mn <= mx ? f64_key((double)mx) : 0ull;
  for (int o = 16; o; o >>= 1) {
    unsigned long long a = __shfl_xor_sync(0xffffffffu, kmn, o);
    unsigned long long b = __shfl_xor_sync(0xffffffffu, kmx, o);
    unsigned long long c = __shfl_xor_sync(0xffffffffu, bad, o);
    kmn = a < kmn ? a : kmn;
    kmx = b > kmx ? b : kmx;
    bad += c;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(out + 0, kmn);
    atomicMax(out + 1, kmx);
    if (bad) atomicAdd(out + 2, bad);
  }
}

__global__ void ecc_minmax_init(unsigned long long* out) {
  out[0] = ~0ull;
  out[1] = 0ull;
  out[2] = 0ull;
}

// ---------------------------------------------------------------------------
// launch helpers
// ---------------------------------------------------------------------------
static int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

static Geom make_geom(const int64_t* dims3, int64_t batch, int64_t zc_hint, int64_t max_ctas, int64_t zb,
                      int64_t ze) {
  Geom g;
  g.D = dims3[0];
  g.H = dims3[1];
  g.W = dims3[2];
  g.zb = zb;
  g.ze = ze;
  const int64_t Dw = ze - zb;
  g.batch = batch;
  g.tiles_x = (g.W + TX - 1) / TX;
  g.tiles_y = (g.H + TY - 1) / TY;
  const int64_t tiles = g.tiles_x * g.tiles_y * batch;
  // pick the z-chunk so that items >= ~4 waves of the persistent grid while
  // keeping the z-halo overhead (2 planes per chunk) small
  int64_t zc = zc_hint > 0 ? zc_hint : 64;
  while (zc > 8 && tiles * ((Dw + zc - 1) / zc) < 4 * max_ctas) zc >>= 1;
  if (zc > Dw) zc = Dw;
  if (zc < 1) zc = 1;
  g.zc = zc;
  g.zchunks = (Dw + zc - 1) / zc;
  g.items = tiles * g.zchunks;
  return g;
}

// function attribute + occupancy once per (kernel, smem bytes, device)
static int sweep_occupancy(const void* kfn, size_t smem, int* occ) {
  // the attribute is raised to the largest dynamic smem any launch of the
  // kernel asked for (a smaller later setting would fail the larger launch)
  static std::mutex mu;
  static std::map<std::tuple<const void*, size_t, int>, int> cache;
  static std::map<std::pair<const void*, int>, size_t> attr;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find({kfn, smem, dev});
  if (it != cache.end()) {
    *occ = it->second;
    return ECC_OK;
  }
  size_t& cur = attr[{kfn, dev}];
  if (smem > 48 * 1024 && smem > cur) {
    cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaFuncSetAttribute(sweep)");
    cur = smem;
  }
  int o = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kfn, NT, smem);
  if (o < 1) return set_error(ECC_EINVAL, "sweep kernel does not fit on an SM");
  cache[{kfn, smem, dev}] = o;
  *occ = o;
  return ECC_OK;
}

template <typename Src, typename Sink>
static int launch_sweep(Src src, Sink sink, const int64_t* dims3, int64_t batch, size_t sink_smem,
                        cudaStream_t stream, int64_t zb = 0, int64_t ze = -1) {
  if (ze < 0) ze = dims3[0];
  using V = typename Src::V;
  const size_t smem = sizeof(V) * NBUF * PLANE + sink_smem;
  auto kfn = ecc_sweep_kernel<Src, Sink>;
  int occ = 0;
  if (int rc = sweep_occupancy(reinterpret_cast<const void*>(kfn), smem, &occ)) return rc;
  const int64_t max_ctas = (int64_t)num_sms() * occ;
  if (ze <= zb) return ECC_OK;
  Geom g = make_geom(dims3, batch, 0, max_ctas, zb, ze);
  int64_t grid = g.items < max_ctas ? g.items : max_ctas;
  if (grid < 1) return ECC_OK;
  kfn<<<(unsigned)grid, NT, smem, stream>>>(src, sink, g);
  return check_launch("ecc_sweep_kernel");
}

}  // namespace ecc

using namespace ecc;

// ---------------------------------------------------------------------------
// C-ABI launchers (declared in include/ecc_b200.h)
// ---------------------------------------------------------------------------
static int dims_to3(int ndim, const int64_t* dims, int64_t out[3]) {
  if (ndim == 2) {
    out[0] = 1;
    out[1] = dims[0];
    out[2] = dims[1];
  } else if (ndim == 3) {
    out[0] = dims[0];
    out[1] = dims[1];
    out[2] = dims[2];
  } else {
    return set_error(ECC_EINVAL, "grid must be 2D or 3D");
  }
  for (int a = 0; a < 3; ++a) {
    if (out[a] < 1) return set_error(ECC_EINVAL, "grid extents must be positive");
    if (out[a] > 2147483647) return set_error(ECC_EINVAL, "grid extent exceeds 2^31 - 1");
  }
  return ECC_OK;
}

namespace ecc {
// non-finite check pass for the kernels that do not check while they sweep
// (the float32 fallbacks; the production rank kernels fuse it)
template <typename T>
__global__ void nonfinite_kernel(const T* __restrict__ x, int64_t n, int* __restrict__ nf) {
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    bad |= !isfinite((double)x[i]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nf, 1);
}
}  // namespace ecc

static int histogram_range_impl(const void* x, int dtype, int ndim, const int64_t* dims, int64_t batch,
                                int64_t plane_begin, int64_t plane_end, const void* table,
                                const ecc_binning* binning, int64_t* hist, int* nf, void* stream) {
  clear_error();
  int64_t d3[3];
  int rc = dims_to3(ndim, dims, d3);
  if (rc) return rc;
  if (!x || !table || !binning || !hist) return set_error(ECC_EINVAL, "null pointer argument");
  if (batch < 1) return set_error(ECC_EINVAL, "batch must be >= 1");
  const int64_t nb = binning->nbins;
  if (nb < 1 || nb > ECC_MAX_BINS) return set_error(ECC_EINVAL, "number of thresholds out of range");
  if (ndim != 3 && (plane_begin != 0 || plane_end != 1))
    return set_error(ECC_EINVAL, "plane ranges apply to 3D grids (axis 0)");
  if (ndim == 2) { plane_begin = 0; plane_end = 1; }
  if (plane_begin < 0 || plane_end > d3[0] || plane_begin > plane_end)
    return set_error(ECC_EINVAL, "plane range outside the grid");
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(hist, 0, sizeof(int64_t) * (size_t)batch * (size_t)(nb + 1), s);
  if (e != cudaSuccess) return set_cuda_error(e, "cudaMemsetAsync(hist)");
  if (nf && (e = cudaMemsetAsync(nf, 0, sizeof(int), s)) != cudaSuccess)
    return set_cuda_error(e, "cudaMemsetAsync(nonfinite flag)");
  BinParams bp;
  bp.t0 = binning->t0;
  bp.inv_w = binning->inv_w;
  bp.nb = nb;
  bp.mode = binning->mode;
  bp.pad = 0;
  auto* h = reinterpret_cast<unsigned long long*>(hist);
  switch (dtype) {
    case ECC_DTYPE_U8: {   // always finite
      if (fast3d_u8_eligible(x, d3[0], d3[1], d3[2], batch, nb) && !variant_generic())
        return fast3d_u8_launch((const uint8_t*)x, d3[0], d3[1], d3[2], batch, plane_begin, plane_end, table,
                                binning, h, s);
      HistSink<float> sk{(const float*)table, h, bp};
      sk.global_mode = HistSink<float>::smem_bytes(nb) > HistSink<float>::kSmemMax;
      return launch_sweep(RawSrc<uint8_t>{(const uint8_t*)x}, sk, d3, batch,
                          sk.global_mode ? 0 : HistSink<float>::smem_bytes(nb), s, plane_begin, plane_end);
    }
    case ECC_DTYPE_F32: {
      bool checked = false;
      if (fast3d_eligible(x, d3[0], d3[1], d3[2], batch, nb) && !variant_generic()) {
        rc = fast3d_launch((const float*)x, d3[0], d3[1], d3[2], batch, plane_begin, plane_end, table, binning, h, s,
                           nf, &checked);
      } else {
        HistSink<float> sk{(const float*)table, h, bp};
        sk.global_mode = HistSink<float>::smem_bytes(nb) > HistSink<float>::kSmemMax;
        rc = launch_sweep(RawSrc<float>{(const float*)x}, sk, d3, batch,
                          sk.global_mode ? 0 : HistSink<float>::smem_bytes(nb), s, plane_begin, plane_end);
      }
      if (rc || !nf || checked) return rc;
      const int64_t n = batch * d3[0] * d3[1] * d3[2];
      nonfinite_kernel<float><<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, s>>>(
          (const float*)x, n, nf);
      return check_launch("nonfinite_kernel");
    }
    case ECC_DTYPE_F64: {
      HistSink<double> sk{(const double*)table, h, bp};
      sk.global_mode = HistSink<double>::smem_bytes(nb) > HistSink<double>::kSmemMax;
      rc = launch_sweep(RawSrc<double>{(const double*)x}, sk, d3, batch,
                        sk.global_mode ? 0 : HistSink<double>::smem_bytes(nb), s, plane_begin, plane_end);
      if (rc || !nf) return rc;
      const int64_t n = batch * d3[0] * d3[1] * d3[2];
      nonfinite_kernel<double><<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, s>>>(
          (const double*)x, n, nf);
      return check_launch("nonfinite_kernel");
    }
    default:
      return set_error(ECC_EINVAL, "unsupported dtype");
  }
}

extern "C" int ecc_histogram_range(const void* x, int dtype, int ndim, const int64_t* dims, int64_t batch,
                                   int64_t plane_begin, int64_t plane_end, const void* table,
                                   const ecc_binning* binning, int64_t* hist, void* stream) {
  return histogram_range_impl(x, dtype, ndim, dims, batch, plane_begin, plane_end, table, binning, hist, nullptr,
                              stream);
}

extern "C" int ecc_histogram_checked(const void* x, int dtype, int ndim, const int64_t* dims, int64_t batch,
                                     int64_t plane_begin, int64_t plane_end, const void* table,
                                     const ecc_binning* binning, int64_t* hist, int32_t* nonfinite, void* stream) {
  if (!nonfinite) {
    clear_error();
    return set_error(ECC_EINVAL, "null pointer argument");
  }
  return histogram_range_impl(x, dtype, ndim, dims, batch, plane_begin, plane_end, table, binning, hist, nonfinite,
                              stream);
}

extern "C" int ecc_histogram(const void* x, int dtype, int ndim, const int64_t* dims, int64_t batch,
                             const void* table, const ecc_binning* binning, int64_t* hist, void* stream) {
  if (ndim != 2 && ndim != 3) {
    clear_error();
    return set_error(ECC_EINVAL, "grid must be 2D or 3D");
  }
  return ecc_histogram_range(x, dtype, ndim, dims, batch, 0, ndim == 3 ? dims[0] : 1, table, binning, hist, stream);
}

extern "C" int ecc_scan(const int64_t* hist, int64_t batch, int64_t nbins, int64_t* curve, void* stream) {
  clear_error();
  if (!hist || !curve) return set_error(ECC_EINVAL, "null pointer argument");
  if (batch < 1 || nbins < 1) return set_error(ECC_EINVAL, "empty scan");
  ecc_scan_kernel<<<(unsigned)batch, 256, 0, (cudaStream_t)stream>>>((const long long*)hist, nbins,
                                                                      (long long*)curve);
  return check_launch("ecc_scan_kernel");
}

extern "C" int ecc_coefficients(const void* x, int dtype, int ndim, const int64_t* dims, int64_t batch, int8_t* out,
                                void* stream) {
  clear_error();
  int64_t d3[3];
  int rc = dims_to3(ndim, dims, d3);
  if (rc) return rc;
  if (!x || !out) return set_error(ECC_EINVAL, "null pointer argument");
  if (batch < 1) return set_error(ECC_EINVAL, "batch must be >= 1");
  CoeffSink sk{out, d3[0], d3[1], d3[2]};
  cudaStream_t s = (cudaStream_t)stream;
  switch (dtype) {
    case ECC_DTYPE_U8: return launch_sweep(RawSrc<uint8_t>{(const uint8_t*)x}, sk, d3, batch, 0, s);
    case ECC_DTYPE_F32: return launch_sweep(RawSrc<float>{(const float*)x}, sk, d3, batch, 0, s);
    case ECC_DTYPE_F64: return launch_sweep(RawSrc<double>{(const double*)x}, sk, d3, batch, 0, s);
    default: return set_error(ECC_EINVAL, "unsupported dtype");
  }
}

extern "C" int ecc_minmax(const void* x, int dtype, int64_t n, uint64_t* out3, void* stream) {
  clear_error();
  if (!x || !out3) return set_error(ECC_EINVAL, "null pointer argument");
  cudaStream_t s = (cudaStream_t)stream;
  auto* o = reinterpret_cast<unsigned long long*>(out3);
  ecc_minmax_init<<<1, 1, 0, s>>>(o);
  int64_t blocks = (n + 255) / 256;
  int64_t cap = (int64_t)num_sms() * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  switch (dtype) {
    case ECC_DTYPE_U8: ecc_minmax_kernel<uint8_t><<<(unsigned)blocks, 256, 0, s>>>((const uint8_t*)x, n, o); break;
    case ECC_DTYPE_F32:
      if (((uintptr_t)x & 15u) == 0) {
        const int64_t n4 = n / 4;
        int64_t b4 = (n4 + 255) / 256;
        if (b4 > cap) b4 = cap;
        if (b4 < 1) b4 = 1;
        ecc_minmax_f32v_kernel<<<(unsigned)b4, 256, 0, s>>>((const float4*)x, n4, (const float*)x + 4 * n4,
                                                              (int)(n - 4 * n4), o);
      } else {
        ecc_minmax_kernel<float><<<(unsigned)blocks, 256, 0, s>>>((const float*)x, n, o);
      }
      break;
    case ECC_DTYPE_F64: ecc_minmax_kernel<double><<<(unsigned)blocks, 256, 0, s>>>((const double*)x, n, o); break;
    default: return set_error(ECC_EINVAL, "unsupported dtype");
  }
  return check_launch("ecc_minmax_kernel");
}

namespace ecc {
// 2D soft prepare: one CTA per 32x8 pixel tile; the float64 effective field of
// the tile and its one-pixel halo is built once in shared memory (NaN outside
// the grid), then each thread writes its pixel's coefficient and centred field.
#ifndef PREP_TH
#define PREP_TH 32   // output rows per CTA of the 2D soft prepare
#endif
template <typename T>
__global__ void __launch_bounds__(256) soft_prep2d_kernel(EffSrc<T> src, double center, int8_t* __restrict__ coeffs,
                                                          float* __restrict__ fc, float* __restrict__ fclo) {
  src.init();
  if (src.pd) {
    center = src.pd->center;
    if (src.pd->factorized) fclo = nullptr;   // only the direct mode reads the remainders
  }
  // 32 x 32 outputs per CTA (8 warps x 4 rows); the 34 x 34 effective-field
  // tile is loaded with all of a thread's global loads in flight at once
  constexpr int TH = PREP_TH, TW = 32, PWD = TW + 2, PHT = TH + 2, NE = PWD * PHT, PER = (NE + 255) / 256;
  __shared__ double tile[PHT][PWD];
  const int64_t n = blockIdx.z;
  const int64_t y0 = (int64_t)blockIdx.y * TH, x0 = (int64_t)blockIdx.x * TW;
  const int64_t H = src.H, W = src.W;
  const int64_t base = n * H * W;
  const double nanv = __longlong_as_double(0x7ff8000000000000ll);
  double vals[PER];
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int e = threadIdx.x + 256 * k;
    const int ry = e / PWD, rx = e - ry * PWD;
    const int64_t yy = y0 - 1 + ry, xx = x0 - 1 + rx;
    vals[k] = (e < NE && yy >= 0 && yy < H && xx >= 0 && xx < W) ? src.at(base + yy * W + xx, 0, yy, xx) : nanv;
  }
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int e = threadIdx.x + 256 * k;
    if (e < NE) tile[e / PWD][e % PWD] = vals[k];
  }
  __syncthreads();
  const int tx = threadIdx.x & 31, wy = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < TH / 8; ++q) {
    const int ty = wy + 8 * q;
    const int64_t y = y0 + ty, x = x0 + tx;
    if (y < H && x < W) {
      double v[3][3];
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) v[a][b] = tile[ty + a][tx + b];
      const int64_t i = base + y * W + x;
      coeffs[i] = (int8_t)coeff2<double>(v);
      const double d = v[1][1] - center;
      const float hi = (float)d;
      fc[i] = hi;
      if (fclo) fclo[i] = (float)(d - (double)hi);
    }
  }
}
}  // namespace ecc

#ifndef ECC_PREP_SGN
#define ECC_PREP_SGN 0   // 1: coeff3_sgn (sign bits of RD/RN differences + funnel shifts) in the 3-D
                         // soft prepare; measured slower at 1024^3 (9.87 vs 9.05 ms: the nine
                         // chained pushes per mask are a longer dependency chain than the
                         // independent predicate selects)
#endif
namespace ecc {
// 3-D soft prepare (C4).  The generic sweep's z-streaming tiling (32 x 16
// outputs per work item, a 4-plane float64 ring in shared memory, a 3 x 4 x 3
// register window per thread), specialised for the effective field: every
// thread stages the same three (row, column) positions of each plane of an
// item, so the position terms of the field are formed once per item and a
// staged voxel costs only
//   t = fma(p0(z), u0, p1(y) u1),  dot = fma(p2(x), u2, t),  f = x + alpha dot
// -- the reference's rounding sequence (soft.py:97-101; OpenBLAS dgemv's fma
// order), bit for bit the generic sweep's EffSrc::make -- with 32-bit index
// and bounds arithmetic per plane.
#ifndef ECC_PREP_MINB
#define ECC_PREP_MINB 2
#endif
template <typename T>
__global__ void __launch_bounds__(NT, ECC_PREP_MINB)
soft_prep3d_kernel(EffSrc<T> src, SoftPrepSink sk, Geom g) {
  __shared__ double planes[NBUF][PLANE];
  src.init();
  sk.init(nullptr);
  const int tx = threadIdx.x & (TX - 1);
  const int wy = threadIdx.x >> 5;
  const double nanv = __longlong_as_double(0x7ff8000000000000ll);
  const int64_t HW = g.H * g.W;
  int sry[LPT], srx[LPT];
#pragma unroll
  for (int k = 0; k < LPT; ++k) {
    const int e = threadIdx.x + k * NT;
    sry[k] = e / PW;
    srx[k] = e - sry[k] * PW;
  }
  // the remainder output is selected once (uniform), not per voxel
  auto run = [&](auto lotag) {
  constexpr bool LO = decltype(lotag)::value;
  for (int64_t item = blockIdx.x; item < g.items; item += gridDim.x) {
    int64_t r = item;
    const int64_t tile_x = r % g.tiles_x; r /= g.tiles_x;
    const int64_t tile_y = r % g.tiles_y; r /= g.tiles_y;
    const int64_t zchunk = r % g.zchunks; r /= g.zchunks;
    const int64_t n = r;
    const int64_t x0 = tile_x * TX, y0 = tile_y * TY;
    const int64_t zs = g.zb + zchunk * g.zc;
    const int64_t ze = min(zs + g.zc, g.ze);
    const T* xb = src.x + n * g.D * HW;
    // per staged position: in-grid flag, in-plane offset, p1 u1 and p2
    bool ok[LPT];
    int64_t off[LPT];
    double p1u1[LPT], p2[LPT];
#pragma unroll
    for (int k = 0; k < LPT; ++k) {
      const int64_t yy = y0 - 1 + sry[k], xx = x0 - 1 + srx[k];
      ok[k] = threadIdx.x + k * NT < PLANE && yy >= 0 && yy < g.H && xx >= 0 && xx < g.W;
      off[k] = ok[k] ? yy * g.W + xx : 0;
      p1u1[k] = __dmul_rn(EffSrc<T>::crd(ok[k] ? yy : 0, g.H, src.sH), src.u1);
      p2[k] = EffSrc<T>::crd(ok[k] ? xx : 0, g.W, src.sW);
    }
    auto load_plane = [&](int64_t z, T (&buf)[LPT]) {
      const bool zin = z >= 0 && z < g.D;
      const T* zp = xb + z * HW;
#pragma unroll
      for (int k = 0; k < LPT; ++k) buf[k] = (zin && ok[k]) ? zp[off[k]] : T(0);
    };
    // alpha = 0 needs no branch: v + 0 * dot == v (dot is finite)
    auto store_plane = [&](int64_t z, const T (&buf)[LPT]) {
      double* dst = planes[(int)((z + 4) & (NBUF - 1))];
      const bool zin = z >= 0 && z < g.D;
      const double t0 = EffSrc<T>::crd(zin ? z : 0, g.D, src.sD);   // p0(z)
#pragma unroll
      for (int k = 0; k < LPT; ++k) {
        const int e = threadIdx.x + k * NT;
        if (k < LPT - 1 || e < PLANE) {
          const double dot = __fma_rn(p2[k], src.u2, __fma_rn(t0, src.u0, p1u1[k]));
          // -0 -> +0 (coeff3_sgn's sign-bit compares; equal values either way)
          const double v = __dadd_rn(__dadd_rn((double)buf[k], __dmul_rn(src.alpha, dot)), 0.0);
          dst[e] = (zin && ok[k]) ? v : nanv;
        }
      }
    };
    {
      T b0[LPT], b1[LPT], b2[LPT];
      load_plane(zs - 1, b0);
      load_plane(zs, b1);
      load_plane(zs + 1, b2);
      store_plane(zs - 1, b0);
      store_plane(zs, b1);
      store_plane(zs + 1, b2);
    }
    __syncthreads();
    double win[3][RY + 2][3];
#pragma unroll
    for (int pz = 0; pz < 2; ++pz) {
      const double* sp = planes[(int)((zs - 1 + pz + 4) & (NBUF - 1))];
#pragma unroll
      for (int rr = 0; rr < RY + 2; ++rr)
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) win[pz + 1][rr][cc] = sp[(RY * wy + rr) * PW + tx + cc];
    }
    const int64_t xg = x0 + tx;
    const int64_t yb = y0 + RY * wy;
    // outputs of this thread: (z, yb + ry, xg); pointers advance by a plane
    const int64_t i0 = ((n * g.D + zs) * g.H + yb) * g.W + xg;
    int8_t* cp = sk.coeffs + i0;
    float* fp = sk.fc + i0;
    float* lp = LO ? sk.fclo + i0 : nullptr;
    bool inb[RY];
#pragma unroll
    for (int ry = 0; ry < RY; ++ry) inb[ry] = xg < g.W && yb + ry < g.H;
    for (int64_t z = zs; z < ze; ++z) {
      T nxt[LPT];
      const bool more = (z + 2 <= ze);
      if (more) load_plane(z + 2, nxt);
      const double* sp = planes[(int)((z + 1 + 4) & (NBUF - 1))];
#pragma unroll
      for (int rr = 0; rr < RY + 2; ++rr)
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) {
          win[0][rr][cc] = win[1][rr][cc];
          win[1][rr][cc] = win[2][rr][cc];
          win[2][rr][cc] = sp[(RY * wy + rr) * PW + tx + cc];
        }
#pragma unroll
      for (int ry = 0; ry < RY; ++ry) {
        double nb[3][3][3];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b)
#pragma unroll
            for (int c = 0; c < 3; ++c) nb[a][b][c] = win[a][ry + b][c];
        const int c = ECC_PREP_SGN ? coeff3_sgn(nb) : coeff3<double>(nb);
        const double d = nb[1][1][1] - sk.center;
        const float hi = (float)d;
        if (inb[ry]) {
          cp[ry * g.W] = (int8_t)c;
          fp[ry * g.W] = hi;
          if (LO) lp[ry * g.W] = (float)(d - (double)hi);
        }
      }
      cp += HW;
      fp += HW;
      if (LO) lp += HW;
      if (more) store_plane(z + 2, nxt);
      __syncthreads();
    }
  }
  };
  if (sk.fclo) run(std::true_type{});
  else run(std::false_type{});
}
}  // namespace ecc

namespace ecc {
// ---------------------------------------------------------------------------
// 3-D soft prepare, row-word formulation (C4; the default for float32 /
// float64 grids).  One warp per work item: a tile of 30 rows x 28 columns
// streamed over a z-chunk.  Lane l owns row y0 - 1 + l (lanes 0 and 31 are
// halo rows: their words serve the neighbours, they write nothing) and walks
// the 30 voxels x0 - 1 .. x0 + 28 of its row once per plane, comparing each
// with its 13 "positive" neighbours (first non-zero offset component +1).
// The sign of RN(q - p) is [q < p] exactly (a difference of distinct doubles
// never rounds to zero; values are canonicalised, -0 -> +0), and a funnel
// shift pushes it into a 32-bit word per direction (bit j = voxel x0 - 1 + j,
// the two end voxels included).  The 13 "negative" relations are the
// complements of the neighbours' positive ones -- [q <= p] = !(p < q) -- taken
// from the lane above (SHFL), the previous plane's words and the shifted own
// words, so each pair of voxels is compared once instead of twice.  The
// lower-star coefficient c = 1 - E + S - C (coefficients.py:109-138) is then
// evaluated bit-sliced on the 26 words -- squares and cubes are ANDs, the
// count a carry-save adder tree -- 32 voxels per instruction, and spread to
// bytes.  Out-of-grid positions hold +inf: never lower, and !(p < +inf) is
// false, so the complements stay right.  A tile whose effective field holds a
// non-finite value is redone voxel by voxel with the IEEE compares (coeff3's
// NaN semantics, the generic sweep's result).
// ---------------------------------------------------------------------------
#ifndef ECC_RW_UNR
#define ECC_RW_UNR 4   // unroll of the staging loops (rows): 1 / 2 / 4 / 8 measured 7.19 / 6.92 / 6.87 / 6.99 ms
#endif
#ifndef ECC_RW_MINB
#define ECC_RW_MINB 1   // resident warps per SM the register budget must allow
#endif
#ifndef ECC_RW_LA
#define ECC_RW_LA 5    // look-ahead of the plane walk's column reads: 1 / 2 / 3 / 5 measured 6.90 / 6.72 / 6.72 / 6.62 ms
#endif
#define ECC_RW_PRAGMA(x) _Pragma(#x)
#define ECC_RW_PRAGMA2(n) ECC_RW_PRAGMA(unroll n)
#define ECC_RW_UNROLL ECC_RW_PRAGMA2(ECC_RW_UNR)
constexpr int RWR = 34;      // staged rows: y0 - 2 .. y0 + 31
constexpr int RWC = 32;      // staged columns: x0 - 2 .. x0 + 29, one per lane
constexpr int RWLD = 33;     // row stride in doubles (odd: lanes reading one column hit distinct banks)
constexpr int RWOUT = 30;    // output rows per tile (lanes 1 .. 30)
constexpr int RWX = 28;      // output columns per tile: x0 .. x0 + 27

template <typename T>
struct RwSmem {
  // effective field of planes z (slot z & 1) and z + 1; a plane's raw values
  // arrive (cp.async) at the end of the slot it is converted into
  double eff[2][RWR * RWLD];
  double p1u1[RWR];            // per staged row: crd(y) * u1
  double q[RWR];               // per staged row of the plane being staged: fma(crd(z), u0, p1u1)
  __device__ __forceinline__ T* raw(int slot) {
    return reinterpret_cast<T*>(reinterpret_cast<char*>(eff[slot]) + sizeof(double) * RWR * RWLD -
                                sizeof(T) * RWR * RWC);
  }
};

__device__ __forceinline__ void fa3(uint32_t a, uint32_t b, uint32_t c, uint32_t& s, uint32_t& cy) {
  s = a ^ b ^ c;
  cy = (a & b) | (c & (a ^ b));
}
__device__ __forceinline__ uint32_t spread4(uint32_t n) { return (n * 0x00204081u) & 0x01010101u; }

template <typename T>
__device__ __forceinline__ void cp_async_t(void* sdst, const T* gsrc, bool in) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(sdst);
  if (sizeof(T) == 4)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(gsrc), "r"(in ? 4 : 0) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(gsrc), "r"(in ? 8 : 0) : "memory");
}

// Words: bit j of a lane's direction word is the voxel x0 - 1 + j of its row
// (j = 0 .. 29: the 28 outputs and one halo voxel each side), so the shifted
// reads of the negative relations are single shifts.
template <typename T>
__global__ void __launch_bounds__(32, ECC_RW_MINB) soft_prep3d_rw_kernel(EffSrc<T> src, SoftPrepSink sk, int64_t batch,
                                                            int64_t tiles_x, int64_t tiles_y, int64_t zc,
                                                            int64_t zchunks, int64_t zb, int64_t zlim) {
  __shared__ __align__(16) RwSmem<T> S;
  src.init();
  sk.init(nullptr);
  const int lane = threadIdx.x;
  const int64_t D = sk.D, H = sk.H, W = sk.W, HW = H * W;
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  int64_t r = blockIdx.x;
  const int64_t tile_x = r % tiles_x; r /= tiles_x;
  const int64_t tile_y = r % tiles_y; r /= tiles_y;
  const int64_t zchunk = r % zchunks; r /= zchunks;
  const int64_t n = r;
  if (n >= batch) return;
  const int64_t x0 = tile_x * RWX, y0 = tile_y * RWOUT;
  const int64_t zs = zb + zchunk * zc, ze = min(zs + zc, zlim);   // output planes [zb, zlim) (halo planes read)
  const T* xb = src.x + n * D * HW;
  // tile and halo inside the grid in x and y: no per-value range checks
  const bool inner = x0 >= 2 && x0 + RWC - 2 <= W && y0 >= 2 && y0 + RWR - 2 <= H;

  const int64_t gx = x0 - 2 + lane;   // this lane's staged column
  const bool cok = gx >= 0 && gx < W;
  const double p2 = EffSrc<T>::crd(cok ? gx : 0, W, src.sW);
  for (int row = lane; row < RWR; row += 32) {
    const int64_t gy = y0 - 2 + row;
    S.p1u1[row] = __dmul_rn(EffSrc<T>::crd(gy >= 0 && gy < H ? gy : 0, H, src.sH), src.u1);
  }
  __syncwarp();

  auto issue = [&](int64_t zp) {   // cp.async plane zp's raw values (zero-filled outside the grid)
    const bool zin = zp >= 0 && zp < D;
    T* raw = S.raw((int)(zp & 1));
    if (inner && zin) {
      const T* rp = xb + zp * HW + (y0 - 2) * W + gx;
ECC_RW_UNROLL
      for (int row = 0; row < RWR; ++row, rp += W) cp_async_t(&raw[row * RWC + lane], rp, true);
    } else {
      const T* pl = xb + (zin ? zp : 0) * HW;
ECC_RW_UNROLL
      for (int row = 0; row < RWR; ++row) {
        const int64_t gy = y0 - 2 + row;
        const bool in = zin && cok && gy >= 0 && gy < H;
        cp_async_t(&raw[row * RWC + lane], pl + (in ? gy * W + gx : 0), in);
      }
    }
    cp_async_commit();
  };
  uint32_t badhi = 0;   // max of the exponent fields of the effective field: 0x7ff00000 = non-finite
  auto convert = [&](int64_t zp) {   // raw -> effective field (the generic sweep's rounding sequence)
    cp_async_wait_all();
    const bool zin = zp >= 0 && zp < D;
    const double t0 = EffSrc<T>::crd(zin ? zp : 0, D, src.sD);
    for (int row = lane; row < RWR; row += 32) S.q[row] = __fma_rn(t0, src.u0, S.p1u1[row]);
    __syncwarp();
    double* dst = S.eff[(int)(zp & 1)];
    // In place: the raw values sit at the end of the slot.  Converted row by
    // row in order, row r's float64 values end before raw row r + 1 starts
    // (264 (r + 1) <= slot - raw + RWC sizeof(T) (r + 1) for r < 34), and
    // within a row every lane's load precedes the warp's store.
    const T* raw = S.raw((int)(zp & 1));
    if (inner && zin) {
ECC_RW_UNROLL
      for (int row = 0; row < RWR; ++row) {
        const double dot = __fma_rn(p2, src.u2, S.q[row]);
        const double v = __dadd_rn(__dadd_rn((double)raw[row * RWC + lane], __dmul_rn(src.alpha, dot)), 0.0);
        badhi = max(badhi, (uint32_t)__double2hiint(v) & 0x7ff00000u);
        dst[row * RWLD + lane] = v;
      }
    } else {
ECC_RW_UNROLL
      for (int row = 0; row < RWR; ++row) {
        const int64_t gy = y0 - 2 + row;
        const bool in = zin && cok && gy >= 0 && gy < H;
        const double dot = __fma_rn(p2, src.u2, S.q[row]);
        const double v = __dadd_rn(__dadd_rn((double)raw[row * RWC + lane], __dmul_rn(src.alpha, dot)), 0.0);
        if (in) badhi = max(badhi, (uint32_t)__double2hiint(v) & 0x7ff00000u);
        dst[row * RWLD + lane] = in ? v : inf;   // outside the grid: never lower
      }
    }
    __syncwarp();
  };

  // one plane walk: the 13 positive-direction words of this lane's row, plus
  // the centred field stores of output planes
  const int sr = lane + 1;
  const int64_t gyl = y0 - 1 + lane;
  const bool rowout = lane >= 1 && lane <= RWOUT && gyl < H;
  // vector stores (float4 field, 4-byte coefficient words) need whole,
  // aligned rows: caller buffers of the C ABI may be arbitrary
  const bool fullx = x0 + RWX <= W && (W & 3) == 0 &&
                     (((uintptr_t)sk.fc | (uintptr_t)sk.fclo) & 15) == 0 && ((uintptr_t)sk.coeffs & 3) == 0;
  auto walk = [&](int64_t z, uint32_t (&Wd)[13], bool out, int64_t obase, auto lotag) {
    constexpr bool LO = decltype(lotag)::value;
    const double* a = S.eff[(int)(z & 1)] + sr * RWLD;
    const double* b = S.eff[(int)(z & 1)] + (sr + 1) * RWLD;
    const double* c0 = S.eff[(int)((z + 1) & 1)] + (sr - 1) * RWLD;
    const double* c1 = S.eff[(int)((z + 1) & 1)] + sr * RWLD;
    const double* c2 = S.eff[(int)((z + 1) & 1)] + (sr + 1) * RWLD;
    double av[RWC], bv[RWC], c0v[RWC], c1v[RWC], c2v[RWC];
    // columns are read ECC_RW_LA steps ahead of their first use
#pragma unroll
    for (int j = RWC - 1; j >= RWC - 1 - ECC_RW_LA; --j) {
      av[j] = a[j]; bv[j] = b[j]; c0v[j] = c0[j]; c1v[j] = c1[j]; c2v[j] = c2[j];
    }
    float f4[4], l4[4];
    const bool wr = out && rowout;
#pragma unroll
    for (int sc = RWC - 2; sc >= 1; --sc) {   // voxel x0 - 2 + sc, bit sc - 1
      if (sc - ECC_RW_LA >= 0) {
        const int j = sc - ECC_RW_LA;
        av[j] = a[j]; bv[j] = b[j]; c0v[j] = c0[j]; c1v[j] = c1[j]; c2v[j] = c2[j];
      }
      const double p = av[sc];
      const double qv[13] = {av[sc + 1], bv[sc - 1], bv[sc], bv[sc + 1], c0v[sc - 1], c0v[sc], c0v[sc + 1],
                             c1v[sc - 1], c1v[sc], c1v[sc + 1], c2v[sc - 1], c2v[sc], c2v[sc + 1]};
#pragma unroll
      for (int d = 0; d < 13; ++d) {
        const uint32_t h = (uint32_t)__double2hiint(__dsub_rn(qv[d], p));   // bit 31 = [q < p]
        Wd[d] = __funnelshift_l(h, Wd[d], 1);
      }
      if (sc >= 2 && sc <= RWX + 1) {
        const int i = sc - 2;   // voxel x0 + i
        const double dd = p - sk.center;
        f4[i & 3] = (float)dd;
        if (LO) l4[i & 3] = (float)(dd - (double)f4[i & 3]);
        if ((i & 3) == 0 && wr) {
          float* fp = sk.fc + obase + i;
          float* lp = LO ? sk.fclo + obase + i : nullptr;
          if (fullx) {
            *reinterpret_cast<float4*>(fp) = make_float4(f4[0], f4[1], f4[2], f4[3]);
            if (LO) *reinterpret_cast<float4*>(lp) = make_float4(l4[0], l4[1], l4[2], l4[3]);
          } else {
#pragma unroll
            for (int t = 0; t < 4; ++t)
              if (x0 + i + t < W) {
                fp[t] = f4[t];
                if (LO) lp[t] = l4[t];
              }
          }
        }
      }
    }
  };

  auto tile = [&](auto lotag) {
    // prologue: planes zs - 1 and zs staged; the walk of plane zs - 1 gives
    // the previous-plane words
    issue(zs - 1);
    convert(zs - 1);
    issue(zs);
    convert(zs);
    uint32_t Wd[13], Pz[9];
    walk(zs - 1, Wd, false, 0, lotag);
#pragma unroll
    for (int d = 0; d < 9; ++d) Pz[d] = Wd[4 + d];
    __syncwarp();
    issue(zs + 1);   // into the slot of zs - 1, done with
    convert(zs + 1);
    int64_t obase = ((n * D + zs) * H + gyl) * W + x0;
    for (int64_t z = zs; z < ze; ++z, obase += HW) {
      // planes z, z + 1 are staged; plane z + 2 is fetched into the slot of
      // plane z once the walk has read it, while the words are evaluated
      walk(z, Wd, true, obase, lotag);
      const bool next = z + 2 <= ze;
      __syncwarp();
      if (next) issue(z + 2);
      // ---- negative relations from the neighbours' positive ones ----------
      // lane above (row r - 1), this plane: directions (0, +1, dx)
      const uint32_t u1 = __shfl_up_sync(0xffffffffu, Wd[1], 1), u2 = __shfl_up_sync(0xffffffffu, Wd[2], 1),
                     u3 = __shfl_up_sync(0xffffffffu, Wd[3], 1);
      // previous plane: rows r + 1 (dy = -1), r (dy = 0), r - 1 (dy = +1)
      uint32_t pd[9];
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        pd[t] = __shfl_down_sync(0xffffffffu, Pz[t], 1);        // (1, -1, dx) of row r + 1
        pd[3 + t] = Pz[3 + t];                                  // (1,  0, dx) of row r
        pd[6 + t] = __shfl_up_sync(0xffffffffu, Pz[6 + t], 1);  // (1, +1, dx) of row r - 1
      }
      // output bit i (voxel x0 + i) reads the source voxel x0 + i - dx, bit i - dx + 1
      auto neg = [](uint32_t w, int dx) -> uint32_t { return ~(w >> (1 - dx)); };
      // L[dz][dy][dx] (offset + 1): the neighbour precedes p; bit i = voxel x0 + i
      uint32_t L[3][3][3];
      L[1][1][2] = Wd[0] >> 1;
      L[1][1][0] = neg(Wd[0], +1);
#pragma unroll
      for (int dx = -1; dx <= 1; ++dx) {
        L[1][2][dx + 1] = Wd[2 + dx] >> 1;
        const uint32_t uw = dx < 0 ? u1 : dx == 0 ? u2 : u3;
        L[1][0][1 - dx] = neg(uw, dx);
      }
#pragma unroll
      for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
        for (int dx = -1; dx <= 1; ++dx) {
          const int d = 3 * (dy + 1) + (dx + 1);
          L[2][dy + 1][dx + 1] = Wd[4 + d] >> 1;
          L[0][1 - dy][1 - dx] = neg(pd[d], dx);
        }
      // ---- bit-sliced lower-star count: c + 13 = #squares + #(not edges) + #(not cubes)
      uint32_t in[26];
      int k = 0;
      uint32_t sxy[2][2], sxz[2][2], syz[2][2];
#pragma unroll
      for (int a1 = 0; a1 < 2; ++a1)
#pragma unroll
        for (int b1 = 0; b1 < 2; ++b1) {
          const int A = 2 * a1, B = 2 * b1;
          sxy[a1][b1] = L[1][A][1] & L[1][1][B] & L[1][A][B];
          sxz[a1][b1] = L[A][1][1] & L[1][1][B] & L[A][1][B];
          syz[a1][b1] = L[A][1][1] & L[1][B][1] & L[A][B][1];
          in[k++] = sxy[a1][b1];
          in[k++] = sxz[a1][b1];
          in[k++] = syz[a1][b1];
        }
      in[k++] = ~L[1][1][0]; in[k++] = ~L[1][1][2]; in[k++] = ~L[1][0][1];
      in[k++] = ~L[1][2][1]; in[k++] = ~L[0][1][1]; in[k++] = ~L[2][1][1];
#pragma unroll
      for (int zz = 0; zz < 2; ++zz)
#pragma unroll
        for (int yy = 0; yy < 2; ++yy)
#pragma unroll
          for (int xx = 0; xx < 2; ++xx)
            in[k++] = ~(sxy[yy][xx] & sxz[zz][xx] & syz[zz][yy] & L[2 * zz][2 * yy][2 * xx]);
      uint32_t s8[8], k8[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) fa3(in[3 * t], in[3 * t + 1], in[3 * t + 2], s8[t], k8[t]);
      uint32_t t0, m0, t1, m1, t2, m2, u0, n0;
      fa3(s8[0], s8[1], s8[2], t0, m0);
      fa3(s8[3], s8[4], s8[5], t1, m1);
      fa3(s8[6], s8[7], in[24], t2, m2);
      fa3(t0, t1, t2, u0, n0);
      const uint32_t b0 = u0 ^ in[25], n1 = u0 & in[25];
      uint32_t a0, e0, a1, e1, a2, e2, a3, e3, bb, f0, b1, f1;
      fa3(k8[0], k8[1], k8[2], a0, e0);
      fa3(k8[3], k8[4], k8[5], a1, e1);
      fa3(k8[6], k8[7], m0, a2, e2);
      fa3(m1, m2, n0, a3, e3);
      fa3(a0, a1, a2, bb, f0);
      fa3(bb, a3, n1, b1, f1);
      uint32_t g0, h0, g1, h1, b3, b4;
      fa3(e0, e1, e2, g0, h0);
      fa3(e3, f0, f1, g1, h1);
      const uint32_t b2 = g0 ^ g1, h2 = g0 & g1;
      fa3(h0, h1, h2, b3, b4);
      // c = (c + 13) - 13: add 19 (10011b) modulo 32, 5-bit two's complement
      const uint32_t c0 = b0;
      const uint32_t s0 = ~b0;
      const uint32_t s1 = ~(b1 ^ c0), c1 = b1 | c0;
      const uint32_t s2 = b2 ^ c1, c2 = b2 & c1;
      const uint32_t s3 = b3 ^ c2, c3 = b3 & c2;
      const uint32_t s4 = ~(b4 ^ c3);
      if (rowout) {
        int8_t* cp = sk.coeffs + obase;
#pragma unroll
        for (int g = 0; g < RWX / 4; ++g) {
          const int sh = 4 * g;
          const uint32_t wv = spread4((s0 >> sh) & 15u) | (spread4((s1 >> sh) & 15u) << 1) |
                              (spread4((s2 >> sh) & 15u) << 2) | (spread4((s3 >> sh) & 15u) << 3) |
                              (spread4((s4 >> sh) & 15u) * 0xF0u);
          if (fullx) {
            reinterpret_cast<uint32_t*>(cp)[g] = wv;
          } else {
#pragma unroll
            for (int t = 0; t < 4; ++t)
              if (x0 + 4 * g + t < W) cp[4 * g + t] = (int8_t)(wv >> (8 * t));
          }
        }
      }
#pragma unroll
      for (int d = 0; d < 9; ++d) Pz[d] = Wd[4 + d];
      if (next) convert(z + 2);
    }
  };
  if (sk.fclo) tile(std::true_type{});
  else tile(std::false_type{});

  // a non-finite effective field: redo the tile voxel by voxel with the IEEE
  // compares (out-of-grid neighbours NaN, as coeff3 expects)
  if (__any_sync(0xffffffffu, badhi == 0x7ff00000u)) {
    const double nanv = __longlong_as_double(0x7ff8000000000000ll);
    const int64_t xg = x0 + lane;
    if (lane < RWX && xg < W) {
      for (int64_t z = zs; z < ze; ++z)
        for (int ry = 0; ry < RWOUT; ++ry) {
          const int64_t yg = y0 + ry;
          if (yg >= H) break;
          double nb[3][3][3];
#pragma unroll
          for (int a1 = 0; a1 < 3; ++a1)
#pragma unroll
            for (int b1 = 0; b1 < 3; ++b1)
#pragma unroll
              for (int c1 = 0; c1 < 3; ++c1) {
                const int64_t zz = z + a1 - 1, yy = yg + b1 - 1, xx = xg + c1 - 1;
                const bool in = zz >= 0 && zz < D && yy >= 0 && yy < H && xx >= 0 && xx < W;
                nb[a1][b1][c1] = in ? src.at(n * D * HW + (zz * H + yy) * W + xx, zz, yy, xx) : nanv;
              }
          const int64_t i = ((n * D + z) * H + yg) * W + xg;
          sk.coeffs[i] = (int8_t)coeff3<double>(nb);
          const double dd = nb[1][1][1] - sk.center;
          const float hf = (float)dd;
          sk.fc[i] = hf;
          if (sk.fclo) sk.fclo[i] = (float)(dd - (double)hf);
        }
    }
  }
}
}  // namespace ecc

namespace ecc {
// 2-D soft prepare, row-word form (C3; the default for float32 / float64
// images): the 3-D kernel's scheme on one plane -- a warp per 30 x 28 tile,
// lane = row, 4 positive compares per voxel (sign of the float64
// difference), the 4 negative relations from the lane above and the own
// shifted word, c = 1 - E + S bit-sliced (c + 3 = #squares + #(not edges)).
// 128 x 1024^2: 650 us (per-voxel tile kernel: 740; several tiles per warp
// with the next tile's loads in flight measured 661-726).
template <typename T>
#ifndef ECC_RW2_MINB
#define ECC_RW2_MINB 1   // resident warps per SM the register budget must allow (16: -3 %, 20 / 24: spills, slower)
#endif
__global__ void __launch_bounds__(32, ECC_RW2_MINB) soft_prep2d_rw_kernel(EffSrc<T> src, double center, int8_t* __restrict__ coeffs,
                                                            float* __restrict__ fc, float* __restrict__ fclo,
                                                            int64_t batch, int64_t tiles_x, int64_t tiles_y) {
  __shared__ __align__(16) double eff[RWR * RWLD];
  __shared__ double p0s[RWR];
  src.init();
  if (src.pd) {
    center = src.pd->center;
    if (src.pd->factorized) fclo = nullptr;   // only the direct mode reads the remainders
  }
  const int lane = threadIdx.x;
  const int64_t H = src.H, W = src.W;
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  int64_t r = blockIdx.x;
  const int64_t tile_x = r % tiles_x; r /= tiles_x;
  const int64_t tile_y = r % tiles_y; r /= tiles_y;
  const int64_t n = r;
  if (n >= batch) return;
  const int64_t x0 = tile_x * RWX, y0 = tile_y * RWOUT;
  const T* xb = src.x + n * H * W;
  const int64_t gx = x0 - 2 + lane;
  const bool cok = gx >= 0 && gx < W;
  const double p1u1 = __dmul_rn(EffSrc<T>::crd(cok ? gx : 0, W, src.sW), src.u1);
  for (int row = lane; row < RWR; row += 32) {
    const int64_t gy = y0 - 2 + row;
    p0s[row] = EffSrc<T>::crd(gy >= 0 && gy < H ? gy : 0, H, src.sH);
  }
  // the tile's raw values, all loads in flight at once (interior tiles: a
  // pointer walk without per-row range checks)
  T rv[RWR];
  const bool inner = x0 >= 2 && x0 + RWC - 2 <= W && y0 >= 2 && y0 + RWR - 2 <= H;
  if (inner) {
    const T* rp = xb + (y0 - 2) * W + gx;
#pragma unroll
    for (int row = 0; row < RWR; ++row, rp += W) rv[row] = *rp;
  } else {
#pragma unroll
    for (int row = 0; row < RWR; ++row) {
      const int64_t gy = y0 - 2 + row;
      rv[row] = (cok && gy >= 0 && gy < H) ? xb[gy * W + gx] : T(0);
    }
  }
  __syncwarp();
  double p0r[RWR];   // every row's p0 read before the conversion chain starts
#pragma unroll
  for (int row = 0; row < RWR; ++row) p0r[row] = p0s[row];
  uint32_t badhi = 0;
  if (inner) {
#pragma unroll
    for (int row = 0; row < RWR; ++row) {
      const double dot = __fma_rn(p0r[row], src.u0, p1u1);   // EffSrc::make, 2-D
      const double v = __dadd_rn(__dadd_rn((double)rv[row], __dmul_rn(src.alpha, dot)), 0.0);   // -0 -> +0
      badhi = max(badhi, (uint32_t)__double2hiint(v) & 0x7ff00000u);
      eff[row * RWLD + lane] = v;
    }
  } else {
#pragma unroll
    for (int row = 0; row < RWR; ++row) {
      const int64_t gy = y0 - 2 + row;
      const bool in = cok && gy >= 0 && gy < H;
      const double dot = __fma_rn(p0r[row], src.u0, p1u1);   // EffSrc::make, 2-D
      const double v = __dadd_rn(__dadd_rn((double)rv[row], __dmul_rn(src.alpha, dot)), 0.0);   // -0 -> +0
      if (in) badhi = max(badhi, (uint32_t)__double2hiint(v) & 0x7ff00000u);
      eff[row * RWLD + lane] = in ? v : inf;
    }
  }
  __syncwarp();

  const int sr = lane + 1;
  const int64_t gyl = y0 - 1 + lane;
  const bool rowout = lane >= 1 && lane <= RWOUT && gyl < H;
  const bool fullx = x0 + RWX <= W && (W & 3) == 0 && (((uintptr_t)fc | (uintptr_t)fclo) & 15) == 0 &&
                     ((uintptr_t)coeffs & 3) == 0;   // vector stores: whole, aligned rows
  const int64_t obase = (n * H + gyl) * W + x0;
  const double* a = eff + sr * RWLD;
  const double* b = eff + (sr + 1) * RWLD;
  double av[RWC], bv[RWC];
#pragma unroll
  for (int j = RWC - 1; j >= RWC - 1 - ECC_RW_LA; --j) { av[j] = a[j]; bv[j] = b[j]; }
  uint32_t Wd[4];
  float f4[4], l4[4];
#pragma unroll
  for (int sc = RWC - 2; sc >= 1; --sc) {   // voxel x0 - 2 + sc, bit sc - 1
    if (sc - ECC_RW_LA >= 0) { av[sc - ECC_RW_LA] = a[sc - ECC_RW_LA]; bv[sc - ECC_RW_LA] = b[sc - ECC_RW_LA]; }
    const double p = av[sc];
    const double qv[4] = {av[sc + 1], bv[sc - 1], bv[sc], bv[sc + 1]};
#pragma unroll
    for (int d = 0; d < 4; ++d) Wd[d] = __funnelshift_l((uint32_t)__double2hiint(__dsub_rn(qv[d], p)), Wd[d], 1);
    if (sc >= 2 && sc <= RWX + 1) {
      const int i = sc - 2;
      const double dd = p - center;
      f4[i & 3] = (float)dd;
      if (fclo) l4[i & 3] = (float)(dd - (double)f4[i & 3]);
      if ((i & 3) == 0 && rowout) {
        if (fullx) {
          *reinterpret_cast<float4*>(fc + obase + i) = make_float4(f4[0], f4[1], f4[2], f4[3]);
          if (fclo) *reinterpret_cast<float4*>(fclo + obase + i) = make_float4(l4[0], l4[1], l4[2], l4[3]);
        } else {
#pragma unroll
          for (int t = 0; t < 4; ++t)
            if (x0 + i + t < W) {
              fc[obase + i + t] = f4[t];
              if (fclo) fclo[obase + i + t] = l4[t];
            }
        }
      }
    }
  }
  // negative relations: the lane above (row r - 1) and the own shifted word
  const uint32_t u1 = __shfl_up_sync(0xffffffffu, Wd[1], 1), u2 = __shfl_up_sync(0xffffffffu, Wd[2], 1),
                 u3 = __shfl_up_sync(0xffffffffu, Wd[3], 1);
  auto neg = [](uint32_t w, int dx) -> uint32_t { return ~(w >> (1 - dx)); };
  uint32_t L[3][3];
  L[1][2] = Wd[0] >> 1;
  L[1][0] = neg(Wd[0], +1);
#pragma unroll
  for (int dx = -1; dx <= 1; ++dx) {
    L[2][dx + 1] = Wd[2 + dx] >> 1;
    L[0][1 - dx] = neg(dx < 0 ? u1 : dx == 0 ? u2 : u3, dx);
  }
  // c + 3 = #squares + #(not edges): 8 one-bit words
  const uint32_t i0 = L[0][1] & L[1][0] & L[0][0], i1 = L[0][1] & L[1][2] & L[0][2];
  const uint32_t i2 = L[2][1] & L[1][0] & L[2][0], i3 = L[2][1] & L[1][2] & L[2][2];
  const uint32_t i4 = ~L[0][1], i5 = ~L[2][1], i6 = ~L[1][0], i7 = ~L[1][2];
  uint32_t s0, k0, s1, k1, t0, m0, x1, n0;
  fa3(i0, i1, i2, s0, k0);
  fa3(i3, i4, i5, s1, k1);
  fa3(s0, s1, i6, t0, m0);
  const uint32_t b0 = t0 ^ i7, m1 = t0 & i7;
  fa3(k0, k1, m0, x1, n0);
  const uint32_t b1 = x1 ^ m1, n1 = x1 & m1;
  const uint32_t b2 = n0 ^ n1, b3 = n0 & n1;
  // c = (c + 3) - 3: add 13 (1101b) modulo 16, 4-bit two's complement
  const uint32_t c0 = b0, s0b = ~b0;
  const uint32_t s1b = b1 ^ c0, c1 = b1 & c0;
  const uint32_t s2b = ~(b2 ^ c1), c2 = b2 | c1;
  const uint32_t s3b = ~(b3 ^ c2);
  if (rowout) {
    int8_t* cp = coeffs + obase;
#pragma unroll
    for (int g = 0; g < RWX / 4; ++g) {
      const int sh = 4 * g;
      const uint32_t wv = spread4((s0b >> sh) & 15u) | (spread4((s1b >> sh) & 15u) << 1) |
                          (spread4((s2b >> sh) & 15u) << 2) | (spread4((s3b >> sh) & 15u) * 0xF8u);
      if (fullx) {
        reinterpret_cast<uint32_t*>(cp)[g] = wv;
      } else {
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (x0 + 4 * g + t < W) cp[4 * g + t] = (int8_t)(wv >> (8 * t));
      }
    }
  }
  // a non-finite effective field: the tile voxel by voxel with the IEEE compares
  if (__any_sync(0xffffffffu, badhi == 0x7ff00000u)) {
    const double nanv = __longlong_as_double(0x7ff8000000000000ll);
    const int64_t xg = x0 + lane;
    if (lane < RWX && xg < W) {
      for (int ry = 0; ry < RWOUT; ++ry) {
        const int64_t yg = y0 + ry;
        if (yg >= H) break;
        double nb[3][3];
#pragma unroll
        for (int b1 = 0; b1 < 3; ++b1)
#pragma unroll
          for (int c1 = 0; c1 < 3; ++c1) {
            const int64_t yy = yg + b1 - 1, xx = xg + c1 - 1;
            const bool in = yy >= 0 && yy < H && xx >= 0 && xx < W;
            nb[b1][c1] = in ? src.at(n * H * W + yy * W + xx, 0, yy, xx) : nanv;
          }
        const int64_t i = (n * H + yg) * W + xg;
        coeffs[i] = (int8_t)coeff2<double>(nb);
        const double dd = nb[1][1] - center;
        const float hf = (float)dd;
        fc[i] = hf;
        if (fclo) fclo[i] = (float)(dd - (double)hf);
      }
    }
  }
}
}  // namespace ecc

// p: host parameters, or (pd != nullptr) parameters resident on the device
// (ecc_soft_setup); the values in *p are then placeholders

// the row-word 3-D prepare of output planes [zb, zlim) (the planes zb - 1 and
// zlim are read as halos): one warp per 30 x 28 tile and z-chunk; the chunk
// is shortened until there are ~4 waves of 9 resident warps per SM
static int soft_prep3d_rw_launch(const void* x, int dtype, const int64_t* d3, int64_t batch, const ecc_soft_params* p,
                                 const ecc_soft_params* pd, const SoftPrepSink& sk, int64_t zb, int64_t zlim,
                                 cudaStream_t s) {
  const int64_t tiles_x = (d3[2] + RWX - 1) / RWX, tiles_y = (d3[1] + RWOUT - 1) / RWOUT;
  const int64_t tiles = tiles_x * tiles_y * batch;
  const int64_t depth = zlim - zb;
  if (depth <= 0) return ECC_OK;
  int64_t zc = 64;
  while (zc > 8 && tiles * ((depth + zc - 1) / zc) < (int64_t)num_sms() * 9 * 4) zc >>= 1;
  if (zc > depth) zc = depth;
  const int64_t zchunks = (depth + zc - 1) / zc;
  const int64_t grid = tiles * zchunks;
  if (grid > 0x7fffffff) return set_error(ECC_EINVAL, "grid too large for the 3-D prepare");
  if (dtype == ECC_DTYPE_F32) {
    EffSrc<float> src{(const float*)x, p->alpha, p->u[0], p->u[1], p->u[2], d3[0], d3[1], d3[2], 3,
                      coord_scale(d3[0]), coord_scale(d3[1]), coord_scale(d3[2]), pd};
    soft_prep3d_rw_kernel<float><<<(unsigned)grid, 32, 0, s>>>(src, sk, batch, tiles_x, tiles_y, zc, zchunks, zb, zlim);
  } else {
    EffSrc<double> src{(const double*)x, p->alpha, p->u[0], p->u[1], p->u[2], d3[0], d3[1], d3[2], 3,
                       coord_scale(d3[0]), coord_scale(d3[1]), coord_scale(d3[2]), pd};
    soft_prep3d_rw_kernel<double><<<(unsigned)grid, 32, 0, s>>>(src, sk, batch, tiles_x, tiles_y, zc, zchunks, zb, zlim);
  }
  return check_launch("soft_prep3d_rw_kernel");
}

static int soft_prepare(const void* x, int dtype, int ndim, const int64_t* dims, int64_t batch,
                        const ecc_soft_params* p, const ecc_soft_params* pd, int8_t* coeffs, float* field_c,
                        float* field_lo, void* stream) {
  clear_error();
  int64_t d3[3];
  int rc = dims_to3(ndim, dims, d3);
  if (rc) return rc;
  if (!x || !p || !coeffs || !field_c) return set_error(ECC_EINVAL, "null pointer argument");
  if (batch < 1) return set_error(ECC_EINVAL, "batch must be >= 1");
  SoftPrepSink sk{coeffs, field_c, field_lo, p->center, d3[0], d3[1], d3[2], pd};
  cudaStream_t s = (cudaStream_t)stream;
  if (ndim == 2 && (dtype == ECC_DTYPE_F32 || dtype == ECC_DTYPE_F64) && !variant_generic() &&
      !variant_soft_prep_old() && d3[1] < (1ll << 30) && d3[2] < (1ll << 30)) {
    const int64_t tiles_x = (d3[2] + RWX - 1) / RWX, tiles_y = (d3[1] + RWOUT - 1) / RWOUT;
    const int64_t grid = tiles_x * tiles_y * batch;
    if (grid > 0x7fffffff) return set_error(ECC_EINVAL, "grid too large for the 2-D prepare");
    if (dtype == ECC_DTYPE_F32) {
      EffSrc<float> src{(const float*)x, p->alpha, p->u[0], p->u[1], 0.0, 1, d3[1], d3[2], 2,
                        0.0, coord_scale(d3[1]), coord_scale(d3[2]), pd};
      soft_prep2d_rw_kernel<float><<<(unsigned)grid, 32, 0, s>>>(src, p->center, coeffs, field_c, field_lo, batch,
                                                                  tiles_x, tiles_y);
    } else {
      EffSrc<double> src{(const double*)x, p->alpha, p->u[0], p->u[1], 0.0, 1, d3[1], d3[2], 2,
                         0.0, coord_scale(d3[1]), coord_scale(d3[2]), pd};
      soft_prep2d_rw_kernel<double><<<(unsigned)grid, 32, 0, s>>>(src, p->center, coeffs, field_c, field_lo, batch,
                                                                   tiles_x, tiles_y);
    }
    return check_launch("soft_prep2d_rw_kernel");
  }
  if (ndim == 2 && batch <= 65535 && (dtype == ECC_DTYPE_F32 || dtype == ECC_DTYPE_F64) &&
      !variant_generic()) {
    dim3 grid((unsigned)((d3[2] + 31) / 32), (unsigned)((d3[1] + PREP_TH - 1) / PREP_TH), (unsigned)batch);
    if (grid.y > 65535) goto generic;
    if (dtype == ECC_DTYPE_F32) {
      EffSrc<float> src{(const float*)x, p->alpha, p->u[0], p->u[1], 0.0, 1, d3[1], d3[2], 2,
                        0.0, coord_scale(d3[1]), coord_scale(d3[2]), pd};
      soft_prep2d_kernel<float><<<grid, 256, 0, s>>>(src, p->center, coeffs, field_c, field_lo);
    } else {
      EffSrc<double> src{(const double*)x, p->alpha, p->u[0], p->u[1], 0.0, 1, d3[1], d3[2], 2,
                         0.0, coord_scale(d3[1]), coord_scale(d3[2]), pd};
      soft_prep2d_kernel<double><<<grid, 256, 0, s>>>(src, p->center, coeffs, field_c, field_lo);
    }
    return check_launch("soft_prep2d_kernel");
  }
generic:
  if (ndim == 3 && !variant_generic() && !variant_soft_prep_old() && (dtype == ECC_DTYPE_F32 || dtype == ECC_DTYPE_F64) &&
      d3[1] < (1ll << 30) && d3[2] < (1ll << 30))
    return soft_prep3d_rw_launch(x, dtype, d3, batch, p, pd, sk, 0, d3[0], s);
  if (ndim == 3 && !variant_generic() && (dtype == ECC_DTYPE_F32 || dtype == ECC_DTYPE_F64)) {
    int occ = 0;
    const void* kfn = dtype == ECC_DTYPE_F32 ? (const void*)soft_prep3d_kernel<float>
                                             : (const void*)soft_prep3d_kernel<double>;
    if (int rc2 = sweep_occupancy(kfn, 0, &occ)) return rc2;
    const int64_t max_ctas = (int64_t)num_sms() * occ;
    Geom g = make_geom(d3, batch, 0, max_ctas, 0, d3[0]);
    const int64_t grid = g.items < max_ctas ? g.items : max_ctas;
    if (grid < 1) return ECC_OK;
    if (dtype == ECC_DTYPE_F32) {
      EffSrc<float> src{(const float*)x, p->alpha, p->u[0], p->u[1], p->u[2], d3[0], d3[1], d3[2], ndim,
                        coord_scale(d3[0]), coord_scale(d3[1]), coord_scale(d3[2]), pd};
      soft_prep3d_kernel<float><<<(unsigned)grid, NT, 0, s>>>(src, sk, g);
    } else {
      EffSrc<double> src{(const double*)x, p->alpha, p->u[0], p->u[1], p->u[2], d3[0], d3[1], d3[2], ndim,
                         coord_scale(d3[0]), coord_scale(d3[1]), coord_scale(d3[2]), pd};
      soft_prep3d_kernel<double><<<(unsigned)grid, NT, 0, s>>>(src, sk, g);
    }
    return check_launch("soft_prep3d_kernel");
  }
  if (dtype == ECC_DTYPE_F32) {
    EffSrc<float> src{(const float*)x, p->alpha, p->u[0], p->u[1], p->u[2], d3[0], d3[1], d3[2], ndim,
                      coord_scale(d3[0]), coord_scale(d3[1]), coord_scale(d3[2]), pd};
    return launch_sweep(src, sk, d3, batch, 0, s);
  } else if (dtype == ECC_DTYPE_F64) {
    EffSrc<double> src{(const double*)x, p->alpha, p->u[0], p->u[1], p->u[2], d3[0], d3[1], d3[2], ndim,
                       coord_scale(d3[0]), coord_scale(d3[1]), coord_scale(d3[2]), pd};
    return launch_sweep(src, sk, d3, batch, 0, s);
  }
  return set_error(ECC_EINVAL, "soft path takes float32 or float64 grids");
}

extern "C" int ecc_soft_prepare(const void* x, int dtype, int ndim, const int64_t* dims, int64_t batch,
                                const ecc_soft_params* p, int8_t* coeffs, float* field_c, float* field_lo,
                                void* stream) {
  return soft_prepare(x, dtype, ndim, dims, batch, p, nullptr, coeffs, field_c, field_lo, stream);
}

extern "C" int ecc_soft_prepare_d(const void* x, int dtype, int ndim, const int64_t* dims, int64_t batch,
                                  const ecc_soft_params* params_dev, int8_t* coeffs, float* field_c, float* field_lo,
                                  void* stream) {
  if (!params_dev) return set_error(ECC_EINVAL, "null pointer argument");
  const ecc_soft_params placeholder{1.0, 0.0, {0.0, 0.0, 0.0}, 0.0, 1, 0};
  return soft_prepare(x, dtype, ndim, dims, batch, &placeholder, params_dev, coeffs, field_c, field_lo, stream);
}

extern "C" int ecc_soft_prepare_range_d(const void* x, int dtype, int ndim, const int64_t* dims, int64_t batch,
                                        const ecc_soft_params* params_dev, int8_t* coeffs, float* field_c,
                                        float* field_lo, int64_t plane_begin, int64_t plane_end, void* stream) {
  clear_error();
  int64_t d3[3];
  int rc = dims_to3(ndim, dims, d3);
  if (rc) return rc;
  if (!x || !params_dev || !coeffs || !field_c) return set_error(ECC_EINVAL, "null pointer argument");
  if (ndim != 3 || batch < 1) return set_error(ECC_EINVAL, "plane ranges are for 3-D grids");
  if (dtype != ECC_DTYPE_F32 && dtype != ECC_DTYPE_F64) return set_error(ECC_EINVAL, "soft path takes float32 or float64 grids");
  if (plane_begin < 0 || plane_end > d3[0] || plane_begin > plane_end) return set_error(ECC_EINVAL, "plane range out of bounds");
  if (d3[1] >= (1ll << 30) || d3[2] >= (1ll << 30)) return set_error(ECC_EINVAL, "grid too large for the 3-D prepare");
  const ecc_soft_params placeholder{1.0, 0.0, {0.0, 0.0, 0.0}, 0.0, 1, 0};
  SoftPrepSink sk{coeffs, field_c, field_lo, placeholder.center, d3[0], d3[1], d3[2], params_dev};
  return soft_prep3d_rw_launch(x, dtype, d3, batch, &placeholder, params_dev, sk, plane_begin, plane_end,
                               (cudaStream_t)stream);
}

namespace ecc {
template <typename T>
__global__ void effective_field_kernel(EffSrc<T> src, int64_t total, double* __restrict__ out) {
  const int64_t per = src.D * src.H * src.W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i % per;
    const int64_t z = r / (src.H * src.W);
    r -= z * src.H * src.W;
    const int64_t y = r / src.W, x = r - y * src.W;
    out[i] = src.at(i, z, y, x);
  }
}
}  // namespace ecc

extern "C" int ecc_effective_field(const void* x, int dtype, int ndim, const int64_t* dims, int64_t batch,
                                   double alpha, const double* u, double* out, void* stream) {
  clear_error();
  int64_t d3[3];
  int rc = dims_to3(ndim, dims, d3);
  if (rc) return rc;
  if (!x || !u || !out) return set_error(ECC_EINVAL, "null pointer argument");
  const int64_t total = batch * d3[0] * d3[1] * d3[2];
  int64_t blocks = (total + 255) / 256;
  if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
  if (blocks < 1) return ECC_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (dtype == ECC_DTYPE_F32) {
    EffSrc<float> src{(const float*)x, alpha, u[0], u[1], ndim == 3 ? u[2] : 0.0, d3[0], d3[1], d3[2], ndim,
                      coord_scale(d3[0]), coord_scale(d3[1]), coord_scale(d3[2])};
    effective_field_kernel<float><<<(unsigned)blocks, 256, 0, s>>>(src, total, out);
  } else if (dtype == ECC_DTYPE_F64) {
    EffSrc<double> src{(const double*)x, alpha, u[0], u[1], ndim == 3 ? u[2] : 0.0, d3[0], d3[1], d3[2], ndim,
                       coord_scale(d3[0]), coord_scale(d3[1]), coord_scale(d3[2])};
    effective_field_kernel<double><<<(unsigned)blocks, 256, 0, s>>>(src, total, out);
  } else {
    return set_error(ECC_EINVAL, "effective field takes float32 or float64 grids");
  }
  return check_launch("effective_field_kernel");
}
