// lithogpu C ABI implementation: contexts, band-sparse kernel stacks, tile
// plans, launch orchestration (include/lithogpu.h documents the contract and
// the reference interface each entry point replaces).
#include <cuda_runtime.h>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/lithogpu.h"
#include "contour_kernels.cuh"
#include "raster_kernels.cuh"
#include "socs_kernels.cuh"
#include "util_kernels.cuh"
#include "socs_fast.h"
#include <cstdlib>
#include <type_traits>

namespace {

thread_local std::string g_last_error;

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define LG_CUDA(call)                                                                      \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      throw std::runtime_error(std::string("CUDA error: ") + cudaGetErrorString(e_) + " (" + \
                               #call + ")");                                               \
  } while (0)

template <typename Fn>
lithogpu_status guarded(Fn&& fn) {
  try {
    fn();
    g_last_error.clear();
    return LITHOGPU_OK;
  } catch (const UsageError& e) {
    g_last_error = e.what();
    return LITHOGPU_ERR_USAGE;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return LITHOGPU_ERR_DOMAIN;
  } catch (...) {
    g_last_error = "unknown error";
    return LITHOGPU_ERR_DOMAIN;
  }
}

// LITHOGPU_UNFUSED=1: the two-pass forms of the fused column kernels (A/B timing)
bool unfused() {
  static const bool v = [] {
    const char* e = std::getenv("LITHOGPU_UNFUSED");
    return e && e[0] == '1';
  }();
  return v;
}

void require(bool ok, const char* msg) {
  if (!ok) throw UsageError(msg);
}

size_t dtype_size(lithogpu_dtype d) {
  switch (d) {
    case LITHOGPU_F32:
      return 4;
    case LITHOGPU_F64:
      return 8;
    case LITHOGPU_U8:
      return 1;
  }
  throw UsageError("unknown dtype");
}

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  void ensure(size_t b) {
    if (b <= bytes) return;
    release();
    if (b == 0) return;
    LG_CUDA(cudaMalloc(&p, b));
    bytes = b;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// device tables of one generic-path transform length (fft.cuh; make_tab)
struct TabBufs {
  DevBuf tw, twM, chirp, bhat;
  bool built = false;
};

// Host -> device upload of a freshly built table that returns only when the
// bytes are in device memory.  A plain cudaMemcpy from pageable memory may
// return once the data is staged, before the DMA lands; the tables are then
// read by kernels on the context's (non-blocking) stream, which does not
// order against the legacy stream — so wait for the legacy stream here.
inline void h2d_blocking(void* dst, const void* src, size_t bytes) {
  LG_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
  LG_CUDA(cudaStreamSynchronize(cudaStreamLegacy));
}

// Non-owning view of a device table (Plan::set_sigma's per-sigma tables).
struct TabView {
  void* p = nullptr;
  template <typename U>
  U* as() const {
    return static_cast<U*>(p);
  }
};
struct GTab {
  DevBuf x, y;
};

// Stream-ordered pool allocation (cudaMallocAsync) for per-call scratch of the
// non-graph entry points (rasterization, contours, EPE, evaluate_epe): no
// cudaMalloc / cudaFree (tens of microseconds to milliseconds) on every call.
struct PoolBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t s = nullptr;
  PoolBuf() = default;
  PoolBuf(const PoolBuf&) = delete;
  PoolBuf& operator=(const PoolBuf&) = delete;
  ~PoolBuf() { release(); }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    bytes = 0;
  }
  void ensure(size_t b, cudaStream_t st) {
    if (b <= bytes && st == s) return;
    release();
    s = st;
    if (b == 0) return;
    static const bool pool_init = [] {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        unsigned long long keep = ~0ull;  // keep freed blocks for reuse
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
      return true;
    }();
    (void)pool_init;
    LG_CUDA(cudaMallocAsync(&p, b, s));
    bytes = b;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

}  // namespace

struct lithogpu_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  long long launches = 0;
  // pinned double buffer for tile I/O (lithogpu_write_aimg)
  void* pinned[2] = {nullptr, nullptr};
  size_t pinned_bytes = 0;
  void pinned_ensure(size_t b) {
    if (b <= pinned_bytes) return;
    for (auto& p : pinned) {
      if (p) cudaFreeHost(p);
      p = nullptr;
    }
    pinned_bytes = 0;
    for (auto& p : pinned) LG_CUDA(cudaMallocHost(&p, b));
    pinned_bytes = b;
  }

  std::vector<std::unique_ptr<DevBuf>> scratch;  // staging pool (per call slots)
  // lithogpu_fft2 transform tables, cached per (length, real type size);
  // immutable once built, so later calls never rewrite a table in use
  std::map<std::pair<int, int>, std::unique_ptr<TabBufs>> fft_tabs;
  DevBuf raster_tmp;
  std::unordered_map<const void*, int> smem_set;
  // optional per-launch CUDA-event timing (lithogpu_ctx_set_profiling)
  bool profiling = false;
  struct Rec {
    const char* name;
    cudaEvent_t a, b;
  };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  struct Agg {
    long long n = 0;
    double ms = 0;
  };
  std::unordered_map<std::string, Agg> agg;

  cudaEvent_t ev() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    LG_CUDA(cudaEventCreate(&e));
    return e;
  }
  void prof_begin(const char* name) {
    if (!profiling) return;
    Rec r{name, ev(), ev()};
    LG_CUDA(cudaEventRecord(r.a, stream));
    recs.push_back(r);
  }
  void prof_end() {
    if (!profiling || recs.empty()) return;
    LG_CUDA(cudaEventRecord(recs.back().b, stream));
  }
  void prof_collect() {
    if (recs.empty()) return;
    LG_CUDA(cudaStreamSynchronize(stream));
    for (auto& r : recs) {
      float ms = 0;
      LG_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
      Agg& g = agg[r.name];
      g.n++;
      g.ms += ms;
      pool.push_back(r.a);
      pool.push_back(r.b);
    }
    recs.clear();
  }
  ~lithogpu_ctx() {
    for (auto& r : recs) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    for (auto e : pool) cudaEventDestroy(e);
    for (auto& p : pinned)
      if (p) cudaFreeHost(p);
  }

  DevBuf& slot(size_t i) {
    while (scratch.size() <= i) scratch.emplace_back(new DevBuf);
    return *scratch[i];
  }
  void activate() const { LG_CUDA(cudaSetDevice(device)); }
  void check_launch() {
    ++launches;
    LG_CUDA(cudaGetLastError());
  }
  template <typename K>
  void smem_attr(K kern, size_t bytes) {
    const void* key = reinterpret_cast<const void*>(kern);
    auto it = smem_set.find(key);
    if (it != smem_set.end() && size_t(it->second) >= bytes) return;
    if (bytes > 48 * 1024)
      LG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
    smem_set[key] = int(bytes);
  }
};

namespace {

// ---- host <-> device staging with dtype conversion ------------------------
template <typename A, typename B>
void convert_dev(lithogpu_ctx* ctx, const A* in, B* out, size_t n) {
  if (n == 0) return;
  const int blocks = int(std::min<size_t>((n + 255) / 256, 148 * 16));
  lg::k_convert<A, B><<<blocks, 256, 0, ctx->stream>>>(in, out, n);
  ctx->check_launch();
}

template <typename B>
void convert_from(lithogpu_ctx* ctx, const void* in, lithogpu_dtype dt, B* out, size_t n) {
  switch (dt) {
    case LITHOGPU_F32:
      convert_dev(ctx, static_cast<const float*>(in), out, n);
      break;
    case LITHOGPU_F64:
      convert_dev(ctx, static_cast<const double*>(in), out, n);
      break;
    case LITHOGPU_U8:
      convert_dev(ctx, static_cast<const unsigned char*>(in), out, n);
      break;
  }
}

template <typename A>
void convert_to(lithogpu_ctx* ctx, const A* in, void* out, lithogpu_dtype dt, size_t n) {
  switch (dt) {
    case LITHOGPU_F32:
      convert_dev(ctx, in, static_cast<float*>(out), n);
      break;
    case LITHOGPU_F64:
      convert_dev(ctx, in, static_cast<double*>(out), n);
      break;
    case LITHOGPU_U8:
      convert_dev(ctx, in, static_cast<unsigned char*>(out), n);
      break;
  }
}

// Input of n elements of dtype dt at user pointer p -> device T array.
// Uses scratch slots [s, s+1].
template <typename T>
const T* stage_in(lithogpu_ctx* ctx, const void* p, lithogpu_dtype dt, size_t n, int s) {
  const bool dev = is_device_ptr(p);
  const size_t bytes = n * dtype_size(dt);
  const void* dsrc = p;
  if (!dev) {
    DevBuf& raw = ctx->slot(s);
    raw.ensure(bytes);
    LG_CUDA(cudaMemcpyAsync(raw.p, p, bytes, cudaMemcpyHostToDevice, ctx->stream));
    dsrc = raw.p;
  }
  const bool same = (sizeof(T) == 4 && dt == LITHOGPU_F32) || (sizeof(T) == 8 && dt == LITHOGPU_F64);
  if (same) return static_cast<const T*>(dsrc);
  DevBuf& cv = ctx->slot(s + 1);
  cv.ensure(n * sizeof(T));
  convert_from(ctx, dsrc, dt, cv.as<T>(), n);
  return cv.as<T>();
}

// Output: returns a device T buffer to compute into; finish_out() moves it to p.
template <typename T>
struct OutStage {
  lithogpu_ctx* ctx;
  void* user;
  lithogpu_dtype dt;
  size_t n;
  bool dev;
  T* work = nullptr;
  int slot;
  OutStage(lithogpu_ctx* c, void* p, lithogpu_dtype d, size_t n_, int s)
      : ctx(c), user(p), dt(d), n(n_), slot(s) {
    if (!p) return;
    dev = is_device_ptr(p);
    const bool same = (sizeof(T) == 4 && dt == LITHOGPU_F32) || (sizeof(T) == 8 && dt == LITHOGPU_F64);
    if (dev && same) {
      work = static_cast<T*>(p);
    } else {
      DevBuf& b = ctx->slot(slot);
      b.ensure(n * sizeof(T));
      work = b.as<T>();
    }
  }
  // returns true if a host copy was queued (caller must sync)
  bool finish() {
    if (!user) return false;
    const bool same = (sizeof(T) == 4 && dt == LITHOGPU_F32) || (sizeof(T) == 8 && dt == LITHOGPU_F64);
    if (dev) {
      if (!same) convert_to(ctx, work, user, dt, n);
      return false;
    }
    const void* src = work;
    if (!same) {
      DevBuf& b = ctx->slot(slot + 1);
      b.ensure(n * dtype_size(dt));
      convert_to(ctx, work, b.p, dt, n);
      src = b.p;
    }
    LG_CUDA(cudaMemcpyAsync(user, src, n * dtype_size(dt), cudaMemcpyDeviceToHost, ctx->stream));
    return true;
  }
};

// ---- geometry --------------------------------------------------------------
// Decimation d: the largest divisor of N whose grid n = N/d still holds the
// intensity band without aliasing (n >= 2P+1) and keeps n >= 32 (fast-path
// transform range).  No such d -> full band on the N grid.
lg::AxisGeom make_axis(int N, int lo, int hi, bool mixed = false) {
  lg::AxisGeom a{};
  a.N = N;
  a.lo = lo;
  a.hi = hi;
  a.B = hi - lo + 1;
  a.Pm = std::max(-lo, hi);
  const int P0 = a.B - 1;
  if (mixed) {
    // fp32 fast path: any supported FFT length n >= 2P+1 works (the samples
    // s N/n of the trigonometric polynomial need not be integer pixels)
    const bool pow2_only = std::getenv("LITHOGPU_POW2_SUBGRID") != nullptr;
    for (int n : lg::kFastLens) {
      if (n > N) break;
      if (pow2_only && !lg::is_pow2(n)) continue;
      if (n >= 2 * P0 + 1 && n >= std::min(N, 32)) {
        a.d = N % n == 0 ? N / n : 0;  // informational (0: fractional decimation)
        a.n = n;
        a.full = 0;
        a.P = P0;
        a.nb2 = 2 * P0 + 1;
        return a;
      }
    }
  }
  // generic path: n need not divide N either (samples at s N / n); every
  // length is O(n log n) (fft.cuh), so take the smallest power of two (radix-16
  // register Stockham) or else the smallest 7-smooth length (mixed radix)
  // >= max(2P+1, min(N, 32)) that fits in N.  LITHOGPU_DIVISOR_SUBGRID=1
  // keeps the divisor rule below (A/B).
  if (!std::getenv("LITHOGPU_DIVISOR_SUBGRID")) {
    const int m = std::max(2 * P0 + 1, std::min(N, 32));
    int n = 16;
    while (n < m) n <<= 1;
    if (n > N) {
      n = m;
      while (lg::fft_kind(n) == lg::kFftBluestein) ++n;
    }
    if (n < N) {
      a.d = N % n == 0 ? N / n : 0;
      a.n = n;
      a.full = 0;
      a.P = P0;
      a.nb2 = 2 * P0 + 1;
      return a;
    }
  }
  int best = 0;
  for (int d = N; d >= 1; --d) {
    if (N % d) continue;
    const int n = N / d;
    if (n >= 2 * P0 + 1 && n >= std::min(N, 32)) {
      best = d;
      break;
    }
  }
  if (best) {
    a.d = best;
    a.n = N / best;
    a.full = 0;
    a.P = P0;
    a.nb2 = 2 * P0 + 1;
  } else {
    a.d = 1;
    a.n = N;
    a.full = 1;
    a.P = N / 2;
    a.nb2 = N;
  }
  return a;
}

// exp(-2 pi i m / L), m < L, fp64 then rounded
template <typename T>
void make_twiddles(int L, DevBuf& buf) {
  std::vector<lg::cx<T>> h(L);
  for (int m = 0; m < L; ++m) {
    // reduce the angle exactly: m/L in [0,1)
    const double a = 2.0 * M_PI * double(m) / double(L);
    h[m].x = T(std::cos(a));
    h[m].y = T(-std::sin(a));
  }
  buf.ensure(sizeof(lg::cx<T>) * L);
  h2d_blocking(buf.p, h.data(), sizeof(lg::cx<T>) * L);
}

// Bluestein chirp w_n = exp(-i pi n^2 / L): n^2 reduced mod 2L in integers so
// the angle is exact before the fp64 sin/cos
static std::complex<double> chirp_at(long long n, int L) {
  const long long m = (n % (2LL * L)) * (n % (2LL * L)) % (2LL * L);
  const double a = M_PI * double(m) / double(L);
  return {std::cos(a), -std::sin(a)};
}

// in-place fp64 radix-2 FFT (host, table setup only), sign -1
static void host_fft_pow2(std::vector<std::complex<double>>& a) {
  const int n = int(a.size());
  for (int i = 1, j = 0; i < n; ++i) {
    int bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) std::swap(a[i], a[j]);
  }
  for (int len = 2; len <= n; len <<= 1) {
    for (int i = 0; i < n; i += len)
      for (int k = 0; k < len / 2; ++k) {
        const double ang = -2.0 * M_PI * double(k) / double(len);
        const std::complex<double> w(std::cos(ang), std::sin(ang));
        const std::complex<double> u = a[i + k], v = a[i + k + len / 2] * w;
        a[i + k] = u + v;
        a[i + k + len / 2] = u - v;
      }
  }
}

// reuse: the buffers already hold this length's tables (only the view is
// rebuilt)
template <typename T>
lg::Tab<T> make_tab(int L, TabBufs& b, bool reuse = false) {
  using C = lg::cx<T>;
  if (!reuse) make_twiddles<T>(L, b.tw);
  lg::Tab<T> t{};
  t.tw = b.tw.as<C>();
  t.L = L;
  t.kind = lg::fft_kind(L);
  t.log2L = t.kind == lg::kFftPow2 ? lg::ilog2(L) : -1;
  t.rad = lg::mixed_radices(L, t.nst);
  t.M = lg::blue_len(L);
  if (t.M) {
    const int M = t.M;
    t.log2M = lg::ilog2(M);
    t.twM = b.twM.as<C>();
    t.chirp = b.chirp.as<C>();
    t.bhat = b.bhat.as<C>();
    if (reuse) return t;
    make_twiddles<T>(M, b.twM);
    std::vector<C> ch(L), bh(M);
    std::vector<std::complex<double>> f(M, 0.0);
    for (int n = 0; n < L; ++n) {
      const std::complex<double> w = chirp_at(n, L);
      ch[n].x = T(w.real());
      ch[n].y = T(w.imag());
      f[n] = std::conj(w);                 // b_m = conj(w_m), m >= 0
      if (n) f[M - n] = std::conj(w);      // and m < 0 (wrapped)
    }
    host_fft_pow2(f);
    for (int k = 0; k < M; ++k) {
      bh[k].x = T(f[k].real());
      bh[k].y = T(f[k].imag());
    }
    b.chirp.ensure(sizeof(C) * L);
    h2d_blocking(b.chirp.p, ch.data(), sizeof(C) * L);
    b.bhat.ensure(sizeof(C) * M);
    h2d_blocking(b.bhat.p, bh.data(), sizeof(C) * M);
    t.twM = b.twM.as<C>();
    t.chirp = b.chirp.as<C>();
    t.bhat = b.bhat.as<C>();
  }
  return t;
}

// 1-D DFT of the reference's truncated unit-sum Gaussian on an N-grid
// (imaging.cpp:292-305: radius min(N/2, ceil(6 sigma_px)+1), unit sum; the
// 2-D kernel is the product of the two axes' 1-D kernels).
std::vector<double> gauss_taps(int N, double sigma_px, int& r) {
  r = std::min(N / 2, int(std::ceil(6 * sigma_px)) + 1);
  std::vector<double> g(2 * r + 1);
  double s = 0;
  for (int d = -r; d <= r; ++d) {
    g[d + r] = std::exp(-0.5 * double(d) * double(d) / (sigma_px * sigma_px));
    s += g[d + r];
  }
  for (auto& v : g) v /= s;
  return g;
}

double gauss_hat(int N, const std::vector<double>& taps, int r, int p) {
  double acc = 0;
  for (int d = -r; d <= r; ++d) acc += taps[d + r] * std::cos(2.0 * M_PI * double(p) * d / N);
  return acc;
}

struct Launch {
  int G, RPC, block;
  size_t smem;
};

template <typename T>
Launch launch_cfg(int LA, int LB, int target = 256) {
  Launch l;
  l.G = lg::group_threads<T>(LA, LB);
  l.RPC = std::max(1, target / l.G);
  l.block = l.RPC * l.G;
  l.smem = size_t(l.RPC) * lg::group_elems<T>(LA, LB) * sizeof(T);
  // one row group must fit a CTA's shared memory (227 KB on sm_100); very long
  // Bluestein lengths in fp64 do not
  if (l.smem > 227u * 1024u)
    throw std::runtime_error("transform length " + std::to_string(std::max(LA, LB)) + " needs " +
                             std::to_string(l.smem / 1024) + " KB of shared memory per row group (" +
                             (sizeof(T) == 8 ? "fp64" : "fp32") + " generic path; limit 227 KB)");
  return l;
}

int cdiv(long long a, long long b) { return int((a + b - 1) / b); }

struct PlanBase {
  virtual ~PlanBase() = default;
};

}  // namespace

// ============================================================================
// Plan: one tile geometry + F x K kernel stacks, templated on the real type
// ============================================================================
template <typename T>
struct Plan : PlanBase {
  using C = lg::cx<T>;
  lithogpu_ctx* ctx;
  lg::Geo<T> g{};
  lithogpu_grid grid{};
  int F = 0, K = 0;
  TabBufs twNx, twNy, twnx, twny;
  DevBuf H, wk;
  // Gaussian transfer cache
  // Gaussian band tables, one immutable device table per resist sigma: a
  // solver or image() call with another sigma never overwrites a table that
  // queued work (or a captured ILT graph) still reads.
  std::map<double, std::unique_ptr<GTab>> gtabs;
  double gsig = -1.0;
  TabView gxh, gyb;
  // work buffers (sized for `cap` tiles)
  int cap = 0;
  DevBuf Mr, Mhat, Tb, Ir, Ic, Rc, Dr, Wc, U, Acc, Gc, costrow, gmaxrow;
  // the ILT whose next-iteration mask rows currently sit in Mr (fused into
  // grad_rows); any other producer of Mr clears it
  const void* mr_owner = nullptr;
  long long gen = 0;  // bumped whenever work buffers are reallocated
  long long s_Mr, s_Mhat, s_T, s_Ir, s_C, s_Dr, s_Wc, s_U, s_Acc, s_Gc, s_cr, s_gm;
  // fp32 fast path (power-of-two tiles, register FFT kernels of socs_fast.cuh)
  bool fast = false;
  lg::FGeo fg{};
  DevBuf ftNx, ftNy, ftnx, ftny, Wsub, Ih, Rh, Wh, Eb, Ht;
  long long s_Wsub = 0, s_band = 0, s_E = 0;
  // ILT: keep the coherent fields E_fk from the forward rows for the adjoint
  // rows (saves one n-point IFFT per (row, kernel)).  Measured faster than
  // recomputing even when they stream through HBM (C4 +9 %, C5 +7 %), so they
  // are kept up to 8 GiB per launch
  bool store_E = false;

  Plan(lithogpu_ctx* c, const lithogpu_grid& gr, int F_, int K_, const double* weights, int S,
       const int32_t* support, const double* values)
      : ctx(c), grid(gr), F(F_), K(K_) {
    const int Nx = gr.nx, Ny = gr.ny;
    // canonical signed support indices and band extent
    std::vector<int> kx(S), ky(S);
    int lox = 1 << 30, hix = -(1 << 30), loy = lox, hiy = hix;
    for (int s = 0; s < S; ++s) {
      int a = ((support[2 * s] % Nx) + Nx) % Nx, b = ((support[2 * s + 1] % Ny) + Ny) % Ny;
      if (a > Nx / 2) a -= Nx;
      if (b > Ny / 2) b -= Ny;
      kx[s] = a;
      ky[s] = b;
      lox = std::min(lox, a);
      hix = std::max(hix, a);
      loy = std::min(loy, b);
      hiy = std::max(hiy, b);
    }
    const bool mixed = std::is_same<T, float>::value && lg::fast_len_ok(Nx) && lg::fast_len_ok(Ny) &&
                       !std::getenv("LITHOGPU_GENERIC");
    g.ax = make_axis(Nx, lox, hix, mixed);
    g.ay = make_axis(Ny, loy, hiy, mixed);
    g.F = F;
    g.K = K;
    auto tab = [&](int L, TabBufs& b) { return make_tab<T>(L, b); };
    g.tNx = tab(Nx, twNx);
    g.tNy = tab(Ny, twNy);
    g.tnx = tab(g.ax.n, twnx);
    g.tny = tab(g.ay.n, twny);
    // dense band kernels [F*K][By][Bx]
    const int Bx = g.ax.B, By = g.ay.B;
    std::vector<C> h(size_t(F) * K * By * Bx);
    for (auto& v : h) v.x = v.y = T(0);
    for (int fk = 0; fk < F * K; ++fk)
      for (int s = 0; s < S; ++s) {
        C& dst = h[(size_t(fk) * By + (ky[s] - loy)) * Bx + (kx[s] - lox)];
        dst.x = T(values[2 * (size_t(fk) * S + s)]);
        dst.y = T(values[2 * (size_t(fk) * S + s) + 1]);
      }
    H.ensure(h.size() * sizeof(C));
    h2d_blocking(H.p, h.data(), h.size() * sizeof(C));
    std::vector<T> w(size_t(F) * K);
    for (size_t i = 0; i < w.size(); ++i) w[i] = T(weights[i]);
    wk.ensure(w.size() * sizeof(T));
    h2d_blocking(wk.p, w.data(), w.size() * sizeof(T));
    // strides (elements)
    const auto& ax = g.ax;
    const auto& ay = g.ay;
    s_Mr = (long long)(ax.Pm + 1) * Ny;
    s_Mhat = (long long)By * Bx;
    s_T = (long long)F * K * ay.n * Bx;
    s_Ir = (long long)F * (ax.P + 1) * ay.n;
    s_C = (long long)F * Ny * (ax.P + 1);
    s_Dr = (long long)F * (ax.P + 1) * Ny;
    s_Wc = (long long)F * ay.n * (ax.P + 1);
    s_U = (long long)F * K * Bx * ay.n;
    s_Acc = (long long)F * K * By * Bx;  // fast path keeps per-(f,k) partials
    s_Gc = (long long)Ny * (ax.Pm + 1);
    s_cr = (long long)F * Ny;
    s_gm = (long long)(Ny + 1) / 2;
    if constexpr (std::is_same<T, float>::value) {
      auto ok = [](int L) { return lg::fast_len_ok(L); };
      fast = ok(Nx) && ok(Ny) && ok(ax.n) && ok(ay.n) && !std::getenv("LITHOGPU_GENERIC");
      if (fast) {
        fg.ax = ax;
        fg.tld = (Bx + 1) & ~1;
        s_T = (long long)F * K * ay.n * fg.tld;
        fg.ay = ay;
        fg.F = F;
        fg.K = K;
        auto table = [](int len, DevBuf& b) {
          std::vector<lg::C32> h(std::max(1, lg::fast_tw_len(len)));
          lg::fast_fill_twiddles(len, h.data());
          b.ensure(h.size() * sizeof(lg::C32));
          h2d_blocking(b.p, h.data(), h.size() * sizeof(lg::C32));
          return b.as<lg::C32>();
        };
        // focus stacks computed on the fast path (mirror stacks merged)
        merge_foci(weights, S, kx, ky, values);
        const int Fc = fg.F;
        // column-major copy of the kernel band for the fast column kernels
        {
          std::vector<lg::C32> ht(size_t(Fc) * K * Bx * By);
          for (int r = 0; r < Fc; ++r)
            for (int k = 0; k < K; ++k)
              for (int jy = 0; jy < By; ++jy)
                for (int jx = 0; jx < Bx; ++jx) {
                  const C& src = h[((size_t(rep_src[r]) * K + k) * By + jy) * Bx + jx];
                  ht[((size_t(r) * K + k) * Bx + jx) * By + jy] = lg::C32{float(src.x), float(src.y)};
                }
          Ht.ensure(ht.size() * sizeof(lg::C32));
          h2d_blocking(Ht.p, ht.data(), ht.size() * sizeof(lg::C32));
          std::vector<float> wf(size_t(Fc) * K);
          for (int r = 0; r < Fc; ++r)
            for (int k = 0; k < K; ++k) wf[size_t(r) * K + k] = float(weights[size_t(rep_src[r]) * K + k]);
          wkf.ensure(wf.size() * sizeof(float));
          h2d_blocking(wkf.p, wf.data(), wf.size() * sizeof(float));
        }
        fg.twNx = table(Nx, ftNx);
        fg.twNy = table(Ny, ftNy);
        fg.twnx = table(ax.n, ftnx);
        fg.twny = table(ay.n, ftny);
        {
          std::vector<double> cw(size_t(Fc) * K), cv(size_t(Fc) * K * S * 2);
          for (int r = 0; r < Fc; ++r) {
            std::copy(weights + size_t(rep_src[r]) * K, weights + size_t(rep_src[r] + 1) * K, cw.begin() + size_t(r) * K);
            std::copy(values + size_t(rep_src[r]) * K * S * 2, values + size_t(rep_src[r] + 1) * K * S * 2,
                      cv.begin() + size_t(r) * K * S * 2);
          }
          make_pairs(cw.data(), S, kx, ky, cv.data());
        }
        s_Wsub = (long long)F * ay.n * ax.n;
        s_band = (long long)F * ay.nb2 * (ax.P + 1);
        s_E = (long long)F * fg.K * ay.n * ax.n;
        const long long npairs = (Ny + 1) / 2;
        const long long wpg = std::max(1, lg::fast_tpr(Nx) / 32);
        s_cr = std::max(s_cr, F * npairs * wpg);
        s_gm = std::max(s_gm, npairs * wpg);
      }
    }
  }

  // ---- kernel pairing (fast path) ----------------------------
  // A kernel whose band is Hermitian-symmetric, H(-q) = conj(H(q)), gives a
  // REAL coherent field E = IFFT(M^ H) for a real mask (M^ is Hermitian); an
  // anti-Hermitian one becomes Hermitian after a -i rotation (|E|^2 and the
  // adjoint are unchanged).  When every kernel qualifies (in-focus stacks of a
  // point-symmetric source: real TCC), kernels a, b are packed into one
  // complex kernel H_a + i H_b: one transform per PAIR yields E_a + i E_b,
  // |E_a|^2 w_a + |E_b|^2 w_b = w_a Re^2 + w_b Im^2, and the adjoint of the
  // pair is exact with the band weight conj(w_a H_a + i w_b H_b) because only
  // the Hermitian part of the accumulated spectrum reaches the real gradient.
  bool paired = false;
  DevBuf Hadj, wRe, wIm, wOne;
  void make_pairs(const double* weights, int S, const std::vector<int>& kx, const std::vector<int>& ky,
                  const double* values) {
    const int Bx = g.ax.B, By = g.ay.B, lox = g.ax.lo, loy = g.ay.lo, F = fg.F;
    if (std::getenv("LITHOGPU_NO_PAIRS") || K < 2 || g.ax.lo != -g.ax.hi || g.ay.lo != -g.ay.hi) return;
    std::vector<int> at(size_t(Bx) * By, -1);  // band slot -> support index
    for (int s2 = 0; s2 < S; ++s2) at[size_t(ky[s2] - loy) * Bx + (kx[s2] - lox)] = s2;
    std::vector<int> mir(S);
    for (int s2 = 0; s2 < S; ++s2) {
      mir[s2] = at[size_t(-ky[s2] - loy) * Bx + (-kx[s2] - lox)];
      if (mir[s2] < 0) return;  // support not point-symmetric
    }
    // per kernel: 0 Hermitian, 1 anti-Hermitian (rotate by -i), -1 neither
    std::vector<int> rot(size_t(F) * K, 0);
    std::vector<char> stack_ok(F, 1);
    for (int fk = 0; fk < F * K; ++fk) {
      const double* v = values + 2 * size_t(fk) * S;
      double hmax = 0, eh = 0, ea = 0;
      for (int s2 = 0; s2 < S; ++s2) {
        const double re = v[2 * s2], im = v[2 * s2 + 1], mr = v[2 * mir[s2]], mi = v[2 * mir[s2] + 1];
        hmax = std::max(hmax, std::hypot(re, im));
        eh = std::max(eh, std::hypot(mr - re, mi + im));  // H(-q) - conj(H(q))
        ea = std::max(ea, std::hypot(mr + re, mi - im));  // H(-q) + conj(H(q))
      }
      rot[fk] = eh <= 1e-9 * hmax ? 0 : (ea <= 1e-9 * hmax ? 1 : -1);
      if (rot[fk] < 0) stack_ok[fk / K] = 0;
    }
    const int npair = int(std::count(stack_ok.begin(), stack_ok.end(), 1));
    if (npair == 0) return;
    // all stacks pair: Kp slots per stack.  Mixed (e.g. the in-focus stack of a
    // through-focus set): K slots per stack; a pairing stack uses its first
    // Kp slots and leaves the rest empty (skipped by every kernel via
    // FGeo::slot_on), the others keep one kernel per slot with w_a = w_b = w
    // (w Re^2 + w Im^2 = w |E|^2, adjoint band w H: the per-kernel path).
    const bool mixed = npair < F;
    const int Kp = (K + 1) / 2, KS = mixed ? K : Kp;
    std::vector<lg::C32> hc(size_t(F) * KS * Bx * By, lg::C32{0.f, 0.f}), ha(hc.size(), lg::C32{0.f, 0.f});
    std::vector<float> wr(size_t(F) * KS, 0.f), wi(wr.size(), 0.f), one(wr.size(), 1.f);
    std::vector<int> on(wr.size(), 0);
    for (int f = 0; f < F; ++f) {
      auto kval = [&](int k, int s2, bool rotate, double& re, double& im) {
        re = im = 0.0;
        if (k >= K) return;
        const double* v = values + 2 * (size_t(f * K + k) * S + s2);
        if (rotate && rot[size_t(f) * K + k] == 1) {  // -i (x + i y) = y - i x
          re = v[1];
          im = -v[0];
        } else {
          re = v[0];
          im = v[1];
        }
      };
      const int nslot = stack_ok[f] ? Kp : K;
      for (int sl = 0; sl < nslot; ++sl) {
        const int a = stack_ok[f] ? 2 * sl : sl, b = stack_ok[f] ? 2 * sl + 1 : -1;
        const double wa = weights[size_t(f) * K + a];
        const double wb = b >= 0 ? (b < K ? weights[size_t(f) * K + b] : 0.0) : wa;
        const size_t si = size_t(f) * KS + sl;
        wr[si] = float(wa);
        wi[si] = float(wb);
        on[si] = (wa != 0.0 || (b >= 0 && wb != 0.0)) ? 1 : 0;
        for (int s2 = 0; s2 < S; ++s2) {
          const size_t o = ((size_t(f) * KS + sl) * Bx + (kx[s2] - lox)) * By + (ky[s2] - loy);
          double ar, ai;
          kval(a, s2, stack_ok[f] != 0, ar, ai);
          if (b >= 0) {  // pair: H_a + i H_b, adjoint w_a H_a + i w_b H_b
            double br, bi;
            kval(b, s2, true, br, bi);
            hc[o] = lg::C32{float(ar - bi), float(ai + br)};
            ha[o] = lg::C32{float(wa * ar - wb * bi), float(wa * ai + wb * br)};
          } else {  // single kernel in its own slot
            hc[o] = lg::C32{float(ar), float(ai)};
            ha[o] = lg::C32{float(wa * ar), float(wa * ai)};
          }
        }
      }
    }
    auto up = [](DevBuf& d, const void* h, size_t bytes) {
      d.ensure(bytes);
      h2d_blocking(d.p, h, bytes);
    };
    up(Ht, hc.data(), hc.size() * sizeof(lg::C32));
    up(Hadj, ha.data(), ha.size() * sizeof(lg::C32));
    up(wRe, wr.data(), wr.size() * sizeof(float));
    up(wIm, wi.data(), wi.size() * sizeof(float));
    up(wOne, one.data(), one.size() * sizeof(float));
    if (mixed) {
      up(slotOn, on.data(), on.size() * sizeof(int));
      fg.slot_on = slotOn.as<int>();
    }
    fg.K = KS;
    paired = true;
  }
  DevBuf slotOn;

  // weights / adjoint band of the fast kernels (paired or per kernel)
  const float* fw1() const { return paired ? wRe.as<float>() : wkf.as<float>(); }
  const float* fw2() const { return paired ? wIm.as<float>() : nullptr; }
  const lg::C32* fadjH() const { return paired ? Hadj.as<lg::C32>() : Ht.as<lg::C32>(); }
  const float* fadjW() const { return paired ? wOne.as<float>() : wkf.as<float>(); }

  // ---- mirror focus stacks (fast path) ----------------------
  // Paraxial defocus flips the pupil phase, P(f; -F) = conj(P(f; F)); with a
  // point-symmetric source the -F stack is the conjugate of the +F stack and
  // both print the same aerial image of a real mask, so a
  // stack that is the conjugate mirror of an earlier one is not recomputed:
  // it is imaged / weighted through its representative.  The test is on the
  // kernel values themselves (any source / generator): equal weights and
  // H_f'(q) = c conj(H_f(-q)) with |c| = 1 per kernel, or H_f'(q) = c conj(H_f(q))
  // with H_f of definite parity.
  std::vector<int> rep;      // focus stack -> computed stack index
  std::vector<int> rep_src;  // computed stack -> its source focus stack
  DevBuf wkf;                // weights of the computed stacks [Fc][K]
  void merge_foci(const double* weights, int S, const std::vector<int>& kx, const std::vector<int>& ky,
                  const double* values) {
    rep.assign(F, 0);
    rep_src.clear();
    const bool off = std::getenv("LITHOGPU_NO_FOCUS_MERGE") != nullptr;
    const int Bx = g.ax.B, lox = g.ax.lo, loy = g.ay.lo;
    std::vector<int> mir(S, -1);
    if (g.ax.lo == -g.ax.hi && g.ay.lo == -g.ay.hi) {
      std::vector<int> at(size_t(Bx) * g.ay.B, -1);
      for (int s2 = 0; s2 < S; ++s2) at[size_t(ky[s2] - loy) * Bx + (kx[s2] - lox)] = s2;
      for (int s2 = 0; s2 < S; ++s2) mir[s2] = at[size_t(-ky[s2] - loy) * Bx + (-kx[s2] - lox)];
    }
    const bool sym_support = std::find(mir.begin(), mir.end(), -1) == mir.end();
    auto kv = [&](int f, int k, int s2, int comp) { return values[2 * ((size_t(f) * K + k) * S + s2) + comp]; };
    auto mirror_of = [&](int f, int f2) {  // is stack f2 the conjugate mirror of stack f?
      if (!sym_support) return false;
      for (int k = 0; k < K; ++k) {
        const double wa = weights[size_t(f) * K + k], wb = weights[size_t(f2) * K + k];
        if (std::abs(wa - wb) > 1e-12 * std::max(std::abs(wa), 1e-300)) return false;
        double hmax = 0;
        int im = 0;
        for (int s2 = 0; s2 < S; ++s2) {
          const double a = std::hypot(kv(f, k, s2, 0), kv(f, k, s2, 1));
          if (a > hmax) {
            hmax = a;
            im = s2;
          }
        }
        if (hmax == 0) continue;
        // parity of H_f (needed for the sigma = +1 form)
        double ep = 0, eo = 0;
        for (int s2 = 0; s2 < S; ++s2) {
          ep = std::max(ep, std::hypot(kv(f, k, mir[s2], 0) - kv(f, k, s2, 0), kv(f, k, mir[s2], 1) - kv(f, k, s2, 1)));
          eo = std::max(eo, std::hypot(kv(f, k, mir[s2], 0) + kv(f, k, s2, 0), kv(f, k, mir[s2], 1) + kv(f, k, s2, 1)));
        }
        const bool parity = std::min(ep, eo) <= 1e-9 * hmax;
        bool ok = false;
        for (int sigma : {-1, 1}) {
          if (sigma == 1 && !parity) continue;
          // c = H_f2(q_m) / conj(H_f(sigma q_m)), |c| = 1
          const int sm = sigma == 1 ? im : mir[im];
          const double xr = kv(f, k, sm, 0), xi = -kv(f, k, sm, 1);  // conj(H_f(sigma q_m))
          const double yr = kv(f2, k, im, 0), yi = kv(f2, k, im, 1);
          const double d = xr * xr + xi * xi;
          if (d == 0) continue;
          double cr = (yr * xr + yi * xi) / d, ci = (yi * xr - yr * xi) / d;
          const double cn = std::hypot(cr, ci);
          if (std::abs(cn - 1.0) > 1e-9) continue;
          double err = 0;
          for (int s2 = 0; s2 < S && err <= 1e-9 * hmax; ++s2) {
            const int ss = sigma == 1 ? s2 : mir[s2];
            const double ar = kv(f, k, ss, 0), ai = -kv(f, k, ss, 1);
            const double pr = cr * ar - ci * ai, pi = cr * ai + ci * ar;
            err = std::max(err, std::hypot(kv(f2, k, s2, 0) - pr, kv(f2, k, s2, 1) - pi));
          }
          if (err <= 1e-9 * hmax) {
            ok = true;
            break;
          }
        }
        if (!ok) return false;
      }
      return true;
    };
    for (int f = 0; f < F; ++f) {
      int r = -1;
      if (!off)
        for (int c = 0; c < int(rep_src.size()) && r < 0; ++c)
          if (mirror_of(rep_src[c], f)) r = c;
      if (r < 0) {
        r = int(rep_src.size());
        rep_src.push_back(f);
      }
      rep[f] = r;
    }
    fg.F = int(rep_src.size());
  }
  int frep(int focus) const { return fast ? rep[focus] : focus; }

  // ---- launch trace (LITHOGPU_TRACE=<path>, diagnostic) ----
  DevBuf trace_buf;
  std::vector<std::string> trace_names;
  static constexpr int kTraceSlots = 64;
  void trace_reset() {
    trace_names.clear();
    trace_buf.ensure(size_t(kTraceSlots) * lg::kTraceCtas * 2 * sizeof(unsigned long long));
    LG_CUDA(cudaMemsetAsync(trace_buf.p, 0, size_t(kTraceSlots) * lg::kTraceCtas * 2 * sizeof(unsigned long long),
                            ctx->stream));
  }
  void trace_dump(const char* path) {
    std::vector<unsigned long long> h(size_t(kTraceSlots) * lg::kTraceCtas * 2);
    LG_CUDA(cudaStreamSynchronize(ctx->stream));
    LG_CUDA(cudaMemcpy(h.data(), trace_buf.p, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    FILE* f = std::fopen(path, "a");
    if (!f) return;
    for (size_t sl = 0; sl < trace_names.size(); ++sl) {
      unsigned long long t0 = ~0ull, t1 = 0;
      int n = 0;
      for (int c = 0; c < lg::kTraceCtas; ++c) {
        const unsigned long long ar = h[(sl * lg::kTraceCtas + c) * 2], b = h[(sl * lg::kTraceCtas + c) * 2 + 1];
        if (!ar) continue;
        const unsigned long long a = ~ar;  // cells keep the complement of the earliest start
        ++n;
        t0 = std::min(t0, a);
        t1 = std::max(t1, b);
      }
      std::fprintf(f, "{\"slot\": %zu, \"name\": \"%s\", \"start_ns\": %llu, \"end_ns\": %llu, \"ctas\": %d}\n", sl,
                   trace_names[sl].c_str(), t0, t1, n);
    }
    std::fclose(f);
  }

  int zflip = 0;
  template <typename Fn>
  void fl(const char* name, Fn&& fn) {
    // LITHOGPU_ABLATE=name[,name..]: skip those launches (timing ablation
    // only, tools/ablate.py; results are then meaningless)
    static const char* ablate = std::getenv("LITHOGPU_ABLATE");
    if (ablate) {
      const std::string list = std::string(",") + ablate + ",";
      if (list.find(std::string(",") + name + ",") != std::string::npos) return;
    }
    if (trace_buf.p && int(trace_names.size()) < kTraceSlots) {
      fg.trace = static_cast<unsigned long long*>(trace_buf.p);
      fg.trace_slot = int(trace_names.size());
      trace_names.push_back(name);
    } else {
      fg.trace = nullptr;
    }
    // alternate the tile order launch by launch (LITHOGPU_NO_ZREV=1: off)
    static const bool zrev_off = std::getenv("LITHOGPU_NO_ZREV") != nullptr;
    fg.zrev = zrev_off ? 0 : (zflip ^= 1);
    ctx->prof_begin(name);
    fn();
    ctx->prof_end();
    try {
      ctx->check_launch();
    } catch (const std::exception& e) {
      fg.trace = nullptr;
      throw std::runtime_error(std::string(name) + ": " + e.what());
    }
    fg.trace = nullptr;
  }

  void set_sigma(double sigma_nm) {
    if (sigma_nm == gsig) return;
    auto hit = gtabs.find(sigma_nm);
    if (hit != gtabs.end()) {
      gxh.p = hit->second->x.p;
      gyb.p = hit->second->y.p;
      gsig = sigma_nm;
      return;
    }
    const auto& ax = g.ax;
    const auto& ay = g.ay;
    std::vector<T> hx(ax.P + 1), hy(ay.nb2);
    if (sigma_nm == 0) {
      std::fill(hx.begin(), hx.end(), T(1));
      std::fill(hy.begin(), hy.end(), T(1));
    } else {
      const double sp = sigma_nm / grid.pitch_nm;
      int rx, ry;
      const auto tx = gauss_taps(ax.N, sp, rx);
      const auto ty = gauss_taps(ay.N, sp, ry);
      for (int p = 0; p <= ax.P; ++p) hx[p] = T(gauss_hat(ax.N, tx, rx, p));
      for (int j = 0; j < ay.nb2; ++j) hy[j] = T(gauss_hat(ay.N, ty, ry, lg::band2_p(ay, j)));
    }
    auto tab = std::make_unique<GTab>();
    tab->x.ensure(hx.size() * sizeof(T));
    tab->y.ensure(hy.size() * sizeof(T));
    h2d_blocking(tab->x.p, hx.data(), hx.size() * sizeof(T));
    h2d_blocking(tab->y.p, hy.data(), hy.size() * sizeof(T));
    gxh.p = tab->x.p;
    gyb.p = tab->y.p;
    gtabs.emplace(sigma_nm, std::move(tab));
    gsig = sigma_nm;
  }

  void reserve(int tiles, bool adjoint) {
    if (tiles > cap) {
      ++gen;
      Eb.release();
      Mr.release(); Mhat.release(); Tb.release(); Ir.release(); Ic.release(); Rc.release();
      Dr.release(); Wc.release(); U.release(); Acc.release(); Gc.release();
      costrow.release(); gmaxrow.release();
      cap = tiles;
    }
    const size_t c = sizeof(C) * size_t(cap);
    if (fast) {
      const char* se = std::getenv("LITHOGPU_STORE_E");
      store_E = adjoint && (se ? se[0] == '1' : c * s_E <= (8ll << 30));
      if (store_E) Eb.ensure(c * s_E);
      Rh.ensure(c * s_band);
      Ih.ensure(c * s_band);
      Wsub.ensure(sizeof(T) * size_t(cap) * s_Wsub);  // W_lp (adjoint) / I_sub (forward) scratch
      if (adjoint) Wh.ensure(c * s_band);
    }
    Mr.ensure(c * s_Mr);
    Mhat.ensure(c * s_Mhat);
    Tb.ensure(c * s_T);
    Ir.ensure(c * s_Ir);
    Rc.ensure(c * s_C);
    if (!adjoint) {
      Ic.ensure(c * s_C);
      return;
    }
    Dr.ensure(c * s_Dr);
    Wc.ensure(c * s_Wc);
    U.ensure(c * s_U);
    Acc.ensure(c * s_Acc);
    Gc.ensure(c * s_Gc);
    costrow.ensure(sizeof(double) * cap * s_cr);
    gmaxrow.ensure(sizeof(double) * cap * s_gm);
  }

  template <typename Kern, typename... Args>
  void go(const char* name, Kern kern, const Launch& l, dim3 grd, Args... args) {
    ctx->smem_attr(kern, l.smem);
    ctx->prof_begin(name);
    kern<<<grd, l.block, l.smem, ctx->stream>>>(args...);
    ctx->prof_end();
    ctx->check_launch();
  }

  // ---- pipeline stages ------------------------------------------------------
  // real images (tile-major, T) -> half-spectrum rows into out [Pout+1][Ny]
  template <int MODE>
  void real_rows_fwd(const T* src, long long src_ts, T steep, int Pout, C* out, long long out_ts,
                     int tiles) {
    const Launch l = launch_cfg<T>(g.ax.N, 0);
    go("real_rows_fwd", lg::k_real_rows_fwd<T, MODE>, l, dim3(cdiv((g.ay.N + 1) / 2, l.RPC), 1, tiles), g, src,
       src_ts, steep, Pout, out, out_ts);
  }
  void mask_cols(int tiles) {
    const Launch l = launch_cfg<T>(g.ay.N, 0);
    go("mask_cols", lg::k_mask_cols<T>, l, dim3(cdiv(g.ax.Pm + 1, l.RPC), 1, tiles), g, Mr.as<C>(), s_Mr,
       Mhat.as<C>(), s_Mhat);
  }
  void socs_cols(int tiles) {
    const Launch l = launch_cfg<T>(g.ay.n, 0);
    go("socs_cols", lg::k_socs_cols<T>, l, dim3(cdiv(g.ax.B, l.RPC), F * K, tiles), g, Mhat.as<C>(), s_Mhat,
       H.as<C>(), Tb.as<C>(), s_T);
  }
  void socs_rows(T dose, int tiles) {
    const Launch l = launch_cfg<T>(g.ax.n, 0);
    go("socs_rows", lg::k_socs_rows<T>, l, dim3(cdiv(g.ay.n, l.RPC), F, tiles), g, Tb.as<C>(), s_T,
       wk.as<T>(), dose, Ir.as<C>(), s_Ir, static_cast<T*>(nullptr), 0LL);
  }
  void isub_cols(bool want_i, bool want_r, int tiles) {
    const Launch l = launch_cfg<T>(g.ay.n, g.ay.N);
    const dim3 grd(cdiv(g.ax.P + 1, l.RPC), F, tiles);
    if (want_i && want_r)
      go("isub_cols", lg::k_isub_cols<T, true, true>, l, grd, g, Ir.as<C>(), s_Ir, gxh.as<T>(), gyb.as<T>(),
         Ic.as<C>(), Rc.as<C>(), s_C);
    else if (want_i)
      go("isub_cols", lg::k_isub_cols<T, true, false>, l, grd, g, Ir.as<C>(), s_Ir, gxh.as<T>(), gyb.as<T>(),
         Ic.as<C>(), Rc.as<C>(), s_C);
    else
      go("isub_cols", lg::k_isub_cols<T, false, true>, l, grd, g, Ir.as<C>(), s_Ir, gxh.as<T>(), gyb.as<T>(),
         Ic.as<C>(), Rc.as<C>(), s_C);
  }
  template <typename OutT>
  void out_rows(bool want_i, bool want_r, OutT* I, OutT* R, unsigned char* pr, long long o_ts,
                T thr, int tiles) {
    if constexpr (std::is_same<T, float>::value && std::is_same<OutT, float>::value) {
      if (fast) {
        fl("out_rows", [&] {
          lg::fl_out_rows(fg, ctx->stream, tiles, want_i ? Ic.as<C>() : nullptr, want_r ? Rc.as<C>() : nullptr,
                          s_C, I, R, pr, o_ts, thr);
        });
        return;
      }
    }
    const Launch l = launch_cfg<T>(g.ax.N, 0);
    go("out_rows", lg::k_out_rows<T, OutT>, l, dim3(cdiv(g.ay.N, l.RPC), F, tiles), g,
       want_i ? static_cast<const C*>(Ic.as<C>()) : nullptr,
       want_r ? static_cast<const C*>(Rc.as<C>()) : nullptr, s_C, I, R, pr, o_ts, thr);
  }
  void resist_rows(const T* target, long long tg_ts, const T* cf, T beta, T thr, int tiles,
                   T* zout = nullptr, long long z_ts = 0) {
    const Launch l = launch_cfg<T>(g.ax.N, 0);
    go("resist_rows", lg::k_resist_rows<T>, l, dim3(cdiv(g.ay.N, l.RPC), (F + 1) / 2, tiles), g, Rc.as<C>(),
       s_C, target, tg_ts, cf, beta, thr, Dr.as<C>(), s_Dr, costrow.as<double>(), s_cr, zout,
       z_ts);
  }
  void wlp_cols(bool gauss, int nf, int tiles) {
    const Launch l = launch_cfg<T>(g.ay.N, g.ay.n);
    const dim3 grd(cdiv(g.ax.P + 1, l.RPC), nf, tiles);
    if (gauss)
      go("wlp_cols", lg::k_wlp_cols<T, true>, l, grd, g, Dr.as<C>(), s_Dr, gxh.as<T>(), gyb.as<T>(),
         Wc.as<C>(), s_Wc);
    else
      go("wlp_cols", lg::k_wlp_cols<T, false>, l, grd, g, Dr.as<C>(), s_Dr, gxh.as<T>(), gyb.as<T>(),
         Wc.as<C>(), s_Wc);
  }
  void adj_rows(bool uniform, int nf, int tiles) {
    const Launch l = launch_cfg<T>(g.ax.n, 0);
    const dim3 grd(cdiv(g.ay.n, l.RPC), nf, tiles);
    if (uniform)
      go("adj_rows", lg::k_adj_rows<T, true>, l, grd, g, Tb.as<C>(), s_T, Wc.as<C>(), s_Wc, U.as<C>(), s_U);
    else
      go("adj_rows", lg::k_adj_rows<T, false>, l, grd, g, Tb.as<C>(), s_T, Wc.as<C>(), s_Wc, U.as<C>(), s_U);
  }
  void adj_cols(T dose, int tiles) {
    const Launch l = launch_cfg<T>(g.ay.n, 0);
    go("adj_cols", lg::k_adj_cols<T>, l, dim3(g.ax.B, 1, tiles), g, U.as<C>(), s_U, H.as<C>(), wk.as<T>(),
       dose, Acc.as<C>(), s_Acc);
  }
  void grad_cols(int tiles, bool with_cost, double* cost_out, long long co_ts) {
    const Launch l = launch_cfg<T>(g.ay.N, 0);
    go("grad_cols", lg::k_grad_cols<T>, l, dim3(cdiv(g.ax.Pm + 1, l.RPC) + 1, 1, tiles), g, Acc.as<C>(),
       s_Acc, Gc.as<C>(), s_Gc, static_cast<const double*>(costrow.as<double>()), s_cr,
       with_cost ? int(F * g.ay.N) : 0, with_cost ? cost_out : nullptr, co_ts);
  }
  template <bool ILT, typename OutT>
  void grad_rows(OutT* grad, long long gr_ts, T* theta, long long th_ts, T steep, T step,
                 double* gm, int tiles) {
    const Launch l = launch_cfg<T>(g.ax.N, 0);
    go("grad_rows", lg::k_grad_rows<T, ILT, OutT>, l, dim3(cdiv((g.ay.N + 1) / 2, l.RPC), 1, tiles), g,
       Gc.as<C>(), s_Gc, grad, gr_ts, theta, th_ts, steep, step, Mr.as<C>(), s_Mr, gm, s_gm);
  }

  // fast path: band resampling columns (fused single pass when the plan pair
  // has a fused kernel, else the two-pass form through the band buffers)
  void isub_cols_fast(int tiles, bool want_i, bool want_r) {
    cudaStream_t s = ctx->stream;
    bool fused = false;
    if (!unfused())
      fl("isub_cols", [&] {
      fused = lg::fl_band_col2(fg, s, tiles, fg.F, true, Ir.as<C>(), s_Ir, gxh.as<T>(), gyb.as<T>(),
                               want_r ? Rc.as<C>() : nullptr, want_i ? Ic.as<C>() : nullptr, s_C);
    });
    if (fused) return;
    fl("isub_colfwd", [&] {
      lg::fl_band_colfwd(fg, s, tiles, fg.F, true, Ir.as<C>(), s_Ir, gxh.as<T>(), gyb.as<T>(),
                         want_r ? Rh.as<C>() : nullptr, want_i ? Ih.as<C>() : nullptr, s_band);
    });
    if (want_i)
      fl("isub_colinv", [&] { lg::fl_band_colinv(fg, s, tiles, fg.F, false, Ih.as<C>(), s_band, Ic.as<C>(), s_C); });
    if (want_r)
      fl("isub_colinv", [&] { lg::fl_band_colinv(fg, s, tiles, fg.F, false, Rh.as<C>(), s_band, Rc.as<C>(), s_C); });
  }
  void wlp_cols_fast(int tiles, int nf, bool gauss) {
    cudaStream_t s = ctx->stream;
    const float* gx = gauss ? gxh.as<T>() : nullptr;
    const float* gy = gauss ? gyb.as<T>() : nullptr;
    bool fused = false;
    if (!unfused())
      fl("wlp_cols", [&] {
      fused = lg::fl_band_col2(fg, s, tiles, nf, false, Dr.as<C>(), s_Dr, gx, gy, Wc.as<C>(), nullptr, s_Wc);
    });
    if (fused) return;
    fl("wlp_colfwd", [&] {
      lg::fl_band_colfwd(fg, s, tiles, nf, false, Dr.as<C>(), s_Dr, gx, gy, Wh.as<C>(), nullptr, s_band);
    });
    fl("wlp_colinv", [&] { lg::fl_band_colinv(fg, s, tiles, nf, true, Wh.as<C>(), s_band, Wc.as<C>(), s_Wc); });
  }

  // ---- composite operations ---------------------------------------------------
  // Forward images for focus stacks (all F computed; caller picks one).
  void forward(const T* mask, long long m_ts, int tiles, T dose, bool want_i, bool want_r) {
    reserve(tiles, false);
    mr_owner = nullptr;
    if constexpr (std::is_same<T, float>::value) {
      if (fast) {
        cudaStream_t s = ctx->stream;
        lg::fast_set_pdl(true);
        fl("real_rows_fwd", [&] { lg::fl_real_rows_fwd(fg, s, tiles, 0, mask, m_ts, 0.f, g.ax.Pm, Mr.as<C>(), s_Mr); });
        fl("mask_cols", [&] { lg::fl_mask_cols(fg, s, tiles, Mr.as<C>(), s_Mr, Mhat.as<C>(), s_Mhat); });
        fl("socs_cols", [&] { lg::fl_socs_cols(fg, s, tiles, Mhat.as<C>(), s_Mhat, Ht.as<C>(), Tb.as<C>(), s_T); });
        fl("socs_rows", [&] {
          lg::fl_socs_rows(fg, s, tiles, Tb.as<C>(), s_T, fw1(), fw2(), dose, Ir.as<C>(), s_Ir, nullptr, 0);
        });
        isub_cols_fast(tiles, want_i, want_r);
        return;
      }
    }
    real_rows_fwd<0>(mask, m_ts, T(0), g.ax.Pm, Mr.as<C>(), s_Mr, tiles);
    mask_cols(tiles);
    socs_cols(tiles);
    socs_rows(dose, tiles);
    isub_cols(want_i, want_r, tiles);
  }

  void gradient(const T* mask, const T* W, T dose, T* grad) {
    reserve(1, true);
    mr_owner = nullptr;
    if constexpr (std::is_same<T, float>::value) {
      if (fast) {
        cudaStream_t s = ctx->stream;
        fl("real_rows_fwd", [&] { lg::fl_real_rows_fwd(fg, s, 1, 0, mask, 0, 0.f, g.ax.Pm, Mr.as<C>(), s_Mr); });
        fl("mask_cols", [&] { lg::fl_mask_cols(fg, s, 1, Mr.as<C>(), s_Mr, Mhat.as<C>(), s_Mhat); });
        fl("socs_cols", [&] { lg::fl_socs_cols(fg, s, 1, Mhat.as<C>(), s_Mhat, Ht.as<C>(), Tb.as<C>(), s_T); });
        if (W) {
          fl("real_rows_fwd", [&] { lg::fl_real_rows_fwd(fg, s, 1, 0, W, 0, 0.f, g.ax.P, Dr.as<C>(), s_Dr); });
          wlp_cols_fast(1, 1, false);
          fl("wlp_rows", [&] { lg::fl_wlp_rows(fg, s, 1, 1, Wc.as<C>(), s_Wc, Wsub.as<T>(), s_Wsub); });
        }
        fl("adj_rows", [&] {
          lg::fl_adj_rows(fg, s, 1, 1, W == nullptr, false, Tb.as<C>(), s_T, Wsub.as<T>(), s_Wsub, U.as<C>(),
                          s_U);
        });
        fl("adj_cols", [&] { lg::fl_adj_cols(fg, s, 1, U.as<C>(), s_U, fadjH(), fadjW(), dose, Acc.as<C>(), s_Acc); });
        fl("grad_cols", [&] {
          lg::fl_grad_cols(fg, s, 1, Acc.as<C>(), s_Acc, fg.F * fg.K, Gc.as<C>(), s_Gc, nullptr, 0, 0, nullptr, 0);
        });
        fl("grad_rows", [&] {
          lg::fl_grad_rows(fg, s, 1, false, Gc.as<C>(), s_Gc, grad, 0, nullptr, 0, 0.f, 0.f, Mr.as<C>(), s_Mr,
                           nullptr, 0);
        });
        return;
      }
    }
    real_rows_fwd<0>(mask, 0, T(0), g.ax.Pm, Mr.as<C>(), s_Mr, 1);
    mask_cols(1);
    socs_cols(1);
    if (W) {
      real_rows_fwd<0>(W, 0, T(0), g.ax.P, Dr.as<C>(), s_Dr, 1);
      wlp_cols(false, 1, 1);
    }
    adj_rows(W == nullptr, 1, 1);
    adj_cols(dose, 1);
    grad_cols(1, false, nullptr, 0);
    grad_rows<false, T>(grad, 0, nullptr, 0, T(0), T(0), nullptr, 1);
  }
};

struct lithogpu_kernels {
  lithogpu_ctx* ctx;
  lithogpu_dtype precision;
  lithogpu_grid grid;
  int F, K;
  std::unique_ptr<PlanBase> plan;
  template <typename T>
  Plan<T>& p() {
    return *static_cast<Plan<T>*>(plan.get());
  }
};

// ============================================================================
// ILT state
// ============================================================================
struct lithogpu_ilt {
  lithogpu_kernels* ks;
  lithogpu_ilt_params prm;
  std::vector<double> cf;
  int tiles;
  DevBuf theta, target, cfd, cost, gmax;
  bool primed = false;
  // captured launch sequences (see ilt_run_impl)
  struct GraphKey {
    int iters;
    bool gmax, prime;
    long long gen;
    const void *cost, *gmaxp;
    bool operator==(const GraphKey& o) const {
      return iters == o.iters && gmax == o.gmax && prime == o.prime && gen == o.gen &&
             cost == o.cost && gmaxp == o.gmaxp;
    }
  };
  struct GraphEntry {
    GraphKey key;
    cudaGraphExec_t exec;
    long long nk;  // kernels per replay
    std::vector<std::string> trace_names;  // launch names per trace slot (LITHOGPU_TRACE)
  };
  std::vector<GraphEntry> graphs;
  std::vector<GraphKey> warm;
  bool warm_key(const GraphKey& k) const {
    for (const auto& w : warm)
      if (w == k) return true;
    return false;
  }
  ~lithogpu_ilt() {
    for (auto& e : graphs) cudaGraphExecDestroy(e.exec);
  }
};

// grad_dev (device, tiles x N^2, nullable): dL/dtheta of the LAST iteration;
// step_override >= 0 replaces params.step (0: evaluate without moving theta —
// theta - 0*g == theta exactly, so the mask spectrum re-derived by grad_rows
// is unchanged).  Graph capture only for the plain run (grad_dev == nullptr).
template <typename T>
static void ilt_run_impl(lithogpu_ilt* ilt, int iters, double* cost_user, double* gmax_user,
                         T* grad_dev = nullptr, double step_override = -1.0) {
  using C = lg::cx<T>;
  Plan<T>& P = ilt->ks->p<T>();
  lithogpu_ctx* ctx = ilt->ks->ctx;
  const int tiles = ilt->tiles;
  const auto& prm = ilt->prm;
  const long long NN = (long long)P.g.ax.N * P.g.ay.N;
  P.reserve(tiles, true);
  P.set_sigma(prm.resist_sigma_nm);
  ilt->cost.ensure(sizeof(double) * size_t(std::max(iters, 1)) * tiles);
  ilt->gmax.ensure(sizeof(double) * size_t(std::max(iters, 1)) * tiles);
  T* theta = ilt->theta.as<T>();
  const T a = T(prm.mask_steepness), step = T(step_override >= 0 ? step_override : prm.step),
          beta = T(prm.resist_beta),
          thr = T(prm.threshold), dose = T(prm.dose);
  // initial mask row pass (subsequent ones are fused into grad_rows)
  const bool need_prime = !(ilt->primed && P.mr_owner == ilt);
  if (iters > 0) {
    ilt->primed = true;
    P.mr_owner = ilt;
  }
  auto enqueue = [&]() {
  if constexpr (std::is_same<T, float>::value) {
    if (P.fast) {
      cudaStream_t s = ctx->stream;
      const lg::FGeo& fg = P.fg;
      static const bool ilt_pdl = [] {
        const char* e = std::getenv("LITHOGPU_ILT_PDL");
        return e && e[0] == '1';
      }();
      lg::fast_set_pdl(ilt_pdl);
      const int F = P.fg.F;  // computed focus stacks (mirrors merged)
      if (need_prime)
        P.fl("real_rows_fwd", [&] { lg::fl_real_rows_fwd(fg, s, tiles, 1, theta, NN, a, P.g.ax.Pm, P.Mr.template as<C>(), P.s_Mr); });
      for (int it = 0; it < iters; ++it) {
        P.fl("mask_cols", [&] { lg::fl_mask_cols(fg, s, tiles, P.Mr.template as<C>(), P.s_Mr, P.Mhat.template as<C>(), P.s_Mhat); });
        P.fl("socs_cols", [&] { lg::fl_socs_cols(fg, s, tiles, P.Mhat.template as<C>(), P.s_Mhat, P.Ht.template as<C>(), P.Tb.template as<C>(), P.s_T); });
        C* Ef = P.store_E ? P.Eb.template as<C>() : nullptr;
        P.fl("socs_rows", [&] {
          lg::fl_socs_rows(fg, s, tiles, P.Tb.template as<C>(), P.s_T, P.fw1(), P.fw2(), dose, P.Ir.template as<C>(),
                           P.s_Ir, Ef, P.s_E);
        });
        P.isub_cols_fast(tiles, false, true);
        P.fl("resist_rows", [&] {
          lg::fl_resist_rows(fg, s, tiles, P.Rc.template as<C>(), P.s_C, ilt->target.as<T>(), NN, ilt->cfd.as<T>(), beta, thr,
                             P.Dr.template as<C>(), P.s_Dr, P.costrow.template as<double>(), P.s_cr);
        });
        P.wlp_cols_fast(tiles, F, true);
        P.fl("wlp_rows", [&] { lg::fl_wlp_rows(fg, s, tiles, F, P.Wc.template as<C>(), P.s_Wc, P.Wsub.template as<T>(), P.s_Wsub); });
        P.fl("adj_rows", [&] {
          lg::fl_adj_rows(fg, s, tiles, F, false, Ef != nullptr, Ef ? Ef : P.Tb.template as<C>(), Ef ? P.s_E : P.s_T,
                          P.Wsub.template as<T>(), P.s_Wsub, P.U.template as<C>(), P.s_U);
        });
        const long long npairs = (P.g.ay.N + 1) / 2;
        const int ncost = int(std::min<long long>(P.s_cr, F * npairs * std::max(1, lg::fast_tpr(P.g.ax.N) / 32)));
        double* cost_it = ilt->cost.as<double>() + size_t(it) * tiles;
        P.fl("adj_cols", [&] {
          lg::fl_adj_cols(fg, s, tiles, P.U.template as<C>(), P.s_U, P.fadjH(), P.fadjW(), dose,
                          P.Acc.template as<C>(), P.s_Acc);
        });
        P.fl("grad_cols", [&] {
          lg::fl_grad_cols(fg, s, tiles, P.Acc.template as<C>(), P.s_Acc, F * fg.K, P.Gc.template as<C>(), P.s_Gc,
                           P.costrow.template as<double>(), P.s_cr, ncost, cost_it, 1);
        });
        P.fl("grad_rows", [&] {
          lg::fl_grad_rows(fg, s, tiles, true, P.Gc.template as<C>(), P.s_Gc, it + 1 == iters ? grad_dev : nullptr,
                           NN, theta, NN, a, step,
                           P.Mr.template as<C>(), P.s_Mr, P.gmaxrow.template as<double>(), P.s_gm);
        });
        if (gmax_user) {
          const int ngm = int(npairs * std::max(1, lg::fast_tpr(P.g.ax.N) / 32));
          lg::k_reduce_max<<<tiles, 32, 0, ctx->stream>>>(P.gmaxrow.template as<double>(), P.s_gm, ngm,
                                                         ilt->gmax.as<double>() + size_t(it) * tiles);
          ctx->check_launch();
        }
      }
      return;
    }
  }
  if (need_prime)
    P.template real_rows_fwd<1>(theta, NN, a, P.g.ax.Pm, P.Mr.template as<C>(), P.s_Mr, tiles);
  for (int it = 0; it < iters; ++it) {
    P.mask_cols(tiles);
    P.socs_cols(tiles);
    P.socs_rows(dose, tiles);
    P.isub_cols(false, true, tiles);
    P.resist_rows(ilt->target.as<T>(), NN, ilt->cfd.as<T>(), beta, thr, tiles);
    P.wlp_cols(true, P.F, tiles);
    P.adj_rows(false, P.F, tiles);
    P.adj_cols(dose, tiles);
    // cost of iteration `it` for each tile -> cost[it*tiles + tile]
    P.grad_cols(tiles, true, ilt->cost.as<double>() + size_t(it) * tiles, 1);
    P.template grad_rows<true, T>(it + 1 == iters ? grad_dev : static_cast<T*>(nullptr), NN, theta, NN, a, step,
                                  P.gmaxrow.template as<double>(), tiles);
    if (gmax_user) {
      lg::k_reduce_max<<<tiles, 32, 0, ctx->stream>>>(
          P.gmaxrow.template as<double>(), P.s_gm, int(P.s_gm),
          ilt->gmax.as<double>() + size_t(it) * tiles);
      ctx->check_launch();
    }
  }
  };  // enqueue

  static const char* trace_path = std::getenv("LITHOGPU_TRACE");
  if (trace_path) P.trace_reset();
  // CUDA graph of the whole `iters`-iteration launch sequence: captured on the
  // second call with an identical configuration, replayed afterwards.
  const bool graphable = ctx->stream != nullptr && !ctx->profiling && iters > 0 && !grad_dev &&
                         step_override < 0 &&
                         !std::getenv("LITHOGPU_NO_GRAPH");
  if (!graphable) {
    enqueue();
  } else {
    const lithogpu_ilt::GraphKey key{iters, gmax_user != nullptr, need_prime, P.gen, ilt->cost.p,
                                     ilt->gmax.p};
    lithogpu_ilt::GraphEntry* hit = nullptr;
    for (auto& e : ilt->graphs)
      if (e.key == key) hit = &e;
    if (!hit && ilt->warm_key(key)) {
      const long long l0 = ctx->launches;
      LG_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
      cudaGraph_t graph = nullptr;
      try {
        enqueue();
      } catch (...) {
        cudaStreamEndCapture(ctx->stream, &graph);
        if (graph) cudaGraphDestroy(graph);
        throw;
      }
      LG_CUDA(cudaStreamEndCapture(ctx->stream, &graph));
      cudaGraphExec_t exec = nullptr;
      const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
      cudaGraphDestroy(graph);
      LG_CUDA(ie);
      ilt->graphs.push_back({key, exec, ctx->launches - l0, P.trace_names});
      ctx->launches = l0;
      hit = &ilt->graphs.back();
    }
    if (hit) {
      if (trace_path) P.trace_names = hit->trace_names;
      LG_CUDA(cudaGraphLaunch(hit->exec, ctx->stream));
      ctx->launches += hit->nk;
    } else {
      enqueue();
      ilt->warm.push_back(key);
    }
  }
  if (trace_path) P.trace_dump(trace_path);

  if (cost_user) {
    const size_t bytes = sizeof(double) * size_t(iters) * tiles;
    LG_CUDA(cudaMemcpyAsync(cost_user, ilt->cost.p, bytes,
                            is_device_ptr(cost_user) ? cudaMemcpyDeviceToDevice
                                                     : cudaMemcpyDeviceToHost,
                            ctx->stream));
  }
  bool host = false;
  if (gmax_user) {
    const size_t bytes = sizeof(double) * size_t(iters) * tiles;
    const bool dev = is_device_ptr(gmax_user);
    host |= !dev;
    LG_CUDA(cudaMemcpyAsync(gmax_user, ilt->gmax.p, bytes,
                            dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, ctx->stream));
  }
  if (cost_user) host |= !is_device_ptr(cost_user);
  // stream-ordered unless results go to host memory
  if (host) LG_CUDA(cudaStreamSynchronize(ctx->stream));
}

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

const char* lithogpu_last_error(void) { return g_last_error.c_str(); }

lithogpu_status lithogpu_ctx_create(int device, lithogpu_ctx** out) {
  if (!out) {
    g_last_error = "lithogpu_ctx_create: null argument";
    return LITHOGPU_ERR_USAGE;
  }
  return guarded([&] {
    int n = 0;
    LG_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) throw UsageError("lithogpu_ctx_create: bad device index");
    auto* c = new lithogpu_ctx;
    c->device = device;
    LG_CUDA(cudaSetDevice(device));
    *out = c;
  });
}

void lithogpu_ctx_destroy(lithogpu_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  delete ctx;
}

lithogpu_status lithogpu_ctx_set_stream(lithogpu_ctx* ctx, void* stream) {
  if (!ctx) {
    g_last_error = "lithogpu_ctx_set_stream: null context";
    return LITHOGPU_ERR_USAGE;
  }
  ctx->stream = static_cast<cudaStream_t>(stream);
  g_last_error.clear();
  return LITHOGPU_OK;
}

lithogpu_status lithogpu_ctx_synchronize(lithogpu_ctx* ctx) {
  if (!ctx) {
    g_last_error = "lithogpu_ctx_synchronize: null context";
    return LITHOGPU_ERR_USAGE;
  }
  return guarded([&] {
    ctx->activate();
    LG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

long long lithogpu_ctx_launch_count(const lithogpu_ctx* ctx) { return ctx ? ctx->launches : -1; }

lithogpu_status lithogpu_ctx_set_profiling(lithogpu_ctx* ctx, int on) {
  if (!ctx) {
    g_last_error = "lithogpu_ctx_set_profiling: null context";
    return LITHOGPU_ERR_USAGE;
  }
  return guarded([&] {
    ctx->activate();
    ctx->prof_collect();
    ctx->profiling = on != 0;
  });
}

lithogpu_status lithogpu_ctx_profile_report(lithogpu_ctx* ctx, char* buf, size_t len, int reset) {
  if (!ctx || !buf || len == 0) {
    g_last_error = "lithogpu_ctx_profile_report: null argument";
    return LITHOGPU_ERR_USAGE;
  }
  return guarded([&] {
    ctx->activate();
    ctx->prof_collect();
    std::string out;
    char line[256];
    for (const auto& kv : ctx->agg) {
      std::snprintf(line, sizeof line, "%s %lld %.9f\n", kv.first.c_str(), kv.second.n, kv.second.ms);
      out += line;
    }
    std::snprintf(buf, len, "%s", out.c_str());
    if (reset) ctx->agg.clear();
  });
}

lithogpu_status lithogpu_fp32_peak(lithogpu_ctx* ctx, double* tflops) {
  if (!ctx || !tflops) {
    g_last_error = "lithogpu_fp32_peak: null argument";
    return LITHOGPU_ERR_USAGE;
  }
  return guarded([&] {
    ctx->activate();
    int dev = 0, sms = 0;
    LG_CUDA(cudaGetDevice(&dev));
    LG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    DevBuf o;
    o.ensure(16);
    cudaEvent_t a, b;
    LG_CUDA(cudaEventCreate(&a));
    LG_CUDA(cudaEventCreate(&b));
    const int blocks = sms * 8, threads = 256, iters = 4096;
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
      LG_CUDA(cudaEventRecord(a, ctx->stream));
      lg::k_ffma_peak<<<blocks, threads, 0, ctx->stream>>>(o.as<float>(), iters, 0.999f, 0.001f);
      LG_CUDA(cudaEventRecord(b, ctx->stream));
      LG_CUDA(cudaEventSynchronize(b));
      float ms = 0;
      LG_CUDA(cudaEventElapsedTime(&ms, a, b));
      if (rep > 0) best = std::min(best, ms);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    const double flops = 2.0 * 8 * 16 * double(iters) * blocks * threads;
    *tflops = flops / (best * 1e-3) / 1e12;
  });
}

lithogpu_status lithogpu_rasterize(lithogpu_ctx* ctx, const lithogpu_grid* grid, const int64_t* xy,
                                   const int64_t* poly_start, int n_poly, double dbu_per_nm,
                                   double* out) {
  if (!ctx || !grid || !out || (n_poly > 0 && (!xy || !poly_start)) || n_poly < 0) {
    g_last_error = "lithogpu_rasterize: null argument";
    return LITHOGPU_ERR_USAGE;
  }
  return guarded([&] {
    ctx->activate();
    if (grid->pitch_nm <= 0) throw std::invalid_argument("rasterize_layer: nonpositive pitch");
    if (grid->nx <= 0 || grid->ny <= 0) throw std::invalid_argument("rasterize_layer: empty grid");
    if (!(dbu_per_nm > 0)) throw std::invalid_argument("rasterize_layer: nonpositive dbu_per_nm");
    const int nx = grid->nx, ny = grid->ny;
    const size_t npix = size_t(nx) * ny;
    std::vector<int64_t> st(size_t(n_poly) + 1, 0);
    if (n_poly > 0) {
      if (is_device_ptr(poly_start))
        LG_CUDA(cudaMemcpy(st.data(), poly_start, sizeof(int64_t) * (n_poly + 1), cudaMemcpyDeviceToHost));
      else
        std::memcpy(st.data(), poly_start, sizeof(int64_t) * (n_poly + 1));
    }
    const int64_t nv = st[n_poly];
    const int nbx = (nx + lg::kRasterBin - 1) / lg::kRasterBin;
    const int nby = (ny + lg::kRasterBin - 1) / lg::kRasterBin;
    const int nbins = nbx * nby;
    // device scratch
    PoolBuf dxy, dst, vx, vy, bb, cnt, off, tmp, rect, rsign;
    dxy.ensure(sizeof(int64_t) * 2 * std::max<int64_t>(nv, 1), ctx->stream);
    dst.ensure(sizeof(int64_t) * (n_poly + 1), ctx->stream);
    vx.ensure(sizeof(double) * std::max<int64_t>(nv, 1), ctx->stream);
    vy.ensure(sizeof(double) * std::max<int64_t>(nv, 1), ctx->stream);
    bb.ensure(sizeof(int4) * std::max(n_poly, 1), ctx->stream);
    rect.ensure(sizeof(double4) * std::max(n_poly, 1), ctx->stream);
    rsign.ensure(sizeof(double) * std::max(n_poly, 1), ctx->stream);
    cnt.ensure(sizeof(int) * (nbins + 1), ctx->stream);
    off.ensure(sizeof(int) * (nbins + 1), ctx->stream);
    if (nv > 0) LG_CUDA(cudaMemcpyAsync(dxy.p, xy, sizeof(int64_t) * 2 * nv, cudaMemcpyDefault, ctx->stream));
    LG_CUDA(cudaMemcpyAsync(dst.p, st.data(), sizeof(int64_t) * (n_poly + 1), cudaMemcpyHostToDevice, ctx->stream));
    if (n_poly > 0) {
      lg::k_raster_prep<<<cdiv(n_poly, 128), 128, 0, ctx->stream>>>(
          dxy.as<int64_t>(), dst.as<int64_t>(), n_poly, 1.0 / dbu_per_nm, grid->origin_x_nm,
          grid->origin_y_nm, grid->pitch_nm, nx, ny, vx.as<double>(), vy.as<double>(), bb.as<int4>(),
          rect.as<double4>(), rsign.as<double>());
      ctx->check_launch();
    }
    LG_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int) * (nbins + 1), ctx->stream));
    lg::k_raster_bin<false><<<nbins, 256, 0, ctx->stream>>>(bb.as<int4>(), n_poly, nbx, cnt.as<int>(), nullptr, nullptr);
    ctx->check_launch();
    size_t tbytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tbytes, cnt.as<int>(), off.as<int>(), nbins + 1, ctx->stream);
    tmp.ensure(std::max<size_t>(tbytes, 16), ctx->stream);
    cub::DeviceScan::ExclusiveSum(tmp.p, tbytes, cnt.as<int>(), off.as<int>(), nbins + 1, ctx->stream);
    int total = 0;
    LG_CUDA(cudaMemcpyAsync(&total, off.as<int>() + nbins, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    LG_CUDA(cudaStreamSynchronize(ctx->stream));
    PoolBuf lists;
    lists.ensure(sizeof(int) * std::max(total, 1), ctx->stream);
    lg::k_raster_bin<true><<<nbins, 256, 0, ctx->stream>>>(bb.as<int4>(), n_poly, nbx, cnt.as<int>(), off.as<int>(), lists.as<int>());
    ctx->check_launch();
    const bool dev_out = is_device_ptr(out);
    PoolBuf obuf;
    double* dout = out;
    if (!dev_out) {
      obuf.ensure(sizeof(double) * npix, ctx->stream);
      dout = obuf.as<double>();
    }
    dim3 blk(32, 8), grd(cdiv(nx, 32), cdiv(ny, 8));
    PoolBuf slow, slist, nslow, stmp;
    slow.ensure(sizeof(int) * npix, ctx->stream);
    slist.ensure(sizeof(int) * npix, ctx->stream);
    nslow.ensure(sizeof(int), ctx->stream);
    lg::k_raster_pixels<<<grd, blk, 0, ctx->stream>>>(vx.as<double>(), vy.as<double>(), dst.as<int64_t>(), bb.as<int4>(),
                                                      rect.as<double4>(), rsign.as<double>(), off.as<int>(),
                                                      cnt.as<int>(), lists.as<int>(), nx, ny, nbx, dout,
                                                      slow.as<int>());
    ctx->check_launch();
    {  // compact the pixels that need the clip chain (edges of rectangles, general polygons)
      cub::CountingInputIterator<int> ids(0);
      size_t sb = 0;
      cub::DeviceSelect::Flagged(nullptr, sb, ids, slow.as<int>(), slist.as<int>(), nslow.as<int>(), int(npix),
                                 ctx->stream);
      stmp.ensure(std::max<size_t>(sb, 16), ctx->stream);
      cub::DeviceSelect::Flagged(stmp.p, sb, ids, slow.as<int>(), slist.as<int>(), nslow.as<int>(), int(npix),
                                 ctx->stream);
    }
    lg::k_raster_pixels_slow<<<148 * 8, 256, 0, ctx->stream>>>(
        vx.as<double>(), vy.as<double>(), dst.as<int64_t>(), bb.as<int4>(), rect.as<double4>(), rsign.as<double>(),
        off.as<int>(), cnt.as<int>(), lists.as<int>(), nx, nbx, slist.as<int>(), nslow.as<int>(), dout);
    ctx->check_launch();
    if (!dev_out) LG_CUDA(cudaMemcpyAsync(out, dout, sizeof(double) * npix, cudaMemcpyDeviceToHost, ctx->stream));
    LG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

lithogpu_status lithogpu_kernels_create(lithogpu_ctx* ctx, const lithogpu_grid* grid,
                                        lithogpu_dtype precision, int n_focus, int order,
                                        const double* weights, int n_support,
                                        const int32_t* support, const double* values,
                                        lithogpu_kernels** out) {
  if (!ctx || !grid || !weights || !support || !values || !out) {
    g_last_error = "lithogpu_kernels_create: null argument";
    return LITHOGPU_ERR_USAGE;
  }
  return guarded([&] {
    require(precision == LITHOGPU_F32 || precision == LITHOGPU_F64,
            "lithogpu_kernels_create: precision must be F32 or F64");
    if (grid->nx <= 0 || grid->ny <= 0 || !(grid->pitch_nm > 0))
      throw std::invalid_argument("lithogpu_kernels_create: bad grid");
    if (n_focus <= 0 || order <= 0 || n_support <= 0)
      throw std::invalid_argument("lithogpu_kernels_create: empty kernel stack");
    for (int i = 0; i < n_focus * order; ++i)
      if (!(weights[i] >= 0) || !std::isfinite(weights[i]))
        throw std::invalid_argument("lithogpu_kernels_create: weights must be finite and >= 0");
    ctx->activate();
    auto* ks = new lithogpu_kernels;
    ks->ctx = ctx;
    ks->precision = precision;
    ks->grid = *grid;
    ks->F = n_focus;
    ks->K = order;
    try {
      if (precision == LITHOGPU_F32)
        ks->plan.reset(new Plan<float>(ctx, *grid, n_focus, order, weights, n_support, support, values));
      else
        ks->plan.reset(new Plan<double>(ctx, *grid, n_focus, order, weights, n_support, support, values));
    } catch (...) {
      delete ks;
      throw;
    }
    *out = ks;
  });
}

void lithogpu_kernels_destroy(lithogpu_kernels* ks) {
  if (!ks) return;
  cudaSetDevice(ks->ctx->device);
  cudaStreamSynchronize(ks->ctx->stream);
  delete ks;
}

lithogpu_status lithogpu_kernels_fast_order(const lithogpu_kernels* ks, int* order) {
  if (!ks || !order) {
    g_last_error = "lithogpu_kernels_fast_order: null argument";
    return LITHOGPU_ERR_USAGE;
  }
  return guarded([&] {
    *order = 0;
    if (ks->precision != LITHOGPU_F32) return;
    auto& p = const_cast<lithogpu_kernels*>(ks)->p<float>();
    if (p.fast) *order = p.fg.K;
  });
}

lithogpu_status lithogpu_kernels_fast_stacks(const lithogpu_kernels* ks, int* stacks) {
  if (!ks || !stacks) {
    g_last_error = "lithogpu_kernels_fast_stacks: null argument";
    return LITHOGPU_ERR_USAGE;
  }
  return guarded([&] {
    *stacks = ks->F;
    if (ks->precision != LITHOGPU_F32) return;
    auto& p = const_cast<lithogpu_kernels*>(ks)->p<float>();
    if (p.fast) *stacks = p.fg.F;
  });
}

lithogpu_status lithogpu_kernels_info(const lithogpu_kernels* ks, int* nx_sub, int* ny_sub,
                                      int* band_x, int* band_y) {
  if (!ks) {
    g_last_error = "lithogpu_kernels_info: null argument";
    return LITHOGPU_ERR_USAGE;
  }
  return guarded([&] {
    const lg::AxisGeom *ax, *ay;
    if (ks->precision == LITHOGPU_F32) {
      auto& p = const_cast<lithogpu_kernels*>(ks)->p<float>();
      ax = &p.g.ax;
      ay = &p.g.ay;
    } else {
      auto& p = const_cast<lithogpu_kernels*>(ks)->p<double>();
      ax = &p.g.ax;
      ay = &p.g.ay;
    }
    if (nx_sub) *nx_sub = ax->n;
    if (ny_sub) *ny_sub = ay->n;
    if (band_x) *band_x = ax->B;
    if (band_y) *band_y = ay->B;
  });
}

}  // extern "C"

namespace {

template <typename T>
void image_impl(lithogpu_kernels* ks, int focus, const void* mask, lithogpu_dtype mdt, double dose,
                double sigma, double thr, void* I, void* R, lithogpu_dtype odt, unsigned char* pr) {
  Plan<T>& P = ks->p<T>();
  lithogpu_ctx* ctx = ks->ctx;
  const size_t n = size_t(P.g.ax.N) * P.g.ay.N;
  const T* m = stage_in<T>(ctx, mask, mdt, n, 0);
  const bool want_r = R || pr;
  const bool want_i = I != nullptr;
  P.set_sigma(want_r ? sigma : 0.0);
  P.forward(m, 0, 1, T(dose), want_i || !want_r, want_r);
  // all F foci are computed by forward(); output rows only for `focus`
  OutStage<T> oi(ctx, I, odt, n, 2), orr(ctx, R, odt, n, 4);
  DevBuf& fullI = ctx->slot(6);
  DevBuf& fullR = ctx->slot(7);
  DevBuf& fullP = ctx->slot(8);
  const size_t Fn = size_t(P.F) * n;
  fullI.ensure(sizeof(T) * Fn);
  fullR.ensure(sizeof(T) * Fn);
  if (pr) fullP.ensure(Fn);
  P.template out_rows<T>(want_i, want_r, want_i ? fullI.as<T>() : nullptr,
                         want_r ? fullR.as<T>() : nullptr, pr ? fullP.as<unsigned char>() : nullptr,
                         0, T(thr), 1);
  if (I)
    LG_CUDA(cudaMemcpyAsync(oi.work, fullI.as<T>() + size_t(P.frep(focus)) * n, sizeof(T) * n,
                            cudaMemcpyDeviceToDevice, ctx->stream));
  if (R)
    LG_CUDA(cudaMemcpyAsync(orr.work, fullR.as<T>() + size_t(P.frep(focus)) * n, sizeof(T) * n,
                            cudaMemcpyDeviceToDevice, ctx->stream));
  bool host = oi.finish();
  host |= orr.finish();
  if (pr) {
    LG_CUDA(cudaMemcpyAsync(pr, fullP.as<unsigned char>() + size_t(P.frep(focus)) * n, n, cudaMemcpyDefault,
                            ctx->stream));
    host |= !is_device_ptr(pr);
  }
  if (host || !is_device_ptr(mask)) LG_CUDA(cudaStreamSynchronize(ctx->stream));
}

}  // namespace

extern "C" {

lithogpu_status lithogpu_image_resist(lithogpu_kernels* ks, int focus, const void* mask,
                                      lithogpu_dtype mask_dtype, double dose, double sigma_nm,
                                      double threshold, void* intensity, void* resist,
                                      lithogpu_dtype out_dtype, unsigned char* print) {
  if (!ks || !mask) {
    g_last_error = "lithogpu_image_resist: null argument";
    return LITHOGPU_ERR_USAGE;
  }
  return guarded([&] {
    if (focus < 0 || focus >= ks->F) throw UsageError("lithogpu_image: focus index out of range");
    if (sigma_nm < 0) throw std::invalid_argument("gaussian_blur: negative sigma");
    dtype_size(mask_dtype);
    dtype_size(out_dtype);
    ks->ctx->activate();
    if (ks->precision == LITHOGPU_F32)
      image_impl<float>(ks, focus, mask, mask_dtype, dose, sigma_nm, threshold, intensity, resist,
                        out_dtype, print);
    else
      image_impl<double>(ks, focus, mask, mask_dtype, dose, sigma_nm, threshold, intensity, resist,
                         out_dtype, print);
  });
}

lithogpu_status lithogpu_image_socs(lithogpu_kernels* ks, int focus, const void* mask,
                                    lithogpu_dtype mask_dtype, double dose, void* intensity,
                                    lithogpu_dtype out_dtype) {
  if (!intensity) {
    g_last_error = "lithogpu_image_socs: null argument";
    return LITHOGPU_ERR_USAGE;
  }
  return lithogpu_image_resist(ks, focus, mask, mask_dtype, dose, 0.0, 0.0, intensity, nullptr,
                               out_dtype, nullptr);
}

lithogpu_status lithogpu_intensity_gradient(lithogpu_kernels* ks, int focus, const void* mask,
                                            lithogpu_dtype mask_dtype, const void* weight,
                                            lithogpu_dtype weight_dtype, double dose, void* grad,
                                            lithogpu_dtype grad_dtype) {
  if (!ks || !mask || !grad) {
    g_last_error = "lithogpu_intensity_gradient: null argument";
    return LITHOGPU_ERR_USAGE;
  }
  return guarded([&] {
    if (focus < 0 || focus >= ks->F) throw UsageError("intensity_gradient: focus out of range");
    ks->ctx->activate();
    auto run = [&](auto tag) {
      using T = decltype(tag);
      Plan<T>& P = ks->p<T>();
      lithogpu_ctx* ctx = ks->ctx;
      const size_t n = size_t(P.g.ax.N) * P.g.ay.N;
      const T* m = stage_in<T>(ctx, mask, mask_dtype, n, 0);
      const T* w = weight ? stage_in<T>(ctx, weight, weight_dtype, n, 2) : nullptr;
      OutStage<T> og(ctx, grad, grad_dtype, n, 4);
      // single focus: temporarily view stack `focus` as a 1-stack plan
      const int F0 = P.F;
      lg::Geo<T> g0 = P.g;
      DevBuf& Hf = ctx->slot(9);
      DevBuf& wf = ctx->slot(10);
      const size_t hsz = size_t(P.K) * P.g.ay.B * P.g.ax.B * sizeof(lg::cx<T>);
      Hf.ensure(hsz);
      wf.ensure(sizeof(T) * P.K);
      LG_CUDA(cudaMemcpyAsync(Hf.p, P.H.template as<char>() + hsz * focus, hsz, cudaMemcpyDeviceToDevice, ctx->stream));
      LG_CUDA(cudaMemcpyAsync(wf.p, P.wk.template as<T>() + size_t(P.K) * focus, sizeof(T) * P.K, cudaMemcpyDeviceToDevice, ctx->stream));
      DevBuf& Htf = ctx->slot(11);
      DevBuf& Haf = ctx->slot(12);
      DevBuf& Wff = ctx->slot(13);
      if (P.fast) {  // fast-path copies of the computed stack of `focus` (kernel pairs when paired)
        const int fr = P.frep(focus);
        const size_t fsz = size_t(P.fg.K) * P.g.ay.B * P.g.ax.B * sizeof(lg::C32);
        Htf.ensure(fsz);
        LG_CUDA(cudaMemcpyAsync(Htf.p, P.Ht.template as<char>() + fsz * fr, fsz, cudaMemcpyDeviceToDevice,
                                ctx->stream));
        std::swap(P.Ht.p, Htf.p);
        if (P.paired) {
          Haf.ensure(fsz);
          LG_CUDA(cudaMemcpyAsync(Haf.p, P.Hadj.template as<char>() + fsz * fr, fsz, cudaMemcpyDeviceToDevice,
                                  ctx->stream));
          std::swap(P.Hadj.p, Haf.p);
        } else {
          Wff.ensure(sizeof(float) * P.K);
          LG_CUDA(cudaMemcpyAsync(Wff.p, P.wkf.template as<float>() + size_t(P.K) * fr, sizeof(float) * P.K,
                                  cudaMemcpyDeviceToDevice, ctx->stream));
          std::swap(P.wkf.p, Wff.p);
        }
      }
      std::swap(P.H.p, Hf.p);
      std::swap(P.wk.p, wf.p);
      const int fgF0 = P.fg.F;
      const int* slot0 = P.fg.slot_on;
      if (P.fast && slot0) P.fg.slot_on = slot0 + size_t(P.frep(focus)) * P.fg.K;  // mixed pairs: this stack's slots
      P.F = 1;
      P.g.F = 1;
      P.fg.F = 1;
      try {
        P.gradient(m, w, T(dose), og.work);
      } catch (...) {
        if (P.fast) std::swap(P.Ht.p, Htf.p);
        if (P.fast && P.paired) std::swap(P.Hadj.p, Haf.p);
        if (P.fast && !P.paired) std::swap(P.wkf.p, Wff.p);
        std::swap(P.H.p, Hf.p);
        std::swap(P.wk.p, wf.p);
        P.F = F0;
        P.g = g0;
        P.fg.F = fgF0;
        P.fg.slot_on = slot0;
        throw;
      }
      if (P.fast) std::swap(P.Ht.p, Htf.p);
      if (P.fast && P.paired) std::swap(P.Hadj.p, Haf.p);
      if (P.fast && !P.paired) std::swap(P.wkf.p, Wff.p);
      std::swap(P.H.p, Hf.p);
      std::swap(P.wk.p, wf.p);
      P.F = F0;
      P.g = g0;
      P.fg.F = fgF0;
      P.fg.slot_on = slot0;
      const bool host = og.finish();
      if (host || !is_device_ptr(mask)) LG_CUDA(cudaStreamSynchronize(ctx->stream));
    };
    if (ks->precision == LITHOGPU_F32)
      run(float{});
    else
      run(double{});
  });
}

lithogpu_status lithogpu_gaussian_blur(lithogpu_ctx* ctx, const lithogpu_grid* grid,
                                       const void* in, lithogpu_dtype dtype, double sigma_nm,
                                       void* out) {
  if (!ctx || !grid || !in || !out) {
    g_last_error = "lithogpu_gaussian_blur: null argument";
    return LITHOGPU_ERR_USAGE;
  }
  return guarded([&] {
    if (sigma_nm < 0) throw std::invalid_argument("gaussian_blur: negative sigma");
    require(dtype == LITHOGPU_F32 || dtype == LITHOGPU_F64, "gaussian_blur: dtype must be F32/F64");
    ctx->activate();
    const int nx = grid->nx, ny = grid->ny;
    const size_t n = size_t(nx) * ny;
    auto run = [&](auto tag) {
      using T = decltype(tag);
      const T* src = stage_in<T>(ctx, in, dtype, n, 0);
      OutStage<T> o(ctx, out, dtype, n, 2);
      if (sigma_nm == 0) {
        LG_CUDA(cudaMemcpyAsync(o.work, src, sizeof(T) * n, cudaMemcpyDeviceToDevice, ctx->stream));
      } else {
        const double sp = sigma_nm / grid->pitch_nm;
        int rx, ry;
        auto tx = gauss_taps(nx, sp, rx);
        auto ty = gauss_taps(ny, sp, ry);
        std::vector<T> hx(tx.begin(), tx.end()), hy(ty.begin(), ty.end());
        DevBuf& dt = ctx->slot(11);
        DevBuf& mid = ctx->slot(12);
        dt.ensure(sizeof(T) * (hx.size() + hy.size()));
        mid.ensure(sizeof(T) * n);
        LG_CUDA(cudaMemcpyAsync(dt.p, hx.data(), sizeof(T) * hx.size(), cudaMemcpyHostToDevice, ctx->stream));
        LG_CUDA(cudaMemcpyAsync(dt.as<T>() + hx.size(), hy.data(), sizeof(T) * hy.size(), cudaMemcpyHostToDevice, ctx->stream));
        dim3 blk(32, 8), grd(cdiv(nx, 32), cdiv(ny, 8));
        lg::k_blur_pass<T, 0><<<grd, blk, 0, ctx->stream>>>(src, mid.as<T>(), nx, ny, dt.as<T>(), rx);
        ctx->check_launch();
        lg::k_blur_pass<T, 1><<<grd, blk, 0, ctx->stream>>>(mid.as<T>(), o.work, nx, ny, dt.as<T>() + hx.size(), ry);
        ctx->check_launch();
        LG_CUDA(cudaStreamSynchronize(ctx->stream));  // host taps lifetime
      }
      const bool host = o.finish();
      if (host) LG_CUDA(cudaStreamSynchronize(ctx->stream));
    };
    if (dtype == LITHOGPU_F32)
      run(float{});
    else
      run(double{});
  });
}

lithogpu_status lithogpu_fft2(lithogpu_ctx* ctx, void* data, lithogpu_dtype dtype, int nx, int ny,
                              int inverse) {
  if (!ctx || !data) {
    g_last_error = "lithogpu_fft2: null argument";
    return LITHOGPU_ERR_USAGE;
  }
  return guarded([&] {
    require(dtype == LITHOGPU_F32 || dtype == LITHOGPU_F64, "fft2: dtype must be F32 or F64");
    if (nx <= 0 || ny <= 0) throw std::invalid_argument("fft2: size mismatch");
    ctx->activate();
    auto run = [&](auto tag) {
      using T = decltype(tag);
      using C = lg::cx<T>;
      const size_t n = size_t(nx) * ny;
      const bool dev = is_device_ptr(data);
      C* d = static_cast<C*>(data);
      if (!dev) {
        DevBuf& b = ctx->slot(13);
        b.ensure(n * sizeof(C));
        LG_CUDA(cudaMemcpyAsync(b.p, data, n * sizeof(C), cudaMemcpyHostToDevice, ctx->stream));
        d = b.as<C>();
      }
      auto cached = [&](int L) {
        auto& tb = ctx->fft_tabs[{L, int(sizeof(T))}];
        if (!tb) tb.reset(new TabBufs);
        const lg::Tab<T> t = make_tab<T>(L, *tb, tb->built);
        tb->built = true;
        return t;
      };
      const lg::Tab<T> tabx = cached(nx), taby = cached(ny);
      auto tab = [&](int L, int) { return L == nx ? tabx : taby; };
      const int tx = 0, ty = 0;
      const Launch lr = launch_cfg<T>(nx, 0), lc = launch_cfg<T>(ny, 0);
      ctx->smem_attr(lg::k_fft2_rows<T, -1>, lr.smem);
      ctx->smem_attr(lg::k_fft2_rows<T, +1>, lr.smem);
      ctx->smem_attr(lg::k_fft2_cols<T, -1>, lc.smem);
      ctx->smem_attr(lg::k_fft2_cols<T, +1>, lc.smem);
      if (inverse) {
        lg::k_fft2_rows<T, +1><<<dim3(cdiv(ny, lr.RPC)), lr.block, lr.smem, ctx->stream>>>(tab(nx, tx), nx, ny, d);
        ctx->check_launch();
        lg::k_fft2_cols<T, +1><<<dim3(cdiv(nx, lc.RPC)), lc.block, lc.smem, ctx->stream>>>(tab(ny, ty), nx, ny, d);
      } else {
        lg::k_fft2_rows<T, -1><<<dim3(cdiv(ny, lr.RPC)), lr.block, lr.smem, ctx->stream>>>(tab(nx, tx), nx, ny, d);
        ctx->check_launch();
        lg::k_fft2_cols<T, -1><<<dim3(cdiv(nx, lc.RPC)), lc.block, lc.smem, ctx->stream>>>(tab(ny, ty), nx, ny, d);
      }
      ctx->check_launch();
      if (!dev)
        LG_CUDA(cudaMemcpyAsync(data, d, n * sizeof(C), cudaMemcpyDeviceToHost, ctx->stream));
      LG_CUDA(cudaStreamSynchronize(ctx->stream));
    };
    if (dtype == LITHOGPU_F32)
      run(float{});
    else
      run(double{});
  });
}

lithogpu_status lithogpu_threshold(lithogpu_ctx* ctx, size_t n, const void* in,
                                   lithogpu_dtype in_dtype, double tau, void* out,
                                   lithogpu_dtype out_dtype) {
  if (!ctx || !in || !out) {
    g_last_error = "lithogpu_threshold: null argument";
    return LITHOGPU_ERR_USAGE;
  }
  return guarded([&] {
    dtype_size(in_dtype);
    dtype_size(out_dtype);
    ctx->activate();
    const double* src = stage_in<double>(ctx, in, in_dtype, n, 0);
    OutStage<double> o(ctx, out, out_dtype, n, 2);
    const int blocks = int(std::min<size_t>((n + 255) / 256, 148 * 16));
    if (n) {
      lg::k_threshold<double, double><<<blocks, 256, 0, ctx->stream>>>(src, o.work, n, tau);
      ctx->check_launch();
    }
    const bool host = o.finish();
    if (host || !is_device_ptr(in)) LG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

lithogpu_status lithogpu_ilt_create(lithogpu_kernels* ks, const lithogpu_ilt_params* params,
                                    int n_tiles, lithogpu_ilt** out) {
  if (!ks || !params || !out || !params->focus_weights) {
    g_last_error = "lithogpu_ilt_create: null argument";
    return LITHOGPU_ERR_USAGE;
  }
  return guarded([&] {
    if (n_tiles <= 0) throw UsageError("lithogpu_ilt_create: n_tiles must be > 0");
    if (params->resist_sigma_nm < 0) throw std::invalid_argument("ilt: negative resist sigma");
    ks->ctx->activate();
    auto* ilt = new lithogpu_ilt;
    ilt->ks = ks;
    ilt->prm = *params;
    ilt->cf.assign(params->focus_weights, params->focus_weights + ks->F);
    ilt->prm.focus_weights = ilt->cf.data();
    ilt->tiles = n_tiles;
    const size_t es = ks->precision == LITHOGPU_F32 ? 4 : 8;
    const size_t n = size_t(ks->grid.nx) * ks->grid.ny * n_tiles;
    try {
      ilt->theta.ensure(es * n);
      ilt->target.ensure(es * n);
      ilt->cfd.ensure(es * ks->F);
      if (es == 4) {
        // fp32 fast path: weights of the computed stacks (mirror stacks add to
        // their representative, Plan::merge_foci)
        auto& P = ks->p<float>();
        std::vector<float> c(ilt->cf.begin(), ilt->cf.end());
        if (P.fast) {
          std::vector<double> m(size_t(P.fg.F), 0.0);
          for (int f = 0; f < ks->F; ++f) m[size_t(P.rep[f])] += ilt->cf[f];
          c.assign(m.begin(), m.end());
          c.resize(size_t(ks->F), 0.f);
        }
        h2d_blocking(ilt->cfd.p, c.data(), 4 * c.size());
      } else {
        h2d_blocking(ilt->cfd.p, ilt->cf.data(), 8 * ilt->cf.size());
      }
      LG_CUDA(cudaMemsetAsync(ilt->theta.p, 0, es * n, ks->ctx->stream));
      LG_CUDA(cudaMemsetAsync(ilt->target.p, 0, es * n, ks->ctx->stream));
    } catch (...) {
      delete ilt;
      throw;
    }
    *out = ilt;
  });
}

void lithogpu_ilt_destroy(lithogpu_ilt* ilt) {
  if (!ilt) return;
  cudaSetDevice(ilt->ks->ctx->device);
  cudaStreamSynchronize(ilt->ks->ctx->stream);
  delete ilt;
}

}  // extern "C"

namespace {

template <typename T>
void ilt_set_impl(lithogpu_ilt* ilt, int tile0, int ntl, const void* target, const void* theta0,
                  lithogpu_dtype dt) {
  lithogpu_ctx* ctx = ilt->ks->ctx;
  const size_t n1 = size_t(ilt->ks->grid.nx) * ilt->ks->grid.ny;
  const size_t n = n1 * ntl;
  const T* tg = stage_in<T>(ctx, target, dt, n, 0);
  T* dtg = ilt->target.as<T>() + n1 * tile0;
  T* dth = ilt->theta.as<T>() + n1 * tile0;
  LG_CUDA(cudaMemcpyAsync(dtg, tg, sizeof(T) * n, cudaMemcpyDeviceToDevice, ctx->stream));
  if (theta0) {
    const T* th = stage_in<T>(ctx, theta0, dt, n, 2);
    LG_CUDA(cudaMemcpyAsync(dth, th, sizeof(T) * n, cudaMemcpyDeviceToDevice, ctx->stream));
  } else {
    const int blocks = int(std::min<size_t>((n + 255) / 256, 148 * 16));
    lg::k_theta_init<T><<<blocks, 256, 0, ctx->stream>>>(dtg, dth, n, T(2.0 / ilt->prm.mask_steepness));
    ctx->check_launch();
  }
  if (!is_device_ptr(target) || (theta0 && !is_device_ptr(theta0)))
    LG_CUDA(cudaStreamSynchronize(ctx->stream));
}

template <typename T>
void ilt_get_impl(lithogpu_ilt* ilt, int tile0, int ntl, void* theta, void* mask, lithogpu_dtype dt) {
  lithogpu_ctx* ctx = ilt->ks->ctx;
  const size_t n1 = size_t(ilt->ks->grid.nx) * ilt->ks->grid.ny;
  const size_t n = n1 * ntl;
  const T* th = ilt->theta.as<T>() + n1 * tile0;
  bool host = false;
  if (theta) {
    OutStage<T> o(ctx, theta, dt, n, 0);
    LG_CUDA(cudaMemcpyAsync(o.work, th, sizeof(T) * n, cudaMemcpyDeviceToDevice, ctx->stream));
    host |= o.finish();
  }
  if (mask) {
    OutStage<T> o(ctx, mask, dt, n, 2);
    const int blocks = int(std::min<size_t>((n + 255) / 256, 148 * 16));
    lg::k_sigmoid<T><<<blocks, 256, 0, ctx->stream>>>(th, o.work, n, T(ilt->prm.mask_steepness));
    ctx->check_launch();
    host |= o.finish();
  }
  if (host) LG_CUDA(cudaStreamSynchronize(ctx->stream));
}

}  // namespace

extern "C" {

lithogpu_status lithogpu_ilt_set_tile(lithogpu_ilt* ilt, int tile, const void* target,
                                      const void* theta0, lithogpu_dtype dtype) {
  if (!ilt || !target) {
    g_last_error = "lithogpu_ilt_set_tile: null argument";
    return LITHOGPU_ERR_USAGE;
  }
  return guarded([&] {
    if (tile < 0 || tile >= ilt->tiles) throw UsageError("lithogpu_ilt_set_tile: tile out of range");
    dtype_size(dtype);
    ilt->ks->ctx->activate();
    ilt->primed = false;
    if (ilt->ks->precision == LITHOGPU_F32)
      ilt_set_impl<float>(ilt, tile, 1, target, theta0, dtype);
    else
      ilt_set_impl<double>(ilt, tile, 1, target, theta0, dtype);
  });
}

lithogpu_status lithogpu_ilt_set_tiles(lithogpu_ilt* ilt, const void* target, const void* theta0,
                                       lithogpu_dtype dtype) {
  if (!ilt || !target) {
    g_last_error = "lithogpu_ilt_set_tiles: null argument";
    return LITHOGPU_ERR_USAGE;
  }
  return guarded([&] {
    dtype_size(dtype);
    ilt->ks->ctx->activate();
    ilt->primed = false;
    if (ilt->ks->precision == LITHOGPU_F32)
      ilt_set_impl<float>(ilt, 0, ilt->tiles, target, theta0, dtype);
    else
      ilt_set_impl<double>(ilt, 0, ilt->tiles, target, theta0, dtype);
  });
}

lithogpu_status lithogpu_ilt_run(lithogpu_ilt* ilt, int iterations, double* cost, double* gmax) {
  if (!ilt) {
    g_last_error = "lithogpu_ilt_run: null argument";
    return LITHOGPU_ERR_USAGE;
  }
  return guarded([&] {
    if (iterations < 0) throw UsageError("lithogpu_ilt_run: negative iteration count");
    ilt->ks->ctx->activate();
    if (ilt->ks->precision == LITHOGPU_F32)
      ilt_run_impl<float>(ilt, iterations, cost, gmax);
    else
      ilt_run_impl<double>(ilt, iterations, cost, gmax);
  });
}

lithogpu_status lithogpu_ilt_gradient(lithogpu_ilt* ilt, double* cost, void* grad, lithogpu_dtype dtype) {
  if (!ilt || !grad) {
    g_last_error = "lithogpu_ilt_gradient: null argument";
    return LITHOGPU_ERR_USAGE;
  }
  return guarded([&] {
    dtype_size(dtype);
    if (dtype == LITHOGPU_U8) throw UsageError("lithogpu_ilt_gradient: gradient dtype must be F32 or F64");
    ilt->ks->ctx->activate();
    lithogpu_ctx* ctx = ilt->ks->ctx;
    const size_t n = size_t(ilt->ks->grid.nx) * ilt->ks->grid.ny * ilt->tiles;
    auto run = [&](auto tag) {
      using T = decltype(tag);
      OutStage<T> o(ctx, grad, dtype, n, 0);
      ilt_run_impl<T>(ilt, 1, cost, nullptr, o.work, 0.0);
      if (o.finish()) LG_CUDA(cudaStreamSynchronize(ctx->stream));
    };
    if (ilt->ks->precision == LITHOGPU_F32)
      run(float{});
    else
      run(double{});
  });
}

static lithogpu_status ilt_get_window_impl(lithogpu_ilt* ilt, int tile, int x0, int y0, int w, int h, void* mask,
                                           int64_t row_stride, lithogpu_dtype dtype, bool async);

lithogpu_status lithogpu_ilt_get_window(lithogpu_ilt* ilt, int tile, int x0, int y0, int w, int h, void* mask,
                                        int64_t row_stride, lithogpu_dtype dtype) {
  return ilt_get_window_impl(ilt, tile, x0, y0, w, h, mask, row_stride, dtype, false);
}

lithogpu_status lithogpu_ilt_get_window_async(lithogpu_ilt* ilt, int tile, int x0, int y0, int w, int h,
                                              void* mask, int64_t row_stride, lithogpu_dtype dtype) {
  return ilt_get_window_impl(ilt, tile, x0, y0, w, h, mask, row_stride, dtype, true);
}

static lithogpu_status ilt_get_window_impl(lithogpu_ilt* ilt, int tile, int x0, int y0, int w, int h, void* mask,
                                           int64_t row_stride, lithogpu_dtype dtype, bool async) {
  if (!ilt || !mask) {
    g_last_error = "lithogpu_ilt_get_window: null argument";
    return LITHOGPU_ERR_USAGE;
  }
  return guarded([&] {
    const int nx = ilt->ks->grid.nx, ny = ilt->ks->grid.ny;
    if (tile < 0 || tile >= ilt->tiles) throw UsageError("lithogpu_ilt_get_window: tile out of range");
    if (x0 < 0 || y0 < 0 || w <= 0 || h <= 0 || x0 + w > nx || y0 + h > ny || row_stride < w)
      throw UsageError("lithogpu_ilt_get_window: window outside the tile");
    if (dtype != LITHOGPU_F32 && dtype != LITHOGPU_F64) throw UsageError("lithogpu_ilt_get_window: dtype");
    lithogpu_ctx* ctx = ilt->ks->ctx;
    ctx->activate();
    const size_t es = dtype_size(dtype);
    const bool dev = is_device_ptr(mask);
    if (async && !dev) {
      cudaPointerAttributes a{};
      if (cudaPointerGetAttributes(&a, mask) != cudaSuccess || a.type != cudaMemoryTypeHost) {
        cudaGetLastError();
        throw UsageError("lithogpu_ilt_get_window_async: mask must be device or page-locked host memory");
      }
    }
    void* dst = mask;
    long long stride = row_stride;
    if (!dev) {  // staging window (stream-ordered reuse: the next call's kernel runs after this copy)
      DevBuf& b = ctx->slot(async ? 22 : 0);
      if (b.bytes < es * size_t(w) * h) {
        if (async) LG_CUDA(cudaStreamSynchronize(ctx->stream));  // a pending copy may still read it
        b.ensure(es * size_t(w) * h);
      }
      dst = b.p;
      stride = w;
    }
    const dim3 grd((w + 255) / 256, h);
    auto launch = [&](auto tag) {
      using T = decltype(tag);
      const T* th = ilt->theta.as<T>() + size_t(nx) * ny * tile;
      if (dtype == LITHOGPU_F32)
        lg::k_sigmoid_window<T, float><<<grd, 256, 0, ctx->stream>>>(th, nx, x0, y0, w, h,
                                                                      T(ilt->prm.mask_steepness),
                                                                      static_cast<float*>(dst), stride);
      else
        lg::k_sigmoid_window<T, double><<<grd, 256, 0, ctx->stream>>>(th, nx, x0, y0, w, h,
                                                                       T(ilt->prm.mask_steepness),
                                                                       static_cast<double*>(dst), stride);
      ctx->check_launch();
    };
    if (ilt->ks->precision == LITHOGPU_F32)
      launch(float{});
    else
      launch(double{});
    if (!dev) {
      LG_CUDA(cudaMemcpy2DAsync(mask, size_t(row_stride) * es, dst, size_t(w) * es, size_t(w) * es, size_t(h),
                                cudaMemcpyDeviceToHost, ctx->stream));
      if (!async) LG_CUDA(cudaStreamSynchronize(ctx->stream));
    }
  });
}

lithogpu_status lithogpu_ilt_get_tile(lithogpu_ilt* ilt, int tile, void* theta, void* mask,
                                      lithogpu_dtype dtype) {
  if (!ilt) {
    g_last_error = "lithogpu_ilt_get_tile: null argument";
    return LITHOGPU_ERR_USAGE;
  }
  return guarded([&] {
    if (tile < 0 || tile >= ilt->tiles) throw UsageError("lithogpu_ilt_get_tile: tile out of range");
    dtype_size(dtype);
    ilt->ks->ctx->activate();
    if (ilt->ks->precision == LITHOGPU_F32)
      ilt_get_impl<float>(ilt, tile, 1, theta, mask, dtype);
    else
      ilt_get_impl<double>(ilt, tile, 1, theta, mask, dtype);
  });
}

lithogpu_status lithogpu_ilt_get_tiles(lithogpu_ilt* ilt, void* theta, void* mask,
                                       lithogpu_dtype dtype) {
  if (!ilt) {
    g_last_error = "lithogpu_ilt_get_tiles: null argument";
    return LITHOGPU_ERR_USAGE;
  }
  return guarded([&] {
    dtype_size(dtype);
    ilt->ks->ctx->activate();
    if (ilt->ks->precision == LITHOGPU_F32)
      ilt_get_impl<float>(ilt, 0, ilt->tiles, theta, mask, dtype);
    else
      ilt_get_impl<double>(ilt, 0, ilt->tiles, theta, mask, dtype);
  });
}

}  // extern "C"

// ===========================================================================
// contours + EPE: contour_kernels.cuh
// ===========================================================================
struct lithogpu_contours {
  lithogpu_ctx* ctx = nullptr;
  lg::CGeo g{};
  long long ne = 0;
  int ncross = 0;
  long long nloops = 0, npts = 0;
  PoolBuf succ, pt, offsets, xs, ys;
};

namespace {
void ms_scan(lithogpu_ctx* ctx, const int* in, int* out, long long n, PoolBuf& tmp) {
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, n, ctx->stream);
  tmp.ensure(std::max<size_t>(tb, 16), ctx->stream);
  cub::DeviceScan::ExclusiveSum(tmp.p, tb, in, out, n, ctx->stream);
}
void ms_scan64(lithogpu_ctx* ctx, const int* in, long long* out, long long n, PoolBuf& tmp) {
  size_t tb = 0;
  cub::DeviceScan::ExclusiveScan(nullptr, tb, in, out, cub::Sum(), 0ll, n, ctx->stream);
  tmp.ensure(std::max<size_t>(tb, 16), ctx->stream);
  cub::DeviceScan::ExclusiveScan(tmp.p, tb, in, out, cub::Sum(), 0ll, n, ctx->stream);
}
template <typename T>
T read_dev(lithogpu_ctx* ctx, const T* p) {
  T v;
  LG_CUDA(cudaMemcpyAsync(&v, p, sizeof(T), cudaMemcpyDeviceToHost, ctx->stream));
  LG_CUDA(cudaStreamSynchronize(ctx->stream));
  return v;
}
}  // namespace

// marching squares of a DEVICE f64 field (internal; see lithogpu_marching_squares)
static std::unique_ptr<lithogpu_contours> ms_build(lithogpu_ctx* ctx, const lithogpu_grid* grid, const double* field,
                                            double threshold) {
  const int nx = grid->nx, ny = grid->ny;
  if (nx <= 0 || ny <= 0) throw std::invalid_argument("marching_squares: empty grid");
  auto c = std::make_unique<lithogpu_contours>();
  c->ctx = ctx;
  c->g = lg::CGeo{nx, ny, grid->pitch_nm, grid->origin_x_nm, grid->origin_y_nm, (long long)(nx - 1) * ny};
  c->ne = c->g.nh + (long long)nx * (ny - 1);
  if (nx < 2 || ny < 2) {  // reference :61
    c->offsets.ensure(sizeof(long long), ctx->stream);
    LG_CUDA(cudaMemsetAsync(c->offsets.p, 0, sizeof(long long), ctx->stream));
    return c;
  }
  const double* f = field;  // device
  const size_t npix = size_t(nx) * ny;
  const int nblk = 256;
  PoolBuf part, mm, flags;
  part.ensure(sizeof(double) * 2 * nblk, ctx->stream);
  mm.ensure(sizeof(double) * 2, ctx->stream);
  flags.ensure(sizeof(int) * 4, ctx->stream);
  LG_CUDA(cudaMemsetAsync(flags.p, 0, sizeof(int) * 4, ctx->stream));
  int* fl = flags.as<int>();  // [0] non-finite, [1] duplicate edge, [2] broken chain
  lg::k_field_minmax<<<nblk, 256, 0, ctx->stream>>>(f, (long long)npix, part.as<double>(), part.as<double>() + nblk, fl);
  ctx->check_launch();
  lg::k_field_minmax_final<<<1, 32, 0, ctx->stream>>>(part.as<double>(), part.as<double>() + nblk, nblk, mm.as<double>());
  ctx->check_launch();
  c->succ.ensure(sizeof(int) * c->ne, ctx->stream);
  c->pt.ensure(sizeof(double2) * c->ne, ctx->stream);
  LG_CUDA(cudaMemsetAsync(c->succ.p, 0xff, sizeof(int) * c->ne, ctx->stream));
  dim3 blk(32, 8), grd(cdiv(nx - 1, 32), cdiv(ny - 1, 8));
  lg::k_ms_cells<<<grd, blk, 0, ctx->stream>>>(c->g, f, threshold, mm.as<double>(), c->succ.as<int>(),
                                             c->pt.as<double2>(), fl + 1);
  ctx->check_launch();
  int hf[4];
  LG_CUDA(cudaMemcpyAsync(hf, fl, sizeof(hf), cudaMemcpyDeviceToHost, ctx->stream));
  LG_CUDA(cudaStreamSynchronize(ctx->stream));
  if (hf[0]) throw std::invalid_argument("marching_squares: non-finite field");
  if (hf[1]) throw std::runtime_error("marching_squares: inconsistent contour graph");
  // compact the crossing edges in edge order
  PoolBuf flag, pos, tmp, idx;
  flag.ensure(sizeof(int) * (c->ne + 1), ctx->stream);
  pos.ensure(sizeof(int) * (c->ne + 1), ctx->stream);
  idx.ensure(sizeof(int) * c->ne, ctx->stream);
  const int gb = 148 * 8;
  lg::k_ms_flags<<<gb, 256, 0, ctx->stream>>>(c->succ.as<int>(), c->ne, flag.as<int>());
  ctx->check_launch();
  LG_CUDA(cudaMemsetAsync(flag.as<int>() + c->ne, 0, sizeof(int), ctx->stream));
  ms_scan(ctx, flag.as<int>(), pos.as<int>(), c->ne + 1, tmp);
  const int n = read_dev(ctx, pos.as<int>() + c->ne);
  c->ncross = n;
  if (n == 0) {
    c->offsets.ensure(sizeof(long long), ctx->stream);
    LG_CUDA(cudaMemsetAsync(c->offsets.p, 0, sizeof(long long), ctx->stream));
    LG_CUDA(cudaStreamSynchronize(ctx->stream));
    return c;
  }
  PoolBuf cedge, csucc, m0, m1, j0, j1, d0, d1, isst, len, lidx, ptoff;
  cedge.ensure(sizeof(int) * n, ctx->stream);
  csucc.ensure(sizeof(int) * n, ctx->stream);
  for (PoolBuf* b : {&m0, &m1, &j0, &j1, &d0, &d1}) b->ensure(sizeof(int) * n, ctx->stream);
  lg::k_ms_compact<<<gb, 256, 0, ctx->stream>>>(c->succ.as<int>(), pos.as<int>(), c->ne, cedge.as<int>(), idx.as<int>());
  ctx->check_launch();
  const int tb = cdiv(n, 256);
  lg::k_ms_link<<<tb, 256, 0, ctx->stream>>>(cedge.as<int>(), c->succ.as<int>(), idx.as<int>(), n, csucc.as<int>(),
                                           m0.as<int>(), fl + 2);
  ctx->check_launch();
  if (read_dev(ctx, fl + 2)) throw std::runtime_error("marching_squares: broken contour chain");
  int rounds = 1;
  while ((1 << rounds) < n) ++rounds;
  // cycle minima
  LG_CUDA(cudaMemcpyAsync(j0.p, csucc.p, sizeof(int) * n, cudaMemcpyDeviceToDevice, ctx->stream));
  int *mA = m0.as<int>(), *mB = m1.as<int>(), *jA = j0.as<int>(), *jB = j1.as<int>();
  for (int r = 0; r < rounds; ++r) {
    lg::k_ms_minjump<<<tb, 256, 0, ctx->stream>>>(mA, jA, n, mB, jB);
    ctx->check_launch();
    std::swap(mA, mB);
    std::swap(jA, jB);
  }
  // distance to the end of each cycle cut before its start
  int *nA = jB, *nB = jA, *dA = d0.as<int>(), *dB = d1.as<int>();
  lg::k_ms_rank_init<<<tb, 256, 0, ctx->stream>>>(csucc.as<int>(), cedge.as<int>(), mA, n, nA, dA);
  ctx->check_launch();
  for (int r = 0; r < rounds; ++r) {
    lg::k_ms_rank_jump<<<tb, 256, 0, ctx->stream>>>(nA, dA, n, nB, dB);
    ctx->check_launch();
    std::swap(nA, nB);
    std::swap(dA, dB);
  }
  isst.ensure(sizeof(int) * (n + 1), ctx->stream);
  len.ensure(sizeof(int) * (n + 1), ctx->stream);
  lidx.ensure(sizeof(int) * (n + 1), ctx->stream);
  ptoff.ensure(sizeof(long long) * (n + 1), ctx->stream);
  lg::k_ms_starts<<<tb, 256, 0, ctx->stream>>>(cedge.as<int>(), mA, dA, n, isst.as<int>(), len.as<int>());
  ctx->check_launch();
  LG_CUDA(cudaMemsetAsync(isst.as<int>() + n, 0, sizeof(int), ctx->stream));
  LG_CUDA(cudaMemsetAsync(len.as<int>() + n, 0, sizeof(int), ctx->stream));
  ms_scan(ctx, isst.as<int>(), lidx.as<int>(), n + 1, tmp);
  ms_scan64(ctx, len.as<int>(), ptoff.as<long long>(), n + 1, tmp);
  c->nloops = read_dev(ctx, lidx.as<int>() + n);
  c->npts = read_dev(ctx, ptoff.as<long long>() + n);
  if (c->npts != n) throw std::runtime_error("marching_squares: broken contour chain");
  c->offsets.ensure(sizeof(long long) * (c->nloops + 1), ctx->stream);
  c->xs.ensure(sizeof(double) * n, ctx->stream);
  c->ys.ensure(sizeof(double) * n, ctx->stream);
  lg::k_ms_offsets<<<tb, 256, 0, ctx->stream>>>(isst.as<int>(), lidx.as<int>(), ptoff.as<long long>(), n,
                                              c->offsets.as<long long>(), c->npts);
  ctx->check_launch();
  lg::k_ms_scatter<<<tb, 256, 0, ctx->stream>>>(cedge.as<int>(), mA, idx.as<int>(), dA, ptoff.as<long long>(),
                                              c->pt.as<double2>(), n, c->xs.as<double>(), c->ys.as<double>());
  ctx->check_launch();
  LG_CUDA(cudaStreamSynchronize(ctx->stream));
  return c;
}

lithogpu_status lithogpu_marching_squares(lithogpu_ctx* ctx, const lithogpu_grid* grid, const double* field,
                                          double threshold, lithogpu_contours** out) {
  if (!ctx || !grid || !field || !out) {
    g_last_error = "lithogpu_marching_squares: null argument";
    return LITHOGPU_ERR_USAGE;
  }
  return guarded([&] {
    ctx->activate();
    if (grid->nx <= 0 || grid->ny <= 0) throw std::invalid_argument("marching_squares: empty grid");
    const double* f = stage_in<double>(ctx, field, LITHOGPU_F64, size_t(grid->nx) * grid->ny, 0);
    *out = ms_build(ctx, grid, f, threshold).release();
  });
}

lithogpu_status lithogpu_contours_size(const lithogpu_contours* c, int64_t* n_loops, int64_t* n_points) {
  if (!c || !n_loops || !n_points) {
    g_last_error = "lithogpu_contours_size: null argument";
    return LITHOGPU_ERR_USAGE;
  }
  *n_loops = c->nloops;
  *n_points = c->npts;
  return LITHOGPU_OK;
}

lithogpu_status lithogpu_contours_get(const lithogpu_contours* c, int64_t* loop_start, double* xs, double* ys) {
  if (!c || (!loop_start && !xs && !ys)) {
    g_last_error = "lithogpu_contours_get: null argument";
    return LITHOGPU_ERR_USAGE;
  }
  return guarded([&] {
    c->ctx->activate();
    cudaStream_t s = c->ctx->stream;
    if (loop_start)
      LG_CUDA(cudaMemcpyAsync(loop_start, c->offsets.p, sizeof(long long) * (c->nloops + 1), cudaMemcpyDefault, s));
    if (xs && c->npts) LG_CUDA(cudaMemcpyAsync(xs, c->xs.p, sizeof(double) * c->npts, cudaMemcpyDefault, s));
    if (ys && c->npts) LG_CUDA(cudaMemcpyAsync(ys, c->ys.p, sizeof(double) * c->npts, cudaMemcpyDefault, s));
    LG_CUDA(cudaStreamSynchronize(s));
  });
}

void lithogpu_contours_destroy(lithogpu_contours* c) { delete c; }

// EPE of DEVICE gauges into DEVICE outputs (internal)
static void epe_run(const lithogpu_contours* c, const double* gauges_dev, int64_t n, double radius, double* epe_dev,
             unsigned char* open_dev) {
  if (n == 0) return;
  const bool grid_ok = c->g.nx >= 2 && c->g.ny >= 2;
  lg::k_epe<<<cdiv(n * 32, 256), 256, 0, c->ctx->stream>>>(
      c->g, grid_ok ? c->succ.as<int>() : nullptr, grid_ok ? c->pt.as<double2>() : nullptr, grid_ok ? c->ncross : 0,
      reinterpret_cast<const lg::Gauge*>(gauges_dev), int(n), radius, epe_dev, open_dev);
  c->ctx->check_launch();
}

lithogpu_status lithogpu_measure_epe(lithogpu_contours* c, const double* gauges, int64_t n, double search_radius_nm,
                                     double* epe_nm, uint8_t* open) {
  if (!c || (n > 0 && (!gauges || !epe_nm || !open)) || n < 0) {
    g_last_error = "lithogpu_measure_epe: null argument";
    return LITHOGPU_ERR_USAGE;
  }
  return guarded([&] {
    if (n == 0) return;
    lithogpu_ctx* ctx = c->ctx;
    ctx->activate();
    const double* gd = stage_in<double>(ctx, gauges, LITHOGPU_F64, size_t(n) * 4, 0);
    const bool dev_e = is_device_ptr(epe_nm), dev_o = is_device_ptr(open);
    PoolBuf eb, ob;
    double* de = epe_nm;
    unsigned char* dob = open;
    if (!dev_e) {
      eb.ensure(sizeof(double) * n, ctx->stream);
      de = eb.as<double>();
    }
    if (!dev_o) {
      ob.ensure(size_t(n), ctx->stream);
      dob = ob.as<unsigned char>();
    }
    epe_run(c, gd, n, search_radius_nm, de, dob);
    if (!dev_e) LG_CUDA(cudaMemcpyAsync(epe_nm, de, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
    if (!dev_o) LG_CUDA(cudaMemcpyAsync(open, dob, size_t(n), cudaMemcpyDeviceToHost, ctx->stream));
    LG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

lithogpu_status lithogpu_measure_epe_loops(lithogpu_ctx* ctx, const int64_t* loop_start, int64_t n_loops,
                                           const double* xs, const double* ys, const double* gauges,
                                           int64_t n, double search_radius_nm, double* epe_nm, uint8_t* open) {
  if (!ctx || n_loops < 0 || n < 0 || (n_loops > 0 && !loop_start) || (n > 0 && (!gauges || !epe_nm || !open))) {
    g_last_error = "lithogpu_measure_epe_loops: null argument";
    return LITHOGPU_ERR_USAGE;
  }
  return guarded([&] {
    if (n == 0) return;
    ctx->activate();
    // segments on the host in loop order (cheap: O(points)), then the GPU scan
    std::vector<int64_t> st(size_t(n_loops) + 1, 0);
    if (n_loops > 0)
      LG_CUDA(cudaMemcpy(st.data(), loop_start, sizeof(int64_t) * (n_loops + 1), cudaMemcpyDefault));
    const int64_t np = n_loops > 0 ? st[n_loops] : 0;
    std::vector<double> hx(size_t(std::max<int64_t>(np, 1))), hy(hx.size());
    if (np > 0) {
      LG_CUDA(cudaMemcpy(hx.data(), xs, sizeof(double) * np, cudaMemcpyDefault));
      LG_CUDA(cudaMemcpy(hy.data(), ys, sizeof(double) * np, cudaMemcpyDefault));
    }
    std::vector<double4> segs;
    segs.reserve(size_t(np));
    for (int64_t l = 0; l < n_loops; ++l)
      for (int64_t i = st[l]; i < st[l + 1]; ++i) {
        const int64_t j = i + 1 < st[l + 1] ? i + 1 : st[l];
        segs.push_back(make_double4(hx[i], hy[i], hx[j], hy[j]));
      }
    PoolBuf ds, eb, ob;
    ds.ensure(sizeof(double4) * std::max<size_t>(segs.size(), 1), ctx->stream);
    if (!segs.empty())
      LG_CUDA(cudaMemcpyAsync(ds.p, segs.data(), sizeof(double4) * segs.size(), cudaMemcpyHostToDevice, ctx->stream));
    const double* gd = stage_in<double>(ctx, gauges, LITHOGPU_F64, size_t(n) * 4, 0);
    const bool dev_e = is_device_ptr(epe_nm), dev_o = is_device_ptr(open);
    double* de = epe_nm;
    unsigned char* dob = open;
    if (!dev_e) {
      eb.ensure(sizeof(double) * n, ctx->stream);
      de = eb.as<double>();
    }
    if (!dev_o) {
      ob.ensure(size_t(n), ctx->stream);
      dob = ob.as<unsigned char>();
    }
    lg::k_epe_segments<<<cdiv(n * 32, 256), 256, 0, ctx->stream>>>(
        ds.as<double4>(), (long long)segs.size(), reinterpret_cast<const lg::Gauge*>(gd), int(n), search_radius_nm,
        de, dob);
    ctx->check_launch();
    if (!dev_e) LG_CUDA(cudaMemcpyAsync(epe_nm, de, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
    if (!dev_o) LG_CUDA(cudaMemcpyAsync(open, dob, size_t(n), cudaMemcpyDeviceToHost, ctx->stream));
    LG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

// ---- evaluate_epe (opc.cpp:140-151) fused on the device ------------------
namespace {
template <typename T>
void evaluate_epe_impl(lithogpu_kernels* ks, int focus, int nm, const void* masks, lithogpu_dtype mdt, double dose,
                       double sigma, double t_eff, const double* gauges, int64_t n, double radius, double* epe_nm,
                       uint8_t* open, double* resist) {
  Plan<T>& P = ks->p<T>();
  lithogpu_ctx* ctx = ks->ctx;
  const long long NN = (long long)P.g.ax.N * P.g.ay.N;
  const T* m = stage_in<T>(ctx, masks, mdt, size_t(nm) * NN, 0);
  P.set_sigma(sigma);
  P.forward(m, NN, nm, T(dose), false, true);  // all tiles in one launch sequence (blockIdx.z)
  PoolBuf fullR, r64, gd, eb, ob;
  fullR.ensure(sizeof(T) * size_t(nm) * P.F * NN, ctx->stream);
  P.template out_rows<T>(false, true, nullptr, fullR.as<T>(), nullptr, (long long)P.F * NN, T(t_eff), nm);
  if (n > 0) {
    gd.ensure(sizeof(double) * 4 * n, ctx->stream);
    LG_CUDA(cudaMemcpyAsync(gd.p, gauges, sizeof(double) * 4 * n, cudaMemcpyDefault, ctx->stream));
    eb.ensure(sizeof(double) * n * nm, ctx->stream);
    ob.ensure(size_t(n) * nm, ctx->stream);
  }
  r64.ensure(sizeof(double) * NN, ctx->stream);
  const lithogpu_grid grid = ks->grid;
  for (int t = 0; t < nm; ++t) {
    const T* rt = fullR.as<T>() + (size_t(t) * P.F + P.frep(focus)) * NN;
    const double* f64;
    if constexpr (std::is_same<T, double>::value) {
      f64 = rt;
    } else {
      convert_dev(ctx, rt, r64.as<double>(), size_t(NN));
      f64 = r64.as<double>();
    }
    if (resist)
      LG_CUDA(cudaMemcpyAsync(resist + size_t(t) * NN, f64, sizeof(double) * NN, cudaMemcpyDefault, ctx->stream));
    auto c = ms_build(ctx, &grid, f64, t_eff);
    if (n > 0) epe_run(c.get(), gd.as<double>(), n, radius, eb.as<double>() + size_t(t) * n,
                       ob.as<unsigned char>() + size_t(t) * n);
  }
  if (n > 0) {
    LG_CUDA(cudaMemcpyAsync(epe_nm, eb.p, sizeof(double) * n * nm, cudaMemcpyDefault, ctx->stream));
    LG_CUDA(cudaMemcpyAsync(open, ob.p, size_t(n) * nm, cudaMemcpyDefault, ctx->stream));
  }
  LG_CUDA(cudaStreamSynchronize(ctx->stream));
}
}  // namespace

lithogpu_status lithogpu_evaluate_epe(lithogpu_kernels* ks, int focus, int n_masks, const void* masks,
                                      lithogpu_dtype mask_dtype, double dose, double sigma_nm, double t_eff,
                                      const double* gauges, int64_t n_gauges, double search_radius_nm,
                                      double* epe_nm, uint8_t* open, double* resist) {
  if (!ks || !masks || n_masks <= 0 || n_gauges < 0 || (n_gauges > 0 && (!gauges || !epe_nm || !open))) {
    g_last_error = "lithogpu_evaluate_epe: null argument";
    return LITHOGPU_ERR_USAGE;
  }
  return guarded([&] {
    if (focus < 0 || focus >= ks->F) throw UsageError("lithogpu_evaluate_epe: focus index out of range");
    if (sigma_nm < 0) throw std::invalid_argument("gaussian_blur: negative sigma");
    dtype_size(mask_dtype);
    ks->ctx->activate();
    if (ks->precision == LITHOGPU_F32)
      evaluate_epe_impl<float>(ks, focus, n_masks, masks, mask_dtype, dose, sigma_nm, t_eff, gauges, n_gauges,
                               search_radius_nm, epe_nm, open, resist);
    else
      evaluate_epe_impl<double>(ks, focus, n_masks, masks, mask_dtype, dose, sigma_nm, t_eff, gauges, n_gauges,
                                search_radius_nm, epe_nm, open, resist);
  });
}

// ---- internal hooks for the other translation units (kernelgen.cu) --------
namespace lg_internal {
cudaStream_t ctx_stream(lithogpu_ctx* ctx) { return ctx->stream; }
void ctx_activate(lithogpu_ctx* ctx) { ctx->activate(); }
void ctx_count_launch(lithogpu_ctx* ctx) { ctx->check_launch(); }
void set_error(const char* msg) { g_last_error = msg ? msg : ""; }
}  // namespace lg_internal

// ---- AIMG tile I/O (io.cpp:317-350) -----------------
lithogpu_status lithogpu_write_aimg(lithogpu_ctx* ctx, const lithogpu_grid* grid, int n_tiles,
                                    const char* const* paths, const void* values, lithogpu_dtype dtype) {
  if (!ctx || !grid || !paths || !values || n_tiles < 0) {
    g_last_error = "lithogpu_write_aimg: null argument";
    return LITHOGPU_ERR_USAGE;
  }
  return guarded([&] {
    const size_t n = size_t(grid->nx) * size_t(grid->ny);
    const size_t es = dtype_size(dtype);
    if (grid->nx <= 0 || grid->ny <= 0) throw std::invalid_argument("write_aimg: size mismatch");
    ctx->activate();
    const bool dev = is_device_ptr(values);
    if (dev) ctx->pinned_ensure(n * sizeof(double));
    DevBuf conv;
    // tile t: D2H (converted to f64 on the device) into pinned buffer t%2; the
    // host writes tile t while tile t+1's copy is in flight
    cudaEvent_t done[2];
    LG_CUDA(cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming));
    LG_CUDA(cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming));
    struct Ev {
      cudaEvent_t* e;
      ~Ev() {
        cudaEventDestroy(e[0]);
        cudaEventDestroy(e[1]);
      }
    } guard{done};
    auto enqueue = [&](int t) {
      const char* src = static_cast<const char*>(values) + size_t(t) * n * es;
      void* dst = ctx->pinned[t & 1];
      if (dtype == LITHOGPU_F64) {
        LG_CUDA(cudaMemcpyAsync(dst, src, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
      } else {
        conv.ensure(n * sizeof(double));
        convert_from(ctx, src, dtype, conv.as<double>(), n);
        LG_CUDA(cudaMemcpyAsync(dst, conv.p, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
      }
      LG_CUDA(cudaEventRecord(done[t & 1], ctx->stream));
    };
    std::vector<double> host_tile;
    if (dev && n_tiles > 0) enqueue(0);
    for (int t = 0; t < n_tiles; ++t) {
      const double* payload;
      if (dev) {
        LG_CUDA(cudaEventSynchronize(done[t & 1]));
        if (t + 1 < n_tiles) enqueue(t + 1);  // overlaps the file write below
        payload = static_cast<const double*>(ctx->pinned[t & 1]);
      } else if (dtype == LITHOGPU_F64) {
        payload = static_cast<const double*>(values) + size_t(t) * n;
      } else {
        host_tile.resize(n);
        const char* b = static_cast<const char*>(values) + size_t(t) * n * es;
        for (size_t i = 0; i < n; ++i)
          host_tile[i] = dtype == LITHOGPU_F32 ? double(reinterpret_cast<const float*>(b)[i])
                                               : double(reinterpret_cast<const unsigned char*>(b)[i]);
        payload = host_tile.data();
      }
      if (!paths[t]) throw UsageError("lithogpu_write_aimg: null path");
      FILE* f = std::fopen(paths[t], "wb");
      if (!f) throw std::runtime_error(std::string("cannot write ") + paths[t]);
      const uint32_t w = uint32_t(grid->nx), h = uint32_t(grid->ny);
      bool ok = std::fwrite("AIMG", 1, 4, f) == 4 && std::fwrite(&w, 4, 1, f) == 1 && std::fwrite(&h, 4, 1, f) == 1 &&
                std::fwrite(&grid->pitch_nm, 8, 1, f) == 1 && std::fwrite(payload, 8, n, f) == n;
      ok = (std::fclose(f) == 0) && ok;
      if (!ok) throw std::runtime_error(std::string("cannot write ") + paths[t]);
    }
  });
}

lithogpu_status lithogpu_read_aimg(lithogpu_ctx* ctx, const char* path, int* nx, int* ny, double* pitch_nm,
                                   double* values) {
  if (!ctx || !path || !nx || !ny || !pitch_nm) {
    g_last_error = "lithogpu_read_aimg: null argument";
    return LITHOGPU_ERR_USAGE;
  }
  return guarded([&] {
    FILE* f = std::fopen(path, "rb");
    if (!f) throw std::runtime_error(std::string("cannot open ") + path);
    struct Closer {
      FILE* f;
      ~Closer() { std::fclose(f); }
    } closer{f};
    char magic[4];
    if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, "AIMG", 4) != 0)
      throw std::runtime_error(std::string(path) + ": not an AIMG file");
    uint32_t w = 0, h = 0;
    double p = 0;
    if (std::fread(&w, 4, 1, f) != 1 || std::fread(&h, 4, 1, f) != 1 || std::fread(&p, 8, 1, f) != 1 || w == 0 ||
        h == 0 || !(p > 0))
      throw std::runtime_error(std::string(path) + ": bad AIMG header");
    *nx = int(w);
    *ny = int(h);
    *pitch_nm = p;
    if (!values) return;
    const size_t n = size_t(w) * h;
    if (is_device_ptr(values)) {
      ctx->activate();
      ctx->pinned_ensure(n * sizeof(double));
      if (std::fread(ctx->pinned[0], 8, n, f) != n) throw std::runtime_error(std::string(path) + ": truncated AIMG payload");
      LG_CUDA(cudaMemcpyAsync(values, ctx->pinned[0], n * 8, cudaMemcpyHostToDevice, ctx->stream));
      LG_CUDA(cudaStreamSynchronize(ctx->stream));
    } else if (std::fread(values, 8, n, f) != n) {
      throw std::runtime_error(std::string(path) + ": truncated AIMG payload");
    }
  });
}
