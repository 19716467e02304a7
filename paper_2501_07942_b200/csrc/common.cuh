// Common layer of the TT-GBF step engine.
//
// The engine is written as CTA-cooperative C++: every routine is executed by
// all threads of one CTA with uniform control flow; parallel loops stride by
// `nt`, serial sections run on thread 0 and publish through memory followed by
// a barrier.  Compiled by nvcc this is the product (one CTA per filter,
// sm_100a).  Compiled by g++ (ENGINE_HOSTSIM) the same source runs as a single
// "thread" -- used only by the CPU test-suite to check the engine's decision
// logic against the oracle; it is never loaded by the product path.
#pragma once

#include <stdint.h>
#include <stddef.h>
#include <math.h>
#include <string.h>

#ifdef __CUDACC__
#define HD __host__ __device__ __forceinline__
#define HDI __host__ __device__
#define HDN static __host__ __device__ __noinline__   // internal linkage: api.cu is compiled once per entry-point group
#else
#define HD inline
#define HDI
#define HDN inline
#endif

#if defined(__CUDA_ARCH__)
#define ENGINE_DEVICE 1
#else
#define ENGINE_DEVICE 0
#endif

namespace tg {

constexpr int MAXD = 16;      // max number of modes (state dimension)
// general SMEM scratch per CTA (doubles): sized so two CTAs need <= 100 KB of
// shared memory and the SM keeps ~156 KB of L1 for the L2-streamed working set
constexpr int SMEM_SCRATCH_DOUBLES = 5632;
constexpr int CTA_WARPS = 8;  // BLOCK_THREADS / 32
// widest TT rank tt_chain_eval can hold: two rank vectors per warp in the scratch
constexpr int CHAIN_MAXR = SMEM_SCRATCH_DOUBLES / (2 * CTA_WARPS);
constexpr int MAXB = 16;      // max measurement dimension

// status codes (mirrored in include/ttgbf.h)
enum Status : int {
  OK = 0,
  E_ARG = 1,          // ValueError: bad shape / config
  E_NONFINITE = 2,    // ValueError: evaluator returned a non-finite value
  E_DEGENERATE = 3,   // DegenerateDensityError
  E_WORKSPACE = 4,    // per-filter workspace exhausted
  E_CACHE = 5,        // evaluator cache capacity exhausted
  E_CUDA = 6,
  E_LINALG = 7,       // singular dynamics (numpy.linalg.LinAlgError)
  E_DENSE_GUARD = 8,  // DenseGuardError
  E_STATE_CAP = 9,    // output TT larger than the state slab (not an arena failure)
};

#define CK(expr) do { int _st = (expr); if (_st) return _st; } while (0)

HD int64_t clk() {
#if ENGINE_DEVICE
  return (int64_t)clock64();
#else
  return 0;
#endif
}
// profile scope: leader accumulates elapsed SM cycles into ctx.prof[cat]
struct ProfScope {
  const int64_t* dummy;
  int64_t* slot;
  int64_t t0;
  HD ProfScope(int64_t* p, int tid, int cat) : dummy(nullptr), slot((p && tid == 0) ? p + cat : nullptr), t0(clk()) {}
  HD ~ProfScope() { if (slot) *slot += clk() - t0; }
};
#define PROF(c, cat) ::tg::ProfScope _prof_##cat((c).prof, (c).tid, cat)

// Quotient / remainder of loop indices: the 32-bit divide when both operands
// are below 2^31 (the 64-bit one costs ~5x more instructions on the device).
HD int64_t qdiv(int64_t e, int64_t d) {
  return ((e | d) >> 31) == 0 ? (int64_t)((unsigned)e / (unsigned)d) : e / d;
}
HD int64_t qmod(int64_t e, int64_t d) {
  return ((e | d) >> 31) == 0 ? (int64_t)((unsigned)e % (unsigned)d) : e % d;
}
HD int imin(int a, int b) { return a < b ? a : b; }
HD int imax(int a, int b) { return a > b ? a : b; }
HD int64_t lmin(int64_t a, int64_t b) { return a < b ? a : b; }
HD int64_t lmax(int64_t a, int64_t b) { return a > b ? a : b; }

// ---------------------------------------------------------------------------
// CTA context
// ---------------------------------------------------------------------------
struct Ctx {
  int tid;
  int nt;
  double* red;   // shared scratch, >= 64 doubles (+ 64 ints after it)
  int* ired;     // shared scratch, >= 64 ints
  int64_t* prof; // optional per-CTA profile counters (leader), may be null

  HD void sync() const {
#if ENGINE_DEVICE
    __syncthreads();
#endif
  }
  HD bool leader() const { return tid == 0; }
};

// Deterministic CTA-wide sum: warp shuffles, then every thread adds the warp
// partials in warp order.  All threads must call; all receive the result.
HD double block_sum(const Ctx& c, double v) {
#if ENGINE_DEVICE
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = c.tid >> 5, l = c.tid & 31, nw = (c.nt + 31) >> 5;
  __syncthreads();
  if (l == 0) c.red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < nw; ++i) s += c.red[i];
  __syncthreads();
  return s;
#else
  (void)c;
  return v;
#endif
}

HD double block_max(const Ctx& c, double v) {
#if ENGINE_DEVICE
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = c.tid >> 5, l = c.tid & 31, nw = (c.nt + 31) >> 5;
  __syncthreads();
  if (l == 0) c.red[w] = v;
  __syncthreads();
  double s = c.red[0];
  for (int i = 1; i < nw; ++i) s = fmax(s, c.red[i]);
  __syncthreads();
  return s;
#else
  (void)c;
  return v;
#endif
}

HD int64_t block_sum_i64(const Ctx& c, int64_t v) {
#if ENGINE_DEVICE
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = c.tid >> 5, l = c.tid & 31, nw = (c.nt + 31) >> 5;
  int64_t* r = reinterpret_cast<int64_t*>(c.red);
  __syncthreads();
  if (l == 0) r[w] = v;
  __syncthreads();
  int64_t s = 0;
  for (int i = 0; i < nw; ++i) s += r[i];
  __syncthreads();
  return s;
#else
  (void)c;
  return v;
#endif
}

// argmax with numpy semantics: largest value, first index among ties.
struct ValIdx {
  double v;
  int64_t i;
};
HD ValIdx vi_better(ValIdx a, ValIdx b) {
  if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}
HD ValIdx block_argmax(const Ctx& c, ValIdx x) {
#if ENGINE_DEVICE
  for (int o = 16; o > 0; o >>= 1) {
    ValIdx y;
    y.v = __shfl_xor_sync(0xffffffffu, x.v, o);
    y.i = __shfl_xor_sync(0xffffffffu, x.i, o);
    x = vi_better(x, y);
  }
  const int w = c.tid >> 5, l = c.tid & 31, nw = (c.nt + 31) >> 5;
  int64_t* ri = reinterpret_cast<int64_t*>(c.red + 32);
  __syncthreads();
  if (l == 0) { c.red[w] = x.v; ri[w] = x.i; }
  __syncthreads();
  ValIdx s{c.red[0], ri[0]};
  for (int i = 1; i < nw; ++i) s = vi_better(s, ValIdx{c.red[i], ri[i]});
  __syncthreads();
  return s;
#else
  (void)c;
  return x;
#endif
}

// Broadcast a value computed by the leader (after a serial section).
HD double bcast(const Ctx& c, double v) {
#if ENGINE_DEVICE
  __syncthreads();
  if (c.tid == 0) c.red[0] = v;
  __syncthreads();
  double r = c.red[0];
  __syncthreads();
  return r;
#else
  (void)c;
  return v;
#endif
}
HD int64_t bcast_i(const Ctx& c, int64_t v) {
#if ENGINE_DEVICE
  int64_t* r = reinterpret_cast<int64_t*>(c.red);
  __syncthreads();
  if (c.tid == 0) r[0] = v;
  __syncthreads();
  int64_t x = r[0];
  __syncthreads();
  return x;
#else
  (void)c;
  return v;
#endif
}

// ---------------------------------------------------------------------------
// Workspace arena (per filter).  Every thread keeps an identical copy and
// performs the same allocation sequence, so pointers agree without barriers.
// ---------------------------------------------------------------------------
struct Arena {
  char* base;
  size_t cap;
  size_t off;
  size_t peak;

  template <class T>
  HD T* alloc(size_t n) {
    size_t a = (off + 255) & ~(size_t)255;
    size_t need = a + n * sizeof(T);
    if (need > cap) return nullptr;
    off = need;
    if (off > peak) peak = off;
    return reinterpret_cast<T*>(base + a);
  }
  HD size_t mark() const { return off; }
  HD void release(size_t m) { off = m; }
};

// arena over slot `item` of a slab of equal workspaces
HD Arena make_ws_arena(void* ws, int64_t ws_bytes, int item) {
  Arena a;
  a.base = reinterpret_cast<char*>(ws) + (int64_t)item * ws_bytes;
  a.cap = (size_t)ws_bytes;
  a.off = 0;
  a.peak = 0;
  return a;
}

#define ALLOC(ptr, T, n, ar) do { (ptr) = (ar).template alloc<T>((size_t)(n)); if (!(ptr)) return ::tg::E_WORKSPACE; } while (0)

// ---------------------------------------------------------------------------
// parallel helpers
// ---------------------------------------------------------------------------
HD void par_fill(const Ctx& c, double* p, int64_t n, double v) {
  for (int64_t i = c.tid; i < n; i += c.nt) p[i] = v;
}
// Copy with 16-byte accesses where dst and src share their alignment (half
// the load/store instructions of the element loop; same bytes written).
HD void par_copy(const Ctx& c, double* dst, const double* src, int64_t n) {
#if ENGINE_DEVICE
  if ((((uintptr_t)dst ^ (uintptr_t)src) & 15) == 0) {
    const int64_t head = (((uintptr_t)dst & 15) != 0) ? 1 : 0;
    if (head && c.tid == 0 && n > 0) dst[0] = src[0];
    const int64_t nv = (n - head) / 2;
    double2* d2 = reinterpret_cast<double2*>(dst + head);
    const double2* s2 = reinterpret_cast<const double2*>(src + head);
    for (int64_t i = c.tid; i < nv; i += c.nt) d2[i] = s2[i];
    for (int64_t i = head + 2 * nv + c.tid; i < n; i += c.nt) dst[i] = src[i];
    return;
  }
#endif
  for (int64_t i = c.tid; i < n; i += c.nt) dst[i] = src[i];
}
// int32 fill with 16-byte stores (p 16-byte aligned -- arena allocations are).
HD void par_fill_i32(const Ctx& c, int32_t* p, int64_t n, int32_t v) {
#if ENGINE_DEVICE
  if (((uintptr_t)p & 15) == 0) {
    const int64_t nv = n / 4;
    int4* p4 = reinterpret_cast<int4*>(p);
    const int4 v4 = make_int4(v, v, v, v);
    const int64_t tid = c.tid, nt = c.nt;   // locals: four stores in flight, no reload of the context
    int64_t i = tid;
    for (; i + 3 * nt < nv; i += 4 * nt) {
      p4[i] = v4;
      p4[i + nt] = v4;
      p4[i + 2 * nt] = v4;
      p4[i + 3 * nt] = v4;
    }
    for (; i < nv; i += nt) p4[i] = v4;
    for (int64_t q = 4 * nv + tid; q < n; q += nt) p[q] = v;
    return;
  }
#endif
  for (int64_t i = c.tid; i < n; i += c.nt) p[i] = v;
}

}  // namespace tg
