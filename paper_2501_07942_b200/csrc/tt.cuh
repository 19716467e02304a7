// Tensor-train operations of the step engine (CTA-cooperative, FP64).
//
// Layout: core k is a C-order block (r[k], n[k], r[k+1]) -- the reference's
// layout (tensor_train.py:1-24) -- so core k viewed column-major is the
// (n[k]*r[k+1]) x r[k] matrix whose thin QR the rounding sweep needs.
#pragma once
#include "common.cuh"
#include "linalg.cuh"
#include "la2.cuh"
#if defined(ENGINE_HOSTSIM) && defined(ENGINE_TRACE)
#include <stdio.h>
#endif

namespace tg {

struct TT {
  int d;
  int n[MAXD];
  int r[MAXD + 1];
  double* c[MAXD];
  HD int64_t size(int k) const { return (int64_t)r[k] * n[k] * r[k + 1]; }
  HD int64_t total() const {
    int64_t s = 0;
    for (int k = 0; k < d; ++k) s += size(k);
    return s;
  }
};

HDN int tt_alloc(Arena& ar, TT& t, int d, const int* n, const int* r) {
  t.d = d;
  for (int k = 0; k < d; ++k) t.n[k] = n[k];
  for (int k = 0; k <= d; ++k) t.r[k] = r[k];
  for (int k = 0; k < d; ++k) ALLOC(t.c[k], double, t.size(k), ar);
  return OK;
}

HDN int tt_clone(const Ctx& c, Arena& ar, const TT& src, TT& dst) {
  CK(tt_alloc(ar, dst, src.d, src.n, src.r));
  for (int k = 0; k < src.d; ++k) par_copy(c, dst.c[k], src.c[k], src.size(k));
  c.sync();
  return OK;
}

// ---------------------------------------------------------------------------
// sum of all entries (tensor_train.py:283-288): v = 1; v = v @ core.sum(1)
// ---------------------------------------------------------------------------
HDN double tt_sum(const Ctx& c, const TT& t, double* ws) {
  // ws: 2 * maxr + blockDim doubles
  int maxr = 1;
  for (int k = 0; k <= t.d; ++k) maxr = imax(maxr, t.r[k]);
  double* v = ws;
  double* w = ws + maxr;
  double* part = ws + 2 * maxr;   // partial sums of the narrow-bond path
  if (c.leader()) v[0] = 1.0;
  c.sync();
  for (int k = 0; k < t.d; ++k) {
    const int rl = t.r[k], n = t.n[k], rr = t.r[k + 1];
    if (2 * rr <= c.nt) {
      // narrow right bond: G = nt / rr thread groups share the left index
      // (group g takes a = g, g + G, ...), partials summed in group order
      const int G = c.nt / rr;
      const int g = c.tid / rr, b = c.tid % rr;
      if (g < G) {
        double acc = 0.0;
        for (int a = g; a < rl; a += G) {
          const double* p = t.c[k] + (int64_t)a * n * rr + b;
          double s = 0.0;
          for (int i = 0; i < n; ++i) s += p[(int64_t)i * rr];
          acc = fma(v[a], s, acc);
        }
        part[g * rr + b] = acc;
      }
      c.sync();
      if (c.tid < rr) {
        double acc = 0.0;
        for (int q = 0; q < G; ++q) acc += part[q * rr + c.tid];
        w[c.tid] = acc;
      }
    } else {
      for (int b = c.tid; b < rr; b += c.nt) {
        double acc = 0.0;
        for (int a = 0; a < rl; ++a) {
          const double* p = t.c[k] + (int64_t)a * n * rr + b;
          double s = 0.0;
          for (int i = 0; i < n; ++i) s += p[(int64_t)i * rr];
          acc = fma(v[a], s, acc);
        }
        w[b] = acc;
      }
    }
    c.sync();
    double* tmp = v; v = w; w = tmp;
  }
  double res = v[0];
  c.sync();
  return res;
}

// scale core 0 (tensor_train.py:291-295)
HDN void tt_scale(const Ctx& c, TT& t, double s) {
  for (int64_t e = c.tid; e < t.size(0); e += c.nt) t.c[0][e] *= s;
  c.sync();
}

// ---------------------------------------------------------------------------
// Moments: for each core the three contractions M_p = sum_i core[:,i,:] x(i)^p
// (p = 0,1,2), then chain products for mass, d first and d(d+1)/2 second raw
// moments (filters.py:297-322 with tt_dot of tensor_train.py:269-275).
// out: [0] = sum (un-normalised), [1..d] first, then second moments (i<=j,
// row-major upper triangle), all un-normalised (divide by sum).
// ---------------------------------------------------------------------------
HDN int tt_moments(const Ctx& c, Arena& ar, const TT& t, const double* const* axes, double* out) {
  const int d = t.d;
  size_t mk = ar.mark();
  double* M[MAXD][3];
  for (int k = 0; k < d; ++k) {
    const int rl = t.r[k], n = t.n[k], rr = t.r[k + 1];
    for (int p = 0; p < 3; ++p) ALLOC(M[k][p], double, (int64_t)rl * rr, ar);
    for (int64_t e = c.tid; e < (int64_t)rl * rr; e += c.nt) {
      const int a = (int)(qdiv(e, rr)), b = (int)(qmod(e, rr));
      const double* g = t.c[k] + (int64_t)a * n * rr + b;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0;
      for (int i = 0; i < n; ++i) {
        const double x = axes[k][i];
        const double v = g[(int64_t)i * rr];
        s0 += v;
        s1 = fma(v, x, s1);
        s2 = fma(v, x * x, s2);
      }
      M[k][0][e] = s0;
      M[k][1][e] = s1;
      M[k][2][e] = s2;
    }
  }
  c.sync();
  int maxr = 1;
  for (int k = 0; k <= d; ++k) maxr = imax(maxr, t.r[k]);
  const int nmom = 1 + d + d * (d + 1) / 2;
  double* vec;
  ALLOC(vec, double, (int64_t)2 * maxr * nmom, ar);
  // each thread handles whole chains for a subset of moments (tiny work)
  for (int q = c.tid; q < nmom; q += c.nt) {
    int pi = -1, pj = -1;
    if (q >= 1 && q <= d) pi = q - 1;
    if (q > d) {
      int idx = q - d - 1;
      for (int i = 0; i < d; ++i)
        for (int j = i; j < d; ++j) {
          if (idx == 0) { pi = i; pj = j; }
          --idx;
        }
    }
    double* v = vec + (int64_t)2 * maxr * q;
    double* w = v + maxr;
    v[0] = 1.0;
    for (int k = 0; k < d; ++k) {
      int p = (k == pi) + (k == pj);
      const double* m = M[k][p];
      const int rl = t.r[k], rr = t.r[k + 1];
      for (int b = 0; b < rr; ++b) {
        double acc = 0.0;
        for (int a = 0; a < rl; ++a) acc = fma(v[a], m[(int64_t)a * rr + b], acc);
        w[b] = acc;
      }
      double* tmp = v; v = w; w = tmp;
    }
    out[q] = v[0];
  }
  c.sync();
  ar.release(mk);
  return OK;
}

// ---------------------------------------------------------------------------
// Point evaluation.  One warp per point; the running row vector lives in
// SMEM (per warp 2*maxr doubles at `sm`).  Integer indices (K x d, int32) for
// tt_eval_many (tensor_train.py:129-158); continuous points with 2-tap
// multilinear weights for tt_eval_at_points (tt_algorithms.py:721-745).
// ---------------------------------------------------------------------------
struct AxisGeom {  // equidistant axis: first value, step, count
  double a0, h;
  int n;
};

// (cell, frac, inside) exactly as tt_algorithms.py:673-684
HD void axis_cell(const AxisGeom& g, double x, int* cell, double* frac, bool* inside) {
  const double pos = (x - g.a0) / g.h;
  const double eps = 1e-9;
  *inside = (pos >= -eps) && (pos <= (double)(g.n - 1) + eps);
  double fl = floor(pos);
  // clip(floor(pos), 0, n-2) as integers (floor of huge values saturates)
  int ci;
  if (!(fl >= 0.0)) ci = 0;
  else if (fl > (double)(g.n - 2)) ci = g.n - 2;
  else ci = (int)fl;
  *cell = ci;
  double f = pos - (double)ci;
  *frac = f < 0.0 ? 0.0 : (f > 1.0 ? 1.0 : f);
}

// generic chain evaluation: `slice(k, a, b)` returns core_k[a, i_k, b] for the
// point; K points; out[K]
#if ENGINE_DEVICE
// Warp-per-point chain with the running row vector held in registers: lane l
// owns entries l, l+32, ... (S slots); v[a] is broadcast by shuffle and each
// lane accumulates its output columns from coalesced core-row loads.
template <int S, int P, class Slice>
__device__ __forceinline__ void chain_regs(const Ctx& c, const TT& t, int64_t K, Slice& s0, double* out) {
  // P points per warp in flight: P independent load streams per step hide
  // the L2 latency of the core-row reads (the cores do not fit in L1).
  Slice sl_[P];
#pragma unroll
  for (int u = 0; u < P; ++u) sl_[u] = s0;
  const int nwarps = c.nt >> 5, warp = c.tid >> 5, lane = c.tid & 31;
  for (int64_t p0 = P * (int64_t)warp; p0 < K; p0 += P * (int64_t)nwarps) {
    double v[P][S];
    bool dead[P], has[P];
#pragma unroll
    for (int u = 0; u < P; ++u) {
      has[u] = p0 + u < K;
      dead[u] = !has[u];
#pragma unroll
      for (int q = 0; q < S; ++q) v[u][q] = (q == 0 && lane == 0) ? 1.0 : 0.0;
    }
    for (int k = 0; k < t.d; ++k) {
      const int rl = t.r[k], rr = t.r[k + 1];
      const int64_t sa = (int64_t)t.n[k] * rr;
      bool all_dead = true;
#pragma unroll
      for (int u = 0; u < P; ++u) {
        if (!dead[u]) dead[u] = !sl_[u].prepare(k, p0 + u);
        all_dead = all_dead && dead[u];
      }
      if (all_dead) break;
      const double *lo[P], *hi[P];
      double wl[P], wh[P];
#pragma unroll
      for (int u = 0; u < P; ++u) {
        if (!dead[u]) sl_[u].row(k, &lo[u], &hi[u], &wl[u], &wh[u]);
        else { lo[u] = hi[u] = t.c[k]; wl[u] = wh[u] = 0.0; }   // finished / outside: row 0, discarded
      }
      double a[P][S];
#pragma unroll
      for (int u = 0; u < P; ++u)
#pragma unroll
        for (int q = 0; q < S; ++q) a[u][q] = 0.0;
#pragma unroll
      for (int sl = 0; sl < S; ++sl) {
        if (sl * 32 < rl) {
          const int amax = imin(32, rl - sl * 32);
          const double* r[P];
          const double* h[P];
#pragma unroll
          for (int u = 0; u < P; ++u) {
            r[u] = lo[u] + (int64_t)(sl * 32) * sa + lane;
            h[u] = hi[u] + (int64_t)(sl * 32) * sa + lane;
          }
#pragma unroll 2
          for (int l = 0; l < amax; ++l) {
            double va[P];
#pragma unroll
            for (int u = 0; u < P; ++u) va[u] = __shfl_sync(0xffffffffu, v[u][sl], l);
#pragma unroll
            for (int q = 0; q < S; ++q) {
              if (q * 32 + lane < rr) {
#pragma unroll
                for (int u = 0; u < P; ++u) {
                  double x = r[u][q * 32];
                  if (Slice::kBlend) x = x * wl[u] + h[u][q * 32] * wh[u];
                  a[u][q] = fma(va[u], x, a[u][q]);
                }
              }
            }
#pragma unroll
            for (int u = 0; u < P; ++u) { r[u] += sa; h[u] += sa; }
          }
        }
      }
#pragma unroll
      for (int u = 0; u < P; ++u)
#pragma unroll
        for (int q = 0; q < S; ++q) v[u][q] = a[u][q];
    }
#pragma unroll
    for (int u = 0; u < P; ++u) {
      const double o = __shfl_sync(0xffffffffu, v[u][0], 0);
      if (lane == 0 && has[u]) out[p0 + u] = dead[u] ? 0.0 : o;
    }
  }
  c.sync();
}
#endif

template <class Slice>
HDN void tt_chain_eval(const Ctx& c, const TT& t, int64_t K, Slice slice, double* out, double* sm) {
  int maxr = 1;
  for (int k = 0; k <= t.d; ++k) maxr = imax(maxr, t.r[k]);
#if ENGINE_DEVICE
  if (maxr <= 32) { chain_regs<1, 4>(c, t, K, slice, out); return; }
  if (maxr <= 64) { chain_regs<2, 2>(c, t, K, slice, out); return; }
  if (maxr <= 128) { chain_regs<4, 2>(c, t, K, slice, out); return; }
  const int nwarps = c.nt >> 5, warp = c.tid >> 5, lane = c.tid & 31;
  double* v = sm + (int64_t)warp * 2 * maxr;
  double* w = v + maxr;
  for (int64_t p = warp; p < K; p += nwarps) {
    if (lane == 0) v[0] = 1.0;
    __syncwarp();
    double* vv = v;
    double* ww = w;
    bool dead = false;
    for (int k = 0; k < t.d; ++k) {
      const int rl = t.r[k], rr = t.r[k + 1];
      if (!slice.prepare(k, p)) { dead = true; break; }
      for (int b = lane; b < rr; b += 32) {
        double acc = 0.0;
        for (int a = 0; a < rl; ++a) acc = fma(vv[a], slice.at(k, a, b), acc);
        ww[b] = acc;
      }
      __syncwarp();
      double* tmp = vv; vv = ww; ww = tmp;
    }
    if (lane == 0) out[p] = dead ? 0.0 : vv[0];
    __syncwarp();
  }
  c.sync();
#else
  double* v = sm;
  double* w = sm + maxr;
  for (int64_t p = 0; p < K; ++p) {
    v[0] = 1.0;
    double* vv = v;
    double* ww = w;
    bool dead = false;
    for (int k = 0; k < t.d; ++k) {
      const int rl = t.r[k], rr = t.r[k + 1];
      if (!slice.prepare(k, p)) { dead = true; break; }
      for (int b = 0; b < rr; ++b) {
        double acc = 0.0;
        for (int a = 0; a < rl; ++a) acc = fma(vv[a], slice.at(k, a, b), acc);
        ww[b] = acc;
      }
      double* tmp = vv; vv = ww; ww = tmp;
    }
    out[p] = dead ? 0.0 : vv[0];
  }
#endif
}

struct IndexSlice {
  const TT* t;
  const int32_t* idx;  // K x d
  int i;
  static constexpr bool kBlend = false;
  HD bool prepare(int k, int64_t p) { i = idx[p * t->d + k]; return true; }
  HD double at(int k, int a, int b) const {
    return t->c[k][((int64_t)a * t->n[k] + i) * t->r[k + 1] + b];
  }
  HD void row(int k, const double** lo, const double** hi, double* wl, double* wh) const {
    *lo = t->c[k] + (int64_t)i * t->r[k + 1];
    *hi = *lo;
    *wl = 1.0;
    *wh = 0.0;
  }
  HD bool locate(int k, int64_t p, int* s, double* wl, double* wh) const {
    *s = idx[p * t->d + k];
    *wl = 1.0;
    *wh = 0.0;
    return true;
  }
};

HDN void tt_eval_idx(const Ctx& c, const TT& t, const int32_t* idx, int64_t K, double* out, double* sm) {
  IndexSlice s{&t, idx, 0};
  tt_chain_eval(c, t, K, s, out, sm);
}

// Evaluation of the TT at continuous points produced by a functor
// `pt(p, k)` (coordinate k of point p) on axes `geo`; zero outside the hull.
template <class PointFn>
struct PointSlice {
  const TT* t;
  const AxisGeom* geo;
  PointFn pt;
  int cell;
  double frac;
  HD bool prepare(int k, int64_t p) {
    bool inside;
    axis_cell(geo[k], pt(p, k), &cell, &frac, &inside);
    return inside;
  }
  static constexpr bool kBlend = true;
  HD double at(int k, int a, int b) const {
    const int64_t rr = t->r[k + 1];
    const double* base = t->c[k] + ((int64_t)a * t->n[k] + cell) * rr + b;
    // lo * (1 - frac) + hi * frac, as tt_algorithms.py:741
    return base[0] * (1.0 - frac) + base[rr] * frac;
  }
  HD void row(int k, const double** lo, const double** hi, double* wl, double* wh) const {
    const int64_t rr = t->r[k + 1];
    *lo = t->c[k] + (int64_t)cell * rr;
    *hi = *lo + rr;
    *wl = 1.0 - frac;
    *wh = frac;
  }
  HD bool locate(int k, int64_t p, int* s, double* wl, double* wh) const {
    int cl;
    double fr;
    bool inside;
    axis_cell(geo[k], pt(p, k), &cl, &fr, &inside);
    *s = cl;
    *wl = 1.0 - fr;
    *wh = fr;
    return inside;
  }
};

struct PtsFn {
  const double* pts;
  int d;
  HD double operator()(int64_t p, int k) const { return pts[p * d + k]; }
};

// ---------------------------------------------------------------------------
// Core-major TT evaluation for batches: for each core the points are
// bucketed by their slice (counting sort), the buckets are cut into tiles of
// 8 points, and each warp takes whole tiles: DMMA (m8n8k4 f64) of the 8
// running row vectors against the slice (and its right neighbour for 2-tap
// interpolation), B fragments read straight from the core in global memory
// (L2-resident), so there is no CTA barrier per slice and warps work on
// different slices at once.  A row's result depends only on its own A row,
// so the (atomic) order of points inside a bucket does not change any value.
// Small batches go through tt_chain_eval.
// ---------------------------------------------------------------------------
constexpr int64_t BUCKET_MIN_K = 64;
constexpr int BUCKET_MAXR = 160;
#ifndef TTGBF_EVAL_TILE
#define TTGBF_EVAL_TILE 16
#endif
constexpr int EVAL_TILE = TTGBF_EVAL_TILE;   // points per warp tile of the bucketed evaluation

template <class Slice>
HDN int tt_eval_bucketed(const Ctx& c, Arena& ar, const TT& t, int64_t K, Slice slice, double* out, double* sm) {
  int maxr = 1, maxn = 1;
  for (int k = 0; k <= t.d; ++k) maxr = imax(maxr, t.r[k]);
  for (int k = 0; k < t.d; ++k) maxn = imax(maxn, t.n[k]);
  if (maxr > BUCKET_MAXR || K < BUCKET_MIN_K || maxn > 1000) {
    tt_chain_eval(c, t, K, slice, out, sm);
    return OK;
  }
  const int d = t.d;
  const size_t mk = ar.mark();
  double *V0, *V1, *wlv, *whv;
  int32_t *sid, *perm;
  uint8_t* dead;
  ALLOC(V0, double, K * maxr, ar);
  ALLOC(V1, double, K * maxr, ar);
  ALLOC(wlv, double, K, ar);
  ALLOC(whv, double, K, ar);
  ALLOC(sid, int32_t, K, ar);
  ALLOC(perm, int32_t, K, ar);
  ALLOC(dead, uint8_t, K, ar);
  // core 0 (left rank 1): V0[p, b] = blended slice row
  {
    const int r1 = t.r[1];
    for (int64_t p = c.tid; p < K; p += c.nt) {
      int sl;
      double wl, wh;
      const bool in = slice.locate(0, p, &sl, &wl, &wh);
      dead[p] = in ? 0 : 1;
      const double* lo = t.c[0] + (int64_t)sl * r1;
      for (int b = 0; b < r1; ++b) {
        double x = lo[b];
        if (Slice::kBlend) x = x * wl + lo[r1 + b] * wh;
        V0[p * maxr + b] = x;
      }
    }
  }
  c.sync();
  double* Vin = V0;
  double* Vout = V1;
  int* cur = reinterpret_cast<int*>(sm);   // bucket cursors   (n + 1 <= 1001)
  int* offs = cur + 1024;                  // bucket offsets   (n + 1)
  int* toffs = offs + 1024;                // tile offsets     (n + 1)
  for (int k = 1; k < d; ++k) {
    const int rl = t.r[k], rr = t.r[k + 1], n = t.n[k];
    for (int q = c.tid; q <= n; q += c.nt) cur[q] = 0;
    c.sync();
    for (int64_t p = c.tid; p < K; p += c.nt) {
      int sl;
      double wl, wh;
      const bool in = slice.locate(k, p, &sl, &wl, &wh);
      if (!in) dead[p] = 1;
      sid[p] = sl;
      wlv[p] = wl;
      whv[p] = wh;
#if ENGINE_DEVICE
      atomicAdd(&cur[sl], 1);
#else
      cur[sl] += 1;
#endif
    }
    c.sync();
    if (c.leader()) {
      int acc = 0, tacc = 0;
      for (int q = 0; q < n; ++q) {
        const int h = cur[q];
        offs[q] = acc;
        toffs[q] = tacc;
        cur[q] = acc;
        acc += h;
        tacc += (h + EVAL_TILE - 1) / EVAL_TILE;
      }
      offs[n] = acc;
      toffs[n] = tacc;
    }
    c.sync();
    for (int64_t p = c.tid; p < K; p += c.nt) {
#if ENGINE_DEVICE
      const int pos = atomicAdd(&cur[sid[p]], 1);
#else
      const int pos = cur[sid[p]]++;
#endif
      perm[pos] = (int32_t)p;
    }
    c.sync();
    const double* G = t.c[k];
    const int64_t sa = (int64_t)n * rr;
#if ENGINE_DEVICE
    {
      // Fragments (PTX m8n8k4 .f64): A(row=lane/4, col=lane%4),
      // B(row=lane%4, col=lane/4), C(row=lane/4, cols 2*(lane%4)+{0,1}).
      const int nwarps = c.nt >> 5, warp = c.tid >> 5, lane = c.tid & 31;
      const int ar_ = lane >> 2, ac = lane & 3;
      const int ntiles = toffs[n];
      for (int tile = warp; tile < ntiles; tile += nwarps) {
        int lo_ = 0, hi_ = n;                     // slice: toffs[s] <= tile < toffs[s+1]
        while (hi_ - lo_ > 1) {
          const int mid = (lo_ + hi_) >> 1;
          if (toffs[mid] <= tile) lo_ = mid; else hi_ = mid;
        }
        const int sl = lo_;
        // EVAL_TILE points of one slice per tile: every B fragment (a 4 x 8
        // piece of the slice, the load the loop waits on) feeds EVAL_TILE / 8
        // A fragments
        constexpr int NA = EVAL_TILE / 8;
        const int q0 = offs[sl] + EVAL_TILE * (tile - toffs[sl]);
        const int end = offs[sl + 1];
        bool rv[NA];
        int pp[NA];
        const double* vr[NA];
        double wl[NA], wh[NA];
#pragma unroll
        for (int a = 0; a < NA; ++a) {
          const int qa = q0 + 8 * a + ar_;
          rv[a] = qa < end;
          pp[a] = perm[rv[a] ? qa : q0];
          vr[a] = Vin + (int64_t)pp[a] * maxr;
          wl[a] = wlv[pp[a]];
          wh[a] = whv[pp[a]];
        }
        const double* Gs = G + (int64_t)sl * rr;
        const bool has_hi = sl + 1 < n;
        for (int n0 = 0; n0 < rr; n0 += 8) {
          double cc[NA][2], ee[NA][2];
#pragma unroll
          for (int a = 0; a < NA; ++a) cc[a][0] = cc[a][1] = ee[a][0] = ee[a][1] = 0.0;
          const int bcol = n0 + ar_;
#pragma unroll 4
          for (int k0 = 0; k0 < rl; k0 += 4) {
            const int ka = k0 + ac;
            double af[NA];
#pragma unroll
            for (int a = 0; a < NA; ++a) af[a] = (rv[a] && ka < rl) ? vr[a][ka] : 0.0;
            const bool bv = ka < rl && bcol < rr;
            const double* gp = Gs + (int64_t)ka * sa + bcol;
            const double bf = bv ? gp[0] : 0.0;
#pragma unroll
            for (int a = 0; a < NA; ++a)
              asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                           : "+d"(cc[a][0]), "+d"(cc[a][1]) : "d"(af[a]), "d"(bf));
            if (Slice::kBlend) {
              const double bf2 = (bv && has_hi) ? gp[rr] : 0.0;
#pragma unroll
              for (int a = 0; a < NA; ++a)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                             : "+d"(ee[a][0]), "+d"(ee[a][1]) : "d"(af[a]), "d"(bf2));
            }
          }
          const int oc = n0 + 2 * ac;
#pragma unroll
          for (int a = 0; a < NA; ++a) {
            if (!rv[a]) continue;
            double* orow = Vout + (int64_t)pp[a] * maxr;
            if (Slice::kBlend) {
              if (oc < rr) orow[oc] = cc[a][0] * wl[a] + ee[a][0] * wh[a];
              if (oc + 1 < rr) orow[oc + 1] = cc[a][1] * wl[a] + ee[a][1] * wh[a];
            } else {
              if (oc < rr) orow[oc] = cc[a][0];
              if (oc + 1 < rr) orow[oc + 1] = cc[a][1];
            }
          }
        }
      }
    }
#else
    for (int sl = 0; sl < n; ++sl) {
      for (int q0 = offs[sl]; q0 < offs[sl + 1]; ++q0) {
        const int p = perm[q0];
        const double wl = wlv[p], wh = whv[p];
        for (int bb = 0; bb < rr; ++bb) {
          double acc = 0.0, acc2 = 0.0;
          for (int a = 0; a < rl; ++a) {
            const double g = G[a * sa + (int64_t)sl * rr + bb];
            acc = fma(Vin[(int64_t)p * maxr + a], g, acc);
            if (Slice::kBlend) {
              const double g2 = (sl + 1 < n) ? G[a * sa + (int64_t)(sl + 1) * rr + bb] : 0.0;
              acc2 = fma(Vin[(int64_t)p * maxr + a], g2, acc2);
            }
          }
          Vout[(int64_t)p * maxr + bb] = Slice::kBlend ? acc * wl + acc2 * wh : acc;
        }
      }
    }
#endif
    c.sync();
    double* tmp = Vin; Vin = Vout; Vout = tmp;
  }
  for (int64_t p = c.tid; p < K; p += c.nt) out[p] = dead[p] ? 0.0 : Vin[p * maxr];
  c.sync();
  ar.release(mk);
  return OK;
}

// ---------------------------------------------------------------------------
// Hadamard product cores (tensor_train.py:252-266)
// ---------------------------------------------------------------------------
HDN int tt_hadamard(const Ctx& c, Arena& ar, const TT& A, const TT& B, TT& out) {
  int n[MAXD], r[MAXD + 1];
  for (int k = 0; k < A.d; ++k) n[k] = A.n[k];
  for (int k = 0; k <= A.d; ++k) r[k] = A.r[k] * B.r[k];
  CK(tt_alloc(ar, out, A.d, n, r));
  for (int k = 0; k < A.d; ++k) {
    const int ra0 = A.r[k], ra1 = A.r[k + 1], rb0 = B.r[k], rb1 = B.r[k + 1], nn = A.n[k];
    // output row (aa0, bb0, i) = outer product of A row (aa0, i, :) and B row
    // (bb0, i, :); rows to warps, row elements to lanes (32-bit index math)
    const int rows = ra0 * rb0 * nn, len = ra1 * rb1;
#if ENGINE_DEVICE
    const int nw = c.nt >> 5, w = c.tid >> 5, lane = c.tid & 31;
#else
    const int nw = 1, w = 0, lane = 0;
#endif
    for (int row = w; row < rows; row += nw) {
      const int i = row % nn, ab = row / nn;
      const int bb0 = ab % rb0, aa0 = ab / rb0;
      const double* ar_ = A.c[k] + ((int64_t)aa0 * nn + i) * ra1;
      const double* br_ = B.c[k] + ((int64_t)bb0 * nn + i) * rb1;
      double* o = out.c[k] + (int64_t)row * len;
#if ENGINE_DEVICE
      for (int col = lane; col < len; col += 32) o[col] = ar_[col / rb1] * br_[col % rb1];
#else
      for (int col = 0; col < len; ++col) o[col] = ar_[col / rb1] * br_[col % rb1];
#endif
    }
  }
  c.sync();
  return OK;
}

// ---------------------------------------------------------------------------
// Separable linear interpolation onto new axes (tt_algorithms.py:687-718)
// ---------------------------------------------------------------------------
HDN int tt_interp(const Ctx& c, Arena& ar, const TT& t, const AxisGeom* old_geo,
                         const double* const* new_axes, TT& out) {
  CK(tt_alloc(ar, out, t.d, t.n, t.r));
  for (int k = 0; k < t.d; ++k) {
    const int rl = t.r[k], n = t.n[k], rr = t.r[k + 1];
    const int64_t tot = out.size(k);
    for (int64_t e = c.tid; e < tot; e += c.nt) {
      const int b = (int)(qmod(e, rr));
      const int j = (int)(qmod(qdiv(e, rr), n));
      const int a = (int)(qdiv(e, (int64_t)rr * n));
      int cell;
      double frac;
      bool inside;
      axis_cell(old_geo[k], new_axes[k][j], &cell, &frac, &inside);
      double v = 0.0;
      if (inside) {
        const double* g = t.c[k] + ((int64_t)a * n + cell) * rr + b;
        v = g[0] * (1.0 - frac) + g[rr] * frac;
      }
      out.c[k][e] = v;
    }
  }
  c.sync();
  return OK;
}

// ---------------------------------------------------------------------------
// Truncation rule (tensor_train.py:165-176)
// ---------------------------------------------------------------------------
HD int keep_rank(const double* s, int k, double delta, int cap, double* tail) {
  int r;
  if (delta > 0.0) {
    double acc = 0.0;
    for (int i = k - 1; i >= 0; --i) { acc += s[i] * s[i]; tail[i] = acc; }
    const double d2 = delta * delta;
    r = k;
    for (int i = 0; i < k; ++i)
      if (tail[i] <= d2) { r = i; break; }
    r = imax(r, 1);
  } else {
    r = imax(k, 1);
  }
  if (cap > 0) r = imin(r, cap);
  return r;
}

// SVD of a row-major (m x n) matrix X (read-only): returns U (m x kk, col-major
// ld m), s (kk), Vt (kk x n, row-major ld n), kk = min(m, n).
HDN int svd_rowmajor(const Ctx& c, Arena& ar, const double* X, int m, int n, double** U_out,
                            double** s_out, double** Vt_out, int* kk_out, double* sm) {
  const int kk = imin(m, n);
  PROF(c, 8);
  double *U, *s, *Vt;
  ALLOC(U, double, (int64_t)m * kk, ar);
  ALLOC(s, double, kk, ar);
  ALLOC(Vt, double, (int64_t)kk * n, ar);
  size_t mk = ar.mark();
  int* perm;
  double* tmp;
  ALLOC(perm, int, kk, ar);
  ALLOC(tmp, double, kk, ar);
  // Work on the orientation with more rows than columns: Y (rows >= cols).
  const bool tall = m >= n;
  const int yr = tall ? m : n, yc = tall ? n : m;   // yc == kk
  double* Y;
  ALLOC(Y, double, (int64_t)yr * yc, ar);
  if (tall) {  // Y = X (col-major copy)
    for (int64_t e = c.tid; e < (int64_t)m * n; e += c.nt) {
      const int i = (int)(qdiv(e, n)), j = (int)(qmod(e, n));
      Y[i + (int64_t)j * m] = X[e];
    }
  } else {     // Y = X^T (col-major (n x m)) == X's buffer
    par_copy(c, Y, X, (int64_t)m * n);
  }
  c.sync();
  // QR preconditioning when Y is much taller than wide
  double* Z = Y;
  int zr = yr;
  double* Qy = nullptr;
  double* Tq = nullptr;
  if (yr > 2 * yc && yc > 1) {
    double* tau;
    ALLOC(tau, double, yc, ar);
    ALLOC(Tq, double, (int64_t)((yc + NB - 1) / NB) * NB * NB, ar);
    CK(geqrf_nb(c, ar, Y, yr, yr, yc, tau, Tq, sm));
    Qy = Y;   // reflectors; Q is applied implicitly below
    ALLOC(Z, double, (int64_t)yc * yc, ar);
    for (int64_t e = c.tid; e < (int64_t)yc * yc; e += c.nt) {
      const int i = (int)(qmod(e, yc)), j = (int)(qdiv(e, yc));
      Z[e] = (i <= j) ? Y[i + (int64_t)j * yr] : 0.0;
    }
    c.sync();
    zr = yc;
  }
  double* Vj;
  ALLOC(Vj, double, (int64_t)yc * yc, ar);
  CK(svd_jacobi(c, Z, zr, zr, yc, Vj, s, perm, tmp));
  // Left vectors of Y: Uy = (Qy *) Z[:, perm]  (yr x kk);  right: Vj[:, perm]
  double* Uy;
  ALLOC(Uy, double, (int64_t)yr * kk, ar);
  if (Qy) {
    // Uy = Q [Z[:, perm]; 0]
    for (int64_t e = c.tid; e < (int64_t)yr * kk; e += c.nt) {
      const int i = (int)(qmod(e, yr)), j = (int)(qdiv(e, yr));
      Uy[e] = (i < zr) ? Z[i + (int64_t)perm[j] * zr] : 0.0;
    }
    c.sync();
    CK(apply_q(c, ar, Qy, yr, yr, yc, Tq, false, Uy, yr, kk, sm));
  } else {
    for (int64_t e = c.tid; e < (int64_t)yr * kk; e += c.nt) {
      const int i = (int)(qmod(e, yr)), j = (int)(qdiv(e, yr));
      Uy[e] = Z[i + (int64_t)perm[j] * zr];
    }
    c.sync();
  }
  if (tall) {  // X = Uy S Vj^T : U = Uy, Vt[j, :] = Vj[:, perm[j]]
    par_copy(c, U, Uy, (int64_t)m * kk);
    for (int64_t e = c.tid; e < (int64_t)kk * n; e += c.nt) {
      const int j = (int)(qdiv(e, n)), q = (int)(qmod(e, n));
      Vt[e] = Vj[q + (int64_t)perm[j] * yc];
    }
  } else {     // X^T = Uy S Vj^T -> X = Vj S Uy^T : U = Vj[:, perm], Vt = Uy^T
    for (int64_t e = c.tid; e < (int64_t)m * kk; e += c.nt) {
      const int i = (int)(qmod(e, m)), j = (int)(qdiv(e, m));
      U[e] = Vj[i + (int64_t)perm[j] * yc];
    }
    for (int64_t e = c.tid; e < (int64_t)kk * n; e += c.nt) {
      const int j = (int)(qdiv(e, n)), q = (int)(qmod(e, n));
      Vt[e] = Uy[q + (int64_t)j * yr];
    }
  }
  c.sync();
  ar.release(mk);
  *U_out = U;
  *s_out = s;
  *Vt_out = Vt;
  *kk_out = kk;
  return OK;
}

// ---------------------------------------------------------------------------
// Rank-revealing truncated SVD of a row-major (m x n) matrix X (read-only).
// Householder QR with column pivoting (largest remaining column first) is
// stopped once the Frobenius norm of the unreduced block falls to eps_abs;
// the p x n leading block [R11 R12] P^T is then factored exactly (QR of its
// transpose + one-sided Jacobi on the p x p triangle).  Dropping the
// unreduced block perturbs every singular value by <= eps_abs and the tail
// energies by <= eps_abs^2, so with eps_abs = 1e-3 * delta the truncation
// rule of tt_round and the kept subspace are unchanged up to ~1e-3 delta.
// eps_abs = 0 gives the full SVD.  s holds all kk = p singular values; only
// the leading nw = min(want, p) vectors are formed (want = 0: all p):
// U (m x nw, col-major), Vt (nw x n, row-major).
// ---------------------------------------------------------------------------
#if ENGINE_DEVICE
// Pivoted-QR trailing update of svd_rrqr: apply the reflector (col, tau t) of
// step j to columns j+1.. (NQ per warp) and recompute their norms below row j.
template <int NQ>
__device__ __forceinline__ void rrqr_update_cols(double* A, int m, int n, int j, const double* col, double t,
                                                 double* cn, int warp, int nwarps, int lane) {
  for (int q0 = j + 1 + warp * NQ; q0 < n; q0 += nwarps * NQ) {
    double w[NQ];
    double* cq[NQ];
#pragma unroll
    for (int u = 0; u < NQ; ++u) {
      w[u] = 0.0;
      cq[u] = A + (int64_t)imin(q0 + u, n - 1) * m;
    }
    for (int r = j + lane; r < m; r += 32) {
      const double v = r == j ? 1.0 : col[r];
#pragma unroll
      for (int u = 0; u < NQ; ++u) w[u] = fma(v, cq[u][r], w[u]);
    }
#pragma unroll
    for (int u = 0; u < NQ; ++u) {
      for (int o = 16; o > 0; o >>= 1) w[u] += __shfl_xor_sync(0xffffffffu, w[u], o);
      w[u] *= t;
    }
    double nr[NQ];
#pragma unroll
    for (int u = 0; u < NQ; ++u) nr[u] = 0.0;
    for (int r = j + lane; r < m; r += 32) {
      const double v = r == j ? 1.0 : col[r];
#pragma unroll
      for (int u = 0; u < NQ; ++u) {
        if (q0 + u < n) {
          const double x = cq[u][r] - w[u] * v;
          cq[u][r] = x;
          if (r > j) nr[u] = fma(x, x, nr[u]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < NQ; ++u) {
      for (int o = 16; o > 0; o >>= 1) nr[u] += __shfl_xor_sync(0xffffffffu, nr[u], o);
      if (lane == 0 && q0 + u < n) cn[q0 + u] = nr[u];
    }
  }
}
#endif

#if ENGINE_DEVICE
// Register-resident form of rrqr_update_cols for columns of at most 32 * RL
// rows below the pivot: a warp loads its column once (all loads in flight),
// forms the dot product, updates and stores it and takes the new norm from
// the registers -- one read and one write of the trailing block per pivot
// step instead of two reads and a write.  Same per-lane accumulation order
// and shuffle tree as rrqr_update_cols, so the values are identical.
template <int RL>
__device__ __noinline__ void rrqr_update_cols_reg(double* A, int m, int n, int j, const double* col, double t,
                                                  double* cn, int warp, int nwarps, int lane) {
  // the reflector is re-read per column (10 KB, L1-resident, shared by the
  // warps): only the column itself is held in registers
  auto vat = [&](int r) { return r == j ? 1.0 : col[r]; };
  for (int qc = j + 1 + warp; qc < n; qc += nwarps) {
    double* cq = A + (int64_t)qc * m;
    double x[RL];
#pragma unroll
    for (int q = 0; q < RL; ++q) {
      const int r = j + lane + 32 * q;
      x[q] = r < m ? cq[r] : 0.0;
    }
    double w = 0.0;
#pragma unroll
    for (int q = 0; q < RL; ++q) {
      const int r = j + lane + 32 * q;
      if (r < m) w = fma(vat(r), x[q], w);
    }
    for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
    w *= t;
    double nr = 0.0;
#pragma unroll
    for (int q = 0; q < RL; ++q) {
      const int r = j + lane + 32 * q;
      if (r < m) {
        const double y = x[q] - w * vat(r);
        cq[r] = y;
        if (r > j) nr = fma(y, y, nr);
      }
    }
    for (int o = 16; o > 0; o >>= 1) nr += __shfl_xor_sync(0xffffffffu, nr, o);
    if (lane == 0) cn[qc] = nr;
  }
}
#endif

HDN int svd_rrqr(const Ctx& c, Arena& ar, const double* X, int m, int n, double eps_abs, double** U_out,
                 double** s_out, double** Vt_out, int* kk_out, double* sm, int want = 0) {
  PROF(c, 8);
  const int kmax = imin(m, n);
  // outputs sized for the worst case (p <= kmax), allocated first
  double *U, *s, *Vt;
  ALLOC(U, double, (int64_t)m * kmax, ar);
  ALLOC(s, double, kmax, ar);
  ALLOC(Vt, double, (int64_t)kmax * n, ar);
  const size_t mk = ar.mark();
  double *A, *cn, *tau;
  int* perm;
  ALLOC(A, double, (int64_t)m * n, ar);     // col-major copy
  ALLOC(cn, double, n, ar);
  ALLOC(tau, double, kmax, ar);
  ALLOC(perm, int, n, ar);
  for (int64_t e = c.tid; e < (int64_t)m * n; e += c.nt) {
    const int i = (int)(qdiv(e, n)), j = (int)(qmod(e, n));
    A[i + (int64_t)j * m] = X[e];
  }
  for (int j = c.tid; j < n; j += c.nt) perm[j] = j;
  c.sync();
#if ENGINE_DEVICE
  const int nwarps = c.nt >> 5, warp = c.tid >> 5, lane = c.tid & 31;
#endif
  // column norms^2 (one warp per column)
#if ENGINE_DEVICE
  for (int j = warp; j < n; j += nwarps) {
    double a = 0.0;
    for (int r = lane; r < m; r += 32) a = fma(A[r + (int64_t)j * m], A[r + (int64_t)j * m], a);
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) cn[j] = a;
  }
#else
  for (int j = 0; j < n; ++j) {
    double a = 0.0;
    for (int r = 0; r < m; ++r) a = fma(A[r + (int64_t)j * m], A[r + (int64_t)j * m], a);
    cn[j] = a;
  }
#endif
  c.sync();
  const double eps2 = eps_abs * eps_abs;
  int p = 0;
  int64_t t_rrqr = clk();
  for (int j = 0; j < kmax; ++j) {
    // remaining energy and pivot
    double part = 0.0;
    ValIdx best{-1.0, 0};
    for (int q = j + c.tid; q < n; q += c.nt) {
      part += cn[q];
      best = vi_better(best, ValIdx{cn[q], q});
    }
    const double rem = block_sum(c, part);
    best = block_argmax(c, best);
    if (rem <= eps2 || best.v <= 0.0) break;
    const int pv = (int)best.i;
    if (pv != j) {
      for (int r = c.tid; r < m; r += c.nt) {
        const double t = A[r + (int64_t)j * m];
        A[r + (int64_t)j * m] = A[r + (int64_t)pv * m];
        A[r + (int64_t)pv * m] = t;
      }
      c.sync();
      if (c.leader()) {
        const int t = perm[j]; perm[j] = perm[pv]; perm[pv] = t;
        const double tc = cn[j]; cn[j] = cn[pv]; cn[pv] = tc;
      }
    }
    c.sync();
    // reflector of column j (rows j..m-1)
    double* col = A + (int64_t)j * m;
    double part2 = 0.0;
    for (int r = j + 1 + c.tid; r < m; r += c.nt) part2 = fma(col[r], col[r], part2);
    const double xn = sqrt(block_sum(c, part2));
    const double alpha = col[j];
    double t, beta, scal;
    larfg(alpha, xn, &t, &beta, &scal);
    for (int r = j + 1 + c.tid; r < m; r += c.nt) col[r] *= scal;
    c.sync();
    if (c.leader()) { col[j] = beta; tau[j] = t; }
    c.sync();
    // apply to the trailing columns and refresh their norms (rows > j)
#if ENGINE_DEVICE
    // several columns per warp when the trailing block is wide: more loads in
    // flight per lane; every column keeps its own accumulation order, so the
    // values are those of the one-column-per-warp loop
    const int ntr = n - j - 1;
    const int rl = (m - j + 31) / 32;
    if (rl <= 8) rrqr_update_cols_reg<8>(A, m, n, j, col, t, cn, warp, nwarps, lane);
    else if (rl <= 16) rrqr_update_cols_reg<16>(A, m, n, j, col, t, cn, warp, nwarps, lane);
    else if (rl <= 28) rrqr_update_cols_reg<28>(A, m, n, j, col, t, cn, warp, nwarps, lane);
    else if (rl <= 42) rrqr_update_cols_reg<42>(A, m, n, j, col, t, cn, warp, nwarps, lane);
    else if (ntr >= 8 * nwarps) rrqr_update_cols<4>(A, m, n, j, col, t, cn, warp, nwarps, lane);
    else if (ntr >= 2 * nwarps) rrqr_update_cols<2>(A, m, n, j, col, t, cn, warp, nwarps, lane);
    else rrqr_update_cols<1>(A, m, n, j, col, t, cn, warp, nwarps, lane);
#else
    for (int q = j + 1; q < n; ++q) {
      double* cq = A + (int64_t)q * m;
      double w = 0.0;
      for (int r = j; r < m; ++r) w = fma(r == j ? 1.0 : col[r], cq[r], w);
      w *= t;
      double nr = 0.0;
      for (int r = j; r < m; ++r) {
        const double v = cq[r] - w * (r == j ? 1.0 : col[r]);
        cq[r] = v;
        if (r > j) nr = fma(v, v, nr);
      }
      cn[q] = nr;
    }
#endif
    c.sync();
    p = j + 1;
  }
  if (c.prof && c.leader()) {
    c.prof[21] += clk() - t_rrqr;
    c.prof[22] += p;            // rank reached by the pivoted QR (sum)
    c.prof[23] += 1;            // svd_rrqr calls
    if (p > c.prof[24]) c.prof[24] = p;
    if (p > 64) c.prof[28] += 1;
  }
  if (p == 0) {   // zero matrix: one zero singular triplet
    for (int64_t e = c.tid; e < m; e += c.nt) U[e] = (e == 0) ? 1.0 : 0.0;
    for (int64_t e = c.tid; e < n; e += c.nt) Vt[e] = (e == 0) ? 1.0 : 0.0;
    if (c.leader()) s[0] = 0.0;
    c.sync();
    ar.release(mk);
    *U_out = U; *s_out = s; *Vt_out = Vt; *kk_out = 1;
    return OK;
  }
  // Bt = (R P^T)^T: n x p col-major, Bt[perm[q], i] = R[i, q] (i <= q)
  int64_t t_sec = clk();
  auto sec = [&](int cat) {
    if (c.prof && c.leader()) { const int64_t t1 = clk(); c.prof[cat] += t1 - t_sec; t_sec = t1; }
  };
  const int nw = want > 0 ? imin(want, p) : p;   // singular vectors needed by the caller
  double *Bt, *tq, *Tq, *Z, *tmp, *Uz, *Vw;
  int* jp;
  ALLOC(Bt, double, (int64_t)n * p, ar);
  for (int64_t e = c.tid; e < (int64_t)n * p; e += c.nt) {
    const int q = (int)(qmod(e, n)), i = (int)(qdiv(e, n));
    Bt[perm[q] + (int64_t)i * n] = (i <= q) ? A[i + (int64_t)q * m] : 0.0;
  }
  c.sync();
  // QR of Bt (n x p, n >= p): Bt = Q2 R2;  R2^T = B's left factor
  ALLOC(tq, double, p, ar);
  ALLOC(Tq, double, (int64_t)((p + NB - 1) / NB) * NB * NB, ar);
  CK(geqrf_nb(c, ar, Bt, n, n, p, tq, Tq, sm));
  // Z = R2^T (p x p, col-major) -> one-sided Jacobi on its columns:
  // R2^T Vj = Uz S  =>  B = R2^T Q2^T = Uz S (Q2 Vj)^T
  ALLOC(Z, double, (int64_t)p * p, ar);
  for (int64_t e = c.tid; e < (int64_t)p * p; e += c.nt) {
    const int i = (int)(qmod(e, p)), j = (int)(qdiv(e, p));     // Z(i, j) = R2(j, i)
    Z[e] = (j <= i) ? Bt[j + (int64_t)i * n] : 0.0;
  }
  ALLOC(tmp, double, p, ar);
  ALLOC(jp, int, p, ar);
  ALLOC(Uz, double, (int64_t)p * nw, ar);   // top nw left vectors of Z (p x nw)
  ALLOC(Vw, double, (int64_t)n * nw, ar);   // [Vj_top; 0] (n x nw), then Q2 * that
  c.sync();
  sec(27);
  bool done = false;
#if ENGINE_DEVICE
  if (c.nt == 256 && p <= 1024) {
    // Jacobi without V: Vj's top columns are recovered as Z0^T Uz S^-1
    // (error eps*|Z|/s_i, times s_i in the truncated product).
    double* Z0;
    ALLOC(Z0, double, (int64_t)p * p, ar);
    par_copy(c, Z0, Z, (int64_t)p * p);
    c.sync();
    if (p <= 32) jacobi_cols_reg<1>(c, Z, p, p, p);
    else if (p <= 64) jacobi_cols_reg<2>(c, Z, p, p, p);
    else if (p <= 128) jacobi_cols_reg<4>(c, Z, p, p, p);
    else if (p <= 256) jacobi_cols_reg<8>(c, Z, p, p, p);
    else if (p <= 512) jacobi_cols_reg<16>(c, Z, p, p, p);
    else jacobi_cols_reg<32>(c, Z, p, p, p);
    jacobi_finish(c, Z, p, p, p, s, jp, tmp);
    for (int64_t e = c.tid; e < (int64_t)p * nw; e += c.nt) {
      const int i = (int)(qmod(e, p)), j = (int)(qdiv(e, p));
      Uz[e] = Z[i + (int64_t)jp[j] * p];
    }
    c.sync();
    // Vw(0:p, j) = Z0^T Uz(:, j) / s_j
    gemm_dm<32>(c, p, nw, p, 1.0, Mat{Z0, p, 1}, Mat{Uz, 1, p}, 0.0, Vw, 1, n, sm);
    for (int64_t e = c.tid; e < (int64_t)n * nw; e += c.nt) {
      const int i = (int)(qmod(e, n)), j = (int)(qdiv(e, n));
      if (i >= p) Vw[e] = 0.0;
      else Vw[e] = s[j] > 0.0 ? Vw[e] / s[j] : 0.0;
    }
    c.sync();
    done = true;
  }
#endif
  if (!done) {
    double* Vj;
    ALLOC(Vj, double, (int64_t)p * p, ar);
    CK(svd_jacobi(c, Z, p, p, p, Vj, s, jp, tmp));
    for (int64_t e = c.tid; e < (int64_t)p * nw; e += c.nt) {
      const int i = (int)(qmod(e, p)), j = (int)(qdiv(e, p));
      Uz[e] = Z[i + (int64_t)jp[j] * p];
    }
    for (int64_t e = c.tid; e < (int64_t)n * nw; e += c.nt) {
      const int i = (int)(qmod(e, n)), j = (int)(qdiv(e, n));
      Vw[e] = (i < p) ? Vj[i + (int64_t)jp[j] * p] : 0.0;
    }
    c.sync();
  }
  sec(25);
  // U = Q1 [Uz; 0]   (m x nw);  Q1 = H_0 .. H_{p-1} of the pivoted QR
  for (int64_t e = c.tid; e < (int64_t)m * nw; e += c.nt) {
    const int i = (int)(qmod(e, m)), j = (int)(qdiv(e, m));
    U[e] = (i < p) ? Uz[i + (int64_t)j * p] : 0.0;
  }
  c.sync();
  CK(apply_refl_blocked(c, ar, A, m, m, p, tau, U, m, nw, sm));
  sec(26);
  // Vt[i, :] = (Q2 [Vj[:, i]; 0])^T  for i < nw
  CK(apply_q(c, ar, Bt, n, n, p, Tq, false, Vw, n, nw, sm));
  for (int64_t e = c.tid; e < (int64_t)nw * n; e += c.nt) {
    const int i = (int)(qdiv(e, n)), q = (int)(qmod(e, n));
    Vt[e] = Vw[q + (int64_t)i * n];
  }
  c.sync();
  sec(27);
  if (c.prof && c.leader() && p > 64) c.prof[29] += clk() - t_rrqr;
  ar.release(mk);
  *U_out = U;
  *s_out = s;
  *Vt_out = Vt;
  *kk_out = p;
  return OK;
}

// ---------------------------------------------------------------------------
// TT rounding (tensor_train.py:327-360): right-to-left Householder QR, then
// left-to-right truncated SVD with the reference's rule and sweep direction.
// The result is written into `out` (allocated here, after the temporaries are
// released, so the caller's arena holds only the output).
// ---------------------------------------------------------------------------
HDN int tt_round(const Ctx& c, Arena& ar, const TT& in, double tol, int cap, TT& out, double* sm,
                 bool destroy_input = false) {
  const int d = in.d;
  PROF(c, 7);
  if (d == 1) return tt_clone(c, ar, in, out);
  size_t mk0 = ar.mark();
  // Right-to-left: blocked Householder QR of core_k^T (rows (i, gamma), cols
  // alpha).  The reflectors stay in place (Q is never formed); R^T is carried
  // into core k-1.  Temporaries are factored in place (no copy).
  TT w;
  if (destroy_input) w = in;
  else CK(tt_clone(c, ar, in, w));
  double* taus[MAXD];
  double* Ts[MAXD];
  int mrow[MAXD], kq[MAXD];
  for (int k = d - 1; k >= 1; --k) {
    const int rl = w.r[k], n = w.n[k], rr = w.r[k + 1];
    const int m = n * rr;
    const int kk = imin(m, rl);
    ALLOC(taus[k], double, kk, ar);
    ALLOC(Ts[k], double, (int64_t)((kk + NB - 1) / NB) * NB * NB, ar);
    {
      PROF(c, 9);
      CK(geqrf_nb(c, ar, w.c[k], m, m, rl, taus[k], Ts[k], sm));
    }
    mrow[k] = m;
    kq[k] = kk;
#if defined(ENGINE_HOSTSIM) && defined(ENGINE_TRACE)
    fprintf(stderr, "RL k=%d m=%d rl=%d kk=%d A:", k, m, rl, kk);
    for (int q = 0; q < m * rl; ++q) fprintf(stderr, " %.4f", w.c[k][q]);
    fprintf(stderr, " T: %.4f %.4f %.4f", Ts[k][0], Ts[k][NB], Ts[k][NB + 1]);
    fprintf(stderr, " tau:");
    for (int q = 0; q < kk; ++q) fprintf(stderr, " %.4f", taus[k][q]);
    fprintf(stderr, "\n");
#endif
    size_t mk = ar.mark();
    double *Rm, *nc;
    ALLOC(Rm, double, (int64_t)kk * rl, ar);   // R (kk x rl) row-major
    for (int64_t e = c.tid; e < (int64_t)kk * rl; e += c.nt) {
      const int i = (int)(qdiv(e, rl)), j = (int)(qmod(e, rl));
      Rm[e] = (i <= j) ? w.c[k][i + (int64_t)j * m] : 0.0;
    }
    const int rpp = w.r[k - 1], np_ = w.n[k - 1];
    // core k-1 <- core k-1 x_3 R^T : (rpp*n', rl) @ R^T (rl x kk), in place
    // by row blocks (output row x lands at x*kk <= x*rl, so a block only
    // overwrites rows already consumed).  R is upper triangular: ktri.
    const int64_t rows = (int64_t)rpp * np_;
    const int rb = (int)lmin(rows, lmax(64, ((int64_t)1 << 20) / imax(kk, 1) / 64 * 64));
    ALLOC(nc, double, (int64_t)rb * kk, ar);
    c.sync();
    PROF(c, 18);
    for (int64_t x0 = 0; x0 < rows; x0 += rb) {
      const int nr = (int)lmin(rb, rows - x0);
      gemm_dm<64>(c, nr, kk, rl, 1.0, Mat{w.c[k - 1] + x0 * rl, rl, 1}, Mat{Rm, 1, rl}, 0.0, nc, kk, 1, sm, true);
      par_copy(c, w.c[k - 1] + x0 * kk, nc, (int64_t)nr * kk);
      c.sync();
    }
    w.r[k] = kk;
    ar.release(mk);
  }
  // Frobenius norm of core 0
  double part = 0.0;
  for (int64_t e = c.tid; e < w.size(0); e += c.nt) part = fma(w.c[0][e], w.c[0][e], part);
  const double nrm = sqrt(block_sum(c, part));
  if (nrm == 0.0) {
    ar.release(mk0);
    int n1[MAXD], r1[MAXD + 1];
    for (int k = 0; k < d; ++k) n1[k] = in.n[k];
    for (int k = 0; k <= d; ++k) r1[k] = 1;
    CK(tt_alloc(ar, out, d, n1, r1));
    for (int k = 0; k < d; ++k) par_fill(c, out.c[k], out.n[k], 0.0);
    c.sync();
    return OK;
  }
  const double delta = tol * nrm / sqrt((double)(d - 1));
  // Left-to-right: X_k = carry Q_k^T, computed as (Q_k [carry^T; 0])^T, then
  // truncated SVD.  New cores are appended in the arena (compacted at the end).
  TT res;
  res.d = d;
  for (int k = 0; k < d; ++k) res.n[k] = w.n[k];
  res.r[0] = 1;
  res.r[d] = 1;
  double* carry = nullptr;
  int rprev = 1;
  for (int k = 0; k < d; ++k) {
    const int n = w.n[k], rr = w.r[k + 1];
    const int mx = rprev * n;          // rows of X_k
    size_t mk = ar.mark();
    double* X;                         // row-major (rprev*n) x rr
    if (k == 0) {
      X = w.c[0];
    } else {
      const int m = mrow[k], kk = kq[k];
      double* Y;                       // col-major m x rprev
      ALLOC(Y, double, (int64_t)m * rprev, ar);
      for (int64_t e = c.tid; e < (int64_t)m * rprev; e += c.nt) {
        const int64_t r = qmod(e, m);
        const int a = (int)(qdiv(e, m));
        Y[e] = (r < kk) ? carry[(int64_t)a * kk + r] : 0.0;
      }
      c.sync();
#if defined(ENGINE_HOSTSIM) && defined(ENGINE_TRACE)
      fprintf(stderr, "Yin:");
      for (int q = 0; q < m * rprev; ++q) fprintf(stderr, " %.4f", Y[q]);
      fprintf(stderr, "\n");
#endif
      {
        PROF(c, 19);
        CK(apply_q(c, ar, w.c[k], m, m, kk, Ts[k], false, Y, m, rprev, sm));
      }
#if defined(ENGINE_HOSTSIM) && defined(ENGINE_TRACE)
      fprintf(stderr, "LR k=%d A:", k);
      for (int q = 0; q < m * kk; ++q) fprintf(stderr, " %.4f", w.c[k][q]);
      fprintf(stderr, " T: %.4f %.4f %.4f | ", Ts[k][0], Ts[k][NB], Ts[k][NB + 1]);
      fprintf(stderr, "k=%d m=%d kk=%d rprev=%d carry:", k, m, kk, rprev);
      for (int q = 0; q < rprev * kk; ++q) fprintf(stderr, " %.4f", carry[q]);
      fprintf(stderr, "\n Y:");
      for (int q = 0; q < m * rprev; ++q) fprintf(stderr, " %.4f", Y[q]);
      fprintf(stderr, "\n");
#endif
      ALLOC(X, double, (int64_t)mx * rr, ar);
      for (int64_t e = c.tid; e < (int64_t)mx * rr; e += c.nt) {
        const int64_t row = qdiv(e, rr);
        const int g = (int)(qmod(e, rr));
        const int a = (int)(qdiv(row, n)), i = (int)(qmod(row, n));
        X[e] = Y[((int64_t)i * rr + g) + (int64_t)a * m];
      }
      c.sync();
    }
    if (k == d - 1) {
      double* core;
      ALLOC(core, double, (int64_t)mx, ar);
      par_copy(c, core, X, mx);
      c.sync();
      res.c[k] = core;
      break;
    }
    double *U, *s, *Vt;
    int kk;
    CK(svd_rrqr(c, ar, X, mx, rr, 1e-3 * delta, &U, &s, &Vt, &kk, sm, cap > 0 ? cap : 0));
    double* tail;
    ALLOC(tail, double, kk, ar);
    int rnew = 0;
    if (c.leader()) rnew = keep_rank(s, kk, delta, cap, tail);
    rnew = (int)bcast_i(c, rnew);
    // stash U[:, :rnew] and carry = s V^T[:rnew] above the temporaries, then
    // move them down to `mk`
    double *core, *cr;
    ALLOC(core, double, (int64_t)mx * rnew, ar);
    ALLOC(cr, double, (int64_t)rnew * rr, ar);
    for (int64_t e = c.tid; e < (int64_t)mx * rnew; e += c.nt) {
      const int64_t i = qdiv(e, rnew);
      const int j = (int)(qmod(e, rnew));
      core[e] = U[i + (int64_t)j * mx];
    }
    for (int64_t e = c.tid; e < (int64_t)rnew * rr; e += c.nt) cr[e] = s[e / rr] * Vt[e];
    c.sync();
    ar.release(mk);
    double *core2, *cr2;
    ALLOC(core2, double, (int64_t)mx * rnew, ar);
    ALLOC(cr2, double, (int64_t)rnew * rr, ar);
    // destinations are below the sources: chunked forward copies
    for (int pass = 0; pass < 2; ++pass) {
      double* dst = pass ? cr2 : core2;
      const double* src = pass ? cr : core;
      const int64_t sz = pass ? (int64_t)rnew * rr : (int64_t)mx * rnew;
      if (dst == src) continue;
      const int64_t chunk = (int64_t)(src - dst);
      for (int64_t s0 = 0; s0 < sz; s0 += chunk) {
        const int64_t s1 = lmin(sz, s0 + chunk);
        for (int64_t e = s0 + c.tid; e < s1; e += c.nt) dst[e] = src[e];
        c.sync();
      }
    }
    c.sync();
    res.c[k] = core2;
    res.r[k + 1] = rnew;
    carry = cr2;
    rprev = rnew;
  }
  // compact the output cores down to mk0 (each destination precedes its source)
  ar.release(mk0);
  CK(tt_alloc(ar, out, d, res.n, res.r));
  for (int k = 0; k < d; ++k) {
    const int64_t sz = out.size(k);
    if (out.c[k] == res.c[k]) continue;
    const int64_t chunk = (int64_t)(res.c[k] - out.c[k]);
    for (int64_t s0 = 0; s0 < sz; s0 += chunk) {
      const int64_t s1 = lmin(sz, s0 + chunk);
      for (int64_t e = s0 + c.tid; e < s1; e += c.nt) out.c[k][e] = res.c[k][e];
      c.sync();
    }
  }
  c.sync();
  return OK;
}

// ---------------------------------------------------------------------------
// FFT convolution in TT form (tt_algorithms.py:642-666): transforms of both
// TTs' mode fibres, Kronecker product in the frequency domain, inverse
// transform (real part, using Hermitian symmetry), then tt_round.
// ---------------------------------------------------------------------------
HDN int tt_fft_conv(const Ctx& c, Arena& ar, const TT& K, const TT& W, double tol, int cap,
                           TT& out, double* sm) {
  const int d = K.d;
  PROF(c, 14);
  size_t mk0 = ar.mark();
  TT P;
  {
    int n[MAXD], r[MAXD + 1];
    for (int k = 0; k < d; ++k) n[k] = K.n[k];
    for (int k = 0; k <= d; ++k) r[k] = K.r[k] * W.r[k];
    CK(tt_alloc(ar, P, d, n, r));
  }
  for (int k = 0; k < d; ++k) {
    PROF(c, 20);
    const int n = K.n[k];
    const int nh = (n - 1) / 2;   // n odd
    size_t mk = ar.mark();
    double *cs, *sn;
    ALLOC(cs, double, n, ar);
    ALLOC(sn, double, n, ar);
    for (int q = c.tid; q < n; q += c.nt) {
      // e^{-2 pi i q / n}: forward twiddles; inverse uses the conjugate
      const double ang = 2.0 * 3.14159265358979323846 * (double)q / (double)n;
      cs[q] = cos(ang);
      sn[q] = sin(ang);
    }
    // spectra: fiber-major layout [a][b][omega] for omega in [0, nh]
    const int ka = K.r[k], kb = K.r[k + 1], wa = W.r[k], wb = W.r[k + 1];
    double *Kr, *Ki, *Wr, *Wi;
    ALLOC(Kr, double, (int64_t)ka * kb * (nh + 1), ar);
    ALLOC(Ki, double, (int64_t)ka * kb * (nh + 1), ar);
    ALLOC(Wr, double, (int64_t)wa * wb * (nh + 1), ar);
    ALLOC(Wi, double, (int64_t)wa * wb * (nh + 1), ar);
    c.sync();
    for (int64_t e = c.tid; e < (int64_t)ka * kb * (nh + 1); e += c.nt) {
      const int om = (int)(qmod(e, nh + 1));
      const int64_t f = qdiv(e, nh + 1);
      const int a = (int)(f / kb), b = (int)(f % kb);
      double re = 0.0, im = 0.0;
      for (int i = 0; i < n; ++i) {
        const double x = K.c[k][((int64_t)a * n + i) * kb + b];
        const int q = (int)(((int64_t)om * i) % n);
        re = fma(x, cs[q], re);
        im = fma(-x, sn[q], im);
      }
      Kr[e] = re;
      Ki[e] = im;
    }
    for (int64_t e = c.tid; e < (int64_t)wa * wb * (nh + 1); e += c.nt) {
      const int om = (int)(qmod(e, nh + 1));
      const int64_t f = qdiv(e, nh + 1);
      const int a = (int)(f / wb), b = (int)(f % wb);
      double re = 0.0, im = 0.0;
      for (int i = 0; i < n; ++i) {
        const double x = W.c[k][((int64_t)a * n + i) * wb + b];
        const int q = (int)(((int64_t)om * i) % n);
        re = fma(x, cs[q], re);
        im = fma(-x, sn[q], im);
      }
      Wr[e] = re;
      Wi[e] = im;
    }
    c.sync();
    // product fibre (a1 a2, j, b1 b2) = (1/n) [P0 + 2 sum_{om=1..nh} Re(P_om e^{+i 2pi om j/n})]
    // as a real GEMM per output row (a1 a2):  out (pr x n) = [Re P | Im P] (pr x 2(nh+1)) @ Tw,
    // Tw(om, j) = w_om cos(2 pi om j / n) / n,  Tw(nh+1+om, j) = -w_om sin(2 pi om j / n) / n,
    // w_0 = 1, w_om = 2.  Output row block lands at P[row, j, col] (stride pr along j).
    const int nk = 2 * (nh + 1);
    const int pr = P.r[k + 1];
    double *Tw, *Ph;
    ALLOC(Tw, double, (int64_t)nk * n, ar);
    ALLOC(Ph, double, (int64_t)pr * nk, ar);
    for (int e = c.tid; e < nk * n; e += c.nt) {
      const int p = e / n, j = e % n;
      const int om = p <= nh ? p : p - (nh + 1);
      const int qq = (int)(((int64_t)om * j) % n);
      const double w = (om == 0 ? 1.0 : 2.0) / (double)n;
      Tw[e] = p <= nh ? w * cs[qq] : -w * sn[qq];
    }
    for (int row = 0; row < ka * wa; ++row) {
      const int a1 = row / wa, a2 = row % wa;
      for (int64_t e = c.tid; e < (int64_t)pr * (nh + 1); e += c.nt) {
        const int col = (int)(qdiv(e, nh + 1)), om = (int)(qmod(e, nh + 1));
        const int b1 = col / wb, b2 = col % wb;
        const int64_t ik = ((int64_t)a1 * kb + b1) * (nh + 1) + om;
        const int64_t iw = ((int64_t)a2 * wb + b2) * (nh + 1) + om;
        const double kr = Kr[ik], ki = Ki[ik], wr = Wr[iw], wi = Wi[iw];
        Ph[(int64_t)col * nk + om] = kr * wr - ki * wi;
        Ph[(int64_t)col * nk + nh + 1 + om] = kr * wi + ki * wr;
      }
      c.sync();
      gemm_dm<32>(c, pr, n, nk, 1.0, Mat{Ph, nk, 1}, Mat{Tw, n, 1}, 0.0, P.c[k] + (int64_t)row * n * pr, 1, pr,
                  sm);
    }
    c.sync();
    ar.release(mk);
  }
  TT R;
  CK(tt_round(c, ar, P, tol, cap, R, sm, true));
  // R sits after P in the arena: move it down over P
  ar.release(mk0);
  TT o;
  CK(tt_alloc(ar, o, d, R.n, R.r));
  for (int k = 0; k < d; ++k) {
    const int64_t sz = o.size(k);
    const int64_t chunk = (int64_t)(R.c[k] - o.c[k]);
    for (int64_t s0 = 0; s0 < sz; s0 += chunk) {
      const int64_t s1 = lmin(sz, s0 + chunk);
      for (int64_t e = s0 + c.tid; e < s1; e += c.nt) o.c[k][e] = R.c[k][e];
      c.sync();
    }
  }
  out = o;
  return OK;
}

// ---------------------------------------------------------------------------
// tt_einsum_tpm (tt_algorithms.py:603-635): contract the 2d-mode transition TT
// with the d-mode weights over modes d..2d-1.  Backward fold
//   z(a, c) = sum_{n, b, e} T_{d+j}(a, n, b) W_j(c, n, e) z(b, e)
// as two GEMMs per mode pair (M = W_j z^T, then T_{d+j} M^T), then core d-1
// of the output = T_{d-1} x_3 z; cores 0..d-2 are T's.  Output in `out`.
// ---------------------------------------------------------------------------
HDN int tt_einsum_tpm(const Ctx& c, Arena& ar, const TT& T, const TT& W, TT& out, double* sm) {
  const int d = W.d;
  if (T.d != 2 * d) return E_ARG;
  for (int k = 0; k < d; ++k)
    if (T.n[d + k] != W.n[k]) return E_ARG;
  int maxz = 1;
  for (int k = 0; k <= T.d; ++k) maxz = imax(maxz, T.r[k]);
  int maxw = 1;
  for (int k = 0; k <= d; ++k) maxw = imax(maxw, W.r[k]);
  int n[MAXD], r[MAXD + 1];
  for (int k = 0; k < d; ++k) n[k] = T.n[k];
  for (int k = 0; k < d; ++k) r[k] = T.r[k];
  r[d] = W.r[0];   // = 1
  CK(tt_alloc(ar, out, d, n, r));
  const size_t mk = ar.mark();
  double *z, *z2, *M;
  int maxn = 1;
  for (int k = 0; k < T.d; ++k) maxn = imax(maxn, T.n[k]);
  ALLOC(z, double, (int64_t)maxz * maxw, ar);
  ALLOC(z2, double, (int64_t)maxz * maxw, ar);
  ALLOC(M, double, (int64_t)maxw * maxn * maxz, ar);
  if (c.leader()) z[0] = 1.0;
  c.sync();
  int zb = 1, ze = 1;   // z is (zb x ze) row-major: rows = T right rank, cols = W right rank
  for (int j = d - 1; j >= 0; --j) {
    const double* Tc = T.c[d + j];
    const double* Wc = W.c[j];
    const int ta = T.r[d + j], tb = T.r[d + j + 1], wc = W.r[j], wd = W.r[j + 1], nn = W.n[j];
    if (tb != zb || wd != ze) return E_ARG;
    // M[(c, n), b] = sum_e W[(c, n), e] z[b, e]            ((wc*nn) x tb)
    gemm(c, wc * nn, tb, wd, 1.0, Wc, wd, 1, z, 1, ze, 0.0, M, tb, 1, sm);
    // z2[a, c] = sum_{(n, b)} T[a, (n, b)] M[(c, n), b]     (ta x wc)
    gemm(c, ta, wc, nn * tb, 1.0, Tc, (int64_t)nn * tb, 1, M, 1, (int64_t)nn * tb, 0.0, z2, wc, 1, sm);
    double* t = z; z = z2; z2 = t;
    zb = ta;
    ze = wc;
  }
  // cores 0..d-2 copied; core d-1: (r, n, zb) x z (zb x 1)
  for (int k = 0; k + 1 < d; ++k) par_copy(c, out.c[k], T.c[k], T.size(k));
  {
    const int ra = T.r[d - 1], nn = T.n[d - 1];
    gemm(c, ra * nn, ze, zb, 1.0, T.c[d - 1], zb, 1, z, ze, 1, 0.0, out.c[d - 1], ze, 1, sm);
  }
  c.sync();
  ar.release(mk);
  return OK;
}

// ---------------------------------------------------------------------------
// Negative mass (filters.py:427-436): exact by full evaluation when the grid
// has at most `guard` points, else the mean of max(-v,0) over the fixed
// probe cells times the point count.  Returns the un-scaled sum or mean.
// ---------------------------------------------------------------------------
HDN int tt_negative_mass(const Ctx& c, Arena& ar, const TT& t, int64_t guard, const int32_t* probes,
                                int nprobes, double* result, double* sm) {
  PROF(c, 15);
  int64_t total = 1;
  bool big = false;
  for (int k = 0; k < t.d; ++k) {
    if (total > guard) big = true;
    total *= t.n[k];
    if (total > guard) big = true;
  }
  size_t mk = ar.mark();
  if (!big) {
    // dense chain: M (prod n_<k, r_k) -> M @ core_k.reshape(r_k, n_k r_{k+1})
    double* M;
    ALLOC(M, double, (int64_t)t.n[0] * t.r[1], ar);
    par_copy(c, M, t.c[0], t.size(0));
    c.sync();
    int64_t rows = t.n[0];
    for (int k = 1; k < t.d; ++k) {
      const int rl = t.r[k], n = t.n[k], rr = t.r[k + 1];
      double* M2;
      ALLOC(M2, double, rows * n * rr, ar);
      gemm(c, (int)rows, n * rr, rl, 1.0, M, rl, 1, t.c[k], (int64_t)n * rr, 1, 0.0, M2, (int64_t)n * rr, 1, sm);
      M = M2;
      rows *= n;
    }
    double part = 0.0;
    for (int64_t e = c.tid; e < rows; e += c.nt)
      if (M[e] < 0.0) part -= M[e];
    *result = block_sum(c, part);
  } else {
    double* vals;
    ALLOC(vals, double, nprobes, ar);
    IndexSlice is{&t, probes, 0};
    CK(tt_eval_bucketed(c, ar, t, nprobes, is, vals, sm));
    double part = 0.0;
    for (int e = c.tid; e < nprobes; e += c.nt) part += fmax(-vals[e], 0.0);
    *result = block_sum(c, part) / (double)nprobes * (double)total;
  }
  ar.release(mk);
  return OK;
}

}  // namespace tg
