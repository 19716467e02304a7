// Dense point-mass filter with FFT time update on the device: the pieces of
// ttpmf.filters.dense_fft_pmf_step (filters.py:888-934) as C-ABI kernels
// over a C-order dense grid (d <= 8) resident in HBM.
//
//   ttgbf_dense_prior        initial_pmd_dense values       filters.py:487-494
//   ttgbf_dense_likelihood   w *= p(z|x) (dense branch)     filters.py:564-566
//   ttgbf_dense_reduce       sums for _finalize_dense and moments_from_pmd
//                                                           filters.py:439-451, 323-333
//   ttgbf_dense_finalize     max(w, 0) / mass               filters.py:446-451
//   ttgbf_dense_interp       RegularGridInterpolator(linear, fill 0) at
//                            grid_pred @ F^-T, into a complex FFT buffer
//                                                           filters.py:911-916
//   ttgbf_dense_kernel       N(disp; 0, Q) cell_volume/|det F| (ifftshift
//                            layout), into a complex FFT buffer filters.py:920-927
//   ttgbf_dense_dft          one axis of fftn / ifftn (direct DFT of the
//                            line, twiddles from a host table) filters.py:732-736
//   ttgbf_dense_cmul / ttgbf_dense_real   spectrum product, real part
//
// Every kernel is a grid-stride pass over the grid: HBM-bound except the
// DFT (8 n flops per element and axis).  Reductions are deterministic: a
// fixed block decomposition, fixed-order block trees, then one block sums
// the block partials in order.
#include <cuda_runtime.h>

#include "common.cuh"
#include "measure.cuh"
#include "../../include/ttgbf.h"

namespace tg {
namespace dn {

constexpr int DMAXD = 8;
constexpr int THREADS = 256;
constexpr int RED_BLOCKS = 148 * 8;   // fixed decomposition of the reductions
constexpr int MAXQ = 1 + DMAXD + DMAXD * (DMAXD + 1) / 2;

struct Geo {
  int d;
  int64_t total;
  int n[DMAXD];
  ttgbf_axis ax[DMAXD];
};

// axis coordinate exactly as numpy builds it (separate multiply and add)
__device__ __forceinline__ double axv(const ttgbf_axis& a, int i) {
  return __dadd_rn(a.base, __dmul_rn(a.step, (double)(i - a.off)));
}

__device__ __forceinline__ void unflat(const Geo& g, int64_t e, int* idx) {
  for (int k = g.d - 1; k >= 0; --k) {
    idx[k] = (int)(e % g.n[k]);
    e /= g.n[k];
  }
}

struct MSpec {   // adapter for eval_h (measure.cuh)
  int d, hkind, b;
  const double* H;
};

__global__ void __launch_bounds__(THREADS) k_prior(Geo g, const ttgbf_gauss* p, double* w) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < g.total; e += (int64_t)gridDim.x * blockDim.x) {
    int idx[DMAXD];
    unflat(g, e, idx);
    double x[MAXD];
    for (int k = 0; k < g.d; ++k) x[k] = axv(g.ax[k], idx[k]) - p->mean[k];
    w[e] = exp(p->logn - 0.5 * tri_quad(SolveLU{p->LU, p->piv, p->inv, MAXD}, g.d, x));
  }
}

__global__ void __launch_bounds__(THREADS) k_likelihood(Geo g, const ttgbf_model* m, const double* z, double* w) {
  const MSpec s{m->d, m->hkind, m->b, m->H};
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < g.total; e += (int64_t)gridDim.x * blockDim.x) {
    int idx[DMAXD];
    unflat(g, e, idx);
    double x[MAXD], hz[MAXB];
    for (int k = 0; k < g.d; ++k) x[k] = axv(g.ax[k], idx[k]);
    eval_h(s, x, hz);
    for (int i = 0; i < s.b; ++i) hz[i] = hz[i] - z[i];
    for (int t = 0; t < m->nang; ++t) {
      const int a = m->ang[t];
      hz[a] = 180.0 - np_mod360(180.0 - hz[a]);
    }
    w[e] = w[e] * exp(m->logn_r - 0.5 * tri_quad(SolveLU{m->LUr, m->pivr, m->invr, MAXB}, s.b, hz));
  }
}

// mode 0: {sum max(w, 0), sum min(w, 0)}             (clipped mass, negative mass)
// mode 1: {sum w cv, sum x_k (w cv)}                       (mass, first moments)
// mode 2: {sum c_i c_j (w cv), i <= j},  c = x - mean      (centred second moments)
__device__ __forceinline__ int nq_of(int mode, int d) {
  return mode == 0 ? 2 : (mode == 1 ? 1 + d : d * (d + 1) / 2);
}

__global__ void __launch_bounds__(THREADS) k_reduce(Geo g, const double* w, int mode, double cv, const double* mean,
                                                    double* partials) {
  __shared__ double red[THREADS / 32][MAXQ];
  const int d = g.d, nq = nq_of(mode, d);
  double acc[MAXQ];
  for (int q = 0; q < nq; ++q) acc[q] = 0.0;
  const int64_t lo = g.total * blockIdx.x / gridDim.x, hi = g.total * (blockIdx.x + 1) / gridDim.x;
  for (int64_t e = lo + threadIdx.x; e < hi; e += blockDim.x) {
    const double v = w[e];
    if (mode == 0) {
      if (v < 0.0) acc[1] += v;
      else acc[0] += v;
      continue;
    }
    int idx[DMAXD];
    unflat(g, e, idx);
    const double wv = v * cv;
    if (mode == 1) {
      acc[0] += wv;
      for (int k = 0; k < d; ++k) acc[1 + k] = fma(axv(g.ax[k], idx[k]), wv, acc[1 + k]);
    } else {
      double c[DMAXD];
      for (int k = 0; k < d; ++k) c[k] = axv(g.ax[k], idx[k]) - mean[k];
      int q = 0;
      for (int i = 0; i < d; ++i)
        for (int j = i; j < d; ++j, ++q) acc[q] = fma(c[i], c[j] * wv, acc[q]);
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int q = 0; q < nq; ++q) {
    double x = acc[q];
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if (lane == 0) red[warp][q] = x;
  }
  __syncthreads();
  if (threadIdx.x < nq) {
    double s = 0.0;
    for (int i = 0; i < THREADS / 32; ++i) s += red[i][threadIdx.x];
    partials[(int64_t)blockIdx.x * MAXQ + threadIdx.x] = s;
  }
}

__global__ void k_reduce_final(const double* partials, int nblocks, int nq, double* out) {
  if (threadIdx.x < nq) {
    double s = 0.0;
    for (int b = 0; b < nblocks; ++b) s += partials[(int64_t)b * MAXQ + threadIdx.x];
    out[threadIdx.x] = s;
  }
}

__global__ void __launch_bounds__(THREADS) k_finalize(double* w, int64_t n, double mass) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    w[e] = fmax(w[e], 0.0) / mass;
}

// scipy find_indices: largest i <= n-2 with axis[i] <= x (0 below the grid)
__device__ __forceinline__ int find_cell(const ttgbf_axis& a, double x) {
  int lo = 0, hi = a.n - 2;
  if (!(axv(a, 0) <= x)) return 0;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (axv(a, mid) <= x) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(THREADS) k_interp(Geo go, Geo gn, const double* Finv, const double* w,
                                                    double2* out) {
  const int d = gn.d;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < gn.total; e += (int64_t)gridDim.x * blockDim.x) {
    int idx[DMAXD];
    unflat(gn, e, idx);
    double y[DMAXD], x[DMAXD];
    for (int k = 0; k < d; ++k) y[k] = axv(gn.ax[k], idx[k]);
    for (int j = 0; j < d; ++j) {   // (points @ F^-T)[j] = sum_k y_k Finv[j, k]
      double s = 0.0;
      for (int k = 0; k < d; ++k) s = fma(y[k], Finv[j * MAXD + k], s);
      x[j] = s;
    }
    bool oob = false;
    int cell[DMAXD];
    double dist[DMAXD];
    for (int k = 0; k < d; ++k) {
      const ttgbf_axis& a = go.ax[k];
      oob = oob || x[k] < axv(a, 0) || x[k] > axv(a, a.n - 1);
      const int i = find_cell(a, x[k]);
      const double g0 = axv(a, i), g1 = axv(a, i + 1);
      cell[k] = i;
      dist[k] = (x[k] - g0) / (g1 - g0);
    }
    double v = 0.0;
    if (!oob) {
      for (int cn = 0; cn < (1 << d); ++cn) {   // itertools.product order: dim 0 slowest
        double wt = 1.0;
        int64_t off = 0;
        for (int k = 0; k < d; ++k) {
          const int bit = (cn >> (d - 1 - k)) & 1;
          wt = wt * (bit ? dist[k] : 1.0 - dist[k]);
          off = off * go.n[k] + cell[k] + bit;
        }
        v = v + w[off] * wt;
      }
    }
    out[e] = make_double2(v, 0.0);
  }
}

__global__ void __launch_bounds__(THREADS) k_kernel(Geo g, const ttgbf_model* m, const double* steps, double cv,
                                                    double absdet, double2* out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < g.total; e += (int64_t)gridDim.x * blockDim.x) {
    int idx[DMAXD];
    unflat(g, e, idx);
    double disp[MAXD];
    for (int k = 0; k < g.d; ++k) {
      const int half = (g.n[k] - 1) / 2;
      const int sg = idx[k] <= half ? idx[k] : idx[k] - g.n[k];
      disp[k] = (double)sg * steps[k];
    }
    const double pdf = exp(m->logn_q - 0.5 * tri_quad(SolveLU{m->LUq, m->pivq, m->invq, MAXD}, g.d, disp));
    out[e] = make_double2(pdf * cv / absdet, 0.0);
  }
}

// One axis of an n-point DFT over `lines` = outer*inner lines (element j of
// line (o, i) at (o*n + j)*inner + i).  A CTA stages LT lines in SMEM.  For
// n = n1*n2 (n1 the smallest prime factor) the transform is two-stage
// Cooley-Tukey in SMEM -- length-n1 DFTs, twiddles W_n^(j2 k1), length-n2
// DFTs -- so an element costs n1 + n2 + 1 complex MACs instead of n; a
// prime n is a direct DFT.  Every twiddle is root[(.) mod n] from the host's
// exp(-2 pi i q / n) table, conjugated and scaled by 1/n for ifft.
constexpr int LT = 16;
__device__ __forceinline__ void cmac(double& re, double& im, const double2 a, const double2 r) {
  re = fma(a.x, r.x, fma(-a.y, r.y, re));
  im = fma(a.x, r.y, fma(a.y, r.x, im));
}

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(THREADS) k_dft(double2* x, int64_t outer, int n, int n1, int64_t inner, int inverse,
                                                 const double2* roots, int use_mma) {
  extern __shared__ double2 sh[];
  double2* xs = sh;               // [n][LT]
  double2* ys = sh + n * LT;      // [n][LT]  stage-1 output
  double2* rt = ys + n * LT;      // [n]
  const int n2 = n / n1;
  // DMMA final stage: the length-n2 DFT matrix W(k2, j2) = root[(j2 k2 n1) mod n]
  // as real and imaginary planes, zero-padded to MP x KP (8 | MP, 4 | KP)
  const int MP = (n2 + 7) & ~7, KP = (n2 + 3) & ~3;
  double* wr = reinterpret_cast<double*>(rt + n);
  double* wi = wr + MP * KP;
  for (int q = threadIdx.x; q < n; q += blockDim.x) {
    const double2 r = roots[q];
    rt[q] = inverse ? make_double2(r.x, -r.y) : r;
  }
  if (use_mma) {
    __syncthreads();
    for (int e = threadIdx.x; e < MP * KP; e += blockDim.x) {
      const int k2 = e / KP, j2 = e % KP;
      double2 w = make_double2(0.0, 0.0);
      if (k2 < n2 && j2 < n2) w = rt[(int)(((int64_t)j2 * k2 * n1) % n)];
      wr[e] = w.x;
      wi[e] = w.y;
    }
  }
  const int64_t lines = outer * inner;
  const double scale = inverse ? 1.0 / (double)n : 1.0;
  for (int64_t l0 = (int64_t)blockIdx.x * LT; l0 < lines; l0 += (int64_t)gridDim.x * LT) {
    __syncthreads();
    for (int e = threadIdx.x; e < n * LT; e += blockDim.x) {
      const int j = e / LT, l = e % LT;
      const int64_t L = l0 + l;
      if (L < lines) {
        const int64_t o = L / inner, i = L % inner;
        xs[e] = x[(o * n + j) * inner + i];
      } else {
        xs[e] = make_double2(0.0, 0.0);
      }
    }
    __syncthreads();
    const double2* src = xs;
    int m = n, stride = 1;          // final stage: length m DFT over src rows j*stride (+ k1)
    if (n1 > 1) {
      // stage 1: Y[j2*n1 + k1] = W_n^(j2 k1) * sum_j1 W_n1^(j1 k1) x[j2 + n2 j1]
      for (int e = threadIdx.x; e < n * LT; e += blockDim.x) {
        const int r = e / LT, l = e % LT;
        const int j2 = r / n1, k1 = r % n1;
        double re = 0.0, im = 0.0;
        int q = 0;
        const int dq = (k1 * n2) % n;
        for (int j1 = 0; j1 < n1; ++j1) {
          cmac(re, im, xs[(j2 + n2 * j1) * LT + l], rt[q]);
          q += dq;
          if (q >= n) q -= n;
        }
        const double2 t = rt[(j2 * k1) % n];
        ys[e] = make_double2(re * t.x - im * t.y, re * t.y + im * t.x);
      }
      __syncthreads();
      src = ys;
      m = n2;
      stride = n1;
    }
    if (use_mma) {
      // final stage on FP64 tensor cores: per k1, OUT (MP x LT) = W (MP x KP) SRC_k1 (KP x LT),
      // complex as four real DMMA products.  Warp task = (k1, 8-row tile, 8-line tile).
      const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, ar = lane >> 2, ac = lane & 3;
      const int tm_n = MP / 8, tasks = stride * tm_n * (LT / 8);
      for (int t = warp; t < tasks; t += blockDim.x >> 5) {
        const int tn = t % (LT / 8), tm = (t / (LT / 8)) % tm_n, k1 = t / (LT / 8 * tm_n);
        double cr0 = 0.0, cr1 = 0.0, ci0 = 0.0, ci1 = 0.0;
        const int row = tm * 8 + ar, col = tn * 8 + ar;
        for (int k0 = 0; k0 < KP; k0 += 4) {
          const int j2 = k0 + ac;
          const double a_r = wr[row * KP + j2], a_i = wi[row * KP + j2];
          const double2 b = j2 < m ? src[(j2 * stride + k1) * LT + col] : make_double2(0.0, 0.0);
          dmma884(cr0, cr1, a_r, b.x);
          dmma884(cr0, cr1, -a_i, b.y);
          dmma884(ci0, ci1, a_r, b.y);
          dmma884(ci0, ci1, a_i, b.x);
        }
        const int k2 = tm * 8 + ar;
        if (k2 < m) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int l = tn * 8 + 2 * ac + h;
            const int64_t L = l0 + l;
            if (L < lines) {
              const int64_t o = L / inner, i = L % inner;
              x[(o * n + k1 + stride * k2) * inner + i] =
                  make_double2((h ? cr1 : cr0) * scale, (h ? ci1 : ci0) * scale);
            }
          }
        }
      }
      continue;
    }
    // final stage: X[k1 + n1 k2] = sum_j2 W_n2^(j2 k2) src[j2*n1 + k1]   (n1 = 1: direct DFT).
    // A thread owns one line and KB consecutive k2 of one k1: each src value is
    // loaded once for KB complex MACs, and the KB accumulators are independent.
    constexpr int KB = 4;
    const int kq = (m + KB - 1) / KB;
    for (int e = threadIdx.x; e < stride * kq * LT; e += blockDim.x) {
      const int l = e % LT, rest = e / LT;
      const int k1 = rest % stride, k2b = (rest / stride) * KB;
      const int64_t L = l0 + l;
      if (L >= lines) continue;
      double re[KB], im[KB];
      int q[KB], dq[KB];
#pragma unroll
      for (int u = 0; u < KB; ++u) {
        re[u] = 0.0;
        im[u] = 0.0;
        q[u] = 0;
        dq[u] = ((k2b + u) * stride) % n;
      }
      for (int j2 = 0; j2 < m; ++j2) {
        const double2 a = src[(j2 * stride + k1) * LT + l];
#pragma unroll
        for (int u = 0; u < KB; ++u) {
          cmac(re[u], im[u], a, rt[q[u]]);
          q[u] += dq[u];
          if (q[u] >= n) q[u] -= n;
        }
      }
      const int64_t o = L / inner, i = L % inner;
#pragma unroll
      for (int u = 0; u < KB; ++u) {
        const int k2 = k2b + u;
        if (k2 < m) x[(o * n + k1 + stride * k2) * inner + i] = make_double2(re[u] * scale, im[u] * scale);
      }
    }
  }
}

__global__ void __launch_bounds__(THREADS) k_cmul(double2* a, const double2* b, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const double2 x = a[e], y = b[e];
    a[e] = make_double2(x.x * y.x - x.y * y.y, x.x * y.y + x.y * y.x);
  }
}

__global__ void __launch_bounds__(THREADS) k_real(const double2* a, double* w, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    w[e] = a[e].x;
}

int grid_for(int64_t n) {
  const int64_t b = (n + THREADS - 1) / THREADS;
  return (int)(b < 148 * 16 ? (b > 0 ? b : 1) : 148 * 16);
}

int make_geo(const ttgbf_axis* axes, int d, Geo* g) {
  if (d < 1 || d > DMAXD) return TTGBF_E_ARG;
  g->d = d;
  g->total = 1;
  for (int k = 0; k < d; ++k) {
    if (axes[k].n < 2) return TTGBF_E_ARG;
    g->ax[k] = axes[k];
    g->n[k] = axes[k].n;
    g->total *= axes[k].n;
  }
  return TTGBF_OK;
}

int done() { return cudaGetLastError() == cudaSuccess ? TTGBF_OK : TTGBF_E_CUDA; }

}  // namespace dn
}  // namespace tg

using namespace tg::dn;

extern "C" {

int ttgbf_dense_prior(const ttgbf_gauss* prior, const ttgbf_axis* axes, int d, double* w, void* stream) {
  Geo g;
  int st = make_geo(axes, d, &g);
  if (st) return st;
  k_prior<<<grid_for(g.total), THREADS, 0, (cudaStream_t)stream>>>(g, prior, w);
  return done();
}

int ttgbf_dense_likelihood(const ttgbf_model* model, const double* z, const ttgbf_axis* axes, int d, double* w,
                           void* stream) {
  Geo g;
  int st = make_geo(axes, d, &g);
  if (st) return st;
  k_likelihood<<<grid_for(g.total), THREADS, 0, (cudaStream_t)stream>>>(g, model, z, w);
  return done();
}

int ttgbf_dense_reduce(const double* w, const ttgbf_axis* axes, int d, int mode, double cell_volume,
                       const double* mean, double* partials, double* out, void* stream) {
  Geo g;
  int st = make_geo(axes, d, &g);
  if (st) return st;
  if (mode < 0 || mode > 2) return TTGBF_E_ARG;
  const int nq = mode == 0 ? 2 : (mode == 1 ? 1 + d : d * (d + 1) / 2);
  k_reduce<<<RED_BLOCKS, THREADS, 0, (cudaStream_t)stream>>>(g, w, mode, cell_volume, mean, partials);
  k_reduce_final<<<1, 64, 0, (cudaStream_t)stream>>>(partials, RED_BLOCKS, nq, out);
  return done();
}

int ttgbf_dense_reduce_blocks(void) { return RED_BLOCKS * MAXQ; }

int ttgbf_dense_finalize(double* w, int64_t n, double mass, void* stream) {
  k_finalize<<<grid_for(n), THREADS, 0, (cudaStream_t)stream>>>(w, n, mass);
  return done();
}

int ttgbf_dense_interp(const double* w_old, const ttgbf_axis* old_axes, const ttgbf_axis* new_axes, int d,
                       const double* Finv, double* out_complex, void* stream) {
  Geo go, gn;
  int st = make_geo(old_axes, d, &go);
  if (!st) st = make_geo(new_axes, d, &gn);
  if (st) return st;
  k_interp<<<grid_for(gn.total), THREADS, 0, (cudaStream_t)stream>>>(go, gn, Finv, w_old,
                                                                     reinterpret_cast<double2*>(out_complex));
  return done();
}

int ttgbf_dense_kernel(const ttgbf_model* model, const ttgbf_axis* axes, int d, const double* steps,
                       double cell_volume, double abs_det_f, double* out_complex, void* stream) {
  Geo g;
  int st = make_geo(axes, d, &g);
  if (st) return st;
  k_kernel<<<grid_for(g.total), THREADS, 0, (cudaStream_t)stream>>>(g, model, steps, cell_volume, abs_det_f,
                                                                     reinterpret_cast<double2*>(out_complex));
  return done();
}

int ttgbf_dense_dft(double* data_complex, const int32_t* shape, int d, int axis, int inverse,
                    const double* roots_complex, void* stream) {
  if (d < 1 || d > DMAXD || axis < 0 || axis >= d) return TTGBF_E_ARG;
  int64_t outer = 1, inner = 1;
  for (int k = 0; k < axis; ++k) outer *= shape[k];
  for (int k = axis + 1; k < d; ++k) inner *= shape[k];
  const int n = shape[axis];
  int n1 = 1;                        // smallest prime factor (two-stage transform) or 1 (prime n)
  for (int p = 2; p * p <= n; ++p)
    if (n % p == 0) { n1 = p; break; }
  const int n2 = n / n1;
  const int use_mma = (n1 > 1 && n2 <= 64) ? 1 : 0;   // tensor-core final stage for n2 <= 64
  const int MP = (n2 + 7) & ~7, KP = (n2 + 3) & ~3;
  const size_t smem = (size_t)(2 * n * LT + n) * sizeof(double2) + (use_mma ? (size_t)2 * MP * KP * sizeof(double) : 0);
  if (smem > 200 * 1024) return TTGBF_E_ARG;
  if (cudaFuncSetAttribute(k_dft, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return TTGBF_E_CUDA;
  const int64_t lines = outer * inner;
  const int64_t blocks = (lines + LT - 1) / LT;
  const int grid = (int)(blocks < 148 * 8 ? blocks : 148 * 8);
  k_dft<<<grid, THREADS, smem, (cudaStream_t)stream>>>(reinterpret_cast<double2*>(data_complex), outer, n, n1, inner,
                                                       inverse, reinterpret_cast<const double2*>(roots_complex), use_mma);
  return done();
}

int ttgbf_dense_cmul(double* a_complex, const double* b_complex, int64_t n, void* stream) {
  k_cmul<<<grid_for(n), THREADS, 0, (cudaStream_t)stream>>>(reinterpret_cast<double2*>(a_complex),
                                                            reinterpret_cast<const double2*>(b_complex), n);
  return done();
}

int ttgbf_dense_real(const double* a_complex, double* w, int64_t n, void* stream) {
  k_real<<<grid_for(n), THREADS, 0, (cudaStream_t)stream>>>(reinterpret_cast<const double2*>(a_complex), w, n);
  return done();
}

}  // extern "C"
