// Blocked dense kernels for TT rounding (CTA-cooperative, FP64 FFMA).
//
//  * gemm_t        C = alpha*A*B + beta*C with SMEM tiles whose global loads
//                  walk the unit-stride dimension (coalesced for every layout
//                  the rounding uses); TM x 64 output tiles, 4x4/2x4 per thread
//  * geqrf_nb      blocked Householder QR, nb = 32: one-pass panel columns
//                  (norm + dots with the previous reflectors in one fused
//                  reduction, T built incrementally as in dlarft), trailing
//                  update W = V^T C, W = T^T W, C -= V W as three tiled GEMMs
//  * apply_q       Q * [X; 0] (or Q^T * X) from the stored reflectors + T's,
//                  used instead of forming Q (dorgqr) in the rounding sweep
#pragma once
#include "common.cuh"
#include "linalg.cuh"
#if defined(ENGINE_HOSTSIM) && defined(ENGINE_TRACE)
#include <stdio.h>
#endif

namespace tg {

constexpr int NB = 32;

// element (i, j) of a strided operand
struct Mat {
  const double* p;
  int64_t rs, cs;   // row stride, column stride
  HD double at(int64_t i, int64_t j) const { return p[i * rs + j * cs]; }
};

// Tiled GEMM.  C(i,j) at C[i*crs + j*ccs].  SMEM: (TM + 64) * 17 doubles.
template <int TM>
HDN void gemm_t(const Ctx& c, int M, int N, int K, double alpha, Mat A, Mat B, double beta, double* C, int64_t crs,
                int64_t ccs, double* sm) {
#if ENGINE_DEVICE
  constexpr int TN = 64, TK = 16;
  constexpr int RM = TM / 16;   // rows per thread (TM = 64 -> 4, TM = 32 -> 2)
  double* As = sm;                    // [TK][TM + 1]
  double* Bs = sm + TK * (TM + 1);    // [TK][TN + 1]
  const int tx = c.tid % 16, ty = c.tid / 16;   // 16 x 16 threads
  const bool a_rowfast = A.rs == 1;             // unit stride along i?
  const bool b_colfast = B.cs == 1;             // unit stride along j?
  for (int i0 = 0; i0 < M; i0 += TM) {
    for (int j0 = 0; j0 < N; j0 += TN) {
      double acc[RM][4];
#pragma unroll
      for (int a = 0; a < RM; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
      for (int p0 = 0; p0 < K; p0 += TK) {
        __syncthreads();
        for (int e = c.tid; e < TK * TM; e += c.nt) {
          int pp, ii;
          if (a_rowfast) { ii = e % TM; pp = e / TM; } else { pp = e % TK; ii = e / TK; }
          const int gi = i0 + ii, gp = p0 + pp;
          As[pp * (TM + 1) + ii] = (gi < M && gp < K) ? A.at(gi, gp) : 0.0;
        }
        for (int e = c.tid; e < TK * TN; e += c.nt) {
          int pp, jj;
          if (b_colfast) { jj = e % TN; pp = e / TN; } else { pp = e % TK; jj = e / TK; }
          const int gj = j0 + jj, gp = p0 + pp;
          Bs[pp * (TN + 1) + jj] = (gj < N && gp < K) ? B.at(gp, gj) : 0.0;
        }
        __syncthreads();
#pragma unroll 4
        for (int pp = 0; pp < TK; ++pp) {
          double av[RM], bv[4];
#pragma unroll
          for (int a = 0; a < RM; ++a) av[a] = As[pp * (TM + 1) + ty + 16 * a];
#pragma unroll
          for (int b = 0; b < 4; ++b) bv[b] = Bs[pp * (TN + 1) + tx + 16 * b];
#pragma unroll
          for (int a = 0; a < RM; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
        }
      }
#pragma unroll
      for (int a = 0; a < RM; ++a) {
        const int gi = i0 + ty + 16 * a;
        if (gi >= M) continue;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int gj = j0 + tx + 16 * b;
          if (gj >= N) continue;
          double* cp = C + gi * crs + gj * ccs;
          *cp = (beta == 0.0) ? alpha * acc[a][b] : fma(alpha, acc[a][b], beta * (*cp));
        }
      }
    }
  }
  __syncthreads();
#else
  (void)c; (void)sm;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      double acc = 0.0;
      for (int p = 0; p < K; ++p) acc = fma(A.at(i, p), B.at(p, j), acc);
      double* cp = C + i * crs + j * ccs;
      *cp = (beta == 0.0) ? alpha * acc : fma(alpha, acc, beta * (*cp));
    }
#endif
}

// CTA reduction of a small vector (nv <= 33): every thread passes its
// partials in v[]; the totals are written to out[] (shared) and returned
// after a barrier.  Deterministic order.
HD void block_reduce_vec(const Ctx& c, double* v, int nv, double* out) {
#if ENGINE_DEVICE
  const int w = c.tid >> 5, l = c.tid & 31, nw = c.nt >> 5;
  double* part = c.red + 64;   // nw x 33 (scan buffer region)
  for (int q = 0; q < nv; ++q) {
    double x = v[q];
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (l == 0) part[w * 33 + q] = x;
  }
  __syncthreads();
  if (c.tid < nv) {
    double s = 0.0;
    for (int i = 0; i < nw; ++i) s += part[i * 33 + c.tid];
    out[c.tid] = s;
  }
  __syncthreads();
#else
  (void)c;
  for (int q = 0; q < nv; ++q) out[q] = v[q];
#endif
}

// Panel factorisation of A[j0:m, j0:j0+jb) plus its T factor (ld NB).
HDN void qr_panel_nb(const Ctx& c, double* A, int64_t lda, int m, int j0, int jb, double* tau, double* T,
                     double* sm) {
  double* red = sm;   // >= 2*NB
  for (int jj = 0; jj < jb; ++jj) {
    const int j = j0 + jj;
    double* col = A + (int64_t)j * lda;
    // pass 1: ||x||^2 and dots of x with the previous reflectors (rows > j)
    double v[NB + 1];
#pragma unroll
    for (int q = 0; q <= NB; ++q) v[q] = 0.0;
    for (int64_t r = j + 1 + c.tid; r < m; r += c.nt) {
      const double x = col[r];
      v[0] = fma(x, x, v[0]);
#pragma unroll
      for (int q = 0; q < NB; ++q)
        if (q < jj) v[1 + q] = fma(A[(int64_t)(j0 + q) * lda + r], x, v[1 + q]);
    }
    block_reduce_vec(c, v, jj + 1, red);
    const double alpha = col[j];
    double t, beta, scal;
    larfg(alpha, sqrt(red[0]), &t, &beta, &scal);
    if (c.leader()) {
      // T(0:jj, jj) = -tau_j T(0:jj, 0:jj) g,  g_q = V(:,q)^T v_j = A[j, q] + scal * dot_q
      double g[NB];
      for (int q = 0; q < jj; ++q) g[q] = A[(int64_t)(j0 + q) * lda + j] + scal * red[1 + q];
      for (int p = 0; p < jj; ++p) {
        double s = 0.0;
        for (int q = p; q < jj; ++q) s += T[p + q * NB] * g[q];
        T[p + jj * NB] = -t * s;
      }
      T[jj + jj * NB] = t;
      for (int p = jj + 1; p < NB; ++p) T[p + jj * NB] = 0.0;   // T is upper triangular
      tau[j] = t;
    }
    // pass 2: scale the reflector, then apply H_j to the rest of the panel
    for (int64_t r = j + 1 + c.tid; r < m; r += c.nt) col[r] *= scal;
    c.sync();
    if (c.leader()) col[j] = beta;
    const int nrem = jb - jj - 1;
    if (nrem > 0 && t != 0.0) {
      double w[NB];
#pragma unroll
      for (int q = 0; q < NB; ++q) w[q] = 0.0;
      for (int64_t r = j + 1 + c.tid; r < m; r += c.nt) {
        const double vr = col[r];
#pragma unroll
        for (int q = 0; q < NB; ++q)
          if (q < nrem) w[q] = fma(vr, A[(int64_t)(j + 1 + q) * lda + r], w[q]);
      }
      block_reduce_vec(c, w, nrem, red + NB);
      // include the unit diagonal row j of v_j, scale by tau
      if (c.leader())
        for (int q = 0; q < nrem; ++q) red[NB + q] = t * (red[NB + q] + A[(int64_t)(j + 1 + q) * lda + j]);
      c.sync();
      for (int64_t r = j + c.tid; r < m; r += c.nt) {
        const double vr = (r == j) ? 1.0 : col[r];
#pragma unroll
        for (int q = 0; q < NB; ++q)
          if (q < nrem) A[(int64_t)(j + 1 + q) * lda + r] -= red[NB + q] * vr;
      }
    }
    c.sync();
  }
}

// Dense copy of the panel's reflectors V (rows j0..m-1, unit diagonal,
// zeros above) into Vc (col-major, ld = m - j0).
HD void copy_v(const Ctx& c, const double* A, int64_t lda, int m, int j0, int jb, double* Vc) {
  const int64_t mr = m - j0;
  for (int64_t e = c.tid; e < mr * jb; e += c.nt) {
    const int64_t r = e % mr;
    const int q = (int)(e / mr);
    double v;
    if (r < q) v = 0.0;
    else if (r == q) v = 1.0;
    else v = A[(int64_t)(j0 + q) * lda + j0 + r];
    Vc[e] = v;
  }
  c.sync();
}

// C[j0:m, 0:nc) <- H^op C with H = I - V T V^T (trans: H^T = I - V T^T V^T)
HDN int apply_block(const Ctx& c, Arena& ar, const double* Vc, int m, int j0, int jb, const double* T, bool trans,
                    double* Cm, int64_t ldc, int nc, double* sm) {
  const int64_t mr = m - j0;
  size_t mk = ar.mark();
  double *W, *W2;
  ALLOC(W, double, (int64_t)jb * nc, ar);
  ALLOC(W2, double, (int64_t)jb * nc, ar);
  // W = V^T C   (jb x nc): A(i,p) = Vc[p + i*mr], B(p,j) = C[j0+p + j*ldc]
  gemm_t<32>(c, jb, nc, (int)mr, 1.0, Mat{Vc, mr, 1}, Mat{Cm + j0, 1, ldc}, 0.0, W, nc, 1, sm);
  // W2 = T^op W: T(p,q) at T[p + q*NB]; T^T(p,q) = T[q + p*NB]
  if (trans) gemm_t<32>(c, jb, nc, jb, 1.0, Mat{T, NB, 1}, Mat{W, nc, 1}, 0.0, W2, nc, 1, sm);
  else gemm_t<32>(c, jb, nc, jb, 1.0, Mat{T, 1, NB}, Mat{W, nc, 1}, 0.0, W2, nc, 1, sm);
#if defined(ENGINE_HOSTSIM) && defined(ENGINE_TRACE)
  fprintf(stderr, "apply_block m=%d j0=%d jb=%d nc=%d ldc=%lld trans=%d W:", m, j0, jb, nc, (long long)ldc, (int)trans);
  for (int q = 0; q < jb * nc; ++q) fprintf(stderr, " %.4f", W[q]);
  fprintf(stderr, " W2:");
  for (int q = 0; q < jb * nc; ++q) fprintf(stderr, " %.4f", W2[q]);
  fprintf(stderr, " V:");
  for (int q = 0; q < (m - j0) * jb; ++q) fprintf(stderr, " %.4f", Vc[q]);
  fprintf(stderr, "\n");
#endif
  // C -= V W2
  gemm_t<64>(c, (int)mr, nc, jb, -1.0, Mat{Vc, 1, mr}, Mat{W2, nc, 1}, 1.0, Cm + j0, 1, ldc, sm);
  ar.release(mk);
  return OK;
}

// Blocked QR of A (m x n, col-major lda).  Ts: ceil(min(m,n)/NB) * NB*NB.
HDN int geqrf_nb(const Ctx& c, Arena& ar, double* A, int64_t lda, int m, int n, double* tau, double* Ts,
                 double* sm) {
  const int k = imin(m, n);
  for (int j0 = 0; j0 < k; j0 += NB) {
    const int jb = imin(NB, k - j0);
    double* T = Ts + (int64_t)(j0 / NB) * NB * NB;
    qr_panel_nb(c, A, lda, m, j0, jb, tau, T, sm);
    if (j0 + jb < n) {
      size_t mk = ar.mark();
      double* Vc;
      ALLOC(Vc, double, (int64_t)(m - j0) * jb, ar);
      copy_v(c, A, lda, m, j0, jb, Vc);
      CK(apply_block(c, ar, Vc, m, j0, jb, T, true, A + (int64_t)(j0 + jb) * lda, lda, n - (j0 + jb), sm));
      ar.release(mk);
    }
  }
  return OK;
}

// X (m x nc, col-major ldx) <- Q X  (trans=false)  or  Q^T X  (trans=true)
// with Q = H_0 ... H_{k-1} stored in A / Ts by geqrf_nb.
HDN int apply_q(const Ctx& c, Arena& ar, const double* A, int64_t lda, int m, int k, const double* Ts, bool trans,
                double* X, int64_t ldx, int nc, double* sm) {
  const int nblk = (k + NB - 1) / NB;
  for (int bi = 0; bi < nblk; ++bi) {
    const int b = trans ? bi : nblk - 1 - bi;
    const int j0 = b * NB, jb = imin(NB, k - j0);
    size_t mk = ar.mark();
    double* Vc;
    ALLOC(Vc, double, (int64_t)(m - j0) * jb, ar);
    copy_v(c, A, lda, m, j0, jb, Vc);
    CK(apply_block(c, ar, Vc, m, j0, jb, Ts + (int64_t)b * NB * NB, trans, X, ldx, nc, sm));
    ar.release(mk);
  }
  return OK;
}

}  // namespace tg
