// Dense FP64 linear algebra for the step engine (CTA-cooperative).
//
//  * gemm            C = alpha*op(A) op(B) + beta*C, arbitrary strides, SMEM tiles
//  * qr_householder  blocked Householder QR (LAPACK dgeqrf semantics: R with
//                    beta = -sign(alpha)*||x|| diagonal, unit-lower V, tau)
//  * qr_form_q       explicit thin Q (dorgqr semantics)
//  * svd_jacobi      one-sided Jacobi SVD (high relative accuracy), sorted
//  * lstsq_pivoted   QR with column pivoting + rank cut at rcond=eps, the
//                    algorithm of LAPACK dgelsy that scipy.linalg.lstsq calls in
//                    the reference cross core solve (tt_algorithms.py:305-307)
//
// Matrices are column-major with explicit leading dimension unless stated.
#pragma once
#include "common.cuh"

namespace tg {

constexpr double DEPS = 2.220446049250313e-16;
constexpr int X_MAXR_SOLVE = 160;   // max r of lstsq_operator (cross max_rank bound)

// ---------------------------------------------------------------------------
// GEMM: C[i,j] = alpha * sum_p A(i,p) B(p,j) + beta * C[i,j]
// element (i,p) of A at A[i*ars + p*acs]; B(p,j) at B[p*brs + j*bcs];
// C(i,j) at C[i*crs + j*ccs].  beta == 0 ignores C's previous contents.
// SMEM: 2 * 16 * 64 doubles (16 KB) taken from `sm`.
// ---------------------------------------------------------------------------
HDN void gemm(const Ctx& c, int M, int N, int K, double alpha,
                     const double* A, int64_t ars, int64_t acs,
                     const double* B, int64_t brs, int64_t bcs, double beta,
                     double* C, int64_t crs, int64_t ccs, double* sm) {
#if ENGINE_DEVICE
  // 64x64 output tiles, K-tiles of 16 staged in SMEM; 256 threads x (4x4).
  constexpr int TM = 64, TN = 64, TK = 16;
  double* As = sm;             // [TK][TM]
  double* Bs = sm + TK * TM;   // [TK][TN]
  const int ti = (c.tid % 16) * 4, tj = (c.tid / 16) * 4;
  for (int i0 = 0; i0 < M; i0 += TM) {
    for (int j0 = 0; j0 < N; j0 += TN) {
      double acc[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
      for (int p0 = 0; p0 < K; p0 += TK) {
        __syncthreads();
        for (int e = c.tid; e < TK * TM; e += c.nt) {
          int pp = e / TM, ii = e % TM;
          int gi = i0 + ii, gp = p0 + pp;
          As[e] = (gi < M && gp < K) ? A[gi * ars + gp * acs] : 0.0;
        }
        for (int e = c.tid; e < TK * TN; e += c.nt) {
          int pp = e / TN, jj = e % TN;
          int gj = j0 + jj, gp = p0 + pp;
          Bs[e] = (gj < N && gp < K) ? B[gp * brs + gj * bcs] : 0.0;
        }
        __syncthreads();
        if (c.tid < 256) {
#pragma unroll 4
          for (int pp = 0; pp < TK; ++pp) {
            double av[4], bv[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) av[a] = As[pp * TM + ti + a];
#pragma unroll
            for (int b = 0; b < 4; ++b) bv[b] = Bs[pp * TN + tj + b];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
              for (int b = 0; b < 4; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
          }
        }
      }
      if (c.tid < 256) {
        for (int a = 0; a < 4; ++a) {
          int gi = i0 + ti + a;
          if (gi >= M) continue;
          for (int b = 0; b < 4; ++b) {
            int gj = j0 + tj + b;
            if (gj >= N) continue;
            double* cp = C + gi * crs + gj * ccs;
            *cp = (beta == 0.0) ? alpha * acc[a][b] : fma(alpha, acc[a][b], beta * (*cp));
          }
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
      for (int p = 0; p < K; ++p) acc = fma(A[i * ars + p * acs], B[p * brs + j * bcs], acc);
      double* cp = C + i * crs + j * ccs;
      *cp = (beta == 0.0) ? alpha * acc : fma(alpha, acc, beta * (*cp));
    }
#endif
}

// ---------------------------------------------------------------------------
// Householder reflector (LAPACK dlarfg): given alpha and ||x||, returns tau
// and beta; the caller scales x by 1/(alpha - beta).
// ---------------------------------------------------------------------------
HD void larfg(double alpha, double xnorm, double* tau, double* beta, double* scal) {
  if (xnorm == 0.0) {
    *tau = 0.0;
    *beta = alpha;
    *scal = 1.0;
    return;
  }
  double b = -copysign(hypot(alpha, xnorm), alpha);
  *tau = (b - alpha) / b;
  *scal = 1.0 / (alpha - b);
  *beta = b;
}

// ---------------------------------------------------------------------------
// LAPACK-faithful pieces of the cross's core solve (dgelsy -> dgeqp3/dlaqp2,
// dlarfg, dlapy2, dnrm2).  The cross black boxes span 300 decades (kernel and
// likelihood tails), so squared norms underflow where LAPACK's do not:
// dnrm2 (OpenBLAS x86-64: an x87 extended-precision sum of squares) is
// emulated by a power-of-two-scaled double-double sum; dlarfg rescales tiny
// reflectors by 1/safmin like LAPACK; dgelsy scales A and B into
// [smlnum, bignum] first.  Serial (one thread) -- r <= 160.
// ---------------------------------------------------------------------------
constexpr double LA_SAFMIN = 2.2250738585072014e-308;   // dlamch('S')
constexpr double LA_EPS = 1.1102230246251565e-16;       // dlamch('E') = 2^-53
constexpr double LA_PREC = 2.220446049250313e-16;       // dlamch('P') = eps * base

HD double nrm2_ser(int n, const double* x, int64_t incx) {
  double amax = 0.0, s2 = 0.0;
  for (int i = 0; i < n; ++i) {
    const double v = x[i * incx];
    amax = fmax(amax, fabs(v));
    s2 = fma(v, v, s2);
  }
  if (amax == 0.0 || !isfinite(amax)) return amax;
  // no under/overflow possible: the plain sum (as before the scaled path)
  if (amax > 1e-140 && amax < 1e140) return sqrt(s2);
  int e;
  frexp(amax, &e);
  const double sc = ldexp(1.0, -e), inv = ldexp(1.0, e);   // exact power-of-two scaling
  double hi = 0.0, lo = 0.0;
  for (int i = 0; i < n; ++i) {
    const double v = x[i * incx] * sc;
    const double p = v * v, pe = fma(v, v, -p);
    const double t = hi + p;                             // two-sum
    const double bp = t - hi;
    const double err = (hi - (t - bp)) + (p - bp);
    hi = t;
    lo += err + pe;
  }
  const double sh = hi + lo, sl = lo - (sh - hi);
  double r = sqrt(sh);
  r = r + (fma(-r, r, sh) + sl) / (2.0 * r);             // one Newton step on the double-double sum
  return r * inv;
}

HD double lapy2(double x, double y) {   // LAPACK dlapy2
  const double xa = fabs(x), ya = fabs(y);
  const double w = fmax(xa, ya), z = fmin(xa, ya);
  if (z == 0.0) return w;
  const double q = z / w;
  const double q2 = q * q;     // separate roundings (reference Fortran, no FMA)
  volatile double one_q2 = 1.0 + q2;
  return w * sqrt(one_q2);
}

// LAPACK dlarfg on alpha / x(0:n) (x scaled in place): tau, beta; x <- v.
HD void larfg_lapack(int n, double* alpha, double* x, int64_t incx, double* tau) {
  if (n <= 0) { *tau = 0.0; return; }
  double xnorm = nrm2_ser(n, x, incx);
  if (xnorm == 0.0) { *tau = 0.0; return; }
  double a = *alpha;
  double beta = -copysign(lapy2(a, xnorm), a);
  const double safmin = LA_SAFMIN / LA_EPS;
  int knt = 0;
  if (fabs(beta) < safmin) {
    const double rsafmn = 1.0 / safmin;
    do {
      ++knt;
      for (int i = 0; i < n; ++i) x[i * incx] *= rsafmn;
      beta *= rsafmn;
      a *= rsafmn;
    } while (fabs(beta) < safmin && knt < 20);
    xnorm = nrm2_ser(n, x, incx);
    beta = -copysign(lapy2(a, xnorm), a);
  }
  *tau = (beta - a) / beta;
  const double sc = 1.0 / (a - beta);
  for (int i = 0; i < n; ++i) x[i * incx] *= sc;
  for (int j = 0; j < knt; ++j) beta *= safmin;
  *alpha = beta;
}

// Unblocked QR of the panel A[j0:m, j0:j0+jb) (column-major, lda); writes
// tau[j0..j0+jb).  Each column: norm via block reduction, then the reflector
// is applied to the remaining panel columns with one fused reduction pass.
HDN void qr_panel(const Ctx& c, double* A, int64_t lda, int m, int j0, int jb, double* tau) {
  for (int j = j0; j < j0 + jb && j < m; ++j) {
    double* col = A + (int64_t)j * lda;
    double part = 0.0;
    for (int64_t r = j + 1 + c.tid; r < m; r += c.nt) part = fma(col[r], col[r], part);
    double xn2 = block_sum(c, part);
    double alpha = col[j];
    double t, beta, scal;
    larfg(alpha, sqrt(xn2), &t, &beta, &scal);
    // LAPACK computes xnorm with dnrm2 (scaled); sqrt of the sum of squares
    // agrees to rounding for the magnitudes seen here.
    for (int64_t r = j + 1 + c.tid; r < m; r += c.nt) col[r] *= scal;
    c.sync();
    if (c.leader()) { col[j] = beta; tau[j] = t; }
    // apply H = I - t v v^T to the remaining panel columns j+1..j0+jb-1
    const int nrem = j0 + jb - (j + 1);
    if (nrem > 0 && t != 0.0) {
      double w[16];
      for (int q = 0; q < nrem; ++q) w[q] = 0.0;
      for (int64_t r = j + c.tid; r < m; r += c.nt) {
        double v = (r == j) ? 1.0 : col[r];
        for (int q = 0; q < nrem; ++q) w[q] = fma(v, A[(int64_t)(j + 1 + q) * lda + r], w[q]);
      }
      for (int q = 0; q < nrem; ++q) w[q] = block_sum(c, w[q]);
      for (int64_t r = j + c.tid; r < m; r += c.nt) {
        double v = (r == j) ? 1.0 : col[r];
        for (int q = 0; q < nrem; ++q) A[(int64_t)(j + 1 + q) * lda + r] -= t * w[q] * v;
      }
    }
    c.sync();
  }
}

// Build the upper-triangular block-reflector factor T (jb x jb, col-major ld jb)
// for V = A[j0:m, j0:j0+jb) (LAPACK dlarft, forward, columnwise).
HDN void qr_larft(const Ctx& c, const double* A, int64_t lda, int m, int j0, int jb,
                         const double* tau, double* T, double* sm) {
  // G = V^T V (upper), computed by per-thread partials then reduced.
  double* G = sm;  // jb*jb
  for (int e = c.tid; e < jb * jb; e += c.nt) G[e] = 0.0;
  c.sync();
  for (int p = 0; p < jb; ++p) {
    for (int q = p + 1; q < jb; ++q) {
      double part = 0.0;
      for (int64_t r = j0 + q + c.tid; r < m; r += c.nt) {
        double vp = (r == j0 + p) ? 1.0 : A[(int64_t)(j0 + p) * lda + r];
        double vq = (r == j0 + q) ? 1.0 : A[(int64_t)(j0 + q) * lda + r];
        part = fma(vp, vq, part);
      }
      double s = block_sum(c, part);
      if (c.leader()) G[p * jb + q] = s;  // G[p][q] = v_p . v_q
    }
  }
  c.sync();
  if (c.leader()) {
    for (int i = 0; i < jb; ++i) {
      for (int r = 0; r < jb; ++r) T[r + i * jb] = 0.0;
      T[i + i * jb] = tau[j0 + i];
      // T(0:i, i) = -tau_i * T(0:i,0:i) * (V(:,0:i)^T v_i)
      double tmp[16];
      for (int p = 0; p < i; ++p) tmp[p] = -tau[j0 + i] * G[p * jb + i];
      for (int p = 0; p < i; ++p) {
        double s = 0.0;
        for (int q = p; q < i; ++q) s += T[p + q * jb] * tmp[q];
        T[p + i * jb] = s;
      }
    }
  }
  c.sync();
}

// Apply the block reflector H = I - V T V^T (trans=true: H^T) from the left to
// C = A[j0:m, c0:c0+nc) (same leading dimension as V's matrix unless given).
// Mapping: a warp owns 32 consecutive columns (lane = column) and streams all
// rows; V rows are broadcast.  W = V^T C is accumulated in registers.
HDN void apply_block_reflector(const Ctx& c, const double* V, int64_t ldv, int m, int j0, int jb,
                                      const double* T, bool trans, double* Cm, int64_t ldc,
                                      int c0, int nc, double* sm) {
  const int nwarps = (c.nt + 31) / 32;
  const int warp = c.tid >> 5;
  const int lane = c.tid & 31;
  double* Ts = sm;  // jb*jb
  for (int e = c.tid; e < jb * jb; e += c.nt) Ts[e] = T[e];
  c.sync();
#if !ENGINE_DEVICE
  (void)nwarps; (void)warp; (void)lane;
  for (int cc = 0; cc < nc; ++cc) {
    double* col = Cm + (int64_t)(c0 + cc) * ldc;
    double w[16], w2[16];
    for (int p = 0; p < jb; ++p) {
      double s = 0.0;
      for (int64_t r = j0 + p; r < m; ++r) {
        double v = (r == j0 + p) ? 1.0 : V[(int64_t)(j0 + p) * ldv + r];
        s = fma(v, col[r], s);
      }
      w[p] = s;
    }
    for (int p = 0; p < jb; ++p) {
      double s = 0.0;
      if (trans) { for (int q = 0; q <= p; ++q) s += Ts[q + p * jb] * w[q]; }
      else { for (int q = p; q < jb; ++q) s += Ts[p + q * jb] * w[q]; }
      w2[p] = s;
    }
    for (int64_t r = j0; r < m; ++r) {
      double s = 0.0;
      for (int p = 0; p < jb && j0 + p <= r; ++p) {
        double v = (r == j0 + p) ? 1.0 : V[(int64_t)(j0 + p) * ldv + r];
        s = fma(v, w2[p], s);
      }
      col[r] -= s;
    }
  }
#else
  for (int cb = warp * 32; cb < nc; cb += nwarps * 32) {
    const int cc = cb + lane;
    const bool active = cc < nc;
    double* col = active ? Cm + (int64_t)(c0 + cc) * ldc : Cm;
    double w[16];
#pragma unroll
    for (int p = 0; p < 16; ++p) w[p] = 0.0;
    for (int64_t r = j0; r < m; ++r) {
      double x = active ? col[r] : 0.0;
      const int pmax = imin(jb, (int)(r - j0) + 1);
#pragma unroll
      for (int p = 0; p < 16; ++p) {
        if (p < pmax) {
          double v = (r == j0 + p) ? 1.0 : V[(int64_t)(j0 + p) * ldv + r];
          w[p] = fma(v, x, w[p]);
        }
      }
    }
    double w2[16];
#pragma unroll
    for (int p = 0; p < 16; ++p) {
      double s = 0.0;
      if (p < jb) {
        if (trans) { for (int q = 0; q <= p; ++q) s += Ts[q + p * jb] * w[q]; }
        else { for (int q = p; q < jb; ++q) s += Ts[p + q * jb] * w[q]; }
      }
      w2[p] = s;
    }
    if (active) {
      for (int64_t r = j0; r < m; ++r) {
        double s = 0.0;
        const int pmax = imin(jb, (int)(r - j0) + 1);
#pragma unroll
        for (int p = 0; p < 16; ++p) {
          if (p < pmax) {
            double v = (r == j0 + p) ? 1.0 : V[(int64_t)(j0 + p) * ldv + r];
            s = fma(v, w2[p], s);
          }
        }
        col[r] -= s;
      }
    }
  }
#endif
  c.sync();
}

constexpr int QR_NB = 16;

// In-place blocked Householder QR of A (m x n, col-major, lda).
// sm: >= 2*QR_NB*QR_NB + 64 doubles of shared scratch.  T: QR_NB^2 doubles.
HDN int qr_householder(const Ctx& c, double* A, int64_t lda, int m, int n, double* tau,
                              double* T, double* sm) {
  const int k = imin(m, n);
  for (int j0 = 0; j0 < k; j0 += QR_NB) {
    const int jb = imin(QR_NB, k - j0);
    qr_panel(c, A, lda, m, j0, jb, tau);
    if (j0 + jb < n) {
      qr_larft(c, A, lda, m, j0, jb, tau, T, sm);
      apply_block_reflector(c, A, lda, m, j0, jb, T, true, A, lda, j0 + jb, n - (j0 + jb), sm);
    }
  }
  return OK;
}

// Explicit thin Q (m x k, col-major ldq) from the reflectors stored in A.
HDN int qr_form_q(const Ctx& c, const double* A, int64_t lda, int m, int k, const double* tau,
                         double* Q, int64_t ldq, double* T, double* sm) {
  for (int64_t e = c.tid; e < (int64_t)m * k; e += c.nt) {
    int64_t j = e / m, i = e % m;
    Q[j * ldq + i] = (i == j) ? 1.0 : 0.0;
  }
  c.sync();
  const int nblk = (k + QR_NB - 1) / QR_NB;
  for (int b = nblk - 1; b >= 0; --b) {
    const int j0 = b * QR_NB;
    const int jb = imin(QR_NB, k - j0);
    qr_larft(c, A, lda, m, j0, jb, tau, T, sm);
    apply_block_reflector(c, A, lda, m, j0, jb, T, false, Q, ldq, j0, k - j0, sm);
  }
  return OK;
}

// ---------------------------------------------------------------------------
// One-sided Jacobi SVD of X (m x n, col-major ldx), m >= n assumed; X is
// overwritten by U*S (columns), V (n x n, ld n) accumulates rotations.
// On return: s[0..n) sorted descending, U columns in X normalised (zero
// columns stay zero), perm applied to both.  Needs n ints + n doubles ws.
// Parallel: round-robin tournament, one warp per column pair.
// ---------------------------------------------------------------------------
HDN int svd_jacobi(const Ctx& c, double* X, int64_t ldx, int m, int n, double* V, double* s,
                          int* perm, double* tmp) {
  for (int64_t e = c.tid; e < (int64_t)n * n; e += c.nt) V[e] = ((e / n) == (e % n)) ? 1.0 : 0.0;
  c.sync();
  if (n == 1) {
    double part = 0.0;
    for (int64_t r = c.tid; r < m; r += c.nt) part = fma(X[r], X[r], part);
    double nrm = sqrt(block_sum(c, part));
    if (c.leader()) { s[0] = nrm; perm[0] = 0; }
    if (nrm > 0.0)
      for (int64_t r = c.tid; r < m; r += c.nt) X[r] /= nrm;
    c.sync();
    return OK;
  }
  const int np = n + (n & 1);            // even number of players
  const int pairs = np / 2;
  const int nwarps = imax(1, c.nt / 32);
  const int warp = c.tid >> 5;
  const int lane = c.tid & 31;
  const double tol = DEPS * sqrt((double)m);
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0;
    for (int round = 0; round < np - 1; ++round) {
#if ENGINE_DEVICE
      for (int pr = warp; pr < pairs; pr += nwarps) {
#else
      for (int pr = 0; pr < pairs; ++pr) {
#endif
        // circle method: player 0 fixed, others rotate
        int a = (pr == 0) ? 0 : 1 + (pr - 1 + round) % (np - 1);
        int b = 1 + (np - 2 - pr + round) % (np - 1);
        if (a >= n || b >= n) continue;
        if (a > b) { int t = a; a = b; b = t; }
        double* xa = X + (int64_t)a * ldx;
        double* xb = X + (int64_t)b * ldx;
        double al = 0.0, be = 0.0, ga = 0.0;
#if ENGINE_DEVICE
        for (int64_t r = lane; r < m; r += 32) {
          double u = xa[r], v = xb[r];
          al = fma(u, u, al); be = fma(v, v, be); ga = fma(u, v, ga);
        }
        for (int o = 16; o > 0; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
#else
        for (int64_t r = 0; r < m; ++r) {
          double u = xa[r], v = xb[r];
          al = fma(u, u, al); be = fma(v, v, be); ga = fma(u, v, ga);
        }
#endif
        if (ga == 0.0 || al == 0.0 || be == 0.0) continue;
        double rel = fabs(ga) / sqrt(al * be);
        if (rel > off) off = rel;
        if (rel <= tol) continue;
        double zeta = (be - al) / (2.0 * ga);
        double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        double cs = 1.0 / sqrt(1.0 + t * t);
        double sn = cs * t;
#if ENGINE_DEVICE
        for (int64_t r = lane; r < m; r += 32) {
#else
        for (int64_t r = 0; r < m; ++r) {
#endif
          double u = xa[r], v = xb[r];
          xa[r] = cs * u - sn * v;
          xb[r] = sn * u + cs * v;
        }
        double* va = V + (int64_t)a * n;
        double* vb = V + (int64_t)b * n;
#if ENGINE_DEVICE
        for (int r = lane; r < n; r += 32) {
#else
        for (int r = 0; r < n; ++r) {
#endif
          double u = va[r], v = vb[r];
          va[r] = cs * u - sn * v;
          vb[r] = sn * u + cs * v;
        }
      }
      c.sync();
    }
    off = block_max(c, off);
    if (off <= tol) break;
  }
  // norms, normalise, sort descending (stable by index)
  for (int j = 0; j < n; ++j) {
    double part = 0.0;
    const double* xj = X + (int64_t)j * ldx;
    for (int64_t r = c.tid; r < m; r += c.nt) part = fma(xj[r], xj[r], part);
    double nr = sqrt(block_sum(c, part));
    if (c.leader()) tmp[j] = nr;
  }
  c.sync();
  if (c.leader()) {
    for (int j = 0; j < n; ++j) perm[j] = j;
    for (int i = 1; i < n; ++i) {  // insertion sort, descending, stable
      int p = perm[i];
      int q = i - 1;
      while (q >= 0 && tmp[perm[q]] < tmp[p]) { perm[q + 1] = perm[q]; --q; }
      perm[q + 1] = p;
    }
    for (int j = 0; j < n; ++j) s[j] = tmp[perm[j]];
  }
  c.sync();
  for (int j = 0; j < n; ++j) {
    double nr = tmp[j];
    if (nr > 0.0) {
      double* xj = X + (int64_t)j * ldx;
      for (int64_t r = c.tid; r < m; r += c.nt) xj[r] /= nr;
    }
  }
  c.sync();
  return OK;
}

#if ENGINE_DEVICE
// One-sided Jacobi on the columns of Z (m x n, col-major ldz), m <= 32*RL,
// without accumulating V: one warp per column pair of the round-robin
// tournament, both columns held in registers (all loads in flight at once).
// Same rotation formulas, order and stopping rule as svd_jacobi.
template <int RL>
__device__ __noinline__ void jacobi_cols_reg(const Ctx& c, double* Z, int64_t ldz, int m, int n) {
  const int np = n + (n & 1), pairs = np / 2;
  const int warp = c.tid >> 5, lane = c.tid & 31, nwarps = c.nt >> 5;
  const double tol = DEPS * sqrt((double)m);
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0;
    for (int round = 0; round < np - 1; ++round) {
      for (int pr = warp; pr < pairs; pr += nwarps) {
        int a = (pr == 0) ? 0 : 1 + (pr - 1 + round) % (np - 1);
        int b = 1 + (np - 2 - pr + round) % (np - 1);
        if (a >= n || b >= n) continue;
        if (a > b) { const int t = a; a = b; b = t; }
        double* xa = Z + (int64_t)a * ldz;
        double* xb = Z + (int64_t)b * ldz;
        double u[RL], v[RL];
#pragma unroll
        for (int q = 0; q < RL; ++q) {
          const int r = lane + 32 * q;
          u[q] = r < m ? xa[r] : 0.0;
          v[q] = r < m ? xb[r] : 0.0;
        }
        double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
        for (int q = 0; q < RL; ++q) {
          al = fma(u[q], u[q], al);
          be = fma(v[q], v[q], be);
          ga = fma(u[q], v[q], ga);
        }
        for (int o = 16; o > 0; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        if (ga == 0.0 || al == 0.0 || be == 0.0) continue;
        const double rel = fabs(ga) / sqrt(al * be);
        if (rel > off) off = rel;
        if (rel <= tol) continue;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / sqrt(1.0 + t * t);
        const double sn = cs * t;
#pragma unroll
        for (int q = 0; q < RL; ++q) {
          const int r = lane + 32 * q;
          if (r < m) {
            xa[r] = cs * u[q] - sn * v[q];
            xb[r] = sn * u[q] + cs * v[q];
          }
        }
      }
      __syncthreads();
    }
    off = block_max(c, off);
    if (off <= tol) break;
  }
}

// column norms of Z -> s (sorted descending, stable), perm, columns normalised
__device__ __noinline__ void jacobi_finish(const Ctx& c, double* Z, int64_t ldz, int m, int n, double* s, int* perm,
                                           double* tmp) {
  const int warp = c.tid >> 5, lane = c.tid & 31, nwarps = c.nt >> 5;
  for (int j = warp; j < n; j += nwarps) {
    const double* zj = Z + (int64_t)j * ldz;
    double a = 0.0;
    for (int r = lane; r < m; r += 32) a = fma(zj[r], zj[r], a);
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) tmp[j] = sqrt(a);
  }
  __syncthreads();
  for (int j = c.tid; j < n; j += c.nt) {
    const double v = tmp[j];
    int rank = 0;
    for (int i = 0; i < n; ++i) rank += (tmp[i] > v || (tmp[i] == v && i < j)) ? 1 : 0;
    perm[rank] = j;
    s[rank] = v;
  }
  __syncthreads();
  for (int j = warp; j < n; j += nwarps) {
    const double nr = tmp[j];
    if (nr > 0.0) {
      double* zj = Z + (int64_t)j * ldz;
      for (int r = lane; r < m; r += 32) zj[r] /= nr;
    }
  }
  __syncthreads();
}
#endif

// LAPACK dlaic1: one step of incremental condition estimation.
// job 1: largest singular value, job 2: smallest.  x has length j, w is the
// new column's top j entries, gamma its diagonal entry.
HD void laic1(int job, int j, const double* x, double sest, const double* w, double gamma, double* sestpr,
              double* s, double* c) {
  const double eps = 1.1102230246251565e-16;   // dlamch('Epsilon')
  double alpha = 0.0;
  for (int i = 0; i < j; ++i) alpha += x[i] * w[i];
  const double absalp = fabs(alpha), absgam = fabs(gamma), absest = fabs(sest);
  if (job == 1) {
    if (sest == 0.0) {
      const double s1 = fmax(absgam, absalp);
      if (s1 == 0.0) { *s = 0.0; *c = 1.0; *sestpr = 0.0; }
      else {
        double ss = alpha / s1, cc = gamma / s1;
        const double tmp = sqrt(ss * ss + cc * cc);
        *s = ss / tmp; *c = cc / tmp; *sestpr = s1 * tmp;
      }
      return;
    } else if (absgam <= eps * absest) {
      *s = 1.0; *c = 0.0;
      const double tmp = fmax(absest, absalp);
      const double s1 = absest / tmp, s2 = absalp / tmp;
      *sestpr = tmp * sqrt(s1 * s1 + s2 * s2);
      return;
    } else if (absalp <= eps * absest) {
      if (absgam <= absest) { *s = 1.0; *c = 0.0; *sestpr = absest; }
      else { *s = 0.0; *c = 1.0; *sestpr = absgam; }
      return;
    } else if (absest <= eps * absalp || absest <= eps * absgam) {
      const double s1 = absgam, s2 = absalp;
      if (s1 <= s2) {
        const double tmp = s1 / s2;
        const double ss = sqrt(1.0 + tmp * tmp);
        *sestpr = s2 * ss;
        *c = (gamma / s2) / ss;
        *s = copysign(1.0, alpha) / ss;
      } else {
        const double tmp = s2 / s1;
        const double cc = sqrt(1.0 + tmp * tmp);
        *sestpr = s1 * cc;
        *s = (alpha / s1) / cc;
        *c = copysign(1.0, gamma) / cc;
      }
      return;
    } else {
      const double z1 = alpha / absest, z2 = gamma / absest;
      const double b = (1.0 - z1 * z1 - z2 * z2) * 0.5;
      const double cc = z1 * z1;
      const double t = (b > 0.0) ? cc / (b + sqrt(b * b + cc)) : sqrt(b * b + cc) - b;
      const double sine = -z1 / t, cosine = -z2 / (1.0 + t);
      const double tmp = sqrt(sine * sine + cosine * cosine);
      *s = sine / tmp; *c = cosine / tmp;
      *sestpr = sqrt(t + 1.0) * absest;
      return;
    }
  }
  // job == 2
  if (sest == 0.0) {
    *sestpr = 0.0;
    double sine, cosine;
    if (fmax(absgam, absalp) == 0.0) { sine = 1.0; cosine = 0.0; }
    else { sine = -gamma; cosine = alpha; }
    const double s1 = fmax(fabs(sine), fabs(cosine));
    double ss = sine / s1, cc = cosine / s1;
    const double tmp = sqrt(ss * ss + cc * cc);
    *s = ss / tmp; *c = cc / tmp;
    return;
  } else if (absgam <= eps * absest) {
    *s = 0.0; *c = 1.0; *sestpr = absgam;
    return;
  } else if (absalp <= eps * absest) {
    if (absgam <= absest) { *s = 0.0; *c = 1.0; *sestpr = absgam; }
    else { *s = 1.0; *c = 0.0; *sestpr = absest; }
    return;
  } else if (absest <= eps * absalp || absest <= eps * absgam) {
    const double s1 = absgam, s2 = absalp;
    if (s1 <= s2) {
      const double tmp = s1 / s2;
      const double cc = sqrt(1.0 + tmp * tmp);
      *sestpr = absest * (tmp / cc);
      *s = -(gamma / s2) / cc;
      *c = copysign(1.0, alpha) / cc;
    } else {
      const double tmp = s2 / s1;
      const double ss = sqrt(1.0 + tmp * tmp);
      *sestpr = absest / ss;
      *c = (alpha / s1) / ss;
      *s = -copysign(1.0, gamma) / ss;
    }
    return;
  }
  const double z1 = alpha / absest, z2 = gamma / absest;
  const double norma = fmax(1.0 + z1 * z1 + fabs(z1 * z2), fabs(z1 * z2) + z2 * z2);
  const double test = 1.0 + 2.0 * (z1 - z2) * (z1 + z2);
  double sine, cosine;
  if (test >= 0.0) {
    const double b = (z1 * z1 + z2 * z2 + 1.0) * 0.5;
    const double cc = z2 * z2;
    const double t = cc / (b + sqrt(fabs(b * b - cc)));
    sine = z1 / (1.0 - t);
    cosine = -z2 / t;
    *sestpr = sqrt(t + 4.0 * eps * eps * norma) * absest;
  } else {
    const double b = (z2 * z2 + z1 * z1 - 1.0) * 0.5;
    const double cc = z1 * z1;
    const double t = (b >= 0.0) ? -cc / (b + sqrt(b * b + cc)) : b - sqrt(b * b + cc);
    sine = -z1 / t;
    cosine = -z2 / (1.0 + t);
    *sestpr = sqrt(1.0 + t + 4.0 * eps * eps * norma) * absest;
  }
  const double tmp = sqrt(sine * sine + cosine * cosine);
  *s = sine / tmp;
  *c = cosine / tmp;
}

// ---------------------------------------------------------------------------
// Least squares  A X = B  with A (r x r), B (r x nrhs): the dgelsy algorithm
// (QR with column pivoting, rank by incremental condition estimation with
// rcond = eps as scipy's default, min-norm solution for rank-deficient A).
// A(i,j) = A[i*lda_r + j*lda_c]; B(i,j) at B[i + j*ldb]; X(i,j) written at
// X[i + j*ldx].  The pivoted QR and the rank-deficient second QR run on
// warp 0 (lanes over columns / rows); right-hand sides are solved one per
// thread with LAPACK's per-column operation order (an explicit solution
// operator M with X = M B loses ~cond(A)*eps on these ill-conditioned
// cross matrices and breaks parity).
// Workspace: W r*r, W2 r*r, tau r, tau2 r, jpvt r (ints), colnorm r.
// ---------------------------------------------------------------------------
HDN int lstsq_pivoted(const Ctx& c, const double* A, int64_t lda_r, int64_t lda_c, int r, const double* B,
                      int64_t ldb, int nrhs, double* X, int64_t ldx, double* W, double* W2, double* tau, double* tau2,
                      int* jpvt, double* cn, int* rank_out, double* sm = nullptr, int sm_doubles = 0) {
  // Small systems (2 r^2 + 4 r + 2 doubles fit the CTA scratch) are factored
  // in shared memory: the pivot search, swaps, reflectors and condition
  // estimation below are chains of dependent loads, and every thread of the
  // solve phase reads all of R.  Same arithmetic in the same order as the
  // global-memory path.
  if (sm && 2 * (int64_t)r * r + 4 * r + 2 <= sm_doubles) {
    W = sm;
    W2 = sm + (int64_t)r * r;
    cn = W2 + (int64_t)r * r;
    tau = cn + r + 1;
    tau2 = tau + r;
    jpvt = reinterpret_cast<int*>(tau2 + r);
    c.sync();
  }
  for (int64_t e = c.tid; e < (int64_t)r * r; e += c.nt) {
    int i = (int)(e % r), j = (int)(e / r);
    W[i + (int64_t)j * r] = A[i * lda_r + j * lda_c];
  }
  for (int j = c.tid; j < r; j += c.nt) jpvt[j] = j;
  c.sync();
  const int64_t t_fact = clk();
#if ENGINE_DEVICE
  const bool w0 = c.tid < 32;
  const int lane = c.tid & 31, L = 32;
#define WSYNC() __syncwarp()
#else
  const bool w0 = true;
  const int L = 1;
#define WSYNC() (void)0
#endif
  if (w0) {
#if !ENGINE_DEVICE
    const int lane = 0;
#endif
    // dgelsy: scale A into [smlnum, bignum] (the solution is rescaled below)
    if (lane == 0) {
      double anrm = 0.0;
      for (int64_t e = 0; e < (int64_t)r * r; ++e) anrm = fmax(anrm, fabs(W[e]));
      const double smlnum = LA_SAFMIN / LA_PREC, bignum = 1.0 / smlnum;
      double ascl = 1.0;
      if (anrm > 0.0 && anrm < smlnum) ascl = smlnum / anrm;
      else if (anrm > bignum) ascl = bignum / anrm;
      if (ascl != 1.0)
        for (int64_t e = 0; e < (int64_t)r * r; ++e) W[e] *= ascl;
      cn[r] = ascl;   // (cn has r + 1 entries)
    }
    WSYNC();
    // dgeqp3 / dlaqp2: partial column norms vn1 (cn) / vn2 (tau2), downdated
    for (int q = lane; q < r; q += L) { cn[q] = nrm2_ser(r, W + (int64_t)q * r, 1); tau2[q] = cn[q]; }
    WSYNC();
    const double tol3z = sqrt(LA_EPS);
    for (int j = 0; j < r; ++j) {
      // idamax (first max) over cn[j..r): lanes scan strided, ties to the lower index
      int best = j;
#if ENGINE_DEVICE
      {
        double bv = -1.0;
        int bi = r;
        for (int q = j + lane; q < r; q += L) {
          const double v = fabs(cn[q]);
          if (v > bv) { bv = v; bi = q; }
        }
        for (int o = 16; o > 0; o >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
        }
        // (a NaN norm never compares greater: the serial scan keeps j as well)
        best = (bi < r && bv > fabs(cn[j])) ? bi : j;
      }
#else
      for (int q = j + 1; q < r; ++q)
        if (fabs(cn[q]) > fabs(cn[best])) best = q;
#endif
      if (best != j) {
        for (int i = lane; i < r; i += L) {
          const double t = W[i + (int64_t)j * r];
          W[i + (int64_t)j * r] = W[i + (int64_t)best * r];
          W[i + (int64_t)best * r] = t;
        }
        if (lane == 0) {
          const int t = jpvt[j]; jpvt[j] = jpvt[best]; jpvt[best] = t;
          cn[best] = cn[j];
          tau2[best] = tau2[j];
        }
      }
      WSYNC();
      if (lane == 0) {
        double t2 = 0.0;
        if (j < r - 1) larfg_lapack(r - j - 1, &W[j + (int64_t)j * r], W + j + 1 + (int64_t)j * r, 1, &t2);
        tau[j] = t2;
      }
      WSYNC();
      const double* col = W + (int64_t)j * r;
      const double t2 = tau[j];
      for (int q = j + 1 + lane; q < r; q += L) {
        double* cq = W + (int64_t)q * r;
        if (t2 != 0.0) {   // dlarf: H C = C - tau v (v^T C), v = [1; col(j+1:)]
          double w = cq[j];
          for (int i = j + 1; i < r; ++i) w = fma(col[i], cq[i], w);
          w *= t2;
          cq[j] -= w;
          for (int i = j + 1; i < r; ++i) cq[i] -= w * col[i];
        }
        if (cn[q] != 0.0) {   // dlaqp2's norm downdate / recomputation
          const double a = fabs(cq[j]) / cn[q];
          const double temp = fmax(1.0 - a * a, 0.0);
          const double ratio = cn[q] / tau2[q];
          if (temp * ratio * ratio <= tol3z) {
            cn[q] = j + 1 < r ? nrm2_ser(r - j - 1, cq + j + 1, 1) : 0.0;
            tau2[q] = cn[q];
          } else {
            cn[q] *= sqrt(temp);
          }
        }
      }
      WSYNC();
    }
    // rank by incremental condition estimation (dgelsy with rcond = eps)
    int rank = 0;
    if (lane == 0) {
      double* xmin = cn;            // reuse: column norms no longer needed
      double* xmax = tau2;          // (tau2 is rewritten below if rank-deficient)
      double smax = fabs(W[0]);
      double smin = smax;
      if (smax != 0.0) {
        rank = 1;
        xmin[0] = 1.0;
        xmax[0] = 1.0;
        while (rank < r) {
          const int i = rank;
          const double* col = W + (int64_t)i * r;
          double sminpr, s1, c1, smaxpr, s2, c2;
          laic1(2, rank, xmin, smin, col, col[i], &sminpr, &s1, &c1);
          laic1(1, rank, xmax, smax, col, col[i], &smaxpr, &s2, &c2);
          if (!(smaxpr * DEPS <= sminpr)) break;
          for (int q = 0; q < rank; ++q) { xmin[q] *= s1; xmax[q] *= s2; }
          xmin[rank] = c1;
          xmax[rank] = c2;
          smin = sminpr;
          smax = smaxpr;
          ++rank;
        }
      }
      c.ired[0] = rank;
    }
    WSYNC();
    rank = c.ired[0];
    // rank-deficient: QR of [R11 R12]^T (r x rank) -> min-norm solution
    if (rank > 0 && rank < r) {
      for (int64_t e = lane; e < (int64_t)r * rank; e += L) {
        const int i = (int)(e % r), j = (int)(e / r);
        W2[i + (int64_t)j * r] = (i >= j) ? W[j + (int64_t)i * r] : 0.0;
      }
      WSYNC();
      for (int j = 0; j < rank; ++j) {
        double* col = W2 + (int64_t)j * r;
        double t2 = 0.0;
        if (lane == 0) {
          if (j < r - 1) larfg_lapack(r - j - 1, &col[j], col + j + 1, 1, &t2);
          tau2[j] = t2;
        }
        WSYNC();
        t2 = tau2[j];
        for (int q = j + 1 + lane; q < rank; q += L) {
          double* cq = W2 + (int64_t)q * r;
          double w = cq[j];
          for (int i = j + 1; i < r; ++i) w = fma(col[i], cq[i], w);
          w *= t2;
          cq[j] -= w;
          for (int i = j + 1; i < r; ++i) cq[i] -= w * col[i];
        }
        WSYNC();
      }
    }
  }
#undef WSYNC
  c.sync();
  if (c.prof && c.leader()) c.prof[31] += clk() - t_fact;   // factorisation + rank (warp 0), the rest is the solve phase
  const int rank = c.ired[0];
  if (rank_out) *rank_out = rank;
  // dgelsy's scaling of B into [smlnum, bignum] (one factor for all of B)
  double bpart = 0.0;
  for (int q = c.tid; q < nrhs; q += c.nt)
    for (int i = 0; i < r; ++i) bpart = fmax(bpart, fabs(B[i + (int64_t)q * ldb]));
  const double bnrm = block_max(c, bpart);
  double bscl = 1.0;
  {
    const double smlnum = LA_SAFMIN / LA_PREC, bignum = 1.0 / smlnum;
    if (bnrm > 0.0 && bnrm < smlnum) bscl = smlnum / bnrm;
    else if (bnrm > bignum) bscl = bignum / bnrm;
  }
  const double xscl = cn[r] / bscl;   // X = (A-scale / B-scale) * solution of the scaled system
  // per right-hand side: y = Q^T b; triangular / min-norm solve; permute
  for (int q = c.tid; q < nrhs; q += c.nt) {
    // one private vector per thread, solved in place (y -> solution): half
    // the local-memory footprint of separate y / solution arrays.  (A fully
    // unrolled register-resident variant was measured slower: ~10k
    // instructions per right-hand side thrash the instruction cache.)
    double yy[X_MAXR_SOLVE];
    double* sol = yy;
    for (int i = 0; i < r; ++i) yy[i] = B[i + (int64_t)q * ldb] * bscl;
    for (int j = 0; j < r; ++j) {
      const double t2 = tau[j];
      if (t2 == 0.0) continue;
      const double* v = W + (int64_t)j * r;
      double w = yy[j];
      for (int i = j + 1; i < r; ++i) w = fma(v[i], yy[i], w);
      w *= t2;
      yy[j] -= w;
      for (int i = j + 1; i < r; ++i) yy[i] -= w * v[i];
    }
    if (rank == 0) {
      for (int i = 0; i < r; ++i) sol[i] = 0.0;
    } else if (rank == r) {
      for (int i = r - 1; i >= 0; --i) {
        double s2 = yy[i];
        for (int k = i + 1; k < r; ++k) s2 -= W[i + (int64_t)k * r] * sol[k];
        sol[i] = s2 / W[i + (int64_t)i * r];
      }
    } else {
      // [R11 R12] = L2^T Q2^T with W2 = Q2 L2 (L2 upper, rank x rank)
      // solve L2^T w = y[0:rank] (forward, in place), sol = Q2 [w; 0]
      for (int i = 0; i < rank; ++i) {
        double s2 = yy[i];
        for (int k = 0; k < i; ++k) s2 -= W2[k + (int64_t)i * r] * yy[k];
        yy[i] = s2 / W2[i + (int64_t)i * r];
      }
      for (int i = rank; i < r; ++i) sol[i] = 0.0;
      for (int j = rank - 1; j >= 0; --j) {
        const double t2 = tau2[j];
        if (t2 == 0.0) continue;
        const double* v = W2 + (int64_t)j * r;
        double w = sol[j];
        for (int i = j + 1; i < r; ++i) w = fma(v[i], sol[i], w);
        w *= t2;
        sol[j] -= w;
        for (int i = j + 1; i < r; ++i) sol[i] -= w * v[i];
      }
    }
    for (int i = 0; i < r; ++i) X[jpvt[i] + (int64_t)q * ldx] = xscl == 1.0 ? sol[i] : sol[i] * xscl;
  }
  c.sync();
  return OK;
}

}  // namespace tg
