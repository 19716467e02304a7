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

// DMMA tiled GEMM (256 threads): C = alpha*A*B + beta*C on FP64 tensor-core
// tiles (mma.sync.m8n8k4.f64).  CTA tile 64 x TN x 16, warps 2 (m) x 4 (n),
// warp tile 32 x TN/4.  SMEM double-buffered with register prefetch of the
// next K-tile; each operand is staged in the layout that keeps both its
// global loads (unit-stride dimension fastest) and the fragment reads
// bank-conflict free:  K-major [16][68] when the operand's unit stride runs
// along its M/N index, M/N-major [64][20] when it runs along K.
// ktri: B(p, j) == 0 for p < j (B = R^T of an upper-triangular R), so column
// tile j0 starts its K loop at j0.  SMEM: 2 * 2 * 1280 doubles.
template <int TN>
HDN void gemm_dm(const Ctx& c, int M, int N, int K, double alpha, Mat A, Mat B, double beta, double* C, int64_t crs,
                 int64_t ccs, double* sm, bool ktri = false) {
#if ENGINE_DEVICE
  if (c.nt != 256) {
    gemm_t<64>(c, M, N, K, alpha, A, B, beta, C, crs, ccs, sm);
    return;
  }
  constexpr int TM = 64, TK = 16, LK = 68, LM = 20, OPS = 1280;
  constexpr int WN = TN / 4, NT = WN / 8;        // warp tile columns, 8-wide n tiles per warp
  constexpr int AL = TM * TK / 256, BL = TN * TK / 256;   // elements each thread loads per K-tile
  const int warp = c.tid >> 5, lane = c.tid & 31;
  const int wm = warp & 1, wn = warp >> 1;
  const int ar = lane >> 2, ac = lane & 3;
  const bool a_kmaj = A.rs == 1;   // unit stride along i -> K-major staging
  const bool b_kmaj = B.cs == 1;   // unit stride along j -> K-major staging
  double ra[AL], rb[BL];
  for (int i0 = 0; i0 < M; i0 += TM) {
    for (int j0 = 0; j0 < N; j0 += TN) {
      const int kbeg = ktri ? (j0 / TK) * TK : 0;
      if (kbeg >= K) {
        // whole K range is zero: C = beta*C
        for (int e = c.tid; e < TM * TN; e += 256) {
          const int gi = i0 + e / TN, gj = j0 + e % TN;
          if (gi < M && gj < N) {
            double* cp = C + gi * crs + gj * ccs;
            *cp = (beta == 0.0) ? 0.0 : beta * (*cp);
          }
        }
        continue;
      }
      double acc[4][NT][2];
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int u = 0; u < NT; ++u) acc[t][u][0] = acc[t][u][1] = 0.0;
      // global -> registers for K-tile p0
      auto load = [&](int p0) {
#pragma unroll
        for (int q = 0; q < AL; ++q) {
          const int e = c.tid + 256 * q;
          int pp, ii;
          if (a_kmaj) { ii = e % TM; pp = e / TM; } else { pp = e % TK; ii = e / TK; }
          const int gi = i0 + ii, gp = p0 + pp;
          ra[q] = (gi < M && gp < K) ? A.at(gi, gp) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < BL; ++q) {
          const int e = c.tid + 256 * q;
          int pp, jj;
          if (b_kmaj) { jj = e % TN; pp = e / TN; } else { pp = e % TK; jj = e / TK; }
          const int gj = j0 + jj, gp = p0 + pp;
          rb[q] = (gj < N && gp < K) ? B.at(gp, gj) : 0.0;
        }
      };
      auto store = [&](int buf) {
        double* As = sm + buf * 2 * OPS;
        double* Bs = As + OPS;
#pragma unroll
        for (int q = 0; q < AL; ++q) {
          const int e = c.tid + 256 * q;
          if (a_kmaj) As[(e / TM) * LK + e % TM] = ra[q];
          else As[(e / TK) * LM + e % TK] = ra[q];
        }
#pragma unroll
        for (int q = 0; q < BL; ++q) {
          const int e = c.tid + 256 * q;
          if (b_kmaj) Bs[(e / TN) * LK + e % TN] = rb[q];
          else Bs[(e / TK) * LM + e % TK] = rb[q];
        }
      };
      __syncthreads();   // previous tile's readers of both buffers are done
      load(kbeg);
      store(0);
      __syncthreads();
      int buf = 0;
      for (int p0 = kbeg; p0 < K; p0 += TK) {
        const bool more = p0 + TK < K;
        if (more) load(p0 + TK);
        const double* As = sm + buf * 2 * OPS;
        const double* Bs = As + OPS;
#pragma unroll
        for (int ks = 0; ks < TK; ks += 4) {
          double fa[4], fb[NT];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int ii = wm * 32 + 8 * t + ar, pp = ks + ac;
            fa[t] = a_kmaj ? As[pp * LK + ii] : As[ii * LM + pp];
          }
#pragma unroll
          for (int u = 0; u < NT; ++u) {
            const int jj = wn * WN + 8 * u + ar, pp = ks + ac;
            fb[u] = b_kmaj ? Bs[pp * LK + jj] : Bs[jj * LM + pp];
          }
#pragma unroll
          for (int t = 0; t < 4; ++t)
#pragma unroll
            for (int u = 0; u < NT; ++u)
              asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                           : "+d"(acc[t][u][0]), "+d"(acc[t][u][1])
                           : "d"(fa[t]), "d"(fb[u]));
        }
        if (more) store(buf ^ 1);
        __syncthreads();
        buf ^= 1;
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int gi = i0 + wm * 32 + 8 * t + ar;
        if (gi >= M) continue;
#pragma unroll
        for (int u = 0; u < NT; ++u)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int gj = j0 + wn * WN + 8 * u + 2 * ac + h;
            if (gj >= N) continue;
            double* cp = C + gi * crs + gj * ccs;
            *cp = (beta == 0.0) ? alpha * acc[t][u][h] : fma(alpha, acc[t][u][h], beta * (*cp));
          }
      }
    }
  }
  __syncthreads();
#else
  (void)ktri;
  gemm_t<64>(c, M, N, K, alpha, A, B, beta, C, crs, ccs, sm);
#endif
}

#if ENGINE_DEVICE
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// W (jb x nc, row-major ld nc) = V^T C for tall V (mr x jb, col-major ld ldv)
// and C (mr x nc, col-major ld ldc), jb <= 8*JT.  Split-K over warps: each
// warp streams its own contiguous row range straight from global memory
// into DMMA fragments (no SMEM staging, no barriers in the loop, 2 row
// steps in flight), accumulating a 32 x 8*JT block of W^T; the 8 partial
// blocks are then summed in a fixed tree order through SMEM (4096 doubles).
template <int JT>
__device__ __noinline__ void gemm_vtc_dev(const Ctx& c, int64_t mr, int jb, int nc, const double* V, int64_t ldv,
                                          const double* C, int64_t ldc, double* W, double* sm) {
  const int warp = c.tid >> 5, lane = c.tid & 31, ar = lane >> 2, ac = lane & 3;
  const int64_t steps = (mr + 3) / 4;
  const int64_t s0 = steps * warp / 8, s1 = steps * (warp + 1) / 8;
  for (int i0 = 0; i0 < nc; i0 += 32) {
    double acc[4][JT][2];
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int u = 0; u < JT; ++u) acc[t][u][0] = acc[t][u][1] = 0.0;
    const double* cp[4];
    const double* vp[JT];
    bool cv[4], vv[JT];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int i = i0 + 8 * t + ar;
      cv[t] = i < nc;
      cp[t] = C + (int64_t)(cv[t] ? i : 0) * ldc + ac;
    }
#pragma unroll
    for (int u = 0; u < JT; ++u) {
      const int j = 8 * u + ar;
      vv[u] = j < jb;
      vp[u] = V + (int64_t)(vv[u] ? j : 0) * ldv + ac;
    }
    int64_t s = s0;
    for (; s + 2 <= s1; s += 2) {
      const int64_t r = 4 * s;
      double fa[2][4], fb[2][JT];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t rr = r + 4 * h;
        const bool ok = rr + ac < mr;
#pragma unroll
        for (int t = 0; t < 4; ++t) fa[h][t] = (cv[t] && ok) ? cp[t][rr] : 0.0;
#pragma unroll
        for (int u = 0; u < JT; ++u) fb[h][u] = (vv[u] && ok) ? vp[u][rr] : 0.0;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
          for (int u = 0; u < JT; ++u) dmma(acc[t][u][0], acc[t][u][1], fa[h][t], fb[h][u]);
    }
    for (; s < s1; ++s) {
      const int64_t rr = 4 * s;
      const bool ok = rr + ac < mr;
      double fa[4], fb[JT];
#pragma unroll
      for (int t = 0; t < 4; ++t) fa[t] = (cv[t] && ok) ? cp[t][rr] : 0.0;
#pragma unroll
      for (int u = 0; u < JT; ++u) fb[u] = (vv[u] && ok) ? vp[u][rr] : 0.0;
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int u = 0; u < JT; ++u) dmma(acc[t][u][0], acc[t][u][1], fa[t], fb[u]);
    }
    // fixed-order tree reduction of the 8 warp partials (4 -> 2 -> 1 rounds)
    constexpr int PS = 4 * JT * 2 * 32;   // doubles per warp partial
    for (int half = 4; half >= 1; half >>= 1) {
      __syncthreads();
      if (warp >= half && warp < 2 * half) {
        double* dst = sm + (warp - half) * PS;
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
          for (int u = 0; u < JT; ++u) {
            dst[((t * JT + u) * 2 + 0) * 32 + lane] = acc[t][u][0];
            dst[((t * JT + u) * 2 + 1) * 32 + lane] = acc[t][u][1];
          }
      }
      __syncthreads();
      if (warp < half) {
        const double* src = sm + warp * PS;
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
          for (int u = 0; u < JT; ++u) {
            acc[t][u][0] += src[((t * JT + u) * 2 + 0) * 32 + lane];
            acc[t][u][1] += src[((t * JT + u) * 2 + 1) * 32 + lane];
          }
      }
    }
    if (warp == 0) {
      // acc[t][u][h] = W^T(i = i0 + 8t + ar, j = 8u + 2ac + h)
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int u = 0; u < JT; ++u)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int i = i0 + 8 * t + ar, j = 8 * u + 2 * ac + h;
            if (i < nc && j < jb) W[(int64_t)j * nc + i] = acc[t][u][h];
          }
    }
  }
  __syncthreads();
}

// C (mr x nc, col-major ld ldc) -= V (mr x jb, col-major ld ldv) W2 (jb x nc,
// row-major ld nc), jb <= 4*KS.  W2 is staged in SMEM in column chunks of
// 160 (ld 164: conflict-free B fragments); warps stream 8-row blocks of C
// and V straight from global memory, C fragments are loaded into the
// accumulators, updated with -V fragments and stored back.
template <int KS>
__device__ __noinline__ void gemm_cmvw_dev(const Ctx& c, int64_t mr, int jb, int nc, const double* V, int64_t ldv,
                                           const double* W2, double* C, int64_t ldc, double* sm) {
  constexpr int CH = 160, LDW = 164;
  static_assert(4 * KS * LDW <= SMEM_SCRATCH_DOUBLES, "W2 chunk exceeds the SMEM scratch");
  const int warp = c.tid >> 5, lane = c.tid & 31, ar = lane >> 2, ac = lane & 3;
  const int64_t nblk = (mr + 7) / 8;
  for (int n0 = 0; n0 < nc; n0 += CH) {
    const int nw = imin(CH, nc - n0);
    __syncthreads();
    for (int e = c.tid; e < 4 * KS * LDW; e += 256) {
      const int k = e / LDW, j = e % LDW;
      sm[e] = (k < jb && j < nw) ? W2[(int64_t)k * nc + n0 + j] : 0.0;
    }
    __syncthreads();
    for (int64_t b = warp; b < nblk; b += 8) {
      const int64_t row = 8 * b + ar;
      const bool rv = row < mr;
      double fa[KS];
#pragma unroll
      for (int s = 0; s < KS; ++s) {
        const int k = 4 * s + ac;
        fa[s] = (rv && k < jb) ? -V[row + (int64_t)k * ldv] : 0.0;
      }
      for (int j0 = 0; j0 < nw; j0 += 32) {
        double acc[4][2];
        double* cp[4][2];
        bool ok[4][2];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int j = j0 + 8 * q + 2 * ac + h;
            ok[q][h] = rv && j < nw;
            cp[q][h] = C + row + (int64_t)(n0 + (ok[q][h] ? j : 0)) * ldc;
            acc[q][h] = ok[q][h] ? *cp[q][h] : 0.0;
          }
#pragma unroll
        for (int s = 0; s < KS; ++s)
#pragma unroll
          for (int q = 0; q < 4; ++q)
            dmma(acc[q][0], acc[q][1], fa[s], sm[(4 * s + ac) * LDW + j0 + 8 * q + ar]);
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            if (ok[q][h]) *cp[q][h] = acc[q][h];
      }
    }
  }
  __syncthreads();
}
#endif

// CTA reduction of a small vector (nv <= 33): every thread passes its
// partials in v[]; the totals are written to out[] (shared) and returned
// after a barrier.  Deterministic order.
// The array is taken by reference and walked by a fully unrolled loop so it
// stays in registers (a runtime-bounded loop over v[] would force the
// caller's accumulators into local memory).
template <int NV>
HD void block_reduce_vec(const Ctx& c, double (&v)[NV], int nv, double* out) {
#if ENGINE_DEVICE
  const int w = c.tid >> 5, l = c.tid & 31, nw = c.nt >> 5;
  double* part = c.red + 64;   // nw x 33 (scan buffer region)
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    if (q < nv) {
      double x = v[q];
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (l == 0) part[w * 33 + q] = x;
    }
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
    // T(0:jj, jj) = -tau_j T(0:jj, 0:jj) g,  g_q = V(:,q)^T v_j = A[j, q] + scal * dot_q.
    // Thread p owns row p of T (it reads only row p, written by itself in
    // earlier columns), so the rows are computed in parallel without barriers.
    for (int p = c.tid; p < NB; p += c.nt) {
      double tv;
      if (p < jj) {
        double s = 0.0;
        for (int q = p; q < jj; ++q) s += T[p + q * NB] * (A[(int64_t)(j0 + q) * lda + j] + scal * red[1 + q]);
        tv = -t * s;
      } else {
        tv = p == jj ? t : 0.0;   // T is upper triangular
      }
      T[p + jj * NB] = tv;
    }
    if (c.leader()) tau[j] = t;
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
      for (int q = c.tid; q < nrem; q += c.nt) red[NB + q] = t * (red[NB + q] + A[(int64_t)(j + 1 + q) * lda + j]);
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

// Left-looking form of qr_panel_nb (same reflectors, T and R up to
// rounding): column j of the panel is brought up to date by the panel's
// earlier reflectors only when it is reached -- w = V^T a_j, a_j -= V T^T w --
// and reflected in the same sweep that writes it (its norm and the dots with
// V for T accumulate while the updated values are stored).  Per column two
// sweeps over the j earlier reflector columns plus one scaling sweep,
// instead of the right-looking form's sweeps over every later column of the
// panel: ~2j + 5 column passes instead of j + 5 + 3 (jb - j - 1).
#ifndef TTGBF_QR_UNROLL
#define TTGBF_QR_UNROLL 4
#endif
template <int PW>
HDN void qr_panel_ll(const Ctx& c, double* A, int64_t lda, int m, int j0, int jb, double* tau, double* T,
                     double* sm) {
  constexpr int QU = TTGBF_QR_UNROLL;   // rows per thread per iteration
  double* red = sm;        // >= NB + 1 reduction outputs
  double* u = sm + 2 * NB; // T^T w (NB)
  for (int jj = 0; jj < jb; ++jj) {
    const int j = j0 + jj;
    double* col = A + (int64_t)j * lda;
    if (jj > 0) {
      // pass A: w_q = V_q^T a_j, V_q = e_{j0+q} + A_q[r > j0+q]
      double w[PW];
#pragma unroll
      for (int q = 0; q < PW; ++q) w[q] = 0.0;
      // QU rows per iteration: their loads are independent, so each thread
      // keeps QU x (jj + 1) loads in flight (the panel streams from L2/HBM)
      for (int64_t r0 = j0 + 1 + c.tid; r0 < m; r0 += (int64_t)QU * c.nt) {
        double x[QU];
#pragma unroll
        for (int u = 0; u < QU; ++u) {
          const int64_t r = r0 + (int64_t)u * c.nt;
          x[u] = r < m ? col[r] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < PW; ++q)
          if (q < jj) {
            const double* aq = A + (int64_t)(j0 + q) * lda;
#pragma unroll
            for (int u = 0; u < QU; ++u) {
              const int64_t r = r0 + (int64_t)u * c.nt;
              if (r < m && r > j0 + q) w[q] = fma(aq[r], x[u], w[q]);
            }
          }
      }
      block_reduce_vec(c, w, jj, red);
      // u = T^T (w + diagonal terms): u_p = sum_{q <= p} T(q, p) w_q
      for (int p = c.tid; p < jj; p += c.nt) {
        double acc = 0.0;
        for (int q = 0; q <= p; ++q) acc += T[q + p * NB] * (red[q] + col[j0 + q]);
        u[p] = acc;
      }
      c.sync();
    }
    // pass B: a_j -= V u (rows >= j0); norm^2 and V^T a_j below row j
    double v[PW + 1];
#pragma unroll
    for (int q = 0; q <= PW; ++q) v[q] = 0.0;
    for (int64_t r0 = j0 + c.tid; r0 < m; r0 += (int64_t)QU * c.nt) {
      double x[QU];
#pragma unroll
      for (int u2 = 0; u2 < QU; ++u2) {
        const int64_t r = r0 + (int64_t)u2 * c.nt;
        x[u2] = r < m ? col[r] : 0.0;
      }
      if (jj > 0) {
#pragma unroll
        for (int q = 0; q < PW; ++q)
          if (q < jj) {
            const int64_t dq = j0 + q;
            const double* aq = A + dq * lda;
#pragma unroll
            for (int u2 = 0; u2 < QU; ++u2) {
              const int64_t r = r0 + (int64_t)u2 * c.nt;
              if (r < m) {
                if (r == dq) x[u2] -= u[q];
                else if (r > dq) x[u2] = fma(-aq[r], u[q], x[u2]);
              }
            }
          }
#pragma unroll
        for (int u2 = 0; u2 < QU; ++u2) {
          const int64_t r = r0 + (int64_t)u2 * c.nt;
          if (r < m) col[r] = x[u2];
        }
      }
#pragma unroll
      for (int u2 = 0; u2 < QU; ++u2) {
        const int64_t r = r0 + (int64_t)u2 * c.nt;
        if (r < m && r > j) {
          v[0] = fma(x[u2], x[u2], v[0]);
#pragma unroll
          for (int q = 0; q < PW; ++q)
            if (q < jj) v[1 + q] = fma(A[(int64_t)(j0 + q) * lda + r], x[u2], v[1 + q]);
        }
      }
    }
    block_reduce_vec(c, v, jj + 1, red);
    const double alpha = col[j];
    double t, beta, scal;
    larfg(alpha, sqrt(red[0]), &t, &beta, &scal);
    for (int p = c.tid; p < NB; p += c.nt) {
      double tv;
      if (p < jj) {
        double s = 0.0;
        for (int q = p; q < jj; ++q) s += T[p + q * NB] * (A[(int64_t)(j0 + q) * lda + j] + scal * red[1 + q]);
        tv = -t * s;
      } else {
        tv = p == jj ? t : 0.0;
      }
      T[p + jj * NB] = tv;
    }
    if (c.leader()) tau[j] = t;
    // pass C: scale the reflector
    for (int64_t r = j + 1 + c.tid; r < m; r += c.nt) col[r] *= scal;
    c.sync();
    if (c.leader()) col[j] = beta;
    c.sync();
  }
}

// Dense copy of the panel's reflectors V (rows j0..m-1, unit diagonal,
// zeros above) into Vc (col-major, ld = m - j0).
HD void copy_v(const Ctx& c, const double* A, int64_t lda, int m, int j0, int jb, double* Vc) {
  const int64_t mr = m - j0;
  for (int q = 0; q < jb; ++q) {
    const double* aq = A + (int64_t)(j0 + q) * lda + j0;
    double* vq = Vc + (int64_t)q * mr;
    for (int64_t r = c.tid; r < mr; r += c.nt) vq[r] = r < q ? 0.0 : (r == q ? 1.0 : aq[r]);
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
#if ENGINE_DEVICE
  if (c.nt == 256) {
    if (jb <= 8) gemm_vtc_dev<1>(c, mr, jb, nc, Vc, mr, Cm + j0, ldc, W, sm);
    else gemm_vtc_dev<4>(c, mr, jb, nc, Vc, mr, Cm + j0, ldc, W, sm);
    if (trans) gemm_t<32>(c, jb, nc, jb, 1.0, Mat{T, NB, 1}, Mat{W, nc, 1}, 0.0, W2, nc, 1, sm);
    else gemm_t<32>(c, jb, nc, jb, 1.0, Mat{T, 1, NB}, Mat{W, nc, 1}, 0.0, W2, nc, 1, sm);
    if (jb <= 8) gemm_cmvw_dev<2>(c, mr, jb, nc, Vc, mr, W2, Cm + j0, ldc, sm);
    else gemm_cmvw_dev<8>(c, mr, jb, nc, Vc, mr, W2, Cm + j0, ldc, sm);
    ar.release(mk);
    return OK;
  }
#endif
  // W = V^T C   (jb x nc), computed as W^T = C^T V (nc x jb) so the DMMA
  // tile's long side runs along nc: A(i,p) = C[j0+p + i*ldc], B(p,j) = Vc[p + j*mr]
  gemm_dm<32>(c, nc, jb, (int)mr, 1.0, Mat{Cm + j0, ldc, 1}, Mat{Vc, 1, mr}, 0.0, W, 1, nc, sm);
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
  gemm_dm<64>(c, (int)mr, nc, jb, -1.0, Mat{Vc, 1, mr}, Mat{W2, nc, 1}, 1.0, Cm + j0, 1, ldc, sm);
  ar.release(mk);
  return OK;
}

// T factor of a block of jb reflectors from their Gram matrix G = V^T V
// (jb x jb, row-major) -- dlarft's recurrence T(0:j, j) = -tau_j T(0:j, 0:j)
// V(:, 0:j)^T v_j with the dot products read from G.  Leader-only, ld NB.
// Row p of T depends only on row p itself (and G), so thread p builds it
// alone: no barriers inside, same operation order as the serial recurrence.
HD void t_from_gram(const Ctx& c, const double* G, int jb, const double* tau, double* T) {
  for (int p = c.tid; p < NB; p += c.nt) {
    for (int j = 0; j < jb; ++j) {
      double tv;
      if (p < j) {
        double s = 0.0;
        for (int q = p; q < j; ++q) s += T[p + q * NB] * G[q * jb + j];
        tv = -tau[j] * s;
      } else {
        tv = p == j ? tau[j] : 0.0;
      }
      T[p + j * NB] = tv;
    }
  }
  c.sync();
}

// Blocked QR of A (m x n, col-major lda).  Ts: ceil(min(m,n)/NB) * NB*NB.
// Two-level blocking: each NB-column panel is factored as NS-column
// sub-panels (level-2) whose block reflectors update the rest of the panel
// with GEMMs, so a tall panel is streamed ~3x instead of ~NB times; the
// panel's T comes from one Gram GEMM of its explicit V (which the trailing
// update needs anyway).
#ifndef TTGBF_QR_NS
#define TTGBF_QR_NS 4   /* measured (two-level at every height): 8 -> 12046, 4 -> 11591, 2 -> 12005 CTA-s per bench launch */
#endif
constexpr int NS = TTGBF_QR_NS;   // sub-panel width of the two-level panel factorisation
#ifndef TTGBF_QR_PANEL_LL
#define TTGBF_QR_PANEL_LL 1
#endif
HDN void qr_panel_blk(const Ctx& c, double* A, int64_t lda, int m, int j0, int jb, double* tau, double* T, double* sm) {
#if TTGBF_QR_PANEL_LL
  // register arrays sized to the panel: sub-panels (jb <= 8) keep their 8 + 9
  // accumulators in registers; the 32-wide instance spills part of them
  if (jb <= 4) qr_panel_ll<4>(c, A, lda, m, j0, jb, tau, T, sm);
  else if (jb <= 8) qr_panel_ll<8>(c, A, lda, m, j0, jb, tau, T, sm);
  else qr_panel_ll<NB>(c, A, lda, m, j0, jb, tau, T, sm);
#else
  qr_panel_nb(c, A, lda, m, j0, jb, tau, T, sm);
#endif
}
#ifndef TTGBF_QR2_MIN_ROWS
#define TTGBF_QR2_MIN_ROWS 0   /* measured: 2048 -> 226, 512 -> 234, 0 -> 237 steps/s (the 32-wide single-level panel spills its accumulators) */
#endif
constexpr int QR2_MIN_ROWS = TTGBF_QR2_MIN_ROWS;   // panels taller than this use two-level blocking
HDN int geqrf_nb(const Ctx& c, Arena& ar, double* A, int64_t lda, int m, int n, double* tau, double* Ts,
                 double* sm) {
  const int k = imin(m, n);
  for (int j0 = 0; j0 < k; j0 += NB) {
    const int jb = imin(NB, k - j0);
    double* T = Ts + (int64_t)(j0 / NB) * NB * NB;
    const int64_t mr = m - j0;
    size_t mk = ar.mark();
    if (mr <= QR2_MIN_ROWS || jb <= NS) {
      PROF(c, 16);
      qr_panel_blk(c, A, lda, m, j0, jb, tau, T, sm);
    } else {
      PROF(c, 16);
      double *Ts_, *Vs;
      ALLOC(Ts_, double, NB * NB, ar);
      ALLOC(Vs, double, mr * NS, ar);
      for (int s0 = 0; s0 < jb; s0 += NS) {
        const int sb = imin(NS, jb - s0);
        qr_panel_blk(c, A, lda, m, j0 + s0, sb, tau, Ts_, sm);
        if (s0 + sb < jb) {
          copy_v(c, A, lda, m, j0 + s0, sb, Vs);
          CK(apply_block(c, ar, Vs, m, j0 + s0, sb, Ts_, true, A + (int64_t)(j0 + s0 + sb) * lda, lda,
                         jb - s0 - sb, sm));
        }
      }
    }
    const bool trail = j0 + jb < n;
    if (trail || !(mr <= QR2_MIN_ROWS || jb <= NS)) {
      PROF(c, 17);
      double *Vc, *G;
      ALLOC(Vc, double, mr * jb, ar);
      copy_v(c, A, lda, m, j0, jb, Vc);
      if (!(mr <= QR2_MIN_ROWS || jb <= NS)) {
        ALLOC(G, double, jb * jb, ar);
        // G = V^T V: A(i,p) = Vc[p + i*mr], B(p,j) = Vc[p + j*mr]
#if ENGINE_DEVICE
        if (c.nt == 256) gemm_vtc_dev<4>(c, mr, jb, jb, Vc, mr, Vc, mr, G, sm);
        else
#endif
        gemm_dm<32>(c, jb, jb, (int)mr, 1.0, Mat{Vc, mr, 1}, Mat{Vc, 1, mr}, 0.0, G, jb, 1, sm);
        t_from_gram(c, G, jb, tau + j0, T);
      }
      if (trail)
        CK(apply_block(c, ar, Vc, m, j0, jb, T, true, A + (int64_t)(j0 + jb) * lda, lda, n - (j0 + jb), sm));
    }
    ar.release(mk);
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

// Y (m x ny, col-major ldy) <- H_0 H_1 ... H_{k-1} Y for reflectors stored
// LAPACK-style in the columns of A (unit diagonal implied) with scalars tau
// but no T factors (e.g. the pivoted QR): blocks of NB get their T from a
// Gram GEMM, then one block-reflector application each (last block first).
HDN int apply_refl_blocked(const Ctx& c, Arena& ar, const double* A, int64_t lda, int m, int k, const double* tau,
                           double* Y, int64_t ldy, int ny, double* sm) {
  const int nblk = (k + NB - 1) / NB;
  for (int b = nblk - 1; b >= 0; --b) {
    const int j0 = b * NB, jb = imin(NB, k - j0);
    const int64_t mr = m - j0;
    size_t mk = ar.mark();
    double *Vc, *G, *T;
    ALLOC(Vc, double, mr * jb, ar);
    ALLOC(G, double, jb * jb, ar);
    ALLOC(T, double, NB * NB, ar);
    copy_v(c, A, lda, m, j0, jb, Vc);
#if ENGINE_DEVICE
    if (c.nt == 256) gemm_vtc_dev<4>(c, mr, jb, jb, Vc, mr, Vc, mr, G, sm);
    else
#endif
    gemm_dm<32>(c, jb, jb, (int)mr, 1.0, Mat{Vc, mr, 1}, Mat{Vc, 1, mr}, 0.0, G, jb, 1, sm);
    t_from_gram(c, G, jb, tau + j0, T);
    CK(apply_block(c, ar, Vc, m, j0, jb, T, false, Y, ldy, ny, sm));
    ar.release(mk);
  }
  return OK;
}

}  // namespace tg
