// Greedy restricted TT-cross on the device (tt_algorithms.py:463-596).
//
// One CTA runs one cross.  Decisions (random candidate sets, sorting,
// pivot adoption, stopping) are taken by the CTA leader with the numpy-
// compatible PCG64 stream (rng.cuh) in exactly the reference's draw order;
// evaluations, error scans, TT point evaluations and the core least-squares
// solves are CTA-parallel.  Constants: tt_algorithms.py:49-58.
#pragma once
#include "common.cuh"
#include "rng.cuh"
#include "rng_warp.cuh"
#include "linalg.cuh"
#include "tt.cuh"
#include "models.cuh"
#include "cache.cuh"

namespace tg {

constexpr int X_INIT = 32, X_CAND = 10, X_ROOK = 2, X_SCAN = 1024, X_BATCH = 24, X_INJECT = 8;
constexpr int X_FRESH = 128, X_SAMPLE = 4096, X_GATE = 32768;
constexpr double X_TINY = 2.2250738585072014e-308;
constexpr int X_MAXR = 160;  // per-thread solve buffers bound the cross rank

struct CrossCfg {
  double tol;
  int max_rank;
  int max_sweeps;
  int validation_count;
  const int32_t* seeds;   // (nseeds x d) or null
  int nseeds;
  Pcg64 rng;              // initial state of default_rng(rng_seed) (host-derived)
  int64_t cache_cap;
};

struct CrossInfo {
  double achieved;
  int64_t calls;
  int sweeps;
  int converged;
};

// Pivot tuples are stored as int16 rows of MAXD entries.
struct XState {
  int d;
  int n[MAXD];
  int maxr;
  int rank[MAXD];           // rank[b], b = 1..d-1
  int16_t* rows[MAXD];      // rows[b][t*MAXD + j], j < b
  int16_t* cols[MAXD];      // cols[b][t*MAXD + j], j < d-b
  double* fib[MAXD];        // (Acap x n x Ccap)
  double* core[MAXD];
  int ccap[MAXD];
  double* ahat[MAXD];       // maxr x maxr row-major
};

struct XShared {           // leader-published scalars
  Pcg64 rng;
  int64_t i0, i1, i2;
  double f0, f1;
};

struct ChoiceWs {
  int32_t* disp;     // virtual arange for tail shuffles (-1 = untouched)
  uint32_t* gset;    // Floyd first-occurrence table when it does not fit shared memory
  uint8_t* flags;    // per-draw collision flags
  int64_t* touch;    // touched positions / shuffle draws
  int64_t* draws;    // pre-drawn bounded values
  const PcgJump* jt; // PCG64 jump-ahead table of this stream
};

HD int x_left(const XState& s, int k) { return k == 0 ? 1 : s.rank[k]; }
HD int x_right(const XState& s, int k) { return k == s.d - 1 ? 1 : s.rank[k + 1]; }
HD int x_limit(const XState& s, int b, int max_rank) {
  return imin(max_rank, imin(x_left(s, b - 1) * s.n[b - 1], s.n[b] * x_right(s, b)));
}
HD const int16_t* x_lrow(const XState& s, int k, int a) { return k == 0 ? nullptr : s.rows[k] + a * MAXD; }
HD const int16_t* x_rcol(const XState& s, int k, int c) { return k == s.d - 1 ? nullptr : s.cols[k + 1] + c * MAXD; }

HD bool tuple_lt(const int16_t* a, const int16_t* b, int len) {
  for (int j = 0; j < len; ++j)
    if (a[j] != b[j]) return a[j] < b[j];
  return false;
}

// leader: order[0..cnt) = indices of list rows [base, base+cnt) sorted by tuple
HD void sort_tuples(const int16_t* list, int base, int cnt, int len, int* order) {
  for (int t = 0; t < cnt; ++t) order[t] = base + t;
  for (int t = 1; t < cnt; ++t) {
    int p = order[t], q = t - 1;
    while (q >= 0 && tuple_lt(list + p * MAXD, list + order[q] * MAXD, len)) { order[q + 1] = order[q]; --q; }
    order[q + 1] = p;
  }
}

// Cartesian block (left(k) x arange(n_k) x right(k)) restricted to the left
// rows [a0, a1) and right cols [c0, c1), enumerated in ascending key order
// (sorted prefixes, mode index, sorted suffixes).  lo[] / co[] receive the
// original row / col of each sorted position.
HDN void x_block_idx(const Ctx& c, const XState& s, int k, int a0, int a1, int c0, int c1, int32_t* idx,
                     int* lo, int* co) {
  const int d = s.d, n = s.n[k];
  const int na = a1 - a0, nc = c1 - c0;
  if (c.leader()) {
    if (k == 0) lo[0] = 0; else sort_tuples(s.rows[k], a0, na, k, lo);
    if (k == d - 1) co[0] = 0; else sort_tuples(s.cols[k + 1], c0, nc, d - k - 1, co);
  }
  c.sync();
  const int64_t tot = (int64_t)na * n * nc;
  for (int64_t e = c.tid; e < tot; e += c.nt) {
    const int cc = (int)(e % nc);
    const int i = (int)((e / nc) % n);
    const int aa = (int)(e / ((int64_t)nc * n));
    int32_t* o = idx + e * d;
    const int16_t* L = x_lrow(s, k, lo[aa]);
    for (int j = 0; j < k; ++j) o[j] = L[j];
    o[k] = i;
    const int16_t* R = x_rcol(s, k, co[cc]);
    for (int j = 0; j < d - k - 1; ++j) o[k + 1 + j] = R[j];
  }
  c.sync();
}

// fibre slab for core k over left rows [a0,a1) and right cols [c0,c1)
HDN int x_fill_fib(const Ctx& c, Arena& ar, Cache* C, const EvalSpec& spec, XState& s, int k,
                          int a0, int a1, int c0, int c1, double* sm) {
  const int n = s.n[k];
  const int64_t tot = (int64_t)(a1 - a0) * n * (c1 - c0);
  if (tot == 0) return OK;
  size_t mk = ar.mark();
  int32_t* idx;
  double* v;
  int *lo, *co;
  ALLOC(idx, int32_t, tot * s.d, ar);
  ALLOC(v, double, tot, ar);
  ALLOC(lo, int, a1 - a0, ar);
  ALLOC(co, int, c1 - c0, ar);
  x_block_idx(c, s, k, a0, a1, c0, c1, idx, lo, co);
  CK(cache_eval(c, ar, C, spec, idx, tot, v, sm, true));
  const int nc = c1 - c0;
  for (int64_t e = c.tid; e < tot; e += c.nt) {
    const int cc = (int)(e % nc);
    const int i = (int)((e / nc) % n);
    const int aa = (int)(e / ((int64_t)nc * n));
    s.fib[k][((int64_t)lo[aa] * n + i) * s.ccap[k] + co[cc]] = v[e];
  }
  c.sync();
  ar.release(mk);
  return OK;
}

// pivot block entries for rows [r0,r1) x cols [q0,q1) of bond b into ahat
HDN int x_fill_ahat(const Ctx& c, Arena& ar, Cache* C, const EvalSpec& spec, XState& s, int b,
                           int r0, int r1, int q0, int q1, double* sm) {
  const int nr = r1 - r0, nq = q1 - q0;
  if (nr <= 0 || nq <= 0) return OK;
  const int d = s.d;
  size_t mk = ar.mark();
  int32_t* idx;
  double* v;
  ALLOC(idx, int32_t, (int64_t)nr * nq * d, ar);
  ALLOC(v, double, (int64_t)nr * nq, ar);
  for (int64_t e = c.tid; e < (int64_t)nr * nq; e += c.nt) {
    const int t = (int)(e / nq), q = (int)(e % nq);
    int32_t* o = idx + e * d;
    const int16_t* R = s.rows[b] + (r0 + t) * MAXD;
    const int16_t* Q = s.cols[b] + (q0 + q) * MAXD;
    for (int j = 0; j < b; ++j) o[j] = R[j];
    for (int j = 0; j < d - b; ++j) o[b + j] = Q[j];
  }
  c.sync();
  CK(cache_eval(c, ar, C, spec, idx, (int64_t)nr * nq, v, sm));
  for (int64_t e = c.tid; e < (int64_t)nr * nq; e += c.nt) {
    const int t = (int)(e / nq), q = (int)(e % nq);
    s.ahat[b][(r0 + t) * s.maxr + q0 + q] = v[e];
  }
  c.sync();
  ar.release(mk);
  return OK;
}

// core k from fibres and the pivot block of bond k+1 (tt_algorithms.py:295-308)
HDN int x_solve_core(const Ctx& c, Arena& ar, XState& s, int k, double* sm) {
  const int d = s.d, n = s.n[k];
  const int A = x_left(s, k);
  const int Cc = x_right(s, k);
  const int cc = s.ccap[k];
  if (k == d - 1) {
    for (int64_t e = c.tid; e < (int64_t)A * n; e += c.nt) s.core[k][e * cc] = s.fib[k][e * cc];
    c.sync();
    return OK;
  }
  PROF(c, 3);
  size_t mk = ar.mark();
  const int r = Cc;
  double *W, *W2, *tau, *tau2, *cn;
  int* jpvt;
  ALLOC(W, double, (int64_t)r * r, ar);
  ALLOC(W2, double, (int64_t)r * r, ar);
  ALLOC(tau, double, r, ar);
  ALLOC(tau2, double, r, ar);
  ALLOC(cn, double, r + 1, ar);
  ALLOC(jpvt, int, r, ar);
  // A_ls = ahat^T: (i,j) -> ahat[j][i]; B(i, row) = fib[row*cc + i]
  int rank_used = 0;
  CK(lstsq_pivoted(c, s.ahat[k + 1], 1, s.maxr, r, s.fib[k], cc, A * n, s.core[k], cc, W, W2, tau, tau2, jpvt,
                   cn, &rank_used, sm, SMEM_SCRATCH_DOUBLES));
#if defined(ENGINE_HOSTSIM) && defined(ENGINE_TRACE)
  {
    double cs = 0.0;
    for (int64_t e = 0; e < (int64_t)A * n; ++e)
      for (int i = 0; i < r; ++i) cs += fabs(s.core[k][e * cc + i]);
    fprintf(stderr, "SOLVE k=%d r=%d rank=%d rows=%d sum=%.17g\n", k, r, rank_used, A * n, cs);
  }
#endif
  ar.release(mk);
  return OK;
}

// compact snapshot of the current interpolant
HDN int x_snapshot(const Ctx& c, Arena& ar, const XState& s, TT& t) {
  PROF(c, 11);
  int r[MAXD + 1];
  r[0] = 1;
  for (int b = 1; b < s.d; ++b) r[b] = s.rank[b];
  r[s.d] = 1;
  CK(tt_alloc(ar, t, s.d, s.n, r));
  for (int k = 0; k < s.d; ++k) {
    const int64_t tot = t.size(k);
    const int rr = t.r[k + 1];
    for (int64_t e = c.tid; e < tot; e += c.nt) {
      const int64_t row = e / rr;
      const int cc = (int)(e % rr);
      t.c[k][e] = s.core[k][row * s.ccap[k] + cc];
    }
  }
  c.sync();
  return OK;
}

HD bool tuple_eq(const int16_t* a, const int16_t* b, int len) {
  for (int j = 0; j < len; ++j)
    if (a[j] != b[j]) return false;
  return true;
}
HD bool tuple_in(const int16_t* list, int cnt, const int16_t* x, int len) {
  for (int t = 0; t < cnt; ++t)
    if (tuple_eq(list + t * MAXD, x, len)) return true;
  return false;
}

// accept new pivots at bond b (tt_algorithms.py:310-335).  New rows/cols are
// already appended to s.rows[b]/s.cols[b] at positions [old, old+m).
HDN int x_accept(const Ctx& c, Arena& ar, Cache* C, const EvalSpec& spec, XState& s, int b, int m,
                        double* sm) {
  PROF(c, 5);
  const int old = s.rank[b];
  // row block (new rows x old cols), then col block (all rows x new cols)
  CK(x_fill_ahat(c, ar, C, spec, s, b, old, old + m, 0, old, sm));
  CK(x_fill_ahat(c, ar, C, spec, s, b, 0, old + m, old, old + m, sm));
  if (c.leader()) s.rank[b] = old + m;
  c.sync();
  // left slabs of fibre b (new rows x n_b x right(b)); right slabs of fibre b-1
  CK(x_fill_fib(c, ar, C, spec, s, b, old, old + m, 0, x_right(s, b), sm));
  CK(x_fill_fib(c, ar, C, spec, s, b - 1, 0, x_left(s, b - 1), old, old + m, sm));
  CK(x_solve_core(c, ar, s, b - 1, sm));
  CK(x_solve_core(c, ar, s, b, sm));
  return OK;
}

// errors |ev(cell) - g_left[row] . f_right[:, col]| for flat (row, col) pairs
struct HuntGeo {
  int b, nl, ns, nrow, ncol, r;
};
HDN int x_errors(const Ctx& c, Arena& ar, Cache* C, const EvalSpec& spec, const XState& s,
                        const HuntGeo& g, const int64_t* rf, const int64_t* cf, int64_t K, double* err, double* sm) {
  const int d = s.d, b = g.b;
  size_t mk = ar.mark();
  int32_t* idx;
  double* v;
  ALLOC(idx, int32_t, K * d, ar);
  ALLOC(v, double, K, ar);
  for (int64_t p = c.tid; p < K; p += c.nt) {
    int32_t* o = idx + p * d;
    const int64_t row = rf[p], col = cf[p];
    const int16_t* L = x_lrow(s, b - 1, (int)(row / g.nl));
    for (int j = 0; j < b - 1; ++j) o[j] = L[j];
    o[b - 1] = (int)(row % g.nl);
    o[b] = (int)(col / g.ns);
    const int16_t* R = x_rcol(s, b, (int)(col % g.ns));
    for (int j = 0; j < d - b - 1; ++j) o[b + 1 + j] = R[j];
  }
  c.sync();
  CK(cache_eval(c, ar, C, spec, idx, K, v, sm));
  const int ccl = s.ccap[b - 1], ccr = s.ccap[b], nb = s.n[b];
  for (int64_t p = c.tid; p < K; p += c.nt) {
    const int64_t row = rf[p], col = cf[p];
    const double* gl = s.core[b - 1] + row * ccl;
    const int i = (int)(col / g.ns), cc = (int)(col % g.ns);
    double acc = 0.0;
    for (int t = 0; t < g.r; ++t) acc = fma(gl[t], s.fib[b][((int64_t)t * nb + i) * ccr + cc], acc);
    err[p] = fabs(v[p] - acc);
  }
  c.sync();
  ar.release(mk);
  return OK;
}

struct Cand {
  int64_t row, col;
  double err;
};

// _hunt_candidates (tt_algorithms.py:341-421).  Writes up to 101 candidates
// (rook winner first) to `cand`, returns count and err_seen.
HDN int x_hunt(const Ctx& c, Arena& ar, Cache* C, const EvalSpec& spec, XState& s, int b, XShared* sh,
                      const ChoiceWs& rws, Cand* cand, int* ncand, double* err_seen, double* sm) {
  PROF(c, 4);
  HuntGeo g;
  g.b = b;
  g.nl = s.n[b - 1];
  g.ns = x_right(s, b);
  g.nrow = x_left(s, b - 1) * g.nl;
  g.ncol = s.n[b] * g.ns;
  g.r = s.rank[b];
  size_t mk = ar.mark();
  const int qr = imin(X_CAND, g.nrow), qc = imin(X_CAND, g.ncol);
  int64_t *cr, *cc, *br, *bc;
  double* e;
  ALLOC(cr, int64_t, X_CAND, ar);
  ALLOC(cc, int64_t, X_CAND, ar);
  ALLOC(br, int64_t, X_SCAN, ar);
  ALLOC(bc, int64_t, X_SCAN, ar);
  ALLOC(e, double, X_SCAN, ar);
  {
    PROF(c, 10);
    warp_choice(c, &sh->rng, rws.jt, g.nrow, qr, cr, rws.disp, rws.touch, rws.draws, rws.flags, reinterpret_cast<uint32_t*>(sm), 2 * SMEM_SCRATCH_DOUBLES, rws.gset);
    warp_choice(c, &sh->rng, rws.jt, g.ncol, qc, cc, rws.disp, rws.touch, rws.draws, rws.flags, reinterpret_cast<uint32_t*>(sm), 2 * SMEM_SCRATCH_DOUBLES, rws.gset);
  }
  for (int e = c.tid; e < qr * qc; e += c.nt) { br[e] = cr[e / qc]; bc[e] = cc[e % qc]; }
  c.sync();
  const int nb = qr * qc;
  CK(x_errors(c, ar, C, spec, s, g, br, bc, nb, e, sm));
  int nc_ = 0;
  double seen = 0.0;
  int64_t rbest = 0, cbest = 0;
  {
    // argsort ascending (stable) then reversed: descending, later index first
    // on ties.  Thread i places element i at its stable rank (the number of
    // elements that precede it), all ranks in parallel.
    double* es = sm;   // nb <= X_CAND^2 errors staged in SMEM
    for (int i = c.tid; i < nb; i += c.nt) es[i] = e[i];
    c.sync();
    for (int i = c.tid; i < nb; i += c.nt) {
      const double ei = es[i];
      int rank = 0;
      for (int j = 0; j < nb; ++j) {
        const double ej = es[j];
        rank += (ej < ei || (ej == ei && j < i)) ? 1 : 0;
      }
      cand[1 + (nb - 1 - rank)] = Cand{br[i], bc[i], ei};
    }
    c.sync();
    if (c.leader()) {
      nc_ = nb;
      if (nb > 0) { seen = cand[1].err; rbest = cand[1].row; cbest = cand[1].col; }
      sh->i0 = rbest; sh->i1 = cbest; sh->f0 = seen;
    }
    c.sync();   // publish the leader's pick before anyone reads it
  }
  rbest = sh->i0; cbest = sh->i1; seen = sh->f0;
  nc_ = nb;
  c.sync();
  for (int it = 0; it < X_ROOK; ++it) {
    // column scan over (sampled) rows
    int nsr = 0;
    if (g.nrow > X_SCAN) {
      PROF(c, 10);
      warp_choice(c, &sh->rng, rws.jt, g.nrow, X_SCAN, br, rws.disp, rws.touch, rws.draws, rws.flags, reinterpret_cast<uint32_t*>(sm), 2 * SMEM_SCRATCH_DOUBLES, rws.gset);
    }
    nsr = imin(g.nrow, X_SCAN);
    if (g.nrow <= X_SCAN)
      for (int i = c.tid; i < nsr; i += c.nt) br[i] = i;
    for (int i = c.tid; i < nsr; i += c.nt) bc[i] = cbest;
    c.sync();
    CK(x_errors(c, ar, C, spec, s, g, br, bc, nsr, e, sm));
    ValIdx best{-1.0, 0};
    for (int i = c.tid; i < nsr; i += c.nt) best = vi_better(best, ValIdx{e[i], i});
    best = block_argmax(c, best);
    const int64_t rnew = br[best.i];
    const double mcol = best.v;
    c.sync();
    int nsc = 0;
    if (g.ncol > X_SCAN) {
      PROF(c, 10);
      warp_choice(c, &sh->rng, rws.jt, g.ncol, X_SCAN, bc, rws.disp, rws.touch, rws.draws, rws.flags, reinterpret_cast<uint32_t*>(sm), 2 * SMEM_SCRATCH_DOUBLES, rws.gset);
    }
    nsc = imin(g.ncol, X_SCAN);
    if (g.ncol <= X_SCAN)
      for (int i = c.tid; i < nsc; i += c.nt) bc[i] = i;
    for (int i = c.tid; i < nsc; i += c.nt) br[i] = rnew;
    c.sync();
    CK(x_errors(c, ar, C, spec, s, g, br, bc, nsc, e, sm));
    ValIdx best2{-1.0, 0};
    for (int i = c.tid; i < nsc; i += c.nt) best2 = vi_better(best2, ValIdx{e[i], i});
    best2 = block_argmax(c, best2);
    const int64_t cnew = bc[best2.i];
    const double mrow = best2.v;
    seen = fmax(seen, fmax(mcol, mrow));
    c.sync();
    if (rnew == rbest && cnew == cbest) break;
    rbest = rnew;
    cbest = cnew;
  }
  if (c.leader()) { br[0] = rbest; bc[0] = cbest; }
  c.sync();
  CK(x_errors(c, ar, C, spec, s, g, br, bc, 1, e, sm));
  if (c.leader()) cand[0] = Cand{rbest, cbest, e[0]};
#if defined(ENGINE_HOSTSIM) && defined(ENGINE_TRACE)
  fprintf(stderr, "HUNT b=%d rook=(%lld,%lld) e=%.17g seen=%.17g top=(%lld,%lld,%.17g)\n", b, (long long)rbest,
          (long long)cbest, e[0], seen, (long long)cand[1].row, (long long)cand[1].col, cand[1].err);
#endif
  c.sync();
  *ncand = nc_ + 1;
  *err_seen = seen;
  ar.release(mk);
  return OK;
}

// split flat (row, col) at bond b into prefix/suffix tuples
HD void x_split(const XState& s, int b, int64_t row, int64_t col, int16_t* rt, int16_t* ct) {
  const int nl = s.n[b - 1], ns = x_right(s, b);
  const int16_t* L = x_lrow(s, b - 1, (int)(row / nl));
  for (int j = 0; j < b - 1; ++j) rt[j] = L[j];
  rt[b - 1] = (int16_t)(row % nl);
  ct[0] = (int16_t)(col / ns);
  const int16_t* R = x_rcol(s, b, (int)(col % ns));
  for (int j = 0; j < s.d - b - 1; ++j) ct[1 + j] = R[j];
}

// _cache_check (tt_algorithms.py:424-433): worst `top` errors over a random
// cache subsample; out_err/out_cell (cells as int32 x d), sorted worst first.
HDN int x_check(const Ctx& c, Arena& ar, Cache* C, XShared* sh, const ChoiceWs& rws, const TT& t,
                       int count, int top, double* out_err, int32_t* out_cell, int* nout, double* sm) {
  const int d = C->d;
  PROF(c, 6);
  size_t mk = ar.mark();
  const int64_t cnt = C->count;
  const int64_t K = cnt > count ? count : cnt;
  int64_t* sel;
  int32_t* idx;
  double *vals, *tv;
  ALLOC(sel, int64_t, K, ar);
  ALLOC(idx, int32_t, K * d, ar);
  ALLOC(vals, double, K, ar);
  ALLOC(tv, double, K, ar);
  if (cnt > count) {
    PROF(c, 10);
    warp_choice(c, &sh->rng, rws.jt, cnt, count, sel, rws.disp, rws.touch, rws.draws, rws.flags, reinterpret_cast<uint32_t*>(sm), 2 * SMEM_SCRATCH_DOUBLES, rws.gset);
  } else if (c.leader()) {
    for (int64_t i = 0; i < cnt; ++i) sel[i] = i;
  }
  c.sync();
  for (int64_t p = c.tid; p < K; p += c.nt) {
    unpack_key(d, C->bits, C->keys[sel[p]], idx + p * d);
    vals[p] = C->vals[sel[p]];
  }
  c.sync();
  {
    PROF(c, 12);
    IndexSlice is{&t, idx, 0};
    CK(tt_eval_bucketed(c, ar, t, K, is, tv, sm));
  }
  for (int64_t p = c.tid; p < K; p += c.nt) tv[p] = fabs(vals[p] - tv[p]);
  c.sync();
  // top-k: repeated arg-max preferring the LAST index on ties (argsort[::-1])
  const int kk = (int)lmin(top, K);
  for (int q = 0; q < kk; ++q) {
    ValIdx best{-1.0, -1};
    for (int64_t p = c.tid; p < K; p += c.nt) {
      const double v = tv[p];
      if (v > best.v || (v == best.v && p > best.i)) best = ValIdx{v, p};
    }
    // reduce with "later index wins ties": negate indices for block_argmax
    best.i = -best.i;
    best = block_argmax(c, best);
    const int64_t pi = -best.i;
    if (c.leader()) {
      out_err[q] = tv[pi];
      for (int j = 0; j < d; ++j) out_cell[q * d + j] = idx[pi * d + j];
      tv[pi] = -2.0;   // exclude (errors are >= 0)
    }
    c.sync();
  }
  *nout = kk;
  ar.release(mk);
  return OK;
}

// _inject_cells (tt_algorithms.py:436-460)
HDN int x_inject(const Ctx& c, Arena& ar, Cache* C, const EvalSpec& spec, XState& s, XShared* sh,
                        const double* oerr, const int32_t* ocell, int nof, double thr, int max_rank,
                        bool* grew, double* sm) {
  const int d = s.d;
  PROF(c, 13);
  int pend[MAXD];
  for (int b = 0; b < d; ++b) pend[b] = 0;
  // leader decides; pending rows/cols are appended to the state's lists
  // (beyond rank[b]) and committed bond by bond in sorted order.
  if (c.leader()) {
    for (int q = 0; q < nof; ++q) {
      if (oerr[q] <= thr) break;
      const int32_t* cell = ocell + q * d;
      for (int b = 1; b < d; ++b) {
        if (s.rank[b] + pend[b] >= x_limit(s, b, max_rank)) continue;
        int16_t rt[MAXD], ct[MAXD];
        for (int j = 0; j < b; ++j) rt[j] = (int16_t)cell[j];
        for (int j = 0; j < d - b; ++j) ct[j] = (int16_t)cell[b + j];
        if (tuple_in(s.rows[b], s.rank[b] + pend[b], rt, b)) continue;
        if (tuple_in(s.cols[b], s.rank[b] + pend[b], ct, d - b)) continue;
        int16_t* dr = s.rows[b] + (s.rank[b] + pend[b]) * MAXD;
        int16_t* dc = s.cols[b] + (s.rank[b] + pend[b]) * MAXD;
        for (int j = 0; j < b; ++j) dr[j] = rt[j];
        for (int j = 0; j < d - b; ++j) dc[j] = ct[j];
        pend[b]++;
        break;
      }
    }
    for (int b = 1; b < d; ++b) sh->rng.s_lo ^= 0, (void)0;
    int64_t* pp = reinterpret_cast<int64_t*>(&sh->i0);
    (void)pp;
  }
  // publish pend[] through the shared scalars area: reuse red via bcast
  bool any = false;
  for (int b = 1; b < d; ++b) {
    const int m = (int)bcast_i(c, pend[b]);
    if (m > 0) {
      CK(x_accept(c, ar, C, spec, s, b, m, sm));
      any = true;
    }
  }
  if (any) *grew = true;
  return OK;
}

// ---------------------------------------------------------------------------
// greedy_cross
// ---------------------------------------------------------------------------
HDN int greedy_cross(const Ctx& c, Arena& ar, const EvalSpec& spec, const CrossCfg& cfg, XShared* sh,
                            TT& out, CrossInfo* info, double* sm) {
  const int d = spec.d;
  if (cfg.max_rank < 1 || cfg.max_rank > X_MAXR || cfg.max_sweeps < 1 || cfg.validation_count < 1 ||
      !(cfg.tol > 0.0))
    return E_ARG;
  Cache* C;
  CK(cache_init(c, ar, C, d, spec.n, cfg.cache_cap));
  if (c.leader()) sh->rng = cfg.rng;
  c.sync();
  // RNG workspace for choice(): up to the gate sample from a large cache
  ChoiceWs rws;
  {
    int maxn = 1;
    for (int k = 0; k < d; ++k) maxn = imax(maxn, spec.n[k]);
    const int64_t dcap = lmax(cfg.cache_cap + 16, (int64_t)cfg.max_rank * maxn + 16);
    ALLOC(rws.gset, uint32_t, 2 * (gen_mask((uint64_t)(1.2 * X_GATE)) + 1), ar);
    ALLOC(rws.flags, uint8_t, X_GATE + X_SCAN, ar);
    ALLOC(rws.disp, int32_t, dcap, ar);
    ALLOC(rws.touch, int64_t, X_GATE + X_SCAN, ar);
    ALLOC(rws.draws, int64_t, X_GATE + X_SCAN, ar);
    PcgJump* jt;
    ALLOC(jt, PcgJump, 1, ar);
    if (c.leader()) pcg_make_jump(cfg.rng, jt);
    rws.jt = jt;
    par_fill_i32(c, rws.disp, dcap, -1);
    c.sync();
  }
  if (d == 1) {
    int32_t* idx;
    double* v;
    ALLOC(idx, int32_t, spec.n[0], ar);
    ALLOC(v, double, spec.n[0], ar);
    for (int i = c.tid; i < spec.n[0]; i += c.nt) idx[i] = i;
    c.sync();
    CK(cache_eval(c, ar, C, spec, idx, spec.n[0], v, sm));
    int n1[1] = {spec.n[0]}, r1[2] = {1, 1};
    CK(tt_alloc(ar, out, 1, n1, r1));
    par_copy(c, out.c[0], v, spec.n[0]);
    c.sync();
    info->achieved = 0.0; info->calls = C->calls; info->sweeps = 0; info->converged = 1;
    return OK;
  }
  // --- seed pivot: argmax |v| over random probes (+ seeds)
  const int nprobe = X_INIT + 4 * d;
  const int64_t K0 = nprobe + cfg.nseeds;
  int32_t* probes;
  double* pv;
  ALLOC(probes, int32_t, K0 * d, ar);
  ALLOC(pv, double, K0, ar);
  warp_integers(c, &sh->rng, rws.jt, spec.n, d, nprobe, probes, rws.draws);
  for (int64_t e = c.tid; e < (int64_t)cfg.nseeds * d; e += c.nt) probes[(int64_t)nprobe * d + e] = cfg.seeds[e];
  c.sync();
  CK(cache_eval(c, ar, C, spec, probes, K0, pv, sm));
  ValIdx bp{-1.0, 0};
  for (int64_t p = c.tid; p < K0; p += c.nt) bp = vi_better(bp, ValIdx{fabs(pv[p]), p});
  bp = block_argmax(c, bp);
  int32_t pivot[MAXD];
  for (int j = 0; j < d; ++j) pivot[j] = probes[bp.i * d + j];
  // --- state
  XState& s = *reinterpret_cast<XState*>(sh + 1);   // lives in the shared block after XShared
  XState* sp = &s;
  (void)sp;
  const int maxr = cfg.max_rank;
  if (c.leader()) {
    s.d = d;
    s.maxr = maxr;
    for (int k = 0; k < d; ++k) s.n[k] = spec.n[k];
  }
  c.sync();
  // allocations (all threads identical)
  int16_t* rowbuf[MAXD];
  int16_t* colbuf[MAXD];
  double* fibb[MAXD];
  double* coreb[MAXD];
  double* ahb[MAXD];
  int ccap[MAXD];
  for (int b = 1; b < d; ++b) {
    ALLOC(rowbuf[b], int16_t, (int64_t)maxr * MAXD, ar);
    ALLOC(colbuf[b], int16_t, (int64_t)maxr * MAXD, ar);
    ALLOC(ahb[b], double, (int64_t)maxr * maxr, ar);
  }
  for (int k = 0; k < d; ++k) {
    const int acap = k == 0 ? 1 : maxr;
    ccap[k] = k == d - 1 ? 1 : maxr;
    ALLOC(fibb[k], double, (int64_t)acap * spec.n[k] * ccap[k], ar);
    ALLOC(coreb[k], double, (int64_t)acap * spec.n[k] * ccap[k], ar);
  }
  if (c.leader()) {
    for (int b = 1; b < d; ++b) {
      s.rows[b] = rowbuf[b];
      s.cols[b] = colbuf[b];
      s.ahat[b] = ahb[b];
      s.rank[b] = 1;
      for (int j = 0; j < b; ++j) rowbuf[b][j] = (int16_t)pivot[j];
      for (int j = 0; j < d - b; ++j) colbuf[b][j] = (int16_t)pivot[b + j];
    }
    for (int k = 0; k < d; ++k) {
      s.fib[k] = fibb[k];
      s.core[k] = coreb[k];
      s.ccap[k] = ccap[k];
    }
  }
  c.sync();
  for (int k = 0; k < d; ++k) CK(x_fill_fib(c, ar, C, spec, s, k, 0, x_left(s, k), 0, x_right(s, k), sm));
  for (int b = 1; b < d; ++b) CK(x_fill_ahat(c, ar, C, spec, s, b, 0, 1, 0, 1, sm));
  for (int k = 0; k < d; ++k) CK(x_solve_core(c, ar, s, k, sm));

  // total grid points for the fresh-probe budget (may exceed int64: saturate)
  int64_t prod = 1;
  bool huge = false;
  for (int k = 0; k < d; ++k) {
    if (prod > ((int64_t)1 << 40)) huge = true;
    prod *= spec.n[k];
  }
  const int64_t fresh = huge ? X_FRESH : lmin(X_FRESH, lmax(4 * d, prod / 64));

  // best interpolant storage
  TT best;
  bool have_best = false;
  {
    int rcap[MAXD + 1];
    rcap[0] = 1; rcap[d] = 1;
    for (int b = 1; b < d; ++b) rcap[b] = maxr;
    CK(tt_alloc(ar, best, d, spec.n, rcap));
  }
  double best_err = INFINITY;
  int sweeps = 0, clean = 0;
  bool converged = false;
  double oerr[X_INJECT];
  int32_t ocell[X_INJECT * MAXD];
  Cand* cand;
  ALLOC(cand, Cand, X_CAND * X_CAND + 1, ar);
  int32_t* fp;
  ALLOC(fp, int32_t, (int64_t)X_FRESH * d, ar);
  double* fv;
  ALLOC(fv, double, X_FRESH, ar);
  double* oerr_s;
  int32_t* ocell_s;
  ALLOC(oerr_s, double, X_INJECT, ar);
  ALLOC(ocell_s, int32_t, X_INJECT * d, ar);

  for (int sw = 0; sw < cfg.max_sweeps; ++sw) {
    ++sweeps;
    double swe = 0.0;
    bool grew = false, full = true;
    for (int b = 1; b < d; ++b) {
      const int r = s.rank[b];
      const int lim = x_limit(s, b, maxr);
      if (r >= lim) continue;
      full = false;
      int ncand = 0;
      double seen = 0.0;
      CK(x_hunt(c, ar, C, spec, s, b, sh, rws, cand, &ncand, &seen, sm));
      swe = fmax(swe, seen);
      const double thr = cfg.tol * fmax(C->max_abs, X_TINY);
      const int bcap = imin(X_BATCH, imin(imax(1, r / 2), lim - r));
      int m = 0;
      if (c.leader()) {
        for (int q = 0; q < ncand; ++q) {
          if (cand[q].err <= thr || m >= bcap) break;
          int16_t rt[MAXD], ct[MAXD];
          x_split(s, b, cand[q].row, cand[q].col, rt, ct);
          if (tuple_in(s.rows[b], r + m, rt, b)) continue;
          if (tuple_in(s.cols[b], r + m, ct, d - b)) continue;
          int16_t* dr = s.rows[b] + (r + m) * MAXD;
          int16_t* dc = s.cols[b] + (r + m) * MAXD;
          for (int j = 0; j < b; ++j) dr[j] = rt[j];
          for (int j = 0; j < d - b; ++j) dc[j] = ct[j];
          ++m;
        }
      }
      m = (int)bcast_i(c, m);
      if (m > 0) {
        CK(x_accept(c, ar, C, spec, s, b, m, sm));
        grew = true;
      }
    }
    // fresh uniform probes
    warp_integers(c, &sh->rng, rws.jt, spec.n, d, fresh, fp, rws.draws);
    c.sync();
    CK(cache_eval(c, ar, C, spec, fp, fresh, fv, sm));
    double thr = cfg.tol * fmax(C->max_abs, X_TINY);
    size_t mk = ar.mark();
    TT now;
    CK(x_snapshot(c, ar, s, now));
    int nof = 0;
    CK(x_check(c, ar, C, sh, rws, now, X_SAMPLE, X_INJECT, oerr_s, ocell_s, &nof, sm));
    for (int q = 0; q < nof; ++q) { oerr[q] = oerr_s[q]; for (int j = 0; j < d; ++j) ocell[q * d + j] = ocell_s[q * d + j]; }
    c.sync();
    swe = fmax(swe, oerr[0]);
    if (swe < best_err) {
      best_err = swe;
      have_best = true;
      for (int k = 0; k <= d; ++k) best.r[k] = now.r[k];
      for (int k = 0; k < d; ++k) par_copy(c, best.c[k], now.c[k], now.size(k));
      c.sync();
    }
    ar.release(mk);
    if (oerr[0] > thr) CK(x_inject(c, ar, C, spec, s, sh, oerr, ocell, nof, thr, maxr, &grew, sm));
    if (full) {
      size_t mk2 = ar.mark();
      TT t2;
      CK(x_snapshot(c, ar, s, t2));
      CK(x_check(c, ar, C, sh, rws, t2, X_GATE, 1, oerr_s, ocell_s, &nof, sm));
      converged = oerr_s[0] <= thr;
      ar.release(mk2);
      break;
    }
    if (swe <= thr) {
      ++clean;
      if (clean >= 2) {
        size_t mk2 = ar.mark();
        TT t2;
        CK(x_snapshot(c, ar, s, t2));
        CK(x_check(c, ar, C, sh, rws, t2, X_GATE, X_INJECT, oerr_s, ocell_s, &nof, sm));
        for (int q = 0; q < nof; ++q) { oerr[q] = oerr_s[q]; for (int j = 0; j < d; ++j) ocell[q * d + j] = ocell_s[q * d + j]; }
        c.sync();
        ar.release(mk2);
        if (oerr[0] <= thr) { converged = true; break; }
        clean = 0;
        CK(x_inject(c, ar, C, spec, s, sh, oerr, ocell, nof, thr, maxr, &grew, sm));
      }
    } else {
      clean = 0;
    }
    if (!grew && clean == 0) break;
  }
  // --- validation
  TT fin;
  CK(x_snapshot(c, ar, s, fin));
  const int nv = cfg.validation_count;
  int32_t* vp;
  double *vref, *vt;
  ALLOC(vp, int32_t, (int64_t)nv * d, ar);
  ALLOC(vref, double, nv, ar);
  ALLOC(vt, double, nv, ar);
  if ((int64_t)nv * d > X_GATE + X_SCAN) return E_ARG;
  warp_integers(c, &sh->rng, rws.jt, spec.n, d, nv, vp, rws.draws);
  c.sync();
  CK(cache_eval(c, ar, C, spec, vp, nv, vref, sm));
  auto validate = [&](const TT& cand_tt, double* res) -> int {
    tt_eval_idx(c, cand_tt, vp, nv, vt, sm);
    double part = 0.0;
    for (int p = c.tid; p < nv; p += c.nt) part = fmax(part, fabs(vref[p] - vt[p]));
    double e1 = block_max(c, part);
    int no = 0;
    CK(x_check(c, ar, C, sh, rws, cand_tt, X_GATE, 1, oerr_s, ocell_s, &no, sm));
    *res = fmax(e1, oerr_s[0]);
    return OK;
  };
  double achieved = 0.0;
  CK(validate(fin, &achieved));
  const TT* chosen = &fin;
  if (have_best && best_err < achieved) {
    double alt = 0.0;
    CK(validate(best, &alt));
    if (alt < achieved) { chosen = &best; achieved = alt; }
  }
  achieved /= fmax(C->max_abs, X_TINY);
  // output (compact copy; caller's arena keeps the cross workspace until released)
  CK(tt_alloc(ar, out, d, chosen->n, chosen->r));
  for (int k = 0; k < d; ++k) par_copy(c, out.c[k], chosen->c[k], chosen->size(k));
  c.sync();
  info->achieved = achieved;
  info->calls = C->calls;
  info->sweeps = sweeps;
  info->converged = converged ? 1 : 0;
  return OK;
}

}  // namespace tg
