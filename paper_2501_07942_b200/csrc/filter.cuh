// Filter stages of Algorithm 3 (filters.py:937-985), one CTA per filter.
//
//   stage_prior    initial_pmd_tt            filters.py:497-513
//   stage_measure  measurement_update (TT) + raw moments
//                                            filters.py:521-563, 287-333
//   stage_time     grid_redesign interp+finalize, kernel cross, FFT conv,
//                  realign cross, finalize   filters.py:799-824, 959-985
// The tiny host-side geometry between the two (SPD repair, Kalman predict,
// grid design, corner pull-back) runs in numpy on the host, exactly as the
// reference computes it.
#pragma once
#include "common.cuh"
#include "tt.cuh"
#include "models.cuh"
#include "cross.cuh"
#include "geom.cuh"
#include "../../include/ttgbf.h"

namespace tg {

constexpr double MASS_FLOOR = 1e-300;   // filters.py:100


HD void log_ranks(ttgbf_diag* dg, int slot, const TT& t) {
  for (int k = 0; k <= TTGBF_MAXD; ++k) dg->ranks[slot][k] = k <= t.d ? t.r[k] : 0;
}

// axis coordinates exactly as numpy builds them: base + step * (i - off)
HD double axis_value(const ttgbf_axis& a, int i) {
#if ENGINE_DEVICE
  return __dadd_rn(a.base, __dmul_rn(a.step, (double)(i - a.off)));
#else
  volatile double t = a.step * (double)(i - a.off);
  return a.base + t;
#endif
}

HDN int materialize_axes(const Ctx& c, Arena& ar, int d, const ttgbf_axis* g, double** axes,
                                AxisGeom* geo, double* steps) {
  for (int k = 0; k < d; ++k) {
    ALLOC(axes[k], double, g[k].n, ar);
    for (int i = c.tid; i < g[k].n; i += c.nt) axes[k][i] = axis_value(g[k], i);
  }
  c.sync();
  for (int k = 0; k < d; ++k) {
    const double a0 = axes[k][0], a1 = axes[k][g[k].n - 1];
    geo[k].a0 = a0;
    geo[k].h = (a1 - a0) / (double)(g[k].n - 1);
    geo[k].n = g[k].n;
    steps[k] = geo[k].h;
  }
  return OK;
}

HD double cell_volume(const double* steps, int d) {
  double v = 1.0;   // np.prod
  for (int k = 0; k < d; ++k) v *= steps[k];
  return v;
}

// packed TT I/O (include/ttgbf.h): header + cores at data + off[k]
HDN int tt_store(const Ctx& c, const TT& t, ttgbf_tt* hdr, double* data, int64_t cap) {
  int64_t need = 0;
  for (int k = 0; k < t.d; ++k) need += t.size(k);
  if (need > cap) return E_STATE_CAP;
  int64_t off = 0;
  for (int k = 0; k < t.d; ++k) {
    par_copy(c, data + off, t.c[k], t.size(k));
    off += t.size(k);
  }
  if (c.leader()) {
    hdr->d = t.d;
    off = 0;
    for (int k = 0; k < t.d; ++k) { hdr->n[k] = t.n[k]; hdr->off[k] = off; off += t.size(k); }
    for (int k = 0; k <= t.d; ++k) hdr->r[k] = t.r[k];
  }
  c.sync();
  return OK;
}

HD TT tt_view(const ttgbf_tt* hdr, double* data) {
  TT t;
  t.d = hdr->d;
  for (int k = 0; k < t.d; ++k) { t.n[k] = hdr->n[k]; t.c[k] = data + hdr->off[k]; }
  for (int k = 0; k <= t.d; ++k) t.r[k] = hdr->r[k];
  return t;
}

// Move a TT that was allocated above `mark` down to `mark` (release the
// temporaries in between).  Destination addresses never exceed the source.
HDN int tt_compact(const Ctx& c, Arena& ar, size_t mark, TT& t) {
  ar.release(mark);
  TT o;
  CK(tt_alloc(ar, o, t.d, t.n, t.r));
  for (int k = 0; k < t.d; ++k) {
    const int64_t sz = o.size(k);
    if (o.c[k] == t.c[k]) continue;
    const int64_t chunk = (int64_t)(t.c[k] - o.c[k]);
    for (int64_t s0 = 0; s0 < sz; s0 += chunk) {
      const int64_t s1 = lmin(sz, s0 + chunk);
      for (int64_t e = s0 + c.tid; e < s1; e += c.nt) o.c[k][e] = t.c[k][e];
      c.sync();
    }
  }
  c.sync();
  t = o;
  return OK;
}

// Exact-rank squeeze of a cross output.  greedy_cross returns cores solved
// from rank-deficient skeleton systems, so about half of its bond directions
// are numerically null (singular values at 1e-16 of the largest; measured on
// the C3 kernel and likelihood crosses).  Dropping them before the Kronecker
// product (FFT convolution, Hadamard) changes the tensor by <= SQUEEZE_TOL
// relative -- rounding noise next to the 1e-8 rounding that follows -- and
// shrinks the product cores ~4x.  `t` must be the last allocation, at `mark`.
#ifndef TTGBF_SQUEEZE
#define TTGBF_SQUEEZE 1
#endif
constexpr double SQUEEZE_TOL = 1e-14;
HDN int tt_squeeze(const Ctx& c, Arena& ar, size_t mark, TT& t, double* sm) {
#if TTGBF_SQUEEZE
  int maxr = 1;
  for (int k = 0; k <= t.d; ++k) maxr = imax(maxr, t.r[k]);
  if (maxr == 1) return OK;
  PROF(c, 30);
  TT r;
  CK(tt_round(c, ar, t, SQUEEZE_TOL, 0, r, sm, true));
  CK(tt_compact(c, ar, mark, r));
  t = r;
#else
  (void)c; (void)ar; (void)mark; (void)t; (void)sm;
#endif
  return OK;
}

HD CrossCfg make_cross_cfg(const ttgbf_cross_cfg& x, const int32_t* seeds, int nseeds) {
  CrossCfg cc;
  cc.tol = x.tol;
  cc.max_rank = x.max_rank;
  cc.max_sweeps = x.max_sweeps;
  cc.validation_count = x.validation_count;
  cc.seeds = seeds;
  cc.nseeds = nseeds;
  cc.rng.s_lo = x.rng_state[0];
  cc.rng.s_hi = x.rng_state[1];
  cc.rng.i_lo = x.rng_state[2];
  cc.rng.i_hi = x.rng_state[3];
  cc.rng.has32 = (uint32_t)x.rng_state[4];
  cc.rng.u32 = (uint32_t)x.rng_state[5];
  cc.cache_cap = x.cache_cap;
  return cc;
}

HD void put_cross(ttgbf_cross_info* o, const CrossInfo& i) {
  o->achieved = i.achieved;
  o->calls = i.calls;
  o->sweeps = i.sweeps;
  o->converged = i.converged;
}

// _finalize_tt (filters.py:454-479): round -> mass -> scale -> negative mass.
// The input TT is a temporary and is consumed (rounded in place).
HDN int finalize_tt(const Ctx& c, Arena& ar, TT& t, const ttgbf_grid_cfg& g, const double* steps,
                           const int32_t* probes, int nprobes, ttgbf_diag* dg, double* sm) {
  const int d = t.d;
  const double dv = cell_volume(steps, d);
  const size_t mk = ar.mark();
  double* ws;
  int wr = 1;
  for (int k = 0; k <= d; ++k) wr = imax(wr, t.r[k]);
  ALLOC(ws, double, 2 * wr + 1024, ar);   // tt_sum: 2 * maxr + blockDim
  TT r;
  if (g.normalize_before_round) {
    const double mass = tt_sum(c, t, ws) * dv;
    if (c.leader()) dg->mass_before_norm = mass;
    if (!isfinite(mass) || mass <= MASS_FLOOR) return E_DEGENERATE;
    tt_scale(c, t, 1.0 / mass);
    CK(tt_round(c, ar, t, g.round_tol, g.round_max_rank, r, sm, true));
  } else {
    CK(tt_round(c, ar, t, g.round_tol, g.round_max_rank, r, sm, true));
    const double mass = tt_sum(c, r, ws) * dv;
    if (c.leader()) dg->mass_before_norm = mass;
    if (!isfinite(mass) || mass <= MASS_FLOOR) return E_DEGENERATE;
    tt_scale(c, r, 1.0 / mass);
  }
  double neg = 0.0;
  CK(tt_negative_mass(c, ar, r, g.densify_guard, probes, nprobes, &neg, sm));
  if (c.leader()) dg->clipped_mass += neg * dv;
  c.sync();
  CK(tt_compact(c, ar, mk, r));
  t = r;
  return OK;
}


// ---------------------------------------------------------------------------
// Evaluator specs
// ---------------------------------------------------------------------------
HDN int spec_alloc(const Ctx& c, Arena& ar, EvalSpec*& sp) {
  ALLOC(sp, EvalSpec, 1, ar);
  (void)c;
  return OK;
}

HD void spec_grid(EvalSpec& s, int d, double* const* axes, const ttgbf_axis* g) {
  s.d = d;
  for (int k = 0; k < d; ++k) { s.n[k] = g[k].n; s.axes[k] = axes[k]; }
}

HD void spec_prior(EvalSpec& s, const ttgbf_gauss& p) {
  s.kind = EV_GAUSS;
  for (int i = 0; i < MAXD * MAXD; ++i) s.LU[i] = p.LU[i];
  for (int i = 0; i < MAXD; ++i) { s.piv[i] = p.piv[i]; s.inv[i] = p.inv[i]; }
  for (int i = 0; i < MAXD; ++i) s.mean[i] = p.mean[i];
  s.log_norm = p.logn;
}

HD void spec_likelihood(EvalSpec& s, const ttgbf_model& m, const double* z) {
  s.kind = EV_LIKELIHOOD;
  s.hkind = m.hkind;
  s.b = m.b;
  s.nang = m.nang;
  for (int i = 0; i < MAXB; ++i) { s.ang[i] = m.ang[i]; s.z[i] = z[i]; }
  for (int i = 0; i < MAXB * MAXB; ++i) s.LUr[i] = m.LUr[i];
  for (int i = 0; i < MAXB; ++i) { s.pivr[i] = m.pivr[i]; s.invr[i] = m.invr[i]; }
  for (int i = 0; i < MAXB * MAXD; ++i) s.H[i] = m.H[i];
  s.log_norm_r = m.logn_r;
}

HD void spec_kernel(EvalSpec& s, const ttgbf_model& m, const double* steps) {
  s.kind = EV_KERNEL;
  for (int i = 0; i < MAXD * MAXD; ++i) { s.F[i] = m.F[i]; s.LU[i] = m.LUq[i]; }
  for (int i = 0; i < MAXD; ++i) { s.piv[i] = m.pivq[i]; s.inv[i] = m.invq[i]; }
  s.log_norm = m.logn_q;
  for (int k = 0; k < s.d; ++k) s.steps[k] = steps[k];
  s.cellvol = cell_volume(steps, s.d);
}

struct StageSmem {
  XShared* xs;   // XShared followed by XState
  double* sm;    // general scratch
};

// ---------------------------------------------------------------------------
// initial_pmd_tt (filters.py:497-513)
// ---------------------------------------------------------------------------
HDN int stage_prior(const Ctx& c, Arena& ar, const ttgbf_model& model, const ttgbf_gauss& prior,
                           const ttgbf_grid_cfg& gcfg, const ttgbf_cross_cfg& xcfg, const ttgbf_filter_io& io,
                           const int32_t* probes, int nprobes, ttgbf_tt* hdr, double* state, int64_t cap,
                           ttgbf_diag* dg, StageSmem S) {
  const int d = model.d;
  double* axes[MAXD];
  AxisGeom geo[MAXD];
  double steps[MAXD];
  CK(materialize_axes(c, ar, d, io.cur, axes, geo, steps));
  EvalSpec* sp;
  CK(spec_alloc(c, ar, sp));
  if (c.leader()) { spec_grid(*sp, d, axes, io.cur); spec_prior(*sp, prior); }
  c.sync();
  const size_t mk = ar.mark();
  TT t;
  CrossInfo ci;
  CK(greedy_cross(c, ar, *sp, make_cross_cfg(xcfg, nullptr, 0), S.xs, t, &ci, S.sm));
  if (c.leader()) put_cross(&dg->cross[0], ci);
  CK(tt_compact(c, ar, mk, t));
  CK(finalize_tt(c, ar, t, gcfg, steps, probes, nprobes, dg, S.sm));
  CK(tt_store(c, t, hdr, state, cap));
  return OK;
}

// Borrow an overflow buffer (spin-acquire): the first class if `need` fits it
// with 50 % headroom, else (or when those are busy) the second, larger class.
// Returns E_WORKSPACE at once when no class can ever hold `need` (instead of
// spinning forever); otherwise *big is the arena over the buffer and *cls /
// *bi identify it for overflow_release.
HD bool overflow_fits(const ttgbf_run_cfg& pool, int64_t need) {
  return (pool.nbig > 0 && need + need / 2 <= pool.big_bytes) || (pool.nbig2 > 0 && need <= pool.big2_bytes) ||
         (pool.nbig2 == 0 && pool.nbig > 0 && need <= pool.big_bytes);
}

HDN int overflow_acquire(const Ctx& c, const ttgbf_run_cfg& pool, int64_t need, ttgbf_diag* dg, Arena* big,
                         int* cls_out, int* bi_out) {
  if (!overflow_fits(pool, need)) return E_WORKSPACE;
  const bool small_ok = pool.nbig > 0 && need + need / 2 <= pool.big_bytes;
  const bool large_ok = pool.nbig2 > 0 && need <= pool.big2_bytes;
  const bool only_small = pool.nbig2 == 0;
  int bi = -1, cls = 0;
  if (c.leader()) {
#if ENGINE_DEVICE
    const int64_t tw = clk();
    while (bi < 0) {
      if (small_ok || only_small)
        for (int i = 0; i < pool.nbig && bi < 0; ++i)
          if (atomicCAS(&pool.big_locks[i], 0, 1) == 0) { bi = i; cls = 0; }
      if (large_ok)
        for (int i = 0; i < pool.nbig2 && bi < 0; ++i)
          if (atomicCAS(&pool.big2_locks[i], 0, 1) == 0) { bi = i; cls = 1; }
      if (bi < 0) __nanosleep(4000);
    }
    dg->big_wait += clk() - tw;
#else
    bi = 0;
    cls = (small_ok || only_small) ? 0 : 1;
#endif
  }
  bi = (int)bcast_i(c, bi);
  cls = (int)bcast_i(c, cls);
  *cls_out = cls;
  *bi_out = bi;
  *big = cls == 0 ? make_ws_arena(pool.big_ws, pool.big_bytes, bi) : make_ws_arena(pool.big2_ws, pool.big2_bytes, bi);
  return OK;
}

HDN void overflow_release(const Ctx& c, const ttgbf_run_cfg& pool, const Arena& big, int cls, int bi,
                          ttgbf_diag* dg) {
  c.sync();
  if (c.leader()) {
    dg->big_used += 1;
    if ((int64_t)big.peak > dg->big_peak) dg->big_peak = (int64_t)big.peak;
#if ENGINE_DEVICE
    __threadfence();
    atomicExch(cls == 0 ? &pool.big_locks[bi] : &pool.big2_locks[bi], 0);
#endif
  }
  c.sync();
}

// ---------------------------------------------------------------------------
// measurement_update (TT branch, filters.py:521-563) + raw moments of the
// filtering density (filters.py:297-322).  Outlier keeps the prior.
// ---------------------------------------------------------------------------
HDN int stage_measure(const Ctx& c, Arena& ar, const ttgbf_model& model, const ttgbf_grid_cfg& gcfg,
                             const ttgbf_cross_cfg& xcfg, const ttgbf_filter_io& io, const int32_t* probes,
                             int nprobes, const int32_t* seeds, int nseeds, ttgbf_tt* hdr, double* state,
                             int64_t cap, ttgbf_diag* dg, StageSmem S, const ttgbf_run_cfg* pool = nullptr) {
  const int d = model.d;
  double* axes[MAXD];
  AxisGeom geo[MAXD];
  double steps[MAXD];
  CK(materialize_axes(c, ar, d, io.cur, axes, geo, steps));
  TT p = tt_view(hdr, state);
  if (c.leader()) log_ranks(dg, 0, p);
  int64_t t0 = clk();
  if (io.has_z) {
    EvalSpec* sp;
    CK(spec_alloc(c, ar, sp));
    if (c.leader()) { spec_grid(*sp, d, axes, io.cur); spec_likelihood(*sp, model, io.z); }
    c.sync();
    const size_t mk = ar.mark();
    TT lik;
    CrossInfo ci;
    CK(greedy_cross(c, ar, *sp, make_cross_cfg(xcfg, seeds, nseeds), S.xs, lik, &ci, S.sm));
    if (c.leader()) { put_cross(&dg->cross[0], ci); log_ranks(dg, 1, lik); }
    CK(tt_compact(c, ar, mk, lik));
    CK(tt_squeeze(c, ar, mk, lik, S.sm));
    if (c.leader()) log_ranks(dg, 8, lik);
    const int64_t t1 = clk();
    if (c.leader()) dg->cycles[0] += t1 - t0;
    t0 = t1;
    const size_t mk2 = ar.mark();
    // Hadamard + finalize on arena A; the state is written only at the end,
    // so a product that outgrows the slot is redone in an overflow buffer
    auto had_fin = [&](Arena& A) -> int {
      const size_t ma = A.mark();
      TT prod;
      CK(tt_hadamard(c, A, p, lik, prod));
      double* ws;
      int wr = 1;
      for (int k = 0; k <= d; ++k) wr = imax(wr, prod.r[k]);
      ALLOC(ws, double, 2 * wr + 1024, A);   // tt_sum: 2 * maxr + blockDim
      const double mass = tt_sum(c, prod, ws) * cell_volume(steps, d);
      if (!isfinite(mass) || mass <= MASS_FLOOR) {
        if (c.leader()) dg->outlier = 1;
        c.sync();
        return OK;
      }
      CK(tt_compact(c, A, ma, prod));
      CK(finalize_tt(c, A, prod, gcfg, steps, probes, nprobes, dg, S.sm));
      CK(tt_store(c, prod, hdr, state, cap));
      return OK;
    };
    const double clipped0 = dg->clipped_mass;
    int hst = had_fin(ar);
    if (hst == E_WORKSPACE && pool && (pool->nbig > 0 || pool->nbig2 > 0)) {
      ar.release(mk2);
      if (c.leader()) dg->clipped_mass = clipped0;
      c.sync();
      int64_t pb = 0;
      for (int k = 0; k < d; ++k) pb += (int64_t)p.r[k] * lik.r[k] * p.n[k] * p.r[k + 1] * lik.r[k + 1] * 8;
      int64_t nd = pb + pb / 16 + ((int64_t)64 << 20);
      if (nd < (int64_t)ar.cap) nd = (int64_t)ar.cap;
      int cls, bi;
      Arena big;
      if (overflow_acquire(c, *pool, nd, dg, &big, &cls, &bi) == OK) {
        hst = had_fin(big);
        overflow_release(c, *pool, big, cls, bi, dg);
      }
    }
    CK(hst);
    p = tt_view(hdr, state);
  }
  if (c.leader()) { log_ranks(dg, 2, p); dg->cycles[1] += clk() - t0; }
  t0 = clk();
  // raw moments of the filtering density
  const double* ax[MAXD];
  for (int k = 0; k < d; ++k) ax[k] = axes[k];
  double* mom;
  ALLOC(mom, double, TTGBF_NMOM, ar);
  CK(tt_moments(c, ar, p, ax, mom));
  const int nmom = 1 + d + d * (d + 1) / 2;
  for (int q = c.tid; q < nmom; q += c.nt) dg->raw_moments[q] = mom[q];
  if (c.leader()) dg->cycles[2] += clk() - t0;
  c.sync();
  return OK;
}

// ---------------------------------------------------------------------------
// time update of tt_fft_pmf_step (filters.py:958-985)
// ---------------------------------------------------------------------------
// FFT convolution + rounding inside a borrowed overflow workspace; the
// rounded TT (small) is copied back into the slot arena at `mark`.
HDN int conv_in_overflow(const Ctx& c, Arena& ar, size_t mark, const TT& ker, const TT& shifted,
                         const ttgbf_grid_cfg& gcfg, const ttgbf_run_cfg& pool, int64_t need, ttgbf_diag* dg,
                         TT& conv, double* sm) {
  int cls, bi;
  Arena big;
  CK(overflow_acquire(c, pool, need, dg, &big, &cls, &bi));
  TT big_conv;
  int st = tt_fft_conv(c, big, ker, shifted, gcfg.round_tol, gcfg.round_max_rank, big_conv, sm);
  if (!st) {
    ar.release(mark);
    st = tt_alloc(ar, conv, big_conv.d, big_conv.n, big_conv.r);
    if (!st) {
      for (int k = 0; k < conv.d; ++k) par_copy(c, conv.c[k], big_conv.c[k], conv.size(k));
    }
  }
  overflow_release(c, pool, big, cls, bi, dg);
  return st;
}

HDN int stage_time(const Ctx& c, Arena& ar, const ttgbf_model& model, const ttgbf_grid_cfg& gcfg,
                          const ttgbf_cross_cfg& xcfg, const ttgbf_filter_io& io, const int32_t* probes,
                          int nprobes, const int32_t* seeds, int nseeds, ttgbf_tt* hdr, double* state,
                          int64_t cap, ttgbf_diag* dg, StageSmem S, const ttgbf_run_cfg* pool = nullptr) {
  const int d = model.d;
  double *ac[MAXD], *af[MAXD], *apd[MAXD];
  AxisGeom gc[MAXD], gf[MAXD], gp[MAXD];
  double sc[MAXD], sf[MAXD], spd[MAXD];
  CK(materialize_axes(c, ar, d, io.cur, ac, gc, sc));
  CK(materialize_axes(c, ar, d, io.filt, af, gf, sf));
  CK(materialize_axes(c, ar, d, io.pred, apd, gp, spd));
  EvalSpec* sp;
  CK(spec_alloc(c, ar, sp));
  // grid_redesign: interpolate the filtering TT onto the new filtering grid
  const size_t m0 = ar.mark();
  TT filt = tt_view(hdr, state);
  TT shifted;
  int64_t t0 = clk();
  {
    const double* na[MAXD];
    for (int k = 0; k < d; ++k) na[k] = af[k];
    CK(tt_interp(c, ar, filt, gc, na, shifted));
  }
  CK(finalize_tt(c, ar, shifted, gcfg, sf, probes, nprobes, dg, S.sm));
  if (c.leader()) { log_ranks(dg, 3, shifted); dg->cycles[3] += clk() - t0; }
  t0 = clk();
  // kernel cross on the filtering grid
  if (c.leader()) { spec_grid(*sp, d, af, io.filt); spec_kernel(*sp, model, sf); }
  c.sync();
  const size_t m1 = ar.mark();
  TT ker;
  CrossInfo ci;
  CK(greedy_cross(c, ar, *sp, make_cross_cfg(xcfg, nullptr, 0), S.xs, ker, &ci, S.sm));
  if (c.leader()) { put_cross(&dg->cross[1], ci); log_ranks(dg, 4, ker); dg->cycles[4] += clk() - t0; }
  t0 = clk();
  CK(tt_compact(c, ar, m1, ker));
  CK(tt_squeeze(c, ar, m1, ker, S.sm));
  if (c.leader()) { log_ranks(dg, 9, ker); dg->cycles[4] += clk() - t0; }
  t0 = clk();
  // FFT convolution + rounding
  TT conv;
  int64_t pbytes = 0;
  for (int k = 0; k < d; ++k)
    pbytes += (int64_t)ker.r[k] * shifted.r[k] * ker.n[k] * ker.r[k + 1] * shifted.r[k + 1] * 8;
  const int64_t need = pbytes + pbytes / 16 + ((int64_t)64 << 20);   // + rounding temporaries
  const bool have_pool = pool && (pool->nbig > 0 || pool->nbig2 > 0);
  int cst = E_WORKSPACE;
  int64_t nd = need;
  if (!have_pool || (int64_t)(ar.cap - ar.off) >= need) {
    // in the slot; if the rounding temporaries outgrow the estimate, the
    // (deterministic) convolution is redone in an overflow buffer
    const size_t mc = ar.mark();
    cst = tt_fft_conv(c, ar, ker, shifted, gcfg.round_tol, gcfg.round_max_rank, conv, S.sm);
    if (cst == OK) {
      CK(tt_compact(c, ar, m0, conv));
    } else {
      if (cst != E_WORKSPACE || !have_pool) return cst;
      ar.release(mc);
      if (nd < (int64_t)ar.cap) nd = (int64_t)ar.cap;
    }
  }
  if (cst != OK) {
    cst = conv_in_overflow(c, ar, m0, ker, shifted, gcfg, *pool, nd, dg, conv, S.sm);
    if (cst == E_WORKSPACE && pool->nbig2 > 0 && pool->big2_bytes > pool->big_bytes && nd + nd / 2 <= pool->big_bytes)
      cst = conv_in_overflow(c, ar, m0, ker, shifted, gcfg, *pool, pool->big_bytes + 1, dg, conv, S.sm);   // large class
    CK(cst);
  }
  if (c.leader()) { log_ranks(dg, 5, conv); dg->cycles[5] += clk() - t0; }
  t0 = clk();
  int maxr = 1;
  for (int k = 0; k <= d; ++k) maxr = imax(maxr, conv.r[k]);
  if (maxr > CHAIN_MAXR) return E_ARG;
  // realign cross on the predictive grid
  if (c.leader()) {
    spec_grid(*sp, d, apd, io.pred);
    sp->kind = EV_REALIGN;
    for (int i = 0; i < MAXD * MAXD; ++i) sp->Finv[i] = model.Finv[i];
    sp->conv = conv;
    for (int k = 0; k < d; ++k) sp->geo[k] = gf[k];
  }
  c.sync();
  const size_t m2 = ar.mark();
  TT rl;
  CK(greedy_cross(c, ar, *sp, make_cross_cfg(xcfg, seeds, nseeds), S.xs, rl, &ci, S.sm));
  if (c.leader()) { put_cross(&dg->cross[2], ci); log_ranks(dg, 6, rl); dg->cycles[6] += clk() - t0; }
  t0 = clk();
  CK(tt_compact(c, ar, m2, rl));
  CK(finalize_tt(c, ar, rl, gcfg, spd, probes, nprobes, dg, S.sm));
  CK(tt_store(c, rl, hdr, state, cap));
  if (c.leader()) { log_ranks(dg, 7, rl); dg->cycles[7] += clk() - t0; }
  return OK;
}


// ---------------------------------------------------------------------------
// Algorithm 2 time update of tt_pmf_step (filters.py:876-885): transition
// cross over the 2d modes (new grid io.pred, old grid io.cur), backward
// contraction with the filtering TT, scale by the old cell volume, finalize
// on the new grid.  The cross info lands in dg->cross[1] ("transition").
// ---------------------------------------------------------------------------
HDN int stage_time_std(const Ctx& c, Arena& ar, const ttgbf_model& model, const ttgbf_grid_cfg& gcfg,
                       const ttgbf_cross_cfg& xcfg, const ttgbf_filter_io& io, const int32_t* probes, int nprobes,
                       ttgbf_tt* hdr, double* state, int64_t cap, ttgbf_diag* dg, StageSmem S) {
  const int d = model.d;
  if (2 * d > MAXD) return E_ARG;
  double *ao[MAXD], *an[MAXD];
  AxisGeom go[MAXD], gn[MAXD];
  double so[MAXD], sn[MAXD];
  CK(materialize_axes(c, ar, d, io.cur, ao, go, so));
  CK(materialize_axes(c, ar, d, io.pred, an, gn, sn));
  EvalSpec* sp;
  CK(spec_alloc(c, ar, sp));
  const double cv_old = cell_volume(so, d);
  if (c.leader()) {
    sp->kind = EV_TRANSITION;
    sp->d = 2 * d;
    sp->dhalf = d;
    for (int k = 0; k < d; ++k) {
      sp->n[k] = io.pred[k].n;
      sp->axes[k] = an[k];
      sp->n[d + k] = io.cur[k].n;
      sp->axes[d + k] = ao[k];
    }
    for (int i = 0; i < MAXD * MAXD; ++i) { sp->F[i] = model.F[i]; sp->LU[i] = model.LUq[i]; }
    for (int i = 0; i < MAXD; ++i) { sp->piv[i] = model.pivq[i]; sp->inv[i] = model.invq[i]; }
    sp->log_norm = model.logn_q;
    sp->cellvol = cv_old;
  }
  c.sync();
  const TT filt = tt_view(hdr, state);
  int64_t t0 = clk();
  const size_t m0 = ar.mark();
  TT tpm;
  CrossInfo ci;
  CK(greedy_cross(c, ar, *sp, make_cross_cfg(xcfg, nullptr, 0), S.xs, tpm, &ci, S.sm));
  if (c.leader()) { put_cross(&dg->cross[1], ci); dg->cycles[4] += clk() - t0; }
  CK(tt_compact(c, ar, m0, tpm));
  t0 = clk();
  const size_t m1 = ar.mark();
  TT raw;
  CK(tt_einsum_tpm(c, ar, tpm, filt, raw, S.sm));
  CK(tt_compact(c, ar, m1, raw));
  tt_scale(c, raw, cv_old);
  CK(finalize_tt(c, ar, raw, gcfg, sn, probes, nprobes, dg, S.sm));
  CK(tt_store(c, raw, hdr, state, cap));
  if (c.leader()) { log_ranks(dg, 7, raw); dg->cycles[5] += clk() - t0; }
  return OK;
}

// ---------------------------------------------------------------------------
// Persistent multi-step run: this filter's loop over rc.steps tt_fft_pmf_step
// calls with device geometry, restarting from the prior after a failure or
// at the end of its trajectory (bench / Monte Carlo driver).
// ---------------------------------------------------------------------------
// one step of the persistent run for this filter; R receives the record
HDN int stage_run_step(const Ctx& c, Arena& ar, const ttgbf_model& model, const ttgbf_gauss& prior,
                       const ttgbf_grid_cfg& gcfg, const ttgbf_cross_cfg& xcfg, const ttgbf_run_cfg& rc,
                       ttgbf_filter_io* io, int32_t* kstep, const double* Z, const int32_t* probes, int nprobes,
                       const int32_t* seeds, int nseeds, ttgbf_tt* hdr, double* state, int64_t cap,
                       ttgbf_diag* dg, ttgbf_step_rec* R, StageSmem S) {
  const int d = model.d, b = model.b;
  const int64_t t_start = clk();
  const size_t mbase = ar.mark();
  GeomOut* go;
  ALLOC(go, GeomOut, 1, ar);
  const size_t m0 = ar.mark();
  if (!io->active) {
    if (c.leader()) {
      for (int k = 0; k < MAXD; ++k) io->cur[k] = rc.prior_grid[k];
      *kstep = 0;
      dg->clipped_mass = 0.0;
    }
    c.sync();
    const int st = stage_prior(c, ar, model, prior, gcfg, xcfg, *io, probes, nprobes, hdr, state, cap, dg, S);
    ar.release(m0);
    if (st) {
      if (c.leader()) { R->status = -1; R->k = -1; R->cycles = clk() - t_start; }
      c.sync();
      ar.release(mbase);
      return OK;
    }
    if (c.leader()) io->active = 1;
    c.sync();
  }
  const int kk = *kstep;
  if (c.leader()) {
    for (int i = 0; i < b; ++i) io->z[i] = Z[(int64_t)kk * b + i];
    io->has_z = 1;
    dg->clipped_mass = 0.0;
    dg->outlier = 0;
    R->k = kk;
    for (int q = 0; q < 3; ++q) dg->cross[q].calls = 0;
    for (int sl = 0; sl < TTGBF_NRANKLOG; ++sl)
      for (int k = 0; k <= TTGBF_MAXD; ++k) dg->ranks[sl][k] = 0;
  }
  c.sync();
  int st = stage_measure(c, ar, model, gcfg, xcfg, *io, probes, nprobes, seeds, nseeds, hdr, state, cap, dg, S, &rc);
  ar.release(m0);
  if (!st) {
    int gst = 0;
    if (c.leader()) {
      double dv = 1.0;
      for (int k = 0; k < d; ++k)
        dv *= (axis_at(io->cur[k], io->cur[k].n - 1) - axis_at(io->cur[k], 0)) / (double)(io->cur[k].n - 1);
      if (!geom_moments(dg->raw_moments, d, dv, go)) {
        gst = E_DEGENERATE;
      } else if (!geom_redesign(go, d, model.F, model.Q, model.Finv, rc.n_per_axis, rc.sigma_mult, io->filt,
                                io->pred)) {
        gst = E_ARG;
      } else {
        for (int i = 0, q = 0; i < d; ++i) {
          R->mean[i] = go->mean[i];
          for (int j = i; j < d; ++j) R->cov[q++] = go->cov[i * d + j];
        }
        R->spd_fixed = go->spd_fixed;
      }
    }
    st = (int)bcast_i(c, gst);
  }
  if (!st) {
    st = stage_time(c, ar, model, gcfg, xcfg, *io, probes, nprobes, seeds, nseeds, hdr, state, cap, dg, S, &rc);
    ar.release(m0);
  }
  if (c.leader()) {
    R->status = st;
    R->outlier = dg->outlier;
    R->mass_before_norm = dg->mass_before_norm;
    R->clipped_mass = dg->clipped_mass;
    for (int q = 0; q < 3; ++q) R->calls[q] = dg->cross[q].calls;
    for (int sl = 0; sl < TTGBF_NRANKLOG; ++sl)
      for (int k = 0; k <= TTGBF_MAXD; ++k) R->ranks[sl][k] = dg->ranks[sl][k];
    R->cycles = clk() - t_start;
    if (st) {
      io->active = 0;
    } else {
      for (int k = 0; k < MAXD; ++k) io->cur[k] = io->pred[k];
      *kstep = kk + 1;
      if (kk + 1 >= rc.kf) io->active = 0;
    }
  }
  c.sync();
  ar.release(mbase);
  return OK;
}

HDN int stage_run(const Ctx& c, Arena& ar, const ttgbf_model& model, const ttgbf_gauss& prior,
                  const ttgbf_grid_cfg& gcfg, const ttgbf_cross_cfg& xcfg, const ttgbf_run_cfg& rc,
                  ttgbf_filter_io* io, int32_t* kstep, const double* Z, const int32_t* probes, int nprobes,
                  const int32_t* seeds, int nseeds, ttgbf_tt* hdr, double* state, int64_t cap, ttgbf_diag* dg,
                  ttgbf_step_rec* rec, StageSmem S) {
  for (int s = 0; s < rc.steps; ++s)
    CK(stage_run_step(c, ar, model, prior, gcfg, xcfg, rc, io, kstep, Z, probes, nprobes, seeds, nseeds, hdr, state,
                      cap, dg, rec + s, S));
  return OK;
}

}  // namespace tg
