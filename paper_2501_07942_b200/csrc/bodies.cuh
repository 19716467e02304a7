// Per-item bodies of the C-ABI entry points.  Each body is what ONE CTA does
// for one filter / one TT item; api.cu wraps them in __global__ kernels
// (blockIdx.x = item), hostsim.cpp (test-only) loops over items.
#pragma once
#include "filter.cuh"

namespace tg {

constexpr int SMEM_RED = 64 + 320;        // reductions + block_reduce_vec partials (8 warps x 33)
constexpr int SMEM_XBLK = 128;            // XShared + XState (doubles)
constexpr int SMEM_SCRATCH = SMEM_SCRATCH_DOUBLES;   // gemm tiles / QR / chain evaluation
constexpr int SMEM_DOUBLES = SMEM_RED + SMEM_XBLK + SMEM_SCRATCH;
constexpr int BLOCK_THREADS = 256;
static_assert(BLOCK_THREADS == 32 * CTA_WARPS, "CHAIN_MAXR assumes CTA_WARPS warps per CTA");
// resident CTAs per SM the kernels are built for (registers <= 64K / (256 *
// this), SMEM_DOUBLES * 8 + 1 KiB <= 228 KiB / this)
#ifndef TTGBF_CTAS_PER_SM
#define TTGBF_CTAS_PER_SM 2
#endif
constexpr int CTAS_PER_SM = TTGBF_CTAS_PER_SM;
static_assert((SMEM_DOUBLES * 8 + 1024) * CTAS_PER_SM <= 228 * 1024, "SMEM too large for CTAS_PER_SM");

static_assert(sizeof(XShared) + sizeof(XState) <= SMEM_XBLK * sizeof(double), "xblk too small");

HD Ctx make_ctx(double* smem, int tid, int nt) {
  Ctx c;
  c.tid = tid;
  c.nt = nt;
  c.red = smem;
  c.ired = reinterpret_cast<int*>(smem + 32);
  c.prof = nullptr;
  return c;
}
HD StageSmem make_stage_smem(double* smem) {
  StageSmem s;
  s.xs = reinterpret_cast<XShared*>(smem + SMEM_RED);
  s.sm = smem + SMEM_RED + SMEM_XBLK;
  return s;
}
HD Arena make_arena(void* ws, int64_t ws_bytes, int item) {
  Arena a;
  a.base = reinterpret_cast<char*>(ws) + (int64_t)item * ws_bytes;
  a.cap = (size_t)ws_bytes;
  a.off = 0;
  a.peak = 0;
  return a;
}

HDN int body_round(const Ctx& c, Arena& ar, const ttgbf_tt* ih, const double* in, double tol, int cap,
                          ttgbf_tt* oh, double* out, int64_t ocap, double* sm) {
  TT t = tt_view(ih, const_cast<double*>(in));
  TT r;
  CK(tt_round(c, ar, t, tol, cap, r, sm));
  return tt_store(c, r, oh, out, ocap);
}

HDN int body_hadamard(const Ctx& c, Arena& ar, const ttgbf_tt* ah, const double* a, const ttgbf_tt* bh,
                             const double* b, ttgbf_tt* oh, double* out, int64_t ocap) {
  TT ta = tt_view(ah, const_cast<double*>(a)), tb = tt_view(bh, const_cast<double*>(b));
  if (ta.d != tb.d) return E_ARG;
  for (int k = 0; k < ta.d; ++k)
    if (ta.n[k] != tb.n[k]) return E_ARG;
  TT r;
  CK(tt_hadamard(c, ar, ta, tb, r));
  return tt_store(c, r, oh, out, ocap);
}

HDN int body_fftconv(const Ctx& c, Arena& ar, const ttgbf_tt* kh, const double* k, const ttgbf_tt* wh,
                            const double* w, double tol, int cap, ttgbf_tt* oh, double* out, int64_t ocap,
                            double* sm) {
  TT tk = tt_view(kh, const_cast<double*>(k)), tw = tt_view(wh, const_cast<double*>(w));
  if (tk.d != tw.d) return E_ARG;
  for (int q = 0; q < tk.d; ++q)
    if (tk.n[q] != tw.n[q] || (tk.n[q] % 2) == 0 || tk.n[q] > 159) return E_ARG;
  TT r;
  CK(tt_fft_conv(c, ar, tk, tw, tol, cap, r, sm));
  return tt_store(c, r, oh, out, ocap);
}

HDN int body_interp(const Ctx& c, Arena& ar, const ttgbf_tt* ih, const double* in, const ttgbf_axis* oa,
                           const ttgbf_axis* na, ttgbf_tt* oh, double* out, int64_t ocap) {
  TT t = tt_view(ih, const_cast<double*>(in));
  double *ao[MAXD], *an[MAXD];
  AxisGeom go[MAXD], gn[MAXD];
  double so[MAXD], sn[MAXD];
  CK(materialize_axes(c, ar, t.d, oa, ao, go, so));
  CK(materialize_axes(c, ar, t.d, na, an, gn, sn));
  const double* nap[MAXD];
  for (int k = 0; k < t.d; ++k) nap[k] = an[k];
  TT r;
  CK(tt_interp(c, ar, t, go, nap, r));
  return tt_store(c, r, oh, out, ocap);
}

HDN int body_eval_many(const Ctx& c, Arena& ar, const ttgbf_tt* h, const double* data, const int32_t* idx,
                              int64_t K, double* out, double* sm) {
  TT t = tt_view(h, const_cast<double*>(data));
  int maxr = 1;
  for (int k = 0; k <= t.d; ++k) maxr = imax(maxr, t.r[k]);
  if (maxr > CHAIN_MAXR) return E_ARG;
  IndexSlice is{&t, idx, 0};
  return tt_eval_bucketed(c, ar, t, K, is, out, sm);
}


HDN int body_eval_points(const Ctx& c, Arena& ar, const ttgbf_tt* h, const double* data,
                                const ttgbf_axis* axes, const double* pts, int64_t K, double* out, double* sm) {
  TT t = tt_view(h, const_cast<double*>(data));
  int maxr = 1;
  for (int k = 0; k <= t.d; ++k) maxr = imax(maxr, t.r[k]);
  if (maxr > CHAIN_MAXR) return E_ARG;
  double* ax[MAXD];
  AxisGeom geo[MAXD];
  double st[MAXD];
  CK(materialize_axes(c, ar, t.d, axes, ax, geo, st));
  PointSlice<PtsFn> ps{&t, geo, PtsFn{pts, t.d}, 0, 0.0};
  return tt_eval_bucketed(c, ar, t, K, ps, out, sm);
}

HDN int body_moments(const Ctx& c, Arena& ar, const ttgbf_tt* h, const double* data, const ttgbf_axis* axes,
                            double* out) {
  TT t = tt_view(h, const_cast<double*>(data));
  double* ax[MAXD];
  AxisGeom geo[MAXD];
  double st[MAXD];
  CK(materialize_axes(c, ar, t.d, axes, ax, geo, st));
  const double* axc[MAXD];
  for (int k = 0; k < t.d; ++k) axc[k] = ax[k];
  return tt_moments(c, ar, t, axc, out);
}

HDN int body_negmass(const Ctx& c, Arena& ar, const ttgbf_tt* h, const double* data, const ttgbf_axis* axes,
                            int64_t guard, const int32_t* probes, int nprobes, double* out, double* sm) {
  TT t = tt_view(h, const_cast<double*>(data));
  double* ax[MAXD];
  AxisGeom geo[MAXD];
  double st[MAXD];
  CK(materialize_axes(c, ar, t.d, axes, ax, geo, st));
  double neg = 0.0;
  CK(tt_negative_mass(c, ar, t, guard, probes, nprobes, &neg, sm));
  if (c.leader()) *out = neg * cell_volume(st, t.d);
  c.sync();
  return OK;
}

HDN int body_cross(const Ctx& c, Arena& ar, int kind, const ttgbf_model& model, const ttgbf_gauss* prior,
                          const ttgbf_cross_cfg& xcfg, const ttgbf_filter_io& io, const int32_t* seeds, int nseeds,
                          ttgbf_tt* oh, double* out, int64_t ocap, ttgbf_diag* dg, StageSmem S) {
  const int d = model.d;
  double* axes[MAXD];
  AxisGeom geo[MAXD];
  double steps[MAXD];
  CK(materialize_axes(c, ar, d, io.cur, axes, geo, steps));
  EvalSpec* sp;
  CK(spec_alloc(c, ar, sp));
  if (c.leader()) {
    spec_grid(*sp, d, axes, io.cur);
    if (kind == 0) spec_prior(*sp, *prior);
    else if (kind == 1) spec_likelihood(*sp, model, io.z);
    else spec_kernel(*sp, model, steps);
  }
  c.sync();
  TT t;
  CrossInfo ci;
  CK(greedy_cross(c, ar, *sp, make_cross_cfg(xcfg, seeds, nseeds), S.xs, t, &ci, S.sm));
  if (c.leader()) put_cross(&dg->cross[0], ci);
  c.sync();
  return tt_store(c, t, oh, out, ocap);
}

// Black-box evaluators at integer indices (no cross, no cache): the values
// greedy_cross sees.  kind TTGBF_BB_GAUSS / _LIKELIHOOD / _KERNEL on io.cur,
// TTGBF_BB_REALIGN: the TT (th, data) on grid io.filt at F^-1 y, y the io.pred
// node of each index (filters.py:969-979).
HDN int body_eval_bb(const Ctx& c, Arena& ar, int kind, const ttgbf_model& model, const ttgbf_gauss* prior,
                     const ttgbf_filter_io& io, const ttgbf_tt* th, const double* data, const int32_t* idx,
                     int64_t K, double* out, double* sm) {
  const int d = model.d;
  if (d < 1 || d > MAXD || K < 0) return E_ARG;
  double* axes[MAXD];
  AxisGeom geo[MAXD];
  double steps[MAXD];
  CK(materialize_axes(c, ar, d, kind == TTGBF_BB_REALIGN ? io.pred : io.cur, axes, geo, steps));
  EvalSpec* sp;
  CK(spec_alloc(c, ar, sp));
  if (kind == TTGBF_BB_REALIGN) {
    if (th == nullptr || th->d != d) return E_ARG;
    const TT t = tt_view(th, const_cast<double*>(data));
    int maxr = 1;
    for (int k = 0; k <= d; ++k) maxr = imax(maxr, t.r[k]);
    if (maxr > CHAIN_MAXR) return E_ARG;
    double* fax[MAXD];
    AxisGeom fgeo[MAXD];
    double fsteps[MAXD];
    CK(materialize_axes(c, ar, d, io.filt, fax, fgeo, fsteps));
    if (c.leader()) {
      spec_grid(*sp, d, axes, io.pred);
      sp->kind = EV_REALIGN;
      for (int i = 0; i < MAXD * MAXD; ++i) sp->Finv[i] = model.Finv[i];
      sp->conv = t;
      for (int k = 0; k < d; ++k) sp->geo[k] = fgeo[k];
    }
    c.sync();
    double* coords;
    ALLOC(coords, double, K * d, ar);
    for (int64_t e = c.tid; e < K * d; e += c.nt) coords[e] = realign_coord(*sp, idx + (e / d) * d, (int)(e % d));
    c.sync();
    PointSlice<PtsFn> ps{&sp->conv, sp->geo, PtsFn{coords, d}, 0, 0.0};
    return tt_eval_bucketed(c, ar, sp->conv, K, ps, out, sm);
  }
  if (c.leader()) {
    spec_grid(*sp, d, axes, io.cur);
    if (kind == TTGBF_BB_GAUSS) spec_prior(*sp, *prior);
    else if (kind == TTGBF_BB_LIKELIHOOD) spec_likelihood(*sp, model, io.z);
    else spec_kernel(*sp, model, steps);
  }
  c.sync();
  for (int64_t j = c.tid; j < K; j += c.nt) out[j] = eval_point(*sp, idx + j * d);
  c.sync();
  return OK;
}

}  // namespace tg
