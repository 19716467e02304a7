// Device form of the step's small dense geometry (leader thread, d <= 16):
// moments -> SPD repair (filters.py:275-333), Kalman predict (filters.py:366-375),
// moment-designed predictive grid (grids.py:148-167), corner pull-back and the
// circumscribing filtering grid (filters.py:769-786, grids.py:72-83).
// Used by the persistent multi-step kernel; the object API keeps the numpy
// host geometry (bit-identical to the reference) instead.
#pragma once
#include "common.cuh"
#include "../../include/ttgbf.h"

namespace tg {

// coordinate i of an axis with numpy's two roundings (no FMA contraction)
HD double axis_at(const ttgbf_axis& a, int i) {
#if ENGINE_DEVICE
  return __dadd_rn(a.base, __dmul_rn(a.step, (double)(i - a.off)));
#else
  volatile double t = a.step * (double)(i - a.off);
  return a.base + t;
#endif
}

// smallest eigenvalue of a symmetric d x d matrix (cyclic Jacobi)
HD double sym_min_eig(const double* A, int d) {
  double a[MAXD * MAXD];
  for (int i = 0; i < d * d; ++i) a[i] = A[i];
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (int i = 0; i < d; ++i) {
      diag += a[i * d + i] * a[i * d + i];
      for (int j = i + 1; j < d; ++j) off += a[i * d + j] * a[i * d + j];
    }
    if (off <= 1e-34 * diag || off == 0.0) break;
    for (int p = 0; p < d; ++p)
      for (int q = p + 1; q < d; ++q) {
        const double apq = a[p * d + q];
        if (apq == 0.0) continue;
        const double theta = (a[q * d + q] - a[p * d + p]) / (2.0 * apq);
        const double t = copysign(1.0, theta) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double cs = 1.0 / sqrt(t * t + 1.0), sn = t * cs;
        for (int k = 0; k < d; ++k) {
          const double akp = a[k * d + p], akq = a[k * d + q];
          a[k * d + p] = cs * akp - sn * akq;
          a[k * d + q] = sn * akp + cs * akq;
        }
        for (int k = 0; k < d; ++k) {
          const double apk = a[p * d + k], aqk = a[q * d + k];
          a[p * d + k] = cs * apk - sn * aqk;
          a[q * d + k] = sn * apk + cs * aqk;
        }
      }
  }
  double lo = a[0];
  for (int i = 1; i < d; ++i) lo = fmin(lo, a[i * d + i]);
  return lo;
}

struct GeomOut {
  double mean[MAXD];
  double cov[MAXD * MAXD];      // d x d, ld d
  double pmean[MAXD];
  double pcov[MAXD * MAXD];
  int spd_fixed;
};

// Raw moments (device dots) -> filtering moments; returns false if the mass
// is non-positive / non-finite (DegenerateDensityError).
HD bool geom_moments(const double* raw, int d, double dv, GeomOut* g) {
  const double mass = raw[0] * dv;
  if (!isfinite(mass) || mass <= 0.0) return false;
  for (int i = 0; i < d; ++i) g->mean[i] = raw[1 + i] * dv / mass;
  double sec[MAXD * MAXD];
  int q = 1 + d;
  for (int i = 0; i < d; ++i)
    for (int j = i; j < d; ++j) {
      const double v = raw[q++] * dv / mass;
      sec[i * d + j] = v;
      sec[j * d + i] = v;
    }
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) g->cov[i * d + j] = sec[i * d + j] - g->mean[i] * g->mean[j];
  double sym[MAXD * MAXD];
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) sym[i * d + j] = 0.5 * (g->cov[i * d + j] + g->cov[j * d + i]);
  for (int i = 0; i < d * d; ++i) g->cov[i] = sym[i];
  const double lo = sym_min_eig(sym, d);
  g->spd_fixed = 0;
  if (!(lo > 0.0)) {
    double tr = 0.0;
    for (int i = 0; i < d; ++i) tr += g->cov[i * d + i];
    const double scale = fmax(tr / d, 1.0);
    const double shift = 1e-9 * scale - fmin(lo, 0.0);
    for (int i = 0; i < d; ++i) g->cov[i * d + i] += shift;
    g->spd_fixed = 1;
  }
  return true;
}

// Kalman predict + grid redesign.  F, Q, Finv row-major with ld MAXD.
// Returns false when a predicted variance is not positive (ValueError).
HD bool geom_redesign(GeomOut* g, int d, const double* F, const double* Q, const double* Finv, int n,
                      double sigma_mult, ttgbf_axis* filt, ttgbf_axis* pred) {
  for (int i = 0; i < d; ++i) {
    double acc = 0.0;
    for (int j = 0; j < d; ++j) acc += g->mean[j] * F[i * MAXD + j];
    g->pmean[i] = acc;
  }
  double FC[MAXD * MAXD];
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) {
      double acc = 0.0;
      for (int k = 0; k < d; ++k) acc += F[i * MAXD + k] * g->cov[k * d + j];
      FC[i * d + j] = acc;
    }
  double P[MAXD * MAXD];
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) {
      double acc = 0.0;
      for (int k = 0; k < d; ++k) acc += FC[i * d + k] * F[j * MAXD + k];
      P[i * d + j] = acc + Q[i * MAXD + j];
    }
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) g->pcov[i * d + j] = 0.5 * (P[i * d + j] + P[j * d + i]);
  // predictive grid: mean +- sigma_mult * sqrt(var), odd n, centre on the mean
  const int off = (n - 1) / 2;
  for (int i = 0; i < d; ++i) {
    const double v = g->pcov[i * d + i];
    if (!(v > 0.0)) return false;
    const double half = sigma_mult * sqrt(v);
    pred[i].base = g->pmean[i];
    pred[i].step = 2.0 * half / (double)(n - 1);
    pred[i].off = off;
    pred[i].n = n;
  }
  // corners of the predictive grid pulled back through F^-1
  double lo[MAXD], hi[MAXD];
  double c0[MAXD], c1[MAXD];
  for (int j = 0; j < d; ++j) {
    c0[j] = axis_at(pred[j], 0);
    c1[j] = axis_at(pred[j], n - 1);
  }
  for (int i = 0; i < d; ++i) { lo[i] = INFINITY; hi[i] = -INFINITY; }
  const int64_t ncorner = (int64_t)1 << d;
  for (int64_t cm = 0; cm < ncorner; ++cm) {
    double x[MAXD];
    for (int j = 0; j < d; ++j) x[j] = ((cm >> (d - 1 - j)) & 1) ? c1[j] : c0[j];
    for (int i = 0; i < d; ++i) {
      double acc = 0.0;
      for (int j = 0; j < d; ++j) acc += x[j] * Finv[i * MAXD + j];
      lo[i] = fmin(lo[i], acc);
      hi[i] = fmax(hi[i], acc);
    }
  }
  for (int i = 0; i < d; ++i) {
    if (!(hi[i] > lo[i])) return false;
    filt[i].base = lo[i];
    filt[i].step = (hi[i] - lo[i]) / (double)(n - 1);
    filt[i].off = 0;
    filt[i].n = n;
  }
  return true;
}

}  // namespace tg
