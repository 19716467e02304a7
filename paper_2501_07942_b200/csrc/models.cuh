// Black-box evaluators of the TT-FFT step (device forms of the reference's
// Python callables):
//   EV_GAUSS      initial prior pdf on the grid           filters.py:502-505
//   EV_LIKELIHOOD p(z | x) with angle wrap                 models.py:72-82,146-153
//   EV_KERNEL     N(disp F^T; 0, Q) * cell volume          filters.py:682-706
//   EV_REALIGN    conv TT at F^{-1} y (multilinear)        filters.py:969-974
//   EV_TRANSITION N(x_new - F x_old; 0, Q) * cell volume(old) over the
//                 2d modes (new grid, old grid)           filters.py:580-588, 653-679
// Gaussian densities follow models.py:30-69: value = exp(log_norm - |L^-1 r|^2/2)
// with L the lower Cholesky factor, solved as numpy.linalg.solve does it
// (tri_quad in measure.cuh, from the dgetrf factors computed on the host).
#pragma once
#include "common.cuh"
#include "tt.cuh"
#include "measure.cuh"

namespace tg {

enum EvalKind : int { EV_GAUSS = 0, EV_LIKELIHOOD = 1, EV_KERNEL = 2, EV_REALIGN = 3, EV_TRANSITION = 4 };


struct EvalSpec {
  int kind;
  int d;
  int n[MAXD];
  const double* axes[MAXD];   // coordinates of the black box's grid
  // Gaussian (prior, or process noise for the kernel): dim == d
  double LU[MAXD * MAXD];     // dgetrf factors of the lower Cholesky factor, row-major
  int32_t piv[MAXD];
  double inv[MAXD];
  double log_norm;
  double mean[MAXD];
  // likelihood
  int hkind;
  int b;
  int nang;
  int ang[MAXB];
  double z[MAXB];
  double LUr[MAXB * MAXB];
  int32_t pivr[MAXB];
  double invr[MAXB];
  double log_norm_r;
  double H[MAXB * MAXD];
  // kernel
  double F[MAXD * MAXD];
  double steps[MAXD];
  double cellvol;
  // transition (Algorithm 2): modes [0, dhalf) new grid, [dhalf, 2 dhalf) old grid
  int dhalf;
  // realign
  double Finv[MAXD * MAXD];
  TT conv;
  AxisGeom geo[MAXD];
};

// value at one integer multi-index (not used for EV_REALIGN)
HD double eval_point(const EvalSpec& s, const int32_t* idx) {
  double x[MAXD];
  const int d = s.d;
  switch (s.kind) {
    case EV_GAUSS: {
      for (int k = 0; k < d; ++k) x[k] = s.axes[k][idx[k]] - s.mean[k];
      return exp(s.log_norm - 0.5 * tri_quad(SolveLU{s.LU, s.piv, s.inv, MAXD}, d, x));
    }
    case EV_LIKELIHOOD: {
      for (int k = 0; k < d; ++k) x[k] = s.axes[k][idx[k]];
      double hz[MAXB];
      eval_h(s, x, hz);
      for (int i = 0; i < s.b; ++i) hz[i] = hz[i] - s.z[i];
      for (int t = 0; t < s.nang; ++t) {
        const int a = s.ang[t];
        hz[a] = 180.0 - np_mod360(180.0 - hz[a]);
      }
      return exp(s.log_norm_r - 0.5 * tri_quad(SolveLU{s.LUr, s.pivr, s.invr, MAXB}, s.b, hz));
    }
    case EV_KERNEL: {
      double disp[MAXD], q[MAXD];
      for (int k = 0; k < d; ++k) {
        const int half = (s.n[k] - 1) / 2;
        const int sg = idx[k] <= half ? idx[k] : idx[k] - s.n[k];
        disp[k] = (double)sg * s.steps[k];
      }
      for (int i = 0; i < d; ++i) {
        double acc = 0.0;
        for (int j = 0; j < d; ++j) acc += disp[j] * s.F[i * MAXD + j];
        q[i] = acc;
      }
      return exp(s.log_norm - 0.5 * tri_quad(SolveLU{s.LU, s.piv, s.inv, MAXD}, d, q)) * s.cellvol;
    }
    case EV_TRANSITION: {
      const int h = s.dhalf;
      double xo[MAXD], diff[MAXD];
      for (int k = 0; k < h; ++k) xo[k] = s.axes[h + k][idx[h + k]];
      for (int i = 0; i < h; ++i) {   // x_new - (x_old @ F^T)
        double acc = 0.0;
        for (int j = 0; j < h; ++j) acc += xo[j] * s.F[i * MAXD + j];
        diff[i] = s.axes[i][idx[i]] - acc;
      }
      return exp(s.log_norm - 0.5 * tri_quad(SolveLU{s.LU, s.piv, s.inv, MAXD}, h, diff)) * s.cellvol;
    }
    default:
      return NAN;
  }
}

// realign point coordinate k for multi-index idx: (F^{-1} y)_k, y = pred grid node
HD double realign_coord(const EvalSpec& s, const int32_t* idx, int k) {
  double acc = 0.0;
  for (int j = 0; j < s.d; ++j) acc += s.axes[j][idx[j]] * s.Finv[k * MAXD + j];
  return acc;
}

}  // namespace tg
