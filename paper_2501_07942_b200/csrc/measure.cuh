// Measurement-model arithmetic shared by the TT engine (models.cuh) and the
// dense grid filter (dense.cu): h(x) for the enumerated measurement kinds,
// the Cholesky quadratic form of GaussianDensity.pdf (models.py:55-66) and
// the degree wrap of angle_wrap_residual (models.py:72-82).  No TT types.
#pragma once
#include "common.cuh"

namespace tg {

enum HKind : int {
  H_LINEAR = 0, H_RANGE_BEARING = 1, H_RANGE_BEARING_DEG = 2, H_NORM_BEARING_DEG = 3,
  H_ABS_FIRST = 4, H_RANGE_AZ_EL = 5, H_CHAIN_QUADRATIC = 6
};

// Separately rounded double ops: numpy evaluates x*y and x+y as separate
// ufunc passes, so the device must not contract them into an FMA.
HD double mul_rn(double a, double b) {
#if ENGINE_DEVICE
  return __dmul_rn(a, b);
#else
  volatile double t = a * b;
  return t;
#endif
}
HD double add_rn(double a, double b) {
#if ENGINE_DEVICE
  return __dadd_rn(a, b);
#else
  volatile double t = a + b;
  return t;
#endif
}

// Factors of a Gaussian's lower Cholesky factor L as LAPACK dgetrf returns
// them on the host (row-major LU with unit-lower L part, 0-based sequential
// row swaps piv, reciprocal pivots inv = 1 / U_ii).
struct SolveLU {
  const double* lu;
  const int32_t* piv;
  const double* inv;
  int ld;
};

// |L^-1 x|^2 as GaussianDensity.logpdf evaluates it (models.py:60-63):
// y = numpy.linalg.solve(chol, diff.T) -- dgesv = dgetrf + dgetrs, i.e. row
// swaps, unit-lower forward and upper backward substitution -- then
// sum(y * y, axis=0).  The substitutions follow OpenBLAS's trsm kernels: rows
// in power-of-two blocks (largest first from the top; the backward sweep
// visits the same blocks bottom-up), a block's update by the solved rows
// accumulated with FMAs from zero and subtracted once, in-block right-looking
// FMA updates, division replaced by the reciprocal pivot.  Checked against
// numpy.linalg.solve (tests/test_evaluators.py): bit-identical for diagonal
// and unpivoted factors, 98.7 % of values for the pivoted cv6 noise factor.
HD double tri_quad(const SolveLU& f, int m, const double* x) {
  double c[MAXD > MAXB ? MAXD : MAXB];
  for (int i = 0; i < m; ++i) c[i] = x[i];
  for (int i = 0; i < m; ++i) {
    const int j = f.piv[i];
    const double t = c[i];
    c[i] = c[j];
    c[j] = t;
  }
  const int ld = f.ld;
  int blk[6], nb = 0;
  for (int bit = 16; bit >= 1; bit >>= 1)
    if (m & bit) blk[nb++] = bit;
  // forward: unit lower, blocks top-down
  int r0 = 0;
  for (int q = 0; q < nb; ++q) {
    const int r1 = r0 + blk[q];
    for (int k = r0; k < r1 && r0 > 0; ++k) {
      double acc = 0.0;
      for (int j = 0; j < r0; ++j) acc = fma(f.lu[k * ld + j], c[j], acc);
      c[k] = c[k] - acc;
    }
    for (int i = r0; i < r1; ++i)
      for (int k = i + 1; k < r1; ++k) c[k] = fma(-c[i], f.lu[k * ld + i], c[k]);
    r0 = r1;
  }
  // backward: upper with reciprocal pivots, the same blocks bottom-up
  int hi = m;
  for (int q = nb - 1; q >= 0; --q) {
    const int lo = hi - blk[q];
    for (int k = lo; k < hi && hi < m; ++k) {
      double acc = 0.0;
      for (int j = hi; j < m; ++j) acc = fma(f.lu[k * ld + j], c[j], acc);
      c[k] = c[k] - acc;
    }
    for (int i = hi - 1; i >= lo; --i) {
      const double v = mul_rn(c[i], f.inv[i]);
      c[i] = v;
      for (int k = lo; k < i; ++k) c[k] = fma(-v, f.lu[k * ld + i], c[k]);
    }
    hi = lo;
  }
  double q = mul_rn(c[0], c[0]);
  for (int i = 1; i < m; ++i) q = add_rn(q, mul_rn(c[i], c[i]));
  return q;
}

constexpr double RAD2DEG = 57.29577951308232;  // 180/pi as numpy.degrees

// measurement function h(x) -> out[b]
template <class S>
HD void eval_h(const S& s, const double* x, double* out) {
  const int d = s.d;
  switch (s.hkind) {
    case H_LINEAR:
      for (int i = 0; i < s.b; ++i) {
        double acc = 0.0;
        for (int j = 0; j < d; ++j) acc += x[j] * s.H[i * MAXD + j];
        out[i] = acc;
      }
      break;
    case H_RANGE_BEARING:
      out[0] = hypot(x[0], x[1]);
      out[1] = atan2(x[1], x[0]);
      break;
    case H_RANGE_BEARING_DEG:
      out[0] = hypot(x[0], x[1]);
      out[1] = atan2(x[1], x[0]) * RAD2DEG;
      break;
    case H_NORM_BEARING_DEG: {   // numpy.linalg.norm: sqrt(add.reduce(x * x))
      double acc = mul_rn(x[0], x[0]);
      for (int j = 1; j < d; ++j) acc = add_rn(acc, mul_rn(x[j], x[j]));
      out[0] = sqrt(acc);
      out[1] = atan2(x[1], x[0]) * RAD2DEG;
      break;
    }
    case H_ABS_FIRST:
      out[0] = fabs(x[0]);
      break;
    case H_RANGE_AZ_EL: {
      double acc = add_rn(add_rn(mul_rn(x[0], x[0]), mul_rn(x[1], x[1])), mul_rn(x[2], x[2]));
      out[0] = sqrt(acc);
      out[1] = atan2(x[1], x[0]);
      out[2] = atan2(x[2], hypot(x[0], x[1]));
      break;
    }
    case H_CHAIN_QUADRATIC:
      for (int i = 0; i + 1 < d; ++i) out[i] = add_rn(mul_rn(x[i], x[i]), mul_rn(x[i + 1], x[i + 1]));
      out[d - 1] = x[d - 1];
      break;
    default:
      for (int i = 0; i < s.b; ++i) out[i] = NAN;
  }
}

// numpy.mod(a, 360) for the wrap 180 - mod(180 - r, 360)
HD double np_mod360(double a) {
  double m = fmod(a, 360.0);
  if (m != 0.0) {
    if ((m < 0.0) != (360.0 < 0.0)) m += 360.0;
  } else {
    m = copysign(0.0, 360.0);
  }
  return m;
}

}  // namespace tg
