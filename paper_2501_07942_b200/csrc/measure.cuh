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

// forward substitution with a lower-triangular row-major L (dim m): |L^-1 x|^2
HD double tri_quad(const double* L, int m, int ld, const double* x) {
  double y[MAXD > MAXB ? MAXD : MAXB];
  double q = 0.0;
  for (int i = 0; i < m; ++i) {
    double s = x[i];
    for (int j = 0; j < i; ++j) s -= L[i * ld + j] * y[j];
    y[i] = s / L[i * ld + i];
  }
  for (int i = 0; i < m; ++i) q += y[i] * y[i];
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
    case H_NORM_BEARING_DEG: {
      double acc = 0.0;
      for (int j = 0; j < d; ++j) acc += x[j] * x[j];
      out[0] = sqrt(acc);
      out[1] = atan2(x[1], x[0]) * RAD2DEG;
      break;
    }
    case H_ABS_FIRST:
      out[0] = fabs(x[0]);
      break;
    case H_RANGE_AZ_EL: {
      double acc = 0.0;
      for (int j = 0; j < 3; ++j) acc += x[j] * x[j];
      out[0] = sqrt(acc);
      out[1] = atan2(x[1], x[0]);
      out[2] = atan2(x[2], hypot(x[0], x[1]));
      break;
    }
    case H_CHAIN_QUADRATIC:
      for (int i = 0; i + 1 < d; ++i) out[i] = x[i] * x[i] + x[i + 1] * x[i + 1];
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
