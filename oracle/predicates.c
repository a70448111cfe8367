/* CPU ORACLE (test infrastructure only): C restatement of the two magnitude
 * algorithms behind the reference's θ-criterion, compiled with
 * -ffp-contract=off so every operation rounds separately.  The CUDA engine
 * uses the same formulas (paper_1205_4611_b200/csrc/common.cuh); the test
 * tests/test_predicates.py pins these against numpy bit for bit.
 *
 *   radius  = np.hypot(hw, hh)      (reference geometry.py:27-29)  -> glibc hypot
 *   distance= np.abs(ca - cb)       (reference geometry.py:40, 53) -> numpy SIMD cabs
 *   criterion: max + θ·min <= θ·d   (reference geometry.py:41; swapped :54)
 */
#include <math.h>
#include <stdint.h>

static double hyp_kernel(double ax, double ay) {
  double h = sqrt(ax * ax + ay * ay);
  double t1, t2;
  if (h <= 2.0 * ay) {
    double d = h - ay;
    t1 = ax * (2.0 * d - ax);
    t2 = (d - 2.0 * (ax - ay)) * d;
  } else {
    double d = h - ax;
    t1 = 2.0 * d * (ax - 2.0 * ay);
    t2 = (4.0 * d - ay) * ay + d * d;
  }
  return h - (t1 + t2) / (2.0 * h);
}

double orc_hypot(double x, double y) {
  const double SCALE = 0x1p-600, LARGE = 0x1p+511, TINY = 0x1p-511, EPS = 0x1p-54;
  x = fabs(x);
  y = fabs(y);
  double ax = x < y ? y : x, ay = x < y ? x : y;
  if (ax > LARGE) {
    if (ay <= ax * EPS) return ax + ay;
    return hyp_kernel(ax * SCALE, ay * SCALE) / SCALE;
  }
  if (ay < TINY) {
    if (ax >= ay / EPS) return ax + ay;
    return hyp_kernel(ax / SCALE, ay / SCALE) * SCALE;
  }
  if (ay <= ax * EPS) return ax + ay;
  return hyp_kernel(ax, ay);
}

double orc_cabs(double dx, double dy) {
  double ax = fabs(dx), ay = fabs(dy);
  double l = ax < ay ? ay : ax, s = ax < ay ? ax : ay;
  if (l == 0.0) return 0.0;
  double q = s / l;
  return l * sqrt(fma(q, q, 1.0));
}

void orc_hypot_v(const double* x, const double* y, double* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = orc_hypot(x[i], y[i]);
}

void orc_cabs_v(const double* x, const double* y, double* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = orc_cabs(x[i], y[i]);
}
