// fp64 decision helpers with the reference's tie rules, shared by the exact
// kernel and the event checks of the traversal kernel.
//   * nearest point for e = 1: the 2-D argmin of |c - s|^2 with the first
//     (lowest) label on ties (detect.py:418-419 argsort(kind="stable")[0]);
//     for square QAM it factorises per axis, ties -> lower Gray label.
//   * the e nearest points: stable order by (|c - s|^2, label).
#pragma once
#include "common.cuh"

namespace mpnl {

// (L-1-2i)/norm exactly as the reference computes its points (a division),
// folded at compile time: no DDIV at run time.
__device__ __forceinline__ double level_value(int i, int L, double nrm) {
  (void)nrm;
  constexpr double n2 = 1.4142135623730951, n4 = 3.1622776601683795, n8 = 6.48074069840786;
  // branch-free (a switch compiles to an indirect jump, and the lanes of a warp
  // index different levels): |lv| from the mirrored index, then the sign --
  // the same compile-time quotients, negation is exact
  const bool neg = 2 * i >= L;
  const int k = neg ? L - 1 - i : i;
  double v;
  if (L == 2) {
    v = 1.0 / n2;
  } else if (L == 4) {
    v = k == 0 ? 3.0 / n4 : 1.0 / n4;
  } else {
    v = k == 0 ? 7.0 / n8 : (k == 1 ? 5.0 / n8 : (k == 2 ? 3.0 / n8 : 1.0 / n8));
  }
  return neg ? -v : v;
}

// level_value for a RUN-TIME index (lanes holding different levels): the same
// constants chosen with predicated selects that ptxas cannot turn back into an
// indirect jump.  (level_value stays foldable for compile-time indices.)
__device__ __forceinline__ double selp_d(double a, double b, bool p) {
  double r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\tselp.f64 %0, %1, %2, q;\n\t}"
      : "=d"(r) : "d"(a), "d"(b), "r"((unsigned)p));
  return r;
}
__device__ __forceinline__ double level_value_rt(int i, int L) {
  constexpr double n2 = 1.4142135623730951, n4 = 3.1622776601683795, n8 = 6.48074069840786;
  const bool neg = 2 * i >= L;
  const int k = neg ? L - 1 - i : i;
  double v;
  if (L == 2) v = 1.0 / n2;
  else if (L == 4) v = selp_d(3.0 / n4, 1.0 / n4, k == 0);
  else v = selp_d(7.0 / n8, selp_d(5.0 / n8, selp_d(3.0 / n8, 1.0 / n8, k == 2), k == 1), k == 0);
  return selp_d(-v, v, neg);
}

static __device__ __noinline__ int nearest_level_f64(double c, int L, double nrm) {
  double bd = 1e300;
  int bg = 1 << 30, bi = 0;
  for (int i = 0; i < L; ++i) {
    const double d = (c - level_value(i, L, nrm)) * (c - level_value(i, L, nrm));
    const int g = gray_code(i);
    if (d < bd || (d == bd && g < bg)) { bd = d; bg = g; bi = i; }
  }
  return bi;
}

// 64-bit mask (bit = i*L + j over level indices) of the e nearest points.
static __device__ __noinline__ unsigned long long nearest_set_f64(double cr, double ci, int L, double nrm,
                                                     int e) {
  const int h = (L == 2) ? 1 : (L == 4 ? 2 : 3);
  const int Q = L * L;
  unsigned long long mask = 0ull;
  for (int q = 0; q < Q; ++q) {
    const int i = q / L, j = q % L;
    const double dr = cr - level_value(i, L, nrm), di = ci - level_value(j, L, nrm);
    const double d = dr * dr + di * di;
    const int lb = (gray_code(i) << h) | gray_code(j);
    int rank = 0;
    for (int q2 = 0; q2 < Q; ++q2) {
      const int i2 = q2 / L, j2 = q2 % L;
      const double er = cr - level_value(i2, L, nrm), ei = ci - level_value(j2, L, nrm);
      const double d2 = er * er + ei * ei;
      const int lb2 = (gray_code(i2) << h) | gray_code(j2);
      rank += (d2 < d) || (d2 == d && lb2 < lb);
    }
    if (rank < e) mask |= 1ull << q;
  }
  return mask;
}

}  // namespace mpnl
