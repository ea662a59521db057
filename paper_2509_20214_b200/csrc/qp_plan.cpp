// Host-only planning helpers of the C ABI (no device work).
//
// qp_optimal_bits: Theorem 1 of the paper, optimal fractional bit allocation with
// ideal Gaussian quantizers, b_l* = max{eta, ln(a_l / n_l) / (2 ln 2) + C} with the C that makes
// the memory budget tight. S(C) = sum_l max{eta, u_l + C} n_l is piecewise linear and
// non-decreasing in C with breakpoints C_l = eta - u_l; the exact C is found by sorting the
// breakpoints and solving the linear piece on which S crosses M (no iteration).
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <numeric>
#include <string>
#include <vector>

#include "qpalette.h"
#include "qp_internal.h"

namespace {
qp_status fail(qp_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  return (qp_status)qp::set_error((int)s, buf);
}
}  // namespace

extern "C" qp_status qp_optimal_bits(const double* a, const double* n, int L, double M, double eta, double* b_out) {
  if (!a || !n || !b_out || L <= 0) return fail(QP_ERR_INVALID_ARG, "qp_optimal_bits: NULL argument or L <= 0");
  double total = 0.0;
  std::vector<double> u(L);
  for (int l = 0; l < L; ++l) {
    if (!(a[l] > 0.0) || !(n[l] > 0.0) || !std::isfinite(a[l]) || !std::isfinite(n[l]))
      return fail(QP_ERR_INVALID_ARG, "qp_optimal_bits: a[%d]=%g, n[%d]=%g must be positive and finite", l, a[l], l,
                      n[l]);
    u[l] = std::log(a[l] / n[l]) / (2.0 * std::log(2.0));
    total += n[l];
  }
  if (!(eta >= 0.0) || !std::isfinite(M))
    return fail(QP_ERR_INVALID_ARG, "qp_optimal_bits: eta=%g must be >= 0 and M finite", eta);
  if (M < eta * total * (1.0 - 1e-12))
    return fail(QP_ERR_CONFIG_MISMATCH, "qp_optimal_bits: budget M=%g below eta * sum(n) = %g (P:172)", M,
                    eta * total);
  // layers leave the floor in order of increasing breakpoint eta - u_l (decreasing u_l)
  std::vector<int> ord(L);
  std::iota(ord.begin(), ord.end(), 0);
  std::sort(ord.begin(), ord.end(), [&](int x, int y) { return u[x] > u[y]; });
  // with the first k layers (in that order) free: S(C) = eta * (total - N_k) + sum_{free} (u_l + C) n_l
  double Nk = 0.0, Uk = 0.0, C = 0.0;
  for (int k = 0; k < L; ++k) {
    const int l = ord[k];
    Nk += n[l];
    Uk += u[l] * n[l];
    C = (M - eta * (total - Nk) - Uk) / Nk;            // solve S(C) = M on this piece
    const double next_bp = k + 1 < L ? eta - u[ord[k + 1]] : INFINITY;
    if (C <= next_bp) break;                            // the next layer stays on the floor
  }
  for (int l = 0; l < L; ++l) b_out[l] = std::max(eta, u[l] + C);
  return QP_OK;
}
