// Offline stage of Polar Express: greedy minimax odd polynomials in fp64.
//
// Paper: arXiv 2505.16932 (/root/reference/PAPER.md, P:<line>).
//   Theorem 1: greedy per-step minimax is optimal; the next
//     interval is [p_t(l_t), 2 - p_t(l_t)] (eq. (newbounds)).
//   Alg. 2 / Listing 1 `optimal_quintic`: degree-5
//     Remez with fixed end points, interior points from the quadratic in x^2.
//   eq. (deg3_solution): closed-form degree-3 optimum.
//   Listing 1 `optimal_composition`: cushion, recentring.
//   Listing 2: safety factor p(x) -> p(x / 1.01).
// Readings R3-R6, R15 are in DESIGN.md.
#include <cmath>
#include <cstddef>

#include "pe.h"

namespace {

constexpr double kPadeThreshold = 1.0 - 5e-6;
constexpr double kRemezTol = 1e-15;
constexpr double kCushion5 = 0.02407327424182761;
constexpr double kCushion3 = 0.039327193224439359;       // R3 (degree-3 analogue)
constexpr int kRemezMaxIters = 50;                       // R6

// p(x) = sum_q c[q] x^(2q+1), Horner in x^2.
double eval_odd(const double* c, int nq, double x) {
  const double y = x * x;
  double h = c[nq - 1];
  for (int q = nq - 2; q >= 0; --q) h = h * y + c[q];
  return x * h;
}

// 4x4 linear solve, Gaussian elimination with partial pivoting.
bool solve4(double A[4][4], double b[4], double x[4]) {
  for (int col = 0; col < 4; ++col) {
    int piv = col;
    for (int r = col + 1; r < 4; ++r)
      if (std::fabs(A[r][col]) > std::fabs(A[piv][col])) piv = r;
    if (A[piv][col] == 0.0) return false;
    if (piv != col) {
      for (int k = 0; k < 4; ++k) { double t = A[col][k]; A[col][k] = A[piv][k]; A[piv][k] = t; }
      double t = b[col]; b[col] = b[piv]; b[piv] = t;
    }
    for (int r = col + 1; r < 4; ++r) {
      const double f = A[r][col] / A[col][col];
      for (int k = col; k < 4; ++k) A[r][k] -= f * A[col][k];
      b[r] -= f * b[col];
    }
  }
  for (int r = 3; r >= 0; --r) {
    double s = b[r];
    for (int k = r + 1; k < 4; ++k) s -= A[r][k] * x[k];
    x[r] = s / A[r][r];
  }
  return true;
}

// Alg. 2: minimax odd quintic for the constant 1 on [l, u].
pe_status quintic(double l, double u, double out[3], bool* pade) {
  *pade = false;
  if (l / u >= kPadeThreshold) {  // Pade branch
    out[0] = (15.0 / 8.0) / u;
    out[1] = (-10.0 / 8.0) / (u * u * u);
    out[2] = (3.0 / 8.0) / (u * u * u * u * u);
    *pade = true;
    return PE_OK;
  }
  double x1 = (3.0 * l + u) / 4.0, x2 = (l + 3.0 * u) / 4.0;
  double E = INFINITY, E_prev = NAN;
  bool first = true;
  double a = 0, b = 0, c = 0;
  for (int it = 0;; ++it) {
    if (!first && std::fabs(E_prev - E) <= kRemezTol) break;  // P:523 / P:876
    if (it >= kRemezMaxIters) return PE_ERR_NO_CONVERGENCE;
    first = false;
    E_prev = E;
    const double pts[4] = {l, x1, x2, u};
    const double sgn[4] = {1.0, -1.0, 1.0, -1.0};  // p = 1 -/+ E alternately
    double A[4][4], rhs[4], sol[4];
    for (int r = 0; r < 4; ++r) {
      const double x = pts[r];
      A[r][0] = x; A[r][1] = x * x * x; A[r][2] = x * x * x * x * x; A[r][3] = sgn[r];
      rhs[r] = 1.0;
    }
    if (!solve4(A, rhs, sol)) return PE_ERR_NO_CONVERGENCE;
    a = sol[0]; b = sol[1]; c = sol[2]; E = sol[3];
    // extrema of 1 - p: roots of 5c x^4 + 3b x^2 + a
    const double disc = std::sqrt(9.0 * b * b - 20.0 * a * c);
    x1 = std::sqrt((-3.0 * b - disc) / (10.0 * c));
    x2 = std::sqrt((-3.0 * b + disc) / (10.0 * c));
    if (!std::isfinite(x1) || !std::isfinite(x2)) return PE_ERR_NO_CONVERGENCE;
  }
  out[0] = a; out[1] = b; out[2] = c;
  return PE_OK;
}

// eq. (deg3_solution): p(x) = beta p_NS(alpha x).
void cubic(double l, double u, double out[2], bool* pade) {
  *pade = (l / u >= kPadeThreshold);
  if (*pade) { out[0] = 1.5; out[1] = -0.5; return; }
  const double alpha = std::sqrt(3.0 / (u * u + l * u + l * l));
  const double beta = 4.0 / (2.0 + l * u * (l + u) * alpha * alpha * alpha);
  out[0] = beta * 1.5 * alpha;
  out[1] = -beta * 0.5 * alpha * alpha * alpha;
}

}  // namespace

extern "C" pe_status pe_coeffs_ex(double ell, int degree, int T, double safety, double cushion,
                                  int flags, double* coeffs, double* ell_trace) {
  if (coeffs == nullptr || !(ell > 0.0 && ell <= 1.0) || T < 1 || !(safety >= 1.0) ||
      !std::isfinite(safety))
    return PE_ERR_INVALID_ARG;
  if (degree != 3 && degree != 5) return PE_ERR_UNSUPPORTED;
  const int nq = (degree + 1) / 2;
  if (cushion < 0.0) cushion = (degree == 5) ? kCushion5 : kCushion3;
  if (!(cushion < 1.0)) return PE_ERR_INVALID_ARG;

  double l = ell, u = 1.0;
  if (ell_trace) ell_trace[0] = l;
  for (int t = 0; t < T; ++t) {
    double p[3] = {0, 0, 0};
    bool pade = false;
    const double lo = std::fmax(l, cushion * u);  // cushion
    if (degree == 5) {
      pe_status s = quintic(lo, u, p, &pade);
      if (s != PE_OK) return s;
      if (pade) { p[0] = 15.0 / 8.0; p[1] = -10.0 / 8.0; p[2] = 3.0 / 8.0; }  // R4
    } else {
      cubic(lo, u, p, &pade);
    }
    if (!pade && !(flags & PE_NO_RECENTER)) {
      // recentre so that 1 - min p = max p - 1 over [l_t, u_t];
      // the quintic's max is at u, the cubic's at its interior extremum (R15).
      const double pl = eval_odd(p, nq, l);
      double pmax = eval_odd(p, nq, u);
      if (degree == 3) {
        double xs = std::sqrt(-p[0] / (3.0 * p[1]));
        xs = std::fmin(std::fmax(xs, l), u);
        pmax = std::fmax(pmax, eval_odd(p, nq, xs));
      }
      const double r = 2.0 / (pl + pmax);
      for (int q = 0; q < nq; ++q) p[q] *= r;
    }
    const double l_next = eval_odd(p, nq, l);
    u = 2.0 - l_next;
    l = l_next;
    if (ell_trace) ell_trace[t + 1] = l;
    // safety (R5 leaves the Pade tail unscaled)
    bool scale = !pade || (flags & PE_SAFETY_ALL);
    if ((flags & PE_SAFETY_NOT_FINAL) && t == T - 1) scale = false;
    double f = safety;
    for (int q = 0; q < nq; ++q) {
      coeffs[t * nq + q] = scale ? p[q] / f : p[q];
      f *= safety * safety;
    }
  }
  return PE_OK;
}

extern "C" pe_status pe_coeffs(double ell, int degree, int T, double safety, double* coeffs) {
  return pe_coeffs_ex(ell, degree, T, safety, -1.0, 0, coeffs, nullptr);
}
