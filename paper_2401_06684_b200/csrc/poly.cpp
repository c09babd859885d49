// Host construction of the preconditioning polynomial q ~ z^{-1/2} (layer L1).
//
// Chebyshev: c_i = (2/pi) int w f T_i (c_0 with 1/pi) evaluated by
// the (deg+1)-point Gauss-Chebyshev rule (reading Q2), i.e.
//   c_i = (2/d) sum_l f(z_l) cos(i theta_l), theta_l = pi (l + 1/2)/d,
//   z_l = (a+b)/2 + (b-a)/2 cos(theta_l), c_0 halved;
// scalar evaluation by the Clenshaw recurrence.
// Newton: Leja order and divided differences of z^{-1/2}.
#include <algorithm>
#include <cmath>

#include "ppf_internal.h"

namespace ppf {

void chebyshev_coefficients(double a, double b, int deg, std::vector<double>& c) {
  const int d = deg + 1;
  const double pi = 3.14159265358979323846;
  std::vector<double> th(d), f(d);
  for (int l = 0; l < d; ++l) {
    th[l] = pi * (l + 0.5) / d;
    const double z = 0.5 * (a + b) + 0.5 * (b - a) * std::cos(th[l]);
    f[l] = 1.0 / std::sqrt(z);
  }
  c.assign(d, 0.0);
  for (int i = 0; i < d; ++i) {
    double s = 0.0;
    for (int l = 0; l < d; ++l) s += f[l] * std::cos(i * th[l]);
    c[i] = 2.0 * s / d;
  }
  c[0] *= 0.5;
}

// Clenshaw: b_k = c_k + 2 t b_{k+1} - b_{k+2}; q = c_0 + t b_1 - b_2.
double chebyshev_eval(const ppf_poly& q, double z) {
  const double t = (2.0 * z - q.a - q.b) / (q.b - q.a);
  double b1 = 0.0, b2 = 0.0;
  for (int k = q.deg; k >= 1; --k) {
    const double b0 = q.c[k] + 2.0 * t * b1 - b2;
    b2 = b1;
    b1 = b0;
  }
  return q.c[0] + t * b1 - b2;
}

zc poly_eval(const ppf_poly& q, zc z) {
  if (q.kind == PPF_POLY_CHEBYSHEV) {
    const zc t = (2.0 * z - q.a - q.b) / (q.b - q.a);
    zc b1 = 0.0, b2 = 0.0;
    for (int k = q.deg; k >= 1; --k) {
      const zc b0 = q.c[k] + 2.0 * t * b1 - b2;
      b2 = b1;
      b1 = b0;
    }
    return q.c[0] + t * b1 - b2;
  }
  // Horner on the Newton form: p = dd_k; p = p (z - theta_j) + dd_j
  zc p = q.dd[q.deg];
  for (int j = q.deg - 1; j >= 0; --j) p = p * (z - q.nodes[j]) + q.dd[j];
  return p;
}

std::vector<zc> leja_order(const std::vector<zc>& nodes) {
  std::vector<zc> pts = nodes;
  std::stable_sort(pts.begin(), pts.end(), [](const zc& x, const zc& y) {
    if (x.real() != y.real()) return x.real() < y.real();
    return x.imag() < y.imag();
  });
  const int n = int(pts.size());
  std::vector<int> chosen;
  std::vector<char> used(n, 0);
  int first = 0;
  for (int i = 1; i < n; ++i)
    if (std::abs(pts[i]) > std::abs(pts[first])) first = i;
  chosen.push_back(first);
  used[first] = 1;
  while (int(chosen.size()) < n) {
    int best = -1;
    double best_val = -HUGE_VAL;
    for (int i = 0; i < n; ++i) {
      if (used[i]) continue;
      double s = 0.0;
      for (int j : chosen) s += std::log(std::abs(pts[i] - pts[j]));
      if (best < 0 || s > best_val) {
        best = i;
        best_val = s;
      }
    }
    chosen.push_back(best);
    used[best] = 1;
  }
  std::vector<zc> out;
  for (int i : chosen) out.push_back(pts[i]);
  return out;
}

std::vector<zc> divided_differences_invsqrt(const std::vector<zc>& x) {
  const int n = int(x.size());
  std::vector<zc> dd(n);
  for (int i = 0; i < n; ++i) dd[i] = 1.0 / std::sqrt(x[i]);
  for (int k = 1; k < n; ++k)
    for (int i = n - 1; i >= k; --i) dd[i] = (dd[i] - dd[i - 1]) / (x[i] - x[i - k]);
  return dd;
}

}  // namespace ppf
