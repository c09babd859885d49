// Host construction of the preconditioning polynomial q ~ z^{-1/2} (layer L1).
//
// Chebyshev: c_i = (2/pi) int w f T_i (c_0 with 1/pi) evaluated by
// the (deg+1)-point Gauss-Chebyshev rule (reading Q2), i.e.
//   c_i = (2/d) sum_l f(z_l) cos(i theta_l), theta_l = pi (l + 1/2)/d,
//   z_l = (a+b)/2 + (b-a)/2 cos(theta_l), c_0 halved;
// scalar evaluation by the Clenshaw recurrence.
// Newton: Leja order and divided differences of z^{-1/2}.
#include <algorithm>
#include <utility>
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

// Certificate (P:334-335 for Chebyshev, P:401-403 for a contour): min Re q
// over the points -- host `pts` of npts R64 or C128 (interleaved) values, or
// (pts == NULL, Chebyshev only) z_k = a + (b-a)k/1000, k = 0..1000.
// NaN anywhere gives NaN (so "min > 0" fails).
double certify_min_re(const ppf_poly& q, const void* pts, int npts, int dtype) {
  double mn = HUGE_VAL;
  auto take = [&](double v) {
    if (std::isnan(v) || std::isnan(mn)) mn = NAN;
    else mn = std::min(mn, v);
  };
  if (!pts) {
    for (int k = 0; k <= 1000; ++k) {
      const double z = q.a + (q.b - q.a) * k / 1000.0;
      take(q.kind == PPF_POLY_CHEBYSHEV ? chebyshev_eval(q, z) : poly_eval(q, zc(z, 0.0)).real());
    }
    return mn;
  }
  const double* p = static_cast<const double*>(pts);
  for (int i = 0; i < npts; ++i) {
    const zc z = dtype == PPF_C128 ? zc(p[2 * i], p[2 * i + 1]) : zc(p[i], 0.0);
    if (q.kind == PPF_POLY_CHEBYSHEV && z.imag() == 0.0) take(chebyshev_eval(q, z.real()));
    else take(poly_eval(q, z).real());
  }
  return mn;
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

// Least-squares q on a discretised contour: Arnoldi on
// diag(z_1..z_N) from [1..1]/sqrt(N) gives the orthonormal basis polynomials
// as the columns of P; alpha = P^H z^{-1/2}; the fit's
// values at the contour points are P alpha.  The device applies q in Newton
// form: q has degree deg, so its interpolant at deg+1 Leja-ordered contour
// points is q itself (divided differences of the fitted values), evaluated by
// the same fused Newton-Horner chain as the Ritz polynomials.  Returns
// min Re q(z_i) (the certificate of P:401-403) through min_re.
void contour_ls_newton(const std::vector<zc>& z, int deg, std::vector<zc>& nodes,
                       std::vector<zc>& dd, double& min_re) {
  const int N = int(z.size()), d = deg + 1;
  std::vector<zc> P(size_t(N) * d, zc(0.0, 0.0));  // column-major N x d
  auto col = [&](int k) { return &P[size_t(k) * N]; };
  for (int i = 0; i < N; ++i) col(0)[i] = 1.0 / std::sqrt(double(N));
  std::vector<zc> w(N), h(d);
  for (int k = 1; k < d; ++k) {
    for (int i = 0; i < N; ++i) w[i] = z[i] * col(k - 1)[i];
    for (int pass = 0; pass < 2; ++pass) {  // CGS with one reorthogonalisation
      for (int j = 0; j < k; ++j) {
        zc s(0.0, 0.0);
        for (int i = 0; i < N; ++i) s += std::conj(col(j)[i]) * w[i];
        h[j] = s;
      }
      for (int j = 0; j < k; ++j)
        for (int i = 0; i < N; ++i) w[i] -= h[j] * col(j)[i];
    }
    double nr = 0.0;
    for (int i = 0; i < N; ++i) nr += std::norm(w[i]);
    nr = std::sqrt(nr);
    if (!(nr > 0.0)) fail(PPF_EINVAL, "contour points do not support degree deg (need deg + 1 distinct points)");
    for (int i = 0; i < N; ++i) col(k)[i] = w[i] / nr;
  }
  std::vector<zc> alpha(d);
  for (int j = 0; j < d; ++j) {
    zc s(0.0, 0.0);
    for (int i = 0; i < N; ++i) s += std::conj(col(j)[i]) * (1.0 / std::sqrt(z[i]));
    alpha[j] = s;
  }
  std::vector<zc> qz(N, zc(0.0, 0.0));
  for (int j = 0; j < d; ++j)
    for (int i = 0; i < N; ++i) qz[i] += alpha[j] * col(j)[i];
  min_re = HUGE_VAL;
  for (int i = 0; i < N; ++i) min_re = std::min(min_re, qz[i].real());
  // deg+1 nodes in Leja order among the contour points (same rule as
  // leja_order: max modulus first, then greedy max sum log distance, ties to
  // the smaller index after sorting by (Re, Im))
  std::vector<int> idx(N);
  for (int i = 0; i < N; ++i) idx[i] = i;
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) {
    if (z[a].real() != z[b].real()) return z[a].real() < z[b].real();
    return z[a].imag() < z[b].imag();
  });
  std::vector<char> used(N, 0);
  std::vector<double> score(N, 0.0);
  std::vector<int> chosen;
  int first = 0;
  for (int t = 1; t < N; ++t)
    if (std::abs(z[idx[t]]) > std::abs(z[idx[first]])) first = t;
  chosen.push_back(first);
  used[first] = 1;
  while (int(chosen.size()) < d) {
    const int last = chosen.back();
    int best = -1;
    for (int t = 0; t < N; ++t) {
      if (used[t]) continue;
      score[t] += std::log(std::abs(z[idx[t]] - z[idx[last]]));
      if (best < 0 || score[t] > score[best]) best = t;
    }
    chosen.push_back(best);
    used[best] = 1;
  }
  nodes.resize(d);
  dd.resize(d);
  for (int j = 0; j < d; ++j) {
    nodes[j] = z[idx[chosen[j]]];
    dd[j] = qz[idx[chosen[j]]];
  }
  for (int k = 1; k < d; ++k)
    for (int i = d - 1; i >= k; --i) dd[i] = (dd[i] - dd[i - 1]) / (nodes[i] - nodes[i - k]);
}

// Contour from Ritz values (reading Q29): the
// convex hull of the values (Andrew's monotone chain; collinear values give
// the segment there and back), densified in steps of length <= step, points
// closer to 0 than r_min projected radially onto |z| = r_min (the circular
// arc replacing that part), then resampled uniformly and re-projected.
std::vector<zc> ritz_polygon(const std::vector<zc>& theta, double r_min, double step) {
  std::vector<std::pair<double, double>> P;
  for (const zc& t : theta) {
    const double x = std::nearbyint(t.real() * 1e15) / 1e15, y = std::nearbyint(t.imag() * 1e15) / 1e15;
    P.push_back({x, y});
  }
  std::sort(P.begin(), P.end());
  P.erase(std::unique(P.begin(), P.end()), P.end());
  if (P.size() < 2) fail(PPF_EINVAL, "need at least two distinct Ritz values");
  auto cross = [](const std::pair<double, double>& o, const std::pair<double, double>& a,
                  const std::pair<double, double>& b) {
    return (a.first - o.first) * (b.second - o.second) - (a.second - o.second) * (b.first - o.first);
  };
  std::vector<std::pair<double, double>> lower, upper;
  for (const auto& p : P) {
    while (lower.size() >= 2 && cross(lower[lower.size() - 2], lower.back(), p) <= 0) lower.pop_back();
    lower.push_back(p);
  }
  for (auto it = P.rbegin(); it != P.rend(); ++it) {
    while (upper.size() >= 2 && cross(upper[upper.size() - 2], upper.back(), *it) <= 0) upper.pop_back();
    upper.push_back(*it);
  }
  std::vector<zc> verts;
  for (size_t i = 0; i + 1 < lower.size(); ++i) verts.push_back(zc(lower[i].first, lower[i].second));
  for (size_t i = 0; i + 1 < upper.size(); ++i) verts.push_back(zc(upper[i].first, upper[i].second));
  std::vector<zc> z;
  const size_t nv = verts.size();
  for (size_t i = 0; i < nv; ++i) {
    const zc a = verts[i], c = verts[(i + 1) % nv];
    const int k = std::max(1, int(std::ceil(std::abs(c - a) / step)));
    for (int t = 0; t < k; ++t) z.push_back(a + (c - a) * (double(t) / k));
  }
  double wind = 0.0;
  for (size_t i = 0; i < z.size(); ++i) wind += std::arg(z[(i + 1) % z.size()] / z[i]);
  if (std::fabs(wind) > M_PI) fail(PPF_EBRANCH, "the Ritz polygon surrounds 0");
  bool close = false;
  for (auto& v : z)
    if (std::abs(v) < r_min) {
      v = std::polar(r_min, std::arg(v));
      close = true;
    }
  if (close) {
    const size_t nz = z.size();
    std::vector<double> s(nz + 1, 0.0);
    for (size_t i = 0; i < nz; ++i) s[i + 1] = s[i] + std::abs(z[(i + 1) % nz] - z[i]);
    std::vector<zc> r;
    size_t i = 0;
    for (double t = 0.0; t < s[nz]; t += step) {
      while (i + 1 < nz && s[i + 1] <= t) ++i;
      const double seg = s[i + 1] - s[i];
      const double f = seg > 0.0 ? (t - s[i]) / seg : 0.0;
      zc v = z[i] + f * (z[(i + 1) % nz] - z[i]);
      if (std::abs(v) < r_min) v = std::polar(r_min, std::arg(v));
      r.push_back(v);
    }
    z = r;
  }
  return z;
}

// Real-arithmetic form of a Newton polynomial whose nodes are closed under
// conjugation (the Ritz values of a real operator): Lejà order with each
// complex node immediately followed by its conjugate, divided differences of
// z^{-1/2} in that order, then the coefficients c_j in the real basis
//   P_0 = 1,  P_{j+1} = (z - a_j) P_j                    (real node, or the first of a pair)
//             P_{j+1} = (z - a_j) P_j + b_j^2 P_{j-1}      (the second of a pair a +- i b)
// (P_{j+2} = ((z-a)^2 + b^2) P_j = N_{j+2}); with N_{j+1} = P_{j+1} - i b P_j
// inside a pair, q = sum dd_j N_j = sum c_j P_j has c_j = dd_j - i b dd_{j+1},
// c_{j+1} = dd_{j+1} there and c_j = dd_j elsewhere -- real for a real q.
void real_pair_form(ppf_poly& q) {
  const int d = int(q.nodes.size());
  std::vector<zc> th = q.nodes;
  const double scale = [&] {
    double m = 0.0;
    for (auto& t : th) m = std::max(m, std::abs(t));
    return m;
  }();
  // representatives: real nodes and the Im > 0 member of each pair
  std::vector<zc> rep;
  std::vector<char> used(d, 0);
  for (int i = 0; i < d; ++i) {
    if (used[i]) continue;
    if (std::fabs(th[i].imag()) <= 1e-12 * scale) {
      rep.push_back(zc(th[i].real(), 0.0));
      used[i] = 1;
      continue;
    }
    int best = -1;
    for (int j = 0; j < d; ++j)
      if (j != i && !used[j] && (best < 0 || std::abs(th[j] - std::conj(th[i])) < std::abs(th[best] - std::conj(th[i]))))
        best = j;
    if (best < 0 || std::abs(th[best] - std::conj(th[i])) > 1e-8 * scale)
      fail(PPF_EINVAL, "nodes are not closed under conjugation: no real-arithmetic form");
    const zc m = 0.5 * (th[i] + std::conj(th[best]));  // symmetrise the pair
    rep.push_back(zc(m.real(), std::fabs(m.imag())));
    used[i] = used[best] = 1;
  }
  // Lejà order over representatives, each complex one followed by its conjugate
  std::stable_sort(rep.begin(), rep.end(), [](const zc& x, const zc& y) {
    if (x.real() != y.real()) return x.real() < y.real();
    return x.imag() < y.imag();
  });
  std::vector<zc> order;
  std::vector<char> taken(rep.size(), 0);
  auto push = [&](size_t r) {
    taken[r] = 1;
    order.push_back(rep[r]);
    if (rep[r].imag() != 0.0) order.push_back(std::conj(rep[r]));
  };
  size_t first = 0;
  for (size_t r = 1; r < rep.size(); ++r)
    if (std::abs(rep[r]) > std::abs(rep[first])) first = r;
  push(first);
  while (order.size() < size_t(d)) {
    size_t best = rep.size();
    double bv = -HUGE_VAL;
    for (size_t r = 0; r < rep.size(); ++r) {
      if (taken[r]) continue;
      double sc = 0.0;
      for (const zc& o : order) sc += std::log(std::abs(rep[r] - o));
      if (best == rep.size() || sc > bv) {
        best = r;
        bv = sc;
      }
    }
    push(best);
  }
  q.nodes = order;
  q.dd = divided_differences_invsqrt(order);
  q.rp_a.assign(d, 0.0);
  q.rp_b2.assign(d, 0.0);
  q.rp_c.assign(d, 0.0);
  double cmax = 0.0, imax = 0.0;
  for (int j = 0; j < d;) {
    if (order[j].imag() == 0.0) {
      q.rp_a[j] = order[j].real();
      q.rp_c[j] = q.dd[j].real();
      imax = std::max(imax, std::fabs(q.dd[j].imag()));
      cmax = std::max(cmax, std::fabs(q.dd[j].real()));
      ++j;
    } else {
      const double a = order[j].real(), bb = order[j].imag();
      q.rp_a[j] = a;
      q.rp_a[j + 1] = a;
      q.rp_b2[j + 1] = bb * bb;  // step from P_{j+1} to P_{j+2} adds b^2 P_j
      const zc cj = q.dd[j] - zc(0.0, bb) * (j + 1 < d ? q.dd[j + 1] : zc(0.0, 0.0));
      const zc cj1 = j + 1 < d ? q.dd[j + 1] : zc(0.0, 0.0);
      q.rp_c[j] = cj.real();
      q.rp_c[j + 1] = cj1.real();
      imax = std::max({imax, std::fabs(cj.imag()), std::fabs(cj1.imag())});
      cmax = std::max({cmax, std::fabs(cj.real()), std::fabs(cj1.real())});
      j += 2;
    }
  }
  if (imax > 1e-8 * std::max(cmax, 1e-300))
    fail(PPF_EINVAL, "real-basis coefficients are not real (nodes not conjugate-symmetric?)");
  q.newton_eval = 2;
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
