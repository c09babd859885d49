// Host dense kernel K10: y = beta0 * H_m^{-1/2} e_1, principal
// branch, for the small projected matrix of Algorithm 1.
//
//  * Hermitian (Lanczos) case: symmetric tridiagonal T = Z diag(theta) Z^T by
//    the implicit-shift QL iteration; y = beta0 Z (theta^{-1/2} .* Z(0,:)^T).
//  * General case, as P:153 suggests: complex Schur H = Q T Q^H by the
//    single-shift implicit QR iteration on the Hessenberg matrix, the upper
//    triangular square root R of T (R_ii = sqrt(T_ii), then the column-wise
//    recurrence R_ij = (T_ij - sum_{i<k<j} R_ik R_kj)/(R_ii + R_jj)), and
//    y = beta0 Q R^{-1} Q^H e_1 by back substitution.
// No LAPACK exists in this image; these are written out here and are
// independent of the oracle (which uses NumPy's eig/eigh).
#include <algorithm>
#include <cmath>

#include "ppf_internal.h"

namespace ppf {

namespace {

// sqrt(a^2 + b^2) without std::hypot's overflow/underflow guards (libm's
// hypot costs ~40 ns, it dominated the QL sweep); the entries of H_m are
// bounded by ||A q(A)^2|| (< 1e8 for every config), far from overflow
inline double fhypot(double a, double b) { return std::sqrt(a * a + b * b); }

inline bool on_branch_cut(zc z) {
  return std::abs(z.imag()) <= 1e-14 * std::max(std::abs(z), 1e-300) && z.real() <= 0.0;
}

}  // namespace

// The eigenvector matrix is never formed: Z = R_1 R_2 ... R_K is a product of
// plane rotations on adjacent columns (i, i+1).  Only e_1^T Z is needed for the
// weights and Z w for the result, so row 0 of Z is tracked through the
// rotations (O(1) each) and w is pushed back through the logged rotations in
// reverse order: O(m^2) instead of O(m^3) (m = 576 at Table 1's d = 1).
void tridiag_invsqrt_e1(int m, const double* dd, const double* ee, double beta0, double* y) {
  std::vector<double> d(dd, dd + m), e(m, 0.0);
  for (int i = 0; i + 1 < m; ++i) e[i] = ee[i];
  struct Rot {
    int i;
    double s, c;
  };
  std::vector<Rot> log;
  log.reserve(size_t(8) * m);
  std::vector<double> z0(m, 0.0);  // row 0 of Z
  z0[0] = 1.0;
  const double eps = 2.220446049250313e-16;
  for (int l = 0; l < m; ++l) {
    int iter = 0;
    int mm;
    do {
      for (mm = l; mm < m - 1; ++mm) {
        const double dsum = std::fabs(d[mm]) + std::fabs(d[mm + 1]);
        if (std::fabs(e[mm]) <= eps * dsum) break;
      }
      if (mm != l) {
        if (iter++ == 100) fail(PPF_EDENSE, "tridiagonal QL iteration did not converge");
        double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
        double r = fhypot(g, 1.0);
        g = d[mm] - d[l] + e[l] / (g + std::copysign(r, g));
        double s = 1.0, c = 1.0, p = 0.0;
        int i;
        bool early = false;
        for (i = mm - 1; i >= l; --i) {
          double f = s * e[i];
          const double b = c * e[i];
          r = fhypot(f, g);
          e[i + 1] = r;
          if (r == 0.0) {
            d[i + 1] -= p;
            e[mm] = 0.0;
            early = true;
            break;
          }
          s = f / r;
          c = g / r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + 2.0 * c * b;
          p = s * r;
          d[i + 1] = g + p;
          g = c * r - b;
          // Z <- Z R: Z[:, i+1] = s Z[:, i] + c Z[:, i+1], Z[:, i] = c Z[:, i] - s Z[:, i+1]
          const double zi = z0[i], zi1 = z0[i + 1];
          z0[i + 1] = s * zi + c * zi1;
          z0[i] = c * zi - s * zi1;
          log.push_back({i, s, c});
        }
        if (early) continue;
        d[l] -= p;
        e[l] = g;
        e[mm] = 0.0;
      }
    } while (mm != l);
  }
  for (int i = 0; i < m; ++i)
    if (!(d[i] > 0.0)) fail(PPF_EBRANCH, "eigenvalue of T_m on (-inf, 0]");
  // y = beta0 Z diag(theta^{-1/2}) Z^T e_1 = Z w, w_i = beta0 z0_i / sqrt(theta_i)
  for (int i = 0; i < m; ++i) y[i] = beta0 * z0[i] / std::sqrt(d[i]);
  for (size_t t = log.size(); t-- > 0;) {
    const Rot& R = log[t];
    const double a = y[R.i], b = y[R.i + 1];
    y[R.i] = R.c * a + R.s * b;
    y[R.i + 1] = -R.s * a + R.c * b;
  }
}

void complex_schur(int m, std::vector<zc>& H, std::vector<zc>& Q) {
  auto h = [&](int i, int j) -> zc& { return H[size_t(i) + size_t(j) * m]; };
  auto q = [&](int i, int j) -> zc& { return Q[size_t(i) + size_t(j) * m]; };
  Q.assign(size_t(m) * m, zc(0.0, 0.0));
  for (int i = 0; i < m; ++i) q(i, i) = 1.0;
  for (int j = 0; j < m; ++j)
    for (int i = j + 2; i < m; ++i) h(i, j) = 0.0;  // Hessenberg input
  const double eps = 2.220446049250313e-16;
  int hi = m - 1, iter = 0, total = 0;
  while (hi > 0) {
    int l = hi;
    while (l > 0) {
      const double s = std::abs(h(l, l)) + std::abs(h(l - 1, l - 1));
      if (std::abs(h(l, l - 1)) <= eps * (s > 0 ? s : 1.0)) break;
      --l;
    }
    if (l > 0) h(l, l - 1) = 0.0;
    if (l == hi) {
      --hi;
      iter = 0;
      continue;
    }
    if (++total > 200 * m) fail(PPF_EDENSE, "complex Schur QR iteration did not converge");
    ++iter;
    // Wilkinson shift from the trailing 2x2 of the active block
    const zc a = h(hi - 1, hi - 1), b = h(hi - 1, hi), c = h(hi, hi - 1), d = h(hi, hi);
    zc mu;
    if (iter % 11 == 10) {
      mu = d + zc(std::abs(c), 0.0);  // exceptional shift
    } else {
      const zc half = (a - d) * 0.5;
      const zc disc = std::sqrt(half * half + b * c);
      const zc e1 = (a + d) * 0.5 + disc, e2 = (a + d) * 0.5 - disc;
      mu = (std::abs(e1 - d) < std::abs(e2 - d)) ? e1 : e2;
    }
    for (int k = l; k < hi; ++k) {
      zc x, y;
      if (k == l) {
        x = h(l, l) - mu;
        y = h(l + 1, l);
      } else {
        x = h(k, k - 1);
        y = h(k + 1, k - 1);
      }
      const double ax = std::abs(x), ay = std::abs(y);
      const double r = std::hypot(ax, ay);
      if (r == 0.0) continue;
      double cg;
      zc sg;
      if (ax == 0.0) {
        cg = 0.0;
        sg = std::conj(y) / ay;
      } else {
        cg = ax / r;
        sg = (x / ax) * std::conj(y) / r;
      }
      // rows k, k+1 (all columns from k-1 or l to the end): G = [c s; -conj(s) c]
      const int j0 = (k == l) ? l : k - 1;
      for (int j = j0; j < m; ++j) {
        const zc h1 = h(k, j), h2 = h(k + 1, j);
        h(k, j) = cg * h1 + sg * h2;
        h(k + 1, j) = -std::conj(sg) * h1 + cg * h2;
      }
      // columns k, k+1 (rows 0 .. min(k+2, hi)): times G^H = [c -s; conj(s) c]
      const int i1 = std::min(k + 2, hi);
      for (int i = 0; i <= i1; ++i) {
        const zc h1 = h(i, k), h2 = h(i, k + 1);
        h(i, k) = cg * h1 + std::conj(sg) * h2;
        h(i, k + 1) = -sg * h1 + cg * h2;
      }
      for (int i = 0; i < m; ++i) {
        const zc q1 = q(i, k), q2 = q(i, k + 1);
        q(i, k) = cg * q1 + std::conj(sg) * q2;
        q(i, k + 1) = -sg * q1 + cg * q2;
      }
      if (k > l) h(k + 1, k - 1) = 0.0;
    }
  }
  for (int j = 0; j < m; ++j)
    for (int i = j + 1; i < m; ++i) h(i, j) = 0.0;
}

std::vector<zc> eigenvalues(int m, std::vector<zc> H) {
  std::vector<zc> Q;
  complex_schur(m, H, Q);
  std::vector<zc> ev(m);
  for (int i = 0; i < m; ++i) ev[i] = H[size_t(i) + size_t(i) * m];
  return ev;
}

void general_invsqrt_e1(int m, const std::vector<zc>& H0, double beta0, std::vector<zc>& y) {
  std::vector<zc> T = H0, Q;
  complex_schur(m, T, Q);
  auto t = [&](int i, int j) -> const zc& { return T[size_t(i) + size_t(j) * m]; };
  std::vector<zc> R(size_t(m) * m, zc(0.0, 0.0));
  auto r = [&](int i, int j) -> zc& { return R[size_t(i) + size_t(j) * m]; };
  for (int i = 0; i < m; ++i) {
    if (on_branch_cut(t(i, i))) fail(PPF_EBRANCH, "eigenvalue of H_m on (-inf, 0]");
    r(i, i) = std::sqrt(t(i, i));  // principal branch
  }
  for (int j = 1; j < m; ++j) {
    for (int i = j - 1; i >= 0; --i) {
      zc s = t(i, j);
      for (int k = i + 1; k < j; ++k) s -= r(i, k) * r(k, j);
      r(i, j) = s / (r(i, i) + r(j, j));
    }
  }
  // u = R^{-1} Q^H e1
  std::vector<zc> u(m);
  for (int i = 0; i < m; ++i) u[i] = std::conj(Q[size_t(0) + size_t(i) * m]);
  for (int i = m - 1; i >= 0; --i) {
    zc s = u[i];
    for (int k = i + 1; k < m; ++k) s -= r(i, k) * u[k];
    u[i] = s / r(i, i);
  }
  y.assign(m, zc(0.0, 0.0));
  for (int k = 0; k < m; ++k)
    for (int i = 0; i < m; ++i) y[i] += Q[size_t(i) + size_t(k) * m] * u[k];
  for (int i = 0; i < m; ++i) y[i] *= beta0;
}

}  // namespace ppf
