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

// Provenance: the QL sweep below is the textbook implicit-shift QL iteration
// for a symmetric tridiagonal matrix in its classical EISPACK tql2 / Numerical
// Recipes tqli form (Wilkinson shift, rotations chased up from the bottom of
// the unreduced block; variable names g, r, s, c, p, f, b follow that form).
// What is added here: the rotations are logged and row 0 of the eigenvector
// matrix is tracked instead of accumulating it.
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

// With `log` non-null the rotations are recorded there instead of being
// accumulated into Q (Q is then left empty): y = Q R^{-1} Q^H e_1 only needs
// Q^H e_1 and Q u, which the log replays in O(#rotations) -- a third of the
// flops of the sweep saved.
void complex_schur(int m, std::vector<zc>& H, std::vector<zc>& Q, std::vector<CRot>* log) {
  auto h = [&](int i, int j) -> zc& { return H[size_t(i) + size_t(j) * m]; };
  auto q = [&](int i, int j) -> zc& { return Q[size_t(i) + size_t(j) * m]; };
  if (log) {
    Q.clear();
    log->clear();
  } else {
    Q.assign(size_t(m) * m, zc(0.0, 0.0));
    for (int i = 0; i < m; ++i) q(i, i) = 1.0;
  }
  for (int j = 0; j < m; ++j)
    for (int i = j + 2; i < m; ++i) h(i, j) = 0.0;  // Hessenberg input
  const double eps = 2.220446049250313e-16;
  std::vector<CRot> sweep;
  sweep.reserve(size_t(m));
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
    sweep.clear();
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
      sweep.push_back({k, cg, sg});
      // rows k, k+1 inside the active window (columns from k-1 or l to hi):
      // G = [c s; -conj(s) c].  The columns right of the window are not read
      // by the sweep: they get its rotations afterwards, column by column.
      const int j0 = (k == l) ? l : k - 1;
      for (int j = j0; j <= hi; ++j) {
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
      if (log) {
        log->push_back({k, cg, sg});
      } else {
        for (int i = 0; i < m; ++i) {
          const zc q1 = q(i, k), q2 = q(i, k + 1);
          q(i, k) = cg * q1 + std::conj(sg) * q2;
          q(i, k + 1) = -sg * q1 + cg * q2;
        }
      }
      if (k > l) h(k + 1, k - 1) = 0.0;
    }
    // the sweep's rotations on the columns right of the window: each column
    // segment (contiguous in column-major, L1-resident) takes all of them in
    // sweep order -- the same operations on the same values as row-pair-wise
    // application over the whole row (bitwise equal; m = 256: 596 -> 141 ms)
    for (int j = hi + 1; j < m; ++j) {
      zc* col = &h(0, j);
      for (const CRot& g : sweep) {
        const zc h1 = col[g.k], h2 = col[g.k + 1];
        col[g.k] = g.c * h1 + g.s * h2;
        col[g.k + 1] = -std::conj(g.s) * h1 + g.c * h2;
      }
    }
  }
  for (int j = 0; j < m; ++j)
    for (int i = j + 1; i < m; ++i) h(i, j) = 0.0;
}

// f with H^H f = e_{m-1} (the last unit vector), Gaussian elimination with
// partial pivoting on the m x m adjoint (column-major H)
std::vector<zc> solve_dense_adjoint_ed(int m, const std::vector<zc>& H) {
  std::vector<zc> M(size_t(m) * m), f(m, zc(0.0, 0.0));
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) M[size_t(i) * m + j] = std::conj(H[size_t(j) + size_t(i) * m]);  // row-major H^H
  f[m - 1] = 1.0;
  for (int c = 0; c < m; ++c) {
    int p = c;
    for (int r = c + 1; r < m; ++r)
      if (std::abs(M[size_t(r) * m + c]) > std::abs(M[size_t(p) * m + c])) p = r;
    if (std::abs(M[size_t(p) * m + c]) == 0.0) fail(PPF_EDENSE, "singular H_d in the harmonic Ritz construction");
    if (p != c) {
      for (int j = 0; j < m; ++j) std::swap(M[size_t(c) * m + j], M[size_t(p) * m + j]);
      std::swap(f[c], f[p]);
    }
    for (int r = c + 1; r < m; ++r) {
      const zc t = M[size_t(r) * m + c] / M[size_t(c) * m + c];
      for (int j = c; j < m; ++j) M[size_t(r) * m + j] -= t * M[size_t(c) * m + j];
      f[r] -= t * f[c];
    }
  }
  for (int c = m - 1; c >= 0; --c) {
    zc t = f[c];
    for (int j = c + 1; j < m; ++j) t -= M[size_t(c) * m + j] * f[j];
    f[c] = t / M[size_t(c) * m + c];
  }
  return f;
}

std::vector<zc> eigenvalues(int m, std::vector<zc> H) {
  std::vector<zc> Q;
  std::vector<CRot> log;
  complex_schur(m, H, Q, &log);
  std::vector<zc> ev(m);
  for (int i = 0; i < m; ++i) ev[i] = H[size_t(i) + size_t(i) * m];
  return ev;
}

void general_invsqrt_e1(int m, const std::vector<zc>& H0, double beta0, std::vector<zc>& y) {
  std::vector<zc> T = H0, Q;
  std::vector<CRot> log;
  log.reserve(size_t(4) * m * m / 2 + 16);
  complex_schur(m, T, Q, &log);
  auto t = [&](int i, int j) -> const zc& { return T[size_t(i) + size_t(j) * m]; };
  std::vector<zc> R(size_t(m) * m, zc(0.0, 0.0));
  auto r = [&](int i, int j) -> zc& { return R[size_t(i) + size_t(j) * m]; };
  for (int i = 0; i < m; ++i) {
    if (on_branch_cut(t(i, i))) fail(PPF_EBRANCH, "eigenvalue of H_m on (-inf, 0]");
    r(i, i) = std::sqrt(t(i, i));  // principal branch
  }
  // R's rows are also kept row-major (Rt): the inner sum walks row i of R and
  // column j of R, both contiguous then (same terms, same order)
  std::vector<zc> Rt(size_t(m) * m, zc(0.0, 0.0));
  for (int i = 0; i < m; ++i) Rt[size_t(i) * m + i] = r(i, i);
  for (int j = 1; j < m; ++j) {
    const zc* rj = &r(0, j);
    for (int i = j - 1; i >= 0; --i) {
      const zc* ri = &Rt[size_t(i) * m];
      zc s = t(i, j);
      for (int k = i + 1; k < j; ++k) s -= ri[k] * rj[k];
      r(i, j) = s / (r(i, i) + r(j, j));
      Rt[size_t(i) * m + j] = r(i, j);
    }
  }
  // u = R^{-1} Q^H e1.  Q = G_1 G_2 ... G_K with G_t acting on columns
  // (k, k+1) as [c, -s; conj(s), c]: Q^H e1 applies G_t^H in order, Q u
  // applies G_t in reverse order.
  std::vector<zc> u(m, zc(0.0, 0.0));
  u[0] = 1.0;
  for (const CRot& t : log) {
    const zc a = u[t.k], b = u[t.k + 1];
    u[t.k] = t.c * a + t.s * b;
    u[t.k + 1] = -std::conj(t.s) * a + t.c * b;
  }
  for (int i = m - 1; i >= 0; --i) {
    zc s = u[i];
    const zc* ri = &Rt[size_t(i) * m];
    for (int k = i + 1; k < m; ++k) s -= ri[k] * u[k];
    u[i] = s / r(i, i);
  }
  for (size_t t = log.size(); t-- > 0;) {
    const CRot& g = log[t];
    const zc a = u[g.k], b = u[g.k + 1];
    u[g.k] = g.c * a - g.s * b;
    u[g.k + 1] = std::conj(g.s) * a + g.c * b;
  }
  y.assign(m, zc(0.0, 0.0));
  for (int i = 0; i < m; ++i) y[i] = beta0 * u[i];
}

// ---------------------------------------------------------------------------
// Real Hessenberg H (a real operator's Arnoldi matrix): the same Schur route
// in real arithmetic, ~5x fewer flops than the complex single-shift QR.
//  * real Schur H = Q T Q^T by the Francis double-shift QR (3x3 Householder
//    bulge chase, 2x2 Givens at the end of each sweep); every converged 2x2
//    block with real eigenvalues is split by one more rotation, so T's 2x2
//    diagonal blocks carry complex-conjugate pairs only;
//  * the principal square root R of T block by block (Higham 1987): 1x1
//    blocks sqrt(t); a 2x2 block B with eigenvalues th +- i mu has
//    R = alpha I + (B - th I)/(2 alpha), alpha = sqrt((th + |th + i mu|)/2);
//    off-diagonal blocks from R_ii X + X R_jj = T_ij - sum_k R_ik R_kj
//    (Kronecker systems of order <= 4);
//  * y = beta0 Q R^{-1} Q^T e_1 by block back substitution.
// Q is never formed: the reflectors/rotations are logged and replayed on the
// two vectors that need them (Q^T e_1 forward, Q u backward).
// ---------------------------------------------------------------------------
namespace {

struct RTrans {
  int k;        // first index
  int kind;     // 3: Householder on k..k+2 (I - tau v v^T, v[0] = 1); 2: rotation on k, k+1
  double v1, v2, tau;  // Householder
  double c, s;         // rotation M = [[c, -s], [s, c]]
};

// solve the n x n system (n <= 4) M x = b by Gaussian elimination with
// partial pivoting; M row-major
void small_solve(int n, double* M, double* b) {
  for (int c = 0; c < n; ++c) {
    int p = c;
    for (int r = c + 1; r < n; ++r)
      if (std::fabs(M[r * n + c]) > std::fabs(M[p * n + c])) p = r;
    if (M[p * n + c] == 0.0) fail(PPF_EDENSE, "singular block system in the real Schur square root");
    if (p != c) {
      for (int j = 0; j < n; ++j) std::swap(M[c * n + j], M[p * n + j]);
      std::swap(b[c], b[p]);
    }
    for (int r = c + 1; r < n; ++r) {
      const double f = M[r * n + c] / M[c * n + c];
      for (int j = c; j < n; ++j) M[r * n + j] -= f * M[c * n + j];
      b[r] -= f * b[c];
    }
  }
  for (int c = n - 1; c >= 0; --c) {
    double t = b[c];
    for (int j = c + 1; j < n; ++j) t -= M[c * n + j] * b[j];
    b[c] = t / M[c * n + c];
  }
}

}  // namespace

void real_invsqrt_e1(int m, const double* H0, int ldh, double beta0, double* y) {
  std::vector<double> H(size_t(m) * m);
  auto h = [&](int i, int j) -> double& { return H[size_t(i) + size_t(j) * m]; };
  for (int j = 0; j < m; ++j)
    for (int i = 0; i < m; ++i) h(i, j) = (i <= j + 1) ? H0[size_t(i) + size_t(j) * ldh] : 0.0;
  std::vector<RTrans> log;
  log.reserve(size_t(4) * m * m / 2 + 16);
  const double eps = 2.220446049250313e-16;
  // apply M^T from the left to rows (k..k+2) and M from the right to columns
  auto house = [&](int k, double v1, double v2, double tau, int c0, int r1) {
    for (int j = c0; j < m; ++j) {
      const double t = tau * (h(k, j) + v1 * h(k + 1, j) + v2 * h(k + 2, j));
      h(k, j) -= t;
      h(k + 1, j) -= t * v1;
      h(k + 2, j) -= t * v2;
    }
    for (int i = 0; i <= r1; ++i) {
      const double t = tau * (h(i, k) + v1 * h(i, k + 1) + v2 * h(i, k + 2));
      h(i, k) -= t;
      h(i, k + 1) -= t * v1;
      h(i, k + 2) -= t * v2;
    }
    log.push_back({k, 3, v1, v2, tau, 0.0, 0.0});
  };
  auto rot = [&](int k, double c, double s, int c0, int r1) {
    // H <- M^T H M, M = [[c, -s], [s, c]] on (k, k+1)
    for (int j = c0; j < m; ++j) {
      const double a = h(k, j), b = h(k + 1, j);
      h(k, j) = c * a + s * b;
      h(k + 1, j) = -s * a + c * b;
    }
    for (int i = 0; i <= r1; ++i) {
      const double a = h(i, k), b = h(i, k + 1);
      h(i, k) = c * a + s * b;
      h(i, k + 1) = -s * a + c * b;
    }
    log.push_back({k, 2, 0.0, 0.0, 0.0, c, s});
  };
  // Householder for (x, y, z): v = [1, v1, v2], tau with (I - tau v v^T)[x y z]^T = [*, 0, 0]^T
  auto make_house = [&](double x, double yv, double z, double& v1, double& v2, double& tau) -> bool {
    const double nrm = std::sqrt(x * x + yv * yv + z * z);
    if (nrm == 0.0) return false;
    const double alpha = (x >= 0.0) ? -nrm : nrm;
    const double u0 = x - alpha;
    if (u0 == 0.0) return false;
    v1 = yv / u0;
    v2 = z / u0;
    tau = (alpha - x) / alpha;  // = 2 / (v^T v)
    return true;
  };
  std::vector<char> split(m, 0);  // split[i]: T(i+1, i) == 0 (block boundary)
  int hi = m - 1, iter = 0, total = 0;
  while (hi >= 0) {
    int l = hi;
    while (l > 0) {
      const double sc = std::fabs(h(l - 1, l - 1)) + std::fabs(h(l, l));
      if (std::fabs(h(l, l - 1)) <= eps * (sc > 0.0 ? sc : 1.0)) break;
      --l;
    }
    if (l > 0) h(l, l - 1) = 0.0;
    if (l == hi) {  // 1x1 block converged
      --hi;
      iter = 0;
      continue;
    }
    if (l == hi - 1) {  // 2x2 block converged: split it if its eigenvalues are real
      const int k = hi - 1;
      const double a = h(k, k), b = h(k, k + 1), c = h(k + 1, k), d = h(k + 1, k + 1);
      const double p = 0.5 * (a - d), disc = p * p + b * c;
      if (disc >= 0.0 && c != 0.0) {
        // eigenvector of lam = d + z from the block's second row, (z, c), with
        // z = p + sign(p) sqrt(p^2 + bc) free of cancellation (cf. LAPACK's
        // dlanv2); M = [v, v_perp] triangularises the block.  (Forming it from
        // the first row, (b, lam - a), loses all digits when b, c ~ eps.)
        const double z = p + (p >= 0.0 ? std::sqrt(disc) : -std::sqrt(disc));
        const double r = std::sqrt(z * z + c * c);
        if (r > 0.0) rot(k, z / r, c / r, k, k + 1);
        h(k + 1, k) = 0.0;
      } else if (disc >= 0.0) {
        h(k + 1, k) = 0.0;
      }
      hi -= 2;
      iter = 0;
      continue;
    }
    if (++total > 100 * m) fail(PPF_EDENSE, "real Schur QR iteration did not converge");
    ++iter;
    // double shift from the trailing 2x2 (exceptional shifts every 10 iterations)
    double sh, th;
    if (iter % 10 == 0) {  // EISPACK hqr's exceptional shift
      const double w = std::fabs(h(hi, hi - 1)) + std::fabs(h(hi - 1, hi - 2));
      const double xx = 0.75 * w + h(hi, hi);
      sh = 2.0 * xx;
      th = xx * xx + 0.4375 * w * w;
    } else {
      sh = h(hi - 1, hi - 1) + h(hi, hi);
      th = h(hi - 1, hi - 1) * h(hi, hi) - h(hi - 1, hi) * h(hi, hi - 1);
    }
    double x = h(l, l) * h(l, l) + h(l, l + 1) * h(l + 1, l) - sh * h(l, l) + th;
    double yv = h(l + 1, l) * (h(l, l) + h(l + 1, l + 1) - sh);
    double z = h(l + 1, l) * h(l + 2, l + 1);
    for (int k = l; k <= hi - 2; ++k) {
      double v1, v2, tau;
      if (make_house(x, yv, z, v1, v2, tau)) {
        house(k, v1, v2, tau, std::max(l, k - 1), std::min(k + 3, hi));
        if (k > l) h(k + 1, k - 1) = h(k + 2, k - 1) = 0.0;
      }
      x = h(k + 1, k);
      yv = h(k + 2, k);
      if (k < hi - 2) z = h(k + 3, k);
    }
    // final 2x2 rotation on (hi-1, hi) zeroing yv against x
    const double r = std::sqrt(x * x + yv * yv);
    if (r > 0.0) {
      rot(hi - 1, x / r, yv / r, hi - 2, hi);
      h(hi, hi - 2) = 0.0;
    }
  }
  for (int j = 0; j < m; ++j)
    for (int i = j + 2; i < m; ++i) h(i, j) = 0.0;
  // blocks of T
  std::vector<int> bs, bz;  // block start, size
  for (int i = 0; i < m;) {
    if (i + 1 < m && h(i + 1, i) != 0.0) {
      bs.push_back(i);
      bz.push_back(2);
      i += 2;
    } else {
      bs.push_back(i);
      bz.push_back(1);
      i += 1;
    }
  }
  const int nb = int(bs.size());
  std::vector<double> R(size_t(m) * m, 0.0);
  auto r = [&](int i, int j) -> double& { return R[size_t(i) + size_t(j) * m]; };
  for (int b = 0; b < nb; ++b) {
    const int i = bs[b];
    if (bz[b] == 1) {
      if (!(h(i, i) > 0.0)) fail(PPF_EBRANCH, "eigenvalue of H_m on (-inf, 0]");
      r(i, i) = std::sqrt(h(i, i));
    } else {
      const double a = h(i, i), bb = h(i, i + 1), c = h(i + 1, i), d = h(i + 1, i + 1);
      const double thv = 0.5 * (a + d);
      const double mu2 = -(0.25 * (a - d) * (a - d) + bb * c);
      if (!(mu2 > 0.0)) fail(PPF_EDENSE, "2x2 Schur block without a complex pair");
      const double alpha = std::sqrt(0.5 * (thv + std::hypot(thv, std::sqrt(mu2))));
      r(i, i) = alpha + (a - thv) / (2.0 * alpha);
      r(i, i + 1) = bb / (2.0 * alpha);
      r(i + 1, i) = c / (2.0 * alpha);
      r(i + 1, i + 1) = alpha + (d - thv) / (2.0 * alpha);
    }
  }
  for (int bj = 1; bj < nb; ++bj) {
    const int j0 = bs[bj], q = bz[bj];
    for (int bi = bj - 1; bi >= 0; --bi) {
      const int i0 = bs[bi], p = bz[bi];
      double C[4];
      for (int ii = 0; ii < p; ++ii)
        for (int jj = 0; jj < q; ++jj) {
          double t = h(i0 + ii, j0 + jj);
          for (int kk = i0 + p; kk < j0; ++kk) t -= r(i0 + ii, kk) * r(kk, j0 + jj);
          C[ii + p * jj] = t;  // column-major p x q
        }
      // (I_q (x) R_ii + R_jj^T (x) I_p) vec(X) = vec(C)
      const int nn = p * q;
      double Mx[16] = {0};
      for (int jj = 0; jj < q; ++jj)
        for (int ii = 0; ii < p; ++ii) {
          const int row = ii + p * jj;
          for (int kk = 0; kk < p; ++kk) Mx[row * nn + (kk + p * jj)] += r(i0 + ii, i0 + kk);
          for (int ll = 0; ll < q; ++ll) Mx[row * nn + (ii + p * ll)] += r(j0 + ll, j0 + jj);
        }
      small_solve(nn, Mx, C);
      for (int ii = 0; ii < p; ++ii)
        for (int jj = 0; jj < q; ++jj) r(i0 + ii, j0 + jj) = C[ii + p * jj];
    }
  }
  // w = Q^T e_1: apply M_t^T in order
  std::vector<double> w(m, 0.0);
  w[0] = 1.0;
  for (const RTrans& t : log) {
    if (t.kind == 3) {
      const double d = t.tau * (w[t.k] + t.v1 * w[t.k + 1] + t.v2 * w[t.k + 2]);
      w[t.k] -= d;
      w[t.k + 1] -= d * t.v1;
      w[t.k + 2] -= d * t.v2;
    } else {
      const double a = w[t.k], b = w[t.k + 1];
      w[t.k] = t.c * a + t.s * b;
      w[t.k + 1] = -t.s * a + t.c * b;
    }
  }
  // u = R^{-1} w (block back substitution)
  for (int b = nb - 1; b >= 0; --b) {
    const int i0 = bs[b], p = bz[b];
    double rhs[2], Mx[4];
    for (int ii = 0; ii < p; ++ii) {
      double t = w[i0 + ii];
      for (int kk = i0 + p; kk < m; ++kk) t -= r(i0 + ii, kk) * w[kk];
      rhs[ii] = t;
      for (int jj = 0; jj < p; ++jj) Mx[ii * p + jj] = r(i0 + ii, i0 + jj);
    }
    small_solve(p, Mx, rhs);
    for (int ii = 0; ii < p; ++ii) w[i0 + ii] = rhs[ii];
  }
  // y = beta0 Q u: apply M_t in reverse order
  for (size_t t = log.size(); t-- > 0;) {
    const RTrans& T = log[t];
    if (T.kind == 3) {
      const double d = T.tau * (w[T.k] + T.v1 * w[T.k + 1] + T.v2 * w[T.k + 2]);
      w[T.k] -= d;
      w[T.k + 1] -= d * T.v1;
      w[T.k + 2] -= d * T.v2;
    } else {
      const double a = w[T.k], b = w[T.k + 1];
      w[T.k] = T.c * a - T.s * b;
      w[T.k + 1] = T.s * a + T.c * b;
    }
  }
  for (int i = 0; i < m; ++i) y[i] = beta0 * w[i];
}

}  // namespace ppf
