// linalg.cpp -- oracle: thin SVD / POD and minimum-norm least squares.
// TEST INFRASTRUCTURE ONLY (see oracle.h).
//
// POD_m: "applies the thin SVD to the argument ... and extracts the m
// left singular vectors".  Gappy coordinates (Eq. 8): y = (P^T Phi)^+ P^T(v - psi).
// Both are written out textbook-style: Householder QR of the tall matrix, then
// one-sided (Hestenes) Jacobi SVD of the small triangular factor (reading A15;
// cut-offs A13/A15).  All inner products are Neumaier-compensated.
#include <algorithm>
#include <cmath>
#include <numeric>
#include "common.hpp"

namespace orc {

// In-place Householder QR of A (m x n, col-major, m >= n).  On exit the upper
// triangle of A holds R; V[j] holds the unit Householder vector of step j
// (length m - j), H_j = I - 2 v v^T acting on rows j..m-1.
void householder_qr(double* A, int64_t m, int n, std::vector<std::vector<double>>& V) {
  V.assign(n, {});
  for (int j = 0; j < n; ++j) {
    double* x = A + (int64_t)j * m + j;
    const int64_t len = m - j;
    const double nrm = std::sqrt(dot(x, x, len));
    std::vector<double> v(x, x + len);
    if (nrm == 0.0) {  // zero column: identity reflector
      V[j].assign(len, 0.0);
      continue;
    }
    const double alpha = (x[0] >= 0.0) ? -nrm : nrm;
    v[0] = x[0] - alpha;
    const double vn = std::sqrt(dot(v.data(), v.data(), len));
    for (auto& t : v) t /= vn;
    // apply to columns j..n-1
    for (int k = j; k < n; ++k) {
      double* a = A + (int64_t)k * m + j;
      const double s = 2.0 * dot(v.data(), a, len);
      for (int64_t i = 0; i < len; ++i) a[i] -= s * v[i];
    }
    x[0] = alpha;
    for (int64_t i = 1; i < len; ++i) x[i] = 0.0;
    V[j] = std::move(v);
  }
}

// x <- Q x, Q = H_0 H_1 ... H_{n-1}
void apply_q(const std::vector<std::vector<double>>& V, int64_t m, double* x) {
  for (int j = (int)V.size() - 1; j >= 0; --j) {
    const auto& v = V[j];
    const int64_t len = m - j;
    const double s = 2.0 * dot(v.data(), x + j, len);
    for (int64_t i = 0; i < len; ++i) x[j + i] -= s * v[i];
  }
}

// x <- Q^T x
void apply_qt(const std::vector<std::vector<double>>& V, int64_t m, double* x) {
  for (size_t j = 0; j < V.size(); ++j) {
    const auto& v = V[j];
    const int64_t len = m - (int64_t)j;
    const double s = 2.0 * dot(v.data(), x + j, len);
    for (int64_t i = 0; i < len; ++i) x[j + i] -= s * v[i];
  }
}

// One-sided Jacobi on B (m x n): B V = U diag(S).  On exit B holds U*diag(S)
// (unsorted), V the accumulated rotations, S the column norms.
void jacobi_svd_square(double* B, int64_t m, int n, double* V, double* S) {
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) V[(int64_t)j * n + i] = (i == j) ? 1.0 : 0.0;
  const double tol = 1e-15;
  for (int sweep = 0; sweep < 100; ++sweep) {
    int rotations = 0;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        double* bp = B + (int64_t)p * m;
        double* bq = B + (int64_t)q * m;
        const double alpha = dot(bp, bp, m);
        const double beta = dot(bq, bq, m);
        const double gamma = dot(bp, bq, m);
        if (gamma == 0.0 || std::fabs(gamma) <= tol * std::sqrt(alpha * beta)) continue;
        ++rotations;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / std::sqrt(1.0 + t * t);
        const double sn = cs * t;
        for (int64_t i = 0; i < m; ++i) {
          const double x = bp[i], y = bq[i];
          bp[i] = cs * x - sn * y;
          bq[i] = sn * x + cs * y;
        }
        double* vp = V + (int64_t)p * n;
        double* vq = V + (int64_t)q * n;
        for (int i = 0; i < n; ++i) {
          const double x = vp[i], y = vq[i];
          vp[i] = cs * x - sn * y;
          vq[i] = sn * x + cs * y;
        }
      }
    if (rotations == 0) break;
  }
  for (int j = 0; j < n; ++j) {
    const double* b = B + (int64_t)j * m;
    S[j] = std::sqrt(dot(b, b, m));
  }
}

}  // namespace orc

using namespace orc;

extern "C" {

// Thin SVD X = U diag(S) V^T, descending S; sign: the largest-|V_ij| entry of
// each right singular vector (ties -> lowest i) is positive (reading A15).
void orc_svd(const double* X, int64_t m, int32_t n, double* U, double* S, double* V) {
  std::vector<double> W(X, X + m * (int64_t)n);
  std::vector<std::vector<double>> H;
  std::vector<double> Vt((int64_t)n * n), St(n);
  int64_t mr;  // row count of the matrix handed to Jacobi
  std::vector<double> R;
  const bool tall = m >= n;
  if (tall) {
    householder_qr(W.data(), m, n, H);
    R.assign((int64_t)n * n, 0.0);
    for (int j = 0; j < n; ++j)
      for (int i = 0; i <= j; ++i) R[(int64_t)j * n + i] = W[(int64_t)j * m + i];
    mr = n;
  } else {
    R = W;
    mr = m;
  }
  jacobi_svd_square(R.data(), mr, n, Vt.data(), St.data());
  std::vector<int> ord(n);
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return St[a] > St[b]; });
  for (int jj = 0; jj < n; ++jj) {
    const int j = ord[jj];
    S[jj] = St[j];
    // sign from V
    int imax = 0;
    double vmax = -1.0;
    for (int i = 0; i < n; ++i) {
      const double a = std::fabs(Vt[(int64_t)j * n + i]);
      if (a > vmax) { vmax = a; imax = i; }
    }
    const double sg = (Vt[(int64_t)j * n + imax] < 0.0) ? -1.0 : 1.0;
    for (int i = 0; i < n; ++i) V[(int64_t)jj * n + i] = sg * Vt[(int64_t)j * n + i];
    if (U) {
      std::vector<double> u(m, 0.0);
      const double* b = R.data() + (int64_t)j * mr;
      for (int64_t i = 0; i < mr; ++i) u[i] = (St[j] > 0.0) ? sg * b[i] / St[j] : 0.0;
      if (tall) apply_q(H, m, u.data());
      std::copy(u.begin(), u.end(), U + (int64_t)jj * m);
    }
  }
}

// POD_r of the w deviation columns: r_eff = #{i < r : S_i^2 >= cut S_0^2}
int32_t orc_pod(const double* X, int64_t m, int32_t w, int32_t r, double cut, double* Phi,
                double* S, double* V) {
  std::vector<double> U(m * (int64_t)w), Sv(w), Vv((int64_t)w * w);
  orc_svd(X, m, w, U.data(), Sv.data(), Vv.data());
  int32_t reff = 0;
  for (int i = 0; i < std::min(r, w); ++i)
    if (Sv[0] > 0.0 && Sv[i] * Sv[i] >= cut * Sv[0] * Sv[0]) ++reff;
    else break;
  if (Phi) std::copy(U.begin(), U.begin() + m * (int64_t)reff, Phi);
  if (S) std::copy(Sv.begin(), Sv.end(), S);
  if (V) std::copy(Vv.begin(), Vv.end(), V);
  return reff;
}

// minimum-norm least squares x = A^+ b, keeping sigma_i^2 >= cut * sigma_1^2 (A13)
int32_t orc_lsq(const double* A, int64_t m, int32_t n, const double* b, double cut, double* x) {
  for (int i = 0; i < n; ++i) x[i] = 0.0;
  if (n == 0 || m == 0) return 0;
  std::vector<double> U(m * (int64_t)n), S(n), V((int64_t)n * n);
  orc_svd(A, m, n, U.data(), S.data(), V.data());
  int32_t rank = 0;
  for (int j = 0; j < n; ++j) {
    if (!(S[0] > 0.0) || !(S[j] * S[j] >= cut * S[0] * S[0])) break;
    ++rank;
    const double coef = dot(U.data() + (int64_t)j * m, b, m) / S[j];
    for (int i = 0; i < n; ++i) x[i] += coef * V[(int64_t)j * n + i];
  }
  return rank;
}

void orc_gram(const double* S, int32_t ncol, int64_t rows, const double* rho, double* C) {
  std::vector<double> a(rows), b(rows);
  for (int i = 0; i < ncol; ++i)
    for (int j = i; j < ncol; ++j) {
      CSum s;
      for (int64_t e = 0; e < rows; ++e) {
        const double x = S[(int64_t)i * rows + e] - (rho ? rho[e] : 0.0);
        const double y = S[(int64_t)j * rows + e] - (rho ? rho[e] : 0.0);
        s.add(x * y);
      }
      C[(int64_t)i * ncol + j] = C[(int64_t)j * ncol + i] = s.value();
    }
}

// Projection of snapshots on a basis (config-5 kernel op; the POD
// coefficients Phi^T (gamma - .) of P:266/P:281): C[i * ncol + j] = sum_e Phi[i][e] S[j][e],
// Phi: m columns of D rows, S: ncol columns of D rows (both column-major), compensated sums.
void orc_project(const double* Phi, int64_t D, int32_t m, const double* S, int32_t ncol, double* C) {
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < ncol; ++j) C[(int64_t)i * ncol + j] = dot(Phi + (int64_t)i * D, S + (int64_t)j * D, D);
}

}  // extern "C"
