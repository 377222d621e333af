// implicit.cpp -- oracle: the paper's own implicit HDM.
// TEST INFRASTRUCTURE ONLY (see oracle.h).
//
//   * Roe flux ("MUSCL ... with Roe flux [roe_1981] and minmod limiter"), no entropy fix
//     (reading A37: the paper is silent; S:151 default), written in the textbook wave form:
//     F = 1/2 (F(U_L) + F(U_R)) - 1/2 sum_k |lambda_k| alpha_k r_k at the Roe average.
//   * Wall boundaries ("All four boundaries are taken to be walls"): two ghost layers
//     mirror the interior cells with the normal momentum negated (reading A38).
//   * BDF of order s (P:170-177 Eq. bdf): sum_j a_j q_{n+j} = dt beta f*(q_{n+s}); BDF2 with
//     a_0 = 1/3, a_1 = -4/3, a_2 = 1, beta = 2/3; the first step k = 1 uses BDF1
//     (a_0 = -1, beta = 1), reading A39.
//   * The HDM residual R_k(q) = q - F_k(q), F_k(q) = dt beta f*(q) - sum_{j<s} a_j q_{k-s+j}
//     (P:179-189 Eq. hdm), solved by Newton's method with GMRES on Jacobian-vector products
//     ("Newton's method ... GMRES"); the products are one-sided finite differences
//     of R (reading A40).  Only the converged root is compared with the GPU, never the
//     iterates: both sides stop at ||R||_inf <= tol.
//   * The partial HDM (Eq. 6b, Eq. partial_hdm2): the same Newton solve restricted
//     to the rows of S-hat, with the values on S-tilde = Neighbors(S-hat) frozen.
#include <algorithm>
#include <cmath>
#include <limits>
#include <vector>
#include "common.hpp"

using namespace orc;

extern "C" {

// Roe flux through a face normal to `axis` (0: x, 1: y), conservative states U_L, U_R.
// Roe averages (Roe 1981): sqrt-density weights for u, v, H; a~^2 = (gamma-1)(H - |u|^2/2).
// Wave strengths from the jumps of the primitive variables (dp, du_n, du_t, drho):
//   alpha_1 = (dp - rho a du_n) / (2 a^2),   lambda_1 = u_n - a,  r_1 = (1, u - a n, H - u_n a)
//   alpha_2 = drho - dp / a^2,               lambda_2 = u_n,      r_2 = (1, u, |u|^2 / 2)
//   alpha_3 = rho du_t   (2D only),          lambda_3 = u_n,      r_3 = (0, t, u_t)
//   alpha_4 = (dp + rho a du_n) / (2 a^2),   lambda_4 = u_n + a,  r_4 = (1, u + a n, H + u_n a)
// Returns 0, or -1 when the Roe average is not admissible (a~^2 <= 0).
int32_t orc_roe(int32_t dim, int32_t axis, double gamma, const double* UL, const double* UR, double* F) {
  const int c = dim + 2;
  double FL[4], FR[4];
  orc_physical_flux(dim, axis, gamma, UL, FL);
  orc_physical_flux(dim, axis, gamma, UR, FR);
  const double rL = UL[0], rR = UR[0];
  const double pL = orc_pressure(dim, gamma, UL), pR = orc_pressure(dim, gamma, UR);
  double uL[2] = {0, 0}, uR[2] = {0, 0};
  for (int d = 0; d < dim; ++d) {
    uL[d] = UL[1 + d] / rL;
    uR[d] = UR[1 + d] / rR;
  }
  const double HL = (UL[c - 1] + pL) / rL, HR = (UR[c - 1] + pR) / rR;
  const double sL = std::sqrt(rL), sR = std::sqrt(rR);
  double u[2] = {0, 0};
  for (int d = 0; d < dim; ++d) u[d] = (sL * uL[d] + sR * uR[d]) / (sL + sR);
  const double H = (sL * HL + sR * HR) / (sL + sR);
  double q2 = 0.0;
  for (int d = 0; d < dim; ++d) q2 += u[d] * u[d];
  const double a2 = (gamma - 1.0) * (H - 0.5 * q2);
  if (!(a2 > 0.0)) {
    for (int v = 0; v < c; ++v) F[v] = std::numeric_limits<double>::quiet_NaN();
    return -1;
  }
  const double a = std::sqrt(a2), rho = sL * sR;
  const int t = 1 - axis;  // tangential axis (2D)
  const double un = u[axis];
  const double drho = rR - rL, dp = pR - pL, dun = uR[axis] - uL[axis];
  const double al1 = (dp - rho * a * dun) / (2.0 * a2);
  const double al2 = drho - dp / a2;
  const double al4 = (dp + rho * a * dun) / (2.0 * a2);
  const double l1 = std::fabs(un - a), l2 = std::fabs(un), l4 = std::fabs(un + a);
  double D[4] = {0, 0, 0, 0};  // sum_k |lambda_k| alpha_k r_k
  // wave 1
  D[0] += l1 * al1;
  for (int d = 0; d < dim; ++d) D[1 + d] += l1 * al1 * (u[d] - (d == axis ? a : 0.0));
  D[c - 1] += l1 * al1 * (H - un * a);
  // wave 2 (entropy)
  D[0] += l2 * al2;
  for (int d = 0; d < dim; ++d) D[1 + d] += l2 * al2 * u[d];
  D[c - 1] += l2 * al2 * 0.5 * q2;
  // wave 3 (shear, 2D)
  if (dim == 2) {
    const double al3 = rho * (uR[t] - uL[t]);
    D[1 + t] += l2 * al3;
    D[c - 1] += l2 * al3 * u[t];
  }
  // wave 4
  D[0] += l4 * al4;
  for (int d = 0; d < dim; ++d) D[1 + d] += l4 * al4 * (u[d] + (d == axis ? a : 0.0));
  D[c - 1] += l4 * al4 * (H + un * a);
  for (int v = 0; v < c; ++v) F[v] = 0.5 * (FL[v] + FR[v]) - 0.5 * D[v];
  return 0;
}

}  // extern "C"

namespace {

// cell (i, j) of the grid including ghosts: transmissive / periodic through Grid::ix/iy; walls
// (bc 2) mirror the interior (ghost -1-m <-> cell m) with the normal momentum negated (A38)
void load_cell(const Grid& G, const double* q, int i, int j, double* U) {
  int ii = i, jj = j;
  bool flip_x = false, flip_y = false;
  if (G.bc == 2) {
    if (ii < 0) { ii = -1 - ii; flip_x = true; }
    if (ii >= G.nx) { ii = 2 * G.nx - 1 - ii; flip_x = true; }
    if (G.dim == 2) {
      if (jj < 0) { jj = -1 - jj; flip_y = true; }
      if (jj >= G.ny) { jj = 2 * G.ny - 1 - jj; flip_y = true; }
    } else {
      jj = 0;
    }
  } else {
    ii = G.ix(i);
    jj = G.iy(j);
  }
  const int64_t n = (int64_t)jj * G.nx + ii;
  for (int v = 0; v < G.c; ++v) U[v] = q[v * G.N + n];
  if (flip_x) U[1] = -U[1];
  if (flip_y) U[2] = -U[2];
}

// numerical flux through the face between (i, j) and the next cell along axis: MUSCL-minmod
// faces (conservative, component-wise, reading A3) then Rusanov (flux 0) or Roe (flux 1)
int face_flux2(const Grid& G, int flux, const double* q, int i, int j, int axis, double* F) {
  double Um1[4], U0[4], U1[4], U2[4], UL[4], UR[4];
  const int di = axis == 0 ? 1 : 0, dj = axis == 0 ? 0 : 1;
  load_cell(G, q, i, j, U0);
  load_cell(G, q, i + di, j + dj, U1);
  if (G.recon == 2) {
    load_cell(G, q, i - di, j - dj, Um1);
    load_cell(G, q, i + 2 * di, j + 2 * dj, U2);
  }
  for (int v = 0; v < G.c; ++v) {
    if (G.recon == 2) {
      double lf, rf;
      orc_muscl_faces(Um1[v], U0[v], U1[v], &lf, &rf);
      UL[v] = rf;
      orc_muscl_faces(U0[v], U1[v], U2[v], &lf, &rf);
      UR[v] = lf;
    } else {
      UL[v] = U0[v];
      UR[v] = U1[v];
    }
  }
  if (flux == 1) return orc_roe(G.dim, axis, G.gamma, UL, UR, F);
  orc_rusanov(G.dim, axis, G.gamma, UL, UR, F);
  return 0;
}

// f*(q) at cell (i, j): -(F_{i+1/2} - F_{i-1/2})/dx - (G_{j+1/2} - G_{j-1/2})/dy
int rhs_cell2(const Grid& G, int flux, const double* q, int i, int j, double* L) {
  double Fp[4], Fm[4];
  int bad = face_flux2(G, flux, q, i, j, 0, Fp);
  bad |= face_flux2(G, flux, q, i - 1, j, 0, Fm);
  for (int v = 0; v < G.c; ++v) L[v] = -(Fp[v] - Fm[v]) / G.dx;
  if (G.dim == 2) {
    double Gp[4], Gm[4];
    bad |= face_flux2(G, flux, q, i, j, 1, Gp);
    bad |= face_flux2(G, flux, q, i, j - 1, 1, Gm);
    for (int v = 0; v < G.c; ++v) L[v] = L[v] - (Gp[v] - Gm[v]) / G.dy;
  }
  return bad;
}

// BDF coefficients (A39): order 1 a = {-1}, beta = 1; order 2
// a = {1/3, -4/3} (for q_{k-2}, q_{k-1}), beta = 2/3
struct Bdf {
  int order;
  double a_m2, a_m1, beta;
  explicit Bdf(int s) : order(s) {
    if (s == 1) { a_m2 = 0.0; a_m1 = -1.0; beta = 1.0; }
    else { a_m2 = 1.0 / 3.0; a_m1 = -4.0 / 3.0; beta = 2.0 / 3.0; }
  }
};

// F_k(q) at cell n (all c variables): dt beta f*(q) - a_{s-1} q_{k-1} - a_{s-2} q_{k-2}
int Fk_cell(const Grid& G, int flux, const Bdf& B, double dt, const double* q, const double* qm1,
            const double* qm2, int64_t n, double* Fout) {
  const int i = (int)(n % G.nx), j = (int)(n / G.nx);
  double L[4];
  const int bad = rhs_cell2(G, flux, q, i, j, L);
  for (int v = 0; v < G.c; ++v) {
    const int64_t e = v * G.N + n;
    double h = B.a_m1 * qm1[e];
    if (B.order == 2) h = h + B.a_m2 * qm2[e];
    Fout[v] = dt * B.beta * L[v] - h;
  }
  return bad;
}

// the system R(q) = 0 on the rows of `cells` (all c variables of each), row r = v * nu + idx
struct Sys {
  const Grid& G;
  int flux;
  Bdf B;
  double dt;
  const double* qm1;
  const double* qm2;
  const std::vector<int64_t>& cells;
  int64_t nu;
  Sys(const Grid& g, int fl, int order, double d, const double* a, const double* b, const std::vector<int64_t>& cl)
      : G(g), flux(fl), B(order), dt(d), qm1(a), qm2(b), cells(cl), nu((int64_t)cl.size() * g.c) {}
  // R on the unknown rows of the state q (values outside `cells` are read as frozen data)
  bool residual(const double* q, std::vector<double>& R) const {
    R.resize(nu);
    const int64_t nc = (int64_t)cells.size();
    bool ok = true;
    for (int64_t idx = 0; idx < nc; ++idx) {
      const int64_t n = cells[idx];
      double F[4];
      if (Fk_cell(G, flux, B, dt, q, qm1, qm2, n, F)) ok = false;
      for (int v = 0; v < G.c; ++v) {
        const double r = q[v * G.N + n] - F[v];
        if (!std::isfinite(r)) ok = false;
        R[v * nc + idx] = r;
      }
    }
    return ok;
  }
  void gather(const double* q, std::vector<double>& x) const {
    const int64_t nc = (int64_t)cells.size();
    x.resize(nu);
    for (int v = 0; v < G.c; ++v)
      for (int64_t idx = 0; idx < nc; ++idx) x[v * nc + idx] = q[v * G.N + cells[idx]];
  }
  void scatter(const std::vector<double>& x, double* q) const {
    const int64_t nc = (int64_t)cells.size();
    for (int v = 0; v < G.c; ++v)
      for (int64_t idx = 0; idx < nc; ++idx) q[v * G.N + cells[idx]] = x[v * nc + idx];
  }
};

double norm2(const std::vector<double>& x) { return std::sqrt(dot(x.data(), x.data(), (int64_t)x.size())); }
double norm_inf(const std::vector<double>& x) {
  double m = 0.0;
  for (double v : x) m = std::max(m, std::fabs(v));
  return m;
}

// admissible state on the unknown cells (rho > 0, p > 0)
bool admissible(const Sys& S, const double* q) {
  for (int64_t n : S.cells) {
    double U[4];
    for (int v = 0; v < S.G.c; ++v) U[v] = q[v * S.G.N + n];
    if (!(U[0] > 0.0) || !(orc_pressure(S.G.dim, S.G.gamma, U) > 0.0)) return false;
  }
  return true;
}

// restarted GMRES(m) with modified Gram-Schmidt and Givens rotations for J x = b, J applied by
// the callback; x starts at 0; stops at ||b - J x||_2 <= rtol ||b||_2 or maxit products
template <class Op>
int gmres(const Op& J, const std::vector<double>& b, std::vector<double>& x, double rtol, int m, int maxit) {
  const int64_t n = (int64_t)b.size();
  x.assign(n, 0.0);
  const double bn = norm2(b);
  if (bn == 0.0) return 0;
  int its = 0;
  std::vector<double> r = b, w(n);
  while (its < maxit) {
    const double beta = norm2(r);
    if (beta <= rtol * bn) break;
    std::vector<std::vector<double>> V(1, std::vector<double>(n));
    for (int64_t i = 0; i < n; ++i) V[0][i] = r[i] / beta;
    std::vector<std::vector<double>> H(m + 1, std::vector<double>(m, 0.0));
    std::vector<double> cs(m), sn(m), g(m + 1, 0.0);
    g[0] = beta;
    int j = 0;
    for (; j < m && its < maxit; ++j, ++its) {
      J(V[j], w);
      for (int i = 0; i <= j; ++i) {  // modified Gram-Schmidt
        H[i][j] = dot(w.data(), V[i].data(), n);
        for (int64_t e = 0; e < n; ++e) w[e] -= H[i][j] * V[i][e];
      }
      H[j + 1][j] = norm2(w);
      V.emplace_back(n);
      if (H[j + 1][j] > 0.0)
        for (int64_t e = 0; e < n; ++e) V[j + 1][e] = w[e] / H[j + 1][j];
      for (int i = 0; i < j; ++i) {  // previous rotations
        const double t = cs[i] * H[i][j] + sn[i] * H[i + 1][j];
        H[i + 1][j] = -sn[i] * H[i][j] + cs[i] * H[i + 1][j];
        H[i][j] = t;
      }
      const double den = std::hypot(H[j][j], H[j + 1][j]);
      cs[j] = den > 0.0 ? H[j][j] / den : 1.0;
      sn[j] = den > 0.0 ? H[j + 1][j] / den : 0.0;
      H[j][j] = den;
      H[j + 1][j] = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      if (std::fabs(g[j + 1]) <= rtol * bn || H[j][j] == 0.0) {
        ++j;
        ++its;
        break;
      }
    }
    // back substitution of the j x j triangle, x += V y
    std::vector<double> y(j, 0.0);
    for (int i = j - 1; i >= 0; --i) {
      double s = g[i];
      for (int k = i + 1; k < j; ++k) s -= H[i][k] * y[k];
      y[i] = H[i][i] != 0.0 ? s / H[i][i] : 0.0;
    }
    for (int i = 0; i < j; ++i)
      for (int64_t e = 0; e < n; ++e) x[e] += y[i] * V[i][e];
    // true residual for the restart
    J(x, w);
    for (int64_t e = 0; e < n; ++e) r[e] = b[e] - w[e];
    if (j == 0) break;
  }
  return its;
}

}  // namespace

namespace orc {
int implicit_Fk_cell(const Grid& G, int flux, int order, double dt, const double* q, const double* qm1,
                     const double* qm2, int64_t n, double* F) {
  return Fk_cell(G, flux, Bdf(order), dt, q, qm1, qm2, n, F);
}
}  // namespace orc

extern "C" {

// f*(q) on every cell with the flux of `flux` (0 Rusanov, 1 Roe) and the grid's BCs (incl. walls)
int32_t orc_rhs2(const orc_grid* g, int32_t flux, const double* q, double* L) {
  Grid G(g);
  int32_t bad = 0;
  for (int j = 0; j < G.ny; ++j)
    for (int i = 0; i < G.nx; ++i) {
      double Lc[4];
      bad |= rhs_cell2(G, flux, q, i, j, Lc);
      for (int v = 0; v < G.c; ++v) L[v * G.N + (int64_t)j * G.nx + i] = Lc[v];
    }
  return bad;
}

// R_k(q) = q - F_k(q) on every cell; order 1 or 2; qm2 unused for order 1
void orc_bdf_residual(const orc_grid* g, int32_t flux, int32_t order, double dt, const double* q,
                      const double* qm1, const double* qm2, double* R) {
  Grid G(g);
  Bdf B(order);
  for (int64_t n = 0; n < G.N; ++n) {
    double F[4];
    Fk_cell(G, flux, B, dt, q, qm1, qm2, n, F);
    for (int v = 0; v < G.c; ++v) R[v * G.N + n] = q[v * G.N + n] - F[v];
  }
}

// Newton-Krylov solve of R_k(q) = 0 on the cells with mask[n] != 0 (mask NULL: every cell);
// q holds the initial guess on those cells and the frozen values elsewhere (only the stencil
// neighbours of the unknown cells are read).  Newton: J dq = -R by GMRES(30) (relative tol
// 1e-8, the accuracy of the difference products; J products by one-sided differences with h = sqrt(eps) (1 + ||q_u||_2) / ||v||_2),
// then q += lambda dq with lambda halved (<= 12 times) until the state is admissible and
// ||R||_2 decreases.  Stops when ||R||_inf <= tol.  Returns the Newton iterations, or -1
// (no convergence within maxit), -2 (non-admissible state / Roe average).
// stats (nullable): [0] final ||R||_inf, [1] total GMRES products.
int32_t orc_newton(const orc_grid* g, int32_t flux, int32_t order, double dt, const double* qm1,
                   const double* qm2, const uint8_t* mask, double* q, double tol, int32_t maxit,
                   double* stats) {
  Grid G(g);
  std::vector<int64_t> cells;
  for (int64_t n = 0; n < G.N; ++n)
    if (!mask || mask[n]) cells.push_back(n);
  Sys S(G, flux, order, dt, qm1, qm2, cells);
  std::vector<double> R, x, dq, Rt;
  if (!S.residual(q, R)) return -2;
  int64_t prods = 0;
  const double sq_eps = std::sqrt(std::numeric_limits<double>::epsilon());
  int it = 0;
  std::vector<double> work(q, q + G.D);
  for (;; ++it) {
    const double rinf = norm_inf(R);
    if (stats) stats[0] = rinf;
    if (rinf <= tol) break;
    if (it >= maxit) return -1;
    S.gather(q, x);
    const double xn = norm2(x);
    auto J = [&](const std::vector<double>& v, std::vector<double>& out) {
      const double vn = norm2(v);
      out.assign(v.size(), 0.0);
      if (vn == 0.0) return;
      const double h = sq_eps * (1.0 + xn) / vn;
      std::copy(q, q + G.D, work.begin());
      std::vector<double> xp(x.size());
      for (size_t e = 0; e < x.size(); ++e) xp[e] = x[e] + h * v[e];
      S.scatter(xp, work.data());
      S.residual(work.data(), Rt);
      for (size_t e = 0; e < v.size(); ++e) out[e] = (Rt[e] - R[e]) / h;
      ++prods;
    };
    std::vector<double> b(R.size());
    for (size_t e = 0; e < R.size(); ++e) b[e] = -R[e];
    gmres(J, b, dq, 1e-8, 30, 300);
    const double r0 = norm2(R);
    double lam = 1.0;
    bool accepted = false;
    for (int ls = 0; ls <= 12; ++ls, lam *= 0.5) {
      std::vector<double> xn2(x.size());
      for (size_t e = 0; e < x.size(); ++e) xn2[e] = x[e] + lam * dq[e];
      std::copy(q, q + G.D, work.begin());
      S.scatter(xn2, work.data());
      if (!admissible(S, work.data())) continue;
      if (!S.residual(work.data(), Rt)) continue;
      if (norm2(Rt) < r0 || ls == 12) {
        std::copy(work.begin(), work.end(), q);
        R = Rt;
        accepted = true;
        break;
      }
    }
    if (!accepted) return -2;
  }
  if (stats) stats[1] = (double)prods;
  return it;
}

}  // extern "C"
