// euler.cpp -- oracle: ideal-gas Euler finite volumes and the explicit HDM step.
// TEST INFRASTRUCTURE ONLY (see oracle.h).
//
// Paper: Euler equations P:674-691 (Eq. euler), ideal gas P:693-698, MUSCL +
// minmod P:701.  BASELINE.json replaces Roe by Rusanov (BJ:7-10, reading A2) and
// BDF2 by SSP-RK3 (reading A1; P:345-347 remark: explicit F_k is computed
// directly).  Conservative, component-wise limiting (reading A3).
#include <algorithm>
#include <cmath>
#include <limits>
#include "common.hpp"

using namespace orc;

extern "C" {

// O2: p = (gamma-1)(E - 1/2 (mx^2 + my^2)/rho)
double orc_pressure(int32_t dim, double gamma, const double* U) {
  double m2 = U[1] * U[1];
  if (dim == 2) m2 += U[2] * U[2];
  return (gamma - 1.0) * (U[dim + 1] - 0.5 * m2 / U[0]);
}

// O5: F(U) = (m_a, m_x u_a + p d_xa, m_y u_a + p d_ya, (E + p) u_a)
void orc_physical_flux(int32_t dim, int32_t axis, double gamma, const double* U, double* F) {
  const int c = dim + 2;
  const double p = orc_pressure(dim, gamma, U);
  const double ua = U[1 + axis] / U[0];
  F[0] = U[1 + axis];
  for (int d = 0; d < dim; ++d) F[1 + d] = U[1 + d] * ua + (d == axis ? p : 0.0);
  F[c - 1] = (U[c - 1] + p) * ua;
}

// minmod(a,b) = 0 if ab <= 0 else sign(a) min(|a|,|b|)
double orc_minmod(double a, double b) {
  if (a * b <= 0.0) return 0.0;
  return a > 0.0 ? std::min(a, b) : std::max(a, b);
}

// MUSCL faces of the middle cell: u0 -+ sigma/2, sigma = minmod(u0-um1, up1-u0)
void orc_muscl_faces(double um1, double u0, double up1, double* left_face, double* right_face) {
  const double s = orc_minmod(u0 - um1, up1 - u0);
  *left_face = u0 - 0.5 * s;
  *right_face = u0 + 0.5 * s;
}

// Rusanov: 1/2 (F(UL)+F(UR)) - 1/2 a (UR-UL), a = max(|u_L|+c_L, |u_R|+c_R)  (O5, A2)
void orc_rusanov(int32_t dim, int32_t axis, double gamma, const double* UL, const double* UR,
                 double* F) {
  const int c = dim + 2;
  double FL[4], FR[4];
  orc_physical_flux(dim, axis, gamma, UL, FL);
  orc_physical_flux(dim, axis, gamma, UR, FR);
  const double pL = orc_pressure(dim, gamma, UL), pR = orc_pressure(dim, gamma, UR);
  const double cL = std::sqrt(gamma * pL / UL[0]), cR = std::sqrt(gamma * pR / UR[0]);
  const double a = std::max(std::fabs(UL[1 + axis] / UL[0]) + cL,
                            std::fabs(UR[1 + axis] / UR[0]) + cR);
  for (int v = 0; v < c; ++v) F[v] = 0.5 * (FL[v] + FR[v]) - 0.5 * a * (UR[v] - UL[v]);
}

}  // extern "C"

namespace {

// load the conservative vector of cell (i, j) (already ghost-mapped)
inline void load(const Grid& G, const double* q, int i, int j, double* U) {
  const int64_t n = (int64_t)j * G.nx + i;
  for (int v = 0; v < G.c; ++v) U[v] = q[v * G.N + n];
}

// numerical flux through the face between cells (i, j) and the next cell along `axis`
// (x: (i+1, j); y: (i, j+1)).  Uses cells -1, 0, +1, +2 along the axis (O4).
void face_flux(const Grid& G, const double* q, int i, int j, int axis, double* F) {
  double Um1[4], U0[4], U1[4], U2[4], UL[4], UR[4];
  if (axis == 0) {
    load(G, q, G.ix(i), G.iy(j), U0);
    load(G, q, G.ix(i + 1), G.iy(j), U1);
    if (G.recon == 2) {
      load(G, q, G.ix(i - 1), G.iy(j), Um1);
      load(G, q, G.ix(i + 2), G.iy(j), U2);
    }
  } else {
    load(G, q, G.ix(i), G.iy(j), U0);
    load(G, q, G.ix(i), G.iy(j + 1), U1);
    if (G.recon == 2) {
      load(G, q, G.ix(i), G.iy(j - 1), Um1);
      load(G, q, G.ix(i), G.iy(j + 2), U2);
    }
  }
  for (int v = 0; v < G.c; ++v) {
    if (G.recon == 2) {
      double lf, rf;
      orc_muscl_faces(Um1[v], U0[v], U1[v], &lf, &rf);
      UL[v] = rf;  // right face of cell 0
      orc_muscl_faces(U0[v], U1[v], U2[v], &lf, &rf);
      UR[v] = lf;  // left face of cell +1
    } else {
      UL[v] = U0[v];
      UR[v] = U1[v];
    }
  }
  orc_rusanov(G.dim, axis, G.gamma, UL, UR, F);
}

// O6: L_n = -(F_{i+1/2} - F_{i-1/2})/dx - (G_{j+1/2} - G_{j-1/2})/dy
void rhs_cell(const Grid& G, const double* q, int i, int j, double* L) {
  double Fp[4], Fm[4];
  face_flux(G, q, i, j, 0, Fp);
  face_flux(G, q, i - 1, j, 0, Fm);
  for (int v = 0; v < G.c; ++v) L[v] = -(Fp[v] - Fm[v]) / G.dx;
  if (G.dim == 2) {
    double Gp[4], Gm[4];
    face_flux(G, q, i, j, 1, Gp);
    face_flux(G, q, i, j - 1, 1, Gm);
    for (int v = 0; v < G.c; ++v) L[v] = L[v] - (Gp[v] - Gm[v]) / G.dy;
  }
}

enum Stage { S1, S2, S3 };

// one SSP-RK3 stage at one cell, expressions in the printed order (O8)
void stage_cell(const Grid& G, Stage st, const double* qn, const double* qin, double dt,
                int i, int j, double* out) {
  double L[4];
  rhs_cell(G, qin, i, j, L);
  const int64_t n = (int64_t)j * G.nx + i;
  for (int v = 0; v < G.c; ++v) {
    const int64_t e = v * G.N + n;
    if (st == S1) out[e] = qn[e] + dt * L[v];
    else if (st == S2) out[e] = 0.75 * qn[e] + 0.25 * (qin[e] + dt * L[v]);
    else out[e] = (1.0 / 3.0) * qn[e] + (2.0 / 3.0) * (qin[e] + dt * L[v]);
  }
}

}  // namespace

extern "C" {

void orc_rhs(const orc_grid* g, const double* q, double* L) {
  Grid G(g);
  for (int j = 0; j < G.ny; ++j)
    for (int i = 0; i < G.nx; ++i) {
      double Lc[4];
      rhs_cell(G, q, i, j, Lc);
      for (int v = 0; v < G.c; ++v) L[v * G.N + (int64_t)j * G.nx + i] = Lc[v];
    }
}

// H1 / O7 (reading A4): dt = CFL / max_n [(|u|+c)/dx + (|v|+c)/dy] over all cells
double orc_dt(const orc_grid* g, const double* q) {
  Grid G(g);
  double smax = 0.0;
  for (int64_t n = 0; n < G.N; ++n) {
    double U[4];
    for (int v = 0; v < G.c; ++v) U[v] = q[v * G.N + n];
    const double p = orc_pressure(G.dim, G.gamma, U);
    const double cs = std::sqrt(G.gamma * p / U[0]);
    double s = (std::fabs(U[1] / U[0]) + cs) / G.dx;
    if (G.dim == 2) s = s + (std::fabs(U[2] / U[0]) + cs) / G.dy;
    if (!(s <= smax)) smax = s;  // NaN propagates as "largest"
  }
  return G.cfl / smax;
}

// O2/O11: lowest cell with rho <= 0 or p <= 0 (or NaN), else -1
int64_t orc_positivity(const orc_grid* g, const double* q) {
  Grid G(g);
  for (int64_t n = 0; n < G.N; ++n) {
    double U[4];
    for (int v = 0; v < G.c; ++v) U[v] = q[v * G.N + n];
    const double p = orc_pressure(G.dim, G.gamma, U);
    if (!(U[0] > 0.0) || !(p > 0.0)) return n;
  }
  return -1;
}

// H2 / O8-O9: full SSP-RK3 step on all cells
void orc_full_step(const orc_grid* g, const double* q, double dt, double* out) {
  Grid G(g);
  std::vector<double> U1(G.D), U2(G.D);
  for (int j = 0; j < G.ny; ++j)
    for (int i = 0; i < G.nx; ++i) stage_cell(G, S1, q, q, dt, i, j, U1.data());
  for (int j = 0; j < G.ny; ++j)
    for (int i = 0; i < G.nx; ++i) stage_cell(G, S2, q, U1.data(), dt, i, j, U2.data());
  for (int j = 0; j < G.ny; ++j)
    for (int i = 0; i < G.nx; ++i) stage_cell(G, S3, q, U2.data(), dt, i, j, out);
}

// H3 / O10.1 (reading A9): stage 1 on A1, stage 2 on A2, stage 3 on T, with
// A2 = T (+) C_h, A1 = A2 (+) C_h.  Values outside a stage's set are NaN, so a
// dilation that is too small shows up as NaN on T.
void orc_masked_step(const orc_grid* g, const double* q, double dt, const uint8_t* mask_T,
                     int32_t h, double* out) {
  Grid G(g);
  std::vector<uint8_t> A2(G.N), A1(G.N);
  orc_dilate_cross(g, mask_T, h, A2.data());
  orc_dilate_cross(g, A2.data(), h, A1.data());
  const double nan = std::numeric_limits<double>::quiet_NaN();
  std::vector<double> U1(G.D, nan), U2(G.D, nan);
  for (int64_t e = 0; e < G.D; ++e) out[e] = nan;
  for (int j = 0; j < G.ny; ++j)
    for (int i = 0; i < G.nx; ++i)
      if (A1[(int64_t)j * G.nx + i]) stage_cell(G, S1, q, q, dt, i, j, U1.data());
  for (int j = 0; j < G.ny; ++j)
    for (int i = 0; i < G.nx; ++i)
      if (A2[(int64_t)j * G.nx + i]) stage_cell(G, S2, q, U1.data(), dt, i, j, U2.data());
  for (int j = 0; j < G.ny; ++j)
    for (int i = 0; i < G.nx; ++i)
      if (mask_T[(int64_t)j * G.nx + i]) stage_cell(G, S3, q, U2.data(), dt, i, j, out);
}

}  // extern "C"
