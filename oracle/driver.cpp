// driver.cpp -- oracle: Algorithm 1, explicit variant, full-HDM period z.
// TEST INFRASTRUCTURE ONLY (see oracle.h).
//
// Schedule: full steps for k+1 <= w or k mod z = 0 (z = infinity by default, A20);
// hybrid steps otherwise.
// Refresh after every step k >= w-1 with (k+1) mod z != 0:
//   G_{k+1} from the indicator (fraction mode A18; bootstrap A19 at k = w-1;
//   after a full step k >= w the same projection rule with Phi_{k+1}, psi_{k+1}, reading G8),
//   Phi_{k+1} = POD_r([gamma_{k-w+1} - psi_k, ..., gamma_k - psi_k])   (lagged A14)
//   psi_{k+1} = mean(gamma_{k-w+1..k})
// Hybrid step k (O10-O13):
//   masked RK3 on S-hat (and the band, for F) -> gappy y (Eq. 8, P = S-hat, A11)
//   -> fill the complement with psi + Phi y -> indicator (A16/A17)
//   -> seam filter (A21-A24) -> indicator on kept cells.
#include <algorithm>
#include <cmath>
#include <deque>
#include <limits>
#include <vector>
#include "common.hpp"

using namespace orc;

struct orc_run {
  orc_grid g;
  orc_params p;
  Grid G;
  int64_t k = 0;
  std::deque<std::vector<double>> snaps;  // gamma_{k-w}..gamma_k (at most w+1)
  std::vector<double> Phi, psi;           // Phi_{k+1} (D x reff), psi_{k+1}
  std::vector<double> sigma;
  int32_t reff = 0;
  std::vector<uint8_t> mask_next, mask_used;
  std::vector<double> eps, y;
  int32_t ny_last = 0;
  double dt = 0.0;
  int64_t kept = 0;
  int32_t sweeps[3] = {0, 0, 0};
  int32_t z = 0;  // full-HDM period; <= 0: infinity
  double delta = 0.0;  // > 0: RRE-delta selection instead of the fraction f
  int32_t odeim_np = 0;  // > 0: S-hat = G u ODEIM points, gappy rows = the points' DOF rows (Eq. 8, 10)
  std::vector<int64_t> prow, prow_next;  // ODEIM DOF rows used by / chosen for the next step
  // NEXT-4: the paper's implicit HDM (BDF2 + MUSCL/Roe, Newton-Krylov) with partial-HDM
  // subiterations; fixed dt
  int32_t imp = 0, flux = 1, jmax = 10, nmaxit = 30;
  double imp_dt = 0.0, eps_y = 1e-4, ntol = 1e-12;
  int32_t J_last = 0;
  int64_t newton_its = 0;
  int32_t imp_fail = 0;
  orc_run(const orc_grid* gg, const orc_params* pp) : g(*gg), p(*pp), G(gg) {}
};

namespace {

std::vector<double> mean_of(const std::deque<std::vector<double>>& s, size_t first, size_t count,
                            int64_t D) {
  std::vector<double> m(D, 0.0);
  for (int64_t e = 0; e < D; ++e) {
    double acc = 0.0;
    for (size_t t = first; t < first + count; ++t) acc += s[t][e];
    m[e] = acc / (double)count;
  }
  return m;
}

// Phi_{k+1}, psi_{k+1}, S from the current window (O14).  `lagged` = psi_k.
void refresh_basis(orc_run* R, const std::vector<double>& psi_k) {
  const int w = R->p.w;
  const int64_t D = R->G.D;
  const size_t ns = R->snaps.size();
  // X = [gamma_{k-w+1} - psi_k, ..., gamma_k - psi_k]: the last w snapshots
  std::vector<double> X((int64_t)w * D);
  for (int j = 0; j < w; ++j) {
    const auto& s = R->snaps[ns - w + j];
    for (int64_t e = 0; e < D; ++e) X[(int64_t)j * D + e] = s[e] - psi_k[e];
  }
  const int r = std::min(R->p.r, w);
  R->Phi.assign((int64_t)r * D, 0.0);
  R->sigma.assign(w, 0.0);
  std::vector<double> V((int64_t)w * w);
  R->reff = orc_pod(X.data(), D, w, r, R->p.eig_rel_cutoff, R->Phi.data(), R->sigma.data(), V.data());
  R->Phi.resize((int64_t)R->reff * D);
  R->psi = mean_of(R->snaps, ns - w, w, D);
}

// S-hat_{k+1} from eps: the fraction rule (A18) or, when set, the RRE-delta rule
// With ODEIM (NEXT-1): S-hat_{k+1} = G_{k+1} u P_{k+1}, P_{k+1} = ODEIM(Phi_{k+1}).
void select_next(orc_run* R) {
  const int64_t N = R->g.nx * (int64_t)R->g.ny;
  if (R->delta > 0.0) orc_select_rre(R->eps.data(), N, R->delta, R->mask_next.data());
  else orc_select(R->eps.data(), N, orc_n_g(R->p.f, N), R->mask_next.data());
  R->prow_next.clear();
  if (R->odeim_np > 0 && R->reff > 0) {
    const int32_t np = (int32_t)std::min<int64_t>(R->odeim_np, N);
    std::vector<int32_t> cells(np);
    R->prow_next.resize(np);
    orc_odeim(R->Phi.data(), R->G.D, R->reff, N, np, R->p.lsq_rel_cutoff, cells.data(), R->prow_next.data());
    for (int32_t q = 0; q < np; ++q) R->mask_next[cells[q]] = 1;
  }
}

void reconstruct(const orc_run* R, const std::vector<double>& y, int64_t n, double* out) {
  // out[v] = psi[v,n] + sum_i Phi[v*N+n, i] y_i
  const int64_t N = R->G.N, D = R->G.D;
  for (int v = 0; v < R->G.c; ++v) {
    const int64_t e = v * N + n;
    double acc = 0.0;
    for (int i = 0; i < R->reff; ++i) acc += R->Phi[(int64_t)i * D + e] * y[i];
    out[v] = R->psi[e] + acc;
  }
}

// eps_n = sum_v [(I - Phi_{k+1} Phi_{k+1}^T)(gamma_k - psi_{k+1})]^2_{v,n}: the projection
// error of the newest snapshot on the basis just built (A19 at k = w-1; G8 after full steps)
void projection_indicator(orc_run* R) {
  const int64_t N = R->G.N, D = R->G.D;
  std::vector<double> d(D);
  const auto& last = R->snaps.back();
  for (int64_t e = 0; e < D; ++e) d[e] = last[e] - R->psi[e];
  for (int i = 0; i < R->reff; ++i) {
    const double c = dot(R->Phi.data() + (int64_t)i * D, d.data(), D);
    for (int64_t e = 0; e < D; ++e) d[e] -= c * R->Phi[(int64_t)i * D + e];
  }
  for (int64_t n = 0; n < N; ++n) {
    double e2 = 0.0;
    for (int v = 0; v < R->G.c; ++v) e2 += d[v * N + n] * d[v * N + n];
    R->eps[n] = e2;
  }
}

// the least-squares coordinates y = (P^T Phi)^+ P^T (v - psi) on the rows erows (Eq. 8)
std::vector<double> gappy_y(const orc_run* R, const std::vector<int64_t>& erows, const double* v) {
  const int64_t m = (int64_t)erows.size(), D = R->G.D;
  const int reff = R->reff;
  std::vector<double> A(m * (int64_t)reff), b(m), y(reff, 0.0);
  for (int64_t row = 0; row < m; ++row) {
    const int64_t e = erows[row];
    b[row] = v[e] - R->psi[e];
    for (int i = 0; i < reff; ++i) A[(int64_t)i * m + row] = R->Phi[(int64_t)i * D + e];
  }
  orc_lsq(A.data(), m, reff, b.data(), R->p.lsq_rel_cutoff, y.data());
  return y;
}

// NEXT-4 hybrid step k (Algorithm 1 lines 7-14, with the subiterations of
// P:317-343): the partial HDM on S-hat with S-tilde = Neighbors(S-hat) frozen (Eq. 6b,
// P:238-245), y from the P rows (Eq. 8), S-tilde refreshed from psi + Phi y, until
// ||y^(j+1) - y^(j)||_2 < eps_y or j = j_max (reading A41: the test needs two iterates, so
// J >= 2 unless j_max = 1); then the fill, the indicator and the filter gated by
// the implicit residual.  Returns 1, or -1 when a partial Newton solve failed.
int implicit_hybrid(orc_run* R, int order, const double* qm1, const double* qm2, std::vector<double>& gam) {
  const Grid& G = R->G;
  const int64_t N = G.N, D = G.D;
  const std::vector<uint8_t>& S = R->mask_next;
  R->mask_used = S;
  std::vector<uint8_t> dil(N), St(N);
  orc_dilate_cross(&R->g, S.data(), R->p.h, dil.data());
  for (int64_t n = 0; n < N; ++n) St[n] = (dil[n] && !S[n]) ? 1 : 0;
  // working state: S-hat u S-tilde from gamma_{k-1} (Alg. 1 line 7); every other entry NaN,
  // so a stencil that reaches past S-tilde shows up as a failed solve
  const double nan = std::numeric_limits<double>::quiet_NaN();
  std::vector<double> v(D, nan);
  for (int64_t n = 0; n < N; ++n)
    if (S[n] || St[n])
      for (int c = 0; c < G.c; ++c) v[c * N + n] = qm1[c * N + n];
  std::vector<int64_t> erows;
  R->prow = R->prow_next;
  if (R->odeim_np > 0) {
    erows = R->prow;
  } else {
    for (int64_t n = 0; n < N; ++n)
      if (S[n])
        for (int c = 0; c < G.c; ++c) erows.push_back(c * N + n);
  }
  std::vector<double> y, yprev;
  int J = 0;
  for (int j = 1; j <= R->jmax; ++j) {
    const int its = orc_newton(&R->g, R->flux, order, R->imp_dt, qm1, qm2, S.data(), v.data(), R->ntol,
                               R->nmaxit, nullptr);
    if (its < 0) return -1;
    R->newton_its += its;
    y = gappy_y(R, erows, v.data());
    J = j;
    if (j > 1) {
      double d2 = 0.0;
      for (size_t i = 0; i < y.size(); ++i) d2 += (y[i] - yprev[i]) * (y[i] - yprev[i]);
      if (std::sqrt(d2) < R->eps_y) break;
    }
    if (j == R->jmax) break;
    for (int64_t n = 0; n < N; ++n)
      if (St[n]) {
        double rec[4];
        reconstruct(R, y, n, rec);
        for (int c = 0; c < G.c; ++c) v[c * N + n] = rec[c];
      }
    yprev = y;
  }
  R->J_last = J;
  R->y = y;
  R->ny_last = R->reff;
  std::fill(R->eps.begin(), R->eps.end(), 0.0);
  for (int64_t n = 0; n < N; ++n) {
    double rec[4];
    reconstruct(R, y, n, rec);
    if (S[n]) {
      double e2 = 0.0;
      for (int c = 0; c < G.c; ++c) {
        gam[c * N + n] = v[c * N + n];
        const double d = v[c * N + n] - rec[c];
        e2 += d * d;
      }
      R->eps[n] = e2;
    } else {
      for (int c = 0; c < G.c; ++c) gam[c * N + n] = rec[c];
    }
  }
  std::vector<uint8_t> kept(N, 0);
  R->kept = orc_seam_filter_implicit(&R->g, &R->p, R->flux, order, R->imp_dt, qm1, qm2, gam.data(), S.data(),
                                     kept.data(), R->sweeps);
  for (int64_t n = 0; n < N; ++n)
    if (kept[n]) {
      double rec[4];
      reconstruct(R, y, n, rec);
      double e2 = 0.0;
      for (int c = 0; c < G.c; ++c) {
        const double d = gam[c * N + n] - rec[c];
        e2 += d * d;
      }
      R->eps[n] = e2;
    }
  return 1;
}

// full implicit HDM step (Alg. 1 line 4): Newton from gamma_{k-1}; -1 on failure
int implicit_full(orc_run* R, int order, const double* qm1, const double* qm2, std::vector<double>& gam) {
  std::copy(qm1, qm1 + R->G.D, gam.begin());
  const int its = orc_newton(&R->g, R->flux, order, R->imp_dt, qm1, qm2, nullptr, gam.data(), R->ntol,
                             R->nmaxit, nullptr);
  if (its < 0) return -1;
  R->newton_its += its;
  return 0;
}

}  // namespace

extern "C" {

orc_run* orc_run_create(const orc_grid* g, const orc_params* p, const double* q0) {
  auto* R = new orc_run(g, p);
  R->snaps.emplace_back(q0, q0 + R->G.D);
  R->mask_next.assign(R->G.N, 0);
  R->mask_used.assign(R->G.N, 0);
  R->eps.assign(R->G.N, 0.0);
  return R;
}

void orc_run_destroy(orc_run* R) { delete R; }

int32_t orc_run_step(orc_run* R, double dt_override) {
  const Grid& G = R->G;
  const int w = R->p.w;
  const int64_t N = G.N, D = G.D;
  const int64_t k = R->k + 1;
  const std::vector<double>& prev = R->snaps.back();
  std::vector<double> gam(D);
  int32_t kind = 0;
  if (R->imp) {
    // NEXT-4: BDF1 at k = 1, BDF2 afterwards (A39); fixed dt
    R->dt = R->imp_dt;
    const int order = (k == 1 || R->snaps.size() < 2) ? 1 : 2;
    const double* qm1 = prev.data();
    const double* qm2 = order == 2 ? R->snaps[R->snaps.size() - 2].data() : prev.data();
    R->J_last = 0;
    if (k + 1 <= w || (R->z > 0 && k % R->z == 0)) {
      std::fill(R->mask_used.begin(), R->mask_used.end(), 1);
      if (implicit_full(R, order, qm1, qm2, gam) < 0) { R->imp_fail = 1; return -1; }
    } else {
      kind = implicit_hybrid(R, order, qm1, qm2, gam);
      if (kind < 0 || orc_positivity(&R->g, gam.data()) >= 0) {  // escalation
        if (implicit_full(R, order, qm1, qm2, gam) < 0) { R->imp_fail = 1; return -1; }
        kind = 2;
      }
    }
  } else {
  R->dt = (dt_override > 0.0) ? dt_override : orc_dt(&R->g, prev.data());
  if (k + 1 <= w || (R->z > 0 && k % R->z == 0)) {
    orc_full_step(&R->g, prev.data(), R->dt, gam.data());
    std::fill(R->mask_used.begin(), R->mask_used.end(), 1);
  } else {
    kind = 1;
    const std::vector<uint8_t>& S = R->mask_next;
    R->mask_used = S;
    // band B = (S (+) Q_W) \ S; the masked step runs on T = S u B (O10.1)
    std::vector<uint8_t> sq(N), T(N);
    orc_dilate_square(&R->g, S.data(), R->p.W, sq.data());
    for (int64_t n = 0; n < N; ++n) T[n] = (S[n] || sq[n]) ? 1 : 0;
    std::vector<double> F(D);
    orc_masked_step(&R->g, prev.data(), R->dt, T.data(), R->p.h, F.data());
    // gappy coordinates on the rows of S-hat (Eq. 8 with P = S-hat, A11, A12), or on the DOF
    // rows of the ODEIM points (Eq. 8 with P = ODEIM(Phi_k))
    std::vector<int64_t> erows;
    R->prow = R->prow_next;
    if (R->odeim_np > 0) {
      erows = R->prow;
    } else {
      for (int64_t n = 0; n < N; ++n)
        if (S[n])
          for (int v = 0; v < G.c; ++v) erows.push_back(v * N + n);
    }
    const int64_t m = (int64_t)erows.size();
    const int reff = R->reff;
    std::vector<double> A(m * (int64_t)reff), b(m);
    for (int64_t row = 0; row < m; ++row) {
      const int64_t e = erows[row];
      b[row] = F[e] - R->psi[e];
      for (int i = 0; i < reff; ++i) A[(int64_t)i * m + row] = R->Phi[(int64_t)i * D + e];
    }
    R->y.assign(reff, 0.0);
    orc_lsq(A.data(), m, reff, b.data(), R->p.lsq_rel_cutoff, R->y.data());
    R->ny_last = reff;
    // assemble gamma_k: S-hat rows from the partial HDM, the rest psi + Phi y
    std::fill(R->eps.begin(), R->eps.end(), 0.0);
    for (int64_t n = 0; n < N; ++n) {
      double rec[4];
      reconstruct(R, R->y, n, rec);
      if (S[n]) {
        double e2 = 0.0;
        for (int v = 0; v < G.c; ++v) {
          gam[v * N + n] = F[v * N + n];
          const double d = F[v * N + n] - rec[v];
          e2 += d * d;
        }
        R->eps[n] = e2;  // P:363, summed over the cell's c variables (A16)
      } else {
        for (int v = 0; v < G.c; ++v) gam[v * N + n] = rec[v];
      }
    }
    // seam filter, F valid on the band
    std::vector<uint8_t> kept(N, 0);
    R->kept = orc_seam_filter(&R->g, &R->p, gam.data(), F.data(), S.data(), kept.data(), R->sweeps);
    for (int64_t n = 0; n < N; ++n)
      if (kept[n]) {
        double rec[4];
        reconstruct(R, R->y, n, rec);
        double e2 = 0.0;
        for (int v = 0; v < G.c; ++v) {
          const double d = gam[v * N + n] - rec[v];
          e2 += d * d;
        }
        R->eps[n] = e2;
      }
    if (orc_positivity(&R->g, gam.data()) >= 0) {  // O11 escalation
      orc_full_step(&R->g, prev.data(), R->dt, gam.data());
      kind = 2;
    }
  }
  }  // explicit
  R->snaps.push_back(std::move(gam));
  while ((int)R->snaps.size() > w + 1) R->snaps.pop_front();
  R->k = k;
  if (R->z > 0 && (k + 1) % R->z == 0) return kind;  // no refresh before a full step
  if (k == w - 1) {
    // offset bootstrap: psi_{w-1} = mean(gamma_0..gamma_{w-1})
    const std::vector<double> psi0 = mean_of(R->snaps, R->snaps.size() - w, w, D);
    refresh_basis(R, psi0);
    if (R->odeim_np > 0) {
      // Algorithm 1: G_w = {} at k = w-1, so S-hat_w = P_w (the ODEIM points only)
      std::fill(R->eps.begin(), R->eps.end(), 0.0);
    } else {
      projection_indicator(R);  // bootstrap indicator (A19: P = S-hat mode, where P_w is empty)
    }
    select_next(R);
  } else if (k >= w) {
    // psi_k = mean(gamma_{k-w..k-1}) (lagged centring, A14; by its formula also
    // when the refresh after step k-1 was skipped, reading G8)
    const std::vector<double> psik = mean_of(R->snaps, 0, w, D);
    refresh_basis(R, psik);
    if (kind == 0) projection_indicator(R);  // after a full step (finite z): reading G8
    select_next(R);
  }
  return kind;
}

void orc_run_set_full_period(orc_run* R, int32_t z) { R->z = z; }
void orc_run_set_rre(orc_run* R, double delta) { R->delta = delta; }
void orc_run_set_odeim(orc_run* R, int32_t n_p) { R->odeim_np = n_p; }
void orc_run_set_implicit(orc_run* R, int32_t flux, double dt, double eps_y, int32_t j_max, double newton_tol,
                          int32_t newton_maxit) {
  R->imp = 1;
  R->flux = flux;
  R->imp_dt = dt;
  R->eps_y = eps_y;
  R->jmax = j_max;
  R->ntol = newton_tol;
  R->nmaxit = newton_maxit;
}
void orc_run_implicit_stats(const orc_run* R, int32_t* J_last, int64_t* newton_its) {
  *J_last = R->J_last;
  *newton_its = R->newton_its;
}
int32_t orc_run_points(const orc_run* R, int64_t* rows) {
  std::copy(R->prow_next.begin(), R->prow_next.end(), rows);
  return (int32_t)R->prow_next.size();
}

int64_t orc_run_k(const orc_run* R) { return R->k; }
void orc_run_state(const orc_run* R, double* q) { std::copy(R->snaps.back().begin(), R->snaps.back().end(), q); }
void orc_run_mask(const orc_run* R, uint8_t* m) { std::copy(R->mask_next.begin(), R->mask_next.end(), m); }
void orc_run_mask_used(const orc_run* R, uint8_t* m) { std::copy(R->mask_used.begin(), R->mask_used.end(), m); }
void orc_run_eps(const orc_run* R, double* e) { std::copy(R->eps.begin(), R->eps.end(), e); }
int32_t orc_run_reff(const orc_run* R) { return R->reff; }
void orc_run_basis(const orc_run* R, double* Phi) { std::copy(R->Phi.begin(), R->Phi.end(), Phi); }
void orc_run_psi(const orc_run* R, double* psi) { std::copy(R->psi.begin(), R->psi.end(), psi); }
void orc_run_sigma(const orc_run* R, double* S) { std::copy(R->sigma.begin(), R->sigma.end(), S); }
int32_t orc_run_y(const orc_run* R, double* y) {
  std::copy(R->y.begin(), R->y.end(), y);
  return (int32_t)R->y.size();
}
double orc_run_dt(const orc_run* R) { return R->dt; }
void orc_run_filter_stats(const orc_run* R, int64_t* kept, int32_t* sweeps) {
  *kept = R->kept;
  for (int i = 0; i < 3; ++i) sweeps[i] = R->sweeps[i];
}

void orc_run_set_window(orc_run* R, int64_t k, const double* snaps, int32_t nsnaps,
                        const uint8_t* mask_next) {
  const int64_t D = R->G.D;
  R->snaps.clear();
  for (int t = 0; t < nsnaps; ++t) R->snaps.emplace_back(snaps + (int64_t)t * D, snaps + (int64_t)(t + 1) * D);
  R->k = k;
  const int w = R->p.w;
  const std::vector<double> psik = mean_of(R->snaps, 0, w, D);  // gamma_{k-w..k-1}
  refresh_basis(R, psik);
  std::copy(mask_next, mask_next + R->G.N, R->mask_next.begin());
  // with ODEIM the given mask is G_{k+1}: add the points of Phi_{k+1} (as select_next does)
  R->prow_next.clear();
  if (R->odeim_np > 0 && R->reff > 0) {
    const int32_t np = (int32_t)std::min<int64_t>(R->odeim_np, R->G.N);
    std::vector<int32_t> cells(np);
    R->prow_next.resize(np);
    orc_odeim(R->Phi.data(), D, R->reff, R->G.N, np, R->p.lsq_rel_cutoff, cells.data(), R->prow_next.data());
    for (int32_t q = 0; q < np; ++q) R->mask_next[cells[q]] = 1;
  }
}

}  // extern "C"
