/* oracle.h -- C shim of the CPU oracle for the hybrid-snapshot step.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load liboracle.so.  The product path
 * (paper_2301_01718_b200, libhrom.so) never includes, links or calls this code,
 * and this code shares nothing with it.
 *
 * A plain, slow, single-threaded fp64 C++17 implementation written from
 * /root/reference/PAPER.md (cited "P:<line>") with the readings of DESIGN.md §3
 * (SURVEY.md §8(c) A1-A34).  No BLAS/LAPACK, no blocking, no fusion; long sums
 * are Neumaier-compensated.  Built with g++ -O2 -ffp-contract=off.
 *
 * Layout everywhere: SoA q[v*N + n], n = j*nx + i; matrices column-major.
 * Masks are uint8 per cell (0/1).
 *
 * Parity status: every function below is pinned by tests/test_oracle_*.py
 * except orc_run_* trajectories, whose end-to-end values are "parity unpinned"
 * against the paper (no explicit-path numbers exist); they
 * are pinned only through the invariants of their parts.
 */
#ifndef HROM_ORACLE_H
#define HROM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t dim, nx, ny;
  double x0, x1, y0, y1;
  int32_t bc;     /* 0 transmissive (zeroth-order ghost), 1 periodic */
  int32_t recon;  /* 1 first order, 2 MUSCL-minmod */
  double gamma, cfl;
} orc_grid;

typedef struct {
  int32_t w, r, h, W;
  double f;
  int32_t filter_orders[3];
  int32_t n_filter_orders;
  int32_t filter_max_sweeps;
  double filter_eps;
  double eig_rel_cutoff;  /* 1e-8 on sigma^2 (A15) */
  double lsq_rel_cutoff;  /* 1e-12 on sigma^2 (A13) */
} orc_params;

/* ---- EOS / flux / RHS (Eq. euler; BJ:7-10 Rusanov) ---- */
double orc_pressure(int32_t dim, double gamma, const double* U);
void orc_physical_flux(int32_t dim, int32_t axis, double gamma, const double* U, double* F);
double orc_minmod(double a, double b);
void orc_muscl_faces(double um1, double u0, double up1, double* left_face, double* right_face);
void orc_rusanov(int32_t dim, int32_t axis, double gamma, const double* UL, const double* UR, double* F);
void orc_rhs(const orc_grid* g, const double* q, double* L);
double orc_dt(const orc_grid* g, const double* q);
int64_t orc_positivity(const orc_grid* g, const double* q); /* lowest bad cell or -1 */

/* ---- explicit HDM step F_k (P:179-189 Eq. hdm, P:345-347 remark) ---- */
void orc_full_step(const orc_grid* g, const double* q, double dt, double* out);
/* masked step (Eq. 6b/7, reading A9): stage 1 on A1, 2 on A2, 3 on T (mask_T).
 * Entries outside T are NaN on output. */
void orc_masked_step(const orc_grid* g, const double* q, double dt, const uint8_t* mask_T,
                     int32_t h, double* out);

/* ---- sampling sets ---- */
void orc_dilate_cross(const orc_grid* g, const uint8_t* in, int32_t h, uint8_t* out);
void orc_dilate_square(const orc_grid* g, const uint8_t* in, int32_t W, uint8_t* out);
/* top-n_g of eps>0, ties by ascending index (A18). returns |G|. */
int64_t orc_select(const double* eps, int64_t N, int64_t n_g, uint8_t* mask_out);
int64_t orc_n_g(double f, int64_t N); /* ceil(f*N) */
/* RRE-delta rule (P:373-380 Eq. rre), used by the NEXT-1 pins */
int64_t orc_select_rre(const double* eps, int64_t N, double delta, uint8_t* mask_out);
/* ODEIM_{n_p} points (Eq. 10; reading A36, greedy DEIM-and-continue of S:279/S:295):
 * Phi D x m col-major, DOF e in cell e mod N; cells_out[n_p], rows_out[n_p] (the DOF rows).
 * Returns n_p, -1 on bad arguments (n_p > N). */
int32_t orc_odeim(const double* Phi, int64_t D, int32_t m, int64_t N, int32_t n_p, double cut,
                  int32_t* cells_out, int64_t* rows_out);

/* ---- dense linear algebra (Eq. 8, Eq. 9) ---- */
/* min-norm LSQ: x = A^+ b discarding sigma_i^2 < cut*sigma_1^2. A m x n col-major.
 * returns numerical rank. */
int32_t orc_lsq(const double* A, int64_t m, int32_t n, const double* b, double cut, double* x);
/* thin SVD via Householder QR + one-sided Jacobi (descending). X is m x n col-major.
 * U: m x n (may be NULL), S: n, V: n x n. sign: largest |V_ij| of each column positive. */
void orc_svd(const double* X, int64_t m, int32_t n, double* U, double* S, double* V);
/* POD_r: Phi = leading r_eff left singular vectors; r_eff per A15. */
int32_t orc_pod(const double* X, int64_t m, int32_t w, int32_t r, double cut,
                double* Phi, double* S, double* V);

/* Gram of shifted columns: C_ij = sum_e (S_ie - rho_e)(S_je - rho_e), S: ncol x rows
 * (row-major per column), rho nullable.  The snapshot Gram of the POD remark P:634. */
void orc_gram(const double* S, int32_t ncol, int64_t rows, const double* rho, double* C);
/* C = Phi^T S (m x ncol, row-major) over D rows, compensated sums (config-5 projection op) */
void orc_project(const double* Phi, int64_t D, int32_t m, const double* S, int32_t ncol, double* C);

/* ---- Shapiro filters and seam filter (A21-A24) ---- */
void orc_shapiro_1d(const double* line, int32_t n, int32_t order, int32_t periodic, double* out);
/* seam filter on band B = (S (+) Q_W) \ S. v is updated in place (SoA state).
 * F: full-step values (valid on B). kept_out (uint8 N, may be NULL): cells ever kept.
 * sweeps_out[3]: sweeps performed per order. returns number of cells ever kept. */
int64_t orc_seam_filter(const orc_grid* g, const orc_params* p, double* v, const double* F,
                        const uint8_t* mask_S, uint8_t* kept_out, int32_t* sweeps_out);

/* ---- Algorithm 1, explicit variant (O1-O16), z = infinity unless set ---- */
typedef struct orc_run orc_run;
orc_run* orc_run_create(const orc_grid* g, const orc_params* p, const double* q0);
void orc_run_destroy(orc_run* R);
/* one step k -> k+1.  dt_override <= 0 uses the CFL rule.  returns 0 full, 1 hybrid,
 * 2 hybrid escalated to full (positivity). */
int32_t orc_run_step(orc_run* R, double dt_override);
/* full-HDM period z of Algorithm 1; <= 0: infinity (the default) */
void orc_run_set_full_period(orc_run* R, int32_t z);
void orc_run_set_rre(orc_run* R, double delta);  /* > 0: RRE-delta sampling */
void orc_run_set_odeim(orc_run* R, int32_t n_p);  /* > 0: S-hat = G u ODEIM points, gappy on their rows */
int32_t orc_run_points(const orc_run* R, int64_t* rows);  /* ODEIM DOF rows chosen for the next step */
int64_t orc_run_k(const orc_run* R);
void orc_run_state(const orc_run* R, double* q);             /* gamma_k */
void orc_run_mask(const orc_run* R, uint8_t* m);             /* S-hat for the NEXT step */
void orc_run_mask_used(const orc_run* R, uint8_t* m);        /* S-hat used by the last step */
void orc_run_eps(const orc_run* R, double* eps);             /* indicator of the last step */
int32_t orc_run_reff(const orc_run* R);                      /* r_eff of Phi_{k+1} */
void orc_run_basis(const orc_run* R, double* Phi);           /* Phi_{k+1}, D x r_eff */
void orc_run_psi(const orc_run* R, double* psi);             /* psi_{k+1} */
void orc_run_sigma(const orc_run* R, double* S);             /* singular values (w) */
int32_t orc_run_y(const orc_run* R, double* y);              /* y_k of the last hybrid step */
double orc_run_dt(const orc_run* R);
void orc_run_filter_stats(const orc_run* R, int64_t* kept, int32_t* sweeps);
/* replay hooks (inputs all come from tests/ generators or the oracle itself):
 * set the window (w+1 snapshots gamma_{k-w}..gamma_k, oldest first), the
 * mask S-hat_{k+1} and k; builds Phi_{k+1}, psi_{k+1} from the window. */
void orc_run_set_window(orc_run* R, int64_t k, const double* snaps, int32_t nsnaps,
                        const uint8_t* mask_next);

/* ---- NEXT-4: the paper's implicit HDM (implicit.cpp) ----
 * Roe flux, walls (bc = 2), BDF1/BDF2, R_k(q) = q - F_k(q)
 * by Newton-Krylov, partial HDM on S-hat with S-tilde frozen (Eq. 6b,
 * P:238-245), subiterations. */
int32_t orc_roe(int32_t dim, int32_t axis, double gamma, const double* UL, const double* UR, double* F);
int32_t orc_rhs2(const orc_grid* g, int32_t flux, const double* q, double* L); /* flux 0 Rusanov, 1 Roe */
void orc_bdf_residual(const orc_grid* g, int32_t flux, int32_t order, double dt, const double* q,
                      const double* qm1, const double* qm2, double* R);
int32_t orc_newton(const orc_grid* g, int32_t flux, int32_t order, double dt, const double* qm1,
                   const double* qm2, const uint8_t* mask, double* q, double tol, int32_t maxit,
                   double* stats);
int64_t orc_seam_filter_implicit(const orc_grid* g, const orc_params* p, int32_t flux, int32_t order,
                                 double dt, const double* qm1, const double* qm2, double* v,
                                 const uint8_t* mask_S, uint8_t* kept_out, int32_t* sweeps_out);
/* Algorithm 1 with the implicit HDM: fixed dt, eps_y / j_max of P:336-340, Newton tolerance
 * on ||R||_inf.  orc_run_step then returns -1 if a full Newton solve failed. */
void orc_run_set_implicit(orc_run* R, int32_t flux, double dt, double eps_y, int32_t j_max, double newton_tol,
                          int32_t newton_maxit);
void orc_run_implicit_stats(const orc_run* R, int32_t* J_last, int64_t* newton_its);

#ifdef __cplusplus
}
#endif
#endif
