/* hrom.h -- C ABI of libhrom, the B200 (sm_100a) hybrid-snapshot step library.
 *
 * Implements the data-parallel hot path of Zucatti & Zahr, "An adaptive,
 * training-free reduced-order model for convection-dominated problems based on
 * hybrid snapshots" (arXiv 2301.01718; /root/reference/PAPER.md, cited "P:<line>"),
 * in its explicit variant (SSP-RK3 + MUSCL-minmod/Rusanov, BASELINE.json configs).
 *
 * Conventions (all entry points):
 *  - State layout: SoA fp64 q[v*N + n], v = rho, rho*u, [rho*v,] rho*E, n = j*nx + i.
 *  - Masks: N-bit bitmaps, row-padded: word j*ceil(nx/32) + i/32, bit i%32 (1 = cell selected).
 *  - Pointers named dev_* must be device pointers; pointers named any_* may be
 *    host (pageable or pinned) or device pointers (copied with cudaMemcpyDefault).
 *    Caller-owned memory is never freed by the library; all workspaces are
 *    allocated in hrom_create and freed in hrom_destroy; step calls never allocate.
 *  - Asynchrony: every call enqueues on the context's stream and returns; argument
 *    and ordering errors are returned synchronously (HROM_E_INVALID, HROM_E_STATE).
 *    Device-side failures (non-positive density/pressure, NaN) are latched and
 *    returned by hrom_sync (HROM_E_POSITIVITY) with the lowest cell in hrom_error_cell.
 *  - Determinism: bitwise run-to-run reproducible (no floating-point atomics).
 *  - Threading: a context is used by one host thread at a time.
 */
#ifndef HROM_H
#define HROM_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hrom_ctx hrom_ctx;

typedef enum {
  HROM_OK = 0,
  HROM_E_INVALID = 1,     /* bad argument (e.g. r > w, h < stencil radius, f outside (0,1]) */
  HROM_E_STATE = 2,       /* call out of order (e.g. hybrid step before the first basis) */
  HROM_E_POSITIVITY = 3,  /* latched device error: rho <= 0 or p <= 0 or NaN */
  HROM_E_RANK = 4,        /* gappy least-squares matrix is zero */
  HROM_E_CUDA = 5,        /* CUDA runtime error */
  HROM_E_NOMEM = 6        /* device allocation failed in hrom_create */
} hrom_status;

/* Grid: cell-centred Cartesian mesh on [x0,x1] x [y0,y1] (ny = 1 when dim = 1). */
typedef struct {
  int32_t dim, nx, ny;
  double x0, x1, y0, y1;
  int32_t bc;     /* 0 transmissive (zeroth-order ghosts), 1 periodic */
  int32_t recon;  /* 1 first order, 2 MUSCL-minmod */
} hrom_grid;

/* Method parameters (notation of DESIGN.md §1 / SURVEY §0.4). */
typedef struct {
  int32_t window;            /* w: snapshots in the POD window */
  int32_t rank;              /* r: POD modes ("m"), r <= w */
  int32_t halo;              /* h: per-RK-stage stencil halo, h >= recon */
  int32_t band;              /* W: seam-band half width (square), reading A21; -1: the whole
                                hybrid state off S-hat (the paper's filter domain) */
  int32_t filter_orders[3];  /* Shapiro cascade, default {2,4,6} */
  int32_t n_filter_orders;
  int32_t filter_max_sweeps; /* j_max^f = 10; n_filter_orders * j_max^f <= 64 */
  double filter_eps;         /* eps_f = 1e-2, relative decrease (A23) */
  double eig_rel_cutoff;     /* keep POD modes with lambda_i >= cut * lambda_1 (1e-8, A15) */
  double lsq_rel_cutoff;     /* pinv cut on lambda(A^T A) (1e-12, A13) */
  double sample_fraction;    /* f: n_g = ceil(f N) HDM cells per hybrid step (A18) */
  int32_t gram_mode;         /* 0 incremental shifted Gram (default), 1 full DMMA Gram every step */
  int32_t rebase_period;     /* steps between shifted-Gram re-bases (<= 0: never; the window Gram
                                is double-double, G11, so the shift's cancellation in the
                                centring algebra stays below fp64 output precision) */
  int32_t gather_mode;       /* 0: gathered Gram of the S-hat rows updated from the previous
                                step (S-hat churn rows + the new snapshot and HDM columns),
                                1: recomputed over all S-hat rows every step (G7) */
  int32_t full_period;       /* z of Algorithm 1: step k is a full HDM step when
                                k+1 <= w or k mod z = 0, and the basis update + sampling after
                                step k is skipped when (k+1) mod z = 0; <= 0: z = infinity */
  int32_t sample_mode;       /* selection rule of hrom_step: 0 fixed fraction (A18), 1 RRE-delta */
  double rre_delta;          /* delta of the RRE rule, in (0, 1] (sample_mode 1) */
  int32_t odeim_points;      /* n_p > 0: S-hat_{k+1} = G_{k+1} u ODEIM_{n_p}(Phi_{k+1}) (Eq. 10)
                                and the gappy rows are the points' DOF rows (Eq. 8); costs a lifted
                                basis (D x r) and n_p arg-max passes per step; 0: P = S-hat (A11) */
} hrom_params;

/* Create a context for one grid.  cuda_stream: a cudaStream_t (NULL = legacy default).
 * Allocates: ring of w+2 snapshots, Gram shift, RK stage buffers, indicator, masks,
 * lists, small-matrix scratch (about (w+8) * 8 * c * N bytes). */
hrom_status hrom_create(const hrom_grid* grid, double gamma, double cfl, const hrom_params* params,
                        void* cuda_stream, hrom_ctx** out);
void hrom_destroy(hrom_ctx* ctx);

/* gamma_0 := q.  Resets the step counter k to 0 and drops any basis. */
hrom_status hrom_set_state(hrom_ctx* ctx, const double* any_q);
/* q := gamma_k (the latest snapshot). */
hrom_status hrom_get_state(hrom_ctx* ctx, double* any_q);

/* H1+H2: gamma_{k+1} = SSP-RK3 full HDM step of gamma_k (explicit F_k).
 * dt_override > 0 replaces the CFL rule dt = cfl / max_n[(|u|+c)/dx + (|v|+c)/dy].
 * dev_dt_out (nullable, device) receives the dt used. */
hrom_status hrom_full_step(hrom_ctx* ctx, double dt_override, double* dev_dt_out);

/* H1, H3-H7: hybrid step k+1: masked RK3 on S-hat (+ its band, for the
 * filter residual), gappy coordinates y (Eq. 8, P = S-hat), fill of the complement
 * with psi + Phi y, indicator eps, seam filter.
 * dev_mask: S-hat bitmap, or NULL to use the sets built by the last hrom_sample.
 * Requires a basis (hrom_update_basis after step >= w-1).
 * Positivity (O11): if the hybrid state has rho <= 0 or p <= 0 anywhere, the step is
 * redone on the device as a full step from gamma_k with the same dt (the indicator of the
 * hybrid step is kept, as in the oracle); only a failure of that full step is latched and
 * returned by hrom_sync.  Escalations are counted in debug counter [15]. */
hrom_status hrom_hybrid_step(hrom_ctx* ctx, const uint32_t* dev_mask, double dt_override,
                             double* dev_dt_out);

/* H9-H12: push gamma_k into the window; Gram (incremental shifted or full DMMA),
 * lagged centring (Eq. 9 / P:585-587), thin eigen, r_eff; psi_{k+1}.
 * No-op while k < w-1.  At k = w-1 it also sets the bootstrap indicator: the projection error
 * (reading A19) when S-hat = G, or zero in ODEIM mode, where G_w = {} and S-hat_w = P_w. */
hrom_status hrom_update_basis(hrom_ctx* ctx);

/* H8: S-hat_{k+1} = top ceil(f N) cells of eps > 0, ties by ascending index,
 * then builds the stage sets, the seam band and their compacted lists.
 * dev_eps: N indicator values, or NULL for the context's own indicator.
 * Outputs (nullable, device): mask bitmap, ascending cell list, count (int32). */
hrom_status hrom_sample(hrom_ctx* ctx, double fraction, const double* dev_eps, uint32_t* dev_mask_out,
                        int32_t* dev_list_out, int32_t* dev_count_out);

/* H8, RRE-delta rule (Eq. rre): S-hat_{k+1} = the n_g cells of largest eps (ties by
 * ascending index), n_g the smallest count whose relative retained error
 * RRE(n_g) = sum of the n_g largest eps / sum of all eps reaches delta.  The sums are exact
 * (integer arithmetic in units of 2^-1074; reading A35), so n_g is decided without rounding.
 * delta in (0, 1] (else HROM_E_INVALID); all-zero eps selects nothing.  Then builds the sets
 * as hrom_sample; same outputs (dev_count_out receives n_g). */
hrom_status hrom_sample_rre(hrom_ctx* ctx, double delta, const double* dev_eps, uint32_t* dev_mask_out,
                            int32_t* dev_list_out, int32_t* dev_count_out);

/* NEXT-1: ODEIM_{n_p} sampling points of a basis (Eq. 10; reading A36 = greedy
 * DEIM-and-continue over DOF rows, one row per cell, ties by lowest DOF index).
 * dev_phi: D x m column-major (D = c N; e.g. the basis of hrom_get_basis), 1 <= m <= 64,
 * 0 <= n_p <= min(256, N) (else HROM_E_INVALID).  Outputs (device): dev_cells_out[n_p] (int32
 * cells), dev_rows_out[n_p] (int64 DOF rows), in selection order.  Enqueued on the stream. */
hrom_status hrom_odeim(hrom_ctx* ctx, const double* dev_phi, int32_t m, int32_t n_p, int32_t* dev_cells_out,
                       int64_t* dev_rows_out);

/* H4-H6 standalone (gappy POD): with the current basis (Phi_{k+1}, psi_{k+1}), take the
 * values of dev_v on the cells of S-hat (dev_mask or the current sets) as HDM values,
 * y = argmin ||Phi_S y - (v - psi)_S|| (min-norm), and overwrite dev_v off S-hat
 * with psi + Phi y.  dev_y_out (nullable): y (r_eff values).
 * dev_eps_out (nullable): per-cell indicator on S-hat, 0 elsewhere. */
hrom_status hrom_reconstruct(hrom_ctx* ctx, const uint32_t* dev_mask, double* dev_v, double* dev_y_out,
                             double* dev_eps_out);

/* H7 standalone: seam filter of dev_v on the band (S-hat (+) Q_W) \ S-hat against the
 * residual reference dev_F (readings A21-A24).  dev_kept_out (nullable):
 * N bytes, 1 where the filtered value was kept in some sweep. */
hrom_status hrom_filter(hrom_ctx* ctx, const uint32_t* dev_mask, double* dev_v, const double* dev_F,
                        uint8_t* dev_kept_out);

/* One step k of Algorithm 1 (explicit variant) with z = params.full_period:
 * a full step when k+1 <= w or k mod z = 0, else a hybrid step; then, when k >= w-1 and
 * (k+1) mod z != 0, update_basis + sample.  After a full step k >= w the sampling indicator
 * is the projection error of gamma_k on the new basis (the bootstrap rule A19 applied at k;
 * DESIGN.md G8).  A skipped update owes the window-Gram row of gamma_k, computed at the next
 * update.  dev_count_out (nullable, device int32): |S-hat| used by this step (N for a full
 * step), for the sampling averages s-bar, s-bar* of P:715-727. */
hrom_status hrom_step(hrom_ctx* ctx, double dt_override);
hrom_status hrom_step_ex(hrom_ctx* ctx, double dt_override, int32_t* dev_count_out);

/* CUDA-graph replay of hrom_step (NEXT-3).  enable != 0: a steady-state step of Algorithm 1
 * (a hybrid step, then the basis update and the sampling; z = infinity, no ODEIM points,
 * incremental Grams, profiling off, no count output) is captured into a CUDA graph the first
 * time its ring phase k mod (w + 2) occurs -- its kernel arguments depend on k only through the
 * ring slots -- and replayed with cudaGraphLaunch afterwards, the host bookkeeping advanced as
 * the captured step left it.  Other steps run eagerly.  In graph mode the eigen-solve of a basis
 * starts with the next step (not with the sampling), so a captured step joins all its side-
 * stream work.  Results are bitwise identical to eager steps.  Graphs are freed by
 * hrom_set_graph(ctx, 0) and hrom_destroy. */
hrom_status hrom_set_graph(hrom_ctx* ctx, int32_t enable);
int64_t hrom_graph_launches(const hrom_ctx* ctx);  /* steps run from a graph so far */

/* Relative L1 error of Algorithm 1: e = sum |a - b| / sum |b| over the D entries
 * of two device states (uniform cell volumes; the per-cell 1-norm over the c variables).
 * Enqueued on the context stream; synchronises and writes the value to *host_out.
 * Fixed-order reductions: bitwise reproducible. */
hrom_status hrom_rel_l1_error(hrom_ctx* ctx, const double* dev_a, const double* dev_b, double* host_out);

/* ODEIM points (n_p)_k used by the latest step k (the p-bar average): the count of
 * points of the basis that step was solved with in ODEIM mode (odeim_points > 0), 0 for a full
 * step or when S-hat = G (odeim_points = 0, reading A11).  Host-side value, no synchronisation. */
int32_t hrom_points_used(const hrom_ctx* ctx);

/* Make the context stream wait for work the library enqueued on its internal side stream (the
 * eigen-solve of the last basis update, band Gram rows): an event recorded on the context stream
 * after this call covers every kernel of the steps enqueued so far.  No host synchronisation. */
hrom_status hrom_join(hrom_ctx* ctx);

/* Synchronise the stream; returns latched device errors. */
hrom_status hrom_sync(hrom_ctx* ctx);
int64_t hrom_error_cell(const hrom_ctx* ctx);        /* lowest offending cell, or -1 */
int64_t hrom_step_index(const hrom_ctx* ctx);        /* k of the latest snapshot */
int32_t hrom_effective_rank(hrom_ctx* ctx);          /* r_eff of the current basis (syncs) */
const char* hrom_status_string(hrom_status s);

/* ---- test / replay hooks ---- */
/* Window gamma_{k-w}..gamma_k (w+1 snapshots, oldest first, D each, any_ memory) and the
 * mask S-hat_{k+1}; builds the basis as hrom_update_basis would after step k (k >= w). */
hrom_status hrom_set_window(hrom_ctx* ctx, int64_t k, const double* any_snaps, int32_t nsnaps,
                            const uint32_t* any_mask_next);
/* Write gamma_k into its ring slot (streams a window column by column, config 5, without a
 * (w+1) x D staging buffer); no basis work.  hrom_rebuild_basis(k) then treats
 * gamma_{k-w}..gamma_k as the window and builds the basis exactly as hrom_set_window. */
hrom_status hrom_put_snapshot(hrom_ctx* ctx, int64_t k, const double* any_q);
hrom_status hrom_rebuild_basis(hrom_ctx* ctx, int64_t k, const uint32_t* any_mask_next);
/* Phi_{k+1} (D x r_eff, column-major) and psi_{k+1} (D), materialised by the lift kernel. */
hrom_status hrom_get_basis(hrom_ctx* ctx, double* dev_phi, double* dev_psi);
hrom_status hrom_get_indicator(hrom_ctx* ctx, double* any_eps);      /* N values */
hrom_status hrom_get_mask(hrom_ctx* ctx, uint32_t* any_mask);        /* current S-hat bitmap */
hrom_status hrom_get_y(hrom_ctx* ctx, double* any_y);                /* y of the last gappy solve (r) */
hrom_status hrom_get_eigen(hrom_ctx* ctx, double* any_lambda);       /* eigenvalues of X^T X (w) */
int64_t hrom_mask_words(const hrom_ctx* ctx);                        /* words per bitmap */
/* Gram of the listed ring columns shifted by a reference: C = (S - rho 1^T)^T (S - rho 1^T)
 * over D rows with FP64 DMMA tensor cores (K11).  dev_cols: ncol device pointers (device array),
 * dev_rho (nullable = 0), dev_C: ncol*ncol output. Standalone op (config 5). */
hrom_status hrom_gram(hrom_ctx* ctx, const double* const* dev_cols, int32_t ncol, int64_t rows,
                      const double* dev_rho, double* dev_C);
/* Projection of the window on a basis (config 5 kernel op):
 * dev_C[i * (w+1) + j] = sum_e Phi[e][i] gamma_{k-w+j}[e] for the w + 1 window columns of the
 * current basis (oldest first), on FP64 tensor cores.  dev_phi: D x m column-major (device,
 * m <= 64; e.g. hrom_get_basis), dev_C: m (w+1) doubles.  Supported (ceil(m/16), ceil((w+1)/16)):
 * (1,1..5) (2,2..5) (4,9), else HROM_E_INVALID.  HROM_E_STATE before the first basis. */
hrom_status hrom_project(hrom_ctx* ctx, const double* dev_phi, int32_t m, double* dev_C);
/* Overwrite gamma_k (the latest snapshot) in place, without touching the schedule
 * (end-to-end benchmarking of host-resident states).  The window Gram and the basis already
 * built from gamma_k are kept: the caller supplies the same state (e.g. a host round trip);
 * to change the trajectory use hrom_set_state / hrom_set_window. */
hrom_status hrom_put_state(hrom_ctx* ctx, const double* any_q);

/* ---- measurement hooks ---- */
/* enable != 0: record CUDA events around each section of the step on the context stream.
 * Sections: 0 dt, 1 masked RK3, 2 gathered Gram, 3 pinv solve, 4 fill pass, 5 indicator,
 * 6 seam filter, 7 band Gram, 8 positivity, 9 basis update (Gram row), 10 sampling, 11 full step,
 * 12 Gram re-base, 13 eigen-solve (side stream, overlaps sections 10, 0-2 of the next step). */
hrom_status hrom_profile(hrom_ctx* ctx, int32_t enable);
/* Synchronises; per-section summed milliseconds and counts since the last read. */
hrom_status hrom_profile_read(hrom_ctx* ctx, double* ms, int64_t* counts, int32_t nsec);
/* Number of kernels this context has launched (host-side count). */
int64_t hrom_launch_count(const hrom_ctx* ctx);
/* Synchronises and copies n <= 32 int32 device counters: [0] r_eff, [2] LSQ status,
 * [4..6] filter sweeps per order, [8] eigen sweeps (basis), [9] eigen sweeps (pinv);
 * [10..14] eigen-solve phase timings (kcycles), [15] positivity escalations;
 * [16 + l] the size of cell list l (0 S-hat, 1 seam band B, 2 T, 3 A2, 4 A1, 5 filter halo). */
hrom_status hrom_debug_counters(hrom_ctx* ctx, int32_t* any_out, int32_t n);
/* Synchronises and copies n <= 128 device timestamps (ns, %globaltimer) written by the last
 * launches: seam filter [0] start, [1] after the compaction prologue, [2 + s] after sweep s;
 * sets kernel [40 + phase]; LSQ solve [64 + phase] (only while profiling is enabled). */
hrom_status hrom_debug_timers(hrom_ctx* ctx, int64_t* host_out, int32_t n);
/* debug read-back of the small matrices of the basis path (joins the side stream; n doubles):
 * which = 0 / 1 window Gram C hi / lo by ring slot (130 x 130), 2 M = X^T X hi then lo (w x w each,
 * packed at 130^2), 3 eigenvectors of hi(M) (w x w), 4 A (w x r, column j at j*w), 5 eigenvalues */
hrom_status hrom_debug_read(hrom_ctx* ctx, int32_t which, double* any_out, int64_t n);

/* ==== NEXT-4: Algorithm 1 with the paper's own implicit HDM ====
 * HDM: R_k(q) = q - F_k(q) = 0, F_k(q) = dt beta f*(q) - sum_{j<s} a_j q_{k-s+j},
 * BDF2 (a = 1/3, -4/3, 1; beta = 2/3) started by BDF1 at k = 1 (reading A39),
 * f*: MUSCL-minmod + Roe (no entropy fix, A37) or Rusanov; walls (bc = 2: ghosts
 * mirror the interior with the normal momentum negated, A38).  Solved by Newton-Krylov:
 * GMRES(30) on exact Jacobian-vector products (forward-mode dual numbers), backtracking line
 * search, stop at ||R_k||_inf <= newton_tol (reading A40).  A hybrid step solves the partial
 * HDM on S-hat with S-tilde = Neighbors(S-hat) frozen (Eq. 6b) and iterates it
 * with the gappy coordinates: y^(j) = (P^T Phi)^+ P^T (v^(j) - psi), S-tilde :=
 * psi + Phi y^(j), until ||y^(j) - y^(j-1)||_2 < eps_y (j >= 2) or j = j_max (reading A41);
 * then the fill and the spatial filter gated by v - F_k(v).  Window, POD,
 * RRE-delta / fraction sampling, ODEIM points and the schedule z are those of hrom_params.
 * Steps synchronise the stream once per subiteration (the eps_y test is a host decision). */
typedef struct hrom_imp_ctx hrom_imp_ctx;
typedef struct {
  int32_t flux;          /* 0 Rusanov (BASELINE), 1 Roe */
  double dt;             /* fixed time step */
  double eps_y;          /* subiteration tolerance (1e-4) */
  int32_t j_max;         /* maximum subiterations (10) */
  double newton_tol;     /* ||R_k||_inf stop of the Newton solves */
  int32_t newton_maxit;  /* Newton iterations before a solve counts as failed */
} hrom_imp_params;
/* grid->bc in {0, 1, 2 = walls}; params: window, rank, halo (>= stencil radius), band (-1: the
 * whole hybrid state off S-hat, the paper's filter domain), filter, cutoffs, sample_mode /
 * sample_fraction / rre_delta, odeim_points, full_period (z).  HROM_E_INVALID on bad values. */
hrom_status hrom_imp_create(const hrom_grid* grid, double gamma, const hrom_params* params,
                            const hrom_imp_params* imp, void* cuda_stream, hrom_imp_ctx** out);
void hrom_imp_destroy(hrom_imp_ctx* ctx);
hrom_status hrom_imp_set_state(hrom_imp_ctx* ctx, const double* any_q);  /* gamma_0, k = 0 */
hrom_status hrom_imp_get_state(hrom_imp_ctx* ctx, double* any_q);        /* gamma_k */
/* One step of Algorithm 1: full implicit HDM when k+1 <= w or k mod z = 0, else the
 * partial HDM with subiterations; then the basis update and sampling as hrom_step.  A failed
 * partial Newton solve or a non-physical hybrid state escalates to a full solve;
 * a failed full solve returns HROM_E_POSITIVITY.  dev_count_out (nullable): |S-hat| used. */
hrom_status hrom_imp_step(hrom_imp_ctx* ctx, int32_t* dev_count_out);
/* host_out[5]: kind of the last step (0 full, 1 hybrid, 2 escalated), J (subiterations), Newton
 * iterations, GMRES products, ODEIM points used (p-bar) */
hrom_status hrom_imp_stats(hrom_imp_ctx* ctx, int32_t* host_out);
hrom_status hrom_imp_get_mask(hrom_imp_ctx* ctx, uint32_t* any_mask);      /* S-hat_{k+1} bitmap */
hrom_status hrom_imp_get_indicator(hrom_imp_ctx* ctx, double* any_eps);   /* N values */
hrom_status hrom_imp_get_y(hrom_imp_ctx* ctx, double* any_y);
int64_t hrom_imp_mask_words(const hrom_imp_ctx* ctx);
int32_t hrom_imp_effective_rank(hrom_imp_ctx* ctx);
hrom_status hrom_imp_sync(hrom_imp_ctx* ctx);
/* standalone pieces (device pointers, D values each; order 1 or 2, qm2 unused for order 1):
 * R_k on every cell; the Newton-Krylov root on the cells of dev_mask (NULL: all) with dev_q the
 * initial guess and the frozen data (host_iters: iterations, HROM_E_POSITIVITY if it failed);
 * the filter of dev_v on the band of dev_mask gated by the implicit residual (host_sweeps[3]). */
hrom_status hrom_imp_residual(hrom_imp_ctx* ctx, int32_t order, const double* dev_q, const double* dev_qm1,
                              const double* dev_qm2, double* dev_R);
hrom_status hrom_imp_newton(hrom_imp_ctx* ctx, int32_t order, const double* dev_qm1, const double* dev_qm2,
                            const uint32_t* dev_mask, double* dev_q, int32_t* host_iters);
hrom_status hrom_imp_filter(hrom_imp_ctx* ctx, int32_t order, const double* dev_qm1, const double* dev_qm2,
                            const uint32_t* dev_mask, double* dev_v, uint8_t* dev_kept_out, int32_t* host_sweeps);
/* measurement hook: block 0's clock64 sums since the last read over the Newton solves:
 * [0] Jacobian products (incl. barriers), [1] Gram-Schmidt, [2] norms + Givens, [3] line
 * searches, [4] whole kernels, [5] products, [6] solves, [7] block 0 thread 0's own face tasks,
 * [8] its wait at the barrier after them; host_out: 10 values; then resets them */
hrom_status hrom_imp_debug_timers(hrom_imp_ctx* ctx, int64_t* host_out);
/* the filter band of the current sets (ascending cells; N int32 + count) */
hrom_status hrom_imp_get_band(hrom_imp_ctx* ctx, int32_t* any_list, int32_t* any_count);
/* replay hook: window gamma_{k-w}..gamma_k (w+1, oldest first) and S-hat_{k+1} (as hrom_set_window) */
hrom_status hrom_imp_set_window(hrom_imp_ctx* ctx, int64_t k, const double* any_snaps, int32_t nsnaps,
                                const uint32_t* any_mask_next);

/* ---- Row-slab sharding of ONE problem across ranks -----------------------------
 * The HDM residual is local (Eq. partial_hdm2), so the grid can be cut into slabs of
 * consecutive rows, one per rank: every rank keeps its rows of the snapshot window, of Phi (implicit),
 * psi and the indicator, plus `halo` = max(3 h, 2 h + W) rows of each neighbour (the reach of a
 * three-stage step with per-stage stencil halo h, and of the set dilations of reading A21).  Per step
 * the ranks exchange: the halo rows of gamma_k (H3/H6) and of S-hat (H8) with their two neighbours,
 * and all-reduce the gathered normal matrix of Eq. 8 (H4, (w+2)^2 double-doubles), the new row of the
 * window Gram of Eq. 9 (H10, w+1 double-doubles), the radix-select histograms of the sampling rule
 * (H8, 2048 counts per pass) and the CFL maximum (H1).  The small solves (H5, H11) are
 * replicated: they run on every rank on bitwise identical inputs.
 *
 * A slab context is an hrom_ctx (destroy with hrom_destroy; hrom_sync, hrom_step_index,
 * hrom_effective_rank, hrom_get_y, hrom_get_eigen apply).  Transport stays outside the library:
 * hrom_slab_step runs the local work up to the next exchange and writes ONE message into the
 * caller's device buffer dev_send (capacity >= max_message_bytes); the caller all-gathers the
 * nranks messages of *send_bytes_out bytes each, in rank order, into one device buffer and passes
 * it to the next call as dev_gathered (NULL on the first call of a step).  *send_bytes_out == 0
 * means the step (stage, basis update and sampling of Algorithm 1, z = infinity, fixed
 * sampling fraction, P = S-hat) is complete.  Every reduction is done by the library itself on the
 * gathered buffer in rank order (double-double sums): all ranks obtain identical bits, and a run
 * is bitwise reproducible.  Messages of all ranks have equal length in every phase.
 * The seam filter runs one exchange per sweep (edge rows + the sweep's keep count and
 * largest relative decrease); its stop decision is taken on the host from the gathered statistics,
 * so a call that consumes a sweep message synchronises the context's stream.
 * Refused (HROM_E_INVALID): dim != 2, ODEIM points, RRE-delta, finite z, W = -1, w + 1 > 68, fewer
 * than `halo` own rows per rank.  Positivity escalation: when any rank's hybrid state is
 * non-physical, every rank redoes the step as a full step with the same dt (host decision on the
 * gathered flags: a call that consumes an END message of a hybrid step synchronises the stream);
 * a state that is still non-physical is latched on every rank (hrom_sync -> HROM_E_POSITIVITY). */
typedef struct {
  int32_t rank, nranks;
  int32_t ny_global;          /* rows of the whole grid */
  int32_t row0, rows_own;     /* first global row and number of rows this rank owns */
  int32_t halo_lo, halo_hi;   /* halo rows kept below / above (0 at a non-periodic end) */
  int32_t halo;               /* halo depth of an interior edge */
  int64_t cells_own, cells_local, cells_global;
  int64_t max_message_bytes;  /* capacity the send buffer needs */
} hrom_slab_info;
/* host-only: the row partition (rows_own differ by at most one; rank r owns rows after rank r-1) */
hrom_status hrom_slab_partition(int32_t ny_global, int32_t nranks, int32_t rank, int32_t periodic, int32_t halo_rows,
                                hrom_slab_info* out);
/* grid: the WHOLE grid; params as hrom_create (gather_mode is ignored) */
hrom_status hrom_slab_create(const hrom_grid* grid, double gamma, double cfl, const hrom_params* params,
                             void* cuda_stream, int32_t rank, int32_t nranks, hrom_ctx** out);
hrom_status hrom_slab_get_info(const hrom_ctx* ctx, hrom_slab_info* out);
/* any_q_global: the whole initial state q[v*N_global + n] (every rank passes the same array) */
hrom_status hrom_slab_set_state(hrom_ctx* ctx, const double* any_q_global);
/* the own rows: q[v*cells_own + n], rows_own*ceil(nx/32) mask words, cells_own indicator values */
hrom_status hrom_slab_get_state(hrom_ctx* ctx, double* any_q_own);
hrom_status hrom_slab_get_mask(hrom_ctx* ctx, uint32_t* any_mask_own);
hrom_status hrom_slab_get_indicator(hrom_ctx* ctx, double* any_eps_own);
hrom_status hrom_slab_step(hrom_ctx* ctx, const void* dev_gathered, void* dev_send, int64_t* send_bytes_out);
/* H8 alone (the slab counterpart of hrom_sample with an explicit indicator): S-hat := the top
 * ceil(f N_global) cells of the ranks' indicators any_eps_own (cells_own values each; eps > 0 only,
 * ties at the threshold by ascending global cell), then the sets.  Starts the selection phases:
 * writes the first message; continue with hrom_slab_step until *send_bytes_out == 0. */
hrom_status hrom_slab_resample(hrom_ctx* ctx, const double* any_eps_own, void* dev_send, int64_t* send_bytes_out);
/* Replay hook (as hrom_set_window): the window gamma_{k-w}..gamma_k (w+1 WHOLE-grid snapshots, oldest
 * first) and the WHOLE-grid S-hat_{k+1} bitmap; every rank copies its rows and halo rows, the window
 * Gram of the own rows is summed over the ranks, the basis and the sets are rebuilt.  Writes the
 * first message; continue with hrom_slab_step until *send_bytes_out == 0. */
hrom_status hrom_slab_set_window(hrom_ctx* ctx, int64_t k, const double* any_snaps_global, int32_t nsnaps,
                                 const uint32_t* any_mask_global, void* dev_send, int64_t* send_bytes_out);
int64_t hrom_slab_escalations(const hrom_ctx* ctx);  /* hybrid steps redone as full steps so far */

#ifdef __cplusplus
}
#endif
#endif
