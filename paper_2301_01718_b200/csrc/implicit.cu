// implicit.cu -- NEXT-4: the paper's own implicit HDM inside Algorithm 1.
//
//   * f*(q): MUSCL-minmod faces (conservative, component-wise, A3) + Roe flux or Rusanov,
//     transmissive / periodic / wall boundaries (reading A38);
//   * R_k(q) = q - F_k(q), F_k(q) = dt beta f*(q) - sum_{j<s} a_j q_{k-s+j}, BDF1 at
//     k = 1 and BDF2 afterwards (a = 1/3, -4/3, beta = 2/3; reading A39);
//   * Newton-Krylov: ONE cooperative kernel per solve runs every Newton iteration, the
//     restarted GMRES on exact Jacobian-vector products (forward-mode dual numbers through the
//     same templated residual: the directional derivative of the discrete residual, minmod
//     branches frozen at the current state) and the backtracking line search; reductions are
//     per-block partials summed in a fixed order, so every block takes the same decisions and
//     the solve is bitwise reproducible.  The unknowns are all cells (full HDM) or the cells of
//     S-hat with the values on S-tilde = Neighbors(S-hat) frozen (partial HDM, Eq. 6b,
//     P:238-245).
//   * the partial-HDM subiterations alternate that solve with the gappy coordinates
//     of the context's explicit machinery (gathered Gram + pinv solve on the rows of P, fill of
//     psi + Phi y off S-hat), until ||y^(j+1) - y^(j)||_2 < eps_y or j = j_max (reading A41);
//   * the spatial filter gated by the implicit residual: one cooperative kernel,
//     the residual v - F_k(v) re-evaluated on the filtered candidate every sweep.
// The window, POD basis, RRE-delta sampling and ODEIM points are the explicit path's (an
// internal hrom_ctx on the same grid): only the HDM function changes (Algorithm 1).
#include <cooperative_groups.h>
#include <algorithm>
#include <cmath>
#include "internal.cuh"

namespace cg = cooperative_groups;

struct hrom_imp_ctx;

namespace hrom {
namespace imp {

// geometry of the implicit residual (bc 2 = walls)
struct IGeo {
  int dim, nx, ny, c, bc, recon, flux;
  int N, D;
  double dx, dy, gamma;
};

// BDF of order s: R = q - (dt beta f*(q) - (a_m1 q_{k-1} + a_m2 q_{k-2}))
struct IBdf {
  int order;
  double a_m2, a_m1, beta, dt;
};

// ---------------- forward-mode dual numbers (value, tangent) ----------------
struct dual {
  double v, d;
};
__device__ __forceinline__ dual operator+(dual a, dual b) { return {a.v + b.v, a.d + b.d}; }
__device__ __forceinline__ dual operator-(dual a, dual b) { return {a.v - b.v, a.d - b.d}; }
__device__ __forceinline__ dual operator-(dual a) { return {-a.v, -a.d}; }
__device__ __forceinline__ dual operator*(dual a, dual b) { return {a.v * b.v, a.d * b.v + a.v * b.d}; }
// one division per dual division: only the tangents of dual results are used (Jacobian products,
// accurate far beyond the GMRES tolerance with a reciprocal), the values come from the double path
__device__ __forceinline__ dual operator/(dual a, dual b) {
  const double r = 1.0 / b.v;
  const double q = a.v * r;
  return {q, (a.d - q * b.d) * r};
}
__device__ __forceinline__ dual operator*(double s, dual a) { return {s * a.v, s * a.d}; }
__device__ __forceinline__ dual operator+(double s, dual a) { return {s + a.v, a.d}; }
__device__ __forceinline__ dual operator-(dual a, double s) { return {a.v - s, a.d}; }
__device__ __forceinline__ double val(double a) { return a; }
__device__ __forceinline__ double val(dual a) { return a.v; }
__device__ __forceinline__ double tsqrt(double a) { return sqrt(a); }
__device__ __forceinline__ dual tsqrt(dual a) {
  const double s = sqrt(a.v);
  return {s, (0.5 * a.d) / s};
}
__device__ __forceinline__ double tabs(double a) { return fabs(a); }
__device__ __forceinline__ dual tabs(dual a) { return a.v < 0.0 ? -a : a; }
template <class T> __device__ __forceinline__ T tzero() { return T{}; }
template <> __device__ __forceinline__ double tzero<double>() { return 0.0; }
template <> __device__ __forceinline__ dual tzero<dual>() { return dual{0.0, 0.0}; }
template <class T> __device__ __forceinline__ T tmk(double v, double d);
template <> __device__ __forceinline__ double tmk<double>(double v, double) { return v; }
template <> __device__ __forceinline__ dual tmk<dual>(double v, double d) { return dual{v, d}; }

// minmod(a, b) = 0 if ab <= 0, else the argument of smaller magnitude (branch by value)
template <class T> __device__ __forceinline__ T minmod(T a, T b) {
  if (val(a) * val(b) <= 0.0) return tzero<T>();
  if (val(a) > 0.0) return val(a) < val(b) ? a : b;
  return val(a) > val(b) ? a : b;
}

// All local state vectors below have compile-time sizes and indices (DIM, AXIS template
// parameters, C = DIM + 2): no local array is indexed by a run-time value, so every one of them
// lives in registers.  (A first version indexed them with g.c / axis at run time; the cooperative
// filter kernel then read stale local-memory copies -- residuals that changed with unrelated code
// and with the initial contents of the arrays.)

// cell (i, j) with ghosts: periodic wrap, transmissive clamp, walls mirror (ghost -1-m <-> m)
// with the normal momentum negated.  The tangent of a cell is V[e] when the cell is an
// unknown of the current solve (unk == nullptr: every cell), else 0.
template <class T, int DIM>
__device__ __forceinline__ void load_cell(const IGeo& g, const double* q, const double* V, const uint8_t* unk, int i,
                                          int j, T (&U)[DIM + 2]) {
  bool fx = false, fy = false;
  if (g.bc == 1) {
    i = (i % g.nx + g.nx) % g.nx;
    j = DIM == 2 ? (j % g.ny + g.ny) % g.ny : 0;
  } else if (g.bc == 2) {
    if (i < 0) { i = -1 - i; fx = true; }
    if (i >= g.nx) { i = 2 * g.nx - 1 - i; fx = true; }
    if (DIM == 2) {
      if (j < 0) { j = -1 - j; fy = true; }
      if (j >= g.ny) { j = 2 * g.ny - 1 - j; fy = true; }
    } else {
      j = 0;
    }
  } else {
    i = i < 0 ? 0 : (i >= g.nx ? g.nx - 1 : i);
    j = DIM == 2 ? (j < 0 ? 0 : (j >= g.ny ? g.ny - 1 : j)) : 0;
  }
  const int n = j * g.nx + i;
  // the tangent loads do not wait for the unknown flag (no control dependency): V of a frozen
  // cell is read and discarded
  double vt[DIM + 2];
#pragma unroll
  for (int v = 0; v < DIM + 2; ++v) vt[v] = V ? V[v * g.N + n] : 0.0;
  const bool tan = V && (!unk || (unk[n] & 1));
#pragma unroll
  for (int v = 0; v < DIM + 2; ++v) U[v] = tmk<T>(q[v * g.N + n], tan ? vt[v] : 0.0);
  if (fx) U[1] = -U[1];
  if (DIM == 2 && fy) U[2] = -U[2];
}

template <class T, int DIM>
__device__ __forceinline__ T pressure(double gamma, const T (&U)[DIM + 2]) {
  T m2 = U[1] * U[1];
  if (DIM == 2) m2 = m2 + U[2] * U[2];
  return (gamma - 1.0) * (U[DIM + 1] - 0.5 * (m2 / U[0]));
}

template <class T, int DIM, int AXIS>
__device__ __forceinline__ void phys_flux(const T (&U)[DIM + 2], const T& p, T (&F)[DIM + 2]) {
  const T ua = U[1 + AXIS] / U[0];
  F[0] = U[1 + AXIS];
#pragma unroll
  for (int d = 0; d < DIM; ++d) F[1 + d] = d == AXIS ? U[1 + d] * ua + p : U[1 + d] * ua;
  F[DIM + 1] = (U[DIM + 1] + p) * ua;
}

// Roe flux in wave form (Roe 1981), no entropy fix (reading A37): false (F = NaN) when
// the Roe average is not admissible (a~^2 <= 0)
template <class T, int DIM, int AXIS>
__device__ __forceinline__ bool roe_flux(double gamma, const T (&UL)[DIM + 2], const T (&UR)[DIM + 2],
                                         T (&F)[DIM + 2]) {
  constexpr int C = DIM + 2, TA = 1 - AXIS;  // TA: tangential axis (2D)
  const T pL = pressure<T, DIM>(gamma, UL), pR = pressure<T, DIM>(gamma, UR);
  T FL[C], FR[C];
  phys_flux<T, DIM, AXIS>(UL, pL, FL);
  phys_flux<T, DIM, AXIS>(UR, pR, FR);
  const T rL = UL[0], rR = UR[0];
  T uL[DIM], uR[DIM];
#pragma unroll
  for (int d = 0; d < DIM; ++d) {
    uL[d] = UL[1 + d] / rL;
    uR[d] = UR[1 + d] / rR;
  }
  const T HL = (UL[C - 1] + pL) / rL, HR = (UR[C - 1] + pR) / rR;
  const T sL = tsqrt(rL), sR = tsqrt(rR), sw = sL + sR;
  T u[DIM];
  T q2 = tzero<T>();
#pragma unroll
  for (int d = 0; d < DIM; ++d) {
    u[d] = (sL * uL[d] + sR * uR[d]) / sw;
    q2 = q2 + u[d] * u[d];
  }
  const T H = (sL * HL + sR * HR) / sw;
  const T a2 = (gamma - 1.0) * (H - 0.5 * q2);
  if (!(val(a2) > 0.0)) {
#pragma unroll
    for (int v = 0; v < C; ++v) F[v] = tmk<T>(__longlong_as_double(0x7ff8000000000000ll), 0.0);
    return false;
  }
  const T a = tsqrt(a2), rho = sL * sR;
  const T un = u[AXIS];
  const T dp = pR - pL, dun = uR[AXIS] - uL[AXIS];
  const T al1 = (dp - rho * a * dun) / (2.0 * a2);
  const T al2 = (rR - rL) - dp / a2;
  const T al4 = (dp + rho * a * dun) / (2.0 * a2);
  const T l1 = tabs(un - a), l2 = tabs(un), l4 = tabs(un + a);
  const T w1 = l1 * al1, w2 = l2 * al2, w4 = l4 * al4;
  T Dv[C];
  Dv[0] = (w1 + w2) + w4;
#pragma unroll
  for (int d = 0; d < DIM; ++d) {
    const T ua = d == AXIS ? a : tzero<T>();
    Dv[1 + d] = (w1 * (u[d] - ua) + w2 * u[d]) + w4 * (u[d] + ua);
  }
  Dv[C - 1] = (w1 * (H - un * a) + w2 * (0.5 * q2)) + w4 * (H + un * a);
  if (DIM == 2) {
    const T w3 = l2 * (rho * (uR[TA] - uL[TA]));
    Dv[1 + TA] = Dv[1 + TA] + w3;
    Dv[C - 1] = Dv[C - 1] + w3 * u[TA];
  }
#pragma unroll
  for (int v = 0; v < C; ++v) F[v] = 0.5 * (FL[v] + FR[v]) - 0.5 * Dv[v];
  return true;
}

// Rusanov (BASELINE flux, A2): 1/2 (F_L + F_R) - 1/2 max(|u_L|+c_L, |u_R|+c_R) (U_R - U_L)
template <class T, int DIM, int AXIS>
__device__ __forceinline__ bool rusanov_flux(double gamma, const T (&UL)[DIM + 2], const T (&UR)[DIM + 2],
                                             T (&F)[DIM + 2]) {
  constexpr int C = DIM + 2;
  const T pL = pressure<T, DIM>(gamma, UL), pR = pressure<T, DIM>(gamma, UR);
  T FL[C], FR[C];
  phys_flux<T, DIM, AXIS>(UL, pL, FL);
  phys_flux<T, DIM, AXIS>(UR, pR, FR);
  const T cL = tsqrt(gamma * pL / UL[0]), cR = tsqrt(gamma * pR / UR[0]);
  const T sLv = tabs(UL[1 + AXIS] / UL[0]) + cL, sRv = tabs(UR[1 + AXIS] / UR[0]) + cR;
  const T s = val(sLv) >= val(sRv) ? sLv : sRv;
#pragma unroll
  for (int v = 0; v < C; ++v) F[v] = 0.5 * (FL[v] + FR[v]) - 0.5 * (s * (UR[v] - UL[v]));
  return val(pL) > 0.0 && val(pR) > 0.0;
}

// numerical flux through the face between (i, j) and the next cell along AXIS
template <class T, int DIM, int AXIS>
__device__ __forceinline__ bool face_flux(const IGeo& g, const double* q, const double* V, const uint8_t* unk, int i,
                                          int j, T (&F)[DIM + 2]) {
  constexpr int C = DIM + 2, di = AXIS == 0 ? 1 : 0, dj = 1 - di;
  T U0[C], U1[C], UL[C], UR[C];
  load_cell<T, DIM>(g, q, V, unk, i, j, U0);
  load_cell<T, DIM>(g, q, V, unk, i + di, j + dj, U1);
  if (g.recon == 2) {
    T Um[C], U2[C];
    load_cell<T, DIM>(g, q, V, unk, i - di, j - dj, Um);
    load_cell<T, DIM>(g, q, V, unk, i + 2 * di, j + 2 * dj, U2);
#pragma unroll
    for (int v = 0; v < C; ++v) {
      UL[v] = U0[v] + 0.5 * minmod(U0[v] - Um[v], U1[v] - U0[v]);
      UR[v] = U1[v] - 0.5 * minmod(U1[v] - U0[v], U2[v] - U1[v]);
    }
  } else {
#pragma unroll
    for (int v = 0; v < C; ++v) {
      UL[v] = U0[v];
      UR[v] = U1[v];
    }
  }
  return g.flux == 1 ? roe_flux<T, DIM, AXIS>(g.gamma, UL, UR, F) : rusanov_flux<T, DIM, AXIS>(g.gamma, UL, UR, F);
}

// R_k at cell n (all C variables) for the state q (+ direction V: dual tangent)
template <class T, int DIM>
__device__ __forceinline__ bool cell_residual_t(const IGeo& g, const IBdf& B, const double* q, const double* V,
                                                const uint8_t* unk, const double* qm1, const double* qm2, int n,
                                                T* R) {
  constexpr int C = DIM + 2;
  const int i = n % g.nx, j = n / g.nx;
  T Fxp[C], Fxm[C], Fyp[C], Fym[C];
  bool ok = face_flux<T, DIM, 0>(g, q, V, unk, i, j, Fxp);
  ok = face_flux<T, DIM, 0>(g, q, V, unk, i - 1, j, Fxm) && ok;
  if (DIM == 2) {
    ok = face_flux<T, DIM, 1>(g, q, V, unk, i, j, Fyp) && ok;
    ok = face_flux<T, DIM, 1>(g, q, V, unk, i, j - 1, Fym) && ok;
  }
  const bool tan = V && (!unk || (unk[n] & 1));
  const double sdt = B.dt * B.beta;
#pragma unroll
  for (int v = 0; v < C; ++v) {
    // f* = -(F_{i+1/2} - F_{i-1/2}) / dx - (G_{j+1/2} - G_{j-1/2}) / dy
    T L = (Fxp[v] - Fxm[v]) / tmk<T>(-g.dx, 0.0);
    if (DIM == 2) L = L - (Fyp[v] - Fym[v]) / tmk<T>(g.dy, 0.0);
    const int e = v * g.N + n;
    double h = B.a_m1 * qm1[e];
    if (B.order == 2) h = h + B.a_m2 * qm2[e];
    const T F = sdt * L - tmk<T>(h, 0.0);
    R[v] = tmk<T>(q[e], tan ? V[e] : 0.0) - F;
  }
  return ok;
}

// run-time dimension dispatch; R has room for 4 values
template <class T>
__device__ __forceinline__ bool cell_residual(const IGeo& g, const IBdf& B, const double* q, const double* V,
                                              const uint8_t* unk, const double* qm1, const double* qm2, int n, T* R) {
  return g.dim == 2 ? cell_residual_t<T, 2>(g, B, q, V, unk, qm1, qm2, n, R)
                    : cell_residual_t<T, 1>(g, B, q, V, unk, qm1, qm2, n, R);
}

// admissibility of a cell state (rho > 0, p > 0)
__device__ __forceinline__ bool admissible_cell(const IGeo& g, const double* U) {
  double m2 = U[1] * U[1];
  if (g.dim == 2) m2 += U[2] * U[2];
  const double p = (g.gamma - 1.0) * (U[g.dim + 1] - 0.5 * (m2 / U[0]));
  return U[0] > 0.0 && p > 0.0;
}

// ---------------- the Newton-Krylov solve (one cooperative kernel) ----------------
constexpr int NK_T = 256, NK_W = NK_T / 32;  // 256: up to 255 registers (dual-number face fluxes)
constexpr int kMaxKrylov = 30;  // GMRES restart length

struct NArgs {
  IGeo g;
  IBdf B;
  const double* qm1;
  const double* qm2;
  double* q;     // state (D): unknown entries are solved for, the rest is frozen data
  double* qt;    // trial state (D)
  const int32_t* cells;  // unknown cells (nullptr: 0..N-1)
  const int32_t* ncell_dev;  // device count of cells (nullptr: ncell)
  int ncell;
  const uint8_t* unk;  // per-cell flags, bit 0 = unknown (nullptr: every cell)
  double tol, rtol;
  int maxit, maxprod;
  double* R;   // D residual (unknown entries)
  double* Rt;  // D trial residual
  double* dq;  // D Newton correction
  double* Vk;  // (kMaxKrylov + 1) D Krylov basis
  double* wv;  // D
  double* part;  // [gridDim][32] block partials
  int* stat;     // [0] Newton iterations (or -1 / -2), [1] J products, [2] final ||R||_inf bits lo, hi
  double* rstat;  // [0] final ||R||_inf
  const int* run_if;  // nullable: run only when *run_if != 0
  double* ff;         // 4 * 4 * ncell face-flux tangents of the face-parallel Jacobian products
  long long* tdbg;    // nullable: block 0's clock64 per phase [0] products (JVP + barriers),
                      // [1] Gram-Schmidt, [2] norms + Givens, [3] line search, [4] whole kernel
};

struct NShared {
  double H[(kMaxKrylov + 1) * kMaxKrylov];
  double cs[kMaxKrylov], sn[kMaxKrylov], gv[kMaxKrylov + 1], y[kMaxKrylov];
  double red[NK_W][32];
  double tot[32];
  double hcol[kMaxKrylov + 1];  // Arnoldi column j (both Gram-Schmidt passes), thread 0
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// barrier of a Newton / filter kernel: a block barrier when the solve runs in ONE block (small
// partial systems: no grid barrier, no global partials), else a cooperative grid barrier
template <bool ONE>
struct GSync {
  __device__ __forceinline__ void sync() const {
    if (ONE) __syncthreads();
    else cg::this_grid().sync();
  }
};

// grid-wide reduction of K <= 32 per-thread values (the caller has put warp results in S.red):
// block partial -> part[blk][k] -> grid sync -> every block sums the partials in block order.
// mode: 0 sum, 1 max.  Result in S.tot[k], identical in every block.
template <class GS>
__device__ void grid_finish(const GS& G, NShared& S, double* part, int K, const int* modes) {
  __syncthreads();
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  if (t < K) {
    double a = S.red[0][t];
    for (int w = 1; w < NK_W; ++w) a = modes && modes[t] ? fmax(a, S.red[w][t]) : a + S.red[w][t];
    part[blockIdx.x * 32 + t] = a;
  }
  G.sync();
  // every block sums the partials in the same fixed order: lane l takes blocks l, l + 32, ...,
  // then a fixed xor tree over the lanes (no serial walk over the blocks)
  const int nb = gridDim.x;
  for (int k = warp; k < K; k += NK_W) {
    const bool mx = modes && modes[k];
    double a = 0.0;  // identity of both (the max mode's values are >= 0)
    for (int b = lane; b < nb; b += 32) a = mx ? fmax(a, part[b * 32 + k]) : a + part[b * 32 + k];
    for (int o = 16; o > 0; o >>= 1) {
      const double x = __shfl_xor_sync(0xffffffffu, a, o);
      a = mx ? fmax(a, x) : a + x;
    }
    if (lane == 0) S.tot[k] = a;
  }
  __syncthreads();
}

__device__ __forceinline__ int cell_of(const NArgs& a, int idx) { return a.cells ? a.cells[idx] : idx; }

// residual of state s on the unknown cells into out; warp partials of ||.||_inf, ||.||_2^2 and
// the "bad" count (non-finite or non-admissible) into S.red[w][0..2]
__device__ void residual_phase(const NArgs& a, int nc, const double* s, double* out, NShared& S) {
  const IGeo& g = a.g;
  double mx = 0.0, s2 = 0.0, bad = 0.0;
  for (int idx = blockIdx.x * NK_T + threadIdx.x; idx < nc; idx += gridDim.x * NK_T) {
    const int n = cell_of(a, idx);
    double R[4];
    const bool ok = cell_residual<double>(g, a.B, s, nullptr, nullptr, a.qm1, a.qm2, n, R);
    double U[4];
    for (int v = 0; v < g.c; ++v) U[v] = s[v * g.N + n];
    const bool adm = admissible_cell(g, U);
    if (!ok || !adm) bad += 1.0;
    for (int v = 0; v < g.c; ++v) {
      out[v * g.N + n] = R[v];
      if (!(fabs(R[v]) <= 1e300)) bad += 1.0;
      mx = fmax(mx, fabs(R[v]));
      s2 = fma(R[v], R[v], s2);
    }
  }
  mx = warp_max(mx);
  s2 = warp_sum(s2);
  bad = warp_sum(bad);
  if ((threadIdx.x & 31) == 0) {
    S.red[threadIdx.x >> 5][0] = mx;
    S.red[threadIdx.x >> 5][1] = s2;
    S.red[threadIdx.x >> 5][2] = bad;
  }
}

// w = J V_j on the unknown cells (directional derivative of R at q)
// the tangent of one face flux of cell n (f: 0 x+, 1 x-, 2 y+, 3 y-) in direction V
template <int DIM>
__device__ __forceinline__ void face_tangent(const NArgs& a, const double* V, int n, int f, double* out) {
  const IGeo& g = a.g;
  int i = n % g.nx, j = n / g.nx;
  if (f == 1) --i;
  else if (f == 3) --j;
  dual F[DIM + 2];
  // two call sites (one per axis), not four: the dual-number Roe flux is long straight-line code,
  // and a per-face copy of it overflowed the instruction cache (~25 us per face task)
  if (DIM == 1 || f < 2) face_flux<dual, DIM, 0>(g, a.q, V, a.unk, i, j, F);
  else face_flux<dual, DIM, DIM - 1>(g, a.q, V, a.unk, i, j, F);
#pragma unroll
  for (int v = 0; v < DIM + 2; ++v) out[v] = F[v].d;
}

// w = J V on the unknown cells (directional derivative of R at q).  Face-parallel: one thread per
// (cell, face) computes the face flux's tangent (a cell's residual is four long dependent chains
// of Roe arithmetic; with one thread per cell a small partial system waits on their latency),
// then one thread per unknown entry combines them as cell_residual does.
template <class GS>
__device__ void jvp_phase(const GS& G, const NArgs& a, int nc, const double* V, double* w, long long* tj = nullptr) {
  const IGeo& g = a.g;
  const int nf = 2 * g.dim;
  const int gt = blockIdx.x * NK_T + threadIdx.x, gs = gridDim.x * NK_T;
  const long long c0 = clock64();
  for (int t = gt; t < nc * nf; t += gs) {
    const int idx = t / nf, f = t - idx * nf;
    double* o = a.ff + (int64_t)t * 4;
    if (g.dim == 2) face_tangent<2>(a, V, cell_of(a, idx), f, o);
    else face_tangent<1>(a, V, cell_of(a, idx), f, o);
  }
  const long long c1 = clock64();
  G.sync();
  if (tj) {
    tj[0] += c1 - c0;          // this thread's face task
    tj[1] += clock64() - c1;   // waiting for the other blocks' tasks + the barrier
  }
  const double sdt = a.B.dt * a.B.beta;
  for (int t = gt; t < nc * g.c; t += gs) {
    const int v = t / nc, idx = t - v * nc;
    const int n = cell_of(a, idx);
    const double* o = a.ff + (int64_t)idx * nf * 4;
    double L = (o[0 * 4 + v] - o[1 * 4 + v]) / (-g.dx);
    if (g.dim == 2) L = L - (o[2 * 4 + v] - o[3 * 4 + v]) / g.dy;
    const int e = v * g.N + n;
    w[e] = V[e] - sdt * L;  // every listed cell is an unknown: its tangent is V[e]
  }
}

// entry e of unknown entry index t, cell-major (t = idx * C + v): no division by the run-time
// cell count in the vector loops
__device__ __forceinline__ int entry(const NArgs& a, int nc, int t) {
  (void)nc;
  int idx, v;
  if (a.g.c == 4) {
    idx = t >> 2;
    v = t & 3;
  } else {
    idx = t / 3;
    v = t - 3 * idx;
  }
  return v * a.g.N + cell_of(a, idx);
}

// dots <x, V_i>, i < K, over the unknown entries with each thread's OWN entries (the mapping of
// the CGS updates and of the norm: no barrier between an update and the next reduction); per
// vector a warp tree, then the fixed-order block / grid sums of grid_finish
template <class GS>
__device__ void dots_phase(const GS& G, const NArgs& a, int nc, const double* x, const double* Vb, int K,
                           NShared& S) {
  const int ne = nc * a.g.c;
  const int64_t D = a.g.D;
  const int gt = blockIdx.x * NK_T + threadIdx.x, gs = gridDim.x * NK_T;
  int es[4];
  int m = 0;
  for (int t = gt; t < ne && m < 4; t += gs) es[m++] = entry(a, nc, t);
  const bool more = gt + 4 * gs < ne;  // (not the case for the launch grids used: <= 4 entries each)
  double xs[4];
  for (int k = 0; k < m; ++k) xs[k] = x[es[k]];
#pragma unroll 4
  for (int i = 0; i < K; ++i) {  // unrolled: four vectors' loads in flight (L2 latency)
    const double* vi = Vb + i * D;
    double sv = 0.0;
    for (int k = 0; k < m; ++k) sv = fma(xs[k], vi[es[k]], sv);
    if (more)
      for (int t = gt + 4 * gs; t < ne; t += gs) {
        const int e = entry(a, nc, t);
        sv = fma(x[e], vi[e], sv);
      }
    sv = warp_sum(sv);
    if ((threadIdx.x & 31) == 0) S.red[threadIdx.x >> 5][i] = sv;
  }
  grid_finish(G, S, a.part, K, nullptr);
}

template <class GS>
__device__ double norm2_phase(const GS& G, const NArgs& a, int nc, const double* x, NShared& S) {
  const int ne = nc * a.g.c;
  double s = 0.0;
  for (int t = blockIdx.x * NK_T + threadIdx.x; t < ne; t += gridDim.x * NK_T) {
    const double v = x[entry(a, nc, t)];
    s = fma(v, v, s);
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) S.red[threadIdx.x >> 5][0] = s;
  grid_finish(G, S, a.part, 1, nullptr);
  return sqrt(S.tot[0]);
}

template <bool ONE>
__global__ void __launch_bounds__(NK_T) newton_kernel(NArgs a) {
  if (a.run_if && *a.run_if == 0) return;
  const GSync<ONE> G;
  const long long t_start = clock64();
  long long tph[4] = {0, 0, 0, 0};
  long long tj[2] = {0, 0};
  __shared__ NShared S;
  const IGeo& g = a.g;
  const int nc = a.ncell_dev ? *a.ncell_dev : a.ncell;
  const int ne = nc * g.c;
  const int64_t D = g.D;
  const int gt = blockIdx.x * NK_T + threadIdx.x, gs = gridDim.x * NK_T;
  // trial state = state (frozen entries included)
  for (int e = gt; e < g.D; e += gs) a.qt[e] = a.q[e];
  G.sync();
  residual_phase(a, nc, a.q, a.R, S);
  const int modes3[3] = {1, 0, 0};  // ||R||_inf (max), ||R||_2^2, bad count (sums)
  grid_finish(G, S, a.part, 3, modes3);
  double rinf = S.tot[0], r2 = sqrt(S.tot[1]);
  bool bad = S.tot[2] > 0.0;
  int it = 0, prods = 0;
  int status = 0;
  // forcing term: 1e-4 first, then 0.9 (||R_k|| / ||R_k-1||)^2 (Eisenstat-Walker choice 2)
  // clipped to [rtol, 1e-4], and rtol once ||R||_inf < 1e4 tol; the Jacobian products are
  // exact, so Newton stays superlinear
  double eta = 1e-4, r2prev = r2;
  if (bad) status = -2;
  while (status == 0) {
    if (rinf <= a.tol) break;
    if (it >= a.maxit) {
      status = -1;
      break;
    }
    // ---- GMRES(m) for J dq = -R, dq = 0 initially
    for (int t = gt; t < ne; t += gs) a.dq[entry(a, nc, t)] = 0.0;
    const double bnorm = r2;
    const double tolk = eta * bnorm;  // inexact Newton: GMRES to eta ||R|| (Eisenstat-Walker)
    double beta = r2;
    // V_0 = -R / beta
    for (int t = gt; t < ne; t += gs) {
      const int e = entry(a, nc, t);
      a.Vk[e] = -a.R[e] / beta;
    }
    bool first = true;
    while (prods < a.maxprod) {
      if (!first) {
        // restart: r = -R - J dq
        G.sync();
        jvp_phase(G, a, nc, a.dq, a.wv);
        ++prods;
        G.sync();
        for (int t = gt; t < ne; t += gs) {
          const int e = entry(a, nc, t);
          a.wv[e] = -a.R[e] - a.wv[e];
        }
        G.sync();
        beta = norm2_phase(G, a, nc, a.wv, S);
        if (beta <= tolk) break;
        for (int t = gt; t < ne; t += gs) {
          const int e = entry(a, nc, t);
          a.Vk[e] = a.wv[e] / beta;
        }
      }
      first = false;
      if (threadIdx.x == 0) {
        S.gv[0] = beta;
        for (int i = 1; i <= kMaxKrylov; ++i) S.gv[i] = 0.0;
      }
      __syncthreads();
      int j = 0;
      for (; j < kMaxKrylov && prods < a.maxprod; ++j) {
        long long c0 = clock64();
        G.sync();  // V_j complete
        jvp_phase(G, a, nc, a.Vk + j * D, a.wv, tj);
        ++prods;
        G.sync();
        // classical Gram-Schmidt, twice (CGS2)
        for (int pass = 0; pass < 2; ++pass) {
          if (pass == 0) {
            const long long c1 = clock64();
            tph[0] += c1 - c0;
            c0 = c1;
          }
          dots_phase(G, a, nc, a.wv, a.Vk, j + 1, S);
          if (threadIdx.x == 0)
            for (int i = 0; i <= j; ++i) S.hcol[i] = (pass ? S.hcol[i] : 0.0) + S.tot[i];
          for (int t = gt; t < ne; t += gs) {
            const int e = entry(a, nc, t);
            double wv = a.wv[e];
#pragma unroll 8
            for (int i = 0; i <= j; ++i) wv = fma(-S.tot[i], a.Vk[i * D + e], wv);
            a.wv[e] = wv;
          }
          // no barrier: the next dots pass and the norm read each thread's own entries
        }
        {
          const long long c1 = clock64();
          tph[1] += c1 - c0;
          c0 = c1;
        }
        const double hn = norm2_phase(G, a, nc, a.wv, S);
        if (hn > 0.0)
          for (int t = gt; t < ne; t += gs) {
            const int e = entry(a, nc, t);
            a.Vk[(j + 1) * D + e] = a.wv[e] / hn;
          }
        // Givens rotations on column j (identical in every block)
        if (threadIdx.x == 0) {
          for (int i = 0; i <= j; ++i) S.H[i * kMaxKrylov + j] = S.hcol[i];
          S.H[(j + 1) * kMaxKrylov + j] = hn;
          for (int i = 0; i < j; ++i) {
            const double x0 = S.H[i * kMaxKrylov + j], x1 = S.H[(i + 1) * kMaxKrylov + j];
            S.H[i * kMaxKrylov + j] = S.cs[i] * x0 + S.sn[i] * x1;
            S.H[(i + 1) * kMaxKrylov + j] = -S.sn[i] * x0 + S.cs[i] * x1;
          }
          const double x0 = S.H[j * kMaxKrylov + j], x1 = S.H[(j + 1) * kMaxKrylov + j];
          const double den = hypot(x0, x1);
          S.cs[j] = den > 0.0 ? x0 / den : 1.0;
          S.sn[j] = den > 0.0 ? x1 / den : 0.0;
          S.H[j * kMaxKrylov + j] = den;
          S.H[(j + 1) * kMaxKrylov + j] = 0.0;
          S.gv[j + 1] = -S.sn[j] * S.gv[j];
          S.gv[j] = S.cs[j] * S.gv[j];
        }
        __syncthreads();
        tph[2] += clock64() - c0;
        if (fabs(S.gv[j + 1]) <= tolk || S.H[j * kMaxKrylov + j] == 0.0) {
          ++j;
          break;
        }
      }
      // y = H^-1 g (j x j upper triangle), dq += V y
      if (threadIdx.x == 0) {
        for (int i = j - 1; i >= 0; --i) {
          double s = S.gv[i];
          for (int k = i + 1; k < j; ++k) s -= S.H[i * kMaxKrylov + k] * S.y[k];
          S.y[i] = S.H[i * kMaxKrylov + i] != 0.0 ? s / S.H[i * kMaxKrylov + i] : 0.0;
        }
      }
      __syncthreads();
      for (int t = gt; t < ne; t += gs) {
        const int e = entry(a, nc, t);
        double x = a.dq[e];
#pragma unroll 8
        for (int i = 0; i < j; ++i) x = fma(S.y[i], a.Vk[i * D + e], x);
        a.dq[e] = x;
      }
      if (fabs(S.gv[j]) <= tolk || j == 0) break;
    }
    G.sync();
    // ---- line search: q + lambda dq, lambda halved until admissible and ||R||_2 decreases
    const long long cls = clock64();
    bool accepted = false;
    double lam = 1.0;
    for (int ls = 0; ls <= 12; ++ls, lam *= 0.5) {
      for (int t = gt; t < ne; t += gs) {
        const int e = entry(a, nc, t);
        a.qt[e] = fma(lam, a.dq[e], a.q[e]);
      }
      G.sync();
      residual_phase(a, nc, a.qt, a.Rt, S);
      grid_finish(G, S, a.part, 3, modes3);
      const bool tbad = S.tot[2] > 0.0;
      const double t2 = sqrt(S.tot[1]);
      if (!tbad && (t2 < r2 || ls == 12)) {
        for (int t = gt; t < ne; t += gs) {
          const int e = entry(a, nc, t);
          a.q[e] = a.qt[e];
          a.R[e] = a.Rt[e];
        }
        rinf = S.tot[0];
        r2 = t2;
        accepted = true;
        break;
      }
    }
    G.sync();
    if (!accepted) {
      status = -2;
      break;
    }
    tph[3] += clock64() - cls;
    eta = fmax(a.rtol, fmin(1e-4, 0.9 * (r2 / r2prev) * (r2 / r2prev)));
    if (rinf < 1e4 * a.tol) eta = a.rtol;  // the last steps tight: the root, not just ||R|| <= tol
    r2prev = r2;
    ++it;
  }
  if (gt == 0) {
    a.stat[0] = status == 0 ? it : status;
    a.stat[1] = prods;
    a.rstat[0] = rinf;
    if (a.tdbg) {
      for (int k = 0; k < 4; ++k) a.tdbg[k] += tph[k];
      a.tdbg[4] += clock64() - t_start;
      a.tdbg[5] += prods;
      a.tdbg[6] += 1;
      a.tdbg[7] += tj[0];  // block 0 thread 0's face tasks
      a.tdbg[8] += tj[1];  // ... and its wait for the other tasks + the barrier after them
    }
  }
}

}  // namespace imp
}  // namespace hrom

namespace hrom {
namespace imp {

// ---------------- the filter gated by the implicit residual (one cooperative kernel) ----------------
// Shapiro cascade (reading A24: orders 2, 4, 6; zeroth-order extrapolation at non-periodic ends,
// P:447) on the cells of the band list; per sweep: x-pass v -> vp, y-pass vp -> vpp (2D), the
// residual v - F_k(v) and vpp - F_k(vpp) at every band cell (F_k re-evaluated on the candidate
// state: band cells filtered, the rest unchanged), keep where max_var |.| decreases; the
// eps_f stop counts cells with r_old > 2^-40 max_var |F_k(v)| (reading A23').
constexpr int FI_T = 256, FI_W = FI_T / 32;

struct FArgs {
  IGeo g;
  IBdf B;
  const double* qm1;
  const double* qm2;
  double* v;       // state (D), filtered in place on kept cells
  double* vp;      // D scratch
  double* vpp;     // D scratch
  double* vorig;   // D copy of the input (indicator of kept cells)
  const int32_t* band;  // band cells
  const int32_t* nband_dev;
  uint8_t* keep;        // per band index, this sweep
  uint8_t* kept_cell;   // N: ever kept (nullable output of the standalone call: written here)
  double* eps;          // N, nullable: sum_var (v - vorig)^2 on kept cells
  int orders[3], norders, maxsweeps;
  double eps_f;
  double* part;         // [grid][32]
  int* sweeps_out;      // 3
};

// Shapiro weights (reading A24): (1,2,1)/4, (-1,4,10,4,-1)/16, (1,-6,15,44,15,-6,1)/64
__device__ __forceinline__ int shapiro_rad(int order) { return order == 2 ? 1 : (order == 4 ? 2 : 3); }
__device__ __forceinline__ double shapiro_den(int order) { return order == 2 ? 4.0 : (order == 4 ? 16.0 : 64.0); }
__device__ __forceinline__ double shapiro_coef(int order, int k) {  // k = m + rad
  if (order == 2) return k == 1 ? 2.0 : 1.0;
  if (order == 4) return k == 2 ? 10.0 : (k == 1 || k == 3 ? 4.0 : -1.0);
  return k == 3 ? 44.0 : (k == 2 || k == 4 ? 15.0 : (k == 1 || k == 5 ? -6.0 : 1.0));
}

__device__ __forceinline__ int wrap_or_clamp(int i, int n, bool periodic) {
  if (periodic) return (i % n + n) % n;
  return i < 0 ? 0 : (i >= n ? n - 1 : i);
}

template <bool ONE>
__global__ void __launch_bounds__(FI_T) imp_filter_kernel(FArgs a) {
  const GSync<ONE> G;
  __shared__ double red[FI_W][2];
  __shared__ double tot[2];
  const IGeo& g = a.g;
  const int nb = *a.nband_dev;
  const int gt = blockIdx.x * FI_T + threadIdx.x, gs = gridDim.x * FI_T;
  const bool per = g.bc == 1;
  for (int e = gt; e < g.D; e += gs) a.vp[e] = a.vpp[e] = a.vorig[e] = a.v[e];
  if (a.kept_cell)
    for (int n = gt; n < g.N; n += gs) a.kept_cell[n] = 0;
  G.sync();
  for (int oi = 0; oi < a.norders; ++oi) {
    const int ord = a.orders[oi];
    const int rad = shapiro_rad(ord);
    const double den = shapiro_den(ord);
    int sweeps = 0;
    for (int sw = 0; sw < a.maxsweeps; ++sw) {
      ++sweeps;
      for (int b = gt; b < nb; b += gs) {  // x-pass
        const int n = a.band[b], i = n % g.nx, j = n / g.nx;
        for (int v = 0; v < g.c; ++v) {
          double s = 0.0;
          for (int m = -rad; m <= rad; ++m)
            s += shapiro_coef(ord, m + rad) * a.v[v * g.N + j * g.nx + wrap_or_clamp(i + m, g.nx, per)];
          a.vp[v * g.N + n] = s / den;
        }
      }
      G.sync();
      for (int b = gt; b < nb; b += gs) {  // y-pass (2D)
        const int n = a.band[b], i = n % g.nx, j = n / g.nx;
        for (int v = 0; v < g.c; ++v) {
          if (g.dim == 2) {
            double s = 0.0;
            for (int m = -rad; m <= rad; ++m)
              s += shapiro_coef(ord, m + rad) * a.vp[v * g.N + wrap_or_clamp(j + m, g.ny, per) * g.nx + i];
            a.vpp[v * g.N + n] = s / den;
          } else {
            a.vpp[v * g.N + n] = a.vp[v * g.N + n];
          }
        }
      }
      G.sync();
      double nk = 0.0, md = 0.0;
      for (int b = gt; b < nb; b += gs) {  // residual gate
        const int n = a.band[b];
        double Ro[4], Rn[4];
        cell_residual<double>(g, a.B, a.v, nullptr, nullptr, a.qm1, a.qm2, n, Ro);
        cell_residual<double>(g, a.B, a.vpp, nullptr, nullptr, a.qm1, a.qm2, n, Rn);
        double rold = 0.0, rnew = 0.0, fs = 0.0;
        for (int v = 0; v < g.c; ++v) {
          const int e = v * g.N + n;
          rold = fmax(rold, fabs(Ro[v]));
          rnew = fmax(rnew, fabs(Rn[v]));
          fs = fmax(fs, fabs(a.v[e] - Ro[v]));  // |F_k(v)|: R = v - F
        }
        const bool k = rnew < rold;
        a.keep[b] = k ? 1 : 0;
        if (k) {
          nk += 1.0;
          if (rold > 0x1p-40 * fs) md = fmax(md, (rold - rnew) / rold);
        }
      }
      nk = warp_sum(nk);
      md = warp_max(md);
      if ((threadIdx.x & 31) == 0) {
        red[threadIdx.x >> 5][0] = nk;
        red[threadIdx.x >> 5][1] = md;
      }
      __syncthreads();
      if (threadIdx.x < 2) {
        double s = red[0][threadIdx.x];
        for (int w = 1; w < FI_W; ++w) s = threadIdx.x ? fmax(s, red[w][1]) : s + red[w][0];
        a.part[blockIdx.x * 32 + threadIdx.x] = s;
      }
      G.sync();
      if (threadIdx.x < 64) {  // fixed-order cross-block sums: lane l takes blocks l, l + 32, ...
        const int k = threadIdx.x >> 5, lane = threadIdx.x & 31;
        double s = 0.0;
        for (int b = lane; b < (int)gridDim.x; b += 32) s = k ? fmax(s, a.part[b * 32 + 1]) : s + a.part[b * 32];
        for (int o = 16; o > 0; o >>= 1) {
          const double x = __shfl_xor_sync(0xffffffffu, s, o);
          s = k ? fmax(s, x) : s + x;
        }
        if (lane == 0) tot[k] = s;
      }
      for (int b = gt; b < nb; b += gs)  // apply the kept values
        if (a.keep[b]) {
          const int n = a.band[b];
          for (int v = 0; v < g.c; ++v) a.v[v * g.N + n] = a.vpp[v * g.N + n];
          if (a.kept_cell) a.kept_cell[n] = 1;
        }
      __syncthreads();
      const double nkept = tot[0], maxdec = tot[1];
      G.sync();
      if (nkept == 0.0) break;
      if (maxdec < a.eps_f) break;
    }
    if (gt == 0) a.sweeps_out[oi] = sweeps;
  }
  if (a.eps && a.kept_cell) {
    G.sync();
    for (int b = gt; b < nb; b += gs) {
      const int n = a.band[b];
      if (!a.kept_cell[n]) continue;
      double e2 = 0.0;
      for (int v = 0; v < g.c; ++v) {
        const double d = a.v[v * g.N + n] - a.vorig[v * g.N + n];
        e2 += d * d;
      }
      a.eps[n] = e2;
    }
  }
}

// R_k on every cell (standalone residual)
__global__ void residual_all_kernel(IGeo g, IBdf B, const double* q, const double* qm1, const double* qm2, double* R) {
  for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < g.N; n += gridDim.x * blockDim.x) {
    double r[4];
    cell_residual<double>(g, B, q, nullptr, nullptr, qm1, qm2, n, r);
    for (int v = 0; v < g.c; ++v) R[v * g.N + n] = r[v];
  }
}

// per-cell flag bit 0 from an N-bit row-padded bitmap (word j*wpr + i/32, bit i%32)
__global__ void flags_from_mask_kernel(IGeo g, int wpr, const uint32_t* mask, uint8_t* flags) {
  for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < g.N; n += gridDim.x * blockDim.x) {
    const int i = n % g.nx, j = n / g.nx;
    flags[n] = (uint8_t)((mask[j * wpr + (i >> 5)] >> (i & 31)) & 1u);
  }
}

// ascending list of the cells with flag bit 0 (one block: ordered ballot compaction)
__global__ void __launch_bounds__(1024) list_from_flags_kernel(int N, const uint8_t* flags, int32_t* list, int32_t* count) {
  __shared__ int wcnt[32];
  __shared__ int base;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c0 = 0; c0 < N; c0 += 1024) {
    const int n = c0 + threadIdx.x;
    const bool f = n < N && (flags[n] & 1);
    const unsigned b = __ballot_sync(0xffffffffu, f);
    if (lane == 0) wcnt[warp] = __popc(b);
    __syncthreads();
    int off = base;
    for (int w = 0; w < warp; ++w) off += wcnt[w];
    if (f) list[off + __popc(b & ((1u << lane) - 1u))] = n;
    __syncthreads();
    if (threadIdx.x == 0)
      for (int w = 0; w < 32; ++w) base += wcnt[w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *count = base;
}

// flag[0] = 1 when some cell has rho <= 0 or p <= 0 (or NaN)
__global__ void positivity_flag_kernel(IGeo g, const double* q, int* flag) {
  for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < g.N; n += gridDim.x * blockDim.x) {
    double U[4];
    for (int v = 0; v < g.c; ++v) U[v] = q[v * g.N + n];
    if (!admissible_cell(g, U)) atomicOr(flag, 1);
  }
}

// ||y - y_prev||_2 over the r_eff coordinates -> out[0]; y_prev := y
__global__ void ycheck_kernel(const double* y, double* yprev, const int32_t* reff, int r, double* out) {
  if (threadIdx.x != 0) return;
  const int n = min(*reff, r);
  double s = 0.0;
  for (int i = 0; i < n; ++i) {
    const double d = y[i] - yprev[i];
    s += d * d;
    yprev[i] = y[i];
  }
  out[0] = sqrt(s);
}

}  // namespace imp
}  // namespace hrom

using namespace hrom;
using namespace hrom::imp;

struct hrom_imp_ctx {
  hrom_ctx* aux = nullptr;  // window, basis, sampling, ODEIM, gappy solve and fill (explicit path)
  IGeo g{};
  hrom_params P{};
  hrom_imp_params I{};
  cudaStream_t st = nullptr;
  int nsm = 0, nk_grid = 0, fi_grid = 0;
  int64_t Dp = 0;
  int64_t k = -1;
  // device buffers (plain layout, Dp each)
  double *q1 = nullptr, *q2 = nullptr, *V = nullptr, *qt = nullptr, *R = nullptr, *Rt = nullptr, *dq = nullptr;
  double *Vk = nullptr, *wv = nullptr, *vp = nullptr, *vpp = nullptr, *vorig = nullptr, *part = nullptr;
  double *yprev = nullptr, *rstat = nullptr, *ff = nullptr;
  uint8_t *flags = nullptr, *keep = nullptr, *kept = nullptr;
  int32_t *list = nullptr, *count = nullptr, *istat = nullptr, *fsweeps = nullptr;
  int* posflag = nullptr;
  long long* tdbg = nullptr;  // Newton phase clocks (hrom_imp_debug_timers)
  // pinned host mirror of small results
  double* hres = nullptr;   // [0] ||dy||, [1] final ||R||_inf
  int32_t* hint = nullptr;  // [0] newton status, [1] products, [2] positivity flag, [3..5] sweeps
  // statistics of the last step
  int kind = 0, J = 0, newton_its = 0, prods = 0;
  int64_t newton_total = 0;
};

namespace {

IBdf bdf_of(const hrom_imp_ctx* c, int order) {
  IBdf B{};
  B.order = order;
  B.dt = c->I.dt;
  if (order == 1) {
    B.a_m2 = 0.0;
    B.a_m1 = -1.0;
    B.beta = 1.0;
  } else {
    B.a_m2 = 1.0 / 3.0;
    B.a_m1 = -4.0 / 3.0;
    B.beta = 2.0 / 3.0;
  }
  return B;
}

// ring slot <-> plain vector (the aux context's slab layout, internal.cuh)
hrom_status slot_copy(hrom_imp_ctx* ic, int64_t kk, const double* src_plain, double* dst_plain) {
  hrom_ctx* c = ic->aux;
  const int64_t D = c->g.D, full = D / TILE, tail = D - full * TILE;
  const size_t row = TILE * sizeof(double), spitch = (size_t)c->g.nsr * TILE * sizeof(double);
  double* base = c->b.ring + (int64_t)c->slot_of(kk) * TILE;
  if (src_plain) {
    if (full) HROM_CK(cudaMemcpy2DAsync(base, spitch, src_plain, row, row, full, cudaMemcpyDeviceToDevice, ic->st));
    if (tail)
      HROM_CK(cudaMemcpyAsync(base + full * c->g.nsr * TILE, src_plain + full * TILE, tail * sizeof(double),
                              cudaMemcpyDeviceToDevice, ic->st));
  } else {
    if (full) HROM_CK(cudaMemcpy2DAsync(dst_plain, row, base, spitch, row, full, cudaMemcpyDeviceToDevice, ic->st));
    if (tail)
      HROM_CK(cudaMemcpyAsync(dst_plain + full * TILE, base + full * c->g.nsr * TILE, tail * sizeof(double),
                              cudaMemcpyDeviceToDevice, ic->st));
  }
  return HROM_OK;
}

// one Newton-Krylov solve on the unknown cells (cells == nullptr: every cell), state in q
hrom_status newton(hrom_imp_ctx* c, int order, const double* qm1, const double* qm2, const int32_t* cells,
                   const int32_t* ncell_dev, const uint8_t* unk, double* q, const int* run_if, int ncells_hint) {
  NArgs a{};
  a.g = c->g;
  a.B = bdf_of(c, order);
  a.qm1 = qm1;
  a.qm2 = qm2 ? qm2 : qm1;
  a.q = q;
  a.qt = c->qt;
  a.cells = cells;
  a.ncell_dev = ncell_dev;
  a.ncell = c->g.N;
  a.unk = unk;
  a.tol = c->I.newton_tol;
  a.rtol = 1e-10;
  a.maxit = c->I.newton_maxit;
  a.maxprod = 400;
  a.R = c->R;
  a.Rt = c->Rt;
  a.dq = c->dq;
  a.Vk = c->Vk;
  a.wv = c->wv;
  a.part = c->part;
  a.stat = c->istat;
  a.rstat = c->rstat;
  a.run_if = run_if;
  a.ff = c->ff;
  a.tdbg = c->tdbg;
  // ~16 cells per block: a small partial system is latency-bound (each face flux is a long
  // dependent chain), so it is spread over many SMs rather than packed into one block
  const int grid = std::max(1, std::min(c->nk_grid, (ncells_hint + 15) / 16));
  if (grid == 1) {
    newton_kernel<true><<<1, NK_T, 0, c->st>>>(a);
  } else {
    void* args[] = {&a};
    HROM_CK(cudaLaunchCooperativeKernel((void*)newton_kernel<false>, dim3(grid), dim3(NK_T), args, 0, c->st));
  }
  HROM_LAUNCH_CK();
  ++c->aux->nlaunch;
  return HROM_OK;
}

hrom_status filter_launch(hrom_imp_ctx* c, int order, const double* qm1, const double* qm2, double* v,
                          const int32_t* band, const int32_t* nband_dev, uint8_t* kept_cell, double* eps,
                          int nband_hint) {
  FArgs a{};
  a.g = c->g;
  a.B = bdf_of(c, order);
  a.qm1 = qm1;
  a.qm2 = qm2 ? qm2 : qm1;
  a.v = v;
  a.vp = c->vp;
  a.vpp = c->vpp;
  a.vorig = c->vorig;
  a.band = band;
  a.nband_dev = nband_dev;
  a.keep = c->keep;
  a.kept_cell = kept_cell;
  a.eps = eps;
  a.norders = c->P.n_filter_orders;
  for (int i = 0; i < 3; ++i) a.orders[i] = c->P.filter_orders[i];
  a.maxsweeps = c->P.filter_max_sweeps;
  a.eps_f = c->P.filter_eps;
  a.part = c->part;
  a.sweeps_out = c->fsweeps;
  const int grid = std::max(1, std::min(c->fi_grid, (nband_hint + FI_T - 1) / FI_T));
  if (grid == 1) {
    imp_filter_kernel<true><<<1, FI_T, 0, c->st>>>(a);
  } else {
    void* args[] = {&a};
    HROM_CK(cudaLaunchCooperativeKernel((void*)imp_filter_kernel<false>, dim3(grid), dim3(FI_T), args, 0, c->st));
  }
  HROM_LAUNCH_CK();
  ++c->aux->nlaunch;
  return HROM_OK;
}

hrom_status read_newton(hrom_imp_ctx* c, int* status) {
  HROM_CK(cudaMemcpyAsync(c->hint, c->istat, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, c->st));
  HROM_CK(cudaMemcpyAsync(c->hres + 1, c->rstat, sizeof(double), cudaMemcpyDeviceToHost, c->st));
  HROM_CK(cudaStreamSynchronize(c->st));
  *status = c->hint[0];
  c->prods += c->hint[1];
  return HROM_OK;
}

// full implicit HDM step into c->V from gamma_{k} (= q1), Alg. 1 line 4
hrom_status full_solve(hrom_imp_ctx* c, int order) {
  HROM_CK(cudaMemcpyAsync(c->V, c->q1, c->g.D * sizeof(double), cudaMemcpyDeviceToDevice, c->st));
  hrom_status s = newton(c, order, c->q1, order == 2 ? c->q2 : c->q1, nullptr, nullptr, nullptr, c->V, nullptr, c->g.N);
  if (s != HROM_OK) return s;
  int st = 0;
  if ((s = read_newton(c, &st)) != HROM_OK) return s;
  if (st < 0) return HROM_E_POSITIVITY;  // the HDM itself failed (latched as a device failure)
  c->newton_its += st;
  return HROM_OK;
}

// hybrid step (Alg. 1 lines 6-14 with the subiterations of P:317-343) into c->V; returns
// kind 1, or 2 when it escalated to a full solve (failed partial Newton or positivity)
hrom_status hybrid_solve(hrom_imp_ctx* c, int order, int* kind) {
  hrom_ctx* x = c->aux;
  const Geo& xg = x->g;
  const double* qm2 = order == 2 ? c->q2 : c->q1;
  hrom_status s;
  basis_join(x);
  // unknown flags from S-hat (the context's current sets), the list is the sets' L_S
  flags_from_mask_kernel<<<c->nsm, 256, 0, c->st>>>(c->g, xg.wpr, x->b.masks + (int64_t)M_S * x->mwords, c->flags);
  HROM_LAUNCH_CK();
  const int32_t* Sl = x->b.lists + (int64_t)L_S * xg.N;
  const int32_t* Sn = x->b.counts + L_S;
  // |S-hat| and |B| on the host: the solve and the filter size their grids by them (one block,
  // block barriers only, when the set fits)
  HROM_CK(cudaMemcpyAsync(c->hint + 6, x->b.counts, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, c->st));
  HROM_CK(cudaStreamSynchronize(c->st));
  const int nS = c->hint[6 + L_S], nB = c->hint[6 + L_B];
  HROM_CK(cudaMemcpyAsync(c->V, c->q1, c->g.D * sizeof(double), cudaMemcpyDeviceToDevice, c->st));
  HROM_CK(cudaMemsetAsync(c->yprev, 0, kMaxR * sizeof(double), c->st));
  const int gm = x->P.gather_mode;
  x->P.gather_mode = 1;  // the gathered Gram of the P rows from scratch (no incremental bookkeeping)
  bool failed = false;
  int J = 0;
  for (int j = 1; j <= c->I.j_max; ++j) {
    if ((s = newton(c, order, c->q1, qm2, Sl, Sn, c->flags, c->V, nullptr, nS)) != HROM_OK) break;
    // y = (P^T Phi)^+ P^T (v - psi) on the rows of P (Eq. 8), then v := psi + Phi y off S-hat
    // (S-tilde included: the next subiteration's frozen values, Alg. 1 line 10)
    if ((s = gram_gathered(x, plain(c->V))) != HROM_OK) break;
    if ((s = small_solve(x)) != HROM_OK) break;
    HROM_CK(cudaMemsetAsync(x->b.eps, 0, xg.N * sizeof(double), c->st));
    if ((s = launch_fill(x, x->win, 0, plain(c->V), plain(c->V), false)) != HROM_OK) break;
    if ((s = launch_eps_cells(x)) != HROM_OK) break;
    ycheck_kernel<<<1, 32, 0, c->st>>>(x->b.y, c->yprev, x->b.ireg, x->r, c->rstat + 1);
    HROM_LAUNCH_CK();
    HROM_CK(cudaMemcpyAsync(c->hres, c->rstat + 1, sizeof(double), cudaMemcpyDeviceToHost, c->st));
    int st = 0;
    if ((s = read_newton(c, &st)) != HROM_OK) break;
    J = j;
    if (st < 0) {
      failed = true;
      break;
    }
    c->newton_its += st;
    if (j > 1 && c->hres[0] < c->I.eps_y) break;
  }
  x->P.gather_mode = gm;
  if (s != HROM_OK) return s;
  c->J = J;
  *kind = 1;
  if (!failed) {
    // filter gated by the implicit residual on the band, indicator on kept cells
    if (c->P.n_filter_orders > 0 && c->P.filter_max_sweeps > 0) {
      if ((s = filter_launch(c, order, c->q1, qm2, c->V, x->b.lists + (int64_t)L_B * xg.N, x->b.counts + L_B, c->kept,
                             x->b.eps, nB)) != HROM_OK)
        return s;
    }
    HROM_CK(cudaMemsetAsync(c->posflag, 0, sizeof(int), c->st));
    positivity_flag_kernel<<<c->nsm, 256, 0, c->st>>>(c->g, c->V, c->posflag);
    HROM_LAUNCH_CK();
    HROM_CK(cudaMemcpyAsync(c->hint + 2, c->posflag, sizeof(int), cudaMemcpyDeviceToHost, c->st));
    HROM_CK(cudaStreamSynchronize(c->st));
    if (c->hint[2]) failed = true;
  }
  if (failed) {  // escalation: the step is redone as a full HDM step
    if ((s = full_solve(c, order)) != HROM_OK) return s;
    *kind = 2;
  }
  return HROM_OK;
}

}  // namespace

extern "C" {

hrom_status hrom_imp_create(const hrom_grid* grid, double gamma, const hrom_params* p, const hrom_imp_params* ip,
                            void* stream, hrom_imp_ctx** out) {
  if (!grid || !p || !ip || !out) return HROM_E_INVALID;
  *out = nullptr;
  if (grid->bc < 0 || grid->bc > 2) return HROM_E_INVALID;
  if (!(ip->dt > 0.0) || !(ip->eps_y > 0.0) || ip->j_max < 1 || !(ip->newton_tol > 0.0) || ip->newton_maxit < 1 ||
      (ip->flux != 0 && ip->flux != 1))
    return HROM_E_INVALID;
  hrom_grid ag = *grid;
  if (ag.bc == 2) ag.bc = 0;  // the sets' dilations treat walls like transmissive ends (no wrap)
  hrom_params ap = *p;
  ap.gather_mode = 1;
  hrom_ctx* aux = nullptr;
  hrom_status s = hrom_create(&ag, gamma, 0.5, &ap, stream, &aux);
  if (s != HROM_OK) return s;
  auto* c = new hrom_imp_ctx();
  c->aux = aux;
  c->P = ap;
  c->I = *ip;
  c->st = (cudaStream_t)stream;
  c->nsm = aux->nsm;
  IGeo& g = c->g;
  g.dim = aux->g.dim;
  g.nx = aux->g.nx;
  g.ny = aux->g.ny;
  g.c = aux->g.c;
  g.bc = grid->bc;
  g.recon = grid->recon;
  g.flux = ip->flux;
  g.N = (int)aux->g.N;
  g.D = (int)aux->g.D;
  g.dx = aux->g.dx;
  g.dy = aux->g.dy;
  g.gamma = gamma;
  c->Dp = aux->g.Dp;
  {  // the residual's flux temporaries need more than the default 1 KB of stack per thread
    size_t lim = 0;
    cudaDeviceGetLimit(&lim, cudaLimitStackSize);
    if (lim < 4096) cudaDeviceSetLimit(cudaLimitStackSize, 4096);
  }
  // cooperative grids: one block per SM at most, and no more blocks than the work needs
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, newton_kernel<false>, NK_T, 0);
  const int want = std::max(1, std::min(c->nsm, (g.N + 15) / 16));
  c->nk_grid = std::max(1, std::min(want, occ * c->nsm));
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, imp_filter_kernel<false>, FI_T, 0);
  c->fi_grid = std::max(1, std::min(want, occ * c->nsm));
  bool ok = true;
  auto al = [&](auto** ptr, size_t n) {
    if (cudaMalloc((void**)ptr, n) != cudaSuccess) ok = false;
    else cudaMemset(*ptr, 0, n);
  };
  const size_t vb = c->Dp * sizeof(double);
  al(&c->q1, vb); al(&c->q2, vb); al(&c->V, vb); al(&c->qt, vb); al(&c->R, vb); al(&c->Rt, vb); al(&c->dq, vb);
  al(&c->Vk, vb * (kMaxKrylov + 1)); al(&c->wv, vb); al(&c->vp, vb); al(&c->vpp, vb); al(&c->vorig, vb);
  al(&c->part, 64 * 32 * sizeof(double) + 4096 * sizeof(double));
  al(&c->yprev, kMaxR * sizeof(double));
  al(&c->ff, (size_t)16 * g.N * sizeof(double));
  al(&c->rstat, 4 * sizeof(double));
  al(&c->flags, g.N);
  al(&c->keep, g.N);
  al(&c->kept, g.N);
  al(&c->list, g.N * sizeof(int32_t));
  al(&c->count, 4 * sizeof(int32_t));
  al(&c->istat, 4 * sizeof(int32_t));
  al(&c->fsweeps, 4 * sizeof(int32_t));
  al(&c->posflag, 4 * sizeof(int));
  al(&c->tdbg, 16 * sizeof(long long));
  if (cudaMallocHost((void**)&c->hres, 4 * sizeof(double)) != cudaSuccess) ok = false;
  if (cudaMallocHost((void**)&c->hint, 16 * sizeof(int32_t)) != cudaSuccess) ok = false;
  if (!ok) {
    hrom_imp_destroy(c);
    return HROM_E_NOMEM;
  }
  *out = c;
  return HROM_OK;
}

void hrom_imp_destroy(hrom_imp_ctx* c) {
  if (!c) return;
  if (c->st) cudaStreamSynchronize(c->st);
  for (void* ptr : {(void*)c->q1, (void*)c->q2, (void*)c->V, (void*)c->qt, (void*)c->R, (void*)c->Rt, (void*)c->dq,
                    (void*)c->Vk, (void*)c->wv, (void*)c->vp, (void*)c->vpp, (void*)c->vorig, (void*)c->part,
                    (void*)c->yprev, (void*)c->rstat, (void*)c->ff, (void*)c->flags, (void*)c->keep, (void*)c->kept, (void*)c->list,
                    (void*)c->count, (void*)c->istat, (void*)c->fsweeps, (void*)c->posflag, (void*)c->tdbg})
    if (ptr) cudaFree(ptr);
  if (c->hres) cudaFreeHost(c->hres);
  if (c->hint) cudaFreeHost(c->hint);
  if (c->aux) hrom_destroy(c->aux);
  delete c;
}

hrom_status hrom_imp_set_state(hrom_imp_ctx* c, const double* any_q) {
  if (!c || !any_q) return HROM_E_INVALID;
  hrom_status s = hrom_set_state(c->aux, any_q);
  if (s != HROM_OK) return s;
  c->k = 0;
  c->newton_total = 0;
  return HROM_OK;
}

hrom_status hrom_imp_get_state(hrom_imp_ctx* c, double* any_q) {
  if (!c || !any_q) return HROM_E_INVALID;
  return hrom_get_state(c->aux, any_q);
}

hrom_status hrom_imp_step(hrom_imp_ctx* c, int32_t* dev_count_out) {
  if (!c) return HROM_E_INVALID;
  if (c->k < 0) return HROM_E_STATE;
  hrom_ctx* x = c->aux;
  const int64_t kn = c->k + 1;
  const int w = x->w;
  const int64_t z = c->P.full_period;
  const bool full = (kn + 1 <= w) || (z > 0 && kn % z == 0);  // Alg. 1 line 3
  const int order = kn == 1 ? 1 : 2;                            // BDF1 start (A39)
  hrom_status s;
  basis_join(x);
  if ((s = slot_copy(c, c->k, nullptr, c->q1)) != HROM_OK) return s;
  if (order == 2 && (s = slot_copy(c, c->k - 1, nullptr, c->q2)) != HROM_OK) return s;
  c->J = 0;
  c->newton_its = 0;
  c->prods = 0;
  int kind = 0;
  if (full || !x->basis_ready || !x->sets_ready) {
    if ((s = full_solve(c, order)) != HROM_OK) return s;
    kind = 0;
    if (dev_count_out) HROM_CK(cudaMemcpyAsync(dev_count_out, &c->g.N, sizeof(int32_t), cudaMemcpyHostToDevice, c->st));
  } else {
    if ((s = hybrid_solve(c, order, &kind)) != HROM_OK) return s;
    if (dev_count_out) {
      if (kind == 1)
        HROM_CK(cudaMemcpyAsync(dev_count_out, x->b.counts + L_S, sizeof(int32_t), cudaMemcpyDeviceToDevice, c->st));
      else
        HROM_CK(cudaMemcpyAsync(dev_count_out, &c->g.N, sizeof(int32_t), cudaMemcpyHostToDevice, c->st));
    }
  }
  c->kind = kind;
  c->newton_total += c->newton_its;
  // gamma_kn into the window ring, then the explicit machinery's bookkeeping of a new snapshot
  if ((s = slot_copy(c, kn, c->V, nullptr)) != HROM_OK) return s;
  x->k = kn;
  x->smax_k = -1;
  x->points_used = (kind == 1 && x->P.odeim_points > 0) ? x->odeim_n : 0;
  x->last_hybrid = false;
  x->full_since_update = kind == 0;  // the projection indicator follows full steps only (G8)
  x->gram_row_ready = false;
  x->sets_ready = false;
  x->eps_sparse = false;
  c->k = kn;
  if (kn >= w - 1) {
    if (z > 0 && (kn + 1) % z == 0) {  // no update before a full step; its Gram row is owed
      if (x->n_owed == 4) {
        for (int i = 0; i < 3; ++i) x->owed_rows[i] = x->owed_rows[i + 1];
        x->n_owed = 3;
      }
      x->owed_rows[x->n_owed++] = kn;
      x->full_since_update = false;
    } else {
      if ((s = hrom_update_basis(x)) != HROM_OK) return s;
      s = c->P.sample_mode == 1 ? hrom_sample_rre(x, c->P.rre_delta, nullptr, nullptr, nullptr, nullptr)
                                : hrom_sample(x, c->P.sample_fraction, nullptr, nullptr, nullptr, nullptr);
      if (s != HROM_OK) return s;
    }
  }
  return HROM_OK;
}

hrom_status hrom_imp_stats(hrom_imp_ctx* c, int32_t* host_out) {
  if (!c || !host_out) return HROM_E_INVALID;
  host_out[0] = c->kind;
  host_out[1] = c->J;
  host_out[2] = c->newton_its;
  host_out[3] = c->prods;
  host_out[4] = (int32_t)c->aux->points_used;
  return HROM_OK;
}

hrom_status hrom_imp_get_mask(hrom_imp_ctx* c, uint32_t* any_mask) { return c ? hrom_get_mask(c->aux, any_mask) : HROM_E_INVALID; }
hrom_status hrom_imp_get_indicator(hrom_imp_ctx* c, double* any_eps) {
  return c ? hrom_get_indicator(c->aux, any_eps) : HROM_E_INVALID;
}
hrom_status hrom_imp_get_y(hrom_imp_ctx* c, double* any_y) { return c ? hrom_get_y(c->aux, any_y) : HROM_E_INVALID; }
int64_t hrom_imp_mask_words(const hrom_imp_ctx* c) { return c ? c->aux->mwords : 0; }
hrom_status hrom_imp_sync(hrom_imp_ctx* c) { return c ? hrom_sync(c->aux) : HROM_E_INVALID; }
int32_t hrom_imp_effective_rank(hrom_imp_ctx* c) { return c ? hrom_effective_rank(c->aux) : -1; }

hrom_status hrom_imp_residual(hrom_imp_ctx* c, int32_t order, const double* dev_q, const double* dev_qm1,
                              const double* dev_qm2, double* dev_R) {
  if (!c || !dev_q || !dev_qm1 || !dev_R || (order != 1 && order != 2) || (order == 2 && !dev_qm2))
    return HROM_E_INVALID;
  residual_all_kernel<<<c->nsm * 2, 256, 0, c->st>>>(c->g, bdf_of(c, order), dev_q, dev_qm1, order == 2 ? dev_qm2 : dev_qm1,
                                                      dev_R);
  HROM_LAUNCH_CK();
  return HROM_OK;
}

hrom_status hrom_imp_newton(hrom_imp_ctx* c, int32_t order, const double* dev_qm1, const double* dev_qm2,
                            const uint32_t* dev_mask, double* dev_q, int32_t* host_iters) {
  if (!c || !dev_qm1 || !dev_q || (order != 1 && order != 2) || (order == 2 && !dev_qm2)) return HROM_E_INVALID;
  hrom_status s;
  c->prods = 0;
  if (dev_mask) {
    flags_from_mask_kernel<<<c->nsm, 256, 0, c->st>>>(c->g, c->aux->g.wpr, dev_mask, c->flags);
    HROM_LAUNCH_CK();
    list_from_flags_kernel<<<1, 1024, 0, c->st>>>(c->g.N, c->flags, c->list, c->count);
    HROM_LAUNCH_CK();
    HROM_CK(cudaMemcpyAsync(c->hint + 6, c->count, sizeof(int32_t), cudaMemcpyDeviceToHost, c->st));
    HROM_CK(cudaStreamSynchronize(c->st));
    s = newton(c, order, dev_qm1, order == 2 ? dev_qm2 : dev_qm1, c->list, c->count, c->flags, dev_q, nullptr,
               c->hint[6]);
  } else {
    s = newton(c, order, dev_qm1, order == 2 ? dev_qm2 : dev_qm1, nullptr, nullptr, nullptr, dev_q, nullptr, c->g.N);
  }
  if (s != HROM_OK) return s;
  int st = 0;
  if ((s = read_newton(c, &st)) != HROM_OK) return s;
  if (host_iters) *host_iters = st;
  return st < 0 ? HROM_E_POSITIVITY : HROM_OK;
}

hrom_status hrom_imp_filter(hrom_imp_ctx* c, int32_t order, const double* dev_qm1, const double* dev_qm2,
                            const uint32_t* dev_mask, double* dev_v, uint8_t* dev_kept_out, int32_t* host_sweeps) {
  if (!c || !dev_qm1 || !dev_mask || !dev_v || (order != 1 && order != 2) || (order == 2 && !dev_qm2))
    return HROM_E_INVALID;
  hrom_ctx* x = c->aux;
  hrom_status s;
  if ((s = build_sets(x, dev_mask)) != HROM_OK) return s;
  x->sets_ready = true;
  HROM_CK(cudaMemcpyAsync(c->hint + 6, x->b.counts + L_B, sizeof(int32_t), cudaMemcpyDeviceToHost, c->st));
  HROM_CK(cudaStreamSynchronize(c->st));
  if ((s = filter_launch(c, order, dev_qm1, order == 2 ? dev_qm2 : dev_qm1, dev_v, x->b.lists + (int64_t)L_B * x->g.N,
                         x->b.counts + L_B, dev_kept_out ? dev_kept_out : c->kept, nullptr, c->hint[6])) != HROM_OK)
    return s;
  if (host_sweeps) {
    HROM_CK(cudaMemcpyAsync(c->hint + 3, c->fsweeps, 3 * sizeof(int32_t), cudaMemcpyDeviceToHost, c->st));
    HROM_CK(cudaStreamSynchronize(c->st));
    for (int i = 0; i < 3; ++i) host_sweeps[i] = i < c->P.n_filter_orders ? c->hint[3 + i] : 0;
  }
  return HROM_OK;
}

hrom_status hrom_imp_debug_timers(hrom_imp_ctx* c, int64_t* host_out) {
  if (!c || !host_out) return HROM_E_INVALID;
  HROM_CK(cudaMemcpyAsync(host_out, c->tdbg, 10 * sizeof(long long), cudaMemcpyDeviceToHost, c->st));
  HROM_CK(cudaStreamSynchronize(c->st));
  HROM_CK(cudaMemsetAsync(c->tdbg, 0, 16 * sizeof(long long), c->st));
  return HROM_OK;
}

hrom_status hrom_imp_get_band(hrom_imp_ctx* c, int32_t* any_list, int32_t* any_count) {
  if (!c || !any_list || !any_count) return HROM_E_INVALID;
  hrom_ctx* x = c->aux;
  HROM_CK(cudaMemcpyAsync(any_count, x->b.counts + L_B, sizeof(int32_t), cudaMemcpyDefault, c->st));
  HROM_CK(cudaMemcpyAsync(any_list, x->b.lists + (int64_t)L_B * x->g.N, x->g.N * sizeof(int32_t), cudaMemcpyDefault,
                          c->st));
  return HROM_OK;
}

// replay hook: window gamma_{k-w}..gamma_k (oldest first) and S-hat_{k+1}; the basis as after step k
hrom_status hrom_imp_set_window(hrom_imp_ctx* c, int64_t k, const double* any_snaps, int32_t nsnaps,
                                const uint32_t* any_mask_next) {
  if (!c) return HROM_E_INVALID;
  hrom_status s = hrom_set_window(c->aux, k, any_snaps, nsnaps, any_mask_next);
  if (s != HROM_OK) return s;
  c->k = k;
  return HROM_OK;
}

}  // extern "C"
