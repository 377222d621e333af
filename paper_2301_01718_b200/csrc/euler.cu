// euler.cu -- H1 (CFL dt), H2 (full SSP-RK3 step) and H3 (masked step) kernels.
//
// Paper: Euler equations + ideal gas, MUSCL + minmod, explicit
// F_k (remark P:345-347).  BASELINE.json: Rusanov flux, SSP-RK3 (BJ:7-10).
// The full and the masked step run the SAME kernel (list == nullptr means all cells),
// so the S-hat rows of a masked step are bitwise the rows of the full step (Eq. 7,
// exact restriction, reading A9).  States are addressed through SRef (slab ring slot
// or plain vector, internal.cuh).
#include <algorithm>
#include <cfloat>
#include "internal.cuh"
#include "async.cuh"

namespace hrom {
namespace {

__device__ __forceinline__ double minmod(double a, double b) {
  if (a * b <= 0.0) return 0.0;
  return a > 0.0 ? fmin(a, b) : fmax(a, b);
}

template <int DIM>
__device__ __forceinline__ double pressure(const double* U, double gm1) {
  double m2 = U[1] * U[1];
  if (DIM == 2) m2 += U[2] * U[2];
  return gm1 * (U[DIM + 1] - 0.5 * m2 / U[0]);
}

// pressure with the reciprocal density supplied (one division per state instead of three)
template <int DIM>
__device__ __forceinline__ double pressure_r(const double* U, double rinv, double gm1) {
  double m2 = U[1] * U[1];
  if (DIM == 2) m2 += U[2] * U[2];
  return gm1 * (U[DIM + 1] - 0.5 * m2 * rinv);
}

// Rusanov flux along AXIS from reconstructed face states (O5).  1/rho is formed once per state
// (u = m / rho, p, c = sqrt(gamma p / rho) all use it): equal to the divided forms to ~1 ulp.
template <int DIM, int AXIS>
__device__ __forceinline__ void rusanov(const double* UL, const double* UR, double gamma, double* F) {
  constexpr int C = DIM + 2;
  const double gm1 = gamma - 1.0;
  const double rL = 1.0 / UL[0], rR = 1.0 / UR[0];
  const double pL = pressure_r<DIM>(UL, rL, gm1), pR = pressure_r<DIM>(UR, rR, gm1);
  const double uL = UL[1 + AXIS] * rL, uR = UR[1 + AXIS] * rR;
  const double cL = sqrt(gamma * pL * rL), cR = sqrt(gamma * pR * rR);
  const double a = fmax(fabs(uL) + cL, fabs(uR) + cR);
  double FL[C], FR[C];
  FL[0] = UL[1 + AXIS];
  FR[0] = UR[1 + AXIS];
#pragma unroll
  for (int d = 0; d < DIM; ++d) {
    FL[1 + d] = UL[1 + d] * uL + (d == AXIS ? pL : 0.0);
    FR[1 + d] = UR[1 + d] * uR + (d == AXIS ? pR : 0.0);
  }
  FL[C - 1] = (UL[C - 1] + pL) * uL;
  FR[C - 1] = (UR[C - 1] + pR) * uR;
#pragma unroll
  for (int v = 0; v < C; ++v) F[v] = 0.5 * (FL[v] + FR[v]) - 0.5 * a * (UR[v] - UL[v]);
}

// flux through the face between cells a and b (am left of a, bp right of b)
template <int DIM, int AXIS, int RECON>
__device__ __forceinline__ void face_flux(const double* Uam, const double* Ua, const double* Ub,
                                          const double* Ubp, double gamma, double* F) {
  constexpr int C = DIM + 2;
  double UL[C], UR[C];
#pragma unroll
  for (int v = 0; v < C; ++v) {
    if (RECON == 2) {
      UL[v] = Ua[v] + 0.5 * minmod(Ua[v] - Uam[v], Ub[v] - Ua[v]);
      UR[v] = Ub[v] - 0.5 * minmod(Ub[v] - Ua[v], Ubp[v] - Ub[v]);
    } else {
      UL[v] = Ua[v];
      UR[v] = Ub[v];
    }
  }
  rusanov<DIM, AXIS>(UL, UR, gamma, F);
}

__device__ __forceinline__ int wrap(int i, int n, int bc) {
  if (bc == 1) {
    // stencil offsets are small: one conditional add / subtract almost always lands in range
    if (i < 0) i += n;
    else if (i >= n) i -= n;
    if ((unsigned)i >= (unsigned)n) {
      i = i % n;
      if (i < 0) i += n;
    }
    return i;
  }
  return i < 0 ? 0 : (i >= n ? n - 1 : i);
}

// L at cell (i, j) of q (O6); loads the cross stencil of radius RECON
template <int DIM, int RECON>
__device__ __forceinline__ void cell_rhs(const Geo& g, const SRef q, int i, int j, double* L) {
  constexpr int C = DIM + 2;
  constexpr int R = RECON;
  double Ux[2 * R + 1][C];
  const int64_t row = (int64_t)j * g.nx;
#pragma unroll
  for (int m = -R; m <= R; ++m) {
    const int64_t n = row + wrap(i + m, g.nx, g.bc);
#pragma unroll
    for (int v = 0; v < C; ++v) Ux[m + R][v] = __ldg(q.p + sidx(q, v * g.N + n));
  }
  double Fp[C], Fm[C];
  // right face (i, i+1) uses cells i-1, i, i+1, i+2; left face uses i-2 .. i+1
  face_flux<DIM, 0, RECON>(Ux[R - (R == 2 ? 1 : 0)], Ux[R], Ux[R + 1], Ux[R + (R == 2 ? 2 : 1)], g.gamma, Fp);
  face_flux<DIM, 0, RECON>(Ux[0], Ux[R - 1], Ux[R], Ux[R + (R == 2 ? 1 : 0)], g.gamma, Fm);
#pragma unroll
  for (int v = 0; v < C; ++v) L[v] = -div_dx(g, Fp[v] - Fm[v]);
  if (DIM == 2) {
    double Uy[2 * R + 1][C];
#pragma unroll
    for (int m = -R; m <= R; ++m) {
      if (m == 0) {
#pragma unroll
        for (int v = 0; v < C; ++v) Uy[R][v] = Ux[R][v];
        continue;
      }
      const int64_t n = (int64_t)wrap(j + m, g.ny, g.bcy) * g.nx + i;
#pragma unroll
      for (int v = 0; v < C; ++v) Uy[m + R][v] = __ldg(q.p + sidx(q, v * g.N + n));
    }
    double Gp[C], Gm[C];
    face_flux<DIM, DIM - 1, RECON>(Uy[R - (R == 2 ? 1 : 0)], Uy[R], Uy[R + 1], Uy[R + (R == 2 ? 2 : 1)], g.gamma, Gp);
    face_flux<DIM, DIM - 1, RECON>(Uy[0], Uy[R - 1], Uy[R], Uy[R + (R == 2 ? 1 : 0)], g.gamma, Gm);
#pragma unroll
    for (int v = 0; v < C; ++v) L[v] = L[v] - div_dy(g, Gp[v] - Gm[v]);
  }
}

// One SSP-RK3 stage (O8, printed order) on all cells (list == nullptr) or a cell list.
template <int DIM, int RECON>
__global__ void __launch_bounds__(256) stage_kernel(Geo g, int stage, const SRef qn, const SRef qin, const SRef out,
                                                    const int32_t* __restrict__ list,
                                                    const int32_t* __restrict__ count,
                                                    const double* __restrict__ dtp,
                                                    const unsigned long long* __restrict__ run_if,
                                                    int32_t* __restrict__ esc_count) {
  constexpr int C = DIM + 2;
  if (run_if && *run_if == ~0ull) return;  // conditional full-step re-run (positivity escalation)
  if (run_if && esc_count && stage == 1 && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(esc_count, 1);
  const int64_t total = list ? (int64_t)(*count) : g.N;
  const double dt = *dtp;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = list ? (int64_t)list[t] : t;
    const int i = (int)(n % g.nx), j = (int)(n / g.nx);
    double L[C];
    cell_rhs<DIM, RECON>(g, qin, i, j, L);
#pragma unroll
    for (int v = 0; v < C; ++v) {
      const int64_t e = v * g.N + n;
      const double un = qn.p[sidx(qn, e)];
      double r;
      if (stage == 1) r = un + dt * L[v];
      else if (stage == 2) r = 0.75 * un + 0.25 * (qin.p[sidx(qin, e)] + dt * L[v]);
      else r = (1.0 / 3.0) * un + (2.0 / 3.0) * (qin.p[sidx(qin, e)] + dt * L[v]);
      out.p[sidx(out, e)] = r;
    }
  }
}

// 2-D SSP-RK3 stage on 32 x 8 cell tiles (one thread per cell): the cross stencil region is
// staged in shared memory once, every face flux is computed ONCE (x-faces 33 x 8, y-faces 32 x 9)
// and shared by its two cells.  Same face_flux arithmetic on the same operands and the same
// L = -(Fp - Fm)/dx - (Gp - Gm)/dy order as cell_rhs: bitwise identical to the per-cell kernel.
// mask (nullable): the stage's cell set (row-padded bitmap; one 32-cell tile row = one word);
// tiles without an active cell exit at once, inactive cells of active tiles are not written.
constexpr int TX = 32, TY = 8, TH = 2;  // tile, halo (MUSCL radius)
// six resident blocks per SM (40 registers, ~120 B of spills): the kernel is bound by barrier and
// memory latency, so the occupancy pays (2048^2 full step 0.90 -> 0.64 ms; 5 blocks: 0.67, 8: 0.85)
#ifndef STAGE_MINB
#define STAGE_MINB 6
#endif
#ifndef STAGE_MINB_MASKED
#define STAGE_MINB_MASKED 4
#endif
template <int RECON, bool MASKED>
__global__ void __launch_bounds__(TX * TY, MASKED ? STAGE_MINB_MASKED : STAGE_MINB) stage_tile_kernel(Geo g, int stage, const SRef qn, const SRef qin,
                                                           const SRef out, const uint32_t* __restrict__ mask,
                                                           const double* __restrict__ dtp,
                                                           const int32_t* __restrict__ tiles,
                                                           const int32_t* __restrict__ ntiles_p,
                                                           unsigned long long* __restrict__ smax_out) {
  constexpr int C = 4, R = RECON;
  constexpr int SX = TX + 2 * TH, SY = TY + 2 * TH;
  __shared__ double U[C][SY][SX];        // cross region (corners unused)
  __shared__ double Fx[C][TY][TX + 1];   // x-face i - 1/2 of tile column i
  __shared__ double Fy[C][TY + 1][TX];   // y-face j - 1/2 of tile row j
  __shared__ int any;
  const int tx = threadIdx.x % TX, ty = threadIdx.x / TX;
  const int ntx = (g.nx + TX - 1) / TX;
  // tiles: persistent loop over the listed active tiles (masked stages), or one tile per block
  // MASKED = false (full step): one tile per block, no bitmap, no tile list
  const int ntiles = MASKED ? *ntiles_p : (int)gridDim.x;
  for (int it = blockIdx.x; it < ntiles; it += (MASKED ? (int)gridDim.x : ntiles)) {
    const int tile = MASKED ? tiles[it] : it;
    const int bx = tile % ntx, by = tile / ntx;
    const int i0 = bx * TX, j0 = by * TY;
    const int i = i0 + tx, j = j0 + ty;
    // active for this stage's set?
    uint32_t myword = 0;
    if (MASKED) {
      __syncthreads();  // U / Fx / Fy / any of the previous tile are consumed
      if (threadIdx.x == 0) any = 0;
      __syncthreads();
      if (j < g.ny) myword = mask[(int64_t)j * g.wpr + bx];
      if (tx == 0 && myword) any = 1;
      __syncthreads();
      if (!any) continue;  // uniform
    }
    // stage the cross region: rows j0-2 .. j0+9 over the tile columns, and the x-halo columns
    for (int idx = threadIdx.x; idx < SY * SX; idx += TX * TY) {
      const int ly = idx / SX, lx = idx % SX;
      const bool xin = lx >= TH && lx < TH + TX, yin = ly >= TH && ly < TH + TY;
      if (!xin && !yin) continue;  // corner
      const int gi = wrap(i0 + lx - TH, g.nx, g.bc), gj = wrap(j0 + ly - TH, g.ny, g.bcy);
      const int64_t n = (int64_t)gj * g.nx + gi;
      // asynchronous 8-byte copies straight into shared memory: every copy of a thread is in flight
      // at once and none passes through a register
#pragma unroll
      for (int v = 0; v < C; ++v) cp_async8(&U[v][ly][lx], qin.p + sidx(qin, v * g.N + n));
    }
    cp_async_commit();
    // gamma_n of this thread's cell for the stage combination: issued now, consumed after the
    // flux phase (stage 1 combines with the staged value itself)
    const bool mine = i < g.nx && j < g.ny && (!MASKED || ((myword >> tx) & 1u));
    double unv[C];
#pragma unroll
    for (int v = 0; v < C; ++v)
      unv[v] = (mine && stage != 1) ? qn.p[sidx(qn, v * g.N + (int64_t)j * g.nx + i)] : 0.0;
    cp_async_wait<0>();
    __syncthreads();
    // x-faces: face f between local columns f-1 and f (f = 0..TX), rows 0..TY-1
    for (int f = threadIdx.x; f < (TX + 1) * TY; f += TX * TY) {
      const int fy = f / (TX + 1), fx = f % (TX + 1);
      const int ly = fy + TH, lx = fx + TH;  // cell "b" (right of the face) in the staged region
      double Uam[C], Ua[C], Ub[C], Ubp[C], F[C];
#pragma unroll
      for (int v = 0; v < C; ++v) {
        Uam[v] = U[v][ly][lx - (R == 2 ? 2 : 1)];
        Ua[v] = U[v][ly][lx - 1];
        Ub[v] = U[v][ly][lx];
        Ubp[v] = U[v][ly][lx + (R == 2 ? 1 : 0)];
      }
      face_flux<2, 0, RECON>(Uam, Ua, Ub, Ubp, g.gamma, F);
#pragma unroll
      for (int v = 0; v < C; ++v) Fx[v][fy][fx] = F[v];
    }
    // y-faces: face f between local rows f-1 and f (f = 0..TY), columns 0..TX-1
    for (int f = threadIdx.x; f < (TY + 1) * TX; f += TX * TY) {
      const int fy = f / TX, fx = f % TX;
      const int ly = fy + TH, lx = fx + TH;
      double Uam[C], Ua[C], Ub[C], Ubp[C], F[C];
#pragma unroll
      for (int v = 0; v < C; ++v) {
        Uam[v] = U[v][ly - (R == 2 ? 2 : 1)][lx];
        Ua[v] = U[v][ly - 1][lx];
        Ub[v] = U[v][ly][lx];
        Ubp[v] = U[v][ly + (R == 2 ? 1 : 0)][lx];
      }
      face_flux<2, 1, RECON>(Uam, Ua, Ub, Ubp, g.gamma, F);
#pragma unroll
      for (int v = 0; v < C; ++v) Fy[v][fy][fx] = F[v];
    }
    __syncthreads();
    double smx = 0.0;  // H1 of the NEXT step, fused into the last stage of a full step (smax_out)
    if (mine) {
      const double dt = *dtp;
      const int64_t n = (int64_t)j * g.nx + i;
      double Unew[C];
#pragma unroll
      for (int v = 0; v < C; ++v) {
        double L = -div_dx(g, Fx[v][ty][tx + 1] - Fx[v][ty][tx]);
        L = L - div_dy(g, Fy[v][ty + 1][tx] - Fy[v][ty][tx]);
        const int64_t e = v * g.N + n;
        const double un = stage == 1 ? U[v][ty + TH][tx + TH] : unv[v];  // stage 1: qin = gamma_n
        double r;
        if (stage == 1) r = un + dt * L;
        else if (stage == 2) r = 0.75 * un + 0.25 * (U[v][ty + TH][tx + TH] + dt * L);
        else r = (1.0 / 3.0) * un + (2.0 / 3.0) * (U[v][ty + TH][tx + TH] + dt * L);
        out.p[sidx(out, e)] = r;
        Unew[v] = r;
      }
      if (!MASKED && smax_out) {
        // the divided forms of the CFL rule (O7), as smax_kernel: the same bits as a separate pass
        const double p = pressure<2>(Unew, g.gamma - 1.0);
        const double cs = sqrt(g.gamma * p / Unew[0]);
        smx = div_dx(g, fabs(Unew[1] / Unew[0]) + cs);
        smx = smx + div_dy(g, fabs(Unew[2] / Unew[0]) + cs);
      }
    }
    if (!MASKED && smax_out) {  // block maximum (NaN sticks), one integer atomicMax per tile
      double m = smx;
      if (m != m) m = __longlong_as_double(0x7ff8000000000000ll);
      for (int o = 16; o > 0; o >>= 1) {
        const double t = __shfl_xor_sync(0xffffffffu, m, o);
        if (!(t <= m)) m = t;
      }
      __shared__ double smw[TX * TY / 32];
      if ((threadIdx.x & 31) == 0) smw[threadIdx.x >> 5] = m;
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int k = 1; k < TX * TY / 32; ++k)
          if (!(smw[k] <= m)) m = smw[k];
        unsigned long long bits = (unsigned long long)__double_as_longlong(m);
        if (m != m) bits = 0x7ff8000000000000ull;
        atomicMax(smax_out, bits);
      }
    }
    if (!MASKED) break;
  }
}

// H1: max_n S_n with S_n = (|u|+c)/dx [+ (|v|+c)/dy]; S_n >= 0 so its IEEE bits order like
// the value and an integer atomicMax is exact and order-free (deterministic).
template <int DIM>
__global__ void __launch_bounds__(256) smax_kernel(Geo g, const SRef q, unsigned long long* __restrict__ smax,
                                                   int64_t n0, int64_t n1) {
  constexpr int C = DIM + 2;
  double m = 0.0;
  for (int64_t n = n0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < n1;
       n += (int64_t)gridDim.x * blockDim.x) {
    double U[C];
#pragma unroll
    for (int v = 0; v < C; ++v) U[v] = q.p[sidx(q, v * g.N + n)];
    // the divided forms of the CFL rule (O7): dt matches the oracle's bit for bit
    const double p = pressure<DIM>(U, g.gamma - 1.0);
    const double cs = sqrt(g.gamma * p / U[0]);
    double s = div_dx(g, fabs(U[1] / U[0]) + cs);
    if (DIM == 2) s = s + div_dy(g, fabs(U[2] / U[0]) + cs);
    if (!(s <= m)) m = s;  // NaN sticks
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double t = __shfl_xor_sync(0xffffffffu, m, o);
    if (!(t <= m)) m = t;
  }
  __shared__ double sm[8];
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
      if (!(sm[k] <= m)) m = sm[k];
    unsigned long long bits = (unsigned long long)__double_as_longlong(m);
    if (m != m) bits = 0x7ff8000000000000ull;  // canonical NaN (largest positive pattern class)
    atomicMax(smax, bits);
  }
}

__global__ void dt_finalize(const unsigned long long* smax, const unsigned long long* smax_alt,
                            const unsigned long long* esc, double cfl, double dt_override, double* dt,
                            unsigned long long* ureg) {
  // smax_alt: the escalated state's maximum when the previous step was redone as a full step
  const unsigned long long* src = (esc && *esc != ~0ull) ? smax_alt : smax;
  const double s = __longlong_as_double((long long)*src);
  // reset the registers of this step's positivity pass (maximum ureg[2], step flag ureg[3],
  // escalated maximum ureg[0]) -- no separate memsets on the critical path
  ureg[0] = 0ull;
  ureg[2] = 0ull;
  ureg[3] = ~0ull;
  *dt = dt_override > 0.0 ? dt_override : cfl / s;
}

// O11: lowest cell with rho <= 0 or p <= 0 (or NaN); fused with H1's max wave speed of the same
// state (the next step's dt reads it instead of a second pass over the state)
template <int DIM>
// Positivity (O11) and the wave-speed maximum of the next dt (H1) in one pass.  The oracle's
// divided forms (O7) are evaluated exactly only where they can matter: a cell is tested with
// the division-free p rho = (gamma - 1)(E rho - |m|^2 / 2) (positive with a 1e-10 relative margin
// => p > 0 in the exact form too) and its wave speed screened in fp32 (relative error < 1e-5);
// the exact divided s is computed when the screen comes within 1e-3 of the thread's running
// screened maximum (the cell that raised it was computed exactly, so no exact maximum is
// missed), and the exact p whenever the margin test is inconclusive.  Same bad-cell latch and
// maximum, bit for bit, at ~1/10 of the divisions.
__global__ void __launch_bounds__(256) positivity_kernel(Geo g, const SRef q, unsigned long long* __restrict__ bad,
                                                         unsigned long long* __restrict__ smax,
                                                         const unsigned long long* __restrict__ run_if,
                                                         int64_t n0, int64_t n1) {
  constexpr int C = DIM + 2;
  if (run_if && *run_if == ~0ull) return;
  const double gm1 = g.gamma - 1.0;
  double m = 0.0;
  float amax = 0.0f;  // running screened maximum (of cells not evaluated exactly, a lower bound)
  const float frdx = (float)(g.pow2 ? g.rdx : 1.0 / g.dx), frdy = (float)(g.pow2 ? g.rdy : 1.0 / g.dy);
  for (int64_t n = n0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < n1;
       n += (int64_t)gridDim.x * blockDim.x) {
    double U[C];
#pragma unroll
    for (int v = 0; v < C; ++v) U[v] = q.p[sidx(q, v * g.N + n)];
    double m2 = U[1] * U[1];
    if (DIM == 2) m2 += U[2] * U[2];
    const double pr = gm1 * fma(U[C - 1], U[0], -0.5 * m2);  // ~ p rho
    const bool sure = U[0] > 0.0 && pr > 1e-10 * gm1 * (fabs(U[C - 1]) * U[0] + 0.5 * m2);
    float sa = 0.0f;
    bool exact = !sure;
    if (sure) {
      const float rf = 1.0f / (float)U[0];
      const float cf = sqrtf((float)(g.gamma * pr)) * rf;
      sa = (fabsf((float)U[1]) * rf + cf) * frdx;
      if (DIM == 2) sa += (fabsf((float)U[2]) * rf + cf) * frdy;
      exact = !(sa < amax * 0.999f);  // NaN / inf: exact
      if (sa > amax) amax = sa;
    }
    if (exact) {
      // the divided forms of the CFL rule (O7): dt matches the oracle's bit for bit
      const double p = pressure<DIM>(U, gm1);
      if (!(U[0] > 0.0) || !(p > 0.0)) atomicMin(bad, (unsigned long long)n);
      const double cs = sqrt(g.gamma * p / U[0]);
      double sx = div_dx(g, fabs(U[1] / U[0]) + cs);
      if (DIM == 2) sx = sx + div_dy(g, fabs(U[2] / U[0]) + cs);
      if (!(sx <= m)) m = sx;  // NaN sticks
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double t = __shfl_xor_sync(0xffffffffu, m, o);
    if (!(t <= m)) m = t;
  }
  __shared__ double sm[8];
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k)
      if (!(sm[k] <= m)) m = sm[k];
    unsigned long long bits = (unsigned long long)__double_as_longlong(m);
    if (m != m) bits = 0x7ff8000000000000ull;
    atomicMax(smax, bits);
  }
}

}  // namespace

hrom_status launch_dt(hrom_ctx* c, SRef q, double dt_override, int64_t kq) {
  const unsigned long long* smax = c->b.ureg;
  const unsigned long long *alt = nullptr, *esc = nullptr;
  int nl = 1;
  if (dt_override <= 0.0) {
    if (c->smax_k == kq) {
      // computed by the positivity pass that closed step kq (ureg[2]); ureg[0] if that step
      // was redone as a full step (ureg[3] != ~0)
      smax = c->b.ureg + 2;
      alt = c->b.ureg;
      esc = c->b.ureg + 3;
    } else {
      HROM_CK(cudaMemsetAsync(c->b.ureg, 0, sizeof(unsigned long long), c->st));
      const int grid = c->nsm * 8;
      if (c->g.dim == 1) smax_kernel<1><<<grid, 256, 0, c->st>>>(c->g, q, c->b.ureg, 0, c->g.N);
      else smax_kernel<2><<<grid, 256, 0, c->st>>>(c->g, q, c->b.ureg, 0, c->g.N);
      HROM_LAUNCH_CK();
      ++nl;
    }
  }
  dt_finalize<<<1, 1, 0, c->st>>>(smax, alt, esc, c->g.cfl, dt_override, c->b.dreg, c->b.ureg);
  HROM_LAUNCH_CK();
  c->nlaunch += nl;
  return HROM_OK;
}

hrom_status launch_stage(hrom_ctx* c, int stage, SRef qn, SRef qin, SRef out, const int32_t* list, int list_idx,
                         double /*dt_override*/, const unsigned long long* run_if, bool fuse_smax) {
  // conditional (escalation) launches almost always exit at once: a small grid-stride grid
  const int grid = run_if ? c->nsm * 2 : c->nsm * 8;
  const int32_t* cnt = list ? c->b.counts + list_idx : nullptr;
  const Geo& g = c->g;
  int32_t* ec = c->b.ireg + 15;
  if (g.dim == 2 && !run_if) {
    // tile kernel: every face once; masked stages restrict to the set's bitmap (A1, A2, T)
    // masked stages: a persistent grid over the active tiles of A1 (listed by the sets kernel;
    // A1 >= A2 >= T), each tile re-checked against its own stage's bitmap
    const uint32_t* mask = list ? c->b.masks + (int64_t)list_idx * c->mwords : nullptr;
    const int tiles = ((g.nx + TX - 1) / TX) * ((g.ny + TY - 1) / TY);
    const int32_t* tl = list ? c->b.lists + (int64_t)L_A2 * g.N : nullptr;  // tile list (2-D)
    const int32_t* tn = c->b.counts + 10;
    const int grid = list ? std::min(tiles, 8 * c->nsm) : tiles;
    // fuse_smax (last stage of a full step over the whole grid): the new state's wave-speed maximum
    // goes to ureg[2] (zeroed by this step's dt_finalize), as after the positivity pass
    unsigned long long* sm = (fuse_smax && !list) ? c->b.ureg + 2 : nullptr;
    if (list) {
      if (g.recon == 1) stage_tile_kernel<1, true><<<grid, TX * TY, 0, c->st>>>(g, stage, qn, qin, out, mask, c->b.dreg, tl, tn, sm);
      else stage_tile_kernel<2, true><<<grid, TX * TY, 0, c->st>>>(g, stage, qn, qin, out, mask, c->b.dreg, tl, tn, sm);
    } else {
      if (g.recon == 1) stage_tile_kernel<1, false><<<grid, TX * TY, 0, c->st>>>(g, stage, qn, qin, out, mask, c->b.dreg, tl, tn, sm);
      else stage_tile_kernel<2, false><<<grid, TX * TY, 0, c->st>>>(g, stage, qn, qin, out, mask, c->b.dreg, tl, tn, sm);
    }
  } else if (g.dim == 1) {
    if (g.recon == 1) stage_kernel<1, 1><<<grid, 256, 0, c->st>>>(g, stage, qn, qin, out, list, cnt, c->b.dreg, run_if, ec);
    else stage_kernel<1, 2><<<grid, 256, 0, c->st>>>(g, stage, qn, qin, out, list, cnt, c->b.dreg, run_if, ec);
  } else {
    if (g.recon == 1) stage_kernel<2, 1><<<grid, 256, 0, c->st>>>(g, stage, qn, qin, out, list, cnt, c->b.dreg, run_if, ec);
    else stage_kernel<2, 2><<<grid, 256, 0, c->st>>>(g, stage, qn, qin, out, list, cnt, c->b.dreg, run_if, ec);
  }
  HROM_LAUNCH_CK();
  c->nlaunch += 1;
  return HROM_OK;
}

// O11 after a hybrid step: per-step flag ureg[3] and the wave-speed maximum ureg[2]; then, only
// if the flag is set (device-side condition, S:478 escalation): the step is redone as a full
// step from gamma_{k-1} with the same dt, re-checked (latched error ureg[1], maximum ureg[0]).
hrom_status launch_positivity_check(hrom_ctx* c, SRef q, int64_t n0, int64_t n1) {
  const int grid = c->nsm * 8;
  unsigned long long* u = c->b.ureg;
  if (n1 < 0) n1 = c->g.N;
  // ureg[0] = 0, ureg[2] = 0, ureg[3] = ~0 were set by this step's dt_finalize
  if (c->g.dim == 1) positivity_kernel<1><<<grid, 256, 0, c->st>>>(c->g, q, u + 3, u + 2, nullptr, n0, n1);
  else positivity_kernel<2><<<grid, 256, 0, c->st>>>(c->g, q, u + 3, u + 2, nullptr, n0, n1);
  HROM_LAUNCH_CK();
  c->nlaunch += 1;
  return HROM_OK;
}

hrom_status launch_positivity_redo(hrom_ctx* c, SRef qprev, SRef q, int64_t kq) {
  unsigned long long* u = c->b.ureg;
  hrom_status s;
  const SRef U1 = plain(c->b.U1), U2 = plain(c->b.U2);
  if ((s = launch_stage(c, 1, qprev, qprev, U1, nullptr, 0, 0.0, u + 3)) != HROM_OK) return s;
  if ((s = launch_stage(c, 2, qprev, U1, U2, nullptr, 0, 0.0, u + 3)) != HROM_OK) return s;
  if ((s = launch_stage(c, 3, qprev, U2, q, nullptr, 0, 0.0, u + 3)) != HROM_OK) return s;
  if (c->g.dim == 1) positivity_kernel<1><<<c->nsm * 2, 256, 0, c->st>>>(c->g, q, u + 1, u, u + 3, 0, c->g.N);
  else positivity_kernel<2><<<c->nsm * 2, 256, 0, c->st>>>(c->g, q, u + 1, u, u + 3, 0, c->g.N);
  HROM_LAUNCH_CK();
  c->nlaunch += 1;
  c->smax_k = kq;
  return HROM_OK;
}

hrom_status launch_positivity(hrom_ctx* c, SRef qprev, SRef q, int64_t kq) {
  hrom_status s = launch_positivity_check(c, q, 0, -1);
  if (s != HROM_OK) return s;
  return launch_positivity_redo(c, qprev, q, kq);
}

// H1's wave-speed maximum of q alone (row slabs exchange it before dt, slab.cu); *dev_out must be
// zeroed by the caller on the same stream
hrom_status launch_smax(hrom_ctx* c, SRef q, unsigned long long* dev_out, int64_t n0, int64_t n1) {
  const int grid = c->nsm * 8;
  if (c->g.dim == 1) smax_kernel<1><<<grid, 256, 0, c->st>>>(c->g, q, dev_out, n0, n1);
  else smax_kernel<2><<<grid, 256, 0, c->st>>>(c->g, q, dev_out, n0, n1);
  HROM_LAUNCH_CK();
  c->nlaunch += 1;
  return HROM_OK;
}

}  // namespace hrom
