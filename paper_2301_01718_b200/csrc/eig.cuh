// eig.cuh -- one-CTA symmetric eigen-solver for the small Gram matrices of H5 (G, r x r) and
// H11 (M = X^T X, w x w): the POD of the window (Eq. 8) and the pinv of the gappy
// least-squares normal matrix.  DESIGN.md §5 "eigen-solve".
//
//   1. Householder tridiagonalisation A = Q T Q^T (three block barriers per column);
//   2. all eigenvalues of T by multisection of Sturm counts (G lanes per eigenvalue, each lane
//      one Sturm count per round: log2(G) bits per round), descending;
//   3. the leading nvec eigenvectors of T by inverse iteration (one thread per vector, three
//      solves with the partially pivoted LU of T - lambda I), then two passes of classical
//      Gram-Schmidt in descending-eigenvalue order so that the vectors are orthonormal to
//      rounding also inside clusters (eigenvalue gaps below the iteration's resolution);
//   4. back-transformation Z <- Q Z, sign: largest |Z_ij| (ties: lowest i) positive.
//
// Cost ~ O(n^3 / threads) + O(n^2) dependent steps instead of the ~10 sweeps x (n - 1) rounds of
// two-sided Jacobi (2.2 ms for n = 64 on one SM, measured).  Accuracy: eigenvalues to
// ~4 eps ||T|| absolute, vectors to ~eps ||T|| / gap -- the same as any backward-stable solver
// applied to the (already rounded) Gram matrix.
#pragma once
#include <float.h>
#include "internal.cuh"

namespace hrom {

struct EigWork {
  double* d;     // kMaxSlots
  double* e;     // kMaxSlots
  double* tau;   // kMaxSlots
  double* vv;    // kMaxSlots
  double* pp;    // kMaxSlots
  double* red;   // 64 (reduction scratch)
  double* lam;   // n, descending
  double* Z;     // n x ldz, Z[i * ldz + j] = component i of eigenvector j
  int ldz;       // >= nvec_cap
  double* fac;   // 4 * n * ldz doubles: LU of T - lambda I per vector, [a][i][j]
  uint8_t* swp;  // n * ldz
};

__device__ __forceinline__ double eig_warp_sum(double s) {
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// number of eigenvalues of T (d, e2 = e^2) strictly below x
__device__ __forceinline__ int sturm_count(const double* d, const double* e2, int n, double x, double pivmin) {
  double q = d[0] - x;
  if (fabs(q) <= pivmin) q = -pivmin;
  int c = q < 0.0;
  for (int i = 1; i < n; ++i) {
    q = d[i] - x - e2[i - 1] / q;
    if (fabs(q) <= pivmin) q = -pivmin;
    c += q < 0.0;
  }
  return c;
}

// deterministic start vector entries in (-1, 1)
__device__ __forceinline__ double eig_start(int i, int j) {
  uint64_t z = 0x9E3779B97F4A7C15ull * (uint64_t)(i + 1) + 0xBF58476D1CE4E5B9ull * (uint64_t)(j + 7);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
}

// A (n x n symmetric, ld ldn, destroyed).  Returns nvec = min(nvec_cap, #{lam_j >= cut lam_0})
// (0 when lam_0 <= 0); lam (all n, descending) and Z[:, 0..nvec) are written.  All threads of
// the block must call it; blockDim.x a multiple of 32, >= 64.
__device__ int sym_eig(double* A, int n, int ldn, const EigWork& W, int nvec_cap, double cut,
                       int32_t* phase_kcycles = nullptr) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  long long t0 = clock64();
  auto mark = [&](int ph) {  // optional per-phase timing (thousands of SM cycles), thread 0
    if (phase_kcycles && tid == 0) {
      const long long t1 = clock64();
      phase_kcycles[ph] = (int32_t)((t1 - t0) / 1000);
      t0 = t1;
    }
  };
  __shared__ double s_scal[4];
  __shared__ int s_nvec;
  // ---- 1. tridiagonalisation: H_k = I - tau v v^T on rows k+1.., v_0 = 1 ----
  constexpr int TPR = 4;  // threads per row of the matrix-vector product
  for (int k = 0; k + 2 < n; ++k) {
    const int m = n - k - 1;
    if (warp == 0) {
      double s = 0.0;
      for (int i = k + 2 + lane; i < n; i += 32) {
        const double x = A[i * ldn + k];
        s += x * x;
      }
      s = eig_warp_sum(s);
      if (lane == 0) {
        const double alpha = A[(k + 1) * ldn + k];
        double tau = 0.0, beta = alpha, scale = 0.0;
        if (s > 0.0) {
          const double nrm = sqrt(alpha * alpha + s);
          beta = alpha >= 0.0 ? -nrm : nrm;
          tau = (beta - alpha) / beta;
          scale = 1.0 / (alpha - beta);
        }
        W.tau[k] = tau;
        W.e[k] = beta;
        W.d[k] = A[k * ldn + k];
        s_scal[0] = scale;
        s_scal[1] = tau;
      }
    }
    __syncthreads();
    const double scale = s_scal[0], tau = s_scal[1];
    if (tau != 0.0) {
      // p = tau A22 v (v computed on the fly), per-warp partials of v^T p
      double part = 0.0;
      for (int base = 0; base < m * TPR; base += nt) {
        const int idx = base + tid, row = idx / TPR, sub = idx % TPR;
        double s = 0.0;
        if (row < m) {
          const double* ar = A + (k + 1 + row) * ldn + (k + 1);
          for (int j = sub; j < m; j += TPR) {
            const double vj = j == 0 ? 1.0 : A[(k + 1 + j) * ldn + k] * scale;
            s += ar[j] * vj;
          }
        }
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        if (row < m && sub == 0) {
          const double vr = row == 0 ? 1.0 : A[(k + 1 + row) * ldn + k] * scale;
          W.pp[row] = tau * s;
          W.vv[row] = vr;
          part += vr * (tau * s);
        }
      }
      part = eig_warp_sum(part);
      if (lane == 0) W.red[warp] = part;
      __syncthreads();
      double vp = 0.0;
      for (int q = 0; q < nw; ++q) vp += W.red[q];
      const double K = 0.5 * tau * vp;
      // A22 -= v q^T + q v^T, q = p - K v; store v below the sub-diagonal of column k
      for (int idx = tid; idx < m * m; idx += nt) {
        const int i = idx / m, j = idx - i * m;
        const double vi = W.vv[i], vj = W.vv[j];
        const double qi = W.pp[i] - K * vi, qj = W.pp[j] - K * vj;
        A[(k + 1 + i) * ldn + (k + 1 + j)] -= vi * qj + qi * vj;
      }
      for (int i = tid; i + 1 < m; i += nt) A[(k + 2 + i) * ldn + k] = W.vv[i + 1];
    }
    __syncthreads();
  }
  if (tid == 0) {
    if (n >= 2) {
      W.d[n - 2] = A[(n - 2) * ldn + (n - 2)];
      W.e[n - 2] = A[(n - 1) * ldn + (n - 2)];
      W.tau[n - 2] = 0.0;
    }
    W.d[n - 1] = A[(n - 1) * ldn + (n - 1)];
    W.e[n - 1] = 0.0;
  }
  __syncthreads();
  mark(0);
  // ---- 2. eigenvalues: multisection of Sturm counts ----
  double* e2 = W.pp;  // reuse
  double tn = 0.0, glo = 0.0, ghi = 0.0, emax2 = 0.0;
  for (int i = 0; i < n; ++i) {  // every thread (n <= 130): identical values, no barrier
    const double el = i > 0 ? fabs(W.e[i - 1]) : 0.0, er = i + 1 < n ? fabs(W.e[i]) : 0.0;
    const double lo = W.d[i] - el - er, hi = W.d[i] + el + er;
    glo = i == 0 ? lo : fmin(glo, lo);
    ghi = i == 0 ? hi : fmax(ghi, hi);
    tn = fmax(tn, fabs(W.d[i]) + el + er);
    emax2 = fmax(emax2, er * er);
  }
  for (int i = tid; i < n; i += nt) e2[i] = i + 1 < n ? W.e[i] * W.e[i] : 0.0;
  __syncthreads();
  const double pivmin = DBL_MIN * fmax(1.0, emax2);
  const double tol = 4.0 * DBL_EPSILON * tn;
  glo -= 2.0 * tol + pivmin;
  ghi += 2.0 * tol + pivmin;
  // only the nl = min(n, nvec_cap) largest eigenvalues are needed (the cut and the basis use
  // lambda_0 .. lambda_{r-1}); lam[j >= nl] are left 0
  const int nl = nvec_cap < n ? nvec_cap : n;
  for (int j = nl + tid; j < n; j += nt) W.lam[j] = 0.0;
  int G = 1;
  while (G < 32 && 2 * G * nl <= nt) G *= 2;
  const int P = G > 1 ? G - 1 : 1;  // evaluation points per group
  const int ngrp = nt / G, grp = tid / G, gl = tid % G, gbase = (lane / G) * G;
  for (int k0 = n - nl; k0 < n; k0 += ngrp) {
    const int k = k0 + grp;  // ascending index
    double lo = glo, hi = ghi;
    for (int round = 0; round < 256; ++round) {
      const bool act = k < n && tn > 0.0 && hi - lo > tol;
      if (!__any_sync(0xffffffffu, act)) break;
      int c = n + 1;
      if (act && gl < P) c = sturm_count(W.d, e2, n, lo + (hi - lo) * (double)(gl + 1) / (double)(P + 1), pivmin);
      const unsigned b = __ballot_sync(0xffffffffu, act && gl < P && c > k);
      if (act) {
        const unsigned mb = (b >> gbase) & ((G >= 32) ? 0xffffffffu : ((1u << G) - 1u));
        const int f = mb ? __ffs(mb) : P + 1;  // first point (1-based) with count > k
        const double span = hi - lo;
        const double nhi = f == P + 1 ? hi : lo + span * (double)f / (double)(P + 1);
        const double nlo = f == 1 ? lo : lo + span * (double)(f - 1) / (double)(P + 1);
        lo = nlo;
        hi = nhi;
      }
    }
    if (k < n && gl == 0) W.lam[n - 1 - k] = tn > 0.0 ? 0.5 * (lo + hi) : 0.0;
  }
  __syncthreads();
  if (tid == 0) {
    int nv = 0;
    const double l0 = W.lam[0];
    if (l0 > 0.0)
      while (nv < nvec_cap && nv < n && W.lam[nv] >= cut * l0) ++nv;
    s_nvec = nv;
  }
  __syncthreads();
  const int nvec = s_nvec;
  mark(1);
  if (nvec == 0) return 0;
  // ---- 3. inverse iteration, one thread per vector ----
  const int ldz = W.ldz;
  const double pert = 4.0 * DBL_EPSILON * tn + pivmin;
  for (int j = tid; j < nvec; j += nt) {
    const double sh = W.lam[j];
    double* u0 = W.fac;
    double* u1 = W.fac + (size_t)n * ldz;
    double* u2 = W.fac + (size_t)2 * n * ldz;
    double* ml = W.fac + (size_t)3 * n * ldz;
    // LU with partial pivoting of T - sh I (rows: p q r | e a e')
    double p = W.d[0] - sh, q = n > 1 ? W.e[0] : 0.0, r = 0.0;
    for (int i = 0; i + 1 < n; ++i) {
      const double ei = W.e[i], an = W.d[i + 1] - sh, en = i + 2 < n ? W.e[i + 1] : 0.0;
      if (fabs(p) >= fabs(ei)) {
        const double mu = p != 0.0 ? ei / p : 0.0;
        u0[i * ldz + j] = p == 0.0 ? pert : p;
        u1[i * ldz + j] = q;
        u2[i * ldz + j] = r;
        ml[i * ldz + j] = mu;
        W.swp[i * ldz + j] = 0;
        p = an - mu * q;
        q = en - mu * r;
        r = 0.0;
      } else {
        const double mu = p / ei;
        u0[i * ldz + j] = ei;
        u1[i * ldz + j] = an;
        u2[i * ldz + j] = en;
        ml[i * ldz + j] = mu;
        W.swp[i * ldz + j] = 1;
        const double np_ = q - mu * an, nq = r - mu * en;
        p = np_;
        q = nq;
        r = 0.0;
      }
    }
    u0[(n - 1) * ldz + j] = fabs(p) < pert ? (p < 0.0 ? -pert : pert) : p;
    // the last row has no super-diagonals: the back substitution multiplies these two entries by
    // z1 = z2 = 0, so they must be finite -- left unwritten they are whatever the previous block
    // on this SM left in shared memory, and a NaN / Inf pattern there sent the vector through
    // the degenerate-restart path (a rounding-level, run-to-run difference of the basis)
    u1[(n - 1) * ldz + j] = 0.0;
    u2[(n - 1) * ldz + j] = 0.0;
    for (int i = 0; i + 1 < n; ++i)
      if (fabs(u0[i * ldz + j]) < pert) u0[i * ldz + j] = u0[i * ldz + j] < 0.0 ? -pert : pert;
    // start vector
    double nrm = 0.0;
    for (int i = 0; i < n; ++i) {
      const double b = eig_start(i, j);
      W.Z[i * ldz + j] = b;
      nrm += b * b;
    }
    for (int it = 0; it < 3; ++it) {
      const double inv = 1.0 / sqrt(nrm);
      // forward: row operations
      double bi = W.Z[0 * ldz + j] * inv;
      for (int i = 0; i + 1 < n; ++i) {
        double bn = W.Z[(i + 1) * ldz + j] * inv;
        if (W.swp[i * ldz + j]) {
          const double t = bi;
          bi = bn;
          bn = t;
        }
        W.Z[i * ldz + j] = bi;
        bi = bn - ml[i * ldz + j] * bi;
      }
      W.Z[(n - 1) * ldz + j] = bi;
      // backward
      double z1 = 0.0, z2 = 0.0;
      nrm = 0.0;
      for (int i = n - 1; i >= 0; --i) {
        const double z = (W.Z[i * ldz + j] - u1[i * ldz + j] * z1 - u2[i * ldz + j] * z2) / u0[i * ldz + j];
        W.Z[i * ldz + j] = z;
        nrm += z * z;
        z2 = z1;
        z1 = z;
      }
      if (!(nrm > 0.0) || !isfinite(nrm)) {  // degenerate: restart from the start vector
        nrm = 0.0;
        for (int i = 0; i < n; ++i) {
          const double b = eig_start(i, j + 1000 * (it + 1));
          W.Z[i * ldz + j] = b;
          nrm += b * b;
        }
      }
    }
    const double inv = 1.0 / sqrt(nrm);
    for (int i = 0; i < n; ++i) W.Z[i * ldz + j] *= inv;
  }
  __syncthreads();
  mark(2);
  // ---- 3b. CGS2 in descending-eigenvalue order ----
  double* coef = W.vv;
  for (int j = 1; j < nvec; ++j) {
    for (int pass = 0; pass < 2; ++pass) {
      for (int i = warp; i < j; i += nw) {
        double s = 0.0;
        for (int rr = lane; rr < n; rr += 32) s += W.Z[rr * ldz + i] * W.Z[rr * ldz + j];
        s = eig_warp_sum(s);
        if (lane == 0) coef[i] = s;
      }
      __syncthreads();
      // z_j -= sum_i coef_i z_i: NP consecutive threads per row split the i range (fixed order:
      // strided partial sums, then a shuffle tree over the NP threads)
      const int NP = nt >= 8 * n ? 8 : (nt >= 4 * n ? 4 : (nt >= 2 * n ? 2 : 1));
      for (int base = 0; base < n * NP; base += nt) {
        const int t = base + tid, rr = t / NP, part = t % NP;
        double s = 0.0;
        if (rr < n)
          for (int i = part; i < j; i += NP) s += coef[i] * W.Z[rr * ldz + i];
        for (int o = 1; o < NP; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (rr < n && part == 0) W.Z[rr * ldz + j] -= s;
      }
      __syncthreads();
    }
    if (warp == 0) {
      double s = 0.0;
      for (int rr = lane; rr < n; rr += 32) s += W.Z[rr * ldz + j] * W.Z[rr * ldz + j];
      s = eig_warp_sum(s);
      if (lane == 0) s_scal[2] = 1.0 / sqrt(s);
    }
    __syncthreads();
    const double inv = s_scal[2];
    for (int rr = tid; rr < n; rr += nt) W.Z[rr * ldz + j] *= inv;
    __syncthreads();
  }
  mark(3);
  // ---- 4. back-transformation Z <- H_0 ... H_{n-3} Z: each warp owns a contiguous run of up to
  // BT eigenvectors and applies every reflector to all of them at once (BT independent dot
  // products and warp reductions in flight); the reflectors are read-only now: no block
  // barriers ----
  {
    constexpr int BT = 8;
    const int per = (nvec + nw - 1) / nw;
    const int jend = min(nvec, (warp + 1) * per);
    for (int j0 = warp * per; j0 < jend; j0 += BT) {
      const int nb = min(BT, jend - j0);
      for (int k = n - 3; k >= 0; --k) {
        const double tau = W.tau[k];
        if (tau == 0.0) continue;  // uniform within the warp
        const int m = n - k - 1;
        double sb[BT];
#pragma unroll
        for (int b = 0; b < BT; ++b) sb[b] = 0.0;
        for (int i = lane; i < m; i += 32) {
          const double v = i == 0 ? 1.0 : A[(k + 1 + i) * ldn + k];
          const double* zr = W.Z + (k + 1 + i) * ldz + j0;
#pragma unroll
          for (int b = 0; b < BT; ++b)
            if (b < nb) sb[b] += v * zr[b];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int b = 0; b < BT; ++b) sb[b] += __shfl_xor_sync(0xffffffffu, sb[b], o);
        for (int i = lane; i < m; i += 32) {
          const double v = i == 0 ? 1.0 : A[(k + 1 + i) * ldn + k];
          double* zr = W.Z + (k + 1 + i) * ldz + j0;
#pragma unroll
          for (int b = 0; b < BT; ++b)
            if (b < nb) zr[b] -= v * (sb[b] * tau);
        }
        __syncwarp();
      }
    }
  }
  __syncthreads();
  // ---- sign ----
  for (int j = tid; j < nvec; j += nt) {
    int im = 0;
    double vm = -1.0;
    for (int i = 0; i < n; ++i) {
      const double a = fabs(W.Z[i * ldz + j]);
      if (a > vm) {
        vm = a;
        im = i;
      }
    }
    if (W.Z[im * ldz + j] < 0.0)
      for (int i = 0; i < n; ++i) W.Z[i * ldz + j] = -W.Z[i * ldz + j];
  }
  __syncthreads();
  mark(4);
  return nvec;
}

}  // namespace hrom
