// linalg.cu -- H4/H5 (gappy normal equations + one-CTA solve), H10-H12 (Gram, thin
// eigen, lift).  FP64 tensor cores: mma.sync.m8n8k4.f64 (SASS DMMA; sm_100a has no
// tcgen05 f64 kind).
//
// Paper: gappy coordinates y = (P^T Phi)^+ P^T (v - psi) (Eq. 8); POD_m of the
// lagged-centred window via a thin SVD (Eq. 9; remark P:634);
// reading A13 (pinv cut 1e-12 on lambda), A14 (lagged centring; shifted Gram with
// periodic re-base), A15 (Gram + Jacobi eigen, keep lambda_i >= 1e-8 lambda_1, sign on V).
#include <algorithm>
#include "internal.cuh"

namespace hrom {
namespace {

constexpr int RT = 64;        // rows per Gram tile
constexpr int LDT = RT + 4;   // padded column stride in smem (conflict-free fragments)
constexpr int GT = 256;       // threads per Gram CTA

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

struct GramArgs {
  int mode;                  // 0 contiguous columns (shift rho), 1 gathered rows of S-hat
  int ncol;                  // real columns
  int nsb;                   // super blocks (16 columns each)
  int64_t rows;              // contiguous rows (mode 0)
  const double* const* cols; // mode 0: column pointers
  int64_t ns;                // mode 0: slab stride of the columns (1 = plain)
  SRef rho;                  // mode 0: shift (rho.p nullable)
  // mode 1
  Geo g;
  Win W;
  const double* ring;
  const int32_t* list;       // S-hat cells
  const int32_t* count;      // |S-hat|
  SRef src_b;                // HDM values on S-hat rows
  double* part;              // [grid][nsb*16][nsb*16]
};

// One tile of the Gram: C += T^T T over RT rows, T in smem column-major (ld LDT).
template <int TPW>
__device__ __forceinline__ void gram_tile(const double* tile, int nsb, double (&acc)[TPW][8]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int ntask = nsb * (nsb + 1) / 2;
#pragma unroll
  for (int kk = 0; kk < RT; kk += 4) {
#pragma unroll
    for (int t = 0; t < TPW; ++t) {
      const int task = warp + t * (GT / 32);
      if (task < ntask) {
        // task -> (sa, sb), sa <= sb, row-major over the upper triangle
        int sa = 0, rem = task;
        while (rem >= nsb - sa) { rem -= nsb - sa; ++sa; }
        const int sb = sa + rem;
        const double a0 = tile[(16 * sa + gid) * LDT + kk + tig];
        const double a1 = tile[(16 * sa + 8 + gid) * LDT + kk + tig];
        const double b0 = tile[(16 * sb + gid) * LDT + kk + tig];
        const double b1 = tile[(16 * sb + 8 + gid) * LDT + kk + tig];
        dmma(acc[t][0], acc[t][1], a0, b0);
        dmma(acc[t][2], acc[t][3], a0, b1);
        dmma(acc[t][4], acc[t][5], a1, b0);
        dmma(acc[t][6], acc[t][7], a1, b1);
      }
    }
  }
}

template <int TPW>
__global__ void __launch_bounds__(GT, (TPW <= 2) ? 2 : 1) gram_kernel(GramArgs a) {
  extern __shared__ double smem[];
  double* tile = smem;                      // [nsb*16][LDT]
  const int ncp = a.nsb * 16;
  double acc[TPW][8];
#pragma unroll
  for (int t = 0; t < TPW; ++t)
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[t][q] = 0.0;
  int64_t total_rows;
  if (a.mode == 0) total_rows = a.rows;
  else total_rows = (int64_t)(*a.count) * a.g.c;
  const int64_t ntiles = (total_rows + RT - 1) / RT;
  for (int64_t tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
    const int64_t r0 = tl * RT;
    if (a.mode == 0) {
      for (int idx = threadIdx.x; idx < ncp * RT; idx += GT) {
        const int col = idx / RT, k = idx % RT;
        const int64_t row = r0 + k;
        double v = 0.0;
        if (col < a.ncol && row < total_rows) {
          v = a.cols[col][sidx(SRef{nullptr, a.ns}, row)];
          if (a.rho.p) v -= a.rho.p[sidx(a.rho, row)];
        }
        tile[col * LDT + k] = v;
      }
    } else {
      // gathered rows: row t -> (var = t / nS, idx = t % nS), element e = var*N + cell.
      // X slot s (s >= nU-w) lands in column s-(nU-w); the psi_prev-only slot (nU = w+1) in
      // column w+1; the HDM value b in column w.  Then centre in place.
      const int nS = *a.count;
      const int nU = a.W.nU, w = a.W.w;
      const int xoff = nU - w;
      double* psi = smem + (size_t)ncp * LDT;  // [2][RT]
      __shared__ int64_t erow[RT];             // DOF of each tile row (-1 past the end)
      if (threadIdx.x < RT) {
        const int64_t row = r0 + threadIdx.x;
        int64_t e = -1;
        if (row < total_rows) {
          const int var = (int)(row / nS), ii = (int)(row % nS);
          e = (int64_t)var * a.g.N + a.list[ii];
        }
        erow[threadIdx.x] = e;
      }
      __syncthreads();
      // all loads of this thread in flight before the first shared store (memory-level parallelism)
      constexpr int QB = 17;  // loads in flight per thread per batch
      const int total = (nU + 1) * RT;
      for (int base = threadIdx.x; base < total; base += QB * GT) {
        double vbuf[QB];
#pragma unroll
        for (int q = 0; q < QB; ++q) {
          const int idx = base + q * GT;
          double v = 0.0;
          if (idx < total) {
            const int s = idx / RT, k = idx % RT;
            const int64_t e = erow[k];
            if (e >= 0)
              v = (s < nU) ? __ldg(a.ring + (int64_t)a.W.slot[s] * TILE + sidx(SRef{nullptr, a.g.nsr}, e))
                           : __ldg(a.src_b.p + sidx(a.src_b, e));
          }
          vbuf[q] = v;
        }
#pragma unroll
        for (int q = 0; q < QB; ++q) {
          const int idx = base + q * GT;
          if (idx < total) {
            const int s = idx / RT, k = idx % RT;
            const int col = (s == nU) ? w : (s >= xoff ? s - xoff : w + 1);
            tile[col * LDT + k] = vbuf[q];
          }
        }
      }
      __syncthreads();
      if (threadIdx.x < RT) {
        const int k = threadIdx.x;
        double sp = 0.0, sc = 0.0;
        for (int i = 0; i < w; ++i) sc += tile[i * LDT + k];
        if (xoff == 1) {
          sp = tile[(w + 1) * LDT + k];
          for (int i = 0; i < w - 1; ++i) sp += tile[i * LDT + k];
        } else {
          sp = sc;
        }
        psi[k] = sp / (double)w;
        psi[RT + k] = sc / (double)w;
      }
      __syncthreads();
      for (int idx = threadIdx.x; idx < ncp * RT; idx += GT) {
        const int col = idx / RT, k = idx % RT;
        const bool valid = r0 + k < total_rows;
        double v;
        if (col < w) v = valid ? tile[col * LDT + k] - psi[k] : 0.0;
        else if (col == w) v = valid ? tile[col * LDT + k] - psi[RT + k] : 0.0;
        else v = 0.0;
        tile[col * LDT + k] = v;
      }
    }
    __syncthreads();
    gram_tile<TPW>(tile, a.nsb, acc);
    __syncthreads();
  }
  // write this CTA's partial (upper super-block pairs)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int ntask = a.nsb * (a.nsb + 1) / 2;
  double* out = a.part + (int64_t)blockIdx.x * ncp * ncp;
#pragma unroll
  for (int t = 0; t < TPW; ++t) {
    const int task = warp + t * (GT / 32);
    if (task < ntask) {
      int sa = 0, rem = task;
      while (rem >= a.nsb - sa) { rem -= a.nsb - sa; ++sa; }
      const int sb = sa + rem;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int bi = 16 * sa + 8 * (q >> 1), bj = 16 * sb + 8 * (q & 1);
        out[(bi + gid) * ncp + bj + 2 * tig] = acc[t][2 * q];
        out[(bi + gid) * ncp + bj + 2 * tig + 1] = acc[t][2 * q + 1];
      }
    }
  }
}

// deterministic fixed-order reduction over CTAs; C[i][j] for i <= j mirrored
__global__ void gram_reduce(const double* __restrict__ part, int nblk, int ncp, int ncol, double* __restrict__ C,
                            int ldc, const int32_t* __restrict__ map) {
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < ncol * ncol; idx += gridDim.x * blockDim.x) {
    const int i = idx / ncol, j = idx % ncol;
    if (i > j) continue;
    double s = 0.0;
    for (int b = 0; b < nblk; ++b) s += part[(int64_t)b * ncp * ncp + i * ncp + j];
    const int ci = map ? map[i] : i, cj = map ? map[j] : j;
    C[ci * ldc + cj] = s;
    C[cj * ldc + ci] = s;
  }
}

// ---------------- one-CTA cyclic Jacobi eigen-solver (n <= 130) ----------------
// A (n x n, ld = ldn, symmetric) is overwritten; V receives eigenvectors (columns);
// lam/perm: eigenvalues in descending order and the column permutation.
__device__ void jacobi_eig(double* A, double* V, int n, int ldn, double* lam, int* perm, double* cs,
                           int* pq, int* flag, int32_t* sweeps_out) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int ne = n + (n & 1);  // even size (padded index has zero row/col)
  for (int idx = tid; idx < ne * ne; idx += nt) {
    const int i = idx / ne, j = idx % ne;
    V[i * ldn + j] = (i == j) ? 1.0 : 0.0;
    if (i >= n || j >= n) A[i * ldn + j] = 0.0;
  }
  __syncthreads();
  __shared__ double floor_abs;
  if (tid == 0) {
    double m = 0.0;
    for (int i = 0; i < n; ++i) m = fmax(m, fabs(A[i * ldn + i]));
    floor_abs = 1e-14 * m;  // below the Gram's own rounding level (~n eps lambda_max): not resolvable
  }
  __syncthreads();
  const int np = ne / 2;
  // round-robin tournament schedule, precomputed: round r pairs positions k and ne-1-k,
  // player(pos) = pos == 0 ? 0 : ((pos - 1 + r) mod (ne - 1)) + 1
  __shared__ short2 ptab[(kMaxSlots - 1) * (kMaxSlots / 2)];
  for (int idx = tid; idx < (ne - 1) * np; idx += nt) {
    const int r = idx / np, k = idx % np;
    auto player = [&](int pos) { return pos == 0 ? 0 : ((pos - 1 + r) % (ne - 1)) + 1; };
    int p = player(k), q = player(ne - 1 - k);
    if (p > q) { const int t = p; p = q; q = t; }
    ptab[idx] = make_short2((short)p, (short)q);
  }
  __syncthreads();
  for (int sweep = 0; sweep < 20; ++sweep) {
    if (tid == 0) *flag = 0;
    __syncthreads();
    for (int rnd = 0; rnd < ne - 1; ++rnd) {
      if (tid < np) {
        const int k = tid;
        const short2 pr = ptab[rnd * np + k];
        const int p = pr.x, q = pr.y;
        const double app = A[p * ldn + p], aqq = A[q * ldn + q], apq = A[p * ldn + q];
        double c = 1.0, s = 0.0;
        if (fabs(apq) > floor_abs && fabs(apq) > 1e-14 * sqrt(fabs(app * aqq))) {
          // t = tan(phi) of the annihilating rotation, written without 1/apq
          const double tau = aqq - app;
          const double t = (tau >= 0.0 ? 2.0 : -2.0) * apq / (fabs(tau) + sqrt(tau * tau + 4.0 * apq * apq));
          c = rsqrt(1.0 + t * t);
          s = t * c;
          *flag = 1;
        }
        cs[2 * k] = c;
        cs[2 * k + 1] = s;
        pq[2 * k] = p;
        pq[2 * k + 1] = q;
      }
      __syncthreads();
      // A' = J^T A J in one pass: every 2x2 block (pair k1 rows, pair k2 cols) is independent
      for (int idx = tid, k1 = tid / np, k2 = tid % np; idx < np * np;
           idx += nt, k2 += nt % np, k1 += nt / np + (k2 >= np ? 1 : 0), k2 -= (k2 >= np ? np : 0)) {
        const double c1 = cs[2 * k1], s1 = cs[2 * k1 + 1], c2 = cs[2 * k2], s2 = cs[2 * k2 + 1];
        if (s1 == 0.0 && s2 == 0.0) continue;
        const int p1 = pq[2 * k1], q1 = pq[2 * k1 + 1], p2 = pq[2 * k2], q2 = pq[2 * k2 + 1];
        const double b00 = A[p1 * ldn + p2], b01 = A[p1 * ldn + q2];
        const double b10 = A[q1 * ldn + p2], b11 = A[q1 * ldn + q2];
        const double r00 = c1 * b00 - s1 * b10, r01 = c1 * b01 - s1 * b11;
        const double r10 = s1 * b00 + c1 * b10, r11 = s1 * b01 + c1 * b11;
        double n00 = c2 * r00 - s2 * r01, n01 = s2 * r00 + c2 * r01;
        double n10 = c2 * r10 - s2 * r11, n11 = s2 * r10 + c2 * r11;
        if (k1 == k2) { n01 = 0.0; n10 = 0.0; }
        A[p1 * ldn + p2] = n00;
        A[p1 * ldn + q2] = n01;
        A[q1 * ldn + p2] = n10;
        A[q1 * ldn + q2] = n11;
      }
      // V' = V J
      for (int idx = tid, i = tid / np, k = tid % np; idx < ne * np;
           idx += nt, k += nt % np, i += nt / np + (k >= np ? 1 : 0), k -= (k >= np ? np : 0)) {
        const double c = cs[2 * k], s = cs[2 * k + 1];
        if (s == 0.0) continue;
        const int p = pq[2 * k], q = pq[2 * k + 1];
        const double vp = V[i * ldn + p], vq = V[i * ldn + q];
        V[i * ldn + p] = c * vp - s * vq;
        V[i * ldn + q] = s * vp + c * vq;
      }
      __syncthreads();
    }
    if (tid == 0 && sweeps_out) *sweeps_out = sweep + 1;
    if (*flag == 0) break;
    __syncthreads();
  }
  // descending order, ties by index
  for (int i = tid; i < n; i += nt) {
    const double li = A[i * ldn + i];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
      const double lj = A[j * ldn + j];
      if (lj > li || (lj == li && j < i)) ++rank;
    }
    perm[rank] = i;
  }
  __syncthreads();
  for (int r = tid; r < n; r += nt) lam[r] = A[perm[r] * ldn + perm[r]];
  // sign: largest |V_i,col| (ties lowest i) positive
  for (int col = tid; col < n; col += nt) {
    int im = 0;
    double vm = -1.0;
    for (int i = 0; i < n; ++i) {
      const double a = fabs(V[i * ldn + col]);
      if (a > vm) { vm = a; im = i; }
    }
    if (V[im * ldn + col] < 0.0)
      for (int i = 0; i < n; ++i) V[i * ldn + col] = -V[i * ldn + col];
  }
  __syncthreads();
}

// basis from the shifted Gram (one CTA): M = X^T X by lagged centring, eigen, A = V_r L_r^-1/2
__global__ void __launch_bounds__(1024) basis_kernel(const double* __restrict__ C, int ldc, Win W, int r, double cut,
                                                     double* __restrict__ Aout, double* __restrict__ lam_out,
                                                     int32_t* __restrict__ reff_out, double* __restrict__ Vg) {
  extern __shared__ double sm[];
  const int w = W.w, nU = W.nU;
  const int ldn = w + (w & 1) + 1;  // odd stride: column sweeps are bank-conflict free
  double* M = sm;                                   // ldn*ldn
  const bool vsm = (2 * ldn * ldn + 4 * kMaxSlots) * 8 <= 200 * 1024;
  double* V = vsm ? sm + ldn * ldn : Vg;
  double* lam = sm + (vsm ? 2 : 1) * ldn * ldn;     // kMaxSlots
  double* mrow = lam + kMaxSlots;                   // kMaxSlots
  double* cs = mrow + kMaxSlots;                    // 2*kMaxSlots
  __shared__ int perm[kMaxSlots];
  __shared__ int pq[2 * kMaxSlots];
  __shared__ int flag;
  __shared__ double mu;
  const int tid = threadIdx.x;
  // m_i = (1/w) sum_{p<w} C[x_i][u_p];  mu = (1/w^2) sum_{p,q<w} C[u_p][u_q]
  for (int i = tid; i < w; i += blockDim.x) {
    const int xi = W.slot[nU - w + i];
    double s = 0.0;
    for (int p = 0; p < w; ++p) s += C[xi * ldc + W.slot[p]];
    mrow[i] = s / (double)w;
  }
  if (tid == 0) {
    double s = 0.0;
    for (int p = 0; p < w; ++p)
      for (int q = 0; q < w; ++q) s += C[W.slot[p] * ldc + W.slot[q]];
    mu = s / ((double)w * (double)w);
  }
  __syncthreads();
  for (int idx = tid; idx < w * w; idx += blockDim.x) {
    const int i = idx / w, j = idx % w;
    const int xi = W.slot[nU - w + i], xj = W.slot[nU - w + j];
    // when psi_prev == psi_cur (bootstrap, nU == w) this is the plain centred Gram
    double mi = mrow[i], mj = mrow[j];
    M[i * ldn + j] = ((C[xi * ldc + xj] - mi) - mj) + mu;
  }
  __syncthreads();
  jacobi_eig(M, V, w, ldn, lam, perm, cs, pq, &flag, reff_out + 8);
  if (tid == 0) {
    int re = 0;
    const double l0 = lam[0];
    for (int i = 0; i < r && i < w; ++i)
      if (l0 > 0.0 && lam[i] >= cut * l0) ++re;
      else break;
    *reff_out = re;
  }
  __syncthreads();
  const int re = *reff_out;
  for (int idx = tid; idx < w * r; idx += blockDim.x) {
    const int i = idx % w, j = idx / w;  // A column-major: A[j*w + i]
    Aout[j * w + i] = (j < re) ? V[i * ldn + perm[j]] / sqrt(lam[j]) : 0.0;
  }
  for (int i = tid; i < w; i += blockDim.x) lam_out[i] = lam[i];
}

// H5: G = A^T K_XX A, rhs = A^T K_Xb, y = G^+ rhs (cut on lambda), c = A y
__global__ void __launch_bounds__(1024) solve_kernel(const double* __restrict__ K, int w, int r,
                                                     const double* __restrict__ A, const int32_t* __restrict__ reffp,
                                                     double cut, double* __restrict__ y_out,
                                                     double* __restrict__ c_out, int32_t* __restrict__ status) {
  extern __shared__ double sm[];
  const int re = *reffp;
  const int ldk = w + 1;
  const int ldn = re + (re & 1) + 1;  // odd stride
  double* T = sm;                 // w x re  (K_XX A)
  double* G = T + w * kMaxR;      // ldn x ldn
  double* V = G + (kMaxR + 2) * (kMaxR + 2);  // ldn x ldn
  double* rhs = V + (kMaxR + 2) * (kMaxR + 2);
  double* lam = rhs + kMaxR;
  double* cs = lam + kMaxR;       // 2*kMaxR
  double* y = cs + 2 * kMaxR;
  __shared__ int perm[kMaxR];
  __shared__ int pq[2 * kMaxR];
  __shared__ int flag;
  const int tid = threadIdx.x;
  for (int idx = tid; idx < w * re; idx += blockDim.x) {
    const int i = idx % w, j = idx / w;
    double s = 0.0;
    for (int p = 0; p < w; ++p) s += K[i * ldk + p] * A[j * w + p];
    T[j * w + i] = s;
  }
  for (int j = tid; j < re; j += blockDim.x) {
    double s = 0.0;
    for (int p = 0; p < w; ++p) s += A[j * w + p] * K[p * ldk + w];
    rhs[j] = s;
  }
  __syncthreads();
  for (int idx = tid; idx < re * re; idx += blockDim.x) {
    const int i = idx / re, j = idx % re;
    if (j < i) continue;
    double s = 0.0;
    for (int p = 0; p < w; ++p) s += A[i * w + p] * T[j * w + p];
    G[i * ldn + j] = s;
    G[j * ldn + i] = s;
  }
  __syncthreads();
  if (re > 0) jacobi_eig(G, V, re, ldn, lam, perm, cs, pq, &flag, status + 7);
  if (tid < kMaxR) y[tid] = 0.0;
  __syncthreads();
  if (tid == 0) {
    int st = 0;
    if (re == 0 || !(lam[0] > 0.0)) st = 1;
    *status = st;
  }
  // y = sum_{kept} v_k (v_k^T rhs) / lam_k
  for (int i = tid; i < re; i += blockDim.x) {
    double s = 0.0;
    if (lam[0] > 0.0)
      for (int kk = 0; kk < re; ++kk) {
        if (!(lam[kk] >= cut * lam[0])) break;
        const int col = perm[kk];
        double d = 0.0;
        for (int p = 0; p < re; ++p) d += V[p * ldn + col] * rhs[p];
        s += V[i * ldn + col] * (d / lam[kk]);
      }
    y[i] = s;
  }
  __syncthreads();
  for (int i = tid; i < kMaxR; i += blockDim.x) y_out[i] = (i < re) ? y[i] : 0.0;
  for (int i = tid; i < w; i += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < re; ++j) s += A[j * w + i] * y[j];
    c_out[i] = s;
  }
}

// Phi_{k+1}[:, j] = X A[:, j] (materialised; tests/config 5), psi_cur
__global__ void lift_kernel(Geo g, Win W, const double* __restrict__ ring, const double* __restrict__ A,
                            const int32_t* __restrict__ reffp, double* __restrict__ phi, double* __restrict__ psi) {
  const int re = *reffp;
  const int w = W.w, nU = W.nU;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < g.D; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t se = sidx(SRef{nullptr, g.nsr}, e);
    double sp = 0.0, sc = 0.0;
    for (int s = 0; s < w; ++s) sp += ring[(int64_t)W.slot[s] * TILE + se];
    for (int s = nU - w; s < nU; ++s) sc += ring[(int64_t)W.slot[s] * TILE + se];
    const double pp = sp / (double)w;
    if (psi) psi[e] = sc / (double)w;
    if (phi)
      for (int j = 0; j < re; ++j) {
        double acc = 0.0;
        for (int i = 0; i < w; ++i) acc += (ring[(int64_t)W.slot[nU - w + i] * TILE + se] - pp) * A[j * w + i];
        phi[(int64_t)j * g.D + e] = acc;
      }
  }
}

template <int TPW>
hrom_status launch_gram(hrom_ctx* c, const GramArgs& a, int grid) {
  const size_t smem = ((size_t)a.nsb * 16 * LDT + 2 * RT) * sizeof(double);
  HROM_CK(cudaFuncSetAttribute(gram_kernel<TPW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  gram_kernel<TPW><<<grid, GT, smem, c->st>>>(a);
  HROM_LAUNCH_CK();
  ++c->nlaunch;
  return HROM_OK;
}

hrom_status dispatch_gram(hrom_ctx* c, GramArgs a, int grid) {
  const int ntask = a.nsb * (a.nsb + 1) / 2;
  const int tpw = (ntask + GT / 32 - 1) / (GT / 32);
  if (tpw <= 1) return launch_gram<1>(c, a, grid);
  if (tpw <= 2) return launch_gram<2>(c, a, grid);
  if (tpw <= 4) return launch_gram<4>(c, a, grid);
  if (tpw <= 6) return launch_gram<6>(c, a, grid);
  if (tpw <= 9) return launch_gram<9>(c, a, grid);
  return HROM_E_INVALID;
}

}  // namespace

// Full Gram of ncol columns over `rows` rows, shifted by rho (nullable): dev_C[i*ldc+j].
hrom_status gram_full(hrom_ctx* c, const double* const* dev_cols, int64_t ns, int ncol, int64_t rows, SRef rho,
                      double* dev_C, int ldc, const int32_t* map) {
  GramArgs a{};
  a.mode = 0;
  a.ncol = ncol;
  a.nsb = (ncol + 15) / 16;
  a.rows = rows;
  a.cols = dev_cols;
  a.ns = ns;
  a.rho = rho;
  const int grid = c->nsm * 2;
  const int ncp = a.nsb * 16;
  if ((int64_t)grid * ncp * ncp > c->b.part_len) return HROM_E_INVALID;
  a.part = c->b.part;
  hrom_status s = dispatch_gram(c, a, grid);
  if (s != HROM_OK) return s;
  gram_reduce<<<64, 256, 0, c->st>>>(c->b.part, grid, ncp, ncol, dev_C, ldc, map);
  HROM_LAUNCH_CK();
  ++c->nlaunch;
  return HROM_OK;
}

// gathered Gram of [X_S, b] over the rows of S-hat -> b.K ((w+1) x (w+1))
hrom_status gram_gathered(hrom_ctx* c, SRef src_b) {
  GramArgs a{};
  a.mode = 1;
  a.ncol = c->win.w + 1;
  a.nsb = (c->win.w + 2 + 15) / 16;  // tile holds the raw w+1 slots + b before centring
  a.g = c->g;
  a.W = c->win;
  a.ring = c->b.ring;
  a.list = c->b.lists + (int64_t)L_S * c->g.N;
  a.count = c->b.counts + L_S;
  a.src_b = src_b;
  // while the one-CTA eigen-solve of the previous update holds an SM (side stream), size the
  // grid to the other SMs: a static tile split with one block left over would double the time
  const int grid = (c->basis_pending ? c->nsm - 1 : c->nsm) * 2;
  const int ncp = a.nsb * 16;
  if ((int64_t)grid * ncp * ncp > c->b.part_len) return HROM_E_INVALID;
  a.part = c->b.part;
  hrom_status s = dispatch_gram(c, a, grid);
  if (s != HROM_OK) return s;
  gram_reduce<<<64, 256, 0, c->st>>>(c->b.part, grid, ncp, a.ncol, c->b.K, a.ncol, nullptr);
  HROM_LAUNCH_CK();
  ++c->nlaunch;
  return HROM_OK;
}

hrom_status small_solve(hrom_ctx* c) {
  const size_t smem = (size_t)(c->win.w * kMaxR + 2 * (kMaxR + 2) * (kMaxR + 2) + 6 * kMaxR) * sizeof(double);
  HROM_CK(cudaFuncSetAttribute(solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  solve_kernel<<<1, 256, smem, c->st>>>(c->b.K, c->win.w, c->r, c->b.A, c->b.ireg, c->P.lsq_rel_cutoff, c->b.y,
                                        c->b.cvec, c->b.ireg + 2);
  HROM_LAUNCH_CK();
  ++c->nlaunch;
  return HROM_OK;
}

hrom_status basis_from_gram(hrom_ctx* c, const Win& W) {
  const int ldn = W.w + (W.w & 1) + 1;
  const bool vsm = (2 * ldn * ldn + 4 * kMaxSlots) * 8 <= 200 * 1024;
  const size_t smem = (size_t)((vsm ? 2 : 1) * ldn * ldn + 4 * kMaxSlots) * sizeof(double);
  HROM_CK(cudaFuncSetAttribute(basis_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  basis_kernel<<<1, 512, smem, c->st>>>(c->b.C, kMaxSlots, W, c->r, c->P.eig_rel_cutoff, c->b.A, c->b.lam,
                                         c->b.ireg, c->b.eigV);
  HROM_LAUNCH_CK();
  ++c->nlaunch;
  return HROM_OK;
}

hrom_status lift(hrom_ctx* c, const Win& W, double* phi, double* psi) {
  lift_kernel<<<c->nsm * 4, 256, 0, c->st>>>(c->g, W, c->b.ring, c->b.A, c->b.ireg, phi, psi);
  HROM_LAUNCH_CK();
  ++c->nlaunch;
  return HROM_OK;
}

}  // namespace hrom
