// odeim.cu -- NEXT-1: ODEIM_{n_p} sampling points of a POD basis (Eq. 10).
//
// Reading A36 (the cited ODEIM paper is not in the container): SPEC's greedy
// DEIM-and-continue.  Phi is D x m (col-major), DOF e belongs to cell e mod N.
// Point j = 0..n_p-1 uses mode l = j mod m: c = least squares of Phi[P, 0..l-1] c = Phi[P, l]
// over the DOF rows P chosen so far, residual rho = phi_l - Phi[:, 0..l-1] c with the rows of
// already chosen cells excluded, p_j = argmax_e |rho_e| (ties: lowest e).  The first m points
// interpolate (DEIM), the rest oversample.
//
// Per point: one CTA solves the small least-squares problem (Householder QR, |P| x l <= 256 x 63,
// in shared memory), then a grid pass over the D rows forms rho and its arg-max (HBM-bound:
// reads l + 1 columns); the last CTA to finish reduces the per-CTA maxima in fixed order and
// appends the point.  Everything stays on the stream; no host round trip between points.
#include <algorithm>
#include <climits>
#include "internal.cuh"

namespace hrom {
namespace {

constexpr int OD_T = 256;

// c = argmin || A c - b ||, A[q][i] = Phi[rows[q], i] (q < np, i < l), b[q] = Phi[rows[q], l].
// Householder QR with the same rank rule as the gappy solve (A13): a column whose R diagonal
// falls below sqrt(cut) |R_00| gets a zero coefficient.
__global__ void __launch_bounds__(OD_T) odeim_solve_kernel(const double* __restrict__ phi, int64_t D,
                                                           const int64_t* __restrict__ rows, int np, int l,
                                                           double cut, double* __restrict__ c) {
  extern __shared__ double sm[];
  double* A = sm;                   // [l + 1][np] column-major; column l = b
  __shared__ double red[OD_T / 32];
  __shared__ double s_alpha[kMaxR + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = OD_T / 32;
  for (int i = 0; i <= l; ++i)
    for (int q = tid; q < np; q += OD_T) A[i * np + q] = phi[(int64_t)i * D + rows[q]];
  __syncthreads();
  for (int k = 0; k < l; ++k) {
    // norm of A[k:, k]
    double s = 0.0;
    for (int q = k + tid; q < np; q += OD_T) s += A[k * np + q] * A[k * np + q];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    double nrm2 = 0.0;
    for (int w = 0; w < nw; ++w) nrm2 += red[w];
    const double akk = A[k * np + k];
    const double alpha = nrm2 > 0.0 ? (akk > 0.0 ? -sqrt(nrm2) : sqrt(nrm2)) : 0.0;
    const double v0 = akk - alpha;
    const double vn2 = nrm2 - akk * akk + v0 * v0;  // |v|^2 with v = A[k:,k] - alpha e_k
    __syncthreads();
    if (vn2 > 0.0) {
      // apply H = I - 2 v v^T / |v|^2 to columns k+1..l (one warp per column)
      for (int i = k + 1 + warp; i <= l; i += nw) {
        double d = 0.0;
        for (int q = k + lane; q < np; q += 32) d += (q == k ? v0 : A[k * np + q]) * A[i * np + q];
        for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
        const double f = 2.0 * d / vn2;
        for (int q = k + lane; q < np; q += 32) A[i * np + q] -= f * (q == k ? v0 : A[k * np + q]);
      }
    }
    if (tid == 0) s_alpha[k] = alpha;  // R_kk
    __syncthreads();
  }
  // back substitution R c = (Q^T b)[0..l) (R above the diagonal in A, diagonal in s_alpha)
  if (tid == 0) {
    const double r00 = l > 0 ? fabs(s_alpha[0]) : 0.0;
    for (int k = l - 1; k >= 0; --k) {
      const double rkk = s_alpha[k];
      double x = A[l * np + k];
      for (int i = k + 1; i < l; ++i) x -= A[i * np + k] * c[i];
      c[k] = (rkk != 0.0 && rkk * rkk >= cut * r00 * r00) ? x / rkk : 0.0;
    }
  }
}

struct ArgMax {
  double v;
  int64_t e;
};
__device__ __forceinline__ ArgMax amax(ArgMax a, ArgMax b) {
  if (b.v > a.v || (b.v == a.v && b.e < a.e)) return b;
  return a;
}
__device__ __forceinline__ ArgMax shfl_amax(ArgMax a) {
  for (int o = 16; o > 0; o >>= 1) {
    ArgMax b;
    b.v = __shfl_xor_sync(0xffffffffu, a.v, o);
    b.e = __shfl_xor_sync(0xffffffffu, a.e, o);
    a = amax(a, b);
  }
  return a;
}

// rho_e = phi_l[e] - sum_{i<l} Phi[e, i] c_i on the free rows; arg-max |rho| (ties: lowest e);
// the last CTA appends point j
__global__ void __launch_bounds__(OD_T) odeim_argmax_kernel(const double* __restrict__ phi, int64_t D, int64_t N,
                                                            int l, const double* __restrict__ cg,
                                                            uint8_t* __restrict__ chosen, double* __restrict__ pv,
                                                            int64_t* __restrict__ pe, unsigned int* __restrict__ cnt,
                                                            int64_t* __restrict__ rows, int j,
                                                            int32_t* __restrict__ cells_out,
                                                            int64_t* __restrict__ rows_out) {
  __shared__ double c[kMaxR + 1];
  __shared__ ArgMax wred[OD_T / 32];
  __shared__ bool last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < l; i += OD_T) c[i] = cg[i];
  __syncthreads();
  ArgMax best{-1.0, INT64_MAX};
  const int64_t stride = (int64_t)gridDim.x * OD_T;
  const double* pl = phi + (int64_t)l * D;
  const bool small = D < (int64_t)INT32_MAX;  // 32-bit cell index (D <= 67 M in every config)
  for (int64_t e = blockIdx.x * (int64_t)OD_T + tid; e < D; e += stride) {
    if (chosen[small ? (int)((unsigned)e % (unsigned)N) : e % N]) continue;
    double r = pl[e];
    const double* col = phi + e;
    int i = 0;
    for (; i + 8 <= l; i += 8) {  // eight column loads in flight before the (ordered) updates
      double p[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) p[u] = col[(int64_t)(i + u) * D];
#pragma unroll
      for (int u = 0; u < 8; ++u) r = __dsub_rn(r, __dmul_rn(p[u], c[i + u]));
    }
    for (; i < l; ++i) r = __dsub_rn(r, __dmul_rn(col[(int64_t)i * D], c[i]));
    best = amax(best, ArgMax{fabs(r), e});
  }
  best = shfl_amax(best);
  if (lane == 0) wred[warp] = best;
  __syncthreads();
  if (warp == 0) {
    ArgMax b = lane < OD_T / 32 ? wred[lane] : ArgMax{-1.0, INT64_MAX};
    b = shfl_amax(b);
    if (lane == 0) {
      pv[blockIdx.x] = b.v;
      pe[blockIdx.x] = b.e;
      __threadfence();
      last = atomicAdd(cnt, 1u) == gridDim.x - 1;
    }
  }
  __syncthreads();
  if (!last) return;
  // fixed-order reduction of the per-CTA maxima (the max is order-free; ties by index)
  ArgMax b{-1.0, INT64_MAX};
  for (int q = tid; q < (int)gridDim.x; q += OD_T) b = amax(b, ArgMax{__ldcg(pv + q), __ldcg(pe + q)});
  b = shfl_amax(b);
  if (lane == 0) wred[warp] = b;
  __syncthreads();
  if (tid == 0) {
    ArgMax r{-1.0, INT64_MAX};
    for (int w = 0; w < OD_T / 32; ++w) r = amax(r, wred[w]);
    rows[j] = r.e;
    rows_out[j] = r.e;
    cells_out[j] = (int32_t)(r.e % N);
    chosen[r.e % N] = 1;
    *cnt = 0u;
  }
}

}  // namespace
}  // namespace hrom

using namespace hrom;

namespace hrom {
// the greedy of hrom_odeim with its chosen-rows workspace `rows_ws` (kOdeimMax entries):
// b.orows for the context's own points (the gappy rows of the ODEIM-mode step), b.orows_pub for
// the public call, so that inspecting another basis never overwrites the rows of the next step
static hrom_status odeim_points(hrom_ctx* c, const double* dev_phi, int32_t m, int32_t n_p, int64_t* rows_ws,
                                int32_t* dev_cells_out, int64_t* dev_rows_out) {
  const int64_t D = c->g.D, N = c->g.N;
  HROM_CK(cudaMemsetAsync(c->b.ochosen, 0, N, c->st));
  const int grid = (int)std::min<int64_t>(kOdeimBlocks, std::max<int64_t>(1, (D + OD_T - 1) / OD_T));
  for (int j = 0; j < n_p; ++j) {
    const int l = j % m;
    if (l > 0) {
      const size_t smem = (size_t)(l + 1) * j * sizeof(double);
      HROM_CK(cudaFuncSetAttribute(odeim_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      odeim_solve_kernel<<<1, OD_T, smem, c->st>>>(dev_phi, D, rows_ws, j, l, c->P.lsq_rel_cutoff, c->b.ocoef);
      HROM_LAUNCH_CK();
      ++c->nlaunch;
    }
    odeim_argmax_kernel<<<grid, OD_T, 0, c->st>>>(dev_phi, D, N, l, c->b.ocoef, c->b.ochosen, c->b.opart_v,
                                                   c->b.opart_e, c->b.ocnt, rows_ws, j, dev_cells_out,
                                                   dev_rows_out);
    HROM_LAUNCH_CK();
    ++c->nlaunch;
  }
  return HROM_OK;
}
}  // namespace hrom

extern "C" hrom_status hrom_odeim(hrom_ctx* c, const double* dev_phi, int32_t m, int32_t n_p,
                                  int32_t* dev_cells_out, int64_t* dev_rows_out) {
  if (!c || !dev_phi || !dev_cells_out || !dev_rows_out) return HROM_E_INVALID;
  if (m < 1 || m > kMaxR || n_p < 0 || n_p > kOdeimMax || n_p > c->g.N) return HROM_E_INVALID;
  return odeim_points(c, dev_phi, m, n_p, c->b.orows_pub, dev_cells_out, dev_rows_out);
}

namespace hrom {
// Algorithm 1 with ODEIM: the points of Phi_{k+1} (lifted into b.ophi) for the next step.  The
// greedy needs r_eff on the host (one stream synchronisation per basis); only in this mode.
hrom_status odeim_for_basis(hrom_ctx* c) {
  if (c->odeim_k == c->k && c->odeim_n > 0) return HROM_OK;
  if (!c->basis_ready) return HROM_E_STATE;
  basis_join(c);
  hrom_status s = lift(c, c->win, c->b.ophi, nullptr);
  if (s != HROM_OK) return s;
  int32_t reff = 0;
  HROM_CK(cudaMemcpyAsync(&reff, c->b.ireg, sizeof(int32_t), cudaMemcpyDeviceToHost, c->st));
  HROM_CK(cudaStreamSynchronize(c->st));
  const int np = (int)std::min<int64_t>(c->P.odeim_points, c->g.N);
  c->odeim_n = 0;
  if (reff < 1) return HROM_OK;
  if ((s = odeim_points(c, c->b.ophi, reff, np, c->b.orows, c->b.ocells, c->b.orows)) != HROM_OK) return s;
  c->odeim_n = np;
  c->odeim_k = c->k;
  return HROM_OK;
}
}  // namespace hrom
