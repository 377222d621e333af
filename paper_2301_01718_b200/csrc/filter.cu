// filter.cu -- H7: residual-gated Shapiro seam filter (one cooperative kernel), plus the
// window-Gram contributions of the seam-band DOFs once their values are final.
//
// Paper: explicit Shapiro filters applied dimension by dimension,
// zeroth-order boundary extrapolation, residual gate: keep filtered values only
// where the residual decreases; stop on an empty keep-set, a decrease below eps_f, or
// j_max^f sweeps; cascade 2 -> 4 -> 6.  Readings A21-A24: band
// B = (S-hat (+) Q_W) \ S-hat, residual per cell ||v - F||_inf over the c variables
// (F = full-RK3 values on B), relative eps_f test, x then y, stencils of S:386.
#include <cooperative_groups.h>
#include <algorithm>
#include "internal.cuh"

namespace cg = cooperative_groups;

namespace hrom {
namespace {

struct FilterArgs {
  Geo g;
  int orders[3];
  int norders, maxsw, rmax;
  double eps_f;
  const int32_t* list;   // band cells B (ascending)
  const int32_t* count;  // |B|
  const uint32_t* mB;    // band bit mask
  uint32_t* mH;          // halo bit mask (zeroed by the launcher)
  int32_t* hlist;        // halo cells (ascending), written here
  int32_t* hcount;       // |halo| (written here)
  int32_t* idx;          // cell -> compact index (band t < nb, halo nb + h); N entries
  int32_t* tab;          // stencil tables: row (d * 7 + m + 3) * N + t, d = 0 x, 1 y
  SRef v;                // gamma_k (read, band values written back)
  SRef F;                // full-step values on B
  double* cur;           // compact: current values [var * N + t]
  double* cur0;          // compact: pre-filter values (band)
  double* Fb;            // compact: F on the band
  double* Vp;            // compact: x-filtered values (band) / fixed values (halo)
  double* Vpp;           // compact: y-filtered values (band)
  uint8_t* flag;         // compact: bit0 ever kept, bits 1/2 keep-set of even/odd sweeps
  uint8_t* kept_cells;   // nullable: per-cell 1 where kept in some sweep (zeroed by the launcher)
  double* eps;
  double* fstat;         // [grid]
  int32_t* fcnt;         // [grid]
  int32_t* sweeps_out;   // [3]
};

constexpr int FT = 512;  // filter threads per block (one block per SM)

__device__ __forceinline__ int wrapf(int i, int n, int bc) {
  if (bc == 1) {
    i %= n;
    return i < 0 ? i + n : i;
  }
  return i < 0 ? 0 : (i >= n ? n - 1 : i);
}

__device__ __forceinline__ bool bitB(const uint32_t* m, const Geo& g, int i, int j) {
  return (m[(int64_t)j * g.wpr + (i >> 5)] >> (i & 31)) & 1u;
}

// (1,2,1)/4, (-1,4,10,4,-1)/16, (1,-6,15,44,15,-6,1)/64  (A24)
__constant__ double c2[3] = {1, 2, 1};
__constant__ double c4[5] = {-1, 4, 10, 4, -1};
__constant__ double c6[7] = {1, -6, 15, 44, 15, -6, 1};

__device__ __forceinline__ int shapiro(int order, const double** c, double* den) {
  if (order == 2) { *c = c2; *den = 4.0; return 1; }
  if (order == 4) { *c = c4; *den = 16.0; return 2; }
  *c = c6; *den = 64.0; return 3;
}

// Compaction of the seam filter: the band B and its halo (cells within the
// largest stencil radius of B along x or y, not in B -- their values are fixed during the
// filter) are gathered once into compact arrays of |B| + |halo| entries with precomputed
// stencil tables, so every sweep works on an L2-resident working set instead of gathering
// through the snapshot slab.  Same arithmetic, same order as the per-cell formulation.
__global__ void __launch_bounds__(FT) filter_kernel(FilterArgs a) {
  cg::grid_group grid = cg::this_grid();
  const Geo& g = a.g;
  const int nb = *a.count;
  const int64_t N = g.N;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  __shared__ double sdec[FT / 32];
  __shared__ int scnt[FT / 32];
  __shared__ int sscan[FT];
  __shared__ int sbase;
  // S0: mark the halo
  for (int64_t t = gtid; t < nb; t += gstride) {
    const int64_t n = a.list[t];
    const int i = (int)(n % g.nx), j = (int)(n / g.nx);
    for (int m = -a.rmax; m <= a.rmax; ++m) {
      if (m == 0) continue;
      const int ii = wrapf(i + m, g.nx, g.bc);
      if (!bitB(a.mB, g, ii, j)) atomicOr(&a.mH[(int64_t)j * g.wpr + (ii >> 5)], 1u << (ii & 31));
      if (g.dim == 2) {
        const int jj = wrapf(j + m, g.ny, g.bc);
        if (!bitB(a.mB, g, i, jj)) atomicOr(&a.mH[(int64_t)jj * g.wpr + (i >> 5)], 1u << (i & 31));
      }
    }
  }
  grid.sync();
  // S1: ordered compaction of the halo mask -- block b owns a contiguous word range
  const int64_t nw = (int64_t)g.ny * g.wpr;
  const int64_t bchunk = (nw + gridDim.x - 1) / gridDim.x;
  const int64_t tchunk = (bchunk + blockDim.x - 1) / blockDim.x;
  const int64_t w0 = blockIdx.x * bchunk + threadIdx.x * tchunk;
  const int64_t w1 = min(min(w0 + tchunk, (int64_t)(blockIdx.x + 1) * bchunk), nw);
  int mine = 0;
  for (int64_t wi = w0; wi < w1; ++wi) mine += __popc(a.mH[wi]);
  sscan[threadIdx.x] = mine;
  __syncthreads();
  for (int o = 1; o < (int)blockDim.x; o <<= 1) {  // inclusive Hillis-Steele scan
    const int x = threadIdx.x >= o ? sscan[threadIdx.x - o] : 0;
    __syncthreads();
    sscan[threadIdx.x] += x;
    __syncthreads();
  }
  if (threadIdx.x == 0) a.fcnt[blockIdx.x] = sscan[blockDim.x - 1];
  grid.sync();
  if (threadIdx.x == 0) {
    int base = 0, tot = 0;
    for (int b = 0; b < (int)gridDim.x; ++b) {
      if (b < (int)blockIdx.x) base += a.fcnt[b];
      tot += a.fcnt[b];
    }
    sbase = base;
    if (blockIdx.x == 0) *a.hcount = tot;
  }
  __syncthreads();
  {
    int pos = sbase + sscan[threadIdx.x] - mine;
    for (int64_t wi = w0; wi < w1; ++wi) {
      uint32_t bits = a.mH[wi];
      const int64_t j = wi / g.wpr, i0 = (wi % g.wpr) * 32;
      while (bits) {
        const int bpos = __ffs(bits) - 1;
        bits &= bits - 1;
        a.hlist[pos++] = (int32_t)(j * g.nx + i0 + bpos);
      }
    }
  }
  grid.sync();
  const int nh = *a.hcount;
  // S2: index map and gathers
  for (int64_t t = gtid; t < nb + nh; t += gstride) {
    const int64_t n = t < nb ? a.list[t] : a.hlist[t - nb];
    a.idx[n] = (int32_t)t;
    for (int var = 0; var < g.c; ++var) {
      const double x = a.v.p[sidx(a.v, var * N + n)];
      a.cur[var * N + t] = x;
      if (t < nb) {
        a.cur0[var * N + t] = x;
        a.Fb[var * N + t] = a.F.p[sidx(a.F, var * N + n)];
      } else {
        a.Vp[var * N + t] = x;
      }
    }
    a.flag[t] = 0;
  }
  grid.sync();
  // S3: stencil tables
  for (int64_t t = gtid; t < nb; t += gstride) {
    const int64_t n = a.list[t];
    const int i = (int)(n % g.nx), j = (int)(n / g.nx);
    for (int m = -a.rmax; m <= a.rmax; ++m) {
      a.tab[(int64_t)(m + 3) * N + t] = a.idx[(int64_t)j * g.nx + wrapf(i + m, g.nx, g.bc)];
      if (g.dim == 2) a.tab[(int64_t)(7 + m + 3) * N + t] = a.idx[(int64_t)wrapf(j + m, g.ny, g.bc) * g.nx + i];
    }
  }
  grid.sync();
  // Sweeps, two grid barriers each: the keep-set of sweep s (flag bit 1 + (s & 1), values in
  // Vpp) is applied lazily by the x-pass of sweep s+1, which reads cur(m) = kept_s(m) ? Vpp(m)
  // : cur(m) and writes its own cell; every block takes the same stop decision.
  int gs = 0;  // sweeps done over all orders
  for (int oi = 0; oi < a.norders; ++oi) {
    const double* cf;
    double den;
    const int rad = shapiro(a.orders[oi], &cf, &den);
    int sweeps = 0;
    for (int sw = 0; sw < a.maxsw; ++sw, ++gs) {
      ++sweeps;
      const uint8_t pbit = (uint8_t)(2u << ((gs + 1) & 1));  // keep bit of the previous sweep
      const uint8_t cbit = (uint8_t)(2u << (gs & 1));        // keep bit of this sweep
      // P1: v' = S^x(cur) on B
      for (int64_t t = gtid; t < nb; t += gstride) {
        int nbr[7];
        bool kp[7];
#pragma unroll
        for (int m = 0; m < 7; ++m) {
          nbr[m] = m <= 2 * rad ? a.tab[(int64_t)(m - rad + 3) * N + t] : 0;
          kp[m] = m <= 2 * rad && gs > 0 && (a.flag[nbr[m]] & pbit);
        }
        const bool own = gs > 0 && (a.flag[t] & pbit);
        for (int var = 0; var < g.c; ++var) {
          const int64_t vb = var * N;
          double s = 0.0;
#pragma unroll
          for (int m = 0; m < 7; ++m) {
            if (m > 2 * rad) break;
            const double x = kp[m] ? a.Vpp[vb + nbr[m]] : a.cur[vb + nbr[m]];
            s += cf[m] * x;
          }
          a.Vp[vb + t] = s / den;
          if (own) a.cur[vb + t] = a.Vpp[vb + t];
        }
      }
      grid.sync();
      // P2: v'' = S^y(v') on B, residual gate
      double mdec = 0.0;
      int cnt = 0;
      for (int64_t t = gtid; t < nb; t += gstride) {
        int nbr[7];
#pragma unroll
        for (int m = 0; m < 7; ++m) nbr[m] = (g.dim == 2 && m <= 2 * rad) ? a.tab[(int64_t)(7 + m - rad + 3) * N + t] : 0;
        double rold = 0.0, rnew = 0.0;
        double vpp[4];
#pragma unroll
        for (int var = 0; var < 4; ++var) {
          if (var >= g.c) break;
          const int64_t vb = var * N;
          double x;
          if (g.dim == 2) {
            double s = 0.0;
#pragma unroll
            for (int m = 0; m < 7; ++m) {
              if (m > 2 * rad) break;
              s += cf[m] * a.Vp[vb + nbr[m]];
            }
            x = s / den;
          } else {
            x = a.Vp[vb + t];
          }
          vpp[var] = x;
          const double fe = a.Fb[vb + t];
          rold = fmax(rold, fabs(a.cur[vb + t] - fe));
          rnew = fmax(rnew, fabs(x - fe));
        }
        uint8_t fl = (uint8_t)(a.flag[t] & ~(pbit | cbit));
        if (rnew < rold) {
#pragma unroll
          for (int var = 0; var < 4; ++var)
            if (var < g.c) a.Vpp[var * N + t] = vpp[var];
          fl |= (uint8_t)(cbit | 1u);
          mdec = fmax(mdec, (rold - rnew) / rold);
          ++cnt;
        }
        a.flag[t] = fl;
      }
      for (int o = 16; o > 0; o >>= 1) {
        mdec = fmax(mdec, __shfl_xor_sync(0xffffffffu, mdec, o));
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
      }
      if ((threadIdx.x & 31) == 0) {
        sdec[threadIdx.x >> 5] = mdec;
        scnt[threadIdx.x >> 5] = cnt;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        double md = 0.0;
        int c = 0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
          md = fmax(md, sdec[k]);
          c += scnt[k];
        }
        a.fstat[blockIdx.x] = md;
        a.fcnt[blockIdx.x] = c;
      }
      grid.sync();
      // identical stop decision in every block (fixed-order reduction of the block stats)
      double md = 0.0;
      long long tot = 0;
      for (int b = 0; b < (int)gridDim.x; ++b) {
        md = fmax(md, a.fstat[b]);
        tot += a.fcnt[b];
      }
      if (tot == 0 || md < a.eps_f) {
        ++gs;
        break;
      }
    }
    if (gtid == 0 && a.sweeps_out) a.sweeps_out[oi] = sweeps;
  }
  // apply the last pending keep-set, write the kept band values back, and the indicator on
  // kept band cells: eps_n = sum_v (v - (psi + Phi y))^2 (pre-filter value = psi + Phi y)
  const uint8_t pbit = (uint8_t)(2u << ((gs + 1) & 1));
  for (int64_t t = gtid; t < nb; t += gstride) {
    const uint8_t fl = a.flag[t];
    if (!(fl & 1)) continue;
    const int64_t n = a.list[t];
    const bool pend = gs > 0 && (fl & pbit);
    double s = 0.0;
    for (int var = 0; var < g.c; ++var) {
      const double x = pend ? a.Vpp[var * N + t] : a.cur[var * N + t];
      a.v.p[sidx(a.v, var * N + n)] = x;
      const double d = x - a.cur0[var * N + t];
      s += d * d;
    }
    if (a.eps) a.eps[n] = s;
    if (a.kept_cells) a.kept_cells[n] = 1;
  }
}

// Gram-row contributions of the band DOFs (final values), partials after the fill blocks
__global__ void __launch_bounds__(256) band_gram_kernel(Geo g, Win W, const double* __restrict__ ring,
                                                        const SRef rho, const SRef v,
                                                        const int32_t* __restrict__ list,
                                                        const int32_t* __restrict__ count, double* __restrict__ part) {
  constexpr int CH = 128;
  constexpr int SPW = (kMaxW + 2 + 7) / 8;
  __shared__ double gt[CH], rh[CH];
  __shared__ int64_t es[CH];
  __shared__ double wsum[8];
  const int nU = W.nU;
  const int nb = *count;
  const int64_t total = (int64_t)nb * g.c;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc[SPW];
#pragma unroll
  for (int q = 0; q < SPW; ++q) acc[q] = 0.0;
  double self = 0.0;
  for (int64_t base = (int64_t)blockIdx.x * CH; base < total; base += (int64_t)gridDim.x * CH) {
    if (threadIdx.x < CH) {
      const int64_t t = base + threadIdx.x;
      if (t < total) {
        const int var = (int)(t / nb), idx = (int)(t % nb);
        const int64_t e = (int64_t)var * g.N + list[idx];
        const double r = rho.p[sidx(rho, e)];
        const double x = v.p[sidx(v, e)] - r;
        gt[threadIdx.x] = x;
        rh[threadIdx.x] = r;
        es[threadIdx.x] = sidx(SRef{nullptr, g.nsr}, e);  // slab offset within a ring slot
        self += x * x;
      } else {
        gt[threadIdx.x] = 0.0;
        rh[threadIdx.x] = 0.0;
        es[threadIdx.x] = -1;
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < SPW; ++q) {
      const int s = warp + q * 8;
      if (s < nU) {
        const double* col = ring + (int64_t)W.slot[s] * TILE;
        double sacc = 0.0;
        for (int el = lane; el < CH; el += 32)
          if (es[el] >= 0) sacc += gt[el] * (col[es[el]] - rh[el]);
        acc[q] += sacc;
      }
    }
    __syncthreads();
  }
  double* out = part + (int64_t)blockIdx.x * (nU + 1);
#pragma unroll
  for (int q = 0; q < SPW; ++q) {
    double x = acc[q];
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    const int s = warp + q * 8;
    if (lane == 0 && s < nU) out[s] = x;
  }
  for (int o = 16; o > 0; o >>= 1) self += __shfl_xor_sync(0xffffffffu, self, o);
  if (lane == 0) wsum[warp] = self;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int k = 0; k < 8; ++k) s += wsum[k];
    out[nU] = s;
  }
}

}  // namespace

hrom_status launch_filter(hrom_ctx* c, SRef v, SRef F, uint8_t* kept_cells) {
  FilterArgs a{};
  a.g = c->g;
  a.rmax = 0;
  for (int i = 0; i < 3; ++i) a.orders[i] = c->P.filter_orders[i];
  a.norders = c->P.n_filter_orders;
  for (int i = 0; i < a.norders; ++i) a.rmax = std::max(a.rmax, a.orders[i] / 2);
  a.maxsw = c->P.filter_max_sweeps;
  a.eps_f = c->P.filter_eps;
  a.list = c->b.lists + (int64_t)L_B * c->g.N;
  a.count = c->b.counts + L_B;
  a.mB = c->b.masks + (int64_t)M_B * c->mwords;
  a.mH = c->b.masks + (int64_t)M_TMP * c->mwords;
  a.hlist = c->b.lists + (int64_t)L_H * c->g.N;
  a.hcount = c->b.counts + L_H;
  a.idx = c->b.fidx;
  a.tab = c->b.ftab;
  a.v = v;
  a.F = F;
  a.cur = c->b.fcur;
  a.cur0 = c->b.Vorig;
  a.Fb = c->b.fF;
  a.Vp = c->b.U1;
  a.Vpp = c->b.U2;
  a.flag = c->b.kept;
  a.kept_cells = kept_cells;
  a.eps = c->b.eps;
  a.fstat = c->b.fstat;
  a.fcnt = c->b.fcnt;
  a.sweeps_out = c->b.ireg + 4;
  HROM_CK(cudaMemsetAsync(a.mH, 0, (size_t)c->g.ny * c->g.wpr * sizeof(uint32_t), c->st));
  if (kept_cells) HROM_CK(cudaMemsetAsync(kept_cells, 0, c->g.N, c->st));
  void* args[] = {&a};
  HROM_CK(cudaLaunchCooperativeKernel((void*)filter_kernel, dim3(c->filter_blocks), dim3(FT), args, 0, c->st));
  ++c->nlaunch;
  return HROM_OK;
}

hrom_status launch_band_gram(hrom_ctx* c, const Win& W, SRef v) {
  band_gram_kernel<<<c->band_blocks, 256, 0, c->st>>>(c->g, W, c->b.ring, c->rho_ref(), v,
                                                       c->b.lists + (int64_t)L_B * c->g.N, c->b.counts + L_B,
                                                       c->b.gpart + (int64_t)c->fill_blocks * (W.nU + 1));
  HROM_LAUNCH_CK();
  ++c->nlaunch;
  return HROM_OK;
}

int filter_occupancy() {
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, filter_kernel, FT, 0);
  return nb;
}

}  // namespace hrom
