// filter.cu -- H7: residual-gated Shapiro seam filter (one cooperative kernel).  The window-Gram
// contributions of the seam-band DOFs (final values) are computed by band_gram_rows (linalg.cu).
//
// Paper: explicit Shapiro filters applied dimension by dimension,
// zeroth-order boundary extrapolation, residual gate: keep filtered values only
// where the residual decreases; stop on an empty keep-set, a decrease below eps_f, or
// j_max^f sweeps; cascade 2 -> 4 -> 6.  Readings A21-A24: band
// B = (S-hat (+) Q_W) \ S-hat, residual per cell ||v - F||_inf over the c variables
// (F = full-RK3 values on B), relative eps_f test above the rounding level (A23'), x then y,
// stencils of S:386.
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
  const int32_t* hlist;  // halo cells (ascending), built with the sets
  const int32_t* hcount; // |halo|
  int32_t* idx;          // cell -> compact index (band t < nb, halo nb + h); N entries
  int32_t* tab;          // stencil tables: row (d * 7 + m + 3) * N + t, d = 0 x, 1 y
  SRef v;                // gamma_k (read, band values written back)
  SRef F;                // full-step values on B
  double* cur;           // compact: current values [var * N + t]
  double* cur0;          // compact: pre-filter values (band)
  double* Fb;            // compact: F on the band
  double* Vp;            // compact: x-filtered values (band) / fixed values (halo)
  double* Vpp;           // compact: second x-filtered buffer (x-passes alternate Vp / Vpp)
  uint8_t* flag;         // compact: bit0 ever kept, bits 1/2 keep-set of even/odd sweeps
  uint8_t* kept_cells;   // nullable: per-cell 1 where kept in some sweep (zeroed by the launcher)
  double* eps;
  unsigned long long* fdec;  // [2 kFilterSlots]: per sweep, max decrease (bits) and kept count
  int32_t* sweeps_out;   // [3]
  long long* tdbg;       // 64 timestamps (debug)
  int smem_bytes;        // dynamic shared memory of the launch (tables staged when they fit)
};

constexpr int FT = 512;  // filter threads per block (one block per SM)
constexpr int kFilterSlots = 64;  // >= orders * max sweeps
constexpr int FILTER_SMEM = 200 * 1024;

__device__ __forceinline__ void stamp(long long* t, int i) {
  if (t && i < 64 && blockIdx.x == 0 && threadIdx.x == 0) {
    long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    t[i] = g;
  }
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
  stamp(a.tdbg, 0);
  // gathers into the compact band + halo arrays (halo list, index map and stencil tables were
  // built with the sets, masks.cu sets_kernel)
  const int nh = *a.hcount;
  for (int64_t t = gtid; t < nb + nh; t += gstride) {
    const int64_t n = t < nb ? a.list[t] : a.hlist[t - nb];
    for (int var = 0; var < g.c; ++var) {
      const double x = a.v.p[sidx(a.v, var * N + n)];
      a.cur[var * N + t] = x;
      if (t < nb) {
        a.cur0[var * N + t] = x;
        a.Fb[var * N + t] = a.F.p[sidx(a.F, var * N + n)];
      } else {
        a.Vp[var * N + t] = x;   // halo: fixed values in both x-pass buffers
        a.Vpp[var * N + t] = x;
      }
    }
    a.flag[t] = 0;
  }
  if (blockIdx.x == 0)
    for (int i = threadIdx.x; i < 2 * kFilterSlots; i += blockDim.x) a.fdec[i] = 0ull;
  grid.sync();
  stamp(a.tdbg, 1);
  // Each CTA owns a contiguous chunk of the band made of WHOLE grid rows (the band list is
  // row-major): the x-stencil of a band cell then only reads cells of its own chunk or fixed
  // halo values, so the x-pass of sweep s+1 follows the y-pass of sweep s after a block barrier,
  // and one grid barrier per sweep remains (the y-pass reads x-filtered values of other rows).
  // The stop decision of sweep s is read after that barrier, so the x-pass of sweep s+1 runs
  // speculatively (its values are scratch when the order stops).  Stencil tables and F of the
  // chunk are staged in shared memory once.
  extern __shared__ double fsm[];
  __shared__ int s_bound[2];
  const int64_t nominal = ((int64_t)nb + gridDim.x - 1) / gridDim.x;
  for (int side = 0; side < 2; ++side) {
    // first list index >= the nominal split that starts a new grid row (one parallel probe:
    // a row holds at most nx band cells)
    const int64_t s0 = min((int64_t)(blockIdx.x + side) * nominal, (int64_t)nb);
    if (threadIdx.x == 0) s_bound[side] = (int)nb;
    __syncthreads();
    if (s0 == 0 || s0 >= nb) {
      if (threadIdx.x == 0) s_bound[side] = (int)s0;
    } else {
      const int r0 = a.list[s0 - 1] / g.nx;
      const int64_t span = g.nx + 1, per = (span + blockDim.x - 1) / blockDim.x;
      for (int64_t q = 0; q < per; ++q) {
        const int64_t t = s0 + (int64_t)threadIdx.x * per + q;
        if (t < nb && a.list[t] / g.nx != r0) {
          atomicMin(&s_bound[side], (int)t);
          break;
        }
      }
    }
    __syncthreads();
  }
  const int64_t c0 = s_bound[0], c1 = max(s_bound[1], s_bound[0]);
  const int64_t chunk = c1 - c0;
  const bool tsm = chunk * (14 * sizeof(int32_t) + g.c * sizeof(double)) <= (size_t)a.smem_bytes;
  double* sFb = fsm;                                      // [var][chunk]
  int32_t* stab = reinterpret_cast<int32_t*>(fsm + (tsm ? g.c * chunk : 0));  // [14][chunk]
  if (tsm) {
    for (int64_t t = c0 + threadIdx.x; t < c1; t += blockDim.x) {
      const int64_t lt = t - c0;
#pragma unroll
      for (int m = 0; m < 14; ++m)
        if (g.dim == 2 || m < 7) stab[m * chunk + lt] = __ldcg(a.tab + (int64_t)m * N + t);
      for (int var = 0; var < g.c; ++var) sFb[var * chunk + lt] = __ldcg(a.Fb + var * N + t);
    }
    __syncthreads();
  }
  const int32_t* __restrict__ tab = a.tab;
  double* __restrict__ cur = a.cur;
  // x-passes alternate between two buffers: the speculative x-pass of sweep s+1 of one CTA may
  // run while another CTA's y-pass of sweep s still reads the x-filtered values of s (the grid
  // barrier after x-pass s+1 orders x-pass s+2, which reuses s's buffer, after every y-pass s)
  double* const Vbuf[2] = {a.Vp, a.Vpp};
  int xp = 0;  // x-passes issued (identical in every CTA)
  const double* __restrict__ Fb = a.Fb;
  uint8_t* __restrict__ flag = a.flag;
  int gs = 0;  // sweeps done over all orders
  for (int oi = 0; oi < a.norders; ++oi) {
    const double* cf;
    double den;
    const int rad = shapiro(a.orders[oi], &cf, &den);
    double cfr[7];
#pragma unroll
    for (int m = 0; m < 7; ++m) cfr[m] = m <= 2 * rad ? cf[m] : 0.0;
    // P1: v' = S^x(cur) on the chunk
    auto x_pass = [&]() {
      double* __restrict__ Vp = Vbuf[xp & 1];
      ++xp;
      for (int64_t t = c0 + threadIdx.x; t < c1; t += blockDim.x) {
        const int64_t lt = t - c0;
        int nbr[7];
#pragma unroll
        for (int m = 0; m < 7; ++m)
          nbr[m] = m <= 2 * rad ? (tsm ? stab[(m - rad + 3) * chunk + lt] : __ldcg(tab + (int64_t)(m - rad + 3) * N + t)) : 0;
        double x[4][7];
#pragma unroll
        for (int var = 0; var < 4; ++var)
#pragma unroll
          for (int m = 0; m < 7; ++m) x[var][m] = (var < g.c && m <= 2 * rad) ? __ldcg(cur + var * N + nbr[m]) : 0.0;
#pragma unroll
        for (int var = 0; var < 4; ++var) {
          if (var >= g.c) break;
          double sx = 0.0;
#pragma unroll
          for (int m = 0; m < 7; ++m)
            if (m <= 2 * rad) sx += cfr[m] * x[var][m];
          Vp[var * N + t] = sx / den;
        }
      }
    };
    int sweeps = 0;
    if (a.maxsw > 0) x_pass();
    for (int sw = 0;; ++sw) {
      grid.sync();  // Vp of sweep sw everywhere; statistics of sweep sw-1 complete
      if (sw > 0) {  // identical stop decision in every block
        const double md = __longlong_as_double((long long)__ldcg(a.fdec + gs - 1));
        const long long tot = (long long)__ldcg(a.fdec + kFilterSlots + gs - 1);
        stamp(a.tdbg, 1 + gs);
        if (tot == 0 || md < a.eps_f) break;
      }
      if (sw == a.maxsw) break;
      ++sweeps;
      // P2: v'' = S^y(v') on the chunk, residual gate, kept values applied in place
      const double* __restrict__ Vp = Vbuf[(xp - 1) & 1];
      double mdec = 0.0;
      int cnt = 0;
      for (int64_t t = c0 + threadIdx.x; t < c1; t += blockDim.x) {
        const int64_t lt = t - c0;
        int nbr[7];
#pragma unroll
        for (int m = 0; m < 7; ++m)
          nbr[m] = (g.dim == 2 && m <= 2 * rad)
                       ? (tsm ? stab[(7 + m - rad + 3) * chunk + lt] : __ldcg(tab + (int64_t)(7 + m - rad + 3) * N + t))
                       : 0;
        double own[4], fe[4], y[4][7];
#pragma unroll
        for (int var = 0; var < 4; ++var) {
          own[var] = var < g.c ? __ldcg(cur + var * N + t) : 0.0;
          fe[var] = var < g.c ? (tsm ? sFb[var * chunk + lt] : __ldcg(Fb + var * N + t)) : 0.0;
#pragma unroll
          for (int m = 0; m < 7; ++m) y[var][m] = (g.dim == 2 && var < g.c && m <= 2 * rad) ? __ldcg(Vp + var * N + nbr[m]) : 0.0;
        }
        double rold = 0.0, rnew = 0.0, fs = 0.0;
        double vpp[4];
#pragma unroll
        for (int var = 0; var < 4; ++var) {
          if (var >= g.c) break;
          double xv;
          if (g.dim == 2) {
            double sy = 0.0;
#pragma unroll
            for (int m = 0; m < 7; ++m)
              if (m <= 2 * rad) sy += cfr[m] * y[var][m];
            xv = sy / den;
          } else {
            xv = __ldcg(Vp + var * N + t);  // 1-D: no y-pass
          }
          vpp[var] = xv;
          rold = fmax(rold, fabs(own[var] - fe[var]));
          rnew = fmax(rnew, fabs(xv - fe[var]));
          fs = fmax(fs, fabs(fe[var]));
        }
        if (rnew < rold) {
#pragma unroll
          for (int var = 0; var < 4; ++var)
            if (var < g.c) cur[var * N + t] = vpp[var];
          if (!(flag[t] & 1)) flag[t] = 1;
          if (rold > 0x1p-40 * fs) mdec = fmax(mdec, (rold - rnew) / rold);  // A23': above rounding level
          ++cnt;
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        mdec = fmax(mdec, __shfl_xor_sync(0xffffffffu, mdec, o));
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
      }
      if ((threadIdx.x & 31) == 0) {
        sdec[threadIdx.x >> 5] = mdec;
        scnt[threadIdx.x >> 5] = cnt;
      }
      __syncthreads();  // also orders this block's cur writes before the next x-pass reads them
      if (threadIdx.x == 0) {
        double md = 0.0;
        int c = 0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
          md = fmax(md, sdec[k]);
          c += scnt[k];
        }
        // one atomic max (non-negative doubles order like their bit patterns) and one integer
        // add per CTA into this sweep's slot: order-independent, so every CTA reads the same
        atomicMax(a.fdec + gs, (unsigned long long)__double_as_longlong(md));
        atomicAdd(a.fdec + kFilterSlots + gs, (unsigned long long)c);
      }
      ++gs;
      if (sw + 1 < a.maxsw) x_pass();  // speculative: scratch if the order stops after sweep sw
    }
    if (gtid == 0 && a.sweeps_out) a.sweeps_out[oi] = sweeps;
    __syncthreads();  // this block's last y-pass before the next order's x-pass
  }
  grid.sync();  // every chunk's final values before the write-back
  // write the kept band values back, and the indicator on kept band cells:
  // eps_n = sum_v (v - (psi + Phi y))^2 (pre-filter value = psi + Phi y)
  for (int64_t t = gtid; t < nb; t += gstride) {
    if (!(flag[t] & 1)) continue;
    const int64_t n = a.list[t];
    double s = 0.0;
    for (int var = 0; var < g.c; ++var) {
      const double x = cur[var * N + t];
      a.v.p[sidx(a.v, var * N + n)] = x;
      const double d = x - a.cur0[var * N + t];
      s += d * d;
    }
    if (a.eps) a.eps[n] = s;
    if (a.kept_cells) a.kept_cells[n] = 1;
  }
}

// Small grids (N <= kFilterSmallN cells): the whole compact band + halo lives in the shared
// memory of ONE block, so a sweep costs two block barriers instead of grid barriers and L2 round
// trips (config 1: 30 sweeps over ~200 band cells).  Same compact layout, tables, arithmetic and
// stop rule as filter_kernel (bit-identical results).
constexpr int kFilterSmallN = 1024;
__global__ void __launch_bounds__(FT) filter_small_kernel(FilterArgs a) {
  const Geo& g = a.g;
  const int nb = *a.count, nh = *a.hcount, M = nb + nh;
  const int64_t N = g.N;
  extern __shared__ double fsm[];
  double* scur = fsm;                 // [c][M]
  double* sVp = scur + g.c * M;       // [c][M] (halo entries: fixed values)
  double* sF = sVp + g.c * M;         // [c][nb]
  int32_t* stab = reinterpret_cast<int32_t*>(sF + g.c * nb);  // [14][nb]
  uint8_t* sflag = reinterpret_cast<uint8_t*>(stab + 14 * nb);
  __shared__ double sdec[FT / 32];
  __shared__ int scnt[FT / 32];
  __shared__ int s_stop;
  for (int t = threadIdx.x; t < M; t += FT) {
    const int64_t n = t < nb ? a.list[t] : a.hlist[t - nb];
    for (int var = 0; var < g.c; ++var) {
      const double x = a.v.p[sidx(a.v, var * N + n)];
      scur[var * M + t] = x;
      if (t < nb) {
        a.cur0[var * N + t] = x;
        sF[var * nb + t] = a.F.p[sidx(a.F, var * N + n)];
      } else {
        sVp[var * M + t] = x;
      }
    }
    if (t < nb) {
      sflag[t] = 0;
      for (int m = 0; m < 14; ++m)
        if (g.dim == 2 || m < 7) stab[m * nb + t] = a.tab[(int64_t)m * N + t];
    }
  }
  __syncthreads();
  for (int oi = 0; oi < a.norders; ++oi) {
    const double* cf;
    double den;
    const int rad = shapiro(a.orders[oi], &cf, &den);
    double cfr[7];
#pragma unroll
    for (int m = 0; m < 7; ++m) cfr[m] = m <= 2 * rad ? cf[m] : 0.0;
    int sweeps = 0;
    for (int sw = 0; sw < a.maxsw; ++sw) {
      ++sweeps;
      for (int t = threadIdx.x; t < nb; t += FT) {  // P1: v' = S^x(cur)
        for (int var = 0; var < g.c; ++var) {
          double sx = 0.0;
#pragma unroll
          for (int m = 0; m < 7; ++m)
            if (m <= 2 * rad) sx += cfr[m] * scur[var * M + stab[(m - rad + 3) * nb + t]];
          sVp[var * M + t] = sx / den;
        }
      }
      __syncthreads();
      double mdec = 0.0;
      int cnt = 0;
      for (int t = threadIdx.x; t < nb; t += FT) {  // P2: v'' = S^y(v'), gate, apply
        double rold = 0.0, rnew = 0.0, fs = 0.0, vpp[4];
        for (int var = 0; var < g.c; ++var) {
          double xv;
          if (g.dim == 2) {
            double sy = 0.0;
#pragma unroll
            for (int m = 0; m < 7; ++m)
              if (m <= 2 * rad) sy += cfr[m] * sVp[var * M + stab[(7 + m - rad + 3) * nb + t]];
            xv = sy / den;
          } else {
            xv = sVp[var * M + t];
          }
          vpp[var] = xv;
          const double fe = sF[var * nb + t];
          rold = fmax(rold, fabs(scur[var * M + t] - fe));
          rnew = fmax(rnew, fabs(xv - fe));
          fs = fmax(fs, fabs(fe));
        }
        if (rnew < rold) {
          for (int var = 0; var < g.c; ++var) scur[var * M + t] = vpp[var];
          sflag[t] = 1;
          if (rold > 0x1p-40 * fs) mdec = fmax(mdec, (rold - rnew) / rold);  // A23': above rounding level
          ++cnt;
        }
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
        for (int k = 0; k < FT / 32; ++k) {
          md = fmax(md, sdec[k]);
          c += scnt[k];
        }
        s_stop = (c == 0 || md < a.eps_f) ? 1 : 0;
      }
      __syncthreads();
      if (s_stop) break;
    }
    if (threadIdx.x == 0 && a.sweeps_out) a.sweeps_out[oi] = sweeps;
  }
  for (int t = threadIdx.x; t < nb; t += FT) {
    if (!sflag[t]) continue;
    const int64_t n = a.list[t];
    double s2 = 0.0;
    for (int var = 0; var < g.c; ++var) {
      const double x = scur[var * M + t];
      a.v.p[sidx(a.v, var * N + n)] = x;
      const double d = x - a.cur0[var * N + t];
      s2 += d * d;
    }
    if (a.eps) a.eps[n] = s2;
    if (a.kept_cells) a.kept_cells[n] = 1;
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
  a.fdec = reinterpret_cast<unsigned long long*>(c->b.fstat);
  a.sweeps_out = c->b.ireg + 4;
  a.tdbg = c->b.dbg;
  if (kept_cells) HROM_CK(cudaMemsetAsync(kept_cells, 0, c->g.N, c->st));
  if (c->g.N <= kFilterSmallN) {
    // |B| + |halo| <= N: sized for the worst case
    const size_t smem = (size_t)c->g.c * 3 * c->g.N * sizeof(double) + (size_t)14 * c->g.N * sizeof(int32_t) + c->g.N;
    HROM_CK(cudaFuncSetAttribute(filter_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    filter_small_kernel<<<1, FT, smem, c->st>>>(a);
    HROM_LAUNCH_CK();
    ++c->nlaunch;
    return HROM_OK;
  }
  a.smem_bytes = FILTER_SMEM;
  HROM_CK(cudaFuncSetAttribute(filter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, FILTER_SMEM));
  void* args[] = {&a};
  HROM_CK(cudaLaunchCooperativeKernel((void*)filter_kernel, dim3(c->filter_blocks), dim3(FT), args, FILTER_SMEM,
                                      c->st));
  ++c->nlaunch;
  return HROM_OK;
}

int filter_occupancy() {
  int nb = 0;
  cudaFuncSetAttribute(filter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, FILTER_SMEM);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, filter_kernel, FT, FILTER_SMEM);
  return nb;
}

}  // namespace hrom
