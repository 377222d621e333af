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
#include "internal.cuh"

namespace cg = cooperative_groups;

namespace hrom {
namespace {

struct FilterArgs {
  Geo g;
  int orders[3];
  int norders, maxsw;
  double eps_f;
  const int32_t* list;   // band cells
  const int32_t* count;
  const uint32_t* mB;
  SRef v;                // gamma_k (in place)
  SRef F;                // full-step values on B
  double* Vp;
  double* Vpp;
  double* Vorig;
  uint8_t* kept;         // bit0: ever kept, bit1: kept this sweep
  double* eps;
  double* fstat;         // [grid]
  int32_t* fcnt;         // [grid]
  int32_t* sweeps_out;   // [3]
};

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

__global__ void __launch_bounds__(256) filter_kernel(FilterArgs a) {
  cg::grid_group grid = cg::this_grid();
  const Geo& g = a.g;
  const int nb = *a.count;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  __shared__ double sdec[8];
  __shared__ int scnt[8];
  for (int64_t t = gtid; t < nb; t += gstride) {
    const int64_t n = a.list[t];
    for (int var = 0; var < g.c; ++var) a.Vorig[var * g.N + n] = a.v.p[sidx(a.v, var * g.N + n)];
  }
  grid.sync();
  // Two grid barriers per sweep: the keep-set of sweep s (flag bit 1 + (s & 1), values in Vpp)
  // is applied lazily by the x-pass of sweep s+1, which reads cur(m) = kept_s(m) ? Vpp(m) : v(m)
  // and writes its own cell; every block takes the same stop decision from per-block stats.
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
      // P1: apply the previous keep-set to the own cell, v' = S^x(cur) on B
      for (int64_t t = gtid; t < nb; t += gstride) {
        const int64_t n = a.list[t];
        const int i = (int)(n % g.nx), j = (int)(n / g.nx);
        const int64_t row = (int64_t)j * g.nx;
        for (int var = 0; var < g.c; ++var) {
          const int64_t rb = var * g.N + row;
          double s = 0.0;
          for (int m = -rad; m <= rad; ++m) {
            const int64_t nn = row + wrapf(i + m, g.nx, g.bc);
            const int64_t e = rb + (nn - row);
            const double cur = (gs > 0 && (a.kept[nn] & pbit)) ? a.Vpp[e] : a.v.p[sidx(a.v, e)];
            s += cf[m + rad] * cur;
          }
          a.Vp[var * g.N + n] = s / den;
        }
        if (gs > 0 && (a.kept[n] & pbit))
          for (int var = 0; var < g.c; ++var) a.v.p[sidx(a.v, var * g.N + n)] = a.Vpp[var * g.N + n];
      }
      grid.sync();
      // P2: v'' = S^y(v') on B, residual gate
      double mdec = 0.0;
      int cnt = 0;
      for (int64_t t = gtid; t < nb; t += gstride) {
        const int64_t n = a.list[t];
        const int i = (int)(n % g.nx), j = (int)(n / g.nx);
        double rold = 0.0, rnew = 0.0;
        double vpp[4];
        for (int var = 0; var < g.c; ++var) {
          const int64_t e = var * g.N + n;
          double x;
          if (g.dim == 2) {
            double s = 0.0;
            for (int m = -rad; m <= rad; ++m) {
              const int jj = wrapf(j + m, g.ny, g.bc);
              const int64_t nn = (int64_t)jj * g.nx + i;
              const double val = bitB(a.mB, g, i, jj) ? a.Vp[var * g.N + nn] : a.v.p[sidx(a.v, var * g.N + nn)];
              s += cf[m + rad] * val;
            }
            x = s / den;
          } else {
            x = a.Vp[e];
          }
          vpp[var] = x;
          const double fe = a.F.p[sidx(a.F, e)];
          rold = fmax(rold, fabs(a.v.p[sidx(a.v, e)] - fe));
          rnew = fmax(rnew, fabs(x - fe));
        }
        uint8_t fl = (uint8_t)(a.kept[n] & ~(pbit | cbit));
        if (rnew < rold) {
          for (int var = 0; var < g.c; ++var) a.Vpp[var * g.N + n] = vpp[var];
          fl |= (uint8_t)(cbit | 1u);
          mdec = fmax(mdec, (rold - rnew) / rold);
          ++cnt;
        }
        a.kept[n] = fl;
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
  // apply the last pending keep-set
  if (gs > 0) {
    const uint8_t pbit = (uint8_t)(2u << ((gs + 1) & 1));
    for (int64_t t = gtid; t < nb; t += gstride) {
      const int64_t n = a.list[t];
      if (a.kept[n] & pbit)
        for (int var = 0; var < g.c; ++var) a.v.p[sidx(a.v, var * g.N + n)] = a.Vpp[var * g.N + n];
    }
  }
  // indicator on kept band cells: eps_n = sum_v (v - (psi + Phi y))^2, pre-filter value = psi + Phi y
  for (int64_t t = gtid; t < nb; t += gstride) {
    const int64_t n = a.list[t];
    if (a.kept[n] & 1) {
      double s = 0.0;
      for (int var = 0; var < g.c; ++var) {
        const double d = a.v.p[sidx(a.v, var * g.N + n)] - a.Vorig[var * g.N + n];
        s += d * d;
      }
      if (a.eps) a.eps[n] = s;
    }
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

hrom_status launch_filter(hrom_ctx* c, SRef v, SRef F) {
  FilterArgs a{};
  a.g = c->g;
  for (int i = 0; i < 3; ++i) a.orders[i] = c->P.filter_orders[i];
  a.norders = c->P.n_filter_orders;
  a.maxsw = c->P.filter_max_sweeps;
  a.eps_f = c->P.filter_eps;
  a.list = c->b.lists + (int64_t)L_B * c->g.N;
  a.count = c->b.counts + L_B;
  a.mB = c->b.masks + (int64_t)M_B * c->mwords;
  a.v = v;
  a.F = F;
  a.Vp = c->b.U1;
  a.Vpp = c->b.U2;
  a.Vorig = c->b.Vorig;
  a.kept = c->b.kept;
  a.eps = c->b.eps;
  a.fstat = c->b.fstat;
  a.fcnt = c->b.fcnt;
  a.sweeps_out = c->b.ireg + 4;
  HROM_CK(cudaMemsetAsync(c->b.kept, 0, c->g.N, c->st));  // keep flags are read at band neighbours
  void* args[] = {&a};
  HROM_CK(cudaLaunchCooperativeKernel((void*)filter_kernel, dim3(c->filter_blocks), dim3(256), args, 0, c->st));
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
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, filter_kernel, 256, 0);
  return nb;
}

}  // namespace hrom
