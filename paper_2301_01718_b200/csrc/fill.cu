// fill.cu -- H6 + H9 + incremental H10: ONE pass over the snapshot window per hybrid step.
//
// For every DOF e the kernel streams the w+1 window columns gamma_{k-w-1..k-1} and the Gram
// shift rho once from HBM and
//   * fills gamma_k[e] = psi_k + Phi_k y_k = psi_cur + sum_i c_i (gamma_{x_i} - psi_prev)
//     (Alg. 1 line P:570; Phi_k = X^{(k-1)} A kept implicit), or takes the
//     partial-HDM value on S-hat (Eq. 6b),
//   * writes the per-DOF squared reconstruction error on S-hat,
//   * accumulates the new row of the shifted window Gram <gamma_k - rho, gamma_s - rho>
//     for every window slot s (reading A14), skipping seam-band cells (added after the
//     filter by filter.cu).
// psi_prev / psi_cur are recomputed from the columns in registers: the
// reference state is never stored or drifted.
//
// Register streaming: thread per DOF; all of a DOF's window loads are in flight at once
// (coalesced 256-byte warp segments per column), the values stay in registers for their
// second use (the Gram row) whose per-thread products accumulate in shared memory.  No
// staging copies, no CTA barrier in the stream.
#include <algorithm>
#include <cstdlib>
#include "internal.cuh"

namespace hrom {
namespace {

constexpr int FILL_THREADS = 128;

enum { MODE_FILL = 0, MODE_READ = 1, MODE_PROJ = 2 };

struct FillArgs {
  Geo g;
  Win W;
  int mode;
  int do_gram;
  const double* ring;
  const double* rho;
  const double* cvec;      // w coefficients (c = A y, or projection z)
  const double* src_S;     // HDM values on S-hat (MODE_FILL)
  double* out;             // gamma_k (MODE_FILL writes, MODE_READ reads)
  const uint32_t* mS;
  const uint32_t* mB;
  double* eps_elem;
  double* part;            // [grid][nU+1]
};

__device__ __forceinline__ double ld_stream(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.f64 %0, [%1];\n" : "=d"(v) : "l"(p));
  return v;
}

// Thread per DOF.  NU: compile-time bound of the window slots (register array of the
// DOF's window values, kept between the two uses); the per-thread Gram-row products are
// accumulated in shared memory (acc[s][thread]), conflict-free.
template <int NU, bool GRAM>
__global__ void __launch_bounds__(FILL_THREADS) fill_kernel(FillArgs a) {
  extern __shared__ double accs[];       // [NU+1][FILL_THREADS] (GRAM only)
  __shared__ double cs[kMaxW + 2];       // c_i, indexed by slot (0 for the psi_prev-only slot)
  const int nU = a.W.nU, w = a.W.w;
  const int xoff = nU - w;  // psi_cur and X use slots >= xoff; psi_prev uses slots < w
  const int tid = threadIdx.x;
  const Geo& g = a.g;
  for (int s = tid; s < nU; s += FILL_THREADS) cs[s] = (s >= xoff && a.cvec) ? a.cvec[s - xoff] : 0.0;
  if (GRAM)
    for (int s = 0; s <= NU; ++s) accs[s * FILL_THREADS + tid] = 0.0;
  __syncthreads();
  double csum = 0.0;
  for (int s = xoff; s < nU; ++s) csum += cs[s];
  const double inv_w = 1.0 / (double)w;
  const int64_t stride = (int64_t)gridDim.x * FILL_THREADS;
  // per-DOF side data (mask words, HDM value / new column) is fetched one iteration ahead
  uint32_t wS = 0, wB = 0;
  int bitpos = 0;
  double pre = 0.0;
  auto fetch = [&](int64_t e) {
    wS = wB = 0;
    pre = 0.0;
    if (e < g.D && a.mode != MODE_PROJ) {
      const int64_t n = e % g.N;
      const int i = (int)(n % g.nx), j = (int)(n / g.nx);
      const int64_t wi = (int64_t)j * g.wpr + (i >> 5);
      bitpos = i & 31;
      if (a.mode == MODE_FILL) {
        wS = a.mS[wi];
        if (a.mB) wB = a.mB[wi];
        pre = a.src_S[e];  // read unconditionally (allocated everywhere); used on S-hat only
      } else {
        pre = a.out[e];
      }
    }
  };
  int64_t e = (int64_t)blockIdx.x * FILL_THREADS + tid;
  fetch(e);
  for (; e < g.D; e += stride) {
    // all window loads of this DOF in flight together
    double x[NU];
#pragma unroll
    for (int s = 0; s < NU; ++s)
      if (s < nU) x[s] = ld_stream(a.ring + (int64_t)a.W.slot[s] * g.Dp + e);
    const double rh = ld_stream(a.rho + e);
    const bool inS = (wS >> bitpos) & 1u, inB = (wB >> bitpos) & 1u;
    const double side = pre;
    fetch(e + stride);
    // pass 1 (x_s = gamma_s - rho): sp = sum_{s<w} x_s, sc = sum_{s>=xoff} x_s,
    //                                tr = sum_{s>=xoff} c_{s-xoff} x_s  (two chains each)
    double sp = 0.0, sc = 0.0, tr = 0.0, sp2 = 0.0, sc2 = 0.0, tr2 = 0.0;
#pragma unroll
    for (int s = 0; s < NU; ++s) {
      if (s < nU) {
        x[s] -= rh;
        if (s & 1) {
          if (s < w) sp2 += x[s];
          if (s >= xoff) sc2 += x[s];
          tr2 += cs[s] * x[s];
        } else {
          if (s < w) sp += x[s];
          if (s >= xoff) sc += x[s];
          tr += cs[s] * x[s];
        }
      }
    }
    sp += sp2;
    sc += sc2;
    tr += tr2;
    double gval = 0.0;
    // psi_prev - rho = sp/w, psi_cur - rho = sc/w;  Phi y = sum_i c_i (x_i - (psi_prev - rho))
    const double dev = tr - (sp * inv_w) * csum;
    if (a.mode == MODE_FILL) {
      const double rec = (rh + sc * inv_w) + dev;
      gval = inS ? side : rec;
      if (inS) {
        const double d = gval - rec;
        a.eps_elem[e] = d * d;
      }
      a.out[e] = gval;
    } else if (a.mode == MODE_READ) {
      gval = side;
    } else {  // MODE_PROJ: residual of the projection onto the basis (bootstrap indicator)
      a.eps_elem[e] = dev * dev;
    }
    // pass 2: new Gram row (band DOFs are added after the filter)
    if (GRAM && !inB) {
      const double gr = gval - rh;
#pragma unroll
      for (int s = 0; s < NU; ++s)
        if (s < nU) accs[s * FILL_THREADS + tid] += gr * x[s];
      accs[NU * FILL_THREADS + tid] += gr * gr;
    }
  }
  if (!GRAM) return;
  // fixed-order reduction over the block's threads -> part[block][*]
  __syncthreads();
  double* outp = a.part + (int64_t)blockIdx.x * (nU + 1);
  for (int s = tid / 32; s <= nU; s += FILL_THREADS / 32) {
    const int row = (s == nU) ? NU : s;
    double v = 0.0;
    for (int t = tid & 31; t < FILL_THREADS; t += 32) v += accs[row * FILL_THREADS + t];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((tid & 31) == 0) outp[s] = v;
  }
}

// C[new][U[s]] = sum over blocks of fill partials (+ band partials), fixed order
__global__ void gram_row_reduce(const double* __restrict__ part, int nblk, Win W, int new_slot,
                                double* __restrict__ C, int ldc) {
  const int nU = W.nU;
  for (int s = threadIdx.x; s <= nU; s += blockDim.x) {
    double acc = 0.0;
    for (int b = 0; b < nblk; ++b) acc += part[(int64_t)b * (nU + 1) + s];
    if (s < nU) {
      C[new_slot * ldc + W.slot[s]] = acc;
      C[W.slot[s] * ldc + new_slot] = acc;
    } else {
      C[new_slot * ldc + new_slot] = acc;
    }
  }
}

// eps_n = sum_v eps_elem[v*N + n] on the listed cells (S-hat), P:363 summed over c (A16)
__global__ void eps_cells_kernel(Geo g, const int32_t* __restrict__ list, const int32_t* __restrict__ count,
                                 const double* __restrict__ eps_elem, double* __restrict__ eps) {
  const int total = *count;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const int64_t n = list[t];
    double s = 0.0;
    for (int v = 0; v < g.c; ++v) s += eps_elem[v * g.N + n];
    eps[n] = s;
  }
}

__global__ void eps_all_kernel(Geo g, const double* __restrict__ eps_elem, double* __restrict__ eps) {
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < g.N; n += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int v = 0; v < g.c; ++v) s += eps_elem[v * g.N + n];
    eps[n] = s;
  }
}

// rho (or psi) = mean of the last w window slots
__global__ void mean_kernel(Geo g, Win W, const double* __restrict__ ring, double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < g.D; e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int q = W.nU - W.w; q < W.nU; ++q) s += ring[(int64_t)W.slot[q] * g.Dp + e];
    out[e] = s / (double)W.w;
  }
}

template <int NU, bool GRAM>
hrom_status launch_fill_t(hrom_ctx* c, const FillArgs& a) {
  const size_t smem = GRAM ? (size_t)(NU + 1) * FILL_THREADS * sizeof(double) : 0;
  HROM_CK(cudaFuncSetAttribute(fill_kernel<NU, GRAM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fill_kernel<NU, GRAM>, FILL_THREADS, smem);
  const int grid = std::min(c->fill_blocks, c->nsm * std::max(occ, 1));
  fill_kernel<NU, GRAM><<<grid, FILL_THREADS, smem, c->st>>>(a);
  HROM_LAUNCH_CK();
  ++c->nlaunch;
  c->fill_grid = grid;
  return HROM_OK;
}

}  // namespace

int fill_max_gram_slots() { return 68; }
hrom_status reduce_band_rows(hrom_ctx* c, const Win& W, int new_slot);

hrom_status launch_fill(hrom_ctx* c, const Win& W, int mode, const double* src_S, double* out, int /*out_slot*/) {
  FillArgs a{};
  a.g = c->g;
  a.W = W;
  a.mode = mode;
  a.do_gram = (mode != MODE_PROJ) && out != nullptr && c->P.gram_mode == 0 ? 1 : 0;
  if (mode == MODE_FILL && out != nullptr && !(out >= c->b.ring && out < c->b.ring + (int64_t)c->nslots * c->g.Dp))
    a.do_gram = 0;  // standalone reconstruct into a caller buffer: no window Gram
  a.ring = c->b.ring;
  a.rho = c->b.rho;
  a.cvec = (mode == MODE_PROJ) ? c->b.zvec : c->b.cvec;
  a.src_S = src_S;
  a.out = out;
  a.mS = c->b.masks + (int64_t)M_S * c->mwords;
  a.mB = (mode == MODE_FILL) ? c->b.masks + (int64_t)M_B * c->mwords : nullptr;
  a.eps_elem = c->b.eps_elem;
  a.part = c->b.gpart;
  if (a.do_gram) {
    if (W.nU <= 12) return launch_fill_t<12, true>(c, a);
    if (W.nU <= 24) return launch_fill_t<24, true>(c, a);
    if (W.nU <= 36) return launch_fill_t<36, true>(c, a);
    if (W.nU <= 52) return launch_fill_t<52, true>(c, a);
    if (W.nU <= 68) return launch_fill_t<68, true>(c, a);
    return HROM_E_INVALID;  // wider windows with a Gram row use gram_mode = 1 (hrom_create)
  }
  if (W.nU <= 12) return launch_fill_t<12, false>(c, a);
  if (W.nU <= 24) return launch_fill_t<24, false>(c, a);
  if (W.nU <= 36) return launch_fill_t<36, false>(c, a);
  if (W.nU <= 68) return launch_fill_t<68, false>(c, a);
  if (W.nU <= 100) return launch_fill_t<100, false>(c, a);
  if (W.nU <= 132) return launch_fill_t<132, false>(c, a);
  return HROM_E_INVALID;
}

hrom_status launch_gram_row(hrom_ctx* c, const Win& W, int new_slot) {
  return launch_fill(c, W, MODE_READ, nullptr, c->b.ring + (int64_t)new_slot * c->g.Dp, new_slot);
}

hrom_status reduce_gram_row(hrom_ctx* c, const Win& W, int new_slot, bool with_band) {
  // fill partials occupy blocks [0, fill_grid); band partials follow at offset fill_blocks
  gram_row_reduce<<<1, 256, 0, c->st>>>(c->b.gpart, c->fill_grid, W, new_slot, c->b.C, kMaxSlots);
  HROM_LAUNCH_CK();
  ++c->nlaunch;
  // band partials are added into the same C entries (fixed order, after the fill part)
  if (with_band) return reduce_band_rows(c, W, new_slot);
  return HROM_OK;
}

__global__ void band_row_add(const double* __restrict__ part, int nblk, Win W, int new_slot, double* __restrict__ C,
                             int ldc) {
  const int nU = W.nU;
  for (int s = threadIdx.x; s <= nU; s += blockDim.x) {
    double acc = 0.0;
    for (int b = 0; b < nblk; ++b) acc += part[(int64_t)b * (nU + 1) + s];
    const int cs_ = (s < nU) ? W.slot[s] : new_slot;
    const double v = C[new_slot * ldc + cs_] + acc;
    C[new_slot * ldc + cs_] = v;
    C[cs_ * ldc + new_slot] = v;
  }
}

hrom_status reduce_band_rows(hrom_ctx* c, const Win& W, int new_slot) {
  band_row_add<<<1, 256, 0, c->st>>>(c->b.gpart + (int64_t)c->fill_blocks * (W.nU + 1), c->band_blocks, W, new_slot,
                                      c->b.C, kMaxSlots);
  HROM_LAUNCH_CK();
  ++c->nlaunch;
  return HROM_OK;
}

hrom_status launch_eps_cells(hrom_ctx* c) {
  eps_cells_kernel<<<c->nsm * 4, 256, 0, c->st>>>(c->g, c->b.lists + (int64_t)L_S * c->g.N, c->b.counts + L_S,
                                                   c->b.eps_elem, c->b.eps);
  HROM_LAUNCH_CK();
  ++c->nlaunch;
  return HROM_OK;
}

hrom_status launch_eps_all(hrom_ctx* c) {
  eps_all_kernel<<<c->nsm * 4, 256, 0, c->st>>>(c->g, c->b.eps_elem, c->b.eps);
  HROM_LAUNCH_CK();
  ++c->nlaunch;
  return HROM_OK;
}

hrom_status launch_mean(hrom_ctx* c, const Win& W, double* out) {
  mean_kernel<<<c->nsm * 8, 256, 0, c->st>>>(c->g, W, c->b.ring, out);
  HROM_LAUNCH_CK();
  ++c->nlaunch;
  return HROM_OK;
}

}  // namespace hrom
