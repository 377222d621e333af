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
// Register streaming: a DOF is owned by a lane pair (lane l and l+16); each lane loads its
// half of the window column values with coalesced 128-byte warp segments, all loads of a
// DOF in flight at once, keeps them in registers for the second use (Gram row) and keeps
// one Gram accumulator per slot.  No shared-memory staging, no CTA barrier in the stream.
#include <algorithm>
#include <cstdlib>
#include "internal.cuh"

namespace hrom {
namespace {

constexpr int FILL_THREADS = 128;
constexpr int FILL_WARPS = FILL_THREADS / 32;

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

// SH: compile-time slots per lane (a DOF's nU slots are split over the two half-warps)
template <int SH>
__global__ void __launch_bounds__(FILL_THREADS) fill_kernel(FillArgs a) {
  __shared__ double cs[kMaxW + 2];       // c_i, indexed by slot (0 for psi_prev-only slot)
  __shared__ double wred[FILL_WARPS][2 * SH + 1];
  const int nU = a.W.nU, w = a.W.w;
  const int xoff = nU - w;  // psi_cur and X use slots >= xoff; psi_prev uses slots < w
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int half = lane >> 4, sub = lane & 15;
  const Geo& g = a.g;
  for (int s = tid; s < nU; s += FILL_THREADS) cs[s] = (s >= xoff && a.cvec) ? a.cvec[s - xoff] : 0.0;
  __syncthreads();
  double csum = 0.0;
  for (int s = xoff; s < nU; ++s) csum += cs[s];
  const double inv_w = 1.0 / (double)w;
  // this lane's slots: half 0 -> [0, h0), half 1 -> [h0, nU)
  const int h0 = (nU + 1) / 2;
  const int s_begin = half ? h0 : 0, s_end = half ? nU : h0;
  double acc[SH];
#pragma unroll
  for (int i = 0; i < SH; ++i) acc[i] = 0.0;
  double acc_self = 0.0;
  const int64_t nchunks = (g.D + 15) / 16;
  const int64_t stride = (int64_t)gridDim.x * FILL_WARPS;
  // per-DOF side data (mask words, HDM value / new column) is fetched one chunk ahead
  uint32_t wS = 0, wB = 0;
  int bitpos = 0;
  double pre = 0.0;
  auto fetch = [&](int64_t chunk) {
    wS = wB = 0;
    pre = 0.0;
    const int64_t e = chunk * 16 + sub;
    if (half == 0 && chunk < nchunks && e < g.D && a.mode != MODE_PROJ) {
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
  int64_t chunk = (int64_t)blockIdx.x * FILL_WARPS + warp;
  fetch(chunk);
  for (; chunk < nchunks; chunk += stride) {
    const int64_t e = chunk * 16 + sub;
    const bool valid = e < g.D;
    const int64_t ec = valid ? e : 0;
    // all window loads of this lane in flight together
    double x[SH];
#pragma unroll
    for (int i = 0; i < SH; ++i) {
      const int s = s_begin + i;
      const double* col = (s < s_end) ? a.ring + (int64_t)a.W.slot[s] * g.Dp : a.rho;
      x[i] = ld_stream(col + ec);
    }
    const double rh = ld_stream(a.rho + ec);
    const bool inS = (wS >> bitpos) & 1u, inB = (wB >> bitpos) & 1u;
    const double sidev = pre;
    fetch(chunk + stride);
    // pass 1 on this lane's slots (x_s = gamma_s - rho):
    //   sp = sum_{s<w} x_s, sc = sum_{s>=xoff} x_s, tr = sum_{s>=xoff} c_{s-xoff} x_s
    double sp = 0.0, sc = 0.0, tr = 0.0;
#pragma unroll
    for (int i = 0; i < SH; ++i) {
      const int s = s_begin + i;
      x[i] -= rh;
      if (s < s_end) {
        if (s < w) sp += x[i];
        if (s >= xoff) sc += x[i];
        tr += cs[s] * x[i];
      }
    }
    // combine the two halves (a + b == b + a: both lanes get identical sums)
    sp += __shfl_xor_sync(0xffffffffu, sp, 16);
    sc += __shfl_xor_sync(0xffffffffu, sc, 16);
    tr += __shfl_xor_sync(0xffffffffu, tr, 16);
    const bool inS_p = __shfl_sync(0xffffffffu, inS, sub);
    const bool inB_p = __shfl_sync(0xffffffffu, inB, sub);
    const double side_p = __shfl_sync(0xffffffffu, sidev, sub);
    double gval = 0.0;
    // psi_prev - rho = sp/w, psi_cur - rho = sc/w;  Phi y = sum_i c_i (x_i - (psi_prev - rho))
    const double dev = tr - (sp * inv_w) * csum;
    if (a.mode == MODE_FILL) {
      const double rec = (rh + sc * inv_w) + dev;
      gval = inS_p ? side_p : rec;
      if (half == 0 && valid) {
        if (inS_p) {
          const double d = gval - rec;
          a.eps_elem[e] = d * d;
        }
        a.out[e] = gval;
      }
    } else if (a.mode == MODE_READ) {
      gval = side_p;
    } else if (half == 0 && valid) {  // MODE_PROJ: residual of the projection (bootstrap indicator)
      a.eps_elem[e] = dev * dev;
    }
    // pass 2: new Gram row on this lane's slots (band DOFs are added after the filter)
    if (a.do_gram && valid && !inB_p) {
      const double gr = gval - rh;
      if (half == 0) acc_self += gr * gr;
#pragma unroll
      for (int i = 0; i < SH; ++i) acc[i] += gr * x[i];
    }
  }
  if (!a.do_gram) return;
  // fixed-order reductions: 16 lanes of each half (shuffle tree), then warps -> part[block][*]
#pragma unroll
  for (int i = 0; i < SH; ++i) {
    double v = acc[i];
    for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (sub == 0) wred[warp][half * SH + i] = v;
  }
  {
    double v = acc_self;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) wred[warp][2 * SH] = v;
  }
  __syncthreads();
  double* outp = a.part + (int64_t)blockIdx.x * (nU + 1);
  for (int s = tid; s <= nU; s += FILL_THREADS) {
    int idx;
    if (s == nU) idx = 2 * SH;
    else idx = (s < h0) ? s : SH + (s - h0);
    double v = 0.0;
    for (int k = 0; k < FILL_WARPS; ++k) v += wred[k][idx];
    outp[s] = v;
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

template <int SH>
hrom_status launch_fill_t(hrom_ctx* c, const FillArgs& a) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fill_kernel<SH>, FILL_THREADS, 0);
  const int grid = std::min(c->fill_blocks, c->nsm * std::max(occ, 1));
  fill_kernel<SH><<<grid, FILL_THREADS, 0, c->st>>>(a);
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
  const int sh = (W.nU + 1) / 2;
  if (sh <= 6) return launch_fill_t<6>(c, a);
  if (sh <= 12) return launch_fill_t<12>(c, a);
  if (sh <= 18) return launch_fill_t<18>(c, a);
  if (sh <= 26) return launch_fill_t<26>(c, a);
  if (sh <= 34) return launch_fill_t<34>(c, a);
  if (!a.do_gram) {
    if (sh <= 50) return launch_fill_t<50>(c, a);
    if (sh <= 66) return launch_fill_t<66>(c, a);
  }
  return HROM_E_INVALID;  // wider windows with a Gram row use gram_mode = 1 (hrom_create)
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
