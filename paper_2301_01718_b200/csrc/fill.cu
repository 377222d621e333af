// fill.cu -- H6 + H9 + incremental H10: ONE pass over the snapshot window per hybrid step.
//
// For every DOF e the kernel streams the w+1 window columns gamma_{k-w-1..k-1} and the Gram
// shift rho through shared memory (cp.async.bulk / TMA 1-D bulk copies, mbarrier pipeline) and
//   * fills gamma_k[e] = psi_k + Phi_k y_k = psi_cur + sum_i c_i (gamma_{x_i} - psi_prev)
//     (Alg. 1 line P:570; Phi_k = X^{(k-1)} A kept implicit), or takes the
//     partial-HDM value on S-hat (Eq. 6b),
//   * writes the per-DOF squared reconstruction error on S-hat,
//   * accumulates the new row of the shifted window Gram <gamma_k - rho, gamma_s - rho>
//     for every window slot s (reading A14), skipping seam-band cells (added after the
//     filter by filter.cu).
// psi_prev / psi_cur are recomputed from the columns in registers: the
// reference state is never stored or drifted.
#include <algorithm>
#include "internal.cuh"

namespace hrom {
namespace {

// Tiles of TE DOFs; 2*TE threads: two threads per DOF share the slot loop (phase A),
// TE/32*2 warps share the window slots in the Gram-row phase (phase B).
constexpr int TE_FILL = 64;

enum { MODE_FILL = 0, MODE_READ = 1, MODE_PROJ = 2 };

struct FillArgs {
  Geo g;
  Win W;
  int mode;
  int do_gram;
  int nstage;
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

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ bool bit_of(const uint32_t* m, const Geo& g, int64_t n) {
  const int i = (int)(n % g.nx), j = (int)(n / g.nx);
  return (m[(int64_t)j * g.wpr + (i >> 5)] >> (i & 31)) & 1u;
}

template <int TE, int SPW>
__global__ void __launch_bounds__(2 * TE) fill_kernel(FillArgs a) {
  constexpr int FT = 2 * TE, NW = FT / 32;
  extern __shared__ __align__(128) unsigned char smraw[];
  const int nU = a.W.nU, w = a.W.w;
  const int ncol = nU + 1;  // window slots + rho
  double* stage0 = reinterpret_cast<double*>(smraw);
  const size_t stage_elems = (size_t)ncol * TE;
  double* gt = stage0 + a.nstage * stage_elems;      // TE: g - rho (0 on band cells)
  double* red = gt + TE;                              // [3][TE] partial sums of part 1
  uint64_t* bars = reinterpret_cast<uint64_t*>(red + 3 * TE);
  __shared__ double cs[kMaxW];
  __shared__ double csum_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Geo& g = a.g;
  for (int i = tid; i < w; i += FT) cs[i] = a.cvec ? a.cvec[i] : 0.0;
  if (tid == 0) {
    for (int s = 0; s < a.nstage; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int i = 0; i < w; ++i) t += cs[i];
    csum_s = t;
  }
  const int64_t ntiles = (g.D + TE - 1) / TE;
  auto issue = [&](int64_t tile, int st) {
    const int64_t e0 = tile * TE;
    const int64_t cnt = (g.D - e0) < TE ? (g.D - e0) : TE;
    const uint32_t bytes = (uint32_t)(((cnt + 1) / 2) * 2 * sizeof(double));
    double* dst = stage0 + st * stage_elems;
    // warp 0 issues the ncol bulk copies lane-parallel (one elected lane arms the barrier)
    if (lane == 0) mbar_expect(&bars[st], bytes * ncol);
    __syncwarp();
    for (int s = lane; s <= nU; s += 32) {
      const double* src = (s < nU) ? a.ring + (int64_t)a.W.slot[s] * g.Dp + e0 : a.rho + e0;
      bulk_g2s(dst + (size_t)s * TE, src, bytes, &bars[st]);
    }
  };
  const int64_t first = blockIdx.x;
  if (warp == 0)
    for (int s = 0; s < a.nstage; ++s)
      if (first + (int64_t)s * gridDim.x < ntiles) issue(first + (int64_t)s * gridDim.x, s);
  double acc[SPW];
#pragma unroll
  for (int q = 0; q < SPW; ++q) acc[q] = 0.0;
  double acc_self = 0.0;
  __syncthreads();
  const double csum = csum_s;
  const int e_loc = tid % TE, part = tid / TE;
  const int xoff = nU - w;  // first X slot (psi_cur and X use slots >= xoff; psi_prev slots < w)
  const int half = (nU + 1) / 2;
  const int s0 = part ? half : 0, s1 = part ? nU : half;
  const double inv_w = 1.0 / (double)w;
  int it = 0;
  for (int64_t tile = first; tile < ntiles; tile += gridDim.x, ++it) {
    const int st = it % a.nstage;
    const uint32_t par = (uint32_t)((it / a.nstage) & 1);
    const int64_t e0 = tile * TE;
    const int64_t e = e0 + e_loc;
    const bool valid = e < g.D;
    // per-DOF global reads are issued before waiting on the stage (latency overlap)
    bool inS = false, inB = false;
    double srcv = 0.0, outv = 0.0;
    if (part == 0 && valid && a.mode != MODE_PROJ) {
      const int64_t n = e % g.N;
      if (a.mode == MODE_FILL) {
        inS = bit_of(a.mS, g, n);
        inB = a.mB && bit_of(a.mB, g, n);
        if (inS) srcv = a.src_S[e];
      } else {
        outv = a.out[e];
      }
    }
    mbar_wait(&bars[st], par);
    const double* T = stage0 + st * stage_elems;
    const double rh = T[nU * TE + e_loc];
    // phase A, one pass over this part's slots, shifted by rho (x_s = gamma_s - rho):
    //   sp = sum_{s<w} x_s,  sc = sum_{s>=xoff} x_s,  tr = sum_{s>=xoff} c_{s-xoff} x_s
    double sp0 = 0.0, sp1 = 0.0, sc0 = 0.0, sc1 = 0.0, tr0 = 0.0, tr1 = 0.0;
    {
      const int l1 = min(s1, xoff);
      for (int s = s0; s < l1; ++s) sp0 += T[s * TE + e_loc] - rh;
      const int m0 = max(s0, xoff), m1 = min(s1, w);
      int s = m0;
      for (; s + 1 < m1; s += 2) {
        const double x0 = T[s * TE + e_loc] - rh, x1 = T[(s + 1) * TE + e_loc] - rh;
        sp0 += x0; sp1 += x1; sc0 += x0; sc1 += x1;
        tr0 += cs[s - xoff] * x0; tr1 += cs[s + 1 - xoff] * x1;
      }
      if (s < m1) {
        const double x0 = T[s * TE + e_loc] - rh;
        sp0 += x0; sc0 += x0; tr0 += cs[s - xoff] * x0;
      }
      for (int s2 = max(s0, w); s2 < s1; ++s2) {
        const double x0 = T[s2 * TE + e_loc] - rh;
        sc1 += x0; tr1 += cs[s2 - xoff] * x0;
      }
    }
    if (part == 1) {
      red[e_loc] = sp0 + sp1;
      red[TE + e_loc] = sc0 + sc1;
      red[2 * TE + e_loc] = tr0 + tr1;
    }
    __syncthreads();
    if (part == 0) {
      double gval = 0.0;
      if (valid) {
        const double sp = (sp0 + sp1) + red[e_loc];
        const double sc = (sc0 + sc1) + red[TE + e_loc];
        const double tr = (tr0 + tr1) + red[2 * TE + e_loc];
        // psi_prev - rho = sp/w, psi_cur - rho = sc/w;  Phi y = sum_i c_i (x_i - (psi_prev - rho))
        const double dev = tr - (sp * inv_w) * csum;
        if (a.mode == MODE_FILL) {
          const double rec = (rh + sc * inv_w) + dev;
          if (inS) {
            gval = srcv;
            const double d = gval - rec;
            a.eps_elem[e] = d * d;
          } else {
            gval = rec;
          }
          a.out[e] = gval;
        } else if (a.mode == MODE_READ) {
          gval = outv;
        } else {  // MODE_PROJ: residual of the projection onto the basis (bootstrap indicator)
          a.eps_elem[e] = dev * dev;
        }
        const bool skip = inB || a.mode == MODE_PROJ;
        const double gr = skip ? 0.0 : gval - rh;
        gt[e_loc] = gr;
        acc_self += gr * gr;
      } else {
        gt[e_loc] = 0.0;
      }
    }
    __syncthreads();
    // phase B: Gram row, warp-per-slot-set, lanes over DOFs (rho and g hoisted per DOF)
    if (a.do_gram) {
      const int cnt = (int)((g.D - e0) < TE ? (g.D - e0) : TE);
#pragma unroll
      for (int j = 0; j < TE / 32; ++j) {
        const int el = lane + 32 * j;
        if (el < cnt) {
          const double gv = gt[el];
          const double r = T[nU * TE + el];
#pragma unroll
          for (int q = 0; q < SPW; ++q) {
            const int s = warp + q * NW;
            if (s < nU) acc[q] += gv * (T[s * TE + el] - r);
          }
        }
      }
    }
    __syncthreads();  // stage fully consumed
    if (warp == 0) {
      const int64_t nt = tile + (int64_t)a.nstage * gridDim.x;
      if (nt < ntiles) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        issue(nt, st);
      }
    }
  }
  if (!a.do_gram) return;
  // fixed-order reductions -> part[block][s], part[block][nU] = self
  double* out = a.part + (int64_t)blockIdx.x * (nU + 1);
#pragma unroll
  for (int q = 0; q < SPW; ++q) {
    double v = acc[q];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int s = warp + q * NW;
    if (lane == 0 && s < nU) out[s] = v;
  }
  double v = acc_self;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __shared__ double wsum[NW];
  if (lane == 0) wsum[warp] = v;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int k = 0; k < NW; ++k) s += wsum[k];
    out[nU] = s;
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

}  // namespace

static int fill_smem_stages(int nU, size_t* bytes) {
  constexpr int TE = TE_FILL;
  const size_t stage = (size_t)(nU + 1) * TE * sizeof(double);
  const size_t fixed = (TE + 3 * TE) * sizeof(double) + 8 * sizeof(uint64_t);
  const size_t budget = 108 * 1024;  // two CTAs per SM
  int ns = (int)((budget - fixed) / stage);
  if (ns > 4) ns = 4;
  if (ns < 2) ns = std::max(1, (int)((220 * 1024 - fixed) / stage));  // very wide windows: one CTA per SM
  if (ns > 4) ns = 4;
  *bytes = ns * stage + fixed;
  return ns;
}

template <int SPW>
static hrom_status launch_fill_t(hrom_ctx* c, const FillArgs& a, size_t smem) {
  constexpr int TE = TE_FILL;
  HROM_CK(cudaFuncSetAttribute(fill_kernel<TE, SPW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  fill_kernel<TE, SPW><<<c->fill_blocks, 2 * TE, smem, c->st>>>(a);
  HROM_LAUNCH_CK();
  ++c->nlaunch;
  return HROM_OK;
}

hrom_status launch_fill(hrom_ctx* c, const Win& W, int mode, const double* src_S, double* out, int /*out_slot*/) {
  FillArgs a{};
  a.g = c->g;
  a.W = W;
  a.mode = mode;
  a.do_gram = (mode != MODE_PROJ) && out != nullptr && c->P.gram_mode == 0 ? 1 : 0;
  if (mode == MODE_FILL && out != nullptr && !(out >= c->b.ring && out < c->b.ring + (int64_t)c->nslots * c->g.Dp))
    a.do_gram = 0;  // standalone reconstruct into a caller buffer: no window Gram
  size_t smem;
  a.nstage = fill_smem_stages(W.nU, &smem);
  if (a.nstage < 1) return HROM_E_INVALID;
  a.ring = c->b.ring;
  a.rho = c->b.rho;
  a.cvec = (mode == MODE_PROJ) ? c->b.zvec : c->b.cvec;
  a.src_S = src_S;
  a.out = out;
  a.mS = c->b.masks + (int64_t)M_S * c->mwords;
  a.mB = (mode == MODE_FILL) ? c->b.masks + (int64_t)M_B * c->mwords : nullptr;
  a.eps_elem = c->b.eps_elem;
  a.part = c->b.gpart;
  constexpr int NW = 2 * TE_FILL / 32;
  const int spw = (W.nU + NW - 1) / NW;
  if (spw <= 3) return launch_fill_t<3>(c, a, smem);
  if (spw <= 6) return launch_fill_t<6>(c, a, smem);
  if (spw <= 9) return launch_fill_t<9>(c, a, smem);
  if (spw <= 17) return launch_fill_t<17>(c, a, smem);
  if (spw <= 33) return launch_fill_t<33>(c, a, smem);
  return HROM_E_INVALID;
}

hrom_status launch_gram_row(hrom_ctx* c, const Win& W, int new_slot) {
  return launch_fill(c, W, MODE_READ, nullptr, c->b.ring + (int64_t)new_slot * c->g.Dp, new_slot);
}

hrom_status reduce_gram_row(hrom_ctx* c, const Win& W, int new_slot, bool with_band) {
  const int nblk = c->fill_blocks + (with_band ? c->band_blocks : 0);
  gram_row_reduce<<<1, 256, 0, c->st>>>(c->b.gpart, nblk, W, new_slot, c->b.C, kMaxSlots);
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
