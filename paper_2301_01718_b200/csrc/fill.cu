// fill.cu -- H6 + H9 + incremental H10: ONE pass over the snapshot window per hybrid step.
//
// For every DOF e the kernel streams the w+1 window columns gamma_{k-w-1..k-1} and the Gram
// shift rho once from HBM and
//   * fills gamma_k[e] = psi_k + Phi_k y_k = psi_cur + sum_i c_i (gamma_{x_i} - psi_prev)
//     (Alg. 1 line P:570; Phi_k = X^{(k-1)} A kept implicit), or takes the
//     partial-HDM value on S-hat (Eq. 6b),
//   * writes the per-DOF squared reconstruction error on S-hat,
//   * accumulates the new row of the shifted window Gram <gamma_k - rho, gamma_s - rho>
//     for every window slot s (reading A14) in double-double (G11), skipping seam-band cells
//     (added after the filter by the band GEMV).
// psi_prev / psi_cur are recomputed from the columns in registers: the
// reference state is never stored or drifted.
//
// Data path: the ring is in slab layout (internal.cuh), so a tile -- all w+3 slab slots of
// TILE DOFs -- is ONE contiguous run fetched by ONE cp.async.bulk (TMA) into a ring of
// shared-memory stages by a producer warp.  NCW compute warps each own 16 DOFs of the tile
// (one lane pair per DOF), run over the slots twice (sums -> gamma_k, then the Gram row into
// per-lane double-double accumulators) and release the stage through an mbarrier: no CTA-wide
// barrier in the stream.
#include <algorithm>
#include "internal.cuh"
#include "async.cuh"
#include "dd.cuh"

namespace hrom {
namespace {

constexpr int NCW = TILE / 16;  // warps (16 DOFs each: one lane pair per DOF); thread 0 also issues the copies
constexpr int FILL_STAGES = 2;  // slab-tile stages in shared memory
constexpr int FILL_THREADS = 32 * NCW;

enum { MODE_FILL = 0, MODE_READ = 1, MODE_PROJ = 2 };

struct FillArgs {
  Geo g;
  Win W;
  int mode;
  int do_gram;
  int nstage;
  int nslots;              // physical snapshot slots (w + 2)
  int rho_slot;            // slab slot of rho
  const double* ring;
  const double* cvec;      // w coefficients (c = A y, or projection z)
  SRef src_S;              // HDM values on S-hat (MODE_FILL)
  SRef out;                // gamma_k (MODE_FILL writes, MODE_READ reads)
  const uint32_t* mS;
  const uint32_t* mB;
  double* eps_elem;
  double* part;            // [grid][nU+1][hi, lo]
  const double* C;         // window Gram (hi) by ring slot: its diagonal sets the accumulator bias
  int ldc;
  const unsigned long long* run_if;  // nullable: run only if *run_if != ~0 (escalated step)
};

// (hi, lo) += a * b with hi biased far above every partial sum and product (|hi| >= |a b|):
// TwoProduct by FMA, then the exact Fast2Sum
__device__ __forceinline__ void biased_fma(double& hi, double& lo, double a, double b) {
  const double p = a * b;
  const double pe = fma(a, b, -p);
  const double s = hi + p;
  const double e = p - (s - hi);
  hi = s;
  lo += e + pe;
}

// SH: compile-time upper bound of the physical slots per half (ceil((w + 2) / 2)).
// A DOF is owned by a lane pair (l, l ^ 16) of a compute warp; each lane reads its half of the
// DOF's slot values from the staged tile and holds SH double-double Gram accumulators.
// GRAM: the instantiation accumulates the Gram row (do_gram); without it the double-double
// accumulators are compiled out (projection mode, wide windows).
template <int SH, bool GRAM>
__global__ void __launch_bounds__(FILL_THREADS, 1) fill_kernel(FillArgs a) {
  if (a.run_if && *a.run_if == ~0ull) return;  // conditional re-run (positivity escalation)
  extern __shared__ __align__(128) unsigned char smraw[];
  const int nU = a.W.nU, w = a.W.w, nsl = a.nslots;
  const int64_t nsr = a.g.nsr;
  double* stage0 = reinterpret_cast<double*>(smraw);
  const size_t stage_elems = (size_t)nsr * TILE;
  uint64_t* full = reinterpret_cast<uint64_t*>(stage0 + a.nstage * stage_elems);
  uint64_t* empty = full + a.nstage;
  // per PHYSICAL slot p: in-window flag (cA) and coefficient c (cX)
  __shared__ double cA[kMaxSlots + 2], cX[kMaxSlots + 2];
  __shared__ double wred[NCW][2 * SH + 1], wredl[NCW][2 * SH + 1];
  __shared__ double s_bias;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Geo& g = a.g;
  const int xoff = nU - w;  // logical: psi_cur and X use slots >= xoff; psi_prev uses slots < w
  for (int q = tid; q < kMaxSlots + 2; q += FILL_THREADS) cA[q] = cX[q] = 0.0;
  __syncthreads();
  for (int s = tid; s < nU; s += FILL_THREADS) {
    const int q = a.W.slot[s];
    cA[q] = 1.0;
    cX[q] = (s >= xoff && a.cvec) ? a.cvec[s - xoff] : 0.0;
  }
  if (tid == 0) {
    for (int q = 0; q < a.nstage; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    // Gram-row accumulator bias B = a power of two >= 256 max_s ||gamma_s - rho||^2 (the window
    // Gram's diagonal): every partial sum and product of the row then stays below B / 2, so
    // hi = B + S is updated by the exact Fast2Sum (3 operations instead of TwoSum's 6) and
    // (hi - B) + lo is the double-double row (G11).  A new snapshot 8x farther from rho than the
    // whole window would only degrade the row towards fp64 accuracy.
    double mc = 0.0;
    if (GRAM && a.C)
      for (int s2 = 0; s2 < nU; ++s2) mc = fmax(mc, a.C[a.W.slot[s2] * (a.ldc + 1)]);
    s_bias = mc > 0.0 ? ldexp(1.0, ilogb(256.0 * mc) + 1) : 1.0;
  }
  __syncthreads();
  const int64_t ntiles = (g.D + TILE - 1) / TILE;
  const int64_t first = blockIdx.x;
  const uint32_t tile_bytes = (uint32_t)(stage_elems * sizeof(double));

  // producer role: thread 0 keeps FILL_STAGES slab tiles in flight, one bulk copy each
  auto issue = [&](int it2) {
    const int64_t tile = first + (int64_t)it2 * gridDim.x;
    if (tile >= ntiles) return;
    const int st = it2 % a.nstage;
    mbar_expect(&full[st], tile_bytes);
    bulk_g2s(stage0 + st * stage_elems, a.ring + tile * stage_elems, tile_bytes, &full[st]);
  };
  if (tid == 0)
    for (int q = 0; q < a.nstage; ++q) issue(q);

  // ---------------- compute warps: DOF el = warp*16 + (lane & 15), slot half = lane >> 4
  const int half = lane >> 4;
  const int el = warp * 16 + (lane & 15);
  const int h0 = (nsl + 1) / 2;                  // physical slots [0, h0) | [h0, nsl)
  const int q0 = half ? h0 : 0, qn = half ? nsl : h0;
  const int p_first = a.W.slot[0], p_last = a.W.slot[nU - 1];
  double csum = 0.0;
  for (int q = 0; q < nsl; ++q) csum += cX[q];
  const double inv_w = 1.0 / (double)w;
  const int roff = a.rho_slot * TILE;
  // Gram-row accumulators in double-double (dd.cuh, G11), biased by B (see s_bias)
  const double bias = s_bias;
  double acc[SH], accl[SH];
#pragma unroll
  for (int i = 0; i < SH; ++i) {
    acc[i] = bias;
    accl[i] = 0.0;
  }
  double acc_self = bias, acc_selfl = 0.0;
  // per-DOF side data (mask words, HDM value / new column) is fetched one tile ahead
  uint32_t wS = 0, wB = 0;
  int bitpos = 0;
  double pre = 0.0;
  auto fetch = [&](int64_t tile) {
    const int64_t e = tile * TILE + el;
    wS = wB = 0;
    pre = 0.0;
    if (half == 0 && tile < ntiles && e < g.D && a.mode != MODE_PROJ) {
      const int64_t n = e % g.N;
      const int i = (int)(n % g.nx), j = (int)(n / g.nx);
      const int64_t wi = (int64_t)j * g.wpr + (i >> 5);
      bitpos = i & 31;
      if (a.mode == MODE_FILL) {
        wS = a.mS[wi];
        if (a.mB) wB = a.mB[wi];
        pre = a.src_S.p[sidx(a.src_S, e)];  // read unconditionally; used on S-hat only
      } else {
        pre = a.out.p[sidx(a.out, e)];
      }
    }
  };
  fetch(first);
  int it = 0;
  for (int64_t tile = first; tile < ntiles; tile += gridDim.x, ++it) {
    const int st = it % a.nstage;
    if (tid == 0 && it >= 1) {
      // the stage of tile it-1 is free once every warp released it: refill it with tile it-1+stages
      const int pst = (it - 1) % a.nstage;
      mbar_wait(&empty[pst], (uint32_t)(((it - 1) / a.nstage) & 1));
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      issue(it - 1 + a.nstage);
    }
    const int64_t e = tile * TILE + el;
    const bool valid = e < g.D;
    const bool inS = __shfl_sync(0xffffffffu, (wS >> bitpos) & 1u, lane & 15);
    const bool inB = __shfl_sync(0xffffffffu, (wB >> bitpos) & 1u, lane & 15);
    const double side = __shfl_sync(0xffffffffu, pre, lane & 15);
    fetch(tile + gridDim.x);
    mbar_wait(&full[st], (uint32_t)((it / a.nstage) & 1));
    const double* T = stage0 + st * stage_elems + el;
    const double rh = T[roff];
    // pass 1 on this lane's physical slots (x = gamma - rho, re-read from shared memory in
    // pass 2: the registers hold the double-double row accumulators):
    //   sa = sum of the window slots, tr = sum_{s>=xoff} c_{s-xoff} x_s
    double sa = 0.0, tr = 0.0, sa2 = 0.0, tr2 = 0.0;
#pragma unroll
    for (int i = 0; i < SH; ++i) {
      const int q = q0 + i;
      if (q < qn) {
        const double xi = T[q * TILE] - rh;
        if (i & 1) {
          sa2 = fma(cA[q], xi, sa2);
          tr2 = fma(cX[q], xi, tr2);
        } else {
          sa = fma(cA[q], xi, sa);
          tr = fma(cX[q], xi, tr);
        }
      }
    }
    sa += sa2;
    tr += tr2;
    // combine the two halves (a + b == b + a: both lanes of the pair get identical sums)
    sa += __shfl_xor_sync(0xffffffffu, sa, 16);
    tr += __shfl_xor_sync(0xffffffffu, tr, 16);
    // psi_prev and psi_cur differ from the window sum by one end slot each (when nU = w + 1)
    double sp = sa, sc = sa;
    if (xoff == 1) {
      sp -= T[p_last * TILE] - rh;
      sc -= T[p_first * TILE] - rh;
    }
    double gval = 0.0;
    if (valid) {
      // psi_prev - rho = sp/w, psi_cur - rho = sc/w;  Phi y = sum_i c_i (x_i - (psi_prev - rho))
      const double dev = tr - (sp * inv_w) * csum;
      if (a.mode == MODE_FILL) {
        const double rec = (rh + sc * inv_w) + dev;
        gval = inS ? side : rec;
        if (half == 0) {
          if (inS) {
            const double d = gval - rec;
            a.eps_elem[e] = d * d;
          }
          a.out.p[sidx(a.out, e)] = gval;
        }
      } else if (a.mode == MODE_READ) {
        gval = side;
      } else if (half == 0) {  // MODE_PROJ: residual of the projection (bootstrap indicator)
        a.eps_elem[e] = dev * dev;
      }
    }
    // pass 2: new Gram row on this lane's physical slots (band DOFs are added after the filter)
    if (GRAM && valid && !inB) {
      const double gr = gval - rh;
      if (half == 0) biased_fma(acc_self, acc_selfl, gr, gr);
      // h0 slots per half (uniform): for an odd slot count the last of half 1 is rho's slot,
      // accumulated and discarded
#pragma unroll
      for (int i = 0; i < SH; ++i)
        if (i < h0) biased_fma(acc[i], accl[i], gr, T[(q0 + i) * TILE] - rh);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
  if constexpr (GRAM) {
  // fixed-order reductions: the 16 lanes of each half (shuffle tree), then warps -> part[block][s]
#pragma unroll
  for (int i = 0; i < SH; ++i) {
    double v = acc[i] - bias, vl = accl[i];  // exact (Sterbenz)
    for (int o = 8; o > 0; o >>= 1) {
      const double oh = __shfl_xor_sync(0xffffffffu, v, o), ol = __shfl_xor_sync(0xffffffffu, vl, o);
      dd_add(v, vl, oh, ol);
    }
    if ((lane & 15) == 0) {
      wred[warp][half * SH + i] = v;
      wredl[warp][half * SH + i] = vl;
    }
  }
  {
    double v = acc_self - bias, vl = acc_selfl;
    for (int o = 16; o > 0; o >>= 1) {
      const double oh = __shfl_xor_sync(0xffffffffu, v, o), ol = __shfl_xor_sync(0xffffffffu, vl, o);
      dd_add(v, vl, oh, ol);
    }
    if (lane == 0) {
      wred[warp][2 * SH] = v;
      wredl[warp][2 * SH] = vl;
    }
  }
  __syncthreads();
  double* outp = a.part + (int64_t)blockIdx.x * (nU + 1) * 2;
  for (int s = tid; s <= nU; s += 32 * NCW) {
    int idx;
    if (s == nU) {
      idx = 2 * SH;
    } else {
      const int q = a.W.slot[s];
      idx = (q < h0) ? q : SH + (q - h0);
    }
    double v = 0.0, vl = 0.0;
    for (int k = 0; k < NCW; ++k) dd_add(v, vl, wred[k][idx], wredl[k][idx]);
    outp[2 * s] = v;
    outp[2 * s + 1] = vl;
  }
  }
}

// C[new][U[s]] = sum over blocks of fill partials, fixed order
// C row of the new slot = sum of the fill partials (+ the seam-band partials), 16 threads per
// entry with a fixed-order tree (deterministic)
// (double-double partials [blk][nU + 1][hi, lo]; row written to Chi / Clo)
__global__ void __launch_bounds__(1024) gram_row_reduce(const double* __restrict__ part, int nblk,
                                                        const double* __restrict__ bpart, int nbblk, Win W,
                                                        int new_slot, double* __restrict__ C, double* __restrict__ Clo,
                                                        int ldc, const unsigned long long* __restrict__ esc) {
  const int nU = W.nU;
  if (esc && *esc != ~0ull) bpart = nullptr;  // escalated step: the row was recomputed from gamma_k
  constexpr int TPE = 16;
  for (int base = 0; base < (nU + 1) * TPE; base += blockDim.x) {
    const int idx = base + threadIdx.x, s = idx / TPE, sub = idx % TPE;
    double a = 0.0, al = 0.0, bsum = 0.0, bl = 0.0;
    if (s <= nU) {
      for (int b = sub; b < nblk; b += TPE) {
        const double* p = part + ((int64_t)b * (nU + 1) + s) * 2;
        dd_add(a, al, p[0], p[1]);
      }
      if (bpart)
        for (int b = sub; b < nbblk; b += TPE) {
          const double* p = bpart + ((int64_t)b * (nU + 1) + s) * 2;
          dd_add(bsum, bl, p[0], p[1]);
        }
    }
    for (int o = TPE / 2; o > 0; o >>= 1) {
      double oh = __shfl_xor_sync(0xffffffffu, a, o), ol = __shfl_xor_sync(0xffffffffu, al, o);
      dd_add(a, al, oh, ol);
      oh = __shfl_xor_sync(0xffffffffu, bsum, o);
      ol = __shfl_xor_sync(0xffffffffu, bl, o);
      dd_add(bsum, bl, oh, ol);
    }
    if (s <= nU && sub == 0) {
      dd_add(a, al, bsum, bl);
      const int cs_ = (s < nU) ? W.slot[s] : new_slot;
      C[new_slot * ldc + cs_] = a;
      C[cs_ * ldc + new_slot] = a;
      Clo[new_slot * ldc + cs_] = al;
      Clo[cs_ * ldc + new_slot] = al;
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

// out (rho or psi) = mean of the last w window slots

template <int NU, bool GRAM>
hrom_status launch_fill_t(hrom_ctx* c, const FillArgs& a, size_t smem) {
  HROM_CK(cudaFuncSetAttribute(fill_kernel<NU, GRAM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  fill_kernel<NU, GRAM><<<c->nsm, FILL_THREADS, smem, c->st>>>(a);
  HROM_LAUNCH_CK();
  ++c->nlaunch;
  c->fill_grid = c->nsm;
  return HROM_OK;
}

}  // namespace

int fill_max_gram_slots() { return 68; }

hrom_status launch_fill(hrom_ctx* c, const Win& W, int mode, SRef src_S, SRef out, bool out_in_ring,
                        const unsigned long long* run_if) {
  FillArgs a{};
  a.run_if = run_if;
  a.g = c->g;
  a.W = W;
  a.mode = mode;
  a.do_gram = (mode != MODE_PROJ) && out_in_ring && c->P.gram_mode == 0 ? 1 : 0;
  const size_t stage = (size_t)c->g.nsr * TILE * sizeof(double);
  a.nstage = FILL_STAGES;
  while (a.nstage > 1 && a.nstage * stage > 216 * 1024) --a.nstage;  // wide windows (w = 128): one stage
  if (a.nstage * stage > 216 * 1024) return HROM_E_INVALID;
  const size_t smem = a.nstage * stage + 2 * a.nstage * sizeof(uint64_t);
  a.rho_slot = c->nslots;
  a.nslots = c->nslots;
  a.ring = c->b.ring;
  a.cvec = (mode == MODE_PROJ) ? c->b.zvec : c->b.cvec;
  a.src_S = src_S;
  a.out = out;
  a.mS = c->b.masks + (int64_t)M_S * c->mwords;
  a.mB = (mode == MODE_FILL) ? c->b.masks + (int64_t)M_B * c->mwords : nullptr;
  a.eps_elem = c->b.eps_elem;
  a.part = c->b.gpart;
  a.C = c->b.C;
  a.ldc = kMaxSlots;
  const int sh = (c->nslots + 1) / 2;
#define FILL_CASE(SH_)                                                                            \
  if (sh <= SH_) return a.do_gram ? launch_fill_t<SH_, true>(c, a, smem) : launch_fill_t<SH_, false>(c, a, smem);
  FILL_CASE(6) FILL_CASE(12) FILL_CASE(18) FILL_CASE(26) FILL_CASE(34)
#undef FILL_CASE
  if (!a.do_gram && sh <= 50) return launch_fill_t<50, false>(c, a, smem);
  if (!a.do_gram && sh <= 66) return launch_fill_t<66, false>(c, a, smem);
  return HROM_E_INVALID;  // wider windows use gram_mode = 1 (hrom_create enforces it)
}

hrom_status launch_gram_row(hrom_ctx* c, const Win& W, int new_slot, const unsigned long long* run_if) {
  return launch_fill(c, W, MODE_READ, plain(nullptr), c->slot_ref(new_slot), true, run_if);
}

hrom_status reduce_gram_row(hrom_ctx* c, const Win& W, int new_slot, bool with_band,
                            const unsigned long long* esc) {
  gram_row_reduce<<<1, 1024, 0, c->st>>>(c->b.gpart, c->fill_grid,
                                         with_band ? c->b.gpart + (int64_t)c->fill_blocks * (W.nU + 1) * 2 : nullptr,
                                         c->band_blocks, W, new_slot, c->b.C, c->b.Clo, kMaxSlots, esc);
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


}  // namespace hrom
