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

constexpr int NQ = 4;            // slot quarters: four warps cooperate on the same 32 DOFs
constexpr int NCW = NQ * TILE / 32;  // compute warps (16); thread 0 also issues the copies
constexpr int FILL_STAGES = 3;   // slab-tile stages in shared memory (at most; launch_fill_t)
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

// SQ: compile-time upper bound of the physical slots per quarter (ceil((w + 2) / 4)).
// Warp w owns DOF group grp = w / 4 (32 DOFs, one per lane) and slot quarter qq = w % 4
// (physical slots [qq SQ, qq SQ + SQ)): every shared-memory load of a warp reads 32 consecutive
// DOFs of one slot (conflict-free), and each lane holds SQ double-double Gram accumulators.
// The four quarters' partial window sums meet in shared memory behind a 128-thread named
// barrier per DOF group (double-buffered by tile parity).
template <int SQ, bool GRAM>
__global__ void __launch_bounds__(FILL_THREADS, 1) fill_kernel(FillArgs a) {
  if (a.run_if && *a.run_if == ~0ull) return;  // conditional re-run (positivity escalation)
  extern __shared__ __align__(128) unsigned char smraw[];
  const int nU = a.W.nU, w = a.W.w, nsl = a.nslots;
  const int64_t nsr = a.g.nsr;
  double* stage0 = reinterpret_cast<double*>(smraw);
  // a stage holds the nsr slab rows of a tile (one bulk copy) and zero rows up to NQ * SQ, so
  // every quarter walks SQ rows without bounds tests (cA = cX = 0 there; its Gram accumulators
  // for rows >= nslots are discarded)
  const int srows = (int)(nsr > NQ * SQ ? nsr : NQ * SQ);
  const size_t stage_elems = (size_t)srows * TILE;
  uint64_t* full = reinterpret_cast<uint64_t*>(stage0 + a.nstage * stage_elems);
  uint64_t* empty = full + a.nstage;
  // per PHYSICAL slot p: in-window flag (cA) and coefficient c (cX)
  __shared__ double cA[kMaxSlots + 2], cX[kMaxSlots + 2];
  // quarter partials [parity][group][quarter][lane]: window sum, c-weighted sum; quarter 0 also
  // publishes the DOF's side data (S-hat / band bits, HDM value)
  __shared__ double xsa[2][NCW / NQ][NQ][32], xtr[2][NCW / NQ][NQ][32], xside[2][NCW / NQ][32];
  __shared__ uint8_t xflag[2][NCW / NQ][32];
  __shared__ double wred[NCW][2 * SQ + 2];  // end-of-kernel row reduction (hi, lo per slot)
  __shared__ double s_bias;
  __shared__ int srel[FILL_STAGES];  // per stage: warps done with it
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = warp / NQ, qq = warp % NQ;
  const Geo& g = a.g;
  const int xoff = nU - w;  // logical: psi_cur and X use slots >= xoff; psi_prev uses slots < w
  for (int q = tid; q < kMaxSlots + 2; q += FILL_THREADS) cA[q] = cX[q] = 0.0;
  if (tid < FILL_STAGES) srel[tid] = 0;
  for (int st = 0; st < a.nstage; ++st)
    for (int i = (int)nsr * TILE + tid; i < srows * TILE; i += FILL_THREADS) stage0[st * stage_elems + i] = 0.0;
  __syncthreads();
  for (int s2 = tid; s2 < nU; s2 += FILL_THREADS) {
    const int q = a.W.slot[s2];
    cA[q] = 1.0;
    cX[q] = (s2 >= xoff && a.cvec) ? a.cvec[s2 - xoff] : 0.0;
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
    s_bias = gram_bias(mc);
  }
  __syncthreads();
  const int64_t ntiles = (g.D + TILE - 1) / TILE;
  const int64_t first = blockIdx.x;
  const uint32_t tile_bytes = (uint32_t)(nsr * TILE * sizeof(double));

  // producer role: thread 0 keeps FILL_STAGES slab tiles in flight, one bulk copy each
  auto issue = [&](int it2, int st) {  // st = it2 mod nstage (tracked by the caller)
    const int64_t tile = first + (int64_t)it2 * gridDim.x;
    if (tile >= ntiles) return;
    mbar_expect(&full[st], tile_bytes);
    bulk_g2s(stage0 + st * stage_elems, a.ring + tile * nsr * TILE, tile_bytes, &full[st]);
  };
  if (tid == 0)
    for (int q = 0; q < a.nstage; ++q) issue(q, q);

  // ---------------- compute warps: DOF el = grp*32 + lane, physical slots [q0, q0 + SQ)
  const int el = grp * 32 + lane;
  const int q0 = qq * SQ;
  const int p_first = a.W.slot[0], p_last = a.W.slot[nU - 1];
  // physical rows of this quarter that are not window slots: padding rows (zero, >= nsr), the
  // rho row (x = 0) and at most one dead snapshot slot (not in the union)
  // (nU = w + 1: one dead slot; nU = w at the bootstrap: two)
  int dead0 = -1, dead1 = -1;
  for (int q = q0; q < min(q0 + SQ, nsl); ++q)
    if (cA[q] == 0.0) {
      if (dead0 < 0) dead0 = q;
      else dead1 = q;
    }
  const int npad_q = max(0, min(q0 + SQ, srows) - max(q0, (int)nsr));
  double csum = 0.0;
  for (int q = 0; q < nsl; ++q) csum += cX[q];
  const double inv_w = 1.0 / (double)w;
  const int roff = a.rho_slot * TILE;
  const double bias = s_bias;
  double acc[SQ], accl[SQ];
#pragma unroll
  for (int i = 0; i < SQ; ++i) {
    acc[i] = bias;
    accl[i] = 0.0;
  }
  double acc_self = bias, acc_selfl = 0.0;
  // per-DOF side data, fetched one tile ahead and spread over the quarters so that no warp of a
  // group carries all of it: quarter 1 the S-hat / band mask bits, quarter 2 the HDM value (or
  // the new column); quarter 0 writes gamma_k, quarter 3 the squared error
  uint32_t wS = 0, wB = 0;
  int bitpos = 0;
  double pre = 0.0;
  // quarter 1's cell (n = e mod N, column i, row j) of the next fetched DOF, advanced by the grid
  // stride each tile without divisions (32-bit unsigned arithmetic: D < 2^31, hrom_create)
  unsigned fn = 0, fi = 0, fj = 0, sN = 0, sdi = 0, sdj = 0;
  if (qq == 1 && a.mode == MODE_FILL) {
    const unsigned e0 = (unsigned)(first * TILE + el), N = (unsigned)g.N, nx = (unsigned)g.nx;
    fn = e0 % N;
    fi = fn % nx;
    fj = fn / nx;
    sN = (unsigned)(((uint64_t)gridDim.x * TILE) % N);
    sdi = sN % nx;
    sdj = sN / nx;
  }
  auto fetch = [&](int64_t tile) {
    const int64_t e = tile * TILE + el;
    wS = wB = 0;
    pre = 0.0;
    if (qq == 1 && a.mode == MODE_FILL) {
      const unsigned i = fi, j = fj;
      // advance to the DOF of tile + gridDim.x: n += s mod N (rows carry, a wrap past N restarts them)
      fn += sN;
      fi += sdi;
      fj += sdj;
      if (fi >= (unsigned)g.nx) {
        fi -= (unsigned)g.nx;
        ++fj;
      }
      if (fn >= (unsigned)g.N) {
        fn -= (unsigned)g.N;
        fj -= (unsigned)g.ny;
      }
      if (tile >= ntiles || e >= g.D) return;
      const unsigned wi = j * (unsigned)g.wpr + (i >> 5);
      bitpos = (int)(i & 31);
      wS = a.mS[wi];
      if (a.mB) wB = a.mB[wi];
    } else if (qq == 2) {
      if (tile >= ntiles || e >= g.D || a.mode == MODE_PROJ) return;
      pre = a.mode == MODE_FILL ? a.src_S.p[sidx(a.src_S, e)]  // read unconditionally; used on S-hat only
                                : a.out.p[sidx(a.out, e)];
    }
  };
  fetch(first);
  int it = 0;
  int st = 0;            // stage of tile it (it mod nstage) and the parity of its use
  uint32_t sphase = 0;   // ((it / nstage) & 1), tracked without divisions
  for (int64_t tile = first; tile < ntiles; tile += gridDim.x, ++it) {
    const int par = it & 1;

    const int64_t e = tile * TILE + el;
    const bool valid = e < g.D;
    if (qq == 1) xflag[par][grp][lane] = (uint8_t)(((wS >> bitpos) & 1u) | (((wB >> bitpos) & 1u) << 1));
    if (qq == 2) xside[par][grp][lane] = pre;
    fetch(tile + gridDim.x);
    mbar_wait(&full[st], sphase);
    const double* T = stage0 + st * stage_elems + el;
    const double rh = T[roff];
    // pass 1 on this quarter's physical slots (x = gamma - rho; re-read in pass 2):
    //   sa = sum of the window slots, tr = sum_{s>=xoff} c_{s-xoff} x_s
    // four independent chains of each sum (fixed order: chain i & 3, then ((0 + 1) + (2 + 3)))
    // every row of the quarter enters sa; rows outside the window are removed after the loop:
    // rho's row contributes x = 0, each zero padding row -rho, the dead slot its own x
    double sa4[4] = {0.0, 0.0, 0.0, 0.0}, tr4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int i = 0; i < SQ; ++i) {
      const int q = q0 + i;
      const double xi = T[q * TILE] - rh;
      sa4[i & 3] += xi;
      tr4[i & 3] = fma(cX[q], xi, tr4[i & 3]);
    }
    double sq_ = (sa4[0] + sa4[1]) + (sa4[2] + sa4[3]);
    if (npad_q) sq_ += npad_q * rh;
    if (dead0 >= 0) sq_ -= T[dead0 * TILE] - rh;
    if (dead1 >= 0) sq_ -= T[dead1 * TILE] - rh;
    xsa[par][grp][qq][lane] = sq_;
    xtr[par][grp][qq][lane] = (tr4[0] + tr4[1]) + (tr4[2] + tr4[3]);
    double sa, tr;
    asm volatile("barrier.sync %0, %1;\n" ::"r"(1 + grp), "n"(32 * NQ) : "memory");  // thread 0 may lag (producer)
    // the four quarters in a fixed order: every warp of the group gets identical sums
    sa = ((xsa[par][grp][0][lane] + xsa[par][grp][1][lane]) + xsa[par][grp][2][lane]) + xsa[par][grp][3][lane];
    tr = ((xtr[par][grp][0][lane] + xtr[par][grp][1][lane]) + xtr[par][grp][2][lane]) + xtr[par][grp][3][lane];
    const uint8_t fl = xflag[par][grp][lane];
    const bool inS = fl & 1, inB = fl & 2;
    const double side = xside[par][grp][lane];
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
        if (qq == 3 && inS) {
          const double d = gval - rec;
          a.eps_elem[e] = d * d;
        }
        if (qq == 0) a.out.p[sidx(a.out, e)] = gval;
      } else if (a.mode == MODE_READ) {
        gval = side;
      } else if (qq == 3) {  // MODE_PROJ: residual of the projection (bootstrap indicator)
        a.eps_elem[e] = dev * dev;
      }
    }
    // pass 2: the new Gram row on this quarter's slots (band DOFs are added after the filter)
    if (GRAM && valid && !inB) {
      const double gr = gval - rh;
      if (qq == 0) biased_fma(acc_self, acc_selfl, gr, gr);
#pragma unroll
      for (int i = 0; i < SQ; ++i) biased_fma(acc[i], accl[i], gr, T[(q0 + i) * TILE] - rh);
    }
    // release the stage: the last warp to finish with it refills it with tile it + nstage (no
    // thread ever blocks waiting for the others)
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      if (atomicAdd(&srel[st], 1) == NCW - 1) {
        srel[st] = 0;
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        issue(it + a.nstage, st);
      }
    }
    if (++st == a.nstage) {
      st = 0;
      sphase ^= 1u;
    }
  }
  if constexpr (GRAM) {
    // fixed-order reductions: the 32 lanes (shuffle tree), then the DOF groups -> part[block][s]
#pragma unroll
    for (int i = 0; i < SQ; ++i) {
      double v = acc[i] - bias, vl = accl[i];  // exact (Sterbenz)
      for (int o = 16; o > 0; o >>= 1) {
        const double oh = __shfl_xor_sync(0xffffffffu, v, o), ol = __shfl_xor_sync(0xffffffffu, vl, o);
        dd_add(v, vl, oh, ol);
      }
      if (lane == 0) {
        wred[warp][2 * i] = v;
        wred[warp][2 * i + 1] = vl;
      }
    }
    {
      double v = acc_self - bias, vl = acc_selfl;
      for (int o = 16; o > 0; o >>= 1) {
        const double oh = __shfl_xor_sync(0xffffffffu, v, o), ol = __shfl_xor_sync(0xffffffffu, vl, o);
        dd_add(v, vl, oh, ol);
      }
      if (lane == 0) {
        wred[warp][2 * SQ] = v;  // meaningful in quarter-0 warps only
        wred[warp][2 * SQ + 1] = vl;
      }
    }
    __syncthreads();
    double* outp = a.part + (int64_t)blockIdx.x * (nU + 1) * 2;
    for (int s2 = tid; s2 <= nU; s2 += FILL_THREADS) {
      int qw, idx;  // quarter and accumulator index of the union slot s2
      if (s2 == nU) {
        qw = 0;
        idx = SQ;
      } else {
        const int q = a.W.slot[s2];
        qw = q / SQ;
        idx = q - qw * SQ;
      }
      double v = 0.0, vl = 0.0;
      for (int k = 0; k < NCW / NQ; ++k) dd_add(v, vl, wred[k * NQ + qw][2 * idx], wred[k * NQ + qw][2 * idx + 1]);
      outp[2 * s2] = v;
      outp[2 * s2 + 1] = vl;
    }
  }
}

// C[new][U[s]] = sum over blocks of fill partials, fixed order
// C row of the new slot = sum of the fill partials (+ the seam-band partials), 16 threads per
// entry with a fixed-order tree (deterministic)
// (double-double partials [blk][nU + 1][hi, lo]; row written to Chi / Clo)
// (one 256-thread block per 16 entries: the per-entry order does not depend on the grid)
__global__ void __launch_bounds__(256) gram_row_reduce(const double* __restrict__ part, int nblk,
                                                        const double* __restrict__ bpart, int nbblk, Win W,
                                                        int new_slot, double* __restrict__ C, double* __restrict__ Clo,
                                                        int ldc, const unsigned long long* __restrict__ esc) {
  const int nU = W.nU;
  if (esc && *esc != ~0ull) bpart = nullptr;  // escalated step: the row was recomputed from gamma_k
  constexpr int TPE = 16;
  {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x, s = idx / TPE, sub = idx % TPE;
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

// stages: as many slab tiles in flight as fit next to the kernel's static shared memory (3 at
// w = 64: the producer can run a tile ahead of the slowest warp)
template <int NU, bool GRAM>
hrom_status launch_fill_t(hrom_ctx* c, FillArgs a, size_t stage) {
  cudaFuncAttributes fa{};
  HROM_CK(cudaFuncGetAttributes(&fa, fill_kernel<NU, GRAM>));
  int dev = 0, optin = 0;
  HROM_CK(cudaGetDevice(&dev));
  HROM_CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const size_t avail = (size_t)optin - fa.sharedSizeBytes;
  a.nstage = FILL_STAGES;
  while (a.nstage > 1 && a.nstage * (stage + 16) > avail) --a.nstage;
  if (a.nstage * (stage + 16) > avail) return HROM_E_INVALID;
  const size_t smem = a.nstage * stage + 2 * a.nstage * sizeof(uint64_t);
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
  const int64_t sq_host = (c->nslots + NQ - 1) / NQ;  // stage rows padded to NQ * SQ (fill_kernel)

  a.rho_slot = c->nslots;
  a.nslots = c->nslots;
  a.ring = c->b.ring;
  a.cvec = (mode == MODE_PROJ) ? c->b.zvec : c->b.cvec;
  a.src_S = src_S;
  a.out = out;
  a.mS = c->b.masks + (int64_t)M_S * c->mwords;
  a.mB = (mode == MODE_FILL) ? (c->fill_mB_override ? c->fill_mB_override : c->b.masks + (int64_t)M_B * c->mwords)
                            : nullptr;
  a.eps_elem = c->b.eps_elem;
  a.part = c->b.gpart;
  a.C = c->b.C;
  a.ldc = kMaxSlots;
  const int sq = (c->nslots + NQ - 1) / NQ;
  (void)sq_host;
#define FILL_STAGE(SQ_) ((size_t)std::max<int64_t>(c->g.nsr, (int64_t)NQ * SQ_) * TILE * sizeof(double))
#define FILL_CASE(SQ_)                                                                            \
  if (sq <= SQ_)                                                                                  \
    return a.do_gram ? launch_fill_t<SQ_, true>(c, a, FILL_STAGE(SQ_)) : launch_fill_t<SQ_, false>(c, a, FILL_STAGE(SQ_));
  FILL_CASE(3) FILL_CASE(6) FILL_CASE(9) FILL_CASE(13) FILL_CASE(17)
#undef FILL_CASE
  if (!a.do_gram && sq <= 25) return launch_fill_t<25, false>(c, a, FILL_STAGE(25));
  if (!a.do_gram && sq <= 33) return launch_fill_t<33, false>(c, a, FILL_STAGE(33));
#undef FILL_STAGE
  return HROM_E_INVALID;  // wider windows use gram_mode = 1 (hrom_create enforces it)
}

hrom_status launch_gram_row(hrom_ctx* c, const Win& W, int new_slot, const unsigned long long* run_if) {
  return launch_fill(c, W, MODE_READ, plain(nullptr), c->slot_ref(new_slot), true, run_if);
}

hrom_status reduce_gram_row(hrom_ctx* c, const Win& W, int new_slot, bool with_band,
                            const unsigned long long* esc) {
  gram_row_reduce<<<((W.nU + 1) * 16 + 255) / 256, 256, 0, c->st>>>(c->b.gpart, c->fill_grid,
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
