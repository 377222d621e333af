// slab.cu -- row-slab sharding of ONE problem across ranks.
//
// The HDM residual is local (Eq. partial_hdm2): a cell's RK3 update reads a
// cross stencil of radius h per stage, so a rank that owns `rows_own` consecutive grid rows and
// keeps H = max(3 h, 2 h + W) halo rows of its neighbours on each side can run the whole masked
// RK3 (H3), the set dilations (H8) and the fill (H6) of its rows without talking to anyone; what
// the ranks must agree on are a handful of small reductions.  A slab context is an ordinary
// hrom_ctx over the local rows [halo | own | halo] whose y ends are open (Geo::bcy = 0; garbage
// from the open ends stays inside the halo, which is overwritten by the next exchange), plus the
// state below.  One step of Algorithm 1 is cut into phases at the exchanges:
//
//   S   max wave speed (H1)                          all-reduce MAX of one word (first step only;
//                                                     later steps carry it in the END message)
//   R   gathered Gram of the own S-hat rows (H4)     all-reduce SUM of (w+2)^2 double-doubles
//   F0  halo rows of the pre-filter gamma_k (H6)       neighbour rows (only when the seam filter is on)
//   Fs  per filter sweep (H7): band values of the edge
//       rows + the sweep's statistics                 neighbour rows + all-reduce MAX / SUM, host decision
//   END halo rows of gamma_k (H3/H6), new window-Gram
//       row (H10), max wave speed, positivity flag   neighbour rows + all-reduce SUM / MAX / MIN
//   B   bootstrap window Gram (k = w-1, H10)         all-reduce SUM of (w+1)^2 double-doubles
//   H0..H5  radix-select histograms (H8)             all-reduce SUM of 2048 counts per pass
//   M   S-hat halo rows (H8)                         neighbour rows
//
// and everything else (dt, masked RK3, solve, fill, eigen-solve, set construction) is local or
// replicated: the eigen-solve and the gappy solve run on every rank on bitwise identical inputs,
// so every rank holds the same basis coefficients and y ("H11 replicated").
//
// Transport is not this file's business: hrom_slab_step() runs the local work of one phase and
// leaves ONE message in a caller-provided device buffer; the caller all-gathers the nranks
// messages in rank order (NCCL all_gather over NVLink, or plain copies between contexts of one
// process) and hands the gathered buffer to the next call, which does every reduction itself in
// rank order (double-double sums with TwoSum: fixed order, so all ranks get identical bits).
// Reductions never include halo rows: S-hat and band sums run on own-row sub-lists, and the
// fused window-Gram row of the fill pass skips halo cells through its band mask.
//
// The seam filter (H7, readings A21-A24, A23') runs sweep by sweep: the x-pass on every
// local band cell (halo rows included: it reads its own row only), the y-pass and the residual gate
// on the own band cells, then the edge rows and the sweep's statistics travel; the stop decision
// (empty keep-set, relative decrease below eps_f, j_max sweeps) is taken on the host from the
// gathered statistics, the same on every rank.  Same arithmetic as filter.cu on the dense field.
//
// Positivity escalation: the ranks' flags travel in the END message; when any rank holds a
// non-physical hybrid state, EVERY rank redoes the step as a full step from gamma_{k-1} with the
// same dt (host decision on the gathered flags), takes the new window-Gram row over all its own
// cells, and a second END exchange follows.
//
// Not supported on a slab (hrom_slab_create refuses): ODEIM points, RRE-delta, finite z, the
// whole-domain filter (W = -1).
#include <algorithm>
#include <cmath>
#include <cstring>
#include "internal.cuh"
#include "dd.cuh"

struct hrom_slab {
  int rank = 0, nranks = 1;
  int ny_g = 0, row0 = 0, own = 0, hlo = 0, hhi = 0, H = 0;
  int bc_g = 0;
  int64_t N_g = 0;
  int phase = 0;
  int sel_pass = 0;
  bool step_hybrid = false;
  int f_order = 0, f_sw = 0;  // seam filter: cascade order and sweep in flight
  int f_sweeps[3] = {0, 0, 0};
  int64_t escalations = 0;  // hybrid steps redone as full steps
  unsigned long long* fstat = nullptr;  // [0] max relative decrease (bits) [1] kept count of the sweep
  // message geometry (bytes)
  int64_t halo_doubles = 0;  // c * H * nx: one edge block of the state
  int64_t mask_words = 0;    // H * wpr: one edge block of a bitmap
  int64_t max_msg = 0;
  // device
  int32_t* listS = nullptr;  // own rows of S-hat (sub-list of L_S)
  int32_t* listB = nullptr;  // own rows of the band
  int32_t* listA = nullptr;  // every own cell
  int32_t* listAdd = nullptr;  // own rows of the cells entering / leaving S-hat at the last sampling (G7)
  int32_t* listRem = nullptr;
  int32_t* cnt = nullptr;    // [0] |listS| [1] |listB| [2] |listA| [3] |listAdd| [4] |listRem|
  bool have_prev = false;    // M_SPREV holds the S-hat of the previous sampling
  uint32_t* mBH = nullptr;   // band u halo rows: cells left out of the fused Gram row
  unsigned long long* sel = nullptr;  // [0] prefix [1] remaining [2] tau [3] quota [4] my ties [5] all-positive flag [6] scratch smax
  int32_t* hist = nullptr;   // 2048
  double* stage = nullptr;   // plain staging vector (Dp)
};

namespace hrom {
namespace {

constexpr int RADIX = 11, NBIN = 1 << RADIX;
constexpr int ROW_SLOTS = kMaxW + 2;  // fixed length of the Gram-row part of an END message

enum Phase { PH_IDLE = 0, PH_SMAX, PH_R, PH_HALO1, PH_FSWEEP, PH_END, PH_END2, PH_BOOT, PH_REBUILD, PH_SEL, PH_MASK };

__host__ __device__ inline int sel_shift(int p) { return p < 5 ? 53 - RADIX * p : 0; }

// rows [row_first, row_first + nrows) of every variable of src -> dst[(v * nrows + jr) * nx + i]
__global__ void pack_rows_kernel(Geo g, SRef src, int row_first, int nrows, double* __restrict__ dst) {
  const int64_t per = (int64_t)nrows * g.nx, total = per * g.c;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int v = (int)(t / per);
    const int64_t q = t - v * per;
    dst[t] = src.p[sidx(src, v * g.N + (int64_t)row_first * g.nx + q)];
  }
}
__global__ void unpack_rows_kernel(Geo g, SRef dst, int row_first, int nrows, const double* __restrict__ src) {
  const int64_t per = (int64_t)nrows * g.nx, total = per * g.c;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int v = (int)(t / per);
    const int64_t q = t - v * per;
    dst.p[sidx(dst, v * g.N + (int64_t)row_first * g.nx + q)] = src[t];
  }
}

// all-reduce MAX of the wave-speed words and MIN of the positivity flags of the gathered
// messages (order-free, exact); sets up the registers launch_dt's fused path reads
__global__ void smax_reduce_kernel(const unsigned char* __restrict__ gath, int64_t stride, int64_t off, int P,
                                   unsigned long long* __restrict__ ureg, int latch_bad) {
  unsigned long long m = 0ull, bad = ~0ull;
  for (int r = 0; r < P; ++r) {
    const unsigned long long* p = reinterpret_cast<const unsigned long long*>(gath + r * stride + off);
    m = p[0] > m ? p[0] : m;
    bad = p[1] < bad ? p[1] : bad;
  }
  ureg[0] = m;
  ureg[2] = m;
  ureg[3] = ~0ull;
  // a slab does not escalate: a non-physical hybrid state on any rank is latched on all of them
  if (latch_bad && bad != ~0ull && ureg[1] == ~0ull) ureg[1] = bad;
}

// double-double all-reduce SUM in rank order: message part = hi[n] then lo[n]
// (il = 1: pairs interleaved [i][hi, lo] on both sides, hi / lo = the arrays' first hi / lo element)
__global__ void dd_sum_kernel(const unsigned char* __restrict__ gath, int64_t stride, int64_t off, int P, int n, int il,
                              double* hi, double* lo) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double h = 0.0, l = 0.0;
    for (int r = 0; r < P; ++r) {
      const double* p = reinterpret_cast<const double*>(gath + r * stride + off);
      if (il) dd_add(h, l, p[2 * i], p[2 * i + 1]);
      else dd_add(h, l, p[i], p[n + i]);
    }
    hi[il ? 2 * i : i] = h;
    lo[il ? 2 * i : i] = l;
  }
}

// bootstrap: the summed gathered Gram R (union order, ncol x ncol) -> window Gram C by ring slot
__global__ void scatter_gram_kernel(const double* __restrict__ Rh, const double* __restrict__ Rl, int ncol, Win W,
                                    double* __restrict__ C, double* __restrict__ Clo, int ldc) {
  const int nU = W.nU;
  for (int t = threadIdx.x; t < nU * nU; t += blockDim.x) {
    const int i = t / nU, j = t - i * nU;
    C[W.slot[i] * ldc + W.slot[j]] = Rh[i * ncol + j];
    Clo[W.slot[i] * ldc + W.slot[j]] = Rl[i * ncol + j];
  }
}

// local part of the new window-Gram row: fill partials + band partials in the same fixed order
// as gram_row_reduce (fill.cu), written to the message (hi[ROW_SLOTS], lo[ROW_SLOTS]) instead of C
__global__ void __launch_bounds__(256) slab_row_reduce(const double* __restrict__ part, int nblk,
                                                        const double* __restrict__ bpart, int nbblk, int nU,
                                                        double* __restrict__ out) {
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
      out[s] = a;
      out[ROW_SLOTS + s] = al;
    }
  }
  if (blockIdx.x == 0)
    for (int s = nU + 1 + threadIdx.x; s < ROW_SLOTS; s += blockDim.x) out[s] = out[ROW_SLOTS + s] = 0.0;
}

// C row / column of the new slot = sum over ranks (rank order) of the row parts
__global__ void slab_row_apply(const unsigned char* __restrict__ gath, int64_t stride, int64_t off, int P, Win W,
                               int new_slot, double* __restrict__ C, double* __restrict__ Clo, int ldc) {
  const int s = threadIdx.x;
  if (s > W.nU) return;
  double h = 0.0, l = 0.0;
  for (int r = 0; r < P; ++r) {
    const double* p = reinterpret_cast<const double*>(gath + r * stride + off);
    dd_add(h, l, p[s], p[ROW_SLOTS + s]);
  }
  const int cs = s < W.nU ? W.slot[s] : new_slot;
  C[new_slot * ldc + cs] = h;
  C[cs * ldc + new_slot] = h;
  Clo[new_slot * ldc + cs] = l;
  Clo[cs * ldc + new_slot] = l;
}

// own-row sub-list of an ascending cell list: cells in [lo_cell, hi_cell)
__global__ void own_list_kernel(const int32_t* __restrict__ src, const int32_t* __restrict__ count, int lo_cell,
                                int hi_cell, int32_t* __restrict__ dst, int32_t* __restrict__ dst_count) {
  __shared__ int s_lo, s_hi;
  const int n = *count;
  if (threadIdx.x == 0) {
    int a = 0, b = n;  // lower bound of lo_cell
    while (a < b) {
      const int m = (a + b) >> 1;
      if (src[m] < lo_cell) a = m + 1;
      else b = m;
    }
    s_lo = a;
    b = n;  // lower bound of hi_cell
    while (a < b) {
      const int m = (a + b) >> 1;
      if (src[m] < hi_cell) a = m + 1;
      else b = m;
    }
    s_hi = a;
  }
  __syncthreads();
  const int lo = s_lo, hi = s_hi;
  for (int t = lo + blockIdx.x * blockDim.x + threadIdx.x; t < hi; t += gridDim.x * blockDim.x) dst[t - lo] = src[t];
  if (blockIdx.x == 0 && threadIdx.x == 0) *dst_count = hi - lo;
}

__global__ void iota_kernel(int32_t* __restrict__ dst, int first, int n, int32_t* __restrict__ cnt) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) dst[t] = first + t;
  if (blockIdx.x == 0 && threadIdx.x == 0) *cnt = n;
}

// mBH = band bits on own rows, every bit on halo rows
__global__ void halo_mask_kernel(const uint32_t* __restrict__ mB, uint32_t* __restrict__ mBH, int wpr, int ny,
                                 int row_lo, int row_hi) {
  const int64_t nw = (int64_t)ny * wpr;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nw; w += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(w / wpr);
    mBH[w] = (j >= row_lo && j < row_hi) ? mB[w] : 0xffffffffu;
  }
}

// ---- distributed top-n_g selection (A18): radix select over the IEEE patterns of eps > 0 ----
// pass p: counts of digit (bits >> shift) among own cells whose higher digits equal the prefix
__global__ void __launch_bounds__(1024) sel_hist_kernel(const double* __restrict__ eps, int lo_cell, int hi_cell,
                                                        int pass, const unsigned long long* __restrict__ sel,
                                                        int32_t* __restrict__ hist) {
  __shared__ int sh[NBIN];
  for (int i = threadIdx.x; i < NBIN; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  const int shift = sel_shift(pass);
  const int width = shift == 0 ? 9 : RADIX;
  const unsigned long long hm = pass == 0 ? 0ull : (~0ull << (shift + width));
  const unsigned long long prefix = pass == 0 ? 0ull : sel[0];  // sel[0] still holds the previous selection's prefix
  const bool skip = pass > 0 && sel[5] != 0ull;  // every positive cell is selected: nothing to count
  int run_bin = -1, run = 0;  // run-length cache: neighbouring cells mostly share a digit
  if (!skip)
    for (int n = lo_cell + blockIdx.x * blockDim.x + threadIdx.x; n < hi_cell; n += gridDim.x * blockDim.x) {
      const unsigned long long bb = (unsigned long long)__double_as_longlong(eps[n]);
      if (bb == 0ull || (bb & hm) != prefix) continue;
      const int bin = (int)((bb >> shift) & (NBIN - 1));
      if (bin == run_bin) {
        ++run;
      } else {
        if (run) atomicAdd(&sh[run_bin], run);
        run_bin = bin;
        run = 1;
      }
    }
  if (run) atomicAdd(&sh[run_bin], run);
  __syncthreads();
  for (int i = threadIdx.x; i < NBIN; i += blockDim.x)
    if (sh[i]) atomicAdd(hist + i, sh[i]);  // integer counts: order-free
}

// every rank, identical: the highest digit d with #(> d) < rem <= #(>= d) over the summed
// histograms; after the last pass the tie quota of this rank (ties by ascending cell = by rank,
// then by cell inside the rank)
__global__ void __launch_bounds__(1024) sel_digit_kernel(const unsigned char* __restrict__ gath, int64_t stride, int P,
                                                         int rank, int pass, long long n_g,
                                                         unsigned long long* __restrict__ sel) {
  __shared__ long long tot[NBIN];
  for (int b = threadIdx.x; b < NBIN; b += blockDim.x) {
    long long t = 0;
    for (int r = 0; r < P; ++r) t += reinterpret_cast<const int32_t*>(gath + r * stride)[b];
    tot[b] = t;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (pass == 0) {
      long long t = 0;
      for (int b = 0; b < NBIN; ++b) t += tot[b];
      sel[0] = 0ull;
      sel[1] = (unsigned long long)n_g;
      sel[5] = n_g >= t ? 1ull : 0ull;  // fewer positive cells than n_g: all of them (no zeros, masks.cu A1)
      sel[2] = 0ull;
      sel[3] = sel[4] = 0ull;
    }
    if (sel[5] == 0ull) {
      const long long rem = (long long)sel[1];
      long long above = 0;
      int digit = 0;
      for (int b = NBIN - 1; b >= 0; --b) {
        if (above < rem && above + tot[b] >= rem) {
          digit = b;
          break;
        }
        above += tot[b];
      }
      const int shift = sel_shift(pass);
      sel[0] |= (unsigned long long)digit << shift;
      sel[1] = (unsigned long long)(rem - above);
      if (pass == 5) {
        long long before = 0;
        for (int r = 0; r < rank; ++r) before += reinterpret_cast<const int32_t*>(gath + r * stride)[digit];
        const long long mine = reinterpret_cast<const int32_t*>(gath + rank * stride)[digit];
        long long quota = (rem - above) - before;
        quota = quota < 0 ? 0 : (quota > mine ? mine : quota);
        sel[2] = sel[0];
        sel[3] = (unsigned long long)quota;
        sel[4] = (unsigned long long)mine;
      }
    }
  }
}

// S-hat bits of the own rows: eps > tau, and the first `quota` ties (eps == tau) of this rank by
// ascending cell.  quota == my ties (or 0) needs no order; otherwise one block walks the rows
__global__ void sel_mark_kernel(Geo g, const double* __restrict__ eps, int row_lo, int row_hi,
                                const unsigned long long* __restrict__ sel, uint32_t* __restrict__ S) {
  const unsigned long long tau = sel[2], quota = sel[3], mine = sel[4];
  const bool all = sel[5] != 0ull;
  const bool ties_all = quota == mine;
  const int64_t nw = (int64_t)(row_hi - row_lo) * g.wpr;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nw; t += (int64_t)gridDim.x * blockDim.x) {
    const int j = row_lo + (int)(t / g.wpr), wi = (int)(t % g.wpr);
    uint32_t bits = 0u;
    for (int b = 0; b < 32; ++b) {
      const int i = 32 * wi + b;
      if (i >= g.nx) break;
      const unsigned long long bb = (unsigned long long)__double_as_longlong(eps[(int64_t)j * g.nx + i]);
      const bool s = all ? bb != 0ull : (bb > tau || (bb == tau && ties_all));
      bits |= (uint32_t)s << b;
    }
    S[(int64_t)j * g.wpr + wi] = bits;
  }
}
__global__ void __launch_bounds__(1024) sel_ties_kernel(Geo g, const double* __restrict__ eps, int row_lo, int row_hi,
                                                        const unsigned long long* __restrict__ sel,
                                                        uint32_t* __restrict__ S) {
  const unsigned long long tau = sel[2], quota = sel[3], mine = sel[4];
  if (sel[5] != 0ull || quota == mine || quota == 0ull) return;
  __shared__ int sc[1024];
  __shared__ int s_base;
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  const int lo = row_lo * g.nx, hi = row_hi * g.nx;
  for (int base = lo; base < hi; base += 1024) {
    const int n = base + threadIdx.x;
    const bool tie = n < hi && (unsigned long long)__double_as_longlong(eps[n]) == tau;
    sc[threadIdx.x] = tie;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {  // inclusive scan
      const int v = threadIdx.x >= o ? sc[threadIdx.x - o] : 0;
      __syncthreads();
      sc[threadIdx.x] += v;
      __syncthreads();
    }
    const int rank_in = s_base + sc[threadIdx.x] - (tie ? 1 : 0);
    if (tie && (unsigned long long)rank_in < quota) {
      const int j = n / g.nx, i = n - j * g.nx;
      atomicOr(&S[(int64_t)j * g.wpr + (i >> 5)], 1u << (i & 31));
    }
    __syncthreads();
    if (threadIdx.x == 1023) s_base += sc[1023];
    __syncthreads();
    if ((unsigned long long)s_base >= quota) break;  // uniform
  }
}

// ---- seam filter on the dense field (same stencils, order of operations and gate as filter.cu) ----
__constant__ double fc2[3] = {1, 2, 1};
__constant__ double fc4[5] = {-1, 4, 10, 4, -1};
__constant__ double fc6[7] = {1, -6, 15, 44, 15, -6, 1};
__device__ __forceinline__ int fshapiro(int order, const double** c, double* den) {
  if (order == 2) { *c = fc2; *den = 4.0; return 1; }
  if (order == 4) { *c = fc4; *den = 16.0; return 2; }
  *c = fc6; *den = 64.0; return 3;
}
__device__ __forceinline__ int fwrap(int i, int n, int bc) {  // periodic wrap, else zeroth-order end
  if (bc == 1) {
    i %= n;
    return i < 0 ? i + n : i;
  }
  return i < 0 ? 0 : (i >= n ? n - 1 : i);
}
// pre-filter values of the own band cells (the indicator on kept cells needs them), flags cleared
__global__ void filt_init_kernel(Geo g, SRef v, const int32_t* __restrict__ list, const int32_t* __restrict__ count,
                                 double* __restrict__ v0, uint8_t* __restrict__ flag) {
  const int nb = *count;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nb; t += gridDim.x * blockDim.x) {
    const int64_t n = list[t];
    for (int var = 0; var < g.c; ++var) v0[var * g.N + n] = v.p[sidx(v, var * g.N + n)];
    flag[n] = 0;
  }
}
// P1: v' = S^x(v) on every local band cell
__global__ void filt_x_kernel(Geo g, SRef v, const int32_t* __restrict__ list, const int32_t* __restrict__ count,
                              int order, double* __restrict__ Vp) {
  const double* cf;
  double den;
  const int rad = fshapiro(order, &cf, &den);
  double cfr[7];
#pragma unroll
  for (int m = 0; m < 7; ++m) cfr[m] = m <= 2 * rad ? cf[m] : 0.0;
  const int nb = *count;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nb; t += gridDim.x * blockDim.x) {
    const int n = list[t];
    const int j = n / g.nx, i = n - j * g.nx;
    for (int var = 0; var < g.c; ++var) {
      double sx = 0.0;
#pragma unroll
      for (int m = 0; m < 7; ++m)
        if (m <= 2 * rad) {
          const int64_t nn = (int64_t)j * g.nx + fwrap(i + m - rad, g.nx, g.bc);
          sx += cfr[m] * v.p[sidx(v, var * g.N + nn)];
        }
      Vp[var * g.N + n] = sx / den;
    }
  }
}
// P2 on the own band cells: v'' = S^y(v') (band neighbours: x-filtered, others: fixed values),
// residual gate against F, kept values applied in place, sweep statistics
__global__ void __launch_bounds__(256) filt_y_kernel(Geo g, SRef v, const double* __restrict__ Vp,
                                                     const double* __restrict__ F, const uint32_t* __restrict__ mB,
                                                     const int32_t* __restrict__ list,
                                                     const int32_t* __restrict__ count, int order,
                                                     uint8_t* __restrict__ flag, unsigned long long* __restrict__ stat) {
  const double* cf;
  double den;
  const int rad = fshapiro(order, &cf, &den);
  double cfr[7];
#pragma unroll
  for (int m = 0; m < 7; ++m) cfr[m] = m <= 2 * rad ? cf[m] : 0.0;
  const int nb = *count;
  double mdec = 0.0;
  int cnt = 0;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nb; t += gridDim.x * blockDim.x) {
    const int n = list[t];
    const int j = n / g.nx, i = n - j * g.nx;
    double rold = 0.0, rnew = 0.0, fs = 0.0, vpp[4];
    for (int var = 0; var < g.c; ++var) {
      double sy = 0.0;
#pragma unroll
      for (int m = 0; m < 7; ++m)
        if (m <= 2 * rad) {
          const int jj = fwrap(j + m - rad, g.ny, g.bcy);
          const int64_t nn = (int64_t)jj * g.nx + i;
          const bool inB = (mB[(int64_t)jj * g.wpr + (i >> 5)] >> (i & 31)) & 1u;
          const double yv = inB ? Vp[var * g.N + nn] : v.p[sidx(v, var * g.N + nn)];
          sy += cfr[m] * yv;
        }
      const double xv = sy / den;
      vpp[var] = xv;
      const double own = v.p[sidx(v, var * g.N + n)], fe = F[var * g.N + n];
      rold = fmax(rold, fabs(own - fe));
      rnew = fmax(rnew, fabs(xv - fe));
      fs = fmax(fs, fabs(fe));
    }
    if (rnew < rold) {
      for (int var = 0; var < g.c; ++var) v.p[sidx(v, var * g.N + n)] = vpp[var];
      flag[n] = 1;
      if (rold > 0x1p-40 * fs) mdec = fmax(mdec, (rold - rnew) / rold);  // A23': above the rounding level
      ++cnt;
    }
  }
  __shared__ double sdec[8];
  __shared__ int scnt[8];
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
    atomicMax(stat, (unsigned long long)__double_as_longlong(md));  // non-negative doubles order like their bits
    atomicAdd(stat + 1, (unsigned long long)c);
  }
}
// indicator on the kept own band cells: eps_n = sum_v (v - (psi + Phi y))^2 (filter.cu write-back)
__global__ void filt_final_kernel(Geo g, SRef v, const int32_t* __restrict__ list, const int32_t* __restrict__ count,
                                  const double* __restrict__ v0, const uint8_t* __restrict__ flag,
                                  double* __restrict__ eps) {
  const int nb = *count;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nb; t += gridDim.x * blockDim.x) {
    const int64_t n = list[t];
    if (!flag[n]) continue;
    double sum = 0.0;
    for (int var = 0; var < g.c; ++var) {
      const double d = v.p[sidx(v, var * g.N + n)] - v0[var * g.N + n];
      sum += d * d;
    }
    eps[n] = sum;
  }
}

template <typename T>
hrom_status salloc(T** p, size_t n) {
  const size_t bytes = std::max<size_t>(n, 1) * sizeof(T);
  if (cudaMalloc((void**)p, bytes) != cudaSuccess) return HROM_E_NOMEM;
  if (cudaMemset(*p, 0, bytes) != cudaSuccess) return HROM_E_CUDA;
  return HROM_OK;
}

int halo_rows(const hrom_params* p) { return std::max(3 * p->halo, 2 * p->halo + std::max(p->band, 0)); }

hrom_status partition(int ny, int P, int rank, int periodic, int H, hrom_slab_info* o) {
  if (ny < 1 || P < 1 || rank < 0 || rank >= P || H < 0) return HROM_E_INVALID;
  const int base = ny / P, rem = ny % P;
  const int own = base + (rank < rem ? 1 : 0);
  const int row0 = rank * base + std::min(rank, rem);
  if (P > 1 && base < H) return HROM_E_INVALID;  // a halo must come from ONE neighbour
  std::memset(o, 0, sizeof(*o));
  o->rank = rank;
  o->nranks = P;
  o->ny_global = ny;
  o->row0 = row0;
  o->rows_own = own;
  o->halo = H;
  o->halo_lo = (P > 1 && (periodic || rank > 0)) ? H : 0;
  o->halo_hi = (P > 1 && (periodic || rank < P - 1)) ? H : 0;
  return HROM_OK;
}

int grid_for(const hrom_ctx* c, int64_t n, int threads = 256) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, 8 * (int64_t)c->nsm));
}

// message offsets
struct EndLayout {
  int64_t first_rows, last_rows, row, tail, bytes;
};
EndLayout end_layout(const hrom_slab* s) {
  EndLayout L;
  L.first_rows = 0;
  L.last_rows = s->halo_doubles * 8;
  L.row = 2 * s->halo_doubles * 8;
  L.tail = L.row + 2 * ROW_SLOTS * 8;
  L.bytes = L.tail + 16;
  return L;
}

hrom_status pack_halo(hrom_ctx* c, SRef q, unsigned char* send) {
  hrom_slab* s = c->slab;
  if (s->H == 0 || s->nranks == 1) return HROM_OK;
  const EndLayout L = end_layout(s);
  const int g = grid_for(c, s->halo_doubles);
  pack_rows_kernel<<<g, 256, 0, c->st>>>(c->g, q, s->hlo, s->H, reinterpret_cast<double*>(send + L.first_rows));
  pack_rows_kernel<<<g, 256, 0, c->st>>>(c->g, q, s->hlo + s->own - s->H, s->H,
                                         reinterpret_cast<double*>(send + L.last_rows));
  HROM_LAUNCH_CK();
  c->nlaunch += 2;
  return HROM_OK;
}

hrom_status unpack_halo(hrom_ctx* c, SRef q, const unsigned char* gath, int64_t stride) {
  hrom_slab* s = c->slab;
  if (s->nranks == 1) return HROM_OK;
  const EndLayout L = end_layout(s);
  const int P = s->nranks, g = grid_for(c, s->halo_doubles);
  if (s->hlo) {  // rows below my first own row = the LAST own rows of rank - 1
    const int nb = (s->rank - 1 + P) % P;
    unpack_rows_kernel<<<g, 256, 0, c->st>>>(c->g, q, 0, s->H,
                                             reinterpret_cast<const double*>(gath + nb * stride + L.last_rows));
    ++c->nlaunch;
  }
  if (s->hhi) {  // rows above my last own row = the FIRST own rows of rank + 1
    const int nb = (s->rank + 1) % P;
    unpack_rows_kernel<<<g, 256, 0, c->st>>>(c->g, q, s->hlo + s->own, s->H,
                                             reinterpret_cast<const double*>(gath + nb * stride + L.first_rows));
    ++c->nlaunch;
  }
  HROM_LAUNCH_CK();
  return HROM_OK;
}

// the sets of the next step from the complete local S-hat bitmap (own + halo rows), then the
// own-row sub-lists and the fill's exclusion mask
hrom_status finish_sets(hrom_ctx* c) {
  hrom_slab* s = c->slab;
  // with the previous S-hat in M_SPREV the sets kernel also lists the churn (G7)
  hrom_status st = s->have_prev ? build_sets_with_churn(c) : build_sets(c, nullptr);
  if (st != HROM_OK) return st;
  const Geo& g = c->g;
  const int lo = s->hlo * g.nx, hi = (s->hlo + s->own) * g.nx;
  if (s->have_prev) {
    own_list_kernel<<<grid_for(c, g.N), 256, 0, c->st>>>(c->b.lists + (int64_t)L_ADD * g.N, c->b.counts + L_ADD, lo, hi,
                                                        s->listAdd, s->cnt + 3);
    own_list_kernel<<<grid_for(c, g.N), 256, 0, c->st>>>(c->b.lists + (int64_t)L_REM * g.N, c->b.counts + L_REM, lo, hi,
                                                        s->listRem, s->cnt + 4);
    c->nlaunch += 2;
  }
  s->have_prev = true;
  own_list_kernel<<<grid_for(c, g.N), 256, 0, c->st>>>(c->b.lists + (int64_t)L_S * g.N, c->b.counts + L_S, lo, hi,
                                                      s->listS, s->cnt + 0);
  own_list_kernel<<<grid_for(c, g.N), 256, 0, c->st>>>(c->b.lists + (int64_t)L_B * g.N, c->b.counts + L_B, lo, hi,
                                                      s->listB, s->cnt + 1);
  halo_mask_kernel<<<grid_for(c, (int64_t)g.ny * g.wpr), 256, 0, c->st>>>(c->b.masks + (int64_t)M_B * c->mwords, s->mBH,
                                                                        g.wpr, g.ny, s->hlo, s->hlo + s->own);
  HROM_LAUNCH_CK();
  c->nlaunch += 3;
  c->sets_ready = true;
  return HROM_OK;
}

// first selection pass: zero the histogram, count the top digit of the own cells' eps > 0
hrom_status sel_pass(hrom_ctx* c, int pass, unsigned char* send) {
  hrom_slab* s = c->slab;
  const Geo& g = c->g;
  HROM_CK(cudaMemsetAsync(s->hist, 0, NBIN * sizeof(int32_t), c->st));
  const int lo = s->hlo * g.nx, hi = (s->hlo + s->own) * g.nx;
  sel_hist_kernel<<<std::min(2 * c->nsm, std::max(1, (hi - lo + 1023) / 1024)), 1024, 0, c->st>>>(c->b.eps, lo, hi, pass,
                                                                                                s->sel, s->hist);
  HROM_LAUNCH_CK();
  ++c->nlaunch;
  HROM_CK(cudaMemcpyAsync(send, s->hist, NBIN * sizeof(int32_t), cudaMemcpyDeviceToDevice, c->st));
  return HROM_OK;
}

// basis update + start of the sampling after step k (k >= w - 1); returns the message length
hrom_status begin_update(hrom_ctx* c, unsigned char* send, int64_t* bytes) {
  hrom_slab* s = c->slab;
  const int64_t k = c->k;
  const Win W = window_of(c, k);
  c->eig_win = W;
  c->eig_todo = true;
  hrom_status st = flush_eigen(c);  // side stream: overlaps the selection passes
  if (st != HROM_OK) return st;
  c->win = W;
  c->basis_ready = true;
  c->gram_row_ready = false;
  c->full_since_update = false;
  if (k == c->w - 1) {  // bootstrap: projection indicator (A19)
    basis_join(c);
    if ((st = launch_zvec(c, c->w, 0.0)) != HROM_OK) return st;
    if ((st = launch_fill(c, W, 2, plain(nullptr), plain(nullptr), false)) != HROM_OK) return st;
    if ((st = launch_eps_all(c)) != HROM_OK) return st;
    c->eps_sparse = false;
  }
  s->sel_pass = 0;
  if ((st = sel_pass(c, 0, send)) != HROM_OK) return st;
  *bytes = NBIN * sizeof(int32_t);
  s->phase = PH_SEL;
  return HROM_OK;
}


bool filter_on(const hrom_ctx* c) { return c->P.n_filter_orders > 0 && c->P.filter_max_sweeps > 0; }

// one filter sweep of cascade order f_order: x-pass on every local band cell, y-pass + gate on the
// own band cells; message = END layout with the edge rows and the sweep's statistics in the tail
hrom_status run_sweep(hrom_ctx* c, unsigned char* send, int64_t* bytes) {
  hrom_slab* s = c->slab;
  const Geo& g = c->g;
  Bufs& b = c->b;
  const SRef v = c->slot_ref(c->slot_of(c->k + 1));
  const int order = c->P.filter_orders[s->f_order];
  const EndLayout L = end_layout(s);
  HROM_CK(cudaMemsetAsync(s->fstat, 0, 2 * sizeof(unsigned long long), c->st));
  const int grid = 4 * c->nsm;
  filt_x_kernel<<<grid, 256, 0, c->st>>>(g, v, b.lists + (int64_t)L_B * g.N, b.counts + L_B, order, b.U1);
  filt_y_kernel<<<grid, 256, 0, c->st>>>(g, v, b.U1, b.U3, b.masks + (int64_t)M_B * c->mwords, s->listB, s->cnt + 1,
                                         order, b.kept, s->fstat);
  HROM_LAUNCH_CK();
  c->nlaunch += 2;
  hrom_status st = pack_halo(c, v, send);
  if (st != HROM_OK) return st;
  HROM_CK(cudaMemsetAsync(send + L.row, 0, 2 * ROW_SLOTS * 8, c->st));
  HROM_CK(cudaMemcpyAsync(send + L.tail, s->fstat, 16, cudaMemcpyDeviceToDevice, c->st));
  ++s->f_sweeps[s->f_order];
  *bytes = L.bytes;
  s->phase = PH_FSWEEP;
  return HROM_OK;
}

// after the fill (and the filter): band part of the Gram row, positivity + wave speeds of the own
// rows, the END message
hrom_status finish_hybrid(hrom_ctx* c, unsigned char* send, int64_t* bytes) {
  hrom_slab* s = c->slab;
  const Geo& g = c->g;
  Bufs& b = c->b;
  const int64_t kn = c->k + 1;
  const SRef out = c->slot_ref(c->slot_of(kn));
  const int64_t own_lo = (int64_t)s->hlo * g.nx, own_hi = (int64_t)(s->hlo + s->own) * g.nx;
  hrom_status st;
  if ((st = band_gram_rows_list(c, c->win, out, s->listB, s->cnt + 1)) != HROM_OK) return st;
  if ((st = launch_positivity_check(c, out, own_lo, own_hi)) != HROM_OK) return st;
  const EndLayout L = end_layout(s);
  slab_row_reduce<<<((c->win.nU + 1) * 16 + 255) / 256, 256, 0, c->st>>>(b.gpart, c->fill_grid, b.gpart + (int64_t)c->fill_blocks * (c->win.nU + 1) * 2,
                                         c->band_blocks, c->win.nU, reinterpret_cast<double*>(send + L.row));
  HROM_LAUNCH_CK();
  ++c->nlaunch;
  if ((st = pack_halo(c, out, send)) != HROM_OK) return st;
  // tail: the own rows' wave-speed maximum (H1 of the next step) and positivity flag
  HROM_CK(cudaMemcpyAsync(send + L.tail, b.ureg + 2, 8, cudaMemcpyDeviceToDevice, c->st));
  HROM_CK(cudaMemcpyAsync(send + L.tail + 8, b.ureg + 3, 8, cudaMemcpyDeviceToDevice, c->st));
  c->k = kn;
  c->points_used = 0;
  c->last_hybrid = true;
  c->eps_sparse = true;
  c->gram_row_ready = false;
  c->sets_ready = false;
  s->step_hybrid = true;
  *bytes = L.bytes;
  s->phase = PH_END;
  return HROM_OK;
}

// the filter is over: indicator on the kept own band cells, sweep counts where the unsharded
// filter reports them (ireg[4..6]), then the rest of the step
hrom_status end_filter(hrom_ctx* c, unsigned char* send, int64_t* bytes) {
  hrom_slab* s = c->slab;
  const SRef v = c->slot_ref(c->slot_of(c->k + 1));
  filt_final_kernel<<<4 * c->nsm, 256, 0, c->st>>>(c->g, v, s->listB, s->cnt + 1, c->b.Vorig, c->b.kept, c->b.eps);
  HROM_LAUNCH_CK();
  ++c->nlaunch;
  int32_t sw[3] = {s->f_sweeps[0], s->f_sweeps[1], s->f_sweeps[2]};
  HROM_CK(cudaMemcpyAsync(c->b.ireg + 4, sw, sizeof(sw), cudaMemcpyHostToDevice, c->st));
  HROM_CK(cudaStreamSynchronize(c->st));  // sw is a stack array
  return finish_hybrid(c, send, bytes);
}

}  // namespace

void slab_destroy(hrom_ctx* c) {
  hrom_slab* s = c->slab;
  if (!s) return;
  void* ptrs[] = {s->listS, s->listB, s->listA, s->listAdd, s->listRem, s->cnt, s->mBH, s->sel, s->hist, s->stage, s->fstat};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  delete s;
  c->slab = nullptr;
}

}  // namespace hrom

using namespace hrom;

extern "C" {

hrom_status hrom_slab_partition(int32_t ny_global, int32_t nranks, int32_t rank, int32_t periodic, int32_t halo_rows_,
                                hrom_slab_info* out) {
  if (!out) return HROM_E_INVALID;
  return partition(ny_global, nranks, rank, periodic, halo_rows_, out);
}

hrom_status hrom_slab_create(const hrom_grid* grid, double gamma, double cfl, const hrom_params* p, void* stream,
                             int32_t rank, int32_t nranks, hrom_ctx** out) {
  if (!grid || !p || !out) return HROM_E_INVALID;
  *out = nullptr;
  if (grid->dim != 2) return HROM_E_INVALID;  // a 1-D grid has no rows to split
  if (nranks < 1 || nranks > 64 || rank < 0 || rank >= nranks) return HROM_E_INVALID;  // host decisions read <= 64 flags
  if (p->odeim_points > 0 || p->sample_mode != 0 || p->full_period > 0 || p->band < 0 || p->gram_mode != 0)
    return HROM_E_INVALID;
  hrom_slab_info info;
  const int H = halo_rows(p);
  hrom_status st = partition(grid->ny, nranks, rank, grid->bc == 1, H, &info);
  if (st != HROM_OK) return st;
  hrom_grid lg = *grid;
  lg.ny = info.rows_own + info.halo_lo + info.halo_hi;
  hrom_params lp = *p;
  lp.gather_mode = 0;  // incremental gathered Gram (G7): the churn lists are rebuilt from M_SPREV (finish_sets)
  hrom_ctx* c = nullptr;
  if ((st = hrom_create(&lg, gamma, cfl, &lp, stream, &c)) != HROM_OK) return st;
  if (c->P.gram_mode != 0) {  // the fused Gram row (w + 1 <= 68) carries the halo exclusion
    hrom_destroy(c);
    return HROM_E_INVALID;
  }
  // the global mesh width (bitwise the unsharded context's dy) and open y ends on split grids
  Geo& g = c->g;
  g.dy = (grid->y1 - grid->y0) / grid->ny;
  g.rdy = 1.0 / g.dy;
  {
    int ex = 0, ey = 0;
    g.pow2 = (std::frexp(g.dx, &ex) == 0.5 && std::frexp(g.dy, &ey) == 0.5) ? 1 : 0;
  }
  if (nranks > 1) g.bcy = 0;
  hrom_slab* s = new hrom_slab();
  c->slab = s;
  s->rank = rank;
  s->nranks = nranks;
  s->ny_g = grid->ny;
  s->row0 = info.row0;
  s->own = info.rows_own;
  s->hlo = info.halo_lo;
  s->hhi = info.halo_hi;
  s->H = nranks > 1 ? H : 0;
  s->bc_g = grid->bc;
  s->N_g = (int64_t)grid->nx * grid->ny;
  s->halo_doubles = (int64_t)g.c * s->H * g.nx;
  s->mask_words = (int64_t)s->H * g.wpr;
  const int64_t r_bytes = (int64_t)(4 * (kMaxW + 2) * (kMaxW + 2) + 2 * (2 * kMaxW + 3)) * 8;
  s->max_msg = std::max<int64_t>({end_layout(s).bytes, r_bytes, (int64_t)NBIN * 4, 2 * s->mask_words * 4, 16});
  auto A = [&](hrom_status r) { if (r != HROM_OK) st = r; };
  A(salloc(&s->listS, g.N));
  A(salloc(&s->listB, g.N));
  A(salloc(&s->listA, g.N));
  A(salloc(&s->listAdd, g.N));
  A(salloc(&s->listRem, g.N));
  A(salloc(&s->cnt, 8));
  A(salloc(&s->mBH, c->mwords));
  A(salloc(&s->sel, 8));
  A(salloc(&s->hist, NBIN));
  A(salloc(&s->stage, g.Dp));
  A(salloc(&s->fstat, 2));
  if (st != HROM_OK) {
    hrom_destroy(c);
    return st;
  }
  iota_kernel<<<grid_for(c, (int64_t)s->own * g.nx), 256, 0, c->st>>>(s->listA, s->hlo * g.nx, s->own * g.nx, s->cnt + 2);
  if (cudaGetLastError() != cudaSuccess) {
    hrom_destroy(c);
    return HROM_E_CUDA;
  }
  *out = c;
  return HROM_OK;
}

hrom_status hrom_slab_get_info(const hrom_ctx* c, hrom_slab_info* out) {
  if (!c || !c->slab || !out) return HROM_E_INVALID;
  const hrom_slab* s = c->slab;
  std::memset(out, 0, sizeof(*out));
  out->rank = s->rank;
  out->nranks = s->nranks;
  out->ny_global = s->ny_g;
  out->row0 = s->row0;
  out->rows_own = s->own;
  out->halo_lo = s->hlo;
  out->halo_hi = s->hhi;
  out->halo = s->H;
  out->cells_own = (int64_t)s->own * c->g.nx;
  out->cells_local = c->g.N;
  out->cells_global = s->N_g;
  out->max_message_bytes = s->max_msg;
  return HROM_OK;
}

hrom_status hrom_slab_set_state(hrom_ctx* c, const double* any_q_global) {
  if (!c || !c->slab || !any_q_global) return HROM_E_INVALID;
  hrom_slab* s = c->slab;
  const Geo& g = c->g;
  // local row jl <-> global row (row0 - halo_lo + jl) mod ny_global, copied in contiguous runs
  for (int v = 0; v < g.c; ++v) {
    int jl = 0;
    while (jl < g.ny) {
      int gj = s->row0 - s->hlo + jl;
      gj = ((gj % s->ny_g) + s->ny_g) % s->ny_g;
      const int run = std::min(g.ny - jl, s->ny_g - gj);
      HROM_CK(cudaMemcpyAsync(s->stage + v * g.N + (int64_t)jl * g.nx, any_q_global + v * s->N_g + (int64_t)gj * g.nx,
                              (size_t)run * g.nx * sizeof(double), cudaMemcpyDefault, c->st));
      jl += run;
    }
  }
  s->phase = PH_IDLE;
  s->have_prev = false;
  return hrom_set_state(c, s->stage);
}

hrom_status hrom_slab_get_state(hrom_ctx* c, double* any_q_own) {
  if (!c || !c->slab || !any_q_own) return HROM_E_INVALID;
  hrom_slab* s = c->slab;
  const Geo& g = c->g;
  hrom_status st = hrom_get_state(c, s->stage);
  if (st != HROM_OK) return st;
  const int64_t per = (int64_t)s->own * g.nx;
  for (int v = 0; v < g.c; ++v)
    HROM_CK(cudaMemcpyAsync(any_q_own + v * per, s->stage + v * g.N + (int64_t)s->hlo * g.nx, per * sizeof(double),
                            cudaMemcpyDefault, c->st));
  return HROM_OK;
}

hrom_status hrom_slab_get_mask(hrom_ctx* c, uint32_t* any_mask_own) {
  if (!c || !c->slab || !any_mask_own) return HROM_E_INVALID;
  const hrom_slab* s = c->slab;
  HROM_CK(cudaMemcpyAsync(any_mask_own, c->b.masks + (int64_t)M_S * c->mwords + (int64_t)s->hlo * c->g.wpr,
                          (size_t)s->own * c->g.wpr * sizeof(uint32_t), cudaMemcpyDefault, c->st));
  return HROM_OK;
}

hrom_status hrom_slab_get_indicator(hrom_ctx* c, double* any_eps_own) {
  if (!c || !c->slab || !any_eps_own) return HROM_E_INVALID;
  const hrom_slab* s = c->slab;
  HROM_CK(cudaMemcpyAsync(any_eps_own, c->b.eps + (int64_t)s->hlo * c->g.nx,
                          (size_t)s->own * c->g.nx * sizeof(double), cudaMemcpyDefault, c->st));
  return HROM_OK;
}

int64_t hrom_slab_escalations(const hrom_ctx* c) { return (c && c->slab) ? c->slab->escalations : -1; }

hrom_status hrom_slab_set_window(hrom_ctx* c, int64_t k, const double* any_snaps_global, int32_t nsnaps,
                                 const uint32_t* any_mask_global, void* dev_send, int64_t* send_bytes_out) {
  if (!c || !c->slab || !any_snaps_global || !any_mask_global || !dev_send || !send_bytes_out) return HROM_E_INVALID;
  if (k < c->w || nsnaps != c->w + 1) return HROM_E_INVALID;
  hrom_slab* s = c->slab;
  const Geo& g = c->g;
  Bufs& b = c->b;
  basis_join(c);
  hrom_status st;
  const int64_t Dg = (int64_t)g.c * s->N_g;
  for (int t = 0; t < nsnaps; ++t) {
    const double* q = any_snaps_global + (int64_t)t * Dg;
    for (int v = 0; v < g.c; ++v) {
      int jl = 0;
      while (jl < g.ny) {
        int gj = s->row0 - s->hlo + jl;
        gj = ((gj % s->ny_g) + s->ny_g) % s->ny_g;
        const int run = std::min(g.ny - jl, s->ny_g - gj);
        HROM_CK(cudaMemcpyAsync(s->stage + v * g.N + (int64_t)jl * g.nx, q + v * s->N_g + (int64_t)gj * g.nx,
                                (size_t)run * g.nx * sizeof(double), cudaMemcpyDefault, c->st));
        jl += run;
      }
    }
    if ((st = hrom_put_snapshot(c, k - c->w + t, s->stage)) != HROM_OK) return st;
  }
  {  // S-hat_{k+1}: the local rows (own + halo) of the global bitmap
    uint32_t* S = b.masks + (int64_t)M_S * c->mwords;
    int jl = 0;
    while (jl < g.ny) {
      int gj = s->row0 - s->hlo + jl;
      gj = ((gj % s->ny_g) + s->ny_g) % s->ny_g;
      const int run = std::min(g.ny - jl, s->ny_g - gj);
      HROM_CK(cudaMemcpyAsync(S + (int64_t)jl * g.wpr, any_mask_global + (int64_t)gj * g.wpr,
                              (size_t)run * g.wpr * sizeof(uint32_t), cudaMemcpyDefault, c->st));
      jl += run;
    }
  }
  HROM_CK(cudaMemsetAsync(b.ureg + 1, 0xff, sizeof(unsigned long long), c->st));
  c->k = k;
  c->last_hybrid = false;
  c->full_since_update = false;
  c->n_owed = 0;
  c->kinc_valid = false;
  c->eps_sparse = false;
  c->basis_ready = false;
  c->gram_row_ready = false;
  c->sets_ready = false;
  c->smax_k = -1;
  s->have_prev = false;
  // window Gram of the own rows (shift rho := the newest snapshot), summed over the ranks next
  const size_t pitch = (size_t)g.nsr * TILE * sizeof(double);
  HROM_CK(cudaMemcpy2DAsync(b.rho, pitch, b.ring + (int64_t)c->slot_of(k) * TILE, pitch, TILE * sizeof(double),
                            (size_t)(g.Dp / TILE), cudaMemcpyDeviceToDevice, c->st));
  const Win W = window_of(c, k);
  if ((st = gram_gathered_list(c, W, c->slot_ref(c->slot_of(k)), s->listA, s->cnt + 2, b.eigV, b.Rlo)) != HROM_OK)
    return st;
  const int ncol = W.nU + 1, n2 = ncol * ncol;
  unsigned char* send = static_cast<unsigned char*>(dev_send);
  HROM_CK(cudaMemcpyAsync(send, b.eigV, (size_t)n2 * 8, cudaMemcpyDeviceToDevice, c->st));
  HROM_CK(cudaMemcpyAsync(send + (size_t)n2 * 8, b.Rlo, (size_t)n2 * 8, cudaMemcpyDeviceToDevice, c->st));
  *send_bytes_out = (int64_t)2 * n2 * 8;
  s->phase = PH_REBUILD;
  return HROM_OK;
}

hrom_status hrom_slab_resample(hrom_ctx* c, const double* any_eps_own, void* dev_send, int64_t* send_bytes_out) {
  if (!c || !c->slab || !any_eps_own || !dev_send || !send_bytes_out) return HROM_E_INVALID;
  hrom_slab* s = c->slab;
  if (s->phase != PH_IDLE) return HROM_E_STATE;
  HROM_CK(cudaMemsetAsync(c->b.eps, 0, c->g.N * sizeof(double), c->st));
  HROM_CK(cudaMemcpyAsync(c->b.eps + (int64_t)s->hlo * c->g.nx, any_eps_own, (size_t)s->own * c->g.nx * sizeof(double),
                          cudaMemcpyDefault, c->st));
  s->sel_pass = 0;
  hrom_status st = sel_pass(c, 0, static_cast<unsigned char*>(dev_send));
  if (st != HROM_OK) return st;
  *send_bytes_out = NBIN * sizeof(int32_t);
  s->phase = PH_SEL;
  return HROM_OK;
}

hrom_status hrom_slab_step(hrom_ctx* c, const void* dev_gathered, void* dev_send, int64_t* send_bytes_out) {
  if (!c || !c->slab || !dev_send || !send_bytes_out) return HROM_E_INVALID;
  if (c->k < 0) return HROM_E_STATE;
  hrom_slab* s = c->slab;
  const Geo& g = c->g;
  Bufs& b = c->b;
  const int P = s->nranks;
  const unsigned char* gath = static_cast<const unsigned char*>(dev_gathered);
  unsigned char* send = static_cast<unsigned char*>(dev_send);
  *send_bytes_out = 0;
  hrom_status st;
  if (s->phase != PH_IDLE && !gath) return HROM_E_STATE;
  // reductions and flags run over the own rows only: the halo rows of a state under construction
  // hold open-end values until the exchange
  const int64_t own_lo = (int64_t)s->hlo * g.nx, own_hi = (int64_t)(s->hlo + s->own) * g.nx;

  if (s->phase == PH_IDLE) {
    if (c->smax_k != c->k) {  // H1's maximum of gamma_k is not known yet (first step / after a set_state)
      HROM_CK(cudaMemsetAsync(s->sel + 6, 0, sizeof(unsigned long long), c->st));
      if ((st = launch_smax(c, c->slot_ref(c->slot_of(c->k)), s->sel + 6, own_lo, own_hi)) != HROM_OK) return st;
      HROM_CK(cudaMemcpyAsync(send, s->sel + 6, 8, cudaMemcpyDeviceToDevice, c->st));
      HROM_CK(cudaMemsetAsync(send + 8, 0xff, 8, c->st));
      *send_bytes_out = 16;
      s->phase = PH_SMAX;
      return HROM_OK;
    }
  } else if (s->phase == PH_SMAX) {
    smax_reduce_kernel<<<1, 1, 0, c->st>>>(gath, 16, 0, P, b.ureg, 0);
    HROM_LAUNCH_CK();
    ++c->nlaunch;
    c->smax_k = c->k;
    s->phase = PH_IDLE;
  }

  if (s->phase == PH_IDLE) {
    // ---- stage part of step k -> k + 1 (Algorithm 1 line P:557: full while k + 1 <= w) ----
    const int64_t kn = c->k + 1;
    const bool full = kn + 1 <= c->w;
    const SRef qn = c->slot_ref(c->slot_of(c->k));
    const SRef out = c->slot_ref(c->slot_of(kn));
    const SRef U1 = plain(b.U1), U2 = plain(b.U2), U3 = plain(b.U3);
    const EndLayout L = end_layout(s);
    if (full) {
      if ((st = launch_dt(c, qn, 0.0, c->k)) != HROM_OK) return st;
      if ((st = launch_stage(c, 1, qn, qn, U1, nullptr, 0, 0.0)) != HROM_OK) return st;
      if ((st = launch_stage(c, 2, qn, U1, U2, nullptr, 0, 0.0)) != HROM_OK) return st;
      if ((st = launch_stage(c, 3, qn, U2, out, nullptr, 0, 0.0)) != HROM_OK) return st;
      // END message: halo rows, an empty Gram row, the wave-speed maximum of the own rows, no flag
      if ((st = pack_halo(c, out, send)) != HROM_OK) return st;
      HROM_CK(cudaMemsetAsync(send + L.row, 0, 2 * ROW_SLOTS * 8, c->st));
      c->k = kn;
      c->points_used = 0;
      c->last_hybrid = false;
      c->full_since_update = true;
      c->gram_row_ready = false;
      c->sets_ready = false;
      s->step_hybrid = false;
      HROM_CK(cudaMemsetAsync(s->sel + 6, 0, sizeof(unsigned long long), c->st));
      if ((st = launch_smax(c, out, s->sel + 6, own_lo, own_hi)) != HROM_OK) return st;
      HROM_CK(cudaMemcpyAsync(send + L.tail, s->sel + 6, 8, cudaMemcpyDeviceToDevice, c->st));
      HROM_CK(cudaMemsetAsync(send + L.tail + 8, 0xff, 8, c->st));
      *send_bytes_out = L.bytes;
      s->phase = PH_END;
      return HROM_OK;
    }
    if (!c->basis_ready || !c->sets_ready) return HROM_E_STATE;
    if ((st = flush_eigen(c)) != HROM_OK) return st;
    if ((st = launch_dt(c, qn, 0.0, c->k)) != HROM_OK) return st;
    const int32_t* Ls = b.lists;
    if ((st = launch_stage(c, 1, qn, qn, U1, Ls + (int64_t)L_A1 * g.N, L_A1, 0.0)) != HROM_OK) return st;
    if ((st = launch_stage(c, 2, qn, U1, U2, Ls + (int64_t)L_A2 * g.N, L_A2, 0.0)) != HROM_OK) return st;
    if ((st = launch_stage(c, 3, qn, U2, U3, Ls + (int64_t)L_T * g.N, L_T, 0.0)) != HROM_OK) return st;
    // H4 on the own rows of S-hat: the full gathered Gram, or (G7) the Grams of the own rows that
    // entered / left S-hat and the two GEMVs -- every part is a sum over rows, so the ranks' parts add
    GatherLists GL{s->listS, s->cnt + 0, s->listAdd, s->cnt + 3, s->listRem, s->cnt + 4};
    if ((st = gram_gathered_partial(c, U3, &GL)) != HROM_OK) return st;
    const int ncol = c->win.nU + 1, n2 = ncol * ncol;
    if (!c->gather_inc) {
      HROM_CK(cudaMemcpyAsync(send, b.eigV, (size_t)n2 * 8, cudaMemcpyDeviceToDevice, c->st));
      HROM_CK(cudaMemcpyAsync(send + (size_t)n2 * 8, b.Rlo, (size_t)n2 * 8, cudaMemcpyDeviceToDevice, c->st));
      *send_bytes_out = (int64_t)2 * n2 * 8;
    } else {
      const size_t S2 = (size_t)(kMaxW + 2) * (kMaxW + 2);
      const int nv = 2 * c->win.nU + 1;
      for (int q = 0; q < 4; ++q)  // R+ hi, lo, R- hi, lo
        HROM_CK(cudaMemcpyAsync(send + (size_t)q * n2 * 8, b.Rd + q * S2, (size_t)n2 * 8, cudaMemcpyDeviceToDevice, c->st));
      HROM_CK(cudaMemcpyAsync(send + (size_t)4 * n2 * 8, gathered_gemv_values(c), (size_t)2 * nv * 8,
                              cudaMemcpyDeviceToDevice, c->st));
      *send_bytes_out = (int64_t)(4 * n2 + 2 * nv) * 8;
    }
    s->phase = PH_R;
    return HROM_OK;
  }

  if (s->phase == PH_R) {
    const int64_t kn = c->k + 1;
    const SRef qn = c->slot_ref(c->slot_of(c->k));
    (void)qn;
    const SRef out = c->slot_ref(c->slot_of(kn));
    const SRef U3 = plain(b.U3);
    const int ncol = c->win.nU + 1, n2 = ncol * ncol;
    if (!c->gather_inc) {
      dd_sum_kernel<<<(n2 + 255) / 256, 256, 0, c->st>>>(gath, (int64_t)2 * n2 * 8, 0, P, n2, 0, b.eigV, b.Rlo);
      ++c->nlaunch;
    } else {
      const size_t S2 = (size_t)(kMaxW + 2) * (kMaxW + 2);
      const int nv = 2 * c->win.nU + 1;
      const int64_t stride = (int64_t)(4 * n2 + 2 * nv) * 8;
      dd_sum_kernel<<<(n2 + 255) / 256, 256, 0, c->st>>>(gath, stride, 0, P, n2, 0, b.Rd, b.Rd + S2);
      dd_sum_kernel<<<(n2 + 255) / 256, 256, 0, c->st>>>(gath, stride, (int64_t)2 * n2 * 8, P, n2, 0, b.Rd + 2 * S2,
                                                         b.Rd + 3 * S2);
      double* v = gathered_gemv_values(c);
      dd_sum_kernel<<<(nv + 255) / 256, 256, 0, c->st>>>(gath, stride, (int64_t)4 * n2 * 8, P, nv, 1, v, v + 1);
      c->nlaunch += 3;
    }
    HROM_LAUNCH_CK();
    if ((st = gram_gathered_finish(c)) != HROM_OK) return st;
    basis_join(c);
    if ((st = small_solve(c)) != HROM_OK) return st;  // H5, replicated: identical y on every rank
    HROM_CK(cudaMemsetAsync(b.eps, 0, g.N * sizeof(double), c->st));
    c->fill_mB_override = s->mBH;
    st = launch_fill(c, c->win, 0, U3, out, true);  // H6 + H9 + the own rows' part of the H10 row
    c->fill_mB_override = nullptr;
    if (st != HROM_OK) return st;
    if ((st = launch_eps_cells(c)) != HROM_OK) return st;
    if (!filter_on(c)) return finish_hybrid(c, send, send_bytes_out);
    // H7: the neighbours' pre-filter rows first (the filter's stencils reach into the halo)
    const EndLayout L = end_layout(s);
    if ((st = pack_halo(c, out, send)) != HROM_OK) return st;
    HROM_CK(cudaMemsetAsync(send + L.row, 0, L.bytes - L.row, c->st));
    *send_bytes_out = L.bytes;
    s->phase = PH_HALO1;
    return HROM_OK;
  }

  if (s->phase == PH_HALO1) {
    const EndLayout L = end_layout(s);
    const SRef v = c->slot_ref(c->slot_of(c->k + 1));
    if ((st = unpack_halo(c, v, gath, L.bytes)) != HROM_OK) return st;
    filt_init_kernel<<<4 * c->nsm, 256, 0, c->st>>>(g, v, s->listB, s->cnt + 1, b.Vorig, b.kept);
    HROM_LAUNCH_CK();
    ++c->nlaunch;
    s->f_order = s->f_sw = 0;
    s->f_sweeps[0] = s->f_sweeps[1] = s->f_sweeps[2] = 0;
    return run_sweep(c, send, send_bytes_out);
  }

  if (s->phase == PH_FSWEEP) {
    const EndLayout L = end_layout(s);
    const SRef v = c->slot_ref(c->slot_of(c->k + 1));
    if ((st = unpack_halo(c, v, gath, L.bytes)) != HROM_OK) return st;
    // stop decision from the gathered statistics (A23): identical on every rank
    unsigned long long hs[2 * 64];
    if (P > 64) return HROM_E_INVALID;
    HROM_CK(cudaMemcpy2DAsync(hs, 16, gath + L.tail, (size_t)L.bytes, 16, (size_t)P, cudaMemcpyDeviceToHost, c->st));
    HROM_CK(cudaStreamSynchronize(c->st));
    unsigned long long mb = 0ull, tot = 0ull;
    for (int r = 0; r < P; ++r) {
      mb = std::max(mb, hs[2 * r]);
      tot += hs[2 * r + 1];
    }
    double md;
    std::memcpy(&md, &mb, sizeof(md));
    const bool stop = tot == 0ull || md < c->P.filter_eps || s->f_sw + 1 == c->P.filter_max_sweeps;
    if (!stop) {
      ++s->f_sw;
      return run_sweep(c, send, send_bytes_out);
    }
    s->f_sw = 0;
    if (++s->f_order < c->P.n_filter_orders) return run_sweep(c, send, send_bytes_out);
    return end_filter(c, send, send_bytes_out);
  }

  if (s->phase == PH_END || s->phase == PH_END2) {
    const bool redo_done = s->phase == PH_END2;
    const EndLayout L = end_layout(s);
    const SRef qk = c->slot_ref(c->slot_of(c->k));
    if ((st = unpack_halo(c, qk, gath, L.bytes)) != HROM_OK) return st;
    if (s->step_hybrid && !redo_done) {
      // positivity flags of all ranks: any non-physical hybrid state -> every rank redoes the step
      // as a full step, decided on the host from the gathered flags (identical everywhere)
      unsigned long long hf[2 * 64];
      if (P > 64) return HROM_E_INVALID;
      HROM_CK(cudaMemcpy2DAsync(hf, 16, gath + L.tail, (size_t)L.bytes, 16, (size_t)P, cudaMemcpyDeviceToHost, c->st));
      HROM_CK(cudaStreamSynchronize(c->st));
      bool bad = false;
      for (int r = 0; r < P; ++r) bad = bad || hf[2 * r + 1] != ~0ull;
      if (bad) {
        ++s->escalations;
        const SRef qprev = c->slot_ref(c->slot_of(c->k - 1));
        const SRef U1 = plain(b.U1), U2 = plain(b.U2);
        if ((st = launch_stage(c, 1, qprev, qprev, U1, nullptr, 0, 0.0)) != HROM_OK) return st;  // dt: still in dreg
        if ((st = launch_stage(c, 2, qprev, U1, U2, nullptr, 0, 0.0)) != HROM_OK) return st;
        if ((st = launch_stage(c, 3, qprev, U2, qk, nullptr, 0, 0.0)) != HROM_OK) return st;
        HROM_CK(cudaMemsetAsync(b.ureg + 2, 0, 8, c->st));
        HROM_CK(cudaMemsetAsync(b.ureg + 3, 0xff, 8, c->st));
        if ((st = launch_positivity_check(c, qk, own_lo, own_hi)) != HROM_OK) return st;
        // the window-Gram row of the final gamma_k over every own cell (the band GEMV on the
        // all-own list), no fill partials
        if ((st = band_gram_rows_list(c, c->win, qk, s->listA, s->cnt + 2)) != HROM_OK) return st;
        slab_row_reduce<<<((c->win.nU + 1) * 16 + 255) / 256, 256, 0, c->st>>>(
            b.gpart, 0, b.gpart + (int64_t)c->fill_blocks * (c->win.nU + 1) * 2, c->band_blocks, c->win.nU,
            reinterpret_cast<double*>(send + L.row));
        HROM_LAUNCH_CK();
        ++c->nlaunch;
        if ((st = pack_halo(c, qk, send)) != HROM_OK) return st;
        HROM_CK(cudaMemcpyAsync(send + L.tail, b.ureg + 2, 8, cudaMemcpyDeviceToDevice, c->st));
        HROM_CK(cudaMemcpyAsync(send + L.tail + 8, b.ureg + 3, 8, cudaMemcpyDeviceToDevice, c->st));
        *send_bytes_out = L.bytes;
        s->phase = PH_END2;
        return HROM_OK;
      }
    }
    // wave-speed maximum of all ranks (and, after a redo, a flag that is still set: latched)
    smax_reduce_kernel<<<1, 1, 0, c->st>>>(gath, L.bytes, L.tail, P, b.ureg, 1);
    HROM_LAUNCH_CK();
    ++c->nlaunch;
    c->smax_k = c->k;  // the maximum of gamma_k over all ranks is in ureg[2]: the next dt reads it
    if (s->step_hybrid) {
      const Win& W = c->win;
      slab_row_apply<<<1, 128, 0, c->st>>>(gath, L.bytes, L.row, P, W, c->slot_of(c->k), b.C, b.Clo, kMaxSlots);
      HROM_LAUNCH_CK();
      ++c->nlaunch;
    }
    const int64_t k = c->k;
    if (k < c->w - 1) {
      s->phase = PH_IDLE;
      return HROM_OK;
    }
    if (k == c->w - 1) {
      // bootstrap window Gram on the own rows: Gram shift rho := the newest snapshot (api.cu),
      // then the gathered Gram over EVERY own cell is the window Gram of the own rows
      const size_t pitch = (size_t)g.nsr * TILE * sizeof(double);
      HROM_CK(cudaMemcpy2DAsync(b.rho, pitch, b.ring + (int64_t)c->slot_of(k) * TILE, pitch, TILE * sizeof(double),
                                (size_t)(g.Dp / TILE), cudaMemcpyDeviceToDevice, c->st));
      const Win W = window_of(c, k);
      if ((st = gram_gathered_list(c, W, qk, s->listA, s->cnt + 2, b.eigV, b.Rlo)) != HROM_OK) return st;
      const int ncol = W.nU + 1, n2 = ncol * ncol;
      HROM_CK(cudaMemcpyAsync(send, b.eigV, (size_t)n2 * 8, cudaMemcpyDeviceToDevice, c->st));
      HROM_CK(cudaMemcpyAsync(send + (size_t)n2 * 8, b.Rlo, (size_t)n2 * 8, cudaMemcpyDeviceToDevice, c->st));
      *send_bytes_out = (int64_t)2 * n2 * 8;
      s->phase = PH_BOOT;
      return HROM_OK;
    }
    return begin_update(c, send, send_bytes_out);
  }

  if (s->phase == PH_BOOT) {
    const Win W = window_of(c, c->k);
    const int ncol = W.nU + 1, n2 = ncol * ncol;
    dd_sum_kernel<<<(n2 + 255) / 256, 256, 0, c->st>>>(gath, (int64_t)2 * n2 * 8, 0, P, n2, 0, b.eigV, b.Rlo);
    scatter_gram_kernel<<<1, 1024, 0, c->st>>>(b.eigV, b.Rlo, ncol, W, b.C, b.Clo, kMaxSlots);
    HROM_LAUNCH_CK();
    c->nlaunch += 2;
    c->rebase_k = c->k;
    return begin_update(c, send, send_bytes_out);
  }

  if (s->phase == PH_REBUILD) {  // replay hook: the summed window Gram -> C, eigen-solve, sets of the given S-hat
    const Win W = window_of(c, c->k);
    const int ncol = W.nU + 1, n2 = ncol * ncol;
    dd_sum_kernel<<<(n2 + 255) / 256, 256, 0, c->st>>>(gath, (int64_t)2 * n2 * 8, 0, P, n2, 0, b.eigV, b.Rlo);
    scatter_gram_kernel<<<1, 1024, 0, c->st>>>(b.eigV, b.Rlo, ncol, W, b.C, b.Clo, kMaxSlots);
    HROM_LAUNCH_CK();
    c->nlaunch += 2;
    c->rebase_k = c->k;
    c->eig_win = W;
    c->eig_todo = true;
    if ((st = flush_eigen(c)) != HROM_OK) return st;
    c->win = W;
    c->basis_ready = true;
    s->phase = PH_IDLE;
    return finish_sets(c);
  }

  if (s->phase == PH_SEL) {
    const long long n_g = (long long)std::ceil(c->P.sample_fraction * (double)s->N_g);
    sel_digit_kernel<<<1, 1024, 0, c->st>>>(gath, NBIN * 4, P, s->rank, s->sel_pass, n_g, s->sel);
    HROM_LAUNCH_CK();
    ++c->nlaunch;
    if (s->sel_pass < 5) {
      ++s->sel_pass;
      if ((st = sel_pass(c, s->sel_pass, send)) != HROM_OK) return st;
      *send_bytes_out = NBIN * 4;
      return HROM_OK;
    }
    // S-hat_{k+1} on the own rows, then its edge rows for the neighbours
    uint32_t* S = b.masks + (int64_t)M_S * c->mwords;
    const int r0 = s->hlo, r1 = s->hlo + s->own;
    HROM_CK(cudaMemcpyAsync(b.masks + (int64_t)M_SPREV * c->mwords, S, c->mwords * sizeof(uint32_t),
                            cudaMemcpyDeviceToDevice, c->st));
    sel_mark_kernel<<<grid_for(c, (int64_t)s->own * g.wpr), 256, 0, c->st>>>(g, b.eps, r0, r1, s->sel, S);
    sel_ties_kernel<<<1, 1024, 0, c->st>>>(g, b.eps, r0, r1, s->sel, S);
    HROM_LAUNCH_CK();
    c->nlaunch += 2;
    if (P == 1) {
      s->phase = PH_IDLE;
      return finish_sets(c);
    }
    const size_t eb = (size_t)s->mask_words * 4;
    HROM_CK(cudaMemcpyAsync(send, S + (int64_t)r0 * g.wpr, eb, cudaMemcpyDeviceToDevice, c->st));
    HROM_CK(cudaMemcpyAsync(send + eb, S + (int64_t)(r1 - s->H) * g.wpr, eb, cudaMemcpyDeviceToDevice, c->st));
    *send_bytes_out = (int64_t)2 * eb;
    s->phase = PH_MASK;
    return HROM_OK;
  }

  if (s->phase == PH_MASK) {
    uint32_t* S = b.masks + (int64_t)M_S * c->mwords;
    const size_t eb = (size_t)s->mask_words * 4;
    const int64_t stride = (int64_t)2 * eb;
    if (s->hlo)
      HROM_CK(cudaMemcpyAsync(S, gath + ((s->rank - 1 + P) % P) * stride + eb, eb, cudaMemcpyDeviceToDevice, c->st));
    if (s->hhi)
      HROM_CK(cudaMemcpyAsync(S + (int64_t)(s->hlo + s->own) * g.wpr, gath + ((s->rank + 1) % P) * stride, eb,
                              cudaMemcpyDeviceToDevice, c->st));
    s->phase = PH_IDLE;
    return finish_sets(c);
  }
  return HROM_E_STATE;
}

}  // extern "C"
