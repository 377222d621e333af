// masks.cu -- H8: sampling sets as N-bit bitmaps, warp-ballot stream compaction into
// ascending cell lists, and the top-ceil(fN) indicator selection (radix select on the
// IEEE bit patterns of eps >= 0).
//
// Paper: sampling matrices S-hat, S-tilde, S-breve (Fig. 1), Neighbors /
// union / setdiff, ordering of the pointwise error.
// Readings: A9 (per-stage cross dilations), A18 (fraction mode, ties by ascending
// index), A21 (square seam band).  Everything here is integer work: bit-exact.
#include <cooperative_groups.h>
#include <cmath>
#include "internal.cuh"

namespace cg = cooperative_groups;

namespace hrom {
hrom_status launch_sets(hrom_ctx* c, bool do_select, const double* eps, long long n_g, bool sparse = false,
                        double rre_delta = 0.0, bool use_prev = false);
namespace {

__device__ __forceinline__ int wrapi(int i, int n, int bc, bool* valid) {
  if (bc == 1) {
    i %= n;
    *valid = true;
    return i < 0 ? i + n : i;
  }
  *valid = (i >= 0 && i < n);
  return i;
}

__device__ __forceinline__ uint32_t get_bit(const uint32_t* m, const Geo& g, int i, int j) {
  return (__ldcg(m + (int64_t)j * g.wpr + (i >> 5)) >> (i & 31)) & 1u;
}

// valid-bit mask of word wi in a row
__device__ __forceinline__ uint32_t row_valid(const Geo& g, int wi) {
  const int rem = g.nx - 32 * wi;
  return rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
}

// x-dilation of one word by radius h: OR_{|a|<=h} in[i+a]
__device__ uint32_t xdil_word(const uint32_t* in, const Geo& g, int j, int wi, int h) {
  const uint32_t* row = in + (int64_t)j * g.wpr;
  const uint32_t cur = __ldcg(row + wi);
  if (g.bc == 1 && (g.nx & 31)) {  // periodic with a ragged last word: per-bit
    uint32_t out = 0;
    const uint32_t vm = row_valid(g, wi);
    for (int b = 0; b < 32; ++b) {
      if (!((vm >> b) & 1u)) continue;
      const int i = 32 * wi + b;
      uint32_t any = 0;
      for (int a = -h; a <= h && !any; ++a) {
        bool ok;
        const int ii = wrapi(i + a, g.nx, 1, &ok);
        any = get_bit(in, g, ii, j);
      }
      out |= any << b;
    }
    return out;
  }
  uint32_t prev, next;
  if (g.bc == 1) {
    prev = __ldcg(row + (wi - 1 + g.wpr) % g.wpr);
    next = __ldcg(row + (wi + 1) % g.wpr);
  } else {
    prev = wi > 0 ? __ldcg(row + wi - 1) : 0u;
    next = wi + 1 < g.wpr ? __ldcg(row + wi + 1) : 0u;
  }
  uint32_t out = cur;
  const unsigned long long hi = ((unsigned long long)next << 32) | cur;   // bits of i+a
  const unsigned long long lo = ((unsigned long long)cur << 32) | prev;   // bits of i-a
  for (int a = 1; a <= h; ++a) {
    out |= (uint32_t)(hi >> a);
    out |= (uint32_t)(lo >> (32 - a));
  }
  return out & row_valid(g, wi);
}

// y-dilation of one word by radius h
__device__ __forceinline__ uint32_t ydil_word(const uint32_t* in, const Geo& g, int j, int wi, int h) {
  uint32_t out = 0;
  for (int b = -h; b <= h; ++b) {
    bool ok;
    const int jj = wrapi(j + b, g.ny, g.bcy, &ok);
    if (ok) out |= __ldcg(in + (int64_t)jj * g.wpr + wi);
  }
  return out;
}

// ---------------- H8 + set construction + seam-filter tables: one cooperative kernel ----------------
// Phases (grid barriers between them): [select: eps > 0 bitmap -> ordered compaction ->
// 11-bit radix select of the n_g-th largest IEEE pattern (6 passes) -> mark S-hat, ties by
// ascending cell] -> x/y dilations (B, T, A2, A1) -> ordered compaction of the 5 sets ->
// seam-filter halo (cells within the largest Shapiro radius of B, not in B), its compaction,
// the cell -> compact index map and the stencil tables used by filter_kernel.
constexpr int ST_T = 1024;
constexpr int RADIX = 11, NBIN = 1 << RADIX;

struct SetsArgs {
  Geo g;
  int do_select;
  int use_prev;            // no selection, but M_SPREV holds the previous S-hat: build the churn lists from it
  const double* eps;
  long long n_g;
  int rre;                 // 1: RRE-delta rule instead of n_g
  unsigned long long rre_dm;  // delta = rre_dm * 2^-rre_sh exactly (rre_dm < 2^53)
  int rre_sh;
  unsigned long long* hsum;  // 3 x 2 x NBIN exact bucket sums (RRE mode)
  const int32_t* extra;      // cells OR'ed into S-hat after the selection (ODEIM points)
  int n_extra;
  int halo, band, rmax;
  uint32_t* masks;     // M_COUNT masks of mwords
  int64_t mwords;
  int32_t* lists;      // L_COUNT lists of N
  int32_t* counts;     // [l] sizes; [8] #eps > 0
  double* sel_val;
  int32_t* sel_cell;
  int32_t* blk;        // per-block scratch (>= 8 * grid)
  int32_t* hist;       // 3 * NBIN
  int32_t* idx;        // cell -> compact filter index
  int32_t* tab;        // stencil tables (14 N)
  long long* tdbg;     // debug timestamps [40..63]
  const int32_t* cand; // nullable: sorted candidate cells for eps > 0 (T list of the current sets)
  const int32_t* ncand;
};

__device__ __forceinline__ void sstamp(long long* t, int& i) {
  if (t && blockIdx.x == 0 && threadIdx.x == 0 && i < 64) {
    long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    t[i] = gt;
  }
  ++i;
}

struct BlockRange {
  int64_t w0, w1;  // this thread's contiguous sub-range
};
__device__ __forceinline__ BlockRange thread_range(int64_t n) {
  const int64_t bchunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t tchunk = (bchunk + blockDim.x - 1) / blockDim.x;
  const int64_t b0 = (int64_t)blockIdx.x * bchunk, b1 = min(b0 + bchunk, n);
  BlockRange r;
  r.w0 = min(b0 + (int64_t)threadIdx.x * tchunk, b1);
  r.w1 = min(r.w0 + tchunk, b1);
  return r;
}

// exclusive block scan of one int per thread (returns exclusive prefix, *total = block sum)
__device__ __forceinline__ int block_excl_scan(int v, int* total, int* sbuf) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int x = v;
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += t;
  }
  __syncthreads();
  if (lane == 31) sbuf[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int y = lane < nw ? sbuf[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, y, o);
      if (lane >= o) y += t;
    }
    sbuf[lane] = y;
  }
  __syncthreads();
  *total = sbuf[nw - 1];
  const int wpre = warp ? sbuf[warp - 1] : 0;
  return wpre + x - v;
}

// offset of this block among all blocks' counts blk[q * G + b], and the total (read via L2):
// one count per thread and a block scan (gridDim.x <= blockDim.x), not a serial loop of loads
__device__ __forceinline__ void block_offset(const int32_t* blk, int q, int* off, int* tot, int* sbuf) {
  __shared__ int s_off;
  const int v = threadIdx.x < gridDim.x ? __ldcg(blk + q * gridDim.x + threadIdx.x) : 0;
  int t;
  const int ex = block_excl_scan(v, &t, sbuf);
  if (threadIdx.x == blockIdx.x) s_off = ex;
  __syncthreads();
  *off = s_off;
  *tot = t;
  __syncthreads();
}

// ---- warp-cooperative ordered compaction of a block's word range [b0, b1) ----
// Each warp owns a contiguous sub-range; words are read once per lane-stride for the count and
// once per word (broadcast) for the write, where lane b emits bit b: coalesced list/value I/O.
__device__ __forceinline__ void warp_range(int64_t b0, int64_t b1, int64_t* w0, int64_t* w1) {
  const int nwarp = blockDim.x >> 5, warp = threadIdx.x >> 5;
  const int64_t wc = (b1 - b0 + nwarp - 1) / nwarp;
  *w0 = min(b0 + (int64_t)warp * wc, b1);
  *w1 = min(*w0 + wc, b1);
}
// per-warp counts into wcnt[warp]; returns the block total (all threads)
__device__ __forceinline__ int blk_count(const uint32_t* M, int64_t b0, int64_t b1, int* wcnt) {
  int64_t w0, w1;
  warp_range(b0, b1, &w0, &w1);
  const int lane = threadIdx.x & 31;
  int c = 0;
  for (int64_t w = w0 + lane; w < w1; w += 32) c += __popc(__ldcg(M + w));
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  __syncthreads();
  if (lane == 0) wcnt[threadIdx.x >> 5] = c;
  __syncthreads();
  int t = 0;
  for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += wcnt[k];
  return t;
}
// write the set bits of [b0, b1) in order from position base (block offset); flat: word w
// covers cells 32w.. (else row-padded words); optional value gather and index map
__device__ __forceinline__ void blk_write(const uint32_t* M, int64_t b0, int64_t b1, int base, const int* wcnt,
                                          const Geo& g, bool flat, int32_t* __restrict__ list,
                                          const double* __restrict__ src, double* __restrict__ vals,
                                          int32_t* __restrict__ idx, int idx_base) {
  int64_t w0, w1;
  warp_range(b0, b1, &w0, &w1);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int pos = base;
  for (int k = 0; k < warp; ++k) pos += wcnt[k];
  for (int64_t wb = w0; wb < w1; wb += 32) {
    // 32 words per coalesced load, broadcast one by one (no load in the dependent chain)
    const uint32_t mine = wb + lane < w1 ? __ldcg(M + wb + lane) : 0u;
    const int nwk = (int)min((int64_t)32, w1 - wb);
    int jrow = flat ? 0 : (int)wb / g.wpr, wcol = flat ? (int)wb : (int)wb - jrow * g.wpr;  // no 64-bit division
    for (int k = 0; k < nwk; ++k) {
      const uint32_t bits = __shfl_sync(0xffffffffu, mine, k);
      if ((bits >> lane) & 1u) {
        const int p = pos + __popc(bits & ((1u << lane) - 1u));
        const int cell = (flat ? 32 * wcol : jrow * g.nx + 32 * wcol) + lane;
        list[p] = cell;
        if (vals) vals[p] = src[cell];
        if (idx) idx[cell] = idx_base + p;
      }
      pos += __popc(bits);
      if (++wcol == g.wpr && !flat) {
        wcol = 0;
        ++jrow;
      }
    }
  }
}


// ---- RRE-delta selection: exact integer arithmetic (reading A35) ----
// A positive double is m 2^(max(be,1) - 1) in units of 2^-1074 (m < 2^53 an integer).  Radix
// bucket b0 = pattern bits 63..53 holds the biased exponents 2 b0 and 2 b0 + 1, so with the
// bucket unit 2^ub, ub = max(2 b0 - 1, 0), every value of the bucket is the integer m or 2m.
// Pass 0 (the bucket b0) works on big naturals (T = sum of all eps, R = ceil(delta T)); the
// later passes stay inside one bucket, where every partial sum is < 2^80 units: 128-bit.
constexpr int RRE_LIMBS = 72;  // 2304 bits > 2^(2046 + 80 + 53)
typedef unsigned __int128 u128;
__device__ __forceinline__ int rre_ub(unsigned b0) { return b0 ? 2 * (int)b0 - 1 : 0; }
__device__ __forceinline__ unsigned long long rre_contrib(unsigned long long bb) {
  const int be = (int)(bb >> 52);
  const unsigned long long f = bb & ((1ull << 52) - 1ull);
  const unsigned long long m = be ? (f | (1ull << 52)) : f;
  return m << ((be ? be - 1 : 0) - rre_ub((unsigned)(bb >> 53)));
}
__device__ __forceinline__ u128 shfl_up_u128(u128 v, int o) {
  const unsigned long long lo = __shfl_up_sync(0xffffffffu, (unsigned long long)v, o);
  const unsigned long long hi = __shfl_up_sync(0xffffffffu, (unsigned long long)(v >> 64), o);
  return ((u128)hi << 64) | lo;
}
// exclusive block scan of one u128 per thread
__device__ __forceinline__ u128 block_excl_scan_u128(u128 v, u128* sbuf) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  u128 x = v;
  for (int o = 1; o < 32; o <<= 1) {
    const u128 t = shfl_up_u128(x, o);
    if (lane >= o) x += t;
  }
  __syncthreads();
  if (lane == 31) sbuf[warp] = x;
  __syncthreads();
  if (warp == 0) {
    u128 y = lane < nw ? sbuf[lane] : (u128)0;
    for (int o = 1; o < 32; o <<= 1) {
      const u128 t = shfl_up_u128(y, o);
      if (lane >= o) y += t;
    }
    sbuf[lane] = y;
  }
  __syncthreads();
  const u128 wpre = warp ? sbuf[warp - 1] : (u128)0;
  __syncthreads();
  return wpre + x - v;
}
// Pass-0 pick of the RRE rule, thread 0 of the block (identical in every block).
// lo/hi: the 1024 bucket sums of pass 0 (sum = hi 2^32 + lo, units 2^ub(b)); acc: T in
// non-normalised 32-bit limbs (u64 each).  Returns the bucket b0 whose cumulative sum (from
// the top) first reaches R = ceil(delta T), and D = ceil((R - sum above b0) / 2^ub(b0)).
__device__ void rre_pick0(const unsigned long long* lo, const unsigned long long* hi, const unsigned long long* acc,
                          unsigned long long dm, int sh, uint32_t* big, int* b_out, u128* D_out) {
  uint32_t T[RRE_LIMBS];
  unsigned long long carry = 0;
  for (int i = 0; i < RRE_LIMBS; ++i) {
    const unsigned long long t = acc[i] + carry;
    T[i] = (uint32_t)t;
    carry = t >> 32;
  }
  // P = T dm (dm < 2^53), in place over T's limbs, then R = ceil(P / 2^sh) into big
  {
    u128 cy = 0;
    for (int i = 0; i < RRE_LIMBS; ++i) {
      const u128 t = (u128)T[i] * dm + cy;
      T[i] = (uint32_t)t;
      cy = t >> 32;
    }
  }
  const int q = sh >> 5, s = sh & 31;
  bool sticky = false;
  for (int i = 0; i < RRE_LIMBS; ++i) {
    if (i < q) sticky |= T[i] != 0u;
  }
  if (s) sticky |= (q < RRE_LIMBS) && (T[q] & ((1u << s) - 1u)) != 0u;
  for (int i = 0; i < RRE_LIMBS; ++i) {
    const int k = i + q;
    const uint32_t a0 = k < RRE_LIMBS ? T[k] : 0u, a1 = k + 1 < RRE_LIMBS ? T[k + 1] : 0u;
    big[i] = s ? (a0 >> s) | (a1 << (32 - s)) : a0;
  }
  if (sticky)
    for (int i = 0; i < RRE_LIMBS; ++i)
      if (++big[i] != 0u) break;
  int top = RRE_LIMBS - 1;
  while (top > 0 && big[top] == 0u) --top;
  // descend the buckets: Dif = R - (sum of the buckets above) > 0
  for (int b = 1023; b >= 0; --b) {
    if (lo[b] == 0ull && hi[b] == 0ull) continue;
    const int ub = rre_ub((unsigned)b), L = ub >> 5;
    const u128 sb = (((u128)hi[b]) << 32) + lo[b];
    const u128 s2 = sb << (ub & 31);  // < 2^111
    uint32_t p[4];
    for (int k = 0; k < 4; ++k) p[k] = (uint32_t)(s2 >> (32 * k));
    int cmp = 0;  // sign of (S_b - Dif)
    if (top > L + 3) cmp = -1;
    else {
      for (int i = L + 3; i >= L && cmp == 0; --i) {
        const uint32_t d = big[i];
        if (p[i - L] != d) cmp = p[i - L] > d ? 1 : -1;
      }
      if (cmp == 0) {
        cmp = 1;  // S_b >= Dif unless Dif has bits below limb L
        for (int i = 0; i < L; ++i)
          if (big[i]) cmp = -1;
      }
    }
    if (cmp >= 0) {  // found: D = ceil(Dif / 2^ub)
      u128 V = 0;
      for (int i = min(top, L + 3); i >= L; --i) V = (V << 32) | big[i];
      const int sb2 = ub & 31;
      bool st = sb2 ? (V & ((((u128)1) << sb2) - 1)) != 0 : false;
      for (int i = 0; i < L; ++i) st |= big[i] != 0u;
      *D_out = (V >> sb2) + (st ? 1 : 0);
      *b_out = b;
      return;
    }
    // Dif -= S_b
    unsigned long long br = 0;
    for (int i = L; i < RRE_LIMBS; ++i) {
      const unsigned long long sub = (i - L < 4 ? p[i - L] : 0u) + br;
      const unsigned long long d = big[i];
      big[i] = (uint32_t)(d - sub);
      br = d < sub ? 1ull : 0ull;
      if (i - L >= 3 && br == 0) break;
    }
    while (top > 0 && big[top] == 0u) --top;
  }
  *b_out = -1;  // R > T: cannot happen for delta <= 1
  *D_out = 0;
}

__global__ void __launch_bounds__(ST_T) sets_kernel(SetsArgs a) {
  cg::grid_group grid = cg::this_grid();
  const Geo& g = a.g;
  const int64_t N = g.N, mw = a.mwords, nw = (int64_t)g.ny * g.wpr;
  uint32_t* S = a.masks + (int64_t)M_S * mw;
  uint32_t* TMP = a.masks + (int64_t)M_TMP * mw;
  uint32_t* FLAT = a.masks + (int64_t)M_TMP2 * mw;
  uint32_t* HM = a.masks + (int64_t)M_H * mw;
  uint32_t* SPREV = a.masks + (int64_t)M_SPREV * mw;
  uint32_t* MADD = a.masks + (int64_t)M_ADD * mw;
  uint32_t* MREM = a.masks + (int64_t)M_REM * mw;
  __shared__ int sbuf[32];
  __shared__ int wcnt[32];
  __shared__ int shist[NBIN];
  __shared__ int s_digit, s_above;
  __shared__ unsigned long long s_lo[NBIN], s_hi[NBIN], s_acc[RRE_LIMBS];
  __shared__ uint32_t s_big[RRE_LIMBS];
  __shared__ u128 s_u128[32];
  __shared__ u128 s_D;
  const int tid = threadIdx.x;
  const int G = gridDim.x;
  int ts = 40;
  sstamp(a.tdbg, ts);
  // ================= select =================
  if (a.do_select) {
    const int64_t fw = (N + 31) / 32;
    // A1: eps > 0 bitmap (flat words; one warp ballot per word, coalesced), zero S-hat, count.
    // Sparse indicator (after a hybrid step eps is nonzero only on S-hat u B, i.e. the T list of
    // the current sets): the candidates are that sorted list instead of all N cells.
    const int ncand = a.cand ? __ldcg(a.ncand) : 0;
    const int64_t cchunk = ((int64_t)ncand + G - 1) / G;
    const int64_t c0 = min((int64_t)blockIdx.x * cchunk, (int64_t)ncand), c1 = min(c0 + cchunk, (int64_t)ncand);
    if (a.cand) {
      int mine = 0;
      const int64_t tch = (c1 - c0 + blockDim.x - 1) / blockDim.x;
      const int64_t t0 = min(c0 + tid * tch, c1), t1 = min(t0 + tch, c1);
      for (int64_t t = t0; t < t1; ++t) mine += a.eps[__ldcg(a.cand + t)] > 0.0;
      const BlockRange rs = thread_range(nw);
      for (int64_t w = rs.w0; w < rs.w1; ++w) {
        SPREV[w] = S[w];
        S[w] = 0u;
      }
      int tot;
      block_excl_scan(mine, &tot, sbuf);
      if (tid == 0) a.blk[0 * G + blockIdx.x] = tot;
    } else {
      const int64_t bchunk = (fw + G - 1) / G;
      const int64_t b0 = min((int64_t)blockIdx.x * bchunk, fw), b1 = min(b0 + bchunk, fw);
      const int lane = tid & 31, warp = tid >> 5;
      int mine = 0;
      constexpr int U = 8;  // words per warp iteration: U independent loads in flight
      const int nwarp = blockDim.x >> 5;
      for (int64_t w = b0 + (int64_t)warp * U; w < b1; w += (int64_t)nwarp * U) {
        double e[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t n = 32 * (w + u) + lane;
          e[u] = (w + u < b1 && n < N) ? a.eps[n] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t bits = __ballot_sync(0xffffffffu, e[u] > 0.0);
          if (lane == 0 && w + u < b1) {
            FLAT[w + u] = bits;
            mine += __popc(bits);
          }
        }
      }
      const BlockRange rs = thread_range(nw);
      for (int64_t w = rs.w0; w < rs.w1; ++w) {
        SPREV[w] = S[w];  // the churn of S-hat feeds the incremental gathered Gram (G7)
        S[w] = 0u;
      }
      int tot;
      block_excl_scan(mine, &tot, sbuf);
      if (tid == 0) a.blk[0 * G + blockIdx.x] = tot;
    }
    grid.sync();
  sstamp(a.tdbg, ts);
    // A2: ordered compaction of eps > 0 -> (sel_cell, sel_val)
    if (a.cand) {
      int off, tot;
      block_offset(a.blk, 0, &off, &tot, sbuf);
      const int64_t tch = (c1 - c0 + blockDim.x - 1) / blockDim.x;
      const int64_t t0 = min(c0 + tid * tch, c1), t1 = min(t0 + tch, c1);
      int mine = 0;
      for (int64_t t = t0; t < t1; ++t) mine += a.eps[__ldcg(a.cand + t)] > 0.0;
      int btot;
      int pos = off + block_excl_scan(mine, &btot, sbuf);
      for (int64_t t = t0; t < t1; ++t) {
        const int cell = __ldcg(a.cand + t);
        const double e = a.eps[cell];
        if (e > 0.0) {
          a.sel_cell[pos] = cell;
          a.sel_val[pos] = e;
          ++pos;
        }
      }
      if (blockIdx.x == 0 && tid == 0) a.counts[8] = tot;
      for (int i = blockIdx.x * blockDim.x + tid; i < 2 * NBIN; i += G * blockDim.x) a.hist[i] = 0;
      if (a.rre)  // the sum buffers of passes 0 and 1
        for (int i = blockIdx.x * blockDim.x + tid; i < 4 * NBIN; i += G * blockDim.x) a.hsum[i] = 0ull;
    } else {
      const int64_t bchunk = (fw + G - 1) / G;
      const int64_t b0 = min((int64_t)blockIdx.x * bchunk, fw), b1 = min(b0 + bchunk, fw);
      int off, tot;
      block_offset(a.blk, 0, &off, &tot, sbuf);
      blk_count(FLAT, b0, b1, wcnt);
      blk_write(FLAT, b0, b1, off, wcnt, g, true, a.sel_cell, a.eps, a.sel_val, nullptr, 0);
      if (blockIdx.x == 0 && tid == 0) a.counts[8] = tot;
      // zero the first two histogram buffers
      for (int i = blockIdx.x * blockDim.x + tid; i < 2 * NBIN; i += G * blockDim.x) a.hist[i] = 0;
      if (a.rre)  // the sum buffers of passes 0 and 1
        for (int i = blockIdx.x * blockDim.x + tid; i < 4 * NBIN; i += G * blockDim.x) a.hsum[i] = 0ull;
    }
    grid.sync();
  sstamp(a.tdbg, ts);
    const int total = __ldcg(a.counts + 8);
    const int ng = (int)(a.n_g < total ? a.n_g : total);
    bool thresh = a.rre ? total > 0 : a.n_g < total;
    unsigned long long prefix = 0ull;
    int rem = a.rre ? 0 : ng;
    // contiguous block chunk of the compacted values
    const int64_t vchunk = ((int64_t)total + G - 1) / G;
    const int64_t v0 = min((int64_t)blockIdx.x * vchunk, (int64_t)total), v1 = min(v0 + vchunk, (int64_t)total);
    if (a.rre && thresh) {
      // RRE-delta: the same 6 radix passes over the IEEE patterns, on exact per-digit sums
      // instead of counts; the target is the remaining sum D (units of the pass-0 bucket)
      u128 Drem = 0;
      for (int p = 0; p < 6; ++p) {
        const int shift = p < 5 ? 53 - RADIX * p : 0;
        const int width = (shift == 0) ? 9 : RADIX;
        const unsigned long long hm = (p == 0) ? 0ull : (~0ull << (shift + width));
        for (int i = tid; i < NBIN; i += blockDim.x) s_lo[i] = s_hi[i] = 0ull;
        __syncthreads();
        for (int64_t t = v0 + tid; t < v1; t += blockDim.x) {
          const unsigned long long bb = (unsigned long long)__double_as_longlong(a.sel_val[t]);
          if ((bb & hm) == prefix) {
            const unsigned long long cv = rre_contrib(bb);
            const int bin = (int)((bb >> shift) & (NBIN - 1));
            atomicAdd(&s_lo[bin], cv & 0xffffffffull);
            if (cv >> 32) atomicAdd(&s_hi[bin], cv >> 32);
          }
        }
        __syncthreads();
        unsigned long long* gs = a.hsum + (p % 3) * 2 * NBIN;
        for (int i = tid; i < NBIN; i += blockDim.x) {
          if (s_lo[i]) atomicAdd(gs + i, s_lo[i]);
          if (s_hi[i]) atomicAdd(gs + NBIN + i, s_hi[i]);
        }
        if (blockIdx.x == 0)
          for (int i = tid; i < 2 * NBIN; i += blockDim.x) a.hsum[((p + 1) % 3) * 2 * NBIN + i] = 0ull;
        grid.sync();
  sstamp(a.tdbg, ts);
        for (int i = tid; i < NBIN; i += blockDim.x) {
          s_lo[i] = __ldcg(gs + i);
          s_hi[i] = __ldcg(gs + NBIN + i);
        }
        __syncthreads();
        if (p == 0) {
          for (int i = tid; i < RRE_LIMBS; i += blockDim.x) s_acc[i] = 0ull;
          __syncthreads();
          for (int b = tid; b < 1024; b += blockDim.x) {
            if (s_lo[b] == 0ull && s_hi[b] == 0ull) continue;
            const int ub = rre_ub((unsigned)b), L = ub >> 5;
            const u128 s2 = ((((u128)s_hi[b]) << 32) + s_lo[b]) << (ub & 31);
            for (int k = 0; k < 4; ++k) {
              const uint32_t piece = (uint32_t)(s2 >> (32 * k));
              if (piece) atomicAdd(&s_acc[L + k], (unsigned long long)piece);
            }
          }
          __syncthreads();
          if (tid == 0) {
            int b0;
            u128 D;
            rre_pick0(s_lo, s_hi, s_acc, a.rre_dm, a.rre_sh, s_big, &b0, &D);
            s_digit = b0;
            s_D = D;
          }
          __syncthreads();
          if (s_digit < 0) {
            thresh = false;  // R > T (delta > 1): every eps > 0 is selected
            break;
          }
          prefix = (unsigned long long)s_digit << 53;
          Drem = s_D;
          __syncthreads();
        } else {
          constexpr int PER = NBIN / ST_T;
          u128 sq[PER];
          u128 mine = 0;
          for (int q = 0; q < PER; ++q) {
            const int bin = NBIN - 1 - (tid * PER + q);
            sq[q] = (((u128)s_hi[bin]) << 32) + s_lo[bin];
            mine += sq[q];
          }
          u128 above = block_excl_scan_u128(mine, s_u128);
          for (int q = 0; q < PER; ++q) {
            if (above < Drem && above + sq[q] >= Drem) {
              s_digit = NBIN - 1 - (tid * PER + q);
              s_D = above;
            }
            above += sq[q];
          }
          __syncthreads();
          prefix |= (unsigned long long)s_digit << shift;
          Drem -= s_D;
          __syncthreads();
        }
      }
      if (thresh) {
        const unsigned long long vt = rre_contrib(prefix);  // tau in the pass-0 bucket's units
        rem = (int)((Drem + vt - 1) / vt);
      }
    } else if (thresh) {
      for (int p = 0; p < 6; ++p) {
        const int shift = p < 5 ? 53 - RADIX * p : 0;  // 53, 42, 31, 20, 9, 0
        const int width = (shift == 0) ? 9 : RADIX;
        const unsigned long long hm = (p == 0) ? 0ull : (~0ull << (shift + width));
        for (int i = tid; i < NBIN; i += blockDim.x) shist[i] = 0;
        __syncthreads();
        for (int64_t t = v0 + tid; t < v1; t += blockDim.x) {
          const unsigned long long bb = (unsigned long long)__double_as_longlong(a.sel_val[t]);
          if ((bb & hm) == prefix) atomicAdd(&shist[(bb >> shift) & (NBIN - 1)], 1);
        }
        __syncthreads();
        int32_t* gh = a.hist + (p % 3) * NBIN;
        for (int i = tid; i < NBIN; i += blockDim.x)
          if (shist[i]) atomicAdd(gh + i, shist[i]);
        if (blockIdx.x == 0)  // buffer of pass p+1 (last read in pass p-2's pick)
          for (int i = tid; i < NBIN; i += blockDim.x) a.hist[((p + 1) % 3) * NBIN + i] = 0;
        grid.sync();
  sstamp(a.tdbg, ts);
        // pick (every block, identical): highest digit d with #(> d) < rem <= #(>= d)
        {
          constexpr int PER = NBIN / ST_T;  // bins per thread, top-down
          int cnt[PER];
          int mine = 0;
          for (int q = 0; q < PER; ++q) {
            const int bin = NBIN - 1 - (tid * PER + q);
            cnt[q] = __ldcg(gh + bin);
            mine += cnt[q];
          }
          int btot;
          int above = block_excl_scan(mine, &btot, sbuf);  // count in higher bins
          for (int q = 0; q < PER; ++q) {
            if (above < rem && above + cnt[q] >= rem) {
              s_digit = NBIN - 1 - (tid * PER + q);
              s_above = above;
            }
            above += cnt[q];
          }
          __syncthreads();
          prefix |= (unsigned long long)s_digit << shift;
          rem -= s_above;
          __syncthreads();
        }
      }
    }
    // A3: ties at tau by ascending cell (the compacted array is in cell order)
    const unsigned long long tau = prefix;
    {
      int mine = 0;
      if (thresh)
        for (int64_t t = v0 + tid; t < v1; t += blockDim.x)
          mine += ((unsigned long long)__double_as_longlong(a.sel_val[t]) == tau);
      int btot;
      block_excl_scan(mine, &btot, sbuf);
      if (tid == 0) a.blk[1 * G + blockIdx.x] = btot;
    }
    grid.sync();
  sstamp(a.tdbg, ts);
    {
      int off, tot;
      block_offset(a.blk, 1, &off, &tot, sbuf);
      // per-thread contiguous sub-chunk keeps the tie order = cell order
      const int64_t len = v1 - v0;
      const int64_t tch = (len + blockDim.x - 1) / blockDim.x;
      const int64_t t0 = min(v0 + tid * tch, v1), t1 = min(t0 + tch, v1);
      int mine = 0;
      if (thresh)
        for (int64_t t = t0; t < t1; ++t) mine += ((unsigned long long)__double_as_longlong(a.sel_val[t]) == tau);
      int btot;
      int tie_rank = off + block_excl_scan(mine, &btot, sbuf);
      for (int64_t t = t0; t < t1; ++t) {
        const unsigned long long bb = (unsigned long long)__double_as_longlong(a.sel_val[t]);
        bool sel = !thresh || bb > tau;
        if (thresh && bb == tau) {
          sel = tie_rank < rem;
          ++tie_rank;
        }
        if (sel) {
          const int64_t cell = a.sel_cell[t];
          const int ci = (int)cell, j = ci / g.nx, i = ci - j * g.nx;
          atomicOr(&S[(int64_t)j * g.wpr + (i >> 5)], 1u << (i & 31));
        }
      }
      if (blockIdx.x == 0)  // S-hat = G u P (ODEIM points)
        for (int q = tid; q < a.n_extra; q += blockDim.x) {
          const int ci = __ldg(a.extra + q), j = ci / g.nx, i = ci - j * g.nx;
          atomicOr(&S[(int64_t)j * g.wpr + (i >> 5)], 1u << (i & 31));
        }
    }
    grid.sync();
  sstamp(a.tdbg, ts);
  }
  // ================= sets =================
  uint32_t* B = a.masks + (int64_t)M_B * mw;
  uint32_t* T = a.masks + (int64_t)M_T * mw;
  uint32_t* A2 = a.masks + (int64_t)M_A2 * mw;
  uint32_t* A1 = a.masks + (int64_t)M_A1 * mw;
  {
    const BlockRange r = thread_range(nw);
    for (int64_t w = r.w0; w < r.w1; ++w) {
      const int wq = (int)w, jq = wq / g.wpr;
      // band < 0: B = every cell off S-hat (whole-domain filter)
      TMP[w] = a.band < 0 ? row_valid(g, wq - jq * g.wpr) : xdil_word(S, g, jq, wq - jq * g.wpr, a.band);
      HM[w] = 0u;
      const uint32_t sn = __ldcg(S + w), sp = (a.do_select || a.use_prev) ? SPREV[w] : sn;
      MADD[w] = sn & ~sp;
      MREM[w] = sp & ~sn;
    }
  }
  grid.sync();
  sstamp(a.tdbg, ts);
  {
    const BlockRange r = thread_range(nw);
    for (int64_t w = r.w0; w < r.w1; ++w) {
      const int j = (int)w / g.wpr, wi = (int)w - j * g.wpr;
      const uint32_t sq = (g.dim == 2 && a.band >= 0) ? ydil_word(TMP, g, j, wi, a.band) : __ldcg(TMP + w);
      const uint32_t sv = __ldcg(S + w);
      B[w] = sq & ~sv;
      T[w] = sq | sv;
    }
  }
  grid.sync();
  sstamp(a.tdbg, ts);
  for (int q = 0; q < 2; ++q) {
    const uint32_t* cin = q == 0 ? T : A2;
    uint32_t* cout_ = q == 0 ? A2 : A1;
    const BlockRange r = thread_range(nw);
    for (int64_t w = r.w0; w < r.w1; ++w) {
      const int j = (int)w / g.wpr, wi = (int)w - j * g.wpr;
      uint32_t o = xdil_word(cin, g, j, wi, a.halo);
      if (g.dim == 2) o |= ydil_word(cin, g, j, wi, a.halo);
      cout_[w] = o;
    }
    grid.sync();
  sstamp(a.tdbg, ts);
  }
  // ordered compaction of S, B, T, A2, A1 and the S-hat churn (entering / leaving cells), all
  // seven at once: each warp loads its words of the seven masks once (kept in registers when the
  // warp's range is <= 32 words), per-warp counts stay in shared memory across the grid barrier
  const int64_t rchunk = (nw + G - 1) / G;
  const int64_t rb0 = min((int64_t)blockIdx.x * rchunk, nw), rb1 = min(rb0 + rchunk, nw);
  constexpr int NSET = 7;
  const int mk[NSET] = {M_S, M_B, M_T, M_A2, M_A1, M_ADD, M_REM};
  const int lk[NSET] = {L_S, L_B, L_T, L_A2, L_A1, L_ADD, L_REM};
  __shared__ int wc5[NSET][32];
  __shared__ int soff5[NSET], stot5[NSET];
  // active 32 x 8 tiles of A1 (2-D): tile (bx, by) <-> words A1[(8 by + r) * wpr + bx], r < 8
  const int ntile = g.dim == 2 ? g.wpr * ((g.ny + 7) / 8) : 0;
  const int64_t tchunk = ((int64_t)ntile + G - 1) / G;
  const int64_t tb0 = min((int64_t)blockIdx.x * tchunk, (int64_t)ntile), tb1 = min(tb0 + tchunk, (int64_t)ntile);
  const int64_t ttch = (tb1 - tb0 + blockDim.x - 1) / blockDim.x;
  const int64_t tt0 = min(tb0 + tid * ttch, tb1), tt1 = min(tt0 + ttch, tb1);
  auto tile_active = [&](int64_t t) -> bool {
    const int bx = (int)(t % g.wpr), by = (int)(t / g.wpr);
    uint32_t o = 0u;
    for (int r = 0; r < 8 && 8 * by + r < g.ny; ++r) o |= __ldcg(a.masks + (int64_t)M_A1 * mw + (int64_t)(8 * by + r) * g.wpr + bx);
    return o != 0u;
  };
  int tmine = 0, texcl = 0;
  if (g.dim == 2) {
    for (int64_t t = tt0; t < tt1; ++t) tmine += tile_active(t);
    int tbt;
    texcl = block_excl_scan(tmine, &tbt, sbuf);
    if (tid == 0) a.blk[15 * G + blockIdx.x] = tbt;
  }
  {
    int64_t ww0, ww1;
    warp_range(rb0, rb1, &ww0, &ww1);
    const int lane = tid & 31, warp = tid >> 5;
    const bool fast = ww1 - ww0 <= 32;  // uniform: every warp gets the same range length
    uint32_t wd[NSET];
    int c5[NSET];
#pragma unroll
    for (int m = 0; m < NSET; ++m) {
      wd[m] = (fast && ww0 + lane < ww1) ? __ldcg(a.masks + (int64_t)mk[m] * mw + ww0 + lane) : 0u;
      c5[m] = __popc(wd[m]);
    }
    if (!fast)
#pragma unroll
      for (int m = 0; m < NSET; ++m)
        for (int64_t w = ww0 + lane; w < ww1; w += 32) c5[m] += __popc(__ldcg(a.masks + (int64_t)mk[m] * mw + w));
#pragma unroll
    for (int m = 0; m < NSET; ++m) {
      for (int o = 16; o > 0; o >>= 1) c5[m] += __shfl_xor_sync(0xffffffffu, c5[m], o);
      if (lane == 0) wc5[m][warp] = c5[m];
    }
    __syncthreads();
    if (tid < NSET) {
      int t = 0;
      for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += wc5[tid][k];
      a.blk[(8 + tid) * G + blockIdx.x] = t;
    }
    grid.sync();
    sstamp(a.tdbg, ts);
    if (warp < NSET) {  // warp m: this block's offset in list m and its total
      int o = 0, t = 0;
      for (int b = lane; b < G; b += 32) {
        const int v = __ldcg(a.blk + (8 + warp) * G + b);
        if (b < (int)blockIdx.x) o += v;
        t += v;
      }
      for (int q = 16; q > 0; q >>= 1) {
        o += __shfl_xor_sync(0xffffffffu, o, q);
        t += __shfl_xor_sync(0xffffffffu, t, q);
      }
      if (lane == 0) {
        soff5[warp] = o;
        stot5[warp] = t;
      }
    }
    __syncthreads();
#pragma unroll
    for (int m = 0; m < NSET; ++m) {
      if (g.dim == 2 && (lk[m] == L_A2 || lk[m] == L_A1)) {  // 2-D stages read the bitmaps, not the lists
        if (blockIdx.x == 0 && tid == 0) a.counts[lk[m]] = stot5[m];
        continue;
      }
      int pos = soff5[m];
      for (int k = 0; k < warp; ++k) pos += wc5[m][k];
      int32_t* L = a.lists + (int64_t)lk[m] * N;
      int32_t* idx = lk[m] == L_B ? a.idx : nullptr;
      for (int64_t wb = ww0; wb < ww1; wb += 32) {
        const uint32_t mine = fast ? wd[m] : (wb + lane < ww1 ? __ldcg(a.masks + (int64_t)mk[m] * mw + wb + lane) : 0u);
        const int nwk = (int)min((int64_t)32, ww1 - wb);
        int jrow = (int)wb / g.wpr, wcol = (int)wb - jrow * g.wpr;  // tracked incrementally
        for (int k = 0; k < nwk; ++k) {
          const uint32_t bits = __shfl_sync(0xffffffffu, mine, k);
          if ((bits >> lane) & 1u) {
            const int p = pos + __popc(bits & ((1u << lane) - 1u));
            const int cell = jrow * g.nx + 32 * wcol + lane;
            L[p] = cell;
            if (idx) idx[cell] = p;
          }
          pos += __popc(bits);
          if (++wcol == g.wpr) {
            wcol = 0;
            ++jrow;
          }
        }
      }
      if (blockIdx.x == 0 && tid == 0) a.counts[lk[m]] = stot5[m];
    }
    if (g.dim == 2) {  // the tile list (into the A2 list, unused in 2-D)
      int off, tot;
      block_offset(a.blk, 15, &off, &tot, sbuf);
      int pos = off + texcl;
      int32_t* TL = a.lists + (int64_t)L_A2 * N;
      for (int64_t t = tt0; t < tt1; ++t)
        if (tile_active(t)) TL[pos++] = (int32_t)t;
      if (blockIdx.x == 0 && tid == 0) a.counts[10] = tot;
    }
  }
  grid.sync();
  sstamp(a.tdbg, ts);
  // ================= seam-filter halo, index map, stencil tables =================
  if (a.rmax <= 0) return;
  const int nb = __ldcg(a.counts + L_B);
  const int32_t* LB = a.lists + (int64_t)L_B * N;
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + tid, gstride = (int64_t)G * blockDim.x;
  for (int64_t t = gtid; t < nb; t += gstride) {
    const int64_t n = LB[t];
    const int j = (int)n / g.nx, i = (int)n - j * g.nx;
    for (int m = -a.rmax; m <= a.rmax; ++m) {
      if (m == 0) continue;
      bool ok;
      const int ii = wrapi(i + m, g.nx, g.bc, &ok) ;
      const int iic = ok ? ii : (i + m < 0 ? 0 : g.nx - 1);  // transmissive: clamp
      if (!get_bit(B, g, iic, j)) atomicOr(&HM[(int64_t)j * g.wpr + (iic >> 5)], 1u << (iic & 31));
      if (g.dim == 2) {
        const int jj = wrapi(j + m, g.ny, g.bcy, &ok);
        const int jjc = ok ? jj : (j + m < 0 ? 0 : g.ny - 1);
        if (!get_bit(B, g, i, jjc)) atomicOr(&HM[(int64_t)jjc * g.wpr + (i >> 5)], 1u << (i & 31));
      }
    }
  }
  grid.sync();
  sstamp(a.tdbg, ts);
  {
    const int t = blk_count(HM, rb0, rb1, wcnt);
    if (tid == 0) a.blk[7 * G + blockIdx.x] = t;
  }
  grid.sync();
  sstamp(a.tdbg, ts);
  {
    int off, tot;
    block_offset(a.blk, 7, &off, &tot, sbuf);
    blk_count(HM, rb0, rb1, wcnt);
    blk_write(HM, rb0, rb1, off, wcnt, g, false, a.lists + (int64_t)L_H * N, nullptr, nullptr, a.idx, nb);
    if (blockIdx.x == 0 && tid == 0) a.counts[L_H] = tot;
  }
  grid.sync();
  sstamp(a.tdbg, ts);
  for (int64_t t = gtid; t < nb; t += gstride) {
    const int64_t n = LB[t];
    const int j = (int)n / g.nx, i = (int)n - j * g.nx;
    for (int m = -a.rmax; m <= a.rmax; ++m) {
      bool ok;
      int ii = wrapi(i + m, g.nx, g.bc, &ok);
      if (!ok) ii = i + m < 0 ? 0 : g.nx - 1;
      a.tab[(int64_t)(m + 3) * N + t] = __ldcg(a.idx + (int64_t)j * g.nx + ii);
      if (g.dim == 2) {
        int jj = wrapi(j + m, g.ny, g.bcy, &ok);
        if (!ok) jj = j + m < 0 ? 0 : g.ny - 1;
        a.tab[(int64_t)(7 + m + 3) * N + t] = __ldcg(a.idx + (int64_t)jj * g.nx + i);
      }
    }
  }
}

}  // namespace

hrom_status launch_sets(hrom_ctx* c, bool do_select, const double* eps, long long n_g, bool sparse,
                        double rre_delta, bool use_prev) {
  SetsArgs a{};
  a.use_prev = use_prev ? 1 : 0;
  if (rre_delta > 0.0) {  // delta = dm 2^-sh exactly
    int ex;
    const double mant = std::frexp(rre_delta, &ex);
    a.rre = 1;
    a.rre_dm = (unsigned long long)std::ldexp(mant, 53);
    a.rre_sh = 53 - ex;
  }
  a.hsum = c->b.hsum;
  if (do_select && c->P.odeim_points > 0) {
    a.extra = c->b.ocells;
    a.n_extra = c->odeim_n;
  }
  a.cand = sparse ? c->b.lists + (int64_t)L_T * c->g.N : nullptr;
  a.ncand = c->b.counts + L_T;
  a.g = c->g;
  a.do_select = do_select ? 1 : 0;
  a.eps = eps;
  a.n_g = n_g;
  a.halo = c->P.halo;
  a.band = c->P.band;
  a.rmax = 0;
  if (c->P.filter_max_sweeps > 0)
    for (int i = 0; i < c->P.n_filter_orders; ++i) a.rmax = std::max(a.rmax, c->P.filter_orders[i] / 2);
  a.masks = c->b.masks;
  a.mwords = c->mwords;
  a.lists = c->b.lists;
  a.counts = c->b.counts;
  a.sel_val = c->b.sel_val;
  a.sel_cell = c->b.sel_cell;
  a.blk = c->b.blk;
  a.hist = c->b.hist;
  a.idx = c->b.fidx;
  a.tab = c->b.ftab;
  a.tdbg = c->b.dbg;
  if ((int64_t)16 * c->sets_blocks > c->b.blk_len) return HROM_E_INVALID;
  void* args[] = {&a};
  const int grid = c->basis_pending ? c->sets_blocks - 1 : c->sets_blocks;  // leave the eigen's SM
  HROM_CK(cudaLaunchCooperativeKernel((void*)sets_kernel, dim3(grid), dim3(ST_T), args, 0, c->st));
  ++c->nlaunch;
  return HROM_OK;
}

int sets_occupancy() {
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, sets_kernel, ST_T, 0);
  return nb;
}

namespace {

}  // namespace

__global__ void or_cells_kernel(Geo g, uint32_t* S, const int32_t* cells, int n) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
    const int ci = cells[q], j = ci / g.nx, i = ci - j * g.nx;
    atomicOr(&S[(int64_t)j * g.wpr + (i >> 5)], 1u << (i & 31));
  }
}

hrom_status or_cells_into_mask(hrom_ctx* c, uint32_t* mask, const int32_t* cells, int n) {
  if (n <= 0) return HROM_OK;
  or_cells_kernel<<<1, 256, 0, c->st>>>(c->g, mask, cells, n);
  HROM_LAUNCH_CK();
  ++c->nlaunch;
  return HROM_OK;
}

// S-hat bitmap (in masks[M_S]) -> B, T, A2, A1 bitmaps, their ascending lists and the
// seam-filter tables.
hrom_status build_sets(hrom_ctx* c, const uint32_t* dev_mask_S) {
  c->samples_since_gather = 99;  // an explicit S-hat: no churn lists for the incremental Gram
  uint32_t* S = c->b.masks + (int64_t)M_S * c->mwords;
  if (dev_mask_S && dev_mask_S != S)
    HROM_CK(cudaMemcpyAsync(S, dev_mask_S, c->mwords * sizeof(uint32_t), cudaMemcpyDeviceToDevice, c->st));
  if (c->P.odeim_points > 0 && c->basis_ready) {  // an explicit mask is G: S-hat = G u ODEIM points
    hrom_status s = odeim_for_basis(c);
    if (s != HROM_OK) return s;
    if ((s = or_cells_into_mask(c, S, c->b.ocells, c->odeim_n)) != HROM_OK) return s;
  }
  return launch_sets(c, false, nullptr, 0);
}

// the sets of an S-hat bitmap already in place whose predecessor is in M_SPREV (row slabs: the
// selection ran across ranks, slab.cu): as build_sets, plus the churn lists of the incremental
// gathered Gram (G7)
hrom_status build_sets_with_churn(hrom_ctx* c) {
  ++c->samples_since_gather;
  return launch_sets(c, false, nullptr, 0, false, 0.0, true);
}

// top-n_g of eps > 0 -> S-hat (ties at the threshold by ascending cell), then build_sets.
hrom_status select_and_build(hrom_ctx* c, const double* eps, int64_t n_g, double rre_delta) {
  ++c->samples_since_gather;
  // the step's own indicator is nonzero only on S-hat u B (the T list): scan that list only
  const bool sparse = eps == c->b.eps && c->eps_sparse;
  return launch_sets(c, true, eps, (long long)n_g, sparse, rre_delta);
}

}  // namespace hrom
