// masks.cu -- H8: sampling sets as N-bit bitmaps, warp-ballot stream compaction into
// ascending cell lists, and the top-ceil(fN) indicator selection (radix select on the
// IEEE bit patterns of eps >= 0).
//
// Paper: sampling matrices S-hat, S-tilde, S-breve (Fig. 1), Neighbors /
// union / setdiff, ordering of the pointwise error.
// Readings: A9 (per-stage cross dilations), A18 (fraction mode, ties by ascending
// index), A21 (square seam band).  Everything here is integer work: bit-exact.
#include "internal.cuh"

namespace hrom {
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
  return (m[(int64_t)j * g.wpr + (i >> 5)] >> (i & 31)) & 1u;
}

// valid-bit mask of word wi in a row
__device__ __forceinline__ uint32_t row_valid(const Geo& g, int wi) {
  const int rem = g.nx - 32 * wi;
  return rem >= 32 ? 0xffffffffu : ((1u << rem) - 1u);
}

// x-dilation of one word by radius h: OR_{|a|<=h} in[i+a]
__device__ uint32_t xdil_word(const uint32_t* in, const Geo& g, int j, int wi, int h) {
  const uint32_t* row = in + (int64_t)j * g.wpr;
  const uint32_t cur = row[wi];
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
    prev = row[(wi - 1 + g.wpr) % g.wpr];
    next = row[(wi + 1) % g.wpr];
  } else {
    prev = wi > 0 ? row[wi - 1] : 0u;
    next = wi + 1 < g.wpr ? row[wi + 1] : 0u;
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
    const int jj = wrapi(j + b, g.ny, g.bc, &ok);
    if (ok) out |= in[(int64_t)jj * g.wpr + wi];
  }
  return out;
}

// cross dilation C_h (x and y arms of the original set)
__global__ void cross_kernel(Geo g, const uint32_t* __restrict__ in, uint32_t* __restrict__ out, int h) {
  const int64_t nw = (int64_t)g.ny * g.wpr;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nw; w += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(w / g.wpr), wi = (int)(w % g.wpr);
    uint32_t o = xdil_word(in, g, j, wi, h);
    if (g.dim == 2) o |= ydil_word(in, g, j, wi, h);
    out[w] = o;
  }
}

__global__ void xdil_kernel(Geo g, const uint32_t* __restrict__ in, uint32_t* __restrict__ out, int h) {
  const int64_t nw = (int64_t)g.ny * g.wpr;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nw; w += (int64_t)gridDim.x * blockDim.x)
    out[w] = xdil_word(in, g, (int)(w / g.wpr), (int)(w % g.wpr), h);
}

// band: B = ydil(xdil(S)) \ S, T = S u B
__global__ void band_kernel(Geo g, const uint32_t* __restrict__ xs, const uint32_t* __restrict__ S,
                            uint32_t* __restrict__ B, uint32_t* __restrict__ T, int W) {
  const int64_t nw = (int64_t)g.ny * g.wpr;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nw; w += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(w / g.wpr), wi = (int)(w % g.wpr);
    const uint32_t sq = (g.dim == 2) ? ydil_word(xs, g, j, wi, W) : xs[w];
    const uint32_t s = S[w];
    B[w] = sq & ~s;
    T[w] = sq | s;
  }
}

// ---------------- ordered compaction (count / scan / write) ----------------
constexpr int CB = 256;  // words per compaction block

struct CmpJob {
  int n;                       // number of masks
  const uint32_t* mask[8];
  int32_t* list[8];
  double* vals[8];             // optional values gathered from src (flat mode)
  const double* src[8];
  int32_t* count_out[8];
  int flat[8];                 // 1: word w covers cells 32w..32w+31 (no rows)
};

__global__ void cmp_count_kernel(CmpJob job, int64_t nwords, int32_t* __restrict__ blkcnt, int nblk) {
  const int m = blockIdx.y;
  const int64_t w = (int64_t)blockIdx.x * CB + threadIdx.x;
  int c = (w < nwords) ? __popc(job.mask[m][w]) : 0;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  __shared__ int s[CB / 32];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int k = 0; k < CB / 32; ++k) t += s[k];
    blkcnt[(int64_t)m * nblk + blockIdx.x] = t;
  }
}

__global__ void cmp_scan_kernel(CmpJob job, int32_t* __restrict__ blkcnt, int nblk) {
  // one block per mask: exclusive scan in place, total -> count_out
  const int m = blockIdx.x;
  int32_t* a = blkcnt + (int64_t)m * nblk;
  __shared__ int carry;
  __shared__ int ws[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < nblk; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const int v = i < nblk ? a[i] : 0;
    int x = v;  // inclusive warp scan
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, x, o);
      if ((threadIdx.x & 31) >= o) x += t;
    }
    if ((threadIdx.x & 31) == 31) ws[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
      int y = threadIdx.x < (int)(blockDim.x >> 5) ? ws[threadIdx.x] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, y, o);
        if (threadIdx.x >= o) y += t;
      }
      ws[threadIdx.x] = y;  // inclusive over warps
    }
    __syncthreads();
    const int wpre = (threadIdx.x >> 5) ? ws[(threadIdx.x >> 5) - 1] : 0;
    const int excl = carry + wpre + x - v;
    __syncthreads();
    if (i < nblk) a[i] = excl;
    if (threadIdx.x == blockDim.x - 1) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0 && job.count_out[m]) *job.count_out[m] = carry;
}

__global__ void cmp_write_kernel(CmpJob job, Geo g, int64_t nwords, const int32_t* __restrict__ blkoff, int nblk) {
  const int m = blockIdx.y;
  const int64_t w = (int64_t)blockIdx.x * CB + threadIdx.x;
  const uint32_t bits = (w < nwords) ? job.mask[m][w] : 0u;
  const int c = __popc(bits);
  int x = c;
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) >= o) x += t;
  }
  __shared__ int ws[CB / 32];
  if ((threadIdx.x & 31) == 31) ws[threadIdx.x >> 5] = x;
  __syncthreads();
  int wpre = 0;
  for (int k = 0; k < (int)(threadIdx.x >> 5); ++k) wpre += ws[k];
  int pos = blkoff[(int64_t)m * nblk + blockIdx.x] + wpre + x - c;
  if (!bits) return;
  int64_t cell0;
  if (job.flat[m]) cell0 = 32 * w;
  else cell0 = (w / g.wpr) * (int64_t)g.nx + 32 * (w % g.wpr);
  uint32_t b = bits;
  while (b) {
    const int bit = __ffs(b) - 1;
    b &= b - 1;
    const int64_t cell = cell0 + bit;
    job.list[m][pos] = (int32_t)cell;
    if (job.vals[m]) job.vals[m][pos] = job.src[m][cell];
    ++pos;
  }
}

hrom_status run_compaction(hrom_ctx* c, const CmpJob& job, int64_t nwords) {
  const int nblk = (int)((nwords + CB - 1) / CB);
  if ((int64_t)nblk * job.n > c->b.blk_len) return HROM_E_INVALID;
  dim3 grid(nblk, job.n);
  cmp_count_kernel<<<grid, CB, 0, c->st>>>(job, nwords, c->b.blk, nblk);
  cmp_scan_kernel<<<job.n, 1024, 0, c->st>>>(job, c->b.blk, nblk);
  cmp_write_kernel<<<grid, CB, 0, c->st>>>(job, c->g, nwords, c->b.blk, nblk);
  HROM_LAUNCH_CK();
  c->nlaunch += 3;
  return HROM_OK;
}

// ---------------- top-n selection ----------------
// flat bitmap of eps > 0 (word w: cells 32w..32w+31)
__global__ void nz_kernel(const double* __restrict__ eps, int64_t N, uint32_t* __restrict__ out) {
  const int64_t nthreads = ((N + 31) / 32) * 32;
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < nthreads; n += (int64_t)gridDim.x * blockDim.x) {
    const bool p = n < N && eps[n] > 0.0;
    const uint32_t b = __ballot_sync(0xffffffffu, p);
    if ((threadIdx.x & 31) == 0) out[n >> 5] = b;
  }
}

// selection state in hist[256 ..]: [0] prefix lo, [1] prefix hi, [2] remaining rank, [3] count_gt,
// [4] mode (0: take all, 1: threshold), [5] need ties
__global__ void sel_init(int32_t* st, const int32_t* cnt, long long n_g) {
  const int total = *cnt;
  st[0] = 0;
  st[1] = 0;
  st[2] = (int)(n_g < total ? n_g : total);
  st[3] = 0;
  st[4] = (n_g < total) ? 1 : 0;
  st[5] = 0;
}

__global__ void sel_hist(const double* __restrict__ vals, const int32_t* __restrict__ cnt,
                         int32_t* __restrict__ hist, const int32_t* __restrict__ st, int shift) {
  if (st[4] == 0) return;
  __shared__ int h[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const unsigned long long prefix = ((unsigned long long)(unsigned)st[1] << 32) | (unsigned)st[0];
  const unsigned long long hm = (shift >= 56) ? 0ull : (~0ull << (shift + 8));
  const int total = *cnt;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(vals[t]);
    if ((b & hm) == prefix) atomicAdd(&h[(b >> shift) & 255], 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    if (h[i]) atomicAdd(&hist[i], h[i]);
}

__global__ void sel_pick(int32_t* hist, int32_t* st, int shift) {
  if (st[4] == 0) return;
  int rem = st[2];
  int above = 0;
  int d = 255;
  for (; d > 0; --d) {
    if (above + hist[d] >= rem) break;
    above += hist[d];
  }
  st[2] = rem - above;
  st[3] += above;
  unsigned long long prefix = ((unsigned long long)(unsigned)st[1] << 32) | (unsigned)st[0];
  prefix |= (unsigned long long)d << shift;
  st[0] = (int)(unsigned)(prefix & 0xffffffffull);
  st[1] = (int)(unsigned)(prefix >> 32);
  if (shift == 0) st[5] = st[2];  // ties to take at the threshold value
  for (int i = 0; i < 256; ++i) hist[i] = 0;
}

// mark selected cells into the (row-padded) S bitmap; ties at tau by ascending cell
__global__ void sel_mark_count(const double* __restrict__ vals, const int32_t* __restrict__ cnt,
                               const int32_t* __restrict__ st, int32_t* __restrict__ blkcnt) {
  const int total = *cnt;
  const unsigned long long tau = ((unsigned long long)(unsigned)st[1] << 32) | (unsigned)st[0];
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool tie = st[4] && t < total && (unsigned long long)__double_as_longlong(vals[t]) == tau;
  int c = __popc(__ballot_sync(0xffffffffu, tie));
  __shared__ int s[32];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int tt = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) tt += s[k];
    blkcnt[blockIdx.x] = tt;
  }
}

__global__ void sel_mark_write(Geo g, const double* __restrict__ vals, const int32_t* __restrict__ cells,
                               const int32_t* __restrict__ cnt, const int32_t* __restrict__ st,
                               const int32_t* __restrict__ blkoff, uint32_t* __restrict__ S) {
  const int total = *cnt;
  const unsigned long long tau = ((unsigned long long)(unsigned)st[1] << 32) | (unsigned)st[0];
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool in = t < total;
  const unsigned long long b = in ? (unsigned long long)__double_as_longlong(vals[t]) : 0ull;
  const bool tie = st[4] && in && b == tau;
  const unsigned bal = __ballot_sync(0xffffffffu, tie);
  __shared__ int s[32];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = __popc(bal);
  __syncthreads();
  int pre = blkoff[blockIdx.x];
  for (int k = 0; k < (int)(threadIdx.x >> 5); ++k) pre += s[k];
  pre += __popc(bal & ((1u << (threadIdx.x & 31)) - 1u));
  bool sel = false;
  if (in) {
    if (st[4] == 0) sel = true;
    else if (b > tau) sel = true;
    else if (tie && pre < st[5]) sel = true;
  }
  if (sel) {
    const int64_t cell = cells[t];
    const int i = (int)(cell % g.nx), j = (int)(cell / g.nx);
    atomicOr(&S[(int64_t)j * g.wpr + (i >> 5)], 1u << (i & 31));
  }
}

}  // namespace

hrom_status compact_masks(hrom_ctx* c, const int* which, int nwhich) {
  CmpJob job{};
  job.n = nwhich;
  for (int k = 0; k < nwhich; ++k) {
    const int l = which[k];  // list index == mask index for S, B, T, A2, A1
    job.mask[k] = c->b.masks + (int64_t)l * c->mwords;
    job.list[k] = c->b.lists + (int64_t)l * c->g.N;
    job.vals[k] = nullptr;
    job.src[k] = nullptr;
    job.count_out[k] = c->b.counts + l;
    job.flat[k] = 0;
  }
  return run_compaction(c, job, c->mwords);
}

// S-hat bitmap (in masks[M_S]) -> B, T, A2, A1 bitmaps and their ascending lists.
hrom_status build_sets(hrom_ctx* c, const uint32_t* dev_mask_S) {
  const Geo& g = c->g;
  uint32_t* M = c->b.masks;
  const int64_t mw = c->mwords;
  uint32_t* S = M + M_S * mw;
  if (dev_mask_S && dev_mask_S != S)
    HROM_CK(cudaMemcpyAsync(S, dev_mask_S, mw * sizeof(uint32_t), cudaMemcpyDeviceToDevice, c->st));
  const int grid = (int)std::min<int64_t>((mw + 255) / 256, (int64_t)c->nsm * 16);
  xdil_kernel<<<grid, 256, 0, c->st>>>(g, S, M + M_TMP * mw, c->P.band);
  band_kernel<<<grid, 256, 0, c->st>>>(g, M + M_TMP * mw, S, M + M_B * mw, M + M_T * mw, c->P.band);
  cross_kernel<<<grid, 256, 0, c->st>>>(g, M + M_T * mw, M + M_A2 * mw, c->P.halo);
  cross_kernel<<<grid, 256, 0, c->st>>>(g, M + M_A2 * mw, M + M_A1 * mw, c->P.halo);
  HROM_LAUNCH_CK();
  c->nlaunch += 4;
  const int which[5] = {L_S, L_B, L_T, L_A2, L_A1};
  return compact_masks(c, which, 5);
}

// top-n_g of eps > 0 -> S bitmap (masks[M_S]); ties at the threshold by ascending cell.
hrom_status select_topn(hrom_ctx* c, const double* eps, int64_t n_g) {
  const int64_t N = c->g.N;
  const int64_t fw = (N + 31) / 32;
  uint32_t* flat = c->b.masks + (int64_t)M_TMP2 * c->mwords;  // mwords >= fw
  int32_t* cnt = c->b.counts + 8;
  int32_t* hist = c->b.hist;
  int32_t* st = c->b.hist + 256;
  const int grid = c->nsm * 8;
  nz_kernel<<<grid, 256, 0, c->st>>>(eps, N, flat);
  HROM_LAUNCH_CK();
  CmpJob job{};
  job.n = 1;
  job.mask[0] = flat;
  job.list[0] = c->b.sel_cell;
  job.vals[0] = c->b.sel_val;
  job.src[0] = eps;
  job.count_out[0] = cnt;
  job.flat[0] = 1;
  hrom_status s = run_compaction(c, job, fw);
  if (s != HROM_OK) return s;
  HROM_CK(cudaMemsetAsync(hist, 0, 256 * sizeof(int32_t), c->st));
  sel_init<<<1, 1, 0, c->st>>>(st, cnt, (long long)n_g);
  for (int shift = 56; shift >= 0; shift -= 8) {
    sel_hist<<<c->nsm * 2, 512, 0, c->st>>>(c->b.sel_val, cnt, hist, st, shift);
    sel_pick<<<1, 1, 0, c->st>>>(hist, st, shift);
  }
  HROM_LAUNCH_CK();
  // mark: count ties per block, scan, write
  uint32_t* S = c->b.masks + (int64_t)M_S * c->mwords;
  HROM_CK(cudaMemsetAsync(S, 0, c->mwords * sizeof(uint32_t), c->st));
  const int nb = (int)((N + 1023) / 1024);
  sel_mark_count<<<nb, 1024, 0, c->st>>>(c->b.sel_val, cnt, st, c->b.blk);
  CmpJob one{};
  one.n = 1;
  one.count_out[0] = nullptr;
  cmp_scan_kernel<<<1, 1024, 0, c->st>>>(one, c->b.blk, nb);
  sel_mark_write<<<nb, 1024, 0, c->st>>>(c->g, c->b.sel_val, c->b.sel_cell, cnt, st, c->b.blk, S);
  HROM_LAUNCH_CK();
  c->nlaunch += 1 + 1 + 16 + 3;
  return HROM_OK;
}

}  // namespace hrom
