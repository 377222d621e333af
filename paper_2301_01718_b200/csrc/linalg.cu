// linalg.cu -- H4/H5 (gappy normal equations + one-CTA solve), H10-H12 (Gram, thin
// eigen, lift).  FP64 tensor cores: mma.sync.m8n8k4.f64 (SASS DMMA; sm_100a has no
// tcgen05 f64 kind).
//
// Paper: gappy coordinates y = (P^T Phi)^+ P^T (v - psi) (Eq. 8); POD_m of the
// lagged-centred window via a thin SVD (Eq. 9; remark P:634);
// reading A13 (pinv cut 1e-12 on lambda), A14 (lagged centring; shifted Gram with
// periodic re-base), A15 (Gram + Jacobi eigen, keep lambda_i >= 1e-8 lambda_1, sign on V).
#include <algorithm>
#include <cstring>
#include <utility>
#include <vector>
#include "internal.cuh"
#include "eig.cuh"
#include "async.cuh"
#include "dd.cuh"

namespace hrom {
namespace {

constexpr int GR_TPE = 16;  // threads per entry of the fixed-order partial reductions


__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// ---------------- H4: gathered Gram of the S-hat rows ----------------
// R = [U - rho, b - rho]^T [U - rho, b - rho] over the c |S-hat| rows (U: the nU union slots in
// window order, b: the HDM value, rho: the Gram shift); the lagged centring (A14) is applied to
// the small R by solve_kernel, exactly as for the window Gram C.
// Warp-specialised, one CTA per SM: GG_PW producer warps own one tile row per thread and gather
// its nU + 1 values with 8-byte cp.async one tile ahead, subtract rho once they land and arrive
// on full[s]; GG_CW consumer warps each own one 16 x 16 super-block pair of the upper triangle
// (DMMA m8n8k4) and release the stage through empty[s].  No CTA-wide barrier in the stream.
// NSB 16-column super blocks (ncol <= 16 NSB), RT rows per tile (= producer threads),
// TPW super-block pairs per consumer warp, CW consumer warps.
// DD: double-double consumers (dd.cuh, G11) instead of DMMA: each consumer thread owns TPW
// 2 x 2 column blocks of the upper triangle and accumulates TwoProduct/TwoSum; odd tile stride
// (conflict-free column gathers of one row).
template <int NSB, int RT, int TPW, int CW, int STAGES, int PW, int LOOK, bool DD = false>
struct GGCfg {
  static constexpr int nsb = NSB, rt = RT, tpw = TPW, cw = CW, stages = STAGES, look = LOOK;
  static constexpr bool dd = DD;
  static constexpr int pw = PW, ncp = 16 * NSB, ldt = DD ? RT + 1 : RT + 4, threads = 32 * (PW + CW);
  static constexpr int parts = 32 * PW / RT;  // producer threads per tile row (columns split)
  // per stage: the tile, then each producer part's copy of the shift of its rows (cp.async'd
  // with the tile, so no pending global load is carried across iterations in registers)
  static constexpr size_t smem = (size_t)STAGES * (ncp * ldt + parts * RT) * sizeof(double);
  static_assert(DD ? 32 * CW * TPW >= (8 * NSB) * (8 * NSB + 1) / 2 : CW * TPW >= NSB * (NSB + 1) / 2, "tasks");
  static_assert((32 * PW) % RT == 0 && STAGES >= LOOK + 2, "producer layout");
};
// producers run LOOK tiles ahead of the tile they publish (DRAM latency of the 8-byte gathers)
using GGSmall = GGCfg<5, 64, 1, 15, 4, 6, 2>;  // ncol <= 80 (w <= 78)
using GGWide = GGCfg<9, 32, 3, 15, 4, 2, 2>;   // ncol <= 144 (w <= kMaxW)
using GGDSmall = GGCfg<5, 64, 2, 15, 4, 6, 2, true>;  // double-double, ncol <= 80
using GGDWide = GGCfg<9, 32, 6, 15, 4, 2, 2, true>;   // double-double, ncol <= 144

struct GGArgs {
  int mode;                  // 0: contiguous rows of ncol columns (cols, slab stride ns), 1: S-hat rows
  // mode 0
  const double* const* cols;
  int64_t ns;
  int ncol0;
  int64_t rows;
  // mode 1
  Geo g;
  Win W;
  const double* ring;
  const int32_t* list;
  const int32_t* count;
  SRef src_b;
  const int64_t* rowlist;    // mode 2: explicit DOF rows (ODEIM points), count nrow2
  int nrow2;
  // both
  SRef rho;                  // shift (rho.p nullable in mode 0)
  double* part;              // [grid][ncp][ncp]
};

template <class CFG>
__global__ void __launch_bounds__(CFG::threads, 1) gather_gram_kernel(GGArgs a) {
  constexpr int RT = CFG::rt, NSB = CFG::nsb, NCP = CFG::ncp, LDT = CFG::ldt, ST = CFG::stages;
  extern __shared__ double smem[];
  __shared__ __align__(8) uint64_t full[ST], empty[ST];
  __shared__ const double* scol[NCP];  // column base pointers (mode 0: caller's; mode 1: ring slots)
  const int nS = a.mode == 1 ? *a.count : 0;
  const int64_t total_rows = a.mode == 1 ? (int64_t)nS * a.g.c : a.mode == 2 ? a.nrow2 : a.rows;
  const int64_t ntiles = (total_rows + RT - 1) / RT;
  const bool gath = a.mode >= 1;
  const int nU = gath ? a.W.nU : a.ncol0;
  const int ncol = gath ? nU + 1 : a.ncol0;  // modes 1, 2: union slots + b
  for (int col = threadIdx.x; col < ncol; col += CFG::threads)
    scol[col] = gath ? (col < nU ? a.ring + (int64_t)a.W.slot[col] * TILE : nullptr) : a.cols[col];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < ST * NCP * LDT; i += CFG::threads) smem[i] = 0.0;  // padding stays 0
  if (threadIdx.x == 0) {
    for (int q = 0; q < ST; ++q) {
      mbar_init(&full[q], 32 * CFG::pw);
      mbar_init(&empty[q], CFG::cw);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int64_t my_tiles = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (warp < CFG::pw) {
    // ---- producers: thread (k, part) owns row k, columns part, part + parts, ... of every tile ----
    constexpr int PARTS = CFG::parts, LOOK = CFG::look;
    const int k = threadIdx.x % RT, part = threadIdx.x / RT;
    const SRef slab{nullptr, gath ? a.g.nsr : a.ns};
    double* ext0 = smem + (size_t)ST * NCP * LDT;  // [stage][part][RT] shifts
    for (int64_t it = 0; it < my_tiles + LOOK; ++it) {
      if (it < my_tiles) {
        const int st = (int)(it % ST);
        if (it >= ST) mbar_wait(&empty[st], (uint32_t)(((it / ST) - 1) & 1));
        double* tile = smem + (size_t)st * NCP * LDT;
        const int64_t row = (blockIdx.x + it * gridDim.x) * RT + k;
        if (row < total_rows) {
          int64_t e;
          if (gath) {
            if (a.mode == 2) {
              e = __ldg(a.rowlist + row);
            } else {
              const int var = (int)row / nS;  // 32-bit: c * |S-hat| < 2^31
              e = (int64_t)var * a.g.N + __ldg(a.list + ((int)row - var * nS));
            }
            const int64_t se = sidx(slab, e);
            for (int col = part; col < nU; col += PARTS) cp_async8(tile + col * LDT + k, scol[col] + se);
            if (nU % PARTS == part) cp_async8(tile + nU * LDT + k, a.src_b.p + sidx(a.src_b, e));
          } else {
            e = row;
            const int64_t se = sidx(slab, e);
            for (int col = part; col < ncol; col += PARTS) cp_async8(tile + col * LDT + k, scol[col] + se);
          }
          double* ext = ext0 + ((size_t)st * PARTS + part) * RT;
          if (a.rho.p) cp_async8(ext + k, a.rho.p + sidx(a.rho, e));
          else ext[k] = 0.0;
        } else {
          for (int col = part; col < ncol; col += PARTS) tile[col * LDT + k] = 0.0;
        }
      }
      cp_async_commit();
      if (it >= LOOK) {  // tile it-LOOK has landed: shift by rho, publish
        cp_async_wait<LOOK>();
        const int64_t pit = it - LOOK;
        const int ps = (int)(pit % ST);
        double* tile = smem + (size_t)ps * NCP * LDT;
        if ((blockIdx.x + pit * gridDim.x) * RT + k < total_rows) {
          const double rh = ext0[((size_t)ps * PARTS + part) * RT + k];
          for (int col = part; col < ncol; col += PARTS) tile[col * LDT + k] -= rh;
        }
        mbar_arrive(&full[ps]);
      }
    }
    cp_async_wait<0>();
  } else if constexpr (CFG::dd) {
    // ---- double-double consumers: thread t owns the 2 x 2 column blocks t, t + T, ... of the
    // upper triangle (bi <= bj over nb = ceil(ncol / 2) block indices) ----
    constexpr int BPT = CFG::tpw, T = 32 * CFG::cw;
    const int t = threadIdx.x - 32 * CFG::pw;
    const int nb = (ncol + 1) / 2, nblk = nb * (nb + 1) / 2;
    int ci[BPT], cj[BPT];
#pragma unroll
    for (int q = 0; q < BPT; ++q) {
      const int task = t + q * T;
      int x = 0, rem = task < nblk ? task : 0;
      while (rem >= nb - x) {
        rem -= nb - x;
        ++x;
      }
      ci[q] = task < nblk ? 2 * x : -1;
      cj[q] = 2 * (x + rem);
    }
    double hi[BPT][4], lo[BPT][4];
#pragma unroll
    for (int q = 0; q < BPT; ++q)
#pragma unroll
      for (int u = 0; u < 4; ++u) hi[q][u] = lo[q][u] = 0.0;
    for (int64_t it = 0; it < my_tiles; ++it) {
      const int st = (int)(it % ST);
      mbar_wait(&full[st], (uint32_t)((it / ST) & 1));
      const double* tile = smem + (size_t)st * NCP * LDT;
#pragma unroll
      for (int q = 0; q < BPT; ++q) {
        if (ci[q] < 0) continue;
        const double* xa = tile + ci[q] * LDT;
        const double* xb = tile + cj[q] * LDT;
        for (int kk = 0; kk < RT; ++kk) {
          const double a0 = xa[kk], a1 = xa[LDT + kk], b0 = xb[kk], b1 = xb[LDT + kk];
          dd_fma(hi[q][0], lo[q][0], a0, b0);
          dd_fma(hi[q][1], lo[q][1], a0, b1);
          dd_fma(hi[q][2], lo[q][2], a1, b0);
          dd_fma(hi[q][3], lo[q][3], a1, b1);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    double* out = a.part + (int64_t)blockIdx.x * NCP * NCP * 2;
#pragma unroll
    for (int q = 0; q < BPT; ++q) {
      if (ci[q] < 0) continue;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = ci[q] + (u >> 1), j = cj[q] + (u & 1);
        if (i > j) continue;  // diagonal block: the lower entry duplicates the upper one
        dd_norm(hi[q][u], lo[q][u]);
        out[2 * (i * NCP + j)] = hi[q][u];
        out[2 * (i * NCP + j) + 1] = lo[q][u];
      }
    }
  } else {
    // ---- consumers: TPW upper super-block pairs (sa <= sb) per warp ----
    const int cwarp = warp - CFG::pw;
    const int gid = lane >> 2, tig = lane & 3;
    // the last super block holds ncol - 16 (NSB - 1) real columns: when <= 8, its pairs only
    // need the first 8-column half (fewer DMMAs, same result: the rest is padding)
    const bool last_half = ncol <= 16 * (NSB - 1) + 8;
    int sa[CFG::tpw], sb[CFG::tpw];
    bool has[CFG::tpw];
#pragma unroll
    for (int t = 0; t < CFG::tpw; ++t) {
      const int task = cwarp + t * CFG::cw;
      has[t] = task < NSB * (NSB + 1) / 2;
      int x = 0, rem = has[t] ? task : 0;
      while (rem >= NSB - x) {
        rem -= NSB - x;
        ++x;
      }
      sa[t] = x;
      sb[t] = x + rem;
    }
    double acc[CFG::tpw][8];
#pragma unroll
    for (int t = 0; t < CFG::tpw; ++t)
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[t][q] = 0.0;
    for (int64_t it = 0; it < my_tiles; ++it) {
      const int st = (int)(it % ST);
      mbar_wait(&full[st], (uint32_t)((it / ST) & 1));
      const double* tile = smem + (size_t)st * NCP * LDT;
#pragma unroll
      for (int t = 0; t < CFG::tpw; ++t) {
        if (!has[t]) continue;
        const bool bh = last_half && sb[t] == NSB - 1;  // b: first half only
        const bool ah = last_half && sa[t] == NSB - 1;  // a: first half only
#pragma unroll
        for (int kk = 0; kk < RT; kk += 4) {
          const double a0 = tile[(16 * sa[t] + gid) * LDT + kk + tig];
          const double b0 = tile[(16 * sb[t] + gid) * LDT + kk + tig];
          dmma(acc[t][0], acc[t][1], a0, b0);
          if (!bh) {
            const double b1 = tile[(16 * sb[t] + 8 + gid) * LDT + kk + tig];
            dmma(acc[t][2], acc[t][3], a0, b1);
            if (!ah) {
              const double a1 = tile[(16 * sa[t] + 8 + gid) * LDT + kk + tig];
              if (sa[t] != sb[t]) dmma(acc[t][4], acc[t][5], a1, b0);  // diagonal pair: lower block unused
              dmma(acc[t][6], acc[t][7], a1, b1);
            }
          } else if (!ah) {
            const double a1 = tile[(16 * sa[t] + 8 + gid) * LDT + kk + tig];
            dmma(acc[t][4], acc[t][5], a1, b0);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    double* out = a.part + (int64_t)blockIdx.x * NCP * NCP;
#pragma unroll
    for (int t = 0; t < CFG::tpw; ++t) {
      if (!has[t]) continue;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int bi = 16 * sa[t] + 8 * (q >> 1), bj = 16 * sb[t] + 8 * (q & 1);
        out[(bi + gid) * NCP + bj + 2 * tig] = acc[t][2 * q];
        out[(bi + gid) * NCP + bj + 2 * tig + 1] = acc[t][2 * q + 1];
      }
    }
  }
}

// ---------------- H10 / K11: window Gram of contiguous (slab) rows ----------------
// C = (S - rho 1^T)^T (S - rho 1^T) over D rows of ncol columns, ncol = 16 NSB + TAIL.  The
// 16 NSB leading columns run on the FP64 tensor cores; the TAIL (<= 2) trailing columns -- the
// "+1" of the w+1 window columns (A14) -- would otherwise cost a whole padded 16-column super
// block of DMMAs (17 of 153 per k-step at w = 128, 9 of 45 at w = 64), so the producer threads
// that already touch every element for the rho shift accumulate them with FMAs instead.
// 4 producer warps (one per SM sub-partition, thread = one tile row, warp = one column part)
// and 16 consumer warps (4 per sub-partition); the upper super-block pairs are assigned by the
// host so that every sub-partition's tensor pipe gets the same DMMA count (warp w runs on
// sub-partition w mod 4).
constexpr int SG_PW = 4, SG_CW = 16, SG_TPW = 3;
constexpr int SG_THREADS = 32 * (SG_PW + SG_CW);
struct SGArgs {
  const double* const* cols;
  int64_t ns;       // slab slots per tile of the columns (1: plain vectors)
  int64_t rows;
  SRef rho;         // shift (rho.p nullable)
  double* part;     // [grid][ncp][ncp]
  int ncp;
  uint8_t task[SG_CW][SG_TPW];  // (sa << 4) | sb, 0xff = none
};
// RPT rows per producer thread (tile = 32 RPT rows: fewer per-tile pipeline drains when the
// per-tile DMMA work is small), STAGES smem stages, LOOK tiles in flight per producer
template <int NSB, int TAIL>
struct SGCfg {
  static constexpr int ncd = 16 * NSB;
  static constexpr int rpt = 2;
  static constexpr int rt = 32 * rpt, ldt = rt + 4;
  // per stage: the tile, and per producer warp the shift and tail values of its rows (landed by
  // cp.async with the tile: no global load result is carried across iterations in registers)
  static constexpr int ext = SG_PW * (1 + TAIL) * rt;
  static constexpr size_t stage_bytes = ((size_t)ncd * ldt + ext) * sizeof(double);
  static constexpr int fit = (int)((225 * 1024) / stage_bytes);
  static constexpr int stages = fit > 8 ? 8 : fit;
  static constexpr int look = stages - 2 < 3 ? stages - 2 : 3;
  static constexpr size_t smem = (size_t)stages * stage_bytes;
};

template <int NSB, int TAIL>
__global__ void __launch_bounds__(SG_THREADS, 1) slab_gram_kernel(SGArgs a) {
  using CF = SGCfg<NSB, TAIL>;
  constexpr int NCD = 16 * NSB, ST = CF::stages, LOOK = CF::look, NPC = NCD / SG_PW;
  constexpr int RPT = CF::rpt, RT = CF::rt, LDT = CF::ldt, TT = TAIL > 0 ? TAIL : 1;
  extern __shared__ double smem[];
  __shared__ __align__(8) uint64_t full[ST], empty[ST];
  __shared__ const double* scol[NCD + 2];
  for (int col = threadIdx.x; col < NCD + TAIL; col += SG_THREADS) scol[col] = a.cols[col];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int q = 0; q < ST; ++q) {
      mbar_init(&full[q], 32 * SG_PW);
      mbar_init(&empty[q], SG_CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int64_t ntiles = (a.rows + RT - 1) / RT;
  const int64_t my_tiles = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  double* out = a.part + (int64_t)blockIdx.x * a.ncp * a.ncp;
  if (warp < SG_PW) {
    // ---- producers: lane = tile rows lane + 32 q (q < RPT), warp = column part (part + 4 i) ----
    const int part = warp;
    const SRef slab{nullptr, a.ns};
    double* ext0 = smem + (size_t)ST * NCD * LDT;  // [stage][part][1 + TAIL][RT]
    double acc[TT][NPC];
    double att[3] = {0.0, 0.0, 0.0};  // tail x tail (part 0)
#pragma unroll
    for (int t = 0; t < TT; ++t)
#pragma unroll
      for (int i = 0; i < NPC; ++i) acc[t][i] = 0.0;
    for (int64_t it = 0; it < my_tiles + LOOK; ++it) {
      if (it < my_tiles) {
        const int st = (int)(it % ST);
        if (it >= ST) mbar_wait(&empty[st], (uint32_t)(((it / ST) - 1) & 1));
        double* tile = smem + (size_t)st * NCD * LDT;
        double* ext = ext0 + ((size_t)st * SG_PW + part) * (1 + TAIL) * RT;
#pragma unroll
        for (int h = 0; h < RPT; ++h) {
          const int k = lane + 32 * h;
          const int64_t row = (blockIdx.x + it * gridDim.x) * RT + k;
          if (row < a.rows) {
            const int64_t se = sidx(slab, row);
#pragma unroll
            for (int i = 0; i < NPC; ++i) cp_async8(tile + (part + SG_PW * i) * LDT + k, scol[part + SG_PW * i] + se);
            if (a.rho.p) cp_async8(ext + k, a.rho.p + sidx(a.rho, row));
            else ext[k] = 0.0;
#pragma unroll
            for (int t = 0; t < TAIL; ++t) cp_async8(ext + (1 + t) * RT + k, scol[NCD + t] + se);
          } else {
#pragma unroll
            for (int i = 0; i < NPC; ++i) tile[(part + SG_PW * i) * LDT + k] = 0.0;
          }
        }
      }
      cp_async_commit();
      if (it >= LOOK) {  // tile it-LOOK has landed: shift by rho, tail products, publish
        cp_async_wait<LOOK>();
        const int64_t pit = it - LOOK;
        const int ps = (int)(pit % ST);
        double* tile = smem + (size_t)ps * NCD * LDT;
        const double* ext = ext0 + ((size_t)ps * SG_PW + part) * (1 + TAIL) * RT;
#pragma unroll
        for (int h = 0; h < RPT; ++h) {
          const int k = lane + 32 * h;
          if ((blockIdx.x + pit * gridDim.x) * RT + k >= a.rows) continue;
          const double rh = ext[k];
          double xt[TT];
#pragma unroll
          for (int t = 0; t < TAIL; ++t) xt[t] = ext[(1 + t) * RT + k] - rh;
#pragma unroll
          for (int i = 0; i < NPC; ++i) {
            double* e = tile + (part + SG_PW * i) * LDT + k;
            const double v = *e - rh;
            *e = v;
#pragma unroll
            for (int t = 0; t < TAIL; ++t) acc[t][i] = fma(xt[t], v, acc[t][i]);
          }
          if (TAIL > 0 && part == 0) {
            att[0] = fma(xt[0], xt[0], att[0]);
            if (TAIL > 1) {
              att[1] = fma(xt[0], xt[TT - 1], att[1]);
              att[2] = fma(xt[TT - 1], xt[TT - 1], att[2]);
            }
          }
        }
        mbar_arrive(&full[ps]);
      }
    }
    cp_async_wait<0>();
    if (TAIL > 0) {  // fixed-order butterfly over the 32 lanes of the warp
#pragma unroll
      for (int t = 0; t < TAIL; ++t)
#pragma unroll
        for (int i = 0; i < NPC; ++i) {
          double v = acc[t][i];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          if (lane == 0) out[(part + SG_PW * i) * a.ncp + NCD + t] = v;
        }
      if (part == 0) {
#pragma unroll
        for (int q = 0; q < 3; ++q)
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) att[q] += __shfl_xor_sync(0xffffffffu, att[q], o);
        if (lane == 0) {
          out[NCD * a.ncp + NCD] = att[0];
          if (TAIL > 1) {
            out[NCD * a.ncp + NCD + 1] = att[1];
            out[(NCD + 1) * a.ncp + NCD + 1] = att[2];
          }
        }
      }
    }
  } else {
    // ---- consumers: up to SG_TPW upper super-block pairs (host-balanced per sub-partition) ----
    const int cwarp = warp - SG_PW;
    const int gid = lane >> 2, tig = lane & 3;
    int sa[SG_TPW], sb[SG_TPW];
    bool has[SG_TPW];
#pragma unroll
    for (int t = 0; t < SG_TPW; ++t) {
      const int v = a.task[cwarp][t];
      has[t] = v != 0xff;
      sa[t] = has[t] ? v >> 4 : 0;
      sb[t] = has[t] ? v & 15 : 0;
    }
    double acc[SG_TPW][8];
#pragma unroll
    for (int t = 0; t < SG_TPW; ++t)
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[t][q] = 0.0;
    for (int64_t it = 0; it < my_tiles; ++it) {
      const int st = (int)(it % ST);
      mbar_wait(&full[st], (uint32_t)((it / ST) & 1));
      const double* tile = smem + (size_t)st * NCD * LDT;
#pragma unroll
      for (int t = 0; t < SG_TPW; ++t) {
        if (!has[t]) continue;
        const double* pa = tile + (16 * sa[t] + gid) * LDT + tig;
        const double* pb = tile + (16 * sb[t] + gid) * LDT + tig;
        if (sa[t] != sb[t]) {
#pragma unroll
          for (int kk = 0; kk < RT; kk += 4) {
            const double a0 = pa[kk], a1 = pa[8 * LDT + kk], b0 = pb[kk], b1 = pb[8 * LDT + kk];
            dmma(acc[t][0], acc[t][1], a0, b0);
            dmma(acc[t][2], acc[t][3], a0, b1);
            dmma(acc[t][4], acc[t][5], a1, b0);
            dmma(acc[t][6], acc[t][7], a1, b1);
          }
        } else {  // diagonal pair: the lower 8 x 8 block is the mirror of the upper one
#pragma unroll
          for (int kk = 0; kk < RT; kk += 4) {
            const double a0 = pa[kk], a1 = pa[8 * LDT + kk];
            dmma(acc[t][0], acc[t][1], a0, a0);
            dmma(acc[t][2], acc[t][3], a0, a1);
            dmma(acc[t][6], acc[t][7], a1, a1);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
#pragma unroll
    for (int t = 0; t < SG_TPW; ++t) {
      if (!has[t]) continue;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int bi = 16 * sa[t] + 8 * (q >> 1), bj = 16 * sb[t] + 8 * (q & 1);
        out[(bi + gid) * a.ncp + bj + 2 * tig] = acc[t][2 * q];
        out[(bi + gid) * a.ncp + bj + 2 * tig + 1] = acc[t][2 * q + 1];
      }
    }
  }
}

// host: balance the upper super-block pairs (diagonal 3 DMMAs per k-step, off-diagonal 4) over
// the 4 sub-partitions (longest first, least-loaded bin), then over each one's 4 warps
bool sg_tasks(int nsb, SGArgs& a) {
  std::vector<std::pair<int, int>> t;  // (cost, code)
  for (int x = 0; x < nsb; ++x)
    for (int y = x; y < nsb; ++y) t.push_back({x == y ? 3 : 4, (x << 4) | y});
  std::stable_sort(t.begin(), t.end(), [](const std::pair<int, int>& u, const std::pair<int, int>& v) {
    return u.first > v.first;
  });
  int load[4] = {0, 0, 0, 0}, cnt[4] = {0, 0, 0, 0};
  std::memset(a.task, 0xff, sizeof(a.task));
  for (auto& q : t) {
    int b = 0;
    for (int i = 1; i < 4; ++i)
      if (load[i] < load[b]) b = i;
    const int slot = cnt[b] / 4, w = b + 4 * (cnt[b] % 4);  // consumer warp w: sub-partition w mod 4
    if (slot >= SG_TPW) return false;
    a.task[w][slot] = (uint8_t)q.second;
    load[b] += q.first;
    ++cnt[b];
  }
  return true;
}

template <int NSB, int TAIL>
hrom_status launch_slab_gram(hrom_ctx* c, SGArgs& a, int grid) {
  const size_t smem = SGCfg<NSB, TAIL>::smem;
  HROM_CK(cudaFuncSetAttribute(slab_gram_kernel<NSB, TAIL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  slab_gram_kernel<NSB, TAIL><<<grid, SG_THREADS, smem, c->st>>>(a);
  HROM_LAUNCH_CK();
  return HROM_OK;
}

// dispatch: returns HROM_E_INVALID when (ncol) has no instantiation (caller falls back)
hrom_status run_slab_gram(hrom_ctx* c, SGArgs& a, int ncol, int grid) {
  const int nsb = ncol / 16, tail = ncol - 16 * nsb;
  if (!sg_tasks(nsb, a)) return HROM_E_INVALID;
#define SG_CASE(N, T) \
  if (nsb == N && tail == T) return launch_slab_gram<N, T>(c, a, grid);
  SG_CASE(2, 0) SG_CASE(2, 1) SG_CASE(2, 2)
  SG_CASE(3, 0) SG_CASE(3, 1) SG_CASE(3, 2)
  SG_CASE(4, 0) SG_CASE(4, 1) SG_CASE(4, 2)
  SG_CASE(6, 0) SG_CASE(6, 1)
  SG_CASE(8, 0) SG_CASE(8, 1)
#undef SG_CASE
  return HROM_E_INVALID;
}

// ---------------- config 5: projection Phi^T S of the window (cross Gram, DMMA) ----------------
// C[i][j] = sum_e Phi[e][i] S_j[e] over the D rows: Phi (D x m, plain columns, m <= 64) against the
// w + 1 ring columns of the window (slab layout).  Same warp specialisation as slab_gram_kernel:
// 4 producer warps (lane = row, warp = column part) stage 32-row tiles of all 16 (NA + NB) columns
// (padding columns stay zero), 16 consumer warps own 16 x 16 (A block, B block) pairs balanced per
// sub-partition by the host.  Per-CTA partials reduced in fixed order by cross_reduce.
constexpr int XG_RT = 32, XG_LDT = XG_RT + 4;
struct XGArgs {
  const double* colA[kMaxR];
  int ncA;
  const double* ring;
  Win W;               // B columns: the nU union slots (window order)
  int64_t nsr, rows;
  double* part;        // [grid][16 NA][16 NB]
  int tma;             // 1: 16-byte aligned column runs (D even): TMA bulk copies
  uint8_t task[SG_CW][SG_TPW];  // (a << 4) | b
};
template <int NA, int NB>
struct XGCfg {
  static constexpr int nc = 16 * (NA + NB);
  static constexpr size_t stage_bytes = (size_t)nc * XG_LDT * sizeof(double);
  static constexpr int fit = (int)((225 * 1024) / stage_bytes);
  static constexpr int stages = fit > 6 ? 6 : fit;
  static constexpr int look = stages - 2 < 3 ? stages - 2 : 3;
  static constexpr size_t smem = (size_t)stages * stage_bytes;
};

template <int NA, int NB>
__global__ void __launch_bounds__(SG_THREADS, 1) cross_gram_kernel(XGArgs a) {
  using CF = XGCfg<NA, NB>;
  constexpr int NC = CF::nc, ST = CF::stages, LOOK = CF::look, RT = XG_RT, LDT = XG_LDT;
  extern __shared__ double smem[];
  __shared__ __align__(8) uint64_t full[ST], empty[ST];
  __shared__ const double* scol[NC];
  __shared__ int64_t sns[NC];
  for (int col = threadIdx.x; col < NC; col += SG_THREADS) {
    const int cb = col - 16 * NA;
    if (col < 16 * NA) {
      scol[col] = col < a.ncA ? a.colA[col] : nullptr;
      sns[col] = 1;
    } else {
      scol[col] = cb < a.W.nU ? a.ring + (int64_t)a.W.slot[cb] * TILE : nullptr;
      sns[col] = a.nsr;
    }
  }
  for (int i = threadIdx.x; i < ST * NC * LDT; i += SG_THREADS) smem[i] = 0.0;  // padding columns stay 0
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int q = 0; q < ST; ++q) {
      mbar_init(&full[q], 32 * SG_PW);
      mbar_init(&empty[q], SG_CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int64_t ntiles = (a.rows + RT - 1) / RT;
  const int64_t my_tiles = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (warp < SG_PW) {
    // ---- producers: 16-byte cp.async, a half-warp per 32-row column run (tiles never straddle
    // a slab run of 128 rows), 8 columns per 4-warp pass; element copies for the ragged last
    // tile or when the runs are not 16-byte aligned.  No producer arithmetic.
    const int half = lane >> 4, ch = lane & 15;
    for (int64_t it = 0; it < my_tiles + LOOK; ++it) {
      if (it < my_tiles) {
        const int st = (int)(it % ST);
        if (it >= ST) mbar_wait(&empty[st], (uint32_t)(((it / ST) - 1) & 1));
        double* tile = smem + (size_t)st * NC * LDT;
        const int64_t row0 = (blockIdx.x + it * gridDim.x) * RT;
        if (a.tma && row0 + RT <= a.rows) {
          for (int col = 2 * warp + half; col < NC; col += 2 * SG_PW) {
            const double* src = scol[col];
            if (src) cp_async16(tile + col * LDT + 2 * ch, src + sidx(SRef{nullptr, sns[col]}, row0) + 2 * ch);
          }
        } else {
          for (int col = warp; col < NC; col += SG_PW) {
            const double* src = scol[col];
            if (!src) continue;
            const int64_t row = row0 + lane;
            if (row < a.rows) cp_async8(tile + col * LDT + lane, src + sidx(SRef{nullptr, sns[col]}, row));
            else tile[col * LDT + lane] = 0.0;
          }
        }
      }
      cp_async_commit();
      if (it >= LOOK) {
        cp_async_wait<LOOK>();
        mbar_arrive(&full[(int)((it - LOOK) % ST)]);
      }
    }
    cp_async_wait<0>();
  } else {
    const int cwarp = warp - SG_PW;
    const int gid = lane >> 2, tig = lane & 3;
    int sa[SG_TPW], sb[SG_TPW];
    bool has[SG_TPW];
#pragma unroll
    for (int t = 0; t < SG_TPW; ++t) {
      const int v = a.task[cwarp][t];
      has[t] = v != 0xff;
      sa[t] = has[t] ? v >> 4 : 0;
      sb[t] = has[t] ? v & 15 : 0;
    }
    double acc[SG_TPW][8];
#pragma unroll
    for (int t = 0; t < SG_TPW; ++t)
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[t][q] = 0.0;
    for (int64_t it = 0; it < my_tiles; ++it) {
      const int st = (int)(it % ST);
      mbar_wait(&full[st], (uint32_t)((it / ST) & 1));
      const double* tile = smem + (size_t)st * NC * LDT;
#pragma unroll
      for (int t = 0; t < SG_TPW; ++t) {
        if (!has[t]) continue;
        const double* pa = tile + (16 * sa[t] + gid) * LDT + tig;
        const double* pb = tile + (16 * (NA + sb[t]) + gid) * LDT + tig;
#pragma unroll
        for (int kk = 0; kk < RT; kk += 4) {
          const double a0 = pa[kk], a1 = pa[8 * LDT + kk], b0 = pb[kk], b1 = pb[8 * LDT + kk];
          dmma(acc[t][0], acc[t][1], a0, b0);
          dmma(acc[t][2], acc[t][3], a0, b1);
          dmma(acc[t][4], acc[t][5], a1, b0);
          dmma(acc[t][6], acc[t][7], a1, b1);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    double* out = a.part + (int64_t)blockIdx.x * (16 * NA) * (16 * NB);
#pragma unroll
    for (int t = 0; t < SG_TPW; ++t) {
      if (!has[t]) continue;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int bi = 16 * sa[t] + 8 * (q >> 1), bj = 16 * sb[t] + 8 * (q & 1);
        out[(bi + gid) * (16 * NB) + bj + 2 * tig] = acc[t][2 * q];
        out[(bi + gid) * (16 * NB) + bj + 2 * tig + 1] = acc[t][2 * q + 1];
      }
    }
  }
}

__global__ void __launch_bounds__(256) cross_reduce(const double* __restrict__ part, int nblk, int lda, int ldb, int m,
                                                    int n, double* __restrict__ C) {
  const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int idx = (int)(gt / GR_TPE), sub = (int)(gt % GR_TPE);
  const int i = idx / n, j = idx % n;
  const bool act = idx < m * n;
  double s = 0.0;
  if (act)
    for (int b = sub; b < nblk; b += GR_TPE) s += part[(int64_t)b * lda * ldb + i * ldb + j];
  for (int o = GR_TPE / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (act && sub == 0) C[i * n + j] = s;
}

// host: all NA x NB pairs cost 4 DMMAs per k-step; round-robin over the sub-partitions
bool xg_tasks(int na, int nb, XGArgs& a) {
  std::memset(a.task, 0xff, sizeof(a.task));
  int cnt[4] = {0, 0, 0, 0}, q = 0;
  for (int x = 0; x < na; ++x)
    for (int y = 0; y < nb; ++y, ++q) {
      const int b = q % 4, slot = cnt[b] / 4, w = b + 4 * (cnt[b] % 4);
      if (slot >= SG_TPW) return false;
      a.task[w][slot] = (uint8_t)((x << 4) | y);
      ++cnt[b];
    }
  return true;
}

template <int NA, int NB>
hrom_status launch_cross(hrom_ctx* c, XGArgs& a, int grid) {
  const size_t smem = XGCfg<NA, NB>::smem;
  HROM_CK(cudaFuncSetAttribute(cross_gram_kernel<NA, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cross_gram_kernel<NA, NB><<<grid, SG_THREADS, smem, c->st>>>(a);
  HROM_LAUNCH_CK();
  return HROM_OK;
}

// ---------------- G7: incremental gathered Gram ----------------
// S-hat moves little from one step to the next (measured churn ~0.1-1 % of its cells at config
// 4), and the union window shifts by one snapshot.  So the Gram of the old columns over the rows
// of S-hat_{k+1} is the previous one plus the Gram of the entering rows minus that of the leaving
// rows (kept per ring slot in double-double), while the columns that are new every step -- the
// newest snapshot and the HDM values b -- come from two GEMVs over all S-hat rows (memory-bound,
// no DMMA).  Re-initialised by the full gathered Gram at a re-base, after set-window/explicit
// masks, or when the previous step was not the preceding hybrid step.

// S-hat GEMVs: v_new[i] = sum_r x_i x_new, v_b[i] = sum_r x_i b, bb = sum_r b^2 over the rows of
// S-hat (x = slot - rho, b = src_b - rho).  Lanes own consecutive rows (one slot load per warp
// instruction = 32 consecutive list DOFs, coalesced); warp w of the CTA owns slots w, w + 8, ...;
// GV_U row chunks in flight per lane (1 with both product vectors, 2 for the band rows' one).
// Per-CTA partials [blk][2 nU + 1], reduced in fixed order.
constexpr int GV_T = 256, GV_W = GV_T / 32;
// dynamic shared memory of gemv_gather_kernel: two stages of (3 + SPW) values x 32 lanes per warp and chunk
constexpr size_t gv_smem(int spw, int gv_u) { return (size_t)2 * GV_W * gv_u * (3 + spw) * 32 * sizeof(double); }
// NEWCOL = false, BANDOUT = true: the seam-band part of the new window Gram row (H10): one
// product vector b = gamma_k on the band rows, partials [blk][nU + 1] ([nU] = sum b^2).
// DD = false: plain fp64 accumulation (the gathered Gram of the gappy normal equations when
// gather_precision = 1, G11; lo parts stay 0)
// NT: threads per block (GV_T for every current launch).
template <int SPW, bool NEWCOL = true, bool BANDOUT = false, bool DD = true, int GV_U = NEWCOL ? 1 : 2, int NT = GV_T>
__global__ void __launch_bounds__(NT, NT == GV_T ? 2 : 1) gemv_gather_kernel(Geo g, Win W, const double* __restrict__ ring,
                                                           const SRef rho, const int32_t* __restrict__ list,
                                                           const int32_t* __restrict__ count, const SRef src_b,
                                                           double* __restrict__ vpart, const double* __restrict__ C) {
  constexpr int NW = NT / 32;
  __shared__ double red[NW][2 * SPW + 1], redl[NW][2 * SPW + 1];
  __shared__ double s_bias;
  if (threadIdx.x == 0) {  // accumulator bias from the window Gram's diagonal (dd.cuh gram_bias)
    double mc = 0.0;
    for (int s2 = 0; s2 < W.nU; ++s2) mc = fmax(mc, C[W.slot[s2] * (kMaxSlots + 1)]);
    s_bias = gram_bias(mc);
  }
  __syncthreads();
  const double bias = DD ? s_bias : 0.0;
  const int nU = W.nU, nS = *count;
  const int64_t total = (int64_t)nS * g.c;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const SRef slab{nullptr, g.nsr};
  const double* xnew_col = ring + (int64_t)W.slot[nU - 1] * TILE;
  int coff[SPW];  // slab offsets of the warp's slots (-1: none); 32-bit to save registers
#pragma unroll
  for (int j = 0; j < SPW; ++j) {
    const int sl = warp + NW * j;
    coff[j] = sl < nU ? W.slot[sl] * TILE : -1;
  }
  // double-double accumulators (G11): these GEMVs are rows / columns of the POD's and the
  // gappy normal equations' Grams
  double an[SPW], ab[SPW], anl[SPW], abl[SPW];
#pragma unroll
  for (int j = 0; j < SPW; ++j) {
    an[j] = ab[j] = bias;
    anl[j] = abl[j] = 0.0;
  }
  double bb = bias, bbl = 0.0;
  const int64_t gstep = (int64_t)gridDim.x * 32 * GV_U;
  // the S-hat list entries of the next chunk are fetched one iteration ahead (the value loads
  // depend on them: without the prefetch every chunk pays two dependent memory latencies)
  int32_t lnext[GV_U];
  auto fetch_list = [&](int64_t b0) {
#pragma unroll
    for (int u = 0; u < GV_U; ++u) {
      const int64_t t = b0 + 32 * u + lane;
      lnext[u] = 0;
      if (t < total) {
        const int var = (int)t / nS;
        lnext[u] = __ldg(list + ((int)t - var * nS));
      }
    }
  };
  if constexpr (NEWCOL) {
    // Value loads run one chunk ahead of the arithmetic through shared memory (cp.async, no
    // registers): stage[s][warp][u][k][lane], k = rho, x_new, b, the warp's SPW slots.  Every lane
    // reads back only what it copied itself; the sums run in the same order as before.
    constexpr int NV = 3 + SPW;
    extern __shared__ double gv_stage[];
    double* mystage = gv_stage + (size_t)warp * GV_U * NV * 32 + lane;
    constexpr size_t STG = (size_t)NW * GV_U * NV * 32;  // doubles per stage
    auto issue = [&](int64_t b0, const int32_t* lcell, int st) {
  #pragma unroll
      for (int u = 0; u < GV_U; ++u) {
        const int64_t t = b0 + 32 * u + lane;
        if (t < total) {
          const int var = (int)t / nS;
          const int64_t e = (int64_t)var * g.N + lcell[u];
          const int64_t se = sidx(slab, e);
          double* d = mystage + st * STG + (size_t)u * NV * 32;
          cp_async8(d, rho.p + sidx(rho, e));
          if (NEWCOL) cp_async8(d + 32, xnew_col + se);
          cp_async8(d + 64, src_b.p + sidx(src_b, e));
  #pragma unroll
          for (int j = 0; j < SPW; ++j)
            if (coff[j] >= 0) cp_async8(d + (3 + j) * 32, ring + coff[j] + se);
        }
      }
      cp_async_commit();
    };
    const int64_t base0 = (int64_t)blockIdx.x * 32 * GV_U;
    fetch_list(base0);
    {
      int32_t l0[GV_U];
  #pragma unroll
      for (int u = 0; u < GV_U; ++u) l0[u] = lnext[u];
      issue(base0, l0, 0);
    }
    fetch_list(base0 + gstep);
    int st = 0;
    for (int64_t base = base0; base < total; base += gstep) {
      {
        int32_t l1[GV_U];
  #pragma unroll
        for (int u = 0; u < GV_U; ++u) l1[u] = lnext[u];
        issue(base + gstep, l1, st ^ 1);  // the next chunk's values (a chunk past the end copies nothing)
      }
      fetch_list(base + 2 * gstep);
      cp_async_wait<1>();  // this chunk's copies have landed (the next chunk's may be in flight)
  #pragma unroll
      for (int u = 0; u < GV_U; ++u) {
        const int64_t t = base + 32 * u + lane;
        if (t >= total) continue;
        const double* d = mystage + st * STG + (size_t)u * NV * 32;
        const double r = d[0];
        const double x = (NEWCOL ? d[32] : 0.0) - r, y = d[64] - r;
  #pragma unroll
        for (int j = 0; j < SPW; ++j) {
          const double v = (coff[j] >= 0 ? d[(3 + j) * 32] : 0.0) - r;
          if (DD) {
            if (NEWCOL) biased_fma(an[j], anl[j], v, x);
            biased_fma(ab[j], abl[j], v, y);
          } else {
            if (NEWCOL) an[j] = fma(v, x, an[j]);
            ab[j] = fma(v, y, ab[j]);
          }
        }
        if (warp == 0) {
          if (DD) biased_fma(bb, bbl, y, y);
          else bb = fma(y, y, bb);
        }
      }
      st ^= 1;
    }
    cp_async_wait<0>();
  } else {
    // band rows (one product vector, two chunks in flight in registers): runs beside the positivity
    // pass, where the staged variant's shared memory cost more than its overlap gained
    fetch_list((int64_t)blockIdx.x * 32 * GV_U);
    for (int64_t base = (int64_t)blockIdx.x * 32 * GV_U; base < total; base += gstep) {
      int32_t lcur[GV_U];
  #pragma unroll
      for (int u = 0; u < GV_U; ++u) lcur[u] = lnext[u];
      fetch_list(base + gstep);
      int64_t se[GV_U];
      double xn[GV_U], bv[GV_U], r[GV_U];
      bool ok[GV_U];
  #pragma unroll
      for (int u = 0; u < GV_U; ++u) {
        const int64_t t = base + 32 * u + lane;
        ok[u] = t < total;
        int64_t e = 0;
        if (ok[u]) {
          const int var = (int)t / nS;
          e = (int64_t)var * g.N + lcur[u];
        }
        se[u] = sidx(slab, e);
        r[u] = ok[u] ? __ldg(rho.p + sidx(rho, e)) : 0.0;
        xn[u] = (NEWCOL && ok[u]) ? __ldg(xnew_col + se[u]) : 0.0;
        bv[u] = ok[u] ? __ldg(src_b.p + sidx(src_b, e)) : 0.0;
      }
      double val[GV_U][SPW];
  #pragma unroll
      for (int u = 0; u < GV_U; ++u)
  #pragma unroll
        for (int j = 0; j < SPW; ++j) val[u][j] = (ok[u] && coff[j] >= 0) ? __ldg(ring + coff[j] + se[u]) : 0.0;
  #pragma unroll
      for (int u = 0; u < GV_U; ++u) {
        if (!ok[u]) continue;
        const double x = xn[u] - r[u], y = bv[u] - r[u];
  #pragma unroll
        for (int j = 0; j < SPW; ++j) {
          const double v = val[u][j] - r[u];
          if (DD) {
            if (NEWCOL) biased_fma(an[j], anl[j], v, x);
            biased_fma(ab[j], abl[j], v, y);
          } else {
            if (NEWCOL) an[j] = fma(v, x, an[j]);
            ab[j] = fma(v, y, ab[j]);
          }
        }
        if (warp == 0) {
          if (DD) biased_fma(bb, bbl, y, y);
          else bb = fma(y, y, bb);
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < SPW; ++j) {  // remove the bias (exact)
    an[j] -= bias;
    ab[j] -= bias;
  }
  bb -= bias;
  auto wsum = [&](double& h, double& l) {
    for (int o = 16; o > 0; o >>= 1) {
      const double oh = __shfl_xor_sync(0xffffffffu, h, o), ol = __shfl_xor_sync(0xffffffffu, l, o);
      dd_add(h, l, oh, ol);
    }
  };
#pragma unroll
  for (int j = 0; j < SPW; ++j) {
    if (NEWCOL) wsum(an[j], anl[j]);
    wsum(ab[j], abl[j]);
    if (lane == 0) {
      red[warp][j] = an[j];
      redl[warp][j] = anl[j];
      red[warp][SPW + j] = ab[j];
      redl[warp][SPW + j] = abl[j];
    }
  }
  wsum(bb, bbl);
  if (lane == 0) {
    red[warp][2 * SPW] = bb;
    redl[warp][2 * SPW] = bbl;
  }
  __syncthreads();
  // partials [blk][n][hi, lo]
  if (BANDOUT) {
    double* out = vpart + (int64_t)blockIdx.x * (nU + 1) * 2;
    for (int k = threadIdx.x; k <= nU; k += NT) {
      const int wi = k == nU ? 0 : k % NW, ji = k == nU ? 2 * SPW : SPW + k / NW;
      out[2 * k] = red[wi][ji];
      out[2 * k + 1] = redl[wi][ji];
    }
    return;
  }
  double* out = vpart + (int64_t)blockIdx.x * (2 * nU + 1) * 2;
  for (int k = threadIdx.x; k <= 2 * nU; k += NT) {
    int wi, ji;
    if (k == 2 * nU) {
      wi = 0;
      ji = 2 * SPW;
    } else {
      const int sl = k < nU ? k : k - nU;  // slot sl is (warp sl % NW, j = sl / NW)
      wi = sl % NW;
      ji = (k < nU ? 0 : SPW) + sl / NW;
    }
    out[2 * k] = red[wi][ji];
    out[2 * k + 1] = redl[wi][ji];
  }
}

// fixed-order reduce of the GEMV partials [blk][n][hi, lo], 16 threads per entry -> v[n][hi, lo]
__global__ void __launch_bounds__(256) vpart_reduce(const double* __restrict__ vpart, int nblk, int n,
                                                    double* __restrict__ v) {
  const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int k = (int)(gt / GR_TPE), sub = (int)(gt % GR_TPE);
  double h = 0.0, l = 0.0;
  if (k < n)
    for (int b = sub; b < nblk; b += GR_TPE) dd_add(h, l, vpart[((int64_t)b * n + k) * 2], vpart[((int64_t)b * n + k) * 2 + 1]);
  for (int o = GR_TPE / 2; o > 0; o >>= 1) {
    const double oh = __shfl_xor_sync(0xffffffffu, h, o), ol = __shfl_xor_sync(0xffffffffu, l, o);
    dd_add(h, l, oh, ol);
  }
  if (k < n && sub == 0) {
    v[2 * k] = h;
    v[2 * k + 1] = l;
  }
}

// Ks (by ring slot) <- update; Rout ((nU+1)^2, union order, hi / lo) <- the gathered Gram for
// the solve.  init: Rout holds a full gathered Gram -> Ks = Rout.  Otherwise: old-old block
// += R+ - R- (all double-double), newest-slot row/column and the b row/column from the reduced
// GEMV partials v[n][hi, lo].
__global__ void __launch_bounds__(512) kinc_update_kernel(Win W, int init, const double* __restrict__ Rp,
                                                          const double* __restrict__ Rpl,
                                                          const double* __restrict__ Rm, const double* __restrict__ Rml,
                                                          const double* __restrict__ v, double* __restrict__ Khi,
                                                          double* __restrict__ Klo, double* __restrict__ Rout,
                                                          double* __restrict__ Routl) {
  const int nU = W.nU, ldr = nU + 1;
  if (init) {
    for (int idx = threadIdx.x; idx < nU * nU; idx += blockDim.x) {
      const int i = idx / nU, j = idx % nU;
      Khi[W.slot[i] * kMaxSlots + W.slot[j]] = Rout[i * ldr + j];
      Klo[W.slot[i] * kMaxSlots + W.slot[j]] = Routl[i * ldr + j];
    }
    return;
  }
  for (int idx = threadIdx.x; idx < nU * nU; idx += blockDim.x) {
    const int i = idx / nU, j = idx % nU;
    const int si = W.slot[i], sj = W.slot[j];
    double hi, lo;
    if (i == nU - 1 || j == nU - 1) {
      const int k = i == nU - 1 ? j : i;
      hi = v[2 * k];
      lo = v[2 * k + 1];
    } else {
      hi = Khi[si * kMaxSlots + sj];
      lo = Klo[si * kMaxSlots + sj];
      dd_add(hi, lo, Rp[i * ldr + j], Rpl[i * ldr + j]);
      dd_add(hi, lo, -Rm[i * ldr + j], -Rml[i * ldr + j]);
    }
    Khi[si * kMaxSlots + sj] = hi;
    Klo[si * kMaxSlots + sj] = lo;
    Rout[i * ldr + j] = hi;
    Routl[i * ldr + j] = lo;
  }
  for (int i = threadIdx.x; i < nU; i += blockDim.x) {
    Rout[i * ldr + nU] = Rout[nU * ldr + i] = v[2 * (nU + i)];
    Routl[i * ldr + nU] = Routl[nU * ldr + i] = v[2 * (nU + i) + 1];
  }
  if (threadIdx.x == 0) {
    Rout[nU * ldr + nU] = v[4 * nU];
    Routl[nU * ldr + nU] = v[4 * nU + 1];
  }
}

// deterministic fixed-order reduction over CTAs, 16 threads per entry (block-strided sub-sums,
// then a fixed shuffle tree); C[i][j] for i <= j mirrored
__global__ void __launch_bounds__(256) gram_reduce(const double* __restrict__ part, int nblk, int ncp, int ncol,
                                                   double* __restrict__ C, int ldc, const int32_t* __restrict__ map) {
  const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int idx = (int)(gt / GR_TPE), sub = (int)(gt % GR_TPE);
  const int i = idx / ncol, j = idx % ncol;
  const bool act = idx < ncol * ncol && i <= j;
  double s = 0.0;
  if (act)
    for (int b = sub; b < nblk; b += GR_TPE) s += part[(int64_t)b * ncp * ncp + i * ncp + j];
  for (int o = GR_TPE / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (act && sub == 0) {
    const int ci = map ? map[i] : i, cj = map ? map[j] : j;
    C[ci * ldc + cj] = s;
    C[cj * ldc + ci] = s;
  }
}

// double-double version of gram_reduce: partials [blk][ncp][ncp][hi, lo] -> (Chi, Clo)
__global__ void __launch_bounds__(256) gram_reduce_dd(const double* __restrict__ part, int nblk, int ncp, int ncol,
                                                      double* __restrict__ Chi, double* __restrict__ Clo, int ldc,
                                                      const int32_t* __restrict__ map) {
  const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int idx = (int)(gt / GR_TPE), sub = (int)(gt % GR_TPE);
  const int i = idx / ncol, j = idx % ncol;
  const bool act = idx < ncol * ncol && i <= j;
  double h = 0.0, l = 0.0;
  if (act)
    for (int b = sub; b < nblk; b += GR_TPE) {
      const double* p = part + ((int64_t)b * ncp * ncp + i * ncp + j) * 2;
      dd_add(h, l, p[0], p[1]);
    }
  for (int o = GR_TPE / 2; o > 0; o >>= 1) {
    const double oh = __shfl_xor_sync(0xffffffffu, h, o), ol = __shfl_xor_sync(0xffffffffu, l, o);
    dd_add(h, l, oh, ol);
  }
  if (act && sub == 0) {
    const int ci = map ? map[i] : i, cj = map ? map[j] : j;
    Chi[ci * ldc + cj] = h;
    Chi[cj * ldc + ci] = h;
    Clo[ci * ldc + cj] = l;
    Clo[cj * ldc + ci] = l;
  }
}

// smem layout of the eigen-solve workspace (eig.cuh), shared by the basis and solve kernels
struct EigLayout {
  int ldn, ldz;
  bool fac_smem;
  bool z_smem;     // eigenvectors in shared memory (else the caller's global gz: w = 128 windows)
  size_t doubles;  // dynamic smem doubles (matrix [+ Z] + vectors [+ LU workspace])
  size_t bytes;
};
__host__ __device__ inline EigLayout eig_layout(int n, int nvec_cap) {
  EigLayout L;
  L.ldn = n + (n & 1) + 1;  // odd strides: column accesses are bank-conflict free
  L.ldz = nvec_cap | 1;
  const size_t zsz = (size_t)n * L.ldz;
  const size_t core = (size_t)L.ldn * L.ldn + 8 * kMaxSlots + 64;
  L.z_smem = (core + zsz) * 8 <= 216 * 1024;
  const size_t base = core + (L.z_smem ? zsz : 0);
  const size_t fac = (size_t)4 * n * L.ldz + ((size_t)n * L.ldz + 7) / 8;
  L.fac_smem = (base + fac) * 8 <= 216 * 1024;
  L.doubles = base + (L.fac_smem ? fac : 0);
  L.bytes = L.doubles * sizeof(double);
  return L;
}
// dynamic doubles of the eigen-solve workspace with the LU factors in (fac_smem) or out of smem
__host__ __device__ inline size_t eig_doubles(int n, int nvec_cap, bool fac_smem, bool z_global = false) {
  const EigLayout L = eig_layout(n, nvec_cap);
  const bool zs = L.z_smem && !z_global;
  const size_t core = (size_t)L.ldn * L.ldn + 8 * kMaxSlots + 64 + (zs ? (size_t)n * L.ldz : 0);
  const size_t fac = (size_t)4 * n * L.ldz + ((size_t)n * L.ldz + 7) / 8;
  return core + (fac_smem ? fac : 0);
}
__device__ inline EigWork eig_work(double* sm, int n, const EigLayout& L, double* gfac, double* gz = nullptr) {
  EigWork W;
  double* p = sm + (size_t)L.ldn * L.ldn;
  if (L.z_smem) {
    W.Z = p;
    p += (size_t)n * L.ldz;
  } else {
    W.Z = gz;
  }
  W.ldz = L.ldz;
  W.d = p; p += kMaxSlots;
  W.e = p; p += kMaxSlots;
  W.tau = p; p += kMaxSlots;
  W.vv = p; p += kMaxSlots;
  W.pp = p; p += kMaxSlots;
  W.lam = p; p += kMaxSlots;
  p += 2 * kMaxSlots;  // caller scratch (mrow, rhs / y)
  W.red = p; p += 64;
  W.fac = L.fac_smem ? p : gfac;
  W.swp = (uint8_t*)(W.fac + (size_t)4 * n * L.ldz);
  return W;
}

// basis from the shifted Gram (one CTA): M = X^T X by lagged centring in double-double (G11),
// all w eigenvectors of hi(M) (eig.cuh) -> Zf, lam; M (hi, lo) -> Mh, Ml for refine_kernel
__global__ void __launch_bounds__(512) basis_kernel(const double* __restrict__ C, const double* __restrict__ Clo,
                                                    int ldc, Win W, double* __restrict__ Mh, double* __restrict__ Ml,
                                                    double* __restrict__ Zf, double* __restrict__ lam_out,
                                                    int32_t* __restrict__ reff_out, double* __restrict__ gfac,
                                                    double* __restrict__ gz) {
  extern __shared__ double sm[];
  const int w = W.w, nU = W.nU;
  const EigLayout L = eig_layout(w, w);
  const int ldn = L.ldn;
  double* M = sm;
  const EigWork E = eig_work(sm, w, L, gfac, gz);
  double* mrow = E.lam + kMaxSlots;  // kMaxSlots: m_i (hi)
  double* mrowl = mrow + kMaxSlots;  // kMaxSlots: m_i (lo)
  __shared__ double msum[2 * kMaxSlots];
  __shared__ double s_mu[2];
  const int tid = threadIdx.x;
  // m_i = (1/w) sum_{p<w} C[x_i][u_p];  mu = (1/w^2) sum_{p,q<w} C[u_p][u_q]  (double-double)
  for (int i = tid; i < w; i += blockDim.x) {
    const int xi = W.slot[nU - w + i];
    double h = 0.0, l = 0.0;
    for (int p = 0; p < w; ++p) dd_add(h, l, C[xi * ldc + W.slot[p]], Clo[xi * ldc + W.slot[p]]);
    dd_div1(h, l, (double)w);
    mrow[i] = h;
    mrowl[i] = l;
  }
  for (int p = tid; p < w; p += blockDim.x) {
    double h = 0.0, l = 0.0;
    for (int q = 0; q < w; ++q) dd_add(h, l, C[W.slot[p] * ldc + W.slot[q]], Clo[W.slot[p] * ldc + W.slot[q]]);
    msum[2 * p] = h;
    msum[2 * p + 1] = l;
  }
  __syncthreads();
  if (tid == 0) {
    double h = 0.0, l = 0.0;
    for (int p = 0; p < w; ++p) dd_add(h, l, msum[2 * p], msum[2 * p + 1]);
    dd_div1(h, l, (double)w * (double)w);
    s_mu[0] = h;
    s_mu[1] = l;
  }
  __syncthreads();
  for (int idx = tid; idx < w * w; idx += blockDim.x) {
    const int i = idx / w, j = idx % w;
    const int xi = W.slot[nU - w + i], xj = W.slot[nU - w + j];
    // when psi_prev == psi_cur (bootstrap, nU == w) this is the plain centred Gram
    double h = C[xi * ldc + xj], l = Clo[xi * ldc + xj];
    dd_add(h, l, -mrow[i], -mrowl[i]);
    dd_add(h, l, -mrow[j], -mrowl[j]);
    dd_add(h, l, s_mu[0], s_mu[1]);
    M[i * ldn + j] = h;
    Mh[i * w + j] = h;
    Ml[i * w + j] = l;
  }
  __syncthreads();
  // every eigenvector (the refinement couples the kept modes with all the others)
  const int nv = sym_eig(M, w, ldn, E, w, -1.0, reff_out + 10);
  if (tid == 0) reff_out[8] = 0;
  for (int idx = tid; idx < w * w; idx += blockDim.x) {
    const int i = idx / w, j = idx % w;
    Zf[idx] = j < nv ? E.Z[i * E.ldz + j] : 0.0;
  }
  for (int i = tid; i < w; i += blockDim.x) lam_out[i] = E.lam[i];
}

// One step of the Ogita-Aishima eigenvector refinement (G11) of the eigen-decomposition of
// hi(M), driven by the double-double M: R = I - Z^T Z, S = Z^T M Z (double-double),
// lam~_i = S_ii / (1 - R_ii), E_ij = (S_ij + lam~_j R_ij) / (lam~_j - lam~_i) for
// |lam~_i - lam~_j| > delta = 2 (||S - diag lam~||_F + ||M||_F ||R||_F), else R_ij / 2;
// Z' = Z + Z E.  The subspace error eps lambda_1 / gap of the fp64 solve becomes its square,
// i.e. the eigenvectors are those of the exact Gram to fp64 precision (SVD class, A15).
// Then r_eff = #{j < r : lam~_j >= cut lam~_0} (consecutive), sign (largest |Z_ij| positive),
// A = V_r L_r^-1/2 (column-major A[j*w + i]), lam_out = lam~.
constexpr int RF_T = 512;
__device__ __forceinline__ double rf_block_sum(double v, double* red) {  // all threads get the sum
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  for (int q = 0; q < RF_T / 32; ++q) t += red[q];  // fixed order
  return t;
}
// Workspace: 5 w (w | 1) doubles in shared memory, or in the global scratch gws (wide windows,
// w > 72: L2-resident)
__global__ void __launch_bounds__(RF_T) refine_kernel(const double* __restrict__ Mh, const double* __restrict__ Ml,
                                                      const double* __restrict__ Zg, int w, int r, double cut,
                                                      double* __restrict__ lam_io, double* __restrict__ Aout,
                                                      int32_t* __restrict__ reff_out, double* gws) {
  extern __shared__ double sm[];
  const int ld = w | 1;
  const size_t B = (size_t)w * ld;
  double* Z = gws ? gws : sm;  // Z[a * ld + j]
  double* Yh = Z + B;        // Y = M Z (hi), then E
  double* Yl = Yh + B;       // Y (lo), then Z' = Z + Z E
  double* M0 = Yl + B;       // M (hi), then S (rounded)
  double* M1 = M0 + B;       // M (lo), then R (rounded)
  __shared__ double lt[kMaxSlots], red[RF_T / 32];
  __shared__ int s_reff;
  const int tid = threadIdx.x;
  for (int idx = tid; idx < w * w; idx += RF_T) {
    const int a = idx / w, j = idx % w;
    Z[a * ld + j] = Zg[idx];
    M0[a * ld + j] = Mh[idx];
    M1[a * ld + j] = Ml[idx];
  }
  __syncthreads();
  // Y = M Z (double-double); ||M||_F
  double fm = 0.0;
  for (int idx = tid; idx < w * w; idx += RF_T) {
    const int a = idx / w, j = idx % w;
    double h = 0.0, l = 0.0;
    for (int b = 0; b < w; ++b) {
      const double z = Z[b * ld + j];
      dd_fma(h, l, M0[a * ld + b], z);
      l = fma(M1[a * ld + b], z, l);
    }
    dd_norm(h, l);
    Yh[a * ld + j] = h;
    Yl[a * ld + j] = l;
    fm += M0[a * ld + j] * M0[a * ld + j];
  }
  const double normM = sqrt(rf_block_sum(fm, red));  // (its barriers also retire M)
  // S = Z^T Y and R = I - Z^T Z (double-double, rounded to fp64) over M's storage
  for (int idx = tid; idx < w * w; idx += RF_T) {
    const int i = idx / w, j = idx % w;
    double sh = 0.0, sl = 0.0, rh = i == j ? 1.0 : 0.0, rl = 0.0;
    for (int a = 0; a < w; ++a) {
      const double zi = Z[a * ld + i];
      dd_fma(sh, sl, zi, Yh[a * ld + j]);
      sl = fma(zi, Yl[a * ld + j], sl);
      dd_fma(rh, rl, -zi, Z[a * ld + j]);
    }
    M0[i * ld + j] = sh + sl;
    M1[i * ld + j] = rh + rl;
  }
  __syncthreads();
  for (int i = tid; i < w; i += RF_T) lt[i] = M0[i * ld + i] / (1.0 - M1[i * ld + i]);
  __syncthreads();
  double fs = 0.0, fr = 0.0;
  for (int idx = tid; idx < w * w; idx += RF_T) {
    const int i = idx / w, j = idx % w;
    const double sv = i == j ? M0[i * ld + i] - lt[i] : M0[i * ld + j];
    fs += sv * sv;
    fr += M1[i * ld + j] * M1[i * ld + j];
  }
  const double nS = sqrt(rf_block_sum(fs, red));
  const double nR = sqrt(rf_block_sum(fr, red));
  const double delta = 2.0 * (nS + normM * nR);
  // E (over Y hi)
  for (int idx = tid; idx < w * w; idx += RF_T) {
    const int i = idx / w, j = idx % w;
    double e;
    if (i == j) e = 0.5 * M1[i * ld + i];
    else if (fabs(lt[i] - lt[j]) > delta) e = (M0[i * ld + j] + lt[j] * M1[i * ld + j]) / (lt[j] - lt[i]);
    else e = 0.5 * M1[i * ld + j];
    Yh[i * ld + j] = e;
  }
  __syncthreads();
  // Z' = Z + Z E (over Y lo)
  for (int idx = tid; idx < w * w; idx += RF_T) {
    const int a = idx / w, j = idx % w;
    double s = 0.0;
    for (int i = 0; i < w; ++i) s = fma(Z[a * ld + i], Yh[i * ld + j], s);
    Yl[a * ld + j] = Z[a * ld + j] + s;
  }
  __syncthreads();
  // sign: the largest |Z'_ij| of each vector (ties: lowest i) positive (A15)
  for (int j = tid; j < w; j += RF_T) {
    int im = 0;
    double vm = -1.0;
    for (int i = 0; i < w; ++i) {
      const double a = fabs(Yl[i * ld + j]);
      if (a > vm) {
        vm = a;
        im = i;
      }
    }
    if (Yl[im * ld + j] < 0.0)
      for (int i = 0; i < w; ++i) Yl[i * ld + j] = -Yl[i * ld + j];
  }
  if (tid == 0) {
    int re = 0;
    const double l0 = lt[0];
    if (l0 > 0.0)
      for (int j = 0; j < min(r, w); ++j) {
        if (lt[j] >= cut * l0) ++re;
        else break;
      }
    s_reff = re;
    *reff_out = re;
  }
  __syncthreads();
  const int re = s_reff;
  for (int idx = tid; idx < w * r; idx += RF_T) {
    const int i = idx % w, j = idx / w;  // A column-major: A[j*w + i]
    Aout[j * w + i] = (j < re) ? Yl[i * ld + j] / sqrt(lt[j]) : 0.0;
  }
  for (int i = tid; i < w; i += RF_T) lam_io[i] = lt[i];
}

// H5 (one CTA): K = lagged centring of the gathered R (A14), G = A^T K_XX A, g = A^T K_Xb,
// y = G^+ g with the 1e-12 cut on lambda (A13), c = A y.
// Fast path: Cholesky G = L L^T.  lambda_min >= 1 / trace(G^-1) = 1 / ||L^-1||_F^2 and
// lambda_max <= ||G||_F, so when 1 / ||L^-1||_F^2 >= 1e-10 ||G||_F no eigenvalue is within
// two orders of magnitude of the cut and y = G^-1 g exactly; otherwise the eigen route (eig.cuh).
// debug timestamps (thread 0 of block 0; t nullable)
__device__ __forceinline__ void sstamp(long long* t, int& i) {
  if (t && blockIdx.x == 0 && threadIdx.x == 0 && i < 16) {
    long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    t[i] = gt;
  }
  ++i;
}

constexpr int SV_T = 256, SV_W = SV_T / 32;
// Workspace of solve_kernel (offsets in doubles of the dynamic shared memory; a buffer whose
// flag is set lives in the global scratch instead -- wide windows).  Region X holds K (hi, lo)
// and T (hi, lo) until G is formed, then the eigen-solve workspace of the pinv route.
struct SolveLayout {
  size_t as, x, kh, kl, th, tl, gh, gl, lm, mp, vec, eig, total;
  bool kg, tg;  // K / T in global memory
};
__host__ __device__ inline SolveLayout solve_layout(int w, int r, bool kg, bool tg, size_t eig_doubles) {
  SolveLayout S;
  S.kg = kg;
  S.tg = tg;
  const size_t ka = (size_t)(w + 1) * (w + 1), ta = (size_t)(w + 1) * r;
  S.as = 0;
  S.x = S.as + ta;
  S.kh = S.x;
  S.kl = S.kh + (kg ? 0 : ka);
  S.th = S.kl + (kg ? 0 : ka);
  S.tl = S.th + (tg ? 0 : ta);
  const size_t xend = S.tl + (tg ? 0 : ta);
  S.eig = S.x;
  S.gh = (xend > S.eig + eig_doubles ? xend : S.eig + eig_doubles);
  S.gl = S.gh + (size_t)r * (r | 1);
  S.lm = S.gl + (size_t)r * (r | 1);
  S.mp = S.lm + (size_t)r * (r | 1);  // mp, mpl, mc, mcl: 4 (kMaxW + 2)
  S.vec = S.mp + 4 * (kMaxW + 2);     // g hi, g lo, y, u, misc, res: 6 kMaxSlots + 2 SV_W
  S.total = S.vec + 6 * kMaxSlots + 2 * SV_W;
  return S;
}

// out(m, n) = sum_p X[m ldx + p] Y[n ldy + p] over p < P, m < M, n < N (shared memory operands).
// Register blocks of RM rows (stride ceil(M / RM): consecutive threads walk consecutive X rows,
// conflict-free for odd ldx) x CN columns (warp-uniform: broadcast Y loads); RM x CN independent
// FMA chains per thread.  Only blocks with some n >= m when UPPER.
template <int RM, int CN, bool UPPER, class F>
__device__ __forceinline__ void smem_gemm_nt(const double* X, int ldx, const double* Y, int ldy, int M, int N, int P,
                                             F store) {
  const int mb = (M + RM - 1) / RM, nb = (N + CN - 1) / CN;
  for (int blk = threadIdx.x; blk < mb * nb; blk += blockDim.x) {
    const int m0 = blk % mb, n0 = CN * (blk / mb);
    if (UPPER && n0 + CN - 1 < m0) continue;
    const double* xr[RM];
    const double* yr[CN];
#pragma unroll
    for (int q = 0; q < RM; ++q) xr[q] = X + (int64_t)min(m0 + q * mb, M - 1) * ldx;
#pragma unroll
    for (int c = 0; c < CN; ++c) yr[c] = Y + (int64_t)min(n0 + c, N - 1) * ldy;
    double acc[RM][CN];
#pragma unroll
    for (int q = 0; q < RM; ++q)
#pragma unroll
      for (int c = 0; c < CN; ++c) acc[q][c] = 0.0;
    for (int p = 0; p < P; ++p) {
      double xv[RM];
#pragma unroll
      for (int q = 0; q < RM; ++q) xv[q] = xr[q][p];
#pragma unroll
      for (int c = 0; c < CN; ++c) {
        const double yv = yr[c][p];
#pragma unroll
        for (int q = 0; q < RM; ++q) acc[q][c] += xv[q] * yv;
      }
    }
#pragma unroll
    for (int q = 0; q < RM; ++q)
#pragma unroll
      for (int c = 0; c < CN; ++c)
        if (m0 + q * mb < M && n0 + c < N) store(m0 + q * mb, n0 + c, acc[q][c]);
  }
}

// One warp, in place: the n x n SPD matrix M (leading dimension ld, odd) -> its lower Cholesky
// factor L (right-looking; lanes own rows i = lane, lane + 32).  Uniformly false when a pivot is
// not positive.  Kept as loops: this code runs once per launch, so an unrolled body would be
// instruction-fetch bound.
__device__ bool chol_warp(double* M, int ld, int n, double* dinv) {
  const int lane = threadIdx.x & 31;
  for (int j = 0; j < n; ++j) {
    const double d = M[j * ld + j];
    if (!(d > 0.0)) return false;
    const double ljj = sqrt(d), rj = 1.0 / ljj;
    __syncwarp();
    for (int i = lane; i < n; i += 32) {
      if (i > j) M[i * ld + j] *= rj;
      else if (i == j) {
        M[j * ld + j] = ljj;
        dinv[j] = rj;
      }
    }
    __syncwarp();
    for (int i = lane; i < n; i += 32) {
      if (i <= j) continue;
      const double lij = M[i * ld + j];
      double* Mi = M + i * ld;
      int k = j + 1;
      for (; k + 3 <= i; k += 4) {  // loads first: four independent updates in flight
        const double a0 = M[k * ld + j], a1 = M[(k + 1) * ld + j], a2 = M[(k + 2) * ld + j], a3 = M[(k + 3) * ld + j];
        const double b0 = Mi[k], b1 = Mi[k + 1], b2 = Mi[k + 2], b3 = Mi[k + 3];
        Mi[k] = b0 - lij * a0;
        Mi[k + 1] = b1 - lij * a1;
        Mi[k + 2] = b2 - lij * a2;
        Mi[k + 3] = b3 - lij * a3;
      }
      for (; k <= i; ++k) Mi[k] -= lij * M[k * ld + j];
    }
    __syncwarp();
  }
  return true;
}

// Forward substitution L x = e_c for the columns c = warp, warp + SV_W, ... (< n: columns of
// L^-1, only their squared norms are kept) and c = n (x = L^-1 g -> u).  Lanes own rows
// lane, lane + 32; the CPW columns of a warp advance together (independent chains).
constexpr int SV_CPW = (kMaxR + 1 + SV_W - 1) / SV_W;
__device__ double trinv_cols(const double* Lm, int ld, int n, const double* dinv, const double* g, double* u) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double x[SV_CPW][2];
#pragma unroll
  for (int m = 0; m < SV_CPW; ++m) {
    const int c = warp + SV_W * m;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int i = lane + 32 * h;
      x[m][h] = c < n ? (i == c ? 1.0 : 0.0) : (c == n && i < n ? g[i] : 0.0);
    }
  }
  for (int k = 0; k < n; ++k) {  // (the columns c > k are still zero above the diagonal)
    const double rk = dinv[k];
    const double l0 = lane > k && lane < n ? Lm[lane * ld + k] : 0.0;
    const double l1 = lane + 32 > k && lane + 32 < n ? Lm[(lane + 32) * ld + k] : 0.0;
#pragma unroll
    for (int m = 0; m < SV_CPW; ++m) {
      if (warp + SV_W * m > n) break;
      const double xk = __shfl_sync(0xffffffffu, k < 32 ? x[m][0] : x[m][1], k & 31) * rk;
      if (lane == (k & 31)) {
        if (k < 32) x[m][0] = xk;
        else x[m][1] = xk;
      }
      x[m][0] -= l0 * xk;
      x[m][1] -= l1 * xk;
    }
  }
  double tr = 0.0;
#pragma unroll
  for (int m = 0; m < SV_CPW; ++m) {
    const int c = warp + SV_W * m;
    if (c < n) tr += x[m][0] * x[m][0] + x[m][1] * x[m][1];
    if (c == n) {
      u[lane] = x[m][0];
      if (lane + 32 < n) u[lane + 32] = x[m][1];
    }
  }
  for (int o = 16; o > 0; o >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, o);
  return tr;
}

// One warp: back substitution L^T y = u (lanes own rows k = lane, lane + 32)
__device__ void trsolve_t_warp(const double* Lm, int ld, int n, const double* dinv, const double* u, double* y) {
  const int lane = threadIdx.x & 31;
  double v0 = lane < n ? u[lane] : 0.0, v1 = lane + 32 < n ? u[lane + 32] : 0.0;
  for (int i = n - 1; i >= 0; --i) {
    const double yi = __shfl_sync(0xffffffffu, i < 32 ? v0 : v1, i & 31) * dinv[i];
    if (lane == (i & 31)) {
      if (i < 32) v0 = yi;
      else v1 = yi;
    }
    if (lane < i) v0 -= Lm[i * ld + lane] * yi;
    if (lane + 32 < i) v1 -= Lm[i * ld + lane + 32] * yi;
  }
  if (lane < n) y[lane] = v0;
  if (lane + 32 < n) y[lane + 32] = v1;
}

// One warp: forward substitution L x = b (lanes own rows lane, lane + 32)
__device__ void trsolve_warp(const double* Lm, int ld, int n, const double* dinv, const double* b, double* x) {
  const int lane = threadIdx.x & 31;
  double v0 = lane < n ? b[lane] : 0.0, v1 = lane + 32 < n ? b[lane + 32] : 0.0;
  for (int k = 0; k < n; ++k) {
    const double xk = __shfl_sync(0xffffffffu, k < 32 ? v0 : v1, k & 31) * dinv[k];
    if (lane == (k & 31)) {
      if (k < 32) v0 = xk;
      else v1 = xk;
    }
    if (lane > k && lane < n) v0 -= Lm[lane * ld + k] * xk;
    if (lane + 32 > k && lane + 32 < n) v1 -= Lm[(lane + 32) * ld + k] * xk;
  }
  if (lane < n) x[lane] = v0;
  if (lane + 32 < n) x[lane + 32] = v1;
}

// out(m, n) = sum_p X(m, p) Y(n, p), X and Y double-double (lo parts nullable), layouts
// X[m ldx + p], Y[n ldy + p]; CN outputs per thread share the X loads; UPPER: only n >= m
template <int CN, bool UPPER, class F>
__device__ __forceinline__ void smem_gemm_dd(const double* Xh, const double* Xl, int ldx, const double* Yh,
                                             const double* Yl, int ldy, int M, int N, int P, F store) {
  const int nb = (N + CN - 1) / CN;
  for (int blk = threadIdx.x; blk < M * nb; blk += blockDim.x) {
    const int m = blk % M, n0 = CN * (blk / M);
    if (UPPER && n0 + CN - 1 < m) continue;
    double h[CN], l[CN];
#pragma unroll
    for (int c = 0; c < CN; ++c) h[c] = l[c] = 0.0;
    const double* xh = Xh + (int64_t)m * ldx;
    const double* xl = Xl ? Xl + (int64_t)m * ldx : nullptr;
    for (int p = 0; p < P; ++p) {
      const double a = xh[p], al = xl ? xl[p] : 0.0;
#pragma unroll
      for (int c = 0; c < CN; ++c) {
        const int n = min(n0 + c, N - 1);
        const double b = Yh[(int64_t)n * ldy + p];
        dd_fma(h[c], l[c], a, b);
        l[c] = fma(al, b, l[c]);
        if (Yl) l[c] = fma(a, Yl[(int64_t)n * ldy + p], l[c]);
      }
    }
#pragma unroll
    for (int c = 0; c < CN; ++c)
      if (n0 + c < N) {
        dd_norm(h[c], l[c]);
        store(m, n0 + c, h[c], l[c]);
      }
  }
}

// H5 (one CTA), double-double throughout (G11): K = lagged centring of the gathered R (A14),
// T = K_XX A, G = A^T T, g = A^T K_Xb; y = G^+ g with the 1e-12 cut on lambda (A13) from
// hi(G) -- Cholesky (fast path, trace(G^-1) bound as before) or the eigen route -- refined
// twice against the double-double G and g (residual g - G y in double-double); c = A y.
__global__ void __launch_bounds__(SV_T) solve_kernel(const double* __restrict__ R, const double* __restrict__ Rlo,
                                                     Win W, int r, const double* __restrict__ A,
                                                     const int32_t* __restrict__ reffp, double cut,
                                                     double* __restrict__ y_out, double* __restrict__ c_out,
                                                     int32_t* __restrict__ status, double* __restrict__ gfac,
                                                     bool fac_smem, double* __restrict__ Kg, double* __restrict__ Tg,
                                                     long long* tdbg, double* __restrict__ gz) {
  extern __shared__ double sm[];
  int ts = 0;
  sstamp(tdbg, ts);
  const int re = *reffp;
  const int w = W.w, nU = W.nU, xoff = nU - w, ldk = w + 1, lda = w + 1, ldl = re | 1, ldg = r | 1;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  EigLayout L = eig_layout(re > 0 ? re : 1, re > 0 ? re : 1);
  L.fac_smem = fac_smem;  // the host sized the smem for r >= r_eff: its choice is safe
  if (gz) L.z_smem = false;  // eigenvectors in global memory (w = 128, r = 64: config 5)
  const SolveLayout S = solve_layout(w, r, Kg != nullptr, Tg != nullptr, eig_doubles(r, r, fac_smem, gz != nullptr));
  const size_t ka = (size_t)(w + 1) * (w + 1), ta = (size_t)(w + 1) * r;
  double* As = sm + S.as;  // As[j * lda + i] = A[j * w + i]
  double* Kh = S.kg ? Kg : sm + S.kh;
  double* Kl = S.kg ? Kg + ka : sm + S.kl;
  double* Th = S.tg ? Tg : sm + S.th;  // T[j * lda + i]
  double* Tl = S.tg ? Tg + ta : sm + S.tl;
  double* Gh = sm + S.gh;  // G[i * ldg + j]
  double* Gl = sm + S.gl;
  double* Lm = sm + S.lm;  // Lm[i * ldl + k]
  double* mp = sm + S.mp;
  double* mpl = mp + (kMaxW + 2);
  double* mc = mpl + (kMaxW + 2);
  double* mcl = mc + (kMaxW + 2);
  double* gh = sm + S.vec;
  double* gl = gh + kMaxSlots;
  double* y = gl + kMaxSlots;
  double* u = y + kMaxSlots;
  double* misc = u + kMaxSlots;
  double* res = misc + kMaxSlots;
  double* wtr = res + kMaxSlots;  // per-warp partials (2 SV_W)
  double* Ge = sm + S.eig;        // eigen route: matrix + workspace over region X
  const EigWork E = eig_work(Ge, re > 0 ? re : 1, L, gfac, gz);
  const int ldn = L.ldn;
  __shared__ double gm[6];
  __shared__ int s_fast;
  // ---- centring of R into K (same algebra as the window Gram, A14), double-double ----
  const int ldr = nU + 1;
  for (int i = tid; i < w * re; i += nt) As[(i / w) * lda + (i % w)] = A[i];
  for (int a = warp; a <= nU; a += SV_W) {  // warp per row of R
    double ph = 0.0, pl = 0.0, ch = 0.0, cl = 0.0;
    for (int q = lane; q < nU; q += 32) {
      const double vh = R[a * ldr + q], vl = Rlo[a * ldr + q];
      if (q < w) dd_add(ph, pl, vh, vl);
      if (q >= xoff) dd_add(ch, cl, vh, vl);
    }
    for (int o = 16; o > 0; o >>= 1) {
      double oh = __shfl_xor_sync(0xffffffffu, ph, o), ol = __shfl_xor_sync(0xffffffffu, pl, o);
      dd_add(ph, pl, oh, ol);
      oh = __shfl_xor_sync(0xffffffffu, ch, o);
      ol = __shfl_xor_sync(0xffffffffu, cl, o);
      dd_add(ch, cl, oh, ol);
    }
    if (lane == 0) {
      dd_div1(ph, pl, (double)w);
      dd_div1(ch, cl, (double)w);
      mp[a] = ph;
      mpl[a] = pl;
      mc[a] = ch;
      mcl[a] = cl;
    }
  }
  __syncthreads();
  sstamp(tdbg, ts);
  if (tid == 0) {
    double pp = 0.0, ppl = 0.0, pc = 0.0, pcl = 0.0, cc = 0.0, ccl = 0.0;
    for (int q = 0; q < w; ++q) {
      dd_add(pp, ppl, mp[q], mpl[q]);
      dd_add(pc, pcl, mc[q], mcl[q]);
      dd_add(cc, ccl, mc[xoff + q], mcl[xoff + q]);
    }
    dd_div1(pp, ppl, (double)w);
    dd_div1(pc, pcl, (double)w);
    dd_div1(cc, ccl, (double)w);
    gm[0] = pp;
    gm[1] = ppl;
    gm[2] = pc;
    gm[3] = pcl;
    gm[4] = cc;
    gm[5] = ccl;
  }
  __syncthreads();
  for (int idx = tid; idx < ldk * ldk; idx += nt) {
    const int i = idx / ldk, j = idx % ldk;
    double h, l;
    if (i < w && j < w) {
      const int a = xoff + i, b = xoff + j;
      h = R[a * ldr + b];
      l = Rlo[a * ldr + b];
      dd_add(h, l, -mp[a], -mpl[a]);
      dd_add(h, l, -mp[b], -mpl[b]);
      dd_add(h, l, gm[0], gm[1]);
    } else if (i < w || j < w) {
      const int a = xoff + (i < w ? i : j);
      h = R[a * ldr + nU];
      l = Rlo[a * ldr + nU];
      dd_add(h, l, -mc[a], -mcl[a]);
      dd_add(h, l, -mp[nU], -mpl[nU]);
      dd_add(h, l, gm[2], gm[3]);
    } else {
      h = R[nU * ldr + nU];
      l = Rlo[nU * ldr + nU];
      dd_add(h, l, -mc[nU], -mcl[nU]);
      dd_add(h, l, -mc[nU], -mcl[nU]);
      dd_add(h, l, gm[4], gm[5]);
    }
    Kh[i * ldk + j] = h;
    Kl[i * ldk + j] = l;
  }
  __syncthreads();
  sstamp(tdbg, ts);
  // ---- T = K_XX A, g = A^T K_Xb, G = A^T T (double-double) ----
  smem_gemm_dd<4, false>(Kh, Kl, ldk, As, nullptr, lda, w, re, w, [&](int i, int j, double h, double l) {
    Th[j * lda + i] = h;
    Tl[j * lda + i] = l;
  });
  for (int j = tid; j < re; j += nt) {
    double h = 0.0, l = 0.0;
    for (int p = 0; p < w; ++p) {
      const double a = As[j * lda + p];
      dd_fma(h, l, a, Kh[p * ldk + w]);
      l = fma(a, Kl[p * ldk + w], l);
    }
    dd_norm(h, l);
    gh[j] = h;
    gl[j] = l;
  }
  __syncthreads();
  sstamp(tdbg, ts);
  smem_gemm_dd<4, true>(Th, Tl, lda, As, nullptr, lda, re, re, w, [&](int i, int j, double h, double l) {
    if (j >= i) {
      Gh[i * ldg + j] = Gh[j * ldg + i] = h;
      Gl[i * ldg + j] = Gl[j * ldg + i] = l;
    }
  });
  __syncthreads();
  sstamp(tdbg, ts);
  // ---- fast path: Cholesky hi(G) = L L^T + trace(G^-1) bound ----
  double gf = 0.0;  // ||G||_F^2
  for (int idx = tid; idx < re * re; idx += nt) {
    const double v = Gh[(idx / re) * ldg + idx % re];
    Lm[(idx / re) * ldl + idx % re] = v;
    gf += v * v;
  }
  for (int o = 16; o > 0; o >>= 1) gf += __shfl_xor_sync(0xffffffffu, gf, o);
  if (lane == 0) wtr[SV_W + warp] = gf;
  __syncthreads();
  if (warp == 0) {
    const bool f = re > 0 && chol_warp(Lm, ldl, re, misc);
    if (lane == 0) s_fast = f ? 1 : 0;
  }
  __syncthreads();
  bool ok = s_fast != 0;
  sstamp(tdbg, ts);
  if (ok) {
    const double tr = trinv_cols(Lm, ldl, re, misc, gh, u);  // trace(G^-1) = ||L^-1||_F^2, u = L^-1 g
    if (lane == 0) wtr[warp] = tr;
    __syncthreads();
    if (warp == 0) {
      double t = lane < SV_W ? wtr[lane] : 0.0;
      gf = lane < SV_W ? wtr[SV_W + lane] : 0.0;
      for (int o = 16; o > 0; o >>= 1) {
        t += __shfl_xor_sync(0xffffffffu, t, o);
        gf += __shfl_xor_sync(0xffffffffu, gf, o);
      }
      const bool f = t > 0.0 && isfinite(t) && 1.0 / t >= 1e-10 * sqrt(gf);
      if (f) trsolve_t_warp(Lm, ldl, re, misc, u, y);
      if (lane == 0) s_fast = f ? 1 : 0;
    }
    __syncthreads();
    ok = s_fast != 0;
  }
  sstamp(tdbg, ts);
  int nk = 0;
  if (!ok) {
    // eigen route on hi(G) (its workspace overlays K and T, dead now)
    for (int idx = tid; idx < re * re; idx += nt) Ge[(idx / re) * ldn + idx % re] = Gh[(idx / re) * ldg + idx % re];
    __syncthreads();
    nk = re > 0 ? sym_eig(Ge, re, ldn, E, re, cut) : 0;
    for (int kk = tid; kk < nk; kk += nt) {
      double d = 0.0;
      for (int p = 0; p < re; ++p) d += E.Z[p * E.ldz + kk] * gh[p];
      misc[kk] = d / E.lam[kk];
    }
    __syncthreads();
    for (int i = tid; i < re; i += nt) {
      double s = 0.0;
      for (int kk = 0; kk < nk; ++kk) s += E.Z[i * E.ldz + kk] * misc[kk];
      y[i] = s;
    }
    __syncthreads();
  }
  if (tid == 0) {
    *status = (!ok && (re == 0 || !(E.lam[0] > 0.0))) ? 1 : 0;
    status[7] = ok ? 0 : 1;  // fast path / eigen route
  }
  // ---- iterative refinement: res = g - G y in double-double, y += G^+ res (same route) ----
  for (int itr = 0; itr < 2 && re > 0; ++itr) {
    for (int i = tid; i < re; i += nt) {
      double h = gh[i], l = gl[i];
      for (int j = 0; j < re; ++j) {
        dd_fma(h, l, -Gh[i * ldg + j], y[j]);
        l = fma(-Gl[i * ldg + j], y[j], l);
      }
      res[i] = h + l;
    }
    __syncthreads();
    if (ok) {
      if (warp == 0) {
        trsolve_warp(Lm, ldl, re, misc, res, u);
        __syncwarp();
        trsolve_t_warp(Lm, ldl, re, misc, u, res);
        __syncwarp();
        for (int i = lane; i < re; i += 32) y[i] += res[i];
      }
    } else {
      for (int kk = tid; kk < nk; kk += nt) {
        double d = 0.0;
        for (int p = 0; p < re; ++p) d += E.Z[p * E.ldz + kk] * res[p];
        misc[kk] = d / E.lam[kk];
      }
      __syncthreads();
      for (int i = tid; i < re; i += nt) {
        double s = 0.0;
        for (int kk = 0; kk < nk; ++kk) s += E.Z[i * E.ldz + kk] * misc[kk];
        y[i] += s;
      }
    }
    __syncthreads();
  }
  sstamp(tdbg, ts);
  for (int i = tid; i < kMaxR; i += nt) y_out[i] = (i < re) ? y[i] : 0.0;
  for (int i = tid; i < w; i += nt) {
    double s = 0.0;
    for (int j = 0; j < re; ++j) s += As[j * lda + i] * y[j];
    c_out[i] = s;
  }
}

// Phi_{k+1}[:, j] = X A[:, j] (materialised; tests/config 5), psi_cur
// H12 lift on FP64 tensor cores: Phi[:, j] = (X - psi_prev 1^T) A[:, j] (D x r, column-major),
// psi_cur = mean of the last w slots.  Warp-specialised like the gathered Gram: LF_PW = 8
// producer warps (LF_NH = 4 threads per tile row, window means split over the four) gather a
// 64-DOF tile of all nU window slots (cp.async), form X - psi_prev in place and publish it; 16 consumer warps each own one 8-DOF block x four 8-mode blocks of the product
// with A (staged in smem once per CTA) and write Phi straight from the accumulators.
constexpr int LF_RT = 64, LF_LDT = LF_RT + 4, LF_PW = 8, LF_CW = 16, LF_T = 32 * (LF_PW + LF_CW);
constexpr int LF_NH = 32 * LF_PW / LF_RT;  // producer threads per tile row
constexpr int LF_STAGES = 2, LF_NCOL = kMaxW + 5, LF_LDA = kMaxR + 4;

__global__ void __launch_bounds__(LF_T, 1) lift_kernel(Geo g, Win W, const double* __restrict__ ring,
                                                       const double* __restrict__ A, const int32_t* __restrict__ reffp,
                                                       double* __restrict__ phi, double* __restrict__ psi) {
  extern __shared__ double smem[];
  __shared__ __align__(8) uint64_t full[LF_STAGES], empty[LF_STAGES];
  const int re = *reffp;
  const int w = W.w, nU = W.nU, xoff = nU - w;
  const int kpad = (w + 3) & ~3;
  double* As = smem;                                // kpad x LF_LDA: As[i][j] = A[j*w + i]
  double* tiles = smem + (size_t)kpad * LF_LDA;     // LF_STAGES x LF_NCOL x LF_LDT
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < kpad * LF_LDA; i += LF_T) {
    const int si = i / LF_LDA, j = i % LF_LDA;
    As[i] = (si < w && j < re) ? A[j * w + si] : 0.0;
  }
  for (int i = threadIdx.x; i < LF_STAGES * LF_NCOL * LF_LDT; i += LF_T) tiles[i] = 0.0;
  if (threadIdx.x == 0) {
    for (int q = 0; q < LF_STAGES; ++q) {
      mbar_init(&full[q], 32 * LF_PW);
      mbar_init(&empty[q], LF_CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int64_t ntiles = (g.D + LF_RT - 1) / LF_RT;
  const int64_t my_tiles = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const double inv_w = 1.0 / (double)w;
  if (warp < LF_PW) {
    // producers: LF_NH threads per tile row (hf = column part); the row's window means are
    // LF_NH part sums exchanged through shared memory
    __shared__ double xch[LF_NH][2][LF_RT];
    const int kt = threadIdx.x, k = kt & (LF_RT - 1), hf = kt / LF_RT;
    const SRef slab{nullptr, g.nsr};
    const int s0 = (w * hf) / LF_NH, s1 = (w * (hf + 1)) / LF_NH;  // this thread's part of each mean
    int64_t e_prev = -1;
    for (int64_t it = 0; it <= my_tiles; ++it) {
      int64_t e_cur = -1;
      if (it < my_tiles) {
        const int st = (int)(it % LF_STAGES);
        if (it >= LF_STAGES) mbar_wait(&empty[st], (uint32_t)(((it / LF_STAGES) - 1) & 1));
        double* tile = tiles + (size_t)st * LF_NCOL * LF_LDT;
        const int64_t e0 = (blockIdx.x + it * gridDim.x) * LF_RT, e = e0 + k;
        if (e0 + LF_RT <= g.D) {
          // full tile: 16-byte cp.async, a half-warp per 32-row column run (a 64-row tile lies
          // inside one slab run of 128 rows, so each run is 256 contiguous bytes)
          const int hw = kt >> 4, ch = kt & 15;
          for (int q = hw; q < 2 * nU; q += 2 * LF_PW) {
            const int col = q >> 1, part = q & 1;
            cp_async16(tile + col * LF_LDT + 32 * part + 2 * ch,
                       ring + (int64_t)W.slot[col] * TILE + sidx(slab, e0 + 32 * part) + 2 * ch);
          }
          e_cur = e;
        } else if (e < g.D) {
          const int64_t se = sidx(slab, e);
          for (int col = hf; col < nU; col += LF_NH) cp_async8(tile + col * LF_LDT + k, ring + (int64_t)W.slot[col] * TILE + se);
          e_cur = e;
        } else {
          for (int col = hf; col < nU; col += LF_NH) tile[col * LF_LDT + k] = 0.0;
        }
      }
      cp_async_commit();
      if (it >= 1) {
        cp_async_wait<1>();
        asm volatile("bar.sync 1, %0;\n" ::"n"(32 * LF_PW) : "memory");  // rows landed by other lanes
        const int ps = (int)((it - 1) % LF_STAGES);
        double* tile = tiles + (size_t)ps * LF_NCOL * LF_LDT;
        double p2[2] = {0.0, 0.0}, c2[2] = {0.0, 0.0};
        if (e_prev >= 0) {
          int s = s0;
          for (; s + 2 <= s1; s += 2) {
            p2[0] += tile[s * LF_LDT + k];
            p2[1] += tile[(s + 1) * LF_LDT + k];
            c2[0] += tile[(xoff + s) * LF_LDT + k];
            c2[1] += tile[(xoff + s + 1) * LF_LDT + k];
          }
          if (s < s1) {
            p2[0] += tile[s * LF_LDT + k];
            c2[0] += tile[(xoff + s) * LF_LDT + k];
          }
          xch[hf][0][k] = p2[0] + p2[1];
          xch[hf][1][k] = c2[0] + c2[1];
        }
        asm volatile("bar.sync 1, %0;\n" ::"n"(32 * LF_PW) : "memory");  // both halves' sums
        if (e_prev >= 0) {
          double sp = xch[0][0][k], sc = xch[0][1][k];
#pragma unroll
          for (int h = 1; h < LF_NH; ++h) {
            sp += xch[h][0][k];
            sc += xch[h][1][k];
          }
          if (psi && hf == 0) psi[e_prev] = sc * inv_w;
          const double pp = sp * inv_w;
          for (int s = xoff + s0; s < xoff + s1; ++s) tile[s * LF_LDT + k] -= pp;
        }
        mbar_arrive(&full[ps]);
      }
      e_prev = e_cur;
    }
    cp_async_wait<0>();
  } else {
    const int cw = warp - LF_PW;
    // r_eff <= 32: each warp takes 2 column blocks so that all 16 warps work (else 4 blocks)
    const int nbk = re > 32 ? 4 : 2;
    const int db = cw & 7, mb0 = (cw >> 3) * nbk;
    const int gid = lane >> 2, tig = lane & 3;
    for (int64_t it = 0; it < my_tiles; ++it) {
      const int st = (int)(it % LF_STAGES);
      mbar_wait(&full[st], (uint32_t)((it / LF_STAGES) & 1));
      const double* tile = tiles + (size_t)st * LF_NCOL * LF_LDT;
      double acc[4][2];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q][0] = acc[q][1] = 0.0;
      if (phi && 8 * mb0 < re) {
        if (nbk == 4) {
          for (int kk = 0; kk < kpad; kk += 4) {
            const double av = tile[(xoff + kk + tig) * LF_LDT + 8 * db + gid];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const double bv = As[(kk + tig) * LF_LDA + 8 * (mb0 + q) + gid];
              dmma(acc[q][0], acc[q][1], av, bv);
            }
          }
        } else {
          for (int kk = 0; kk < kpad; kk += 4) {
            const double av = tile[(xoff + kk + tig) * LF_LDT + 8 * db + gid];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const double bv = As[(kk + tig) * LF_LDA + 8 * (mb0 + q) + gid];
              dmma(acc[q][0], acc[q][1], av, bv);
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      if (phi) {
        const int64_t e0 = (blockIdx.x + it * gridDim.x) * LF_RT + 8 * db + gid;
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int j = 8 * (mb0 + q) + 2 * tig + h;
            if (q < nbk && j < re && e0 < g.D) phi[(int64_t)j * g.D + e0] = acc[q][h];
          }
      }
    }
  }
}

// double-double Gram (G11): GGDSmall / GGDWide consumers, partials reduced into (Chi, Clo)
hrom_status run_gather_gram_dd(hrom_ctx* c, GGArgs& a, int ncol, int grid, double* Chi, double* Clo, int ldc,
                               const int32_t* map) {
  a.part = c->b.part;
  int ncp;
  if (ncol <= GGDSmall::ncp) {
    ncp = GGDSmall::ncp;
    if ((int64_t)grid * ncp * ncp * 2 > c->b.part_len) return HROM_E_INVALID;
    HROM_CK(cudaFuncSetAttribute(gather_gram_kernel<GGDSmall>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)GGDSmall::smem));
    gather_gram_kernel<GGDSmall><<<grid, GGDSmall::threads, GGDSmall::smem, c->st>>>(a);
  } else if (ncol <= GGDWide::ncp) {
    ncp = GGDWide::ncp;
    if ((int64_t)grid * ncp * ncp * 2 > c->b.part_len) return HROM_E_INVALID;
    HROM_CK(cudaFuncSetAttribute(gather_gram_kernel<GGDWide>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)GGDWide::smem));
    gather_gram_kernel<GGDWide><<<grid, GGDWide::threads, GGDWide::smem, c->st>>>(a);
  } else {
    return HROM_E_INVALID;
  }
  HROM_LAUNCH_CK();
  ++c->nlaunch;
  gram_reduce_dd<<<(ncol * ncol * GR_TPE + 255) / 256, 256, 0, c->st>>>(c->b.part, grid, ncp, ncol, Chi, Clo, ldc,
                                                                         map);
  HROM_LAUNCH_CK();
  ++c->nlaunch;
  return HROM_OK;
}

// launch the pipelined Gram (both modes) and reduce its per-CTA partials into C
hrom_status run_gather_gram(hrom_ctx* c, GGArgs& a, int ncol, int grid, double* dev_C, int ldc,
                                   const int32_t* map) {
  a.part = c->b.part;
  int ncp;
  if (ncol <= GGSmall::ncp) {
    ncp = GGSmall::ncp;
    if ((int64_t)grid * ncp * ncp > c->b.part_len) return HROM_E_INVALID;
    HROM_CK(cudaFuncSetAttribute(gather_gram_kernel<GGSmall>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)GGSmall::smem));
    gather_gram_kernel<GGSmall><<<grid, GGSmall::threads, GGSmall::smem, c->st>>>(a);
  } else if (ncol <= GGWide::ncp) {
    ncp = GGWide::ncp;
    if ((int64_t)grid * ncp * ncp > c->b.part_len) return HROM_E_INVALID;
    HROM_CK(cudaFuncSetAttribute(gather_gram_kernel<GGWide>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)GGWide::smem));
    gather_gram_kernel<GGWide><<<grid, GGWide::threads, GGWide::smem, c->st>>>(a);
  } else {
    return HROM_E_INVALID;
  }
  HROM_LAUNCH_CK();
  ++c->nlaunch;
  gram_reduce<<<(ncol * ncol * GR_TPE + 255) / 256, 256, 0, c->st>>>(c->b.part, grid, ncp, ncol, dev_C, ldc, map);
  HROM_LAUNCH_CK();
  ++c->nlaunch;
  return HROM_OK;
}

}  // namespace

// Full Gram of ncol columns over `rows` rows, shifted by rho (nullable): dev_C[i*ldc+j].
hrom_status gram_full(hrom_ctx* c, const double* const* dev_cols, int64_t ns, int ncol, int64_t rows, SRef rho,
                      double* dev_C, int ldc, const int32_t* map) {
  const int grid = c->basis_pending ? c->nsm - 1 : c->nsm;
  {
    SGArgs sg{};
    sg.cols = dev_cols;
    sg.ns = ns;
    sg.rows = rows;
    sg.rho = rho;
    sg.part = c->b.part;
    sg.ncp = 16 * (ncol / 16) + 16;
    if ((int64_t)grid * sg.ncp * sg.ncp <= c->b.part_len && run_slab_gram(c, sg, ncol, grid) == HROM_OK) {
      ++c->nlaunch;
      gram_reduce<<<(ncol * ncol * GR_TPE + 255) / 256, 256, 0, c->st>>>(c->b.part, grid, sg.ncp, ncol, dev_C, ldc,
                                                                         map);
      HROM_LAUNCH_CK();
      ++c->nlaunch;
      return HROM_OK;
    }
  }
  GGArgs a{};
  a.mode = 0;
  a.cols = dev_cols;
  a.ns = ns;
  a.ncol0 = ncol;
  a.rows = rows;
  a.rho = rho;
  return run_gather_gram(c, a, ncol, c->basis_pending ? c->nsm - 1 : c->nsm, dev_C, ldc, map);
}

// Window Gram of the basis path in double-double (G11): dev_Chi / dev_Clo[i*ldc+j] (mapped),
// rows of ncol slab columns shifted by rho, FMA consumers (gather_gram_kernel<GGD*>)
hrom_status gram_full_dd(hrom_ctx* c, const double* const* dev_cols, int64_t ns, int ncol, int64_t rows, SRef rho,
                         double* dev_Chi, double* dev_Clo, int ldc, const int32_t* map) {
  GGArgs a{};
  a.mode = 0;
  a.cols = dev_cols;
  a.ns = ns;
  a.ncol0 = ncol;
  a.rows = rows;
  a.rho = rho;
  return run_gather_gram_dd(c, a, ncol, c->basis_pending ? c->nsm - 1 : c->nsm, dev_Chi, dev_Clo, ldc, map);
}

// config 5: C = Phi^T S over the w + 1 window columns (S = the ring slots of the current window)
hrom_status project_window(hrom_ctx* c, const double* const* phicols, int m, double* dev_C) {
  const Win& W = c->win;
  const int na = (m + 15) / 16, nb = (W.nU + 15) / 16;
  XGArgs a{};
  for (int i = 0; i < m; ++i) a.colA[i] = phicols[i];
  a.ncA = m;
  a.ring = c->b.ring;
  a.W = W;
  a.nsr = c->g.nsr;
  a.rows = c->g.D;
  a.part = c->b.part;
  a.tma = (c->g.D % 2 == 0) ? 1 : 0;
  for (int i = 0; i < m; ++i)
    if ((reinterpret_cast<uintptr_t>(phicols[i]) & 15) != 0) a.tma = 0;
  const int grid = c->basis_pending ? c->nsm - 1 : c->nsm;
  if ((int64_t)grid * 256 * na * nb > c->b.part_len || !xg_tasks(na, nb, a)) return HROM_E_INVALID;
  hrom_status s = HROM_E_INVALID;
#define XG_CASE(A_, B_) \
  if (na == A_ && nb == B_) s = launch_cross<A_, B_>(c, a, grid);
  XG_CASE(1, 1) XG_CASE(1, 2) XG_CASE(1, 3) XG_CASE(1, 4) XG_CASE(1, 5)
  XG_CASE(2, 2) XG_CASE(2, 3) XG_CASE(2, 4) XG_CASE(2, 5) XG_CASE(4, 9)
#undef XG_CASE
  if (s != HROM_OK) return s;
  ++c->nlaunch;
  cross_reduce<<<(m * W.nU * GR_TPE + 255) / 256, 256, 0, c->st>>>(c->b.part, grid, 16 * na, 16 * nb, m, W.nU, dev_C);
  HROM_LAUNCH_CK();
  ++c->nlaunch;
  return HROM_OK;
}

// gathered Gram R of [U, b] over the rows of S-hat (shifted by rho, union order, (nU+1)^2,
// double-double: hi in b.eigV, lo in b.Rlo); the lagged centring is applied by solve_kernel.
// Two halves, so that a row slab (slab.cu) can sum the ranks' partials in between: `partial`
// leaves this context's sums over the rows of the given lists -- the full Gram in (b.eigV, b.Rlo),
// or, on the incremental route (G7), the Grams of the entering / leaving rows in b.Rd and the two
// GEMVs' reduced values behind the GEMV partials -- and `finish` turns them into R (and the
// per-slot state Khi / Klo).  Every quantity is linear in the rows.
hrom_status gram_gathered_partial(hrom_ctx* c, SRef src_b, const GatherLists* L) {
  GGArgs a{};
  a.g = c->g;
  a.W = c->win;
  a.ring = c->b.ring;
  a.rho = c->rho_ref();
  a.list = L ? L->S : c->b.lists + (int64_t)L_S * c->g.N;
  a.count = L ? L->nS : c->b.counts + L_S;
  a.src_b = src_b;
  a.mode = 1;
  // while the one-CTA eigen-solve of the previous update holds an SM (side stream), leave it
  // out: a static tile split with one block left over would double the time
  const int grid = c->basis_pending ? c->nsm - 1 : c->nsm;
  const int ncol = a.W.nU + 1;
  double* R = c->b.eigV;
  double* Rl = c->b.Rlo;
  auto gram = [&](GGArgs& aa, double* hi, double* lo) -> hrom_status {
    return run_gather_gram_dd(c, aa, ncol, grid, hi, lo, ncol, nullptr);
  };
  c->gather_inc = false;
  if (c->P.odeim_points > 0) {  // gappy rows = the DOF rows of the ODEIM points (Eq. 8, 10)
    a.mode = 2;
    a.rowlist = c->b.orows;
    a.nrow2 = c->odeim_n;
    c->kinc_valid = false;
    c->samples_since_gather = 0;
    c->gather_skip_finish = true;
    return gram(a, R, Rl);
  }
  c->gather_skip_finish = false;
  const bool inc = c->P.gather_mode == 0 && c->kinc_valid && c->samples_since_gather == 1 && c->kinc_newest == c->k - 1 &&
                   c->kinc_rebase == c->rebase_k;
  c->gather_inc = inc;
  hrom_status s;
  if (!inc) return gram(a, R, Rl);
  // rows entering and leaving S-hat (cells of the last sampling's churn), double-double
  const size_t S2 = (size_t)(kMaxW + 2) * (kMaxW + 2);
  double* Rp = c->b.Rd;
  double* Rpl = Rp + S2;
  double* Rm = Rp + 2 * S2;
  double* Rml = Rp + 3 * S2;
  GGArgs d = a;
  d.list = L ? L->add : c->b.lists + (int64_t)L_ADD * c->g.N;
  d.count = L ? L->nadd : c->b.counts + L_ADD;
  if ((s = gram(d, Rp, Rpl)) != HROM_OK) return s;
  d.list = L ? L->rem : c->b.lists + (int64_t)L_REM * c->g.N;
  d.count = L ? L->nrem : c->b.counts + L_REM;
  if ((s = gram(d, Rm, Rml)) != HROM_OK) return s;
  // GEMVs of the newest snapshot and of b over all S-hat rows: one wave (2 CTAs per SM), static
  // split that avoids the eigen's SM.  (Tried: 512 threads with 5 slots per warp and 4 row
  // chunks in flight -- 0.64 ms against 0.47 ms for the whole gathered Gram: the 16 warps'
  // redundant rho / x_new / b loads of the same rows cost more than the extra memory-level
  // parallelism gains.)
  const int gblocks = 2 * (c->basis_pending ? c->nsm - 1 : c->nsm);
  const int nv = 2 * a.W.nU + 1;
  if (a.W.nU <= 9 * GV_W)
  {
    HROM_CK(cudaFuncSetAttribute(gemv_gather_kernel<9>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gv_smem(9, 1)));
    gemv_gather_kernel<9><<<gblocks, GV_T, gv_smem(9, 1), c->st>>>(c->g, a.W, a.ring, a.rho, a.list, a.count, src_b,
                                                                   c->b.vpart, c->b.C);
  }
  else
  {
    HROM_CK(cudaFuncSetAttribute(gemv_gather_kernel<17>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gv_smem(17, 1)));
    gemv_gather_kernel<17><<<gblocks, GV_T, gv_smem(17, 1), c->st>>>(c->g, a.W, a.ring, a.rho, a.list, a.count, src_b,
                                                                     c->b.vpart, c->b.C);
  }
  HROM_LAUNCH_CK();
  double* v = gathered_gemv_values(c);
  vpart_reduce<<<(nv * GR_TPE + 255) / 256, 256, 0, c->st>>>(c->b.vpart, gblocks, nv, v);
  HROM_LAUNCH_CK();
  c->nlaunch += 2;
  return HROM_OK;
}

// reduced GEMV values v[2 nU + 1][hi, lo] of the incremental route: behind the largest possible
// block of GEMV partials (fixed place: the same whatever grid the GEMV ran on)
double* gathered_gemv_values(hrom_ctx* c) { return c->b.vpart + (size_t)2 * c->nsm * (2 * kMaxSlots + 2) * 2; }

hrom_status gram_gathered_finish(hrom_ctx* c) {
  if (c->gather_skip_finish) return HROM_OK;
  const Win& W = c->win;
  double* R = c->b.eigV;
  double* Rl = c->b.Rlo;
  if (!c->gather_inc) {
    if (c->P.gather_mode == 0) {
      kinc_update_kernel<<<1, 512, 0, c->st>>>(W, 1, nullptr, nullptr, nullptr, nullptr, nullptr, c->b.Khi, c->b.Klo, R, Rl);
      HROM_LAUNCH_CK();
      ++c->nlaunch;
    }
  } else {
    const size_t S2 = (size_t)(kMaxW + 2) * (kMaxW + 2);
    double* Rp = c->b.Rd;
    kinc_update_kernel<<<1, 512, 0, c->st>>>(W, 0, Rp, Rp + S2, Rp + 2 * S2, Rp + 3 * S2, gathered_gemv_values(c), c->b.Khi,
                                             c->b.Klo, R, Rl);
    HROM_LAUNCH_CK();
    ++c->nlaunch;
  }
  if (c->P.gather_mode == 0) {
    c->kinc_valid = true;
    c->kinc_newest = c->k;
    c->kinc_rebase = c->rebase_k;
  }
  c->samples_since_gather = 0;
  return HROM_OK;
}

hrom_status gram_gathered(hrom_ctx* c, SRef src_b) {
  hrom_status s = gram_gathered_partial(c, src_b, nullptr);
  if (s != HROM_OK) return s;
  return gram_gathered_finish(c);
}

// seam-band part of the new window Gram row (band DOFs' final values), double-double partials
// after the fill's
hrom_status band_gram_rows_list(hrom_ctx* c, const Win& W, SRef v, const int32_t* list, const int32_t* count) {
  if (W.nU > 9 * GV_W) return HROM_E_INVALID;  // the fused row is limited to nU <= 68 anyway
  gemv_gather_kernel<9, false, true><<<c->band_blocks, GV_T, 0, c->st>>>(
      c->g, W, c->b.ring, c->rho_ref(), list, count, v, c->b.gpart + (int64_t)c->fill_blocks * (W.nU + 1) * 2, c->b.C);
  HROM_LAUNCH_CK();
  ++c->nlaunch;
  return HROM_OK;
}

hrom_status band_gram_rows(hrom_ctx* c, const Win& W, SRef v) {
  return band_gram_rows_list(c, W, v, c->b.lists + (int64_t)L_B * c->g.N, c->b.counts + L_B);
}

// gathered Gram of [U, b] over the DOF rows of an explicit cell list (row slabs: the own rows of
// S-hat, or every own cell for the window Gram of the bootstrap), (nU+1)^2 double-double
hrom_status gram_gathered_list(hrom_ctx* c, const Win& W, SRef src_b, const int32_t* list, const int32_t* count,
                               double* Rhi, double* Rlo) {
  GGArgs a{};
  a.g = c->g;
  a.W = W;
  a.ring = c->b.ring;
  a.rho = c->rho_ref();
  a.list = list;
  a.count = count;
  a.src_b = src_b;
  a.mode = 1;
  const int ncol = a.W.nU + 1;
  return run_gather_gram_dd(c, a, ncol, c->basis_pending ? c->nsm - 1 : c->nsm, Rhi, Rlo, ncol, nullptr);
}

hrom_status small_solve(hrom_ctx* c) {
  // the solve reads r_eff on the device: size the workspace for the largest possible (r)
  const int w = c->win.w, r = c->r;
  bool fac = eig_layout(r, r).fac_smem;
  const size_t lim = 220 * 1024 / sizeof(double);
  bool kg = false, tg = false;
  SolveLayout S = solve_layout(w, r, kg, tg, eig_doubles(r, r, fac));
  if (S.total > lim) S = solve_layout(w, r, kg = true, tg, eig_doubles(r, r, fac));  // wide windows: K in global
  if (S.total > lim) S = solve_layout(w, r, kg, tg = true, eig_doubles(r, r, fac));  // ... and T
  if (S.total > lim) S = solve_layout(w, r, kg, tg, eig_doubles(r, r, fac = false));  // ... and the eigen LU
  bool zg = false;  // ... and the eigenvectors of the eigen route (the double-double G, g need the room)
  if (S.total > lim) S = solve_layout(w, r, kg, tg, eig_doubles(r, r, fac, zg = true));
  if (S.total > lim) return HROM_E_INVALID;
  const size_t smem = S.total * sizeof(double);
  HROM_CK(cudaFuncSetAttribute(solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  solve_kernel<<<1, SV_T, smem, c->st>>>(c->b.eigV, c->b.Rlo, c->win, r, c->b.A, c->b.ireg, c->P.lsq_rel_cutoff,
                                         c->b.y, c->b.cvec, c->b.ireg + 2, c->b.eigA, fac,
                                         kg ? c->b.K : nullptr, tg ? c->b.Tg : nullptr,
                                         c->prof ? c->b.dbg + 64 : nullptr, zg ? c->b.eigZ : nullptr);
  HROM_LAUNCH_CK();
  ++c->nlaunch;
  return HROM_OK;
}

hrom_status basis_from_gram(hrom_ctx* c, const Win& W) {
  const EigLayout L = eig_layout(W.w, W.w);
  const size_t smem = L.bytes + 2 * kMaxSlots * sizeof(double);  // + the centring row means (hi, lo)
  HROM_CK(cudaFuncSetAttribute(basis_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  double* Mh = c->b.Mdd;
  double* Ml = c->b.Mdd + (size_t)kMaxSlots * kMaxSlots;
  basis_kernel<<<1, 512, smem, c->st>>>(c->b.C, c->b.Clo, kMaxSlots, W, Mh, Ml, c->b.Zf, c->b.lam, c->b.ireg,
                                        c->b.eigA, c->b.eigZ);
  HROM_LAUNCH_CK();
  size_t rsm = (size_t)5 * W.w * (W.w | 1) * sizeof(double);
  double* gws = nullptr;
  if (rsm > 200 * 1024) {  // wide windows: workspace in the (L2-resident) global scratch
    gws = c->b.rfws;
    rsm = 0;
  }
  HROM_CK(cudaFuncSetAttribute(refine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsm));
  refine_kernel<<<1, RF_T, rsm, c->st>>>(Mh, Ml, c->b.Zf, W.w, c->r, c->P.eig_rel_cutoff, c->b.lam, c->b.A,
                                         c->b.ireg, gws);
  HROM_LAUNCH_CK();
  c->nlaunch += 2;
  return HROM_OK;
}

hrom_status lift(hrom_ctx* c, const Win& W, double* phi, double* psi) {
  if (W.w > kMaxW || c->r > kMaxR) return HROM_E_INVALID;
  const int kpad = (W.w + 3) & ~3;
  const size_t smem = ((size_t)kpad * LF_LDA + (size_t)LF_STAGES * LF_NCOL * LF_LDT) * sizeof(double);
  HROM_CK(cudaFuncSetAttribute(lift_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  lift_kernel<<<c->nsm, LF_T, smem, c->st>>>(c->g, W, c->b.ring, c->b.A, c->b.ireg, phi, psi);
  HROM_LAUNCH_CK();
  ++c->nlaunch;
  return HROM_OK;
}

}  // namespace hrom
