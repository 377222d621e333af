// internal.cuh -- shared definitions of libhrom (product path; no oracle code).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../include/hrom.h"

#define HROM_CK(x)                                                                        \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess) {                                                              \
      fprintf(stderr, "libhrom: CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, \
              __LINE__);                                                                  \
      return HROM_E_CUDA;                                                                 \
    }                                                                                     \
  } while (0)

// HROM_SYNC_DEBUG=1: synchronise after every launch so a fault names its kernel (debug only)
inline bool hrom_sync_debug() {
  static const bool on = getenv("HROM_SYNC_DEBUG") != nullptr;
  return on;
}
#define HROM_LAUNCH_CK()                 \
  do {                                   \
    if (hrom_sync_debug()) cudaDeviceSynchronize(); \
    cudaError_t e_ = cudaGetLastError(); \
    if (e_ != cudaSuccess) {             \
      fprintf(stderr, "libhrom: launch error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return HROM_E_CUDA;                \
    }                                    \
  } while (0)

namespace hrom {

// Slab layout of the snapshot ring: DOFs are grouped in tiles of TILE; tile t
// of slot s lives at ring[(t * NSR + s) * TILE ..], NSR = w + 3 (w + 2 snapshot slots and the
// Gram shift rho).  One fill tile -- every window column of TILE DOFs -- is therefore ONE
// contiguous (w+3) KB run: a single TMA bulk copy (measured 7.3 TB/s vs 4.9 TB/s for w+2
// separate 1 KB copies).  A plain vector is the same layout with NSR = 1.
constexpr int TILE = 128;
constexpr int TILE_SHIFT = 7;
struct SRef {
  double* p;   // base (ring + slot * TILE for a ring slot)
  int64_t ns;  // slots per slab tile (1 for a plain vector)
};
__host__ __device__ __forceinline__ int64_t sidx(const SRef& r, int64_t e) {
  return (((e >> TILE_SHIFT) * r.ns) << TILE_SHIFT) + (e & (TILE - 1));
}
__host__ __device__ __forceinline__ SRef plain(const double* p) { return SRef{const_cast<double*>(p), 1}; }

constexpr int kMaxW = 128;           // largest window supported (config 5)
constexpr int kMaxSlots = kMaxW + 2; // ring slots
constexpr int kMaxR = 64;
constexpr int kL1Blocks = 1024;  // relative-L1 partial sums
constexpr int kOdeimMax = 256;   // ODEIM points per call (n_p)
constexpr int kOdeimBlocks = 4 * 148;

// Geometry passed by value to kernels.
struct Geo {
  int dim, nx, ny, c, bc, recon, wpr;  // wpr = mask words per row
  int bcy;  // boundary rule of the y ends (= bc; 0 on a row slab whose y ends are halo rows, slab.cu)
  int64_t N, D, Dp;                    // Dp: D rounded up to a multiple of TILE
  int64_t nsr;                         // slab slots per tile (w + 3)
  double dx, dy, gamma, cfl;
  double rdx, rdy;  // 1/dx, 1/dy: used instead of the divisions only when dx, dy are powers of two
  int pow2;         // (then x / dx == x * rdx bit for bit)
};

// Slot descriptor of the basis: union slots (oldest first), psi_prev = mean of the first w,
// psi_cur = mean of the last w, X columns = the last w union slots.
struct Win {
  int nU, w;
  int slot[kMaxW + 1];
};

// mask indices
// M_H: seam-filter halo; M_SPREV: S-hat of the previous sampling; M_ADD / M_REM: its churn
enum { M_S = 0, M_B, M_T, M_A2, M_A1, M_TMP, M_TMP2, M_H, M_SPREV, M_ADD, M_REM, M_COUNT };
// list indices
// L_H: seam-filter halo; L_ADD / L_REM: cells entering / leaving S-hat at the last sampling
enum { L_S = 0, L_B, L_T, L_A2, L_A1, L_H, L_ADD, L_REM, L_COUNT };

struct Bufs {
  double* ring = nullptr;     // slab: (Dp / TILE) tiles x nsr slots x TILE
  double* rho = nullptr;      // = ring + nslots * TILE (slab slot nslots)
  double* U1 = nullptr;       // Dp (stage outputs / filter scratch)
  double* U2 = nullptr;
  double* U3 = nullptr;
  double* Vorig = nullptr;    // Dp
  double* eps = nullptr;      // N
  double* eps_elem = nullptr; // Dp
  uint32_t* masks = nullptr;  // M_COUNT * mwords
  int32_t* lists = nullptr;   // L_COUNT * N
  int32_t* counts = nullptr;  // 16 ints (device)
  uint8_t* kept = nullptr;    // N bytes (compact seam-filter flags)
  int32_t* fidx = nullptr;    // N: cell -> compact seam-filter index
  int32_t* ftab = nullptr;    // 14 N: seam-filter stencil tables
  double* fcur = nullptr;     // Dp: compact current values (seam filter)
  double* fF = nullptr;       // Dp: compact full-step values on the band
  double* C = nullptr;        // kMaxSlots^2 window Gram by ring slot (hi part; double-double, G11)
  double* Clo = nullptr;      // kMaxSlots^2 (lo part)
  double* Rlo = nullptr;      // (kMaxW+2)^2: lo part of the gathered Gram R (hi: eigV)
  double* Mdd = nullptr;      // 2 kMaxSlots^2: M = X^T X (hi, lo) for the eigenvector refinement
  double* Zf = nullptr;       // kMaxSlots^2: all w eigenvectors of hi(M) (refined by refine_kernel)
  double* rfws = nullptr;     // 5 kMaxSlots^2: refine_kernel workspace for wide windows
  double* Tg = nullptr;       // 2 (kMaxW+1) kMaxR: solve_kernel's T = K A (hi, lo) for wide windows
  double* part = nullptr;     // partial sums
  int64_t part_len = 0;
  double* gpart = nullptr;    // Gram-row partials (fill + band)
  int64_t gpart_len = 0;
  double* K = nullptr;        // 2 (kMaxW+2)^2 centred gathered Gram (hi, lo) when not in smem
  double* Khi = nullptr;      // kMaxSlots^2: incremental gathered Gram by ring slot (double-double)
  double* Klo = nullptr;
  double* Rd = nullptr;       // 4 (kMaxW+2)^2: Gram of the rows entering / leaving S-hat (hi, lo each)
  double* vpart = nullptr;    // per-CTA partials of the S-hat GEMVs
  double* A = nullptr;        // w x r (column j: mode j)
  double* lam = nullptr;      // w eigenvalues
  double* y = nullptr;        // r
  double* cvec = nullptr;     // w
  double* zvec = nullptr;     // w (bootstrap projection coefficients)
  double* eigV = nullptr;     // kMaxSlots^2 scratch (eigenvectors when not in smem)
  double* eigA = nullptr;     // kMaxSlots^2 scratch
  double* eigZ = nullptr;     // kMaxSlots (kMaxSlots + 1): the basis eigen-solve's eigenvectors when
                              // they do not fit shared memory (w = 128)
  int32_t* ireg = nullptr;    // small int registers: [0] reff, [1] err cell lo, ...
  double* dreg = nullptr;     // small double registers: [0] dt, ...
  unsigned long long* ureg = nullptr;  // [0] smax bits, [1] latched min bad cell, [2] fused smax, [3] step flag
  long long* dbg = nullptr;   // 64 debug timestamps (seam filter)
  // sampling scratch
  double* sel_val = nullptr;   // N
  int32_t* sel_cell = nullptr; // N
  int32_t* blk = nullptr;      // block counts/offsets for compaction (max blocks * L_COUNT * 2)
  int64_t blk_len = 0;
  int32_t* hist = nullptr;     // 3 x 2048 radix histograms
  unsigned long long* hsum = nullptr;  // 3 x 2 x 2048 exact radix bucket sums (RRE-delta)
  // filter stats per block
  double* fstat = nullptr;
  double* l1part = nullptr;   // 2 * kL1Blocks partial sums (relative L1 error)
  int32_t* fcnt = nullptr;
  const double** colptr = nullptr;  // device array of column pointers (Gram)
  int32_t* slot_tab = nullptr;      // slot_tab[i] = i mod nslots
  // ODEIM workspace (odeim.cu)
  uint8_t* ochosen = nullptr;       // N: cell already a point
  double* ocoef = nullptr;          // kMaxR + 1 LSQ coefficients
  int64_t* orows = nullptr;         // kOdeimMax chosen DOF rows (the context's points: gappy rows)
  int64_t* orows_pub = nullptr;     // kOdeimMax: workspace of the public hrom_odeim
  double* opart_v = nullptr;        // per-block argmax partials
  int64_t* opart_e = nullptr;
  unsigned int* ocnt = nullptr;     // last-block counter
  int32_t* ocells = nullptr;        // kOdeimMax point cells (Algorithm 1 with ODEIM)
  double* ophi = nullptr;           // D x r materialised basis (only when odeim_points > 0)
};

}  // namespace hrom

namespace hrom {
// Host bookkeeping of a context that one step of Algorithm 1 advances (graph replay, api.cu):
// a steady-state step changes only k and the fields that track it.
struct HostSnap {
  int64_t k, rebase_k, smax_k, kinc_newest, kinc_rebase, odeim_k, nlaunch, last_err_cell;
  bool basis_ready, sets_ready, gram_row_ready, full_since_update, last_hybrid, basis_pending, eig_todo,
      bg_pending, kinc_valid, eps_sparse;
  int n_owed, samples_since_gather, fill_grid, odeim_n, points_used;
  int64_t owed_rows[4];
  double dt_override;
  Win win, eig_win;
};
// one captured steady-state step per ring phase k mod nslots (its kernel arguments depend on k
// only through the ring slots)
struct GraphSlot {
  cudaGraphExec_t exec = nullptr;
  HostSnap pre{}, post{};
};
}  // namespace hrom

struct hrom_slab;  // slab.cu: row-slab state of a sharded problem

struct hrom_ctx {
  hrom_slab* slab = nullptr;                 // non-null: this context owns one row slab of a sharded grid
  const uint32_t* fill_mB_override = nullptr;  // fill pass: cells left out of the fused Gram row (band u halo rows)
  hrom::Geo g;
  hrom_params P;
  int w, r, nslots;
  cudaStream_t st;
  int nsm;
  int64_t mwords;
  hrom::Bufs b;
  // host bookkeeping
  int64_t k = -1;            // index of the latest snapshot
  bool basis_ready = false;  // basis for step k+1 available
  bool sets_ready = false;   // S-hat_{k+1} sets built
  bool gram_row_ready = false;
  int64_t rebase_k = -1000000;
  // Algorithm 1 with finite z: the last step was a full step (the update after it sets the
  // projection indicator, G8); window-Gram rows owed by skipped updates
  bool full_since_update = false;
  int64_t owed_rows[4] = {0, 0, 0, 0};
  int n_owed = 0;
  hrom::Win win{};           // window of the current basis
  int fill_blocks = 0;       // max grid of the fill kernel (Gram-row partial slots)
  int fill_grid = 0;         // grid of the last fill launch
  int band_blocks = 0;
  int filter_blocks = 0;
  int sets_blocks = 0;       // cooperative sets kernel grid (one block per SM)
  int64_t last_err_cell = -1;
  int64_t smax_k = -1;       // state index whose max wave speed is in ureg[2] (positivity pass)
  bool last_hybrid = false;  // the latest step was a hybrid step (its positivity flag is ureg[3])
  int64_t nlaunch = 0;       // kernels launched by this context (host-side count)
  // optional per-section CUDA-event timing (hrom_profile)
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, std::pair<int, int>>> ev_pairs;  // (section, (start ev, stop ev))
  int ev_next = 0;
  int ev_open[16] = {0};
  // the one-CTA eigen-solve of the basis update runs on a side stream, overlapping the
  // sampling and the next step's dt / masked RK3 / gathered Gram (which do not need it)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_basis_in = nullptr, ev_basis_done = nullptr;
  int odeim_n = 0;            // ODEIM points of the current basis (0: none / not computed)
  int points_used = 0;        // ODEIM points used by the latest step (p-bar)
  int64_t odeim_k = -1;       // k of the basis they belong to
  bool basis_pending = false;  // eigen-solve launched on the side stream, not yet joined
  bool eig_todo = false;       // eigen-solve deferred (launched after the sampling kernel)
  cudaEvent_t ev_bg_in = nullptr, ev_bg_done = nullptr;
  bool bg_pending = false;     // band Gram partials computed on the side stream, not yet joined
  // incremental gathered Gram (G7): valid for the S-hat of the last sampling, shift rebase_k and
  // the union whose newest snapshot is kinc_newest
  bool kinc_valid = false;
  int samples_since_gather = 99;  // samplings since the last gathered Gram (churn lists valid iff 1)
  bool eps_sparse = false;   // the indicator is nonzero only on the T list (set by a hybrid step)
  bool gather_inc = false;          // the gathered Gram in flight took the incremental route (G7)
  bool gather_skip_finish = false;  // ... or the ODEIM rows (no per-slot state)
  int64_t kinc_newest = -1, kinc_rebase = -1;
  hrom::Win eig_win{};
  // CUDA-graph replay of steady-state steps (hrom_set_graph)
  bool graph_on = false;
  std::vector<hrom::GraphSlot> graphs;
  int64_t graph_launches = 0, graph_captures = 0;
  cudaStream_t gst = nullptr;               // capture / replay stream of the graphs
  cudaEvent_t ev_g0 = nullptr, ev_g1 = nullptr;
  int slot_of(int64_t kk) const { return (int)(kk % nslots); }
  hrom::SRef slot_ref(int s) const { return hrom::SRef{b.ring + (int64_t)s * hrom::TILE, g.nsr}; }
  hrom::SRef rho_ref() const { return hrom::SRef{b.rho, g.nsr}; }
};

namespace hrom {
hrom_status flush_eigen(hrom_ctx* c);  // api.cu: launch a deferred eigen-solve on the side stream
inline void basis_join(hrom_ctx* c) {
  if (c->bg_pending) {
    cudaStreamWaitEvent(c->st, c->ev_bg_done, 0);
    c->bg_pending = false;
  }
  if (c->eig_todo) flush_eigen(c);
  if (c->basis_pending) {
    cudaStreamWaitEvent(c->st, c->ev_basis_done, 0);
    c->basis_pending = false;
  }
}
}  // namespace hrom

namespace hrom {
enum Section { SEC_DT = 0, SEC_MASKED, SEC_GATHER, SEC_SOLVE, SEC_FILL, SEC_EPS, SEC_FILTER, SEC_BANDGRAM,
               SEC_POS, SEC_BASIS, SEC_SAMPLE, SEC_FULL, SEC_REBASE, SEC_EIGEN, SEC_COUNT };
inline void prof_begin(hrom_ctx* c, int sec) {
  if (!c->prof || c->ev_next + 2 > (int)c->ev_pool.size()) return;
  c->ev_open[sec] = c->ev_next;
  cudaEventRecord(c->ev_pool[c->ev_next++], c->st);
}
inline void prof_end(hrom_ctx* c, int sec) {
  if (!c->prof || c->ev_next + 1 > (int)c->ev_pool.size()) return;
  cudaEventRecord(c->ev_pool[c->ev_next], c->st);
  c->ev_pairs.push_back({sec, {c->ev_open[sec], c->ev_next}});
  ++c->ev_next;
}
}  // namespace hrom

namespace hrom {
__host__ __device__ __forceinline__ double div_dx(const Geo& g, double x) { return g.pow2 ? x * g.rdx : x / g.dx; }
__host__ __device__ __forceinline__ double div_dy(const Geo& g, double x) { return g.pow2 ? x * g.rdy : x / g.dy; }
// euler.cu
hrom_status launch_dt(hrom_ctx* c, SRef q, double dt_override, int64_t kq);
hrom_status launch_stage(hrom_ctx* c, int stage, SRef qn, SRef qin, SRef out, const int32_t* list, int list_idx,
                         double dt_override, const unsigned long long* run_if = nullptr, bool fuse_smax = false);
hrom_status launch_positivity(hrom_ctx* c, SRef qprev, SRef q, int64_t kq);
// flag ureg[3] and maximum ureg[2] over the cells [n0, n1) (n1 < 0: all)
hrom_status launch_positivity_check(hrom_ctx* c, SRef q, int64_t n0, int64_t n1);
hrom_status launch_positivity_redo(hrom_ctx* c, SRef qprev, SRef q, int64_t kq);  // conditional full-step redo
// max wave speed bits of the cells [n0, n1) (atomicMax into *dev_out)
hrom_status launch_smax(hrom_ctx* c, SRef q, unsigned long long* dev_out, int64_t n0, int64_t n1);
// masks.cu
hrom_status build_sets(hrom_ctx* c, const uint32_t* dev_mask_S);
hrom_status build_sets_with_churn(hrom_ctx* c);  // S-hat in place, its predecessor in M_SPREV
hrom_status select_and_build(hrom_ctx* c, const double* eps, int64_t n_g, double rre_delta = 0.0);
hrom_status odeim_for_basis(hrom_ctx* c);
hrom_status project_window(hrom_ctx* c, const double* const* phicols, int m, double* dev_C);           // ODEIM points of the current basis (odeim.cu)
hrom_status or_cells_into_mask(hrom_ctx* c, uint32_t* mask, const int32_t* cells, int n);
int sets_occupancy();
// linalg.cu
// dev_cols: column base pointers, all with slab stride ns (1 = plain vectors); rho: SRef or p == nullptr
hrom_status gram_full(hrom_ctx* c, const double* const* dev_cols, int64_t ns, int ncol, int64_t rows, SRef rho,
                      double* dev_C, int ldc, const int32_t* map);
hrom_status gram_full_dd(hrom_ctx* c, const double* const* dev_cols, int64_t ns, int ncol, int64_t rows, SRef rho,
                         double* dev_Chi, double* dev_Clo, int ldc, const int32_t* map);
hrom_status gram_gathered(hrom_ctx* c, SRef src_b);
// the two halves of gram_gathered with explicit cell lists (row slabs: own-row sub-lists)
struct GatherLists {
  const int32_t *S, *nS, *add, *nadd, *rem, *nrem;
};
hrom_status gram_gathered_partial(hrom_ctx* c, SRef src_b, const GatherLists* L);
hrom_status gram_gathered_finish(hrom_ctx* c);
double* gathered_gemv_values(hrom_ctx* c);
hrom_status band_gram_rows(hrom_ctx* c, const Win& W, SRef v);
// the same kernels on an explicit cell list (row slabs: the own rows of a set)
hrom_status band_gram_rows_list(hrom_ctx* c, const Win& W, SRef v, const int32_t* list, const int32_t* count);
hrom_status gram_gathered_list(hrom_ctx* c, const Win& W, SRef src_b, const int32_t* list, const int32_t* count,
                               double* Rhi, double* Rlo);
hrom_status small_solve(hrom_ctx* c);
hrom_status basis_from_gram(hrom_ctx* c, const Win& W);
hrom_status lift(hrom_ctx* c, const Win& W, double* phi, double* psi);
// fill.cu
hrom_status launch_fill(hrom_ctx* c, const Win& W, int mode, SRef src_S, SRef out, bool out_in_ring,
                        const unsigned long long* run_if = nullptr);
hrom_status launch_gram_row(hrom_ctx* c, const Win& W, int new_slot, const unsigned long long* run_if = nullptr);
hrom_status reduce_gram_row(hrom_ctx* c, const Win& W, int new_slot, bool with_band,
                            const unsigned long long* esc = nullptr);
hrom_status launch_eps_cells(hrom_ctx* c);
// api.cu
Win window_of(const hrom_ctx* c, int64_t k);           // slots of the window whose newest snapshot is gamma_k
hrom_status launch_zvec(hrom_ctx* c, int w, double am);  // projection-indicator coefficients (A19, G8)
hrom_status launch_eps_all(hrom_ctx* c);
// slab.cu
void slab_destroy(hrom_ctx* c);
// filter.cu
hrom_status launch_filter(hrom_ctx* c, SRef v, SRef F, uint8_t* kept_cells);
}  // namespace hrom
