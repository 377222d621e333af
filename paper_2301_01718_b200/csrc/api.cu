// api.cu -- the C ABI of libhrom (include/hrom.h): context, schedule and orchestration.
//
// One hybrid step (Algorithm 1, explicit variant, z = infinity):
//   H1 dt -> H3 masked RK3 on A1 / A2 / T = S-hat u B -> H4 gathered Gram [X_S, b] (DMMA)
//   -> H5 one-CTA pinv solve (y, c = A y) -> H6+H9+H10 fused fill / indicator / Gram-row pass
//   -> H7 seam filter (cooperative) -> band Gram rows
// then hrom_update_basis (H10 reduce / re-base, H11 eigen) and hrom_sample (H8).
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include "internal.cuh"

namespace hrom {
hrom_status launch_eps_all(hrom_ctx* c);
int filter_occupancy();
int fill_max_gram_slots();

namespace {

__global__ void zvec_kernel(const double* __restrict__ A, const double* __restrict__ lam,
                            const int32_t* __restrict__ reffp, int w, double am, double* __restrict__ z) {
  // projection indicator (A19 at k = w-1; G8 after a full step k >= w): gamma_k - psi_{k+1} =
  // X alpha with alpha = e_{w-1} - am 1 (am = 0 at the bootstrap, where psi_{w-1} = psi_w;
  // am = 1/w for the lagged centring, k >= w), and Phi Phi^T X alpha = X V_r V_r^T alpha, so
  // the residual is X z with z = alpha - V_r V_r^T alpha, V_r[:, j] = A[:, j] sqrt(lam_j)
  const int re = *reffp;
  __shared__ double t[kMaxR];
  for (int j = threadIdx.x; j < re; j += blockDim.x) {  // t_j = sqrt(lam_j) A[:, j]^T alpha
    const double sl = sqrt(lam[j]);
    double sum = 0.0;
    for (int i = 0; i < w; ++i) sum += A[j * w + i];
    t[j] = A[j * w + (w - 1)] * sl - am * (sum * sl);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < w; i += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < re; ++j) s += (A[j * w + i] * sqrt(lam[j])) * t[j];
    z[i] = ((i == w - 1 ? 1.0 : 0.0) - am) - s;
  }
}

__global__ void set_i32_kernel(int32_t* p, int32_t v) { *p = v; }

// relative L1 error: per-block partial sums over a fixed grid-stride assignment,
// then one block sums the partials in a fixed tree order (bitwise reproducible)
__global__ void __launch_bounds__(256) l1_partial_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                                         int64_t n, double* __restrict__ part) {
  __shared__ double s0[8], s1[8];
  double num = 0.0, den = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double bv = b[i];
    num += fabs(a[i] - bv);
    den += fabs(bv);
  }
  for (int o = 16; o > 0; o >>= 1) {
    num += __shfl_xor_sync(0xffffffffu, num, o);
    den += __shfl_xor_sync(0xffffffffu, den, o);
  }
  if ((threadIdx.x & 31) == 0) {
    s0[threadIdx.x >> 5] = num;
    s1[threadIdx.x >> 5] = den;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0.0, y = 0.0;
    for (int k = 0; k < 8; ++k) {
      x += s0[k];
      y += s1[k];
    }
    part[blockIdx.x] = x;
    part[gridDim.x + blockIdx.x] = y;
  }
}

__global__ void __launch_bounds__(1024) l1_final_kernel(const double* __restrict__ part, int nb, double* __restrict__ out) {
  __shared__ double s0[32], s1[32];
  double x = 0.0, y = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    x += part[i];
    y += part[nb + i];
  }
  for (int o = 16; o > 0; o >>= 1) {
    x += __shfl_xor_sync(0xffffffffu, x, o);
    y += __shfl_xor_sync(0xffffffffu, y, o);
  }
  if ((threadIdx.x & 31) == 0) {
    s0[threadIdx.x >> 5] = x;
    s1[threadIdx.x >> 5] = y;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int k = 0; k < 32; ++k) {
      a += s0[k];
      b += s1[k];
    }
    out[0] = a;
    out[1] = b;
  }
}

// every workspace starts zeroed: a context's results never depend on what an earlier allocation
// left in the memory (two runs are bitwise identical whatever ran before them)
template <typename T>
hrom_status dalloc(T** p, size_t n) {
  const size_t bytes = std::max<size_t>(n, 1) * sizeof(T);
  if (cudaMalloc((void**)p, bytes) != cudaSuccess) return HROM_E_NOMEM;
  if (cudaMemset(*p, 0, bytes) != cudaSuccess) return HROM_E_CUDA;
  return HROM_OK;
}

Win window_at(const hrom_ctx* c, int64_t k) {
  Win W{};
  W.w = c->w;
  if (k == c->w - 1) {
    W.nU = c->w;
    for (int i = 0; i < c->w; ++i) W.slot[i] = c->slot_of(i);
  } else {
    W.nU = c->w + 1;
    for (int i = 0; i <= c->w; ++i) W.slot[i] = c->slot_of(k - c->w + i);
  }
  return W;
}

}  // namespace
}  // namespace hrom

using namespace hrom;

namespace hrom {
Win window_of(const hrom_ctx* c, int64_t k) { return window_at(c, k); }
hrom_status launch_zvec(hrom_ctx* c, int w, double am) {
  zvec_kernel<<<1, 128, 0, c->st>>>(c->b.A, c->b.lam, c->b.ireg, w, am, c->b.zvec);
  HROM_LAUNCH_CK();
  ++c->nlaunch;
  return HROM_OK;
}
hrom_status flush_eigen(hrom_ctx* c) {
  if (!c->eig_todo) return HROM_OK;
  c->eig_todo = false;
  HROM_CK(cudaEventRecord(c->ev_basis_in, c->st));
  HROM_CK(cudaStreamWaitEvent(c->side, c->ev_basis_in, 0));
  cudaStream_t main_st = c->st;
  c->st = c->side;
  prof_begin(c, SEC_EIGEN);
  const hrom_status s = basis_from_gram(c, c->eig_win);
  prof_end(c, SEC_EIGEN);
  c->st = main_st;
  if (s != HROM_OK) return s;
  HROM_CK(cudaEventRecord(c->ev_basis_done, c->side));
  c->basis_pending = true;
  return HROM_OK;
}

}  // namespace hrom

extern "C" {

const char* hrom_status_string(hrom_status s) {
  switch (s) {
    case HROM_OK: return "ok";
    case HROM_E_INVALID: return "invalid argument";
    case HROM_E_STATE: return "call out of order";
    case HROM_E_POSITIVITY: return "non-positive density or pressure";
    case HROM_E_RANK: return "zero least-squares matrix";
    case HROM_E_CUDA: return "CUDA error";
    case HROM_E_NOMEM: return "out of device memory";
  }
  return "unknown";
}

hrom_status hrom_create(const hrom_grid* grid, double gamma, double cfl, const hrom_params* p, void* stream,
                        hrom_ctx** out) {
  if (!grid || !p || !out) return HROM_E_INVALID;
  *out = nullptr;
  const int dim = grid->dim;
  if (dim != 1 && dim != 2) return HROM_E_INVALID;
  const int ny = dim == 1 ? 1 : grid->ny;
  if (grid->nx < 1 || ny < 1 || (grid->bc != 0 && grid->bc != 1) || (grid->recon != 1 && grid->recon != 2))
    return HROM_E_INVALID;
  if ((int64_t)grid->nx * ny * (dim + 2) >= (int64_t)INT32_MAX * 2) return HROM_E_INVALID;
  if (!(gamma > 1.0) || !(cfl > 0.0)) return HROM_E_INVALID;
  if (p->window < 2 || p->window > kMaxW || p->rank < 1 || p->rank > p->window || p->rank > kMaxR)
    return HROM_E_INVALID;
  if (p->halo < grid->recon || p->halo > 16 || p->band < -1 || p->band > 16) return HROM_E_INVALID;
  if (p->n_filter_orders < 0 || p->n_filter_orders > 3 || p->filter_max_sweeps < 0 ||
      p->n_filter_orders * p->filter_max_sweeps > 64)
    return HROM_E_INVALID;
  for (int i = 0; i < p->n_filter_orders; ++i)
    if (p->filter_orders[i] != 2 && p->filter_orders[i] != 4 && p->filter_orders[i] != 6) return HROM_E_INVALID;
  if (!(p->sample_fraction > 0.0 && p->sample_fraction <= 1.0)) return HROM_E_INVALID;
  if (p->sample_mode != 0 && p->sample_mode != 1) return HROM_E_INVALID;
  if (p->odeim_points < 0 || p->odeim_points > kOdeimMax ||
      (int64_t)p->odeim_points > (int64_t)grid->nx * (grid->dim == 2 ? grid->ny : 1))
    return HROM_E_INVALID;
  if (p->sample_mode == 1 && !(p->rre_delta > 0.0 && p->rre_delta <= 1.0)) return HROM_E_INVALID;
  if (p->gram_mode != 0 && p->gram_mode != 1) return HROM_E_INVALID;
  if (p->gather_mode != 0 && p->gather_mode != 1) return HROM_E_INVALID;

  hrom_ctx* c = new hrom_ctx();
  c->P = *p;
  // the window Gram is double-double (G11): the shift's cancellation in the centring algebra
  // costs nothing at fp64 output precision, so by default the shift is never re-based
  if (c->P.rebase_period <= 0) c->P.rebase_period = INT32_MAX;
  c->w = p->window;
  c->r = p->rank;
  c->nslots = c->w + 2;
  c->st = (cudaStream_t)stream;
  Geo& g = c->g;
  g.dim = dim;
  g.nx = grid->nx;
  g.ny = ny;
  g.c = dim + 2;
  g.bc = grid->bc;
  g.bcy = grid->bc;
  g.recon = grid->recon;
  g.wpr = (grid->nx + 31) / 32;
  g.N = (int64_t)g.nx * g.ny;
  g.D = g.c * g.N;
  g.Dp = (g.D + TILE - 1) / TILE * TILE;
  g.nsr = c->nslots + 1;  // slab: w+2 snapshot slots + rho
  g.dx = (grid->x1 - grid->x0) / grid->nx;
  g.dy = dim == 2 ? (grid->y1 - grid->y0) / ny : 1.0;
  g.gamma = gamma;
  g.cfl = cfl;
  {
    int ex = 0, ey = 0;
    const bool px = std::frexp(g.dx, &ex) == 0.5, py = std::frexp(g.dy, &ey) == 0.5;
    g.pow2 = (px && py) ? 1 : 0;
    g.rdx = 1.0 / g.dx;
    g.rdy = 1.0 / g.dy;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, dev);
  c->mwords = std::max<int64_t>((int64_t)g.ny * g.wpr, (g.N + 31) / 32);
  c->fill_blocks = 8 * c->nsm;  // upper bound of the fill grid (fill.cu sizes it by occupancy)
  // the fused Gram row keeps one accumulator per window slot per lane: wider windows
  // (w + 1 > 68) take the full DMMA Gram every step instead
  if (c->w + 1 > fill_max_gram_slots()) c->P.gram_mode = 1;
  c->band_blocks = 4 * c->nsm;
  if (filter_occupancy() < 1) {  // the cooperative seam filter needs one resident block per SM
    delete c;
    return HROM_E_CUDA;
  }
  c->filter_blocks = c->nsm;  // one block per SM: cheapest grid barrier
  if (sets_occupancy() < 1) {
    delete c;
    return HROM_E_CUDA;
  }
  c->sets_blocks = c->nsm;

  Bufs& b = c->b;
  hrom_status s = HROM_OK;
  auto A = [&](hrom_status r) { if (r != HROM_OK) s = r; };
  A(dalloc(&b.ring, (size_t)g.nsr * g.Dp));
  if (b.ring) b.rho = b.ring + (int64_t)c->nslots * TILE;  // slab slot nslots
  A(dalloc(&b.U1, g.Dp));
  A(dalloc(&b.U2, g.Dp));
  A(dalloc(&b.U3, g.Dp));
  A(dalloc(&b.Vorig, g.Dp));
  A(dalloc(&b.eps, g.N));
  A(dalloc(&b.eps_elem, g.Dp));
  A(dalloc(&b.masks, (size_t)M_COUNT * c->mwords));
  A(dalloc(&b.lists, (size_t)L_COUNT * g.N));
  A(dalloc(&b.counts, 16));
  A(dalloc(&b.kept, g.N));
  A(dalloc(&b.fidx, g.N));
  A(dalloc(&b.ftab, (size_t)14 * g.N));
  A(dalloc(&b.fcur, g.Dp));
  A(dalloc(&b.fF, g.Dp));
  A(dalloc(&b.C, (size_t)kMaxSlots * kMaxSlots));
  A(dalloc(&b.Clo, (size_t)kMaxSlots * kMaxSlots));
  A(dalloc(&b.Rlo, (size_t)(kMaxW + 2) * (kMaxW + 2)));
  A(dalloc(&b.Mdd, (size_t)2 * kMaxSlots * kMaxSlots));
  A(dalloc(&b.Zf, (size_t)kMaxSlots * kMaxSlots));
  A(dalloc(&b.rfws, (size_t)5 * kMaxSlots * kMaxSlots));
  A(dalloc(&b.Tg, (size_t)2 * (kMaxW + 1) * kMaxR));
  b.part_len = (int64_t)2 * c->nsm * 144 * 144;
  A(dalloc(&b.part, b.part_len));
  b.gpart_len = (int64_t)(c->fill_blocks + c->band_blocks) * (kMaxSlots + 1) * 2;  // double-double
  A(dalloc(&b.gpart, b.gpart_len));
  A(dalloc(&b.K, (size_t)2 * (kMaxW + 2) * (kMaxW + 2)));
  A(dalloc(&b.Khi, (size_t)kMaxSlots * kMaxSlots));
  A(dalloc(&b.Klo, (size_t)kMaxSlots * kMaxSlots));
  A(dalloc(&b.Rd, (size_t)4 * (kMaxW + 2) * (kMaxW + 2)));
  A(dalloc(&b.vpart, (size_t)2 * 8 * c->nsm * (2 * kMaxSlots + 2)));
  A(dalloc(&b.A, (size_t)kMaxW * kMaxR));
  A(dalloc(&b.lam, kMaxSlots));
  A(dalloc(&b.y, kMaxR));
  A(dalloc(&b.cvec, kMaxW));
  A(dalloc(&b.zvec, kMaxW));
  A(dalloc(&b.eigV, (size_t)kMaxSlots * kMaxSlots));
  A(dalloc(&b.eigA, (size_t)5 * kMaxSlots * (kMaxSlots + 1)));  // eigen-solve LU workspace when not in smem
  A(dalloc(&b.eigZ, (size_t)kMaxSlots * (kMaxSlots + 1)));      // eigenvectors when not in smem (w = 128)
  A(dalloc(&b.ireg, 16));
  A(dalloc(&b.dreg, 16));
  A(dalloc(&b.ureg, 4));
  A(dalloc(&b.dbg, 128));
  A(dalloc(&b.sel_val, g.N));
  A(dalloc(&b.sel_cell, g.N));
  b.blk_len = std::max<int64_t>(8 * ((c->mwords + 255) / 256 + 2) + (g.N + 1023) / 1024 + 16, 16 * (int64_t)c->nsm + 64);
  A(dalloc(&b.blk, b.blk_len));
  A(dalloc(&b.hist, 3 * 2048));
  A(dalloc(&b.hsum, 3 * 2 * 2048));
  A(dalloc(&b.fstat, std::max(c->filter_blocks, 128)));  // also the filter's per-sweep slots
  A(dalloc(&b.l1part, 2 * kL1Blocks));
  A(dalloc(&b.fcnt, c->filter_blocks));
  A(dalloc(&b.colptr, 2 * kMaxSlots));
  A(dalloc(&b.slot_tab, 2 * kMaxSlots));
  A(dalloc(&b.ochosen, g.N));
  A(dalloc(&b.ocoef, kMaxR + 1));
  A(dalloc(&b.orows, kOdeimMax));
  A(dalloc(&b.orows_pub, kOdeimMax));
  A(dalloc(&b.opart_v, kOdeimBlocks));
  A(dalloc(&b.opart_e, kOdeimBlocks));
  A(dalloc(&b.ocnt, 1));
  A(dalloc(&b.ocells, kOdeimMax));
  if (c->P.odeim_points > 0) A(dalloc(&b.ophi, (size_t)c->r * g.D));
  if (s == HROM_OK && cudaMemset(b.ocnt, 0, sizeof(unsigned int)) != cudaSuccess) s = HROM_E_CUDA;
  if (s != HROM_OK) {
    hrom_destroy(c);
    return s;
  }
  // pointer table: colptr[i] = slot (i mod nslots), so any run of consecutive slots is contiguous
  std::vector<const double*> tab(2 * kMaxSlots);
  for (int i = 0; i < 2 * kMaxSlots; ++i) tab[i] = b.ring + (int64_t)(i % c->nslots) * TILE;
  std::vector<int32_t> stab(2 * kMaxSlots);
  for (int i = 0; i < 2 * kMaxSlots; ++i) stab[i] = i % c->nslots;
  if (cudaMemcpy(b.colptr, tab.data(), tab.size() * sizeof(double*), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(b.slot_tab, stab.data(), stab.size() * sizeof(int32_t), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemset(b.C, 0, sizeof(double) * kMaxSlots * kMaxSlots) != cudaSuccess ||
      cudaMemset(b.Clo, 0, sizeof(double) * kMaxSlots * kMaxSlots) != cudaSuccess ||
      cudaMemset(b.ureg, 0xff, 4 * sizeof(unsigned long long)) != cudaSuccess ||
      cudaMemset(b.ireg, 0, 16 * sizeof(int32_t)) != cudaSuccess ||
      cudaMemset(b.eps, 0, g.N * sizeof(double)) != cudaSuccess ||
      cudaMemset(b.masks, 0, (size_t)M_COUNT * c->mwords * sizeof(uint32_t)) != cudaSuccess ||
      cudaMemset(b.counts, 0, 16 * sizeof(int32_t)) != cudaSuccess ||
      cudaMemset(b.ring, 0, (size_t)g.nsr * g.Dp * sizeof(double)) != cudaSuccess) {
    hrom_destroy(c);
    return HROM_E_CUDA;
  }
  if (cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_basis_in, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_basis_done, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_bg_in, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_bg_done, cudaEventDisableTiming) != cudaSuccess) {
    hrom_destroy(c);
    return HROM_E_CUDA;
  }
  *out = c;
  return HROM_OK;
}

void hrom_destroy(hrom_ctx* c) {
  if (!c) return;
  if (c->side) cudaStreamSynchronize(c->side);
  if (c->st) cudaStreamSynchronize(c->st);
  else cudaDeviceSynchronize();
  if (c->side) cudaStreamDestroy(c->side);
  if (c->ev_basis_in) cudaEventDestroy(c->ev_basis_in);
  if (c->ev_basis_done) cudaEventDestroy(c->ev_basis_done);
  if (c->ev_bg_in) cudaEventDestroy(c->ev_bg_in);
  if (c->ev_bg_done) cudaEventDestroy(c->ev_bg_done);
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  for (auto& gs : c->graphs)
    if (gs.exec) cudaGraphExecDestroy(gs.exec);
  if (c->gst) {
    cudaStreamSynchronize(c->gst);
    cudaStreamDestroy(c->gst);
  }
  if (c->ev_g0) cudaEventDestroy(c->ev_g0);
  if (c->ev_g1) cudaEventDestroy(c->ev_g1);
  Bufs& b = c->b;
  void* ptrs[] = {b.ring, b.U1, b.U2, b.U3, b.Vorig, b.eps, b.eps_elem, b.masks, b.lists, b.counts,
                  b.kept, b.fidx, b.ftab, b.fcur, b.fF, b.C, b.Clo, b.Rlo, b.Mdd, b.Zf, b.rfws, b.Tg, b.part, b.gpart, b.K, b.Khi, b.Klo, b.Rd, b.vpart, b.A, b.lam, b.y, b.cvec, b.zvec, b.eigV, b.eigA, b.eigZ, b.ireg,
                  b.dreg, b.ureg, b.dbg, b.sel_val, b.sel_cell, b.blk, b.hist, b.hsum, b.fstat, b.l1part, b.fcnt, (void*)b.colptr, b.slot_tab, b.ochosen, b.ocoef, b.orows, b.orows_pub, b.opart_v, b.opart_e, b.ocnt, b.ocells, b.ophi};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  slab_destroy(c);
  delete c;
}

// plain vector <-> slab ring slot (2-D copy: TILE-element rows, pitches TILE and nsr*TILE)
static hrom_status copy_slot(hrom_ctx* c, int slot, const double* src_plain, double* dst_plain) {
  const int64_t D = c->g.D, full = D / TILE, tail = D - full * TILE;
  const size_t row = TILE * sizeof(double), spitch = (size_t)c->g.nsr * TILE * sizeof(double);
  double* base = c->b.ring + (int64_t)slot * TILE;
  if (src_plain) {
    c->smax_k = -1;  // the state changed under the fused wave-speed maximum
    if (full) HROM_CK(cudaMemcpy2DAsync(base, spitch, src_plain, row, row, full, cudaMemcpyDefault, c->st));
    if (tail)
      HROM_CK(cudaMemcpyAsync(base + full * c->g.nsr * TILE, src_plain + full * TILE, tail * sizeof(double),
                              cudaMemcpyDefault, c->st));
  } else {
    if (full) HROM_CK(cudaMemcpy2DAsync(dst_plain, row, base, spitch, row, full, cudaMemcpyDefault, c->st));
    if (tail)
      HROM_CK(cudaMemcpyAsync(dst_plain + full * TILE, base + full * c->g.nsr * TILE, tail * sizeof(double),
                              cudaMemcpyDefault, c->st));
  }
  return HROM_OK;
}

hrom_status hrom_set_state(hrom_ctx* c, const double* any_q) {
  if (!c || !any_q) return HROM_E_INVALID;
  hrom_status s0 = copy_slot(c, 0, any_q, nullptr);
  if (s0 != HROM_OK) return s0;
  HROM_CK(cudaMemsetAsync(c->b.ureg + 1, 0xff, sizeof(unsigned long long), c->st));
  c->k = 0;
  c->last_hybrid = false;
  c->full_since_update = false;
  c->n_owed = 0;
  c->kinc_valid = false;
  c->eps_sparse = false;
  c->basis_ready = c->sets_ready = c->gram_row_ready = false;
  c->rebase_k = -1000000;
  c->last_err_cell = -1;
  return HROM_OK;
}

hrom_status hrom_get_state(hrom_ctx* c, double* any_q) {
  if (!c || !any_q) return HROM_E_INVALID;
  if (c->k < 0) return HROM_E_STATE;
  return copy_slot(c, c->slot_of(c->k), nullptr, any_q);
}

hrom_status hrom_full_step(hrom_ctx* c, double dt_override, double* dev_dt_out) {
  if (!c) return HROM_E_INVALID;
  if (c->k < 0) return HROM_E_STATE;
  const int64_t kn = c->k + 1;
  const SRef qn = c->slot_ref(c->slot_of(c->k));
  const SRef out = c->slot_ref(c->slot_of(kn));
  const SRef U1 = plain(c->b.U1), U2 = plain(c->b.U2);
  hrom_status s;
  prof_begin(c, SEC_FULL);
  if ((s = launch_dt(c, qn, dt_override, c->k)) != HROM_OK) return s;
  if (dev_dt_out) HROM_CK(cudaMemcpyAsync(dev_dt_out, c->b.dreg, sizeof(double), cudaMemcpyDefault, c->st));
  if ((s = launch_stage(c, 1, qn, qn, U1, nullptr, 0, dt_override)) != HROM_OK) return s;
  if ((s = launch_stage(c, 2, qn, U1, U2, nullptr, 0, dt_override)) != HROM_OK) return s;
  // 2-D: the last stage also takes the new state's wave-speed maximum (the next step's H1)
  const bool fuse = c->g.dim == 2 && !c->slab && dt_override <= 0.0;
  if ((s = launch_stage(c, 3, qn, U2, out, nullptr, 0, dt_override, nullptr, fuse)) != HROM_OK) return s;
  prof_end(c, SEC_FULL);
  if (fuse) c->smax_k = kn;
  c->k = kn;
  c->points_used = 0;
  c->last_hybrid = false;
  c->full_since_update = true;
  c->gram_row_ready = false;
  c->sets_ready = false;
  return HROM_OK;
}

hrom_status hrom_hybrid_step(hrom_ctx* c, const uint32_t* dev_mask, double dt_override, double* dev_dt_out) {
  if (!c) return HROM_E_INVALID;
  if (!c->basis_ready) return HROM_E_STATE;
  hrom_status s;
  if ((s = flush_eigen(c)) != HROM_OK) return s;
  if (dev_mask) {
    if ((s = build_sets(c, dev_mask)) != HROM_OK) return s;
    c->sets_ready = true;
  }
  if (!c->sets_ready) return HROM_E_STATE;
  const Geo& g = c->g;
  Bufs& b = c->b;
  const int64_t kn = c->k + 1;
  const SRef qn = c->slot_ref(c->slot_of(c->k));
  const SRef out = c->slot_ref(c->slot_of(kn));
  const SRef U1 = plain(b.U1), U2 = plain(b.U2), U3 = plain(b.U3);
  // H1
  prof_begin(c, SEC_DT);
  if ((s = launch_dt(c, qn, dt_override, c->k)) != HROM_OK) return s;
  prof_end(c, SEC_DT);
  if (dev_dt_out) HROM_CK(cudaMemcpyAsync(dev_dt_out, b.dreg, sizeof(double), cudaMemcpyDefault, c->st));
  // H3: stage 1 on A1, stage 2 on A2, stage 3 on T = S-hat u B (F on the band)
  const int32_t* L = b.lists;
  prof_begin(c, SEC_MASKED);
  if ((s = launch_stage(c, 1, qn, qn, U1, L + (int64_t)L_A1 * g.N, L_A1, dt_override)) != HROM_OK) return s;
  if ((s = launch_stage(c, 2, qn, U1, U2, L + (int64_t)L_A2 * g.N, L_A2, dt_override)) != HROM_OK) return s;
  if ((s = launch_stage(c, 3, qn, U2, U3, L + (int64_t)L_T * g.N, L_T, dt_override)) != HROM_OK) return s;
  prof_end(c, SEC_MASKED);
  // H4 + H5
  prof_begin(c, SEC_GATHER);
  if ((s = gram_gathered(c, U3)) != HROM_OK) return s;
  prof_end(c, SEC_GATHER);
  basis_join(c);  // the eigen-solve of the previous update ran on the side stream
  prof_begin(c, SEC_SOLVE);
  if ((s = small_solve(c)) != HROM_OK) return s;
  prof_end(c, SEC_SOLVE);
  // H6 (+H9, H10 row)
  HROM_CK(cudaMemsetAsync(b.eps, 0, g.N * sizeof(double), c->st));
  prof_begin(c, SEC_FILL);
  if ((s = launch_fill(c, c->win, 0, U3, out, true)) != HROM_OK) return s;
  prof_end(c, SEC_FILL);
  prof_begin(c, SEC_EPS);
  if ((s = launch_eps_cells(c)) != HROM_OK) return s;
  prof_end(c, SEC_EPS);
  // H7
  prof_begin(c, SEC_FILTER);
  if (c->P.n_filter_orders > 0 && c->P.filter_max_sweeps > 0)
    if ((s = launch_filter(c, out, U3, nullptr)) != HROM_OK) return s;
  prof_end(c, SEC_FILTER);
  if (c->P.gram_mode == 0) {
    // H10 band part on the side stream, concurrently with the positivity pass (both only read
    // gamma_k; an escalated step discards the band partials); joined in basis_join()
    HROM_CK(cudaEventRecord(c->ev_bg_in, c->st));
    HROM_CK(cudaStreamWaitEvent(c->side, c->ev_bg_in, 0));
    cudaStream_t main_st = c->st;
    c->st = c->side;
    prof_begin(c, SEC_BANDGRAM);
    s = band_gram_rows(c, c->win, out);
    prof_end(c, SEC_BANDGRAM);
    c->st = main_st;
    if (s != HROM_OK) return s;
    HROM_CK(cudaEventRecord(c->ev_bg_done, c->side));
    c->bg_pending = true;
  }
  prof_begin(c, SEC_POS);
  if ((s = launch_positivity(c, qn, out, kn)) != HROM_OK) return s;
  prof_end(c, SEC_POS);
  c->k = kn;
  c->points_used = (c->P.odeim_points > 0 && c->odeim_k == c->k - 1) ? c->odeim_n : 0;
  c->last_hybrid = true;
  c->eps_sparse = true;  // eps: memset, then written on S-hat (fill) and kept band cells (filter)
  c->gram_row_ready = (c->P.gram_mode == 0);
  c->sets_ready = false;
  return HROM_OK;
}

hrom_status hrom_update_basis(hrom_ctx* c) {
  if (!c) return HROM_E_INVALID;
  if (c->k < 0) return HROM_E_STATE;
  const int w = c->w;
  const int64_t k = c->k;
  if (k < w - 1) return HROM_OK;
  c->odeim_k = -1;  // a new basis: its ODEIM points are computed by the next sampling
  hrom_status s;
  basis_join(c);  // C is rewritten below
  prof_begin(c, SEC_BASIS);
  const Win W = window_at(c, k);
  const bool rebase = (k == w - 1) || c->P.gram_mode == 1 || (k - c->rebase_k >= c->P.rebase_period) ||
                      (!c->gram_row_ready && !c->basis_ready);
  if (rebase) {
    prof_end(c, SEC_BASIS);
    prof_begin(c, SEC_REBASE);
    // Gram shift rho := the newest snapshot (any fixed reference inside the window controls the
    // cancellation of the centring algebra, G2; a slab-strided copy instead of a mean pass)
    {
      const size_t pitch = (size_t)c->g.nsr * TILE * sizeof(double);
      HROM_CK(cudaMemcpy2DAsync(c->b.rho, pitch, c->b.ring + (int64_t)c->slot_of(k) * TILE, pitch,
                                TILE * sizeof(double), (size_t)(c->g.Dp / TILE), cudaMemcpyDeviceToDevice, c->st));
    }
    const int s0 = W.slot[0];
    // consecutive slots are contiguous in the pointer table (see hrom_create); the Gram is
    // written straight into the slot-indexed C through the slot table
    if ((s = gram_full_dd(c, c->b.colptr + s0, c->g.nsr, W.nU, c->g.D, c->rho_ref(), c->b.C, c->b.Clo, kMaxSlots,
                          c->b.slot_tab + s0)) != HROM_OK)
      return s;
    prof_end(c, SEC_REBASE);
    prof_begin(c, SEC_BASIS);
    c->rebase_k = k;
  } else if (c->n_owed > 0) {
    // rows owed by skipped updates (finite z) and this step's row (a full step: a skip
    // at k-1 means k mod z = 0), each against the whole new window (covers the pairs between them)
    for (int i = 0; i < c->n_owed; ++i) {
      const int64_t kk = c->owed_rows[i];
      if (kk <= k - w || kk >= k) continue;
      if ((s = launch_gram_row(c, W, c->slot_of(kk))) != HROM_OK) return s;
      if ((s = reduce_gram_row(c, W, c->slot_of(kk), false)) != HROM_OK) return s;
    }
    if ((s = launch_gram_row(c, W, c->slot_of(k))) != HROM_OK) return s;
    if ((s = reduce_gram_row(c, W, c->slot_of(k), false)) != HROM_OK) return s;
  } else if (!c->gram_row_ready) {
    if ((s = launch_gram_row(c, c->win, c->slot_of(k))) != HROM_OK) return s;
    if ((s = reduce_gram_row(c, c->win, c->slot_of(k), false)) != HROM_OK) return s;
  } else {
    // fused row of the fill pass + band; if the step was redone as a full step (device flag
    // ureg[3]), the row is recomputed from the final gamma_k instead
    const unsigned long long* esc = c->last_hybrid ? c->b.ureg + 3 : nullptr;
    if (esc && (s = launch_gram_row(c, c->win, c->slot_of(k), esc)) != HROM_OK) return s;
    if ((s = reduce_gram_row(c, c->win, c->slot_of(k), true, esc)) != HROM_OK) return s;
  }
  prof_end(c, SEC_BASIS);
  // eigen-solve: deferred to the side stream after the sampling kernel (a cooperative kernel
  // that needs every SM), overlapping the next step's dt / masked RK3 / gathered Gram;
  // consumers call basis_join()
  c->eig_win = W;
  c->eig_todo = true;
  c->win = W;
  c->basis_ready = true;
  c->gram_row_ready = false;
  c->n_owed = 0;
  const bool proj = k == w - 1 || c->full_since_update;
  c->full_since_update = false;
  if (proj && k == w - 1 && c->P.odeim_points > 0) {
    // Algorithm 1: G_w = {} at k = w-1, so S-hat_w = P_w, the ODEIM points alone
    HROM_CK(cudaMemsetAsync(c->b.eps, 0, c->g.N * sizeof(double), c->st));
    c->eps_sparse = false;
  } else if (proj) {  // projection indicator: bootstrap (reading A19, P = S-hat mode), or after a full step k >= w (G8)
    basis_join(c);
    zvec_kernel<<<1, 128, 0, c->st>>>(c->b.A, c->b.lam, c->b.ireg, w, k == w - 1 ? 0.0 : 1.0 / w, c->b.zvec);
    HROM_LAUNCH_CK();
    ++c->nlaunch;
    if ((s = launch_fill(c, W, 2, plain(nullptr), plain(nullptr), false)) != HROM_OK) return s;
    if ((s = launch_eps_all(c)) != HROM_OK) return s;
    c->eps_sparse = false;
  }
  return HROM_OK;
}

static hrom_status sample_outputs(hrom_ctx* c, uint32_t* dev_mask_out, int32_t* dev_list_out,
                                  int32_t* dev_count_out);

hrom_status hrom_sample(hrom_ctx* c, double fraction, const double* dev_eps, uint32_t* dev_mask_out,
                        int32_t* dev_list_out, int32_t* dev_count_out) {
  if (!c) return HROM_E_INVALID;
  if (!(fraction > 0.0 && fraction <= 1.0)) return HROM_E_INVALID;
  const int64_t n_g = (int64_t)std::ceil(fraction * (double)c->g.N);
  hrom_status s;
  // the deferred eigen-solve starts first on the side stream; the cooperative sampling kernel
  // then runs on the other SMs (grid nsm - 1), so the eigen overlaps the sampling too.  In graph
  // mode it starts with the next step instead (a captured step must join its side-stream work)
  if (!c->graph_on && (s = flush_eigen(c)) != HROM_OK) return s;
  if (c->P.odeim_points > 0 && (s = odeim_for_basis(c)) != HROM_OK) return s;
  prof_begin(c, SEC_SAMPLE);
  if ((s = select_and_build(c, dev_eps ? dev_eps : c->b.eps, n_g)) != HROM_OK) return s;
  prof_end(c, SEC_SAMPLE);
  c->sets_ready = true;
  return sample_outputs(c, dev_mask_out, dev_list_out, dev_count_out);
}

static hrom_status sample_outputs(hrom_ctx* c, uint32_t* dev_mask_out, int32_t* dev_list_out,
                                  int32_t* dev_count_out) {
  if (dev_mask_out)
    HROM_CK(cudaMemcpyAsync(dev_mask_out, c->b.masks + (int64_t)M_S * c->mwords, c->mwords * sizeof(uint32_t),
                            cudaMemcpyDefault, c->st));
  if (dev_list_out)
    HROM_CK(cudaMemcpyAsync(dev_list_out, c->b.lists + (int64_t)L_S * c->g.N, c->g.N * sizeof(int32_t),
                            cudaMemcpyDefault, c->st));
  if (dev_count_out)
    HROM_CK(cudaMemcpyAsync(dev_count_out, c->b.counts + L_S, sizeof(int32_t), cudaMemcpyDefault, c->st));
  return HROM_OK;
}

hrom_status hrom_sample_rre(hrom_ctx* c, double delta, const double* dev_eps, uint32_t* dev_mask_out,
                            int32_t* dev_list_out, int32_t* dev_count_out) {
  if (!c) return HROM_E_INVALID;
  if (!(delta > 0.0 && delta <= 1.0)) return HROM_E_INVALID;
  hrom_status s;
  if (!c->graph_on && (s = flush_eigen(c)) != HROM_OK) return s;
  if (c->P.odeim_points > 0 && (s = odeim_for_basis(c)) != HROM_OK) return s;
  prof_begin(c, SEC_SAMPLE);
  if ((s = select_and_build(c, dev_eps ? dev_eps : c->b.eps, 0, delta)) != HROM_OK) return s;
  prof_end(c, SEC_SAMPLE);
  c->sets_ready = true;
  return sample_outputs(c, dev_mask_out, dev_list_out, dev_count_out);
}

hrom_status hrom_reconstruct(hrom_ctx* c, const uint32_t* dev_mask, double* dev_v, double* dev_y_out,
                             double* dev_eps_out) {
  if (!c || !dev_v) return HROM_E_INVALID;
  if (!c->basis_ready) return HROM_E_STATE;
  hrom_status s;
  if ((s = flush_eigen(c)) != HROM_OK) return s;
  if (dev_mask) {
    if ((s = build_sets(c, dev_mask)) != HROM_OK) return s;
    c->sets_ready = true;
  }
  if (!c->sets_ready) return HROM_E_STATE;
  prof_begin(c, SEC_GATHER);
  if ((s = gram_gathered(c, plain(dev_v))) != HROM_OK) return s;
  prof_end(c, SEC_GATHER);
  basis_join(c);
  prof_begin(c, SEC_SOLVE);
  if ((s = small_solve(c)) != HROM_OK) return s;
  prof_end(c, SEC_SOLVE);
  HROM_CK(cudaMemsetAsync(c->b.eps, 0, c->g.N * sizeof(double), c->st));
  prof_begin(c, SEC_FILL);
  if ((s = launch_fill(c, c->win, 0, plain(dev_v), plain(dev_v), false)) != HROM_OK) return s;
  prof_end(c, SEC_FILL);
  if ((s = launch_eps_cells(c)) != HROM_OK) return s;
  if (dev_y_out) HROM_CK(cudaMemcpyAsync(dev_y_out, c->b.y, c->r * sizeof(double), cudaMemcpyDefault, c->st));
  if (dev_eps_out)
    HROM_CK(cudaMemcpyAsync(dev_eps_out, c->b.eps, c->g.N * sizeof(double), cudaMemcpyDefault, c->st));
  return HROM_OK;
}

hrom_status hrom_filter(hrom_ctx* c, const uint32_t* dev_mask, double* dev_v, const double* dev_F,
                        uint8_t* dev_kept_out) {
  if (!c || !dev_v || !dev_F) return HROM_E_INVALID;
  hrom_status s;
  if (dev_mask) {
    if ((s = build_sets(c, dev_mask)) != HROM_OK) return s;
    c->sets_ready = true;
  }
  if (!c->sets_ready) return HROM_E_STATE;
  prof_begin(c, SEC_FILTER);
  if ((s = launch_filter(c, plain(dev_v), plain(dev_F), dev_kept_out)) != HROM_OK) return s;
  prof_end(c, SEC_FILTER);
  return HROM_OK;
}

namespace {
HostSnap snap_get(const hrom_ctx* c, double dt_override) {
  HostSnap h;
  h.k = c->k;
  h.rebase_k = c->rebase_k;
  h.smax_k = c->smax_k;
  h.kinc_newest = c->kinc_newest;
  h.kinc_rebase = c->kinc_rebase;
  h.odeim_k = c->odeim_k;
  h.nlaunch = c->nlaunch;
  h.last_err_cell = c->last_err_cell;
  h.basis_ready = c->basis_ready;
  h.sets_ready = c->sets_ready;
  h.gram_row_ready = c->gram_row_ready;
  h.full_since_update = c->full_since_update;
  h.last_hybrid = c->last_hybrid;
  h.basis_pending = c->basis_pending;
  h.eig_todo = c->eig_todo;
  h.bg_pending = c->bg_pending;
  h.kinc_valid = c->kinc_valid;
  h.eps_sparse = c->eps_sparse;
  h.n_owed = c->n_owed;
  h.samples_since_gather = c->samples_since_gather;
  h.fill_grid = c->fill_grid;
  h.odeim_n = c->odeim_n;
  h.points_used = c->points_used;
  for (int i = 0; i < 4; ++i) h.owed_rows[i] = c->owed_rows[i];
  h.dt_override = dt_override;
  h.win = c->win;
  h.eig_win = c->eig_win;
  return h;
}
// the entry state of a captured step, up to the shift of the k-tracking fields by a whole
// number of ring periods
bool snap_same(const HostSnap& a, const HostSnap& b, int nslots) {
  const int64_t dk = b.k - a.k;
  return dk % nslots == 0 && b.smax_k - a.smax_k == dk && b.kinc_newest - a.kinc_newest == dk &&
         a.rebase_k == b.rebase_k && a.kinc_rebase == b.kinc_rebase && a.odeim_k == b.odeim_k &&
         a.basis_ready == b.basis_ready && a.sets_ready == b.sets_ready && a.gram_row_ready == b.gram_row_ready &&
         a.full_since_update == b.full_since_update && a.last_hybrid == b.last_hybrid &&
         a.basis_pending == b.basis_pending && a.eig_todo == b.eig_todo && a.bg_pending == b.bg_pending &&
         a.kinc_valid == b.kinc_valid && a.eps_sparse == b.eps_sparse && a.n_owed == b.n_owed &&
         a.samples_since_gather == b.samples_since_gather && a.fill_grid == b.fill_grid &&
         a.odeim_n == b.odeim_n && a.dt_override == b.dt_override;
}
void snap_apply(hrom_ctx* c, const HostSnap& post, int64_t dk, int64_t dlaunch) {
  c->k = post.k + dk;
  c->rebase_k = post.rebase_k;
  c->smax_k = post.smax_k + dk;
  c->kinc_newest = post.kinc_newest + dk;
  c->kinc_rebase = post.kinc_rebase;
  c->odeim_k = post.odeim_k;
  c->nlaunch += dlaunch;
  c->basis_ready = post.basis_ready;
  c->sets_ready = post.sets_ready;
  c->gram_row_ready = post.gram_row_ready;
  c->full_since_update = post.full_since_update;
  c->last_hybrid = post.last_hybrid;
  c->basis_pending = post.basis_pending;
  c->eig_todo = post.eig_todo;
  c->bg_pending = post.bg_pending;
  c->kinc_valid = post.kinc_valid;
  c->eps_sparse = post.eps_sparse;
  c->n_owed = post.n_owed;
  c->samples_since_gather = post.samples_since_gather;
  c->fill_grid = post.fill_grid;
  c->odeim_n = post.odeim_n;
  c->points_used = post.points_used;
  c->win = post.win;
  c->eig_win = post.eig_win;
}
// a step the graph path may capture / replay: Algorithm 1 in its steady state (a hybrid step
// followed by the basis update and the sampling, z = infinity), no host-visible outputs
bool graph_eligible(const hrom_ctx* c, int32_t* dev_count_out) {
  static const bool nocap = getenv("HROM_GRAPH_NOCAPTURE") != nullptr;  // debug: graph-mode order, eager launches
  return c->graph_on && !nocap && !c->prof && dev_count_out == nullptr && c->P.full_period <= 0 && c->P.odeim_points == 0 &&
         c->P.gram_mode == 0 && c->P.gather_mode == 0 && c->k >= c->w + 1 && c->last_hybrid && c->sets_ready &&
         c->basis_ready && c->eig_todo && !c->basis_pending && !c->bg_pending && c->kinc_valid &&
         c->samples_since_gather == 1 && c->kinc_newest == c->k - 1 && c->smax_k == c->k && c->n_owed == 0 &&
         !hrom_sync_debug();
}
hrom_status step_eager(hrom_ctx* c, double dt_override, int32_t* dev_count_out);
}  // namespace

hrom_status hrom_step_ex(hrom_ctx* c, double dt_override, int32_t* dev_count_out) {
  if (!c) return HROM_E_INVALID;
  if (c->k < 0) return HROM_E_STATE;
  if (!graph_eligible(c, dev_count_out)) return step_eager(c, dt_override, dev_count_out);
  GraphSlot& gs = c->graphs[c->slot_of(c->k)];
  const HostSnap entry = snap_get(c, dt_override);
  // graphs run on the library's own capture stream, ordered after / before the context stream
  // (which may be the legacy default stream, where capture is not permitted)
  cudaStream_t user = c->st;
  HROM_CK(cudaEventRecord(c->ev_g0, user));
  HROM_CK(cudaStreamWaitEvent(c->gst, c->ev_g0, 0));
  if (gs.exec && snap_same(gs.pre, entry, c->nslots)) {
    snap_apply(c, gs.post, entry.k - gs.pre.k, gs.post.nlaunch - gs.pre.nlaunch);
    HROM_CK(cudaGraphLaunch(gs.exec, c->gst));
  } else {
    // capture this step (nothing executes while capturing), instantiate, then launch it
    if (gs.exec) {
      cudaGraphExecDestroy(gs.exec);
      gs.exec = nullptr;
    }
    HROM_CK(cudaStreamBeginCapture(c->gst, cudaStreamCaptureModeThreadLocal));
    c->st = c->gst;
    const hrom_status s = step_eager(c, dt_override, nullptr);
    c->st = user;
    cudaGraph_t graph = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(c->gst, &graph);
    if (s != HROM_OK) {
      if (graph) cudaGraphDestroy(graph);
      return s;
    }
    HROM_CK(ec);
    const cudaError_t ei = cudaGraphInstantiate(&gs.exec, graph, 0);
    cudaGraphDestroy(graph);
    HROM_CK(ei);
    gs.pre = entry;
    gs.post = snap_get(c, dt_override);
    ++c->graph_captures;
    HROM_CK(cudaGraphLaunch(gs.exec, c->gst));
  }
  ++c->graph_launches;
  HROM_CK(cudaEventRecord(c->ev_g1, c->gst));
  HROM_CK(cudaStreamWaitEvent(user, c->ev_g1, 0));
  return HROM_OK;
}

hrom_status hrom_set_graph(hrom_ctx* c, int32_t enable) {
  if (!c) return HROM_E_INVALID;
  c->graph_on = enable != 0;
  if (c->graph_on && c->graphs.empty()) c->graphs.resize(c->nslots);
  if (c->graph_on && !c->gst) {
    HROM_CK(cudaStreamCreateWithFlags(&c->gst, cudaStreamNonBlocking));
    HROM_CK(cudaEventCreateWithFlags(&c->ev_g0, cudaEventDisableTiming));
    HROM_CK(cudaEventCreateWithFlags(&c->ev_g1, cudaEventDisableTiming));
  }
  if (!c->graph_on) {
    // the eager path flushes the deferred eigen-solve at the sampling; a pending one (graph mode
    // defers it to the next step) is launched by the next step's flush_eigen as well
    for (auto& gs : c->graphs)
      if (gs.exec) {
        cudaGraphExecDestroy(gs.exec);
        gs.exec = nullptr;
      }
  }
  return HROM_OK;
}

int64_t hrom_graph_launches(const hrom_ctx* c) { return c ? c->graph_launches : 0; }

namespace {
hrom_status step_eager(hrom_ctx* c, double dt_override, int32_t* dev_count_out) {
  const int64_t kn = c->k + 1;
  const int64_t z = c->P.full_period;
  // Algorithm 1 line P:557: full HDM step while k+1 <= w or k mod z = 0
  const bool full = (kn + 1 <= c->w) || (z > 0 && kn % z == 0);
  hrom_status s;
  if (full) {
    s = hrom_full_step(c, dt_override, nullptr);
    if (s == HROM_OK && dev_count_out) {
      set_i32_kernel<<<1, 1, 0, c->st>>>(dev_count_out, (int32_t)c->g.N);
      HROM_LAUNCH_CK();
      ++c->nlaunch;
    }
  } else {
    s = hrom_hybrid_step(c, nullptr, dt_override, nullptr);
    if (s == HROM_OK && dev_count_out)
      HROM_CK(cudaMemcpyAsync(dev_count_out, c->b.counts + L_S, sizeof(int32_t), cudaMemcpyDeviceToDevice, c->st));
  }
  if (s != HROM_OK) return s;
  if (kn >= c->w - 1) {
    if (z > 0 && (kn + 1) % z == 0) {
      // no basis update / sampling before a full step; the window-Gram row of
      // gamma_kn is owed to the next update (only the last w can still be in a window)
      if (c->n_owed == 4) {
        for (int i = 0; i < 3; ++i) c->owed_rows[i] = c->owed_rows[i + 1];
        c->n_owed = 3;
      }
      c->owed_rows[c->n_owed++] = kn;
      c->full_since_update = false;  // the next update follows the next (full) step
    } else {
      if ((s = hrom_update_basis(c)) != HROM_OK) return s;
      s = c->P.sample_mode == 1 ? hrom_sample_rre(c, c->P.rre_delta, nullptr, nullptr, nullptr, nullptr)
                                : hrom_sample(c, c->P.sample_fraction, nullptr, nullptr, nullptr, nullptr);
      if (s != HROM_OK) return s;
    }
  }
  return HROM_OK;
}
}  // namespace

hrom_status hrom_step(hrom_ctx* c, double dt_override) { return hrom_step_ex(c, dt_override, nullptr); }

hrom_status hrom_rel_l1_error(hrom_ctx* c, const double* dev_a, const double* dev_b, double* host_out) {
  if (!c || !dev_a || !dev_b || !host_out) return HROM_E_INVALID;
  const int nb = std::min<int64_t>(kL1Blocks, std::max<int64_t>(1, (c->g.D + 255) / 256));
  l1_partial_kernel<<<nb, 256, 0, c->st>>>(dev_a, dev_b, c->g.D, c->b.l1part);
  HROM_LAUNCH_CK();
  l1_final_kernel<<<1, 1024, 0, c->st>>>(c->b.l1part, nb, c->b.dreg + 8);
  HROM_LAUNCH_CK();
  c->nlaunch += 2;
  double r[2];
  HROM_CK(cudaMemcpyAsync(r, c->b.dreg + 8, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->st));
  HROM_CK(cudaStreamSynchronize(c->st));
  *host_out = r[0] / r[1];
  return HROM_OK;
}

hrom_status hrom_sync(hrom_ctx* c) {
  if (!c) return HROM_E_INVALID;
  basis_join(c);
  HROM_CK(cudaStreamSynchronize(c->st));
  unsigned long long bad = 0;
  HROM_CK(cudaMemcpy(&bad, c->b.ureg + 1, sizeof(bad), cudaMemcpyDeviceToHost));
  if (bad != ~0ull) {
    c->last_err_cell = (int64_t)bad;
    return HROM_E_POSITIVITY;
  }
  return HROM_OK;
}

int32_t hrom_points_used(const hrom_ctx* c) { return c ? c->points_used : 0; }

hrom_status hrom_join(hrom_ctx* c) {
  if (!c) return HROM_E_INVALID;
  basis_join(c);
  return HROM_OK;
}

int64_t hrom_error_cell(const hrom_ctx* c) { return c ? c->last_err_cell : -1; }
int64_t hrom_step_index(const hrom_ctx* c) { return c ? c->k : -1; }
int64_t hrom_mask_words(const hrom_ctx* c) { return c ? c->mwords : 0; }

int32_t hrom_effective_rank(hrom_ctx* c) {
  if (!c) return -1;
  int32_t r = 0;
  basis_join(c);
  if (cudaStreamSynchronize(c->st) != cudaSuccess) return -1;
  if (cudaMemcpy(&r, c->b.ireg, sizeof(r), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
  return r;
}

hrom_status hrom_put_snapshot(hrom_ctx* c, int64_t k, const double* any_q) {
  if (!c || !any_q || k < 0) return HROM_E_INVALID;
  return copy_slot(c, c->slot_of(k), any_q, nullptr);
}

hrom_status hrom_rebuild_basis(hrom_ctx* c, int64_t k, const uint32_t* any_mask_next) {
  if (!c) return HROM_E_INVALID;
  if (k < c->w) return HROM_E_INVALID;
  basis_join(c);
  HROM_CK(cudaMemsetAsync(c->b.ureg + 1, 0xff, sizeof(unsigned long long), c->st));
  c->k = k;
  c->last_hybrid = false;
  c->full_since_update = false;
  c->n_owed = 0;
  c->kinc_valid = false;
  c->eps_sparse = false;
  c->basis_ready = false;
  c->gram_row_ready = false;
  c->rebase_k = -1000000;
  hrom_status s = hrom_update_basis(c);
  if (s != HROM_OK) return s;
  if (any_mask_next) {
    uint32_t* S = c->b.masks + (int64_t)M_S * c->mwords;
    HROM_CK(cudaMemcpyAsync(S, any_mask_next, c->mwords * sizeof(uint32_t), cudaMemcpyDefault, c->st));
    if ((s = build_sets(c, nullptr)) != HROM_OK) return s;
    c->sets_ready = true;
  }
  return HROM_OK;
}

hrom_status hrom_set_window(hrom_ctx* c, int64_t k, const double* any_snaps, int32_t nsnaps,
                            const uint32_t* any_mask_next) {
  if (!c || !any_snaps) return HROM_E_INVALID;
  if (k < c->w || nsnaps != c->w + 1) return HROM_E_INVALID;
  for (int t = 0; t < nsnaps; ++t) {
    hrom_status s0 = hrom_put_snapshot(c, k - c->w + t, any_snaps + (int64_t)t * c->g.D);
    if (s0 != HROM_OK) return s0;
  }
  return hrom_rebuild_basis(c, k, any_mask_next);
}

hrom_status hrom_get_basis(hrom_ctx* c, double* dev_phi, double* dev_psi) {
  if (!c) return HROM_E_INVALID;
  if (!c->basis_ready) return HROM_E_STATE;
  basis_join(c);
  return lift(c, c->win, dev_phi, dev_psi);
}

hrom_status hrom_get_indicator(hrom_ctx* c, double* any_eps) {
  if (!c || !any_eps) return HROM_E_INVALID;
  HROM_CK(cudaMemcpyAsync(any_eps, c->b.eps, c->g.N * sizeof(double), cudaMemcpyDefault, c->st));
  return HROM_OK;
}

hrom_status hrom_get_mask(hrom_ctx* c, uint32_t* any_mask) {
  if (!c || !any_mask) return HROM_E_INVALID;
  HROM_CK(cudaMemcpyAsync(any_mask, c->b.masks + (int64_t)M_S * c->mwords, c->mwords * sizeof(uint32_t),
                          cudaMemcpyDefault, c->st));
  return HROM_OK;
}

hrom_status hrom_get_y(hrom_ctx* c, double* any_y) {
  if (!c || !any_y) return HROM_E_INVALID;
  HROM_CK(cudaMemcpyAsync(any_y, c->b.y, c->r * sizeof(double), cudaMemcpyDefault, c->st));
  return HROM_OK;
}

hrom_status hrom_get_eigen(hrom_ctx* c, double* any_lambda) {
  if (!c || !any_lambda) return HROM_E_INVALID;
  basis_join(c);
  HROM_CK(cudaMemcpyAsync(any_lambda, c->b.lam, c->w * sizeof(double), cudaMemcpyDefault, c->st));
  return HROM_OK;
}

hrom_status hrom_gram(hrom_ctx* c, const double* const* dev_cols, int32_t ncol, int64_t rows, const double* dev_rho,
                      double* dev_C) {
  if (!c || !dev_cols || !dev_C || ncol < 1 || ncol > kMaxSlots + 14 || rows < 0) return HROM_E_INVALID;
  return gram_full(c, dev_cols, 1, ncol, rows, plain(dev_rho), dev_C, ncol, nullptr);
}

hrom_status hrom_project(hrom_ctx* c, const double* dev_phi, int32_t m, double* dev_C) {
  if (!c || !dev_phi || !dev_C || m < 1 || m > kMaxR) return HROM_E_INVALID;
  if (!c->basis_ready) return HROM_E_STATE;
  basis_join(c);
  std::vector<const double*> cols(m);
  for (int i = 0; i < m; ++i) cols[i] = dev_phi + (int64_t)i * c->g.D;
  return project_window(c, cols.data(), m, dev_C);
}

hrom_status hrom_put_state(hrom_ctx* c, const double* any_q) {
  if (!c || !any_q) return HROM_E_INVALID;
  if (c->k < 0) return HROM_E_STATE;
  return copy_slot(c, c->slot_of(c->k), any_q, nullptr);
}

hrom_status hrom_profile(hrom_ctx* c, int32_t enable) {
  if (!c) return HROM_E_INVALID;
  basis_join(c);
  HROM_CK(cudaStreamSynchronize(c->st));
  c->ev_pairs.clear();
  c->ev_next = 0;
  c->prof = enable != 0;
  if (c->prof && c->ev_pool.empty()) {
    c->ev_pool.resize(1 << 15);
    for (auto& e : c->ev_pool) HROM_CK(cudaEventCreate(&e));
  }
  return HROM_OK;
}

hrom_status hrom_profile_read(hrom_ctx* c, double* ms, int64_t* counts, int32_t nsec) {
  if (!c || !ms || !counts) return HROM_E_INVALID;
  basis_join(c);
  HROM_CK(cudaStreamSynchronize(c->st));
  for (int i = 0; i < nsec; ++i) {
    ms[i] = 0.0;
    counts[i] = 0;
  }
  for (const auto& p : c->ev_pairs) {
    float t = 0.f;
    HROM_CK(cudaEventElapsedTime(&t, c->ev_pool[p.second.first], c->ev_pool[p.second.second]));
    if (p.first < nsec) {
      ms[p.first] += t;
      counts[p.first] += 1;
    }
  }
  c->ev_pairs.clear();
  c->ev_next = 0;
  return HROM_OK;
}

int64_t hrom_launch_count(const hrom_ctx* c) { return c ? c->nlaunch : 0; }

hrom_status hrom_debug_counters(hrom_ctx* c, int32_t* any_out, int32_t n) {
  if (!c || !any_out || n < 0 || n > 32) return HROM_E_INVALID;
  basis_join(c);
  HROM_CK(cudaStreamSynchronize(c->st));
  HROM_CK(cudaMemcpy(any_out, c->b.ireg, std::min(n, 16) * sizeof(int32_t), cudaMemcpyDefault));
  if (n > 16) HROM_CK(cudaMemcpy(any_out + 16, c->b.counts, (n - 16) * sizeof(int32_t), cudaMemcpyDefault));
  return HROM_OK;
}

hrom_status hrom_debug_read(hrom_ctx* c, int32_t which, double* any_out, int64_t n) {
  if (!c || !any_out || n < 0) return HROM_E_INVALID;
  basis_join(c);
  const double* src = nullptr;
  int64_t cap = 0;
  const int64_t k2 = (int64_t)kMaxSlots * kMaxSlots;
  switch (which) {
    case 0: src = c->b.C; cap = k2; break;
    case 1: src = c->b.Clo; cap = k2; break;
    case 2: src = c->b.Mdd; cap = 2 * k2; break;
    case 3: src = c->b.Zf; cap = k2; break;
    case 4: src = c->b.A; cap = (int64_t)kMaxW * kMaxR; break;
    case 5: src = c->b.lam; cap = kMaxSlots; break;
    default: return HROM_E_INVALID;
  }
  if (n > cap) return HROM_E_INVALID;
  HROM_CK(cudaMemcpyAsync(any_out, src, n * sizeof(double), cudaMemcpyDefault, c->st));
  return HROM_OK;
}

hrom_status hrom_debug_timers(hrom_ctx* c, int64_t* host_out, int32_t n) {
  if (!c || !host_out || n < 0 || n > 128) return HROM_E_INVALID;
  basis_join(c);
  HROM_CK(cudaStreamSynchronize(c->st));
  HROM_CK(cudaMemcpy(host_out, c->b.dbg, n * sizeof(int64_t), cudaMemcpyDeviceToHost));
  return HROM_OK;
}

}  // extern "C"
