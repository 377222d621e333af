// sampling_filter.cpp -- oracle: sampling sets, indicator selection, Shapiro seam filter.
// TEST INFRASTRUCTURE ONLY (see oracle.h).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include "common.hpp"

using namespace orc;

extern "C" {

// Neighbors (Fig. 1): cross C_h = {(+-a,0),(0,+-b): a,b <= h} (O10.1).
// Transmissive grids clip at the boundary, periodic grids wrap (reading A9).
void orc_dilate_cross(const orc_grid* g, const uint8_t* in, int32_t h, uint8_t* out) {
  Grid G(g);
  for (int j = 0; j < G.ny; ++j)
    for (int i = 0; i < G.nx; ++i) {
      bool any = false;
      for (int a = -h; a <= h && !any; ++a) {
        const int ii = i + a;
        if (G.bc == 0 && (ii < 0 || ii >= G.nx)) continue;
        if (in[(int64_t)j * G.nx + G.ix(ii)]) any = true;
      }
      if (G.dim == 2)
        for (int b = -h; b <= h && !any; ++b) {
          const int jj = j + b;
          if (G.bc == 0 && (jj < 0 || jj >= G.ny)) continue;
          if (in[(int64_t)G.iy(jj) * G.nx + i]) any = true;
        }
      out[(int64_t)j * G.nx + i] = any ? 1 : 0;
    }
}

// square Q_W = {(a,b): |a|,|b| <= W} (O13 band, reading A21)
// W < 0: the whole grid (the paper's filter over the whole hybrid state; NEXT-2)
void orc_dilate_square(const orc_grid* g, const uint8_t* in, int32_t W, uint8_t* out) {
  Grid G(g);
  if (W < 0) {
    for (int64_t n = 0; n < G.N; ++n) out[n] = 1;
    return;
  }
  const int Wy = (G.dim == 2) ? W : 0;
  for (int j = 0; j < G.ny; ++j)
    for (int i = 0; i < G.nx; ++i) {
      bool any = false;
      for (int b = -Wy; b <= Wy && !any; ++b) {
        const int jj = j + b;
        if (G.bc == 0 && (jj < 0 || jj >= G.ny)) continue;
        for (int a = -W; a <= W && !any; ++a) {
          const int ii = i + a;
          if (G.bc == 0 && (ii < 0 || ii >= G.nx)) continue;
          if (in[(int64_t)G.iy(jj) * G.nx + G.ix(ii)]) any = true;
        }
      }
      out[(int64_t)j * G.nx + i] = any ? 1 : 0;
    }
}

int64_t orc_n_g(double f, int64_t N) { return (int64_t)std::ceil(f * (double)N); }

// H8 / O15 (reading A18): order cells by descending eps, ties by
// ascending index; G = the first min(n_g, #{eps>0}) cells with eps > 0.
int64_t orc_select(const double* eps, int64_t N, int64_t n_g, uint8_t* mask_out) {
  std::vector<int64_t> idx;
  for (int64_t n = 0; n < N; ++n) {
    mask_out[n] = 0;
    if (eps[n] > 0.0) idx.push_back(n);
  }
  std::stable_sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) { return eps[a] > eps[b]; });
  const int64_t k = std::min<int64_t>(n_g, (int64_t)idx.size());
  for (int64_t t = 0; t < k; ++t) mask_out[idx[t]] = 1;
  return k;
}

// RRE-delta rule (Eq. rre): order cells by descending eps (ties by ascending index,
// as in the fraction rule) and take the smallest n_g with
//   RRE(n_g) = sum_{j <= n_g} eps_{i_j} / sum_j eps_j >= delta.
// The sums are the exact real sums (reading A35: no rounding decides the integer n_g): every
// double eps >= 0 is an integer multiple of 2^-1074, so the sums are exact big integers in that
// unit, and RRE(n) >= delta  <=>  S_n >= delta T  <=>  S_n >= ceil(delta T) (S_n integer).
// An all-zero indicator selects nothing.
namespace {
struct BigNat {  // little-endian base-2^32 natural number
  std::vector<uint64_t> l;
  void add_shifted(uint64_t m, int shift) {  // += m * 2^shift
    const int w = shift / 32, b = shift % 32;
    unsigned __int128 v = (unsigned __int128)m << b;
    size_t i = (size_t)w;
    while (v != 0) {
      if (l.size() <= i) l.resize(i + 1, 0);
      const unsigned __int128 t = (unsigned __int128)l[i] + (uint64_t)(v & 0xffffffffu);
      l[i] = (uint64_t)(t & 0xffffffffu);
      v = (v >> 32) + (t >> 32);
      ++i;
    }
  }
  void trim() {
    while (!l.empty() && l.back() == 0) l.pop_back();
  }
};
int cmp(BigNat a, BigNat b) {
  a.trim();
  b.trim();
  if (a.l.size() != b.l.size()) return a.l.size() < b.l.size() ? -1 : 1;
  for (size_t i = a.l.size(); i-- > 0;)
    if (a.l[i] != b.l[i]) return a.l[i] < b.l[i] ? -1 : 1;
  return 0;
}
// eps = m * 2^(e - 1074) with m < 2^53 an integer (e >= 0)
void split(double x, uint64_t* m, int* e) {
  uint64_t bits;
  std::memcpy(&bits, &x, 8);
  const int be = (int)((bits >> 52) & 0x7ff);
  const uint64_t f = bits & ((1ull << 52) - 1);
  *m = be == 0 ? f : (f | (1ull << 52));
  *e = be == 0 ? 0 : be - 1;
}
}  // namespace

int64_t orc_select_rre(const double* eps, int64_t N, double delta, uint8_t* mask_out) {
  std::vector<int64_t> idx;
  BigNat T;
  for (int64_t n = 0; n < N; ++n) {
    mask_out[n] = 0;
    if (eps[n] > 0.0) {
      idx.push_back(n);
      uint64_t m;
      int e;
      split(eps[n], &m, &e);
      T.add_shifted(m, e);
    }
  }
  if (idx.empty() || !(delta > 0.0)) return 0;
  std::stable_sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) { return eps[a] > eps[b]; });
  // R = ceil(delta T): delta = dm 2^-sh (dm < 2^53), R = ceil(T dm / 2^sh)
  int ex;
  const double mant = std::frexp(delta, &ex);
  const uint64_t dm = (uint64_t)std::ldexp(mant, 53);
  const int sh = 53 - ex;
  BigNat P;  // T * dm
  for (size_t i = 0; i < T.l.size(); ++i)
    if (T.l[i]) {
      P.add_shifted(T.l[i] * (dm & 0xffffffffu), 32 * (int)i);
      P.add_shifted(T.l[i] * (dm >> 32), 32 * (int)i + 32);
    }
  BigNat R;  // floor(P / 2^sh) + (remainder != 0)
  bool rem = false;
  for (size_t i = 0; i < P.l.size(); ++i) {
    const int bitpos = 32 * (int)i;  // limb i covers bits [bitpos, bitpos + 32)
    for (int b = 0; b < 32; ++b) {
      if (!((P.l[i] >> b) & 1u)) continue;
      const int q = bitpos + b - sh;
      if (q < 0) rem = true;
      else R.add_shifted(1, q);
    }
  }
  if (rem) R.add_shifted(1, 0);
  BigNat S;
  int64_t ng = 0;
  for (size_t t = 0; t < idx.size(); ++t) {
    uint64_t m;
    int e;
    split(eps[idx[t]], &m, &e);
    S.add_shifted(m, e);
    mask_out[idx[t]] = 1;
    ng = (int64_t)t + 1;
    if (cmp(S, R) >= 0) break;
  }
  return ng;
}

// ODEIM_{n_p}(Phi) (Eq. 10; NEXT-1).  The cited algorithm is not in the container:
// reading A36 = SPEC's greedy DEIM-and-continue.  Phi is D x m (col-major,
// orthonormal columns), DOF e belongs to cell e mod N.  Point j = 1..n_p uses mode
// l = ((j-1) mod m) + 1: c = min-norm LSQ of Phi[P, 1..l-1] c = phi_l[P] (A13 cut; P = the DOF
// rows chosen so far), residual rho = phi_l - Phi[:, 1..l-1] c with the rows of already chosen
// cells excluded, p_j = argmax_e |rho_e| (ties: lowest e).  The first m points are DEIM
// (interpolation), the rest oversample.  Returns n_p, or -1 if n_p > N or m < 1.
int32_t orc_odeim(const double* Phi, int64_t D, int32_t m, int64_t N, int32_t n_p, double cut,
                  int32_t* cells_out, int64_t* rows_out) {
  if (m < 1 || n_p < 0 || n_p > N) return -1;
  std::vector<uint8_t> chosen(N, 0);
  std::vector<int64_t> P;
  for (int32_t j = 0; j < n_p; ++j) {
    const int l = j % m;  // 0-based mode index
    const double* phil = Phi + (int64_t)l * D;
    std::vector<double> c(l, 0.0);
    if (l > 0) {
      const int64_t np = (int64_t)P.size();
      std::vector<double> A(np * l), b(np);
      for (int i = 0; i < l; ++i)
        for (int64_t q = 0; q < np; ++q) A[(int64_t)i * np + q] = Phi[(int64_t)i * D + P[q]];
      for (int64_t q = 0; q < np; ++q) b[q] = phil[P[q]];
      orc_lsq(A.data(), np, l, b.data(), cut, c.data());
    }
    int64_t best = -1;
    double bv = -1.0;
    for (int64_t e = 0; e < D; ++e) {
      if (chosen[e % N]) continue;
      double r = phil[e];
      for (int i = 0; i < l; ++i) r -= Phi[(int64_t)i * D + e] * c[i];
      const double a = std::fabs(r);
      if (a > bv) {  // strict: ties keep the lowest e
        bv = a;
        best = e;
      }
    }
    P.push_back(best);
    chosen[best % N] = 1;
    cells_out[j] = (int32_t)(best % N);
    rows_out[j] = best;
  }
  return n_p;
}

// Shapiro stencils (reading A24): order 2 (1,2,1)/4, 4 (-1,4,10,4,-1)/16,
// 6 (1,-6,15,44,15,-6,1)/64.  Line ends: zeroth-order extrapolation or wrap.
static int shapiro_coef(int order, const double** c, double* den) {
  static const double c2[3] = {1, 2, 1};
  static const double c4[5] = {-1, 4, 10, 4, -1};
  static const double c6[7] = {1, -6, 15, 44, 15, -6, 1};
  if (order == 2) { *c = c2; *den = 4.0; return 1; }
  if (order == 4) { *c = c4; *den = 16.0; return 2; }
  *c = c6; *den = 64.0; return 3;
}

void orc_shapiro_1d(const double* line, int32_t n, int32_t order, int32_t periodic, double* out) {
  const double* c;
  double den;
  const int rad = shapiro_coef(order, &c, &den);
  for (int i = 0; i < n; ++i) {
    double s = 0.0;
    for (int m = -rad; m <= rad; ++m) {
      int k = i + m;
      if (periodic) k = ((k % n) + n) % n;
      else k = k < 0 ? 0 : (k >= n ? n - 1 : k);
      s += c[m + rad] * line[k];
    }
    out[i] = s / den;
  }
}

}  // extern "C"

namespace {

// H7 / O13 seam filter (readings A21-A24).  Fcell(state, n, F4) gives the HDM
// function F_k at cell n for the given state: the explicit path's F does not depend on the
// state (the full RK3 map of gamma_{k-1}, A22); the implicit path's F_k(v) does (NEXT-4,
// P:179-189), so the residual v - F_k(v) is re-evaluated on the filtered candidate.
template <class FC>
int64_t seam_filter_impl(const orc_grid* g, const orc_params* p, double* v, const uint8_t* mask_S,
                         uint8_t* kept_out, int32_t* sweeps_out, const FC& Fcell) {
  Grid G(g);
  std::vector<uint8_t> sq(G.N), B(G.N), kept(G.N, 0);
  orc_dilate_square(g, mask_S, p->W, sq.data());
  std::vector<int64_t> band;
  for (int64_t n = 0; n < G.N; ++n) {
    B[n] = (sq[n] && !mask_S[n]) ? 1 : 0;
    if (B[n]) band.push_back(n);
  }
  std::vector<double> vp(G.D), vpp(G.D);
  for (int oi = 0; oi < p->n_filter_orders; ++oi) {
    const int order = p->filter_orders[oi];
    const double* c;
    double den;
    const int rad = shapiro_coef(order, &c, &den);
    int sweeps = 0;
    for (int sw = 0; sw < p->filter_max_sweeps; ++sw) {
      ++sweeps;
      // v' = S^x(v) on B; off-B values unchanged (read-only)
      std::copy(v, v + G.D, vp.begin());
      for (int64_t n : band) {
        const int i = (int)(n % G.nx), j = (int)(n / G.nx);
        for (int var = 0; var < G.c; ++var) {
          double s = 0.0;
          for (int m = -rad; m <= rad; ++m)
            s += c[m + rad] * v[var * G.N + (int64_t)j * G.nx + G.ix(i + m)];
          vp[var * G.N + n] = s / den;
        }
      }
      // v'' = S^y(v') on B (2D only)
      std::copy(vp.begin(), vp.end(), vpp.begin());
      if (G.dim == 2)
        for (int64_t n : band) {
          const int i = (int)(n % G.nx), j = (int)(n / G.nx);
          for (int var = 0; var < G.c; ++var) {
            double s = 0.0;
            for (int m = -rad; m <= rad; ++m)
              s += c[m + rad] * vp[var * G.N + (int64_t)G.iy(j + m) * G.nx + i];
            vpp[var * G.N + n] = s / den;
          }
        }
      // residual gate: r = max_var |v - F| per cell; keep where r_new < r_old.
      // eps_f stop (reading A23'): the relative decrease counts only cells whose old residual is
      // above the rounding level of the state, r_old > 2^-40 max_var |F| (rounding noise would
      // otherwise decide the sweep count)
      int64_t nkept = 0;
      double maxdec = 0.0;
      // (all residuals of the sweep are evaluated before v changes)
      std::vector<double> Fo((size_t)band.size() * G.c), Fn((size_t)band.size() * G.c);
      for (size_t b = 0; b < band.size(); ++b) {
        Fcell(v, band[b], &Fo[b * G.c]);
        Fcell(vpp.data(), band[b], &Fn[b * G.c]);
      }
      for (size_t b = 0; b < band.size(); ++b) {
        const int64_t n = band[b];
        double rold = 0.0, rnew = 0.0, fs = 0.0;
        for (int var = 0; var < G.c; ++var) {
          const int64_t e = var * G.N + n;
          rold = std::max(rold, std::fabs(v[e] - Fo[b * G.c + var]));
          rnew = std::max(rnew, std::fabs(vpp[e] - Fn[b * G.c + var]));
          fs = std::max(fs, std::fabs(Fo[b * G.c + var]));
        }
        if (rnew < rold) {
          ++nkept;
          kept[n] = 1;
          if (rold > 0x1p-40 * fs) maxdec = std::max(maxdec, (rold - rnew) / rold);
          for (int var = 0; var < G.c; ++var) v[var * G.N + n] = vpp[var * G.N + n];
        }
      }
      if (nkept == 0) break;                  // empty keep-set: stop this order
      if (maxdec < p->filter_eps) break;      // relative decrease < eps_f
    }
    if (sweeps_out) sweeps_out[oi] = sweeps;
  }
  int64_t total = 0;
  for (int64_t n = 0; n < G.N; ++n) {
    if (kept_out) kept_out[n] = kept[n];
    total += kept[n];
  }
  return total;
}

}  // namespace

extern "C" {

int64_t orc_seam_filter(const orc_grid* g, const orc_params* p, double* v, const double* F,
                        const uint8_t* mask_S, uint8_t* kept_out, int32_t* sweeps_out) {
  Grid G(g);
  auto Fcell = [&](const double*, int64_t n, double* F4) {
    for (int var = 0; var < G.c; ++var) F4[var] = F[var * G.N + n];
  };
  return seam_filter_impl(g, p, v, mask_S, kept_out, sweeps_out, Fcell);
}

// the same filter gated by the implicit residual v - F_k(v) (NEXT-4; P:419-432 with Eq. hdm)
int64_t orc_seam_filter_implicit(const orc_grid* g, const orc_params* p, int32_t flux, int32_t order,
                                 double dt, const double* qm1, const double* qm2, double* v,
                                 const uint8_t* mask_S, uint8_t* kept_out, int32_t* sweeps_out) {
  Grid G(g);
  auto Fcell = [&](const double* state, int64_t n, double* F4) {
    implicit_Fk_cell(G, flux, order, dt, state, qm1, qm2, n, F4);
  };
  return seam_filter_impl(g, p, v, mask_S, kept_out, sweeps_out, Fcell);
}

}  // extern "C"
