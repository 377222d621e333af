// common.hpp -- internal helpers of the CPU oracle (TEST INFRASTRUCTURE ONLY; see oracle.h).
#pragma once
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>
#include "oracle.h"

namespace orc {

// Neumaier-compensated running sum: every reduction over more than a few terms
// in the oracle goes through it (SURVEY §8(c) "Reductions"), so the oracle is at
// least as accurate as any ordering the GPU may use.
struct CSum {
  double s = 0.0, c = 0.0;
  inline void add(double x) {
    double t = s + x;
    if (std::fabs(s) >= std::fabs(x)) c += (s - t) + x;
    else c += (x - t) + s;
    s = t;
  }
  inline double value() const { return s + c; }
};

inline double dot(const double* a, const double* b, int64_t n) {
  CSum s;
  for (int64_t i = 0; i < n; ++i) s.add(a[i] * b[i]);
  return s.value();
}

struct Grid {
  int dim, nx, ny, c, bc, recon;
  int64_t N, D;
  double dx, dy, gamma, cfl;
  explicit Grid(const orc_grid* g)
      : dim(g->dim), nx(g->nx), ny(g->dim == 1 ? 1 : g->ny), c(g->dim + 2), bc(g->bc),
        recon(g->recon), gamma(g->gamma), cfl(g->cfl) {
    N = (int64_t)nx * ny;
    D = (int64_t)c * N;
    dx = (g->x1 - g->x0) / nx;
    dy = (dim == 2) ? (g->y1 - g->y0) / ny : 1.0;
  }
  // ghost handling (O3): transmissive = nearest interior cell (zeroth order,
  // two layers), periodic = wrap.
  inline int ix(int i) const {
    if (bc == 1) return ((i % nx) + nx) % nx;
    return i < 0 ? 0 : (i >= nx ? nx - 1 : i);
  }
  inline int iy(int j) const {
    if (bc == 1) return ((j % ny) + ny) % ny;
    return j < 0 ? 0 : (j >= ny ? ny - 1 : j);
  }
};

// dense helpers (column-major)
void householder_qr(double* A, int64_t m, int n, std::vector<std::vector<double>>& V);
void apply_q(const std::vector<std::vector<double>>& V, int64_t m, double* x);
void apply_qt(const std::vector<std::vector<double>>& V, int64_t m, double* x);
void jacobi_svd_square(double* B, int64_t m, int n, double* V, double* S);

// implicit HDM function F_k(q) at cell n (implicit.cpp; NEXT-4); returns nonzero
// when a Roe average was not admissible
int implicit_Fk_cell(const Grid& G, int flux, int order, double dt, const double* q, const double* qm1,
                     const double* qm2, int64_t n, double* F);

}  // namespace orc
