// cell_stencil.h — S~ applied matrix-free from its entry formula, 3D:
//   (S~ f)_i = S~_ii f_i - sum over the interior faces k of cell i of w_k f_{nb(k)},
//   w_k = 1 / M~_kk, S~_ii = C~_ii + sum_{k in F(i)} w_k,
// from the cell-major weight arrays built by kernel_sparse.cu (cellw_kernel):
//   cw[0][i] = S~_ii, cw[1..3][i] = w of the cell's +x / +y / +z face (0 on the domain boundary
//   or an eliminated face), cw[4][X + n_x Y] = the -z face of a slab whose lower neighbour is a
//   ghost; a cell's -x / -y / -z weights are its neighbours' + weights.  Shared by the Chebyshev
//   step (solver.cu) and AMG's level-0 passes (amg.cu).  L2 numbering: e p^3 + a + p (b + p c).
#pragma once

#include "internal.h"

namespace hdiv {

struct CellGeo {
  long long n;                       // local cells (n_l2)
  long long nx, ny, nz;              // local subcell counts
  long long ghost_lo, ghost_hi;      // first ghost cell below / above the slab, -1 if none
  int NL[3];
  unsigned long long mx, my;         // ceil(2^64 / NL0), ceil(2^64 / NL1) (0 <-> divisor 1)
  const double* cw;
};

inline CellGeo make_cellgeo(const hdiv_ctx* h) {
  CellGeo g;
  g.n = h->nl2;
  g.nx = h->n[0]; g.ny = h->n[1]; g.nz = h->n[2];
  const long long lplane = h->n[0] * h->n[1];
  g.ghost_lo = (h->rank > 0) ? h->nl2 : -1;
  g.ghost_hi = (h->rank < h->nranks - 1) ? h->nl2 + lplane : -1;
  for (int a = 0; a < 3; ++a) g.NL[a] = (int)h->NL[a];
  auto magic = [](unsigned long long D) { return D <= 1 ? 0ull : (~0ull) / D + 1ull; };
  g.mx = magic((unsigned long long)h->NL[0]);
  g.my = magic((unsigned long long)h->NL[1]);
  g.cw = h->d_cw;
  return g;
}

__device__ __forceinline__ unsigned cell_fdiv(unsigned v, unsigned long long m) {
  return m ? (unsigned)__umul64hi((unsigned long long)v, m) : v;
}

// sum_j S~_ij f(j) for row i; GHOSTS: couplings to the ghost layers of the neighbouring slabs
// (false: dropped, AMG's block-Jacobi per slab, reading A9c).  Off-diagonals accumulate in the
// face order -x, +x, -y, +y, -z, +z; the diagonal term last.
template <int P, bool GHOSTS, class F>
__device__ __forceinline__ double cell_apply(const CellGeo& g, long long i, F f) {
  constexpr int PD = P * P * P;
  const long long rowx = (long long)g.NL[0] * PD;
  const long long lay = rowx * g.NL[1];
  const double* __restrict__ cw = g.cw;
  const double* __restrict__ cwx = cw + g.n;
  const double* __restrict__ cwy = cw + 2 * g.n;
  const double* __restrict__ cwz = cw + 3 * g.n;
  const unsigned e = (unsigned)(i / PD);
  const int il = (int)(i - (long long)e * PD);
  const int a = il % P, b = (il / P) % P, c = il / (P * P);
  const unsigned t = cell_fdiv(e, g.mx);
  const int ex = (int)(e - t * (unsigned)g.NL[0]);
  const unsigned u = cell_fdiv(t, g.my);
  const int ey = (int)(t - u * (unsigned)g.NL[1]);
  const int ez = (int)u;
  const long long X = (long long)ex * P + a, Y = (long long)ey * P + b, Z = (long long)ez * P + c;
  double sd = 0.0;
  if (X > 0) { const long long j = a > 0 ? i - 1 : i - PD + (P - 1); sd = fma(cwx[j], f(j), sd); }
  if (X + 1 < g.nx) sd = fma(cwx[i], f(a < P - 1 ? i + 1 : i + PD - (P - 1)), sd);
  if (Y > 0) { const long long j = b > 0 ? i - P : i - rowx + P * (P - 1); sd = fma(cwy[j], f(j), sd); }
  if (Y + 1 < g.ny) sd = fma(cwy[i], f(b < P - 1 ? i + P : i + rowx - P * (P - 1)), sd);
  if (Z > 0) {
    const long long j = c > 0 ? i - P * P : i - lay + P * P * (P - 1);
    sd = fma(cwz[j], f(j), sd);
  } else if (GHOSTS && g.ghost_lo >= 0) {
    sd = fma(cw[4 * g.n + X + g.nx * Y], f(g.ghost_lo + X + g.nx * Y), sd);
  }
  if (Z + 1 < g.nz) sd = fma(cwz[i], f(c < P - 1 ? i + P * P : i + lay - P * P * (P - 1)), sd);
  else if (GHOSTS && g.ghost_hi >= 0) sd = fma(cwz[i], f(g.ghost_hi + X + g.nx * Y), sd);
  return cw[i] * f(i) - sd;
}

// AMG accessor (amg.cu's A.dot interface): level 0 through the cell stencil, slab-local
template <int P>
struct CellA {
  CellGeo g;
  template <class F>
  __device__ __forceinline__ double dot(long long i, F f) const { return cell_apply<P, false>(g, i, f); }
};

}  // namespace hdiv
