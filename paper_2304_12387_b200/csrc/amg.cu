// amg.cu — NEXT-1: one algebraic-multigrid V-cycle as S^-1 (the paper's Schur preconditioner,
// P:889-891 "one V-cycle of AMG"; l1-Jacobi smoothing P:900-901; Galerkin coarse
// operators).  The paper leaves coarsening, interpolation, sweeps and coarse solve open
// (reading A9); this build fixes them as reading A9b, identical in oracle/amg.py:
//
//   aggregates   3 x 3 (x 3) blocks of the structured subcell grid (deterministic)
//   P            (I - omega D^-1 A) P_tent,  omega = 4 / (3 max_i sum_j |a_ij| / a_ii)
//   A_{l+1}      P^T A_l P   (27-point / 9-point on every coarse level)
//   smoother     nu sweeps of l1-Jacobi before and after the coarse correction
//   coarsest     <= max_coarse unknowns: dense inverse (host Gauss-Jordan at setup)
//
// B200 layout: level 0 is S~ itself (SELL-32 copy for the SpMVs, its 7-point face form for the
// setup); levels >= 1 are structured stencils stored as [3^d][n] (SoA: coalesced per offset),
// lexicographic x-fastest numbering.  Multi-rank (slabs): every rank builds the hierarchy of its
// own diagonal block of S~ (slab-local aggregates, ghost couplings dropped: the face terms of the
// interface stay on the diagonal) and the V-cycles act independently — the block-Jacobi of the
// per-slab V-cycles (reading A9c), no communication inside a V-cycle; in 3D, S^-1 wraps them (or
// their A9d polynomial) once in the balancing form with a replicated global coarse operator
// A0 = R S~ R^T over blocks of ceil(N/8) elements (reading A9e, amg_global_apply below).
// P and P^T are never stored: P e = inject(e) - omega D^-1 A
// inject(e) and P^T r = aggregate-sum(r - omega A D^-1 r) reuse the level's SpMV.  The Galerkin
// product is formed matrix-free per coarse row (one CTA: phi_I on the 5^d box, A phi_I on 7^d,
// (I - omega A D^-1) A phi_I on 9^d, summed per neighbouring aggregate), no SpGEMM.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "cell_stencil.h"
#include "internal.h"

namespace hdiv {

struct AmgLevel {
  int dim = 3;
  long long d[3] = {1, 1, 1};   // grid extents
  long long n = 0;
  double* st = nullptr;         // [3^dim][n] stencil (levels >= 1)
  double* dinv = nullptr;       // 1 / a_ii
  double* dl1inv = nullptr;     // 1 / sum_j |a_ij|
  double omega = 0.0;           // prolongator smoothing weight (levels with a coarser one)
  double *xa = nullptr, *xb = nullptr, *r = nullptr, *sv = nullptr;
  double *b = nullptr, *e = nullptr;   // levels >= 1: restricted rhs, coarse correction
};

// reading A9e: the balancing global coarse correction across slabs (3D)
struct GlobalCoarse {
  long long n0 = 0;          // global aggregates
  int g[3] = {1, 1, 1};      // aggregate extents (global subcells)
  int cd[3] = {1, 1, 1};     // aggregate grid
  long long z0c = 0;         // the slab's first global subcell layer
  double* a0inv = nullptr;   // [n0][n0] (A0 = R S~ R^T, pinned for the pure-Neumann S~)
  double* part = nullptr;    // [n0] this rank's aggregate sums
  double* glob = nullptr;    // [P][n0] all ranks' sums
  double* c = nullptr;       // [n0] summed in rank order
  double* e0 = nullptr;      // [n0]
  double* e1 = nullptr;      // [n0]
  double* rp = nullptr;      // [n_l2] r - S~ R^T e0, later S~ w
  double* w = nullptr;       // [n_l2 + 2 plane] the block-Jacobi V-cycles (ghost space)
  double* u = nullptr;       // [n_l2 + 2 plane] R^T e0 (ghost space)
  double* es = nullptr;      // [E] per-element sums
  int32_t* eagg = nullptr;   // [E] element -> aggregate
};

struct AmgHier {
  GlobalCoarse* gc = nullptr;
  std::vector<AmgLevel> L;
  int32_t* agg0 = nullptr;      // level-0 row -> level-1 aggregate
  double* cinv = nullptr;       // dense inverse of the coarsest operator [nc][nc]
  long long nc = 0;
  int nu = 2;
  double* red = nullptr;        // reduction scratch
};

namespace {

constexpr int ANT = 256;
constexpr int ABLK = 148 * 8;

// ---- level-0 operator: S~ in its 7/5-point face form, L2 element-major rows ----
struct Op0 {
  long long n[3], off[3], NL[3];
  int p, dim;
  int ess;               // eliminated essential sides (NEXT-3): their faces are not in F(i)
  const double* mdiag;
  const double* ctil;
  __device__ __forceinline__ long long idx(long long X, long long Y, long long Z) const {
    long long e = (X / p) + NL[0] * ((Y / p) + NL[1] * (Z / p));
    long long a = X % p, b = Y % p, c = Z % p;
    if (dim == 2) return e * p * p + a + p * b;
    return e * p * p * p + a + p * (b + p * c);
  }
  __device__ __forceinline__ bool in(long long X, long long Y, long long Z) const {
    return X >= 0 && Y >= 0 && Z >= 0 && X < n[0] && Y < n[1] && (dim == 2 ? Z == 0 : Z < n[2]);
  }
  __device__ __forceinline__ void coords(long long r, long long* X, long long* Y,
                                         long long* Z) const {
    const long long pd = (dim == 2) ? (long long)p * p : (long long)p * p * p;
    const long long e = r / pd, il = r % pd;
    const long long ex = e % NL[0], ey = (e / NL[0]) % NL[1];
    const long long ez = (dim == 3) ? e / (NL[0] * NL[1]) : 0;
    *X = ex * p + il % p;
    *Y = ey * p + (il / p) % p;
    *Z = (dim == 3) ? ez * p + il / (p * p) : 0;
  }
  // a[k], k = (dx+1) + 3(dy+1) (+ 9(dz+1)): the row of S~ at cell (X,Y,Z); zeros elsewhere
  __device__ __forceinline__ void row(long long X, long long Y, long long Z, double* a) const {
    const int NS = (dim == 3) ? 27 : 9;
    for (int k = 0; k < NS; ++k) a[k] = 0.0;
    const int C = (dim == 3) ? 13 : 4;
    long long f[6];
    int nf;
    if (dim == 3) {
      f[0] = off[0] + X + (n[0] + 1) * (Y + n[1] * Z);
      f[1] = f[0] + 1;
      f[2] = off[1] + X + n[0] * (Y + (n[1] + 1) * Z);
      f[3] = f[2] + n[0];
      f[4] = off[2] + X + n[0] * (Y + n[1] * Z);
      f[5] = f[4] + n[0] * n[1];
      nf = 6;
    } else {
      f[0] = off[0] + X + (n[0] + 1) * Y;
      f[1] = f[0] + 1;
      f[2] = off[1] + X + n[0] * Y;
      f[3] = f[2] + n[0];
      nf = 4;
    }
    double d = ctil[idx(X, Y, Z)];
    const int step[3] = {1, 3, 9};
    const long long ext[3] = {n[0], n[1], n[2]};
    const long long crd[3] = {X, Y, Z};
    for (int k = 0; k < nf; ++k) {
      const int ax = k >> 1;
      const bool up = k & 1;
      const bool has = up ? (crd[ax] + 1 < ext[ax]) : (crd[ax] > 0);
      if (!has && ((ess >> k) & 1)) continue;   // k = 2 axis + side: the ess bit layout
      const double w = 1.0 / mdiag[f[k]];
      d += w;
      if (has) a[C + (up ? step[ax] : -step[ax])] = -w;
    }
    a[C] = d;
  }
};

// ---- level >= 1: stored structured stencil ----
struct OpS {
  long long d[3], n;
  int dim;
  const double* st;
  __device__ __forceinline__ long long idx(long long X, long long Y, long long Z) const {
    return X + d[0] * (Y + d[1] * Z);
  }
  __device__ __forceinline__ bool in(long long X, long long Y, long long Z) const {
    return X >= 0 && Y >= 0 && Z >= 0 && X < d[0] && Y < d[1] && Z < d[2];
  }
  __device__ __forceinline__ void coords(long long r, long long* X, long long* Y,
                                         long long* Z) const {
    *X = r % d[0];
    *Y = (r / d[0]) % d[1];
    *Z = r / (d[0] * d[1]);
  }
  __device__ __forceinline__ void row(long long X, long long Y, long long Z, double* a) const {
    const int NS = (dim == 3) ? 27 : 9;
    const long long i = idx(X, Y, Z);
    for (int k = 0; k < NS; ++k) a[k] = st[k * n + i];
  }
};

// stencil slot k -> offset: k = (dx+1) + 3(dy+1) (+ 9(dz+1) in 3D)
template <int DIM>
__device__ __forceinline__ void off_of(int k, int* dx, int* dy, int* dz) {
  *dx = k % 3 - 1;
  *dy = (k / 3) % 3 - 1;
  *dz = (DIM == 3) ? k / 9 - 1 : 0;
}

// diag / l1 / Gershgorin ratio per row; part[block] = max ratio of the block
template <class Op>
__global__ void __launch_bounds__(ANT) level_diag_kernel(Op A, long long nrow, double* dinv,
                                                        double* dl1inv, double* part) {
  __shared__ double red[ANT / 32];
  double mx = 0.0;
  const int NS = (A.dim == 3) ? 27 : 9;
  for (long long r = blockIdx.x * (long long)ANT + threadIdx.x; r < nrow;
       r += (long long)gridDim.x * ANT) {
    long long X, Y, Z;
    A.coords(r, &X, &Y, &Z);
    double a[27];
    A.row(X, Y, Z, a);
    double l1 = 0.0;
    for (int k = 0; k < NS; ++k) l1 += fabs(a[k]);
    const double dg = a[NS / 2];
    dinv[r] = 1.0 / dg;
    dl1inv[r] = 1.0 / l1;
    mx = fmax(mx, l1 / dg);
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int w = 0; w < ANT / 32; ++w) m = fmax(m, red[w]);
    part[blockIdx.x] = m;
  }
}

// Galerkin row I of A_c = P^T A P (one CTA per coarse point; DIM 2 or 3)
template <int DIM, class Op>
__global__ void __launch_bounds__(128) rap_kernel(Op A, const double* __restrict__ dinv,
                                                  long long cd0, long long cd1, long long cd2,
                                                  double omega, double* __restrict__ stc) {
  constexpr int B5 = (DIM == 3) ? 125 : 25, B7 = (DIM == 3) ? 343 : 49, B9 = (DIM == 3) ? 729 : 81;
  constexpr int NS = (DIM == 3) ? 27 : 9;
  __shared__ double phi[B5], psi[B7], chi[B7], xi[B9];
  const long long nc = cd0 * cd1 * cd2;
  const long long I = blockIdx.x;
  const long long IX = I % cd0, IY = (I / cd0) % cd1, IZ = (DIM == 3) ? I / (cd0 * cd1) : 0;
  const long long ox = 3 * IX, oy = 3 * IY, oz = 3 * IZ;   // aggregate origin (fine coords)
  auto inagg = [&](long long X, long long Y, long long Z) {
    return X >= ox && X < ox + 3 && Y >= oy && Y < oy + 3 && (DIM == 2 || (Z >= oz && Z < oz + 3));
  };
  auto box = [&](int t, int w, long long lo, long long* X, long long* Y, long long* Z) {
    *X = ox + lo + t % w;
    *Y = oy + lo + (t / w) % w;
    *Z = (DIM == 3) ? oz + lo + t / (w * w) : 0;
  };
  auto bidx = [&](long long X, long long Y, long long Z, int w, long long lo) -> int {
    const long long x = X - ox - lo, y = Y - oy - lo, z = (DIM == 3) ? Z - oz - lo : 0;
    if (x < 0 || y < 0 || z < 0 || x >= w || y >= w || z >= w) return -1;
    return (int)(x + w * (y + w * z));
  };
  double a[27];
  // phi_I = (I - omega D^-1 A) 1_agg(I) on the 5^d box [o-1, o+3]
  for (int t = threadIdx.x; t < B5; t += blockDim.x) {
    long long X, Y, Z;
    box(t, 5, -1, &X, &Y, &Z);
    double v = 0.0;
    if (A.in(X, Y, Z)) {
      A.row(X, Y, Z, a);
      double sacc = 0.0;
      for (int k = 0; k < NS; ++k) {
        int dx, dy, dz;
        off_of<DIM>(k, &dx, &dy, &dz);
        if (inagg(X + dx, Y + dy, Z + dz) && A.in(X + dx, Y + dy, Z + dz)) sacc += a[k];
      }
      v = (inagg(X, Y, Z) ? 1.0 : 0.0) - omega * dinv[A.idx(X, Y, Z)] * sacc;
    }
    phi[t] = v;
  }
  __syncthreads();
  // psi = A phi on the 7^d box [o-2, o+4]; chi = D^-1 psi
  for (int t = threadIdx.x; t < B7; t += blockDim.x) {
    long long X, Y, Z;
    box(t, 7, -2, &X, &Y, &Z);
    double v = 0.0, c = 0.0;
    if (A.in(X, Y, Z)) {
      A.row(X, Y, Z, a);
      for (int k = 0; k < NS; ++k) {
        int dx, dy, dz;
        off_of<DIM>(k, &dx, &dy, &dz);
        const int q = bidx(X + dx, Y + dy, Z + dz, 5, -1);
        if (q >= 0 && a[k] != 0.0) v += a[k] * phi[q];
      }
      c = dinv[A.idx(X, Y, Z)] * v;
    }
    psi[t] = v;
    chi[t] = c;
  }
  __syncthreads();
  // xi = psi - omega A chi on the 9^d box [o-3, o+5]
  for (int t = threadIdx.x; t < B9; t += blockDim.x) {
    long long X, Y, Z;
    box(t, 9, -3, &X, &Y, &Z);
    double v = 0.0;
    if (A.in(X, Y, Z)) {
      A.row(X, Y, Z, a);
      double ac = 0.0;
      for (int k = 0; k < NS; ++k) {
        int dx, dy, dz;
        off_of<DIM>(k, &dx, &dy, &dz);
        const int q = bidx(X + dx, Y + dy, Z + dz, 7, -2);
        if (q >= 0 && a[k] != 0.0) ac += a[k] * chi[q];
      }
      const int q0 = bidx(X, Y, Z, 7, -2);
      v = (q0 >= 0 ? psi[q0] : 0.0) - omega * ac;
    }
    xi[t] = v;
  }
  __syncthreads();
  // A_c[I][J] = sum of xi over aggregate J = I + delta
  for (int k = threadIdx.x; k < NS; k += blockDim.x) {
    int dx, dy, dz;
    off_of<DIM>(k, &dx, &dy, &dz);
    const long long JX = IX + dx, JY = IY + dy, JZ = IZ + dz;
    double v = 0.0;
    if (JX >= 0 && JY >= 0 && JZ >= 0 && JX < cd0 && JY < cd1 && JZ < cd2) {
      for (int cz = 0; cz < (DIM == 3 ? 3 : 1); ++cz)
        for (int cy = 0; cy < 3; ++cy)
          for (int cx = 0; cx < 3; ++cx) {
            const long long X = 3 * JX + cx, Y = 3 * JY + cy, Z = (DIM == 3) ? 3 * JZ + cz : 0;
            if (!A.in(X, Y, Z)) continue;
            const int q = bidx(X, Y, Z, 9, -3);
            v += xi[q];
          }
    }
    stc[k * nc + I] = v;
  }
}

// level-0 row -> aggregate (lexicographic coarse numbering)
__global__ void agg0_kernel(Op0 A, long long cd0, long long cd1, int32_t* agg, long long nrow) {
  long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (r >= nrow) return;
  const long long pd = (A.dim == 2) ? (long long)A.p * A.p : (long long)A.p * A.p * A.p;
  const long long e = r / pd, il = r % pd;
  const long long ex = e % A.NL[0], ey = (e / A.NL[0]) % A.NL[1];
  const long long ez = (A.dim == 3) ? e / (A.NL[0] * A.NL[1]) : 0;
  const long long X = ex * A.p + il % A.p, Y = ey * A.p + (il / A.p) % A.p;
  const long long Z = (A.dim == 3) ? ez * A.p + il / (A.p * A.p) : 0;
  (void)X;
  agg[r] = (int32_t)(X / 3 + cd0 * (Y / 3 + cd1 * (Z / 3)));
}

// ---- V-cycle kernels.  SpMV access: level 0 through SELL-32 (width W), levels >= 1 stencil ----
struct SellA {
  const int32_t* col;
  const double* val;
  int W;
  int nloc;   // local rows: slab ghost columns (>= nloc) are dropped — multi-rank AMG is the
              // block-Jacobi of the per-slab V-cycles (reading A9c)
  template <class F>
  __device__ __forceinline__ double dot(long long i, F f) const {
    const long long base = (i >> 5) * (32LL * W) + (i & 31);
    double s = 0.0;
    for (int k = 0; k < W; ++k) {
      const int c = col[base + 32 * k];
      if (c < nloc) s = fma(val[base + 32 * k], f(c), s);
    }
    return s;
  }
};

struct StA {
  long long d[3], n;
  int dim;
  const double* st;
  int id[3];   // 32-bit extents: coarse levels have < 2^31 rows (row coordinates in 32-bit)
  // sum_k st[k][i] f(j_k, x_k, y_k, z_k) over the in-range 3^d neighbours (x_k, y_k, z_k) of row i
  template <class F>
  __device__ __forceinline__ double dot_xyz(long long i, F f) const {
    const int ii = (int)i;
    const int X = ii % id[0], r = ii / id[0], Y = r % id[1], Z = r / id[1];
    const int NS = (dim == 3) ? 27 : 9;
    double s = 0.0;
#pragma unroll 9
    for (int k = 0; k < NS; ++k) {
      const int dx = k % 3 - 1, dy = (k / 3) % 3 - 1, dz = (dim == 3) ? k / 9 - 1 : 0;
      const int x = X + dx, y = Y + dy, z = Z + dz;
      if (x < 0 || y < 0 || z < 0 || x >= id[0] || y >= id[1] || z >= id[2]) continue;
      s = fma(st[k * n + i], f(ii + dx + id[0] * (dy + id[1] * dz), x, y, z), s);
    }
    return s;
  }
  template <class F>
  __device__ __forceinline__ double dot(long long i, F f) const {
    return dot_xyz(i, [&](int j, int, int, int) { return f((long long)j); });
  }
  __device__ __forceinline__ long long agg(long long j, long long cd0, long long cd1) const {
    const long long X = j % d[0], Y = (j / d[0]) % d[1], Z = j / (d[0] * d[1]);
    return X / 3 + cd0 * (Y / 3 + cd1 * (Z / 3));
  }
};

// level-0 sweeps: 8 resident 256-thread CTAs per SM (the reduction / sweep grid is 148 x 8: one
// wave; at 36-48 registers only 5-7 fit and the last CTAs ran as a second, mostly empty wave)
#ifndef AMG_MINB
#define AMG_MINB 8
#endif
#define AMG_LOOP(n) \
  for (long long i = blockIdx.x * (long long)ANT + threadIdx.x; i < (n); i += (long long)gridDim.x * ANT)

// the last level-0 post-smoothing sweep with the MINRES partial <x_out, b> (b = the V-cycle's
// right-hand side = v_q): saves the separate dot pass; part has gridDim.x entries
template <class Acc>
__global__ void __launch_bounds__(ANT, AMG_MINB) jacobi_dot_kernel(Acc A, long long n,
                                                         const double* __restrict__ b,
                                                         const double* __restrict__ xin,
                                                         double* __restrict__ xout,
                                                         const double* __restrict__ dl1inv,
                                                         double* __restrict__ part,
                                                         const int* __restrict__ done) {
  if (done && *done) return;
  __shared__ double red[ANT / 32];
  double sdot = 0.0;
  AMG_LOOP(n) {
    const double ax = A.dot(i, [&](long long j) { return xin[j]; });
    const double bi = b[i];
    const double xo = xin[i] + dl1inv[i] * (bi - ax);
    xout[i] = xo;
    sdot = fma(xo, bi, sdot);
  }
  for (int o = 16; o > 0; o >>= 1) sdot += __shfl_down_sync(0xffffffffu, sdot, o);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  if (l == 0) red[w] = sdot;
  __syncthreads();
  if (threadIdx.x < 32) {
    double r = (l < ANT / 32) ? red[l] : 0.0;
    for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
    if (l == 0) part[blockIdx.x] = r;
  }
}

// x_out = x_in + Dl1^-1 (b - A x_in); x_in = nullptr means x_in = Dl1^-1 b (first sweep from 0)
template <class Acc>
__global__ void __launch_bounds__(ANT, AMG_MINB) jacobi_kernel(Acc A, long long n, const double* __restrict__ b,
                                                     const double* __restrict__ xin,
                                                     double* __restrict__ xout,
                                                     const double* __restrict__ dl1inv,
                                                     const int* __restrict__ done) {
  if (done && *done) return;
  AMG_LOOP(n) {
    double ax, xi;
    if (xin) {
      ax = A.dot(i, [&](long long j) { return xin[j]; });
      xi = xin[i];
    } else {
      ax = A.dot(i, [&](long long j) { return dl1inv[j] * b[j]; });
      xi = dl1inv[i] * b[i];
    }
    xout[i] = xi + dl1inv[i] * (b[i] - ax);
  }
}

__global__ void __launch_bounds__(ANT) scale_kernel(long long n, const double* __restrict__ b,
                                                    const double* __restrict__ dl1inv,
                                                    double* __restrict__ x,
                                                    const int* __restrict__ done) {
  if (done && *done) return;
  AMG_LOOP(n) x[i] = dl1inv[i] * b[i];
}

// s = r - omega A D^-1 r with r = b - A x  (computed in two passes: r then s)
// r = b - A x and t = D^-1 r (so the next pass gathers one vector, not two)
template <class Acc>
__global__ void __launch_bounds__(ANT, AMG_MINB) resid_kernel(Acc A, long long n, const double* __restrict__ b,
                                                    const double* __restrict__ x,
                                                    double* __restrict__ r,
                                                    const double* __restrict__ dinv,
                                                    double* __restrict__ t,
                                                    const int* __restrict__ done) {
  if (done && *done) return;
  AMG_LOOP(n) {
    const double ri = b[i] - A.dot(i, [&](long long j) { return x[j]; });
    r[i] = ri;
    t[i] = dinv[i] * ri;
  }
}

// s = r - omega A t, t = D^-1 r
template <class Acc>
__global__ void __launch_bounds__(ANT, AMG_MINB) smooth_r_kernel(Acc A, long long n,
                                                       const double* __restrict__ r,
                                                       const double* __restrict__ t, double omega,
                                                       double* __restrict__ s,
                                                       const int* __restrict__ done) {
  if (done && *done) return;
  AMG_LOOP(n) s[i] = r[i] - omega * A.dot(i, [&](long long j) { return t[j]; });
}

// b_c[I] = sum over aggregate I of s (level 0: element-major fine rows); the 3 x 3 (x 3)
// subcells' element / local coordinates per axis once, 32-bit (level 0 has < 2^31 rows), then
// the 27 (9) row indices by adds; summation order x fastest as before
__global__ void __launch_bounds__(ANT) aggsum0_kernel(Op0 A, long long cd0, long long cd1,
                                                      long long nc, const double* __restrict__ s,
                                                      double* __restrict__ bc,
                                                      const int* __restrict__ done) {
  if (done && *done) return;
  const int p = A.p;
  const int pd = (A.dim == 2) ? p * p : p * p * p;
  AMG_LOOP(nc) {
    const long long IX = i % cd0, IY = (i / cd0) % cd1, IZ = (A.dim == 3) ? i / (cd0 * cd1) : 0;
    int ox[3], oy[3], oz[3];   // element offset * pd + local offset per coordinate
    bool vx[3], vy[3], vz[3];
    for (int k = 0; k < 3; ++k) {
      const int X = (int)(3 * IX) + k, Y = (int)(3 * IY) + k, Z = (int)(3 * IZ) + k;
      vx[k] = X < A.n[0];
      vy[k] = Y < A.n[1];
      vz[k] = (A.dim == 3) ? (Z < A.n[2]) : (k == 0);
      const int ex = X / p, ey = Y / p, ez = (A.dim == 3) ? Z / p : 0;
      ox[k] = ex * pd + (X - ex * p);
      oy[k] = ey * (int)A.NL[0] * pd + p * (Y - ey * p);
      oz[k] = (A.dim == 3) ? ez * (int)(A.NL[0] * A.NL[1]) * pd + p * p * (Z - ez * p) : 0;
    }
    double v = 0.0;
    for (int cz = 0; cz < (A.dim == 3 ? 3 : 1); ++cz) {
      if (!vz[cz]) continue;
      for (int cy = 0; cy < 3; ++cy) {
        if (!vy[cy]) continue;
        for (int cx = 0; cx < 3; ++cx)
          if (vx[cx]) v += s[(long long)ox[cx] + oy[cy] + oz[cz]];
      }
    }
    bc[i] = v;
  }
}

__global__ void __launch_bounds__(ANT) aggsumS_kernel(long long d0, long long d1, long long d2,
                                                      long long cd0, long long cd1, long long nc,
                                                      int dim, const double* __restrict__ s,
                                                      double* __restrict__ bc,
                                                      const int* __restrict__ done) {
  if (done && *done) return;
  AMG_LOOP(nc) {
    const long long IX = i % cd0, IY = (i / cd0) % cd1, IZ = (dim == 3) ? i / (cd0 * cd1) : 0;
    double v = 0.0;
    for (int cz = 0; cz < (dim == 3 ? 3 : 1); ++cz)
      for (int cy = 0; cy < 3; ++cy)
        for (int cx = 0; cx < 3; ++cx) {
          const long long X = 3 * IX + cx, Y = 3 * IY + cy, Z = 3 * IZ + cz;
          if (X < d0 && Y < d1 && Z < d2) v += s[X + d0 * (Y + d1 * Z)];
        }
    bc[i] = v;
  }
}

// x_out = x + e_f - omega D^-1 A e_f,  e_f(j) = e_c[agg(j)]
template <class Acc, class Agg>
__global__ void __launch_bounds__(ANT, AMG_MINB) prolong_kernel(Acc A, Agg agg, long long n,
                                                      const double* __restrict__ x,
                                                      const double* __restrict__ ec,
                                                      const double* __restrict__ dinv, double omega,
                                                      double* __restrict__ xout,
                                                      const int* __restrict__ done) {
  if (done && *done) return;
  AMG_LOOP(n) {
    const double ae = A.dot(i, [&](long long j) { return ec[agg(j)]; });
    xout[i] = x[i] + ec[agg(i)] - omega * dinv[i] * ae;
  }
}

// stencil levels: the aggregate of a neighbour from its coordinates (no index division)
__global__ void __launch_bounds__(ANT) prolong_st_kernel(StA A, long long cd0, long long cd1,
                                                         long long n, const double* __restrict__ x,
                                                         const double* __restrict__ ec,
                                                         const double* __restrict__ dinv,
                                                         double omega, double* __restrict__ xout,
                                                         const int* __restrict__ done) {
  if (done && *done) return;
  const int c0 = (int)cd0, c1 = (int)cd1;
  AMG_LOOP(n) {
    const double ae = A.dot_xyz(i, [&](int, int x, int y, int z) {
      return ec[x / 3 + c0 * (y / 3 + c1 * (z / 3))];
    });
    const int ii = (int)i;
    const int X = ii % A.id[0], r = ii / A.id[0], Y = r % A.id[1], Z = r / A.id[1];
    xout[i] = x[i] + ec[X / 3 + c0 * (Y / 3 + c1 * (Z / 3))] - omega * dinv[i] * ae;
  }
}

struct Agg0 {
  const int32_t* a;
  __device__ __forceinline__ long long operator()(long long j) const { return a[j]; }
};

// coarsest: x = A^-1 b (dense): one warp per row, lanes over the columns (coalesced row reads,
// fixed-order lane sums -> deterministic); many CTAs so the inverse streams from all SMs
__global__ void __launch_bounds__(ANT) coarse_kernel(const double* __restrict__ cinv, long long nc,
                                                     const double* __restrict__ b,
                                                     double* __restrict__ x,
                                                     const int* __restrict__ done) {
  if (done && *done) return;
  const long long w = blockIdx.x * (long long)(ANT / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (w >= nc) return;
  const double* row = cinv + w * nc;
  double s = 0.0;
  for (long long j = lane; j < nc; j += 32) s = fma(row[j], b[j], s);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) x[w] = s;
}

inline unsigned nbk(long long n) {
  long long b = (n + ANT - 1) / ANT;
  return (unsigned)std::max(1LL, std::min<long long>(b, ABLK));
}

Op0 make_op0(const hdiv_ctx* h) {
  Op0 o;
  for (int a = 0; a < 3; ++a) { o.n[a] = h->n[a]; o.off[a] = h->off[a]; o.NL[a] = h->NL[a]; }
  if (h->dim == 2) o.n[2] = 1;
  o.p = h->p;
  o.dim = h->dim;
  o.ess = h->ess;
  o.mdiag = h->d_mdiag;
  o.ctil = h->d_ctil;
  return o;
}

OpS make_ops(const AmgLevel& L) {
  OpS o;
  for (int a = 0; a < 3; ++a) o.d[a] = L.d[a];
  o.n = L.n;
  o.dim = L.dim;
  o.st = L.st;
  return o;
}

StA make_sta(const AmgLevel& L) {
  StA o;
  for (int a = 0; a < 3; ++a) o.id[a] = (int)L.d[a];
  for (int a = 0; a < 3; ++a) o.d[a] = L.d[a];
  o.n = L.n;
  o.dim = L.dim;
  o.st = L.st;
  return o;
}

// Gauss-Jordan inverse with partial pivoting (host, coarsest level only)
bool invert_dense(std::vector<double>& A, long long n) {
  std::vector<double> Inv(n * n, 0.0);
  for (long long i = 0; i < n; ++i) Inv[i * n + i] = 1.0;
  for (long long c = 0; c < n; ++c) {
    long long piv = c;
    for (long long r = c + 1; r < n; ++r)
      if (std::fabs(A[r * n + c]) > std::fabs(A[piv * n + c])) piv = r;
    if (A[piv * n + c] == 0.0) return false;
    if (piv != c)
      for (long long j = 0; j < n; ++j) {
        std::swap(A[c * n + j], A[piv * n + j]);
        std::swap(Inv[c * n + j], Inv[piv * n + j]);
      }
    const double d = A[c * n + c];
    for (long long j = 0; j < n; ++j) { A[c * n + j] /= d; Inv[c * n + j] /= d; }
    for (long long r = 0; r < n; ++r) {
      if (r == c) continue;
      const double f = A[r * n + c];
      if (f == 0.0) continue;
      for (long long j = 0; j < n; ++j) { A[r * n + j] -= f * A[c * n + j]; Inv[r * n + j] -= f * Inv[c * n + j]; }
    }
  }
  A.swap(Inv);
  return true;
}

}  // namespace

void amg_free(hdiv_ctx* h) {
  if (!h->amg) return;
  for (auto& L : h->amg->L) {
    cudaFree(L.st); cudaFree(L.dinv); cudaFree(L.dl1inv);
    cudaFree(L.xa); cudaFree(L.xb); cudaFree(L.r); cudaFree(L.sv); cudaFree(L.b); cudaFree(L.e);
  }
  if (GlobalCoarse* G = h->amg->gc) {
    cudaFree(G->a0inv); cudaFree(G->part); cudaFree(G->glob); cudaFree(G->c); cudaFree(G->e0);
    cudaFree(G->e1); cudaFree(G->rp); cudaFree(G->w); cudaFree(G->u); cudaFree(G->es); cudaFree(G->eagg);
    delete G;
  }
  cudaFree(h->amg->agg0);
  cudaFree(h->amg->cinv);
  cudaFree(h->amg->red);
  delete h->amg;
  h->amg = nullptr;
}

static hdiv_status gc_setup(hdiv_ctx* h, cudaStream_t s);

hdiv_status amg_setup(hdiv_ctx* h, cudaStream_t s) {
  auto* H = new AmgHier();
  h->amg = H;
  H->nu = h->opts.amg_sweeps;
  HDIV_CUDA_TRY(cudaMalloc(&H->red, sizeof(double) * ABLK));
  std::vector<double> part(ABLK);
  const int dim = h->dim;
  const int NS = (dim == 3) ? 27 : 9;
  // level 0
  {
    AmgLevel L;
    L.dim = dim;
    L.d[0] = h->n[0]; L.d[1] = h->n[1]; L.d[2] = (dim == 3) ? h->n[2] : 1;
    L.n = h->nl2;
    HDIV_CUDA_TRY(cudaMalloc(&L.dinv, sizeof(double) * L.n));
    HDIV_CUDA_TRY(cudaMalloc(&L.dl1inv, sizeof(double) * L.n));
    HDIV_CUDA_TRY(cudaMemsetAsync(H->red, 0, sizeof(double) * ABLK, s));
    level_diag_kernel<Op0><<<ABLK, ANT, 0, s>>>(make_op0(h), L.n, L.dinv, L.dl1inv, H->red);
    HDIV_CUDA_TRY(cudaGetLastError());
    HDIV_CUDA_TRY(cudaMemcpyAsync(part.data(), H->red, sizeof(double) * ABLK, cudaMemcpyDeviceToHost, s));
    HDIV_CUDA_TRY(cudaStreamSynchronize(s));
    double mx = 0.0;
    for (double v : part) mx = std::max(mx, v);
    L.omega = 4.0 / (3.0 * mx);
    H->L.push_back(L);
  }
  for (;;) {
    AmgLevel& F = H->L.back();
    long long cd[3] = {(F.d[0] + 2) / 3, (F.d[1] + 2) / 3, (dim == 3) ? (F.d[2] + 2) / 3 : 1};
    const bool same = cd[0] == F.d[0] && cd[1] == F.d[1] && cd[2] == F.d[2];
    if (F.n <= h->opts.amg_max_coarse || same || H->L.size() >= 25) break;
    AmgLevel Cl;
    Cl.dim = dim;
    for (int a = 0; a < 3; ++a) Cl.d[a] = cd[a];
    Cl.n = cd[0] * cd[1] * cd[2];
    HDIV_CUDA_TRY(cudaMalloc(&Cl.st, sizeof(double) * NS * Cl.n));
    const bool first = H->L.size() == 1;
    if (dim == 3) {
      if (first) rap_kernel<3, Op0><<<(unsigned)Cl.n, 128, 0, s>>>(make_op0(h), F.dinv, cd[0], cd[1], cd[2], F.omega, Cl.st);
      else rap_kernel<3, OpS><<<(unsigned)Cl.n, 128, 0, s>>>(make_ops(F), F.dinv, cd[0], cd[1], cd[2], F.omega, Cl.st);
    } else {
      if (first) rap_kernel<2, Op0><<<(unsigned)Cl.n, 128, 0, s>>>(make_op0(h), F.dinv, cd[0], cd[1], cd[2], F.omega, Cl.st);
      else rap_kernel<2, OpS><<<(unsigned)Cl.n, 128, 0, s>>>(make_ops(F), F.dinv, cd[0], cd[1], cd[2], F.omega, Cl.st);
    }
    HDIV_CUDA_TRY(cudaGetLastError());
    if (first) {
      HDIV_CUDA_TRY(cudaMalloc(&H->agg0, sizeof(int32_t) * F.n));
      agg0_kernel<<<(unsigned)((F.n + 255) / 256), 256, 0, s>>>(make_op0(h), cd[0], cd[1], H->agg0, F.n);
      HDIV_CUDA_TRY(cudaGetLastError());
    }
    HDIV_CUDA_TRY(cudaMalloc(&Cl.dinv, sizeof(double) * Cl.n));
    HDIV_CUDA_TRY(cudaMalloc(&Cl.dl1inv, sizeof(double) * Cl.n));
    HDIV_CUDA_TRY(cudaMemsetAsync(H->red, 0, sizeof(double) * ABLK, s));
    level_diag_kernel<OpS><<<ABLK, ANT, 0, s>>>(make_ops(Cl), Cl.n, Cl.dinv, Cl.dl1inv, H->red);
    HDIV_CUDA_TRY(cudaGetLastError());
    HDIV_CUDA_TRY(cudaMemcpyAsync(part.data(), H->red, sizeof(double) * ABLK, cudaMemcpyDeviceToHost, s));
    HDIV_CUDA_TRY(cudaStreamSynchronize(s));
    double mx = 0.0;
    for (double v : part) mx = std::max(mx, v);
    Cl.omega = 4.0 / (3.0 * mx);
    H->L.push_back(Cl);
  }
  // work vectors
  for (size_t l = 0; l < H->L.size(); ++l) {
    AmgLevel& L = H->L[l];
    const size_t b = sizeof(double) * L.n;
    HDIV_CUDA_TRY(cudaMalloc(&L.xa, b));
    HDIV_CUDA_TRY(cudaMalloc(&L.xb, b));
    HDIV_CUDA_TRY(cudaMalloc(&L.r, b));
    HDIV_CUDA_TRY(cudaMalloc(&L.sv, b));
    if (l > 0) {
      HDIV_CUDA_TRY(cudaMalloc(&L.b, b));
      HDIV_CUDA_TRY(cudaMalloc(&L.e, b));
    }
  }
  // coarsest dense inverse
  AmgLevel& Lc = H->L.back();
  const long long nc = Lc.n;
  if (nc > 8192) {
    set_error("AMG coarsest level too large for the dense solve (raise amg_max_coarse coverage)");
    return HDIV_ERR_UNSUPPORTED;
  }
  std::vector<double> Ad(nc * nc, 0.0);
  if (H->L.size() == 1) {   // the fine operator itself: from the CSR of S~
    std::vector<int64_t> rp(nc + 1);
    HDIV_CUDA_TRY(cudaMemcpyAsync(rp.data(), h->d_srow, sizeof(int64_t) * (nc + 1), cudaMemcpyDeviceToHost, s));
    HDIV_CUDA_TRY(cudaStreamSynchronize(s));
    std::vector<int32_t> col(rp[nc]);
    std::vector<double> val(rp[nc]);
    HDIV_CUDA_TRY(cudaMemcpyAsync(col.data(), h->d_scol, sizeof(int32_t) * rp[nc], cudaMemcpyDeviceToHost, s));
    HDIV_CUDA_TRY(cudaMemcpyAsync(val.data(), h->d_sval, sizeof(double) * rp[nc], cudaMemcpyDeviceToHost, s));
    HDIV_CUDA_TRY(cudaStreamSynchronize(s));
    for (long long i = 0; i < nc; ++i)
      for (int64_t t = rp[i]; t < rp[i + 1]; ++t)
        if (col[t] < nc) Ad[i * nc + col[t]] = val[t];   // slab ghost columns dropped (A9c)
  } else {
    std::vector<double> st(NS * nc);
    HDIV_CUDA_TRY(cudaMemcpyAsync(st.data(), Lc.st, sizeof(double) * NS * nc, cudaMemcpyDeviceToHost, s));
    HDIV_CUDA_TRY(cudaStreamSynchronize(s));
    for (long long i = 0; i < nc; ++i) {
      const long long X = i % Lc.d[0], Y = (i / Lc.d[0]) % Lc.d[1], Z = i / (Lc.d[0] * Lc.d[1]);
      for (int k = 0; k < NS; ++k) {
        const long long x = X + k % 3 - 1, y = Y + (k / 3) % 3 - 1;
        const long long z = Z + ((dim == 3) ? k / 9 - 1 : 0);
        if (x < 0 || y < 0 || z < 0 || x >= Lc.d[0] || y >= Lc.d[1] || z >= Lc.d[2]) continue;
        Ad[i * nc + (x + Lc.d[0] * (y + Lc.d[1] * z))] = st[k * nc + i];
      }
    }
  }
  // singular pure-Neumann S~ (NEXT-3, reading A21): pin the last unknown (identity row and
  // column) — one rank only: a slab's block keeps its interface weights on the diagonal and is
  // nonsingular (reading A9c)
  if (h->opts.project_mean && h->nranks == 1) {
    for (long long i = 0; i < nc; ++i) {
      Ad[(nc - 1) * nc + i] = 0.0;
      Ad[i * nc + (nc - 1)] = 0.0;
    }
    Ad[(nc - 1) * nc + (nc - 1)] = 1.0;
  }
  if (!invert_dense(Ad, nc)) {
    set_error("AMG: singular coarsest operator");
    return HDIV_ERR_BREAKDOWN;
  }
  if (h->opts.project_mean && h->nranks == 1) {   // the pinned unknown is 0 and its (redundant)
    for (long long i = 0; i < nc; ++i) {           // equation is dropped: B stays semidefinite
      Ad[(nc - 1) * nc + i] = 0.0;
      Ad[i * nc + (nc - 1)] = 0.0;
    }
  }
  H->nc = nc;
  HDIV_CUDA_TRY(cudaMalloc(&H->cinv, sizeof(double) * nc * nc));
  HDIV_CUDA_TRY(cudaMemcpyAsync(H->cinv, Ad.data(), sizeof(double) * nc * nc, cudaMemcpyHostToDevice, s));
  HDIV_CUDA_TRY(cudaStreamSynchronize(s));
  if (h->opts.amg_global_coarse && h->nranks > 1 && h->dim == 3) return gc_setup(h, s);   // A9e
  return HDIV_OK;
}

// one V-cycle at level l: x = B_l b (x written, b read)
static hdiv_status vcycle(hdiv_ctx* h, size_t l, const double* b, double* x, const int* done,
                          cudaStream_t s, double* part = nullptr, int nbpart = 0) {
  AmgHier* H = h->amg;
  AmgLevel& L = H->L[l];
  if (l + 1 == H->L.size()) {
    coarse_kernel<<<(unsigned)((L.n + ANT / 32 - 1) / (ANT / 32)), ANT, 0, s>>>(H->cinv, L.n, b, x,
                                                                               done);
    return cudaGetLastError() == cudaSuccess ? HDIV_OK : HDIV_ERR_CUDA;
  }
  AmgLevel& C = H->L[l + 1];
  const int nu = H->nu;
  const long long n = L.n;
  const unsigned g = nbk(n);
  StA sta = make_sta(L);
  const bool lev0 = (l == 0);
  // level 0 (S~ itself): the cell stencil in 3D (cell_stencil.h), the SELL copy in 2D
  auto lev0_acc = [&](auto&& fn) {
    if (h->d_cw) {
      const CellGeo cg = make_cellgeo(h);
      switch (h->p) {
        case 1: fn(CellA<1>{cg}); break;
        case 2: fn(CellA<2>{cg}); break;
        case 3: fn(CellA<3>{cg}); break;
        case 4: fn(CellA<4>{cg}); break;
        case 5: fn(CellA<5>{cg}); break;
        default: fn(CellA<6>{cg}); break;
      }
    } else {
      fn(SellA{h->d_ecol, h->d_eval, 2 * h->dim + 1, (int)h->nl2});
    }
  };
  // buffers: pre-smoothing ping-pong in xa/xb, final post-smoothing output in x
  double* cur = L.xa;
  double* nxt = L.xb;
  auto jac = [&](const double* xin, double* xout) {
    if (lev0)
      lev0_acc([&](auto acc) {
        jacobi_kernel<decltype(acc)><<<g, ANT, 0, s>>>(acc, n, b, xin, xout, L.dl1inv, done);
      });
    else jacobi_kernel<StA><<<g, ANT, 0, s>>>(sta, n, b, xin, xout, L.dl1inv, done);
  };
  if (nu >= 1) {
    // (forming x_1 = D^-1 b on the fly inside the second sweep instead of storing it measured
    //  slower at config 4: 25.0 -> 25.5 ms per MINRES iteration — two loads per neighbour)
    scale_kernel<<<g, ANT, 0, s>>>(n, b, L.dl1inv, cur, done);
    for (int k = 1; k < nu; ++k) { jac(cur, nxt); std::swap(cur, nxt); }
  } else {
    HDIV_CUDA_TRY(cudaMemsetAsync(cur, 0, sizeof(double) * n, s));
  }
  // r = b - A x ; s = r - omega A D^-1 r ; b_c = aggregate sums of s
  if (lev0) {
    lev0_acc([&](auto acc) {
      resid_kernel<decltype(acc)><<<g, ANT, 0, s>>>(acc, n, b, cur, L.r, L.dinv, nxt, done);
      smooth_r_kernel<decltype(acc)><<<g, ANT, 0, s>>>(acc, n, L.r, nxt, L.omega, L.sv, done);
    });
    aggsum0_kernel<<<nbk(C.n), ANT, 0, s>>>(make_op0(h), C.d[0], C.d[1], C.n, L.sv, C.b, done);
  } else {
    resid_kernel<StA><<<g, ANT, 0, s>>>(sta, n, b, cur, L.r, L.dinv, nxt, done);
    smooth_r_kernel<StA><<<g, ANT, 0, s>>>(sta, n, L.r, nxt, L.omega, L.sv, done);
    aggsumS_kernel<<<nbk(C.n), ANT, 0, s>>>(L.d[0], L.d[1], L.d[2], C.d[0], C.d[1], C.n, L.dim,
                                            L.sv, C.b, done);
  }
  HDIV_CUDA_TRY(cudaGetLastError());
  // coarse correction e_c = B_{l+1} b_c
  hdiv_status st = vcycle(h, l + 1, C.b, C.e, done, s);
  if (st != HDIV_OK) return st;
  const double* ecv = C.e;
  // prolongate: cur + P e_c -> nxt
  if (lev0)
    lev0_acc([&](auto acc) {
      prolong_kernel<decltype(acc), Agg0><<<g, ANT, 0, s>>>(acc, Agg0{H->agg0}, n, cur, ecv, L.dinv,
                                                             L.omega, nxt, done);
    });
  else
    prolong_st_kernel<<<g, ANT, 0, s>>>(sta, C.d[0], C.d[1], n, cur, ecv, L.dinv, L.omega, nxt,
                                        done);
  HDIV_CUDA_TRY(cudaGetLastError());
  std::swap(cur, nxt);
  // post-smoothing; the last sweep writes x
  if (nu == 0) {
    HDIV_CUDA_TRY(cudaMemcpyAsync(x, cur, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  }
  for (int k = 0; k < nu; ++k) {
    double* out = (k == nu - 1) ? x : nxt;
    if (k == nu - 1 && part && lev0)
      lev0_acc([&](auto acc) {
        jacobi_dot_kernel<decltype(acc)><<<nbpart, ANT, 0, s>>>(acc, n, b, cur, out, L.dl1inv, part,
                                                                 done);
      });
    else
      jac(cur, out);
    if (k < nu - 1) std::swap(cur, nxt);
  }
  HDIV_CUDA_TRY(cudaGetLastError());
  return HDIV_OK;
}

// ---- reading A9e: B = B0 + (I - B0 S~) B_bj (I - S~ B0), B0 = R^T A0^-1 R ----
hdiv_status comm_l2_ghosts(hdiv_ctx* h, double* x, cudaStream_t s);
hdiv_status comm_allgather(hdiv_ctx* h, const double* loc, double* glob, int k, cudaStream_t s);

namespace {

struct GcGeo {
  CellGeo g;
  int p;
  int gx, gy, gz, cdx, cdy;
  long long nzg, z0c;
};

// es[e] = sum of v over the P^3 cells of local element e (one warp per element, fixed order)
template <int P>
__global__ void __launch_bounds__(ANT) gc_elem_sum_kernel(long long E, const double* __restrict__ v,
                                                          double* __restrict__ es,
                                                          const int* __restrict__ done) {
  if (done && *done) return;
  constexpr int PD = P * P * P;
  const long long e = blockIdx.x * (long long)(ANT / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (e >= E) return;
  double t = 0.0;
  for (int k = lane; k < PD; k += 32) t += v[e * PD + k];
  for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
  if (lane == 0) es[e] = t;
}

// part[I] = sum over this slab's elements of aggregate I of es (one CTA per aggregate, each
// thread a fixed strided subset, then a fixed-order tree)
__global__ void __launch_bounds__(ANT) gc_agg_sum_kernel(GcGeo G, const double* __restrict__ es,
                                                         double* __restrict__ part,
                                                         const int* __restrict__ done) {
  if (done && *done) return;
  __shared__ double red[ANT / 32];
  const long long I = blockIdx.x;
  const long long gx = G.gx / G.p, gy = G.gy / G.p, gz = G.gz / G.p;
  const long long Ix = I % G.cdx, Iy = (I / G.cdx) % G.cdy, Iz = I / ((long long)G.cdx * G.cdy);
  const long long NLx = G.g.NL[0], NLy = G.g.NL[1], NLz = G.g.NL[2];
  const long long ez0g = G.z0c / G.p;
  const long long x0 = Ix * gx, x1 = min(x0 + gx, NLx), y0 = Iy * gy, y1 = min(y0 + gy, NLy);
  const long long z0 = max(Iz * gz, ez0g), z1 = min((Iz + 1) * gz, ez0g + NLz);
  double acc = 0.0;
  if (z1 > z0 && x1 > x0 && y1 > y0) {
    const long long bx = x1 - x0, by = y1 - y0, cnt = bx * by * (z1 - z0);
    for (long long t = threadIdx.x; t < cnt; t += ANT) {
      const long long ex = x0 + t % bx, ey = y0 + (t / bx) % by, ez = z0 - ez0g + t / (bx * by);
      acc += es[ex + NLx * (ey + NLy * ez)];
    }
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < ANT / 32; ++w) t += red[w];
    part[I] = t;
  }
}

__global__ void gc_sum_kernel(const double* __restrict__ glob, int P, long long n0,
                              double* __restrict__ c, const int* __restrict__ done) {
  if (done && *done) return;
  const long long I = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (I >= n0) return;
  double t = 0.0;
  for (int r = 0; r < P; ++r) t += glob[r * n0 + I];
  c[I] = t;
}

// u = R^T e (injection of the aggregate values into the cells)
template <int P>
__global__ void __launch_bounds__(ANT) gc_inject_kernel(GcGeo G, const int32_t* __restrict__ eagg,
                                                        const double* __restrict__ e0,
                                                        double* __restrict__ u,
                                                        const int* __restrict__ done) {
  if (done && *done) return;
  constexpr int PD = P * P * P;
  AMG_LOOP(G.g.n) u[i] = e0[eagg[i / PD]];
}

// out = b - S~ u (SUB) or S~ u, through the cell stencil with the slab ghosts
template <int P, bool SUB>
__global__ void __launch_bounds__(ANT, AMG_MINB) gc_smul_kernel(CellGeo g, const double* __restrict__ b,
                                                       const double* __restrict__ u,
                                                       double* __restrict__ out,
                                                       const int* __restrict__ done) {
  if (done && *done) return;
  AMG_LOOP(g.n) {
    const double su = cell_apply<P, true>(g, i, [&](long long j) { return u[j]; });
    out[i] = SUB ? b[i] - su : su;
  }
}

// x = u + w - R^T e1   (u = R^T e0)
template <int P>
__global__ void __launch_bounds__(ANT) gc_final_kernel(GcGeo G, const int32_t* __restrict__ eagg,
                                                       const double* __restrict__ u,
                                                       const double* __restrict__ w,
                                                       const double* __restrict__ e1,
                                                       double* __restrict__ x,
                                                       const int* __restrict__ done) {
  if (done && *done) return;
  constexpr int PD = P * P * P;
  AMG_LOOP(G.g.n) x[i] = (u[i] + w[i]) - e1[eagg[i / PD]];
}

GcGeo make_gcgeo(const hdiv_ctx* h) {
  const GlobalCoarse* C = h->amg->gc;
  GcGeo G;
  G.g = make_cellgeo(h);
  G.p = h->p;
  G.gx = C->g[0]; G.gy = C->g[1]; G.gz = C->g[2];
  G.cdx = C->cd[0]; G.cdy = C->cd[1];
  G.nzg = h->N[2] * h->p;
  G.z0c = C->z0c;
  return G;
}

}  // namespace

static hdiv_status gc_setup(hdiv_ctx* h, cudaStream_t s) {
  auto* C = new GlobalCoarse();
  h->amg->gc = C;
  const int p = h->p;
  const long long ng[3] = {h->N[0] * p, h->N[1] * p, h->N[2] * p};
  long long n0 = 1;
  (void)ng;
  for (int a = 0; a < 3; ++a) {   // blocks of ceil(N_a / 8) whole elements (oracle/amg.py)
    const long long ge = std::max(1LL, (long long)(h->N[a] + 7) / 8);
    C->g[a] = (int)(ge * p);
    C->cd[a] = (int)((h->N[a] + ge - 1) / ge);
    n0 *= C->cd[a];
  }
  C->n0 = n0;
  C->z0c = h->ez0 * p;
  const long long n = h->nl2, plane = h->n[0] * h->n[1];
  HDIV_CUDA_TRY(cudaMalloc(&C->a0inv, sizeof(double) * n0 * n0));
  HDIV_CUDA_TRY(cudaMalloc(&C->part, sizeof(double) * n0));
  HDIV_CUDA_TRY(cudaMalloc(&C->glob, sizeof(double) * n0 * h->nranks));
  HDIV_CUDA_TRY(cudaMalloc(&C->c, sizeof(double) * n0));
  HDIV_CUDA_TRY(cudaMalloc(&C->e0, sizeof(double) * n0));
  HDIV_CUDA_TRY(cudaMalloc(&C->e1, sizeof(double) * n0));
  HDIV_CUDA_TRY(cudaMalloc(&C->rp, sizeof(double) * n));
  HDIV_CUDA_TRY(cudaMalloc(&C->w, sizeof(double) * (n + 2 * plane)));
  HDIV_CUDA_TRY(cudaMemsetAsync(C->w, 0, sizeof(double) * (n + 2 * plane), s));
  HDIV_CUDA_TRY(cudaMalloc(&C->u, sizeof(double) * (n + 2 * plane)));
  HDIV_CUDA_TRY(cudaMemsetAsync(C->u, 0, sizeof(double) * (n + 2 * plane), s));
  HDIV_CUDA_TRY(cudaMalloc(&C->es, sizeof(double) * std::max<long long>(1, h->E)));
  {
    std::vector<int32_t> ea(h->E);
    const long long ge[3] = {C->g[0] / p, C->g[1] / p, C->g[2] / p};
    for (long long e = 0; e < h->E; ++e) {
      const long long ex = e % h->NL[0], ey = (e / h->NL[0]) % h->NL[1], ez = e / (h->NL[0] * h->NL[1]);
      ea[e] = (int32_t)(ex / ge[0] + C->cd[0] * (ey / ge[1] + (long long)C->cd[1] * ((h->ez0 + ez) / ge[2])));
    }
    HDIV_CUDA_TRY(cudaMalloc(&C->eagg, sizeof(int32_t) * std::max<long long>(1, h->E)));
    HDIV_CUDA_TRY(cudaMemcpyAsync(C->eagg, ea.data(), sizeof(int32_t) * h->E, cudaMemcpyHostToDevice, s));
    HDIV_CUDA_TRY(cudaStreamSynchronize(s));
  }
  // A0 = R S~ R^T: this rank's rows of S~ (the CSR, ghost columns for the slab neighbours),
  // summed per aggregate pair on the host in row order, all-gathered and summed in rank order
  std::vector<int64_t> rp(n + 1);
  HDIV_CUDA_TRY(cudaMemcpyAsync(rp.data(), h->d_srow, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost, s));
  HDIV_CUDA_TRY(cudaStreamSynchronize(s));
  const int64_t nnz = rp[n];
  std::vector<int32_t> col(nnz);
  std::vector<double> val(nnz);
  HDIV_CUDA_TRY(cudaMemcpyAsync(col.data(), h->d_scol, sizeof(int32_t) * nnz, cudaMemcpyDeviceToHost, s));
  HDIV_CUDA_TRY(cudaMemcpyAsync(val.data(), h->d_sval, sizeof(double) * nnz, cudaMemcpyDeviceToHost, s));
  HDIV_CUDA_TRY(cudaStreamSynchronize(s));
  const long long pd = (long long)p * p * p;
  auto agg_of = [&](long long j) -> long long {
    long long X, Y, Zg;
    if (j < n) {
      const long long e = j / pd, il = j - e * pd;
      const long long ex = e % h->NL[0], ey = (e / h->NL[0]) % h->NL[1], ez = e / (h->NL[0] * h->NL[1]);
      X = ex * p + il % p;
      Y = ey * p + (il / p) % p;
      Zg = C->z0c + ez * p + il / (p * p);
    } else {
      const long long q = j - n;
      const bool lo = q < plane;
      const long long idx = lo ? q : q - plane;
      X = idx % h->n[0];
      Y = idx / h->n[0];
      Zg = lo ? C->z0c - 1 : C->z0c + h->n[2];
    }
    return X / C->g[0] + C->cd[0] * (Y / C->g[1] + (long long)C->cd[1] * (Zg / C->g[2]));
  };
  std::vector<double> A0(n0 * n0, 0.0);
  for (long long i = 0; i < n; ++i) {
    const long long I = agg_of(i);
    for (int64_t t = rp[i]; t < rp[i + 1]; ++t) A0[I * n0 + agg_of(col[t])] += val[t];
  }
  double* dA0 = nullptr;
  double* dG = nullptr;
  HDIV_CUDA_TRY(cudaMalloc(&dA0, sizeof(double) * n0 * n0));
  HDIV_CUDA_TRY(cudaMalloc(&dG, sizeof(double) * n0 * n0 * h->nranks));
  HDIV_CUDA_TRY(cudaMemcpyAsync(dA0, A0.data(), sizeof(double) * n0 * n0, cudaMemcpyHostToDevice, s));
  hdiv_status st = comm_allgather(h, dA0, dG, (int)(n0 * n0), s);
  if (st != HDIV_OK) { cudaFree(dA0); cudaFree(dG); return st; }
  std::vector<double> all(n0 * n0 * h->nranks);
  HDIV_CUDA_TRY(cudaMemcpyAsync(all.data(), dG, sizeof(double) * all.size(), cudaMemcpyDeviceToHost, s));
  HDIV_CUDA_TRY(cudaStreamSynchronize(s));
  cudaFree(dA0);
  cudaFree(dG);
  for (long long k = 0; k < n0 * n0; ++k) {
    double t = 0.0;
    for (int r = 0; r < h->nranks; ++r) t += all[r * n0 * n0 + k];
    A0[k] = t;
  }
  const bool pin = h->opts.project_mean != 0;   // A0 singular: constants (A21)
  if (pin) {
    for (long long i = 0; i < n0; ++i) { A0[(n0 - 1) * n0 + i] = 0.0; A0[i * n0 + (n0 - 1)] = 0.0; }
    A0[(n0 - 1) * n0 + (n0 - 1)] = 1.0;
  }
  if (!invert_dense(A0, n0)) {
    set_error("AMG: singular global coarse operator");
    return HDIV_ERR_BREAKDOWN;
  }
  if (pin)
    for (long long i = 0; i < n0; ++i) { A0[(n0 - 1) * n0 + i] = 0.0; A0[i * n0 + (n0 - 1)] = 0.0; }
  HDIV_CUDA_TRY(cudaMemcpyAsync(C->a0inv, A0.data(), sizeof(double) * n0 * n0, cudaMemcpyHostToDevice, s));
  HDIV_CUDA_TRY(cudaStreamSynchronize(s));
  return HDIV_OK;
}

// e = A0^-1 R v (R: sums over the aggregates' cells; this rank's share, all-gathered)
static hdiv_status gc_restrict(hdiv_ctx* h, const GcGeo& G, const double* v, double* e,
                               const int* done, cudaStream_t s) {
  GlobalCoarse* C = h->amg->gc;
  const unsigned ge = (unsigned)((h->E + ANT / 32 - 1) / (ANT / 32));
  switch (h->p) {
    case 1: gc_elem_sum_kernel<1><<<ge, ANT, 0, s>>>(h->E, v, C->es, done); break;
    case 2: gc_elem_sum_kernel<2><<<ge, ANT, 0, s>>>(h->E, v, C->es, done); break;
    case 3: gc_elem_sum_kernel<3><<<ge, ANT, 0, s>>>(h->E, v, C->es, done); break;
    case 4: gc_elem_sum_kernel<4><<<ge, ANT, 0, s>>>(h->E, v, C->es, done); break;
    case 5: gc_elem_sum_kernel<5><<<ge, ANT, 0, s>>>(h->E, v, C->es, done); break;
    default: gc_elem_sum_kernel<6><<<ge, ANT, 0, s>>>(h->E, v, C->es, done); break;
  }
  gc_agg_sum_kernel<<<(unsigned)C->n0, ANT, 0, s>>>(G, C->es, C->part, done);
  HDIV_CUDA_TRY(cudaGetLastError());
  hdiv_status st = comm_allgather(h, C->part, C->glob, (int)C->n0, s);
  if (st != HDIV_OK) return st;
  gc_sum_kernel<<<(unsigned)((C->n0 + 255) / 256), 256, 0, s>>>(C->glob, h->nranks, C->n0, C->c, done);
  coarse_kernel<<<(unsigned)((C->n0 + ANT / 32 - 1) / (ANT / 32)), ANT, 0, s>>>(C->a0inv, C->n0, C->c,
                                                                                e, done);
  HDIV_CUDA_TRY(cudaGetLastError());
  return HDIV_OK;
}

template <int P>
static hdiv_status gc_apply_p(hdiv_ctx* h, const GcGeo& G, const double* b, double* x,
                              const int* done, cudaStream_t s, AmgInner inner) {
  GlobalCoarse* C = h->amg->gc;
  const unsigned g = nbk(h->nl2);
  hdiv_status st = gc_restrict(h, G, b, C->e0, done, s);                      // e0 = A0^-1 R b
  if (st != HDIV_OK) return st;
  gc_inject_kernel<P><<<g, ANT, 0, s>>>(G, C->eagg, C->e0, C->u, done);               // u = R^T e0
  HDIV_CUDA_TRY(cudaGetLastError());
  if ((st = comm_l2_ghosts(h, C->u, s)) != HDIV_OK) return st;
  gc_smul_kernel<P, true><<<g, ANT, 0, s>>>(G.g, b, C->u, C->rp, done);       // rp = b - S~ u
  HDIV_CUDA_TRY(cudaGetLastError());
  if ((st = inner(h, C->rp, C->w, done, s)) != HDIV_OK) return st;          // w = M rp
  if ((st = comm_l2_ghosts(h, C->w, s)) != HDIV_OK) return st;
  gc_smul_kernel<P, false><<<g, ANT, 0, s>>>(G.g, nullptr, C->w, C->rp, done);  // S~ w
  HDIV_CUDA_TRY(cudaGetLastError());
  if ((st = gc_restrict(h, G, C->rp, C->e1, done, s)) != HDIV_OK) return st;  // e1 = A0^-1 R S~ w
  gc_final_kernel<P><<<g, ANT, 0, s>>>(G, C->eagg, C->u, C->w, C->e1, x, done);
  HDIV_CUDA_TRY(cudaGetLastError());
  return HDIV_OK;
}

bool amg_has_global_coarse(const hdiv_ctx* h) { return h->amg && h->amg->gc; }

// reading A9e: x = S^-1 b in the balancing form around the inner preconditioner M (the
// block-Jacobi V-cycles or their A9d polynomial):  e0 = A0^-1 R b, u = R^T e0,
// w = M (b - S~ u), x = u + w - R^T A0^-1 R S~ w
hdiv_status amg_global_apply(hdiv_ctx* h, const double* b, double* x, const int* done,
                             cudaStream_t s, AmgInner inner) {
  if (!amg_has_global_coarse(h)) return inner(h, b, x, done, s);
  const GcGeo G = make_gcgeo(h);
  switch (h->p) {
    case 1: return gc_apply_p<1>(h, G, b, x, done, s, inner);
    case 2: return gc_apply_p<2>(h, G, b, x, done, s, inner);
    case 3: return gc_apply_p<3>(h, G, b, x, done, s, inner);
    case 4: return gc_apply_p<4>(h, G, b, x, done, s, inner);
    case 5: return gc_apply_p<5>(h, G, b, x, done, s, inner);
    default: return gc_apply_p<6>(h, G, b, x, done, s, inner);
  }
}

hdiv_status amg_vcycle(hdiv_ctx* h, const double* b, double* x, const int* done, cudaStream_t s,
                       double* part, int nbpart) {
  if (!h->amg) {
    set_error("AMG hierarchy missing");
    return HDIV_ERR_UNSUPPORTED;
  }
  if (part && (h->amg->nu < 1 || h->amg->L.size() < 2)) return HDIV_ERR_UNSUPPORTED;
  return vcycle(h, 0, b, x, done, s, part, nbpart);
}

int amg_num_levels(const hdiv_ctx* h) { return h->amg ? (int)h->amg->L.size() : 0; }

hdiv_status amg_level_info(const hdiv_ctx* h, int l, int64_t* dims, int64_t* n, double* omega,
                           const double** st) {
  if (!h->amg || l < 0 || l >= (int)h->amg->L.size()) {
    set_error("AMG level out of range");
    return HDIV_ERR_SHAPE;
  }
  const AmgLevel& L = h->amg->L[l];
  for (int a = 0; a < 3; ++a) dims[a] = L.d[a];
  *n = L.n;
  *omega = L.omega;
  *st = L.st;
  return HDIV_OK;
}

}  // namespace hdiv
