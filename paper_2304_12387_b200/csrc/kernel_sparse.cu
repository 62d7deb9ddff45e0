// kernel_sparse.cu — topological divergence, Algorithm 1, the Schur approximation S~ in CSR,
// its SpMV, and setup helpers.
//
// D_ij = sigma_ij = +-1 for subcell face j of subcell volume i.
// P:843-873 Algorithm 1: row i of D has 2d entries at I[i] = 2 d i.
// P:463-473 eq.(approx-schur-entries): S~_ii = C~_ii + sum_{k in F(i)} 1/M~_kk,
//           S~_ij = -1/M~_kk for the cell j across interior face k.
// Structured slab: subcell (X,Y,Z) of the local grid, element (X/p, Y/p, Z/p),
// L2 index e p^3 + (X%p) + p((Y%p) + p (Z%p)); RT indices canonical.
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include "internal.h"

namespace hdiv {
namespace {

struct Grid {
  long long NL[3], n[3], off[3];
  int p, dim;
  int ess;                        // eliminated essential sides (NEXT-3), local bitmask
  long long ghost_lo, ghost_hi;   // first ghost column below / above the slab, -1 if none
  __device__ __forceinline__ long long l2(long long X, long long Y, long long Z) const {
    long long e = (X / p) + NL[0] * ((Y / p) + NL[1] * (Z / p));
    long long a = X % p, b = Y % p, c = Z % p;
    if (dim == 2) return e * p * p + a + p * b;
    return e * p * p * p + a + p * (b + p * c);
  }
  // RT index of the face of component c at subcell-face coordinates (I,J,K)
  __device__ __forceinline__ long long rt(int c, long long I, long long J, long long K) const {
    if (dim == 2) {
      if (c == 0) return off[0] + I + (n[0] + 1) * J;
      return off[1] + I + n[0] * J;
    }
    if (c == 0) return off[0] + I + (n[0] + 1) * (J + n[1] * K);
    if (c == 1) return off[1] + I + n[0] * (J + (n[1] + 1) * K);
    return off[2] + I + n[0] * (J + n[1] * K);
  }
  __device__ __forceinline__ void cell_of_l2(long long i, long long* X, long long* Y,
                                             long long* Z) const {
    long long pd = (dim == 2) ? (long long)p * p : (long long)p * p * p;
    long long e = i / pd, il = i % pd;
    long long ex = e % NL[0], ey = (e / NL[0]) % NL[1], ez = (dim == 3) ? e / (NL[0] * NL[1]) : 0;
    *X = ex * p + il % p;
    *Y = ey * p + (il / p) % p;
    *Z = (dim == 3) ? ez * p + il / (p * p) : 0;
  }
};

Grid make_grid(const hdiv_ctx* h) {
  Grid g;
  for (int d = 0; d < 3; ++d) { g.NL[d] = h->NL[d]; g.n[d] = h->n[d]; g.off[d] = h->off[d]; }
  g.p = h->p; g.dim = h->dim; g.ess = h->ess;
  const long long lplane = (h->dim == 3) ? h->n[0] * h->n[1] : h->n[0];
  g.ghost_lo = (h->rank > 0) ? h->nl2 : -1;
  g.ghost_hi = (h->rank < h->nranks - 1) ? h->nl2 + lplane : -1;
  return g;
}

inline unsigned nblocks(long long n, int nt) { return (unsigned)((n + nt - 1) / nt); }

// (D u)_i = sum over the 2d faces of cell i, +1 on the + side, -1 on the - side
__global__ void div_kernel(Grid g, const double* __restrict__ u, double* __restrict__ yq,
                           long long nl2) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= nl2) return;
  long long X, Y, Z;
  g.cell_of_l2(i, &X, &Y, &Z);
  // eliminated essential faces act as zero (NEXT-3: the (2,1) block is D F)
  auto uu = [&](int c, long long I, long long J, long long K) {
    const long long idx = (c == 0) ? I : (c == 1) ? J : K;
    return face_masked(g.ess, c, idx, g.n[c]) ? 0.0 : u[g.rt(c, I, J, K)];
  };
  double s = uu(0, X + 1, Y, Z) - uu(0, X, Y, Z);
  s += uu(1, X, Y + 1, Z) - uu(1, X, Y, Z);
  if (g.dim == 3) s += uu(2, X, Y, Z + 1) - uu(2, X, Y, Z);
  yq[i] = s;
}

// (D^T q)_f = q(cell on - side) - q(cell on + side)
__global__ void divT_kernel(Grid g, const double* __restrict__ q, double* __restrict__ yu,
                            long long nrt) {
  long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (f >= nrt) return;
  int c = (g.dim == 3 && f >= g.off[2]) ? 2 : (f >= g.off[1] ? 1 : 0);
  long long r = f - g.off[c];
  long long e0 = g.n[0] + (c == 0), e1 = g.n[1] + (c == 1);
  long long I = r % e0, J = (r / e0) % e1, K = (g.dim == 3) ? r / (e0 * e1) : 0;
  long long idx[3] = {I, J, K};
  long long nn = g.n[c];
  if (face_masked(g.ess, c, idx[c], nn)) { yu[f] = 0.0; return; }   // F D^T (NEXT-3)
  double s = 0.0;
  if (idx[c] > 0) {
    long long m[3] = {I, J, K};
    m[c] -= 1;
    s += q[g.l2(m[0], m[1], m[2])];
  }
  if (idx[c] < nn) s -= q[g.l2(I, J, K)];
  yu[f] = s;
}

// Algorithm 1: I[i] = 2 d i ; order (-x,+x,-y,+y,-z,+z); sigma_loc sigma_glob
__global__ void div_csr_kernel(Grid g, int64_t* rp, int64_t* col, double* val, long long nl2) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i > nl2) return;
  int nd = 2 * g.dim;
  rp[i] = nd * i;
  if (i == nl2) return;
  long long X, Y, Z;
  g.cell_of_l2(i, &X, &Y, &Z);
  long long* c = (long long*)col + nd * i;
  double* v = val + nd * i;
  c[0] = g.rt(0, X, Y, Z); v[0] = -1.0;
  c[1] = g.rt(0, X + 1, Y, Z); v[1] = 1.0;
  c[2] = g.rt(1, X, Y, Z); v[2] = -1.0;
  c[3] = g.rt(1, X, Y + 1, Z); v[3] = 1.0;
  if (g.dim == 3) {
    c[4] = g.rt(2, X, Y, Z); v[4] = -1.0;
    c[5] = g.rt(2, X, Y, Z + 1); v[5] = 1.0;
  }
}

// neighbours of cell (X,Y,Z) in face order (-x,+x,-y,+y,-z,+z); -1 if outside the local grid
__device__ __forceinline__ int faces_of(const Grid& g, long long X, long long Y, long long Z,
                                        long long* face, long long* nb) {
  int nd = 2 * g.dim;
  face[0] = g.rt(0, X, Y, Z);     nb[0] = X > 0 ? g.l2(X - 1, Y, Z) : -1;
  face[1] = g.rt(0, X + 1, Y, Z); nb[1] = X + 1 < g.n[0] ? g.l2(X + 1, Y, Z) : -1;
  face[2] = g.rt(1, X, Y, Z);     nb[2] = Y > 0 ? g.l2(X, Y - 1, Z) : -1;
  face[3] = g.rt(1, X, Y + 1, Z); nb[3] = Y + 1 < g.n[1] ? g.l2(X, Y + 1, Z) : -1;
  if (g.dim == 3) {
    face[4] = g.rt(2, X, Y, Z);     nb[4] = Z > 0 ? g.l2(X, Y, Z - 1) : -1;
    face[5] = g.rt(2, X, Y, Z + 1); nb[5] = Z + 1 < g.n[2] ? g.l2(X, Y, Z + 1) : -1;
    // slab interfaces: the neighbour across is a ghost cell (ordered by subcell X + n_x Y)
    if (Z == 0 && g.ghost_lo >= 0) nb[4] = g.ghost_lo + X + g.n[0] * Y;
    if (Z + 1 == g.n[2] && g.ghost_hi >= 0) nb[5] = g.ghost_hi + X + g.n[0] * Y;
  } else {
    if (Y == 0 && g.ghost_lo >= 0) nb[2] = g.ghost_lo + X;
    if (Y + 1 == g.n[1] && g.ghost_hi >= 0) nb[3] = g.ghost_hi + X;
  }
  return nd;
}

__global__ void schur_count_kernel(Grid g, int64_t* cnt, long long nl2) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i > nl2) return;
  if (i == nl2) { cnt[i] = 0; return; }
  long long X, Y, Z, face[6], nb[6];
  g.cell_of_l2(i, &X, &Y, &Z);
  int nd = faces_of(g, X, Y, Z, face, nb);
  int c = 1;
  for (int k = 0; k < nd; ++k) c += (nb[k] >= 0);
  cnt[i] = c;
}

__global__ void schur_fill_kernel(Grid g, const double* __restrict__ mdiag,
                                  const double* __restrict__ ctil, const int64_t* __restrict__ rp,
                                  int32_t* col, double* val, double* sdinv, long long nl2) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= nl2) return;
  long long X, Y, Z, face[6], nb[6];
  g.cell_of_l2(i, &X, &Y, &Z);
  int nd = faces_of(g, X, Y, Z, face, nb);
  long long cc[7];
  double vv[7];
  int m = 0;
  double d = ctil[i];
  for (int k = 0; k < nd; ++k) {
    // an eliminated boundary face (k = 2 axis + side, the ess bit layout) is not in F(i)
    if (nb[k] < 0 && ((g.ess >> k) & 1)) continue;
    double w = 1.0 / mdiag[face[k]];
    d += w;
    if (nb[k] >= 0) { cc[m] = nb[k]; vv[m] = -w; ++m; }
  }
  cc[m] = i; vv[m] = d; ++m;
  for (int a = 1; a < m; ++a) {   // insertion sort by column
    long long kc = cc[a]; double kv = vv[a]; int b = a - 1;
    while (b >= 0 && cc[b] > kc) { cc[b + 1] = cc[b]; vv[b + 1] = vv[b]; --b; }
    cc[b + 1] = kc; vv[b + 1] = kv;
  }
  long long r0 = rp[i];
  for (int a = 0; a < m; ++a) { col[r0 + a] = (int32_t)cc[a]; val[r0 + a] = vv[a]; }
  sdinv[i] = 1.0 / d;
}

// Cell-major face weights of S~ for the matrix-free Chebyshev stencil (3D): cw[0] = S~_ii (the
// same sum in the same face order as schur_fill_kernel), cw[1..3] = w_k = 1/M~_kk of the cell's
// +x / +y / +z face when a neighbour (or a ghost) lies across it, else 0; cw[4] (one plane,
// indexed X + n_x Y) = the -z interface face of a slab whose lower neighbour is a ghost.  The
// -x / -y / -z weights of a cell are its neighbours' + weights, so every array is read
// coalesced in the L2 (element-major) numbering.
__global__ void cellw_kernel(Grid g, const double* __restrict__ mdiag,
                             const double* __restrict__ ctil, double* __restrict__ cw,
                             long long nl2) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= nl2) return;
  long long X, Y, Z, face[6], nb[6];
  g.cell_of_l2(i, &X, &Y, &Z);
  faces_of(g, X, Y, Z, face, nb);
  double d = ctil[i], w[6];
  for (int k = 0; k < 6; ++k) {
    w[k] = 0.0;
    if (nb[k] < 0 && ((g.ess >> k) & 1)) continue;   // eliminated: not in F(i)
    w[k] = 1.0 / mdiag[face[k]];
    d += w[k];
  }
  cw[i] = d;
  cw[nl2 + i] = nb[1] >= 0 ? w[1] : 0.0;
  cw[2 * nl2 + i] = nb[3] >= 0 ? w[3] : 0.0;
  cw[3 * nl2 + i] = nb[5] >= 0 ? w[5] : 0.0;
  if (Z == 0 && g.ghost_lo >= 0) cw[4 * nl2 + X + g.n[0] * Y] = w[4];
}

// CSR -> SELL-32 with fixed width W: entry (row, k) at (row/32)*32*W + k*32 + row%32
__global__ void sell_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ c,
                            const double* __restrict__ v, int32_t* ec, double* ev, long long n,
                            int W) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long base = (i / 32) * 32 * W + (i % 32);
  const long long r0 = rp[i], r1 = rp[i + 1];
  for (int k = 0; k < W; ++k) {
    const long long t = r0 + k;
    ec[base + 32 * k] = (t < r1) ? c[t] : (int32_t)i;
    ev[base + 32 * k] = (t < r1) ? v[t] : 0.0;
  }
}

// NEXT-3: y_b = x_b (x != nullptr) or cval on the faces of the eliminated sides; blockIdx.y =
// 2 c + side, one thread per face of that side's plane
__global__ void ess_fixup_kernel(Grid g, const double* __restrict__ x, double* __restrict__ y,
                                 double cval, const int* __restrict__ skip) {
  if (skip && *skip) return;
  const int k = blockIdx.y, c = k >> 1, side = k & 1;
  if (c >= g.dim || !((g.ess >> k) & 1)) return;
  // the two tangential axes (2D: one) of component c
  const int t0 = (c == 0) ? 1 : 0, t1 = (c == 2) ? 1 : 2;
  const long long n0 = g.n[t0], n1 = (g.dim == 3) ? g.n[t1] : 1;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n0 * n1) return;
  long long idx[3] = {0, 0, 0};
  idx[c] = side ? g.n[c] : 0;
  idx[t0] = i % n0;
  if (g.dim == 3) idx[t1] = i / n0;
  const long long f = g.rt(c, idx[0], idx[1], idx[2]);
  y[f] = x ? x[f] : cval;
}

__global__ void recip_kernel(const double* __restrict__ a, double* __restrict__ r, long long n) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) r[i] = 1.0 / a[i];
}

__global__ void schur_export_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ c,
                                    const double* __restrict__ v, int64_t* rp_o, int64_t* c_o,
                                    double* v_o, long long nl2) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i > nl2) return;
  rp_o[i] = rp[i];
  if (i == nl2) return;
  for (long long t = rp[i]; t < rp[i + 1]; ++t) { c_o[t] = c[t]; v_o[t] = v[t]; }
}

__global__ void spmv_kernel(const int64_t* __restrict__ rp, const int32_t* __restrict__ c,
                            const double* __restrict__ v, const double* __restrict__ x,
                            double* __restrict__ y, long long nl2) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= nl2) return;
  double s = 0.0;
  for (long long t = rp[i]; t < rp[i + 1]; ++t) s = fma(v[t], x[c[t]], s);
  y[i] = s;
}

// C~ from diag(W_1) (w1 = sum_q w_q psi_a^2 / det J) and the per-element coefficient c2:
//   grad-div  C~ = 1 / diag(W_alpha) = 1 / (alpha_e w1)
//   Darcy     C~ = diag(W_gamma) / diag(W)^2 = gamma_e w1 / (w1 w1)
__global__ void ctil_kernel(const double* __restrict__ w1, const double* __restrict__ c2,
                            double* ctil, long long nl2, long long pd, int darcy) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= nl2) return;
  double w = w1[i], c = c2[i / pd];
  ctil[i] = darcy ? (c * w) / (w * w) : 1.0 / (c * w);
}

__global__ void geom_check_kernel(const double* __restrict__ vert, Tab1D tab, long long NLx,
                                  long long NLy, long long E, int dim, int* bad) {
  long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= E) return;
  long long ex = e % NLx, ey = (e / NLx) % NLy, ez = (dim == 3) ? e / (NLx * NLy) : 0;
  double X[8][3];
  for (int v = 0; v < (1 << dim); ++v) {
    int a = v & 1, b = (v >> 1) & 1, c = (v >> 2) & 1;
    long long gv = (dim == 3) ? ((ez + c) * (NLy + 1) + (ey + b)) * (NLx + 1) + (ex + a)
                              : (ey + b) * (NLx + 1) + (ex + a);
    for (int d = 0; d < dim; ++d) X[v][d] = vert[gv * dim + d];
  }
  int Q = tab.Q;
  for (int qz = 0; qz < (dim == 3 ? Q : 1); ++qz)
    for (int qy = 0; qy < Q; ++qy)
      for (int qx = 0; qx < Q; ++qx) {
        double xh = tab.xq[qx], yh = tab.xq[qy], zh = (dim == 3) ? tab.xq[qz] : 0.0;
        double J[3][3];
        double det;
        if (dim == 2) {
          for (int d = 0; d < 2; ++d) {
            J[d][0] = (1 - yh) * (X[1][d] - X[0][d]) + yh * (X[3][d] - X[2][d]);
            J[d][1] = (1 - xh) * (X[2][d] - X[0][d]) + xh * (X[3][d] - X[1][d]);
          }
          det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
        } else {
          for (int d = 0; d < 3; ++d) {
            J[d][0] = (1 - yh) * (1 - zh) * (X[1][d] - X[0][d]) + yh * (1 - zh) * (X[3][d] - X[2][d]) +
                      (1 - yh) * zh * (X[5][d] - X[4][d]) + yh * zh * (X[7][d] - X[6][d]);
            J[d][1] = (1 - xh) * (1 - zh) * (X[2][d] - X[0][d]) + xh * (1 - zh) * (X[3][d] - X[1][d]) +
                      (1 - xh) * zh * (X[6][d] - X[4][d]) + xh * zh * (X[7][d] - X[5][d]);
            J[d][2] = (1 - xh) * (1 - yh) * (X[4][d] - X[0][d]) + xh * (1 - yh) * (X[5][d] - X[1][d]) +
                      (1 - xh) * yh * (X[6][d] - X[2][d]) + xh * yh * (X[7][d] - X[3][d]);
          }
          det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
        }
        if (!(det > 0.0)) { atomicExch(bad, 1); return; }
      }
}

}  // namespace

cudaError_t launch_ess_fixup(const hdiv_ctx* h, const double* x, double* y, double cval,
                             const int* skip, cudaStream_t s) {
  if (!h->ess) return cudaSuccess;
  long long mx = 0;
  for (int c = 0; c < h->dim; ++c) {
    long long pl = 1;
    for (int a = 0; a < h->dim; ++a)
      if (a != c) pl *= h->n[a];
    if (pl > mx) mx = pl;
  }
  dim3 grid(nblocks(mx, 256), 2 * h->dim);
  count_op();
  ess_fixup_kernel<<<grid, 256, 0, s>>>(make_grid(h), x, y, cval, skip);
  return cudaGetLastError();
}

cudaError_t launch_div(const hdiv_ctx* h, const double* u, double* yq, cudaStream_t s) {
  div_kernel<<<nblocks(h->nl2, 256), 256, 0, s>>>(make_grid(h), u, yq, h->nl2);
  return cudaGetLastError();
}

cudaError_t launch_divT(const hdiv_ctx* h, const double* q, double* yu, cudaStream_t s) {
  divT_kernel<<<nblocks(h->nrt, 256), 256, 0, s>>>(make_grid(h), q, yu, h->nrt);
  return cudaGetLastError();
}

cudaError_t launch_div_csr(const hdiv_ctx* h, int64_t* rp, int64_t* col, double* val,
                           cudaStream_t s) {
  div_csr_kernel<<<nblocks(h->nl2 + 1, 256), 256, 0, s>>>(make_grid(h), rp, col, val, h->nl2);
  return cudaGetLastError();
}

cudaError_t launch_geometry_check(const hdiv_ctx* h, int* bad, cudaStream_t s) {
  geom_check_kernel<<<nblocks(h->E, 128), 128, 0, s>>>(h->d_vert, h->tab, h->NL[0], h->NL[1],
                                                        h->E, h->dim, bad);
  return cudaGetLastError();
}

cudaError_t launch_l2_diag(const hdiv_ctx* h, double* w1, cudaStream_t s);   // kernel_general.cu
cudaError_t launch_l2_diag_gamma(const hdiv_ctx* h, double* wg, cudaStream_t s);

// general gamma (NEXT-3): C~ = diag(W_gamma) / diag(W)^2
__global__ void ctil_g_kernel(const double* __restrict__ w1, const double* __restrict__ wg,
                              double* ctil, long long nl2) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= nl2) return;
  const double w = w1[i];
  ctil[i] = wg[i] / (w * w);
}

cudaError_t launch_ctil(const hdiv_ctx* h, const double* d_c2, double* ctil, cudaStream_t s) {
  cudaError_t e = launch_l2_diag(h, ctil, s);   // w1 into ctil, then transform in place
  if (e != cudaSuccess) return e;
  if (h->d_gvert) {
    double* wg = nullptr;
    if ((e = cudaMallocAsync(&wg, sizeof(double) * h->nl2, s)) != cudaSuccess) return e;
    if ((e = launch_l2_diag_gamma(h, wg, s)) != cudaSuccess) return e;
    ctil_g_kernel<<<nblocks(h->nl2, 256), 256, 0, s>>>(ctil, wg, ctil, h->nl2);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    return cudaFreeAsync(wg, s);
  }
  long long pd = (h->dim == 2) ? (long long)h->p * h->p : (long long)h->p * h->p * h->p;
  ctil_kernel<<<nblocks(h->nl2, 256), 256, 0, s>>>(ctil, d_c2, ctil, h->nl2, pd,
                                                  h->kind == HDIV_DARCY);
  return cudaGetLastError();
}

hdiv_status build_schur(hdiv_ctx* h, cudaStream_t s) {
  const long long n = h->nl2;
  Grid g = make_grid(h);
  int64_t* cnt = nullptr;
  HDIV_CUDA_TRY(cudaMalloc(&h->d_srow, sizeof(int64_t) * (n + 1)));
  HDIV_CUDA_TRY(cudaMalloc(&cnt, sizeof(int64_t) * (n + 1)));
  schur_count_kernel<<<nblocks(n + 1, 256), 256, 0, s>>>(g, cnt, n);
  HDIV_CUDA_TRY(cudaGetLastError());
  size_t tmp_bytes = 0;
  HDIV_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, h->d_srow, n + 1, s));
  void* tmp = nullptr;
  HDIV_CUDA_TRY(cudaMalloc(&tmp, tmp_bytes));
  HDIV_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, h->d_srow, n + 1, s));
  int64_t nnz = 0;
  HDIV_CUDA_TRY(cudaMemcpyAsync(&nnz, h->d_srow + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  HDIV_CUDA_TRY(cudaStreamSynchronize(s));
  cudaFree(tmp);
  cudaFree(cnt);
  h->snnz = nnz;
  HDIV_CUDA_TRY(cudaMalloc(&h->d_scol, sizeof(int32_t) * (nnz > 0 ? nnz : 1)));
  HDIV_CUDA_TRY(cudaMalloc(&h->d_sval, sizeof(double) * (nnz > 0 ? nnz : 1)));
  HDIV_CUDA_TRY(cudaMalloc(&h->d_sdinv, sizeof(double) * (n > 0 ? n : 1)));
  schur_fill_kernel<<<nblocks(n, 256), 256, 0, s>>>(g, h->d_mdiag, h->d_ctil, h->d_srow,
                                                    h->d_scol, h->d_sval, h->d_sdinv, n);
  HDIV_CUDA_TRY(cudaGetLastError());
  if (h->dim == 3) {   // S~ inside S^-1 (Chebyshev, AMG level 0): the cell stencil's weights
    const long long lplane = h->n[0] * h->n[1];
    HDIV_CUDA_TRY(cudaMalloc(&h->d_cw, sizeof(double) * (4 * n + lplane)));
    HDIV_CUDA_TRY(cudaMemsetAsync(h->d_cw, 0, sizeof(double) * (4 * n + lplane), s));
    cellw_kernel<<<nblocks(n, 256), 256, 0, s>>>(g, h->d_mdiag, h->d_ctil, h->d_cw, n);
    HDIV_CUDA_TRY(cudaGetLastError());
    return HDIV_OK;
  }
  // 2D: sliced-ELL copy used by the SpMV inside S^-1 (coalesced slot loads)
  const int W = 2 * h->dim + 1;
  const long long ns = (n + 31) / 32;
  HDIV_CUDA_TRY(cudaMalloc(&h->d_ecol, sizeof(int32_t) * ns * 32 * W));
  HDIV_CUDA_TRY(cudaMalloc(&h->d_eval, sizeof(double) * ns * 32 * W));
  HDIV_CUDA_TRY(cudaMemsetAsync(h->d_ecol, 0, sizeof(int32_t) * ns * 32 * W, s));
  HDIV_CUDA_TRY(cudaMemsetAsync(h->d_eval, 0, sizeof(double) * ns * 32 * W, s));
  sell_kernel<<<nblocks(n, 256), 256, 0, s>>>(h->d_srow, h->d_scol, h->d_sval, h->d_ecol,
                                              h->d_eval, n, W);
  HDIV_CUDA_TRY(cudaGetLastError());
  return HDIV_OK;
}

cudaError_t launch_schur_export(const hdiv_ctx* h, int64_t* rp, int64_t* col, double* val,
                                cudaStream_t s) {
  schur_export_kernel<<<nblocks(h->nl2 + 1, 256), 256, 0, s>>>(h->d_srow, h->d_scol, h->d_sval,
                                                               rp, col, val, h->nl2);
  return cudaGetLastError();
}

cudaError_t launch_spmv(const hdiv_ctx* h, const double* x, double* y, cudaStream_t s) {
  spmv_kernel<<<nblocks(h->nl2, 256), 256, 0, s>>>(h->d_srow, h->d_scol, h->d_sval, x, y, h->nl2);
  return cudaGetLastError();
}

}  // namespace hdiv
