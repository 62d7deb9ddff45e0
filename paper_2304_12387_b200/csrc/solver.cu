// solver.cu — block-diagonal preconditioner and MINRES, device resident.
//
// P:411-421 Remark: P = diag(tau M~, S^);  P:668 M~^-1 is diagonal scaling;
// S^-1 = Chebyshev-Jacobi polynomial on S~ (reading A9/A10; the paper uses one AMG V-cycle,
// P:889, which is NEXT-1).  P:169 / P:663: MINRES; rtol 1e-12 on the preconditioned
// residual (reading A8).  Recurrence: Elman-Silvester-Wathen preconditioned MINRES
// (SURVEY §8(c) step 10), written with the unnormalised z (A z/gamma = (A z)/gamma).
//
// Per iteration (all on the handle's stream, captured in a CUDA graph of 6 iterations so the
// buffer rotation v(3) / w(3) / z(2) is baked into the graph):
//   apply_block(z) -> Az                      (kernel_affine / kernel_general [+ reverse-add])
//   dot(Az, z) -> local scalar [-> allgather] -> delta = <Az,z>/gamma^2
//   vupd: v_new, z_new_u = v_new_u/(tau M~), partial <z_u, v_u>
//   Chebyshev steps on v_new_q -> z_new_q [ghost refresh before each SpMV], partial <z_q, v_q>
//   scalar: gamma_new, Givens rotation, eta, convergence flag
//   wupd: w_new, x += c eta w_new
// Reductions: fixed grid, fixed-order block and partial sums, and (multi-GPU) an all-gather of
// the per-rank scalars summed in rank order -> deterministic and identical on every rank.
// Every kernel reads the device `done` flag and returns early once converged.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "cell_stencil.h"
#include "internal.h"

namespace hdiv {

hdiv_status comm_l2_ghosts(hdiv_ctx* h, double* x, cudaStream_t s);
hdiv_status comm_allgather(hdiv_ctx* h, const double* loc, double* glob, int k, cudaStream_t s);
bool comm_is_loopback(const hdiv_ctx* h);

namespace {

constexpr int RED_BLOCKS = 148 * 8;   // 8 x 256 threads per SM: bytes in flight
constexpr int RED_NT = 256;

struct MState {
  double gamma, gamma_old, eta, gamma1, s, s_old, c, c_old, delta;
  double wz, wa3, wa2, xc, rtol, rel;
  double xcp;   // deferred x-update coefficient of w_{j-1} (odd iterations defer, see wstep)
  int done, iters, maxit, breakdown, conv, pend;
};

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double red[RED_NT / 32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  if (l == 0) red[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x < 32) {
    r = (l < RED_NT / 32) ? red[l] : 0.0;
    for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
  }
  __syncthreads();
  return r;   // valid in thread 0
}

// partial sums of a.b over [0,n) excluding [ex_lo, ex_hi) (replicated interface plane)
__global__ void __launch_bounds__(RED_NT)
dot_kernel(const double* __restrict__ a, const double* __restrict__ b, long long n,
           long long ex_lo, long long ex_hi, double* __restrict__ part,
           const int* __restrict__ done) {
  if (done && *done) return;
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)RED_NT + threadIdx.x; i < n;
       i += (long long)gridDim.x * RED_NT)
    if (i < ex_lo || i >= ex_hi) s = fma(a[i], b[i], s);
  s = block_sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__device__ __forceinline__ double sum_partials(const double* part, int nb) {
  double s = 0.0;
  for (int i = threadIdx.x; i < nb; i += RED_NT) s += part[i];
  return block_sum(s);
}

// loc[0] = sum(part_a) (+ sum(part_b)); nb = the reduction grid of the partials
__global__ void __launch_bounds__(RED_NT)
local_reduce_kernel(const double* part_a, const double* part_b, double* loc,
                    const int* __restrict__ done, int nb) {
  if (done && *done) return;
  double s = sum_partials(part_a, nb);
  double t = part_b ? sum_partials(part_b, nb) : 0.0;
  if (threadIdx.x == 0) loc[0] = s + t;
}

__device__ __forceinline__ double rank_sum(const double* glob, int P) {
  double s = 0.0;
  for (int r = 0; r < P; ++r) s += glob[r];
  return s;
}


// delta = <Az, z>/gamma^2 from the all-gathered partial (fused: no separate scalar launch);
// v_new = Az/g - (delta/g) v - (g/g_old) v_old ; z_new_u = v_new_u / (tau M~)
__global__ void __launch_bounds__(RED_NT)
vupd_kernel(const double* __restrict__ Az, const double* __restrict__ v,
            const double* __restrict__ v_old, double* __restrict__ v_new,
            double* __restrict__ z_new, const double* __restrict__ mdiag, double tau,
            long long nrt, long long n, long long ex_lo, long long ex_hi,
            MState* __restrict__ st, const double* __restrict__ glob, int P,
            const double* __restrict__ dpart, int nb, double* part) {
  if (st->done) return;
  const double g = st->gamma, ig = 1.0 / g;
  // single rank: every block sums the <Az, z> partials itself (same order as the reduction
  // kernel it replaces, so bitwise the same delta); multi-rank: the all-gathered scalars
  __shared__ double sdel;
  if (dpart) {
    const double t = sum_partials(dpart, nb);
    if (threadIdx.x == 0) sdel = t;
    __syncthreads();
  }
  const double delta = (dpart ? sdel : rank_sum(glob, P)) / (g * g);
  const double cd = delta * ig, co = g / st->gamma_old;
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)RED_NT + threadIdx.x; i < n;
       i += (long long)gridDim.x * RED_NT) {
    double vn = Az[i] * ig - cd * v[i] - co * v_old[i];
    v_new[i] = vn;
    if (i < nrt) {
      double zn = vn * mdiag[i];   // mdiag here: the precomputed 1 / (tau M~)
      z_new[i] = zn;
      if (i < ex_lo || i >= ex_hi) s = fma(zn, vn, s);
    }
  }
  s = block_sum(s);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = s;
    if (blockIdx.x == 0) st->delta = delta;   // for scalar_kernel (a later launch)
  }
}

// Chebyshev semi-iteration (reading A10), first term: y_0 = D^-1 v / theta.  `last` adds <y, v>.
__global__ void __launch_bounds__(RED_NT)
cheb_first_kernel(const double* __restrict__ rin, const double* __restrict__ dinv, double itheta,
                  double* __restrict__ d, double* __restrict__ y, long long n, int last,
                  double* part, const int* __restrict__ done) {
  if (done && *done) return;
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)RED_NT + threadIdx.x; i < n;
       i += (long long)gridDim.x * RED_NT) {
    double di = dinv[i] * rin[i] * itheta;
    d[i] = di;
    y[i] = di;
    if (last) s = fma(di, rin[i], s);
  }
  if (last && part) {
    s = block_sum(s);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
  }
}

// Chebyshev step as a three-term recurrence on the iterate (the same polynomial as the r/d form
// of reading A10: d_i = y_i - y_{i-1}, r_i = v - S~ y_{i-1}):
//   y_i = y_{i-1} + c1 (y_{i-1} - y_{i-2}) + c2 D^-1 (v - S~ y_{i-1})        (y_{-1} = 0)
// S~ through the SELL-32 copy; per row: the slots, y_{i-1} (gathered), y_{i-2}, v, D^-1 -> y_i
// (124 B instead of the r/d form's 140: no residual / direction vectors are written).
template <int W>
__global__ void __launch_bounds__(RED_NT)
cheb3_kernel(const int32_t* __restrict__ ecol, const double* __restrict__ eval,
             const double* __restrict__ v, const double* ym1, const double* ym2,
             const double* __restrict__ dinv, double* yout, double c1, double c2, long long n,
             int last, double* part, const int* __restrict__ done) {
  if (done && *done) return;
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)RED_NT + threadIdx.x; i < n;
       i += (long long)gridDim.x * RED_NT) {
    const long long base = (i >> 5) * (32 * W) + (i & 31);
    double sd = 0.0;
#pragma unroll
    for (int k = 0; k < W; ++k) sd = fma(eval[base + 32 * k], ym1[ecol[base + 32 * k]], sd);
    const double y = ym1[i];
    const double dprev = ym2 ? y - ym2[i] : y;
    const double yn = y + (c1 * dprev + c2 * dinv[i] * (v[i] - sd));
    yout[i] = yn;
    if (last) s = fma(yn, v[i], s);
  }
  if (last && part) {
    s = block_sum(s);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
  }
}

// The same step with S~ y from the cell-major weights (3D, one thread per cell, lanes over
// consecutive cells: every stream coalesced, the six neighbours shifted copies of the same
// rows): per cell diag, three + weights, y_{i-1}, y_{i-2}, v, y_i = 64 B, vs SELL's 124.
#ifndef HDIV_CHEB3C_MINB
#define HDIV_CHEB3C_MINB 8
#endif
// Y0 = 1: y_{i-1} is the first term y_0 = D^-1 v / theta, formed on the fly from v and D^-1 at
// each stencil point (the first term is never stored: one pass over the L2 vectors fewer);
// Y0 = 2: y_{i-2} is y_0 (the second step), likewise
template <int P, int Y0>
__global__ void __launch_bounds__(RED_NT, HDIV_CHEB3C_MINB)
cheb3c_kernel(CellGeo g, const double* __restrict__ v, const double* __restrict__ ym1,
              const double* ym2, const double* __restrict__ dinv, double itheta, double* yout,
              double c1, double c2, int last, double* part, const int* __restrict__ done) {
  if (done && *done) return;
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)RED_NT + threadIdx.x; i < g.n;
       i += (long long)gridDim.x * RED_NT) {
    double sy, y;
    if constexpr (Y0 == 1) {
      sy = cell_apply<P, false>(g, i, [&](long long j) { return dinv[j] * v[j] * itheta; });
      y = dinv[i] * v[i] * itheta;
    } else {
      sy = cell_apply<P, true>(g, i, [&](long long j) { return ym1[j]; });
      y = ym1[i];
    }
    const double yo = (Y0 == 2) ? dinv[i] * v[i] * itheta : (ym2 ? ym2[i] : 0.0);
    const double dprev = (Y0 == 1) ? y : y - yo;
    const double yn = y + (c1 * dprev + c2 * ((v[i] - sy) / g.cw[i]));
    yout[i] = yn;
    if (last) s = fma(yn, v[i], s);
  }
  if (last && part) {
    s = block_sum(s);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
  }
}

// Reading A9d: Chebyshev polynomial in B S~ (B = one AMG V-cycle) in the r/d form of the
// oracle (oracle/amg.py AMGSchur.__call__): d_0 = B r / theta, y = d_0; for i >= 1:
// r_i = r_{i-1} - S~ d_{i-1}, d_i = c1 d_{i-1} + c2 B r_i, y += d_i.
// pcheb_first: d = t / theta, y = d (t = B r_0); `last` (degree 1 never gets here) unused.
__global__ void __launch_bounds__(RED_NT)
pcheb_first_kernel(const double* __restrict__ t, double itheta, double* __restrict__ d,
                   double* __restrict__ y, long long n, const int* __restrict__ done) {
  if (done && *done) return;
  for (long long i = blockIdx.x * (long long)RED_NT + threadIdx.x; i < n;
       i += (long long)gridDim.x * RED_NT) {
    const double di = t[i] * itheta;
    d[i] = di;
    y[i] = di;
  }
}

// r_out = r_in - S~ d through the cell stencil (3D; d in ghost space for slabs)
template <int P>
__global__ void __launch_bounds__(RED_NT, HDIV_CHEB3C_MINB)
pcheb_res_cell_kernel(CellGeo g, const double* __restrict__ rin, const double* __restrict__ d,
                      double* __restrict__ rout, const int* __restrict__ done) {
  if (done && *done) return;
  for (long long i = blockIdx.x * (long long)RED_NT + threadIdx.x; i < g.n;
       i += (long long)gridDim.x * RED_NT)
    rout[i] = rin[i] - cell_apply<P, true>(g, i, [&](long long j) { return d[j]; });
}

// the same through the SELL-32 copy (2D; ghost columns >= n read from d's ghost space)
template <int W>
__global__ void __launch_bounds__(RED_NT)
pcheb_res_sell_kernel(const int32_t* __restrict__ ecol, const double* __restrict__ eval,
                      const double* __restrict__ rin, const double* __restrict__ d,
                      double* __restrict__ rout, long long n, const int* __restrict__ done) {
  if (done && *done) return;
  for (long long i = blockIdx.x * (long long)RED_NT + threadIdx.x; i < n;
       i += (long long)gridDim.x * RED_NT) {
    const long long base = (i >> 5) * (32 * W) + (i & 31);
    double sd = 0.0;
#pragma unroll
    for (int k = 0; k < W; ++k) sd = fma(eval[base + 32 * k], d[ecol[base + 32 * k]], sd);
    rout[i] = rin[i] - sd;
  }
}

// d = c1 d + c2 t, y += d; `last` adds the partial <y, v>
__global__ void __launch_bounds__(RED_NT)
pcheb_upd_kernel(const double* __restrict__ t, double* __restrict__ d, double* __restrict__ y,
                 const double* __restrict__ v, double c1, double c2, long long n, int last,
                 double* part, const int* __restrict__ done) {
  if (done && *done) return;
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)RED_NT + threadIdx.x; i < n;
       i += (long long)gridDim.x * RED_NT) {
    const double dn = c1 * d[i] + c2 * t[i];
    d[i] = dn;
    const double yn = y[i] + dn;
    y[i] = yn;
    if (last) s = fma(yn, v[i], s);
  }
  if (last && part) {
    s = block_sum(s);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
  }
}

// 1 / (tau M~) once per handle (the (1,1) preconditioner block as a multiply, not a division)
__global__ void tau_minv_kernel(const double* __restrict__ mdiag, double tau, double* __restrict__ r,
                                long long n) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) r[i] = 1.0 / (tau * mdiag[i]);
}


__global__ void scale_minv_kernel(const double* __restrict__ v, const double* __restrict__ minv,
                                  double* __restrict__ z, long long n) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) z[i] = v[i] * minv[i];
}

__global__ void init_kernel(const double* glob, int P, MState* st, double rtol, int maxit) {
  if (threadIdx.x != 0) return;
  double g2 = rank_sum(glob, P);
  MState m{};
  m.rtol = rtol; m.maxit = maxit;
  m.gamma_old = 1.0; m.c = 1.0; m.c_old = 1.0; m.s = 0.0; m.s_old = 0.0;
  if (g2 < 0.0) { m.breakdown = 1; m.done = 1; }
  double g = std::sqrt(g2 > 0 ? g2 : 0.0);
  m.gamma = g; m.gamma1 = g; m.eta = g; m.rel = 1.0;
  if (g == 0.0 && !m.breakdown) { m.done = 1; m.conv = 1; m.rel = 0.0; }
  *st = m;
}

// one MINRES scalar step: Givens rotation from (delta, gamma_new),
// the w/x update coefficients, eta and the stopping test (done = 2: converged this iteration)
__device__ __forceinline__ MState scalar_step(MState m, double g2) {
  if (g2 < 0.0) { m.breakdown = 1; m.done = 1; return m; }
  const double gn = std::sqrt(g2);
  const double delta = m.delta, g = m.gamma;
  const double a0 = m.c * delta - m.c_old * m.s * g;
  const double a1 = hypot(a0, gn);
  const double a2 = m.s * delta + m.c_old * m.c * g;
  const double a3 = m.s_old * g;
  const double cn = a0 / a1, sn = gn / a1;
  m.wz = 1.0 / (g * a1);      // w_new = z/g/a1 - (a3/a1) w_old - (a2/a1) w
  m.wa3 = a3 / a1;
  m.wa2 = a2 / a1;
  m.xc = cn * m.eta;          // x += c_new eta w_new
  m.eta = -sn * m.eta;
  m.gamma_old = g; m.gamma = gn;
  m.c_old = m.c; m.c = cn;
  m.s_old = m.s; m.s = sn;
  m.iters += 1;
  m.rel = fabs(m.eta) / m.gamma1;
  if (fabs(m.eta) <= m.rtol * m.gamma1 || gn == 0.0) { m.conv = 1; m.done = 2; }
  else if (m.iters >= m.maxit) m.done = 2;
  return m;
}

// Fused end of an iteration: every block derives the new scalars from the old state S and
// gamma^2 (single rank: sum(pa) + sum(pb), summed here in the reduction kernel's order;
// multi-rank: the all-gathered scalars) — identical in every block — then
// w_new = wz z - wa3 w_old - wa2 w, x += xc w_new; block 0 publishes the new state in the
// OTHER state slot (double-buffered: no block can see a half-updated state), with done = 2
// (converged in this iteration, whose update still runs) latched to 1.
__global__ void __launch_bounds__(RED_NT)
wstep_kernel(const double* __restrict__ glob, int P, const MState* __restrict__ S,
             MState* __restrict__ Snext, const double* __restrict__ pa,
             const double* __restrict__ pb, int nb, const double* __restrict__ z,
             const double* __restrict__ w_old, const double* __restrict__ w,
             double* __restrict__ w_new, double* __restrict__ x, long long n) {
  __shared__ MState sm;
  if (S->done) {   // (done is 0 or 1 here) propagate the finished state
    if (blockIdx.x == 0 && threadIdx.x == 0) *Snext = *S;
    return;
  }
  double red = 0.0;
  if (pa) {
    const double a = sum_partials(pa, nb);
    const double b = sum_partials(pb, nb);
    red = a + b;
  }
  if (threadIdx.x == 0) sm = scalar_step(*S, pa ? red : rank_sum(glob, P));
  __syncthreads();
  const MState m = sm;
  // x += c_j eta_j w_j is applied two iterations at a time: an odd iteration only records its
  // coefficient (x is neither read nor written), the next one adds xcp w_{j-1} + xc w_j — w_{j-1}
  // is the `w` this pass reads anyway — so x streams through HBM every other iteration; a
  // finishing iteration (done = 2) always flushes
  const bool defer = (m.iters & 1) && m.done != 2;
  if (!m.breakdown) {
    const double wz = m.wz, wa3 = m.wa3, wa2 = m.wa2, xc = m.xc;
    if (defer) {
      for (long long i = blockIdx.x * (long long)RED_NT + threadIdx.x; i < n;
           i += (long long)gridDim.x * RED_NT)
        w_new[i] = wz * z[i] - wa3 * w_old[i] - wa2 * w[i];
    } else {
      const double xcp = m.pend ? m.xcp : 0.0;
      for (long long i = blockIdx.x * (long long)RED_NT + threadIdx.x; i < n;
           i += (long long)gridDim.x * RED_NT) {
        const double wi = w[i];
        const double wn = wz * z[i] - wa3 * w_old[i] - wa2 * wi;
        w_new[i] = wn;
        x[i] = fma(xc, wn, fma(xcp, wi, x[i]));
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    MState o = m;
    if (!o.breakdown) {
      o.pend = defer ? 1 : 0;
      o.xcp = defer ? m.xc : 0.0;
    }
    if (o.done == 2) o.done = 1;
    *Snext = o;
  }
}

// NEXT-3 orthogonalization after S^-1 (reading A21): partial sums of y, then
// y -= mean (the rank-ordered global sum / n) fused with the partial <y, v> MINRES needs
__global__ void __launch_bounds__(RED_NT)
sum_kernel(const double* __restrict__ y, long long n, double* __restrict__ part,
           const int* __restrict__ done) {
  if (done && *done) return;
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)RED_NT + threadIdx.x; i < n;
       i += (long long)gridDim.x * RED_NT)
    s += y[i];
  s = block_sum(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void __launch_bounds__(RED_NT)
mean_sub_kernel(double* __restrict__ y, long long n, const double* __restrict__ glob, int P,
                double inv_n, const double* __restrict__ v, double* __restrict__ part,
                const int* __restrict__ done) {
  if (done && *done) return;
  const double mean = rank_sum(glob, P) * inv_n;
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)RED_NT + threadIdx.x; i < n;
       i += (long long)gridDim.x * RED_NT) {
    const double t = y[i] - mean;
    y[i] = t;
    if (part) s = fma(t, v[i], s);
  }
  if (part) {
    s = block_sum(s);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
  }
}

inline unsigned nb(long long n, int nt) { return (unsigned)((n + nt - 1) / nt); }

}  // namespace

struct MinresWork {
  long long n = 0;
  int nb = 0;                      // reduction grid: min(RED_BLOCKS, ceil(n / RED_NT))
  double* buf = nullptr;           // all vectors
  double *v[3], *w[3], *z[2], *Az, *r, *d[2];
  double *part_a, *part_b, *part_c, *loc, *glob;
  double* mtinv = nullptr;         // 1 / (tau M~) [n_rt]
  double* part_t = nullptr;        // box kernel, one rank: per-tile partials of <A z, z>
  long long ntiles = 0;
  MState* st = nullptr;            // [2]: iteration j reads st[j & 1], publishes st[(j + 1) & 1]
  MState* st_host = nullptr;       // pinned
  cudaStream_t stream = nullptr;   // own non-blocking stream (graph capture needs one)
  std::vector<double> c1, c2;      // Chebyshev step constants
  double itheta = 0;
  long long ex_lo = 0, ex_hi = 0;  // RT range excluded from dots (replicated plane)
};

static hdiv_status ensure_work(hdiv_ctx* h) {
  if (h->mw) return HDIV_OK;
  auto* mw = new MinresWork();
  h->mw = mw;
  const long long n = h->nrt + h->nl2, nq = h->nl2;
  const long long lplane = (h->dim == 3) ? h->n[0] * h->n[1] : h->n[0];
  const long long nqg = nq + (h->nranks > 1 ? 2 * lplane : 0);   // + ghost layers
  mw->n = n;
  mw->nb = (int)std::max(1LL, std::min<long long>(RED_BLOCKS, (n + RED_NT - 1) / RED_NT));
  size_t tot = 9 * (size_t)n + (size_t)nq + 2 * (size_t)nqg + 3 * RED_BLOCKS + 2 + 2 * h->nranks;
  HDIV_CUDA_TRY(cudaMalloc(&mw->buf, tot * sizeof(double)));
  HDIV_CUDA_TRY(cudaMemset(mw->buf, 0, tot * sizeof(double)));
  double* p = mw->buf;
  for (int i = 0; i < 3; ++i) { mw->v[i] = p; p += n; }
  for (int i = 0; i < 3; ++i) { mw->w[i] = p; p += n; }
  for (int i = 0; i < 2; ++i) { mw->z[i] = p; p += n; }
  mw->Az = p; p += n;
  mw->r = p; p += nq;
  for (int i = 0; i < 2; ++i) { mw->d[i] = p; p += nqg; }
  mw->part_a = p; p += RED_BLOCKS;
  mw->part_b = p; p += RED_BLOCKS;
  mw->part_c = p; p += RED_BLOCKS;
  mw->loc = p; p += 2;
  mw->glob = (h->nranks > 1) ? p : mw->loc;
  p += 2 * h->nranks;
  if (h->rank > 0) {   // the lower rank owns the shared interface plane
    const int last = h->dim - 1;
    mw->ex_lo = h->off[last];
    mw->ex_hi = h->off[last] + lplane;
  }
  HDIV_CUDA_TRY(cudaMalloc(&mw->st, 2 * sizeof(MState)));
  if (h->kernel == 2 && h->nranks == 1) {   // <A z, z> fused into the block apply
    mw->ntiles = affine_num_tiles(h);
    HDIV_CUDA_TRY(cudaMalloc(&mw->part_t, sizeof(double) * mw->ntiles));
  }
  HDIV_CUDA_TRY(cudaMalloc(&mw->mtinv, sizeof(double) * (h->nrt > 0 ? h->nrt : 1)));
  tau_minv_kernel<<<nb(h->nrt, 256), 256>>>(h->d_mdiag, h->opts.tau, mw->mtinv, h->nrt);
  HDIV_CUDA_TRY(cudaGetLastError());
  HDIV_CUDA_TRY(cudaDeviceSynchronize());   // double-buffered (wstep_kernel)
  HDIV_CUDA_TRY(cudaMallocHost(&mw->st_host, sizeof(MState)));
  HDIV_CUDA_TRY(cudaStreamCreateWithFlags(&mw->stream, cudaStreamNonBlocking));
  // Chebyshev constants on [lmax/ratio, lmax], lmax = 2 (reading A10)
  const int k = h->opts.cheb_degree;
  const double lmax = 2.0, a = lmax / h->opts.cheb_ratio, b = lmax;
  const double theta = 0.5 * (a + b), delta = 0.5 * (b - a), sigma = theta / delta;
  double rho = 1.0 / sigma;
  mw->itheta = 1.0 / theta;
  for (int i = 1; i < k; ++i) {
    double rn = 1.0 / (2.0 * sigma - rho);
    mw->c1.push_back(rn * rho);
    mw->c2.push_back(2.0 * rn / delta);
    rho = rn;
  }
  return HDIV_OK;
}

void minres_free(hdiv_ctx* h) {
  if (!h->mw) return;
  cudaFree(h->mw->buf);
  cudaFree(h->mw->st);
  cudaFree(h->mw->mtinv);
  cudaFree(h->mw->part_t);
  cudaFreeHost(h->mw->st_host);
  if (h->mw->stream) cudaStreamDestroy(h->mw->stream);
  delete h->mw;
  h->mw = nullptr;
}

template <int Y0>
static cudaError_t cheb3c_y0(const hdiv_ctx* h, const CellGeo& g, const double* v, const double* ym1,
                             const double* ym2, double* yo, double c1, double c2, int last,
                             double* part, const int* done, cudaStream_t s) {
  const unsigned nbk = h->mw->nb;   // the reduction grid (the consumers sum nb partials)
  const double* di = h->d_sdinv;
  const double it = h->mw->itheta;
  switch (h->p) {
    case 1: cheb3c_kernel<1, Y0><<<nbk, RED_NT, 0, s>>>(g, v, ym1, ym2, di, it, yo, c1, c2, last, part, done); break;
    case 2: cheb3c_kernel<2, Y0><<<nbk, RED_NT, 0, s>>>(g, v, ym1, ym2, di, it, yo, c1, c2, last, part, done); break;
    case 3: cheb3c_kernel<3, Y0><<<nbk, RED_NT, 0, s>>>(g, v, ym1, ym2, di, it, yo, c1, c2, last, part, done); break;
    case 4: cheb3c_kernel<4, Y0><<<nbk, RED_NT, 0, s>>>(g, v, ym1, ym2, di, it, yo, c1, c2, last, part, done); break;
    case 5: cheb3c_kernel<5, Y0><<<nbk, RED_NT, 0, s>>>(g, v, ym1, ym2, di, it, yo, c1, c2, last, part, done); break;
    case 6: cheb3c_kernel<6, Y0><<<nbk, RED_NT, 0, s>>>(g, v, ym1, ym2, di, it, yo, c1, c2, last, part, done); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// step i of the recurrence through the cell stencil; y0: 1 = y_{i-1} is y_0 (formed on the fly),
// 2 = y_{i-2} is y_0, 0 = both stored
static cudaError_t launch_cheb3c(const hdiv_ctx* h, const double* v, const double* ym1,
                                 const double* ym2, double* yo, double c1, double c2, int last,
                                 double* part, const int* done, cudaStream_t s, int y0 = 0) {
  const CellGeo g = make_cellgeo(h);
  if (y0 == 1) return cheb3c_y0<1>(h, g, v, ym1, ym2, yo, c1, c2, last, part, done, s);
  if (y0 == 2) return cheb3c_y0<2>(h, g, v, ym1, ym2, yo, c1, c2, last, part, done, s);
  return cheb3c_y0<0>(h, g, v, ym1, ym2, yo, c1, c2, last, part, done, s);
}

static hdiv_status reduce_scalar(hdiv_ctx* h, const double* pa, const double* pb, const int* done,
                                 cudaStream_t s);

// Reading A9d: y = the degree-k Chebyshev polynomial in B S~ applied to vq (B = one V-cycle);
// d in mw->d[0] (ghost space for slabs), r in mw->d[1], t = B r in mw->r
static hdiv_status amg_cheb_apply(hdiv_ctx* h, const double* vq, double* y, double* part,
                                  const int* done, cudaStream_t s) {
  MinresWork* mw = h->mw;
  const long long n = h->nl2;
  const int k = h->opts.amg_cheb_degree;
  // spectrum of B S~: (0, 1] for one V-cycle, (0, 2] for the block-Jacobi over a chain of
  // slabs (two colours, oracle/amg.py) -> b = 1.1 / 2.2
  const double b = (h->nranks > 1) ? 2.2 : 1.1, a = b / h->opts.amg_cheb_ratio;
  const double theta = 0.5 * (b + a), delta = 0.5 * (b - a), sigma = theta / delta;
  double* d = mw->d[0];
  double* r = mw->d[1];
  double* t = mw->r;
  hdiv_status st = amg_vcycle(h, vq, t, done, s);
  if (st != HDIV_OK) return st;
  pcheb_first_kernel<<<mw->nb, RED_NT, 0, s>>>(t, 1.0 / theta, d, y, n, done);
  HDIV_CUDA_TRY(cudaGetLastError());
  double rho = 1.0 / sigma;
  for (int i = 1; i < k; ++i) {
    if (h->nranks > 1 && (st = comm_l2_ghosts(h, d, s)) != HDIV_OK) return st;
    const double* rin = (i == 1) ? vq : r;
    if (h->d_cw) {
      const CellGeo g = make_cellgeo(h);
      switch (h->p) {
        case 1: pcheb_res_cell_kernel<1><<<mw->nb, RED_NT, 0, s>>>(g, rin, d, r, done); break;
        case 2: pcheb_res_cell_kernel<2><<<mw->nb, RED_NT, 0, s>>>(g, rin, d, r, done); break;
        case 3: pcheb_res_cell_kernel<3><<<mw->nb, RED_NT, 0, s>>>(g, rin, d, r, done); break;
        case 4: pcheb_res_cell_kernel<4><<<mw->nb, RED_NT, 0, s>>>(g, rin, d, r, done); break;
        case 5: pcheb_res_cell_kernel<5><<<mw->nb, RED_NT, 0, s>>>(g, rin, d, r, done); break;
        case 6: pcheb_res_cell_kernel<6><<<mw->nb, RED_NT, 0, s>>>(g, rin, d, r, done); break;
        default: return HDIV_ERR_UNSUPPORTED;
      }
    } else {
      pcheb_res_sell_kernel<5><<<mw->nb, RED_NT, 0, s>>>(h->d_ecol, h->d_eval, rin, d, r, n, done);
    }
    HDIV_CUDA_TRY(cudaGetLastError());
    if ((st = amg_vcycle(h, r, t, done, s)) != HDIV_OK) return st;
    const double rn = 1.0 / (2.0 * sigma - rho);
    pcheb_upd_kernel<<<mw->nb, RED_NT, 0, s>>>(t, d, y, vq, rn * rho, 2.0 * rn / delta, n,
                                               i == k - 1, part, done);
    HDIV_CUDA_TRY(cudaGetLastError());
    rho = rn;
  }
  return HDIV_OK;
}

// the inner preconditioners of the A9e balancing form
static hdiv_status amg_poly_inner(hdiv_ctx* h, const double* b, double* x, const int* done,
                                  cudaStream_t s) {
  return amg_cheb_apply(h, b, x, nullptr, done, s);
}
static hdiv_status amg_vc_inner(hdiv_ctx* h, const double* b, double* x, const int* done,
                                cudaStream_t s) {
  return amg_vcycle(h, b, x, done, s);
}

// Chebyshev-Jacobi S^-1 applied to vq -> y (uses mw->r, mw->d); partial <y, vq> if part
static hdiv_status cheb_apply_raw(hdiv_ctx* h, const double* vq, double* y, double* part,
                                  const int* done, cudaStream_t s) {
  MinresWork* mw = h->mw;
  if (h->opts.schur_solver == HDIV_SCHUR_AMG && amg_has_global_coarse(h)) {
    // reading A9e: the balancing global coarse correction around the polynomial / V-cycles
    hdiv_status st = amg_global_apply(h, vq, y, done, s,
                                      h->opts.amg_cheb_degree >= 2 ? amg_poly_inner : amg_vc_inner);
    if (st != HDIV_OK) return st;
    if (part) {
      dot_kernel<<<h->mw->nb, RED_NT, 0, s>>>(y, vq, h->nl2, 0, 0, part, done);
      HDIV_CUDA_TRY(cudaGetLastError());
    }
    return HDIV_OK;
  }
  if (h->opts.schur_solver == HDIV_SCHUR_AMG && h->opts.amg_cheb_degree >= 2)
    return amg_cheb_apply(h, vq, y, part, done, s);
  if (h->opts.schur_solver == HDIV_SCHUR_AMG) {   // NEXT-1: one V-cycle
    if (part) {   // the partial <y, vq> fused into the last level-0 smoothing sweep
      hdiv_status st = amg_vcycle(h, vq, y, done, s, part, h->mw->nb);
      if (st == HDIV_OK) return HDIV_OK;
      if (st != HDIV_ERR_UNSUPPORTED) return st;
    }
    hdiv_status st = amg_vcycle(h, vq, y, done, s);
    if (st != HDIV_OK) return st;
    if (part) {
      dot_kernel<<<h->mw->nb, RED_NT, 0, s>>>(y, vq, h->nl2, 0, 0, part, done);
      HDIV_CUDA_TRY(cudaGetLastError());
    }
    return HDIV_OK;
  }
  const long long n = h->nl2;
  const int k = h->opts.cheb_degree;
  // three-term recurrence on the iterate: y_i in d[i & 1] (ghost space for slabs), the last
  // one straight into y; S~ y_{i-1} by the cell stencil (3D) or the SELL copy (2D)
  // one rank, cell stencil, degree >= 2: y_0 = D^-1 v / theta is never stored (steps 1 and 2
  // form it on the fly); otherwise the first term is written by its own pass
  // (A/B on one box, config 4: 17.83 -> 17.40 ms per MINRES iteration)
  const bool y0_fly = h->d_cw && h->nranks == 1 && k >= 2;
  if (!y0_fly) {
    cheb_first_kernel<<<h->mw->nb, RED_NT, 0, s>>>(vq, h->d_sdinv, mw->itheta, mw->d[0],
                                                    k == 1 ? y : mw->d[0], n, k == 1, part, done);
    HDIV_CUDA_TRY(cudaGetLastError());
  }
  for (int i = 1; i < k; ++i) {
    double* ym1 = mw->d[(i - 1) & 1];
    if (h->nranks > 1) {
      hdiv_status st = comm_l2_ghosts(h, ym1, s);
      if (st != HDIV_OK) return st;
    }
    double* yo = (i == k - 1) ? y : mw->d[i & 1];
    const double* ym2 = (i == 1) ? nullptr : mw->d[i & 1];
    if (h->d_cw) {
      const int y0 = y0_fly ? (i == 1 ? 1 : i == 2 ? 2 : 0) : 0;
      HDIV_CUDA_TRY(launch_cheb3c(h, vq, ym1, ym2, yo, mw->c1[i - 1], mw->c2[i - 1], i == k - 1,
                                  part, done, s, y0));
    } else {
      cheb3_kernel<5><<<h->mw->nb, RED_NT, 0, s>>>(h->d_ecol, h->d_eval, vq, ym1, ym2, h->d_sdinv,
                                                    yo, mw->c1[i - 1], mw->c2[i - 1], n, i == k - 1,
                                                    part, done);
      HDIV_CUDA_TRY(cudaGetLastError());
    }
  }
  return HDIV_OK;
}

// S^-1 (Chebyshev or AMG) followed, with options.project_mean, by the orthogonalization step
// of P:1038-1040; the partial <y, vq> is taken after the projection
static hdiv_status cheb_apply(hdiv_ctx* h, const double* vq, double* y, double* part,
                              const int* done, cudaStream_t s) {
  if (!h->opts.project_mean) return cheb_apply_raw(h, vq, y, part, done, s);
  MinresWork* mw = h->mw;
  hdiv_status st = cheb_apply_raw(h, vq, y, nullptr, done, s);
  if (st != HDIV_OK) return st;
  sum_kernel<<<h->mw->nb, RED_NT, 0, s>>>(y, h->nl2, mw->part_b, done);
  HDIV_CUDA_TRY(cudaGetLastError());
  if ((st = reduce_scalar(h, mw->part_b, nullptr, done, s)) != HDIV_OK) return st;
  mean_sub_kernel<<<h->mw->nb, RED_NT, 0, s>>>(y, h->nl2, mw->glob, h->nranks,
                                                1.0 / (double)h->nl2_g, vq, part, done);
  HDIV_CUDA_TRY(cudaGetLastError());
  return HDIV_OK;
}

hdiv_status apply_precond(hdiv_ctx* h, const double* v, double* z, cudaStream_t s) {
  hdiv_status st = ensure_work(h);
  if (st != HDIV_OK) return st;
  scale_minv_kernel<<<nb(h->nrt, 256), 256, 0, s>>>(v, h->mw->mtinv, z, h->nrt);
  HDIV_CUDA_TRY(cudaGetLastError());
  return cheb_apply(h, v + h->nrt, z + h->nrt, nullptr, nullptr, s);
}

// y = S^-1 vq (Chebyshev or AMG per options), for other solvers (GMRES)
hdiv_status schur_inv_apply(hdiv_ctx* h, const double* vq, double* y, cudaStream_t s) {
  hdiv_status st = ensure_work(h);
  if (st != HDIV_OK) return st;
  return cheb_apply(h, vq, y, nullptr, nullptr, s);
}

// local scalar -> (all-gather) -> glob
static hdiv_status reduce_scalar(hdiv_ctx* h, const double* pa, const double* pb, const int* done,
                                 cudaStream_t s) {
  MinresWork* mw = h->mw;
  local_reduce_kernel<<<1, RED_NT, 0, s>>>(pa, pb, mw->loc, done, mw->nb);
  HDIV_CUDA_TRY(cudaGetLastError());
  if (h->nranks > 1) return comm_allgather(h, mw->loc, mw->glob, 1, s);
  return HDIV_OK;
}

hdiv_status minres(hdiv_ctx* h, const double* b, double* x, double rtol, int maxit,
                   hdiv_report* rep, cudaStream_t caller) {
  hdiv_status stt = ensure_work(h);
  if (stt != HDIV_OK) return stt;
  MinresWork* mw = h->mw;
  const long long n = mw->n, nrt = h->nrt;
  // state slots: init writes st[1]; iteration j (1..6 per graph launch) reads st[j & 1] and
  // publishes st[(j + 1) & 1], so after every 6 iterations the latest state is in st[1]
  MState* const st_last = mw->st + 1;
  const int P = h->nranks;
  // the solve runs on the handle's own (capturable) stream, ordered after `caller`
  cudaStream_t s = mw->stream;
  cudaEvent_t e0, e1;
  HDIV_CUDA_TRY(cudaEventCreate(&e0));
  HDIV_CUDA_TRY(cudaEventCreate(&e1));
  HDIV_CUDA_TRY(cudaEventRecord(e0, caller));
  HDIV_CUDA_TRY(cudaStreamWaitEvent(s, e0, 0));
  HDIV_CUDA_TRY(cudaEventRecord(e0, s));
  // x0 = 0, v0 = 0 (v_old), w0 = w1 = 0, v1 = b, z1 = P^-1 v1, gamma1 = sqrt(<z1, v1>)
  HDIV_CUDA_TRY(cudaMemsetAsync(x, 0, n * sizeof(double), s));
  HDIV_CUDA_TRY(cudaMemsetAsync(mw->v[0], 0, n * sizeof(double), s));
  HDIV_CUDA_TRY(cudaMemsetAsync(mw->w[0], 0, n * sizeof(double), s));
  HDIV_CUDA_TRY(cudaMemsetAsync(mw->w[1], 0, n * sizeof(double), s));
  HDIV_CUDA_TRY(cudaMemcpyAsync(mw->v[1], b, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  scale_minv_kernel<<<nb(nrt, 256), 256, 0, s>>>(mw->v[1], mw->mtinv, mw->z[0], nrt);
  dot_kernel<<<h->mw->nb, RED_NT, 0, s>>>(mw->z[0], mw->v[1], nrt, mw->ex_lo, mw->ex_hi,
                                           mw->part_a, nullptr);
  HDIV_CUDA_TRY(cudaGetLastError());
  if ((stt = cheb_apply(h, mw->v[1] + nrt, mw->z[0] + nrt, mw->part_b, nullptr, s)) != HDIV_OK)
    return stt;
  if ((stt = reduce_scalar(h, mw->part_a, mw->part_b, nullptr, s)) != HDIV_OK) return stt;
  init_kernel<<<1, 32, 0, s>>>(mw->glob, P, st_last, rtol, maxit);
  HDIV_CUDA_TRY(cudaGetLastError());

  // iteration j: (v_old, v, v_new) = v[(j-1)%3], v[j%3], v[(j+1)%3]; same for w;
  //              (z, z_new) = z[(j-1)%2], z[j%2]
  auto iteration = [&](int j) -> hdiv_status {
    double* vo = mw->v[(j + 2) % 3];
    double* vc = mw->v[j % 3];
    double* vn = mw->v[(j + 1) % 3];
    double* wo = mw->w[(j + 2) % 3];
    double* wc = mw->w[j % 3];
    double* wn = mw->w[(j + 1) % 3];
    double* zc = mw->z[(j + 1) % 2];
    double* zn = mw->z[j % 2];
    MState* stc = mw->st + (j & 1);
    MState* stn = mw->st + ((j + 1) & 1);
    const int* done = &stc->done;
    const bool one = (P == 1);
    hdiv_status st = HDIV_OK;
    const double* dpart = nullptr;   // vupd sums these nb partials itself (single rank)
    if (mw->part_t) {
      // box kernel, one rank: <A z, z> fused into the block apply (one partial per tile, summed
      // in tile order) — the separate pass over A z and z is saved
      HDIV_CUDA_TRY(launch_affine_apply_dot(h, zc, mw->Az, done, mw->part_t, s));
      local_reduce_kernel<<<1, RED_NT, 0, s>>>(mw->part_t, nullptr, mw->loc, done, (int)mw->ntiles);
      HDIV_CUDA_TRY(cudaGetLastError());
    } else {
      HDIV_CUDA_TRY(apply_block_dev(h, zc, mw->Az, done, s));
      // single rank: the consumers (vupd, scalar) sum the partials themselves — two launches
      // fewer per iteration; multi-rank: local reduction + all-gather as before
      dot_kernel<<<h->mw->nb, RED_NT, 0, s>>>(mw->Az, zc, n, mw->ex_lo, mw->ex_hi, mw->part_c,
                                               done);
      HDIV_CUDA_TRY(cudaGetLastError());
      if (!one && (st = reduce_scalar(h, mw->part_c, nullptr, done, s)) != HDIV_OK) return st;
      if (one) dpart = mw->part_c;
    }
    vupd_kernel<<<h->mw->nb, RED_NT, 0, s>>>(mw->Az, vc, vo, vn, zn, mw->mtinv, h->opts.tau,
                                              nrt, n, mw->ex_lo, mw->ex_hi, stc, mw->glob, P,
                                              dpart, mw->nb, mw->part_a);
    HDIV_CUDA_TRY(cudaGetLastError());
    if ((st = cheb_apply(h, vn + nrt, zn + nrt, mw->part_b, done, s)) != HDIV_OK) return st;
    if (!one && (st = reduce_scalar(h, mw->part_a, mw->part_b, done, s)) != HDIV_OK) return st;
    wstep_kernel<<<h->mw->nb, RED_NT, 0, s>>>(mw->glob, P, stc, stn, one ? mw->part_a : nullptr,
                                              mw->part_b, mw->nb, zc, wo, wc, wn, x, n);
    HDIV_CUDA_TRY(cudaGetLastError());
    return HDIV_OK;
  };
  // capture 6 iterations (the buffer pattern repeats with period 6)
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  // (the loopback test communicator meets its peers at host barriers: no graph capture)
  bool use_graph = !comm_is_loopback(h);
  if (!use_graph || cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    use_graph = false;
    cudaGetLastError();
  } else {
    hdiv_status e = HDIV_OK;
    for (int j = 1; j <= 6 && e == HDIV_OK; ++j) e = iteration(j);
    cudaError_t ec = cudaStreamEndCapture(s, &graph);
    if (e != HDIV_OK || ec != cudaSuccess || cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) {
      use_graph = false;
      cudaGetLastError();
      if (graph) cudaGraphDestroy(graph);
      graph = nullptr;
      exec = nullptr;
    }
  }
  int launched = 0;
  for (;;) {
    if (use_graph) {
      HDIV_CUDA_TRY(cudaGraphLaunch(exec, s));
    } else {
      for (int j = 1; j <= 6; ++j) {
        hdiv_status e = iteration(j);
        if (e != HDIV_OK) return e;
      }
    }
    launched += 6;
    HDIV_CUDA_TRY(cudaMemcpyAsync(mw->st_host, st_last, sizeof(MState), cudaMemcpyDeviceToHost, s));
    if (hdiv_status e = comm_sync(h, s); e != HDIV_OK) return e;
    if (mw->st_host->done || launched >= maxit + 6) break;
  }
  HDIV_CUDA_TRY(cudaEventRecord(e1, s));
  HDIV_CUDA_TRY(cudaStreamWaitEvent(caller, e1, 0));
  HDIV_CUDA_TRY(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (exec) cudaGraphExecDestroy(exec);
  if (graph) cudaGraphDestroy(graph);
  MState m = *mw->st_host;
  if (rep) {
    rep->iters = m.iters;
    rep->converged = m.conv;
    rep->rel_resid = m.rel;
    rep->t_solve_ms = ms;
  }
  if (m.breakdown) {
    set_error("MINRES breakdown: <z, v> < 0");
    return HDIV_ERR_BREAKDOWN;
  }
  return HDIV_OK;
}

}  // namespace hdiv
