// gmres.cu — NEXT-4: block upper-triangular preconditioner + right-preconditioned GMRES(m).
//
// P:423-438 Remark: B = [M, B^T; 0, S] gives sigma(B^-1 A) = {1} with a degree-2 minimal
// polynomial, so GMRES converges in at most two iterations with exact blocks; in practice the
// diagonal blocks are replaced by tau M~ and S^ (the same M~ and S^-1 as the MINRES
// preconditioner, options.schur_solver).  With this build's A = [M, D^T; D, -Z] the Schur
// complement is -S, so  B = [tau M~, D^T; 0, -S^]  and
//     B^-1 v:  z_q = -S^-1 v_q ,  z_u = (tau M~)^-1 (v_u - D^T z_q).
// GMRES(m) (Saad Alg. 9.5, right preconditioning: the least-squares residual is the true
// residual), x0 = 0, Arnoldi with classical Gram-Schmidt applied twice; the (m+1)-vector
// projections are ONE pass over w and the basis (per-thread partial sums for every basis
// vector, fixed-order reductions), the update one pass; the tiny Hessenberg / Givens algebra
// runs on the host between the device passes (identical arithmetic to oracle/solvers.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "internal.h"

namespace hdiv {

hdiv_status comm_reverse_add(hdiv_ctx* h, double* y_rt, cudaStream_t s);   // comm.cu
hdiv_status comm_allgather(hdiv_ctx* h, const double* loc, double* glob, int k, cudaStream_t s);

constexpr int GMAX = 64;   // maximum restart length

struct GmresWork {
  long long n = 0;
  int m = 0;
  double* V = nullptr;      // (m+1) x n basis
  double* w = nullptr;
  double* t = nullptr;      // B^-1 V_j and the final correction
  double* tq = nullptr;     // S^-1 scratch (n_l2) and D^T scratch (n_rt)
  double* tu = nullptr;
  double* part = nullptr;   // [GMAX+1][GBLK] partial sums
  double* hd = nullptr;     // device copy of the projection coefficients
  double* glob = nullptr;   // multi-rank: all-gathered per-rank projections [P][GMAX+1]
  long long ex_lo = 0, ex_hi = 0;   // RT range excluded from dots (replicated interface plane)
  std::vector<double> hh;   // host
  std::vector<double> hg;   // host copy of glob
};

namespace {

constexpr int GNT = 256;
constexpr int GBLK = 148 * 4;
constexpr int KB = 8;       // basis vectors per projection pass (register tile)

__device__ __forceinline__ double gblock_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  if (l == 0) red[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x < 32) {
    r = (l < GNT / 32) ? red[l] : 0.0;
    for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
  }
  __syncthreads();
  return r;
}

// part[k][blk] = partial <V_{k0+k}, w> for k < nk (<= KB), entries [ex_lo, ex_hi) excluded
// (multi-rank: the interface plane replicated on the upper rank counts once)
__global__ void __launch_bounds__(GNT) proj_kernel(const double* __restrict__ V, long long n,
                                                   int k0, int nk, const double* __restrict__ w,
                                                   double* __restrict__ part, long long ex_lo,
                                                   long long ex_hi) {
  __shared__ double red[GNT / 32];
  double s[KB];
#pragma unroll
  for (int k = 0; k < KB; ++k) s[k] = 0.0;
  for (long long i = blockIdx.x * (long long)GNT + threadIdx.x; i < n;
       i += (long long)gridDim.x * GNT) {
    const double wi = (i >= ex_lo && i < ex_hi) ? 0.0 : w[i];
#pragma unroll
    for (int k = 0; k < KB; ++k)
      if (k < nk) s[k] = fma(V[(long long)(k0 + k) * n + i], wi, s[k]);
  }
#pragma unroll
  for (int k = 0; k < KB; ++k) {
    if (k >= nk) break;
    const double r = gblock_sum(s[k], red);
    if (threadIdx.x == 0) part[(long long)(k0 + k) * GBLK + blockIdx.x] = r;
  }
}

// out[k] = sum_blk part[k][blk] (fixed order), k < nk
__global__ void __launch_bounds__(GNT) proj_final_kernel(const double* __restrict__ part, int nk,
                                                         double* __restrict__ out) {
  __shared__ double red[GNT / 32];
  for (int k = 0; k < nk; ++k) {
    double s = 0.0;
    for (int i = threadIdx.x; i < GBLK; i += GNT) s += part[(long long)k * GBLK + i];
    s = gblock_sum(s, red);
    if (threadIdx.x == 0) out[k] = s;
  }
}

// w -= sum_{k<nk} h[k] V_k   (sign = -1)   or   t = sum_k h[k] V_k (sign = 0: overwrite)
__global__ void __launch_bounds__(GNT) combo_kernel(const double* __restrict__ V, long long n,
                                                    int nk, const double* __restrict__ h,
                                                    double* __restrict__ w, int overwrite) {
  for (long long i = blockIdx.x * (long long)GNT + threadIdx.x; i < n;
       i += (long long)gridDim.x * GNT) {
    double s = 0.0;
    for (int k = 0; k < nk; ++k) s = fma(h[k], V[(long long)k * n + i], s);
    w[i] = overwrite ? s : w[i] - s;
  }
}

__global__ void scale_copy_kernel(const double* __restrict__ a, double c, double* __restrict__ b,
                                  long long n) {
  for (long long i = blockIdx.x * (long long)GNT + threadIdx.x; i < n;
       i += (long long)gridDim.x * GNT)
    b[i] = c * a[i];
}

__global__ void sub_kernel(const double* __restrict__ b, const double* __restrict__ ax,
                           double* __restrict__ r, long long n) {
  for (long long i = blockIdx.x * (long long)GNT + threadIdx.x; i < n;
       i += (long long)gridDim.x * GNT)
    r[i] = b[i] - ax[i];
}

__global__ void axpy_kernel(const double* __restrict__ z, double* __restrict__ x, long long n) {
  for (long long i = blockIdx.x * (long long)GNT + threadIdx.x; i < n;
       i += (long long)gridDim.x * GNT)
    x[i] += z[i];
}

// z_u = (v_u + t_u) / (tau M~) with t_u = D^T y ; z_q = -y
__global__ void tri_u_kernel(const double* __restrict__ vu, const double* __restrict__ tu,
                             const double* __restrict__ mdiag, double tau, double* __restrict__ zu,
                             long long nrt) {
  for (long long i = blockIdx.x * (long long)GNT + threadIdx.x; i < nrt;
       i += (long long)gridDim.x * GNT)
    zu[i] = (vu[i] + tu[i]) / (tau * mdiag[i]);
}

__global__ void neg_kernel(const double* __restrict__ y, double* __restrict__ z, long long n) {
  for (long long i = blockIdx.x * (long long)GNT + threadIdx.x; i < n;
       i += (long long)gridDim.x * GNT)
    z[i] = -y[i];
}

}  // namespace

void gmres_free(hdiv_ctx* h) {
  if (!h->gw) return;
  cudaFree(h->gw->V); cudaFree(h->gw->w); cudaFree(h->gw->t); cudaFree(h->gw->tq);
  cudaFree(h->gw->tu); cudaFree(h->gw->part); cudaFree(h->gw->hd); cudaFree(h->gw->glob);
  delete h->gw;
  h->gw = nullptr;
}

static hdiv_status ensure_gw(hdiv_ctx* h, int m) {
  if (h->gw && h->gw->m >= m) return HDIV_OK;
  gmres_free(h);
  auto* g = new GmresWork();
  h->gw = g;
  g->n = h->nrt + h->nl2;
  g->m = m;
  HDIV_CUDA_TRY(cudaMalloc(&g->V, sizeof(double) * (size_t)(m + 1) * g->n));
  HDIV_CUDA_TRY(cudaMalloc(&g->w, sizeof(double) * g->n));
  HDIV_CUDA_TRY(cudaMalloc(&g->t, sizeof(double) * g->n));
  HDIV_CUDA_TRY(cudaMalloc(&g->tq, sizeof(double) * (h->nl2 > 0 ? h->nl2 : 1)));
  HDIV_CUDA_TRY(cudaMalloc(&g->tu, sizeof(double) * (h->nrt > 0 ? h->nrt : 1)));
  HDIV_CUDA_TRY(cudaMalloc(&g->part, sizeof(double) * (GMAX + 1) * GBLK));
  HDIV_CUDA_TRY(cudaMalloc(&g->hd, sizeof(double) * (GMAX + 1)));
  HDIV_CUDA_TRY(cudaMalloc(&g->glob, sizeof(double) * (GMAX + 1) * h->nranks));
  g->hh.resize(GMAX + 1);
  g->hg.resize((size_t)(GMAX + 1) * h->nranks);
  if (h->rank > 0) {   // the lower rank owns the shared interface plane
    const int last = h->dim - 1;
    const long long lplane = (h->dim == 3) ? h->n[0] * h->n[1] : h->n[0];
    g->ex_lo = h->off[last];
    g->ex_hi = h->off[last] + lplane;
  }
  return HDIV_OK;
}

hdiv_status apply_precond_tri(hdiv_ctx* h, const double* v, double* z, cudaStream_t s) {
  hdiv_status st = ensure_gw(h, h->gw ? h->gw->m : 1);
  if (st != HDIV_OK) return st;
  GmresWork* g = h->gw;
  // y = S^-1 v_q ; t_u = D^T y ; z_u = (v_u + t_u)/(tau M~) ; z_q = -y
  st = schur_inv_apply(h, v + h->nrt, g->tq, s);
  if (st != HDIV_OK) return st;
  HDIV_CUDA_TRY(launch_divT(h, g->tq, g->tu, s));
  if (h->nranks > 1 && (st = comm_reverse_add(h, g->tu, s)) != HDIV_OK) return st;
  tri_u_kernel<<<GBLK, GNT, 0, s>>>(v, g->tu, h->d_mdiag, h->opts.tau, z, h->nrt);
  neg_kernel<<<GBLK, GNT, 0, s>>>(g->tq, z + h->nrt, h->nl2);
  HDIV_CUDA_TRY(cudaGetLastError());
  return HDIV_OK;
}

// the nk projections in g->hd (this rank's) -> global values on the host: multi-rank, the P
// per-rank vectors are all-gathered and summed in rank order (identical on every rank)
static hdiv_status global_proj(hdiv_ctx* h, int nk, double* out, cudaStream_t s) {
  GmresWork* g = h->gw;
  if (h->nranks == 1) {
    HDIV_CUDA_TRY(cudaMemcpyAsync(out, g->hd, sizeof(double) * nk, cudaMemcpyDeviceToHost, s));
    HDIV_CUDA_TRY(cudaStreamSynchronize(s));
    return HDIV_OK;
  }
  hdiv_status st = comm_allgather(h, g->hd, g->glob, nk, s);
  if (st != HDIV_OK) return st;
  HDIV_CUDA_TRY(cudaMemcpyAsync(g->hg.data(), g->glob, sizeof(double) * nk * h->nranks,
                                cudaMemcpyDeviceToHost, s));
  if ((st = comm_sync(h, s)) != HDIV_OK) return st;
  for (int k = 0; k < nk; ++k) {
    double v = 0.0;
    for (int r = 0; r < h->nranks; ++r) v += g->hg[(size_t)r * nk + k];
    out[k] = v;
  }
  return HDIV_OK;
}

// <a,b> over the whole (global) vector (deterministic), via the projection kernels with V = a
static hdiv_status dot_host(hdiv_ctx* h, const double* a, const double* b, long long n,
                            double* out, cudaStream_t s) {
  GmresWork* g = h->gw;
  proj_kernel<<<GBLK, GNT, 0, s>>>(a, n, 0, 1, b, g->part, g->ex_lo, g->ex_hi);
  proj_final_kernel<<<1, GNT, 0, s>>>(g->part, 1, g->hd);
  HDIV_CUDA_TRY(cudaGetLastError());
  return global_proj(h, 1, out, s);
}

hdiv_status gmres(hdiv_ctx* h, const double* b, double* x, double rtol, int maxit, int restart,
                  hdiv_report* rep, cudaStream_t s) {
  const int m = std::max(1, std::min(restart, GMAX));
  hdiv_status st = ensure_gw(h, m);
  if (st != HDIV_OK) return st;
  GmresWork* g = h->gw;
  const long long n = g->n;
  cudaEvent_t e0, e1;
  HDIV_CUDA_TRY(cudaEventCreate(&e0));
  HDIV_CUDA_TRY(cudaEventCreate(&e1));
  HDIV_CUDA_TRY(cudaEventRecord(e0, s));
  HDIV_CUDA_TRY(cudaMemsetAsync(x, 0, sizeof(double) * n, s));
  double bb = 0.0;
  if ((st = dot_host(h, b, b, n, &bb, s)) != HDIV_OK) return st;
  const double bnorm = std::sqrt(bb);
  int it = 0;
  bool conv = (bnorm == 0.0);
  double rel = conv ? 0.0 : 1.0;
  std::vector<double> H((m + 1) * m), cs(m), sn(m), gv(m + 1), y(m);
  auto Hij = [&](int i, int j) -> double& { return H[(size_t)i * m + j]; };
  while (!conv && it < maxit) {
    // r = b - A x ; V_0 = r / ||r||
    HDIV_CUDA_TRY(apply_block_dev(h, x, g->w, nullptr, s));
    sub_kernel<<<GBLK, GNT, 0, s>>>(b, g->w, g->w, n);
    double rr = 0.0;
    if ((st = dot_host(h, g->w, g->w, n, &rr, s)) != HDIV_OK) return st;
    const double beta = std::sqrt(rr);
    rel = beta / bnorm;
    if (beta <= rtol * bnorm) { conv = true; break; }
    scale_copy_kernel<<<GBLK, GNT, 0, s>>>(g->w, 1.0 / beta, g->V, n);
    std::fill(H.begin(), H.end(), 0.0);
    std::fill(gv.begin(), gv.end(), 0.0);
    gv[0] = beta;
    int k = 0;
    for (int j = 0; j < m; ++j) {
      // w = A B^-1 V_j
      if ((st = apply_precond_tri(h, g->V + (size_t)j * n, g->t, s)) != HDIV_OK) return st;
      HDIV_CUDA_TRY(apply_block_dev(h, g->t, g->w, nullptr, s));
      for (int pass = 0; pass < 2; ++pass) {   // classical Gram-Schmidt, twice
        for (int k0 = 0; k0 <= j; k0 += KB)
          proj_kernel<<<GBLK, GNT, 0, s>>>(g->V, n, k0, std::min(KB, j + 1 - k0), g->w, g->part,
                                           g->ex_lo, g->ex_hi);
        proj_final_kernel<<<1, GNT, 0, s>>>(g->part, j + 1, g->hd);
        HDIV_CUDA_TRY(cudaGetLastError());
        if ((st = global_proj(h, j + 1, g->hh.data(), s)) != HDIV_OK) return st;
        if (h->nranks > 1)   // the global projections back to the device for the update
          HDIV_CUDA_TRY(cudaMemcpyAsync(g->hd, g->hh.data(), sizeof(double) * (j + 1),
                                        cudaMemcpyHostToDevice, s));
        combo_kernel<<<GBLK, GNT, 0, s>>>(g->V, n, j + 1, g->hd, g->w, 0);
        HDIV_CUDA_TRY(cudaGetLastError());
        for (int i = 0; i <= j; ++i) Hij(i, j) += g->hh[i];
      }
      double ww = 0.0;
      if ((st = dot_host(h, g->w, g->w, n, &ww, s)) != HDIV_OK) return st;
      Hij(j + 1, j) = std::sqrt(ww);
      if (Hij(j + 1, j) > 0.0)
        scale_copy_kernel<<<GBLK, GNT, 0, s>>>(g->w, 1.0 / Hij(j + 1, j), g->V + (size_t)(j + 1) * n, n);
      for (int i = 0; i < j; ++i) {   // previous rotations
        const double t = cs[i] * Hij(i, j) + sn[i] * Hij(i + 1, j);
        Hij(i + 1, j) = -sn[i] * Hij(i, j) + cs[i] * Hij(i + 1, j);
        Hij(i, j) = t;
      }
      const double den = std::hypot(Hij(j, j), Hij(j + 1, j));
      cs[j] = Hij(j, j) / den;
      sn[j] = Hij(j + 1, j) / den;
      Hij(j, j) = den;
      Hij(j + 1, j) = 0.0;
      gv[j + 1] = -sn[j] * gv[j];
      gv[j] = cs[j] * gv[j];
      ++it;
      k = j + 1;
      rel = std::fabs(gv[j + 1]) / bnorm;
      if (std::fabs(gv[j + 1]) <= rtol * bnorm || it >= maxit) {
        conv = std::fabs(gv[j + 1]) <= rtol * bnorm;
        break;
      }
    }
    // x += B^-1 V_k y, H y = g (back substitution on the host)
    for (int i = k - 1; i >= 0; --i) {
      double v = gv[i];
      for (int c = i + 1; c < k; ++c) v -= Hij(i, c) * y[c];
      y[i] = v / Hij(i, i);
    }
    HDIV_CUDA_TRY(cudaMemcpyAsync(g->hd, y.data(), sizeof(double) * k, cudaMemcpyHostToDevice, s));
    combo_kernel<<<GBLK, GNT, 0, s>>>(g->V, n, k, g->hd, g->w, 1);
    if ((st = apply_precond_tri(h, g->w, g->t, s)) != HDIV_OK) return st;
    axpy_kernel<<<GBLK, GNT, 0, s>>>(g->t, x, n);
    HDIV_CUDA_TRY(cudaGetLastError());
    HDIV_CUDA_TRY(cudaStreamSynchronize(s));
  }
  HDIV_CUDA_TRY(cudaEventRecord(e1, s));
  HDIV_CUDA_TRY(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (rep) {
    rep->iters = it;
    rep->converged = conv ? 1 : 0;
    rep->rel_resid = rel;
    rep->t_solve_ms = ms;
  }
  return HDIV_OK;
}

}  // namespace hdiv
