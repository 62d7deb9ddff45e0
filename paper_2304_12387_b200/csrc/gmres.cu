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
// vector, fixed-order reductions), the update one pass.  The tiny Hessenberg / Givens algebra
// runs on the device too (one-thread kernels on a device-resident state, the arithmetic of
// oracle/solvers.py): the host launches a whole restart cycle without waiting and reads the
// state once per cycle; a converged state turns the rest of the cycle's scalar updates into
// no-ops (the basis passes after it are wasted but harmless).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
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
  struct GState* st = nullptr;   // device-resident Hessenberg / Givens state
  struct GState* st_host = nullptr;   // pinned copy (read once per restart cycle)
  int* flags = nullptr;             // pinned: cycle_done after each Arnoldi step
  cudaEvent_t ev[GMAX] = {};        // ... and its completion
};

// device state of one GMRES(m) cycle (column-major H: H[i + (GMAX + 1) j])
struct GState {
  double H[(GMAX + 1) * GMAX];
  double cs[GMAX], sn[GMAX], gv[GMAX + 1], y[GMAX];
  double bnorm, rtol, rel, inv;   // inv: the scale of the next basis vector (0: none)
  int it, maxit, k, conv, done, cycle_done, pad[2];
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
                                                    double* __restrict__ w, int overwrite,
                                                    const int* __restrict__ nkp = nullptr) {
  if (nkp) nk = *nkp;   // the device state's basis size (vectors beyond it may be stale)
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

// multi-rank: the all-gathered per-rank values [P][nk] summed in rank order (identical on
// every rank) -> out[nk]
__global__ void rank_sum_kernel(const double* __restrict__ glob, int P, int nk, double* out) {
  const int k = threadIdx.x;
  if (k >= nk) return;
  double v = 0.0;
  for (int r = 0; r < P; ++r) v += glob[(size_t)r * nk + k];
  out[k] = v;
}

// cycle start: beta = ||r|| from hd[0]; converged (or the iteration budget spent) -> done
__global__ void g_start_kernel(GState* st, const double* __restrict__ hd) {
  GState& g = *st;
  const double beta = sqrt(hd[0]);
  for (int i = 0; i < (GMAX + 1) * GMAX; ++i) g.H[i] = 0.0;
  for (int i = 0; i <= GMAX; ++i) g.gv[i] = 0.0;
  g.gv[0] = beta;
  g.k = 0;
  g.cycle_done = 0;
  g.rel = beta / g.bnorm;
  if (beta <= g.rtol * g.bnorm) { g.conv = 1; g.done = 1; }
  if (g.it >= g.maxit) g.done = 1;
  g.inv = g.done ? 0.0 : 1.0 / beta;
}

// H(0..j, j) += hd[0..j]   (one classical Gram-Schmidt pass)
__global__ void g_hcol_kernel(GState* st, const double* __restrict__ hd, int j) {
  GState& g = *st;
  if (g.done || g.cycle_done) return;
  for (int i = 0; i <= j; ++i) g.H[i + (GMAX + 1) * j] += hd[i];
}

// after the two passes: H(j+1, j) = ||w|| (hd[0]), the previous rotations on column j, the new
// rotation, the residual estimate and the stopping test; inv = 1 / H(j+1, j) for V_{j+1}
__global__ void g_step_kernel(GState* st, const double* __restrict__ hd, int j, int m) {
  GState& g = *st;
  if (g.done || g.cycle_done) { g.inv = 0.0; return; }
  double* H = g.H;
  auto Hij = [&](int i, int c) -> double& { return H[i + (GMAX + 1) * c]; };
  Hij(j + 1, j) = sqrt(hd[0]);
  g.inv = Hij(j + 1, j) > 0.0 ? 1.0 / Hij(j + 1, j) : 0.0;
  for (int i = 0; i < j; ++i) {   // previous rotations
    const double t = g.cs[i] * Hij(i, j) + g.sn[i] * Hij(i + 1, j);
    Hij(i + 1, j) = -g.sn[i] * Hij(i, j) + g.cs[i] * Hij(i + 1, j);
    Hij(i, j) = t;
  }
  const double den = hypot(Hij(j, j), Hij(j + 1, j));
  g.cs[j] = Hij(j, j) / den;
  g.sn[j] = Hij(j + 1, j) / den;
  Hij(j, j) = den;
  Hij(j + 1, j) = 0.0;
  g.gv[j + 1] = -g.sn[j] * g.gv[j];
  g.gv[j] = g.cs[j] * g.gv[j];
  g.it += 1;
  g.k = j + 1;
  g.rel = fabs(g.gv[j + 1]) / g.bnorm;
  if (fabs(g.gv[j + 1]) <= g.rtol * g.bnorm) { g.conv = 1; g.cycle_done = 1; }
  else if (g.it >= g.maxit || j + 1 == m) g.cycle_done = 1;
}

// back substitution H y = g on the k x k triangle -> y into out[0..k) (coefficients of V)
__global__ void g_solve_kernel(GState* st, double* out) {
  GState& g = *st;
  const int k = g.k;
  for (int i = k - 1; i >= 0; --i) {
    double v = g.gv[i];
    for (int c = i + 1; c < k; ++c) v -= g.H[i + (GMAX + 1) * c] * g.y[c];
    g.y[i] = v / g.H[i + (GMAX + 1) * i];
  }
  for (int i = 0; i < GMAX; ++i) out[i] = i < k ? g.y[i] : 0.0;
  if (g.conv || g.it >= g.maxit) g.done = 1;
}

// b = inv * a (inv read from the device state; 0 leaves b untouched)
__global__ void scale_dev_kernel(const double* __restrict__ a, const GState* __restrict__ st,
                                 double* __restrict__ b, long long n) {
  const double c = st->inv;
  if (c == 0.0) return;
  for (long long i = blockIdx.x * (long long)GNT + threadIdx.x; i < n;
       i += (long long)gridDim.x * GNT)
    b[i] = c * a[i];
}

}  // namespace

void gmres_free(hdiv_ctx* h) {
  if (!h->gw) return;
  cudaFree(h->gw->V); cudaFree(h->gw->w); cudaFree(h->gw->t); cudaFree(h->gw->tq);
  cudaFree(h->gw->tu); cudaFree(h->gw->part); cudaFree(h->gw->hd); cudaFree(h->gw->glob);
  cudaFree(h->gw->st); cudaFreeHost(h->gw->st_host); cudaFreeHost(h->gw->flags);
  for (int j = 0; j < GMAX; ++j)
    if (h->gw->ev[j]) cudaEventDestroy(h->gw->ev[j]);
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
  HDIV_CUDA_TRY(cudaMalloc(&g->st, sizeof(GState)));
  HDIV_CUDA_TRY(cudaMallocHost(&g->st_host, sizeof(GState)));
  HDIV_CUDA_TRY(cudaMallocHost(&g->flags, sizeof(int) * GMAX));
  for (int j = 0; j < GMAX; ++j)
    HDIV_CUDA_TRY(cudaEventCreateWithFlags(&g->ev[j], cudaEventDisableTiming));
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

// the nk projections in g->hd (this rank's partial sums) -> global values in g->hd: multi-rank,
// the P per-rank vectors are all-gathered and summed in rank order on the device
static hdiv_status global_proj_dev(hdiv_ctx* h, int nk, cudaStream_t s) {
  GmresWork* g = h->gw;
  if (h->nranks == 1) return HDIV_OK;
  hdiv_status st = comm_allgather(h, g->hd, g->glob, nk, s);
  if (st != HDIV_OK) return st;
  rank_sum_kernel<<<1, GMAX + 1, 0, s>>>(g->glob, h->nranks, nk, g->hd);
  HDIV_CUDA_TRY(cudaGetLastError());
  return HDIV_OK;
}

// hd[0] = <a, b> over the whole (global) vector (deterministic), via the projection kernels
static hdiv_status dot_dev(hdiv_ctx* h, const double* a, const double* b, long long n, cudaStream_t s) {
  GmresWork* g = h->gw;
  proj_kernel<<<GBLK, GNT, 0, s>>>(a, n, 0, 1, b, g->part, g->ex_lo, g->ex_hi);
  proj_final_kernel<<<1, GNT, 0, s>>>(g->part, 1, g->hd);
  HDIV_CUDA_TRY(cudaGetLastError());
  return global_proj_dev(h, 1, s);
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
  // ||b|| once, on the host (the state's reference norm)
  if ((st = dot_dev(h, b, b, n, s)) != HDIV_OK) return st;
  double bb = 0.0;
  HDIV_CUDA_TRY(cudaMemcpyAsync(&bb, g->hd, sizeof(double), cudaMemcpyDeviceToHost, s));
  HDIV_CUDA_TRY(cudaStreamSynchronize(s));
  {
    GState* hs = g->st_host;
    std::memset(hs, 0, sizeof(GState));
    hs->bnorm = std::sqrt(bb);
    hs->rtol = rtol;
    hs->maxit = maxit;
    hs->rel = 1.0;
    if (hs->bnorm == 0.0) { hs->conv = 1; hs->done = 1; hs->rel = 0.0; }
    HDIV_CUDA_TRY(cudaMemcpyAsync(g->st, hs, sizeof(GState), cudaMemcpyHostToDevice, s));
  }
  while (!g->st_host->done) {
    // one restart cycle, launched without host round trips:
    // r = b - A x ; beta = ||r|| ; V_0 = r / beta (the start kernel decides done)
    HDIV_CUDA_TRY(apply_block_dev(h, x, g->w, nullptr, s));
    sub_kernel<<<GBLK, GNT, 0, s>>>(b, g->w, g->w, n);
    if ((st = dot_dev(h, g->w, g->w, n, s)) != HDIV_OK) return st;
    g_start_kernel<<<1, 1, 0, s>>>(g->st, g->hd);
    scale_dev_kernel<<<GBLK, GNT, 0, s>>>(g->w, g->st, g->V, n);
    HDIV_CUDA_TRY(cudaGetLastError());
    // the host stays at most LAG Arnoldi steps ahead of the device and stops launching once a
    // completed step reports the cycle finished (at most LAG wasted steps, no idle device)
    constexpr int LAG = 2;
    for (int j = 0; j < m; ++j) {
      if (j >= LAG) {
        HDIV_CUDA_TRY(cudaEventSynchronize(g->ev[j - LAG]));
        if (g->flags[j - LAG]) break;
      }
      // w = A B^-1 V_j
      if ((st = apply_precond_tri(h, g->V + (size_t)j * n, g->t, s)) != HDIV_OK) return st;
      HDIV_CUDA_TRY(apply_block_dev(h, g->t, g->w, nullptr, s));
      for (int pass = 0; pass < 2; ++pass) {   // classical Gram-Schmidt, twice
        for (int k0 = 0; k0 <= j; k0 += KB)
          proj_kernel<<<GBLK, GNT, 0, s>>>(g->V, n, k0, std::min(KB, j + 1 - k0), g->w, g->part,
                                           g->ex_lo, g->ex_hi);
        proj_final_kernel<<<1, GNT, 0, s>>>(g->part, j + 1, g->hd);
        HDIV_CUDA_TRY(cudaGetLastError());
        if ((st = global_proj_dev(h, j + 1, s)) != HDIV_OK) return st;
        combo_kernel<<<GBLK, GNT, 0, s>>>(g->V, n, j + 1, g->hd, g->w, 0);
        g_hcol_kernel<<<1, 1, 0, s>>>(g->st, g->hd, j);
        HDIV_CUDA_TRY(cudaGetLastError());
      }
      if ((st = dot_dev(h, g->w, g->w, n, s)) != HDIV_OK) return st;
      g_step_kernel<<<1, 1, 0, s>>>(g->st, g->hd, j, m);
      if (j + 1 < m) scale_dev_kernel<<<GBLK, GNT, 0, s>>>(g->w, g->st, g->V + (size_t)(j + 1) * n, n);
      HDIV_CUDA_TRY(cudaGetLastError());
      HDIV_CUDA_TRY(cudaMemcpyAsync(&g->flags[j], &g->st->cycle_done, sizeof(int),
                                    cudaMemcpyDeviceToHost, s));
      HDIV_CUDA_TRY(cudaEventRecord(g->ev[j], s));
    }
    // x += B^-1 V_k y, H y = g (back substitution on the device; k = 0 adds nothing)
    g_solve_kernel<<<1, 1, 0, s>>>(g->st, g->hd);
    combo_kernel<<<GBLK, GNT, 0, s>>>(g->V, n, m, g->hd, g->w, 1, &g->st->k);
    HDIV_CUDA_TRY(cudaGetLastError());
    if ((st = apply_precond_tri(h, g->w, g->t, s)) != HDIV_OK) return st;
    axpy_kernel<<<GBLK, GNT, 0, s>>>(g->t, x, n);
    HDIV_CUDA_TRY(cudaGetLastError());
    HDIV_CUDA_TRY(cudaMemcpyAsync(g->st_host, g->st, sizeof(GState), cudaMemcpyDeviceToHost, s));
    if ((st = comm_sync(h, s)) != HDIV_OK) return st;
  }
  HDIV_CUDA_TRY(cudaEventRecord(e1, s));
  HDIV_CUDA_TRY(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (rep) {
    rep->iters = g->st_host->it;
    rep->converged = g->st_host->conv;
    rep->rel_resid = g->st_host->rel;
    rep->t_solve_ms = ms;
  }
  return HDIV_OK;
}

}  // namespace hdiv
