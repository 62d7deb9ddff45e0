// api.cu — the C-ABI of libhdiv (include/hdiv.h).  Argument marshalling, validation and
// dispatch only; every step of the hot path runs in the kernels of this directory.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "internal.h"

namespace hdiv {

static thread_local std::string g_err;
void set_error(const std::string& s) { g_err = s; }

hdiv_status comm_init(hdiv_ctx* h, const void* id, cudaStream_t s);      // comm.cu
void comm_free(hdiv_ctx* h);
hdiv_status comm_reverse_add(hdiv_ctx* h, double* y_rt, cudaStream_t s);  // interface planes
hdiv_status comm_setup_schur_ghosts(hdiv_ctx* h, cudaStream_t s);
void comm_overlap_handles(const hdiv_ctx* h, cudaStream_t* cs, cudaEvent_t* fork, cudaEvent_t* join);

// Slab apply with the interface exchange overlapped: the first and last z-tile
// layers, which alone write the two interface planes, run first; the reverse-add exchange and
// its add kernel run on the comm stream while the interior tile layers compute, joined before
// return.  Box meshes with >= 3 tile layers per slab (HDIV_SLAB_OVERLAP=0 disables).
static bool slab_overlap(const hdiv_ctx* h, int* ntz) {
  if (h->nranks < 2 || h->kernel != 2) return false;
  static const bool on = [] {
    const char* e = getenv("HDIV_SLAB_OVERLAP");
    return !(e && atoi(e) == 0);
  }();
  if (!on) return false;
  int TZ = 0;
  if (launch_affine_apply_range(h, nullptr, nullptr, 0, 0, &TZ, nullptr) != cudaSuccess || TZ <= 0)
    return false;
  *ntz = (int)((h->NL[2] + TZ - 1) / TZ);
  return *ntz >= 3;
}

static hdiv_status fail(hdiv_status st, const std::string& msg) {
  set_error(msg);
  return st;
}

// Vertex corner X[v][d] of local element (ex,ey,ez), v = a + 2b + 4c
static void corners(const std::vector<double>& V, int dim, int64_t NLx, int64_t NLy, int64_t ex,
                    int64_t ey, int64_t ez, double X[8][3]) {
  for (int v = 0; v < (1 << dim); ++v) {
    int a = v & 1, b = (v >> 1) & 1, c = (v >> 2) & 1;
    int64_t g = (dim == 3) ? ((ez + c) * (NLy + 1) + (ey + b)) * (NLx + 1) + (ex + a)
                           : (ey + b) * (NLx + 1) + (ex + a);
    for (int d = 0; d < dim; ++d) X[v][d] = V[g * dim + d];
  }
}

cudaError_t apply_block_dev(hdiv_ctx* h, const double* x, double* y, const int* skip,
                            cudaStream_t s) {
  int ntz = 0;
  if (slab_overlap(h, &ntz)) {
    cudaStream_t cs;
    cudaEvent_t fork, join;
    comm_overlap_handles(h, &cs, &fork, &join);
    cudaError_t e = launch_affine_apply_range(h, x, y, 0, 1, nullptr, s, skip);
    if (e == cudaSuccess) e = launch_affine_apply_range(h, x, y, ntz - 1, ntz, nullptr, s, skip);
    if (e == cudaSuccess) e = cudaEventRecord(fork, s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, fork, 0);
    if (e != cudaSuccess) return e;
    if (comm_reverse_add(h, y, cs) != HDIV_OK) return cudaErrorUnknown;
    e = cudaEventRecord(join, cs);
    if (e == cudaSuccess) e = launch_affine_apply_range(h, x, y, 1, ntz - 1, nullptr, s, skip);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, join, 0);
    return e;
  }
  cudaError_t e = (h->kernel == 2)  ? launch_affine_apply(h, x, y, MODE_BLOCK, skip, s)
                   : (h->dim == 3) ? launch_trilinear_apply(h, x, y, MODE_BLOCK, skip, s)
                                   : launch_general_apply(h, x, y, MODE_BLOCK, skip, s);
  if (e != cudaSuccess) return e;
  // eliminated essential faces: identity rows (the box kernel writes them itself)
  if (h->ess && h->kernel != 2) {
    e = launch_ess_fixup(h, x, y, 0.0, skip, s);
    if (e != cudaSuccess) return e;
  }
  if (h->nranks > 1) {
    if (comm_reverse_add(h, y, s) != HDIV_OK) return cudaErrorUnknown;
  }
  return cudaSuccess;
}

}  // namespace hdiv

using namespace hdiv;

extern "C" {

int hdiv_version(void) { return 1; }

const char* hdiv_last_error(void) { return g_err.c_str(); }

const char* hdiv_status_string(hdiv_status s) {
  switch (s) {
    case HDIV_OK: return "ok";
    case HDIV_ERR_INVALID_ORDER: return "invalid order";
    case HDIV_ERR_INVALID_MESH: return "invalid mesh";
    case HDIV_ERR_COEFFICIENT: return "coefficient error";
    case HDIV_ERR_SHAPE: return "shape error";
    case HDIV_ERR_CUDA: return "CUDA error";
    case HDIV_ERR_NCCL: return "NCCL error";
    case HDIV_ERR_BREAKDOWN: return "MINRES breakdown (preconditioner not SPD)";
    case HDIV_ERR_UNSUPPORTED: return "unsupported";
    case HDIV_ERR_NULL: return "null argument";
  }
  return "unknown";
}

void hdiv_destroy(hdiv_handle h) {
  if (!h) return;
  minres_free(h);
  comm_free(h);
  cudaFree(h->d_vert);
  cudaFree(h->d_coef);
  cudaFree(h->d_mdiag);
  cudaFree(h->d_ctil);
  cudaFree(h->d_c2);
  cudaFree(h->d_sdinv);
  cudaFree(h->d_srow);
  cudaFree(h->d_scol);
  cudaFree(h->d_sval);
  cudaFree(h->d_ecol);
  cudaFree(h->d_cw);
  cudaFree(h->d_zcoef);
  cudaFree(h->d_winv);
  cudaFree(h->d_geo);
  cudaFree(h->d_gvert);
  amg_free(h);
  gmres_free(h);
  cudaFree(h->d_eval);
  cudaFree(h->d_scratch);
  cudaFree(h->d_xbuf);
  cudaFree(h->d_ybuf);
  for (int i = 0; i < 3; ++i)
    if (h->hs[i]) cudaStreamDestroy(h->hs[i]);
  for (int k = 0; k < 2; ++k)
    for (int c = 0; c < hdiv_ctx::kMaxChunks; ++c)
      if (h->hev[k][c]) cudaEventDestroy(h->hev[k][c]);
  delete h;
}

hdiv_status hdiv_setup(const hdiv_mesh_desc* mesh, int p, const hdiv_coeffs* co, hdiv_kind kind,
                       const hdiv_options* opts, const void* nccl_id, int rank, int nranks,
                       void* stream, hdiv_handle* out) {
  HDIV_NVTX();
  if (!out) return fail(HDIV_ERR_NULL, "out is NULL");
  *out = nullptr;
  if (!mesh || !co) return fail(HDIV_ERR_NULL, "mesh/coeffs NULL");
  if (p < 1 || p > HDIV_MAX_ORDER) return fail(HDIV_ERR_INVALID_ORDER, "p out of [1,6]");
  if (mesh->dim != 2 && mesh->dim != 3) return fail(HDIV_ERR_SHAPE, "dim must be 2 or 3");
  if (kind != HDIV_GRAD_DIV && kind != HDIV_DARCY) return fail(HDIV_ERR_SHAPE, "bad kind");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(HDIV_ERR_SHAPE, "bad rank");
  if (nranks > 1 && !nccl_id) return fail(HDIV_ERR_NULL, "nccl id required for nranks > 1");
  const int dim = mesh->dim;
  const int64_t N[3] = {mesh->nx, mesh->ny, dim == 3 ? mesh->nz : 1};
  for (int d = 0; d < dim; ++d)
    if (N[d] < 1) return fail(HDIV_ERR_INVALID_MESH, "element counts must be >= 1");
  const int last = dim - 1;
  if (mesh->ez_begin < 0 || mesh->ez_end > N[last] || mesh->ez_end <= mesh->ez_begin)
    return fail(HDIV_ERR_INVALID_MESH, "bad slab range");
  if (nranks == 1 && (mesh->ez_begin != 0 || mesh->ez_end != N[last]))
    return fail(HDIV_ERR_INVALID_MESH, "single rank must own the whole mesh");
  cudaStream_t s = (cudaStream_t)stream;

  auto* h = new hdiv_ctx();
  h->dim = dim; h->p = p; h->Q = p + 2; h->kind = kind;
  h->rank = rank; h->nranks = nranks;
  h->opts.tau = (opts && opts->tau > 0) ? opts->tau : 1.0;
  h->opts.cheb_degree = (opts && opts->cheb_degree > 0) ? opts->cheb_degree : 4;
  h->opts.cheb_ratio = (opts && opts->cheb_ratio > 0) ? opts->cheb_ratio : 30.0;
  h->opts.kernel = opts ? opts->kernel : 0;
  h->opts.schur_solver = opts ? opts->schur_solver : HDIV_SCHUR_CHEBYSHEV;
  h->opts.amg_sweeps = (opts && opts->amg_sweeps > 0) ? opts->amg_sweeps : 2;
  h->opts.amg_max_coarse = (opts && opts->amg_max_coarse > 0) ? opts->amg_max_coarse : 512;
  h->opts.essential_sides = opts ? opts->essential_sides : 0;
  h->opts.project_mean = opts ? (opts->project_mean != 0) : 0;
  h->opts.tri_geometry = opts ? opts->tri_geometry : 0;
  h->opts.amg_cheb_degree = opts ? opts->amg_cheb_degree : 0;   // 0: auto (after the coefficients)
  h->opts.amg_cheb_ratio = (opts && opts->amg_cheb_ratio > 0) ? opts->amg_cheb_ratio : 20.0;
  {
    const int gc = opts ? opts->amg_global_coarse : 0;
    h->opts.amg_global_coarse = (dim == 3 && nranks > 1 && gc != 2) ? 1 : 0;   // A9e
  }
  if (h->opts.tri_geometry < 0 || h->opts.tri_geometry > 2) {
    delete h;
    return fail(HDIV_ERR_SHAPE, "options.tri_geometry must be 0, 1 or 2");
  }
  if (h->opts.essential_sides < 0 || h->opts.essential_sides >= (1 << (2 * dim))) {
    delete h;
    return fail(HDIV_ERR_SHAPE, "essential_sides: bits 0..2 dim - 1 only");
  }
  if (h->opts.schur_solver != HDIV_SCHUR_CHEBYSHEV && h->opts.schur_solver != HDIV_SCHUR_AMG &&
      h->opts.schur_solver != HDIV_SCHUR_AUTO) {
    delete h;
    return fail(HDIV_ERR_SHAPE, "schur_solver must be HDIV_SCHUR_CHEBYSHEV, _AMG or _AUTO");
  }
  for (int d = 0; d < 3; ++d) { h->N[d] = N[d]; h->NL[d] = N[d]; }
  h->ez0 = mesh->ez_begin; h->ez1 = mesh->ez_end;
  h->NL[last] = h->ez1 - h->ez0;
  if (dim == 2) h->NL[2] = 1;
  for (int d = 0; d < 3; ++d) h->n[d] = (d < dim) ? h->NL[d] * p : 1;
  {   // local eliminated sides: the last axis' sides only where the slab meets the boundary
    int ess = h->opts.essential_sides;
    if (h->ez0 > 0) ess &= ~(1 << (2 * last));
    if (h->ez1 < N[last]) ess &= ~(1 << (2 * last + 1));
    h->ess = ess;
  }
  h->E = h->NL[0] * h->NL[1] * h->NL[2];
  auto rt_count = [&](const int64_t* n) -> int64_t {
    if (dim == 2) return (n[0] + 1) * n[1] + n[0] * (n[1] + 1);
    return (n[0] + 1) * n[1] * n[2] + n[0] * (n[1] + 1) * n[2] + n[0] * n[1] * (n[2] + 1);
  };
  h->nrt = rt_count(h->n);
  const int64_t pd = (dim == 2) ? (int64_t)p * p : (int64_t)p * p * p;
  h->nl2 = h->E * pd;
  {
    int64_t ng[3] = {N[0] * p, N[1] * p, dim == 3 ? N[2] * p : 1};
    h->nrt_g = rt_count(ng);
    h->nl2_g = N[0] * N[1] * N[2] * pd;
    // auto S^-1: the fixed Chebyshev polynomial is not h-robust (config 3: 1903 MINRES iterations
    // vs 695 with the AMG V-cycle; config 4 does not converge in 600) but is the cheaper one on
    // small grids (config 2: 120 its / 4.2 ms vs 105 / 5.6 ms)
    if (h->opts.schur_solver == HDIV_SCHUR_AUTO)
      h->opts.schur_solver = (h->nl2_g >= kAutoAmgRows) ? HDIV_SCHUR_AMG : HDIV_SCHUR_CHEBYSHEV;
  }
  if (dim == 2) {
    h->off[0] = 0; h->off[1] = (h->n[0] + 1) * h->n[1]; h->off[2] = h->nrt;
  } else {
    h->off[0] = 0;
    h->off[1] = (h->n[0] + 1) * h->n[1] * h->n[2];
    h->off[2] = h->off[1] + h->n[0] * (h->n[1] + 1) * h->n[2];
  }

  // ---- vertices (host) ----
  const int64_t nvx = h->NL[0] + 1, nvy = h->NL[1] + 1, nvz = (dim == 3) ? h->NL[2] + 1 : 1;
  const int64_t nv = nvx * nvy * nvz;
  std::vector<double> V(nv * dim);
  if (mesh->vertices) {
    std::memcpy(V.data(), mesh->vertices, sizeof(double) * V.size());
  } else {   // uniform unit box
    for (int64_t k = 0; k < nvz; ++k)
      for (int64_t j = 0; j < nvy; ++j)
        for (int64_t i = 0; i < nvx; ++i) {
          int64_t g = (k * nvy + j) * nvx + i;
          V[g * dim + 0] = (double)i / N[0];
          if (dim == 2) V[g * dim + 1] = (double)(j + h->ez0) / N[1];
          else {
            V[g * dim + 1] = (double)j / N[1];
            V[g * dim + 2] = (double)(k + h->ez0) / N[2];
          }
        }
  }

  // ---- coefficients (host validation) ----
  const int64_t E = h->E;
  std::vector<double> mw(E), c2(E);
  bool any_gamma = false;
  // NEXT-3: general gamma as a trilinear vertex field (reading A22)
  const bool gvert = (kind == HDIV_DARCY && co->gamma_vertex != nullptr);
  if (gvert) {
    if (dim != 3) {
      delete h;
      return fail(HDIV_ERR_UNSUPPORTED, "general (vertex-field) gamma is 3D only");
    }
    if (opts && opts->kernel == 2) {
      delete h;
      return fail(HDIV_ERR_UNSUPPORTED, "general gamma needs the quadrature kernel");
    }
    const int64_t nvg = (h->NL[0] + 1) * (h->NL[1] + 1) * (h->NL[2] + 1);
    for (int64_t v = 0; v < nvg; ++v) {
      if (!(co->gamma_vertex[v] >= 0)) {
        delete h;
        return fail(HDIV_ERR_COEFFICIENT, "gamma_vertex must be >= 0");
      }
      if (co->gamma_vertex[v] > 0) any_gamma = true;
    }
  }
  for (int64_t e = 0; e < E; ++e) {
    if (kind == HDIV_GRAD_DIV) {
      double al = co->alpha ? co->alpha[e] : co->alpha0;
      double be = co->beta ? co->beta[e] : co->beta0;
      if (!(al > 0) || !(be > 0)) {
        delete h;
        return fail(HDIV_ERR_COEFFICIENT, "alpha, beta must be > 0");
      }
      mw[e] = be; c2[e] = al;
    } else {
      double ep = co->eps ? co->eps[e] : co->eps0;
      double ga = gvert ? 1.0 : (co->gamma ? co->gamma[e] : co->gamma0);   // gvert: s_e = 1
      if (!(ep > 0) || !(ga >= 0)) {
        delete h;
        return fail(HDIV_ERR_COEFFICIENT, "eps > 0 and gamma >= 0 required");
      }
      mw[e] = 1.0 / ep; c2[e] = ga;
      if (ga > 0 && !gvert) any_gamma = true;
    }
  }
  h->has_z = (kind == HDIV_GRAD_DIV) || any_gamma;
  // A9d auto degree.  One rank: the polynomial where one V-cycle of the geometric aggregation
  // degrades — element-wise contrast of the mass weight above 10^2 (config 3: 890 -> 330 MINRES
  // iterations, 3.6 -> 2.7 s); else the plain V-cycle (config 4: 155 its / 3.7 s, the polynomial
  // no faster).  Slabs: with the A9e global coarse space the plain V-cycle (config-3 mesh 32^3
  // p=4, 2..16 slabs: 544..553 its, flat, at half the cost per iteration of the polynomial's
  // 285..348); without it (2D, or switched off) the polynomial (block-Jacobi: 737 -> 356 at 8)
  if (h->opts.amg_cheb_degree <= 0) {
    double lo = mw.empty() ? 1.0 : mw[0], hi = lo;
    for (double v : mw) { lo = std::min(lo, v); hi = std::max(hi, v); }
    if (nranks > 1) h->opts.amg_cheb_degree = h->opts.amg_global_coarse ? 1 : 3;
    else h->opts.amg_cheb_degree = (hi > 100.0 * lo) ? 3 : 1;
  }

  // ---- geometry classification per element (host) ----
  bool all_box = true, all_affine = true;
  std::vector<double> coef(4 * E);
  for (int64_t e = 0; e < E && (all_box || all_affine); ++e) {
    int64_t ex = e % h->NL[0], ey = (e / h->NL[0]) % h->NL[1], ez = (dim == 3) ? e / (h->NL[0] * h->NL[1]) : 0;
    double X[8][3];
    corners(V, dim, h->NL[0], h->NL[1], ex, ey, ez, X);
    double scale = 0.0;
    for (int v = 1; v < (1 << dim); ++v)
      for (int d = 0; d < dim; ++d) scale = std::fmax(scale, std::fabs(X[v][d] - X[0][d]));
    const double tol = 1e-13 * scale;
    // parallelogram / parallelepiped: X_v = X_0 + sum of the axis edge vectors
    for (int v = 3; v < (1 << dim); ++v) {
      if (v == 4) continue;
      int a = v & 1, b = (v >> 1) & 1, c = (v >> 2) & 1;
      for (int d = 0; d < dim; ++d) {
        double pred = X[0][d] + a * (X[1][d] - X[0][d]) + b * (X[2][d] - X[0][d]) +
                      (dim == 3 ? c * (X[4][d] - X[0][d]) : 0.0);
        if (std::fabs(pred - X[v][d]) > tol) all_affine = false;
      }
    }
    // axis-aligned box: edge vectors along the axes
    double hsz[3] = {X[1][0] - X[0][0], X[2][1] - X[0][1], dim == 3 ? X[4][2] - X[0][2] : 1.0};
    for (int d = 0; d < dim; ++d) {
      if (d != 0 && std::fabs(X[1][d] - X[0][d]) > tol) all_box = false;
      if (d != 1 && std::fabs(X[2][d] - X[0][d]) > tol) all_box = false;
      if (dim == 3 && d != 2 && std::fabs(X[4][d] - X[0][d]) > tol) all_box = false;
    }
    if (!all_affine) all_box = false;
    for (int d = 0; d < dim; ++d)
      if (all_box && !(hsz[d] > 0)) {
        delete h;
        return fail(HDIV_ERR_INVALID_MESH, "det J <= 0 (inverted box element)");
      }
  }
  h->geom = all_box ? GEOM_BOX : (all_affine ? GEOM_AFFINE : GEOM_TRILINEAR);
  int want = h->opts.kernel;
  if (want == 2 && !(dim == 3 && all_box)) {
    delete h;
    return fail(HDIV_ERR_UNSUPPORTED, "affine tile kernel needs 3D axis-aligned boxes");
  }
  h->kernel = (want == 1 || gvert) ? 1 : ((dim == 3 && all_box) ? 2 : 1);
  for (int64_t e = 0; e < E; ++e) {
    int64_t ex = e % h->NL[0], ey = (e / h->NL[0]) % h->NL[1], ez = (dim == 3) ? e / (h->NL[0] * h->NL[1]) : 0;
    double X[8][3];
    corners(V, dim, h->NL[0], h->NL[1], ex, ey, ez, X);
    double zc = 0.0;
    if (h->geom != GEOM_TRILINEAR) {
      double det;
      double J[3][3] = {{0}};
      for (int d = 0; d < dim; ++d) {
        J[d][0] = X[1][d] - X[0][d];
        J[d][1] = X[2][d] - X[0][d];
        if (dim == 3) J[d][2] = X[4][d] - X[0][d];
      }
      if (dim == 2) det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
      else
        det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
              J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
              J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
      if (!(det > 0)) {
        delete h;
        return fail(HDIV_ERR_INVALID_MESH, "det J <= 0");
      }
      // Z_e = z_e (M_h^-1)^{(x)d}: grad-div det/alpha ; Darcy gamma det
      zc = (kind == HDIV_GRAD_DIV) ? det / c2[e] : c2[e] * det;
      if (h->kernel == 2) {
        double hx = J[0][0], hy = J[1][1], hz = J[2][2];
        coef[4 * e + 0] = mw[e] * hx / (hy * hz);
        coef[4 * e + 1] = mw[e] * hy / (hx * hz);
        coef[4 * e + 2] = mw[e] * hz / (hx * hy);
        coef[4 * e + 3] = zc;
        continue;
      }
    }
    coef[4 * e + 0] = mw[e];
    // 3D quadrature kernel: Z = s_e W_1^-1 by element-local CG (any geometry), s_e = 1/alpha
    // (grad-div) | gamma (Darcy); 2D kernel: exact Kronecker with z_e = det/alpha | gamma det on
    // parallelograms, s_e with a dense element solve on general quadrilaterals
    coef[4 * e + 1] = (dim == 3 || h->geom == GEOM_TRILINEAR)
                          ? ((kind == HDIV_GRAD_DIV) ? 1.0 / c2[e] : c2[e]) : zc;
    coef[4 * e + 2] = 0.0;
    coef[4 * e + 3] = 0.0;
  }
  // general-kernel coefficients are needed for the diagonal even on the box path
  std::vector<double> gcoef(4 * E);
  for (int64_t e = 0; e < E; ++e) {
    gcoef[4 * e] = mw[e];
    gcoef[4 * e + 1] = 0.0;
    gcoef[4 * e + 2] = gcoef[4 * e + 3] = 0.0;
  }

  std::string err;
  if (!build_tables(p, h->Q, &h->tab, &err)) {
    delete h;
    return fail(HDIV_ERR_INVALID_ORDER, err);
  }
  std::memcpy(h->taff.Ml, h->tab.Ml, sizeof(h->taff.Ml));
  std::memcpy(h->taff.Mh, h->tab.Mh, sizeof(h->taff.Mh));
  std::memcpy(h->taff.Mhinv, h->tab.Mhinv, sizeof(h->taff.Mhinv));

#define SETUP_TRY(expr)                                                                  \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess) {                                                             \
      set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));                     \
      hdiv_destroy(h);                                                                   \
      return HDIV_ERR_CUDA;                                                              \
    }                                                                                    \
  } while (0)

  SETUP_TRY(cudaMalloc(&h->d_vert, sizeof(double) * V.size()));
  SETUP_TRY(cudaMalloc(&h->d_coef, sizeof(double) * 4 * E));
  SETUP_TRY(cudaMalloc(&h->d_c2, sizeof(double) * E));
  if (dim == 3) {   // {mass weight, s_e} for the Z-only path (any geometry)
    std::vector<double> zc(4 * E, 0.0);
    for (int64_t e = 0; e < E; ++e) {
      zc[4 * e] = mw[e];
      zc[4 * e + 1] = (kind == HDIV_GRAD_DIV) ? 1.0 / c2[e] : c2[e];
    }
    SETUP_TRY(cudaMalloc(&h->d_zcoef, sizeof(double) * 4 * E));
    SETUP_TRY(cudaMemcpy(h->d_zcoef, zc.data(), sizeof(double) * 4 * E, cudaMemcpyHostToDevice));
  }
  SETUP_TRY(cudaMalloc(&h->d_mdiag, sizeof(double) * h->nrt));
  SETUP_TRY(cudaMalloc(&h->d_ctil, sizeof(double) * h->nl2));
  SETUP_TRY(cudaMemcpyAsync(h->d_vert, V.data(), sizeof(double) * V.size(), cudaMemcpyHostToDevice, s));
  SETUP_TRY(cudaMemcpyAsync(h->d_c2, c2.data(), sizeof(double) * E, cudaMemcpyHostToDevice, s));
  if (gvert) {
    const size_t nvg = (size_t)((h->NL[0] + 1) * (h->NL[1] + 1) * (h->NL[2] + 1));
    SETUP_TRY(cudaMalloc(&h->d_gvert, sizeof(double) * nvg));
    SETUP_TRY(cudaMemcpyAsync(h->d_gvert, co->gamma_vertex, sizeof(double) * nvg,
                              cudaMemcpyHostToDevice, s));
  }
  // the diagonal kernel reads {mass weight} from d_coef: upload general layout first
  SETUP_TRY(cudaMemcpyAsync(h->d_coef, gcoef.data(), sizeof(double) * 4 * E, cudaMemcpyHostToDevice, s));
  if (h->geom == GEOM_TRILINEAR) {
    int* bad = nullptr;
    SETUP_TRY(cudaMalloc(&bad, sizeof(int)));
    SETUP_TRY(cudaMemsetAsync(bad, 0, sizeof(int), s));
    SETUP_TRY(launch_geometry_check(h, bad, s));
    int hb = 0;
    SETUP_TRY(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
    SETUP_TRY(cudaStreamSynchronize(s));
    cudaFree(bad);
    if (hb) {
      hdiv_destroy(h);
      return fail(HDIV_ERR_INVALID_MESH, "det J <= 0 at a quadrature point");
    }
  }
  // W^-1 by precomputed explicit element inverses on trilinear meshes at
  // p <= 4 when they fit (<= 16 GB and a quarter of the free memory; env HDIV_WINV=cg: local CG)
  if (dim == 3 && h->geom == GEOM_TRILINEAR && h->has_z && !gvert && h->p <= 4) {
    const char* wm = getenv("HDIV_WINV");
    const size_t n3 = (size_t)h->p * h->p * h->p;
    const size_t bytes = sizeof(double) * n3 * n3 * (size_t)E;
    size_t fr = 0, tot = 0;
    SETUP_TRY(cudaMemGetInfo(&fr, &tot));
    const bool want = !(wm && std::string(wm) == "cg");
    if (want && bytes <= ((size_t)16 << 30) && bytes <= fr / 4) {
      SETUP_TRY(cudaMalloc(&h->d_winv, bytes));
      SETUP_TRY(build_winv(h, s));
    }
  }
  // stored Piola factors at the quadrature points (partial assembly) for the
  // trilinear mass / gamma = 0 applies: 48 Q^3 B per element (config 3, p = 4: 2.7 GB)
  if (dim == 3 && h->geom == GEOM_TRILINEAR && h->kernel == 1 && !gvert && h->opts.tri_geometry != 1) {
    const size_t bytes = sizeof(double) * 6 * (size_t)h->Q * h->Q * h->Q * (size_t)E;
    size_t fr = 0, tot = 0;
    SETUP_TRY(cudaMemGetInfo(&fr, &tot));
    if (h->opts.tri_geometry == 2 || bytes <= fr / 4) {
      SETUP_TRY(cudaMalloc(&h->d_geo, bytes));
      SETUP_TRY(build_tri_geo(h, s));
    }
  }
  SETUP_TRY(launch_mass_diag(h, h->d_mdiag, s));
  if (h->ess) SETUP_TRY(launch_ess_fixup(h, nullptr, h->d_mdiag, 1.0, nullptr, s));   // M~_b = 1
  SETUP_TRY(launch_ctil(h, h->d_c2, h->d_ctil, s));
  SETUP_TRY(cudaMemcpyAsync(h->d_coef, coef.data(), sizeof(double) * 4 * E, cudaMemcpyHostToDevice, s));
  if (nranks > 1) {
    hdiv_status cs = comm_init(h, nccl_id, s);
    if (cs != HDIV_OK) { hdiv_destroy(h); return cs; }
    cs = comm_reverse_add(h, h->d_mdiag, s);   // interface faces: sum of both sides
    if (cs != HDIV_OK) { hdiv_destroy(h); return cs; }
  }
  {
    // S~ inside S^-1: the cell stencil (3D, kernel_sparse.cu / cell_stencil.h) or a SELL-32
    // copy (2D); the CSR itself serves the ABI exports and hdiv_apply_schur
    hdiv_status ss = build_schur(h, s);
    if (ss != HDIV_OK) { hdiv_destroy(h); return ss; }
    if (nranks > 1) {
      ss = comm_setup_schur_ghosts(h, s);
      if (ss != HDIV_OK) { hdiv_destroy(h); return ss; }
    }
    if (h->opts.schur_solver == HDIV_SCHUR_AMG) {
      ss = amg_setup(h, s);
      if (ss != HDIV_OK) { hdiv_destroy(h); return ss; }
    }
  }
  SETUP_TRY(cudaStreamSynchronize(s));
  SETUP_TRY(cudaGetLastError());
#undef SETUP_TRY
  *out = h;
  return HDIV_OK;
}

hdiv_status hdiv_sizes(hdiv_handle h, int64_t* nrt, int64_t* nl2, int64_t* nrt_g, int64_t* nl2_g) {
  if (!h) return fail(HDIV_ERR_NULL, "NULL handle");
  if (nrt) *nrt = h->nrt;
  if (nl2) *nl2 = h->nl2;
  if (nrt_g) *nrt_g = h->nrt_g;
  if (nl2_g) *nl2_g = h->nl2_g;
  return HDIV_OK;
}

hdiv_status hdiv_apply_mass(hdiv_handle h, const double* u, double* yu, void* stream) {
  HDIV_NVTX();
  if (!h || !u || !yu) return fail(HDIV_ERR_NULL, "NULL argument");
  cudaStream_t s = (cudaStream_t)stream;
  HDIV_CUDA_TRY(h->kernel == 2  ? launch_affine_apply(h, u, yu, MODE_MASS, nullptr, s)
                : (h->dim == 3) ? launch_trilinear_apply(h, u, yu, MODE_MASS, nullptr, s)
                                : launch_general_apply(h, u, yu, MODE_MASS, nullptr, s));
  if (h->ess && h->kernel != 2) HDIV_CUDA_TRY(launch_ess_fixup(h, u, yu, 0.0, nullptr, s));
  if (h->nranks > 1) return comm_reverse_add(h, yu, s);
  return HDIV_OK;
}

hdiv_status hdiv_apply_div(hdiv_handle h, const double* u, double* yq, void* stream) {
  HDIV_NVTX();
  if (!h || !u || !yq) return fail(HDIV_ERR_NULL, "NULL argument");
  HDIV_CUDA_TRY(launch_div(h, u, yq, (cudaStream_t)stream));
  return HDIV_OK;
}

hdiv_status hdiv_apply_divT(hdiv_handle h, const double* q, double* yu, void* stream) {
  HDIV_NVTX();
  if (!h || !q || !yu) return fail(HDIV_ERR_NULL, "NULL argument");
  cudaStream_t s = (cudaStream_t)stream;
  HDIV_CUDA_TRY(launch_divT(h, q, yu, s));
  if (h->nranks > 1) return comm_reverse_add(h, yu, s);
  return HDIV_OK;
}

hdiv_status hdiv_apply_block(hdiv_handle h, const double* x, double* y, void* stream) {
  HDIV_NVTX();
  if (!h || !x || !y) return fail(HDIV_ERR_NULL, "NULL argument");
  g_ops = 0;
  HDIV_CUDA_TRY(apply_block_dev(h, x, y, nullptr, (cudaStream_t)stream));
  h->last_apply_ops = g_ops;
  return HDIV_OK;
}

hdiv_status hdiv_apply_z(hdiv_handle h, const double* q, double* y, void* stream) {
  HDIV_NVTX();
  if (!h || !q || !y) return fail(HDIV_ERR_NULL, "NULL argument");
  if (h->dim == 2) {
    if (!h->has_z) {   // Darcy gamma = 0: Z = 0
      HDIV_CUDA_TRY(cudaMemsetAsync(y, 0, sizeof(double) * h->nl2, (cudaStream_t)stream));
      return HDIV_OK;
    }
    HDIV_CUDA_TRY(launch_general_z(h, q, y, (cudaStream_t)stream));
    return HDIV_OK;
  }
  HDIV_CUDA_TRY(launch_trilinear_apply(h, q, y, MODE_ZONLY, nullptr, (cudaStream_t)stream));
  return HDIV_OK;
}

hdiv_status hdiv_apply_precond_tri(hdiv_handle h, const double* v, double* z, void* stream) {
  HDIV_NVTX();
  if (!h || !v || !z) return fail(HDIV_ERR_NULL, "NULL argument");
  return apply_precond_tri(h, v, z, (cudaStream_t)stream);
}

hdiv_status hdiv_gmres_solve(hdiv_handle h, const double* b, double* x, double rtol, int maxit,
                             int restart, hdiv_report* report, void* stream) {
  HDIV_NVTX();
  if (!h || !b || !x) return fail(HDIV_ERR_NULL, "NULL argument");
  if (!(rtol > 0) || maxit < 1 || restart < 1 || restart > 64)
    return fail(HDIV_ERR_SHAPE, "gmres: rtol > 0, maxit >= 1, 1 <= restart <= 64 required");
  return gmres(h, b, x, rtol, maxit, restart, report, (cudaStream_t)stream);
}

hdiv_status hdiv_apply_launches(hdiv_handle h, int* n) {
  if (!h || !n) return fail(HDIV_ERR_NULL, "NULL argument");
  // counted at the launch sites during the last hdiv_apply_block on this handle (kernels +
  // memsets of this rank: the fused apply, the memset of the quadrature paths, a separate
  // explicit-W^-1 apply, the eliminated-face fixup, the interface add of multi-rank applies);
  // 0 before the first apply
  *n = h->last_apply_ops;
  return HDIV_OK;
}

// End-to-end host apply on box meshes (one rank): the mesh is cut into chunks of element
// layers along z (whole halo tiles) and the chunks are pipelined over three streams —
// H2D of chunk c+1 and D2H of chunk c-1 overlap the fused apply of chunk c (PCIe is full
// duplex).  Chunk c needs x for its own layers plus the - halo layer and the top z-face plane
// (already sent with chunks <= c); it owns the outputs of its layers except the top z-face
// plane, which belongs to chunk c+1 (the + tile owns a shared plane).
static hdiv_status apply_block_host_pipelined(hdiv_ctx* h, const double* xh, double* yh,
                                              cudaStream_t caller) {
  int TZ = 0;
  HDIV_CUDA_TRY(launch_affine_apply_range(h, nullptr, nullptr, 0, 0, &TZ, caller));
  const int64_t NLz = h->NL[2], P = h->p;
  const char* ec = getenv("HDIV_HOST_CHUNKS");
  const int64_t want = ec ? std::max(1, atoi(ec)) : 32;   // fill + drain cost ~2/want of a transfer
  int64_t cz = (NLz + want - 1) / want;
  cz = ((cz + TZ - 1) / TZ) * TZ;
  const int nch = (int)((NLz + cz - 1) / cz);
  if (nch > hdiv_ctx::kMaxChunks) return HDIV_ERR_UNSUPPORTED;
  for (int i = 0; i < 3; ++i)
    if (!h->hs[i]) HDIV_CUDA_TRY(cudaStreamCreateWithFlags(&h->hs[i], cudaStreamNonBlocking));
  for (int k = 0; k < 2; ++k)
    for (int c = 0; c < nch; ++c)
      if (!h->hev[k][c]) HDIV_CUDA_TRY(cudaEventCreateWithFlags(&h->hev[k][c], cudaEventDisableTiming));
  cudaEvent_t start;
  HDIV_CUDA_TRY(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
  HDIV_CUDA_TRY(cudaEventRecord(start, caller));
  for (int i = 0; i < 3; ++i) HDIV_CUDA_TRY(cudaStreamWaitEvent(h->hs[i], start, 0));
  cudaEventDestroy(start);
  const int64_t n0 = h->n[0], n1 = h->n[1];
  const int64_t sx = (n0 + 1) * n1, sy = n0 * (n1 + 1), sz = n0 * n1;   // doubles per K plane
  const int64_t sq = h->NL[0] * h->NL[1] * P * P * P;                   // per element layer
  double* dx = h->d_xbuf;
  double* dy = h->d_ybuf;
  auto cpy = [&](double* dst, const double* src, int64_t off, int64_t cnt, cudaMemcpyKind kd,
                 cudaStream_t st) -> cudaError_t {
    if (cnt <= 0) return cudaSuccess;
    return cudaMemcpyAsync(dst + off, src + off, sizeof(double) * cnt, kd, st);
  };
  for (int c = 0; c < nch; ++c) {
    const int64_t z0 = c * cz, z1 = std::min<int64_t>(NLz, z0 + cz);
    const bool last = (z1 == NLz);
    const cudaMemcpyKind H2D = cudaMemcpyHostToDevice, D2H = cudaMemcpyDeviceToHost;
    // H2D: x/y faces of planes [z0 P, z1 P), z faces (previous top, z1 P], q layers [z0, z1)
    const int64_t Ka = (c == 0) ? 0 : z0 * P + 1, Kb = z1 * P + 1;
    HDIV_CUDA_TRY(cpy(dx, xh, h->off[0] + sx * z0 * P, sx * (z1 - z0) * P, H2D, h->hs[0]));
    HDIV_CUDA_TRY(cpy(dx, xh, h->off[1] + sy * z0 * P, sy * (z1 - z0) * P, H2D, h->hs[0]));
    HDIV_CUDA_TRY(cpy(dx, xh, h->off[2] + sz * Ka, sz * (Kb - Ka), H2D, h->hs[0]));
    HDIV_CUDA_TRY(cpy(dx, xh, h->nrt + sq * z0, sq * (z1 - z0), H2D, h->hs[0]));
    HDIV_CUDA_TRY(cudaEventRecord(h->hev[0][c], h->hs[0]));
    // fused apply of the chunk's tiles
    HDIV_CUDA_TRY(cudaStreamWaitEvent(h->hs[1], h->hev[0][c], 0));
    HDIV_CUDA_TRY(launch_affine_apply_range(h, dx, dy, (int)(z0 / TZ), (int)((z1 + TZ - 1) / TZ),
                                            nullptr, h->hs[1]));
    HDIV_CUDA_TRY(cudaEventRecord(h->hev[1][c], h->hs[1]));
    // D2H of the owned outputs
    HDIV_CUDA_TRY(cudaStreamWaitEvent(h->hs[2], h->hev[1][c], 0));
    const int64_t Ke = last ? z1 * P + 1 : z1 * P;
    HDIV_CUDA_TRY(cpy(yh, dy, h->off[0] + sx * z0 * P, sx * (z1 - z0) * P, D2H, h->hs[2]));
    HDIV_CUDA_TRY(cpy(yh, dy, h->off[1] + sy * z0 * P, sy * (z1 - z0) * P, D2H, h->hs[2]));
    HDIV_CUDA_TRY(cpy(yh, dy, h->off[2] + sz * z0 * P, sz * (Ke - z0 * P), D2H, h->hs[2]));
    HDIV_CUDA_TRY(cpy(yh, dy, h->nrt + sq * z0, sq * (z1 - z0), D2H, h->hs[2]));
  }
  HDIV_CUDA_TRY(cudaStreamSynchronize(h->hs[2]));
  HDIV_CUDA_TRY(cudaStreamSynchronize(h->hs[1]));
  HDIV_CUDA_TRY(cudaStreamSynchronize(h->hs[0]));
  return HDIV_OK;
}

hdiv_status hdiv_apply_block_host(hdiv_handle h, const double* xh, double* yh, void* stream) {
  HDIV_NVTX();
  if (!h || !xh || !yh) return fail(HDIV_ERR_NULL, "NULL argument");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t bytes = sizeof(double) * (h->nrt + h->nl2);
  if (!h->d_xbuf) HDIV_CUDA_TRY(cudaMalloc(&h->d_xbuf, bytes));
  if (!h->d_ybuf) HDIV_CUDA_TRY(cudaMalloc(&h->d_ybuf, bytes));
  const char* ep = getenv("HDIV_HOST_PIPELINE");
  const bool pipe = !(ep && atoi(ep) == 0);
  if (pipe && h->kernel == 2 && h->dim == 3 && h->nranks == 1 && h->NL[2] >= 2) {
    hdiv_status st = apply_block_host_pipelined(h, xh, yh, s);
    if (st != HDIV_ERR_UNSUPPORTED) return st;
  }
  HDIV_CUDA_TRY(cudaMemcpyAsync(h->d_xbuf, xh, bytes, cudaMemcpyHostToDevice, s));
  HDIV_CUDA_TRY(apply_block_dev(h, h->d_xbuf, h->d_ybuf, nullptr, s));
  HDIV_CUDA_TRY(cudaMemcpyAsync(yh, h->d_ybuf, bytes, cudaMemcpyDeviceToHost, s));
  HDIV_CUDA_TRY(cudaStreamSynchronize(s));
  return HDIV_OK;
}

hdiv_status hdiv_assemble_mass_diag(hdiv_handle h, double* diag, void* stream) {
  HDIV_NVTX();
  if (!h || !diag) return fail(HDIV_ERR_NULL, "NULL argument");
  HDIV_CUDA_TRY(cudaMemcpyAsync(diag, h->d_mdiag, sizeof(double) * h->nrt,
                                cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return HDIV_OK;
}

hdiv_status hdiv_assemble_schur_diag_term(hdiv_handle h, double* ctil, void* stream) {
  HDIV_NVTX();
  if (!h || !ctil) return fail(HDIV_ERR_NULL, "NULL argument");
  HDIV_CUDA_TRY(cudaMemcpyAsync(ctil, h->d_ctil, sizeof(double) * h->nl2,
                                cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return HDIV_OK;
}

hdiv_status hdiv_schur_nnz(hdiv_handle h, int64_t* nnz) {
  if (!h || !nnz) return fail(HDIV_ERR_NULL, "NULL argument");
  *nnz = h->snnz;
  return HDIV_OK;
}

hdiv_status hdiv_assemble_schur_csr(hdiv_handle h, int64_t* rp, int64_t* col, double* val,
                                    void* stream) {
  HDIV_NVTX();
  if (!h || !rp || !col || !val) return fail(HDIV_ERR_NULL, "NULL argument");
  HDIV_CUDA_TRY(launch_schur_export(h, rp, col, val, (cudaStream_t)stream));
  return HDIV_OK;
}

hdiv_status hdiv_apply_schur(hdiv_handle h, const double* x, double* y, void* stream) {
  HDIV_NVTX();
  if (!h || !x || !y) return fail(HDIV_ERR_NULL, "NULL argument");
  if (h->nranks > 1) return fail(HDIV_ERR_UNSUPPORTED, "apply_schur with ghosts: use minres");
  HDIV_CUDA_TRY(launch_spmv(h, x, y, (cudaStream_t)stream));
  return HDIV_OK;
}

hdiv_status hdiv_export_div_csr(hdiv_handle h, int64_t* rp, int64_t* col, double* val,
                                void* stream) {
  HDIV_NVTX();
  if (!h || !rp || !col || !val) return fail(HDIV_ERR_NULL, "NULL argument");
  HDIV_CUDA_TRY(launch_div_csr(h, rp, col, val, (cudaStream_t)stream));
  return HDIV_OK;
}

hdiv_status hdiv_apply_precond(hdiv_handle h, const double* v, double* z, void* stream) {
  HDIV_NVTX();
  if (!h || !v || !z) return fail(HDIV_ERR_NULL, "NULL argument");
  return apply_precond(h, v, z, (cudaStream_t)stream);
}

hdiv_status hdiv_minres_solve(hdiv_handle h, const double* b, double* x, double rtol, int maxit,
                              hdiv_report* rep, void* stream) {
  HDIV_NVTX();
  if (!h || !b || !x) return fail(HDIV_ERR_NULL, "NULL argument");
  if (maxit < 1) return fail(HDIV_ERR_SHAPE, "maxit < 1");
  return minres(h, b, x, rtol, maxit, rep, (cudaStream_t)stream);
}

hdiv_status hdiv_amg_levels(hdiv_handle h, int* nlevels) {
  if (!h || !nlevels) return fail(HDIV_ERR_NULL, "NULL argument");
  if (!h->amg) return fail(HDIV_ERR_UNSUPPORTED, "handle has no AMG hierarchy");
  *nlevels = amg_num_levels(h);
  return HDIV_OK;
}

hdiv_status hdiv_amg_level(hdiv_handle h, int level, int64_t* dims, int64_t* n, double* omega,
                           double* st, void* stream) {
  if (!h || !dims || !n || !omega) return fail(HDIV_ERR_NULL, "NULL argument");
  if (!h->amg) return fail(HDIV_ERR_UNSUPPORTED, "handle has no AMG hierarchy");
  const double* src = nullptr;
  hdiv_status st_ = amg_level_info(h, level, dims, n, omega, &src);
  if (st_ != HDIV_OK) return st_;
  if (st && src) {
    const int NS = (h->dim == 3) ? 27 : 9;
    HDIV_CUDA_TRY(cudaMemcpyAsync(st, src, sizeof(double) * NS * (*n), cudaMemcpyDeviceToDevice,
                                  (cudaStream_t)stream));
  }
  return HDIV_OK;
}

hdiv_status hdiv_debug_gl_tables(int p, int Q, double* BG, double* HG) {
  Tab1D t;
  std::string err;
  if (!build_tables(p, Q, &t, &err)) return fail(HDIV_ERR_INVALID_ORDER, err);
  for (int q = 0; q < Q; ++q)
    for (int b = 0; b < p; ++b) if (BG) BG[q * p + b] = t.BG[q][b];
  for (int a = 0; a < p; ++a)
    for (int b = 0; b < p; ++b) if (HG) HG[a * p + b] = t.HG[a][b];
  return HDIV_OK;
}

hdiv_status hdiv_debug_tables(int p, int Q, double* xq, double* wq, double* Bl, double* Bh,
                              double* Ml, double* Mh, double* Mhinv) {
  Tab1D t;
  std::string err;
  if (!build_tables(p, Q, &t, &err)) return fail(HDIV_ERR_INVALID_ORDER, err);
  for (int q = 0; q < Q; ++q) {
    if (xq) xq[q] = t.xq[q];
    if (wq) wq[q] = t.wq[q];
    for (int i = 0; i <= p; ++i) if (Bl) Bl[q * (p + 1) + i] = t.Bl[q][i];
    for (int j = 0; j < p; ++j) if (Bh) Bh[q * p + j] = t.Bh[q][j];
  }
  for (int i = 0; i <= p; ++i)
    for (int j = 0; j <= p; ++j) if (Ml) Ml[i * (p + 1) + j] = t.Ml[i][j];
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j) {
      if (Mh) Mh[i * p + j] = t.Mh[i][j];
      if (Mhinv) Mhinv[i * p + j] = t.Mhinv[i][j];
    }
  return HDIV_OK;
}

}  // extern "C"
