// internal.h — libhdiv internals (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdint>
#include <string>
#include <vector>

#include "hdiv.h"

namespace hdiv {

constexpr int MAXP = HDIV_MAX_ORDER;
constexpr long long kAutoAmgRows = 1000000;   // HDIV_SCHUR_AUTO: AMG from this many L2 rows
constexpr int MAXQ = MAXP + 2;

// 1D tables on [0,1].  Passed to kernels by value (__grid_constant__).
struct Tab1D {
  int p, Q;
  double xq[MAXQ], wq[MAXQ];            // Gauss-Legendre rule, Q = p+2 (reading A3)
  double Bl[MAXQ][MAXP + 1];            // l_i(x_q)   Lagrange on GLL nodes
  double Bh[MAXQ][MAXP];                // h_j(x_q)   histopolation, h_j = -sum_{i<=j} l_i'
  double Ml[MAXP + 1][MAXP + 1];        // 1D masses B^T W B
  double Mh[MAXP][MAXP];
  double Mhinv[MAXP][MAXP];
  // Gauss-Legendre nodal basis of Q_{p-1} (p GL points g_b) for the local CG of W^-1
  // (P:606): BG[q][b] = L_b(x_q), HG[a][b] = integral over subinterval a of L_b
  // (histopolation coefficients of L_b, i.e. the change of basis GL-nodal -> histopolation)
  double BG[MAXQ][MAXP];
  double HG[MAXP][MAXP];
};

// Small table set for the affine (axis-aligned box) kernels.
struct TabAffine {
  double Ml[MAXP + 1][MAXP + 1];
  double Mh[MAXP][MAXP];
  double Mhinv[MAXP][MAXP];
};

bool build_tables(int p, int Q, Tab1D* t, std::string* err);

// Geometry kind of the local mesh
enum GeomKind { GEOM_BOX = 0, GEOM_AFFINE = 1, GEOM_TRILINEAR = 2 };

struct MinresWork;   // solver.cu
struct Comm;         // comm.cu
struct AmgHier;      // amg.cu
struct GmresWork;    // gmres.cu

}  // namespace hdiv

struct hdiv_ctx {
  int dim = 3, p = 1, Q = 3;
  hdiv_kind kind = HDIV_GRAD_DIV;
  hdiv_options opts{};
  int64_t N[3] = {1, 1, 1};       // global element counts
  int64_t NL[3] = {1, 1, 1};      // local element counts (last axis = slab thickness)
  int64_t ez0 = 0, ez1 = 1;       // slab along the last axis
  int64_t n[3] = {1, 1, 1};       // local subcell counts n_a = NL_a p
  int64_t E = 1;                  // local elements
  int64_t nrt = 0, nl2 = 0, nrt_g = 0, nl2_g = 0;
  int64_t off[3] = {0, 0, 0};     // RT component offsets (local numbering)
  int geom = hdiv::GEOM_BOX;
  bool has_z = true;              // (2,2) block nonzero
  int kernel = 2;                 // 1 general quadrature kernel, 2 affine tile kernel
  hdiv::Tab1D tab{};
  hdiv::TabAffine taff{};
  // device data
  double* d_vert = nullptr;       // local vertices [layers][(ny+1)][(nx+1)][dim]
  double* d_coef = nullptr;       // per element: box {cx, cy, cz, z}; general {w, z, 0, 0}
  double* d_mdiag = nullptr;      // M~ (assembled, interface-summed)
  double* d_ctil = nullptr;       // C~
  double* d_c2 = nullptr;         // per element alpha (grad-div) | gamma (Darcy)
  double* d_zcoef = nullptr;      // 3D: per element {mass weight, s_e = 1/alpha | gamma, 0, 0}
  double* d_winv = nullptr;       // [E][p^3][p^3] explicit W^e inverses (nullptr: local CG)
  double* d_geo = nullptr;        // [E][6][Q^3] stored G_q = w_q mw / det J J^T J (nullptr: on the fly)
  double* d_gvert = nullptr;      // NEXT-3 general gamma: per local vertex (nullptr: per element)
  double* d_sdinv = nullptr;      // 1 / diag(S~)
  int64_t* d_srow = nullptr;      // S~ CSR (local rows; ghost columns >= nl2 for multi-GPU)
  int32_t* d_scol = nullptr;
  double* d_sval = nullptr;
  int32_t* d_ecol = nullptr;      // 2D: S~ as SELL-32, fixed width 2d+1 (padding: col=row,
  double* d_eval = nullptr;       //   val=0) for the SpMVs inside S^-1
  double* d_cw = nullptr;         // 3D: [4][n_l2] diag(S~), +x/+y/+z face weights, + one plane
                                  //   (the cell stencil inside S^-1, cell_stencil.h)
  int64_t snnz = 0;
  double* d_scratch = nullptr;    // reduction partials etc.
  double* d_xbuf = nullptr;       // host-API staging (lazily allocated)
  double* d_ybuf = nullptr;
  cudaStream_t hs[3] = {nullptr, nullptr, nullptr};   // host pipeline: H2D, compute, D2H
  static constexpr int kMaxChunks = 64;
  cudaEvent_t hev[2][kMaxChunks] = {};                // H2D done / compute done per chunk
  // NEXT-3: essential (eliminated) RT sides of THIS rank's slab, bit 2a = side x_a = min of
  // the local grid, bit 2a+1 = max (the last-axis bits only where the slab touches the domain
  // boundary); 0 = natural everywhere
  int ess = 0;
  int rank = 0, nranks = 1;
  hdiv::Comm* comm = nullptr;
  hdiv::MinresWork* mw = nullptr;
  hdiv::AmgHier* amg = nullptr;   // NEXT-1 hierarchy when opts.schur_solver == HDIV_SCHUR_AMG
  hdiv::GmresWork* gw = nullptr;  // NEXT-4 Krylov basis (lazily allocated)
  int last_apply_ops = 0;         // device operations of the last hdiv_apply_block
};

// error plumbing
namespace hdiv {
void set_error(const std::string& s);
}
#define HDIV_CUDA_TRY(expr)                                                           \
  do {                                                                                \
    cudaError_t _e = (expr);                                                          \
    if (_e != cudaSuccess) {                                                          \
      hdiv::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));            \
      return HDIV_ERR_CUDA;                                                           \
    }                                                                                 \
  } while (0)

namespace hdiv {
// kernel launchers (return cudaGetLastError())
cudaError_t launch_affine_apply_range(const hdiv_ctx* h, const double* x, double* y, int tz0,
                                      int tz1, int* tz_out, cudaStream_t s,
                                      const int* skip = nullptr);
cudaError_t launch_affine_apply(const hdiv_ctx* h, const double* x, double* y, int mode,
                                const int* skip, cudaStream_t s);
// box-kernel block apply with the fused MINRES partial <y, x> (one partial per tile)
cudaError_t launch_affine_apply_dot(const hdiv_ctx* h, const double* x, double* y, const int* skip,
                                    double* dpart, cudaStream_t s);
long long affine_num_tiles(const hdiv_ctx* h);
cudaError_t launch_general_apply(const hdiv_ctx* h, const double* x, double* y, int mode,
                                 const int* skip, cudaStream_t s);
cudaError_t launch_l2_diag(const hdiv_ctx* h, double* w1, cudaStream_t s);
cudaError_t launch_general_z(const hdiv_ctx* h, const double* q, double* y, cudaStream_t s);
cudaError_t launch_trilinear_apply(const hdiv_ctx* h, const double* x, double* y, int mode,
                                   const int* skip, cudaStream_t s);
cudaError_t apply_block_dev(hdiv_ctx* h, const double* x, double* y, const int* skip,
                            cudaStream_t s);
cudaError_t launch_div(const hdiv_ctx* h, const double* u, double* yq, cudaStream_t s);
cudaError_t launch_divT(const hdiv_ctx* h, const double* q, double* yu, cudaStream_t s);
cudaError_t launch_mass_diag(const hdiv_ctx* h, double* diag, cudaStream_t s);
cudaError_t launch_ctil(const hdiv_ctx* h, const double* d_c2, double* ctil, cudaStream_t s);
cudaError_t launch_geometry_check(const hdiv_ctx* h, int* bad, cudaStream_t s);
cudaError_t build_winv(hdiv_ctx* h, cudaStream_t s);   // explicit W^e inverses (trilinear, p <= 4)
cudaError_t build_tri_geo(hdiv_ctx* h, cudaStream_t s);   // stored quadrature-point factors
cudaError_t launch_div_csr(const hdiv_ctx* h, int64_t* rp, int64_t* col, double* val,
                           cudaStream_t s);
hdiv_status build_schur(hdiv_ctx* h, cudaStream_t s);
cudaError_t launch_schur_export(const hdiv_ctx* h, int64_t* rp, int64_t* col, double* val,
                                cudaStream_t s);
cudaError_t launch_spmv(const hdiv_ctx* h, const double* x, double* y, cudaStream_t s);
hdiv_status apply_precond(hdiv_ctx* h, const double* v, double* z, cudaStream_t s);
hdiv_status minres(hdiv_ctx* h, const double* b, double* x, double rtol, int maxit,
                   hdiv_report* rep, cudaStream_t s);
void minres_free(hdiv_ctx* h);
hdiv_status schur_inv_apply(hdiv_ctx* h, const double* vq, double* y, cudaStream_t s);
hdiv_status apply_precond_tri(hdiv_ctx* h, const double* v, double* z, cudaStream_t s);
hdiv_status gmres(hdiv_ctx* h, const double* b, double* x, double rtol, int maxit, int restart,
                  hdiv_report* rep, cudaStream_t s);
void gmres_free(hdiv_ctx* h);
hdiv_status amg_setup(hdiv_ctx* h, cudaStream_t s);
void amg_free(hdiv_ctx* h);
// part != nullptr: the last level-0 sweep also writes the partial <x, b> into part[0..nbpart)
// (HDIV_ERR_UNSUPPORTED, nothing launched, when the hierarchy has no such sweep)
hdiv_status amg_vcycle(hdiv_ctx* h, const double* b, double* x, const int* done, cudaStream_t s,
                       double* part = nullptr, int nbpart = 0);
// reading A9e (3D slabs): S^-1 in the balancing form with the global coarse space around the
// inner preconditioner `inner` (block-Jacobi V-cycles or their A9d polynomial)
typedef hdiv_status (*AmgInner)(hdiv_ctx* h, const double* b, double* x, const int* done,
                                 cudaStream_t s);
bool amg_has_global_coarse(const hdiv_ctx* h);
hdiv_status amg_global_apply(hdiv_ctx* h, const double* b, double* x, const int* done,
                             cudaStream_t s, AmgInner inner);
int amg_num_levels(const hdiv_ctx* h);
hdiv_status amg_level_info(const hdiv_ctx* h, int l, int64_t* dims, int64_t* n, double* omega,
                           const double** st);

// multi-rank: NCCL asynchronous-error poll, and a stream sync that polls it while waiting
hdiv_status comm_check_async(const hdiv_ctx* h);
hdiv_status comm_sync(const hdiv_ctx* h, cudaStream_t s);

// device operations (kernel launches + memsets) issued by the current host thread; reset and
// read around an apply by hdiv_apply_block (hdiv_apply_launches reports the last count)
inline thread_local int g_ops = 0;
inline void count_op(int n = 1) { g_ops += n; }

// NVTX range around every C-ABI entry point (header-only NVTX v3: no link dependency)
struct NvtxScope {
  explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
  ~NvtxScope() { nvtxRangePop(); }
};
#define HDIV_NVTX() ::hdiv::NvtxScope _hdiv_nvtx_scope(__func__)

// apply modes
enum { MODE_MASS = 1, MODE_BLOCK = 2, MODE_ZONLY = 3 };

// NEXT-3: is the face of component c at subcell-face coordinate idx (along c) on an
// eliminated side?  ess: local side bitmask (hdiv_ctx::ess), n_c: local subcells along c
__host__ __device__ __forceinline__ bool face_masked(int ess, int c, long long idx, long long n_c) {
  return ((ess >> (2 * c)) & 1 && idx == 0) || ((ess >> (2 * c + 1)) & 1 && idx == n_c);
}
// y_b = x_b on the eliminated faces (x == nullptr: y_b = cval)
cudaError_t launch_ess_fixup(const hdiv_ctx* h, const double* x, double* y, double cval,
                             const int* skip, cudaStream_t s);
}  // namespace hdiv
