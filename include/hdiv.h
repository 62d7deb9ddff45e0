/* hdiv.h — C-ABI of libhdiv: the B200 hot path of arXiv 2304.12387's matrix-free
 * block-preconditioned saddle-point solver for RT_p / L2_{p-1} (interpolation-histopolation
 * basis) grad-div and Darcy problems on structured quadrilateral / hexahedral meshes.
 *
 * Citations: P:n = /root/reference/PAPER.md line n.
 *
 * Conventions for every call
 *  - Vectors are DEVICE pointers (fp64), caller-owned (e.g. torch tensors), in the canonical
 *    numbering of DESIGN.md §Layout (the library's HBM layout IS the canonical numbering):
 *      RT (3D): x-faces I+(n_x+1)(J+n_y K), then y-faces I+n_x(J+(n_y+1)K), then z-faces
 *               I+n_x(J+n_y K);  n_a = N_a p subcells per axis;  (2D: x-faces, y-faces).
 *      L2     : element-contiguous e p^d + (a + p(b + p c)), e = ex + N_x(ey + N_y ez).
 *      block  : x = [u (n_rt) ; q~ (n_l2)].
 *    With nranks > 1 the vectors are this rank's slab (its own canonical numbering; the
 *    interface face plane is replicated on both ranks and kept bitwise identical).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream). Applies are
 *    asynchronous on that stream; nothing is synchronised unless stated.
 *  - Inputs and outputs must not alias unless stated.
 *  - Errors are returned as hdiv_status; nothing propagates across the ABI. Validation
 *    (order, det J > 0 at every quadrature point, coefficient signs, shapes) happens in
 *    hdiv_setup before any device work.  A CUDA launch error is HDIV_ERR_CUDA.
 *  - ONE call in flight per handle.  Several calls keep scratch in the handle (the MINRES /
 *    GMRES workspaces, the Chebyshev and AMG work vectors used by hdiv_apply_precond and
 *    hdiv_apply_schur, the explicit-inverse / local-CG buffers of hdiv_apply_precond_tri, the
 *    host-pipeline buffers, streams and events of hdiv_apply_block_host, the interface send /
 *    receive buffers and the comm stream of multi-rank applies), and some of it is allocated
 *    lazily on first use.  Calls on one handle must therefore be ordered by the caller: issue
 *    them from one host thread and on one stream (or on streams the caller orders with
 *    events).  Distinct handles are independent.  There is no internal lock.
 */
#ifndef HDIV_H
#define HDIV_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hdiv_ctx* hdiv_handle;          /* opaque, library-owned */

typedef enum {
  HDIV_OK = 0,
  HDIV_ERR_INVALID_ORDER = 1,   /* p < 1 or p > HDIV_MAX_ORDER                        */
  HDIV_ERR_INVALID_MESH = 2,    /* det J <= 0 at a quadrature point, bad counts/slab   */
  HDIV_ERR_COEFFICIENT = 3,     /* alpha, beta, eps <= 0 or gamma < 0                  */
  HDIV_ERR_SHAPE = 4,           /* inconsistent sizes / dim                            */
  HDIV_ERR_CUDA = 5,            /* CUDA runtime error (allocation, launch)             */
  HDIV_ERR_NCCL = 6,            /* NCCL error                                          */
  HDIV_ERR_BREAKDOWN = 7,       /* MINRES gamma^2 < 0: preconditioner not SPD          */
  HDIV_ERR_UNSUPPORTED = 8,     /* a combination this build does not provide              */
  HDIV_ERR_NULL = 9             /* NULL handle or required pointer                      */
} hdiv_status;

#define HDIV_MAX_ORDER 6

typedef enum {
  HDIV_GRAD_DIV = 0,  /* [M_beta, D^T; D, -W_alpha^-1]            */
  HDIV_DARCY = 1      /* [M_{1/eps}, D^T; D, -W^-1 W_gamma W^-1];   */
                      /* gamma piecewise constant, gamma = 0 allowed (zero (2,2) block)     */
} hdiv_kind;

typedef struct {
  int dim;                    /* 2 or 3                                                      */
  int64_t nx, ny, nz;         /* GLOBAL element counts (2D: nz = 1)                          */
  int64_t ez_begin, ez_end;   /* this rank's slab of element layers [begin, end) along the   */
                              /* last axis (z in 3D, y in 2D); single GPU: [0, nz) / [0, ny) */
  const double* vertices;     /* HOST, vertex layers begin..end inclusive of the slab,       */
                              /* [layers][..][nx+1][dim], x fastest; NULL => uniform unit box */
} hdiv_mesh_desc;

typedef struct {              /* HOST per-element arrays of the slab [E_local], or NULL       */
  const double *alpha, *beta, *gamma, *eps;
  double alpha0, beta0, gamma0, eps0;   /* constants used where an array is NULL              */
  /* NEXT-3 (reading A22): Darcy with a general (not piecewise-constant) gamma —
   * HOST per-vertex values of the slab's vertex layers (layout of hdiv_mesh_desc.vertices
   * without the coordinate axis), gamma(x) = their trilinear interpolant, >= 0.  When set,
   * `gamma`/`gamma0` are ignored and the (2,2) block is the full W^-1 W_gamma W^-1 (two
   * element-local W^-1 solves per apply); 3D only (HDIV_ERR_UNSUPPORTED in 2D), always on the
   * quadrature kernel. */
  const double* gamma_vertex;
} hdiv_coeffs;

typedef struct {
  double tau;          /* (1,1) preconditioner scale tau M~; <= 0 => 1 (A7)      */
  int cheb_degree;     /* S^-1 = Chebyshev-Jacobi polynomial degree on S~; <= 0 => 4 (A10)   */
  double cheb_ratio;   /* interval [2/ratio, 2]; <= 0 => 30                                  */
  int kernel;          /* 0 auto, 1 force the general quadrature kernel, 2 force affine tile */
  int schur_solver;    /* S^-1: HDIV_SCHUR_CHEBYSHEV (0, reading A10), HDIV_SCHUR_AMG (1):    */
                       /* one smoothed-aggregation V-cycle (reading A9b); with     */
                       /* slabs the block-Jacobi of per-slab V-cycles (reading A9c), or      */
                       /* HDIV_SCHUR_AUTO (2: AMG at >= 10^6 global L2 rows, else Chebyshev) */
  int amg_sweeps;      /* l1-Jacobi sweeps before and after the coarse correction; <= 0 => 2 */
  int amg_max_coarse;  /* dense solve once a level has <= this many rows; <= 0 => 512        */
  /* NEXT-3 (reading A21).  essential_sides: bitmask of domain sides whose RT
   * DOFs carry an essential (prescribed-flux) condition, eliminated by identity rows and
   * columns: bit 2a = side x_a = min, bit 2a+1 = side x_a = max (a = 0..dim-1; global sides —
   * with slabs the library applies the last-axis bits only on the first / last rank).  In
   * every apply the eliminated DOFs act as zero inputs and their outputs are the identity
   * (y_b = x_b in hdiv_apply_block / hdiv_apply_mass, 0 in hdiv_apply_divT); M~ = 1 there
   * and they are dropped from the face sets F(i) of S~.  The caller lifts inhomogeneous
   * data into b.  0 = natural conditions everywhere (A11). */
  int essential_sides;
  /* project_mean != 0: every application of S^-1 is followed by the orthogonalization step
   * of P:1038-1040 (subtract the mean of the coefficient vector, reading A11) and the AMG
   * coarsest solve pins its last unknown — for the singular pure-Neumann Darcy problem
   * (all sides essential, gamma = 0). */
  int project_mean;
  /* Trilinear (non-affine) 3D elements, mass / gamma = 0 applies: where the Piola factors
   * G_q = w_q mw_e / det J_q  J_q^T J_q come from.  0 = auto (stored when they fit: 48 Q^3 B
   * per element, <= 1/4 of the free memory), 1 = recomputed from the vertices every apply,
   * 2 = stored at setup (the paper's partial assembly: geometric factors precomputed at the
   * quadrature points; HDIV_ERR_CUDA if they do not fit).  The block apply
   * with the explicit W^-1 inverses fused (HBM-bound) always recomputes J. */
  int tri_geometry;
  /* schur_solver == HDIV_SCHUR_AMG (reading A9d): S^-1 = the degree-amg_cheb_degree Chebyshev
   * polynomial in B S~ (B = the V-cycle above) on [b / amg_cheb_ratio, b], b = 1.1 (one rank)
   * or 2.2 (slabs: block-Jacobi over a chain, spectrum <= 2) — the r/d
   * recurrence of reading A10 with B in place of D^-1, amg_cheb_degree V-cycles and
   * amg_cheb_degree - 1 S~ applies per S^-1.  1 = the plain V-cycle; <= 0 = auto:
   * one rank: 3 when the element mass weights (beta | 1/eps) span more than 10^2, else 1;
   * slabs: 1 with the A9e global coarse space (amg_global_coarse), else 3;
   * amg_cheb_ratio <= 0 => 20. */
  int amg_cheb_degree;
  double amg_cheb_ratio;
  /* schur_solver == HDIV_SCHUR_AMG with 3D slabs (reading A9e): S^-1 = B0 + (I - B0 S~) M
   * (I - S~ B0), the balancing two-level form around M = the per-slab V-cycles (or their A9d
   * polynomial) with a global coarse space, B0 = R^T A0^-1 R, R the sums over the aggregates of
   * a fixed grid of blocks of ceil(N_a / 8) elements of the global mesh, A0 = R S~ R^T (dense,
   * replicated on every rank) — it restores the slab coupling the block-Jacobi drops (per S^-1:
   * two S~ applies, two aggregate restrictions, two all-gathers of one double per aggregate).  1 = on, 2 = off, 0 = auto (on with >= 2 slabs in
   * 3D); ignored on one rank and in 2D. */
  int amg_global_coarse;
} hdiv_options;

/* HDIV_SCHUR_AUTO: the AMG V-cycle when the global L2 space has >= 10^6 rows (the Chebyshev
 * polynomial is not h-robust), else Chebyshev; the choice is made once at setup. */
enum { HDIV_SCHUR_CHEBYSHEV = 0, HDIV_SCHUR_AMG = 1, HDIV_SCHUR_AUTO = 2 };

typedef struct {
  int iters;           /* first j with |eta_j| <= rtol * gamma_1 (reading A8)         */
  int converged;       /* 0 on iteration limit (not an error)                                */
  double rel_resid;    /* |eta| / gamma_1 at exit                                            */
  double t_solve_ms;   /* device time of the solve (CUDA events on `stream`)                 */
} hdiv_report;

/* Setup (setup list of SURVEY §3): validates, uploads 1D tables, precomputes
 * per-element geometry/coefficients, assembles diag(M), diag(W), the
 * Schur approximation S~ (CSR) and allocates the MINRES workspace.
 * nccl_unique_id: 128-byte ncclUniqueId (rank 0's, broadcast by the caller) or NULL for one
 * GPU; the library creates and owns the communicator.  Blocks until setup is complete.
 * Returns the handle in *out (NULL on error). */
hdiv_status hdiv_setup(const hdiv_mesh_desc* mesh, int p, const hdiv_coeffs* coeffs,
                       hdiv_kind kind, const hdiv_options* opts,
                       const void* nccl_unique_id, int rank, int nranks,
                       void* stream, hdiv_handle* out);

void hdiv_destroy(hdiv_handle h);
const char* hdiv_status_string(hdiv_status s);
const char* hdiv_last_error(void);      /* thread-local detail of the last error              */
int hdiv_version(void);

/* Local (this rank) and global vector sizes. */
hdiv_status hdiv_sizes(hdiv_handle h, int64_t* n_rt_local, int64_t* n_l2_local,
                       int64_t* n_rt_global, int64_t* n_l2_global);

/* y_u = M_beta u  (sum-factorised).  u, y_u: [n_rt]. */
hdiv_status hdiv_apply_mass(hdiv_handle h, const double* u, double* y_u, void* stream);
/* y_q = D u  (topological +-1).  u: [n_rt], y_q: [n_l2].  Eliminated
 * essential DOFs (options.essential_sides) act as zero (the (2,1) block D F of A). */
hdiv_status hdiv_apply_div(hdiv_handle h, const double* u, double* y_q, void* stream);
/* y_u = D^T q  .  q: [n_l2], y_u: [n_rt]. */
hdiv_status hdiv_apply_divT(hdiv_handle h, const double* q, double* y_u, void* stream);
/* y = A x with A = [M, D^T; D, -Z], Z = W_alpha^-1 (grad-div) or W^-1 W_gamma W^-1 (Darcy)
 * (P:207-211).  x, y: [n_rt + n_l2].  Multi-GPU: includes the interface
 * reverse-add over NCCL. */
hdiv_status hdiv_apply_block(hdiv_handle h, const double* x, double* y, void* stream);
/* y_q = Z q: the (2,2) block alone, Z = W_alpha^-1 (grad-div) or gamma_e W^-1 (Darcy, piecewise-
 * constant gamma), P:235-238, P:535-553 — on every 3D geometry through the element-local CG in
 * the Gauss-Legendre nodal basis (exact Kronecker case converges in one
 * step); on trilinear meshes at p <= 4 through precomputed explicit element inverses built at
 * setup when they fit the memory budget (env HDIV_WINV=cg keeps the CG); 2D: the quadrature kernel (exact Kronecker inverse on parallelograms, Cholesky of the
 * quadrature-assembled W on general quadrilaterals); Z = 0 gives y_q = 0.  q, y_q: DEVICE [n_l2]. */
hdiv_status hdiv_apply_z(hdiv_handle h, const double* q, double* y_q, void* stream);
/* Same as hdiv_apply_block with HOST x, y (pinned or pageable): H2D copy, apply, D2H copy,
 * ordered after `stream`; blocks until y is on the host (end-to-end path).  On box meshes (one
 * rank) the copies and the fused apply are pipelined over ~16 chunks of element layers along z
 * on three library streams (H2D of chunk c+1 and D2H of chunk c-1 overlap the apply of chunk c;
 * the result is bitwise the device apply's; HDIV_HOST_PIPELINE=0 disables it).  Device staging
 * buffers (2 vectors) are allocated on first use. */
hdiv_status hdiv_apply_block_host(hdiv_handle h, const double* x_host, double* y_host,
                                  void* stream);
/* Device operations (kernel launches + memsets of this rank, communication excluded) that the
 * most recent hdiv_apply_block on this handle issued, counted at the launch sites; 0 before
 * the first apply (launch accounting for bench.py's gpu_launches). */
hdiv_status hdiv_apply_launches(hdiv_handle h, int* n);

/* diag(M_beta) = M~, assembled (interface-summed).  diag: [n_rt]. */
hdiv_status hdiv_assemble_mass_diag(hdiv_handle h, double* diag, void* stream);
/* C~ = W~^-1 (grad-div) or diag(W)^-1 diag(W_gamma) diag(W)^-1 (Darcy). [n_l2] */
hdiv_status hdiv_assemble_schur_diag_term(hdiv_handle h, double* ctil, void* stream);

/* S~ = C~ + D M~^-1 D^T in CSR (eq. approx-schur-entries), rows = local L2 DOFs,
 * columns sorted ascending (local numbering; multi-GPU ghost columns are not exported).
 * Query nnz first; caller allocates row_ptr[n_l2+1], col[nnz], val[nnz] (device). */
hdiv_status hdiv_schur_nnz(hdiv_handle h, int64_t* nnz);
hdiv_status hdiv_assemble_schur_csr(hdiv_handle h, int64_t* row_ptr, int64_t* col,
                                    double* val, void* stream);
/* y = S~ x (the SpMV used inside S^-1).  x, y: [n_l2]. */
hdiv_status hdiv_apply_schur(hdiv_handle h, const double* x, double* y, void* stream);
/* D in CSR by Algorithm 1: row_ptr[n_l2+1] (= 2d i), col[2d n_l2], val.  Always
 * the unmasked incidence (essential_sides does not change it). */
hdiv_status hdiv_export_div_csr(hdiv_handle h, int64_t* row_ptr, int64_t* col, double* val,
                                void* stream);
/* z = P^-1 v with P = diag(tau M~, S^), S^-1 = Chebyshev-Jacobi on S~. */
hdiv_status hdiv_apply_precond(hdiv_handle h, const double* v, double* z, void* stream);

/* Block-diagonally preconditioned MINRES for A x = b, x0 = 0, stopping at
 * |eta| <= rtol * gamma_1.  b, x: [n_rt + n_l2] device.  Blocks until done; fills
 * *report.  Non-convergence is HDIV_OK with converged = 0. */
hdiv_status hdiv_minres_solve(hdiv_handle h, const double* b, double* x, double rtol,
                              int maxit, hdiv_report* report, void* stream);

/* NEXT-4 (P:423-438 Remark): z = B^-1 v with the block upper-triangular preconditioner
 * B = [tau M~, D^T; 0, -S^] (S^-1 per options.schur_solver):  z_q = -S^-1 v_q,
 * z_u = (tau M~)^-1 (v_u - D^T z_q).  v, z: DEVICE [n_rt + n_l2].  Slabs: D^T reverse-added. */
hdiv_status hdiv_apply_precond_tri(hdiv_handle h, const double* v, double* z, void* stream);

/* NEXT-4: right-preconditioned restarted GMRES(restart) with B above, x0 = 0;
 * Arnoldi with classical Gram-Schmidt applied twice, Givens rotations; stops when the
 * least-squares residual (the true residual norm, right preconditioning) <= rtol ||b||.
 * restart <= 64; the (restart+1) basis vectors are allocated on first use (8 (restart+1) n
 * bytes).  Synchronous (host-driven Hessenberg algebra).  Slabs: every projection is
 * all-gathered and summed in rank order (the interface plane counted once), so all ranks build
 * the same Hessenberg matrix and take the same decisions. */
hdiv_status hdiv_gmres_solve(hdiv_handle h, const double* b, double* x, double rtol, int maxit,
                             int restart, hdiv_report* report, void* stream);

/* Multi-GPU helper: writes a fresh 128-byte ncclUniqueId (rank 0 calls it and broadcasts the
 * bytes, e.g. with torch.distributed, before every rank calls hdiv_setup).  NCCL is resolved
 * at run time (dlopen); HDIV_ERR_NCCL if it is unavailable. */
hdiv_status hdiv_nccl_unique_id(void* out, int64_t len);

/* Diagnostic, host only (no GPU needed): the library's 1D tables for order p with Q points
 * (reading A3: Q = p+2).  Outputs (caller-owned host arrays): xq[Q], wq[Q] Gauss-Legendre on
 * [0,1]; Bl[Q][p+1] = l_i(x_q); Bh[Q][p] = h_j(x_q); Ml[(p+1)^2], Mh[p^2], Mhinv[p^2]. */
hdiv_status hdiv_debug_tables(int p, int Q, double* xq, double* wq, double* Bl, double* Bh,
                              double* Ml, double* Mh, double* Mhinv);

/* Diagnostic, host only: the Gauss-Legendre nodal tables of the W^-1 local CG.
 * BG[Q][p] = L_b(x_q) (L_b the Lagrange basis on the p-point Gauss rule, x_q the Q-point rule);
 * HG[p][p] with HG[a][b] = integral of L_b over GLL subinterval a.  Caller-owned host arrays. */
/* AMG hierarchy introspection (parity tests): number of levels, and for level l the grid
 * extents dims[3] (level 0: the subcell grid), rows n, prolongator weight omega, and (levels
 * >= 1) a copy of the 3^d-point stencil into the caller's DEVICE buffer st[3^d][n] (offset
 * k = (dx+1) + 3(dy+1) + 9(dz+1), lexicographic x-fastest rows; NULL skips the copy).
 * HDIV_ERR_UNSUPPORTED if the handle has no AMG hierarchy. */
hdiv_status hdiv_amg_levels(hdiv_handle h, int* nlevels);
hdiv_status hdiv_amg_level(hdiv_handle h, int level, int64_t* dims, int64_t* n, double* omega,
                           double* st, void* stream);

hdiv_status hdiv_debug_gl_tables(int p, int Q, double* BG, double* HG);

#ifdef __cplusplus
}
#endif
#endif /* HDIV_H */
