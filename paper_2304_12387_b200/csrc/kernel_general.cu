// kernel_general.cu — element-by-element quadrature kernels for arbitrary (bi/tri)linear
// geometry in 2D and 3D:
//
//   M^e u = sum_q w_q (mw_e / det J_q) J_q^T J_q  u_hat(x_q)   tested against phi_hat
//   u_hat(x_q) by sum factorisation with the 1D tables B_l, B_h; quadrature
//   Gauss-Legendre Q = p+2 per direction (reading A3); J, det J evaluated on the fly from the
//   element's 2^d vertices (stored-G vs on-the-fly: DESIGN.md §Kernels).
//
// One CTA per element.  Face DOFs on the element boundary receive two contributions and
// are accumulated with fp64 atomics onto a zeroed output (0 + a + b is order independent,
// so results are bitwise deterministic); interior DOFs are stored.  Modes:
//   MODE_MASS   y_u  = M u
//   MODE_BLOCK  y    = [M u + D^T q ; D u - Z q]   (Z only for constant-J elements)
//   GMODE_DIAGM diag(M) (squared tables, atomics)
//   GMODE_DIAGW diag(W_1) per L2 DOF, i.e. sum_q w_q psi_a^2 / det J (store)
#include <cuda_runtime.h>

#include "internal.h"

namespace hdiv {
namespace {

enum { GMODE_MASS = 1, GMODE_BLOCK = 2, GMODE_DIAGM = 3, GMODE_DIAGW = 4, GMODE_ZONLY = 5 };

struct GenArgs {
  const double* x;      // [u ; q]  (MASS: u)
  double* y;            // [y_u ; y_q] (MASS/DIAGM: y_u ; DIAGW: [n_l2])
  const double* vert;   // [layers][NLy+1][NLx+1][dim]
  const double* coef;   // [E][4] {mass weight, z, -, -}
  long long NL[3];
  long long n[3];
  long long off[3];
  long long nrt;
  int has_z;
  int ess;              // eliminated essential sides (NEXT-3): zero inputs, outputs skipped
  const double* gvert;  // DIAGW: weight by the trilinear gamma field (NEXT-3), else nullptr
  int dense_z;          // 2D non-affine quadrilaterals: Z = s_e W^-1 by a dense element solve
  const int* skip;
};

template <int DIM>
struct Pow;
template <>
struct Pow<2> { static constexpr int v(int a) { return a * a; } };
template <>
struct Pow<3> { static constexpr int v(int a) { return a * a * a; } };

// out[o-index replaces axis ax] = sum_t T(o,t) in[t at axis ax]; dims d[0..2] of `in`
// (d[0] fastest).  T(o,t) = tab[o*so + t*st].
template <int NT>
__device__ __forceinline__ void contract(const double* in, double* out, const double* tab,
                                         int so, int st, int nin, int nout, int ax, int d0,
                                         int d1, int d2) {
  int e0 = d0, e1 = d1, e2 = d2;
  if (ax == 0) e0 = nout; else if (ax == 1) e1 = nout; else e2 = nout;
  const int total = e0 * e1 * e2;
  for (int it = threadIdx.x; it < total; it += NT) {
    int o0 = it % e0, r = it / e0, o1 = r % e1, o2 = r / e1;
    double s = 0.0;
    if (ax == 0) {
      const double* b = in + (o2 * d1 + o1) * d0;
      for (int t = 0; t < nin; ++t) s = fma(tab[o0 * so + t * st], b[t], s);
    } else if (ax == 1) {
      const double* b = in + o2 * d1 * d0 + o0;
      for (int t = 0; t < nin; ++t) s = fma(tab[o1 * so + t * st], b[t * d0], s);
    } else {
      const double* b = in + o1 * d0 + o0;
      for (int t = 0; t < nin; ++t) s = fma(tab[o2 * so + t * st], b[t * d0 * d1], s);
    }
    out[it] = s;
  }
}

template <int DIM, int P, int NT, int MODE>
__global__ void __launch_bounds__(NT) general_kernel(const GenArgs a,
                                                     const __grid_constant__ Tab1D tab) {
  constexpr int Q = P + 2;
  constexpr int NQ = Pow<DIM>::v(Q);
  constexpr int NC = (P + 1) * Pow<DIM>::v(P) / P;     // DOFs per component
  constexpr int NL2 = Pow<DIM>::v(P);
  constexpr bool BLOCK = (MODE == GMODE_BLOCK);
  constexpr bool ZO = (MODE == GMODE_ZONLY);   // y = Z q alone (hdiv_apply_z, 2D)
  if (a.skip && *a.skip) return;
  __shared__ double sBl[Q * (P + 1)], sBh[Q * P], sw[Q], sx[Q];
  __shared__ double sX[8 * 3];
  __shared__ double su[DIM * NC];      // inputs u^c (local tensor order, i fastest)
  __shared__ double sV[DIM * NQ];      // quadrature values per component
  __shared__ double sT1[NQ], sT2[NQ];  // contraction scratch
  __shared__ double sq[BLOCK || ZO ? NL2 : 1], sy[BLOCK || ZO || MODE == GMODE_DIAGW ? NL2 : 1];
  __shared__ double sMhi[P * P];
  __shared__ double scoef[2];
  __shared__ double sG[8];   // vertex gamma values (DIAGW with a.gvert)
  // 2D non-affine: the element's W (P^2 x P^2) for the dense Cholesky solve of Z
  __shared__ double sW[(DIM == 2 && (BLOCK || ZO)) ? Pow<DIM>::v(P) * Pow<DIM>::v(P) : 1];

  const int tid = threadIdx.x;
  const long long e = blockIdx.x;
  const long long NLx = a.NL[0], NLy = a.NL[1];
  const int ex = (int)(e % NLx);
  const int ey = (int)((e / NLx) % NLy);
  const int ez = (DIM == 3) ? (int)(e / (NLx * NLy)) : 0;
  const bool SQUARE = (MODE == GMODE_DIAGM || MODE == GMODE_DIAGW);

  for (int i = tid; i < Q * (P + 1); i += NT) {
    double v = tab.Bl[i / (P + 1)][i % (P + 1)];
    sBl[i] = SQUARE ? v * v : v;
  }
  for (int i = tid; i < Q * P; i += NT) {
    double v = tab.Bh[i / P][i % P];
    sBh[i] = SQUARE ? v * v : v;
  }
  for (int i = tid; i < Q; i += NT) { sw[i] = tab.wq[i]; sx[i] = tab.xq[i]; }
  for (int i = tid; i < P * P; i += NT) sMhi[i] = tab.Mhinv[i / P][i % P];
  if (tid < 2) scoef[tid] = a.coef[4 * e + tid];
  for (int i = tid; i < (1 << DIM) * DIM; i += NT) {
    int v = i / DIM, d = i % DIM;
    int ca = v & 1, cb = (v >> 1) & 1, cc = (v >> 2) & 1;
    long long g = (DIM == 3)
                      ? (((long long)(ez + cc) * (NLy + 1) + (ey + cb)) * (NLx + 1) + (ex + ca))
                      : ((long long)(ey + cb) * (NLx + 1) + (ex + ca));
    sX[v * DIM + d] = a.vert[g * DIM + d];
    if (DIM == 3 && MODE == GMODE_DIAGW && a.gvert && d == 0) sG[v] = a.gvert[g];
  }
  const long long nx = a.n[0], ny = a.n[1];
  // global index of local DOF (component c, local tensor index (i,j,k))
  auto gidx = [&](int c, int i, int j, int k) -> long long {
    long long I = (long long)ex * P + i, J = (long long)ey * P + j, K = (long long)ez * P + k;
    if (DIM == 2) {
      if (c == 0) return a.off[0] + I + (nx + 1) * J;
      return a.off[1] + I + nx * J;
    }
    if (c == 0) return a.off[0] + I + (nx + 1) * (J + ny * K);
    if (c == 1) return a.off[1] + I + nx * (J + (ny + 1) * K);
    return a.off[2] + I + nx * (J + ny * K);
  };
  // component c local extents (n0 fastest): P+1 along axis c, P elsewhere
  auto ext = [&](int c, int ax) -> int { return ax == c ? P + 1 : P; };

  if (MODE == GMODE_MASS || BLOCK) {
    for (int i = tid; i < DIM * NC; i += NT) {
      int c = i / NC, l = i % NC;
      int n0 = ext(c, 0), n1 = ext(c, 1);
      int ii = l % n0, jj = (l / n0) % n1, kk = (DIM == 3) ? l / (n0 * n1) : 0;
      double v = a.x[gidx(c, ii, jj, kk)];
      if (a.ess) {   // eliminated essential face: acts as zero (NEXT-3)
        const long long gi = (c == 0) ? (long long)ex * P + ii : (c == 1) ? (long long)ey * P + jj
                                                                         : (long long)ez * P + kk;
        if (face_masked(a.ess, c, gi, a.n[c])) v = 0.0;
      }
      su[i] = v;
    }
  }
  if constexpr (BLOCK || ZO) {
    const double* q = ZO ? a.x : a.x + a.nrt;
    for (int i = tid; i < NL2; i += NT) sq[i] = q[e * NL2 + i];
  }
  __syncthreads();

  // ---- D u - Z q (element-local) ----
  if constexpr (BLOCK || ZO) {
    for (int i = tid; i < NL2; i += NT) {
      if constexpr (ZO) { sy[i] = 0.0; continue; }
      int A = i % P, B = (i / P) % P, C = (DIM == 3) ? i / (P * P) : 0;
      double d = 0.0;
      // x faces: component 0 index A + (P+1)(B + P C)
      d += su[(A + 1) + (P + 1) * (B + P * C)] - su[A + (P + 1) * (B + P * C)];
      // y faces: component 1 index A + P(B + (P+1) C)
      d += su[NC + A + P * ((B + 1) + (P + 1) * C)] - su[NC + A + P * (B + (P + 1) * C)];
      if (DIM == 3)
        d += su[2 * NC + A + P * (B + P * (C + 1))] - su[2 * NC + A + P * (B + P * C)];
      sy[i] = d;
    }
    if (DIM == 2 && a.has_z && a.dense_z) {
      // 2D non-affine quadrilateral: Z q = s_e W^-1 q with W_ab = sum_q w_q psi_a psi_b / det J_q
      // (P:117), psi_a = h_i(x) h_j(y); W assembled by quadrature, factored by a
      // right-looking Cholesky across the CTA, solved by substitution
      constexpr int N = NL2;
      for (int qi = tid; qi < Q * Q; qi += NT) {   // w_q / det J_q at the Q^2 points -> sT1
        const int qx = qi % Q, qy = qi / Q;
        const double xh = sx[qx], yh = sx[qy];
        const double* X = sX;
        double J[2][2];
        for (int d = 0; d < 2; ++d) {
          J[d][0] = (1 - yh) * (X[1 * 2 + d] - X[0 * 2 + d]) + yh * (X[3 * 2 + d] - X[2 * 2 + d]);
          J[d][1] = (1 - xh) * (X[2 * 2 + d] - X[0 * 2 + d]) + xh * (X[3 * 2 + d] - X[1 * 2 + d]);
        }
        sT1[qi] = sw[qx] * sw[qy] / (J[0][0] * J[1][1] - J[0][1] * J[1][0]);
      }
      __syncthreads();
      for (int idx = tid; idx < N * N; idx += NT) {
        const int ra = idx / N, cb = idx % N;
        const int i1 = ra % P, j1 = ra / P, i2 = cb % P, j2 = cb / P;
        double w = 0.0;
        for (int qy = 0; qy < Q; ++qy) {
          double t = 0.0;
          for (int qx = 0; qx < Q; ++qx) t = fma(sT1[qx + Q * qy], sBh[qx * P + i1] * sBh[qx * P + i2], t);
          w = fma(t, sBh[qy * P + j1] * sBh[qy * P + j2], w);
        }
        sW[idx] = w;
      }
      __syncthreads();
      for (int k = 0; k < N; ++k) {   // W = L L^T in place (lower triangle)
        if (tid == 0) sW[k * N + k] = sqrt(sW[k * N + k]);
        __syncthreads();
        for (int i = k + 1 + tid; i < N; i += NT) sW[i * N + k] /= sW[k * N + k];
        __syncthreads();
        for (int idx = tid; idx < (N - k - 1) * (N - k - 1); idx += NT) {
          const int i = k + 1 + idx / (N - k - 1), j = k + 1 + idx % (N - k - 1);
          if (j <= i) sW[i * N + j] -= sW[i * N + k] * sW[j * N + k];
        }
        __syncthreads();
      }
      if (tid == 0) {   // L y = q, L^T z = y  -> sT2
        for (int i = 0; i < N; ++i) {
          double v = sq[i];
          for (int j = 0; j < i; ++j) v -= sW[i * N + j] * sT2[j];
          sT2[i] = v / sW[i * N + i];
        }
        for (int i = N - 1; i >= 0; --i) {
          double v = sT2[i];
          for (int j = i + 1; j < N; ++j) v -= sW[j * N + i] * sT2[j];
          sT2[i] = v / sW[i * N + i];
        }
      }
      __syncthreads();
      for (int i = tid; i < NL2; i += NT) sy[i] -= scoef[1] * sT2[i];
    } else if (a.has_z) {
      // Z q = z (Mh^-1)^{(x)d} q   (constant-J elements)
      contract<NT>(sq, sT1, sMhi, P, 1, P, P, 0, P, P, DIM == 3 ? P : 1);
      __syncthreads();
      contract<NT>(sT1, sT2, sMhi, P, 1, P, P, 1, P, P, DIM == 3 ? P : 1);
      __syncthreads();
      if (DIM == 3) {
        contract<NT>(sT2, sT1, sMhi, P, 1, P, P, 2, P, P, P);
        __syncthreads();
      }
      const double* zq = (DIM == 3) ? sT1 : sT2;
      for (int i = tid; i < NL2; i += NT) sy[i] -= scoef[1] * zq[i];
    }
    __syncthreads();
    if constexpr (ZO) {   // y = Z q = -(0 - Z q)
      for (int i = tid; i < NL2; i += NT) a.y[e * NL2 + i] = -sy[i];
      return;
    }
  }

  // ---- forward: component values at quadrature points ----
  if (MODE == GMODE_MASS || BLOCK) {
    for (int c = 0; c < DIM; ++c) {
      const double* in = su + c * NC;
      double* V = sV + c * NQ;
      int d0 = ext(c, 0), d1 = ext(c, 1), d2 = (DIM == 3) ? ext(c, 2) : 1;
      // axis 0
      const double* t0 = (c == 0) ? sBl : sBh;
      int st0 = (c == 0) ? 1 : 1, so0 = (c == 0) ? (P + 1) : P;
      contract<NT>(in, sT1, t0, so0, st0, d0, Q, 0, d0, d1, d2);
      __syncthreads();
      const double* t1 = (c == 1) ? sBl : sBh;
      int so1 = (c == 1) ? (P + 1) : P;
      contract<NT>(sT1, (DIM == 3) ? sT2 : V, t1, so1, 1, d1, Q, 1, Q, d1, d2);
      __syncthreads();
      if (DIM == 3) {
        const double* t2 = (c == 2) ? sBl : sBh;
        int so2 = (c == 2) ? (P + 1) : P;
        contract<NT>(sT2, V, t2, so2, 1, d2, Q, 2, Q, Q, d2);
        __syncthreads();
      }
    }
  }

  // ---- quadrature-point operator ----
  for (int qi = tid; qi < NQ; qi += NT) {
    int qx = qi % Q, qy = (qi / Q) % Q, qz = (DIM == 3) ? qi / (Q * Q) : 0;
    double xh = sx[qx], yh = sx[qy], zh = (DIM == 3) ? sx[qz] : 0.0;
    double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    double det;
    if (DIM == 2) {
      const double* X = sX;   // X[v*2+d], v = a + 2b
      for (int d = 0; d < 2; ++d) {
        J[d][0] = (1 - yh) * (X[1 * 2 + d] - X[0 * 2 + d]) + yh * (X[3 * 2 + d] - X[2 * 2 + d]);
        J[d][1] = (1 - xh) * (X[2 * 2 + d] - X[0 * 2 + d]) + xh * (X[3 * 2 + d] - X[1 * 2 + d]);
      }
      det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    } else {
      const double* X = sX;   // X[v*3+d], v = a + 2b + 4c
      for (int d = 0; d < 3; ++d) {
        auto x = [&](int va, int vb, int vc) { return X[(va + 2 * vb + 4 * vc) * 3 + d]; };
        J[d][0] = (1 - yh) * (1 - zh) * (x(1, 0, 0) - x(0, 0, 0)) + yh * (1 - zh) * (x(1, 1, 0) - x(0, 1, 0)) +
                  (1 - yh) * zh * (x(1, 0, 1) - x(0, 0, 1)) + yh * zh * (x(1, 1, 1) - x(0, 1, 1));
        J[d][1] = (1 - xh) * (1 - zh) * (x(0, 1, 0) - x(0, 0, 0)) + xh * (1 - zh) * (x(1, 1, 0) - x(1, 0, 0)) +
                  (1 - xh) * zh * (x(0, 1, 1) - x(0, 0, 1)) + xh * zh * (x(1, 1, 1) - x(1, 0, 1));
        J[d][2] = (1 - xh) * (1 - yh) * (x(0, 0, 1) - x(0, 0, 0)) + xh * (1 - yh) * (x(1, 0, 1) - x(1, 0, 0)) +
                  (1 - xh) * yh * (x(0, 1, 1) - x(0, 1, 0)) + xh * yh * (x(1, 1, 1) - x(1, 1, 0));
      }
      det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
            J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
            J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
    }
    double wq = sw[qx] * sw[qy] * (DIM == 3 ? sw[qz] : 1.0);
    if (MODE == GMODE_DIAGW) {
      double gw = 1.0;
      if (DIM == 3 && a.gvert) {   // gamma(x_hat_q), trilinear in the vertex values
        gw = 0.0;
        for (int v = 0; v < 8; ++v)
          gw += sG[v] * ((v & 1) ? xh : 1 - xh) * ((v & 2) ? yh : 1 - yh) * ((v & 4) ? zh : 1 - zh);
      }
      sT1[qi] = gw * wq / det;
      continue;
    }
    double s = wq * scoef[0] / det;
    if (MODE == GMODE_DIAGM) {   // G_cc = (J^T J)_cc
      for (int c = 0; c < DIM; ++c) {
        double g = 0.0;
        for (int d = 0; d < DIM; ++d) g += J[d][c] * J[d][c];
        sV[c * NQ + qi] = s * g;
      }
      continue;
    }
    double uh[3], Ju[3];
    for (int c = 0; c < DIM; ++c) uh[c] = sV[c * NQ + qi];
    for (int d = 0; d < DIM; ++d) {
      double t = 0.0;
      for (int c = 0; c < DIM; ++c) t += J[d][c] * uh[c];
      Ju[d] = t;
    }
    for (int c = 0; c < DIM; ++c) {
      double t = 0.0;
      for (int d = 0; d < DIM; ++d) t += J[d][c] * Ju[d];
      sV[c * NQ + qi] = s * t;
    }
  }
  __syncthreads();

  if constexpr (MODE == GMODE_DIAGW) {
    // sum_q (w/det) psi_a^2 with squared h tables
    contract<NT>(sT1, sT2, sBh, 1, P, Q, P, 0, Q, Q, DIM == 3 ? Q : 1);
    __syncthreads();
    contract<NT>(sT2, (DIM == 3) ? sT1 : sy, sBh, 1, P, Q, P, 1, P, Q, DIM == 3 ? Q : 1);
    __syncthreads();
    if (DIM == 3) {
      contract<NT>(sT1, sy, sBh, 1, P, Q, P, 2, P, P, Q);
      __syncthreads();
    }
    for (int i = tid; i < NL2; i += NT) a.y[e * NL2 + i] = sy[i];
    return;
  } else {
    // ---- backward: test against phi_hat, then scatter ----
    for (int c = 0; c < DIM; ++c) {
      double* V = sV + c * NQ;
      int d0 = ext(c, 0), d1 = ext(c, 1), d2 = (DIM == 3) ? ext(c, 2) : 1;
      double* out;
      if (DIM == 3) {
        const double* t2 = (c == 2) ? sBl : sBh;
        int n2 = (c == 2) ? (P + 1) : P;
        contract<NT>(V, sT1, t2, 1, n2, Q, d2, 2, Q, Q, Q);   // T(o=k,t=q) = B[q][k]
        __syncthreads();
        const double* t1 = (c == 1) ? sBl : sBh;
        int n1 = (c == 1) ? (P + 1) : P;
        contract<NT>(sT1, sT2, t1, 1, n1, Q, d1, 1, Q, Q, d2);
        __syncthreads();
        const double* t0 = (c == 0) ? sBl : sBh;
        int n0 = (c == 0) ? (P + 1) : P;
        contract<NT>(sT2, sT1, t0, 1, n0, Q, d0, 0, Q, d1, d2);
        __syncthreads();
        out = sT1;
      } else {
        const double* t1 = (c == 1) ? sBl : sBh;
        int n1 = (c == 1) ? (P + 1) : P;
        contract<NT>(V, sT1, t1, 1, n1, Q, d1, 1, Q, Q, 1);
        __syncthreads();
        const double* t0 = (c == 0) ? sBl : sBh;
        int n0 = (c == 0) ? (P + 1) : P;
        contract<NT>(sT1, sT2, t0, 1, n0, Q, d0, 0, Q, d1, 1);
        __syncthreads();
        out = sT2;
      }
      for (int l = tid; l < NC; l += NT) {
        int ii = l % d0, jj = (l / d0) % d1, kk = (DIM == 3) ? l / (d0 * d1) : 0;
        double v = out[l];
        int ic = (c == 0) ? ii : (c == 1) ? jj : kk;   // index along the normal axis
        if constexpr (BLOCK) {
          // (D^T q)_face: + q(cell on - side, inside this element), - q(cell on + side)
          int A = ii, B = jj, C = kk;
          if (ic > 0) {
            int cm = (c == 0) ? (A - 1) + P * (B + P * C)
                   : (c == 1) ? A + P * ((B - 1) + P * C) : A + P * (B + P * (C - 1));
            v += sq[cm];
          }
          if (ic < P) {
            int cp = A + P * (B + P * C);
            v -= sq[cp];
          }
        }
        long long g = gidx(c, ii, jj, kk);
        if (ic == 0 || ic == P) {
          const long long gi = (c == 0) ? (long long)ex * P + ii : (c == 1) ? (long long)ey * P + jj
                                                                           : (long long)ez * P + kk;
          if (!(a.ess && face_masked(a.ess, c, gi, a.n[c]))) atomicAdd(a.y + g, v);
        } else {
          a.y[g] = v;
        }
      }
      __syncthreads();
    }
    if constexpr (BLOCK) {
      double* yq = a.y + a.nrt;
      for (int i = tid; i < NL2; i += NT) yq[e * NL2 + i] = sy[i];
    }
  }
}

template <int DIM, int P, int MODE>
cudaError_t launch_g(const hdiv_ctx* h, const double* x, double* y, const int* skip,
                     cudaStream_t s) {
  constexpr int NT = (DIM == 3) ? 128 : 64;
  GenArgs a;
  a.x = x; a.y = y; a.vert = h->d_vert; a.coef = h->d_coef;
  for (int d = 0; d < 3; ++d) { a.NL[d] = h->NL[d]; a.n[d] = h->n[d]; a.off[d] = h->off[d]; }
  a.nrt = h->nrt;
  a.has_z = h->has_z ? 1 : 0;
  a.ess = (MODE == GMODE_MASS || MODE == GMODE_BLOCK) ? h->ess : 0;
  a.gvert = nullptr;
  a.dense_z = (DIM == 2 && h->geom == GEOM_TRILINEAR) ? 1 : 0;
  if (MODE == GMODE_ZONLY) a.has_z = 1;
  a.skip = skip;
  count_op();
  general_kernel<DIM, P, NT, MODE><<<(unsigned)h->E, NT, 0, s>>>(a, h->tab);
  return cudaGetLastError();
}

template <int MODE>
cudaError_t dispatch(const hdiv_ctx* h, const double* x, double* y, const int* k,
                     cudaStream_t s) {
  if (h->dim == 2) {
    switch (h->p) {
      case 1: return launch_g<2, 1, MODE>(h, x, y, k, s);
      case 2: return launch_g<2, 2, MODE>(h, x, y, k, s);
      case 3: return launch_g<2, 3, MODE>(h, x, y, k, s);
      case 4: return launch_g<2, 4, MODE>(h, x, y, k, s);
      case 5: return launch_g<2, 5, MODE>(h, x, y, k, s);
      case 6: return launch_g<2, 6, MODE>(h, x, y, k, s);
    }
  } else {
    switch (h->p) {
      case 1: return launch_g<3, 1, MODE>(h, x, y, k, s);
      case 2: return launch_g<3, 2, MODE>(h, x, y, k, s);
      case 3: return launch_g<3, 3, MODE>(h, x, y, k, s);
      case 4: return launch_g<3, 4, MODE>(h, x, y, k, s);
      case 5: return launch_g<3, 5, MODE>(h, x, y, k, s);
      case 6: return launch_g<3, 6, MODE>(h, x, y, k, s);
    }
  }
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_general_apply(const hdiv_ctx* h, const double* x, double* y, int mode,
                                 const int* skip, cudaStream_t s) {
  count_op();
  cudaError_t e = cudaMemsetAsync(y, 0, sizeof(double) * h->nrt, s);
  if (e != cudaSuccess) return e;
  if (mode == MODE_BLOCK) return dispatch<GMODE_BLOCK>(h, x, y, skip, s);
  return dispatch<GMODE_MASS>(h, x, y, skip, s);
}

// y = Z q, the (2,2) block alone, 2D (3D: the trilinear kernel's W^-1 path)
cudaError_t launch_general_z(const hdiv_ctx* h, const double* q, double* y, cudaStream_t s) {
  return dispatch<GMODE_ZONLY>(h, q, y, nullptr, s);
}

cudaError_t launch_mass_diag(const hdiv_ctx* h, double* diag, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(diag, 0, sizeof(double) * h->nrt, s);
  if (e != cudaSuccess) return e;
  return dispatch<GMODE_DIAGM>(h, nullptr, diag, nullptr, s);
}

// diag(W_1) per L2 DOF into `w1` (sum_q w_q psi_hat_a^2 / det J)
cudaError_t launch_l2_diag(const hdiv_ctx* h, double* w1, cudaStream_t s) {
  return dispatch<GMODE_DIAGW>(h, nullptr, w1, nullptr, s);
}

// diag(W_gamma) per L2 DOF for the general (vertex-field) gamma, 3D (NEXT-3)
template <int P>
static cudaError_t launch_wg(const hdiv_ctx* h, double* wg, cudaStream_t s) {
  GenArgs a;
  a.x = nullptr; a.y = wg; a.vert = h->d_vert; a.coef = h->d_coef;
  for (int d = 0; d < 3; ++d) { a.NL[d] = h->NL[d]; a.n[d] = h->n[d]; a.off[d] = h->off[d]; }
  a.nrt = h->nrt;
  a.has_z = 0;
  a.ess = 0;
  a.gvert = h->d_gvert;
  a.dense_z = 0;
  a.skip = nullptr;
  general_kernel<3, P, 128, GMODE_DIAGW><<<(unsigned)h->E, 128, 0, s>>>(a, h->tab);
  return cudaGetLastError();
}

cudaError_t launch_l2_diag_gamma(const hdiv_ctx* h, double* wg, cudaStream_t s) {
  switch (h->p) {
    case 1: return launch_wg<1>(h, wg, s);
    case 2: return launch_wg<2>(h, wg, s);
    case 3: return launch_wg<3>(h, wg, s);
    case 4: return launch_wg<4>(h, wg, s);
    case 5: return launch_wg<5>(h, wg, s);
    case 6: return launch_wg<6>(h, wg, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace hdiv
