// kernel_trilinear.cu — 3D block-operator apply on (tri)linear hexahedra, element by element.
//
//   M^e u = sum_q w_q (mw_e / det J_q) J_q^T J_q u_hat(x_q) tested against phi_hat
//   (P:84 Piola, P:135 eq. matrices), Gauss-Legendre Q = p+2 (reading A3).
//
// One CTA per element, all three components advanced together so a sum-factorisation stage
// costs one barrier: 3 forward contractions (B_l / B_h tables), the pointwise G_q = w mw
// J^T J / det J (J from per-element column factors: dT/dx_hat depends on (y_hat,z_hat) only,
// etc., so the three columns are tabulated on the Q^2 faces once), 3 transposed contractions,
// then D^T q~ and the scatter (fp64 atomics on element-boundary faces onto a zeroed y, plain
// stores inside).  All extents are compile-time.  Z (constant-J elements only) and D u are
// element-local.  Bound: FP64 issue.
#include <cuda_runtime.h>

#include "internal.h"

namespace hdiv {
namespace {

struct TriArgs {
  const double* x;      // [u ; q]  (MASS: u)
  double* y;            // zeroed RT part on entry
  const double* vert;   // [layers][NLy+1][NLx+1][3]
  const double* coef;   // [E][4] {mass weight, z, -, -}
  long long NL[3];
  long long n[3];
  long long off[3];
  long long nrt;
  int has_z;
  const int* skip;
};

// out(i0,i1,i2) = sum_t T[o][t] in(.. t at axis AX ..); in extents (N0,N1,N2), out extent NO
// along AX; T(o, t) = tab[o*SO + t*ST].  Thread-strided over the outputs.
template <int NT, int N0, int N1, int N2, int AX, int NO, int SO, int ST>
__device__ __forceinline__ void contract(const double* in, double* out, const double* tab) {
  constexpr int NIN = (AX == 0) ? N0 : (AX == 1) ? N1 : N2;
  constexpr int E0 = (AX == 0) ? NO : N0;
  constexpr int E1 = (AX == 1) ? NO : N1;
  constexpr int E2 = (AX == 2) ? NO : N2;
  constexpr int TOT = E0 * E1 * E2;
  constexpr int SIN = (AX == 0) ? 1 : (AX == 1) ? N0 : N0 * N1;
#pragma unroll 2
  for (int it = threadIdx.x; it < TOT; it += NT) {
    const int o0 = it % E0, r = it / E0, o1 = r % E1, o2 = r / E1;
    const int o = (AX == 0) ? o0 : (AX == 1) ? o1 : o2;
    const double* b = in + (AX == 0 ? 0 : o0) + (AX == 1 ? 0 : o1 * N0) + (AX == 2 ? 0 : o2 * N0 * N1);
    double s = 0.0;
#pragma unroll
    for (int t = 0; t < NIN; ++t) s = fma(tab[o * SO + t * ST], b[t * SIN], s);
    out[it] = s;
  }
}

template <int P, int NT, bool BLOCK>
__global__ void __launch_bounds__(NT) tri_kernel(const TriArgs a, const __grid_constant__ Tab1D tab) {
  constexpr int Q = P + 2;
  constexpr int NQ = Q * Q * Q;
  constexpr int NC = (P + 1) * P * P;
  constexpr int P3 = P * P * P;
  if (a.skip && *a.skip) return;
  __shared__ double sBl[Q * (P + 1)], sBh[Q * P], sw[Q], sx[Q], sMhi[P * P];
  __shared__ double sX[8 * 3];
  __shared__ double sJ[3][Q * Q][3];   // column factors: sJ[c][pair][d] = dT_d/dx_hat_c
  __shared__ double su[3 * NC];        // inputs / outputs per component
  __shared__ double sT1[3 * NQ], sT2[3 * NQ];
  double* const sV = sT1;              // V is live only while T1 is dead (F3 .. B1)
  __shared__ double sq[BLOCK ? P3 : 1], sy[BLOCK ? P3 : 1], sz1[BLOCK ? P3 : 1], sz2[BLOCK ? P3 : 1];
  __shared__ double scoef[2];

  const int tid = threadIdx.x;
  const long long e = blockIdx.x;
  const long long NLx = a.NL[0], NLy = a.NL[1];
  const int ex = (int)(e % NLx), ey = (int)((e / NLx) % NLy), ez = (int)(e / (NLx * NLy));
  const long long nx = a.n[0], ny = a.n[1];

  for (int i = tid; i < Q * (P + 1); i += NT) sBl[i] = tab.Bl[i / (P + 1)][i % (P + 1)];
  for (int i = tid; i < Q * P; i += NT) sBh[i] = tab.Bh[i / P][i % P];
  for (int i = tid; i < Q; i += NT) { sw[i] = tab.wq[i]; sx[i] = tab.xq[i]; }
  for (int i = tid; i < P * P; i += NT) sMhi[i] = tab.Mhinv[i / P][i % P];
  if (tid < 2) scoef[tid] = a.coef[4 * e + tid];
  for (int i = tid; i < 24; i += NT) {
    const int v = i / 3, d = i % 3;
    const long long g = ((long long)(ez + (v >> 2)) * (NLy + 1) + (ey + ((v >> 1) & 1))) * (NLx + 1) +
                        (ex + (v & 1));
    sX[i] = a.vert[g * 3 + d];
  }
  // gather u (component c, local (i,j,k), i fastest; extent P+1 along c)
  for (int i = tid; i < 3 * NC; i += NT) {
    const int c = i / NC, l = i % NC;
    int li, lj, lk;
    long long g;
    if (c == 0) {
      li = l % (P + 1); lj = (l / (P + 1)) % P; lk = l / ((P + 1) * P);
      g = a.off[0] + (ex * P + li) + (nx + 1) * ((ey * P + lj) + ny * (long long)(ez * P + lk));
    } else if (c == 1) {
      li = l % P; lj = (l / P) % (P + 1); lk = l / (P * (P + 1));
      g = a.off[1] + (ex * P + li) + nx * ((ey * P + lj) + (ny + 1) * (long long)(ez * P + lk));
    } else {
      li = l % P; lj = (l / P) % P; lk = l / (P * P);
      g = a.off[2] + (ex * P + li) + nx * ((ey * P + lj) + ny * (long long)(ez * P + lk));
    }
    su[i] = a.x[g];
  }
  if constexpr (BLOCK) {
    const double* q = a.x + a.nrt;
    for (int i = tid; i < P3; i += NT) sq[i] = q[e * P3 + i];
  }
  __syncthreads();

  // column factors of the trilinear Jacobian on the Q x Q point pairs
  for (int i = tid; i < 3 * Q * Q * 3; i += NT) {
    const int c = i / (Q * Q * 3), r = i % (Q * Q * 3), pr = r / 3, d = r % 3;
    const double s = sx[pr % Q], t = sx[pr / Q];
    auto X = [&](int va, int vb, int vc) { return sX[(va + 2 * vb + 4 * vc) * 3 + d]; };
    double v;
    if (c == 0)        // (s,t) = (y,z)
      v = (1 - s) * (1 - t) * (X(1, 0, 0) - X(0, 0, 0)) + s * (1 - t) * (X(1, 1, 0) - X(0, 1, 0)) +
          (1 - s) * t * (X(1, 0, 1) - X(0, 0, 1)) + s * t * (X(1, 1, 1) - X(0, 1, 1));
    else if (c == 1)   // (s,t) = (x,z)
      v = (1 - s) * (1 - t) * (X(0, 1, 0) - X(0, 0, 0)) + s * (1 - t) * (X(1, 1, 0) - X(1, 0, 0)) +
          (1 - s) * t * (X(0, 1, 1) - X(0, 0, 1)) + s * t * (X(1, 1, 1) - X(1, 0, 1));
    else               // (s,t) = (x,y)
      v = (1 - s) * (1 - t) * (X(0, 0, 1) - X(0, 0, 0)) + s * (1 - t) * (X(1, 0, 1) - X(1, 0, 0)) +
          (1 - s) * t * (X(0, 1, 1) - X(0, 1, 0)) + s * t * (X(1, 1, 1) - X(1, 1, 0));
    sJ[c][pr][d] = v;
  }
  // forward stage 1 (axis 0) for the 3 components, + D u and Z stage 1
  contract<NT, P + 1, P, P, 0, Q, P + 1, 1>(su, sT1, sBl);
  contract<NT, P, P + 1, P, 0, Q, P, 1>(su + NC, sT1 + NQ, sBh);
  contract<NT, P, P, P + 1, 0, Q, P, 1>(su + 2 * NC, sT1 + 2 * NQ, sBh);
  if constexpr (BLOCK) {
    for (int i = tid; i < P3; i += NT) {
      const int A = i % P, B = (i / P) % P, C = i / (P * P);
      double d = su[(A + 1) + (P + 1) * (B + P * C)] - su[A + (P + 1) * (B + P * C)];
      d += su[NC + A + P * ((B + 1) + (P + 1) * C)] - su[NC + A + P * (B + (P + 1) * C)];
      d += su[2 * NC + A + P * (B + P * (C + 1))] - su[2 * NC + A + P * (B + P * C)];
      sy[i] = d;
    }
    if (a.has_z) contract<NT, P, P, P, 0, P, P, 1>(sq, sz1, sMhi);
  }
  __syncthreads();
  // forward stage 2 (axis 1)
  contract<NT, Q, P, P, 1, Q, P, 1>(sT1, sT2, sBh);
  contract<NT, Q, P + 1, P, 1, Q, P + 1, 1>(sT1 + NQ, sT2 + NQ, sBl);
  contract<NT, Q, P, P + 1, 1, Q, P, 1>(sT1 + 2 * NQ, sT2 + 2 * NQ, sBh);
  if constexpr (BLOCK) if (a.has_z) contract<NT, P, P, P, 1, P, P, 1>(sz1, sz2, sMhi);
  __syncthreads();
  // forward stage 3 (axis 2)
  contract<NT, Q, Q, P, 2, Q, P, 1>(sT2, sV, sBh);
  contract<NT, Q, Q, P, 2, Q, P, 1>(sT2 + NQ, sV + NQ, sBh);
  contract<NT, Q, Q, P + 1, 2, Q, P + 1, 1>(sT2 + 2 * NQ, sV + 2 * NQ, sBl);
  if constexpr (BLOCK) if (a.has_z) contract<NT, P, P, P, 2, P, P, 1>(sz2, sz1, sMhi);
  __syncthreads();
  // pointwise G_q = w_q mw / det J  J^T J
  const double mw = scoef[0];
  for (int qi = tid; qi < NQ; qi += NT) {
    const int qx = qi % Q, qy = (qi / Q) % Q, qz = qi / (Q * Q);
    const double* c0 = sJ[0][qy + Q * qz];
    const double* c1 = sJ[1][qx + Q * qz];
    const double* c2 = sJ[2][qx + Q * qy];
    const double det = c0[0] * (c1[1] * c2[2] - c1[2] * c2[1]) - c1[0] * (c0[1] * c2[2] - c0[2] * c2[1]) +
                       c2[0] * (c0[1] * c1[2] - c0[2] * c1[1]);
    const double s = sw[qx] * sw[qy] * sw[qz] * mw / det;
    const double u0 = sV[qi], u1 = sV[NQ + qi], u2 = sV[2 * NQ + qi];
    double Ju[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) Ju[d] = c0[d] * u0 + c1[d] * u1 + c2[d] * u2;
    sV[qi] = s * (c0[0] * Ju[0] + c0[1] * Ju[1] + c0[2] * Ju[2]);
    sV[NQ + qi] = s * (c1[0] * Ju[0] + c1[1] * Ju[1] + c1[2] * Ju[2]);
    sV[2 * NQ + qi] = s * (c2[0] * Ju[0] + c2[1] * Ju[1] + c2[2] * Ju[2]);
  }
  __syncthreads();
  // backward stage 1 (axis 2): T(o=k, t=q) = B[q][k]
  contract<NT, Q, Q, Q, 2, P, 1, P>(sV, sT2, sBh);
  contract<NT, Q, Q, Q, 2, P, 1, P>(sV + NQ, sT2 + NQ, sBh);
  contract<NT, Q, Q, Q, 2, P + 1, 1, P + 1>(sV + 2 * NQ, sT2 + 2 * NQ, sBl);
  __syncthreads();
  contract<NT, Q, Q, P, 1, P, 1, P>(sT2, sT1, sBh);
  contract<NT, Q, Q, P, 1, P + 1, 1, P + 1>(sT2 + NQ, sT1 + NQ, sBl);
  contract<NT, Q, Q, P + 1, 1, P, 1, P>(sT2 + 2 * NQ, sT1 + 2 * NQ, sBh);
  __syncthreads();
  contract<NT, Q, P, P, 0, P + 1, 1, P + 1>(sT1, su, sBl);
  contract<NT, Q, P + 1, P, 0, P, 1, P>(sT1 + NQ, su + NC, sBh);
  contract<NT, Q, P, P + 1, 0, P, 1, P>(sT1 + 2 * NQ, su + 2 * NC, sBh);
  __syncthreads();
  // D^T q~ and scatter
  for (int i = tid; i < 3 * NC; i += NT) {
    const int c = i / NC, l = i % NC;
    int li, lj, lk, ic;
    long long g;
    if (c == 0) {
      li = l % (P + 1); lj = (l / (P + 1)) % P; lk = l / ((P + 1) * P); ic = li;
      g = a.off[0] + (ex * P + li) + (nx + 1) * ((ey * P + lj) + ny * (long long)(ez * P + lk));
    } else if (c == 1) {
      li = l % P; lj = (l / P) % (P + 1); lk = l / (P * (P + 1)); ic = lj;
      g = a.off[1] + (ex * P + li) + nx * ((ey * P + lj) + (ny + 1) * (long long)(ez * P + lk));
    } else {
      li = l % P; lj = (l / P) % P; lk = l / (P * P); ic = lk;
      g = a.off[2] + (ex * P + li) + nx * ((ey * P + lj) + ny * (long long)(ez * P + lk));
    }
    double v = su[i];
    if constexpr (BLOCK) {
      const int cstep = (c == 0) ? 1 : (c == 1) ? P : P * P;
      const int cell = li + P * (lj + P * lk);   // valid when ic < P (the + side cell)
      if (ic > 0) v += sq[cell - cstep];
      if (ic < P) v -= sq[cell];
    }
    if (ic == 0 || ic == P) atomicAdd(a.y + g, v);
    else a.y[g] = v;
  }
  if constexpr (BLOCK) {
    double* yq = a.y + a.nrt;
    const double z = scoef[1];
    for (int i = tid; i < P3; i += NT) yq[e * P3 + i] = a.has_z ? sy[i] - z * sz1[i] : sy[i];
  }
}

template <int P, bool BLOCK>
cudaError_t launch_p(const hdiv_ctx* h, const double* x, double* y, const int* skip,
                     cudaStream_t s) {
  constexpr int NT = 128;
  TriArgs a;
  a.x = x; a.y = y; a.vert = h->d_vert; a.coef = h->d_coef;
  for (int d = 0; d < 3; ++d) { a.NL[d] = h->NL[d]; a.n[d] = h->n[d]; a.off[d] = h->off[d]; }
  a.nrt = h->nrt;
  a.has_z = h->has_z ? 1 : 0;
  a.skip = skip;
  tri_kernel<P, NT, BLOCK><<<(unsigned)h->E, NT, 0, s>>>(a, h->tab);
  return cudaGetLastError();
}

template <bool BLOCK>
cudaError_t dispatch(const hdiv_ctx* h, const double* x, double* y, const int* k, cudaStream_t s) {
  switch (h->p) {
    case 1: return launch_p<1, BLOCK>(h, x, y, k, s);
    case 2: return launch_p<2, BLOCK>(h, x, y, k, s);
    case 3: return launch_p<3, BLOCK>(h, x, y, k, s);
    case 4: return launch_p<4, BLOCK>(h, x, y, k, s);
    case 5: return launch_p<5, BLOCK>(h, x, y, k, s);
    case 6: return launch_p<6, BLOCK>(h, x, y, k, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

// y (RT part zeroed here) = M u  /  [M u + D^T q ; D u - Z q], 3D, any trilinear geometry
cudaError_t launch_trilinear_apply(const hdiv_ctx* h, const double* x, double* y, int mode,
                                   const int* skip, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(y, 0, sizeof(double) * h->nrt, s);
  if (e != cudaSuccess) return e;
  if (mode == MODE_BLOCK) return dispatch<true>(h, x, y, skip, s);
  return dispatch<false>(h, x, y, skip, s);
}

}  // namespace hdiv
