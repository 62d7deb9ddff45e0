// kernel_trilinear.cu — 3D block-operator apply on (tri)linear hexahedra, element by element.
//
//   M^e u = sum_q w_q (mw_e / det J_q) J_q^T J_q u_hat(x_q) tested against phi_hat
//   (P:84 Piola, P:135 eq. matrices), Gauss-Legendre Q = p+2 (reading A3).
//
// One CTA (64 threads) per element; the three components advance together so every
// sum-factorisation stage costs one barrier.  Each contraction is a register-blocked line
// pass: a thread loads the NIN inputs of one line, applies the 1D table (B_l / B_h, compile-
// time indices -> constant-bank operands) and writes the NO outputs, i.e. ~(NIN+NO)/(NIN NO)
// shared-memory accesses per FMA.  All smem arrays use odd-padded strides (lanes run over an
// odd stride -> conflict free).  The trilinear Jacobian columns are tabulated on the Q^2 point
// pairs (dT/dx_hat depends on (y_hat, z_hat) only, etc.).  Element-boundary faces are
// accumulated with fp64 atomics onto a zeroed y (0 + a + b: order independent), interior
// faces stored.  Z (constant-J elements only) and D u are element-local.
#include <cuda_runtime.h>

#include <cstdlib>

#include "internal.h"
#include "tri_layouts.h"

namespace hdiv {
namespace {

constexpr int odd_up(int v) { return (v % 2) ? v : v + 1; }

// 8-byte global -> shared copy, asynchronous; !ok writes 0 (src-size 0: nothing is read)
__device__ __forceinline__ void cp_async8z(double* smem, const double* gmem, bool ok) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem),
               "r"(ok ? 8 : 0) : "memory");
}

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
  int ess;              // eliminated essential sides (NEXT-3): zero inputs, outputs skipped
  const double* gvert;  // general gamma (NEXT-3): per-vertex field; Z = W^-1 W_gamma W^-1
  const int* skip;
  const double* winv;   // explicit W^e inverses fused into tri_multi_kernel's y_q store (or nullptr)
  const double* zc;     // {., s_e, ., .} per element (with winv)
  const double* geo;    // stored quadrature-point factors [E][6][Q^3] (tri_multi_kernel<SG>)
};

// padded layout of a (D0, D1, D2) array of the order-PP kernel: the strides with the fewest
// modelled bank-conflict wavefronts over every pass that touches arrays of this shape
// (tri_layouts.h, scripts/tri_layout_model.py), else odd-padded extents
template <int D0, int D1, int D2, int PP = 0>
struct Lay {
  static constexpr int LI = find_tri_layout(PP, 64, D0, D1, D2);
  static constexpr int S1 = LI >= 0 ? kTriLayouts[LI].S1 : odd_up(D0);
  static constexpr int S2 = LI >= 0 ? kTriLayouts[LI].S2 : S1 * odd_up(D1);
  static constexpr int SIZE = S2 * D2;
  static_assert(S1 >= D0 && S2 >= S1 * D1, "overlapping layout");
};

// 1D tables: B_l, B_h, M_h^-1, GL-nodal basis at the quadrature points (BG), its square
// (diagonal of W in the GL basis), the change of basis GL-nodal -> histopolation (HG) and HG^T
enum { TB_L = 0, TB_H = 1, TB_HI = 2, TB_G = 3, TB_G2 = 4, TB_HG = 5, TB_HGT = 6 };

template <int KIND, bool FWD>
__device__ __forceinline__ double tcoef(const Tab1D& tab, int o, int t) {
  if (KIND == TB_HI) return tab.Mhinv[o][t];
  if (KIND == TB_HG) return tab.HG[o][t];
  if (KIND == TB_HGT) return tab.HG[t][o];
  if (KIND == TB_G) return FWD ? tab.BG[o][t] : tab.BG[t][o];
  if (KIND == TB_G2) return FWD ? tab.BG[o][t] * tab.BG[o][t] : tab.BG[t][o] * tab.BG[t][o];
  if (FWD) return (KIND == TB_L) ? tab.Bl[o][t] : tab.Bh[o][t];   // T(o=q, t=i) = B[q][i]
  return (KIND == TB_L) ? tab.Bl[t][o] : tab.Bh[t][o];            // T(o=i, t=q) = B[q][i]
}

// sum over the CTA of a per-thread value (all threads return the total)
template <int NT>
__device__ __forceinline__ double cta_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int w = 0; w < NT / 32; ++w) s += red[w];
  __syncthreads();
  return s;
}

// line contraction along AX: in (N0,N1,N2) layout LI -> out (.. NO at AX ..) layout LO
// EPC > 1: the lines of EPC elements whose arrays sit ES doubles apart form one item space
template <int NT, int N0, int N1, int N2, int AX, int NO, int KIND, bool FWD, class LI, class LO,
          int EPC = 1, int ES = 0>
__device__ __forceinline__ void lines(const double* in, double* out, const Tab1D& tab,
                                      int start = -1, int stride = NT) {
  constexpr int NIN = (AX == 0) ? N0 : (AX == 1) ? N1 : N2;
  // the two other axes (lanes over the first: odd stride)
  constexpr int B0 = (AX == 0) ? N1 : N0;
  constexpr int B1 = (AX == 2) ? N1 : N2;
  constexpr int SI_A = (AX == 0) ? 1 : (AX == 1) ? LI::S1 : LI::S2;
  constexpr int SI_0 = (AX == 0) ? LI::S1 : 1;
  constexpr int SI_1 = (AX == 2) ? LI::S1 : LI::S2;
  constexpr int SO_A = (AX == 0) ? 1 : (AX == 1) ? LO::S1 : LO::S2;
  constexpr int SO_0 = (AX == 0) ? LO::S1 : 1;
  constexpr int SO_1 = (AX == 2) ? LO::S1 : LO::S2;
  constexpr int NB = B0 * B1;
#pragma unroll 1
  for (int it = (start < 0 ? (int)threadIdx.x : start); it < EPC * NB; it += stride) {
    const int el = (EPC > 1) ? it / NB : 0;
    const int r = (EPC > 1) ? it - el * NB : it;
    const int b0 = r % B0, b1 = r / B0;
    const double* pi = in + el * ES + b0 * SI_0 + b1 * SI_1;
    double* po = out + el * ES + b0 * SO_0 + b1 * SO_1;
    double v[NIN];
#pragma unroll
    for (int t = 0; t < NIN; ++t) v[t] = pi[t * SI_A];
#pragma unroll
    for (int o = 0; o < NO; ++o) {
      double s = 0.0;
#pragma unroll
      for (int t = 0; t < NIN; ++t) s = fma(tcoef<KIND, FWD>(tab, o, t), v[t], s);
      po[o * SO_A] = s;
    }
  }
}

// the same line pass with every output multiplied by scale[] (laid out like `out`): the
// pointwise quadrature weights folded into the last forward contraction
template <int NT, int N0, int N1, int N2, int AX, int NO, int KIND, bool FWD, class LI, class LO>
__device__ __forceinline__ void lines_scaled(const double* in, double* out,
                                             const double* __restrict__ scale, const Tab1D& tab) {
  constexpr int NIN = (AX == 0) ? N0 : (AX == 1) ? N1 : N2;
  constexpr int B0 = (AX == 0) ? N1 : N0;
  constexpr int B1 = (AX == 2) ? N1 : N2;
  constexpr int SI_A = (AX == 0) ? 1 : (AX == 1) ? LI::S1 : LI::S2;
  constexpr int SI_0 = (AX == 0) ? LI::S1 : 1;
  constexpr int SI_1 = (AX == 2) ? LI::S1 : LI::S2;
  constexpr int SO_A = (AX == 0) ? 1 : (AX == 1) ? LO::S1 : LO::S2;
  constexpr int SO_0 = (AX == 0) ? LO::S1 : 1;
  constexpr int SO_1 = (AX == 2) ? LO::S1 : LO::S2;
#pragma unroll 1
  for (int it = threadIdx.x; it < B0 * B1; it += NT) {
    const int b0 = it % B0, b1 = it / B0;
    const double* pi = in + b0 * SI_0 + b1 * SI_1;
    const int oo = b0 * SO_0 + b1 * SO_1;
    double v[NIN];
#pragma unroll
    for (int t = 0; t < NIN; ++t) v[t] = pi[t * SI_A];
#pragma unroll
    for (int o = 0; o < NO; ++o) {
      double s = 0.0;
#pragma unroll
      for (int t = 0; t < NIN; ++t) s = fma(tcoef<KIND, FWD>(tab, o, t), v[t], s);
      out[oo + o * SO_A] = s * scale[oo + o * SO_A];
    }
  }
}

// one component's line pass of a stage: with 96-thread CTAs warp COMP takes component COMP's
// lines (the three components run side by side, no divergence), else all threads take them
template <int NT, int COMP, int N0, int N1, int N2, int AX, int NO, int KIND, bool FWD, class LI,
          class LO, int EPC = 1, int ES = 0>
__device__ __forceinline__ void lines_c(const double* in, double* out, const Tab1D& tab) {
  if constexpr (NT == 96) {
    if ((int)(threadIdx.x >> 5) == COMP)
      lines<NT, N0, N1, N2, AX, NO, KIND, FWD, LI, LO, EPC, ES>(in, out, tab, threadIdx.x & 31, 32);
  } else {
    lines<NT, N0, N1, N2, AX, NO, KIND, FWD, LI, LO, EPC, ES>(in, out, tab);
  }
}

template <int P>
struct TG {   // per-component layouts at every stage
  static constexpr int Q = P + 2;
  using U0 = Lay<P + 1, P, P, P>;  using U1 = Lay<P, P + 1, P, P>;  using U2 = Lay<P, P, P + 1, P>;
  using A0 = Lay<Q, P, P, P>;      using A1 = Lay<Q, P + 1, P, P>;  using A2 = Lay<Q, P, P + 1, P>;
  using B0 = Lay<Q, Q, P, P>;      using B1 = Lay<Q, Q, P, P>;      using B2 = Lay<Q, Q, P + 1, P>;
  using V = Lay<Q, Q, Q, P>;
  using L2 = Lay<P, P, P, P>;
  static constexpr int SU = (U0::SIZE > U1::SIZE ? (U0::SIZE > U2::SIZE ? U0::SIZE : U2::SIZE)
                                                  : (U1::SIZE > U2::SIZE ? U1::SIZE : U2::SIZE));
  static constexpr int SA = A2::SIZE > A1::SIZE ? A2::SIZE : A1::SIZE;
  static constexpr int SB = B2::SIZE;
  static constexpr int SV = V::SIZE;
  static constexpr int SL = L2::SIZE;
};

// MODE 0: y_u = M u ; 1: block apply ; 2: y = Z q only (the (2,2) block, W^-1 benchmark)
template <int P, int NT, int MODE>
__global__ void __launch_bounds__(NT) tri_kernel(const TriArgs a, const __grid_constant__ Tab1D tab) {
  constexpr bool BLOCK = (MODE == 1), ZONLY = (MODE == 2), HASQ = (MODE >= 1);
  using T = TG<P>;
  constexpr int Q = P + 2;
  constexpr int NQ = Q * Q * Q;
  constexpr int P3 = P * P * P;
  if (a.skip && *a.skip) return;
  __shared__ double sX[8 * 3];
  __shared__ double sJ[3][Q * Q][3];   // column factors: sJ[c][pair][d] = dT_d/dx_hat_c
  // lifetimes: su (load..F1, B3..scatter) / sB (F2..F3, B1..B2) share region R1;
  //            sA (F1..F2, B2..B3) / sV (F3..B1) share region R2
  constexpr int R1 = (3 * T::SU > 3 * T::SB) ? 3 * T::SU : 3 * T::SB;
  constexpr int R2 = (3 * T::SA > 3 * T::SV) ? 3 * T::SA : 3 * T::SV;
  __shared__ double sreg[R1 + R2];
#define su(c) (sreg + (c) * T::SU)
#define sB(c) (sreg + (c) * T::SB)
#define sA(c) (sreg + R1 + (c) * T::SA)
#define sV(c) (sreg + R1 + (c) * T::SV)
  __shared__ double sq[HASQ ? T::SL : 1], sy[BLOCK ? P3 : 1], sz1[HASQ ? T::SL : 1],
      sz2[HASQ ? T::SL : 1];
  __shared__ double scoef[2];
  __shared__ double sG[8];   // vertex gamma values (general gamma)

  const int tid = threadIdx.x;
  const long long e = blockIdx.x;
  const long long NLx = a.NL[0], NLy = a.NL[1];
  // element coordinates in 32-bit (the grid is < 2^31 CTAs)
  const unsigned eu = blockIdx.x, nlx = (unsigned)NLx, nly = (unsigned)NLy;
  const unsigned eyz = eu / nlx;
  const int ex = (int)(eu - eyz * nlx), ey = (int)(eyz % nly), ez = (int)(eyz / nly);
  const long long nx = a.n[0], ny = a.n[1];

  if (tid < 2) scoef[tid] = a.coef[4 * e + tid];
  // inputs land by cp.async at p <= 4 and for Z alone (all loads of the element in flight at
  // once: the register-path gather was the top long-scoreboard stall); the p = 5, 6 block apply
  // with the local CG ran 4-7 % slower that way (r01 A/B, scripts/tri_z_time.py)
  constexpr bool ASYNC = (P <= 4) || ZONLY;
  auto ld = [&](double* dst, const double* src, bool ok) {
    if constexpr (ASYNC) cp_async8z(dst, ok ? src : a.x, ok);
    else *dst = ok ? *src : 0.0;
  };
  for (int i = tid; i < 24; i += NT) {
    const int v = i / 3, d = i % 3;
    const long long g = ((long long)(ez + (v >> 2)) * (NLy + 1) + (ey + ((v >> 1) & 1))) * (NLx + 1) +
                        (ex + (v & 1));
    ld(&sX[i], a.vert + g * 3 + d, true);
    if (HASQ && a.gvert && d == 0) ld(&sG[v], a.gvert + g, true);
  }
  // gather u per component (compile-time extents, i fastest; padded smem layouts)
  if constexpr (!ZONLY) {
    const long long gx = a.off[0] + (long long)ex * P + (nx + 1) * ((long long)ey * P + ny * (long long)ez * P);
    const long long gy = a.off[1] + (long long)ex * P + nx * ((long long)ey * P + (ny + 1) * (long long)ez * P);
    const long long gz = a.off[2] + (long long)ex * P + nx * ((long long)ey * P + ny * (long long)ez * P);
    // eliminated essential faces (NEXT-3) act as zero inputs
    for (int l = tid; l < (P + 1) * P * P; l += NT) {
      const int li = l % (P + 1), lj = (l / (P + 1)) % P, lk = l / ((P + 1) * P);
      const bool m = a.ess && face_masked(a.ess, 0, (long long)ex * P + li, nx);
      ld(su(0) + li + T::U0::S1 * lj + T::U0::S2 * lk, a.x + gx + li + (nx + 1) * (lj + ny * lk), !m);
    }
    for (int l = tid; l < (P + 1) * P * P; l += NT) {
      const int li = l % P, lj = (l / P) % (P + 1), lk = l / (P * (P + 1));
      const bool m = a.ess && face_masked(a.ess, 1, (long long)ey * P + lj, ny);
      ld(su(1) + li + T::U1::S1 * lj + T::U1::S2 * lk, a.x + gy + li + nx * (lj + (ny + 1) * lk), !m);
    }
    for (int l = tid; l < (P + 1) * P * P; l += NT) {
      const int li = l % P, lj = (l / P) % P, lk = l / (P * P);
      const bool m = a.ess && face_masked(a.ess, 2, (long long)ez * P + lk, a.n[2]);
      ld(su(2) + li + T::U2::S1 * lj + T::U2::S2 * lk, a.x + gz + li + nx * (lj + ny * lk), !m);
    }
  }
  if constexpr (HASQ) {
    const double* q = ZONLY ? a.x : a.x + a.nrt;
    for (int i = tid; i < P3; i += NT) {
      const int A = i % P, B = (i / P) % P, C = i / (P * P);
      ld(sq + A + T::L2::S1 * B + T::L2::S2 * C, q + e * P3 + i, true);
    }
  }
  if constexpr (ASYNC) asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();

  // trilinear Jacobian column factors on the Q x Q point pairs: dT/dx_hat_c is bilinear in the
  // other two reference coordinates (s, t) with the four edge vectors along c as coefficients
  // E[c][k] (k = corner (s, t) in {0,1}^2); first the 36 edge-vector entries, then one item per
  // (c, point pair) evaluating the three coordinates
  __shared__ double sE[3][4][3];
  for (int i = tid; i < 36; i += NT) {   // (NT may be 32)
    const int c = i / 12, k = (i / 3) % 4, d = i % 3;
    const int s1 = k & 1, t1 = k >> 1;   // corner along the (first, second) other axis
    int lo[3], hi[3];
    const int o0 = (c == 0) ? 1 : 0, o1 = (c == 2) ? 1 : 2;
    lo[c] = 0; hi[c] = 1;
    lo[o0] = hi[o0] = s1;
    lo[o1] = hi[o1] = t1;
    sE[c][k][d] = sX[(hi[0] + 2 * hi[1] + 4 * hi[2]) * 3 + d] - sX[(lo[0] + 2 * lo[1] + 4 * lo[2]) * 3 + d];
  }
  __syncthreads();
  for (int i = tid; i < 3 * Q * Q; i += NT) {
    const int c = i / (Q * Q), pr = i % (Q * Q);
    const double s = tab.xq[pr % Q], t = tab.xq[pr / Q];
    const double w00 = (1 - s) * (1 - t), w10 = s * (1 - t), w01 = (1 - s) * t, w11 = s * t;
#pragma unroll
    for (int d = 0; d < 3; ++d)
      sJ[c][pr][d] = w00 * sE[c][0][d] + w10 * sE[c][1][d] + w01 * sE[c][2][d] + w11 * sE[c][3][d];
  }
  if constexpr (!ZONLY) {
  // ---- forward: axis 0, 1, 2 (3 components per stage), + D u and Z q~ ----
  lines_c<NT, 0, P + 1, P, P, 0, Q, TB_L, true, typename T::U0, typename T::A0>(su(0), sA(0), tab);
  lines_c<NT, 1, P, P + 1, P, 0, Q, TB_H, true, typename T::U1, typename T::A1>(su(1), sA(1), tab);
  lines_c<NT, 2, P, P, P + 1, 0, Q, TB_H, true, typename T::U2, typename T::A2>(su(2), sA(2), tab);
  if constexpr (BLOCK) {
    for (int i = tid; i < P3; i += NT) {
      const int A = i % P, B = (i / P) % P, C = i / (P * P);
      const double* u0 = su(0) + A + T::U0::S1 * B + T::U0::S2 * C;
      const double* u1 = su(1) + A + T::U1::S1 * B + T::U1::S2 * C;
      const double* u2 = su(2) + A + T::U2::S1 * B + T::U2::S2 * C;
      sy[i] = (u0[1] - u0[0]) + (u1[T::U1::S1] - u1[0]) + (u2[T::U2::S2] - u2[0]);
    }
  }
  __syncthreads();
  lines_c<NT, 0, Q, P, P, 1, Q, TB_H, true, typename T::A0, typename T::B0>(sA(0), sB(0), tab);
  lines_c<NT, 1, Q, P + 1, P, 1, Q, TB_L, true, typename T::A1, typename T::B1>(sA(1), sB(1), tab);
  lines_c<NT, 2, Q, P, P + 1, 1, Q, TB_H, true, typename T::A2, typename T::B2>(sA(2), sB(2), tab);
  __syncthreads();
  lines_c<NT, 0, Q, Q, P, 2, Q, TB_H, true, typename T::B0, typename T::V>(sB(0), sV(0), tab);
  lines_c<NT, 1, Q, Q, P, 2, Q, TB_H, true, typename T::B1, typename T::V>(sB(1), sV(1), tab);
  lines_c<NT, 2, Q, Q, P + 1, 2, Q, TB_L, true, typename T::B2, typename T::V>(sB(2), sV(2), tab);
  __syncthreads();
  // ---- pointwise G_q = w_q mw / det J  J^T J ----
  const double mw = scoef[0];
  for (int qi = tid; qi < NQ; qi += NT) {
    const int qx = qi % Q, qy = (qi / Q) % Q, qz = qi / (Q * Q);
    const double* c0 = sJ[0][qy + Q * qz];
    const double* c1 = sJ[1][qx + Q * qz];
    const double* c2 = sJ[2][qx + Q * qy];
    const double det = c0[0] * (c1[1] * c2[2] - c1[2] * c2[1]) - c1[0] * (c0[1] * c2[2] - c0[2] * c2[1]) +
                       c2[0] * (c0[1] * c1[2] - c0[2] * c1[1]);
    const double s = tab.wq[qx] * tab.wq[qy] * tab.wq[qz] * mw / det;
    const int o = qx + T::V::S1 * qy + T::V::S2 * qz;
    const double u0 = sV(0)[o], u1 = sV(1)[o], u2 = sV(2)[o];
    double Ju[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) Ju[d] = c0[d] * u0 + c1[d] * u1 + c2[d] * u2;
    sV(0)[o] = s * (c0[0] * Ju[0] + c0[1] * Ju[1] + c0[2] * Ju[2]);
    sV(1)[o] = s * (c1[0] * Ju[0] + c1[1] * Ju[1] + c1[2] * Ju[2]);
    sV(2)[o] = s * (c2[0] * Ju[0] + c2[1] * Ju[1] + c2[2] * Ju[2]);
  }
  __syncthreads();
  // ---- backward: axis 2, 1, 0 ----
  lines_c<NT, 0, Q, Q, Q, 2, P, TB_H, false, typename T::V, typename T::B0>(sV(0), sB(0), tab);
  lines_c<NT, 1, Q, Q, Q, 2, P, TB_H, false, typename T::V, typename T::B1>(sV(1), sB(1), tab);
  lines_c<NT, 2, Q, Q, Q, 2, P + 1, TB_L, false, typename T::V, typename T::B2>(sV(2), sB(2), tab);
  __syncthreads();
  lines_c<NT, 0, Q, Q, P, 1, P, TB_H, false, typename T::B0, typename T::A0>(sB(0), sA(0), tab);
  lines_c<NT, 1, Q, Q, P, 1, P + 1, TB_L, false, typename T::B1, typename T::A1>(sB(1), sA(1), tab);
  lines_c<NT, 2, Q, Q, P + 1, 1, P, TB_H, false, typename T::B2, typename T::A2>(sB(2), sA(2), tab);
  __syncthreads();
  lines_c<NT, 0, Q, P, P, 0, P + 1, TB_L, false, typename T::A0, typename T::U0>(sA(0), su(0), tab);
  lines_c<NT, 1, Q, P + 1, P, 0, P, TB_H, false, typename T::A1, typename T::U1>(sA(1), su(1), tab);
  lines_c<NT, 2, Q, P, P + 1, 0, P, TB_H, false, typename T::A2, typename T::U2>(sA(2), su(2), tab);
  __syncthreads();
  // ---- D^T q~ and scatter (per component; boundary faces by atomics) ----
  {
    const long long gx = a.off[0] + (long long)ex * P + (nx + 1) * ((long long)ey * P + ny * (long long)ez * P);
    const long long gy = a.off[1] + (long long)ex * P + nx * ((long long)ey * P + (ny + 1) * (long long)ez * P);
    const long long gz = a.off[2] + (long long)ex * P + nx * ((long long)ey * P + ny * (long long)ez * P);
    // element-boundary faces by atomics onto the zeroed output; eliminated essential faces
    // are skipped (their identity rows are written by the fixup kernel)
    auto put = [&](double* g, double v, int ic, int c, long long gi) {
      if (ic == 0 || ic == P) {
        if (!(a.ess && face_masked(a.ess, c, gi, a.n[c]))) atomicAdd(g, v);
      } else {
        *g = v;
      }
    };
    for (int l = tid; l < (P + 1) * P * P; l += NT) {
      const int li = l % (P + 1), lj = (l / (P + 1)) % P, lk = l / ((P + 1) * P);
      double v = su(0)[li + T::U0::S1 * lj + T::U0::S2 * lk];
      if constexpr (BLOCK) {
        const int cell = li + T::L2::S1 * lj + T::L2::S2 * lk;
        if (li > 0) v += sq[cell - 1];
        if (li < P) v -= sq[cell];
      }
      put(a.y + gx + li + (nx + 1) * (lj + ny * lk), v, li, 0, (long long)ex * P + li);
    }
    for (int l = tid; l < (P + 1) * P * P; l += NT) {
      const int li = l % P, lj = (l / P) % (P + 1), lk = l / (P * (P + 1));
      double v = su(1)[li + T::U1::S1 * lj + T::U1::S2 * lk];
      if constexpr (BLOCK) {
        const int cell = li + T::L2::S1 * lj + T::L2::S2 * lk;
        if (lj > 0) v += sq[cell - T::L2::S1];
        if (lj < P) v -= sq[cell];
      }
      put(a.y + gy + li + nx * (lj + (ny + 1) * lk), v, lj, 1, (long long)ey * P + lj);
    }
    for (int l = tid; l < (P + 1) * P * P; l += NT) {
      const int li = l % P, lj = (l / P) % P, lk = l / (P * P);
      double v = su(2)[li + T::U2::S1 * lj + T::U2::S2 * lk];
      if constexpr (BLOCK) {
        const int cell = li + T::L2::S1 * lj + T::L2::S2 * lk;
        if (lk > 0) v += sq[cell - T::L2::S2];
        if (lk < P) v -= sq[cell];
      }
      put(a.y + gz + li + nx * (lj + ny * lk), v, lk, 2, (long long)ez * P + lk);
    }
  }
  }  // !ZONLY
  if constexpr (HASQ) {
    if (ZONLY || a.has_z) {
      // ---- Z q~ = s_e W_1^-1 q~ (s_e = 1/alpha | gamma) by a fused
      //      element-local PCG in the Gauss-Legendre nodal basis with Jacobi preconditioning
      //      (P:606-609): W_h^-1 = H W_g^-1 H^T, W_g = H^T W_h H, H = HG^{(x)3}.
      //      W_g v = B_G^T diag(w_q / det J_q) B_G v by sum factorisation (Q = p+2 points).
      using GA = Lay<Q, P, P, P>;
      using GB = Lay<Q, Q, P, P>;
      using GV = Lay<Q, Q, Q, P>;
      using L2 = typename T::L2;
      __syncthreads();   // sreg is free: the mass part is done
      double* ta = sreg;
      double* tb = ta + GA::SIZE;
      double* tv = tb + GB::SIZE;
      double* gq = tv + GV::SIZE;        // w_q / det J_q (GV layout)
      double* vz = gq + GV::SIZE;        // CG iterate (GL basis)
      double* vp = vz + L2::SIZE;        // search direction
      double* vap = vp + L2::SIZE;       // W_g p
      double* vr = sz2;                  // residual
      double* vd = sz1;                  // diag(W_g), later the result
      __shared__ double red[NT / 32];
      for (int qi = tid; qi < NQ; qi += NT) {
        const int qx = qi % Q, qy = (qi / Q) % Q, qz = qi / (Q * Q);
        const double* c0 = sJ[0][qy + Q * qz];
        const double* c1 = sJ[1][qx + Q * qz];
        const double* c2 = sJ[2][qx + Q * qy];
        const double det = c0[0] * (c1[1] * c2[2] - c1[2] * c2[1]) -
                           c1[0] * (c0[1] * c2[2] - c0[2] * c2[1]) +
                           c2[0] * (c0[1] * c1[2] - c0[2] * c1[1]);
        gq[qx + GV::S1 * qy + GV::S2 * qz] = tab.wq[qx] * tab.wq[qy] * tab.wq[qz] / det;
      }
      // r = H^T q~ ; d = diag(W_g) = (B_G^2)^T g
      lines<NT, P, P, P, 0, P, TB_HGT, true, L2, L2>(sq, vz, tab);
      __syncthreads();
      lines<NT, P, P, P, 1, P, TB_HGT, true, L2, L2>(vz, vap, tab);
      lines<NT, Q, Q, Q, 2, P, TB_G2, false, GV, GB>(gq, tb, tab);
      __syncthreads();
      lines<NT, P, P, P, 2, P, TB_HGT, true, L2, L2>(vap, vr, tab);
      lines<NT, Q, Q, P, 1, P, TB_G2, false, GB, GA>(tb, ta, tab);
      __syncthreads();
      lines<NT, Q, P, P, 0, P, TB_G2, false, GA, L2>(ta, vd, tab);
      __syncthreads();
      // general gamma: Z = W^-1 W_gamma W^-1 — two passes of the local CG
      // with t = W_gamma (W^-1 q~) in between; piecewise-constant gamma: one pass, Z = s_e W^-1
      const int npass = a.gvert ? 2 : 1;
      for (int pass = 0; pass < npass; ++pass) {
      if (pass == 1) {
        // t = W_gamma y in the histopolation basis: B_h^T diag(w_q gamma_q / det J_q) B_h,
        // y = W^-1 q~ (sz1) -> sq (free: D^T q~ was scattered before)
        lines<NT, P, P, P, 0, Q, TB_H, true, L2, GA>(sz1, ta, tab);
        __syncthreads();
        lines<NT, Q, P, P, 1, Q, TB_H, true, GA, GB>(ta, tb, tab);
        __syncthreads();
        lines<NT, Q, Q, P, 2, Q, TB_H, true, GB, GV>(tb, tv, tab);
        __syncthreads();
        for (int qi = tid; qi < NQ; qi += NT) {
          const int qx = qi % Q, qy = (qi / Q) % Q, qz = qi / (Q * Q);
          const double xh = tab.xq[qx], yh = tab.xq[qy], zh = tab.xq[qz];
          double g = 0.0;
#pragma unroll
          for (int v = 0; v < 8; ++v)
            g += sG[v] * ((v & 1) ? xh : 1 - xh) * ((v & 2) ? yh : 1 - yh) * ((v & 4) ? zh : 1 - zh);
          const int o = qx + GV::S1 * qy + GV::S2 * qz;
          tv[o] *= g * gq[o];
        }
        __syncthreads();
        lines<NT, Q, Q, Q, 2, P, TB_H, false, GV, GB>(tv, tb, tab);
        __syncthreads();
        lines<NT, Q, Q, P, 1, P, TB_H, false, GB, GA>(tb, ta, tab);
        __syncthreads();
        lines<NT, Q, P, P, 0, P, TB_H, false, GA, L2>(ta, sq, tab);
        __syncthreads();
        // r = H^T t for the second solve; diag(W_g) again into vd (= sz1, which held y)
        lines<NT, P, P, P, 0, P, TB_HGT, true, L2, L2>(sq, vz, tab);
        lines<NT, Q, Q, Q, 2, P, TB_G2, false, GV, GB>(gq, tb, tab);
        __syncthreads();
        lines<NT, P, P, P, 1, P, TB_HGT, true, L2, L2>(vz, vap, tab);
        lines<NT, Q, Q, P, 1, P, TB_G2, false, GB, GA>(tb, ta, tab);
        __syncthreads();
        lines<NT, P, P, P, 2, P, TB_HGT, true, L2, L2>(vap, vr, tab);
        lines<NT, Q, P, P, 0, P, TB_G2, false, GA, L2>(ta, vd, tab);
        __syncthreads();
      }
      // PCG with the iterate, residual, direction and diagonal in registers (KP entries per
      // thread); only the direction goes through shared memory for the W_g apply
      constexpr int KP = (P3 + NT - 1) / NT;
      auto off = [&](int i) { return i % P + L2::S1 * ((i / P) % P) + L2::S2 * (i / (P * P)); };
      double rz[KP], rr[KP], rp[KP], rd[KP], ra[KP];
      double rs = 0.0;
#pragma unroll
      for (int k = 0; k < KP; ++k) {   // z = 0, p = D^-1 r
        const int i = tid + k * NT;
        rz[k] = 0.0;
        rr[k] = 0.0; rd[k] = 1.0; rp[k] = 0.0;
        if (i < P3) {
          const int o = off(i);
          rr[k] = vr[o];
          rd[k] = vd[o];
          rp[k] = rr[k] / rd[k];
          vp[o] = rp[k];
          rs += rr[k] * rp[k];
        }
      }
      rs = cta_sum<NT>(rs, red);
      const double rs0 = rs;
      for (int it = 0; it < 40 && rs > 1e-30 * rs0 && rs > 0.0; ++it) {
        // ap = W_g p (the pointwise w_q / det J_q folded into the last forward pass)
        lines<NT, P, P, P, 0, Q, TB_G, true, L2, GA>(vp, ta, tab);
        __syncthreads();
        lines<NT, Q, P, P, 1, Q, TB_G, true, GA, GB>(ta, tb, tab);
        __syncthreads();
        lines_scaled<NT, Q, Q, P, 2, Q, TB_G, true, GB, GV>(tb, tv, gq, tab);
        __syncthreads();
        lines<NT, Q, Q, Q, 2, P, TB_G, false, GV, GB>(tv, tb, tab);
        __syncthreads();
        lines<NT, Q, Q, P, 1, P, TB_G, false, GB, GA>(tb, ta, tab);
        __syncthreads();
        lines<NT, Q, P, P, 0, P, TB_G, false, GA, L2>(ta, vap, tab);
        __syncthreads();
        double pap = 0.0;
#pragma unroll
        for (int k = 0; k < KP; ++k) {
          const int i = tid + k * NT;
          ra[k] = (i < P3) ? vap[off(i)] : 0.0;
          pap += rp[k] * ra[k];
        }
        pap = cta_sum<NT>(pap, red);
        const double al = rs / pap;
        double rsn = 0.0;
#pragma unroll
        for (int k = 0; k < KP; ++k) {
          rz[k] += al * rp[k];
          rr[k] -= al * ra[k];
          rsn += rr[k] * (rr[k] / rd[k]);
        }
        rsn = cta_sum<NT>(rsn, red);
        const double be = rsn / rs;
#pragma unroll
        for (int k = 0; k < KP; ++k) {
          const int i = tid + k * NT;
          rp[k] = rr[k] / rd[k] + be * rp[k];
          if (i < P3) vp[off(i)] = rp[k];
        }
        rs = rsn;
        __syncthreads();
      }
#pragma unroll
      for (int k = 0; k < KP; ++k) {
        const int i = tid + k * NT;
        if (i < P3) vz[off(i)] = rz[k];
      }
      __syncthreads();
      // y = H z (histopolation basis) -> sz1
      lines<NT, P, P, P, 0, P, TB_HG, true, L2, L2>(vz, vap, tab);
      __syncthreads();
      lines<NT, P, P, P, 1, P, TB_HG, true, L2, L2>(vap, vp, tab);
      __syncthreads();
      lines<NT, P, P, P, 2, P, TB_HG, true, L2, L2>(vp, sz1, tab);
      __syncthreads();
      }   // pass
    }
    const double z = scoef[1];
    if constexpr (ZONLY) {
      for (int i = tid; i < P3; i += NT) {
        const int A = i % P, B = (i / P) % P, C = i / (P * P);
        a.y[e * P3 + i] = z * sz1[A + T::L2::S1 * B + T::L2::S2 * C];
      }
    } else {
      double* yq = a.y + a.nrt;
      for (int i = tid; i < P3; i += NT) {
        const int A = i % P, B = (i / P) % P, C = i / (P * P);
        yq[e * P3 + i] = a.has_z ? sy[i] - z * sz1[A + T::L2::S1 * B + T::L2::S2 * C] : sy[i];
      }
    }
  }
}

// Mass apply / gamma = 0 block apply with EPC elements per 96-thread CTA: warp c takes the line
// passes of RT component c for all EPC elements, so a stage's lines fill the lanes (one element
// leaves 37 % of them idle at p = 4: 16-24 lines per component and stage) — same arithmetic,
// same order per output as tri_kernel<P, 96, MODE>.
template <int P, int EPC, bool BLOCK, bool SG = false, bool ESS = true>
__global__ void __launch_bounds__(96) tri_multi_kernel(const TriArgs a,
                                                       const __grid_constant__ Tab1D tab,
                                                       long long E) {
  constexpr int NT = 96;
  using T = TG<P>;
  constexpr int Q = P + 2;
  constexpr int NQ = Q * Q * Q;
  constexpr int P3 = P * P * P;
  constexpr int NU = (P + 1) * P * P;
  if (a.skip && *a.skip) return;
  constexpr int R1 = (3 * T::SU > 3 * T::SB) ? 3 * T::SU : 3 * T::SB;
  constexpr int R2 = (3 * T::SA > 3 * T::SV) ? 3 * T::SA : 3 * T::SV;
  constexpr int ES = R1 + R2;   // per-element stride of the stage arrays
  __shared__ double sreg[EPC * ES];
  constexpr int EJ = SG ? 1 : EPC;   // Jacobian scratch (on-the-fly variant only)
  __shared__ double sX[EJ][24];
  __shared__ double sE[EJ][3][4][3];
  __shared__ double sJ[EJ][3][Q * Q][3];
  __shared__ double sq[BLOCK ? EPC * T::SL : 1], sy[BLOCK ? EPC * P3 : 1];
  __shared__ double smw[EPC];
  __shared__ int sEc[EPC][4];   // ex, ey, ez, valid
  const int tid = threadIdx.x;
  const long long e0 = (long long)blockIdx.x * EPC;
  const long long NLx = a.NL[0], NLy = a.NL[1];
  const long long nx = a.n[0], ny = a.n[1];
  if (tid < EPC) {
    const long long e = e0 + tid;
    const bool ok = e < E;
    const unsigned eu = ok ? (unsigned)e : 0u, nlx = (unsigned)NLx, nly = (unsigned)NLy;
    const unsigned eyz = eu / nlx;
    sEc[tid][0] = (int)(eu - eyz * nlx);
    sEc[tid][1] = (int)(eyz % nly);
    sEc[tid][2] = (int)(eyz / nly);
    sEc[tid][3] = ok ? 1 : 0;
    smw[tid] = ok ? a.coef[4 * e] : 0.0;
  }
  if constexpr (SG) {   // stored factors: pull the CTA's G block toward L2 while the passes run
    constexpr int NLINE = (EPC * 6 * NQ * 8 + 127) / 128;
    const char* gb = (const char*)(a.geo + e0 * 6 * NQ);
    const long long lim = (E - e0) * 6 * NQ * 8;
    for (int i = tid; i < NLINE; i += NT)
      if ((long long)i * 128 < lim) asm volatile("prefetch.global.L2 [%0];\n" ::"l"(gb + i * 128));
  }
  __syncthreads();
  // every input lands by cp.async (all loads in flight at once; masked / absent -> 0)
  for (int i = tid; i < (SG ? 0 : EPC * 24); i += NT) {
    const int el = i / 24, v = (i % 24) / 3, d = i % 3;
    const bool ok = sEc[el][3];
    const long long g = ((long long)(sEc[el][2] + (v >> 2)) * (NLy + 1) + (sEc[el][1] + ((v >> 1) & 1))) *
                            (NLx + 1) + (sEc[el][0] + (v & 1));
    cp_async8z(&sX[el][v * 3 + d], a.vert + (ok ? g * 3 + d : 0), ok);
  }
  // gather u (eliminated essential faces act as zero inputs; absent elements as zeros)
  // component strides (64-bit, once): face (li, lj, lk) of component c of element (ex, ey, ez)
  // at g_c(e) + li + lj s1_c + lk s2_c
  const long long s1x = nx + 1, s2x = (nx + 1) * ny, s1y = nx, s2y = nx * (ny + 1), s1z = nx, s2z = nx * ny;
  auto gbase = [&](int c, int ex, int ey, int ez) -> long long {
    const long long X = (long long)ex * P, Y = (long long)ey * P, Z = (long long)ez * P;
    return c == 0 ? a.off[0] + X + Y * s1x + Z * s2x
         : c == 1 ? a.off[1] + X + Y * s1y + Z * s2y : a.off[2] + X + Y * s1z + Z * s2z;
  };
  for (int l = tid; l < EPC * NU; l += NT) {
    const int el = l / NU, r = l - (l / NU) * NU;
    const int ex = sEc[el][0], ey = sEc[el][1], ez = sEc[el][2];
    double* sr = sreg + el * ES;
    {
      const int li = r % (P + 1), lj = (r / (P + 1)) % P, lk = r / ((P + 1) * P);
      const long long g = gbase(0, ex, ey, ez) + li + lj * s1x + lk * s2x;
      const bool m = !sEc[el][3] || (ESS && a.ess && face_masked(a.ess, 0, (long long)ex * P + li, nx));
      cp_async8z(sr + 0 * T::SU + li + T::U0::S1 * lj + T::U0::S2 * lk, a.x + (m ? 0 : g), !m);
    }
    {
      const int li = r % P, lj = (r / P) % (P + 1), lk = r / (P * (P + 1));
      const long long g = gbase(1, ex, ey, ez) + li + lj * s1y + lk * s2y;
      const bool m = !sEc[el][3] || (ESS && a.ess && face_masked(a.ess, 1, (long long)ey * P + lj, ny));
      cp_async8z(sr + 1 * T::SU + li + T::U1::S1 * lj + T::U1::S2 * lk, a.x + (m ? 0 : g), !m);
    }
    {
      const int li = r % P, lj = (r / P) % P, lk = r / (P * P);
      const long long g = gbase(2, ex, ey, ez) + li + lj * s1z + lk * s2z;
      const bool m = !sEc[el][3] || (ESS && a.ess && face_masked(a.ess, 2, (long long)ez * P + lk, a.n[2]));
      cp_async8z(sr + 2 * T::SU + li + T::U2::S1 * lj + T::U2::S2 * lk, a.x + (m ? 0 : g), !m);
    }
  }
  if constexpr (BLOCK) {
    const double* q = a.x + a.nrt;
    for (int i = tid; i < EPC * P3; i += NT) {
      const int el = i / P3, r = i - (i / P3) * P3;
      const int A = r % P, B = (r / P) % P, C = r / (P * P);
      const bool ok = sEc[el][3];
      cp_async8z(sq + el * T::SL + A + T::L2::S1 * B + T::L2::S2 * C, q + (ok ? (e0 + el) * P3 + r : 0), ok);
    }
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  for (int i = tid; i < (SG ? 0 : EPC * 36); i += NT) {
    const int el = i / 36, j = i % 36;
    const int c = j / 12, k = (j / 3) % 4, d = j % 3;
    const int s1 = k & 1, t1 = k >> 1;
    int lo[3], hi[3];
    const int o0 = (c == 0) ? 1 : 0, o1 = (c == 2) ? 1 : 2;
    lo[c] = 0; hi[c] = 1;
    lo[o0] = hi[o0] = s1;
    lo[o1] = hi[o1] = t1;
    sE[el][c][k][d] = sX[el][(hi[0] + 2 * hi[1] + 4 * hi[2]) * 3 + d] - sX[el][(lo[0] + 2 * lo[1] + 4 * lo[2]) * 3 + d];
  }
  if constexpr (!SG) __syncthreads();
  for (int i = tid; i < (SG ? 0 : EPC * 3 * Q * Q); i += NT) {
    const int el = i / (3 * Q * Q), j = i % (3 * Q * Q);
    const int c = j / (Q * Q), pr = j % (Q * Q);
    const double s = tab.xq[pr % Q], t = tab.xq[pr / Q];
    const double w00 = (1 - s) * (1 - t), w10 = s * (1 - t), w01 = (1 - s) * t, w11 = s * t;
#pragma unroll
    for (int d = 0; d < 3; ++d)
      sJ[el][c][pr][d] = w00 * sE[el][c][0][d] + w10 * sE[el][c][1][d] + w01 * sE[el][c][2][d] + w11 * sE[el][c][3][d];
  }
  // ---- forward: axis 0, 1, 2 (warp c: component c of every element), + D u ----
  lines_c<NT, 0, P + 1, P, P, 0, Q, TB_L, true, typename T::U0, typename T::A0, EPC, ES>(su(0), sA(0), tab);
  lines_c<NT, 1, P, P + 1, P, 0, Q, TB_H, true, typename T::U1, typename T::A1, EPC, ES>(su(1), sA(1), tab);
  lines_c<NT, 2, P, P, P + 1, 0, Q, TB_H, true, typename T::U2, typename T::A2, EPC, ES>(su(2), sA(2), tab);
  if constexpr (BLOCK) {
    for (int i = tid; i < EPC * P3; i += NT) {
      const int el = i / P3, r = i - (i / P3) * P3;
      const int A = r % P, B = (r / P) % P, C = r / (P * P);
      const double* u0 = su(0) + el * ES + A + T::U0::S1 * B + T::U0::S2 * C;
      const double* u1 = su(1) + el * ES + A + T::U1::S1 * B + T::U1::S2 * C;
      const double* u2 = su(2) + el * ES + A + T::U2::S1 * B + T::U2::S2 * C;
      sy[i] = (u0[1] - u0[0]) + (u1[T::U1::S1] - u1[0]) + (u2[T::U2::S2] - u2[0]);
    }
  }
  __syncthreads();
  lines_c<NT, 0, Q, P, P, 1, Q, TB_H, true, typename T::A0, typename T::B0, EPC, ES>(sA(0), sB(0), tab);
  lines_c<NT, 1, Q, P + 1, P, 1, Q, TB_L, true, typename T::A1, typename T::B1, EPC, ES>(sA(1), sB(1), tab);
  lines_c<NT, 2, Q, P, P + 1, 1, Q, TB_H, true, typename T::A2, typename T::B2, EPC, ES>(sA(2), sB(2), tab);
  __syncthreads();
  lines_c<NT, 0, Q, Q, P, 2, Q, TB_H, true, typename T::B0, typename T::V, EPC, ES>(sB(0), sV(0), tab);
  lines_c<NT, 1, Q, Q, P, 2, Q, TB_H, true, typename T::B1, typename T::V, EPC, ES>(sB(1), sV(1), tab);
  lines_c<NT, 2, Q, Q, P + 1, 2, Q, TB_L, true, typename T::B2, typename T::V, EPC, ES>(sB(2), sV(2), tab);
  __syncthreads();
  // ---- pointwise G_q = w_q mw / det J  J^T J (stored: read from the setup table) ----
  if constexpr (SG) {
    for (int i = tid; i < EPC * NQ; i += NT) {
      const int el = i / NQ, qi = i - (i / NQ) * NQ;
      if (!sEc[el][3]) continue;
      const int qx = qi % Q, qy = (qi / Q) % Q, qz = qi / (Q * Q);
      const double* g = a.geo + (e0 + el) * 6 * NQ + qi;
      const double g00 = __ldcs(g), g11 = __ldcs(g + NQ), g22 = __ldcs(g + 2 * NQ);
      const double g01 = __ldcs(g + 3 * NQ), g02 = __ldcs(g + 4 * NQ), g12 = __ldcs(g + 5 * NQ);
      const int o = el * ES + qx + T::V::S1 * qy + T::V::S2 * qz;
      const double u0 = sV(0)[o], u1 = sV(1)[o], u2 = sV(2)[o];
      sV(0)[o] = g00 * u0 + g01 * u1 + g02 * u2;
      sV(1)[o] = g01 * u0 + g11 * u1 + g12 * u2;
      sV(2)[o] = g02 * u0 + g12 * u1 + g22 * u2;
    }
  }
  for (int i = tid; i < (SG ? 0 : EPC * NQ); i += NT) {
    const int el = i / NQ, qi = i - (i / NQ) * NQ;
    const int qx = qi % Q, qy = (qi / Q) % Q, qz = qi / (Q * Q);
    const double* c0 = sJ[el][0][qy + Q * qz];
    const double* c1 = sJ[el][1][qx + Q * qz];
    const double* c2 = sJ[el][2][qx + Q * qy];
    const double det = c0[0] * (c1[1] * c2[2] - c1[2] * c2[1]) - c1[0] * (c0[1] * c2[2] - c0[2] * c2[1]) +
                       c2[0] * (c0[1] * c1[2] - c0[2] * c1[1]);
    const double s = tab.wq[qx] * tab.wq[qy] * tab.wq[qz] * smw[el] / det;
    const int o = el * ES + qx + T::V::S1 * qy + T::V::S2 * qz;
    const double u0 = sV(0)[o], u1 = sV(1)[o], u2 = sV(2)[o];
    double Ju[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) Ju[d] = c0[d] * u0 + c1[d] * u1 + c2[d] * u2;
    sV(0)[o] = s * (c0[0] * Ju[0] + c0[1] * Ju[1] + c0[2] * Ju[2]);
    sV(1)[o] = s * (c1[0] * Ju[0] + c1[1] * Ju[1] + c1[2] * Ju[2]);
    sV(2)[o] = s * (c2[0] * Ju[0] + c2[1] * Ju[1] + c2[2] * Ju[2]);
  }
  __syncthreads();
  // ---- backward: axis 2, 1, 0 ----
  lines_c<NT, 0, Q, Q, Q, 2, P, TB_H, false, typename T::V, typename T::B0, EPC, ES>(sV(0), sB(0), tab);
  lines_c<NT, 1, Q, Q, Q, 2, P, TB_H, false, typename T::V, typename T::B1, EPC, ES>(sV(1), sB(1), tab);
  lines_c<NT, 2, Q, Q, Q, 2, P + 1, TB_L, false, typename T::V, typename T::B2, EPC, ES>(sV(2), sB(2), tab);
  __syncthreads();
  lines_c<NT, 0, Q, Q, P, 1, P, TB_H, false, typename T::B0, typename T::A0, EPC, ES>(sB(0), sA(0), tab);
  lines_c<NT, 1, Q, Q, P, 1, P + 1, TB_L, false, typename T::B1, typename T::A1, EPC, ES>(sB(1), sA(1), tab);
  lines_c<NT, 2, Q, Q, P + 1, 1, P, TB_H, false, typename T::B2, typename T::A2, EPC, ES>(sB(2), sA(2), tab);
  __syncthreads();
  lines_c<NT, 0, Q, P, P, 0, P + 1, TB_L, false, typename T::A0, typename T::U0, EPC, ES>(sA(0), su(0), tab);
  lines_c<NT, 1, Q, P + 1, P, 0, P, TB_H, false, typename T::A1, typename T::U1, EPC, ES>(sA(1), su(1), tab);
  lines_c<NT, 2, Q, P, P + 1, 0, P, TB_H, false, typename T::A2, typename T::U2, EPC, ES>(sA(2), su(2), tab);
  __syncthreads();
  // ---- D^T q~ and scatter (boundary faces by atomics onto the zeroed y, eliminated faces skipped) ----
  auto put = [&](double* g, double v, int ic, int c, long long gi) {
    if (ic == 0 || ic == P) {
      if (!(ESS && a.ess && face_masked(a.ess, c, gi, a.n[c]))) atomicAdd(g, v);
    } else {
      *g = v;
    }
  };
  for (int l = tid; l < EPC * NU; l += NT) {
    const int el = l / NU, r = l - (l / NU) * NU;
    if (!sEc[el][3]) continue;
    const int ex = sEc[el][0], ey = sEc[el][1], ez = sEc[el][2];
    const double* sr = sreg + el * ES;
    const double* sqe = sq + (BLOCK ? el * T::SL : 0);
    {
      const int li = r % (P + 1), lj = (r / (P + 1)) % P, lk = r / ((P + 1) * P);
      double v = sr[0 * T::SU + li + T::U0::S1 * lj + T::U0::S2 * lk];
      if constexpr (BLOCK) {
        const int cell = li + T::L2::S1 * lj + T::L2::S2 * lk;
        if (li > 0) v += sqe[cell - 1];
        if (li < P) v -= sqe[cell];
      }
      put(a.y + gbase(0, ex, ey, ez) + li + lj * s1x + lk * s2x, v, li, 0, (long long)ex * P + li);
    }
    {
      const int li = r % P, lj = (r / P) % (P + 1), lk = r / (P * (P + 1));
      double v = sr[1 * T::SU + li + T::U1::S1 * lj + T::U1::S2 * lk];
      if constexpr (BLOCK) {
        const int cell = li + T::L2::S1 * lj + T::L2::S2 * lk;
        if (lj > 0) v += sqe[cell - T::L2::S1];
        if (lj < P) v -= sqe[cell];
      }
      put(a.y + gbase(1, ex, ey, ez) + li + lj * s1y + lk * s2y, v, lj, 1, (long long)ey * P + lj);
    }
    {
      const int li = r % P, lj = (r / P) % P, lk = r / (P * P);
      double v = sr[2 * T::SU + li + T::U2::S1 * lj + T::U2::S2 * lk];
      if constexpr (BLOCK) {
        const int cell = li + T::L2::S1 * lj + T::L2::S2 * lk;
        if (lk > 0) v += sqe[cell - T::L2::S2];
        if (lk < P) v -= sqe[cell];
      }
      put(a.y + gbase(2, ex, ey, ez) + li + lj * s1z + lk * s2z, v, lk, 2, (long long)ez * P + lk);
    }
  }
  if constexpr (BLOCK) {
    double* yq = a.y + a.nrt;
    if (a.winv) {   // y_q = D u - s_e W_e^-1 q~_e: the stored inverse streamed column by column
      for (int i = tid; i < EPC * P3; i += NT) {
        const int el = i / P3, r = i - (i / P3) * P3;
        if (!sEc[el][3]) continue;
        const long long e = e0 + el;
        const double* w = a.winv + e * (long long)(P3 * P3) + r;
        const double* qe = sq + el * T::SL;
        double acc = 0.0;
#pragma unroll 8
        for (int c = 0; c < P3; ++c)
          acc = fma(w[c * P3], qe[(c % P) + T::L2::S1 * ((c / P) % P) + T::L2::S2 * (c / (P * P))], acc);
        yq[e0 * P3 + i] = sy[i] - a.zc[4 * e + 1] * acc;
      }
    } else {
      for (int i = tid; i < EPC * P3; i += NT) {
        const int el = i / P3;
        if (sEc[el][3]) yq[e0 * P3 + i] = sy[i];
      }
    }
  }
}

// Z q for p <= 2: one thread per element assembles W^e = sum_q (w_q / det J_q) psi psi^T
// (P^3 x P^3, P:117/P:135 with the histopolation tensor basis) and solves it by Cholesky in
// registers — the paper's "explicit inverse for p <= 2" regime, where a
// 64-thread CTA per element would leave most lanes idle.
template <int P>
__global__ void __launch_bounds__(128) tri_z_direct_kernel(const TriArgs a,
                                                           const __grid_constant__ Tab1D tab,
                                                           long long E) {
  constexpr int Q = P + 2, N = P * P * P;
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= E) return;
  const long long NLx = a.NL[0], NLy = a.NL[1];
  const long long ex = e % NLx, ey = (e / NLx) % NLy, ez = e / (NLx * NLy);
  double X[8][3];
#pragma unroll
  for (int v = 0; v < 8; ++v) {
    const long long g = ((ez + (v >> 2)) * (NLy + 1) + (ey + ((v >> 1) & 1))) * (NLx + 1) + (ex + (v & 1));
#pragma unroll
    for (int d = 0; d < 3; ++d) X[v][d] = a.vert[g * 3 + d];
  }
  double W[N][N];
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) W[i][j] = 0.0;
#pragma unroll 1
  for (int qz = 0; qz < Q; ++qz)
#pragma unroll 1
    for (int qy = 0; qy < Q; ++qy)
#pragma unroll
      for (int qx = 0; qx < Q; ++qx) {
        const double xh = tab.xq[qx], yh = tab.xq[qy], zh = tab.xq[qz];
        double J[3][3];
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          J[d][0] = (1 - yh) * (1 - zh) * (X[1][d] - X[0][d]) + yh * (1 - zh) * (X[3][d] - X[2][d]) +
                    (1 - yh) * zh * (X[5][d] - X[4][d]) + yh * zh * (X[7][d] - X[6][d]);
          J[d][1] = (1 - xh) * (1 - zh) * (X[2][d] - X[0][d]) + xh * (1 - zh) * (X[3][d] - X[1][d]) +
                    (1 - xh) * zh * (X[6][d] - X[4][d]) + xh * zh * (X[7][d] - X[5][d]);
          J[d][2] = (1 - xh) * (1 - yh) * (X[4][d] - X[0][d]) + xh * (1 - yh) * (X[5][d] - X[1][d]) +
                    (1 - xh) * yh * (X[6][d] - X[2][d]) + xh * yh * (X[7][d] - X[3][d]);
        }
        const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                           J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                           J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
        const double g = tab.wq[qx] * tab.wq[qy] * tab.wq[qz] / det;
        double phi[N];
#pragma unroll
        for (int c = 0; c < P; ++c)
#pragma unroll
          for (int b = 0; b < P; ++b)
#pragma unroll
            for (int aa = 0; aa < P; ++aa)
              phi[aa + P * (b + P * c)] = tab.Bh[qx][aa] * tab.Bh[qy][b] * tab.Bh[qz][c];
#pragma unroll
        for (int i = 0; i < N; ++i)
#pragma unroll
          for (int j = 0; j <= i; ++j) W[i][j] = fma(g * phi[i], phi[j], W[i][j]);
      }
  // Cholesky (lower) in place, then forward / backward substitution
#pragma unroll
  for (int j = 0; j < N; ++j) {
    double d = W[j][j];
#pragma unroll
    for (int k = 0; k < j; ++k) d -= W[j][k] * W[j][k];
    d = sqrt(d);
    W[j][j] = d;
#pragma unroll
    for (int i = j + 1; i < N; ++i) {
      double v = W[i][j];
#pragma unroll
      for (int k = 0; k < j; ++k) v -= W[i][k] * W[j][k];
      W[i][j] = v / d;
    }
  }
  double y[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double v = a.x[e * N + i];
#pragma unroll
    for (int k = 0; k < i; ++k) v -= W[i][k] * y[k];
    y[i] = v / W[i][i];
  }
#pragma unroll
  for (int i = N - 1; i >= 0; --i) {
    double v = y[i];
#pragma unroll
    for (int k = i + 1; k < N; ++k) v -= W[k][i] * y[k];
    y[i] = v / W[i][i];
  }
  const double z = a.coef[4 * e + 1];
#pragma unroll
  for (int i = 0; i < N; ++i) a.y[e * N + i] = z * y[i];
}

// elements per CTA of the mass / gamma = 0 applies (r01 A/B, scripts/tri_epc.py on config 3's
// mesh); 0 = the one-element tri_kernel.  Env HDIV_TRI_EPC overrides (clamped to what fits).
static int tri_epc(int p, int mode) {
  const char* e = getenv("HDIV_TRI_EPC");
  if (e) return atoi(e);
  (void)mode;
  // block apply (mass-only) per apply, one-element tri_kernel -> chosen EPC:
  if (p <= 2) return 4;                      // p1 0.50 -> 0.21, p2 0.76 -> 0.34 ms
  if (p == 3) return 2;                      // 1.09 -> 0.78 (0.95 -> 0.71)
  if (p == 4) return (mode == 1) ? 1 : 2;    // 1.55 -> 1.32 (1.25 -> 1.18)
  if (p == 5) return 1;                      // 3.20 -> 2.76 (2.58 -> 2.43)
  return (mode == 1) ? 1 : 0;                // p6 2.52 -> 2.12 (mass: 1.77 stays, 1.91 with EPC 1)
}

// noz: the block apply without its Z term (added by the explicit-inverse apply afterwards)
template <int P, int MODE>
cudaError_t launch_p(const hdiv_ctx* h, const double* x, double* y, const int* skip,
                     cudaStream_t s, bool noz = false, bool* fused = nullptr) {
  const bool hz = h->has_z && !noz;
  // CTA size (r01 A/B of 64 vs 96 threads per order): W^-1 alone at p = 3 — one warp per element (its
  // barriers are warp-synchronous); mass-only / gamma = 0 applies at p = 4, 5 — three warps,
  // one per RT component in every line-pass stage; otherwise 64 threads (the local CG prefers it)
  constexpr int NT = (MODE == 2) ? (P == 3 ? 32 : 64) : 64;
  const bool wide = (MODE != 2) && (P == 4 || P == 5) && !(MODE == 1 && hz);
  TriArgs a;
  a.x = x; a.y = y;
  a.vert = h->d_vert;
  a.coef = (MODE == 2) ? h->d_zcoef : h->d_coef;
  for (int d = 0; d < 3; ++d) { a.NL[d] = h->NL[d]; a.n[d] = h->n[d]; a.off[d] = h->off[d]; }
  a.nrt = h->nrt;
  a.has_z = hz ? 1 : 0;
  a.ess = (MODE == 2) ? 0 : h->ess;
  a.gvert = h->d_gvert;
  a.skip = skip;
  a.winv = nullptr;
  a.zc = h->d_zcoef;
  a.geo = nullptr;
  if constexpr (MODE == 2 && P <= 2) {
    if (!h->d_gvert) {
      count_op();
      tri_z_direct_kernel<P><<<(unsigned)((h->E + 127) / 128), 128, 0, s>>>(a, h->tab, h->E);
      return cudaGetLastError();
    }
  }
  if constexpr (MODE != 2) {
    // EPC elements per 96-thread CTA (mass / gamma = 0 applies), inputs landed by cp.async
    const int epc = tri_epc(P, MODE);
    if (!(MODE == 1 && hz) && epc >= 1) {
      if (MODE == 1 && noz && fused && h->d_winv) {   // Z by the stored inverses, in the epilogue
        a.winv = h->d_winv;
        *fused = true;
      }
      // stored quadrature-point factors (partial assembly) — not with the fused
      // explicit W^-1 epilogue: that path is HBM-bound (streaming the inverses), and the 48 Q^3
      // B per element of G cost more than the Jacobian they save (r02: p = 4 1.97 -> 2.35 ms)
      if (h->d_geo && !a.winv) {
        a.geo = h->d_geo;
        count_op();
        if (P <= 4 && epc >= 2) {   // (two elements fit the 48 KB of static shared memory)
          auto k2 = h->ess ? tri_multi_kernel<P, (P <= 4 ? 2 : 1), MODE == 1, true, true>
                           : tri_multi_kernel<P, (P <= 4 ? 2 : 1), MODE == 1, true, false>;
          k2<<<(unsigned)((h->E + (P <= 4 ? 1 : 0)) / (P <= 4 ? 2 : 1)), 96, 0, s>>>(a, h->tab, h->E);
        } else {
          auto k1 = h->ess ? tri_multi_kernel<P, 1, MODE == 1, true, true>
                           : tri_multi_kernel<P, 1, MODE == 1, true, false>;
          k1<<<(unsigned)h->E, 96, 0, s>>>(a, h->tab, h->E);
        }
        return cudaGetLastError();
      }
      if constexpr (P <= 3) {
        if (epc >= 4) {
          count_op();
          tri_multi_kernel<P, 4, MODE == 1><<<(unsigned)((h->E + 3) / 4), 96, 0, s>>>(a, h->tab, h->E);
          return cudaGetLastError();
        }
      }
      if constexpr (P <= 4) {   // three elements fit the 48 KB of static shared memory
        if (epc >= 3) {
          count_op();
          tri_multi_kernel<P, 3, MODE == 1><<<(unsigned)((h->E + 2) / 3), 96, 0, s>>>(a, h->tab, h->E);
          return cudaGetLastError();
        }
      }
      if constexpr (P <= 5) {
        if (epc >= 2) {
          count_op();
          tri_multi_kernel<P, 2, MODE == 1><<<(unsigned)((h->E + 1) / 2), 96, 0, s>>>(a, h->tab, h->E);
          return cudaGetLastError();
        }
      }
      count_op();
      tri_multi_kernel<P, 1, MODE == 1><<<(unsigned)h->E, 96, 0, s>>>(a, h->tab, h->E);
      return cudaGetLastError();
    }
  }
  if constexpr (MODE != 2 && (P == 4 || P == 5)) {
    if (wide) {
      count_op();
      tri_kernel<P, 96, MODE><<<(unsigned)h->E, 96, 0, s>>>(a, h->tab);
      return cudaGetLastError();
    }
  }
  count_op();
  tri_kernel<P, NT, MODE><<<(unsigned)h->E, NT, 0, s>>>(a, h->tab);
  return cudaGetLastError();
}

template <int MODE>
cudaError_t dispatch(const hdiv_ctx* h, const double* x, double* y, const int* k, cudaStream_t s,
                     bool noz = false, bool* fused = nullptr) {
  switch (h->p) {
    case 1: return launch_p<1, MODE>(h, x, y, k, s, noz, fused);
    case 2: return launch_p<2, MODE>(h, x, y, k, s, noz, fused);
    case 3: return launch_p<3, MODE>(h, x, y, k, s, noz, fused);
    case 4: return launch_p<4, MODE>(h, x, y, k, s, noz, fused);
    case 5: return launch_p<5, MODE>(h, x, y, k, s, noz, fused);
    case 6: return launch_p<6, MODE>(h, x, y, k, s, noz, fused);
  }
  return cudaErrorInvalidValue;
}


// ---- explicit element inverses of W (the paper's "precomputed explicit inverse", P:706-715,
//      P:770; on B200's 180 GB affordable up to p = 4) ----
// Build: one CTA per element assembles W^e_ab = sum_q (w_q / det J_q) psi_a psi_b in the
// histopolation basis psi_a = h_i h_j h_k, factors it W = L L^T in shared
// memory (right-looking, CTA-parallel) and stores (W^e)^-1 column by column: winv[e][c][i] =
// (W^-1)_{ic}, found by the two triangular solves of L L^T x = e_c (one thread per column).
template <int P>
__global__ void __launch_bounds__(128) winv_build_kernel(const double* __restrict__ vert,
                                                         long long NLx, long long NLy,
                                                         const __grid_constant__ Tab1D tab,
                                                         double* __restrict__ winv) {
  constexpr int N = P * P * P, Q = P + 2, NQ = Q * Q * Q, NT = 128;
  extern __shared__ double wsm[];
  double* W = wsm;            // N x N, lower triangle -> L
  double* Y = W + N * N;      // N x N, columns of the inverse
  double* g = Y + N * N;      // NQ: w_q / det J_q
  __shared__ double sX[24];
  const int tid = threadIdx.x;
  const long long e = blockIdx.x;
  const long long ex = e % NLx, ey = (e / NLx) % NLy, ez = e / (NLx * NLy);
  if (tid < 24) {
    const int v = tid / 3, d = tid % 3;
    const long long gv = ((ez + (v >> 2)) * (NLy + 1) + (ey + ((v >> 1) & 1))) * (NLx + 1) + (ex + (v & 1));
    sX[tid] = vert[gv * 3 + d];
  }
  __syncthreads();
  for (int qi = tid; qi < NQ; qi += NT) {
    const int qx = qi % Q, qy = (qi / Q) % Q, qz = qi / (Q * Q);
    const double xh = tab.xq[qx], yh = tab.xq[qy], zh = tab.xq[qz];
    double J[3][3];
    for (int d = 0; d < 3; ++d) {
      auto X = [&](int a, int b, int c) { return sX[(a + 2 * b + 4 * c) * 3 + d]; };
      J[d][0] = (1 - yh) * (1 - zh) * (X(1, 0, 0) - X(0, 0, 0)) + yh * (1 - zh) * (X(1, 1, 0) - X(0, 1, 0)) +
                (1 - yh) * zh * (X(1, 0, 1) - X(0, 0, 1)) + yh * zh * (X(1, 1, 1) - X(0, 1, 1));
      J[d][1] = (1 - xh) * (1 - zh) * (X(0, 1, 0) - X(0, 0, 0)) + xh * (1 - zh) * (X(1, 1, 0) - X(1, 0, 0)) +
                (1 - xh) * zh * (X(0, 1, 1) - X(0, 0, 1)) + xh * zh * (X(1, 1, 1) - X(1, 0, 1));
      J[d][2] = (1 - xh) * (1 - yh) * (X(0, 0, 1) - X(0, 0, 0)) + xh * (1 - yh) * (X(1, 0, 1) - X(1, 0, 0)) +
                (1 - xh) * yh * (X(0, 1, 1) - X(0, 1, 0)) + xh * yh * (X(1, 1, 1) - X(1, 1, 0));
    }
    const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                       J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                       J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
    g[qi] = tab.wq[qx] * tab.wq[qy] * tab.wq[qz] / det;
  }
  __syncthreads();
  for (int idx = tid; idx < N * N; idx += NT) {   // lower triangle (a >= b)
    const int a = idx / N, b = idx % N;
    if (b > a) continue;
    const int ia = a % P, ja = (a / P) % P, ka = a / (P * P);
    const int ib = b % P, jb = (b / P) % P, kb = b / (P * P);
    double w = 0.0;
    for (int qz = 0; qz < Q; ++qz) {
      double ty = 0.0;
      for (int qy = 0; qy < Q; ++qy) {
        double tx = 0.0;
        const double* gr = g + Q * (qy + Q * qz);
        for (int qx = 0; qx < Q; ++qx) tx = fma(gr[qx], tab.Bh[qx][ia] * tab.Bh[qx][ib], tx);
        ty = fma(tx, tab.Bh[qy][ja] * tab.Bh[qy][jb], ty);
      }
      w = fma(ty, tab.Bh[qz][ka] * tab.Bh[qz][kb], w);
    }
    W[a * N + b] = w;
  }
  __syncthreads();
  for (int k = 0; k < N; ++k) {   // W = L L^T, L in the lower triangle
    if (tid == 0) W[k * N + k] = sqrt(W[k * N + k]);
    __syncthreads();
    const double dk = W[k * N + k];
    for (int i = k + 1 + tid; i < N; i += NT) W[i * N + k] /= dk;
    __syncthreads();
    const int m = N - k - 1;
    for (int idx = tid; idx < m * m; idx += NT) {
      const int i = k + 1 + idx / m, j = k + 1 + idx % m;
      if (j <= i) W[i * N + j] -= W[i * N + k] * W[j * N + k];
    }
    __syncthreads();
  }
  if (tid < N) {   // column c of W^-1: L y = e_c, L^T x = y (in place in Y's column c)
    const int c = tid;
    for (int i = 0; i < N; ++i) {
      double v = (i == c) ? 1.0 : 0.0;
      for (int k = 0; k < i; ++k) v -= W[i * N + k] * Y[k * N + c];
      Y[i * N + c] = v / W[i * N + i];
    }
    for (int i = N - 1; i >= 0; --i) {
      double v = Y[i * N + c];
      for (int k = i + 1; k < N; ++k) v -= W[k * N + i] * Y[k * N + c];
      Y[i * N + c] = v / W[i * N + i];
    }
    double* out = winv + e * (long long)(N * N) + (long long)c * N;
    for (int i = 0; i < N; ++i) out[i] = Y[i * N + c];
  }
}

// y_q = s_e W_e^-1 q_e (ACC: y_q -= s_e W_e^-1 q_e), one warp per element: for every column c
// the warp streams winv[e][c][0..N) (contiguous) and adds q_c times it into lane rows
// r = lane, lane + 32 (fixed order: deterministic)
template <int P, bool ACC>
__global__ void __launch_bounds__(128) winv_apply_kernel(const double* __restrict__ winv,
                                                         const double* __restrict__ q,
                                                         double* __restrict__ y,
                                                         const double* __restrict__ zcoef,
                                                         long long E, const int* skip) {
  constexpr int N = P * P * P;
  static_assert(N <= 64, "two rows per lane");
  if (skip && *skip) return;
  const int lane = threadIdx.x & 31;
  const long long e = (long long)blockIdx.x * 4 + (threadIdx.x >> 5);
  if (e >= E) return;
  const double* qe = q + e * N;
  const double q0 = lane < N ? qe[lane] : 0.0;
  const double q1 = lane + 32 < N ? qe[lane + 32] : 0.0;
  const double* we = winv + e * (long long)(N * N);
  double a0 = 0.0, a1 = 0.0;
#pragma unroll 8
  for (int c = 0; c < N; ++c) {
    const double qc = __shfl_sync(0xffffffffu, c < 32 ? q0 : q1, c & 31);
    const double* col = we + c * N;
    if (lane < N) a0 = fma(col[lane], qc, a0);
    if (lane + 32 < N) a1 = fma(col[lane + 32], qc, a1);
  }
  const double s = zcoef[4 * e + 1];
  double* ye = y + e * N;
  if (lane < N) ye[lane] = ACC ? ye[lane] - s * a0 : s * a0;
  if (lane + 32 < N) ye[lane + 32] = ACC ? ye[lane + 32] - s * a1 : s * a1;
}

// p <= 2 (p^3 <= 8 rows): one thread per (element, row), columns in order
template <int P, bool ACC>
__global__ void __launch_bounds__(256) winv_apply_small_kernel(const double* __restrict__ winv,
                                                               const double* __restrict__ q,
                                                               double* __restrict__ y,
                                                               const double* __restrict__ zcoef,
                                                               long long E, const int* skip) {
  constexpr int N = P * P * P;
  if (skip && *skip) return;
  const long long t = (long long)blockIdx.x * 256 + threadIdx.x;
  if (t >= E * N) return;
  const long long e = t / N;
  const int r = (int)(t - e * N);
  const double* we = winv + e * (N * N) + r;
  const double* qe = q + e * N;
  double a = 0.0;
#pragma unroll
  for (int c = 0; c < N; ++c) a = fma(we[c * N], qe[c], a);
  const double s = zcoef[4 * e + 1];
  y[t] = ACC ? y[t] - s * a : s * a;
}

template <int P>
cudaError_t winv_build_p(hdiv_ctx* h, cudaStream_t s) {
  constexpr int N = P * P * P, Q = P + 2;
  const size_t smem = sizeof(double) * (2 * N * N + Q * Q * Q);
  cudaError_t e = cudaFuncSetAttribute(winv_build_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  winv_build_kernel<P><<<(unsigned)h->E, 128, smem, s>>>(h->d_vert, h->NL[0], h->NL[1], h->tab, h->d_winv);
  return cudaGetLastError();
}

template <int P, bool ACC>
cudaError_t winv_apply_p(const hdiv_ctx* h, const double* q, double* y, const int* skip, cudaStream_t s) {
  if constexpr (P <= 2) {
    const long long n = h->E * P * P * P;
    count_op();
    winv_apply_small_kernel<P, ACC><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(h->d_winv, q, y, h->d_zcoef, h->E, skip);
    return cudaGetLastError();
  }
  count_op();
  winv_apply_kernel<P, ACC><<<(unsigned)((h->E + 3) / 4), 128, 0, s>>>(h->d_winv, q, y, h->d_zcoef, h->E, skip);
  return cudaGetLastError();
}

template <bool ACC>
cudaError_t winv_apply(const hdiv_ctx* h, const double* q, double* y, const int* skip, cudaStream_t s) {
  switch (h->p) {
    case 1: return winv_apply_p<1, ACC>(h, q, y, skip, s);
    case 2: return winv_apply_p<2, ACC>(h, q, y, skip, s);
    case 3: return winv_apply_p<3, ACC>(h, q, y, skip, s);
    case 4: return winv_apply_p<4, ACC>(h, q, y, skip, s);
  }
  return cudaErrorInvalidValue;
}
// Stored quadrature-point factors (the paper's partial assembly: geometric factors precomputed
// at the quadrature points): G_q = w_q mw_e / det J_q  J_q^T J_q (symmetric, 6
// entries {00, 11, 22, 01, 02, 12}), layout [E][6][Q^3] (q fastest: the pointwise stage reads
// each entry coalesced).  One thread per (element, point); J from the 8 vertices (trilinear map).
template <int P>
__global__ void __launch_bounds__(256) geo_build_kernel(const double* __restrict__ vert, long long NLx,
                                                        long long NLy, const __grid_constant__ Tab1D tab,
                                                        const double* __restrict__ coef, long long E,
                                                        double* __restrict__ geo) {
  constexpr int Q = P + 2, NQ = Q * Q * Q;
  const long long t = (long long)blockIdx.x * 256 + threadIdx.x;
  if (t >= E * NQ) return;
  const long long e = t / NQ;
  const int qi = (int)(t - e * NQ);
  const int qx = qi % Q, qy = (qi / Q) % Q, qz = qi / (Q * Q);
  const long long ex = e % NLx, ey = (e / NLx) % NLy, ez = e / (NLx * NLy);
  double X[8][3];
#pragma unroll
  for (int v = 0; v < 8; ++v) {
    const long long g = ((ez + (v >> 2)) * (NLy + 1) + (ey + ((v >> 1) & 1))) * (NLx + 1) + (ex + (v & 1));
#pragma unroll
    for (int d = 0; d < 3; ++d) X[v][d] = vert[g * 3 + d];
  }
  const double xh = tab.xq[qx], yh = tab.xq[qy], zh = tab.xq[qz];
  double c[3][3];   // c[k][d] = dT_d / dx_hat_k
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    c[0][d] = (1 - yh) * (1 - zh) * (X[1][d] - X[0][d]) + yh * (1 - zh) * (X[3][d] - X[2][d]) +
              (1 - yh) * zh * (X[5][d] - X[4][d]) + yh * zh * (X[7][d] - X[6][d]);
    c[1][d] = (1 - xh) * (1 - zh) * (X[2][d] - X[0][d]) + xh * (1 - zh) * (X[3][d] - X[1][d]) +
              (1 - xh) * zh * (X[6][d] - X[4][d]) + xh * zh * (X[7][d] - X[5][d]);
    c[2][d] = (1 - xh) * (1 - yh) * (X[4][d] - X[0][d]) + xh * (1 - yh) * (X[5][d] - X[1][d]) +
              (1 - xh) * yh * (X[6][d] - X[2][d]) + xh * yh * (X[7][d] - X[3][d]);
  }
  const double det = c[0][0] * (c[1][1] * c[2][2] - c[1][2] * c[2][1]) -
                     c[1][0] * (c[0][1] * c[2][2] - c[0][2] * c[2][1]) +
                     c[2][0] * (c[0][1] * c[1][2] - c[0][2] * c[1][1]);
  const double sc = tab.wq[qx] * tab.wq[qy] * tab.wq[qz] * coef[4 * e] / det;
  auto dot = [&](int i, int j) { return c[i][0] * c[j][0] + c[i][1] * c[j][1] + c[i][2] * c[j][2]; };
  double* g = geo + e * 6 * NQ + qi;
  g[0] = sc * dot(0, 0);
  g[NQ] = sc * dot(1, 1);
  g[2 * NQ] = sc * dot(2, 2);
  g[3 * NQ] = sc * dot(0, 1);
  g[4 * NQ] = sc * dot(0, 2);
  g[5 * NQ] = sc * dot(1, 2);
}

template <int P>
cudaError_t geo_build_p(hdiv_ctx* h, cudaStream_t s) {
  constexpr int Q = P + 2;
  const long long n = h->E * Q * Q * Q;
  geo_build_kernel<P><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(h->d_vert, h->NL[0], h->NL[1], h->tab,
                                                                  h->d_coef, h->E, h->d_geo);
  return cudaGetLastError();
}
}  // namespace

// stored quadrature-point factors for the mass / gamma = 0 applies (d_coef[4e] = mass weight)
cudaError_t build_tri_geo(hdiv_ctx* h, cudaStream_t s) {
  switch (h->p) {
    case 1: return geo_build_p<1>(h, s);
    case 2: return geo_build_p<2>(h, s);
    case 3: return geo_build_p<3>(h, s);
    case 4: return geo_build_p<4>(h, s);
    case 5: return geo_build_p<5>(h, s);
    case 6: return geo_build_p<6>(h, s);
  }
  return cudaErrorInvalidValue;
}

// the explicit element inverses of W (p <= 4), built at setup when they fit the memory budget
cudaError_t build_winv(hdiv_ctx* h, cudaStream_t s) {
  switch (h->p) {
    case 1: return winv_build_p<1>(h, s);
    case 2: return winv_build_p<2>(h, s);
    case 3: return winv_build_p<3>(h, s);
    case 4: return winv_build_p<4>(h, s);
  }
  return cudaErrorInvalidValue;
}

// y (RT part zeroed here) = M u  /  [M u + D^T q ; D u - Z q], 3D, any trilinear geometry.
// With the explicit inverses: Z q by the streaming inverse apply (block: the gamma = 0 kernel
// writes [M u + D^T q ; D u], then y_q -= s_e W_e^-1 q_e)
cudaError_t launch_trilinear_apply(const hdiv_ctx* h, const double* x, double* y, int mode,
                                   const int* skip, cudaStream_t s) {
  if (mode == MODE_ZONLY) {
    if (h->d_winv) return winv_apply<false>(h, x, y, skip, s);
    return dispatch<2>(h, x, y, skip, s);   // y (L2) fully written
  }
  count_op();
  cudaError_t e = cudaMemsetAsync(y, 0, sizeof(double) * h->nrt, s);
  if (e != cudaSuccess) return e;
  if (mode == MODE_BLOCK) {
    if (h->d_winv) {
      static const bool fuse = [] {
        const char* v = getenv("HDIV_WINV_FUSE");
        return !(v && atoi(v) == 0);
      }();
      bool fused = false;
      e = dispatch<1>(h, x, y, skip, s, true, fuse ? &fused : nullptr);
      if (e != cudaSuccess || fused) return e;
      return winv_apply<true>(h, x + h->nrt, y + h->nrt, skip, s);
    }
    return dispatch<1>(h, x, y, skip, s);
  }
  return dispatch<0>(h, x, y, skip, s);
}

}  // namespace hdiv
