// kernel_affine.cu — fused block-operator apply on axis-aligned box elements (3D).
//
//   y_u = M_beta u + D^T q~ ,  y_q = D u - Z q~
//
// On a box element with sizes (hx,hy,hz) the Piola-mapped RT mass is block diagonal in the
// components and each block is a Kronecker product of 1D masses (exact):
//   M^e_x = c_x (M_h (x) M_h (x) M_l),  c_x = beta hx / (hy hz)   (and cyclic)
//   Z^e   = z_e (M_h^-1)^{(x)3},        z_e = detJ/alpha (grad-div) | gamma detJ (Darcy)
// D is the signed subcell-face incidence: (D u)_cell = sum over the 6 faces +-u.
//
// B200 design:
//  * one CTA per tile of TXxTYxTZ elements; every DOF is read once from HBM (cp.async into
//    shared memory) and written once — no atomics, no zero-fill;
//  * a face plane shared by two tiles is OWNED by the tile on its + side; that tile
//    recomputes the - side neighbour element's contribution from a one-element halo of the
//    single component involved (1/T of one component; neighbours' reads hit L2);
//  * sum factorisation: two element-local M_h passes, then one line pass along the component
//    direction that applies c_e M_l element by element, carries the shared-plane sum in a
//    register and adds D^T q~; one thread owns a whole line, smem row strides are odd, so
//    the passes are bank-conflict free;
//  * D u and -Z q~ are accumulated in registers by the thread that owns each cell and stored
//    coalesced (the L2 DOFs of a tile row are contiguous in HBM).
#include <cuda_runtime.h>

#include "internal.h"

namespace hdiv {
namespace {

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

constexpr int odd_up(int v) { return (v % 2) ? v : v + 1; }

template <int P, int TX, int TY, int TZ>
struct Geo {
  // x-component tile: [K][J][I'], I' in [0,(TX+1)P], I' = 0 <-> global plane (ex0-1)P
  static constexpr int XI = odd_up((TX + 1) * P + 1), XJ = TY * P, XK = TZ * P;
  // y-component tile: [K][J'][I]
  static constexpr int YI = odd_up(TX * P), YJ = (TY + 1) * P + 1, YK = TZ * P;
  // z-component tile: [K'][J][I]
  static constexpr int ZI = odd_up(TX * P), ZJ = TY * P, ZK = (TZ + 1) * P + 1;
  static constexpr int SX = XI * XJ * XK, SY = YI * YJ * YK, SZ = ZI * ZJ * ZK;
  static constexpr int P3 = P * P * P;
  static constexpr int NE = TX * TY * TZ;
  static constexpr int NCELL = NE * P3;
  static constexpr int RQ = odd_up(P);                 // padded a-row of the Z scratch
  static constexpr int SZQ = NE * RQ * P * P;
  static constexpr int SU0 = SX > SY ? (SX > SZ ? SX : SZ) : (SY > SZ ? SY : SZ);
  static constexpr int SU = SU0 > SZQ ? SU0 : SZQ;
  static constexpr int HQX = TZ * P * TY * P, HQY = TZ * P * TX * P, HQZ = TY * P * TX * P;
  static constexpr int NCO = (TX + 1) * (TY + 1) * (TZ + 1);
  static constexpr size_t smem_doubles(bool block) {
    return (size_t)SU + (block ? (size_t)NCELL + HQX + HQY + HQZ : 0) + 4 * NCO;
  }
};

struct AffArgs {
  const double* x;     // [u ; q]
  double* y;           // [y_u ; y_q]
  const double* coef;  // [E][4] = {cx, cy, cz, z}
  long long NL[3];     // local element counts
  long long n[3];      // local subcell counts
  long long off[3];    // RT component offsets
  long long nrt;
  int ntile[3];
  int has_z;
  const int* skip;   // MINRES done flag (nullptr: never skip)
};

template <int P>
__device__ __forceinline__ void matvec_h(const double (*M)[MAXP], double* v) {
  double w[P];
#pragma unroll
  for (int i = 0; i < P; ++i) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < P; ++j) s = fma(M[i][j], v[j], s);
    w[i] = s;
  }
#pragma unroll
  for (int i = 0; i < P; ++i) v[i] = w[i];
}

// In-place element-local contraction along one axis.  Element k of line (i0,i1,blk) lives at
// s[off + i0*s0 + i1*s1 + blk*sb + k*se]; lanes run over i0 first.
template <int P, int NT>
__device__ __forceinline__ void hpass(double* s, const double (*M)[MAXP], int off, int n0,
                                      int s0, int n1, int s1, int nb, int sb, int se) {
  const int total = n0 * n1 * nb;
  for (int it = threadIdx.x; it < total; it += NT) {
    const int i0 = it % n0;
    const int r = it / n0;
    const int i1 = r % n1;
    const int blk = r / n1;
    double* b = s + off + i0 * s0 + i1 * s1 + blk * sb;
    double v[P];
#pragma unroll
    for (int k = 0; k < P; ++k) v[k] = b[k * se];
    matvec_h<P>(M, v);
#pragma unroll
    for (int k = 0; k < P; ++k) b[k * se] = v[k];
  }
}

// Line pass along the component axis AX (0 x, 1 y, 2 z).  Lines are indexed by the two other
// subcell coordinates (l0 = lane-fast, l1).  Element et (in [-h, m)) covers positions
// (et+1)P .. (et+1)P+P of the line (stride sl).  Applies c_e M_l, sums the shared planes,
// adds D^T q~ (BLOCK), writes the owned planes [P, (m+1)P) (+ the last plane if `last`).
template <int P, int TX, int TY, int TZ, int NT, int AX, bool BLOCK>
__device__ __forceinline__ void lpass(double* su, const double* sq, const double* hq,
                                      const double* sco, const TabAffine& tab, int n0, int s0,
                                      int n1, int s1, int sl, int m, int h, bool last) {
  using G = Geo<P, TX, TY, TZ>;
  constexpr int P3 = G::P3;
  const int total = n0 * n1;
  for (int it = threadIdx.x; it < total; it += NT) {
    const int l0 = it % n0, l1 = it / n0;
    double* line = su + l0 * s0 + l1 * s1;
    // other-axis element / local coordinates of this line
    int e_o0, loc_o0, e_o1, loc_o1;   // (x: J->y, K->z ; y: I->x, K->z ; z: I->x, J->y)
    e_o0 = l0 / P; loc_o0 = l0 % P;
    e_o1 = l1 / P; loc_o1 = l1 % P;
    int ex = 0, ey = 0, ez = 0;
    // q~ addressing: cell (ex,ey,ez ; a,b,c) -> ((ez*TY+ey)*TX+ex)*P3 + a + P b + P^2 c
    int qbase = 0, qstep_loc = 1, qstep_el = P3, hqi = 0;
    if (AX == 0) {
      ey = e_o0; ez = e_o1;
      qbase = ((ez * TY + ey) * TX) * P3 + P * loc_o0 + P * P * loc_o1;
      qstep_loc = 1; qstep_el = P3;
      hqi = l1 * (TY * P) + l0;
    } else if (AX == 1) {
      ex = e_o0; ez = e_o1;
      qbase = ((ez * TY) * TX + ex) * P3 + loc_o0 + P * P * loc_o1;
      qstep_loc = P; qstep_el = TX * P3;
      hqi = l1 * (TX * P) + l0;
    } else {
      ex = e_o0; ey = e_o1;
      qbase = (ey * TX + ex) * P3 + loc_o0 + P * loc_o1;
      qstep_loc = P * P; qstep_el = TX * TY * P3;
      hqi = l1 * (TX * P) + l0;
    }
    auto cof = [&](int et) -> double {
      int cx = (AX == 0) ? et : ex, cy = (AX == 1) ? et : ey, cz = (AX == 2) ? et : ez;
      return sco[4 * (((cz + 1) * (TY + 1) + (cy + 1)) * (TX + 1) + (cx + 1)) + AX];
    };
    double carry = 0.0;
    if (h) {   // halo element et = -1: only its contribution to plane P
      double v[P + 1];
#pragma unroll
      for (int i = 0; i <= P; ++i) v[i] = line[i * sl];
      double s = 0.0;
#pragma unroll
      for (int j = 0; j <= P; ++j) s = fma(tab.Ml[P][j], v[j], s);
      carry = cof(-1) * s;
    }
    double qprev = 0.0;   // q~ of the cell on the - side of the current plane
    if (BLOCK && h) qprev = hq[hqi];
    for (int et = 0; et < m; ++et) {
      double* eb = line + (et + 1) * P * sl;
      double v[P + 1];
#pragma unroll
      for (int i = 0; i <= P; ++i) v[i] = eb[i * sl];
      const double c = cof(et);
      double w[P + 1];
#pragma unroll
      for (int i = 0; i <= P; ++i) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j <= P; ++j) s = fma(tab.Ml[i][j], v[j], s);
        w[i] = c * s;
      }
      w[0] += carry;
      if constexpr (BLOCK) {
        const double* qe = sq + qbase + et * qstep_el;
#pragma unroll
        for (int i = 0; i < P; ++i) {
          double qc = qe[i * qstep_loc];
          w[i] += qprev - qc;   // (D^T q)_face = q(- side cell) - q(+ side cell)
          qprev = qc;
        }
      }
#pragma unroll
      for (int i = 0; i < P; ++i) eb[i * sl] = w[i];
      carry = w[P];
    }
    if (last) line[(m + 1) * P * sl] = carry + (BLOCK ? qprev : 0.0);
  }
}

template <int P, int TX, int TY, int TZ, int NT, bool BLOCK>
__global__ void __launch_bounds__(NT)
affine_apply_kernel(const AffArgs a, const __grid_constant__ TabAffine tab) {
  using G = Geo<P, TX, TY, TZ>;
  constexpr int P3 = G::P3;
  if (a.skip && *a.skip) return;
  extern __shared__ double smem[];
  double* su = smem;                                  // component tile / Z scratch
  double* sq = su + G::SU;                            // q~ tile (element-major)
  double* hqx = sq + (BLOCK ? G::NCELL : 0);          // halo q~ for owned -x planes [K][J]
  double* hqy = hqx + (BLOCK ? G::HQX : 0);           // [K][I]
  double* hqz = hqy + (BLOCK ? G::HQY : 0);           // [J][I]
  double* sco = hqz + (BLOCK ? G::HQZ : 0);           // coefficients [(TZ+1)][(TY+1)][(TX+1)][4]

  const int tid = threadIdx.x;
  int t = blockIdx.x;
  const int tx = t % a.ntile[0];
  t /= a.ntile[0];
  const int ty = t % a.ntile[1];
  const int tz = t / a.ntile[1];
  const long long NLx = a.NL[0], NLy = a.NL[1], NLz = a.NL[2];
  const int ex0 = tx * TX, ey0 = ty * TY, ez0 = tz * TZ;
  const int mx = (int)min((long long)TX, NLx - ex0);
  const int my = (int)min((long long)TY, NLy - ey0);
  const int mz = (int)min((long long)TZ, NLz - ez0);
  const int hx = ex0 > 0, hy = ey0 > 0, hz = ez0 > 0;
  const bool lastx = (ex0 + mx == NLx), lasty = (ey0 + my == NLy), lastz = (ez0 + mz == NLz);
  const long long nx = a.n[0], ny = a.n[1];
  const double* u = a.x;
  const double* q = a.x + a.nrt;

  // ---- coefficients of the tile and its - halo ----
  for (int i = tid; i < G::NCO; i += NT) {
    int ix = i % (TX + 1), iy = (i / (TX + 1)) % (TY + 1), iz = i / ((TX + 1) * (TY + 1));
    long long ex = ex0 - 1 + ix, ey = ey0 - 1 + iy, ez = ez0 - 1 + iz;
    if (ex >= 0 && ey >= 0 && ez >= 0 && ex < ex0 + mx && ey < ey0 + my && ez < ez0 + mz) {
      const double* c = a.coef + 4 * ((ez * NLy + ey) * NLx + ex);
#pragma unroll
      for (int k = 0; k < 4; ++k) cp_async8(sco + 4 * i + k, c + k);
    }
  }

  constexpr int NQR = (G::NCELL + NT - 1) / NT;
  double acc[NQR];
#pragma unroll
  for (int k = 0; k < NQR; ++k) acc[k] = 0.0;

  if constexpr (BLOCK) {
    for (int i = tid; i < G::NCELL; i += NT) {
      int e = i / P3, il = i % P3;
      int etx = e % TX, ety = (e / TX) % TY, etz = e / (TX * TY);
      if (etx < mx && ety < my && etz < mz) {
        long long ge = ((long long)(ez0 + etz) * NLy + (ey0 + ety)) * NLx + (ex0 + etx);
        cp_async8(sq + i, q + ge * P3 + il);
      }
    }
    if (hx)
      for (int i = tid; i < my * P * mz * P; i += NT) {
        int J = i % (my * P), K = i / (my * P);
        long long ge = ((long long)(ez0 + K / P) * NLy + (ey0 + J / P)) * NLx + (ex0 - 1);
        cp_async8(hqx + K * (TY * P) + J, q + ge * P3 + (P - 1) + P * ((J % P) + P * (K % P)));
      }
    if (hy)
      for (int i = tid; i < mx * P * mz * P; i += NT) {
        int I = i % (mx * P), K = i / (mx * P);
        long long ge = ((long long)(ez0 + K / P) * NLy + (ey0 - 1)) * NLx + (ex0 + I / P);
        cp_async8(hqy + K * (TX * P) + I, q + ge * P3 + (I % P) + P * ((P - 1) + P * (K % P)));
      }
    if (hz)
      for (int i = tid; i < mx * P * my * P; i += NT) {
        int I = i % (mx * P), J = i / (mx * P);
        long long ge = ((long long)(ez0 - 1) * NLy + (ey0 + J / P)) * NLx + (ex0 + I / P);
        cp_async8(hqz + J * (TX * P) + I, q + ge * P3 + (I % P) + P * ((J % P) + P * (P - 1)));
      }
  }
  cp_async_wait_all();
  __syncthreads();

  if constexpr (BLOCK) {
    if (a.has_z) {
      // -Z q~ = -z_e (Mh^-1)^{(x)3} q~_e ; scratch layout [e][c][b][a] with a-row stride RQ
      constexpr int RQ = G::RQ, EST = RQ * P * P;
      for (int i = tid; i < G::NCELL; i += NT) {
        int e = i / P3, il = i % P3;
        su[e * EST + (il / P) * RQ + il % P] = sq[i];
      }
      __syncthreads();
      // a-lines: lanes over (b,c) rows [stride RQ, odd] then elements
      hpass<P, NT>(su, tab.Mhinv, 0, P * P, RQ, G::NE, EST, 1, 0, 1);
      __syncthreads();
      // b-lines: lanes over a, then (c, e)
      hpass<P, NT>(su, tab.Mhinv, 0, P, 1, P * G::NE, RQ * P, 1, 0, RQ);
      __syncthreads();
      // c-lines: lanes over a, then (b, e) -- i1 = b + P e is not affine in memory, so run
      // over b explicitly
      for (int b = 0; b < P; ++b)
        hpass<P, NT>(su, tab.Mhinv, b * RQ, P, 1, G::NE, EST, 1, 0, RQ * P);
      __syncthreads();
#pragma unroll
      for (int k = 0; k < NQR; ++k) {
        int i = tid + k * NT;
        if (i < G::NCELL) {
          int e = i / P3, il = i % P3;
          int etx = e % TX, ety = (e / TX) % TY, etz = e / (TX * TY);
          if (etx < mx && ety < my && etz < mz) {
            double z = sco[4 * (((etz + 1) * (TY + 1) + (ety + 1)) * (TX + 1) + (etx + 1)) + 3];
            acc[k] = -z * su[e * EST + (il / P) * RQ + il % P];
          }
        }
      }
      __syncthreads();
    }
  }

  // ======================= x component =======================
  {
    constexpr int XI = G::XI, XJ = G::XJ;
    const int ilo = hx ? 0 : P;
    const int nI = (mx + 1) * P + 1 - ilo;
    const int nJ = my * P, nK = mz * P;
    const long long gI0 = (long long)(ex0 - 1) * P;
    for (int i = tid; i < nI * nJ * nK; i += NT) {
      int I = i % nI + ilo, r = i / nI, J = r % nJ, K = r / nJ;
      long long g = a.off[0] + (gI0 + I) + (nx + 1) * ((long long)(ey0 * P + J) + ny * (ez0 * P + K));
      cp_async8(su + (K * XJ + J) * XI + I, u + g);
    }
    cp_async_wait_all();
    __syncthreads();
    if constexpr (BLOCK) {
#pragma unroll
      for (int k = 0; k < NQR; ++k) {
        int i = tid + k * NT;
        int e = i / P3, il = i % P3;
        int etx = e % TX, ety = (e / TX) % TY, etz = e / (TX * TY);
        if (i < G::NCELL && etx < mx && ety < my && etz < mz) {
          int A = il % P, B = (il / P) % P, C = il / (P * P);
          const double* s = su + ((etz * P + C) * XJ + ety * P + B) * XI + (etx + 1) * P + A;
          acc[k] += s[1] - s[0];
        }
      }
      __syncthreads();
    }
    hpass<P, NT>(su, tab.Mh, ilo, nI, 1, nJ, XI, mz, P * XI * XJ, XI * XJ);      // K
    __syncthreads();
    hpass<P, NT>(su, tab.Mh, ilo, nI, 1, nK, XI * XJ, my, P * XI, XI);           // J
    __syncthreads();
    lpass<P, TX, TY, TZ, NT, 0, BLOCK>(su, sq, hqx, sco, tab, nJ, XI, nK, XI * XJ, 1, mx, hx,
                                      lastx);
    __syncthreads();
    const int nO = mx * P + (lastx ? 1 : 0);
    for (int i = tid; i < nO * nJ * nK; i += NT) {
      int I = i % nO + P, r = i / nO, J = r % nJ, K = r / nJ;
      long long g = a.off[0] + (gI0 + I) + (nx + 1) * ((long long)(ey0 * P + J) + ny * (ez0 * P + K));
      a.y[g] = su[(K * XJ + J) * XI + I];
    }
    __syncthreads();
  }
  // ======================= y component =======================
  {
    constexpr int YI = G::YI, YJ = G::YJ;
    const int jlo = hy ? 0 : P;
    const int nJ = (my + 1) * P + 1 - jlo;
    const int nI = mx * P, nK = mz * P;
    const long long gJ0 = (long long)(ey0 - 1) * P;
    for (int i = tid; i < nI * nJ * nK; i += NT) {
      int I = i % nI, r = i / nI, J = r % nJ + jlo, K = r / nJ;
      long long g = a.off[1] + (ex0 * P + I) + nx * ((gJ0 + J) + (ny + 1) * (long long)(ez0 * P + K));
      cp_async8(su + (K * YJ + J) * YI + I, u + g);
    }
    cp_async_wait_all();
    __syncthreads();
    if constexpr (BLOCK) {
#pragma unroll
      for (int k = 0; k < NQR; ++k) {
        int i = tid + k * NT;
        int e = i / P3, il = i % P3;
        int etx = e % TX, ety = (e / TX) % TY, etz = e / (TX * TY);
        if (i < G::NCELL && etx < mx && ety < my && etz < mz) {
          int A = il % P, B = (il / P) % P, C = il / (P * P);
          const double* s = su + ((etz * P + C) * YJ + (ety + 1) * P + B) * YI + etx * P + A;
          acc[k] += s[YI] - s[0];
        }
      }
      __syncthreads();
    }
    hpass<P, NT>(su, tab.Mh, jlo * YI, nJ, YI, nK, YI * YJ, mx, P, 1);           // I
    __syncthreads();
    hpass<P, NT>(su, tab.Mh, jlo * YI, nI, 1, nJ, YI, mz, P * YI * YJ, YI * YJ);  // K
    __syncthreads();
    lpass<P, TX, TY, TZ, NT, 1, BLOCK>(su, sq, hqy, sco, tab, nI, 1, nK, YI * YJ, YI, my, hy,
                                      lasty);
    __syncthreads();
    const int nO = my * P + (lasty ? 1 : 0);
    for (int i = tid; i < nI * nO * nK; i += NT) {
      int I = i % nI, r = i / nI, J = r % nO + P, K = r / nO;
      long long g = a.off[1] + (ex0 * P + I) + nx * ((gJ0 + J) + (ny + 1) * (long long)(ez0 * P + K));
      a.y[g] = su[(K * YJ + J) * YI + I];
    }
    __syncthreads();
  }
  // ======================= z component =======================
  {
    constexpr int ZI = G::ZI, ZJ = G::ZJ;
    const int klo = hz ? 0 : P;
    const int nK = (mz + 1) * P + 1 - klo;
    const int nI = mx * P, nJ = my * P;
    const long long gK0 = (long long)(ez0 - 1) * P;
    for (int i = tid; i < nI * nJ * nK; i += NT) {
      int I = i % nI, r = i / nI, J = r % nJ, K = r / nJ + klo;
      long long g = a.off[2] + (ex0 * P + I) + nx * ((long long)(ey0 * P + J) + ny * (gK0 + K));
      cp_async8(su + (K * ZJ + J) * ZI + I, u + g);
    }
    cp_async_wait_all();
    __syncthreads();
    if constexpr (BLOCK) {
#pragma unroll
      for (int k = 0; k < NQR; ++k) {
        int i = tid + k * NT;
        int e = i / P3, il = i % P3;
        int etx = e % TX, ety = (e / TX) % TY, etz = e / (TX * TY);
        if (i < G::NCELL && etx < mx && ety < my && etz < mz) {
          int A = il % P, B = (il / P) % P, C = il / (P * P);
          const double* s = su + (((etz + 1) * P + C) * ZJ + ety * P + B) * ZI + etx * P + A;
          acc[k] += s[ZI * ZJ] - s[0];
        }
      }
      __syncthreads();
    }
    hpass<P, NT>(su, tab.Mh, klo * ZI * ZJ, nJ, ZI, nK, ZI * ZJ, mx, P, 1);      // I
    __syncthreads();
    hpass<P, NT>(su, tab.Mh, klo * ZI * ZJ, nI, 1, nK, ZI * ZJ, my, P * ZI, ZI);  // J
    __syncthreads();
    lpass<P, TX, TY, TZ, NT, 2, BLOCK>(su, sq, hqz, sco, tab, nI, 1, nJ, ZI, ZI * ZJ, mz, hz,
                                      lastz);
    __syncthreads();
    const int nO = mz * P + (lastz ? 1 : 0);
    for (int i = tid; i < nI * nJ * nO; i += NT) {
      int I = i % nI, r = i / nI, J = r % nJ, K = r / nJ + P;
      long long g = a.off[2] + (ex0 * P + I) + nx * ((long long)(ey0 * P + J) + ny * (gK0 + K));
      a.y[g] = su[(K * ZJ + J) * ZI + I];
    }
  }
  // ======================= L2 block =======================
  if constexpr (BLOCK) {
    double* yq = a.y + a.nrt;
#pragma unroll
    for (int k = 0; k < NQR; ++k) {
      int i = tid + k * NT;
      int e = i / P3, il = i % P3;
      int etx = e % TX, ety = (e / TX) % TY, etz = e / (TX * TY);
      if (i < G::NCELL && etx < mx && ety < my && etz < mz) {
        long long ge = ((long long)(ez0 + etz) * NLy + (ey0 + ety)) * NLx + (ex0 + etx);
        yq[ge * P3 + il] = acc[k];
      }
    }
  }
}

template <int P, int TX, int TY, int TZ, bool BLOCK>
cudaError_t launch_t(const hdiv_ctx* h, const double* x, double* y, const int* skip,
                     cudaStream_t s) {
  constexpr int NT = 256;
  using G = Geo<P, TX, TY, TZ>;
  AffArgs a;
  a.x = x; a.y = y; a.coef = h->d_coef;
  for (int d = 0; d < 3; ++d) { a.NL[d] = h->NL[d]; a.n[d] = h->n[d]; a.off[d] = h->off[d]; }
  a.nrt = h->nrt;
  a.ntile[0] = (int)((h->NL[0] + TX - 1) / TX);
  a.ntile[1] = (int)((h->NL[1] + TY - 1) / TY);
  a.ntile[2] = (int)((h->NL[2] + TZ - 1) / TZ);
  a.has_z = h->has_z ? 1 : 0;
  a.skip = skip;
  const size_t smem = G::smem_doubles(BLOCK) * sizeof(double);
  auto kern = affine_apply_kernel<P, TX, TY, TZ, NT, BLOCK>;
  static bool attr_done = false;   // per instantiation
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  const long long nblk = (long long)a.ntile[0] * a.ntile[1] * a.ntile[2];
  kern<<<(unsigned)nblk, NT, smem, s>>>(a, h->taff);
  return cudaGetLastError();
}

template <bool BLOCK>
cudaError_t dispatch(const hdiv_ctx* h, const double* x, double* y, const int* k,
                     cudaStream_t s) {
  switch (h->p) {
    case 1: return launch_t<1, 8, 8, 8, BLOCK>(h, x, y, k, s);
    case 2: return launch_t<2, 8, 8, 4, BLOCK>(h, x, y, k, s);
    case 3: return launch_t<3, 4, 4, 4, BLOCK>(h, x, y, k, s);
    case 4: return launch_t<4, 4, 4, 2, BLOCK>(h, x, y, k, s);
    case 5: return launch_t<5, 4, 2, 2, BLOCK>(h, x, y, k, s);
    case 6: return launch_t<6, 2, 2, 2, BLOCK>(h, x, y, k, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_affine_apply(const hdiv_ctx* h, const double* x, double* y, int mode,
                                const int* skip, cudaStream_t s) {
  if (mode == MODE_BLOCK) return dispatch<true>(h, x, y, skip, s);
  return dispatch<false>(h, x, y, skip, s);
}

}  // namespace hdiv
