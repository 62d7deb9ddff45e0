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
//    shared memory) and written once (streaming stores) — no atomics, no zero fill;
//  * a face plane shared by two tiles is OWNED by the tile on its + side; that tile
//    recomputes the - side neighbour element's contribution from a one-element halo of the
//    single component involved (1/T of one component; neighbours' reads hit L2);
//  * per component: one register-blocked pass applies M_h (x) M_h across the two histopolation
//    directions (P x P block per thread), one line pass applies c_e M_l along the component
//    direction element by element with the shared-plane sum carried in a register, and D^T q~
//    is added in the coalesced copy-out;
//  * tile geometry is compile-time (loops unrolled, constant divisors); partial tiles at the
//    domain edge are handled with predicates; every smem extent is padded to an odd number of
//    doubles so that all lane strides are odd -> bank-conflict free;
//  * D u and -Z q~ accumulate in registers per owned cell; stored coalesced (a tile row of
//    L2 DOFs is contiguous in HBM).
#include <cuda_runtime.h>

#include <cstdlib>

#include "affine_layouts.h"
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
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

constexpr int odd_up(int v) { return (v % 2) ? v : v + 1; }
constexpr int cmax(int a, int b) { return a > b ? a : b; }
// x component: 1 = store the owned planes straight from the line pass (per-lane runs along x;
// full sectors merge in L2), 0 = write back to smem + coalesced copy-out
#ifndef HDIV_X_DIRECT
#define HDIV_X_DIRECT 1
#endif
constexpr bool kXDirect = HDIV_X_DIRECT;

// smem box of component AX: extent (T_AX+1)P+1 along AX (position 0 <-> global plane
// (e0_AX - 1) P), T P along the others.  Strides: the generated per-tile layout
// (affine_layouts.h, fewest modelled bank-conflict wavefronts), else extents 0 and 1 padded odd.
template <int P, int TX, int TY, int TZ, int AX>
struct CG {
  static constexpr int LI = find_tile_layout(P, TX, TY, TZ);
  static constexpr int E0 = (AX == 0) ? (TX + 1) * P + 1 : TX * P;
  static constexpr int E1 = (AX == 1) ? (TY + 1) * P + 1 : TY * P;
  static constexpr int E2 = (AX == 2) ? (TZ + 1) * P + 1 : TZ * P;
  static constexpr int S1 = LI >= 0 ? kTileLayouts[LI].S[AX][0] : odd_up(E0);
  static constexpr int S2 = LI >= 0 ? kTileLayouts[LI].S[AX][1] : S1 * odd_up(E1);
  static_assert(S1 >= E0 && S2 >= S1 * E1, "component layout overlaps");
  // lane maps: M_l / halo lines and M_h (x) M_h positions padded to half-warps or packed
  static constexpr bool PADL = LI >= 0 ? kTileLayouts[LI].padL[AX] != 0 : true;
  static constexpr bool PADA = LI >= 0 ? kTileLayouts[LI].padA[AX] != 0 : true;
  static constexpr int SIZE = S2 * E2;
  static constexpr int EA = (AX == 0) ? E0 : (AX == 1) ? E1 : E2;   // extent along AX
  static constexpr int SA = (AX == 0) ? 1 : (AX == 1) ? S1 : S2;    // stride along AX
  // the two histopolation axes A1 < A2
  static constexpr int A1 = (AX == 0) ? 1 : 0;
  static constexpr int A2 = (AX == 2) ? 1 : 2;
  static constexpr int SA1 = (A1 == 0) ? 1 : S1;
  static constexpr int SA2 = (A2 == 1) ? S1 : S2;
  static constexpr int TA = (AX == 0) ? TX : (AX == 1) ? TY : TZ;
  static constexpr int TA1 = (A1 == 0) ? TX : TY;
  static constexpr int TA2 = (A2 == 1) ? TY : TZ;
};

template <int P, int TX, int TY, int TZ>
struct Geo {
  static constexpr int P3 = P * P * P;
  static constexpr int NE = TX * TY * TZ;
  static constexpr int NCELL = NE * P3;
  // cell tile (subcell-major, odd-padded): cell (X,Y,Z) at X + Q1 Y + Q2 Z
  static constexpr int CX = TX * P, CY = TY * P, CZ = TZ * P;
  static constexpr int LI = find_tile_layout(P, TX, TY, TZ);
  static constexpr int Q1 = LI >= 0 ? kTileLayouts[LI].Q[0] : odd_up(CX);
  static constexpr int Q2 = LI >= 0 ? kTileLayouts[LI].Q[1] : Q1 * odd_up(CY);
  static_assert(Q1 >= CX && Q2 >= Q1 * CY, "q tile layout overlaps");
  static constexpr int SQSIZE = Q2 * CZ;
  static constexpr int SU = cmax(cmax(CG<P, TX, TY, TZ, 0>::SIZE, CG<P, TX, TY, TZ, 1>::SIZE),
                                 cmax(CG<P, TX, TY, TZ, 2>::SIZE, SQSIZE));
  static constexpr int HQ0 = CY * CZ, HQ1 = CX * CZ, HQ2 = CX * CY;
  static constexpr int NCO = (TX + 1) * (TY + 1) * (TZ + 1);
  static constexpr size_t smem_doubles(bool block, bool db = true) {   // db: double buffer
    return (db ? 2 : 1) * (size_t)SU + (block ? (size_t)SQSIZE + HQ0 + HQ1 + HQ2 : 0) + 4 * NCO;
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
  // packed (the argument block keeps its round-1 size: ptxas allocated registers differently,
  // and the p=3/4 kernels ran 4-8 % slower, when two ints were added here):
  // bit 0 = (2,2) block nonzero, bits 1..6 = eliminated essential sides (NEXT-3),
  // bits 8.. = first z tile of this launch (z-chunked host pipeline)
  int flags;
  const int* skip;     // MINRES done flag (nullptr: never skip)
  __device__ __forceinline__ int has_z() const { return flags & 1; }
  __device__ __forceinline__ int ess() const { return (flags >> 1) & 63; }
  __device__ __forceinline__ int tz0() const { return flags >> 8; }
};

// z-tile range of the next halo-tile launch (host side, set by launch_affine_apply_range):
// tz1 < 0 = all tiles; tz_out != nullptr = only report the variant's TZ, launch nothing
struct TileRange {
  int tz0 = 0, tz1 = -1;
  int* tz_out = nullptr;
};
static thread_local TileRange g_range;

struct TileInfo {
  int e0[3];    // first element of the tile
  int m[3];     // valid elements per axis (<= T)
  int h[3];     // - side halo element present
  int last[3];  // tile touches the + domain boundary
};

// Row loops.  The box (i0 < L, i1 < R1, i2 < R2) is contiguous along i0 in both smem and HBM;
// warps take i2 planes round-robin, lanes run along rows (rows shorter than 16 are packed
// RPI per warp), and the row loop is unrolled with incremental addresses so each entry costs
// a predicate, an address add and the access.  act(global_ptr, smem_ptr) per valid entry;
// ok0(i0) / ok1(i1) / ok2(i2) are the per-axis validity predicates.
template <int NT, int L, int R1, int R2, int S1, int S2, class GT, class OK0, class OK1,
          class OK2, class ACT>
__device__ __forceinline__ void rows(GT* gbase, long long ext0, long long ext01, double* sbase,
                                     OK0 ok0, OK1 ok1, OK2 ok2, ACT act) {
  static_assert(L <= 32, "row longer than a warp");
  constexpr int LP = L <= 2 ? 2 : L <= 4 ? 4 : L <= 8 ? 8 : L <= 16 ? 16 : 32;
  constexpr int RPI = 32 / LP;
  constexpr int NJ = (R1 + RPI - 1) / RPI;
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = lane % LP, rs = lane / LP;
  if (c >= L || !ok0(c)) return;
  const long long gstep = RPI * ext0;
  for (int i2 = warp; i2 < R2; i2 += NW) {
    if (!ok2(i2)) continue;
    GT* g = gbase + (i2 * ext01 + rs * ext0 + c);
    double* s = sbase + (i2 * S2 + rs * S1 + c);
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const int i1 = j * RPI + rs;
      if (i1 < R1 && ok1(i1)) act(g, s + j * RPI * S1);
      g += gstep;
    }
  }
}

// X- and Y-lines of (M_h^-1)^{(x)2} on the q~ tile in one register-blocked pass: a thread owns
// the P x P (X, Y) block of one element column at one cell layer Z (lanes over Z first; the
// element columns of consecutive item groups in the order of the layout's zmap), reads it from
// src once, contracts along X then Y (the order of two separate line passes: same arithmetic)
// and writes it to dst once
template <int P, int TX, int TY, int TZ, int NT>
__device__ __forceinline__ void z_xy_block(const double* src, double* dst, const double (*Mi)[MAXP]) {
  using G = Geo<P, TX, TY, TZ>;
  constexpr int LI = find_tile_layout(P, TX, TY, TZ);
  constexpr int ZMAP = LI >= 0 ? kTileLayouts[LI].zmap : 0;
  constexpr int CZ = G::CZ;
  constexpr int NIT = CZ * TX * TY;
#pragma unroll 1
  for (int it = threadIdx.x; it < NIT; it += NT) {
    const int zc = it % CZ, b = it / CZ;
    const int by = b / TX, r = b % TX;
    const int bx = (ZMAP == 1 && TX % 2 == 0) ? (r / 2) + (r % 2) * (TX / 2) : r;
    const int o = bx * P + G::Q1 * (by * P) + G::Q2 * zc;
    double w[P][P];
#pragma unroll
    for (int k2 = 0; k2 < P; ++k2) {
      double v[P];
#pragma unroll
      for (int k1 = 0; k1 < P; ++k1) v[k1] = src[o + k1 + G::Q1 * k2];
#pragma unroll
      for (int i = 0; i < P; ++i) {
        double t = 0.0;
#pragma unroll
        for (int j = 0; j < P; ++j) t = fma(Mi[i][j], v[j], t);
        w[k2][i] = t;
      }
    }
#pragma unroll
    for (int k1 = 0; k1 < P; ++k1)
#pragma unroll
      for (int k2 = 0; k2 < P; ++k2) {
        double t = 0.0;
#pragma unroll
        for (int j = 0; j < P; ++j) t = fma(Mi[k2][j], w[j][k1], t);
        dst[o + k1 + G::Q1 * k2] = t;
      }
  }
}

// L2-cell ownership: thread t owns the cell columns (X, Y) = col % CX, col / CX for
// col = t + j NT (j < JC) and all Z of the tile -> acc[j * CZ + Z]; addresses are a per-column
// base plus compile-time offsets, and lanes run along X (conflict free).
template <int P, int TX, int TY, int TZ, int NT>
struct Own {
  using G = Geo<P, TX, TY, TZ>;
  static constexpr int NCOL = G::CX * G::CY;
  static constexpr int JC = (NCOL + NT - 1) / NT;
  static constexpr int NACC = JC * G::CZ;
};

// global tile origin of component AX (position 0 of its smem box) and its face-grid extents
template <int P, int AX>
struct CompAddr {
  long long ext0, ext01, gtile;
  __device__ __forceinline__ CompAddr(const AffArgs& a, const TileInfo& ti) {
    ext0 = a.n[0] + (AX == 0);
    const long long ext1 = a.n[1] + (AX == 1);
    ext01 = ext0 * ext1;
    long long gorg[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) gorg[d] = (long long)(ti.e0[d] - (d == AX ? 1 : 0)) * P;
    gtile = a.off[AX] + gorg[0] + ext0 * (gorg[1] + ext1 * gorg[2]);
  }
};

// issue the cp.async loads of component AX's tile (+ - halo) into `su` and commit a group
template <int P, int TX, int TY, int TZ, int NT, int AX>
__device__ __forceinline__ void load_component(const AffArgs& a, const TileInfo& ti, double* su) {
  using C = CG<P, TX, TY, TZ, AX>;
  const CompAddr<P, AX> ca(a, ti);
  const int lo_a = ti.h[AX] ? 0 : P;                  // first loaded position along AX
  const int hi_a = (ti.m[AX] + 1) * P;                // last valid position along AX
  const int hi0 = ti.m[0] * P, hi1 = ti.m[1] * P, hi2 = ti.m[2] * P;
  auto okd = [&](int d, int pos) {
    if (d == AX) return pos >= lo_a && pos <= hi_a;
    return pos < (d == 0 ? hi0 : d == 1 ? hi1 : hi2);
  };
  rows<NT, C::E0, C::E1, C::E2, C::S1, C::S2>(
      a.x + ca.gtile, ca.ext0, ca.ext01, su, [&](int i) { return okd(0, i); },
      [&](int i) { return okd(1, i); }, [&](int i) { return okd(2, i); },
      [&](const double* g, double* s) { cp_async8(s, g); });
  cp_async_commit();
}

// -------- one component phase (AX), data already in `su` ------------------------------------
template <int P, int TX, int TY, int TZ, int NT, int AX, bool BLOCK, bool XD = kXDirect,
          bool ESS = false, bool DOT = false>
__device__ __forceinline__ void component(const AffArgs& a, const TileInfo& ti,
                                          const TabAffine& tab, double* su, const double* sq,
                                          const double* hq, const double* sco, double* acc,
                                          double& dsum) {
  using C = CG<P, TX, TY, TZ, AX>;
  using G = Geo<P, TX, TY, TZ>;
  using O = Own<P, TX, TY, TZ, NT>;
  const int tid = threadIdx.x;
  const CompAddr<P, AX> ca(a, ti);
  const long long ext0 = ca.ext0, ext01 = ca.ext01, gtile = ca.gtile;
  const int hi0 = ti.m[0] * P, hi1 = ti.m[1] * P, hi2 = ti.m[2] * P;
  constexpr int EL1 = C::TA1 * P, EL2 = C::TA2 * P;

  // ---- NEXT-3: eliminated essential planes act as zero inputs (the tile's first plane when
  //      it starts at the domain's - side, its last when it ends at the + side) ----
  // (ESS instantiations only: the common path compiles exactly as without eliminated sides)
  const bool ess_lo = ESS && ((a.ess() >> (2 * AX)) & 1) && ti.e0[AX] == 0;
  const bool ess_hi = ESS && ((a.ess() >> (2 * AX + 1)) & 1) && ti.last[AX];
  if (ESS && (ess_lo || ess_hi)) {   // block-uniform
    for (int it = tid; it < EL1 * EL2; it += NT) {
      double* line = su + (it % EL1) * C::SA1 + (it / EL1) * C::SA2;
      if (ess_lo) line[P * C::SA] = 0.0;
      if (ess_hi) line[(ti.m[AX] + 1) * P * C::SA] = 0.0;
    }
    __syncthreads();
  }

  // ---- D u: this component's two faces of every owned cell ----
  if constexpr (BLOCK) {
#pragma unroll
    for (int j = 0; j < O::JC; ++j) {
      const int col = tid + j * NT;
      if (col < O::NCOL) {
        int pos[3] = {col % G::CX, col / G::CX, 0};
        pos[AX] += P;
        const double* s = su + pos[0] + C::S1 * pos[1] + C::S2 * pos[2];
        if constexpr (AX == 2) {   // walk up the column: each z face read once
          double lo = s[0];
#pragma unroll
          for (int z = 0; z < G::CZ; ++z) {
            const double hi = s[(z + 1) * C::S2];
            acc[j * G::CZ + z] += hi - lo;
            lo = hi;
          }
        } else {
#pragma unroll
          for (int z = 0; z < G::CZ; ++z)
            acc[j * G::CZ + z] += s[z * C::S2 + C::SA] - s[z * C::S2];
        }
      }
    }
    __syncthreads();
  }

  // ---- halo element: only its contribution to the shared plane is needed, and by
  //      linearity c_h sum_j M_l[P][j] (M_h (x) M_h) u_j = c_h (M_h (x) M_h) sum_j M_l[P][j] u_j,
  //      so the raw halo planes are combined first into position P-1 (one plane to transform)
  constexpr int EL1P = C::PADL ? (EL1 + 15) / 16 * 16 : EL1;   // half-warp aligned lane rows
  const int m_a = ti.m[AX], h_a = ti.h[AX];
  if (h_a) {
#pragma unroll 1
    for (int it = tid; it < EL1P * EL2; it += NT) {
      const int l1 = it % EL1P, l2 = it / EL1P;
      if (l1 >= EL1) continue;
      double* line = su + l1 * C::SA1 + l2 * C::SA2;
      double s = 0.0;
#pragma unroll
      for (int j = 0; j <= P; ++j) s = fma(tab.Ml[P][j], line[j * C::SA], s);
      line[(P - 1) * C::SA] = s;
    }
    __syncthreads();
  }

  // ---- M_h (x) M_h over the two histopolation axes: one P x P block per thread, positions
  //      P-1 (combined halo) .. (T+1)P; lanes run along AX (odd stride), the position range
  //      padded to a multiple of 16 so a half-warp never straddles two blocks ----
  constexpr int EAH = C::EA - (P - 1);
  constexpr int EAP = C::PADA ? (EAH + 15) / 16 * 16 : EAH;
  constexpr int NH = EAP * C::TA1 * C::TA2;
#pragma unroll 2
  for (int it = tid; it < NH; it += NT) {
    const int pa = it % EAP + (P - 1), b1 = (it / EAP) % C::TA1, b2 = it / (EAP * C::TA1);
    if (pa >= C::EA) continue;
    double* base = su + pa * C::SA + b1 * P * C::SA1 + b2 * P * C::SA2;
    // row by row: only one input row and the P x P intermediate are live (register pressure)
    double w[P][P];
#pragma unroll
    for (int k2 = 0; k2 < P; ++k2) {
      double v[P];
#pragma unroll
      for (int k1 = 0; k1 < P; ++k1) v[k1] = base[k1 * C::SA1 + k2 * C::SA2];
#pragma unroll
      for (int k1 = 0; k1 < P; ++k1) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < P; ++j) s = fma(tab.Mh[k1][j], v[j], s);
        w[k2][k1] = s;
      }
    }
#pragma unroll
    for (int k1 = 0; k1 < P; ++k1)
#pragma unroll
      for (int k2 = 0; k2 < P; ++k2) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < P; ++j) s = fma(tab.Mh[k2][j], w[j][k1], s);
        base[k1 * C::SA1 + k2 * C::SA2] = s;
      }
  }
  __syncthreads();

  // ---- c_e M_l along AX element by element (shared-plane sum carried in a register),
  //      + D^T q~ ; y/z: owned planes stored straight to HBM (lanes run along x: coalesced),
  //      x: written back to smem for a coalesced copy-out ----
  constexpr int NL = EL1P * EL2;
  constexpr int QA1 = (C::A1 == 0) ? 1 : G::Q1;
  constexpr int QA2 = (C::A2 == 1) ? G::Q1 : G::Q2;
  constexpr int QS = (AX == 0) ? 1 : (AX == 1) ? G::Q1 : G::Q2;
  const long long gs1 = (C::A1 == 0) ? 1 : ext0;        // HBM strides along A1, A2, AX
  const long long gs2 = (C::A2 == 1) ? ext0 : ext01;
  const long long gsa = (AX == 0) ? 1 : (AX == 1) ? ext0 : ext01;
  const int hiA1 = (C::A1 == 0) ? hi0 : hi1, hiA2 = (C::A2 == 1) ? hi1 : hi2;
  double* yt = a.y + gtile;
#pragma unroll 1
  for (int it = tid; it < NL; it += NT) {
    const int l1 = it % EL1P, l2 = it / EL1P;
    if (l1 >= EL1) continue;
    const bool line_ok = l1 < hiA1 && l2 < hiA2;
    if ((AX != 0 || XD) && !line_ok) continue;
    double* line = su + l1 * C::SA1 + l2 * C::SA2;
    double* gl = yt + (l1 * gs1 + l2 * gs2);
    int ec[3];
    ec[C::A1] = l1 / P;
    ec[C::A2] = l2 / P;
    ec[AX] = 0;
    const double* cbase =
        sco + 4 * (((ec[2] + 1) * (TY + 1) + (ec[1] + 1)) * (TX + 1) + (ec[0] + 1)) + AX;
    constexpr int CSTEP = 4 * ((AX == 0) ? 1 : (AX == 1) ? (TX + 1) : (TX + 1) * (TY + 1));
    const double* ql = sq + l1 * QA1 + l2 * QA2;
    double carry = 0.0, qprev = 0.0;
    if (h_a) {   // transformed combined halo plane (position P-1)
      carry = cbase[-CSTEP] * line[(P - 1) * C::SA];
      if (BLOCK) qprev = hq[l2 * EL1 + l1];
    }
#pragma unroll
    for (int et = 0; et < C::TA; ++et) {
      if (et < m_a) {
        double* eb = line + (et + 1) * P * C::SA;
        double v[P + 1];
#pragma unroll
        for (int i = 0; i <= P; ++i) v[i] = eb[i * C::SA];
        const double c = cbase[et * CSTEP];
#pragma unroll
        for (int i = 0; i < P; ++i) {
          double s = 0.0;
#pragma unroll
          for (int j = 0; j <= P; ++j) s = fma(tab.Ml[i][j], v[j], s);
          double o = (i == 0) ? fma(c, s, carry) : c * s;
          if constexpr (BLOCK) {   // (D^T q)_face = q(- side cell) - q(+ side cell)
            const double qc = ql[(et * P + i) * QS];
            o += qprev - qc;
            qprev = qc;
          }
          if (ESS && i == 0 && et == 0 && ess_lo)   // identity row of the eliminated plane
            o = a.x[gtile + (l1 * gs1 + l2 * gs2) + P * gsa];
          if (AX == 0 && !XD) eb[i * C::SA] = o;
          else {
            __stcs(gl + ((et + 1) * P + i) * gsa, o);
            if constexpr (DOT) dsum = fma(o, __ldg(a.x + (gl - a.y) + ((et + 1) * P + i) * gsa), dsum);
          }
        }
        double s = 0.0;
#pragma unroll
        for (int j = 0; j <= P; ++j) s = fma(tab.Ml[P][j], v[j], s);
        carry = c * s;
      }
    }
    if (ti.last[AX]) {
      const double o = (ESS && ess_hi) ? a.x[gtile + (l1 * gs1 + l2 * gs2) + (m_a + 1) * P * gsa]
                              : carry + (BLOCK ? qprev : 0.0);
      if (AX == 0 && !XD) line[(m_a + 1) * P * C::SA] = o;
      else {
        __stcs(gl + (m_a + 1) * P * gsa, o);
        if constexpr (DOT) dsum = fma(o, __ldg(a.x + (gl - a.y) + (m_a + 1) * P * gsa), dsum);
      }
    }
  }
  __syncthreads();

  if constexpr (AX == 0 && !XD) {
    // ---- copy-out of the owned x planes (coalesced, streaming) ----
    constexpr int NO0 = TX * P + 1;
    const int own_hi = m_a * P + (ti.last[0] ? 1 : 0);   // exclusive, relative to position P
    rows<NT, NO0, C::E1, C::E2, C::S1, C::S2>(
        yt + P, ext0, ext01, su + P, [&](int i) { return i < own_hi; },
        [&](int i) { return i < hi1; }, [&](int i) { return i < hi2; },
        [&](double* g, const double* s) {
          __stcs(g, *s);
          if constexpr (DOT) dsum = fma(*s, __ldg(a.x + (g - a.y)), dsum);
        });
    __syncthreads();
  }
}

// DOT: the MINRES partial <y, x> of this tile's owned outputs -> dpart[blockIdx.x] (the separate
// dot pass over both vectors is saved; x is re-read where each output is stored: L1/L2 hits)
template <int P, int TX, int TY, int TZ, int NT, bool BLOCK, bool DB, int MINB, bool XD,
          bool ESS = false, bool DOT = false>
__global__ void __launch_bounds__(NT, MINB)
affine_apply_kernel(const AffArgs a, const __grid_constant__ TabAffine tab, double* __restrict__ dpart) {
  using G = Geo<P, TX, TY, TZ>;
  using O = Own<P, TX, TY, TZ, NT>;
  constexpr int P3 = G::P3;
  if (a.skip && *a.skip) return;
  extern __shared__ double smem[];
  double* bufA = smem;                                // component buffers (DB: double buffered;
  double* bufB = DB ? smem + G::SU : smem;            // else one buffer, more CTAs per SM)
  double* sq = bufB + G::SU;                          // q~ tile, subcell-major
  double* hq0 = sq + (BLOCK ? G::SQSIZE : 0);         // halo q~ for owned -x planes [K][J]
  double* hq1 = hq0 + (BLOCK ? G::HQ0 : 0);           // [K][I]
  double* hq2 = hq1 + (BLOCK ? G::HQ1 : 0);           // [J][I]
  double* sco = hq2 + (BLOCK ? G::HQ2 : 0);           // coefficients [(TZ+1)][(TY+1)][(TX+1)][4]

  const int tid = threadIdx.x;
  TileInfo ti;
  {
    int t = blockIdx.x;
    const int tx = t % a.ntile[0];
    t /= a.ntile[0];
    const int ty = t % a.ntile[1];
    const int tz = t / a.ntile[1] + a.tz0();
    const int T3[3] = {TX, TY, TZ};
    const int tt[3] = {tx, ty, tz};
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      ti.e0[d] = tt[d] * T3[d];
      ti.m[d] = (int)min((long long)T3[d], a.NL[d] - ti.e0[d]);
      ti.h[d] = ti.e0[d] > 0;
      ti.last[d] = (ti.e0[d] + ti.m[d] == a.NL[d]);
    }
  }
  const long long NLx = a.NL[0], NLy = a.NL[1];
  const double* q = a.x + a.nrt;
  auto elem_ok = [&](int ex, int ey, int ez) {
    return ex < ti.m[0] && ey < ti.m[1] && ez < ti.m[2];
  };
  auto gelem = [&](int ex, int ey, int ez) -> long long {
    return ((long long)(ti.e0[2] + ez) * NLy + (ti.e0[1] + ey)) * NLx + (ti.e0[0] + ex);
  };

  // ---- group 0: coefficients of the tile and its - halo, q~ tile, halo q~ ----
  for (int l = tid; l < 4 * G::NCO; l += NT) {   // lanes over (slot, k): contiguous runs
    const int i = l >> 2, k = l & 3;
    const int ix = i % (TX + 1), iy = (i / (TX + 1)) % (TY + 1), iz = i / ((TX + 1) * (TY + 1));
    const int ex = ti.e0[0] - 1 + ix, ey = ti.e0[1] - 1 + iy, ez = ti.e0[2] - 1 + iz;
    if (ex >= 0 && ey >= 0 && ez >= 0 && ix <= ti.m[0] && iy <= ti.m[1] && iz <= ti.m[2])
      cp_async8(sco + l, a.coef + 4 * (((long long)ez * NLy + ey) * NLx + ex) + k);
  }
  if constexpr (BLOCK) {
    // q~ tile, subcell-major, loaded per owned column (X, Y): lanes run along X (conflict-free
    // smem writes; HBM runs of P doubles per element)
#pragma unroll
    for (int j = 0; j < O::JC; ++j) {
      const int col = tid + j * NT;
      if (col < O::NCOL) {
        const int X = col % G::CX, Y = col / G::CX;
        if (X < ti.m[0] * P && Y < ti.m[1] * P) {
          const double* qc = q + gelem(X / P, Y / P, 0) * P3 + (X % P) + P * (Y % P);
          double* sc = sq + X + G::Q1 * Y;
#pragma unroll
          for (int z = 0; z < G::CZ; ++z)
            if (z < ti.m[2] * P)
              cp_async8(sc + z * G::Q2, qc + (long long)(z / P) * NLx * NLy * P3 + P * P * (z % P));
        }
      }
    }
    // halo q~ of the - neighbour's adjacent cell layer (for D^T at the owned - planes)
    if (ti.h[0])
      for (int i = tid; i < G::HQ0; i += NT) {
        const int J = i % G::CY, K = i / G::CY;
        if (J < ti.m[1] * P && K < ti.m[2] * P) {
          const long long ge = ((long long)(ti.e0[2] + K / P) * NLy + (ti.e0[1] + J / P)) * NLx +
                               (ti.e0[0] - 1);
          cp_async8(hq0 + i, q + ge * P3 + (P - 1) + P * ((J % P) + P * (K % P)));
        }
      }
    if (ti.h[1])
      for (int i = tid; i < G::HQ1; i += NT) {
        const int I = i % G::CX, K = i / G::CX;
        if (I < ti.m[0] * P && K < ti.m[2] * P) {
          const long long ge = ((long long)(ti.e0[2] + K / P) * NLy + (ti.e0[1] - 1)) * NLx +
                               (ti.e0[0] + I / P);
          cp_async8(hq1 + i, q + ge * P3 + (I % P) + P * ((P - 1) + P * (K % P)));
        }
      }
    if (ti.h[2])
      for (int i = tid; i < G::HQ2; i += NT) {
        const int I = i % G::CX, J = i / G::CX;
        if (I < ti.m[0] * P && J < ti.m[1] * P) {
          const long long ge = ((long long)(ti.e0[2] - 1) * NLy + (ti.e0[1] + J / P)) * NLx +
                               (ti.e0[0] + I / P);
          cp_async8(hq2 + i, q + ge * P3 + (I % P) + P * ((J % P) + P * (P - 1)));
        }
      }
  }
  cp_async_commit();
  // ---- group 1 (DB): x component -> A, overlapping the Z passes (scratch B) ----
  if constexpr (DB) load_component<P, TX, TY, TZ, NT, 0>(a, ti, bufA);

  double acc[O::NACC];
#pragma unroll
  for (int k = 0; k < O::NACC; ++k) acc[k] = 0.0;
  double dsum = 0.0;

  if constexpr (DB) cp_async_wait_group<1>();
  else cp_async_wait_group<0>();
  __syncthreads();
  if constexpr (BLOCK) {
    if (a.has_z()) {
      // -Z q~ = -z_e (Mh^-1)^{(x)3} q~_e in B (subcell-major like sq):
      // X-lines (lanes over Y, odd stride Q1; sq -> B), then Y- and Z-lines (lanes over X)
      z_xy_block<P, TX, TY, TZ, NT>(sq, bufB, tab.Mhinv);
      __syncthreads();
      // Z-lines in registers: every thread owns whole z-columns of cells
#pragma unroll
      for (int j = 0; j < O::JC; ++j) {
        const int col = tid + j * NT;
        if (col < O::NCOL) {
          const int X = col % G::CX, Y = col / G::CX;
          const double* sz = sco + 4 * (((Y / P) + 1) * (TX + 1) + (X / P) + 1) + 3;
          const double* s = bufB + X + G::Q1 * Y;
#pragma unroll
          for (int zb = 0; zb < TZ; ++zb) {
            double v[P];
#pragma unroll
            for (int k = 0; k < P; ++k) v[k] = s[(zb * P + k) * G::Q2];
            const double ze = sz[4 * (TX + 1) * (TY + 1) * (zb + 1)];
#pragma unroll
            for (int i = 0; i < P; ++i) {
              double t = 0.0;
#pragma unroll
              for (int k = 0; k < P; ++k) t = fma(tab.Mhinv[i][k], v[k], t);
              acc[j * G::CZ + zb * P + i] = -ze * t;
            }
          }
        }
      }
      __syncthreads();
    }
  }
  if constexpr (DB) {
    // ---- group 2: y component -> B ; compute x from A ----
    load_component<P, TX, TY, TZ, NT, 1>(a, ti, bufB);
    cp_async_wait_group<1>();
    __syncthreads();
    component<P, TX, TY, TZ, NT, 0, BLOCK, XD, ESS, DOT>(a, ti, tab, bufA, sq, hq0, sco, acc, dsum);
    // ---- group 3: z component -> A ; compute y from B ----
    load_component<P, TX, TY, TZ, NT, 2>(a, ti, bufA);
    cp_async_wait_group<1>();
    __syncthreads();
    component<P, TX, TY, TZ, NT, 1, BLOCK, XD, ESS, DOT>(a, ti, tab, bufB, sq, hq1, sco, acc, dsum);
    cp_async_wait_group<0>();
    __syncthreads();
    component<P, TX, TY, TZ, NT, 2, BLOCK, XD, ESS, DOT>(a, ti, tab, bufA, sq, hq2, sco, acc, dsum);
  } else {
    load_component<P, TX, TY, TZ, NT, 0>(a, ti, bufA);
    cp_async_wait_group<0>();
    __syncthreads();
    component<P, TX, TY, TZ, NT, 0, BLOCK, XD, ESS, DOT>(a, ti, tab, bufA, sq, hq0, sco, acc, dsum);
    load_component<P, TX, TY, TZ, NT, 1>(a, ti, bufA);
    cp_async_wait_group<0>();
    __syncthreads();
    component<P, TX, TY, TZ, NT, 1, BLOCK, XD, ESS, DOT>(a, ti, tab, bufA, sq, hq1, sco, acc, dsum);
    load_component<P, TX, TY, TZ, NT, 2>(a, ti, bufA);
    cp_async_wait_group<0>();
    __syncthreads();
    component<P, TX, TY, TZ, NT, 2, BLOCK, XD, ESS, DOT>(a, ti, tab, bufA, sq, hq2, sco, acc, dsum);
  }

  if constexpr (BLOCK) {
    // y_q straight from the accumulators: per owned column, runs of P doubles per element
    double* yq = a.y + a.nrt;
#pragma unroll
    for (int j = 0; j < O::JC; ++j) {
      const int col = tid + j * NT;
      if (col < O::NCOL) {
        const int X = col % G::CX, Y = col / G::CX;
        if (X < ti.m[0] * P && Y < ti.m[1] * P) {
          double* yc = yq + gelem(X / P, Y / P, 0) * P3 + (X % P) + P * (Y % P);
#pragma unroll
          for (int z = 0; z < G::CZ; ++z)
            if (z < ti.m[2] * P) {
              const long long off = (long long)(z / P) * NLx * NLy * P3 + P * P * (z % P);
              __stcs(yc + off, acc[j * G::CZ + z]);
              if constexpr (DOT) dsum = fma(acc[j * G::CZ + z], __ldg(a.x + (yc - a.y) + off), dsum);
            }
        }
      }
    }
  }
  if constexpr (DOT) {   // fixed-order block sum -> this tile's partial
    __shared__ double red[NT / 32];
    for (int o = 16; o > 0; o >>= 1) dsum += __shfl_down_sync(0xffffffffu, dsum, o);
    if ((tid & 31) == 0) red[tid >> 5] = dsum;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < NT / 32; ++w) t += red[w];
      dpart[blockIdx.x] = t;
    }
  }
}

template <int P, int TX, int TY, int TZ, int NT, bool BLOCK, bool DB = true, int MINB = 0, bool XD = kXDirect,
          bool ESS = false, bool DOT = false>
cudaError_t launch_t(const hdiv_ctx* h, const double* x, double* y, const int* skip,
                     cudaStream_t s, double* dpart = nullptr) {
  using G = Geo<P, TX, TY, TZ>;
  AffArgs a;
  a.x = x; a.y = y; a.coef = h->d_coef;
  for (int d = 0; d < 3; ++d) { a.NL[d] = h->NL[d]; a.n[d] = h->n[d]; a.off[d] = h->off[d]; }
  a.nrt = h->nrt;
  a.ntile[0] = (int)((h->NL[0] + TX - 1) / TX);
  a.ntile[1] = (int)((h->NL[1] + TY - 1) / TY);
  a.ntile[2] = (int)((h->NL[2] + TZ - 1) / TZ);
  a.flags = (h->has_z ? 1 : 0) | (h->ess << 1);
  a.skip = skip;
  if (g_range.tz_out) {   // query: the variant's tile depth along z
    *g_range.tz_out = TZ;
    return cudaSuccess;
  }
  const int tz1 = (g_range.tz1 < 0) ? a.ntile[2] : min(g_range.tz1, a.ntile[2]);
  const int tz0 = g_range.tz0;
  a.flags |= tz0 << 8;
  if (tz1 <= tz0) return cudaSuccess;
  const size_t smem = G::smem_doubles(BLOCK, DB) * sizeof(double);
  auto kern = affine_apply_kernel<P, TX, TY, TZ, NT, BLOCK, DB, MINB, XD, ESS, DOT>;
  static bool attr_done = false;   // per instantiation
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  const long long nblk = (long long)a.ntile[0] * a.ntile[1] * (tz1 - tz0);
  count_op();
  kern<<<(unsigned)nblk, NT, smem, s>>>(a, h->taff, dpart);
  return cudaGetLastError();
}

// one production tile per order (r01 sweeps, profiles/r01_variant_sweep_v*.txt): TXxTYxTZ
// elements, NT threads, DB = double-buffered component boxes (p <= 2; single-buffered tiles
// give more CTAs per SM at p >= 3), MINB = __launch_bounds__ min blocks (p = 4: 7 -> 72 registers,
// 7 CTAs per SM, the shared-memory limit; 2.30 -> 2.26 ms, profiles/r02_box_experiments_late.txt),
// XD = x planes stored
// straight from the line pass (else written back and copied out coalesced, p = 5, 6).
// Eliminated essential sides use an instantiation of their own (ESS).
template <bool BLOCK, int P, int TX, int TY, int TZ, int NT, bool DB, int MINB, bool XD>
cudaError_t launch_tile(const hdiv_ctx* h, const double* x, double* y, const int* k,
                        cudaStream_t s, double* dpart) {
  if (dpart) {   // block apply with the fused MINRES partial <y, x> (whole grid, one launch)
    if constexpr (BLOCK) {
      if (h->ess) return launch_t<P, TX, TY, TZ, NT, BLOCK, DB, MINB, XD, true, true>(h, x, y, k, s, dpart);
      return launch_t<P, TX, TY, TZ, NT, BLOCK, DB, MINB, XD, false, true>(h, x, y, k, s, dpart);
    }
    return cudaErrorInvalidValue;
  }
  if (h->ess) return launch_t<P, TX, TY, TZ, NT, BLOCK, DB, MINB, XD, true>(h, x, y, k, s);
  return launch_t<P, TX, TY, TZ, NT, BLOCK, DB, MINB, XD, false>(h, x, y, k, s);
}

// tiles of h's production tile shape (the DOT partials: one per tile)
template <int TX, int TY, int TZ>
long long ntiles_of(const hdiv_ctx* h) {
  return ((h->NL[0] + TX - 1) / TX) * ((h->NL[1] + TY - 1) / TY) * ((h->NL[2] + TZ - 1) / TZ);
}

template <bool BLOCK>
cudaError_t dispatch(const hdiv_ctx* h, const double* x, double* y, const int* k,
                     cudaStream_t s, double* dpart = nullptr) {
  switch (h->p) {
    case 1: return launch_tile<BLOCK, 1, 8, 8, 4, 128, true, 0, kXDirect>(h, x, y, k, s, dpart);
    case 2: return launch_tile<BLOCK, 2, 8, 4, 4, 128, true, 0, kXDirect>(h, x, y, k, s, dpart);
    case 3: return launch_tile<BLOCK, 3, 4, 4, 2, 160, false, 0, kXDirect>(h, x, y, k, s, dpart);
    case 4: return launch_tile<BLOCK, 4, 4, 2, 2, 128, false, 7, kXDirect>(h, x, y, k, s, dpart);
    case 5: return launch_tile<BLOCK, 5, 3, 2, 2, 160, false, 0, false>(h, x, y, k, s, dpart);
    case 6: return launch_tile<BLOCK, 6, 3, 2, 2, 224, false, 2, false>(h, x, y, k, s, dpart);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

// the block apply with the fused partial <y, x>: one partial per tile into dpart (the caller
// sums affine_num_tiles(h) of them); single launch over all tiles
cudaError_t launch_affine_apply_dot(const hdiv_ctx* h, const double* x, double* y, const int* skip,
                                    double* dpart, cudaStream_t s) {
  return dispatch<true>(h, x, y, skip, s, dpart);
}

long long affine_num_tiles(const hdiv_ctx* h) {
  switch (h->p) {
    case 1: return ntiles_of<8, 8, 4>(h);
    case 2: return ntiles_of<8, 4, 4>(h);
    case 3: return ntiles_of<4, 4, 2>(h);
    case 4: return ntiles_of<4, 2, 2>(h);
    default: return ntiles_of<3, 2, 2>(h);
  }
}

cudaError_t launch_affine_apply(const hdiv_ctx* h, const double* x, double* y, int mode,
                                const int* skip, cudaStream_t s) {
  if (mode == MODE_BLOCK) return dispatch<true>(h, x, y, skip, s);
  return dispatch<false>(h, x, y, skip, s);
}

// the block apply restricted to the halo tiles with z-tile index in [tz0, tz1) (the z-chunked
// host pipeline of hdiv_apply_block_host); tz_out != nullptr: report the tile depth only
cudaError_t launch_affine_apply_range(const hdiv_ctx* h, const double* x, double* y, int tz0,
                                      int tz1, int* tz_out, cudaStream_t s, const int* skip) {
  g_range.tz0 = tz0;
  g_range.tz1 = tz1;
  g_range.tz_out = tz_out;
  cudaError_t e = dispatch<true>(h, x, y, skip, s);
  g_range = TileRange();
  return e;
}

}  // namespace hdiv
