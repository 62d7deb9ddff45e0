// tables.cpp — 1D node sets and the interpolation-histopolation tables (host, once per setup).
//
// P:178  GLL subcell vertices; P:181-182 RT/L2 DOFs via 1D interpolation / histopolation.
// Construction (independent of the oracle's):
//   GLL nodes  = roots of P_{p+1}(t) - P_{p-1}(t)  (= c (1-t^2) P_p'(t)), Newton, derivative
//                (2p+1) P_p(t).
//   GL rule    = Newton on P_Q, w = 2 / ((1-t^2) P_Q'(t)^2), mapped to [0,1].
//   l_i        = barycentric Lagrange on the GLL nodes.
//   h_j        = -sum_{i<=j} l_i'   (integral of l_i' over subinterval m is d_{i,m+1}-d_{i,m},
//                so these h_j have unit subinterval integrals: the histopolation DOFs).
#include <cmath>

#include "internal.h"

namespace hdiv {

static void legendre(int n, double t, double* P, double* dP) {
  double p0 = 1.0, p1 = t;
  if (n == 0) { *P = 1.0; *dP = 0.0; return; }
  for (int k = 2; k <= n; ++k) {
    double p2 = ((2.0 * k - 1.0) * t * p1 - (k - 1.0) * p0) / k;
    p0 = p1; p1 = p2;
  }
  *P = p1;
  // P_n' = n (t P_n - P_{n-1}) / (t^2 - 1), endpoints closed form
  if (std::fabs(std::fabs(t) - 1.0) < 1e-300)
    *dP = (t > 0 ? 1.0 : ((n % 2) ? 1.0 : -1.0)) * 0.5 * n * (n + 1);
  else
    *dP = n * (t * p1 - p0) / (t * t - 1.0);
}

static bool gll(int p, double* x) {
  // t-nodes in [-1,1] ascending
  std::vector<double> t(p + 1);
  for (int k = 0; k <= p; ++k) t[k] = -std::cos(M_PI * k / p);
  for (int k = 1; k < p; ++k) {
    double tk = t[k];
    for (int it = 0; it < 100; ++it) {
      double a, da, b, db, c, dc;
      legendre(p + 1, tk, &a, &da);
      legendre(p - 1, tk, &b, &db);
      legendre(p, tk, &c, &dc);
      double f = a - b, fp = (2.0 * p + 1.0) * c;
      double d = f / fp;
      tk -= d;
      if (std::fabs(d) < 1e-17) break;
    }
    t[k] = tk;
  }
  t[0] = -1.0; t[p] = 1.0;
  for (int k = 0; k <= p; ++k) x[k] = 0.5 * (t[k] + 1.0);
  x[0] = 0.0; x[p] = 1.0;
  for (int k = 0; k < p; ++k) if (!(x[k] < x[k + 1])) return false;
  return true;
}

static void gauss(int Q, double* x, double* w) {
  for (int k = 0; k < Q; ++k) {
    double tk = -std::cos(M_PI * (k + 0.75) / (Q + 0.5));
    double P = 0, dP = 1;
    for (int it = 0; it < 100; ++it) {
      legendre(Q, tk, &P, &dP);
      double d = P / dP;
      tk -= d;
      if (std::fabs(d) < 1e-17) break;
    }
    legendre(Q, tk, &P, &dP);
    x[k] = 0.5 * (tk + 1.0);
    w[k] = 1.0 / ((1.0 - tk * tk) * dP * dP);   // (2/((1-t^2)P'^2)) / 2
  }
}

// l_i(x) and l_i'(x) on nodes xi[0..n-1] (barycentric form)
static void lagrange(int n, const double* xi, double x, double* L, double* dL) {
  double lam[MAXP + 1];
  for (int i = 0; i < n; ++i) {
    double d = 1.0;
    for (int m = 0; m < n; ++m) if (m != i) d *= (xi[i] - xi[m]);
    lam[i] = 1.0 / d;
  }
  int hit = -1;
  for (int i = 0; i < n; ++i) if (x == xi[i]) hit = i;
  if (hit < 0) {
    double ell = 1.0, s = 0.0;
    for (int m = 0; m < n; ++m) { ell *= (x - xi[m]); s += 1.0 / (x - xi[m]); }
    for (int i = 0; i < n; ++i) {
      L[i] = ell * lam[i] / (x - xi[i]);
      dL[i] = L[i] * (s - 1.0 / (x - xi[i]));
    }
  } else {   // differentiation-matrix row at a node
    for (int i = 0; i < n; ++i) L[i] = (i == hit) ? 1.0 : 0.0;
    double diag = 0.0;
    for (int i = 0; i < n; ++i) {
      if (i == hit) continue;
      dL[i] = (lam[i] / lam[hit]) / (xi[hit] - xi[i]);
      diag -= dL[i];
    }
    dL[hit] = diag;
  }
}

static bool invert_spd(int n, const double* A, double* Ainv) {
  // Gauss-Jordan with partial pivoting (n <= 6)
  double M[MAXP][2 * MAXP];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < 2 * n; ++j) M[i][j] = (j < n) ? A[i * MAXP + j] : (j - n == i ? 1.0 : 0.0);
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int r = c + 1; r < n; ++r) if (std::fabs(M[r][c]) > std::fabs(M[piv][c])) piv = r;
    if (M[piv][c] == 0.0) return false;
    if (piv != c) for (int j = 0; j < 2 * n; ++j) std::swap(M[c][j], M[piv][j]);
    double d = M[c][c];
    for (int j = 0; j < 2 * n; ++j) M[c][j] /= d;
    for (int r = 0; r < n; ++r) {
      if (r == c) continue;
      double f = M[r][c];
      if (f != 0.0) for (int j = 0; j < 2 * n; ++j) M[r][j] -= f * M[c][j];
    }
  }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) Ainv[i * MAXP + j] = M[i][j + n];
  return true;
}

bool build_tables(int p, int Q, Tab1D* t, std::string* err) {
  *t = Tab1D{};
  t->p = p; t->Q = Q;
  if (p < 1 || p > MAXP || Q < 1 || Q > MAXQ) { *err = "order out of range"; return false; }
  double xi[MAXP + 1];
  if (!gll(p, xi)) { *err = "GLL Newton failed"; return false; }
  gauss(Q, t->xq, t->wq);
  for (int q = 0; q < Q; ++q) {
    double L[MAXP + 1], dL[MAXP + 1];
    lagrange(p + 1, xi, t->xq[q], L, dL);
    double acc = 0.0;
    for (int i = 0; i <= p; ++i) t->Bl[q][i] = L[i];
    for (int j = 0; j < p; ++j) { acc -= dL[j]; t->Bh[q][j] = acc; }
  }
  for (int i = 0; i <= p; ++i)
    for (int j = 0; j <= p; ++j) {
      double s = 0.0;
      for (int q = 0; q < Q; ++q) s += t->wq[q] * t->Bl[q][i] * t->Bl[q][j];
      t->Ml[i][j] = s;
    }
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j) {
      double s = 0.0;
      for (int q = 0; q < Q; ++q) s += t->wq[q] * t->Bh[q][i] * t->Bh[q][j];
      t->Mh[i][j] = s;
    }
  if (!invert_spd(p, &t->Mh[0][0], &t->Mhinv[0][0])) { *err = "M_h singular"; return false; }
  // GL-nodal basis on the p-point Gauss rule
  double g[MAXP + 2], gw[MAXP + 2];
  gauss(p, g, gw);
  for (int q = 0; q < Q; ++q) {
    double L[MAXP + 1], dL[MAXP + 1];
    lagrange(p, g, t->xq[q], L, dL);
    for (int b = 0; b < p; ++b) t->BG[q][b] = L[b];
  }
  // HG[a][b] = integral_{xi_a}^{xi_{a+1}} L_b, by a (p+1)-point Gauss rule per subinterval
  double sx[MAXP + 2], sw[MAXP + 2];
  gauss(p + 1, sx, sw);
  for (int a = 0; a < p; ++a)
    for (int b = 0; b < p; ++b) {
      double s = 0.0;
      for (int k = 0; k <= p; ++k) {
        const double x = xi[a] + (xi[a + 1] - xi[a]) * sx[k];
        double L[MAXP + 1], dL[MAXP + 1];
        lagrange(p, g, x, L, dL);
        s += (xi[a + 1] - xi[a]) * sw[k] * L[b];
      }
      t->HG[a][b] = s;
    }
  return true;
}

}  // namespace hdiv
