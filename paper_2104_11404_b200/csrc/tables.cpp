// tables.cpp -- the library's 1D basis/quadrature tables, computed on the host in
// IEEE binary128 (__float128) and rounded once to double (correctly rounded).
//
// Readings (R5/R6; PAPER P:384-394 defers the FE spaces to Dobrev 2012):
//   reference element [0,1]^d; tensor Gauss-Legendre quadrature with q points/dim;
//   H1 basis: degree-k Lagrange on the k+1 Gauss-Lobatto points {0, roots of P_k', 1};
//   L2 basis: degree-(k-1) Lagrange on the k Gauss-Legendre points.
// Independent of the oracle's mpmath tables (oracle/tables.py); a not-gpu test demands
// the two agree bit for bit, which holds because both are correctly rounded.
#include <cmath>
#include <cstring>

#include "hydro_internal.h"

namespace {
typedef __float128 qf;

qf qabs(qf x) { return x < 0 ? -x : x; }

// Legendre P_n and derivatives at x by the three-term recurrence.
void legendre(int n, qf x, qf *p, qf *dp, qf *d2p) {
  qf p0 = 1, p1 = x, d0 = 0, d1 = 1, s0 = 0, s1 = 0;
  if (n == 0) { *p = 1; *dp = 0; *d2p = 0; return; }
  for (int m = 1; m < n; ++m) {
    qf p2 = ((2 * m + 1) * x * p1 - m * p0) / (m + 1);
    qf d2 = d0 + (2 * m + 1) * p1;       // P'_{m+1} = P'_{m-1} + (2m+1) P_m
    qf s2 = s0 + (2 * m + 1) * d1;       // P''_{m+1} = P''_{m-1} + (2m+1) P'_m
    p0 = p1; p1 = p2; d0 = d1; d1 = d2; s0 = s1; s1 = s2;
  }
  *p = p1; *dp = d1; *d2p = s1;
}

// Gauss-Legendre points/weights on [-1,1], ascending.
void gauss_legendre(int n, qf *x, qf *w) {
  for (int i = 0; i < n; ++i) {
    qf t = (qf)-std::cos(M_PI * (i + 0.75) / (n + 0.5));
    for (int it = 0; it < 100; ++it) {
      qf p, dp, d2;
      legendre(n, t, &p, &dp, &d2);
      qf dx = p / dp;
      t -= dx;
      if (qabs(dx) < (qf)1e-33) break;
    }
    qf p, dp, d2;
    legendre(n, t, &p, &dp, &d2);
    x[i] = t;
    w[i] = 2 / ((1 - t * t) * dp * dp);
  }
}

// Gauss-Lobatto points on [-1,1] (k+1 of them), ascending.
void gauss_lobatto(int k, qf *x) {
  x[0] = -1;
  x[k] = 1;
  for (int i = 1; i < k; ++i) {
    qf t = (qf)-std::cos(M_PI * i / k);
    for (int it = 0; it < 100; ++it) {
      qf p, dp, d2;
      legendre(k, t, &p, &dp, &d2);
      qf dx = dp / d2;
      t -= dx;
      if (qabs(dx) < (qf)1e-33) break;
    }
    x[i] = t;
  }
}

qf lagrange(const qf *nodes, int n, int j, qf t) {
  qf v = 1;
  for (int m = 0; m < n; ++m)
    if (m != j) v *= (t - nodes[m]) / (nodes[j] - nodes[m]);
  return v;
}

qf lagrange_d(const qf *nodes, int n, int j, qf t) {
  qf s = 0;
  for (int i = 0; i < n; ++i) {
    if (i == j) continue;
    qf term = 1 / (nodes[j] - nodes[i]);
    for (int m = 0; m < n; ++m)
      if (m != j && m != i) term *= (t - nodes[m]) / (nodes[j] - nodes[m]);
    s += term;
  }
  return s;
}
}  // namespace

int hydro_make_tables(int k, int q, hydro_tables_t *T) {
  if (k < 1 || k > HYDRO_MAXN - 1 || q < 1 || q > HYDRO_MAXQ) return 1;
  std::memset(T, 0, sizeof(*T));
  T->k = k;
  T->q = q;
  qf g[HYDRO_MAXQ], gw[HYDRO_MAXQ], gll[HYDRO_MAXN], gl2[HYDRO_MAXN];
  gauss_legendre(q, g, gw);
  gauss_lobatto(k, gll);
  {
    qf tmpw[HYDRO_MAXN];
    gauss_legendre(k, gl2, tmpw);
  }
  qf xi[HYDRO_MAXQ];
  for (int i = 0; i < q; ++i) {
    xi[i] = (g[i] + 1) / 2;
    T->xi[i] = (double)xi[i];
    T->w[i] = (double)(gw[i] / 2);
  }
  qf n1[HYDRO_MAXN], n2[HYDRO_MAXN];
  for (int a = 0; a <= k; ++a) n1[a] = (gll[a] + 1) / 2;
  for (int j = 0; j < k; ++j) n2[j] = (gl2[j] + 1) / 2;
  for (int i = 0; i < q; ++i) {
    for (int a = 0; a <= k; ++a) {
      T->B[i][a] = (double)lagrange(n1, k + 1, a, xi[i]);
      T->G[i][a] = (double)lagrange_d(n1, k + 1, a, xi[i]);
    }
    for (int j = 0; j < k; ++j) T->Bl[i][j] = (double)lagrange(n2, k, j, xi[i]);
  }
  return 0;
}
