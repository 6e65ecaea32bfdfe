/*
 * hydro_oracle.c -- plain, slow, CPU reference of the corner-force evaluation.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  It shares no code,
 * header, table or constant generator with the CUDA path (paper_2104_11404_b200/).
 *
 * What it computes (Sec. 2):
 *   Semi-discrete Lagrangian hydro (Eq. fom):
 *     M_V dv/dt = -F.1,  M_E de/dt = F^T.v,  with F1 = F.1 and FTv = F^T.v
 *     (Eq. forceOneforceTv).
 *   F (never written in the paper, which defers to Dobrev 2012) is the
 *   weak form of the momentum equation rho dv/dt = div(sigma) (Eq. euler)
 *   tested with phi_a e_c and expanded in the L2 basis psi_j (DESIGN R1):
 *     F_K[(a,c)][j] = sum_q w_q detJ_q [sigma_q J_q^{-T} gradhat(phi_a)(xi_q)]_c psi_j(xi_q)
 *   sigma = -p I + mu eps(v)   (DESIGN R3), p = (gamma-1) rho e (Eq. EOS,
 *   P:372-376), rho_q = m_q / detJ_q with m_q = rho0_K detJ0_q (density elimination,
 *   P:389-391, DESIGN R11).
 *   dt = min over all quadrature points of
 *     alpha / (c_s/h + alpha_mu mu/(rho h^2))   (Eq. adaptive-timestep),
 *   h = minimal singular value of the zone Jacobian (DESIGN R2).
 *
 * How (step by step, no blocking or fusion beyond the definition):
 *   1. per element: gather X, V, W (W = V when w == NULL), E_K, gamma_K;
 *   2. per quadrature point: J, grad(v), grad(w), e_q by the canonical contraction
 *      order (DESIGN "Evaluation contract" A.2), J0 from x0 likewise -> m_q;
 *   3. pointwise physics in the contract order A.3 (no FMA), lmin3 per A.4 (R30);
 *   4. the DENSE element matrix F_K (not sum-factorised), then F_K.1 and F_K^T.w;
 *   5. F.1 assembled serially in ascending element order; F^T.w element-local;
 *   6. dt = min over (K, q); NaN if any dt_q is NaN; lowest tangled element.
 * Also returns per-entry magnitude scales M (sum of |terms|) used by the parity
 * tolerance (DESIGN "Tolerances").
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp -shared -fPIC
 * (no FMA contraction; every FMA is written as fma()).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define MAXN 4   /* H1 nodes per dim (k+1 <= 4) */
#define MAXQ 6   /* GL points per dim */
#define MAXM 3   /* L2 nodes per dim (k <= 3) */

typedef struct {
  int dim, k, q;
  double xi[MAXQ], w[MAXQ];
  double B[MAXQ][MAXN], G[MAXQ][MAXN], Bl[MAXQ][MAXM];
} otab;

/* ---------------------------------------------------------------- A.4 lmin3 */
/* Smallest eigenvalue of a symmetric 3x3 matrix (DESIGN A.4, reading R30).
 *
 * Closed form (the trigonometric characterisation of the eigenvalues of a symmetric
 * 3x3 matrix): with q = tr(A)/3, B = A - qI, p = sqrt(tr(B^2)/6), the eigenvalues are
 * q + 2p c where c runs over the roots of 4c^3 - 3c = r, r = det(B)/(2p^3) in [-1, 1]
 * (c = cos(theta/3 + 2 pi k/3), r = cos(theta)); lambda_min takes the smallest root,
 * c in [-1, -1/2].  That root is found from a cubic initial guess in s = sqrt((1-r)/2)
 * (c = cos(2pi/3 + (2/3) asin s)) refined by two Newton steps on 4c^3 - 3c - r.  It is
 * ill-conditioned only near r = 1, where lambda_min is a double eigenvalue: there
 * (r > 1 - 2^-13, or r NaN) the cyclic Jacobi method below is used instead.  A = qI
 * (p2 == 0) returns q.  IEEE ops, FMA only where written as fma().
 *
 * Jacobi fallback: at most four cyclic sweeps over the pairs (0,1), (0,2), (1,2); a pair
 * whose off-diagonal is negligible (<= 2^-53 max|a_ij|, which also covers a_pq == 0) is
 * skipped -- this also removes the 0/0 of a re-introduced subnormal a_pq on an exactly
 * degenerate diagonal. IEEE ops only, no FMA. */
/* instrumentation for bench.py's algorithmic-work count (not part of the method):
 * Jacobi rotations performed / lmin3 calls / Jacobi fallbacks, summed over threads */
static int64_t g_rot = 0, g_calls = 0, g_fallback = 0;
static __thread int64_t t_rot = 0, t_calls = 0, t_fallback = 0;

void oracle_stats(int64_t *rotations, int64_t *calls, int reset) {
  if (rotations) *rotations = g_rot;
  if (calls) *calls = g_calls;
  if (reset) { g_rot = 0; g_calls = 0; g_fallback = 0; }
}

void oracle_stats2(int64_t *rotations, int64_t *calls, int64_t *fallbacks, int reset) {
  if (rotations) *rotations = g_rot;
  if (calls) *calls = g_calls;
  if (fallbacks) *fallbacks = g_fallback;
  if (reset) { g_rot = 0; g_calls = 0; g_fallback = 0; }
}

static double lmin3_jacobi(const double a_in[6]);

double oracle_lmin3(const double a_in[6] /* a00 a11 a22 a01 a02 a12 */) {
  ++t_calls;
  const double a00 = a_in[0], a11 = a_in[1], a22 = a_in[2];
  const double a01 = a_in[3], a02 = a_in[4], a12 = a_in[5];
  const double third = 0x1.5555555555555p-2, sixth = 0x1.5555555555555p-3;  /* RN(1/3), RN(1/6) */
  const double q = ((a00 + a11) + a22) * third;
  const double b0 = a00 - q, b1 = a11 - q, b2 = a22 - q;
  const double p1 = (a01 * a01 + a02 * a02) + a12 * a12;
  const double p2 = ((b0 * b0 + b1 * b1) + b2 * b2) + 2.0 * p1;
  if (p2 == 0.0) return q;                                /* A = qI */
  const double p = sqrt(p2 * sixth);
  const double det = (b0 * (b1 * b2 - a12 * a12) - a01 * (a01 * b2 - a12 * a02)) +
                     a02 * (a01 * a12 - b1 * a02);
  double r = det / ((2.0 * p) * (p * p));
  if (!(r <= 1.0 - 0x1p-13)) {                            /* near-double lambda_min or NaN */
    ++t_fallback;
    return lmin3_jacobi(a_in);
  }
  r = fmax(r, -1.0);
  const double s = sqrt((1.0 - r) * 0.5);
  /* c0(s) = -1/2 - s/sqrt(3) + s^2 (K2 + s (K3 + s (K4 + s K5))), Horner with fma */
  double u = fma(s, -0.005042, 0.021433);
  u = fma(s, u, -0.04969);
  u = fma(s, u, 0.110644);
  u = fma(s, u, -0x1.279a74590331cp-1);                  /* -RN(1/sqrt(3)) */
  double c = fma(s, u, -0.5);
  for (int it = 0; it < 2; ++it) {                        /* Newton on f(c) = c (4c^2 - 3) - r */
    const double c2 = c * c;
    const double f = fma(c, fma(4.0, c2, -3.0), -r);
    const double fp = fma(12.0, c2, -3.0);
    c = c - f / fp;
  }
  return fma(2.0 * p, c, q);
}

static double lmin3_jacobi(const double a_in[6]) {
  double a[3][3];
  a[0][0] = a_in[0]; a[1][1] = a_in[1]; a[2][2] = a_in[2];
  a[0][1] = a[1][0] = a_in[3];
  a[0][2] = a[2][0] = a_in[4];
  a[1][2] = a[2][1] = a_in[5];
  static const int P[3] = {0, 0, 1}, Qp[3] = {1, 2, 2};
  /* negligibility threshold (DESIGN A.4): |a_pq| <= 2^-53 * max|a_ij| is skipped */
  double amax = fabs(a_in[0]);
  for (int i = 1; i < 6; ++i) amax = fmax(amax, fabs(a_in[i]));
  const double tol = amax * 0x1p-53;
  for (int sweep = 0; sweep < 4; ++sweep) {
    for (int r = 0; r < 3; ++r) {
      const int p = P[r], q = Qp[r];
      const double apq = a[p][q];
      if (fabs(apq) <= tol) continue;
      ++t_rot;
      const double dlt = 0.5 * (a[q][q] - a[p][p]);
      const double rr = sqrt(dlt * dlt + apq * apq);
      double t = apq / (fabs(dlt) + rr);
      if (dlt < 0.0) t = -t;
      const double c = 1.0 / sqrt(1.0 + t * t);
      const double s = t * c;
      const int r3 = 3 - p - q;
      const double arp = a[r3][p], arq = a[r3][q];
      a[p][p] = a[p][p] - t * apq;
      a[q][q] = a[q][q] + t * apq;
      a[p][q] = a[q][p] = 0.0;
      a[r3][p] = a[p][r3] = c * arp - s * arq;
      a[r3][q] = a[q][r3] = s * arp + c * arq;
    }
  }
  return fmin(fmin(a[0][0], a[1][1]), a[2][2]);
}

/* ---------------------------------------------------------------- A.2 contractions */
/* Canonical FMA chain: acc = t0*u0; acc = fma(ti, ui, acc), i ascending. */
#define CHAIN(N, T, U, OUT)                              \
  do {                                                   \
    double acc_ = (T(0)) * (U(0));                       \
    for (int i_ = 1; i_ < (N); ++i_) acc_ = fma((T(i_)), (U(i_)), acc_); \
    (OUT) = acc_;                                        \
  } while (0)

/* 2D gradient of one scalar field X[a2][a1] at all qps: D[q2][q1][delta]. */
static void grad2(const otab *T, const double *X, double D[MAXQ][MAXQ][2]) {
  const int n = T->k + 1, q = T->q;
  double UB[MAXQ][MAXN], UG[MAXQ][MAXN];
  for (int q1 = 0; q1 < q; ++q1)
    for (int a2 = 0; a2 < n; ++a2) {
#define TB(i) T->B[q1][i]
#define TG(i) T->G[q1][i]
#define UX(i) X[a2 * n + (i)]
      CHAIN(n, TB, UX, UB[q1][a2]);
      CHAIN(n, TG, UX, UG[q1][a2]);
#undef TB
#undef TG
#undef UX
    }
  for (int q2 = 0; q2 < q; ++q2)
    for (int q1 = 0; q1 < q; ++q1) {
#define TB(i) T->B[q2][i]
#define TG(i) T->G[q2][i]
#define UGq(i) UG[q1][i]
#define UBq(i) UB[q1][i]
      CHAIN(n, TB, UGq, D[q2][q1][0]);
      CHAIN(n, TG, UBq, D[q2][q1][1]);
#undef TB
#undef TG
#undef UGq
#undef UBq
    }
}

/* 3D gradient of one scalar field X[a3][a2][a1] at all qps: D[q3][q2][q1][delta]. */
static void grad3(const otab *T, const double *X, double D[MAXQ][MAXQ][MAXQ][3]) {
  const int n = T->k + 1, q = T->q;
  double UB[MAXQ][MAXN][MAXN], UG[MAXQ][MAXN][MAXN];          /* [q1][a2][a3] */
  double P1[MAXQ][MAXQ][MAXN], P2[MAXQ][MAXQ][MAXN], P3[MAXQ][MAXQ][MAXN]; /* [q1][q2][a3] */
  for (int q1 = 0; q1 < q; ++q1)
    for (int a2 = 0; a2 < n; ++a2)
      for (int a3 = 0; a3 < n; ++a3) {
#define TB(i) T->B[q1][i]
#define TG(i) T->G[q1][i]
#define UX(i) X[(a3 * n + a2) * n + (i)]
        CHAIN(n, TB, UX, UB[q1][a2][a3]);
        CHAIN(n, TG, UX, UG[q1][a2][a3]);
#undef TB
#undef TG
#undef UX
      }
  for (int q1 = 0; q1 < q; ++q1)
    for (int q2 = 0; q2 < q; ++q2)
      for (int a3 = 0; a3 < n; ++a3) {
#define TB(i) T->B[q2][i]
#define TG(i) T->G[q2][i]
#define UGq(i) UG[q1][i][a3]
#define UBq(i) UB[q1][i][a3]
        CHAIN(n, TB, UGq, P1[q1][q2][a3]);
        CHAIN(n, TG, UBq, P2[q1][q2][a3]);
        CHAIN(n, TB, UBq, P3[q1][q2][a3]);
#undef TB
#undef TG
#undef UGq
#undef UBq
      }
  for (int q3 = 0; q3 < q; ++q3)
    for (int q2 = 0; q2 < q; ++q2)
      for (int q1 = 0; q1 < q; ++q1) {
#define TB(i) T->B[q3][i]
#define TG(i) T->G[q3][i]
#define V1(i) P1[q1][q2][i]
#define V2(i) P2[q1][q2][i]
#define V3(i) P3[q1][q2][i]
        CHAIN(n, TB, V1, D[q3][q2][q1][0]);
        CHAIN(n, TB, V2, D[q3][q2][q1][1]);
        CHAIN(n, TG, V3, D[q3][q2][q1][2]);
#undef TB
#undef TG
#undef V1
#undef V2
#undef V3
      }
}

/* L2 interpolation e_q (canonical order: j1, then j2, then j3). */
static void interp2(const otab *T, const double *E, double eq[MAXQ][MAXQ]) {
  const int m = T->k, q = T->q;
  double U[MAXQ][MAXM];
  for (int q1 = 0; q1 < q; ++q1)
    for (int j2 = 0; j2 < m; ++j2) {
#define TB(i) T->Bl[q1][i]
#define UX(i) E[j2 * m + (i)]
      CHAIN(m, TB, UX, U[q1][j2]);
#undef TB
#undef UX
    }
  for (int q2 = 0; q2 < q; ++q2)
    for (int q1 = 0; q1 < q; ++q1) {
#define TB(i) T->Bl[q2][i]
#define UX(i) U[q1][i]
      CHAIN(m, TB, UX, eq[q2][q1]);
#undef TB
#undef UX
    }
}

static void interp3(const otab *T, const double *E, double eq[MAXQ][MAXQ][MAXQ]) {
  const int m = T->k, q = T->q;
  double U1[MAXQ][MAXM][MAXM], U2[MAXQ][MAXQ][MAXM];
  for (int q1 = 0; q1 < q; ++q1)
    for (int j2 = 0; j2 < m; ++j2)
      for (int j3 = 0; j3 < m; ++j3) {
#define TB(i) T->Bl[q1][i]
#define UX(i) E[(j3 * m + j2) * m + (i)]
        CHAIN(m, TB, UX, U1[q1][j2][j3]);
#undef TB
#undef UX
      }
  for (int q1 = 0; q1 < q; ++q1)
    for (int q2 = 0; q2 < q; ++q2)
      for (int j3 = 0; j3 < m; ++j3) {
#define TB(i) T->Bl[q2][i]
#define UX(i) U1[q1][i][j3]
        CHAIN(m, TB, UX, U2[q1][q2][j3]);
#undef TB
#undef UX
      }
  for (int q3 = 0; q3 < q; ++q3)
    for (int q2 = 0; q2 < q; ++q2)
      for (int q1 = 0; q1 < q; ++q1) {
#define TB(i) T->Bl[q3][i]
#define UX(i) U2[q1][q2][i]
        CHAIN(m, TB, UX, eq[q3][q2][q1]);
#undef TB
#undef UX
      }
}

/* ---------------------------------------------------------------- A.3 pointwise */
typedef struct {
  double gamma, q1, q2, alpha, alpha_mu;
  int visc;
} phys;

/* Determinant and inverse (contract formulas). Returns det. */
static double det_inv(int dim, const double J[3][3], double Ji[3][3]) {
  if (dim == 2) {
    const double det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    const double inv = 1.0 / det;
    Ji[0][0] = J[1][1] * inv; Ji[0][1] = -(J[0][1] * inv);
    Ji[1][0] = -(J[1][0] * inv); Ji[1][1] = J[0][0] * inv;
    return det;
  }
  double C[3][3];
  C[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
  C[0][1] = J[1][2] * J[2][0] - J[1][0] * J[2][2];
  C[0][2] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
  C[1][0] = J[0][2] * J[2][1] - J[0][1] * J[2][2];
  C[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
  C[1][2] = J[0][1] * J[2][0] - J[0][0] * J[2][1];
  C[2][0] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
  C[2][1] = J[0][2] * J[1][0] - J[0][0] * J[1][2];
  C[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
  const double det = (J[0][0] * C[0][0] + J[0][1] * C[0][1]) + J[0][2] * C[0][2];
  const double inv = 1.0 / det;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) Ji[i][j] = C[j][i] * inv;
  return det;
}

static double det_only(int dim, const double J[3][3]) {
  double Ji[3][3];
  return det_inv(dim, J, Ji);
}

/* Pointwise physics at one qp. Inputs J (J[c][d] = dx_c/dxi_d), Gv (grad-hat v),
 * e_q, m_q. Outputs sigma (dim x dim), Ji, det; returns dt_q. */
static double pointwise(int dim, const phys *P, const double J[3][3], const double Gv[3][3],
                        double eq, double mq, double sigma[3][3], double Ji[3][3], double *det_out) {
  const double det = det_inv(dim, J, Ji);
  *det_out = det;
  const double rho = mq / det;
  const double gam = P->gamma;
  const double p = ((gam - 1.0) * rho) * eq;
  /* no clamp: e < 0 or NaN gives NaN -> dt NaN -> status NONFINITE (DESIGN R12) */
  const double cs = sqrt((gam * (gam - 1.0)) * eq);
  double h;
  if (dim == 2) {
    const double c00 = J[0][0] * J[0][0] + J[1][0] * J[1][0];
    const double c11 = J[0][1] * J[0][1] + J[1][1] * J[1][1];
    const double c01 = J[0][0] * J[0][1] + J[1][0] * J[1][1];
    const double kk = 0.5 * (c00 - c11);
    const double smax2 = 0.5 * (c00 + c11) + sqrt(kk * kk + c01 * c01);
    h = det / sqrt(smax2);
  } else {
    double c[6];
    const int ii[6] = {0, 1, 2, 0, 0, 1}, jj[6] = {0, 1, 2, 1, 2, 2};
    for (int r = 0; r < 6; ++r) {
      const int i = ii[r], j = jj[r];
      c[r] = (J[0][i] * J[0][j] + J[1][i] * J[1][j]) + J[2][i] * J[2][j];
    }
    h = sqrt(fmax(oracle_lmin3(c), 0.0));
  }
  double mu = 0.0;
  double eps[3][3] = {{0}};
  if (P->visc) {
    double gv[3][3];
    for (int c = 0; c < dim; ++c)
      for (int d = 0; d < dim; ++d) {
        double s = Gv[c][0] * Ji[0][d];
        for (int i = 1; i < dim; ++i) s = s + Gv[c][i] * Ji[i][d];
        gv[c][d] = s;
      }
    for (int c = 0; c < dim; ++c) {
      eps[c][c] = gv[c][c];
      for (int d = 0; d < dim; ++d)
        if (d != c) eps[c][d] = 0.5 * (gv[c][d] + gv[d][c]);
    }
    double lam;
    if (dim == 2) {
      const double k = 0.5 * (eps[0][0] - eps[1][1]);
      lam = 0.5 * (eps[0][0] + eps[1][1]) - sqrt(k * k + eps[0][1] * eps[0][1]);
    } else {
      const double a[6] = {eps[0][0], eps[1][1], eps[2][2], eps[0][1], eps[0][2], eps[1][2]};
      lam = oracle_lmin3(a);
    }
    const double lneg = fmin(lam, 0.0);
    mu = (rho * h) * ((P->q1 * cs) + ((P->q2 * h) * (-lneg)));
  }
  const double den = (rho * h) * h;
  const double inv_dt = cs / h + (P->alpha_mu * mu) / den;
  const double dtq = P->alpha / inv_dt;
  /* stress (outside the dt contract; tolerance only) */
  for (int c = 0; c < dim; ++c)
    for (int d = 0; d < dim; ++d) sigma[c][d] = mu * eps[c][d] - (c == d ? p : 0.0);
  return dtq;
}

/* total order on non-NaN doubles with -0 < +0 */
static int dt_less(double a, double b) {
  return a < b || (a == b && signbit(a) && !signbit(b));
}

/* ---------------------------------------------------------------- element driver */
typedef struct {
  int dim, nd, ne, nq;      /* nodes/elem, L2 dofs/elem, qps/elem */
} shape_t;

/* Dense tensor-product basis derivative Dphi[qp][a][delta] and psi[qp][j]. */
static void dense_basis(const otab *T, double *Dphi, double *psi) {
  const int n = T->k + 1, m = T->k, q = T->q, dim = T->dim;
  const int nd = dim == 2 ? n * n : n * n * n;
  const int ne = dim == 2 ? m * m : m * m * m;
  const int nq = dim == 2 ? q * q : q * q * q;
  for (int qp = 0; qp < nq; ++qp) {
    const int q1 = qp % q, q2 = (qp / q) % q, q3 = dim == 3 ? qp / (q * q) : 0;
    for (int a = 0; a < nd; ++a) {
      const int a1 = a % n, a2 = (a / n) % n, a3 = dim == 3 ? a / (n * n) : 0;
      if (dim == 2) {
        Dphi[(qp * nd + a) * 3 + 0] = T->G[q1][a1] * T->B[q2][a2];
        Dphi[(qp * nd + a) * 3 + 1] = T->B[q1][a1] * T->G[q2][a2];
        Dphi[(qp * nd + a) * 3 + 2] = 0.0;
      } else {
        Dphi[(qp * nd + a) * 3 + 0] = T->G[q1][a1] * T->B[q2][a2] * T->B[q3][a3];
        Dphi[(qp * nd + a) * 3 + 1] = T->B[q1][a1] * T->G[q2][a2] * T->B[q3][a3];
        Dphi[(qp * nd + a) * 3 + 2] = T->B[q1][a1] * T->B[q2][a2] * T->G[q3][a3];
      }
    }
    for (int j = 0; j < ne; ++j) {
      const int j1 = j % m, j2 = (j / m) % m, j3 = dim == 3 ? j / (m * m) : 0;
      psi[qp * ne + j] = dim == 2 ? T->Bl[q1][j1] * T->Bl[q2][j2]
                                  : T->Bl[q1][j1] * T->Bl[q2][j2] * T->Bl[q3][j3];
    }
  }
}

/* Forward gradients of a [dim][n_nodes] SoA field gathered into Xl[c][a]:
 * out[qp][c][delta] (qp lexicographic q1 fastest). */
static void forward_grad(const otab *T, const double *Xl /*[dim][nd]*/, int nd, double *out) {
  const int q = T->q, dim = T->dim;
  if (dim == 2) {
    double D[MAXQ][MAXQ][2];
    for (int c = 0; c < 2; ++c) {
      grad2(T, Xl + c * nd, D);
      for (int q2 = 0; q2 < q; ++q2)
        for (int q1 = 0; q1 < q; ++q1)
          for (int d = 0; d < 2; ++d) out[((q2 * q + q1) * 3 + c) * 3 + d] = D[q2][q1][d];
    }
  } else {
    static __thread double D[MAXQ][MAXQ][MAXQ][3];
    for (int c = 0; c < 3; ++c) {
      grad3(T, Xl + c * nd, D);
      for (int q3 = 0; q3 < q; ++q3)
        for (int q2 = 0; q2 < q; ++q2)
          for (int q1 = 0; q1 < q; ++q1)
            for (int d = 0; d < 3; ++d)
              out[(((q3 * q + q2) * q + q1) * 3 + c) * 3 + d] = D[q3][q2][q1][d];
    }
  }
}

static void forward_interp(const otab *T, const double *El, double *eq) {
  const int q = T->q;
  if (T->dim == 2) {
    double D[MAXQ][MAXQ];
    interp2(T, El, D);
    for (int q2 = 0; q2 < q; ++q2)
      for (int q1 = 0; q1 < q; ++q1) eq[q2 * q + q1] = D[q2][q1];
  } else {
    double D[MAXQ][MAXQ][MAXQ];
    interp3(T, El, D);
    for (int q3 = 0; q3 < q; ++q3)
      for (int q2 = 0; q2 < q; ++q2)
        for (int q1 = 0; q1 < q; ++q1) eq[(q3 * q + q2) * q + q1] = D[q3][q2][q1];
  }
}

typedef struct {
  int64_t first_bad;  /* lowest element with detJ <= 0 (or n_elem if none) */
  int any_nan;
} ostatus;

/*
 * oracle_force: see the file header. Arguments
 *   tab               : tables (dim, k, q and the 1D arrays)
 *   n_elem, n_nodes   : mesh sizes
 *   elem_nodes        : [n_elem][(k+1)^dim] int32
 *   x0, rho0          : initial positions [dim][n_nodes], density [n_elem]
 *   x, v, e, w, gamma : state; w == NULL means w = v
 *   elist, n_list     : elements to evaluate (NULL => all, ascending)
 *   mode              : 0 = forces + dt, 1 = dt only
 * Outputs (any may be NULL): F1 [dim][n_nodes] (zeroed then assembled over the
 *   listed elements), FTw [n_elem][k^dim] (only listed elements written), F1mag,
 *   FTwmag (magnitude scales), dt (scalar), first_bad (lowest tangled element or -1),
 *   dtq_out [n_list][nq] per-qp dt (optional).
 * Returns 0, or 4 if an element is tangled, 5 if a dt_q is NaN.
 */
int oracle_force(const otab *tab, int64_t n_elem, int64_t n_nodes, const int32_t *elem_nodes,
                 const double *x0, const double *rho0, const double *x, const double *v,
                 const double *e, const double *w, const double *gamma, int visc, double q1,
                 double q2, double alpha, double alpha_mu, const int32_t *elist, int64_t n_list,
                 int mode, double *F1, double *FTw, double *F1mag, double *FTwmag, double *dt,
                 int64_t *first_bad, double *dtq_out, int nthreads) {
  const int dim = tab->dim, n = tab->k + 1, m = tab->k, q = tab->q;
  const int nd = dim == 2 ? n * n : n * n * n;
  const int ne = dim == 2 ? m * m : m * m * m;
  const int nq = dim == 2 ? q * q : q * q * q;
  if (!elist) n_list = n_elem;
  double *Dphi = (double *)malloc(sizeof(double) * nq * nd * 3);
  double *psi = (double *)malloc(sizeof(double) * nq * ne);
  dense_basis(tab, Dphi, psi);
  double *F1loc = NULL, *F1locmag = NULL;
  if (mode == 0 && F1) {
    F1loc = (double *)malloc(sizeof(double) * (size_t)n_list * nd * dim);
    F1locmag = (double *)malloc(sizeof(double) * (size_t)n_list * nd * dim);
  }
  double dt_min = INFINITY;
  int any_nan = 0;
  int64_t bad = INT64_MAX;
  /* nthreads > 0: that many threads for this call only; 0: every host core */
#ifdef _OPENMP
  const int nt_use = nthreads > 0 ? nthreads : omp_get_num_procs();
#else
  const int nt_use = 1;
#endif
  (void)nt_use;
#pragma omp parallel num_threads(nt_use)
  {
    double *Xl = (double *)malloc(sizeof(double) * 3 * nd * 4);
    double *Vl = Xl + 3 * nd, *Wl = Xl + 6 * nd, *X0l = Xl + 9 * nd;
    double El[MAXM * MAXM * MAXM];
    double *gx = (double *)malloc(sizeof(double) * nq * 9 * 3);
    double *gv = gx + nq * 9, *gw = gx + 2 * nq * 9;
    double *gx0 = (double *)malloc(sizeof(double) * nq * 9);
    double *eqv = (double *)malloc(sizeof(double) * nq);
    double *S = (double *)malloc(sizeof(double) * nq * 9);
    double *Smag = (double *)malloc(sizeof(double) * nq * 9);
    double *FK = (double *)malloc(sizeof(double) * nd * 3 * ne);
    double my_dt = INFINITY;
    int my_nan = 0;
    int64_t my_bad = INT64_MAX;
#pragma omp for schedule(dynamic, 16)
    for (int64_t li = 0; li < n_list; ++li) {
      const int64_t K = elist ? elist[li] : li;
      const int32_t *en = elem_nodes + K * nd;
      for (int c = 0; c < dim; ++c)
        for (int a = 0; a < nd; ++a) {
          const int64_t g = (int64_t)c * n_nodes + en[a];
          Xl[c * nd + a] = x[g];
          Vl[c * nd + a] = v[g];
          Wl[c * nd + a] = w ? w[g] : v[g];
          X0l[c * nd + a] = x0[g];
        }
      for (int j = 0; j < ne; ++j) El[j] = e[K * ne + j];
      /* step 2: forward */
      forward_grad(tab, Xl, nd, gx);
      forward_grad(tab, Vl, nd, gv);
      forward_grad(tab, Wl, nd, gw);
      forward_grad(tab, X0l, nd, gx0);
      forward_interp(tab, El, eqv);
      phys P = {gamma[K], q1, q2, alpha, alpha_mu, visc};
      int tangled = 0;
      for (int qp = 0; qp < nq; ++qp) {
        double J[3][3] = {{0}}, J0[3][3] = {{0}}, G[3][3] = {{0}}, sig[3][3], Ji[3][3] = {{0}};
        for (int c = 0; c < dim; ++c)
          for (int d = 0; d < dim; ++d) {
            J[c][d] = gx[(qp * 3 + c) * 3 + d];
            J0[c][d] = gx0[(qp * 3 + c) * 3 + d];
            G[c][d] = gv[(qp * 3 + c) * 3 + d];
          }
        /* density elimination: m_q = rho0_K * detJ0 (setup quantity) */
        const double mq = rho0[K] * det_only(dim, J0);
        double det;
        const double dtq = pointwise(dim, &P, J, G, eqv[qp], mq, sig, Ji, &det);
        if (!(det > 0.0)) tangled = 1;
        if (isnan(dtq)) my_nan = 1;
        else if (dt_less(dtq, my_dt)) my_dt = dtq;
        if (dtq_out) dtq_out[li * nq + qp] = dtq;
        if (mode != 0) continue;
        /* S_q = (w_q detJ) sigma J^{-T};  (sigma J^{-T})[c][d] = sum_i sigma[c][i] Ji[d][i] */
        const int qq1 = qp % q, qq2 = (qp / q) % q, qq3 = dim == 3 ? qp / (q * q) : 0;
        const double wq = dim == 2 ? tab->w[qq1] * tab->w[qq2]
                                   : tab->w[qq1] * tab->w[qq2] * tab->w[qq3];
        for (int c = 0; c < dim; ++c)
          for (int d = 0; d < dim; ++d) {
            double s = 0.0, sm = 0.0;
            for (int i = 0; i < dim; ++i) {
              s += sig[c][i] * Ji[d][i];
              sm += fabs(sig[c][i] * Ji[d][i]);
            }
            S[qp * 9 + c * 3 + d] = (wq * det) * s;
            Smag[qp * 9 + c * 3 + d] = fabs(wq * det) * sm;
          }
      }
      if (tangled && K < my_bad) my_bad = K;
      if (mode != 0) continue;
      /* step 4: dense element force matrix F_K[(a,c)][j] */
      memset(FK, 0, sizeof(double) * nd * 3 * ne);
      for (int qp = 0; qp < nq; ++qp)
        for (int a = 0; a < nd; ++a)
          for (int c = 0; c < dim; ++c) {
            double t = 0.0;
            for (int d = 0; d < dim; ++d) t += S[qp * 9 + c * 3 + d] * Dphi[(qp * nd + a) * 3 + d];
            for (int j = 0; j < ne; ++j) FK[(a * 3 + c) * ne + j] += t * psi[qp * ne + j];
          }
      /* F_K . 1 and F_K^T . w */
      if (F1loc) {
        for (int a = 0; a < nd; ++a)
          for (int c = 0; c < dim; ++c) {
            double s = 0.0;
            for (int j = 0; j < ne; ++j) s += FK[(a * 3 + c) * ne + j];
            F1loc[(li * nd + a) * dim + c] = s;
            double mg = 0.0;
            for (int qp = 0; qp < nq; ++qp)
              for (int d = 0; d < dim; ++d)
                mg += Smag[qp * 9 + c * 3 + d] * fabs(Dphi[(qp * nd + a) * 3 + d]);
            F1locmag[(li * nd + a) * dim + c] = mg;
          }
      }
      if (FTw) {
        for (int j = 0; j < ne; ++j) {
          double s = 0.0;
          for (int a = 0; a < nd; ++a)
            for (int c = 0; c < dim; ++c) s += FK[(a * 3 + c) * ne + j] * Wl[c * nd + a];
          FTw[K * ne + j] = s;
        }
      }
      if (FTwmag) {
        for (int j = 0; j < ne; ++j) {
          double mg = 0.0;
          for (int qp = 0; qp < nq; ++qp) {
            double inner = 0.0;
            for (int c = 0; c < dim; ++c)
              for (int d = 0; d < dim; ++d) {
                double gm = 0.0;
                for (int a = 0; a < nd; ++a) gm += fabs(Wl[c * nd + a] * Dphi[(qp * nd + a) * 3 + d]);
                inner += Smag[qp * 9 + c * 3 + d] * gm;
              }
            mg += fabs(psi[qp * ne + j]) * inner;
          }
          FTwmag[K * ne + j] = mg;
        }
      }
    }
#pragma omp critical
    {
      g_rot += t_rot; g_calls += t_calls; g_fallback += t_fallback;
      t_rot = 0; t_calls = 0; t_fallback = 0;
      if (my_nan) any_nan = 1;
      if (dt_less(my_dt, dt_min)) dt_min = my_dt;
      if (my_bad < bad) bad = my_bad;
    }
    free(Xl); free(gx); free(gx0); free(eqv); free(S); free(Smag); free(FK);
  }
  /* step 5: serial assembly in ascending element order */
  if (F1loc) {
    memset(F1, 0, sizeof(double) * (size_t)dim * n_nodes);
    if (F1mag) memset(F1mag, 0, sizeof(double) * (size_t)dim * n_nodes);
    for (int64_t li = 0; li < n_list; ++li) {
      const int64_t K = elist ? elist[li] : li;
      const int32_t *en = elem_nodes + K * nd;
      for (int a = 0; a < nd; ++a)
        for (int c = 0; c < dim; ++c) {
          F1[(int64_t)c * n_nodes + en[a]] += F1loc[(li * nd + a) * dim + c];
          if (F1mag) F1mag[(int64_t)c * n_nodes + en[a]] += F1locmag[(li * nd + a) * dim + c];
        }
    }
  }
  free(F1loc); free(F1locmag); free(Dphi); free(psi);
  if (dt) *dt = any_nan ? NAN : dt_min;
  if (first_bad) *first_bad = bad == INT64_MAX ? -1 : bad;
  if (bad != INT64_MAX) return 4;
  if (any_nan) return 5;
  return 0;
}

/* ---------------------------------------------------------------- ROM (S7, S9) */
/* Lift (PAPER Eq. discretesolrepresentation):
 *   out[r][b] = os[r][b or broadcast] + sum_k Phi[r][k] Y[k][b], ascending k. */
void oracle_lift(int64_t rows, int n, int B, const double *Phi, const double *os, int os_batched,
                 const double *Y, double *out) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < rows; ++r)
    for (int b = 0; b < B; ++b) {
      double s = 0.0;
      for (int k = 0; k < n; ++k) s += Phi[r * n + k] * Y[(int64_t)k * B + b];
      out[r * B + b] = (os_batched ? os[r * B + b] : os[r]) + s;
    }
}

/* Projection (PAPER Eq. sol-ls-hyper): r[i][b] = sum_s P[i][s] f[s][b]. */
void oracle_project(int n, int64_t s_rows, int B, const double *P, const double *f, double *r) {
#pragma omp parallel for schedule(static)
  for (int i = 0; i < n; ++i)
    for (int b = 0; b < B; ++b) {
      double acc = 0.0;
      for (int64_t s = 0; s < s_rows; ++s) acc += P[(int64_t)i * s_rows + s] * f[s * B + b];
      r[(int64_t)i * B + b] = acc;
    }
}

/* exported helpers for the pins */
double oracle_det(int dim, const double *J9) {
  double J[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) J[i][j] = J9[i * 3 + j];
  return det_only(dim, J);
}

int oracle_sizeof_tab(void) { return (int)sizeof(otab); }
