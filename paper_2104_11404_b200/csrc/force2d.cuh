// force2d.cuh -- the corner-force kernel specialised for 2D Q2/Q1 with 4x4 Gauss points
// (BASELINE configs C0 and C1: 16 points per element, 9 H1 nodes, 4 L2 dofs).
//
// ONE THREAD PER ELEMENT (per unit in batched mode).  A 2D Q2 element is small enough that
// every intermediate of the sum-factorised contractions stays in the thread's registers,
// so the element needs no shared-memory exchange at all.  The earlier element-per-
// half-warp layout was bound by shared-memory wavefronts (9.0 M per C1 call, ~32 us of a
// 47 us kernel: profiles/r01_v5_c1_force_full.txt); here shared memory holds only each
// thread's own gathered dofs and F1 accumulators, in a lane-interleaved layout that is
// conflict-free (consecutive threads -> consecutive 8-byte words).
//
// Per element (canonical contract order, DESIGN A.2-A.4; identical values to force_kernel):
//   gather   x, v (, w) at the 9 nodes -> shared [36 (54)][NT];  e (4) -> registers
//   for q1 = 0..3:                                                  (rolled loop)
//     U_B/U_G[fc][a2] = sum_a1 B/G[q1][a1] X[fc][a1,a2]              (registers, 24 (36))
//     E1[j2]          = sum_j1 Bl[q1][j1] E[j1,j2]
//     for q2 = 0..3:                                                 (rolled)
//       J, gradhat v (, w) = B/G[q2] . U ; e_q = Bl[q2] . E1
//       S3 pointwise (fast div/sqrt) -> S_q, A_q, dt_q
//       T[c][d][a2] += (d ? G : B)[q2][a2] S[c][d] ;  f1[j2] += Bl[q2][j2] A   (S4, q2 stage)
//     (if a fast path left its range for any of the 4 points: redo the q2 loop with IEEE ops)
//     F1[c][a1,a2] += G[q1][a1] T[c][0][a2] + B[q1][a1] T[c][1][a2]           (S4, q1 stage)
//     FTw[j1,j2]   += Bl[q1][j1] f1[j2]
//   F1 -> assembly slots (evec), FTw -> element-local output; dt: warp min, 1 atomic / CTA
// The 1D tables live in __constant__ memory (c_t24, filled at context creation).
#pragma once

#include "force_kernel.cuh"

namespace hk {

// (Tab24 / c_t24 are defined in force_kernel.cuh, shared with the blocked 3D stages)

struct ColOut {
  double T[2][2][3];  // T[c][d][a2] of this q1
  double f1[2];
  unsigned long long kmin;
  bool tangled, nan;
};

// The q2 loop of one q1 column: forward last stage, pointwise, first backward stage.
constexpr int F2D_NT = 64;

// Threads per element (r02): TPE threads share an element's gathered dofs and take its q1
// columns in turn (q1 = sub, sub + TPE, ...); their F.1 / F^T.w column sums are combined in
// ascending sub at the end (fixed order).  TPE = 1 is the round-1 layout.
#ifndef F2D_TPE
#define F2D_TPE 1
#endif
constexpr int F2D_TPE_K = F2D_TPE;

// U rows of the xi_1 contraction (canonical order): ub = sum_a1 B[q1][a1] X[fc][a1,a2],
// ug = sum_a1 G[q1][a1] X[fc][a1,a2]; Xs is the thread's lane-interleaved dof column.
// gathered dofs are interleaved over the CTA's elements: stride F2D_NT / TPE
__device__ __forceinline__ void u_row(int q1, const double *Xs, int fc, int a2, double &ub,
                                      double &ug) {
  constexpr int XS = F2D_NT / F2D_TPE;
  const double x0 = Xs[(fc * 9 + a2 * 3 + 0) * XS];
  const double x1 = Xs[(fc * 9 + a2 * 3 + 1) * XS];
  const double x2 = Xs[(fc * 9 + a2 * 3 + 2) * XS];
  ub = c_t24.B[q1][0] * x0;
  ug = c_t24.G[q1][0] * x0;
  ub = __fma_rn(c_t24.B[q1][1], x1, ub);
  ug = __fma_rn(c_t24.G[q1][1], x1, ug);
  ub = __fma_rn(c_t24.B[q1][2], x2, ub);
  ug = __fma_rn(c_t24.G[q1][2], x2, ug);
}

#ifndef F2D_Q2_UNROLL
#define F2D_Q2_UNROLL 2
#endif
constexpr int F2D_Q2_UNROLL_K = F2D_Q2_UNROLL;
// unroll of the q1 column loop (1: rolled; the register budget caps it)
#ifndef F2D_Q1_UNROLL
#define F2D_Q1_UNROLL 1
#endif
constexpr int F2D_Q1_UNROLL_K = F2D_Q1_UNROLL;

// F2D_KEEP: how many of the (field, component) rows of U stay in registers across the q2
// loop (the position rows, 2); the velocity (and w) rows are re-contracted from the gathered
// dofs in shared memory at every point -- the same canonical FMA chain, so the same bits --
// trading ~27 FP64 instructions per point for ~24 registers, which removes the local-memory
// spills the all-register version had (they missed L1: profiles/r01_ab14_*).
#ifndef F2D_KEEP
#define F2D_KEEP 2
#endif

template <bool VISC, bool HAS_W, class AR>
__device__ __forceinline__ void column2d(AR &ar, int q1, const double (&UB)[6][3],
                                         const double (&UG)[6][3], const double *Xs,
                                         const double (&E1)[2],
                                         const double *__restrict__ mqp, double mq0,
                                         double &mq_next, double gam, const PhysIn &ph,
                                         ColOut &o, double *Sst) {
#pragma unroll
  for (int c = 0; c < 2; ++c)
#pragma unroll
    for (int d = 0; d < 2; ++d)
#pragma unroll
      for (int a2 = 0; a2 < 3; ++a2) o.T[c][d][a2] = 0.0;
  o.f1[0] = o.f1[1] = 0.0;
  o.kmin = ~0ull;
  o.tangled = o.nan = false;
  const double wq1 = c_t24.w[q1];
  // m_q is software-prefetched one point ahead (a rotating register, no indexed array):
  // the global load's latency hides behind the previous point's pointwise stage.  After
  // the last point mq_next holds m_q(q1 + 1, 0) (mqp[1]; a harmless re-read for q1 = 3).
  double mq_cur = mq0;
#pragma unroll (F2D_Q2_UNROLL_K)
  for (int q2 = 0; q2 < 4; ++q2) {
    const double mq = mq_cur;
    mq_cur = __ldg(q2 < 3 ? mqp + 4 * (q2 + 1) : mqp + (q1 + F2D_TPE_K < 4 ? F2D_TPE_K : 0));
    double J[3][3], Gv[3][3], Gw[3][3];
    constexpr int NF = HAS_W ? 3 : 2;
#pragma unroll
    for (int f = 0; f < NF; ++f)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int fc = f * 2 + c;
        double ugv[3], ubv[3];
#pragma unroll
        for (int a2 = 0; a2 < 3; ++a2) {
          if (fc < F2D_KEEP) {
            ugv[a2] = UG[fc][a2];
            ubv[a2] = UB[fc][a2];
          } else {
            u_row(q1, Xs, fc, a2, ubv[a2], ugv[a2]);
          }
        }
        double d0 = c_t24.B[q2][0] * ugv[0], d1 = c_t24.G[q2][0] * ubv[0];
#pragma unroll
        for (int a2 = 1; a2 < 3; ++a2) {
          d0 = __fma_rn(c_t24.B[q2][a2], ugv[a2], d0);
          d1 = __fma_rn(c_t24.G[q2][a2], ubv[a2], d1);
        }
        double *dst = f == 0 ? J[c] : (f == 1 ? Gv[c] : Gw[c]);
        dst[0] = d0;
        dst[1] = d1;
      }
    if (!HAS_W) {
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int d = 0; d < 3; ++d) Gw[c][d] = 0.0;
    }
    double eq = c_t24.Bl[q2][0] * E1[0];
    eq = __fma_rn(c_t24.Bl[q2][1], E1[1], eq);
    PointOut po;
    pointwise<2, VISC, HAS_W, false>(ar, J, Gv, Gw, eq, mq, gam, wq1 * c_t24.w[q2], ph, po);
    if (Sst) {  // stored S_q = w_q detJ sigma J^-T, [cd][q] with q = q1 + 4 q2
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int d = 0; d < 2; ++d) Sst[(c * 2 + d) * 16 + q1 + 4 * q2] = po.S[c][d];
    }
    o.tangled = o.tangled || !(po.det > 0.0);
    if (isnan(po.dtq)) o.nan = true;
    else {
      const unsigned long long k = dt_key(po.dtq);
      o.kmin = k < o.kmin ? k : o.kmin;
    }
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int a2 = 0; a2 < 3; ++a2) {
        o.T[c][0][a2] = __fma_rn(c_t24.B[q2][a2], po.S[c][0], o.T[c][0][a2]);
        o.T[c][1][a2] = __fma_rn(c_t24.G[q2][a2], po.S[c][1], o.T[c][1][a2]);
      }
    o.f1[0] = __fma_rn(c_t24.Bl[q2][0], po.A, o.f1[0]);
    o.f1[1] = __fma_rn(c_t24.Bl[q2][1], po.A, o.f1[1]);
  }
  mq_next = mq_cur;
}

template <int NF>
struct G2 {
  static constexpr int NT = F2D_NT;
  static constexpr int TPE = F2D_TPE;
  static constexpr int UPB = NT / TPE;   // elements (units) per CTA
  // per element: gathered dofs NF*2*9 + e 4; per thread: F1 column sums 18
  static constexpr size_t SMEM = sizeof(double) * (size_t)((NF * 2 * 9 + 4) * UPB + 18 * NT);
};

#ifndef F2D_MAXNREG
#define F2D_MAXNREG 128
#endif
template <bool VISC, int MODE, bool BATCHED, bool HAS_W>
__global__ void __maxnreg__(F2D_MAXNREG) force2d_kernel(const Params P) {
  constexpr int NF = HAS_W ? 3 : 2;
  constexpr int ND = 9, NE = 4, NQ = 16, NT = F2D_NT, TPE = F2D_TPE, UPB = NT / TPE;
  constexpr int NX = NF * 2 * ND;
  static_assert(NT % TPE == 0 && (TPE == 1 || TPE == 2 || TPE == 4), "F2D_TPE");
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x;
  // element slot e of the CTA and this thread's place among its element's TPE threads (the
  // TPE threads of an element are adjacent lanes)
  const int e = tid / TPE, sub = tid % TPE;
  double *Xs = smem + e;                        // [NX][UPB]  gathered x, v (, w) per element
  double *Es = smem + NX * UPB + e;             // [4][UPB]   e dofs
  double *Fs = smem + (NX + 4) * UPB + tid;     // [18][NT]   this thread's F1 column sums [c][a2][a1]
  __shared__ unsigned long long skey[NT / 32];

  const int g0 = blockIdx.x * UPB + e;
  const bool valid = g0 < P.n_units;
  const int g = valid ? g0 : P.n_units - 1;   // ragged tail: compute a copy, write nothing
  const int B = BATCHED ? P.B : 1;
  const int l = BATCHED ? g / B : g;
  const int b = BATCHED ? g % B : 0;
  const int gid = P.elem_gid ? __ldg(P.elem_gid + l) : l;
  const double gam = __ldg(P.gamma + gid);

  // --- S1 gather (the element's TPE threads split the nodes)
  {
#pragma unroll
    for (int a = sub; a < ND; a += TPE) {
      const int nd = __ldg(P.elem_nodes + (int64_t)l * ND + a);
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        const double *src = f == 0 ? P.x : (f == 1 ? P.v : P.w);
#pragma unroll
        for (int c = 0; c < 2; ++c)
          Xs[((f * 2 + c) * ND + a) * UPB] = __ldg(src + ((int64_t)c * P.ld_nodes + nd) * B + b);
      }
    }
  }
#pragma unroll
  for (int j = sub; j < NE; j += TPE) Es[j * UPB] = __ldg(P.e + ((int64_t)l * NE + j) * B + b);
  if (TPE > 1) __syncwarp();
  double FT[2][2];  // FTw[j1][j2] accumulators
#pragma unroll
  for (int j = 0; j < 2; ++j) FT[j][0] = FT[j][1] = 0.0;
  if (MODE == MODE_FORCE) {
#pragma unroll
    for (int k = 0; k < 18; ++k) Fs[k * NT] = 0.0;
  }
  const PhysIn ph{P.q1, P.q2, P.alpha, P.alpha_mu};
  unsigned long long kmin = ~0ull;
  bool tangled = false, nan = false;
  double *Sst = nullptr;
  if (MODE == MODE_FORCE && P.S_store && valid) {
    const int64_t si = s_index(P, g, l, b);
    if (si >= 0) Sst = P.S_store + si * 4 * NQ;
  }
  double mq0 = __ldg(P.mq + (int64_t)gid * NQ + sub);  // m_q(sub, 0); then prefetched point by point

#pragma unroll (F2D_Q1_UNROLL_K)
  for (int q1 = sub; q1 < 4; q1 += TPE) {
    // S2a: contract xi_1 for this q1 (canonical order)
    double UB[6][3], UG[6][3];
#pragma unroll
    for (int fc = 0; fc < NF * 2; ++fc)
#pragma unroll
      for (int a2 = 0; a2 < 3; ++a2) {
        if (fc < F2D_KEEP) u_row(q1, Xs, fc, a2, UB[fc][a2], UG[fc][a2]);
        else UB[fc][a2] = UG[fc][a2] = 0.0;  // unused: re-contracted per point
      }
    double E1[2];
#pragma unroll
    for (int j2 = 0; j2 < 2; ++j2) {
      const double acc = c_t24.Bl[q1][0] * Es[(j2 * 2 + 0) * UPB];
      E1[j2] = __fma_rn(c_t24.Bl[q1][1], Es[(j2 * 2 + 1) * UPB], acc);
    }
    const double *mqp = P.mq + (int64_t)gid * NQ + q1;  // m_q at (q1, q2) = mqp[4 q2]

    // S2b + S3 + S4 (q2 stage): fast pass; exact IEEE re-run of the column if needed
    ColOut co;
    {
      ArithFast af;
      double mqn;
      column2d<VISC, HAS_W>(af, q1, UB, UG, Xs, E1, mqp, mq0, mqn, gam, ph, co, Sst);
      if (!af.ok) {
        ArithIeee ai;
        column2d<VISC, HAS_W>(ai, q1, UB, UG, Xs, E1, mqp, mq0, mqn, gam, ph, co, Sst);
      }
      mq0 = mqn;
    }
    kmin = co.kmin < kmin ? co.kmin : kmin;
    tangled = tangled || co.tangled;
    nan = nan || co.nan;

    if (MODE == MODE_FORCE) {
      // S4, q1 stage (same FMA order as force_kernel's b2/b3: G.T0 then B.T1, ascending q1
      // within this thread's columns)
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int a2 = 0; a2 < 3; ++a2)
#pragma unroll
          for (int a1 = 0; a1 < 3; ++a1) {
            double acc = Fs[((c * 3 + a2) * 3 + a1) * NT];
            acc = __fma_rn(c_t24.G[q1][a1], co.T[c][0][a2], acc);
            acc = __fma_rn(c_t24.B[q1][a1], co.T[c][1][a2], acc);
            Fs[((c * 3 + a2) * 3 + a1) * NT] = acc;
          }
#pragma unroll
      for (int j1 = 0; j1 < 2; ++j1)
#pragma unroll
        for (int j2 = 0; j2 < 2; ++j2) FT[j1][j2] = __fma_rn(c_t24.Bl[q1][j1], co.f1[j2], FT[j1][j2]);
    }
  }

  // combine the element's TPE threads (sub 0 collects, ascending sub)
  if (TPE > 1) {
#pragma unroll
    for (int o = 1; o < TPE; o <<= 1) {
      const unsigned long long ko = __shfl_down_sync(0xffffffffu, kmin, o);
      const int fl = __shfl_down_sync(0xffffffffu, (int)tangled | ((int)nan << 1), o);
      kmin = ko < kmin ? ko : kmin;
      tangled = tangled || (fl & 1);
      nan = nan || (fl & 2);
    }
    if (MODE == MODE_FORCE) {
      __syncwarp();
      if (sub == 0) {
#pragma unroll
        for (int k = 0; k < 18; ++k) {
          double acc = Fs[k * NT];
#pragma unroll
          for (int t = 1; t < TPE; ++t) acc = acc + Fs[k * NT + t];
          Fs[k * NT] = acc;
        }
      }
#pragma unroll
      for (int j1 = 0; j1 < 2; ++j1)
#pragma unroll
        for (int j2 = 0; j2 < 2; ++j2) {
          double acc = FT[j1][j2];
          double part[TPE];
#pragma unroll
          for (int t = 1; t < TPE; ++t) part[t] = __shfl_down_sync(0xffffffffu, acc, t);
#pragma unroll
          for (int t = 1; t < TPE; ++t) acc = acc + part[t];
          FT[j1][j2] = acc;
        }
    }
  }

  // --- S6 dt: flags, warp min of keys, one atomic per CTA (per unit in batched mode)
  const bool lead = valid && sub == 0;
  if (lead) {
    if (tangled) atomicMin(&P.st[b].first_bad, (unsigned long long)gid);
    if (nan) atomicOr(&P.st[b].nan_flag, 1u);
  }
  if (!lead) kmin = ~0ull;
  if (BATCHED) {
    if (lead && kmin != ~0ull) atomicMin(&P.st[b].dt_key, kmin);
  } else {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const unsigned long long o = __shfl_xor_sync(0xffffffffu, kmin, off);
      kmin = o < kmin ? o : kmin;
    }
    if ((tid & 31) == 0) skey[tid >> 5] = kmin;
    __syncthreads();
    if (tid == 0) {
      unsigned long long k = skey[0];
#pragma unroll
      for (int i = 1; i < NT / 32; ++i) k = skey[i] < k ? skey[i] : k;
      if (k != ~0ull) atomicMin(&P.st[0].dt_key, k);
    }
  }

  // --- S5 outputs (the element's first thread)
  if (MODE == MODE_FORCE && lead) {
#pragma unroll
    for (int a = 0; a < ND; ++a) {
      const int s = __ldg(P.slot + (int64_t)l * ND + a);
      if (s >= 0) {
        P.evec[((int64_t)s * 2 + 0) * B + b] = Fs[((0 * 3 + a / 3) * 3 + a % 3) * NT];
        P.evec[((int64_t)s * 2 + 1) * B + b] = Fs[((1 * 3 + a / 3) * 3 + a % 3) * NT];
      }
    }
    const int row = P.ftw_row ? __ldg(P.ftw_row + l) : l;
    if (row >= 0) {
#pragma unroll
      for (int j = 0; j < NE; ++j) P.FTw[((int64_t)row * NE + j) * B + b] = FT[j & 1][j >> 1];
    }
  }
  pdl_trigger();
}

}  // namespace hk
