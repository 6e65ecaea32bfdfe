// force3d.cuh -- the corner-force kernel for 3D hexahedra (Q2/Q1 with 4^3 points: C2, C4;
// Q3/Q2 with 6^3 points: C3).  One thread per Gauss point, one element at a time per CTA.
//
// Same stages and arithmetic as force_kernel (contract parts bit-identical: forward_point,
// pointwise), restructured after the r01 v4 profile (profiles/r01_v4_c2_force_full.txt:
// issue slots 65 % busy with FP64 only 37 % of instructions; index decoding in the
// contraction loops was the largest integer cost, gather latency 16 % of stall samples):
//   * PERSISTENT CTAs: CTA c evaluates units c, c + gridDim.x, ...; each lane's stage
//     tasks are decoded once, outside the unit loop (no div/mod in the loops);
//   * each contraction stage maps one lane to one (q, a, a) pencil and loops over the
//     fields at compile time, computing the B and G contractions (and all three stage-2
//     kinds) of a pencil together;
//   * two-stage software pipeline for the gather: while unit i computes, unit i+1's dofs
//     are copied into the other shared buffer with cp.async and unit i+2's node ids,
//     unit i+1's masses / gamma / slots are loaded into registers;
//   * dt keys are min'd per thread across units (full mode) and reduced once per CTA.
// Lane roles (NT = 32-rounded point count; "hi" lanes are the top lanes of the CTA):
//   S1   lane (q1,a2,a3) < Q N^2     : U_B/U_G[fc][q1][a2][a3] = sum_a1 B/G[q1][a1] X[fc][a1,a2,a3]
//        hi lane (q1,j2,j3)           : E1[q1][j2][j3] = sum_j1 Bl[q1][j1] E[j1,j2,j3]
//   S2   lane (q1,q2,a3) < Q^2 N     : d/dxi1: B[q2].U_G, d/dxi2: G[q2].U_B, d/dxi3: B[q2].U_B
//        hi lane (q1,q2,j3)           : E2[q1][q2][j3] = sum_j2 Bl[q2][j2] E1[q1][j2][j3]
//   S2b  lane = point                 : contract a3 (forward_point), S3 pointwise
//   S4a  lane (q1,q2,a3) < Q^2 N     : T[dl][c][q1][q2][a3] = sum_q3 (dl==2 ? G : B)[q3][a3] S[c][dl]
//        hi lane (q1,q2,j3)           : f1[q1][q2][j3] = sum_q3 Bl[q3][j3] A
//   S4b  lane (q1,a2,a3) < Q N^2     : W1 = sum_q2 B[q2][a2] T0 ; W23 = sum_q2 G[q2][a2] T1 + B[q2][a2] T2
//        hi lane (q1,j2,j3)           : f2 = sum_q2 Bl[q2][j2] f1
//   S4c  lane a < N^3                 : F1[c][a] = sum_q1 G[q1][a1] W1 + B[q1][a1] W23 -> slot
//        hi lane j < M^3              : FTw[j] = sum_q1 Bl[q1][j1] f2
#pragma once

#include "force_kernel.cuh"

namespace hk {

__device__ __forceinline__ void cp_async8(double *dst, const double *src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

__device__ __forceinline__ int opaque_tid() {
  int t;
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(t));
  return t;
}

#ifndef F3D_MINB
#define F3D_MINB 10
#endif

template <int K, int Q, int NF>
struct G3 {
  using G = Geo<3, K, Q, NF>;
  static constexpr int N = K + 1, M = K, ND = N * N * N, NE = M * M * M, NQ = Q * Q * Q;
  static constexpr int NT = ((NQ + 31) / 32) * 32;
  static constexpr int XE = NF * 3 * ND + NE;  // gathered doubles per unit (one buffer)
  static constexpr int TABD = G::TABD;
  static constexpr int WORK = G::WORK;
  static constexpr size_t SMEM = sizeof(double) * (size_t)(TABD + 2 * XE + WORK);
  // occupancy target (registers): ~96/thread for Q=4 (10 CTAs of 64); Q=6: 2 x 224 threads
  // (~144 registers: the 3 x 224 budget of 80 registers spilled heavily)
  static constexpr int MINB = NT >= 224 ? 2 : F3D_MINB;
};

// The exact IEEE re-run of one point (rare: a fast-path range check failed), out of line so
// that its ~1 500 instructions do not sit inside the unit loop's instruction footprint.
template <int K, int Q, int NF, bool VISC, bool HAS_W>
__device__ __noinline__ void rerun_point_ieee(const double *sB, const double *sG, const double *sBl,
                                              const double *Wk, int q1i, int q2i, int q3i,
                                              double mq, double gam, double wq, PhysIn ph,
                                              PointOut *po) {
  double J[3][3], Gv[3][3], Gw[3][3], eq = 0.0;
  forward_point<3, K, Q, NF, true>(sB, sG, sBl, Wk, q1i, q2i, q3i, J, Gv, Gw, eq);
  if (!HAS_W) {
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int d = 0; d < 3; ++d) Gw[c][d] = 0.0;
  }
  ArithIeee ai;
  pointwise<3, VISC, HAS_W, false>(ai, J, Gv, Gw, eq, mq, gam, wq, ph, *po);
}

template <int K, int Q, bool VISC, int MODE, bool BATCHED, bool HAS_W>
__global__ void __launch_bounds__(G3<K, Q, HAS_W ? 3 : 2>::NT, G3<K, Q, HAS_W ? 3 : 2>::MINB)
force3d_kernel(const Params P) {
  constexpr int NF = HAS_W ? 3 : 2;
  using L = G3<K, Q, NF>;
  using G = typename L::G;
  constexpr int N = L::N, M = L::M, ND = L::ND, NE = L::NE, NQ = L::NQ, NT = L::NT, XE = L::XE;
  extern __shared__ __align__(16) double smem[];
  double *sW = smem;              // [Q]
  double *sB = sW + Q;            // [Q][N]
  double *sG = sB + Q * N;        // [Q][N]
  double *sBl = sG + Q * N;       // [Q][M]
  double *Xb = smem + L::TABD;    // [2][XE]
  double *Wk = Xb + 2 * XE;       // work region
  double *S1b = Wk;                                   // [NF*3][2][Q][N][N]
  double *S2b = Wk + NF * 3 * 2 * G::S1;              // [NF*3][3][Q][Q][N]
  double *E1b = S2b + NF * 3 * 3 * G::S2;             // [Q][M][M]
  double *E2b = E1b + G::E1;                          // [Q][Q][M]
  double *Ss = Wk;                                    // [9][NQ]   (backward, aliases forward)
  double *As = Ss + 9 * NQ;                           // [NQ]
  double *Tb = As + NQ;                               // [3][3][Q][Q][N]
  double *Wb = Tb + G::TB;                            // [2][3][Q][N][N]
  double *F1b = Wb + G::WB;                           // [Q][Q][M]
  double *F2b = F1b + G::F1B;                         // [Q][M][M]
  __shared__ unsigned long long skey[NT / 32];

  const int lt = threadIdx.x;
  const int B = BATCHED ? P.B : 1;
  for (int i = lt; i < Q; i += NT) sW[i] = P.tab_w[i];
  for (int i = lt; i < Q * N; i += NT) { sB[i] = P.tab_B[i]; sG[i] = P.tab_G[i]; }
  for (int i = lt; i < Q * M; i += NT) sBl[i] = P.tab_Bl[i];

  // ---- per-lane task decode.  The decodes are cheap (constant divisors); they are
  // re-derived inside each stage from an opaque copy of the thread index so that the
  // compiler does not hoist ~20 loop-invariant integers into registers for the whole
  // unit loop (it spilled them instead of rematerialising).
  const int lq = lt < NQ ? lt : 0;                       // point (pad lanes: a copy of 0)
  const int q1i = lq % Q, q2i = (lq / Q) % Q, q3i = lq / (Q * Q);
  constexpr int nE1 = Q * M * M, nE2 = Q * Q * M;
  const int U = P.n_units;
  // unit u -> (element l, instance b) = (u / B, u % B) without an integer division (it was
  // ~3 % of the instructions and stall samples on C4): for u < 2^24 (exact in float) the
  // float quotient is off by at most one; the correction loops make it exact for any u.
  const float invB = 1.0f / (float)B;
  auto unit_parts = [&](int u, int &l, int &b) {
    if (BATCHED) {
      int q = __float2int_rz(__int2float_rz(u) * invB);
      int r = u - q * B;
      while (r < 0) { --q; r += B; }
      while (r >= B) { ++q; r -= B; }
      l = q;
      b = r;
    } else {
      l = u;
      b = 0;
    }
  };
  // gather issue for unit u (lanes < ND: their node's NF*3 values; next NE lanes: e)
  auto issue_gather = [&](int u, int nid, double *dst) {
    int l, b;
    unit_parts(u, l, b);
    if (lt < ND) {
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        const double *src = f == 0 ? P.x : (f == 1 ? P.v : P.w);
#pragma unroll
        for (int c = 0; c < 3; ++c)
          cp_async8(dst + (f * 3 + c) * ND + lt, src + ((int64_t)c * P.ld_nodes + nid) * B + b);
      }
    } else if (lt < ND + NE) {
      const int j = lt - ND;
      cp_async8(dst + NF * 3 * ND + j, P.e + ((int64_t)l * NE + j) * B + b);
    }
  };
  auto node_id = [&](int u) -> int {
    if (lt >= ND || u >= U) return 0;
    int l, b;
    unit_parts(u, l, b);
    return __ldg(P.elem_nodes + (int64_t)l * ND + lt);
  };
  struct Scal { double mq, gam; int gid, slot; };
  auto scalars = [&](int u) {
    Scal s{1.0, 1.4, 0, -1};
    if (u >= U) return s;
    int l, b;
    unit_parts(u, l, b);
    s.gid = P.elem_gid ? __ldg(P.elem_gid + l) : l;
    s.mq = __ldg(P.mq + (int64_t)s.gid * NQ + lq);
    s.gam = __ldg(P.gamma + s.gid);
    if (MODE == MODE_FORCE && lt < ND) s.slot = __ldg(P.slot + (int64_t)l * ND + lt);
    return s;
  };

  // ---- pipeline prologue
  int u = blockIdx.x;
  if (u < U) issue_gather(u, node_id(u), Xb);
  cp_async_commit();
  int nid_next = node_id(u + gridDim.x);
  Scal sc = scalars(u);
  unsigned long long kmin = ~0ull;

  for (int it = 0; u < U; ++it, u += gridDim.x) {
    const double *X = Xb + (it & 1) * XE;
    const int un = u + gridDim.x;
    if (un < U) issue_gather(un, nid_next, Xb + ((it + 1) & 1) * XE);
    cp_async_commit();
    nid_next = node_id(un + gridDim.x);
    const Scal scn = scalars(un);
    cp_async_wait1();
    __syncthreads();  // B0: this unit's dofs visible; previous unit's buffers free
    int l, b;
    unit_parts(u, l, b);

    // ---- S1: contract a1 (and E: j1)
    if (const int t = opaque_tid(); t < Q * N * N) {
      const int s1_q = t % Q, s1_a2 = (t / Q) % N, s1_a3 = t / Q / N;
      double tb[N], tg[N];
#pragma unroll
      for (int a = 0; a < N; ++a) { tb[a] = sB[s1_q * N + a]; tg[a] = sG[s1_q * N + a]; }
#pragma unroll
      for (int fc = 0; fc < NF * 3; ++fc) {
        const double *src = X + fc * ND + (s1_a3 * N + s1_a2) * N;
        double ub = tb[0] * src[0], ug = tg[0] * src[0];
#pragma unroll
        for (int a1 = 1; a1 < N; ++a1) {
          ub = __fma_rn(tb[a1], src[a1], ub);
          ug = __fma_rn(tg[a1], src[a1], ug);
        }
        S1b[((fc * 2 + 0) * Q + s1_q) * N * N + s1_a2 * N + s1_a3] = ub;
        S1b[((fc * 2 + 1) * Q + s1_q) * N * N + s1_a2 * N + s1_a3] = ug;
      }
    }
    if (const int e1 = opaque_tid() - (NT - nE1); e1 >= 0) {
      const int e1_q = e1 % Q, e1_j2 = (e1 / Q) % M, e1_j3 = e1 / Q / M;
      const double *tab = sBl + e1_q * M;
      const double *src = X + NF * 3 * ND + (e1_j3 * M + e1_j2) * M;
      double acc = tab[0] * src[0];
#pragma unroll
      for (int j1 = 1; j1 < M; ++j1) acc = __fma_rn(tab[j1], src[j1], acc);
      E1b[(e1_q * M + e1_j2) * M + e1_j3] = acc;
    }
    __syncthreads();  // B1

    // ---- S2: contract a2 (and E: j2)
    if (const int t = opaque_tid(); t < Q * Q * N) {
      const int s2_q1 = t % Q, s2_q2 = (t / Q) % Q, s2_a3 = t / Q / Q;
      double tb[N], tg[N];
#pragma unroll
      for (int a = 0; a < N; ++a) { tb[a] = sB[s2_q2 * N + a]; tg[a] = sG[s2_q2 * N + a]; }
#pragma unroll
      for (int fc = 0; fc < NF * 3; ++fc) {
        const double *uB = S1b + ((fc * 2 + 0) * Q + s2_q1) * N * N + s2_a3;
        const double *uG = S1b + ((fc * 2 + 1) * Q + s2_q1) * N * N + s2_a3;
        double d1 = tb[0] * uG[0], d2 = tg[0] * uB[0], d3 = tb[0] * uB[0];
#pragma unroll
        for (int a2 = 1; a2 < N; ++a2) {
          d1 = __fma_rn(tb[a2], uG[a2 * N], d1);
          d2 = __fma_rn(tg[a2], uB[a2 * N], d2);
          d3 = __fma_rn(tb[a2], uB[a2 * N], d3);
        }
        const int o = (s2_q1 * Q + s2_q2) * N + s2_a3;
        S2b[(fc * 3 + 0) * Q * Q * N + o] = d1;
        S2b[(fc * 3 + 1) * Q * Q * N + o] = d2;
        S2b[(fc * 3 + 2) * Q * Q * N + o] = d3;
      }
    }
    if (const int e2 = opaque_tid() - (NT - nE2); e2 >= 0) {
      const int e2_q1 = e2 % Q, e2_q2 = (e2 / Q) % Q, e2_j3 = e2 / Q / Q;
      const double *tab = sBl + e2_q2 * M;
      const double *src = E1b + e2_q1 * M * M + e2_j3;
      double acc = tab[0] * src[0];
#pragma unroll
      for (int j2 = 1; j2 < M; ++j2) acc = __fma_rn(tab[j2], src[j2 * M], acc);
      E2b[(e2_q1 * Q + e2_q2) * M + e2_j3] = acc;
    }
    __syncthreads();  // B2

    // ---- S2b + S3: the point (fast pass, exact IEEE re-run where needed)
    double J[3][3], Gv[3][3], Gw[3][3], eq = 0.0;
    forward_point<3, K, Q, NF, true>(sB, sG, sBl, Wk, q1i, q2i, q3i, J, Gv, Gw, eq);
    if (!HAS_W) {
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int d = 0; d < 3; ++d) Gw[c][d] = 0.0;
    }
    double wq = sW[q1i] * sW[q2i];
    wq = wq * sW[q3i];
    const PhysIn ph{P.q1, P.q2, P.alpha, P.alpha_mu};
    PointOut po;
    {
      ArithFast af;
      pointwise<3, VISC, HAS_W, true, ArithFast, true>(af, J, Gv, Gw, eq, sc.mq, sc.gam, wq, ph, po);
      count_rerun(!af.ok);
      if (!af.ok) rerun_point_ieee<K, Q, NF, VISC, HAS_W>(sB, sG, sBl, Wk, q1i, q2i, q3i, sc.mq,
                                                           sc.gam, wq, ph, &po);
    }
    // ---- S6 dt: flags; key min per thread (full) or per unit (batched)
    const bool pt = lt < NQ;
    if (MODE == MODE_FORCE && P.S_store && pt) {
      const int64_t si = s_index(P, u, l, b);
      if (si >= 0) {
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int d = 0; d < 3; ++d) P.S_store[(si * 9 + c * 3 + d) * NQ + lt] = po.S[c][d];
      }
    }
    if (pt) {
      if (!(po.det > 0.0)) atomicMin(&P.st[b].first_bad, (unsigned long long)sc.gid);
      if (isnan(po.dtq)) atomicOr(&P.st[b].nan_flag, 1u);
      else {
        const unsigned long long k = dt_key(po.dtq);
        kmin = k < kmin ? k : kmin;
      }
    }
    if (BATCHED) {
      unsigned long long key = kmin;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, key, off);
        key = o < key ? o : key;
      }
      if ((lt & 31) == 0 && key != ~0ull) atomicMin(&P.st[b].dt_key, key);
      kmin = ~0ull;
    }
    __syncthreads();  // B3: forward buffers dead

    if (MODE == MODE_FORCE) {
      // ---- S4a: contract q3 (and A: q3)
      if (pt) {
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int d = 0; d < 3; ++d) Ss[(c * 3 + d) * NQ + lt] = po.S[c][d];
        As[lt] = po.A;
      }
      __syncthreads();  // B4
      if (const int t = opaque_tid(); t < Q * Q * N) {
        const int s2_q1 = t % Q, s2_q2 = (t / Q) % Q, s2_a3 = t / Q / Q;
        double tb[Q], tg[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) { tb[q] = sB[q * N + s2_a3]; tg[q] = sG[q * N + s2_a3]; }
        const double *src0 = Ss + s2_q1 + Q * s2_q2;
#pragma unroll
        for (int dl = 0; dl < 3; ++dl)
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const double *src = src0 + (c * 3 + dl) * NQ;
            double acc = 0.0;
#pragma unroll
            for (int q3 = 0; q3 < Q; ++q3) acc = __fma_rn(dl == 2 ? tg[q3] : tb[q3], src[q3 * Q * Q], acc);
            Tb[(((dl * 3 + c) * Q + s2_q1) * Q + s2_q2) * N + s2_a3] = acc;
          }
      }
      if (const int e2 = opaque_tid() - (NT - nE2); e2 >= 0) {  // f1[q1][q2][j3]
        const int e2_q1 = e2 % Q, e2_q2 = (e2 / Q) % Q, e2_j3 = e2 / Q / Q;
        double acc = 0.0;
#pragma unroll
        for (int q3 = 0; q3 < Q; ++q3)
          acc = __fma_rn(sBl[q3 * M + e2_j3], As[e2_q1 + Q * e2_q2 + Q * Q * q3], acc);
        F1b[(e2_q1 * Q + e2_q2) * M + e2_j3] = acc;
      }
      __syncthreads();  // B5
      // ---- S4b: contract q2
      if (const int t = opaque_tid(); t < Q * N * N) {
        const int s1_q = t % Q, s1_a2 = (t / Q) % N, s1_a3 = t / Q / N;
        double tb[Q], tg[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) { tb[q] = sB[q * N + s1_a2]; tg[q] = sG[q * N + s1_a2]; }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double *t0 = Tb + ((0 * 3 + c) * Q + s1_q) * Q * N + s1_a3;
          const double *t1 = Tb + ((1 * 3 + c) * Q + s1_q) * Q * N + s1_a3;
          const double *t2 = Tb + ((2 * 3 + c) * Q + s1_q) * Q * N + s1_a3;
          double w1 = 0.0, w23 = 0.0;
#pragma unroll
          for (int q2 = 0; q2 < Q; ++q2) {
            w1 = __fma_rn(tb[q2], t0[q2 * N], w1);
            w23 = __fma_rn(tg[q2], t1[q2 * N], w23);
            w23 = __fma_rn(tb[q2], t2[q2 * N], w23);
          }
          Wb[((0 * 3 + c) * Q + s1_q) * N * N + s1_a2 * N + s1_a3] = w1;
          Wb[((1 * 3 + c) * Q + s1_q) * N * N + s1_a2 * N + s1_a3] = w23;
        }
      }
      if (const int e1 = opaque_tid() - (NT - nE1); e1 >= 0) {  // f2[q1][j2][j3]
        const int e1_q = e1 % Q, e1_j2 = (e1 / Q) % M, e1_j3 = e1 / Q / M;
        double acc = 0.0;
#pragma unroll
        for (int q2 = 0; q2 < Q; ++q2)
          acc = __fma_rn(sBl[q2 * M + e1_j2], F1b[(e1_q * Q + q2) * M + e1_j3], acc);
        F2b[(e1_q * M + e1_j2) * M + e1_j3] = acc;
      }
      __syncthreads();  // B6
      // ---- S4c: contract q1, outputs
      if (u < U) {
        if (const int t = opaque_tid(); t < ND) {
          const int na1 = t % N, na2 = (t / N) % N, na3 = t / N / N;
          double val[3];
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            double acc = 0.0;
#pragma unroll
            for (int q1 = 0; q1 < Q; ++q1) {
              acc = __fma_rn(sG[q1 * N + na1], Wb[((0 * 3 + c) * Q + q1) * N * N + na2 * N + na3], acc);
              acc = __fma_rn(sB[q1 * N + na1], Wb[((1 * 3 + c) * Q + q1) * N * N + na2 * N + na3], acc);
            }
            val[c] = acc;
          }
          if (sc.slot >= 0) {
#pragma unroll
            for (int c = 0; c < 3; ++c) P.evec[((int64_t)sc.slot * 3 + c) * B + b] = val[c];
          }
        }
        if (const int fe = opaque_tid() - (NT - NE); fe >= 0) {
          const int fe_j1 = fe % M, fe_j2 = (fe / M) % M, fe_j3 = fe / M / M;
          const int row = P.ftw_row ? __ldg(P.ftw_row + l) : l;
          if (row >= 0) {
            double acc = 0.0;
#pragma unroll
            for (int q1 = 0; q1 < Q; ++q1)
              acc = __fma_rn(sBl[q1 * M + fe_j1], F2b[(q1 * M + fe_j2) * M + fe_j3], acc);
            P.FTw[((int64_t)row * NE + fe) * B + b] = acc;
          }
        }
      }
    }
    sc = scn;
  }

  if (!BATCHED) {  // one dt atomic per CTA
    unsigned long long key = kmin;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const unsigned long long o = __shfl_xor_sync(0xffffffffu, key, off);
      key = o < key ? o : key;
    }
    if ((lt & 31) == 0) skey[lt >> 5] = key;
    __syncthreads();
    if (lt == 0) {
      unsigned long long k = skey[0];
#pragma unroll
      for (int i = 1; i < NT / 32; ++i) k = skey[i] < k ? skey[i] : k;
      if (k != ~0ull) atomicMin(&P.st[0].dt_key, k);
    }
  }
  pdl_trigger();
}

}  // namespace hk
