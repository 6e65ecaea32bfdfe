// force2d.cuh -- the corner-force kernel specialised for 2D Q2/Q1 with 4x4 Gauss points
// (BASELINE configs C0 and C1: 16 points per element, 9 H1 nodes, 4 L2 dofs).
//
// Same stages and the same arithmetic as force_kernel (the contract parts are bit
// identical: see forward_point / pointwise), but laid out for a 16-point element:
//   * one element per half-warp (lane = q1 + 4 q2), 8 elements per 128-thread CTA; all
//     of an element's shared-memory exchange stays inside its warp (__syncwarp, no CTA
//     barriers after the table load), so elements never wait on each other;
//   * every contraction stage is a fixed per-lane task with compile-time indices (no
//     runtime index decoding; the generic kernel spent ~25 % of its C1 instructions
//     there -- profiles/r01_v2_c1_force_full.txt);
//   * persistent CTAs with a two-stage software pipeline: the next round's dofs are
//     copied into a second shared buffer with cp.async (and the round after's node ids,
//     masses, gamma and slots are loaded into registers) while the current round computes;
//   * dt keys are min'd per thread across rounds and reduced once per CTA;
//   * S5/S6 in the programmatic dependent assembly launch (griddepcontrol).
// Lane roles per stage (u = element in CTA, lt = lane in element, q1 = lt&3, q2 = lt>>2):
//   S1  lane a < 9 gathers node a's x, v (, w); lanes 9..12 gather e_j.
//   S2a lane (q1, fc=q2 [+4]) : U_B/U_G[fc][q1][a2] = sum_a1 B/G[q1][a1] X[fc][a1,a2]
//       lane (q1, j2=q2 < 2)  : E1[q1][j2] = sum_j1 Bl[q1][j1] E[j1,j2]
//   S2b lane (q1, q2)         : J, gradhat v (, w), e_q at the point  (forward_point)
//   S3  lane (q1, q2)         : pointwise, fast pass + exact re-run   (pointwise)
//   S4a lane (q1, (c,d)=q2)   : T[c][d][q1][a2] = sum_q2' (d ? G : B)[q2'][a2] S[c][d](q1,q2')
//       lane (q1, j2=q2 < 2)  : f1[q1][j2] = sum_q2' Bl[q2'][j2] A(q1,q2')
//   S4b lane a < 9            : F1[c][a] = sum_q1 G[q1][a1] T[c][0][q1][a2] + B[q1][a1] T[c][1][q1][a2]
//       lanes 9..12           : FTw[j1,j2] = sum_q1 Bl[q1][j1] f1[q1][j2]
#pragma once

#include "force_kernel.cuh"

namespace hk {

template <int NF>
struct G2 {
  static constexpr int Q = 4, N = 3, M = 2, NQ = 16, ND = 9, NE = 4, EPB = 8, NT = 128;
  // per-element shared layout (doubles)
  static constexpr int U = 0;                         // [NF*2][2][4][3]
  static constexpr int E1 = U + NF * 2 * 2 * Q * N;   // [4][2]
  static constexpr int S = E1 + Q * M;                // [4][16]  (c*2+d, lane)
  static constexpr int A = S + 4 * NQ;                // [16]
  static constexpr int T = A + NQ;                    // [2][2][4][3]
  static constexpr int F1 = T + 2 * 2 * Q * N;        // [4][2]
  static constexpr int UNIT = F1 + Q * M;
  static constexpr int TABD = Q + Q * N * 2 + Q * M;  // w, B, G, Bl
  static constexpr int XE = NF * 2 * ND + NE;         // gathered dofs per unit
  static constexpr size_t SMEM = sizeof(double) * (size_t)(TABD + EPB * UNIT + EPB * 2 * XE);
};

__device__ __forceinline__ void cp_async8(double *dst, const double *src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// Persistent CTAs: CTA c handles rounds c, c + gridDim.x, ... (a round = 8 units, one per
// half-warp).  While round r is computed, round r+1's dofs are already in flight into
// the other shared buffer (cp.async) and round r+2's node ids into registers, so the
// gather latency (the top stall of the non-pipelined kernel: long_scoreboard, ~27 % of
// samples, profiles/r01_v4_c1_force_full.txt) overlaps compute.
template <bool VISC, int MODE, bool BATCHED, bool HAS_W>
__global__ void __launch_bounds__(128, 6) force2d_kernel(const Params P) {
  constexpr int NF = HAS_W ? 3 : 2;
  using L = G2<NF>;
  constexpr int Q = 4, N = 3, M = 2, NQ = 16, ND = 9, NE = 4, EPB = 8;
  constexpr int XE = NF * 2 * ND + NE;  // gathered doubles per unit (one buffer)
  extern __shared__ __align__(16) double smem[];
  double *sW = smem;              // [4]
  double *sB = sW + Q;            // [4][3]
  double *sG = sB + Q * N;        // [4][3]
  double *sBl = sG + Q * N;       // [4][2]
  __shared__ unsigned long long skey[EPB];

  const int tid = threadIdx.x;
  const int u = tid >> 4, lt = tid & 15;
  const int q1 = lt & 3, q2 = lt >> 2;
  const int B = BATCHED ? P.B : 1;
  const int R = (P.n_units + EPB - 1) / EPB;
  double *Us = smem + L::TABD + u * L::UNIT;
  double *Xb = smem + L::TABD + EPB * L::UNIT + u * 2 * XE;  // [2][XE] double buffer

  for (int i = tid; i < Q; i += 128) sW[i] = P.tab_w[i];
  for (int i = tid; i < Q * N; i += 128) { sB[i] = P.tab_B[i]; sG[i] = P.tab_G[i]; }
  for (int i = tid; i < Q * M; i += 128) sBl[i] = P.tab_Bl[i];

  auto unit_of = [&](int r) {
    const int g = r * EPB + u;
    return g < P.n_units ? g : P.n_units - 1;  // ragged tail: compute a copy, write nothing
  };
  auto node_id = [&](int r) -> int {
    if (lt >= ND || r >= R) return 0;
    const int g = unit_of(r);
    return __ldg(P.elem_nodes + (int64_t)(BATCHED ? g / B : g) * ND + lt);
  };
  auto issue_gather = [&](int r, int nid, double *dst) {
    const int g = unit_of(r);
    const int l = BATCHED ? g / B : g, b = BATCHED ? g % B : 0;
    if (lt < ND) {
#pragma unroll
      for (int f = 0; f < NF; ++f) {
        const double *src = f == 0 ? P.x : (f == 1 ? P.v : P.w);
#pragma unroll
        for (int c = 0; c < 2; ++c)
          cp_async8(dst + (f * 2 + c) * ND + lt, src + ((int64_t)c * P.ld_nodes + nid) * B + b);
      }
    } else if (lt < ND + NE) {
      const int j = lt - ND;
      cp_async8(dst + NF * 2 * ND + j, P.e + ((int64_t)l * NE + j) * B + b);
    }
  };
  struct Scal { double mq, gam; int slot, gid; };
  auto scalars = [&](int r) {
    Scal sc{1.0, 1.4, -1, 0};
    if (r >= R) return sc;
    const int g = unit_of(r);
    const int l = BATCHED ? g / B : g;
    sc.gid = P.elem_gid ? __ldg(P.elem_gid + l) : l;
    sc.mq = __ldg(P.mq + (int64_t)sc.gid * NQ + lt);
    sc.gam = __ldg(P.gamma + sc.gid);
    if (MODE == MODE_FORCE && lt < ND) sc.slot = __ldg(P.slot + (int64_t)l * ND + lt);
    return sc;
  };

  // pipeline prologue
  int r = blockIdx.x;
  issue_gather(r, node_id(r), Xb);
  cp_async_commit();
  int nid_next = node_id(r + gridDim.x);
  Scal sc = scalars(r);
  unsigned long long kmin = ~0ull;  // running dt key min of this thread (full mode)
  __syncthreads();                  // tables

  for (int it = 0; r < R; ++it, r += gridDim.x) {
    double *Xc = Xb + (it & 1) * XE;
    const int rn = r + gridDim.x;
    if (rn < R) issue_gather(rn, nid_next, Xb + ((it + 1) & 1) * XE);
    cp_async_commit();
    nid_next = node_id(rn + gridDim.x);
    const Scal scn = scalars(rn);
    cp_async_wait1();
    __syncwarp();

    const int g0 = r * EPB + u;
    const bool valid = g0 < P.n_units;
    const int g = valid ? g0 : P.n_units - 1;
    const int l = BATCHED ? g / B : g;
    const int b = BATCHED ? g % B : 0;

    // --- S2a: contract xi_1 (canonical order, DESIGN A.2)
    {
      const double b0 = sB[q1 * N + 0], b1 = sB[q1 * N + 1], b2 = sB[q1 * N + 2];
      const double g0_ = sG[q1 * N + 0], g1 = sG[q1 * N + 1], g2 = sG[q1 * N + 2];
#pragma unroll
      for (int fc = q2; fc < NF * 2; fc += 4) {
        const double *x = Xc + fc * ND;
#pragma unroll
        for (int a2 = 0; a2 < N; ++a2) {
          const double x0 = x[a2 * N + 0], x1 = x[a2 * N + 1], x2 = x[a2 * N + 2];
          double ub = b0 * x0, ug = g0_ * x0;
          ub = __fma_rn(b1, x1, ub); ug = __fma_rn(g1, x1, ug);
          ub = __fma_rn(b2, x2, ub); ug = __fma_rn(g2, x2, ug);
          Us[L::U + ((fc * 2 + 0) * Q + q1) * N + a2] = ub;
          Us[L::U + ((fc * 2 + 1) * Q + q1) * N + a2] = ug;
        }
      }
      if (q2 < M) {
        const double *e = Xc + NF * 2 * ND + q2 * M;
        double acc = sBl[q1 * M + 0] * e[0];
        acc = __fma_rn(sBl[q1 * M + 1], e[1], acc);
        Us[L::E1 + q1 * M + q2] = acc;
      }
    }
    __syncwarp();

    // --- S2b: the point's J, gradhat v (, gradhat w), e_q
    double J[3][3], Gv[3][3], Gw[3][3], eq = 0.0;
    forward_point<2, 2, 4, NF, true>(sB, sG, sBl, Us + L::U, q1, q2, 0, J, Gv, Gw, eq);
    if (!HAS_W) {
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int d = 0; d < 3; ++d) Gw[c][d] = 0.0;
    }

    // --- S3 pointwise: fast pass, exact IEEE re-run where a fast path left its range
    const double wq = sW[q1] * sW[q2];
    const PhysIn ph{P.q1, P.q2, P.alpha, P.alpha_mu};
    PointOut po;
    {
      ArithFast af;
      pointwise<2, VISC, HAS_W, true>(af, J, Gv, Gw, eq, sc.mq, sc.gam, wq, ph, po);
      if (!af.ok) {
        forward_point<2, 2, 4, NF, true>(sB, sG, sBl, Us + L::U, q1, q2, 0, J, Gv, Gw, eq);
        if (!HAS_W) {
#pragma unroll
          for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int d = 0; d < 3; ++d) Gw[c][d] = 0.0;
        }
        ArithIeee ai;
        pointwise<2, VISC, HAS_W, false>(ai, J, Gv, Gw, eq, sc.mq, sc.gam, wq, ph, po);
      }
    }

    // --- S6 dt: flags; keys min'd per thread across rounds (full mode) or per unit
    if (valid) {
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
      for (int off = 8; off > 0; off >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, key, off);
        key = o < key ? o : key;
      }
      if (lt == 0 && valid && key != ~0ull) atomicMin(&P.st[b].dt_key, key);
      kmin = ~0ull;
    }

    if (MODE == MODE_FORCE) {
      // --- S4a: contract q2 (backward)
      Us[L::S + 0 * NQ + lt] = po.S[0][0];
      Us[L::S + 1 * NQ + lt] = po.S[0][1];
      Us[L::S + 2 * NQ + lt] = po.S[1][0];
      Us[L::S + 3 * NQ + lt] = po.S[1][1];
      Us[L::A + lt] = po.A;
      __syncwarp();
      {
        const int cd = q2;            // (c, d) = (cd >> 1, cd & 1)
        const double *tab = (cd & 1) ? sG : sB;
        const double *src = Us + L::S + cd * NQ + q1;  // S[c][d](q1, q2') at src[4 q2']
        const double s0 = src[0], s1 = src[4], s2 = src[8], s3 = src[12];
#pragma unroll
        for (int a2 = 0; a2 < N; ++a2) {
          double acc = 0.0;
          acc = __fma_rn(tab[0 * N + a2], s0, acc);
          acc = __fma_rn(tab[1 * N + a2], s1, acc);
          acc = __fma_rn(tab[2 * N + a2], s2, acc);
          acc = __fma_rn(tab[3 * N + a2], s3, acc);
          Us[L::T + (cd * Q + q1) * N + a2] = acc;   // T[c][d][q1][a2], cd = c*2+d
        }
        if (q2 < M) {
          const double *a = Us + L::A + q1;
          double acc = 0.0;
#pragma unroll
          for (int k = 0; k < Q; ++k) acc = __fma_rn(sBl[k * M + q2], a[4 * k], acc);
          Us[L::F1 + q1 * M + q2] = acc;
        }
      }
      __syncwarp();

      // --- S4b: contract q1, outputs
      if (valid) {
        if (lt < ND) {
          const int a1 = lt % N, a2 = lt / N;
          double val[2];
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const double *t0 = Us + L::T + ((c * 2 + 0) * Q) * N + a2;
            const double *t1 = Us + L::T + ((c * 2 + 1) * Q) * N + a2;
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < Q; ++k) {
              acc = __fma_rn(sG[k * N + a1], t0[k * N], acc);
              acc = __fma_rn(sB[k * N + a1], t1[k * N], acc);
            }
            val[c] = acc;
          }
          if (sc.slot >= 0) {
            P.evec[((int64_t)sc.slot * 2 + 0) * B + b] = val[0];
            P.evec[((int64_t)sc.slot * 2 + 1) * B + b] = val[1];
          }
        } else if (lt < ND + NE) {
          const int j = lt - ND, j1 = j & 1, j2 = j >> 1;
          const int row = P.ftw_row ? __ldg(P.ftw_row + l) : l;
          if (row >= 0) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < Q; ++k) acc = __fma_rn(sBl[k * M + j1], Us[L::F1 + k * M + j2], acc);
            P.FTw[((int64_t)row * NE + j) * B + b] = acc;
          }
        }
      }
    }
    __syncwarp();  // this round's shared buffers are free for the next prefetch
    sc = scn;
  }

  if (!BATCHED) {
    // one dt atomic per CTA
    unsigned long long key = kmin;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const unsigned long long o = __shfl_xor_sync(0xffffffffu, key, off);
      key = o < key ? o : key;
    }
    if ((tid & 31) == 0) skey[tid >> 5] = key;
    __syncthreads();
    if (tid == 0) {
      unsigned long long k = skey[0];
#pragma unroll
      for (int i = 1; i < 4; ++i) k = skey[i] < k ? skey[i] : k;
      if (k != ~0ull) atomicMin(&P.st[0].dt_key, k);
    }
  }
  pdl_trigger();
}

}  // namespace hk
