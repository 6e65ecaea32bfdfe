// force2d_pl.cuh -- 2D Q2/Q1 corner-force kernel with ONE LANE PER GAUSS POINT and the
// xi_1 index q1 uniform over each warp (BASELINE configs C0/C1 shape: 16 points per element,
// 9 H1 nodes, 4 L2 dofs; PAPER Eq. fom, Eq. forceOneforceTv).
//
// Why: the one-thread-per-element kernel (force2d.cuh) gives C1 (65 536 elements) only
// 13.8 warps per SM at 128 registers, one wave, bound by the fixed latencies of the pointwise
// chains (profiles/r02_v4_c1_force_full.txt: FP64 pipe 41 %, `wait` the top stall).  Here a
// CTA of 4 warps evaluates 8 elements: warp w is Gauss column q1 = w, lane = q2 * 8 + e.
// Every table index of q1 is warp-uniform (constant-bank operands), the q2 rows are loaded
// into registers once, and a point's live state is small enough for 16x the threads.
//
// Per CTA (canonical contract order for everything dt depends on, DESIGN A.2-A.4):
//   S1  gather the 8 elements' x, v (9 nodes x 2 x 2) and e (4) into shared memory;
//   S2a lane (s, e) of warp q1 contracts xi_1 for field-component fc = s:
//       U_B[fc][a2] = sum_a1 B[q1][a1] X[fc][a1,a2], U_G likewise (the element kernel's u_row);
//       the four lanes of (q1, e) exchange their rows through shared memory (__syncwarp);
//   S2b J / gradhat v at (q1, q2 = s): B/G[q2] . U (same FMA chains as column2d); e_q;
//   S3  pointwise (fast div/sqrt, exact IEEE re-run of the lane if a fast path left its range);
//   S4  S_q, A_q to shared memory; barrier; warp (c, d) contracts q2 for lane (q1, e):
//       T[c][d][q1][a2] = sum_q2 (d ? G : B)[q2][a2] S_q[c][d]  (warps 0/1 also f1[j2]);
//       barrier; F1[c][a1,a2] = sum_q1 G[q1][a1] T[c][0] + B[q1][a1] T[c][1],
//       FTw[j1,j2] = sum_q1 Bl[q1][j1] f1[q1][j2]  (one output per thread);
//   S5  F1 to the assembly slots (evec), FTw element-local; S6 dt: warp REDUX min, CTA min,
//       one atomicMin per CTA.
// The backward sums run over q2 then q1 in ascending order (tolerance-only, A.5; the sums
// differ from force2d's only in association, within 1e-11 / 1e-12).
#pragma once

#include "force_kernel.cuh"

namespace hk {

struct G2L {
  static constexpr int NT = 128;     // 4 warps: q1 = warp
  static constexpr int UPB = 8;      // elements (units) per CTA
  static constexpr int XS = 37;      // per-element stride of the gathered dofs (36 + 1: banks)
  static constexpr int US = 26;      // per-(q1, e) stride of the U rows (24 + 2: LDS.128 banks)
  static constexpr int SQ = 40;      // q2 stride of the point-value block [cd][q2][q1*8 + e]
  // shared layout (doubles): tables 24 | X 8*37 | E 32 | U 4*8*26 | S 5*4*40 | T 12*32 | f1 2*32
  static constexpr int O_TB = 0, O_X = 24, O_E = O_X + UPB * XS, O_U = (O_E + 4 * UPB + 1) & ~1,
                       O_S = O_U + 4 * UPB * US, O_T = O_S + 5 * 4 * SQ, O_F = O_T + 12 * 32,
                       TOTAL = O_F + 2 * 32;
  static constexpr size_t SMEM = sizeof(double) * TOTAL;
};

#ifndef F2L_MINB
#define F2L_MINB 8
#endif

template <bool VISC, int MODE, bool BATCHED>
__global__ void __launch_bounds__(G2L::NT, F2L_MINB) force2d_pl_kernel(const Params P) {
  constexpr int ND = 9, NE = 4, NQ = 16, UPB = G2L::UPB;
  extern __shared__ __align__(16) double smem[];
  double *sTB = smem + G2L::O_TB;    // B[4][3], G[4][3] (per-lane indexed reads in the last pass)
  double *Xs = smem + G2L::O_X;      // [e][fc*9 + a]
  double *Es = smem + G2L::O_E;      // [j][e]
  double *Us = smem + G2L::O_U;      // [q1][e][fc*6 + 2*a2 + (0: U_B, 1: U_G)]
  double *Ss = smem + G2L::O_S;      // [cd (4: A)][q2][q1*8 + e]
  double *Ts = smem + G2L::O_T;      // [c][d][a2][q1*8 + e]
  double *F1s = smem + G2L::O_F;     // [j2][q1*8 + e]
  __shared__ unsigned long long skey[4];
  __shared__ int sflag[UPB];
  __shared__ int sslot[ND * UPB];   // assembly slot of (a, e), loaded with the node ids

  const int tid = threadIdx.x;
  const int w = tid >> 5, lane = tid & 31;
  const int B = BATCHED ? P.B : 1;
  const int64_t unit0 = (int64_t)blockIdx.x * UPB;

  // --- S1 gather: thread (a, eg) for a < 9 loads node a of element eg (4 values); 72..103 the
  // e dofs; 104..127 the tables and flags
  if (tid < 72 + 32) {
    const int eg = tid & 7;
    const int64_t g0 = unit0 + eg;
    const int64_t g = g0 < P.n_units ? g0 : P.n_units - 1;  // ragged tail: a copy, never written
    const int64_t l = BATCHED ? g / B : g;
    const int64_t b = BATCHED ? g - l * B : 0;
    if (tid < 72) {
      const int a = tid >> 3;
      const int nd = __ldg(P.elem_nodes + l * ND + a);
      // the slot of this node's F.1 partial: its latency hides behind the whole element here
      // instead of sitting in front of the final stores
      if (MODE == MODE_FORCE) sslot[tid] = __ldg(P.slot + l * ND + a);
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        const double *src = f == 0 ? P.x : P.v;
#pragma unroll
        for (int c = 0; c < 2; ++c)
          Xs[eg * G2L::XS + (f * 2 + c) * ND + a] = __ldg(src + ((int64_t)c * P.ld_nodes + nd) * B + b);
      }
    } else {
      const int j = (tid - 72) >> 3;
      Es[j * UPB + eg] = __ldg(P.e + (l * NE + j) * B + b);
    }
  } else {
    const int i = tid - 104;  // 24 threads: B and G tables
    sTB[i] = i < 12 ? (&c_t24.B[0][0])[i] : (&c_t24.G[0][0])[i - 12];
    if (i < UPB) sflag[i] = 0;
  }
  // this lane's point: (q1 = w, q2 = s) of element e
  const int s = lane >> 3, e = lane & 7;
  const int q1 = w;
  const int64_t gu0 = unit0 + e;
  const bool valid = gu0 < P.n_units;
  const int64_t gu = valid ? gu0 : P.n_units - 1;
  const int64_t lu = BATCHED ? gu / B : gu;
  const int64_t bu = BATCHED ? gu - lu * B : 0;
  const int gid = P.elem_gid ? __ldg(P.elem_gid + lu) : (int)lu;
  const double gam = __ldg(P.gamma + gid);
  const double mq = __ldg(P.mq + (int64_t)gid * NQ + q1 + 4 * s);
  double tB[3], tG[3], tBl[2];
#pragma unroll
  for (int a = 0; a < 3; ++a) { tB[a] = c_t24.B[s][a]; tG[a] = c_t24.G[s][a]; }
  tBl[0] = c_t24.Bl[s][0];
  tBl[1] = c_t24.Bl[s][1];
  __syncthreads();

  // --- S2a: this lane's U row (fc = s), the element kernel's u_row chain
  {
    const double *x = Xs + e * G2L::XS + s * ND;
    double *u = Us + (q1 * UPB + e) * G2L::US + s * 6;
#pragma unroll
    for (int a2 = 0; a2 < 3; ++a2) {
      const double x0 = x[a2 * 3 + 0], x1 = x[a2 * 3 + 1], x2 = x[a2 * 3 + 2];
      double ub = c_t24.B[q1][0] * x0;
      double ug = c_t24.G[q1][0] * x0;
      ub = __fma_rn(c_t24.B[q1][1], x1, ub);
      ug = __fma_rn(c_t24.G[q1][1], x1, ug);
      ub = __fma_rn(c_t24.B[q1][2], x2, ub);
      ug = __fma_rn(c_t24.G[q1][2], x2, ug);
      *reinterpret_cast<double2 *>(u + 2 * a2) = make_double2(ub, ug);
    }
  }
  // E1[j2] = Bl[q1] . E[., j2]; e_q = Bl[q2] . E1 (column2d's order)
  double eq;
  {
    double E1[2];
#pragma unroll
    for (int j2 = 0; j2 < 2; ++j2) {
      const double acc = c_t24.Bl[q1][0] * Es[(j2 * 2 + 0) * UPB + e];
      E1[j2] = __fma_rn(c_t24.Bl[q1][1], Es[(j2 * 2 + 1) * UPB + e], acc);
    }
    eq = tBl[0] * E1[0];
    eq = __fma_rn(tBl[1], E1[1], eq);
  }
  __syncwarp();

  // --- S2b: J (fc 0, 1) and gradhat v (fc 2, 3) at (q1, q2)
  double J[3][3], Gv[3][3], Gw[3][3];
  {
    const double *u = Us + (q1 * UPB + e) * G2L::US;
#pragma unroll
    for (int fc = 0; fc < 4; ++fc) {
      const double2 p0 = *reinterpret_cast<const double2 *>(u + fc * 6 + 0);
      const double2 p1 = *reinterpret_cast<const double2 *>(u + fc * 6 + 2);
      const double2 p2 = *reinterpret_cast<const double2 *>(u + fc * 6 + 4);
      double d0 = tB[0] * p0.y, d1 = tG[0] * p0.x;
      d0 = __fma_rn(tB[1], p1.y, d0);
      d1 = __fma_rn(tG[1], p1.x, d1);
      d0 = __fma_rn(tB[2], p2.y, d0);
      d1 = __fma_rn(tG[2], p2.x, d1);
      double *dst = fc < 2 ? J[fc] : Gv[fc - 2];
      dst[0] = d0;
      dst[1] = d1;
    }
  }
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int d = 0; d < 3; ++d) Gw[c][d] = 0.0;

  // --- S3 pointwise
  const PhysIn ph{P.q1, P.q2, P.alpha, P.alpha_mu};
  const double wq = c_t24.w[q1] * c_t24.w[s];
  PointOut po;
  {
    ArithFast af;
    pointwise<2, VISC, false, false>(af, J, Gv, Gw, eq, mq, gam, wq, ph, po);
    if (!af.ok) {
      ArithIeee ai;
      pointwise<2, VISC, false, false>(ai, J, Gv, Gw, eq, mq, gam, wq, ph, po);
    }
  }
  unsigned long long key = ~0ull;
  if (valid) {
    if (!(po.det > 0.0)) atomicMin(&P.st[bu].first_bad, (unsigned long long)gid);
    if (isnan(po.dtq)) sflag[e] = 1;  // (benign race: every writer stores 1)
    else key = dt_key(po.dtq);
  }

  if (MODE == MODE_FORCE) {
    if (P.S_store && valid) {  // stored S_q = w_q detJ sigma J^-T, [cd][q] with q = q1 + 4 q2
      const int64_t si = s_index(P, (int)gu, (int)lu, (int)bu);
      if (si >= 0) {
        double *Sst = P.S_store + si * 4 * NQ;
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int d = 0; d < 2; ++d) Sst[(c * 2 + d) * 16 + q1 + 4 * s] = po.S[c][d];
      }
    }
    const int col = q1 * UPB + e;
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int d = 0; d < 2; ++d) Ss[((c * 2 + d) * 4 + s) * G2L::SQ + col] = po.S[c][d];
    Ss[(4 * 4 + s) * G2L::SQ + col] = po.A;
  }

  // --- S6 dt: warp min of the keys; CTA min after the barrier; one atomic per CTA (per unit
  // in batched mode: the 8 units of a CTA may be different instances)
  if (BATCHED) {
    // min over the 16 points of each unit: lanes e, e+8, e+16, e+24 of the 4 warps
#pragma unroll
    for (int off = 8; off < 32; off <<= 1) {
      const unsigned long long o = __shfl_xor_sync(0xffffffffu, key, off);
      key = o < key ? o : key;
    }
  } else {
    key = warp_min_u64(key);
  }
  __shared__ unsigned long long skeyu[4][UPB];
  if (BATCHED) {
    if (s == 0) skeyu[w][e] = key;
  } else if (lane == 0) {
    skey[w] = key;
  }
  __syncthreads();
  if (BATCHED) {
    if (tid < UPB && unit0 + tid < P.n_units) {
      unsigned long long k = skeyu[0][tid];
#pragma unroll
      for (int i = 1; i < 4; ++i) k = skeyu[i][tid] < k ? skeyu[i][tid] : k;
      const int64_t g = unit0 + tid;
      const int64_t bb = g - (g / B) * B;
      if (k != ~0ull) atomicMin(&P.st[bb].dt_key, k);
      if (sflag[tid]) atomicOr(&P.st[bb].nan_flag, 1u);
    }
  } else if (tid == 0) {
    unsigned long long k = skey[0];
#pragma unroll
    for (int i = 1; i < 4; ++i) k = skey[i] < k ? skey[i] : k;
    if (k != ~0ull) atomicMin(&P.st[0].dt_key, k);
    int nf = 0;
#pragma unroll
    for (int i = 0; i < UPB; ++i) nf |= sflag[i];
    if (nf) atomicOr(&P.st[0].nan_flag, 1u);
  }

  if (MODE == MODE_FORCE) {
    // --- S4, q2 stage: warp (c, d) = (w >> 1, w & 1), lane (q1', e') = (lane >> 3, lane & 7)
    {
      const int c = w >> 1, d = w & 1;
      const double *sp = Ss + (c * 2 + d) * 4 * G2L::SQ + lane;
      double sv[4];
#pragma unroll
      for (int q2 = 0; q2 < 4; ++q2) sv[q2] = sp[q2 * G2L::SQ];
      double T[3];
      if (d == 0) {
#pragma unroll
        for (int a2 = 0; a2 < 3; ++a2) {
          double acc = c_t24.B[0][a2] * sv[0];
#pragma unroll
          for (int q2 = 1; q2 < 4; ++q2) acc = __fma_rn(c_t24.B[q2][a2], sv[q2], acc);
          T[a2] = acc;
        }
      } else {
#pragma unroll
        for (int a2 = 0; a2 < 3; ++a2) {
          double acc = c_t24.G[0][a2] * sv[0];
#pragma unroll
          for (int q2 = 1; q2 < 4; ++q2) acc = __fma_rn(c_t24.G[q2][a2], sv[q2], acc);
          T[a2] = acc;
        }
      }
#pragma unroll
      for (int a2 = 0; a2 < 3; ++a2) Ts[((c * 2 + d) * 3 + a2) * 32 + lane] = T[a2];
      if (w < 2) {  // f1[q1'][j2 = w] = sum_q2 Bl[q2][j2] A_q
        const double *ap = Ss + 4 * 4 * G2L::SQ + lane;
        double acc = c_t24.Bl[0][w] * ap[0];
#pragma unroll
        for (int q2 = 1; q2 < 4; ++q2) acc = __fma_rn(c_t24.Bl[q2][w], ap[q2 * G2L::SQ], acc);
        F1s[w * 32 + lane] = acc;
      }
    }
    __syncthreads();
    // --- S4, q1 stage + S5: output t = (r, e') with r = c*9 + a2*3 + a1 (t < 144), then the
    // 32 FTw outputs (j, e')
#pragma unroll
    for (int t = tid; t < 144 + 32; t += G2L::NT) {
      const int ee = t & 7;
      const int64_t g0 = unit0 + ee;
      if (g0 >= P.n_units) continue;
      const int64_t l = BATCHED ? g0 / B : g0;
      const int64_t b = BATCHED ? g0 - l * B : 0;
      if (t < 144) {
        const int r = t >> 3;
        const int c = r / 9, a = r - c * 9, a2 = a / 3, a1 = a - a2 * 3;
        const double *t0 = Ts + ((c * 2 + 0) * 3 + a2) * 32 + ee;
        const double *t1 = Ts + ((c * 2 + 1) * 3 + a2) * 32 + ee;
        double acc = 0.0;
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
          acc = __fma_rn(sTB[12 + qq * 3 + a1], t0[qq * 8], acc);
          acc = __fma_rn(sTB[qq * 3 + a1], t1[qq * 8], acc);
        }
        const int sl = sslot[a * UPB + ee];
        if (sl >= 0) P.evec[((int64_t)sl * 2 + c) * B + b] = acc;
      } else {
        const int j = (t - 144) >> 3, j1 = j & 1, j2 = j >> 1;
        const double *fp = F1s + j2 * 32 + ee;
        double acc = 0.0;
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) acc = __fma_rn(c_t24.Bl[qq][j1], fp[qq * 8], acc);
        const int row = P.ftw_row ? __ldg(P.ftw_row + l) : (int)l;
        if (row >= 0) P.FTw[((int64_t)row * NE + j) * B + b] = acc;
      }
    }
  }
  pdl_trigger();
}

}  // namespace hk
