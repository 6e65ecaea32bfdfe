// force_kernel.cuh -- fused corner-force kernel for sm_100a (FP64).
//
// One CTA evaluates EPB "units" (a unit = one element in full-order mode, one
// (closure element, instance) pair in batched ROM mode); one thread per Gauss
// point of its unit.  Stages (DESIGN "Kernels"):
//   S1 gather    element dofs of x, v (w) and e into shared memory;
//   S2 forward   sum-factorised contractions J = dx/dxi, gradhat v, (gradhat w), e_q,
//                each output an FMA chain in the canonical order of DESIGN A.2;
//   S3 pointwise detJ, J^-1, rho = m_q/detJ, p, cs, h, grad v, eps, lambda_min, mu,
//                sigma, dt_q -- the exact IEEE sequence of DESIGN A.3/A.4 (this file
//                is compiled with -fmad=false; every FMA is written as __fma_rn).  The
//                stage runs with the branch-free fast div/sqrt of ieee_fast.cuh (the
//                two Jacobi eigen-solves of a 3D viscous point interleaved for ILP) and
//                is re-run with the plain IEEE operators on the rare points where a
//                fast path left its valid range -- bit-identical either way;
//   S4 backward  S_q = w_q detJ sigma J^-T, A_q = w_q detJ sigma : grad w, then the
//                sum-factorised transposes F1_K[a][c] = sum_q (S_q gradhat phi_a)_c,
//                FTw_K[j] = sum_q psi_j A_q;
//   S5 outputs   F1_K to its assembly slots (summed per node in fixed order by
//                assemble_kernel, a programmatic dependent launch), FTw_K element-local;
//   S6 dt        warp/CTA min of order-preserving keys, one atomicMin per CTA (exact).
// PAPER anchors: Eq. fom, Eq. forceOneforceTv, Eq. EOS P:374-376,
// stress split P:367-370, density elimination P:389-391, Eq. adaptive-timestep P:533-544.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "hydro_internal.h"
#include "ieee_fast.cuh"

namespace hk {

enum Mode { MODE_FORCE = 0, MODE_DT = 1, MODE_MQ = 2, MODE_FTW = 3 };
// MODE_FTW: F^T w from stored S_q (no pointwise stage): gather w, its reference gradient,
// A_q = S_q : gradhat w, the L2 backward contraction.

// EPB_: units per CTA (0 = default: 8 for 16-point 2D elements, else 1).
#ifndef GEN_SEPS
#define GEN_SEPS 0
#endif
// one dt-key atomic per warp instead of a CTA-wide shared-memory reduction and barrier
#ifndef GEN_WARP_KEY
#define GEN_WARP_KEY 1
#endif
// one-unit 3D CTAs gather node ids and values in the same thread (no barrier in between)
// Vectorised (LDS.128) reads of the stage-2 pencils in the last forward stage (3D, even N)
#ifndef FP_VEC
#define FP_VEC 1
#endif
#ifndef GEN_GATHER1
#define GEN_GATHER1 1
#endif
// q1-stride padding (doubles) of the Q3 stage-2 blocks (see Geo::S2Q1) and stage-1 blocks (S1Q1)
#ifndef S2PAD_K3
#define S2PAD_K3 6
#endif
#ifndef S1PAD_K3
#define S1PAD_K3 0
#endif
// 3D Q2 (K = 2) bank-conflict layouts of the contraction stage buffers (r02; tools/bank_sim.py):
// 1 = padded strides and a q1-fastest stage-2 task order (modelled shared wavefronts per unit
// 756 -> 666), Wb / f2 placed over the dead point stresses; 0 = the round-1 layout.
#ifndef LAYOUT_K2
#define LAYOUT_K2 1
#endif
#ifndef XS_UNDER_K2
#define XS_UNDER_K2 1
#endif
#ifndef EJ_K2
#define EJ_K2 1
#endif
#ifndef S1FCPAD_K3
#define S1FCPAD_K3 2
#endif
// 3D Q3: bank-conflict-avoiding order of the stage-2 tasks (see the stage-2 loop); 0 = plain order
#ifndef PERM_K3
#define PERM_K3 1
#endif

template <int DIM_, int K_, int Q_, int NF_, int EPB_ = 0>
struct Geo {
  static constexpr int DIM = DIM_, K = K_, Q = Q_;
  static constexpr int N = K + 1, M = K;
  static constexpr int ND = DIM == 2 ? N * N : N * N * N;
  static constexpr int NE = DIM == 2 ? M * M : M * M * M;
  static constexpr int NQ = DIM == 2 ? Q * Q : Q * Q * Q;
  static constexpr int EPB = EPB_ > 0 ? EPB_ : (NQ <= 16 ? 8 : 1);
  static constexpr int NT = ((EPB * NQ + 31) / 32) * 32;
  static constexpr int NF = NF_;  // gathered H1 fields: x, v (, w)
  // per-unit shared-memory layout (doubles)
  // 3D stage-1 block [q1][a3][a2] with q1 stride S1Q1 = N^2 + S1PAD_K3 (Q3; padding 2 halves
  // stage 2's modelled LDS.128 conflicts but measured +0.8 % on C3: profiles/ab/r02_ab24_*, so 0)
  static constexpr int S1Q1 = (DIM == 3 && K == 3) ? N * N + S1PAD_K3 : N * N;
  static constexpr int S1 = DIM == 3 ? Q * S1Q1 : Q * N;         // one stage-1 block
  // stage-2 block [q1][q2][a3] with q1 stride S2Q1: for Q3 (Q = 6, N = 4) padded 24 -> 30 doubles
  // so that the per-point LDS.128 pencil reads of forward_point spread over all 32 banks
  // (unpadded: 3-way conflicts, 80 wavefronts per 7 warps instead of 38; ideal 28)
  static constexpr int S2Q1 = (DIM == 3 && K == 3) ? Q * N + S2PAD_K3 : Q * N;
  static constexpr int S2 = DIM == 3 ? Q * S2Q1 : 0;             // one stage-2 block
  static constexpr bool LK2 = DIM == 3 && K == 2 && LAYOUT_K2;
  // K = 2 layout (modelled wavefronts per unit 756 -> 666 within +24 doubles, which keeps the
  // 196 KB shared carve-out at 14 CTAs/SM -- a wider padding (-17 %, +386 doubles) pushed the
  // carve-out to 228 KB and cost C4 9 % through the smaller L1): stage-1 fc stride 73 (was 72),
  // stage-2 fc stride 147 (was 144), Tb c stride 50 (was 48), Wb [w: 162][c: 54][a2 a3: 6][q1]
  // XK2 (XS_UNDER_K2): the gathered dofs live inside the stage-2 span (dead once stage 1 has
  // read them), which pays for a stage-1 q1 stride of 12 (conflict-free stage-2 pencil reads:
  // modelled 54 -> 30 wavefronts per unit) at +22 doubles per unit
  static constexpr bool XK2 = LK2 && XS_UNDER_K2;
  static constexpr int S1Q1X = XK2 ? 12 : S1Q1;                   // stage-1 q1 stride
  static constexpr int S1X = DIM == 3 ? Q * S1Q1X : S1;           // stage-1 B|G stride
  // stage-1 fc stride: K = 2 as above; Q3 with the PERM_K3 stage-2 order: +2 doubles, so that the
  // four consecutive fc of a half-warp read their stage-1 pencils from distinct banks (modelled
  // stage-2 loads 144 -> 72 wavefronts per element)
  static constexpr int S1FC = XK2 ? 2 * S1X + 9
                                  : (LK2 ? 2 * S1X + 1 : (DIM == 3 && K == 3 && PERM_K3 ? 2 * S1X + S1FCPAD_K3 : 2 * S1X));
  static constexpr int S2FC = LK2 ? 3 * S2 + 3 : 3 * S2;          // stage-2 fc stride
  static constexpr int S1TOT = DIM == 3 ? NF * DIM * S1FC : NF * DIM * 2 * S1;
  static constexpr int S2TOT = DIM == 3 ? NF * DIM * S2FC : 0;
  // Tb: XK2 leaves the backward region room under the forward one, so Tb takes the strides that
  // make both the b1 stores and the b2 pencil reads conflict-free (with q1-fastest b2 tasks):
  // [dl: 246][c: 82][q1: 20][a3: 6][q2]
  static constexpr int TA3 = XK2 ? 6 : Q, TQ1 = XK2 ? 20 : Q * N,
                       TC = XK2 ? 82 : (LK2 ? Q * Q * N + 2 : Q * Q * N), TDL = DIM * TC;
  static constexpr int WA = LK2 ? 6 : Q, WC = LK2 ? 54 : N * N * Q, WW = LK2 ? 162 : DIM * N * N * Q;
  static constexpr int E1 = DIM == 3 ? Q * M * M : Q * M;
  static constexpr int E2 = DIM == 3 ? Q * Q * M : 0;
  static constexpr int FWD = S1TOT + S2TOT + E1 + E2;
  static constexpr int TB = DIM == 3 ? DIM * TDL : DIM * DIM * Q * N;
  static constexpr int WB = DIM == 3 ? 2 * WW : 0;
  static constexpr int F1B = DIM == 3 ? Q * Q * M : Q * M;
  static constexpr int F2B = DIM == 3 ? Q * M * M : 0;
  // LK2: Wb and f2 live over the point stresses S_q (dead once b1 has read them)
  static_assert(!LK2 || WB + F2B <= DIM * DIM * NQ, "LK2 Wb placement");
  static constexpr int BWD = DIM * DIM * NQ + NQ + TB + F1B + (LK2 ? 0 : WB + F2B);
  // SEPS (3D Q3 and larger): the point stresses S_q, A_q get their own region after the
  // forward buffers, so they can be written without waiting for every warp to finish its
  // forward reads (one barrier fewer per element); the backward work arrays still overlap
  // the forward buffers.  Costs 2 160 doubles per C3 element (4 CTAs/SM still fit).
  static constexpr bool SEPS = DIM == 3 && NQ >= 128 && GEN_SEPS;
  static constexpr int WORK = SEPS ? FWD + DIM * DIM * NQ + NQ : (FWD > BWD ? FWD : BWD);
  static_assert(!SEPS || TB + WB + F1B + F2B <= FWD, "SEPS layout");
  // the work region starts 16-byte aligned (NEP: NE rounded up to even) so that stage outputs
  // can be read as double2 (LDS.128); every unit is an even number of doubles
  static constexpr int NEP = (NE + 1) & ~1;
  // unit layout: [gathered dofs Xs | e dofs | work] or, XK2, [work] with Xs, Es at XOFF (inside
  // the stage-2 span: written by the gather, read by stage 1, overwritten by stage 2)
  static constexpr int XOFF = XK2 ? S1TOT : 0;
  static constexpr int WKOFF = XK2 ? 0 : NF * DIM * ND + NEP;
  static_assert(!XK2 || NF * DIM * ND + NEP <= S2TOT, "XK2 placement");
  static_assert(!XK2 || NF != 2 || BWD <= FWD, "XK2: the backward region stays under the forward one");
  static constexpr int UNIT = (WKOFF + WORK + 1) & ~1;
  static constexpr int TABD = Q + Q * N * 2 + Q * M;             // w, B, G, Bl
  static constexpr size_t SMEM =
      sizeof(double) * (size_t)(TABD + EPB * UNIT) + sizeof(int) * ((EPB * ND + 1) / 2 * 2) +
      sizeof(unsigned long long) * EPB;
};

struct Params {
  int32_t n_units;          // full: n_elem; batched: n_cl_elem * B
  int B;                    // instances (1 in full mode)
  int b_shift;              // log2(B) when B is a power of two, else -1 (set by launch_force)
  int64_t ld_nodes;         // H1 component stride in nodes (n_nodes or n_cl_nodes)
  const int32_t *elem_nodes;  // [n_l][ND] node ids (closure-local in batched mode)
  const int32_t *elem_gid;    // batched: closure-local -> global element id; NULL = identity
  const double *x, *v, *w, *e, *gamma, *mq, *rho0;
  double q1, q2, alpha, alpha_mu;
  int visc;
  double *evec;             // F1 slot buffer [slot][DIM][B]
  const int32_t *slot;      // [n_l][ND] slot or -1
  double *FTw;              // [row][NE][B]
  const int32_t *ftw_row;   // [n_l] row or -1; NULL = identity
  double *mq_out;           // MODE_MQ: [n_elem][NQ]
  hydro_devstatus *st;      // [B]
  const double *tab_w, *tab_B, *tab_G, *tab_Bl;  // device tables [Q], [Q][N], [Q][N], [Q][M]
  // fused deterministic assembly (S5) and dt finalisation (S6)
  const int32_t *anode;     // [n_l][ND] assembly-node index of (element, local node) or -1
  const int32_t *off;       // [n_asm + 1] CSR: slots of assembly node n are off[n]..off[n+1)
  unsigned *cnt;            // [n_asm][B] arrival counters (zero between calls)
  unsigned *done;           // CTA completion counter (zero between calls)
  double *F1;               // [DIM][n_asm][B] assembled output
  int64_t n_asm;            // assembly nodes (n_nodes, or S0 nodes in sampled mode)
  double *dt_out;           // [B] or NULL
  // stored point stresses S_q = w_q detJ sigma J^-T (optional): [unit][DIM*DIM][NQ]
  double *S_store;          // written by MODE_FORCE when non-NULL
  const double *S_load;     // read by MODE_FTW
  // S index of unit (l, b): sampled mode (ftw_row != NULL) keeps only the S0 elements,
  // compacted to ftw_row[l] * B + b (-1: not stored); full mode: the unit index itself.
  // MODE_FTW over compacted units: unit_elem[row] = the closure element of S0 row `row`.
  const int32_t *unit_elem;
};

// unit -> (element row, instance) of the batched layout unit = l * B + b: a shift for the usual
// power-of-two instance counts (the signed division by a runtime B was ~2 % of all warp
// instructions of the C4 kernel, computed twice per CTA)
__device__ __forceinline__ int unit_row(const Params &P, int g) {
  return P.b_shift >= 0 ? (int)((unsigned)g >> P.b_shift) : (int)((unsigned)g / (unsigned)P.B);
}

__device__ __forceinline__ int64_t s_index(const Params &P, int unit, int l, int b) {
  if (!P.ftw_row) return unit;
  const int row = __ldg(P.ftw_row + l);
  return row < 0 ? -1 : (int64_t)row * P.B + b;
}

// ----------------------------------------------------------------------------- helpers
// min of a 64-bit key over the full warp with two 32-bit REDUX operations (high words, then the
// low words of the lanes holding the minimal high word)
__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long k) {
  const unsigned hi = (unsigned)(k >> 32);
  const unsigned mh = __reduce_min_sync(0xffffffffu, hi);
  const unsigned ml = __reduce_min_sync(0xffffffffu, hi == mh ? (unsigned)k : 0xffffffffu);
  return ((unsigned long long)mh << 32) | ml;
}

__device__ __forceinline__ unsigned long long dt_key(double d) {
  // order-preserving map of a double to uint64 (-0 < +0); NaN never reaches here
  unsigned long long b = (unsigned long long)__double_as_longlong(d);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ double key_to_dt(unsigned long long k) {
  unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}

// Device-side completion of a call, in the dependent launch that follows the force kernel:
// dt = min key (NaN if any dt_q was NaN); the per-call state is reset for the next call
// and the NaN condition is folded into the sticky word read by status_sync.
__device__ __forceinline__ void finalize_one(hydro_devstatus *st, double *dt_out) {
  double d = key_to_dt(st->dt_key);
  if (st->nan_flag) {
    d = __longlong_as_double(0x7ff8000000000000ll);
    st->nan_sticky = 1u;
  }
  if (dt_out) *dt_out = d;
  st->dt_key = dt_key(__longlong_as_double(0x7ff0000000000000ll));  // +inf
  st->nan_flag = 0u;
}

// Programmatic dependent launch (PDL): the force kernel signals that its dependent (the
// assembly / dt-finalisation kernel) may be scheduled; the dependent waits for the force
// grid's completion and memory flush before reading.  Hides the second launch's latency.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// One cyclic-Jacobi rotation of DESIGN A.4 on pair (p,q) with r3 = the third index,
// skipped when |a_pq| <= tol.  Written without branches (the skipped case computes on
// harmless stand-in values and keeps the old entries) so that two independent matrices'
// rotations can be interleaved by the scheduler.  The rotated entries are exactly the
// contract's: dlt = 0.5(a_qq - a_pp), r = sqrt(dlt^2 + a_pq^2), t = a_pq/(|dlt| + r)
// (negated if dlt < 0), c = 1/sqrt(1 + t^2), s = t c.
#ifdef HYDRO_COUNT_ROT
// diagnostic build only (tools/rot_count.py): [0] lane-slots of executed rotations,
// [1] rotations a lane actually needed (not skipped)
__device__ unsigned long long g_rot_count[2];
__device__ unsigned long long g_sweep_count[4][2];  // [sweep]: lanes live (a + e), lane-slots executed
__device__ unsigned long long g_rerun_count[2];     // points re-run with IEEE ops, warps affected
__device__ __forceinline__ void count_rerun(bool rerun) {
  const unsigned m = __activemask();
  const unsigned b = __ballot_sync(m, rerun);
  if ((threadIdx.x & 31) == __ffs(m) - 1 && b) {
    atomicAdd(&g_rerun_count[0], (unsigned long long)__popc(b));
    atomicAdd(&g_rerun_count[1], 1ull);
  }
}
__device__ __forceinline__ void count_sweep(int sweep, bool la, bool le, bool wa, bool we) {
  const unsigned b = __ballot_sync(0xffffffffu, la), c = __ballot_sync(0xffffffffu, le);
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&g_sweep_count[sweep][0], (unsigned long long)(__popc(b) + __popc(c)));
    atomicAdd(&g_sweep_count[sweep][1], (unsigned long long)(32 * ((int)wa + (int)we)));
  }
}
__device__ __forceinline__ void count_rot(bool go) {
  const unsigned m = __activemask();
  const unsigned b = __ballot_sync(m, go);
  if ((threadIdx.x & 31) == __ffs(m) - 1) {
    atomicAdd(&g_rot_count[0], (unsigned long long)__popc(m));
    atomicAdd(&g_rot_count[1], (unsigned long long)__popc(b));
  }
}
#else
__device__ __forceinline__ void count_rot(bool) {}
__device__ __forceinline__ void count_sweep(int, bool, bool, bool, bool) {}
__device__ __forceinline__ void count_rerun(bool) {}
#endif

// !(|x| <= tol) for a tolerance tol >= +0 or NaN.  GEN_INT_CMP: on the integer ALU --
// for non-negative doubles the bit patterns order like the values, so |x| > tol is
// (bits(x) & ~sign) > bits(tol) as int64, which also sends NaN x to "above"; a NaN tol
// (bits above +inf's) makes every x "above", as the FP comparison does.  Same predicate
// bit for bit, off the FP64 pipe -- but measured 0.9 % slower on C2 and 1.2 % on TG (0.5 %
// faster on C3; profiles/ab/r01_ab43_*), so the FP comparison stays the default.
#ifndef GEN_INT_CMP
#define GEN_INT_CMP 0
#endif
__device__ __forceinline__ bool above_tol(double x, double tol) {
#if GEN_INT_CMP
  const long long xb = __double_as_longlong(x) & 0x7fffffffffffffffll;
  const long long tb = __double_as_longlong(tol);
  return xb > tb || tb > 0x7ff0000000000000ll;
#else
  return !(fabs(x) <= tol);
#endif
}

template <class AR>
__device__ __forceinline__ void jacobi_rot(AR &ar, double &app, double &aqq, double &apq,
                                           double &arp, double &arq, const double tol) {
  const bool go = above_tol(apq, tol);
  count_rot(go);
  const double a_ = go ? apq : 1.0;
  const double dl = go ? 0.5 * (aqq - app) : 0.0;
  const double rr = ar.sqrt_(dl * dl + a_ * a_);
  double t = ar.div(a_, fabs(dl) + rr);
  t = dl < 0.0 ? -t : t;
  // t = a_/(|dl| + sqrt(dl^2 + a_^2)) has |t| <= 1 (plus rounding) whenever the checked
  // sqrt and div passed, so 1 + t^2 lies in [1, 2] and its root in [1, 1.5): both fast
  // paths are valid there and their range checks are redundant (unit variants).  If a
  // checked op failed, the whole point is re-run with IEEE operators anyway.
  const double c = ar.rcp_unit(ar.sqrt_unit(1.0 + t * t));
  const double s = t * c;
  const double rp = arp, rq = arq;
  const double napp = app - t * apq;
  const double naqq = aqq + t * apq;
  const double narp = c * rp - s * rq;
  const double narq = s * rp + c * rq;
  app = go ? napp : app;
  aqq = go ? naqq : aqq;
  apq = go ? 0.0 : apq;
  arp = go ? narp : arp;
  arq = go ? narq : arq;
}

// Two independent rotations (one per matrix), written step by step in lockstep so the
// scheduler sees the two dependency chains side by side (ptxas otherwise emitted the first
// rotation's whole sqrt -> div -> sqrt -> rcp chain before the second's).  Each rotation's
// arithmetic is exactly jacobi_rot's.
template <class AR>
__device__ __forceinline__ void jacobi_rot2(AR &ar, double &app, double &aqq, double &apq,
                                            double &arp, double &arq, const double ta,
                                            double &epp, double &eqq, double &epq,
                                            double &erp, double &erq, const double te) {
  const bool ga = above_tol(apq, ta), ge = above_tol(epq, te);
  count_rot(ga);
  count_rot(ge);
  const double a_ = ga ? apq : 1.0, e_ = ge ? epq : 1.0;
  const double dla = ga ? 0.5 * (aqq - app) : 0.0, dle = ge ? 0.5 * (eqq - epp) : 0.0;
  const double sa = dla * dla + a_ * a_, se = dle * dle + e_ * e_;
  const double rra = ar.sqrt_(sa), rre = ar.sqrt_(se);
  const double dna = fabs(dla) + rra, dne = fabs(dle) + rre;
  double tA = ar.div(a_, dna), tE = ar.div(e_, dne);
  tA = dla < 0.0 ? -tA : tA;
  tE = dle < 0.0 ? -tE : tE;
  const double ua = 1.0 + tA * tA, ue = 1.0 + tE * tE;
  const double qa = ar.sqrt_unit(ua), qe = ar.sqrt_unit(ue);  // in [1, 2]: see jacobi_rot
  const double ca = ar.rcp_unit(qa), ce = ar.rcp_unit(qe);
  const double sA = tA * ca, sE = tE * ce;
  const double rpa = arp, rqa = arq, rpe = erp, rqe = erq;
  const double nppa = app - tA * apq, nppe = epp - tE * epq;
  const double nqqa = aqq + tA * apq, nqqe = eqq + tE * epq;
  const double nrpa = ca * rpa - sA * rqa, nrpe = ce * rpe - sE * rqe;
  const double nrqa = sA * rpa + ca * rqa, nrqe = sE * rpe + ce * rqe;
  app = ga ? nppa : app;  epp = ge ? nppe : epp;
  aqq = ga ? nqqa : aqq;  eqq = ge ? nqqe : eqq;
  apq = ga ? 0.0 : apq;   epq = ge ? 0.0 : epq;
  arp = ga ? nrpa : arp;  erp = ge ? nrpe : erp;
  arq = ga ? nrqa : arq;  erq = ge ? nrqe : erq;
}

__device__ __forceinline__ double amax6(double a00, double a11, double a22, double a01, double a02,
                                        double a12) {
  double amax = fabs(a00);
  amax = fmax(amax, fabs(a11));
  amax = fmax(amax, fabs(a22));
  amax = fmax(amax, fabs(a01));
  amax = fmax(amax, fabs(a02));
  amax = fmax(amax, fabs(a12));
  return amax;
}

__device__ __forceinline__ bool offdiag_live(double a01, double a02, double a12, double tol) {
  return above_tol(a01, tol) || above_tol(a02, tol) || above_tol(a12, tol);
}

// The remaining sweeps [sweep0, 4) of lmin3_pair once at most 32 matrices of the warp
// (either kind, over all lanes) are still live: they are compacted onto the first lanes
// (lane i takes the i-th live matrix; __fns finds its owner) and rotated one matrix per lane,
// so the slots the converged lanes would have skipped cost nothing.  Each matrix sees the
// same rotation sequence with the same arithmetic (jacobi_rot), so its lambda_min is
// bit-identical to the uncompacted schedule's; a matrix that was not live keeps its entries.
template <class AR>
__device__ __forceinline__ void lmin3_pair_compact(AR &ar, int sweep0, unsigned ba, unsigned be,
                                                 double a00, double a11, double a22, double a01,
                                                 double a02, double a12, double ta, double e00,
                                                 double e11, double e22, double e01, double e02,
                                                 double e12, double te, double &la, double &le) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int na = __popc(ba), n = na + __popc(be);
  const bool mine = lane < n, isE = lane >= na;
  const int src = mine ? (int)__fns(isE ? be : ba, 0, (isE ? lane - na : lane) + 1) : lane;
  // both shuffles are issued by every lane (the source lane does not know which is wanted)
  const double sa00 = __shfl_sync(full, a00, src), se00 = __shfl_sync(full, e00, src);
  const double sa11 = __shfl_sync(full, a11, src), se11 = __shfl_sync(full, e11, src);
  const double sa22 = __shfl_sync(full, a22, src), se22 = __shfl_sync(full, e22, src);
  const double sa01 = __shfl_sync(full, a01, src), se01 = __shfl_sync(full, e01, src);
  const double sa02 = __shfl_sync(full, a02, src), se02 = __shfl_sync(full, e02, src);
  const double sa12 = __shfl_sync(full, a12, src), se12 = __shfl_sync(full, e12, src);
  const double sta = __shfl_sync(full, ta, src), ste = __shfl_sync(full, te, src);
  double m00 = isE ? se00 : sa00, m11 = isE ? se11 : sa11, m22 = isE ? se22 : sa22;
  double m01 = isE ? se01 : sa01, m02 = isE ? se02 : sa02, m12 = isE ? se12 : sa12;
  const double tm = isE ? ste : sta;
  if (!mine) m01 = m02 = m12 = 0.0;  // idle lanes: nothing live, never keeps the loop going
#pragma unroll 1
  for (int sweep = sweep0; sweep < 4; ++sweep) {
    if (!__any_sync(full, offdiag_live(m01, m02, m12, tm))) break;
    jacobi_rot(ar, m00, m11, m01, m02, m12, tm);  // (0,1), r3 = 2
    jacobi_rot(ar, m00, m22, m02, m01, m12, tm);  // (0,2), r3 = 1
    jacobi_rot(ar, m11, m22, m12, m01, m02, tm);  // (1,2), r3 = 0
  }
  const double lam = fmin(fmin(m00, m11), m22);
  const unsigned lt = (1u << lane) - 1u;
  const double lA = __shfl_sync(full, lam, __popc(ba & lt));
  const double lE = __shfl_sync(full, lam, (na + __popc(be & lt)) & 31);
  la = ((ba >> lane) & 1u) ? lA : fmin(fmin(a00, a11), a22);
  le = ((be >> lane) & 1u) ? lE : fmin(fmin(e00, e11), e22);
}

// Smallest eigenvalues of two symmetric 3x3 matrices (DESIGN A.4), their rotations
// interleaved.  COMPACT: from the third sweep on, once <= 32 matrices of the warp are live,
// finish in lmin3_pair_compact (force3d: C2 -5.5 %; the 72-register generic kernel spills
// more with it and loses 5 %, so it does not use it).  EARLY: the warp leaves the sweep loop once no lane has a live
// off-diagonal in either matrix (every remaining rotation would be a skip) -- needs all
// 32 lanes converged, so only the fast (non-divergent) pass uses it.
template <class AR, bool EARLY, bool COMPACT = false>
__device__ __forceinline__ void lmin3_pair(AR &ar, double a00, double a11, double a22,
                                           double a01, double a02, double a12, double e00,
                                           double e11, double e22, double e01, double e02,
                                           double e12, double &la_out, double &le_out) {
  const double ta = amax6(a00, a11, a22, a01, a02, a12) * 0x1p-53;
  const double te = amax6(e00, e11, e22, e01, e02, e12) * 0x1p-53;
#pragma unroll 1
  for (int sweep = 0; sweep < 4; ++sweep) {
    if (EARLY) {
      // warp-uniform scheduling: a rotation slot of a matrix is executed only if some lane
      // needs it (skipped lanes keep their entries), and the two matrices' rotations are
      // interleaved only when both are live -- a converged matrix costs nothing
      const bool la = offdiag_live(a01, a02, a12, ta), le = offdiag_live(e01, e02, e12, te);
      const bool wa = __any_sync(0xffffffffu, la), we = __any_sync(0xffffffffu, le);
      count_sweep(sweep, la, le, wa, we);
      if (!(wa || we)) break;
      // (a sweep with only one kind live always fits: its single-matrix code paths below
      // are then dead and compiled out, which keeps the kernel's hot loop smaller)
      if (COMPACT && (sweep >= 2 || !(wa && we))) {
        const unsigned ba = __ballot_sync(0xffffffffu, la), be = __ballot_sync(0xffffffffu, le);
        if (__popc(ba) + __popc(be) <= 32) {
          lmin3_pair_compact(ar, sweep, ba, be, a00, a11, a22, a01, a02, a12, ta, e00, e11, e22,
                             e01, e02, e12, te, la_out, le_out);
          return;
        }
      }
      if (wa && we) {
        jacobi_rot2(ar, a00, a11, a01, a02, a12, ta, e00, e11, e01, e02, e12, te);  // (0,1)
        jacobi_rot2(ar, a00, a22, a02, a01, a12, ta, e00, e22, e02, e01, e12, te);  // (0,2)
        jacobi_rot2(ar, a11, a22, a12, a01, a02, ta, e11, e22, e12, e01, e02, te);  // (1,2)
      } else if (COMPACT) {
        __builtin_unreachable();  // handled by lmin3_pair_compact above
      } else if (wa) {
        jacobi_rot(ar, a00, a11, a01, a02, a12, ta);
        jacobi_rot(ar, a00, a22, a02, a01, a12, ta);
        jacobi_rot(ar, a11, a22, a12, a01, a02, ta);
      } else {
        jacobi_rot(ar, e00, e11, e01, e02, e12, te);
        jacobi_rot(ar, e00, e22, e02, e01, e12, te);
        jacobi_rot(ar, e11, e22, e12, e01, e02, te);
      }
    } else {
      jacobi_rot(ar, a00, a11, a01, a02, a12, ta);  // (0,1), r3 = 2
      jacobi_rot(ar, e00, e11, e01, e02, e12, te);
      jacobi_rot(ar, a00, a22, a02, a01, a12, ta);  // (0,2), r3 = 1
      jacobi_rot(ar, e00, e22, e02, e01, e12, te);
      jacobi_rot(ar, a11, a22, a12, a01, a02, ta);  // (1,2), r3 = 0
      jacobi_rot(ar, e11, e22, e12, e01, e02, te);
    }
  }
  la_out = fmin(fmin(a00, a11), a22);
  le_out = fmin(fmin(e00, e11), e22);
}

template <class AR, bool EARLY>
__device__ __forceinline__ double lmin3(AR &ar, double a00, double a11, double a22, double a01,
                                        double a02, double a12) {
  const double ta = amax6(a00, a11, a22, a01, a02, a12) * 0x1p-53;
#pragma unroll 1
  for (int sweep = 0; sweep < 4; ++sweep) {
    if (EARLY) {
      if (!__any_sync(0xffffffffu, offdiag_live(a01, a02, a12, ta))) break;
    }
    jacobi_rot(ar, a00, a11, a01, a02, a12, ta);
    jacobi_rot(ar, a00, a22, a02, a01, a12, ta);
    jacobi_rot(ar, a11, a22, a12, a01, a02, ta);
  }
  return fmin(fmin(a00, a11), a22);
}

// Smallest eigenvalue of a symmetric 3x3 matrix by the closed form of DESIGN A.4 / R30:
// q = tr/3, B = A - qI, p = sqrt(tr(B^2)/6), r = det(B)/(2p^3); lambda_min = q + 2p c with c
// the smallest root of 4c^3 - 3c = r (a cubic guess in s = sqrt((1-r)/2), two Newton steps).
// fb = true where the root is ill-conditioned (r > 1 - 2^-13: a near-double lambda_min) or r is
// NaN: the caller then takes the Jacobi value instead.  A = qI (p2 == 0) gives q.  Operation
// for operation the oracle's oracle_lmin3 (oracle/hydro_oracle.c).  The guards below only keep
// operands inside the fast paths' exact range; each reproduces the IEEE result exactly:
// p2 == 0 returns q anyway, 0 / den = det (den > 0), and a zero Newton residual leaves c.
template <class AR>
__device__ __forceinline__ double lmin3_cf(AR &ar, double a00, double a11, double a22, double a01,
                                           double a02, double a12, bool &fb) {
  const double q = ((a00 + a11) + a22) * 0x1.5555555555555p-2;
  const double b0 = a00 - q, b1 = a11 - q, b2 = a22 - q;
  const double p1 = (a01 * a01 + a02 * a02) + a12 * a12;
  const double p2 = ((b0 * b0 + b1 * b1) + b2 * b2) + 2.0 * p1;
  const bool iso = p2 == 0.0;
  const double p = ar.sqrt_((iso ? 1.0 : p2) * 0x1.5555555555555p-3);
  const double det = (b0 * (b1 * b2 - a12 * a12) - a01 * (a01 * b2 - a12 * a02)) + a02 * (a01 * a12 - b1 * a02);
  const double den = (2.0 * p) * (p * p);
  double r = (det == 0.0 && den > 0.0) ? det : ar.div(det, den);
  fb = !iso && !(r <= 1.0 - 0x1p-13);
  r = (fb || iso) ? 0.0 : fmax(r, -1.0);  // (branch values unused when fb or iso)
  // r, s, c, f, f' are scale-free: (1 - r)/2 lies in [2^-14, 1], f' = 12c^2 - 3 >= 0.05 and a
  // nonzero f is far above 2^-967, so these fast paths need no range checks (*_unit)
  const double s = ar.sqrt_unit((1.0 - r) * 0.5);
  double u = __fma_rn(s, -0.005042, 0.021433);
  u = __fma_rn(s, u, -0.04969);
  u = __fma_rn(s, u, 0.110644);
  u = __fma_rn(s, u, -0x1.279a74590331cp-1);
  double c = __fma_rn(s, u, -0.5);
#pragma unroll
  for (int it = 0; it < 2; ++it) {
    const double c2 = c * c;
    const double f = __fma_rn(c, __fma_rn(4.0, c2, -3.0), -r);
    const double fp = __fma_rn(12.0, c2, -3.0);
    c = c - (f == 0.0 ? f : ar.div_unit(f, fp));
  }
  return iso ? q : __fma_rn(2.0 * p, c, q);
}

// Determinant / inverse by cofactors (DESIGN A.3).
template <int DIM, class AR>
__device__ __forceinline__ double det_inv(AR &ar, const double (&J)[3][3], double (&Ji)[3][3]) {
  if (DIM == 2) {
    const double det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    const double inv = ar.rcp(det);
    Ji[0][0] = J[1][1] * inv;
    Ji[0][1] = -(J[0][1] * inv);
    Ji[1][0] = -(J[1][0] * inv);
    Ji[1][1] = J[0][0] * inv;
    return det;
  } else {
    const double C00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
    const double C01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
    const double C02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
    const double C10 = J[0][2] * J[2][1] - J[0][1] * J[2][2];
    const double C11 = J[0][0] * J[2][2] - J[0][2] * J[2][0];
    const double C12 = J[0][1] * J[2][0] - J[0][0] * J[2][1];
    const double C20 = J[0][1] * J[1][2] - J[0][2] * J[1][1];
    const double C21 = J[0][2] * J[1][0] - J[0][0] * J[1][2];
    const double C22 = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    const double det = (J[0][0] * C00 + J[0][1] * C01) + J[0][2] * C02;
    const double inv = ar.rcp(det);
    Ji[0][0] = C00 * inv; Ji[0][1] = C10 * inv; Ji[0][2] = C20 * inv;
    Ji[1][0] = C01 * inv; Ji[1][1] = C11 * inv; Ji[1][2] = C21 * inv;
    Ji[2][0] = C02 * inv; Ji[2][1] = C12 * inv; Ji[2][2] = C22 * inv;
    return det;
  }
}

template <int DIM>
__device__ __forceinline__ double det_only(const double (&J)[3][3]) {
  if (DIM == 2) return J[0][0] * J[1][1] - J[0][1] * J[1][0];
  const double C00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
  const double C01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
  const double C02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
  return (J[0][0] * C00 + J[0][1] * C01) + J[0][2] * C02;
}

struct PhysIn {
  double q1, q2, alpha, alpha_mu;
};

struct PointOut {
  double S[3][3];  // w_q detJ sigma J^-T (DIM x DIM)
  double A;        // w_q detJ sigma : grad w
  double det, dtq;
};

// Pointwise stage (DESIGN A.3/A.4) through arithmetic policy AR; everything dt_q depends
// on follows the contract exactly.  Gw: gradhat of the field F^T is applied to (== Gv
// when w is v).  S and A are tolerance-only (A.5).
template <int DIM, bool VISC, bool HAS_W, bool EARLY, class AR, bool COMPACT = false>
__device__ __forceinline__ void pointwise(AR &ar, const double (&J)[3][3], const double (&Gv)[3][3],
                                          const double (&Gw)[3][3], double eq, double mq,
                                          double gam, double wq, const PhysIn &ph, PointOut &o) {
  double Ji[3][3];
  const double det = det_inv<DIM>(ar, J, Ji);
  const double rho = ar.div(mq, det);
  const double p = ((gam - 1.0) * rho) * eq;
  const double cs = ar.sqrt_((gam * (gam - 1.0)) * eq);
  // physical velocity gradient (contract order: ascending i, plain mul/add)
  double gv[3][3];
#pragma unroll
  for (int c = 0; c < DIM; ++c)
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      double s = Gv[c][0] * Ji[0][d];
#pragma unroll
      for (int i = 1; i < DIM; ++i) s = s + Gv[c][i] * Ji[i][d];
      gv[c][d] = s;
    }
  double eps[3][3];
#pragma unroll
  for (int c = 0; c < DIM; ++c) {
    eps[c][c] = gv[c][c];
#pragma unroll
    for (int d = 0; d < DIM; ++d)
      if (d != c) eps[c][d] = 0.5 * (gv[c][d] + gv[d][c]);
  }
  double h, lam = 0.0;
  if (DIM == 2) {
    const double c00 = J[0][0] * J[0][0] + J[1][0] * J[1][0];
    const double c11 = J[0][1] * J[0][1] + J[1][1] * J[1][1];
    const double c01 = J[0][0] * J[0][1] + J[1][0] * J[1][1];
    const double kk = 0.5 * (c00 - c11);
    const double smax2 = 0.5 * (c00 + c11) + ar.sqrt_(kk * kk + c01 * c01);
    h = ar.div(det, ar.sqrt_(smax2));
    if (VISC) {
      const double k = 0.5 * (eps[0][0] - eps[1][1]);
      lam = 0.5 * (eps[0][0] + eps[1][1]) - ar.sqrt_(k * k + eps[0][1] * eps[0][1]);
    }
  } else {
    const double c00 = (J[0][0] * J[0][0] + J[1][0] * J[1][0]) + J[2][0] * J[2][0];
    const double c11 = (J[0][1] * J[0][1] + J[1][1] * J[1][1]) + J[2][1] * J[2][1];
    const double c22 = (J[0][2] * J[0][2] + J[1][2] * J[1][2]) + J[2][2] * J[2][2];
    const double c01 = (J[0][0] * J[0][1] + J[1][0] * J[1][1]) + J[2][0] * J[2][1];
    const double c02 = (J[0][0] * J[0][2] + J[1][0] * J[1][2]) + J[2][0] * J[2][2];
    const double c12 = (J[0][1] * J[0][2] + J[1][1] * J[1][2]) + J[2][1] * J[2][2];
    // DESIGN A.4 / R30: closed form, Jacobi only where the closed form is ill-conditioned
    bool fa = false, fe = false;
    double lj = lmin3_cf(ar, c00, c11, c22, c01, c02, c12, fa);
    if (VISC) lam = lmin3_cf(ar, eps[0][0], eps[1][1], eps[2][2], eps[0][1], eps[0][2], eps[1][2], fe);
    if (EARLY) {
      // warp-uniform fallback: lanes without a fallback pass diagonal matrices (no live
      // off-diagonal: no rotation slot is executed for them) and keep their closed form
      if (__any_sync(0xffffffffu, fa || fe)) {
        double ja, je = 0.0;
        if (VISC) {
          lmin3_pair<AR, true, COMPACT>(ar, c00, c11, c22, fa ? c01 : 0.0, fa ? c02 : 0.0, fa ? c12 : 0.0,
                                        eps[0][0], eps[1][1], eps[2][2], fe ? eps[0][1] : 0.0,
                                        fe ? eps[0][2] : 0.0, fe ? eps[1][2] : 0.0, ja, je);
        } else {
          ja = lmin3<AR, true>(ar, c00, c11, c22, fa ? c01 : 0.0, fa ? c02 : 0.0, fa ? c12 : 0.0);
        }
        lj = fa ? ja : lj;
        lam = fe ? je : lam;
      }
    } else {
      if (fa) lj = lmin3<AR, false>(ar, c00, c11, c22, c01, c02, c12);
      if (VISC && fe) lam = lmin3<AR, false>(ar, eps[0][0], eps[1][1], eps[2][2], eps[0][1], eps[0][2], eps[1][2]);
    }
    h = ar.sqrt_(fmax(lj, 0.0));
  }
  double mu = 0.0, visc_term;
  const double den = (rho * h) * h;
  if (VISC) {
    const double lneg = fmin(lam, 0.0);
    mu = (rho * h) * ((ph.q1 * cs) + ((ph.q2 * h) * (-lneg)));
    visc_term = ar.div(ph.alpha_mu * mu, den);
  } else {
    // (alpha_mu * 0) / den with IEEE semantics, no division: +-0 (sign xor) unless den is
    // 0 or NaN (then NaN); a NaN numerator (alpha_mu infinite) stays NaN.
    const double num = ph.alpha_mu * mu;
    const bool nanres = (num != num) || (den == 0.0) || (den != den);
    const double z = (signbit(num) != signbit(den)) ? -0.0 : 0.0;
    visc_term = nanres ? __longlong_as_double(0x7ff8000000000000ll) : z;
  }
  const double inv_dt = ar.div(cs, h) + visc_term;
  o.dtq = ar.div(ph.alpha, inv_dt);
  o.det = det;
  // sigma = -p I + mu eps;  S = w_q detJ sigma J^-T;  A = w_q detJ sigma : grad w
  double sig[3][3];
#pragma unroll
  for (int c = 0; c < DIM; ++c)
#pragma unroll
    for (int d = 0; d < DIM; ++d) sig[c][d] = (VISC ? mu * eps[c][d] : 0.0) - (c == d ? p : 0.0);
  const double wd = wq * det;
  double A = 0.0;
#pragma unroll
  for (int c = 0; c < DIM; ++c)
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
      double s = sig[c][0] * Ji[d][0];
#pragma unroll
      for (int i = 1; i < DIM; ++i) s = __fma_rn(sig[c][i], Ji[d][i], s);
      o.S[c][d] = wd * s;
      double g;
      if (HAS_W) {
        g = Gw[c][0] * Ji[0][d];
#pragma unroll
        for (int i = 1; i < DIM; ++i) g = __fma_rn(Gw[c][i], Ji[i][d], g);
      } else {
        g = eps[c][d];  // sigma symmetric: sigma : grad v = sigma : eps
      }
      A = __fma_rn(sig[c][d], g, A);
    }
  o.A = wd * A;
}

// Last forward stage for one Gauss point (DESIGN A.2, canonical order): 3D contracts a3
// from the stage-2 blocks, 2D contracts a2 from the stage-1 blocks; e_q likewise.  Reads
// shared memory only, so the exact IEEE re-run of S3 can recompute its inputs instead of
// keeping them live in registers through the fast pass.
template <int DIM, int K, int Q, int NF, bool WANT_E>
__device__ __forceinline__ void forward_point(const double *sB, const double *sG,
                                              const double *sBl, const double *Wk, int q1i,
                                              int q2i, int q3i, double (&J)[3][3],
                                              double (&Gv)[3][3], double (&Gw)[3][3],
                                              double &eq) {
  using G = Geo<DIM, K, Q, NF>;
  constexpr int N = G::N, M = G::M;
  if (DIM == 3) {
    const double *S2b = Wk + G::S1TOT;                   // [NF*DIM: S2FC][3][Q][S2Q1: Q][N]
    const double *E2b = S2b + G::S2TOT + G::E1;          // [Q][Q][M]
    double tB[N], tG[N];
#pragma unroll
    for (int a3 = 0; a3 < N; ++a3) { tB[a3] = sB[q3i * N + a3]; tG[a3] = sG[q3i * N + a3]; }
#pragma unroll
    for (int f = 0; f < NF; ++f) {
#pragma unroll
      for (int c = 0; c < DIM; ++c) {
        const int fc = f * DIM + c;
        const double *p1 = S2b + fc * G::S2FC + 0 * G::S2 + q1i * G::S2Q1 + q2i * N;
        const double *p2 = S2b + fc * G::S2FC + 1 * G::S2 + q1i * G::S2Q1 + q2i * N;
        const double *p3 = S2b + fc * G::S2FC + 2 * G::S2 + q1i * G::S2Q1 + q2i * N;
        double d0, d1, d2;
        if constexpr (N % 2 == 0 && FP_VEC) {   // 16-byte aligned pencils: LDS.128
          double v1[N], v2[N], v3[N];
#pragma unroll
          for (int a3 = 0; a3 < N; a3 += 2) {
            const double2 x1 = *reinterpret_cast<const double2 *>(p1 + a3);
            const double2 x2 = *reinterpret_cast<const double2 *>(p2 + a3);
            const double2 x3 = *reinterpret_cast<const double2 *>(p3 + a3);
            v1[a3] = x1.x; v1[a3 + 1] = x1.y;
            v2[a3] = x2.x; v2[a3 + 1] = x2.y;
            v3[a3] = x3.x; v3[a3 + 1] = x3.y;
          }
          d0 = tB[0] * v1[0]; d1 = tB[0] * v2[0]; d2 = tG[0] * v3[0];
#pragma unroll
          for (int a3 = 1; a3 < N; ++a3) {
            d0 = __fma_rn(tB[a3], v1[a3], d0);
            d1 = __fma_rn(tB[a3], v2[a3], d1);
            d2 = __fma_rn(tG[a3], v3[a3], d2);
          }
        } else {
          d0 = tB[0] * p1[0]; d1 = tB[0] * p2[0]; d2 = tG[0] * p3[0];
#pragma unroll
          for (int a3 = 1; a3 < N; ++a3) {
            d0 = __fma_rn(tB[a3], p1[a3], d0);
            d1 = __fma_rn(tB[a3], p2[a3], d1);
            d2 = __fma_rn(tG[a3], p3[a3], d2);
          }
        }
        double *dst = f == 0 ? J[c] : (f == 1 ? Gv[c] : Gw[c]);
        dst[0] = d0; dst[1] = d1; dst[2] = d2;
      }
    }
    if (WANT_E) {
      // E2b: [q1][q2][j3], or [j3][q1][q2] for K = 2 (EJ_K2: a half-warp's 16 points read 16
      // consecutive doubles, one wavefront instead of two)
      constexpr bool EJ = G::LK2 && EJ_K2;
      const double *tb = sBl + q3i * M;
      const double *src = EJ ? E2b + q1i * Q + q2i : E2b + (q1i * Q + q2i) * M;
      constexpr int ES = EJ ? Q * Q : 1;
      double acc = tb[0] * src[0];
#pragma unroll
      for (int j3 = 1; j3 < M; ++j3) acc = __fma_rn(tb[j3], src[j3 * ES], acc);
      eq = acc;
    }
  } else {
    const double *S1b = Wk;                              // [NF*DIM][2][Q][N]
    const double *E1b = Wk + G::NF * DIM * 2 * G::S1;    // [Q][M]
    double tB[N], tG[N];
#pragma unroll
    for (int a2 = 0; a2 < N; ++a2) { tB[a2] = sB[q2i * N + a2]; tG[a2] = sG[q2i * N + a2]; }
#pragma unroll
    for (int f = 0; f < NF; ++f) {
#pragma unroll
      for (int c = 0; c < DIM; ++c) {
        const int fc = f * DIM + c;
        const double *uB = S1b + ((fc * 2 + 0) * Q + q1i) * N;
        const double *uG = S1b + ((fc * 2 + 1) * Q + q1i) * N;
        double d0 = tB[0] * uG[0], d1 = tG[0] * uB[0];
#pragma unroll
        for (int a2 = 1; a2 < N; ++a2) {
          d0 = __fma_rn(tB[a2], uG[a2], d0);
          d1 = __fma_rn(tG[a2], uB[a2], d1);
        }
        double *dst = f == 0 ? J[c] : (f == 1 ? Gv[c] : Gw[c]);
        dst[0] = d0; dst[1] = d1;
      }
    }
    if (WANT_E) {
      const double *tb = sBl + q2i * M;
      const double *src = E1b + q1i * M;
      double acc = tb[0] * src[0];
#pragma unroll
      for (int j2 = 1; j2 < M; ++j2) acc = __fma_rn(tb[j2], src[j2], acc);
      eq = acc;
    }
  }
}

// Warp-compacted final Jacobi sweeps in the generic kernel (3D Q2 only; Q3 at 72 registers
// spills more with it): see lmin3_pair.  Off by default: on the blocked generic kernel it is
// neutral (C2 +0.8 %, C4 -0.3 %: profiles/ab/r01_ab23_*); force3d keeps it.
#ifndef F3_COMPACT
#define F3_COMPACT 0
#endif
// CTAs per SM targeted for the 224-thread (3D Q3) generic kernel (registers: 4 -> 72)
#ifndef GEN_MINB224
#define GEN_MINB224 4
#endif
// ... and for the 64-thread (3D Q2) one: 14 -> 72 registers, 28 warps/SM; with the blocked
// stages the occupancy pays for the extra spills (10/12/13/14/16 measured: profiles/ab/r01_ab30_*)
#ifndef GEN_MINB64
#define GEN_MINB64 14
#endif
#ifndef F3_COMPACT_Q3
#define F3_COMPACT_Q3 0
#endif
// Task splits of the 3D contraction stages (r02): a stage's pencils are split into SPLIT parts
// along one output index so that more of the CTA's threads work per round.  Each part reloads
// its pencil's inputs; every output keeps its FMA chain (the forward ones: DESIGN A.2).  Parts
// occupy contiguous task ranges (warp-uniform except at a range boundary) and each part's body
// is compiled with its table indices as constants (constant-bank operands, no LDC).
// forward stage 1 (q1 ranges), stage 2 (q2 ranges); backward b1 (per dl), b2 (per a2 range),
// b3 (per a1 range).  Q2 (64-thread) / Q3 (224-thread) defaults; -D overrides for A/B builds.
#ifndef SPLIT_F1_K2
#define SPLIT_F1_K2 1
#endif
#ifndef SPLIT_F2_K2
#define SPLIT_F2_K2 1
#endif
#ifndef SPLIT_B1_K2
#define SPLIT_B1_K2 1
#endif
#ifndef SPLIT_B2_K2
#define SPLIT_B2_K2 1
#endif
#ifndef SPLIT_B3_K2
#define SPLIT_B3_K2 1
#endif
#ifndef SPLIT_F1_K3
#define SPLIT_F1_K3 1
#endif
#ifndef SPLIT_F2_K3
#define SPLIT_F2_K3 1
#endif
#ifndef SPLIT_B1_K3
#define SPLIT_B1_K3 1
#endif
#ifndef SPLIT_B2_K3
#define SPLIT_B2_K3 1
#endif
#ifndef SPLIT_B3_K3
#define SPLIT_B3_K3 1
#endif
// Unroll of the table-indexed loops of the 3D Q3 contraction stages (r02).  On sm_100a the
// FP64 instructions take table entries as uniform-register operands (LDCU into URs); fully
// unrolled, a Q3 stage keeps 48 table doubles live and the uniform file spills into regular
// registers (R2UR / MOV.SPILL / IMAD.U32 moves: ~10 instructions per FP64 one in stage 1,
// profiles/r02_v3_c3_*).  K3_ROLL_Q / K3_ROLL_N > 0 unroll the loops over Gauss points / over
// nodes and dofs by that factor only (Q2 keeps full unrolling: its 24 entries fit).  Same FMA
// chains, so the same bits.  C3 force call (profiles/ab/r02_ab19-20_*): full 6.56 ms; Q 3 with
// N full 6.27 ms (kept); Q 2 / N full 6.27; Q 3 / N 2 6.41; Q 1 / N 1 6.56; Q full / N 2 6.56.
#ifndef K3_ROLL_Q
#define K3_ROLL_Q 3
#endif
#ifndef K3_ROLL_N
#define K3_ROLL_N 0
#endif
#ifndef K3_ROLL_B1
#define K3_ROLL_B1 0
#endif
#ifndef K3_ROLL_DL
#define K3_ROLL_DL 1
#endif
// Fill the per-CTA shared table copy from the __constant__ tables (1) or from global memory (0)
#ifndef TAB_CONST
#define TAB_CONST 1
#endif
// Units per CTA of the batched 3D force kernel (r02): a CTA evaluates GEN_UPC consecutive units
// (consecutive instances of one closure element) in turn, loading the 1D tables once.
#ifndef GEN_UPC
#define GEN_UPC 1
#endif
template <int DIM, int EPB, int MODE, bool BATCHED>
__host__ __device__ constexpr int units_per_cta() {
  return (DIM == 3 && EPB == 1 && BATCHED && MODE == MODE_FORCE) ? GEN_UPC : 1;
}
template <int K>
struct Split {
  static constexpr int F1 = K == 2 ? SPLIT_F1_K2 : SPLIT_F1_K3;   // divides Q
  static constexpr int F2 = K == 2 ? SPLIT_F2_K2 : SPLIT_F2_K3;   // divides Q
  static constexpr int B1 = K == 2 ? SPLIT_B1_K2 : SPLIT_B1_K3;   // 1 or 3
  static constexpr int B2 = K == 2 ? SPLIT_B2_K2 : SPLIT_B2_K3;   // divides N
  static constexpr int B3 = K == 2 ? SPLIT_B3_K2 : SPLIT_B3_K3;   // divides N
};
template <int V>
struct IC {
  static constexpr int value = V;
};
// body(IC<part>{}) for the runtime part in [0, S): one compiled copy per part
template <int S, int P = 0, class F>
__device__ __forceinline__ void part_dispatch(int part, F &&body) {
  if constexpr (P + 1 >= S) {
    body(IC<P>{});
  } else {
    if (part == P) body(IC<P>{});
    else part_dispatch<S, P + 1>(part, body);
  }
}

// ----------------------------------------------------------------------------- tables
// The 1D tables in __constant__ memory (filled at context creation, packed order w, B, G, Bl):
// in the register-blocked 3D stages below every table index is a compile-time constant, so the
// entries are read as uniform constant-bank operands (no shared-memory loads).
struct Tab24 {
  double w[4];
  double B[4][3];
  double G[4][3];
  double Bl[4][2];
};
struct Tab36 {
  double w[6];
  double B[6][4];
  double G[6][4];
  double Bl[6][3];
};
__constant__ Tab24 c_t24;
__constant__ Tab36 c_t36;
template <int K, int Q>
struct CTab;
template <>
struct CTab<2, 4> {
  static __device__ __forceinline__ double B(int q, int a) { return c_t24.B[q][a]; }
  static __device__ __forceinline__ double G(int q, int a) { return c_t24.G[q][a]; }
  static __device__ __forceinline__ double Bl(int q, int j) { return c_t24.Bl[q][j]; }
};
template <>
struct CTab<3, 6> {
  static __device__ __forceinline__ double B(int q, int a) { return c_t36.B[q][a]; }
  static __device__ __forceinline__ double G(int q, int a) { return c_t36.G[q][a]; }
  static __device__ __forceinline__ double Bl(int q, int j) { return c_t36.Bl[q][j]; }
};

// ----------------------------------------------------------------------------- kernel
template <int DIM, int K, int Q, int NF, int EPB_>
struct KCfg {
  using G = Geo<DIM, K, Q, NF, EPB_>;
  // occupancy target.  3D Q3 (224-thread CTAs): 4 CTAs/SM at 72 registers measured best
  // (10.75 ms on C3 vs 12.0 ms at 3 CTAs / 80 registers, 11.2 ms at 5 CTAs / 56 registers:
  // occupancy outweighs the extra spills; profiles/ab/).
  static constexpr int MINB = G::NT >= 224 ? GEN_MINB224 : (G::NT >= 128 ? 5 : GEN_MINB64);
};

template <int MODE, bool HAS_W>
__host__ __device__ constexpr int nfields() { return (MODE == MODE_MQ || MODE == MODE_FTW) ? 1 : (HAS_W ? 3 : 2); }

template <int DIM, int K, int Q, bool VISC, int MODE, bool BATCHED, bool HAS_W, int EPB_ = 0>
__global__ void __launch_bounds__(KCfg<DIM, K, Q, nfields<MODE, HAS_W>(), EPB_>::G::NT,
                                  KCfg<DIM, K, Q, nfields<MODE, HAS_W>(), EPB_>::MINB)
force_kernel(const Params P) {
  constexpr int NF = nfields<MODE, HAS_W>();
  constexpr bool WANT_E = MODE != MODE_MQ && MODE != MODE_FTW;
  constexpr int K3UQ = (K == 3 && K3_ROLL_Q > 0) ? K3_ROLL_Q : 64;  // loops over q
  constexpr int K3UN = (K == 3 && K3_ROLL_N > 0) ? K3_ROLL_N : 64;  // loops over a / j
  constexpr int K3UB1 = (K == 3 && K3_ROLL_B1 > 0) ? K3_ROLL_B1 : 64;  // b1: loop over a3
  constexpr int K3UD = (K == 3 && K3_ROLL_DL > 0) ? K3_ROLL_DL : 64;   // b1: loop over dl
  using G = Geo<DIM, K, Q, NF, EPB_>;
  constexpr int N = G::N, M = G::M, ND = G::ND, NE = G::NE, NQ = G::NQ, EPB = G::EPB,
                NT = G::NT;
  extern __shared__ __align__(16) double smem[];
  double *sW = smem;                    // [Q]
  double *sB = sW + Q;                  // [Q][N]
  double *sG = sB + Q * N;              // [Q][N]
  double *sBl = sG + Q * N;             // [Q][M]
  double *units = smem + G::TABD;       // EPB * UNIT
  int *snode = (int *)(units + EPB * G::UNIT);             // [EPB][ND]
  unsigned long long *skey = (unsigned long long *)(snode + (EPB * ND + 1) / 2 * 2);  // [EPB]

  const int tid = threadIdx.x;
  const int u = tid / NQ;               // unit within CTA (may be >= EPB for pad threads)
  const int lt = tid - u * NQ;          // Gauss point within unit
  constexpr int UPC = units_per_cta<DIM, EPB, MODE, BATCHED>();
  const int B = BATCHED ? P.B : 1;

  // --- tables to shared memory (from the __constant__ copy where there is one: a constant-
  // cache hit instead of a global load at every CTA's start)
  if constexpr (TAB_CONST && ((K == 2 && Q == 4) || (K == 3 && Q == 6))) {
    const double *ct = K == 2 ? &c_t24.w[0] : &c_t36.w[0];  // packed w, B, G, Bl = sW.. layout
    for (int i = tid; i < Q + 2 * Q * N + Q * M; i += NT) sW[i] = ct[i];
  } else {
    for (int i = tid; i < Q; i += NT) sW[i] = P.tab_w[i];
    for (int i = tid; i < Q * N; i += NT) { sB[i] = P.tab_B[i]; sG[i] = P.tab_G[i]; }
    for (int i = tid; i < Q * M; i += NT) sBl[i] = P.tab_Bl[i];
  }
#pragma unroll 1
  for (int iu = 0; iu < UPC; ++iu) {
  const int unit0 = (blockIdx.x * UPC + iu) * EPB;
  if (UPC > 1) {
    if (unit0 >= P.n_units) break;      // (uniform over the CTA)
    if (iu > 0) __syncthreads();        // the previous unit's last shared-memory reads
  }
  for (int i = tid; i < EPB; i += NT) skey[i] = ~0ull;

  // --- S1 gather
  constexpr bool GATHER1 = GEN_GATHER1 && DIM == 3 && EPB == 1 && NT >= ND + NE;
  if constexpr (GATHER1) {
    // one unit per CTA: thread a < ND loads node a's id and then its NF x DIM values (no
    // barrier between the two), threads ND .. ND+NE-1 load the e dofs
    const int gu = unit0;
    if (gu < P.n_units) {
      const int lr = BATCHED ? unit_row(P, gu) : gu;
      const int l0 = P.unit_elem ? P.unit_elem[lr] : lr;
      const int b0 = BATCHED ? gu - lr * B : 0;
      if (tid < ND) {
        const int nd = __ldg(P.elem_nodes + (int64_t)l0 * ND + tid);
        // the node's assembly slot, for the F.1 write-out at the end (snode is free here)
        if (MODE == MODE_FORCE) snode[tid] = __ldg(P.slot + (int64_t)l0 * ND + tid);
#pragma unroll
        for (int f = 0; f < NF; ++f) {
          const double *src = NF == 1 ? P.x : (f == 0 ? P.x : (f == 1 ? P.v : P.w));
#pragma unroll
          for (int c = 0; c < DIM; ++c)
            units[G::XOFF + (f * DIM + c) * ND + tid] = __ldg(src + ((int64_t)c * P.ld_nodes + nd) * B + b0);
        }
      } else if (WANT_E && tid < ND + NE) {
        const int j = tid - ND;
        units[G::XOFF + G::NF * DIM * ND + j] = __ldg(P.e + ((int64_t)l0 * NE + j) * B + b0);
      }
    } else {
      for (int i = tid; i < G::NF * DIM * ND + NE; i += NT) units[G::XOFF + i] = 0.0;
    }
  } else {
  // node ids, then fields (unit fastest for coalescing across instances)
  for (int i = tid; i < EPB * ND; i += NT) {
    const int uu = i % EPB, a = i / EPB;
    const int gu = unit0 + uu;
    int nd = 0;
    if (gu < P.n_units) {
      const int lr = BATCHED ? unit_row(P, gu) : gu;
      nd = P.elem_nodes[(P.unit_elem ? P.unit_elem[lr] : lr) * ND + a];
    }
    snode[uu * ND + a] = nd;
  }
  __syncthreads();
  {
    constexpr int total = EPB * NF * DIM * ND;
    for (int i = tid; i < total; i += NT) {
      const int uu = i % EPB;
      int r = i / EPB;
      const int a = r % ND; r /= ND;
      const int c = r % DIM;
      const int f = r / DIM;
      const int gu = unit0 + uu;
      double val = 0.0;
      if (gu < P.n_units) {
        const int b = BATCHED ? gu - unit_row(P, gu) * B : 0;
        const int64_t idx = ((int64_t)c * P.ld_nodes + snode[uu * ND + a]) * B + b;
        const double *src = NF == 1 ? P.x : (f == 0 ? P.x : (f == 1 ? P.v : P.w));
        val = __ldg(src + idx);
      }
      units[uu * G::UNIT + G::XOFF + (f * DIM + c) * ND + a] = val;
    }
    if (WANT_E) {
      for (int i = tid; i < EPB * NE; i += NT) {
        const int uu = i % EPB, j = i / EPB;
        const int gu = unit0 + uu;
        double val = 0.0;
        if (gu < P.n_units) {
          const int l = BATCHED ? unit_row(P, gu) : gu, b = BATCHED ? gu - l * B : 0;
          val = __ldg(P.e + ((int64_t)l * NE + j) * B + b);
        }
        units[uu * G::UNIT + G::XOFF + G::NF * DIM * ND + j] = val;
      }
    }
  }
  }  // !GATHER1
  __syncthreads();

  const bool active = (u < EPB) && (unit0 + u < P.n_units) && (lt < NQ);
  const int uc = u < EPB ? u : EPB - 1;  // clamp pad threads onto a real unit buffer (reads only)
  double *U = units + uc * G::UNIT;
  double *Xs = U + G::XOFF;               // [NF][DIM][ND]
  double *Es = Xs + G::NF * DIM * ND;     // [NE]
  double *Wk = U + G::WKOFF;              // work region (16-byte aligned)
  const int gu = (unit0 + uc < P.n_units) ? unit0 + uc : 0;  // safe unit for reads
  const int lraw = BATCHED ? unit_row(P, gu) : gu;  // element (or, over compacted units, S0 row)
  const int l = P.unit_elem ? P.unit_elem[lraw] : lraw;
  const int b = BATCHED ? gu - lraw * B : 0;
  const int gid = P.elem_gid ? P.elem_gid[l] : l;

  // --- S2 forward contractions (canonical order, DESIGN A.2)
  double J[3][3], Gv[3][3], Gw[3][3];
  double eq = 0.0;
  int q1i, q2i, q3i = 0;
  const int lq = lt < NQ ? lt : 0;
  if (DIM == 2) { q1i = lq % Q; q2i = lq / Q; }
  else { q1i = lq % Q; q2i = (lq / Q) % Q; q3i = lq / (Q * Q); }

  if (DIM == 3) {
    double *S1b = Wk;                              // [NF*DIM: S1FC][2: S1X][Q: S1Q1X][N][N]
    double *S2b = Wk + G::S1TOT;                   // [NF*DIM: S2FC][3][Q][S2Q1: Q][N]
    double *E1b = S2b + G::S2TOT;                  // [Q][M][M]
    double *E2b = E1b + G::E1;                     // [Q][Q][M]
    using CT = CTab<K, Q>;
    if (u < EPB) {
      // stage 1: contract a1.  One task per (field comp, a2, a3) line: its N dofs are loaded
      // once and give all Q x {B, G} outputs (canonical FMA order per output, DESIGN A.2).
      constexpr int SP1 = Split<K>::F1, QP1 = Q / SP1, T1 = NF * DIM * N * N;
      static_assert(Q % SP1 == 0, "SPLIT_F1 must divide Q");
      for (int t = lt; t < T1 * SP1; t += NQ) {
        const int t1 = t % T1;
        const int a23 = t1 % (N * N), fc = t1 / (N * N);
        const int a2 = a23 % N, a3 = a23 / N;
        const double *src = Xs + fc * ND + (a3 * N + a2) * N;
        double x[N];
        if constexpr (N % 2 == 0 && FP_VEC) {   // 16-byte aligned line: LDS.128
#pragma unroll
          for (int a1 = 0; a1 < N; a1 += 2) {
            const double2 x2 = *reinterpret_cast<const double2 *>(src + a1);
            x[a1] = x2.x;
            x[a1 + 1] = x2.y;
          }
        } else {
#pragma unroll
          for (int a1 = 0; a1 < N; ++a1) x[a1] = src[a1];
        }
        // S1b layout [fc][B|G][q1][a3][a2] (a2 fastest: stage 2 reads its pencils contiguously)
        double *dB = S1b + fc * G::S1FC + a3 * N + a2;
        double *dG = S1b + fc * G::S1FC + G::S1X + a3 * N + a2;
        part_dispatch<SP1>(t / T1, [&](auto pc) {
          constexpr int part = decltype(pc)::value;
#pragma unroll (K3UQ)
          for (int qq = 0; qq < QP1; ++qq) {
            const int q1 = part * QP1 + qq;
            double ab = CT::B(q1, 0) * x[0], ag = CT::G(q1, 0) * x[0];
#pragma unroll
            for (int a1 = 1; a1 < N; ++a1) {
              ab = __fma_rn(CT::B(q1, a1), x[a1], ab);
              ag = __fma_rn(CT::G(q1, a1), x[a1], ag);
            }
            dB[q1 * G::S1Q1X] = ab;
            dG[q1 * G::S1Q1X] = ag;
          }
        });
      }
      if (WANT_E) {  // (j2, j3) lines, on the highest lanes
        for (int t = NQ - 1 - lt; t < M * M; t += NQ) {
          const int j2 = t % M, j3 = t / M;
          const double *src = Es + (j3 * M + j2) * M;
          double ev[M];
#pragma unroll
          for (int j1 = 0; j1 < M; ++j1) ev[j1] = src[j1];
#pragma unroll (K3UQ)
          for (int q1 = 0; q1 < Q; ++q1) {
            double acc = CT::Bl(q1, 0) * ev[0];
#pragma unroll
            for (int j1 = 1; j1 < M; ++j1) acc = __fma_rn(CT::Bl(q1, j1), ev[j1], acc);
            E1b[(q1 * M + j2) * M + j3] = acc;
          }
        }
      }
    }
    __syncthreads();
    if (u < EPB) {
      // stage 2: contract a2 ; kind 0: B.UG (d/dxi1), 1: G.UB (d/dxi2), 2: B.UB (d/dxi3).
      // One task per (field comp, q1, a3): its 2N stage-1 values give all Q x 3 outputs.
      constexpr int SP2 = Split<K>::F2, QP2 = Q / SP2, T2 = NF * DIM * Q * N;
      static_assert(Q % SP2 == 0, "SPLIT_F2 must divide Q");
      for (int t = lt; t < T2 * SP2; t += NQ) {
        const int t2 = t % T2;
        // LK2: q1 fastest over the lanes (conflict-free stage-2 stores with the padded strides)
        int a3 = G::LK2 ? (t2 / Q) % N : t2 % N;
        int q1 = G::LK2 ? t2 % Q : (t2 / N) % Q;
        int fc = t2 / (Q * N);
        if constexpr (PERM_K3 && K == 3 && G::NF * DIM == 6 && N == 4 && Q == 6) {
          // Q3: each half-warp takes four (fc, q1) pencils whose stage-2 store offsets are
          // {0, 4, 8, 12} mod 16 doubles (fc stride 540, q1 stride 30): four consecutive fc of
          // one q1, then {4, 5} x {q1, q1 + 4} for q1 = 0, 1, then {4, 5} x {2, 3}
          // (modelled stage-2 store wavefronts per element 324 -> 180, tools/bank_sim.py)
          const int pc = t2 >> 2;
          a3 = t2 & 3;
          if (pc < 24) {
            q1 = pc >> 2;
            fc = pc & 3;
          } else {
            const int r = pc - 24, g = r >> 2, wi = r & 3;
            fc = 4 + (wi & 1);
            q1 = g + (wi >> 1) * (g < 2 ? 4 : 1);
          }
        }
        const double *pB = S1b + fc * G::S1FC + q1 * G::S1Q1X + a3 * N;
        const double *pG = pB + G::S1X;
        double uB[N], uG[N];
#pragma unroll
        for (int a2 = 0; a2 < N; ++a2) { uB[a2] = pB[a2]; uG[a2] = pG[a2]; }
        double *dst = S2b + fc * G::S2FC + q1 * G::S2Q1 + a3;
        part_dispatch<SP2>(t / T2, [&](auto pc) {
          constexpr int part = decltype(pc)::value;
#pragma unroll (K3UQ)
          for (int qq = 0; qq < QP2; ++qq) {
            const int q2 = part * QP2 + qq;
            double d1 = CT::B(q2, 0) * uG[0], d2 = CT::G(q2, 0) * uB[0], d3 = CT::B(q2, 0) * uB[0];
#pragma unroll
            for (int a2 = 1; a2 < N; ++a2) {
              d1 = __fma_rn(CT::B(q2, a2), uG[a2], d1);
              d2 = __fma_rn(CT::G(q2, a2), uB[a2], d2);
              d3 = __fma_rn(CT::B(q2, a2), uB[a2], d3);
            }
            dst[0 * G::S2 + q2 * N] = d1;
            dst[1 * G::S2 + q2 * N] = d2;
            dst[2 * G::S2 + q2 * N] = d3;
          }
        });
      }
      if (WANT_E) {  // (q1, j3) lines, on the highest lanes
        for (int t = NQ - 1 - lt; t < Q * M; t += NQ) {
          const int j3 = t % M, q1 = t / M;
          const double *src = E1b + q1 * M * M + j3;
          double ev[M];
#pragma unroll
          for (int j2 = 0; j2 < M; ++j2) ev[j2] = src[j2 * M];
#pragma unroll (K3UQ)
          for (int q2 = 0; q2 < Q; ++q2) {
            double acc = CT::Bl(q2, 0) * ev[0];
#pragma unroll
            for (int j2 = 1; j2 < M; ++j2) acc = __fma_rn(CT::Bl(q2, j2), ev[j2], acc);
            if constexpr (G::LK2 && EJ_K2) E2b[(j3 * Q + q1) * Q + q2] = acc;
            else E2b[(q1 * Q + q2) * M + j3] = acc;
          }
        }
      }
    }
    __syncthreads();
    // stage 3 (per Gauss point): contract a3 -- see forward_point
  } else {
    double *S1b = Wk;                              // [NF*DIM][2][Q][N]
    double *E1b = Wk + G::NF * DIM * 2 * G::S1;    // [Q][M]
    if (u < EPB) {
      constexpr int cnt1 = NF * DIM * 2 * Q * N;
      for (int o = lt; o < cnt1; o += NQ) {
        int r = o;
        const int a2 = r % N; r /= N;
        const int q1 = r % Q; r /= Q;
        const int bg = r % 2;
        const int fc = r / 2;
        const double *tab = (bg ? sG : sB) + q1 * N;
        const double *src = Xs + fc * ND + a2 * N;
        double acc = tab[0] * src[0];
#pragma unroll
        for (int a1 = 1; a1 < N; ++a1) acc = __fma_rn(tab[a1], src[a1], acc);
        S1b[((fc * 2 + bg) * Q + q1) * N + a2] = acc;
      }
      if (WANT_E) {
        for (int o = lt; o < Q * M; o += NQ) {
          const int j2 = o % M, q1 = o / M;
          const double *tab = sBl + q1 * M;
          const double *src = Es + j2 * M;
          double acc = tab[0] * src[0];
#pragma unroll
          for (int j1 = 1; j1 < M; ++j1) acc = __fma_rn(tab[j1], src[j1], acc);
          E1b[q1 * M + j2] = acc;
        }
      }
    }
    __syncthreads();
  }
  forward_point<DIM, K, Q, NF, WANT_E>(sB, sG, sBl, Wk, q1i, q2i, q3i, J, Gv, Gw, eq);

  // --- MODE_FTW: FTw[j] = sum_q psi_j(xi_q) (S_q : gradhat w_q) from the stored S_q
  if (MODE == MODE_FTW) {
    __syncthreads();                      // forward buffers dead
    double *As = Wk;                      // [NQ]
    double *F1b = As + NQ;                // f1
    double *F2b = F1b + G::F1B;           // f2 (3D)
    if (u < EPB && lt < NQ) {
      const double *S = P.S_load + (int64_t)(unit0 + uc) * DIM * DIM * NQ + lt;
      double A = 0.0;
#pragma unroll
      for (int c = 0; c < DIM; ++c)
#pragma unroll
        for (int d = 0; d < DIM; ++d) A = __fma_rn(S[(c * DIM + d) * NQ], J[c][d], A);
      As[lt] = A;
    }
    __syncthreads();
    const int row = (u < EPB && unit0 + u < P.n_units)
                        ? (P.unit_elem ? lraw : (P.ftw_row ? P.ftw_row[l] : l)) : -1;
    if (DIM == 3) {
      if (u < EPB)
        for (int o = lt; o < Q * Q * M; o += NQ) {
          const int j3 = o % M, q2 = (o / M) % Q, q1 = o / (M * Q);
          double acc = 0.0;
#pragma unroll
          for (int q3 = 0; q3 < Q; ++q3) acc = __fma_rn(sBl[q3 * M + j3], As[q1 + Q * q2 + Q * Q * q3], acc);
          F1b[o] = acc;
        }
      __syncthreads();
      if (u < EPB)
        for (int o = lt; o < Q * M * M; o += NQ) {
          const int j3 = o % M, j2 = (o / M) % M, q1 = o / (M * M);
          double acc = 0.0;
#pragma unroll
          for (int q2 = 0; q2 < Q; ++q2) acc = __fma_rn(sBl[q2 * M + j2], F1b[(q1 * Q + q2) * M + j3], acc);
          F2b[o] = acc;
        }
      __syncthreads();
      if (row >= 0)
        for (int o = lt; o < NE; o += NQ) {
          const int j1 = o % M, j2 = (o / M) % M, j3 = o / (M * M);
          double acc = 0.0;
#pragma unroll
          for (int q1 = 0; q1 < Q; ++q1) acc = __fma_rn(sBl[q1 * M + j1], F2b[(q1 * M + j2) * M + j3], acc);
          P.FTw[((int64_t)row * NE + o) * B + b] = acc;
        }
    } else {
      if (u < EPB)
        for (int o = lt; o < Q * M; o += NQ) {
          const int j2 = o % M, q1 = o / M;
          double acc = 0.0;
#pragma unroll
          for (int q2 = 0; q2 < Q; ++q2) acc = __fma_rn(sBl[q2 * M + j2], As[q1 + Q * q2], acc);
          F1b[o] = acc;
        }
      __syncthreads();
      if (row >= 0)
        for (int o = lt; o < NE; o += NQ) {
          const int j1 = o % M, j2 = o / M;
          double acc = 0.0;
#pragma unroll
          for (int q1 = 0; q1 < Q; ++q1) acc = __fma_rn(sBl[q1 * M + j1], F1b[q1 * M + j2], acc);
          P.FTw[((int64_t)row * NE + o) * B + b] = acc;
        }
    }
    return;
  }

  // --- MODE_MQ: m_q = rho0_K detJ0 (density elimination)
  if (MODE == MODE_MQ) {
    if (active) {
      const double det0 = det_only<DIM>(J);
      P.mq_out[(int64_t)gid * NQ + lt] = P.rho0[gid] * det0;
    }
    return;
  }
  if (!HAS_W) {
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int d = 0; d < 3; ++d) Gw[c][d] = 0.0;
  }

  // --- S3 pointwise: fast pass, exact IEEE re-run where a fast path was out of range
  const double gam = __ldg(P.gamma + gid);
  const double mq = __ldg(P.mq + (int64_t)gid * NQ + lq);
  double wq = sW[q1i] * sW[q2i];
  if (DIM == 3) wq = wq * sW[q3i];
  const PhysIn ph{P.q1, P.q2, P.alpha, P.alpha_mu};
  PointOut po;
  {
    ArithFast af;
    pointwise<DIM, VISC, HAS_W, true, ArithFast,
              DIM == 3 && ((F3_COMPACT && K == 2) || (F3_COMPACT_Q3 && K == 3))>(
        af, J, Gv, Gw, eq, mq, gam, wq, ph, po);
    if (!af.ok) {
      // rare: some fast div/sqrt left its exact range; recompute the inputs from shared
      // memory (not kept live across the fast pass) and re-run with IEEE operators.
      forward_point<DIM, K, Q, NF, true>(sB, sG, sBl, Wk, q1i, q2i, q3i, J, Gv, Gw, eq);
      if (!HAS_W) {
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int d = 0; d < 3; ++d) Gw[c][d] = 0.0;
      }
      ArithIeee ai;
      pointwise<DIM, VISC, HAS_W, false>(ai, J, Gv, Gw, eq, __ldg(P.mq + (int64_t)gid * NQ + lq),
                                         __ldg(P.gamma + gid), wq, ph, po);
    }
  }

  if (MODE == MODE_FORCE && P.S_store && active) {
    const int64_t si = s_index(P, unit0 + u, l, b);
    if (si >= 0) {
#pragma unroll
      for (int c = 0; c < DIM; ++c)
#pragma unroll
        for (int d = 0; d < DIM; ++d)
          P.S_store[(si * DIM * DIM + c * DIM + d) * NQ + lt] = po.S[c][d];
    }
  }

  // --- S6 dt: status flags, then min of order-preserving keys
  unsigned long long key = ~0ull;
  if (active) {
    if (!(po.det > 0.0)) atomicMin(&P.st[b].first_bad, (unsigned long long)gid);
    if (isnan(po.dtq)) atomicOr(&P.st[b].nan_flag, 1u);
    else key = dt_key(po.dtq);
  }
  if (GEN_WARP_KEY && DIM == 3 && EPB == 1) {
    // one unit per CTA: each warp's minimum goes straight to the unit's status word (no
    // shared-memory reduction, no CTA barrier before the backward pass)
    key = warp_min_u64(key);
    if ((tid & 31) == 0 && key != ~0ull && unit0 < P.n_units) atomicMin(&P.st[b].dt_key, key);
  } else {
  {
    constexpr bool WARP_IN_UNIT = (NQ % 32 == 0) || (EPB == 1);
    constexpr bool HALF = (NQ == 16);
    if (WARP_IN_UNIT || HALF) {
      constexpr int width = WARP_IN_UNIT ? 32 : 16;
#pragma unroll
      for (int off = width / 2; off > 0; off >>= 1) {
        const unsigned long long o = __shfl_xor_sync(0xffffffffu, key, off);
        key = o < key ? o : key;
      }
      if ((tid & (width - 1)) == 0 && u < EPB) atomicMin(&skey[u], key);
    } else {
      if (u < EPB) atomicMin(&skey[u], key);
    }
  }
  __syncthreads();
  if (!BATCHED) {
    if (tid == 0) {
      unsigned long long k = skey[0];
      for (int i = 1; i < EPB; ++i) k = skey[i] < k ? skey[i] : k;
      if (k != ~0ull) atomicMin(&P.st[0].dt_key, k);
    }
  } else if (tid < EPB) {
    const int g2 = unit0 + tid;
    if (g2 < P.n_units && skey[tid] != ~0ull) atomicMin(&P.st[g2 - unit_row(P, g2) * B].dt_key, skey[tid]);
  }
  }
  if (MODE == MODE_DT) {
    pdl_trigger();
    return;
  }
  if (!G::SEPS) __syncthreads();  // forward buffers are dead from here on (S4 reuses them)

  // --- S4 backward
  double *Ss = G::SEPS ? Wk + G::FWD : Wk;  // [DIM*DIM][NQ]
  double *As = Ss + DIM * DIM * NQ;         // [NQ]
  double *Tb = G::SEPS ? Wk : As + NQ;
  double *F1b = G::LK2 ? Tb + G::TB : Tb + G::TB + G::WB;
  double *Wb = G::LK2 ? Ss : Tb + G::TB;          // LK2: over the dead point stresses
  double *F2b = G::LK2 ? Ss + G::WB : F1b + G::F1B;
  // (the __syncthreads above separates the last forward read from these writes)
  // 3D Q3: point stresses stored [c][d][q1][q2][q3] (q3 fastest: the b1 / f1 pencils over q3
  // are contiguous; C3 -1 %); Q2 and 2D: [c][d][q] with q = q1 + Q q2 (+ Q^2 q3) -- for Q = 4
  // the q3-fastest store is an 8-way bank conflict (C2 +6 %: profiles/ab/r02_ab5_*)
  constexpr bool SQ3 = DIM == 3 && K == 3;
  const int spos = SQ3 ? (q1i + Q * q2i) * Q + q3i : lt;
  if (u < EPB && lt < NQ) {
#pragma unroll
    for (int c = 0; c < DIM; ++c)
#pragma unroll
      for (int d = 0; d < DIM; ++d) Ss[(c * DIM + d) * NQ + spos] = po.S[c][d];
    As[spos] = po.A;
  }
  __syncthreads();
  const int64_t slot_base = (int64_t)l * ND;
  if (DIM == 3) {
    using CT = CTab<K, Q>;
    if (u < EPB) {
      // b1: T[dl][c][q1][q2][a3] = sum_q3 (dl==2 ? G : B)[q3][a3] S[c][dl](q1,q2,q3); one task
      // per (c, q1, q2) pencil: its 3Q stresses give all 3 x N outputs
      constexpr int SB1 = Split<K>::B1, DLP = 3 / SB1, TB1 = DIM * Q * Q;
      static_assert(3 % SB1 == 0, "SPLIT_B1 must divide 3");
      for (int t = lt; t < TB1 * SB1; t += NQ) {
        const int tb = t % TB1;
        const int q12 = tb % (Q * Q), c = tb / (Q * Q);
        const int q1 = q12 % Q, q2 = q12 / Q;
        part_dispatch<SB1>(t / TB1, [&](auto pc) {
          constexpr int part = decltype(pc)::value;
#pragma unroll (K3UD)
          for (int dd = 0; dd < DLP; ++dd) {
            const int dl = part * DLP + dd;
            const double *src = Ss + (c * DIM + dl) * NQ + (SQ3 ? q12 * Q : q12);
            double sv[Q];
#pragma unroll
            for (int q3 = 0; q3 < Q; ++q3) sv[q3] = src[SQ3 ? q3 : q3 * Q * Q];
            // Tb layout [dl][c][q1][a3][q2] (q2 fastest: b2 reads its pencils contiguously)
            double *dst = Tb + dl * G::TDL + c * G::TC + q1 * G::TQ1 + q2;
#pragma unroll (K3UB1)
            for (int a3 = 0; a3 < N; ++a3) {
              double acc = 0.0;
#pragma unroll
              for (int q3 = 0; q3 < Q; ++q3)
                acc = __fma_rn(dl == 2 ? CT::G(q3, a3) : CT::B(q3, a3), sv[q3], acc);
              dst[a3 * G::TA3] = acc;
            }
          }
        });
      }
      // f1[q1][q2][j3] = sum_q3 Bl[q3][j3] A(q1,q2,q3), (q1, q2) pencils on the highest lanes
      for (int t = NQ - 1 - lt; t < Q * Q; t += NQ) {
        double av[Q];
#pragma unroll
        for (int q3 = 0; q3 < Q; ++q3) av[q3] = As[SQ3 ? t * Q + q3 : t + Q * Q * q3];
        const int q1 = t % Q, q2 = t / Q;
#pragma unroll (K3UN)
        for (int j3 = 0; j3 < M; ++j3) {
          double acc = 0.0;
#pragma unroll
          for (int q3 = 0; q3 < Q; ++q3) acc = __fma_rn(CT::Bl(q3, j3), av[q3], acc);
          F1b[(q1 * Q + q2) * M + j3] = acc;
        }
      }
    }
    __syncthreads();
    if (u < EPB) {
      // b2: W1[c][q1][a2][a3] = sum_q2 B[q2][a2] T0 ; W23 = sum_q2 G[q2][a2] T1 + B[q2][a2] T2;
      // one task per (c, q1, a3) pencil
      constexpr int SB2 = Split<K>::B2, A2P = N / SB2, TB2 = DIM * Q * N;
      static_assert(N % SB2 == 0, "SPLIT_B2 must divide N");
      for (int t = lt; t < TB2 * SB2; t += NQ) {
        const int tb = t % TB2;
        const int a3 = G::XK2 ? (tb / Q) % N : tb % N;   // XK2: q1 fastest over the lanes
        const int q1 = G::XK2 ? tb % Q : (tb / N) % Q;
        const int c = tb / (Q * N);
        const double *t0 = Tb + 0 * G::TDL + c * G::TC + q1 * G::TQ1 + a3 * G::TA3;
        const double *t1 = Tb + 1 * G::TDL + c * G::TC + q1 * G::TQ1 + a3 * G::TA3;
        const double *t2 = Tb + 2 * G::TDL + c * G::TC + q1 * G::TQ1 + a3 * G::TA3;
        double v0[Q], v1[Q], v2[Q];
#pragma unroll
        for (int q2 = 0; q2 < Q; ++q2) { v0[q2] = t0[q2]; v1[q2] = t1[q2]; v2[q2] = t2[q2]; }
        // Wb layout [W1|W23][c][a2][a3][q1] (q1 fastest: b3 reads its pencils contiguously)
        double *w1 = Wb + 0 * G::WW + c * G::WC + a3 * G::WA + q1;
        double *w23 = Wb + 1 * G::WW + c * G::WC + a3 * G::WA + q1;
        part_dispatch<SB2>(t / TB2, [&](auto pc) {
          constexpr int part = decltype(pc)::value;
#pragma unroll (K3UN)
          for (int aa = 0; aa < A2P; ++aa) {
            const int a2 = part * A2P + aa;
            double acc1 = 0.0, acc23 = 0.0;
#pragma unroll
            for (int q2 = 0; q2 < Q; ++q2) {
              acc1 = __fma_rn(CT::B(q2, a2), v0[q2], acc1);
              acc23 = __fma_rn(CT::G(q2, a2), v1[q2], acc23);
              acc23 = __fma_rn(CT::B(q2, a2), v2[q2], acc23);
            }
            w1[a2 * N * G::WA] = acc1;
            w23[a2 * N * G::WA] = acc23;
          }
        });
      }
      // f2[q1][j2][j3] = sum_q2 Bl[q2][j2] f1[q1][q2][j3], (q1, j3) pencils on the highest lanes
      for (int t = NQ - 1 - lt; t < Q * M; t += NQ) {
        const int j3 = t % M, q1 = t / M;
        double fv[Q];
#pragma unroll
        for (int q2 = 0; q2 < Q; ++q2) fv[q2] = F1b[(q1 * Q + q2) * M + j3];
#pragma unroll (K3UN)
        for (int j2 = 0; j2 < M; ++j2) {
          double acc = 0.0;
#pragma unroll
          for (int q2 = 0; q2 < Q; ++q2) acc = __fma_rn(CT::Bl(q2, j2), fv[q2], acc);
          F2b[(q1 * M + j2) * M + j3] = acc;
        }
      }
    }
    __syncthreads();
    if (u < EPB && unit0 + u < P.n_units) {
      // b3: F1[c][a] = sum_q1 G[q1][a1] W1[c][q1][a2][a3] + B[q1][a1] W23[c][q1][a2][a3];
      // one task per (c, a2, a3) pencil writes the N nodes a1 = 0..N-1 of component c
      constexpr int SB3 = Split<K>::B3, A1P = N / SB3, TB3 = DIM * N * N;
      static_assert(N % SB3 == 0, "SPLIT_B3 must divide N");
      for (int t = lt; t < TB3 * SB3; t += NQ) {
        const int tb = t % TB3;
        const int a23 = tb % (N * N), c = tb / (N * N);
        double w1v[Q], w23v[Q];
#pragma unroll
        for (int q1 = 0; q1 < Q; ++q1) {
          w1v[q1] = Wb[0 * G::WW + c * G::WC + a23 * G::WA + q1];
          w23v[q1] = Wb[1 * G::WW + c * G::WC + a23 * G::WA + q1];
        }
        const int a2 = a23 / N, a3 = a23 % N;  // Wb index a2 * N + a3
        const int a0 = (a3 * N + a2) * N;      // node a = a1 + N a2 + N^2 a3
        part_dispatch<SB3>(t / TB3, [&](auto pc) {
          constexpr int part = decltype(pc)::value;
#pragma unroll (K3UN)
          for (int aa = 0; aa < A1P; ++aa) {
            const int a1 = part * A1P + aa;
            double acc = 0.0;
#pragma unroll
            for (int q1 = 0; q1 < Q; ++q1) {
              acc = __fma_rn(CT::G(q1, a1), w1v[q1], acc);
              acc = __fma_rn(CT::B(q1, a1), w23v[q1], acc);
            }
            const int s = GATHER1 && MODE == MODE_FORCE ? snode[a0 + a1] : P.slot[slot_base + a0 + a1];
            if (s >= 0) P.evec[((int64_t)s * DIM + c) * B + b] = acc;
          }
        });
      }
      const int row = P.ftw_row ? P.ftw_row[l] : l;
      if (row >= 0) {  // (j2, j3) pencils on the highest lanes
        for (int t = NQ - 1 - lt; t < M * M; t += NQ) {
          const int j2 = t % M, j3 = t / M;
          double fv[Q];
#pragma unroll
          for (int q1 = 0; q1 < Q; ++q1) fv[q1] = F2b[(q1 * M + j2) * M + j3];
#pragma unroll (K3UN)
          for (int j1 = 0; j1 < M; ++j1) {
            double acc = 0.0;
#pragma unroll
            for (int q1 = 0; q1 < Q; ++q1) acc = __fma_rn(CT::Bl(q1, j1), fv[q1], acc);
            P.FTw[((int64_t)row * NE + (j3 * M + j2) * M + j1) * B + b] = acc;
          }
        }
      }
    }
  } else {
    if (u < EPB) {
      // b1: T[dl][c][q1][a2] = sum_q2 (dl==1 ? G : B)[q2][a2] S[c][dl](q1,q2)
      for (int o = lt; o < DIM * DIM * Q * N; o += NQ) {
        int r = o;
        const int a2 = r % N; r /= N;
        const int q1 = r % Q; r /= Q;
        const int c = r % DIM;
        const int dl = r / DIM;
        const double *tab = dl == 1 ? sG : sB;
        const double *src = Ss + (c * DIM + dl) * NQ + q1;
        double acc = 0.0;
#pragma unroll
        for (int q2 = 0; q2 < Q; ++q2) acc = __fma_rn(tab[q2 * N + a2], src[q2 * Q], acc);
        Tb[o] = acc;
      }
      for (int o = lt; o < Q * M; o += NQ) {
        const int j2 = o % M, q1 = o / M;
        double acc = 0.0;
#pragma unroll
        for (int q2 = 0; q2 < Q; ++q2) acc = __fma_rn(sBl[q2 * M + j2], As[q1 + Q * q2], acc);
        F1b[o] = acc;
      }
    }
    __syncthreads();
    if (u < EPB && unit0 + u < P.n_units) {
      for (int a = lt; a < ND; a += NQ) {
        const int a1 = a % N, a2 = a / N;
        double val[3];
#pragma unroll
        for (int c = 0; c < DIM; ++c) {
          double acc = 0.0;
#pragma unroll
          for (int q1 = 0; q1 < Q; ++q1) {
            acc = __fma_rn(sG[q1 * N + a1], Tb[((0 * DIM + c) * Q + q1) * N + a2], acc);
            acc = __fma_rn(sB[q1 * N + a1], Tb[((1 * DIM + c) * Q + q1) * N + a2], acc);
          }
          val[c] = acc;
        }
        const int s = P.slot[slot_base + a];
        if (s >= 0) {
#pragma unroll
          for (int c = 0; c < DIM; ++c) P.evec[((int64_t)s * DIM + c) * B + b] = val[c];
        }
      }
      const int row = P.ftw_row ? P.ftw_row[l] : l;
      if (row >= 0) {
        for (int o = lt; o < NE; o += NQ) {
          const int j1 = o % M, j2 = o / M;
          double acc = 0.0;
#pragma unroll
          for (int q1 = 0; q1 < Q; ++q1) acc = __fma_rn(sBl[q1 * M + j1], F1b[q1 * M + j2], acc);
          P.FTw[((int64_t)row * NE + o) * B + b] = acc;
        }
      }
    }
  }
  }  // units of this CTA
  pdl_trigger();
}

}  // namespace hk

namespace hk {
// ----------------------------------------------------------------------------- assembly
// S5 + S6 completion, launched as a programmatic dependent of the force kernel:
// F1[c][node] (or F1_rows[(c*n_nodes + node)*B + b]) = sum over the node's slots in
// ascending order (slots are laid out by ascending element) -- deterministic; then the
// call's dt is finalised.
template <int DIM>
__global__ void assemble_kernel(int64_t n_nodes, int B, const int32_t *__restrict__ off,
                                const double *__restrict__ evec, double *__restrict__ F1,
                                hydro_devstatus *st, double *dt_out) {
  pdl_wait();
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n_nodes * B) {
    const int64_t node = B == 1 ? t : t / B;
    const int b = B == 1 ? 0 : (int)(t % B);
    const int s0 = off[node], s1 = off[node + 1];
    // one pass over the node's slots for all components (each component still summed in
    // ascending slot order: the same bits as a per-component pass)
    double acc[DIM];
#pragma unroll
    for (int c = 0; c < DIM; ++c) acc[c] = 0.0;
    for (int s = s0; s < s1; ++s) {
      const double *e = evec + (int64_t)s * DIM * B + b;
#pragma unroll
      for (int c = 0; c < DIM; ++c) acc[c] += e[(int64_t)c * B];
    }
#pragma unroll
    for (int c = 0; c < DIM; ++c) F1[((int64_t)c * n_nodes + node) * B + b] = acc[c];
  }
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i < B; i += blockDim.x) finalize_one(st + i, dt_out ? dt_out + i : nullptr);
  }
}

__global__ void finalize_dt_kernel(int B, hydro_devstatus *st, double *dt_out) {
  pdl_wait();
  for (int i = threadIdx.x; i < B; i += blockDim.x) finalize_one(st + i, dt_out ? dt_out + i : nullptr);
}

// ----------------------------------------------------------------------------- self-test
// Bit-equality of the ieee_fast.cuh fast paths against the IEEE operators on seeded
// operands (SplitMix64 counter stream).  dist 0: random sign/mantissa, exponent uniform in
// [-64, 64]; dist 1: raw 64-bit patterns (NaN, inf, subnormals, extremes).  op 0: a/b,
// 1: 1/b, 2: sqrt(|x|) (dist 1: sqrt(x)).  counts[0] += fast-path-valid results whose bits
// differ (must stay 0), counts[1] += operands outside the fast range, counts[2] += total.
__device__ __forceinline__ unsigned long long st_mix(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double st_operand(unsigned long long r, int dist) {
  if (dist == 1) return __longlong_as_double((long long)r);
  const unsigned long long mant = r & 0x000FFFFFFFFFFFFFull;
  const long long ex = (long long)((r >> 52) & 127) - 64 + 1023;
  const unsigned long long sg = (r >> 63) << 63;
  return __longlong_as_double((long long)(sg | ((unsigned long long)ex << 52) | mant));
}

__global__ void selftest_ieee_kernel(unsigned long long seed, long long n, int op, int dist,
                                     unsigned long long *counts) {
  unsigned long long bad = 0, slow = 0, tot = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const unsigned long long r1 = st_mix(seed ^ (2ull * (unsigned long long)i));
    const unsigned long long r2 = st_mix(seed ^ (2ull * (unsigned long long)i + 1ull));
    double a = st_operand(r1, dist), b = st_operand(r2, dist);
    bool ok = true;
    double f, ref;
    if (op == 0) { f = div_fast(a, b, ok); ref = __ddiv_rn(a, b); }
    else if (op == 1) { f = rcp_fast(b, ok); ref = __ddiv_rn(1.0, b); }
    else { if (dist == 0) a = fabs(a); f = sqrt_fast(a, ok); ref = __dsqrt_rn(a); }
    ++tot;
    if (!ok) ++slow;
    else if (__double_as_longlong(f) != __double_as_longlong(ref)) ++bad;
  }
  atomicAdd(counts + 0, bad);
  atomicAdd(counts + 1, slow);
  atomicAdd(counts + 2, tot);
}
}  // namespace hk
