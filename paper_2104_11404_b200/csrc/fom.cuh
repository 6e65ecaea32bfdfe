// fom.cuh -- kernels of the full-order RK2-average time step:
// the kinematic mass operator M_V (matrix-free, sum-factorised, deterministic slot
// assembly), its diagonal (Jacobi preconditioner), the thermodynamic mass blocks M_E,K
// and their inverses, deterministic dot products and the vector updates of
// Eq. RK2-avg.  M_V and M_E are constant in time (Lagrangian mass
// conservation):
//     M_V[a][b]   = sum_K sum_q w_q m_q phi_a(xi_q) phi_b(xi_q)   (each velocity component)
//     M_E,K[i][j] = sum_q w_q m_q psi_i(xi_q) psi_j(xi_q)
// with m_q = rho0_K detJ0(xi_q), the per-point masses the force path already uses.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace hk {

struct MassParams {
  int32_t n_elem;
  int64_t n_nodes;
  const int32_t *elem_nodes;  // [E][ND]
  const int32_t *slot;        // [E][ND]
  const double *mq;           // [E][NQ]
  const double *in;           // [DIM][n_nodes]
  double *evec;               // [slot][DIM]
  int mode;                   // 0: M_V in (per component), 1: diagonal of M_V (in unused)
  const double *tab_w, *tab_B;
};

// One element per CTA, one thread per point (or node): interpolate, weight, project.
template <int DIM, int K, int Q>
__global__ void __launch_bounds__(DIM == 3 ? (Q == 4 ? 64 : 224) : 64)
mass_apply_kernel(const MassParams P) {
  constexpr int N = K + 1, ND = DIM == 3 ? N * N * N : N * N, NQ = DIM == 3 ? Q * Q * Q : Q * Q;
  constexpr int NT = DIM == 3 ? (Q == 4 ? 64 : 224) : 64;
  constexpr int S1 = DIM == 3 ? DIM * Q * N * N : DIM * Q * N;   // stage buffers (doubles)
  constexpr int S2 = DIM == 3 ? DIM * Q * Q * N : 0;
  __shared__ double sW[Q], sB[Q * N];
  __shared__ double X[DIM * ND], U1[S1], U2[S2 > 0 ? S2 : 1], V[DIM * NQ], Y[DIM * ND];
  __shared__ int snode[ND];
  const int tid = threadIdx.x;
  const int e = blockIdx.x;
  for (int i = tid; i < Q; i += NT) sW[i] = P.tab_w[i];
  for (int i = tid; i < Q * N; i += NT) sB[i] = P.tab_B[i];
  for (int a = tid; a < ND; a += NT) snode[a] = P.elem_nodes[(int64_t)e * ND + a];
  __syncthreads();
  if (P.mode == 1) {
    // diagonal: d_a = sum_q w_q m_q phi_a(xi_q)^2  (phi_a = prod of 1D B factors)
    for (int a = tid; a < ND; a += NT) {
      const int a1 = a % N, a2 = (a / N) % N, a3 = a / (N * N);
      double acc = 0.0;
      for (int q = 0; q < NQ; ++q) {
        const int q1 = q % Q, q2 = (q / Q) % Q, q3 = q / (Q * Q);
        double phi = sB[q1 * N + a1] * sB[q2 * N + a2];
        double wq = sW[q1] * sW[q2];
        if (DIM == 3) { phi = phi * sB[q3 * N + a3]; wq = wq * sW[q3]; }
        acc = __fma_rn(wq * P.mq[(int64_t)e * NQ + q], phi * phi, acc);
      }
      const int s = P.slot[(int64_t)e * ND + a];
      for (int c = 0; c < DIM; ++c) P.evec[(int64_t)s * DIM + c] = acc;
    }
    return;
  }
  for (int i = tid; i < DIM * ND; i += NT) {
    const int c = i / ND, a = i % ND;
    X[i] = P.in[(int64_t)c * P.n_nodes + snode[a]];
  }
  __syncthreads();
  // interpolate to the points: contract a1, a2 (, a3) with B
  if (DIM == 3) {
    for (int o = tid; o < S1; o += NT) {  // U1[c][q1][a2][a3]
      const int a3 = o % N, a2 = (o / N) % N, q1 = (o / (N * N)) % Q, c = o / (N * N * Q);
      const double *x = X + c * ND + (a3 * N + a2) * N;
      double acc = sB[q1 * N] * x[0];
      for (int a1 = 1; a1 < N; ++a1) acc = __fma_rn(sB[q1 * N + a1], x[a1], acc);
      U1[o] = acc;
    }
    __syncthreads();
    for (int o = tid; o < S2; o += NT) {  // U2[c][q1][q2][a3]
      const int a3 = o % N, q2 = (o / N) % Q, q1 = (o / (N * Q)) % Q, c = o / (N * Q * Q);
      const double *u = U1 + ((c * Q + q1) * N) * N + a3;
      double acc = sB[q2 * N] * u[0];
      for (int a2 = 1; a2 < N; ++a2) acc = __fma_rn(sB[q2 * N + a2], u[a2 * N], acc);
      U2[o] = acc;
    }
    __syncthreads();
    for (int o = tid; o < DIM * NQ; o += NT) {  // V[c][q] with q = q1 + Q q2 + Q^2 q3
      const int q = o % NQ, c = o / NQ;
      const int q1 = q % Q, q2 = (q / Q) % Q, q3 = q / (Q * Q);
      const double *u = U2 + ((c * Q + q1) * Q + q2) * N;
      double acc = sB[q3 * N] * u[0];
      for (int a3 = 1; a3 < N; ++a3) acc = __fma_rn(sB[q3 * N + a3], u[a3], acc);
      const double wq = (sW[q1] * sW[q2]) * sW[q3];
      V[o] = acc * (wq * P.mq[(int64_t)e * NQ + q]);
    }
  } else {
    for (int o = tid; o < S1; o += NT) {  // U1[c][q1][a2]
      const int a2 = o % N, q1 = (o / N) % Q, c = o / (N * Q);
      const double *x = X + c * ND + a2 * N;
      double acc = sB[q1 * N] * x[0];
      for (int a1 = 1; a1 < N; ++a1) acc = __fma_rn(sB[q1 * N + a1], x[a1], acc);
      U1[o] = acc;
    }
    __syncthreads();
    for (int o = tid; o < DIM * NQ; o += NT) {
      const int q = o % NQ, c = o / NQ;
      const int q1 = q % Q, q2 = q / Q;
      const double *u = U1 + (c * Q + q1) * N;
      double acc = sB[q2 * N] * u[0];
      for (int a2 = 1; a2 < N; ++a2) acc = __fma_rn(sB[q2 * N + a2], u[a2], acc);
      V[o] = acc * ((sW[q1] * sW[q2]) * P.mq[(int64_t)e * NQ + q]);
    }
  }
  __syncthreads();
  // project back: Y[c][a] = sum_q phi_a(xi_q) V[c][q]  (transposed stages, reusing U1/U2)
  if (DIM == 3) {
    for (int o = tid; o < S2; o += NT) {  // P1[c][q1][q2][a3] = sum_q3 B[q3][a3] V
      const int a3 = o % N, q2 = (o / N) % Q, q1 = (o / (N * Q)) % Q, c = o / (N * Q * Q);
      double acc = 0.0;
      for (int q3 = 0; q3 < Q; ++q3) acc = __fma_rn(sB[q3 * N + a3], V[c * NQ + q1 + Q * q2 + Q * Q * q3], acc);
      U2[o] = acc;
    }
    __syncthreads();
    for (int o = tid; o < S1; o += NT) {  // P2[c][q1][a2][a3] = sum_q2 B[q2][a2] P1
      const int a3 = o % N, a2 = (o / N) % N, q1 = (o / (N * N)) % Q, c = o / (N * N * Q);
      double acc = 0.0;
      for (int q2 = 0; q2 < Q; ++q2) acc = __fma_rn(sB[q2 * N + a2], U2[((c * Q + q1) * Q + q2) * N + a3], acc);
      U1[o] = acc;
    }
    __syncthreads();
    for (int o = tid; o < DIM * ND; o += NT) {  // Y[c][a1,a2,a3] = sum_q1 B[q1][a1] P2
      const int a = o % ND, c = o / ND;
      const int a1 = a % N, a2 = (a / N) % N, a3 = a / (N * N);
      double acc = 0.0;
      for (int q1 = 0; q1 < Q; ++q1) acc = __fma_rn(sB[q1 * N + a1], U1[((c * Q + q1) * N + a2) * N + a3], acc);
      Y[o] = acc;
    }
  } else {
    for (int o = tid; o < S1; o += NT) {  // P1[c][q1][a2] = sum_q2 B[q2][a2] V
      const int a2 = o % N, q1 = (o / N) % Q, c = o / (N * Q);
      double acc = 0.0;
      for (int q2 = 0; q2 < Q; ++q2) acc = __fma_rn(sB[q2 * N + a2], V[c * NQ + q1 + Q * q2], acc);
      U1[o] = acc;
    }
    __syncthreads();
    for (int o = tid; o < DIM * ND; o += NT) {
      const int a = o % ND, c = o / ND;
      const int a1 = a % N, a2 = a / N;
      double acc = 0.0;
      for (int q1 = 0; q1 < Q; ++q1) acc = __fma_rn(sB[q1 * N + a1], U1[(c * Q + q1) * N + a2], acc);
      Y[o] = acc;
    }
  }
  __syncthreads();
  for (int o = tid; o < DIM * ND; o += NT) {
    const int a = o % ND, c = o / ND;
    const int s = P.slot[(int64_t)e * ND + a];
    P.evec[(int64_t)s * DIM + c] = Y[o];
  }
}

// M_V apply for 3D Q2/Q1 with 4^3 points (C2/C4 meshes), one thread per (element,
// component, q1): the lane's slice of the sum-factorised interpolation / projection lives in
// registers (tables are compile-time constant-bank operands), the final q1 contraction
// exchanges the four lanes' partial sums through shared memory (fixed order, deterministic).
// wm: precomputed w_q m_q [E][64].  evec: [slot][3].
__constant__ double c_mB24[4][3];  // Q2 GLL basis at the 4 GL points (filled at FOM setup)

#ifdef MASS3_MINB
#define MASS3_BOUNDS __launch_bounds__(256, MASS3_MINB)
#else
#define MASS3_BOUNDS __launch_bounds__(256)
#endif
__global__ void MASS3_BOUNDS mass_apply3_q2_kernel(int32_t n_elem, int64_t n_nodes,
                                                            const int32_t *__restrict__ elem_nodes,
                                                            const int32_t *__restrict__ slot,
                                                            const double *__restrict__ wm,
                                                            const double *__restrict__ in,
                                                            double *__restrict__ evec) {
  // CTA = 64 (element, component) groups of 4 lanes (q1); elements [e0, e0 + 22) overlap it
  __shared__ int sNode[23][27];
  __shared__ double sX[64][27];
  __shared__ double sP2[64][4][9];  // [group][q1][a2 + 3 a3]
  const int tid = threadIdx.x;
  const int q1 = tid & 3, grp = tid >> 2;
  const int ec0 = blockIdx.x * 64;
  const int e0 = ec0 / 3;
  const int ec = ec0 + grp;
  const bool valid = ec < n_elem * 3;
  const int e = valid ? ec / 3 : 0, c = valid ? ec % 3 : 0;
  const int le = e - e0;                       // element within the CTA window (0..22)
  // (1) node ids of the window's elements (coalesced rows)
  const int ne_win = min(23, n_elem - e0);
  for (int i = tid; i < ne_win * 27; i += 256) sNode[i / 27][i % 27] = __ldg(elem_nodes + (int64_t)e0 * 27 + i);
  __syncthreads();
  // (2) each lane gathers a quarter of its group's 27 dofs
  const double *src = in + (int64_t)c * n_nodes;
  if (valid)
    for (int a = q1; a < 27; a += 4) sX[grp][a] = __ldg(src + sNode[le][a]);
  __syncthreads();
  const double *X = sX[grp];
  // stage 1: U1[a2][a3] = sum_a1 B[q1][a1] X[a1, a2, a3]
  double b0, b1, b2;
  if (q1 == 0) { b0 = c_mB24[0][0]; b1 = c_mB24[0][1]; b2 = c_mB24[0][2]; }
  else if (q1 == 1) { b0 = c_mB24[1][0]; b1 = c_mB24[1][1]; b2 = c_mB24[1][2]; }
  else if (q1 == 2) { b0 = c_mB24[2][0]; b1 = c_mB24[2][1]; b2 = c_mB24[2][2]; }
  else { b0 = c_mB24[3][0]; b1 = c_mB24[3][1]; b2 = c_mB24[3][2]; }
  double U1[9];
#pragma unroll
  for (int r = 0; r < 9; ++r) U1[r] = __fma_rn(b2, X[3 * r + 2], __fma_rn(b1, X[3 * r + 1], b0 * X[3 * r]));
  // stage 2: U2[q2][a3] = sum_a2 B[q2][a2] U1[a2][a3]
  double U2[4][3];
#pragma unroll
  for (int q2 = 0; q2 < 4; ++q2)
#pragma unroll
    for (int a3 = 0; a3 < 3; ++a3)
      U2[q2][a3] = __fma_rn(c_mB24[q2][2], U1[2 + 3 * a3],
                            __fma_rn(c_mB24[q2][1], U1[1 + 3 * a3], c_mB24[q2][0] * U1[3 * a3]));
  // stage 3 + weights + first projection: P1[q2][a3] = sum_q3 B[q3][a3] wm V
  const double *w = wm + (int64_t)e * 64 + q1;
  double P1[4][3];
#pragma unroll
  for (int q2 = 0; q2 < 4; ++q2) {
    P1[q2][0] = P1[q2][1] = P1[q2][2] = 0.0;
#pragma unroll
    for (int q3 = 0; q3 < 4; ++q3) {
      double vq = __fma_rn(c_mB24[q3][2], U2[q2][2],
                           __fma_rn(c_mB24[q3][1], U2[q2][1], c_mB24[q3][0] * U2[q2][0]));
      vq = vq * __ldg(w + 4 * q2 + 16 * q3);
#pragma unroll
      for (int a3 = 0; a3 < 3; ++a3) P1[q2][a3] = __fma_rn(c_mB24[q3][a3], vq, P1[q2][a3]);
    }
  }
  // P2[a2][a3] = sum_q2 B[q2][a2] P1[q2][a3]  -> shared, per lane q1
#pragma unroll
  for (int a2 = 0; a2 < 3; ++a2)
#pragma unroll
    for (int a3 = 0; a3 < 3; ++a3) {
      double acc = 0.0;
#pragma unroll
      for (int q2 = 0; q2 < 4; ++q2) acc = __fma_rn(c_mB24[q2][a2], P1[q2][a3], acc);
      sP2[grp][q1][a2 + 3 * a3] = acc;
    }
  __syncwarp();
  // Y[a1, a2, a3] = sum_q1 B[q1][a1] P2[q1][a2][a3]: lane q1 writes nodes a = q1, q1+4, ...
  if (valid) {
    const int32_t *sl = slot + (int64_t)e * 27;
    for (int a = q1; a < 27; a += 4) {
      const int a1 = a % 3, r = a / 3;
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < 4; ++k) acc = __fma_rn(c_mB24[k][a1], sP2[grp][k][r], acc);
      evec[(int64_t)__ldg(sl + a) * 3 + c] = acc;
    }
  }
}

__global__ void wm_setup_kernel(int64_t n, int Q, int dim, const double *__restrict__ tab_w,
                                const double *__restrict__ mq, double *__restrict__ wm) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int nq = dim == 3 ? Q * Q * Q : Q * Q;
  if (t >= n * nq) return;
  const int q = (int)(t % nq);
  const int q1 = q % Q, q2 = (q / Q) % Q, q3 = q / (Q * Q);
  double w = tab_w[q1] * tab_w[q2];
  if (dim == 3) w = w * tab_w[q3];
  wm[t] = w * mq[t];
}

// y[c][node] = mask * sum over the node's slots (ascending) -- deterministic assembly
template <int DIM>
__global__ void assemble_masked_kernel(int64_t n_nodes, const int32_t *__restrict__ off,
                                       const double *__restrict__ evec,
                                       const double *__restrict__ mask, double *__restrict__ y,
                                       int invert) {
  const int64_t node = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (node >= n_nodes) return;
  const int s0 = off[node], s1 = off[node + 1];
#pragma unroll
  for (int c = 0; c < DIM; ++c) {
    double acc = 0.0;
    for (int s = s0; s < s1; ++s) acc += evec[(int64_t)s * DIM + c];
    const int64_t i = (int64_t)c * n_nodes + node;
    const double m = mask ? mask[i] : 1.0;
    y[i] = invert ? (m != 0.0 ? 1.0 / acc : 0.0) : m * acc;
  }
}

// M_E,K (kept in Mblk for hydro_mass_e_apply), its inverse (Gauss-Jordan on the SPD block, no pivoting needed) and its row sums
// (c_K[j] = 1^T M_E,K e_j, the internal-energy weights).  One thread per element.
template <int DIM, int K, int Q>
__global__ void mass_e_setup_kernel(int32_t n_elem, const double *__restrict__ mq,
                                    const double *__restrict__ tab_w,
                                    const double *__restrict__ tab_Bl, double *__restrict__ Minv,
                                    double *__restrict__ csum, double *__restrict__ Mblk) {
  constexpr int M = K, NE = DIM == 3 ? M * M * M : M * M, NQ = DIM == 3 ? Q * Q * Q : Q * Q;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_elem) return;
  double A[NE][2 * NE];
  for (int i = 0; i < NE; ++i)
    for (int j = 0; j < 2 * NE; ++j) A[i][j] = (j - NE == i) ? 1.0 : 0.0;
  for (int q = 0; q < NQ; ++q) {
    const int q1 = q % Q, q2 = (q / Q) % Q, q3 = q / (Q * Q);
    double wq = tab_w[q1] * tab_w[q2];
    if (DIM == 3) wq = wq * tab_w[q3];
    const double wm = wq * mq[(int64_t)e * NQ + q];
    double psi[NE];
    for (int i = 0; i < NE; ++i) {
      const int i1 = i % M, i2 = (i / M) % M, i3 = i / (M * M);
      double p = tab_Bl[q1 * M + i1] * tab_Bl[q2 * M + i2];
      if (DIM == 3) p = p * tab_Bl[q3 * M + i3];
      psi[i] = p;
    }
    for (int i = 0; i < NE; ++i)
      for (int j = 0; j < NE; ++j) A[i][j] = __fma_rn(wm * psi[i], psi[j], A[i][j]);
  }
  for (int i = 0; i < NE; ++i) {
    double s = 0.0;
    for (int j = 0; j < NE; ++j) s += A[i][j];
    csum[(int64_t)e * NE + i] = s;
    if (Mblk)
      for (int j = 0; j < NE; ++j) Mblk[((int64_t)e * NE + i) * NE + j] = A[i][j];
  }
  for (int p = 0; p < NE; ++p) {
    const double inv = 1.0 / A[p][p];
    for (int j = 0; j < 2 * NE; ++j) A[p][j] *= inv;
    for (int i = 0; i < NE; ++i) {
      if (i == p) continue;
      const double f = A[i][p];
      if (f != 0.0)
        for (int j = 0; j < 2 * NE; ++j) A[i][j] = __fma_rn(-f, A[p][j], A[i][j]);
    }
  }
  for (int i = 0; i < NE; ++i)
    for (int j = 0; j < NE; ++j) Minv[((int64_t)e * NE + i) * NE + j] = A[i][NE + j];
}

// out_K = a_K + s * Minv_K rhs_K    (element-local energy update; one thread per dof)
template <int NE>
__global__ void mass_e_update_kernel(int32_t n_elem, const double *__restrict__ Minv,
                                     const double *__restrict__ a, const double *__restrict__ rhs,
                                     double s, double *__restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)n_elem * NE) return;
  const int64_t e = t / NE;
  const int i = (int)(t % NE);
  const double *m = Minv + (e * NE + i) * NE;
  const double *r = rhs + e * NE;
  double acc = 0.0;
#pragma unroll
  for (int j = 0; j < NE; ++j) acc = __fma_rn(m[j], r[j], acc);
  out[t] = a[t] + s * acc;
}

// ---- deterministic dot product: fixed grid, fixed-order block trees, one final block
constexpr int DOT_BLOCKS = 148 * 8, DOT_THREADS = 256;

__global__ void __launch_bounds__(DOT_THREADS) dot_partial_kernel(int64_t n, const double *__restrict__ a,
                                                                  const double *__restrict__ b,
                                                                  double *__restrict__ part) {
  __shared__ double sh[DOT_THREADS];
  const int64_t chunk = (n + DOT_BLOCKS - 1) / DOT_BLOCKS;
  const int64_t lo = (int64_t)blockIdx.x * chunk;
  const int64_t hi = lo + chunk < n ? lo + chunk : n;
  double acc = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += DOT_THREADS) acc = __fma_rn(a[i], b[i], acc);
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int w = DOT_THREADS / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}



// Block-partial of a dot product inside another kernel's grid: each block writes the
// fixed-order tree sum of its threads' values to part[blockIdx.x] (grid = DOT_BLOCKS
// blocks of DOT_THREADS threads, each covering one contiguous chunk: deterministic).
__device__ __forceinline__ void block_partial(double v, double *part) {
  __shared__ double sh[DOT_THREADS];
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int w = DOT_THREADS / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

// Ap = mask * assemble(evec) and part = block partials of p . Ap  (fused)
// 8 CTAs per SM (32 registers, a few spilled words): all DOT_BLOCKS CTAs resident in one wave
#ifndef ASM_DOT_MINB
#define ASM_DOT_MINB 8
#endif
template <int DIM>
__global__ void __launch_bounds__(DOT_THREADS, ASM_DOT_MINB) assemble_dot_kernel(
    int64_t n_nodes, const int32_t *__restrict__ off, const double *__restrict__ evec,
    const double *__restrict__ mask, const double *__restrict__ p, double *__restrict__ Ap,
    double *__restrict__ part) {
  const int64_t chunk = (n_nodes + DOT_BLOCKS - 1) / DOT_BLOCKS;
  const int64_t lo = (int64_t)blockIdx.x * chunk;
  const int64_t hi = lo + chunk < n_nodes ? lo + chunk : n_nodes;
  double acc = 0.0;
  for (int64_t node = lo + threadIdx.x; node < hi; node += DOT_THREADS) {
    const int s0 = off[node], s1 = off[node + 1];
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
      double y = 0.0;
      for (int s = s0; s < s1; ++s) y += evec[(int64_t)s * DIM + c];
      const int64_t i = (int64_t)c * n_nodes + node;
      y = mask[i] * y;
      Ap[i] = y;
      acc = __fma_rn(p[i], y, acc);
    }
  }
  block_partial(acc, part);
}

// Fixed-order sum of the DOT_BLOCKS partials by one 256-thread block: thread t adds
// partials t, t+256, ... in order, then a fixed tree (deterministic, ~2 us instead of a
// serial loop's ~40 us).
__device__ __forceinline__ double sum_partials(const double *__restrict__ part) {
  __shared__ double sh[256];
  double acc = 0.0;
  for (int i = threadIdx.x; i < DOT_BLOCKS; i += 256) acc += part[i];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  return sh[0];
}

__global__ void __launch_bounds__(256) dot_final_kernel(const double *__restrict__ part,
                                                        double *__restrict__ out) {
  const double s_ = sum_partials(part);
  if (threadIdx.x == 0) *out = s_;
}

// The two per-iteration vector passes of PCG with the dot finalisations folded in (4 launches
// per iteration instead of 6): every CTA sums the DOT_BLOCKS partials of the preceding kernel
// itself, in sum_partials' fixed order, so all CTAs hold the same bits as the former one-block
// finalisation kernels.  The partials a kernel reads (pin) and writes (pout) are different
// arrays, and r.z lives in two slots of sc used alternately (rz_in is read by every CTA,
// rz_out written by CTA 0), so no CTA reads what another writes.
// x += alpha p; r -= alpha Ap; z = Dinv r; pout = block partials of r.z;  alpha = rz / p.Ap
// (8 CTAs per SM: all DOT_BLOCKS = 148 x 8 CTAs resident in one wave -- at 40 registers only 6 fit and the
// last 296 CTAs ran as a third-full second wave)
#ifndef CG_XR_MINB
#define CG_XR_MINB 8
#endif
__global__ void __launch_bounds__(DOT_THREADS, CG_XR_MINB) cg_xr_dot_fused_kernel(
    int64_t n, double *__restrict__ sc, int rz_in, const double *__restrict__ pin,
    const double *__restrict__ p, const double *__restrict__ Ap, const double *__restrict__ dinv,
    double *__restrict__ x, double *__restrict__ r, double *__restrict__ z, double *__restrict__ pout) {
  const double pAp = sum_partials(pin);
  const double rz = sc[rz_in];
  // a zero residual (rz = 0) or a vanishing p.Ap would give 0/0: the iterate is final
  const double al = (rz == 0.0 || pAp == 0.0) ? 0.0 : rz / pAp;
  if (blockIdx.x == 0 && threadIdx.x == 0) { sc[1] = pAp; sc[2] = al; }
  const int64_t chunk = (n + DOT_BLOCKS - 1) / DOT_BLOCKS;
  const int64_t lo = (int64_t)blockIdx.x * chunk;
  const int64_t hi = lo + chunk < n ? lo + chunk : n;
  double acc = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += DOT_THREADS) {
    x[i] = __fma_rn(al, p[i], x[i]);
    const double ri = __fma_rn(-al, Ap[i], r[i]);
    r[i] = ri;
    const double zi = dinv[i] * ri;
    z[i] = zi;
    acc = __fma_rn(ri, zi, acc);
  }
  block_partial(acc, pout);
}
// p = z + beta p;  beta = rz_new / rz with rz_new the sum of pin; sc[rz_out] = rz_new
__global__ void __launch_bounds__(DOT_THREADS) cg_p_fused_kernel(
    int64_t n, double *__restrict__ sc, int rz_in, int rz_out, const double *__restrict__ pin,
    const double *__restrict__ z, double *__restrict__ p) {
  const double rzn = sum_partials(pin);
  const double rz = sc[rz_in];
  const double be = rz == 0.0 ? 0.0 : rzn / rz;
  if (blockIdx.x == 0 && threadIdx.x == 0) { sc[3] = rzn; sc[4] = be; sc[rz_out] = rzn; }
  const int64_t chunk = (n + DOT_BLOCKS - 1) / DOT_BLOCKS;
  const int64_t lo = (int64_t)blockIdx.x * chunk;
  const int64_t hi = lo + chunk < n ? lo + chunk : n;
  for (int64_t i = lo + threadIdx.x; i < hi; i += DOT_THREADS) p[i] = __fma_rn(be, p[i], z[i]);
}

// ---- PCG (Jacobi) pieces.  sc: [0] / [8] rz (alternating), [1] pAp, [2] alpha, [3] rz_new,
// [4] beta, [5] rz0
__global__ void cg_init_kernel(int64_t n, const double *__restrict__ b, const double *__restrict__ mask,
                               const double *__restrict__ dinv, double *__restrict__ x,
                               double *__restrict__ r, double *__restrict__ z, double *__restrict__ p) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double ri = mask[i] * b[i];
  x[i] = 0.0;
  r[i] = ri;
  const double zi = dinv[i] * ri;
  z[i] = zi;
  p[i] = zi;
}
// warm start: r = mask b - Ap (Ap = mask M x0, r = mask b on entry), z = D^-1 r, p = z
__global__ void cg_residual_kernel(int64_t n, const double *__restrict__ Ap,
                                   const double *__restrict__ dinv, double *__restrict__ r,
                                   double *__restrict__ z, double *__restrict__ p) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double ri = r[i] - Ap[i];
  r[i] = ri;
  const double zi = dinv[i] * ri;
  z[i] = zi;
  p[i] = zi;
}
// out = mask * (a + s * b)   (masked: the v.n = 0 components stay exactly 0 when a has 0 there)
__global__ void axpy_kernel(int64_t n, const double *__restrict__ a, double s,
                            const double *__restrict__ b, const double *__restrict__ mask,
                            double *__restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double v = a[i] + s * b[i];
  out[i] = mask ? mask[i] * v : v;
}

// vbar = (a + b) / 2
__global__ void avg_kernel(int64_t n, const double *__restrict__ a, const double *__restrict__ b,
                           double *__restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = 0.5 * (a[i] + b[i]);
}

// ---- hyper-reduced ROM step vector ops on [n][B] arrays (instance fastest), per-instance dt
// out[i][b] = a[i][b] + s * dt[b] * r[i][b]
__global__ void rom_axpy_kernel(int64_t n, int B, const double *__restrict__ a, double s,
                                const double *__restrict__ dt, const double *__restrict__ r,
                                double *__restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * B) return;
  const int b = (int)(t % B);
  out[t] = a[t] + (s * dt[b]) * r[t];
}

// Per-instance accept/restore of the step controller: Y[:, b] = keep[b] ? Y : Ybak (layout [n][B])
__global__ void rom_select_kernel(int64_t n, int B, const double *__restrict__ keep,
                                  const double *__restrict__ bak, double *__restrict__ Y) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * B) return;
  if (keep[t % B] == 0.0) Y[t] = bak[t];
}

__global__ void min2_kernel(int B, const double *__restrict__ a, const double *__restrict__ b,
                            double *__restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < B) {
    const double x = a[i], y = b[i];
    out[i] = (x != x || y != y) ? __longlong_as_double(0x7ff8000000000000ll) : fmin(x, y);  // NaN in either propagates
  }
}

}  // namespace hk
