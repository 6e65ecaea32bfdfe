// rom_kernels.cuh -- FP64 GEMM-shaped kernels of the hyper-reduced ROM online step.
//
// lift:    out[r][b] = os[r] (or os[r][b]) + sum_k Phi[r][k] Y[k][b]
//          (PAPER Eq. discretesolrepresentation, on sample-mesh rows only,
//          P:893-894).  Tall-skinny: rows ~ 3.5e6, n = 40, B = 64 -> bound by the Phi
//          read + out write (~6 flop/B, near the FP64 ridge).  64-row x 64-col CTA tile,
//          Phi tile and Y staged in shared memory, 4x4 register tile per thread.
// project: r[i][b] = sum_s P[i][s] f[s][b]  (Eq. sol-ls-hyper P:778-799 with the
//          precomputed (Z^T Phi)^dagger).  Short-wide: n = 40, s ~ 4e5 -> deterministic
//          split-K: CTA g reduces a fixed contiguous s-range into a partial [n][B] tile,
//          a second kernel sums the partials in ascending g.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace hk {

constexpr int LIFT_RT = 64;      // rows per CTA
constexpr int LIFT_CB = 64;      // columns per CTA
constexpr int LIFT_THREADS = 256;

// dynamic smem: (n * LIFT_CB + LIFT_RT * (n + 1)) doubles
__global__ void __launch_bounds__(LIFT_THREADS)
lift_kernel(int64_t rows, int n, int B, const double *__restrict__ Phi,
            const double *__restrict__ os, int os_batched, const double *__restrict__ Y,
            double *__restrict__ out) {
  extern __shared__ __align__(16) double sm[];
  double *sY = sm;                       // [n][LIFT_CB]
  double *sP = sm + n * LIFT_CB;         // [LIFT_RT][n+1] (padded)
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int64_t r0 = (int64_t)blockIdx.x * LIFT_RT;
  const int c0 = blockIdx.y * LIFT_CB;
  for (int i = tid; i < n * LIFT_CB; i += LIFT_THREADS) {
    const int k = i / LIFT_CB, cb = i % LIFT_CB;
    sY[i] = (c0 + cb < B) ? Y[(int64_t)k * B + c0 + cb] : 0.0;
  }
  for (int i = tid; i < LIFT_RT * n; i += LIFT_THREADS) {
    const int rr = i / n, k = i % n;
    const int64_t r = r0 + rr;
    sP[rr * (n + 1) + k] = r < rows ? Phi[r * n + k] : 0.0;
  }
  __syncthreads();
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (int k = 0; k < n; ++k) {
    double pv[4], yv[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) pv[i] = sP[(ty * 4 + i) * (n + 1) + k];
#pragma unroll
    for (int j = 0; j < 4; ++j) yv[j] = sY[k * LIFT_CB + tx + 16 * j];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = __fma_rn(pv[i], yv[j], acc[i][j]);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = r0 + ty * 4 + i;
    if (r >= rows) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int b = c0 + tx + 16 * j;
      if (b >= B) continue;
      const double o = os_batched ? os[r * B + b] : os[r];
      out[r * B + b] = o + acc[i][j];
    }
  }
}

constexpr int PROJ_THREADS = 256;
constexpr int PROJ_TS = 32;      // s-rows per shared tile
constexpr int PROJ_MAXN = 64;
constexpr int PROJ_MAXB = 64;

// Partial r over s in [s_begin(g), s_end(g)). Thread owns column b = tid % B and rows
// i = tid / B + (256 / B) * j.  Requires n <= 64, B <= 64.
__global__ void __launch_bounds__(PROJ_THREADS)
project_partial_kernel(int n, int64_t s_rows, int B, int64_t chunk, const double *__restrict__ P,
                       const double *__restrict__ f, double *__restrict__ part) {
  __shared__ double sP[PROJ_MAXN][PROJ_TS + 1];
  __shared__ double sF[PROJ_TS][PROJ_MAXB];
  const int tid = threadIdx.x;
  const int64_t s_begin = (int64_t)blockIdx.x * chunk;
  const int64_t s_end = s_begin + chunk < s_rows ? s_begin + chunk : s_rows;
  const int b = tid % B;
  const int rstep = PROJ_THREADS / B;
  const int i0 = tid / B;
  const bool has_col = tid < rstep * B;
  double acc[PROJ_MAXN / 4];  // rows i0 + rstep*j, j < ceil(n / rstep); rstep >= 4
#pragma unroll
  for (int j = 0; j < PROJ_MAXN / 4; ++j) acc[j] = 0.0;
  for (int64_t s0 = s_begin; s0 < s_end; s0 += PROJ_TS) {
    const int ts = (int)((s_end - s0) < PROJ_TS ? (s_end - s0) : PROJ_TS);
    __syncthreads();
    for (int i = tid; i < n * PROJ_TS; i += PROJ_THREADS) {
      const int row = i / PROJ_TS, ss = i % PROJ_TS;
      sP[row][ss] = ss < ts ? P[(int64_t)row * s_rows + s0 + ss] : 0.0;
    }
    for (int i = tid; i < PROJ_TS * B; i += PROJ_THREADS) {
      const int ss = i / B, bb = i % B;
      sF[ss][bb] = ss < ts ? f[(s0 + ss) * B + bb] : 0.0;
    }
    __syncthreads();
    if (has_col) {
      for (int ss = 0; ss < ts; ++ss) {
        const double fv = sF[ss][b];
#pragma unroll
        for (int j = 0; j < PROJ_MAXN / 4; ++j) {
          const int i = i0 + rstep * j;
          if (i < n) acc[j] = __fma_rn(sP[i][ss], fv, acc[j]);
        }
      }
    }
  }
  if (has_col) {
#pragma unroll
    for (int j = 0; j < PROJ_MAXN / 4; ++j) {
      const int i = i0 + rstep * j;
      if (i < n) part[((int64_t)blockIdx.x * n + i) * B + b] = acc[j];
    }
  }
}

__global__ void project_reduce_kernel(int n, int B, int G, const double *__restrict__ part,
                                      double *__restrict__ r) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * B) return;
  double acc = 0.0;
  for (int g = 0; g < G; ++g) acc += part[(int64_t)g * n * B + t];
  r[t] = acc;
}

}  // namespace hk
