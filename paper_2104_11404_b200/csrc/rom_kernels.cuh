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

// ---------------------------------------------------------------------------- FP64 MMA
// D (8x8) = A (8x4, row) B (4x8, col) + C on the FP64 tensor pipe (mma.sync m8n8k4 f64, the
// DMMA path: 256 FMAs per warp instruction at the same 37 TF/s as DFMA, measured
// profiles/r01_fp64_dmma_rate.txt).  Fragments (lane l): A[l>>2][l&3], B[l&3][l>>2],
// C/D[l>>2][2(l&3) + {0,1}].  Not volatile: the scheduler may move loads across it.
__device__ __forceinline__ void dmma_m8n8k4(double &d0, double &d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------- cp.async
__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gmem_src, bool pred) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  const int sz = pred ? 16 : 0;   // src-size 0: zero-fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(gmem_src), "r"(sz));
}
__device__ __forceinline__ void cp_async8(void *smem_dst, const void *gmem_src, bool pred) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  const int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(gmem_src), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

// lift on the tensor pipe: out[r][c] = os + sum_k Phi[r][k] Y[k][c] for n <= 4 NKS, B <= 64
// per column block (grid.y).  Persistent CTAs of 8 warps over 128-row tiles (16 rows = two
// m-tiles per warp); Y's column block is staged once per CTA in shared memory in fragment
// order (conflict-free LDS.64); each warp preloads its 2 x NKS A fragments (Phi rows, 32 B
// per row per k-step: full sectors) and issues 16 DMMAs per k-step from 32 accumulators.
// WM m-tiles (8 rows each) per warp, MINB CTAs per SM: (2, 2) for shared offsets (x, v: the
// tensor pipe binds, 2 m-tiles reuse each B fragment), (1, 4) for per-instance offsets (e: the
// offset read makes it HBM-bound; 4 CTAs per SM keep more bytes in flight) -- measured
// (profiles/ab/r02_ab13_lift_warp_tile.txt).
constexpr int LIFT_MMA_THREADS = 256;
template <int NKS, int WM, int MINB>
__global__ void __launch_bounds__(LIFT_MMA_THREADS, MINB)
lift_mma_kernel(int64_t rows, int n, int B, const double *__restrict__ Phi,
                const double *__restrict__ os, int os_batched, const double *__restrict__ Y,
                double *__restrict__ out) {
  constexpr int LIFT_MMA_RT = 8 * 8 * WM;
  __shared__ double sY[NKS * 8 * 32];   // [kstep][ntile][lane]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c0 = blockIdx.y * 64;
  for (int i = threadIdx.x; i < NKS * 8 * 32; i += LIFT_MMA_THREADS) {
    const int l = i & 31, nt = (i >> 5) & 7, ks = i >> 8;
    const int k = ks * 4 + (l & 3), c = c0 + nt * 8 + (l >> 2);
    sY[i] = (k < n && c < B) ? Y[(int64_t)k * B + c] : 0.0;
  }
  __syncthreads();
  const int64_t ntiles = (rows + LIFT_MMA_RT - 1) / LIFT_MMA_RT;
  const int ar = lane >> 2, ak = lane & 3;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t rw = t * LIFT_MMA_RT + warp * 8 * WM;   // this warp's first row
    double a[WM][NKS];
#pragma unroll
    for (int mt = 0; mt < WM; ++mt) {
      const int64_t r = rw + mt * 8 + ar;
#pragma unroll
      for (int ks = 0; ks < NKS; ++ks) {
        const int k = ks * 4 + ak;
        a[mt][ks] = (r < rows && k < n) ? __ldg(Phi + r * n + k) : 0.0;
      }
    }
    double acc[WM][8][2];
#pragma unroll
    for (int mt = 0; mt < WM; ++mt)
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < NKS; ++ks) {
      double b[8];
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) b[nt] = sY[(ks * 8 + nt) * 32 + lane];
#pragma unroll
      for (int mt = 0; mt < WM; ++mt)
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) dmma_m8n8k4(acc[mt][nt][0], acc[mt][nt][1], a[mt][ks], b[nt]);
    }
#pragma unroll
    for (int mt = 0; mt < WM; ++mt) {
      const int64_t r = rw + mt * 8 + ar;
      if (r >= rows) continue;
      const double o1 = os_batched ? 0.0 : __ldg(os + r);
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        const int c = c0 + nt * 8 + 2 * ak;
        if (c + 1 < B) {
          double2 o;
          if (os_batched) {
            o = __ldg(reinterpret_cast<const double2 *>(os + r * B + c));
          } else {
            o.x = o1;
            o.y = o1;
          }
          double2 v;
          v.x = o.x + acc[mt][nt][0];
          v.y = o.y + acc[mt][nt][1];
          *reinterpret_cast<double2 *>(out + r * B + c) = v;
        } else if (c < B) {
          out[r * B + c] = (os_batched ? __ldg(os + r * B + c) : o1) + acc[mt][nt][0];
        }
      }
    }
  }
}

// projection on the tensor pipe, split-K: CTA g reduces a fixed contiguous range of s into
// a partial [n][B] (n <= 8 MT, B <= 64).  Within the CTA, warp w = 2 kg + nh takes every 4th
// k-step of the range (k-group kg, fixed) for the column half nh (4 n-tiles) and all MT m-tiles
// (40 accumulators for MT = 5); the four k-group partials of each half are summed in a fixed
// tree through shared memory; project_mma_reduce sums the CTA partials in ascending g (fixed
// order, parallel over 8 sub-ranges per output).  Deterministic.
constexpr int PROJ_MMA_THREADS = 256;
// AT: A is stored transposed, A(m, k) = P[k * lda + m] (basis products Phi^T X with Phi
// [s][lda] row-major); otherwise A(m, k) = P[m * lda + k] (the projector [n][s], lda = s).
// B(k, c) = f[k * ldf + c].
template <int MT, bool AT = false>
__global__ void __launch_bounds__(PROJ_MMA_THREADS, 2)
project_mma_kernel(int n, int64_t s_rows, int B, int64_t chunk, const double *__restrict__ P,
                   int64_t lda, const double *__restrict__ f, int64_t ldf, double *__restrict__ part) {
  extern __shared__ __align__(16) double sred[];   // [4 slots][MT*4 tiles][2][32]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nh = warp & 1, kg = warp >> 1;
  const int64_t s_begin = (int64_t)blockIdx.x * chunk;
  const int64_t s_end = s_begin + chunk < s_rows ? s_begin + chunk : s_rows;
  const int ar = lane >> 2, ak = lane & 3;
  double acc[MT][4][2];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
  const bool fullB = B == 64;
#pragma unroll 2
  for (int64_t k0 = s_begin + kg * 4; k0 < s_end; k0 += 16) {
    const int64_t k = k0 + ak;   // A: P(m, k) (m = 8 mt + (l >> 2)); B: f[k][c] (c = 8 nt + (l >> 2))
    const bool kin = k < s_end;
    double a[MT], b[4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int m = mt * 8 + ar;
      a[mt] = (kin && m < n) ? __ldg(P + (AT ? k * lda + m : (int64_t)m * lda + k)) : 0.0;
    }
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int c = (nh * 4 + nt) * 8 + ar;
      b[nt] = (kin && (fullB || c < B)) ? __ldg(f + k * ldf + c) : 0.0;
    }
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) dmma_m8n8k4(acc[mt][nt][0], acc[mt][nt][1], a[mt], b[nt]);
  }
  // fixed tree over the k-groups of each column half: (kg, kg + 2), then (0, 1)
  constexpr int TS = MT * 4 * 2 * 32;
#pragma unroll
  for (int half = 2; half >= 1; half >>= 1) {
    if (kg >= half && kg < 2 * half) {
      double *dst = sred + ((kg - half) * 2 + nh) * TS;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          dst[((mt * 4 + nt) * 2 + 0) * 32 + lane] = acc[mt][nt][0];
          dst[((mt * 4 + nt) * 2 + 1) * 32 + lane] = acc[mt][nt][1];
        }
    }
    __syncthreads();
    if (kg < half) {
      const double *src = sred + (kg * 2 + nh) * TS;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          acc[mt][nt][0] += src[((mt * 4 + nt) * 2 + 0) * 32 + lane];
          acc[mt][nt][1] += src[((mt * 4 + nt) * 2 + 1) * 32 + lane];
        }
    }
    __syncthreads();
  }
  if (kg == 0) {
    double *pg = part + (int64_t)blockIdx.x * n * B;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int m = mt * 8 + ar;
      if (m >= n) continue;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int c = (nh * 4 + nt) * 8 + 2 * ak;
        if (c < B) pg[m * B + c] = acc[mt][nt][0];
        if (c + 1 < B) pg[m * B + c + 1] = acc[mt][nt][1];
      }
    }
  }
}

// Projection v3 (r02): a streaming split-K GEMM.  CTA g reduces a fixed contiguous range of s in
// chunks of PK rows; each chunk of P ([n][PK], 8 PK bytes per row) and f ([PK][64]) is copied into a
// PS-stage shared-memory ring with cp.async (16-byte copies, no registers held while in flight),
// and warp w computes the column tile w (8 columns) for all MT m-tiles from shared memory (4 MMAs
// of k 4 per m-tile and chunk; 2 MT accumulators).  The CTA partial is written per warp (no
// cross-warp reduction); project_mma_reduce sums the CTA partials in ascending g.  Requires
// n <= 8 MT, B <= 64 and even, P and f 16-byte aligned.  Deterministic.
#ifndef PROJ3_PK_
#define PROJ3_PK_ 32
#endif
#ifndef PROJ3_PS_
#define PROJ3_PS_ 3
#endif
// column tiles (8 columns each) per warp: 1 -- warp w takes column tile w over every k-step;
// 2 -- warp w takes the column pair w % 4 over the k-steps of parity w / 4, so each A fragment
// loaded from shared memory feeds two MMAs (0.7 instead of 1.2 shared loads per MMA); the two
// k-parity partials are summed in a fixed order (even + odd) before the CTA partial is written.
#ifndef PROJ3_NTW_
#define PROJ3_NTW_ 2
#endif
// resident CTAs per SM (the split-K group count is 148 x this): the ring holds PS stages of
// (8 MT (PK + 4) + 72 PK) doubles per CTA
#ifndef PROJ3_MINB_
#define PROJ3_MINB_ 2
#endif
constexpr int PROJ3_MINB = PROJ3_MINB_;
constexpr int PROJ3_PK = PROJ3_PK_, PROJ3_PS = PROJ3_PS_, PROJ3_SPS = PROJ3_PK + 4, PROJ3_SFS = 72,
              PROJ3_NTW = PROJ3_NTW_;
static_assert(PROJ3_NTW == 1 || PROJ3_NTW == 2, "PROJ3_NTW");
// P8: s_rows odd -- the rows of P are only 8-byte aligned, so P is copied in 8-byte pieces.
template <int MT, bool P8 = false>
__global__ void __launch_bounds__(256, PROJ3_MINB)
project_mma3_kernel(int n, int64_t s_rows, int B, int64_t chunk, const double *__restrict__ P,
                    const double *__restrict__ f, double *__restrict__ part) {
  extern __shared__ __align__(16) double sm3[];
  constexpr int PK = PROJ3_PK, PS = PROJ3_PS, SPS = PROJ3_SPS, SFS = PROJ3_SFS;
  constexpr int PSZ = MT * 8 * SPS;
  constexpr int STAGE = PSZ + PK * SFS;                   // doubles per stage
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ar = lane >> 2, ak = lane & 3;
  const int64_t s_begin = (int64_t)blockIdx.x * chunk;
  const int64_t s_end = s_begin + chunk < s_rows ? s_begin + chunk : s_rows;
  const int nchunks = (int)((s_end - s_begin + PK - 1) / PK);
  auto issue = [&](int ci) {
    double *sP = sm3 + (ci % PS) * STAGE;
    double *sF = sP + PSZ;
    const int64_t k0 = s_begin + (int64_t)ci * PK;
    if (P8) {
      for (int i = tid; i < MT * 8 * PK; i += 256) {        // MT*8 rows of P, PK doubles each
        const int m = i / PK, j = i % PK;
        const bool ok = m < n && k0 + j < s_end;
        cp_async8(sP + m * SPS + j, ok ? P + (int64_t)m * s_rows + k0 + j : P, ok);
      }
    } else {
      for (int i = tid; i < MT * 8 * (PK / 2); i += 256) {
        const int m = i / (PK / 2), j = (i % (PK / 2)) * 2;
        const bool ok = m < n && k0 + j < s_end;   // s_rows even and k0 even: pairs never straddle
        cp_async16(sP + m * SPS + j, ok ? P + (int64_t)m * s_rows + k0 + j : P, ok);
      }
    }
    // f: 16 rows x B doubles (B/2 copies per row)
    const int bh = (B + 1) / 2;
    for (int i = tid; i < PK * bh; i += 256) {
      const int r = i / bh, c = (i % bh) * 2;
      const bool row = k0 + r < s_end;
      if (c + 1 < B) {
        cp_async16(sF + r * SFS + c, row ? f + (k0 + r) * B + c : f, row);
      } else {   // odd B: the last column by a plain store (its pair is zero)
        sF[r * SFS + c] = row ? f[(k0 + r) * B + c] : 0.0;
        sF[r * SFS + c + 1] = 0.0;
      }
    }
  };
  constexpr int NTW = PROJ3_NTW;
  double acc[MT][NTW][2];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int t = 0; t < NTW; ++t) acc[mt][t][0] = acc[mt][t][1] = 0.0;
  // column base and first k-step of this warp
  const int cb = NTW == 1 ? warp * 8 : (warp & 3) * 16;
  const int kg = NTW == 1 ? 0 : warp >> 2;
#pragma unroll
  for (int ci = 0; ci < PS - 1; ++ci) {
    if (ci < nchunks) issue(ci);
    cp_async_commit();
  }
  for (int ci = 0; ci < nchunks; ++ci) {
    if (ci + PS - 1 < nchunks) issue(ci + PS - 1);
    cp_async_commit();
    cp_async_wait<PS - 1>();
    __syncthreads();
    const double *sP = sm3 + (ci % PS) * STAGE;
    const double *sF = sP + PSZ;
#pragma unroll
    for (int k2 = 0; k2 < PK / 4 / NTW; ++k2) {
      const int kk = k2 * NTW + kg;
      double b[NTW];
#pragma unroll
      for (int t = 0; t < NTW; ++t) b[t] = sF[(kk * 4 + ak) * SFS + cb + t * 8 + ar];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int m = mt * 8 + ar;
        const double a = sP[m * SPS + kk * 4 + ak];
#pragma unroll
        for (int t = 0; t < NTW; ++t) dmma_m8n8k4(acc[mt][t][0], acc[mt][t][1], a, b[t]);
      }
    }
    __syncthreads();
  }
  if (NTW == 2) {  // odd-parity warps hand their partial to the even ones (the ring is free)
    double *xs = sm3 + ((warp & 3) * 32 + lane) * (MT * 4);
    if (kg == 1) {
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          xs[(mt * 2 + t) * 2 + 0] = acc[mt][t][0];
          xs[(mt * 2 + t) * 2 + 1] = acc[mt][t][1];
        }
    }
    __syncthreads();
    if (kg == 1) return;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        acc[mt][t][0] = acc[mt][t][0] + xs[(mt * 2 + t) * 2 + 0];
        acc[mt][t][1] = acc[mt][t][1] + xs[(mt * 2 + t) * 2 + 1];
      }
  }
  double *pg = part + (int64_t)blockIdx.x * n * B;
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int t = 0; t < NTW; ++t) {
      const int m = mt * 8 + ar, c = cb + t * 8 + 2 * ak;
      if (m < n) {
        if (c < B) pg[m * B + c] = acc[mt][t][0];
        if (c + 1 < B) pg[m * B + c + 1] = acc[mt][t][1];
      }
    }
}

// r[o] = sum_g part[g][o] in ascending g: 8 threads per output sum fixed contiguous g-ranges,
// combined in ascending range order through shared memory.
constexpr int PROJ_RED_OUT = 32;
__global__ void __launch_bounds__(256) project_mma_reduce_kernel(int nB, int G, const double *__restrict__ part,
                                                                 double *__restrict__ r) {
  __shared__ double ssum[8][PROJ_RED_OUT];
  const int o = blockIdx.x * PROJ_RED_OUT + (threadIdx.x & 31);
  const int j = threadIdx.x >> 5;
  const int per = (G + 7) / 8;
  const int g0 = j * per, g1 = min(G, g0 + per);
  double acc = 0.0;
  if (o < nB)
    for (int g = g0; g < g1; ++g) acc += __ldg(part + (int64_t)g * nB + o);
  ssum[j][threadIdx.x & 31] = acc;
  __syncthreads();
  if (j == 0 && o < nB) {
    double t = ssum[0][threadIdx.x];
#pragma unroll
    for (int i = 1; i < 8; ++i) t += ssum[i][threadIdx.x];
    r[o] = t;
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
