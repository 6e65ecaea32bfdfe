// offline.cuh -- the ROM offline phase on the GPU (PAPER Sec. 4.3-4.5,
// P:908-1051): the snapshot Gram matrix for POD by the method of snapshots, the basis
// formation Phi = S^T V Sigma^-1, and the greedy DEIM index selection (Algorithm 1 of
// Chaturantabut-Sorensen, as described at P:1003-1016).  All reductions are fixed-order
// (split over fixed row chunks, then a fixed-order sum), so results are run-to-run
// deterministic.  The small dense pieces (the ns x ns eigenproblem, the j x j DEIM solves)
// run on the host in hydro_api.cu.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "rom_kernels.cuh"  // dmma_m8n8k4, project_mma_reduce_kernel

namespace hk {

constexpr int GRAM_T = 16;        // output tile (GRAM_T x GRAM_T per block)
constexpr int GRAM_KT = 64;       // rows staged per smem tile
constexpr int GRAM_CHUNKS = 148 * 2;

// partial[c][i][j] = sum over k in chunk c of A(i, k) A(j, k), A(i, k) = A[i * si + k * sk]
// (snapshots S [ns][N]: si = N, sk = 1; the columns of a row-major basis Phi [N][ldp]:
// si = 1, sk = ldp), for the upper-triangle tile (blockIdx.y, blockIdx.z), tile_i <= tile_j.
// The smem loader walks the unit-stride index fastest so the loads coalesce either way.
__global__ void __launch_bounds__(GRAM_T *GRAM_T) gram_partial_kernel(
    int ns, int64_t N, int64_t chunk, int64_t si_, int64_t sk_, const double *__restrict__ S,
    double *__restrict__ partial) {
  const int ti = blockIdx.y, tj = blockIdx.z;
  if (ti > tj) return;
  __shared__ double si[GRAM_T][GRAM_KT + 1], sj[GRAM_T][GRAM_KT + 1];
  const int tx = threadIdx.x % GRAM_T, ty = threadIdx.x / GRAM_T;
  const int i = ti * GRAM_T + ty, j = tj * GRAM_T + tx;
  const int64_t k0 = (int64_t)blockIdx.x * chunk;
  const int64_t k1 = k0 + chunk < N ? k0 + chunk : N;
  const bool kfast = sk_ == 1;
  double acc = 0.0;
  for (int64_t kb = k0; kb < k1; kb += GRAM_KT) {
    for (int t = threadIdx.x; t < GRAM_T * GRAM_KT; t += GRAM_T * GRAM_T) {
      const int r = kfast ? t / GRAM_KT : t % GRAM_T;
      const int kk = kfast ? t % GRAM_KT : t / GRAM_T;
      const int64_t k = kb + kk;
      const int ri = ti * GRAM_T + r, rj = tj * GRAM_T + r;
      si[r][kk] = (ri < ns && k < k1) ? S[ri * si_ + k * sk_] : 0.0;
      sj[r][kk] = (rj < ns && k < k1) ? S[rj * si_ + k * sk_] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < GRAM_KT; ++kk) acc = __fma_rn(si[ty][kk], sj[tx][kk], acc);
    __syncthreads();
  }
  if (i < ns && j < ns) partial[((int64_t)blockIdx.x * ns + i) * ns + j] = acc;
}

// G[i][j] = G[j][i] = sum over chunks (ascending) of partial[c][min][max]
__global__ void gram_reduce_kernel(int ns, int chunks, const double *__restrict__ partial,
                                   double *__restrict__ G) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ns * ns) return;
  int i = t / ns, j = t % ns;
  if (i > j) { const int x = i; i = j; j = x; }
  double acc = 0.0;
  for (int c = 0; c < chunks; ++c) acc += partial[((int64_t)c * ns + i) * ns + j];
  G[t] = acc;
}

// Phi[r][c] = sum_j S[j][r] W[j][c]  (S: [ns][N], W: [ns][k], Phi: [N][ldp], c < k); one
// thread per row r, output columns in groups of 8 registers.
__global__ void snapshot_combine_kernel(int ns, int64_t N, int k, int ldp, const double *__restrict__ S,
                                        const double *__restrict__ W, double *__restrict__ Phi) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= N) return;
  for (int c0 = 0; c0 < k; c0 += 8) {
    double acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.0;
    for (int j = 0; j < ns; ++j) {
      const double sv = S[(int64_t)j * N + r];
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (c0 + q < k) acc[q] = __fma_rn(sv, W[j * k + c0 + q], acc[q]);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (c0 + q < k) Phi[r * ldp + c0 + q] = acc[q];
  }
}

constexpr int POD_MAXK = 128;

// Phi[r][:k] <- Phi[r][:k] R^{-1} (Rinv: [k][k] upper triangular), one thread per row, the
// row held in a per-thread array (k <= POD_MAXK).
__global__ void right_mult_kernel(int64_t N, int k, int ldp, const double *__restrict__ Rinv,
                                  double *__restrict__ Phi) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= N) return;
  double t[POD_MAXK];
  double *row = Phi + r * ldp;
  for (int j = 0; j < k; ++j) t[j] = row[j];
  for (int c = 0; c < k; ++c) {
    double acc = 0.0;
    for (int j = 0; j <= c; ++j) acc = __fma_rn(t[j], Rinv[j * k + c], acc);
    row[c] = acc;
  }
}

// P[i][j] = sum_{k >= i} Rinv[i][k] Q[j][k]  (P = R^-1 Q^T: [m][s]; Q [s][m] row-major, Rinv
// [m][m] upper triangular), one thread per column j of P -- consecutive threads write
// consecutive entries of every row of P (hydro_gappy_pinv).
__global__ void pinv_apply_kernel(int64_t s, int m, const double *__restrict__ Rinv,
                                  const double *__restrict__ Q, double *__restrict__ P) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= s) return;
  double q[POD_MAXK];
  for (int k = 0; k < m; ++k) q[k] = Q[j * m + k];
  for (int i = 0; i < m; ++i) {
    double acc = 0.0;
    for (int k = i; k < m; ++k) acc = __fma_rn(Rinv[i * m + k], q[k], acc);
    P[(int64_t)i * s + j] = acc;
  }
}

// DEIM residual of basis column j: res[r] = U[r][j] - sum_{i<j} U[r][i] c[i]  (U: [N][m]),
// with per-block argmax of |res| (ties: lowest row) written to (bval, bidx).
constexpr int DEIM_BLOCKS = 148 * 4, DEIM_THREADS = 256;
// mask (optional): rows with mask[r] != 0 are skipped (the oversampled greedy's chosen set).
__global__ void __launch_bounds__(DEIM_THREADS) deim_residual_kernel(
    int64_t N, int m, int j, const double *__restrict__ U, const double *__restrict__ c,
    double *__restrict__ bval, int64_t *__restrict__ bidx,
    const unsigned char *__restrict__ mask = nullptr, double *__restrict__ absr = nullptr) {
  __shared__ double sv[DEIM_THREADS];
  __shared__ int64_t si[DEIM_THREADS];
  const int64_t chunk = (N + DEIM_BLOCKS - 1) / DEIM_BLOCKS;
  const int64_t lo = (int64_t)blockIdx.x * chunk;
  const int64_t hi = lo + chunk < N ? lo + chunk : N;
  double best = -1.0;
  int64_t bi = -1;
  for (int64_t r = lo + threadIdx.x; r < hi; r += DEIM_THREADS) {
    if (mask && mask[r]) continue;
    const double *row = U + r * m;
    double acc = 0.0;
    for (int i = 0; i < j; ++i) acc = __fma_rn(row[i], c[i], acc);
    const double v = fabs(row[j] - acc);
    if (absr) absr[r] = v;   // kept for the oversampled greedy's further picks of column j
    if (v > best) { best = v; bi = r; }   // ascending r per thread: first maximum kept
  }
  sv[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int w = DEIM_THREADS / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      const double a = sv[threadIdx.x], b = sv[threadIdx.x + w];
      const int64_t ia = si[threadIdx.x], ib = si[threadIdx.x + w];
      if (b > a || (b == a && ib >= 0 && (ia < 0 || ib < ia))) { sv[threadIdx.x] = b; si[threadIdx.x] = ib; }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) { bval[blockIdx.x] = sv[0]; bidx[blockIdx.x] = si[0]; }
}

// Q-DEIM (QR with column pivoting of U^T = pivoted Gram-Schmidt on the rows of U), one
// step on the residual Rt held column-major ([m][N], so every access below is coalesced
// across rows): every residual row r loses its component along the unit vector q (the last
// pivot's normalised residual), R[r] -= (R[r].q) q, and its squared norm nu[r] is recomputed
// from the updated entries; the block-wise arg-max of nu (ties: the lowest row) is written
// for the next pivot.  Rows already chosen keep a zero residual and are never picked again.
__global__ void __launch_bounds__(DEIM_THREADS) qdeim_step_kernel(
    int64_t N, int m, const double *__restrict__ q, double *__restrict__ Rt,
    double *__restrict__ bval, int64_t *__restrict__ bidx, int first) {
  __shared__ double sv[DEIM_THREADS];
  __shared__ int64_t si[DEIM_THREADS];
  const int64_t chunk = (N + DEIM_BLOCKS - 1) / DEIM_BLOCKS;
  const int64_t lo = (int64_t)blockIdx.x * chunk;
  const int64_t hi = lo + chunk < N ? lo + chunk : N;
  double best = -1.0;
  int64_t bi = -1;
  for (int64_t r = lo + threadIdx.x; r < hi; r += DEIM_THREADS) {
    double n2 = 0.0;
    if (first) {
      for (int j = 0; j < m; ++j) {
        const double v = Rt[(int64_t)j * N + r];
        n2 = __fma_rn(v, v, n2);
      }
    } else {
      double c = 0.0;
      for (int j = 0; j < m; ++j) c = __fma_rn(Rt[(int64_t)j * N + r], q[j], c);
      for (int j = 0; j < m; ++j) {
        const double v = __fma_rn(-c, q[j], Rt[(int64_t)j * N + r]);
        Rt[(int64_t)j * N + r] = v;
        n2 = __fma_rn(v, v, n2);
      }
    }
    if (n2 > best) { best = n2; bi = r; }
  }
  sv[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int w = DEIM_THREADS / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      const double a = sv[threadIdx.x], b = sv[threadIdx.x + w];
      const int64_t ia = si[threadIdx.x], ib = si[threadIdx.x + w];
      if (b > a || (b == a && ib >= 0 && (ia < 0 || ib < ia))) { sv[threadIdx.x] = b; si[threadIdx.x] = ib; }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) { bval[blockIdx.x] = sv[0]; bidx[blockIdx.x] = si[0]; }
}

// [N][m] row-major -> [m][N], 32x32 tiles through shared memory; a 1D grid of
// ceil(N/32) * ceil(m/32) tiles (row tile fastest), so either extent may be large.
__global__ void transpose_kernel(int64_t N, int64_t m, const double *__restrict__ A,
                                 double *__restrict__ At) {
  __shared__ double t[32][33];
  const int64_t tiles_r = (N + 31) / 32;
  const int64_t r0 = ((int64_t)blockIdx.x % tiles_r) * 32;
  const int64_t j0 = ((int64_t)blockIdx.x / tiles_r) * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int64_t r = r0 + i;
    const int64_t j = j0 + threadIdx.x;
    if (r < N && j < m) t[i][threadIdx.x] = A[r * m + j];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int64_t j = j0 + i;
    const int64_t r = r0 + threadIdx.x;
    if (r < N && j < m) At[j * N + r] = t[threadIdx.x][i];
  }
}

// Cross products G = A^T X over N rows (A: [N][lda] first na columns, X: [N][ldx] first nx
// columns), split-K over row chunks like the Gram kernel: one GRAM_T x GRAM_T output tile per
// block (y, z) and row chunk (x), staged through shared memory; partial[chunk][na][nx].
__global__ void __launch_bounds__(GRAM_T *GRAM_T) xprod_partial_kernel(
    int na, int nx, int64_t N, int64_t chunk, const double *__restrict__ A, int64_t lda,
    const double *__restrict__ X, int64_t ldx, double *__restrict__ partial) {
  __shared__ double sa[GRAM_KT][GRAM_T + 1], sx[GRAM_KT][GRAM_T + 1];
  const int tx = threadIdx.x % GRAM_T, ty = threadIdx.x / GRAM_T;
  const int i = blockIdx.y * GRAM_T + ty, j = blockIdx.z * GRAM_T + tx;
  const int64_t k0 = (int64_t)blockIdx.x * chunk;
  const int64_t k1 = k0 + chunk < N ? k0 + chunk : N;
  double acc = 0.0;
  for (int64_t kb = k0; kb < k1; kb += GRAM_KT) {
    for (int t = threadIdx.x; t < GRAM_T * GRAM_KT; t += GRAM_T * GRAM_T) {
      const int c = t % GRAM_T, kk = t / GRAM_T;   // consecutive threads: consecutive columns
      const int64_t k = kb + kk;
      const int ca = blockIdx.y * GRAM_T + c, cx = blockIdx.z * GRAM_T + c;
      sa[kk][c] = (ca < na && k < k1) ? A[k * lda + ca] : 0.0;
      sx[kk][c] = (cx < nx && k < k1) ? X[k * ldx + cx] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < GRAM_KT; ++kk) acc = __fma_rn(sa[kk][ty], sx[kk][tx], acc);
    __syncthreads();
  }
  if (i < na && j < nx) partial[((int64_t)blockIdx.x * na + i) * nx + j] = acc;
}

// G[i][j] = sum over chunks (ascending) of partial[c][i][j]
__global__ void xprod_reduce_kernel(int na, int nx, int chunks, const double *__restrict__ partial,
                                    double *__restrict__ G) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= na * nx) return;
  double acc = 0.0;
  for (int c = 0; c < chunks; ++c) acc += partial[(int64_t)c * na * nx + t];
  G[t] = acc;
}

// d = a - b (elementwise; the offset difference of a window transition)
__global__ void sub_kernel(int64_t n, const double *__restrict__ a, const double *__restrict__ b,
                           double *__restrict__ d) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) d[i] = a[i] - b[i];
}

// out[r] = (f ? f[r] : 0) - sgn * sum_j A[r][j] y[j]   (A: [N][lda], first n columns)
__global__ void gemv_kernel(int64_t N, int n, const double *__restrict__ A, int64_t lda,
                            const double *__restrict__ y, const double *__restrict__ f, double sgn,
                            double *__restrict__ out) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= N) return;
  const double *a = A + r * lda;
  double acc = 0.0;
  for (int j = 0; j < n; ++j) acc = __fma_rn(a[j], y[j], acc);
  out[r] = (f ? f[r] : 0.0) - sgn * acc;
}

// out[i][j] = A[idx[i]][j]  (i < s, j < n; A: [N][lda])
__global__ void gather_rows_kernel(int s, int n, const int64_t *__restrict__ idx,
                                   const double *__restrict__ A, int64_t lda, double *__restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= s * n) return;
  const int i = t / n, j = t % n;
  out[t] = A[idx[i] * lda + j];
}

// dst[c * ld_dst + di] (+)= src[c * ld_src + si] for i < n, c < dim, with si = src_idx[i] (or
// i) and di = dst_idx[i] (or i) -- the gather / fixed-order accumulate / scatter of the
// sharded force's halo sum.  Indices within one call are distinct (no write conflicts).
__global__ void index_copy_add_kernel(int64_t n, int dim, const double *__restrict__ src, int64_t ld_src,
                                      const int64_t *__restrict__ src_idx, double *__restrict__ dst,
                                      int64_t ld_dst, const int64_t *__restrict__ dst_idx, int add) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * dim) return;
  const int c = (int)(t / n);
  const int64_t i = t % n;
  const int64_t si = src_idx ? src_idx[i] : i, di = dst_idx ? dst_idx[i] : i;
  const double v = src[c * ld_src + si];
  double *d = dst + c * ld_dst + di;
  *d = add ? *d + v : v;
}

// ------------------------------------------------------------------ FP64 tensor-pipe GEMMs
// Gram matrices of the offline phase on the tensor pipe (DMMA m8n8k4): partial[c][i][j] =
// sum over k in chunk c of A(i, k) A(j, k), A(i, k) = KFAST ? A[i * ld + k] (snapshots S [ns][N])
// : A[k * ld + i] (the columns of a row-major basis Phi [N][ld]).  CTA (c, ti, tj) computes the
// 64 x 64 output tile (ti, tj) over row chunk c in k-blocks of 32: every warp stages the eight
// 8 x 4 fragments of one k-step into shared memory in fragment order (lane = row * 4 + k: each
// lane's global load is one double of a fully used 32-byte sector; the fragment reads are
// conflict-free LDS.64), the next k-block is loaded into registers while the current one is
// multiplied; warp w owns m-tiles 2 (w & 3) .. + 1 and n-tiles 4 (w >> 2) .. + 3 (8 DMMAs per
// k-step).  A B fragment (k x n8) of the Gram is the A fragment of n-tile nt, so a diagonal
// tile stages one operand.  Partials are summed by project_mma_reduce_kernel in ascending
// chunk order: deterministic.
constexpr int GMMA_T = 64;     // output tile
constexpr int GMMA_KB = 32;    // k-block (8 k-steps of 4)
template <bool KFAST>
__global__ void __launch_bounds__(256, 2)
gram_mma_kernel(int n, int64_t N, int64_t chunk, int64_t ld, const double *__restrict__ A,
                double *__restrict__ partial) {
  __shared__ double sF[2][8 * 8 * 32];   // [operand][k-step][8-row tile][lane]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ti = blockIdx.y, tj = blockIdx.z;
  const bool same = ti == tj;
  const int64_t k0 = (int64_t)blockIdx.x * chunk;
  const int64_t k1 = k0 + chunk < N ? k0 + chunk : N;
  const int fr = lane >> 2, fk = lane & 3;
  double ra[8], rb[8];
  // warp w stages k-step w of a k-block: fragment (ks = w, tile q) = rows q*8 + fr, k = 4w + fk
  auto load = [&](int64_t kb) {
    const int64_t k = kb + warp * 4 + fk;
    const bool kin = k < k1;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int i = ti * GMMA_T + q * 8 + fr, j = tj * GMMA_T + q * 8 + fr;
      ra[q] = (kin && i < n) ? __ldg(KFAST ? A + (int64_t)i * ld + k : A + k * ld + i) : 0.0;
      if (!same) rb[q] = (kin && j < n) ? __ldg(KFAST ? A + (int64_t)j * ld + k : A + k * ld + j) : 0.0;
    }
  };
  double acc[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int mt0 = (warp & 3) * 2, nt0 = (warp >> 2) * 4;
  if (k0 < k1) load(k0);
  for (int64_t kb = k0; kb < k1; kb += GMMA_KB) {
    __syncthreads();   // the previous k-block's fragment reads are done
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      sF[0][(warp * 8 + q) * 32 + lane] = ra[q];
      if (!same) sF[1][(warp * 8 + q) * 32 + lane] = rb[q];
    }
    __syncthreads();
    if (kb + GMMA_KB < k1) load(kb + GMMA_KB);
    const double *fa = sF[0], *fb = same ? sF[0] : sF[1];
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const double a0 = fa[(ks * 8 + mt0) * 32 + lane], a1 = fa[(ks * 8 + mt0 + 1) * 32 + lane];
      double b[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) b[t] = fb[(ks * 8 + nt0 + t) * 32 + lane];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        dmma_m8n8k4(acc[0][t][0], acc[0][t][1], a0, b[t]);
        dmma_m8n8k4(acc[1][t][0], acc[1][t][1], a1, b[t]);
      }
    }
  }
  double *out = partial + (int64_t)blockIdx.x * n * n;
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const int i = ti * GMMA_T + (mt0 + a) * 8 + fr;
    if (i >= n) continue;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int j = tj * GMMA_T + (nt0 + t) * 8 + 2 * fk;
      if (j < n) out[(int64_t)i * n + j] = acc[a][t][0];
      if (j + 1 < n) out[(int64_t)i * n + j + 1] = acc[a][t][1];
    }
  }
}

// out[r][c] = sum_k A(r, k) Y[k][c] for c < B <= 64, k < K <= 4 NKS, A(r, k) = AT ? A[k * lda + r]
// (Phi = S^T W from the snapshots S [ns][N]) : A[r * lda + k] (Phi <- Phi R^-1); out row stride
// ldo.  The lift kernel's scheme (lift_mma_kernel): persistent CTAs of 8 warps over 128-row
// tiles, Y staged once per CTA in fragment order, each warp 2 m-tiles x 8 n-tiles.  A warp
// reads all of its rows' A fragments before it writes any of its outputs and no other warp
// touches those rows, so with !AT the call may be in place (out == A, ldo == lda): A and out
// are deliberately not __restrict__.
template <bool AT, int NKS>
__global__ void __launch_bounds__(256, 2)
tall_mma_kernel(int64_t rows, int K, int B, const double *A, int64_t lda,
                const double *__restrict__ Y, double *out, int64_t ldo) {
  __shared__ double sY[NKS * 8 * 32];   // [kstep][ntile][lane]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < NKS * 8 * 32; i += 256) {
    const int l = i & 31, nt = (i >> 5) & 7, ks = i >> 8;
    const int k = ks * 4 + (l & 3), c = nt * 8 + (l >> 2);
    sY[i] = (k < K && c < B) ? Y[(int64_t)k * B + c] : 0.0;
  }
  __syncthreads();
  const int64_t ntiles = (rows + 127) / 128;
  const int ar = lane >> 2, ak = lane & 3;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t rw = t * 128 + warp * 16;
    double a[2][NKS];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int64_t r = rw + mt * 8 + ar;
#pragma unroll
      for (int ks = 0; ks < NKS; ++ks) {
        const int k = ks * 4 + ak;
        a[mt][ks] = (r < rows && k < K) ? __ldg(AT ? A + (int64_t)k * lda + r : A + r * lda + k) : 0.0;
      }
    }
    double acc[2][8][2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < NKS; ++ks) {
      double b[8];
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) b[nt] = sY[(ks * 8 + nt) * 32 + lane];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 8; ++nt) dmma_m8n8k4(acc[mt][nt][0], acc[mt][nt][1], a[mt][ks], b[nt]);
    }
    __syncwarp();
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int64_t r = rw + mt * 8 + ar;
      if (r >= rows) continue;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        const int c = nt * 8 + 2 * ak;
        if (c < B) out[r * ldo + c] = acc[mt][nt][0];
        if (c + 1 < B) out[r * ldo + c + 1] = acc[mt][nt][1];
      }
    }
  }
}

// Q-DEIM by column-norm downdating (the pivoted QR of U^T the way LAPACK's geqp3 tracks its
// column norms): nu[r] = |u_r|^2 - sum_{l<k} (q_l . u_r)^2 is the squared norm of row r's
// residual after k pivots (q_l: the orthonormalised pivot residuals), so a step reads each row
// once (Ut column-major [m][N], coalesced) and updates nu in place -- no residual matrix is
// rewritten.  Where the downdate cancels (nu <= sqrt(eps) nu0, nu0 the original norm) the
// row's residual norm is recomputed from u_r against all k+1 directions Q [k+1][m] (MGS order,
// as geqp3 recomputes).  Chosen rows carry nu = -1 and are never picked again.  step == 0:
// nu = nu0 = |u_r|^2.  Block-wise arg-max of nu (ties: the lowest row) into (bval, bidx).
// |u_r - sum_{l<k} q_l (q_l . res)|^2 by modified Gram-Schmidt against Q [k][m] (m <= 64);
// out of line so that its 64-entry row does not raise the register count of the main loop
__device__ __noinline__ double qdeim_recompute(const double *__restrict__ Ut, int64_t N, int m, int64_t r,
                                               const double *__restrict__ Q, int k) {
  double u[64];
  for (int j = 0; j < m; ++j) u[j] = Ut[(int64_t)j * N + r];
  for (int l = 0; l < k; ++l) {
    const double *ql = Q + (int64_t)l * m;
    double d = 0.0;
    for (int j = 0; j < m; ++j) d = __fma_rn(u[j], ql[j], d);
    for (int j = 0; j < m; ++j) u[j] = __fma_rn(-d, ql[j], u[j]);
  }
  double n2 = 0.0;
  for (int j = 0; j < m; ++j) n2 = __fma_rn(u[j], u[j], n2);
  return n2;
}

template <int M>
__global__ void __launch_bounds__(DEIM_THREADS) qdeim_dd_kernel(
    int64_t N, int m, int step, const double *__restrict__ Q, const double *__restrict__ Ut,
    double *__restrict__ nu, double *__restrict__ nu0, double *__restrict__ bval,
    int64_t *__restrict__ bidx) {
  __shared__ double sv[DEIM_THREADS];
  __shared__ int64_t si[DEIM_THREADS];
  __shared__ double sq[M];
  const double *qk = Q + (int64_t)(step > 0 ? step - 1 : 0) * m;   // the newest direction
  for (int j = threadIdx.x; j < M; j += DEIM_THREADS) sq[j] = (step > 0 && j < m) ? qk[j] : 0.0;
  __syncthreads();
  const int64_t chunk = (N + DEIM_BLOCKS - 1) / DEIM_BLOCKS;
  const int64_t lo = (int64_t)blockIdx.x * chunk;
  const int64_t hi = lo + chunk < N ? lo + chunk : N;
  const double tol = 1.4901161193847656e-08;   // sqrt(DBL_EPSILON)
  double best = -1.0;
  int64_t bi = -1;
  for (int64_t r = lo + threadIdx.x; r < hi; r += DEIM_THREADS) {
    double n2;
    if (step == 0) {
      n2 = 0.0;
#pragma unroll 8
      for (int j = 0; j < m; ++j) {
        const double v = Ut[(int64_t)j * N + r];
        n2 = __fma_rn(v, v, n2);
      }
      nu0[r] = n2;
    } else {
      n2 = nu[r];
      if (n2 < 0.0) continue;   // chosen
      double c = 0.0;
#pragma unroll 8
      for (int j = 0; j < m; ++j) c = __fma_rn(Ut[(int64_t)j * N + r], sq[j], c);
      n2 = n2 - c * c;
      const double n0 = nu0[r];
      if (!(n2 > tol * n0)) n2 = n0 > 0.0 ? qdeim_recompute(Ut, N, m, r, Q, step) : 0.0;   // cancellation
    }
    nu[r] = n2;
    if (n2 > best) { best = n2; bi = r; }   // ascending r per thread: first maximum kept
  }
  sv[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int w = DEIM_THREADS / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      const double a = sv[threadIdx.x], b = sv[threadIdx.x + w];
      const int64_t ia = si[threadIdx.x], ib = si[threadIdx.x + w];
      if (b > a || (b == a && ib >= 0 && (ia < 0 || ib < ia))) { sv[threadIdx.x] = b; si[threadIdx.x] = ib; }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) { bval[blockIdx.x] = sv[0]; bidx[blockIdx.x] = si[0]; }
}

__global__ void mark_chosen_kernel(double *nu, int64_t p) { nu[p] = -1.0; }

// block-wise arg-max of stored |res| over the rows outside the mask (ties: the lowest row)
__global__ void __launch_bounds__(DEIM_THREADS) argmax_masked_kernel(
    int64_t N, const double *__restrict__ absr, const unsigned char *__restrict__ mask,
    double *__restrict__ bval, int64_t *__restrict__ bidx) {
  __shared__ double sv[DEIM_THREADS];
  __shared__ int64_t si[DEIM_THREADS];
  const int64_t chunk = (N + DEIM_BLOCKS - 1) / DEIM_BLOCKS;
  const int64_t lo = (int64_t)blockIdx.x * chunk;
  const int64_t hi = lo + chunk < N ? lo + chunk : N;
  double best = -1.0;
  int64_t bi = -1;
  for (int64_t r = lo + threadIdx.x; r < hi; r += DEIM_THREADS) {
    if (mask[r]) continue;
    const double v = absr[r];
    if (v > best) { best = v; bi = r; }
  }
  sv[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int w = DEIM_THREADS / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      const double a = sv[threadIdx.x], b = sv[threadIdx.x + w];
      const int64_t ia = si[threadIdx.x], ib = si[threadIdx.x + w];
      if (b > a || (b == a && ib >= 0 && (ia < 0 || ib < ia))) { sv[threadIdx.x] = b; si[threadIdx.x] = ib; }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) { bval[blockIdx.x] = sv[0]; bidx[blockIdx.x] = si[0]; }
}

}  // namespace hk
