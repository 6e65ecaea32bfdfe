// DMMA (mma.sync m8n8k4 f64) throughput on this part, alone and mixed with DFMA, and whether
// a DMMA with C = 0 equals the sequential FMA chain fma(a3,b3,fma(a2,b2,fma(a1,b1,a0*b0)))
// bit for bit.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 dmma_rate.cu -o dmma_rate
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
               : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

template <int MODE>  // 0: DMMA only, 1: DFMA only, 2: both
__global__ void rate(int iters, double *out, double seed) {
  double a = seed + threadIdx.x * 1e-3, b = seed * 0.5, acc[8], f[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { acc[i] = 0.0; f[i] = seed + i; }
  for (int it = 0; it < iters; ++it) {
    if (MODE != 1) {
#pragma unroll
      for (int i = 0; i < 8; i += 2) dmma(acc[i], acc[i + 1], a, b, acc[i], acc[i + 1]);
    }
    if (MODE != 0) {
#pragma unroll
      for (int i = 0; i < 8; ++i) f[i] = __fma_rn(f[i], 0.999999, 1e-7);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i] + f[i];
  if (s == 12345.678) out[0] = s;
}

// exactness: lane layout of m8n8k4 (row.col): A fragment: lane l holds A[l/4][l%4]; B: lane l
// holds B[l%4][l/4]; C/D: lane l holds D[l/4][2*(l%4)], D[l/4][2*(l%4)+1]
__global__ void exact(const double *A, const double *B, double *D, double *Dref) {
  const int l = threadIdx.x;
  double a = A[(l / 4) * 4 + l % 4], b = B[(l % 4) * 8 + l / 4], d0, d1;
  dmma(d0, d1, a, b, 0.0, 0.0);
  D[(l / 4) * 8 + 2 * (l % 4)] = d0;
  D[(l / 4) * 8 + 2 * (l % 4) + 1] = d1;
  if (l < 8) {
    for (int j = 0; j < 8; ++j) {
      double acc = A[l * 4 + 0] * B[0 * 8 + j];
      for (int k = 1; k < 4; ++k) acc = __fma_rn(A[l * 4 + k], B[k * 8 + j], acc);
      Dref[l * 8 + j] = acc;
    }
  }
}

int main() {
  double *out;
  cudaMalloc(&out, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000, blocks = sms * 8, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char *names[3] = {"DMMA only", "DFMA only", "DMMA+DFMA"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) rate<0><<<blocks, threads>>>(iters, out, 1.0);
      if (mode == 1) rate<1><<<blocks, threads>>>(iters, out, 1.0);
      if (mode == 2) rate<2><<<blocks, threads>>>(iters, out, 1.0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double warps = (double)blocks * threads / 32;
      const double dmma_flop = (mode != 1) ? warps * iters * 4 * (8.0 * 8 * 4 * 2) : 0;  // 4 mma/iter
      const double dfma_flop = (mode != 0) ? (double)blocks * threads * iters * 8 * 2 : 0;
      if (rep) printf("%-10s %8.3f ms  DMMA %6.2f TF  DFMA %6.2f TF  total %6.2f TF\n", names[mode], ms,
                      dmma_flop / ms / 1e9, dfma_flop / ms / 1e9, (dmma_flop + dfma_flop) / ms / 1e9);
    }
  }
  // exactness on random operands
  const int trials = 2000;
  double hA[32], hB[32], hD[64], hR[64];
  double *dA, *dB, *dD, *dR;
  cudaMalloc(&dA, 256); cudaMalloc(&dB, 256); cudaMalloc(&dD, 512); cudaMalloc(&dR, 512);
  uint64_t st = 88172645463325252ull;
  auto rnd = [&]() { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return (double)(st >> 11) / 9007199254740992.0 * 2 - 1; };
  long mismatch = 0, total = 0;
  for (int t = 0; t < trials; ++t) {
    for (int i = 0; i < 32; ++i) { hA[i] = rnd() * (1 + (t % 7) * 1e3); hB[i] = rnd(); }
    cudaMemcpy(dA, hA, 256, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice);
    exact<<<1, 32>>>(dA, dB, dD, dR);
    cudaMemcpy(hD, dD, 512, cudaMemcpyDeviceToHost);
    cudaMemcpy(hR, dR, 512, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 64; ++i) { total++; if (hD[i] != hR[i]) mismatch++; }
  }
  printf("DMMA vs sequential FMA chain (C = 0): %ld / %ld entries differ\n", mismatch, total);
  return 0;
}
