// FP64-pipe rate of the contract's Jacobi pair (lmin3_pair, fast arithmetic) in isolation:
// every thread solves `reps` pairs of seeded symmetric 3x3 matrices shaped like C2's
// (J^T J near h^2 I with +-5% shape noise; eps random), no memory traffic.  Reports the
// executed-rotation count and algorithmic FP64 instructions per second (48 per rotation +
// setup) against the measured DFMA peak, for several occupancies.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2104_11404_b200/csrc/force_kernel.cuh"

__device__ unsigned long long g_rot;

__device__ __forceinline__ double u01(unsigned long long &s) {
  s += 0x9E3779B97F4A7C15ull;
  unsigned long long z = s;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (double)(z >> 11) * 0x1p-53;
}

template <int MINB>
__global__ void __launch_bounds__(64, MINB) jk(int reps, double *out) {
  unsigned long long s = 0x2104ull * (blockIdx.x * 64 + threadIdx.x + 1);
  double acc = 0.0;
  unsigned long long rot = 0;
  for (int r = 0; r < reps; ++r) {
    const double h = 0.01875;
    double J[3][3];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) J[i][j] = (i == j ? h : 0.0) + 0.05 * h * (2 * u01(s) - 1);
    const double c00 = (J[0][0] * J[0][0] + J[1][0] * J[1][0]) + J[2][0] * J[2][0];
    const double c11 = (J[0][1] * J[0][1] + J[1][1] * J[1][1]) + J[2][1] * J[2][1];
    const double c22 = (J[0][2] * J[0][2] + J[1][2] * J[1][2]) + J[2][2] * J[2][2];
    const double c01 = (J[0][0] * J[0][1] + J[1][0] * J[1][1]) + J[2][0] * J[2][1];
    const double c02 = (J[0][0] * J[0][2] + J[1][0] * J[1][2]) + J[2][0] * J[2][2];
    const double c12 = (J[0][1] * J[0][2] + J[1][1] * J[1][2]) + J[2][1] * J[2][2];
    double e[6];
    for (int i = 0; i < 6; ++i) e[i] = 2 * u01(s) - 1;
    hk::ArithFast af;
    double la, le;
    hk::lmin3_pair<hk::ArithFast, true>(af, c00, c11, c22, c01, c02, c12, e[0], e[1], e[2], e[3],
                                        e[4], e[5], la, le);
    acc += la + le + (af.ok ? 0.0 : 1.0);
  }
  out[blockIdx.x * 64 + threadIdx.x] = acc;
}

template <int MINB>
void run(int blocks_per_sm) {
  int sms = 148;
  const int blocks = sms * blocks_per_sm, reps = 200;
  double *o;
  cudaMalloc(&o, sizeof(double) * blocks * 64);
  jk<MINB><<<blocks, 64>>>(10, o);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  jk<MINB><<<blocks, 64>>>(reps, o);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  int regs = 0;
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, jk<MINB>);
  regs = fa.numRegs;
  const double pairs = (double)blocks * 64 * reps;
  // assume ~9.06 rotations per lmin3 (C2) -> 2 x 9.06 x 48 instr + 2 (tol) per pair
  const double instr = pairs * (2 * 9.06 * 48 + 2);
  printf("CTAs/SM %2d  regs %3d  %.3f ms  pair-solves/s %.3e  algorithmic FP64 instr/s %.3e  "
         "= %.1f %% of 1.71e13 DFMA/s\n", blocks_per_sm, regs, ms, pairs / (ms * 1e-3),
         instr / (ms * 1e-3), 100.0 * instr / (ms * 1e-3) / 1.71e13);
  cudaFree(o);
}

int main() {
  run<10>(10);
  run<10>(20);
  run<16>(16);
  run<16>(32);
  run<8>(8);
  return 0;
}
