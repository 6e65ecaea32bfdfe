// Throughput (not latency) of the FP64 seed instructions and of the exact fast paths:
// 8 independent chains per thread, full occupancy, all SMs.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2104_11404_b200/csrc/ieee_fast.cuh"

template <int OP>
__global__ void __launch_bounds__(256) tp(double *out, int n) {
  double x[8], y[8];
  bool ok = true;
  for (int k = 0; k < 8; ++k) x[k] = y[k] = 1.0 + (threadIdx.x + k) * 1e-7;
#pragma unroll 1
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (OP == 0) x[k] = __fma_rn(x[k], 0.9999999, 1e-7);
      if (OP == 1) x[k] = __hiloint2double(__double2hiint(hk::rcp_seed(x[k])), 0x3ff00000) ;
      if (OP == 2) x[k] = __hiloint2double(__double2hiint(hk::rsq_seed(x[k])), 0x3ff00000);
      if (OP == 3) x[k] = hk::div_fast(1.0, x[k], ok);
      if (OP == 4) x[k] = hk::sqrt_fast(x[k], ok);
      if (OP == 5) x[k] = hk::rcp_fast(x[k], ok);
      if (OP == 6) { float f = __double2float_rn(x[k]); asm("rcp.approx.ftz.f32 %0, %0;" : "+f"(f)); x[k] = f; }
      if (OP == 7) {  // 4 DFMA + 1 MUFU.RCP64H per k (independent): do they share a pipe?
        x[k] = __fma_rn(x[k], 0.9999999, 1e-7);
        x[k] = __fma_rn(x[k], 0.9999999, 1e-7);
        x[k] = __fma_rn(x[k], 0.9999999, 1e-7);
        x[k] = __fma_rn(x[k], 0.9999999, 1e-7);
        y[k] = __hiloint2double(__double2hiint(hk::rcp_seed(y[k])), 0x3ff00000);
      }
    }
  }
  double s = 0;
  for (int k = 0; k < 8; ++k) s += x[k] + y[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + ok;
}

template <int OP>
void run(const char *name) {
  const int blocks = 148 * 8, n = 2000;
  double *o;
  cudaMalloc(&o, sizeof(double) * blocks * 256);
  tp<OP><<<blocks, 256>>>(o, 10);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  tp<OP><<<blocks, 256>>>(o, n);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double ops = (double)blocks * 256 * n * 8;
  printf("%-34s %.3e ops/s  = %6.2f per clk per SM at 1965 MHz\n", name, ops / (ms * 1e-3),
         ops / (ms * 1e-3) / 148 / 1.965e9);
  cudaFree(o);
}

int main() {
  run<0>("DFMA");
  run<1>("MUFU.RCP64H (+hi/lo moves)");
  run<2>("MUFU.RSQ64H (+hi/lo moves)");
  run<3>("div_fast");
  run<4>("sqrt_fast");
  run<5>("rcp_fast");
  run<6>("F2F + MUFU.RCP f32 + F2F");
  run<7>("mix: 4 DFMA + 1 MUFU.RCP64H (per op)");
  return 0;
}
