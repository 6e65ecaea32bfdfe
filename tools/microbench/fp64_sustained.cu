// Sustained FP64 peak on this part ("DFMA loop, all 148 SMs,
// sustained >= 4 s"): DFMA (8 independent chains per thread) and DMMA (mma.sync m8n8k4 f64)
// kernels launched back to back for `seconds` each; per ~0.5 s window the achieved TFLOP/s
// (CUDA events), then the overall rate.  Run with nvidia-smi sampling the SM clock beside it
// (tools/fp64_sustained.sh).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64_sustained.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int MODE>  // 0: DFMA, 1: DMMA
__global__ void burn(int iters, double *out, double seed) {
  double a = seed + threadIdx.x * 1e-3, b = seed * 0.5, acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = seed + i;
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = __fma_rn(acc[i], 0.999999, 1e-7);
    } else {
#pragma unroll
      for (int i = 0; i < 8; i += 2) dmma(acc[i], acc[i + 1], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

int main(int argc, char **argv) {
  const double seconds = argc > 1 ? atof(argv[1]) : 5.0;
  double *out;
  cudaMalloc(&out, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256;
  const char *names[2] = {"DFMA", "DMMA"};
  for (int mode = 0; mode < 2; ++mode) {
    // per launch: DFMA 8 fma x 2 flop per thread-iteration; DMMA 4 mma x 512 flop per warp-iteration
    const int iters = mode == 0 ? 200000 : 50000;
    const double flop = mode == 0 ? (double)blocks * threads * iters * 16.0
                                  : (double)blocks * threads / 32 * iters * 4 * 512.0;
    cudaEvent_t e0, e1, w0;
    cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&w0);
    // warm-up launch
    if (mode == 0) burn<0><<<blocks, threads>>>(iters / 10, out, 1.0); else burn<1><<<blocks, threads>>>(iters / 10, out, 1.0);
    cudaDeviceSynchronize();
    double total_ms = 0, total_flop = 0, win_ms = 0, win_flop = 0;
    int win = 0;
    cudaEventRecord(w0);
    while (total_ms < seconds * 1e3) {
      cudaEventRecord(e0);
      if (mode == 0) burn<0><<<blocks, threads>>>(iters, out, 1.0); else burn<1><<<blocks, threads>>>(iters, out, 1.0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      total_ms += ms; total_flop += flop; win_ms += ms; win_flop += flop;
      if (win_ms >= 500.0) {
        printf("%s window %2d: %7.1f ms  %6.2f TFLOP/s\n", names[mode], win++, win_ms, win_flop / win_ms / 1e9);
        fflush(stdout);
        win_ms = win_flop = 0;
      }
    }
    printf("%s sustained over %.2f s: %6.2f TFLOP/s\n", names[mode], total_ms / 1e3, total_flop / total_ms / 1e9);
    fflush(stdout);
  }
  return 0;
}
