// FP64 pipe microbenchmark: DFMA peak, and IEEE div / sqrt throughput on sm_100a.
// Used once to fix the roofline denominators in DESIGN.md (not part of the product).
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

template<int ILP>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double acc[ILP];
  #pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = __fma_rn(acc[i], a, b);
  }
  double s = 0; 
  #pragma unroll
  for (int i = 0; i < ILP; ++i) s += acc[i];
  if (s == 1.2345) out[threadIdx.x] = s;
}
template<int ILP>
__global__ void ddiv_loop(double* out, int iters, double a) {
  double acc[ILP];
  #pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = 1.0 + threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = a / acc[i];
  }
  double s = 0;
  #pragma unroll
  for (int i = 0; i < ILP; ++i) s += acc[i];
  if (s == 1.2345) out[threadIdx.x] = s;
}
template<int ILP>
__global__ void dsqrt_loop(double* out, int iters) {
  double acc[ILP];
  #pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = 2.0 + threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = sqrt(acc[i]) + 1.5;
  }
  double s = 0;
  #pragma unroll
  for (int i = 0; i < ILP; ++i) s += acc[i];
  if (s == 1.2345) out[threadIdx.x] = s;
}

int main() {
  double* out; CK(cudaMalloc(&out, 1 << 20));
  int dev; cudaGetDevice(&dev); cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int sms = p.multiProcessorCount;
  printf("device %s sms=%d\n", p.name, sms);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int threads = 512, blocksPerSM = 4;
  int grid = sms * blocksPerSM;
  // DFMA: run ~4 s sustained and also a short burst
  for (int rep = 0; rep < 2; ++rep) {
    int iters = rep == 0 ? 20000 : 400000;
    dfma_loop<8><<<grid, threads>>>(out, 100, 1.0000001, 1e-7);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dfma_loop<8><<<grid, threads>>>(out, iters, 1.0000001, 1e-7);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * (double)iters * threads * grid;
    printf("dfma %s: %.3f ms  %.2f TFLOP/s\n", rep ? "sustained" : "burst", ms, flops / ms / 1e9);
  }
  {
    int iters = 20000;
    ddiv_loop<4><<<grid, threads>>>(out, 100, 3.0); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    ddiv_loop<4><<<grid, threads>>>(out, iters, 3.0);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = 4.0 * iters * threads * grid;
    printf("ddiv: %.3f ms  %.2f Gdiv/s  (%.2f div/clk/SM at %d MHz)\n", ms, ops / ms / 1e6,
           ops / (ms * 1e-3) / sms / (p.clockRate * 1e3), p.clockRate / 1000);
  }
  {
    int iters = 20000;
    dsqrt_loop<4><<<grid, threads>>>(out, 100); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dsqrt_loop<4><<<grid, threads>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = 4.0 * iters * threads * grid;
    printf("dsqrt(+add): %.3f ms  %.2f Gsqrt/s\n", ms, ops / ms / 1e6);
  }
  return 0;
}
