// FP64 peak microbenchmarks for B200 (sm_100a): DMMA (mma.sync m8n8k4 f64),
// DFMA (fma.rn.f64) and, from the Python side, cuBLAS DGEMM.  MEASURED_PEAKS.json
// carries no FP64 figure, so the roofline denominator for this path comes from here.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

template <int CHAINS>
__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i];
  if (s == 12345.0) out[threadIdx.x] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  double* out; CK(cudaMalloc(&out, 1 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  printf("{\"sms\": %d, \"clock_khz\": %d}\n", sms, clk);
  const int iters = 20000;
  for (int warps : {4, 8, 16}) {
    for (int bps : {1, 2, 4}) {
      dim3 grid(sms * bps), block(32 * warps);
      dmma_loop<8><<<grid, block>>>(out, 100);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      dmma_loop<8><<<grid, block>>>(out, iters);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 256.0 * 8 * iters * (double)grid.x * warps;
      printf("{\"kind\": \"dmma_m8n8k4\", \"warps\": %d, \"blocks_per_sm\": %d, \"tflops\": %.3f, \"ms\": %.3f}\n",
             warps, bps, flops / ms / 1e9, ms);
    }
  }
  for (int warps : {8, 16, 32}) {
    dim3 grid(sms * 2), block(32 * warps);
    dfma_loop<8><<<grid, block>>>(out, 100);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dfma_loop<8><<<grid, block>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * iters * (double)grid.x * block.x;
    printf("{\"kind\": \"dfma\", \"warps\": %d, \"tflops\": %.3f, \"ms\": %.3f}\n", warps, flops / ms / 1e9, ms);
  }
  // sustained DMMA: ~4 s back to back
  {
    dim3 grid(sms * 2), block(32 * 8);
    cudaEventRecord(e0);
    int reps = 0; float ms = 0;
    while (ms < 4000.f) {
      dmma_loop<8><<<grid, block>>>(out, iters);
      ++reps;
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    }
    double flops = 2.0 * 256.0 * 8 * iters * (double)grid.x * 8 * reps;
    printf("{\"kind\": \"dmma_sustained_4s\", \"tflops\": %.3f, \"ms\": %.1f}\n", flops / ms / 1e9, ms);
  }
  return 0;
}
