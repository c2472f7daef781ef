// Microbenchmark of the 64x64 leaf (factor + inverse) in isolation: one CTA,
// clock64 stamps.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2504_19171_b200/csrc
#define TIB_LEAF_TIMING
#include "../paper_2504_19171_b200/csrc/kernels.cu"
#include <cstdio>
#include <vector>
using namespace tib;

__global__ void leaf_bench_kernel(const double* A, double* L, double* X, DevStatus* st, double* ld, long long* cyc, int reps) {
  extern __shared__ __align__(16) double smem[];
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r)
    leaf_potrf_inv<true>(A, 64, L, X, 64, 64, 0, st, ld, smem);
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / reps;
}

int main() {
  std::vector<double> a(64 * 64);
  for (int i = 0; i < 64; ++i)
    for (int j = 0; j < 64; ++j) a[i * 64 + j] = (i == j) ? 70.0 : 1.0 / (1 + i + j);
  double *dA, *dL, *dX, *dld; DevStatus* st; long long* cyc;
  cudaMalloc(&dA, 64 * 64 * 8); cudaMalloc(&dL, 64 * 64 * 8); cudaMalloc(&dX, 64 * 64 * 8);
  cudaMalloc(&dld, 8); cudaMalloc(&st, 8); cudaMalloc(&cyc, 8);
  cudaMemcpy(dA, a.data(), 64 * 64 * 8, cudaMemcpyHostToDevice);
  cudaMemset(st, 0xff, 8);
  cudaFuncSetAttribute(leaf_bench_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kFlowSmemBytes);
  for (int it = 0; it < 3; ++it) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    leaf_bench_kernel<<<1, 128, kFlowSmemBytes>>>(dA, dL, dX, st, dld, cyc, 20);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("{\"leaf_cycles\": %lld, \"us_per_leaf\": %.2f, \"err\": \"%s\"}\n", c, ms * 1000 / 20, cudaGetErrorString(cudaGetLastError()));
  }
  std::vector<double> l(64 * 64), x(64 * 64);
  cudaMemcpy(l.data(), dL, 64 * 64 * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(x.data(), dX, 64 * 64 * 8, cudaMemcpyDeviceToHost);
  double e1 = 0, e2 = 0;
  for (int i = 0; i < 64; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = 0; for (int k = 0; k <= j; ++k) s += l[i * 64 + k] * l[j * 64 + k];
      e1 = fmax(e1, fabs(s - a[i * 64 + j]));
      double t = 0; for (int k = j; k <= i; ++k) t += l[i * 64 + k] * x[k * 64 + j];
      e2 = fmax(e2, fabs(t - (i == j)));
    }
  long long tim[8]; cudaMemcpyFromSymbol(tim, g_leaf_timing, 64);
  printf("{\"compute\": %lld, \"store\": %lld, \"leaf32a\": %lld, \"gemm2\": %lld, \"leaf32b\": %lld, \"gemm2b\": %lld}\n", tim[0] / 60, tim[1] / 60, tim[2]/60, tim[3]/60, tim[4]/60, tim[5]/60);
  printf("{\"llt_err\": %.3e, \"lx_err\": %.3e}\n", e1, e2);
  return 0;
}
