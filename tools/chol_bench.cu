// Microbenchmark of the warp-level 32x32 Cholesky + inverse (chol32_warp) and
// the 64x64 leaf in isolation: one CTA, clock64 stamps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2504_19171_b200/csrc chol_bench.cu -o chol_bench
#define TIB_LEAF_TIMING
#include "../paper_2504_19171_b200/csrc/kernels.cu"
#include <cstdio>
#include <vector>
using namespace tib;

template <bool F, bool WX = true, bool BK = true>
__global__ void chol_kernel(const double* A, double* out, long long* cyc, int reps) {
  extern __shared__ __align__(16) double smem[];
  double* SA = smem;
  double* SX = smem + kLeaf * kLs;
  double* vec = SX + kLeaf * kLs;
  for (int i = threadIdx.x; i < 32 * 32; i += blockDim.x) SA[(i / 32) * kLs + i % 32] = A[i];
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (threadIdx.x < 32) chol32_warp<F, WX, BK>(SA, SX, vec, vec + 128, vec + 256);
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / reps;
  for (int i = threadIdx.x; i < 32 * 32; i += blockDim.x) out[i] = SX[(i / 32) * kLs + i % 32];
}

// warp-specialised chol32 (chol32_l on warp 0, chol32_x on warp 1)
__global__ void split_kernel(const double* A, double* out, long long* cyc, int reps) {
  extern __shared__ __align__(16) double smem[];
  double* SA = smem;
  double* SX = smem + kLeaf * kLs;
  double* vec = SX + kLeaf * kLs;
  for (int i = threadIdx.x; i < 32 * 32; i += blockDim.x) SA[(i / 32) * kLs + i % 32] = A[i];
  __syncthreads();
  long long t0 = clock64();
  volatile int* flag = reinterpret_cast<volatile int*>(vec + 7 * kL2);
  for (int r = 0; r < reps; ++r) {
    if (threadIdx.x == 0) *flag = 0;
    __syncthreads();
    if (threadIdx.x < 32) chol32_l<true>(SA, SX + kL2, vec + 128, vec + 288, vec + 192, flag);
    else if (threadIdx.x < 64) chol32_x(SX, SX + kL2, vec + 192, flag);
    __syncthreads();
    for (int i = threadIdx.x; i < 32 * 32; i += blockDim.x) SA[(i / 32) * kLs + i % 32] = A[i];
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / reps;
}

__global__ void chol2_kernel(const double* A, long long* cyc, int mode) {
  extern __shared__ __align__(16) double smem[];
  double* SA = smem;
  double* SX = smem + kLeaf * kLs;
  double* vec = SX + kLeaf * kLs;
  for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) SA[(i / 64) * kLs + i % 64] = (i % 64 <= i / 64) ? A[i] : 0.0;
  __syncthreads();
  long long t0 = clock64();
  if (threadIdx.x < 32) chol32_warp<true>(SA, SX, vec, vec + 128, vec + 288);
  __syncthreads();
  long long t1 = clock64();
  if (mode == 1) {
    cta_dmma<32, 32>(SA + 32 * kLs, kLs, SA + 32 * kLs, kLs, SX, kLs, true, kL2, 1.0, false);
    cta_dmma<32, 32>(SA + 32 * kLs + 32, kLs, SA + 32 * kLs, kLs, SA + 32 * kLs, kLs, true, kL2, -1.0, true);
  }
  long long t2 = clock64();
  if (threadIdx.x < 32) chol32_warp<true>(SA + 32 * kLs + 32, SX + 32 * kLs + 32, vec, vec + 160, vec + 320);
  __syncthreads();
  long long t3 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}

// copy of the leaf's compute sequence with a compile-time factor flag
__device__ __noinline__ void leafT_body(const double* Ain, long long* cyc, int reps, double* smem) {
  double* SA = smem;
  double* SX = smem + kLeaf * kLs;
  double* SP = SX + kLeaf * kLs;
  double* vec = SP + kLeaf * kLs;
  double* dv = vec + 9 * kL2;
  double* piv = vec + 4 * kL2;
  const int t = threadIdx.x;
  long long c0 = 0, c1 = 0, c2 = 0;
  for (int rep = 0; rep < reps; ++rep) {
    for (int idx = t; idx < 64 * 64; idx += blockDim.x) SA[(idx / 64) * kLs + idx % 64] = (idx % 64 <= idx / 64) ? Ain[idx] : 0.0;
    __syncthreads();
    long long a0 = clock64();
    if (t < 32) chol32_warp<true>(SA, SX, vec, piv, dv);
    __syncthreads();
    long long a1 = clock64();
    cta_dmma<32, 32>(SA + 32 * kLs, kLs, SA + 32 * kLs, kLs, SX, kLs, true, kL2, 1.0, false);
    cta_dmma<32, 32>(SA + 32 * kLs + 32, kLs, SA + 32 * kLs, kLs, SA + 32 * kLs, kLs, true, kL2, -1.0, true);
    long long a2 = clock64();
    if (t < 32) chol32_warp<true>(SA + 32 * kLs + 32, SX + 32 * kLs + 32, vec, piv + kL2, dv + kL2);
    __syncthreads();
    long long a3 = clock64();
    c0 += a1 - a0; c1 += a2 - a1; c2 += a3 - a2;
  }
  if (t == 0) { cyc[0] = c0 / reps; cyc[1] = c1 / reps; cyc[2] = c2 / reps; }
}
__global__ void leafT_kernel(const double* Ain, long long* cyc, int reps) {
  extern __shared__ __align__(16) double smem[];
  leafT_body(Ain, cyc, reps, smem);
}

__global__ void leaf_kernel(const double* A, double* L, double* X, DevStatus* st, double* ld, long long* cyc, int reps) {
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
  std::vector<double> a32(32 * 32);
  for (int i = 0; i < 32; ++i)
    for (int j = 0; j < 32; ++j) a32[i * 32 + j] = (i == j) ? 40.0 : 1.0 / (1 + i + j);
  double *dA, *dA32, *dL, *dX, *dld, *dout; DevStatus* st; long long* cyc;
  cudaMalloc(&dA, 64 * 64 * 8); cudaMalloc(&dA32, 32 * 32 * 8); cudaMalloc(&dL, 64 * 64 * 8); cudaMalloc(&dX, 64 * 64 * 8);
  cudaMalloc(&dld, 8); cudaMalloc(&st, 8); cudaMalloc(&cyc, 64); cudaMalloc(&dout, 32 * 32 * 8);
  cudaMemcpy(dA, a.data(), 64 * 64 * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dA32, a32.data(), 32 * 32 * 8, cudaMemcpyHostToDevice);
  cudaMemset(st, 0xff, 8);
  cudaFuncSetAttribute(leaf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kFlowSmemBytes);
  cudaFuncSetAttribute(chol_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFlowSmemBytes);
  cudaFuncSetAttribute(chol_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFlowSmemBytes);
  long long c;
  for (int threads : {32, 128}) {
    for (int it = 0; it < 2; ++it) {
      chol_kernel<true><<<1, threads, kFlowSmemBytes>>>(dA32, dout, cyc, it == 0 ? 1 : 20);
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      printf("{\"chol32_factor_cycles\": %lld, \"threads\": %d, \"err\": \"%s\"}\n", c, threads, cudaGetErrorString(cudaGetLastError()));
      chol_kernel<false><<<1, threads, kFlowSmemBytes>>>(dA32, dout, cyc, it == 0 ? 1 : 20);
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      printf("{\"chol32_inverse_only_cycles\": %lld, \"threads\": %d}\n", c, threads);
    }
  }
  cudaFuncSetAttribute(chol_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFlowSmemBytes);
  for (int it = 0; it < 2; ++it) {
    chol_kernel<true, false><<<1, 32, kFlowSmemBytes>>>(dA32, dout, cyc, 20);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("{\"chol32_factor_noX_cycles\": %lld}\n", c);
  }
  cudaFuncSetAttribute(chol_kernel<true, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFlowSmemBytes);
  for (int it = 0; it < 2; ++it) {
    chol_kernel<true, false, false><<<1, 32, kFlowSmemBytes>>>(dA32, dout, cyc, 20);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("{\"chol32_chain_only_cycles\": %lld}\n", c);
  }
  cudaFuncSetAttribute(split_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kFlowSmemBytes);
  for (int it = 0; it < 2; ++it) {
    split_kernel<<<1, 128, kFlowSmemBytes>>>(dA32, dout, cyc, 20);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("{\"chol32_split_cycles_incl_reload\": %lld}\n", c);
  }
  cudaFuncSetAttribute(chol2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kFlowSmemBytes);
  for (int mode : {0, 1, 0, 1}) {
    long long cc[3];
    chol2_kernel<<<1, 128, kFlowSmemBytes>>>(dA, cyc, mode);
    cudaMemcpy(cc, cyc, 24, cudaMemcpyDeviceToHost);
    printf("{\"chol2_mode\": %d, \"first\": %lld, \"dmma\": %lld, \"second\": %lld}\n", mode, cc[0], cc[1], cc[2]);
  }
  cudaFuncSetAttribute(leafT_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kFlowSmemBytes);
  for (int it = 0; it < 2; ++it) {
    long long cc[3];
    leafT_kernel<<<1, 128, kFlowSmemBytes>>>(dA, cyc, 10);
    cudaMemcpy(cc, cyc, 24, cudaMemcpyDeviceToHost);
    printf("{\"leafT_chol_a\": %lld, \"dmma\": %lld, \"chol_b\": %lld}\n", cc[0], cc[1], cc[2]);
  }
  for (int it = 0; it < 3; ++it) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    leaf_kernel<<<1, 128, kFlowSmemBytes>>>(dA, dL, dX, st, dld, cyc, 20);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
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
  const int n = 60;
  printf("{\"compute\": %lld, \"store\": %lld, \"chol_a\": %lld, \"gemm2\": %lld, \"chol_b\": %lld, \"gemm2b\": %lld, \"chol32_inside_total\": %lld, \"chol32_calls\": %lld}\n",
         tim[0] / n, tim[1] / n, tim[2] / n, tim[3] / n, tim[4] / n, tim[5] / n, tim[6], tim[7]);
  printf("{\"llt_err\": %.3e, \"lx_err\": %.3e}\n", e1, e2);
  return 0;
}
