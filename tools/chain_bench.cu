// Microbenchmark of the chain step in isolation (one CTA, no scheduler):
// leaf (Cholesky + inverse of the carried 64x64 block) + the fat second phase
// (next panel block, next diagonal update), repeated.  Variants time the leaf
// alone with and without the global load, to compare with the in-sweep step.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2504_19171_b200/csrc chain_bench.cu -o chain_bench
#include "../paper_2504_19171_b200/csrc/kernels.cu"
#include <cstdio>
#include <vector>
using namespace tib;

// mode 0: leaf with global load; 1: leaf on the carried block (reload SA from a
// copy first, outside the timed region); 2: leaf + fat (full chain step)
__global__ void chain_kernel(const double* A, const double* P, const double* Dn, double* L, double* X, double* Pout,
                             DevStatus* st, double* ld, long long* cyc, int steps, int mode) {
  extern __shared__ __align__(16) double smem[];
  long long total = 0, leaf_t = 0, fat_t = 0, fat_t0 = 0;
  for (int s = 0; s < steps; ++s) {
    if (mode != 0) {
      for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) smem[(i / 64) * kLs + i % 64] = (i % 64 <= i / 64) ? A[i] : 0.0;
      __syncthreads();
    }
    const long long t0 = clock64();
    PROF(-1);
    if (mode == 4) {
      // the sweep's pipelining: the previous step's D' tail on warps 2-3 during
      // the first 32x32 sweep (operands: whatever SP / SA hold)
      if (threadIdx.x < 64) leaf_first<true>(smem);
      else chain_fat_tail(smem);
      __syncthreads();
      leaf_rest<true>(L, X, 64, 64, 0, st, ld, smem);
    } else {
      leaf_potrf_inv<true>(mode == 0 ? A : nullptr, 64, L, X, 64, 64, 0, st, ld, smem);
    }
    const long long t1 = clock64();
    if (mode == 2 || mode == 4) {
      chain_fat_prefetch(P, Dn, 64, smem);
      double* SX = smem + kLeaf * kLs;
      for (int idx = threadIdx.x; idx < kL2 * kL2; idx += kGemmThreads) SX[(idx / kL2) * kLs + kL2 + (idx % kL2)] = 0.0;
      cp_async_wait<0>();
      __syncthreads();
      PROF(6);
      fat_t0 = clock64();
      chain_fat_head(Pout, 64, smem);
      fat_t += clock64() - fat_t0;
      PROF(7);
      if (threadIdx.x >= 64) chain_fat_tail(smem);
      __syncthreads();
    }
    if (false) {
      // code pollution: a block GEMM task between steps (like the sweep kernel's other paths)
      RSeg sg{P, Dn, 64, 64, 0, 64, kTransB, 0};
      RTask t{};
      t.C = Pout;
      t.ldc = t.ldc0 = 64;
      t.seg_count = 1;
      t.mode = kFull;
      gemm_task(t, LocalSegs{&sg, 1}, smem);
      chain_fat(P, Pout, Dn, 64, smem);
      __syncthreads();
    }
    const long long t2 = clock64();
    total += t2 - t0;
    leaf_t += t1 - t0;
  }
  if (threadIdx.x == 0) {
    cyc[0] = total / steps;
    cyc[1] = leaf_t / steps;
    cyc[2] = fat_t / steps;
  }
}

int main() {
  std::vector<double> a(64 * 64), p(64 * 64);
  for (int i = 0; i < 64; ++i)
    for (int j = 0; j < 64; ++j) {
      a[i * 64 + j] = (i == j) ? 70.0 : 1.0 / (1 + i + j);
      p[i * 64 + j] = 0.01 * ((i * 7 + j * 3) % 11 - 5);
    }
  double *dA, *dP, *dL, *dX, *dPo, *dld;
  DevStatus* st;
  long long* cyc;
  cudaMalloc(&dA, 32768); cudaMalloc(&dP, 32768); cudaMalloc(&dL, 32768); cudaMalloc(&dX, 32768);
  cudaMalloc(&dPo, 32768); cudaMalloc(&dld, 8); cudaMalloc(&st, 8); cudaMalloc(&cyc, 32);
  cudaMemcpy(dA, a.data(), 32768, cudaMemcpyHostToDevice);
  cudaMemcpy(dP, p.data(), 32768, cudaMemcpyHostToDevice);
  cudaMemset(st, 0xff, 8);
  cudaFuncSetAttribute(chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kFlowSmemBytes);
#ifdef TIB_PROF
  long long* prof;
  cudaMalloc(&prof, 16 * 8);
  cudaMemcpyToSymbol(g_prof, &prof, sizeof(prof));
#endif
  for (int mode : {0, 1, 2, 4, 0, 1, 2, 4}) {
#ifdef TIB_PROF
    cudaMemset(prof, 0, 16 * 8);
#endif
    chain_kernel<<<1, 128, kFlowSmemBytes>>>(dA, dP, dA, dL, dX, dPo, st, dld, cyc, 50, mode);
    long long c[3];
    cudaMemcpy(c, cyc, 24, cudaMemcpyDeviceToHost);
    printf("{\"mode\": %d, \"step_cycles\": %lld, \"leaf_cycles\": %lld, \"fat_dmma_cycles\": %lld, \"err\": \"%s\"}\n", mode, c[0], c[1], c[2],
           cudaGetErrorString(cudaGetLastError()));
#ifdef TIB_PROF
    long long h[16];
    cudaMemcpy(h, prof, 16 * 8, cudaMemcpyDeviceToHost);
    printf("  prof per step:");
    for (int i = 0; i < 10; ++i) printf(" p%d=%lld", i, h[i] / 50);
    printf("\n");
#endif
  }
  return 0;
}
