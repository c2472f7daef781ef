// Device task formats and launch wrappers for the sm_100a kernels of the tile
// path (kernels.cu).  Host code (engine.cpp) only sees these; no torch types.
#pragma once

#include <cuda_runtime.h>

#include "gemm_dmma.cuh"

namespace tib {

// Device-side error word: first non-positive pivot (global scalar index),
// ULLONG_MAX when the factorization succeeded.
struct DevStatus {
  unsigned long long first_bad_pivot;
};

int configure_kernels();  // smem attribute; returns cudaError_t
int dataflow_grid(int device);
void launch_dataflow(const DTask* tasks, const Seg* segs, const Dep* deps, const int* sigs, QueueDesc q0,
                     QueueDesc q1, int batch, const BaseTable* tables, int* claim, int grid, cudaStream_t s,
                     unsigned long long* trace = nullptr);
void launch_zero_strips(const ZeroStrip* z, int count, int ld, int batch, const BaseTable* tables, cudaStream_t s);
void launch_fill(double* p, double v, size_t count, cudaStream_t s);

}  // namespace tib
