// Launch wrappers for the sm_100a kernels of the tile path (kernels.cu).
// Host code (engine.cpp) only sees these; no torch types anywhere.
#pragma once

#include <cuda_runtime.h>

#include "gemm_dmma.cuh"

namespace tib {

// Device-side error word: first non-positive pivot (global scalar index),
// ULLONG_MAX when the factorization succeeded.
struct DevStatus {
  unsigned long long first_bad_pivot;
};

// One diagonal tile to factor and/or invert on one thread-block cluster.
//   mode kFactorInvert: L = chol(A lower), X = L^{-1}   (factor sweep, phase 1 fused)
//   mode kInvertOnly  : X = L^{-1} from an existing L   (standalone phase 1)
// Offsets are in doubles into the matrix's stores (A, L, P1, scratch,
// logdet), resolved through the per-matrix BaseTable like block tasks.
enum DiagMode : int { kFactorInvert = 0, kInvertOnly = 1 };
constexpr int kStoreLogdet = 6;
struct DiagJob {
  long long a_off, l_off, x_off, t_off, logdet_off;
  long long pivot_base;  // global scalar index of the tile's first row (j * b)
  int valid_rows;        // rows of this tile that are real matrix rows
  int mode;
};

constexpr int kDiagCluster = 16;  // CTAs per diagonal tile (non-portable cluster size)

// tasks[0..count) x tables[0..batch): grid (count, batch), one block task per CTA.
void launch_gemm_tasks(const Task* tasks, const Seg* segs, int count, const BaseTable* tables,
                       int batch, cudaStream_t s);
// jobs[0..count) x tables[0..batch), one cluster of `cluster` CTAs each;
// status[matrix] is the table's kStoreStatus entry.
void launch_diag_jobs(const DiagJob* jobs, int count, const BaseTable* tables, int batch, int bp,
                      int cluster, cudaStream_t s);
void launch_fill(double* p, double v, size_t count, cudaStream_t s);
int configure_kernels();  // sets smem / cluster attributes once; returns cudaError_t

}  // namespace tib
