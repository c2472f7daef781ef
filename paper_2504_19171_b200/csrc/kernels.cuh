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
// Everything the persistent sweep kernel reads: the plan (device copies),
// the per-matrix base tables, and the per-sweep scheduler state.
struct FlowArgs {
  const DTask* tasks;
  const Seg* segs;
  const Dep* deps;
  const int* sigs;
  const int* vbase;  // counters + 1
  const int* vidx;
  const int* wl;
  QueueDesc q0, q1;
  int batch, ntasks;
  const BaseTable* tables;
  int* missing;  // batch x ntasks
  int* slots0;   // q0.count x batch
  int* slots1;   // q1.count x batch
  int* ctl;      // head0, tail0, head1, tail1 (128-byte apart)
  const DTask* chain;  // chain steps (kChainTask)
  int dedicate;        // chains get their SM to themselves
  int static_chains;   // chains run on worker 0 of CTAs 0 .. batch-1 (q0 items 0 .. batch-1 skipped)
  int poll_shift;      // polling backoff caps scaled by 2^poll_shift
  int agent;           // with dedicate + static_chains: the chain's sibling worker raises its signals
  int poll_uploads;    // streamed upload: tasks wait for their A-store column (DTask::poll)
  int c0_prefetch;     // plain tasks stage C0 in shared memory during their main loop
  unsigned long long watchdog_ns;  // a spin longer than this aborts the sweep (TIB_ERR_CUDA)
  unsigned long long* trace;
};

// Sticky watchdog record {flag, counter, value, dep index}; cleared once read.
int read_watchdog(int* rec);
// Chain phase profile accumulator (16 long longs of device memory) or null.
int set_chain_profile(long long* p);

void launch_dataflow(const FlowArgs& a, const int* need, const int* init0, int n_init0, const int* init1, int n_init1,
                     int grid, cudaStream_t s);
void launch_zero_strips(const ZeroStrip* z, int count, int ld, int batch, const BaseTable* tables, cudaStream_t s);
void launch_fill(double* p, double v, size_t count, cudaStream_t s);
// generate.cu: density-1 arrowhead generator (matgen.cpp:59-120) into a tile
// store over a pattern given as device CSC (colptr[N + 1], rows), row stride bp.
int launch_generate_arrowhead(long n, long w, long t, unsigned long long seed, int b, int bp, int N, const int* colptr,
                              const int* rows, int max_col_slots, double* out, cudaStream_t s);

}  // namespace tib
