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
  int static_chains;   // chain tasks per matrix (q0 tasks 0 ..), run on worker 0 of CTAs 0 .. static_chains * batch - 1
  int poll_shift;      // polling backoff caps scaled by 2^poll_shift
  int agent;           // with dedicate + static_chains: the chain's sibling worker raises its signals
  int poll_uploads;    // streamed upload: tasks wait for their A-store column (DTask::poll)
  int c0_prefetch;     // plain tasks stage C0 in shared memory during their main loop
  int early_ticket;    // bulk workers take their next q1 ticket once a task's waits are over (atomic latency hidden under the epilogue)
  // streamed two-chain upload (one matrix): worker 1 of the last t_agents CTAs
  // places the staged tiles of each column (upload order t_cols; entries
  // t_off[c] .. t_off[c+1]: Sigma-store slot t_src -> A-store slot t_dst,
  // transposed when t_tr) once the copy engine has set the column's raw
  // counter, then sets its upload counter; counters complete in upload order
  int t_agents, t_ncols, t_bp;
  const int* t_cols;
  const int* t_off;
  const int* t_dst;
  const int* t_src;
  const unsigned char* t_tr;
  long long t_raw, t_upl, t_arrive;  // counter offsets (raw per column, upload per column, arrivals per column)
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
void launch_gather(const double* src, const long long* idx, double* out, long long n, cudaStream_t s);
void launch_permute_tiles(double* dst, const double* src, const int* d, const int* s, const unsigned char* tr,
                          int count, int bp, int max_blocks, cudaStream_t st);
void launch_permute_rows(double* dst, const double* src, const int* d, const int* s, int count, int bp, cudaStream_t st);
// generate.cu: density-1 arrowhead generator (matgen.cpp:59-120) into a tile
// store over a pattern given as device CSC (colptr[N + 1], rows), row stride bp.
int launch_generate_arrowhead(long n, long w, long t, unsigned long long seed, int b, int bp, int N, const int* colptr,
                              const int* rows, int max_col_slots, double* out, cudaStream_t s,
                              const unsigned long long* seeds = nullptr, int count = 1, long long stride = 0);

}  // namespace tib
