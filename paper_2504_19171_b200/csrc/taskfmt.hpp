// Plain-old-data task formats shared by the host planner (plan.cpp, built
// with the host compiler) and the device kernels (gemm_dmma.cuh, kernels.cu).
#pragma once

namespace tib {

constexpr int kBM = 64;
constexpr int kBN = 64;
constexpr int kBK = 16;

enum SegFlags : int { kTransA = 1, kTransB = 2, kNegate = 4 };

// Plans are built once per (pattern, request) on the host and must not depend
// on where the stores live (results get fresh allocations; a batch of
// matrices shares one plan), so tasks address operands as (store id, offset
// in doubles); a per-matrix base table resolves them at run time.
enum StoreId : int {
  kStoreA = 0,      // working copy of A (receives the Schur updates in place)
  kStoreL = 1,      // factor tiles L
  kStoreP1 = 2,     // phase-1 tiles: X_j = L_jj^{-1} on the diagonal, W_kj off it
  kStoreSigma = 3,  // selected-inverse tiles
  kStoreVar = 4,    // marginal variances (N * bp)
  kStoreScratch = 5,
  kStoreLogdet = 6,    // logdet partials (N * bp/64)
  kStoreStatus = 7,    // DevStatus word of the matrix
  kStoreCounters = 8,  // dataflow dependency counters (int)
  kStoreNone = 255,
};
constexpr int kMaxStores = 10;
struct BaseTable {
  double* p[kMaxStores];
};

// One K segment.  op(A) rows are the task's block rows, op(B) columns the
// task's block columns; offsets point at the operand matrix origin (a tile or
// a sub-block of one) with leading dimensions lda/ldb.
struct Seg {
  long long a_off, b_off;
  int lda, ldb;
  short k_lo, k_hi;  // K range [k_lo, k_hi), multiples of kBK
  unsigned char flags, a_store, b_store, pad;
};

enum TaskMode : int {
  kFull = 0,       // write the whole block to C
  kSymDiag = 1,    // diagonal block of a symmetric tile: lower part -> C and mirrored
  kMirror = 2,     // off-diagonal block of a symmetric tile: C and transpose into Cm
};

struct Task {
  long long c_off, c0_off, cm_off, diag_off;
  int ldc, ldc0;
  int m0, n0;
  int seg_begin, seg_count;
  unsigned char mode, c_store, c0_store, cm_store;
  unsigned char diag_store, pad0, pad1, pad2;
};

// Leaf / chain-step mode bits (DTask::mode of a kLeafTask): 1 invert only,
// 2 fat leaf, 4 tile-boundary leaf, kCarry: the block the step updates last
// is the next chain step's, which may take it from shared memory.
constexpr int kCarry = 16;

enum TaskKind : unsigned char { kGemmTask = 0, kLeafTask = 1, kSplitTask = 2, kChainTask = 3 };

// One schedulable unit of a sweep.  kGemmTask: C / C0 / Cm / diag stores and
// offsets as Task, segments [seg_begin, seg_begin + seg_count).  kLeafTask:
// c_off = A block (input, ld = ldc0), c0_off = L block, cm_off = X block
// (ld = ldc), diag_off = logdet slot, m0 = valid rows, n0 = global pivot
// index of the block's first row, mode = 0 factor + invert / 1 invert only
// (| 2: fat leaf, also the next panel block and next diagonal-block update).
// kSplitTask: one K-part of a split-K block GEMM: writes its partial product
// to scratch slot p_off + part * 64*64, bumps the arrival counter aux0, and
// the last of the `parts` arrivals (aux1 = part << 8 | parts) reduces all
// partials in part order (deterministic), adds C0 and runs the epilogue of
// `mode` like a kGemmTask.  Only the reducer signals.
// kChainTask: the whole diagonal chain of one matrix run by one CTA: steps
// [seg_begin, seg_begin + seg_count) of the plan's chain list, each a (fat)
// leaf descriptor executed in order, waiting on its own dependencies and
// keeping the next diagonal block in shared memory between steps.
// Dependencies: deps [dep_begin, dep_begin + dep_count) are waited before the
// task starts; the next dep2_count are waited before its second phase (the
// fat part of a leaf, the reduction of a split task) -- typically the
// update-ordering counter of the block it writes.  Signals: the last
// sig2_count of a leaf's signals are raised after its second phase, the
// others as soon as its first phase is done.
struct DTask {
  long long c_off, c0_off, cm_off, diag_off, p_off;
  int ldc, ldc0;
  int m0, n0;
  int seg_begin, seg_count;
  int dep_begin, sig_begin;
  int aux0, aux1;
  int poll;    // streamed upload: counter (>= 1 once the A-store column the task touches is uploaded), or -1
  int chunks;  // GEMM / split tasks: K chunks over all segments (set by the plan; the main loop needs no count pass)
  unsigned short dep_count, sig_count;
  unsigned char kind, mode, c_store, c0_store, cm_store, diag_store, dep2_count, sig2_count;
};

// wait until counters[counter] >= value
struct Dep {
  int counter;
  int value;
};

// 64 rows x (blocks * 64) doubles at `off` in the L and phase-1 stores, zeroed.
struct ZeroStrip {
  long long off;
  int blocks, pad;
};

// A queue is a contiguous range of the task array; `workers` CTAs serve q0
// (the critical chain) only, the rest of the grid serves q0 first, then q1.
struct QueueDesc {
  int first, count, workers, pad;
};

// Push-model scheduling (plan.hpp vbase / vidx / wl): for every counter and
// value, the tasks whose dependency that value completes.  The task whose
// signal brings a counter to the value decrements each such waiter's
// missing-dependency count, and the one that reaches zero enqueues it.

}  // namespace tib
