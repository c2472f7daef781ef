// Dataflow task plans for the two device sweeps (kernels.cu dataflow_kernel).
//
// A plan is a pointer-free task list (store id + offset addressing, see
// taskfmt.hpp) with per-task dependency lists and completion signals on
// integer counters.  It is built once per tile pattern (and per closure for
// phase 2), cached, and shared by every matrix with that pattern -- including
// all members of a batch.  Building it is pure integer work on the host.
#pragma once

#include <vector>

#include "planner.hpp"
#include "taskfmt.hpp"

namespace tib {

struct DataflowPlan {
  Layout L;
  int bp = 0, nb = 0;
  std::vector<DTask> tasks;  // queue 0 (critical chain) then queue 1 (bulk)
  std::vector<Seg> segs;
  std::vector<Dep> deps;
  std::vector<int> sigs;
  QueueDesc q0{}, q1{};
  long counters = 0;          // ints per matrix
  size_t scratch_doubles = 0; // per matrix
  size_t logdet_doubles = 0;  // per matrix
  double task_flops = 0;      // FLOPs actually executed by the block tasks (2 per FMA)
  // 64-row strips right of each diagonal block that must read zero in the L and
  // phase-1 stores (upper triangle of the diagonal tiles): origin offset and
  // width in 64-column blocks; cleared by a separate kernel before the sweep.
  std::vector<ZeroStrip> zero;
  std::vector<Coord> slot_tiles;  // tile coordinates of the store slots (diagnostics: task traces)
  // push-model scheduling tables (finalize_waiters): per task the number of
  // first-phase dependencies not satisfied initially, per counter its waiters
  // (CSR, sorted by value), and the initially ready tasks of each queue
  // waiters of counter c reaching value v: wl[vidx[vbase[c] + v] .. vidx[vbase[c] + v + 1]),
  // for 1 <= v <= vbase[c + 1] - vbase[c] - 2
  std::vector<int> need, vbase, vidx, init0, init1;
  std::vector<int> wl;
  std::vector<DTask> chain;  // leaf steps of the chain task (kChainTask), in order
  // streamed upload (factor sweep): counter upl + c is set to 1 by the copy
  // stream once tile column c of A is resident; every task and chain step that
  // touches the A store polls the counter of the latest column it touches
  long upl = -1;
  // order in which the copy stream uploads the tile columns: by the first
  // column whose elimination touches them (the arrow tip, updated by every
  // column, goes up with the first columns instead of last); each task polls
  // the counter of the touched column uploaded last
  std::vector<int> upload_order;
};

// Fused factorization + phase 1 over the FILLED pattern: per column, the
// diagonal-tile chain (64x64 leaves + intra-tile panel / trailing / inverse
// rows) on queue 0; panel GEMMs L_kj = A_kj X_j^T, Schur updates (critical
// column first) and deferred W_kj = L_kj X_j on queue 1.
// fat_leaf fuses the next panel block and diagonal-block update into the leaf task.
// chain: the leaves (fat) become the steps of one persistent chain task per matrix.
// boundary: the last leaf of each tile also forms row 0 of the next tile's last
// panel block and the last update term of the next diagonal block (S trick).
// split > 0: columns [split, N) form a second elimination chain independent of
// [0, split) until they meet (two_chain_order): two chain tasks, one scratch
// ring each.
// coarse_second (with split): the second off-diagonal tile's panel and update
// as whole-K bulk tasks instead of the progressive split-K parts.
// ugroup > 1: the bulk updates of a tile are grouped, up to ugroup terms
// (ascending column) per task -- one multi-segment GEMM of K = ugroup * bp
// instead of ugroup K = bp tasks; a tile's pending terms go out before the
// tile's next non-bulk use (its panel, leaf or critical split update).
DataflowPlan build_factor_dataflow(const Pattern& filled, int crit_workers, int defer_w, bool fat_leaf,
                                   bool chain = false, bool boundary = false, int split = -1,
                                   bool coarse_second = false, int ugroup = 1);

// Phase 1 alone (selinv.cpp:195-237) from a given factor L (a factor read back
// from a tile file): X_j = L_jj^{-1} and W_kj = L_kj X_j, every column
// independent, all on the bulk queue.  The sweep's A-store entry must point at
// the L store (the invert-only leaves read their block from there).
DataflowPlan build_phase1_dataflow(const Pattern& filled);

// Phase 2 over a closure: per column descending, off-diagonal targets split
// into an early part and the k == j term, diagonal targets into LAUUM + early
// terms and the first-row term; the first-row chain is queue 0.
// split > 0 (two-chain order): the columns below split get their own ring of
// split-K slots (an independent chain once the columns above are done).
// group: late (critical) terms per split-K part.
DataflowPlan build_phase2_dataflow(const Pattern& filled, const Closure& sel, int crit_workers, int split = -1,
                                   int group = 1);

// Simulates the plan in its global emission order (queue 0 and queue 1 are
// both subsequences of it) and throws ConsistencyError if any dependency is
// not produced by an earlier task -- the property that makes in-order claiming
// deadlock-free.
void validate_dataflow(const DataflowPlan& plan, const std::vector<int>& global_order);

}  // namespace tib
