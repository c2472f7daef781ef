// Host engine of the B200 path: builds pointer-free task plans from the
// symbolic planner (plan.cpp), owns device stores, runs the two sweeps -- each
// one launch of the persistent dataflow executor (kernels.cu), captured into a
// CUDA graph per plan and batch size -- and implements the C ABI declared in
// include/tileinv_b200.h.
//
// Device data layout: every store is one contiguous allocation
// of `tiles x bp x bp` doubles in pattern slot order (column-major over the
// tile grid, diagonal first in each column), bp = b rounded up to 64 with
// identity padding on diagonal tiles.  Stores: A (working copy, Schur updates
// in place), L (factor), P1 (X_j = L_jj^{-1} on diagonal slots, W_kj = L_kj X_j
// off them), Sigma (closure slots), Var (N x bp marginal variances), Scratch
// (T-term accumulators, split-K partials), Logdet (N x bp/64 partial sums),
// Counters (dependency, arrival and upload counters).
//
// Sweeps: the fused factorization + phase 1 (64x64 block tasks:
// the diagonal chain, panels L_kj = A_kj X_j^T, Schur updates, W_kj), then
// phase 2 per closure column descending (selinv.cpp:239-345).  Single-matrix
// calls run in the two-chain elimination order when it pays off
// (selected_inverse_split); host inputs stream up under the factor sweep;
// batches are one launch per sweep (or pipelined groups for host batches).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <functional>
#include <atomic>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/tileinv_b200.h"
#include "kernels.cuh"
#include "plan.hpp"
#include "planner.hpp"

namespace tib {

#define CK(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess) throw Error(kErrCuda, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)


// ---------------------------------------------------------------------------
// memory
struct DevBuf {
  double* p = nullptr;
  size_t n = 0;  // doubles
  int dev = 0;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(size_t doubles, int device, cudaStream_t stream) : n(doubles), dev(device), s(stream) {
    if (n) CK(cudaMallocAsync(reinterpret_cast<void**>(&p), n * sizeof(double), s));
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), dev(o.dev), s(o.s) {
    o.p = nullptr;
    o.n = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      n = o.n;
      dev = o.dev;
      s = o.s;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
  // stream-ordered free back into the device pool (release threshold = max)
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  ~DevBuf() { release(); }
};

template <class T>
struct DevArray {
  T* p = nullptr;
  size_t n = 0;
  void upload(const std::vector<T>& v, cudaStream_t s) {
    if (p) cudaFree(p);
    p = nullptr;
    n = v.size();
    if (n) {
      CK(cudaMalloc(reinterpret_cast<void**>(&p), n * sizeof(T)));
      CK(cudaMemcpyAsync(p, v.data(), n * sizeof(T), cudaMemcpyHostToDevice, s));
    }
  }
  ~DevArray() {
    if (p) cudaFree(p);
  }
};

// Pinned host staging (falls back to pageable memory without a device).
struct HostBuf {
  double* p = nullptr;
  size_t n = 0;
  bool pinned = false;
  HostBuf() = default;
  explicit HostBuf(size_t doubles) { alloc(doubles); }
  void alloc(size_t doubles) {
    free_();
    n = doubles;
    if (!n) return;
    if (cudaMallocHost(reinterpret_cast<void**>(&p), n * sizeof(double)) == cudaSuccess) {
      pinned = true;
    } else {
      cudaGetLastError();
      p = static_cast<double*>(std::malloc(n * sizeof(double)));
      if (!p) throw Error(kErrGeneric, "host allocation failed");
      pinned = false;
    }
  }
  void free_() {
    if (p) {
      if (pinned) cudaFreeHost(p);
      else std::free(p);
    }
    p = nullptr;
    n = 0;
  }
  HostBuf(const HostBuf&) = delete;
  HostBuf& operator=(const HostBuf&) = delete;
  HostBuf(HostBuf&& o) noexcept : p(o.p), n(o.n), pinned(o.pinned) {
    o.p = nullptr;
    o.n = 0;
  }
  HostBuf& operator=(HostBuf&& o) noexcept {
    if (this != &o) {
      free_();
      p = o.p;
      n = o.n;
      pinned = o.pinned;
      o.p = nullptr;
      o.n = 0;
    }
    return *this;
  }
  ~HostBuf() { free_(); }
};

// ---------------------------------------------------------------------------
// per-device runtime
constexpr int kOnes = 256;
struct DeviceRt {
  int dev = -1;
  cudaStream_t stream = nullptr;
  cudaStream_t upload = nullptr;  // streamed H2D of the A store, concurrent with the factor sweep
  cudaStream_t permute = nullptr; // two-chain order: transposes of streamed tiles on the SMs the sweep leaves free
  int* one = nullptr;             // pinned host 1s (kOnes): the copy engine writes them into upload counters
  bool ready = false;
};
static std::mutex g_rt_mu;
static DeviceRt g_rt[16];

static DeviceRt& runtime(int device) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    throw Error(kErrCuda, "no CUDA device available (the B200 path has no CPU fallback)");
  }
  if (device < 0 || device >= count || device >= 16)
    throw Error(kErrInvalidArgument, "device index " + std::to_string(device) + " out of range");
  std::lock_guard<std::mutex> lk(g_rt_mu);
  DeviceRt& rt = g_rt[device];
  CK(cudaSetDevice(device));
  if (!rt.ready) {
    cudaMemPool_t pool;
    CK(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thresh = UINT64_MAX;
    CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh));
    CK(cudaStreamCreateWithFlags(&rt.stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&rt.upload, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&rt.permute, cudaStreamNonBlocking));
    CK(cudaMallocHost(reinterpret_cast<void**>(&rt.one), kOnes * sizeof(int)));
    for (int i = 0; i < kOnes; ++i) rt.one[i] = 1;
    CK(static_cast<cudaError_t>(configure_kernels()));
    rt.dev = device;
    rt.ready = true;
  }
  return rt;
}

// ---------------------------------------------------------------------------
// plans: host-built dataflow task lists (plan.cpp), uploaded once per device
// and replayed through a CUDA graph per batch size.
struct GraphCache {
  struct Entry {
    cudaGraphExec_t exec = nullptr;
    BaseTable* tables = nullptr;  // device copy of the per-matrix base tables, owned here
    int* sched = nullptr;         // scheduler state: ctl[128], missing[batch x T], slots0, slots1
  };
  std::map<int, Entry> by_batch;
  Entry& get(int batch, size_t ntasks, bool poll = false, int grid = 0) {
    Entry& e = by_batch[(grid * 65536 + batch) * 2 + (poll ? 1 : 0)];
    if (!e.tables) CK(cudaMalloc(reinterpret_cast<void**>(&e.tables), sizeof(BaseTable) * batch));
    if (!e.sched) CK(cudaMalloc(reinterpret_cast<void**>(&e.sched), (128 + 256 + 2 * ntasks * batch) * sizeof(int)));
    return e;
  }
  ~GraphCache() {
    for (auto& kv : by_batch) {
      if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
      if (kv.second.tables) cudaFree(kv.second.tables);
      if (kv.second.sched) cudaFree(kv.second.sched);
    }
  }
};

struct DevPlan {
  DataflowPlan host;
  int device = -1;
  int grid = 0;
  DevArray<DTask> tasks;
  DevArray<Seg> segs;
  DevArray<Dep> deps;
  DevArray<int> sigs;
  DevArray<ZeroStrip> zero;
  DevArray<int> need, vbase, vidx, wl, init0, init1;
  DevArray<DTask> chain;
  GraphCache graphs;
  std::mutex mu;
  // reserved critical-queue workers when a launch carries more matrices than
  // get dedicated chain SMs (-1: the plan's count).  Many chains keep q0 busy
  // by themselves, and the bulk queue needs the workers more.
  int crit_batch = -1;
  int c0_prefetch = 1;  // FlowArgs::c0_prefetch
};

struct FactorPlan2 {
  FactorPlan sym;  // filled pattern + reference task counts
  std::shared_ptr<DevPlan> flow;
  Layout L;
  int bp = 0, nb = 0;
};

struct Phase2Plan {
  Closure sel;
  std::shared_ptr<DevPlan> flow;
  int bp = 0, nb = 0;
};

constexpr int kDeferW = 2;  // phase-1 W tasks of column j are emitted with column j + 2 (bulk filler)

static int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e && *e ? std::atoi(e) : dflt;
}
// Streamed uploads overlap copies on one stream with the persistent sweep on
// another, the sweep polling for the copies.  A profiler that serialises the
// device's work (Nsight Compute: its injection leaves NV_COMPUTE_PROFILER_* /
// NV_NSIGHT_INJECTION_* in the environment) would hold the copies behind the
// sweep and stall it until the watchdog fires: then (and with
// TIB_STREAM_UPLOAD=0) A goes up before the sweep.
static bool streaming_allowed() {
  if (env_int("TIB_STREAM_UPLOAD", 1) == 0) return false;
  for (const char* v : {"CUDA_INJECTION64_PATH", "NV_COMPUTE_PROFILER_PERFWORKS_DIR", "NV_NSIGHT_INJECTION_TRANSPORT_TYPE"}) {
    const char* e = std::getenv(v);
    if (e && *e) return false;
  }
  return true;
}
// CTAs reserved for the critical queue: the factor sweep's q0 (the chain's
// helpers) is heavy and latency-sensitive, phase 2's (diagonal parts) is light
static int crit_workers(bool factor) {
  const int all = env_int("TIB_CRIT_WORKERS", 0);
  if (all > 0) return all;
  return factor ? env_int("TIB_CRIT_WORKERS_FACTOR", 56) : env_int("TIB_CRIT_WORKERS_P2", 12);
}
static int crit_workers_batch(bool factor) {
  return factor ? env_int("TIB_CRIT_BATCH_FACTOR", 32) : env_int("TIB_CRIT_BATCH_P2", 40);
}

static std::shared_ptr<DevPlan> upload_plan(DataflowPlan&& host, int device, cudaStream_t s) {
  auto d = std::make_shared<DevPlan>();
  d->host = std::move(host);
  d->device = device;
  d->grid = dataflow_grid(device);
  if (kWorkers * d->grid <= d->host.q0.workers) throw Error(kErrCuda, "persistent grid too small for the critical queue");
  // test hook: one task of the plan can never become ready, so the sweep
  // stalls and must end through the executor's watchdog (tests/test_gpu_parity.py)
  if (env_int("TIB_TEST_STALL", 0) && !d->host.need.empty()) d->host.need.back() += 1;
  d->tasks.upload(d->host.tasks, s);
  d->segs.upload(d->host.segs, s);
  d->deps.upload(d->host.deps, s);
  d->sigs.upload(d->host.sigs, s);
  d->zero.upload(d->host.zero, s);
  d->need.upload(d->host.need, s);
  d->vbase.upload(d->host.vbase, s);
  d->vidx.upload(d->host.vidx, s);
  d->wl.upload(d->host.wl, s);
  d->init0.upload(d->host.init0, s);
  d->init1.upload(d->host.init1, s);
  d->chain.upload(d->host.chain, s);
  CK(cudaStreamSynchronize(s));
  return d;
}

// plan caches (keyed by layout + pattern tiles [+ closure tiles])
static uint64_t pattern_hash(const Pattern& p, uint64_t seed) {
  Fnv h;
  h.h ^= seed;
  const Layout& L = p.layout();
  h.mix(&L.n, sizeof(L.n));
  h.mix(&L.b, sizeof(L.b));
  for (const Coord& c : p.tiles()) h.mix(&c, sizeof(c));
  return h.h;
}
static std::mutex g_plan_mu;
static std::map<std::pair<int, uint64_t>, std::shared_ptr<FactorPlan2>> g_fplans;
static std::map<std::pair<int, uint64_t>, std::shared_ptr<Phase2Plan>> g_p2plans;

// Update work per elimination step relative to the chain: (tiles per column)^2
// x (blocks per tile)^2.  Above TIB_SPLIT_WORK the sweeps are throughput bound
// even with one chain (Kronecker), below it a single chain bounds them.
static double chain_work(const Pattern& F) {
  const int N = F.layout().N;
  const double per_col = static_cast<double>(F.size() - static_cast<size_t>(N)) / N;
  const double nbk = static_cast<double>((F.layout().b + 63) / 64);
  return per_col * per_col * nbk * nbk;
}

// batch > 4 (chains share their SMs): no chain task.  A batch is throughput
// bound; a chain task would tie one worker per matrix for the whole sweep
// (64 x 157 ms at config 5, ~11 % of it computing) and its fat steps wait in
// the second phase for a backlogged bulk queue.  Plain leaves (no fat part,
// no boundary trick) are ordinary tasks that never wait inside.
// Only launches of many matrices: with fewer in flight (the host batch's
// pipelined groups of 16) each matrix's chain of leaf tasks, every step a trip
// through the queues, becomes the bound (groups of 16: 447 -> 475 ms e2e).
static bool batch_leaves(int batch) {
  return batch >= env_int("TIB_BATCH_LEAVES_MIN", 32) && env_int("TIB_BATCH_CHAIN", 0) == 0;
}

// Bulk update terms per factor task (build_factor_dataflow's ugroup): four
// terms to a multi-segment GEMM (K = 4 bp), except in a single natural-order
// chain that bounds its sweep (each term as early as its column: large
// natural order 93.8 vs 95.6 ms grouped).  tools/ab_env.py, one B200: factor
// sweep large 85.8 -> 81.1 ms, Kronecker 248 -> 229, batch 131.5 -> 113.9,
// medium 29.0 -> 27.5 (flat from 4 to 16 terms).
static int factor_update_group(const Pattern& F, int batch, int split) {
  const int forced = env_int("TIB_UPD_GROUP", 0);
  if (forced > 0) return std::min(forced, 16);  // two signals per term, <= 32 per task
  const bool chain_bound = split <= 0 && !batch_leaves(batch) && chain_work(F) <= env_int("TIB_SPLIT_WORK", 3000);
  return chain_bound ? 1 : 4;
}

static std::shared_ptr<FactorPlan2> factor_plan_for(const Pattern& pattern, int device, cudaStream_t s,
                                                    int split = -1, int batch = 1) {
  const bool leaves = batch_leaves(batch);
  // (the grouping is a function of the filled pattern, batch and split; only a
  // forced TIB_UPD_GROUP needs to be in the key)
  const uint64_t key = pattern_hash(pattern, 1 + 0x9e3779b97f4a7c15ull * static_cast<uint64_t>(split + 2) +
                                                 (leaves ? 0x51ed27ull : 0) +
                                                 0x2545f491ull * static_cast<uint64_t>(env_int("TIB_UPD_GROUP", 0)));
  {
    std::lock_guard<std::mutex> lk(g_plan_mu);
    auto it = g_fplans.find({device, key});
    if (it != g_fplans.end() && it->second->L.n == pattern.layout().n) return it->second;
  }
  auto plan = std::make_shared<FactorPlan2>();
  plan->sym = symbolic_cholesky(pattern);
  plan->L = plan->sym.filled.layout();
  const int ug = factor_update_group(plan->sym.filled, batch, split);
  // two chains keep the critical queue busier per reserved worker (tools/ab_env.py: 24 / 12 best with
  // grouped updates, profiles/r02_s4_ab_crit.log);
  // a throughput-bound single chain (chain work above TIB_SPLIT_WORK: Kronecker) needs few
  // (Kronecker factor sweep 276 -> 248 ms at 8)
  const bool tput = chain_work(plan->sym.filled) > env_int("TIB_SPLIT_WORK", 3000);
  const int crit = split > 0 ? env_int("TIB_CRIT_SPLIT_FACTOR", 24)
                             : (tput ? env_int("TIB_CRIT_TPUT_FACTOR", 8) : crit_workers(true));
  // the device sweep: chain task, fat leaves and the tile-boundary trick, or
  // (batches) plain leaf tasks -- the two configurations the executor is tested with
  plan->flow = upload_plan(leaves ? build_factor_dataflow(plan->sym.filled, crit, kDeferW, false, false, false, split,
                                                          false, ug)
                                  : build_factor_dataflow(plan->sym.filled, crit, kDeferW, true, true, true, split,
                                                          env_int("TIB_COARSE_SECOND", 1) != 0, ug),
                           device, s);
  // reserved critical workers of launches without dedicated chain SMs: more
  // for leaf tasks (the whole chain goes through the critical queue)
  plan->flow->crit_batch = leaves ? crit_workers_batch(true) : env_int("TIB_CRIT_BATCH_CHAINS", 8);
  plan->flow->c0_prefetch = env_int("TIB_C0_PF_FACTOR", 1);
  plan->bp = plan->flow->host.bp;
  plan->nb = plan->flow->host.nb;
  std::lock_guard<std::mutex> lk(g_plan_mu);
  if (g_fplans.size() > 8) g_fplans.clear();
  g_fplans[{device, key}] = plan;
  return plan;
}

// Late terms per phase-2 split-K part.  Batches, and the two-chain order with
// large tiles (>= 8 blocks), run a throughput-bound phase 2, where fewer,
// larger parts win (two-chain large 101.3 -> 99.8 ms, batch 137 -> 128 ms at
// 3); a single chain is latency-bound there (natural-order large 101.8 ->
// 117.5 ms, two-chain medium 17 -> 27 ms at 3), so one term per part.
static int phase2_group(const Pattern& F, int batch, int split) {
  const int forced = env_int("TIB_P2_GROUP", 0);
  if (forced > 0) return forced;
  const int nb = (F.layout().b + 63) / 64;
  // launches of many matrices: 8 (batch config 125.6 -> 120.9 ms; 6: 121.3, 12: 121.5)
  if (batch_leaves(batch)) return 8;
  const bool throughput = batch > 4 || (split > 0 && nb >= 8) || chain_work(F) > env_int("TIB_SPLIT_WORK", 3000);
  return throughput ? 3 : 1;
}

// Reserved critical workers of a two-chain phase-2 plan: a throughput-bound
// phase 2 (late terms grouped) needs few (large: 8 vs 12, 97.9 vs 98.2 ms), a
// chain-bound one more (medium: 32 vs 24, 16.4 vs 16.9 ms; profiles/r02_s4_ab_knobs.log).
static int crit_split_p2(const Pattern& F, int split) {
  return env_int("TIB_CRIT_SPLIT_P2", phase2_group(F, 1, split) > 1 ? 8 : 32);
}

static std::shared_ptr<Phase2Plan> phase2_plan_for(const Pattern& F, const Closure& sel, int device,
                                                   cudaStream_t s, int crit = -1, int split = -1, int batch = 1) {
  if (crit < 0)
    crit = chain_work(F) > env_int("TIB_SPLIT_WORK", 3000) ? env_int("TIB_CRIT_TPUT_P2", 6) : crit_workers(false);
  const int group = phase2_group(F, batch, split);
  const uint64_t key = pattern_hash(
      sel.closure, pattern_hash(F, 2 + 7919ull * static_cast<uint64_t>(crit) + 104729ull * static_cast<uint64_t>(split + 2) +
                                       1299709ull * static_cast<uint64_t>(group)));
  {
    std::lock_guard<std::mutex> lk(g_plan_mu);
    auto it = g_p2plans.find({device, key});
    if (it != g_p2plans.end()) return it->second;
  }
  auto plan = std::make_shared<Phase2Plan>();
  plan->sel = sel;
  plan->flow = upload_plan(build_phase2_dataflow(F, plan->sel, crit, split, group), device, s);
  plan->flow->crit_batch = crit_workers_batch(false);
  plan->flow->c0_prefetch = env_int("TIB_C0_PF_P2", 1);
  plan->bp = plan->flow->host.bp;
  plan->nb = plan->flow->host.nb;
  std::lock_guard<std::mutex> lk(g_plan_mu);
  if (g_p2plans.size() > 16) g_p2plans.clear();
  g_p2plans[{device, key}] = plan;
  return plan;
}

static std::map<std::pair<int, uint64_t>, std::shared_ptr<DevPlan>> g_p1plans;
static std::shared_ptr<DevPlan> phase1_plan_for(const Pattern& F, int device, cudaStream_t s) {
  const uint64_t key = pattern_hash(F, 3);
  {
    std::lock_guard<std::mutex> lk(g_plan_mu);
    auto it = g_p1plans.find({device, key});
    if (it != g_p1plans.end()) return it->second;
  }
  auto plan = upload_plan(build_phase1_dataflow(F), device, s);
  std::lock_guard<std::mutex> lk(g_plan_mu);
  if (g_p1plans.size() > 8) g_p1plans.clear();
  g_p1plans[{device, key}] = plan;
  return plan;
}

// ---------------------------------------------------------------------------
// sweeps
static bool use_graphs() {
  const char* e = std::getenv("TIB_GRAPH");
  return !(e && e[0] == '0');
}

// Task trace (TIB_TRACE=<prefix>): per executed task claim / ready / done
// globaltimer stamps + (task, matrix, SM), written to <prefix>.<n>.bin
// together with the plan's task kinds; tools/trace_report.py reads them.
static const char* trace_prefix() {
  const char* e = std::getenv("TIB_TRACE");
  return e && *e ? e : nullptr;
}
static std::atomic<int> g_trace_seq{0};

static void write_trace(DevPlan& P, int batch, unsigned long long* d_trace, cudaStream_t s) {
  const size_t n = (P.host.tasks.size() + 2 * P.host.chain.size()) * batch * 4;  // tasks, chain steps (worker 0, worker 1)
  std::vector<unsigned long long> h(n);
  CK(cudaMemcpyAsync(h.data(), d_trace, n * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const std::string path = std::string(trace_prefix()) + "." + std::to_string(g_trace_seq++) + ".bin";
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) return;
  // v2: header, then the raw plan (tasks, deps, sigs, segs) so tools/trace_report.py
  // can rebuild every dependency edge and walk the critical path
  const long long hdr[11] = {-4,
                            static_cast<long long>(P.host.tasks.size()),
                            batch,
                            P.host.q0.count,
                            P.host.nb,
                            static_cast<long long>(P.host.deps.size()),
                            static_cast<long long>(P.host.sigs.size()),
                            static_cast<long long>(P.host.segs.size()),
                            static_cast<long long>(P.host.slot_tiles.size()),
                            P.host.bp,
                            static_cast<long long>(P.host.chain.size())};
  std::fwrite(hdr, sizeof(hdr), 1, f);
  std::fwrite(P.host.tasks.data(), sizeof(DTask), P.host.tasks.size(), f);
  std::fwrite(P.host.deps.data(), sizeof(Dep), P.host.deps.size(), f);
  std::fwrite(P.host.sigs.data(), sizeof(int), P.host.sigs.size(), f);
  std::fwrite(P.host.segs.data(), sizeof(Seg), P.host.segs.size(), f);
  std::fwrite(P.host.slot_tiles.data(), sizeof(Coord), P.host.slot_tiles.size(), f);
  std::fwrite(P.host.chain.data(), sizeof(DTask), P.host.chain.size(), f);
  std::fwrite(h.data(), 8, n, f);
  std::fclose(f);
}

// Uploads the base tables into the plan-owned buffer, zeroes each matrix's
// dependency counters and runs the persistent sweep (captured once per batch
// size into a CUDA graph; its only baked-in pointers are plan-owned).
// pre_launch (streamed upload): issued after the counters are cleared and
// before the sweep kernel; tasks then poll their A-store column's counter.
// Chain tasks of a plan: the leading queue-0 tasks of kind kChainTask, each
// initially ready (they are the first items of init0).
static int chains_of(const DevPlan& P) {
  int c = 0;
  while (c < static_cast<int>(P.host.tasks.size()) && c < static_cast<int>(P.host.init0.size()) &&
         P.host.tasks[static_cast<size_t>(c)].kind == kChainTask && P.host.init0[static_cast<size_t>(c)] == c)
    ++c;
  return c;
}

// grid > 0: launch that many persistent CTAs instead of one per SM (the
// two-chain streamed upload leaves SMs free for its transposes).
// Streamed two-chain upload: the in-kernel transpose agents' work lists.
struct TransposeAgents {
  int agents = 0, ncols = 0, bp = 0;
  const int* cols = nullptr;
  const int* off = nullptr;
  const int* dst = nullptr;
  const int* src = nullptr;
  const unsigned char* tr = nullptr;
  long long raw = 0, upl = 0, arrive = 0;
};

static void run_flow(DevPlan& P, const std::vector<BaseTable>& tables, cudaStream_t s,
                     const std::function<void()>* pre_launch = nullptr, cudaEvent_t cleared = nullptr, int grid = 0,
                     const TransposeAgents* ta = nullptr) {
  std::lock_guard<std::mutex> lk(P.mu);
  const int batch = static_cast<int>(tables.size());
  const size_t nt = P.host.tasks.size();
  const bool poll = pre_launch != nullptr;
  if (grid <= 0 || grid > P.grid) grid = P.grid;
  GraphCache::Entry& e = P.graphs.get(batch, nt, poll, ta ? 1 : (grid == P.grid ? 0 : grid));
  CK(cudaMemcpyAsync(e.tables, tables.data(), sizeof(BaseTable) * batch, cudaMemcpyHostToDevice, s));
  for (const BaseTable& t : tables)
    CK(cudaMemsetAsync(t.p[kStoreCounters], 0, static_cast<size_t>(P.host.counters) * sizeof(int), s));
  if (cleared) CK(cudaEventRecord(cleared, s));  // the copy stream's counter writes come after this
  // streamed upload: the copies are enqueued on the copy stream once the sweep
  // is launched (its tasks poll the column counters), so the host's issue of
  // thousands of copies overlaps the sweep instead of delaying its launch
  auto launched = [&]() {
    if (pre_launch) (*pre_launch)();
  };
  FlowArgs a{};
  a.tasks = P.tasks.p;
  a.segs = P.segs.p;
  a.deps = P.deps.p;
  a.sigs = P.sigs.p;
  a.vbase = P.vbase.p;
  a.vidx = P.vidx.p;
  a.wl = P.wl.p;
  a.q0 = P.host.q0;
  a.q1 = P.host.q1;
  a.batch = batch;
  a.ntasks = static_cast<int>(nt);
  a.tables = e.tables;
  a.ctl = e.sched;
  a.missing = e.sched + 128 + 256;  // (ctl lines, 256 spare ints, then the per-task counts)
  a.chain = P.chain.p;
  const int nchains = chains_of(P);
  a.dedicate = batch * std::max(nchains, 1) <= env_int("TIB_DEDICATE_MAX_BATCH", 4) ? 1 : 0;
  a.static_chains = nchains > 0 && batch * nchains <= grid ? nchains : 0;
  // the chains' workers are reserved ones (worker 0 of the first CTAs): keep
  // the plan's count of reserved workers for the chain's helpers
  if (!a.dedicate && P.crit_batch >= 0 && a.q0.workers > 0) a.q0.workers = P.crit_batch;
  a.q0.workers += batch * a.static_chains;
  a.poll_shift = env_int("TIB_POLL_SHIFT", 0);
  a.agent = a.dedicate && a.static_chains && env_int("TIB_AGENT", 1) ? 1 : 0;
  a.poll_uploads = poll ? 1 : 0;
  a.c0_prefetch = P.c0_prefetch;
  // early q1 tickets: launches of many matrices only (batch 236.1 -> 234.4 ms;
  // large within noise, chain-bound medium 41.7 -> 43.4: a held ticket delays the
  // critical item that lands in its slot)
  a.early_ticket = env_int("TIB_EARLY_TICKET", batch_leaves(batch) ? 1 : 0);
  a.watchdog_ns = static_cast<unsigned long long>(env_int("TIB_WATCHDOG_S", 60)) * 1000000000ull;
  if (ta && batch == 1) {
    a.t_agents = ta->agents;
    a.t_ncols = ta->ncols;
    a.t_bp = ta->bp;
    a.t_cols = ta->cols;
    a.t_off = ta->off;
    a.t_dst = ta->dst;
    a.t_src = ta->src;
    a.t_tr = ta->tr;
    a.t_raw = ta->raw;
    a.t_upl = ta->upl;
    a.t_arrive = ta->arrive;
  }
  a.slots0 = a.missing + nt * batch;
  a.slots1 = a.slots0 + static_cast<size_t>(P.host.q0.count) * batch;
  a.trace = nullptr;
  auto enqueue = [&]() {
    launch_zero_strips(P.zero.p, static_cast<int>(P.zero.n), P.host.bp, batch, e.tables, s);
    launch_dataflow(a, P.need.p, P.init0.p, static_cast<int>(P.init0.n), P.init1.p, static_cast<int>(P.init1.n), grid, s);
  };
  if (std::getenv("TIB_CHAIN_PROF") && set_chain_profile(nullptr) == cudaSuccess) {
    // phases: 0 leaf (10 chol32 A00, 11 coupling DMMA, 12 chol32 A11, 13 X10 DMMA, rest: logdet + stores),
    // 5 phase-1 signals, 6 second-phase wait + operand prefetch issue, 7 fat part, 8 phase-2 signals,
    // 9 step dependency wait
    long long* prof = nullptr;
    CK(cudaMalloc(reinterpret_cast<void**>(&prof), 16 * sizeof(long long)));
    CK(cudaMemsetAsync(prof, 0, 16 * sizeof(long long), s));
    CK(static_cast<cudaError_t>(set_chain_profile(prof)));
    enqueue();
    CK(cudaGetLastError());
    launched();
    long long h[16];
    CK(cudaMemcpyAsync(h, prof, sizeof(h), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    CK(static_cast<cudaError_t>(set_chain_profile(nullptr)));
    cudaFree(prof);
    const double n = static_cast<double>(std::max<size_t>(P.host.chain.size(), 1)) * batch;
    std::fprintf(stderr, "chain profile (cycles per step):");
    for (int i = 0; i < 16; ++i) std::fprintf(stderr, " p%d=%.0f", i, h[i] / n);
    std::fprintf(stderr, "\n");
    return;
  }
  if (trace_prefix()) {
    unsigned long long* d_trace = nullptr;
    const size_t n = (nt + 2 * P.host.chain.size()) * batch * 4;
    CK(cudaMallocAsync(reinterpret_cast<void**>(&d_trace), n * 8, s));
    CK(cudaMemsetAsync(d_trace, 0, n * 8, s));
    a.trace = d_trace;
    enqueue();
    CK(cudaGetLastError());
    launched();
    write_trace(P, batch, d_trace, s);
    CK(cudaFreeAsync(d_trace, s));
    return;
  }
  if (!use_graphs() || ta) {  // (the agents' work lists are per call: no cached graph)
    enqueue();
    CK(cudaGetLastError());
    launched();
    return;
  }
  if (!e.exec) {
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    enqueue();
    const cudaError_t le = cudaGetLastError();
    CK(cudaStreamEndCapture(s, &g));
    CK(le);
    CK(cudaGraphInstantiate(&e.exec, g, 0));
    cudaGraphDestroy(g);
  }
  CK(cudaGraphLaunch(e.exec, s));
  launched();
}

// Largest batch one launch may carry: every chain needs its own CTA (static
// chain assignment, worker 0 of CTA m runs matrix m's chain) and queue items
// pack (matrix, task) into a non-negative int.  Bigger batches run as several
// launches of the same plan.
static size_t max_batch(const DevPlan& P) {
  const size_t by_items = static_cast<size_t>(INT_MAX) / std::max<size_t>(P.host.tasks.size(), 1);
  const size_t by_chains =
      P.host.chain.empty() ? by_items : static_cast<size_t>(P.grid) / static_cast<size_t>(std::max(chains_of(P), 1));
  return std::max<size_t>(1, std::min(by_items, by_chains));
}

static void run_flow_chunked(DevPlan& P, const std::vector<BaseTable>& tables, cudaStream_t s,
                             const std::function<void()>* pre_launch = nullptr, cudaEvent_t cleared = nullptr,
                             int grid = 0, const TransposeAgents* ta = nullptr) {
  const size_t mb = max_batch(P);
  if (tables.size() <= mb) {
    run_flow(P, tables, s, pre_launch, cleared, grid, ta);
    return;
  }
  if (pre_launch) throw Error(kErrInvalidArgument, "streamed upload is single-launch only");
  for (size_t i = 0; i < tables.size(); i += mb) {
    const std::vector<BaseTable> part(tables.begin() + static_cast<long>(i),
                                      tables.begin() + static_cast<long>(std::min(tables.size(), i + mb)));
    run_flow(P, part, s);
  }
}

// TIB_HOST_TIMING=1: wall-clock phase marks of a public call on stderr (each
// mark synchronises the stream, so only for diagnosis).
struct HostTimer {
  bool on;
  cudaStream_t s;
  std::chrono::steady_clock::time_point t0, last;
  explicit HostTimer(cudaStream_t st) : on(env_int("TIB_HOST_TIMING", 0) != 0), s(st) {
    t0 = last = std::chrono::steady_clock::now();
  }
  void mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[tib timing] %-28s %9.3f ms (total %9.3f)\n", what,
                 std::chrono::duration<double, std::milli>(now - last).count(),
                 std::chrono::duration<double, std::milli>(now - t0).count());
    last = now;
  }
};

// ---------------------------------------------------------------------------
// objects behind the handles
struct MatrixObj {
  Layout layout;
  Pattern pattern;
  mutable HostBuf payload;  // pattern.size() * b * b, pinned when a device exists
  // device-generated matrix (tib_matrix_generate_device): the values are made
  // on the device straight into each sweep's A store; the host payload is
  // materialised (from the device) only when a host-side API asks for it
  struct DevGen {
    bool on = false;
    long n = 0, w = 0, t = 0;
    uint64_t seed = 0;
    int device = 0;
  } gen;
};

// Generator on the device (generate.cu) into a tile store over `pat` with row
// stride bp (identity padding), stream-ordered.
// A batch of device-generated matrices with the same parameters but their own
// seeds (ms[k]'s store at out + k * stride) is one launch per kernel.
static void device_generate(const std::vector<const MatrixObj*>& ms, const Pattern& pat, int bp, double* out,
                            size_t stride, cudaStream_t s) {
  const MatrixObj& m = *ms[0];
  const int N = pat.layout().N;
  std::vector<int> meta(static_cast<size_t>(N) + 1 + pat.size());  // colptr (N + 1), then rows
  int maxc = 0;
  for (int j = 0; j <= N; ++j) meta[static_cast<size_t>(j)] = static_cast<int>(pat.col_start(j));
  for (int j = 0; j < N; ++j) maxc = std::max(maxc, static_cast<int>(pat.col_start(j + 1) - pat.col_start(j)));
  for (size_t k = 0; k < pat.size(); ++k) meta[static_cast<size_t>(N) + 1 + k] = pat.tiles()[k].i;
  std::vector<unsigned long long> seeds;
  for (const MatrixObj* x : ms) seeds.push_back(x->gen.seed);
  int* d_meta = nullptr;
  unsigned long long* d_seeds = nullptr;
  CK(cudaMallocAsync(reinterpret_cast<void**>(&d_meta), meta.size() * sizeof(int), s));
  CK(cudaMallocAsync(reinterpret_cast<void**>(&d_seeds), seeds.size() * sizeof(unsigned long long), s));
  CK(cudaMemcpyAsync(d_meta, meta.data(), meta.size() * sizeof(int), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(d_seeds, seeds.data(), seeds.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice, s));
  CK(static_cast<cudaError_t>(launch_generate_arrowhead(m.gen.n, m.gen.w, m.gen.t, m.gen.seed, m.layout.b, bp, N,
                                                        d_meta, d_meta + N + 1, maxc, out, s, d_seeds,
                                                        static_cast<int>(ms.size()), static_cast<long long>(stride))));
  CK(cudaFreeAsync(d_meta, s));
  CK(cudaFreeAsync(d_seeds, s));
  CK(cudaStreamSynchronize(s));  // the host vectors above die with this scope
}
static void device_generate(const MatrixObj& m, const Pattern& pat, int bp, double* out, cudaStream_t s) {
  device_generate(std::vector<const MatrixObj*>{&m}, pat, bp, out, 0, s);
}

static DeviceRt& runtime(int device);

// Host payload of m (materialised from the device generator on first use).
static const double* host_payload(const MatrixObj& m) {
  if (m.gen.on && m.payload.n == 0) {
    DeviceRt& rt = runtime(m.gen.device);
    const size_t bb = static_cast<size_t>(m.layout.b) * m.layout.b;
    DevBuf d(m.pattern.size() * bb, m.gen.device, rt.stream);
    device_generate(m, m.pattern, m.layout.b, d.p, rt.stream);
    m.payload.alloc(d.n);
    CK(cudaMemcpyAsync(m.payload.p, d.p, d.n * sizeof(double), cudaMemcpyDeviceToHost, rt.stream));
    CK(cudaStreamSynchronize(rt.stream));
  }
  return m.payload.p;
}

// Host payload of m in the two-chain order, bp-layout tiles over so.permuted
// (identity on the padded diagonal, zero fill-in): permuted tile (i, j) is
// original tile (order[i], order[j]), or the transpose of (order[j], order[i]).
static void permuted_payload(const MatrixObj& m, const SplitOrder& so, int bp, double* out) {
  const int b = m.layout.b;
  const double* src = host_payload(m);
  const size_t bb = static_cast<size_t>(b) * b, bpp = static_cast<size_t>(bp) * bp;
  const Pattern& P = so.permuted;
  for (size_t k = 0; k < P.size(); ++k) {
    const Coord& c = P.tiles()[k];
    double* dst = out + k * bpp;
    std::memset(dst, 0, bpp * sizeof(double));
    bool tr = false;
    const Coord o = split_source(so, c.i, c.j, tr);
    const long sl = m.pattern.slot(o.i, o.j);
    if (sl >= 0) {
      const double* t = src + static_cast<size_t>(sl) * bb;
      if (!tr) {
        for (int r = 0; r < b; ++r) std::memcpy(dst + static_cast<size_t>(r) * bp, t + static_cast<size_t>(r) * b, b * sizeof(double));
      } else {
        for (int r = 0; r < b; ++r)
          for (int q = 0; q < b; ++q) dst[static_cast<size_t>(r) * bp + q] = t[static_cast<size_t>(q) * b + r];
      }
    }
    if (c.i == c.j)
      for (int r = b; r < bp; ++r) dst[static_cast<size_t>(r) * bp + r] = 1.0;
  }
}

// TiledFactor (storage.hpp:46-51), device resident.  has_L: the factor tiles L
// are held (PhaseTag kFactor -- factorize, or a kFactor tile file); without,
// only the phase-1 tiles (a kPhase1 tile file: U_j = X_j^T and W_kj).
struct FactorObj {
  int device = 0;
  Layout layout;
  Pattern F;  // the factor's (filled) tile pattern
  int bp = 0, nb = 0;
  bool has_L = true;
  DevBuf L, P1;
  double logdet = 0;
};

struct Unpermute;
struct SigmaObj {
  int device = 0;
  Layout layout;
  Request req;
  std::shared_ptr<Phase2Plan> plan;
  DevBuf S, var;
  double logdet = 0;
  std::unique_ptr<HostBuf> host;  // lazily downloaded bp-layout tiles
  // two-chain order: Sigma and the variances stay in the permuted order (Sp,
  // var); S is un-permuted on the device the first time a whole-store
  // accessor needs it, entries and the diagonal are mapped directly
  std::shared_ptr<const Unpermute> unperm;
  DevBuf Sp;
};

static void fill_matrix(MatrixObj& m, HostMatrix&& hm) {
  m.layout = hm.layout;
  m.pattern = std::move(hm.pattern);
  m.payload.alloc(hm.payload.size());
  std::memcpy(m.payload.p, hm.payload.data(), hm.payload.size() * sizeof(double));
}

// Host matrix -> bp-layout A store over the FILLED pattern (fill-in tiles zero,
// identity on the padded diagonal).
// Uploads the filled-pattern slots of tile columns [c0, c1) of m (b = bp): runs
// of slots present in m's pattern with consecutive host slots are one H2D
// copy (copies = true), runs of fill-in slots one memset (zeros = true) -- no
// host staging.  A streamed upload issues the memsets on the sweep stream
// before the sweep: a memset is a kernel and cannot start while the persistent
// sweep holds every SM, so on the copy stream it would stall the copies behind it.
static void upload_columns(const MatrixObj& m, const Pattern& F, int c0, int c1, double* dA, cudaStream_t s,
                           bool copies = true, bool zeros = true) {
  const size_t bb = static_cast<size_t>(m.layout.b) * m.layout.b;
  long k = F.col_start(c0);
  const long kend = F.col_start(c1);
  while (k < kend) {
    const long src = m.pattern.slot(F.tiles()[static_cast<size_t>(k)].i, F.tiles()[static_cast<size_t>(k)].j);
    long e = k + 1;
    if (src >= 0) {
      while (e < kend && m.pattern.slot(F.tiles()[static_cast<size_t>(e)].i, F.tiles()[static_cast<size_t>(e)].j) ==
                             src + (e - k))
        ++e;
      if (copies)
        CK(cudaMemcpyAsync(dA + static_cast<size_t>(k) * bb, m.payload.p + static_cast<size_t>(src) * bb,
                           static_cast<size_t>(e - k) * bb * sizeof(double), cudaMemcpyHostToDevice, s));
    } else {
      while (e < kend && m.pattern.slot(F.tiles()[static_cast<size_t>(e)].i, F.tiles()[static_cast<size_t>(e)].j) < 0)
        ++e;
      if (zeros)
        CK(cudaMemsetAsync(dA + static_cast<size_t>(k) * bb, 0, static_cast<size_t>(e - k) * bb * sizeof(double), s));
    }
    k = e;
  }
}

static void upload_matrix(const MatrixObj& m, const Pattern& filled, int bp, double* dA, cudaStream_t s,
                          HostBuf* staging_keep = nullptr) {
  if (m.gen.on) {  // no host values: generate in place
    device_generate(m, filled, bp, dA, s);
    return;
  }
  const int b = m.layout.b;
  const size_t bb = static_cast<size_t>(b) * b, bpp = static_cast<size_t>(bp) * bp;
  if (bp == b && filled == m.pattern) {
    CK(cudaMemcpyAsync(dA, m.payload.p, filled.size() * bb * sizeof(double), cudaMemcpyHostToDevice, s));
    return;
  }
  if (bp == b && m.payload.pinned) {
    upload_columns(m, filled, 0, m.layout.N, dA, s);
    CK(cudaStreamSynchronize(s));
    return;
  }
  HostBuf local;
  HostBuf& st = staging_keep ? *staging_keep : local;
  st.alloc(filled.size() * bpp);
  std::memset(st.p, 0, st.n * sizeof(double));
  for (size_t k = 0; k < filled.size(); ++k) {
    const Coord& c = filled.tiles()[k];
    double* dst = st.p + k * bpp;
    const long src = m.pattern.slot(c.i, c.j);
    if (src >= 0)
      for (int r = 0; r < b; ++r)
        std::memcpy(dst + static_cast<size_t>(r) * bp, m.payload.p + static_cast<size_t>(src) * bb + static_cast<size_t>(r) * b,
                    b * sizeof(double));
    if (c.i == c.j)
      for (int r = b; r < bp; ++r) dst[static_cast<size_t>(r) * bp + r] = 1.0;
  }
  CK(cudaMemcpyAsync(dA, st.p, st.n * sizeof(double), cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));
}

struct SweepStores {
  DevBuf A, L, P1, scratch, logdet, counters;
  size_t scratch_stride = 0;  // doubles of scratch per matrix
  DevBuf status;  // DevStatus per matrix (as doubles storage)
  long cstride = 0;  // ints of counters per matrix
  double* ctr(int k) const { return reinterpret_cast<double*>(reinterpret_cast<int*>(counters.p) + cstride * k); }
};

static DevBuf alloc_counters(long per_matrix, int batch, int dev, cudaStream_t s) {
  return DevBuf((static_cast<size_t>(per_matrix) * batch + 1) / 2, dev, s);
}

static void alloc_factor_stores(SweepStores& st, const FactorPlan2& P, int batch, int dev, cudaStream_t s,
                                long min_counters = 0, size_t min_scratch = 0) {
  const size_t tile = static_cast<size_t>(P.bp) * P.bp;
  const size_t T = P.sym.filled.size();
  st.A = DevBuf(T * tile * batch, dev, s);
  st.L = DevBuf(T * tile * batch, dev, s);
  st.P1 = DevBuf(T * tile * batch, dev, s);
  st.scratch_stride = std::max(P.flow->host.scratch_doubles, min_scratch);
  st.scratch = DevBuf(st.scratch_stride * batch, dev, s);
  st.logdet = DevBuf(P.flow->host.logdet_doubles * batch, dev, s);
  st.cstride = std::max<long>(P.flow->host.counters, min_counters);
  st.counters = alloc_counters(st.cstride, batch, dev, s);
  st.status = DevBuf(static_cast<size_t>(batch), dev, s);
}

// After a stream sync: a sweep that hit the executor's watchdog (kernels.cu
// Spin) raises TIB_ERR_CUDA with the dependency it gave up on.
static void check_watchdog() {
  int rec[4] = {0, 0, 0, 0};
  CK(static_cast<cudaError_t>(read_watchdog(rec)));
  if (rec[0])
    throw Error(kErrCuda, "dataflow watchdog: a sweep waited longer than TIB_WATCHDOG_S on counter " +
                              std::to_string(rec[1]) + " >= " + std::to_string(rec[2]) + " (dependency " +
                              std::to_string(rec[3]) + "); results discarded");
}

static void check_status(const DevBuf& status, int batch, const Layout& L, cudaStream_t s, int* bad_index = nullptr) {
  std::vector<unsigned long long> h(static_cast<size_t>(batch));
  CK(cudaMemcpyAsync(h.data(), status.p, batch * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  check_watchdog();
  for (int k = 0; k < batch; ++k)
    if (h[static_cast<size_t>(k)] != ULLONG_MAX) {
      const long pivot = static_cast<long>(h[static_cast<size_t>(k)]);
      const int tile = static_cast<int>(pivot / L.b);
      if (bad_index) *bad_index = k;
      throw NotSpd("matrix is not positive definite", pivot, tile, tile);
    }
}

static double reduce_logdet(const double* parts, int N, int nb) {
  double s = 0.0;
  for (int j = 0; j < N; ++j)
    for (int k = 0; k < nb; ++k) s += parts[static_cast<size_t>(j) * nb + k];
  return 2.0 * s;
}

// Runs the fused factor sweep for the matrices already resident in their A stores.
static void factor_sweep(FactorPlan2& P, SweepStores& st, cudaStream_t s, const std::vector<BaseTable>& tables,
                         const std::function<void()>* pre_launch = nullptr, cudaEvent_t cleared = nullptr,
                         int grid = 0, const TransposeAgents* ta = nullptr) {
  CK(cudaMemsetAsync(st.status.p, 0xff, tables.size() * sizeof(unsigned long long), s));
  run_flow_chunked(*P.flow, tables, s, pre_launch, cleared, grid, ta);
}

static void phase2_sweep(Phase2Plan& P, cudaStream_t s, const std::vector<BaseTable>& tables) {
  run_flow_chunked(*P.flow, tables, s);
}

static BaseTable make_table(double* A, double* L, double* P1, double* Sg, double* var, double* scratch,
                            double* logdet, double* status, double* counters) {
  BaseTable t{};
  t.p[kStoreA] = A;
  t.p[kStoreL] = L;
  t.p[kStoreP1] = P1;
  t.p[kStoreSigma] = Sg;
  t.p[kStoreVar] = var;
  t.p[kStoreScratch] = scratch;
  t.p[kStoreLogdet] = logdet;
  t.p[kStoreStatus] = status;
  t.p[kStoreCounters] = counters;
  return t;
}

static Request make_request(int preset, const long* rows, const long* cols, long n) {
  Request r;
  r.preset = preset;
  if (preset == kNone) {
    if (n < 0 || (n > 0 && (!rows || !cols))) throw Error(kErrInvalidArgument, "entry list pointers are null");
    r.entries.reserve(static_cast<size_t>(n));
    for (long k = 0; k < n; ++k) r.entries.push_back({rows[k], cols[k]});
  } else if (preset < 0 || preset > 3) {
    throw Error(kErrInvalidArgument, "unknown selection preset " + std::to_string(preset));
  }
  return r;
}

// ---------------------------------------------------------------------------
// Two-chain order of a single-matrix call (planner.hpp two_chain_order): the
// sweeps run on the symmetrically permuted matrix, whose factor has two
// independent elimination chains; Sigma comes back in the natural order.
struct SplitCall {
  FactorPlan natural;  // the matrix's own filled pattern
  Closure sel;         // the request's closure (== natural.filled)
  SplitOrder so;
  // per permuted slot: source slot in m.pattern (-1: fill-in), in the natural
  // filled pattern, and whether the permuted tile is the source's transpose
  std::vector<int> src, src_filled;
  std::vector<unsigned char> tr;
};

static bool split_call(const MatrixObj& m, const Request& req, SplitCall& sc) {
  if (env_int("TIB_SPLIT", 1) == 0) return false;
  sc.natural = symbolic_cholesky(m.pattern);
  const Pattern& F = sc.natural.filled;
  // chain-bound sweeps only
  if (chain_work(F) > env_int("TIB_SPLIT_WORK", 3000)) return false;
  sc.sel = symbolic_inversion(select_tiles(F.layout(), F, req), F);
  if (!(sc.sel.closure == F)) return false;  // Sigma on the whole factor pattern only
  sc.so = two_chain_order(F);
  if (sc.so.split <= 0) return false;
  const Pattern& P = sc.so.permuted;
  sc.src.resize(P.size());
  sc.src_filled.resize(P.size());
  sc.tr.resize(P.size());
  for (size_t k = 0; k < P.size(); ++k) {
    bool t = false;
    const Coord o = split_source(sc.so, P.tiles()[k].i, P.tiles()[k].j, t);
    sc.src[k] = static_cast<int>(m.pattern.slot(o.i, o.j));
    sc.src_filled[k] = static_cast<int>(F.slot(o.i, o.j));
    sc.tr[k] = t ? 1 : 0;
  }
  return true;
}

template <class T>
static DevBuf to_device(const std::vector<T>& v, int dev, cudaStream_t s) {
  DevBuf d((v.size() * sizeof(T) + 7) / 8 + 1, dev, s);
  if (!v.empty()) CK(cudaMemcpyAsync(d.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));  // the host vector may die with the caller's scope
  return d;
}

// Sigma' (permuted closure = permuted filled pattern) -> the natural closure
// store; marginal variances likewise (tile rows).  Device maps built once.
struct Unpermute {
  DevBuf d, src, tr, rd, rs;
  int count = 0, N = 0;
  std::vector<int> slot_of, pos;            // natural closure slot -> permuted slot; tile -> position
  std::vector<unsigned char> transposed;    // ... whether the permuted tile is its transpose
  Unpermute(const SplitCall& sc, int dev, cudaStream_t s) {
    const Pattern& C = sc.sel.closure;
    const Pattern& P = sc.so.permuted;
    std::vector<int> vd(C.size()), vs(C.size());
    std::vector<unsigned char> vt(C.size());
    for (size_t k = 0; k < C.size(); ++k) {
      const Coord c = C.tiles()[k];
      const int a = sc.so.pos[static_cast<size_t>(c.i)], b = sc.so.pos[static_cast<size_t>(c.j)];
      vd[k] = static_cast<int>(k);
      vs[k] = static_cast<int>(a >= b ? P.slot(a, b) : P.slot(b, a));
      vt[k] = a < b ? 1 : 0;
    }
    N = C.layout().N;
    std::vector<int> vrd(static_cast<size_t>(N)), vrs(static_cast<size_t>(N));
    for (int i = 0; i < N; ++i) {
      vrd[static_cast<size_t>(i)] = i;
      vrs[static_cast<size_t>(i)] = sc.so.pos[static_cast<size_t>(i)];
    }
    count = static_cast<int>(C.size());
    slot_of = vs;
    transposed = vt;
    pos = sc.so.pos;
    d = to_device(vd, dev, s);
    src = to_device(vs, dev, s);
    tr = to_device(vt, dev, s);
    rd = to_device(vrd, dev, s);
    rs = to_device(vrs, dev, s);
  }
  void run(const double* from, double* to, const double* var_from, double* var_to, int bp, cudaStream_t s) const {
    launch_permute_tiles(to, from, reinterpret_cast<const int*>(d.p), reinterpret_cast<const int*>(src.p),
                         reinterpret_cast<const unsigned char*>(tr.p), count, bp, 148 * 8, s);
    if (var_to)
      launch_permute_rows(var_to, var_from, reinterpret_cast<const int*>(rd.p), reinterpret_cast<const int*>(rs.p), N,
                          bp, s);
    CK(cudaGetLastError());
  }
  // offset of natural closure element (slot, r, c) in the permuted store
  long long offset(long slot, int r, int c, int bp) const {
    const long long k = slot_of[static_cast<size_t>(slot)];
    return k * bp * bp + (transposed[static_cast<size_t>(slot)] ? static_cast<long long>(c) * bp + r
                                                                 : static_cast<long long>(r) * bp + c);
  }
};

static SigmaObj* selected_inverse_split(const MatrixObj& m, const Request& req, int device, SplitCall& sc,
                                        bool streamed) {
  DeviceRt& rt = runtime(device);
  cudaStream_t s = rt.stream;
  HostTimer tm(s);
  auto fp = factor_plan_for(sc.so.permuted, device, s, sc.so.split);
  const Pattern& Fp = fp->sym.filled;
  Request preq;
  preq.preset = kFactorPattern;
  const Closure selp = symbolic_inversion(select_tiles(Fp.layout(), Fp, preq), Fp);
  auto p2 = phase2_plan_for(Fp, selp, device, s, crit_split_p2(Fp, sc.so.split), sc.so.split);
  tm.mark("plans");
  const int bp = fp->bp, N = m.layout.N;
  const size_t bb = static_cast<size_t>(bp) * bp, T = Fp.size();
  SweepStores st;
  // counters: the plans', then (streamed upload) a raw upload counter and an
  // agents' arrival counter per column
  const long fc = fp->flow->host.counters;
  alloc_factor_stores(st, *fp, 1, device, s, std::max<long>(p2->flow->host.counters, fc + 2L * N),
                      p2->flow->host.scratch_doubles);
  auto* res = new SigmaObj;
  std::unique_ptr<SigmaObj> guard(res);
  res->device = device;
  res->layout = m.layout;
  res->req = req;
  auto nat = std::make_shared<Phase2Plan>();  // the natural closure (accessors); no device plan
  nat->sel = sc.sel;
  nat->bp = bp;
  nat->nb = p2->nb;
  res->plan = nat;
  const bool host_tiles = !m.gen.on && bp == m.layout.b && m.payload.pinned;  // natural tiles copy as they are
  const bool stream_up = streamed && host_tiles && streaming_allowed() && fp->flow->host.upl >= 0;
  // generator output / uploaded natural tiles land here before they are placed into A
  DevBuf staging(m.gen.on || host_tiles ? sc.sel.closure.size() * bb : 0, device, s);
  res->var = DevBuf(static_cast<size_t>(N) * bp, device, s);  // permuted order
  DevBuf& varp = res->var;
  tm.mark("allocations");
  // factor sweep on the permuted A store; phase 2 writes Sigma' over A (dead by then)
  std::vector<BaseTable> tf{make_table(st.A.p, st.L.p, st.P1.p, staging.p, varp.p, st.scratch.p, st.logdet.p,
                                       st.status.p, st.ctr(0))};
  std::vector<BaseTable> tp{make_table(st.A.p, st.L.p, st.P1.p, st.A.p, varp.p, st.scratch.p, st.logdet.p,
                                       st.status.p, st.ctr(0))};
  if (m.gen.on) {
    // natural tiles from the device generator into the staging store, then permuted
    device_generate(m, sc.natural.filled, bp, staging.p, s);
    std::vector<int> d(T);
    for (size_t k = 0; k < T; ++k) d[k] = static_cast<int>(k);
    DevBuf dd = to_device(d, device, s), ds = to_device(sc.src_filled, device, s), dt = to_device(sc.tr, device, s);
    launch_permute_tiles(st.A.p, staging.p, reinterpret_cast<const int*>(dd.p), reinterpret_cast<const int*>(ds.p),
                         reinterpret_cast<const unsigned char*>(dt.p), static_cast<int>(T), bp, 148 * 8, s);
    CK(cudaGetLastError());
    tm.mark("generate");
    factor_sweep(*fp, st, s, tf);
  } else if (host_tiles && !stream_up) {
    // the natural tiles in one copy, then placed (copied / transposed) on the device
    CK(cudaMemcpyAsync(staging.p, m.payload.p, m.pattern.size() * bb * sizeof(double), cudaMemcpyHostToDevice, s));
    std::vector<int> d, src;
    std::vector<unsigned char> tr;
    for (size_t k = 0; k < T; ++k)
      if (sc.src[k] >= 0) {
        d.push_back(static_cast<int>(k));
        src.push_back(sc.src[k]);
        tr.push_back(sc.tr[k]);
      }
    if (d.size() < T) CK(cudaMemsetAsync(st.A.p, 0, T * bb * sizeof(double), s));  // fill-in tiles
    DevBuf dd = to_device(d, device, s), ds = to_device(src, device, s), dt = to_device(tr, device, s);
    launch_permute_tiles(st.A.p, staging.p, reinterpret_cast<const int*>(dd.p), reinterpret_cast<const int*>(ds.p),
                         reinterpret_cast<const unsigned char*>(dt.p), static_cast<int>(d.size()), bp, 148 * 8, s);
    CK(cudaGetLastError());
    tm.mark("upload");
    factor_sweep(*fp, st, s, tf);
  } else if (!stream_up) {
    HostBuf hb(T * bb);
    permuted_payload(m, sc.so, bp, hb.p);
    CK(cudaMemcpyAsync(st.A.p, hb.p, T * bb * sizeof(double), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    tm.mark("upload");
    factor_sweep(*fp, st, s, tf);
  } else {
    // Streamed, permuted column by column in the plan's upload order.  A
    // natural tile column whose tiles all land, in order, in one permuted
    // column (I_0, the arrow) goes up as one copy straight into A; every
    // other natural column goes up as one copy into the staging store (the
    // Sigma store, in the matrix's own slot layout), and the kernel's agents
    // (worker 1 of the last TIB_SPLIT_AGENTS CTAs) copy or transpose its
    // tiles into A.  The copy engine sets a raw counter per permuted column
    // once every source column it needs is up; the agents release the
    // column's upload counter in upload order (tasks poll one column: the
    // touched one uploaded last).  (A second kernel beside the persistent
    // sweep would share a hardware queue with it and wait behind it.)
    int* ctr = reinterpret_cast<int*>(st.ctr(0));
    const bool fill = !(sc.natural.filled == m.pattern);
    if (fill) CK(cudaMemsetAsync(st.A.p, 0, T * bb * sizeof(double), s));
    CK(cudaMemsetAsync(ctr + fc, 0, 2 * static_cast<size_t>(N) * sizeof(int), s));
    const Pattern& Mp = m.pattern;
    // direct natural columns: slot k of column j -> permuted slot base + (k - start)
    std::vector<long> direct(static_cast<size_t>(N), -1);
    for (int j = 0; j < N; ++j) {
      const long k0 = Mp.col_start(j), k1 = Mp.col_start(j + 1);
      const int pj = sc.so.pos[static_cast<size_t>(j)];
      long base = -1;
      bool ok = k1 > k0;
      for (long k = k0; k < k1 && ok; ++k) {
        const int pi = sc.so.pos[static_cast<size_t>(Mp.tiles()[static_cast<size_t>(k)].i)];
        if (pi < pj) {
          ok = false;
          break;
        }
        const long d = Fp.slot(pi, pj);
        if (k == k0) base = d;
        ok = d == base + (k - k0);
      }
      if (ok) direct[static_cast<size_t>(j)] = base;
    }
    // agents' entries per permuted column, and each column's source columns
    std::vector<int> edst, esrc, eoff(static_cast<size_t>(N) + 1, 0);
    std::vector<unsigned char> etr;
    std::vector<std::vector<int>> need(static_cast<size_t>(N));
    for (int c = 0; c < N; ++c) {
      for (long k = Fp.col_start(c); k < Fp.col_start(c + 1); ++k) {
        const int sk = sc.src[static_cast<size_t>(k)];
        if (sk < 0) continue;  // fill-in: zeroed above
        const int nj = Mp.tiles()[static_cast<size_t>(sk)].j;
        need[static_cast<size_t>(c)].push_back(nj);
        if (direct[static_cast<size_t>(nj)] >= 0) continue;
        edst.push_back(static_cast<int>(k));
        esrc.push_back(sk);
        etr.push_back(sc.tr[static_cast<size_t>(k)]);
      }
      eoff[static_cast<size_t>(c) + 1] = static_cast<int>(edst.size());
    }
    DevBuf dd = to_device(edst, device, s), dsrc = to_device(esrc, device, s), dtr = to_device(etr, device, s),
           doff = to_device(eoff, device, s), dcols = to_device(fp->flow->host.upload_order, device, s);
    TransposeAgents ta;
    ta.agents = std::max(1, std::min(env_int("TIB_SPLIT_AGENTS", 8), fp->flow->grid - 4));
    ta.ncols = N;
    ta.bp = bp;
    ta.cols = reinterpret_cast<const int*>(dcols.p);
    ta.off = reinterpret_cast<const int*>(doff.p);
    ta.dst = reinterpret_cast<const int*>(dd.p);
    ta.src = reinterpret_cast<const int*>(dsrc.p);
    ta.tr = reinterpret_cast<const unsigned char*>(dtr.p);
    ta.raw = fc;
    ta.arrive = fc + N;
    ta.upl = fp->flow->host.upl;
    cudaEvent_t cleared, uploaded;
    CK(cudaEventCreateWithFlags(&cleared, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&uploaded, cudaEventDisableTiming));
    std::vector<char> sent(static_cast<size_t>(N), 0);
    std::function<void()> up = [&]() {
      CK(cudaStreamWaitEvent(rt.upload, cleared, 0));
      for (const int c : fp->flow->host.upload_order) {
        for (const int nj : need[static_cast<size_t>(c)]) {
          if (sent[static_cast<size_t>(nj)]) continue;
          sent[static_cast<size_t>(nj)] = 1;
          const long k0 = Mp.col_start(nj), k1 = Mp.col_start(nj + 1);
          const long d = direct[static_cast<size_t>(nj)];
          double* dst = d >= 0 ? st.A.p + static_cast<size_t>(d) * bb : staging.p + static_cast<size_t>(k0) * bb;
          CK(cudaMemcpyAsync(dst, m.payload.p + static_cast<size_t>(k0) * bb, static_cast<size_t>(k1 - k0) * bb * sizeof(double),
                             cudaMemcpyHostToDevice, rt.upload));
        }
        CK(cudaMemcpyAsync(ctr + fc + c, rt.one, sizeof(int), cudaMemcpyHostToDevice, rt.upload));
      }
      CK(cudaEventRecord(uploaded, rt.upload));
    };
    factor_sweep(*fp, st, s, tf, &up, cleared, 0, &ta);
    CK(cudaStreamWaitEvent(s, uploaded, 0));
    CK(cudaStreamSynchronize(s));  // the events and device lists die with this scope
    cudaEventDestroy(cleared);
    cudaEventDestroy(uploaded);
  }
  tm.mark("factor sweep");
  phase2_sweep(*p2, s, tp);
  tm.mark("phase-2 sweep");
  staging.release();
  res->unperm = std::make_shared<const Unpermute>(sc, device, s);
  res->Sp = std::move(st.A);  // Sigma' (phase 2 wrote it over the A store)
  std::vector<double> parts(fp->flow->host.logdet_doubles);
  CK(cudaMemcpyAsync(parts.data(), st.logdet.p, parts.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
  check_status(st.status, 1, m.layout, s);  // a NotSpd here is re-run in the natural order by the caller
  tm.mark("read-back");
  res->logdet = reduce_logdet(parts.data(), N, fp->nb);
  return guard.release();
}

// fused factorize + phase 2 for one matrix; returns the result object
static SigmaObj* selected_inverse_matrix(const MatrixObj& m, const Request& req, int device, bool allow_split = true) {
  // The two-chain order pays off when the factor sweep is bound by its chain:
  // always for A already on the device (the device generator).  A host matrix
  // that would stream up under the sweep keeps the natural order, streamed,
  // unless the natural chain (~30 us per 64-column step) is clearly longer
  // than the upload (~50 GB/s) -- otherwise the sweep waits for the upload in
  // either order (large config) -- and then goes up before the split sweep
  // and is placed on the device (medium: 82 -> ~72 ms).  TIB_SPLIT_STREAMED=1
  // streams the split order (in-kernel placement agents; a rare stall with
  // 8 agents is unresolved, so it is not the default).
  const bool streams = !m.gen.on && m.payload.pinned && m.layout.b % 64 == 0 && streaming_allowed();
  const int forced = env_int("TIB_SPLIT_STREAMED", 0);
  bool split_ok = !streams || forced != 0;
  if (streams && !split_ok) {
    const double chain_ms = m.layout.N * ((m.layout.b + 63) / 64) * 0.030;
    const double upload_ms = static_cast<double>(m.pattern.size()) * m.layout.b * m.layout.b * 8 / 50e6;
    split_ok = chain_ms > 1.3 * upload_ms;
  }
  if (allow_split && split_ok) {
    SplitCall sc;
    if (split_call(m, req, sc)) {
      try {
        return selected_inverse_split(m, req, device, sc, streams && forced != 0);
      } catch (const NotSpd&) {
        // the failing pivot of the permuted elimination is not the reference's:
        // the natural order reports the first non-positive pivot like factorize
        return selected_inverse_matrix(m, req, device, false);
      }
    }
  }
  DeviceRt& rt = runtime(device);
  cudaStream_t s = rt.stream;
  HostTimer tm(s);
  auto fp = factor_plan_for(m.pattern, device, s);
  const Pattern& F = fp->sym.filled;
  const Closure sel = symbolic_inversion(select_tiles(F.layout(), F, req), F);
  auto p2 = phase2_plan_for(F, sel, device, s);
  tm.mark("plans");
  SweepStores st;
  alloc_factor_stores(st, *fp, 1, device, s, p2->flow->host.counters, p2->flow->host.scratch_doubles);
  tm.mark("allocations");
  // The A store goes up tile column by tile column on the upload stream while
  // the factor sweep runs (tasks poll each column's counter); only possible
  // when the host tiles already have the device layout (b = bp; fill-in slots
  // are zeroed on the upload stream).
  const bool stream_up = !m.gen.on && fp->bp == m.layout.b && m.payload.pinned &&
                         streaming_allowed() && fp->flow->host.upl >= 0;
  if (!stream_up) upload_matrix(m, F, fp->bp, st.A.p, s);
  auto* res = new SigmaObj;
  std::unique_ptr<SigmaObj> guard(res);
  res->device = device;
  res->layout = m.layout;
  res->req = req;
  res->plan = p2;
  const size_t tile = static_cast<size_t>(fp->bp) * fp->bp;
  res->S = DevBuf(p2->sel.closure.size() * tile, device, s);
  res->var = DevBuf(static_cast<size_t>(m.layout.N) * fp->bp, device, s);
  std::vector<BaseTable> tables{make_table(st.A.p, st.L.p, st.P1.p, res->S.p, res->var.p, st.scratch.p, st.logdet.p, st.status.p, st.ctr(0))};
  if (stream_up) {
    cudaEvent_t cleared, uploaded, t_start = nullptr, t_up = nullptr, t_sweep = nullptr;
    CK(cudaEventCreateWithFlags(&cleared, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&uploaded, cudaEventDisableTiming));
    const size_t bb = static_cast<size_t>(fp->bp) * fp->bp;
    int* upl = reinterpret_cast<int*>(st.ctr(0)) + fp->flow->host.upl;
    const bool same = F == m.pattern;
    // fill-in slots are zero: one memset of the store on the sweep stream
    // (a kernel cannot run beside the persistent sweep), then the copies
    if (!same) CK(cudaMemsetAsync(st.A.p, 0, F.size() * bb * sizeof(double), s));
    std::function<void()> up = [&]() {
      const auto h0 = std::chrono::steady_clock::now();
      CK(cudaStreamWaitEvent(rt.upload, cleared, 0));
      for (const int c : fp->flow->host.upload_order) {
        const size_t t0 = static_cast<size_t>(F.col_start(c)), t1 = static_cast<size_t>(F.col_start(c + 1));
        if (same)
          CK(cudaMemcpyAsync(st.A.p + t0 * bb, m.payload.p + t0 * bb, (t1 - t0) * bb * sizeof(double),
                             cudaMemcpyHostToDevice, rt.upload));
        else
          upload_columns(m, F, c, c + 1, st.A.p, rt.upload, true, false);
        CK(cudaMemcpyAsync(upl + c, rt.one, sizeof(int), cudaMemcpyHostToDevice, rt.upload));
      }
      CK(cudaEventRecord(uploaded, rt.upload));
      if (tm.on) {
        CK(cudaEventRecord(t_up, rt.upload));
        std::fprintf(stderr, "[tib timing] copies enqueued in %.3f ms (host)\n",
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count());
      }
    };
    if (tm.on) {
      CK(cudaEventCreate(&t_start));
      CK(cudaEventCreate(&t_up));
      CK(cudaEventCreate(&t_sweep));
      CK(cudaEventRecord(t_start, s));
    }
    factor_sweep(*fp, st, s, tables, &up, cleared);
    if (tm.on) {
      CK(cudaEventRecord(t_sweep, s));
      CK(cudaEventSynchronize(t_sweep));
      CK(cudaEventSynchronize(t_up));
      float u = 0, w = 0;
      cudaEventElapsedTime(&u, t_start, t_up);
      cudaEventElapsedTime(&w, t_start, t_sweep);
      std::fprintf(stderr, "[tib timing] streamed upload done at %.3f ms, factor sweep at %.3f ms (%.1f GB/s)\n", u, w,
                   static_cast<double>(F.size()) * bb * 8 / (u * 1e6));
    }
    CK(cudaStreamWaitEvent(s, uploaded, 0));
    cudaEventDestroy(cleared);
    cudaEventDestroy(uploaded);
  } else {
    tm.mark("upload");
    factor_sweep(*fp, st, s, tables);
  }
  tm.mark("factor sweep");
  phase2_sweep(*p2, s, tables);
  tm.mark("phase-2 sweep");
  std::vector<double> parts(fp->flow->host.logdet_doubles);
  CK(cudaMemcpyAsync(parts.data(), st.logdet.p, parts.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
  check_status(st.status, 1, m.layout, s);
  tm.mark("read-back");
  res->logdet = reduce_logdet(parts.data(), m.layout.N, fp->nb);
  return guard.release();
}

static void download_tiles(const DevBuf& store, const Pattern& pat, int b, int bp, int* ti, int* tj, double* payload,
                           cudaStream_t s, bool transpose_diag) {
  const size_t bb = static_cast<size_t>(b) * b, bpp = static_cast<size_t>(bp) * bp;
  HostBuf h(pat.size() * bpp);
  CK(cudaMemcpyAsync(h.p, store.p, h.n * sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  for (size_t k = 0; k < pat.size(); ++k) {
    const Coord& c = pat.tiles()[k];
    if (ti) ti[k] = c.i;
    if (tj) tj[k] = c.j;
    if (!payload) continue;
    double* dst = payload + k * bb;
    const double* src = h.p + k * bpp;
    if (transpose_diag && c.i == c.j) {
      for (int r = 0; r < b; ++r)
        for (int q = 0; q < b; ++q) dst[static_cast<size_t>(r) * b + q] = src[static_cast<size_t>(q) * bp + r];
    } else {
      for (int r = 0; r < b; ++r) std::memcpy(dst + static_cast<size_t>(r) * b, src + static_cast<size_t>(r) * bp, b * sizeof(double));
    }
  }
}

// The natural-order Sigma store (un-permuted on first use after a two-chain call).
static const DevBuf& sigma_store(SigmaObj& sg) {
  if (sg.unperm && !sg.S.p) {
    DeviceRt& rt = runtime(sg.device);
    const int bp = sg.plan->bp;
    sg.S = DevBuf(sg.plan->sel.closure.size() * static_cast<size_t>(bp) * bp, sg.device, rt.stream);
    sg.unperm->run(sg.Sp.p, sg.S.p, nullptr, nullptr, bp, rt.stream);
    CK(cudaStreamSynchronize(rt.stream));
  }
  return sg.S;
}

static const double* sigma_host(SigmaObj& sg) {
  if (!sg.host) {
    DeviceRt& rt = runtime(sg.device);
    const DevBuf& S = sigma_store(sg);
    auto h = std::make_unique<HostBuf>(S.n);
    CK(cudaMemcpyAsync(h->p, S.p, h->n * sizeof(double), cudaMemcpyDeviceToHost, rt.stream));
    CK(cudaStreamSynchronize(rt.stream));
    sg.host = std::move(h);
  }
  return sg.host->p;
}

static uint64_t checksum_store(const double* hostbp, const Pattern& pat, int b, int bp) {
  Fnv h;
  const size_t bpp = static_cast<size_t>(bp) * bp;
  for (size_t k = 0; k < pat.size(); ++k) {
    const Coord& c = pat.tiles()[k];
    const uint64_t key = tile_key(c.i, c.j);
    h.mix(&key, sizeof(key));
    const double* src = hostbp + k * bpp;
    for (int r = 0; r < b; ++r) h.mix(src + static_cast<size_t>(r) * bp, b * sizeof(double));
  }
  return h.h;
}

// Host tiles (reference layout: b*b row-major per slot of F) -> a bp-layout
// device store; diagonal tiles optionally transposed (U_j -> X_j) and their
// padding set to the identity (so X = L^{-1} holds on the padded block).
static void upload_host_tiles(const Pattern& F, int b, int bp, const double* pay, double* dst, cudaStream_t s,
                              bool transpose_diag) {
  const size_t bb = static_cast<size_t>(b) * b, bpp = static_cast<size_t>(bp) * bp;
  HostBuf st(F.size() * bpp);
  std::memset(st.p, 0, st.n * sizeof(double));
  for (size_t k = 0; k < F.size(); ++k) {
    const Coord& c = F.tiles()[k];
    double* d = st.p + k * bpp;
    const double* src = pay + k * bb;
    if (transpose_diag && c.i == c.j) {
      for (int r = 0; r < b; ++r)
        for (int q = 0; q < b; ++q) d[static_cast<size_t>(r) * bp + q] = src[static_cast<size_t>(q) * b + r];
    } else {
      for (int r = 0; r < b; ++r) std::memcpy(d + static_cast<size_t>(r) * bp, src + static_cast<size_t>(r) * b, b * sizeof(double));
    }
    if (c.i == c.j)
      for (int r = b; r < bp; ++r) d[static_cast<size_t>(r) * bp + r] = 1.0;
  }
  CK(cudaMemcpyAsync(dst, st.p, st.n * sizeof(double), cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));
}

// The phase-1 transform (X_j = L_jj^{-1}, W_kj = L_kj X_j) of a factor's L
// store on the device (build_phase1_dataflow; selinv.cpp:195-223).
static void run_phase1(FactorObj& f) {
  DeviceRt& rt = runtime(f.device);
  cudaStream_t s = rt.stream;
  auto plan = phase1_plan_for(f.F, f.device, s);
  DevBuf scratch(plan->host.scratch_doubles, f.device, s);
  DevBuf logdet(plan->host.logdet_doubles, f.device, s);
  DevBuf status(1, f.device, s);
  CK(cudaMemsetAsync(status.p, 0xff, sizeof(unsigned long long), s));
  DevBuf ctr = alloc_counters(plan->host.counters, 1, f.device, s);
  // the invert-only leaves read their block through the A-store entry: L
  std::vector<BaseTable> tables{make_table(f.L.p, f.L.p, f.P1.p, nullptr, nullptr, scratch.p, logdet.p, status.p, ctr.p)};
  run_flow_chunked(*plan, tables, s);
  CK(cudaStreamSynchronize(s));
  check_watchdog();
}

// Tiles (i, j) of a factor store <-> host b x b row-major payloads.
static void factor_tile_copy(FactorObj& f, const DevBuf& store, long count, const int* ti, const int* tj, double* host,
                             bool to_device) {
  DeviceRt& rt = runtime(f.device);
  const int b = f.layout.b;
  const size_t bpp = static_cast<size_t>(f.bp) * f.bp, bb = static_cast<size_t>(b) * b;
  for (long k = 0; k < count; ++k) {
    const long slot = f.F.slot(ti[k], tj[k]);
    if (slot < 0)
      throw Error(kErrContract, "tile (" + std::to_string(ti[k]) + ", " + std::to_string(tj[k]) + ") is not in the factor");
    double* d = store.p + static_cast<size_t>(slot) * bpp;
    double* h = host + static_cast<size_t>(k) * bb;
    if (to_device)
      CK(cudaMemcpy2DAsync(d, f.bp * sizeof(double), h, b * sizeof(double), b * sizeof(double), b,
                           cudaMemcpyHostToDevice, rt.stream));
    else
      CK(cudaMemcpy2DAsync(h, b * sizeof(double), d, f.bp * sizeof(double), b * sizeof(double), b,
                           cudaMemcpyDeviceToHost, rt.stream));
  }
  CK(cudaStreamSynchronize(rt.stream));
}

// A factor from host tiles (factor_from_tile_file, tileio.cpp:109-117): phase 1
// = the factor L (phase 1 then runs on the device: build_phase1_dataflow),
// phase 2 = phase-1 tiles U / W (used as they are; selinv.cpp:355 skips
// phase 1 for them).  logdet from the diagonal: 2 sum log L_rr = -2 sum log U_rr.
static FactorObj* factor_from_host(const Layout& L, int phase, const Pattern& P, const double* pay, int device) {
  if (phase != 1 && phase != 2)
    throw Error(kErrFormat, "expected a factor tile file, found phase tag " + std::to_string(phase));
  if (!P.has_all_diagonals()) throw Error(kErrStructure, "factor tiles must include every diagonal tile");
  DeviceRt& rt = runtime(device);
  cudaStream_t s = rt.stream;
  auto f = std::make_unique<FactorObj>();
  f->device = device;
  f->layout = L;
  f->F = P;
  f->bp = (L.b + 63) / 64 * 64;
  f->nb = f->bp / 64;
  const size_t tile = static_cast<size_t>(f->bp) * f->bp, bb = static_cast<size_t>(L.b) * L.b;
  double ld = 0.0;
  for (long r = 0; r < L.n; ++r) {
    const int j = static_cast<int>(r / L.b);
    const double v = pay[static_cast<size_t>(P.col_start(j)) * bb + static_cast<size_t>(r % L.b) * L.b + (r % L.b)];
    if (!(v > 0.0)) throw Error(kErrConsistency, "factor diagonal entry " + std::to_string(r) + " is not positive");
    ld += std::log(v);
  }
  f->logdet = phase == 1 ? 2.0 * ld : -2.0 * ld;
  f->P1 = DevBuf(P.size() * tile, device, s);
  if (phase == 2) {
    f->has_L = false;
    upload_host_tiles(P, L.b, f->bp, pay, f->P1.p, s, true);
    return f.release();
  }
  f->L = DevBuf(P.size() * tile, device, s);
  upload_host_tiles(P, L.b, f->bp, pay, f->L.p, s, false);
  run_phase1(*f);
  return f.release();
}

// ---------------------------------------------------------------------------
// error plumbing
static thread_local std::string t_err;
static thread_local long t_pivot = -1;
static thread_local int t_ti = -1, t_tj = -1;

template <class F>
static int guarded(F&& f) {
  try {
    f();
    return kOk;
  } catch (const NotSpd& e) {
    t_err = e.what();
    t_pivot = e.pivot;
    t_ti = e.tile_i;
    t_tj = e.tile_j;
    return kErrNotSpd;
  } catch (const Error& e) {
    t_err = e.what();
    return e.status;
  } catch (const std::bad_alloc&) {
    t_err = "out of host memory";
    return kErrGeneric;
  } catch (const std::exception& e) {
    t_err = e.what();
    return kErrGeneric;
  }
}

template <class T>
static T* need(T* p, const char* what) {
  if (!p) throw Error(kErrInvalidArgument, std::string("null ") + what + " handle");
  return p;
}

}  // namespace tib

using namespace tib;

struct tib_matrix_s : MatrixObj {};
struct tib_factor_s : FactorObj {};
struct tib_sigma_s : SigmaObj {};

extern "C" {

const char* tib_version(void) { return "0.1.0"; }
const char* tib_last_error_message(void) { return t_err.c_str(); }
int tib_last_not_spd(long* pivot, int* ti, int* tj) {
  if (pivot) *pivot = t_pivot;
  if (ti) *ti = t_ti;
  if (tj) *tj = t_tj;
  return kOk;
}
int tib_device_count(int* count) {
  return guarded([&] {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
      cudaGetLastError();
      c = 0;
    }
    *count = c;
  });
}

static tib_matrix wrap(HostMatrix&& hm) {
  auto* out = new tib_matrix_s;
  fill_matrix(*out, std::move(hm));
  return out;
}

int tib_matrix_generate(long n, long w, long t, double density, uint64_t seed, int b, tib_matrix* out) {
  return guarded([&] { *out = wrap(generate_arrowhead(n, w, t, density, seed, b)); });
}
int tib_matrix_from_dense(long n, int b, const double* a, tib_matrix* out) {
  return guarded([&] {
    if (n < 1 || !a) throw Error(kErrInvalidArgument, "from_dense needs a square 2-D array");
    *out = wrap(matrix_from_dense(n, b, a));
  });
}
int tib_matrix_from_tiles(long n, int b, long count, const int* ti, const int* tj, const double* payload,
                          tib_matrix* out) {
  return guarded([&] { *out = wrap(matrix_from_tiles(n, b, count, ti, tj, payload)); });
}
int tib_matrix_read_mm(const char* text, size_t len, int b, tib_matrix* out) {
  return guarded([&] { *out = wrap(read_matrix_market(std::string(text, len), b)); });
}
int tib_matrix_write_mm(tib_matrix m, char* buf, size_t* len) {
  return guarded([&] {
    need(m, "matrix");
    HostMatrix hm;
    hm.layout = m->layout;
    hm.pattern = m->pattern;
    const double* pay = host_payload(*m);
    hm.payload.assign(pay, pay + m->payload.n);
    const std::string text = write_matrix_market(hm);
    if (buf && *len >= text.size()) std::memcpy(buf, text.data(), text.size());
    *len = text.size();
  });
}
int tib_matrix_info(tib_matrix m, long* n, int* b, int* N, long* stored) {
  return guarded([&] {
    need(m, "matrix");
    if (n) *n = m->layout.n;
    if (b) *b = m->layout.b;
    if (N) *N = m->layout.N;
    if (stored) *stored = static_cast<long>(m->pattern.size());
  });
}
int tib_matrix_tiles(tib_matrix m, int* ti, int* tj, double* payload) {
  return guarded([&] {
    need(m, "matrix");
    for (size_t k = 0; k < m->pattern.size(); ++k) {
      if (ti) ti[k] = m->pattern.tiles()[k].i;
      if (tj) tj[k] = m->pattern.tiles()[k].j;
    }
    if (payload) {
      const double* pay = host_payload(*m);
      std::memcpy(payload, pay, m->payload.n * sizeof(double));
    }
  });
}
int tib_matrix_generate_kronecker(int nt, int nx, int ny, int p, double rho, double kappa2, double tau,
                                  double tau_y, double q_beta, uint64_t seed, int b, tib_matrix* out) {
  return guarded([&] { *out = wrap(generate_kronecker(nt, nx, ny, p, rho, kappa2, tau, tau_y, q_beta, seed, b)); });
}
int tib_matrix_generate_device(long n, long w, long t, uint64_t seed, int b, int device, tib_matrix* out) {
  return guarded([&] {
    runtime(device);  // no device: TIB_ERR_CUDA (no host fallback for a device matrix)
    auto* m = new tib_matrix_s;
    m->pattern = arrowhead_pattern(n, w, t, b);
    m->layout = m->pattern.layout();
    m->gen.on = true;
    m->gen.n = n;
    m->gen.w = w;
    m->gen.t = t;
    m->gen.seed = seed;
    m->gen.device = device;
    *out = m;
  });
}
int tib_matrix_checksum(tib_matrix m, uint64_t* out) {
  return guarded([&] {
    need(m, "matrix");
    *out = checksum_store(host_payload(*m), m->pattern, m->layout.b, m->layout.b);
  });
}
int tib_matrix_free(tib_matrix m) {
  delete m;
  return kOk;
}

int tib_symbolic_pattern(tib_matrix m, long* count, int* ti, int* tj) {
  return guarded([&] {
    need(m, "matrix");
    const Pattern F = symbolic_fill(m->pattern);
    *count = static_cast<long>(F.size());
    if (ti && tj)
      for (size_t k = 0; k < F.size(); ++k) {
        ti[k] = F.tiles()[k].i;
        tj[k] = F.tiles()[k].j;
      }
  });
}
int tib_symbolic_closure(tib_matrix m, int preset, const long* rows, const long* cols, long ne, long* count,
                         int* ti, int* tj, int* growth) {
  return guarded([&] {
    need(m, "matrix");
    const Pattern F = symbolic_fill(m->pattern);
    const Closure c = symbolic_inversion(select_tiles(F.layout(), F, make_request(preset, rows, cols, ne)), F);
    *count = static_cast<long>(c.closure.size());
    if (growth) *growth = c.growth_warning ? 1 : 0;
    if (ti && tj)
      for (size_t k = 0; k < c.closure.size(); ++k) {
        ti[k] = c.closure.tiles()[k].i;
        tj[k] = c.closure.tiles()[k].j;
      }
  });
}
int tib_flops(tib_matrix m, int preset, const long* rows, const long* cols, long ne, double* f, double* p1,
              double* p2) {
  return guarded([&] {
    need(m, "matrix");
    const FactorPlan plan = symbolic_cholesky(m->pattern);
    const Closure c = symbolic_inversion(select_tiles(plan.filled.layout(), plan.filled, make_request(preset, rows, cols, ne)),
                                         plan.filled);
    const Flops fl = count_flops(plan, &c);
    if (f) *f = fl.factorize;
    if (p1) *p1 = fl.phase1;
    if (p2) *p2 = fl.phase2;
  });
}

static void put_report(const KernelReport& r, long long* out) {
  const long long v[9] = {r.n_tiles, r.band_b, r.trsm, r.trmm, r.lauum, r.gemm_actual, r.gemm_predicted,
                          r.critical_path, r.match ? 1 : 0};
  std::memcpy(out, v, sizeof(v));
}
int tib_dag_report(int n_tiles, int band, long long* report) {
  return guarded([&] { put_report(count_task_kernels(band_arrow_task_graph(n_tiles, band > 0 ? band : n_tiles)), report); });
}
int tib_dag_report_matrix(tib_matrix m, int preset, const long* rows, const long* cols, long ne, long long* report) {
  return guarded([&] {
    need(m, "matrix");
    const FactorPlan plan = symbolic_cholesky(m->pattern);
    const Closure c = symbolic_inversion(select_tiles(plan.filled.layout(), plan.filled, make_request(preset, rows, cols, ne)),
                                         plan.filled);
    put_report(count_task_kernels(build_task_graph(c, plan.filled)), report);
  });
}
int tib_dag_export_dot(int n_tiles, int band, int cores, char* buf, size_t* len) {
  return guarded([&] {
    TaskGraph g = band_arrow_task_graph(n_tiles, band > 0 ? band : n_tiles);
    if (cores > 0) assign_task_cores(g, cores);
    const std::string text = task_graph_dot(g);
    if (buf && *len >= text.size()) std::memcpy(buf, text.data(), text.size());
    *len = text.size();
  });
}
int tib_predict_gemm_count(int n_tiles, int band, long long* out) {
  return guarded([&] { *out = predict_gemm_count(n_tiles, band); });
}

int tib_factorize(tib_matrix m, int device, tib_factor* out) {
  return guarded([&] {
    need(m, "matrix");
    DeviceRt& rt = runtime(device);
    cudaStream_t s = rt.stream;
    auto fp = factor_plan_for(m->pattern, device, s);
    SweepStores st;
    alloc_factor_stores(st, *fp, 1, device, s);
    upload_matrix(*m, fp->sym.filled, fp->bp, st.A.p, s);
    std::vector<BaseTable> tables{make_table(st.A.p, st.L.p, st.P1.p, nullptr, nullptr, st.scratch.p, st.logdet.p, st.status.p, st.ctr(0))};
    factor_sweep(*fp, st, s, tables);
    std::vector<double> parts(static_cast<size_t>(m->layout.N) * fp->nb);
    CK(cudaMemcpyAsync(parts.data(), st.logdet.p, parts.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    check_status(st.status, 1, m->layout, s);
    auto* f = new tib_factor_s;
    f->device = device;
    f->layout = m->layout;
    f->F = fp->sym.filled;
    f->bp = fp->bp;
    f->nb = fp->nb;
    f->L = std::move(st.L);
    f->P1 = std::move(st.P1);
    f->logdet = reduce_logdet(parts.data(), m->layout.N, fp->nb);
    *out = f;
  });
}
int tib_factor_info(tib_factor f, long* n, int* b, long* stored) {
  return guarded([&] {
    need(f, "factor");
    if (n) *n = f->layout.n;
    if (b) *b = f->layout.b;
    if (stored) *stored = static_cast<long>(f->F.size());
  });
}
int tib_factor_get_tiles(tib_factor f, long count, const int* ti, const int* tj, double* payload) {
  return guarded([&] {
    need(f, "factor");
    if (!f->has_L) throw Error(kErrContract, "the factor holds phase-1 tiles only (kPhase1 input)");
    if (count < 0 || (count > 0 && (!ti || !tj || !payload))) throw Error(kErrInvalidArgument, "null tile arrays");
    factor_tile_copy(*f, f->L, count, ti, tj, payload, false);
  });
}
int tib_factor_replace_tiles(tib_factor f, long count, const int* ti, const int* tj, const double* payload) {
  return guarded([&] {
    need(f, "factor");
    if (!f->has_L) throw Error(kErrContract, "the factor holds phase-1 tiles only (kPhase1 input)");
    if (count < 0 || (count > 0 && (!ti || !tj || !payload))) throw Error(kErrInvalidArgument, "null tile arrays");
    const int b = f->layout.b;
    const size_t bb = static_cast<size_t>(b) * b;
    // logdet: swap the replaced diagonal tiles' terms
    double delta = 0.0;
    std::vector<double> old(bb);
    for (long k = 0; k < count; ++k) {
      if (ti[k] != tj[k]) continue;
      factor_tile_copy(*f, f->L, 1, ti + k, tj + k, old.data(), false);
      for (int r = 0; r < b; ++r) {
        const long row = static_cast<long>(ti[k]) * b + r;
        if (row >= f->layout.n) break;
        const double v = payload[static_cast<size_t>(k) * bb + static_cast<size_t>(r) * b + r];
        if (!(v > 0.0)) throw Error(kErrConsistency, "factor diagonal entry " + std::to_string(row) + " is not positive");
        delta += std::log(v) - std::log(old[static_cast<size_t>(r) * b + r]);
      }
    }
    factor_tile_copy(*f, f->L, count, ti, tj, const_cast<double*>(payload), true);
    f->logdet += 2.0 * delta;
    run_phase1(*f);
  });
}
int tib_factor_logdet(tib_factor f, double* out) {
  return guarded([&] { *out = need(f, "factor")->logdet; });
}
int tib_factor_tiles(tib_factor f, int phase, int* ti, int* tj, double* payload) {
  return guarded([&] {
    need(f, "factor");
    if (phase != 1 && phase != 2) throw Error(kErrInvalidArgument, "phase must be 1 (factor) or 2 (phase-1 tiles)");
    if (phase == 1 && !f->has_L) throw Error(kErrContract, "the factor holds phase-1 tiles only (kPhase1 input)");
    DeviceRt& rt = runtime(f->device);
    download_tiles(phase == 1 ? f->L : f->P1, f->F, f->layout.b, f->bp, ti, tj, payload, rt.stream, phase == 2);
  });
}
int tib_factor_checksum(tib_factor f, uint64_t* out) {
  return guarded([&] {
    need(f, "factor");
    DeviceRt& rt = runtime(f->device);
    if (f->has_L) {
      HostBuf h(f->L.n);
      CK(cudaMemcpyAsync(h.p, f->L.p, h.n * sizeof(double), cudaMemcpyDeviceToHost, rt.stream));
      CK(cudaStreamSynchronize(rt.stream));
      *out = checksum_store(h.p, f->F, f->layout.b, f->bp);
    } else {  // the phase-1 tiles in the reference's form (U_j = X_j^T)
      const size_t bb = static_cast<size_t>(f->layout.b) * f->layout.b;
      std::vector<double> pay(f->F.size() * bb);
      download_tiles(f->P1, f->F, f->layout.b, f->bp, nullptr, nullptr, pay.data(), rt.stream, true);
      *out = checksum_store(pay.data(), f->F, f->layout.b, f->layout.b);
    }
  });
}
int tib_factor_free(tib_factor f) {
  delete f;
  return kOk;
}
int tib_factor_phase(tib_factor f, int* phase) {
  return guarded([&] { *phase = need(f, "factor")->has_L ? 1 : 2; });
}
int tib_factor_from_tiles(long n, int b, int phase, long count, const int* ti, const int* tj, const double* payload,
                          int device, tib_factor* out) {
  return guarded([&] {
    if (count < 1 || !ti || !tj || !payload) throw Error(kErrInvalidArgument, "factor tiles are empty");
    const Layout L = build_layout(n, b);
    std::vector<Coord> c(static_cast<size_t>(count));
    for (long k = 0; k < count; ++k) c[static_cast<size_t>(k)] = {ti[k], tj[k]};
    const Pattern P(L, c);
    if (static_cast<long>(P.size()) != count) throw Error(kErrInvalidArgument, "duplicate factor tiles");
    const size_t bb = static_cast<size_t>(b) * b;
    std::vector<double> pay(P.size() * bb);
    for (long k = 0; k < count; ++k)
      std::memcpy(&pay[static_cast<size_t>(P.slot(ti[k], tj[k])) * bb], payload + static_cast<size_t>(k) * bb, bb * sizeof(double));
    FactorObj* f = factor_from_host(L, phase, P, pay.data(), device);
    auto* o = new tib_factor_s;
    static_cast<FactorObj&>(*o) = std::move(*f);
    delete f;
    *out = o;
  });
}
int tib_factor_read_stls(const char* path, int device, tib_factor* out) {
  return guarded([&] {
    if (!path) throw Error(kErrInvalidArgument, "null path");
    const TileFileData d = read_tile_file(path);
    FactorObj* f = factor_from_host(d.layout, d.phase, d.pattern, d.payload.data(), device);
    auto* o = new tib_factor_s;
    static_cast<FactorObj&>(*o) = std::move(*f);
    delete f;
    *out = o;
  });
}
int tib_factor_write_stls(tib_factor f, int phase, const char* path) {
  return guarded([&] {
    need(f, "factor");
    if (!path) throw Error(kErrInvalidArgument, "null path");
    if (phase != 1 && phase != 2) throw Error(kErrInvalidArgument, "phase must be 1 (factor) or 2 (phase-1 tiles)");
    if (phase == 1 && !f->has_L) throw Error(kErrContract, "the factor holds phase-1 tiles only (kPhase1 input)");
    DeviceRt& rt = runtime(f->device);
    const size_t bb = static_cast<size_t>(f->layout.b) * f->layout.b;
    std::vector<double> pay(f->F.size() * bb);
    download_tiles(phase == 1 ? f->L : f->P1, f->F, f->layout.b, f->bp, nullptr, nullptr, pay.data(), rt.stream, phase == 2);
    write_tile_file(path, f->layout, phase, f->F, pay.data());
  });
}
int tib_matrix_read_stls(const char* path, tib_matrix* out) {
  return guarded([&] {
    if (!path) throw Error(kErrInvalidArgument, "null path");
    TileFileData d = read_tile_file(path);
    if (d.phase != 0) throw Error(kErrFormat, "expected a matrix tile file, found phase tag " + std::to_string(d.phase));
    HostMatrix hm;
    hm.layout = d.layout;
    hm.pattern = std::move(d.pattern);
    hm.payload = std::move(d.payload);
    *out = wrap(std::move(hm));
  });
}
int tib_matrix_write_stls(tib_matrix m, const char* path) {
  return guarded([&] {
    need(m, "matrix");
    if (!path) throw Error(kErrInvalidArgument, "null path");
    write_tile_file(path, m->layout, 0, m->pattern, host_payload(*m));
  });
}

int tib_selected_inverse(tib_matrix m, int preset, const long* rows, const long* cols, long ne, int device,
                         tib_sigma* out) {
  return guarded([&] {
    need(m, "matrix");
    const Request req = make_request(preset, rows, cols, ne);
    SigmaObj* r = selected_inverse_matrix(*m, req, device);
    auto* o = new tib_sigma_s;
    static_cast<SigmaObj&>(*o) = std::move(*r);
    delete r;
    *out = o;
  });
}

int tib_selected_inverse_of_factor(tib_factor f, int preset, const long* rows, const long* cols, long ne,
                                   tib_sigma* out) {
  return guarded([&] {
    need(f, "factor");
    DeviceRt& rt = runtime(f->device);
    cudaStream_t s = rt.stream;
    const Request req = make_request(preset, rows, cols, ne);
    const Pattern& F = f->F;
    const Closure sel = symbolic_inversion(select_tiles(F.layout(), F, req), F);
    auto p2 = phase2_plan_for(F, sel, f->device, s);
    auto* res = new tib_sigma_s;
    std::unique_ptr<tib_sigma_s> guard(res);
    res->device = f->device;
    res->layout = f->layout;
    res->req = req;
    res->plan = p2;
    res->logdet = f->logdet;
    const size_t tile = static_cast<size_t>(p2->bp) * p2->bp;
    res->S = DevBuf(p2->sel.closure.size() * tile, f->device, s);
    res->var = DevBuf(static_cast<size_t>(f->layout.N) * p2->bp, f->device, s);
    DevBuf ctr = alloc_counters(p2->flow->host.counters, 1, f->device, s);
    DevBuf scratch(p2->flow->host.scratch_doubles, f->device, s);
    std::vector<BaseTable> tables{make_table(nullptr, f->L.p, f->P1.p, res->S.p, res->var.p, scratch.p, nullptr, nullptr, ctr.p)};
    phase2_sweep(*p2, s, tables);
    CK(cudaStreamSynchronize(s));
    check_watchdog();
    *out = guard.release();
  });
}

int tib_sigma_info(tib_sigma sg, long* n, int* b, long* closure_tiles, int* growth) {
  return guarded([&] {
    need(sg, "result");
    if (n) *n = sg->layout.n;
    if (b) *b = sg->layout.b;
    if (closure_tiles) *closure_tiles = static_cast<long>(sg->plan->sel.closure.size());
    if (growth) *growth = sg->plan->sel.growth_warning ? 1 : 0;
  });
}
int tib_sigma_logdet(tib_sigma sg, double* out) {
  return guarded([&] { *out = need(sg, "result")->logdet; });
}
int tib_sigma_diagonal(tib_sigma sg, double* out) {
  return guarded([&] {
    need(sg, "result");
    const Layout& L = sg->layout;
    for (int i = 0; i < L.N; ++i)
      if (!sg->plan->sel.closure.has(i, i))
        throw Error(kErrContract, "entry (" + std::to_string(static_cast<long>(i) * L.b) + ", " +
                                      std::to_string(static_cast<long>(i) * L.b) + ") lies outside the computed closure");
    DeviceRt& rt = runtime(sg->device);
    const int bp = sg->plan->bp;
    std::vector<double> v(sg->var.n);
    CK(cudaMemcpyAsync(v.data(), sg->var.p, v.size() * sizeof(double), cudaMemcpyDeviceToHost, rt.stream));
    CK(cudaStreamSynchronize(rt.stream));
    // (two-chain order: tile row i of the variances is at position pos[i])
    const std::vector<int>* pos = sg->unperm ? &sg->unperm->pos : nullptr;
    for (long r = 0; r < L.n; ++r) {
      const long i = r / L.b;
      out[r] = v[static_cast<size_t>(pos ? (*pos)[static_cast<size_t>(i)] : i) * bp + static_cast<size_t>(r % L.b)];
    }
  });
}
int tib_sigma_entries(tib_sigma sg, long* count, long* rows, long* cols, double* vals) {
  return guarded([&] {
    need(sg, "result");
    const Layout& L = sg->layout;
    const Pattern& C = sg->plan->sel.closure;
    const int bp = sg->plan->bp;
    const bool want = rows || cols || vals;
    // extract_entries order (selinv.cpp:387-439); the values are gathered on
    // the device unless the request reads a large part of the store anyway
    std::vector<long long> at;
    long k = 0;
    for_each_request_entry(L, C, sg->plan->sel.requested, sg->req, [&](long r, long c) {
      const Address a = map_entry_to_tile(L, r, c);
      const long slot = C.slot(a.tile.i, a.tile.j);
      if (slot < 0)
        throw Error(kErrContract, "entry (" + std::to_string(r) + ", " + std::to_string(c) +
                                      ") lies outside the computed closure");
      if (want) {
        if (rows) rows[k] = r;
        if (cols) cols[k] = c;
        if (vals)
          at.push_back(static_cast<long long>(slot) * bp * bp + static_cast<long long>(a.row_off) * bp + a.col_off);
        if (vals && sg->unperm && !sg->S.p) at.back() = sg->unperm->offset(slot, a.row_off, a.col_off, bp);
      }
      ++k;
    });
    *count = k;
    if (!vals || at.empty()) return;
    const bool permuted = sg->unperm && !sg->S.p;  // offsets above are into Sp
    const size_t store = permuted ? sg->Sp.n : sg->S.n;
    if (sg->host || at.size() * 16 > store) {  // most of the store (or already on the host)
      if (permuted) {  // natural offsets again, into the un-permuted host copy
        long e = 0;
        for_each_request_entry(L, C, sg->plan->sel.requested, sg->req, [&](long r, long c) {
          const Address a = map_entry_to_tile(L, r, c);
          at[static_cast<size_t>(e++)] = static_cast<long long>(C.slot(a.tile.i, a.tile.j)) * bp * bp +
                                         static_cast<long long>(a.row_off) * bp + a.col_off;
        });
      }
      const double* h = sigma_host(*sg);
      for (size_t e = 0; e < at.size(); ++e) vals[e] = h[at[e]];
      return;
    }
    DeviceRt& rt = runtime(sg->device);
    DevBuf idx((at.size() + 0), sg->device, rt.stream), out(at.size(), sg->device, rt.stream);
    CK(cudaMemcpyAsync(idx.p, at.data(), at.size() * sizeof(long long), cudaMemcpyHostToDevice, rt.stream));
    launch_gather(permuted ? sg->Sp.p : sg->S.p, reinterpret_cast<const long long*>(idx.p), out.p,
                  static_cast<long long>(at.size()), rt.stream);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(vals, out.p, at.size() * sizeof(double), cudaMemcpyDeviceToHost, rt.stream));
    CK(cudaStreamSynchronize(rt.stream));
  });
}
int tib_sigma_tiles(tib_sigma sg, int* ti, int* tj, double* payload) {
  return guarded([&] {
    need(sg, "result");
    DeviceRt& rt = runtime(sg->device);
    download_tiles(sigma_store(*sg), sg->plan->sel.closure, sg->layout.b, sg->plan->bp, ti, tj, payload, rt.stream, false);
  });
}
int tib_sigma_checksum(tib_sigma sg, uint64_t* out) {
  return guarded([&] {
    need(sg, "result");
    *out = checksum_store(sigma_host(*sg), sg->plan->sel.closure, sg->layout.b, sg->plan->bp);
  });
}
int tib_sigma_write_stls(tib_sigma sg, const char* path) {
  return guarded([&] {
    need(sg, "result");
    if (!path) throw Error(kErrInvalidArgument, "null path");
    DeviceRt& rt = runtime(sg->device);
    const Pattern& C = sg->plan->sel.closure;
    const size_t bb = static_cast<size_t>(sg->layout.b) * sg->layout.b;
    std::vector<double> pay(C.size() * bb);
    download_tiles(sigma_store(*sg), C, sg->layout.b, sg->plan->bp, nullptr, nullptr, pay.data(), rt.stream, false);
    write_tile_file(path, sg->layout, 3, C, pay.data());
  });
}
int tib_sigma_free(tib_sigma sg) {
  delete sg;
  return kOk;
}

int tib_selected_inverse_batch(const tib_matrix* ms, int count, int device, double* logdet, double* diag) {
  return guarded([&] {
    if (count < 1 || !ms) throw Error(kErrInvalidArgument, "batch needs at least one matrix");
    const MatrixObj& m0 = *need(ms[0], "matrix");
    for (int k = 1; k < count; ++k)
      if (!(need(ms[k], "matrix")->pattern == m0.pattern) || ms[k]->layout.n != m0.layout.n)
        throw Error(kErrInvalidArgument, "batched matrices must share one tile pattern");
    DeviceRt& rt = runtime(device);
    cudaStream_t s = rt.stream;
    HostTimer tm(s);
    // (a host batch runs as pipelined launches of TIB_BATCH_PIPE matrices)
    const int pipe_n = env_int("TIB_BATCH_PIPE", 16);
    bool host_batch = true;
    for (int k = 0; k < count; ++k) host_batch = host_batch && !ms[k]->gen.on && ms[k]->payload.pinned;
    const int launch_n = host_batch && pipe_n > 0 && count > pipe_n ? pipe_n : count;
    auto fp = factor_plan_for(m0.pattern, device, s, -1, launch_n);
    const Pattern& F = fp->sym.filled;
    Request req;
    req.preset = kFactorPattern;
    const Closure sel = symbolic_inversion(select_tiles(F.layout(), F, req), F);
    auto p2 = phase2_plan_for(F, sel, device, s, -1, -1, count);
    tm.mark("plans");
    const size_t tile = static_cast<size_t>(fp->bp) * fp->bp;
    SweepStores st;
    alloc_factor_stores(st, *fp, count, device, s, p2->flow->host.counters, p2->flow->host.scratch_doubles);
    DevBuf Sg(p2->sel.closure.size() * tile * count, device, s);
    DevBuf var(static_cast<size_t>(m0.layout.N) * fp->bp * count, device, s);
    tm.mark("allocations");
    std::vector<BaseTable> tables;
    const size_t T = F.size();
    // streamed upload (as the single path): tile column c of every matrix goes
    // up on the copy stream, column-major over the batch, while the batched
    // factor sweep runs; each matrix's tasks poll that matrix's column counters
    bool host_ready = fp->bp == m0.layout.b;
    for (int k = 0; k < count; ++k) host_ready = host_ready && !ms[k]->gen.on && ms[k]->payload.pinned;
    // pipelined batch: groups of `pipe` matrices, each group's upload (one
    // copy per matrix on the copy stream) overlapping the previous group's
    // two sweeps.  A batch streamed column-wise under one launch stalls: with
    // tens of matrices every worker ends up waiting in a task whose target
    // column has not arrived, and the sweep runs after the upload, not under it.
    const int pipe = env_int("TIB_BATCH_PIPE", 16);
    const bool pipelined = host_ready && F == m0.pattern && pipe > 0 && count > pipe;
    bool stream_up = !pipelined && host_ready && streaming_allowed() && fp->flow->host.upl >= 0 &&
                     static_cast<size_t>(count) <= max_batch(*fp->flow);
    // device-generated members with one parameter set: one generator launch
    bool gen_all = !stream_up && !pipelined;
    for (int k = 0; k < count && gen_all; ++k)
      gen_all = ms[k]->gen.on && ms[k]->gen.n == m0.gen.n && ms[k]->gen.w == m0.gen.w && ms[k]->gen.t == m0.gen.t;
    if (gen_all) {
      std::vector<const MatrixObj*> mm;
      for (int k = 0; k < count; ++k) mm.push_back(ms[k]);
      device_generate(mm, F, fp->bp, st.A.p, T * tile, s);
    }
    for (int k = 0; k < count; ++k) {
      if (!stream_up && !pipelined && !gen_all) upload_matrix(*ms[k], F, fp->bp, st.A.p + T * tile * k, s);
      tables.push_back(make_table(st.A.p + T * tile * k, st.L.p + T * tile * k, st.P1.p + T * tile * k,
                                  Sg.p + p2->sel.closure.size() * tile * k, var.p + static_cast<size_t>(m0.layout.N) * fp->bp * k,
                                  st.scratch.p + st.scratch_stride * k,
                                  st.logdet.p + fp->flow->host.logdet_doubles * k, st.status.p + k, st.ctr(k)));
    }
    if (pipelined) {
      CK(cudaMemsetAsync(st.status.p, 0xff, static_cast<size_t>(count) * sizeof(unsigned long long), s));
      std::vector<cudaEvent_t> evs;
      cudaEvent_t ready;
      CK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
      CK(cudaEventRecord(ready, s));  // the stores are allocated (stream-ordered) before the copies
      CK(cudaStreamWaitEvent(rt.upload, ready, 0));
      evs.push_back(ready);
      for (int c0 = 0; c0 < count; c0 += pipe) {
        const int c1 = std::min(count, c0 + pipe);
        for (int k = c0; k < c1; ++k)
          CK(cudaMemcpyAsync(st.A.p + T * tile * k, ms[k]->payload.p, T * tile * sizeof(double), cudaMemcpyHostToDevice,
                             rt.upload));
        cudaEvent_t ev;
        CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        CK(cudaEventRecord(ev, rt.upload));
        CK(cudaStreamWaitEvent(s, ev, 0));
        evs.push_back(ev);
        const std::vector<BaseTable> part(tables.begin() + c0, tables.begin() + c1);
        run_flow_chunked(*fp->flow, part, s);
        run_flow_chunked(*p2->flow, part, s);
      }
      tm.mark("pipelined sweeps");
      CK(cudaStreamSynchronize(s));
      for (cudaEvent_t e : evs) cudaEventDestroy(e);
    } else if (stream_up) {
      cudaEvent_t cleared, uploaded, t_start = nullptr, t_up = nullptr, t_sweep = nullptr;
      CK(cudaEventCreateWithFlags(&cleared, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&uploaded, cudaEventDisableTiming));
      const bool same = F == m0.pattern;
      // groups of columns per copy (~48 groups per matrix): fewer API calls than
      // the copy engine needs time for, while each chain waits for little more
      // than its first group
      const int N = m0.layout.N, grp = std::max(1, std::min(kOnes, (N + 47) / 48));
      if (!same) CK(cudaMemsetAsync(st.A.p, 0, T * tile * count * sizeof(double), s));
      std::function<void()> up = [&]() {
        CK(cudaStreamWaitEvent(rt.upload, cleared, 0));
        // runs of consecutive columns in the plan's upload order, <= grp per copy
        const std::vector<int>& ord = fp->flow->host.upload_order;
        std::vector<std::pair<int, int>> runs;
        for (size_t x = 0; x < ord.size();) {
          size_t y = x + 1;
          while (y < ord.size() && ord[y] == ord[y - 1] + 1 && static_cast<int>(y - x) < grp) ++y;
          runs.push_back({ord[x], ord[y - 1] + 1});
          x = y;
        }
        for (const auto& [c, ce] : runs)
          for (int k = 0; k < count; ++k) {
            double* dA = st.A.p + T * tile * k;
            const size_t t0 = static_cast<size_t>(F.col_start(c)), t1 = static_cast<size_t>(F.col_start(ce));
            if (same)
              CK(cudaMemcpyAsync(dA + t0 * tile, ms[k]->payload.p + t0 * tile, (t1 - t0) * tile * sizeof(double),
                                 cudaMemcpyHostToDevice, rt.upload));
            else
              upload_columns(*ms[k], F, c, ce, dA, rt.upload, true, false);
            CK(cudaMemcpyAsync(reinterpret_cast<int*>(st.ctr(k)) + fp->flow->host.upl + c, rt.one,
                               static_cast<size_t>(ce - c) * sizeof(int), cudaMemcpyHostToDevice, rt.upload));
          }
        CK(cudaEventRecord(uploaded, rt.upload));
        if (tm.on) CK(cudaEventRecord(t_up, rt.upload));
      };
      if (tm.on) {
        CK(cudaEventCreate(&t_start));
        CK(cudaEventCreate(&t_up));
        CK(cudaEventCreate(&t_sweep));
        CK(cudaEventRecord(t_start, s));
      }
      factor_sweep(*fp, st, s, tables, &up, cleared);
      if (tm.on) {
        CK(cudaEventRecord(t_sweep, s));
        CK(cudaEventSynchronize(t_sweep));
        CK(cudaEventSynchronize(t_up));
        float u = 0, w = 0;
        cudaEventElapsedTime(&u, t_start, t_up);
        cudaEventElapsedTime(&w, t_start, t_sweep);
        std::fprintf(stderr, "[tib timing] streamed upload done at %.3f ms, factor sweep at %.3f ms (%.1f GB/s)\n", u, w,
                     static_cast<double>(T) * tile * count * 8 / (u * 1e6));
      }
      CK(cudaStreamWaitEvent(s, uploaded, 0));
      cudaEventDestroy(cleared);
      cudaEventDestroy(uploaded);
    } else {
      tm.mark("uploads");
      factor_sweep(*fp, st, s, tables);
    }
    if (!pipelined) {
      tm.mark("factor sweep");
      phase2_sweep(*p2, s, tables);
      tm.mark("phase-2 sweep");
    }
    std::vector<double> parts(static_cast<size_t>(m0.layout.N) * fp->nb * count);
    std::vector<double> v(var.n);
    CK(cudaMemcpyAsync(parts.data(), st.logdet.p, parts.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(v.data(), var.p, v.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    check_status(st.status, count, m0.layout, s);
    tm.mark("read-back");
    const Layout& L = m0.layout;
    for (int k = 0; k < count; ++k) {
      if (logdet) logdet[k] = reduce_logdet(parts.data() + static_cast<size_t>(L.N) * fp->nb * k, L.N, fp->nb);
      if (diag)
        for (long r = 0; r < L.n; ++r)
          diag[static_cast<size_t>(k) * L.n + r] =
              v[static_cast<size_t>(L.N) * fp->bp * k + static_cast<size_t>(r / L.b) * fp->bp + static_cast<size_t>(r % L.b)];
    }
  });
}

int tib_matrix_two_chain_order(tib_matrix m, int* order, int* split) {
  return guarded([&] {
    need(m, "matrix");
    const SplitOrder so = two_chain_order(symbolic_cholesky(m->pattern).filled);
    if (split) *split = so.split;
    if (order && so.split > 0) std::copy(so.order.begin(), so.order.end(), order);
  });
}

int tib_matrix_two_chain_permuted(tib_matrix m, tib_matrix* out) {
  return guarded([&] {
    need(m, "matrix");
    if (!out) throw Error(kErrInvalidArgument, "null output handle");
    const SplitOrder so = two_chain_order(symbolic_cholesky(m->pattern).filled);
    if (so.split <= 0) throw Error(kErrInvalidArgument, "the tile pattern admits no two-chain order");
    const int b = m->layout.b;
    HostBuf hb(so.permuted.size() * static_cast<size_t>(b) * b);
    permuted_payload(*m, so, b, hb.p);
    auto* r = new tib_matrix_s;
    r->layout = m->layout;
    r->pattern = so.permuted;
    r->payload = std::move(hb);
    *out = r;
  });
}

int tib_plan_export(tib_matrix m, int preset, const long* rows, const long* cols, long ne, int which,
                    int crit_workers, int split, int batch, double* sizes, void* tasks, void* segs, void* deps,
                    void* sigs) {
  return guarded([&] {
    need(m, "matrix");
    if (which != 0 && which != 1) throw Error(kErrInvalidArgument, "which must be 0 (factor) or 1 (phase 2)");
    if (crit_workers < 1) throw Error(kErrInvalidArgument, "at least one reserved critical-queue worker");
    const FactorPlan sym = symbolic_cholesky(m->pattern);
    DataflowPlan P;
    if (which == 0) {
      // the CPU simulator runs the same decomposition as the GPU chain, with the
      // chain's steps kept as (fat / boundary) leaf tasks
      const int ug = factor_update_group(sym.filled, batch, split);
      P = batch_leaves(batch) ? build_factor_dataflow(sym.filled, crit_workers, kDeferW, false, false, false, split,
                                                      false, ug)
                              : build_factor_dataflow(sym.filled, crit_workers, kDeferW, true, false, true, split,
                                                      env_int("TIB_COARSE_SECOND", 1) != 0, ug);
    } else {
      const Closure sel =
          symbolic_inversion(select_tiles(sym.filled.layout(), sym.filled, make_request(preset, rows, cols, ne)), sym.filled);
      P = build_phase2_dataflow(sym.filled, sel, crit_workers, split, phase2_group(sym.filled, batch, split));
    }
    if (sizes) {
      sizes[0] = static_cast<double>(P.tasks.size());
      sizes[1] = P.q0.count;
      sizes[2] = static_cast<double>(P.segs.size());
      sizes[3] = static_cast<double>(P.deps.size());
      sizes[4] = static_cast<double>(P.sigs.size());
      sizes[5] = static_cast<double>(P.counters);
      sizes[6] = P.bp;
      sizes[7] = static_cast<double>(P.scratch_doubles);
      sizes[8] = P.task_flops;
      sizes[9] = sizeof(DTask);
    }
    if (tasks) std::memcpy(tasks, P.tasks.data(), P.tasks.size() * sizeof(DTask));
    if (segs) std::memcpy(segs, P.segs.data(), P.segs.size() * sizeof(Seg));
    if (deps) std::memcpy(deps, P.deps.data(), P.deps.size() * sizeof(Dep));
    if (sigs) std::memcpy(sigs, P.sigs.data(), P.sigs.size() * sizeof(int));
  });
}

}  // extern "C"

struct tib_resident_s {
  int device = 0;
  int count = 1;  // matrices (one tile pattern), run as one batch
  Layout layout;
  std::shared_ptr<FactorPlan2> fp;
  std::shared_ptr<Phase2Plan> p2;
  SweepStores st;
  DevBuf A0, Sg, var;
  std::vector<BaseTable> tables;
  double logdet = 0;
  double model_flops = 0;
  // two-chain order (one matrix): the stores hold the permuted matrix (like a
  // public call's result, Sigma stays in that order until an accessor needs it)
  std::unique_ptr<SplitCall> split;
};

extern "C" {

int tib_resident_create(tib_matrix m, int device, tib_resident* out) {
  return tib_resident_create_batch(&m, 1, device, out);
}

int tib_resident_create_batch(const tib_matrix* ms, int count, int device, tib_resident* out) {
  return guarded([&] {
    if (count < 1 || !ms) throw Error(kErrInvalidArgument, "batch needs at least one matrix");
    const MatrixObj* m = need(ms[0], "matrix");
    for (int k = 1; k < count; ++k)
      if (!(need(ms[k], "matrix")->pattern == m->pattern) || ms[k]->layout.n != m->layout.n)
        throw Error(kErrInvalidArgument, "batched matrices must share one tile pattern");
    DeviceRt& rt = runtime(device);
    cudaStream_t s = rt.stream;
    auto r = std::make_unique<tib_resident_s>();
    r->device = device;
    r->count = count;
    r->layout = m->layout;
    // a single matrix runs in the two-chain order (bit-for-bit the work of the
    // public call, which uses it too)
    const FactorPlan natural = symbolic_cholesky(m->pattern);
    Request req;
    req.preset = kFactorPattern;
    {
      auto sc = std::make_unique<SplitCall>();
      if (count == 1 && split_call(*m, req, *sc)) r->split = std::move(sc);
    }
    const SplitOrder* so = r->split ? &r->split->so : nullptr;
    r->fp = so ? factor_plan_for(so->permuted, device, s, so->split) : factor_plan_for(m->pattern, device, s, -1, count);
    const Pattern& F = r->fp->sym.filled;
    const Closure sel = symbolic_inversion(select_tiles(F.layout(), F, req), F);
    r->p2 = so ? phase2_plan_for(F, sel, device, s, crit_split_p2(F, so->split), so->split)
               : phase2_plan_for(F, sel, device, s, -1, -1, count);
    // the reference's task model counts the reference's own (natural) order
    const Closure sel_nat = symbolic_inversion(select_tiles(natural.filled.layout(), natural.filled, req), natural.filled);
    const Flops fl = count_flops(natural, &sel_nat);
    r->model_flops = fl.total() * count;
    const size_t tile = static_cast<size_t>(r->fp->bp) * r->fp->bp;
    const size_t T = F.size(), C = r->p2->sel.closure.size(), nv = static_cast<size_t>(m->layout.N) * r->fp->bp;
    alloc_factor_stores(r->st, *r->fp, count, device, s, r->p2->flow->host.counters,
                        r->p2->flow->host.scratch_doubles);
    r->A0 = DevBuf(T * tile * count, device, s);
    for (int k = 0; k < count; ++k) {
      if (so) {
        HostBuf hb(T * tile);
        permuted_payload(*ms[k], *so, r->fp->bp, hb.p);
        CK(cudaMemcpyAsync(r->A0.p + T * tile * k, hb.p, T * tile * sizeof(double), cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));
      } else {
        upload_matrix(*ms[k], F, r->fp->bp, r->A0.p + T * tile * k, s);
      }
    }
    r->Sg = DevBuf(C * tile * count, device, s);
    r->var = DevBuf(nv * count, device, s);

    for (int k = 0; k < count; ++k)
      r->tables.push_back(make_table(r->st.A.p + T * tile * k, r->st.L.p + T * tile * k, r->st.P1.p + T * tile * k,
                                     r->Sg.p + C * tile * k, r->var.p + nv * k,
                                     r->st.scratch.p + r->st.scratch_stride * k,
                                     r->st.logdet.p + r->fp->flow->host.logdet_doubles * k, r->st.status.p + k,
                                     r->st.ctr(k)));
    CK(cudaStreamSynchronize(s));
    *out = r.release();
  });
}

int tib_resident_run(tib_resident r, int reps, double* ms_total, double* ms_factor, double* ms_phase2) {
  return guarded([&] {
    need(r, "resident");
    if (reps < 1) throw Error(kErrInvalidArgument, "reps >= 1");
    DeviceRt& rt = runtime(r->device);
    cudaStream_t s = rt.stream;
    std::vector<cudaEvent_t> ev(static_cast<size_t>(3 * reps));
    for (auto& e : ev) CK(cudaEventCreate(&e));
    for (int it = 0; it < reps; ++it) {
      CK(cudaMemcpyAsync(r->st.A.p, r->A0.p, r->A0.n * sizeof(double), cudaMemcpyDeviceToDevice, s));
      CK(cudaEventRecord(ev[3 * it], s));
      factor_sweep(*r->fp, r->st, s, r->tables);
      CK(cudaEventRecord(ev[3 * it + 1], s));
      phase2_sweep(*r->p2, s, r->tables);
      CK(cudaEventRecord(ev[3 * it + 2], s));
    }
    CK(cudaEventSynchronize(ev.back()));
    double total = 0;
    float tf = 0, tp = 0;
    for (int it = 0; it < reps; ++it) {
      CK(cudaEventElapsedTime(&tf, ev[3 * it], ev[3 * it + 1]));
      CK(cudaEventElapsedTime(&tp, ev[3 * it + 1], ev[3 * it + 2]));
      total += tf + tp;
    }
    for (auto& e : ev) cudaEventDestroy(e);
    std::vector<double> parts(r->fp->flow->host.logdet_doubles);  // matrix 0's
    CK(cudaMemcpyAsync(parts.data(), r->st.logdet.p, parts.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    check_status(r->st.status, r->count, r->layout, s);
    r->logdet = reduce_logdet(parts.data(), r->layout.N, r->fp->nb);
    if (ms_total) *ms_total = total;
    if (ms_factor) *ms_factor = tf;
    if (ms_phase2) *ms_phase2 = tp;
  });
}

int tib_resident_info(tib_resident r, double* model, double* executed, double* logdet, long* launches) {
  return guarded([&] {
    need(r, "resident");
    if (model) *model = r->model_flops;
    if (executed) *executed = (r->fp->flow->host.task_flops + r->p2->flow->host.task_flops) * r->count;
    if (logdet) *logdet = r->logdet;
    // per sweep: scheduler init + the persistent dataflow kernel (+ the zero-strip
    // kernel when the plan has strips)
    if (launches)
      *launches = 4 + (r->fp->flow->host.zero.empty() ? 0 : 1) + (r->p2->flow->host.zero.empty() ? 0 : 1);
  });
}

int tib_resident_free(tib_resident r) {
  delete r;
  return kOk;
}

int tib_bench_resident(tib_matrix m, int device, int reps, int warmup, double* ms_per_rep, double* ms_factor,
                       double* ms_phase2, double* logdet) {
  tib_resident r = nullptr;
  int st = tib_resident_create(m, device, &r);
  if (st != kOk) return st;
  double tot = 0;
  if (warmup > 0) st = tib_resident_run(r, warmup, &tot, nullptr, nullptr);
  if (st == kOk) st = tib_resident_run(r, reps, &tot, ms_factor, ms_phase2);
  if (st == kOk) {
    if (ms_per_rep) *ms_per_rep = tot / reps;
    if (logdet) *logdet = r->logdet;
  }
  tib_resident_free(r);
  return st;
}

}  // extern "C"
