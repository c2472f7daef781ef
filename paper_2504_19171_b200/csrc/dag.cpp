// Task-graph / complexity analyzer of the selected inversion, host side.
//
// Restates the reference's analysis layer (proj/src/dag.cpp:79-342,
// proj/include/tileinv/dag.hpp:12-77) on this library's symbolic types:
// one node per kernel invocation of the two inversion phases at tile
// granularity -- TRSM_INV per factor diagonal, TRMM per off-diagonal factor
// tile, LAUUM per closure diagonal, GEMM per (target, k) accumulation term --
// with the reference's canonical node order, edge set, critical path, DOT text
// and closed-form GEMM prediction, so reports and DOT files are byte-identical.
//
// It is analysis only (off the device path).  The library also uses it to
// cross-check the dataflow planner: the phase-2 GEMM terms the GPU plan
// executes must equal this graph's GEMM node count (tests/test_dag.py).
#include <algorithm>
#include <cstdint>
#include <sstream>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "planner.hpp"

namespace tib {

// ---- node identity ---------------------------------------------------------
// kinds in rank order (dag.cpp:17-25): the rank is the tie-break of the order
enum DagKind : int { kTrsmInv = 0, kTrmm = 1, kLauum = 2, kGemm = 3 };
static const char* kKindName[4] = {"TRSM_INV", "TRMM", "LAUUM", "GEMM"};

// (phase, kind, i, j, k) in one word: tiles < 2^20, k = -1 stored as 0
static uint64_t node_key(int phase, int kind, int i, int j, int k) {
  return (static_cast<uint64_t>(phase - 1) << 63) | (static_cast<uint64_t>(kind) << 61) |
         (static_cast<uint64_t>(i) << 41) | (static_cast<uint64_t>(j) << 21) | static_cast<uint64_t>(k + 1);
}

// canonical order (dag.hpp:58-59): phase ascending, column descending, row
// descending, kernel rank, accumulation term ascending
static bool canonical_before(const DagNode& a, const DagNode& b) {
  if (a.phase != b.phase) return a.phase < b.phase;
  if (a.j != b.j) return a.j > b.j;
  if (a.i != b.i) return a.i > b.i;
  if (a.kind != b.kind) return a.kind < b.kind;
  return a.k < b.k;
}

namespace {

// successor lists + indegrees of a graph (edges are unique)
struct Adjacency {
  std::vector<int> start, to, indeg;
  explicit Adjacency(const TaskGraph& g) {
    const size_t n = g.nodes.size();
    start.assign(n + 1, 0);
    indeg.assign(n, 0);
    for (const auto& e : g.edges) {
      ++start[static_cast<size_t>(e.first) + 1];
      ++indeg[static_cast<size_t>(e.second)];
    }
    for (size_t v = 0; v < n; ++v) start[v + 1] += start[v];
    to.resize(g.edges.size());
    std::vector<int> fill(start.begin(), start.end() - 1);
    for (const auto& e : g.edges) to[static_cast<size_t>(fill[static_cast<size_t>(e.first)]++)] = e.second;
  }
};

// Longest path in nodes (Kahn order); throws on a cycle like dag.cpp:46-77.
int longest_path_nodes(const TaskGraph& g) {
  const int n = static_cast<int>(g.nodes.size());
  if (n == 0) return 0;
  Adjacency adj(g);
  std::vector<int> depth(static_cast<size_t>(n), 1), queue;
  queue.reserve(static_cast<size_t>(n));
  for (int v = 0; v < n; ++v)
    if (adj.indeg[static_cast<size_t>(v)] == 0) queue.push_back(v);
  int best = 0;
  for (size_t q = 0; q < queue.size(); ++q) {
    const int v = queue[q];
    best = std::max(best, depth[static_cast<size_t>(v)]);
    for (int e = adj.start[static_cast<size_t>(v)]; e < adj.start[static_cast<size_t>(v) + 1]; ++e) {
      const int w = adj.to[static_cast<size_t>(e)];
      depth[static_cast<size_t>(w)] = std::max(depth[static_cast<size_t>(w)], depth[static_cast<size_t>(v)] + 1);
      if (--adj.indeg[static_cast<size_t>(w)] == 0) queue.push_back(w);
    }
  }
  if (static_cast<int>(queue.size()) != n) throw Error(kErrConsistency, "task graph contains a cycle");
  return best;
}

}  // namespace

// dag.cpp:79-190
TaskGraph build_task_graph(const Closure& sel, const Pattern& factor) {
  const Layout& L = factor.layout();
  const int N = L.N;
  if (sel.closure.layout().N != N) throw Error(kErrContract, "selection closure built for a different tile grid");
  if (N >= (1 << 20)) throw Error(kErrInvalidArgument, "task graph limited to fewer than 2^20 tile columns");
  // rows below the diagonal of factor column j: the accumulation terms k > j
  auto terms_of = [&](int j) {
    std::vector<int> t;
    for (const int* r = factor.rows_begin(j); r != factor.rows_end(j); ++r)
      if (*r > j) t.push_back(*r);
    return t;
  };

  TaskGraph g;
  g.n_tiles = N;
  for (int i = 0; i < N; ++i) {
    g.nodes.push_back({kTrsmInv, i, i, -1, 1});
    for (int k : terms_of(i)) g.nodes.push_back({kTrmm, k, i, -1, 1});
  }
  for (const ColumnWork& cw : sel.columns) {
    const std::vector<int> t = terms_of(cw.col);
    for (int row : cw.offdiag_rows)
      for (int k : t) g.nodes.push_back({kGemm, row, cw.col, k, 2});
    if (cw.diagonal) {
      g.nodes.push_back({kLauum, cw.col, cw.col, -1, 2});
      for (int k : t) g.nodes.push_back({kGemm, cw.col, cw.col, k, 2});
    }
  }
  std::sort(g.nodes.begin(), g.nodes.end(), canonical_before);

  std::unordered_map<uint64_t, int> id_of;
  id_of.reserve(g.nodes.size() * 2);
  for (size_t v = 0; v < g.nodes.size(); ++v) {
    const DagNode& d = g.nodes[v];
    id_of.emplace(node_key(d.phase, d.kind, d.i, d.j, d.k), static_cast<int>(v));
  }
  auto id = [&](int phase, int kind, int i, int j, int k) {
    const auto it = id_of.find(node_key(phase, kind, i, j, k));
    if (it == id_of.end()) throw Error(kErrConsistency, "dangling task reference");
    return it->second;
  };
  // the task that finalises Sigma(i, j): its last accumulation term, else the
  // LAUUM of a diagonal, else none (the tile stays zero)
  auto last_writer = [&](int i, int j) {
    const std::vector<int> t = terms_of(j);
    if (!t.empty()) return id(2, kGemm, i, j, t.back());
    if (i == j) return id(2, kLauum, j, j, -1);
    return -1;
  };

  for (int i = 0; i < N; ++i) {
    const int tr = id(1, kTrsmInv, i, i, -1);
    for (int k : terms_of(i)) g.edges.emplace_back(tr, id(1, kTrmm, k, i, -1));
  }
  for (const ColumnWork& cw : sel.columns) {
    const int i = cw.col;
    const std::vector<int> t = terms_of(i);
    // one accumulation chain per target: (prev term) -> term, W(k, i) -> term,
    // Sigma operand's last writer -> term
    auto chain = [&](int row, int prev) {
      for (int k : t) {
        const int gm = id(2, kGemm, row, i, k);
        if (prev >= 0) g.edges.emplace_back(prev, gm);
        g.edges.emplace_back(id(1, kTrmm, k, i, -1), gm);
        const int op = last_writer(std::max(row, k), std::min(row, k));
        if (op >= 0) g.edges.emplace_back(op, gm);
        prev = gm;
      }
    };
    for (int row : cw.offdiag_rows) chain(row, -1);
    if (cw.diagonal) {
      const int la = id(2, kLauum, i, i, -1);
      g.edges.emplace_back(id(1, kTrsmInv, i, i, -1), la);
      chain(i, la);
    }
  }
  std::sort(g.edges.begin(), g.edges.end());
  g.edges.erase(std::unique(g.edges.begin(), g.edges.end()), g.edges.end());

  // band tag (dag.cpp:163-176): the closure IS the factor pattern and that is
  // a band+arrow pattern of some width (N for the dense grid)
  if (sel.closure == factor) {
    if (sel.closure.size() == static_cast<size_t>(N) * (static_cast<size_t>(N) + 1) / 2) {
      g.band_b = N;
    } else {
      int bw = 1;
      for (const Coord& c : sel.closure.tiles())
        if (c.i != c.j && c.i != N - 1) bw = std::max(bw, c.i - c.j + 1);
      if (band_arrow_pattern(L, bw) == sel.closure) g.band_b = bw;
    }
  }
  longest_path_nodes(g);  // acyclicity check
  return g;
}

// dag.cpp:192-205 -- a scalar-free grid: layout (n = N, b = 1)
TaskGraph band_arrow_task_graph(int n_tiles, int band_b) {
  if (n_tiles < 1) throw Error(kErrInvalidArgument, "tile count must be at least 1");
  if (band_b < 1 || band_b > n_tiles) throw Error(kErrInvalidArgument, "band width must lie in [1, n_tiles]");
  const Pattern p = band_arrow_pattern(build_layout(n_tiles, 1), band_b);
  TaskGraph g = build_task_graph(symbolic_inversion(p.tiles(), p), p);
  g.band_b = band_b;
  return g;
}

// dag.cpp:207-214: column c belongs to core (N - 1 - c) mod P
void assign_task_cores(TaskGraph& g, int cores) {
  if (cores < 1) throw Error(kErrInvalidArgument, "core count must be at least 1");
  g.core_of.resize(g.nodes.size());
  for (size_t v = 0; v < g.nodes.size(); ++v) g.core_of[v] = (g.n_tiles - 1 - g.nodes[v].j) % cores;
}

int task_graph_critical_path(const TaskGraph& g) { return longest_path_nodes(g); }

// dag.cpp:247-270
std::string task_graph_dot(const TaskGraph& g) {
  static const char* kColors[8] = {"#a6cee3", "#1f78b4", "#b2df8a", "#33a02c",
                                   "#fb9a99", "#e31a1c", "#fdbf6f", "#ff7f00"};
  std::ostringstream os;
  os << "digraph tasks {\n  rankdir=TB;\n  node [shape=box];\n";
  for (size_t v = 0; v < g.nodes.size(); ++v) {
    const DagNode& d = g.nodes[v];
    os << "  n" << v << " [label=\"" << kKindName[d.kind] << "(" << d.i << "," << d.j << ")\"";
    if (!g.core_of.empty()) os << ", style=filled, fillcolor=\"" << kColors[g.core_of[v] % 8] << "\"";
    os << "];\n";
  }
  for (const auto& e : g.edges) os << "  n" << e.first << " -> n" << e.second << ";\n";
  os << "}\n";
  return os.str();
}

// dag.cpp:272-280: closed-form GEMM count of the band+arrow recursion,
// N_GEMM = (N-B)B + B(B-1)/2 + B^2(N-B-1) + B(B+1)(2B+1)/6
long long predict_gemm_count(int n_tiles, int band_b) {
  if (n_tiles < 1) throw Error(kErrInvalidArgument, "tile count must be at least 1");
  if (band_b < 1 || band_b > n_tiles) throw Error(kErrInvalidArgument, "band width must lie in [1, n_tiles]");
  const long long n = n_tiles, b = band_b;
  return (n - b) * b + b * (b - 1) / 2 + b * b * (n - b - 1) + b * (b + 1) * (2 * b + 1) / 6;
}

// dag.cpp:282-340: kernel counts of the graph against the closed form
KernelReport count_task_kernels(const TaskGraph& g) {
  KernelReport r;
  r.n_tiles = g.n_tiles;
  r.band_b = g.band_b;
  for (const DagNode& d : g.nodes) {
    if (d.kind == kTrsmInv) ++r.trsm;
    else if (d.kind == kTrmm) ++r.trmm;
    else if (d.kind == kLauum) ++r.lauum;
    else ++r.gemm_actual;
  }
  r.critical_path = longest_path_nodes(g);
  if (g.band_b > 0) {
    // predicted: TRSM_INV = LAUUM = N, TRMM = off-diagonal tiles of the band+arrow pattern
    const int N = g.n_tiles;
    const bool dense = g.band_b == N;
    const long long trmm = dense ? static_cast<long long>(N) * (N - 1) / 2
                                 : static_cast<long long>(band_arrow_pattern(build_layout(N, 1), g.band_b).size()) - N;
    r.gemm_predicted = predict_gemm_count(N, g.band_b);
    r.match = r.gemm_actual == r.gemm_predicted && r.trsm == N && r.trmm == trmm && r.lauum == N;
  }
  return r;
}

}  // namespace tib
