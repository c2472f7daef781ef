// Host-side symbolic planner for the B200 tile Cholesky + selected inversion.
//
// Integer-only work that decides WHICH tiles exist and in WHAT order they are
// touched.  Every function here is a from-scratch restatement of the
// reference's symbolic layer and must produce bit-identical tile sets and
// orders (tests compare them tile-for-tile with oracle/_ref):
//
//   build_layout          <- proj/src/layout.cpp:11-20
//   map_entry_to_tile     <- proj/src/layout.cpp:22-34
//   Pattern               <- TilePattern, proj/src/layout.cpp:36-53
//   symbolic_fill         <- proj/src/layout.cpp:62-87
//   band_arrow_pattern    <- proj/src/layout.cpp:89-100
//   factor task counts    <- symbolic_cholesky, proj/src/cholesky.cpp:17-49
//   select_tiles          <- proj/src/selinv.cpp:51-83
//   symbolic_inversion    <- proj/src/selinv.cpp:85-150
//   extract (entry order) <- extract_entries, proj/src/selinv.cpp:387-439
//   payload_checksum      <- proj/src/storage.cpp:34-48
//   task graph analyzer   <- proj/src/dag.cpp:79-342 (dag.cpp)
//
// Numeric payloads never live here: the device store (store.cuh) owns them.
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace tib {

// ---- error convention (mirrors proj/include/tileinv/errors.hpp:8-58) --------
enum Status : int {
  kOk = 0,
  kErrGeneric = 1,        // tileinv::Error
  kErrInvalidArgument = 2,
  kErrNotSpd = 3,
  kErrSingularTile = 4,
  kErrContract = 5,
  kErrConsistency = 6,
  kErrStructure = 7,
  kErrParse = 8,
  kErrFormat = 9,
  kErrCuda = 10,
};

struct Error : std::runtime_error {
  int status;
  Error(int st, const std::string& msg) : std::runtime_error(msg), status(st) {}
};
struct NotSpd : Error {
  long pivot;
  int tile_i, tile_j;
  NotSpd(const std::string& msg, long p, int ti, int tj)
      : Error(kErrNotSpd, msg), pivot(p), tile_i(ti), tile_j(tj) {}
};

// ---- layout ----------------------------------------------------------------
struct Layout {
  long n = 0;
  int b = 0;
  int N = 0;
  long n_padded = 0;
};
Layout build_layout(long n, int b);

struct Coord {
  int i = 0, j = 0;
  bool operator==(const Coord& o) const { return i == o.i && j == o.j; }
};
inline bool tile_before(const Coord& a, const Coord& b) {
  return a.j != b.j ? a.j < b.j : a.i < b.i;
}
inline uint64_t tile_key(int i, int j) {
  return (static_cast<uint64_t>(static_cast<uint32_t>(j)) << 32) | static_cast<uint32_t>(i);
}

struct Address {
  Coord tile;
  int row_off = 0, col_off = 0;
};
Address map_entry_to_tile(const Layout& L, long r, long c);

// Lower-triangular tile pattern.  Tiles are kept sorted column-major, which is
// also the SLOT order of the packed device store: slot(i, j) is the position
// of (i, j) in tiles(), so column j's tiles are contiguous (diagonal first,
// then ascending rows) and a column panel of m off-diagonal b x b row-major
// tiles is one row-major (m*b) x b matrix in HBM.
class Pattern {
 public:
  Pattern() = default;
  Pattern(Layout layout, std::vector<Coord> tiles);

  const Layout& layout() const { return layout_; }
  const std::vector<Coord>& tiles() const { return tiles_; }
  // ascending rows of column j (includes j itself when stored)
  const int* rows_begin(int j) const { return rows_.data() + col_start_[j]; }
  const int* rows_end(int j) const { return rows_.data() + col_start_[j + 1]; }
  int col_count(int j) const { return static_cast<int>(col_start_[j + 1] - col_start_[j]); }
  long col_start(int j) const { return col_start_[j]; }
  // slot of (i, j) or -1
  long slot(int i, int j) const;
  bool has(int i, int j) const { return slot(i, j) >= 0; }
  size_t size() const { return tiles_.size(); }
  bool has_all_diagonals() const;
  bool operator==(const Pattern& o) const;

 private:
  Layout layout_;
  std::vector<Coord> tiles_;
  std::vector<long> col_start_;  // N + 1
  std::vector<int> rows_;        // rows per column, ascending
};

Pattern symbolic_fill(const Pattern& p);
Pattern band_arrow_pattern(const Layout& L, int band_b);

// ---- factorization plan summary ---------------------------------------------
// The reference's FactorPlan (cholesky.hpp:11-26) is a task list; the device
// sweep only needs the filled pattern (per-column window = neighbours > j), so
// the plan keeps the pattern plus the task counts used for FLOP accounting.
struct FactorCounts {
  long potrf = 0, trsm = 0, syrk = 0, gemm = 0;
};
struct FactorPlan {
  Pattern filled;
  FactorCounts counts;
};
FactorPlan symbolic_cholesky(const Pattern& pattern);

// ---- selection ----------------------------------------------------------------
enum Preset : int { kNone = 0, kDiagonal = 1, kFactorPattern = 2, kAll = 3 };
struct Request {
  int preset = kFactorPattern;
  std::vector<std::pair<long, long>> entries;
};
std::vector<Coord> select_tiles(const Layout& L, const Pattern& factor, const Request& req);

struct ColumnWork {
  int col = 0;
  std::vector<int> offdiag_rows;  // descending
  bool diagonal = false;
};
struct Closure {
  std::vector<Coord> requested;  // sorted column-major
  Pattern closure;
  std::vector<ColumnWork> columns;  // descending column order
  bool growth_warning = false;
};
Closure symbolic_inversion(const std::vector<Coord>& requested, const Pattern& factor);

// Task-model FLOPs: POTRF b^3/3, TRSM b^3, SYRK b^3, GEMM 2b^3,
// TRTRI b^3/3, TRMM b^3, LAUUM b^3/3, phase-2 GEMM 2b^3 per (target, k).
struct Flops {
  double factorize = 0, phase1 = 0, phase2 = 0;
  double total() const { return factorize + phase1 + phase2; }
};
Flops count_flops(const FactorPlan& plan, const Closure* sel);
double phase2_flops(const Pattern& factor, const Closure& sel);

// Canonical entry list of a request (extract_entries order).  Calls
// visit(r, c) for each entry; throws like the reference.
template <class F>
void for_each_request_entry(const Layout& L, const Pattern& closure,
                            const std::vector<Coord>& requested, const Request& req, F&& visit);

uint64_t fnv1a_keys(const std::vector<Coord>& tiles);

// ---- two-chain elimination order (the device's single-matrix path) ----------
// The reference eliminates tile columns 0 .. N-1, one sequential chain of
// diagonal factorizations.  For a band + arrow tile pattern (band width s
// tiles, arrow = the trailing full tile rows) the order
//     [I_0 ascending, I_1 descending, S, arrow]
// with I_0 = [0, h), S = [h, h + s), I_1 = [h + s, M) (M = band columns) has
// two independent chains -- I_1 eliminated from its far end meets the
// separator S last, like I_0 -- and, at tile granularity, no fill beyond the
// matrix's own (checked symbolically).  order[k] = original tile of position
// k; split = first position of the second chain (I_1 then S then arrow).
struct SplitOrder {
  std::vector<int> order, pos;  // pos = inverse permutation
  int split = -1;               // -1: no admissible split
  Pattern permuted;             // the filled pattern in the new order
};
SplitOrder two_chain_order(const Pattern& filled);
// Tile (i, j) of the permuted matrix (i >= j) -> original tile and whether the
// stored original tile is its transpose.
inline Coord split_source(const SplitOrder& so, int i, int j, bool& transposed) {
  const int a = so.order[static_cast<size_t>(i)], b = so.order[static_cast<size_t>(j)];
  transposed = a < b;
  return transposed ? Coord{b, a} : Coord{a, b};
}

// ---- task-graph / complexity analyzer (dag.cpp; reference dag.hpp:12-77) ------
struct DagNode {
  int kind = 0;  // 0 TRSM_INV, 1 TRMM, 2 LAUUM, 3 GEMM (the reference's rank order)
  int i = 0, j = 0;
  int k = -1;    // accumulation term of a GEMM
  int phase = 1;
};
struct TaskGraph {
  int n_tiles = 0;
  int band_b = -1;  // band width when closure == factor == band+arrow, else -1
  std::vector<DagNode> nodes;  // canonical order; ids are indices
  std::vector<std::pair<int, int>> edges;
  std::vector<int> core_of;    // empty until assign_task_cores
};
struct KernelReport {
  int n_tiles = 0, band_b = -1, critical_path = 0;
  long long trsm = 0, trmm = 0, lauum = 0, gemm_actual = 0, gemm_predicted = -1;
  bool match = false;
};
TaskGraph build_task_graph(const Closure& sel, const Pattern& factor);
TaskGraph band_arrow_task_graph(int n_tiles, int band_b);
void assign_task_cores(TaskGraph& g, int cores);
int task_graph_critical_path(const TaskGraph& g);
std::string task_graph_dot(const TaskGraph& g);
long long predict_gemm_count(int n_tiles, int band_b);
KernelReport count_task_kernels(const TaskGraph& g);


// FNV-1a over (tile key, b*b payload) in column-major tile order.
struct Fnv {
  uint64_t h = 1469598103934665603ull;
  void mix(const void* data, size_t len) {
    const unsigned char* p = static_cast<const unsigned char*>(data);
    for (size_t i = 0; i < len; ++i) {
      h ^= p[i];
      h *= 1099511628211ull;
    }
  }
};

// ---- input side: generator and Matrix Market ---------------------------------
// Host tiled symmetric matrix in the reference's value semantics: pattern +
// payload per pattern slot (b*b row-major, diagonal tiles lower only).
struct HostMatrix {
  Layout layout;
  Pattern pattern;
  std::vector<double> payload;  // pattern.size() * b * b
};

// Bit-exact restatement of generate_arrowhead (proj/src/matgen.cpp:59-120).
HostMatrix generate_arrowhead(long n, long w, long t, double density, uint64_t seed, int b);
// Its tile pattern at density 1 (no values; the device generator fills them).
Pattern arrowhead_pattern(long n, long w, long t, int b);
// STLS tile files (tileio.cpp; reference tileio.cpp:30-94).  payload: per
// pattern slot, b*b row-major.
struct TileFileData {
  Layout layout;
  int phase = 0;  // PhaseTag: 0 matrix, 1 factor, 2 phase-1, 3 selected inverse
  Pattern pattern;
  std::vector<double> payload;
};
TileFileData read_tile_file(const std::string& path);
void write_tile_file(const std::string& path, const Layout& layout, int phase, const Pattern& pattern,
                     const double* payload);

// BASELINE config 4: AR1(rho, nt) (x) SPDE(nx x ny lattice) latent field plus p
// fixed effects, as the joint INLA precision (kronecker.cpp).
HostMatrix generate_kronecker(int nt, int nx, int ny, int p, double rho, double kappa2, double tau, double tau_y,
                              double q_beta, uint64_t seed, int b);
HostMatrix matrix_from_dense(long n, int b, const double* a);  // module.cpp:46-74
HostMatrix matrix_from_tiles(long n, int b, long count, const int* ti, const int* tj,
                             const double* payload);
HostMatrix read_matrix_market(const std::string& text, int b);   // matgen.cpp:208-319
std::string write_matrix_market(const HostMatrix& m);             // matgen.cpp:146-184

// ---- implementation of the template --------------------------------------------
template <class F>
void for_each_request_entry(const Layout& L, const Pattern& closure,
                            const std::vector<Coord>& requested, const Request& req, F&& visit) {
  const long n = L.n;
  const int b = L.b;
  switch (req.preset) {
    case kDiagonal:
      for (long r = 0; r < n; ++r) visit(r, r);
      break;
    case kAll:
      for (long c = 0; c < n; ++c)
        for (long r = c; r < n; ++r) visit(r, c);
      break;
    case kFactorPattern: {
      const Pattern rq(L, requested);
      for (int j = 0; j < L.N; ++j) {
        for (int oc = 0; oc < b; ++oc) {
          const long c = static_cast<long>(j) * b + oc;
          if (c >= n) break;
          for (const int* it = rq.rows_begin(j); it != rq.rows_end(j); ++it) {
            for (int orr = 0; orr < b; ++orr) {
              const long r = static_cast<long>(*it) * b + orr;
              if (r >= n) break;
              if (r < c) continue;
              visit(r, c);
            }
          }
        }
      }
      break;
    }
    default: {
      std::vector<uint64_t> seen;
      seen.reserve(req.entries.size());
      for (const auto& [r, c] : req.entries) {
        if (r < 0 || c < 0 || r >= n || c >= n)
          throw Error(kErrInvalidArgument, "requested entry (" + std::to_string(r) + ", " +
                                               std::to_string(c) + ") outside the matrix");
      }
      // keep request order minus duplicates (selinv.cpp:410-425)
      std::vector<std::pair<uint64_t, size_t>> keys;
      keys.reserve(req.entries.size());
      for (size_t k = 0; k < req.entries.size(); ++k)
        keys.push_back({static_cast<uint64_t>(req.entries[k].first) * static_cast<uint64_t>(n) +
                            static_cast<uint64_t>(req.entries[k].second),
                        k});
      std::vector<char> keep(req.entries.size(), 1);
      std::sort(keys.begin(), keys.end());
      for (size_t k = 1; k < keys.size(); ++k)
        if (keys[k].first == keys[k - 1].first) keep[keys[k].second] = 0;
      for (size_t k = 0; k < req.entries.size(); ++k)
        if (keep[k]) visit(req.entries[k].first, req.entries[k].second);
      break;
    }
  }
  (void)closure;
}

}  // namespace tib
