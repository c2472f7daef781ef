// Host symbolic planner: see planner.hpp for the reference file:line each
// routine restates.  Integer code only; bit-identical tile sets and orders.
#include "planner.hpp"

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <set>
#include <sstream>

namespace tib {

// layout.cpp:11-20
Layout build_layout(long n, int b) {
  if (n < 1) throw Error(kErrInvalidArgument, "matrix dimension must be positive, got " + std::to_string(n));
  if (b < 1) throw Error(kErrInvalidArgument, "tile size must be positive, got " + std::to_string(b));
  Layout L;
  L.n = n;
  L.b = b;
  L.N = static_cast<int>((n + b - 1) / b);
  L.n_padded = static_cast<long>(L.N) * b;
  return L;
}

// layout.cpp:22-34
Address map_entry_to_tile(const Layout& L, long r, long c) {
  if (r < 0 || c < 0 || r >= L.n || c >= L.n)
    throw Error(kErrInvalidArgument, "entry (" + std::to_string(r) + ", " + std::to_string(c) +
                                         ") outside matrix of dimension " + std::to_string(L.n));
  if (r < c) std::swap(r, c);
  Address a;
  a.tile.i = static_cast<int>(r / L.b);
  a.tile.j = static_cast<int>(c / L.b);
  a.row_off = static_cast<int>(r % L.b);
  a.col_off = static_cast<int>(c % L.b);
  return a;
}

// layout.cpp:36-53: validate, sort column-major, dedupe, per-column rows.
Pattern::Pattern(Layout layout, std::vector<Coord> tiles) : layout_(layout), tiles_(std::move(tiles)) {
  for (const Coord& t : tiles_) {
    if (t.j < 0 || t.j > t.i || t.i >= layout_.N)
      throw Error(kErrStructure, "tile (" + std::to_string(t.i) + ", " + std::to_string(t.j) +
                                     ") outside the lower triangle of a " +
                                     std::to_string(layout_.N) + "-tile grid");
  }
  std::sort(tiles_.begin(), tiles_.end(), tile_before);
  tiles_.erase(std::unique(tiles_.begin(), tiles_.end()), tiles_.end());
  col_start_.assign(static_cast<size_t>(layout_.N) + 1, 0);
  rows_.resize(tiles_.size());
  for (const Coord& t : tiles_) ++col_start_[static_cast<size_t>(t.j) + 1];
  for (int j = 0; j < layout_.N; ++j) col_start_[j + 1] += col_start_[j];
  for (size_t k = 0; k < tiles_.size(); ++k) rows_[k] = tiles_[k].i;
}

long Pattern::slot(int i, int j) const {
  if (j < 0 || j >= layout_.N) return -1;
  const int* b = rows_begin(j);
  const int* e = rows_end(j);
  const int* it = std::lower_bound(b, e, i);
  if (it == e || *it != i) return -1;
  return col_start_[j] + (it - b);
}

bool Pattern::has_all_diagonals() const {
  for (int i = 0; i < layout_.N; ++i)
    if (!has(i, i)) return false;
  return true;
}

bool Pattern::operator==(const Pattern& o) const { return tiles_ == o.tiles_; }

// layout.cpp:62-87: one ascending pass; additions land in later columns.
Pattern symbolic_fill(const Pattern& p) {
  const int N = p.layout().N;
  for (int i = 0; i < N; ++i)
    if (!p.has(i, i))
      throw Error(kErrStructure, "symbolic fill requires every diagonal tile, column " +
                                     std::to_string(i) + " has none");
  std::vector<std::set<int>> cols(static_cast<size_t>(N));
  for (const Coord& t : p.tiles()) cols[static_cast<size_t>(t.j)].insert(t.i);
  for (int k = 0; k < N; ++k) {
    std::vector<int> below(cols[static_cast<size_t>(k)].upper_bound(k), cols[static_cast<size_t>(k)].end());
    for (size_t a = 0; a < below.size(); ++a)
      for (size_t c = a; c < below.size(); ++c) cols[static_cast<size_t>(below[a])].insert(below[c]);
  }
  std::vector<Coord> tiles;
  for (int j = 0; j < N; ++j)
    for (int i : cols[static_cast<size_t>(j)]) tiles.push_back({i, j});
  return Pattern(p.layout(), std::move(tiles));
}

// layout.cpp:89-100 (band_b counts the diagonal: offsets <= band_b - 1).
Pattern band_arrow_pattern(const Layout& L, int band_b) {
  if (band_b < 1 || band_b > L.N)
    throw Error(kErrInvalidArgument, "band width " + std::to_string(band_b) + " outside [1, " +
                                         std::to_string(L.N) + "]");
  std::vector<Coord> tiles;
  for (int j = 0; j < L.N; ++j) {
    for (int i = j; i < L.N && i - j <= band_b - 1; ++i) tiles.push_back({i, j});
    if (L.N - 1 - j > band_b - 1) tiles.push_back({L.N - 1, j});
  }
  return Pattern(L, std::move(tiles));
}

// cholesky.cpp:17-49.  Per column j: POTRF, TRSM per row > j, and for each
// pair a >= b' of rows > j a SYRK (a == b') or GEMM.
FactorPlan symbolic_cholesky(const Pattern& pattern) {
  FactorPlan plan;
  plan.filled = symbolic_fill(pattern);
  if (!plan.filled.has_all_diagonals())
    throw Error(kErrStructure, "factorization needs every diagonal tile present");
  const int N = plan.filled.layout().N;
  for (int j = 0; j < N; ++j) {
    const long m = plan.filled.col_count(j) - 1;  // rows > j (diagonal is first)
    plan.counts.potrf += 1;
    plan.counts.trsm += m;
    plan.counts.syrk += m;
    plan.counts.gemm += m * (m - 1) / 2;
  }
  return plan;
}

// selinv.cpp:51-83
std::vector<Coord> select_tiles(const Layout& L, const Pattern& factor, const Request& req) {
  std::vector<Coord> tiles;
  switch (req.preset) {
    case kDiagonal:
      tiles.reserve(static_cast<size_t>(L.N));
      for (int i = 0; i < L.N; ++i) tiles.push_back({i, i});
      break;
    case kFactorPattern:
      tiles = factor.tiles();
      break;
    case kAll:
      tiles.reserve(static_cast<size_t>(L.N) * (L.N + 1) / 2);
      for (int j = 0; j < L.N; ++j)
        for (int i = j; i < L.N; ++i) tiles.push_back({i, j});
      break;
    case kNone:
      tiles.reserve(req.entries.size());
      for (const auto& [r, c] : req.entries) {
        if (r < 0 || c < 0 || r >= L.n || c >= L.n)
          throw Error(kErrInvalidArgument, "requested entry (" + std::to_string(r) + ", " +
                                               std::to_string(c) + ") outside the matrix");
        tiles.push_back(map_entry_to_tile(L, r, c).tile);
      }
      std::sort(tiles.begin(), tiles.end(), tile_before);
      tiles.erase(std::unique(tiles.begin(), tiles.end()), tiles.end());
      break;
    default:
      throw Error(kErrInvalidArgument, "unknown selection preset " + std::to_string(req.preset));
  }
  return tiles;
}

// selinv.cpp:85-150: single ascending sweep to the least fixpoint.
Closure symbolic_inversion(const std::vector<Coord>& requested, const Pattern& factor) {
  const Layout& L = factor.layout();
  const int N = L.N;
  if (!factor.has_all_diagonals())
    throw Error(kErrStructure, "symbolic inversion needs every factor diagonal tile");
  std::vector<Coord> wanted = requested;
  std::sort(wanted.begin(), wanted.end(), tile_before);
  wanted.erase(std::unique(wanted.begin(), wanted.end()), wanted.end());
  for (const Coord& t : wanted)
    if (t.j < 0 || t.i < t.j || t.i >= N)
      throw Error(kErrInvalidArgument, "requested tile (" + std::to_string(t.i) + ", " +
                                           std::to_string(t.j) + ") outside the lower tile grid");
  std::vector<std::set<int>> col_rows(static_cast<size_t>(N));
  for (const Coord& t : wanted) col_rows[static_cast<size_t>(t.j)].insert(t.i);
  for (int i = 0; i < N; ++i) {
    std::set<int>& rows = col_rows[static_cast<size_t>(i)];
    if (rows.empty()) continue;
    if (rows.count(i))
      for (const int* k = factor.rows_begin(i); k != factor.rows_end(i); ++k)
        if (*k > i) rows.insert(*k);
    for (int r : rows) {
      if (r <= i) continue;
      for (const int* k = factor.rows_begin(i); k != factor.rows_end(i); ++k) {
        if (*k <= i) continue;
        col_rows[static_cast<size_t>(std::min(r, *k))].insert(std::max(r, *k));
      }
    }
  }
  std::vector<Coord> ctiles;
  Closure out;
  for (int i = 0; i < N; ++i)
    for (int r : col_rows[static_cast<size_t>(i)]) ctiles.push_back({r, i});
  for (int i = N - 1; i >= 0; --i) {
    const std::set<int>& rows = col_rows[static_cast<size_t>(i)];
    if (rows.empty()) continue;
    ColumnWork w;
    w.col = i;
    w.diagonal = rows.count(i) != 0;
    for (auto it = rows.rbegin(); it != rows.rend(); ++it)
      if (*it > i) w.offdiag_rows.push_back(*it);
    out.columns.push_back(std::move(w));
  }
  out.growth_warning = ctiles.size() > 4 * wanted.size();
  out.requested = std::move(wanted);
  out.closure = Pattern(L, std::move(ctiles));
  return out;
}

double phase2_flops(const Pattern& factor, const Closure& sel) {
  const double b = factor.layout().b, b3 = b * b * b;
  double f = 0;
  for (const ColumnWork& c : sel.columns) {
    const double nk = factor.col_count(c.col) - 1;
    f += 2 * b3 * nk * static_cast<double>(c.offdiag_rows.size());
    if (c.diagonal) f += b3 / 3 + 2 * b3 * nk;
  }
  return f;
}

Flops count_flops(const FactorPlan& plan, const Closure* sel) {
  const double b = plan.filled.layout().b, b3 = b * b * b;
  Flops f;
  f.factorize = plan.counts.potrf * b3 / 3 + plan.counts.trsm * b3 + plan.counts.syrk * b3 +
                plan.counts.gemm * 2 * b3;
  f.phase1 = plan.counts.potrf * b3 / 3 + plan.counts.trsm * b3;
  if (sel) f.phase2 = phase2_flops(plan.filled, *sel);
  return f;
}

// selinv.cpp:156-169
uint64_t fnv1a_keys(const std::vector<Coord>& tiles) {
  Fnv h;
  for (const Coord& t : tiles) {
    const uint64_t key = tile_key(t.i, t.j);
    for (int byte = 0; byte < 8; ++byte) {
      const unsigned char v = static_cast<unsigned char>((key >> (byte * 8)) & 0xffu);
      h.mix(&v, 1);
    }
  }
  return h.h;
}

// ---------------------------------------------------------------------------
// Input side.
namespace {

// SplitMix64 (matgen.cpp:17-29): draw k = mix(seed + (k+1) * golden).
struct SplitMix64 {
  uint64_t s;
  explicit SplitMix64(uint64_t seed) : s(seed) {}
  uint64_t next() {
    s += 0x9e3779b97f4a7c15ull;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};

}  // namespace

// matgen.cpp:59-120.  Scalar draw order is (r ascending, c ascending); the
// diagonal is the row's |v| sum (accumulated in draw order) + 1.  Two passes
// over the same SplitMix64 stream: the first decides which tiles receive an
// entry (with density < 1 a band tile may stay empty), the second writes
// values straight into the packed slot-ordered payload.
// Tile pattern of generate_arrowhead at density 1 (every band slot accepted):
// the touched tiles follow from the index ranges alone.
Pattern arrowhead_pattern(long n, long w, long t, int b) {
  if (n < 1) throw Error(kErrInvalidArgument, "generator: n must be positive");
  if (t < 0 || t >= n) throw Error(kErrInvalidArgument, "generator: thickness must satisfy 0 <= t < n");
  if (w < 0 || w >= n - t) throw Error(kErrInvalidArgument, "generator: bandwidth must satisfy 0 <= w < n - t");
  const Layout L = build_layout(n, b);
  std::vector<std::vector<char>> touched(static_cast<size_t>(L.N));
  for (int j = 0; j < L.N; ++j) touched[static_cast<size_t>(j)].assign(static_cast<size_t>(L.N - j), 0);
  for (long r = 0; r < n; ++r) {
    const int ti = static_cast<int>(r / b);
    const long c0 = r < n - t ? std::max(0l, r - w) : 0;
    if (c0 >= r) continue;
    for (int tj = static_cast<int>(c0 / b); tj <= static_cast<int>((r - 1) / b); ++tj)
      touched[static_cast<size_t>(tj)][static_cast<size_t>(ti - tj)] = 1;
  }
  std::vector<Coord> tiles;
  for (int j = 0; j < L.N; ++j) {
    touched[static_cast<size_t>(j)][0] = 1;
    for (int d = 0; d < L.N - j; ++d)
      if (touched[static_cast<size_t>(j)][static_cast<size_t>(d)]) tiles.push_back({j + d, j});
  }
  return Pattern(L, std::move(tiles));
}

HostMatrix generate_arrowhead(long n, long w, long t, double density, uint64_t seed, int b) {
  if (n < 1) throw Error(kErrInvalidArgument, "generator: n must be positive");
  if (t < 0 || t >= n) throw Error(kErrInvalidArgument, "generator: thickness must satisfy 0 <= t < n");
  if (w < 0 || w >= n - t) throw Error(kErrInvalidArgument, "generator: bandwidth must satisfy 0 <= w < n - t");
  if (!(density > 0.0) || density > 1.0) throw Error(kErrInvalidArgument, "generator: density must lie in (0, 1]");
  const Layout L = build_layout(n, b);
  std::vector<std::vector<char>> touched(static_cast<size_t>(L.N));
  for (int j = 0; j < L.N; ++j) touched[static_cast<size_t>(j)].assign(static_cast<size_t>(L.N - j), 0);
  if (density >= 1.0) {
    // every slot is accepted: the touched tiles follow from the index ranges
    for (long r = 0; r < n; ++r) {
      const int ti = static_cast<int>(r / b);
      const long c0 = r < n - t ? std::max(0l, r - w) : 0;
      if (c0 >= r) continue;
      for (int tj = static_cast<int>(c0 / b); tj <= static_cast<int>((r - 1) / b); ++tj)
        touched[static_cast<size_t>(tj)][static_cast<size_t>(ti - tj)] = 1;
    }
  } else {
    SplitMix64 rng(seed);
    for (long r = 0; r < n; ++r) {
      const int ti = static_cast<int>(r / b);
      if (r < n - t) {
        for (long c = std::max(0l, r - w); c < r; ++c)
          if (rng.unit() < density) {
            rng.next();
            touched[static_cast<size_t>(c / b)][static_cast<size_t>(ti - c / b)] = 1;
          }
      } else {
        for (long c = 0; c < r; ++c) rng.next();
        for (int tj = 0; r > 0 && tj <= static_cast<int>((r - 1) / b); ++tj)
          touched[static_cast<size_t>(tj)][static_cast<size_t>(ti - tj)] = 1;
      }
    }
  }
  std::vector<Coord> tiles;
  for (int j = 0; j < L.N; ++j) {
    touched[static_cast<size_t>(j)][0] = 1;  // diagonal tiles always exist
    for (int d = 0; d < L.N - j; ++d)
      if (touched[static_cast<size_t>(j)][static_cast<size_t>(d)]) tiles.push_back({j + d, j});
  }
  HostMatrix m;
  m.layout = L;
  m.pattern = Pattern(L, std::move(tiles));
  const size_t bb = static_cast<size_t>(b) * b;
  m.payload.assign(m.pattern.size() * bb, 0.0);
  std::vector<double> rowsum(static_cast<size_t>(n), 0.0);
  SplitMix64 rng(seed);
  for (long r = 0; r < n; ++r) {
    const int ti = static_cast<int>(r / b);
    const size_t roff = static_cast<size_t>(r % b) * b;
    const bool band = r < n - t;
    const long c0 = band ? std::max(0l, r - w) : 0;
    int cur_tj = -1;
    double* tile = nullptr;
    for (long c = c0; c < r; ++c) {
      if (band && !(rng.unit() < density)) continue;
      const double v = 2.0 * rng.unit() - 1.0;
      const int tj = static_cast<int>(c / b);
      if (tj != cur_tj) {
        tile = &m.payload[static_cast<size_t>(m.pattern.slot(ti, tj)) * bb];
        cur_tj = tj;
      }
      tile[roff + static_cast<size_t>(c % b)] = v;
      rowsum[static_cast<size_t>(r)] += std::abs(v);
      rowsum[static_cast<size_t>(c)] += std::abs(v);
    }
  }
  for (long r = 0; r < L.n_padded; ++r) {
    const long slot = m.pattern.col_start(static_cast<int>(r / b));  // diagonal is first in its column
    m.payload[static_cast<size_t>(slot) * bb + static_cast<size_t>(r % b) * b + (r % b)] =
        r < n ? rowsum[static_cast<size_t>(r)] + 1.0 : 1.0;
  }
  return m;
}

// module.cpp:46-74: lower triangle, zeros off the diagonal skipped, every
// diagonal tile present, padding diagonal = 1.
HostMatrix matrix_from_dense(long n, int b, const double* a) {
  const Layout L = build_layout(n, b);
  std::vector<Coord> tiles;
  std::vector<std::vector<char>> touched(static_cast<size_t>(L.N));
  for (int j = 0; j < L.N; ++j) touched[static_cast<size_t>(j)].assign(static_cast<size_t>(L.N - j), 0);
  for (long r = 0; r < n; ++r)
    for (long c = 0; c <= r; ++c) {
      const double v = a[static_cast<size_t>(r) * n + c];
      if (v == 0.0 && r != c) continue;
      touched[static_cast<size_t>(c / b)][static_cast<size_t>(r / b - c / b)] = 1;
    }
  for (int j = 0; j < L.N; ++j) {
    touched[static_cast<size_t>(j)][0] = 1;
    for (int d = 0; d < L.N - j; ++d)
      if (touched[static_cast<size_t>(j)][static_cast<size_t>(d)]) tiles.push_back({j + d, j});
  }
  HostMatrix m;
  m.layout = L;
  m.pattern = Pattern(L, std::move(tiles));
  const size_t bb = static_cast<size_t>(b) * b;
  m.payload.assign(m.pattern.size() * bb, 0.0);
  for (long r = 0; r < n; ++r)
    for (long c = 0; c <= r; ++c) {
      const double v = a[static_cast<size_t>(r) * n + c];
      if (v == 0.0 && r != c) continue;
      const long s = m.pattern.slot(static_cast<int>(r / b), static_cast<int>(c / b));
      m.payload[static_cast<size_t>(s) * bb + static_cast<size_t>(r % b) * b + (c % b)] = v;
    }
  for (long r = n; r < L.n_padded; ++r) {
    const long s = m.pattern.col_start(static_cast<int>(r / b));
    m.payload[static_cast<size_t>(s) * bb + static_cast<size_t>(r % b) * b + (r % b)] = 1.0;
  }
  return m;
}

HostMatrix matrix_from_tiles(long n, int b, long count, const int* ti, const int* tj,
                             const double* payload) {
  const Layout L = build_layout(n, b);
  std::vector<Coord> tiles;
  tiles.reserve(static_cast<size_t>(count) + static_cast<size_t>(L.N));
  for (long k = 0; k < count; ++k) tiles.push_back({ti[k], tj[k]});
  for (int i = 0; i < L.N; ++i) tiles.push_back({i, i});
  HostMatrix m;
  m.layout = L;
  m.pattern = Pattern(L, std::move(tiles));
  const size_t bb = static_cast<size_t>(b) * b;
  m.payload.assign(m.pattern.size() * bb, 0.0);
  for (long k = 0; k < count; ++k) {
    const long s = m.pattern.slot(ti[k], tj[k]);
    std::memcpy(&m.payload[static_cast<size_t>(s) * bb], payload + static_cast<size_t>(k) * bb,
                bb * sizeof(double));
  }
  return m;
}

namespace {
std::string lower_copy(std::string s) {
  for (char& ch : s) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
  return s;
}
const char* skip_ws(const char* p, const char* end) {
  while (p < end && (*p == ' ' || *p == '\t' || *p == '\r')) ++p;
  return p;
}
[[noreturn]] void parse_fail(const std::string& msg, long line) {
  throw Error(kErrParse, msg + " (line " + std::to_string(line) + ")");
}
}  // namespace

// Matrix Market coordinate real symmetric, lower triangle, 1-based
// (matgen.cpp:208-319 semantics, including its error classes).
HostMatrix read_matrix_market(const std::string& text, int b) {
  long line_no = 0;
  const char* p = text.data();
  const char* end = text.data() + text.size();
  auto next_line = [&](const char** lb, const char** le) {
    if (p >= end) return false;
    *lb = p;
    const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(end - p)));
    *le = nl ? nl : end;
    p = nl ? nl + 1 : end;
    ++line_no;
    return true;
  };
  const char *lb, *le;
  if (!next_line(&lb, &le)) parse_fail("empty matrix market input", 1);
  {
    std::istringstream header(std::string(lb, le));
    std::string banner, object, format, field, symmetry;
    header >> banner >> object >> format >> field >> symmetry;
    if (banner != "%%MatrixMarket") parse_fail("unknown banner '" + banner + "'", line_no);
    if (lower_copy(object) != "matrix" || lower_copy(format) != "coordinate")
      throw Error(kErrFormat, "unsupported matrix market layout: " + object + " " + format);
    if (lower_copy(field) != "real") throw Error(kErrFormat, "unsupported field type: " + field);
    if (lower_copy(symmetry) != "symmetric")
      throw Error(kErrFormat, "only symmetric matrices are supported, got: " + symmetry);
  }
  long n = 0, mm = 0;
  long long nnz = 0;
  for (;;) {
    if (!next_line(&lb, &le)) parse_fail("missing size line", line_no);
    lb = skip_ws(lb, le);
    if (lb == le || *lb == '%') continue;
    auto r1 = std::from_chars(lb, le, n);
    if (r1.ec != std::errc{}) parse_fail("malformed size line", line_no);
    const char* q = skip_ws(r1.ptr, le);
    auto r2 = std::from_chars(q, le, mm);
    if (r2.ec != std::errc{}) parse_fail("malformed size line", line_no);
    q = skip_ws(r2.ptr, le);
    auto r3 = std::from_chars(q, le, nnz);
    if (r3.ec != std::errc{}) parse_fail("malformed size line", line_no);
    break;
  }
  if (n != mm) throw Error(kErrFormat, "matrix is not square: " + std::to_string(n) + " x " + std::to_string(mm));
  if (n < 1) parse_fail("non-positive dimension", line_no);
  const Layout L = build_layout(n, b);
  struct Ent { long r, c; double v; };
  std::vector<Ent> ents;
  ents.reserve(static_cast<size_t>(nnz));
  long long parsed = 0;
  while (parsed < nnz) {
    if (!next_line(&lb, &le))
      parse_fail("expected " + std::to_string(nnz) + " entries, found " + std::to_string(parsed), line_no);
    lb = skip_ws(lb, le);
    if (lb == le || *lb == '%') continue;
    long r = 0, c = 0;
    double v = 0.0;
    auto r1 = std::from_chars(lb, le, r);
    if (r1.ec != std::errc{}) parse_fail("malformed entry", line_no);
    const char* q = skip_ws(r1.ptr, le);
    auto r2 = std::from_chars(q, le, c);
    if (r2.ec != std::errc{}) parse_fail("malformed entry", line_no);
    q = skip_ws(r2.ptr, le);
    auto r3 = std::from_chars(q, le, v);
    if (r3.ec != std::errc{}) parse_fail("malformed entry value", line_no);
    if (r < 1 || c < 1 || r > n || c > n) parse_fail("entry index out of range", line_no);
    if (c > r)
      throw Error(kErrFormat, "upper-triangle entry (" + std::to_string(r) + ", " + std::to_string(c) +
                                  ") in a symmetric lower-triangle file at line " + std::to_string(line_no));
    ents.push_back({r - 1, c - 1, v});
    ++parsed;
  }
  {
    std::vector<uint64_t> seen;
    seen.reserve(ents.size());
    for (const Ent& e : ents) seen.push_back(static_cast<uint64_t>(e.r) * static_cast<uint64_t>(n) + static_cast<uint64_t>(e.c));
    std::sort(seen.begin(), seen.end());
    if (std::adjacent_find(seen.begin(), seen.end()) != seen.end())
      throw Error(kErrFormat, "duplicate entry in matrix market input");
  }
  std::vector<Coord> tiles;
  tiles.reserve(ents.size() / 4 + static_cast<size_t>(L.N));
  for (const Ent& e : ents) tiles.push_back({static_cast<int>(e.r / b), static_cast<int>(e.c / b)});
  for (int i = 0; i < L.N; ++i) tiles.push_back({i, i});
  HostMatrix m;
  m.layout = L;
  m.pattern = Pattern(L, std::move(tiles));
  const size_t bb = static_cast<size_t>(b) * b;
  m.payload.assign(m.pattern.size() * bb, 0.0);
  for (const Ent& e : ents) {
    const long s = m.pattern.slot(static_cast<int>(e.r / b), static_cast<int>(e.c / b));
    m.payload[static_cast<size_t>(s) * bb + static_cast<size_t>(e.r % b) * b + (e.c % b)] = e.v;
  }
  for (long r = n; r < L.n_padded; ++r) {
    const long s = m.pattern.col_start(static_cast<int>(r / b));
    m.payload[static_cast<size_t>(s) * bb + static_cast<size_t>(r % b) * b + (r % b)] = 1.0;
  }
  return m;
}

// matgen.cpp:146-184: column-major over tiles, lower triangle, nonzeros, %.17g.
std::string write_matrix_market(const HostMatrix& m) {
  const Layout& L = m.layout;
  const int b = L.b;
  const size_t bb = static_cast<size_t>(b) * b;
  std::string body;
  long long count = 0;
  char line[96];
  for (int j = 0; j < L.N; ++j) {
    for (int oc = 0; oc < b; ++oc) {
      const long c = static_cast<long>(j) * b + oc;
      if (c >= L.n) break;
      for (long s = m.pattern.col_start(j); s < m.pattern.col_start(j + 1); ++s) {
        const int i = m.pattern.tiles()[static_cast<size_t>(s)].i;
        for (int orr = 0; orr < b; ++orr) {
          const long r = static_cast<long>(i) * b + orr;
          if (r >= L.n) break;
          if (r < c) continue;
          const double v = m.payload[static_cast<size_t>(s) * bb + static_cast<size_t>(orr) * b + oc];
          if (v == 0.0) continue;
          ++count;
          const int len = std::snprintf(line, sizeof(line), "%ld %ld %.17g\n", r + 1, c + 1, v);
          body.append(line, static_cast<size_t>(len));
        }
      }
    }
  }
  std::string out = "%%MatrixMarket matrix coordinate real symmetric\n";
  out += std::to_string(L.n) + " " + std::to_string(L.n) + " " + std::to_string(count) + "\n";
  out += body;
  return out;
}

// Two-chain elimination order (planner.hpp).  Admissible when the pattern is a
// band of s >= 1 tiles plus trailing full arrow rows, only the last tile is
// partial (it stays last: with no arrow a partial last tile is kept as a
// one-tile arrow, and the fill check below decides), each interior has at
// least s columns, and the permuted pattern fills in nothing.
SplitOrder two_chain_order(const Pattern& F) {
  SplitOrder so;
  const Layout& L = F.layout();
  const int N = L.N;
  if (N < 4 || !F.has_all_diagonals()) return so;
  std::vector<int> per_row(static_cast<size_t>(N), 0);
  for (const Coord& c : F.tiles()) ++per_row[static_cast<size_t>(c.i)];
  int na = 0;
  while (na < N - 1 && per_row[static_cast<size_t>(N - 1 - na)] == N - na) ++na;
  if (na == 0 && L.n % L.b != 0) na = 1;
  const int M = N - na;
  int s = 0;
  for (const Coord& c : F.tiles())
    if (c.i < M) s = std::max(s, c.i - c.j);
  if (s < 1 || M < 3 * s + 2) return so;
  const int h = (M - s) / 2;
  so.order.reserve(static_cast<size_t>(N));
  for (int j = 0; j < h; ++j) so.order.push_back(j);
  for (int j = M - 1; j >= h + s; --j) so.order.push_back(j);
  for (int j = h; j < h + s; ++j) so.order.push_back(j);
  for (int j = M; j < N; ++j) so.order.push_back(j);
  so.pos.assign(static_cast<size_t>(N), 0);
  for (int k = 0; k < N; ++k) so.pos[static_cast<size_t>(so.order[static_cast<size_t>(k)])] = k;
  std::vector<Coord> tiles;
  tiles.reserve(F.size());
  for (const Coord& c : F.tiles()) {
    const int a = so.pos[static_cast<size_t>(c.i)], b = so.pos[static_cast<size_t>(c.j)];
    tiles.push_back(a >= b ? Coord{a, b} : Coord{b, a});
  }
  Pattern P(L, std::move(tiles));
  Pattern filled = symbolic_fill(P);
  if (filled.size() != F.size()) {
    so.order.clear();
    so.pos.clear();
    return so;
  }
  so.permuted = std::move(filled);
  so.split = h;
  return so;
}

}  // namespace tib

