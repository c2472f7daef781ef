// Timing / golden driver over the UNMODIFIED reference library (oracle/_ref,
// built by oracle/Makefile from /root/reference/proj/src).  Test
// infrastructure: it is the CPU baseline (`cpu_baseline.kind = "reference"`)
// and the source of golden scalars; the product never links it.
//
// It mirrors the reference CLI's timing method (proj/tools/tileinv_main.cpp:
// 173-203): steady_clock around symbolic_cholesky+factorize, phase1(std::move),
// and phase2, generation excluded.
//
//   ref_driver bench  n w t b seed workers [density]
//       -> one JSON line {factorize_s, phase1_s, phase2_s, total_s, gflop, ...}
//   ref_driver bench_mm file.mtx b workers   (the same for a Matrix Market input)
//   ref_driver golden n w t b seed workers prefix [density]
//   ref_driver golden_mm file.mtx b workers prefix
//       -> golden summary files (see golden_run) and a JSON line
//   ref_driver checksum n w t b seed [density]  -> payload_checksum of the matrix
//   ref_driver dump   n w t b seed workers out_prefix [density]
//   ref_driver symbolic n w t b seed density selection
//       -> {"factor": [[i,j],...], "closure": [[i,j],...], "requested": [...],
//           "columns": [[col, diag, [rows...]], ...], "growth_warning": b}
//          selection = diagonal | pattern | all | r,c;r,c;...
//       -> <prefix>.diag.f64 (n doubles), <prefix>.sigma.f64 (closure tiles,
//          column-major tile order, each b*b row-major) and a JSON line.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>
#include <vector>

#include "tileinv/cholesky.hpp"
#include "tileinv/matgen.hpp"
#include "tileinv/selinv.hpp"
#include "tileinv/tileio.hpp"

using namespace tileinv;
using Clock = std::chrono::steady_clock;

static double secs(Clock::time_point a, Clock::time_point b) {
  return std::chrono::duration<double>(b - a).count();
}

struct Flops {
  double fact = 0, p1 = 0, p2 = 0;
};

// Task-model FLOPs: POTRF b^3/3, TRSM b^3, SYRK b^3, GEMM 2b^3;
// TRTRI b^3/3, TRMM b^3; LAUUM b^3/3, GEMM 2b^3 per (target, k) term.
static Flops count_flops(const FactorPlan& plan, const SelectedTileSet& sel,
                         const TilePattern& fpat) {
  const double b = fpat.layout().b, b3 = b * b * b;
  Flops f;
  for (const FactorTask& t : plan.tasks) {
    switch (t.kind) {
      case FactorKernel::kPotrf: f.fact += b3 / 3; break;
      case FactorKernel::kTrsm: f.fact += b3; break;
      case FactorKernel::kSyrk: f.fact += b3; break;
      case FactorKernel::kGemm: f.fact += 2 * b3; break;
    }
  }
  for (int j = 0; j < fpat.layout().N; ++j) {
    f.p1 += b3 / 3;
    for (int i : fpat.neighbors(j))
      if (i > j) f.p1 += b3;
  }
  for (const ColumnWork& c : sel.columns) {
    int nk = 0;
    for (int k : fpat.neighbors(c.col))
      if (k > c.col) ++nk;
    f.p2 += 2 * b3 * nk * static_cast<double>(c.offdiag_rows.size());
    if (c.diagonal) f.p2 += b3 / 3 + 2 * b3 * nk;
  }
  return f;
}

static void print_tiles(const char* name, const std::vector<TileCoord>& t) {
  std::printf("\"%s\": [", name);
  for (size_t k = 0; k < t.size(); ++k) std::printf("%s[%d,%d]", k ? "," : "", t[k].i, t[k].j);
  std::printf("]");
}

static int symbolic_main(int argc, char** argv) {
  const long n = std::atol(argv[2]), w = std::atol(argv[3]), t = std::atol(argv[4]);
  const int b = std::atoi(argv[5]);
  const unsigned long long seed = std::strtoull(argv[6], nullptr, 10);
  const double density = std::atof(argv[7]);
  const std::string sel = argc > 8 ? argv[8] : "pattern";
  SelectionRequest req;
  if (sel == "diagonal") req = SelectionRequest::diagonal();
  else if (sel == "pattern") req = SelectionRequest::factor_pattern();
  else if (sel == "all") req = SelectionRequest::all();
  else {
    std::vector<std::pair<long, long>> e;
    size_t pos = 0;
    while (pos < sel.size()) {
      size_t semi = sel.find(';', pos);
      if (semi == std::string::npos) semi = sel.size();
      const std::string item = sel.substr(pos, semi - pos);
      const size_t comma = item.find(',');
      e.emplace_back(std::atol(item.substr(0, comma).c_str()), std::atol(item.substr(comma + 1).c_str()));
      pos = semi + 1;
    }
    req = SelectionRequest::of(e);
  }
  GeneratedMatrix gen = generate_arrowhead({n, w, t, density, seed}, b);
  const FactorPlan plan = symbolic_cholesky(gen.matrix.pattern);
  const std::vector<TileCoord> tiles = select_tiles(gen.matrix.layout, plan.filled, req);
  const SelectedTileSet s = symbolic_inversion(tiles, plan.filled);
  std::printf("{");
  print_tiles("factor", plan.filled.tiles());
  std::printf(", ");
  print_tiles("closure", s.closure.tiles());
  std::printf(", ");
  print_tiles("requested", s.requested);
  std::printf(", \"columns\": [");
  for (size_t k = 0; k < s.columns.size(); ++k) {
    std::printf("%s[%d,%d,[", k ? "," : "", s.columns[k].col, s.columns[k].diagonal ? 1 : 0);
    for (size_t r = 0; r < s.columns[k].offdiag_rows.size(); ++r)
      std::printf("%s%d", r ? "," : "", s.columns[k].offdiag_rows[r]);
    std::printf("]]");
  }
  std::printf("], \"growth_warning\": %s, \"tasks\": %zu}\n", s.growth_warning ? "true" : "false",
              plan.tasks.size());
  return 0;
}

// Golden summary of a selected inverse (ref_driver golden / golden_mm): the
// reference's own numbers at the BASELINE configs, small enough to commit.
//   <prefix>.diag.f64    diag(Sigma), n doubles (marginal variances)
//   <prefix>.tstats.f64  per closure tile (column-major): Frobenius norm, sum,
//                        weighted sum with w(r, c) = ((7 r + 13 c) mod 11) - 5
//   <prefix>.blocks.f64  for each sampled tile: the leading s x s block and the
//                        trailing s x s block of its valid region (s = min(64, b);
//                        starting at row / column max(0, valid - s))
//   stdout               JSON: logdet, trace, checksums, sampled tile list
static int golden_run(const TiledSymmetricMatrix& m, int workers, const std::string& prefix) {
  const long n = m.layout.n;
  const int b = m.layout.b;
  const auto t0 = Clock::now();
  const FactorPlan plan = symbolic_cholesky(m.pattern);
  TiledFactor factor = factorize(m, plan, workers);
  double logdet = 0.0;
  for (long r = 0; r < n; ++r) {
    const auto& d = factor.blocks.at(static_cast<int>(r / b), static_cast<int>(r / b));
    logdet += 2.0 * std::log(d[static_cast<std::size_t>(r % b) * b + (r % b)]);
  }
  const std::uint64_t msum = payload_checksum(m.blocks);
  const std::uint64_t fsum = payload_checksum(factor.blocks);
  const SelectedTileSet sel =
      symbolic_inversion(select_tiles(factor.layout, factor.pattern, SelectionRequest::factor_pattern()),
                         factor.pattern);
  factor = phase1(std::move(factor), workers);
  SelectedInverse sigma = phase2(factor, sel, workers);
  const auto t1 = Clock::now();
  const int N = m.layout.N;
  std::vector<double> diag(static_cast<std::size_t>(n));
  double trace = 0.0;
  for (long r = 0; r < n; ++r) {
    const auto& d = sigma.blocks.at(static_cast<int>(r / b), static_cast<int>(r / b));
    diag[static_cast<std::size_t>(r)] = d[static_cast<std::size_t>(r % b) * b + (r % b)];
    trace += diag[static_cast<std::size_t>(r)];
  }
  std::vector<double> stats;
  std::vector<TileCoord> sampled;
  for (const auto& [key, p] : sigma.blocks.map()) {
    const int i = static_cast<int>(key & 0xffffffffu), j = static_cast<int>(key >> 32);
    double fro = 0, sum = 0, wsum = 0;
    for (int r = 0; r < b; ++r)
      for (int c = 0; c < b; ++c) {
        const double v = p[static_cast<std::size_t>(r) * b + c];
        fro += v * v;
        sum += v;
        wsum += v * static_cast<double>(((7 * r + 13 * c) % 11) - 5);
      }
    stats.push_back(std::sqrt(fro));
    stats.push_back(sum);
    stats.push_back(wsum);
    const bool pick = j >= N - 3 || j == N / 2 || (i == N - 1 && (j == 0 || j == N / 2 || j == N - 4));
    if (pick) sampled.push_back({i, j});
  }
  const int s = b < 64 ? b : 64;
  std::ofstream bl(prefix + ".blocks.f64", std::ios::binary);
  for (const TileCoord& tc : sampled) {
    const auto& p = sigma.blocks.at(tc.i, tc.j);
    const long vr = std::min<long>(b, n - static_cast<long>(tc.i) * b), vc = std::min<long>(b, n - static_cast<long>(tc.j) * b);
    for (int part = 0; part < 2; ++part) {
      const long r0 = part ? std::max(0l, vr - s) : 0, c0 = part ? std::max(0l, vc - s) : 0;
      for (long r = r0; r < r0 + s; ++r)
        bl.write(reinterpret_cast<const char*>(p.data() + r * b + c0), static_cast<std::streamsize>(s * sizeof(double)));
    }
  }
  std::ofstream dg(prefix + ".diag.f64", std::ios::binary);
  dg.write(reinterpret_cast<const char*>(diag.data()), static_cast<std::streamsize>(diag.size() * sizeof(double)));
  std::ofstream ts(prefix + ".tstats.f64", std::ios::binary);
  ts.write(reinterpret_cast<const char*>(stats.data()), static_cast<std::streamsize>(stats.size() * sizeof(double)));
  std::printf("{\"n\": %ld, \"b\": %d, \"N\": %d, \"workers\": %d, \"closure_tiles\": %zu, \"seconds\": %.3f, "
              "\"logdet\": %.17g, \"trace\": %.17g, \"matrix_checksum\": %llu, \"factor_checksum\": %llu, "
              "\"result_checksum\": %llu, \"block\": %d, ",
              n, b, N, workers, sigma.closure.size(), secs(t0, t1), logdet, trace,
              static_cast<unsigned long long>(msum), static_cast<unsigned long long>(fsum),
              static_cast<unsigned long long>(payload_checksum(sigma.blocks)), s);
  print_tiles("sampled", sampled);
  std::printf("}\n");
  return 0;
}

// ref_driver bench_mm file.mtx b workers: the bench timing of a Matrix Market
// input (read_matrix_market_file, matgen.cpp:321-327; read time excluded).
static int bench_mm(const std::string& path, int b, int workers) {
  const auto g0 = Clock::now();
  const TiledSymmetricMatrix m = read_matrix_market_file(path, b);
  const auto g1 = Clock::now();
  const auto t0 = Clock::now();
  const FactorPlan plan = symbolic_cholesky(m.pattern);
  TiledFactor factor = factorize(m, plan, workers);
  const auto t1 = Clock::now();
  const SelectedTileSet sel =
      symbolic_inversion(select_tiles(factor.layout, factor.pattern, SelectionRequest::factor_pattern()),
                         factor.pattern);
  const auto t2 = Clock::now();
  factor = phase1(std::move(factor), workers);
  const auto t3 = Clock::now();
  SelectedInverse sigma = phase2(factor, sel, workers);
  const auto t4 = Clock::now();
  const Flops fl = count_flops(plan, sel, factor.pattern);
  const double total = secs(t0, t1) + secs(t2, t3) + secs(t3, t4);
  const double gflop = (fl.fact + fl.p1 + fl.p2) / 1e9;
  std::printf("{\"n\": %ld, \"b\": %d, \"workers\": %d, \"N\": %d, \"tiles\": %zu, \"read_s\": %.6f, "
              "\"factorize_s\": %.6f, \"phase1_s\": %.6f, \"phase2_s\": %.6f, \"total_s\": %.6f, "
              "\"gflop\": %.6f, \"gflops\": %.4f, \"closure_tiles\": %zu}\n",
              m.layout.n, b, workers, m.layout.N, factor.pattern.size(), secs(g0, g1), secs(t0, t1), secs(t2, t3),
              secs(t3, t4), total, gflop, gflop / total, sigma.closure.size());
  return 0;
}

int main(int argc, char** argv) {
  if (argc >= 8 && std::string(argv[1]) == "symbolic") return symbolic_main(argc, argv);
  if (argc >= 5 && std::string(argv[1]) == "bench_mm") return bench_mm(argv[2], std::atoi(argv[3]), std::atoi(argv[4]));
  // ref_driver golden n w t b seed workers prefix [density]
  if (argc >= 9 && std::string(argv[1]) == "golden") {
    const double density = argc > 9 ? std::atof(argv[9]) : 1.0;
    GeneratedMatrix gen = generate_arrowhead(
        {std::atol(argv[2]), std::atol(argv[3]), std::atol(argv[4]), density, std::strtoull(argv[6], nullptr, 10)},
        std::atoi(argv[5]));
    return golden_run(gen.matrix, std::atoi(argv[7]), argv[8]);
  }
  // ref_driver golden_mm file.mtx b workers prefix   (read_matrix_market_file, matgen.cpp:321-327)
  if (argc >= 6 && std::string(argv[1]) == "golden_mm") {
    const TiledSymmetricMatrix m = read_matrix_market_file(argv[2], std::atoi(argv[3]));
    return golden_run(m, std::atoi(argv[4]), argv[5]);
  }
  // ref_driver stls n w t b seed prefix: the reference's own tile files of one
  // case -- <prefix>.matrix.stls (kMatrix), .factor.stls (kFactor, factorize),
  // .phase1.stls (kPhase1, phase1), .sigma.stls (write_selected_inverse, pattern)
  if (argc >= 8 && std::string(argv[1]) == "stls") {
    GeneratedMatrix gen = generate_arrowhead(
        {std::atol(argv[2]), std::atol(argv[3]), std::atol(argv[4]), 1.0, std::strtoull(argv[6], nullptr, 10)},
        std::atoi(argv[5]));
    const std::string pre = argv[7];
    write_tile_file(pre + ".matrix.stls", gen.matrix.layout, PhaseTag::kMatrix, gen.matrix.blocks);
    TiledFactor f = factorize(gen.matrix, symbolic_cholesky(gen.matrix.pattern), 1);
    write_tile_file(pre + ".factor.stls", f.layout, f.phase, f.blocks);
    TiledFactor p1 = phase1(f, 1);
    write_tile_file(pre + ".phase1.stls", p1.layout, p1.phase, p1.blocks);
    const SelectedInverse s = selected_inverse(f, SelectionRequest::factor_pattern(), 1);
    write_selected_inverse(pre + ".sigma.stls", s);
    return 0;
  }
  // ref_driver checksum n w t b seed [density]: payload_checksum of the generated matrix
  if (argc >= 7 && std::string(argv[1]) == "checksum") {
    const double density = argc > 7 ? std::atof(argv[7]) : 1.0;
    GeneratedMatrix gen = generate_arrowhead(
        {std::atol(argv[2]), std::atol(argv[3]), std::atol(argv[4]), density, std::strtoull(argv[6], nullptr, 10)},
        std::atoi(argv[5]));
    std::printf("%llu\n", static_cast<unsigned long long>(payload_checksum(gen.matrix.blocks)));
    return 0;
  }
  if (argc < 8) {
    std::fprintf(stderr, "usage: ref_driver bench|dump n w t b seed workers [prefix] [density]\n");
    return 2;
  }
  const std::string mode = argv[1];
  const long n = std::atol(argv[2]), w = std::atol(argv[3]), t = std::atol(argv[4]);
  const int b = std::atoi(argv[5]);
  const unsigned long long seed = std::strtoull(argv[6], nullptr, 10);
  const int workers = std::atoi(argv[7]);
  std::string prefix;
  int argi = 8;
  if (mode == "dump") prefix = argv[argi++];
  const double density = argc > argi ? std::atof(argv[argi]) : 1.0;

  const auto g0 = Clock::now();
  GeneratedMatrix gen = generate_arrowhead({n, w, t, density, seed}, b);
  const auto g1 = Clock::now();

  const auto t0 = Clock::now();
  const FactorPlan plan = symbolic_cholesky(gen.matrix.pattern);
  TiledFactor factor = factorize(gen.matrix, plan, workers);
  const auto t1 = Clock::now();
  // logdet is not a reference API: 2 * sum log L_rr, r < n.
  double logdet = 0.0;
  for (long r = 0; r < n; ++r) {
    const auto& d = factor.blocks.at(static_cast<int>(r / b), static_cast<int>(r / b));
    logdet += 2.0 * std::log(d[static_cast<std::size_t>(r % b) * b + (r % b)]);
  }
  const std::uint64_t fsum = payload_checksum(factor.blocks);
  const std::vector<TileCoord> tiles =
      select_tiles(factor.layout, factor.pattern, SelectionRequest::factor_pattern());
  const SelectedTileSet sel = symbolic_inversion(tiles, factor.pattern);
  const auto t2 = Clock::now();
  factor = phase1(std::move(factor), workers);
  const auto t3 = Clock::now();
  SelectedInverse sigma = phase2(factor, sel, workers);
  const auto t4 = Clock::now();

  const Flops fl = count_flops(plan, sel, factor.pattern);
  double trace = 0.0;
  std::vector<double> diag(static_cast<std::size_t>(n));
  for (long r = 0; r < n; ++r) {
    const auto& d = sigma.blocks.at(static_cast<int>(r / b), static_cast<int>(r / b));
    diag[static_cast<std::size_t>(r)] = d[static_cast<std::size_t>(r % b) * b + (r % b)];
    trace += diag[static_cast<std::size_t>(r)];
  }
  const double total = secs(t0, t1) + secs(t2, t3) + secs(t3, t4);
  const double gflop = (fl.fact + fl.p1 + fl.p2) / 1e9;
  std::printf(
      "{\"n\": %ld, \"w\": %ld, \"t\": %ld, \"b\": %d, \"seed\": %llu, \"workers\": %d, "
      "\"N\": %d, \"tiles\": %zu, \"closure_tiles\": %zu, \"generate_s\": %.6f, "
      "\"factorize_s\": %.6f, \"phase1_s\": %.6f, \"phase2_s\": %.6f, \"total_s\": %.6f, "
      "\"gflop_factorize\": %.6f, \"gflop_phase1\": %.6f, \"gflop_phase2\": %.6f, "
      "\"gflop\": %.6f, \"gflops\": %.4f, \"logdet\": %.17g, \"trace\": %.17g, "
      "\"factor_checksum\": %llu, \"result_checksum\": %llu}\n",
      n, w, t, b, seed, workers, gen.matrix.layout.N, factor.pattern.size(),
      sigma.closure.size(), secs(g0, g1), secs(t0, t1), secs(t2, t3), secs(t3, t4), total,
      fl.fact / 1e9, fl.p1 / 1e9, fl.p2 / 1e9, gflop, gflop / total, logdet, trace,
      static_cast<unsigned long long>(fsum),
      static_cast<unsigned long long>(payload_checksum(sigma.blocks)));

  if (mode == "dump") {
    std::ofstream dg(prefix + ".diag.f64", std::ios::binary);
    dg.write(reinterpret_cast<const char*>(diag.data()),
             static_cast<std::streamsize>(diag.size() * sizeof(double)));
    std::ofstream sg(prefix + ".sigma.f64", std::ios::binary);
    for (const auto& [key, payload] : sigma.blocks.map()) {
      (void)key;
      sg.write(reinterpret_cast<const char*>(payload.data()),
               static_cast<std::streamsize>(payload.size() * sizeof(double)));
    }
  }
  return 0;
}
