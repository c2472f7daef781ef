// BASELINE config 4: the spatio-temporal INLA precision of a Gaussian model
// with an AR1-in-time x SPDE-in-space latent field and fixed effects -- the
// "Kronecker arrowhead" the reference cannot generate itself (
// it reads it as Matrix Market through read_matrix_market_file,
// /root/reference/proj/src/matgen.cpp:321-327).
//
//   latent x (time-major, index t * S + s, S = nx * ny sites):
//     Q_x = Q_t (x) Q_s
//     Q_t = AR1(rho) precision, unit marginal variance:
//           1 / (1 - rho^2) * tridiag(-rho; 1, 1 + rho^2, ..., 1 + rho^2, 1; -rho)
//     Q_s = tau^2 K^2, K = kappa^2 I + G, G the 5-point graph Laplacian of the
//           nx x ny lattice (SPDE alpha = 2, unit lumped mass): a 13-point stencil
//   fixed effects beta (p of them): prior precision q_beta I
//   observations y = x + Z beta + e, e ~ N(0, 1 / tau_y), Z[i, k] = 2u - 1 with
//   u the (i * p + k)-th SplitMix64 draw of `seed` (matgen.cpp:17-29)
//   joint precision of (x, beta):
//     [[Q_x + tau_y I,  tau_y Z            ],
//      [tau_y Z^T,      q_beta I + tau_y Z^T Z]]
// SPD by construction (prior precision plus a PSD likelihood term).  The
// last p rows are the dense arrow; the band is S + 2 nx (time neighbours at
// +-S with the spatial stencil around them).  Every value is a fixed
// sequence of IEEE operations (no contraction: this file is compiled with
// -ffp-contract=off), so the matrix is reproducible bit for bit.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "planner.hpp"

namespace tib {

namespace {

struct Kron {
  int nt, nx, ny, p;
  double rho, kappa2, tau, tau_y, q_beta;
  long S() const { return static_cast<long>(nx) * ny; }
  long nlat() const { return S() * nt; }
  // AR1 precision entry (|a - b| <= 1)
  double qt(int a, int b) const {
    const double c = 1.0 / (1.0 - rho * rho);
    if (a != b) return -(c * rho);
    return (a == 0 || a == nt - 1) ? c : c * (1.0 + rho * rho);
  }
  int deg(long s) const {
    const int x = static_cast<int>(s % nx), y = static_cast<int>(s / nx);
    return (x > 0) + (x < nx - 1) + (y > 0) + (y < ny - 1);
  }
  // (K^2)[a, b] for lattice sites a, b (0 outside the 13-point stencil)
  double k2(long a, long b) const {
    const int ax = static_cast<int>(a % nx), ay = static_cast<int>(a / nx);
    const int bx = static_cast<int>(b % nx), by = static_cast<int>(b / nx);
    const int dx = std::abs(ax - bx), dy = std::abs(ay - by);
    if (dx + dy == 0) {
      const double kaa = kappa2 + deg(a);
      return kaa * kaa + deg(a);
    }
    if (dx + dy == 1) return -((kappa2 + deg(a)) + (kappa2 + deg(b)));
    if (dx + dy == 2) return (dx == 1 && dy == 1) ? 2.0 : 1.0;  // common neighbours
    return 0.0;
  }
  double z(long i, int k, uint64_t seed) const {
    SplitMix64Draw d(seed);
    return 2.0 * d.unit(static_cast<uint64_t>(i) * p + k) - 1.0;
  }
  struct SplitMix64Draw {
    uint64_t seed;
    explicit SplitMix64Draw(uint64_t s) : seed(s) {}
    double unit(uint64_t k) const {
      uint64_t zz = seed + (k + 1) * 0x9e3779b97f4a7c15ull;
      zz = (zz ^ (zz >> 30)) * 0xbf58476d1ce4e5b9ull;
      zz = (zz ^ (zz >> 27)) * 0x94d049bb133111ebull;
      zz ^= zz >> 31;
      return static_cast<double>(zz >> 11) * 0x1.0p-53;
    }
  };
};

}  // namespace

HostMatrix generate_kronecker(int nt, int nx, int ny, int p, double rho, double kappa2, double tau, double tau_y,
                              double q_beta, uint64_t seed, int b) {
  if (nt < 1 || nx < 1 || ny < 1 || p < 0) throw Error(kErrInvalidArgument, "kronecker: sizes must be positive");
  if (!(std::fabs(rho) < 1.0)) throw Error(kErrInvalidArgument, "kronecker: |rho| must be < 1");
  if (!(kappa2 > 0.0) || !(tau > 0.0) || !(tau_y > 0.0) || !(q_beta > 0.0))
    throw Error(kErrInvalidArgument, "kronecker: kappa^2, tau, tau_y and q_beta must be positive");
  const Kron K{nt, nx, ny, p, rho, kappa2, tau, tau_y, q_beta};
  const long S = K.S(), nl = K.nlat(), n = nl + p;
  const Layout L = build_layout(n, b);
  const double tau2 = tau * tau;
  // stencil offsets (dx, dy) with (dy, dx) lexicographically before (0, 0): the
  // strictly lower part within one time slice
  std::vector<std::pair<int, int>> lower_st;
  for (int dy = -2; dy <= 2; ++dy)
    for (int dx = -2; dx <= 2; ++dx)
      if (std::abs(dx) + std::abs(dy) <= 2 && (dy < 0 || (dy == 0 && dx < 0))) lower_st.push_back({dx, dy});
  // visit every stored lower entry (r, c, value), r >= c
  auto visit = [&](auto&& put) {
    for (long r = 0; r < nl; ++r) {
      const int tr = static_cast<int>(r / S);
      const long sr = r % S;
      const int xr = static_cast<int>(sr % nx), yr = static_cast<int>(sr / nx);
      // previous time slice: the whole stencil, ascending column
      if (tr > 0) {
        const double q = K.qt(tr, tr - 1);
        for (int dy = -2; dy <= 2; ++dy)
          for (int dx = -2; dx <= 2; ++dx) {
            if (std::abs(dx) + std::abs(dy) > 2) continue;
            const int x = xr + dx, y = yr + dy;
            if (x < 0 || x >= nx || y < 0 || y >= ny) continue;
            const long sc = static_cast<long>(y) * nx + x;
            const double qs = tau2 * K.k2(sr, sc);
            put(r, static_cast<long>(tr - 1) * S + sc, q * qs);
          }
      }
      const double q = K.qt(tr, tr);
      for (const auto& [dx, dy] : lower_st) {
        const int x = xr + dx, y = yr + dy;
        if (x < 0 || x >= nx || y < 0 || y >= ny) continue;
        const long sc = static_cast<long>(y) * nx + x;
        const double qs = tau2 * K.k2(sr, sc);
        put(r, static_cast<long>(tr) * S + sc, q * qs);
      }
      const double qs = tau2 * K.k2(sr, sr);
      put(r, r, q * qs + tau_y);
    }
    // arrow: tau_y Z^T, then the fixed-effect block q_beta I + tau_y Z^T Z
    std::vector<double> ztz(static_cast<size_t>(p) * p, 0.0);
    for (long i = 0; i < nl; ++i)
      for (int k = 0; k < p; ++k) {
        const double zk = K.z(i, k, seed);
        for (int l = 0; l <= k; ++l) ztz[static_cast<size_t>(k) * p + l] += zk * K.z(i, l, seed);
      }
    for (int k = 0; k < p; ++k) {
      const long r = nl + k;
      for (long i = 0; i < nl; ++i) put(r, i, tau_y * K.z(i, k, seed));
      for (int l = 0; l < k; ++l) put(r, nl + l, tau_y * ztz[static_cast<size_t>(k) * p + l]);
      put(r, r, q_beta + tau_y * ztz[static_cast<size_t>(k) * p + k]);
    }
  };
  std::vector<std::vector<char>> touched(static_cast<size_t>(L.N));
  for (int j = 0; j < L.N; ++j) touched[static_cast<size_t>(j)].assign(static_cast<size_t>(L.N - j), 0);
  visit([&](long r, long c, double) { touched[static_cast<size_t>(c / b)][static_cast<size_t>(r / b - c / b)] = 1; });
  std::vector<Coord> tiles;
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
  int cur_i = -1, cur_j = -1;
  double* tile = nullptr;
  visit([&](long r, long c, double v) {
    const int ti = static_cast<int>(r / b), tj = static_cast<int>(c / b);
    if (ti != cur_i || tj != cur_j) {
      tile = &m.payload[static_cast<size_t>(m.pattern.slot(ti, tj)) * bb];
      cur_i = ti;
      cur_j = tj;
    }
    tile[static_cast<size_t>(r % b) * b + static_cast<size_t>(c % b)] = v;
  });
  for (long r = n; r < L.n_padded; ++r) {
    const long s = m.pattern.col_start(static_cast<int>(r / b));
    m.payload[static_cast<size_t>(s) * bb + static_cast<size_t>(r % b) * b + (r % b)] = 1.0;
  }
  return m;
}

}  // namespace tib
