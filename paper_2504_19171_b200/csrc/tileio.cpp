// STLS binary tile files (the reference's checkpoint / resume format,
// /root/reference/proj/src/tileio.cpp:30-94, tileio.hpp:9-15), byte for byte:
//   "STLS" | version u32 = 1 | n u32 | b u32 | N u32 | phase u32 | count u32
//   then per tile, column-major over the grid: i u32, j u32, b*b float64 row-major.
// Phase tags (storage.hpp:11-16): 0 matrix, 1 factor, 2 phase-1, 3 selected
// inverse.  Errors follow the reference: unreadable file -> Error, bad magic /
// version / truncation / grid mismatch / upper-triangle tile / unknown phase ->
// ParseError, wrong phase for the consumer -> FormatError (checked by callers).
#include <cstdio>
#include <cstring>
#include <map>

#include "planner.hpp"

namespace tib {

namespace {

struct File {
  std::FILE* f = nullptr;
  File(const std::string& path, const char* mode) : f(std::fopen(path.c_str(), mode)) {}
  ~File() {
    if (f) std::fclose(f);
  }
};

uint32_t get_u32(std::FILE* f, const char* what) {
  uint32_t v = 0;
  if (std::fread(&v, sizeof(v), 1, f) != 1) throw Error(kErrParse, std::string("tile file truncated reading ") + what);
  return v;
}

}  // namespace

TileFileData read_tile_file(const std::string& path) {
  File in(path, "rb");
  if (!in.f) throw Error(kErrGeneric, "cannot open " + path);
  char magic[4];
  if (std::fread(magic, 1, 4, in.f) != 4 || std::memcmp(magic, "STLS", 4) != 0)
    throw Error(kErrParse, "not a tile file (bad magic): " + path);
  const uint32_t version = get_u32(in.f, "version");
  if (version != 1) throw Error(kErrParse, "unsupported tile file version " + std::to_string(version));
  const uint32_t n = get_u32(in.f, "n");
  const uint32_t b = get_u32(in.f, "b");
  const uint32_t N = get_u32(in.f, "N");
  const uint32_t phase = get_u32(in.f, "phase");
  const uint32_t count = get_u32(in.f, "tile count");
  if (phase > 3) throw Error(kErrParse, "unknown phase tag " + std::to_string(phase));
  TileFileData d;
  d.layout = build_layout(static_cast<long>(n), static_cast<int>(b));
  if (d.layout.N != static_cast<int>(N))
    throw Error(kErrParse, "tile grid mismatch: header says " + std::to_string(N) + ", n and b give " +
                               std::to_string(d.layout.N));
  d.phase = static_cast<int>(phase);
  const size_t bb = static_cast<size_t>(b) * b;
  // a later copy of a tile replaces an earlier one (TileBlocks::ensure)
  std::map<uint64_t, std::vector<double>> tiles;
  for (uint32_t t = 0; t < count; ++t) {
    const uint32_t i = get_u32(in.f, "tile row");
    const uint32_t j = get_u32(in.f, "tile column");
    if (j > i || i >= N)
      throw Error(kErrParse, "tile (" + std::to_string(i) + ", " + std::to_string(j) + ") outside the lower triangle");
    std::vector<double>& blk = tiles[tile_key(static_cast<int>(i), static_cast<int>(j))];
    blk.resize(bb);
    if (std::fread(blk.data(), sizeof(double), bb, in.f) != bb)
      throw Error(kErrParse, "tile file truncated in payload of tile " + std::to_string(t));
  }
  std::vector<Coord> coords;
  coords.reserve(tiles.size());
  for (const auto& kv : tiles) coords.push_back({static_cast<int>(kv.first & 0xffffffffu), static_cast<int>(kv.first >> 32)});
  d.pattern = Pattern(d.layout, std::move(coords));
  d.payload.resize(d.pattern.size() * bb);
  size_t k = 0;
  for (const auto& kv : tiles) std::memcpy(&d.payload[bb * k++], kv.second.data(), bb * sizeof(double));
  return d;
}

void write_tile_file(const std::string& path, const Layout& L, int phase, const Pattern& pattern,
                     const double* payload) {
  File out(path, "wb");
  if (!out.f) throw Error(kErrGeneric, "cannot open " + path + " for writing");
  const uint32_t hdr[6] = {1u, static_cast<uint32_t>(L.n), static_cast<uint32_t>(L.b), static_cast<uint32_t>(L.N),
                           static_cast<uint32_t>(phase), static_cast<uint32_t>(pattern.size())};
  bool ok = std::fwrite("STLS", 1, 4, out.f) == 4 && std::fwrite(hdr, sizeof(uint32_t), 6, out.f) == 6;
  const size_t bb = static_cast<size_t>(L.b) * L.b;
  for (size_t k = 0; ok && k < pattern.size(); ++k) {
    const uint32_t ij[2] = {static_cast<uint32_t>(pattern.tiles()[k].i), static_cast<uint32_t>(pattern.tiles()[k].j)};
    ok = std::fwrite(ij, sizeof(uint32_t), 2, out.f) == 2 && std::fwrite(payload + k * bb, sizeof(double), bb, out.f) == bb;
  }
  if (!ok) throw Error(kErrGeneric, "short write to " + path);
}

}  // namespace tib
