// Device-side generator of the reference's synthetic arrowhead matrices
// (generate_arrowhead, /root/reference/proj/src/matgen.cpp:59-120) at
// density 1, bit-identical to the host generator (planner.cpp) and to the
// reference.
//
// At density 1 every band slot is accepted, so the SplitMix64 draw that
// produces an entry has a closed-form index: a band row r
// (r < n - t) draws two numbers per slot c in [max(0, r - w), r) --
// acceptance, then value -- and an arrow row draws one per c < r.  With
// S(r) = sum_{r' < r} min(r', w) the band rows start at draw 2 S(r), the arrow
// rows at 2 S(n - t) + sum_{r' = n-t}^{r-1} r'.  Draw k is
// mix(seed + (k + 1) * 0x9e3779b97f4a7c15) (matgen.cpp:17-29), the value
// 2 u - 1 with u = (x >> 11) 2^-53.  The diagonal is 1 + the row's absolute
// off-diagonal sum accumulated in draw order (own row ascending in c, then
// column entries in ascending row), one sequential sum per row as in the
// reference, so it matches to the last bit.
//
// Two kernels: rowsum (one thread per row, sequential) and fill (every
// element of every stored tile, 16-byte stores, identity on the padding).
// The target is a tile store in pattern slot order with row stride bp >= b
// (the engine's A store), HBM-write bound.
#include <cuda_runtime.h>

#include <cstdint>

namespace tib {

namespace {

struct Gen {
  long long n, w, t;
  unsigned long long seed;
  int b, bp;
};

__device__ __forceinline__ double draw_value(unsigned long long seed, unsigned long long k) {
  unsigned long long z = seed + (k + 1ull) * 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  z ^= z >> 31;
  const double u = static_cast<double>(z >> 11) * 0x1.0p-53;
  return __dadd_rn(__dmul_rn(2.0, u), -1.0);
}

// sum_{r' < r} min(r', w)
__device__ __forceinline__ unsigned long long band_slots_before(long long r, long long w) {
  if (r <= w + 1) return static_cast<unsigned long long>(r) * static_cast<unsigned long long>(r > 0 ? r - 1 : 0) / 2ull;
  return static_cast<unsigned long long>(w) * static_cast<unsigned long long>(w + 1) / 2ull +
         static_cast<unsigned long long>(r - 1 - w) * static_cast<unsigned long long>(w);
}

// value of the strictly lower entry (r, c) (0 when outside the band / arrow)
__device__ __forceinline__ double entry(const Gen& g, long long r, long long c) {
  const long long ab = g.n - g.t;  // first arrow row
  if (r < ab) {
    if (r - c > g.w) return 0.0;
    const long long c0 = r - g.w > 0 ? r - g.w : 0;
    const unsigned long long k = 2ull * band_slots_before(r, g.w) + 2ull * static_cast<unsigned long long>(c - c0) + 1ull;
    return draw_value(g.seed, k);
  }
  const unsigned long long base = 2ull * band_slots_before(ab, g.w) +
                                  static_cast<unsigned long long>(r - 1 + ab) * static_cast<unsigned long long>(r - ab) / 2ull;
  return draw_value(g.seed, base + static_cast<unsigned long long>(c));
}

__global__ void rowsum_kernel(Gen g, double* __restrict__ diag) {
  const long long x = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= g.n) return;
  const long long ab = g.n - g.t;
  double s = 0.0;
  // own row, c ascending
  const long long c0 = x < ab ? (x - g.w > 0 ? x - g.w : 0) : 0;
  for (long long c = c0; c < x; ++c) s += fabs(entry(g, x, c));
  // column entries (r, x), r ascending: band rows within w, then every arrow row
  const long long rb = x + g.w < ab - 1 ? x + g.w : ab - 1;
  for (long long r = x + 1; r <= rb; ++r) s += fabs(entry(g, r, x));
  for (long long r = (ab > x + 1 ? ab : x + 1); r < g.n; ++r) s += fabs(entry(g, r, x));
  diag[x] = s + 1.0;
}

// one CTA per tile: every (row, column pair) of the bp x bp tile
__global__ void fill_kernel(Gen g, const int* __restrict__ ti, const int* __restrict__ tj,
                            const double* __restrict__ diag, double* __restrict__ out) {
  const long long k = blockIdx.x;
  const int I = __ldg(ti + k), J = __ldg(tj + k);
  const int half = g.bp / 2;
  double* tile = out + k * g.bp * g.bp;
  for (int e = threadIdx.x; e < g.bp * half; e += blockDim.x) {
    const int rr = e / half, cc = (e - rr * half) * 2;
    double v[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int c2 = cc + q;
      double x = 0.0;
      if (rr >= g.b || c2 >= g.b) {
        x = (I == J && rr == c2) ? 1.0 : 0.0;  // bp padding: identity on diagonal tiles
      } else {
        const long long r = static_cast<long long>(I) * g.b + rr, c = static_cast<long long>(J) * g.b + c2;
        if (r == c) x = r < g.n ? diag[r] : 1.0;  // n_padded rows: identity (matgen.cpp:103-106)
        else if (c < r && r < g.n) x = entry(g, r, c);
      }
      v[q] = x;
    }
    *reinterpret_cast<double2*>(tile + static_cast<long long>(rr) * g.bp + cc) = make_double2(v[0], v[1]);
  }
}

}  // namespace

// diag_scratch: n doubles of device memory
int launch_generate_arrowhead(long n, long w, long t, unsigned long long seed, int b, int bp, const int* slot_ti,
                              const int* slot_tj, long slots, double* diag_scratch, double* out, cudaStream_t s) {
  const Gen g{n, w, t, seed, b, bp};
  rowsum_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(g, diag_scratch);
  if (slots > 0) fill_kernel<<<static_cast<unsigned>(slots), 256, 0, s>>>(g, slot_ti, slot_tj, diag_scratch, out);
  return static_cast<int>(cudaGetLastError());
}

}  // namespace tib
