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
// mix(seed + (k + 1) * 0x9e3779b97f4a7c15) (matgen.cpp:17-29) and the value
// 2 u - 1 with u = (x >> 11) 2^-53 -- computed here as m 2^-52 - 1 with
// m = x >> 11 split into two exact 32-bit conversions: every step is exact,
// so the bits equal the reference's whatever the operation order.
//
// Two kernels, HBM-write bound then HBM-read bound:
//   fill    one CTA per tile, one warp per row: every strictly lower entry,
//           zeros elsewhere, identity on the padding (the diagonal comes next)
//   rowsum  one thread per band row x: the diagonal is 1 + the row's absolute
//           off-diagonal sum accumulated in the reference's draw order (own
//           row ascending in c, then column x ascending in r), read back from
//           the tiles just written -- the same sequential sum as the
//           reference, so it matches to the last bit; one warp per arrow row
//           (arrow_rowsum_kernel), whose own row spans the whole matrix.
// The target is a tile store in pattern slot order with row stride bp >= b
// (the engine's A store; the slots may include fill-in tiles, which stay 0).
#include <cuda_runtime.h>

#include <cstdint>

namespace tib {

namespace {

constexpr unsigned long long kGamma = 0x9e3779b97f4a7c15ull;

struct Gen {
  long long n, w, t;
  unsigned long long seed;
  int b, bp, N;
  const int* colptr;  // CSC of the target pattern: slots of tile column j are colptr[j] .. colptr[j+1]-1
  const int* rows;    // tile row of every slot
  // a batch (one launch): matrix m (the last grid dimension) has seed
  // seeds[m] and its store at out + m * stride
  const unsigned long long* seeds;
  long long stride;
};

__device__ __forceinline__ double draw_value(unsigned long long state) {
  unsigned long long z = state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  z ^= z >> 31;
  const unsigned long long m = z >> 11;  // < 2^53
  const double md = __dadd_rn(__dmul_rn(static_cast<double>(static_cast<unsigned>(m >> 32)), 4294967296.0),
                              static_cast<double>(static_cast<unsigned>(m)));
  return __dadd_rn(__dmul_rn(md, 0x1.0p-52), -1.0);  // 2 u - 1, exact
}

// sum_{r' < r} min(r', w)
__device__ __forceinline__ unsigned long long band_slots_before(long long r, long long w) {
  if (r <= w + 1) return static_cast<unsigned long long>(r) * static_cast<unsigned long long>(r > 0 ? r - 1 : 0) / 2ull;
  return static_cast<unsigned long long>(w) * static_cast<unsigned long long>(w + 1) / 2ull +
         static_cast<unsigned long long>(r - 1 - w) * static_cast<unsigned long long>(w);
}

// row r: first nonzero column c0, draw index of its first value (c0), draws per column step
struct RowDraw {
  long long c0;
  unsigned long long k0;
  unsigned step;
};
__device__ __forceinline__ RowDraw row_draw(const Gen& g, long long r) {
  const long long ab = g.n - g.t;
  RowDraw d;
  if (r < ab) {
    d.c0 = r - g.w > 0 ? r - g.w : 0;
    d.k0 = 2ull * band_slots_before(r, g.w) + 1ull;  // the acceptance draw comes first
    d.step = 2;
  } else {
    d.c0 = 0;
    d.k0 = 2ull * band_slots_before(ab, g.w) +
           static_cast<unsigned long long>(r - 1 + ab) * static_cast<unsigned long long>(r - ab) / 2ull;
    d.step = 1;
  }
  return d;
}

__device__ __forceinline__ long long slot_of(const Gen& g, int i, int j) {
  for (int s = __ldg(g.colptr + j); s < __ldg(g.colptr + j + 1); ++s)
    if (__ldg(g.rows + s) == i) return s;
  return -1;
}

__global__ void fill_kernel(Gen g, double* __restrict__ out) {
  if (g.seeds) {
    g.seed = g.seeds[blockIdx.z];
    out += blockIdx.z * g.stride;
  }
  const long long k = blockIdx.x;
  const int J = blockIdx.y;  // tile column (grid.y), slot k = colptr[J] + blockIdx.x
  const int s0 = __ldg(g.colptr + J), s1 = __ldg(g.colptr + J + 1);
  if (s0 + k >= s1) return;
  const long long slot = s0 + k;
  const int I = __ldg(g.rows + slot);
  double* tile = out + slot * g.bp * g.bp;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int rr = warp; rr < g.bp; rr += blockDim.x >> 5) {
    const long long r = static_cast<long long>(I) * g.b + rr;
    const bool real = rr < g.b && r < g.n;
    RowDraw d{0, 0, 0};
    if (real) d = row_draw(g, r);
    for (int cc = 2 * lane; cc < g.bp; cc += 64) {
      double v[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int c2 = cc + q;
        const long long c = static_cast<long long>(J) * g.b + c2;
        double x = 0.0;
        if (rr >= g.b || c2 >= g.b) {
          x = (I == J && rr == c2) ? 1.0 : 0.0;  // bp padding: identity on diagonal tiles
        } else if (!real) {
          x = (I == J && rr == c2) ? 1.0 : 0.0;  // n_padded rows (matgen.cpp:103-106)
        } else if (c < r && c >= d.c0) {
          const unsigned long long kd = d.k0 + static_cast<unsigned long long>(c - d.c0) * d.step;
          x = draw_value(g.seed + (kd + 1ull) * kGamma);
        }
        v[q] = x;
      }
      *reinterpret_cast<double2*>(tile + static_cast<long long>(rr) * g.bp + cc) = make_double2(v[0], v[1]);
    }
  }
}

// s + |p[0]| + |p[st]| + ... (len terms) strictly in order: the loads of the
// next 16 terms are issued before the 16 dependent adds of the current ones,
// so the chain runs at the FP64 add latency instead of the load latency (the
// arrow rows sum n terms each; they are the generator's critical path).
__device__ __forceinline__ double seq_abs_sum(double s, const double* __restrict__ p, long long len, long long st) {
  constexpr int U = 16;
  double cur[U], nxt[U];
  long long i = 0;
  if (len >= U) {
#pragma unroll
    for (int q = 0; q < U; ++q) cur[q] = __ldg(p + q * st);
    for (i = U; i + U <= len; i += U) {
#pragma unroll
      for (int q = 0; q < U; ++q) nxt[q] = __ldg(p + (i + q) * st);
#pragma unroll
      for (int q = 0; q < U; ++q) s += fabs(cur[q]);
#pragma unroll
      for (int q = 0; q < U; ++q) cur[q] = nxt[q];
    }
#pragma unroll
    for (int q = 0; q < U; ++q) s += fabs(cur[q]);
  }
  for (; i < len; ++i) s += fabs(__ldg(p + i * st));
  return s;
}

// After fill: diagonal entry x = 1 + sum |v| in draw order, from the stored
// tiles -- band rows (x < n - t), one thread each.
__global__ void rowsum_kernel(Gen g, double* __restrict__ out) {
  out += blockIdx.y * g.stride;
  const long long x = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x >= g.n - g.t) return;
  const long long ab = g.n - g.t;
  const long long bpp = static_cast<long long>(g.bp) * g.bp;
  const int X = static_cast<int>(x / g.b), xo = static_cast<int>(x % g.b);
  double s = 0.0;
  // own row, c ascending, one contiguous run per tile
  const long long c0 = x < ab ? (x - g.w > 0 ? x - g.w : 0) : 0;
  for (long long c = c0; c < x;) {
    const int Jc = static_cast<int>(c / g.b);
    const long long ce = (static_cast<long long>(Jc) + 1) * g.b < x ? (static_cast<long long>(Jc) + 1) * g.b : x;
    const double* row = out + slot_of(g, X, Jc) * bpp + static_cast<long long>(xo) * g.bp + (c - static_cast<long long>(Jc) * g.b);
    s = seq_abs_sum(s, row, ce - c, 1);
    c = ce;
  }
  // column x: band rows within w, then every arrow row, r ascending (stride bp per tile)
  auto column = [&](long long r, long long re) {
    while (r < re) {
      const int Ir = static_cast<int>(r / g.b);
      const long long e = (static_cast<long long>(Ir) + 1) * g.b < re ? (static_cast<long long>(Ir) + 1) * g.b : re;
      const double* col = out + slot_of(g, Ir, X) * bpp + xo + (r - static_cast<long long>(Ir) * g.b) * g.bp;
      s = seq_abs_sum(s, col, e - r, g.bp);
      r = e;
    }
  };
  const long long rb = x + g.w < ab - 1 ? x + g.w : ab - 1;
  column(x + 1, rb + 1);
  column(ab > x + 1 ? ab : x + 1, g.n);
  out[slot_of(g, X, X) * bpp + static_cast<long long>(xo) * g.bp + xo] = s + 1.0;
}

// Arrow rows (x >= n - t), one warp each: the own row has x terms (up to n),
// a serial chain that one thread would run at the load latency.  The warp
// loads 256 consecutive terms (8 per lane) one chunk ahead, and every lane adds
// the chunk in order from the shuffled values -- the same sequence of
// additions (an added +0.0 past a chunk's end leaves s >= 0 unchanged), so the
// same bits, at the FP64 add latency.
__global__ void arrow_rowsum_kernel(Gen g, double* __restrict__ out) {
  out += blockIdx.y * g.stride;
  const int lane = threadIdx.x & 31;
  const long long x = g.n - g.t + (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  if (x >= g.n) return;
  const long long bpp = static_cast<long long>(g.bp) * g.bp;
  const int X = static_cast<int>(x / g.b), xo = static_cast<int>(x % g.b);
  // chunk c .. c + len (len <= 256, within one tile)
  auto chunk_end = [&](long long c) {
    const long long te = (c / g.b + 1) * g.b;
    const long long e = c + 256 < te ? c + 256 : te;
    return e < x ? e : x;
  };
  auto load = [&](long long c, long long e, double (&v)[8]) {
    const int Jc = static_cast<int>(c / g.b);
    const double* row = out + slot_of(g, X, Jc) * bpp + static_cast<long long>(xo) * g.bp + (c - static_cast<long long>(Jc) * g.b);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const long long i = lane * 8 + q;
      v[q] = c + i < e ? __ldg(row + i) : 0.0;
    }
  };
  double s = 0.0, cur[8], nxt[8];
  long long c = 0, e = chunk_end(0);
  if (c < x) load(c, e, cur);
  while (c < x) {
    const long long c2 = e, e2 = c2 < x ? chunk_end(c2) : c2;
    if (c2 < x) load(c2, e2, nxt);
#pragma unroll
    for (int l = 0; l < 32; ++l)
#pragma unroll
      for (int q = 0; q < 8; ++q) s += fabs(__shfl_sync(0xffffffffu, cur[q], l));
#pragma unroll
    for (int q = 0; q < 8; ++q) cur[q] = nxt[q];
    c = c2;
    e = e2;
  }
  if (lane != 0) return;
  // column x: the arrow rows below, r ascending
  for (long long r = x + 1; r < g.n;) {
    const int Ir = static_cast<int>(r / g.b);
    const long long re = (static_cast<long long>(Ir) + 1) * g.b < g.n ? (static_cast<long long>(Ir) + 1) * g.b : g.n;
    const double* col = out + slot_of(g, Ir, X) * bpp + xo + (r - static_cast<long long>(Ir) * g.b) * g.bp;
    s = seq_abs_sum(s, col, re - r, g.bp);
    r = re;
  }
  out[slot_of(g, X, X) * bpp + static_cast<long long>(xo) * g.bp + xo] = s + 1.0;
}

}  // namespace

// colptr (N + 1) and rows (slots) describe the target pattern in device memory.
int launch_generate_arrowhead(long n, long w, long t, unsigned long long seed, int b, int bp, int N, const int* colptr,
                              const int* rows, int max_col_slots, double* out, cudaStream_t s,
                              const unsigned long long* seeds, int count, long long stride) {
  const Gen g{n, w, t, seed, b, bp, N, colptr, rows, seeds, stride};
  const unsigned nm = static_cast<unsigned>(count > 0 ? count : 1);
  if (N > 0 && max_col_slots > 0)
    fill_kernel<<<dim3(static_cast<unsigned>(max_col_slots), static_cast<unsigned>(N), nm), 256, 0, s>>>(g, out);
  if (n - t > 0) rowsum_kernel<<<dim3(static_cast<unsigned>((n - t + 255) / 256), nm), 256, 0, s>>>(g, out);
  if (t > 0) arrow_rowsum_kernel<<<dim3(static_cast<unsigned>((t + 3) / 4), nm), 128, 0, s>>>(g, out);
  return static_cast<int>(cudaGetLastError());
}

}  // namespace tib
