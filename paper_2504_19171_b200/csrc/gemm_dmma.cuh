// FP64 tensor-core (DMMA) tile-block GEMM for sm_100a.
//
// There is no FP64 kind for tcgen05.mma on sm_100a (ptxas rejects it) and no
// wgmma; the FP64 tensor path on B200 is mma.sync.m8n8k4.f64, which lowers to
// DMMA.8x8x4 and was measured at 37.2 TFLOP/s chip-wide (profiles/
// r01_fp64_peak.jsonl) vs 34.2 for DFMA.  So every dense FP64 tile contraction
// of the path runs through this one block routine:
//
//   C[BM x BN] = C0 + sum_s sign_s * op(A_s) op(B_s)       (K = sum of segment ranges)
//
// One CTA owns one 64 x 64 output block of a b x b tile and walks every K
// segment in a fixed order, so the accumulation order is deterministic and no
// atomics are needed (the reference fixes ascending-k order for bitwise
// reproducibility, kernels.hpp:26-27; we fix ours the same way).
//
// Operands are staged global -> shared with cp.async (16 B, .cg = L2 only)
// through a STAGES-deep ring; transposed and non-transposed operands land in
// two padded shared layouts chosen per K chunk, both conflict-free for the
// 64-bit fragment loads (row stride = 4 mod 16 doubles).  4 warps, each a
// 32 x 32 sub-block = 4 x 4 m8n8 accumulators (64 registers).
#pragma once

#include <cstdint>
#include <type_traits>

#include "taskfmt.hpp"

namespace tib {

constexpr int kStages = 4;
constexpr int kGemmThreads = 128;  // threads of one worker (4 warps)
constexpr int kWorkers = 2;         // workers per CTA (one CTA per SM)

// Worker-local thread index and barrier: each CTA runs kWorkers independent
// task loops on its halves, synchronised by named barrier 1 + half (barrier
// 0 stays the whole CTA).
__device__ __forceinline__ int wtid() { return threadIdx.x & (kGemmThreads - 1); }
__device__ __forceinline__ int whalf() { return threadIdx.x / kGemmThreads; }
__device__ __forceinline__ void wsync() {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + static_cast<int>(threadIdx.x / kGemmThreads)), "n"(kGemmThreads) : "memory");
}
constexpr int kLdN = kBK + 4;   // [row][k] layout stride (doubles)
constexpr int kLdT = kBM + 4;   // [k][row] layout stride (doubles)
constexpr int kStageDoubles = (kBM * kLdN > kBK * kLdT ? kBM * kLdN : kBK * kLdT);
constexpr int kGemmSmemBytes = kStages * 2 * kStageDoubles * 8;

// Resolved forms used by the block routine.
struct RSeg {
  const double* A;
  const double* B;
  int lda, ldb, k_lo, k_hi, flags, pad;
};
struct RTask {
  double* C;         // block origin in the output
  const double* C0;  // block origin of the initial value (may alias C), or null
  double* Cm;        // kMirror: origin of the transposed block
  double* diag;      // kSymDiag: if non-null receives C[r][r] (marginal variances)
  int ldc, ldc0;
  int m0, n0;        // block offsets into op(A) rows / op(B) columns
  int seg_count, mode;
};

__device__ __forceinline__ double* resolve(const BaseTable& bt, unsigned char store, long long off) {
  return store == kStoreNone ? nullptr : bt.p[store] + off;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// Stage one BK-wide K chunk of segment s (at k0) into shared buffers.
__device__ __forceinline__ void load_chunk(const RSeg& s, int m0, int n0, int k0, double* As,
                                           double* Bs, int tid) {
  // A: BM x BK of op(A); 512 16-byte pieces, 4 per thread.
  if (!(s.flags & kTransA)) {
    // op(A)[m][k] = A[m0+m][k]: rows of 16 doubles = 8 pieces.
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int idx = tid + p * kGemmThreads;
      const int m = idx >> 3, kq = (idx & 7) * 2;
      cp_async16(As + m * kLdN + kq, s.A + static_cast<size_t>(m0 + m) * s.lda + k0 + kq);
    }
  } else {
    // op(A)[m][k] = A[k][m0+m]: rows of 64 doubles = 32 pieces.
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int idx = tid + p * kGemmThreads;
      const int k = idx >> 5, mq = (idx & 31) * 2;
      cp_async16(As + k * kLdT + mq, s.A + static_cast<size_t>(k0 + k) * s.lda + m0 + mq);
    }
  }
  if (!(s.flags & kTransB)) {
    // op(B)[k][n] = B[k][n0+n]
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int idx = tid + p * kGemmThreads;
      const int k = idx >> 5, nq = (idx & 31) * 2;
      cp_async16(Bs + k * kLdT + nq, s.B + static_cast<size_t>(k0 + k) * s.ldb + n0 + nq);
    }
  } else {
    // op(B)[k][n] = B[n0+n][k]
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int idx = tid + p * kGemmThreads;
      const int n = idx >> 3, kq = (idx & 7) * 2;
      cp_async16(Bs + n * kLdN + kq, s.B + static_cast<size_t>(n0 + n) * s.ldb + k0 + kq);
    }
  }
}

// Segment sources for gemm_task: plan segments in global memory resolved
// through a base table, or ready-made segments (e.g. built in shared memory).
struct GlobalSegs {
  const Seg* segs;
  const BaseTable* bt;
  int count;
  __device__ __forceinline__ RSeg get(int i) const {
    const Seg s = segs[i];
    RSeg r;
    r.A = bt->p[s.a_store] + s.a_off;
    r.B = bt->p[s.b_store] + s.b_off;
    r.lda = s.lda;
    r.ldb = s.ldb;
    r.k_lo = s.k_lo;
    r.k_hi = s.k_hi;
    r.flags = s.flags;
    r.pad = 0;
    return r;
  }
};
struct LocalSegs {
  const RSeg* segs;
  int count;
  __device__ __forceinline__ RSeg get(int i) const { return segs[i]; }
};

// Main loop of one task on the calling CTA (kGemmThreads threads): the block
// product sum_s sign_s op(A_s) op(B_s) into acc (the warp's 32 x 32 patch as
// 4 x 4 m8n8 fragments).  smem must hold kGemmSmemBytes; ends with the ring
// drained (no barrier: the epilogue does not touch shared memory).
//
// Inner loop: the two shared layouts differ only in strides, so fragment
// addresses are (stage base) + k*sK + row*sM with per-stage strides -- no
// branches, and the next k-step's fragments are loaded while the current
// 16 DMMAs issue.  A segment's sign is applied by negating the accumulators
// when the sign changes between chunks (at most a couple of times per task)
// instead of per fragment.
// C0 prefetch: a task whose initial value is final when it starts (no
// second-phase dependency) stages C0 into the two ring stages the last chunks
// free -- rows 0-31 and 32-63, row stride kLdC0 (conflict-free double2 reads)
// -- so the epilogue's read of C0 is a shared-memory read, not an exposed
// global round trip.  gemm_mainloop returns the ring stage of rows 0-31 (rows
// 32-63 are in the next stage, mod kStages), or -1 when nothing was staged.
constexpr int kLdC0 = kBN + 4;
static_assert(32 * kLdC0 <= 2 * kStageDoubles, "a ring stage holds half a C0 block");

template <class Src>
__device__ __forceinline__ int gemm_mainloop(const RTask& t, const Src& src, double* smem, double (&acc)[4][4][2],
                                             bool prefetch_c0 = false, int nchunks_hint = -1) {
  const int tid = wtid();
  const int lane = tid & 31, warp = tid >> 5;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const int fr = lane >> 2, fc = lane & 3;

#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // Flattened chunk sequence over segments, walked by a producer cursor.
  // (plan tasks carry the count: no pass over the segments before the first load)
  int nchunks = nchunks_hint;
  if (nchunks < 0) {
    nchunks = 0;
    for (int s = 0; s < src.count; ++s) {
      const RSeg g = src.get(s);
      nchunks += (g.k_hi - g.k_lo) / kBK;
    }
  }
  prefetch_c0 = prefetch_c0 && t.C0 != nullptr && nchunks >= 4;
  int ls = 0, lk = 0;
  RSeg cur;
  cur.k_hi = 0;
  cur.k_lo = 0;
  cur.flags = 0;
  if (src.count > 0) {
    cur = src.get(0);
    lk = cur.k_lo;
  }
  auto settle = [&]() {  // move to the next segment with chunks left
    while (ls < src.count && lk >= cur.k_hi) {
      ++ls;
      if (ls < src.count) {
        cur = src.get(ls);
        lk = cur.k_lo;
      }
    }
  };
  settle();
  uint32_t stage_flags = 0;  // 3 bits per stage
#pragma unroll
  for (int st = 0; st < kStages - 1; ++st) {
    if (st < nchunks) {
      double* As = smem + st * 2 * kStageDoubles;
      load_chunk(cur, t.m0, t.n0, lk, As, As + kStageDoubles, tid);
      stage_flags |= static_cast<uint32_t>(cur.flags & 7) << (3 * st);
      lk += kBK;
      settle();
    }
    cp_async_commit();
  }

  bool negated = false;
  // one K chunk; the C0 prefetch is only compiled into the last iterations'
  // copy (the main loop stays as it is without it)
  auto chunk = [&](int it, auto with_c0) {
    cp_async_wait<kStages - 2>();
    wsync();
    {
      const int nx = it + kStages - 1;
      if (nx < nchunks) {
        const int st = nx % kStages;
        double* As = smem + st * 2 * kStageDoubles;
        load_chunk(cur, t.m0, t.n0, lk, As, As + kStageDoubles, tid);
        stage_flags = (stage_flags & ~(7u << (3 * st))) | (static_cast<uint32_t>(cur.flags & 7) << (3 * st));
        lk += kBK;
        settle();
      }
      if (decltype(with_c0)::value && it < nchunks - 1) {
        // the stage of chunk it - 1: consumed (barrier above) and never refilled
        double* dst = smem + ((it + kStages - 1) % kStages) * 2 * kStageDoubles;
        const double* src0 = t.C0 + static_cast<size_t>(it - (nchunks - 3)) * 32 * t.ldc0;
#pragma unroll
        for (int p = 0; p < 8; ++p) {
          const int idx = tid + p * kGemmThreads;
          const int r = idx >> 5, cq = (idx & 31) * 2;
          cp_async16(dst + r * kLdC0 + cq, src0 + static_cast<size_t>(r) * t.ldc0 + cq);
        }
      }
      cp_async_commit();
    }
    const int st = it % kStages;
    const int fl = (stage_flags >> (3 * st)) & 7;
    const bool neg = fl & kNegate;
    if (neg != negated) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc[i][j][0] = -acc[i][j][0];
          acc[i][j][1] = -acc[i][j][1];
        }
      negated = neg;
    }
    // element (row, k) of the A chunk is at As[k * aK + row * aM]; (k, col) of B at Bs[k * bK + col * bN]
    const int aK = (fl & kTransA) ? kLdT : 1, aM = (fl & kTransA) ? 1 : kLdN;
    const int bK = (fl & kTransB) ? 1 : kLdT, bN = (fl & kTransB) ? kLdN : 1;
    const double* Ap = smem + st * 2 * kStageDoubles + fc * aK + (wm + fr) * aM;
    const double* Bp = smem + st * 2 * kStageDoubles + kStageDoubles + fc * bK + (wn + fr) * bN;
    double a[2][4], b[2][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      a[0][i] = Ap[i * 8 * aM];
      b[0][i] = Bp[i * 8 * bN];
    }
#pragma unroll
    for (int ks = 0; ks < kBK / 4; ++ks) {
      const int cb = ks & 1;
      if (ks + 1 < kBK / 4) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          a[cb ^ 1][i] = Ap[(ks + 1) * 4 * aK + i * 8 * aM];
          b[cb ^ 1][i] = Bp[(ks + 1) * 4 * bK + i * 8 * bN];
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], a[cb][i], b[cb][j]);
    }
  };
  const int pf_from = prefetch_c0 ? nchunks - 3 : nchunks;  // C0 halves at chunks nchunks-3, nchunks-2
  int it = 0;
  for (; it < pf_from; ++it) chunk(it, std::false_type{});
  for (; it < nchunks; ++it) chunk(it, std::true_type{});
  cp_async_wait<0>();
  if (negated) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        acc[i][j][0] = -acc[i][j][0];
        acc[i][j][1] = -acc[i][j][1];
      }
  }
  wsync();  // every warp is done with the ring before the next task refills it (and sees the staged C0)
  return prefetch_c0 ? (nchunks + kStages - 4) % kStages : -1;
}

// Position of fragment (i, j, h) of the calling thread in the 64 x 64 block.
__device__ __forceinline__ int frag_row(int i) {
  const int lane = threadIdx.x & 31, warp = wtid() >> 5;
  return (warp >> 1) * 32 + i * 8 + (lane >> 2);
}
__device__ __forceinline__ int frag_col(int j) {
  const int lane = threadIdx.x & 31, warp = wtid() >> 5;
  return (warp & 1) * 32 + j * 8 + (lane & 3) * 2;
}

// Epilogue: C = C0 + acc, written per mode; ends with a barrier so thread 0
// may release the task's signals.
// C0 comes from the ring stages gemm_mainloop staged it in (c0_stage >= 0,
// smem = the ring) or from global memory.
__device__ __forceinline__ void gemm_epilogue(const RTask& t, const double (&acc)[4][4][2], const double* smem = nullptr,
                                              int c0_stage = -1) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int r = frag_row(i), c = frag_col(j);
      double v0 = acc[i][j][0], v1 = acc[i][j][1];
      if (c0_stage >= 0) {
        const double* sc = smem + ((c0_stage + (r >> 5)) % kStages) * 2 * kStageDoubles + (r & 31) * kLdC0 + c;
        const double2 o = *reinterpret_cast<const double2*>(sc);
        v0 += o.x;
        v1 += o.y;
      } else if (t.C0) {
        const double2 o = __ldcg(reinterpret_cast<const double2*>(t.C0 + static_cast<size_t>(r) * t.ldc0 + c));
        v0 += o.x;
        v1 += o.y;
      }
      if (t.mode == kFull) {
        *reinterpret_cast<double2*>(t.C + static_cast<size_t>(r) * t.ldc + c) = make_double2(v0, v1);
      } else if (t.mode == kMirror) {
        *reinterpret_cast<double2*>(t.C + static_cast<size_t>(r) * t.ldc + c) = make_double2(v0, v1);
        t.Cm[static_cast<size_t>(c) * t.ldc + r] = v0;
        t.Cm[static_cast<size_t>(c + 1) * t.ldc + r] = v1;
      } else {  // kSymDiag: lower part wins, mirrored exactly
        if (r >= c) {
          t.C[static_cast<size_t>(r) * t.ldc + c] = v0;
          t.C[static_cast<size_t>(c) * t.ldc + r] = v0;
          if (r == c && t.diag) t.diag[r] = v0;
        }
        if (r >= c + 1) {
          t.C[static_cast<size_t>(r) * t.ldc + c + 1] = v1;
          t.C[static_cast<size_t>(c + 1) * t.ldc + r] = v1;
          if (r == c + 1 && t.diag) t.diag[r] = v1;
        }
      }
    }
  }
  wsync();
}

// Split-K: a part's accumulators -> its 64 x 64 scratch slot (row-major).
__device__ __forceinline__ void split_store(double* slot, const double (&acc)[4][4][2]) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
      __stcg(reinterpret_cast<double2*>(slot + frag_row(i) * kBN + frag_col(j)), make_double2(acc[i][j][0], acc[i][j][1]));
}

// Reducer: acc = P_0 + P_1 + ... + P_{parts-1} in part order, every part read
// back from its slot (the caller's own included, bitwise what it stored), so
// the result does not depend on which part arrived last.
__device__ __forceinline__ void split_reduce(const double* slots, int parts, double (&acc)[4][4][2]) {
  for (int p = 0; p < parts; ++p) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double2 v =
            __ldcg(reinterpret_cast<const double2*>(slots + static_cast<size_t>(p) * kBM * kBN + frag_row(i) * kBN + frag_col(j)));
        acc[i][j][0] = p == 0 ? v.x : acc[i][j][0] + v.x;
        acc[i][j][1] = p == 0 ? v.y : acc[i][j][1] + v.y;
      }
  }
}

// One plain task: main loop + epilogue.
template <class Src>
__device__ __forceinline__ void gemm_task(const RTask& t, const Src& src, double* smem) {
  double acc[4][4][2];
  const int c0s = gemm_mainloop(t, src, smem, acc, true);
  gemm_epilogue(t, acc, smem, c0s);
}

__device__ __forceinline__ RTask resolve_task(const Task& s, const BaseTable& bt) {
  RTask t;
  t.C = resolve(bt, s.c_store, s.c_off);
  t.C0 = resolve(bt, s.c0_store, s.c0_off);
  t.Cm = resolve(bt, s.cm_store, s.cm_off);
  t.diag = resolve(bt, s.diag_store, s.diag_off);
  t.ldc = s.ldc;
  t.ldc0 = s.ldc0;
  t.m0 = s.m0;
  t.n0 = s.n0;
  t.seg_count = s.seg_count;
  t.mode = s.mode;
  return t;
}

}  // namespace tib
