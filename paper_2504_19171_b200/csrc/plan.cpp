// Dataflow plans (plan.hpp).  The task decomposition restates the reference
// schedule at 64x64 block granularity:
//   factorize   cholesky.cpp:17-49 (POTRF, TRSM per row, SYRK/GEMM per pair)
//   phase 1     selinv.cpp:195-223 (U_i = trtri(L_ii^T), W_ki = L_ki U_i^T)
//   phase 2     selinv.cpp:239-345 (Sigma_ji = -sum_k M_jk W_ki,
//               Sigma_ii = U_i U_i^T - sum_k W_ki^T Sigma_ki, mirrored)
// with X_j = L_jj^{-1} = U_j^T stored in the diagonal phase-1 slot.
#include "plan.hpp"

#include <algorithm>
#include <string>

namespace tib {

namespace {

constexpr int kB = 64;

struct Builder {
  DataflowPlan& P;
  std::vector<DTask> all;
  std::vector<unsigned char> queue;
  explicit Builder(DataflowPlan& p) : P(p) {}

  DTask& add(int q, const std::vector<Dep>& deps, const std::vector<int>& sigs) {
    DTask t{};
    t.dep_begin = static_cast<int>(P.deps.size());
    t.dep_count = static_cast<unsigned short>(deps.size());
    P.deps.insert(P.deps.end(), deps.begin(), deps.end());
    t.sig_begin = static_cast<int>(P.sigs.size());
    t.sig_count = static_cast<unsigned short>(sigs.size());
    P.sigs.insert(P.sigs.end(), sigs.begin(), sigs.end());
    t.c0_store = t.cm_store = t.diag_store = kStoreNone;
    t.c_store = kStoreNone;
    t.ldc = t.ldc0 = P.bp;
    t.seg_begin = static_cast<int>(P.segs.size());
    all.push_back(t);
    queue.push_back(static_cast<unsigned char>(q));
    return all.back();
  }
  void seg(DTask& t, unsigned char as, long long ao, unsigned char bs, long long bo, int klo, int khi, int flags) {
    Seg s{};
    s.a_store = as;
    s.a_off = ao;
    s.b_store = bs;
    s.b_off = bo;
    s.lda = s.ldb = P.bp;
    s.k_lo = static_cast<short>(klo);
    s.k_hi = static_cast<short>(khi);
    s.flags = static_cast<unsigned char>(flags);
    P.segs.push_back(s);
    ++t.seg_count;
    P.task_flops += 2.0 * kB * kB * (khi - klo);
  }
  // Splits the emission order into the two queues; returns the global order
  // expressed in final task indices.
  std::vector<int> finish(int crit_workers) {
    std::vector<int> pos(all.size());
    P.tasks.clear();
    P.tasks.reserve(all.size());
    for (size_t i = 0; i < all.size(); ++i)
      if (queue[i] == 0) {
        pos[i] = static_cast<int>(P.tasks.size());
        P.tasks.push_back(all[i]);
      }
    const int n0 = static_cast<int>(P.tasks.size());
    for (size_t i = 0; i < all.size(); ++i)
      if (queue[i] == 1) {
        pos[i] = static_cast<int>(P.tasks.size());
        P.tasks.push_back(all[i]);
      }
    P.q0 = QueueDesc{0, n0, n0 > 0 ? crit_workers : 0, 0};
    P.q1 = QueueDesc{n0, static_cast<int>(P.tasks.size()) - n0, 0, 0};
    return pos;
  }
};

long long tile_off(long slot, int bp) { return static_cast<long long>(slot) * bp * bp; }
long long blk_off(long slot, int bp, int p, int q) {
  return tile_off(slot, bp) + static_cast<long long>(p) * kB * bp + static_cast<long long>(q) * kB;
}

}  // namespace

void validate_dataflow(const DataflowPlan& plan, const std::vector<int>& order) {
  std::vector<int> cnt(static_cast<size_t>(plan.counters), 0);
  for (int ti : order) {
    const DTask& t = plan.tasks[static_cast<size_t>(ti)];
    for (int d = t.dep_begin; d < t.dep_begin + t.dep_count; ++d) {
      const Dep& dp = plan.deps[static_cast<size_t>(d)];
      if (dp.counter < 0 || dp.counter >= plan.counters || cnt[static_cast<size_t>(dp.counter)] < dp.value)
        throw Error(kErrConsistency, "dataflow plan: task " + std::to_string(ti) + " depends on counter " +
                                         std::to_string(dp.counter) + " >= " + std::to_string(dp.value) +
                                         " not produced earlier in emission order");
    }
    for (int s = t.sig_begin; s < t.sig_begin + t.sig_count; ++s) ++cnt[static_cast<size_t>(plan.sigs[static_cast<size_t>(s)])];
  }
}

DataflowPlan build_factor_dataflow(const Pattern& F, int crit_workers, int defer_w, bool fat_leaf) {
  DataflowPlan P;
  P.L = F.layout();
  const Layout& L = P.L;
  const int bp = (L.b + kB - 1) / kB * kB, nb = bp / kB, NB2 = nb * nb;
  P.bp = bp;
  P.nb = nb;
  const long T = static_cast<long>(F.size());
  const int N = L.N;
  // counter spaces
  const long cAord = 0, cAfin = cAord + T * NB2, cLblk = cAfin + T, cLfin = cLblk + T * NB2,
             cXblk = cLfin + T, cXfin = cXblk + static_cast<long>(N) * NB2, cTblk = cXfin + N,
             cWfin = cTblk + static_cast<long>(N) * NB2, cEnd = cWfin + T;
  P.counters = cEnd;
  P.scratch_doubles = static_cast<size_t>(N) * bp * bp;
  P.logdet_doubles = static_cast<size_t>(N) * nb;
  auto aord = [&](long s, int p, int q) { return static_cast<int>(cAord + s * NB2 + p * nb + q); };
  auto afin = [&](long s) { return static_cast<int>(cAfin + s); };
  auto lblk = [&](long s, int p, int q) { return static_cast<int>(cLblk + s * NB2 + p * nb + q); };
  auto lfin = [&](long s) { return static_cast<int>(cLfin + s); };
  auto xblk = [&](int j, int p, int q) { return static_cast<int>(cXblk + static_cast<long>(j) * NB2 + p * nb + q); };
  auto xfin = [&](int j) { return static_cast<int>(cXfin + j); };
  auto tblk = [&](int j, int p, int q) { return static_cast<int>(cTblk + static_cast<long>(j) * NB2 + p * nb + q); };
  auto wfin = [&](long s) { return static_cast<int>(cWfin + s); };
  const int xdone = nb * (nb + 1) / 2;
  const long long tsz = static_cast<long long>(bp) * bp;

  Builder B(P);
  std::vector<int> ord(static_cast<size_t>(T), 0);  // update columns applied so far, per tile

  auto emit_w = [&](int j) {
    const long ds = F.col_start(j);
    for (const int* r = F.rows_begin(j); r != F.rows_end(j); ++r) {
      if (*r <= j) continue;
      const long sk = F.slot(*r, j);
      for (int p = 0; p < nb; ++p)
        for (int q = 0; q < nb; ++q) {
          DTask& t = B.add(1, {{lfin(sk), NB2}, {xfin(j), xdone}}, {wfin(sk)});
          t.kind = kGemmTask;
          t.c_store = kStoreP1;
          t.c_off = blk_off(sk, bp, p, q);
          t.m0 = p * kB;
          t.n0 = q * kB;
          B.seg(t, kStoreL, tile_off(sk, bp), kStoreP1, tile_off(ds, bp), q * kB, bp, 0);
        }
    }
  };

  for (int j = 0; j < N; ++j) {
    const long ds = F.col_start(j);
    const int U = ord[static_cast<size_t>(ds)];
    const int valid = static_cast<int>(std::min<long>(L.b, L.n - static_cast<long>(j) * L.b));
    // ---- diagonal-tile chain (queue 0): blocked POTRF + TRTRI of tile (j, j)
    // Fat leaf: factor + invert block (kk, kk), then (kk + 1 < nb) the next
    // panel block L(kk+1, kk) = A(kk+1, kk) X_kk^T and the next diagonal block
    // update A(kk+1, kk+1) -= L(kk+1, kk) L(kk+1, kk)^T in the same task, so the
    // tile's diagonal chain advances one block per task.
    auto leaf = [&](int kk) {
      std::vector<Dep> d{{aord(ds, kk, kk), U + kk}};
      std::vector<int> sg{lblk(ds, kk, kk), lfin(ds), xblk(j, kk, kk), xfin(j)};
      const bool fat = fat_leaf && kk + 1 < nb;
      if (fat) {
        d.push_back({aord(ds, kk + 1, kk), U + kk});
        d.push_back({aord(ds, kk + 1, kk + 1), U + kk});
        sg.push_back(lblk(ds, kk + 1, kk));
        sg.push_back(lfin(ds));
        sg.push_back(aord(ds, kk + 1, kk + 1));
      }
      DTask& t = B.add(0, d, sg);
      t.kind = kLeafTask;
      t.mode = fat ? 2 : 0;
      t.c_off = t.c0_off = t.cm_off = blk_off(ds, bp, kk, kk);
      t.diag_off = static_cast<long long>(j) * nb + kk;
      t.m0 = valid - kk * kB;
      t.n0 = static_cast<int>(static_cast<long>(j) * L.b + kk * kB);
      t.seg_count = 0;
      if (kk + 1 < nb) P.zero.push_back(ZeroStrip{blk_off(ds, bp, kk, kk) + kB, nb - 1 - kk, 0});
      t.ldc = t.ldc0 = bp;
      P.task_flops += 2.0 * (kB * kB * kB / 6.0) * 2;  // chol + inverse of the leaf
      if (fat) P.task_flops += 2.0 * kB * kB * kB * 2;
    };
    auto paneld = [&](int i, int kk) {
      DTask& t = B.add(0, {{lblk(ds, kk, kk), 1}, {aord(ds, i, kk), U + kk}}, {lblk(ds, i, kk), lfin(ds)});
      t.kind = kGemmTask;
      t.c_store = kStoreL;
      t.c_off = blk_off(ds, bp, i, kk);
      B.seg(t, kStoreA, blk_off(ds, bp, i, kk), kStoreP1, blk_off(ds, bp, kk, kk), 0, kB, kTransB);
    };
    auto traild = [&](int i, int p, int kk) {
      DTask& t = B.add(0, {{lblk(ds, i, kk), 1}, {lblk(ds, p, kk), 1}, {aord(ds, i, p), U + kk}}, {aord(ds, i, p)});
      t.kind = kGemmTask;
      t.c_store = t.c0_store = kStoreA;
      t.c_off = t.c0_off = blk_off(ds, bp, i, p);
      B.seg(t, kStoreL, blk_off(ds, bp, i, kk), kStoreL, blk_off(ds, bp, p, kk), 0, kB, kTransB | kNegate);
    };
    auto trow = [&](int kk, int k) {
      std::vector<Dep> d;
      for (int l = k; l < kk; ++l) {
        d.push_back({lblk(ds, kk, l), 1});
        d.push_back({xblk(j, l, k), 1});
      }
      DTask& t = B.add(0, d, {tblk(j, kk, k)});
      t.kind = kGemmTask;
      t.c_store = kStoreScratch;
      t.c_off = tsz * j + static_cast<long long>(kk) * kB * bp + k * kB;
      for (int l = k; l < kk; ++l) B.seg(t, kStoreL, blk_off(ds, bp, kk, l), kStoreP1, blk_off(ds, bp, l, k), 0, kB, 0);
    };
    auto xrow = [&](int kk, int k) {
      DTask& t = B.add(0, {{xblk(j, kk, kk), 1}, {tblk(j, kk, k), 1}}, {xblk(j, kk, k), xfin(j)});
      t.kind = kGemmTask;
      t.c_store = kStoreP1;
      t.c_off = blk_off(ds, bp, kk, k);
      B.seg(t, kStoreP1, blk_off(ds, bp, kk, kk), kStoreScratch,
            tsz * j + static_cast<long long>(kk) * kB * bp + k * kB, 0, kB, kNegate);
    };
    for (int kk = 0; kk < nb; ++kk) {
      leaf(kk);
      if (!fat_leaf && kk + 1 < nb) {
        paneld(kk + 1, kk);
        traild(kk + 1, kk + 1, kk);
      }
      for (int k = 0; k < kk; ++k) xrow(kk, k);
      for (int i = kk + 2; i < nb; ++i) paneld(i, kk);
      for (int p = kk + 1; p < nb; ++p)
        for (int i = p; i < nb; ++i)
          if (!(i == kk + 1 && p == kk + 1)) traild(i, p, kk);
      if (kk + 1 < nb)
        for (int k = 0; k <= kk; ++k) trow(kk + 1, k);
    }
    // ---- bulk (queue 1)
    std::vector<int> krows;
    std::vector<long> ks;
    for (const int* r = F.rows_begin(j); r != F.rows_end(j); ++r)
      if (*r > j) {
        krows.push_back(*r);
        ks.push_back(F.slot(*r, j));
      }
    auto panel = [&](size_t ia) {
      const long sk = ks[ia];
      const int Uk = ord[static_cast<size_t>(sk)];
      for (int p = 0; p < nb; ++p)
        for (int q = 0; q < nb; ++q) {
          DTask& t = B.add(1, {{afin(sk), Uk * NB2}, {xfin(j), xdone}}, {lfin(sk)});
          t.kind = kGemmTask;
          t.c_store = kStoreL;
          t.c_off = blk_off(sk, bp, p, q);
          t.m0 = p * kB;
          t.n0 = q * kB;
          B.seg(t, kStoreA, tile_off(sk, bp), kStoreP1, tile_off(ds, bp), 0, (q + 1) * kB, kTransB);
        }
    };
    auto update = [&](size_t ia, size_t ic) {
      const int a = krows[ia], c = krows[ic];
      const long ts = F.slot(a, c);
      if (ts < 0) throw Error(kErrConsistency, "update target outside the filled pattern");
      const int u = ord[static_cast<size_t>(ts)]++;
      for (int p = 0; p < nb; ++p)
        for (int q = 0; q < (a == c ? p + 1 : nb); ++q) {
          std::vector<int> sg{aord(ts, p, q)};
          if (a != c) sg.push_back(afin(ts));
          DTask& t = B.add(1, {{lfin(ks[ia]), NB2}, {lfin(ks[ic]), NB2}, {aord(ts, p, q), u}}, sg);
          t.kind = kGemmTask;
          t.c_store = t.c0_store = kStoreA;
          t.c_off = t.c0_off = blk_off(ts, bp, p, q);
          t.m0 = p * kB;
          t.n0 = q * kB;
          B.seg(t, kStoreL, tile_off(ks[ia], bp), kStoreL, tile_off(ks[ic], bp), 0, bp, kTransB | kNegate);
        }
    };
    if (!krows.empty()) {
      panel(0);
      update(0, 0);  // feeds the next diagonal tile
      for (size_t ia = 1; ia < krows.size(); ++ia) panel(ia);
      for (size_t ia = 1; ia < krows.size(); ++ia) update(ia, 0);
      for (size_t ic = 1; ic < krows.size(); ++ic)
        for (size_t ia = ic; ia < krows.size(); ++ia) update(ia, ic);
    }
    if (j - defer_w >= 0) emit_w(j - defer_w);
  }
  for (int j = std::max(0, N - defer_w); j < N; ++j) emit_w(j);
  const std::vector<int> pos = B.finish(crit_workers);
  std::vector<int> order(pos.begin(), pos.end());
  validate_dataflow(P, order);
  return P;
}

DataflowPlan build_phase2_dataflow(const Pattern& F, const Closure& sel, int crit_workers) {
  DataflowPlan P;
  P.L = F.layout();
  const int bp = (P.L.b + kB - 1) / kB * kB, nb = bp / kB, NB2 = nb * nb;
  P.bp = bp;
  P.nb = nb;
  const Pattern& C = sel.closure;
  const long Tc = static_cast<long>(C.size());
  const long cSpart = 0, cSfin = cSpart + Tc * NB2;
  P.counters = cSfin + Tc;
  auto spart = [&](long s, int p, int q) { return static_cast<int>(cSpart + s * NB2 + p * nb + q); };
  auto sfin = [&](long s) { return static_cast<int>(cSfin + s); };
  auto cslot = [&](int i, int j) {
    const long s = C.slot(i, j);
    if (s < 0)
      throw Error(kErrConsistency, "operand tile (" + std::to_string(i) + ", " + std::to_string(j) +
                                       ") missing from the closure");
    return s;
  };
  auto final_count = [&](long s) { return C.tiles()[static_cast<size_t>(s)].i == C.tiles()[static_cast<size_t>(s)].j ? nb * (nb + 1) / 2 : NB2; };
  Builder B(P);
  for (const ColumnWork& cw : sel.columns) {
    const int i = cw.col;
    std::vector<int> K;
    for (const int* r = F.rows_begin(i); r != F.rows_end(i); ++r)
      if (*r > i) K.push_back(*r);
    const int kcrit = K.empty() ? -1 : K[0];
    auto mseg = [&](DTask& t, int j, int k) {
      const long ms = cslot(std::max(j, k), std::min(j, k));
      B.seg(t, kStoreSigma, tile_off(ms, bp), kStoreP1, tile_off(F.slot(k, i), bp), 0, bp,
            (k > j ? kTransA : 0) | kNegate);
    };
    struct Off {
      int j;
      long ts;
      bool has_early, has_crit;
    };
    std::vector<Off> offs;
    for (int j : cw.offdiag_rows) {
      Off o{j, cslot(j, i), false, false};
      for (int k : K) (k == j ? o.has_crit : o.has_early) = true;
      offs.push_back(o);
    }
    // early parts (and targets without a k == j term)
    for (const Off& o : offs) {
      if (!o.has_early) continue;
      for (int p = 0; p < nb; ++p)
        for (int q = 0; q < nb; ++q) {
          std::vector<Dep> d;
          for (int k : K)
            if (k != o.j) {
              const long ms = cslot(std::max(o.j, k), std::min(o.j, k));
              d.push_back({sfin(ms), final_count(ms)});
            }
          std::sort(d.begin(), d.end(), [](const Dep& x, const Dep& y) { return x.counter < y.counter; });
          d.erase(std::unique(d.begin(), d.end(), [](const Dep& x, const Dep& y) { return x.counter == y.counter; }),
                  d.end());
          DTask& t = B.add(1, d, {o.has_crit ? spart(o.ts, p, q) : sfin(o.ts)});
          t.kind = kGemmTask;
          t.c_store = kStoreSigma;
          t.c_off = blk_off(o.ts, bp, p, q);
          t.m0 = p * kB;
          t.n0 = q * kB;
          for (int k : K)
            if (k != o.j) mseg(t, o.j, k);
        }
    }
    auto emit_crit = [&](const Off& o, int queue) {
      const long dj = cslot(o.j, o.j);
      for (int p = 0; p < nb; ++p)
        for (int q = 0; q < nb; ++q) {
          std::vector<Dep> d{{sfin(dj), final_count(dj)}};
          if (o.has_early) d.push_back({spart(o.ts, p, q), 1});
          DTask& t = B.add(queue, d, {sfin(o.ts)});
          t.kind = kGemmTask;
          t.c_store = kStoreSigma;
          t.c_off = blk_off(o.ts, bp, p, q);
          if (o.has_early) {
            t.c0_store = kStoreSigma;
            t.c0_off = t.c_off;
          }
          t.m0 = p * kB;
          t.n0 = q * kB;
          mseg(t, o.j, o.j);
        }
    };
    for (const Off& o : offs)
      if (o.has_crit && o.j != kcrit) emit_crit(o, 1);
    if (cw.diagonal) {
      const long dsl = cslot(i, i);
      const long xs = F.col_start(i);
      const bool split = kcrit >= 0;
      auto diag_task = [&](int p, int q, bool early) {
        std::vector<Dep> d;
        std::vector<int> sg;
        if (early) {
          for (int k : K)
            if (k != kcrit) d.push_back({sfin(cslot(k, i)), NB2});
          sg.push_back(spart(dsl, p, q));
        } else {
          if (split) {
            d.push_back({spart(dsl, p, q), 1});
            d.push_back({sfin(cslot(kcrit, i)), NB2});
          }
          sg.push_back(sfin(dsl));
        }
        DTask& t = B.add(early ? 1 : 0, d, sg);
        t.kind = kGemmTask;
        t.c_store = kStoreSigma;
        t.c_off = blk_off(dsl, bp, p, q);
        t.m0 = p * kB;
        t.n0 = q * kB;
        if (!early) {
          if (split) {
            t.c0_store = kStoreSigma;
            t.c0_off = t.c_off;
          }
          if (p == q) {
            t.mode = kSymDiag;
            t.diag_store = kStoreVar;
            t.diag_off = static_cast<long long>(i) * bp + p * kB;
          } else {
            t.mode = kMirror;
            t.cm_store = kStoreSigma;
            t.cm_off = blk_off(dsl, bp, q, p);
          }
        }
        if (early || !split) {
          // U U^T = X^T X; rows >= p*64 of X carry the nonzeros for block row p >= q
          B.seg(t, kStoreP1, tile_off(xs, bp), kStoreP1, tile_off(xs, bp), p * kB, bp, kTransA);
          for (int k : K)
            if (k != kcrit || !split)
              B.seg(t, kStoreP1, tile_off(F.slot(k, i), bp), kStoreSigma, tile_off(cslot(k, i), bp), 0, bp,
                    kTransA | kNegate);
        } else {
          B.seg(t, kStoreP1, tile_off(F.slot(kcrit, i), bp), kStoreSigma, tile_off(cslot(kcrit, i), bp), 0, bp,
                kTransA | kNegate);
        }
      };
      if (split)
        for (int p = 0; p < nb; ++p)
          for (int q = 0; q <= p; ++q) diag_task(p, q, true);
      for (const Off& o : offs)
        if (o.has_crit && o.j == kcrit) emit_crit(o, 0);
      for (int p = 0; p < nb; ++p)
        for (int q = 0; q <= p; ++q) diag_task(p, q, false);
    } else {
      for (const Off& o : offs)
        if (o.has_crit && o.j == kcrit) emit_crit(o, 0);
    }
  }
  const std::vector<int> pos = B.finish(crit_workers);
  std::vector<int> order(pos.begin(), pos.end());
  validate_dataflow(P, order);
  return P;
}

}  // namespace tib
