// Dataflow plans (plan.hpp).  The task decomposition restates the reference
// schedule at 64x64 block granularity:
//   factorize   cholesky.cpp:17-49 (POTRF, TRSM per row, SYRK/GEMM per pair)
//   phase 1     selinv.cpp:195-223 (U_i = trtri(L_ii^T), W_ki = L_ki U_i^T)
//   phase 2     selinv.cpp:239-345 (Sigma_ji = -sum_k M_jk W_ki,
//               Sigma_ii = U_i U_i^T - sum_k W_ki^T Sigma_ki, mirrored)
// with X_j = L_jj^{-1} = U_j^T stored in the diagonal phase-1 slot.
#include "plan.hpp"

#include <algorithm>
#include <set>
#include <string>

namespace tib {

namespace {

constexpr int kB = 64;

struct Builder {
  DataflowPlan& P;
  std::vector<DTask> all;
  std::vector<unsigned char> queue;
  std::vector<int> conv;  // emission index -> index after the chain conversion
  explicit Builder(DataflowPlan& p) : P(p) {}

  DTask& add(int q, const std::vector<Dep>& deps, const std::vector<int>& sigs, const std::vector<Dep>& deps2 = {}) {
    DTask t{};
    t.poll = -1;
    t.dep_begin = static_cast<int>(P.deps.size());
    t.dep_count = static_cast<unsigned short>(deps.size());
    t.dep2_count = static_cast<unsigned char>(deps2.size());
    P.deps.insert(P.deps.end(), deps.begin(), deps.end());
    P.deps.insert(P.deps.end(), deps2.begin(), deps2.end());
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
  // Appends signal c to task t (its signal list is copied to the end of sigs).
  void add_sig(DTask& t, int c) {
    const int nb0 = static_cast<int>(P.sigs.size());
    for (int s = t.sig_begin; s < t.sig_begin + t.sig_count; ++s) P.sigs.push_back(P.sigs[static_cast<size_t>(s)]);
    P.sigs.push_back(c);
    t.sig_begin = nb0;
    ++t.sig_count;
  }
  // Adds a first-phase dependency to task t (its dependency list is copied).
  void add_dep(DTask& t, Dep d) {
    const int nb0 = static_cast<int>(P.deps.size());
    for (int k = t.dep_begin; k < t.dep_begin + t.dep_count; ++k) P.deps.push_back(P.deps[static_cast<size_t>(k)]);
    P.deps.push_back(d);
    for (int k = t.dep_begin + t.dep_count; k < t.dep_begin + t.dep_count + t.dep2_count; ++k)
      P.deps.push_back(P.deps[static_cast<size_t>(k)]);
    t.dep_begin = nb0;
    ++t.dep_count;
  }
  // Splits the emission order into the two queues; returns the global order
  // expressed in final task indices.
  std::vector<int> finish(int crit_workers, bool chain = false, int split = -1) {
    // dependency check in emission order (before any restructuring)
    P.tasks = all;
    std::vector<int> ident(all.size());
    for (size_t i = 0; i < all.size(); ++i) ident[i] = static_cast<int>(i);
    validate_dataflow(P, ident);
    if (chain) {
      // the leaves become chain steps, in emission order (one persistent task runs them)
      std::vector<DTask> rest;
      std::vector<unsigned char> rq;
      P.chain.clear();
      conv.assign(all.size(), -1);
      const bool any_leaf = std::any_of(all.begin(), all.end(), [](const DTask& t) { return t.kind == kLeafTask; });
      // (two chains: the first chain's leaves, then the second's -- the
      // columns may be emitted interleaved)
      for (int pass = 0; pass < (split > 0 ? 2 : 1); ++pass)
        for (size_t i = 0; i < all.size(); ++i)
          if (all[i].kind == kLeafTask && (split <= 0 || (all[i].n0 / P.L.b >= split) == (pass == 1)))
            P.chain.push_back(all[i]);
      for (size_t i = 0; i < all.size(); ++i) {
        if (all[i].kind == kLeafTask) {
        } else {
          conv[i] = static_cast<int>(rest.size()) + (any_leaf ? 1 : 0);
          rest.push_back(all[i]);
          rq.push_back(queue[i]);
        }
      }
      // one chain task per elimination chain: steps of columns < split, then
      // the rest (partitioned by chain above, column order within each)
      std::vector<int> bounds{0};
      if (split > 0) {
        int k = 0;
        while (k < static_cast<int>(P.chain.size()) && P.chain[static_cast<size_t>(k)].n0 / P.L.b < split) ++k;
        if (k > 0 && k < static_cast<int>(P.chain.size())) bounds.push_back(k);
      }
      bounds.push_back(static_cast<int>(P.chain.size()));
      const int nchains = P.chain.empty() ? 0 : static_cast<int>(bounds.size()) - 1;
      if (nchains > 1)
        for (int& x : conv)
          if (x >= 0) x += nchains - 1;
      all.clear();
      queue.clear();
      for (int q = 0; q < nchains; ++q) {
        DTask c{};
        c.poll = -1;
        c.kind = kChainTask;
        c.c_store = c.c0_store = c.cm_store = c.diag_store = kStoreNone;
        c.seg_begin = bounds[static_cast<size_t>(q)];
        c.seg_count = bounds[static_cast<size_t>(q) + 1] - bounds[static_cast<size_t>(q)];
        all.push_back(c);
        queue.push_back(0);
      }
      all.insert(all.end(), rest.begin(), rest.end());
      queue.insert(queue.end(), rq.begin(), rq.end());
      // a boundary leaf may carry its block to the next step only if that step
      // is the block's leaf and no other column updates the block in between
      // (the leaf's dependency value is the count this step's signal reaches)
      for (size_t s = 0; s + 1 < P.chain.size(); ++s) {
        if (std::find(bounds.begin(), bounds.end(), static_cast<int>(s) + 1) != bounds.end()) continue;
        DTask& c0 = P.chain[s];
        const DTask& c1 = P.chain[s + 1];
        if (!(c0.mode & 4) || c1.dep_count < 1) continue;
        const Seg& sx = P.segs[static_cast<size_t>(c0.seg_begin)];
        const Dep& d = P.deps[static_cast<size_t>(c1.dep_begin)];
        const int aord_sig = P.sigs[static_cast<size_t>(c0.sig_begin + c0.sig_count - 2)];
        if (c1.c_off == sx.b_off && d.counter == aord_sig && d.value == c0.aux0) c0.mode |= kCarry;
      }
    }
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
    for (DTask& t : P.tasks) {
      t.chunks = 0;
      if (t.kind == kGemmTask || t.kind == kSplitTask)
        for (int k = t.seg_begin; k < t.seg_begin + t.seg_count; ++k)
          t.chunks += (P.segs[static_cast<size_t>(k)].k_hi - P.segs[static_cast<size_t>(k)].k_lo) / kBK;
    }
    finalize_waiters();
    return pos;
  }
  void finalize_waiters() {
    const size_t nt = P.tasks.size();
    const size_t nc = static_cast<size_t>(P.counters);
    P.need.assign(nt, 0);
    std::vector<int> maxv(nc, 0);
    std::vector<std::pair<long long, int>> w;  // ((counter << 32) | value, task)
    for (size_t t = 0; t < nt; ++t) {
      const DTask& k = P.tasks[t];
      for (int d = k.dep_begin; d < k.dep_begin + k.dep_count; ++d) {
        const Dep& dp = P.deps[static_cast<size_t>(d)];
        if (dp.value <= 0) continue;
        ++P.need[t];
        maxv[static_cast<size_t>(dp.counter)] = std::max(maxv[static_cast<size_t>(dp.counter)], dp.value);
        w.push_back({(static_cast<long long>(dp.counter) << 32) | dp.value, static_cast<int>(t)});
      }
    }
    std::stable_sort(w.begin(), w.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
    P.wl.resize(w.size());
    for (size_t i = 0; i < w.size(); ++i) P.wl[i] = w[i].second;
    P.vbase.assign(nc + 1, 0);
    for (size_t c = 0; c < nc; ++c) P.vbase[c + 1] = P.vbase[c] + maxv[c] + 2;
    P.vidx.assign(static_cast<size_t>(P.vbase[nc]), 0);
    size_t pos = 0;
    for (size_t c = 0; c < nc; ++c) {
      for (int v = 0; v <= maxv[c] + 1; ++v) {
        const long long key = (static_cast<long long>(c) << 32) | v;
        while (pos < w.size() && w[pos].first < key) ++pos;
        P.vidx[static_cast<size_t>(P.vbase[c] + v)] = static_cast<int>(pos);
      }
    }
    P.init0.clear();
    P.init1.clear();
    for (size_t t = 0; t < nt; ++t)
      if (P.need[t] == 0) (static_cast<int>(t) < P.q0.count ? P.init0 : P.init1).push_back(static_cast<int>(t));
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
    for (int d = t.dep_begin; d < t.dep_begin + t.dep_count + t.dep2_count; ++d) {
      const Dep& dp = plan.deps[static_cast<size_t>(d)];
      if (dp.counter < 0 || dp.counter >= plan.counters || cnt[static_cast<size_t>(dp.counter)] < dp.value)
        throw Error(kErrConsistency, "dataflow plan: task " + std::to_string(ti) + " depends on counter " +
                                         std::to_string(dp.counter) + " >= " + std::to_string(dp.value) +
                                         " not produced earlier in emission order");
    }
    // a split group signals once, through its reducer (the last part to arrive;
    // in emission order, the last part)
    if (t.kind == kSplitTask && (t.aux1 >> 8) != (t.aux1 & 255) - 1) continue;
    for (int s = t.sig_begin; s < t.sig_begin + t.sig_count; ++s) ++cnt[static_cast<size_t>(plan.sigs[static_cast<size_t>(s)])];
  }
}

DataflowPlan build_factor_dataflow(const Pattern& F, int crit_workers, int defer_w, bool fat_leaf, bool chain,
                                   bool boundary, int split, bool coarse_second, int ugroup) {
  if (chain) fat_leaf = true;
  if (boundary) fat_leaf = true;
  DataflowPlan P;
  P.L = F.layout();
  const Layout& L = P.L;
  const int bp = (L.b + kB - 1) / kB * kB, nb = bp / kB, NB2 = nb * nb;
  P.bp = bp;
  P.nb = nb;
  const long T = static_cast<long>(F.size());
  const int N = L.N;
  // split-K shapes of the critical tail (see below)
  auto panel_parts = [&](int q) { return (q + 1) * kB > 256 ? (q + 2) / 2 : 1; };  // K = 64 (q+1), parts of <= 128
  const int upd_parts = nb > 2 ? (nb + 1) / 2 : 1;                                // K = bp, parts of 128
  // per column: the progressive panels of the first two off-diagonal tiles and
  // the split updates of tiles (k0, k0) and (k1, k0)
  int panel_slots = 0;
  for (int q = 0; q < nb; ++q)
    if (panel_parts(q) > 1) panel_slots += nb * panel_parts(q);
  const int upd_slots = upd_parts > 1 ? NB2 * upd_parts : 0;
  // tile-boundary trick (boundary && nb >= 2): per row p of the first tile,
  // S_p = sum_{k < nb-1} A(k0, j)[p, k] T(nb-1, k)^T split over parts of <= 128,
  // plus the reduced S_p block itself
  // With the boundary trick every block column q >= 1 of the first tile's panel
  // is formed the same way: S^q_p = sum_{k<q} A(k0, j)[p, k] T(q, k)^T (reduced
  // while leaf q runs), L(k0, j)[p, q] = (A(k0, j)[p, q] - S^q_p) X_q^T -- no
  // row of X_j on the path.
  const bool bnd = boundary && nb >= 2;
  // S^q_p sums l < q - 1 (the last term L(k0, j)[p, q-1] L(j, j)[q, q-1]^T goes
  // into the panel task through M_q, below) -- except row 0 of the last block
  // column, which the boundary leaf takes fully reduced (l < q)
  auto s_terms = [&](int q, int p) { return (q == nb - 1 && p == 0) ? q : q - 1; };
  auto s_parts = [&](int q) { return (q + 1) / 2; };  // the most parts of any row: K = 64 q, parts of <= 128
  std::vector<int> sq_part_base(static_cast<size_t>(nb) + 1, 0), sq_out_base(static_cast<size_t>(nb) + 1, 0);
  int s_slots = 0;
  if (bnd)
    for (int q = 1; q < nb; ++q) {
      sq_part_base[static_cast<size_t>(q)] = s_slots;
      s_slots += s_parts(q) > 1 ? nb * s_parts(q) : 0;
      sq_out_base[static_cast<size_t>(q)] = s_slots;
      s_slots += nb;
    }
  const int m_slots = bnd ? nb : 0;  // M_q = X_q L(j, j)[q, q-1] per block column
  const int sp_slots = bnd ? 2 * NB2 : 0;  // the two parts of each S-trick panel block
  const int slots_per_col = 2 * panel_slots + 2 * upd_slots + s_slots + m_slots + sp_slots;
  constexpr int kRing = 4;  // columns of partial slots in flight (see the reuse argument below)
  // counter spaces
  const long cAord = 0, cAfin = cAord + T * NB2, cLblk = cAfin + T, cLfin = cLblk + T * NB2,
             cXblk = cLfin + T, cXfin = cXblk + static_cast<long>(N) * NB2, cTblk = cXfin + N,
             cWfin = cTblk + static_cast<long>(N) * NB2, cXrow = cWfin + T, cArrive = cXrow + static_cast<long>(N) * nb,
             cSdone = cArrive + static_cast<long>(N) * slots_per_col, cUpl = cSdone + static_cast<long>(N) * NB2,
             cMdone = cUpl + N, cClip = cMdone + static_cast<long>(N) * nb, cRing = cClip + N, cEnd = cRing + N;
  P.upl = cUpl;
  P.counters = cEnd;
  const size_t t_doubles = static_cast<size_t>(N) * bp * bp;
  // one ring per elimination chain (columns [0, split) and [split, N)): the
  // chains run concurrently, so a column must not wait for a column of the
  // other chain to release its slots
  const bool two = split > 0 && split < N;
  P.scratch_doubles = t_doubles + static_cast<size_t>(two ? 2 : 1) * kRing * slots_per_col * kB * kB;
  P.logdet_doubles = static_cast<size_t>(N) * nb;
  auto aord = [&](long s, int p, int q) { return static_cast<int>(cAord + s * NB2 + p * nb + q); };
  auto afin = [&](long s) { return static_cast<int>(cAfin + s); };
  auto lblk = [&](long s, int p, int q) { return static_cast<int>(cLblk + s * NB2 + p * nb + q); };
  auto lfin = [&](long s) { return static_cast<int>(cLfin + s); };
  auto xblk = [&](int j, int p, int q) { return static_cast<int>(cXblk + static_cast<long>(j) * NB2 + p * nb + q); };
  auto xfin = [&](int j) { return static_cast<int>(cXfin + j); };
  auto tcnt = [&](int j, int p, int q) { return static_cast<int>(cTblk + static_cast<long>(j) * NB2 + p * nb + q); };
  auto wfin = [&](long s) { return static_cast<int>(cWfin + s); };
  auto xrowc = [&](int j, int q) { return static_cast<int>(cXrow + static_cast<long>(j) * nb + q); };
  auto sdone = [&](int j, int q, int p) { return static_cast<int>(cSdone + static_cast<long>(j) * NB2 + q * nb + p); };
  auto mdone = [&](int j, int q) { return static_cast<int>(cMdone + static_cast<long>(j) * nb + q); };
  // clipped part of column j's update of block (0, 0) of tile (k0, k0) done
  // (the boundary leaf applies the last term and is the block's one update signal)
  auto clipdone = [&](int j) { return static_cast<int>(cClip + j); };
  // ring release: split groups (and the boundary leaf) of column j finished with
  // the column's scratch ring slots
  auto ringdone = [&](int j) { return static_cast<int>(cRing + j); };
  // ring slot of column j (columns kRing apart share one)
  auto ring_of = [&](int j) {
    return static_cast<long long>(two && j >= split ? kRing + (j - split) % kRing : j % kRing);
  };
  const int xdone = nb * (nb + 1) / 2;
  const long long tsz = static_cast<long long>(bp) * bp;

  P.slot_tiles = F.tiles();
  Builder B(P);
  std::vector<int> ord(static_cast<size_t>(T), 0);  // update columns applied so far, per tile
  // grouped bulk updates (ugroup > 1): pending terms (source slots of L(a, k),
  // L(c, k)) per target slot, emitted as one multi-segment task per block with
  // ordinals ord .. ord + terms - 1 (its signals are repeated once per term, so
  // every waiter on an intermediate count is still woken)
  std::vector<std::vector<std::pair<long, long>>> pend(ugroup > 1 ? static_cast<size_t>(T) : 0);
  auto flush = [&](long ts) {
    if (ugroup <= 1 || ts < 0) return;
    auto& terms = pend[static_cast<size_t>(ts)];
    if (terms.empty()) return;
    const Coord tc = F.tiles()[static_cast<size_t>(ts)];
    const int u = ord[static_cast<size_t>(ts)];
    const int n = static_cast<int>(terms.size());
    ord[static_cast<size_t>(ts)] += n;
    for (int p = 0; p < nb; ++p)
      for (int q = 0; q < (tc.i == tc.j ? p + 1 : nb); ++q) {
        std::vector<Dep> d;
        for (const auto& tm : terms) {
          d.push_back({lfin(tm.first), NB2});
          if (tm.second != tm.first) d.push_back({lfin(tm.second), NB2});
        }
        d.push_back({aord(ts, p, q), u});
        std::vector<int> sg;
        for (int x = 0; x < n; ++x) {
          sg.push_back(aord(ts, p, q));
          if (tc.i != tc.j) sg.push_back(afin(ts));
        }
        DTask& t = B.add(1, d, sg);
        t.kind = kGemmTask;
        t.c_store = t.c0_store = kStoreA;
        t.c_off = t.c0_off = blk_off(ts, bp, p, q);
        t.m0 = p * kB;
        t.n0 = q * kB;
        for (const auto& tm : terms)
          B.seg(t, kStoreL, tile_off(tm.first, bp), kStoreL, tile_off(tm.second, bp), 0, bp, kTransB | kNegate);
      }
    terms.clear();
  };

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

  std::vector<int> ring_count(static_cast<size_t>(N), 0);
  // emission order of the columns: ascending, or -- two chains -- the chains'
  // columns interleaved by elimination step (column k runs at step k, or
  // k - split in the second chain).  Update ordinals follow emission order, so
  // a tile both chains update (separator, arrow) takes their terms in the order
  // they become available instead of all of the first chain's before any of
  // the second's (which serialised ~190 arrow-tip terms after the first chain
  // ended: the last ~7 ms of the large config's factor sweep).
  std::vector<int> seq;
  seq.reserve(static_cast<size_t>(N));
  if (two) {
    int a = 0, c = split;
    while (a < split || c < N) {
      if (c >= N || (a < split && a <= c - split)) seq.push_back(a++);
      else seq.push_back(c++);
    }
  } else {
    for (int j = 0; j < N; ++j) seq.push_back(j);
  }
  for (int jx = 0; jx < N; ++jx) {
    const int j = seq[static_cast<size_t>(jx)];
    const long ds = F.col_start(j);
    const int valid = static_cast<int>(std::min<long>(L.b, L.n - static_cast<long>(j) * L.b));
    std::vector<int> krows;
    std::vector<long> ks;
    for (const int* r = F.rows_begin(j); r != F.rows_end(j); ++r)
      if (*r > j) {
        krows.push_back(*r);
        ks.push_back(F.slot(*r, j));
      }
    // every tile this column reads or updates outside the grouped bulk terms
    if (ugroup > 1) {
      flush(ds);
      for (long sk : ks) flush(sk);
      if (!krows.empty()) flush(F.slot(krows[0], krows[0]));
      if (krows.size() > 1) flush(F.slot(krows[1], krows[0]));
    }
    const size_t col_first = B.all.size();
    const int U = ord[static_cast<size_t>(ds)];
    // first off-diagonal tile of the column and its update ordinals (the
    // progressive tail below), needed by the boundary leaf
    const bool tail0 = !krows.empty(), tail1 = krows.size() > 1;
    const long sk0 = tail0 ? ks[0] : -1;
    const long ts00 = tail0 ? F.slot(krows[0], krows[0]) : -1;
    const int Uk0 = tail0 ? ord[static_cast<size_t>(sk0)] : 0;
    int u00 = 0, u10 = 0;
    if (tail0) u00 = ord[static_cast<size_t>(ts00)]++;
    if (tail1) u10 = ord[static_cast<size_t>(F.slot(krows[1], krows[0]))]++;
    const bool bnd_col = bnd && tail0;
    auto s_off = [&](int q, int p) {  // reduced S^q_p block of this column (ring slot)
      return static_cast<long long>(t_doubles) +
             (ring_of(j) * slots_per_col + 2 * panel_slots + 2 * upd_slots +
              sq_out_base[static_cast<size_t>(q)] + p) *
                 kB * kB;
    };
    auto m_off = [&](int q) {  // M_q of this column (ring slot)
      return static_cast<long long>(t_doubles) +
             (ring_of(j) * slots_per_col + 2 * panel_slots + 2 * upd_slots + s_slots + q) * kB * kB;
    };
    // ---- diagonal-tile chain (queue 0): blocked POTRF + TRTRI of tile (j, j)
    // Fat leaf: factor + invert block (kk, kk), then (kk + 1 < nb, after the
    // second-phase dependencies) the next panel block L(kk+1, kk) = A(kk+1, kk)
    // X_kk^T and the next diagonal block update A(kk+1, kk+1) -= L L^T.
    auto leaf = [&](int kk) {
      std::vector<Dep> d{{aord(ds, kk, kk), U + kk}}, d2;
      std::vector<int> sg{lblk(ds, kk, kk), lfin(ds), xblk(j, kk, kk), xfin(j), xrowc(j, kk)};
      const bool fat = fat_leaf && kk + 1 < nb;
      // boundary leaf (last block of the tile): its second phase forms row 0 of
      // the first off-diagonal tile's last block column, L(k0, j)[0, nb-1] =
      // (A(k0, j)[0, nb-1] - S_0) X_{nb-1}^T, and the last update term of block
      // (0, 0) of tile (k0, k0) -- the next chain step's block
      const bool bleaf = bnd_col && kk == nb - 1;
      if (fat) {
        d2.push_back({aord(ds, kk + 1, kk), U + kk});
        d2.push_back({aord(ds, kk + 1, kk + 1), U + kk});
        sg.push_back(lblk(ds, kk + 1, kk));
        sg.push_back(lfin(ds));
        sg.push_back(aord(ds, kk + 1, kk + 1));
      } else if (bleaf) {
        d2.push_back({sdone(j, nb - 1, 0), 1});
        d2.push_back({afin(sk0), Uk0 * NB2});
        d2.push_back({clipdone(j), 1});
        sg.push_back(lblk(sk0, 0, nb - 1));
        sg.push_back(lfin(sk0));
        sg.push_back(aord(ts00, 0, 0));
        sg.push_back(ringdone(j));
      }
      DTask& t = B.add(0, d, sg, d2);
      t.sig2_count = fat ? 3 : (bleaf ? 4 : 0);
      t.kind = kLeafTask;
      // kCarry: the chain may keep the block this step updates last (the next
      // diagonal block) in shared memory for its next step -- always within a
      // tile; for a boundary leaf decided once the consumer is known (finish)
      t.mode = fat ? (2 | kCarry) : (bleaf ? 4 : 0);
      if (bleaf) t.aux0 = u00 + 1;  // block (0, 0) update count after this leaf
      if (bleaf) {
        t.p_off = blk_off(sk0, bp, 0, nb - 1);  // P in the A store; L(k0, j)[0, nb-1] at the same offset in L
        Seg sgx{};
        sgx.a_store = kStoreScratch;
        sgx.a_off = s_off(nb - 1, 0);            // S^{nb-1}_0
        sgx.b_store = kStoreA;
        sgx.b_off = blk_off(ts00, bp, 0, 0);     // next diagonal block
        sgx.lda = kB;  // S_0 is a 64x64 block
        sgx.ldb = bp;
        t.seg_begin = static_cast<int>(P.segs.size());
        t.seg_count = 1;
        P.segs.push_back(sgx);
        P.task_flops += 2.0 * kB * kB * kB * 2;
      }
      t.c_off = t.c0_off = t.cm_off = blk_off(ds, bp, kk, kk);
      t.diag_off = static_cast<long long>(j) * nb + kk;
      t.m0 = valid - kk * kB;
      t.n0 = static_cast<int>(static_cast<long>(j) * L.b + kk * kB);
      t.ldc = t.ldc0 = bp;
      if (kk + 1 < nb) P.zero.push_back(ZeroStrip{blk_off(ds, bp, kk, kk) + kB, nb - 1 - kk, 0});
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
    // X_j off-diagonal blocks, assembled right-looking so that row kk of X is
    // one task behind leaf kk:  T(kk, k) = sum_{l=k}^{kk-1} L(kk, l) X(l, k)
    // accumulated term by term (tterm, ascending l), X(kk, k) = -X(kk, kk) T(kk, k).
    auto tterm = [&](int kk, int k, int l) {
      DTask& t = B.add(0, {{lblk(ds, kk, l), 1}, {xblk(j, l, k), 1}, {tcnt(j, kk, k), l - k}}, {tcnt(j, kk, k)});
      t.kind = kGemmTask;
      t.c_store = kStoreScratch;
      t.c_off = tsz * j + static_cast<long long>(kk) * kB * bp + k * kB;
      if (l > k) {
        t.c0_store = kStoreScratch;
        t.c0_off = t.c_off;
      }
      B.seg(t, kStoreL, blk_off(ds, bp, kk, l), kStoreP1, blk_off(ds, bp, l, k), 0, kB, 0);
    };
    auto xrow = [&](int kk, int k) {
      DTask& t = B.add(0, {{xblk(j, kk, kk), 1}, {tcnt(j, kk, k), kk - k}}, {xblk(j, kk, k), xfin(j), xrowc(j, kk)});
      t.kind = kGemmTask;
      t.c_store = kStoreP1;
      t.c_off = blk_off(ds, bp, kk, k);
      B.seg(t, kStoreP1, blk_off(ds, bp, kk, kk), kStoreScratch,
            tsz * j + static_cast<long long>(kk) * kB * bp + k * kB, 0, kB, kNegate);
    };
    // ---- critical tail, progressive with the chain: the panels of the first
    // two off-diagonal tiles L(k, j) = A(k, j) X_j^T by block column q as soon
    // as row q of X_j is complete (split-K over parts of <= 128 when K > 256),
    // and the updates of tiles (k0, k0) -- the next diagonal tile when k0 = j+1
    // -- and (k1, k0) -- the next column's first panel tile -- split over
    // k-block pairs, each part issued once its panel columns exist.  The
    // reducer of an update waits (second phase) for the block's earlier updates.
    auto panel_prog = [&](size_t ia, int q, int queue, int slot_base) {
      const long sk = ks[ia];
      const int Uk = ord[static_cast<size_t>(sk)];
      const int parts = panel_parts(q), K = (q + 1) * kB;
      int base = slot_base;
      for (int qq = 0; qq < q; ++qq) base += panel_parts(qq) > 1 ? nb * panel_parts(qq) : 0;
      for (int p = 0; p < nb; ++p) {
        for (int r = 0; r < parts; ++r) {
          DTask& t = B.add(queue, {{afin(sk), Uk * NB2}, {xrowc(j, q), q + 1}}, {lblk(sk, p, q), lfin(sk)});
          t.kind = parts > 1 ? kSplitTask : kGemmTask;
          t.c_store = kStoreL;
          t.c_off = blk_off(sk, bp, p, q);
          t.m0 = p * kB;
          t.n0 = q * kB;
          if (parts > 1) {
            const int slot = base + p * parts;
            t.p_off = static_cast<long long>(t_doubles) +
                      (ring_of(j) * slots_per_col + slot) * kB * kB;
            t.aux0 = static_cast<int>(cArrive + static_cast<long>(j) * slots_per_col + slot);
            t.aux1 = (r << 8) | parts;
          }
          const int klo = parts > 1 ? r * 2 * kB : 0, khi = parts > 1 ? std::min(K, (r + 1) * 2 * kB) : K;
          B.seg(t, kStoreA, tile_off(sk, bp), kStoreP1, tile_off(ds, bp), klo, khi, kTransB);
        }
      }
    };
    // k-blocks [2r, 2r + 2) of the update of tile (krows[ia], krows[ic]); u = its ordinal
    // which: 0 every block, 1 all but block (0, 0), 2 only block (0, 0).  With
    // the boundary trick, block (0, 0) of tile (k0, k0) takes k < nb-1 only (the
    // chain applies the last term), so its parts are clipped and counted apart.
    auto update_split = [&](size_t ia, size_t ic, int r, int u, int queue, int slot_base, int which = 0) {
      const int a = krows[ia], c = krows[ic];
      const long ts = F.slot(a, c);
      if (ts < 0) throw Error(kErrConsistency, "update target outside the filled pattern");
      for (int p = 0; p < nb; ++p)
        for (int q = 0; q < (a == c ? p + 1 : nb); ++q) {
          const bool b00 = p == 0 && q == 0;
          if ((which == 1 && b00) || (which == 2 && !b00)) continue;
          const bool clip = bnd_col && ia == 0 && ic == 0 && b00;
          const int kend = clip ? nb - 1 : nb;
          const int klo = upd_parts > 1 ? 2 * r : 0, khi = upd_parts > 1 ? std::min(kend, 2 * r + 2) : kend;
          if (khi <= klo) continue;
          const int parts = upd_parts > 1 ? (clip ? nb / 2 : upd_parts) : 1;
          std::vector<Dep> d;
          for (int k = klo; k < khi; ++k) {
            d.push_back({lblk(ks[ia], p, k), 1});
            if (!(ia == ic && q == p)) d.push_back({lblk(ks[ic], q, k), 1});
          }
          std::vector<Dep> d2{{aord(ts, p, q), u}};
          if (parts == 1) d.insert(d.end(), d2.begin(), d2.end());
          std::vector<int> sg{aord(ts, p, q)};
          if (a != c) sg.push_back(afin(ts));
          if (clip) sg = {clipdone(j)};
          DTask& t = B.add(queue, d, sg, parts > 1 ? d2 : std::vector<Dep>{});
          t.kind = parts > 1 ? kSplitTask : kGemmTask;
          t.c_store = t.c0_store = kStoreA;
          t.c_off = t.c0_off = blk_off(ts, bp, p, q);
          t.m0 = p * kB;
          t.n0 = q * kB;
          if (upd_parts > 1) {
            // the parts of one block are emitted in different steps of the chain,
            // so their slots are addressed by block index
            const int slot = slot_base + (p * nb + q) * upd_parts;
            t.p_off = static_cast<long long>(t_doubles) +
                      (ring_of(j) * slots_per_col + slot) * kB * kB;
            t.aux0 = static_cast<int>(cArrive + static_cast<long>(j) * slots_per_col + slot);
            t.aux1 = (r << 8) | parts;
            if (parts == 1) t.kind = kGemmTask;
          }
          B.seg(t, kStoreL, tile_off(ks[ia], bp), kStoreL, tile_off(ks[ic], bp), klo * kB, khi * kB,
                kTransB | kNegate);
        }
    };
    const int upd_step_parts = upd_parts;  // parts issued at chain steps kk = 1, 3, 5, ... and nb - 1
    auto upd_part_at = [&](int kk) {
      if (upd_step_parts > 1) return (kk % 2 == 1 || kk == nb - 1) ? kk / 2 : -1;
      return kk == nb - 1 ? 0 : -1;
    };

    // S^q_p = sum_{l < q} L(k0, j)[p, l] L(j, j)[q, l]^T (= sum_{k<q} A(k0, j)[p, k]
    // T(q, k)^T, the right-looking form: no row of X_j needed), split-K over
    // parts of <= 128 in l; each part runs once its panel blocks exist
    auto s_tasks = [&](int q) {
      for (int p = 0; p < nb; ++p) {
        const int nt = s_terms(q, p);
        if (nt < 1) continue;
        const int K = nt * kB, sp = (nt + 1) / 2;
        for (int r = 0; r < sp; ++r) {
          const int klo = sp > 1 ? r * 2 * kB : 0, khi = sp > 1 ? std::min(K, (r + 1) * 2 * kB) : K;
          std::vector<Dep> d;
          for (int l = klo / kB; l < khi / kB; ++l) {
            d.push_back({lblk(sk0, p, l), 1});
            d.push_back({lblk(ds, q, l), 1});
          }
          DTask& t = B.add(0, d, {sdone(j, q, p)});
          t.kind = sp > 1 ? kSplitTask : kGemmTask;
          t.c_store = kStoreScratch;
          t.c_off = s_off(q, p);
          t.ldc = kB;
          if (sp > 1) {
            const int slot = 2 * panel_slots + 2 * upd_slots + sq_part_base[static_cast<size_t>(q)] + p * s_parts(q);
            t.p_off = static_cast<long long>(t_doubles) +
                      (ring_of(j) * slots_per_col + slot) * kB * kB;
            t.aux0 = static_cast<int>(cArrive + static_cast<long>(j) * slots_per_col + slot);
            t.aux1 = (r << 8) | sp;
          }
          for (int l = klo / kB; l < khi / kB; ++l)
            B.seg(t, kStoreL, blk_off(sk0, bp, p, l), kStoreL, blk_off(ds, bp, q, l), 0, kB, kTransB);
        }
      }
    };
    // M_q = X_q L(j, j)[q, q-1] (q >= 1), once leaf q and the panel block of
    // step q-1 exist: the last S term folded into the panel task,
    //   L(k0, j)[p, q-1] L(j, j)[q, q-1]^T X_q^T = L(k0, j)[p, q-1] M_q^T,
    // so each block column of the panel is one task after the previous one.
    auto m_task = [&](int q) {
      DTask& t = B.add(0, {{xblk(j, q, q), 1}, {lblk(ds, q, q - 1), 1}}, {mdone(j, q)});
      t.kind = kGemmTask;
      t.c_store = kStoreScratch;
      t.c_off = m_off(q);
      t.ldc = kB;
      B.seg(t, kStoreP1, blk_off(ds, bp, q, q), kStoreL, blk_off(ds, bp, q, q - 1), 0, kB, 0);
    };
    // L(k0, j)[p, q] = (A(k0, j)[p, q] - S^q_p) X_q^T - L(k0, j)[p, q-1] M_q^T
    // (for q = nb-1, row 0 is the chain's)
    auto s_panel = [&](int q) {
      const long long xd = blk_off(ds, bp, q, q);
      auto scratch_seg = [&](DTask& t, long long a_off, unsigned char bs, long long b_off, int ldb,
                             unsigned char as = kStoreScratch, int lda = kB) {
        Seg& sg = P.segs.emplace_back();
        sg = Seg{};
        sg.a_store = as;
        sg.a_off = a_off;
        sg.lda = lda;
        sg.b_store = bs;
        sg.b_off = b_off;
        sg.ldb = ldb;
        sg.k_lo = 0;
        sg.k_hi = kB;
        sg.flags = kTransB | kNegate;
        ++t.seg_count;
        P.task_flops += 2.0 * kB * kB * kB;
      };
      // two split parts, so the row's hop is only the last one (K = 64):
      //   part 0: (A - S) X_q^T  (X_q and S^q_p exist early)
      //   part 1: -L(k0, j)[p, q-1] M_q^T  (the previous block of the row)
      for (int p = q == nb - 1 ? 1 : 0; p < nb; ++p) {
        const bool has_s = s_terms(q, p) >= 1;
        const int slot = 2 * panel_slots + 2 * upd_slots + s_slots + m_slots + 2 * (q * nb + p);
        auto part = [&](int r, const std::vector<Dep>& d) -> DTask& {
          DTask& t = B.add(0, d, {lblk(sk0, p, q), lfin(sk0)});
          t.kind = kSplitTask;
          t.c_store = kStoreL;
          t.c_off = blk_off(sk0, bp, p, q);
          t.p_off = static_cast<long long>(t_doubles) +
                    (ring_of(j) * slots_per_col + slot) * kB * kB;
          t.aux0 = static_cast<int>(cArrive + static_cast<long>(j) * slots_per_col + slot);
          t.aux1 = (r << 8) | 2;
          return t;
        };
        std::vector<Dep> d0{{xblk(j, q, q), 1}, {afin(sk0), Uk0 * NB2}};
        if (has_s) d0.push_back({sdone(j, q, p), 1});
        DTask& t0 = part(0, d0);
        B.seg(t0, kStoreA, blk_off(sk0, bp, p, q), kStoreP1, xd, 0, kB, kTransB);
        if (has_s) scratch_seg(t0, s_off(q, p), kStoreP1, xd, bp);
        DTask& t1 = part(1, {{mdone(j, q), 1}, {lblk(sk0, p, q - 1), 1}});
        scratch_seg(t1, blk_off(sk0, bp, p, q - 1), kStoreScratch, m_off(q), kB, kStoreL, bp);
      }
    };
    for (int kk = 0; kk < nb; ++kk) {
      leaf(kk);
      if (kk + 1 < nb && !fat_leaf) {
        paneld(kk + 1, kk);
        traild(kk + 1, kk + 1, kk);
      }
      for (int k = 0; k < kk; ++k) xrow(kk, k);
      for (int k = 0; k <= kk && kk + 1 < nb; ++k) tterm(kk + 1, k, kk);
      for (int i = kk + 2; i < nb; ++i) paneld(i, kk);
      for (int p = kk + 1; p < nb; ++p)
        for (int i = p; i < nb; ++i)
          if (!(i == kk + 1 && p == kk + 1)) traild(i, p, kk);
      for (int kk2 = kk + 2; kk2 < nb; ++kk2)
        for (int k = 0; k <= kk; ++k) tterm(kk2, k, kk);
      if (tail0 && !bnd_col) {
        panel_prog(0, kk, 0, 0);
        const int r = upd_part_at(kk);
        if (r >= 0) update_split(0, 0, r, u00, 0, 2 * panel_slots);
      } else if (tail0) {
        if (kk == 0) {
          panel_prog(0, 0, 0, 0);
        } else {
          m_task(kk);
          s_panel(kk);
        }
        const int r = upd_part_at(kk);
        // the next diagonal tile's updates (all but block (0, 0)) go to the bulk
        // queue: in q0 their bursts at odd steps delayed the chain's helpers
        if (r >= 0) update_split(0, 0, r, u00, 1, 2 * panel_slots, 1);
        // block (0, 0): its clipped last part goes out one step early
        if (upd_parts > 1) {
          for (int rr = 0; rr < upd_parts; ++rr) {
            const int last = std::min(nb - 1, 2 * rr + 2) - 1;
            if (2 * rr < nb - 1 && last == kk) update_split(0, 0, rr, u00, 0, 2 * panel_slots, 2);
          }
        } else if (kk == nb - 2) {
          update_split(0, 0, 0, u00, 0, 2 * panel_slots, 2);
        }
        if (kk + 1 < nb) s_tasks(kk + 1);
      }
    }
    const bool coarse1 = two && coarse_second;
    if (tail1 && !coarse1) {
      // second tile: same progression, issued on the bulk queue right after the chain
      for (int kk = 0; kk < nb; ++kk) {
        panel_prog(1, kk, 1, panel_slots);
        const int r = upd_part_at(kk);
        if (r >= 0) update_split(1, 0, r, u10, 1, 2 * panel_slots + upd_slots);
      }
    }
    // ---- bulk (queue 1): the other panels, the other updates, deferred W
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
    auto update_with = [&](size_t ia, size_t ic, int u) {
      const int a = krows[ia], c = krows[ic];
      const long ts = F.slot(a, c);
      if (ts < 0) throw Error(kErrConsistency, "update target outside the filled pattern");
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
    auto update = [&](size_t ia, size_t ic) {
      const long ts = F.slot(krows[ia], krows[ic]);
      if (ts < 0) throw Error(kErrConsistency, "update target outside the filled pattern");
      if (ugroup > 1) {
        auto& terms = pend[static_cast<size_t>(ts)];
        terms.emplace_back(ks[ia], ks[ic]);
        if (static_cast<int>(terms.size()) >= ugroup) flush(ts);
        return;
      }
      update_with(ia, ic, ord[static_cast<size_t>(ts)]++);
    };
    // two chains (the sweep is throughput-bound, not chain-bound): the second
    // tile's panel and its update of tile (k1, k0) as whole-K bulk tasks
    // instead of the progressive split-K parts
    if (tail1 && coarse1) {
      panel(1);
      update_with(1, 0, u10);
    }
    for (size_t ia = 2; ia < krows.size(); ++ia) panel(ia);
    for (size_t ia = 2; ia < krows.size(); ++ia) update(ia, 0);
    for (size_t ic = 1; ic < krows.size(); ++ic)
      for (size_t ia = ic; ia < krows.size(); ++ia) update(ia, ic);
    // scratch ring: every split group of column j (and its boundary leaf, which
    // reads S_0) signals ringdone(j) when done with the column's ring slots;
    // the ring writers of column j wait for the column that used the same
    // slots before (kRing columns earlier) to be done with them -- implied by
    // the data dependencies on band patterns, required for any other
    {
      std::set<int> groups;  // arrival counters (parts of one group are not contiguous)
      for (size_t x = col_first; x < B.all.size(); ++x) {
        DTask& t = B.all[x];
        if (t.kind != kSplitTask) continue;
        groups.insert(t.aux0);
        B.add_sig(t, ringdone(j));
      }
      ring_count[static_cast<size_t>(j)] = static_cast<int>(groups.size()) + (bnd_col ? 1 : 0);
      const int prev = j - kRing;
      const bool same_chain = !(two && j >= split && prev < split);
      if (prev >= 0 && same_chain && ring_count[static_cast<size_t>(prev)] > 0)
        for (size_t x = col_first; x < B.all.size(); ++x) {
          DTask& t = B.all[x];
          const bool writer = t.kind == kSplitTask || (t.kind == kGemmTask && t.c_store == kStoreScratch &&
                                                        t.c_off >= static_cast<long long>(t_doubles));
          if (writer) B.add_dep(t, {ringdone(prev), ring_count[static_cast<size_t>(prev)]});
        }
    }
    if (jx - defer_w >= 0) emit_w(seq[static_cast<size_t>(jx - defer_w)]);
  }
  for (int jx = std::max(0, N - defer_w); jx < N; ++jx) emit_w(seq[static_cast<size_t>(jx)]);
  for (long ts = 0; ts < (ugroup > 1 ? T : 0); ++ts) flush(ts);  // none left on a consistent pattern
  // streamed upload: each task polls the upload counter of the latest tile
  // column of A it reads or writes
  {
    // upload order: column c by the first elimination step that touches it --
    // step k reads column k and updates the tiles (r, c) of every c with
    // (c, k) in F -- where the steps of the two chains (split) run side by
    // side: step k comes at time k, or k - split in the second chain
    std::vector<int> first(static_cast<size_t>(N));
    auto when = [&](int k) { return two && k >= split ? k - split : k; };
    for (int c = 0; c < N; ++c) first[static_cast<size_t>(c)] = when(c);
    for (const Coord& t : F.tiles())
      if (t.i > t.j) first[static_cast<size_t>(t.i)] = std::min(first[static_cast<size_t>(t.i)], when(t.j));
    P.upload_order.resize(static_cast<size_t>(N));
    for (int c = 0; c < N; ++c) P.upload_order[static_cast<size_t>(c)] = c;
    std::stable_sort(P.upload_order.begin(), P.upload_order.end(),
                     [&](int x, int y) { return first[static_cast<size_t>(x)] < first[static_cast<size_t>(y)]; });
    std::vector<int> rank(static_cast<size_t>(N));
    for (int r = 0; r < N; ++r) rank[static_cast<size_t>(P.upload_order[static_cast<size_t>(r)])] = r;
    auto later = [&](int a, int b) { return a < 0 ? b : (b < 0 ? a : (rank[static_cast<size_t>(b)] > rank[static_cast<size_t>(a)] ? b : a)); };
    const long long tsz2 = static_cast<long long>(bp) * bp;
    auto col_of = [&](long long off) { return F.tiles()[static_cast<size_t>(off / tsz2)].j; };
    for (DTask& t : B.all) {
      int c = -1;
      if (t.kind == kLeafTask) {
        c = col_of(t.c_off);
        if (t.mode & 4) c = later(c, col_of(P.segs[static_cast<size_t>(t.seg_begin)].b_off));
        if (t.mode & 4) c = later(c, col_of(t.p_off));
      } else {
        if (t.c_store == kStoreA) c = later(c, col_of(t.c_off));
        if (t.c0_store == kStoreA) c = later(c, col_of(t.c0_off));
        for (int k = t.seg_begin; k < t.seg_begin + t.seg_count; ++k) {
          const Seg& g = P.segs[static_cast<size_t>(k)];
          if (g.a_store == kStoreA) c = later(c, col_of(g.a_off));
          if (g.b_store == kStoreA) c = later(c, col_of(g.b_off));
        }
      }
      t.poll = c >= 0 ? static_cast<int>(cUpl + c) : -1;
    }
  }
  B.finish(crit_workers, chain, two ? split : -1);
  return P;
}

DataflowPlan build_phase1_dataflow(const Pattern& F) {
  DataflowPlan P;
  P.L = F.layout();
  const Layout& L = P.L;
  const int bp = (L.b + kB - 1) / kB * kB, nb = bp / kB, NB2 = nb * nb;
  P.bp = bp;
  P.nb = nb;
  const long T = static_cast<long>(F.size());
  const int N = L.N;
  // counters: X blocks and per-column X completion, T-term accumulation
  // ordinals, W completion per tile
  const long cXblk = 0, cXfin = cXblk + static_cast<long>(N) * NB2, cTblk = cXfin + N,
             cWfin = cTblk + static_cast<long>(N) * NB2, cEnd = cWfin + T;
  P.counters = cEnd;
  const size_t t_doubles = static_cast<size_t>(N) * bp * bp;
  P.scratch_doubles = t_doubles;
  P.logdet_doubles = static_cast<size_t>(N) * nb;
  auto xblk = [&](int j, int p, int q) { return static_cast<int>(cXblk + static_cast<long>(j) * NB2 + p * nb + q); };
  auto xfin = [&](int j) { return static_cast<int>(cXfin + j); };
  auto tcnt = [&](int j, int p, int q) { return static_cast<int>(cTblk + static_cast<long>(j) * NB2 + p * nb + q); };
  auto wfin = [&](long s) { return static_cast<int>(cWfin + s); };
  const int xdone = nb * (nb + 1) / 2;
  const long long tsz = static_cast<long long>(bp) * bp;
  P.slot_tiles = F.tiles();
  Builder B(P);
  for (int j = 0; j < N; ++j) {
    const long ds = F.col_start(j);
    const int valid = static_cast<int>(std::min<long>(L.b, L.n - static_cast<long>(j) * L.b));
    // X_j = L_jj^{-1}: every 64-block leaf inverts its (given) diagonal block of L
    // at once; the blocks below the diagonal follow right-looking, T(kk, k) =
    // sum_{l=k}^{kk-1} L(kk, l) X(l, k) term by term, X(kk, k) = -X(kk, kk) T(kk, k)
    for (int kk = 0; kk < nb; ++kk) {
      DTask& t = B.add(1, {}, {xblk(j, kk, kk), xfin(j)});
      t.kind = kLeafTask;
      t.mode = 1;  // invert only: the input block (A-store slot of the sweep's table = L) is a factor block
      t.c_off = t.c0_off = t.cm_off = blk_off(ds, bp, kk, kk);
      t.diag_off = static_cast<long long>(j) * nb + kk;
      t.m0 = valid - kk * kB;
      t.n0 = static_cast<int>(static_cast<long>(j) * L.b + kk * kB);
      if (kk + 1 < nb) P.zero.push_back(ZeroStrip{blk_off(ds, bp, kk, kk) + kB, nb - 1 - kk, 0});
      P.task_flops += 2.0 * (kB * kB * kB / 6.0);
    }
    for (int kk = 1; kk < nb; ++kk)
      for (int k = 0; k < kk; ++k) {
        for (int l = k; l < kk; ++l) {
          DTask& t = B.add(1, {{xblk(j, l, k), 1}, {tcnt(j, kk, k), l - k}}, {tcnt(j, kk, k)});
          t.kind = kGemmTask;
          t.c_store = kStoreScratch;
          t.c_off = tsz * j + static_cast<long long>(kk) * kB * bp + k * kB;
          if (l > k) {
            t.c0_store = kStoreScratch;
            t.c0_off = t.c_off;
          }
          B.seg(t, kStoreL, blk_off(ds, bp, kk, l), kStoreP1, blk_off(ds, bp, l, k), 0, kB, 0);
        }
        DTask& t = B.add(1, {{xblk(j, kk, kk), 1}, {tcnt(j, kk, k), kk - k}}, {xblk(j, kk, k), xfin(j)});
        t.kind = kGemmTask;
        t.c_store = kStoreP1;
        t.c_off = blk_off(ds, bp, kk, k);
        B.seg(t, kStoreP1, blk_off(ds, bp, kk, kk), kStoreScratch, tsz * j + static_cast<long long>(kk) * kB * bp + k * kB,
              0, kB, kNegate);
      }
    // W_kj = L_kj X_j (trmm_tile(kRight, kTrans) by U_j^T, selinv.cpp:203-216)
    for (const int* r = F.rows_begin(j); r != F.rows_end(j); ++r) {
      if (*r <= j) continue;
      const long sk = F.slot(*r, j);
      for (int p = 0; p < nb; ++p)
        for (int q = 0; q < nb; ++q) {
          DTask& t = B.add(1, {{xfin(j), xdone}}, {wfin(sk)});
          t.kind = kGemmTask;
          t.c_store = kStoreP1;
          t.c_off = blk_off(sk, bp, p, q);
          t.m0 = p * kB;
          t.n0 = q * kB;
          B.seg(t, kStoreL, tile_off(sk, bp), kStoreP1, tile_off(ds, bp), q * kB, bp, 0);
        }
    }
  }
  B.finish(0);
  return P;
}

DataflowPlan build_phase2_dataflow(const Pattern& F, const Closure& sel, int crit_workers, int split, int group) {
  DataflowPlan P;
  P.L = F.layout();
  const int bp = (P.L.b + kB - 1) / kB * kB, nb = bp / kB, NB2 = nb * nb;
  P.bp = bp;
  P.nb = nb;
  const Pattern& C = sel.closure;
  const long Tc = static_cast<long>(C.size());
  const int N = P.L.N;
  // Split-K partial slots: per column, the parts of its late (critical) targets,
  // on a ring of kRing columns.  A column's split parts additionally wait for
  // the targets of the column kRing places later in processing order, which
  // frees the ring slot (implied by the data dependencies on band patterns,
  // enforced for any other closure).
  constexpr int kRing = 4;
  // late terms are split-K parts of `group` terms each (K = 512 * group at b = 512)
  const int G = std::max(1, group);
  auto groups = [&](int terms) { return (terms + G - 1) / G; };
  std::vector<int> col_slots(static_cast<size_t>(N), 0);
  std::vector<std::vector<int>> Kof(static_cast<size_t>(N));
  for (const ColumnWork& cw : sel.columns) {
    const int i = cw.col;
    std::vector<int>& K = Kof[static_cast<size_t>(i)];
    for (const int* r = F.rows_begin(i); r != F.rows_end(i); ++r)
      if (*r > i) K.push_back(*r);
    if (K.empty()) continue;
    const int kc = K[0];
    int n = 0;
    for (int j : cw.offdiag_rows) {
      int late = 0;
      for (int k : K) late += std::min(j, k) == kc ? 1 : 0;
      const int g = groups(late);
      if (g > 1) n += NB2 * g;
    }
    if (cw.diagonal) n += nb * (nb + 1) / 2 * (1 + groups(static_cast<int>(K.size())));
    col_slots[static_cast<size_t>(i)] = n;
  }
  const int slots_per_col = *std::max_element(col_slots.begin(), col_slots.end());
  const long cSpart = 0, cSfin = cSpart + Tc * NB2, cArrive = cSfin + Tc;
  P.counters = cArrive + static_cast<long>(N) * slots_per_col;
  // two-chain order (split > 0): the columns below the split are a second,
  // independent chain once the columns above are done -- its own ring, so
  // it does not wait for the other chain's columns to release slots
  const bool two = split > 0 && split < N;
  P.scratch_doubles = static_cast<size_t>(two ? 2 : 1) * kRing * slots_per_col * kB * kB;
  auto ring_slot = [&](int i) { return two && i < split ? kRing + i % kRing : i % kRing; };
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
  // completion deps of every target of a column (ring-slot release)
  std::vector<std::vector<Dep>> col_done(static_cast<size_t>(N));
  for (const ColumnWork& cw : sel.columns) {
    const int i = cw.col;
    for (int j : cw.offdiag_rows) col_done[static_cast<size_t>(i)].push_back({sfin(cslot(j, i)), NB2});
    if (cw.diagonal) col_done[static_cast<size_t>(i)].push_back({sfin(cslot(i, i)), nb * (nb + 1) / 2});
  }
  P.slot_tiles = C.tiles();
  Builder B(P);
  for (size_t ci = 0; ci < sel.columns.size(); ++ci) {
    const ColumnWork& cw = sel.columns[ci];
    const int i = cw.col;
    const std::vector<int>& K = Kof[static_cast<size_t>(i)];
    const int kcrit = K.empty() ? -1 : K[0];
    // ring release: the column processed kRing steps earlier on the same ring
    // must be complete
    std::vector<Dep> ring_deps;
    {
      int seen = 0;
      for (size_t cj = ci; cj-- > 0;) {
        const int pc = sel.columns[cj].col;
        if (two && ((pc < split) != (i < split))) continue;
        if (++seen == kRing) {
          ring_deps = col_done[static_cast<size_t>(pc)];
          break;
        }
      }
    }
    int slot_next = 0;
    auto take = [&](int parts, DTask& t, int part, int base) {
      t.kind = kSplitTask;
      t.p_off = (static_cast<long long>(ring_slot(i)) * slots_per_col + base) * kB * kB;
      t.aux0 = static_cast<int>(cArrive + static_cast<long>(i) * slots_per_col + base);
      t.aux1 = (part << 8) | parts;
    };
    auto mseg = [&](DTask& t, int j, int k) {
      const long ms = cslot(std::max(j, k), std::min(j, k));
      B.seg(t, kStoreSigma, tile_off(ms, bp), kStoreP1, tile_off(F.slot(k, i), bp), 0, bp,
            (k > j ? kTransA : 0) | kNegate);
    };
    auto mdep = [&](int j, int k) {
      const long ms = cslot(std::max(j, k), std::min(j, k));
      return Dep{sfin(ms), final_count(ms)};
    };
    // off-diagonal targets: Sigma_ji = -sum_k M_jk W_ki.  Terms whose M tile
    // lies in column kcrit (the column processed just before) are late; the
    // others (older columns) form one early task that runs ahead.
    for (int j : cw.offdiag_rows) {
      const long ts = cslot(j, i);
      std::vector<int> early, late;
      for (int k : K) (std::min(j, k) == kcrit ? late : early).push_back(k);
      const int parts = groups(static_cast<int>(late.size()));
      for (int p = 0; p < nb; ++p)
        for (int q = 0; q < nb; ++q) {
          if (!early.empty()) {
            std::vector<Dep> d;
            for (int k : early) d.push_back(mdep(j, k));
            std::sort(d.begin(), d.end(), [](const Dep& x, const Dep& y) { return x.counter < y.counter; });
            d.erase(std::unique(d.begin(), d.end(), [](const Dep& x, const Dep& y) { return x.counter == y.counter; }),
                    d.end());
            DTask& t = B.add(1, d, {late.empty() ? sfin(ts) : spart(ts, p, q)});
            t.kind = kGemmTask;
            t.c_store = kStoreSigma;
            t.c_off = blk_off(ts, bp, p, q);
            t.m0 = p * kB;
            t.n0 = q * kB;
            for (int k : early) mseg(t, j, k);
          }
          const int base = slot_next;
          for (int r = 0; r < parts; ++r) {
            const size_t g0 = static_cast<size_t>(r) * G, g1 = std::min(late.size(), g0 + G);
            std::vector<Dep> d;
            for (size_t x = g0; x < g1; ++x) d.push_back(mdep(j, late[x]));
            std::sort(d.begin(), d.end(), [](const Dep& x, const Dep& y) { return x.counter < y.counter; });
            d.erase(std::unique(d.begin(), d.end(), [](const Dep& x, const Dep& y) { return x.counter == y.counter; }),
                    d.end());
            std::vector<Dep> d2;
            if (!early.empty()) d2.push_back({spart(ts, p, q), 1});
            if (parts > 1) d.insert(d.end(), ring_deps.begin(), ring_deps.end());
            else d.insert(d.end(), d2.begin(), d2.end());
            DTask& t = B.add(1, d, {sfin(ts)}, parts > 1 ? d2 : std::vector<Dep>{});
            t.kind = kGemmTask;
            t.c_store = kStoreSigma;
            t.c_off = blk_off(ts, bp, p, q);
            if (!early.empty()) {
              t.c0_store = kStoreSigma;
              t.c0_off = t.c_off;
            }
            t.m0 = p * kB;
            t.n0 = q * kB;
            if (parts > 1) take(parts, t, r, base);
            for (size_t x = g0; x < g1; ++x) mseg(t, j, late[x]);
          }
          if (parts > 1) slot_next += parts;
        }
    }
    // diagonal target: Sigma_ii = X_i^T X_i - sum_k W_ki^T Sigma_ki (LAUUM +
    // one part per term, all depending on this column's off-diagonal tiles),
    // lower part mirrored exactly, diagonal -> marginal variances.
    if (cw.diagonal) {
      const long dsl = cslot(i, i);
      const long xs = F.col_start(i);
      const int parts = 1 + groups(static_cast<int>(K.size()));
      for (int p = 0; p < nb; ++p)
        for (int q = 0; q <= p; ++q) {
          const int base = slot_next;
          for (int r = 0; r < parts; ++r) {
            std::vector<Dep> d;
            const size_t g0 = r == 0 ? 0 : static_cast<size_t>(r - 1) * G, g1 = r == 0 ? 0 : std::min(K.size(), g0 + G);
            if (r == 0) {
              // the LAUUM part runs when the column becomes active
              if (kcrit >= 0 && C.slot(kcrit, kcrit) >= 0) d.push_back(mdep(kcrit, kcrit));
            } else {
              for (size_t x = g0; x < g1; ++x) d.push_back({sfin(cslot(K[x], i)), NB2});
            }
            if (parts > 1) d.insert(d.end(), ring_deps.begin(), ring_deps.end());
            DTask& t = B.add(0, d, {sfin(dsl)});
            t.kind = kGemmTask;
            t.c_store = kStoreSigma;
            t.c_off = blk_off(dsl, bp, p, q);
            t.m0 = p * kB;
            t.n0 = q * kB;
            if (p == q) {
              t.mode = kSymDiag;
              t.diag_store = kStoreVar;
              t.diag_off = static_cast<long long>(i) * bp + p * kB;
            } else {
              t.mode = kMirror;
              t.cm_store = kStoreSigma;
              t.cm_off = blk_off(dsl, bp, q, p);
            }
            if (parts > 1) take(parts, t, r, base);
            if (r == 0) {
              // U U^T = X^T X; rows >= p*64 of X carry the nonzeros for block row p >= q
              B.seg(t, kStoreP1, tile_off(xs, bp), kStoreP1, tile_off(xs, bp), p * kB, bp, kTransA);
            } else {
              for (size_t x = g0; x < g1; ++x) {
                const int k = K[x];
                B.seg(t, kStoreP1, tile_off(F.slot(k, i), bp), kStoreSigma, tile_off(cslot(k, i), bp), 0, bp,
                      kTransA | kNegate);
              }
            }
          }
          if (parts > 1) slot_next += parts;
        }
    }
  }
  B.finish(crit_workers);
  return P;
}

}  // namespace tib
