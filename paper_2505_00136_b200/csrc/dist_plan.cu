// Multi-GPU schedule of the tiled GP: the per-rank operation lists (gpb200.h
// schedule IR) of the 2D block-cyclic tiled Cholesky, the beta / alpha solves
// and the replica-free gradient.  Host code only; the device executor is
// dist.cu, the CPU interpreter tests/dist_interp.py.
//
// Process grid P x Q, rank = p Q + q; lower tile (i, j) on rank
// (i mod P) Q + (j mod Q).  Per panel k of the right-looking
// tiled Cholesky (taskgp tiled.py:168-204):
//   POTRF(k) on the owner of (k, k); L_kk^-1 down process column k mod Q;
//   TRSM: column k mod Q solves its tiles (i, k) into the row-panel buffer;
//   row stage: each process row p broadcasts its share of the panel from
//     rank (p, k mod Q) along the row (row communicator, one call);
//   column stage: rank (p', q) packs the panel tiles j = p' (mod P),
//     j = q (mod Q) into the column-panel buffer and broadcasts them down
//     process column q (column communicator, P calls);
//   the trailing updates read A from the row panel and B from the column panel.
// Panels are grouped exactly as on one GPU (plan_common.h): in-group updates
// (K = b) and the next group's columns (K = G' b) on the high-priority critical
// stream, the rest of the trailing update (K = G' b) on the main stream.  Every
// tile receives the same sequence of GEMMs with the same K split as in the
// single-GPU plan, so the factor is bitwise the single-GPU one.
#include <algorithm>
#include <cstdlib>
#include <string>

#include "dist_plan.h"
#include "plan_common.h"

namespace gpb {

namespace {

constexpr int kBlk = 128;  // GEMM block (gemm.cuh GBM = GBN)
enum { MAIN = 0, CRIT = 1 };
enum { WORLD = 0, ROWG = 1, COLG = 2 };

struct Ref {
  int buf;
  int64_t off;
};

class Builder {
 public:
  std::vector<gpb_op>* ops;
  std::vector<gpb_op_job>* jobs;

  gpb_op base(int kind, int stream) {
    gpb_op o{};
    o.kind = kind;
    o.stream = stream;
    o.buf[0] = o.buf[1] = o.buf[2] = -1;
    return o;
  }
  void push(const gpb_op& o) { ops->push_back(o); }
  void zero(int stream, Ref a, int64_t count) {
    if (count <= 0) return;
    gpb_op o = base(GPB_OP_ZERO, stream);
    o.buf[0] = a.buf;
    o.off[0] = a.off;
    o.count = count;
    push(o);
  }
  void record(int stream, int ev) {
    gpb_op o = base(GPB_OP_RECORD, stream);
    o.i = ev;
    push(o);
  }
  void wait(int stream, int ev) {
    gpb_op o = base(GPB_OP_WAIT, stream);
    o.i = ev;
    push(o);
  }
  void coll(int kind, int stream, int group, int root, Ref a, int64_t count) {
    if (count <= 0) return;
    gpb_op o = base(kind, stream);
    o.group = group;
    o.root = root;
    o.buf[0] = a.buf;
    o.off[0] = a.off;
    o.count = count;
    push(o);
  }
  // job list helpers: start a list, add jobs, close it into an op
  size_t j0 = 0;
  void begin() { j0 = jobs->size(); }
  void job(Ref a, Ref b, Ref cin, Ref cout, int k = 0, int lower = 0, int i = 0, int j = 0) {
    gpb_op_job q{};
    const Ref r[4] = {a, b, cin, cout};
    for (int t = 0; t < 4; ++t) {
      q.buf[t] = r[t].buf;
      q.off[t] = r[t].off;
    }
    q.k = k;
    q.lower = lower;
    q.i = i;
    q.j = j;
    jobs->push_back(q);
  }
  int64_t pending() const { return static_cast<int64_t>(jobs->size() - j0); }
  // close the open job list into `o` (dropped when empty)
  void close(gpb_op o) {
    o.job0 = static_cast<int64_t>(j0);
    o.njobs = pending();
    if (o.njobs > 0) push(o);
  }
  gpb_op gemm(int stream, int mblk, int nblk, int64_t ld, bool ak, bool bk, double alpha, double beta) {
    gpb_op o = base(GPB_OP_GEMM, stream);
    o.mblk = mblk;
    o.nblk = nblk;
    o.lda = o.ldb = o.ldc = ld;
    o.ak = ak;
    o.bk = bk;
    o.alpha = alpha;
    o.beta = beta;
    return o;
  }
};

const Ref kNone{-1, 0};

}  // namespace

// group sizes of the factorisation (plan_common.h; the planes' rule on large grids as on one GPU)
std::vector<int> dist_group_sizes(const DistLayout& L) {
  return L.planes > 0 && L.Ti >= 48 ? chol_group_sizes(L.Ti, L.G, 4, 0) : chol_group_sizes(L.Ti, L.G);
}

int col_pos(const DistLayout& L, int j) {
  int c = 0;
  for (int t = 0; t < j; ++t)
    if (t % L.P == j % L.P && t % L.Q == j % L.Q) ++c;
  return c;
}

int col_cnt_max(const DistLayout& L, int q) {
  std::vector<int> cnt(L.P, 0);
  for (int j = q; j < L.Ti; j += L.Q) ++cnt[j % L.P];
  return *std::max_element(cnt.begin(), cnt.end());
}

int dist_layout(int rank, int world, int P, int Q, int64_t n, int64_t T, DistLayout* out, std::string* err,
                int exchange) {
  DistLayout& L = *out;
  if (world < 1 || P < 1 || Q < 1 || P * Q != world || rank < 0 || rank >= world) {
    if (err) *err = "process grid " + std::to_string(P) + " x " + std::to_string(Q) + " does not match " +
                    std::to_string(world) + " ranks (rank " + std::to_string(rank) + ")";
    return GPB_INVALID_CONFIG;
  }
  int64_t lay[6];
  if (int s = gpb_layout(n, T, lay)) {
    if (err) *err = "tiles_per_dim=" + std::to_string(T) + " must divide the " + std::to_string(n) +
                    " training points";
    return s;
  }
  L = DistLayout();
  L.rank = rank;
  L.world = world;
  L.P = P;
  L.Q = Q;
  L.my_p = rank / Q;
  L.my_q = rank % Q;
  L.n = n;
  L.bi = static_cast<int>(lay[0]);
  L.Ti = static_cast<int>(lay[1]);
  L.np_ = lay[2];
  L.bp_user = static_cast<int>(lay[3]);
  L.b_user = static_cast<int>(lay[4]);
  L.bi2 = int64_t(L.bi) * L.bi;
  // Trailing updates on the tcgen05 int8 pipe (ozaki.cuh), as on one GPU: GPB_OZAKI planes
  // per operand (default 8), for 512-wide tiles (the smaller grids of the tests keep the
  // DMMA kernels and stay bitwise equal to the single-GPU DMMA factor); GPB_DIST_PLANES=0: off
  {
    const char* e = getenv("GPB_OZAKI");
    int planes = e ? atoi(e) : 8;
    planes = planes <= 0 ? 0 : std::min(8, std::max(4, planes));
    const char* d = getenv("GPB_DIST_PLANES");
    L.planes = (L.bi >= 512 && !(d && atoi(d) == 0)) ? planes : 0;
  }
  // panels per group: plan_common.h; with the planes the single-GPU rule (gpb_api.cu choose_panels)
  L.G = chol_panels(L.Ti);
  if (L.planes > 0 && !getenv("GPB_PANELS")) L.G = L.Ti >= 48 ? 8 : L.Ti >= 16 ? 4 : L.G;
  const int Ti = L.Ti;
  L.slot.assign(size_t(Ti) * Ti, -1);
  for (int i = 0; i < Ti; ++i)
    for (int j = 0; j <= i; ++j)
      if (L.owner(i, j) == rank) {
        L.slot[size_t(i) * Ti + j] = L.nown();
        L.own_i.push_back(i);
        L.own_j.push_back(j);
      }
  L.rows_per = (Ti + P - 1) / P;
  std::vector<int> cnt(P, 0);
  L.jpos.assign(Ti, -1);
  for (int j = 0; j < Ti; ++j)
    if (j % Q == L.my_q) L.jpos[j] = cnt[j % P]++;
  L.cnt_max = *std::max_element(cnt.begin(), cnt.end());
  std::vector<int> cr(Q, 0);
  L.rpos.assign(Ti, -1);
  for (int r = 0; r < Ti; ++r)
    if (r % P == L.my_p) L.rpos[r] = cr[r % Q]++;
  L.cntx = *std::max_element(cr.begin(), cr.end());
  const int64_t bi2 = L.bi2, nown = std::max(1, L.nown());
  L.bufsz[GPB_BUF_L] = nown * bi2;
  L.bufsz[GPB_BUF_DINV] = int64_t(Ti) * bi2;
  L.bufsz[GPB_BUF_ROW] = 2 * int64_t(L.G) * L.rows_per * bi2;
  L.bufsz[GPB_BUF_COL] = P > 1 ? 2 * int64_t(P) * L.G * std::max(1, L.cnt_max) * bi2 : 0;
  // vector slots start on 256-byte boundaries (the copy kernels move 16-byte words);
  // BETA, ALPHA, LOGDIAG stay contiguous for the one replicating all-reduce
  const int64_t np_ = L.np_;
  auto up = [](int64_t x) { return (x + 31) / 32 * 32; };
  L.vec[V_Y] = 0;
  L.vec[V_BETA] = up(np_);
  L.vec[V_ALPHA] = L.vec[V_BETA] + np_;
  L.vec[V_LOGDIAG] = L.vec[V_ALPHA] + np_;
  L.vec[V_ACC] = up(L.vec[V_LOGDIAG] + Ti);
  L.vec[V_TMP] = up(L.vec[V_ACC] + np_);
  L.vec[V_RECV] = up(L.vec[V_TMP] + L.bi);
  L.vec[V_RED] = up(L.vec[V_RECV] + L.bi);
  L.bufsz[GPB_BUF_VEC] = L.vec[V_RED] + 32;
  L.bufsz[GPB_BUF_X] = nown * bi2;
  L.bufsz[GPB_BUF_KINV] = nown * bi2;
  // gradient exchange buffers: two sets (row k + 1 is published while step k reads row k)
  L.bufsz[GPB_BUF_XCOL] = P > 1 ? 2 * int64_t((Ti + Q - 1) / Q) * bi2 : 0;
  L.bufsz[GPB_BUF_XROW] = Q > 1 ? 2 * int64_t(Q) * std::max(1, L.cntx) * bi2 : 0;
  L.bufsz[GPB_BUF_LCOL] = Q > 1 ? 2 * int64_t(L.rows_per) * bi2 : 0;
  const int ng = static_cast<int>(dist_group_sizes(L).size());
  L.p2p = exchange == 1 && world > 1;
  L.nevents = std::max(3 * ng + 2, 2 * Ti + 1);  // factorisation / gradient schedules
  return GPB_OK;
}

namespace {

// ---- phase 0: assembly + factorisation ------------------------------------
void plan_factor(const DistLayout& L, Builder& b) {
  const int Ti = L.Ti, bi = L.bi, nb = bi / kBlk, P = L.P, Q = L.Q, G = L.G;
  const int64_t bi2 = L.bi2;
  auto slot = [&](int i, int j) { return L.slot[size_t(i) * Ti + j]; };
  auto lt = [&](int i, int j) { return Ref{GPB_BUF_L, int64_t(slot(i, j)) * bi2}; };
  auto rowt = [&](int set, int g, int i) {
    return Ref{GPB_BUF_ROW, ((int64_t(set) * G + g) * L.rows_per + i / P) * bi2};
  };
  // column-panel tile j (j mod Q == my_q); with P == 1 the row panel holds every row
  auto colt = [&](int set, int g, int j) {
    if (P == 1) return rowt(set, g, j);
    return Ref{GPB_BUF_COL, (((int64_t(set) * P + j % P) * G + g) * L.cnt_max + L.jpos[j]) * bi2};
  };
  const int64_t a_walk = int64_t(L.rows_per) * bi2;
  const int64_t b_walk = P == 1 ? a_walk : int64_t(L.cnt_max) * bi2;
  const std::vector<int> sizes = dist_group_sizes(L);
  const int ng = static_cast<int>(sizes.size());
  const int ev_start = 0, ev_end = 1 + 3 * ng;
  auto ev_panel = [&](int s) { return 1 + s; };
  auto ev_upd = [&](int s) { return 1 + ng + s; };
  auto ev_next = [&](int s) { return 1 + 2 * ng + s; };

  // ---- peer-memory exchange (L.p2p): who sends panel k's tiles to whom.
  // Tile i > k of panel k is solved by rank (i mod P, k mod Q); process row
  // i mod P reads it from its row panel, process column i mod Q from its
  // column panel (with P == 1 the row panel serves both).
  auto has_rows = [&](int pp, int k) {  // a panel tile i > k in process row pp
    for (int i = k + 1; i < Ti; ++i)
      if (i % P == pp) return true;
    return false;
  };
  auto has_tiles = [&](int pp, int q, int k) {  // ... that process column q reads
    for (int i = k + 1; i < Ti; ++i)
      if (i % P == pp && i % Q == q) return true;
    return false;
  };
  auto rank_of = [&](int p, int q) { return p * Q + q; };
  // destinations (rank, buffer, offset) of tile i of panel g in set `set`
  auto dests = [&](int set, int g, int i) {
    std::vector<std::pair<int, Ref>> d;
    const int pp = i % P;
    if (Q > 1)  // the producer's process row (same row-panel layout on every member)
      for (int q = 0; q < Q; ++q)
        if (q != L.my_q) d.push_back({rank_of(pp, q), rowt(set, g, i)});
    if (P > 1) {  // process column i mod Q, in its column-panel layout
      const int q = i % Q;
      const int64_t off = (((int64_t(set) * P + pp) * G + g) * col_cnt_max(L, q) + col_pos(L, i)) * bi2;
      for (int p = 0; p < P; ++p) d.push_back({rank_of(p, q), Ref{GPB_BUF_COL, off}});
    }
    return d;
  };
  auto sources = [&](int k) {  // ranks whose stores this rank waits for at panel k
    std::vector<int> src;
    const int kq = k % Q;
    if (Q > 1 && L.my_q != kq && has_rows(L.my_p, k)) src.push_back(rank_of(L.my_p, kq));
    if (P > 1)
      for (int pp = 0; pp < P; ++pp)
        if (has_tiles(pp, L.my_q, k) && rank_of(pp, kq) != L.rank) src.push_back(rank_of(pp, kq));
    std::sort(src.begin(), src.end());
    src.erase(std::unique(src.begin(), src.end()), src.end());
    return src;
  };
  auto flag_op = [&](int kind, int stream, int peer, int which, int64_t value) {
    gpb_op o = b.base(kind, stream);
    o.i = peer;
    o.j = which;
    o.count = value;
    b.push(o);
  };

  b.zero(MAIN, {GPB_BUF_VEC, L.vec[V_LOGDIAG]}, Ti);
  b.begin();
  for (int s = 0; s < L.nown(); ++s)
    b.job(kNone, kNone, kNone, {GPB_BUF_L, s * bi2}, 0, 0, L.own_i[s], L.own_j[s]);
  {
    gpb_op o = b.base(GPB_OP_ASSEMBLE, MAIN);
    o.flag = 1;  // noise on the global diagonal
    b.close(o);
  }
  b.record(MAIN, ev_start);
  b.wait(CRIT, ev_start);


  for (int s = 0, k0 = 0; s < ng; k0 += sizes[s], ++s) {
    const int gs = sizes[s], k1 = k0 + gs - 1, set = s % 2;
    if (s >= 2) b.wait(CRIT, ev_upd(s - 2));
    // Digit planes (L.planes > 0): every rank slices the row and column panel tiles it
    // received right after panel g's exchange; NEXT / UPD run from the planes (flag 1), and
    // the in-group updates become left-looking: before POTRF(k0 + g) one product with
    // K = g bi brings column k0 + g up to date from panels 0 .. g - 1 (LL), instead of g
    // right-looking DMMA updates with K = bi (the single-GPU schedule, gpb_api.cu).
    const bool oz_grp = L.planes > 0 && int64_t(gs) * bi >= 512 && k1 + 1 < Ti;
    auto slice_panel = [&](int g) {
      const int k = k0 + g;
      auto slice = [&](Ref first, int64_t cnt) {
        gpb_op o = b.base(GPB_OP_SLICE, CRIT);
        o.buf[0] = first.buf;
        o.off[0] = first.off;
        o.count = cnt;
        b.push(o);
      };
      int first = k + 1;
      while (first < Ti && first % P != L.my_p) ++first;
      if (first < Ti) slice(rowt(set, g, first), (Ti - 1 - first) / P + 1);
      if (P > 1)
        for (int pp = 0; pp < P; ++pp) {
          int j0 = -1, cnt = 0;
          for (int j = k + 1; j < Ti; ++j)
            if (j % P == pp && j % Q == L.my_q) {
              if (j0 < 0) j0 = j;
              ++cnt;
            }
          if (cnt > 0) slice(colt(set, g, j0), cnt);
        }
    };
    if (L.p2p && s >= 2) {
      // this rank's stores of group s land in panel set s mod 2 of its peers:
      // wait until each has finished group s - 2 (its "free" flag)
      std::vector<int> tg;
      for (int k = k0; k <= k1 && k + 1 < Ti; ++k)
        if (L.my_q == k % Q)
          for (int i = k + 1; i < Ti; ++i)
            if (slot(i, k) >= 0)
              for (auto& d : dests(set, k - k0, i))
                if (d.first != L.rank) tg.push_back(d.first);
      std::sort(tg.begin(), tg.end());
      tg.erase(std::unique(tg.begin(), tg.end()), tg.end());
      for (int r : tg) flag_op(GPB_OP_WAITFLAG, CRIT, r, 1, s - 1);
    }
    for (int g = 0; g < gs; ++g) {
      const int k = k0 + g;
      if (oz_grp && g > 0) {  // LL(g): owned tiles of column k from the group's earlier panels
        b.begin();
        for (int s2 = 0; s2 < L.nown(); ++s2) {
          const int i = L.own_i[s2], j = L.own_j[s2];
          if (j != k) continue;
          b.job(rowt(set, 0, i), colt(set, 0, j), lt(i, j), lt(i, j), g * bi, i == j, i, j);
        }
        gpb_op o = b.gemm(CRIT, nb, nb, bi, true, true, -1.0, 1.0);
        o.a_ktile = o.b_ktile = bi;
        o.a_kstride = a_walk;
        o.b_kstride = b_walk;
        o.flag = 1;
        b.close(o);
      }
      if (L.my_q == k % Q) {
        if (L.rank == L.owner(k, k)) {
          gpb_op o = b.base(GPB_OP_POTRF, CRIT);
          o.buf[0] = GPB_BUF_L;
          o.off[0] = lt(k, k).off;
          o.buf[1] = GPB_BUF_DINV;
          o.off[1] = int64_t(k) * bi2;
          o.i = k;
          b.push(o);
        }
        if (P > 1) b.coll(GPB_OP_BCAST, CRIT, COLG, k % P, {GPB_BUF_DINV, int64_t(k) * bi2}, bi2);
        // TRSM X_i = L(i, k) L_kk^-T: Dinv_k is lower triangular, so output
        // column block c needs k < (c + 1) 128 (one job per column block)
        b.begin();
        for (int i = k + 1; i < Ti; ++i) {
          if (slot(i, k) < 0) continue;
          for (int c = 0; c < nb; ++c)
            b.job(lt(i, k), {GPB_BUF_DINV, int64_t(k) * bi2 + int64_t(c) * kBlk * bi}, kNone,
                  {GPB_BUF_ROW, rowt(set, g, i).off + c * kBlk}, (c + 1) * kBlk, 0, i, k);
        }
        const int64_t trsm0 = static_cast<int64_t>(b.jobs->size()) - b.pending();
        const int64_t ntrsm = b.pending();
        b.close(b.gemm(CRIT, nb, 1, bi, true, true, 1.0, 0.0));
        if (L.p2p && ntrsm > 0) {
          // the TRSM's epilogue also stores every tile where its readers keep it
          std::vector<int> tg;
          b.begin();
          for (int64_t t = 0; t < ntrsm; ++t) {
            const gpb_op_job jb = (*b.jobs)[trsm0 + t];
            const int c = static_cast<int>((jb.off[3] - rowt(set, g, jb.i).off) / kBlk);
            for (auto& d : dests(set, g, jb.i)) {
              b.job(kNone, kNone, kNone, {d.second.buf, d.second.off + c * kBlk}, static_cast<int>(t), 0,
                    d.first, 0);
              if (d.first != L.rank) tg.push_back(d.first);
            }
          }
          b.close(b.base(GPB_OP_MIRROR, CRIT));
          std::sort(tg.begin(), tg.end());
          tg.erase(std::unique(tg.begin(), tg.end()), tg.end());
          for (int r : tg) flag_op(GPB_OP_SIGNAL, CRIT, r, 0, k + 1);  // panel k ready
        }
      }
      if (k + 1 == Ti) break;
      if (L.p2p) {  // wait for the stores of every rank that solved tiles this rank reads
        for (int r : sources(k)) flag_op(GPB_OP_WAITFLAG, CRIT, r, 0, k + 1);
      } else if (Q > 1) {  // row stage: this process row's panel tiles from rank (my_p, k mod Q)
        int first = k + 1;
        while (first < Ti && first % P != L.my_p) ++first;
        const int64_t cnt = first < Ti ? (Ti - 1 - first) / P + 1 : 0;
        if (cnt > 0) b.coll(GPB_OP_BCAST, CRIT, ROWG, k % Q, rowt(set, g, first), cnt * bi2);
      }
      // column stage: panel tiles j = p' (mod P), j = my_q (mod Q) from rank (p', my_q)
      if (P > 1 && !L.p2p) {
        for (int pp = 0; pp < P; ++pp) {
          std::vector<int> js;
          for (int j = k + 1; j < Ti; ++j)
            if (j % P == pp && j % Q == L.my_q) js.push_back(j);
          if (js.empty()) continue;
          if (L.my_p == pp) {
            b.begin();
            for (int j : js) b.job(rowt(set, g, j), kNone, kNone, colt(set, g, j));
            gpb_op o = b.base(GPB_OP_COPY, CRIT);
            o.count = bi2;
            b.close(o);
          }
          b.coll(GPB_OP_BCAST, CRIT, COLG, pp, colt(set, g, js.front()), int64_t(js.size()) * bi2);
        }
      }
      if (oz_grp) {
        slice_panel(g);
        continue;
      }
      // in-group update: the group's later columns get panel k (K = b)
      b.begin();
      for (int s2 = 0; s2 < L.nown(); ++s2) {
        const int i = L.own_i[s2], j = L.own_j[s2];
        if (j <= k || j > k1) continue;
        b.job(rowt(set, g, i), colt(set, g, j), lt(i, j), lt(i, j), bi, i == j, i, j);
      }
      b.close(b.gemm(CRIT, nb, nb, bi, true, true, -1.0, 1.0));
    }
    b.record(CRIT, ev_panel(s));
    const int c_next = k0 + gs;
    const int c_upd = std::min(Ti, c_next + (s + 1 < ng ? sizes[s + 1] : 0));
    auto update = [&](int stream, int jlo, int jhi) {
      b.begin();
      for (int s2 = 0; s2 < L.nown(); ++s2) {
        const int i = L.own_i[s2], j = L.own_j[s2];
        if (j < jlo || j >= jhi) continue;
        b.job(rowt(set, 0, i), colt(set, 0, j), lt(i, j), lt(i, j), gs * bi, i == j, i, j);
      }
      gpb_op o = b.gemm(stream, nb, nb, bi, true, true, -1.0, 1.0);
      // tiled-k walk: k tile g of row i is panel g's tile i, which keeps its
      // slot in every panel (rowt(set, g, i) = rowt(set, 0, i) + g rows_per b^2)
      o.a_ktile = o.b_ktile = bi;
      o.a_kstride = a_walk;
      o.b_kstride = b_walk;
      o.flag = oz_grp ? 1 : 0;
      b.close(o);
    };
    if (c_next < Ti) {
      // lookahead: the next group's columns need UPD(s - 1), which covered them
      if (s >= 1) b.wait(CRIT, ev_upd(s - 1));
      update(CRIT, c_next, c_upd);
    }
    b.record(CRIT, ev_next(s));
    // main stream: copy the solved panel tiles back into L, then the rest of the update
    b.wait(MAIN, ev_panel(s));
    b.begin();
    for (int g = 0; g < gs; ++g) {
      const int k = k0 + g;
      if (L.my_q != k % Q) continue;
      for (int i = k + 1; i < Ti; ++i)
        if (slot(i, k) >= 0) b.job(rowt(set, g, i), kNone, kNone, lt(i, k));
    }
    {
      gpb_op o = b.base(GPB_OP_COPY, MAIN);
      o.count = bi2;
      b.close(o);
    }
    update(MAIN, c_upd, Ti);
    b.record(MAIN, ev_upd(s));
    if (L.p2p && s + 2 < ng) {
      // panel set s mod 2 is no longer read here (UPD(s) and NEXT(s) done): tell the peers
      b.wait(MAIN, ev_next(s));
      for (int r = 0; r < L.world; ++r)
        if (r != L.rank) flag_op(GPB_OP_SIGNAL, MAIN, r, 1, s + 1);
    }
  }
  b.record(CRIT, ev_end);
  b.wait(MAIN, ev_end);
  // every rank gets every L_kk^-1 (solves on the diagonal owners, gradient rows)
  if (L.world > 1)
    for (int k = 0; k < Ti; ++k)
      b.coll(GPB_OP_BCAST, MAIN, WORLD, L.owner(k, k), {GPB_BUF_DINV, int64_t(k) * bi2}, bi2);
}

// ---- phase 1: beta = L^-1 y, alpha = L^-T beta (tiled.py:215-260) ----------
void plan_solve(const DistLayout& L, Builder& b) {
  const int Ti = L.Ti, bi = L.bi, P = L.P, Q = L.Q;
  const int64_t bi2 = L.bi2;
  if (L.world == 1) {  // one rank holds the packed factor: the one-launch dataflow solve
    b.push(b.base(GPB_OP_SOLVE_FLOW, MAIN));
    return;
  }
  auto slot = [&](int i, int j) { return L.slot[size_t(i) * Ti + j]; };
  auto v = [&](int which, int64_t at = 0) { return Ref{GPB_BUF_VEC, L.vec[which] + at}; };
  const Ref tmp = v(V_TMP), recv = v(V_RECV);
  auto combine = [&](Ref base, Ref part) {  // TMP = base - part
    gpb_op o = b.base(GPB_OP_COMBINE, MAIN);
    o.buf[0] = base.buf;
    o.off[0] = base.off;
    o.buf[1] = part.buf;
    o.off[1] = part.off;
    o.buf[2] = tmp.buf;
    o.off[2] = tmp.off;
    o.count = bi;
    b.push(o);
  };
  auto gemv = [&](bool trans, bool acc) {
    gpb_op o = b.base(GPB_OP_GEMV, MAIN);
    o.flag = trans;
    o.alpha = 1.0;
    o.beta = acc ? 1.0 : 0.0;
    return o;
  };
  auto copy_vec = [&](Ref src, Ref dst) {
    b.begin();
    b.job(src, kNone, kNone, dst);
    gpb_op o = b.base(GPB_OP_COPY, MAIN);
    o.count = bi;
    b.close(o);
  };
  b.zero(MAIN, v(V_BETA), 2 * L.np_);
  b.zero(MAIN, v(V_ACC), L.np_);
  // forward, right-looking: partial sums of row i reduced onto the diagonal
  // owner along process row i mod P; beta_i down process column i mod Q
  for (int i = 0; i < Ti; ++i) {
    const int64_t seg = int64_t(i) * bi;
    if (Q > 1 && L.my_p == i % P) b.coll(GPB_OP_REDUCE, MAIN, ROWG, i % Q, v(V_ACC, seg), bi);
    if (L.rank == L.owner(i, i)) {
      combine(v(V_Y, seg), v(V_ACC, seg));
      b.begin();
      b.job({GPB_BUF_DINV, int64_t(i) * bi2}, tmp, kNone, v(V_BETA, seg));
      b.close(gemv(false, false));
      copy_vec(v(V_BETA, seg), recv);
    }
    if (L.my_q == i % Q) {
      if (P > 1) b.coll(GPB_OP_BCAST, MAIN, COLG, i % P, recv, bi);
      b.begin();
      for (int r = i + 1; r < Ti; ++r)
        if (slot(r, i) >= 0) b.job({GPB_BUF_L, int64_t(slot(r, i)) * bi2}, recv, kNone, v(V_ACC, int64_t(r) * bi));
      b.close(gemv(false, true));
    }
  }
  b.zero(MAIN, v(V_ACC), L.np_);
  // backward: partial sums of column i reduced along process column i mod Q;
  // alpha_i along process row i mod P
  for (int i = Ti - 1; i >= 0; --i) {
    const int64_t seg = int64_t(i) * bi;
    if (P > 1 && L.my_q == i % Q) b.coll(GPB_OP_REDUCE, MAIN, COLG, i % P, v(V_ACC, seg), bi);
    if (L.rank == L.owner(i, i)) {
      combine(v(V_BETA, seg), v(V_ACC, seg));
      b.begin();
      b.job({GPB_BUF_DINV, int64_t(i) * bi2}, tmp, kNone, v(V_ALPHA, seg));
      b.close(gemv(true, false));
      copy_vec(v(V_ALPHA, seg), recv);
    }
    if (L.my_p == i % P) {
      if (Q > 1) b.coll(GPB_OP_BCAST, MAIN, ROWG, i % Q, recv, bi);
      b.begin();
      for (int j = 0; j < i; ++j)
        if (slot(i, j) >= 0) b.job({GPB_BUF_L, int64_t(slot(i, j)) * bi2}, recv, kNone, v(V_ACC, int64_t(j) * bi));
      b.close(gemv(true, true));
    }
  }
  // beta, alpha and the per-tile log-diagonal sums live on the diagonal
  // owners (zero elsewhere): one all-reduce replicates them exactly
  b.coll(GPB_OP_ALLREDUCE, MAIN, WORLD, 0, v(V_BETA), 2 * L.np_ + Ti);  // contiguous slots
}

// ---- phase 2: gradient terms (model.py:341-435) ----------------------------
// X = L^-1 right-looking with the K^-1 buffer as the accumulator
// A(i, j) = -sum_{m=j}^{i-1} L(i, m) X(m, j), and K^-1 = X^T X in outer-product
// form, both on the block-cyclic tiles.  Row k of X is "published" by:
//   F_k (process row k mod P): X(k, j) = Dinv_k A(k, j), j < k; X(k, k) = Dinv_k;
//   row k of X down the process columns (root k mod P), L(:, k) along the
//   process rows (root k mod Q), row k of X along the process rows (roots:
//   rank (p, r mod Q) for tile r)  -- into exchange set k mod 2.
// Step k then applies, on the main stream,
//   U_k: A(i, j) -= L(i, k) X(k, j) for the rank's tiles i > k + 1, j <= k;
//   LAUUM_k: K^-1(r, c) += X(k, r)^T X(k, c), c <= r <= k (written, not
//     accumulated, at r == k: that slot's A(k, c) was consumed by F_k),
// while the critical stream runs U_k on row k + 1 and publishes row k + 1
// (one-row lookahead, as in the single-GPU gradient).  Then the fused trace
// pass over each rank's K^-1 tiles and an all-reduce of the three partial
// sums.  No rank ever holds more than its own tiles plus two tile rows /
// columns of X and L.
void plan_gradient(const DistLayout& L, Builder& b) {
  const int Ti = L.Ti, bi = L.bi, nb = bi / kBlk, P = L.P, Q = L.Q;
  const int64_t bi2 = L.bi2;
  auto slot = [&](int i, int j) { return L.slot[size_t(i) * Ti + j]; };
  auto xt = [&](int i, int j) { return Ref{GPB_BUF_X, int64_t(slot(i, j)) * bi2}; };
  auto kt = [&](int i, int j) { return Ref{GPB_BUF_KINV, int64_t(slot(i, j)) * bi2}; };
  auto add = [](Ref r, int64_t o) { return Ref{r.buf, r.off + o}; };
  const int64_t xcol_set = L.bufsz[GPB_BUF_XCOL] / 2, xrow_set = L.bufsz[GPB_BUF_XROW] / 2,
                lcol_set = L.bufsz[GPB_BUF_LCOL] / 2;
  // X(k, j) as the B operand on this rank (j mod Q == my_q, j <= k)
  auto xk = [&](int k, int j) {
    return P == 1 ? xt(k, j) : Ref{GPB_BUF_XCOL, (k % 2) * xcol_set + int64_t(j / Q) * bi2};
  };
  // X(k, r) as the A operand (r mod P == my_p, r <= k)
  auto xr = [&](int k, int r) {
    return Q == 1 ? xk(k, r)
                  : Ref{GPB_BUF_XROW, (k % 2) * xrow_set + (int64_t(r % Q) * L.cntx + L.rpos[r]) * bi2};
  };
  // L(i, k) as the A operand (i mod P == my_p, i > k)
  auto lc = [&](int k, int i) {
    return Q == 1 ? Ref{GPB_BUF_L, int64_t(slot(i, k)) * bi2}
                  : Ref{GPB_BUF_LCOL, (k % 2) * lcol_set + int64_t(i / P) * bi2};
  };
  const int ev_zero = 0;
  auto ev_x = [&](int k) { return 1 + k; };       // row k of X published (critical stream)
  auto ev_u = [&](int k) { return 1 + Ti + k; };  // step k applied to rows > k + 1 (main stream)
  auto copy_op = [&](int stream) {
    gpb_op o = b.base(GPB_OP_COPY, stream);
    o.count = bi2;
    b.close(o);
  };
  // U_k on the rank's tiles of rows [ilo, ihi): A(i, j) -= L(i, k) X(k, j), j <= k
  auto update = [&](int stream, int k, int ilo, int ihi) {
    b.begin();
    for (int s = 0; s < L.nown(); ++s) {
      const int i = L.own_i[s], j = L.own_j[s];
      if (i >= ilo && i < ihi && j < k) b.job(lc(k, i), xk(k, j), kt(i, j), kt(i, j), bi, 0, i, j);
    }
    b.close(b.gemm(stream, nb, nb, bi, true, false, -1.0, 1.0));
    // j = k: X(k, k) = Dinv_k is lower triangular, so output column block cb
    // needs only k >= cb 128 (one job per column block, K = b - cb 128)
    b.begin();
    for (int i = std::max(ilo, k + 1); i < ihi; ++i) {
      if (slot(i, k) < 0) continue;
      for (int cb = 0; cb < nb; ++cb) {
        const int64_t o = int64_t(cb) * kBlk;
        b.job(add(lc(k, i), o), add(xk(k, k), o * bi + o), add(kt(i, k), o), add(kt(i, k), o),
              bi - static_cast<int>(o), 0, i, k);
      }
    }
    b.close(b.gemm(stream, nb, 1, bi, true, false, -1.0, 1.0));
  };
  // finalise row k of X on its process row and publish it with L(:, k) (exchange set k mod 2)
  auto publish = [&](int k) {
    if (L.my_p == k % P) {
      // F_k: Dinv_k is lower triangular, so output row block r needs k < (r + 1) 128
      b.begin();
      for (int j = 0; j < k; ++j) {
        if (slot(k, j) < 0) continue;
        for (int r = 0; r < nb; ++r)
          b.job({GPB_BUF_DINV, int64_t(k) * bi2 + int64_t(r) * kBlk * bi}, kt(k, j), kNone,
                add(xt(k, j), int64_t(r) * kBlk * bi), (r + 1) * kBlk, 0, k, j);
      }
      b.close(b.gemm(CRIT, 1, nb, bi, true, false, 1.0, 0.0));
      if (L.rank == L.owner(k, k)) {
        b.begin();
        b.job({GPB_BUF_DINV, int64_t(k) * bi2}, kNone, kNone, xt(k, k));
        copy_op(CRIT);
      }
    }
    if (P > 1) {  // row k of X down process column my_q (root: process row k mod P)
      int cnt = 0;
      b.begin();
      for (int j = L.my_q; j <= k; j += Q) {
        ++cnt;
        if (L.my_p == k % P) b.job(xt(k, j), kNone, kNone, xk(k, j));
      }
      copy_op(CRIT);
      b.coll(GPB_OP_BCAST, CRIT, COLG, k % P, xk(k, L.my_q), int64_t(cnt) * bi2);
    }
    if (Q > 1 && k + 1 < Ti) {  // L(:, k) along process row my_p (root: column k mod Q)
      int first = k + 1;
      while (first < Ti && first % P != L.my_p) ++first;
      const int64_t cnt = first < Ti ? (Ti - 1 - first) / P + 1 : 0;
      if (cnt > 0) {
        b.begin();
        if (L.my_q == k % Q)
          for (int i = first; i < Ti; i += P) b.job({GPB_BUF_L, int64_t(slot(i, k)) * bi2}, kNone, kNone, lc(k, i));
        copy_op(CRIT);
        b.coll(GPB_OP_BCAST, CRIT, ROWG, k % Q, lc(k, first), cnt * bi2);
      }
    }
    if (Q > 1) {  // row k of X along process row my_p: tiles r = q' (mod Q) from rank (my_p, q')
      for (int qq = 0; qq < Q; ++qq) {
        int cnt = 0, first = -1;
        b.begin();
        for (int r = 0; r <= k; ++r) {
          if (r % P != L.my_p || r % Q != qq) continue;
          if (first < 0) first = r;
          ++cnt;
          if (L.my_q == qq) b.job(xk(k, r), kNone, kNone, xr(k, r));
        }
        if (cnt == 0) continue;
        copy_op(CRIT);
        b.coll(GPB_OP_BCAST, CRIT, ROWG, qq, xr(k, first), int64_t(cnt) * bi2);
      }
    }
    b.record(CRIT, ev_x(k));
  };

  b.zero(MAIN, {GPB_BUF_KINV, 0}, int64_t(L.nown()) * bi2);
  b.record(MAIN, ev_zero);
  b.wait(CRIT, ev_zero);
  publish(0);
  for (int k = 0; k < Ti; ++k) {
    // main: the bulk of step k once row k of X is published
    b.wait(MAIN, ev_x(k));
    update(MAIN, k, k + 2, Ti);
    // LAUUM_k: K^-1(r, c) (+)= X(k, r)^T X(k, c), both operands M/N-major
    for (int fresh = 1; fresh >= 0; --fresh) {
      b.begin();
      for (int s = 0; s < L.nown(); ++s) {
        const int r = L.own_i[s], c = L.own_j[s];
        if (r > k || (r == k) != (fresh == 1)) continue;
        b.job(xr(k, r), xk(k, c), fresh ? kNone : kt(r, c), kt(r, c), bi, r == c, r, c);
      }
      b.close(b.gemm(MAIN, nb, nb, bi, false, false, 1.0, fresh ? 0.0 : 1.0));
    }
    b.record(MAIN, ev_u(k));
    if (k + 1 < Ti) {
      // critical: row k + 1 has U_0 .. U_{k-1} from the main stream (and the main
      // stream is done with exchange set (k + 1) mod 2); apply U_k to it, publish it
      if (k >= 1) b.wait(CRIT, ev_u(k - 1));
      update(CRIT, k, k + 1, k + 2);
      publish(k + 1);
    }
  }
  b.begin();
  for (int s = 0; s < L.nown(); ++s)
    b.job({GPB_BUF_KINV, int64_t(s) * bi2}, kNone, kNone, kNone, 0, 0, L.own_i[s], L.own_j[s]);
  {
    gpb_op o = b.base(GPB_OP_TRACE, MAIN);
    o.buf[2] = GPB_BUF_VEC;
    o.off[2] = L.vec[V_RED];
    b.close(o);
  }
  if (L.world > 1) b.coll(GPB_OP_ALLREDUCE, MAIN, WORLD, 0, {GPB_BUF_VEC, L.vec[V_RED]}, 3);
}

}  // namespace

void dist_plan(const DistLayout& L, int phase, std::vector<gpb_op>* ops, std::vector<gpb_op_job>* jobs) {
  Builder b;
  b.ops = ops;
  b.jobs = jobs;
  if (phase == 0) plan_factor(L, b);
  if (phase == 1) plan_solve(L, b);
  if (phase == 2) plan_gradient(L, b);
}

}  // namespace gpb

extern "C" int gpb_plugin_fail(int code, const char* msg);

extern "C" int gpb_dist_plan(int rank, int world, int P, int Q, int64_t n, int64_t tiles_per_dim, int phase,
                             int exchange, gpb_op* ops, int64_t* nops, gpb_op_job* jobs, int64_t* njobs,
                             int64_t bufsz[GPB_NBUF], int64_t meta[16]) {
  if (phase < 0 || phase > 2) return gpb_plugin_fail(GPB_INVALID_CONFIG, "phase must be 0, 1 or 2");
  gpb::DistLayout L;
  std::string err;
  if (int s = gpb::dist_layout(rank, world, P, Q, n, tiles_per_dim, &L, &err, exchange))
    return gpb_plugin_fail(s, err.c_str());
  std::vector<gpb_op> o;
  std::vector<gpb_op_job> j;
  gpb::dist_plan(L, phase, &o, &j);
  if (ops) {
    if (!nops || !njobs || *nops < static_cast<int64_t>(o.size()) || *njobs < static_cast<int64_t>(j.size()))
      return gpb_plugin_fail(GPB_INVALID_CONFIG, "operation buffers too small");
    std::copy(o.begin(), o.end(), ops);
    std::copy(j.begin(), j.end(), jobs);
  }
  if (nops) *nops = static_cast<int64_t>(o.size());
  if (njobs) *njobs = static_cast<int64_t>(j.size());
  if (bufsz)
    for (int t = 0; t < GPB_NBUF; ++t) bufsz[t] = L.bufsz[t];
  if (meta) {
    const int64_t m[16] = {L.bi, L.Ti, L.np_, L.P, L.Q, L.G, L.nown(), L.nevents,
                           L.vec[gpb::V_Y], L.vec[gpb::V_BETA], L.vec[gpb::V_ALPHA], L.vec[gpb::V_LOGDIAG],
                           L.vec[gpb::V_ACC], L.vec[gpb::V_TMP], L.vec[gpb::V_RECV], L.vec[gpb::V_RED]};
    std::copy(m, m + 16, meta);
  }
  return GPB_OK;
}
