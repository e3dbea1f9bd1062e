// Batched sweeps (new entry points; the reference's loop is
// tools/sched_main.cpp:452-502). Host work here is once-per-graph analysis
// (cached on the graph): decide whether the closed form of SURVEY Appendix A.2
// applies and find the chain classes; per oracle the classes are weighted
// into the tables the device kernel folds over (O(n)). Otherwise every seed
// runs through the exact device event simulator.
#include "sweep.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <array>
#include <map>
#include <memory>
#include <set>
#include <thread>

#include "../device/csk.h"
#include "rng_host.hpp"

namespace tictac {

namespace {

// Chain-class tables of one worker (graph or cluster worker partition).
struct ChainTables {
  int32_t R = 0, nc = 0;
  std::vector<int64_t> d;      // per recv column
  std::vector<int32_t> first;  // per recv column
  std::vector<int64_t> pwsuf;  // nc + 1
  int64_t send_total = 0;
  // general DAGs (not nested): weights of the join classes (program order),
  // of the classes whose set is one recv (per recv column), of the classes
  // with no recv ancestor
  std::vector<int64_t> wj, wr;
  int64_t w0 = 0;
  int32_t nch = 1;
  std::vector<int32_t> ch;          // per recv column: channel
  std::vector<int64_t> send_by_ch;  // per channel: send time
};

// Straight-line program for general worker DAGs (sweep.cu dag_sweep_kernel):
// per join class (recv-ancestor set with >= 2 recvs), in increasing set
// size, its latest recv position = max over generators, each a recv column
// (value index c < R: that recv's position) or an earlier join held in a
// live slot (value index R + slot). Records of three generators and one
// output (value index; -1 = discard), a join with more generators chained
// through temporary slots. Records come in groups of four that never read a
// slot written inside the same group (the kernel loads a group's generators
// before storing its outputs); groups are padded with no-op records.
// Duration-independent: per oracle, record r weighs rec_join[r]'s class
// (-1: no weight).
constexpr int32_t kDagAcc = -2;  // generator: the previous record's result (register)
constexpr int32_t kDagPad = -3;  // padding record (no effect)
struct DagProgram {
  int32_t J = 0, L = 0;  // join classes, live slots
  std::vector<std::array<int32_t, 4>> recs;
  std::vector<int32_t> rec_join;    // join index per record, -1 for temporaries and padding
  std::vector<int32_t> join_class;  // class id of every join, program order
  std::vector<int32_t> single;      // per class: recv column when its set is {recv}, else -1
  std::vector<int32_t> empty;       // classes with no recv ancestor
};

// Duration-independent part of the closed form for one worker (graph or
// cluster worker partition): preconditions of A.2, nested recv-ancestor
// classes, first class of every recv column, the send ops. Computed once per
// graph (Graph::memo); durations only weight it (chain_tables).
struct ChainShape {
  bool ok = false;
  std::string why;
  int32_t R = 0, nc = 0;
  std::vector<int32_t> first;     // per recv column: first class containing it
  std::vector<int32_t> class_of;  // per op: class of a non-transfer op, else -1
  std::vector<int32_t> sends;     // send ops (cluster workers)
  bool nested = true;             // chain classes (fold kernel), else `dag`
  DagProgram dag;
  // channels of the worker (resource order; several when the cluster has
  // several parameter servers): channel of every recv column / send op
  int32_t nch = 1;
  std::vector<int32_t> recv_ch, send_ch;
};
constexpr int32_t kMaxChannels = 4;

// Compiles the join program from the classes' recv-ancestor bitsets (rep[j]
// = a member op, sets ordered by size). Generators of class j: the classes
// of the predecessors of one member that has no predecessor in j (its set
// is their union), minus generators whose set is contained in another's.
bool dag_program(const Graph& g, const std::vector<uint64_t>& bits, int32_t W, const std::vector<int32_t>& col,
                 const std::vector<int32_t>& rep, const std::vector<int32_t>& class_of, DagProgram& out,
                 std::string& why) {
  const int32_t nc = static_cast<int32_t>(rep.size());
  const int32_t R = static_cast<int32_t>(g.recv_ops().size());
  auto set_of = [&](int32_t j) { return &bits[static_cast<size_t>(rep[j]) * W]; };
  std::vector<int32_t> pop(nc, 0);
  for (int32_t j = 0; j < nc; ++j)
    for (int32_t q = 0; q < W; ++q) pop[j] += __builtin_popcountll(set_of(j)[q]);
  auto subset = [&](int32_t a, int32_t b) {  // set(a) within set(b)
    const uint64_t *x = set_of(a), *y = set_of(b);
    for (int32_t q = 0; q < W; ++q)
      if (x[q] & ~y[q]) return false;
    return true;
  };
  auto has = [&](int32_t j, int32_t c) { return (set_of(j)[c >> 6] >> (c & 63)) & 1; };
  // generators per class: g >= 0 class, g < 0 recv column -(g+1)
  std::vector<std::vector<int32_t>> gens(nc);
  std::vector<char> done(nc, 0);
  out.single.assign(nc, -1);
  out.empty.clear();
  for (int32_t v = 0; v < g.n(); ++v) {
    const int32_t j = class_of[v];
    if (j < 0) continue;
    std::vector<int32_t> gl;
    bool own = false;
    for (int32_t e = g.pred_off()[v]; e < g.pred_off()[v + 1]; ++e) {
      const int32_t p = g.pred_idx()[e];
      if (col[p] >= 0) {
        gl.push_back(-(col[p] + 1));
      } else if (class_of[p] >= 0) {
        own |= class_of[p] == j;
        gl.push_back(class_of[p]);
      } else {
        return why = "compute op depends on a non-recv transfer", false;
      }
    }
    if (own) continue;  // not a first member of its class
    std::sort(gl.begin(), gl.end());
    gl.erase(std::unique(gl.begin(), gl.end()), gl.end());
    std::vector<int32_t> red;
    for (int32_t x : gl) {
      bool drop = false;
      for (int32_t y : gl) {
        if (y < 0 || y == x) continue;
        if (x < 0 ? has(y, -(x + 1)) : (subset(x, y) && (pop[x] < pop[y] || x > y))) drop = true;
      }
      if (!drop) red.push_back(x);
    }
    if (!done[j] || red.size() < gens[j].size()) gens[j] = red;
    done[j] = 1;
  }
  // join classes in set-size order (classes are sorted that way already)
  std::vector<int32_t> joins, jpos(nc, -1);
  for (int32_t j = 0; j < nc; ++j) {
    if (pop[j] == 0) {
      out.empty.push_back(j);
    } else if (pop[j] == 1) {
      for (int32_t c = 0; c < R; ++c)
        if (has(j, c)) out.single[j] = c;
    } else {
      if (!done[j] || gens[j].size() < 2) return why = "internal: join class without generators", false;
      jpos[j] = static_cast<int32_t>(joins.size());
      joins.push_back(j);
    }
  }
  // 1. records over virtual values (recv column c < R; value v >= R: output
  //    v - R, joins first, then temporaries for joins of > 3 generators)
  struct VRec {
    std::array<int32_t, 3> in;
    int32_t out;   // virtual value id
    int32_t join;  // weighted join, or -1
  };
  std::vector<VRec> vr;
  const int32_t J = static_cast<int32_t>(joins.size());
  int32_t nvals = J;
  for (int32_t k = 0; k < J; ++k) {
    const int32_t j = joins[k];
    std::vector<int32_t> idx;
    for (int32_t x : gens[j]) {
      if (x < 0) {
        idx.push_back(-(x + 1));
      } else if (out.single[x] >= 0) {
        idx.push_back(out.single[x]);
      } else if (jpos[x] >= 0) {
        if (jpos[x] >= k) return why = "internal: generator used before its definition", false;
        idx.push_back(R + jpos[x]);
      }  // else an empty-set generator: position -inf, no effect on the max
    }
    std::sort(idx.begin(), idx.end());
    idx.erase(std::unique(idx.begin(), idx.end()), idx.end());
    if (idx.empty()) return why = "internal: join without recv generators", false;
    while (idx.size() > 3) {  // max of three into a temporary
      vr.push_back({{idx[0], idx[1], idx[2]}, nvals, -1});
      idx.erase(idx.begin(), idx.begin() + 3);
      idx.push_back(R + nvals++);
    }
    while (idx.size() < 3) idx.push_back(idx.back());
    vr.push_back({{idx[0], idx[1], idx[2]}, k, k});
  }
  // 2. list schedule into groups of four: a record's first generator may be
  //    the previous record's result, forwarded in a register (ACC); every
  //    other value it reads must come from an earlier group. Longest
  //    remaining dependency chain first; a chain continues through ACC.
  const int32_t N = static_cast<int32_t>(vr.size());
  std::vector<int32_t> producer(nvals, -1);
  for (int32_t r = 0; r < N; ++r) producer[vr[r].out] = r;
  std::vector<std::vector<int32_t>> users(N);
  for (int32_t r = 0; r < N; ++r)
    for (int32_t x : std::set<int32_t>(vr[r].in.begin(), vr[r].in.end()))
      if (x >= R) users[producer[x - R]].push_back(r);
  std::vector<int32_t> height(N, 1);
  for (int32_t r = N - 1; r >= 0; --r)
    for (int32_t u : users[r]) height[r] = std::max(height[r], height[u] + 1);
  std::vector<int32_t> group_of(N, -1), order;
  std::vector<char> acc(N, 0);
  int32_t placed = 0, gq = 0;
  while (placed < N) {
    int32_t prev = -1;  // record at the previous position of this group
    for (int32_t i = 0; i < 4; ++i) {
      int32_t best = -1;
      bool best_acc = false;
      for (int32_t r = 0; r < N; ++r) {
        if (group_of[r] >= 0) continue;
        bool ok = true, via_acc = false;
        for (int32_t x : vr[r].in) {
          if (x < R) continue;
          const int32_t pr = producer[x - R];
          if (group_of[pr] >= 0 && group_of[pr] < gq) continue;
          if (pr == prev && prev >= 0) {
            via_acc = true;
            continue;
          }
          ok = false;
          break;
        }
        if (!ok) continue;
        if (best < 0 || height[r] > height[best] || (height[r] == height[best] && via_acc && !best_acc)) {
          best = r;
          best_acc = via_acc;
        }
      }
      if (best < 0) break;
      group_of[best] = gq;
      order.push_back(best);
      acc[best] = best_acc ? 1 : 0;
      prev = best;
      ++placed;
    }
    while (order.size() % 4) order.push_back(-1);
    ++gq;
  }
  // the forwarded generator first; its other occurrences become fillers
  for (size_t i = 1; i < order.size(); ++i) {
    const int32_t r = order[i];
    if (r < 0 || !acc[r]) continue;
    const int32_t pv = R + vr[order[i - 1]].out;
    auto& in = vr[r].in;
    for (int q = 0; q < 3; ++q)
      if (in[q] == pv) {
        std::swap(in[0], in[q]);
        break;
      }
    for (int u = 1; u < 3; ++u)
      if (in[u] == pv) in[u] = -1;
    if (in[1] < 0) std::swap(in[1], in[2]);
    if (in[1] < 0) return why = "internal: join with one generator", false;
    if (in[2] < 0) in[2] = in[1];
  }
  const int32_t ngroups = static_cast<int32_t>(order.size() / 4);
  // 3. slots by linear scan over groups: a value lives from its group to
  //    the group of its last non-forwarded reader (a group reads before it
  //    writes, so a slot freed by a group's reads can take that group's
  //    outputs)
  std::vector<int32_t> last_group(nvals, -1);
  for (int32_t r = 0; r < N; ++r)
    for (int q = acc[r] ? 1 : 0; q < 3; ++q)
      if (vr[r].in[q] >= R) last_group[vr[r].in[q] - R] = std::max(last_group[vr[r].in[q] - R], group_of[r]);
  std::vector<int32_t> slot(nvals, -1), free_slots;
  int32_t nslots = 0;
  out.recs.clear();
  out.rec_join.clear();
  for (int32_t gq = 0; gq < ngroups; ++gq) {
    std::array<std::array<int32_t, 4>, 4> recs{};
    for (int32_t i = 0; i < 4; ++i) {
      const int32_t r = order[4 * gq + i];
      if (r < 0) {
        recs[i] = {kDagPad, kDagPad, kDagPad, kDagPad};
        continue;
      }
      for (int q = 0; q < 3; ++q) {
        const int32_t x = vr[r].in[q];
        if (q == 0 && acc[r]) {
          recs[i][q] = kDagAcc;
        } else {
          recs[i][q] = x < R ? x : R + slot[x - R];
        }
      }
      recs[i][3] = -1;
    }
    for (int32_t i = 0; i < 4; ++i) {  // release values last read here
      const int32_t r = order[4 * gq + i];
      if (r < 0) continue;
      for (int q = acc[r] ? 1 : 0; q < 3; ++q) {
        const int32_t x = vr[r].in[q];
        if (x >= R && last_group[x - R] == gq && slot[x - R] >= 0) {
          free_slots.push_back(slot[x - R]);
          slot[x - R] = -1 - slot[x - R];
        }
      }
    }
    for (int32_t i = 0; i < 4; ++i) {  // outputs read later from a slot
      const int32_t r = order[4 * gq + i];
      if (r < 0 || last_group[vr[r].out] < 0) continue;
      int32_t t;
      if (free_slots.empty()) {
        t = nslots++;
      } else {
        t = free_slots.back();
        free_slots.pop_back();
      }
      slot[vr[r].out] = t;
      recs[i][3] = R + t;
    }
    for (int32_t i = 0; i < 4; ++i) {
      out.recs.push_back(recs[i]);
      const int32_t r = order[4 * gq + i];
      out.rec_join.push_back(r < 0 ? -1 : vr[r].join);
    }
    if (R + nslots >= (1 << 15)) return why = "program too large", false;
  }
  out.J = static_cast<int32_t>(joins.size());
  out.L = nslots;
  out.join_class = joins;
  return true;
}

ChainShape chain_shape(const Graph& g, bool allow_sends) {
  ChainShape cs;
  auto no = [&](const char* why) {
    cs.why = why;
    return cs;
  };
  const int32_t n = g.n();
  const auto& ops = g.ops();
  const int32_t R = static_cast<int32_t>(g.recv_ops().size());
  if (R == 0) return no("no recv ops");
  int32_t cpu = -1;
  std::vector<int32_t> chans;  // channel resources, ascending (resource order)
  for (int32_t i = 0; i < n; ++i) {
    const int32_t r = g.res_of()[i];
    if (ops[i].kind == kRecv || ops[i].kind == kSend) {
      if (ops[i].kind == kSend && !allow_sends) return no("send ops on the worker");
      if (std::find(chans.begin(), chans.end(), r) == chans.end()) chans.push_back(r);
    } else {
      if (cpu >= 0 && cpu != r) return no("more than one compute unit");
      cpu = r;
    }
    if (ops[i].kind == kRecv && g.npred(i) > 0) return no("recv with predecessors");
  }
  std::sort(chans.begin(), chans.end());
  if (static_cast<int32_t>(chans.size()) > kMaxChannels) return no("more than four channels");
  cs.nch = std::max<int32_t>(1, static_cast<int32_t>(chans.size()));
  auto chan_index = [&](int32_t op) {
    return static_cast<int32_t>(std::lower_bound(chans.begin(), chans.end(), g.res_of()[op]) - chans.begin());
  };
  for (int32_t c = 0; c < R; ++c) cs.recv_ch.push_back(chan_index(g.recv_ops()[c]));
  // recv-ancestor sets of every compute op (bitsets over recv columns)
  const int32_t W = (R + 63) / 64;
  if (static_cast<int64_t>(n) * W > (int64_t{1} << 27)) return no("graph too large for tables");
  std::vector<int32_t> col(n, -1);
  for (int32_t c = 0; c < R; ++c) col[g.recv_ops()[c]] = c;
  std::vector<int32_t> order, missing(n);
  for (int32_t i = 0; i < n; ++i)
    if ((missing[i] = g.npred(i)) == 0) order.push_back(i);
  for (size_t h = 0; h < order.size(); ++h)
    for (int32_t e = g.succ_off()[order[h]]; e < g.succ_off()[order[h] + 1]; ++e)
      if (--missing[g.succ_idx()[e]] == 0) order.push_back(g.succ_idx()[e]);
  std::vector<uint64_t> bits(static_cast<size_t>(n) * W, 0);
  for (int32_t v : order) {
    uint64_t* row = &bits[static_cast<size_t>(v) * W];
    for (int32_t e = g.pred_off()[v]; e < g.pred_off()[v + 1]; ++e) {
      const uint64_t* pr = &bits[static_cast<size_t>(g.pred_idx()[e]) * W];
      for (int32_t q = 0; q < W; ++q) row[q] |= pr[q];
    }
    if (col[v] >= 0) row[col[v] >> 6] |= 1ULL << (col[v] & 63);
  }
  // classes = distinct sets among non-transfer ops, ordered by size
  std::vector<int32_t> comp;
  for (int32_t i = 0; i < n; ++i)
    if (!transfer(ops[i].kind)) comp.push_back(i);
  std::vector<int64_t> pop(n, 0);
  for (int32_t v : comp)
    for (int32_t q = 0; q < W; ++q) pop[v] += __builtin_popcountll(bits[static_cast<size_t>(v) * W + q]);
  auto less = [&](int32_t a, int32_t b) {
    if (pop[a] != pop[b]) return pop[a] < pop[b];
    return std::lexicographical_compare(&bits[static_cast<size_t>(a) * W], &bits[static_cast<size_t>(a) * W] + W,
                                        &bits[static_cast<size_t>(b) * W], &bits[static_cast<size_t>(b) * W] + W);
  };
  std::sort(comp.begin(), comp.end(), less);
  std::vector<int32_t> rep;  // class representative
  cs.class_of.assign(n, -1);
  for (int32_t v : comp) {
    if (rep.empty() || less(rep.back(), v)) rep.push_back(v);
    cs.class_of[v] = static_cast<int32_t>(rep.size()) - 1;
  }
  const int32_t nc = static_cast<int32_t>(rep.size());
  for (int32_t j = 1; j < nc && cs.nested; ++j) {  // nested?
    const uint64_t* a = &bits[static_cast<size_t>(rep[j - 1]) * W];
    const uint64_t* b = &bits[static_cast<size_t>(rep[j]) * W];
    for (int32_t q = 0; q < W; ++q)
      if (a[q] & ~b[q]) cs.nested = false;
  }
  cs.R = R;
  cs.nc = nc;
  if (cs.nested && !std::getenv("TICTAC_SWEEP_FORCE_DAG")) {
    cs.first.assign(R, nc);
    for (int32_t j = nc - 1; j >= 0; --j)
      for (int32_t c = 0; c < R; ++c)
        if ((bits[static_cast<size_t>(rep[j]) * W + (c >> 6)] >> (c & 63)) & 1) cs.first[c] = j;
  } else {
    cs.nested = false;
    if (cs.nch > 1) return no("recv-ancestor sets are not nested and the worker has several channels");
    std::string why;
    if (!dag_program(g, bits, W, col, rep, cs.class_of, cs.dag, why)) return no(why.c_str());
  }
  // sends: must be released exactly when the last compute finishes, i.e.
  // depend on every compute op that has no compute successor.
  if (allow_sends) {
    std::set<int32_t> sinks;
    for (int32_t v : comp) {
      bool has = false;
      for (int32_t e = g.succ_off()[v]; e < g.succ_off()[v + 1]; ++e)
        has |= !transfer(ops[g.succ_idx()[e]].kind);
      if (!has) sinks.insert(v);
    }
    for (int32_t i = 0; i < n; ++i) {
      if (ops[i].kind != kSend) continue;
      std::set<int32_t> pre(g.pred_idx().begin() + g.pred_off()[i], g.pred_idx().begin() + g.pred_off()[i + 1]);
      for (int32_t p : pre)
        if (transfer(ops[p].kind)) return no("send depends on a transfer");
      if (sinks.empty() || !std::includes(pre.begin(), pre.end(), sinks.begin(), sinks.end()))
        return no("send not released by the last compute");
      cs.sends.push_back(i);
      cs.send_ch.push_back(chan_index(i));
    }
  }
  cs.ok = true;
  return cs;
}

// Send phase of clusters whose parameter-server ops take time (sweep.cu
// cluster_ps_kernel): duration-independent structure, memoised per graph.
struct PsShape {
  bool ok = false;
  std::string why;
  int32_t S = 0, Q = 0, nps = 0, nch = 1;
  std::vector<int16_t> recv_sb;                // [R] the worker's sends before recv column c (op-index order)
  std::vector<uint32_t> ch_mask;               // [nch][sw] sends on each channel
  std::vector<std::vector<int32_t>> sends;      // per worker: send ops (graph index), op-index order
  std::vector<int32_t> send_succ_off;           // [W*S + 1]
  std::vector<int16_t> send_succ;               // PS op indices
  std::vector<int32_t> ps_ops;                  // graph indices, op-index order
  std::vector<uint8_t> ps_missing;              // predecessor counts
  std::vector<int32_t> ps_succ_off;
  std::vector<int16_t> ps_succ;
  std::vector<uint32_t> core_mask;             // [nps][qw] PS ops of each core
  std::vector<int32_t> slots;                  // resource order: core k -> -1-k, channel (w, ch) -> w*nch + ch
  std::vector<int32_t> last_compute;           // per worker: graph index of its last compute op
};

PsShape ps_shape(const Graph& g, const std::vector<std::string>& workers) {
  PsShape ps;
  auto no = [&](const char* why) {
    ps.why = why;
    return ps;
  };
  const int32_t n = g.n();
  const auto& ops = g.ops();
  std::unordered_map<std::string, int32_t> widx;
  for (size_t i = 0; i < workers.size(); ++i) widx[workers[i]] = static_cast<int32_t>(i);
  std::vector<int32_t> wof(n, -1), psix(n, -1);
  std::map<std::string, int32_t> ps_res;  // PS device -> its one resource
  for (int32_t i = 0; i < n; ++i) {
    auto it = widx.find(ops[i].res.device);
    if (it != widx.end()) {
      wof[i] = it->second;
      continue;
    }
    if (transfer(ops[i].kind)) return no("transfer on a parameter-server device");
    auto pr = ps_res.emplace(ops[i].res.device, g.res_of()[i]);
    if (pr.second == false && pr.first->second != g.res_of()[i])
      return no("a parameter-server device with more than one resource");
    psix[i] = static_cast<int32_t>(ps.ps_ops.size());
    ps.ps_ops.push_back(i);  // ascending graph index = op-index order
  }
  ps.Q = static_cast<int32_t>(ps.ps_ops.size());
  ps.nps = static_cast<int32_t>(ps_res.size());
  if (ps.Q == 0) return no("no parameter-server ops");
  if (ps.Q >= (1 << 15)) return no("too many parameter-server ops");
  if (ps.nps > 16) return no("more than 16 parameter servers");
  std::vector<int32_t> core_res;  // resource of core k, cores in resource order
  for (const auto& [dev, r] : ps_res) core_res.push_back(r);
  std::sort(core_res.begin(), core_res.end());
  const int32_t qw = (ps.Q + 31) / 32;
  ps.core_mask.assign(static_cast<size_t>(ps.nps) * qw, 0);
  for (int32_t x = 0; x < ps.Q; ++x) {
    const int32_t k = static_cast<int32_t>(std::lower_bound(core_res.begin(), core_res.end(),
                                                            g.res_of()[ps.ps_ops[x]]) - core_res.begin());
    ps.core_mask[static_cast<size_t>(k) * qw + (x >> 5)] |= 1u << (x & 31);
  }
  for (int32_t x = 0; x < ps.Q; ++x) {
    const int32_t v = ps.ps_ops[x];
    int32_t np = 0;
    for (int32_t e = g.pred_off()[v]; e < g.pred_off()[v + 1]; ++e) {
      const int32_t u = g.pred_idx()[e];
      if (psix[u] < 0 && ops[u].kind != kSend) return no("parameter-server op fed by a non-send worker op");
      ++np;
    }
    if (np == 0) return no("parameter-server op without predecessors");
    if (np > 255) return no("parameter-server op with more than 255 predecessors");
    ps.ps_missing.push_back(static_cast<uint8_t>(np));
  }
  ps.ps_succ_off.push_back(0);
  for (int32_t x = 0; x < ps.Q; ++x) {
    const int32_t v = ps.ps_ops[x];
    for (int32_t e = g.succ_off()[v]; e < g.succ_off()[v + 1]; ++e) {
      const int32_t u = g.succ_idx()[e];
      if (psix[u] < 0) return no("parameter-server op feeding a worker");
      ps.ps_succ.push_back(static_cast<int16_t>(psix[u]));
    }
    ps.ps_succ_off.push_back(static_cast<int32_t>(ps.ps_succ.size()));
  }
  // per worker: channels (resource order), sends, recvs, compute total order
  const int32_t W = static_cast<int32_t>(workers.size());
  ps.sends.assign(W, {});
  std::vector<std::vector<int32_t>> recvs(W), comp(W), chans(W);
  for (int32_t i = 0; i < n; ++i) {
    const int32_t w = wof[i];
    if (w < 0) continue;
    if (ops[i].kind == kSend) ps.sends[w].push_back(i);
    else if (ops[i].kind == kRecv) recvs[w].push_back(i);
    else comp[w].push_back(i);
    if (transfer(ops[i].kind) &&
        std::find(chans[w].begin(), chans[w].end(), g.res_of()[i]) == chans[w].end())
      chans[w].push_back(g.res_of()[i]);
  }
  ps.S = static_cast<int32_t>(ps.sends[0].size());
  ps.nch = static_cast<int32_t>(chans[0].size());
  const int32_t R = static_cast<int32_t>(recvs[0].size());
  const int32_t sw = (ps.S + 31) / 32;
  for (int32_t w = 0; w < W; ++w) {
    std::sort(chans[w].begin(), chans[w].end());
    if (static_cast<int32_t>(ps.sends[w].size()) != ps.S || static_cast<int32_t>(recvs[w].size()) != R ||
        static_cast<int32_t>(chans[w].size()) != ps.nch)
      return no("workers differ in their transfers");
    if (ps.nch == 0) return no("worker without a channel");
    std::vector<int16_t> sb(R);
    for (int32_t c = 0; c < R; ++c)
      sb[c] = static_cast<int16_t>(std::lower_bound(ps.sends[w].begin(), ps.sends[w].end(), recvs[w][c]) -
                                   ps.sends[w].begin());
    std::vector<uint32_t> mask(static_cast<size_t>(ps.nch) * sw, 0);
    for (int32_t x = 0; x < ps.S; ++x) {
      const int32_t ch = static_cast<int32_t>(std::lower_bound(chans[w].begin(), chans[w].end(),
                                                               g.res_of()[ps.sends[w][x]]) - chans[w].begin());
      mask[static_cast<size_t>(ch) * sw + (x >> 5)] |= 1u << (x & 31);
    }
    if (w == 0) {
      ps.recv_sb = sb;
      ps.ch_mask = mask;
    } else if (sb != ps.recv_sb || mask != ps.ch_mask) {
      return no("workers differ in their channel op order");
    }
    // compute ops totally ordered (so the core never has two candidates):
    // the longest path over compute->compute edges covers all of them
    if (comp[w].empty()) return no("worker without compute ops");
    std::unordered_map<int32_t, int32_t> depth, miss;
    for (int32_t v : comp[w]) depth[v] = 0, miss[v] = 0;
    std::vector<int32_t> order;
    for (int32_t v : comp[w]) {
      for (int32_t e = g.pred_off()[v]; e < g.pred_off()[v + 1]; ++e)
        if (depth.count(g.pred_idx()[e])) ++miss[v];
      if (miss[v] == 0) order.push_back(v);
    }
    int32_t best = 0, last = -1;
    for (size_t h = 0; h < order.size(); ++h) {
      const int32_t v = order[h];
      depth[v] += 1;
      if (depth[v] > best) best = depth[v], last = v;
      for (int32_t e = g.succ_off()[v]; e < g.succ_off()[v + 1]; ++e) {
        const int32_t u = g.succ_idx()[e];
        auto it = depth.find(u);
        if (it == depth.end()) continue;
        it->second = std::max(it->second, depth[v]);
        if (--miss[u] == 0) order.push_back(u);
      }
    }
    if (best != static_cast<int32_t>(comp[w].size())) return no("worker compute ops not totally ordered");
    ps.last_compute.push_back(last);
    for (int32_t s_ : ps.sends[w]) {
      for (int32_t e = g.succ_off()[s_]; e < g.succ_off()[s_ + 1]; ++e) {
        const int32_t u = g.succ_idx()[e];
        if (psix[u] < 0) return no("send feeding a worker op");
        ps.send_succ.push_back(static_cast<int16_t>(psix[u]));
      }
      ps.send_succ_off.push_back(static_cast<int32_t>(ps.send_succ.size()));
    }
  }
  ps.send_succ_off.insert(ps.send_succ_off.begin(), 0);
  // active resources in resource order: the PS cores and every worker channel
  std::vector<std::pair<int32_t, int32_t>> act;  // (resource index, slot)
  for (int32_t k = 0; k < ps.nps; ++k) act.emplace_back(core_res[k], -1 - k);
  for (int32_t w = 0; w < W; ++w)
    for (int32_t ch = 0; ch < ps.nch; ++ch) act.emplace_back(chans[w][ch], w * ps.nch + ch);
  std::sort(act.begin(), act.end());
  for (const auto& [r, sl] : act) ps.slots.push_back(sl);
  ps.ok = true;
  return ps;
}

// Weights the shape with one oracle's durations (O(n)).
bool chain_tables(const ChainShape& cs, const Graph& g, const std::vector<int64_t>& dur, ChainTables& t,
                  std::string& why) {
  if (!cs.ok) return why = cs.why, false;
  t.R = cs.R;
  t.nc = cs.nc;
  t.first = cs.first;
  t.d.resize(cs.R);
  for (int32_t c = 0; c < cs.R; ++c) t.d[c] = dur[g.recv_ops()[c]];
  std::vector<int64_t> weight(cs.nc, 0);
  for (int32_t v = 0; v < g.n(); ++v)
    if (cs.class_of[v] >= 0) weight[cs.class_of[v]] += dur[v];
  if (cs.nested) {
    t.pwsuf.assign(cs.nc + 1, 0);
    for (int32_t j = cs.nc - 1; j >= 0; --j) t.pwsuf[j] = t.pwsuf[j + 1] + weight[j];
  } else {
    t.wj.resize(cs.dag.recs.size());
    for (size_t r = 0; r < cs.dag.recs.size(); ++r)
      t.wj[r] = cs.dag.rec_join[r] < 0 ? 0 : weight[cs.dag.join_class[cs.dag.rec_join[r]]];
    t.wr.assign(cs.R, 0);
    for (int32_t j = 0; j < cs.nc; ++j)
      if (cs.dag.single[j] >= 0) t.wr[cs.dag.single[j]] += weight[j];
    t.w0 = 0;
    for (int32_t j : cs.dag.empty) t.w0 += weight[j];
  }
  t.send_total = 0;
  for (int32_t i : cs.sends) t.send_total += dur[i];
  t.nch = cs.nch;
  t.ch = cs.recv_ch;
  t.send_by_ch.assign(cs.nch, 0);
  for (size_t k = 0; k < cs.sends.size(); ++k) t.send_by_ch[cs.send_ch[k]] += dur[cs.sends[k]];
  for (int64_t x : t.d)
    if (x >= (int64_t{1} << 31)) return why = "recv duration beyond 32 bits", false;
  return true;
}

}  // namespace

SweepCtx::~SweepCtx() {
  if (plan) csk_sweep_plan_free(plan);
  if (d_order_) cudaFree(d_order_);
  if (d_ms_) cudaFree(d_ms_);
}

int64_t SweepCtx::order_makespan(const std::vector<int32_t>& order) {
  std::lock_guard<std::mutex> lock(mu_);
  auto ck = [](cudaError_t e) {
    if (e != cudaSuccess) fail(kInternal, std::string("CUDA error: ") + cudaGetErrorString(e));
  };
  if (!d_order_) {
    ck(cudaMalloc(&d_order_, sizeof(int32_t) * std::max<size_t>(order.size(), 1)));
    ck(cudaMalloc(&d_ms_, sizeof(int64_t)));
  }
  ck(cudaMemcpy(d_order_, order.data(), sizeof(int32_t) * order.size(), cudaMemcpyHostToDevice));
  char err[256] = {0};
  if (csk_sweep_orders(plan, d_order_, 1, nullptr, d_ms_, err)) fail(kInternal, err);
  int64_t m = 0;
  ck(cudaMemcpy(&m, d_ms_, sizeof(int64_t), cudaMemcpyDeviceToHost));
  return m;
}

std::unique_ptr<SweepCtx> make_sweep(std::shared_ptr<const Graph> g, const TimeOracle& o,
                                     const Policy& p) {
  auto s = std::make_unique<SweepCtx>();
  const auto t0 = std::chrono::steady_clock::now();
  s->g = g;
  s->dur = o.durations(*g);
  if (p.noise < 0.0 || p.noise > 1.0) fail(kParameter, "reorder_noise must be within [0, 1]");
  s->policy = p;
  std::tie(s->U, s->L) = bounds(*g, o);
  s->cluster = g->cluster();
  if (s->cluster) {
    s->workers = g->worker_devices();
    std::unordered_map<std::string, int32_t> widx;
    for (size_t i = 0; i < s->workers.size(); ++i) widx[s->workers[i]] = static_cast<int32_t>(i);
    for (int32_t r : g->recv_ops()) {
      auto it = widx.find(g->ops()[r].res.device);
      s->recv_worker.push_back(it == widx.end() ? 0 : it->second);
    }
    // every worker partition must validate, as schedule_for builds them
    for (const auto& dv : s->workers) (void)g->partition(dv);
  } else {
    s->workers = {};
    s->recv_worker.assign(g->recv_ops().size(), 0);
  }
  // fast path?
  // Gated: reorder noise only permutes the gate sequence up front, which the
  // sweep kernel applies before folding (explicit-order and single-run
  // callers, which do not, check `noisy`). Ungated: noise is ignored
  // (sim.cpp:106) and, with distinct recv priorities — every random order
  // and permutation — the channel still runs the recvs back-to-back in
  // priority order without a draw, i.e. exactly the gated run; callers with
  // explicit priorities check distinctness (capi.cpp).
  s->noisy = p.gated && p.noise > 0.0;
  if (cudaGetDevice(&s->device) != cudaSuccess) s->device = 0;
  bool ok = s->U < (int64_t{1} << 37);
  if (!ok) s->why = "makespan bound beyond the statistics key range";
  if (ok && std::getenv("TICTAC_SWEEP_FORCE_EXACT")) {  // test knob: the exact event replica
    ok = false;
    s->why = "forced by TICTAC_SWEEP_FORCE_EXACT";
  }
  std::vector<ChainTables> tabs;
  std::shared_ptr<const ChainShape> shape0;  // worker 0's shape (the program the workers share)
  std::shared_ptr<const PsShape> pshape;      // clusters whose PS ops take time
  bool need_ps = false;
  if (ok && !s->cluster) {
    tabs.emplace_back();
    shape0 = g->memo<ChainShape>("chain", [&] { return chain_shape(*g, false); });
    ok = chain_tables(*shape0, *g, s->dur, tabs.back(), s->why);
  } else if (ok) {
    // The full makespan (every event, the parameter servers' included) is
    // the slowest worker's when the PS devices add no time: their ops only
    // wait for the workers' sends and take zero time (config 3's
    // expand_to_mr(…, ps_op_time = 0)); otherwise only the exact replica
    // gives it (SURVEY A.2 covers the workers).
    std::set<std::string> wset(s->workers.begin(), s->workers.end());
    for (int32_t i = 0; i < g->n(); ++i)
      if (!wset.count(g->ops()[i].res.device) && s->dur[i] != 0) need_ps = true;
    if (need_ps && std::getenv("TICTAC_SWEEP_NO_PS")) {
      ok = false;
      s->why = "parameter-server ops take time (send phase disabled by TICTAC_SWEEP_NO_PS)";
    }
    if (need_ps && ok) {  // the send phase of cluster_ps_kernel
      pshape = g->memo<PsShape>("ps", [&] { return ps_shape(*g, s->workers); });
      if (!pshape->ok) {
        ok = false;
        s->why = "parameter-server ops take time and " + pshape->why;
      }
      for (size_t w = 0; ok && w < pshape->last_compute.size(); ++w)
        if (s->dur[pshape->last_compute[w]] <= 0) {
          ok = false;
          s->why = "parameter-server ops take time and a worker's last compute op takes none";
        }
    }
    // devices other than workers must not feed back into workers
    for (const auto& dv : s->workers) {
      auto part = g->partition(dv);
      std::vector<int64_t> pd(part->n());
      for (int32_t i = 0; i < part->n(); ++i) pd[i] = s->dur[g->at(part->ops()[i].id)];
      for (int32_t i = 0; i < g->n(); ++i)
        if (g->ops()[i].res.device != dv)
          for (int32_t e = g->succ_off()[i]; e < g->succ_off()[i + 1]; ++e)
            if (g->ops()[g->succ_idx()[e]].res.device == dv) {
              ok = false;
              s->why = "worker depends on another device";
            }
      if (!ok) break;
      tabs.emplace_back();
      const auto shape = g->memo<ChainShape>("chain:" + dv, [&] { return chain_shape(*part, true); });
      if (!(ok = chain_tables(*shape, *part, pd, tabs.back(), s->why))) break;
      if (!shape0) shape0 = shape;
      if (tabs.back().R != tabs[0].R || tabs.back().nc != tabs[0].nc || shape->nested != shape0->nested ||
          shape->nch != shape0->nch ||
          (!shape->nested && (shape->dag.recs != shape0->dag.recs || shape->dag.rec_join != shape0->dag.rec_join))) {
        ok = false;
        s->why = "workers differ in shape";
        break;
      }
    }
  }
  const auto t1 = std::chrono::steady_clock::now();
  if (std::getenv("TICTAC_SWEEP_TRACE") && shape0)
    std::fprintf(stderr, "[make_sweep] ok=%d nested=%d R=%d classes=%d joins=%d slots=%d words=%zu (%s)\n", ok ? 1 : 0,
                 shape0->nested ? 1 : 0, shape0->R, shape0->nc, shape0->dag.J, shape0->dag.L,
                 shape0->dag.recs.size(), s->why.c_str());
  if (ok) {
    const int32_t W = static_cast<int32_t>(tabs.size()), R = tabs[0].R, nc = tabs[0].nc;
    std::vector<int64_t> d, pw, send, send_ch;
    std::vector<int32_t> first, ch;
    for (const auto& t : tabs) {
      d.insert(d.end(), t.d.begin(), t.d.end());
      first.insert(first.end(), t.first.begin(), t.first.end());
      pw.insert(pw.end(), t.pwsuf.begin(), t.pwsuf.end());
      send.push_back(t.send_total);
      ch.insert(ch.end(), t.ch.begin(), t.ch.end());
      send_ch.insert(send_ch.end(), t.send_by_ch.begin(), t.send_by_ch.end());
    }
    const int32_t nch = tabs[0].nch;
    s->nch = nch;
    char err[256] = {0};
    uint64_t noise_thr = 0;  // unit() < p  <=>  (output >> 11) < p * 2^53 (integers below 2^53)
    if (s->noisy) {
      const double t = std::ldexp(p.noise, 53);
      noise_thr = t == std::floor(t) ? static_cast<uint64_t>(t) : static_cast<uint64_t>(std::floor(t)) + 1;
    }
    const bool fail_ps = need_ps && (!shape0->nested || pshape->nch != nch);
    if (fail_ps) {
    } else if (shape0->nested) {
      s->plan = csk_sweep_plan(W, R, nc, d.data(), first.data(), pw.data(), nch, ch.data(),
                               nch > 1 ? send_ch.data() : send.data(), s->cluster ? 1 : 0, s->U, s->L, noise_thr,
                               err);
      if (s->plan && need_ps) {
        const PsShape& q = *pshape;
        std::vector<int64_t> sd, qd;
        for (const auto& sv : q.sends)
          for (int32_t x : sv) sd.push_back(s->dur[x]);
        for (int32_t x : q.ps_ops) qd.push_back(s->dur[x]);
        if (csk_sweep_plan_add_ps(s->plan, q.S, q.recv_sb.data(), q.ch_mask.data(), sd.data(),
                                  q.send_succ_off.data(), q.send_succ.data(), q.Q, qd.data(), q.ps_missing.data(),
                                  q.ps_succ_off.data(), q.ps_succ.data(), q.nps, q.core_mask.data(),
                                  static_cast<int32_t>(q.slots.size()), q.slots.data(), err)) {
          csk_sweep_plan_free(s->plan);
          s->plan = nullptr;
          fail(kInternal, err);
        }
        s->ps = true;
      }
    } else {
      const DagProgram& dp = shape0->dag;
      std::vector<int64_t> wr, wj, w0;
      for (const auto& t : tabs) {
        wr.insert(wr.end(), t.wr.begin(), t.wr.end());
        wj.insert(wj.end(), t.wj.begin(), t.wj.end());
        w0.push_back(t.w0);
      }
      std::vector<int32_t> recs;
      for (const auto& r : dp.recs) recs.insert(recs.end(), r.begin(), r.end());
      const int32_t nrec = static_cast<int32_t>(dp.recs.size());
      s->plan = csk_sweep_plan_dag(W, R, d.data(), wr.data(), nrec, recs.data(), wj.data(), w0.data(), dp.L,
                                   send.data(), s->cluster ? 1 : 0, s->U, s->L, noise_thr, err);
      s->dag = true;
      s->joins = dp.J;
      s->slots = dp.L;
      s->prog_words = nrec;
    }
    if (!fail_ps && !s->plan) fail(kInternal, err);
    s->fast = !fail_ps;
    if (fail_ps) s->why = "parameter-server ops take time and the workers are not chain-class";
    s->nc = nc;
    s->R = R;
  }
  if (std::getenv("TICTAC_SWEEP_TRACE")) {
    const auto t2 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[make_sweep] analysis %.3f ms, plan %.3f ms\n",
                 std::chrono::duration<double, std::milli>(t1 - t0).count(),
                 std::chrono::duration<double, std::milli>(t2 - t1).count());
  }
  return s;
}

void finish_stats(const SweepCtx& s, const int64_t* i64, const double* f64, uint64_t key_base,
                  cs_sweep_stats* out) {
  std::memset(out, 0, sizeof(*out));
  out->count = i64[3];
  out->upper_us = s.U;
  out->lower_us = s.L;
  if (out->count > 0) {
    const uint64_t kmin = static_cast<uint64_t>(i64[0]), kmax = static_cast<uint64_t>(i64[1]);
    const int kb = csk_key_bits(s.U);
    const uint64_t mask = (1ULL << kb) - 1;
    out->min_us = static_cast<int64_t>(kmin >> kb);
    out->argmin_seed = key_base + (kmin & mask);
    out->max_us = static_cast<int64_t>(kmax >> kb);
    out->argmax_seed = key_base + (mask - (kmax & mask));
  }
  out->sum_us = i64[2];
  out->sumsq_us = f64[0];
  for (int k = 0; k < CS_HIST_BINS; ++k) {
    out->e_hist[k] = i64[8 + k];
    out->straggler_hist[k] = i64[1008 + k];
  }
  out->n_workers = s.cluster ? static_cast<int64_t>(s.workers.size()) : 0;
  out->straggler_sum = f64[1];
  if (s.cluster && out->count > 0) {  // iteration time (slowest worker), keys as above
    const int kb = csk_key_bits(s.U);
    const uint64_t mask = (1ULL << kb) - 1;
    const uint64_t kmin = static_cast<uint64_t>(i64[4]), kmax = static_cast<uint64_t>(i64[5]);
    out->iter_min_us = static_cast<int64_t>(kmin >> kb);
    out->iter_argmin_seed = key_base + (kmin & mask);
    out->iter_max_us = static_cast<int64_t>(kmax >> kb);
    out->iter_argmax_seed = key_base + (mask - (kmax & mask));
    out->iter_sum_us = i64[6];
  }
}

// Exact path: device event simulator over seeds, stats reduced on the device (these
// inputs are outside the closed form, so this is the general replica).
void sweep_exact(SweepCtx& s, uint64_t seed_lo, int64_t count, int64_t* makespans,
                 int64_t* worker_ms, cs_sweep_stats* stats) {
  const Graph& g = *s.g;
  DeviceGraph* dg = g.device();
  const int32_t nw = s.cluster ? static_cast<int32_t>(s.workers.size()) : 1;
  // device index per worker (devices sorted as in the DeviceGraph upload)
  std::vector<std::string> devs;
  for (const Resource& r : g.resources()) devs.push_back(r.device);
  std::sort(devs.begin(), devs.end());
  devs.erase(std::unique(devs.begin(), devs.end()), devs.end());
  std::vector<int32_t> wdev;
  for (const auto& w : s.workers)
    wdev.push_back(static_cast<int32_t>(std::lower_bound(devs.begin(), devs.end(), w) - devs.begin()));
  if (wdev.empty()) wdev.push_back(0);
  // Statistics are reduced on the device per chunk (csk_event_stats: min/max
  // with their lowest run index, sums, histograms); the host only combines
  // the chunks' blocks in seed order. Per-run makespans and device ends are
  // copied back only when the caller asked for them.
  struct Ext {
    int64_t lo = INT64_MAX, hi = INT64_MIN;
    uint64_t alo = 0, ahi = 0;
    void add(int64_t clo, int64_t chi, uint64_t slo, uint64_t shi) {
      if (clo < lo) lo = clo, alo = slo;  // chunks in seed order: ties keep the earlier
      if (chi > hi) hi = chi, ahi = shi;
    }
  } mk, it;
  cs_sweep_stats acc;
  std::memset(&acc, 0, sizeof(acc));
  auto part = std::make_unique<csk_event_stats>();
  const int64_t chunk = 1 << 20;
  std::vector<int64_t> dev_end;
  for (int64_t base = 0; base < count; base += chunk) {
    const int32_t B = static_cast<int32_t>(std::min(chunk, count - base));
    const bool want_dev = s.cluster && worker_ms;
    if (want_dev) dev_end.resize(static_cast<size_t>(B) * devs.size());
    char err[256] = {0};
    const auto t0 = std::chrono::steady_clock::now();
    const uint64_t seed0 = seed_lo + static_cast<uint64_t>(base);
    const int rc = csk_event_sweep(dg, s.dur.data(), seed0, B, s.cluster ? 1 : 0, s.recv_worker.data(), nw,
                                   s.policy.gated ? 1 : 0, s.policy.noise, makespans ? makespans + base : nullptr,
                                   nullptr, nullptr, want_dev ? dev_end.data() : nullptr, wdev.data(), s.U, s.L,
                                   part.get(), err);
    if (rc) fail(kInternal, err);
    if (std::getenv("TICTAC_EVENT_TRACE"))
      std::fprintf(stderr, "[sweep_exact] csk_event_sweep %.3f ms\n",
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    const csk_event_stats& c = *part;
    if (c.stalled) fail(kValidation, "simulation stalled with no runnable op");
    if (want_dev)
      for (int32_t b = 0; b < B; ++b)
        for (int32_t w = 0; w < nw; ++w)
          worker_ms[(base + b) * nw + w] = dev_end[static_cast<size_t>(b) * devs.size() + wdev[w]];
    mk.add(c.min_m, c.max_m, seed0 + static_cast<uint64_t>(c.argmin), seed0 + static_cast<uint64_t>(c.argmax));
    if (s.cluster)
      it.add(c.imin, c.imax, seed0 + static_cast<uint64_t>(c.iargmin), seed0 + static_cast<uint64_t>(c.iargmax));
    acc.count += c.count;
    acc.sum_us += c.sum_m;
    acc.sumsq_us += c.sumsq;
    acc.iter_sum_us += c.isum;
    acc.straggler_sum += c.ssum;
    for (int k = 0; k < CS_HIST_BINS; ++k) {
      acc.e_hist[k] += c.e_hist[k];
      acc.straggler_hist[k] += c.s_hist[k];
    }
  }
  if (!stats) return;
  std::memset(stats, 0, sizeof(*stats));
  stats->count = acc.count;
  stats->upper_us = s.U;
  stats->lower_us = s.L;
  if (stats->count > 0) {
    stats->min_us = mk.lo;
    stats->argmin_seed = mk.alo;
    stats->max_us = mk.hi;
    stats->argmax_seed = mk.ahi;
  }
  stats->sum_us = acc.sum_us;
  stats->sumsq_us = acc.sumsq_us;
  for (int k = 0; k < CS_HIST_BINS; ++k) {
    stats->e_hist[k] = acc.e_hist[k];
    stats->straggler_hist[k] = s.cluster ? acc.straggler_hist[k] : 0;
  }
  stats->n_workers = s.cluster ? nw : 0;
  stats->straggler_sum = acc.straggler_sum;
  if (s.cluster && stats->count > 0) {
    stats->iter_min_us = it.lo;
    stats->iter_argmin_seed = it.alo;
    stats->iter_max_us = it.hi;
    stats->iter_argmax_seed = it.ahi;
    stats->iter_sum_us = acc.iter_sum_us;
  }
}

// ---------------------------------------------------------------------------
// Closed-form sweep execution shared by cs_sweep_random (one device) and
// cs_sweep_random_multi (several devices, one NCCL reduction per round).

namespace {

void cudacheck(cudaError_t e) {
  if (e != cudaSuccess) fail(kInternal, std::string("CUDA error: ") + cudaGetErrorString(e));
}

// Per-call device buffer from the stream-ordered pool (legacy stream).
struct DevBuf {
  void* p = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) cudaFreeAsync(p, 0);
  }
  void alloc(size_t bytes) { cudacheck(cudaMallocAsync(&p, bytes ? bytes : 8, 0)); }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// Page-locked staging buffers for pipelined read-backs, kept for the life of
// the process (pinning is expensive per call) up to a cap; a caller that
// finds none free and would exceed the cap reads back without the pipeline.
class PinnedPool {
 public:
  static constexpr size_t kCapBytes = size_t{1} << 30;
  struct Lease {
    PinnedPool* pool = nullptr;
    char* p = nullptr;
    size_t bytes = 0;
    Lease() = default;
    Lease(const Lease&) = delete;
    Lease& operator=(const Lease&) = delete;
    ~Lease() {
      if (p) pool->put(p, bytes);
    }
  };
  static PinnedPool& get() {
    static PinnedPool* pool = new PinnedPool();  // never destroyed: the OS reclaims at exit
    return *pool;
  }
  bool lease(size_t bytes, Lease& out) {
    std::lock_guard<std::mutex> lock(mu_);
    for (size_t i = 0; i < free_.size(); ++i)
      if (free_[i].second >= bytes) {
        out.pool = this;
        out.p = free_[i].first;
        out.bytes = free_[i].second;
        free_.erase(free_.begin() + static_cast<std::ptrdiff_t>(i));
        return true;
      }
    if (total_ + bytes > kCapBytes) return false;
    void* h = nullptr;
    if (cudaMallocHost(&h, bytes) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    total_ += bytes;
    out.pool = this;
    out.p = static_cast<char*>(h);
    out.bytes = bytes;
    return true;
  }

 private:
  std::mutex mu_;
  size_t total_ = 0;
  std::vector<std::pair<char*, size_t>> free_;
  void put(char* p, size_t bytes) {
    std::lock_guard<std::mutex> lock(mu_);
    free_.emplace_back(p, bytes);
  }
};

// Streams and events of one pipelined read-back. Declared after the staging
// lease, so on every exit path (exceptions included) the destructor first
// waits for both streams — nothing is still copying into the staging buffer
// when it returns to the pool — then destroys them.
struct PipeGuard {
  cudaStream_t sa = nullptr, sb = nullptr;
  cudaEvent_t ready = nullptr;
  std::vector<cudaEvent_t> events;
  PipeGuard() = default;
  PipeGuard(const PipeGuard&) = delete;
  PipeGuard& operator=(const PipeGuard&) = delete;
  cudaEvent_t event() {
    cudaEvent_t e = nullptr;
    cudacheck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    events.push_back(e);
    return e;
  }
  ~PipeGuard() {
    if (sa) cudaStreamSynchronize(sa);
    if (sb) cudaStreamSynchronize(sb);
    for (cudaEvent_t e : events) cudaEventDestroy(e);
    if (ready) cudaEventDestroy(ready);
    if (sa) cudaStreamDestroy(sa);
    if (sb) cudaStreamDestroy(sb);
  }
};

// Runs seeds [lo, lo + n) (n <= 2^26) on the current device, accumulating
// into the device statistics (keys relative to key_base) and copying
// per-seed makespans to the host buffers when given (large spans: launches
// of kSub seeds on one stream, each slice read back on a second stream
// through pinned staging while the next ones run).
void run_span(SweepCtx& ctx, uint64_t lo, int64_t n, uint64_t key_base, int64_t* d_ms, int64_t* d_wms,
              int64_t* d_i64, double* d_f64, int64_t* ms_host, int64_t* wms_host) {
  char err[256] = {0};
  const int64_t W = ctx.cluster ? static_cast<int64_t>(ctx.workers.size()) : 1;
  constexpr int64_t kSub = int64_t{1} << 19;
  PinnedPool::Lease stage;
  const size_t slice_bytes = 8 * static_cast<size_t>(kSub) * ((d_ms ? 1 : 0) + (d_wms ? W : 0));
  const bool piped = (d_ms || d_wms) && n >= 4 * kSub && PinnedPool::get().lease(2 * slice_bytes, stage);
  if (!piped) {
    if (csk_sweep_run(ctx.plan, lo, n, key_base, nullptr, d_ms, d_wms, d_i64, d_f64, err)) fail(kInternal, err);
    if (d_ms) cudacheck(cudaMemcpy(ms_host, d_ms, 8 * n, cudaMemcpyDeviceToHost));
    if (d_wms) cudacheck(cudaMemcpy(wms_host, d_wms, 8 * n * W, cudaMemcpyDeviceToHost));
    return;
  }
  PipeGuard pg;
  cudacheck(cudaStreamCreateWithFlags(&pg.sa, cudaStreamNonBlocking));
  cudacheck(cudaStreamCreateWithFlags(&pg.sb, cudaStreamNonBlocking));
  cudacheck(cudaEventCreateWithFlags(&pg.ready, cudaEventDisableTiming));
  const int64_t K = (n + kSub - 1) / kSub;
  std::vector<cudaEvent_t> ran(static_cast<size_t>(K)), copied(static_cast<size_t>(K));
  for (int64_t k = 0; k < K; ++k) {
    ran[k] = pg.event();
    copied[k] = pg.event();
  }
  cudacheck(cudaEventRecord(pg.ready, 0));  // buffers and the reset, issued on the legacy stream
  cudacheck(cudaStreamWaitEvent(pg.sa, pg.ready, 0));
  for (int64_t k = 0; k < K; ++k) {
    const int64_t off = k * kSub, nk = std::min(kSub, n - off);
    if (csk_sweep_run(ctx.plan, lo + static_cast<uint64_t>(off), nk, key_base, pg.sa, d_ms ? d_ms + off : nullptr,
                      d_wms ? d_wms + off * W : nullptr, d_i64, d_f64, err))
      fail(kInternal, err);
    cudacheck(cudaEventRecord(ran[k], pg.sa));
  }
  auto land = [&](int64_t k) {  // staging slot k % 2 -> the caller's buffers
    cudacheck(cudaEventSynchronize(copied[k]));
    const int64_t off = k * kSub, nk = std::min(kSub, n - off);
    const char* src = stage.p + (k & 1) * slice_bytes;
    if (d_ms) {
      std::memcpy(ms_host + off, src, 8 * nk);
      src += 8 * kSub;
    }
    if (d_wms) std::memcpy(wms_host + off * W, src, 8 * nk * W);
  };
  for (int64_t k = 0; k < K; ++k) {
    const int64_t off = k * kSub, nk = std::min(kSub, n - off);
    char* dst = stage.p + (k & 1) * slice_bytes;
    cudacheck(cudaStreamWaitEvent(pg.sb, ran[k], 0));
    if (d_ms) {
      cudacheck(cudaMemcpyAsync(dst, d_ms + off, 8 * nk, cudaMemcpyDeviceToHost, pg.sb));
      dst += 8 * kSub;
    }
    if (d_wms) cudacheck(cudaMemcpyAsync(dst, d_wms + off * W, 8 * nk * W, cudaMemcpyDeviceToHost, pg.sb));
    cudacheck(cudaEventRecord(copied[k], pg.sb));
    if (k >= 1) land(k - 1);
  }
  land(K - 1);
}

}  // namespace

void merge_stats(cs_sweep_stats& total, const cs_sweep_stats& part, bool first) {
  if (first) {
    total = part;
    return;
  }
  if (part.count <= 0) return;
  if (total.count <= 0) {
    const int64_t U = total.upper_us, L = total.lower_us;
    total = part;
    total.upper_us = U;
    total.lower_us = L;
    return;
  }
  if (part.min_us < total.min_us) total.min_us = part.min_us, total.argmin_seed = part.argmin_seed;
  if (part.max_us > total.max_us) total.max_us = part.max_us, total.argmax_seed = part.argmax_seed;
  if (part.iter_min_us < total.iter_min_us)
    total.iter_min_us = part.iter_min_us, total.iter_argmin_seed = part.iter_argmin_seed;
  if (part.iter_max_us > total.iter_max_us)
    total.iter_max_us = part.iter_max_us, total.iter_argmax_seed = part.iter_argmax_seed;
  total.count += part.count;
  total.sum_us += part.sum_us;
  total.iter_sum_us += part.iter_sum_us;
  total.sumsq_us += part.sumsq_us;
  total.straggler_sum += part.straggler_sum;
  for (int k = 0; k < CS_HIST_BINS; ++k) {
    total.e_hist[k] += part.e_hist[k];
    total.straggler_hist[k] += part.straggler_hist[k];
  }
}

cs_sweep_stats sweep_fast(const std::vector<SweepCtx*>& ctxs, uint64_t seed_lo, int64_t count,
                          int64_t* makespans, int64_t* worker_ms, const DeviceReducer* reducer) {
  const int nd = static_cast<int>(ctxs.size());
  const SweepCtx& c0 = *ctxs[0];
  const int64_t W = c0.cluster ? static_cast<int64_t>(c0.workers.size()) : 1;
  const int kb = csk_key_bits(c0.U);
  // a round's seed offsets must stay below 2^key_bits; a device's span
  // within a round below 2^26 (its per-seed buffers)
  const int64_t per_dev_cap = int64_t{1} << 26;
  const int64_t round = std::min<int64_t>(int64_t{1} << std::min(kb, 40), per_dev_cap * nd);
  cs_sweep_stats total{};
  bool first = true;
  std::vector<int64_t> i64(CS_DSTATS_I64);
  std::vector<double> f64(CS_DSTATS_F64);
  for (int64_t base = 0; base < count || (first && count == 0); base += round) {
    const int64_t rn = std::min(round, count - base);
    const uint64_t rlo = seed_lo + static_cast<uint64_t>(base);
    std::vector<std::string> errors(nd);
    auto device_part = [&](int d) {
      try {
        cudacheck(cudaSetDevice(ctxs[d]->device));
        const int64_t per = (rn + nd - 1) / nd;
        const int64_t off = std::min<int64_t>(rn, d * per), n = std::min<int64_t>(per, rn - off);
        DevBuf st, ms, wms;  // statistics: i64 then f64 words
        st.alloc(8 * (CS_DSTATS_I64 + CS_DSTATS_F64));
        int64_t* d_i64 = st.as<int64_t>();
        double* d_f64 = reinterpret_cast<double*>(d_i64 + CS_DSTATS_I64);
        char err[256] = {0};
        if (csk_sweep_reset(ctxs[d]->plan, nullptr, d_i64, d_f64, err)) fail(kInternal, err);
        if (makespans && n > 0) ms.alloc(8 * n);
        if (worker_ms && c0.cluster && n > 0) wms.alloc(8 * n * W);
        if (n > 0)
          run_span(*ctxs[d], rlo + static_cast<uint64_t>(off), n, rlo, ms.as<int64_t>(), wms.as<int64_t>(), d_i64,
                   d_f64, makespans ? makespans + base + off : nullptr,
                   worker_ms && c0.cluster ? worker_ms + (base + off) * W : nullptr);
        if (nd > 1) {
          reducer->reduce(d, d_i64, d_f64, d == 0 ? i64.data() : nullptr, d == 0 ? f64.data() : nullptr);
        } else {
          std::vector<char> h(8 * (CS_DSTATS_I64 + CS_DSTATS_F64));
          cudacheck(cudaMemcpy(h.data(), d_i64, h.size(), cudaMemcpyDeviceToHost));
          std::memcpy(i64.data(), h.data(), 8 * CS_DSTATS_I64);
          std::memcpy(f64.data(), h.data() + 8 * CS_DSTATS_I64, 8 * CS_DSTATS_F64);
        }
      } catch (const std::exception& e) {
        errors[d] = e.what();
      }
    };
    if (nd == 1) {
      device_part(0);
    } else {
      std::vector<std::thread> th;
      for (int d = 0; d < nd; ++d) th.emplace_back(device_part, d);
      for (auto& t : th) t.join();
    }
    for (const auto& e : errors)
      if (!e.empty()) fail(kInternal, e);
    cs_sweep_stats part{};
    finish_stats(c0, i64.data(), f64.data(), rlo, &part);
    merge_stats(total, part, first);
    first = false;
    if (count == 0) break;
  }
  return total;
}

}  // namespace tictac
