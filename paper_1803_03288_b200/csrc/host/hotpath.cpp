// Host orchestration of the hot path: argument checks and error semantics
// of the reference, then the device kernels (../device/csk.h) do the work.
//   properties  -> properties.cpp:68-109   (csk_properties)
//   tic / tac   -> schedule.cpp:21-71      (csk_tic / csk_tac)
//   random      -> schedule.cpp:73-84      (csk_random_orders)
//   simulate    -> sim.cpp:61-256          (csk_event_sim; csk_event_a2 for event
//                                           lists inside A.2's regime; the
//                                           closed form via csk_sweep_orders
//                                           when only the makespan is needed)
//   brute force -> metrics.cpp:37-72       (csk_brute_force_closed / csk_brute_force)
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <set>

#include "../device/csk.h"
#include "core.hpp"
#include "rng_host.hpp"

namespace tictac {

static void check(int rc, const char* err) {
  if (rc) fail(rc == kValidation ? kValidation : kInternal, err);
}

PropMode prop_mode(std::string_view s) {  // properties.cpp:15-19
  if (s == "literal") return PropMode::Literal;
  if (s == "amended") return PropMode::Amended;
  fail(kParameter, "unknown property mode: " + std::string(s));
}

Json properties_json(const Graph& g, const TimeOracle& o, PropMode mode) {
  const std::vector<int64_t> d = o.durations(g);  // check_covers, properties.cpp:76
  const int32_t n = g.n(), R = static_cast<int32_t>(g.recv_ops().size());
  const int32_t w = std::max(1, (R + 63) / 64);
  std::vector<uint64_t> bits(static_cast<size_t>(n) * w);
  std::vector<int64_t> M(n), P(std::max(R, 1)), Mp(std::max(R, 1));
  char err[256] = {0};
  check(csk_properties(g.device(), d.data(), mode == PropMode::Amended, bits.data(), M.data(),
                       P.data(), Mp.data(), err),
        err);
  const std::vector<std::string> recvs = g.recv_ids();
  Json j;
  j["mode"] = mode == PropMode::Literal ? "literal" : "amended";
  j["dep"] = Json::object();
  for (int32_t v = 0; v < n; ++v) {
    Json list = Json::array();
    for (int32_t c = 0; c < R; ++c)
      if ((bits[static_cast<size_t>(v) * w + (c >> 6)] >> (c & 63)) & 1) list.push_back(recvs[c]);
    j["dep"][g.ops()[v].id] = std::move(list);
  }
  j["M"] = Json::object();
  for (int32_t v = 0; v < n; ++v) j["M"][g.ops()[v].id] = M[v];
  j["P"] = Json::object();
  for (int32_t c = 0; c < R; ++c) j["P"][recvs[c]] = P[c];
  j["M_plus"] = Json::object();
  for (int32_t c = 0; c < R; ++c) {
    if (Mp[c] == INT64_MAX) j["M_plus"][recvs[c]] = nullptr;
    else j["M_plus"][recvs[c]] = Mp[c];
  }
  return j;
}

static Schedule ranks_to_schedule(const Graph& g, const char* algo, const std::vector<int32_t>& pr,
                                  bool total) {
  Schedule s;
  s.graph = g.name();
  s.algorithm = algo;
  const auto& ro = g.recv_ops();
  // recv columns follow op index = byte-lexicographic id order, which is the
  // map's order: append with an end hint (amortised O(1) per recv)
  for (size_t c = 0; c < ro.size(); ++c) s.prio.emplace_hint(s.prio.end(), g.ops()[ro[c]].id, pr[c]);
  s.total = total;
  return s;
}

Schedule tic(const Graph& g, PropMode mode) {
  const int32_t R = static_cast<int32_t>(g.recv_ops().size());
  std::vector<int32_t> pr(std::max(R, 1));
  int total = 1;
  char err[256] = {0};
  check(csk_tic(g.device(), mode == PropMode::Amended, pr.data(), &total, err), err);
  return ranks_to_schedule(g, "tic", pr, total != 0);
}

Schedule tac(const Graph& g, const TimeOracle& o) {
  const int32_t R = static_cast<int32_t>(g.recv_ops().size());
  std::vector<int32_t> pr(std::max(R, 1));
  if (R > 0) {  // the reference touches the oracle only inside a round
    const std::vector<int64_t> d = o.durations(g);
    char err[256] = {0};
    check(csk_tac(g.device(), d.data(), pr.data(), err), err);
  }
  return ranks_to_schedule(g, "tac", pr, true);
}

Schedule random_schedule(const Graph& g, uint64_t seed) {
  const int32_t R = static_cast<int32_t>(g.recv_ops().size());
  std::vector<int32_t> perm(std::max(R, 1)), pr(std::max(R, 1));
  if (R > 0) {
    char err[256] = {0};
    check(csk_random_orders(R, 1, &seed, perm.data(), err), err);
    for (int32_t k = 0; k < R; ++k) pr[perm[k]] = k;
  }
  return ranks_to_schedule(g, "random", pr, true);
}

Schedule schedule_for(const Graph& g, const std::string& algo, PropMode mode, uint64_t seed,
                      const TimeOracle* o) {
  auto one = [&](const Graph& target, uint64_t s) {
    if (algo == "tic") return tic(target, mode);
    if (algo == "tac") {
      if (!o) fail(kParameter, "tac needs a time oracle");
      return tac(target, *o);
    }
    if (algo == "random") return random_schedule(target, s);
    fail(kParameter, "unknown scheduling algorithm: " + algo);
  };
  if (!g.cluster()) return one(g, seed);
  Schedule merged;
  merged.graph = g.name();
  merged.algorithm = algo;
  const std::vector<std::string> devices = g.worker_devices();
  bool total = true;
  for (size_t i = 0; i < devices.size(); ++i) {
    const auto part = g.partition(devices[i]);
    const uint64_t derived = splitmix64(seed ^ (0x9e3779b97f4a7c15ULL * (i + 1)));
    Schedule s = one(*part, derived);
    total = total && s.total;
    for (const auto& kv : s.prio) merged.prio[kv.first] = kv.second;
  }
  merged.total = total && devices.size() <= 1;  // ranks restart per worker
  return merged;
}

static void policy_check(const Policy& p) {
  if (p.noise < 0.0 || p.noise > 1.0) fail(kParameter, "reorder_noise must be within [0, 1]");
}

SimInputs prepare_sim(const Graph& g, const TimeOracle& o, const Schedule* s, const Policy& p) {
  SimInputs in;
  in.d = o.durations(g);  // sim.cpp:63
  policy_check(p);
  in.prio.assign(g.n(), -1);
  if (s) {
    for (const auto& [id, rank] : s->prio) {  // sim.cpp:79-88
      if (!g.has(id)) fail(kValidation, "schedule references unknown op: " + id);
      const int32_t i = g.at(id);
      if (g.ops()[i].kind != kRecv) fail(kValidation, "schedule priority on non-recv op: " + id);
      in.prio[i] = rank;
    }
  }
  in.all_recvs_prioritized = true;
  for (int32_t r : g.recv_ops()) in.all_recvs_prioritized &= in.prio[r] >= 0;
  return in;
}

Report simulate(const Graph& g, const TimeOracle& o, const Schedule* s, const Policy& p) {
  const SimInputs in = prepare_sim(g, o, s, p);
  return simulate_prepared(g, in.d, in.prio, p);
}

namespace {

// Report from per-op start/end times (events sorted by start, resource, op).
Report make_report(const Graph& g, const std::vector<int64_t>& st, const std::vector<int64_t>& en, int64_t m,
                   int64_t viol) {
  const int32_t n = g.n();
  Report r;
  r.makespan = m;
  r.violations = viol;
  r.resources = g.resources();
  r.graph = g.shared_from_this();
  r.events.reserve(n);
  for (int32_t i = 0; i < n; ++i) r.events.push_back({i, g.res_of()[i], st[i], en[i]});
  // order by (start, resource, op id): one LSD radix sort over the packed key
  // when start | resource | op fit 64 bits (always, for real graphs)
  auto bits = [](uint64_t v) { return v ? 64 - __builtin_clzll(v) : 0; };
  int64_t smax = 0;
  bool nonneg = true;
  for (int32_t i = 0; i < n; ++i) smax = std::max(smax, st[i]), nonneg = nonneg && st[i] >= 0;
  const int bo = bits(static_cast<uint64_t>(std::max(n - 1, 0))), br = bits(r.resources.size());
  const int bs = bits(static_cast<uint64_t>(smax));
  if (nonneg && n > 1 && bs + br + bo <= 64) {
    std::vector<uint64_t> key(n), tmp(n);
    for (int32_t i = 0; i < n; ++i)
      key[i] = (static_cast<uint64_t>(st[i]) << (br + bo)) | (static_cast<uint64_t>(g.res_of()[i]) << bo) |
               static_cast<uint64_t>(i);
    const int total = bs + br + bo;
    for (int shift = 0; shift < total; shift += 11) {
      size_t cnt[2049] = {0};
      for (uint64_t k : key) ++cnt[((k >> shift) & 2047) + 1];
      for (int d = 0; d < 2048; ++d) cnt[d + 1] += cnt[d];
      for (uint64_t k : key) tmp[cnt[(k >> shift) & 2047]++] = k;
      key.swap(tmp);
    }
    const uint64_t mask = bo ? (~uint64_t{0} >> (64 - bo)) : 0;
    for (int32_t k = 0; k < n; ++k) {
      const int32_t i = static_cast<int32_t>(key[k] & mask);
      r.events[k] = {i, g.res_of()[i], st[i], en[i]};
    }
  } else {
    std::sort(r.events.begin(), r.events.end(), [](const Report::Event& a, const Report::Event& b) {
      if (a.start != b.start) return a.start < b.start;
      if (a.res != b.res) return a.res < b.res;
      return a.op < b.op;
    });
  }
  if (g.cluster()) {  // iteration_stats, sim.cpp:258-279
    std::map<std::string, int64_t> pw;
    for (const std::string& dv : g.worker_devices()) pw[dv] = 0;
    for (const auto& e : r.events) {
      auto it = pw.find(r.resources[e.res].device);
      if (it != pw.end()) it->second = std::max(it->second, e.end);
    }
    if (pw.empty()) fail(kValidation, "graph has no worker devices");
    int64_t lo = INT64_MAX, hi = 0;
    for (const auto& [dv, mm] : pw) {
      lo = std::min(lo, mm);
      hi = std::max(hi, mm);
      r.per_worker.emplace_back(dv, mm);
    }
    r.has_stats = true;
    r.iteration = hi;
    if (hi == 0) {
      r.strag_num = 0;
      r.strag_den = 1;
    } else {
      const Rational q(hi - lo, hi);
      r.strag_num = q.num;
      r.strag_den = q.den;
    }
  }
  return r;
}

}  // namespace

Report simulate_prepared(const Graph& g, const std::vector<int64_t>& d, const std::vector<int32_t>& prio,
                         const Policy& p) {
  const int32_t n = g.n();
  std::vector<int64_t> st(n), en(n);
  int64_t m = 0, viol = 0;
  int32_t status = 0;
  const uint64_t seed = p.choice_seed;
  char err[256] = {0};
  check(csk_event_sim(g.device(), d.data(), 1, prio.data(), nullptr, 0, &seed, p.gated ? 1 : 0,
                      p.noise, &m, &viol, &status, st.data(), en.data(), nullptr, err),
        err);
  if (status) fail(kValidation, "simulation stalled with no runnable op");
  return make_report(g, st, en, m, viol);
}

int64_t apply_gate_noise(std::vector<int32_t>& order, const Policy& p) {
  if (!p.gated || p.noise <= 0.0) return 0;
  HostRng nr(splitmix64(p.choice_seed ^ 0x9e3779b97f4a7c15ULL));
  int64_t swaps = 0;
  for (size_t pos = 1; pos < order.size(); ++pos)
    if (nr.unit() < p.noise) {
      std::swap(order[pos - 1], order[pos]);
      ++swaps;
    }
  return swaps;
}

Report simulate_a2(const Graph& g, const std::vector<int64_t>& d, const std::vector<int32_t>& prio,
                   const Policy& p) {
  // gate sequence: recvs by (priority, id) (sim.cpp:95-104), then the reorder
  // noise swaps; recvs complete in gate order, so the violations are the
  // swaps and nothing is force-released
  const bool trace = std::getenv("TICTAC_EVENT_TRACE") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<int32_t> order(g.recv_ops().begin(), g.recv_ops().end());
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return prio[a] < prio[b]; });
  const int64_t swaps = apply_gate_noise(order, p);
  const int32_t n = g.n();
  std::vector<int64_t> st(n), en(n);
  int64_t m = 0;
  char err[256] = {0};
  check(csk_event_a2(g.device(), d.data(), order.data(), static_cast<int32_t>(order.size()), p.choice_seed, &m,
                     st.data(), en.data(), err),
        err);
  const auto t1 = std::chrono::steady_clock::now();
  Report r = make_report(g, st, en, m, swaps);
  if (trace)
    std::fprintf(stderr, "[simulate_a2] device call %.3f ms, report build %.3f ms\n",
                 std::chrono::duration<double, std::milli>(t1 - t0).count(),
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count());
  return r;
}

std::pair<int64_t, int64_t> bounds(const Graph& g, const TimeOracle& o) {
  // metrics.cpp:10-22; U/L are per-graph constants, summed once here.
  const std::vector<int64_t> d = o.durations(g);
  int64_t U = 0, L = 0;
  std::vector<int64_t> per(g.resources().size(), 0);
  for (int32_t i = 0; i < g.n(); ++i) {
    U += d[i];
    per[g.res_of()[i]] += d[i];
  }
  for (int64_t x : per) L = std::max(L, x);
  return {U, L};
}

Json brute_force(const Graph& g, const TimeOracle& o, const Policy& p, int max_recvs) {
  std::vector<std::string> recvs = g.recv_ids();
  if (static_cast<int>(recvs.size()) > max_recvs)
    fail(kParameter, "brute force refused: " + std::to_string(recvs.size()) +
                         " recv ops exceed " + std::to_string(max_recvs));
  const std::vector<int64_t> d = o.durations(g);
  policy_check(p);
  const int32_t R = static_cast<int32_t>(recvs.size());
  int64_t perms = 1;
  for (int32_t k = 2; k <= R; ++k) perms *= k;
  std::vector<int64_t> ms(static_cast<size_t>(perms));
  char err[256] = {0};
  check(csk_brute_force(g.device(), d.data(), R, p.choice_seed, p.noise, ms.data(), err), err);
  int64_t best = 0, arg = 0;
  for (int64_t k = 0; k < perms; ++k) {
    if (ms[k] < 0) fail(kValidation, "simulation stalled with no runnable op");
    if (k == 0 || ms[k] < best) {
      best = ms[k];
      arg = k;
    }
  }
  // Unrank the lexicographic index (recvs are already ascending).
  std::vector<std::string> pool = recvs, order;
  int64_t rem = arg, f = perms;
  for (int32_t k = R; k >= 1; --k) {
    f /= k;
    const int64_t q = rem / f;
    rem %= f;
    order.push_back(pool[static_cast<size_t>(q)]);
    pool.erase(pool.begin() + q);
  }
  std::sort(ms.begin(), ms.end());
  ms.erase(std::unique(ms.begin(), ms.end()), ms.end());
  Json j;
  j["order"] = order;
  j["makespan_us"] = best;
  j["distribution"] = ms;
  return j;
}

}  // namespace tictac
