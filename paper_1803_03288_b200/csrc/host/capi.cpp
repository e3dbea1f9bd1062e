// The drop-in C ABI (include/commsched.h): the reference's 40 cs_* entry
// points with identical signatures, status codes, ownership and
// thread-local error messages (reference capi.cpp:21-424), plus the batched
// extensions. Compute entry points run on the GPU through ../device/csk.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../../include/commsched.h"
#include "../device/csk.h"
#include "core.hpp"
#include "sweep.hpp"

using namespace tictac;

namespace {
std::atomic<uint64_t> g_oracle_ids{1};
}

struct cs_graph {
  std::shared_ptr<Graph> g;
  // Last sweep plan built per CUDA device for (oracle id, policy): graph and
  // oracle handles are immutable, so repeated sweeps reuse the device tables.
  struct Cached {
    std::shared_ptr<SweepCtx> ctx;
    uint64_t oracle = 0;
    bool gated = true;
    double noise = 0.0;
  };
  std::mutex mu;
  std::map<int, Cached> sweep;
};
struct cs_oracle {
  TimeOracle o;
  uint64_t id = g_oracle_ids.fetch_add(1);
};
struct cs_schedule {
  Schedule s;
};
// A simulation report. Makespan and violations are always present; the
// event list is either computed eagerly (exact device event simulator) or,
// when the closed form of SURVEY A.2 produced the makespan, on first request
// from the retained inputs (graph, durations, priorities, policy).
struct cs_report {
  int64_t makespan = 0, violations = 0;
  bool has_stats = false;
  std::shared_ptr<const Graph> g;
  std::vector<int64_t> d;
  std::vector<int32_t> prio;
  Policy pol;
  mutable std::mutex mu;
  mutable std::unique_ptr<Report> full;
  const Report& report() const {
    std::lock_guard<std::mutex> lock(mu);
    if (!full) {
      // Deferred reports exist only inside the closed form's regime; the
      // specialised replica also needs the compute ops unprioritized.
      bool compute_prio = false;
      for (int32_t i = 0; i < g->n() && !compute_prio; ++i)
        compute_prio = g->ops()[i].kind != kRecv && prio[i] >= 0;
      if (compute_prio || std::getenv("TICTAC_NO_A2"))
        full = std::make_unique<Report>(simulate_prepared(*g, d, prio, pol));
      else
        full = std::make_unique<Report>(simulate_a2(*g, d, prio, pol));
    }
    return *full;
  }
};
struct cs_sweep_plan {
  std::unique_ptr<SweepCtx> ctx;
};

namespace {

thread_local std::string t_error;

template <typename F>
int guarded(F&& f) {  // capi.cpp:39-52: exceptions -> status + message
  try {
    t_error.clear();
    f();
    return CS_OK;
  } catch (const Failure& e) {
    t_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    t_error = e.what();
    return CS_ERR_INTERNAL;
  }
}

void need(const void* p, const char* what) {
  if (!p) fail(kValidation, std::string("null argument: ") + what);
}

char* dup(const std::string& s) {
  char* out = new char[s.size() + 1];
  std::memcpy(out, s.c_str(), s.size() + 1);
  return out;
}

// Closed-form plan of (graph, oracle, gating/noise), kept on the graph
// handle: handles are immutable, so repeated sweeps/simulations reuse it.
std::shared_ptr<SweepCtx> cached_sweep(const cs_graph* g, const cs_oracle* o, const Policy& p) {
  auto* gm = const_cast<cs_graph*>(g);
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  std::lock_guard<std::mutex> lock(gm->mu);
  cs_graph::Cached& c = gm->sweep[dev];
  if (c.ctx && c.oracle == o->id && c.gated == p.gated && c.noise == p.noise) return c.ctx;
  std::shared_ptr<SweepCtx> ctx = make_sweep(g->g, o->o, p);
  c = {ctx, o->id, p.gated, p.noise};
  return ctx;
}

// Per-call device buffer from the stream-ordered pool (legacy stream, like
// the kernels these calls launch); freed on every exit path.
struct DevPtr {
  void* p = nullptr;
  DevPtr() = default;
  DevPtr(const DevPtr&) = delete;
  DevPtr& operator=(const DevPtr&) = delete;
  ~DevPtr() {
    if (p) cudaFreeAsync(p, 0);
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

Policy policy_of(const cs_sim_policy* p) {  // capi.cpp:64-73 defaults
  Policy q;
  if (p) {
    q.gated = p->counter_gate != 0;
    q.choice_seed = p->choice_seed;
    q.noise = p->reorder_noise;
  }
  return q;
}

}  // namespace

#pragma GCC visibility push(default)
extern "C" {

int cs_graph_parse(const char* json_text, cs_graph** out) {
  return guarded([&] {
    need(json_text, "json_text");
    need(out, "out");
    *out = new cs_graph{Graph::parse(json_text)};
  });
}

int cs_graph_serialize(const cs_graph* g, char** out_json) {
  return guarded([&] {
    need(g, "graph");
    need(out_json, "out_json");
    *out_json = dup(g->g->serialize());
  });
}

int cs_graph_generate(const char* shape, int layers, int params_per_layer,
                      const char* comm_comp_ratio, uint64_t seed, cs_graph** out) {
  return guarded([&] {
    need(shape, "shape");
    need(comm_comp_ratio, "comm_comp_ratio");
    need(out, "out");
    *out = new cs_graph{generate_synthetic(shape, layers, params_per_layer, comm_comp_ratio, seed)};
  });
}

int cs_graph_expand(const cs_graph* worker, int n_workers, int n_ps, int64_t ps_op_time_us,
                    cs_graph** out) {
  return guarded([&] {
    need(worker, "worker");
    need(out, "out");
    *out = new cs_graph{expand_mr(*worker->g, n_workers, n_ps, ps_op_time_us)};
  });
}

int cs_graph_name(const cs_graph* g, char** out) {
  return guarded([&] {
    need(g, "graph");
    need(out, "out");
    *out = dup(g->g->name());
  });
}

int cs_graph_op_count(const cs_graph* g, int64_t* out) {
  return guarded([&] {
    need(g, "graph");
    need(out, "out");
    *out = g->g->n();
  });
}

int cs_graph_edge_count(const cs_graph* g, int64_t* out) {
  return guarded([&] {
    need(g, "graph");
    need(out, "out");
    *out = static_cast<int64_t>(g->g->edges().size());
  });
}

int cs_graph_recv_count(const cs_graph* g, int64_t* out) {
  return guarded([&] {
    need(g, "graph");
    need(out, "out");
    *out = static_cast<int64_t>(g->g->recv_ops().size());
  });
}

int cs_graph_is_cluster(const cs_graph* g, int* out) {
  return guarded([&] {
    need(g, "graph");
    need(out, "out");
    *out = g->g->cluster() ? 1 : 0;
  });
}

int cs_graph_topo_order(const cs_graph* g, char** out_json) {
  return guarded([&] {
    need(g, "graph");
    need(out_json, "out_json");
    *out_json = dup(dump_doc(Json(g->g->topo_order())));
  });
}

int cs_graph_worker_devices(const cs_graph* g, char** out_json) {
  return guarded([&] {
    need(g, "graph");
    need(out_json, "out_json");
    *out_json = dup(dump_doc(Json(g->g->worker_devices())));
  });
}

int cs_graph_worker_partition(const cs_graph* g, const char* device, cs_graph** out) {
  return guarded([&] {
    need(g, "graph");
    need(device, "device");
    need(out, "out");
    *out = new cs_graph{g->g->partition(device)};
  });
}

void cs_graph_free(cs_graph* g) { delete g; }

int cs_oracle_declared(const cs_graph* g, cs_oracle** out) {
  return guarded([&] {
    need(g, "graph");
    need(out, "out");
    *out = new cs_oracle{TimeOracle::declared(g->g)};
  });
}

int cs_oracle_general(const cs_graph* g, cs_oracle** out) {
  return guarded([&] {
    need(g, "graph");
    need(out, "out");
    *out = new cs_oracle{TimeOracle::general(g->g)};
  });
}

int cs_oracle_from_traces(const cs_graph* g, const char* trace_jsonl, cs_oracle** out) {
  return guarded([&] {
    need(g, "graph");
    need(trace_jsonl, "trace_jsonl");
    need(out, "out");
    *out = new cs_oracle{TimeOracle::traces(g->g, trace_jsonl)};
  });
}

int cs_oracle_bandwidth(const cs_graph* g, int64_t bytes_per_us, cs_oracle** out) {
  return guarded([&] {
    need(g, "graph");
    need(out, "out");
    *out = new cs_oracle{TimeOracle::bandwidth(g->g, bytes_per_us)};
  });
}

int cs_oracle_json(const cs_oracle* o, char** out_json) {
  return guarded([&] {
    need(o, "oracle");
    need(out_json, "out_json");
    *out_json = dup(dump_doc(o->o.to_json()));
  });
}

void cs_oracle_free(cs_oracle* o) { delete o; }

int cs_properties_json(const cs_graph* g, const cs_oracle* o, const char* mode, char** out_json) {
  return guarded([&] {
    need(g, "graph");
    need(o, "oracle");
    need(mode, "mode");
    need(out_json, "out_json");
    const PropMode m = prop_mode(mode);
    *out_json = dup(dump_doc(properties_json(*g->g, o->o, m)));
  });
}

int cs_schedule_tic(const cs_graph* g, const char* mode, cs_schedule** out) {
  return guarded([&] {
    need(g, "graph");
    need(mode, "mode");
    need(out, "out");
    *out = new cs_schedule{schedule_for(*g->g, "tic", prop_mode(mode), 0, nullptr)};
  });
}

int cs_schedule_tac(const cs_graph* g, const cs_oracle* o, cs_schedule** out) {
  return guarded([&] {
    need(g, "graph");
    need(o, "oracle");
    need(out, "out");
    *out = new cs_schedule{schedule_for(*g->g, "tac", PropMode::Amended, 0, &o->o)};
  });
}

int cs_schedule_random(const cs_graph* g, uint64_t seed, cs_schedule** out) {
  return guarded([&] {
    need(g, "graph");
    need(out, "out");
    *out = new cs_schedule{schedule_for(*g->g, "random", PropMode::Amended, seed, nullptr)};
  });
}

int cs_schedule_parse(const char* json_text, cs_schedule** out) {
  return guarded([&] {
    need(json_text, "json_text");
    need(out, "out");
    *out = new cs_schedule{Schedule::parse(json_text)};
  });
}

int cs_schedule_serialize(const cs_schedule* s, char** out_json) {
  return guarded([&] {
    need(s, "schedule");
    need(out_json, "out_json");
    *out_json = dup(s->s.serialize());
  });
}

int cs_schedule_total_order(const cs_schedule* s, int* out) {
  return guarded([&] {
    need(s, "schedule");
    need(out, "out");
    *out = s->s.total ? 1 : 0;
  });
}

void cs_schedule_free(cs_schedule* s) { delete s; }

int cs_simulate(const cs_graph* g, const cs_oracle* o, const cs_schedule* s,
                const cs_sim_policy* policy, cs_report** out) {
  return guarded([&] {
    need(g, "graph");
    need(o, "oracle");
    need(out, "out");
    const Policy p = policy_of(policy);
    SimInputs in = prepare_sim(*g->g, o->o, s ? &s->s : nullptr, p);  // reference checks, same order
    auto rep = std::make_unique<cs_report>();
    rep->g = g->g;
    rep->pol = p;
    std::shared_ptr<SweepCtx> ctx;
    bool closed = !g->g->cluster() && in.all_recvs_prioritized;
    if (closed && !p.gated) {  // ungated: only distinct priorities avoid channel draws
      std::vector<int32_t> pr;
      for (int32_t r : g->g->recv_ops()) pr.push_back(in.prio[r]);
      std::sort(pr.begin(), pr.end());
      closed = std::adjacent_find(pr.begin(), pr.end()) == pr.end();
    }
    if (closed) ctx = cached_sweep(g, o, p);
    if (ctx && ctx->fast && !ctx->cluster && ctx->nch == 1) {
      // Closed form: the gate order is the recvs sorted by
      // (priority, id) (sim.cpp:95-104), then the reorder-noise swaps; recvs
      // are roots, so the violations are the swaps (A.4) and nothing is
      // force-released.
      const auto& ro = g->g->recv_ops();
      std::vector<int32_t> order(ro.size());
      for (size_t c = 0; c < ro.size(); ++c) order[c] = static_cast<int32_t>(c);
      std::stable_sort(order.begin(), order.end(),
                       [&](int32_t a, int32_t b) { return in.prio[ro[a]] < in.prio[ro[b]]; });
      rep->violations = apply_gate_noise(order, p);
      rep->makespan = ctx->order_makespan(order);
      rep->d = std::move(in.d);
      rep->prio = std::move(in.prio);
    } else {
      rep->full = std::make_unique<Report>(simulate_prepared(*g->g, in.d, in.prio, p));
      rep->makespan = rep->full->makespan;
      rep->violations = rep->full->violations;
      rep->has_stats = rep->full->has_stats;
    }
    *out = rep.release();
  });
}

int cs_report_makespan(const cs_report* r, int64_t* out_us) {
  return guarded([&] {
    need(r, "report");
    need(out_us, "out_us");
    *out_us = r->makespan;
  });
}

int cs_report_violations(const cs_report* r, int64_t* out) {
  return guarded([&] {
    need(r, "report");
    need(out, "out");
    *out = r->violations;
  });
}

int cs_report_json(const cs_report* r, char** out_json) {
  return guarded([&] {
    need(r, "report");
    need(out_json, "out_json");
    const Report& rep = r->report();
    const auto t0 = std::chrono::steady_clock::now();
    *out_json = dup(rep.json_text());
    if (std::getenv("TICTAC_EVENT_TRACE"))
      std::fprintf(stderr, "[cs_report_json] text %.3f ms\n",
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  });
}

int cs_report_chrome_trace(const cs_report* r, char** out_json) {
  return guarded([&] {
    need(r, "report");
    need(out_json, "out_json");
    *out_json = dup(r->report().chrome_trace_text());
  });
}

int cs_report_iteration_json(const cs_report* r, char** out_json) {
  return guarded([&] {
    need(r, "report");
    need(out_json, "out_json");
    if (!r->has_stats) fail(kValidation, "iteration stats need a cluster simulation");
    *out_json = dup(dump_doc(r->report().iteration_json()));
  });
}

void cs_report_free(cs_report* r) { delete r; }

int cs_makespan_bounds(const cs_graph* g, const cs_oracle* o, int64_t* upper_us, int64_t* lower_us) {
  return guarded([&] {
    need(g, "graph");
    need(o, "oracle");
    need(upper_us, "upper_us");
    need(lower_us, "lower_us");
    const auto b = bounds(*g->g, o->o);
    *upper_us = b.first;
    *lower_us = b.second;
  });
}

int cs_metrics_json(const cs_graph* g, const cs_oracle* o, const cs_report* r, char** out_json) {
  return guarded([&] {
    need(g, "graph");
    need(o, "oracle");
    need(r, "report");
    need(out_json, "out_json");
    const auto b = bounds(*g->g, o->o);
    *out_json = dup(dump_doc(metrics_json(b.first, b.second, r->makespan, r->has_stats ? &r->report() : nullptr)));
  });
}

int cs_brute_force(const cs_graph* g, const cs_oracle* o, const cs_sim_policy* policy, int max_recvs,
                   char** out_json) {
  return guarded([&] {
    need(g, "graph");
    need(o, "oracle");
    need(out_json, "out_json");
    const Graph& G = *g->g;
    const Policy p = policy_of(policy);
    const int64_t R = static_cast<int64_t>(G.recv_ops().size());
    if (R > max_recvs)  // metrics.cpp:40-43, checked before anything else
      fail(kParameter, "brute force refused: " + std::to_string(R) + " recv ops exceed " +
                           std::to_string(max_recvs));
    Policy gp = p;
    gp.gated = true;  // metrics.cpp:45-46
    if (!G.cluster() && p.noise == 0.0 && R >= 1 && R <= 20) {
      std::shared_ptr<SweepCtx> ctx = cached_sweep(g, o, gp);  // coverage/noise checks as simulate()
      if (ctx->fast && !ctx->cluster && !ctx->noisy && ctx->nch == 1) {
        int64_t perms = 1;
        for (int64_t k = 2; k <= R; ++k) perms *= k;
        int64_t best_m = 0, best_k = 0, nd = 0;
        std::vector<int64_t> dist(1 << 16);
        char err[256] = {0};
        if (csk_brute_force_closed(ctx->plan, perms, &best_m, &best_k, dist.data(),
                                   static_cast<int64_t>(dist.size()), &nd, err))
          fail(kInternal, err);
        if (nd > static_cast<int64_t>(dist.size())) {
          dist.resize(static_cast<size_t>(nd));
          if (csk_brute_force_closed(ctx->plan, perms, &best_m, &best_k, dist.data(), nd, &nd, err))
            fail(kInternal, err);
        }
        dist.resize(static_cast<size_t>(nd));
        std::vector<std::string> pool = G.recv_ids(), order;  // unrank best_k
        int64_t rem = best_k, f = perms;
        for (int64_t k = R; k >= 1; --k) {
          f /= k;
          order.push_back(pool[static_cast<size_t>(rem / f)]);
          pool.erase(pool.begin() + rem / f);
          rem %= f;
        }
        Json j;
        j["order"] = order;
        j["makespan_us"] = best_m;
        j["distribution"] = dist;
        *out_json = dup(dump_doc(j));
        return;
      }
    }
    *out_json = dup(dump_doc(brute_force(G, o->o, p, max_recvs)));
  });
}

const char* cs_last_error(void) { return t_error.c_str(); }

void cs_string_free(char* s) { delete[] s; }

const char* cs_version(void) { return "0.1.0"; }

// ---------------------------------------------------------------------------
// Batched extensions

int cs_sweep_random(const cs_graph* g, const cs_oracle* o, uint64_t seed_lo, int64_t count,
                    const cs_sim_policy* policy, int64_t* makespans_out, int64_t* worker_makespans_out,
                    cs_sweep_stats* stats_out) {
  return guarded([&] {
    need(g, "graph");
    need(o, "oracle");
    if (count < 0) fail(kParameter, "count must be non-negative");
    Policy p = policy_of(policy);
    const auto t0 = std::chrono::steady_clock::now();
    std::shared_ptr<SweepCtx> ctx = cached_sweep(g, o, p);
    if (!ctx->fast) {
      const auto t1 = std::chrono::steady_clock::now();
      sweep_exact(*ctx, seed_lo, count, makespans_out, worker_makespans_out, stats_out);
      if (std::getenv("TICTAC_EVENT_TRACE")) {
        const auto t2 = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[cs_sweep_random] ctx %.3f ms, exact sweep %.3f ms\n",
                     std::chrono::duration<double, std::milli>(t1 - t0).count(),
                     std::chrono::duration<double, std::milli>(t2 - t1).count());
      }
      return;
    }
    const cs_sweep_stats total = sweep_fast({ctx.get()}, seed_lo, count, makespans_out, worker_makespans_out,
                                            nullptr);
    if (stats_out) *stats_out = total;
  });
}

int cs_sweep_random_multi(const cs_graph* g, const cs_oracle* o, uint64_t seed_lo, int64_t count,
                          const cs_sim_policy* policy, int n_devices, int64_t* makespans_out,
                          int64_t* worker_makespans_out, cs_sweep_stats* stats_out) {
  return guarded([&] {
    need(g, "graph");
    need(o, "oracle");
    if (count < 0) fail(kParameter, "count must be non-negative");
    int avail = 0;
    if (cudaGetDeviceCount(&avail) != cudaSuccess) avail = 0;
    if (n_devices < 1 || n_devices > avail)
      fail(kParameter, "n_devices must be within [1, " + std::to_string(avail) + "]");
    const Policy p = policy_of(policy);
    int caller = 0;
    if (cudaGetDevice(&caller) != cudaSuccess) caller = 0;
    // one plan per device, built on that device (cached on the graph handle)
    std::vector<std::shared_ptr<SweepCtx>> ctx(n_devices);
    std::vector<std::string> errors(n_devices);
    {
      std::vector<std::thread> th;
      for (int d = 0; d < n_devices; ++d)
        th.emplace_back([&, d] {
          try {
            if (cudaSetDevice(d) != cudaSuccess) fail(kInternal, "cudaSetDevice failed");
            ctx[d] = cached_sweep(g, o, p);
          } catch (const std::exception& e) {
            errors[d] = e.what();
          }
        });
      for (auto& t : th) t.join();
    }
    for (const auto& e : errors)
      if (!e.empty()) fail(kInternal, e);
    const int64_t W = ctx[0]->cluster ? static_cast<int64_t>(ctx[0]->workers.size()) : 1;
    if (!ctx[0]->fast) {
      // exact replica: contiguous shards, one host thread per device, host merge
      std::vector<cs_sweep_stats> parts(n_devices);
      const int64_t per = (count + n_devices - 1) / n_devices;
      std::vector<std::thread> th;
      for (int d = 0; d < n_devices; ++d)
        th.emplace_back([&, d] {
          try {
            if (cudaSetDevice(d) != cudaSuccess) fail(kInternal, "cudaSetDevice failed");
            const int64_t off = std::min<int64_t>(count, d * per), n = std::min<int64_t>(per, count - off);
            sweep_exact(*ctx[d], seed_lo + static_cast<uint64_t>(off), n, makespans_out ? makespans_out + off : nullptr,
                        worker_makespans_out && ctx[d]->cluster ? worker_makespans_out + off * W : nullptr, &parts[d]);
          } catch (const std::exception& e) {
            errors[d] = e.what();
          }
        });
      for (auto& t : th) t.join();
      for (const auto& e : errors)
        if (!e.empty()) fail(kInternal, e);
      cs_sweep_stats total{};
      for (int d = 0; d < n_devices; ++d) merge_stats(total, parts[d], d == 0);
      if (stats_out) *stats_out = total;
      return;
    }
    std::vector<SweepCtx*> raw;
    for (auto& c : ctx) raw.push_back(c.get());
    std::unique_lock<std::mutex> hold;
    const DeviceReducer* red = n_devices > 1 ? &nccl_reducer(n_devices, hold) : nullptr;
    const cs_sweep_stats total = sweep_fast(raw, seed_lo, count, makespans_out, worker_makespans_out, red);
    cudaSetDevice(caller);
    if (stats_out) *stats_out = total;
  });
}

int cs_simulate_orders(const cs_graph* g, const cs_oracle* o, const int32_t* orders, int64_t n,
                       const cs_sim_policy* policy, int64_t* makespans_out, int64_t* violations_out) {
  return guarded([&] {
    need(g, "graph");
    need(o, "oracle");
    need(makespans_out, "makespans_out");
    if (n < 0) fail(kParameter, "n must be non-negative");
    if (n > 0) need(orders, "orders");
    const Graph& G = *g->g;
    const int32_t R = static_cast<int32_t>(G.recv_ops().size());
    const Policy p = policy_of(policy);
    auto ctx = make_sweep(g->g, o->o, p);
    if (n == 0) return;
    if (ctx->fast && !ctx->cluster && ctx->nch == 1) {  // rows validated by the kernel as it reads them
      // every row shares the choice seed, hence the same reorder-noise swaps
      // (positions whose noise draw fired, sim.cpp:106-114): applied to each
      // rank-order row they give its gate order; violations = swaps (A.4)
      std::vector<int32_t> pos(R);
      for (int32_t k = 0; k < R; ++k) pos[k] = k;
      const int64_t swaps = apply_gate_noise(pos, p);
      std::vector<int32_t> gated_rows;
      const int32_t* rows = orders;
      if (swaps) {
        gated_rows.resize(static_cast<size_t>(n) * R);
        for (int64_t b = 0; b < n; ++b)
          for (int32_t k = 0; k < R; ++k) gated_rows[b * R + k] = orders[b * R + pos[k]];
        rows = gated_rows.data();
      }
      auto cudacheck = [&](cudaError_t e) {
        if (e != cudaSuccess) fail(kInternal, std::string("CUDA error: ") + cudaGetErrorString(e));
      };
      DevPtr b_o, b_m;
      cudacheck(cudaMallocAsync(&b_o.p, 4 * n * R + 4, 0));
      cudacheck(cudaMallocAsync(&b_m.p, 8 * n, 0));
      cudacheck(cudaMemcpy(b_o.p, rows, 4 * n * R, cudaMemcpyHostToDevice));
      char err[256] = {0};
      const int rc = csk_sweep_orders(ctx->plan, b_o.as<int32_t>(), n, nullptr, b_m.as<int64_t>(), err);
      if (rc) fail(rc == 4 ? kParameter : kInternal, err);
      cudacheck(cudaMemcpy(makespans_out, b_m.p, 8 * n, cudaMemcpyDeviceToHost));
      if (violations_out)
        for (int64_t k = 0; k < n; ++k) violations_out[k] = swaps;
      return;
    }
    {  // every row a permutation of the recv columns (checked as the kernel does)
      std::vector<uint8_t> seen(static_cast<size_t>(R));
      for (int64_t b = 0; b < n; ++b) {
        std::fill(seen.begin(), seen.end(), 0);
        for (int32_t k = 0; k < R; ++k) {
          const int32_t c = orders[b * R + k];
          if (c < 0 || c >= R) fail(kParameter, "order entry out of range");
          if (seen[c]++) fail(kParameter, "order rows must be permutations of the recv columns");
        }
      }
    }
    std::vector<uint64_t> seeds(static_cast<size_t>(n), p.choice_seed);
    std::vector<int64_t> viol(static_cast<size_t>(n));
    std::vector<int32_t> st(static_cast<size_t>(n));
    char err[256] = {0};
    const int64_t chunk = 1 << 20;
    for (int64_t b = 0; b < n; b += chunk) {
      const int32_t B = static_cast<int32_t>(std::min(chunk, n - b));
      if (csk_event_sim(G.device(), ctx->dur.data(), B, nullptr, orders + b * R, R, seeds.data() + b,
                        p.gated ? 1 : 0, p.noise, makespans_out + b, viol.data() + b, st.data() + b,
                        nullptr, nullptr, nullptr, err))
        fail(kInternal, err);
    }
    for (int64_t k = 0; k < n; ++k)
      if (st[k]) fail(kValidation, "simulation stalled with no runnable op");
    if (violations_out) std::memcpy(violations_out, viol.data(), 8 * n);
  });
}

int cs_sweep_plan_create(const cs_graph* g, const cs_oracle* o, const cs_sim_policy* policy,
                         cs_sweep_plan** out) {
  return guarded([&] {
    need(g, "graph");
    need(o, "oracle");
    need(out, "out");
    auto ctx = make_sweep(g->g, o->o, policy_of(policy));
    if (!ctx->fast) fail(kParameter, "closed-form sweep does not apply: " + ctx->why);
    *out = new cs_sweep_plan{std::move(ctx)};
  });
}

int cs_sweep_path_json(const cs_graph* g, const cs_oracle* o, const cs_sim_policy* policy, char** out_json) {
  return guarded([&] {
    need(g, "graph");
    need(o, "oracle");
    need(out_json, "out_json");
    std::shared_ptr<SweepCtx> c = cached_sweep(g, o, policy_of(policy));
    Json j;
    j["path"] = !c->fast ? "event_sim_kernel"
                : c->dag ? "dag_sweep_kernel"
                : c->ps  ? "cluster_ps_kernel"
                         : "chain_sweep_kernel";
    j["why"] = c->fast ? "" : c->why;
    j["kernel"] = c->fast && c->plan ? csk_sweep_plan_kernel(c->plan) : "event_sim_kernel";
    *out_json = dup(dump_doc(j));
  });
}

int cs_sweep_plan_info(const cs_sweep_plan* p, char** out_json) {
  return guarded([&] {
    need(p, "plan");
    need(out_json, "out_json");
    const SweepCtx& c = *p->ctx;
    Json j;
    j["graph"] = c.g->name();
    j["ops"] = c.g->n();
    j["edges"] = static_cast<int64_t>(c.g->edges().size());
    j["recvs_per_worker"] = c.R;
    j["classes"] = c.nc;
    j["kernel"] = csk_sweep_plan_kernel(c.plan);
    if (c.dag) {
      j["joins"] = c.joins;
      j["slots"] = c.slots;
      j["program_records"] = c.prog_words;
    }
    j["workers"] = c.cluster ? static_cast<int64_t>(c.workers.size()) : 1;
    int64_t erecv = 0;
    for (int32_t r : c.g->recv_ops()) erecv += c.g->nsucc(r);
    j["recv_edges"] = erecv;
    j["U_us"] = c.U;
    j["L_us"] = c.L;
    j["cluster"] = c.cluster;
    j["key_bits"] = csk_key_bits(c.U);
    j["uploaded_bytes"] = csk_sweep_plan_uploaded(c.plan);
    *out_json = dup(dump_doc(j));
  });
}

int cs_sweep_plan_reset(const cs_sweep_plan* p, void* stream, int64_t* d_stats_i64, double* d_stats_f64) {
  return guarded([&] {
    need(p, "plan");
    need(d_stats_i64, "d_stats_i64");
    need(d_stats_f64, "d_stats_f64");
    char err[256] = {0};
    if (csk_sweep_reset(p->ctx->plan, stream, d_stats_i64, d_stats_f64, err)) fail(kInternal, err);
  });
}

int cs_sweep_plan_run(const cs_sweep_plan* p, uint64_t seed_lo, int64_t count, uint64_t key_base,
                      void* stream, int64_t* d_makespans, int64_t* d_stats_i64, double* d_stats_f64) {
  return guarded([&] {
    need(p, "plan");
    need(d_stats_i64, "d_stats_i64");
    need(d_stats_f64, "d_stats_f64");
    if (count < 0) fail(kParameter, "count must be non-negative");
    const int kb = csk_key_bits(p->ctx->U);
    if (seed_lo < key_base || seed_lo - key_base + static_cast<uint64_t>(count) > (uint64_t{1} << kb))
      fail(kParameter, "seed - key_base must stay below 2^" + std::to_string(kb));
    char err[256] = {0};
    if (csk_sweep_run(p->ctx->plan, seed_lo, count, key_base, stream, d_makespans, nullptr, d_stats_i64,
                      d_stats_f64, err))
      fail(kInternal, err);
  });
}

int cs_sweep_stats_finish(const cs_sweep_plan* p, const int64_t* h_stats_i64, const double* h_stats_f64,
                          uint64_t key_base, cs_sweep_stats* out) {
  return guarded([&] {
    need(p, "plan");
    need(h_stats_i64, "h_stats_i64");
    need(h_stats_f64, "h_stats_f64");
    need(out, "out");
    finish_stats(*p->ctx, h_stats_i64, h_stats_f64, key_base, out);
  });
}

int cs_sweep_stats_pack(const int64_t* d_stats_i64, const double* d_stats_f64, int rank, int world,
                        int64_t* d_packed, void* stream) {
  return guarded([&] {
    need(d_stats_i64, "d_stats_i64");
    need(d_stats_f64, "d_stats_f64");
    need(d_packed, "d_packed");
    if (world < 1 || rank < 0 || rank >= world) fail(kParameter, "rank must be within [0, world)");
    char err[256] = {0};
    if (csk_stats_pack(d_stats_i64, d_stats_f64, rank, world, d_packed, stream, err)) fail(kInternal, err);
  });
}

int cs_sweep_stats_unpack(const int64_t* d_packed, int world, int64_t* d_stats_i64, double* d_stats_f64,
                          void* stream) {
  return guarded([&] {
    need(d_packed, "d_packed");
    need(d_stats_i64, "d_stats_i64");
    need(d_stats_f64, "d_stats_f64");
    if (world < 1) fail(kParameter, "world must be positive");
    char err[256] = {0};
    if (csk_stats_unpack(d_packed, world, d_stats_i64, d_stats_f64, stream, err)) fail(kInternal, err);
  });
}

void cs_sweep_plan_free(cs_sweep_plan* p) { delete p; }

int cs_graph_generate_model(const char* model, uint64_t seed, cs_graph** out) {
  return guarded([&] {
    need(model, "model");
    need(out, "out");
    *out = new cs_graph{generate_model(model, seed)};
  });
}

int cs_tac_traffic(const cs_graph* g, const cs_oracle* o, int64_t* out, int n_out) {
  return guarded([&] {
    need(g, "graph");
    need(o, "oracle");
    need(out, "out");
    if (n_out < 7) fail(kParameter, "n_out must be at least 7");
    const Graph& G = *g->g;
    const std::vector<int64_t> d = o->o.durations(G);
    char err[256] = {0};
    if (csk_tac_stats(G.device(), d.data(), out, err)) fail(kInternal, err);
  });
}

int64_t cs_device_launches(void) { return csk_launches(); }

}  // extern "C"
#pragma GCC visibility pop
