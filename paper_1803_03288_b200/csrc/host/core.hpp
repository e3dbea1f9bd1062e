// Host-side data model of the drop-in library: graphs, oracles, schedules,
// reports. Host code parses, validates and formats; all scheduling and
// simulation arithmetic runs on the device (../device/csk.h).
//
// Behaviour follows the reference (file:line cited per function) so that
// every JSON artifact, status code and message is byte-identical.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <unordered_map>
#include <utility>
#include <vector>

#include "json.hpp"

struct DeviceGraph;  // device/csk.h

namespace tictac {

// Status codes double as reference exit codes (errors.hpp:11-17). Domain
// errors surface as 2 (errors.hpp:26-30).
enum Code : int { kInternal = 1, kValidation = 2, kCoverage = 3, kParameter = 4, kIo = 5 };

struct Failure : std::runtime_error {
  int code;
  Failure(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& msg) { throw Failure(code, msg); }

using Json = nlohmann::ordered_json;  // byte-stable key order (json_io.hpp:14)
Json parse_doc(std::string_view text, std::string_view what);
inline std::string dump_doc(const Json& j) { return j.dump(2) + "\n"; }

enum OpKind : int8_t { kCompute = 0, kRecv = 1, kSend = 2, kPsAggregate = 3, kPsRead = 4, kPsUpdate = 5 };
const char* kind_str(OpKind k);
inline bool transfer(OpKind k) { return k == kRecv || k == kSend; }

struct Resource {
  std::string device;
  bool channel = false;  // unit: Compute < Channel (graph.hpp:36-40)
  std::string name;
  std::string key() const { return device + (channel ? "/channel/" : "/compute/") + name; }
  bool operator==(const Resource& o) const {
    return channel == o.channel && device == o.device && name == o.name;
  }
  bool operator<(const Resource& o) const {
    if (device != o.device) return device < o.device;
    if (channel != o.channel) return !channel;
    return name < o.name;
  }
};

struct Op {
  std::string id;
  OpKind kind = kCompute;
  Resource res;
  std::optional<int64_t> time_us, bytes;
  bool operator==(const Op& o) const {
    return id == o.id && kind == o.kind && res == o.res && time_us == o.time_us && bytes == o.bytes;
  }
};

// Immutable DAG in the reference index model: ops sorted by id (byte
// order), edges sorted/deduped, CSR adjacency with ascending lists.
class Graph : public std::enable_shared_from_this<Graph> {
 public:
  static std::shared_ptr<Graph> make(std::string name, bool cluster, std::vector<Op> ops,
                                     std::vector<std::pair<std::string, std::string>> edges);
  static std::shared_ptr<Graph> parse(std::string_view text);
  std::string serialize() const;

  const std::string& name() const { return name_; }
  bool cluster() const { return cluster_; }
  int32_t n() const { return static_cast<int32_t>(ops_.size()); }
  const std::vector<Op>& ops() const { return ops_; }
  const std::vector<std::pair<std::string, std::string>>& edges() const { return edges_; }
  bool has(const std::string& id) const { return index_.count(id) != 0; }
  int32_t at(const std::string& id) const;  // throws Domain (-> 2) "unknown op: "

  const std::vector<int32_t>& pred_off() const { return pred_off_; }
  const std::vector<int32_t>& pred_idx() const { return pred_idx_; }
  const std::vector<int32_t>& succ_off() const { return succ_off_; }
  const std::vector<int32_t>& succ_idx() const { return succ_idx_; }
  int32_t npred(int32_t v) const { return pred_off_[v + 1] - pred_off_[v]; }
  int32_t nsucc(int32_t v) const { return succ_off_[v + 1] - succ_off_[v]; }

  const std::vector<Resource>& resources() const { return resources_; }  // unique, sorted
  const std::vector<int32_t>& res_of() const { return res_of_; }        // per op
  const std::vector<int32_t>& recv_ops() const { return recv_ops_; }    // ascending
  std::vector<std::string> recv_ids() const;
  std::vector<std::string> topo_order() const;  // graph.cpp:158-185
  std::vector<std::string> worker_devices() const;  // sim.cpp:27-41
  std::shared_ptr<Graph> partition(const std::string& device) const;  // sim.cpp:43-59

  // Lazily uploaded device copy of the structure (thread-safe).
  DeviceGraph* device() const;
  ~Graph();

  // Per-graph memo of derived, duration-independent analyses (thread-safe;
  // the graph is immutable, so an entry never goes stale).
  template <class T, class F>
  std::shared_ptr<const T> memo(const std::string& key, F&& make) const {
    std::lock_guard<std::mutex> lock(aux_mu_);
    auto it = aux_.find(key);
    if (it != aux_.end()) return std::static_pointer_cast<const T>(it->second);
    std::shared_ptr<const T> v = std::make_shared<const T>(make());
    aux_.emplace(key, v);
    return v;
  }

 private:
  void index_and_validate();
  std::string name_;
  bool cluster_ = false;
  std::vector<Op> ops_;
  std::vector<std::pair<std::string, std::string>> edges_;
  std::unordered_map<std::string, int32_t> index_;
  std::vector<int32_t> pred_off_, pred_idx_, succ_off_, succ_idx_;
  std::vector<Resource> resources_;
  std::vector<int32_t> res_of_, recv_ops_;
  mutable std::mutex dev_mu_;
  mutable std::map<int, DeviceGraph*> dev_;  // per CUDA device (multi-GPU sweeps)
  mutable std::mutex aux_mu_;
  mutable std::map<std::string, std::shared_ptr<const void>> aux_;
};

// Total map op id -> microseconds (time_oracle.hpp:28-58).
// The reference keeps an id -> µs map (time_oracle.hpp:28-58). Every oracle
// is built from one graph and covers exactly its ops, so here it keeps that
// graph and the values by its op index (= id order): durations() for the same
// graph is a copy, for another graph one merge walk over the two id-ordered
// op lists, and to_json iterates in the map's order without building it.
struct TimeOracle {
  std::shared_ptr<const Graph> src;
  std::vector<int64_t> us;  // by src op index
  std::string origin;       // measured | declared | general | synthetic
  static TimeOracle declared(std::shared_ptr<const Graph> g);
  static TimeOracle general(std::shared_ptr<const Graph> g);
  static TimeOracle traces(std::shared_ptr<const Graph> g, std::string_view jsonl);
  static TimeOracle bandwidth(std::shared_ptr<const Graph> g, int64_t bytes_per_us);
  // check_covers (time_oracle.cpp:143-149), then durations by op index.
  std::vector<int64_t> durations(const Graph& g) const;
  Json to_json() const;
};

struct Schedule {
  std::string graph;
  std::string algorithm;  // tic | tac | random
  std::map<std::string, int> prio;
  bool total = false;
  std::string serialize() const;            // schedule.cpp:86-93
  static Schedule parse(std::string_view);  // schedule.cpp:95-123
};

struct Policy {
  bool gated = true;
  uint64_t choice_seed = 0;
  double noise = 0.0;
};

struct Report {
  int64_t makespan = 0, violations = 0;
  std::vector<Resource> resources;
  struct Event { int32_t op; int32_t res; int64_t start, end; };
  std::vector<Event> events;  // sorted (start, resource, op id)
  std::shared_ptr<const Graph> graph;  // op ids by index (kept alive with the report)
  const std::string& op_id(int32_t op) const { return graph->ops()[op].id; }
  bool has_stats = false;
  std::vector<std::pair<std::string, int64_t>> per_worker;  // ascending device
  int64_t iteration = 0, strag_num = 0, strag_den = 1;
  Json to_json() const;       // sim.cpp:305-321
  Json chrome_trace() const;  // sim.cpp:323-366
  // The same documents as dump_doc(to_json()) / dump_doc(chrome_trace()),
  // written directly (one pass, no per-event JSON nodes).
  std::string json_text() const;
  std::string chrome_trace_text() const;
  Json iteration_json() const;  // sim.cpp:368-376
};

// ---- hot-path entry points (host orchestration of device kernels) -------
enum class PropMode { Literal, Amended };
PropMode prop_mode(std::string_view s);  // properties.cpp:15-19
Json properties_json(const Graph& g, const TimeOracle& o, PropMode mode);
Schedule tic(const Graph& g, PropMode mode);
Schedule tac(const Graph& g, const TimeOracle& o);
Schedule random_schedule(const Graph& g, uint64_t seed);
Schedule schedule_for(const Graph& g, const std::string& algo, PropMode mode, uint64_t seed,
                      const TimeOracle* o);  // cluster.cpp:91-122
Report simulate(const Graph& g, const TimeOracle& o, const Schedule* s, const Policy& p);
// simulate() split in two: validation + per-op arrays (sim.cpp:63-88), then
// the exact device event simulation and report assembly.
struct SimInputs {
  std::vector<int64_t> d;
  std::vector<int32_t> prio;
  bool all_recvs_prioritized = false;
};
SimInputs prepare_sim(const Graph& g, const TimeOracle& o, const Schedule* s, const Policy& p);
Report simulate_prepared(const Graph& g, const std::vector<int64_t>& d, const std::vector<int32_t>& prio,
                         const Policy& p);
// One run inside SURVEY A.2's regime (worker graph, one compute unit and one
// channel, gated, noiseless, every recv prioritized and no compute op): the
// specialised device replica (csk_event_a2), same Report as simulate_prepared.
// Gated reorder noise on a single channel's gate sequence (sim.cpp:106-114):
// adjacent swaps at positions 1..n-1 whose draw of the separate stream
// Rng(splitmix64(choice_seed ^ salt)) has unit() < p. Returns the number of
// swaps, which is the run's violation count in SURVEY A.2's regime (A.4:
// each left-to-right swap adds exactly one inversion; recvs are roots, so
// nothing is force-released).
int64_t apply_gate_noise(std::vector<int32_t>& order, const Policy& p);
Report simulate_a2(const Graph& g, const std::vector<int64_t>& d, const std::vector<int32_t>& prio,
                   const Policy& p);
std::pair<int64_t, int64_t> bounds(const Graph& g, const TimeOracle& o);  // metrics.cpp:10-22
Json metrics_json(int64_t U, int64_t L, int64_t m, const Report* stats);
Json brute_force(const Graph& g, const TimeOracle& o, const Policy& p, int max_recvs);

// ---- host-only builders -------------------------------------------------
std::shared_ptr<Graph> expand_mr(const Graph& worker, int n_workers, int n_ps, int64_t ps_us);
std::shared_ptr<Graph> generate_synthetic(const std::string& shape, int layers, int params,
                                          const std::string& ratio, uint64_t seed);
std::shared_ptr<Graph> generate_model(const std::string& model, uint64_t seed);

// Exact rationals (rational.hpp:13-155): int64 num/den via __int128.
struct Rational {
  int64_t num = 0, den = 1;
  Rational() = default;
  Rational(int64_t n, int64_t d);
  static Rational parse(const std::string& text);
};

}  // namespace tictac
