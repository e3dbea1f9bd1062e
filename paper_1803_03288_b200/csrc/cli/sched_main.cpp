// tictac_sched: the reference CLI's batched `sweep` and `bruteforce`
// subcommands (reference tools/sched_main.cpp) as a native client of the C
// ABI only (include/commsched.h), like the reference's own driver (RAII
// handles over the cs_* calls, sched_main.cpp:38-54). The per-seed loop of
// cmd_sweep (sched_main.cpp:452-502) becomes one cs_sweep_random call per
// contiguous run of seeds when the schedule is random.
//
//   tictac_sched sweep --graph g.json --algo random --seeds 1..100000 --out sweep.csv [--gpus N]
//   tictac_sched bruteforce --graph g.json --max-recvs 12 [--out best.json]
//
// Flags as `--name value` or `--name=value`; `--config file.json` supplies
// defaults (JSON keys = flag names, flags win; sched_main.cpp:142-255); seed
// lists `a..b` (fewer than 10^6 seeds) or `a,b,c` (sched_main.cpp:112-140);
// artifacts are written all-or-nothing (sched_main.cpp:65-87); the exit code
// is the status code, errors print "error: <message>" on stderr.
// paper_1803_03288_b200/sched.py is the same driver in Python; the tests run
// both against the reference library's per-seed loop.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include "commsched.h"
#include "json.hpp"

namespace {

using Json = nlohmann::ordered_json;

struct Exit {
  int code;
  std::string message;
};

[[noreturn]] void quit(int code, std::string message) { throw Exit{code, std::move(message)}; }

// cs_* status -> Exit with the library's thread-local message
void check(int rc) {
  if (rc != CS_OK) quit(rc, cs_last_error());
}

template <typename T, void (*Free)(T*)>
struct Handle {
  T* p = nullptr;
  Handle() = default;
  Handle(const Handle&) = delete;
  Handle& operator=(const Handle&) = delete;
  ~Handle() {
    if (p) Free(p);
  }
};
using GraphH = Handle<cs_graph, cs_graph_free>;
using OracleH = Handle<cs_oracle, cs_oracle_free>;
using ScheduleH = Handle<cs_schedule, cs_schedule_free>;
using ReportH = Handle<cs_report, cs_report_free>;

std::string take(char* s) {  // library-owned string -> std::string
  std::string out(s ? s : "");
  cs_string_free(s);
  return out;
}

std::string read_file(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) quit(CS_ERR_IO, "cannot read " + path);
  std::ostringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

// sched_main.cpp:89-101: six places, half away from zero
std::string decimal6(int64_t num, int64_t den) {
  __int128 scaled = static_cast<__int128>(num) * 1000000;
  const bool neg = scaled < 0;
  if (neg) scaled = -scaled;
  __int128 q = scaled / den, r = scaled % den;
  if (2 * r >= den) ++q;
  char buf[64];
  std::snprintf(buf, sizeof buf, "%s%lld.%06lld", neg ? "-" : "", static_cast<long long>(q / 1000000),
                static_cast<long long>(q % 1000000));
  return buf;
}

// std::stoull semantics: leading whitespace and '+' accepted, the whole
// string must be digits, value < 2^64
uint64_t parse_uint(const std::string& s) {
  size_t i = s.find_first_not_of(" \t\n\v\f\r");
  std::string t = i == std::string::npos ? "" : s.substr(i);
  if (!t.empty() && t[0] == '+') t = t.substr(1);
  bool ok = !t.empty();
  unsigned __int128 v = 0;
  for (char c : t) {
    if (c < '0' || c > '9') {
      ok = false;
      break;
    }
    v = v * 10 + static_cast<unsigned>(c - '0');
    if (v >> 64) {
      ok = false;
      break;
    }
  }
  if (!ok) quit(CS_ERR_PARAMETER, "bad seed value: " + s);
  return static_cast<uint64_t>(v);
}

std::vector<uint64_t> parse_seeds(const std::string& text) {
  std::vector<uint64_t> seeds;
  const size_t dots = text.find("..");
  if (dots != std::string::npos) {
    const uint64_t lo = parse_uint(text.substr(0, dots)), hi = parse_uint(text.substr(dots + 2));
    if (hi < lo) quit(CS_ERR_PARAMETER, "seed range is empty: " + text);
    if (hi - lo >= 1000000) quit(CS_ERR_PARAMETER, "seed range too large: " + text);
    for (uint64_t s = lo;; ++s) {
      seeds.push_back(s);
      if (s == hi) break;
    }
    return seeds;
  }
  size_t pos = 0;
  while (pos <= text.size()) {
    size_t comma = text.find(',', pos);
    if (comma == std::string::npos) comma = text.size();
    if (comma > pos) seeds.push_back(parse_uint(text.substr(pos, comma - pos)));
    pos = comma + 1;
  }
  if (seeds.empty()) quit(CS_ERR_PARAMETER, "no seeds in: " + text);
  return seeds;
}

// all-or-nothing artifact writes (sched_main.cpp:65-87)
struct Artifacts {
  std::vector<std::pair<std::string, std::string>> files;
  void add(const std::string& path, std::string content) {
    if (!path.empty()) files.emplace_back(path, std::move(content));
  }
  void commit() {
    std::vector<std::string> written;
    for (const auto& [path, content] : files) {
      std::ofstream f(path, std::ios::binary | std::ios::trunc);
      if (f) f.write(content.data(), static_cast<std::streamsize>(content.size()));
      if (!f) {
        for (const auto& w : written) std::remove(w.c_str());
        std::remove(path.c_str());
        quit(CS_ERR_IO, "cannot write " + path);
      }
      written.push_back(path);
    }
  }
};

enum class Type { Str, Int, Float };
struct Flag {
  const char* name;  // flag spelling without "--"
  const char* key;   // config-file key
  Type type;
  const char* dflt;  // nullptr: no default (choice-seed falls back to --seed)
};
const Flag kFlags[] = {
    {"graph", "graph", Type::Str, ""},          {"oracle", "oracle", Type::Str, "declared"},
    {"traces", "traces", Type::Str, ""},        {"bandwidth", "bandwidth", Type::Int, "0"},
    {"algo", "algo", Type::Str, "none"},        {"mode", "mode", Type::Str, "amended"},
    {"seed", "seed", Type::Int, "0"},           {"schedule", "schedule", Type::Str, ""},
    {"enforce", "enforce", Type::Str, "counter"}, {"noise", "noise", Type::Float, "0"},
    {"choice-seed", "choice-seed", Type::Int, nullptr}, {"seeds", "seeds", Type::Str, ""},
    {"out", "out", Type::Str, ""},              {"max-recvs", "max-recvs", Type::Int, "8"},
    {"gpus", "gpus", Type::Int, "1"},
};
bool sweep_only(const std::string& f) {
  return f == "seeds" || f == "algo" || f == "mode" || f == "seed" || f == "schedule" || f == "choice-seed" ||
         f == "gpus";
}

struct Options {
  std::string cmd;
  std::map<std::string, std::string> v;  // resolved values as text
  const std::string& s(const char* k) const { return v.at(k); }
  int64_t i(const char* k) const { return std::stoll(v.at(k)); }
  bool has(const char* k) const { return v.count(k) != 0; }
};

void check_type(const Flag& f, const std::string& text) {
  try {
    size_t used = 0;
    if (f.type == Type::Int) (void)std::stoll(text, &used);
    else if (f.type == Type::Float) (void)std::stod(text, &used);
    else return;
    if (used != text.size()) throw std::invalid_argument(text);
  } catch (const std::exception&) {
    quit(CS_ERR_PARAMETER, std::string("--") + f.name + ": invalid value '" + text + "'");
  }
}

Options options(int argc, char** argv) {
  if (argc < 2 || (std::strcmp(argv[1], "sweep") != 0 && std::strcmp(argv[1], "bruteforce") != 0))
    quit(CS_ERR_PARAMETER, "usage: tictac_sched {sweep|bruteforce} [--flag value ...]");
  Options o;
  o.cmd = argv[1];
  std::map<std::string, std::string> given;
  std::string config;
  for (int a = 2; a < argc; ++a) {
    std::string arg = argv[a];
    if (arg.rfind("--", 0) != 0) quit(CS_ERR_PARAMETER, "unexpected argument: " + arg);
    std::string name = arg.substr(2), value;
    const size_t eq = name.find('=');
    if (eq != std::string::npos) {
      value = name.substr(eq + 1);
      name = name.substr(0, eq);
    } else {
      if (a + 1 >= argc) quit(CS_ERR_PARAMETER, "--" + name + " needs a value");
      value = argv[++a];
    }
    if (name == "config") {
      config = value;
      continue;
    }
    const Flag* f = nullptr;
    for (const Flag& k : kFlags)
      if (name == k.name && !(o.cmd == "bruteforce" && sweep_only(name))) f = &k;
    if (!f) quit(CS_ERR_PARAMETER, "unknown option: --" + name);
    check_type(*f, value);
    given[name] = value;
  }
  Json cfg = Json::object();
  if (!config.empty()) {
    try {
      cfg = Json::parse(read_file(config));
    } catch (const Json::parse_error& e) {
      quit(CS_ERR_VALIDATION, std::string("config: ") + e.what());
    }
    if (!cfg.is_object()) quit(CS_ERR_VALIDATION, "config must be a JSON object");
  }
  for (const Flag& f : kFlags) {
    auto it = given.find(f.name);
    if (it != given.end()) {  // flags win over the config file
      o.v[f.name] = it->second;
    } else if (!(o.cmd == "bruteforce" && sweep_only(f.name)) && cfg.contains(f.key)) {
      const Json& j = cfg[f.key];
      std::string text;
      if (j.is_string()) text = j.get<std::string>();
      else if (j.is_number_integer()) text = std::to_string(j.get<int64_t>());
      else if (j.is_number()) text = f.type == Type::Int ? std::to_string(static_cast<int64_t>(j.get<double>()))
                                                         : j.dump();
      else quit(CS_ERR_VALIDATION, std::string("config: bad value for ") + f.key);
      check_type(f, text);
      o.v[f.name] = text;
    } else if (f.dflt) {
      o.v[f.name] = f.dflt;
    }
  }
  return o;
}

void load(const Options& o, GraphH& g, OracleH& oracle) {
  if (o.s("graph").empty()) quit(CS_ERR_PARAMETER, "--graph is required");
  check(cs_graph_parse(read_file(o.s("graph")).c_str(), &g.p));
  const std::string& src = o.s("oracle");
  if (src == "declared") {
    check(cs_oracle_declared(g.p, &oracle.p));
  } else if (src == "general") {
    check(cs_oracle_general(g.p, &oracle.p));
  } else if (src == "traces") {
    if (o.s("traces").empty()) quit(CS_ERR_PARAMETER, "--oracle traces needs --traces");
    check(cs_oracle_from_traces(g.p, read_file(o.s("traces")).c_str(), &oracle.p));
  } else if (src == "bandwidth") {
    if (o.i("bandwidth") <= 0) quit(CS_ERR_PARAMETER, "--oracle bandwidth needs --bandwidth > 0");
    check(cs_oracle_bandwidth(g.p, o.i("bandwidth"), &oracle.p));
  } else {
    quit(CS_ERR_PARAMETER, "unknown oracle source: " + src);
  }
}

cs_sim_policy make_policy(const Options& o) {
  const std::string& e = o.s("enforce");
  if (e != "counter" && e != "none") quit(CS_ERR_PARAMETER, "unknown enforcement: " + e);
  cs_sim_policy p{};
  p.counter_gate = e == "counter" ? 1 : 0;
  p.choice_seed = static_cast<uint64_t>(o.has("choice-seed") ? o.i("choice-seed") : o.i("seed"));
  p.reorder_noise = std::stod(o.s("noise"));
  return p;
}

void fixed_schedule(const Options& o, const GraphH& g, const OracleH& oracle, ScheduleH& s) {
  const std::string& algo = o.s("algo");
  if (!o.s("schedule").empty() && algo != "file") quit(CS_ERR_PARAMETER, "--schedule needs --algo file");
  if (algo == "none") return;
  if (algo == "tic") return check(cs_schedule_tic(g.p, o.s("mode").c_str(), &s.p));
  if (algo == "tac") return check(cs_schedule_tac(g.p, oracle.p, &s.p));
  if (algo == "file") {
    if (o.s("schedule").empty()) quit(CS_ERR_PARAMETER, "--algo file needs --schedule");
    const std::string text = read_file(o.s("schedule"));
    check(cs_schedule_parse(text.c_str(), &s.p));
    char* name = nullptr;
    check(cs_graph_name(g.p, &name));
    const std::string gname = take(name), sname = Json::parse(text)["graph"].get<std::string>();
    if (sname != gname)
      quit(CS_ERR_VALIDATION, "schedule was computed for graph '" + sname + "', not '" + gname + "'");
    return;
  }
  quit(CS_ERR_PARAMETER, "unknown algorithm: " + algo);
}

int cmd_sweep(const Options& o) {
  if (o.s("out").empty()) quit(CS_ERR_PARAMETER, "--out is required");
  if (o.s("seeds").empty()) quit(CS_ERR_PARAMETER, "--seeds is required");
  const std::vector<uint64_t> seeds = parse_seeds(o.s("seeds"));
  GraphH g;
  OracleH oracle;
  load(o, g, oracle);
  int cluster = 0;
  check(cs_graph_is_cluster(g.p, &cluster));
  const cs_sim_policy pol = make_policy(o);
  std::string csv = cluster ? "seed,makespan_us,iteration_us,straggler\n" : "seed,makespan_us\n";
  int64_t lo_all = INT64_MAX, hi_all = INT64_MIN;
  auto row = [&](uint64_t seed, int64_t m, const std::vector<int64_t>* wm, const Json* it) {
    lo_all = std::min(lo_all, m);
    hi_all = std::max(hi_all, m);
    csv += std::to_string(seed) + "," + std::to_string(m);
    if (wm) {  // sim.cpp:258-279 from the per-worker makespans
      int64_t hi = INT64_MIN, lo = INT64_MAX;
      for (int64_t x : *wm) hi = std::max(hi, x), lo = std::min(lo, x);
      csv += "," + std::to_string(hi) + "," + (hi ? decimal6(hi - lo, hi) : decimal6(0, 1));
    } else if (it) {
      csv += "," + std::to_string((*it)["iteration_us"].get<int64_t>()) + "," +
             decimal6((*it)["straggler"]["num"].get<int64_t>(), (*it)["straggler"]["den"].get<int64_t>());
    }
    csv += "\n";
  };
  if (o.s("algo") == "random") {
    int64_t workers = 0;
    if (cluster) {
      char* dv = nullptr;
      check(cs_graph_worker_devices(g.p, &dv));
      workers = static_cast<int64_t>(Json::parse(take(dv)).size());
    }
    for (size_t a = 0; a < seeds.size();) {  // maximal contiguous ascending runs
      size_t b = a + 1;
      while (b < seeds.size() && seeds[b] == seeds[b - 1] + 1) ++b;
      const int64_t n = static_cast<int64_t>(b - a);
      std::vector<int64_t> ms(static_cast<size_t>(n)), wms(static_cast<size_t>(n * std::max<int64_t>(workers, 1)));
      cs_sweep_stats st{};
      const int gpus = static_cast<int>(o.i("gpus"));
      if (gpus > 1) setenv("NCCL_DEBUG", "WARN", 0);  // keep NCCL's banner off the summary stream
      if (gpus > 1)  // seeds sharded over this process's GPUs, one NCCL reduction
        check(cs_sweep_random_multi(g.p, oracle.p, seeds[a], n, &pol, gpus, ms.data(),
                                    cluster ? wms.data() : nullptr, &st));
      else
        check(cs_sweep_random(g.p, oracle.p, seeds[a], n, &pol, ms.data(), cluster ? wms.data() : nullptr, &st));
      for (int64_t k = 0; k < n; ++k) {
        if (cluster) {
          const std::vector<int64_t> wm(wms.begin() + k * workers, wms.begin() + (k + 1) * workers);
          row(seeds[a] + static_cast<uint64_t>(k), ms[static_cast<size_t>(k)], &wm, nullptr);
        } else {
          row(seeds[a] + static_cast<uint64_t>(k), ms[static_cast<size_t>(k)], nullptr, nullptr);
        }
      }
      a = b;
    }
  } else {
    ScheduleH fixed;
    fixed_schedule(o, g, oracle, fixed);
    for (uint64_t s : seeds) {
      cs_sim_policy p = pol;
      p.choice_seed = s;
      ReportH r;
      check(cs_simulate(g.p, oracle.p, fixed.p, &p, &r.p));
      int64_t m = 0;
      check(cs_report_makespan(r.p, &m));
      if (cluster) {
        char* it = nullptr;
        check(cs_report_iteration_json(r.p, &it));
        const Json j = Json::parse(take(it));
        row(s, m, nullptr, &j);
      } else {
        row(s, m, nullptr, nullptr);
      }
    }
  }
  Artifacts arts;
  arts.add(o.s("out"), std::move(csv));
  arts.commit();
  std::printf("sweep seeds=%zu min_us=%lld max_us=%lld\n", seeds.size(), static_cast<long long>(lo_all),
              static_cast<long long>(hi_all));
  return CS_OK;
}

int cmd_bruteforce(const Options& o) {
  GraphH g;
  OracleH oracle;
  load(o, g, oracle);
  const cs_sim_policy pol = make_policy(o);
  char* out = nullptr;
  check(cs_brute_force(g.p, oracle.p, &pol, static_cast<int>(o.i("max-recvs")), &out));
  const std::string text = take(out);
  Artifacts arts;
  arts.add(o.s("out"), text);
  arts.commit();
  const Json res = Json::parse(text);
  std::string order;
  for (const auto& id : res["order"]) order += (order.empty() ? "" : ",") + id.get<std::string>();
  std::printf("best m_us=%lld order=%s\n", static_cast<long long>(res["makespan_us"].get<int64_t>()), order.c_str());
  return CS_OK;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const Options o = options(argc, argv);
    return o.cmd == "sweep" ? cmd_sweep(o) : cmd_bruteforce(o);
  } catch (const Exit& e) {
    std::fprintf(stderr, "error: %s\n", e.message.c_str());
    return e.code;
  } catch (const std::exception& e) {  // the reference's catch-all
    std::fprintf(stderr, "error: %s\n", e.what());
    return CS_ERR_INTERNAL;
  }
}
