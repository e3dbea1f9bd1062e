// TEST / BASELINE INFRASTRUCTURE ONLY. Drives the *reference* libcommsched
// (built from /root/reference by oracle/Makefile into oracle/_ref/) through its
// own C ABI, exactly the way `sched sweep` does (tools/sched_main.cpp:452-502):
// per seed cs_schedule_random(g, seed) + cs_simulate with choice_seed = seed.
// The reference has no threads; independent seeds are split over P pthreads
// (contiguous slices), which is what BASELINE.md §3 prescribes for the CPU arm.
//
// usage:
//   ref_sweep sweep <graph.json> <oracle> <seed_lo> <count> <threads> [out.bin] [noise]
//   ref_sweep sweeplist <graph.json> <oracle> <seeds.bin> <threads> [out.bin] [noise]
//     (seeds.bin: uint64 seeds, any order; results in that order)
//   ref_sweep tac   <graph.json> <oracle>      -> schedule JSON on stdout, seconds on stderr
//   ref_sweep tic   <graph.json> <mode>        -> schedule JSON on stdout, seconds on stderr
// <oracle> is "declared" or "bw:<bytes_per_us>".
// sweep prints one JSON line: {"seconds","sims","min","argmin","sum"}; out.bin gets
// int64 makespans (and for cluster graphs, int64 per-worker makespans after them).

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "commsched.h"

namespace {

std::string slurp(const char* path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) {
    std::fprintf(stderr, "cannot read %s\n", path);
    std::exit(5);
  }
  std::ostringstream s;
  s << in.rdbuf();
  return s.str();
}

void check(int rc, const char* what) {
  if (rc != CS_OK) {
    std::fprintf(stderr, "%s failed (%d): %s\n", what, rc, cs_last_error());
    std::exit(rc);
  }
}

cs_oracle* make_oracle(cs_graph* g, const std::string& kind) {
  cs_oracle* o = nullptr;
  if (kind == "declared") {
    check(cs_oracle_declared(g, &o), "cs_oracle_declared");
  } else if (kind.rfind("bw:", 0) == 0) {
    check(cs_oracle_bandwidth(g, std::atoll(kind.c_str() + 3), &o),
          "cs_oracle_bandwidth");
  } else if (kind == "general") {
    check(cs_oracle_general(g, &o), "cs_oracle_general");
  } else {
    std::fprintf(stderr, "unknown oracle %s\n", kind.c_str());
    std::exit(4);
  }
  return o;
}

// Per-worker makespans out of cs_report_iteration_json without a JSON
// library: the object is {"per_worker_makespan_us": {"w0": N, ...}, ...}.
void per_worker(const char* json, std::vector<int64_t>& out) {
  const char* p = std::strstr(json, "per_worker_makespan_us");
  if (!p) return;
  p = std::strchr(p, '{');
  const char* end = std::strchr(p, '}');
  while (p && p < end) {
    const char* colon = std::strchr(p, ':');
    if (!colon || colon > end) break;
    out.push_back(std::strtoll(colon + 1, nullptr, 10));
    p = colon + 1;
  }
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 4) {
    std::fprintf(stderr, "usage: see header\n");
    return 4;
  }
  const std::string mode = argv[1];
  const std::string text = slurp(argv[2]);
  cs_graph* g = nullptr;
  check(cs_graph_parse(text.c_str(), &g), "cs_graph_parse");

  if (mode == "tac" || mode == "tic") {
    cs_schedule* s = nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    if (mode == "tac") {
      cs_oracle* o = make_oracle(g, argv[3]);
      check(cs_schedule_tac(g, o, &s), "cs_schedule_tac");
    } else {
      check(cs_schedule_tic(g, argv[3], &s), "cs_schedule_tic");
    }
    const double sec = std::chrono::duration<double>(
                           std::chrono::steady_clock::now() - t0).count();
    char* js = nullptr;
    check(cs_schedule_serialize(s, &js), "cs_schedule_serialize");
    std::fputs(js, stdout);
    std::fprintf(stderr, "{\"seconds\": %.9f}\n", sec);
    cs_string_free(js);
    return 0;
  }

  const bool list = mode == "sweeplist";
  if ((mode != "sweep" || argc < 7) && (!list || argc < 6)) {
    std::fprintf(stderr, "bad arguments\n");
    return 4;
  }
  cs_oracle* o = make_oracle(g, argv[3]);
  std::vector<uint64_t> seeds;
  if (list) {
    std::ifstream in(argv[4], std::ios::binary);
    uint64_t v = 0;
    while (in.read(reinterpret_cast<char*>(&v), sizeof v)) seeds.push_back(v);
  } else {
    const uint64_t lo0 = std::strtoull(argv[4], nullptr, 10);
    const int64_t n0 = std::atoll(argv[5]);
    for (int64_t i = 0; i < n0; ++i) seeds.push_back(lo0 + static_cast<uint64_t>(i));
  }
  const int ai = list ? 5 : 6;  // index of <threads>
  const int64_t count = static_cast<int64_t>(seeds.size());
  int threads = std::atoi(argv[ai]);
  if (threads <= 0) threads = static_cast<int>(std::thread::hardware_concurrency());
  const char* out_path = argc > ai + 1 && std::strcmp(argv[ai + 1], "-") != 0 ? argv[ai + 1] : nullptr;
  const double noise = argc > ai + 2 ? std::atof(argv[ai + 2]) : 0.0;
  int cluster = 0;
  check(cs_graph_is_cluster(g, &cluster), "cs_graph_is_cluster");

  std::vector<int64_t> ms(static_cast<size_t>(count));
  std::vector<std::vector<int64_t>> pw(static_cast<size_t>(cluster ? count : 0));
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  const int64_t per = (count + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    const int64_t a = t * per, b = std::min<int64_t>(count, a + per);
    if (a >= b) break;
    pool.emplace_back([&, a, b] {
      for (int64_t i = a; i < b; ++i) {
        const uint64_t seed = seeds[static_cast<size_t>(i)];
        cs_schedule* s = nullptr;
        check(cs_schedule_random(g, seed, &s), "cs_schedule_random");
        cs_sim_policy policy{1, seed, noise};
        cs_report* r = nullptr;
        check(cs_simulate(g, o, s, &policy, &r), "cs_simulate");
        check(cs_report_makespan(r, &ms[static_cast<size_t>(i)]), "makespan");
        if (cluster) {
          char* js = nullptr;
          check(cs_report_iteration_json(r, &js), "iteration_json");
          per_worker(js, pw[static_cast<size_t>(i)]);
          cs_string_free(js);
        }
        cs_report_free(r);
        cs_schedule_free(s);
      }
    });
  }
  for (auto& th : pool) th.join();
  const double sec = std::chrono::duration<double>(
                         std::chrono::steady_clock::now() - t0).count();
  int64_t best = 0, arg = 0, sum = 0;
  for (int64_t i = 0; i < count; ++i) {
    if (i == 0 || ms[static_cast<size_t>(i)] < best) {
      best = ms[static_cast<size_t>(i)];
      arg = static_cast<int64_t>(seeds[static_cast<size_t>(i)]);
    }
    sum += ms[static_cast<size_t>(i)];
  }
  if (out_path) {
    std::ofstream out(out_path, std::ios::binary);
    out.write(reinterpret_cast<const char*>(ms.data()),
              static_cast<std::streamsize>(ms.size() * sizeof(int64_t)));
    for (const auto& v : pw)
      out.write(reinterpret_cast<const char*>(v.data()),
                static_cast<std::streamsize>(v.size() * sizeof(int64_t)));
  }
  std::printf(
      "{\"seconds\": %.9f, \"sims\": %lld, \"threads\": %d, \"min\": %lld, "
      "\"argmin\": %lld, \"sum\": %lld}\n",
      sec, static_cast<long long>(count), threads, static_cast<long long>(best),
      static_cast<long long>(arg), static_cast<long long>(sum));
  cs_oracle_free(o);
  cs_graph_free(g);
  return 0;
}
