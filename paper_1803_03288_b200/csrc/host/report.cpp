// Report / metrics JSON formatting (reference sim.cpp:305-376,
// metrics.cpp:82-105). The numbers come from the device simulator.
#include <algorithm>

#include "core.hpp"

namespace tictac {

Json Report::to_json() const {
  Json j;
  j["makespan_us"] = makespan;
  j["violations"] = violations;
  std::map<std::string, int64_t> busy;  // resource key -> occupied us
  for (const Event& e : events) busy[resources[e.res].key()] += e.end - e.start;
  j["busy"] = Json::object();
  for (const auto& [k, us] : busy) j["busy"][k] = us;
  j["events"] = Json::array();
  for (const Event& e : events) {
    Json je;
    je["op"] = op_ids[e.op];
    je["resource"] = resources[e.res].key();
    je["start_us"] = e.start;
    je["end_us"] = e.end;
    j["events"].push_back(std::move(je));
  }
  return j;
}

Json Report::chrome_trace() const {
  std::vector<std::string> devices;
  for (const Resource& r : resources) devices.push_back(r.device);
  std::sort(devices.begin(), devices.end());
  devices.erase(std::unique(devices.begin(), devices.end()), devices.end());
  auto pid = [&](const std::string& d) {
    return static_cast<int>(std::lower_bound(devices.begin(), devices.end(), d) - devices.begin());
  };
  Json trace = Json::array();
  for (size_t d = 0; d < devices.size(); ++d) {
    Json m;
    m["name"] = "process_name";
    m["ph"] = "M";
    m["pid"] = static_cast<int>(d);
    m["args"] = {{"name", devices[d]}};
    trace.push_back(std::move(m));
  }
  for (size_t r = 0; r < resources.size(); ++r) {
    Json m;
    m["name"] = "thread_name";
    m["ph"] = "M";
    m["pid"] = pid(resources[r].device);
    m["tid"] = static_cast<int>(r);
    m["args"] = {{"name", std::string(resources[r].channel ? "channel" : "compute") + "/" +
                              resources[r].name}};
    trace.push_back(std::move(m));
  }
  for (const Event& e : events) {
    Json x;
    x["name"] = op_ids[e.op];
    x["cat"] = resources[e.res].channel ? "channel" : "compute";
    x["ph"] = "X";
    x["pid"] = pid(resources[e.res].device);
    x["tid"] = static_cast<int>(e.res);
    x["ts"] = e.start;
    x["dur"] = e.end - e.start;
    trace.push_back(std::move(x));
  }
  Json j;
  j["traceEvents"] = std::move(trace);
  return j;
}

Json Report::iteration_json() const {
  Json j;
  j["per_worker_makespan_us"] = Json::object();
  for (const auto& [d, m] : per_worker) j["per_worker_makespan_us"][d] = m;
  j["iteration_us"] = iteration;
  j["straggler"] = {{"num", strag_num}, {"den", strag_den}};
  return j;
}

Json metrics_json(int64_t U, int64_t L, int64_t m, const Report* stats) {
  Json j;
  j["U_us"] = U;
  j["L_us"] = L;
  j["m_us"] = m;
  if (U == L) {
    j["E"] = nullptr;
  } else {
    const Rational e(U - m, U - L);  // efficiency, metrics.cpp:24-29
    j["E"] = {{"num", e.num}, {"den", e.den}};
  }
  if (L == 0) {
    j["S"] = nullptr;
  } else {
    const Rational s(U - L, L);  // speedup, metrics.cpp:31-35
    j["S"] = {{"num", s.num}, {"den", s.den}};
  }
  if (stats && stats->has_stats)
    j["straggler"] = {{"num", stats->strag_num}, {"den", stats->strag_den}};
  else
    j["straggler"] = nullptr;
  return j;
}

}  // namespace tictac
