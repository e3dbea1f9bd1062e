// Report / metrics JSON formatting (reference sim.cpp:305-376,
// metrics.cpp:82-105). The numbers come from the device simulator.
#include <algorithm>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <string_view>

#include "core.hpp"

namespace tictac {

namespace {

// Streaming writer for nlohmann's dump(2) layout: members/elements on their
// own lines at 2-space indent, "key": value, empty containers as {} / [],
// strings escaped as its serializer does with ensure_ascii = false.
class JsonText {
 public:
  std::string s;
  void open(char c) {
    s += c;
    first_.push_back(true);
  }
  void close(char c) {
    const bool empty = first_.back();
    first_.pop_back();
    if (!empty) newline();
    s += c;
  }
  void item() {  // before each array element
    if (!first_.back()) s += ',';
    first_.back() = false;
    newline();
  }
  void key(std::string_view k) {
    item();
    str(k);
    s += ": ";
  }
  void num(int64_t v) {
    char buf[24];
    const auto res = std::to_chars(buf, buf + sizeof(buf), v);
    s.append(buf, res.ptr);
  }
  void str(std::string_view v) {
    s += '"';
    // bulk-append runs that need no escaping
    size_t run = 0;
    for (size_t i = 0; i < v.size(); ++i) {
      const unsigned char c = static_cast<unsigned char>(v[i]);
      if (c > 0x1f && c != '"' && c != '\\') continue;
      s.append(v.data() + run, i - run);
      run = i + 1;
      switch (c) {
        case '"': s += "\\\""; break;
        case '\\': s += "\\\\"; break;
        case '\b': s += "\\b"; break;
        case '\f': s += "\\f"; break;
        case '\n': s += "\\n"; break;
        case '\r': s += "\\r"; break;
        case '\t': s += "\\t"; break;
        default: {
          char buf[8];
          std::snprintf(buf, sizeof(buf), "\\u%04x", c);
          s += buf;
        }
      }
    }
    s.append(v.data() + run, v.size() - run);
    s += '"';
  }

 private:
  std::vector<bool> first_;
  void newline() {
    s += '\n';
    s.append(2 * first_.size(), ' ');
  }
};

}  // namespace

std::string Report::json_text() const {
  std::vector<std::string> keys(resources.size());
  for (size_t r = 0; r < resources.size(); ++r) keys[r] = resources[r].key();
  std::map<std::string, int64_t> busy;
  for (const Event& e : events) busy[keys[e.res]] += e.end - e.start;
  JsonText w;
  w.s.reserve(128 * events.size() + 256);
  w.open('{');
  w.key("makespan_us");
  w.num(makespan);
  w.key("violations");
  w.num(violations);
  w.key("busy");
  w.open('{');
  for (const auto& [k, us] : busy) {
    w.key(k);
    w.num(us);
  }
  w.close('}');
  w.key("events");
  if (events.empty()) {
    w.s += "[]";
  } else {  // fixed per-event layout (depths 2 and 3), fragments appended directly
    std::vector<std::string> qres(resources.size());
    for (size_t r = 0; r < resources.size(); ++r) {
      JsonText q;
      q.str(keys[r]);
      qres[r] = std::move(q.s);
    }
    // one pass into a buffer sized from the fragments' exact lengths
    static constexpr std::string_view kOpen = ",\n    {\n      \"op\": ", kRes = ",\n      \"resource\": ",
                                      kStart = ",\n      \"start_us\": ", kEnd = ",\n      \"end_us\": ",
                                      kClose = "\n    }";
    size_t bound = w.s.size() + 8;
    for (const Event& e : events)
      bound += kOpen.size() + kRes.size() + kStart.size() + kEnd.size() + kClose.size() + 6 * op_id(e.op).size() +
               2 + qres[e.res].size() + 40;
    const size_t at = w.s.size();
    w.s.resize(bound);
    char* p = w.s.data() + at;
    auto put = [&p](std::string_view f) {
      std::memcpy(p, f.data(), f.size());
      p += f.size();
    };
    *p++ = '[';
    for (size_t i = 0; i < events.size(); ++i) {
      const Event& e = events[i];
      put(i ? kOpen : kOpen.substr(1));
      const std::string& id = op_id(e.op);
      *p++ = '"';
      if (std::all_of(id.begin(), id.end(), [](char c) {
            const unsigned char u = static_cast<unsigned char>(c);
            return u > 0x1f && u != '"' && u != '\\';
          })) {
        put(id);
      } else {  // rare: ids that need escaping
        JsonText q;
        q.str(id);
        put(std::string_view(q.s).substr(1, q.s.size() - 2));
      }
      *p++ = '"';
      put(kRes);
      put(qres[e.res]);
      put(kStart);
      p = std::to_chars(p, p + 24, e.start).ptr;
      put(kEnd);
      p = std::to_chars(p, p + 24, e.end).ptr;
      put(kClose);
    }
    put("\n  ]");
    w.s.resize(static_cast<size_t>(p - w.s.data()));
  }
  w.close('}');
  w.s += '\n';
  return std::move(w.s);
}

std::string Report::chrome_trace_text() const {
  std::vector<std::string> devices;
  for (const Resource& r : resources) devices.push_back(r.device);
  std::sort(devices.begin(), devices.end());
  devices.erase(std::unique(devices.begin(), devices.end()), devices.end());
  std::vector<int64_t> pid(resources.size());
  for (size_t r = 0; r < resources.size(); ++r)
    pid[r] = std::lower_bound(devices.begin(), devices.end(), resources[r].device) - devices.begin();
  JsonText w;
  w.s.reserve(160 * events.size() + 256);
  w.open('{');
  w.key("traceEvents");
  w.open('[');
  for (size_t d = 0; d < devices.size(); ++d) {
    w.item();
    w.open('{');
    w.key("name");
    w.str("process_name");
    w.key("ph");
    w.str("M");
    w.key("pid");
    w.num(static_cast<int64_t>(d));
    w.key("args");
    w.open('{');
    w.key("name");
    w.str(devices[d]);
    w.close('}');
    w.close('}');
  }
  for (size_t r = 0; r < resources.size(); ++r) {
    w.item();
    w.open('{');
    w.key("name");
    w.str("thread_name");
    w.key("ph");
    w.str("M");
    w.key("pid");
    w.num(pid[r]);
    w.key("tid");
    w.num(static_cast<int64_t>(r));
    w.key("args");
    w.open('{');
    w.key("name");
    w.str(std::string(resources[r].channel ? "channel" : "compute") + "/" + resources[r].name);
    w.close('}');
    w.close('}');
  }
  for (const Event& e : events) {  // fixed layout: fragments appended directly
    w.item();
    w.s += "{\n      \"name\": ";
    w.str(op_id(e.op));
    w.s += resources[e.res].channel ? ",\n      \"cat\": \"channel\",\n      \"ph\": \"X\",\n      \"pid\": "
                                    : ",\n      \"cat\": \"compute\",\n      \"ph\": \"X\",\n      \"pid\": ";
    w.num(pid[e.res]);
    w.s += ",\n      \"tid\": ";
    w.num(e.res);
    w.s += ",\n      \"ts\": ";
    w.num(e.start);
    w.s += ",\n      \"dur\": ";
    w.num(e.end - e.start);
    w.s += "\n    }";
  }
  w.close(']');
  w.close('}');
  w.s += '\n';
  return std::move(w.s);
}

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
    je["op"] = op_id(e.op);
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
    x["name"] = op_id(e.op);
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
