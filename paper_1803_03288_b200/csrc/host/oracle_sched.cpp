// Time oracles, schedule documents and exact rationals — host-side I/O
// (reference time_oracle.cpp:22-159, schedule.cpp:86-123, rational.hpp).
#include <algorithm>
#include <numeric>
#include <set>

#include "core.hpp"

namespace tictac {

static std::string joined(const std::vector<std::string>& ids) {
  std::string s;
  for (size_t i = 0; i < ids.size(); ++i) s += (i ? ", " : "") + ids[i];
  return s;
}

static TimeOracle checked(std::shared_ptr<const Graph> g, std::vector<int64_t> us, const char* origin) {
  // time_oracle.cpp:64-70: every entry must be non-negative.
  for (size_t i = 0; i < us.size(); ++i)
    if (us[i] < 0) fail(kValidation, "oracle entry " + g->ops()[i].id + ": negative duration");
  return TimeOracle{std::move(g), std::move(us), origin};
}

TimeOracle TimeOracle::declared(std::shared_ptr<const Graph> g) {  // time_oracle.cpp:72-84
  std::vector<int64_t> us(g->n());
  std::vector<std::string> missing;
  for (int32_t i = 0; i < g->n(); ++i) {
    const Op& op = g->ops()[i];
    if (op.time_us) us[i] = *op.time_us;
    else missing.push_back(op.id);
  }
  if (!missing.empty()) fail(kCoverage, "ops without declared time: " + joined(missing));
  return checked(std::move(g), std::move(us), "declared");
}

TimeOracle TimeOracle::general(std::shared_ptr<const Graph> g) {  // time_oracle.cpp:86-91
  std::vector<int64_t> us(g->n());
  for (int32_t i = 0; i < g->n(); ++i) us[i] = g->ops()[i].kind == kRecv ? 1 : 0;
  return checked(std::move(g), std::move(us), "general");
}

TimeOracle TimeOracle::traces(std::shared_ptr<const Graph> g, std::string_view text) {
  // parse_trace_jsonl (time_oracle.cpp:22-52) then the min rule (93-112).
  std::map<std::string, int64_t> best;
  size_t pos = 0, line_no = 0;
  while (pos <= text.size()) {
    const size_t nl = text.find('\n', pos);
    const std::string_view line =
        text.substr(pos, nl == std::string_view::npos ? std::string_view::npos : nl - pos);
    ++line_no;
    pos = nl == std::string_view::npos ? text.size() + 1 : nl + 1;
    if (line.find_first_not_of(" \t\r") == std::string_view::npos) continue;
    const std::string tag = "trace line " + std::to_string(line_no);
    Json j = parse_doc(line, tag);
    if (!j.is_object() || !j.contains("op") || !j["op"].is_string() || !j.contains("run") ||
        !j["run"].is_number_integer() || !j.contains("us") || !j["us"].is_number_integer())
      fail(kValidation, tag + ": expected {\"op\", \"run\", \"us\"}");
    const std::string op = j["op"].get<std::string>();
    const int64_t run = j["run"].get<int64_t>(), us = j["us"].get<int64_t>();
    if (run < 0) fail(kValidation, tag + ": negative run index");
    if (us < 0) fail(kValidation, tag + ": negative duration");
    auto it = best.find(op);
    if (it == best.end()) best.emplace(op, us);
    else it->second = std::min(it->second, us);
  }
  std::vector<std::string> missing;
  std::vector<int64_t> us(g->n());
  for (int32_t i = 0; i < g->n(); ++i) {
    const auto it = best.find(g->ops()[i].id);
    if (it == best.end()) missing.push_back(g->ops()[i].id);
    else us[i] = it->second;
  }
  if (!missing.empty()) fail(kCoverage, "ops without trace records: " + joined(missing));
  return checked(std::move(g), std::move(us), "measured");
}

TimeOracle TimeOracle::bandwidth(std::shared_ptr<const Graph> g, int64_t bw) {  // time_oracle.cpp:114-134
  if (bw <= 0) fail(kParameter, "bandwidth must be positive bytes per microsecond");
  std::vector<int64_t> us(g->n());
  std::vector<std::string> missing;
  for (int32_t i = 0; i < g->n(); ++i) {
    const Op& op = g->ops()[i];
    if (transfer(op.kind) && op.bytes) us[i] = (2 * *op.bytes + bw) / (2 * bw);
    else if (op.time_us) us[i] = *op.time_us;
    else missing.push_back(op.id);
  }
  if (!missing.empty()) fail(kCoverage, "ops without bytes or declared time: " + joined(missing));
  return checked(std::move(g), std::move(us), "synthetic");
}

std::vector<int64_t> TimeOracle::durations(const Graph& g) const {
  if (&g == src.get()) return us;
  std::vector<int64_t> d(g.n());
  std::vector<std::string> missing;
  // both op lists are in id order: one merge pass
  const auto& have = src->ops();
  size_t j = 0;
  for (int32_t i = 0; i < g.n(); ++i) {
    const std::string& id = g.ops()[i].id;
    while (j < have.size() && have[j].id < id) ++j;
    if (j == have.size() || have[j].id != id) missing.push_back(id);
    else d[i] = us[j];
  }
  if (!missing.empty()) fail(kCoverage, "oracle missing entries for: " + joined(missing));
  return d;
}

Json TimeOracle::to_json() const {  // time_oracle.cpp:151-157 (map order = op index order)
  Json j;
  j["origin"] = origin;
  j["entries"] = Json::object();
  for (int32_t i = 0; i < src->n(); ++i) j["entries"][src->ops()[i].id] = us[i];
  return j;
}

std::string Schedule::serialize() const {
  Json doc;
  doc["graph"] = graph;
  doc["algorithm"] = algorithm;
  doc["priorities"] = Json::object();
  for (const auto& [id, r] : prio) doc["priorities"][id] = r;
  return dump_doc(doc);
}

Schedule Schedule::parse(std::string_view text) {
  Json doc = parse_doc(text, "schedule");
  if (!doc.is_object() || !doc.contains("graph") || !doc["graph"].is_string() ||
      !doc.contains("algorithm") || !doc["algorithm"].is_string() ||
      !doc.contains("priorities") || !doc["priorities"].is_object())
    fail(kValidation, "schedule document needs graph, algorithm and priorities");
  Schedule s;
  s.graph = doc["graph"].get<std::string>();
  s.algorithm = doc["algorithm"].get<std::string>();
  if (s.algorithm != "tic" && s.algorithm != "tac" && s.algorithm != "random")
    fail(kValidation, "unknown schedule algorithm: " + s.algorithm);
  for (auto& [id, rank] : doc["priorities"].items()) {
    if (!rank.is_number_integer() || rank.get<int64_t>() < 0)
      fail(kValidation, "priority for " + id + " must be a non-negative integer");
    s.prio[id] = rank.get<int>();
  }
  // Total order iff the ranks are a bijection onto [0, n).
  std::set<int> seen;
  for (const auto& kv : s.prio) seen.insert(kv.second);
  s.total = seen.size() == s.prio.size() &&
            (s.prio.empty() ||
             (*seen.begin() == 0 && *seen.rbegin() == static_cast<int>(s.prio.size()) - 1));
  return s;
}

// ---- Rational ----------------------------------------------------------

Rational::Rational(int64_t n, int64_t d) {
  if (d == 0) throw std::invalid_argument("rational with zero denominator");
  if (d < 0) {
    n = -n;
    d = -d;
  }
  const int64_t g = std::gcd(n < 0 ? -n : n, d);
  if (g > 1) {
    n /= g;
    d /= g;
  }
  num = n;
  den = n == 0 ? 1 : d;
}

static int64_t strict_int(const std::string& t) {
  size_t used = 0;
  const int64_t v = std::stoll(t, &used);
  if (used != t.size()) throw std::invalid_argument("not an integer: " + t);
  return v;
}

Rational Rational::parse(const std::string& text) {  // rational.hpp:103-128
  if (text.empty()) throw std::invalid_argument("not a rational: " + text);
  const size_t slash = text.find('/');
  if (slash != std::string::npos)
    return Rational(strict_int(text.substr(0, slash)), strict_int(text.substr(slash + 1)));
  const size_t dot = text.find('.');
  if (dot == std::string::npos) return Rational(strict_int(text), 1);
  const std::string whole = text.substr(0, dot), frac = text.substr(dot + 1);
  if (frac.empty() || frac.size() > 18) throw std::invalid_argument("not a rational: " + text);
  int64_t scale = 1;
  for (size_t i = 0; i < frac.size(); ++i) scale *= 10;
  const bool neg = !whole.empty() && whole[0] == '-';
  const int64_t w = whole.empty() || whole == "-" ? 0 : strict_int(whole);
  const int64_t f = strict_int(frac);
  if (f < 0) throw std::invalid_argument("not a rational: " + text);
  return Rational(neg ? w * scale - f : w * scale + f, scale);
}

}  // namespace tictac
