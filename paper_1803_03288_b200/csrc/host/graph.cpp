// Graph model: parse / validate / serialize and the index model the device
// kernels consume (reference graph.cpp:54-290, sim.cpp:27-59).
#include <algorithm>
#include <set>

#include "../device/csk.h"
#include <cuda_runtime.h>

#include "core.hpp"

namespace tictac {

Json parse_doc(std::string_view text, std::string_view what) {
  // json_io.hpp:18-37: nlohmann parse errors re-reported as line/column.
  try {
    return Json::parse(text);
  } catch (const nlohmann::json::parse_error& e) {
    size_t off = e.byte > 0 ? e.byte - 1 : 0;
    off = std::min(off, text.size());
    size_t line = 1, col = 1;
    for (size_t i = 0; i < off; ++i) {
      if (text[i] == '\n') {
        ++line;
        col = 1;
      } else {
        ++col;
      }
    }
    fail(kValidation, std::string(what) + ": parse error at line " + std::to_string(line) +
                          ", column " + std::to_string(col));
  }
}

static const char* const kKindNames[] = {"compute", "recv", "send", "ps_aggregate", "ps_read",
                                         "ps_update"};
const char* kind_str(OpKind k) { return kKindNames[static_cast<int>(k)]; }

static OpKind kind_parse(const std::string& s) {  // graph.cpp:25-33
  for (int k = 0; k < 6; ++k)
    if (s == kKindNames[k]) return static_cast<OpKind>(k);
  fail(kValidation, "unknown op kind: " + s);
}

static bool unit_parse(const std::string& s) {  // graph.cpp:39-43
  if (s == "compute") return false;
  if (s == "channel") return true;
  fail(kValidation, "unknown resource unit: " + s);
}

std::shared_ptr<Graph> Graph::make(std::string name, bool cluster, std::vector<Op> ops,
                                   std::vector<std::pair<std::string, std::string>> edges) {
  auto g = std::make_shared<Graph>();
  g->name_ = std::move(name);
  g->cluster_ = cluster;
  std::sort(ops.begin(), ops.end(), [](const Op& a, const Op& b) { return a.id < b.id; });
  std::sort(edges.begin(), edges.end());
  edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
  g->ops_ = std::move(ops);
  g->edges_ = std::move(edges);
  g->index_and_validate();
  return g;
}

void Graph::index_and_validate() {
  // Index + adjacency (graph.cpp:71-96).
  const int32_t n = static_cast<int32_t>(ops_.size());
  index_.reserve(ops_.size());
  for (int32_t i = 0; i < n; ++i) {
    if (ops_[i].id.empty()) fail(kValidation, "op has empty id");
    if (!index_.emplace(ops_[i].id, i).second)
      fail(kValidation, "duplicate op id: " + ops_[i].id);
  }
  std::vector<int32_t> indeg(n + 1, 0), outdeg(n + 1, 0);
  std::vector<std::pair<int32_t, int32_t>> ix;
  ix.reserve(edges_.size());
  for (const auto& [from, to] : edges_) {
    auto a = index_.find(from), b = index_.find(to);
    const std::string tag = "edge " + from + " -> " + to + ": ";
    if (a == index_.end()) fail(kValidation, tag + "unknown op " + from);
    if (b == index_.end()) fail(kValidation, tag + "unknown op " + to);
    if (a->second == b->second) fail(kValidation, tag + "self loop");
    ix.emplace_back(a->second, b->second);
    outdeg[a->second]++;
    indeg[b->second]++;
  }
  pred_off_.assign(n + 1, 0);
  succ_off_.assign(n + 1, 0);
  for (int32_t i = 0; i < n; ++i) {
    pred_off_[i + 1] = pred_off_[i] + indeg[i];
    succ_off_[i + 1] = succ_off_[i] + outdeg[i];
  }
  pred_idx_.assign(ix.size(), 0);
  succ_idx_.assign(ix.size(), 0);
  std::vector<int32_t> pf(pred_off_.begin(), pred_off_.end() - 1),
      sf(succ_off_.begin(), succ_off_.end() - 1);
  for (auto [a, b] : ix) {
    succ_idx_[sf[a]++] = b;
    pred_idx_[pf[b]++] = a;
  }
  for (int32_t i = 0; i < n; ++i) {
    std::sort(pred_idx_.begin() + pred_off_[i], pred_idx_.begin() + pred_off_[i + 1]);
    std::sort(succ_idx_.begin() + succ_off_[i], succ_idx_.begin() + succ_off_[i + 1]);
  }

  // Validation (graph.cpp:98-145), same order and messages.
  if (ops_.empty()) fail(kValidation, "graph has no ops");
  for (const Op& op : ops_) {
    if (op.bytes && !transfer(op.kind))
      fail(kValidation, "op " + op.id + ": bytes set on non-transfer op");
    if (op.bytes && *op.bytes < 0) fail(kValidation, "op " + op.id + ": negative bytes");
    if (op.time_us && *op.time_us < 0) fail(kValidation, "op " + op.id + ": negative time_us");
    if (transfer(op.kind) && !op.res.channel)
      fail(kValidation, "op " + op.id + ": transfer op assigned to a compute resource");
    if (!transfer(op.kind) && op.res.channel)
      fail(kValidation, "op " + op.id + ": non-transfer op assigned to a channel resource");
  }
  if (!cluster_) {
    for (int32_t i = 0; i < n; ++i) {
      if (ops_[i].kind == kRecv && npred(i) > 0)
        fail(kValidation, "op " + ops_[i].id + ": recv op has incoming edge");
      if (ops_[i].kind == kSend && nsucc(i) > 0)
        fail(kValidation, "op " + ops_[i].id + ": send op has outgoing edge");
    }
  }
  // Cycle check: the reference's colored iterative DFS, reproduced step for
  // step so the reported op is the same one.
  std::vector<uint8_t> color(n, 0);
  std::vector<int32_t> stack;
  for (int32_t root = 0; root < n; ++root) {
    if (color[root]) continue;
    stack.push_back(root);
    while (!stack.empty()) {
      const int32_t v = stack.back();
      if (color[v] == 0) {
        color[v] = 1;
        for (int32_t e = succ_off_[v]; e < succ_off_[v + 1]; ++e) {
          const int32_t w = succ_idx_[e];
          if (color[w] == 1) fail(kValidation, "cycle detected at op " + ops_[w].id);
          if (color[w] == 0) stack.push_back(w);
        }
      } else {
        color[v] = 2;
        stack.pop_back();
      }
    }
  }

  std::set<Resource> seen;
  for (const Op& op : ops_) seen.insert(op.res);
  resources_.assign(seen.begin(), seen.end());
  res_of_.resize(n);
  for (int32_t i = 0; i < n; ++i)
    res_of_[i] = static_cast<int32_t>(
        std::lower_bound(resources_.begin(), resources_.end(), ops_[i].res) - resources_.begin());
  for (int32_t i = 0; i < n; ++i)
    if (ops_[i].kind == kRecv) recv_ops_.push_back(i);
}

Graph::~Graph() {
  for (auto& [d, dg] : dev_) csk_graph_free(dg);
}

int32_t Graph::at(const std::string& id) const {
  auto it = index_.find(id);
  if (it == index_.end()) fail(kValidation, "unknown op: " + id);
  return it->second;
}

std::shared_ptr<Graph> Graph::parse(std::string_view text) {  // graph.cpp:200-268
  Json doc = parse_doc(text, "graph");
  if (!doc.is_object()) fail(kValidation, "graph document must be an object");
  for (auto& [key, value] : doc.items()) {
    (void)value;
    if (key != "name" && key != "partition" && key != "ops" && key != "edges")
      fail(kValidation, "graph document has unknown key: " + key);
  }
  if (!doc.contains("name") || !doc["name"].is_string())
    fail(kValidation, "graph document needs a string \"name\"");
  if (!doc.contains("partition") || !doc["partition"].is_string())
    fail(kValidation, "graph document needs a string \"partition\"");
  const std::string part = doc["partition"].get<std::string>();
  if (part != "worker" && part != "cluster") fail(kValidation, "unknown partition: " + part);
  if (!doc.contains("ops") || !doc["ops"].is_array())
    fail(kValidation, "graph document needs an \"ops\" array");
  std::vector<Op> ops;
  for (const Json& j : doc["ops"]) {
    if (!j.is_object()) fail(kValidation, "op entry must be an object");
    Op op;
    if (!j.contains("id") || !j["id"].is_string())
      fail(kValidation, "op entry needs a string \"id\"");
    op.id = j["id"].get<std::string>();
    if (!j.contains("kind") || !j["kind"].is_string())
      fail(kValidation, "op " + op.id + ": needs a string \"kind\"");
    op.kind = kind_parse(j["kind"].get<std::string>());
    if (!j.contains("resource") || !j["resource"].is_object())
      fail(kValidation, "op " + op.id + ": needs a \"resource\" object");
    const Json& r = j["resource"];
    if (!r.contains("device") || !r["device"].is_string() || !r.contains("unit") ||
        !r["unit"].is_string() || !r.contains("name") || !r["name"].is_string())
      fail(kValidation, "op " + op.id + ": resource needs device/unit/name strings");
    op.res.device = r["device"].get<std::string>();
    op.res.channel = unit_parse(r["unit"].get<std::string>());
    op.res.name = r["name"].get<std::string>();
    if (j.contains("time_us")) {
      if (!j["time_us"].is_number_integer())
        fail(kValidation, "op " + op.id + ": time_us must be an integer");
      op.time_us = j["time_us"].get<int64_t>();
    }
    if (j.contains("bytes")) {
      if (!j["bytes"].is_number_integer())
        fail(kValidation, "op " + op.id + ": bytes must be an integer");
      op.bytes = j["bytes"].get<int64_t>();
    }
    ops.push_back(std::move(op));
  }
  std::vector<std::pair<std::string, std::string>> edges;
  if (doc.contains("edges")) {
    if (!doc["edges"].is_array()) fail(kValidation, "graph \"edges\" must be an array");
    for (const Json& e : doc["edges"]) {
      if (!e.is_array() || e.size() != 2 || !e[0].is_string() || !e[1].is_string())
        fail(kValidation, "edge entry must be a [from, to] string pair");
      edges.emplace_back(e[0].get<std::string>(), e[1].get<std::string>());
    }
  }
  return make(doc["name"].get<std::string>(), part == "cluster", std::move(ops),
              std::move(edges));
}

std::string Graph::serialize() const {  // graph.cpp:270-290
  Json doc;
  doc["name"] = name_;
  doc["partition"] = cluster_ ? "cluster" : "worker";
  doc["ops"] = Json::array();
  for (const Op& op : ops_) {
    Json j;
    j["id"] = op.id;
    j["kind"] = kind_str(op.kind);
    j["resource"] = {{"device", op.res.device},
                     {"unit", op.res.channel ? "channel" : "compute"},
                     {"name", op.res.name}};
    if (op.time_us) j["time_us"] = *op.time_us;
    if (op.bytes) j["bytes"] = *op.bytes;
    doc["ops"].push_back(std::move(j));
  }
  doc["edges"] = Json::array();
  for (const auto& [a, b] : edges_) doc["edges"].push_back(Json::array({a, b}));
  return dump_doc(doc);
}

std::vector<std::string> Graph::recv_ids() const {
  std::vector<std::string> out;
  for (int32_t i : recv_ops_) out.push_back(ops_[i].id);
  return out;
}

std::vector<std::string> Graph::topo_order() const {  // graph.cpp:158-185
  const int32_t n = this->n();
  std::vector<int64_t> depth(n, 0);
  std::vector<int32_t> missing(n), q;
  for (int32_t i = 0; i < n; ++i)
    if ((missing[i] = npred(i)) == 0) q.push_back(i);
  for (size_t h = 0; h < q.size(); ++h) {
    const int32_t v = q[h];
    for (int32_t e = succ_off_[v]; e < succ_off_[v + 1]; ++e) {
      const int32_t w = succ_idx_[e];
      depth[w] = std::max(depth[w], depth[v] + 1);
      if (--missing[w] == 0) q.push_back(w);
    }
  }
  std::vector<int32_t> order(n);
  for (int32_t i = 0; i < n; ++i) order[i] = i;
  // Ops are already in id order, so (depth, index) == (depth, id).
  std::stable_sort(order.begin(), order.end(),
                   [&](int32_t a, int32_t b) { return depth[a] < depth[b]; });
  std::vector<std::string> ids;
  ids.reserve(n);
  for (int32_t i : order) ids.push_back(ops_[i].id);
  return ids;
}

std::vector<std::string> Graph::worker_devices() const {  // sim.cpp:27-41
  std::set<std::string> d;
  for (const Op& op : ops_)
    if (op.kind == kRecv || op.kind == kSend || op.kind == kCompute) d.insert(op.res.device);
  return {d.begin(), d.end()};
}

std::shared_ptr<Graph> Graph::partition(const std::string& device) const {  // sim.cpp:43-59
  std::vector<Op> ops;
  std::set<std::string> kept;
  for (const Op& op : ops_)
    if (op.res.device == device) {
      ops.push_back(op);
      kept.insert(op.id);
    }
  if (ops.empty()) fail(kValidation, "no ops on device: " + device);
  std::vector<std::pair<std::string, std::string>> edges;
  for (const auto& e : edges_)
    if (kept.count(e.first) && kept.count(e.second)) edges.push_back(e);
  return make(name_ + "/" + device, false, std::move(ops), std::move(edges));
}

DeviceGraph* Graph::device() const {
  std::lock_guard<std::mutex> lock(dev_mu_);
  int cur = 0;
  if (cudaGetDevice(&cur) != cudaSuccess) cur = 0;
  DeviceGraph*& dg = dev_[cur];
  if (!dg) {
    std::vector<int8_t> kind(n()), chan(resources_.size());
    for (int32_t i = 0; i < n(); ++i) kind[i] = static_cast<int8_t>(ops_[i].kind);
    for (size_t r = 0; r < resources_.size(); ++r) chan[r] = resources_[r].channel ? 1 : 0;
    // device index per resource (devices sorted, as the chrome trace pids)
    std::vector<std::string> devs;
    for (const Resource& r : resources_) devs.push_back(r.device);
    std::sort(devs.begin(), devs.end());
    devs.erase(std::unique(devs.begin(), devs.end()), devs.end());
    std::vector<int32_t> rdev(resources_.size());
    for (size_t r = 0; r < resources_.size(); ++r)
      rdev[r] = static_cast<int32_t>(std::lower_bound(devs.begin(), devs.end(), resources_[r].device) -
                                     devs.begin());
    char err[256] = {0};
    dg = csk_graph_upload(n(), pred_off_.data(), pred_idx_.data(), succ_off_.data(),
                          succ_idx_.data(), kind.data(), res_of_.data(),
                          static_cast<int32_t>(resources_.size()), chan.data(), rdev.data(),
                          static_cast<int32_t>(devs.size()), err);
    if (!dg) {
      dev_.erase(cur);
      fail(kInternal, err);
    }
  }
  return dg;
}

}  // namespace tictac
