// Host-side input builders: model-replica cluster expansion (reference
// cluster.cpp:12-89), the reference's synthetic generators (synthetic.cpp)
// and the model-shaped DAGs of the benchmark configs (new).
// These build graphs once; they are not on the per-ordering hot path.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <numeric>

#include "core.hpp"
#include "rng_host.hpp"

namespace tictac {

std::shared_ptr<Graph> expand_mr(const Graph& worker, int nw, int nps, int64_t ps_us) {
  if (nw < 1) fail(kParameter, "n_workers must be positive");
  if (nps < 1) fail(kParameter, "n_ps must be positive");
  if (ps_us < 0) fail(kParameter, "ps_op_time must be >= 0");
  if (worker.cluster()) fail(kParameter, "expansion needs a worker graph");
  for (const Op& op : worker.ops())
    if (op.kind == kSend) fail(kParameter, "worker graph with send ops not supported: " + op.id);

  const std::vector<std::string> params = worker.recv_ids();
  std::unordered_map<std::string, size_t> param_of;
  for (size_t p = 0; p < params.size(); ++p) param_of[params[p]] = p;
  auto ps_name = [&](size_t p) { return std::to_string(static_cast<int>(p % nps)); };

  // Gradient pushes hang off the compute sinks (all sinks if none compute).
  std::vector<std::string> sources;
  for (int32_t i = 0; i < worker.n(); ++i)
    if (worker.nsucc(i) == 0 && worker.ops()[i].kind == kCompute)
      sources.push_back(worker.ops()[i].id);
  if (sources.empty())
    for (int32_t i = 0; i < worker.n(); ++i)
      if (worker.nsucc(i) == 0) sources.push_back(worker.ops()[i].id);

  std::vector<Op> ops;
  std::vector<std::pair<std::string, std::string>> edges;
  for (int w = 0; w < nw; ++w) {
    const std::string dev = "w" + std::to_string(w), pre = dev + "/";
    for (const Op& op : worker.ops()) {
      Op c = op;
      c.id = pre + op.id;
      c.res.device = dev;
      if (op.kind == kRecv) c.res.name = dev + "-ps" + ps_name(param_of.at(op.id));
      ops.push_back(std::move(c));
    }
    for (const auto& [a, b] : worker.edges()) edges.emplace_back(pre + a, pre + b);
    for (size_t p = 0; p < params.size(); ++p) {
      const Op& orig = worker.ops()[worker.at(params[p])];
      Op grad;
      grad.id = pre + "grad/" + orig.id;
      grad.kind = kSend;
      grad.res = Resource{dev, true, dev + "-ps" + ps_name(p)};
      grad.time_us = orig.time_us;
      grad.bytes = orig.bytes;
      ops.push_back(std::move(grad));
      for (const std::string& s : sources) edges.emplace_back(pre + s, pre + "grad/" + orig.id);
    }
  }
  for (size_t p = 0; p < params.size(); ++p) {
    const std::string& rid = params[p];
    const std::string psdev = "ps" + ps_name(p);
    const Resource cpu{psdev, false, "cpu0"};
    const std::string agg = psdev + "/agg/" + rid, upd = psdev + "/upd/" + rid,
                      read = psdev + "/read/" + rid;
    ops.push_back(Op{agg, kPsAggregate, cpu, ps_us, std::nullopt});
    ops.push_back(Op{upd, kPsUpdate, cpu, ps_us, std::nullopt});
    ops.push_back(Op{read, kPsRead, cpu, ps_us, std::nullopt});
    for (int w = 0; w < nw; ++w) edges.emplace_back("w" + std::to_string(w) + "/grad/" + rid, agg);
    edges.emplace_back(agg, upd);
    edges.emplace_back(upd, read);
  }
  return Graph::make(worker.name() + "-mr" + std::to_string(nw) + "x" + std::to_string(nps), true,
                     std::move(ops), std::move(edges));
}

// ---- reference synthetic generators (synthetic.cpp:14-179) --------------

static std::string padded(const char* prefix, size_t i, size_t count) {
  size_t width = 3;
  for (size_t hi = 1000; hi < count; hi *= 10) ++width;
  char buf[48];
  std::snprintf(buf, sizeof buf, "%s%0*zu", prefix, static_cast<int>(width), i);
  return buf;
}

namespace {
struct Block {
  std::vector<size_t> src, snk;
};
Block compose(size_t lo, size_t hi, HostRng& rng, std::vector<std::pair<size_t, size_t>>& out) {
  if (hi - lo == 1) return Block{{lo}, {lo}};
  const size_t split = lo + 1 + static_cast<size_t>(rng.bounded(hi - lo - 1));
  const bool series = rng.bounded(2) == 0;
  Block l = compose(lo, split, rng, out);
  Block r = compose(split, hi, rng, out);
  if (series) {
    for (size_t a : l.snk)
      for (size_t b : r.src) out.emplace_back(a, b);
    return Block{std::move(l.src), std::move(r.snk)};
  }
  Block m;
  std::merge(l.src.begin(), l.src.end(), r.src.begin(), r.src.end(), std::back_inserter(m.src));
  std::merge(l.snk.begin(), l.snk.end(), r.snk.begin(), r.snk.end(), std::back_inserter(m.snk));
  return m;
}
}  // namespace

std::shared_ptr<Graph> generate_synthetic(const std::string& shape, int layers, int params,
                                          const std::string& ratio_text, uint64_t seed) {
  int kind;
  if (shape == "chain") kind = 0;
  else if (shape == "layered") kind = 1;
  else if (shape == "seriesparallel") kind = 2;
  else fail(kParameter, "unknown shape: " + shape);
  Rational ratio;
  try {
    ratio = Rational::parse(ratio_text);
  } catch (const std::exception&) {
    fail(kParameter, "not a ratio: " + ratio_text);
  }
  if (layers < 1) fail(kParameter, "layers must be positive");
  if (params < 1) fail(kParameter, "params_per_layer must be positive");
  if (ratio.num <= 0) fail(kParameter, "comm_comp_ratio must be positive");

  const size_t nr = static_cast<size_t>(layers) * static_cast<size_t>(params);
  HostRng rng(seed);
  size_t nc = 0;
  std::vector<std::pair<size_t, size_t>> cedges, redges;
  if (kind == 0) {
    nc = nr;
    for (size_t i = 0; i < nc; ++i) {
      redges.emplace_back(i, i);
      if (i) cedges.emplace_back(i - 1, i);
    }
  } else if (kind == 1) {
    nc = static_cast<size_t>(layers);
    for (size_t l = 0; l < nc; ++l) {
      for (int k = 0; k < params; ++k) redges.emplace_back(l * static_cast<size_t>(params) + k, l);
      if (l) cedges.emplace_back(l - 1, l);
    }
  } else {
    nc = nr;
    for (size_t i = 0; i < nc; ++i) redges.emplace_back(i, i);
    compose(0, nc, rng, cedges);
  }
  std::vector<int64_t> ct(nc);
  for (auto& t : ct) t = 500 + static_cast<int64_t>(rng.bounded(1000));
  const int64_t total = std::accumulate(ct.begin(), ct.end(), int64_t{0});
  const int64_t rn = ratio.num, rd = ratio.den;
  const int64_t target = (2 * total * rn + rd) / (2 * rd);
  const int64_t drift = target * rd > total * rn ? target * rd - total * rn : total * rn - target * rd;
  if (100 * drift > total * rn)
    fail(kParameter, "comm_comp_ratio unachievable within 1% at integer microseconds");
  // Largest-remainder apportioning of the channel total, ties to lower index.
  std::vector<int64_t> wts(nr);
  for (auto& w : wts) w = 1 + static_cast<int64_t>(rng.bounded(1000));
  const int64_t tw = std::accumulate(wts.begin(), wts.end(), int64_t{0});
  std::vector<int64_t> rt(nr);
  std::vector<std::pair<int64_t, size_t>> rem;
  int64_t assigned = 0;
  for (size_t i = 0; i < nr; ++i) {
    rt[i] = target * wts[i] / tw;
    assigned += rt[i];
    rem.emplace_back(target * wts[i] % tw, i);
  }
  std::sort(rem.begin(), rem.end(), [](const auto& a, const auto& b) {
    return a.first != b.first ? a.first > b.first : a.second < b.second;
  });
  for (int64_t k = 0; k < target - assigned; ++k) ++rt[rem[static_cast<size_t>(k)].second];

  const Resource chan{"w0", true, "net0"}, cpu{"w0", false, "cpu0"};
  std::vector<Op> ops;
  for (size_t i = 0; i < nr; ++i) ops.push_back(Op{padded("recv", i, nr), kRecv, chan, rt[i], std::nullopt});
  for (size_t i = 0; i < nc; ++i) ops.push_back(Op{padded("comp", i, nc), kCompute, cpu, ct[i], std::nullopt});
  std::vector<std::pair<std::string, std::string>> edges;
  for (auto [r, c] : redges) edges.emplace_back(padded("recv", r, nr), padded("comp", c, nc));
  for (auto [a, b] : cedges) edges.emplace_back(padded("comp", a, nc), padded("comp", b, nc));
  static const char* const names[] = {"chain", "layered", "seriesparallel"};
  char name[160];
  std::snprintf(name, sizeof name, "%s-l%d-k%d-r%lld-%lld-s%llu", names[kind], layers, params,
                static_cast<long long>(rn), static_cast<long long>(rd),
                static_cast<unsigned long long>(seed));
  return Graph::make(name, false, std::move(ops), std::move(edges));
}

// ---- model-shaped worker DAGs (new) ----------------------
//
// "Backbone" DAGs: one compute chain with a residual skip edge into every
// third op, recv roots attached evenly along the forward part, one channel
// w0/channel/net0 and one core w0/compute/cpu0. Recv bytes are log-uniform
// draws scaled to the paper's Table 1 parameter total and
// timed by the bandwidth oracle at 1250 B/us; compute times ~ U[500,1500)
// rescaled so the compute total equals the channel total at that bandwidth.
// Everything is drawn from one mt19937_64 stream seeded with `seed`.

namespace {
struct Shape {
  const char* name;
  int R, V;
  double mib;
  bool training;
};
const Shape kShapes[] = {
    {"resnet_v2_50_inference", 125, 1423, 97.45, false},
    {"resnet_v2_50_training", 125, 2813, 97.45, true},
    {"inception_v3_training", 196, 3672, 103.54, true},
    {"vgg16_training", 32, 758, 527.79, true},
    {"resnet_v2_101_training", 244, 5380, 169.86, true},
};

// VGG-16 parameter tensors (13 conv + 3 fc, weight then bias), elements.
std::vector<int64_t> vgg16_params() {
  const int convs[13][2] = {{3, 64},    {64, 64},   {64, 128},  {128, 128}, {128, 256},
                            {256, 256}, {256, 256}, {256, 512}, {512, 512}, {512, 512},
                            {512, 512}, {512, 512}, {512, 512}};
  std::vector<int64_t> p;
  for (auto& c : convs) {
    p.push_back(int64_t{9} * c[0] * c[1]);
    p.push_back(c[1]);
  }
  const int64_t fcs[3][2] = {{25088, 4096}, {4096, 4096}, {4096, 1000}};
  for (auto& f : fcs) {
    p.push_back(f[0] * f[1]);
    p.push_back(f[1]);
  }
  return p;  // 138,357,544 floats = 527.79 MiB
}
}  // namespace

std::shared_ptr<Graph> generate_model(const std::string& model, uint64_t seed) {
  const int64_t kBw = 1250;  // bytes per microsecond (10 Gb/s)
  HostRng rng(seed);
  int R = 0, V = 0;
  bool training = false;
  std::vector<int64_t> bytes;
  std::string name = model;
  bool layered = false, branchy = false;
  int64_t lay_v = 0, lay_r = 0;
  if (model.rfind("layered:", 0) == 0) {
    // layered:<V>:<R> — R/10 layers, 10 recvs feeding the head of a
    // (V/R*10 - 10)-compute chain per layer, layers linked head-to-tail.
    if (std::sscanf(model.c_str() + 8, "%lld:%lld", reinterpret_cast<long long*>(&lay_v),
                    reinterpret_cast<long long*>(&lay_r)) != 2 ||
        lay_r < 10 || lay_r % 10 || lay_v <= lay_r || (lay_v - lay_r) % (lay_r / 10))
      fail(kParameter, "bad layered model spec: " + model);
    layered = true;
    R = static_cast<int>(lay_r);
    V = static_cast<int>(lay_v);
  } else {
    // "<model>_branchy": the same recvs, bytes and compute times, arranged
    // as Inception-style modules (below) instead of a backbone chain.
    std::string base = model;
    const std::string suffix = "_branchy";
    if (base.size() > suffix.size() && base.compare(base.size() - suffix.size(), suffix.size(), suffix) == 0) {
      base.resize(base.size() - suffix.size());
      branchy = true;
    }
    const Shape* s = nullptr;
    for (const Shape& k : kShapes)
      if (base == k.name) s = &k;
    if (!s) fail(kParameter, "unknown model: " + model);
    R = s->R;
    V = s->V;
    training = s->training;
    const double total = s->mib * 1024.0 * 1024.0;
    if (base == "vgg16_training") {
      for (int64_t e : vgg16_params()) bytes.push_back(4 * e);
    } else {
      // log-uniform over [2^8, 2^24) bytes, then scaled to the total.
      std::vector<double> w(R);
      double sum = 0;
      for (auto& x : w) {
        x = std::exp2(8.0 + 16.0 * (static_cast<double>(rng.next() >> 11) * 0x1.0p-53));
        sum += x;
      }
      int64_t acc = 0;
      for (int i = 0; i < R; ++i) {
        const int64_t b = i + 1 < R ? static_cast<int64_t>(std::llround(w[i] / sum * total))
                                    : static_cast<int64_t>(std::llround(total)) - acc;
        bytes.push_back(std::max<int64_t>(b, 4));
        acc += bytes.back();
      }
    }
  }
  const int nc = V - R;
  std::vector<int64_t> ctime(nc);
  int64_t ctotal = 0, rtotal = 0;
  for (auto& t : ctime) ctotal += (t = 500 + static_cast<int64_t>(rng.bounded(1000)));
  std::vector<int64_t> rtime(R);
  if (layered) {
    for (auto& t : rtime) rtotal += (t = 500 + static_cast<int64_t>(rng.bounded(1000)));
  } else {
    for (int i = 0; i < R; ++i) rtotal += (rtime[i] = (2 * bytes[i] + kBw) / (2 * kBw));
  }
  // Rescale compute so its total matches the channel total (ratio 1).
  int64_t acc = 0;
  for (int i = 0; i < nc; ++i) {
    const int64_t t = i + 1 < nc ? static_cast<int64_t>(static_cast<__int128>(ctime[i]) * rtotal / ctotal)
                                 : rtotal - acc;
    ctime[i] = std::max<int64_t>(t, 0);
    acc += ctime[i];
  }

  const Resource chan{"w0", true, "net0"}, cpu{"w0", false, "cpu0"};
  std::vector<Op> ops;
  std::vector<std::pair<std::string, std::string>> edges;
  for (int i = 0; i < R; ++i) {
    Op op{padded("recv", i, R), kRecv, chan, rtime[i], std::nullopt};
    if (!layered) op.bytes = bytes[i];
    ops.push_back(std::move(op));
  }
  for (int i = 0; i < nc; ++i) ops.push_back(Op{padded("comp", i, nc), kCompute, cpu, ctime[i], std::nullopt});
  auto comp = [&](int i) { return padded("comp", i, nc); };
  if (layered) {
    const int per = nc / (R / 10);
    for (int l = 0; l < R / 10; ++l) {
      const int head = l * per;
      for (int k = 0; k < 10; ++k) edges.emplace_back(padded("recv", l * 10 + k, R), comp(head));
      for (int i = head + 1; i < head + per; ++i) edges.emplace_back(comp(i - 1), comp(i));
      if (l) edges.emplace_back(comp(head - 1), comp(head));
    }
    name = "layered-v" + std::to_string(V) + "-r" + std::to_string(R);
  } else if (branchy) {
    // Inception-style modules: split -> four parallel branches of 1, 3, 4
    // and 2 ops -> concat (12 ops), after a short stem chain. Recvs (one per
    // parameter tensor) attach evenly to the forward convolutions (stem and
    // branch ops, not split/concat), so ops in different branches of a
    // module depend on different recvs: recv-ancestor sets are not nested.
    // Training appends a mirrored backward pass whose branch ops also read
    // their forward counterpart's activations.
    constexpr int kBranch[4] = {1, 3, 4, 2};
    constexpr int kMod = 12;
    const int F = training ? std::max(1, nc / 2) : nc;
    std::vector<int> conv;  // forward convolutions, in order
    // lays out `count` ops starting at `first`; returns per-module op lists
    auto lay = [&](int first, int count, bool fwd, std::vector<std::vector<int>>* mods) {
      const int nm = count >= kMod + 8 ? (count - 8) / kMod : 0;
      const int stem = count - nm * kMod;
      int prev = -1;
      if (!fwd && first > 0) prev = first - 1;  // backward starts after the forward pass
      for (int i = first; i < first + stem; ++i) {
        if (prev >= 0) edges.emplace_back(comp(prev), comp(i));
        if (fwd) conv.push_back(i);
        prev = i;
      }
      int at = first + stem;
      for (int m = 0; m < nm; ++m) {
        std::vector<int> ids;
        const int split = at++;
        ids.push_back(split);
        if (prev >= 0) edges.emplace_back(comp(prev), comp(split));
        std::vector<int> tails;
        for (int b = 0; b < 4; ++b) {
          int p = split;
          for (int k = 0; k < kBranch[b]; ++k) {
            const int op = at++;
            ids.push_back(op);
            edges.emplace_back(comp(p), comp(op));
            if (fwd) conv.push_back(op);
            p = op;
          }
          tails.push_back(p);
        }
        const int cat = at++;
        ids.push_back(cat);
        for (int t : tails) edges.emplace_back(comp(t), comp(cat));
        prev = cat;
        if (mods) mods->push_back(std::move(ids));
      }
    };
    std::vector<std::vector<int>> fmods, bmods;
    lay(0, F, true, &fmods);
    if (nc > F) {
      lay(F, nc - F, false, &bmods);
      for (size_t m = 0; m < bmods.size() && m < fmods.size(); ++m) {
        const auto& f = fmods[fmods.size() - 1 - m];
        for (int k = 1; k + 1 < kMod; ++k) edges.emplace_back(comp(f[k]), comp(bmods[m][k]));
      }
    }
    const int ncv = static_cast<int>(conv.size());
    for (int i = 0; i < R; ++i)
      edges.emplace_back(padded("recv", i, R), comp(conv[static_cast<size_t>(int64_t{i} * ncv / R)]));
  } else {
    for (int i = 1; i < nc; ++i) {
      edges.emplace_back(comp(i - 1), comp(i));
      if (i % 3 == 0 && i >= 3) edges.emplace_back(comp(i - 3), comp(i));  // residual skip
    }
    // Recvs attach evenly over the forward half (training) or everything.
    const int span = training ? std::max(1, nc / 2) : nc;
    for (int i = 0; i < R; ++i)
      edges.emplace_back(padded("recv", i, R), comp(static_cast<int>(int64_t{i} * span / R)));
  }
  return Graph::make(name + "-s" + std::to_string(seed), false, std::move(ops), std::move(edges));
}

}  // namespace tictac
