// Batched sweep context shared by the C ABI (capi.cpp) and sweep.cpp.
#pragma once

#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../../include/commsched.h"
#include "core.hpp"

struct SweepPlan;  // device/csk.h

namespace tictac {

struct SweepCtx {
  std::shared_ptr<const Graph> g;
  std::vector<int64_t> dur;
  Policy policy;
  int64_t U = 0, L = 0;
  bool cluster = false, fast = false;
  bool noisy = false;  // gated with reorder noise: the sweep kernel applies it; explicit orders do not
  std::vector<std::string> workers;  // worker_devices() order (clusters)
  std::vector<int32_t> recv_worker;  // per recv column
  SweepPlan* plan = nullptr;
  int32_t R = 0, nc = 0;
  bool dag = false;  // general-DAG program (not nested chain classes)
  bool ps = false;   // cluster send phase (parameter-server ops take time)
  int32_t nch = 1;   // channels per worker (> 1: statistics sweeps only; explicit
                     // orders and single runs use the exact replica)
  int32_t joins = 0, slots = 0, prog_words = 0;
  std::string why;  // why the closed form does not apply
  int device = 0;   // CUDA ordinal the plan lives on
  // Closed-form makespan of one gate order (recv columns, rank order) on a
  // worker-graph plan: one kernel launch on small cached device buffers.
  int64_t order_makespan(const std::vector<int32_t>& order);
  ~SweepCtx();

 private:
  std::mutex mu_;
  int32_t* d_order_ = nullptr;
  int64_t* d_ms_ = nullptr;
};

std::unique_ptr<SweepCtx> make_sweep(std::shared_ptr<const Graph> g, const TimeOracle& o,
                                     const Policy& p);
void finish_stats(const SweepCtx& s, const int64_t* i64, const double* f64, uint64_t key_base,
                  cs_sweep_stats* out);
void sweep_exact(SweepCtx& s, uint64_t seed_lo, int64_t count, int64_t* makespans,
                 int64_t* worker_ms, cs_sweep_stats* stats);
// Accumulates `part` into `total` (first: total = part).
void merge_stats(cs_sweep_stats& total, const cs_sweep_stats& part, bool first);

// Combines per-device statistics buffers (CS_DSTATS layout) across devices
// in one collective; device 0's caller receives the reduced words.
struct DeviceReducer {
  virtual ~DeviceReducer() = default;
  virtual void reduce(int device, const int64_t* d_i64, const double* d_f64, int64_t* h_i64,
                      double* h_f64) const = 0;
};

// NCCL communicators over devices 0..n_devices-1 (process-lifetime, cached
// per count); `hold` keeps concurrent multi-GPU sweeps from interleaving
// collectives on the same communicators.
const DeviceReducer& nccl_reducer(int n_devices, std::unique_lock<std::mutex>& hold);

// Closed-form sweep of seeds [seed_lo, seed_lo + count) over ctxs (one
// plan per device, ctxs[d]->device its CUDA ordinal): contiguous shards,
// rounds of at most 2^key_bits seeds, statistics combined by `reducer`
// (needed when ctxs.size() > 1). Per-seed outputs go to the host buffers.
cs_sweep_stats sweep_fast(const std::vector<SweepCtx*>& ctxs, uint64_t seed_lo, int64_t count,
                          int64_t* makespans, int64_t* worker_ms, const DeviceReducer* reducer);

}  // namespace tictac
