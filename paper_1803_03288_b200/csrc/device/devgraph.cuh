// DeviceGraph layout shared by the kernels (see graph.cu).
#pragma once

#include <cstdint>
#include <vector>

struct DeviceGraph {
  int32_t n = 0, nres = 0, ndev = 0, R = 0, rb_words = 0;
  // device arrays
  int32_t *pred_off = nullptr, *pred_idx = nullptr, *succ_off = nullptr, *succ_idx = nullptr;
  int8_t* kind = nullptr;
  int32_t* res = nullptr;
  int8_t* chan = nullptr;
  int32_t* res_dev = nullptr;
  int32_t *rops_off = nullptr, *rops = nullptr, *lidx = nullptr, *rb_off = nullptr;
  int32_t *recv_ops = nullptr, *col = nullptr;
  // host mirrors (structure only)
  std::vector<int32_t> h_pred_off, h_pred_idx, h_succ_off, h_succ_idx, h_res, h_res_dev;
  std::vector<int8_t> h_kind, h_chan;
  std::vector<int32_t> h_recv_ops, h_col;
};
