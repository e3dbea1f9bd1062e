// DeviceGraph layout shared by the kernels (see graph.cu).
#pragma once

#include <cstdint>
#include <memory>
#include <mutex>
#include <vector>

// Row structure of the dependency closure (props.cu): ops grouped into rows
// with identical recv-ancestor sets. Graph-only, so built once per handle.
struct Rows {
  int32_t nrows = 0, W = 1;             // W = 32-bit words per row
  std::vector<int32_t> row_of;          // per op
  std::vector<int32_t> self_col;        // per row: recv column or -1
  std::vector<int32_t> pre_off, pre;    // per row: predecessor rows
  std::vector<int32_t> succ_off, succ;  // per recv column: direct-successor rows (TAC)
  std::vector<int32_t> g1;              // per recv column: its one direct-successor row, -1 several, -2 none
  // Rows with predecessor rows, in topological order, and their closure
  // terms encoded for closure_seq_kernel: -1 = the previous such row (kept
  // in a register); -(2 + q) followed by a mask = bits of word q contributed
  // directly (the row's own column and predecessor rows without predecessors
  // of their own); else a row index.
  std::vector<int32_t> nt_row, nt_off, nt_term;
  std::vector<int32_t> nt_chunk;  // row ranges staged through shared memory together
  std::vector<int32_t> has_rows;  // rows with compute members (column-list entries), ascending
  // device copies of the arrays above (uploaded with the structure, freed
  // with the graph by csk_graph_free)
  int32_t *d_self = nullptr, *d_preoff = nullptr, *d_pre = nullptr, *d_rowof = nullptr, *d_succoff = nullptr,
          *d_succ = nullptr, *d_ntrow = nullptr, *d_ntoff = nullptr, *d_ntterm = nullptr, *d_ntchunk = nullptr,
          *d_hasrows = nullptr, *d_g1 = nullptr;
};

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
  std::mutex rows_mu;
  std::shared_ptr<const Rows> rows;  // built on first use (props.cu)
};
