// TIC / TAC / property kernels (reference properties.cpp:19-109,
// schedule.cpp:12-71) on the GPU.
//
// Design (restated on groups):
//  * Row aliasing: a non-recv op with exactly one predecessor has that
//    predecessor's dependency set, so it shares its row. Rows are built in
//    topological order; each row's recv-dependency bitset (bit c = recv
//    column c) is the OR of its predecessor rows (plus itself for recvs) —
//    `closure_*_kernel`, one thread per 32-bit word walking the rows.
//  * Groups = rows with at least one non-recv member. All members of a group
//    share cnt = |dep ∩ outstanding|, M = Σ T over it, and the owner (XOR of
//    columns when cnt == 1), so P and M+ fold over groups with weight
//    W_g = Σ T(members).
//  * Column lists col[c] = groups containing recv c (CSR) drive the literal
//    and amended M+ (min of M over col[c] with cnt ≥ 2 / ≥ 1) and TAC's
//    retire step (cnt−−, M −= T(c), xr ^= c over col[c]; P[owner] += W_g
//    when a group drops to one outstanding recv).
//  * TAC rounds run in one persistent kernel: amended M+ from each
//    outstanding recv's direct-successor groups (exact because recvs are
//    roots in every graph tac() sees), the reference's left fold as a
//    find-first-beater chain (exact for the non-transitive comparator;
//    SURVEY A.3), then the retire step. Variants by size: one block with the
//    state in shared memory (tac_smem_kernel; tac_kernel when it does not
//    fit), one 16-CTA cluster with DSMEM mins (tac_cluster_kernel), and
//    grid-wide cooperative kernels with register-resident candidates
//    (tac_own_kernel) or re-read candidates (tac_dist_kernel).
#include <cooperative_groups.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cub/cub.cuh>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "csk.h"
#include "devgraph.cuh"

namespace cg = cooperative_groups;

namespace tictac_dev {
namespace {

constexpr int64_t kInf = INT64_MAX;

// Per-call device arrays: stream-ordered allocations on the legacy stream
// (the pool keeps its reservation between calls, graph.cu).
struct DevArr {
  void* p = nullptr;
  DevArr() = default;
  DevArr(const DevArr&) = delete;
  ~DevArr() {
    if (p) cudaFreeAsync(p, 0);
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

template <typename T>
int alloc(DevArr& a, size_t count, char* err) {
  CK(cudaMallocAsync(&a.p, round16(sizeof(T) * (count ? count : 1)), 0));  // padded for bulk copies
  return 0;
}
template <typename T>
int put(DevArr& a, const std::vector<T>& v, char* err) {
  CK(cudaMallocAsync(&a.p, round16(sizeof(T) * (v.empty() ? 1 : v.size())), 0));
  if (!v.empty()) CK(cudaMemcpy(a.p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
  return 0;
}

// Host-side row structure (graph-only, O(V+E); cached on the graph handle).
constexpr int kSeqRows = 1024, kSeqTerms = 4096;  // closure_seq_kernel's shared-memory chunk

void build_rows(const DeviceGraph* g, Rows& rw) {
  const int32_t n = g->n;
  std::vector<int32_t> order, missing(n);
  order.reserve(n);
  for (int32_t i = 0; i < n; ++i)
    if ((missing[i] = g->h_pred_off[i + 1] - g->h_pred_off[i]) == 0) order.push_back(i);
  for (size_t h = 0; h < order.size(); ++h) {
    const int32_t v = order[h];
    for (int32_t e = g->h_succ_off[v]; e < g->h_succ_off[v + 1]; ++e)
      if (--missing[g->h_succ_idx[e]] == 0) order.push_back(g->h_succ_idx[e]);
  }
  rw.row_of.assign(n, -1);
  rw.pre_off.assign(1, 0);
  std::vector<int32_t> tmp;
  for (int32_t v : order) {
    const int32_t np = g->h_pred_off[v + 1] - g->h_pred_off[v];
    const bool recv = g->h_kind[v] == 1;
    if (!recv && np == 1) {
      rw.row_of[v] = rw.row_of[g->h_pred_idx[g->h_pred_off[v]]];
      continue;
    }
    tmp.clear();
    for (int32_t e = g->h_pred_off[v]; e < g->h_pred_off[v + 1]; ++e)
      tmp.push_back(rw.row_of[g->h_pred_idx[e]]);
    std::sort(tmp.begin(), tmp.end());
    tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
    if (!recv && tmp.size() == 1) {  // all preds share one row
      rw.row_of[v] = tmp[0];
      continue;
    }
    rw.row_of[v] = rw.nrows++;
    rw.self_col.push_back(recv ? g->h_col[v] : -1);
    rw.pre.insert(rw.pre.end(), tmp.begin(), tmp.end());
    rw.pre_off.push_back(static_cast<int32_t>(rw.pre.size()));
  }
  rw.nt_off.assign(1, 0);
  for (int32_t k = 0; k < rw.nrows; ++k) {
    if (rw.pre_off[k] == rw.pre_off[k + 1]) continue;
    const int32_t last = rw.nt_row.empty() ? -1 : rw.nt_row.back();
    tmp.clear();  // recv columns contributed directly: own column, root predecessor rows
    if (rw.self_col[k] >= 0) tmp.push_back(rw.self_col[k]);
    for (int32_t e = rw.pre_off[k]; e < rw.pre_off[k + 1]; ++e) {
      const int32_t p = rw.pre[e];
      if (p == last) rw.nt_term.push_back(-1);
      else if (rw.pre_off[p] != rw.pre_off[p + 1]) rw.nt_term.push_back(p);
      else if (rw.self_col[p] >= 0) tmp.push_back(rw.self_col[p]);
    }
    std::sort(tmp.begin(), tmp.end());
    for (size_t a = 0; a < tmp.size();) {  // one (word, mask) pair per word touched
      const int32_t q = tmp[a] >> 5;
      uint32_t mask = 0;
      for (; a < tmp.size() && (tmp[a] >> 5) == q; ++a) mask |= 1u << (tmp[a] & 31);
      rw.nt_term.push_back(-2 - q);
      rw.nt_term.push_back(static_cast<int32_t>(mask));
    }
    rw.nt_row.push_back(k);
    rw.nt_off.push_back(static_cast<int32_t>(rw.nt_term.size()));
  }
  {
    std::vector<uint8_t> has(rw.nrows, 0);
    for (int32_t v = 0; v < n; ++v)
      if (g->h_kind[v] != 1) has[rw.row_of[v]] = 1;
    for (int32_t k = 0; k < rw.nrows; ++k)
      if (has[k]) rw.has_rows.push_back(k);
  }
  const int32_t n_nt = static_cast<int32_t>(rw.nt_row.size());
  rw.nt_chunk.assign(1, 0);
  for (int32_t i = 0; i < n_nt;) {  // <= kSeqRows rows and <= kSeqTerms terms (or one oversized row)
    int32_t j = i + 1;
    while (j < n_nt && j - i < kSeqRows && rw.nt_off[j + 1] - rw.nt_off[i] <= kSeqTerms) ++j;
    rw.nt_chunk.push_back(j);
    i = j;
  }
  rw.W = std::max(1, (g->R + 31) / 32);
  rw.succ_off.assign(1, 0);
  for (int32_t c = 0; c < g->R; ++c) {
    const int32_t r = g->h_recv_ops[c];
    tmp.clear();
    for (int32_t e = g->h_succ_off[r]; e < g->h_succ_off[r + 1]; ++e)
      if (g->h_kind[g->h_succ_idx[e]] != 1) tmp.push_back(rw.row_of[g->h_succ_idx[e]]);
    std::sort(tmp.begin(), tmp.end());
    tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
    rw.succ.insert(rw.succ.end(), tmp.begin(), tmp.end());
    rw.succ_off.push_back(static_cast<int32_t>(rw.succ.size()));
    rw.g1.push_back(tmp.size() == 1 ? tmp[0] : (tmp.empty() ? -2 : -1));
  }
}

// ---- closure: thread q owns word q of every row; rows in topo order ------
__global__ void closure_smem_kernel(int32_t nrows, int32_t W, const int32_t* __restrict__ self_col,
                                    const int32_t* __restrict__ pre_off,
                                    const int32_t* __restrict__ pre, uint32_t* __restrict__ out) {
  extern __shared__ uint32_t sm[];
  for (int q = threadIdx.x; q < W; q += blockDim.x) {
    for (int32_t k = 0; k < nrows; ++k) {
      uint32_t w = 0;
      for (int32_t e = pre_off[k]; e < pre_off[k + 1]; ++e) w |= sm[pre[e] * W + q];
      const int32_t c = self_col[k];
      if (c >= 0 && (c >> 5) == q) w |= 1u << (c & 31);
      sm[k * W + q] = w;
    }
  }
  __syncthreads();
  for (int64_t i = threadIdx.x; i < static_cast<int64_t>(nrows) * W; i += blockDim.x) out[i] = sm[i];
}

// Large closures: rows without predecessor rows hold their own bit only and
// are written by one parallel pass; the rows with predecessors follow in
// topological order, thread q owning word q, with the previous such row's
// word in a register and bits of root rows folded in from their column — so
// on backbone/layered DAGs the sequential pass reads no closure words at all.
__global__ void closure_roots_kernel(int32_t nrows, int32_t W, const int32_t* __restrict__ self_col,
                                     const int32_t* __restrict__ pre_off, uint32_t* __restrict__ out) {
  for (int32_t k = blockIdx.x; k < nrows; k += gridDim.x) {
    if (pre_off[k] != pre_off[k + 1]) continue;
    const int32_t c = self_col[k];
    for (int32_t q = threadIdx.x; q < W; q += blockDim.x)
      out[static_cast<int64_t>(k) * W + q] = c >= 0 && (c >> 5) == q ? 1u << (c & 31) : 0u;
  }
}

__global__ void __launch_bounds__(128) closure_seq_kernel(int32_t n_chunks, int32_t W,
                                                          const int32_t* __restrict__ chunk,
                                                          const int32_t* __restrict__ nt_row,
                                                          const int32_t* __restrict__ nt_off,
                                                          const int32_t* __restrict__ nt_term,
                                                          uint32_t* __restrict__ out) {
  // the row metadata is the same for every word: each chunk of rows is
  // staged once per block, then every thread walks it from shared memory
  __shared__ int32_t s_off[kSeqRows + 1], s_row[kSeqRows], s_term[kSeqTerms];
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t carry = 0;
  for (int32_t h = 0; h < n_chunks; ++h) {
    const int32_t i0 = chunk[h], i1 = chunk[h + 1], base = nt_off[i0];
    const int32_t nterm = nt_off[i1] - base;
    const bool staged = nterm <= kSeqTerms;
    for (int32_t j = threadIdx.x; j <= i1 - i0; j += blockDim.x) s_off[j] = nt_off[i0 + j] - base;
    for (int32_t j = threadIdx.x; j < i1 - i0; j += blockDim.x) s_row[j] = nt_row[i0 + j];
    if (staged)
      for (int32_t j = threadIdx.x; j < nterm; j += blockDim.x) s_term[j] = nt_term[base + j];
    __syncthreads();
    if (q < W) {
      const int32_t* term = staged ? s_term : nt_term + base;
      for (int32_t j = 0; j < i1 - i0; ++j) {
        uint32_t w = 0;
        const int32_t e1 = s_off[j + 1];
        for (int32_t e = s_off[j]; e < e1; ++e) {
          const int32_t p = term[e];
          if (p == -1) {
            w |= carry;
          } else if (p < -1) {  // (word, mask) pair
            ++e;
            if (-2 - p == q) w |= static_cast<uint32_t>(term[e]);
          } else {
            w |= out[static_cast<int64_t>(p) * W + q];
          }
        }
        out[static_cast<int64_t>(s_row[j]) * W + q] = w;
        carry = w;
      }
    }
    __syncthreads();
  }
}

// Group weights W_g = Σ T(non-recv member); has[g] marks groups.
__global__ void weights_kernel(int32_t n, const int32_t* __restrict__ row_of,
                               const int8_t* __restrict__ kind, const int64_t* __restrict__ dur,
                               unsigned long long* __restrict__ wsum, int32_t* __restrict__ has) {
  for (int32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    if (kind[v] == 1) continue;
    atomicAdd(&wsum[row_of[v]], static_cast<unsigned long long>(dur[v]));
    has[row_of[v]] = 1;
  }
}

// Per row (warp): cnt, M, xr with every recv outstanding. Rows without
// predecessor rows hold at most their own column: no scan.
__global__ void rowstate_kernel(int32_t nrows, int32_t W, const uint32_t* __restrict__ bits,
                                const int32_t* __restrict__ pre_off, const int32_t* __restrict__ self_col,
                                const int64_t* __restrict__ tcol, const int32_t* __restrict__ has,
                                int32_t* __restrict__ cnt, int64_t* __restrict__ M,
                                int32_t* __restrict__ xr) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t k = wid; k < nrows; k += nw) {
    if (pre_off[k] == pre_off[k + 1]) {
      if (lane == 0) {
        const int32_t c = self_col[k];
        cnt[k] = c >= 0;
        M[k] = c >= 0 ? tcol[c] : 0;
        xr[k] = c >= 0 ? c : 0;
      }
      continue;
    }
    int c_cnt = 0, c_xr = 0;
    int64_t m = 0;
    for (int q = lane; q < W; q += 32) {
      uint32_t w = bits[k * W + q];
      while (w) {
        const int c = (q << 5) + __ffs(w) - 1;
        w &= w - 1;
        ++c_cnt;
        c_xr ^= c;
        m += tcol[c];
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      c_cnt += __shfl_xor_sync(~0u, c_cnt, o);
      c_xr ^= __shfl_xor_sync(~0u, c_xr, o);
      m += __shfl_xor_sync(~0u, m, o);
    }
    if (lane == 0) {
      cnt[k] = c_cnt;
      M[k] = m;
      xr[k] = c_xr;
    }
  }
}

// Column lists (recv column -> rows with compute members whose closure holds
// it) without atomics. A warp owns one closure word q (32 columns) over one
// chunk of the rows with compute members and walks it 32 rows at a time:
// lane i loads row i's word, and per column j a ballot gives the rows that
// hold it. Pass 1 counts per (chunk, column); a per-column scan over chunks
// turns counts into offsets; pass 2 writes each ballot as one contiguous run,
// so every list comes out in ascending row order with coalesced stores.
__global__ void colcount_warp_kernel(int32_t nhas, int32_t W, int32_t R, int32_t nchunks, int32_t chunk_rows,
                                     const uint32_t* __restrict__ bits, const int32_t* __restrict__ has_rows,
                                     int32_t* __restrict__ counts) {
  const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wid >= static_cast<int64_t>(W) * nchunks) return;
  const int q = static_cast<int>(wid % W), h = static_cast<int>(wid / W);
  const int32_t i1 = min(nhas, (h + 1) * chunk_rows);
  int32_t cnt = 0;
  for (int32_t i0 = h * chunk_rows; i0 < i1; i0 += 32) {
    const int32_t i = i0 + lane;
    const uint32_t w = i < i1 ? bits[static_cast<int64_t>(has_rows[i]) * W + q] : 0u;
#pragma unroll 8
    for (int j = 0; j < 32; ++j) {
      const uint32_t b = __ballot_sync(~0u, (w >> j) & 1u);
      if (lane == j) cnt += __popc(b);
    }
  }
  const int c = q * 32 + lane;
  if (c < R) counts[static_cast<int64_t>(h) * R + c] = cnt;
}

__global__ void colprefix_kernel(int32_t R, int32_t nchunks, int32_t* __restrict__ counts,
                                 int32_t* __restrict__ colcount) {
  for (int32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < R; c += gridDim.x * blockDim.x) {
    int32_t run = 0;
    for (int32_t h = 0; h < nchunks; ++h) {
      int32_t* p = counts + static_cast<int64_t>(h) * R + c;
      const int32_t v = *p;
      *p = run;
      run += v;
    }
    colcount[c] = run;
  }
}

__global__ void colfill_warp_kernel(int32_t nhas, int32_t W, int32_t R, int32_t nchunks, int32_t chunk_rows,
                                    const uint32_t* __restrict__ bits, const int32_t* __restrict__ has_rows,
                                    const int32_t* __restrict__ counts, const int32_t* __restrict__ coloff,
                                    int32_t* __restrict__ col) {
  const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wid >= static_cast<int64_t>(W) * nchunks) return;
  const int q = static_cast<int>(wid % W), h = static_cast<int>(wid / W);
  const int32_t i1 = min(nhas, (h + 1) * chunk_rows);
  const int c = q * 32 + lane;
  int32_t pos = c < R ? coloff[c] + counts[static_cast<int64_t>(h) * R + c] : 0;  // lane j: column q*32+j
  const uint32_t below = (1u << lane) - 1u;
  for (int32_t i0 = h * chunk_rows; i0 < i1; i0 += 32) {
    const int32_t i = i0 + lane;
    const int32_t k = i < i1 ? has_rows[i] : 0;
    const uint32_t w = i < i1 ? bits[static_cast<int64_t>(k) * W + q] : 0u;
#pragma unroll 4
    for (int j = 0; j < 32; ++j) {
      const uint32_t b = __ballot_sync(~0u, (w >> j) & 1u);
      if (!b) continue;
      const int32_t at = __shfl_sync(~0u, pos, j);
      if ((w >> j) & 1u) col[at + __popc(b & below)] = k;
      if (lane == j) pos += __popc(b);
    }
  }
}

// P and M+ with every recv outstanding (properties.cpp:92-107 on groups):
// a warp per recv column, lanes striding its (ascending) row list.
__global__ void props_kernel(int32_t R, int amended, const int32_t* __restrict__ col_off,
                             const int32_t* __restrict__ col, const int32_t* __restrict__ cnt,
                             const int64_t* __restrict__ M, const int32_t* __restrict__ xr,
                             const unsigned long long* __restrict__ wsum, int64_t* __restrict__ P,
                             int64_t* __restrict__ Mp) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t c = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; c < R; c += nw) {
    int64_t mp = kInf, p = 0;
    for (int32_t e = col_off[c] + lane; e < col_off[c + 1]; e += 32) {
      const int32_t g = col[e];
      const int k = cnt[g];
      if (k >= 2 || (amended && k == 1)) mp = min(mp, M[g]);
      if (k == 1 && xr[g] == c) p += static_cast<int64_t>(wsum[g]);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      p += __shfl_xor_sync(~0u, p, o);
      mp = min(mp, __shfl_xor_sync(~0u, mp, o));
    }
    if (lane == 0) {
      P[c] = p;
      Mp[c] = mp;
    }
  }
}

inline int props_blocks(int32_t R) { return std::max(1, std::min((R * 32 + 255) / 256, 148 * 16)); }

// precedes (schedule.cpp:12-19); kInf = nullopt sorts last.
__device__ __forceinline__ bool precedes(int a, int64_t ap, int64_t am, int64_t amp, int b, int64_t bp,
                                         int64_t bm, int64_t bmp) {
  const int64_t ab = min(bp, am), ba = min(ap, bm);
  if (ab != ba) return ab < ba;
  if (amp != bmp) return amp < bmp;
  return a < b;
}

struct TacArgs {
  int32_t R;
  const int64_t* tcol;      // T(recv column)
  const int32_t* succ_off;  // direct-successor groups per column
  const int32_t* succ;
  const int32_t* g1;        // per column: its one direct-successor group, -1 several, -2 none
  const int32_t* col_off;   // groups per column
  const int32_t* col;
  const unsigned long long* wsum;
  int32_t* cnt;
  int64_t* M;
  int32_t* xr;
  int64_t* P;
  int64_t* mp;
  uint8_t* out;
  int32_t* prio;
};

// Block-wide min with one barrier: warp min, one shared atomicMin per warp
// into slot sp % 3 of a ring; the slot for the next call is reset now (its
// last readers finished before the previous call's barrier). `red` holds
// the 3 slots (all 0x7fffffff at kernel start); `sp` is block-uniform.
__device__ __forceinline__ int block_min_int(int v, int* red, int& sp) {
  v = __reduce_min_sync(~0u, v);
  if ((threadIdx.x & 31) == 0 && v != 0x7fffffff) atomicMin(&red[sp % 3], v);
  if (threadIdx.x == 0) red[(sp + 1) % 3] = 0x7fffffff;
  __syncthreads();
  const int r = *reinterpret_cast<volatile int*>(&red[sp % 3]);
  ++sp;
  return r;
}

__device__ __forceinline__ void init_red(int* red) {
  if (threadIdx.x < 3) red[threadIdx.x] = 0x7fffffff;
  __syncthreads();
}

// A one-block cooperative grid only needs a block barrier.
__device__ __forceinline__ void grid_bar(cg::grid_group& grid) {
  if (gridDim.x == 1)
    __syncthreads();
  else
    grid.sync();
}

// The R rounds of one-block TAC (phases A-C below) over the state `a` points
// at — global memory (tac_kernel) or a shared-memory copy (tac_smem_kernel).
// Three kinds of block barrier per round: the first block-wide min (which also
// publishes phase A's M+), one per find-first step (the last one orders every
// read of P/out/M+ before the retire writes them), and one after the retire.
template <typename ColT>
__device__ __forceinline__ void tac_rounds(const TacArgs& a, const ColT* __restrict__ col, int* red, int& sp) {
  const int R = a.R;
  for (int round = 0; round < R; ++round) {
    // Phase A: amended M+ of every outstanding recv = min M over its
    // direct-successor groups; the lowest outstanding column.
    int first = 0x7fffffff;
    for (int c = threadIdx.x; c < R; c += blockDim.x) {
      if (!a.out[c]) continue;
      int64_t m = kInf;
      for (int32_t e = a.succ_off[c]; e < a.succ_off[c + 1]; ++e) m = min(m, a.M[a.succ[e]]);
      a.mp[c] = m;
      first = min(first, c);
    }
    // Phase B: the reference's left fold over outstanding recvs in id order
    // == find-first-beater chain.
    int best = block_min_int(first, red, sp);
    for (;;) {
      const int64_t bp = a.P[best], bm = a.tcol[best], bmp = a.mp[best];
      int nxt = 0x7fffffff;
      for (int c = best + 1 + threadIdx.x; c < R; c += blockDim.x)
        if (a.out[c] && precedes(c, a.P[c], a.tcol[c], a.mp[c], best, bp, bm, bmp)) {
          nxt = c;
          break;
        }
      nxt = block_min_int(nxt, red, sp);
      if (nxt == 0x7fffffff) break;
      best = nxt;
    }
    // Phase C: retire `best`.
    const int64_t t = a.tcol[best];
    for (int32_t e = a.col_off[best] + threadIdx.x; e < a.col_off[best + 1]; e += blockDim.x) {
      const int32_t g = col[e];
      const int k = --a.cnt[g];
      a.M[g] -= t;
      const int x = (a.xr[g] ^= best);
      if (k == 1) atomicAdd(reinterpret_cast<unsigned long long*>(&a.P[x]), a.wsum[g]);
    }
    if (threadIdx.x == 0) {
      a.prio[best] = round;
      a.out[best] = 0;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(1024) tac_kernel(TacArgs a) {  // one block
  __shared__ int red[3];
  int sp = 0;
  init_red(red);
  tac_rounds(a, a.col, red, sp);
}

// Shared-memory bytes of tac_smem_kernel's state copy.
// (every array 16-byte aligned and padded: each is one bulk copy)
__host__ __device__ inline size_t tac_smem_bytes(int nrows, int R, int nsucc) {
  return 2 * round16(8ull * nrows) + 3 * round16(8ull * R) + 2 * round16(4ull * nrows) +
         2 * round16(4ull * (R + 1)) + round16(4ull * nsucc) + round16(R);
}
// plus the column lists as 16-bit row ids, when they fit (ncol > 0)
__host__ __device__ inline size_t tac_smem_col_bytes(int64_t ncol) { return (2ull * ncol + 15) & ~size_t(15); }

// One block with every per-round array in shared memory: the rounds' dependent
// reads of values other threads just wrote (M, cnt, xr, P, mp, out) cost a
// shared-memory round trip instead of an L2 one. Column lists (the retire
// work lists) and prio stay in global memory.
__global__ void __launch_bounds__(1024) tac_smem_kernel(TacArgs g, int nrows, int nsucc, int ncol) {
  extern __shared__ __align__(16) char tac_sm[];
  __shared__ int red[3];
  int sp = 0;
  const int R = g.R;
  char* q = tac_sm;
  auto* col16 = reinterpret_cast<uint16_t*>(q);  // first: 16-byte aligned
  q += ncol > 0 ? tac_smem_col_bytes(ncol) : 0;
  for (int e = threadIdx.x; e < ncol; e += blockDim.x) col16[e] = static_cast<uint16_t>(g.col[e]);
  // Every array arrives by one bulk copy on the TMA engine (device
  // allocations are padded to 16 bytes, DevArr), all on one mbarrier.
  __shared__ uint64_t staged;
  if (threadIdx.x == 0) mbar_init(&staged, 1);
  __syncthreads();
  uint32_t total = 0;
  auto take = [&](const void* src, size_t bytes) {
    char* p = q;
    const uint32_t b = static_cast<uint32_t>(round16(bytes));
    q += b;
    if (threadIdx.x == 0 && b > 0) bulk_g2s(p, src, b, &staged);
    total += b;
    return p;
  };
  if (threadIdx.x == 0) mbar_expect_tx(&staged, static_cast<uint32_t>(tac_smem_bytes(nrows, R, nsucc)));
  auto* M = reinterpret_cast<int64_t*>(take(g.M, 8ull * nrows));
  auto* wsum = reinterpret_cast<unsigned long long*>(take(g.wsum, 8ull * nrows));
  auto* P = reinterpret_cast<int64_t*>(take(g.P, 8ull * R));
  auto* mp = reinterpret_cast<int64_t*>(take(g.mp, 8ull * R));
  auto* tcol = reinterpret_cast<int64_t*>(take(g.tcol, 8ull * R));
  auto* cnt = reinterpret_cast<int32_t*>(take(g.cnt, 4ull * nrows));
  auto* xr = reinterpret_cast<int32_t*>(take(g.xr, 4ull * nrows));
  auto* succ_off = reinterpret_cast<int32_t*>(take(g.succ_off, 4ull * (R + 1)));
  auto* col_off = reinterpret_cast<int32_t*>(take(g.col_off, 4ull * (R + 1)));
  auto* succ = reinterpret_cast<int32_t*>(take(g.succ, 4ull * nsucc));
  auto* out = reinterpret_cast<uint8_t*>(take(g.out, R));
  (void)total;
  mbar_wait(&staged, 0);
  init_red(red);  // also the barrier after the column-list conversion
  TacArgs a = g;
  a.tcol = tcol;
  a.succ_off = succ_off;
  a.col_off = col_off;
  a.succ = succ;
  a.wsum = wsum;
  a.cnt = cnt;
  a.M = M;
  a.xr = xr;
  a.P = P;
  a.mp = mp;
  a.out = out;
  if (ncol > 0)
    tac_rounds(a, col16, red, sp);
  else
    tac_rounds(a, a.col, red, sp);
}

// Multi-block TAC: the selection fold is distributed too. Every find-first
// step is a grid-wide min (per-block reduction + atomicMin into a 3-slot
// ring; the slot for step p+1 is reset during step p, two barriers after its
// last reader). Rounds cost (chain length + 3) grid barriers but the O(R_t)
// candidate scan is spread over every SM instead of repeated per block.
__device__ __forceinline__ int grid_min_step(int v, int* ring, int& p, int* red, int& sp,
                                             cg::grid_group& grid) {
  v = block_min_int(v, red, sp);
  if (threadIdx.x == 0 && v != 0x7fffffff) atomicMin(&ring[p % 3], v);
  if (blockIdx.x == 0 && threadIdx.x == 0) ring[(p + 1) % 3] = 0x7fffffff;
  grid.sync();
  const int r = *reinterpret_cast<volatile int*>(&ring[p % 3]);
  ++p;
  return r;
}

__global__ void __launch_bounds__(1024) tac_dist_kernel(TacArgs a, int* ring) {
  cg::grid_group grid = cg::this_grid();
  __shared__ int red[3];
  int sp = 0;
  init_red(red);
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int R = a.R;
  int p = 0;  // ring slot of the next grid-wide min (ring[0] preset by the host)
  for (int round = 0; round < R; ++round) {
    int first = 0x7fffffff;
    for (int64_t c = tid; c < R; c += nthreads) {
      if (!a.out[c]) continue;
      int64_t m = kInf;
      for (int32_t e = a.succ_off[c]; e < a.succ_off[c + 1]; ++e) m = min(m, a.M[a.succ[e]]);
      a.mp[c] = m;
      first = min(first, static_cast<int>(c));
    }
    int best = grid_min_step(first, ring, p, red, sp, grid);  // also publishes mp[]
    for (;;) {
      const int64_t bp = a.P[best], bm = a.tcol[best], bmp = a.mp[best];
      int nxt = 0x7fffffff;
      for (int64_t c = best + 1 + tid; c < R; c += nthreads)
        if (a.out[c] && precedes(static_cast<int>(c), a.P[c], a.tcol[c], a.mp[c], best, bp, bm, bmp)) {
          nxt = static_cast<int>(c);
          break;
        }
      nxt = grid_min_step(nxt, ring, p, red, sp, grid);
      if (nxt == 0x7fffffff) break;
      best = nxt;
    }
    const int64_t t = a.tcol[best];
    for (int64_t e = a.col_off[best] + tid; e < a.col_off[best + 1]; e += nthreads) {
      const int32_t g = a.col[e];
      const int k = --a.cnt[g];
      a.M[g] -= t;
      const int x = (a.xr[g] ^= best);
      if (k == 1) atomicAdd(reinterpret_cast<unsigned long long*>(&a.P[x]), a.wsum[g]);
    }
    if (tid == 0) {
      a.prio[best] = round;
      a.out[best] = 0;
    }
    grid.sync();
  }
}

// Multi-block TAC with the candidates resident in registers: thread t owns
// recv columns t, t + T, ... (at most kOwn), caching T(c), its successor
// range and its outstanding flag across rounds. Amended M+ is evaluated
// inline (min M over direct-successor groups) when a candidate is compared,
// so a round is the find-first chain (one grid-wide min per step, the first
// step starting from the lowest outstanding column, which every thread
// tracks identically) plus the retire: chain length + 1 grid barriers.
template <int kOwn>
__global__ void __launch_bounds__(1024) tac_own_kernel(TacArgs a, int* ring, longlong4* win) {
  // win[slot][block]: {P, T, M+} of the block's winning candidate of a
  // find-first step, written before the step's grid barrier, so the next
  // step reads the new incumbent with one load instead of a dependent chain
  cg::grid_group grid = cg::this_grid();
  __shared__ int red[3];
  int sp = 0;
  init_red(red);
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int nthreads = gridDim.x * blockDim.x;
  const int R = a.R;
  int64_t t_own[kOwn];
  int s0[kOwn], s1[kOwn], g1[kOwn], c0[kOwn], c1[kOwn];
  bool live[kOwn];
#pragma unroll
  for (int k = 0; k < kOwn; ++k) {
    const int c = tid + k * nthreads;
    live[k] = c < R;
    t_own[k] = live[k] ? a.tcol[c] : 0;
    s0[k] = live[k] ? a.succ_off[c] : 0;
    s1[k] = live[k] ? a.succ_off[c + 1] : 0;
    // the single direct-successor group, when there is one (the usual case):
    // M+ is then one load per round instead of a dependent pair
    g1[k] = live[k] && s1[k] - s0[k] == 1 ? a.succ[s0[k]] : -1;
    c0[k] = live[k] ? a.col_off[c] : 0;  // this column's retire list
    c1[k] = live[k] ? a.col_off[c + 1] : 0;
  }
  auto mplus = [&](int e0, int e1) {
    int64_t m = kInf;
    for (int e = e0; e < e1; ++e) m = min(m, a.M[a.succ[e]]);
    return m;
  };
  int p = 0;
  int first = 0;  // lowest outstanding column (identical in every thread)
  // the incumbent's static data, loaded as soon as `first` is known (before
  // the barrier that publishes the round's P and M): T, its one successor
  // group, its column range, and this thread's retire entry of that column
  int64_t f_t = 0;
  int f_g1 = -2;
  int32_t f_c0 = 0, f_c1 = 0, f_g = -1;
  auto load_first = [&]() {
    if (first >= R) return;
    f_t = a.tcol[first];
    f_g1 = a.g1[first];
    f_c0 = a.col_off[first];
    f_c1 = a.col_off[first + 1];
    f_g = f_c0 + tid < f_c1 ? a.col[f_c0 + tid] : -1;
  };
  load_first();
  for (int round = 0; round < R; ++round) {
    // this round's P and amended M+ of the owned outstanding candidates
    int64_t P_own[kOwn], mp_own[kOwn];
#pragma unroll
    for (int k = 0; k < kOwn; ++k) {
      P_own[k] = live[k] ? a.P[tid + k * nthreads] : 0;
      mp_own[k] = !live[k] ? kInf : g1[k] >= 0 ? a.M[g1[k]] : mplus(s0[k], s1[k]);
    }
    int best = first;
    int64_t bp = a.P[best], bm = f_t,
            bmp = f_g1 >= 0 ? a.M[f_g1] : (f_g1 == -2 ? kInf : mplus(a.succ_off[best], a.succ_off[best + 1]));
    int64_t bcol = (static_cast<int64_t>(f_c0) << 32) | static_cast<uint32_t>(f_c1);  // best's column range
    for (;;) {
      int nxt = 0x7fffffff;
      int64_t np = 0, nt = 0, nm = 0, ncol = 0;
#pragma unroll
      for (int k = 0; k < kOwn; ++k) {
        const int c = tid + k * nthreads;
        if (live[k] && c > best && c < nxt && precedes(c, P_own[k], t_own[k], mp_own[k], best, bp, bm, bmp)) {
          nxt = c;
          np = P_own[k];
          nt = t_own[k];
          nm = mp_own[k];
          ncol = (static_cast<int64_t>(c0[k]) << 32) | static_cast<uint32_t>(c1[k]);
        }
      }
      // grid-wide min (grid_min_step, inlined to publish the block winner)
      const int slot = p % 3;
      const int v = block_min_int(nxt, red, sp);
      if (nxt == v && v != 0x7fffffff) {
        win[slot * gridDim.x + blockIdx.x] = make_longlong4(np, nt, nm, ncol);
        atomicMin(&ring[slot], v);
      }
      if (blockIdx.x == 0 && threadIdx.x == 0) ring[(p + 1) % 3] = 0x7fffffff;
      grid.sync();
      nxt = *reinterpret_cast<volatile int*>(&ring[slot]);
      ++p;
      if (nxt == 0x7fffffff) break;
      best = nxt;
      const longlong4 w = win[slot * gridDim.x + (nxt % nthreads) / blockDim.x];  // ordered by grid.sync
      bp = w.x;
      bm = w.y;
      bmp = w.z;
      bcol = w.w;
    }
    const int64_t t = bm;  // T(best)
    const int32_t e0 = static_cast<int32_t>(bcol >> 32);
    const int32_t e1 = static_cast<int32_t>(bcol & 0xffffffff);
    const bool won_first = best == first;
    const int32_t g_pre = f_g;
    if (won_first) {  // the next incumbent is known now: its static data loads overlap the retire
      do ++first;
      while (first < R && (first == best || !*reinterpret_cast<volatile uint8_t*>(&a.out[first])));
      load_first();
    }
    for (int64_t e = e0 + tid; e < e1; e += nthreads) {
      const int32_t g = (won_first && e == e0 + tid) ? g_pre : a.col[e];  // prefetched when the incumbent won
      const int k = --a.cnt[g];
      a.M[g] -= t;
      const int x = (a.xr[g] ^= best);
      if (k == 1) atomicAdd(reinterpret_cast<unsigned long long*>(&a.P[x]), a.wsum[g]);
    }
#pragma unroll
    for (int k = 0; k < kOwn; ++k)
      if (tid + k * nthreads == best) live[k] = false;
    if (tid == 0) {
      a.prio[best] = round;
      a.out[best] = 0;
    }
    grid.sync();
  }
  if (tid == 0) ring[3] = p;  // find-first steps taken (trace)
}

// Speculative multi-block TAC: one grid barrier per round when the lowest
// outstanding column wins (on the layered config-5 graphs it always does:
// every find-first chain is empty). Interval r compares every owned
// candidate against `first` AND retires `first` speculatively; the barrier
// then either confirms it (no beater: round done) or the retire is undone and
// the round continues as tac_own_kernel's chain. What makes the overlap
// race-free: nothing the comparison reads is written in the same interval.
//   - amended M+: a thread keeps the M of each of its columns' direct-
//     successor groups in registers (<= kSpecS groups per column) and applies
//     a retire of column s as M -= T(s) where the closure bit (group, s) is
//     set (static data); the global group M is not needed at all;
//   - P: the retire's additions (a group dropping to one outstanding recv)
//     go to a per-interval delta buffer D[iv % 4] that owners apply one
//     interval later (zeroed two intervals later, flags reset three later);
//   - the incumbent's values: the owner of the next outstanding column
//     publishes them (P without this interval's deltas, M+ after the
//     speculative retire) for the next interval;
//   - closure bits of the incumbent-to-be are loaded two intervals ahead.
// cnt / xr (retire-only state) are touched by one thread per group.
constexpr int kSpecS = 4;

__device__ __forceinline__ longlong4 ldcg4(const longlong4* p) {  // L2 (another SM wrote it)
  const longlong2 lo = __ldcg(reinterpret_cast<const longlong2*>(p)), hi = __ldcg(reinterpret_cast<const longlong2*>(p) + 1);
  return make_longlong4(lo.x, lo.y, hi.x, hi.y);
}

struct TacSpecWs {
  const uint32_t* bits;  // closure [row][W]
  int32_t W;
  long long* D;          // [4][R] P deltas per interval
  int* flag;             // [4] interval had deltas
  longlong4* pub;        // [2] next incumbent {P, M+, T, column}
  int* ring;             // [3] grid-min slots, [3] trace: misspeculated rounds
  longlong4* win;        // [3][blocks] per-block winner records
};

template <int kOwn, int kS>
__global__ void __launch_bounds__(1024) tac_spec_kernel(TacArgs a, TacSpecWs ws) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ uint32_t live_s[];  // this block's replica of the outstanding set, [(R + 31) / 32]
  __shared__ int red[3];
  int sp = 0;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int nthreads = gridDim.x * blockDim.x;
  const int R = a.R;
  const int kInt = 0x7fffffff;
  for (int w = threadIdx.x; w < (R + 31) / 32; w += blockDim.x) {
    uint32_t bits = 0;
    for (int b = 0; b < 32 && w * 32 + b < R; ++b) bits |= (a.out[w * 32 + b] ? 1u : 0u) << b;
    live_s[w] = bits;
  }
  init_red(red);  // (and the bitset's barrier)
  long long T_[kOwn], P_[kOwn], mg[kOwn][kS];
  int sg[kOwn][kS], ns[kOwn], c0[kOwn], c1[kOwn];
  uint32_t bpre[kOwn], bnext[kOwn];
  bool live[kOwn];
#pragma unroll
  for (int k = 0; k < kOwn; ++k) {
    const int c = tid + k * nthreads;
    live[k] = c < R && a.out[c];
    T_[k] = c < R ? a.tcol[c] : 0;
    P_[k] = c < R ? a.P[c] : 0;
    ns[k] = c < R ? a.succ_off[c + 1] - a.succ_off[c] : 0;
#pragma unroll
    for (int s = 0; s < kS; ++s) {
      sg[k][s] = s < ns[k] ? a.succ[a.succ_off[c] + s] : 0;
      mg[k][s] = s < ns[k] ? a.M[sg[k][s]] : kInf;
    }
    c0[k] = c < R ? a.col_off[c] : 0;
    c1[k] = c < R ? a.col_off[c + 1] : 0;
    bpre[k] = bnext[k] = 0;
  }
  auto mplus = [&](int k) {
    long long m = kInf;
#pragma unroll
    for (int s = 0; s < kS; ++s) m = min(m, mg[k][s]);
    return m;
  };
  // bit s: direct-successor group s of owned column k depends on column col
  auto bitmask = [&](int k, int col) -> uint32_t {
    uint32_t m = 0;
    if (col < R && tid + k * nthreads < R) {
#pragma unroll
      for (int s = 0; s < kS; ++s)
        if (s < ns[k])
          m |= ((__ldg(&ws.bits[static_cast<size_t>(sg[k][s]) * ws.W + (col >> 5)]) >> (col & 31)) & 1u) << s;
    }
    return m;
  };
  // next outstanding column after c in the replica, skipping columns whose
  // retirement the replica may not show yet
  auto next_live = [&](int c, int skip1, int skip2) {
    do ++c;
    while (c < R && (c == skip1 || c == skip2 || !((live_s[c >> 5] >> (c & 31)) & 1u)));
    return c;
  };
  auto publish = [&](int col, int iv) {  // owner of col: its values for the next interval
#pragma unroll
    for (int k = 0; k < kOwn; ++k)
      if (tid + k * nthreads == col) ws.pub[iv & 1] = make_longlong4(P_[k], mplus(k), T_[k], col);
  };
  // start-of-interval delta bookkeeping: apply the previous interval's P
  // additions (fl1), zero the buffer of two intervals back (fl2), reset the
  // flag of two intervals back (every thread read it after that barrier)
  auto deltas = [&](int iv, bool fl1, bool fl2) {
#pragma unroll
    for (int k = 0; k < kOwn; ++k) {
      const int c = tid + k * nthreads;
      if (c >= R) continue;
      if (fl1) P_[k] += __ldcg(&ws.D[static_cast<size_t>((iv - 1) & 3) * R + c]);
      if (fl2) ws.D[static_cast<size_t>((iv - 2) & 3) * R + c] = 0;
    }
    if (tid == 0) ws.flag[(iv - 2) & 3] = 0;
  };
  auto add_p = [&](int iv, int x, unsigned long long wsum) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&ws.D[static_cast<size_t>(iv & 3) * R + x]), wsum);
    ws.flag[iv & 3] = 1;
  };
  // a retire's (sign 1) or an undo's (sign -1) group updates beyond this
  // thread's first entry of the list
  auto retire_rest = [&](int col, int e0, int e1, int iv, int sign) {
    for (int e = e0 + tid + nthreads; e < e1; e += nthreads) {
      const int32_t g = a.col[e];
      const int k = (a.cnt[g] -= sign);
      const int x = (a.xr[g] ^= col);
      if (sign > 0 && k == 1) add_p(iv, x, a.wsum[g]);
    }
  };
  int iv = 1;
  int first = next_live(-1, -1, -1), prev = -1;
  int f_c0 = 0, f_c1 = 0, f_g = -1;  // the incumbent's retire list and this thread's first entry
  auto load_first = [&](int col) {
    f_c0 = col < R ? a.col_off[col] : 0;
    f_c1 = col < R ? a.col_off[col + 1] : 0;
    f_g = f_c0 + tid < f_c1 ? a.col[f_c0 + tid] : -1;
  };
  if (first < R) {
    publish(first, 0);
    const int second = next_live(first, -1, -1);
#pragma unroll
    for (int k = 0; k < kOwn; ++k) {
      bpre[k] = bitmask(k, first);
      bnext[k] = bitmask(k, second);
    }
    load_first(first);
  }
  int misses = 0;
  bool fl1 = false, fl2 = false;
  grid.sync();
  longlong4 pubv = ldcg4(&ws.pub[0]);
  for (int round = 0; round < R; ++round) {
    // ---- speculative interval: compare against `first`, retire `first`
    if (threadIdx.x == 0 && prev >= 0) live_s[prev >> 5] &= ~(1u << (prev & 31));  // (seen after block_min)
    const int second = next_live(first, first, prev);
    const int third = second < R ? next_live(second, first, prev) : R;
    uint32_t bnn[kOwn];
#pragma unroll
    for (int k = 0; k < kOwn; ++k) bnn[k] = bitmask(k, third);  // used two intervals on
    int g_cnt = 0, g_xr = 0;
    if (f_g >= 0) {  // the speculative retire's first group, read early
      g_cnt = __ldcg(&a.cnt[f_g]);
      g_xr = __ldcg(&a.xr[f_g]);
    }
    deltas(iv, fl1, fl2);
    const long long Pf = pubv.x + (fl1 ? __ldcg(&ws.D[static_cast<size_t>((iv - 1) & 3) * R + first]) : 0);
    const long long Mf = pubv.y, Tf = pubv.z;
    int nxt = kInt;
    longlong4 rec = make_longlong4(0, 0, 0, 0);
#pragma unroll
    for (int k = 0; k < kOwn; ++k) {
      const int c = tid + k * nthreads;
      if (live[k] && c > first && c < nxt && precedes(c, P_[k], T_[k], mplus(k), first, Pf, Tf, Mf)) {
        nxt = c;
        rec = make_longlong4(P_[k], T_[k], mplus(k), (static_cast<long long>(c0[k]) << 32) | static_cast<uint32_t>(c1[k]));
      }
    }
    {
      const int slot = iv % 3;
      const int v = block_min_int(nxt, red, sp);
      if (nxt == v && v != kInt) {
        ws.win[slot * gridDim.x + blockIdx.x] = rec;
        atomicMin(&ws.ring[slot], v);
      }
      if (blockIdx.x == 0 && threadIdx.x == 0) ws.ring[(iv + 1) % 3] = kInt;
    }
    if (f_g >= 0) {
      a.cnt[f_g] = g_cnt - 1;
      a.xr[f_g] = g_xr ^ first;
      if (g_cnt - 1 == 1) add_p(iv, g_xr ^ first, a.wsum[f_g]);
    }
    retire_rest(first, f_c0, f_c1, iv, 1);
    if (tid == 0) {
      a.out[first] = 0;
      a.prio[first] = round;
    }
#pragma unroll
    for (int k = 0; k < kOwn; ++k) {
#pragma unroll
      for (int s = 0; s < kS; ++s)
        if ((bpre[k] >> s) & 1u) mg[k][s] -= Tf;
      if (tid + k * nthreads == first) live[k] = false;
    }
    publish(second, iv);
    const int sf_c0 = f_c0, sf_c1 = f_c1, sf_g = f_g;
    load_first(second);
    grid.sync();
    ++iv;
    nxt = __ldcg(&ws.ring[(iv - 1) % 3]);
    fl2 = fl1;
    fl1 = __ldcg(&ws.flag[(iv - 1) & 3]) != 0;
    pubv = ldcg4(&ws.pub[(iv - 1) & 1]);
    if (nxt == kInt) {  // confirmed: `first` was the winner
      prev = first;
      first = second;
#pragma unroll
      for (int k = 0; k < kOwn; ++k) {
        bpre[k] = bnext[k];
        bnext[k] = bnn[k];
      }
      continue;
    }
    // ---- misspeculation: undo the retire of `first` (its P additions, in
    // the previous interval's buffer, are never applied), then the chain
    ++misses;
    prev = -1;  // (cleared in the replica already)
    deltas(iv, false, fl2);
    if (sf_g >= 0) {
      ++a.cnt[sf_g];
      a.xr[sf_g] ^= first;
    }
    retire_rest(first, sf_c0, sf_c1, iv, -1);
    if (tid == 0) a.out[first] = 1;
#pragma unroll
    for (int k = 0; k < kOwn; ++k) {
#pragma unroll
      for (int s = 0; s < kS; ++s)
        if ((bpre[k] >> s) & 1u) mg[k][s] += Tf;
      if (tid + k * nthreads == first) live[k] = true;
    }
    f_c0 = sf_c0;
    f_c1 = sf_c1;
    f_g = sf_g;
    int best = nxt;
    longlong4 w = ldcg4(&ws.win[((iv - 1) % 3) * gridDim.x + (nxt % nthreads) / blockDim.x]);
    for (bool undo_iv = true;; undo_iv = false) {  // one find-first step per interval
      if (!undo_iv) deltas(iv, fl1, fl2);
      nxt = kInt;
#pragma unroll
      for (int k = 0; k < kOwn; ++k) {
        const int c = tid + k * nthreads;
        if (live[k] && c > best && c < nxt && precedes(c, P_[k], T_[k], mplus(k), best, w.x, w.y, w.z)) {
          nxt = c;
          rec = make_longlong4(P_[k], T_[k], mplus(k), (static_cast<long long>(c0[k]) << 32) | static_cast<uint32_t>(c1[k]));
        }
      }
      const int slot = iv % 3;
      const int v = block_min_int(nxt, red, sp);
      if (nxt == v && v != kInt) {
        ws.win[slot * gridDim.x + blockIdx.x] = rec;
        atomicMin(&ws.ring[slot], v);
      }
      if (blockIdx.x == 0 && threadIdx.x == 0) ws.ring[(iv + 1) % 3] = kInt;
      grid.sync();
      ++iv;
      nxt = __ldcg(&ws.ring[(iv - 1) % 3]);
      fl2 = fl1;
      fl1 = __ldcg(&ws.flag[(iv - 1) & 3]) != 0;
      if (nxt == kInt) break;
      best = nxt;
      w = ldcg4(&ws.win[((iv - 1) % 3) * gridDim.x + (nxt % nthreads) / blockDim.x]);
    }
    // ---- retire `best` (the incumbent `first` stays for the next round)
    deltas(iv, fl1, fl2);
    if (blockIdx.x == 0 && threadIdx.x == 0) ws.ring[(iv + 1) % 3] = kInt;  // the next interval's min slot
    {
      const int e0 = static_cast<int>(w.w >> 32), e1 = static_cast<int>(w.w & 0xffffffff);
      if (e0 + tid < e1) {
        const int32_t g = a.col[e0 + tid];
        const int k = --a.cnt[g];
        const int x = (a.xr[g] ^= best);
        if (k == 1) add_p(iv, x, a.wsum[g]);
      }
      retire_rest(best, e0, e1, iv, 1);
    }
    if (tid == 0) {
      a.out[best] = 0;
      a.prio[best] = round;
    }
#pragma unroll
    for (int k = 0; k < kOwn; ++k) {
      const uint32_t m = bitmask(k, best);
#pragma unroll
      for (int s = 0; s < kS; ++s)
        if ((m >> s) & 1u) mg[k][s] -= w.y;
      if (tid + k * nthreads == best) live[k] = false;
    }
    publish(first, iv);
    const int second2 = next_live(first, best, -1);
#pragma unroll
    for (int k = 0; k < kOwn; ++k) bnext[k] = bitmask(k, second2);
    grid.sync();
    ++iv;
    fl2 = fl1;
    fl1 = __ldcg(&ws.flag[(iv - 1) & 3]) != 0;
    pubv = ldcg4(&ws.pub[(iv - 1) & 1]);
    prev = best;
  }
  if (tid == 0) ws.ring[3] = misses;
}

// TAC on one thread-block cluster (kClusterMax CTAs): cluster barriers are
// hardware (≈0.3 µs on B200 against ≈1.25 µs for a cooperative grid sync),
// and the rounds are barrier-bound. CTA k owns recv columns
// [k·per, (k+1)·per); each column's static data (T, successor range,
// outstanding flag) and this round's P / amended M+ sit in the owner's shared
// memory. A cluster-wide min = block min → own slot of a 3-slot ring → cluster
// barrier → warp 0 reads every CTA's slot over DSMEM → block broadcast. A
// round: one min for the lowest outstanding column, one per find-first step,
// the retire (column list spread over the cluster), one cluster barrier.
constexpr int kClusterMax = 16;

__host__ __device__ inline size_t tac_cluster_smem(int per) { return 33ull * per + 64; }

__global__ void __launch_bounds__(1024) tac_cluster_kernel(TacArgs a, int per) {
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) char csm[];
  __shared__ int bred[3], ring[3], bcast[3];
  int sp = 0, q = 0;
  const int R = a.R, cs = static_cast<int>(cluster.num_blocks());
  const int rank = static_cast<int>(cluster.block_rank());
  const int base = rank * per, n_own = max(0, min(per, R - base));
  auto* t_s = reinterpret_cast<int64_t*>(csm);
  auto* P_s = t_s + per;
  auto* mp_s = P_s + per;
  auto* s0_s = reinterpret_cast<int32_t*>(mp_s + per);
  auto* s1_s = s0_s + per;
  auto* live_s = reinterpret_cast<uint8_t*>(s1_s + per);
  for (int j = threadIdx.x; j < n_own; j += blockDim.x) {
    const int c = base + j;
    t_s[j] = a.tcol[c];
    s0_s[j] = a.succ_off[c];
    s1_s[j] = a.succ_off[c + 1];
    live_s[j] = a.out[c];
  }
  if (threadIdx.x < 3) {
    bred[threadIdx.x] = 0x7fffffff;
    ring[threadIdx.x] = 0x7fffffff;
  }
  cluster.sync();  // copies and rings ready in every CTA
  auto mplus = [&](int e0, int e1) {
    int64_t m = kInf;
    for (int e = e0; e < e1; ++e) m = min(m, a.M[a.succ[e]]);
    return m;
  };
  auto cluster_min = [&](int v) {
    v = block_min_int(v, bred, sp);
    const int slot = q % 3;
    if (threadIdx.x == 0) ring[slot] = v;
    cluster.sync();
    if (threadIdx.x < 32) {
      int r = 0x7fffffff;
      if (static_cast<int>(threadIdx.x) < cs) r = *cluster.map_shared_rank(&ring[slot], threadIdx.x);
      r = __reduce_min_sync(~0u, r);
      if (threadIdx.x == 0) bcast[slot] = r;
    }
    __syncthreads();
    const int r = bcast[slot];
    ++q;
    return r;
  };
  const int tid = rank * blockDim.x + threadIdx.x, nthreads = cs * blockDim.x;
  for (int round = 0; round < R; ++round) {
    // this round's P and amended M+ of the owned outstanding columns, four at
    // a time so their global loads overlap
    int first = 0x7fffffff;
    for (int j0 = threadIdx.x; j0 < n_own; j0 += 4 * blockDim.x) {
      int64_t pv[4], mv[4];
      bool lv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = j0 + u * blockDim.x;
        lv[u] = j < n_own && live_s[j];
        pv[u] = lv[u] ? a.P[base + j] : 0;
        mv[u] = lv[u] ? mplus(s0_s[j], s1_s[j]) : kInf;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = j0 + u * blockDim.x;
        if (!lv[u]) continue;
        P_s[j] = pv[u];
        mp_s[j] = mv[u];
        first = min(first, base + j);
      }
    }
    int best = cluster_min(first);
    for (;;) {
      const int64_t bp = a.P[best], bm = a.tcol[best], bmp = mplus(a.succ_off[best], a.succ_off[best + 1]);
      int nxt = 0x7fffffff;
      for (int j = max(best + 1 - base, 0) + threadIdx.x; j < n_own; j += blockDim.x)
        if (live_s[j] && precedes(base + j, P_s[j], t_s[j], mp_s[j], best, bp, bm, bmp)) {
          nxt = base + j;
          break;
        }
      nxt = cluster_min(nxt);
      if (nxt == 0x7fffffff) break;
      best = nxt;
    }
    const int64_t t = a.tcol[best];
    for (int32_t e = a.col_off[best] + tid; e < a.col_off[best + 1]; e += nthreads) {
      const int32_t g = a.col[e];
      const int k = --a.cnt[g];
      a.M[g] -= t;
      const int x = (a.xr[g] ^= best);
      if (k == 1) atomicAdd(reinterpret_cast<unsigned long long*>(&a.P[x]), a.wsum[g]);
    }
    if (best >= base && best < base + n_own && threadIdx.x == 0) live_s[best - base] = 0;
    if (tid == 0) {
      a.prio[best] = round;
      a.out[best] = 0;
    }
    cluster.sync();  // retire visible cluster-wide before the next round reads P / M
  }
}

// TAC on one thread-block cluster with every per-round value in distributed
// shared memory. CTA k of cs owns recv columns [k*per, (k+1)*per) (P and T
// in its shared memory, a thread keeps kOwn columns' amended M+ in
// registers) and the groups g with g % cs == k (cnt, M, owner XOR); every
// CTA keeps a replica of the outstanding-column bitset, so the lowest
// outstanding column is tracked locally. A round: amended M+ of the owned
// columns from the groups' owners (DSMEM loads), the find-first chain (one
// cluster-wide min per step over a 3-slot ring of per-CTA winner records
// {column, P, T, M+}), the retire spread over the cluster (DSMEM
// read-modify-writes of the retired column's groups, DSMEM atomics into the
// owners' P), one cluster barrier. Nothing on the round's critical path
// touches global memory but the retired column's group list.
struct TacRec {
  long long P, T, mp;
  int c, pad;
};

__host__ __device__ inline size_t tac_dsm_smem(int per, int gper, int R) {
  return 20ull * per + 16ull * gper + 4ull * ((R + 31) / 32) + 3ull * sizeof(TacRec) + 64;
}

template <int kOwn>
__global__ void __launch_bounds__(1024) tac_dsm_kernel(TacArgs a, int per, int gper, int ngroups) {
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) char dsm[];
  __shared__ int bred[3];
  __shared__ TacRec bcast;
  int sp = 0, q = 0;
  const int R = a.R, cs = static_cast<int>(cluster.num_blocks());
  const int rank = static_cast<int>(cluster.block_rank());
  const int base = rank * per, n_own = max(0, min(per, R - base));
  auto* P_s = reinterpret_cast<long long*>(dsm);          // [per]
  auto* T_s = P_s + per;                                   // [per]
  auto* gM = reinterpret_cast<long long*>(T_s + per);      // [gper] groups g = rank + cs*l
  auto* gcnt = reinterpret_cast<int*>(gM + gper);          // [gper]
  auto* gxr = gcnt + gper;                                 // [gper]
  auto* live = reinterpret_cast<uint32_t*>(gxr + gper);    // [(R+31)/32] replicated
  auto* rec = reinterpret_cast<TacRec*>(live + (R + 31) / 32);  // 3-slot ring
  auto* g1_s = reinterpret_cast<int*>(rec + 3);           // [per] single successor group, -1 several, -2 none
  for (int j = threadIdx.x; j < n_own; j += blockDim.x) {
    P_s[j] = a.P[base + j];
    T_s[j] = a.tcol[base + j];
    const int e0 = a.succ_off[base + j], e1 = a.succ_off[base + j + 1];
    g1_s[j] = e1 - e0 == 1 ? a.succ[e0] : (e1 == e0 ? -2 : -1);
  }
  for (int l = threadIdx.x; l < gper; l += blockDim.x) {
    const int g = rank + cs * l;
    gM[l] = g < ngroups ? a.M[g] : 0;
    gcnt[l] = g < ngroups ? a.cnt[g] : 0;
    gxr[l] = g < ngroups ? a.xr[g] : 0;
  }
  for (int w = threadIdx.x; w < (R + 31) / 32; w += blockDim.x) {
    uint32_t bits = 0;
    for (int b = 0; b < 32 && w * 32 + b < R; ++b) bits |= (a.out[w * 32 + b] ? 1u : 0u) << b;
    live[w] = bits;
  }
  if (threadIdx.x < 3) {
    bred[threadIdx.x] = 0x7fffffff;
    rec[threadIdx.x].c = 0x7fffffff;
  }
  cluster.sync();  // every CTA's slices and rings ready
  auto Mg = [&](int g) -> long long {  // M of group g, at its owner
    return *cluster.map_shared_rank(&gM[g / cs], g % cs);
  };
  auto mplus = [&](int c) -> long long {  // owned or remote column c
    const int o = c / per;
    const int g1 = *cluster.map_shared_rank(&g1_s[c - o * per], o);
    if (g1 >= 0) return Mg(g1);
    if (g1 == -2) return kInf;
    long long m = kInf;
    for (int32_t e = a.succ_off[c]; e < a.succ_off[c + 1]; ++e) m = min(m, Mg(a.succ[e]));
    return m;
  };
  __shared__ long long first_p, first_mp;  // the incumbent's values, fetched once per CTA
  auto is_live = [&](int c) { return (live[c >> 5] >> (c & 31)) & 1u; };
  int first = 0;
  while (first < R && !is_live(first)) ++first;
  const int tid = rank * blockDim.x + threadIdx.x, nthreads = cs * blockDim.x;
  for (int round = 0; round < R; ++round) {
    // owned columns: amended M+ of this round in registers (P and T are
    // read from this CTA's shared memory where they are compared)
    long long mk[kOwn];
#pragma unroll
    for (int k = 0; k < kOwn; ++k) {
      const int j = threadIdx.x + k * blockDim.x;
      mk[k] = j < n_own && is_live(base + j) ? mplus(base + j) : kInf;
    }
    int best = first;
    if (threadIdx.x == 0) {
      first_p = *cluster.map_shared_rank(&P_s[best - (best / per) * per], best / per);
      first_mp = mplus(best);
    }
    __syncthreads();
    long long bp = first_p, bm = a.tcol[best], bmp = first_mp;
    for (;;) {
      int nxt = 0x7fffffff;
      long long np = 0, nt = 0, nm = 0;
#pragma unroll
      for (int k = 0; k < kOwn; ++k) {
        const int j = threadIdx.x + k * blockDim.x;
        const int c = base + j;
        if (j < n_own && c > best && c < nxt && is_live(c) && precedes(c, P_s[j], T_s[j], mk[k], best, bp, bm, bmp)) {
          nxt = c;
          np = P_s[j];
          nt = T_s[j];
          nm = mk[k];
        }
      }
      const int slot = q % 3;
      const int v = block_min_int(nxt, bred, sp);
      if (nxt == v && v != 0x7fffffff) {
        rec[slot].P = np;
        rec[slot].T = nt;
        rec[slot].mp = nm;
      }
      if (threadIdx.x == 0) rec[slot].c = v;
      cluster.sync();
      if (threadIdx.x < 32) {
        int c = 0x7fffffff;
        if (static_cast<int>(threadIdx.x) < cs) c = cluster.map_shared_rank(&rec[slot], threadIdx.x)->c;
        const int m = __reduce_min_sync(~0u, c);
        if (m != 0x7fffffff && c == m) bcast = *cluster.map_shared_rank(&rec[slot], threadIdx.x);
        if (threadIdx.x == 0 && m == 0x7fffffff) bcast.c = m;
      }
      __syncthreads();
      const TacRec w = bcast;
      ++q;
      if (w.c == 0x7fffffff) break;
      best = w.c;
      bp = w.P;
      bm = w.T;
      bmp = w.mp;
      __syncthreads();  // bcast is rewritten by the next step
    }
    // retire the winner: its groups (each listed once) at their owners
    const long long t = bm;
    for (int32_t e = a.col_off[best] + tid; e < a.col_off[best + 1]; e += nthreads) {
      const int32_t g = a.col[e];
      const int o = g % cs, l = g / cs;
      int* cp = cluster.map_shared_rank(&gcnt[l], o);
      const int k = --*cp;
      *cluster.map_shared_rank(&gM[l], o) -= t;
      int* xp = cluster.map_shared_rank(&gxr[l], o);
      const int x = (*xp ^= best);
      if (k == 1)
        atomicAdd(reinterpret_cast<unsigned long long*>(cluster.map_shared_rank(&P_s[x - (x / per) * per], x / per)),
                  a.wsum[g]);
    }
    if (threadIdx.x == 0) live[best >> 5] &= ~(1u << (best & 31));
    if (tid == 0) {
      a.prio[best] = round;
      a.out[best] = 0;
    }
    cluster.sync();  // retire and the outstanding bit visible before the next round reads them
    if (best == first)
      do ++first;
      while (first < R && !is_live(first));
  }
}

// Speculative TAC on one 16-CTA thread-block cluster: tac_spec_kernel's
// one-barrier rounds (compare every candidate against `first` and retire
// `first` in the same interval) with every per-round value in distributed
// shared memory, so a round is one hardware cluster barrier (~0.3 us) and
// DSMEM reads instead of a grid barrier and L2 round trips. CTA k owns
// columns [k*per, (k+1)*per): P, the direct-successor groups' M (amended M+
// is their min) and a P-delta slot per column in its shared memory, T in
// registers; each thread caches the closure words (group, first / 32) of
// its columns' groups, reloaded when `first` crosses a 32-column boundary.
// P additions of a retire (rare: a group dropping to one outstanding recv)
// go to the owners' delta slots and raise a flag in every CTA; the next
// interval then applies them and republishes the incumbent ("fixup") before
// speculating again. Group cnt / owner XOR stay in global memory (one
// thread per group per retire).
struct CSpecPub {
  long long P, mp, T;
  int c, pad;
};

// V: the value width, int when every time sum fits 31 bits (host check),
// which makes a candidate's comparison a handful of 32-bit instructions
// (the rounds are issue-bound at 10^5 candidates on 16 SMs).
__host__ __device__ inline size_t tac_cspec_smem(int per, int kS, int R, size_t vb) {
  return (vb + vb * kS + vb) * per + 8ull * ((R + 63) / 64) + 3 * sizeof(TacRec) + 2 * sizeof(CSpecPub) + 64;
}

template <typename V>
__device__ __forceinline__ bool precedes_v(int a, V ap, V am, V amp, int b, V bp, V bm, V bmp) {
  const V ab = min(bp, am), ba = min(ap, bm);
  if (ab != ba) return ab < ba;
  if (amp != bmp) return amp < bmp;
  return a < b;
}

// Shared-memory loads/stores through a held 32-bit address (volatile and
// ordered like the plain accesses they replace).
template <typename V>
__device__ __forceinline__ V lds_v(uint32_t a) {
  if constexpr (sizeof(V) == 8) {
    long long v;
    asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
    return static_cast<V>(v);
  } else {
    int v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return static_cast<V>(v);
  }
}
template <typename V>
__device__ __forceinline__ void sts_v(uint32_t a, V v) {
  if constexpr (sizeof(V) == 8)
    asm volatile("st.shared.b64 [%0], %1;" :: "r"(a), "l"(static_cast<long long>(v)) : "memory");
  else
    asm volatile("st.shared.b32 [%0], %1;" :: "r"(a), "r"(static_cast<int>(v)) : "memory");
}

template <int kOwn, int kS, typename V>
__global__ void __launch_bounds__(1024) tac_cspec_kernel(TacArgs a, const uint32_t* __restrict__ bits, int W, int per,
                                                         int* trace) {
  constexpr int kCT = 1024;  // threads per CTA (the launch's block size)
  constexpr V kInfV = sizeof(V) == 8 ? static_cast<V>(kInf) : static_cast<V>(0x7fffffff);
  constexpr V kDead = sizeof(V) == 8 ? static_cast<V>(INT64_MIN) : static_cast<V>(INT32_MIN);  // P of a retired column
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) char csp[];
  __shared__ int bred[3];
  __shared__ TacRec bcast;
  __shared__ CSpecPub fpub;
  __shared__ int dflag[2];  // some retire added to a P of this CTA's columns, per interval parity (set remotely)
  __shared__ __align__(16) int mins[3][kClusterMax];  // every CTA's block min, pushed into every CTA (3-slot ring)
  __shared__ CSpecPub pubs[2];             // the next incumbent's values, pushed by its owner
  int sp = 0, q = 0, iv = 0;
  const int R = a.R, cs = static_cast<int>(cluster.num_blocks());
  const int rank = static_cast<int>(cluster.block_rank());
  // columns are interleaved over the CTAs (c % 16 owns c, at local index
  // c / 16), so every CTA keeps the same share of outstanding columns as
  // they retire in order
  constexpr int kCS = kClusterMax;
  const int n_own = max(0, (R - rank + kCS - 1) / kCS);
  (void)cs;
  // [per] P of outstanding columns (>= 0); kDead + 1 + round once retired in
  // that round (written to a.prio at the end: no global store inside a round,
  // so the barrier's release fence has nothing of ours in flight); kDead
  // when not outstanding at the start
  auto* P_s = reinterpret_cast<V*>(csp);
  auto* D_s = P_s + per;                                      // [per] P additions of the last retire
  auto* Mg_s = D_s + per;                                     // [kS][per] M of direct-successor groups
  auto* live = reinterpret_cast<uint32_t*>(csp + round16((2 + kS) * sizeof(V) * per));  // replicated outstanding bitset
  auto* rec = reinterpret_cast<TacRec*>(live + 2 * ((R + 63) / 64));  // 3-slot winner ring
  auto* pub = reinterpret_cast<CSpecPub*>(rec + 3);                    // [2] next incumbent (at its owner)
  const int kInt = 0x7fffffff;
  V T_[kOwn];
  int sg[kOwn][kS], ns[kOwn];
  uint32_t bwv[kOwn][kS];  // closure words (group, wc) of own columns' groups
#pragma unroll
  for (int k = 0; k < kOwn; ++k) {
    const int j = threadIdx.x + k * kCT, c = j * kCS + rank;
    const bool own = j < n_own;
    T_[k] = own ? static_cast<V>(a.tcol[c]) : V(0);
    ns[k] = own ? a.succ_off[c + 1] - a.succ_off[c] : 0;
#pragma unroll
    for (int s = 0; s < kS; ++s) {
      sg[k][s] = s < ns[k] ? a.succ[a.succ_off[c] + s] : 0;
      if (own) Mg_s[s * per + j] = s < ns[k] ? static_cast<V>(a.M[sg[k][s]]) : kInfV;
      bwv[k][s] = 0;
    }
    if (own) {
      P_s[j] = a.out[c] ? static_cast<V>(a.P[c]) : kDead;
      D_s[j] = 0;
    }
  }
  for (int w = threadIdx.x; w < (R + 31) / 32; w += kCT) {
    uint32_t b = 0;
    for (int i = 0; i < 32 && w * 32 + i < R; ++i) b |= (a.out[w * 32 + i] ? 1u : 0u) << i;
    live[w] = b;
  }
  if (threadIdx.x < 3) {
    bred[threadIdx.x] = kInt;
    rec[threadIdx.x].c = kInt;
  }
  if (threadIdx.x < 2) dflag[threadIdx.x] = 0;
  auto is_live = [&](int c) { return (live[c >> 5] >> (c & 31)) & 1u; };
  auto owner = [&](int c) { return c & (kCS - 1); };
  auto local = [&](int c) { return c >> 4; };
  static_assert(kCS == 16, "interleave");
  // this thread owns column c (local index threadIdx.x + k * 1024)
  auto mine_col = [&](int c) { return owner(c) == rank && (local(c) & (kCT - 1)) == static_cast<int>(threadIdx.x); };
  // 32-bit shared-window addresses of the per-column arrays, computed once
  // and held (the hot loops otherwise re-derive the window base from the
  // CTA's cluster id for every column: an S2R and three dependent
  // instructions before each load)
  uint32_t pa = static_cast<uint32_t>(__cvta_generic_to_shared(P_s));
  uint32_t ma = static_cast<uint32_t>(__cvta_generic_to_shared(Mg_s));
  asm volatile("" : "+r"(pa), "+r"(ma));
  auto mplus_j = [&](int j) {
    V m = kInfV;
#pragma unroll
    for (int s = 0; s < kS; ++s) m = min(m, lds_v<V>(ma + static_cast<uint32_t>(sizeof(V) * (s * per + j))));
    return m;
  };
  auto next_live = [&](int c, int skip) {
    do ++c;
    while (c < R && (c == skip || !is_live(c)));
    return c;
  };
  int wc = -1;  // closure word index cached in bwv
  auto load_words = [&](int word) {
#pragma unroll
    for (int k = 0; k < kOwn; ++k)
#pragma unroll
      for (int s = 0; s < kS; ++s)
        bwv[k][s] = s < ns[k] ? __ldg(&bits[static_cast<size_t>(sg[k][s]) * W + word]) : 0u;
    wc = word;
  };
  // M of own columns' groups after retiring column col (sign -1: undo)
  auto apply_retire = [&](int col, V t, int sign) {
    if ((col >> 5) != wc) load_words(col >> 5);
#pragma unroll
    for (int k = 0; k < kOwn; ++k) {
      const int j = threadIdx.x + k * kCT;
      if (j >= n_own) continue;
#pragma unroll
      for (int s = 0; s < kS; ++s)
        if ((bwv[k][s] >> (col & 31)) & 1u) {
          const uint32_t ad = ma + static_cast<uint32_t>(sizeof(V) * (s * per + j));
          sts_v<V>(ad, lds_v<V>(ad) - sign * t);
        }
    }
  };
  // the owner of col pushes its values for the next interval into every
  // CTA: its warp broadcasts them and 16 lanes store one CTA each (called by
  // every thread)
  auto publish = [&](int col, int slot) {
    const bool own = col < R && mine_col(col);
    const unsigned ball = __ballot_sync(~0u, own);
    if (ball == 0) return;
    long long pv = 0, mv = 0, tv = 0;
    if (own) {
      const int j = local(col), kk = j >> 10;
      V t = 0;
#pragma unroll
      for (int k = 0; k < kOwn; ++k)
        if (k == kk) t = T_[k];
      pv = P_s[j];
      mv = mplus_j(j);
      tv = t;
    }
    const int src = __ffs(ball) - 1;
    pv = __shfl_sync(~0u, pv, src);
    mv = __shfl_sync(~0u, mv, src);
    tv = __shfl_sync(~0u, tv, src);
    const int lane = threadIdx.x & 31;
    if (lane < kCS) *cluster.map_shared_rank(&pubs[slot], lane) = CSpecPub{pv, mv, tv, col, 0};
  };
  auto apply_deltas = [&]() {
#pragma unroll
    for (int k = 0; k < kOwn; ++k) {
      const int j = threadIdx.x + k * kCT;
      if (j < n_own && D_s[j] != 0) {
        P_s[j] += D_s[j];
        D_s[j] = 0;
      }
    }
  };
  const int tid = rank * kCT + threadIdx.x, nthreads = cs * kCT;
  // group updates of a retire (sign 1) or undo (sign -1) over the column's
  // list from entry e0 + tid + skip on (atomics: the state lives at L2
  // whatever the L1s hold; one thread per group)
  auto add_p = [&](int x, unsigned long long wsum) {
    if constexpr (sizeof(V) == 8)
      atomicAdd(reinterpret_cast<unsigned long long*>(cluster.map_shared_rank(&D_s[local(x)], owner(x))), wsum);
    else
      atomicAdd(cluster.map_shared_rank(&D_s[local(x)], owner(x)), static_cast<V>(wsum));
    for (int r = 0; r < cs; ++r) *cluster.map_shared_rank(&dflag[iv & 1], r) = 1;
  };
  auto retire_groups = [&](int col, int e0, int e1, int skip, int sign) {
    for (int e = e0 + tid + skip; e < e1; e += nthreads) {
      const int32_t g = a.col[e];
      const int kk = atomicSub(&a.cnt[g], sign) - sign;
      const int x = atomicXor(&a.xr[g], col) ^ col;
      if (sign > 0 && kk == 1) add_p(x, a.wsum[g]);
    }
  };
  // end of an interval: the cluster barrier; returns this CTA's delta flag
  // for the interval just ended (reset after everyone has read it)
  auto end_interval = [&]() {
    cluster.sync();
    ++iv;
    return dflag[(iv - 1) & 1] != 0;
  };
  auto reset_flag = [&]() {  // after a block barrier that follows end_interval's read
    if (threadIdx.x == 0) dflag[(iv - 1) & 1] = 0;
  };
  // cluster-wide min of v with the winners' records (its own interval)
  auto cluster_min_rec = [&](int v, const TacRec& mine) -> TacRec {
    const int slot = q % 3;
    const int bv = block_min_int(v, bred, sp);
    if (v == bv && bv != kInt) rec[slot] = mine;
    if (threadIdx.x == 0) rec[slot].c = bv;
    end_interval();
    if (threadIdx.x < 32) {
      int c = kInt;
      if (static_cast<int>(threadIdx.x) < cs) c = cluster.map_shared_rank(&rec[slot], threadIdx.x)->c;
      const int m = __reduce_min_sync(~0u, c);
      if (m != kInt && c == m) bcast = *cluster.map_shared_rank(&rec[slot], threadIdx.x);
      if (threadIdx.x == 0 && m == kInt) bcast.c = m;
    }
    __syncthreads();
    const TacRec w = bcast;
    reset_flag();
    ++q;
    __syncthreads();  // bcast is rewritten by the next call
    return w;
  };
  auto read_pub = [&](int slot) {  // after the interval that published it (pushed here)
    const CSpecPub v = pubs[slot];
    __syncthreads();
    reset_flag();
    return v;
  };
  cluster.sync();  // slices, bitsets and rings ready in every CTA
  int first = next_live(-1, -1);
  int pslot = 0;  // pub slot holding the incumbent's values
  publish(first, pslot);
  int f_c0 = 0, f_c1 = 0, f_g = -1;
  auto load_first = [&](int col) {
    f_c0 = col < R ? a.col_off[col] : 0;
    f_c1 = col < R ? a.col_off[col + 1] : 0;
    f_g = f_c0 + tid < f_c1 ? a.col[f_c0 + tid] : -1;
  };
  load_first(first);
  if (first < R) load_words(first >> 5);
  // the list bounds of the column after the incumbent, one interval ahead
  int c2_end = 0;
  auto next_c0 = [&](int col, int skip) {
    const int c = next_live(col, skip);
    c2_end = c < R ? a.col_off[c + 1] : 0;
    return c < R ? a.col_off[c] : 0;
  };
  int c2_0 = first < R ? next_c0(first, -1) : 0, c2_1 = c2_end;
  end_interval();
  CSpecPub fp = read_pub(pslot);
  int misses = 0, fixups = 0;
  for (int round = 0; round < R; ++round) {
    // ---- speculative interval: retire `first` (its group updates issued
    // first: nothing this interval reads them), compare against it
    const int second = next_live(first, first);
    int r_cnt = 0, r_xr = 0;  // the atomics' old values, consumed at the end of the interval
    if (f_g >= 0) {
      r_cnt = atomicSub(&a.cnt[f_g], 1);
      r_xr = atomicXor(&a.xr[f_g], first);
    }
    retire_groups(first, f_c0, f_c1, nthreads, 1);  // entries beyond one per thread (rare)
    // this thread's entry of the next incumbent's list (its bounds loaded
    // last interval) and the bounds of the one after it: one memory hop each
    const int n_c0 = c2_0, n_c1 = c2_1;
    const int n_g = n_c0 + tid < n_c1 ? a.col[n_c0 + tid] : -1;
    const int c3_0 = second < R ? next_c0(second, first) : 0, c3_1 = second < R ? c2_end : 0;
    if ((first >> 5) != wc) load_words(first >> 5);
    int nxt = kInt;
    TacRec mine{0, 0, 0, kInt, 0};
    const V fP = static_cast<V>(fp.P), fT = static_cast<V>(fp.T), fM = static_cast<V>(fp.mp);
#pragma unroll
    for (int k = 0; k < kOwn; ++k) {  // every column <= first is retired (kDead)
      const int j = threadIdx.x + k * kCT, c = j * kCS + rank;
      if (j < n_own && c < nxt) {
        const V pc = lds_v<V>(pa + static_cast<uint32_t>(sizeof(V) * j));
        if (pc >= 0) {
          const V mc = mplus_j(j);
          if (precedes_v(c, pc, T_[k], mc, first, fP, fT, fM)) {
            nxt = c;
            mine = TacRec{pc, T_[k], mc, c, 0};
          }
        }
      }
    }
    const int slot = q % 3;
    const int bv = block_min_int(nxt, bred, sp);  // (every compare of this CTA is done)
    reset_flag();  // the previous interval's flag: every thread read it before this barrier
    if (nxt == bv && bv != kInt) rec[slot] = mine;  // (pulled only on a misspeculation)
    if (threadIdx.x < kCS) *cluster.map_shared_rank(&mins[slot][rank], threadIdx.x) = bv;  // push
    apply_retire(first, static_cast<V>(fp.T), 1);
    const int npslot = pslot ^ 1;
    publish(second, npslot);  // M+ after this retire, P without its additions
    // (the asm keeps the compiler from waiting on the atomics where they issue)
    asm volatile("" : "+r"(r_cnt), "+r"(r_xr));
    if (f_g >= 0 && r_cnt - 1 == 1) add_p(r_xr ^ first, a.wsum[f_g]);
    const bool deltas = end_interval();
    int m = kInt;
#pragma unroll
    for (int r = 0; r < kCS / 4; ++r) {  // four 16-byte loads
      const int4 mv = reinterpret_cast<const int4*>(mins[slot])[r];
      m = min(m, min(min(mv.x, mv.y), min(mv.z, mv.w)));
    }
    const CSpecPub np = pubs[npslot];
    ++q;
    if (m == kInt) {  // confirmed: `first` was the winner
      if (threadIdx.x == 0) live[first >> 5] &= ~(1u << (first & 31));
      if (mine_col(first)) P_s[local(first)] = kDead + 1 + round;
      first = second;
      pslot = npslot;
      fp = np;
      f_c0 = n_c0;
      f_c1 = n_c1;
      f_g = n_g;
      c2_0 = c3_0;
      c2_1 = c3_1;
      if (deltas) {  // (every CTA's flag was raised: the fixup is cluster-uniform)
        ++fixups;
        apply_deltas();
        __syncthreads();
        reset_flag();
        pslot ^= 1;
        publish(first, pslot);
        end_interval();
        fp = read_pub(pslot);
      }
      continue;
    }
    // the winner's record, from the CTA that owns it
    if (threadIdx.x == 0) bcast = *cluster.map_shared_rank(&rec[slot], owner(m));
    __syncthreads();
    TacRec w = bcast;
    reset_flag();  // (the speculative retire's additions are dropped below)
    __syncthreads();  // bcast is rewritten later
    // ---- misspeculation: undo the retire of `first` (its P additions are
    // dropped), then the chain from w, then retire the chain's winner
    ++misses;
    retire_groups(first, f_c0, f_c1, 0, -1);
    apply_retire(first, static_cast<V>(fp.T), -1);
#pragma unroll
    for (int k = 0; k < kOwn; ++k) {
      const int j = threadIdx.x + k * kCT;
      if (j < n_own) D_s[j] = 0;
    }
    end_interval();  // undo complete everywhere
    __syncthreads();
    reset_flag();
    for (;;) {
      const int best = w.c;
      int nb = kInt;
      TacRec mb{0, 0, 0, kInt, 0};
#pragma unroll
      for (int k = 0; k < kOwn; ++k) {
        const int j = threadIdx.x + k * kCT, c = j * kCS + rank;
        if (j < n_own && c > best && c < nb) {
          const V pc = lds_v<V>(pa + static_cast<uint32_t>(sizeof(V) * j));
          if (pc >= 0) {
            const V mc = mplus_j(j);
            if (precedes_v(c, pc, T_[k], mc, best, static_cast<V>(w.P), static_cast<V>(w.T), static_cast<V>(w.mp))) {
              nb = c;
              mb = TacRec{pc, T_[k], mc, c, 0};
            }
          }
        }
      }
      const TacRec nw = cluster_min_rec(nb, mb);
      if (nw.c == kInt) break;
      w = nw;
    }
    const int best = w.c;
    retire_groups(best, a.col_off[best], a.col_off[best + 1], 0, 1);
    apply_retire(best, static_cast<V>(w.T), 1);
    end_interval();  // the retire's additions have landed
    if (threadIdx.x == 0) live[best >> 5] &= ~(1u << (best & 31));
    if (mine_col(best)) P_s[local(best)] = kDead + 1 + round;
    apply_deltas();
    __syncthreads();
    reset_flag();
    pslot ^= 1;
    publish(first, pslot);
    end_interval();
    fp = read_pub(pslot);
    if ((first >> 5) != wc) load_words(first >> 5);
    c2_0 = next_c0(first, -1);
    c2_1 = c2_0 >= 0 ? c2_end : 0;
  }
#pragma unroll
  for (int k = 0; k < kOwn; ++k) {
    const int j = threadIdx.x + k * kCT;
    if (j < n_own && P_s[j] != kDead) a.prio[j * kCS + rank] = static_cast<int32_t>(P_s[j] - kDead - 1);
  }
  if (trace && rank == 0 && threadIdx.x == 0) {
    trace[0] = misses;
    trace[1] = fixups;
  }
}

// Shared setup for properties / tic / tac: rows, closure, group state,
// column lists. `dur` per op (host).
struct GroupState {
  std::shared_ptr<const Rows> rw;
  DevArr d_counts, d_bits, d_rowof, d_wsum, d_has, d_cnt, d_M, d_xr, d_colcount,
      d_coloff, d_col, d_tcol, d_dur, d_tmp;
  int64_t nnz = 0;
};

int group_setup(DeviceGraph* g, const int64_t* dur, GroupState& S, char* err) {
  if (ensure_device(err)) return 1;
  {
    std::lock_guard<std::mutex> lock(g->rows_mu);
    if (!g->rows) {
      auto r = std::make_shared<Rows>();
      build_rows(g, *r);
      auto up = [&](int32_t*& d, const std::vector<int32_t>& v) -> int {
        CK(cudaMalloc(&d, round16(4 * std::max<size_t>(v.size(), 1))));
        if (!v.empty()) CK(cudaMemcpy(d, v.data(), 4 * v.size(), cudaMemcpyHostToDevice));
        return 0;
      };
      if (up(r->d_self, r->self_col) || up(r->d_preoff, r->pre_off) || up(r->d_pre, r->pre) ||
          up(r->d_rowof, r->row_of) || up(r->d_succoff, r->succ_off) || up(r->d_succ, r->succ) ||
          up(r->d_g1, r->g1) ||
          up(r->d_ntrow, r->nt_row) || up(r->d_ntoff, r->nt_off) || up(r->d_ntterm, r->nt_term) ||
          up(r->d_ntchunk, r->nt_chunk) || up(r->d_hasrows, r->has_rows)) {
        const int32_t* ps[] = {r->d_self,  r->d_preoff, r->d_pre,    r->d_rowof,   r->d_succoff, r->d_succ,
                               r->d_ntrow, r->d_ntoff,  r->d_ntterm, r->d_ntchunk, r->d_hasrows, r->d_g1};
        for (const int32_t* q : ps)
          if (q) cudaFree(const_cast<int32_t*>(q));
        return 1;
      }
      g->rows = std::move(r);
    }
    S.rw = g->rows;
  }
  const Rows& rw = *S.rw;
  const int32_t nrows = std::max(rw.nrows, 1), W = rw.W;
  std::vector<int64_t> tcol(std::max(g->R, 1));
  for (int c = 0; c < g->R; ++c) tcol[c] = dur[g->h_recv_ops[c]];
  std::vector<int64_t> hd(dur, dur + g->n);
  if (put(S.d_tcol, tcol, err) || put(S.d_dur, hd, err)) return 1;
  if (alloc<uint32_t>(S.d_bits, static_cast<size_t>(nrows) * W, err) ||
      alloc<unsigned long long>(S.d_wsum, nrows, err) || alloc<int32_t>(S.d_has, nrows, err) ||
      alloc<int32_t>(S.d_cnt, nrows, err) || alloc<int64_t>(S.d_M, nrows, err) ||
      alloc<int32_t>(S.d_xr, nrows, err) || alloc<int32_t>(S.d_colcount, g->R + 1, err) ||
      alloc<int32_t>(S.d_coloff, g->R + 1, err))
    return 1;
  CK(cudaMemset(S.d_wsum.p, 0, 8ull * nrows));
  CK(cudaMemset(S.d_has.p, 0, 4ull * nrows));
  CK(cudaMemset(S.d_colcount.p, 0, 4ull * (g->R + 1)));
  const size_t smem = static_cast<size_t>(rw.nrows) * W * 4;
  if (rw.nrows > 0) {
    // (TICTAC_CLOSURE_GLOBAL: test knob forcing the large-closure kernels)
    if (smem <= 200 * 1024 && !std::getenv("TICTAC_CLOSURE_GLOBAL")) {
      CK(allow_max_dynamic_smem(reinterpret_cast<const void*>(closure_smem_kernel)));
      closure_smem_kernel<<<1, 256, smem>>>(rw.nrows, W, rw.d_self,
                                            rw.d_preoff, rw.d_pre,
                                            S.d_bits.as<uint32_t>());
    } else {
      closure_roots_kernel<<<std::min(rw.nrows, 148 * 16), 256>>>(rw.nrows, W, rw.d_self,
                                                                  rw.d_preoff, S.d_bits.as<uint32_t>());
      LAUNCHED();
      if (!rw.nt_row.empty())
        closure_seq_kernel<<<(W + 127) / 128, 128>>>(static_cast<int32_t>(rw.nt_chunk.size()) - 1, W,
                                                     rw.d_ntchunk, rw.d_ntrow,
                                                     rw.d_ntoff, rw.d_ntterm,
                                                     S.d_bits.as<uint32_t>());
    }
    LAUNCHED();
    CK(cudaGetLastError());
  }
  weights_kernel<<<std::max(1, std::min((g->n + 255) / 256, 1184)), 256>>>(
      g->n, rw.d_rowof, g->kind, S.d_dur.as<int64_t>(), S.d_wsum.as<unsigned long long>(),
      S.d_has.as<int32_t>());
  LAUNCHED();
  const int rblocks = std::max(1, std::min((rw.nrows * 32 + 255) / 256, 2368));
  // column-list warps: one per (closure word, chunk of rows with compute
  // members), enough of them to fill the GPU
  const int32_t nhas = static_cast<int32_t>(rw.has_rows.size());
  int32_t nchunks = std::max(1, std::min((nhas + 31) / 32, (148 * 64 + W - 1) / W));
  const int32_t chunk_rows = std::max(32, ((nhas + nchunks - 1) / nchunks + 31) / 32 * 32);
  nchunks = std::max(1, (nhas + chunk_rows - 1) / chunk_rows);
  const int64_t cwarps = static_cast<int64_t>(W) * nchunks;
  const int cblocks = static_cast<int>((cwarps * 32 + 255) / 256);
  if (alloc<int32_t>(S.d_counts, static_cast<size_t>(nchunks) * std::max(g->R, 1), err)) return 1;
  if (rw.nrows > 0) {
    rowstate_kernel<<<rblocks, 256>>>(rw.nrows, W, S.d_bits.as<uint32_t>(), rw.d_preoff,
                                      rw.d_self, S.d_tcol.as<int64_t>(),
                                      S.d_has.as<int32_t>(), S.d_cnt.as<int32_t>(),
                                      S.d_M.as<int64_t>(), S.d_xr.as<int32_t>());
    LAUNCHED();
    if (g->R > 0) {
      colcount_warp_kernel<<<cblocks, 256>>>(nhas, W, g->R, nchunks, chunk_rows, S.d_bits.as<uint32_t>(),
                                             rw.d_hasrows, S.d_counts.as<int32_t>());
      LAUNCHED();
      colprefix_kernel<<<std::max(1, std::min((g->R + 255) / 256, 1184)), 256>>>(
          g->R, nchunks, S.d_counts.as<int32_t>(), S.d_colcount.as<int32_t>());
      LAUNCHED();
    }
  }
  CK(cudaGetLastError());
  // exclusive scan of column counts -> offsets (R+1 entries)
  size_t tmp_bytes = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, S.d_colcount.as<int32_t>(),
                                   S.d_coloff.as<int32_t>(), g->R + 1));
  CK(cudaMallocAsync(&S.d_tmp.p, std::max<size_t>(tmp_bytes, 16), 0));
  CK(cub::DeviceScan::ExclusiveSum(S.d_tmp.p, tmp_bytes, S.d_colcount.as<int32_t>(),
                                   S.d_coloff.as<int32_t>(), g->R + 1));
  LAUNCHED();
  int32_t nnz = 0;
  CK(cudaMemcpy(&nnz, S.d_coloff.as<int32_t>() + g->R, 4, cudaMemcpyDeviceToHost));
  S.nnz = nnz;
  if (alloc<int32_t>(S.d_col, nnz, err)) return 1;
  if (rw.nrows > 0 && g->R > 0) {
    colfill_warp_kernel<<<cblocks, 256>>>(nhas, W, g->R, nchunks, chunk_rows, S.d_bits.as<uint32_t>(),
                                          rw.d_hasrows, S.d_counts.as<int32_t>(),
                                          S.d_coloff.as<int32_t>(), S.d_col.as<int32_t>());
    LAUNCHED();
  }
  CK(cudaGetLastError());
  return 0;
}

__global__ void dense_rank_kernel(int32_t R, const int64_t* __restrict__ sorted_unique, int32_t u,
                                  const int64_t* __restrict__ vals, int32_t* __restrict__ prio) {
  for (int32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < R; c += gridDim.x * blockDim.x) {
    int32_t lo = 0, hi = u;
    const int64_t v = vals[c];
    while (lo < hi) {
      const int32_t mid = (lo + hi) >> 1;
      if (sorted_unique[mid] < v) lo = mid + 1;
      else hi = mid;
    }
    prio[c] = lo;
  }
}

}  // namespace
}  // namespace tictac_dev

using namespace tictac_dev;

extern "C" int csk_properties(DeviceGraph* g, const int64_t* dur, int mode, uint64_t* dep_bits,
                              int64_t* M, int64_t* P, int64_t* Mplus, char* err) {
  GroupState S;
  if (group_setup(g, dur, S, err)) return 1;
  const int R = g->R;
  DevArr d_P, d_Mp;
  if (alloc<int64_t>(d_P, R, err) || alloc<int64_t>(d_Mp, R, err)) return 1;
  if (R > 0) {
    props_kernel<<<props_blocks(R), 256>>>(
        R, mode, S.d_coloff.as<int32_t>(), S.d_col.as<int32_t>(), S.d_cnt.as<int32_t>(),
        S.d_M.as<int64_t>(), S.d_xr.as<int32_t>(), S.d_wsum.as<unsigned long long>(),
        d_P.as<int64_t>(), d_Mp.as<int64_t>());
    LAUNCHED();
    CK(cudaGetLastError());
    CK(cudaMemcpy(P, d_P.p, 8ull * R, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(Mplus, d_Mp.p, 8ull * R, cudaMemcpyDeviceToHost));
  }
  // per-op rows back to the host formatter
  const int W = S.rw->W, w64 = std::max(1, (R + 63) / 64);
  std::vector<uint32_t> bits(static_cast<size_t>(std::max(S.rw->nrows, 1)) * W);
  std::vector<int64_t> rowM(std::max(S.rw->nrows, 1));
  if (S.rw->nrows > 0) {
    CK(cudaMemcpy(bits.data(), S.d_bits.p, 4ull * S.rw->nrows * W, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(rowM.data(), S.d_M.p, 8ull * S.rw->nrows, cudaMemcpyDeviceToHost));
  }
  for (int32_t v = 0; v < g->n; ++v) {
    const int32_t k = S.rw->row_of[v];
    uint64_t* dst = dep_bits + static_cast<size_t>(v) * w64;
    for (int q = 0; q < w64; ++q) dst[q] = 0;
    for (int q = 0; q < W; ++q)
      dst[q >> 1] |= static_cast<uint64_t>(bits[static_cast<size_t>(k) * W + q]) << (32 * (q & 1));
    M[v] = rowM[k];
  }
  return 0;
}

extern "C" int csk_tic(DeviceGraph* g, int mode, int32_t* prio, int* total, char* err) {
  const int R = g->R;
  *total = 1;
  if (R == 0) return 0;
  std::vector<int64_t> unit(g->n);
  for (int32_t v = 0; v < g->n; ++v) unit[v] = g->h_kind[v] == 1 ? 1 : 0;  // general oracle
  GroupState S;
  if (group_setup(g, unit.data(), S, err)) return 1;
  DevArr d_P, d_Mp, d_sorted, d_unique, d_nu, d_tmp, d_prio;
  if (alloc<int64_t>(d_P, R, err) || alloc<int64_t>(d_Mp, R, err) || alloc<int64_t>(d_sorted, R, err) ||
      alloc<int64_t>(d_unique, R, err) || alloc<int32_t>(d_nu, 1, err) || alloc<int32_t>(d_prio, R, err))
    return 1;
  props_kernel<<<props_blocks(R), 256>>>(
      R, mode, S.d_coloff.as<int32_t>(), S.d_col.as<int32_t>(), S.d_cnt.as<int32_t>(),
      S.d_M.as<int64_t>(), S.d_xr.as<int32_t>(), S.d_wsum.as<unsigned long long>(), d_P.as<int64_t>(),
      d_Mp.as<int64_t>());
  LAUNCHED();
  // dense rank: radix sort, unique, binary search (schedule.cpp:27-40)
  size_t b1 = 0, b2 = 0;
  CK(cub::DeviceRadixSort::SortKeys(nullptr, b1, d_Mp.as<int64_t>(), d_sorted.as<int64_t>(), R));
  CK(cub::DeviceSelect::Unique(nullptr, b2, d_sorted.as<int64_t>(), d_unique.as<int64_t>(),
                               d_nu.as<int32_t>(), R));
  CK(cudaMallocAsync(&d_tmp.p, std::max<size_t>(std::max(b1, b2), 16), 0));
  CK(cub::DeviceRadixSort::SortKeys(d_tmp.p, b1, d_Mp.as<int64_t>(), d_sorted.as<int64_t>(), R));
  CK(cub::DeviceSelect::Unique(d_tmp.p, b2, d_sorted.as<int64_t>(), d_unique.as<int64_t>(),
                               d_nu.as<int32_t>(), R));
  LAUNCHED();
  LAUNCHED();
  int32_t u = 0;
  CK(cudaMemcpy(&u, d_nu.p, 4, cudaMemcpyDeviceToHost));
  dense_rank_kernel<<<std::max(1, std::min((R + 255) / 256, 1184)), 256>>>(
      R, d_unique.as<int64_t>(), u, d_Mp.as<int64_t>(), d_prio.as<int32_t>());
  LAUNCHED();
  CK(cudaGetLastError());
  CK(cudaMemcpy(prio, d_prio.p, 4ull * R, cudaMemcpyDeviceToHost));
  *total = u == R;
  return 0;
}

extern "C" int csk_tac(DeviceGraph* g, const int64_t* dur, int32_t* prio, char* err) {
  const int R = g->R;
  if (R == 0) return 0;
  const bool trace = std::getenv("TICTAC_TAC_TRACE") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  const auto t0 = now();
  GroupState S;
  if (group_setup(g, dur, S, err)) return 1;
  if (trace) cudaDeviceSynchronize();
  const auto t1 = now();
  DevArr d_P, d_Mp, d_out, d_prio;
  if (alloc<int64_t>(d_P, R, err) || alloc<int64_t>(d_Mp, R, err) || alloc<uint8_t>(d_out, R, err) ||
      alloc<int32_t>(d_prio, R, err))
    return 1;
  CK(cudaMemset(d_out.p, 1, R));
  // initial P (amended M+ is recomputed inside the rounds)
  props_kernel<<<props_blocks(R), 256>>>(
      R, 1, S.d_coloff.as<int32_t>(), S.d_col.as<int32_t>(), S.d_cnt.as<int32_t>(), S.d_M.as<int64_t>(),
      S.d_xr.as<int32_t>(), S.d_wsum.as<unsigned long long>(), d_P.as<int64_t>(), d_Mp.as<int64_t>());
  LAUNCHED();
  CK(cudaGetLastError());
  TacArgs a{R,
            S.d_tcol.as<int64_t>(),
            S.rw->d_succoff,
            S.rw->d_succ,
            S.rw->d_g1,
            S.d_coloff.as<int32_t>(),
            S.d_col.as<int32_t>(),
            S.d_wsum.as<unsigned long long>(),
            S.d_cnt.as<int32_t>(),
            S.d_M.as<int64_t>(),
            S.d_xr.as<int32_t>(),
            d_P.as<int64_t>(),
            d_Mp.as<int64_t>(),
            d_out.as<uint8_t>(),
            d_prio.as<int32_t>()};
  // One block is latency-optimal until the per-round work (retire list and
  // candidate scan) outgrows it; then spread over the SMs.
  int dev = 0, sms = 148, per_sm = 1;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tac_dist_kernel, 1024, 0));
  // Per-round work = candidate scan (R_t) + retire list (nnz/R on average).
  const int64_t work = S.nnz / std::max(R, 1) + R;
  int blocks = work > 16384 ? static_cast<int>(std::min<int64_t>(sms * std::max(per_sm, 1), (work + 1023) / 1024)) : 1;
  // Test knob: force the block count (the multi-block path is otherwise
  // only taken on graphs too large for the CPU oracle).
  if (const char* env = std::getenv("TICTAC_TAC_BLOCKS")) {
    const int forced = std::atoi(env);
    if (forced > 0) blocks = std::min(forced, sms * std::max(per_sm, 1));
  }
  blocks = std::max(blocks, 1);
  const auto t2 = now();
  // One thread-block cluster when one block's shared memory cannot hold the
  // state but the round work still fits one block's worth of threads per
  // CTA, and the columns fit the cluster's shared memory. TICTAC_TAC_CLUSTER=0 disables it, =1 forces it
  // (tests); a forced block count (TICTAC_TAC_BLOCKS) keeps the grid kernels.
  const char* cl_env = std::getenv("TICTAC_TAC_CLUSTER");
  const bool cl_force = cl_env && std::atoi(cl_env) == 1, cl_off = cl_env && std::atoi(cl_env) == 0;
  const bool forced_blocks = std::getenv("TICTAC_TAC_BLOCKS") != nullptr;
  auto try_cluster = [&]() -> bool {
    CK(allow_max_dynamic_smem(reinterpret_cast<const void*>(tac_cluster_kernel)));
    CK(cudaFuncSetAttribute(reinterpret_cast<const void*>(tac_cluster_kernel),
                            cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    for (int cs = kClusterMax; cs >= 2; cs /= 2) {
      const int per = (R + cs - 1) / cs;
      const size_t smem = tac_cluster_smem(per);
      if (smem > 220 * 1024) return false;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs);
      cfg.blockDim = dim3(1024);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = cs;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      int nclusters = 0;
      if (cudaOccupancyMaxActiveClusters(&nclusters, tac_cluster_kernel, &cfg) != cudaSuccess || nclusters < 1) {
        cudaGetLastError();
        continue;
      }
      CK(cudaLaunchKernelEx(&cfg, tac_cluster_kernel, a, per));
      if (trace) std::fprintf(stderr, "[tac] cluster of %d CTAs, %d columns each\n", cs, per);
      return true;
    }
    return false;
  };
  int32_t smem_rows = S.rw->nrows, smem_succ = static_cast<int>(S.rw->succ.size());
  const bool one_block_fits = tac_smem_bytes(smem_rows, R, smem_succ) <= 220 * 1024;
  bool launched = false;
  // The DSMEM cluster kernel: every per-round value in the cluster's shared
  // memory. TICTAC_TAC_DSM=0 disables it, =1 forces it (tests).
  const char* dsm_env = std::getenv("TICTAC_TAC_DSM");
  const bool dsm_force = dsm_env && std::atoi(dsm_env) == 1, dsm_off = dsm_env && std::atoi(dsm_env) == 0;
  auto try_dsm = [&]() -> bool {
    const int cs = kClusterMax, per = (R + cs - 1) / cs, gper = (smem_rows + cs - 1) / cs;
    const int kown = (per + 1023) / 1024;
    const size_t smem = tac_dsm_smem(per, gper, R);
    // measured: 10^5 ops / 10^4 recvs 56 -> 47 ms (one column per thread);
    // with seven columns per thread (10^6 / 10^5) the grid kernels' 103 SMs
    // win (0.63 s against 1.34 s), so the default stops at two per thread
    if (smem > 220 * 1024 || kown > 8 || (!dsm_force && kown > 2)) return false;
    const void* fn = kown <= 1   ? reinterpret_cast<const void*>(tac_dsm_kernel<1>)
                     : kown <= 2 ? reinterpret_cast<const void*>(tac_dsm_kernel<2>)
                     : kown <= 4 ? reinterpret_cast<const void*>(tac_dsm_kernel<4>)
                                 : reinterpret_cast<const void*>(tac_dsm_kernel<8>);
    CK(allow_max_dynamic_smem(fn));
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(1024);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, fn, &cfg) != cudaSuccess || nclusters < 1) {
      cudaGetLastError();
      return false;
    }
    if (kown <= 1) CK(cudaLaunchKernelEx(&cfg, tac_dsm_kernel<1>, a, per, gper, smem_rows));
    else if (kown <= 2) CK(cudaLaunchKernelEx(&cfg, tac_dsm_kernel<2>, a, per, gper, smem_rows));
    else if (kown <= 4) CK(cudaLaunchKernelEx(&cfg, tac_dsm_kernel<4>, a, per, gper, smem_rows));
    else CK(cudaLaunchKernelEx(&cfg, tac_dsm_kernel<8>, a, per, gper, smem_rows));
    if (trace) std::fprintf(stderr, "[tac] DSMEM cluster of %d CTAs, %d columns and %d groups each\n", cs, per, gper);
    return true;
  };
  // The speculative cluster kernel: TICTAC_TAC_CSPEC=0 disables it, =1 forces it (tests).
  const char* cspec_env = std::getenv("TICTAC_TAC_CSPEC");
  const bool cspec_force = cspec_env && std::atoi(cspec_env) == 1, cspec_off = cspec_env && std::atoi(cspec_env) == 0;
  int trace_misses = -1;
  auto try_cspec = [&]() -> bool {
    const int cs = kClusterMax, per = (R + cs - 1) / cs, kown = (per + 1023) / 1024;
    int max_succ = 0;
    for (int c = 0; c < R; ++c) max_succ = std::max(max_succ, S.rw->succ_off[c + 1] - S.rw->succ_off[c]);
    const int kS = max_succ <= 1 ? 1 : 2;
    // 32-bit values when every duration sum fits (P <= all compute, M <= all recv time)
    int64_t total = 0;
    for (int v = 0; v < g->n; ++v) total += dur[v];
    const bool narrow = total < 0x7fff0000LL && !std::getenv("TICTAC_TAC_WIDE");
    const size_t smem = tac_cspec_smem(per, kS, R, narrow ? 4 : 8);
    if (smem > 220 * 1024 || kown > 8 || max_succ > 2) return false;
    using KF = void (*)(TacArgs, const uint32_t*, int, int, int*);
    KF fn = nullptr;
#define CSPEC_PICK(V)                                                                                          \
  (kS == 1 ? (kown <= 1   ? tac_cspec_kernel<1, 1, V>                                                          \
              : kown <= 2 ? tac_cspec_kernel<2, 1, V>                                                          \
              : kown <= 4 ? tac_cspec_kernel<4, 1, V>                                                          \
              : kown <= 7 ? tac_cspec_kernel<7, 1, V>                                                          \
                          : tac_cspec_kernel<8, 1, V>)                                                         \
           : (kown <= 1   ? tac_cspec_kernel<1, 2, V>                                                          \
              : kown <= 2 ? tac_cspec_kernel<2, 2, V>                                                          \
              : kown <= 4 ? tac_cspec_kernel<4, 2, V>                                                          \
                          : tac_cspec_kernel<8, 2, V>))
    fn = narrow ? CSPEC_PICK(int) : CSPEC_PICK(long long);
#undef CSPEC_PICK
    CK(allow_max_dynamic_smem(reinterpret_cast<const void*>(fn)));
    CK(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(1024);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, fn, &cfg) != cudaSuccess || nclusters < 1) {
      cudaGetLastError();
      return false;
    }
    DevArr d_tr;
    if (alloc<int>(d_tr, 2, err)) return false;
    CK(cudaMemset(d_tr.p, 0, 8));
    int* tp = d_tr.as<int>();
    const uint32_t* bp = S.d_bits.as<uint32_t>();
    const int Wd = S.rw->W;
    CK(cudaLaunchKernelEx(&cfg, fn, a, bp, Wd, per, tp));
    if (trace) {
      int tr[2] = {0, 0};
      CK(cudaMemcpy(tr, tp, 8, cudaMemcpyDeviceToHost));
      trace_misses = tr[0];
      std::fprintf(stderr, "[tac] speculative cluster of %d CTAs, %d columns each, %d fixup intervals, %d misspeculated\n",
                   cs, per, tr[1], tr[0]);
    }
    return true;
  };
  if (cspec_force || (!cspec_off && !dsm_force && !cl_force && !forced_blocks && !one_block_fits)) launched = try_cspec();
  if (!launched && (dsm_force || (!dsm_off && !cl_force && !forced_blocks && !one_block_fits))) launched = try_dsm();
  // (measured: 10^5 ops / 10^4 recvs 61 → 55 ms; at 10^6 / 10^5 the grid
  // kernels' memory parallelism over 100+ SMs wins, 0.80 s vs 1.23 s)
  if (!launched && (cl_force || (!cl_off && !forced_blocks && blocks == 1 && !one_block_fits)))
    launched = try_cluster();
  if (launched) {
    // (cluster kernel in flight; completion below)
  } else if (blocks == 1) {
    int nrows = S.rw->nrows, nsucc = static_cast<int>(S.rw->succ.size());
    size_t smem = tac_smem_bytes(nrows, R, nsucc);
    constexpr size_t kSmemMax = 220 * 1024;
    // column lists in shared memory too when 16-bit row ids fit beside the state
    int ncol = 0;
    if (nrows < 65536 && S.nnz > 0 && smem + tac_smem_col_bytes(S.nnz) <= kSmemMax &&
        !std::getenv("TICTAC_TAC_NO_SMEM_COL")) {
      ncol = static_cast<int>(S.nnz);
      smem += tac_smem_col_bytes(ncol);
    }
    if (smem <= kSmemMax && !std::getenv("TICTAC_TAC_NO_SMEM")) {
      CK(allow_max_dynamic_smem(reinterpret_cast<const void*>(tac_smem_kernel)));
      void* args[] = {&a, &nrows, &nsucc, &ncol};
      // a block sized to the per-round work: idle warps only lengthen barriers
      int threads = R <= 512 ? 512 : 1024;
      if (const char* env = std::getenv("TICTAC_TAC_THREADS")) threads = std::max(32, std::min(1024, std::atoi(env)));
      CK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(tac_smem_kernel), 1, threads, args, smem, nullptr));
    } else {
      void* args[] = {&a};
      CK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(tac_kernel), 1, 1024, args, 0, nullptr));
    }
  } else {
    DevArr d_ring;
    const std::vector<int32_t> ring = {0x7fffffff, 0x7fffffff, 0x7fffffff, 0};  // [3]: steps taken (trace)
    if (put(d_ring, ring, err)) return 1;
    int* rp = d_ring.as<int>();
    void* args[] = {&a, &rp};
    // register-resident candidates when every column has an owner slot
    const int64_t per = (R + static_cast<int64_t>(blocks) * 1024 - 1) / (static_cast<int64_t>(blocks) * 1024);
    DevArr d_win;  // per-block winner slots of tac_own_kernel (3-slot ring)
    if (alloc<longlong4>(d_win, 3ull * blocks, err)) return 1;
    longlong4* wp = d_win.as<longlong4>();
    void* args_own[] = {&a, &rp, &wp};
    void* kern = reinterpret_cast<void*>(tac_dist_kernel);
    // the speculative kernel when every column's direct-successor groups fit
    // its registers (TICTAC_TAC_SPEC=0: tac_own_kernel)
    int max_succ = 0;
    for (int c = 0; c < R; ++c) max_succ = std::max(max_succ, S.rw->succ_off[c + 1] - S.rw->succ_off[c]);
    const char* spec_env = std::getenv("TICTAC_TAC_SPEC");
    if (!std::getenv("TICTAC_TAC_NO_OWN") && !(spec_env && std::atoi(spec_env) == 0) && per <= 4 &&
        max_succ <= kSpecS) {
      DevArr d_D, d_flag, d_pub;
      if (alloc<long long>(d_D, 4ull * R, err) || alloc<int>(d_flag, 4, err) || alloc<longlong4>(d_pub, 2, err))
        return 1;
      CK(cudaMemset(d_D.p, 0, 32ull * R));
      CK(cudaMemset(d_flag.p, 0, 16));
      TacSpecWs ws{S.d_bits.as<uint32_t>(), S.rw->W, d_D.as<long long>(), d_flag.as<int>(), d_pub.as<longlong4>(), rp, wp};
      void* args_spec[] = {&a, &ws};
      void* sk = nullptr;
      if (max_succ <= 1)
        sk = per <= 1 ? reinterpret_cast<void*>(tac_spec_kernel<1, 1>)
             : per <= 2 ? reinterpret_cast<void*>(tac_spec_kernel<2, 1>)
                        : reinterpret_cast<void*>(tac_spec_kernel<4, 1>);
      else if (max_succ <= 2)
        sk = per <= 1 ? reinterpret_cast<void*>(tac_spec_kernel<1, 2>)
             : per <= 2 ? reinterpret_cast<void*>(tac_spec_kernel<2, 2>)
                        : reinterpret_cast<void*>(tac_spec_kernel<4, 2>);
      else
        sk = per <= 1 ? reinterpret_cast<void*>(tac_spec_kernel<1, 4>)
             : per <= 2 ? reinterpret_cast<void*>(tac_spec_kernel<2, 4>)
                        : reinterpret_cast<void*>(tac_spec_kernel<4, 4>);
      const size_t spec_smem = 4ull * ((R + 31) / 32);
      CK(allow_max_dynamic_smem(sk));
      int per_sm_spec = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_spec, sk, 1024, spec_smem));
      if (spec_smem <= 200 * 1024 && per_sm_spec * sms >= blocks) {
        CK(cudaLaunchCooperativeKernel(sk, blocks, 1024, args_spec, spec_smem, nullptr));
        LAUNCHED();
        CK(cudaGetLastError());
        CK(cudaMemcpy(prio, d_prio.p, 4ull * R, cudaMemcpyDeviceToHost));
        if (trace) {
          int misses = 0;
          CK(cudaMemcpy(&misses, rp + 3, 4, cudaMemcpyDeviceToHost));
          std::fprintf(stderr, "[tac] setup %.3f ms, state %.3f ms, rounds (%d blocks, speculative) %.3f ms, %d misspeculated\n",
                       ms(t0, t1), ms(t1, t2), blocks, ms(t2, now()), misses);
        }
        return 0;
      }
    }
    if (!std::getenv("TICTAC_TAC_NO_OWN")) {
      if (per <= 1)
        kern = reinterpret_cast<void*>(tac_own_kernel<1>);
      else if (per <= 2)
        kern = reinterpret_cast<void*>(tac_own_kernel<2>);
      else if (per <= 4)
        kern = reinterpret_cast<void*>(tac_own_kernel<4>);
    }
    CK(cudaLaunchCooperativeKernel(kern, blocks, 1024, kern == reinterpret_cast<void*>(tac_dist_kernel) ? args : args_own,
                                   0, nullptr));
    LAUNCHED();
    CK(cudaGetLastError());
    CK(cudaMemcpy(prio, d_prio.p, 4ull * R, cudaMemcpyDeviceToHost));
    if (trace) {
      int steps = 0;
      CK(cudaMemcpy(&steps, rp + 3, 4, cudaMemcpyDeviceToHost));
      std::fprintf(stderr, "[tac] setup %.3f ms, state %.3f ms, rounds (%d blocks) %.3f ms, %d find-first steps\n",
                   ms(t0, t1), ms(t1, t2), blocks, ms(t2, now()), steps);
    }
    return 0;
  }
  LAUNCHED();
  CK(cudaGetLastError());
  CK(cudaMemcpy(prio, d_prio.p, 4ull * R, cudaMemcpyDeviceToHost));
  if (trace)
    std::fprintf(stderr, "[tac] setup %.3f ms, state %.3f ms, rounds (%s) %.3f ms\n", ms(t0, t1), ms(t1, t2),
                 launched ? "cluster" : "1 block", ms(t2, now()));
  return 0;
}

// SURVEY §8d TAC traffic inputs from the device closure: out[0] V, [1] R,
// [2] E, [3] E_recv (edges leaving recvs), [4] nnz = Σ_r |{ops depending on
// r}| (recvs count themselves, properties.cpp:19-66), [5] closure rows,
// [6] row-level (row, recv) pairs the kernels actually retire over.
extern "C" int csk_tac_stats(DeviceGraph* g, const int64_t* dur, int64_t* out, char* err) {
  for (int k = 0; k < 7; ++k) out[k] = 0;
  out[0] = g->n;
  out[1] = g->R;
  out[2] = g->h_succ_off.empty() ? 0 : g->h_succ_off.back();
  for (int32_t v = 0; v < g->n; ++v)
    if (g->h_kind[v] == 1) out[3] += g->h_succ_off[v + 1] - g->h_succ_off[v];
  if (g->R == 0) return 0;
  GroupState S;
  if (group_setup(g, dur, S, err)) return 1;
  std::vector<int32_t> cnt(std::max(S.rw->nrows, 1));
  if (S.rw->nrows > 0) CK(cudaMemcpy(cnt.data(), S.d_cnt.p, 4ull * S.rw->nrows, cudaMemcpyDeviceToHost));
  int64_t nnz = 0;
  for (int32_t v = 0; v < g->n; ++v) nnz += g->h_kind[v] == 1 ? 1 : cnt[S.rw->row_of[v]];
  out[4] = nnz;
  out[5] = S.rw->nrows;
  out[6] = S.nnz;
  return 0;
}
