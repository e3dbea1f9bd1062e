// Exact event simulator on the GPU — replicas of the reference's
// discrete-event loop (sim.cpp:61-256) for everything outside the closed form
// of SURVEY Appendix A.2, and for event lists.
//
// event_sim_kernel<kL, S>: the general replica. Per-resource ready queues are
// bitsets over that resource's ops (ascending op index = the reference's
// sorted queue); fully prioritized channels also index their ready ops by
// rank, so a start walks from the lowest ready rank. The choice stream is the
// reference's mt19937_64 (shared by all resources, consumed in round order),
// the reorder-noise stream is Rng(splitmix64(choice_seed ^ salt)) consumed in
// resource order. Two run shapes: a thread per run (kL = 1, batches, state
// lane-interleaved in HBM) and a warp per run (kL = 32, small batches, state in
// shared memory, the chain on lane 0).
//
// event_a2_kernel: one run inside A.2's regime (one compute unit + one
// channel, gated, noiseless, recvs prioritized) for its event list — the same
// round structure with the channel reduced to "next recv in gate order" and
// both resources' state in registers.
//
// Used for batches and sweeps outside the closed form, brute force outside
// it, and every report's event list.
#include <algorithm>
#include <climits>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "csk.h"
#include "devgraph.cuh"

namespace tictac_dev {

namespace {

constexpr int kWarpsPerBlock = 4;
constexpr int64_t kThreadModeMin = 2048;        // batch size from which a thread runs a whole sim
constexpr int kThreadMinBlocks = 6;            // thread mode: 24 resident warps/SM (<= 85 registers)
constexpr size_t kThreadScratch = 16ull << 30;  // cap on thread-mode state in HBM
constexpr int kEmptyLo = 1 << 29;  // "no ready word" (no overflow when lanes are added)

struct GraphView {
  int32_t n, nres, ndev, R;
  const int32_t *pred_off, *succ_off, *succ_idx, *res, *res_dev, *rops_off, *rops, *lidx, *rb_off,
      *recv_ops;
  const int8_t* chan;
  const int64_t* dur;
};

// How a run obtains its priorities.
enum PrioMode : int { kPrioExplicit = 0, kPrioOrders = 1, kPrioRandom = 2, kPrioLex = 3 };

struct RunSpec {
  int mode;
  const int32_t* prio;    // kPrioExplicit: [B][n]
  const int32_t* orders;  // kPrioOrders: [B][R]
  uint64_t seed_lo;       // kPrioRandom: seed = seed_lo + b ; kPrioLex: choice seed
  const uint64_t* seeds;  // per-run choice seeds (explicit/orders modes)
  int cluster;            // kPrioRandom: derive per-worker seeds
  const int32_t* wcols_off;  // kPrioRandom: worker w's recv columns
  const int32_t* wcols;
  int32_t n_workers;
  const uint64_t* lim;    // bounded() constants for n = 0..R
  const uint64_t* mag;
  int gated;
  double noise;
  int64_t* makespan;
  int64_t* violations;
  int32_t* status;
  int64_t* start;  // run 0 only
  int64_t* end;
  int64_t* dev_end;  // [B][ndev]
};

// Per-run state. "Hot" arrays (touched every event) live in shared memory
// when a slot fits, else in global scratch; "cold" arrays always in global.
//
// Two run shapes share one kernel body (template kL = lanes per run):
//  kL = 32: a warp per run — setup and violation counting spread over the
//           lanes, the event chain on lane 0 (few, long runs);
//  kL = 1:  a thread per run, 32 runs per warp in lockstep — for large
//           batches. State is lane-interleaved (element i of lane l at
//           [i * 32 + l], stride S = 32), so the per-resource loops that all
//           lanes walk in the same order coalesce into one line per access.
template <typename T, int S>
struct Arr {
  T* p;
  __device__ __forceinline__ T& operator[](int64_t i) const { return p[i * S]; }
};

template <int S>
struct Slot {
  // hot
  Arr<int32_t, S> missing, gate, running, comp_len, ready_cnt, lo, hi, haspri;
  Arr<uint32_t, S> ready, forced, rready, pmask;
  Arr<int64_t, S> run_end, counter;
  Arr<uint64_t, S> mt;
  // cold
  Arr<int32_t, S> orig, seq, prio, items, comp, rop;
  Arr<int64_t, S> dev_end;
  Arr<uint64_t, S> mt2;
};

__host__ __device__ inline size_t align8(size_t x) { return (x + 7) & ~size_t(7); }

// Bytes of one slot group (S runs interleaved; S = 1 for a warp-per-run slot).
__host__ __device__ inline size_t hot_bytes(int n, int nres, int rbw, int S = 1) {
  return align8(4ull * n * S) * 2 + align8(4ull * nres * S) * 6 + align8(4ull * (rbw + 1) * S) * 3 +
         align8(4ull * ((n + 31) / 32 + 1) * S) + align8(8ull * nres * S) * 2 + 8ull * 312 * S;
}

__host__ __device__ inline size_t cold_bytes(int n, int ndev, int R, int S = 1) {
  return align8(4ull * n * S) * 5 + align8(4ull * (R + 1) * S) + align8(8ull * (ndev + 1) * S) +
         8ull * 312 * S;
}

template <int S>
__device__ Slot<S> carve(char* hot, char* cold, int lane, int n, int nres, int ndev, int rbw, int R) {
  Slot<S> s;
  auto take = [lane](auto& arr, char*& base, size_t count) {
    using T = typename std::remove_reference_t<decltype(*arr.p)>;
    arr.p = reinterpret_cast<T*>(base) + lane;
    base += align8(sizeof(T) * count * S);
  };
  take(s.missing, hot, n);
  take(s.gate, hot, n);
  take(s.running, hot, nres);
  take(s.comp_len, hot, nres);
  take(s.ready_cnt, hot, nres);
  take(s.lo, hot, nres);
  take(s.hi, hot, nres);
  take(s.haspri, hot, nres);
  take(s.ready, hot, rbw + 1);
  take(s.rready, hot, rbw + 1);
  take(s.pmask, hot, rbw + 1);
  take(s.forced, hot, (n + 31) / 32 + 1);
  take(s.run_end, hot, nres);
  take(s.counter, hot, nres);
  take(s.mt, hot, 312);
  take(s.orig, cold, n);
  take(s.seq, cold, n);
  take(s.prio, cold, n);
  take(s.comp, cold, n);
  take(s.rop, cold, n);
  take(s.items, cold, R + 1);
  take(s.dev_end, cold, ndev + 1);
  take(s.mt2, cold, 312);
  return s;
}

// Serial helpers over a full mt19937_64 state in scratch.
template <typename M>
__device__ uint64_t bounded_full(M& m, uint64_t n, const RunSpec& rs) {
  if (n < 2) return 0;
  uint64_t lim, mag;
  if (n <= static_cast<uint64_t>(0x7fffffff) && rs.lim && n < 4096) {
    lim = rs.lim[n];
    mag = rs.mag[n];
    uint64_t v;
    do v = m.next();
    while (v > lim);
    return fastmod(v, n, mag);
  }
  const uint64_t limit = UINT64_MAX - (UINT64_MAX % n + 1) % n;
  uint64_t v;
  do v = m.next();
  while (v > limit);
  return v % n;
}

template <int S>
__device__ __forceinline__ bool admitted(const Slot<S>& s, int op, int r, int gated) {
  const int gt = s.gate[op];
  if (!gated || gt < 0) return true;
  if ((s.forced[op >> 5] >> (op & 31)) & 1u) return true;
  return static_cast<int64_t>(gt) <= s.counter[r];
}

template <int kL>
__device__ __forceinline__ void group_sync() {
  if constexpr (kL == 32) __syncwarp();
}

template <int kL, int S>
__device__ void fill_priorities(const GraphView& G, const RunSpec& rs, const Slot<S>& s, int64_t b,
                                int lane, uint64_t* choice_seed) {
  const int n = G.n;
  if (rs.mode == kPrioExplicit) {
    const int32_t* p = rs.prio + b * n;
    for (int i = lane; i < n; i += kL) s.prio[i] = p[i];
    *choice_seed = rs.seeds[b];
    return;
  }
  for (int i = lane; i < n; i += kL) s.prio[i] = -1;
  group_sync<kL>();
  if (rs.mode == kPrioOrders) {
    const int32_t* o = rs.orders + b * G.R;
    for (int k = lane; k < G.R; k += kL) s.prio[G.recv_ops[o[k]]] = k;
    *choice_seed = rs.seeds[b];
  } else if (rs.mode == kPrioLex) {
    *choice_seed = rs.seed_lo;
    if (lane == 0) {  // unrank b in the factorial number system
      const int R = G.R;
      for (int k = 0; k < R; ++k) s.items[k] = k;
      int64_t f = 1;
      for (int k = 2; k < R; ++k) f *= k;
      int64_t rem = b;
      for (int pos = 0; pos < R; ++pos) {
        const int64_t q = f ? rem / f : 0;
        rem = f ? rem % f : 0;
        const int pick = s.items[q];
        for (int k = static_cast<int>(q); k + 1 < R - pos; ++k) s.items[k] = s.items[k + 1];
        s.prio[G.recv_ops[pick]] = pos;
        if (R - 1 - pos > 0) f /= (R - 1 - pos);
      }
    }
  } else {  // kPrioRandom: random_schedule per worker (schedule_for)
    const uint64_t seed = rs.seed_lo + static_cast<uint64_t>(b);
    *choice_seed = seed;
    if (lane == 0) {
      for (int w = 0; w < rs.n_workers; ++w) {
        const int c0 = rs.wcols_off[w], Rw = rs.wcols_off[w + 1] - c0;
        const uint64_t ws = rs.cluster ? splitmix64(seed ^ (kPhi * static_cast<uint64_t>(w + 1))) : seed;
        for (int k = 0; k < Rw; ++k) s.items[k] = k;
        MtLazyP<Arr<uint64_t, S>> m;  // register cursors (R <= 311 draws), scratch state beyond
        m.full = {s.mt2, 0};
        m.seed(ws);
        for (int i = Rw; i > 1; --i) {
          const int j = static_cast<int>(bounded_full(m, static_cast<uint64_t>(i), rs));
          const int t = s.items[i - 1];
          s.items[i - 1] = s.items[j];
          s.items[j] = t;
        }
        for (int k = 0; k < Rw; ++k) s.prio[G.recv_ops[rs.wcols[c0 + s.items[k]]]] = k;
      }
    }
  }
  group_sync<kL>();
}

template <int kL, int S>
__global__ void __launch_bounds__(32 * kWarpsPerBlock, kL == 1 ? kThreadMinBlocks : 4)
    event_sim_kernel(GraphView G, RunSpec rs, int64_t B, char* hot_global, size_t hot_sz, char* cold_scr,
                     size_t cold_sz, int rbw) {
  // S = element stride of the per-run state: 32 = lane-interleaved groups of
  // 32 runs (one per warp), 1 = each run's state contiguous
  extern __shared__ __align__(16) char smem_hot[];
  const int lane = kL == 32 ? (threadIdx.x & 31) : 0;
  const int64_t gtid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t slot_id = kL == 32 ? (gtid >> 5) : gtid;
  const int64_t unit = S == 32 ? (gtid >> 5) : slot_id;  // index of this thread's state block
  const int64_t nslots = (static_cast<int64_t>(gridDim.x) * blockDim.x) / kL;
  char* hot = hot_global ? hot_global + unit * hot_sz : smem_hot + (threadIdx.x >> 5) * hot_sz;
  const Slot<S> s = carve<S>(hot, cold_scr + unit * cold_sz, S == 32 ? (threadIdx.x & 31) : 0, G.n, G.nres,
                             G.ndev, rbw, G.R);
  const int n = G.n, nres = G.nres;

  for (int64_t b = slot_id; b < B; b += nslots) {
    uint64_t choice_seed = 0;
    fill_priorities<kL>(G, rs, s, b, lane, &choice_seed);
    // ---- setup (sim.cpp:74-123)
    for (int w = lane; w < rbw; w += kL) {
      s.ready[w] = 0;
      s.rready[w] = 0;
      s.pmask[w] = 0;
    }
    for (int w = lane; w < (n + 31) / 32; w += kL) s.forced[w] = 0;
    for (int r = lane; r < nres; r += kL) {
      s.running[r] = -1;
      s.run_end[r] = 0;
      s.counter[r] = 0;
      s.comp_len[r] = 0;
      s.ready_cnt[r] = 0;
      s.lo[r] = kEmptyLo;  // scan window of non-empty ready words (empty: lo > hi)
      s.hi[r] = -1;
      s.haspri[r] = 0;
    }
    for (int d = lane; d < G.ndev; d += kL) s.dev_end[d] = 0;
    group_sync<kL>();
    const bool explicit_prio = rs.mode == kPrioExplicit;
    for (int i = lane; i < n; i += kL) {
      const int deg = G.pred_off[i + 1] - G.pred_off[i];
      s.missing[i] = deg;
      s.gate[i] = -1;
      s.orig[i] = -1;
      if (explicit_prio && s.prio[i] >= 0) s.haspri[G.res[i]] = 1;
      if (deg == 0) {
        const int r = G.res[i], l = G.lidx[i];
        if constexpr (kL == 32) {
          atomicOr(&s.ready[G.rb_off[r] + (l >> 5)], 1u << (l & 31));
          atomicAdd(&s.ready_cnt[r], 1);
          atomicMin(&s.lo[r], l >> 5);
          atomicMax(&s.hi[r], l >> 5);
        } else {
          s.ready[G.rb_off[r] + (l >> 5)] |= 1u << (l & 31);
          s.ready_cnt[r] += 1;
          s.lo[r] = min(s.lo[r], l >> 5);
          s.hi[r] = max(s.hi[r], l >> 5);
        }
      }
    }
    if (!explicit_prio)  // only recvs carry priorities
      for (int k = lane; k < G.R; k += kL) {
        const int i = G.recv_ops[k];
        if (s.prio[i] >= 0) s.haspri[G.res[i]] = 1;
      }
    // dense per-channel ranks from (priority, id), then noise swaps
    MtLazyP<Arr<uint64_t, S>> noise;
    noise.full = {s.mt2, 0};
    const bool noisy = rs.gated && rs.noise > 0.0;
    if (lane == 0 && noisy) noise.seed(splitmix64(choice_seed ^ kNoiseSalt));
    for (int r = 0; r < nres; ++r) {
      if (!G.chan[r]) continue;
      const int o0 = G.rops_off[r], o1 = G.rops_off[r + 1];
      int mine = 0;
      if (kL == 1 && rs.mode != kPrioExplicit) {
        // priorities here are positions in a permutation, so distinct: rank
        // by walking the values instead of counting pairs (items = scratch)
        int pmin = 0x7fffffff, pmax = -1;
        for (int a = o0; a < o1; ++a) {
          const int i = G.rops[a];
          const int pi = s.prio[i];
          if (pi < 0) continue;
          s.items[pi] = i;
          pmin = min(pmin, pi);
          pmax = max(pmax, pi);
        }
        for (int p = pmin; p <= pmax; ++p) {
          const int i = s.items[p];
          // stale (or never written) entry from another channel
          if (static_cast<unsigned>(i) >= static_cast<unsigned>(n) || G.res[i] != r || s.prio[i] != p) continue;
          s.orig[i] = mine;
          s.seq[o0 + mine] = i;
          s.rop[o0 + mine] = i;
          ++mine;
        }
      } else
      for (int a = o0 + lane; a < o1; a += kL) {
        const int i = G.rops[a];
        const int pi = s.prio[i];
        if (pi < 0) continue;
        int rank = 0;
        for (int c = o0; c < o1; ++c) {
          const int j = G.rops[c];
          const int pj = s.prio[j];
          rank += (pj >= 0) && (pj < pi || (pj == pi && j < i));
        }
        s.orig[i] = rank;
        s.seq[o0 + rank] = i;
        s.rop[o0 + rank] = i;
        ++mine;
      }
      int k = mine;
      if constexpr (kL == 32) k = warp_sum(mine);
      group_sync<kL>();
      if (k > 0 && k == o1 - o0) {
        // every op on the channel is prioritized: also index ready ops by
        // rank, so a start walks from the lowest ready rank (try_start)
        if (lane == 0) s.haspri[r] = 2;
        for (int a = o0 + lane; a < o1; a += kL) {
          const int i = G.rops[a];
          if (s.missing[i] != 0) continue;
          const int q = s.orig[i];
          if constexpr (kL == 32)
            atomicOr(&s.rready[G.rb_off[r] + (q >> 5)], 1u << (q & 31));
          else
            s.rready[G.rb_off[r] + (q >> 5)] |= 1u << (q & 31);
        }
        group_sync<kL>();
      } else if (k > 0) {
        // prioritized and unprioritized ops share the channel (a worker's
        // recvs and gradient sends): prioritized ready ops indexed by rank
        // as above, the others found through the complement of pmask
        if (lane == 0) s.haspri[r] = 3;
        for (int a = o0 + lane; a < o1; a += kL) {
          const int i = G.rops[a];
          const int q = s.orig[i];
          if (q < 0) continue;
          const int l = G.lidx[i];
          if constexpr (kL == 32) {
            atomicOr(&s.pmask[G.rb_off[r] + (l >> 5)], 1u << (l & 31));
            if (s.missing[i] == 0) atomicOr(&s.rready[G.rb_off[r] + (q >> 5)], 1u << (q & 31));
          } else {
            s.pmask[G.rb_off[r] + (l >> 5)] |= 1u << (l & 31);
            if (s.missing[i] == 0) s.rready[G.rb_off[r] + (q >> 5)] |= 1u << (q & 31);
          }
        }
        group_sync<kL>();
      }
      if (!rs.gated) continue;
      if (lane == 0 && noisy)
        for (int p = 1; p < k; ++p) {
          const double u = static_cast<double>(noise.next() >> 11) * 0x1.0p-53;
          if (u < rs.noise) {
            const int t = s.seq[o0 + p - 1];
            s.seq[o0 + p - 1] = s.seq[o0 + p];
            s.seq[o0 + p] = t;
          }
        }
      group_sync<kL>();
      for (int p = lane; p < k; p += kL) s.gate[s.seq[o0 + p]] = p;
      group_sync<kL>();
    }
    MtInPlaceP<Arr<uint64_t, S>> choice{s.mt, 0};
    if (lane == 0) choice.seed(choice_seed);
    group_sync<kL>();

    // ---- event loop (sim.cpp:194-233), run serially by lane 0 on the
    // shared-memory state: the replica is a dependent chain, and warp-wide
    // bookkeeping per event costs more than it saves. Resources that could
    // start are tracked in a bitmask so each pass visits only those, still in
    // ascending resource order (the order of the reference's draws).
    int64_t t = 0, mk = 0, nforced = 0;
    int stalled = 0;
    const int gated = rs.gated;
    const bool rec = (b == 0) && rs.start;
    if (lane == 0) {
      int finished = 0;
      // With <= 64 resources, three masks replace the per-step scans over all
      // resources (same visiting order, ascending r): avail = idle with ready
      // ops (try_start candidates), busy = running, due = running and ending
      // at the current t (complete_now). Above 64 the scans run as written.
      const bool small = nres <= 64;
      uint64_t avail = 0, busy = 0, due = 0;
      if (small)
        for (int r = 0; r < nres; ++r)
          if (s.ready_cnt[r] > 0) avail |= 1ull << r;
      auto start_op = [&](int r, int op) {
        const int l = G.lidx[op];
        s.ready[G.rb_off[r] + (l >> 5)] &= ~(1u << (l & 31));
        if (s.haspri[r] >= 2) {
          const int q = s.orig[op];
          if (q >= 0) s.rready[G.rb_off[r] + (q >> 5)] &= ~(1u << (q & 31));
        }
        s.ready_cnt[r] -= 1;
        s.running[r] = op;
        const int64_t e = t + G.dur[op];
        s.run_end[r] = e;
        if (rec) {
          rs.start[op] = t;
          rs.end[op] = e;
        }
        const int d = G.res_dev[r];
        if (e > s.dev_end[d]) s.dev_end[d] = e;
        mk = max(mk, e);
        if (small) {
          avail &= ~(1ull << r);
          busy |= 1ull << r;
          if (e == t) due |= 1ull << r;
        }
      };
      // sim.cpp:163-192 for one resource; returns true when an op started
      auto try_start = [&](int r) -> bool {
        if (s.running[r] >= 0 || s.ready_cnt[r] == 0) return false;
        if (s.haspri[r] == 2) {
          // Fully prioritized channel: ranks ascend with (priority, id), so
          // the reference's candidates (admitted ops at the minimum admitted
          // priority, in id order) are the admitted ops of one equal-priority
          // run of ranks, starting at the first admitted ready rank.
          const int wb = G.rb_off[r], o0 = G.rops_off[r];
          const int nw = (G.rops_off[r + 1] - o0 + 31) >> 5;
          int best = -1, total = 0;
          bool done = false;
          for (int w = 0; w < nw && !done; ++w) {
            uint32_t bits = s.rready[wb + w];
            while (bits) {
              const int bit = __ffs(bits) - 1;
              bits &= bits - 1;
              const int op = s.rop[o0 + (w << 5) + bit];
              const int p = s.prio[op];
              if (best >= 0 && p != best) {
                done = true;
                break;
              }
              if (admitted(s, op, r, gated)) {
                best = p;
                ++total;
              }
            }
          }
          if (total == 0) return false;
          int k = total > 1 ? static_cast<int>(bounded_full(choice, static_cast<uint64_t>(total), rs)) : 0;
          for (int w = 0; w < nw; ++w) {
            uint32_t bits = s.rready[wb + w];
            while (bits) {
              const int bit = __ffs(bits) - 1;
              bits &= bits - 1;
              const int op = s.rop[o0 + (w << 5) + bit];
              if (s.prio[op] != best || !admitted(s, op, r, gated)) continue;
              if (k-- == 0) {
                start_op(r, op);
                return true;
              }
            }
          }
          return false;  // unreachable
        }
        if (s.haspri[r] == 3) {
          // candidates (sim.cpp:170-181): every ready unprioritized op, plus
          // the admitted ready ops at the minimum admitted priority — the
          // admitted ops of one equal-priority run of ranks (ranks ascend
          // with (priority, id)) — merged in op-index order
          const int wb = G.rb_off[r], o0 = G.rops_off[r];
          const int nw = (G.rops_off[r + 1] - o0 + 31) >> 5;
          constexpr int kMaxBest = 2;  // tied best-priority candidates kept in registers
          int bl0 = -1, bl1 = -1;
          int best = -1, nb = 0;
          bool done = false;
          for (int w = 0; w < nw && !done; ++w) {
            uint32_t bits = s.rready[wb + w];
            while (bits) {
              const int bit = __ffs(bits) - 1;
              bits &= bits - 1;
              const int op = s.rop[o0 + (w << 5) + bit];
              const int p = s.prio[op];
              if (best >= 0 && p != best) {
                done = true;
                break;
              }
              if (admitted(s, op, r, gated)) {
                best = p;
                if (nb == 0) bl0 = G.lidx[op];
                else if (nb == 1) bl1 = G.lidx[op];
                ++nb;
              }
            }
          }
          if (nb <= kMaxBest) {
            int nu = 0;
            for (int w = s.lo[r], wh = s.hi[r]; w <= wh; ++w) nu += __popc(s.ready[wb + w] & ~s.pmask[wb + w]);
            const int total = nu + nb;
            if (total == 0) return false;
            int k = total > 1 ? static_cast<int>(bounded_full(choice, static_cast<uint64_t>(total), rs)) : 0;
            for (int w = s.lo[r], wh = s.hi[r]; w <= wh; ++w) {
              uint32_t m = s.ready[wb + w] & ~s.pmask[wb + w];
              if (nb > 0 && (bl0 >> 5) == w) m |= 1u << (bl0 & 31);
              if (nb > 1 && (bl1 >> 5) == w) m |= 1u << (bl1 & 31);
              const int c = __popc(m);
              if (k < c) {
                start_op(r, G.rops[o0 + (w << 5) + nth_bit(m, k)]);
                return true;
              }
              k -= c;
            }
            return false;  // unreachable
          }
          // more than kMaxBest tied candidates: the general scan below
        }
        const bool pri = s.haspri[r] != 0;
        const int wb = G.rb_off[r], ob = G.rops_off[r];
        if (!pri) {
          // no priorities here: every ready op is a candidate, so draw over
          // ready_cnt and walk once to the k-th ready op (tightening lo)
          const int total = s.ready_cnt[r];
          int k = total > 1 ? static_cast<int>(bounded_full(choice, static_cast<uint64_t>(total), rs)) : 0;
          bool seen = false;
          for (int w = s.lo[r], wh = s.hi[r]; w <= wh; ++w) {
            const uint32_t bits = s.ready[wb + w];
            if (!bits) continue;
            if (!seen) {
              s.lo[r] = w;
              seen = true;
            }
            const int c = __popc(bits);
            if (k < c) {
              start_op(r, G.rops[ob + (w << 5) + nth_bit(bits, k)]);
              return true;
            }
            k -= c;
          }
          return false;  // unreachable: ready_cnt counts the set bits
        }
        int nlo = kEmptyLo, nhi = -1, best = 0x7fffffff;
        for (int w = s.lo[r]; w <= s.hi[r]; ++w) {
          uint32_t bits = s.ready[wb + w];
          if (!bits) continue;
          nlo = min(nlo, w);
          nhi = w;
          if (!pri) continue;
          while (bits) {
            const int bit = __ffs(bits) - 1;
            bits &= bits - 1;
            const int op = G.rops[ob + (w << 5) + bit];
            const int p = s.prio[op];
            if (p >= 0 && p < best && admitted(s, op, r, gated)) best = p;
          }
        }
        s.lo[r] = nlo;
        s.hi[r] = nhi;
        auto cmask = [&](int w) -> uint32_t {
          uint32_t bits = s.ready[wb + w];
          if (!pri) return bits;
          uint32_t m = 0;
          while (bits) {
            const int bit = __ffs(bits) - 1;
            bits &= bits - 1;
            const int op = G.rops[ob + (w << 5) + bit];
            const int p = s.prio[op];
            if (p < 0 || (p == best && admitted(s, op, r, gated))) m |= 1u << bit;
          }
          return m;
        };
        int total = 0;
        for (int w = nlo; w <= nhi; ++w) total += __popc(cmask(w));
        if (total == 0) return false;
        int k = total > 1 ? static_cast<int>(bounded_full(choice, static_cast<uint64_t>(total), rs)) : 0;
        for (int w = nlo; w <= nhi; ++w) {
          const uint32_t m = cmask(w);
          const int c = __popc(m);
          if (k < c) {
            start_op(r, G.rops[ob + (w << 5) + nth_bit(m, k)]);
            return true;
          }
          k -= c;
        }
        return false;  // unreachable
      };
      auto push_ready = [&](int w_op) {
        const int rw = G.res[w_op], l = G.lidx[w_op];
        s.ready[G.rb_off[rw] + (l >> 5)] |= 1u << (l & 31);
        if (s.haspri[rw] >= 2) {
          const int q = s.orig[w_op];
          if (q >= 0) s.rready[G.rb_off[rw] + (q >> 5)] |= 1u << (q & 31);
        }
        s.ready_cnt[rw] += 1;
        s.lo[rw] = min(s.lo[rw], l >> 5);
        s.hi[rw] = max(s.hi[rw], l >> 5);
        if (small && s.running[rw] < 0) avail |= 1ull << rw;
      };
      // sim.cpp:144-161
      auto complete_one = [&](int r, int i) {
        ++finished;
        s.running[r] = -1;
        if (G.chan[r] && s.prio[i] >= 0) {
          s.counter[r] += 1;
          s.comp[G.rops_off[r] + s.comp_len[r]] = s.orig[i];
          s.comp_len[r] += 1;
        }
        if (small) {
          busy &= ~(1ull << r);
          if (s.ready_cnt[r] > 0) avail |= 1ull << r;
        }
        for (int e = G.succ_off[i]; e < G.succ_off[i + 1]; ++e) {
          const int w = G.succ_idx[e];
          if (--s.missing[w] == 0) push_ready(w);
        }
      };
      auto complete_now = [&]() -> bool {
        if (small) {  // completions never start anything: `due` is stable here
          const bool any = due != 0;
          while (due) {
            const int r = __ffsll(static_cast<long long>(due)) - 1;
            due &= due - 1;
            complete_one(r, s.running[r]);
          }
          return any;
        }
        bool any = false;
        for (int r = 0; r < nres; ++r) {
          const int i = s.running[r];
          if (i < 0 || s.run_end[r] != t) continue;
          any = true;
          complete_one(r, i);
        }
        return any;
      };
      while (finished < n) {
        bool progress = true;
        while (progress) {
          progress = false;
          if (small && (avail | due) == 0) break;  // nothing can start or end at t
          if (small) {  // a start only clears its own resource's bit
            for (uint64_t m = avail; m; m &= m - 1)
              progress = try_start(__ffsll(static_cast<long long>(m)) - 1) || progress;
          } else {
            for (int r = 0; r < nres; ++r) progress = try_start(r) || progress;
          }
          progress = complete_now() || progress;
        }
        if (finished == n) break;
        int64_t next_t = INT64_MAX;
        if (small) {  // earliest end over running resources, and which end then
          due = 0;
          for (uint64_t m = busy; m; m &= m - 1) {
            const int r = __ffsll(static_cast<long long>(m)) - 1;
            const int64_t e = s.run_end[r];
            if (e < next_t) {
              next_t = e;
              due = 1ull << r;
            } else if (e == next_t) {
              due |= 1ull << r;
            }
          }
        } else {
          for (int r = 0; r < nres; ++r)
            if (s.running[r] >= 0) next_t = min(next_t, s.run_end[r]);
        }
        if (next_t == INT64_MAX) {  // forced release, sim.cpp:211-229
          int64_t key = INT64_MAX;
          for (int r = 0; r < nres; ++r)
            for (int w = s.lo[r]; w <= s.hi[r]; ++w) {
              uint32_t bits = s.ready[G.rb_off[r] + w];
              while (bits) {
                const int bit = __ffs(bits) - 1;
                bits &= bits - 1;
                const int op = G.rops[G.rops_off[r] + (w << 5) + bit];
                if (s.gate[op] < 0 || admitted(s, op, r, gated)) continue;
                key = min(key, (static_cast<int64_t>(s.gate[op]) << 32) | op);
              }
            }
          if (key == INT64_MAX) {
            stalled = 1;
            break;
          }
          const int victim = static_cast<int>(key & 0xffffffff);
          s.forced[victim >> 5] |= 1u << (victim & 31);
          ++nforced;
          continue;
        }
        t = next_t;
        complete_now();
      }
    }
    if constexpr (kL == 32) {
      __syncwarp();
      mk = __shfl_sync(~0u, mk, 0);
      nforced = __shfl_sync(~0u, nforced, 0);
      stalled = __shfl_sync(~0u, stalled, 0);
    }

    // violations: rank inversions per channel completion sequence + forced
    int64_t inv = 0;
    for (int r = 0; r < nres; ++r) {
      if (!G.chan[r]) continue;
      const int base = G.rops_off[r];
      const int len = s.comp_len[r];
      if constexpr (kL == 1) {
        // completion ranks are distinct and < the channel's op count: count
        // the smaller ranks seen to the right with a bitset (rready's segment
        // for this channel is free once the loop has ended)
        const int wb = G.rb_off[r], nw = (G.rops_off[r + 1] - base + 31) >> 5;
        for (int w = 0; w < nw; ++w) s.rready[wb + w] = 0;
        for (int a = len - 1; a >= 0; --a) {
          const int v = s.comp[base + a];
          int below = 0;
          for (int w = 0; w < (v >> 5); ++w) below += __popc(s.rready[wb + w]);
          below += __popc(s.rready[wb + (v >> 5)] & ((1u << (v & 31)) - 1u));
          inv += below;
          s.rready[wb + (v >> 5)] |= 1u << (v & 31);
        }
      } else {
        for (int a = lane; a < len; a += kL)
          for (int c = a + 1; c < len; ++c) inv += s.comp[base + a] > s.comp[base + c];
      }
    }
    if constexpr (kL == 32) {
#pragma unroll
      for (int o = 16; o; o >>= 1) inv += __shfl_xor_sync(~0u, inv, o);
    }
    if (lane == 0) {
      rs.makespan[b] = mk;
      rs.violations[b] = inv + nforced;
      rs.status[b] = stalled ? 2 : 0;
      if (rs.dev_end)
        for (int d = 0; d < G.ndev; ++d) rs.dev_end[b * G.ndev + d] = s.dev_end[d];
    }
    group_sync<kL>();
  }
}

// Per-call buffers: stream-ordered allocations on the legacy stream (the
// pool keeps its reservation, graph.cu), so a single report costs no
// cudaMalloc/cudaFree round trips.
struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFreeAsync(p, 0);
  }
};

template <typename T>
int dev_copy(DevBuf& buf, const T* src, size_t count, char* err) {
  CK(cudaMallocAsync(&buf.p, sizeof(T) * (count ? count : 1), 0));
  if (count && src) CK(cudaMemcpy(buf.p, src, sizeof(T) * count, cudaMemcpyHostToDevice));
  return 0;
}

// bounded() constants for n < 4096, built and uploaded once per device
int bounded_tables(int dev, const uint64_t** lim, const uint64_t** mag, char* err) {
  static std::mutex m;
  static uint64_t* tab[64] = {};
  std::lock_guard<std::mutex> lock(m);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!tab[dev]) {
    std::vector<uint64_t> h(2 * 4096);
    for (uint64_t k = 0; k < 4096; ++k) bounded_consts(k, &h[k], &h[4096 + k]);
    void* p = nullptr;
    CK(cudaMalloc(&p, 8 * h.size()));
    CK(cudaMemcpy(p, h.data(), 8 * h.size(), cudaMemcpyHostToDevice));
    tab[dev] = static_cast<uint64_t*>(p);
  }
  *lim = tab[dev];
  *mag = tab[dev] + 4096;
  return 0;
}

// Grow-only per-device scratch for the per-run state: thread-per-run
// batches take gigabytes, which are not worth re-allocating each call. The
// lock is held for the whole (synchronous) run.
struct ScratchPool {
  std::mutex m;
  void* p[64] = {};
  size_t cap[64] = {};
  char* get(int dev, size_t bytes, char* err) {
    if (dev < 0 || dev >= 64) dev = 0;
    if (cap[dev] < bytes) {
      if (p[dev]) cudaFree(p[dev]);
      p[dev] = nullptr;
      cap[dev] = 0;
      if (cudaMalloc(&p[dev], bytes) != cudaSuccess) {
        cudaGetLastError();
        std::snprintf(err, 256, "cannot allocate %zu bytes of simulator scratch", bytes);
        return nullptr;
      }
      cap[dev] = bytes;
    }
    return static_cast<char*>(p[dev]);
  }
};
ScratchPool& scratch_pool() {
  static ScratchPool* pool = new ScratchPool;  // never destroyed: process-lifetime device memory
  return *pool;
}

// Sweep statistics of a batch reduced where the runs' outputs already are
// (the reference's sweep summary, sched_main.cpp:480-502, plus the E and
// straggler histograms): pass 1 folds extremes, sums and histograms (shared
// histograms, one atomic per block and field), pass 2 finds the lowest run
// index reaching each extreme. Integer bins as in the host fold.
struct StatsReq {
  int cluster;
  const int32_t* d_wdev;  // worker w's device index
  int32_t nw;
  int64_t U, L;
  csk_event_stats* out;  // host
};

struct StatsArgs {
  const int64_t *ms, *dev_end;
  const int32_t *status, *wdev;
  int64_t B;
  int ndev, nw, cluster;
  int64_t U, L;
  csk_event_stats* acc;  // device
};

__device__ __forceinline__ void run_iter(const StatsArgs& a, int64_t b, int64_t* hi, int64_t* lo) {
  int64_t h = 0, l = INT64_MAX;
  for (int w = 0; w < a.nw; ++w) {
    const int64_t v = a.dev_end[b * a.ndev + a.wdev[w]];
    h = max(h, v);
    l = min(l, v);
  }
  *hi = h;
  *lo = l;
}

__global__ void __launch_bounds__(256) event_stats_kernel(StatsArgs a) {
  __shared__ int s_e[1000], s_s[1000];
  for (int k = threadIdx.x; k < 1000; k += blockDim.x) s_e[k] = s_s[k] = 0;
  __syncthreads();
  long long mn = LLONG_MAX, mx = LLONG_MIN, imn = LLONG_MAX, imx = LLONG_MIN;
  unsigned long long sum = 0, isum = 0, cnt = 0, stl = 0;
  double sq = 0.0, ss = 0.0;
  for (int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; b < a.B;
       b += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t m = a.ms[b];
    stl += a.status[b] != 0;
    mn = min(mn, static_cast<long long>(m));
    mx = max(mx, static_cast<long long>(m));
    sum += static_cast<unsigned long long>(m);
    ++cnt;
    sq += static_cast<double>(m) * static_cast<double>(m);
    if (a.U != a.L) {
      const int64_t bin = (1000 * (a.U - m)) / (a.U - a.L);
      atomicAdd(&s_e[static_cast<int>(min(int64_t{999}, max(int64_t{0}, bin)))], 1);
    }
    if (a.cluster) {
      int64_t hi, lo;
      run_iter(a, b, &hi, &lo);
      int bin = 0;
      if (hi > 0) {
        ss += static_cast<double>(hi - lo) / static_cast<double>(hi);
        bin = static_cast<int>(min(int64_t{999}, (1000 * (hi - lo)) / hi));
      }
      atomicAdd(&s_s[bin], 1);
      imn = min(imn, static_cast<long long>(hi));
      imx = max(imx, static_cast<long long>(hi));
      isum += static_cast<unsigned long long>(hi);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(~0u, mn, o));
    mx = max(mx, __shfl_xor_sync(~0u, mx, o));
    imn = min(imn, __shfl_xor_sync(~0u, imn, o));
    imx = max(imx, __shfl_xor_sync(~0u, imx, o));
    sum += __shfl_xor_sync(~0u, sum, o);
    isum += __shfl_xor_sync(~0u, isum, o);
    cnt += __shfl_xor_sync(~0u, cnt, o);
    stl += __shfl_xor_sync(~0u, stl, o);
    sq += __shfl_xor_sync(~0u, sq, o);
    ss += __shfl_xor_sync(~0u, ss, o);
  }
  csk_event_stats* acc = a.acc;
  if ((threadIdx.x & 31) == 0 && cnt > 0) {
    atomicMin(reinterpret_cast<long long*>(&acc->min_m), mn);
    atomicMax(reinterpret_cast<long long*>(&acc->max_m), mx);
    atomicAdd(reinterpret_cast<unsigned long long*>(&acc->sum_m), sum);
    atomicAdd(reinterpret_cast<unsigned long long*>(&acc->count), cnt);
    atomicAdd(reinterpret_cast<unsigned long long*>(&acc->stalled), stl);
    atomicAdd(&acc->sumsq, sq);
    if (a.cluster) {
      atomicMin(reinterpret_cast<long long*>(&acc->imin), imn);
      atomicMax(reinterpret_cast<long long*>(&acc->imax), imx);
      atomicAdd(reinterpret_cast<unsigned long long*>(&acc->isum), isum);
      atomicAdd(&acc->ssum, ss);
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < 1000; k += blockDim.x) {
    if (s_e[k]) atomicAdd(reinterpret_cast<unsigned long long*>(&acc->e_hist[k]), static_cast<unsigned long long>(s_e[k]));
    if (s_s[k]) atomicAdd(reinterpret_cast<unsigned long long*>(&acc->s_hist[k]), static_cast<unsigned long long>(s_s[k]));
  }
}

__global__ void __launch_bounds__(256) event_argext_kernel(StatsArgs a) {
  csk_event_stats* acc = a.acc;
  const int64_t mn = acc->min_m, mx = acc->max_m, imn = acc->imin, imx = acc->imax;
  for (int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; b < a.B;
       b += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t m = a.ms[b];
    if (m == mn) atomicMin(reinterpret_cast<long long*>(&acc->argmin), b);
    if (m == mx) atomicMin(reinterpret_cast<long long*>(&acc->argmax), b);
    if (a.cluster) {
      int64_t hi, lo;
      run_iter(a, b, &hi, &lo);
      if (hi == imn) atomicMin(reinterpret_cast<long long*>(&acc->iargmin), b);
      if (hi == imx) atomicMin(reinterpret_cast<long long*>(&acc->iargmax), b);
    }
  }
}

int reduce_stats(const StatsReq& q, const int64_t* d_ms, const int64_t* d_dev, const int32_t* d_st, int64_t B,
                 int ndev, int sms, char* err) {
  DevBuf d_acc;
  csk_event_stats init{};
  init.min_m = init.imin = INT64_MAX;
  init.max_m = init.imax = INT64_MIN;
  init.argmin = init.argmax = init.iargmin = init.iargmax = INT64_MAX;
  if (dev_copy(d_acc, &init, 1, err)) return 1;
  StatsArgs a{d_ms, d_dev, d_st, q.d_wdev, B, ndev, q.cluster ? q.nw : 0, q.cluster, q.U, q.L,
              static_cast<csk_event_stats*>(d_acc.p)};
  const int blocks = static_cast<int>(std::min<int64_t>((B + 255) / 256, 2LL * sms));
  event_stats_kernel<<<blocks, 256>>>(a);
  LAUNCHED();
  CK(cudaGetLastError());
  event_argext_kernel<<<blocks, 256>>>(a);
  LAUNCHED();
  CK(cudaGetLastError());
  CK(cudaMemcpy(q.out, d_acc.p, sizeof(csk_event_stats), cudaMemcpyDeviceToHost));
  return 0;
}

int run_event(DeviceGraph* g, const int64_t* dur, int64_t B, RunSpec rs, int64_t* makespan,
              int64_t* violations, int32_t* status, int64_t* start, int64_t* end, int64_t* dev_end,
              char* err, const StatsReq* sreq = nullptr) {
  if (ensure_device(err)) return 1;
  if (B <= 0) return 0;
  DevBuf d_dur, d_ms, d_vio, d_st, d_start, d_end, d_dev;
  ScratchPool& pool = scratch_pool();
  std::lock_guard<std::mutex> lock(pool.m);
  int sms = 148, dev = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  if (dev_copy(d_dur, dur, g->n, err)) return 1;
  if (bounded_tables(dev, &rs.lim, &rs.mag, err)) return 1;
  if (dev_copy<int64_t>(d_ms, nullptr, B, err) || dev_copy<int64_t>(d_vio, nullptr, B, err) ||
      dev_copy<int32_t>(d_st, nullptr, B, err))
    return 1;
  rs.makespan = static_cast<int64_t*>(d_ms.p);
  rs.violations = static_cast<int64_t*>(d_vio.p);
  rs.status = static_cast<int32_t*>(d_st.p);
  rs.start = rs.end = nullptr;
  if (start) {
    if (dev_copy<int64_t>(d_start, nullptr, g->n, err) || dev_copy<int64_t>(d_end, nullptr, g->n, err))
      return 1;
    rs.start = static_cast<int64_t*>(d_start.p);
    rs.end = static_cast<int64_t*>(d_end.p);
  }
  rs.dev_end = nullptr;
  if (dev_end || (sreq && sreq->cluster)) {
    if (dev_copy<int64_t>(d_dev, nullptr, static_cast<size_t>(B) * g->ndev, err)) return 1;
    rs.dev_end = static_cast<int64_t*>(d_dev.p);
  }
  GraphView G{g->n,        g->nres,     g->ndev,     g->R,        g->pred_off, g->succ_off,
              g->succ_idx, g->res,      g->res_dev,  g->rops_off, g->rops,     g->lidx,
              g->rb_off,   g->recv_ops, g->chan,     static_cast<int64_t*>(d_dur.p)};
  // Large batches: a thread per run (32 interleaved runs per warp) keeps
  // 32x more runs in flight than a warp per run; the lockstep lanes walk the
  // resource loops together, so their state accesses coalesce.
  const bool trace = std::getenv("TICTAC_EVENT_TRACE") != nullptr;
  const auto wall0 = std::chrono::steady_clock::now();
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  if (trace) {
    cudaEventCreate(&ev0);
    cudaEventCreate(&ev1);
    cudaEventRecord(ev0);
  }
  int lanes = B >= kThreadModeMin ? 1 : 32;
  if (const char* env = std::getenv("TICTAC_EVENT_LANES")) lanes = std::atoi(env) == 1 ? 1 : 32;
  if (lanes == 1) {
    bool inter = true;  // lane-interleaved state
    if (const char* env = std::getenv("TICTAC_EVENT_LAYOUT")) inter = std::atoi(env) != 1;
    const int lay = inter ? 32 : 1;
    const size_t hg = align8(hot_bytes(g->n, g->nres, g->rb_words, lay));
    const size_t cg = align8(cold_bytes(g->n, g->ndev, g->R, lay));
    const size_t per_group = inter ? 1 : 32;  // state blocks per 32-run warp
    // as many 32-run warps per SM as are resident (latency-bound chains)
    int occ = 1;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, event_sim_kernel<1, 32>, 32 * kWarpsPerBlock, 0));
    int per_sm = std::max(1, occ) * kWarpsPerBlock;
    if (const char* env = std::getenv("TICTAC_EVENT_GROUPS")) per_sm = std::max(1, std::atoi(env));
    int64_t groups = std::min<int64_t>((B + 31) / 32, static_cast<int64_t>(sms) * per_sm);
    groups = std::max<int64_t>(
        1, std::min<int64_t>(groups, static_cast<int64_t>(kThreadScratch / ((hg + cg) * per_group))));
    // fewer runs in flight when HBM is short (the GPU may be shared)
    int blocks = 0;
    size_t total = 0;
    char* scr = nullptr;
    for (;;) {
      blocks = static_cast<int>((groups + kWarpsPerBlock - 1) / kWarpsPerBlock);
      total = static_cast<size_t>(blocks) * kWarpsPerBlock * per_group;
      if ((scr = pool.get(dev, (hg + cg) * total, err)) || groups <= kWarpsPerBlock) break;
      groups /= 2;
    }
    if (!scr) return 1;
    if (inter)
      event_sim_kernel<1, 32><<<blocks, 32 * kWarpsPerBlock>>>(G, rs, B, scr, hg, scr + hg * total, cg, g->rb_words);
    else
      event_sim_kernel<1, 1><<<blocks, 32 * kWarpsPerBlock>>>(G, rs, B, scr, hg, scr + hg * total, cg, g->rb_words);
  } else {
    // Hot per-run state in shared memory when a slot fits (up to
    // kWarpsPerBlock runs per block), otherwise in global scratch.
    const size_t hsz = align8(hot_bytes(g->n, g->nres, g->rb_words));
    const size_t csz = align8(cold_bytes(g->n, g->ndev, g->R));
    // Shared memory wins per run (~1.7x) but caps runs per SM; large batches
    // of long runs keep more warps in flight with global scratch instead.
    constexpr size_t kSmemBudget = 200 * 1024;
    const int64_t smem_runs =
        static_cast<int64_t>(sms) * std::max<int64_t>(1, (227 * 1024) / std::max<size_t>(hsz, 1));
    const bool in_smem = hsz <= kSmemBudget && (B <= smem_runs || hsz <= 16 * 1024);
    // Few runs: one run per block, so the unused shared-memory carve-out stays
    // L1 for the graph arrays the (latency-bound) event chain reads.
    const int wpb = !in_smem ? kWarpsPerBlock
                    : B <= sms ? 1
                               : static_cast<int>(std::min<size_t>(kWarpsPerBlock, kSmemBudget / hsz));
    int per_sm = 16;
    if (in_smem) {
      CK(allow_max_dynamic_smem(reinterpret_cast<const void*>(event_sim_kernel<32, 1>)));
      const int carve =
          static_cast<int>(std::min<size_t>(100, (hsz * wpb * 100 + 228 * 1024 - 1) / (228 * 1024) + 3));
      CK(cudaFuncSetAttribute(event_sim_kernel<32, 1>, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
      int occ = 1;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, event_sim_kernel<32, 1>, 32 * wpb, hsz * wpb));
      per_sm = std::max(1, occ) * wpb;
    }
    int64_t slots = std::min<int64_t>(B, static_cast<int64_t>(sms) * per_sm);
    int blocks = 0;
    size_t hot_total = 0;
    int64_t total_slots = 0;
    char* scr = nullptr;
    for (;;) {  // fewer runs in flight when HBM is short
      blocks = static_cast<int>((slots + wpb - 1) / wpb);
      total_slots = static_cast<int64_t>(blocks) * wpb;
      hot_total = in_smem ? 0 : hsz * static_cast<size_t>(total_slots);
      if ((scr = pool.get(dev, hot_total + csz * static_cast<size_t>(total_slots), err)) || slots <= wpb) break;
      slots /= 2;
    }
    if (!scr) return 1;
    event_sim_kernel<32, 1><<<blocks, 32 * wpb, in_smem ? hsz * wpb : 0>>>(
        G, rs, B, in_smem ? nullptr : scr, hsz, scr + hot_total, csz, g->rb_words);
  }
  LAUNCHED();
  CK(cudaGetLastError());
  if (trace) cudaEventRecord(ev1);
  CK(cudaDeviceSynchronize());
  if (trace) {
    float ms = 0;
    cudaEventElapsedTime(&ms, ev0, ev1);
    const double wall = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - wall0).count();
    std::fprintf(stderr, "[event_sim] B=%lld lanes=%d kernel %.3f ms (run_event so far %.3f ms)\n",
                 static_cast<long long>(B), lanes, ms, wall);
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
  }
  if (sreq &&
      reduce_stats(*sreq, static_cast<const int64_t*>(d_ms.p), static_cast<const int64_t*>(d_dev.p),
                   static_cast<const int32_t*>(d_st.p), B, g->ndev, sms, err))
    return 1;
  // per-run outputs only where the caller asked for them
  if (makespan) CK(cudaMemcpy(makespan, d_ms.p, 8 * B, cudaMemcpyDeviceToHost));
  if (violations) CK(cudaMemcpy(violations, d_vio.p, 8 * B, cudaMemcpyDeviceToHost));
  if (status) CK(cudaMemcpy(status, d_st.p, 4 * B, cudaMemcpyDeviceToHost));
  if (start) {
    CK(cudaMemcpy(start, d_start.p, 8ull * g->n, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(end, d_end.p, 8ull * g->n, cudaMemcpyDeviceToHost));
  }
  if (dev_end) CK(cudaMemcpy(dev_end, d_dev.p, 8ull * B * g->ndev, cudaMemcpyDeviceToHost));
  return 0;
}

// One exact run inside SURVEY A.2's regime — worker graph with one compute
// unit and one channel, counter gate, no noise, every recv prioritized (and
// no compute op prioritized) — for its event list. The round structure is the
// generic replica's (try_start compute then channel, complete compute then
// channel, repeat while anything moved, then advance time); what the regime
// removes is every per-resource lookup: the channel always starts the next
// recv of the gate order (its only admitted candidate, no draw), both
// resources' state lives in registers, and only the compute unit draws from
// the choice stream. One thread runs the chain; the block initialises.
constexpr int kA2Tab = 256;  // bounded() constants staged for n < kA2Tab

// Shared-memory bytes of event_a2_kernel (the graph arrays stay in global
// memory: the fallback for runs whose nodes do not fit event_a2p_kernel).
__host__ __device__ inline size_t a2_smem(int n, int ncpu) {
  return 8 * 312 + 16ull * kA2Tab + 4ull * n + 4ull * ((ncpu + 31) / 32 + 1);
}

__global__ void __launch_bounds__(256) event_a2_kernel(GraphView G, const int32_t* __restrict__ gate_order,
                                                       int cpu_r, uint64_t choice_seed, const uint64_t* lim,
                                                       const uint64_t* mag, int64_t* start, int64_t* end,
                                                       int64_t* makespan) {
  extern __shared__ __align__(16) char a2_sm[];
  const int n = G.n, R = G.R;
  const int ncpu = cpu_r >= 0 ? G.rops_off[cpu_r + 1] - G.rops_off[cpu_r] : 0;
  const int nw = (ncpu + 31) / 32;
  auto* mt = reinterpret_cast<uint64_t*>(a2_sm);
  auto* s_lim = mt + 312;
  auto* s_mag = s_lim + kA2Tab;
  auto* missing = reinterpret_cast<int32_t*>(s_mag + kA2Tab);
  auto* ready = reinterpret_cast<uint32_t*>(missing + n);
  const int64_t* dur = G.dur;
  const int32_t *succ_off = G.succ_off, *succ_idx = G.succ_idx, *lidx = G.lidx, *order = gate_order;
  const int32_t* cpu_ops = cpu_r >= 0 ? G.rops + G.rops_off[cpu_r] : nullptr;
  for (int k = threadIdx.x; k < kA2Tab; k += blockDim.x) {
    s_lim[k] = lim[k];
    s_mag[k] = mag[k];
  }
  for (int w = threadIdx.x; w < nw; w += blockDim.x) ready[w] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int deg = G.pred_off[i + 1] - G.pred_off[i];
    missing[i] = deg;
    if (deg == 0 && G.res[i] == cpu_r) atomicOr(&ready[G.lidx[i] >> 5], 1u << (G.lidx[i] & 31));
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  MtFullP<uint64_t*> choice{mt, 0};
  choice.seed(choice_seed);
  // bounded(n) (rng.hpp:21-30): staged constants for small n (the ready set
  // of a compute unit is small), the host-built table otherwise
  auto bounded = [&](uint64_t m) -> uint64_t {
    const bool small = m < kA2Tab;
    const uint64_t lm = small ? s_lim[m] : lim[m], mg = small ? s_mag[m] : mag[m];
    uint64_t v;
    do v = choice.next();
    while (v > lm);
    return fastmod(v, m, mg);
  };
  int ready_cnt = 0, lo = 0;  // lo: no set bit below word lo
  for (int w = 0; w < nw; ++w) ready_cnt += __popc(ready[w]);
  constexpr int64_t kNever = INT64_MAX;
  int64_t t = 0, cpu_end = 0, chan_end = 0;
  int cpu_op = -1, chan_op = -1, chan_next = 0, finished = 0;
  auto complete = [&](int op) {
    ++finished;
    for (int e = succ_off[op]; e < succ_off[op + 1]; ++e) {
      const int w = succ_idx[e];
      if (--missing[w] == 0) {  // successors are compute ops (recvs are roots)
        const int l = lidx[w];
        ready[l >> 5] |= 1u << (l & 31);
        ++ready_cnt;
        lo = min(lo, l >> 5);
      }
    }
  };
  while (finished < n) {
    bool progress = true;
    while (progress) {
      progress = false;
      if (cpu_op < 0 && ready_cnt > 0) {  // try_start(compute): every ready op is a candidate
        int k = ready_cnt > 1 ? static_cast<int>(bounded(static_cast<uint64_t>(ready_cnt))) : 0;
        while (!ready[lo]) ++lo;
        int w = lo;
        for (;; ++w) {
          const int c = __popc(ready[w]);
          if (k < c) break;
          k -= c;
        }
        const int bit = nth_bit(ready[w], k);
        ready[w] &= ~(1u << bit);
        --ready_cnt;
        cpu_op = cpu_ops[(w << 5) + bit];
        cpu_end = t + dur[cpu_op];
        start[cpu_op] = t;
        end[cpu_op] = cpu_end;
        progress = true;
      }
      if (chan_op < 0 && chan_next < R) {  // try_start(channel): next in gate order
        chan_op = order[chan_next++];
        chan_end = t + dur[chan_op];
        start[chan_op] = t;
        end[chan_op] = chan_end;
        progress = true;
      }
      if (cpu_op >= 0 && cpu_end == t) {  // complete_now, resource order
        complete(cpu_op);
        cpu_op = -1;
        progress = true;
      }
      if (chan_op >= 0 && chan_end == t) {
        complete(chan_op);
        chan_op = -1;
        progress = true;
      }
    }
    if (finished == n) break;
    t = min(cpu_op >= 0 ? cpu_end : kNever, chan_op >= 0 ? chan_end : kNever);
    if (cpu_op >= 0 && cpu_end == t) {
      complete(cpu_op);
      cpu_op = -1;
    }
    if (chan_op >= 0 && chan_end == t) {
      complete(chan_op);
      chan_op = -1;
    }
  }
  *makespan = static_cast<int64_t>(t);  // every op has ended by the time of the last completion
}

// The packed single-report replica: the graph re-laid per run node in shared
// memory, nodes numbered u = compute op's index in the unit's op list (the
// candidate order of try_start), then R + ... recvs by gate rank. Node u's
// duration and successor range are one 16-byte load; successors are stored as
// unit indices, so a completion touches only `missing` and the ready bitset
// (both by unit index) — each step of the chain is one shared-memory round
// trip instead of several dependent generic loads. Start times stay in shared
// memory; the block writes start/end per op id at the end.
struct alignas(16) A2Node {
  long long dur;
  int beg, end;  // successors: a2_succ[beg..end)
};

__host__ __device__ inline size_t a2p_smem(int n, int E, int ncpu, size_t tbytes) {
  const int nw = (ncpu + 31) / 32 + 1;
  return 8 * 312 + 16ull * kA2Tab + 16ull * n + round16(tbytes * n) + round16(4ull * E) + 2 * round16(4ull * ncpu) +
         4ull * nw;
}

template <typename Tm>
__global__ void __launch_bounds__(256) event_a2p_kernel(GraphView G, const int32_t* __restrict__ gate_order,
                                                        int cpu_r, uint64_t choice_seed, const uint64_t* lim,
                                                        const uint64_t* mag, int64_t* start, int64_t* end,
                                                        int64_t* makespan) {
  extern __shared__ __align__(16) char a2_sm[];
  const int n = G.n, R = G.R;
  const int ncpu = G.rops_off[cpu_r + 1] - G.rops_off[cpu_r];
  const int32_t* cpu_ops = G.rops + G.rops_off[cpu_r];
  const int nw = (ncpu + 31) / 32;
  const int E = G.succ_off[n];
  auto* mt = reinterpret_cast<uint64_t*>(a2_sm);
  auto* s_lim = mt + 312;
  auto* s_mag = s_lim + kA2Tab;
  auto* node = reinterpret_cast<A2Node*>(s_mag + kA2Tab);
  auto* st = reinterpret_cast<Tm*>(node + n);
  auto* succ = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(st) + round16(sizeof(Tm) * n));
  auto* missing = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(succ) + round16(4ull * E));
  auto* nxt = reinterpret_cast<int32_t*>(reinterpret_cast<char*>(missing) + round16(4ull * ncpu));
  auto* ready = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(nxt) + round16(4ull * ncpu));
  for (int u = threadIdx.x; u < n; u += blockDim.x) {
    const int op = u < ncpu ? cpu_ops[u] : gate_order[u - ncpu];
    A2Node a;
    a.dur = G.dur[op];
    a.beg = G.succ_off[op];
    a.end = G.succ_off[op + 1];
    node[u] = a;
  }
  for (int e = threadIdx.x; e < E; e += blockDim.x) {  // ~l: the successor has one predecessor
    const int w = G.succ_idx[e];
    succ[e] = G.pred_off[w + 1] - G.pred_off[w] == 1 ? ~G.lidx[w] : G.lidx[w];
  }
  for (int k = threadIdx.x; k < kA2Tab; k += blockDim.x) {
    s_lim[k] = lim[k];
    s_mag[k] = mag[k];
  }
  for (int w = threadIdx.x; w <= nw; w += blockDim.x) ready[w] = 0;
  __syncthreads();
  for (int l = threadIdx.x; l < ncpu; l += blockDim.x) {
    const int op = cpu_ops[l];
    const int deg = G.pred_off[op + 1] - G.pred_off[op];
    missing[l] = deg;
    if (deg == 0) atomicOr(&ready[l >> 5], 1u << (l & 31));
    // chain successor: op's only out-edge goes to an op with one predecessor
    // and a positive duration (what the unit runs next when nothing else is
    // ready and the channel completes nothing first)
    int nx = -1;
    if (G.succ_off[op + 1] - G.succ_off[op] == 1) {
      const int w = G.succ_idx[G.succ_off[op]];
      if (G.pred_off[w + 1] - G.pred_off[w] == 1 && G.dur[w] > 0) nx = G.lidx[w];
    }
    nxt[l] = nx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    MtFullP<uint64_t*> choice{mt, 0};
    choice.seed(choice_seed);
    int ready_cnt = 0, lo = 0;  // lo: no set bit below word lo
    for (int w = 0; w < nw; ++w) ready_cnt += __popc(ready[w]);
    int hint = -1;  // the last op made ready while it stays ready: the pick when it is the only one
    Tm t = 0, cpu_end = 0, chan_end = 0;
    int cpu_u = -1, chan_u = -1, chan_next = 0;
    auto complete = [&](int u) {  // successors are compute ops (recvs are roots)
      const A2Node nd = node[u];
      for (int e = nd.beg; e < nd.end; ++e) {
        int l = succ[e];
        if (l < 0) {  // single-predecessor op: ready now
          l = ~l;
        } else {
          const int m = missing[l] - 1;
          missing[l] = m;
          if (m) continue;
        }
        ready[l >> 5] |= 1u << (l & 31);
        ++ready_cnt;
        lo = min(lo, l >> 5);
        hint = l;
      }
    };
    auto start_cpu = [&]() {  // try_start(compute): every ready op is a candidate
      int u;
      if (ready_cnt == 1 && hint >= 0) {
        u = hint;
        ready[u >> 5] &= ~(1u << (u & 31));
      } else {
        int k = 0;
        if (ready_cnt > 1) {  // bounded(ready_cnt), rng.hpp:21-30
          const uint64_t m = static_cast<uint64_t>(ready_cnt);
          const bool small = m < kA2Tab;
          const uint64_t lm = small ? s_lim[m] : lim[m], mg = small ? s_mag[m] : mag[m];
          uint64_t v;
          do v = choice.next();
          while (v > lm);
          k = static_cast<int>(fastmod(v, m, mg));
        }
        while (!ready[lo]) ++lo;
        int w = lo;
        uint32_t word = ready[w];
        for (;;) {
          const int c = __popc(word);
          if (k < c) break;
          k -= c;
          word = ready[++w];
        }
        const int bit = nth_bit(word, k);
        ready[w] = word & ~(1u << bit);
        u = (w << 5) + bit;
      }
      if (u == hint) hint = -1;
      --ready_cnt;
      cpu_u = u;
      st[u] = t;
      cpu_end = t + static_cast<Tm>(node[u].dur);
    };
    auto start_chan = [&]() {  // try_start(channel): next in gate order
      chan_u = ncpu + chan_next++;
      st[chan_u] = t;
      chan_end = t + static_cast<Tm>(node[chan_u].dur);
    };
    for (;;) {
      // The round at time t: try_start in resource order. Busy resources end
      // after t here, so complete_now can only fire for an op started now
      // with zero duration; then the generic passes take over (sim.cpp:117-233).
      bool zero = false;
      if (cpu_u < 0 && ready_cnt > 0) {
        start_cpu();
        zero = cpu_end == t;
      }
      if (chan_u < 0 && chan_next < R) {
        start_chan();
        zero |= chan_end == t;
      }
      // Compute-only rounds: while the channel is done or completes strictly
      // after the running compute op, the channel's try_start and
      // completions are no-ops, so each round is "complete the op at its end,
      // pick the next one". Along a chain — the op's only successor is a
      // single-predecessor op with positive duration and nothing else is
      // ready — the round reduces further to "start the successor" (no draw,
      // no other state change).
      while (!zero && cpu_u >= 0 && (chan_u < 0 || cpu_end < chan_end)) {
        if (ready_cnt == 0) {
          const int v = nxt[cpu_u];
          if (v >= 0) {
            t = cpu_end;
            cpu_u = v;
            st[v] = t;
            cpu_end = t + static_cast<Tm>(node[v].dur);
            continue;
          }
        }
        t = cpu_end;
        complete(cpu_u);
        cpu_u = -1;
        if (ready_cnt == 0) break;
        start_cpu();
        zero = cpu_end == t;
      }
      if (zero) {
        if (cpu_u >= 0 && cpu_end == t) {
          complete(cpu_u);
          cpu_u = -1;
        }
        if (chan_u >= 0 && chan_end == t) {
          complete(chan_u);
          chan_u = -1;
        }
        for (bool progress = true; progress;) {
          progress = false;
          if (cpu_u < 0 && ready_cnt > 0) {
            start_cpu();
            progress = true;
          }
          if (chan_u < 0 && chan_next < R) {
            start_chan();
            progress = true;
          }
          if (cpu_u >= 0 && cpu_end == t) {
            complete(cpu_u);
            cpu_u = -1;
            progress = true;
          }
          if (chan_u >= 0 && chan_end == t) {
            complete(chan_u);
            chan_u = -1;
            progress = true;
          }
        }
      }
      if (cpu_u < 0 && chan_u < 0) break;  // nothing running or startable: every op of the DAG has ended
      t = cpu_u < 0 ? chan_end : chan_u < 0 ? cpu_end : min(cpu_end, chan_end);
      if (cpu_u >= 0 && cpu_end == t) {
        complete(cpu_u);
        cpu_u = -1;
      }
      if (chan_u >= 0 && chan_end == t) {
        complete(chan_u);
        chan_u = -1;
      }
    }
    *makespan = static_cast<int64_t>(t);  // every op has ended by the time of the last completion
  }
  __syncthreads();
  for (int u = threadIdx.x; u < n; u += blockDim.x) {
    const int op = u < ncpu ? cpu_ops[u] : gate_order[u - ncpu];
    const int64_t s0 = static_cast<int64_t>(st[u]);
    start[op] = s0;
    end[op] = s0 + node[u].dur;
  }
}

}  // namespace

}  // namespace tictac_dev

using namespace tictac_dev;

extern "C" int csk_event_sim(DeviceGraph* g, const int64_t* dur, int32_t B, const int32_t* prio,
                             const int32_t* orders, int32_t R, const uint64_t* seeds, int gated,
                             double noise, int64_t* makespan, int64_t* violations, int32_t* status,
                             int64_t* start, int64_t* end, int64_t* dev_end, char* err) {
  if (ensure_device(err)) return 1;
  DevBuf d_p, d_s;
  RunSpec rs{};
  if (prio) {
    if (dev_copy(d_p, prio, static_cast<size_t>(B) * g->n, err)) return 1;
    rs.mode = kPrioExplicit;
    rs.prio = static_cast<int32_t*>(d_p.p);
  } else {
    if (R != g->R) {
      std::snprintf(err, 256, "orders have %d recvs, graph has %d", R, g->R);
      return 4;
    }
    if (dev_copy(d_p, orders, static_cast<size_t>(B) * R, err)) return 1;
    rs.mode = kPrioOrders;
    rs.orders = static_cast<int32_t*>(d_p.p);
  }
  if (dev_copy(d_s, seeds, B, err)) return 1;
  rs.seeds = static_cast<uint64_t*>(d_s.p);
  rs.gated = gated;
  rs.noise = noise;
  return run_event(g, dur, B, rs, makespan, violations, status, start, end, dev_end, err);
}

extern "C" int csk_event_sweep(DeviceGraph* g, const int64_t* dur, uint64_t seed_lo, int32_t B,
                               int cluster, const int32_t* recv_worker, int32_t n_workers, int gated,
                               double noise, int64_t* makespan, int64_t* violations, int32_t* status,
                               int64_t* dev_end, const int32_t* worker_dev, int64_t U, int64_t L,
                               csk_event_stats* stats, char* err) {
  if (ensure_device(err)) return 1;
  std::vector<int32_t> off(n_workers + 1, 0), cols(g->R);
  for (int c = 0; c < g->R; ++c) off[recv_worker[c] + 1]++;
  for (int w = 0; w < n_workers; ++w) off[w + 1] += off[w];
  std::vector<int32_t> fill(off.begin(), off.end() - 1);
  for (int c = 0; c < g->R; ++c) cols[fill[recv_worker[c]]++] = c;
  DevBuf d_off, d_cols;
  if (dev_copy(d_off, off.data(), off.size(), err) || dev_copy(d_cols, cols.data(), cols.size(), err))
    return 1;
  RunSpec rs{};
  rs.mode = kPrioRandom;
  rs.seed_lo = seed_lo;
  rs.cluster = cluster;
  rs.wcols_off = static_cast<int32_t*>(d_off.p);
  rs.wcols = static_cast<int32_t*>(d_cols.p);
  rs.n_workers = n_workers;
  rs.gated = gated;
  rs.noise = noise;
  if (!stats) return run_event(g, dur, B, rs, makespan, violations, status, nullptr, nullptr, dev_end, err);
  DevBuf d_wdev;
  if (cluster && dev_copy(d_wdev, worker_dev, static_cast<size_t>(n_workers), err)) return 1;
  const StatsReq q{cluster, static_cast<const int32_t*>(d_wdev.p), n_workers, U, L, stats};
  return run_event(g, dur, B, rs, makespan, violations, status, nullptr, nullptr, dev_end, err, &q);
}

extern "C" int csk_brute_force(DeviceGraph* g, const int64_t* dur, int32_t R, uint64_t choice_seed,
                               double noise, int64_t* makespans, char* err) {
  if (ensure_device(err)) return 1;
  if (R != g->R || R > 20) {
    std::snprintf(err, 256, "brute force over %d recvs unsupported", R);
    return 4;
  }
  int64_t perms = 1;
  for (int k = 2; k <= R; ++k) perms *= k;
  std::vector<int32_t> status(static_cast<size_t>(perms));
  RunSpec rs{};
  rs.mode = kPrioLex;
  rs.seed_lo = choice_seed;
  rs.gated = 1;
  rs.noise = noise;
  if (run_event(g, dur, perms, rs, makespans, nullptr, status.data(), nullptr, nullptr, nullptr, err))
    return 1;
  for (int64_t k = 0; k < perms; ++k)
    if (status[k]) makespans[k] = -1;
  return 0;
}

extern "C" int csk_event_a2(DeviceGraph* g, const int64_t* dur, const int32_t* gate_order, int32_t R,
                            uint64_t choice_seed, int64_t* makespan, int64_t* start, int64_t* end, char* err) {
  if (ensure_device(err)) return 1;
  if (R != g->R) {
    std::snprintf(err, 256, "gate order has %d recvs, graph has %d", R, g->R);
    return 4;
  }
  int cpu_r = -1;  // the compute unit: the resource of any non-recv op
  for (int32_t i = 0; i < g->n && cpu_r < 0; ++i)
    if (g->h_kind[i] != 1) cpu_r = g->h_res[i];
  int dev = 0;
  CK(cudaGetDevice(&dev));
  DevBuf d_dur, d_order, d_start, d_end, d_ms;
  if (dev_copy(d_dur, dur, g->n, err) || dev_copy(d_order, gate_order, R, err) ||
      dev_copy<int64_t>(d_start, nullptr, g->n, err) || dev_copy<int64_t>(d_end, nullptr, g->n, err) ||
      dev_copy<int64_t>(d_ms, nullptr, 1, err))
    return 1;
  RunSpec tabs{};
  if (bounded_tables(dev, &tabs.lim, &tabs.mag, err)) return 1;
  GraphView G{g->n,        g->nres,     g->ndev,     g->R,        g->pred_off, g->succ_off,
              g->succ_idx, g->res,      g->res_dev,  g->rops_off, g->rops,     g->lidx,
              g->rb_off,   g->recv_ops, g->chan,     static_cast<int64_t*>(d_dur.p)};
  int ncpu = 0;
  for (int32_t i = 0; i < g->n; ++i) ncpu += g->h_res[i] == cpu_r;
  const int E = g->h_succ_off.empty() ? 0 : g->h_succ_off.back();
  int64_t U = 0;  // every event time is at most the sum of all durations
  for (int32_t i = 0; i < g->n; ++i) U += dur[i];
  const bool narrow = U < (int64_t{1} << 31);
  // the packed kernel when the run's nodes fit in shared memory, else the
  // replica over the global graph arrays
  const size_t smem_p = a2p_smem(g->n, E, ncpu, narrow ? 4 : 8);
  const bool packed = cpu_r >= 0 && smem_p <= 220 * 1024 && !std::getenv("TICTAC_A2_GLOBAL");
  const size_t smem = packed ? smem_p : a2_smem(g->n, ncpu);
  if (smem > 220 * 1024) {
    std::snprintf(err, 256, "graph too large for the single-report kernel");
    return 4;
  }
  const void* kfn = !packed ? reinterpret_cast<const void*>(event_a2_kernel)
                    : narrow ? reinterpret_cast<const void*>(event_a2p_kernel<int32_t>)
                             : reinterpret_cast<const void*>(event_a2p_kernel<int64_t>);
  CK(allow_max_dynamic_smem(kfn));
  const bool trace = std::getenv("TICTAC_EVENT_TRACE") != nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  if (trace) {
    cudaEventCreate(&ev0);
    cudaEventCreate(&ev1);
    cudaEventRecord(ev0);
  }
  auto* ordp = static_cast<int32_t*>(d_order.p);
  auto *stp = static_cast<int64_t*>(d_start.p), *enp = static_cast<int64_t*>(d_end.p),
       *msp = static_cast<int64_t*>(d_ms.p);
  if (packed && narrow)
    event_a2p_kernel<int32_t><<<1, 256, smem>>>(G, ordp, cpu_r, choice_seed, tabs.lim, tabs.mag, stp, enp, msp);
  else if (packed)
    event_a2p_kernel<int64_t><<<1, 256, smem>>>(G, ordp, cpu_r, choice_seed, tabs.lim, tabs.mag, stp, enp, msp);
  else
    event_a2_kernel<<<1, 256, smem>>>(G, ordp, cpu_r, choice_seed, tabs.lim, tabs.mag, stp, enp, msp);
  LAUNCHED();
  CK(cudaGetLastError());
  if (trace) {
    cudaEventRecord(ev1);
    cudaEventSynchronize(ev1);
    float ms = 0;
    cudaEventElapsedTime(&ms, ev0, ev1);
    std::fprintf(stderr, "[event_a2] n=%d kernel %.3f ms\n", g->n, ms);
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
  }
  CK(cudaMemcpy(makespan, d_ms.p, 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(start, d_start.p, 8ull * g->n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(end, d_end.p, 8ull * g->n, cudaMemcpyDeviceToHost));
  return 0;
}
