// Batched random-order sweep — the throughput kernel (SURVEY §8a rows
// a8/a10/a11/a12, Appendix A.2).
//
// One thread owns one seed end to end: the reference's random_schedule
// (mt19937_64(seed) + bounded() + Fisher–Yates from the top, rng.hpp:21-46,
// schedule.cpp:73-84) and the closed-form makespan of a gated, fully
// prioritized run, fused so that nothing per-ordering touches HBM.
//
// Closed form on "chain-class" graphs (host analysis in csrc/host/sweep.cpp):
// group compute ops by their recv-ancestor set; when these sets are nested
// (C_0 ⊂ C_1 ⊂ … ⊂ C_{nc-1}) a compute class j is released when the last of
// its recvs completes, i.e. at position lp(C_j) = max{k : first[perm[k]] ≤ j}.
// With G_k = min_{k' ≥ k} first[perm[k']] (a suffix minimum), the single-core
// earliest-release-date pass gives
//     T_cpu = max over k with G_k < G_{k+1} of  c_k + S(G_k),
// c_k = completion of the k-th transfer = Ctot − Σ_{k' > k} d, S(j) = Σ weights
// of classes ≥ j. Every term is available right-to-left, and Fisher–Yates
// finalises positions right-to-left, so each draw is folded the moment its
// slot is final: O(R) work, O(R) bytes of shared memory per seed, no arrays.
//   worker graph:   m   = max(T_cpu, Ctot)
//   cluster worker: m_w = max(T_cpu, max(Ctot, T_cpu) + Σ sends)
// The shuffle array lives in shared memory as bytes (R ≤ 256) or halves,
// laid out [k/4][thread] so every lane always hits its own bank.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <cub/cub.cuh>
#include <iterator>
#include <vector>

#include "common.cuh"
#include "csk.h"

namespace tictac_dev {
namespace {

constexpr int kSweepThreads = 256;
constexpr int kMaxChannelsDev = 4;  // channels per worker of chain_multi_kernel
constexpr int kBins = 1000;

struct ChainArgs {
  int W, R, stride;  // workers, recvs per worker, pwsuf stride (nc+1)
  int nc;
  int nch;           // channels per worker (ctot / send_tot are [W][nch])
  const uint2* tab;         // [W][R] {first class, duration}
  const int64_t* pwsuf;     // [W][stride]
  const int64_t* ctot;      // [W]
  const int64_t* send_tot;  // [W]
  int cluster;
  const uint64_t* lim;  // [R+1] bounded() constants
  const uint64_t* mag;
  uint64_t seed_lo, key_base;
  int64_t count;
  int64_t U, L;
  int do_e;
  int key_bits;           // statistics keys: (m << key_bits) | offset
  int force_slow;         // test knob: every shuffle through the generic engine
  const void* blob;       // table image in the kernel's shared-memory layout (bulk-copied), or null
  uint32_t blob_bytes;
  uint32_t mbar_off;      // byte offset of the copy's mbarrier in dynamic shared memory
  const int32_t* orders;  // explicit orders mode (W == 1)
  int* bad_order;         // explicit orders: set when an entry is out of [0, R)
  uint64_t noise_thr;     // gated reorder noise: swap when (output >> 11) < thr (0: none)
  int64_t* makespans;
  int64_t* worker_ms;
  unsigned long long* i64;
  double* f64;
};

template <typename T, int NT = kSweepThreads>
struct Items;  // per-thread array in shared memory, [k / per_word][thread]

template <int NT>
struct Items<uint8_t, NT> {
  using value_type = uint8_t;
  uint32_t* base;
  // byte (k & 3) of word (k >> 2) of this thread's column:
  // (k >> 2) * 4 * NT + (k & 3) == k * NT - (k & 3) * (NT - 1)
  __device__ __forceinline__ uint8_t* at(int k) const {
    return reinterpret_cast<uint8_t*>(base) + k * NT - (k & 3) * (NT - 1);
  }
  // slot 4m and the byte offset of slot 4m + r from it (aligned groups of
  // four slots: one address per group, the rest immediate offsets)
  __device__ __forceinline__ uint8_t* at4(int m) const { return reinterpret_cast<uint8_t*>(base) + m * 4 * NT; }
  static constexpr int goff(int r) { return r; }
  static constexpr int kGroupBytes = 4 * NT;  // at4(m) - at4(m - 1)
  __device__ __forceinline__ void init(int R) const {
    for (int q = 0; q < (R + 3) >> 2; ++q) base[q * NT] = 0x03020100u + 0x04040404u * static_cast<uint32_t>(q);
  }
  static constexpr int words(int n) { return (n + 3) >> 2; }
};
template <int NT>
struct Items<uint16_t, NT> {
  using value_type = uint16_t;
  uint32_t* base;
  __device__ __forceinline__ uint16_t* at(int k) const {
    return reinterpret_cast<uint16_t*>(base + (k >> 1) * NT) + (k & 1);
  }
  __device__ __forceinline__ uint16_t* at4(int m) const { return reinterpret_cast<uint16_t*>(base + 2 * m * NT); }
  static constexpr int goff(int r) { return (r >> 1) * 4 * NT + (r & 1) * 2; }
  static constexpr int kGroupBytes = 8 * NT;
  __device__ __forceinline__ void init(int R) const {
    for (int q = 0; q < (R + 1) >> 1; ++q)
      base[q * NT] = (static_cast<uint32_t>(2 * q + 1) << 16) | static_cast<uint32_t>(2 * q);
  }
  static constexpr int words(int n) { return (n + 1) >> 1; }
};

// Right-to-left suffix-min fold of one ordering; V = int32_t when every
// time sum fits 31 bits (U < 2^31, checked on the host), else int64_t.
template <typename V>
struct FoldT {
  int G;
  V suffix, best;
  // The term is taken unconditionally: when gk == G it is dominated by the
  // term taken when G got its value (the suffix only grows), and before the
  // first class (G == nc, S(nc) = 0) it is a transfer completion c_k <= Ctot,
  // which every consumer of best already maxes with (m = max(T_cpu, Ctot),
  // cluster m_w = max(T_cpu, max(Ctot, T_cpu) + sends)). No predicate, one
  // ALU instruction less per draw.
  __device__ __forceinline__ void add(uint2 e, V ctot, const V* pw) {
    const int gk = min(static_cast<int>(e.x), G);
    best = max(best, ctot - suffix + pw[gk]);
    G = gk;
    suffix += static_cast<V>(e.y);
  }
};

// tab[x] for a table in shared memory, addressed as one IMAD from a 32-bit
// shared-window base (the compiler's LEA form runs on the ALU pipe, which
// bounds the shuffle).
__device__ __forceinline__ uint2 tab_at(const uint2* tab, uint32_t x) {
  uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(tab)), addr;
  asm("mad.lo.u32 %0, %1, 8, %2;" : "=r"(addr) : "r"(x), "r"(base));
  uint2 e;
  asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(e.x), "=r"(e.y) : "r"(addr));  // read-only table
  return e;
}

// One Fisher–Yates draw at slot i (1-based count of unfinished slots) with
// bounded() value j: the element landing in its final slot i-1 is folded.
// kStore: keep the permutation instead (the element is written to slot i-1).
template <typename It, typename V, bool kStore = false>
__device__ __forceinline__ void fy_draw_at(const It& items, typename It::value_type* pl, int j, FoldT<V>& f,
                                           const uint2* tab, V ctot, const V* pw) {
  using T = typename It::value_type;
  T* pj = items.at(j);
  const T x = *pj;
  if constexpr (kStore) {
    *pj = *pl;
    *pl = x;
  } else {
    *pj = *pl;
    f.add(tab_at(tab, x), ctot, pw);
  }
}
template <typename It, typename V, bool kStore = false>
__device__ __forceinline__ void fy_draw(const It& items, int i, int j, FoldT<V>& f, const uint2* tab,
                                        V ctot, const V* pw) {
  fy_draw_at<It, V, kStore>(items, items.at(i - 1), j, f, tab, ctot, pw);
}

// Generic continuation after a bounded() rejection (probability ~R·2^-64
// per draw) or past the first 311 outputs: full mt19937_64 state in local
// memory, advanced to output `out` (0-based), then the reference loop.
// (Everything by value: no address-taken locals in the hot caller.)
template <typename It, typename V, bool kStore = false>
__device__ __noinline__ FoldT<V> shuffle_slow(uint64_t seed, int out, int i, It items, FoldT<V> f,
                                              const uint2* tab, V ctot, const V* pw) {
  uint64_t st[312];
  MtFull m{st, 0};
  m.seed(seed);
  for (int k = 0; k < out; ++k) m.next();
  for (; i > 1; --i) {
    const uint64_t n = static_cast<uint64_t>(i);
    const uint64_t limit = UINT64_MAX - (UINT64_MAX % n + 1) % n;
    uint64_t v;
    do v = m.next();
    while (v > limit);
    fy_draw<It, V, kStore>(items, i, static_cast<int>(v % n), f, tab, ctot, pw);
  }
  if constexpr (!kStore) f.add(tab[*items.at(0)], ctot, pw);
  return f;
}

// Draws d..d+K-1 with outputs v[] (pre-checked only by maybe_reject):
// precise bounded() rejection test, then the swaps. Returns true when a
// rejection sent the rest of the shuffle to the exact slow path. kAligned
// (K == 4, (R - d) % 4 == 0): the group's final slots R-1-d .. R-4-d are the
// four slots of one aligned group, addressed from one pointer.
template <int K, typename It, typename V, bool kStore = false, bool kAligned = false>
__device__ __forceinline__ bool draw_group(uint64_t seed, int R, int d, const uint64_t (&v)[K],
                                           const It& items, FoldT<V>& f, const uint2* tab, V ctot,
                                           const V* pw, const uint64_t* s_lim, const uint64_t* s_mag,
                                           unsigned char* pg = nullptr) {
  using T = typename It::value_type;
  static_assert(!kAligned || K == 4, "aligned groups are four draws");
  int j[K];
  const uint32_t nneg0 = static_cast<uint32_t>(d - R);  // -(slot count) of draw 0
  uint32_t low = ~0u;  // min over draws of (high word + 1): 0 iff some high word is all ones
#pragma unroll
  for (int q = 0; q < K; ++q) {
    const int i = R - d - q;
    // (the two remainder forms measure differently per kernel: the folding
    // chain kernels take the cheaper quotient, the storing ones the exact)
    if constexpr (kStore)
      j[q] = static_cast<int>(fastmod32n_exact(v[q], nneg0 + q, s_mag[i]));
    else
      j[q] = static_cast<int>(fastmod32n(v[q], nneg0 + q, s_mag[i]));
    low = min(low, static_cast<uint32_t>(v[q] >> 32) + 1u);
  }
  if (low == 0) {  // maybe_reject: probability ~2^-32 per draw; exact handling, draw by draw
#pragma unroll  // (static indices: keeps v[] and j[] in registers)
    for (int q = 0; q < K; ++q) {
      const int i = R - d - q;
      if (v[q] > s_lim[i]) {
        f = shuffle_slow<It, V, kStore>(seed, d + q + 1, i, items, f, tab, ctot, pw);
        return true;
      }
      fy_draw<It, V, kStore>(items, i, j[q], f, tab, ctot, pw);
    }
    return false;
  }
  if constexpr (kAligned) {  // pg == items.at4((R - 4 - d) >> 2), kept by the caller
#pragma unroll
    for (int q = 0; q < 4; ++q)
      fy_draw_at<It, V, kStore>(items, reinterpret_cast<T*>(pg + It::goff(3 - q)), j[q], f, tab, ctot, pw);
  } else {
#pragma unroll
    for (int q = 0; q < K; ++q) fy_draw<It, V, kStore>(items, R - d - q, j[q], f, tab, ctot, pw);
  }
  return false;
}

// random_schedule(seed) over R recv columns folded right-to-left. Fast path:
// draw d uses mt output d (no rejection) computed by register cursors —
// phase 1 (d < 156): t_d = f(s_d, s_d+1) ^ s_{d+156}; phase 2 (d < 311):
// t_d = f(s_d, s_d+1) ^ t_{d-156}, t_{d-156} = f(s_{d-156}, s_{d-155}) ^ s_d.
// Four draws per iteration: four independent twist/temper/bounded chains
// before the dependent shared-memory swaps.
// kSave: phase 1 keeps its untempered outputs t_d (d < R - 157) in a local
// array, and phase 2 reads t_{d-156} back instead of re-walking the seeding
// from s_0 with a third cursor (about 16 instructions per phase-2 draw for
// one 8-byte store and load; the array stays in L2 — 87 entries per thread at
// config 4 — where the shuffle's issue-bound loop hides its latency).
template <typename It, typename V, bool kStore = false, bool kSave = false>
__device__ __forceinline__ void shuffle_fold(uint64_t seed, int R, const It& items, FoldT<V>& f,
                                             const uint2* tab, V ctot, const V* pw,
                                             const uint64_t* s_lim, const uint64_t* s_mag) {
  uint64_t ts[kSave ? 156 : 1];
  const int save_lim = R - 157;  // t_d is read back by phase 2 iff d < R - 157
  items.init(R);
  uint64_t a0 = seed, a1 = mt_step(seed, 1), b = seed;
#pragma unroll 4
  for (uint32_t k = 1; k <= 156; ++k) b = mt_step(b, k);
  const int draws = R - 1;
  const int n1 = min(draws, 156);
  int d = 0;
  for (; d < n1 && ((R - d) & 3) != 0; ++d) {  // single draws up to an aligned group
    const uint64_t t = mt_twist(a0, a1, b);
    if constexpr (kSave)
      if (d < save_lim) ts[d] = t;
    const uint64_t v[1] = {mt_temper(kSave ? t : mt_twist(a0, a1, b))};
    a0 = a1;
    a1 = mt_step(a1, static_cast<uint32_t>(d + 2));
    b = mt_step(b, static_cast<uint32_t>(d + 157));
    if (draw_group<1, It, V, kStore>(seed, R, d, v, items, f, tab, ctot, pw, s_lim, s_mag)) return;
  }
  unsigned char* pg = reinterpret_cast<unsigned char*>(items.at4((R - 4 - d) >> 2));  // aligned groups
  for (; d + 3 < n1; d += 4, pg -= It::kGroupBytes) {  // phase 1, a = (s_d, s_d+1), b = s_d+156
    const uint32_t u = static_cast<uint32_t>(d);
    const uint64_t a2 = mt_step(a1, u + 2), a3 = mt_step(a2, u + 3), a4 = mt_step(a3, u + 4);
    const uint64_t b1 = mt_step(b, u + 157), b2 = mt_step(b1, u + 158), b3 = mt_step(b2, u + 159);
    if constexpr (kSave) {
      const uint64_t t[4] = {mt_twist(a0, a1, b), mt_twist(a1, a2, b1), mt_twist(a2, a3, b2), mt_twist(a3, a4, b3)};
      if (d < save_lim) {  // (uniform: R is; the group's tail entries past the limit are never read)
        ts[d] = t[0];
        ts[d + 1] = t[1];
        ts[d + 2] = t[2];
        ts[d + 3] = t[3];
      }
      const uint64_t v[4] = {mt_temper(t[0]), mt_temper(t[1]), mt_temper(t[2]), mt_temper(t[3])};
      a0 = a4;
      a1 = mt_step(a4, u + 5);
      b = mt_step(b3, u + 160);
      if (draw_group<4, It, V, kStore, true>(seed, R, d, v, items, f, tab, ctot, pw, s_lim, s_mag, pg)) return;
    } else {
      const uint64_t v[4] = {mt_temper(mt_twist(a0, a1, b)), mt_temper(mt_twist(a1, a2, b1)),
                             mt_temper(mt_twist(a2, a3, b2)), mt_temper(mt_twist(a3, a4, b3))};
      a0 = a4;
      a1 = mt_step(a4, u + 5);
      b = mt_step(b3, u + 160);
      if (draw_group<4, It, V, kStore, true>(seed, R, d, v, items, f, tab, ctot, pw, s_lim, s_mag, pg)) return;
    }
  }
  for (; d < n1; ++d) {
    const uint64_t t = mt_twist(a0, a1, b);
    if constexpr (kSave)
      if (d < save_lim) ts[d] = t;
    const uint64_t v[1] = {mt_temper(kSave ? t : mt_twist(a0, a1, b))};
    a0 = a1;
    a1 = mt_step(a1, static_cast<uint32_t>(d + 2));
    b = mt_step(b, static_cast<uint32_t>(d + 157));
    if (draw_group<1, It, V, kStore>(seed, R, d, v, items, f, tab, ctot, pw, s_lim, s_mag)) return;
  }
  if (kSave && d < draws && d == 156) {  // phase 2 from the saved outputs: t_d = f(s_d, s_d+1) ^ t_{d-156}
    const int n2 = min(draws, 311);
    for (; d < n2 && ((R - d) & 3) != 0; ++d) {
      const uint64_t v[1] = {mt_temper(mt_twist(a0, a1, ts[d - 156]))};
      a0 = a1;
      a1 = mt_step(a1, static_cast<uint32_t>(d + 2));
      if (draw_group<1, It, V, kStore>(seed, R, d, v, items, f, tab, ctot, pw, s_lim, s_mag)) return;
    }
    pg = reinterpret_cast<unsigned char*>(items.at4((R - 4 - d) >> 2));
    for (; d + 3 < n2; d += 4, pg -= It::kGroupBytes) {
      const uint32_t u = static_cast<uint32_t>(d);
      const uint64_t a2 = mt_step(a1, u + 2), a3 = mt_step(a2, u + 3), a4 = mt_step(a3, u + 4);
      const uint64_t v[4] = {mt_temper(mt_twist(a0, a1, ts[d - 156])), mt_temper(mt_twist(a1, a2, ts[d - 155])),
                             mt_temper(mt_twist(a2, a3, ts[d - 154])), mt_temper(mt_twist(a3, a4, ts[d - 153]))};
      a0 = a4;
      a1 = mt_step(a4, u + 5);
      if (draw_group<4, It, V, kStore, true>(seed, R, d, v, items, f, tab, ctot, pw, s_lim, s_mag, pg)) return;
    }
    for (; d < n2; ++d) {
      const uint64_t v[1] = {mt_temper(mt_twist(a0, a1, ts[d - 156]))};
      a0 = a1;
      a1 = mt_step(a1, static_cast<uint32_t>(d + 2));
      if (draw_group<1, It, V, kStore>(seed, R, d, v, items, f, tab, ctot, pw, s_lim, s_mag)) return;
    }
    if (d < draws) {  // beyond the first block (R > 312)
      f = shuffle_slow<It, V, kStore>(seed, d, R - d, items, f, tab, ctot, pw);
      return;
    }
  } else if (d < draws) {  // phase 2, c = (s_d-156, s_d-155)
    uint64_t c0 = seed, c1 = mt_step(seed, 1);
    const int n2 = min(draws, 311);
    for (; d < n2 && ((R - d) & 3) != 0; ++d) {  // single draws up to an aligned group
      const uint64_t v[1] = {mt_temper(mt_twist(a0, a1, mt_twist(c0, c1, a0)))};
      a0 = a1;
      a1 = mt_step(a1, static_cast<uint32_t>(d + 2));
      c0 = c1;
      c1 = mt_step(c1, static_cast<uint32_t>(d - 154));
      if (draw_group<1, It, V, kStore>(seed, R, d, v, items, f, tab, ctot, pw, s_lim, s_mag)) return;
    }
    pg = reinterpret_cast<unsigned char*>(items.at4((R - 4 - d) >> 2));
    for (; d + 3 < n2; d += 4, pg -= It::kGroupBytes) {
      const uint32_t u = static_cast<uint32_t>(d);
      const uint64_t a2 = mt_step(a1, u + 2), a3 = mt_step(a2, u + 3), a4 = mt_step(a3, u + 4);
      const uint64_t c2 = mt_step(c1, u - 154), c3 = mt_step(c2, u - 153), c4 = mt_step(c3, u - 152);
      const uint64_t v[4] = {mt_temper(mt_twist(a0, a1, mt_twist(c0, c1, a0))),
                             mt_temper(mt_twist(a1, a2, mt_twist(c1, c2, a1))),
                             mt_temper(mt_twist(a2, a3, mt_twist(c2, c3, a2))),
                             mt_temper(mt_twist(a3, a4, mt_twist(c3, c4, a3)))};
      a0 = a4;
      a1 = mt_step(a4, u + 5);
      c0 = c4;
      c1 = mt_step(c4, u - 151);
      if (draw_group<4, It, V, kStore, true>(seed, R, d, v, items, f, tab, ctot, pw, s_lim, s_mag, pg)) return;
    }
    for (; d < n2; ++d) {
      const uint64_t v[1] = {mt_temper(mt_twist(a0, a1, mt_twist(c0, c1, a0)))};
      a0 = a1;
      a1 = mt_step(a1, static_cast<uint32_t>(d + 2));
      c0 = c1;
      c1 = mt_step(c1, static_cast<uint32_t>(d - 154));
      if (draw_group<1, It, V, kStore>(seed, R, d, v, items, f, tab, ctot, pw, s_lim, s_mag)) return;
    }
    if (d < draws) {  // beyond the first block (R > 312)
      f = shuffle_slow<It, V, kStore>(seed, d, R - d, items, f, tab, ctot, pw);
      return;
    }
  }
  if constexpr (!kStore)
    if (R >= 1) f.add(tab[*items.at(0)], ctot, pw);
}

// Shared-memory layout of one block (bytes); hist bins only when used.
// Table image at the start of a block's shared memory: bounded() limits and
// magics (R+2 each), the {first class, duration} table, the class suffix
// weights in the fold's width V; 16-byte padded so one bulk copy moves it.
__host__ __device__ inline size_t sweep_table_bytes(int R, int W, int stride, size_t vbytes) {
  return round16(16 * static_cast<size_t>(R + 2) + 8 * static_cast<size_t>(W) * R + vbytes * W * stride);
}
__host__ __device__ inline size_t sweep_smem(int R, int W, int stride, int nhist, size_t vbytes) {
  const int per_word = R <= 256 ? 4 : 2;
  return sweep_table_bytes(R, W, stride, vbytes) + 4 * static_cast<size_t>(nhist) * kBins +
         4 * static_cast<size_t>(kSweepThreads) * ((R + per_word - 1) / per_word + 1) + 16;  // + mbarrier
}

// Outputs 0..n-1 of mt19937_64(seed), four per iteration from the same
// phase-split register cursors as shuffle_fold (n <= 311: first block only),
// each handed to `use(d, v)` in order.
template <typename F>
__device__ __forceinline__ void mt_outputs(uint64_t seed, int n, F&& use) {
  uint64_t a0 = seed, a1 = mt_step(seed, 1), b = seed;
#pragma unroll 4
  for (uint32_t k = 1; k <= 156; ++k) b = mt_step(b, k);
  const int n1 = min(n, 156);
  int d = 0;
  for (; d + 3 < n1; d += 4) {
    const uint32_t u = static_cast<uint32_t>(d);
    const uint64_t a2 = mt_step(a1, u + 2), a3 = mt_step(a2, u + 3), a4 = mt_step(a3, u + 4);
    const uint64_t b1 = mt_step(b, u + 157), b2 = mt_step(b1, u + 158), b3 = mt_step(b2, u + 159);
    const uint64_t v0 = mt_temper(mt_twist(a0, a1, b)), v1 = mt_temper(mt_twist(a1, a2, b1)),
                   v2 = mt_temper(mt_twist(a2, a3, b2)), v3 = mt_temper(mt_twist(a3, a4, b3));
    a0 = a4;
    a1 = mt_step(a4, u + 5);
    b = mt_step(b3, u + 160);
    use(d, v0);
    use(d + 1, v1);
    use(d + 2, v2);
    use(d + 3, v3);
  }
  for (; d < n1; ++d) {
    use(d, mt_temper(mt_twist(a0, a1, b)));
    a0 = a1;
    a1 = mt_step(a1, static_cast<uint32_t>(d + 2));
    b = mt_step(b, static_cast<uint32_t>(d + 157));
  }
  if (d < n) {
    uint64_t c0 = seed, c1 = mt_step(seed, 1);
    for (; d < n; ++d) {
      use(d, mt_temper(mt_twist(a0, a1, mt_twist(c0, c1, a0))));
      a0 = a1;
      a1 = mt_step(a1, static_cast<uint32_t>(d + 2));
      c0 = c1;
      c1 = mt_step(c1, static_cast<uint32_t>(d - 154));
    }
  }
}

// Per-thread sweep statistics: packed min/max keys (m << key_bits) | offset
// (lowest seed wins ties), sums, the E histogram and, for clusters, the
// straggler histogram in shared memory; reduced per warp, then one set of
// global atomics per block (flush).
struct StatAcc {
  unsigned long long kmin = ~0ULL, kmax = 0, ikmin = ~0ULL, ikmax = 0;  // makespan / iteration-time keys
  long long msum = 0, cnt = 0, isum = 0;
  double sq = 0.0, ssum = 0.0;
  __device__ __forceinline__ void add(const ChainArgs& a, uint64_t seed, int64_t m, int64_t hi, int64_t lo,
                                      int* s_hist, int* s_shist) {
    const unsigned long long off = seed - a.key_base;
    kmin = min(kmin, (static_cast<unsigned long long>(m) << a.key_bits) | off);
    kmax = max(kmax, (static_cast<unsigned long long>(m) << a.key_bits) | ((1ULL << a.key_bits) - 1 - off));
    if (a.cluster) {  // iteration time = slowest worker (differs from m when PS ops take time)
      ikmin = min(ikmin, (static_cast<unsigned long long>(hi) << a.key_bits) | off);
      ikmax = max(ikmax, (static_cast<unsigned long long>(hi) << a.key_bits) | ((1ULL << a.key_bits) - 1 - off));
      isum += hi;
    }
    msum += m;
    ++cnt;
    sq += static_cast<double>(m) * static_cast<double>(m);
    if (a.do_e) {
      const int bin = static_cast<int>(floor(1000.0 * static_cast<double>(a.U - m) /
                                             static_cast<double>(a.U - a.L)));
      atomicAdd(&s_hist[min(max(bin, 0), kBins - 1)], 1);
    }
    if (a.cluster) {
      int bin = 0;
      if (hi > 0) {
        ssum += static_cast<double>(hi - lo) / static_cast<double>(hi);
        bin = min(static_cast<int>(floor(1000.0 * static_cast<double>(hi - lo) / static_cast<double>(hi))),
                  kBins - 1);
      }
      atomicAdd(&s_shist[bin], 1);
    }
  }
  __device__ __forceinline__ void flush(const ChainArgs& a, const int* s_hist, const int* s_shist) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      kmin = min(kmin, __shfl_xor_sync(~0u, kmin, o));
      kmax = max(kmax, __shfl_xor_sync(~0u, kmax, o));
      ikmin = min(ikmin, __shfl_xor_sync(~0u, ikmin, o));
      ikmax = max(ikmax, __shfl_xor_sync(~0u, ikmax, o));
      isum += __shfl_xor_sync(~0u, isum, o);
      msum += __shfl_xor_sync(~0u, msum, o);
      cnt += __shfl_xor_sync(~0u, cnt, o);
      sq += __shfl_xor_sync(~0u, sq, o);
      ssum += __shfl_xor_sync(~0u, ssum, o);
    }
    if (!a.i64) return;  // explicit-orders calls without statistics
    if ((threadIdx.x & 31) == 0 && cnt > 0) {
      atomicMin(&a.i64[0], kmin);
      atomicMax(&a.i64[1], kmax);
      atomicAdd(&a.i64[2], static_cast<unsigned long long>(msum));
      atomicAdd(&a.i64[3], static_cast<unsigned long long>(cnt));
      if (a.cluster) {
        atomicMin(&a.i64[4], ikmin);
        atomicMax(&a.i64[5], ikmax);
        atomicAdd(&a.i64[6], static_cast<unsigned long long>(isum));
      }
      atomicAdd(&a.f64[0], sq);
      atomicAdd(&a.f64[1], ssum);
    }
    __syncthreads();
    if (a.do_e)
      for (int k = threadIdx.x; k < kBins; k += blockDim.x)
        if (s_hist[k]) atomicAdd(&a.i64[8 + k], static_cast<unsigned long long>(s_hist[k]));
    if (a.cluster)
      for (int k = threadIdx.x; k < kBins; k += blockDim.x)
        if (s_shist[k]) atomicAdd(&a.i64[8 + kBins + k], static_cast<unsigned long long>(s_shist[k]));
  }
};

// Gated runs with reorder noise: the noise only permutes the
// gate sequence up front — adjacent swaps with probability p, one draw of the
// separate stream Rng(splitmix64(choice_seed ^ salt)) per position, channels
// in resource order (sim.cpp:94-114) — so the closed form still applies to
// the permuted sequence. The shuffle then has to be stored whole (the fused
// right-to-left fold needs the final order), hence a separate path.
template <bool kOn>
struct NoiseState {
  __device__ __forceinline__ void init(uint64_t) {}
};
template <>
struct NoiseState<true> {
  MtStream m;
  __device__ __forceinline__ void init(uint64_t s) { m.init(s); }
};

template <typename T, bool kOrders, typename V, bool kNoisy = false>
__global__ void __launch_bounds__(kSweepThreads, 3) chain_sweep_kernel(ChainArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int R = a.R, W = a.W;
  uint64_t* s_lim = reinterpret_cast<uint64_t*>(smem);
  uint64_t* s_mag = s_lim + (R + 2);
  uint2* s_tab = reinterpret_cast<uint2*>(s_mag + (R + 2));
  V* s_pw = reinterpret_cast<V*>(s_tab + W * R);
  int* s_hist = reinterpret_cast<int*>(smem + sweep_table_bytes(R, W, a.stride, sizeof(V)));
  const int nhist = (a.do_e ? 1 : 0) + (a.cluster ? 1 : 0);
  int* s_shist = s_hist + (a.do_e ? kBins : 0);  // straggler bins (clusters)
  uint32_t* s_items = reinterpret_cast<uint32_t*>(s_hist + nhist * kBins);
  // mbarrier in the last 16 bytes of the dynamic region (sweep_smem)
  uint64_t* tables_ready = reinterpret_cast<uint64_t*>(smem + a.mbar_off);
  if (a.blob) {  // the whole table image in one bulk copy on the TMA engine
    if (threadIdx.x == 0) mbar_init(tables_ready, 1);
    __syncthreads();
    if (threadIdx.x == 0) {
      mbar_expect_tx(tables_ready, a.blob_bytes);
      bulk_g2s(smem, a.blob, a.blob_bytes, tables_ready);
    }
  } else {
    for (int k = threadIdx.x; k < R + 2; k += blockDim.x) {
      s_lim[k] = a.lim[k];
      s_mag[k] = a.mag[k];
    }
    for (int k = threadIdx.x; k < W * R; k += blockDim.x) s_tab[k] = a.tab[k];
    for (int k = threadIdx.x; k < W * a.stride; k += blockDim.x) s_pw[k] = static_cast<V>(a.pwsuf[k]);
  }
  for (int k = threadIdx.x; k < nhist * kBins; k += blockDim.x) s_hist[k] = 0;
  if (a.blob) mbar_wait(tables_ready, 0);
  __syncthreads();
  const Items<T> items{s_items + threadIdx.x};

  StatAcc acc;
  const int64_t nthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < a.count;
       idx += nthreads) {
    const uint64_t seed = a.seed_lo + static_cast<uint64_t>(idx);
    int64_t hi = 0, lo = INT64_MAX;
    NoiseState<kNoisy> noise;  // one stream per run, across the workers' channels
    if constexpr (kNoisy) noise.init(splitmix64(seed ^ kNoiseSalt));
    for (int w = 0; w < W; ++w) {
      const uint2* tab = s_tab + w * R;
      const V* pw = s_pw + w * a.stride;
      const V ctot = static_cast<V>(a.ctot[w]);
      FoldT<V> f{a.nc, 0, -1};
      if constexpr (kOrders) {
        // rows validated here as they are read (not on the host): entries in
        // [0, R) (bad bit 1), no repeats (bit 2; the shuffle area is free in
        // this mode and holds a per-thread seen-bitset)
        const int32_t* o = a.orders + idx * R;
        uint32_t* seen = s_items + threadIdx.x;  // word q at seen[q * kSweepThreads]
        for (int q = 0; q < (R + 31) / 32; ++q) seen[q * kSweepThreads] = 0;
        int bad = 0;
        for (int k = R - 1; k >= 0; --k) {
          int32_t c = o[k];
          if (static_cast<uint32_t>(c) >= static_cast<uint32_t>(R)) {
            bad |= 1;
            c = 0;
          } else {
            uint32_t& wd = seen[(c >> 5) * kSweepThreads];
            bad |= (wd >> (c & 31)) & 1u ? 2 : 0;
            wd |= 1u << (c & 31);
          }
          f.add(tab[c], ctot, pw);
        }
        if (bad) atomicOr(a.bad_order, bad);
      } else {
        const uint64_t ws = a.cluster ? splitmix64(seed ^ (kPhi * static_cast<uint64_t>(w + 1))) : seed;
        if constexpr (kNoisy) {
          shuffle_fold<Items<T>, V, true>(ws, R, items, f, tab, ctot, pw, s_lim, s_mag);  // rank order = the shuffle
          auto swap_at = [&](int pos, uint64_t v) {   // noise swaps -> gate order
            if ((v >> 11) < a.noise_thr) {
              T* p0 = items.at(pos - 1);
              T* p1 = items.at(pos);
              const T x = *p0;
              *p0 = *p1;
              *p1 = x;
            }
          };
          if (W == 1 && R - 1 <= 311) {  // the run's only channel: the stream's first R-1 outputs
            mt_outputs(splitmix64(seed ^ kNoiseSalt), R - 1, [&](int d, uint64_t v) { swap_at(d + 1, v); });
          } else {
            for (int pos = 1; pos < R; ++pos) swap_at(pos, noise.m.next());
          }
          for (int pos = R - 1; pos >= 0; --pos) f.add(tab[*items.at(pos)], ctot, pw);
        } else if (a.force_slow) {
          items.init(R);
          f = shuffle_slow(ws, 0, R, items, f, tab, ctot, pw);
        } else {
          shuffle_fold<Items<T>, V, false, true>(ws, R, items, f, tab, ctot, pw, s_lim, s_mag);
        }
      }
      if (f.G > 0) f.best = max(f.best, pw[0]);  // bin 0: computes needing no recv
      const int64_t tcpu = f.best < 0 ? 0 : static_cast<int64_t>(f.best);
      const int64_t c64 = static_cast<int64_t>(ctot);
      const int64_t mw = a.cluster ? max(tcpu, max(c64, tcpu) + a.send_tot[w]) : max(tcpu, c64);
      if (a.worker_ms) a.worker_ms[idx * W + w] = mw;
      hi = max(hi, mw);
      lo = min(lo, mw);
    }
    const int64_t m = hi;  // worker graph: the makespan; cluster: iteration time
    if (a.makespans) a.makespans[idx] = m;
    acc.add(a, seed, m, hi, lo, s_hist, s_shist);
  }
  acc.flush(a, s_hist, s_shist);
}

// ---- workers with several channels (clusters with several parameter
// servers): each channel runs its recvs back to back in the gate order
// restricted to it, so a recv's completion c(r) is a prefix sum on its own
// channel. With nested classes the ERD value over release times becomes
//     T_cpu = max(S(0), max over recvs r of c(r) + S(first[r]))
// (class j is released at max{c(r) : first[r] <= j}, and S is non-increasing
// in j), a right-to-left pass over the stored shuffle with one suffix sum per
// channel. Reorder noise permutes each channel's subsequence with one stream
// across the channels in resource order (sim.cpp:94-114). tab[].x carries the
// channel in bits 24..31.
template <typename T, typename V, bool kNoisy>
__global__ void __launch_bounds__(kSweepThreads, 3) chain_multi_kernel(ChainArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int R = a.R, W = a.W, nch = a.nch;
  uint64_t* s_lim = reinterpret_cast<uint64_t*>(smem);
  uint64_t* s_mag = s_lim + (R + 2);
  uint2* s_tab = reinterpret_cast<uint2*>(s_mag + (R + 2));
  V* s_pw = reinterpret_cast<V*>(s_tab + W * R);
  int* s_hist = reinterpret_cast<int*>(smem + sweep_table_bytes(R, W, a.stride, sizeof(V)));
  const int nhist = (a.do_e ? 1 : 0) + (a.cluster ? 1 : 0);
  int* s_shist = s_hist + (a.do_e ? kBins : 0);
  uint32_t* s_items = reinterpret_cast<uint32_t*>(s_hist + nhist * kBins);
  uint64_t* tables_ready = reinterpret_cast<uint64_t*>(smem + a.mbar_off);
  if (threadIdx.x == 0) mbar_init(tables_ready, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(tables_ready, a.blob_bytes);
    bulk_g2s(smem, a.blob, a.blob_bytes, tables_ready);
  }
  for (int k = threadIdx.x; k < nhist * kBins; k += blockDim.x) s_hist[k] = 0;
  mbar_wait(tables_ready, 0);
  __syncthreads();
  const Items<T> items{s_items + threadIdx.x};
  StatAcc acc;
  const int64_t nthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < a.count;
       idx += nthreads) {
    const uint64_t seed = a.seed_lo + static_cast<uint64_t>(idx);
    int64_t hi = 0, lo = INT64_MAX;
    NoiseState<kNoisy> noise;
    if constexpr (kNoisy) noise.init(splitmix64(seed ^ kNoiseSalt));
    for (int w = 0; w < W; ++w) {
      const uint2* tab = s_tab + w * R;
      const V* pw = s_pw + w * a.stride;
      FoldT<V> f{0, 0, 0};
      const uint64_t ws = a.cluster ? splitmix64(seed ^ (kPhi * static_cast<uint64_t>(w + 1))) : seed;
      shuffle_fold<Items<T>, V, true>(ws, R, items, f, nullptr, V(0), nullptr, s_lim, s_mag);
      if constexpr (kNoisy)
        for (int ch = 0; ch < nch; ++ch) {
          int prev = -1;
          for (int pos = 0; pos < R; ++pos) {
            T* p1 = items.at(pos);
            if (static_cast<int>(tab[*p1].x >> 24) != ch) continue;
            if (prev >= 0 && (noise.m.next() >> 11) < a.noise_thr) {
              T* p0 = items.at(prev);
              const T x = *p0;
              *p0 = *p1;
              *p1 = x;
            }
            prev = pos;
          }
        }
      V ct[kMaxChannelsDev], sfx[kMaxChannelsDev];
#pragma unroll
      for (int ch = 0; ch < kMaxChannelsDev; ++ch) {
        ct[ch] = ch < nch ? static_cast<V>(a.ctot[w * nch + ch]) : V(0);
        sfx[ch] = 0;
      }
      V best = pw[0];  // S(0): every class's work after time 0
      for (int pos = R - 1; pos >= 0; --pos) {
        const uint2 e = tab[*items.at(pos)];
        const int ch = static_cast<int>(e.x >> 24);
        V c = 0;
#pragma unroll
        for (int k = 0; k < kMaxChannelsDev; ++k)
          if (k == ch) c = ct[k] - sfx[k];
        best = max(best, c + pw[e.x & 0xFFFFFFu]);
#pragma unroll
        for (int k = 0; k < kMaxChannelsDev; ++k)
          if (k == ch) sfx[k] += static_cast<V>(e.y);
      }
      const int64_t tcpu = static_cast<int64_t>(best);
      int64_t mw = tcpu;
#pragma unroll
      for (int k = 0; k < kMaxChannelsDev; ++k)
        if (k < nch) {
          const int64_t c64 = static_cast<int64_t>(ct[k]);
          mw = max(mw, a.cluster ? max(c64, tcpu) + a.send_tot[w * nch + k] : c64);
        }
      if (a.worker_ms) a.worker_ms[idx * W + w] = mw;
      hi = max(hi, mw);
      lo = min(lo, mw);
    }
    if (a.makespans) a.makespans[idx] = hi;
    acc.add(a, seed, hi, hi, lo, s_hist, s_shist);
  }
  acc.flush(a, s_hist, s_shist);
}

// ---- general worker DAGs: SURVEY Appendix A.2 without the nesting ------
//
// When the compute ops' recv-ancestor sets are not nested (branches, series-
// parallel DAGs) the fold above does not apply, but A.2 still does: the
// channel runs the gate order back to back (completion of position k is the
// prefix sum c_k), and the single compute server's completion is the ERD
// value over release positions,
//     T_cpu = max over k in [-1, R) of  c_k + S(k),   S(k) = Σ w_j [lp_j >= k],
// where class j (compute ops sharing one recv-ancestor set) is released at
// its latest recv position lp_j = max{pos[r] : r in set(j)} (c_{-1} = 0, the
// classes with no recv ancestor count only at k = -1). The host compiles the
// graph once into a straight-line program over "join" classes (sets with two
// or more recvs), each as the max over a few generators — recv positions or
// earlier joins held in live slots (csrc/host/sweep.cpp) — so one ordering
// costs the shuffle, one scatter of positions, the program (a few shared-
// memory reads per generator) and one right-to-left pass over the position
// bins. Classes whose set is a single recv {r} are weighed with the recv's
// table entry instead of a bin. One thread owns one ordering; its arrays
// (gate order, positions + slots, bins) sit in shared memory as
// [index][thread] columns so every access hits the thread's own bank
// whatever the index; the program and tables are read by all lanes at the
// same address (broadcast).
constexpr int kDagThreads = 64;

template <typename V>
struct DagEnt {  // per recv column: duration, weight of the classes whose set is {recv}
  V d, wr;
};

struct DagArgs {
  int nrec, L;                      // program records (multiple of 4), live slots
  int64_t lex_first;                // lexicographic source: permutation number of idx 0
  const unsigned long long* fact;   // k! for k <= 20 (lexicographic source)
};

// Table image: lim/mag (R+2 each), program records [nrec] (uint4: byte
// offsets of three generators and the output inside a thread's value
// column), DagEnt [W][R], record weights [W][nrec], empty-set weights [W];
// 16-byte padded (one bulk copy).
__host__ __device__ inline size_t dag_table_bytes(int R, int W, int nrec, size_t vb) {
  return round16(16 * static_cast<size_t>(R + 2) + 16 * static_cast<size_t>(nrec) + 2 * vb * W * R +
                 vb * W * nrec + vb * W);
}
// per thread: gate order (R items), values (R recv positions + L slots + 1
// discard), bins (R + 1)
__host__ __device__ inline size_t dag_thread_bytes(int R, int L, size_t tb, size_t vb) {
  const int per = tb == 1 ? 4 : 2;
  return 4 * static_cast<size_t>((R + per - 1) / per + (R + L + 1 + per - 1) / per) + vb * (R + 1);
}
__host__ __device__ inline size_t dag_smem(int R, int W, int nrec, int L, int nhist, size_t tb, size_t vb) {
  return round16(dag_table_bytes(R, W, nrec, vb) + 4 * static_cast<size_t>(nhist) * kBins +
                 kDagThreads * dag_thread_bytes(R, L, tb, vb)) + 16;  // + mbarrier
}
// record flags: first generator = the previous record's result (ACC);
// output of a real record (updates ACC; padding records do not)
constexpr uint32_t kDagAccFlag = 0x80000000u, kDagRealFlag = 0x80000000u, kDagOffMask = 0x7FFFFFFFu;
// byte offset of item k inside a thread's Items<T, nt> column
__host__ __device__ inline uint32_t dag_item_off(int k, size_t tb, int nt = kDagThreads) {
  return tb == 1 ? static_cast<uint32_t>(k * nt - (k & 3) * (nt - 1))
                 : static_cast<uint32_t>((k >> 1) * nt * 4 + (k & 1) * 2);
}

// kSrc: 0 random_schedule(seed) (per-worker derived seeds on clusters),
// 1 explicit orders (rows validated as read), 2 lexicographic permutation
// number lex_first + idx (brute force; R <= 20, worker plans).
template <typename T, typename V, bool kNoisy, int kSrc>
__global__ void __launch_bounds__(kDagThreads) dag_sweep_kernel(ChainArgs a, DagArgs g) {
  constexpr int NT = kDagThreads;
  extern __shared__ __align__(16) unsigned char smem[];
  const int R = a.R, W = a.W, NR = g.nrec;
  const size_t vb = sizeof(V);
  const uint64_t* s_lim = reinterpret_cast<const uint64_t*>(smem);
  const uint64_t* s_mag = s_lim + (R + 2);
  const uint4* s_rec = reinterpret_cast<const uint4*>(s_mag + (R + 2));
  const DagEnt<V>* s_ent = reinterpret_cast<const DagEnt<V>*>(s_rec + NR);
  const V* s_wj = reinterpret_cast<const V*>(s_ent + W * R);
  const V* s_w0 = s_wj + W * NR;
  const int nhist = (a.do_e ? 1 : 0) + (a.cluster ? 1 : 0);
  int* s_hist = reinterpret_cast<int*>(smem + dag_table_bytes(R, W, NR, vb));
  int* s_shist = s_hist + (a.do_e ? kBins : 0);
  V* s_bins = reinterpret_cast<V*>(s_hist + nhist * kBins) + threadIdx.x;  // [k][NT]
  uint32_t* s_words = reinterpret_cast<uint32_t*>(reinterpret_cast<V*>(s_hist + nhist * kBins) + (R + 1) * NT);
  const Items<T, NT> perm{s_words + threadIdx.x};
  const Items<T, NT> val{s_words + Items<T, NT>::words(R) * NT + threadIdx.x};
  uint64_t* tables_ready = reinterpret_cast<uint64_t*>(smem + a.mbar_off);
  if (threadIdx.x == 0) mbar_init(tables_ready, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(tables_ready, a.blob_bytes);
    bulk_g2s(smem, a.blob, a.blob_bytes, tables_ready);
  }
  for (int k = threadIdx.x; k < nhist * kBins; k += blockDim.x) s_hist[k] = 0;
  for (int k = 0; k <= R; ++k) s_bins[k * NT] = V(0);  // the fold re-zeroes every bin it reads
  mbar_wait(tables_ready, 0);
  __syncthreads();
  unsigned char* vcol = reinterpret_cast<unsigned char*>(val.base);  // value column (byte offsets)

  StatAcc acc;
  const int64_t nthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < a.count;
       idx += nthreads) {
    const uint64_t seed = a.seed_lo + static_cast<uint64_t>(idx);
    int64_t hi = 0, lo = INT64_MAX;
    NoiseState<kNoisy> noise;
    if constexpr (kNoisy) noise.init(splitmix64(seed ^ kNoiseSalt));
    for (int w = 0; w < W; ++w) {
      const DagEnt<V>* ent = s_ent + w * R;
      // 1. gate order (recv column at each position) and positions
      if constexpr (kSrc == 1) {
        const int32_t* o = a.orders + idx * R;
        const T none = static_cast<T>(~T(0));
        for (int c = 0; c < R; ++c) *val.at(c) = none;
        int bad = 0;
        for (int k = 0; k < R; ++k) {
          int32_t c = o[k];
          if (static_cast<uint32_t>(c) >= static_cast<uint32_t>(R)) {
            bad |= 1;
            c = 0;
          } else if (*val.at(c) != none) {
            bad |= 2;
          }
          *val.at(c) = static_cast<T>(k);
          *perm.at(k) = static_cast<T>(c);
        }
        if (bad) atomicOr(a.bad_order, bad);
      } else {
        if constexpr (kSrc == 2) {
          unsigned long long k = static_cast<unsigned long long>(g.lex_first + idx);
          uint32_t left = (R >= 32) ? ~0u : ((1u << R) - 1u);
          for (int pos = 0; pos < R; ++pos) {
            const unsigned long long f = g.fact[R - 1 - pos];
            const int q = static_cast<int>(k / f);
            k -= static_cast<unsigned long long>(q) * f;
            const int c = nth_bit(left, q);
            left &= ~(1u << c);
            *perm.at(pos) = static_cast<T>(c);
          }
        } else {
          const uint64_t ws = a.cluster ? splitmix64(seed ^ (kPhi * static_cast<uint64_t>(w + 1))) : seed;
          FoldT<V> f{0, 0, 0};
          shuffle_fold<Items<T, NT>, V, true>(ws, R, perm, f, nullptr, V(0), nullptr, s_lim, s_mag);
          if constexpr (kNoisy) {  // noise swaps on the rank order -> gate order (sim.cpp:106-114)
            auto swap_at = [&](int pos, uint64_t v) {
              if ((v >> 11) < a.noise_thr) {
                T* p0 = perm.at(pos - 1);
                T* p1 = perm.at(pos);
                const T x = *p0;
                *p0 = *p1;
                *p1 = x;
              }
            };
            if (W == 1 && R - 1 <= 311) {
              mt_outputs(splitmix64(seed ^ kNoiseSalt), R - 1, [&](int d, uint64_t v) { swap_at(d + 1, v); });
            } else {
              for (int pos = 1; pos < R; ++pos) swap_at(pos, noise.m.next());
            }
          }
        }
        for (int k = 0; k < R; ++k) *val.at(*perm.at(k)) = static_cast<T>(k);
      }
      // 2. latest recv position of every join class, weights into bins:
      // groups of four records, generators loaded before outputs stored
      {
        const V* wj = s_wj + w * NR;
        int accv = 0;  // the previous real record's result
        for (int q = 0; q < NR; q += 4) {
          uint4 rc[4];
          V wt[4];
          int lp[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            rc[i] = s_rec[q + i];
            wt[i] = wj[q + i];
          }
          int x[4], y[4], z[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            x[i] = *reinterpret_cast<const T*>(vcol + (rc[i].x & kDagOffMask));
            y[i] = *reinterpret_cast<const T*>(vcol + rc[i].y);
            z[i] = *reinterpret_cast<const T*>(vcol + rc[i].z);
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            lp[i] = max(max((rc[i].x & kDagAccFlag) ? accv : x[i], y[i]), z[i]);
            accv = (rc[i].w & kDagRealFlag) ? lp[i] : accv;
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) *reinterpret_cast<T*>(vcol + (rc[i].w & kDagOffMask)) = static_cast<T>(lp[i]);
          // equal positions inside the group: the later record carries the sum
#pragma unroll
          for (int j = 1; j < 4; ++j)
#pragma unroll
            for (int i = 0; i < j; ++i)
              if (lp[i] == lp[j]) {
                wt[j] += wt[i];
                wt[i] = V(0);
              }
          V old[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) old[i] = s_bins[lp[i] * NT];
#pragma unroll
          for (int i = 0; i < 4; ++i) s_bins[lp[i] * NT] = old[i] + wt[i];
        }
      }
      // 3. right-to-left: c_k + S(k); every bin is re-zeroed as it is read
      const V ctot = static_cast<V>(a.ctot[w]);
      V S = 0, suffix = 0, best = 0;
      auto step = [&](int r, int k) {
        const DagEnt<V> e = ent[r];
        S += s_bins[k * NT] + e.wr;
        s_bins[k * NT] = V(0);
        best = max(best, ctot - suffix + S);
        suffix += e.d;
      };
      int k = R - 1;
      if constexpr (sizeof(T) == 1) {
        for (; k >= 0 && (k & 3) != 3; --k) step(*perm.at(k), k);
        for (; k >= 3; k -= 4) {  // four positions per word of the gate-order column
          const uint32_t wd = perm.base[(k >> 2) * NT];
          step(wd >> 24, k);
          step((wd >> 16) & 0xFF, k - 1);
          step((wd >> 8) & 0xFF, k - 2);
          step(wd & 0xFF, k - 3);
        }
      } else {
        for (; k >= 0; --k) step(*perm.at(k), k);
      }
      best = max(best, S + s_w0[w]);
      const int64_t tcpu = static_cast<int64_t>(best);
      const int64_t c64 = static_cast<int64_t>(ctot);
      const int64_t mw = a.cluster ? max(tcpu, max(c64, tcpu) + a.send_tot[w]) : max(tcpu, c64);
      if (a.worker_ms) a.worker_ms[idx * W + w] = mw;
      hi = max(hi, mw);
      lo = min(lo, mw);
    }
    if (a.makespans) a.makespans[idx] = hi;
    acc.add(a, seed, hi, hi, lo, s_hist, s_shist);
  }
  acc.flush(a, s_hist, s_shist);
}

// ---- clusters whose parameter-server ops take time ----------------------
//
// With PS ops of positive duration the full makespan depends on the order in
// which each worker's channels send its gradients, which the reference picks
// with draws from the run's shared choice stream (sim.cpp:163-186: the sends
// are unprioritized, so every ready send is a candidate), and on the PS
// cores' choices among ready PS ops (again draws). Everything before a
// worker's last compute op completes is still SURVEY A.2: on chain-class
// workers whose compute ops are totally ordered there are no draws there
// (one candidate at a time on the core; a channel admits only its next recv
// in gate order, the sends are not ready yet), each channel's recv
// completions are prefix sums of its gate order and the release of the
// sends is the fold's T_cpu (the multi-channel form of chain_multi_kernel).
// So a run is: per worker the shuffle and the fold, then an exact replica of
// sim.cpp:194-233 restricted to the resources that can draw — the PS cores
// and each released channel — with the reference's round structure
// (completions at t, then passes of try_start in resource order + same-time
// completions of zero-duration ops until nothing changes). Candidates come
// in op-index order: a channel's are its unsent ready sends plus its next
// recv in gate order (the only admitted one), a PS core's are its ready ops.
// Host checks (csrc/host/sweep.cpp): PS devices with one compute unit each,
// fed only by sends, workers as above, every worker's last compute op of
// positive duration (its completion, hence the release of the sends,
// happens at the start of a time step).
struct PsArgs {
  int S, Q, nps, nslot;           // sends per worker, PS ops, PS cores, active resources
  int sw, qw;                     // 32-bit words of a send bitset / a PS-op bitset
  const int16_t* recv_sb;         // [R] the worker's sends before recv column c (op-index order)
  const uint32_t* ch_mask;        // [nch][sw] sends on each channel
  const int64_t* send_d;          // [W][S]
  const int32_t* send_succ_off;   // [W*S + 1]
  const int16_t* send_succ;       // PS op indices
  const int64_t* ps_d;            // [Q]
  const uint8_t* ps_missing;      // [Q] predecessor counts
  const int32_t* ps_succ_off;     // [Q + 1]
  const int16_t* ps_succ;
  const uint32_t* core_mask;      // [nps][qw] PS ops of each core
  const int32_t* slots;           // [nslot] resource order: PS core k -> -1 - k, channel (w, ch) -> w * nch + ch
};
constexpr int kPsThreads = 64;

// per thread: gate orders (W x R items), pending-send bits (W x sw words),
// PS missing counts (Q bytes), PS ready bits (qw words), worker scalars
// (5 words: release time, device end, released), channel scalars (4 words:
// end, running, next gate position), core scalars (3 words: op, end)
__host__ __device__ inline size_t ps_thread_bytes(int W, int R, int S, int Q, int nch, int nps, size_t tb) {
  const int per = tb == 1 ? 4 : 2;
  return 4 * (static_cast<size_t>(W) * ((R + per - 1) / per) + static_cast<size_t>(W) * ((S + 31) / 32) +
              static_cast<size_t>((Q + 3) / 4) + static_cast<size_t>((Q + 31) / 32) + 5 * static_cast<size_t>(W) +
              4 * static_cast<size_t>(W) * nch + 3 * static_cast<size_t>(nps));
}

template <typename T, typename V, bool kNoisy>
__global__ void __launch_bounds__(kPsThreads) cluster_ps_kernel(ChainArgs a, PsArgs q) {
  constexpr int NT = kPsThreads;
  extern __shared__ __align__(16) unsigned char smem[];
  const int R = a.R, W = a.W, S = q.S, Q = q.Q, nch = a.nch, nps = q.nps;
  uint64_t* s_lim = reinterpret_cast<uint64_t*>(smem);
  const int nk = max(S + 2, Q + 1) + 1;  // bounded() constants for n < nk
  uint64_t* s_mag = s_lim + nk;
  uint2* s_tab = reinterpret_cast<uint2*>(s_mag + nk);
  V* s_pw = reinterpret_cast<V*>(s_tab + W * R);
  int* s_hist = reinterpret_cast<int*>(smem + round16(16ull * nk + 8ull * W * R + sizeof(V) * W * a.stride));
  const int nhist = (a.do_e ? 1 : 0) + 1;
  int* s_shist = s_hist + (a.do_e ? kBins : 0);
  uint32_t* col = reinterpret_cast<uint32_t*>(s_hist + nhist * kBins) + threadIdx.x;  // this thread's column
  const int gw = Items<T, NT>::words(R);
  auto gate = [&](int w) { return Items<T, NT>{col + static_cast<size_t>(w) * gw * NT}; };
  uint32_t* pend = col + static_cast<size_t>(W) * gw * NT;        // [w][sw] words
  uint32_t* qmiss_base = pend + static_cast<size_t>(W) * q.sw * NT;  // Q bytes
  const Items<uint8_t, NT> qmiss{qmiss_base};
  uint32_t* qready = qmiss_base + static_cast<size_t>((Q + 3) / 4) * NT;  // qw words
  uint32_t* wsc = qready + static_cast<size_t>(q.qw) * NT;                // [w][5] words
  uint32_t* csc = wsc + static_cast<size_t>(5 * W) * NT;                   // [w*nch + ch][4] words
  uint32_t* ksc = csc + static_cast<size_t>(4 * W * nch) * NT;             // [k][3] words
  auto ld64 = [&](uint32_t* base, int word) -> int64_t {
    const uint32_t lo = base[static_cast<size_t>(word) * NT], hi = base[static_cast<size_t>(word + 1) * NT];
    return static_cast<int64_t>((static_cast<uint64_t>(hi) << 32) | lo);
  };
  auto st64 = [&](uint32_t* base, int word, int64_t v) {
    base[static_cast<size_t>(word) * NT] = static_cast<uint32_t>(v);
    base[static_cast<size_t>(word + 1) * NT] = static_cast<uint32_t>(static_cast<uint64_t>(v) >> 32);
  };
  auto w32 = [&](uint32_t* base, int word) -> int32_t& {
    return *reinterpret_cast<int32_t*>(&base[static_cast<size_t>(word) * NT]);
  };
  // worker w: T at 5w, device end at 5w+2, released at 5w+4
  // channel i = w*nch + ch: end at 4i, running at 4i+2 (-1 idle, -2 recv, s send), next gate position at 4i+3
  // core k: op at 3k, end at 3k+1
  uint64_t* tables_ready = reinterpret_cast<uint64_t*>(smem + a.mbar_off);
  if (threadIdx.x == 0) mbar_init(tables_ready, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(tables_ready, a.blob_bytes);
    bulk_g2s(smem, a.blob, a.blob_bytes, tables_ready);
  }
  for (int k = threadIdx.x; k < nhist * kBins; k += blockDim.x) s_hist[k] = 0;
  mbar_wait(tables_ready, 0);
  __syncthreads();
  const int16_t* recv_sb = q.recv_sb;

  StatAcc acc;
  const int64_t nthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < a.count;
       idx += nthreads) {
    const uint64_t seed = a.seed_lo + static_cast<uint64_t>(idx);
    NoiseState<kNoisy> noise;
    if constexpr (kNoisy) noise.init(splitmix64(seed ^ kNoiseSalt));
    int64_t t = INT64_MAX, mk = 0;
    // 1. per worker: gate order, T_cpu (fold), each channel's state at the release
    for (int w = 0; w < W; ++w) {
      const Items<T, NT> g = gate(w);
      const uint2* tab = s_tab + w * R;
      const V* pw = s_pw + w * a.stride;
      FoldT<V> f{0, 0, 0};
      const uint64_t ws = splitmix64(seed ^ (kPhi * static_cast<uint64_t>(w + 1)));
      shuffle_fold<Items<T, NT>, V, true>(ws, R, g, f, nullptr, V(0), nullptr, s_lim, s_mag);
      if constexpr (kNoisy)
        for (int ch = 0; ch < nch; ++ch) {
          int prev = -1;
          for (int pos = 0; pos < R; ++pos) {
            T* p1 = g.at(pos);
            if (static_cast<int>(tab[*p1].x >> 24) != ch) continue;
            if (prev >= 0 && (noise.m.next() >> 11) < a.noise_thr) {
              T* p0 = g.at(prev);
              const T x = *p0;
              *p0 = *p1;
              *p1 = x;
            }
            prev = pos;
          }
        }
      V ct[kMaxChannelsDev], sfx[kMaxChannelsDev];
#pragma unroll
      for (int ch = 0; ch < kMaxChannelsDev; ++ch) {
        ct[ch] = ch < nch ? static_cast<V>(a.ctot[w * nch + ch]) : V(0);
        sfx[ch] = 0;
      }
      V best = pw[0];
      for (int pos = R - 1; pos >= 0; --pos) {
        const uint2 e = tab[*g.at(pos)];
        const int ch = static_cast<int>(e.x >> 24);
        V c = 0;
#pragma unroll
        for (int k = 0; k < kMaxChannelsDev; ++k)
          if (k == ch) c = ct[k] - sfx[k];
        best = max(best, c + pw[e.x & 0xFFFFFFu]);
#pragma unroll
        for (int k = 0; k < kMaxChannelsDev; ++k)
          if (k == ch) sfx[k] += static_cast<V>(e.y);
      }
      const int64_t T0 = static_cast<int64_t>(best);
      st64(wsc, 5 * w, T0);
      int64_t dev = T0;
      // per channel: recvs starting before T0 ran back to back before the release
      for (int ch = 0; ch < nch; ++ch) {
        int64_t c = 0;
        int pos = 0, last = -1;
        for (; pos < R; ++pos) {
          const uint2 e = tab[*g.at(pos)];
          if (static_cast<int>(e.x >> 24) != ch) continue;
          if (c >= T0) break;
          c += static_cast<int64_t>(e.y);
          last = pos;
        }
        const int i = w * nch + ch;
        const bool busy = last >= 0 && c > T0;  // the channel's last started recv still runs at T0
        st64(csc, 4 * i, busy ? c : 0);
        w32(csc, 4 * i + 2) = busy ? -2 : -1;
        w32(csc, 4 * i + 3) = pos;  // next gate position to consider on this channel
        if (busy) dev = max(dev, c);
      }
      st64(wsc, 5 * w + 2, dev);
      w32(wsc, 5 * w + 4) = 0;
      mk = max(mk, dev);
      t = min(t, T0);
      for (int x = 0; x < q.sw; ++x) pend[static_cast<size_t>(w * q.sw + x) * NT] = 0;
    }
    for (int x = 0; x < Q; ++x) *qmiss.at(x) = q.ps_missing[x];
    for (int x = 0; x < q.qw; ++x) qready[static_cast<size_t>(x) * NT] = 0;
    for (int k = 0; k < nps; ++k) w32(ksc, 3 * k) = -1;
    MtStream choice;
    choice.init(seed);
    auto draw = [&](int n) -> int {  // bounded(n) of the shared choice stream
      if (n < 2) return 0;
      uint64_t v;
      do v = choice.next();
      while (v > s_lim[n]);
      return static_cast<int>(fastmod32(v, static_cast<uint32_t>(n), s_mag[n]));
    };
    auto ps_ready = [&](int x) {
      uint8_t* m = qmiss.at(x);
      if (--*m == 0) qready[static_cast<size_t>(x >> 5) * NT] |= 1u << (x & 31);
    };
    auto core_complete = [&](int k) {
      const int op = w32(ksc, 3 * k);
      w32(ksc, 3 * k) = -1;
      for (int e = q.ps_succ_off[op]; e < q.ps_succ_off[op + 1]; ++e) ps_ready(q.ps_succ[e]);
    };
    auto chan_complete = [&](int w, int i) {
      const int sid = w32(csc, 4 * i + 2);
      w32(csc, 4 * i + 2) = -1;
      if (sid < 0) return;  // a recv: nothing downstream after the release
      const int base = w * S + sid;
      for (int e = q.send_succ_off[base]; e < q.send_succ_off[base + 1]; ++e) ps_ready(q.send_succ[e]);
    };
    auto core_try = [&](int k) -> bool {
      if (w32(ksc, 3 * k) >= 0) return false;
      const uint32_t* cm = q.core_mask + static_cast<size_t>(k) * q.qw;
      int n = 0;
      for (int x = 0; x < q.qw; ++x) n += __popc(qready[static_cast<size_t>(x) * NT] & cm[x]);
      if (n == 0) return false;
      int j = draw(n);
      for (int x = 0;; ++x) {
        const uint32_t bits = qready[static_cast<size_t>(x) * NT] & cm[x];
        const int cnt = __popc(bits);
        if (j < cnt) {
          const int b = nth_bit(bits, j);
          qready[static_cast<size_t>(x) * NT] &= ~(1u << b);
          const int op = (x << 5) + b;
          w32(ksc, 3 * k) = op;
          const int64_t e = t + q.ps_d[op];
          st64(ksc, 3 * k + 1, e);
          mk = max(mk, e);
          return true;
        }
        j -= cnt;
      }
    };
    auto chan_try = [&](int w, int ch) -> bool {
      const int i = w * nch + ch;
      if (!w32(wsc, 5 * w + 4) || w32(csc, 4 * i + 2) != -1) return false;
      const Items<T, NT> g = gate(w);
      const uint2* tab = s_tab + w * R;
      int pos = w32(csc, 4 * i + 3);  // next recv of this channel in gate order
      while (pos < R && static_cast<int>(tab[*g.at(pos)].x >> 24) != ch) ++pos;
      w32(csc, 4 * i + 3) = pos;
      const int rc = pos < R ? static_cast<int>(*g.at(pos)) : -1;
      uint32_t* pw_ = pend + static_cast<size_t>(w * q.sw) * NT;
      const uint32_t* cm = q.ch_mask + static_cast<size_t>(ch) * q.sw;
      int ns = 0;
      for (int x = 0; x < q.sw; ++x) ns += __popc(pw_[static_cast<size_t>(x) * NT] & cm[x]);
      const int n = ns + (rc >= 0 ? 1 : 0);
      if (n == 0) return false;
      int j = draw(n);
      int64_t d;
      if (rc >= 0) {  // the recv's place among the candidates: this channel's pending sends before it
        const int sb = recv_sb[rc];
        int before = 0;
        for (int x = 0; x < (sb >> 5); ++x) before += __popc(pw_[static_cast<size_t>(x) * NT] & cm[x]);
        if (sb & 31) before += __popc(pw_[static_cast<size_t>(sb >> 5) * NT] & cm[sb >> 5] & ((1u << (sb & 31)) - 1u));
        if (j == before) {
          w32(csc, 4 * i + 2) = -2;
          w32(csc, 4 * i + 3) = pos + 1;
          d = static_cast<int64_t>(tab[rc].y);
          goto started;
        }
        if (j > before) --j;
      }
      for (int x = 0;; ++x) {
        const uint32_t bits = pw_[static_cast<size_t>(x) * NT] & cm[x];
        const int cnt = __popc(bits);
        if (j < cnt) {
          const int b = nth_bit(bits, j);
          pw_[static_cast<size_t>(x) * NT] &= ~(1u << b);
          const int sid = (x << 5) + b;
          w32(csc, 4 * i + 2) = sid;
          d = q.send_d[w * S + sid];
          break;
        }
        j -= cnt;
      }
    started:
      const int64_t e = t + d;
      st64(csc, 4 * i, e);
      if (e > ld64(wsc, 5 * w + 2)) st64(wsc, 5 * w + 2, e);
      mk = max(mk, e);
      return true;
    };
    auto complete_now = [&]() -> bool {  // every op ending at t (completions never draw)
      bool any = false;
      for (int k = 0; k < nps; ++k)
        if (w32(ksc, 3 * k) >= 0 && ld64(ksc, 3 * k + 1) == t) {
          core_complete(k);
          any = true;
        }
      for (int w = 0; w < W; ++w)
        for (int ch = 0; ch < nch; ++ch) {
          const int i = w * nch + ch;
          if (w32(csc, 4 * i + 2) != -1 && ld64(csc, 4 * i) == t) {
            chan_complete(w, i);
            any = true;
          }
        }
      return any;
    };
    // 2. the send phase: sim.cpp:194-233 over the PS cores and the released channels
    while (t != INT64_MAX) {
      for (int w = 0; w < W; ++w)  // last compute op done: the sends are ready
        if (!w32(wsc, 5 * w + 4) && ld64(wsc, 5 * w) == t) {
          w32(wsc, 5 * w + 4) = 1;
          uint32_t* pw_ = pend + static_cast<size_t>(w * q.sw) * NT;
          for (int x = 0; x < q.sw; ++x) {
            const int lo = x << 5;
            pw_[static_cast<size_t>(x) * NT] = S - lo >= 32 ? ~0u : ((1u << (S - lo)) - 1u);
          }
        }
      complete_now();
      bool progress = true;
      while (progress) {  // passes: try_start in resource order, then same-time completions
        progress = false;
        for (int si = 0; si < q.nslot; ++si) {
          const int sl = q.slots[si];
          if (sl < 0) progress = core_try(-1 - sl) || progress;
          else progress = chan_try(sl / nch, sl % nch) || progress;
        }
        progress = complete_now() || progress;
      }
      int64_t nt = INT64_MAX;
      for (int k = 0; k < nps; ++k)
        if (w32(ksc, 3 * k) >= 0) nt = min(nt, ld64(ksc, 3 * k + 1));
      for (int w = 0; w < W; ++w) {
        if (!w32(wsc, 5 * w + 4)) nt = min(nt, ld64(wsc, 5 * w));
        for (int ch = 0; ch < nch; ++ch) {
          const int i = w * nch + ch;
          if (w32(csc, 4 * i + 2) != -1) nt = min(nt, ld64(csc, 4 * i));
        }
      }
      t = nt;
    }
    int64_t hi = 0, lo = INT64_MAX;
    for (int w = 0; w < W; ++w) {
      const int64_t mw = ld64(wsc, 5 * w + 2);
      if (a.worker_ms) a.worker_ms[idx * W + w] = mw;
      hi = max(hi, mw);
      lo = min(lo, mw);
    }
    if (a.makespans) a.makespans[idx] = mk;
    acc.add(a, seed, mk, hi, lo, s_hist, s_shist);
  }
  acc.flush(a, s_hist, s_shist);
}

// ---- dag_pair_kernel: the same sweep with the positions/bins arrays shared
// by the kW warps of a block. A run is phase A (the shuffle, and the noise
// swaps, into the thread's own gate-order column: R bytes) and phase B
// (positions, the join program, the fold: R + L + 1 bytes of positions and
// slots and 4(R + 1) bytes of bins). Phase A is about three times phase B,
// so while one warp runs phase B on the block's single set of
// positions/bins columns (lane l uses column l) the others run phase A, and
// named barriers pass the columns round the warps in a fixed ring (barrier
// 1 + w: warp w - 1 hands them to warp w). Shared memory per thread drops
// from ~6R to ~R + 5R/kW bytes, which is what bounds occupancy here.

__host__ __device__ inline size_t dag_pair_smem(int R, int W, int nrec, int L, int nhist, size_t tb, size_t vb,
                                                int nwarps = 2) {
  const int per = tb == 1 ? 4 : 2;
  const size_t vbins = vb * (R + 1) * 32, vals = 4ull * ((R + L + 1 + per - 1) / per) * 32;
  const size_t perms = 4ull * ((R + per - 1) / per) * 32 * nwarps;
  return round16(dag_table_bytes(R, W, nrec, vb) + 4 * static_cast<size_t>(nhist) * kBins + vbins + vals + perms) + 16;
}

// named barriers between two warps (64 threads: one arrives, one waits)
__device__ __forceinline__ void named_sync(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id)); }
__device__ __forceinline__ void named_arrive(int id) { asm volatile("bar.arrive %0, 64;" ::"r"(id)); }

template <typename T, typename V, bool kNoisy, int kW>
__global__ void __launch_bounds__(32 * kW) dag_pair_kernel(ChainArgs a, DagArgs g) {
  constexpr int NT = 32 * kW;
  extern __shared__ __align__(16) unsigned char smem[];
  const int R = a.R, W = a.W, NR = g.nrec;
  const size_t vb = sizeof(V);
  const uint64_t* s_lim = reinterpret_cast<const uint64_t*>(smem);
  const uint64_t* s_mag = s_lim + (R + 2);
  const uint4* s_rec = reinterpret_cast<const uint4*>(s_mag + (R + 2));
  const DagEnt<V>* s_ent = reinterpret_cast<const DagEnt<V>*>(s_rec + NR);
  const V* s_wj = reinterpret_cast<const V*>(s_ent + W * R);
  const V* s_w0 = s_wj + W * NR;
  const int nhist = (a.do_e ? 1 : 0) + (a.cluster ? 1 : 0);
  int* s_hist = reinterpret_cast<int*>(smem + dag_table_bytes(R, W, NR, vb));
  int* s_shist = s_hist + (a.do_e ? kBins : 0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  V* s_bins = reinterpret_cast<V*>(s_hist + nhist * kBins) + lane;  // [k][32], shared by the pair
  uint32_t* vwords = reinterpret_cast<uint32_t*>(reinterpret_cast<V*>(s_hist + nhist * kBins) + (R + 1) * 32);
  const Items<T, 32> val{vwords + lane};
  uint32_t* pwords = vwords + Items<T, 32>::words(R + g.L + 1) * 32;
  const Items<T, NT> perm{pwords + threadIdx.x};
  uint64_t* tables_ready = reinterpret_cast<uint64_t*>(smem + a.mbar_off);
  if (threadIdx.x == 0) mbar_init(tables_ready, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(tables_ready, a.blob_bytes);
    bulk_g2s(smem, a.blob, a.blob_bytes, tables_ready);
  }
  for (int k = threadIdx.x; k < nhist * kBins; k += blockDim.x) s_hist[k] = 0;
  if (warp == 0)
    for (int k = 0; k <= R; ++k) s_bins[k * 32] = V(0);  // the fold re-zeroes every bin it reads
  mbar_wait(tables_ready, 0);
  __syncthreads();
  unsigned char* vcol = reinterpret_cast<unsigned char*>(val.base);

  StatAcc acc;
  const int64_t nthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
  // every thread of the block runs the same number of units (ordering x
  // worker: the count of the block's first thread), so the named barriers
  // always match; threads past the end only keep the handshake
  const int64_t first0 = static_cast<int64_t>(blockIdx.x) * blockDim.x;
  const int64_t n_ord = first0 < a.count ? (a.count - first0 + nthreads - 1) / nthreads : 0;
  const int64_t units = n_ord * W;
  const int64_t idx0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  int64_t hi = 0, lo = INT64_MAX;
  NoiseState<kNoisy> noise;
  auto phase_a = [&](int64_t u) {  // gate order of unit u into this thread's column
    const int64_t j = u / W;
    const int w = static_cast<int>(u % W);
    const int64_t idx = idx0 + j * nthreads;
    if (idx >= a.count) return;
    const uint64_t seed = a.seed_lo + static_cast<uint64_t>(idx);
    if constexpr (kNoisy)
      if (w == 0) noise.init(splitmix64(seed ^ kNoiseSalt));
    const uint64_t ws = a.cluster ? splitmix64(seed ^ (kPhi * static_cast<uint64_t>(w + 1))) : seed;
    FoldT<V> f{0, 0, 0};
    shuffle_fold<Items<T, NT>, V, true>(ws, R, perm, f, nullptr, V(0), nullptr, s_lim, s_mag);
    if constexpr (kNoisy) {
      auto swap_at = [&](int pos, uint64_t v) {
        if ((v >> 11) < a.noise_thr) {
          T* p0 = perm.at(pos - 1);
          T* p1 = perm.at(pos);
          const T x = *p0;
          *p0 = *p1;
          *p1 = x;
        }
      };
      if (W == 1 && R - 1 <= 311) {
        mt_outputs(splitmix64(seed ^ kNoiseSalt), R - 1, [&](int d, uint64_t v) { swap_at(d + 1, v); });
      } else {
        for (int pos = 1; pos < R; ++pos) swap_at(pos, noise.m.next());
      }
    }
  };
  auto phase_b = [&](int64_t u) {  // positions, program and fold of unit u
    const int64_t j = u / W;
    const int w = static_cast<int>(u % W);
    const int64_t idx = idx0 + j * nthreads;
    if (idx >= a.count) return;
    const DagEnt<V>* ent = s_ent + w * R;
    for (int k = 0; k < R; ++k) *val.at(*perm.at(k)) = static_cast<T>(k);
    {
      const V* wj = s_wj + w * NR;
      int accv = 0;
      for (int q = 0; q < NR; q += 4) {
        uint4 rc[4];
        V wt[4];
        int lp[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          rc[i] = s_rec[q + i];
          wt[i] = wj[q + i];
        }
        int x[4], y[4], z[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          x[i] = *reinterpret_cast<const T*>(vcol + (rc[i].x & kDagOffMask));
          y[i] = *reinterpret_cast<const T*>(vcol + rc[i].y);
          z[i] = *reinterpret_cast<const T*>(vcol + rc[i].z);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          lp[i] = max(max((rc[i].x & kDagAccFlag) ? accv : x[i], y[i]), z[i]);
          accv = (rc[i].w & kDagRealFlag) ? lp[i] : accv;
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) *reinterpret_cast<T*>(vcol + (rc[i].w & kDagOffMask)) = static_cast<T>(lp[i]);
#pragma unroll
        for (int jj = 1; jj < 4; ++jj)
#pragma unroll
          for (int i = 0; i < jj; ++i)
            if (lp[i] == lp[jj]) {
              wt[jj] += wt[i];
              wt[i] = V(0);
            }
        V old[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) old[i] = s_bins[lp[i] * 32];
#pragma unroll
        for (int i = 0; i < 4; ++i) s_bins[lp[i] * 32] = old[i] + wt[i];
      }
    }
    const V ctot = static_cast<V>(a.ctot[w]);
    V S = 0, suffix = 0, best = 0;
    auto step = [&](int r, int k) {
      const DagEnt<V> e = ent[r];
      S += s_bins[k * 32] + e.wr;
      s_bins[k * 32] = V(0);
      best = max(best, ctot - suffix + S);
      suffix += e.d;
    };
    int k = R - 1;
    if constexpr (sizeof(T) == 1) {
      for (; k >= 0 && (k & 3) != 3; --k) step(*perm.at(k), k);
      for (; k >= 3; k -= 4) {
        const uint32_t wd = perm.base[(k >> 2) * NT];
        step(wd >> 24, k);
        step((wd >> 16) & 0xFF, k - 1);
        step((wd >> 8) & 0xFF, k - 2);
        step(wd & 0xFF, k - 3);
      }
    } else {
      for (; k >= 0; --k) step(*perm.at(k), k);
    }
    best = max(best, S + s_w0[w]);
    const int64_t tcpu = static_cast<int64_t>(best);
    const int64_t c64 = static_cast<int64_t>(ctot);
    const int64_t mw = a.cluster ? max(tcpu, max(c64, tcpu) + a.send_tot[w]) : max(tcpu, c64);
    if (a.worker_ms) a.worker_ms[idx * W + w] = mw;
    hi = max(hi, mw);
    lo = min(lo, mw);
    if (w == W - 1) {
      if (a.makespans) a.makespans[idx] = hi;
      acc.add(a, a.seed_lo + static_cast<uint64_t>(idx), hi, hi, lo, s_hist, s_shist);
      hi = 0;
      lo = INT64_MAX;
    }
  };
  // phase B in a fixed ring: warp 0 B(0), warp 1 B(0), ..., warp kW-1 B(0),
  // warp 0 B(1), ...; barrier 1 + w hands the columns from warp w - 1 to w
  if constexpr (kW == 2) {  // (the two-warp form as straight-line code)
    for (int64_t u = 0; u < units; ++u) {
      phase_a(u);
      if (warp == 0) {
        if (u > 0) named_sync(2);
        phase_b(u);
        named_arrive(1);
      } else {
        named_sync(1);
        phase_b(u);
        named_arrive(2);
      }
    }
    if (warp == 0 && units > 0) named_sync(2);
  } else {
    const int next_bar = warp + 1 == kW ? 1 : warp + 2;
    for (int64_t u = 0; u < units; ++u) {
      phase_a(u);
      if (warp != 0 || u > 0) named_sync(1 + warp);
      phase_b(u);
      named_arrive(next_bar);
    }
    if (warp == 0 && units > 0) named_sync(1);  // consume the last warp's final hand-back
  }
  __syncthreads();
  acc.flush(a, s_hist, s_shist);
}

// Brute force (metrics.cpp:37-72) on the closed form: permutation number k
// in lexicographic order of the recv columns (std::next_permutation order
// over ascending ids) is unranked in the factorial number system into a
// per-thread shared-memory row, then folded right-to-left like a random
// order. out[k - first] = makespan.
template <typename V>
__global__ void __launch_bounds__(kSweepThreads) lex_kernel(ChainArgs a, int64_t first, int64_t count,
                                                            const unsigned long long* __restrict__ fact,
                                                            int64_t* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int R = a.R;
  uint2* s_tab = reinterpret_cast<uint2*>(smem);
  V* s_pw = reinterpret_cast<V*>(s_tab + R);
  uint8_t* s_row = reinterpret_cast<uint8_t*>(s_pw + a.stride) + threadIdx.x * 32;
  for (int k = threadIdx.x; k < R; k += blockDim.x) s_tab[k] = a.tab[k];
  for (int k = threadIdx.x; k < a.stride; k += blockDim.x) s_pw[k] = static_cast<V>(a.pwsuf[k]);
  __syncthreads();
  const V ctot = static_cast<V>(a.ctot[0]);
  const int64_t nthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < count; idx += nthreads) {
    unsigned long long k = static_cast<unsigned long long>(first + idx);
    uint32_t left = (R >= 32) ? ~0u : ((1u << R) - 1u);  // remaining columns (R <= 20)
    for (int pos = 0; pos < R; ++pos) {
      const unsigned long long f = fact[R - 1 - pos];
      const int q = static_cast<int>(k / f);
      k -= static_cast<unsigned long long>(q) * f;
      const int c = nth_bit(left, q);
      left &= ~(1u << c);
      s_row[pos] = static_cast<uint8_t>(c);
    }
    FoldT<V> fo{a.nc, 0, -1};
    for (int pos = R - 1; pos >= 0; --pos) fo.add(s_tab[s_row[pos]], ctot, s_pw);
    if (fo.G > 0) fo.best = max(fo.best, s_pw[0]);
    const int64_t tcpu = fo.best < 0 ? 0 : static_cast<int64_t>(fo.best);
    out[idx] = max(tcpu, static_cast<int64_t>(ctot));
  }
}

// Multi-process reduction of the statistics (one SUM all-reduce): pack this
// rank's words into its slots of a zeroed buffer — keys 0, 1, 4, 5 into
// slots [k*world + rank], words 2..2007 (keys zeroed) summed, the float sums'
// bit patterns into [kw + 2006 + 2*rank] — and unpack the reduced buffer.
__global__ void stats_pack_kernel(const unsigned long long* i64, const double* f64, int rank, int world,
                                  unsigned long long* buf) {
  const int kw = 4 * world, nw = kw + 2006 + 2 * world;
  for (int k = threadIdx.x; k < nw; k += blockDim.x) buf[k] = 0;
  __syncthreads();
  if (threadIdx.x < 4) {
    const int word[4] = {0, 1, 4, 5};
    buf[threadIdx.x * world + rank] = i64[word[threadIdx.x]];
  }
  for (int k = threadIdx.x; k < 2006; k += blockDim.x) {
    const int w = k + 2;
    buf[kw + k] = (w == 4 || w == 5) ? 0ULL : i64[w];
  }
  if (threadIdx.x < 2) buf[kw + 2006 + 2 * rank + threadIdx.x] = __double_as_longlong(f64[threadIdx.x]);
}
__global__ void stats_unpack_kernel(const unsigned long long* buf, int world, unsigned long long* i64,
                                    double* f64) {
  const int kw = 4 * world;
  for (int k = threadIdx.x; k < 2006; k += blockDim.x) i64[k + 2] = buf[kw + k];
  __syncthreads();
  if (threadIdx.x < 4) {
    const int word[4] = {0, 1, 4, 5};
    const bool is_min = threadIdx.x == 0 || threadIdx.x == 2;
    unsigned long long v = is_min ? ~0ULL : 0ULL;  // an idle rank's min key is all ones
    for (int r = 0; r < world; ++r) {
      const unsigned long long x = buf[threadIdx.x * world + r];
      v = is_min ? min(v, x) : max(v, x);
    }
    i64[word[threadIdx.x]] = v;
  }
  if (threadIdx.x < 2) {
    double acc = 0.0;  // rank order: deterministic
    for (int r = 0; r < world; ++r) acc += __longlong_as_double(buf[kw + 2006 + 2 * r + threadIdx.x]);
    f64[threadIdx.x] = acc;
  }
}

__global__ void reset_kernel(unsigned long long* i64, double* f64) {
  for (int k = threadIdx.x; k < 2008; k += blockDim.x) i64[k] = (k == 0 || k == 4) ? ~0ULL : 0ULL;
  if (threadIdx.x < 2) f64[threadIdx.x] = 0.0;
}

__global__ void random_orders_kernel(int R, int S, const uint64_t* __restrict__ seeds,
                                     const uint64_t* __restrict__ lim, const uint64_t* __restrict__ mag,
                                     int32_t* __restrict__ perms) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < S; s += gridDim.x * blockDim.x) {
    int32_t* p = perms + static_cast<int64_t>(s) * R;
    for (int k = 0; k < R; ++k) p[k] = k;
    // register cursors for the first 311 outputs, then a full state in
    // local memory continuing the same stream (linear in R)
    MtLazy lz;
    lz.init(seeds[s]);
    uint64_t st[312];
    MtFull full{st, 0};
    bool on_full = false;
    auto next = [&]() -> uint64_t {
      if (!on_full) {
        if (!lz.exhausted()) return lz.next_raw();
        full.seed(lz.seed);
        for (int k = 0; k < lz.i; ++k) full.next();
        on_full = true;
      }
      return full.next();
    };
    for (int i = R; i > 1; --i) {
      uint64_t v = next(), j;
      if (i < 4096) {
        while (v > lim[i]) v = next();
        j = fastmod(v, static_cast<uint64_t>(i), mag[i]);
      } else {
        const uint64_t n = static_cast<uint64_t>(i);
        const uint64_t limit = UINT64_MAX - (UINT64_MAX % n + 1) % n;
        while (v > limit) v = next();
        j = v % n;
      }
      const int32_t t = p[i - 1];
      p[i - 1] = p[j];
      p[j] = t;
    }
  }
}

}  // namespace
}  // namespace tictac_dev

using namespace tictac_dev;

struct SweepPlan {
  int W = 1, R = 0, nc = 0, cluster = 0, stride = 1, narrow = 0, nch = 1;
  int64_t U = 0, L = 0;
  void *tab = nullptr, *pwsuf = nullptr, *ctot = nullptr, *send = nullptr, *lim = nullptr, *mag = nullptr;
  void* blob = nullptr;  // shared-memory table image of the sweep kernels
  size_t blob_bytes = 0;
  size_t smem = 0, smem_orders = 0;
  int blocks = 0;
  uint64_t noise_thr = 0;
  // general-DAG plans (dag_sweep_kernel): program records, slots,
  // shared-memory item width (1: R <= 255, else 2)
  int dag = 0, J = 0, Ls = 0, tb = 1;
  int blocks_orders = 0;
  // dag_pair_kernel (random sweeps): its own image (records with offsets in
  // the 32-column layout), shared memory, grid
  void* pair_blob = nullptr;
  size_t pair_smem = 0;
  int pair_blocks = 0;
  int pair_warps = 4;  // warps sharing one phase-B set (TICTAC_DAG_WARPS: 2, 3, 4, 6)
  // cluster send phase (cluster_ps_kernel): device tables and its own image
  int ps = 0, ps_blocks = 0;
  PsArgs psa{};
  void* ps_blob = nullptr;
  size_t ps_blob_bytes = 0, ps_smem = 0;
  std::vector<void*> ps_bufs;
  size_t uploaded = 0;  // host->device bytes copied when the plan was built
};

using DagFn = void (*)(ChainArgs, DagArgs);
template <int kW>
static DagFn pair_fn_w(const SweepPlan* p) {
  const bool nz = p->noise_thr != 0;
  if (p->tb == 1) {
    if (nz) return p->narrow ? dag_pair_kernel<uint8_t, int32_t, true, kW> : dag_pair_kernel<uint8_t, int64_t, true, kW>;
    return p->narrow ? dag_pair_kernel<uint8_t, int32_t, false, kW> : dag_pair_kernel<uint8_t, int64_t, false, kW>;
  }
  if (nz) return p->narrow ? dag_pair_kernel<uint16_t, int32_t, true, kW> : dag_pair_kernel<uint16_t, int64_t, true, kW>;
  return p->narrow ? dag_pair_kernel<uint16_t, int32_t, false, kW> : dag_pair_kernel<uint16_t, int64_t, false, kW>;
}
static DagFn pair_fn(const SweepPlan* p) {
  switch (p->pair_warps) {
    case 2: return pair_fn_w<2>(p);
    case 3: return pair_fn_w<3>(p);
    case 6: return pair_fn_w<6>(p);
    default: return pair_fn_w<4>(p);
  }
}
template <int kSrc>
static DagFn dag_fn(const SweepPlan* p, bool noisy) {
  if (kSrc == 0 && noisy) {
    if (p->tb == 1)
      return p->narrow ? dag_sweep_kernel<uint8_t, int32_t, true, 0> : dag_sweep_kernel<uint8_t, int64_t, true, 0>;
    return p->narrow ? dag_sweep_kernel<uint16_t, int32_t, true, 0> : dag_sweep_kernel<uint16_t, int64_t, true, 0>;
  }
  if (p->tb == 1)
    return p->narrow ? dag_sweep_kernel<uint8_t, int32_t, false, kSrc> : dag_sweep_kernel<uint8_t, int64_t, false, kSrc>;
  return p->narrow ? dag_sweep_kernel<uint16_t, int32_t, false, kSrc> : dag_sweep_kernel<uint16_t, int64_t, false, kSrc>;
}

using SweepFn = void (*)(ChainArgs);
static SweepFn sweep_fn(const SweepPlan* p) {
  if (p->nch > 1) {
    const bool nz = p->noise_thr != 0;
    if (p->R <= 256) {
      if (nz) return p->narrow ? chain_multi_kernel<uint8_t, int32_t, true> : chain_multi_kernel<uint8_t, int64_t, true>;
      return p->narrow ? chain_multi_kernel<uint8_t, int32_t, false> : chain_multi_kernel<uint8_t, int64_t, false>;
    }
    if (nz) return p->narrow ? chain_multi_kernel<uint16_t, int32_t, true> : chain_multi_kernel<uint16_t, int64_t, true>;
    return p->narrow ? chain_multi_kernel<uint16_t, int32_t, false> : chain_multi_kernel<uint16_t, int64_t, false>;
  }
  if (p->noise_thr) {
    if (p->R <= 256)
      return p->narrow ? chain_sweep_kernel<uint8_t, false, int32_t, true>
                       : chain_sweep_kernel<uint8_t, false, int64_t, true>;
    return p->narrow ? chain_sweep_kernel<uint16_t, false, int32_t, true>
                     : chain_sweep_kernel<uint16_t, false, int64_t, true>;
  }
  if (p->R <= 256)
    return p->narrow ? chain_sweep_kernel<uint8_t, false, int32_t> : chain_sweep_kernel<uint8_t, false, int64_t>;
  return p->narrow ? chain_sweep_kernel<uint16_t, false, int32_t> : chain_sweep_kernel<uint16_t, false, int64_t>;
}

extern "C" SweepPlan* csk_sweep_plan(int32_t W, int32_t R, int32_t nc, const int64_t* d,
                                     const int32_t* first, const int64_t* pwsuf, int32_t nch,
                                     const int32_t* chan, const int64_t* send_total, int cluster, int64_t U,
                                     int64_t L, uint64_t noise_thr, char* err) {
  if (ensure_device(err)) return nullptr;
  if (nch < 1 || nch > kMaxChannelsDev || nc >= (1 << 24)) {
    std::snprintf(err, 256, "sweep plan: unsupported channel or class count");
    return nullptr;
  }
  auto* p = new SweepPlan();
  p->nch = nch;
  p->noise_thr = noise_thr;
  p->W = W;
  p->R = R;
  p->nc = nc;
  p->cluster = cluster;
  p->stride = nc + 1;
  p->U = U;
  p->L = L;
  std::vector<uint2> tab(static_cast<size_t>(W) * R);
  std::vector<int64_t> ctot(static_cast<size_t>(W) * nch, 0);
  for (int w = 0; w < W; ++w)
    for (int c = 0; c < R; ++c) {
      const int ch = nch > 1 ? chan[w * R + c] : 0;
      tab[w * R + c] = make_uint2(static_cast<unsigned>(first[w * R + c]) | (static_cast<unsigned>(ch) << 24),
                                  static_cast<unsigned>(d[w * R + c]));
      ctot[w * nch + ch] += d[w * R + c];
    }
  std::vector<uint64_t> lim(R + 2), mag(R + 2);
  for (int n = 0; n <= R + 1; ++n) bounded_consts(static_cast<uint64_t>(n), &lim[n], &mag[n]);
  auto up = [&](void** dst, const void* src, size_t bytes) {
    if (cudaMalloc(dst, bytes ? bytes : 8) != cudaSuccess) return false;
    p->uploaded += bytes;
    return bytes == 0 || cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice) == cudaSuccess;
  };
  if (!up(&p->tab, tab.data(), tab.size() * sizeof(uint2)) ||
      !up(&p->pwsuf, pwsuf, sizeof(int64_t) * W * p->stride) ||
      !up(&p->ctot, ctot.data(), sizeof(int64_t) * W * nch) ||
      !up(&p->send, send_total, sizeof(int64_t) * W * nch) ||
      !up(&p->lim, lim.data(), sizeof(uint64_t) * lim.size()) ||
      !up(&p->mag, mag.data(), sizeof(uint64_t) * mag.size())) {
    std::snprintf(err, 256, "CUDA allocation for the sweep plan failed");
    csk_sweep_plan_free(p);
    return nullptr;
  }
  // 32-bit fold when every prefix/suffix time sum fits (U bounds them all)
  p->narrow = U < (int64_t{1} << 31) ? 1 : 0;
  {  // the sweep kernels' shared-memory table image, built once per plan
    const size_t vb = p->narrow ? 4 : 8;
    p->blob_bytes = sweep_table_bytes(R, W, p->stride, vb);
    std::vector<unsigned char> img(p->blob_bytes, 0);
    unsigned char* q = img.data();
    std::memcpy(q, lim.data(), 8ull * (R + 2));
    std::memcpy(q + 8ull * (R + 2), mag.data(), 8ull * (R + 2));
    std::memcpy(q + 16ull * (R + 2), tab.data(), 8ull * W * R);
    unsigned char* pwq = q + 16ull * (R + 2) + 8ull * W * R;
    for (int k = 0; k < W * p->stride; ++k) {
      if (p->narrow) {
        const int32_t v = static_cast<int32_t>(pwsuf[k]);
        std::memcpy(pwq + 4ull * k, &v, 4);
      } else {
        std::memcpy(pwq + 8ull * k, &pwsuf[k], 8);
      }
    }
    if (!up(&p->blob, img.data(), img.size())) {
      std::snprintf(err, 256, "CUDA allocation for the sweep plan failed");
      csk_sweep_plan_free(p);
      return nullptr;
    }
  }
  const int nhist = (U != L ? 1 : 0) + (cluster ? 1 : 0);
  p->smem = sweep_smem(R, W, p->stride, nhist, p->narrow ? 4 : 8);
  p->smem_orders = sweep_smem(R, W, p->stride, nhist, 8);
  int dev = 0, sms = 148, occ = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const void* fn = reinterpret_cast<const void*>(sweep_fn(p));
  allow_max_dynamic_smem(fn);
  allow_max_dynamic_smem(reinterpret_cast<const void*>(chain_sweep_kernel<uint8_t, true, int64_t>));
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kSweepThreads, p->smem);
  if (occ < 1) {
    std::snprintf(err, 256, "sweep plan needs %zu bytes of shared memory per block", p->smem);
    csk_sweep_plan_free(p);
    return nullptr;
  }
  p->blocks = sms * occ;
  return p;
}

extern "C" SweepPlan* csk_sweep_plan_dag(int32_t W, int32_t R, const int64_t* d, const int64_t* wr, int32_t nrec,
                                         const int32_t* recs, const int64_t* wj, const int64_t* w0, int32_t Ls,
                                         const int64_t* send_total, int cluster, int64_t U, int64_t L,
                                         uint64_t noise_thr, char* err) {
  if (ensure_device(err)) return nullptr;
  if (nrec % 4) {
    std::snprintf(err, 256, "DAG program records must come in groups of four");
    return nullptr;
  }
  auto* p = new SweepPlan();
  p->dag = 1;
  p->noise_thr = noise_thr;
  p->W = W;
  p->R = R;
  p->J = nrec;
  p->Ls = Ls;
  p->cluster = cluster;
  p->U = U;
  p->L = L;
  p->tb = R <= 255 ? 1 : 2;
  p->narrow = U < (int64_t{1} << 31) ? 1 : 0;
  std::vector<int64_t> ctot(W, 0);
  for (int w = 0; w < W; ++w)
    for (int c = 0; c < R; ++c) ctot[w] += d[w * R + c];
  std::vector<uint64_t> lim(R + 2), mag(R + 2);
  for (int n = 0; n <= R + 1; ++n) bounded_consts(static_cast<uint64_t>(n), &lim[n], &mag[n]);
  const size_t vb = p->narrow ? 4 : 8;
  p->blob_bytes = dag_table_bytes(R, W, nrec, vb);
  std::vector<unsigned char> img(p->blob_bytes, 0);
  unsigned char* q = img.data();
  auto put = [&](int64_t v) {  // one value in the fold's width
    if (p->narrow) {
      const int32_t x = static_cast<int32_t>(v);
      std::memcpy(q, &x, 4);
    } else {
      std::memcpy(q, &v, 8);
    }
    q += vb;
  };
  std::memcpy(q, lim.data(), 8ull * (R + 2));
  q += 8ull * (R + 2);
  std::memcpy(q, mag.data(), 8ull * (R + 2));
  q += 8ull * (R + 2);
  const int discard = R + Ls;  // value index of the discard slot
  for (int r = 0; r < nrec; ++r) {
    const bool pad = recs[4 * r + 3] == -3;
    for (int f = 0; f < 4; ++f) {
      const int v = recs[4 * r + f];
      uint32_t off;
      if (v == -2 && f == 0) {
        off = kDagAccFlag;  // forwarded: the previous record's result
      } else if (pad) {
        off = f == 3 ? dag_item_off(discard, p->tb) : 0;
      } else if (f == 3) {
        off = dag_item_off(v < 0 ? discard : v, p->tb) | kDagRealFlag;
      } else if (v >= 0 && v < discard) {
        off = dag_item_off(v, p->tb);
      } else {
        std::snprintf(err, 256, "DAG program value index out of range");
        delete p;
        return nullptr;
      }
      std::memcpy(q, &off, 4);
      q += 4;
    }
  }
  for (int k = 0; k < W * R; ++k) {
    put(d[k]);
    put(wr[k]);
  }
  for (int k = 0; k < W * nrec; ++k) put(wj[k]);
  for (int w = 0; w < W; ++w) put(w0[w]);
  // the pair kernel's image: the same bytes with the records' offsets in
  // the 32-column layout of its shared positions array
  std::vector<unsigned char> pimg = img;
  {
    unsigned char* rq = pimg.data() + 16ull * (R + 2);
    for (int r = 0; r < nrec; ++r) {
      const bool pad = recs[4 * r + 3] == -3;
      for (int f = 0; f < 4; ++f) {
        const int v = recs[4 * r + f];
        uint32_t off;
        if (v == -2 && f == 0) off = kDagAccFlag;
        else if (pad) off = f == 3 ? dag_item_off(discard, p->tb, 32) : 0;
        else if (f == 3) off = dag_item_off(v < 0 ? discard : v, p->tb, 32) | kDagRealFlag;
        else off = dag_item_off(v, p->tb, 32);
        std::memcpy(rq, &off, 4);
        rq += 4;
      }
    }
  }
  auto up = [&](void** dst, const void* src, size_t bytes) {
    if (cudaMalloc(dst, bytes ? bytes : 8) != cudaSuccess) return false;
    p->uploaded += bytes;
    return bytes == 0 || cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice) == cudaSuccess;
  };
  if (!up(&p->blob, img.data(), img.size()) || !up(&p->pair_blob, pimg.data(), pimg.size()) ||
      !up(&p->ctot, ctot.data(), sizeof(int64_t) * W) || !up(&p->send, send_total, sizeof(int64_t) * W)) {
    std::snprintf(err, 256, "CUDA allocation for the sweep plan failed");
    csk_sweep_plan_free(p);
    return nullptr;
  }
  const int nhist = (U != L ? 1 : 0) + (cluster ? 1 : 0);
  p->smem = dag_smem(R, W, nrec, Ls, nhist, p->tb, vb);
  p->smem_orders = dag_smem(R, W, nrec, Ls, 0, p->tb, vb);
  int dev = 0, sms = 148, occ = 0, occ_o = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const void* fns[] = {reinterpret_cast<const void*>(dag_fn<0>(p, noise_thr != 0)),
                       reinterpret_cast<const void*>(dag_fn<1>(p, false)),
                       reinterpret_cast<const void*>(dag_fn<2>(p, false))};
  for (const void* fn : fns) allow_max_dynamic_smem(fn);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fns[0], kDagThreads, p->smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_o, fns[1], kDagThreads, p->smem_orders);
  if (occ < 1 || occ_o < 1) {
    std::snprintf(err, 256, "DAG sweep plan needs %zu bytes of shared memory per block", p->smem);
    csk_sweep_plan_free(p);
    return nullptr;
  }
  p->blocks = sms * occ;
  p->blocks_orders = sms * occ_o;
  {  // the shared-phase-B kernel for random sweeps, when it fits
    auto occupancy = [&](int w, size_t* smem_out) {
      p->pair_warps = w;
      *smem_out = dag_pair_smem(R, W, nrec, Ls, nhist, p->tb, vb, w);
      const void* pf = reinterpret_cast<const void*>(pair_fn(p));
      allow_max_dynamic_smem(pf);
      int occ = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, pf, 32 * w, *smem_out) != cudaSuccess) {
        cudaGetLastError();
        occ = 0;
      }
      return occ;
    };
    // two warps per phase-B set unless four of them fit half again as many
    // warps per SM (measured: phase B serialises beyond two per set unless
    // occupancy grows that much: branchy Inception 0.62 -> 0.72 G with four,
    // branchy ResNet-101 slower with four than two)
    size_t smem2 = 0, smem4 = 0;
    const int occ4 = occupancy(4, &smem4), occ2 = occupancy(2, &smem2);
    int w = 4 * occ4 * 2 >= 3 * (2 * occ2) && occ4 > 0 ? 4 : 2;
    if (const char* e = std::getenv("TICTAC_DAG_WARPS")) {
      const int f = std::atoi(e);
      if (f == 2 || f == 3 || f == 4 || f == 6) w = f;
    }
    size_t sm = 0;
    const int occ = occupancy(w, &sm);
    p->pair_smem = sm;
    p->pair_blocks = std::getenv("TICTAC_DAG_NO_PAIR") ? 0 : sms * occ;
  }
  return p;
}

using PsFn = void (*)(ChainArgs, PsArgs);
static PsFn ps_fn(const SweepPlan* p) {
  const bool noisy = p->noise_thr != 0;
  if (p->R <= 256) {
    if (noisy) return p->narrow ? cluster_ps_kernel<uint8_t, int32_t, true> : cluster_ps_kernel<uint8_t, int64_t, true>;
    return p->narrow ? cluster_ps_kernel<uint8_t, int32_t, false> : cluster_ps_kernel<uint8_t, int64_t, false>;
  }
  if (noisy) return p->narrow ? cluster_ps_kernel<uint16_t, int32_t, true> : cluster_ps_kernel<uint16_t, int64_t, true>;
  return p->narrow ? cluster_ps_kernel<uint16_t, int32_t, false> : cluster_ps_kernel<uint16_t, int64_t, false>;
}

extern "C" int csk_sweep_plan_add_ps(SweepPlan* p, int32_t S, const int16_t* recv_sb, const uint32_t* ch_mask,
                                     const int64_t* send_d, const int32_t* send_succ_off, const int16_t* send_succ,
                                     int32_t Q, const int64_t* ps_d, const uint8_t* ps_missing,
                                     const int32_t* ps_succ_off, const int16_t* ps_succ, int32_t nps,
                                     const uint32_t* core_mask, int32_t nslot, const int32_t* slots, char* err) {
  if (p->dag || !p->cluster) {
    std::snprintf(err, 256, "the send phase extends cluster chain plans only");
    return 4;
  }
  const int W = p->W, R = p->R;
  auto up = [&](const void* src, size_t bytes) -> void* {
    void* d = nullptr;
    if (cudaMalloc(&d, bytes ? bytes : 8) != cudaSuccess) return nullptr;
    p->ps_bufs.push_back(d);
    p->uploaded += bytes;
    if (bytes && cudaMemcpy(d, src, bytes, cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
    return d;
  };
  PsArgs& a = p->psa;
  a.S = S;
  a.Q = Q;
  a.nps = nps;
  a.nslot = nslot;
  a.sw = (S + 31) / 32;
  a.qw = (Q + 31) / 32;
  const int32_t nss = send_succ_off[W * S], nqs = ps_succ_off[Q];
  a.recv_sb = static_cast<const int16_t*>(up(recv_sb, 2ull * R));
  a.ch_mask = static_cast<const uint32_t*>(up(ch_mask, 4ull * p->nch * a.sw));
  a.send_d = static_cast<const int64_t*>(up(send_d, 8ull * W * S));
  a.send_succ_off = static_cast<const int32_t*>(up(send_succ_off, 4ull * (W * S + 1)));
  a.send_succ = static_cast<const int16_t*>(up(send_succ, 2ull * nss));
  a.ps_d = static_cast<const int64_t*>(up(ps_d, 8ull * Q));
  a.ps_missing = static_cast<const uint8_t*>(up(ps_missing, static_cast<size_t>(Q)));
  a.ps_succ_off = static_cast<const int32_t*>(up(ps_succ_off, 4ull * (Q + 1)));
  a.ps_succ = static_cast<const int16_t*>(up(ps_succ, 2ull * nqs));
  a.core_mask = static_cast<const uint32_t*>(up(core_mask, 4ull * nps * a.qw));
  a.slots = static_cast<const int32_t*>(up(slots, 4ull * nslot));
  for (void* x : p->ps_bufs)
    if (!x) {
      std::snprintf(err, 256, "CUDA allocation for the send-phase tables failed");
      return 1;
    }
  // shared-memory image: bounded() constants (n < nk), the chain tables
  const int nk = std::max(S + 2, Q + 1) + 1;
  const size_t vb = p->narrow ? 4 : 8;
  std::vector<uint64_t> lim(nk), mag(nk);
  for (int n = 0; n < nk; ++n) bounded_consts(static_cast<uint64_t>(n), &lim[n], &mag[n]);
  std::vector<uint2> tab(static_cast<size_t>(W) * R);
  std::vector<int64_t> pw(static_cast<size_t>(W) * p->stride);
  if (cudaMemcpy(tab.data(), p->tab, 8ull * W * R, cudaMemcpyDeviceToHost) != cudaSuccess ||
      cudaMemcpy(pw.data(), p->pwsuf, 8ull * W * p->stride, cudaMemcpyDeviceToHost) != cudaSuccess) {
    std::snprintf(err, 256, "CUDA copy of the chain tables failed");
    return 1;
  }
  p->ps_blob_bytes = round16(16ull * nk + 8ull * W * R + vb * W * p->stride);
  std::vector<unsigned char> img(p->ps_blob_bytes, 0);
  unsigned char* q = img.data();
  std::memcpy(q, lim.data(), 8ull * nk);
  std::memcpy(q + 8ull * nk, mag.data(), 8ull * nk);
  std::memcpy(q + 16ull * nk, tab.data(), 8ull * W * R);
  unsigned char* pq = q + 16ull * nk + 8ull * W * R;
  for (size_t k = 0; k < pw.size(); ++k) {
    if (p->narrow) {
      const int32_t v = static_cast<int32_t>(pw[k]);
      std::memcpy(pq + 4 * k, &v, 4);
    } else {
      std::memcpy(pq + 8 * k, &pw[k], 8);
    }
  }
  p->ps_blob = up(img.data(), img.size());
  if (!p->ps_blob) {
    std::snprintf(err, 256, "CUDA allocation for the send-phase image failed");
    return 1;
  }
  const int nhist = (p->U != p->L ? 1 : 0) + 1;
  p->ps_smem = round16(p->ps_blob_bytes + 4ull * nhist * kBins +
                       kPsThreads * ps_thread_bytes(W, R, S, Q, p->nch, nps, R <= 256 ? 1 : 2)) + 16;
  int dev = 0, sms = 148, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const void* fn = reinterpret_cast<const void*>(ps_fn(p));
  allow_max_dynamic_smem(fn);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kPsThreads, p->ps_smem);
  if (occ < 1) {
    std::snprintf(err, 256, "send-phase plan needs %zu bytes of shared memory per block", p->ps_smem);
    return 1;
  }
  p->ps_blocks = sms * occ;
  p->ps = 1;
  return 0;
}

extern "C" int64_t csk_sweep_plan_uploaded(const SweepPlan* p) { return static_cast<int64_t>(p->uploaded); }

extern "C" const char* csk_sweep_plan_kernel(const SweepPlan* p) {
  if (p->ps) return "cluster_ps_kernel";
  if (p->dag) return p->pair_blocks > 0 ? "dag_pair_kernel" : "dag_sweep_kernel";
  return p->nch > 1 ? "chain_multi_kernel" : "chain_sweep_kernel";
}

extern "C" void csk_sweep_plan_free(SweepPlan* p) {
  if (!p) return;
  void* ptrs[] = {p->tab, p->pwsuf, p->ctot, p->send, p->lim, p->mag, p->blob, p->pair_blob};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  for (void* q : p->ps_bufs)
    if (q) cudaFree(q);
  delete p;
}

extern "C" int csk_stats_pack(const int64_t* d_i64, const double* d_f64, int rank, int world, int64_t* d_buf,
                              void* stream, char* err) {
  stats_pack_kernel<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const unsigned long long*>(d_i64), d_f64, rank, world,
      reinterpret_cast<unsigned long long*>(d_buf));
  LAUNCHED();
  CK(cudaGetLastError());
  return 0;
}

extern "C" int csk_stats_unpack(const int64_t* d_buf, int world, int64_t* d_i64, double* d_f64, void* stream,
                                char* err) {
  stats_unpack_kernel<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const unsigned long long*>(d_buf), world, reinterpret_cast<unsigned long long*>(d_i64),
      d_f64);
  LAUNCHED();
  CK(cudaGetLastError());
  return 0;
}

extern "C" int csk_sweep_reset(SweepPlan*, void* stream, int64_t* d_i64, double* d_f64, char* err) {
  reset_kernel<<<1, 1024, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<unsigned long long*>(d_i64), d_f64);
  LAUNCHED();
  CK(cudaGetLastError());
  return 0;
}

static ChainArgs chain_args(SweepPlan* p) {
  ChainArgs a{};
  a.W = p->W;
  a.R = p->R;
  a.stride = p->stride;
  a.nc = p->nc;
  a.nch = p->nch;
  a.tab = static_cast<const uint2*>(p->tab);
  a.pwsuf = static_cast<const int64_t*>(p->pwsuf);
  a.ctot = static_cast<const int64_t*>(p->ctot);
  a.send_tot = static_cast<const int64_t*>(p->send);
  a.cluster = p->cluster;
  a.lim = static_cast<const uint64_t*>(p->lim);
  a.mag = static_cast<const uint64_t*>(p->mag);
  a.U = p->U;
  a.L = p->L;
  a.do_e = p->U != p->L;
  a.key_bits = csk_key_bits(p->U);
  a.noise_thr = p->noise_thr;
  a.force_slow = std::getenv("TICTAC_SWEEP_FORCE_SLOW") != nullptr;
  a.blob = nullptr;  // per-element staging unless the caller's kernel matches the image
  a.blob_bytes = 0;
  return a;
}

extern "C" int csk_sweep_run(SweepPlan* p, uint64_t seed_lo, int64_t count, uint64_t key_base,
                             void* stream, int64_t* d_makespans, int64_t* d_worker_makespans,
                             int64_t* d_i64, double* d_f64, char* err) {
  if (count <= 0) return 0;
  ChainArgs a = chain_args(p);
  a.seed_lo = seed_lo;
  a.key_base = key_base;
  a.count = count;
  a.makespans = d_makespans;
  a.worker_ms = d_worker_makespans;
  a.i64 = reinterpret_cast<unsigned long long*>(d_i64);
  a.f64 = d_f64;
  if (!std::getenv("TICTAC_SWEEP_NO_BULK") || p->nch > 1) {  // sweep_fn(p) folds in the image's width
    a.blob = p->blob;
    a.blob_bytes = static_cast<uint32_t>(p->blob_bytes);
    a.mbar_off = static_cast<uint32_t>(p->smem - 16);
  }
  auto st = static_cast<cudaStream_t>(stream);
  if (p->ps) {
    a.blob = p->ps_blob;
    a.blob_bytes = static_cast<uint32_t>(p->ps_blob_bytes);
    a.mbar_off = static_cast<uint32_t>(p->ps_smem - 16);
    const int64_t need = (count + kPsThreads - 1) / kPsThreads;
    const int blocks = static_cast<int>(std::min<int64_t>(p->ps_blocks, need));
    ps_fn(p)<<<blocks, kPsThreads, p->ps_smem, st>>>(a, p->psa);
    LAUNCHED();
    CK(cudaGetLastError());
    return 0;
  }
  if (p->dag && p->pair_blocks > 0) {
    a.blob = p->pair_blob;
    a.blob_bytes = static_cast<uint32_t>(p->blob_bytes);
    a.mbar_off = static_cast<uint32_t>(p->pair_smem - 16);
    const int nt = 32 * p->pair_warps;
    const int64_t need = (count + nt - 1) / nt;
    const int blocks = static_cast<int>(std::min<int64_t>(p->pair_blocks, need));
    pair_fn(p)<<<blocks, nt, p->pair_smem, st>>>(a, DagArgs{p->J, p->Ls, 0, nullptr});
    LAUNCHED();
    CK(cudaGetLastError());
    return 0;
  }
  if (p->dag) {
    a.blob = p->blob;
    a.blob_bytes = static_cast<uint32_t>(p->blob_bytes);
    a.mbar_off = static_cast<uint32_t>(p->smem - 16);
    const int64_t need = (count + kDagThreads - 1) / kDagThreads;
    const int blocks = static_cast<int>(std::min<int64_t>(p->blocks, need));
    dag_fn<0>(p, p->noise_thr != 0)<<<blocks, kDagThreads, p->smem, st>>>(a, DagArgs{p->J, p->Ls, 0, nullptr});
    LAUNCHED();
    CK(cudaGetLastError());
    return 0;
  }
  const int64_t need = (count + kSweepThreads - 1) / kSweepThreads;
  const int blocks = static_cast<int>(std::min<int64_t>(p->blocks, need));
  sweep_fn(p)<<<blocks, kSweepThreads, p->smem, st>>>(a);
  LAUNCHED();
  CK(cudaGetLastError());
  return 0;
}

extern "C" int csk_sweep_orders(SweepPlan* p, const int32_t* d_orders, int64_t n, void* stream,
                                int64_t* d_makespans, char* err) {
  if (p->W != 1 || p->nch != 1) {
    std::snprintf(err, 256, "explicit orders need a worker graph plan");
    return 4;
  }
  if (n <= 0) return 0;
  auto st = static_cast<cudaStream_t>(stream);
  ChainArgs a = chain_args(p);
  a.count = n;
  a.orders = d_orders;
  a.makespans = d_makespans;
  a.i64 = nullptr;  // per-order makespans only, no statistics
  a.f64 = nullptr;
  a.do_e = 0;
  DevMem d_bad;
  CK(cudaMallocAsync(&d_bad.p, sizeof(int), 0));
  CK(cudaMemsetAsync(d_bad.p, 0, sizeof(int), st));
  a.bad_order = d_bad.as<int>();
  if (p->dag) {
    a.blob = p->blob;
    a.blob_bytes = static_cast<uint32_t>(p->blob_bytes);
    a.mbar_off = static_cast<uint32_t>(p->smem_orders - 16);
    a.cluster = 0;
    const int blocks = static_cast<int>(std::min<int64_t>(p->blocks_orders, (n + kDagThreads - 1) / kDagThreads));
    dag_fn<1>(p, false)<<<blocks, kDagThreads, p->smem_orders, st>>>(a, DagArgs{p->J, p->Ls, 0, nullptr});
  } else {
    const int blocks = static_cast<int>(std::min<int64_t>(p->blocks, (n + kSweepThreads - 1) / kSweepThreads));
    chain_sweep_kernel<uint8_t, true, int64_t><<<blocks, kSweepThreads, p->smem_orders, st>>>(a);
  }
  LAUNCHED();
  CK(cudaGetLastError());
  int bad = 0;
  CK(cudaMemcpyAsync(&bad, d_bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (bad) {
    std::snprintf(err, 256, "%s",
                  (bad & 1) ? "order entry out of range" : "order rows must be permutations of the recv columns");
    return 4;
  }
  return 0;
}

extern "C" int csk_sweep_lex(SweepPlan* p, int64_t first, int64_t count, int64_t* d_out, char* err) {
  if (p->W != 1 || p->cluster || p->R > 20 || p->nch != 1) {
    std::snprintf(err, 256, "lexicographic brute force needs a worker plan with at most 20 recvs");
    return 4;
  }
  if (count <= 0) return 0;
  std::vector<unsigned long long> fact(21, 1);
  for (int i = 1; i <= 20; ++i) fact[i] = fact[i - 1] * static_cast<unsigned long long>(i);
  DevMem d_fact;
  CK(cudaMallocAsync(&d_fact.p, sizeof(unsigned long long) * fact.size(), 0));
  CK(cudaMemcpy(d_fact.p, fact.data(), sizeof(unsigned long long) * fact.size(), cudaMemcpyHostToDevice));
  ChainArgs a = chain_args(p);
  if (p->dag) {
    a.blob = p->blob;
    a.blob_bytes = static_cast<uint32_t>(p->blob_bytes);
    a.mbar_off = static_cast<uint32_t>(p->smem_orders - 16);
    a.do_e = 0;
    a.cluster = 0;
    a.count = count;
    a.makespans = d_out;
    a.i64 = nullptr;
    a.f64 = nullptr;
    const int blocks = static_cast<int>(std::min<int64_t>(p->blocks_orders, (count + kDagThreads - 1) / kDagThreads));
    dag_fn<2>(p, false)<<<blocks, kDagThreads, p->smem_orders>>>(a, DagArgs{p->J, p->Ls, first,
                                                                   d_fact.as<const unsigned long long>()});
    LAUNCHED();
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    return 0;
  }
  const size_t vb = p->narrow ? 4 : 8;
  const size_t smem = 8 * static_cast<size_t>(p->R) + ((vb * p->stride + 7) & ~size_t(7)) + 32 * kSweepThreads;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int blocks = static_cast<int>(std::min<int64_t>(sms * 8, (count + kSweepThreads - 1) / kSweepThreads));
  const auto* f = d_fact.as<const unsigned long long>();
  if (p->narrow) {
    CK(allow_max_dynamic_smem(reinterpret_cast<const void*>(lex_kernel<int32_t>)));
    lex_kernel<int32_t><<<blocks, kSweepThreads, smem>>>(a, first, count, f, d_out);
  } else {
    CK(allow_max_dynamic_smem(reinterpret_cast<const void*>(lex_kernel<int64_t>)));
    lex_kernel<int64_t><<<blocks, kSweepThreads, smem>>>(a, first, count, f, d_out);
  }
  LAUNCHED();
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  return 0;
}

extern "C" int csk_brute_force_closed(SweepPlan* p, int64_t perms, int64_t* best_m, int64_t* best_k,
                                      int64_t* distinct, int64_t cap, int64_t* n_distinct, char* err) {
  // Chunks of <= 2^26 permutations in lexicographic order: makespans, CUB
  // arg-min (first minimum = the reference's first optimum), then sort +
  // unique for the distribution; chunk results merge on the host. Buffers
  // come from the stream-ordered pool, so repeated calls reuse them.
  const int64_t chunk = std::min<int64_t>(perms, int64_t{1} << 26);
  DevMem m_ms, m_sorted, m_uniq, m_nu, m_arg, m_tmp;
  size_t tmp_bytes = 0, b1 = 0, b2 = 0, b3 = 0;
  const int nc = static_cast<int>(chunk);
  CK(cub::DeviceReduce::ArgMin(nullptr, b1, static_cast<int64_t*>(nullptr),
                               static_cast<cub::KeyValuePair<int, int64_t>*>(nullptr), nc));
  CK(cub::DeviceRadixSort::SortKeys(nullptr, b2, static_cast<int64_t*>(nullptr), static_cast<int64_t*>(nullptr), nc));
  CK(cub::DeviceSelect::Unique(nullptr, b3, static_cast<int64_t*>(nullptr), static_cast<int64_t*>(nullptr),
                               static_cast<int*>(nullptr), nc));
  tmp_bytes = std::max(b1, std::max(b2, b3));
  CK(cudaMallocAsync(&m_ms.p, 8 * chunk, 0));
  CK(cudaMallocAsync(&m_sorted.p, 8 * chunk, 0));
  CK(cudaMallocAsync(&m_uniq.p, 8 * chunk, 0));
  CK(cudaMallocAsync(&m_nu.p, 8, 0));
  CK(cudaMallocAsync(&m_arg.p, sizeof(cub::KeyValuePair<int, int64_t>), 0));
  CK(cudaMallocAsync(&m_tmp.p, std::max<size_t>(tmp_bytes, 16), 0));
  void *d_ms = m_ms.p, *d_sorted = m_sorted.p, *d_uniq = m_uniq.p, *d_nu = m_nu.p, *d_arg = m_arg.p,
       *d_tmp = m_tmp.p;
  std::vector<int64_t> all;
  bool have = false;
  int rc = 0;
  for (int64_t base = 0; base < perms && rc == 0; base += chunk) {
    const int n = static_cast<int>(std::min(chunk, perms - base));
    rc = csk_sweep_lex(p, base, n, static_cast<int64_t*>(d_ms), err);
    if (rc) break;
    size_t t = tmp_bytes;
    cudaError_t e = cub::DeviceReduce::ArgMin(d_tmp, t, static_cast<int64_t*>(d_ms),
                                              static_cast<cub::KeyValuePair<int, int64_t>*>(d_arg), n);
    cub::KeyValuePair<int, int64_t> h{};
    if (e == cudaSuccess) e = cudaMemcpy(&h, d_arg, sizeof(h), cudaMemcpyDeviceToHost);
    t = tmp_bytes;
    if (e == cudaSuccess)
      e = cub::DeviceRadixSort::SortKeys(d_tmp, t, static_cast<int64_t*>(d_ms), static_cast<int64_t*>(d_sorted), n);
    t = tmp_bytes;
    if (e == cudaSuccess)
      e = cub::DeviceSelect::Unique(d_tmp, t, static_cast<int64_t*>(d_sorted), static_cast<int64_t*>(d_uniq),
                                    static_cast<int*>(d_nu), n);
    int nu = 0;
    if (e == cudaSuccess) e = cudaMemcpy(&nu, d_nu, sizeof(int), cudaMemcpyDeviceToHost);
    std::vector<int64_t> u(static_cast<size_t>(nu));
    if (e == cudaSuccess && nu) e = cudaMemcpy(u.data(), d_uniq, 8ull * nu, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
      std::snprintf(err, 256, "CUDA error %s in brute force", cudaGetErrorString(e));
      rc = 1;
      break;
    }
    LAUNCHED();
    if (!have || h.value < *best_m) {
      *best_m = h.value;
      *best_k = base + h.key;
      have = true;
    }
    std::vector<int64_t> merged;
    std::merge(all.begin(), all.end(), u.begin(), u.end(), std::back_inserter(merged));
    merged.erase(std::unique(merged.begin(), merged.end()), merged.end());
    all.swap(merged);
  }
  if (rc) return rc;
  *n_distinct = static_cast<int64_t>(all.size());
  if (static_cast<int64_t>(all.size()) <= cap) std::copy(all.begin(), all.end(), distinct);
  return 0;
}

extern "C" int csk_random_orders(int32_t R, int32_t S, const uint64_t* seeds, int32_t* perms, char* err) {
  if (ensure_device(err)) return 1;
  if (R <= 0 || S <= 0) return 0;
  std::vector<uint64_t> lim(4096), mag(4096);
  for (uint64_t k = 0; k < 4096; ++k) bounded_consts(k, &lim[k], &mag[k]);
  DevMem d_seeds, d_lim, d_mag, d_perm;
  CK(cudaMallocAsync(&d_seeds.p, 8ull * S, 0));
  CK(cudaMallocAsync(&d_lim.p, 8ull * lim.size(), 0));
  CK(cudaMallocAsync(&d_mag.p, 8ull * mag.size(), 0));
  CK(cudaMallocAsync(&d_perm.p, 4ull * R * S, 0));
  CK(cudaMemcpy(d_seeds.p, seeds, 8ull * S, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_lim.p, lim.data(), 8ull * lim.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_mag.p, mag.data(), 8ull * mag.size(), cudaMemcpyHostToDevice));
  random_orders_kernel<<<std::max(1, std::min((S + 127) / 128, 1184)), 128>>>(
      R, S, d_seeds.as<uint64_t>(), d_lim.as<uint64_t>(), d_mag.as<uint64_t>(), d_perm.as<int32_t>());
  LAUNCHED();
  CK(cudaGetLastError());
  CK(cudaMemcpy(perms, d_perm.p, 4ull * R * S, cudaMemcpyDeviceToHost));
  return 0;
}
