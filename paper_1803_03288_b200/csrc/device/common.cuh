// Shared device helpers: error plumbing, launch accounting, and the
// reference's random streams (rng.hpp:14-54) bit-exact on the GPU.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstring>

namespace tictac_dev {

extern std::atomic<int64_t> g_launches;

struct CudaError {
  int code;
};

// Every CUDA call goes through CK; a failure becomes a message in `err`.
#define CK(call)                                                                   \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) {                                                       \
      std::snprintf(err, 256, "CUDA error %s at %s:%d (%s)", cudaGetErrorString(e_), \
                    __FILE__, __LINE__, #call);                                    \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

#define LAUNCHED() tictac_dev::g_launches.fetch_add(1, std::memory_order_relaxed)

int ensure_device(char* err);  // selects/initialises the current device

// Lets a kernel launch with up to the device's opt-in shared memory. The
// limit is a per-function attribute, not per launch: setting it to one call's
// need would race with (or shrink below) another caller's, so every caller
// sets the same maximum (idempotent).
inline cudaError_t allow_max_dynamic_smem(const void* fn) {
  int dev = 0, optin = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa{};
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, fn);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             optin - static_cast<int>(fa.sharedSizeBytes));
  return e;
}

// Owned device allocation (freed on every exit path).
// Per-call device buffer from the stream-ordered pool (allocate with
// cudaMallocAsync on the legacy stream; freed in stream order).
struct DevMem {
  void* p = nullptr;
  DevMem() = default;
  DevMem(const DevMem&) = delete;
  DevMem& operator=(const DevMem&) = delete;
  ~DevMem() {
    if (p) cudaFreeAsync(p, 0);
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// ------------------------------------------------- bulk copies (TMA) ----
// 1-D bulk global->shared copies on the TMA engine (cp.async.bulk, SASS
// UBLKCP), completion tracked by a shared-memory mbarrier. Addresses 16-byte
// aligned, sizes multiples of 16.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.b32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
}
__host__ __device__ constexpr size_t round16(size_t x) { return (x + 15) & ~size_t(15); }

// ---------------------------------------------------------------- RNG ----
constexpr uint64_t kMtMul = 6364136223846793005ULL;
constexpr uint64_t kMtMatrix = 0xB5026F5AA96619E9ULL;
constexpr uint64_t kUpper = 0xFFFFFFFF80000000ULL;
constexpr uint64_t kLower = 0x7FFFFFFFULL;
constexpr uint64_t kPhi = 0x9e3779b97f4a7c15ULL;

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// mt19937_64 seeding recurrence: s[i] = K * (s[i-1] ^ (s[i-1] >> 62)) + i.
__device__ __forceinline__ uint64_t mt_step(uint64_t prev, uint32_t i) {
  return kMtMul * (prev ^ (prev >> 62)) + i;
}
__device__ __forceinline__ uint32_t lo32(uint64_t x) { return static_cast<uint32_t>(x); }
__device__ __forceinline__ uint32_t hi32(uint64_t x) { return static_cast<uint32_t>(x >> 32); }
__device__ __forceinline__ uint64_t join64(uint32_t lo, uint32_t hi) {
  return (static_cast<uint64_t>(hi) << 32) | lo;
}

// One twist element: c ^ ((a&U | b&L) >> 1) ^ (odd ? MATRIX : 0), on 32-bit
// halves (x.hi = a.hi; x.lo = a.lo&0x80000000 | b.lo&0x7fffffff, one LOP3
// select; the odd term is (b & 1) * MATRIX half on the FMA pipe, folded
// into a three-input XOR — the RNG is bound by the ALU pipe).
__device__ __forceinline__ uint32_t sel_upper(uint32_t a, uint32_t b) {
  uint32_t r;  // (a & 0x80000000) | (b & 0x7fffffff) as one LOP3 (ptxas would narrow the mask to two)
  asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(r) : "r"(a), "r"(b), "n"(0x80000000u));
  return r;
}
template <uint32_t C>
__device__ __forceinline__ uint32_t mulc(uint32_t x) {
  uint32_t r;
  asm("mul.lo.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "n"(C));
  return r;
}
__device__ __forceinline__ uint64_t mt_twist(uint64_t a, uint64_t b, uint64_t c) {
  const uint32_t xh = hi32(a);
  const uint32_t xl = sel_upper(lo32(a), lo32(b));
  const uint32_t odd = lo32(b) & 1u;
  const uint32_t rl = lo32(c) ^ ((xl >> 1) | (xh << 31)) ^ mulc<0xA96619E9u>(odd);
  const uint32_t rh = hi32(c) ^ (xh >> 1) ^ mulc<0xB5026F5Au>(odd);
  return join64(rl, rh);
}
// x ^ (y & C) as one LOP3 (ptxas tends to split a chain of these into three).
template <uint32_t C>
__device__ __forceinline__ uint32_t xor_and(uint32_t x, uint32_t y) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0x78;" : "=r"(r) : "r"(x), "r"(y), "n"(C));
  return r;
}
__device__ __forceinline__ uint64_t mt_temper(uint64_t y) {
  uint32_t l = lo32(y), h = hi32(y);
  l = xor_and<0x55555555u>(l, (l >> 29) | (h << 3));  // y ^= (y >> 29) & 0x5555555555555555
  h = xor_and<0x5u>(h, h >> 29);
  h = xor_and<0x71D67FFFu>(h, (h << 17) | (l >> 15));  // y ^= (y << 17) & 0x71D67FFFEDA60000
  l = xor_and<0xEDA60000u>(l, l << 17);
  h = xor_and<0xFFF7EEE0u>(h, l << 5);                  // y ^= (y << 37) & 0xFFF7EEE000000000
  l ^= h >> 11;                                         // y ^= y >> 43
  return join64(l, h);
}

// Full-state engine for streams of any length (state in memory owned by the
// caller: 312 words). Used by single-lane consumers.
// State behind any indexable P (a pointer, or a strided view).
template <typename P>
struct MtFullP {
  P mt;
  int idx;
  __device__ void seed(uint64_t s) {
    mt[0] = s;
    for (uint32_t i = 1; i < 312; ++i) mt[i] = mt_step(mt[i - 1], i);
    idx = 312;
  }
  __device__ uint64_t next() {
    if (idx >= 312) {
      for (int i = 0; i < 312; ++i) mt[i] = mt_twist(mt[i], mt[(i + 1) % 312], mt[(i + 156) % 312]);
      idx = 0;
    }
    return mt_temper(mt[idx++]);
  }
};
using MtFull = MtFullP<uint64_t*>;

// The same sequence with the twist done in place one element per draw:
// output i of a block needs s[i], s[i+1] and s[i+156] of the previous
// block, or, for i >= 156, the already-twisted t[i-156] (and t[0] for
// i = 311) — exactly what the array holds when elements are twisted in draw
// order. No 312-element burst, so 32 lockstep runs that draw at different
// times (the event replica's choice streams) do not serialise a whole
// twist loop each.
template <typename P>
struct MtInPlaceP {
  P mt;
  int idx;
  __device__ void seed(uint64_t s) {
    uint64_t prev = s;
    mt[0] = s;
    for (uint32_t i = 1; i < 312; ++i) {
      prev = mt_step(prev, i);
      mt[i] = prev;
    }
    idx = 0;
  }
  __device__ __forceinline__ uint64_t next() {
    const int i = idx;
    const int i1 = i == 311 ? 0 : i + 1;
    const int im = i < 156 ? i + 156 : i - 156;
    const uint64_t v = mt_twist(mt[i], mt[i1], mt[im]);
    mt[i] = v;
    idx = i1;
    return mt_temper(v);
  }
};

// Register-only engine for the first 311 outputs (SURVEY §7 hard part 2:
// every random order with R <= 312 lives in the first block). Outputs
// i < 156 need s[i], s[i+1], s[i+156]; outputs 156 <= i < 311 need the
// already-twisted t[i-156] = s[i] ^ f(s[i-156], s[i-155]). Two seeding
// cursors run 156 apart, so no state array is stored.
struct MtLazy {
  uint64_t seed, a0, a1, b, c0, c1;
  int i;
  __device__ __forceinline__ void init(uint64_t s) {
    seed = s;
    a0 = s;
    a1 = mt_step(s, 1);
    b = s;
#pragma unroll 4
    for (uint32_t k = 1; k <= 156; ++k) b = mt_step(b, k);
    c0 = c1 = 0;
    i = 0;
  }
  __device__ __forceinline__ bool exhausted() const { return i >= 311; }
  __device__ __forceinline__ uint64_t next_raw() {
    uint64_t t;
    if (i < 156) {
      t = mt_twist(a0, a1, b);
      a0 = a1;
      a1 = mt_step(a1, static_cast<uint32_t>(i + 2));
      b = mt_step(b, static_cast<uint32_t>(i + 157));
      if (i == 155) {
        c0 = seed;
        c1 = mt_step(seed, 1);
      }
    } else {
      const uint64_t back = mt_twist(c0, c1, a0);  // t[i-156]
      t = mt_twist(a0, a1, back);
      a0 = a1;
      a1 = mt_step(a1, static_cast<uint32_t>(i + 2));
      c0 = c1;
      c1 = mt_step(c1, static_cast<uint32_t>(i - 154));
    }
    ++i;
    return mt_temper(t);
  }
};

// The same over a caller-owned state P (312 words, e.g. a strided view into
// scratch) that is only seeded and used once the first 311 outputs are spent.
template <typename P>
struct MtLazyP {
  MtLazy lz;
  MtFullP<P> full;
  bool on_full;
  __device__ __forceinline__ void seed(uint64_t s) {
    lz.init(s);
    on_full = false;
  }
  __device__ __forceinline__ uint64_t next() {
    if (!on_full) {
      if (!lz.exhausted()) return lz.next_raw();
      full.seed(lz.seed);
      for (int k = 0; k < lz.i; ++k) full.next();
      on_full = true;
    }
    return full.next();
  }
};

// A stream of any length: the first 311 outputs from MtLazy's register
// cursors, then a full state in local memory continuing the same sequence.
struct MtStream {
  MtLazy lz;
  uint64_t st[312];
  int idx;
  bool full;
  __device__ __forceinline__ void init(uint64_t s) {
    lz.init(s);
    full = false;
  }
  __device__ __forceinline__ uint64_t next() {
    if (!full) {
      if (!lz.exhausted()) return lz.next_raw();
      MtFull m{st, 0};
      m.seed(lz.seed);
      for (int k = 0; k < lz.i; ++k) m.next();
      idx = m.idx;
      full = true;
    }
    MtFull m{st, idx};
    const uint64_t v = m.next();
    idx = m.idx;
    return v;
  }
};

constexpr uint64_t kNoiseSalt = 0x9e3779b97f4a7c15ULL;  // reorder-noise stream salt, sim.cpp:14

// Bounded draw (rng.hpp:21-30) with host-precomputed per-n constants:
// limit = UINT64_MAX - (2^64 mod n), magic = floor(2^64 / n).
__device__ __forceinline__ uint64_t fastmod(uint64_t v, uint64_t n, uint64_t magic) {
  const uint64_t q = __umul64hi(v, magic);
  uint64_t r = v - q * n;
  if (r >= n) r -= n;
  return r;
}

// Same, remainder only: r = v - q*n < 2n < 2^32 is exact in the low word;
// the conditional subtract is an unsigned min (r - n wraps when r < n).
__device__ __forceinline__ uint32_t fastmod32(uint64_t v, uint32_t n, uint64_t magic) {
  const uint64_t q = __umul64hi(v, magic);
  const uint32_t r = static_cast<uint32_t>(v) - static_cast<uint32_t>(q) * n;
  return min(r, r - n);
}

// The same with the negated modulus (-n mod 2^32), which callers stepping
// through consecutive n keep in a counter.
__device__ __forceinline__ uint32_t fastmod32n_exact(uint64_t v, uint32_t nneg, uint64_t magic) {
  const uint64_t q = __umul64hi(v, magic);
  const uint32_t r = static_cast<uint32_t>(v) + static_cast<uint32_t>(q) * nneg;
  return min(r, r + nneg);
}

// ... and with a cheaper quotient: bits
// 64..95 of v * magic without the lo*lo partial product (and without the
// carries above bit 95), so q is floor(v/n) - {0, 1, 2} (the dropped term is
// below 2^64, i.e. below one unit of q) and two conditional subtracts finish
// the remainder (r < 3n < 2^32 is exact in 32 bits).
__device__ __forceinline__ uint32_t fastmod32n(uint64_t v, uint32_t nneg, uint64_t magic) {
  const uint32_t vl = static_cast<uint32_t>(v), vh = static_cast<uint32_t>(v >> 32);
  const uint32_t ml = static_cast<uint32_t>(magic), mh = static_cast<uint32_t>(magic >> 32);
  uint32_t q;
  asm("{\n\t.reg .u64 c;\n\t.reg .u32 cl, ch;\n\t"
      "mul.wide.u32 c, %1, %2;\n\tmad.wide.u32 c, %3, %4, c;\n\t"
      "mov.b64 {cl, ch}, c;\n\tmad.lo.u32 %0, %1, %4, ch;\n\t}"
      : "=r"(q)
      : "r"(vh), "r"(ml), "r"(vl), "r"(mh));
  uint32_t r = vl + q * nneg;
  r = min(r, r + nneg);
  return min(r, r + nneg);
}

// bounded() rejects v > UINT64_MAX - (2^64 mod n); for n < 2^32 that needs
// the high word to be all ones, so the common test is one 32-bit compare.
__device__ __forceinline__ bool maybe_reject(uint64_t v) {
  return static_cast<uint32_t>(v >> 32) == 0xFFFFFFFFu;
}

inline void bounded_consts(uint64_t n, uint64_t* limit, uint64_t* magic) {
  if (n < 2) {
    *limit = ~0ULL;
    *magic = 0;
    return;
  }
  const uint64_t rem = (UINT64_MAX % n + 1) % n;
  *limit = UINT64_MAX - rem;
  *magic = static_cast<uint64_t>((static_cast<unsigned __int128>(1) << 64) / n);
}

// ----------------------------------------------------------- warp ops ----
__device__ __forceinline__ int64_t warp_min64(int64_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = min(v, static_cast<int64_t>(__shfl_xor_sync(~0u, v, o)));
  return v;
}
__device__ __forceinline__ int64_t warp_max64(int64_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = max(v, static_cast<int64_t>(__shfl_xor_sync(~0u, v, o)));
  return v;
}
__device__ __forceinline__ int warp_sum(int v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(~0u, v, o);
  return v;
}
// position of the k-th (0-based) set bit of x
__device__ __forceinline__ int nth_bit(uint32_t x, int k) {
  for (int j = 0; j < k; ++j) x &= x - 1;
  return __ffs(x) - 1;
}

}  // namespace tictac_dev
