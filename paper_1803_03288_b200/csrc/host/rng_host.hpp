// Host RNG (rng.hpp:14-54): the input builders (graph generators) and the
// reorder-noise swaps of single closed-form simulations (apply_gate_noise,
// hotpath.cpp). The batched streams (random orders, simulator choices, noise
// per seed) are generated on the device by ../device/common.cuh with the
// same definitions.
#pragma once

#include <cstdint>
#include <random>

namespace tictac {

// rng.hpp:14-33 — raw std::mt19937_64 output is pinned by the standard; the
// bounded draw is rejection sampling without modulo bias.
struct HostRng {
  std::mt19937_64 eng;
  explicit HostRng(uint64_t seed) : eng(seed) {}
  uint64_t next() { return eng(); }
  uint64_t bounded(uint64_t n) {
    if (n < 2) return 0;
    const uint64_t limit = UINT64_MAX - (UINT64_MAX % n + 1) % n;
    uint64_t v;
    do v = next();
    while (v > limit);
    return v % n;
  }
  double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }  // rng.hpp:33
};

inline uint64_t splitmix64(uint64_t x) {  // rng.hpp:49-54
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

}  // namespace tictac
