// NumPy's default_rng on the device: SeedSequence hash-mix -> PCG64
// (128-bit LCG, XSL-RR output), the bitgen's buffered 32-bit halves (low
// half first), `random_interval` (Generator.permutation's masked rejection)
// and `integers(n)` (Lemire's bounded rejection on next_uint32; no draw for
// n == 1).  Replica checked against NumPy in tests/test_oracle_kats.py.
#pragma once
#include "gs_internal.cuh"

namespace gs {

typedef unsigned __int128 u128;

// ---------------------------------------------------------------- RNG ----
struct Pcg64 {
  u128 state, inc;
  uint32_t buf;
  bool has_buf;

  __device__ static uint32_t hashmix(uint32_t v, uint32_t& hc) {
    v ^= hc;
    hc *= 0x931E8875u;
    v *= hc;
    return v ^ (v >> 16);
  }
  __device__ static uint32_t mix(uint32_t x, uint32_t y) {
    uint32_t r = 0xCA01F9DDu * x - 0x4973F715u * y;
    return r ^ (r >> 16);
  }
  // SeedSequence(entropy = uint32 words).generate_state(4, uint64)
  __device__ void seed(const uint32_t* ent, int n_ent) {
    uint32_t pool[4];
    uint32_t hc = 0x43B0D7E5u;
    for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < n_ent ? ent[i] : 0u, hc);
    for (int s = 0; s < 4; ++s)
      for (int d = 0; d < 4; ++d)
        if (s != d) pool[d] = mix(pool[d], hashmix(pool[s], hc));
    for (int s = 4; s < n_ent; ++s)
      for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(ent[s], hc));
    uint32_t o[8];
    uint32_t hb = 0x8B51F9DDu;
    for (int i = 0; i < 8; ++i) {
      uint32_t v = pool[i & 3];
      v ^= hb;
      hb *= 0x58F38DEDu;
      v *= hb;
      o[i] = v ^ (v >> 16);
    }
    uint64_t w[4];
    for (int i = 0; i < 4; ++i) w[i] = (uint64_t)o[2 * i] | ((uint64_t)o[2 * i + 1] << 32);
    const u128 sd = ((u128)w[0] << 64) | w[1];
    const u128 sq = ((u128)w[2] << 64) | w[3];
    inc = (sq << 1) | 1;
    state = 0;
    step();
    state += sd;
    step();
    has_buf = false;
    buf = 0;
  }
  __device__ void step() {
    const u128 mult = ((u128)0x2360ED051FC65DA4ULL << 64) | 0x4385DF649FCCF645ULL;
    state = state * mult + inc;
  }
  __device__ uint64_t next64() {
    step();
    uint64_t x = (uint64_t)(state >> 64) ^ (uint64_t)state;
    unsigned rot = (unsigned)(state >> 122);
    return (x >> rot) | (x << ((64 - rot) & 63));
  }
  __device__ uint32_t next32() {
    if (has_buf) { has_buf = false; return buf; }
    uint64_t v = next64();
    has_buf = true;
    buf = (uint32_t)(v >> 32);
    return (uint32_t)v;
  }
  __device__ uint64_t interval(uint64_t mx) {   // numpy random_interval
    if (mx == 0) return 0;
    uint64_t mask = mx;
    mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4;
    mask |= mask >> 8; mask |= mask >> 16; mask |= mask >> 32;
    if (mx <= 0xFFFFFFFFull) {
      uint64_t v;
      while ((v = (next32() & mask)) > mx) {}
      return v;
    }
    uint64_t v;
    while ((v = (next64() & mask)) > mx) {}
    return v;
  }
  __device__ double next_double() { return (double)(next64() >> 11) * (1.0 / 9007199254740992.0); }
  // Generator.integers(n), n >= 1 and < 2^32 (distributions.c
  // buffered_bounded_lemire_uint32 via random_bounded_uint64_fill)
  __device__ uint32_t integers(uint32_t n) {
    const uint32_t rng = n - 1;
    if (rng == 0) return 0;
    const uint32_t ex = n;
    uint64_t m = (uint64_t)next32() * ex;
    uint32_t lo = (uint32_t)m;
    if (lo < ex) {
      const uint32_t th = (0xFFFFFFFFu - rng) % ex;
      while (lo < th) {
        m = (uint64_t)next32() * ex;
        lo = (uint32_t)m;
      }
    }
    return (uint32_t)(m >> 32);
  }
};

__device__ inline int words_of(uint64_t x, uint32_t* out) {
  if (x == 0) { out[0] = 0; return 1; }
  int n = 0;
  while (x) { out[n++] = (uint32_t)x; x >>= 32; }
  return n;
}

__device__ inline void seed_pair(Pcg64& g, uint64_t a, uint64_t b) {
  uint32_t ent[4];
  int n = words_of(a, ent);
  n += words_of(b, ent + n);
  g.seed(ent, n);
}

}  // namespace gs
