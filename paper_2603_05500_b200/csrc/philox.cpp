// H1: numpy-compatible Philox4x64-10 permutation sampler (host C++).
//
// The reference samples every permutation through numpy's
// Generator(Philox) (linalg.py:264-291 `Rng`, permute.py:79-83
// `sample_permutation`, drawn at layer.py:139-140 and 310-311).  This is a
// restatement of numpy 2.x's algorithm so the B200 build can resample at
// merge time without numpy and stay bit-exact:
//   * Philox4x64 with 10 rounds, multipliers 0xD2E7470EE14C6C93 /
//     0xCA5A826395121157, Weyl increments 0x9E3779B97F4A7C15 /
//     0xBB67AE8584CAA73B;
//   * the 256-bit counter is pre-incremented before each block; a block
//     fills a 4-word buffer consumed in order;
//   * 32-bit draws take the low half of a 64-bit word, then the high half;
//   * bounded integers use masked rejection (uint32 path when max < 2^32);
//   * permutation(n) = arange(n) then Fisher-Yates for i = n-1 .. 1.
#include <cstdint>
#include <vector>

#include "common.cuh"

namespace {

constexpr uint64_t kM0 = 0xD2E7470EE14C6C93ULL;
constexpr uint64_t kM1 = 0xCA5A826395121157ULL;
constexpr uint64_t kW0 = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t kW1 = 0xBB67AE8584CAA73BULL;

inline void mulhilo(uint64_t a, uint64_t b, uint64_t* hi, uint64_t* lo) {
  unsigned __int128 p = static_cast<unsigned __int128>(a) * b;
  *hi = static_cast<uint64_t>(p >> 64);
  *lo = static_cast<uint64_t>(p);
}

void philox_block(const uint64_t ctr_in[4], const uint64_t key_in[2], uint64_t out[4]) {
  uint64_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint64_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; ++r) {
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo(kM0, c0, &hi0, &lo0);
    mulhilo(kM1, c2, &hi1, &lo1);
    uint64_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += kW0;
    k1 += kW1;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

uint64_t next64(poetx_philox_state* s) {
  if (s->buffer_pos < 4) return s->buffer[s->buffer_pos++];
  for (int i = 0; i < 4; ++i) {
    if (++s->counter[i] != 0) break;
  }
  philox_block(s->counter, s->key, s->buffer);
  s->buffer_pos = 1;
  return s->buffer[0];
}

uint32_t next32(poetx_philox_state* s) {
  if (s->has_uint32) {
    s->has_uint32 = 0;
    return static_cast<uint32_t>(s->uinteger);
  }
  uint64_t v = next64(s);
  s->has_uint32 = 1;
  s->uinteger = v >> 32;
  return static_cast<uint32_t>(v & 0xffffffffULL);
}

uint64_t bounded(poetx_philox_state* s, uint64_t mx) {
  if (mx == 0) return 0;
  uint64_t mask = mx;
  mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4;
  mask |= mask >> 8; mask |= mask >> 16; mask |= mask >> 32;
  if (mx <= 0xffffffffULL) {
    uint64_t v;
    while ((v = (next32(s) & mask)) > mx) {}
    return v;
  }
  uint64_t v;
  while ((v = (next64(s) & mask)) > mx) {}
  return v;
}

}  // namespace

extern "C" int poetx_philox_seed(poetx_philox_state* st, uint64_t seed, uint64_t stream) {
  POETX_REQUIRE(st != nullptr, POETX_ESHAPE, "poetx_philox_seed: null state");
  for (int i = 0; i < 4; ++i) { st->counter[i] = 0; st->buffer[i] = 0; }
  st->key[0] = seed;
  st->key[1] = stream;
  st->buffer_pos = 4;
  st->has_uint32 = 0;
  st->uinteger = 0;
  return POETX_OK;
}

extern "C" int poetx_philox_permutation(poetx_philox_state* st, int64_t n, int32_t* fwd,
                                        int32_t* inv) {
  POETX_REQUIRE(st != nullptr && fwd != nullptr, POETX_ESHAPE,
                "poetx_philox_permutation: null pointer");
  POETX_REQUIRE(n > 0, POETX_ESHAPE, "permutation size must be positive, got %lld",
                static_cast<long long>(n));
  POETX_REQUIRE(n <= INT32_MAX, POETX_ESHAPE, "permutation size %lld exceeds int32",
                static_cast<long long>(n));
  for (int64_t i = 0; i < n; ++i) fwd[i] = static_cast<int32_t>(i);
  for (int64_t i = n - 1; i >= 1; --i) {
    uint64_t j = bounded(st, static_cast<uint64_t>(i));
    int32_t t = fwd[i];
    fwd[i] = fwd[j];
    fwd[j] = t;
  }
  if (inv) {
    for (int64_t i = 0; i < n; ++i) inv[fwd[i]] = static_cast<int32_t>(i);
  }
  return POETX_OK;
}
