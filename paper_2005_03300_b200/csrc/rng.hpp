// xoshiro256** seeded through splitmix64 — the reference generator
// (rng.hpp:29-90) — plus GF(2) jump-ahead so that the GPU can start any
// sub-stream at an arbitrary draw index and reproduce the reference's
// sequential draws bit for bit.
#pragma once

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <vector>

namespace cagnet {

struct Xoshiro {
  uint64_t s[4];

  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

  explicit Xoshiro(uint64_t seed) {  // rng.hpp:31-40
    uint64_t x = seed;
    for (auto& w : s) {
      x += 0x9e3779b97f4a7c15ULL;
      uint64_t z = x;
      z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
      z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
      w = z ^ (z >> 31);
    }
  }
  uint64_t next() {  // rng.hpp:43-53
    const uint64_t result = rotl(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return result;
  }
  double next_double() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * next_double(); }
  uint64_t bounded(uint64_t bound) {  // rng.hpp:64-71
    if (bound == 0) throw std::invalid_argument("Rng::bounded: bound must be positive");
    const uint64_t threshold = (0 - bound) % bound;
    for (;;) {
      const uint64_t r = next();
      if (r >= threshold) return r % bound;
    }
  }
};

// 256x256 matrices over GF(2) acting on the xoshiro state (bit b of word w is
// state bit 64w+b).  Row r holds the input bits that XOR into output bit r.
struct Gf2Mat {
  uint64_t rows[256][4];
};

inline void gf2_mul(const Gf2Mat& a, const Gf2Mat& b, Gf2Mat& out) {
  for (int r = 0; r < 256; ++r) {
    uint64_t acc[4] = {0, 0, 0, 0};
    for (int w = 0; w < 4; ++w) {
      uint64_t bits = a.rows[r][w];
      while (bits) {
        const int j = 64 * w + __builtin_ctzll(bits);
        bits &= bits - 1;
        for (int q = 0; q < 4; ++q) acc[q] ^= b.rows[j][q];
      }
    }
    std::memcpy(out.rows[r], acc, sizeof(acc));
  }
}

inline void gf2_apply(const Gf2Mat& m, const uint64_t in[4], uint64_t out[4]) {
  uint64_t res[4] = {0, 0, 0, 0};
  for (int r = 0; r < 256; ++r) {
    const int p = __builtin_popcountll(m.rows[r][0] & in[0]) + __builtin_popcountll(m.rows[r][1] & in[1]) +
                  __builtin_popcountll(m.rows[r][2] & in[2]) + __builtin_popcountll(m.rows[r][3] & in[3]);
    if (p & 1) res[r >> 6] |= 1ull << (r & 63);
  }
  std::memcpy(out, res, sizeof(res));
}

// One xoshiro state-update step as a GF(2) matrix.
inline Gf2Mat xoshiro_step_matrix() {
  Gf2Mat t;
  std::memset(&t, 0, sizeof(t));
  for (int j = 0; j < 256; ++j) {
    uint64_t s[4] = {0, 0, 0, 0};
    s[j >> 6] = 1ull << (j & 63);
    const uint64_t tt = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= tt;
    s[3] = Xoshiro::rotl(s[3], 45);
    for (int r = 0; r < 256; ++r)
      if ((s[r >> 6] >> (r & 63)) & 1) t.rows[r][j >> 6] |= 1ull << (j & 63);
  }
  return t;
}

// Powers J^(2^i), i < nbits, of J = T^step.
inline std::vector<Gf2Mat> jump_powers(uint64_t step, int nbits) {
  Gf2Mat t = xoshiro_step_matrix();
  // J = T^step by square-and-multiply.
  Gf2Mat acc;
  std::memset(&acc, 0, sizeof(acc));
  for (int r = 0; r < 256; ++r) acc.rows[r][r >> 6] = 1ull << (r & 63);
  Gf2Mat base = t, tmp;
  uint64_t e = step;
  while (e) {
    if (e & 1) {
      gf2_mul(acc, base, tmp);
      acc = tmp;
    }
    e >>= 1;
    if (e) {
      gf2_mul(base, base, tmp);
      base = tmp;
    }
  }
  std::vector<Gf2Mat> out(static_cast<size_t>(nbits));
  if (nbits > 0) out[0] = acc;
  for (int i = 1; i < nbits; ++i) gf2_mul(out[i - 1], out[i - 1], out[i]);
  return out;
}

}  // namespace cagnet
