#pragma once
// Counter-based random numbers shared by the generators and the solver's
// start vectors.  The reference ships no RNG (SPEC.md
// "Random vectors: standard normal entries"), so the stream definition is
// ours and frozen here:
//
//   mix(z)        = splitmix64 finaliser
//   key(seed, s)  = mix(seed * G + s * S + C)
//   u64(key, c)   = mix(key + (c + 1) * G)
//   uniform       = ((u64 >> 11) + 0.5) * 2^-53            in (0, 1)
//   normal[i]     = Box-Muller on uniforms (2*(i/2), 2*(i/2)+1):
//                   r = sqrt(-2 ln u1), t = 2*pi*u2,
//                   i even -> r cos t, i odd -> r sin t
//
// Everything is evaluated on the host with the platform libm so that the
// product and the oracle (an independent restatement) agree bit for bit.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

namespace ppa {
namespace rng {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kStreamMul = 0xD1B54A32D192ED03ull;
constexpr uint64_t kKeyOffset = 0x8BB84B93962EACC9ull;

// Stream identifiers.
enum Stream : uint64_t {
  kNormEstimate = 1,
  kPolyStart = 2,
  kArnoldiStart = 3,
  kPoly2Start = 4,
  kMatrix = 5,
  kBreakdownRestart = 6,
};

inline uint64_t mix(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

inline uint64_t key(uint64_t seed, uint64_t stream) {
  return mix(seed * kGolden + stream * kStreamMul + kKeyOffset);
}

inline uint64_t u64(uint64_t k, uint64_t ctr) { return mix(k + (ctr + 1) * kGolden); }

inline double uniform(uint64_t k, uint64_t ctr) {
  return (static_cast<double>(u64(k, ctr) >> 11) + 0.5) * 0x1p-53;
}

/// Entry i of the standard-normal vector of stream key k.
inline double normal_at(uint64_t k, uint64_t i) {
  const uint64_t p = i >> 1;
  const double u1 = uniform(k, 2 * p);
  const double u2 = uniform(k, 2 * p + 1);
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double t = 6.283185307179586 * u2;
  return (i & 1) ? r * std::sin(t) : r * std::cos(t);
}

/// Entries are independent (counter-based), so the host threads split the
/// range without changing a bit of the result.  Each Box-Muller pair is
/// evaluated once for both of its members (same r and t as normal_at).
inline void fill_normal(double* v, long long n, uint64_t seed, uint64_t stream) {
  const uint64_t k = key(seed, stream);
  auto fill = [&](long long b, long long e) {  // b even
    for (long long i = b; i < e; i += 2) {
      const uint64_t p = static_cast<uint64_t>(i) >> 1;
      const double r = std::sqrt(-2.0 * std::log(uniform(k, 2 * p)));
      const double t = 6.283185307179586 * uniform(k, 2 * p + 1);
      v[i] = r * std::cos(t);
      if (i + 1 < e) v[i + 1] = r * std::sin(t);
    }
  };
  const unsigned hw = std::thread::hardware_concurrency();
  const long long nt = n < (1 << 16) ? 1 : std::max(1u, std::min(hw, 64u));
  if (nt == 1) {
    fill(0, n);
    return;
  }
  std::vector<std::thread> pool;
  const long long chunk = ((n + nt - 1) / nt + 1) & ~1LL;
  for (long long t = 0; t < nt && t * chunk < n; ++t) {
    pool.emplace_back(fill, t * chunk, std::min(n, (t + 1) * chunk));
  }
  for (auto& th : pool) th.join();
}

inline std::vector<double> normal_vector(long long n, uint64_t seed, uint64_t stream) {
  std::vector<double> v(static_cast<size_t>(n));
  fill_normal(v.data(), n, seed, stream);
  return v;
}

/// Sequential per-row draws used by the random sparse generator.
struct RowStream {
  uint64_t k;
  uint64_t ctr = 0;
  RowStream(uint64_t matrix_key, uint64_t row) : k(mix(matrix_key + (row + 1) * kStreamMul)) {}
  double uniform() { return rng::uniform(k, ctr++); }
  double normal() {  // first Box-Muller member of a fresh pair
    const double u1 = uniform();
    const double u2 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
  }
};

}  // namespace rng
}  // namespace ppa
