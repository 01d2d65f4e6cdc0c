// util.hpp -- drop-in facade of the reference's util.hpp (proj/include/safekv/util.hpp:14-109) for
// the B200 admission path.  SplitMix64 / derive_seed / Fnv1a64 are host value utilities of the
// reference's vocabulary (workload generation, test seeding); the admission path's digests run on
// the device (token_seq_digest in core.hpp calls the CUDA library).
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <string_view>

namespace safekv {

// util.hpp:14-49
class SplitMix64 {
 public:
  explicit SplitMix64(uint64_t seed = 0) : state_(seed) {}
  uint64_t next() {
    uint64_t z = (state_ += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  uint64_t next_below(uint64_t bound) { return bound ? next() % bound : 0; }
  double next_double() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  // util.hpp:33-39 (Box-Muller, the reference's explicit formula)
  double next_normal() {
    double u1 = next_double();
    const double u2 = next_double();
    if (u1 <= 0.0) u1 = 0x1.0p-53;
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
  }

 private:
  uint64_t state_;
};

// util.hpp:52-55
inline uint64_t derive_seed(uint64_t root, uint64_t tag) {
  SplitMix64 r(root ^ (0x51a1c9e3b7d24f85ULL * (tag + 1)));
  return r.next();
}

// util.hpp:58-81
class Fnv1a64 {
 public:
  void update(const void* data, size_t n) {
    const auto* p = static_cast<const unsigned char*>(data);
    for (size_t i = 0; i < n; ++i) h_ = (h_ ^ p[i]) * 0x100000001b3ULL;
  }
  void update(std::string_view s) { update(s.data(), s.size()); }
  void update_u32(uint32_t v) {
    for (int i = 0; i < 4; ++i) h_ = (h_ ^ ((v >> (8 * i)) & 0xff)) * 0x100000001b3ULL;
  }
  void update_u64(uint64_t v) {
    update_u32(static_cast<uint32_t>(v));
    update_u32(static_cast<uint32_t>(v >> 32));
  }
  uint64_t digest() const { return h_; }

 private:
  uint64_t h_ = 0xcbf29ce484222325ULL;
};

inline uint64_t fnv1a64(std::string_view s) {
  Fnv1a64 f;
  f.update(s);
  return f.digest();
}

}  // namespace safekv
