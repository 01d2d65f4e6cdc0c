// route.hpp -- the multi-GPU request router's key arithmetic, shared by
// the product router (route.cpp, skv_route) and the bench/test workload generator
// (workload/skv_gen.cpp, which emits the prompts one rank owns).
//
// Ownership rule: entries at depth < D (the first D blocks of any prompt) are REPLICATED on every
// rank; an entry at depth >= D belongs to the rank of the key h_D of its depth-D ancestor, which is
// the same for every prompt through it (keys are chained, A.2).  A prompt with more than D full
// blocks is therefore routed by h_D; a prompt with at most D blocks touches replicated entries only
// and goes to prompt_id % world.  D = 0 is pure prefix-forest partitioning (route by the root).
// Keys: d_b = token_seq_digest (core.hpp:68-73), h_b = Fnv1a64(u64 h_{b-1} || u64 d_b) (util.hpp:58-81).
#pragma once

#include <cstdint>

namespace skvroute {

constexpr uint64_t kFnvOff = 0xcbf29ce484222325ULL, kFnvP = 0x100000001b3ULL;

inline uint64_t fnv_u32(uint64_t h, uint32_t v) {
  for (int i = 0; i < 4; ++i) h = (h ^ ((v >> (8 * i)) & 0xff)) * kFnvP;
  return h;
}
inline uint64_t fnv_u64(uint64_t h, uint64_t v) { return fnv_u32(fnv_u32(h, static_cast<uint32_t>(v)), v >> 32); }

inline uint64_t block_digest(const uint32_t* t, uint32_t B) {
  uint64_t d = fnv_u32(kFnvOff, B);
  for (uint32_t i = 0; i < B; ++i) d = fnv_u32(d, t[i]);
  return d;
}

// chained key h_D of block D (the caller guarantees (D + 1) * B tokens)
inline uint64_t key_at(const uint32_t* t, uint32_t B, uint32_t D) {
  uint64_t h = 0;
  for (uint32_t b = 0; b <= D; ++b) h = fnv_u64(fnv_u64(kFnvOff, h), block_digest(t + static_cast<uint64_t>(b) * B, B));
  return h;
}

inline uint32_t rank_of_key(uint64_t h, uint32_t world) {
  uint64_t z = h + 0x9e3779b97f4a7c15ULL;  // SplitMix64 finalizer, then multiply-high range map
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  z ^= z >> 31;
  return static_cast<uint32_t>((static_cast<unsigned __int128>(z) * world) >> 64);
}

inline uint32_t route_one(const uint32_t* t, uint64_t len, uint32_t B, uint32_t D, uint64_t prompt_id,
                          uint32_t world) {
  if (world <= 1) return 0;
  if (len < static_cast<uint64_t>(D + 1) * B) return static_cast<uint32_t>(prompt_id % world);
  return rank_of_key(key_at(t, B, D), world);
}

}  // namespace skvroute
