// skv_gen.cpp -- deterministic synthetic prompt batches for the bench configs and tests
// (SURVEY.md section 8(d)).  BENCH / TEST INFRASTRUCTURE, not product code (see skv_gen.h).  Built from the reference's generator primitives, restated:
//   SplitMix64 / derive_seed      (util.hpp:14-55)
//   detail::filler, base36        (workload.hpp:243-266)  letters-only, unique prefix
//   detail::make_secret           (workload.hpp:182-241)  8 PII template families
// Every prompt p is a pure function of (seed, prompt_id_base + p), so shards of a
// global batch generated on different ranks are bit-identical to the single-rank batch.
#include <algorithm>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "skv_gen.h"
#include "../paper_2508_08438_b200/csrc/route.hpp"

namespace {

struct SplitMix64 {
  uint64_t s;
  explicit SplitMix64(uint64_t seed) : s(seed) {}
  uint64_t next() {
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  double next_double() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  uint64_t next_below(uint64_t bound) { return next() % bound; }
};

uint64_t derive_seed(uint64_t root, uint64_t tag) {
  SplitMix64 r(root ^ (0x51a1c9e3b7d24f85ULL * (tag + 1)));
  return r.next();
}

std::string base36(uint64_t v) {
  static const char* a = "0123456789abcdefghijklmnopqrstuvwxyz";
  std::string s;
  do {
    s.push_back(a[v % 36]);
    v /= 36;
  } while (v);
  std::reverse(s.begin(), s.end());
  return s;
}

std::string filler(uint64_t uniq, size_t n, SplitMix64& rng) {
  std::string s = "u" + base36(uniq) + " ";
  while (s.size() < n) {
    size_t len = 3 + rng.next_below(6);
    for (size_t i = 0; i < len && s.size() < n; ++i) s.push_back(static_cast<char>('a' + rng.next_below(26)));
    if (s.size() < n) s.push_back(' ');
  }
  s.resize(n, 'x');
  return s;
}

std::string digits(SplitMix64& rng, size_t n) {
  std::string s;
  for (size_t i = 0; i < n; ++i) s.push_back(static_cast<char>('0' + rng.next_below(10)));
  return s;
}

std::string hex_pairs(SplitMix64& rng, size_t n) {
  static const char* hx = "0123456789abcdef";
  std::string s;
  for (size_t i = 0; i < n; ++i) {
    if (i) s.push_back(':');
    s.push_back(hx[rng.next_below(16)]);
    s.push_back(hx[rng.next_below(16)]);
  }
  return s;
}

std::string make_secret(size_t family, SplitMix64& rng) {
  switch (family % 8) {
    case 0: return "account number " + digits(rng, 8);
    case 1: {
      std::string a = digits(rng, 3), b = digits(rng, 2), c = digits(rng, 4);
      return "my ssn is " + a + "-" + b + "-" + c;
    }
    case 2: {
      std::string a = digits(rng, 3), b = digits(rng, 3), c = digits(rng, 4);
      return "call me at (" + a + ") " + b + "-" + c;
    }
    case 3: {
      std::string a = digits(rng, 4), b = digits(rng, 2);
      return "email me at user" + a + "@mail" + b + ".com";
    }
    case 4: {
      std::string a = digits(rng, 4), b = digits(rng, 4), c = digits(rng, 4), d = digits(rng, 4);
      return "card number " + a + "-" + b + "-" + c + "-" + d;
    }
    case 5: {
      uint64_t a = rng.next_below(200), b = rng.next_below(200), c = rng.next_below(200);
      return "server at 10." + std::to_string(a) + "." + std::to_string(b) + "." + std::to_string(c);
    }
    case 6: return "device mac " + hex_pairs(rng, 6);
    default: return "imei " + digits(rng, 15);
  }
}

constexpr uint64_t kPoolTag = 0x706f6f6c00000000ULL;   // "pool"
constexpr uint64_t kPoolUniq = 0x10000000000ULL;       // filler counters of pool prefixes
constexpr uint64_t kBodyUniq = 0x20000000000ULL;       // filler counters of prompt bodies

std::string pool_prefix(const skvgen_spec& s, uint64_t i) {
  SplitMix64 rng(derive_seed(s.seed, kPoolTag + i));
  return filler(kPoolUniq + i, s.pool_tokens, rng);
}

// Unique body of `n` bytes with PII phrases planted at the configured density.
std::string body(const skvgen_spec& s, uint64_t gid, size_t n, SplitMix64& rng) {
  std::string b = filler(kBodyUniq + gid, n, rng);
  double rate = s.pii_per_kib;  // phrases per KiB
  if (s.pii_mix) {
    double u = rng.next_double();
    rate = u < 0.6 ? 0.0 : (u < 0.9 ? 0.5 : 4.0);  // none / one per 2 KiB / one per 256 B
  }
  double x = rate * static_cast<double>(n) / 1024.0;
  uint64_t k = static_cast<uint64_t>(x);
  if (rng.next_double() < x - static_cast<double>(k)) ++k;
  if (k == 0 || n < 64) return b;
  // keep the first 24 bytes (the unique "u<id> ..." head) intact
  size_t avail = n - 24;
  size_t seg = avail / k;
  for (uint64_t j = 0; j < k; ++j) {
    std::string ph = " " + make_secret(rng.next_below(8), rng) + " ";
    if (ph.size() + 1 >= seg) break;
    size_t at = 24 + j * seg + rng.next_below(seg - ph.size());
    std::memcpy(&b[at], ph.data(), ph.size());
  }
  return b;
}

}  // namespace

extern "C" {

int skvgen_generate_pool(const skvgen_spec* s, uint32_t* tokens, uint64_t* offsets, uint64_t* users,
                      uint8_t* owners) {
  if (!s || !tokens || !offsets) return 1;
  for (uint64_t i = 0; i < s->pool_size; ++i) {
    std::string t = pool_prefix(*s, i);
    offsets[i] = i * s->pool_tokens;
    for (size_t k = 0; k < t.size(); ++k) tokens[i * s->pool_tokens + k] = static_cast<unsigned char>(t[k]);
    if (users) users[i] = s->first_user + i % std::max<uint64_t>(s->n_users, 1);
    if (owners) owners[i] = 0;
  }
  offsets[s->pool_size] = s->pool_size * s->pool_tokens;
  return 0;
}

int skvgen_route(const uint32_t* tokens, const uint64_t* offsets, uint32_t n_prompts, uint32_t block_tokens,
                 uint32_t depth, const uint64_t* prompt_ids, uint32_t world, uint32_t* rank_out) {
  if (!offsets || !rank_out || (n_prompts && !tokens) || block_tokens == 0 || world == 0) return 1;
  for (uint32_t p = 0; p < n_prompts; ++p) {
    if (offsets[p + 1] < offsets[p]) return 1;
    rank_out[p] = skvroute::route_one(tokens + offsets[p], offsets[p + 1] - offsets[p], block_tokens, depth,
                                       prompt_ids ? prompt_ids[p] : p, world);
  }
  return 0;
}

int skvgen_generate(const skvgen_spec* s, uint32_t* tokens, uint64_t* offsets, uint64_t* users, uint8_t* owners,
                 int nthreads) {
  if (!s || !tokens || !offsets) return 1;
  if (s->n_users == 0 || s->prompt_tokens == 0) return 4;
  if (s->shared_fraction > 0 && (s->pool_size == 0 || s->pool_tokens >= s->prompt_tokens)) return 4;
  if (s->route_world > 1 && (s->route_rank >= s->route_world || s->route_block_tokens == 0)) return 4;
  const uint64_t N = s->n_prompts, L = s->prompt_tokens;
  std::vector<std::string> pool;
  if (s->shared_fraction > 0)
    for (uint64_t i = 0; i < s->pool_size; ++i) pool.push_back(pool_prefix(*s, i));
  auto text_of = [&](uint64_t gid) {
    SplitMix64 rng(derive_seed(s->seed, gid));
    std::string text;
    if (s->shared_fraction > 0 && rng.next_double() < s->shared_fraction) text = pool[rng.next_below(s->pool_size)];
    text += body(*s, gid, L - text.size(), rng);
    return text;
  };
  // global prompt ids of the batch: prompt_id_base + [0, N), or -- routed -- the first N
  // ids from prompt_id_base on whose prompt routes to route_rank (skv_route)
  std::vector<uint64_t> gids(N);
  if (s->route_world <= 1) {
    for (uint64_t p = 0; p < N; ++p) gids[p] = s->prompt_id_base + p;
  } else {
    const uint32_t B = s->route_block_tokens, G = s->route_world, D = s->route_depth;
    const uint64_t need = static_cast<uint64_t>(D + 1) * B;  // tokens that decide the rank
    std::vector<int> pool_rank(pool.size(), -1);
    std::vector<uint32_t> tb(need);
    auto tok_rank = [&](const std::string& t, uint64_t gid) {
      if (L < need) return static_cast<uint32_t>(gid % G);
      for (uint64_t i = 0; i < need; ++i) tb[i] = static_cast<unsigned char>(t[i]);
      return skvroute::route_one(tb.data(), L, B, D, gid, G);
    };
    for (uint64_t gid = s->prompt_id_base, p = 0; p < N; ++gid) {
      SplitMix64 rng(derive_seed(s->seed, gid));
      uint32_t r;
      if (s->shared_fraction > 0 && rng.next_double() < s->shared_fraction && s->pool_tokens >= need) {
        const uint64_t i = rng.next_below(s->pool_size);  // the deciding tokens are the pool prefix's
        if (pool_rank[i] < 0) pool_rank[i] = static_cast<int>(tok_rank(pool[i], gid));
        r = static_cast<uint32_t>(pool_rank[i]);
      } else {
        r = tok_rank(text_of(gid), gid);
      }
      if (r == s->route_rank) gids[p++] = gid;
    }
  }
  auto work = [&](uint64_t p0, uint64_t p1) {
    for (uint64_t p = p0; p < p1; ++p) {
      const uint64_t gid = gids[p];
      std::string text = text_of(gid);
      uint32_t* t = tokens + p * L;
      for (uint64_t k = 0; k < L; ++k) t[k] = static_cast<unsigned char>(text[k]);
      offsets[p] = p * L;
      if (users) users[p] = s->first_user + gid % s->n_users;
      if (owners) owners[p] = 0;
      if (s->prompt_ids_out) s->prompt_ids_out[p] = gid;
    }
  };
  if (nthreads <= 0) nthreads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  uint64_t per = (N + nthreads - 1) / nthreads;
  std::vector<std::thread> th;
  for (int i = 0; i < nthreads; ++i) {
    uint64_t a = i * per, b = std::min(N, a + per);
    if (a < b) th.emplace_back(work, a, b);
  }
  for (auto& t : th) t.join();
  offsets[N] = N * L;
  return 0;
}

}  // extern "C"
