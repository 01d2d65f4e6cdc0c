// kernels.cu -- sm_100a kernels of the SafeKV admission hot path.
//
// Stage map (reference symbols they replace, proj/include/safekv/...):
//   k_hash_scan   token_seq_digest (core.hpp:68-73) + CompiledRuleSet::scan
//                 (detection.hpp:148-170) on every block window
//   k_chain       Fnv1a64 chained prefix key (util.hpp:58-81, A.2) + inherited label (A.4)
//   k_probe       RadixCacheIndex::match_prefix / visible / lowest_tier
//                 (cache_index.hpp:213-237, 483-485) over the flat index (A.5)
//   k_record      AccessStats::record (access_stats.hpp:27-37) -- exact, order-preserving
//   k_commit          RadixCacheIndex::insert first-creator-wins + resolve_block (A.7)
//   k_epoch_*     EntropyMonitor::epoch_pass / check_anomaly (monitor.hpp:56-99),
//                 set_label propagation (cache_index.hpp:654-685), AccessStats::roll
// No tensor cores: nothing here is a contraction.  Everything is integer/byte work
// bounded by HBM, shared-memory lookups or memory latency.
#include <cooperative_groups.h>
#include <algorithm>
#include <stdexcept>
#include <string>
#include <vector>
#include <cub/cub.cuh>

#include "../../include/safekv_b200.h"
#include "ctx.hpp"

namespace skv {
namespace {

__host__ __device__ inline uint32_t round16(uint32_t x) { return (x + 15u) & ~15u; }

constexpr uint64_t kFnvOff = 0xcbf29ce484222325ULL;
constexpr uint64_t kFnvP = 0x100000001b3ULL;
constexpr uint64_t kFnvP4 = kFnvP * kFnvP * kFnvP * kFnvP;  // (h^t)*P^4 == update_u32(t) for t < 256

// (h ^ b) * P with P = 2^40 + 0x1b3: lo * 0x1b3 as one wide multiply, then the high word
// gains hi * 0x1b3 and (lo << 8) -- three IMADs instead of a generic 64-bit multiply
// (chained keys in k_chain_probe: 0.229 -> 0.222 ms per config-2 batch)
__device__ __forceinline__ uint64_t fnv_byte(uint64_t h, uint32_t b) {
  const uint32_t lo = static_cast<uint32_t>(h) ^ b, hi = static_cast<uint32_t>(h >> 32);
  uint32_t rlo, rhi;
  asm("{\n\t.reg .u64 w;\n\t.reg .u32 wh;\n\t"
      "mul.wide.u32 w, %2, 0x1b3;\n\t"
      "mov.b64 {%0, wh}, w;\n\t"
      "mad.lo.u32 wh, %3, 0x1b3, wh;\n\t"
      "mad.lo.u32 %1, %2, 256, wh;\n\t}"
      : "=r"(rlo), "=r"(rhi)
      : "r"(lo), "r"(hi));
  return (static_cast<uint64_t>(rhi) << 32) | rlo;
}
__device__ __forceinline__ uint64_t fnv_u32(uint64_t h, uint32_t v) {
  h = fnv_byte(h, v & 0xff);
  h = fnv_byte(h, (v >> 8) & 0xff);
  h = fnv_byte(h, (v >> 16) & 0xff);
  return fnv_byte(h, v >> 24);
}
__device__ __forceinline__ uint64_t fnv_u64(uint64_t h, uint64_t v) {
  h = fnv_u32(h, static_cast<uint32_t>(v));
  return fnv_u32(h, static_cast<uint32_t>(v >> 32));
}
// A.2: h_b = FNV(u64 h_{b-1} || u64 d_b), h_{-1} = 0
__device__ __forceinline__ uint64_t chain_key(uint64_t prev, uint64_t d) {
  return fnv_u64(fnv_u64(kFnvOff, prev), d);
}

__device__ __forceinline__ uint64_t slot_hash(uint64_t h, uint64_t d) {
  uint64_t x = h ^ (d * 0x9e3779b97f4a7c15ULL);
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

// Home slot of the key of block b of a prompt.  Blocks are grouped by kGroup along the
// prompt; a group's region of kGroup consecutive 128-B lines (2 x 64-B entries each) is
// chosen by the hash of the group's first key (h_L, d_L), L = b - b % kGroup, and block
// b's home is the first entry of line b % kGroup.  Every lookup and insert walks a prompt
// from its root, so the group leader's key is always at hand, and a key always sits at
// the same depth under the same prefix, so its home is a function of the key.  Linear
// probing from the home slot visits the line's second entry first.
// kGroup = 1 (every key hashed on its own) is the default: grouping a prompt's blocks
// into shared DRAM pages speeds the probe slightly, but the commit's claim + parent-link
// traffic then concentrates on adjacent lines and slows down more (measured on B200,
// config 2: kGroup 1/2/4/8 -> commit 0.88/0.93/1.22/1.54 ms, probe 0.238/0.216/0.237/
// 0.254 ms), although isolated grouped CAS streams are ~1.9x faster
// (profiles/r01_randmem_microbench.jsonl).
#ifndef SKV_COMMIT_FLAT
#define SKV_COMMIT_FLAT 0  // measured slower (DESIGN 5.3); kept as the documented alternative
#endif
#ifndef SKV_GROUP
#define SKV_GROUP 1
#endif
constexpr uint32_t kGroup = SKV_GROUP;
__device__ __forceinline__ uint64_t home_slot(const Index& ix, uint64_t hL, uint64_t dL, uint32_t b) {
  return (slot_hash(hL, dL) & ix.mask & ~static_cast<uint64_t>(2 * kGroup - 1)) + 2 * (b % kGroup);
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }
constexpr uint32_t kFull = 0xffffffffu;

__device__ __forceinline__ uint4 ldg_stream(const uint32_t* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// ---------------------------------------------------------------------------------
// K0: blocks per prompt
// ---------------------------------------------------------------------------------
__global__ void k_block_counts(const uint64_t* __restrict__ off, uint32_t n, uint32_t B, uint32_t* counts,
                               uint32_t* plen) {
  uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) {
    const uint64_t L = off[p + 1] - off[p];
    counts[p] = static_cast<uint32_t>(L / B);
    plen[p] = static_cast<uint32_t>(min(L, static_cast<uint64_t>(0xffffffffu)));
  }
  if (p == n) counts[p] = 0;
}

// ---------------------------------------------------------------------------------
// Serving observables of an admitted batch (probe epilogue): per prompt
//   ttft = max(t_base + c_prefill * (L - m*B) + sum_{b<m} penalty[tier_b] * B + noise, t_base)
// in the reference's summation order (CostModel::ttft, serving_sim.hpp:50-56; one
// handle per matched block), noise = sigma * Box-Muller normal of
// SplitMix64(derive_seed(seed, request_id)) (util.hpp:14-55), and the reuse attribution
// of ServingSimulator::attribute_reuse (serving_sim.hpp:313-324): matched tokens on
// entries the user created (intra) vs created by others (inter).
// ---------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t splitmix_next(uint64_t& st) {
  uint64_t z = (st += 0x9e3779b97f4a7c15ULL);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__global__ void k_ttft(const uint32_t* __restrict__ blk_off, const uint32_t* __restrict__ matched,
                       const uint32_t* __restrict__ plen, const uint8_t* __restrict__ bmeta,
                       const uint64_t* __restrict__ request_ids, uint64_t request_base, uint32_t n, uint32_t B,
                       CostModelDev cm, double* __restrict__ ttft, uint32_t* __restrict__ intra,
                       uint32_t* __restrict__ inter) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const uint32_t m = matched[p], bo = blk_off[p];
  double t = cm.t_base + cm.c_prefill * static_cast<double>(static_cast<uint64_t>(plen[p]) - static_cast<uint64_t>(m) * B);
  uint32_t own = 0;
  for (uint32_t b = 0; b < m; ++b) {
    const uint32_t x = bmeta[bo + b];
    t += cm.penalty[x & 3u] * static_cast<double>(B);
    own += x >> 2;
  }
  double noise = 0.0;
  if (cm.sigma != 0.0) {
    const uint64_t rid = request_ids ? request_ids[p] : request_base + p;
    uint64_t st = cm.seed ^ (0x51a1c9e3b7d24f85ULL * (rid + 1));
    uint64_t st2 = splitmix_next(st);  // derive_seed(seed, request_id)
    const double u1r = static_cast<double>(splitmix_next(st2) >> 11) * 0x1.0p-53;
    const double u2 = static_cast<double>(splitmix_next(st2) >> 11) * 0x1.0p-53;
    const double u1 = u1r <= 0.0 ? 0x1.0p-53 : u1r;
    noise = cm.sigma * (sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2));
  }
  t += noise;
  ttft[p] = t > cm.t_base ? t : cm.t_base;
  intra[p] = own * B;
  inter[p] = (m - own) * B;
}

// ---------------------------------------------------------------------------------
// K12: fused block digest + rule-DFA window scan.
//
// Warp-autonomous persistent kernel: warp w of the grid owns global blocks
// [w*nb/NW, (w+1)*nb/NW) and walks them in chunks of 32 consecutive blocks (a chunk may
// span prompts), with no CTA-wide barrier after the DFA table load.  Per chunk:
//   staging  the chunk's token span [first window start, last window end) HBM -> the
//            warp's SMEM buffers with coalesced 128-bit streaming loads (every token is
//            read from HBM once; only the W-token right context of the last window is
//            re-read by the next chunk, from L2), converted to pre-scaled DFA byte
//            classes and raw bytes.  The next chunk's span is prefetched into L2 by TMA.
//   lane l owns window l (block b of prompt p, window [bB, min(L, bB+B+W))):
//   phase A  digest of block b (token_seq_digest, core.hpp:68-73) and the DFA run over
//            block b from the start state; records the state after kConv bytes (Z),
//            after W' = min(W,B) bytes (SW) and at the block end (X).
//   phase B  window l continues over the next block from X.  Window l+1 (block b+1)
//            ran those bytes from the start state; two runs of a DFA in the same state
//            at the same byte are identical from there on, so after kConv bytes window
//            l compares its state with lane l+1's Z: equal (the common case -- the runs
//            synchronise within a few bytes) -> window l's run over the rest of that
//            block IS window l+1's own-block run (its row-OR and state SW are reused
//            through a shuffle); otherwise window l steps the bytes itself.
//   phase C  (W = 2B) the same argument at the second block boundary: if window l is in
//            lane l+1's phase-B start state X, window l's last block is lane l+1's
//            phase-B run.
// So a window costs B + kConv DFA steps instead of B + W.  The fast pass only tracks
// WHETHER an accepting transition was taken (bit 15 of the OR of visited row offsets:
// accepting transitions land in copy rows >= 32 KB); the exact enabled-rule mask of the
// few windows that accepted is recomputed per flagged segment (own block / first /
// second context block) from its known start state, one lane per segment.
// ---------------------------------------------------------------------------------
#ifndef SKV_HS_WARPS
#define SKV_HS_WARPS 16
#endif
constexpr uint32_t kHSWarps = SKV_HS_WARPS;  // warps per CTA
constexpr uint32_t kConv = 4;  // context bytes stepped before comparing with the neighbour's run

__device__ __forceinline__ uint32_t lds16(const uint8_t* base, uint32_t off) {
  return *reinterpret_cast<const uint16_t*>(base + off);
}

// Rule mask carried by an accepting-copy row offset r (>= kAccRegion):
// copy index j = (r - kAccRegion) / row_bytes via a 32-bit reciprocal (exact: r is a
// multiple of row_bytes), mask = acc_tab[j] (SMEM, u16).
__device__ __forceinline__ uint32_t copy_mask(const uint16_t* acc_tab, uint32_t r, uint32_t inv) {
  return (r & kAccRegion) ? acc_tab[__umulhi(r - kAccRegion, inv)] : 0u;
}

// 4 DFA steps over the 4 class bytes of w; the visited row offsets are OR-ed into acc
__device__ __forceinline__ uint32_t step4(const uint8_t* __restrict__ tab, uint32_t row, uint32_t w,
                                          uint32_t& acc) {
  const uint32_t r0 = lds16(tab, row + __byte_perm(w, 0u, 0x4440u));
  const uint32_t r1 = lds16(tab, r0 + __byte_perm(w, 0u, 0x4441u));
  const uint32_t r2 = lds16(tab, r1 + __byte_perm(w, 0u, 0x4442u));
  const uint32_t r3 = lds16(tab, r2 + __byte_perm(w, 0u, 0x4443u));
  acc |= r0 | r1 | r2 | r3;
  return r3;
}

// DFA run over cls[o, end) from row (any alignment); OR of visited rows into acc
__device__ __forceinline__ uint32_t run_or(const uint8_t* __restrict__ tab, const uint8_t* __restrict__ cls,
                                           uint32_t o, uint32_t end, uint32_t row, uint32_t& acc) {
  uint32_t m = 0;
  while (o < end && (o & 3)) {
    row = lds16(tab, row + cls[o++]);
    m |= row;
  }
  for (; o + 4 <= end; o += 4) row = step4(tab, row, *reinterpret_cast<const uint32_t*>(cls + o), m);
  while (o < end) {
    row = lds16(tab, row + cls[o++]);
    m |= row;
  }
  acc |= m;
  return row;
}

// exact run: the enabled-rule mask of every accepting transition OR-ed into *mask
__device__ __forceinline__ uint32_t run_exact(const uint8_t* __restrict__ tab, const uint8_t* __restrict__ cls,
                                              const uint16_t* __restrict__ acc_tab, uint32_t inv, uint32_t o,
                                              uint32_t end, uint32_t row, uint32_t* mask) {
  uint32_t m = 0;
  for (; o < end; ++o) {
    row = lds16(tab, row + cls[o]);
    m |= copy_mask(acc_tab, row, inv);
  }
  *mask |= m;
  return row;
}

__device__ __forceinline__ uint64_t digest_bytes(const uint8_t* __restrict__ raw, uint32_t o, uint32_t n,
                                                 uint64_t h) {
  const uint32_t end = o + n;
  while (o < end && (o & 3)) h = (h ^ raw[o++]) * kFnvP4;
  for (; o + 4 <= end; o += 4) {
    const uint32_t w = *reinterpret_cast<const uint32_t*>(raw + o);
#pragma unroll
    for (int k = 0; k < 4; ++k) h = (h ^ __byte_perm(w, 0u, 0x4440u + k)) * kFnvP4;
  }
  for (; o < end; ++o) h = (h ^ raw[o]) * kFnvP4;
  return h;
}

__device__ __forceinline__ uint64_t digest16(uint4 v, uint64_t h) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int k = 0; k < 4; ++k) h = (h ^ __byte_perm(w[q], 0u, 0x4440u + k)) * kFnvP4;
  return h;
}

__device__ __forceinline__ void stage4(uint8_t* cls, uint8_t* raw, const uint8_t* cmap, uint32_t q, uint32_t t0,
                                       uint32_t t1, uint32_t t2, uint32_t t3, uint32_t& wide) {
  wide |= t0 | t1 | t2 | t3;
  const uint32_t c = cmap[t0 & 0xff] | (cmap[t1 & 0xff] << 8) | (cmap[t2 & 0xff] << 16) |
                     (static_cast<uint32_t>(cmap[t3 & 0xff]) << 24);
  reinterpret_cast<uint32_t*>(cls)[q] = c;
  reinterpret_cast<uint32_t*>(raw)[q] = __byte_perm(__byte_perm(t0, t1, 0x0040), __byte_perm(t2, t3, 0x0040), 0x5410);
}

__device__ __forceinline__ uint64_t shfl64(uint64_t v, uint32_t src) {
  const uint32_t lo = __shfl_sync(kFull, static_cast<uint32_t>(v), src);
  const uint32_t hi = __shfl_sync(kFull, static_cast<uint32_t>(v >> 32), src);
  return (static_cast<uint64_t>(hi) << 32) | lo;
}

// Deferred exact-mask task: a flagged segment (<= 16 tokens) of a window, its start row
// and where its mask goes.  32 B, one SMEM slot.
struct SegTask {
  unsigned long long tok;  // first token index of the segment
  uint32_t meta;           // start row | len << 16
  uint32_t gb, p, b;
  uint32_t pad;
};

// exact run over tokens[tok, tok+len) (len <= 16) from row: OR of the enabled-rule masks
// of every accepting transition
__device__ __forceinline__ uint32_t exact_tokens(const uint8_t* __restrict__ tab, const uint8_t* __restrict__ cmap,
                                                 const uint16_t* __restrict__ acc_tab, uint32_t inv,
                                                 const uint32_t* __restrict__ tokens, uint64_t tok, uint32_t len,
                                                 uint32_t row) {
  uint32_t t[16];
#pragma unroll
  for (uint32_t j = 0; j < 16; ++j) t[j] = j < len ? tokens[tok + j] : 0u;
  uint32_t m = 0;
#pragma unroll
  for (uint32_t j = 0; j < 16; ++j) {
    if (j < len) {
      row = lds16(tab, row + cmap[t[j] & 0xffu]);
      m |= copy_mask(acc_tab, row, inv);
    }
  }
  return m;
}

#ifndef SKV_QCAP
#define SKV_QCAP 64
#endif
constexpr uint32_t kQCap = SKV_QCAP;  // deferred tasks per warp (multiple of 32)

__device__ __forceinline__ void flush_tasks(const SegTask* q, uint32_t qn, uint32_t lane, const uint8_t* tab,
                                            const uint8_t* cmap, const uint16_t* acc_tab, uint32_t inv,
                                            const HashScanArgs& a) {
  __syncwarp();
  for (uint32_t k = lane; k < qn; k += 32) {
    const SegTask t = q[k];
    const uint32_t m = exact_tokens(tab, cmap, acc_tab, inv, a.tokens, t.tok, t.meta >> 16, t.meta & 0xffffu);
    if (m) {
      atomicOr(&a.mask_out[t.gb], m << a.mask_shift);
      atomicMin(&a.first_sens[t.p], t.b);
    }
  }
  __syncwarp();
}

// DFA run over tokens[o, e) from row (global loads, L1/L2 hits: the warp has just read
// these lines); OR of the visited rows into acc.  Used off the fast path only.
__device__ __forceinline__ uint32_t run_tokens(const uint8_t* __restrict__ tab, const uint8_t* __restrict__ cmap,
                                               const uint32_t* __restrict__ tokens, uint32_t o, uint32_t e,
                                               uint32_t row, uint32_t& acc) {
  uint32_t m = 0;
  for (; o < e; ++o) {
    row = lds16(tab, row + cmap[tokens[o] & 0xffu]);
    m |= row;
  }
  acc |= m;
  return row;
}

// FNV-1a step of a byte token: (h ^ t) * P^4 mod 2^64 in four 32-bit multiplies
#ifndef SKV_FNV4
#define SKV_FNV4 1
#endif
__device__ __forceinline__ uint64_t fnv_tok(uint64_t h, uint32_t t) {
  const uint32_t lo = static_cast<uint32_t>(h) ^ t, hi = static_cast<uint32_t>(h >> 32);
  uint32_t rlo, rhi;
#if SKV_FNV4
  // lo * P_lo as one wide multiply (no zeroed addend register), then the two cross terms
  // into the high word: XOR + IMAD.WIDE + 2 IMAD per token
  asm("{\n\t.reg .u64 w;\n\t.reg .u32 wh;\n\t"
      "mul.wide.u32 w, %2, %4;\n\t"
      "mov.b64 {%0, wh}, w;\n\t"
      "mad.lo.u32 wh, %2, %5, wh;\n\t"
      "mad.lo.u32 %1, %3, %4, wh;\n\t}"
      : "=r"(rlo), "=r"(rhi)
      : "r"(lo), "r"(hi), "r"(static_cast<uint32_t>(kFnvP4)), "r"(static_cast<uint32_t>(kFnvP4 >> 32)));
  return (static_cast<uint64_t>(rhi) << 32) | rlo;
#endif
  asm("{\n\t.reg .u32 c;\n\t"
      "mul.lo.u32 c, %2, %4;\n\t"
      "mad.lo.u32 c, %3, %5, c;\n\t"
      "mul.lo.u32 %0, %3, %4;\n\t"
      "mad.hi.u32 %1, %3, %4, c;\n\t}"
      : "=r"(rlo), "=r"(rhi)
      : "r"(hi), "r"(lo), "r"(static_cast<uint32_t>(kFnvP4)), "r"(static_cast<uint32_t>(kFnvP4 >> 32)));
  return (static_cast<uint64_t>(rhi) << 32) | rlo;
}

#ifndef SKV_TOK_LDQ
#define SKV_TOK_LDQ ".L1::no_allocate"  // the lines were prefetched into L1; a hit stays, a miss does not
                                         // evict the next chunk (A/B run 96: 0.1964 -> 0.1948 ms)
#endif
__device__ __forceinline__ void ldg_tokens16(const uint32_t* p, uint32_t (&t)[16], bool a8) {
  if (a8) {  // 32-B aligned: two 256-bit loads
#pragma unroll
    for (uint32_t k = 0; k < 2; ++k)
      asm volatile("ld.global.nc" SKV_TOK_LDQ ".v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(t[8 * k]), "=r"(t[8 * k + 1]), "=r"(t[8 * k + 2]), "=r"(t[8 * k + 3]), "=r"(t[8 * k + 4]),
                     "=r"(t[8 * k + 5]), "=r"(t[8 * k + 6]), "=r"(t[8 * k + 7])
                   : "l"(p + 8 * k));
  } else {
#pragma unroll
    for (uint32_t k = 0; k < 4; ++k) {
      const uint4 v = *reinterpret_cast<const uint4*>(p + 4 * k);
      t[4 * k] = v.x, t[4 * k + 1] = v.y, t[4 * k + 2] = v.z, t[4 * k + 3] = v.w;
    }
  }
}

#ifndef SKV_HS_PFCTX
#define SKV_HS_PFCTX 0
#endif
#ifndef SKV_HS_PFDIST
#define SKV_HS_PFDIST 1  // bit 0: next chunk, bit 1: the chunk after
#endif
// The next chunk's new token lines into L1 while this chunk computes: its windows start
// nout blocks on, so lane l touches block (nout + l) of the contiguous token stream (one
// 64-B segment per lane; exact within a prompt, harmless past its end); with
// SKV_HS_PFCTX the right-context blocks past the chunk too.
__device__ __forceinline__ void l1_prefetch_next(const uint32_t* tokens, uint64_t n_tokens, uint64_t T0,
                                                 uint32_t nout, uint32_t lane, uint32_t B, uint32_t W) {
#if SKV_HS_PFDIST & 1
  const uint64_t nt = T0 + static_cast<uint64_t>(nout + lane) * B;
  if (nt < n_tokens) asm volatile("prefetch.global.L1 [%0];" ::"l"(tokens + nt));
#endif
#if SKV_HS_PFDIST & 2
  const uint64_t nt2 = T0 + static_cast<uint64_t>(2 * nout + lane) * B;
  if (nt2 < n_tokens) asm volatile("prefetch.global.L1 [%0];" ::"l"(tokens + nt2));
#endif
#if SKV_HS_PFCTX
  if (lane * B < W) {
    const uint64_t ct = T0 + static_cast<uint64_t>(nout + 32 + lane) * B;
    if (ct < n_tokens) asm volatile("prefetch.global.L1 [%0];" ::"l"(tokens + ct));
  }
#endif
}

#ifndef SKV_HS_MINB
#define SKV_HS_MINB 2
#endif
#ifndef SKV_HS_L1PF
#define SKV_HS_L1PF 2  // 1: before phase B, 2: before phase A
#endif
__global__ void __launch_bounds__(kHSWarps * 32, SKV_HS_MINB) k_hash_scan(HashScanArgs a) {
  extern __shared__ __align__(16) uint8_t sm[];
  // row offsets index the DFA image [row_base, fast_bytes), which sits at sm[0..)
  const uint8_t* tab = sm - a.rules.row_base;
  uint16_t* acc_tab = reinterpret_cast<uint16_t*>(sm + a.off_list);
  __shared__ uint8_t cmap[256];
  __shared__ SegTask s_q[kHSWarps][kQCap];
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nwarps = blockDim.x >> 5;
  // start-up: the DFA image loads, this warp's block range and the prompt search are
  // all in flight before the first barrier
  const uint32_t n_img = (a.rules.fast_bytes - a.rules.row_base + 15) / 16;
  const uint4* img_src = reinterpret_cast<const uint4*>(a.rules.fast) + a.rules.row_base / 16;
  uint4 img[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t i = tid + k * blockDim.x;
    if (i < n_img) img[k] = img_src[i];
  }
  const uint32_t* __restrict__ tokens = a.tokens;
  const uint32_t inv = a.rules.copy_inv;
  const uint32_t N = a.n_prompts;
  const uint32_t nb = a.blk_off[N];  // device-side block count (no host round trip)
  const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * nwarps + wid, TW = static_cast<uint64_t>(gridDim.x) * nwarps;
  const uint32_t G0 = static_cast<uint32_t>(gw * nb / TW), G1 = static_cast<uint32_t>((gw + 1) * nb / TW);
  uint32_t pp = 0;
  if (G0 < G1) {  // prompt containing G0 (the last with blk_off <= G0): 32-ary search, one
                  // load per lane per round (4 dependent rounds for 65,536 prompts, not 16)
    uint32_t lo = 0, hi = N;
    while (hi - lo > 1) {
      const uint32_t step = (hi - lo + 31) / 32;
      const uint32_t m = lo + lane * step;
      const uint32_t bal = __ballot_sync(kFull, m < hi && a.blk_off[m] <= G0);  // a prefix of the lanes
      const uint32_t k = 31 - __clz(bal);
      lo += k * step;
      hi = min(hi, lo + step);
    }
    pp = lo;
  }
  {  // DFA rows and accepting copies [row_base, fast_bytes) -> SMEM
    uint4* dst = reinterpret_cast<uint4*>(sm);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t i = tid + k * blockDim.x;
      if (i < n_img) dst[i] = img[k];
    }
    for (uint32_t i = tid + 4 * blockDim.x; i < n_img; i += blockDim.x) dst[i] = img_src[i];
    if (tid < 64) reinterpret_cast<uint32_t*>(cmap)[tid] = reinterpret_cast<const uint32_t*>(a.rules.class2)[tid];
    for (uint32_t i = tid; i < a.rules.n_copies; i += blockDim.x) acc_tab[i] = a.rules.copy_acc[i];
  }
  __syncthreads();
  SegTask* q = s_q[wid];
  if (G0 >= G1) return;
  uint32_t g = G0, qn = 0;
  const uint32_t B = a.B, W = a.W;
  const uint32_t Wp = min(W, B), kc = min(kConv, Wp);
  const uint32_t start_row = a.rules.start_row, eos2 = a.rules.eos2;
  const bool b16 = B == 16 && W >= kConv;
  const bool bseg = B > 16 && B % 16 == 0;  // long blocks: 16-token segments with 256-bit loads
  const bool defer = W <= 2 * B && B <= 16;  // every flagged segment fits one 16-token task
  // prompt metadata of prompts pbase .. pbase+32 held in lanes (so = first block, st = first
  // token); reloaded only when a chunk reaches past it
  uint32_t pbase = 0xffffffffu, so = 0, so32 = 0;
  uint64_t st = 0, st32 = 0;
  while (g < G1) {
    if (pp < pbase || pp >= pbase + 31 || (so32 <= g + 31 && pbase + 32 < N && pp > pbase)) {
      pbase = pp;
      const uint32_t pl = min(pp + lane, N), p32 = min(pp + 32, N);
      so = a.blk_off[pl];
      st = a.tok_off[pl];
      so32 = a.blk_off[p32];
      st32 = a.tok_off[p32];
    }
    const uint32_t d = pp - pbase;  // lane of prompt pp
    // ---- chunk: up to 32 consecutive blocks within the loaded prompts
    uint32_t nw = min(32u, G1 - g);
    if (pbase + 32 <= N) nw = min(nw, so32 - g);
    const uint32_t lastg = g + nw - 1;
    // prompt starts inside the chunk (lanes > d whose first block is <= lastg)
    const uint32_t starts = __ballot_sync(kFull, lane > d && so <= lastg);
    const uint32_t il = __popc(starts);
    // windows >= nout are helpers: their phase A/B results serve the windows before
    // them, and they are redone as the first windows of the next chunk
    const uint32_t nout = (g + nw == G1 || nw <= 2) ? nw : nw - 2;
    const uint32_t gb = g + lane;
    uint32_t i, bm;  // prompt lane of this window; bit w = a prompt starts at window w
    if (il == 0) {   // the whole chunk lies in prompt pp
      i = d;
      bm = 0;
    } else {
      const uint32_t pos = ((starts >> lane) & 1u) ? so - g : 32u;
      bm = __reduce_or_sync(kFull, pos < 32 ? 1u << pos : 0u);
      if (__popc(bm) == il) {  // distinct starts (no empty prompt inside the chunk)
        i = d + __popc(bm & (0xffffffffu >> (31 - lane)));
      } else {
        i = d;
#pragma unroll
        for (uint32_t s = 16; s >= 1; s >>= 1) {
          const uint32_t v = __shfl_sync(kFull, so, min(i + s, 31u));
          if (i + s <= d + il && v <= gb) i += s;
        }
      }
    }
    // token positions relative to T0 = the chunk's first window start (32-bit)
    const uint64_t T0 = shfl64(st, d) + static_cast<uint64_t>(g - __shfl_sync(kFull, so, d)) * B;
    const uint32_t* __restrict__ tk0 = tokens + T0;
    const uint32_t rel = static_cast<uint32_t>(st - T0), rel32 = static_cast<uint32_t>(st32 - T0);
    const uint32_t i1 = min(i + 1, 31u);
    const uint32_t r_i = __shfl_sync(kFull, rel, i), r_1 = __shfl_sync(kFull, rel, i1);
    const uint32_t so_i = __shfl_sync(kFull, so, i);
    const uint32_t r_i1 = i + 1 < 32 ? r_1 : rel32;  // end of prompt pbase + i
    const uint32_t b = gb - so_i, p = pbase + i;
    const uint32_t ws = r_i + b * B;
    const uint32_t we = min(r_i1, ws + B + W);
    const bool act = lane < nw, out = lane < nout;
    const bool nbr = lane + 1 < nw && !((bm >> (lane + 1)) & 1u);  // block b+1: same prompt, this chunk
#if SKV_HS_L1PF == 2
    l1_prefetch_next(tokens, a.n_tokens, T0, nout, lane, B, W);
#endif
    // ---- phase A: the block's tokens, digest, DFA over the block from the start state
    uint32_t A = 0, X = 0, Z = 0, SW = 0, amid = 0, cw0 = 0;
    if (act) {
      uint64_t dg = a.digest_init;
      const uint32_t al = static_cast<uint32_t>(T0) + ws;  // alignment of the absolute position
      if (b16 && (al & 3) == 0) {
        uint32_t t[16];
        ldg_tokens16(tk0 + ws, t, (al & 7) == 0);
        uint32_t any = 0;
#pragma unroll
        for (uint32_t k = 0; k < 16; ++k) any |= t[k];
        if (any >> 8) {  // a token >= 256: full update_u32 digest, low bytes for the scan
#pragma unroll 1
          for (uint32_t k = 0; k < 16; ++k) dg = fnv_u32(dg, tk0[ws + k]);
#pragma unroll
          for (uint32_t k = 0; k < 16; ++k) t[k] &= 0xffu;
        }
        uint32_t c[16];
#pragma unroll
        for (uint32_t k = 0; k < 16; ++k) c[k] = cmap[t[k]];
        // digest and DFA are independent chains in one basic block
        uint64_t h = a.digest_init;
        uint32_t row = start_row, alo = 0;
#pragma unroll
        for (uint32_t k = 0; k < 16; ++k) {
          h = fnv_tok(h, t[k]);
          row = lds16(tab, row + c[k]);
          if (k < 4) {
            alo |= row;
          } else {
            amid |= row;
          }
          if (k == 3) Z = row;
        }
        if (!(any >> 8)) dg = h;
        X = SW = row;
        A = alo | amid;
        cw0 = c[0] | (c[1] << 8) | (c[2] << 16) | (c[3] << 24);
      } else if (bseg && (al & 3) == 0) {
        // B = 16k: the block in 16-token segments (two 256-bit loads each), byte-token FNV
        // steps; a segment with a token >= 256 switches the digest to update_u32 over the
        // whole block (recomputed after the run)
        uint64_t h = a.digest_init;
        bool wide = false;
        uint32_t row = start_row;
        for (uint32_t k0 = 0; k0 < B; k0 += 16) {
          uint32_t t[16];
          ldg_tokens16(tk0 + ws + k0, t, ((al + k0) & 7) == 0);
          uint32_t any = 0;
#pragma unroll
          for (uint32_t k = 0; k < 16; ++k) any |= t[k];
          if (any >> 8) {
            wide = true;
#pragma unroll
            for (uint32_t k = 0; k < 16; ++k) t[k] &= 0xffu;
          }
#pragma unroll
          for (uint32_t k = 0; k < 16; ++k) {
            const uint32_t gk = k0 + k;
            if (!wide) h = fnv_tok(h, t[k]);
            const uint32_t ck = cmap[t[k]];
            row = lds16(tab, row + ck);
            if (gk < kc) {
              A |= row;
            } else if (gk < Wp) {
              amid |= row;
            } else {
              A |= row;
            }
            if (gk + 1 == kc) Z = row;
            if (gk + 1 == Wp) SW = row;
            if (gk < 4) cw0 |= ck << (8 * gk);
          }
        }
        if (wide) {
#pragma unroll 1
          for (uint32_t k = 0; k < B; ++k) dg = fnv_u32(dg, tk0[ws + k]);
        } else {
          dg = h;
        }
        if (kc == 0) Z = start_row;
        if (Wp == 0) SW = start_row;
        X = row;
        A |= amid;
      } else {  // generic shape / alignment: token by token
        uint32_t row = start_row;
        for (uint32_t k = 0; k < B; ++k) {
          const uint32_t tv = tk0[ws + k];
          dg = fnv_u32(dg, tv);
          const uint32_t ck = cmap[tv & 0xffu];
          row = lds16(tab, row + ck);
          if (k < kc) {
            A |= row;
          } else if (k < Wp) {
            amid |= row;
          } else {
            A |= row;
          }
          if (k + 1 == kc) Z = row;
          if (k + 1 == Wp) SW = row;
          if (k < 4) cw0 |= ck << (8 * k);
        }
        if (kc == 0) Z = start_row;
        if (Wp == 0) SW = start_row;
        X = row;
        A |= amid;
      }
      if (out && a.first) a.d_out[gb] = dg;
    }
#if SKV_HS_L1PF == 1
    l1_prefetch_next(tokens, a.n_tokens, T0, nout, lane, B, W);
#endif
    // ---- phase B: [ws+B, min(we, ws+B+W')), shared with window l+1 once the runs meet
    const uint32_t nZ = __shfl_down_sync(kFull, Z | ((amid & kAccRegion) << 1), 1);
    const uint32_t nSW = __shfl_down_sync(kFull, SW, 1);
    const uint32_t nX = __shfl_down_sync(kFull, X, 1);
    const uint32_t ncw = __shfl_down_sync(kFull, cw0, 1);  // the next block's first classes
    uint32_t Y = X, C = 0;
    const uint32_t sb = ws + B, eb = min(we, ws + B + Wp);
    if (act && lane <= nout && sb < eb) {  // window nout's run serves window nout-1's phase C
      if (nbr && kc == kConv) {
        uint32_t ac = 0;
        const uint32_t V = step4(tab, X, ncw, ac);
        if (V == (nZ & 0xffffu)) {
          C = ac | (nZ >> 1);  // bit 16 (neighbour's rows over [kConv, W')) -> bit 15
          Y = nSW;
        } else {
          Y = run_tokens(tab, cmap, tk0, sb + kConv, eb, V, C);
          C |= ac;
        }
      } else {
        Y = run_tokens(tab, cmap, tk0, sb, eb, X, C);
      }
    }
    // ---- phase C: [ws+2B, we) (W > B); end-of-window transition; flags
    const uint32_t Cf = C & kAccRegion;
    const uint32_t nYC = __shfl_down_sync(kFull, Y | (Cf << 1), 1);
    uint32_t f = 0;
    const uint32_t sc = ws + 2 * B;
    if (out) {
      uint32_t fin = Y, C2 = 0;
      if (W > B && sc < we) {
        if (W == 2 * B && nbr && Y == nX) {
          C2 = nYC >> 1;
          fin = nYC & 0xffffu;
        } else {
          fin = run_tokens(tab, cmap, tk0, sc, we, Y, C2);
        }
      }
      const uint32_t me = copy_mask(acc_tab, lds16(tab, fin + eos2), inv);  // end-of-window transition
      if (a.first)
        a.mask_out[gb] = me;
      else if (me)
        atomicOr(&a.mask_out[gb], me << a.mask_shift);  // a later rule group (bits shifted to its rules)
      if (me) atomicMin(&a.first_sens[p], b);
      f = ((A & kAccRegion) ? 1u : 0u) | (Cf ? 2u : 0u) | ((C2 & kAccRegion) ? 4u : 0u);
    }
    // ---- exact rule masks of the flagged segments (segment s of a window: 0 = block,
    // 1 = phase B, 2 = phase C).  Deferred: every flagged segment gets a queue slot
    // (rank = exclusive prefix of the per-lane counts, one pass); the queue runs 32
    // tasks per lane-pass once full.  In place: segments longer than 16 tokens, or a
    // chunk with more flagged segments than the queue holds.
    if (__any_sync(kFull, f != 0)) {
      const uint32_t cnt = __popc(f);
      const uint32_t c0 = __ballot_sync(kFull, cnt & 1u), c1 = __ballot_sync(kFull, cnt >> 1);
      const uint32_t tot = __popc(c0) + 2 * __popc(c1);
      const bool queue = defer && tot <= kQCap;
      if (queue && qn + tot > kQCap) {
        flush_tasks(q, qn, lane, tab, cmap, acc_tab, inv, a);
        qn = 0;
      }
      const uint32_t lt = (1u << lane) - 1u;
      uint32_t k = qn + __popc(c0 & lt) + 2 * __popc(c1 & lt);
      for (uint32_t ff = f; ff; ff &= ff - 1) {
        const uint32_t sg = __ffs(ff) - 1;
        uint32_t o, e, row;
        if (sg == 0) {
          o = ws, e = ws + B, row = start_row;
        } else if (sg == 1) {
          o = sb, e = eb, row = X;
        } else {
          o = sc, e = we, row = Y;
        }
        if (queue) {
          SegTask t;
          t.tok = T0 + o;
          t.meta = row | ((e - o) << 16);
          t.gb = gb, t.p = p, t.b = b, t.pad = 0;
          q[k++] = t;
        } else {
          uint32_t m = 0;
          for (; o < e; ++o) {
            row = lds16(tab, row + cmap[tk0[o] & 0xffu]);
            m |= copy_mask(acc_tab, row, inv);
          }
          if (m) {
            atomicOr(&a.mask_out[gb], m << a.mask_shift);
            atomicMin(&a.first_sens[p], b);
          }
        }
      }
      if (queue) qn += tot;
    }
    // ---- next chunk
    g += nout;
    pp = pbase + d + __popc(__ballot_sync(kFull, lane > d && so <= g));  // last loaded prompt start <= g
    if (pp == pbase + 31 && pbase + 32 <= N && so32 <= g) {  // past the loaded prompts
      pp = pbase + 32;
      while (pp < N && a.blk_off[pp + 1] <= g) ++pp;
    }
  }
  flush_tasks(q, qn, lane, tab, cmap, acc_tab, inv, a);
}

#include "hash_scan16.cuh"

// find_slot: used by set_tiers (point lookups of block b, group leader key (hL, dL))
__device__ __forceinline__ uint32_t find_slot(const Index& ix, uint64_t h, uint64_t d, uint64_t hL, uint64_t dL,
                                              uint32_t b, Rec* out) {
  uint64_t s = home_slot(ix, hL, dL, b);
  for (uint64_t i = 0; i <= ix.mask; ++i) {
    const ulonglong2* rp = reinterpret_cast<const ulonglong2*>(&ix.e[s].rec);
    ulonglong2 k = rp[0];
    if (k.x == h && k.y == d) {
      *out = ix.e[s].rec;
      return meta_live(out->meta) ? static_cast<uint32_t>(s) : kNone;  // a tombstone is missing
    }
    if (k.x == 0 && k.y == 0) return kNone;
    s = (s + 1) & ix.mask;
  }
  return kNone;
}

__device__ __forceinline__ bool cas128(unsigned long long* addr, unsigned long long cmp_lo, unsigned long long cmp_hi,
                                       unsigned long long new_lo, unsigned long long new_hi,
                                       unsigned long long* old_lo, unsigned long long* old_hi) {
  asm volatile(
      "{\n\t.reg .b128 c, n, d;\n\t"
      "mov.b128 c, {%2, %3};\n\t"
      "mov.b128 n, {%4, %5};\n\t"
      "atom.global.cas.b128 d, [%6], c, n;\n\t"
      "mov.b128 {%0, %1}, d;\n\t}"
      : "=l"(*old_lo), "=l"(*old_hi)
      : "l"(cmp_lo), "l"(cmp_hi), "l"(new_lo), "l"(new_hi), "l"(addr)
      : "memory");
  return *old_lo == cmp_lo && *old_hi == cmp_hi;
}

// ---------------------------------------------------------------------------------
// Monitor record (A.6, AccessStats::record access_stats.hpp:27-37), fused into the probe.
//
// hit_cur is order-independent: one atomic per access.  The distinct-user count is
// order-dependent only for an entry whose tracked set crosses 64 users within the
// batch (which 64 get admitted depends on prompt order).  So every access inserts its
// user into the entry's set table (128-bit CAS); a set that was already full (64
// admitted users) counts every non-member access directly, again order-independent.
// k_record_finish then applies the distinct-insert count of every touched entry whose
// set did not cross 64 in this batch; the rare crossing entries are replayed in prompt
// order by k_record_replay.
// ---------------------------------------------------------------------------------
// the batch / window stamps of a graph-replayed step from the device step state (MonCtx::st)
__device__ __forceinline__ MonCtx mon_live(MonCtx M) {
  if (M.st) {
    const uint32_t cur = M.st[2];
    M.batch = M.st[0];
    M.wstart = M.st[1];
    M.touched = cur ? M.tl[1] : M.tl[0];  // a select, not a dynamic index (that would put M in local memory)
    M.n_touched = M.ntb + (cur ? 1 : 0);
  }
  return M;
}

__device__ __forceinline__ uint32_t mix32(uint64_t u) {
  u ^= u >> 33;
  u *= 0xff51afd7ed558ccdULL;
  u ^= u >> 33;
  return static_cast<uint32_t>(u);
}

__device__ __forceinline__ ulonglong2 ld_relaxed128(const ulonglong2* p) {
  ulonglong2 v;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p) : "memory");
  return v;
}

// Two independent 128-bit claims (compare with empty = 0) issued back to back in one asm
// block: the results are copied out only after both are in flight (separate asm
// statements let the register allocator place a copy of the first result -- a wait on
// its DRAM round trip -- before the second CAS).  Predicated off -> old = all ones.
__device__ __forceinline__ void cas128_empty_x2(unsigned long long* a0, unsigned long long* a1, bool p0, bool p1,
                                                unsigned long long n0l, unsigned long long n0h,
                                                unsigned long long n1l, unsigned long long n1h,
                                                unsigned long long* o0l, unsigned long long* o0h,
                                                unsigned long long* o1l, unsigned long long* o1h) {
  asm volatile(
      "{\n\t.reg .pred q0, q1;\n\t.reg .b128 z, d0, d1, n0, n1;\n\t"
      "setp.ne.u32 q0, %4, 0;\n\t"
      "setp.ne.u32 q1, %5, 0;\n\t"
      "mov.b128 z, {0, 0};\n\t"
      "mov.b128 d0, {-1, -1};\n\t"
      "mov.b128 d1, {-1, -1};\n\t"
      "mov.b128 n0, {%6, %7};\n\t"
      "mov.b128 n1, {%8, %9};\n\t"
      "@q0 atom.global.cas.b128 d0, [%10], z, n0;\n\t"
      "@q1 atom.global.cas.b128 d1, [%11], z, n1;\n\t"
      "mov.b128 {%0, %1}, d0;\n\t"
      "mov.b128 {%2, %3}, d1;\n\t}"
      : "=l"(*o0l), "=l"(*o0h), "=l"(*o1l), "=l"(*o1h)
      : "r"(static_cast<uint32_t>(p0)), "r"(static_cast<uint32_t>(p1)), "l"(n0l), "l"(n0h), "l"(n1l), "l"(n1h),
        "l"(a0), "l"(a1)
      : "memory");
}

__device__ __forceinline__ bool cas128_dev(ulonglong2* addr, ulonglong2 cmp, ulonglong2 val, ulonglong2* old) {
  return cas128(reinterpret_cast<unsigned long long*>(addr), cmp.x, cmp.y, val.x, val.y, &old->x, &old->y);
}

// pool slot of the entry's set for this window (allocated on first touch)
__device__ __forceinline__ uint32_t acquire_set(Entry& e, uint32_t slot, const MonCtx& M) {
  volatile uint32_t* sp = &e.aux.set_idx;
  uint32_t si = *sp;
  if (si < kPendingSet) return si;
  if (si == kNone && atomicCAS(const_cast<uint32_t*>(sp), kNone, kPendingSet) == kNone) {
    si = atomicAdd(M.pool_count, 1u);
    if (si >= M.pool_cap) {
      atomicOr(M.err, 1u);
      atomicExch(const_cast<uint32_t*>(sp), kNone);
      return kNone;
    }
    SetHdr& h = M.hdr[si];
    h.size = 0;
    h.touch = 0;
    h.ovf = 0;
    h.cnt = 0;
    M.touched[atomicAdd(M.n_touched, 1u)] = slot;
    __threadfence();
    atomicExch(const_cast<uint32_t*>(sp), si);
    return si;
  }
  while ((si = *sp) == kPendingSet) {
  }
  return si;
}

__device__ __forceinline__ uint32_t count_insert(unsigned long long* cnt, uint32_t batch) {
  unsigned long long old = *reinterpret_cast<volatile unsigned long long*>(cnt);
  for (;;) {
    const unsigned long long nv = (static_cast<uint32_t>(old >> 32) == batch)
                                      ? old + 1
                                      : ((static_cast<unsigned long long>(batch) << 32) | 1ull);
    const unsigned long long got = atomicCAS(cnt, old, nv);
    if (got == old) return static_cast<uint32_t>(nv);
    old = got;
  }
}

// the distinct-user part of AccessStats::record (the hit count is applied by the caller)
__device__ void record_user(const Index& ix, const MonCtx& M, uint32_t slot, uint64_t user) {
  Entry& e = ix.e[slot];
  const uint32_t si = acquire_set(e, slot, M);
  if (si == kNone) return;
  SetHdr& hd = M.hdr[si];
  const uint32_t size = *reinterpret_cast<volatile uint32_t*>(&hd.size);
  ulonglong2* tab = M.tab + static_cast<uint64_t>(si) * kSetSlots;
  uint32_t pos = mix32(user) & (kSetSlots - 1);
  for (uint32_t i = 0; i < kSetSlots;) {
    const ulonglong2 v = ld_relaxed128(&tab[pos]);
    const bool live = v.y >= M.wstart;
    if (live && v.x == user) return;  // tracked already (access_stats.hpp:30)
    if (live) {
      pos = (pos + 1) & (kSetSlots - 1);
      ++i;
      continue;
    }
    if (size >= kMaxSetUsers) {  // saturated: an untracked user counts as new (access_stats.hpp:33)
      atomicAdd(&e.stats.u_cnt, 1u);
      return;
    }
    ulonglong2 old;
    if (cas128_dev(&tab[pos], v, make_ulonglong2(user, M.batch), &old)) {
      if (size + count_insert(&hd.cnt, M.batch) > kMaxSetUsers) atomicExch(&hd.ovf, M.batch);
      return;
    }
    // lost the slot to a concurrent insert: re-examine the same position
  }
  atomicExch(&hd.ovf, M.batch);  // table full: resolve by ordered replay
}

// one thread per entry touched in the current monitor window
__global__ void k_record_finish(Index ix, MonCtx M, uint32_t* replay, uint32_t* n_replay) {
  M = mon_live(M);
  const uint32_t n = *M.n_touched;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t slot = M.touched[i];
    Entry& e = ix.e[slot];
    SetHdr& hd = M.hdr[e.aux.set_idx];
    if (hd.ovf == M.batch) {
      replay[atomicAdd(n_replay, 1u)] = slot;
      continue;
    }
    const uint32_t c = static_cast<uint32_t>(hd.cnt >> 32) == M.batch ? static_cast<uint32_t>(hd.cnt) : 0u;
    e.stats.u_cnt += c;
    hd.size += c;
  }
}

// A.6 record, one warp per prompt, lanes = its matched blocks (order-independent part)
// Warp = prompt, lanes = its matched blocks, kRecRounds x 32 accesses with their
// dependent loads in flight together.  Fast path (the common case once an entry's set
// exists): the user already sits at its home position of the set table -> nothing but
// the hit count changes.  Everything else takes the full record_user path.
#ifndef SKV_KRECROUNDS
#define SKV_KRECROUNDS 1
#endif
constexpr int kRecRounds = SKV_KRECROUNDS;

// replicated layer: an access to an entry at depth < rep.depth is aggregated per (entry, user)
// -- lowest prompt of the batch and count -- for the cross-rank merge instead of being recorded
__device__ void rep_pair_add(const RepLayer& R, uint32_t slot, uint64_t user, uint32_t p) {
  const ulonglong2 key = make_ulonglong2(user, static_cast<unsigned long long>(slot) + 1);
  uint32_t h = (mix32(user ^ (static_cast<uint64_t>(slot) << 32)) ^ slot * 0x9e3779b9u) & R.pair_mask;
  for (uint32_t i = 0; i <= R.pair_mask; ++i, h = (h + 1) & R.pair_mask) {
    ulonglong2 cur = ld_relaxed128(&R.pair_key[h]);
    if (cur.x == 0 && cur.y == 0) {
      ulonglong2 old;
      cas128_dev(&R.pair_key[h], make_ulonglong2(0, 0), key, &old);
      cur = old.x == 0 && old.y == 0 ? key : old;
    }
    if (cur.x == key.x && cur.y == key.y) {
      atomicMin(&R.pair_first[h], p);
      atomicAdd(&R.pair_cnt[h], 1u);
      return;
    }
  }
  atomicOr(R.err, 1u);
}

__device__ __forceinline__ void record_prompt(const Index& ix, const MonCtx& M, const uint32_t* __restrict__ slot_in,
                                              uint32_t bo, uint32_t m, uint64_t u, uint32_t lane, uint32_t p) {
  const uint32_t pos = mix32(u) & (kSetSlots - 1);
  const uint32_t rd = min(ix.rep.depth, m);
  for (uint32_t b = lane; b < rd; b += 32) rep_pair_add(ix.rep, slot_in[bo + b], u, p);
  bo += rd;
  m -= rd;
  for (uint32_t base = 0; base < m; base += 32 * kRecRounds) {
    uint32_t sl[kRecRounds], si[kRecRounds];
#pragma unroll
    for (int r = 0; r < kRecRounds; ++r) {
      const uint32_t b = base + 32 * r + lane;
      sl[r] = b < m ? slot_in[bo + b] : kNone;
    }
#pragma unroll
    for (int r = 0; r < kRecRounds; ++r)
      if (sl[r] != kNone) {
        atomicAdd(&ix.e[sl[r]].stats.hit_cur, 1u);
        si[r] = *reinterpret_cast<volatile uint32_t*>(&ix.e[sl[r]].aux.set_idx);
      }
    ulonglong2 v[kRecRounds];
#pragma unroll
    for (int r = 0; r < kRecRounds; ++r) {
      v[r] = make_ulonglong2(0, 0);
      if (sl[r] != kNone && si[r] < kPendingSet) v[r] = ld_relaxed128(&M.tab[static_cast<uint64_t>(si[r]) * kSetSlots + pos]);
    }
#pragma unroll
    for (int r = 0; r < kRecRounds; ++r)
      if (sl[r] != kNone && !(si[r] < kPendingSet && v[r].x == u && v[r].y >= M.wstart))
        record_user(ix, M, sl[r], u);
  }
}

__global__ void __launch_bounds__(256) k_record(Index ix, MonCtx M, const uint32_t* __restrict__ slot_in,
                                                const uint32_t* __restrict__ blk_off,
                                                const uint32_t* __restrict__ matched,
                                                const uint64_t* __restrict__ users, uint32_t n_prompts) {
  const uint32_t p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (p >= n_prompts) return;
  record_prompt(ix, M, slot_in, blk_off[p], matched[p], users[p], lane_id(), p);
}

// accesses (slot << 32 | prompt) of the entries that need an ordered replay
__global__ void k_replay_emit(Index ix, MonCtx M, const uint32_t* __restrict__ slot_in,
                              const uint32_t* __restrict__ blk_off, const uint32_t* __restrict__ matched,
                              uint32_t n_prompts, unsigned long long* keys, uint32_t* n_keys) {
  const uint32_t p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (p >= n_prompts) return;
  const uint32_t bo = blk_off[p], m = matched[p];
  for (uint32_t b = ix.rep.depth + lane_id(); b < m; b += 32) {  // replicated entries: merged, not recorded
    const uint32_t s = slot_in[bo + b];
    if (M.hdr[ix.e[s].aux.set_idx].ovf == M.batch)
      keys[atomicAdd(n_keys, 1u)] = (static_cast<unsigned long long>(s) << 32) | p;
  }
}

// One warp per replayed entry: the batch's accesses in prompt order against the set as
// it stood before the batch, exactly as AccessStats::record (register-resident set,
// __match_any_sync for repeats within a 32-access chunk); then rebuild the table.
__global__ void __launch_bounds__(256) k_record_replay(Index ix, MonCtx M, const uint32_t* __restrict__ replay,
                                                       const uint32_t* __restrict__ n_replay,
                                                       const unsigned long long* __restrict__ keys, uint32_t n_keys,
                                                       const uint64_t* __restrict__ users) {
  const uint32_t lane = lane_id();
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < *n_replay; r += nw) {
    const uint32_t slot = replay[r];
    Entry& e = ix.e[slot];
    const uint32_t si = e.aux.set_idx;
    SetHdr& hd = M.hdr[si];
    ulonglong2* tab = M.tab + static_cast<uint64_t>(si) * kSetSlots;
    // pre-batch members (live stamps < batch), compacted into lanes: m0 = member lane, m1 = lane + 32
    unsigned long long m0 = 0, m1 = 0, s0 = 0, s1 = 0;
    uint32_t size = 0;
    for (uint32_t base = 0; base < kSetSlots; base += 32) {
      const ulonglong2 v = tab[base + lane];
      const bool pre = v.y >= M.wstart && v.y < M.batch;
      const uint32_t bal = __ballot_sync(kFull, pre);
      for (uint32_t src = 0; src < 32; ++src) {
        if (!(bal >> src & 1u)) continue;
        const uint32_t rk = size + __popc(bal & ((1u << src) - 1u));
        const unsigned long long ux = __shfl_sync(kFull, v.x, src), sy = __shfl_sync(kFull, v.y, src);
        if (lane == (rk & 31)) {
          if (rk < 32) {
            m0 = ux;
            s0 = sy;
          } else if (rk < 64) {
            m1 = ux;
            s1 = sy;
          }
        }
      }
      size += __popc(bal);
    }
    size = min(size, kMaxSetUsers);
    // this entry's accesses: [lo, hi) in the sorted key list
    const unsigned long long k0 = static_cast<unsigned long long>(slot) << 32;
    uint32_t lo = 0, hi = n_keys;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (keys[mid] < k0) lo = mid + 1; else hi = mid;
    }
    uint32_t end = lo, top = n_keys;
    while (end < top) {
      const uint32_t mid = (end + top) >> 1;
      if ((keys[mid] >> 32) <= slot) end = mid + 1; else top = mid;
    }
    const uint32_t size0 = size;
    uint32_t add_total = 0;
    for (uint32_t c0 = lo; c0 < end; c0 += 32) {
      const uint32_t i = c0 + lane;
      const bool valid = i < end;
      const unsigned long long u = valid ? users[static_cast<uint32_t>(keys[i])] : 0ull;
      bool member = false;
      for (uint32_t j = 0; j < size; ++j) {
        const unsigned long long mj = __shfl_sync(kFull, j < 32 ? m0 : m1, j & 31);
        member |= (mj == u);
      }
      const bool nonmem = valid && !member;
      const uint32_t nm_mask = __ballot_sync(kFull, nonmem);
      const uint32_t peers = __match_any_sync(kFull, u) & nm_mask;
      const uint32_t leader = nonmem ? static_cast<uint32_t>(__ffs(peers) - 1) : 0u;
      const bool is_leader = nonmem && leader == lane;
      const uint32_t leaders = __ballot_sync(kFull, is_leader);
      const uint32_t room = kMaxSetUsers - size;
      const uint32_t lrank = __popc(leaders & ((1u << leader) - 1u));
      const bool admitted = nonmem && lrank < room;
      add_total += nonmem ? (admitted ? (is_leader ? 1u : 0u) : 1u) : 0u;
      uint32_t adm = __ballot_sync(kFull, is_leader && admitted);
      uint32_t pos = size;
      while (adm) {
        const uint32_t ll = __ffs(adm) - 1;
        adm &= adm - 1;
        const unsigned long long v = __shfl_sync(kFull, u, ll);
        if (lane == (pos & 31)) {
          if (pos < 32) {
            m0 = v;
            s0 = M.batch;
          } else {
            m1 = v;
            s1 = M.batch;
          }
        }
        ++pos;
      }
      size = pos;
    }
    add_total = __reduce_add_sync(kFull, add_total);
    // rebuild the table with exactly the admitted users
    for (uint32_t base = 0; base < kSetSlots; base += 32) tab[base + lane] = make_ulonglong2(0ull, 0ull);
    __syncwarp();
    for (uint32_t j = 0; j < size; ++j) {
      const unsigned long long u = __shfl_sync(kFull, j < 32 ? m0 : m1, j & 31);
      const unsigned long long st = __shfl_sync(kFull, j < 32 ? s0 : s1, j & 31);
      if (lane == 0) {
        uint32_t pos = mix32(u) & (kSetSlots - 1);
        while (tab[pos].y != 0) pos = (pos + 1) & (kSetSlots - 1);
        tab[pos] = make_ulonglong2(u, st);
      }
    }
    if (lane == 0) {
      e.stats.u_cnt += add_total;
      hd.size = size;
    }
    (void)size0;
  }
}

// ---------------------------------------------------------------------------------
// K3: chained prefix keys + inherited labels + warp-cooperative index probe, fused.
//
// A warp owns 32 consecutive prompts.  For each 32-block tile it
//   1. stages the tile's block digests HBM -> SMEM (one coalesced 256-B load per prompt);
//   2. runs the serial FNV chain lane-per-prompt (A.2: SIMD across prompts, the chain
//      is serial along one prompt) and the prefix-OR label (A.4);
//   3. writes keys and labels back coalesced;
//   4. probes the tile for every prompt whose commit point is still unknown: lanes =
//      32 consecutive blocks, up to 4 prompts' first-slot loads in flight per lane;
//      ballots give the first invisible block (match length m, A.5: label == Public
//      or creator == user, cache_index.hpp:483-485) and the first missing block (k,
//      where the commit starts).  Probing stops at the tile holding the first miss.
// ---------------------------------------------------------------------------------
#ifndef SKV_KCPWARPS
#define SKV_KCPWARPS 2
#endif
constexpr int kCPWarps = SKV_KCPWARPS;     // warps per CTA (8.4 KB of SMEM tiles each)
#ifndef SKV_KCPPROMPTS
#define SKV_KCPPROMPTS 16
#endif
constexpr int kCPPrompts = SKV_KCPPROMPTS;  // prompts per warp: 4096 warps for config 2 (latency-bound chain + probes)
#ifndef SKV_KCPINFLIGHT
#define SKV_KCPINFLIGHT 8
#endif
constexpr int kCPInFlight = SKV_KCPINFLIGHT;  // prompts whose probe loads are in flight together

constexpr int kPitch = 33;  // u64 per SMEM tile row (odd pitch: conflict-free transposes)

struct Probe {
  uint32_t slot;
  uint32_t creator;  // interned user index
  uint32_t meta;     // Rec::meta
};

__device__ __forceinline__ Probe probe_resolve(const Index& ix, uint64_t h, uint64_t d, uint64_t s, ulonglong2 k,
                                               ulonglong2 m) {
  for (uint64_t i = 0; i <= ix.mask; ++i) {
    if (k.x == h && k.y == d)
      return Probe{static_cast<uint32_t>(s), static_cast<uint32_t>(m.x), static_cast<uint32_t>(m.x >> 32)};
    if (k.x == 0 && k.y == 0) break;
    s = (s + 1) & ix.mask;
    const ulonglong2* rp = reinterpret_cast<const ulonglong2*>(&ix.e[s].rec);
    k = rp[0];
    m = rp[1];
  }
  return Probe{kNone, 0, 0};
}

#ifndef SKV_KCP_MINB
#define SKV_KCP_MINB 1
#endif
#ifndef SKV_KCP_GRID_PER_SM
#define SKV_KCP_GRID_PER_SM 0  // > 0: at most this many CTAs per SM; warps stride over prompt groups
#endif
// Chained keys (A.2) for a prefetched batch, on the side stream while the previous batch
// commits: warp = 32 prompts, lane = prompt, its serial FNV chain (16 byte-steps per
// block) with all 32 lanes busy; digest tiles in and key tiles out coalesced through an
// SMEM transpose (the chain overwrites each digest cell with its key).  Also the labels
// (prefix-OR from the first sensitive block) and the probe's slot initialisation, so the
// probe of that batch (k_chain_probe<true>) is lookups only.
constexpr int kCHWarps = 4;
__global__ void __launch_bounds__(kCHWarps * 32) k_chain(const uint64_t* __restrict__ dk,
                                                         const uint32_t* __restrict__ blk_off,
                                                         const uint32_t* __restrict__ first_sens, uint32_t n_prompts,
                                                         uint64_t* __restrict__ hk, uint8_t* __restrict__ label,
                                                         uint32_t* __restrict__ slot_out) {
  __shared__ uint64_t s_t[kCHWarps][32][kPitch];
  const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
  const uint32_t p0 = (blockIdx.x * kCHWarps + wid) * 32;
  if (p0 >= n_prompts) return;
  const uint32_t p = p0 + lane;
  const bool has = p < n_prompts;
  const uint32_t bo = has ? blk_off[p] : 0, n = has ? blk_off[p + 1] - bo : 0;
  const uint32_t fs = has ? first_sens[p] : 0;
  uint64_t (*t)[kPitch] = s_t[wid];
  uint64_t h = 0;
  const uint32_t nmax = __reduce_max_sync(kFull, n);
  for (uint32_t t0 = 0; t0 < nmax; t0 += 32) {
    const uint32_t b = t0 + lane;
    for (uint32_t j = 0; j < 32; ++j) {
      const uint32_t bj = __shfl_sync(kFull, bo, j), nj = __shfl_sync(kFull, n, j);
      if (b < nj) {
        const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&t[j][lane]));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(dk + bj + b) : "memory");
      }
    }
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    const uint32_t cnt = n > t0 ? min(32u, n - t0) : 0u;
    for (uint32_t c = 0; c < cnt; ++c) {
      h = chain_key(h, t[lane][c]);
      t[lane][c] = h;
    }
    __syncwarp();
    for (uint32_t j = 0; j < 32; ++j) {
      const uint32_t bj = __shfl_sync(kFull, bo, j), nj = __shfl_sync(kFull, n, j);
      const uint32_t fsj = __shfl_sync(kFull, fs, j);
      if (b < nj) {
        hk[bj + b] = t[j][lane];
        label[bj + b] = b >= fsj ? SKV_LABEL_PRIVATE : SKV_LABEL_PUBLIC;
        slot_out[bj + b] = kNone;
      }
    }
    __syncwarp();
  }
}

template <bool kPre>  // kPre: keys, labels and slot init come from k_chain (the prefetch stage)
__global__ void __launch_bounds__(kCPWarps * 32, SKV_KCP_MINB) k_chain_probe(
    Index ix, const uint64_t* __restrict__ dk, const uint32_t* __restrict__ blk_off,
    const uint32_t* __restrict__ first_sens, const uint32_t* __restrict__ uidx, uint32_t n_prompts,
    uint64_t* __restrict__ hk, uint8_t* __restrict__ label, uint8_t* __restrict__ decision,
    uint32_t* __restrict__ slot_out, uint32_t* __restrict__ matched, uint32_t* __restrict__ exist,
    uint8_t* __restrict__ tier, uint8_t* __restrict__ bmeta, MonCtx mon, uint32_t* __restrict__ bprompt,
    uint32_t split_from) {
  __shared__ uint64_t s_d[kCPWarps][kCPPrompts][kPitch];
  __shared__ uint64_t s_h[kCPWarps][kCPPrompts][kPitch];
  const uint32_t lane = lane_id(), wid = threadIdx.x >> 5;
  // warp = kCPPrompts prompts; a grid smaller than that strides over the prompt groups
  for (uint32_t p0 = (blockIdx.x * kCPWarps + wid) * kCPPrompts; p0 < n_prompts;
       p0 += gridDim.x * kCPWarps * kCPPrompts) {
  const uint32_t p = p0 + lane;
  const bool has = lane < kCPPrompts && p < n_prompts;
  const uint32_t bo = has ? blk_off[p] : 0, n = has ? blk_off[p + 1] - bo : 0;
  const uint32_t fs = has ? first_sens[p] : 0;
  const uint32_t user = has ? uidx[p] : 0xffffffffu;
  uint64_t (*td)[kPitch] = s_d[wid];
  uint64_t (*th)[kPitch] = s_h[wid];
  uint64_t h = 0;
  uint32_t m = n, k = n, tmax = 0;  // m, k == n: not determined yet
  const uint32_t nmax = __reduce_max_sync(kFull, n);
  for (uint32_t t0 = 0; t0 < nmax; t0 += 32) {
    const uint32_t b = t0 + lane;
    // keys precomputed: tiles past every prompt's first miss are not read at all (config 2:
    // half of the key and digest rows)
    if constexpr (kPre)
      if (!__ballot_sync(kFull, has && k == n && n > t0)) break;
    // all the warp's prompts' digest rows in flight at once (cp.async: global -> SMEM)
    for (uint32_t j = 0; j < kCPPrompts; ++j) {
      const uint32_t bj = __shfl_sync(kFull, bo, j), nj = __shfl_sync(kFull, n, j);
      if (b < nj) {
        const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&td[j][lane]));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(dk + bj + b) : "memory");
        if constexpr (kPre) {
          const uint32_t dsth = static_cast<uint32_t>(__cvta_generic_to_shared(&th[j][lane]));
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dsth), "l"(hk + bj + b) : "memory");
        }
      }
    }
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
    __syncwarp();
    if constexpr (!kPre) {
    const uint32_t cnt = n > t0 ? min(32u, n - t0) : 0u;
    for (uint32_t c = 0; c < cnt; ++c) {
      h = chain_key(h, td[lane][c]);
      th[lane][c] = h;
    }
    __syncwarp();
    for (uint32_t j = 0; j < kCPPrompts; ++j) {
      const uint32_t bj = __shfl_sync(kFull, bo, j), nj = __shfl_sync(kFull, n, j);
      const uint32_t fsj = __shfl_sync(kFull, fs, j);
      if (b < nj) {
        hk[bj + b] = th[j][lane];
        label[bj + b] = b >= fsj ? SKV_LABEL_PRIVATE : SKV_LABEL_PUBLIC;
        slot_out[bj + b] = kNone;  // missing before the batch unless the probe below finds it
#if SKV_COMMIT_FLAT
        bprompt[bj + b] = p0 + j;  // block -> prompt, for the flat commit
#endif
      }
    }
    }  // !kPre
    // tiles from split_from on are probed in two waves of 16 blocks: the second half only for prompts
    // whose first half found no miss, so the tile holding a prompt's first miss wastes at most 15
    // random probes past it instead of 31 (config 2: ~23 -> ~7 per prompt); the host picks split_from
    // from the previous batch's match lengths (capi.cpp probe_split_from)
    const uint32_t waves = t0 >= split_from ? 2u : 1u;
    for (uint32_t half = 0; half < waves; ++half) {
    const uint32_t lo_b = t0 + half * (32 / waves);
    const bool in_half = waves == 1 || (lane >> 4) == half;
    uint32_t todo = __ballot_sync(kFull, has && k == n && n > lo_b);
    while (todo) {
      uint32_t js[kCPInFlight];
      int ng = 0;
#pragma unroll
      for (int q = 0; q < kCPInFlight; ++q) {
        js[q] = todo ? static_cast<uint32_t>(__ffs(todo) - 1) : 32u;
        if (todo) {
          todo &= todo - 1;
          ++ng;
        }
      }
      // issue up to kCPInFlight independent first-slot loads per lane
      ulonglong2 kk[kCPInFlight], mm[kCPInFlight];
      uint64_t ss[kCPInFlight];
#pragma unroll
      for (int q = 0; q < kCPInFlight; ++q) {
        const uint32_t j = js[q] & (kCPPrompts - 1);
        const uint32_t nj = __shfl_sync(kFull, n, j);
        kk[q] = make_ulonglong2(0, 0);
        mm[q] = make_ulonglong2(0, 0);
        ss[q] = 0;
        if (q < ng && b < nj && in_half) {
          ss[q] = home_slot(ix, th[j][lane & ~(kGroup - 1)], td[j][lane & ~(kGroup - 1)], b);
          const ulonglong2* rp = reinterpret_cast<const ulonglong2*>(&ix.e[ss[q]].rec);
          kk[q] = rp[0];
          mm[q] = rp[1];
        }
      }
#pragma unroll
      for (int q = 0; q < kCPInFlight; ++q) {
        if (q >= ng) break;
        const uint32_t j = js[q];
        const uint32_t bj = __shfl_sync(kFull, bo, j), nj = __shfl_sync(kFull, n, j);
        const uint32_t uj = __shfl_sync(kFull, user, j);
        const uint32_t mj = __shfl_sync(kFull, m, j);
        const bool act = b < nj && in_half;
        Probe pr{kNone, 0, 0};
        if (act) pr = probe_resolve(ix, th[j][lane], td[j][lane], ss[q], kk[q], mm[q]);
        const bool found = pr.slot != kNone && meta_live(pr.meta);  // a tombstone is missing
        const uint32_t lab = meta_label(pr.meta);
        const bool vis = found && (lab == SKV_LABEL_PUBLIC || pr.creator == uj);
        const uint32_t nf = __ballot_sync(kFull, act && !found);
        const uint32_t nv = __ballot_sync(kFull, act && !vis);
        const uint32_t new_m = (mj == nj && nv) ? t0 + __ffs(nv) - 1 : mj;
        const uint32_t new_k = nf ? t0 + __ffs(nf) - 1 : nj;
        uint32_t tm = 0;
        if (act) {
          if (b < new_m) {
            decision[bj + b] = lab == SKV_LABEL_PUBLIC ? SKV_PUBLIC_HIT : SKV_OWNER_HIT;
            tm = meta_tier(pr.meta);
            // TTFT epilogue inputs: the matched block's tier and whether the user created it
            bmeta[bj + b] = static_cast<uint8_t>(tm | ((pr.creator == uj) ? 4u : 0u));
          }
          if (b < new_k) slot_out[bj + b] = pr.slot;
        }
        tm = __reduce_max_sync(kFull, tm);
        if (lane == j) {
          m = new_m;
          k = new_k;
          tmax = max(tmax, tm);
        }
      }
    }
    }  // halves
    __syncwarp();
  }
  if (has) {
    matched[p] = m;
    exist[p] = k;
    tier[p] = static_cast<uint8_t>(tmax);
  }
  const uint32_t msum = __reduce_add_sync(kFull, has ? m : 0u);
  if (lane == 0 && msum) atomicAdd(mon.matched_total, msum);
  __syncwarp();
  }  // prompt groups
}

// ---------------------------------------------------------------------------------
// K6: commit (insert the new blocks of the batch).
// ---------------------------------------------------------------------------------

// Four independent 128-bit claims (compare with empty = 0) in one asm block, for 4
// rounds of claims in flight (SKV_COMMIT_ROUNDS=4); see cas128_empty_x2.
constexpr int kClaimQ = 4;
static_assert(kGroup == 1 || !SKV_COMMIT_FLAT, "the flat commit hashes every key on its own");

__device__ __forceinline__ void cas128_empty_x4(const uint64_t* sl, const bool* act, const uint64_t* h,
                                                const uint64_t* d, Entry* e, unsigned long long* ol,
                                                unsigned long long* oh) {
  asm volatile(
      "{\n\t.reg .pred q0, q1, q2, q3;\n\t.reg .b128 z, d0, d1, d2, d3, n0, n1, n2, n3;\n\t"
      "setp.ne.u32 q0, %8, 0;\n\tsetp.ne.u32 q1, %9, 0;\n\tsetp.ne.u32 q2, %10, 0;\n\tsetp.ne.u32 q3, %11, 0;\n\t"
      "mov.b128 z, {0, 0};\n\t"
      "mov.b128 d0, {-1, -1};\n\tmov.b128 d1, {-1, -1};\n\tmov.b128 d2, {-1, -1};\n\tmov.b128 d3, {-1, -1};\n\t"
      "mov.b128 n0, {%12, %13};\n\tmov.b128 n1, {%14, %15};\n\tmov.b128 n2, {%16, %17};\n\tmov.b128 n3, {%18, %19};\n\t"
      "@q0 atom.global.cas.b128 d0, [%20], z, n0;\n\t"
      "@q1 atom.global.cas.b128 d1, [%21], z, n1;\n\t"
      "@q2 atom.global.cas.b128 d2, [%22], z, n2;\n\t"
      "@q3 atom.global.cas.b128 d3, [%23], z, n3;\n\t"
      "mov.b128 {%0, %1}, d0;\n\tmov.b128 {%2, %3}, d1;\n\tmov.b128 {%4, %5}, d2;\n\tmov.b128 {%6, %7}, d3;\n\t}"
      : "=l"(ol[0]), "=l"(oh[0]), "=l"(ol[1]), "=l"(oh[1]), "=l"(ol[2]), "=l"(oh[2]), "=l"(ol[3]), "=l"(oh[3])
      : "r"(static_cast<uint32_t>(act[0])), "r"(static_cast<uint32_t>(act[1])), "r"(static_cast<uint32_t>(act[2])),
        "r"(static_cast<uint32_t>(act[3])), "l"(h[0]), "l"(d[0]), "l"(h[1]), "l"(d[1]), "l"(h[2]), "l"(d[2]),
        "l"(h[3]), "l"(d[3]), "l"(&e[sl[0]].rec), "l"(&e[sl[1]].rec), "l"(&e[sl[2]].rec), "l"(&e[sl[3]].rec)
      : "memory");
}



// Commit (A.7).  Lanes of the warp of prompt p walk its new blocks b >= k_p (k_p = the
// first block missing before the batch, from k_chain_probe):
//   * CAS the key into its slot.  The inserting thread writes ITS payload (creator,
//     parent slot, label, owner, tier = HBM, live) with one 16-B store and links the
//     entry under its parent (the previous block's slot -- identical for every
//     duplicate of the key) exactly once;
//   * the inserter records its prompt index in Rec::meta;
//   * a claimant whose CAS found the key already inserted by this batch is an
//     intra-batch duplicate: it appends (slot, depth, prompt) to a (rare) fix-up list.
//     Stream-ordered after this kernel, k_commit_fixup_min folds the duplicates'
//     prompts into Rec::meta with atomicMin (lowest prompt = first creator in prompt
//     order, cache_index.hpp:164-168) and k_commit_fixup rewrites the payload from the
//     winning prompt.
// Everything an insert writes is in sector 0 of the entry (the sibling link only on a
// branch), so a new block costs one DRAM sector round trip.
#ifndef SKV_COMMIT_ROUNDS
#define SKV_COMMIT_ROUNDS 2
#endif
constexpr int kCommitRounds = SKV_COMMIT_ROUNDS;

#ifndef SKV_COMMIT_MINB
#define SKV_COMMIT_MINB 3  // 74 registers (profiles/r02_z_*: config 2 0.963 -> 0.946 ms per step; 4 / 64 registers 0.939 but
                           // the system-prompt workload 1.27 -> 1.59 ms, its prefetch no longer fits beside the commit)
#endif
#ifndef SKV_COMMIT_PERSIST
#define SKV_COMMIT_PERSIST 8  // CTAs per SM; each warp then strides over ~7 prompts (0.72 -> 0.60 ms, run 103)
#endif
#ifndef SKV_COMMIT_MINB_NOREC
#define SKV_COMMIT_MINB_NOREC 1
#endif
template <bool kRec>  // kRec: the batch's monitor records ride along (else k_record runs beside it)
__global__ void __launch_bounds__(256, kRec ? SKV_COMMIT_MINB : SKV_COMMIT_MINB_NOREC) k_commit(Index ix, const uint64_t* __restrict__ hk,
                                                const uint64_t* __restrict__ dk, const uint32_t* __restrict__ blk_off,
                                                const uint32_t* __restrict__ exist, const uint8_t* __restrict__ label,
                                                const uint32_t* __restrict__ uidx, const uint8_t* __restrict__ owners,
                                                uint32_t n_prompts, uint32_t* __restrict__ slot_out,
                                                unsigned long long* n_new, uint32_t* fix_list, uint32_t* n_fix,
                                                uint32_t fix_cap, uint32_t* err_flag,
                                                const uint32_t* __restrict__ matched,
                                                const uint64_t* __restrict__ users, MonCtx M, int with_record,
                                                int pending_labels) {
  constexpr int R = kCommitRounds;  // rounds of 32 blocks whose claims are in flight together
  const uint32_t lane = lane_id();
  uint32_t inserted = 0;
  if constexpr (kRec) M = mon_live(M);
  // the admit of this batch overflowed the user table (k_intern_users, err bit 8): its creator
  // indices are invalid, so nothing is inserted or recorded (the host raises CapacityExhausted)
  if (*reinterpret_cast<volatile uint32_t*>(err_flag) & 8u) return;
  // warp = prompt; a grid smaller than one warp per prompt strides over them
  const uint32_t stride = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < n_prompts; p += stride) {
  const uint32_t bo = blk_off[p], n = blk_off[p + 1] - bo, k0 = exist[p];
  if (k0 >= n) {
    if constexpr (kRec)
      if (with_record) record_prompt(ix, M, slot_out, bo, matched[p], users[p], lane, p);
    continue;
  }
  const uint32_t creator = uidx[p];
  const uint32_t owner = owners ? owners[p] : 0u;
  uint32_t carry = k0 > 0 ? slot_out[bo + k0 - 1] : kNone;  // parent of the first new block
  bool carry_mine = false;     // previous block's key claimed by this prompt (first new block: old parent)
  uint32_t carry_fix = kNone;  // previous block's duplicate fix-up entry, if it was a duplicate
  // sibling links of the previous round set, applied once the next set's claims are in
  // flight (the exchange results are not waited for on the critical path)
  uint32_t q_slot[R], q_sib[R];
#pragma unroll
  for (int r = 0; r < R; ++r) q_sib[r] = kNone, q_slot[r] = kNone;
  for (uint32_t base = k0; base < n; base += 32 * R) {
    uint64_t h[R], d[R];
    uint32_t s32[R], lab[R];
    bool mine[R];
    // claims: the first CAS of every round is issued before any result is awaited, so a
    // warp keeps R random DRAM round trips in flight instead of serialising them
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const uint32_t b = base + 32 * r + lane;
      s32[r] = kNone;
      mine[r] = false;
      lab[r] = 0;
      h[r] = d[r] = 0;
      if (b < n) {
        h[r] = hk[bo + b];
        d[r] = dk[bo + b];
        lab[r] = label[bo + b];
      }
    }
    // claims: a 128-bit CAS straight on every round's home slot, all rounds in flight
    // together (one DRAM round trip; the CAS returns the resident key, so no separate
    // load is needed); rare: the slot holds another key or the CAS lost a race -> linear
    // probing with CAS, every pending round's next CAS again in flight together.
    uint64_t sl[R];
    unsigned long long ol[R], oh[R];
    bool pend[R];
    // every round's home slot first (group leader = lane rounded down to kGroup, same
    // round), then the CASes back to back: no load between two claims, so the compiler
    // cannot place a wait for the first claim's result before the second is issued
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const uint64_t hL = __shfl_sync(kFull, h[r], lane & ~(kGroup - 1));
      const uint64_t dL = __shfl_sync(kFull, d[r], lane & ~(kGroup - 1));
      sl[r] = home_slot(ix, hL, dL, base + 32 * r + lane);
      pend[r] = false;
    }
    if constexpr (R == kClaimQ) {
      bool act[R];
#pragma unroll
      for (int r = 0; r < R; ++r) act[r] = base + 32 * r + lane < n;
      cas128_empty_x4(sl, act, h, d, ix.e, ol, oh);
    } else if constexpr (R == 2) {
      cas128_empty_x2(reinterpret_cast<unsigned long long*>(&ix.e[sl[0]].rec),
                      reinterpret_cast<unsigned long long*>(&ix.e[sl[1]].rec), base + lane < n, base + 32 + lane < n,
                      h[0], d[0], h[1], d[1], &ol[0], &oh[0], &ol[1], &oh[1]);
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        ol[r] = oh[r] = ~0ull;
        if (base + 32 * r + lane < n)
          cas128(reinterpret_cast<unsigned long long*>(&ix.e[sl[r]].rec), 0ull, 0ull, h[r], d[r], &ol[r], &oh[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) mine[r] = (ol[r] | oh[r]) == 0ull;
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (q_sib[r] != kNone) ix.e[q_slot[r]].aux.next_sibling = q_sib[r];
    // the batch's monitor records (AccessStats::record of the matched blocks, which
    // precede block k0) run while the first claims are in flight: L2 atomics overlap the
    // claims' DRAM round trips (record and commit touch disjoint fields)
    if constexpr (kRec)
      if (with_record && base == k0) record_prompt(ix, M, slot_out, bo, matched[p], users[p], lane, p);
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (base + 32 * r + lane < n) pend[r] = !mine[r] && !(ol[r] == h[r] && oh[r] == d[r]);
    for (uint64_t i = 1;; ++i) {
      bool any = false;
#pragma unroll
      for (int r = 0; r < R; ++r) any |= pend[r];
      if (!any) break;
      if (i > ix.mask) {  // table full
        atomicOr(err_flag, 2u);
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (pend[r]) {
            pend[r] = false;
            sl[r] = ~0ull;
          }
        break;
      }
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (pend[r]) {
          sl[r] = (sl[r] + 1) & ix.mask;
          mine[r] = cas128(reinterpret_cast<unsigned long long*>(&ix.e[sl[r]].rec), 0ull, 0ull, h[r], d[r], &ol[r],
                           &oh[r]);
        }
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (pend[r]) pend[r] = !mine[r] && !(ol[r] == h[r] && oh[r] == d[r]);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (base + 32 * r + lane >= n || sl[r] == ~0ull) continue;
      s32[r] = static_cast<uint32_t>(sl[r]);
      slot_out[bo + base + 32 * r + lane] = s32[r];
      if (mine[r] && base + 32 * r + lane < ix.rep.depth) {  // a replicated-layer entry this batch created
        const uint32_t k = atomicAdd(ix.rep.new_n, 1u);
        if (k < ix.rep.new_cap)
          ix.rep.new_list[k] = s32[r];
        else
          atomicOr(ix.rep.err, 2u);
      }
    }
    // payloads and parent links (parent = previous block's slot); sector 0 only
    uint32_t par[R];
    bool pmine[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      par[r] = __shfl_up_sync(kFull, s32[r], 1);
      pmine[r] = __shfl_up_sync(kFull, mine[r], 1);
      if (lane == 0) par[r] = carry, pmine[r] = carry_mine;
      carry = __shfl_sync(kFull, s32[r], 31);
      carry_mine = __shfl_sync(kFull, mine[r], 31);
    }
    // this prompt's own child of each block, when this prompt claimed it and it is in
    // this iteration (lane + 1, or the next round's lane 0); the last lane of the last
    // round links its child from the next iteration by a plain store instead
    uint32_t own_child[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const uint32_t cs = __shfl_down_sync(kFull, s32[r], 1);
      const bool cm = __shfl_down_sync(kFull, mine[r], 1);
      uint32_t ns = kNone;
      bool nm = false;
      if (r + 1 < R) {
        ns = __shfl_sync(kFull, s32[r + 1 < R ? r + 1 : r], 0);
        nm = __shfl_sync(kFull, mine[r + 1 < R ? r + 1 : r], 0);
      }
      own_child[r] = lane < 31 ? (cm ? cs : kNone) : (nm ? ns : kNone);
    }
    uint32_t sib[R], fidx[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      sib[r] = kNone;
      fidx[r] = kNone;
      if (s32[r] == kNone) continue;
      Entry& e = ix.e[s32[r]];
#ifdef SKV_EXP_NOPAY
      if (mine[r]) { ++inserted; continue; }
#endif
      if (mine[r]) {
        // creator, meta (with this prompt as the claimant), parent and this prompt's own
        // child in ONE 16-B store: no other child is linked under a fresh entry inside
        // this kernel (other prompts' children of it are duplicate claimants' and are
        // linked by the fix-up pass)
        const uint32_t meta = make_meta(pending_labels ? SKV_LABEL_PENDING : lab[r], owner, SKV_TIER_HBM, p);
        *reinterpret_cast<uint4*>(&e.rec.creator) = make_uint4(creator, meta, par[r], own_child[r]);
        if (ix.em) {  // speculative node id: exact unless this batch has duplicate claims
          const uint32_t b = base + 32 * r + lane, f = n - k0, j = b - k0;
          const uint32_t X = ix.em_next + ix.em_base[p];
          ix.em[s32[r]] = EvictMeta{ix.em_epoch, j + 1 < f ? X + 1 + j : X, b, 0u};
        }
        // the parent link: under a parent that existed before the batch children race ->
        // exchange; under a parent this prompt claimed, the parent's own 16-B store wrote
        // the link, except across iterations (plain store); under a parent another
        // prompt claimed -> linked by the fix-up pass
        if (par[r] != kNone) {
          const uint32_t b = base + 32 * r + lane;
          if (b == k0)
            sib[r] = atomicExch(&ix.e[par[r]].rec.first_child, s32[r]);
          else if (pmine[r] && lane == 0 && r == 0)
            ix.e[par[r]].rec.first_child = s32[r];
        }
        ++inserted;
      } else {
        const uint32_t f = atomicAdd(n_fix, 1u);
        if (f < fix_cap) {
          fix_list[f] = s32[r];
          fix_list[fix_cap + f] = base + 32 * r + lane;  // block depth of this key
          fix_list[2 * fix_cap + f] = p;
          fix_list[3 * fix_cap + f] = kNone;  // this prompt's child under the duplicate, if it claimed one
          fidx[r] = f;
        } else {
          atomicOr(err_flag, 4u);
        }
      }
    }
    __syncwarp();
    // a claimed block under a duplicate parent: hand the link to the parent's fix-up entry
#pragma unroll
    for (int r = 0; r < R; ++r) {
      uint32_t pf = __shfl_up_sync(kFull, fidx[r], 1);
      if (lane == 0) pf = carry_fix;
      carry_fix = __shfl_sync(kFull, fidx[r], 31);
      if (mine[r] && pf != kNone) fix_list[3 * fix_cap + pf] = s32[r];
    }
    // a child chained in front of existing siblings (branching only: under a fresh
    // parent the exchange returns kNone, which is the init value) -- deferred
#pragma unroll
    for (int r = 0; r < R; ++r) {
      q_slot[r] = s32[r];
      q_sib[r] = mine[r] ? sib[r] : kNone;
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (q_sib[r] != kNone) ix.e[q_slot[r]].aux.next_sibling = q_sib[r];
  }  // prompts
  inserted = __reduce_add_sync(kFull, inserted);
  if (lane == 0 && inserted) atomicAdd(n_new, static_cast<unsigned long long>(inserted));
}

// Flat commit (default): warp = 32 x R CONSECUTIVE blocks of the batch (prompt
// boundaries anywhere), grid-stride over such groups -- every warp is busy with claims
// from its first instruction (no per-prompt prologue), which keeps ~2x more claims in
// flight than a warp per prompt.  Lane = block i of prompt p = bprompt[i]:
//   * matched block (b < matched[p]): its monitor record (AccessStats::record), issued
//     while the group's claims are in flight;
//   * new block (the probe left slot = kNone): 128-bit CAS on its home slot (linear
//     probing on a foreign key); the CAS winner writes creator, meta, parent slot and its
//     own child's slot (block i+1, when the same lane group claimed it) in one 16-B store
//     into sector 0 while the line is in L2; a claimant that found its key inserted by
//     another prompt of the batch appends a duplicate fix-up entry;
//   * child links not covered by a parent's own store -- parent existed before the batch,
//     parent claimed by another prompt, or parent in the previous lane group (its slot
//     may not be written yet) -- go to the late list as (child slot, parent block) and
//     are exchanged into the parent's first-child list by k_commit_links after the
//     kernel, once every slot is known.
template <bool kRec>
__global__ void __launch_bounds__(256) k_commit_flat(
    Index ix, const uint64_t* __restrict__ hk, const uint64_t* __restrict__ dk, const uint32_t* __restrict__ blk_off,
    const uint32_t* __restrict__ bprompt, const uint8_t* __restrict__ label, const uint32_t* __restrict__ uidx,
    const uint8_t* __restrict__ owners, uint32_t n_prompts, uint32_t* slot_io, unsigned long long* n_new,
    uint32_t* fix_list, uint32_t* n_fix, uint32_t fix_cap, uint32_t* late, uint32_t* n_late, uint32_t* err_flag,
    const uint32_t* __restrict__ matched, const uint64_t* __restrict__ users, MonCtx M, int pending_labels) {
  constexpr int R = kCommitRounds;
  constexpr uint32_t G = 32 * R;
  const uint32_t lane = lane_id();
  const uint32_t nb = blk_off[n_prompts];
  const uint64_t nw = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  uint32_t inserted = 0;
  for (uint64_t g0 = ((static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * G; g0 < nb;
       g0 += nw * G) {
    uint32_t s32[R], pr[R], bb[R], pend_n[R], lab[R];
    uint64_t h[R], d[R], sl[R];
    bool nw_[R], mine[R], act[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const uint64_t i = g0 + 32 * r + lane;
      act[r] = i < nb;
      s32[r] = act[r] ? slot_io[i] : kNone;
      nw_[r] = act[r] && s32[r] == kNone;
      pr[r] = act[r] ? bprompt[i] : 0;
      h[r] = d[r] = 0;
      lab[r] = 0;
      if (nw_[r]) {
        h[r] = hk[i];
        d[r] = dk[i];
        lab[r] = label[i];
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const uint32_t o = act[r] ? blk_off[pr[r]] : 0;
      bb[r] = static_cast<uint32_t>(g0 + 32 * r + lane - o);
      pend_n[r] = act[r] ? blk_off[pr[r] + 1] - o : 0;  // blocks of the prompt
      sl[r] = home_slot(ix, h[r], d[r], 0);
    }
    unsigned long long ol[R], oh[R];
    if constexpr (R == kClaimQ) {
      cas128_empty_x4(sl, nw_, h, d, ix.e, ol, oh);
    } else if constexpr (R == 2) {
      cas128_empty_x2(reinterpret_cast<unsigned long long*>(&ix.e[sl[0]].rec),
                      reinterpret_cast<unsigned long long*>(&ix.e[sl[1]].rec), nw_[0], nw_[1], h[0], d[0], h[1],
                      d[1], &ol[0], &oh[0], &ol[1], &oh[1]);
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        ol[r] = oh[r] = ~0ull;
        if (nw_[r])
          cas128(reinterpret_cast<unsigned long long*>(&ix.e[sl[r]].rec), 0ull, 0ull, h[r], d[r], &ol[r], &oh[r]);
      }
    }
    // the monitor records of the group's matched blocks while the claims are in flight
    if constexpr (kRec) {
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (act[r] && !nw_[r] && bb[r] < matched[pr[r]]) {
          const uint64_t u = users[pr[r]];
          Entry& e = ix.e[s32[r]];
          atomicAdd(&e.stats.hit_cur, 1u);
          const uint32_t si = *reinterpret_cast<volatile uint32_t*>(&e.aux.set_idx);
          bool fast = false;
          if (si < kPendingSet) {
            const ulonglong2 v = ld_relaxed128(&M.tab[static_cast<uint64_t>(si) * kSetSlots + (mix32(u) & (kSetSlots - 1))]);
            fast = v.x == u && v.y >= M.wstart;
          }
          if (!fast) record_user(ix, M, s32[r], u);
        }
    }
    bool pend[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      mine[r] = nw_[r] && (ol[r] | oh[r]) == 0ull;
      pend[r] = nw_[r] && !mine[r] && !(ol[r] == h[r] && oh[r] == d[r]);
    }
    for (uint64_t k = 1;; ++k) {
      bool any = false;
#pragma unroll
      for (int r = 0; r < R; ++r) any |= pend[r];
      if (!any) break;
      if (k > ix.mask) {  // table full
        atomicOr(err_flag, 2u);
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (pend[r]) pend[r] = false, sl[r] = ~0ull;
        break;
      }
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (pend[r]) {
          sl[r] = (sl[r] + 1) & ix.mask;
          mine[r] = cas128(reinterpret_cast<unsigned long long*>(&ix.e[sl[r]].rec), 0ull, 0ull, h[r], d[r], &ol[r],
                           &oh[r]);
          pend[r] = !mine[r] && !(ol[r] == h[r] && oh[r] == d[r]);
        }
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (nw_[r]) {
        s32[r] = sl[r] == ~0ull ? kNone : static_cast<uint32_t>(sl[r]);
        slot_io[g0 + 32 * r + lane] = s32[r];
      }
    // neighbours inside the group: block i-1 (parent) and i+1 (own child)
#pragma unroll
    for (int r = 0; r < R; ++r) {
      uint32_t ps = __shfl_up_sync(kFull, s32[r], 1);
      bool pm = __shfl_up_sync(kFull, mine[r], 1);
      uint32_t cs = __shfl_down_sync(kFull, s32[r], 1);
      bool cm = __shfl_down_sync(kFull, mine[r], 1);
      const uint32_t ps_prev = __shfl_sync(kFull, s32[r > 0 ? r - 1 : 0], 31);
      const bool pm_prev = __shfl_sync(kFull, mine[r > 0 ? r - 1 : 0], 31);
      const uint32_t cs_next = __shfl_sync(kFull, s32[r + 1 < R ? r + 1 : r], 0);
      const bool cm_next = __shfl_sync(kFull, mine[r + 1 < R ? r + 1 : r], 0);
      bool p_in = true;  // the parent block belongs to this lane group
      if (lane == 0) {
        if (r > 0) {
          ps = ps_prev, pm = pm_prev;
        } else {
          p_in = false;
        }
      }
      bool c_in = true;
      if (lane == 31) {
        if (r + 1 < R) {
          cs = cs_next, cm = cm_next;
        } else {
          c_in = false;
        }
      }
      if (!nw_[r] || s32[r] == kNone) continue;
      const uint32_t b = bb[r], p = pr[r];
      if (mine[r]) {
        uint32_t parent = kNone;
        bool late_link = false, need_parent = false;
        if (b > 0) {
          if (p_in) {
            parent = ps;
            late_link = !pm;
          } else {  // previous lane group: its slot may not be written yet
            parent = *reinterpret_cast<volatile uint32_t*>(&slot_io[g0 + 32 * r + lane - 1]);
            late_link = true;
            need_parent = parent == kNone;
          }
        }
        const uint32_t child = (b + 1 < pend_n[r] && c_in && cm) ? cs : kNone;
        const uint32_t meta = make_meta(pending_labels ? SKV_LABEL_PENDING : lab[r], owners ? owners[p] : 0u,
                                        SKV_TIER_HBM, p);
        *reinterpret_cast<uint4*>(&ix.e[s32[r]].rec.creator) = make_uint4(uidx[p], meta, parent, child);
        if (ix.em) ix.em[s32[r]] = EvictMeta{0u, kNone, b, 0u};
        if (late_link) {
          const uint32_t f = atomicAdd(n_late, 1u);
          if (f < fix_cap) {
            late[2 * f] = s32[r];
            late[2 * f + 1] = static_cast<uint32_t>(g0 + 32 * r + lane - 1) | (need_parent ? 0x80000000u : 0u);
          } else {
            atomicOr(err_flag, 4u);
          }
        }
        ++inserted;
      } else {
        const uint32_t f = atomicAdd(n_fix, 1u);
        if (f < fix_cap) {
          fix_list[f] = s32[r];
          fix_list[fix_cap + f] = b;  // block depth of this key
          fix_list[2 * fix_cap + f] = p;
          fix_list[3 * fix_cap + f] = kNone;
        } else {
          atomicOr(err_flag, 4u);
        }
      }
    }
  }
  inserted = __reduce_add_sync(kFull, inserted);
  if (lane == 0 && inserted) atomicAdd(n_new, static_cast<unsigned long long>(inserted));
}

// Late child links of the flat commit: every slot is known now.
__global__ void k_commit_links(Index ix, const uint32_t* __restrict__ slot, const uint32_t* __restrict__ late,
                               const uint32_t* __restrict__ n_late, uint32_t cap) {
  const uint32_t n = min(*n_late, cap);
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const uint32_t c = late[2 * k], pb = late[2 * k + 1];
    const uint32_t ps = slot[pb & 0x7fffffffu];
    if (pb >> 31) ix.e[c].rec.parent = ps;
    const uint32_t sib = atomicExch(&ix.e[ps].rec.first_child, c);
    if (sib != kNone) ix.e[c].aux.next_sibling = sib;
  }
}

// Intra-batch duplicates, pass 1: lowest claiming prompt (all claims are complete).
__global__ void k_commit_fixup_min(Index ix, const uint32_t* __restrict__ fix_list, const uint32_t* __restrict__ n_fix,
                                   uint32_t fix_cap) {
  const uint32_t nf = min(*n_fix, fix_cap);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nf; i += gridDim.x * blockDim.x)
    atomicMin(&ix.e[fix_list[i]].rec.meta, (fix_list[2 * fix_cap + i] << 8) | 0xffu);
}

// Pass 2: the winner's payload (creator, label, owner, tier = HBM, live, winner prompt).
__global__ void k_commit_fixup(Index ix, const uint32_t* __restrict__ blk_off, const uint8_t* __restrict__ label,
                               const uint32_t* __restrict__ uidx, const uint8_t* __restrict__ owners,
                               const uint32_t* __restrict__ fix_list, const uint32_t* __restrict__ n_fix,
                               uint32_t fix_cap, int pending_labels, uint32_t* n_revived, MonCtx P) {
  P = mon_live(P);
  const uint32_t nf = min(*n_fix, fix_cap);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nf; i += gridDim.x * blockDim.x) {
    const uint32_t s = fix_list[i], b = fix_list[fix_cap + i];
    Rec& r = ix.e[s].rec;
    const uint32_t pw = meta_prompt(r.meta);
    const uint32_t meta = make_meta(pending_labels ? SKV_LABEL_PENDING : label[blk_off[pw] + b],
                                    owners ? owners[pw] : 0u, SKV_TIER_HBM, pw);
    *reinterpret_cast<uint2*>(&r.creator) = make_uint2(uidx[pw], meta);
    // a re-inserted tombstone is a fresh node (cache_index.hpp:192-201); its first claimant
    // resets it, and it is still in its parent's child list
    if (ix.em && ix.em[s].dead && atomicExch(&ix.em[s].dead, 0u)) {
      ix.e[s].stats = Stats{0u, 0u, 0u, 0u};
      // an entry already listed in the current window (set_idx set) keeps its place in the list
      // (acquire_set must not append it twice) but gets a fresh, empty user set: a set allocated
      // in this window has no live member (pool sets are only reused across windows)
      if (ix.e[s].aux.set_idx != kNone && P.hdr) {
        const uint32_t si = atomicAdd(P.pool_count, 1u);
        if (si >= P.pool_cap) {
          atomicOr(P.err, 1u);
        } else {
          P.hdr[si] = SetHdr{0u, 0u, 0u, 0u, 0ull};
          ix.e[s].aux.set_idx = si;
        }
      }
      ix.e[s].aux.mark = 0;
      ix.em[s].node_id = kNone;  // assigned by the exact pass (duplicate claims exist)
      ix.em[s].depth = b;
      ix.em[s].access_epoch = ix.em_epoch;
      atomicAdd(n_revived, 1u);
    }
    // the duplicate claimant's own child under this entry (k_commit left it unlinked)
    const uint32_t c = fix_list[3 * fix_cap + i];
    if (c != kNone) {
      const uint32_t sib = atomicExch(&r.first_child, c);
      if (sib != kNone) ix.e[c].aux.next_sibling = sib;
    }
  }
}

// ---------------------------------------------------------------------------------
// K5: monitor epoch (A.6).  Candidates = Public entries whose FP64 predicate holds
// (monitor.hpp:68-70); a candidate fires iff no ancestor is a candidate (the
// reference's pre-order pass relabels a fired node's subtree before visiting it);
// fired nodes relabel their subtree; then every touched window rolls.
// ---------------------------------------------------------------------------------
struct DevEvent {
  uint64_t h, d;
  uint8_t action, owner, pad[6];
  double now, prev;
  uint64_t u_pre, epoch;
};
static_assert(sizeof(DevEvent) == sizeof(skv_event), "event layout");

__global__ void k_epoch_candidates(Index ix, const uint32_t* __restrict__ list, const uint32_t* __restrict__ n_list,
                                   int only_untouched, uint32_t stamp, double jump, uint64_t u_pre_max,
                                   uint32_t* __restrict__ cands, uint32_t* __restrict__ n_cands,
                                   const uint32_t* __restrict__ guard) {
  if (guard && (guard[5] | guard[8])) return;  // a speculative pass behind a failed / replaying commit
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= *n_list) return;
  uint32_t s = list[i];
  // the entry's label and its monitor sector in ONE round trip (independent loads before any test)
  const uint32_t meta = ix.e[s].rec.meta;
  const Stats st = ix.e[s].stats;
  const uint32_t set_idx = ix.e[s].aux.set_idx;
  if (only_untouched && set_idx != kNone) return;
  if (!meta_live(meta) || meta_label(meta) != SKV_LABEL_PUBLIC) return;
  if (st.hit_pre == 0) return;
  double now = st.hit_cur ? static_cast<double>(st.u_cnt) / static_cast<double>(st.hit_cur) : 0.0;
  double prev = static_cast<double>(st.u_pre) / static_cast<double>(st.hit_pre);
  if ((now - prev) >= jump && static_cast<uint64_t>(st.u_pre) <= u_pre_max) {
    ix.e[s].aux.mark = stamp;
    cands[atomicAdd(n_cands, 1u)] = s;
  }
}

__global__ void k_epoch_fire(Index ix, const uint32_t* __restrict__ cands, const uint32_t* __restrict__ n_cands,
                             uint32_t stamp, uint64_t epoch, DevEvent* __restrict__ events,
                             uint32_t* __restrict__ n_events, uint32_t* __restrict__ fired,
                             const uint32_t* __restrict__ guard) {
  if (guard && (guard[5] | guard[8])) return;  // a speculative pass behind a failed / replaying commit
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= *n_cands) return;
  uint32_t s = cands[i];
  for (uint32_t a = ix.e[s].rec.parent; a != kNone; a = ix.e[a].rec.parent)
    if (ix.e[a].aux.mark == stamp) return;
  Stats st = ix.e[s].stats;
  const Rec& r = ix.e[s].rec;
  uint32_t e = atomicAdd(n_events, 1u);
  DevEvent ev;
  ev.h = r.h;
  ev.d = r.d;
  ev.owner = static_cast<uint8_t>(meta_owner(r.meta));
  ev.action = ev.owner == 0 ? SKV_ACTION_DOWNGRADE : SKV_ACTION_RESTRICT;
  for (int k = 0; k < 6; ++k) ev.pad[k] = 0;
  ev.now = st.hit_cur ? static_cast<double>(st.u_cnt) / static_cast<double>(st.hit_cur) : 0.0;
  ev.prev = static_cast<double>(st.u_pre) / static_cast<double>(st.hit_pre);
  ev.u_pre = st.u_pre;
  ev.epoch = epoch;
  events[e] = ev;
  fired[e] = s;
}

// Relabel a fired entry's whole subtree (monitor.hpp:88-95 -> apply_label_subtree): a DFS whose
// per-node loads (label, first child, next sibling) are issued together -- one dependent round trip
// per node -- with the pending siblings on a per-thread stack instead of climbing parent links back
// up (a 256-deep chain of config 4 cost ~3 round trips per node).  A stack overflow (deeper branching
// than kRelabelStack levels) falls back to the parent-climbing walk, which relabels everything again
// (idempotent).
#ifndef SKV_RELABEL_STACK
#define SKV_RELABEL_STACK 64
#endif
constexpr int kRelabelStack = SKV_RELABEL_STACK;
__device__ void relabel_subtree(const Index& ix, uint32_t root, uint32_t lab) {
  ix.e[root].rec.meta = (ix.e[root].rec.meta & ~3u) | lab;
  uint32_t stack[kRelabelStack];
  int sp = 0;
  bool overflow = false;
  uint32_t cur = ix.e[root].rec.first_child;
  for (;;) {
    if (cur == kNone) {
      if (sp == 0) break;
      cur = stack[--sp];
      continue;
    }
    const uint32_t m = ix.e[cur].rec.meta, fc = ix.e[cur].rec.first_child, ns = ix.e[cur].aux.next_sibling;
    ix.e[cur].rec.meta = (m & ~3u) | lab;
    if (ns != kNone) {
      if (sp < kRelabelStack) {
        stack[sp++] = ns;
      } else {
        overflow = true;
        break;
      }
    }
    cur = fc;
  }
  if (!overflow) return;
  cur = ix.e[root].rec.first_child;
  while (cur != kNone) {
    ix.e[cur].rec.meta = (ix.e[cur].rec.meta & ~3u) | lab;
    const uint32_t c = ix.e[cur].rec.first_child;
    if (c != kNone) {
      cur = c;
      continue;
    }
    while (cur != root && ix.e[cur].aux.next_sibling == kNone) cur = ix.e[cur].rec.parent;
    if (cur == root) break;
    cur = ix.e[cur].aux.next_sibling;
  }
}

__global__ void k_epoch_propagate(Index ix, const uint32_t* __restrict__ fired, const uint32_t* __restrict__ n_fired,
                                  const uint32_t* __restrict__ guard) {
  if (guard && (guard[5] | guard[8])) return;  // a speculative pass behind a failed / replaying commit
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= *n_fired) return;
  const uint32_t root = fired[i];
  relabel_subtree(ix, root, meta_owner(ix.e[root].rec.meta) == 0 ? SKV_LABEL_PRIVATE : SKV_LABEL_RESTRICTED);
}

__global__ void k_epoch_roll(Index ix, const uint32_t* __restrict__ list, const uint32_t* __restrict__ n_list,
                             int prev_list, const uint32_t* __restrict__ guard) {
  if (guard && (guard[5] | guard[8])) return;  // a speculative pass behind a failed / replaying commit
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= *n_list) return;
  uint32_t s = list[i];
  if (prev_list) {
    if (ix.e[s].aux.set_idx != kNone) return;  // rolled by the current-window list
    Stats z{0, 0, 0, 0};
    ix.e[s].stats = z;
  } else {
    Stats st = ix.e[s].stats;
    Stats r{0, 0, st.hit_cur, st.u_cnt};
    ix.e[s].stats = r;
    ix.e[s].aux.set_idx = kNone;
  }
}

// The whole epoch pass in ONE cooperative launch (grid syncs between the phases instead of
// six kernel boundaries): a small batch's epoch is otherwise launch-bound (config 1 / 5:
// ~50 us of mostly empty grids sized for the window lists' capacity).  Same phases, same
// order, each a grid-stride loop over the device-side list lengths:
//   candidates (current list, then the untouched previous-window entries) | fire (an
//   ancestor marked this epoch suppresses, monitor.hpp:88-95) | propagate | roll previous |
//   roll current; then the window swap's counter resets.
// the split pass's window swap (its counter resets), skipped with the pass
__global__ void k_epoch_reset(uint32_t* pool_count, uint32_t* prev_count, const uint32_t* __restrict__ guard) {
  if (guard && (guard[5] | guard[8])) return;
  *pool_count = 0;
  *prev_count = 0;
}

__device__ __forceinline__ void epoch_candidate(Index& ix, uint32_t s, bool only_untouched, uint32_t stamp,
                                                double jump, uint64_t u_pre_max, uint32_t* cands,
                                                uint32_t* n_cands) {
  const uint32_t meta = ix.e[s].rec.meta;  // one round trip: every load before any test
  const Stats st = ix.e[s].stats;
  const uint32_t set_idx = ix.e[s].aux.set_idx;
  if (only_untouched && set_idx != kNone) return;
  if (!meta_live(meta) || meta_label(meta) != SKV_LABEL_PUBLIC) return;
  if (st.hit_pre == 0) return;
  double now = st.hit_cur ? static_cast<double>(st.u_cnt) / static_cast<double>(st.hit_cur) : 0.0;
  double prev = static_cast<double>(st.u_pre) / static_cast<double>(st.hit_pre);
  if ((now - prev) >= jump && static_cast<uint64_t>(st.u_pre) <= u_pre_max) {
    ix.e[s].aux.mark = stamp;
    cands[atomicAdd(n_cands, 1u)] = s;
  }
}

__global__ void __launch_bounds__(256) k_epoch_fused(Index ix, uint32_t* l0, uint32_t* l1, uint32_t* ntb, int cur_in,
                                                     uint32_t stamp, double jump, uint64_t u_pre_max, uint32_t* cands,
                                                     uint32_t* n_cands, uint64_t epoch, DevEvent* events,
                                                     uint32_t* n_events, uint32_t* fired, uint32_t* pool_count,
                                                     const uint32_t* st, const uint32_t* guard) {
  namespace cg = cooperative_groups;
  // a speculative pass behind a commit that failed or needs the ordered replay: nothing happens
  // (every thread leaves before the first grid sync)
  if (guard && (!st || st[6]) && (guard[5] | guard[8])) return;
  cg::grid_group grid = cg::this_grid();
  const uint32_t t0 = blockIdx.x * blockDim.x + threadIdx.x, T = gridDim.x * blockDim.x;
  uint32_t cur = static_cast<uint32_t>(cur_in);
  if (st) {  // a graph-replayed epoch: window and stamps from the device step state
    cur = st[2];
    stamp = st[3];
    epoch = static_cast<uint64_t>(st[4]) | (static_cast<uint64_t>(st[5]) << 32);
  }
  const uint32_t* cur_list = cur ? l1 : l0;
  const uint32_t* prev_list = cur ? l0 : l1;
  uint32_t* prev_count = ntb + (1 - cur);
  const uint32_t nc = ntb[cur], np = *prev_count;
  for (uint32_t i = t0; i < nc + np; i += T)
    epoch_candidate(ix, i < nc ? cur_list[i] : prev_list[i - nc], i >= nc, stamp, jump, u_pre_max, cands, n_cands);
  grid.sync();
  const uint32_t nk = *n_cands;
  for (uint32_t i = t0; i < nk; i += T) {
    const uint32_t s = cands[i];
    bool sup = false;
    for (uint32_t a = ix.e[s].rec.parent; a != kNone && !sup; a = ix.e[a].rec.parent) sup = ix.e[a].aux.mark == stamp;
    if (sup) continue;
    Stats st = ix.e[s].stats;
    const Rec& r = ix.e[s].rec;
    const uint32_t e = atomicAdd(n_events, 1u);
    DevEvent ev;
    ev.h = r.h;
    ev.d = r.d;
    ev.owner = static_cast<uint8_t>(meta_owner(r.meta));
    ev.action = ev.owner == 0 ? SKV_ACTION_DOWNGRADE : SKV_ACTION_RESTRICT;
    for (int k = 0; k < 6; ++k) ev.pad[k] = 0;
    ev.now = st.hit_cur ? static_cast<double>(st.u_cnt) / static_cast<double>(st.hit_cur) : 0.0;
    ev.prev = static_cast<double>(st.u_pre) / static_cast<double>(st.hit_pre);
    ev.u_pre = st.u_pre;
    ev.epoch = epoch;
    events[e] = ev;
    fired[e] = s;
  }
  grid.sync();
  const uint32_t nf = *n_events;
  for (uint32_t i = t0; i < nf; i += T) {
    const uint32_t root = fired[i];
    relabel_subtree(ix, root, meta_owner(ix.e[root].rec.meta) == 0 ? SKV_LABEL_PRIVATE : SKV_LABEL_RESTRICTED);
  }
  for (uint32_t i = t0; i < np; i += T) {  // the previous window's untouched entries roll to zero
    const uint32_t s = prev_list[i];
    if (ix.e[s].aux.set_idx != kNone) continue;  // rolled below with the current window
    ix.e[s].stats = Stats{0, 0, 0, 0};
  }
  grid.sync();
  for (uint32_t i = t0; i < nc; i += T) {
    const uint32_t s = cur_list[i];
    const Stats st = ix.e[s].stats;
    ix.e[s].stats = Stats{0, 0, st.hit_cur, st.u_cnt};
    ix.e[s].aux.set_idx = kNone;
  }
  if (t0 == 0) {  // the window swap: the pool and the list that becomes current start empty
    *pool_count = 0;
    *prev_count = 0;
  }
}

// ---------------------------------------------------------------------------------
// misc: tiers, export, per-call wrappers
// ---------------------------------------------------------------------------------
// ---------------------------------------------------------------------------------
// Label landing (RadixCacheIndex::resolve_block, cache_index.hpp:321-343): the
// classification block of prompt p is its blocks [first[p], n_p) (keys prompt-major from
// block 0).  Public: every block of the chain, no propagation (promotion never
// propagates, :657-662).  Private / Restricted: set_label on the chain's top block with
// propagation to every descendant (:663-666, apply_label_subtree :679-686).
// ---------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t prompt_of(const uint32_t* boff, uint32_t n_prompts, uint32_t i) {
  uint32_t lo = 0, hi = n_prompts;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (boff[mid] <= i)
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}

__device__ __forceinline__ void set_meta_label(Rec& r, uint32_t lab) {
  uint32_t old = r.meta;
  for (;;) {
    const uint32_t nv = (old & ~3u) | lab;
    if (nv == old) return;
    const uint32_t got = atomicCAS(&r.meta, old, nv);
    if (got == old) return;
    old = got;
  }
}

__global__ void k_resolve_public(Index ix, const uint64_t* h, const uint64_t* d, const uint32_t* boff,
                                 uint32_t n_prompts, const uint32_t* first, const uint8_t* labels, uint32_t n,
                                 uint32_t* missing) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t p = prompt_of(boff, n_prompts, i);
  const uint32_t b = i - boff[p];
  if (labels[p] != SKV_LABEL_PUBLIC || b < first[p]) return;
  const uint32_t L = boff[p] + (b & ~(kGroup - 1));
  Rec r;
  const uint32_t s = find_slot(ix, h[i], d[i], h[L], d[L], b, &r);
  if (s == kNone) {
    atomicAdd(missing, 1u);
    return;
  }
  set_meta_label(ix.e[s].rec, SKV_LABEL_PUBLIC);
}

__global__ void k_resolve_private(Index ix, const uint64_t* h, const uint64_t* d, const uint32_t* boff,
                                  uint32_t n_prompts, const uint32_t* first, const uint8_t* labels, uint32_t lab,
                                  uint32_t* missing) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_prompts || labels[p] != lab || boff[p] + first[p] >= boff[p + 1]) return;
  const uint32_t b = first[p], i = boff[p] + b, L = boff[p] + (b & ~(kGroup - 1));
  Rec r;
  const uint32_t root = find_slot(ix, h[i], d[i], h[L], d[L], b, &r);
  if (root == kNone) {
    atomicAdd(missing, 1u);
    return;
  }
  set_meta_label(ix.e[root].rec, lab);
  uint32_t cur = ix.e[root].rec.first_child;
  while (cur != kNone) {
    set_meta_label(ix.e[cur].rec, lab);
    const uint32_t c = ix.e[cur].rec.first_child;
    if (c != kNone) {
      cur = c;
      continue;
    }
    while (cur != root && ix.e[cur].aux.next_sibling == kNone) cur = ix.e[cur].rec.parent;
    if (cur == root) break;
    cur = ix.e[cur].aux.next_sibling;
  }
}

__global__ void k_set_tiers(Index ix, const uint64_t* h, const uint64_t* d, const uint32_t* boff, uint32_t n_prompts,
                            const uint8_t* tiers, uint32_t n) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t lo = 0, hi = n_prompts;  // prompt holding block i
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (boff[mid] <= i)
      lo = mid;
    else
      hi = mid;
  }
  const uint32_t b = i - boff[lo], L = boff[lo] + (b & ~(kGroup - 1));
  Rec r;
  uint32_t s = find_slot(ix, h[i], d[i], h[L], d[L], b, &r);
  if (s == kNone) return;
  // demote (cache_index.hpp:362-381): a tier only moves down HBM -> DRAM -> SSD, so
  // repeated tags of one entry keep the slowest (the reference's demote-until loop)
  uint32_t* meta = &ix.e[s].rec.meta;
  uint32_t old = *meta;
  for (;;) {
    const uint32_t t = max(meta_tier(old), static_cast<uint32_t>(tiers[i]));
    const uint32_t nv = (old & ~(3u << 3)) | (t << 3);
    if (nv == old) break;
    const uint32_t got = atomicCAS(meta, old, nv);
    if (got == old) break;
    old = got;
  }
}

__global__ void k_export(Index ix, const uint64_t* __restrict__ user_rev, skv_entry* out, uint32_t* n_out,
                         uint32_t cap) {
  uint64_t s = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s > ix.mask) return;
  const Rec& r = ix.e[s].rec;
  if ((r.h == 0 && r.d == 0) || !meta_live(r.meta)) return;
  Stats st = ix.e[s].stats;
  skv_entry e;
  e.h = r.h;
  e.d = r.d;
  e.creator = user_rev[r.creator];
  e.label = static_cast<uint8_t>(meta_label(r.meta));
  e.owner = static_cast<uint8_t>(meta_owner(r.meta));
  e.tier = static_cast<uint8_t>(meta_tier(r.meta));
  e.hit_cur = st.hit_cur;
  e.u_cnt = st.u_cnt;
  e.hit_pre = st.hit_pre;
  e.u_pre = st.u_pre;
  const uint32_t k = atomicAdd(n_out, 1u);
  if (k < cap) out[k] = e;  // the count is exact even past cap (the host re-sizes and retries)
}

__global__ void k_scan_text(const uint8_t* text, uint32_t len, DevRules r, uint32_t* mask, uint32_t shift) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  uint32_t row = r.start_row, acc = 0;
  for (uint32_t i = 0; i < len; ++i) {
    const uint32_t e = r.full[(row - r.row_base + r.class2[text[i]]) >> 1];
    acc |= e;
    row = e & 0xffffu;
  }
  acc |= r.full[(row - r.row_base + r.eos2) >> 1];
  *mask |= (acc >> 16) << shift;
}

// A batch of independent texts (DetectionPipeline drains: CompiledRuleSet::scan per pending
// block, detection.hpp:148-170, 547-552): one thread per text -- pipeline texts are a block plus
// its context, a few dozen bytes, so a text is one thread's sequential walk of the search DFA.
__global__ void k_scan_texts(const uint8_t* __restrict__ text, const uint64_t* __restrict__ off, uint32_t n,
                             DevRules r, uint32_t* __restrict__ masks, uint32_t shift) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t row = r.start_row, acc = 0;
  for (uint64_t k = off[i], e = off[i + 1]; k < e; ++k) {
    const uint32_t v = r.full[(row - r.row_base + r.class2[text[k]]) >> 1];
    acc |= v;
    row = v & 0xffffu;
  }
  acc |= r.full[(row - r.row_base + r.eos2) >> 1];
  masks[i] |= (acc >> 16) << shift;
}

__global__ void k_digest(const uint32_t* t, uint32_t n, uint64_t* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  uint64_t h = fnv_u32(kFnvOff, n);
  for (uint32_t i = 0; i < n; ++i) h = fnv_u32(h, t[i]);
  *out = h;
}

inline uint32_t cdiv(uint64_t a, uint64_t b) { return static_cast<uint32_t>((a + b - 1) / b); }

}  // namespace

// =================================================================================
// launchers
// =================================================================================
void launch_block_counts(const uint64_t* tok_off, uint32_t n, uint32_t B, uint32_t* counts, uint32_t* plen,
                         cudaStream_t s) {
  k_block_counts<<<cdiv(n + 1, 256), 256, 0, s>>>(tok_off, n, B, counts, plen);
}

void launch_ttft(const uint32_t* blk_off, const uint32_t* matched, const uint32_t* plen, const uint8_t* bmeta,
                 const uint64_t* request_ids, uint64_t request_base, uint32_t n, uint32_t B, const CostModelDev& cm,
                 double* ttft, uint32_t* intra, uint32_t* inter, cudaStream_t s) {
  if (n)
    k_ttft<<<cdiv(n, 256), 256, 0, s>>>(blk_off, matched, plen, bmeta, request_ids, request_base, n, B, cm, ttft,
                                        intra, inter);
}

size_t scan_temp_bytes(uint32_t n) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, static_cast<const uint32_t*>(nullptr),
                                static_cast<uint32_t*>(nullptr), n);
  return bytes;
}

void launch_exclusive_scan(void* temp, size_t temp_bytes, const uint32_t* in, uint32_t* out, uint32_t n,
                           cudaStream_t s) {
  cub::DeviceScan::ExclusiveSum(temp, temp_bytes, in, out, n, s);
}

HSLayout hash_scan_layout(const DevRules& r, uint32_t B, uint32_t W) {
  // dynamic SMEM = the DFA image [row_base, fast_bytes) + the accepting-copy masks; the
  // tokens are read straight from HBM (no staging buffers)
  (void)B;
  (void)W;
  HSLayout L{};
  L.off_list = round16(r.fast_bytes - r.row_base);
  L.warps = kHSWarps;
  L.total = L.off_list + round16(r.n_copies * 2 + 2);
  return L;
}

// The dynamic-SMEM opt-in is a per-function attribute shared by every context and rule group of
// the process: set it to the device maximum (occupancy follows each launch's own smem), never to
// one group's footprint -- a later, smaller group would otherwise make a larger one fail to launch.
static bool optin_max_smem(const void* fn, int device) {
  int optin = 0;
  cudaFuncAttributes fa;
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device) != cudaSuccess ||
      cudaFuncGetAttributes(&fa, fn) != cudaSuccess)
    return false;
  const int dyn = optin - static_cast<int>(fa.sharedSizeBytes);  // the opt-in covers static + dynamic
  return dyn > 0 && cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn) == cudaSuccess;
}

int hash_scan_grid(int device, uint32_t smem, uint32_t threads) {
  if (!optin_max_smem(reinterpret_cast<const void*>(k_hash_scan), device)) return -1;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_hash_scan, static_cast<int>(threads), smem) !=
      cudaSuccess)
    return -1;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  if (per_sm < 1) per_sm = 1;
  return per_sm * sms;
}

void launch_hash_scan(const HashScanArgs& a, int grid, uint32_t smem, uint32_t threads, cudaStream_t s) {
  // a.n_blocks is a host-side hint (0 = unknown); the kernel reads the count from blk_off[N]
  const uint32_t wpc = threads / 32;
  const uint32_t g = a.n_blocks ? std::min<uint32_t>(grid, (a.n_blocks + wpc - 1) / wpc) : static_cast<uint32_t>(grid);
  if (a.n_prompts == 0 || g == 0) return;
  k_hash_scan<<<g, threads, smem, s>>>(a);
}

uint32_t hash_scan16_smem(uint32_t img_bytes, uint32_t q_cap, uint32_t warps) {
  const uint32_t w = warps ? warps : kH16Warps;
  return round16(img_bytes) + 4 * w * static_cast<uint32_t>(sizeof(Slot16)) +
         w * q_cap * static_cast<uint32_t>(sizeof(H16Task));
}

int hash_scan16_grid(int device, uint32_t smem) {
  if (!optin_max_smem(reinterpret_cast<const void*>(k_hash_scan16), device)) return -1;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_hash_scan16, kH16Warps * 32, smem) != cudaSuccess ||
      per_sm < 1)
    return -1;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  return per_sm * sms;
}

void launch_hash_scan16(const HS16Args& a, int grid, uint32_t smem, cudaStream_t s, int warps) {
  if (a.n_prompts == 0 || grid <= 0) return;
  const int w = warps > 0 && warps < static_cast<int>(kH16Warps) ? warps : static_cast<int>(kH16Warps);
  k_hash_scan16<<<grid, w * 32, smem, s>>>(a);
}

__global__ void k_block_prompts(const uint32_t* __restrict__ blk_off, uint32_t n, uint32_t* __restrict__ map) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < n; p += (gridDim.x * blockDim.x) >> 5)
    for (uint32_t b = blk_off[p] + lane; b < blk_off[p + 1]; b += 32) map[b] = p;
}

void launch_block_prompts(const uint32_t* blk_off, uint32_t n, uint32_t* map, cudaStream_t s) {
  if (n) k_block_prompts<<<static_cast<unsigned>(std::min<uint64_t>(cdiv(static_cast<uint64_t>(n) * 32, 256), 4096)),
                           256, 0, s>>>(blk_off, n, map);
}

void launch_chain_probe(const Index& ix, const uint64_t* d, const uint32_t* blk_off, const uint32_t* first_sens,
                        const uint32_t* users, uint32_t n, uint64_t* h, uint8_t* label, uint8_t* decision,
                        uint32_t* slot, uint32_t* matched, uint32_t* exist, uint8_t* tier, uint8_t* bmeta,
                        const MonCtx& mon, uint32_t* bprompt, int prechained, uint32_t split_from,
                        cudaStream_t s) {
  auto* kern = prechained ? k_chain_probe<true> : k_chain_probe<false>;
  if (n)
    kern<<<static_cast<unsigned>(std::min<uint64_t>(cdiv(n, kCPPrompts * kCPWarps),
                                                             SKV_KCP_GRID_PER_SM ? SKV_KCP_GRID_PER_SM * 148ull
                                                                                 : ~0ull)),
                    kCPWarps * 32, 0, s>>>(ix, d, blk_off, first_sens, users, n, h, label,
                                                                   decision, slot, matched, exist, tier, bmeta, mon,
                                                                   bprompt, split_from);
}

uint32_t record_grid(int device) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  return static_cast<uint32_t>(sms) * 8;
}

void launch_record(const Index& ix, const MonCtx& mon, const uint32_t* slot, const uint32_t* blk_off,
                   const uint32_t* matched, const uint64_t* users, uint32_t n, cudaStream_t s) {
  if (n)
    k_record<<<cdiv(static_cast<uint64_t>(n) * 32, 256), 256, 0, s>>>(ix, mon, slot, blk_off, matched, users, n);
}

void launch_record_finish(const Index& ix, const MonCtx& mon, uint32_t* replay, uint32_t* n_replay, int grid,
                          cudaStream_t s) {
  k_record_finish<<<grid, 256, 0, s>>>(ix, mon, replay, n_replay);
}

void launch_replay_emit(const Index& ix, const MonCtx& mon, const uint32_t* slot, const uint32_t* blk_off,
                        const uint32_t* matched, uint32_t n, unsigned long long* keys, uint32_t* n_keys,
                        cudaStream_t s) {
  if (n)
    k_replay_emit<<<cdiv(static_cast<uint64_t>(n) * 32, 256), 256, 0, s>>>(ix, mon, slot, blk_off, matched, n, keys,
                                                                          n_keys);
}

size_t sort_keys_temp_bytes(uint32_t n, int end_bit) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, bytes, static_cast<const unsigned long long*>(nullptr),
                                 static_cast<unsigned long long*>(nullptr), n, 0, end_bit);
  return bytes;
}

void launch_sort_keys(void* temp, size_t temp_bytes, const unsigned long long* in, unsigned long long* out, uint32_t n,
                      int end_bit, cudaStream_t s) {
  cub::DeviceRadixSort::SortKeys(temp, temp_bytes, in, out, n, 0, end_bit, s);
}

// ---------------------------------------------------------------------------------
// Diagnostic (no reference counterpart): per entry matched by the last admitted
// batch, the histogram of that batch's accesses over users and its Shannon entropy in bits.
// (entry slot, user) keys of every matched block -> radix sort -> run-length encode (per-user
// counts) -> reduce by entry (accesses T, distinct users D, sum c log2 c) -> H = log2 T - S / T.
// The monitor's flags stay on the reference predicate (u / h, monitor.hpp:68-70).
// ---------------------------------------------------------------------------------
struct EntHist {
  unsigned long long accesses;
  unsigned long long users;
  double clogc;  // sum over users of c * log2(c)
};
struct EntHistSum {
  __host__ __device__ EntHist operator()(const EntHist& a, const EntHist& b) const {
    return EntHist{a.accesses + b.accesses, a.users + b.users, a.clogc + b.clogc};
  }
};

__global__ void k_entropy_emit(const uint32_t* __restrict__ blk_off, const uint32_t* __restrict__ matched,
                               const uint32_t* __restrict__ slot, const uint32_t* __restrict__ uidx, uint32_t n,
                               unsigned long long* keys, uint32_t* n_keys, uint32_t cap) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; p < n; p += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t bo = blk_off[p], m = matched[p];
    const unsigned long long u = uidx[p];
    for (uint32_t b = lane; b < m; b += 32) {
      const uint32_t k = atomicAdd(n_keys, 1u);
      if (k < cap) keys[k] = (static_cast<unsigned long long>(slot[bo + b]) << 32) | u;
    }
  }
}

__global__ void k_entropy_runs(const unsigned long long* __restrict__ ukeys, const uint32_t* __restrict__ counts,
                               const uint32_t* __restrict__ n_runs, uint32_t* __restrict__ eslot,
                               EntHist* __restrict__ vals) {
  const uint32_t n = *n_runs;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double c = counts[i];
    eslot[i] = static_cast<uint32_t>(ukeys[i] >> 32);
    vals[i] = EntHist{counts[i], 1ull, c * log2(c)};
  }
}

__global__ void k_entropy_out(Index ix, const uint32_t* __restrict__ eslot, const EntHist* __restrict__ h,
                              const uint32_t* __restrict__ n_seg, uint64_t* __restrict__ out_h,
                              uint64_t* __restrict__ out_d, uint64_t* __restrict__ out_acc,
                              uint64_t* __restrict__ out_users, double* __restrict__ out_bits) {
  const uint32_t n = *n_seg;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const Rec& r = ix.e[eslot[i]].rec;
    const double T = static_cast<double>(h[i].accesses);
    out_h[i] = r.h;
    out_d[i] = r.d;
    out_acc[i] = h[i].accesses;
    out_users[i] = h[i].users;
    out_bits[i] = log2(T) - h[i].clogc / T;
  }
}

// Returns the entries written (<= cap); *total = the batch's matched entries
uint32_t launch_access_entropy(const Index& ix, const uint32_t* blk_off, const uint32_t* matched,
                               const uint32_t* slot, const uint32_t* uidx, uint32_t n_prompts, uint32_t n_access,
                               uint64_t* out_h, uint64_t* out_d, uint64_t* out_acc, uint64_t* out_users,
                               double* out_bits, uint32_t cap, uint32_t* total, cudaStream_t s) {
  std::vector<void*> tmp;
  auto alloc = [&](size_t bytes) {
    void* p = nullptr;
    if (cudaMalloc(&p, std::max<size_t>(bytes, 16)) != cudaSuccess) {
      for (void* q : tmp) cudaFree(q);
      throw std::runtime_error("cudaMalloc: access entropy scratch");
    }
    tmp.push_back(p);
    return p;
  };
  const uint32_t n = std::max<uint32_t>(n_access, 1);
  auto* keys = static_cast<unsigned long long*>(alloc(8ull * n));
  auto* sorted = static_cast<unsigned long long*>(alloc(8ull * n));
  auto* ukeys = static_cast<unsigned long long*>(alloc(8ull * n));
  auto* counts = static_cast<uint32_t*>(alloc(4ull * n));
  auto* eslot = static_cast<uint32_t*>(alloc(4ull * n));
  auto* seg = static_cast<uint32_t*>(alloc(4ull * n));
  auto* vals = static_cast<EntHist*>(alloc(sizeof(EntHist) * n));
  auto* hist = static_cast<EntHist*>(alloc(sizeof(EntHist) * n));
  auto* ctr = static_cast<uint32_t*>(alloc(16));
  cudaMemsetAsync(ctr, 0, 16, s);
  k_entropy_emit<<<std::max<uint32_t>(1, std::min<uint32_t>(cdiv(static_cast<uint64_t>(n_prompts) * 32, 256), 4096)),
                   256, 0, s>>>(blk_off, matched, slot, uidx, n_prompts, keys, ctr, n);
  size_t b1 = 0, b2 = 0, b3 = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, b1, keys, sorted, n_access, 0, 64, s);
  cub::DeviceRunLengthEncode::Encode(nullptr, b2, sorted, ukeys, counts, ctr + 1, n_access, s);
  cub::DeviceReduce::ReduceByKey(nullptr, b3, eslot, seg, vals, hist, ctr + 2, EntHistSum{}, n_access, s);
  void* t = alloc(std::max({b1, b2, b3}));
  const size_t tb = std::max({b1, b2, b3});
  cub::DeviceRadixSort::SortKeys(t, b1 = tb, keys, sorted, n_access, 0, 64, s);
  cub::DeviceRunLengthEncode::Encode(t, b2 = tb, sorted, ukeys, counts, ctr + 1, n_access, s);
  uint32_t h_runs = 0;
  cudaMemcpyAsync(&h_runs, ctr + 1, 4, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  k_entropy_runs<<<std::max<uint32_t>(1, cdiv(h_runs, 256)), 256, 0, s>>>(ukeys, counts, ctr + 1, eslot, vals);
  cub::DeviceReduce::ReduceByKey(t, b3 = tb, eslot, seg, vals, hist, ctr + 2, EntHistSum{}, h_runs, s);
  uint32_t h_seg = 0;
  cudaMemcpyAsync(&h_seg, ctr + 2, 4, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  const uint32_t w = std::min(h_seg, cap);
  if (w) {
    cudaMemcpyAsync(ctr + 3, &w, 4, cudaMemcpyHostToDevice, s);
    k_entropy_out<<<cdiv(w, 256), 256, 0, s>>>(ix, seg, hist, ctr + 3, out_h, out_d, out_acc, out_users, out_bits);
  }
  const cudaError_t e = cudaStreamSynchronize(s);
  for (void* q : tmp) cudaFree(q);
  if (e != cudaSuccess) throw std::runtime_error(std::string("access entropy: ") + cudaGetErrorString(e));
  *total = h_seg;
  return w;
}

// ---------------------------------------------------------------------------------
// Eviction (RadixCacheIndex::evict / select_victim, cache_index.hpp:281-292,697-728).
//
// The reference frees, one at a time, the unpinned HBM leaf with the oldest access epoch,
// Public before non-Public, then the smallest node id; freeing a leaf can expose its
// parent.  A parent's access epoch is never below a child's (every match or insert walk
// that refreshes a node refreshes its whole root path), so this greedy order is the
// order of eff(X) = max(key(X), eff(children)) with children before parents on equal
// eff (a parent that inherits its deepest descendant's key goes right after it); a node
// off HBM never leaves, and blocks every ancestor (eff = +inf).  One evict(V) therefore
// tombstones the V smallest (eff, depth desc) live entries: eff by upward atomicMax,
// then two stable radix sorts (depth desc, then eff).
// ---------------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long evict_key(const Index& ix, uint64_t s) {
  const uint32_t m = ix.e[s].rec.meta;
  if (meta_tier(m) != SKV_TIER_HBM) return ~0ull;
  const EvictMeta em = ix.em[s];
  return (static_cast<unsigned long long>(em.access_epoch) << 32) |
         (static_cast<unsigned long long>(meta_label(m) != SKV_LABEL_PUBLIC) << 31) | (em.node_id & 0x7fffffffu);
}

__global__ void k_touch_matched(Index ix, const uint32_t* __restrict__ slot, const uint32_t* __restrict__ blk_off,
                                const uint32_t* __restrict__ matched, uint32_t n, uint32_t epoch) {
  const uint32_t p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (p >= n) return;
  const uint32_t bo = blk_off[p], m = matched[p];
  for (uint32_t b = lane_id(); b < m; b += 32) ix.em[slot[bo + b]].access_epoch = epoch;
}

// Node ids (cache_index.hpp:193,537): insert() allocates id X for a prompt's new suffix
// node, ensure_boundary then splits off its top block f-1 times, each split's upper half
// taking the next id -- block j of the f created blocks gets X+1+j, the deepest keeps X;
// X runs over the prompts in order.  The commit writes these ids speculatively with
// f = blocks missing before the batch; only a batch with duplicate claims (a lower prompt
// creating a block first, or a tombstone re-inserted) needs the exact pass below.
__global__ void k_nodes_spec(const uint32_t* __restrict__ blk_off, const uint32_t* __restrict__ exist, uint32_t n,
                             uint32_t* counts) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) counts[p] = blk_off[p + 1] - blk_off[p] - exist[p];
}

// every block before the prompt's first new one was walked by its insert: access epoch
__global__ void k_path_epochs(Index ix, const uint32_t* __restrict__ slot, const uint32_t* __restrict__ blk_off,
                              const uint32_t* __restrict__ exist, uint32_t n, uint32_t epoch) {
  const uint32_t p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (p >= n) return;
  const uint32_t bo = blk_off[p], k0 = exist[p];
  for (uint32_t b = lane_id(); b < k0; b += 32) ix.em[slot[bo + b]].access_epoch = epoch;
}

// exact pass, 1: blocks this prompt created = new blocks whose final claimant it is
__global__ void k_nodes_count(Index ix, const uint32_t* __restrict__ slot, const uint32_t* __restrict__ blk_off,
                              const uint32_t* __restrict__ exist, uint32_t n, uint32_t* counts) {
  const uint32_t p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (p >= n) return;
  const uint32_t bo = blk_off[p], nb = blk_off[p + 1] - bo;
  uint32_t f = 0;
  for (uint32_t b = exist[p] + lane_id(); b < nb; b += 32) {
    const uint32_t s = slot[bo + b];
    f += (s != kNone && meta_prompt(ix.e[s].rec.meta) == p) ? 1u : 0u;
  }
  f = __reduce_add_sync(kFull, f);
  if (lane_id() == 0) counts[p] = f;
}

// exact pass, 2: the created blocks are the prompt's last f (a lower prompt sharing block
// b shares every block before it)
__global__ void k_nodes_assign(Index ix, const uint32_t* __restrict__ slot, const uint32_t* __restrict__ blk_off,
                               uint32_t n, const uint32_t* __restrict__ counts, const uint32_t* __restrict__ incl,
                               uint64_t next_id) {
  const uint32_t p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (p >= n) return;
  const uint32_t f = counts[p];
  if (!f) return;
  const uint32_t bo = blk_off[p], nb = blk_off[p + 1] - bo, k = nb - f;
  const uint64_t X = next_id + incl[p] - f;
  for (uint32_t j = lane_id(); j < f; j += 32)
    ix.em[slot[bo + k + j]].node_id = static_cast<uint32_t>(j + 1 < f ? X + 1 + j : X);
}

__global__ void k_evict_init(Index ix, unsigned long long* eff) {
  const uint64_t s = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s > ix.mask) return;
  const Rec& r = ix.e[s].rec;
  eff[s] = ((r.h == 0 && r.d == 0) || !meta_live(r.meta)) ? 0ull : evict_key(ix, s);
}

__global__ void k_evict_propagate(Index ix, unsigned long long* eff) {
  const uint64_t s = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s > ix.mask) return;
  unsigned long long v = eff[s];
  if (!v) return;
  for (uint32_t p = ix.e[s].rec.parent; p != kNone; p = ix.e[p].rec.parent) {
    const unsigned long long old = atomicMax(&eff[p], v);
    if (old >= v) break;
  }
}

__global__ void k_evict_compact(Index ix, const unsigned long long* __restrict__ eff, unsigned long long* keys,
                                uint32_t* vals, uint32_t* n_live) {
  const uint64_t s = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s > ix.mask) return;
  const unsigned long long v = eff[s];
  if (v == 0 || v == ~0ull) return;
  const uint32_t i = atomicAdd(n_live, 1u);
  keys[i] = ~static_cast<unsigned long long>(ix.em[s].depth) & 0xffffffffull;  // deeper first
  vals[i] = static_cast<uint32_t>(s);
}

// tiered demotion (RadixCacheIndex tiered_demotion, evict_or_demote :743-766, lower tiers
// unbounded): a victim moves HBM -> DRAM and stays in the tree as a leaf, so no parent is
// ever exposed and the victims are simply the smallest-key HBM leaves
__global__ void k_evict_children(Index ix, unsigned long long* flag) {
  const uint64_t s = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s > ix.mask) return;
  const Rec& r = ix.e[s].rec;
  if ((r.h == 0 && r.d == 0) || !meta_live(r.meta)) return;
  if (r.parent != kNone) flag[r.parent] = 1;
}

__global__ void k_evict_leaves(Index ix, const unsigned long long* __restrict__ flag, unsigned long long* keys,
                               uint32_t* vals, uint32_t* n_live) {
  const uint64_t s = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s > ix.mask) return;
  const Rec& r = ix.e[s].rec;
  if ((r.h == 0 && r.d == 0) || !meta_live(r.meta) || flag[s]) return;
  const unsigned long long k = evict_key(ix, s);
  if (k == ~0ull) return;  // not in HBM
  const uint32_t i = atomicAdd(n_live, 1u);
  keys[i] = k;
  vals[i] = static_cast<uint32_t>(s);
}

__global__ void k_evict_demote(Index ix, const uint32_t* __restrict__ vals, uint32_t v, uint64_t* vh, uint64_t* vd) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= v) return;
  Rec& r = ix.e[vals[i]].rec;
  r.meta = (r.meta & ~(3u << 3)) | (static_cast<uint32_t>(SKV_TIER_DRAM) << 3);
  if (vh) vh[i] = r.h;
  if (vd) vd[i] = r.d;
}

__global__ void k_evict_gather(const unsigned long long* __restrict__ eff, const uint32_t* __restrict__ vals,
                               unsigned long long* keys, const uint32_t* n_live) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < *n_live) keys[i] = eff[vals[i]];
}

// tombstones: the key stays (linear probing and re-insertion find it), live = 0, the
// claiming-prompt field at its maximum so a re-insert's atomicMin picks its claimant
__global__ void k_evict_mark(Index ix, const uint32_t* __restrict__ vals, uint32_t v, uint64_t* vh, uint64_t* vd) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= v) return;
  const uint32_t s = vals[i];
  Rec& r = ix.e[s].rec;
  r.meta = (r.meta & 0x1fu) | 0xffffff00u;  // label/owner/tier kept, live cleared
  ix.em[s].dead = 1;
  if (vh) vh[i] = r.h;
  if (vd) vd[i] = r.d;
}

void launch_touch_matched(const Index& ix, const uint32_t* slot, const uint32_t* blk_off, const uint32_t* matched,
                          uint32_t n, uint32_t epoch, cudaStream_t s) {
  if (n) k_touch_matched<<<cdiv(static_cast<uint64_t>(n) * 32, 256), 256, 0, s>>>(ix, slot, blk_off, matched, n, epoch);
}

bool node_ids_speculative() { return !SKV_COMMIT_FLAT; }  // the flat commit leaves them to the exact pass

void launch_chain(const uint64_t* d, const uint32_t* blk_off, const uint32_t* first_sens, uint32_t n, uint64_t* h,
                  uint8_t* label, uint32_t* slot, cudaStream_t s) {
  if (n) k_chain<<<cdiv(n, 32 * kCHWarps), 32 * kCHWarps, 0, s>>>(d, blk_off, first_sens, n, h, label, slot);
}

void launch_node_bases(const uint32_t* blk_off, const uint32_t* exist, uint32_t n, uint32_t* counts, uint32_t* base,
                       void* temp, size_t temp_bytes, cudaStream_t s) {
  if (!n) return;
  k_nodes_spec<<<cdiv(n, 256), 256, 0, s>>>(blk_off, exist, n, counts);
  cub::DeviceScan::ExclusiveSum(temp, temp_bytes, counts, base, n, s);
}

void launch_path_epochs(const Index& ix, const uint32_t* slot, const uint32_t* blk_off, const uint32_t* exist,
                        uint32_t n, uint32_t epoch, cudaStream_t s) {
  if (n) k_path_epochs<<<cdiv(static_cast<uint64_t>(n) * 32, 256), 256, 0, s>>>(ix, slot, blk_off, exist, n, epoch);
}

void launch_assign_nodes(const Index& ix, const uint32_t* slot, const uint32_t* blk_off, const uint32_t* exist,
                         uint32_t n, uint32_t* counts, uint32_t* incl, uint64_t next_id, void* temp,
                         size_t temp_bytes, cudaStream_t s) {
  if (!n) return;
  const unsigned g = static_cast<unsigned>(cdiv(static_cast<uint64_t>(n) * 32, 256));
  k_nodes_count<<<g, 256, 0, s>>>(ix, slot, blk_off, exist, n, counts);
  cub::DeviceScan::InclusiveSum(temp, temp_bytes, counts, incl, n, s);
  k_nodes_assign<<<g, 256, 0, s>>>(ix, slot, blk_off, n, counts, incl, next_id);
}

size_t evict_temp_bytes(uint32_t n_prompts, uint64_t cap) {
  size_t a = 0, b = 0;
  cub::DeviceScan::InclusiveSum(nullptr, a, static_cast<const uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                                std::max<uint32_t>(n_prompts, 1));
  cub::DeviceRadixSort::SortPairs(nullptr, b, static_cast<const unsigned long long*>(nullptr),
                                  static_cast<unsigned long long*>(nullptr), static_cast<const uint32_t*>(nullptr),
                                  static_cast<uint32_t*>(nullptr), static_cast<int>(std::min<uint64_t>(cap, 1u << 31)));
  return std::max(a, b);
}

uint32_t launch_evict(const Index& ix, uint64_t needed, unsigned long long* eff, unsigned long long* keys_a,
                      unsigned long long* keys_b, uint32_t* vals_a, uint32_t* vals_b, uint32_t* n_live, void* temp,
                      size_t temp_bytes, uint64_t* victims_h, uint64_t* victims_d, uint32_t* host_n, int tiered,
                      cudaStream_t s) {
  const unsigned g = static_cast<unsigned>(cdiv(ix.cap, 256));
  cudaMemsetAsync(n_live, 0, 4, s);
  if (tiered) {
    cudaMemsetAsync(eff, 0, ix.cap * sizeof(unsigned long long), s);
    k_evict_children<<<g, 256, 0, s>>>(ix, eff);
    k_evict_leaves<<<g, 256, 0, s>>>(ix, eff, keys_a, vals_a, n_live);
    cudaMemcpyAsync(host_n, n_live, 4, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    const uint32_t n = *host_n;
    if (n) cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_a, keys_b, vals_a, vals_b, static_cast<int>(n), 0, 64, s);
    const uint32_t v = static_cast<uint32_t>(std::min<uint64_t>(needed, n));
    if (v) k_evict_demote<<<cdiv(v, 256), 256, 0, s>>>(ix, vals_b, v, victims_h, victims_d);
    return v;
  }
  k_evict_init<<<g, 256, 0, s>>>(ix, eff);
  k_evict_propagate<<<g, 256, 0, s>>>(ix, eff);
  k_evict_compact<<<g, 256, 0, s>>>(ix, eff, keys_a, vals_a, n_live);
  cudaMemcpyAsync(host_n, n_live, 4, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  const uint32_t n = *host_n;
  if (n) {
    cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_a, keys_b, vals_a, vals_b, static_cast<int>(n), 0, 32, s);
    k_evict_gather<<<cdiv(n, 256), 256, 0, s>>>(eff, vals_b, keys_a, n_live);
    cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_a, keys_b, vals_b, vals_a, static_cast<int>(n), 0, 64, s);
  }
  const uint32_t v = static_cast<uint32_t>(std::min<uint64_t>(needed, n));
  if (v) k_evict_mark<<<cdiv(v, 256), 256, 0, s>>>(ix, vals_a, v, victims_h, victims_d);
  return v;
}

void launch_record_replay(const Index& ix, const MonCtx& mon, const uint32_t* replay, const uint32_t* n_replay,
                          const unsigned long long* keys, uint32_t n_keys, const uint64_t* users, int grid,
                          cudaStream_t s) {
  k_record_replay<<<grid, 256, 0, s>>>(ix, mon, replay, n_replay, keys, n_keys, users);
}

void launch_commit(const Index& ix, const uint64_t* h, const uint64_t* d, const uint32_t* blk_off,
                   const uint32_t* exist, const uint8_t* label, const uint32_t* users, const uint8_t* owners,
                   uint32_t n, uint32_t* slot, unsigned long long* n_new, uint32_t* fix_list, uint32_t* n_fix,
                   uint32_t fix_cap, uint32_t* err_flag, int fix_grid, const uint32_t* matched,
                   const uint64_t* users64, const MonCtx* mon, int pending_labels, uint64_t n_blocks, int n_sm,
                   const uint32_t* bprompt, uint32_t* late, uint32_t* n_late, uint32_t* n_revived,
                   const MonCtx& pool, cudaStream_t s) {
  const MonCtx M = mon ? *mon : MonCtx{};
  if (!n) return;
#if SKV_COMMIT_FLAT
  {
    auto* kern = mon ? k_commit_flat<true> : k_commit_flat<false>;
    kern<<<static_cast<unsigned>(std::min<uint64_t>(cdiv(std::max<uint64_t>(n_blocks, 1), 32ull * kCommitRounds * 8),
                                                    8ull * n_sm)),
           256, 0, s>>>(ix, h, d, blk_off, bprompt, label, users, owners, n, slot, n_new, fix_list, n_fix, fix_cap,
                        late, n_late, err_flag, matched, users64, M, pending_labels);
    k_commit_fixup_min<<<fix_grid, 256, 0, s>>>(ix, fix_list, n_fix, fix_cap);
    k_commit_fixup<<<fix_grid, 256, 0, s>>>(ix, blk_off, label, users, owners, fix_list, n_fix, fix_cap,
                                            pending_labels, n_revived, pool);
    k_commit_links<<<fix_grid, 256, 0, s>>>(ix, slot, late, n_late, fix_cap);
    return;
  }
#endif
  auto* kern = mon ? k_commit<true> : k_commit<false>;
#if SKV_COMMIT_PERSIST
  const unsigned cgrid = static_cast<unsigned>(std::min<uint64_t>(cdiv(static_cast<uint64_t>(n) * 32, 256),
                                                                   static_cast<uint64_t>(SKV_COMMIT_PERSIST) * n_sm));
#else
  const unsigned cgrid = static_cast<unsigned>(cdiv(static_cast<uint64_t>(n) * 32, 256));
#endif
  kern<<<cgrid, 256, 0, s>>>(
ix, h, d, blk_off, exist, label, users, owners, n,
                                                                    slot, n_new, fix_list, n_fix, fix_cap, err_flag,
                                                                    matched, users64, M, mon ? 1 : 0,
                                                                    pending_labels);
  k_commit_fixup_min<<<fix_grid, 256, 0, s>>>(ix, fix_list, n_fix, fix_cap);
  k_commit_fixup<<<fix_grid, 256, 0, s>>>(ix, blk_off, label, users, owners, fix_list, n_fix, fix_cap,
                                          pending_labels, n_revived, pool);
}

void launch_epoch_candidates(const Index& ix, const uint32_t* list, const uint32_t* n_list, uint32_t grid_n,
                             int only_untouched, uint32_t stamp, double jump, uint64_t u_pre_max, uint32_t* cands,
                             uint32_t* n_cands, cudaStream_t s, const uint32_t* guard) {
  if (grid_n)
    k_epoch_candidates<<<cdiv(grid_n, 256), 256, 0, s>>>(ix, list, n_list, only_untouched, stamp, jump, u_pre_max,
                                                          cands, n_cands, guard);
}

void launch_epoch_fire(const Index& ix, const uint32_t* cands, const uint32_t* n_cands, uint32_t grid_n,
                       uint32_t stamp, uint64_t epoch, void* events, uint32_t* n_events, uint32_t* fired,
                       cudaStream_t s, const uint32_t* guard) {
  if (grid_n)
    k_epoch_fire<<<cdiv(grid_n, 256), 256, 0, s>>>(ix, cands, n_cands, stamp, epoch, static_cast<DevEvent*>(events),
                                                    n_events, fired, guard);
}

void launch_epoch_propagate(const Index& ix, const uint32_t* fired, const uint32_t* n_events, uint32_t grid_n,
                            cudaStream_t s, const uint32_t* guard) {
  if (grid_n) k_epoch_propagate<<<cdiv(grid_n, 256), 256, 0, s>>>(ix, fired, n_events, guard);
}

int epoch_fused_grid(int device) {
  static int grid[16] = {};
  if (device < 0 || device >= 16) return 0;
  if (!grid[device]) {
    int per_sm = 0, n_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_epoch_fused, 256, 0) != cudaSuccess ||
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, device) != cudaSuccess)
      return 0;
    // two CTAs per SM: the fused pass serves small windows (large ones take the six kernels), where
    // the grid syncs, not memory parallelism, bound it (config 2: 0.037 -> 0.030 ms)
    grid[device] = std::max(1, std::min(per_sm, 2) * n_sm);
  }
  return grid[device];
}

cudaError_t launch_epoch_fused(const Index& ix, uint32_t* const lists[2], uint32_t* ntb, int cur, uint32_t stamp,
                               double jump, uint64_t u_pre_max, uint32_t* cands, uint32_t* n_cands, uint64_t epoch,
                               void* events, uint32_t* n_events, uint32_t* fired, uint32_t* pool_count,
                               const uint32_t* st, const uint32_t* guard, int device, cudaStream_t s) {
  Index ixv = ix;
  DevEvent* ev = static_cast<DevEvent*>(events);
  uint32_t* l0 = lists[0];
  uint32_t* l1 = lists[1];
  void* args[] = {&ixv, &l0, &l1, &ntb, &cur, &stamp, &jump, &u_pre_max, &cands, &n_cands,
                  &epoch, &ev, &n_events, &fired, &pool_count, &st, &guard};
  const int grid = epoch_fused_grid(device);
  if (grid <= 0) return cudaErrorCooperativeLaunchTooLarge;
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_epoch_fused), dim3(grid), dim3(256), args, 0, s);
}

void launch_epoch_roll(const Index& ix, const uint32_t* list, const uint32_t* n_list, uint32_t grid_n, int prev_list,
                       cudaStream_t s, const uint32_t* guard) {
  if (grid_n) k_epoch_roll<<<cdiv(grid_n, 256), 256, 0, s>>>(ix, list, n_list, prev_list, guard);
}

void launch_epoch_reset(uint32_t* pool_count, uint32_t* prev_count, const uint32_t* guard, cudaStream_t s) {
  k_epoch_reset<<<1, 1, 0, s>>>(pool_count, prev_count, guard);
}

void launch_resolve(const Index& ix, const uint64_t* h, const uint64_t* d, const uint32_t* boff, uint32_t n_prompts,
                    const uint32_t* first, const uint8_t* labels, uint32_t n, uint32_t* missing, cudaStream_t s) {
  if (!n_prompts) return;
  if (n) k_resolve_public<<<cdiv(n, 256), 256, 0, s>>>(ix, h, d, boff, n_prompts, first, labels, n, missing);
  // severity order: Private landings, then Restricted (a Restricted ancestor wins an overlap)
  k_resolve_private<<<cdiv(n_prompts, 128), 128, 0, s>>>(ix, h, d, boff, n_prompts, first, labels,
                                                          SKV_LABEL_PRIVATE, missing);
  k_resolve_private<<<cdiv(n_prompts, 128), 128, 0, s>>>(ix, h, d, boff, n_prompts, first, labels,
                                                          SKV_LABEL_RESTRICTED, missing);
}

void launch_set_tiers(const Index& ix, const uint64_t* h, const uint64_t* d, const uint32_t* boff, uint32_t n_prompts,
                      const uint8_t* tiers, uint32_t n, cudaStream_t s) {
  if (n) k_set_tiers<<<cdiv(n, 256), 256, 0, s>>>(ix, h, d, boff, n_prompts, tiers, n);
}

void launch_export(const Index& ix, const uint64_t* user_rev, void* out, uint32_t* n_out, uint32_t cap,
                   cudaStream_t s) {
  k_export<<<cdiv(ix.cap, 256), 256, 0, s>>>(ix, user_rev, static_cast<skv_entry*>(out), n_out, cap);
}

void launch_scan_text(const uint8_t* text, uint32_t len, DevRules r, uint32_t* mask, uint32_t shift, cudaStream_t s) {
  k_scan_text<<<1, 32, 0, s>>>(text, len, r, mask, shift);
}

void launch_scan_texts(const uint8_t* text, const uint64_t* off, uint32_t n, DevRules r, uint32_t* masks,
                       uint32_t shift, cudaStream_t s) {
  if (n) k_scan_texts<<<cdiv(n, 128), 128, 0, s>>>(text, off, n, r, masks, shift);
}

void launch_digest(const uint32_t* tokens, uint32_t n, uint64_t* out, cudaStream_t s) {
  k_digest<<<1, 32, 0, s>>>(tokens, n, out);
}

}  // namespace skv

namespace skv {
namespace {
__global__ void k_init_entries(Index ix) {
  const uint64_t s = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s > ix.mask) return;
  ulonglong2* p = reinterpret_cast<ulonglong2*>(&ix.e[s]);
  const ulonglong2 z = {0ull, 0ull};
  p[0] = z;                                        // key (0,0) = empty
  p[1] = {0ull, 0xffffffffffffffffull};            // creator, meta = 0; parent, first_child = none
  p[2] = z;                                        // AccessStats window
  p[3] = {0xffffffffffffffffull, 0ull};            // next_sibling, set_idx = none; mark = 0
}
}  // namespace

// UserId -> u32 index (insert if absent).  One thread per prompt; the slot's inserter
// allocates the index, everyone else waits for it to be published.
__global__ void k_intern_users(UserTable t, const uint64_t* __restrict__ users, uint32_t n, uint32_t* __restrict__ uidx,
                               uint32_t* err) {
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const unsigned long long u = users[p];
  if (u == kNoUser) {  // index 0 is reserved for the one UserId equal to the empty marker
    uidx[p] = 0;
    return;
  }
  uint32_t s = static_cast<uint32_t>(slot_hash(u, 0x5bd1e995ull)) & t.mask;
  for (uint32_t i = 0; i <= t.mask; ++i, s = (s + 1) & t.mask) {
    unsigned long long k = *reinterpret_cast<volatile unsigned long long*>(&t.keys[s]);
    if (k == kNoUser) k = atomicCAS(&t.keys[s], kNoUser, u);
    if (k == kNoUser) {  // inserted: allocate (index 0 is reserved)
      const uint32_t id = atomicAdd(t.count, 1u) + 1;
      if (id >= t.cap) atomicOr(err, 8u);  // k_commit then inserts nothing (no creator past the table)
      if (id < t.cap) t.rev[id] = u;
      __threadfence();
      atomicExch(&t.idx[s], id + 1);
      uidx[p] = id < t.cap ? id : 0u;
      return;
    }
    if (k == u) {
      uint32_t v;
      while ((v = *reinterpret_cast<volatile uint32_t*>(&t.idx[s])) == 0) {
      }
      uidx[p] = v - 1 < t.cap ? v - 1 : 0u;
      return;
    }
  }
  atomicOr(err, 8u);
}

void launch_intern_users(const UserTable& t, const uint64_t* users, uint32_t n, uint32_t* uidx, uint32_t* err,
                         cudaStream_t s) {
  if (n) k_intern_users<<<cdiv(n, 256), 256, 0, s>>>(t, users, n, uidx, err);
}

void launch_init_entries(const Index& ix, cudaStream_t s) {
  k_init_entries<<<static_cast<uint32_t>((ix.cap + 255) / 256), 256, 0, s>>>(ix);
}

// ---------------------------------------------------------------------------------
// Replicated layer (multi-GPU): export of a rank's new replicated-layer
// entries and aggregated accesses, application of the merge of all ranks' exports.
// ---------------------------------------------------------------------------------
namespace {
static_assert(sizeof(skv_rep_entry) == 56 && sizeof(skv_rep_access) == 40, "replica record layouts");

__global__ void k_rep_export_new(Index ix, const uint64_t* __restrict__ user_rev, const uint64_t* __restrict__ gids,
                                 skv_rep_entry* out, uint32_t n) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Rec r = ix.e[ix.rep.new_list[i]].rec;
  skv_rep_entry o;
  o.h = r.h;
  o.d = r.d;
  o.ph = o.pd = 0;
  if (r.parent != kNone) {
    o.ph = ix.e[r.parent].rec.h;
    o.pd = ix.e[r.parent].rec.d;
  }
  o.creator = user_rev[r.creator];
  o.gid = gids[meta_prompt(r.meta)];
  o.label = static_cast<uint8_t>(meta_label(r.meta));
  o.owner = static_cast<uint8_t>(meta_owner(r.meta));
  for (int k = 0; k < 6; ++k) o.pad[k] = 0;
  out[i] = o;
}

__global__ void k_rep_export_acc(Index ix, const uint64_t* __restrict__ gids, skv_rep_access* out, uint32_t* n_out,
                                 uint32_t cap) {
  const uint32_t h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h > ix.rep.pair_mask) return;
  const ulonglong2 key = ix.rep.pair_key[h];
  if (key.y == 0) return;
  const uint32_t slot = static_cast<uint32_t>(key.y - 1);
  const uint32_t k = atomicAdd(n_out, 1u);
  if (k >= cap) return;
  skv_rep_access o;
  o.h = ix.e[slot].rec.h;
  o.d = ix.e[slot].rec.d;
  o.user = key.x;
  o.gid = gids[ix.rep.pair_first[h]];
  o.count = ix.rep.pair_cnt[h];
  out[k] = o;
}

__global__ void k_rep_clear(RepLayer R) {
  const uint32_t h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h > R.pair_mask) return;
  R.pair_key[h] = make_ulonglong2(0ull, 0ull);
  R.pair_first[h] = 0xffffffffu;
  R.pair_gid[h] = ~0ull;
  R.pair_cnt[h] = 0;
}

// slot of an existing key (the replicated layer is identical on every rank), kNone if absent
__device__ uint32_t rep_find(const Index& ix, uint64_t h, uint64_t d) {
  uint64_t s = home_slot(ix, h, d, 0);
  for (uint64_t i = 0; i <= ix.mask; ++i, s = (s + 1) & ix.mask) {
    const ulonglong2 k = *reinterpret_cast<const ulonglong2*>(&ix.e[s].rec);
    if (k.x == h && k.y == d) return static_cast<uint32_t>(s);
    if (k.x == 0 && k.y == 0) return kNone;
  }
  return kNone;
}

// merged entries (one per key, the global first creator's payload): claim absent keys, write the
// winner's creator / label / owner into every copy
__global__ void k_rep_apply_claim(Index ix, const skv_rep_entry* __restrict__ ents, const uint32_t* __restrict__ uidx,
                                  uint32_t n, uint32_t* slot_out, uint32_t* n_claimed, uint32_t* err) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const skv_rep_entry r = ents[i];
  uint64_t s = home_slot(ix, r.h, r.d, 0);
  bool claimed = false, ok = false;
  for (uint64_t k = 0; k <= ix.mask; ++k, s = (s + 1) & ix.mask) {
    unsigned long long ol, oh;
    if (cas128(reinterpret_cast<unsigned long long*>(&ix.e[s].rec), 0ull, 0ull, r.h, r.d, &ol, &oh)) {
      claimed = ok = true;
      break;
    }
    if (ol == r.h && oh == r.d) {
      ok = true;
      break;
    }
  }
  if (!ok) {
    atomicOr(err, 2u);
    slot_out[i] = kNone;
    return;
  }
  Rec& e = ix.e[s].rec;
  const uint32_t old = claimed ? 0u : e.meta;
  *reinterpret_cast<uint2*>(&e.creator) =
      make_uint2(uidx[i], make_meta(r.label, r.owner, claimed ? SKV_TIER_HBM : meta_tier(old), meta_prompt(old)));
  slot_out[i] = claimed ? (static_cast<uint32_t>(s) | 0x80000000u) : static_cast<uint32_t>(s);
  if (claimed) atomicAdd(n_claimed, 1u);
}

// parent links of the entries the claim pass created (their parents exist now)
__global__ void k_rep_apply_link(Index ix, const skv_rep_entry* __restrict__ ents, const uint32_t* __restrict__ slots,
                                 uint32_t n, uint32_t* err) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || slots[i] == kNone || !(slots[i] & 0x80000000u)) return;
  const uint32_t s = slots[i] & 0x7fffffffu;
  const skv_rep_entry r = ents[i];
  if (r.ph == 0 && r.pd == 0) return;  // a root
  const uint32_t ps = rep_find(ix, r.ph, r.pd);
  if (ps == kNone) {
    atomicOr(err, 4u);
    return;
  }
  ix.e[s].rec.parent = ps;
  const uint32_t sib = atomicExch(&ix.e[ps].rec.first_child, s);
  if (sib != kNone) ix.e[s].aux.next_sibling = sib;
}

// Device merge of the ranks' raw access exports (all ranks' records, any order): per (entry, user)
// the lowest first prompt id and the summed count (pair table keyed {user, slot + 1}) ...
__global__ void k_rep_merge_insert(Index ix, const skv_rep_access* __restrict__ accs, uint32_t n, uint32_t* err) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const skv_rep_access a = accs[i];
  const uint32_t slot = rep_find(ix, a.h, a.d);
  if (slot == kNone) {
    atomicOr(err, 8u);
    return;
  }
  const RepLayer& R = ix.rep;
  const ulonglong2 key = make_ulonglong2(a.user, static_cast<unsigned long long>(slot) + 1);
  uint32_t h = (mix32(a.user ^ (static_cast<uint64_t>(slot) << 32)) ^ slot * 0x9e3779b9u) & R.pair_mask;
  for (uint32_t t = 0; t <= R.pair_mask; ++t, h = (h + 1) & R.pair_mask) {
    ulonglong2 cur = ld_relaxed128(&R.pair_key[h]);
    if (cur.x == 0 && cur.y == 0) {
      ulonglong2 old;
      cas128_dev(&R.pair_key[h], make_ulonglong2(0, 0), key, &old);
      cur = old.x == 0 && old.y == 0 ? key : old;
    }
    if (cur.x == key.x && cur.y == key.y) {
      atomicMin(&R.pair_gid[h], static_cast<unsigned long long>(a.gid));
      atomicAdd(&R.pair_cnt[h], static_cast<uint32_t>(a.count));
      return;
    }
  }
  atomicOr(err, 1u);
}

// ... compacted as (first gid -> pair) for a sort by gid, then a stable sort by entry slot ...
__global__ void k_rep_merge_compact(RepLayer R, unsigned long long* gid_keys, uint32_t* vals, uint32_t* n_out) {
  const uint32_t h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h > R.pair_mask || R.pair_key[h].y == 0) return;
  const uint32_t k = atomicAdd(n_out, 1u);
  gid_keys[k] = R.pair_gid[h];
  vals[k] = h;
}

__global__ void k_rep_merge_slotkeys(RepLayer R, const uint32_t* __restrict__ vals, const uint32_t* __restrict__ n,
                                     uint32_t* slot_keys) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= *n) return;
  slot_keys[i] = static_cast<uint32_t>(R.pair_key[vals[i]].y - 1);
}

// ... and each entry's merged accesses replayed, one thread per entry, in global order against its
// window set (AccessStats::record, access_stats.hpp:27-37, with a user's repeats folded into its
// count: once admitted a user's later accesses add 0; a user not admitted on its first access
// never is, so each of its accesses adds 1)
__global__ void k_rep_apply_acc(Index ix, MonCtx M, const uint32_t* __restrict__ slot_keys,
                                const uint32_t* __restrict__ vals, const uint32_t* __restrict__ n_ptr) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t n = *n_ptr;
  if (i >= n || (i > 0 && slot_keys[i - 1] == slot_keys[i])) return;  // not the entry's first
  const RepLayer& R = ix.rep;
  const uint32_t s = slot_keys[i];
  Entry& e = ix.e[s];
  const uint32_t si = acquire_set(e, s, M);
  if (si == kNone) return;  // pool exhausted (M.err)
  SetHdr& hd = M.hdr[si];
  ulonglong2* tab = M.tab + static_cast<uint64_t>(si) * kSetSlots;
  uint32_t size = hd.size, hits = 0, ucnt = 0;
  for (uint32_t j = i; j < n && slot_keys[j] == s; ++j) {
    const uint32_t v = vals[j];
    const uint64_t u = R.pair_key[v].x;
    const uint32_t c = R.pair_cnt[v];
    hits += c;
    uint32_t pos = mix32(u) & (kSetSlots - 1), free_pos = kNone;
    bool member = false;
    for (uint32_t t = 0; t < kSetSlots; ++t, pos = (pos + 1) & (kSetSlots - 1)) {
      const ulonglong2 x = tab[pos];
      if (x.y < M.wstart) {
        free_pos = pos;
        break;
      }
      if (x.x == u) {
        member = true;
        break;
      }
    }
    if (member) continue;
    if (size < kMaxSetUsers && free_pos != kNone) {
      tab[free_pos] = make_ulonglong2(u, M.batch);
      ++size;
      ucnt += 1;
    } else {
      ucnt += c;  // saturated: every access of an untracked user counts as new (access_stats.hpp:33)
    }
  }
  e.stats.hit_cur += hits;
  e.stats.u_cnt += ucnt;
  hd.size = size;
}
}  // namespace

void launch_rep_export(const Index& ix, const uint64_t* user_rev, const uint64_t* gids, uint32_t n_new,
                       void* ents, void* accs, uint32_t* n_accs, uint32_t acc_cap, cudaStream_t s) {
  if (n_new) k_rep_export_new<<<cdiv(n_new, 256), 256, 0, s>>>(ix, user_rev, gids, static_cast<skv_rep_entry*>(ents),
                                                               n_new);
  k_rep_export_acc<<<cdiv(ix.rep.pair_mask + 1ull, 256), 256, 0, s>>>(ix, gids, static_cast<skv_rep_access*>(accs),
                                                                       n_accs, acc_cap);
}

void launch_rep_clear(const Index& ix, cudaStream_t s) {
  k_rep_clear<<<cdiv(ix.rep.pair_mask + 1ull, 256), 256, 0, s>>>(ix.rep);
}

size_t rep_sort_temp_bytes(uint32_t n) {
  size_t a = 0, b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, a, static_cast<const unsigned long long*>(nullptr),
                                  static_cast<unsigned long long*>(nullptr), static_cast<const uint32_t*>(nullptr),
                                  static_cast<uint32_t*>(nullptr), n);
  cub::DeviceRadixSort::SortPairs(nullptr, b, static_cast<const uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr),
                                  static_cast<const uint32_t*>(nullptr), static_cast<uint32_t*>(nullptr), n);
  return std::max(a, b);
}

void launch_rep_apply(const Index& ix, const MonCtx& M, const void* ents, const uint32_t* uidx, uint32_t n_ents,
                      uint32_t* slots, uint32_t* n_claimed, const void* accs, uint32_t n_accs, const RepScratch& W,
                      uint32_t* err, cudaStream_t s) {
  const auto* E = static_cast<const skv_rep_entry*>(ents);
  if (n_ents) {
    k_rep_apply_claim<<<cdiv(n_ents, 256), 256, 0, s>>>(ix, E, uidx, n_ents, slots, n_claimed, err);
    k_rep_apply_link<<<cdiv(n_ents, 256), 256, 0, s>>>(ix, E, slots, n_ents, err);
  }
  if (!n_accs) return;
  const uint32_t cap = ix.rep.pair_mask + 1;
  k_rep_merge_insert<<<cdiv(n_accs, 256), 256, 0, s>>>(ix, static_cast<const skv_rep_access*>(accs), n_accs, err);
  cudaMemsetAsync(W.n, 0, 4, s);
  k_rep_merge_compact<<<cdiv(cap, 256), 256, 0, s>>>(ix.rep, W.gid_a, W.val_a, W.n);
  // the pair count bounds the sorts: read it (one small copy) so they sort only the used pairs
  uint32_t np = 0;
  cudaMemcpyAsync(W.host_n, W.n, 4, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  np = *W.host_n;
  if (!np) return;
  size_t tb = W.temp_bytes;
  cub::DeviceRadixSort::SortPairs(W.temp, tb, W.gid_a, W.gid_b, W.val_a, W.val_b, np, 0, 64, s);
  k_rep_merge_slotkeys<<<cdiv(np, 256), 256, 0, s>>>(ix.rep, W.val_b, W.n, W.slot_a);
  int bits = 1;
  while ((1ull << bits) <= ix.mask) ++bits;
  tb = W.temp_bytes;
  cub::DeviceRadixSort::SortPairs(W.temp, tb, W.slot_a, W.slot_b, W.val_b, W.val_a, np, 0, bits, s);
  k_rep_apply_acc<<<cdiv(np, 256), 256, 0, s>>>(ix, M, W.slot_b, W.val_a, W.n);
}

// ---------------------------------------------------------------------------------
// Per-entry calls of the reference-API facade (include/safekv/): set_label / record_access /
// roll_window / check_anomaly on given entries, in call order (one thread: these are the
// reference's per-call operations, cache_index.hpp:312-315,385-393, monitor.hpp:56-81)
// ---------------------------------------------------------------------------------
namespace {
__global__ void k_find_entries(Index ix, const uint64_t* __restrict__ h, const uint64_t* __restrict__ d, uint32_t n,
                               uint32_t* slots) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t s = rep_find(ix, h[i], d[i]);
  slots[i] = (s != kNone && meta_live(ix.e[s].rec.meta)) ? s : kNone;
}

__device__ uint32_t label_subtree(const Index& ix, uint32_t root, uint32_t lab) {
  uint32_t changed = 0;
  uint32_t cur = ix.e[root].rec.first_child;
  while (cur != kNone) {
    const uint32_t m = ix.e[cur].rec.meta;
    if (meta_label(m) != lab) {
      ix.e[cur].rec.meta = (m & ~3u) | lab;
      ++changed;
    }
    const uint32_t c = ix.e[cur].rec.first_child;
    if (c != kNone) {
      cur = c;
      continue;
    }
    while (cur != root && ix.e[cur].aux.next_sibling == kNone) cur = ix.e[cur].rec.parent;
    if (cur == root) break;
    cur = ix.e[cur].aux.next_sibling;
  }
  return changed;
}

// label the entries (a facade node's blocks, root-first); with propagate, also every descendant
// of the last one (apply_label_subtree, cache_index.hpp:672-685)
__global__ void k_label_entries(Index ix, const uint32_t* __restrict__ slots, uint32_t n, uint32_t lab, int propagate,
                                unsigned long long* changed) {
  uint32_t ch = 0;
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t s = slots[i];
    const uint32_t m = ix.e[s].rec.meta;
    if (meta_label(m) != lab) {
      ix.e[s].rec.meta = (m & ~3u) | lab;
      ++ch;
    }
    if (propagate && i + 1 == n) ch += label_subtree(ix, s, lab);
  }
  *changed = ch;
}

// AccessStats::record of (entry, user) pairs in order, against the entries' window sets
__global__ void k_record_list(Index ix, MonCtx M, const uint32_t* __restrict__ slots,
                              const uint64_t* __restrict__ users, uint32_t n) {
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t s = slots[i];
    Entry& e = ix.e[s];
    const uint32_t si = acquire_set(e, s, M);
    if (si == kNone) return;
    SetHdr& hd = M.hdr[si];
    ulonglong2* tab = M.tab + static_cast<uint64_t>(si) * kSetSlots;
    const uint64_t u = users[i];
    e.stats.hit_cur += 1;
    uint32_t pos = mix32(u) & (kSetSlots - 1), free_pos = kNone;
    bool member = false;
    for (uint32_t t = 0; t < kSetSlots; ++t, pos = (pos + 1) & (kSetSlots - 1)) {
      const ulonglong2 x = tab[pos];
      if (x.y < M.wstart) {
        free_pos = pos;
        break;
      }
      if (x.x == u) {
        member = true;
        break;
      }
    }
    if (member) continue;
    if (hd.size < kMaxSetUsers && free_pos != kNone) {
      tab[free_pos] = make_ulonglong2(u, M.batch);
      hd.size += 1;
    }
    e.stats.u_cnt += 1;  // a new member, or saturated: counted as new (access_stats.hpp:30-36)
  }
}

// AccessStats::roll (access_stats.hpp:39-45) of given entries outside the epoch pass: the entry
// keeps (or gets) its place in the current window list, with a fresh empty set
__global__ void k_roll_list(Index ix, MonCtx M, const uint32_t* __restrict__ slots, uint32_t n) {
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t s = slots[i];
    Entry& e = ix.e[s];
    if (acquire_set(e, s, M) == kNone) return;  // listed in the current window from now on
    const uint32_t si = atomicAdd(M.pool_count, 1u);
    if (si >= M.pool_cap) {
      atomicOr(M.err, 1u);
      return;
    }
    M.hdr[si] = SetHdr{0u, 0u, 0u, 0u, 0ull};
    e.aux.set_idx = si;
    const Stats st = e.stats;
    e.stats = Stats{0u, 0u, st.hit_cur, st.u_cnt};
  }
}

// EntropyMonitor::check_anomaly (monitor.hpp:56-81) on one entry: the event's values always, the
// downgrade / restrict with subtree propagation when the predicate holds on a Public entry
__global__ void k_check_one(Index ix, uint32_t s, double jump, uint64_t u_pre_max, uint64_t epoch, DevEvent* ev,
                            int* fired) {
  const Rec& r = ix.e[s].rec;
  const Stats st = ix.e[s].stats;
  DevEvent o;
  o.h = r.h;
  o.d = r.d;
  o.owner = static_cast<uint8_t>(meta_owner(r.meta));
  for (int k = 0; k < 6; ++k) o.pad[k] = 0;
  o.now = st.hit_cur ? static_cast<double>(st.u_cnt) / static_cast<double>(st.hit_cur) : 0.0;
  o.prev = st.hit_pre ? static_cast<double>(st.u_pre) / static_cast<double>(st.hit_pre) : 0.0;
  o.u_pre = st.u_pre;
  o.epoch = epoch;
  o.action = SKV_ACTION_NONE;
  *fired = 0;
  if (meta_label(r.meta) == SKV_LABEL_PUBLIC && st.hit_pre > 0 && (o.now - o.prev) >= jump &&
      static_cast<uint64_t>(st.u_pre) <= u_pre_max) {
    const uint32_t lab = o.owner == 0 ? SKV_LABEL_PRIVATE : SKV_LABEL_RESTRICTED;
    o.action = o.owner == 0 ? SKV_ACTION_DOWNGRADE : SKV_ACTION_RESTRICT;
    ix.e[s].rec.meta = (r.meta & ~3u) | lab;
    label_subtree(ix, s, lab);
    *fired = 1;
  }
  *ev = o;
}
}  // namespace

void launch_find_entries(const Index& ix, const uint64_t* h, const uint64_t* d, uint32_t n, uint32_t* slots,
                         cudaStream_t s) {
  if (n) k_find_entries<<<cdiv(n, 256), 256, 0, s>>>(ix, h, d, n, slots);
}
void launch_label_entries(const Index& ix, const uint32_t* slots, uint32_t n, uint32_t label, int propagate,
                          unsigned long long* changed, cudaStream_t s) {
  k_label_entries<<<1, 1, 0, s>>>(ix, slots, n, label, propagate, changed);
}
void launch_record_list(const Index& ix, const MonCtx& M, const uint32_t* slots, const uint64_t* users, uint32_t n,
                        cudaStream_t s) {
  if (n) k_record_list<<<1, 1, 0, s>>>(ix, M, slots, users, n);
}
void launch_roll_list(const Index& ix, const MonCtx& M, const uint32_t* slots, uint32_t n, cudaStream_t s) {
  if (n) k_roll_list<<<1, 1, 0, s>>>(ix, M, slots, n);
}
void launch_check_one(const Index& ix, uint32_t slot, double jump, uint64_t u_pre_max, uint64_t epoch, void* ev,
                      int* fired, cudaStream_t s) {
  k_check_one<<<1, 1, 0, s>>>(ix, slot, jump, u_pre_max, epoch, static_cast<DevEvent*>(ev), fired);
}

// ---------------------------------------------------------------------------------
// A.8 evaluation leak flag (serving_sim.hpp:379-392 with block_truth, workload.hpp:137-147): a
// block of the last admitted batch is a leak iff it is labeled Public and overlaps a planted span
// that is sensitive on its own (SpanSensitivity::Always).  One thread per block.
// ---------------------------------------------------------------------------------
namespace {
__global__ void k_leak_flags(const uint32_t* __restrict__ blk_off, const uint8_t* __restrict__ label,
                             const uint32_t* __restrict__ span_off, const uint64_t* __restrict__ sb,
                             const uint64_t* __restrict__ se, uint32_t n_prompts, uint32_t B, uint8_t* flags,
                             unsigned long long* n_leaks) {
  const uint32_t p = blockIdx.x;
  if (p >= n_prompts) return;
  const uint32_t b0 = blk_off[p], nb = blk_off[p + 1] - b0, s0 = span_off[p], s1 = span_off[p + 1];
  uint32_t leaks = 0;
  for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) {
    const uint64_t lo = static_cast<uint64_t>(b) * B, hi = lo + B;
    bool hit = false;
    for (uint32_t k = s0; k < s1 && !hit; ++k) hit = !(se[k] <= lo || sb[k] >= hi);
    const bool leak = hit && label[b0 + b] == SKV_LABEL_PUBLIC;
    if (flags) flags[b0 + b] = leak ? 1 : 0;
    leaks += leak;
  }
  if (leaks) atomicAdd(n_leaks, static_cast<unsigned long long>(leaks));
}
}  // namespace

void launch_leak_flags(const uint32_t* blk_off, const uint8_t* label, const uint32_t* span_off, const uint64_t* sb,
                       const uint64_t* se, uint32_t n_prompts, uint32_t B, uint8_t* flags,
                       unsigned long long* n_leaks, cudaStream_t s) {
  if (n_prompts) k_leak_flags<<<n_prompts, 128, 0, s>>>(blk_off, label, span_off, sb, se, n_prompts, B, flags, n_leaks);
}

// byte tokens (ByteVocabulary) -> TokenIds: 16 bytes per thread in, 4 x 16 B out
namespace {
__global__ void k_widen(const uint8_t* __restrict__ in, uint32_t* __restrict__ out, uint64_t n) {
  const uint64_t i = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 16ull;
  if (i >= n) return;
  if (i + 16 <= n && (reinterpret_cast<uintptr_t>(in) & 15) == 0) {
    const uint4 v = *reinterpret_cast<const uint4*>(in + i);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint4* o = reinterpret_cast<uint4*>(out + i);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      o[q] = make_uint4(w[q] & 0xffu, (w[q] >> 8) & 0xffu, (w[q] >> 16) & 0xffu, w[q] >> 24);
  } else {
    for (uint64_t k = i; k < n && k < i + 16; ++k) out[k] = in[k];
  }
}
}  // namespace

void launch_widen(const uint8_t* in, uint32_t* out, uint64_t n, cudaStream_t s) {
  if (n) k_widen<<<static_cast<uint32_t>((n + 16 * 256 - 1) / (16 * 256)), 256, 0, s>>>(in, out, n);
}
}  // namespace skv

// =================================================================================
// A.9: insert-time make_room under a bounded HBM budget (cache_index.hpp:183-190,
// 801-806; serving pins, serving_sim.hpp:195-215).  The batch commits in rounds over
// prompt ranges [lo, next): per round a dry claim pass gives every prompt the blocks it
// would create (lowest prompt wins a key), the victim order V is the untiered eviction
// order of the entries no prompt of the batch has matched (pinned), and one thread walks
// the prompts in order, taking victims from V for each prompt's make_room.  A round ends
// early where V stops being the reference's order: an eviction cutting a later prompt's
// insert walk (it re-walks next round), or a victim of the current epoch (this batch's own
// nodes compete with it) after the round's first prompt.  Every round commits >= 1 prompt.
// =================================================================================
namespace skv {
namespace {
constexpr uint32_t kStampNone = 0xffffffffu;

__global__ void k_new_bound(const uint32_t* __restrict__ blk_off, const uint32_t* __restrict__ exist, uint32_t lo,
                            uint32_t hi, unsigned long long* out) {
  const uint32_t p = lo + blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t v = 0;
  if (p < hi) {
    const uint32_t n = blk_off[p + 1] - blk_off[p];
    v = n - min(exist[p], n);
  }
  v = __reduce_add_sync(kFull, v);
  if (lane_id() == 0 && v) atomicAdd(out, static_cast<unsigned long long>(v));
}

// pinned (matched by any prompt of the batch) = 0; walked by prompt p in [lo, hi) = p + 1 (the
// first such p); every newly marked slot is listed for clearing
__device__ __forceinline__ void mark_slot(uint32_t* vstamp, uint32_t s, uint32_t v, uint32_t* list, uint32_t* n_list,
                                          uint32_t cap) {
  const uint32_t old = atomicMin(&vstamp[s], v);
  if (old == kStampNone) {
    const uint32_t i = atomicAdd(n_list, 1u);
    if (i < cap) list[i] = s;
  }
}

__global__ void k_mark_paths(const uint32_t* __restrict__ slot, const uint32_t* __restrict__ blk_off,
                             const uint32_t* __restrict__ exist, const uint32_t* __restrict__ matched, uint32_t lo,
                             uint32_t hi, uint32_t* vstamp, uint32_t* list, uint32_t* n_list, uint32_t cap) {
  const uint32_t p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (p >= hi) return;
  const uint32_t bo = blk_off[p], m = matched[p], k = p >= lo ? exist[p] : m;
  for (uint32_t b = lane_id(); b < k; b += 32) mark_slot(vstamp, slot[bo + b], b < m ? 0u : p + 1, list, n_list, cap);
}

__global__ void k_clear_marks(uint32_t* vstamp, const uint32_t* __restrict__ list, const uint32_t* __restrict__ n_list,
                              uint32_t cap) {
  const uint32_t n = min(*n_list, cap);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    vstamp[list[i]] = kStampNone;
}

// the structural walk of prompts [lo, hi) after the previous rounds (their inserts and victims)
__global__ void k_reprobe(Index ix, const uint64_t* __restrict__ hk, const uint64_t* __restrict__ dk,
                          const uint32_t* __restrict__ blk_off, uint32_t lo, uint32_t hi, uint32_t* exist,
                          uint32_t* slot_out) {
  const uint32_t p = lo + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (p >= hi) return;
  const uint32_t lane = lane_id(), bo = blk_off[p], n = blk_off[p + 1] - bo;
  uint32_t k = n;
  for (uint32_t base = 0; base < n && base < k; base += 32) {
    const uint32_t b = base + lane;
    uint64_t h = 0, d = 0;
    if (b < n) h = hk[bo + b], d = dk[bo + b];
    const uint64_t hL = __shfl_sync(kFull, h, lane & ~(kGroup - 1)), dL = __shfl_sync(kFull, d, lane & ~(kGroup - 1));
    uint32_t s = kNone;
    if (b < n) {
      Rec r;
      s = find_slot(ix, h, d, hL, dL, b, &r);
      if (s != kNone) slot_out[bo + b] = s;
    }
    const uint32_t miss = __ballot_sync(kFull, b < n && s == kNone);
    if (miss) k = min(k, base + __ffs(miss) - 1);
  }
  if (lane == 0) exist[p] = k;
}

// dry claims: the blocks every prompt of [lo, hi) would create, duplicates won by the lowest prompt
__global__ void k_dry_claims(const uint64_t* __restrict__ hk, const uint64_t* __restrict__ dk,
                             const uint32_t* __restrict__ blk_off, const uint32_t* __restrict__ exist, uint32_t lo,
                             uint32_t hi, ulonglong2* tab, uint32_t* minp, uint64_t tmask, uint32_t* dslot) {
  const uint32_t p = lo + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (p >= hi) return;
  const uint32_t bo = blk_off[p], n = blk_off[p + 1] - bo;
  for (uint32_t b = exist[p] + lane_id(); b < n; b += 32) {
    const uint64_t h = hk[bo + b], d = dk[bo + b];
    uint64_t s = slot_hash(h, d) & tmask;
    for (uint64_t i = 0; i <= tmask; ++i, s = (s + 1) & tmask) {
      unsigned long long ol, oh;
      const bool won = cas128(reinterpret_cast<unsigned long long*>(&tab[s]), 0ull, 0ull, h, d, &ol, &oh);
      if (won || (ol == h && oh == d)) {
        atomicMin(&minp[s], p);
        dslot[bo + b] = static_cast<uint32_t>(s);
        break;
      }
    }
  }
}

__global__ void k_dry_count(const uint32_t* __restrict__ blk_off, const uint32_t* __restrict__ exist, uint32_t lo,
                            uint32_t hi, const uint32_t* __restrict__ minp, const uint32_t* __restrict__ dslot,
                            uint32_t* needed) {
  const uint32_t p = lo + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (p >= hi) return;
  const uint32_t bo = blk_off[p], n = blk_off[p + 1] - bo;
  uint32_t f = 0;
  for (uint32_t b = exist[p] + lane_id(); b < n; b += 32) f += minp[dslot[bo + b]] == p ? 1u : 0u;
  f = __reduce_add_sync(kFull, f);
  if (lane_id() == 0) needed[p - lo] = f;
}

// the order key of an entry, with the batch's pinned entries blocking (k_evict_init)
__global__ void k_evict_init_pinned(Index ix, const uint32_t* __restrict__ vstamp, unsigned long long* eff) {
  const uint64_t s = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s > ix.mask) return;
  const Rec& r = ix.e[s].rec;
  if ((r.h == 0 && r.d == 0) || !meta_live(r.meta))
    eff[s] = 0ull;
  else
    eff[s] = vstamp[s] == 0u ? ~0ull : evict_key(ix, s);
}

// one thread: the prompts of the round in order, each insert's make_room taking victims from V
__global__ void k_budget_sim(const uint32_t* __restrict__ needed, uint32_t lo, uint32_t hi, unsigned long long used,
                             unsigned long long cap, const uint32_t* __restrict__ vals, uint32_t nv,
                             const unsigned long long* __restrict__ eff, const uint32_t* __restrict__ vstamp,
                             uint32_t epoch, uint32_t* victims, BudgetSim* out) {
  if (threadIdx.x || blockIdx.x) return;
  uint32_t i = 0, nvict = 0, cut = kNone, p = lo, dropped = kNone;
  for (; p < hi; ++p) {
    if (p == cut) break;  // an eviction cut this prompt's insert walk: it walks again next round
    const uint32_t need = needed[p - lo];
    const uint32_t nvict0 = nvict, i0 = i;
    const unsigned long long used0 = used;
    bool stop = false, fail = false;
    while (used + need > cap) {
      // stamped by an insert walk of this round at or before p: the walk refreshed its epoch
      // (young now, and no longer a leaf unless it ends the walk)
      while (i < nv) {
        const uint32_t st = vstamp[vals[i]];
        if (st != kStampNone && st - 1 >= lo && st - 1 <= p)
          ++i;
        else
          break;
      }
      if (i == nv) {
        fail = true;
        break;
      }
      if (p > lo && (eff[vals[i]] >> 32) == epoch) {
        stop = true;
        break;
      }
      const uint32_t st = vstamp[vals[i]];
      if (st != kStampNone && st - 1 > p) cut = min(cut, st - 1);
      victims[nvict++] = vals[i++];
      --used;
    }
    if (fail && p > lo) stop = true;  // the round's own new nodes may still be candidates
    if (stop) {                       // p's make_room is redone next round
      nvict = nvict0;
      i = i0;
      used = used0;
      break;
    }
    if (fail) {  // CapacityExhausted: its victims stay evicted, the prompt is dropped
      dropped = p;
      ++p;
      break;
    }
    used += need;
  }
  out->used = used;
  out->n_victims = nvict;
  out->next_lo = p;
  out->dropped = dropped;
  out->pad = 0;
}

__global__ void k_evict_mark_list(Index ix, const uint32_t* __restrict__ vals, uint32_t v) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= v) return;
  const uint32_t s = vals[i];
  Rec& r = ix.e[s].rec;
  r.meta = (r.meta & 0x1fu) | 0xffffff00u;
  ix.em[s].dead = 1;
}
}  // namespace

void launch_new_bound(const uint32_t* blk_off, const uint32_t* exist, uint32_t lo, uint32_t hi,
                      unsigned long long* out, cudaStream_t s) {
  cudaMemsetAsync(out, 0, 8, s);
  if (hi > lo) k_new_bound<<<cdiv(hi - lo, 256), 256, 0, s>>>(blk_off, exist, lo, hi, out);
}

void launch_mark_paths(const uint32_t* slot, const uint32_t* blk_off, const uint32_t* exist, const uint32_t* matched,
                       uint32_t lo, uint32_t hi, uint32_t* vstamp, uint32_t* list, uint32_t* n_list, uint32_t cap,
                       cudaStream_t s) {
  if (hi) k_mark_paths<<<cdiv(static_cast<uint64_t>(hi) * 32, 256), 256, 0, s>>>(slot, blk_off, exist, matched, lo, hi,
                                                                                 vstamp, list, n_list, cap);
}

void launch_clear_marks(uint32_t* vstamp, const uint32_t* list, const uint32_t* n_list, uint32_t cap, cudaStream_t s) {
  k_clear_marks<<<256, 256, 0, s>>>(vstamp, list, n_list, cap);
}

void launch_reprobe(const Index& ix, const uint64_t* h, const uint64_t* d, const uint32_t* blk_off, uint32_t lo,
                    uint32_t hi, uint32_t* exist, uint32_t* slot_out, cudaStream_t s) {
  if (hi > lo)
    k_reprobe<<<cdiv(static_cast<uint64_t>(hi - lo) * 32, 256), 256, 0, s>>>(ix, h, d, blk_off, lo, hi, exist, slot_out);
}

void launch_dry_needed(const uint64_t* h, const uint64_t* d, const uint32_t* blk_off, const uint32_t* exist,
                       uint32_t lo, uint32_t hi, ulonglong2* tab, uint32_t* minp, uint64_t tcap, uint32_t* dslot,
                       uint32_t* needed, cudaStream_t s) {
  if (hi <= lo) return;
  cudaMemsetAsync(tab, 0, tcap * sizeof(ulonglong2), s);
  cudaMemsetAsync(minp, 0xff, tcap * sizeof(uint32_t), s);
  const unsigned g = static_cast<unsigned>(cdiv(static_cast<uint64_t>(hi - lo) * 32, 256));
  k_dry_claims<<<g, 256, 0, s>>>(h, d, blk_off, exist, lo, hi, tab, minp, tcap - 1, dslot);
  k_dry_count<<<g, 256, 0, s>>>(blk_off, exist, lo, hi, minp, dslot, needed);
}

uint32_t launch_evict_order(const Index& ix, const uint32_t* vstamp, unsigned long long* eff,
                            unsigned long long* keys_a, unsigned long long* keys_b, uint32_t* vals_a, uint32_t* vals_b,
                            uint32_t* n_live, void* temp, size_t temp_bytes, uint32_t* host_n, cudaStream_t s) {
  const unsigned g = static_cast<unsigned>(cdiv(ix.cap, 256));
  cudaMemsetAsync(n_live, 0, 4, s);
  k_evict_init_pinned<<<g, 256, 0, s>>>(ix, vstamp, eff);
  k_evict_propagate<<<g, 256, 0, s>>>(ix, eff);
  k_evict_compact<<<g, 256, 0, s>>>(ix, eff, keys_a, vals_a, n_live);
  cudaMemcpyAsync(host_n, n_live, 4, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  const uint32_t n = *host_n;
  if (n) {  // deeper first, then by effective key (stable): V in vals_a
    cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_a, keys_b, vals_a, vals_b, static_cast<int>(n), 0, 32, s);
    k_evict_gather<<<cdiv(n, 256), 256, 0, s>>>(eff, vals_b, keys_a, n_live);
    cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_a, keys_b, vals_b, vals_a, static_cast<int>(n), 0, 64, s);
  }
  return n;
}

void launch_budget_sim(const uint32_t* needed, uint32_t lo, uint32_t hi, uint64_t used, uint64_t cap,
                       const uint32_t* vals, uint32_t nv, const unsigned long long* eff, const uint32_t* vstamp,
                       uint32_t epoch, uint32_t* victims, BudgetSim* out, cudaStream_t s) {
  k_budget_sim<<<1, 32, 0, s>>>(needed, lo, hi, used, cap, vals, nv, eff, vstamp, epoch, victims, out);
}

// ---- A.9 with tiered demotion (evict_or_demote, cache_index.hpp:732-766): bounded DRAM / SSD.
// A victim moves one tier down and stays a leaf; a full lower tier first demotes (or, from SSD,
// frees) its own smallest-key leaf; with no such leaf the victim is freed outright.  Frees
// expose parents, so the per-tier candidate pools are the round's sorted leaves plus a heap of
// nodes that became candidates during the round (demoted victims, exposed parents).
namespace {
__device__ __forceinline__ unsigned long long tier_key(const Index& ix, uint32_t s) {
  const EvictMeta em = ix.em[s];
  return (static_cast<unsigned long long>(em.access_epoch) << 32) |
         (static_cast<unsigned long long>(meta_label(ix.e[s].rec.meta) != SKV_LABEL_PUBLIC) << 31) |
         (em.node_id & 0x7fffffffu);
}

__global__ void k_child_counts(Index ix, uint32_t* cc) {
  const uint64_t s = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s > ix.mask) return;
  const Rec& r = ix.e[s].rec;
  if ((r.h == 0 && r.d == 0) || !meta_live(r.meta) || r.parent == kNone) return;
  atomicAdd(&cc[r.parent], 1u);
}

__global__ void k_tier_leaves(Index ix, const uint32_t* __restrict__ cc, const uint32_t* __restrict__ vstamp,
                              unsigned long long* keys, uint32_t* vals, uint32_t* n3, uint64_t cap_each) {
  const uint64_t s = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s > ix.mask) return;
  const Rec& r = ix.e[s].rec;
  if ((r.h == 0 && r.d == 0) || !meta_live(r.meta) || cc[s] || (vstamp && vstamp[s] == 0u)) return;
  const uint32_t t = meta_tier(r.meta);
  const uint32_t i = atomicAdd(&n3[t], 1u);
  keys[t * cap_each + i] = tier_key(ix, static_cast<uint32_t>(s));
  vals[t * cap_each + i] = static_cast<uint32_t>(s);
}

struct TPool {  // one tier's candidates: the round's sorted leaves, then a min-heap of arrivals
  const unsigned long long* lk;
  const uint32_t* lv;
  uint32_t ln, li;
  unsigned long long* hk;
  uint32_t* hv;
  uint32_t hn;
};

__device__ void heap_push(TPool& P, unsigned long long k, uint32_t v) {
  uint32_t i = P.hn++;
  while (i) {
    const uint32_t par = (i - 1) >> 1;
    if (P.hk[par] <= k) break;
    P.hk[i] = P.hk[par];
    P.hv[i] = P.hv[par];
    i = par;
  }
  P.hk[i] = k;
  P.hv[i] = v;
}

__device__ void heap_pop(TPool& P) {
  const unsigned long long k = P.hk[--P.hn];
  const uint32_t v = P.hv[P.hn];
  uint32_t i = 0;
  for (;;) {
    uint32_t c = 2 * i + 1;
    if (c >= P.hn) break;
    if (c + 1 < P.hn && P.hk[c + 1] < P.hk[c]) ++c;
    if (P.hk[c] >= k) break;
    P.hk[i] = P.hk[c];
    P.hv[i] = P.hv[c];
    i = c;
  }
  if (P.hn) {
    P.hk[i] = k;
    P.hv[i] = v;
  }
}

struct TSim {
  Index ix;
  TPool pool[3];
  uint32_t* cc;
  const uint32_t* vstamp;
  uint8_t* tier;  // current tier of every slot this round touched (255 = freed); init = table tier
  uint32_t* act;  // actions in order: slot | kind << 30 (0 free, 1 -> DRAM, 2 -> SSD)
  uint32_t n_act, act_cap;
  unsigned long long used[3], cap[3];
  uint32_t lo, p, cut, epoch;
  unsigned long long hbm_out;  // blocks that left HBM (freed or demoted)
  bool stop;
};

// the smallest-key current candidate of tier t (kNone: none).  Skipped for good: entries that
// left the tier, and entries an insert walk of this round at or before prompt p refreshed (young,
// and attach points: the current-epoch region ends the round, below)
__device__ uint32_t pool_pop(TSim& S, uint32_t t) {
  TPool& P = S.pool[t];
  for (;;) {
    uint32_t v = kNone;
    unsigned long long k = 0;
    const bool from_heap = P.hn && (P.li >= P.ln || P.hk[0] < P.lk[P.li]);
    if (from_heap) {
      v = P.hv[0], k = P.hk[0];
      heap_pop(P);
    } else if (P.li < P.ln) {
      v = P.lv[P.li], k = P.lk[P.li];
      ++P.li;
    } else {
      return kNone;
    }
    if (S.tier[v] != t) continue;
    const uint32_t st = S.vstamp ? S.vstamp[v] : kStampNone;
    if (st != kStampNone && st - 1 >= S.lo && st - 1 <= S.p) continue;
    if (S.p > S.lo && (k >> 32) == S.epoch) {  // the batch's own nodes may precede it: end the round
      S.stop = true;
      return kNone;
    }
    return v;
  }
}

__device__ bool sim_free(TSim& S, uint32_t v) {
  const uint32_t t = S.tier[v];
  S.used[t]--;
  if (t == 0) ++S.hbm_out;
  S.tier[v] = 255;
  if (S.n_act < S.act_cap) S.act[S.n_act++] = v;
  const uint32_t st = S.vstamp ? S.vstamp[v] : kStampNone;
  if (st != kStampNone && st - 1 > S.p) S.cut = min(S.cut, st - 1);  // a later insert walks it
  const uint32_t par = S.ix.e[v].rec.parent;
  if (par != kNone && --S.cc[par] == 0 && S.tier[par] < 3 && !(S.vstamp && S.vstamp[par] == 0u))
    heap_push(S.pool[S.tier[par]], tier_key(S.ix, par), par);  // the parent became a leaf
  return true;
}

// evict_or_demote(v, t): false when a pool query ended the round
__device__ bool sim_evict_or_demote(TSim& S, uint32_t v, uint32_t t) {
  if (t == 2) return sim_free(S, v);
  const uint32_t target = t + 1;
  while (S.used[target] + 1 > S.cap[target]) {
    const uint32_t lv = pool_pop(S, target);
    if (S.stop) return false;
    if (lv == kNone) return sim_free(S, v);  // lower tiers full and unfreeable: drop outright
    if (!sim_evict_or_demote(S, lv, target)) return false;
  }
  S.used[t]--;
  if (t == 0) ++S.hbm_out;
  S.used[target]++;
  S.tier[v] = static_cast<uint8_t>(target);
  if (S.n_act < S.act_cap) S.act[S.n_act++] = v | (target << 30);
  heap_push(S.pool[target], tier_key(S.ix, v), v);  // still a leaf, now in the lower tier
  return true;
}

// needed == nullptr: RadixCacheIndex::evict(need_evict) instead of a commit round
__global__ void k_budget_sim_tiered(TSim S, const uint32_t* __restrict__ needed, uint32_t hi, uint64_t need_evict,
                                    BudgetSim* out, unsigned long long* used_out, uint32_t* n_act_out) {
  if (threadIdx.x || blockIdx.x) return;
  S.cut = kNone;
  S.stop = false;
  S.hbm_out = 0;
  uint32_t p = S.lo, dropped = kNone;
  if (!needed) {
    S.p = S.lo;
    uint64_t freed = 0;
    while (freed < need_evict) {
      const uint32_t v = pool_pop(S, 0);
      if (v == kNone) {
        dropped = 0;  // CapacityExhausted after freeing what it could
        break;
      }
      sim_evict_or_demote(S, v, 0);
      ++freed;
    }
    p = hi;
  } else {
    for (; p < hi; ++p) {
      if (p == S.cut) break;
      S.p = p;
      const uint32_t need = needed[p - S.lo];
      bool fail = false;
      while (S.used[0] + need > S.cap[0]) {
        const uint32_t v = pool_pop(S, 0);
        if (S.stop) break;
        if (v == kNone) {
          fail = true;
          break;
        }
        if (!sim_evict_or_demote(S, v, 0)) break;
      }
      if (fail && p > S.lo) S.stop = true;
      if (S.stop) break;  // the caller re-runs the round up to p (its make_room is redone next round)
      if (fail) {
        dropped = p;
        ++p;
        break;
      }
      S.used[0] += need;
    }
  }
  out->used = S.used[0];
  out->n_victims = S.n_act;
  out->next_lo = p;
  out->dropped = S.stop ? kNone - 1 : dropped;
  out->pad = S.n_act >= S.act_cap ? 1u : 0u;
  for (int t = 0; t < 3; ++t) used_out[t] = S.used[t];
  used_out[3] = S.hbm_out;
  *n_act_out = S.n_act;
}

// apply the actions in order (a slot can move down twice, then be freed)
__global__ void k_apply_actions(Index ix, const uint32_t* __restrict__ act, uint32_t n) {
  if (threadIdx.x || blockIdx.x) return;
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t s = act[i] & 0x3fffffffu, kind = act[i] >> 30;
    Rec& r = ix.e[s].rec;
    if (kind == 0) {
      r.meta = (r.meta & 0x1fu) | 0xffffff00u;
      ix.em[s].dead = 1;
    } else {
      r.meta = (r.meta & ~(3u << 3)) | (kind << 3);
    }
  }
}

__global__ void k_tier_init(Index ix, uint8_t* tier) {
  const uint64_t s = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s > ix.mask) return;
  const Rec& r = ix.e[s].rec;
  tier[s] = ((r.h == 0 && r.d == 0) || !meta_live(r.meta)) ? 255 : static_cast<uint8_t>(meta_tier(r.meta));
}

__global__ void k_count_tiers(Index ix, unsigned long long* out3) {
  const uint64_t s = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  uint32_t t = 3;
  if (s <= ix.mask) {
    const Rec& r = ix.e[s].rec;
    if (!(r.h == 0 && r.d == 0) && meta_live(r.meta)) t = meta_tier(r.meta);
  }
#pragma unroll
  for (uint32_t k = 0; k < 3; ++k) {
    const uint32_t c = __popc(__ballot_sync(kFull, t == k));
    if (lane_id() == 0 && c) atomicAdd(&out3[k], static_cast<unsigned long long>(c));
  }
}
}  // namespace

// One tiered round (or one tiered evict call): candidate pools, then the sequential simulation.
// Work buffers (TieredWork) hold cap-sized arrays; returns the round's BudgetSim in host memory.
BudgetSim launch_budget_tiered(const Index& ix, const TieredWork& w, const uint32_t* vstamp, const uint32_t* needed,
                               uint32_t lo, uint32_t hi, uint64_t need_evict, const uint64_t* used3,
                               const uint64_t* cap3, uint32_t epoch, uint32_t* host, cudaStream_t s) {
  const unsigned g = static_cast<unsigned>(cdiv(ix.cap, 256));
  cudaMemsetAsync(w.cc, 0, ix.cap * 4, s);
  k_child_counts<<<g, 256, 0, s>>>(ix, w.cc);
  cudaMemsetAsync(w.n3, 0, 12, s);
  k_tier_leaves<<<g, 256, 0, s>>>(ix, w.cc, vstamp, w.keys_a, w.vals_a, w.n3, w.cap_each);
  cudaMemcpyAsync(host, w.n3, 12, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  uint32_t n3[3] = {host[0], host[1], host[2]};
  size_t tb = w.temp_bytes;
  for (int t = 0; t < 3; ++t)
    if (n3[t])
      cub::DeviceRadixSort::SortPairs(w.temp, tb, w.keys_a + t * w.cap_each, w.keys_b + t * w.cap_each,
                                      w.vals_a + t * w.cap_each, w.vals_b + t * w.cap_each, static_cast<int>(n3[t]),
                                      0, 64, s);
  // a stopped round is re-run up to its stop prompt from the same start state
  uint32_t hi_run = hi;
  BudgetSim r{};
  for (int attempt = 0; attempt < 2; ++attempt) {
    cudaMemcpyAsync(w.cc_work, w.cc, ix.cap * 4, cudaMemcpyDeviceToDevice, s);
    k_tier_init<<<g, 256, 0, s>>>(ix, w.tier);
    TSim S{};
    S.ix = ix;
    for (int t = 0; t < 3; ++t) {
      S.pool[t] = TPool{w.keys_b + t * w.cap_each, w.vals_b + t * w.cap_each, n3[t], 0u,
                        w.hk + t * w.cap_each, w.hv + t * w.cap_each, 0u};
      S.used[t] = used3[t];
      S.cap[t] = cap3[t];
    }
    S.cc = w.cc_work;
    S.vstamp = vstamp;
    S.tier = w.tier;
    S.act = w.act;
    S.act_cap = static_cast<uint32_t>(std::min<uint64_t>(w.act_cap, 0x3fffffffull));
    S.n_act = 0;
    S.lo = lo;
    S.epoch = epoch;
    k_budget_sim_tiered<<<1, 32, 0, s>>>(S, needed, hi_run, need_evict, w.res, w.used3, w.n_act);
    cudaMemcpyAsync(host, w.res, sizeof(BudgetSim), cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(host + 8, w.used3, 32, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    std::memcpy(&r, host, sizeof(r));
    if (r.dropped != kNone - 1) break;  // not stopped
    hi_run = r.next_lo;                 // stopped at prompt next_lo > lo: redo the round up to it
  }
  if (r.n_victims) k_apply_actions<<<1, 32, 0, s>>>(ix, w.act, r.n_victims);
  return r;
}

void launch_count_tiers(const Index& ix, unsigned long long* out3, cudaStream_t s) {
  cudaMemsetAsync(out3, 0, 24, s);
  k_count_tiers<<<cdiv(ix.cap, 256), 256, 0, s>>>(ix, out3);
}

void launch_evict_mark_list(const Index& ix, const uint32_t* vals, uint32_t v, cudaStream_t s) {
  if (v) k_evict_mark_list<<<cdiv(v, 256), 256, 0, s>>>(ix, vals, v);
}
}  // namespace skv
