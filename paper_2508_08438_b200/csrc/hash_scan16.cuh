// hash_scan16.cuh -- K12 for the configs' block shape (B = 16 tokens, W = 32 right-context
// tokens): block digest (token_seq_digest, core.hpp:68-73) + rule-tier window scan
// (CompiledRuleSet::scan on the window string, detection.hpp:148-170).
// Included by kernels.cu inside namespace skv::{anon}; the general kernel (k_hash_scan)
// serves every other shape.
//
// What differs from k_hash_scan:
//  * Byte-indexed automaton.  The SMEM image is column-major over BYTES (128 columns for
//    bytes 0..127 plus an end-of-text column): entry (byte t, state s) sits at byte offset
//    t * colbytes + v(s), v(s) = 2 * index(s), so one DFA step is IMAD + LDS (no byte-class
//    lookup).  Bytes >= 128 (rare) take a global twin table.
//  * Sticky acceptance.  Every state has a shadow copy (index + S); a transition that
//    accepts some rule lands in the shadow copy and shadow states stay shadow, so "this
//    segment accepted" is one compare of its final state (v >= 2S) instead of an OR per
//    step.  Runs restart from the base copy at segment boundaries (block edges and after the
//    first kConv16 bytes), so per-segment flags are exact.  The EOS column holds the exact
//    end-of-text rule mask.
//  * No helper lanes.  Warps walk their block range in chunks of 32 (stride 32); lane l
//    runs phase A of block g+l, phase B of window g+l-1 over its own block and phase C of
//    window g+l-2 over its own block, and finalises window g+l-2.  The two windows that
//    reach past a chunk are finished by the next chunk with a 2-block lag: their inputs
//    come from the previous chunk's lanes 30/31 through the same shuffle (the sending lane
//    offers its previous-chunk value).
//  * Prompt geometry from three warp-uniform prompt slots (previous, current, next);
//    chunks whose span they do not cover (prompts shorter than ~34 blocks) look their
//    prompts up per lane.
// The exact enabled-rule masks of flagged segments are recomputed from the global
// transition table (queued per warp, as in k_hash_scan).

#ifndef SKV_H16_WARPS
#define SKV_H16_WARPS 32
#endif
constexpr uint32_t kH16Warps = SKV_H16_WARPS;
constexpr uint32_t kConv16 = 4;

struct Slot16 {
  unsigned long long base;  // token index of block 0 of the prompt's block numbering (tok_off - blk_start * 16)
  uint32_t tend;            // low 32 bits of the prompt's token end
  uint32_t start;           // first block of the prompt
};

#ifndef SKV_H16_PF
#define SKV_H16_PF 2  // prefetch of the next chunk's token lines: 0 none, 1 L1, 2 L2
#endif

__device__ __forceinline__ uint32_t h16_base(uint32_t v, uint32_t s2) { return v >= s2 ? v - s2 : v; }

// one DFA step on a byte < 128 (SMEM)
__device__ __forceinline__ uint32_t h16_step(const uint8_t* __restrict__ tab, uint32_t colbytes, uint32_t v,
                                             uint32_t t) {
  return *reinterpret_cast<const uint16_t*>(tab + t * colbytes + v);
}

// one DFA step on any byte (SMEM below 128, the global twin above)
__device__ __forceinline__ uint32_t h16_step_any(const uint8_t* __restrict__ tab, const uint16_t* __restrict__ hi,
                                                 uint32_t colbytes, uint32_t v, uint32_t b) {
  return b < 128 ? h16_step(tab, colbytes, v, b)
                 : __ldg(reinterpret_cast<const uint16_t*>(reinterpret_cast<const uint8_t*>(hi) +
                                                           (b - 128) * colbytes + v));
}

// exact run over tokens[tok, tok+len) from base state v: OR of the enabled-rule masks of
// every accepting transition.  The walk steps through the SMEM image (an accepting
// transition lands in a shadow state: the walk notes it and continues from the state's base
// copy) and reads the global [256][S] table only at accepting transitions, so its
// dependent chain is SMEM latency, not L2 latency (a small batch's flagged windows are its
// tail: config 1 spends most of the kernel here otherwise)
__device__ __forceinline__ uint32_t h16_exact(const uint8_t* __restrict__ tab, const uint16_t* __restrict__ hi,
                                              uint32_t colbytes, uint32_t s2, const uint32_t* __restrict__ full,
                                              const uint32_t* __restrict__ tokens, uint64_t tok, uint32_t len,
                                              uint32_t v) {
  const uint32_t S = s2 >> 1;
  uint32_t m = 0;
#pragma unroll 4
  for (uint32_t j = 0; j < len; ++j) {
    const uint32_t b = tokens[tok + j] & 0xffu;
    const uint32_t nv = h16_step_any(tab, hi, colbytes, v, b);
    if (nv >= s2) {  // accepting transition out of base state v
      m |= __ldg(full + b * S + (v >> 1)) >> 16;
      v = nv - s2;
    } else {
      v = nv;
    }
  }
  return m;
}

// run over tokens[tok, tok+len) (global loads) from base state v; returns the final state
// (shadow if anything accepted)
__device__ __forceinline__ uint32_t h16_run_global(const uint8_t* __restrict__ tab, const uint16_t* __restrict__ hi,
                                                   uint32_t colbytes, const uint32_t* __restrict__ tokens,
                                                   uint64_t tok, uint32_t len, uint32_t v) {
#pragma unroll 1
  for (uint32_t j = 0; j < len; ++j) v = h16_step_any(tab, hi, colbytes, v, tokens[tok + j] & 0xffu);
  return v;
}

// last prompt p with blk_off[p] <= k (non-empty: blk_off[p + 1] > k for k < nb)
__device__ __forceinline__ uint32_t h16_prompt_of(const uint32_t* __restrict__ blk_off, uint32_t N, uint32_t k) {
  uint32_t lo = 0, hi = N;
  while (hi - lo > 1) {
    const uint32_t m = (lo + hi) >> 1;
    if (__ldg(blk_off + m) <= k)
      lo = m;
    else
      hi = m;
  }
  return lo;
}

// first non-empty prompt >= q (N if none)
__device__ __forceinline__ uint32_t h16_nonempty(const uint32_t* __restrict__ blk_off, uint32_t N, uint32_t q) {
  while (q < N && __ldg(blk_off + q + 1) == __ldg(blk_off + q)) ++q;
  return q;
}

__device__ __forceinline__ Slot16 h16_slot(const HS16Args& a, uint32_t p) {
  Slot16 s;
  if (p >= a.n_prompts) {
    s.base = 0;
    s.tend = 0;
    s.start = 0;
    return s;
  }
  s.start = a.blk_off[p];
  s.base = a.tok_off[p] - 16ull * s.start;
  s.tend = static_cast<uint32_t>(a.tok_off[p + 1]);
  return s;
}

// a flagged segment whose exact rule mask is recomputed: first token (bits 0-39), length
// (40-45), start state v (46-61); the window's block and prompt.  16 B.
struct H16Task {
  unsigned long long tokv;
  uint32_t gb, p;
};

__device__ __forceinline__ void h16_flush(H16Task* q, uint32_t qn, uint32_t lane, const HS16Args& a,
                                          const uint8_t* __restrict__ tab) {
  __syncwarp();
  for (uint32_t k = lane; k < qn; k += 32) {
    const H16Task t = q[k];
    const uint32_t m = h16_exact(tab, a.hi, a.colbytes, a.s2, a.full, a.tokens, t.tokv & 0xffffffffffull,
                                 (t.tokv >> 40) & 63u, static_cast<uint32_t>(t.tokv >> 46));
    if (m) {
      atomicOr(&a.mask_out[t.gb], m << a.mask_shift);
      atomicMin(&a.first_sens[t.p], t.gb - a.blk_off[t.p]);
    }
  }
  __syncwarp();
}

// The automaton image -> SMEM by bulk (TMA) copies issued by one thread, completion counted on an
// mbarrier (transaction bytes): the image arrives at the copy engine's rate instead of one L2
// round trip per 16-B load and thread (which bounds a CTA of few warps -- a small batch's launch
// shape -- at ~70 dependent round trips)
__device__ __forceinline__ void h16_load_image(uint8_t* sm, const void* src, uint32_t bytes, uint64_t* mbar) {
  const uint32_t bar = static_cast<uint32_t>(__cvta_generic_to_shared(mbar));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
    for (uint32_t off = 0; off < bytes; off += 32768u) {
      const uint32_t n = min(32768u, bytes - off);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       dst + off),
                   "l"(static_cast<const uint8_t*>(src) + off), "r"(n), "r"(bar)
                   : "memory");
    }
  }
  __syncthreads();  // the barrier is initialised before anyone waits on it
  asm volatile(
      "{\n\t.reg .pred p;\n\tH16_WAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
      "@!p bra H16_WAIT_%=;\n\t}" ::"r"(bar)
      : "memory");
}

// blockDim.x = 32 x WPC warps (kH16Warps for large batches; a small batch spreads its chunks over
// more SMs with fewer warps each, capi.cpp stage12)
__global__ void __launch_bounds__(kH16Warps * 32, kH16Warps <= 16 ? 2 : 1) k_hash_scan16(HS16Args a) {
  extern __shared__ __align__(16) uint8_t sm[];
  const uint8_t* tab = sm;
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, WPC = blockDim.x >> 5;
  const uint32_t img_al = (a.img_bytes + 15) & ~15u;
  Slot16* slots = reinterpret_cast<Slot16*>(sm + img_al) + 4 * wid;  // prev, cur, next; [3].start..: prompt ids
  uint32_t* slot_p = reinterpret_cast<uint32_t*>(slots + 3);
  H16Task* q = reinterpret_cast<H16Task*>(sm + img_al + 4 * WPC * sizeof(Slot16)) + wid * a.q_cap;
  __shared__ uint64_t img_bar;
  h16_load_image(sm, a.img, img_al, &img_bar);
  const uint32_t N = a.n_prompts;
  const uint32_t nb = a.blk_off[N];
  const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * WPC + wid, TW = static_cast<uint64_t>(gridDim.x) * WPC;
  const uint32_t G0 = static_cast<uint32_t>(gw * nb / TW), G1 = static_cast<uint32_t>((gw + 1) * nb / TW);
  __syncthreads();
  if (G0 >= G1) return;
  const uint32_t colbytes = a.colbytes, s2 = a.s2, v_start = a.v_start;
  const uint8_t* eos = tab + 128u * colbytes;
  const uint32_t* __restrict__ tokens = a.tokens;
  // ---- prompt slots (warp-uniform): prev / cur / next non-empty prompts around block g
  uint32_t prev_s = 0, cur_s = 0, cur_e = 0, next_e = 0, cur_p = 0, next_p = 0;
  auto load_slots = [&](uint32_t g) {
    cur_p = a.bmap ? __ldg(a.bmap + min(g, nb - 1)) : h16_prompt_of(a.blk_off, N, min(g, nb - 1));
    cur_s = a.blk_off[cur_p];
    cur_e = a.blk_off[cur_p + 1];
    const uint32_t pp = cur_s > 0 ? (a.bmap ? __ldg(a.bmap + cur_s - 1) : h16_prompt_of(a.blk_off, N, cur_s - 1)) : cur_p;
    prev_s = cur_s > 0 ? a.blk_off[pp] : cur_s;
    next_p = h16_nonempty(a.blk_off, N, cur_p + 1);
    next_e = next_p < N ? a.blk_off[next_p + 1] : cur_e;
    __syncwarp();  // every lane's reads of the previous slots precede their rewrite
    if (lane < 3) {
      const uint32_t sp = lane == 0 ? pp : (lane == 1 ? cur_p : next_p);
      slots[lane] = h16_slot(a, sp);
      slot_p[lane] = sp;
    }
    __syncwarp();
  };
  load_slots(G0);
  uint32_t qn = 0;
  uint32_t Pprev = 0, Qprev = 0;  // this lane's packed phase-A / phase-B results of the previous chunk
  for (uint32_t g = G0; g < G1 + 2; g += 32) {
    // advance the slots to the prompt of block g (at most one step for prompts >= 32 blocks)
    if (g >= cur_e && g < nb) {
      if (g < next_e) {
        Slot16 nx{};
        uint32_t nxp = 0;
        if (lane < 2) nx = slots[lane + 1], nxp = slot_p[lane + 1];
        __syncwarp();  // reads (this shift's and the previous chunk's) before the writes
        if (lane < 2) slots[lane] = nx, slot_p[lane] = nxp;
        __syncwarp();
        prev_s = cur_s;
        cur_s = cur_e;
        cur_e = next_e;
        cur_p = next_p;
        next_p = h16_nonempty(a.blk_off, N, cur_p + 1);
        next_e = next_p < N ? a.blk_off[next_p + 1] : cur_e;
        if (lane == 2) {
          slots[2] = h16_slot(a, next_p);
          slot_p[2] = next_p;
        }
        __syncwarp();
      } else {
        load_slots(g);
      }
    }
    const uint32_t k0 = g + lane;              // this lane's block (phase A)
    const uint32_t w = k0 - 2;                 // the window this lane finalises
    const uint32_t lo = max(g, G0 + 2) - 2;    // lowest block whose geometry the chunk needs
    const uint32_t hi_b = min(g + 32, nb);     // one past the highest
    const bool fast = __all_sync(kFull, lo >= prev_s && hi_b <= next_e);  // warp-uniform (a vote)
    unsigned long long tok0 = 0, tokw = 0;
    uint32_t ew = 0, pw = 0, bw = 0;
    if (fast) {
      tok0 = slots[(k0 >= cur_s) + (k0 >= cur_e)].base + 16ull * k0;
      const uint32_t iw = (w >= cur_s) + (w >= cur_e);
      const Slot16 sw = slots[iw];
      tokw = sw.base + 16ull * w;
      ew = sw.tend - static_cast<uint32_t>(tokw);
      bw = w - sw.start;
      pw = iw;  // slot index for now: the prompt id is read only when needed (below)
    } else {  // short prompts: per-lane lookups
      if (k0 < nb) {  // the batch's block -> prompt map when the host built one (short prompts)
        const uint32_t p0 = a.bmap ? __ldg(a.bmap + k0) : h16_prompt_of(a.blk_off, N, k0);
        tok0 = a.tok_off[p0] + 16ull * (k0 - a.blk_off[p0]);
      }
      if (w >= G0 && w < G1) {
        pw = a.bmap ? __ldg(a.bmap + w) : h16_prompt_of(a.blk_off, N, w);
        bw = w - a.blk_off[pw];
        tokw = a.tok_off[pw] + 16ull * bw;
        ew = static_cast<uint32_t>(a.tok_off[pw + 1] - tokw);
      }
    }
    // ---- phase A: own block k0 (digest + DFA from the start state)
    const bool own = k0 < nb && k0 < G1 + 2;
    if (!own) tok0 = 0;  // lanes without a block read the batch's first block (results unused)
    uint32_t t[16];
    uint32_t any = 0;
    if ((tok0 & 3) == 0) {
      ldg_tokens16(tokens + tok0, t, (tok0 & 7) == 0);
    } else {  // a prompt starting at an unaligned token (ragged batches)
#pragma unroll
      for (uint32_t k = 0; k < 16; ++k) t[k] = tokens[tok0 + k];
    }
#if SKV_H16_PF
    {
      const uint64_t nt = tok0 + 512;  // the next chunk's block (exact inside a prompt)
#if SKV_H16_PF == 1
      if (nt < a.n_tokens) asm volatile("prefetch.global.L1 [%0];" ::"l"(tokens + nt));
#else
      if (nt < a.n_tokens) asm volatile("prefetch.global.L2 [%0];" ::"l"(tokens + nt));
#endif
    }
#endif
#pragma unroll
    for (uint32_t k = 0; k < 16; ++k) any |= t[k];
    uint32_t Zb, Xb, faw;  // base states after kConv16 / 16 bytes; flags: bit 0 = [0,4) accepted, bit 1 = [4,16)
    uint64_t dg;
    // a byte >= 128 (or a wide token) in any lane's block: the whole warp takes the general steps
    // (warp-uniform, so the fast path carries no divergence bookkeeping)
    const bool slow_bytes = __any_sync(kFull, any >= 128u);
    if (!slow_bytes) {
      uint64_t h = a.digest_init;
      uint32_t v = v_start;
#pragma unroll
      for (uint32_t k = 0; k < 16; ++k) {
        h = fnv_tok(h, t[k]);
        v = h16_step(tab, colbytes, v, t[k]);
        if (k + 1 == kConv16) {
          faw = v >= s2 ? 1u : 0u;
          v = h16_base(v, s2);
          Zb = v;
        }
      }
      faw |= v >= s2 ? 2u : 0u;
      Xb = h16_base(v, s2);
      dg = h;
    } else {  // a byte >= 128 or a wide token: re-read the (L1-hot) tokens, general steps
      const uint32_t* tp = tokens + tok0;
      uint64_t h = a.digest_init;
      uint32_t v = v_start;
      for (uint32_t k = 0; k < 16; ++k) {
        const uint32_t tv = tp[k];
        h = (any >> 8) ? fnv_u32(h, tv) : fnv_tok(h, tv);
        v = h16_step_any(tab, a.hi, colbytes, v, tv & 0xffu);  // the scan reads the low byte (A.3)
        if (k + 1 == kConv16) {
          faw = v >= s2 ? 1u : 0u;
          v = h16_base(v, s2);
          Zb = v;
        }
      }
      faw |= v >= s2 ? 2u : 0u;
      Xb = h16_base(v, s2);
      dg = h;
    }
    if (a.first && own && k0 >= G0 && k0 < G1) a.d_out[k0] = dg;
    const uint32_t P = own ? (Xb | (faw << 16)) : 0u;
    // ---- phase B: window k0-1 over this block, from X(k0-1)
    const uint32_t Pd1 = __shfl_sync(kFull, lane == 31 ? Pprev : P, (lane + 31) & 31);
    const uint32_t Xp = Pd1 & 0xffffu;
    uint32_t V = Xp;
    if (!slow_bytes) {
#pragma unroll
      for (uint32_t k = 0; k < kConv16; ++k) V = h16_step(tab, colbytes, V, t[k]);
    } else {
      V = h16_run_global(tab, a.hi, colbytes, tokens, tok0, kConv16, V);
    }
    uint32_t C1 = V >= s2 ? 1u : 0u;
    const uint32_t Vb = h16_base(V, s2);
    const bool met = Vb == Zb;  // the runs met: window k0-1's run over [4,16) is this block's own
    uint32_t Y1 = Xb;
    C1 |= met ? faw >> 1 : 0u;
    if (!__all_sync(kFull, met)) {  // a lane whose runs did not meet: the warp steps the rest (uniformly)
      uint32_t v = Vb;
      if (!slow_bytes) {
#pragma unroll
        for (uint32_t k = kConv16; k < 16; ++k) v = h16_step(tab, colbytes, v, t[k]);
      } else {
        v = h16_run_global(tab, a.hi, colbytes, tokens, tok0 + kConv16, 16 - kConv16, v);
      }
      if (!met) {
        C1 |= v >= s2 ? 1u : 0u;
        Y1 = h16_base(v, s2);
      }
    }
    const uint32_t Q = Y1 | (C1 << 16);
    // ---- window w = k0 - 2: its block (lane l-2), its phase B (lane l-1), phase C here
    const uint32_t Pd2 = __shfl_sync(kFull, lane >= 30 ? Pprev : P, (lane + 30) & 31);
    const uint32_t Qd1 = __shfl_sync(kFull, lane == 31 ? Qprev : Q, (lane + 31) & 31);
    Pprev = P;
    Qprev = Q;
    const bool win = w >= G0 && w < G1;
    uint32_t f = 0, sX = 0, sY = 0;
    if (win) {
      const uint32_t Xw = Pd2 & 0xffffu, fa = Pd2 >> 16;
      const uint32_t Yw = Qd1 & 0xffffu, Cw = Qd1 >> 16;
      uint32_t fin;
      if (ew >= 48) {
        uint32_t C2;
        if (Yw == Xp) {  // window w meets window w+1 at this block: its phase C is w+1's phase B
          fin = Y1;
          C2 = C1;
        } else {
          uint32_t v = Yw;
          if (!slow_bytes) {
#pragma unroll
            for (uint32_t k = 0; k < 16; ++k) v = h16_step(tab, colbytes, v, t[k]);
          } else {
            v = h16_run_global(tab, a.hi, colbytes, tokens, tok0, 16, v);
          }
          C2 = v >= s2 ? 1u : 0u;
          fin = h16_base(v, s2);
        }
        f = (fa ? 1u : 0u) | (Cw ? 2u : 0u) | (C2 ? 4u : 0u);
      } else if (ew >= 32) {  // the prompt ends inside [32, 48): block w+1 then the tail
        uint32_t C2 = 0;
        fin = Yw;
        if (ew > 32) {
          const uint32_t v = h16_run_global(tab, a.hi, colbytes, tokens, tokw + 32, ew - 32, Yw);
          C2 = v >= s2 ? 1u : 0u;
          fin = h16_base(v, s2);
        }
        f = (fa ? 1u : 0u) | (Cw ? 2u : 0u) | (C2 ? 4u : 0u);
      } else {  // the prompt ends inside [16, 32)
        uint32_t C1w = 0;
        fin = Xw;
        if (ew > 16) {
          const uint32_t v = h16_run_global(tab, a.hi, colbytes, tokens, tokw + 16, ew - 16, Xw);
          C1w = v >= s2 ? 1u : 0u;
          fin = h16_base(v, s2);
        }
        f = (fa ? 1u : 0u) | (C1w ? 2u : 0u);
      }
      const uint32_t me = *reinterpret_cast<const uint16_t*>(eos + fin);  // end-of-text transition (exact)
      if (a.first)
        a.mask_out[w] = me;
      else if (me)
        atomicOr(&a.mask_out[w], me << a.mask_shift);  // a later rule group (bits shifted to its rules)
      if (fast && (me || f)) pw = slot_p[pw];
      if (me) atomicMin(&a.first_sens[pw], bw);
      sX = Xw;  // segment start states for the exact masks: block w+1 from X(w), block w+2 from Y(w)
      sY = Yw;
    }
    // ---- exact masks of the flagged segments (queued per warp; a pass runs 32 tasks per lane)
    if (__any_sync(kFull, f != 0)) {
      const uint32_t cnt = __popc(f);
      const uint32_t c0 = __ballot_sync(kFull, cnt & 1u), c1 = __ballot_sync(kFull, cnt >> 1);
      const uint32_t tot = __popc(c0) + 2 * __popc(c1);
      if (qn + tot > a.q_cap) {  // q_cap >= 96 = 3 segments x 32 lanes
        h16_flush(q, qn, lane, a, tab);
        qn = 0;
      }
      const uint32_t lt = (1u << lane) - 1u;
      uint32_t k = qn + __popc(c0 & lt) + 2 * __popc(c1 & lt);
      for (uint32_t ff = f; ff; ff &= ff - 1) {
        const uint32_t sg = __ffs(ff) - 1;
        const uint32_t v = sg == 0 ? v_start : (sg == 1 ? sX : sY);
        const uint32_t len = min(16u, ew - 16 * sg);
        H16Task tk;
        tk.tokv = (tokw + 16ull * sg) | (static_cast<unsigned long long>(len) << 40) |
                  (static_cast<unsigned long long>(v) << 46);
        tk.gb = w;
        tk.p = pw;
        q[k++] = tk;
      }
      qn += tot;
    }
  }
  h16_flush(q, qn, lane, a, tab);
}
