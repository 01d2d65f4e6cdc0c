// ctx.hpp -- internal device-side layout shared by capi.cpp and kernels.cu.
//
// HBM layout of the flattened privacy-aware index (replaces the pointer radix tree of
// reference cache_index.hpp:65-98,127-836): one 64-B
// Entry per slot,
//   sector 0 (Rec, 32 B)  key (h,d) + creator + parent slot + label/owner/tier/state
//   sector 1 (32 B)       AccessStats window (hit_cur, u_cnt, hit_pre, u_pre) and
//                         Aux (child-list links, user-set handle, claim/candidate mark)
// Open addressing with linear probing; a slot is empty iff its key is (0,0).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace skv {

constexpr uint32_t kNone = 0xffffffffu;
constexpr uint32_t kMaxSetUsers = 64;  // AccessStats::kMaxTrackedUsers (access_stats.hpp:15)

struct __align__(32) Rec {
  uint64_t h, d;         // chained prefix key, block digest
  uint32_t creator;      // interned UserId of the first inserter (UserTable index)
  uint32_t meta;         // label:2 | owner:1 | tier:2 | live:1 | - :2 | claiming prompt:24 (meta_* helpers)
  uint32_t parent;       // slot of the previous block's entry, kNone for block 0
  uint32_t first_child;  // subtree walk for label propagation (children chained by Aux::next_sibling)
};
static_assert(sizeof(Rec) == 32, "record must be one 32-B sector");

__host__ __device__ inline uint32_t meta_label(uint32_t m) { return m & 3u; }
__host__ __device__ inline uint32_t meta_owner(uint32_t m) { return (m >> 2) & 1u; }
__host__ __device__ inline uint32_t meta_tier(uint32_t m) { return (m >> 3) & 3u; }
__host__ __device__ inline uint32_t meta_prompt(uint32_t m) { return m >> 8; }
__host__ __device__ inline uint32_t make_meta(uint32_t label, uint32_t owner, uint32_t tier, uint32_t prompt) {
  return (label & 3u) | ((owner & 1u) << 2) | ((tier & 3u) << 3) | (1u << 5) | (prompt << 8);
}
constexpr uint32_t kMaxBatchPrompts = 1u << 24;  // the claiming-prompt field of Rec::meta
__host__ __device__ inline bool meta_live(uint32_t m) { return (m >> 5) & 1u; }

// Eviction bookkeeping (skv_enable_eviction), a parallel array beside the entries so the
// admission path's two-sector entry is unchanged: the fields the reference's victim
// order reads (cache_index.hpp:697-728) plus the tombstone flag.
struct __align__(16) EvictMeta {
  uint32_t access_epoch;  // CacheNode::access_epoch: epoch of the last match / insert walk
  uint32_t node_id;       // CacheNode::node_id as the reference assigns it; kNone = assign at this commit
  uint32_t depth;         // block index (children before parents on equal effective keys)
  uint32_t dead;          // 1 = evicted: the key stays as a tombstone until re-inserted
};

struct __align__(16) Stats {
  uint32_t hit_cur, u_cnt, hit_pre, u_pre;
};

struct __align__(16) Aux {
  uint32_t next_sibling;  // next child of the same parent (written only when the parent already had one)
  uint32_t set_idx;       // user-set pool slot for the current window, kNone if untouched
  uint32_t mark;          // epoch: candidate stamp
  uint32_t spare;
};

// One index slot = 64 B.  Sector 0 (Rec) is everything a probe reads AND everything an
// insert writes (claim CAS, payload, the parent's first_child): a commit touches one
// sector per new block.  Sector 1 holds the monitor window and the sibling link.
struct __align__(64) Entry {
  Rec rec;
  Stats stats;
  Aux aux;
};
static_assert(sizeof(Entry) == 64, "entry must be two 32-B sectors");

// Interned user ids (UserId::value -> u32), so that a record's creator fits sector 0.
// Open addressing on keys (empty = kNoUser); idx[slot] = index + 1 once assigned;
// rev[index] = the UserId.
constexpr unsigned long long kNoUser = ~0ull;
struct UserTable {
  unsigned long long* keys = nullptr;
  uint32_t* idx = nullptr;
  uint64_t* rev = nullptr;
  uint32_t* count = nullptr;
  uint32_t mask = 0;   // slots - 1
  uint32_t cap = 0;    // max distinct users
};

// Device forms of the compiled rule DFA (built by capi.cpp upload_rules).
//
// fast  (u16, SMEM-resident in k_hash_scan): row of state s at byte offset
//        row_base + s*row_bytes (the rows end at 32768, so [row_base, fast_bytes) is one
//        contiguous SMEM image),
//        entry (s, c) at +2c = byte offset of the next row.  A transition that ACCEPTS
//        some rule instead points at a copy of the target row placed at >= 32768
//        (kAccRegion), so "this window matched something" is bit 15 of the OR of all
//        visited offsets -- no per-step mask work.  Entries of the EOS column are 0 or a
//        pseudo offset >= 32768.
// full  (u32, global, read through L1): entry (s, c) at index s*(C+1)+c =
//        (enabled-rule mask << 16) | canonical next-row byte offset (fast format, < 32768).
//        Used to compute the exact rule mask of the (rare) windows the fast pass flags,
//        and by the per-call tier1_scan wrapper.
constexpr uint32_t kAccRegion = 32768;

struct DevRules {
  uint16_t* fast = nullptr;
  uint32_t* full = nullptr;
  uint8_t* class2 = nullptr;  // [256] byte -> 2 * class
  uint32_t fast_bytes = 0;    // kAccRegion + accepting-copy rows
  uint32_t norm_bytes = 0;    // n_states * row_bytes (< kAccRegion)
  uint32_t row_base = 0;      // offset of state 0's row: rows fill [row_base, kAccRegion)
  uint32_t row_bytes = 0;     // 2 * (n_classes + 1)
  uint32_t start_row = 0;     // start * row_bytes
  uint32_t eos2 = 0;          // 2 * n_classes
  uint32_t n_enabled = 0;
  uint16_t* copy_acc = nullptr;  // [n_copies] rule mask of accepting-copy row j
  uint32_t n_copies = 0;
  uint32_t copy_inv = 0;  // ceil(2^32 / row_bytes): j = umulhi(offset - kAccRegion, copy_inv)
};

// The B = 16 / W = 32 automaton of k_hash_scan16 (hash_scan16.cuh): byte-indexed
// columns (entry (byte t, state) at t * colbytes + v, v = 2 * state index), every state with a
// shadow copy (index + S) that accepting transitions enter and never leave.
struct DevRules16 {
  bool ok = false;       // built (B == 16, W == 32 and the image fits SMEM beside the task queues)
  uint16_t* img = nullptr;   // 129 columns (bytes 0..127, then EOS rule masks) x 2S, SMEM image
  uint32_t img_bytes = 0;
  uint16_t* hi = nullptr;    // bytes 128..255 (global)
  uint32_t* full = nullptr;  // [256][S]: (rule mask << 16) | v(next), base states (exact masks)
  uint32_t colbytes = 0, s2 = 0, v_start = 0, q_cap = 0, smem = 0;
  int grid = 0;
};

struct HS16Args {
  const uint32_t* tokens;
  const uint64_t* tok_off;
  const uint32_t* blk_off;
  uint32_t n_prompts;
  uint64_t n_tokens;
  uint64_t digest_init;
  const uint16_t* img;
  uint32_t img_bytes;
  const uint16_t* hi;
  const uint32_t* full;
  uint32_t colbytes;  // 4S
  uint32_t s2;        // 2S: v >= s2 <=> shadow (accepted) state
  uint32_t v_start;
  uint32_t q_cap;  // deferred exact tasks per warp (>= 96)
  uint32_t mask_shift;  // bit of this rule group's first rule in the window masks
  uint32_t first;       // 1: the first group (stores digests and masks); else masks are OR-ed in
  uint64_t* d_out;
  uint32_t* mask_out;
  uint32_t* first_sens;
  const uint32_t* bmap = nullptr;  // block -> prompt (short-prompt batches), else binary searches
};

struct HashScanArgs {
  const uint32_t* tokens;
  const uint64_t* tok_off;
  const uint32_t* blk_off;
  uint32_t n_prompts;
  uint64_t n_tokens;
  uint32_t n_blocks;
  uint32_t B, W;
  uint64_t digest_init;  // FNV state after update_u32(B)
  DevRules rules;
  uint32_t mask_shift;  // bit of this rule group's first rule in the window masks
  uint32_t first;       // 1: the first group (stores digests and masks); else masks are OR-ed in
  uint64_t* d_out;
  uint32_t* mask_out;
  uint32_t* first_sens;
  // dynamic shared-memory layout (hash_scan_layout)
  uint32_t off_list, stage, buf_gap, n_gap, buf_tail;  // hash_scan_layout
};

struct HSLayout {
  uint32_t stage, off_list, buf_gap, n_gap, buf_tail, warps, total;
};

// Replicated layer (multi-GPU, skv_set_replicated_depth): entries at depth < depth exist on every
// rank.  Their accesses are not recorded locally but aggregated per (entry, user) -- first prompt of
// the batch, access count -- into an open-addressed pair table (key {user, slot + 1}, empty = 0), and
// the commit lists the replicated-layer entries it creates; both are exported, merged over the ranks
// and applied identically everywhere (skv_replica_export / skv_replica_apply).
struct RepLayer {
  uint32_t depth = 0;           // 0: nothing replicated
  ulonglong2* pair_key = nullptr;
  uint32_t* pair_first = nullptr;  // lowest local prompt index (init ~0)
  unsigned long long* pair_gid = nullptr;  // apply: lowest global prompt id (init ~0)
  uint32_t* pair_cnt = nullptr;
  uint32_t pair_mask = 0;
  uint32_t* new_list = nullptr;  // slots the commit created at depth < depth
  uint32_t* new_n = nullptr;
  uint32_t new_cap = 0;
  uint32_t* err = nullptr;       // bit 0: pair table full, bit 1: new list full
};

struct Index {
  Entry* e = nullptr;
  uint64_t cap = 0, mask = 0;
  RepLayer rep;
  EvictMeta* em = nullptr;  // null unless eviction is enabled
  // per commit (eviction enabled): speculative node-id bases (exclusive prefix over prompts of
  // the blocks each would create), the next node id and the insert epoch
  const uint32_t* em_base = nullptr;
  uint32_t em_next = 0, em_epoch = 0;
};

// Monitor user sets (AccessStats::user_set, access_stats.hpp:21-37), one per entry touched
// in the current monitor window, allocated from a pool on first touch.  A set is a
// 128-slot open-addressed table of {user, stamp} (128-bit CAS inserts); a slot is live iff
// its stamp (admit-batch id) >= the window's first batch id, so tables never need
// clearing.  `size` = users admitted before the current batch.
constexpr uint32_t kSetSlots = 128;
constexpr uint32_t kPendingSet = 0xfffffffeu;

struct SetHdr {
  uint32_t size;   // admitted members at the start of the current batch
  uint32_t touch;  // unused
  uint32_t ovf;    // batch in which the first-64 boundary was crossed (needs ordered replay)
  uint32_t pad;
  unsigned long long cnt;  // (batch << 32) | distinct users inserted in that batch
};

struct MonCtx {
  SetHdr* hdr;
  ulonglong2* tab;  // pool_cap * kSetSlots
  uint32_t pool_cap;
  uint32_t* pool_count;
  uint32_t* touched;    // entries touched in the current window
  uint32_t* n_touched;
  uint32_t batch;   // admit-batch id (>= 1)
  uint32_t wstart;  // first batch id of the current window
  uint32_t* err;
  uint32_t* matched_total;
  // graph-replayed steps (capi.cpp "CUDA graphs"): the window and batch stamps live on the device
  // ({batch, wstart, cur} at st[0..2], written before each graph launch); kernels then take the
  // current window list from tl[cur] and its count from ntb[cur].  st == nullptr: the fields above.
  const uint32_t* st = nullptr;
  uint32_t* tl[2] = {nullptr, nullptr};
  uint32_t* ntb = nullptr;
};

// CostModel (serving_sim.hpp:25-57) in device form
struct CostModelDev {
  double t_base = 10.0, c_prefill = 1.0;
  double penalty[4] = {0.0, 0.2, 0.5, 0.0};  // HBM, DRAM, SSD (index 3 unused)
  double sigma = 0.0;
  uint64_t seed = 0;
};

void launch_init_entries(const Index& ix, cudaStream_t s);
void launch_widen(const uint8_t* in, uint32_t* out, uint64_t n, cudaStream_t s);
// eviction (kernels.cu): access epochs of matched blocks at admit; node ids + access epochs
// of every committed block at commit; evict(needed) = effective keys, sort, tombstones
void launch_touch_matched(const Index& ix, const uint32_t* slot, const uint32_t* blk_off, const uint32_t* matched,
                          uint32_t n, uint32_t epoch, cudaStream_t s);
bool node_ids_speculative();
void launch_node_bases(const uint32_t* blk_off, const uint32_t* exist, uint32_t n, uint32_t* counts, uint32_t* base,
                       void* temp, size_t temp_bytes, cudaStream_t s);
void launch_path_epochs(const Index& ix, const uint32_t* slot, const uint32_t* blk_off, const uint32_t* exist,
                        uint32_t n, uint32_t epoch, cudaStream_t s);
void launch_assign_nodes(const Index& ix, const uint32_t* slot, const uint32_t* blk_off, const uint32_t* exist,
                         uint32_t n, uint32_t* counts, uint32_t* incl, uint64_t next_id, void* temp,
                         size_t temp_bytes, cudaStream_t s);
size_t evict_temp_bytes(uint32_t n_prompts, uint64_t cap);
// A.9 budgeted commit (kernels.cu)
struct BudgetSim {
  unsigned long long used;  // HBM blocks after the round
  uint32_t n_victims, next_lo, dropped, pad;
};
void launch_new_bound(const uint32_t* blk_off, const uint32_t* exist, uint32_t lo, uint32_t hi,
                      unsigned long long* out, cudaStream_t s);
void launch_mark_paths(const uint32_t* slot, const uint32_t* blk_off, const uint32_t* exist, const uint32_t* matched,
                       uint32_t lo, uint32_t hi, uint32_t* vstamp, uint32_t* list, uint32_t* n_list, uint32_t cap,
                       cudaStream_t s);
void launch_clear_marks(uint32_t* vstamp, const uint32_t* list, const uint32_t* n_list, uint32_t cap, cudaStream_t s);
void launch_reprobe(const Index& ix, const uint64_t* h, const uint64_t* d, const uint32_t* blk_off, uint32_t lo,
                    uint32_t hi, uint32_t* exist, uint32_t* slot_out, cudaStream_t s);
void launch_dry_needed(const uint64_t* h, const uint64_t* d, const uint32_t* blk_off, const uint32_t* exist,
                       uint32_t lo, uint32_t hi, ulonglong2* tab, uint32_t* minp, uint64_t tcap, uint32_t* dslot,
                       uint32_t* needed, cudaStream_t s);
uint32_t launch_evict_order(const Index& ix, const uint32_t* vstamp, unsigned long long* eff,
                            unsigned long long* keys_a, unsigned long long* keys_b, uint32_t* vals_a, uint32_t* vals_b,
                            uint32_t* n_live, void* temp, size_t temp_bytes, uint32_t* host_n, cudaStream_t s);
void launch_budget_sim(const uint32_t* needed, uint32_t lo, uint32_t hi, uint64_t used, uint64_t cap,
                       const uint32_t* vals, uint32_t nv, const unsigned long long* eff, const uint32_t* vstamp,
                       uint32_t epoch, uint32_t* victims, BudgetSim* out, cudaStream_t s);
void launch_evict_mark_list(const Index& ix, const uint32_t* vals, uint32_t v, cudaStream_t s);
void launch_count_tiers(const Index& ix, unsigned long long* out3, cudaStream_t s);
// tiered rounds (bounded DRAM / SSD): cap-sized work arrays, 3 tiers x cap_each candidates
struct TieredWork {
  uint32_t* cc = nullptr;       // live children per slot (round start)
  uint32_t* cc_work = nullptr;  // the simulation's copy
  uint8_t* tier = nullptr;      // current tier per slot during the simulation
  unsigned long long *keys_a = nullptr, *keys_b = nullptr, *hk = nullptr;
  uint32_t *vals_a = nullptr, *vals_b = nullptr, *hv = nullptr;
  uint64_t cap_each = 0;
  uint32_t* n3 = nullptr;
  uint32_t* act = nullptr;  // actions (slot | kind << 30)
  uint64_t act_cap = 0;
  uint32_t* n_act = nullptr;
  unsigned long long* used3 = nullptr;
  BudgetSim* res = nullptr;
  void* temp = nullptr;
  size_t temp_bytes = 0;
};
BudgetSim launch_budget_tiered(const Index& ix, const TieredWork& w, const uint32_t* vstamp, const uint32_t* needed,
                               uint32_t lo, uint32_t hi, uint64_t need_evict, const uint64_t* used3,
                               const uint64_t* cap3, uint32_t epoch, uint32_t* host, cudaStream_t s);
uint32_t launch_evict(const Index& ix, uint64_t needed, unsigned long long* eff, unsigned long long* keys_a,
                      unsigned long long* keys_b, uint32_t* vals_a, uint32_t* vals_b, uint32_t* n_live, void* temp,
                      size_t temp_bytes, uint64_t* victims_h, uint64_t* victims_d, uint32_t* host_n, int tiered,
                      cudaStream_t s);
void launch_intern_users(const UserTable& t, const uint64_t* users, uint32_t n, uint32_t* uidx, uint32_t* err,
                         cudaStream_t s);
void launch_ttft(const uint32_t* blk_off, const uint32_t* matched, const uint32_t* plen, const uint8_t* bmeta,
                 const uint64_t* request_ids, uint64_t request_base, uint32_t n, uint32_t B, const CostModelDev& cm,
                 double* ttft, uint32_t* intra, uint32_t* inter, cudaStream_t s);

// kernel launchers (kernels.cu)
void launch_block_counts(const uint64_t* tok_off, uint32_t n, uint32_t B, uint32_t* counts, uint32_t* plen,
                         cudaStream_t s);
size_t scan_temp_bytes(uint32_t n);
void launch_exclusive_scan(void* temp, size_t temp_bytes, const uint32_t* in, uint32_t* out, uint32_t n,
                           cudaStream_t s);
int hash_scan_grid(int device, uint32_t smem_bytes, uint32_t threads);
HSLayout hash_scan_layout(const DevRules& r, uint32_t B, uint32_t W);
void launch_hash_scan(const HashScanArgs& a, int grid, uint32_t smem, uint32_t threads, cudaStream_t s);
// k_hash_scan16: fixed task-queue / slot layout; returns the dynamic SMEM bytes for an image and
// queue capacity, and the persistent grid (-1 on failure)
uint32_t hash_scan16_smem(uint32_t img_bytes, uint32_t q_cap, uint32_t warps = 0);
int hash_scan16_grid(int device, uint32_t smem);
void launch_hash_scan16(const HS16Args& a, int grid, uint32_t smem, cudaStream_t s, int warps = 0);
// diagnostic: per entry matched by the last admitted batch, its accesses, distinct users and the
// Shannon entropy (bits) of the batch's accesses over users; returns the entries written
uint32_t launch_access_entropy(const Index& ix, const uint32_t* blk_off, const uint32_t* matched,
                               const uint32_t* slot, const uint32_t* uidx, uint32_t n_prompts, uint32_t n_access,
                               uint64_t* out_h, uint64_t* out_d, uint64_t* out_acc, uint64_t* out_users,
                               double* out_bits, uint32_t cap, uint32_t* total, cudaStream_t s);
// block -> prompt map of a batch (warp per prompt), for short-prompt batches
void launch_block_prompts(const uint32_t* blk_off, uint32_t n_prompts, uint32_t* map, cudaStream_t s);
void launch_chain_probe(const Index& ix, const uint64_t* d, const uint32_t* blk_off, const uint32_t* first_sens,
                        const uint32_t* uidx, uint32_t n_prompts, uint64_t* h, uint8_t* label, uint8_t* decision,
                        uint32_t* slot, uint32_t* matched, uint32_t* exist, uint8_t* tier, uint8_t* bmeta,
                        const MonCtx& mon, uint32_t* bprompt, int prechained, uint32_t split_from, cudaStream_t s);
void launch_chain(const uint64_t* d, const uint32_t* blk_off, const uint32_t* first_sens, uint32_t n, uint64_t* h,
                  uint8_t* label, uint32_t* slot, cudaStream_t s);
void launch_record(const Index& ix, const MonCtx& mon, const uint32_t* slot, const uint32_t* blk_off,
                   const uint32_t* matched, const uint64_t* users, uint32_t n_prompts, cudaStream_t s);
void launch_record_finish(const Index& ix, const MonCtx& mon, uint32_t* replay, uint32_t* n_replay, int grid,
                          cudaStream_t s);
void launch_replay_emit(const Index& ix, const MonCtx& mon, const uint32_t* slot, const uint32_t* blk_off,
                        const uint32_t* matched, uint32_t n_prompts, unsigned long long* keys, uint32_t* n_keys,
                        cudaStream_t s);
size_t sort_keys_temp_bytes(uint32_t n, int end_bit);
void launch_sort_keys(void* temp, size_t temp_bytes, const unsigned long long* in, unsigned long long* out, uint32_t n,
                      int end_bit, cudaStream_t s);
void launch_record_replay(const Index& ix, const MonCtx& mon, const uint32_t* replay, const uint32_t* n_replay,
                          const unsigned long long* keys, uint32_t n_keys, const uint64_t* users, int grid,
                          cudaStream_t s);
void launch_commit(const Index& ix, const uint64_t* h, const uint64_t* d, const uint32_t* blk_off,
                   const uint32_t* exist, const uint8_t* label, const uint32_t* uidx, const uint8_t* owners,
                   uint32_t n_prompts, uint32_t* slot, unsigned long long* n_new, uint32_t* fix_list, uint32_t* n_fix,
                   uint32_t fix_cap, uint32_t* err_flag, int fix_grid, const uint32_t* matched,
                   const uint64_t* users64, const MonCtx* mon, int pending_labels, uint64_t n_blocks, int n_sm,
                   const uint32_t* bprompt, uint32_t* late, uint32_t* n_late, uint32_t* n_revived,
                   const MonCtx& pool, cudaStream_t s);
void launch_resolve(const Index& ix, const uint64_t* h, const uint64_t* d, const uint32_t* boff, uint32_t n_prompts,
                    const uint32_t* first, const uint8_t* labels, uint32_t n, uint32_t* missing, cudaStream_t s);
void launch_epoch_candidates(const Index& ix, const uint32_t* list, const uint32_t* n_list, uint32_t grid_n,
                             int only_untouched, uint32_t stamp, double jump, uint64_t u_pre_max, uint32_t* cands,
                             uint32_t* n_cands, cudaStream_t s, const uint32_t* guard = nullptr);
void launch_epoch_fire(const Index& ix, const uint32_t* cands, const uint32_t* n_cands, uint32_t grid_n,
                       uint32_t stamp, uint64_t epoch, void* events, uint32_t* n_events, uint32_t* fired,
                       cudaStream_t s, const uint32_t* guard = nullptr);
void launch_epoch_propagate(const Index& ix, const uint32_t* fired, const uint32_t* n_events, uint32_t grid_n,
                            cudaStream_t s, const uint32_t* guard = nullptr);
// the whole epoch pass (candidates, fire, propagate, rolls, window-swap resets) in one
// cooperative launch
// (st != nullptr: cur, stamp and epoch from the device step state st[2], st[3], st[4..5]; the lists
// are lists[cur] / lists[1 - cur] with counts ntb[cur] / ntb[1 - cur].  guard != nullptr -- and,
// with st, st[6] != 0 -- arms a speculative pass: it returns untouched when guard[5] (commit
// errors) or guard[8] (ordered replay pending) is set.)
cudaError_t launch_epoch_fused(const Index& ix, uint32_t* const lists[2], uint32_t* ntb, int cur, uint32_t stamp,
                               double jump, uint64_t u_pre_max, uint32_t* cands, uint32_t* n_cands, uint64_t epoch,
                               void* events, uint32_t* n_events, uint32_t* fired, uint32_t* pool_count,
                               const uint32_t* st, const uint32_t* guard, int device, cudaStream_t s);
void launch_epoch_roll(const Index& ix, const uint32_t* list, const uint32_t* n_list, uint32_t grid_n, int prev_list,
                       cudaStream_t s, const uint32_t* guard = nullptr);
void launch_epoch_reset(uint32_t* pool_count, uint32_t* prev_count, const uint32_t* guard, cudaStream_t s);
void launch_set_tiers(const Index& ix, const uint64_t* h, const uint64_t* d, const uint32_t* boff, uint32_t n_prompts,
                      const uint8_t* tiers, uint32_t n,
                      cudaStream_t s);
void launch_export(const Index& ix, const uint64_t* user_rev, void* out, uint32_t* n_out, uint32_t cap,
                   cudaStream_t s);
void launch_scan_text(const uint8_t* text, uint32_t len, DevRules r, uint32_t* mask, uint32_t shift, cudaStream_t s);
void launch_scan_texts(const uint8_t* text, const uint64_t* off, uint32_t n, DevRules r, uint32_t* masks,
                       uint32_t shift, cudaStream_t s);
void launch_digest(const uint32_t* tokens, uint32_t n, uint64_t* out, cudaStream_t s);
uint32_t record_grid(int device);
void launch_leak_flags(const uint32_t* blk_off, const uint8_t* label, const uint32_t* span_off, const uint64_t* sb,
                       const uint64_t* se, uint32_t n_prompts, uint32_t B, uint8_t* flags,
                       unsigned long long* n_leaks, cudaStream_t s);
// per-entry calls of the reference-API facade (kernels.cu)
void launch_find_entries(const Index& ix, const uint64_t* h, const uint64_t* d, uint32_t n, uint32_t* slots,
                         cudaStream_t s);
void launch_label_entries(const Index& ix, const uint32_t* slots, uint32_t n, uint32_t label, int propagate,
                          unsigned long long* changed, cudaStream_t s);
void launch_record_list(const Index& ix, const MonCtx& M, const uint32_t* slots, const uint64_t* users, uint32_t n,
                        cudaStream_t s);
void launch_roll_list(const Index& ix, const MonCtx& M, const uint32_t* slots, uint32_t n, cudaStream_t s);
void launch_check_one(const Index& ix, uint32_t slot, double jump, uint64_t u_pre_max, uint64_t epoch, void* ev,
                      int* fired, cudaStream_t s);
// replicated layer (multi-GPU): export / clear / apply (kernels.cu)
void launch_rep_export(const Index& ix, const uint64_t* user_rev, const uint64_t* gids, uint32_t n_new, void* ents,
                       void* accs, uint32_t* n_accs, uint32_t acc_cap, cudaStream_t s);
void launch_rep_clear(const Index& ix, cudaStream_t s);
// device merge scratch of skv_replica_apply (pair capacity each)
struct RepScratch {
  unsigned long long *gid_a = nullptr, *gid_b = nullptr;
  uint32_t *val_a = nullptr, *val_b = nullptr, *slot_a = nullptr, *slot_b = nullptr, *n = nullptr;
  uint32_t* host_n = nullptr;  // pinned
  void* temp = nullptr;
  size_t temp_bytes = 0;
};
size_t rep_sort_temp_bytes(uint32_t n);
void launch_rep_apply(const Index& ix, const MonCtx& M, const void* ents, const uint32_t* uidx, uint32_t n_ents,
                      uint32_t* slots, uint32_t* n_claimed, const void* accs, uint32_t n_accs, const RepScratch& W,
                      uint32_t* err, cudaStream_t s);

}  // namespace skv
