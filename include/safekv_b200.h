/* safekv_b200.h -- C ABI of the B200-native SafeKV admission hot path.
 *
 * This is the drop-in boundary for the per-batch admission path of the SafeKV
 * reference (arxiv 2508.08438, /root/reference/proj/include/safekv).  The reference is
 * header-only C++ with no FFI of its own; each entry point below names the reference
 * interface it replaces (file:line under proj/include/safekv/).  The C++ facade in
 * include/safekv_b200/safekv.hpp re-exposes these under the reference's class and
 * method names; INTEGRATION.md shows how ServingSimulator::submit would call them.
 *
 * Conventions
 *  - Every call returns an int status (SKV_OK == 0).  The facade rethrows the
 *    matching safekv::Error subclass (core.hpp:19-59).
 *  - The caller owns all buffers it passes; the context owns device memory.
 *  - One CUDA stream per context; calls on one context are serialised, mirroring the
 *    reference's single-writer contract (cache_index.hpp:122-127).
 *  - There is no CPU fallback: without a CUDA device skv_create fails with
 *    SKV_ERR_CUDA.  Rule compilation (skv_rules_*) is host-only, like the
 *    reference's std::regex construction (detection.hpp:120-144).
 */
#ifndef SAFEKV_B200_H_
#define SAFEKV_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SKV_ABI_VERSION 1

enum {
  SKV_OK = 0,
  SKV_ERR_ARG = 1,       /* bad argument (null pointer, size mismatch)            */
  SKV_ERR_PARSE = 2,     /* safekv::ParseError      (detection.hpp:224-279)      */
  SKV_ERR_COMPILE = 3,   /* safekv::CompileError    (detection.hpp:126-137)      */
  SKV_ERR_CONFIG = 4,    /* safekv::ConfigError                                   */
  SKV_ERR_CAPACITY = 5,  /* safekv::CapacityExhausted (cache_index.hpp:801-806)   */
  SKV_ERR_STATE = 6,     /* call-order violation (e.g. commit with no admitted batch) */
  SKV_ERR_CUDA = 7,      /* no sm_100 device, or a CUDA runtime failure           */
  SKV_ERR_INTERNAL = 8
};

/* SensitivityLabel values (core.hpp:167) */
enum { SKV_LABEL_PRIVATE = 0, SKV_LABEL_PUBLIC = 1, SKV_LABEL_PENDING = 2, SKV_LABEL_RESTRICTED = 3 };
/* MemTier values (core.hpp:145) */
enum { SKV_TIER_HBM = 0, SKV_TIER_DRAM = 1, SKV_TIER_SSD = 2 };
/* per-block lookup decision */
enum { SKV_MISS = 0, SKV_PUBLIC_HIT = 1, SKV_OWNER_HIT = 2 };
/* AnomalyAction (monitor.hpp:17) */
enum { SKV_ACTION_NONE = 0, SKV_ACTION_DOWNGRADE = 1, SKV_ACTION_RESTRICT = 2 };

/* ------------------------------------------------------------------------------
 * Rule sets (host).  Replaces CompiledRuleSet::compile (detection.hpp:120-144),
 * RuleEngine::load_rules_json (detection.hpp:222-242) and default_pattern_rules
 * (detection.hpp:185-204).  A skv_rules is an immutable snapshot (the reference's
 * shared_ptr<const CompiledRuleSet>); the rule list is compiled into one search DFA.
 * ------------------------------------------------------------------------------ */
typedef struct skv_rules skv_rules;

int skv_rules_default(skv_rules** out);
/* err receives the reference-style message ("rule 'b': bad regex: ..."). */
int skv_rules_from_json(const char* json, size_t len, skv_rules** out, char* err, size_t errcap);
void skv_rules_free(skv_rules* r);
uint64_t skv_rules_version(const skv_rules* r);
uint32_t skv_rules_count(const skv_rules* r);
/* rule i: id, category, kind (0 regex, 1 blacklist), enabled */
int skv_rules_info(const skv_rules* r, uint32_t i, const char** rule_id, const char** category, int* kind,
                   int* enabled);
size_t skv_rules_warning_count(const skv_rules* r);
const char* skv_rules_warning(const skv_rules* r, size_t i);
/* The device runs a rule set as consecutive groups of <= 16 enabled rules whose automata fit its
 * tables (one scan pass per group; no group straddles a 32-rule mask word), so rule libraries of
 * up to 32 * SKV_MAX_MASK_WORDS enabled rules load whatever their automaton size (the reference
 * accepts any size, detection.hpp:222-242; beyond the maximum: SKV_ERR_COMPILE at load). */
#define SKV_MAX_MASK_WORDS 32
uint32_t skv_rules_group_count(const skv_rules* r);
/* Device rule masks use bit j = j-th ENABLED rule; this maps j -> rule list index. */
uint32_t skv_rules_enabled_count(const skv_rules* r);
uint32_t skv_rules_enabled_rule(const skv_rules* r, uint32_t j);
/* u32 words of a window's rule mask: ceil(enabled / 32), at least 1.  Word w holds bits
 * 32w .. 32w+31; every per-window mask output below with more than one word is word-major
 * (word w of all windows, then word w + 1). */
uint32_t skv_rules_mask_words(const skv_rules* r);

/* Read-only view of the compiled automaton (tests / tooling); SKV_ERR_COMPILE for a set of more
 * than 32 enabled rules (it exists only as its groups' automata). */
typedef struct {
  uint32_t n_states, n_classes, start;
  const uint8_t* class_map; /* [256] byte -> class                     */
  const uint16_t* next;     /* [n_states * n_classes]                   */
  const uint32_t* acc;      /* [n_states * (n_classes + 1)], last = EOS */
  uint32_t nfa_states, dfa_states_unminimized;
} skv_dfa_view;
int skv_rules_dfa(const skv_rules* r, skv_dfa_view* out);

/* ------------------------------------------------------------------------------
 * Context.  Holds the device-resident index (flattened, hash-addressed replacement
 * of RadixCacheIndex, cache_index.hpp:127-836), the monitor state (EntropyMonitor,
 * monitor.hpp:44-113) and the active rule DFA.
 * ------------------------------------------------------------------------------ */
typedef struct skv_ctx skv_ctx;

typedef struct {
  int device;                  /* CUDA device ordinal                                 */
  uint32_t block_tokens;       /* B: tokens per KV block (1..4096; the facade uses 1)  */
  uint32_t window_tokens;      /* W: right-context tokens of a block's scan window    */
  uint64_t index_capacity;     /* entry slots (rounded up to a power of two)          */
  uint64_t max_prompts;        /* per batch (<= 2^24)                                 */
  uint64_t max_tokens;         /* per batch                                           */
  uint64_t max_window_entries; /* distinct entries touched per monitor window         */
  double entropy_jump;         /* MonitorConfig::entropy_jump (monitor.hpp:12)        */
  uint64_t u_pre_max;          /* MonitorConfig::u_pre_max    (monitor.hpp:13)        */
  uint64_t max_users;          /* distinct UserIds the context can intern (creators)  */
} skv_config;

void skv_config_default(skv_config* c);
int skv_create(const skv_config* c, skv_ctx** out);
int skv_destroy(skv_ctx* ctx);
const char* skv_last_error(const skv_ctx* ctx);
/* Atomic snapshot swap; takes effect at the next skv_admit (RuleEngine::load_rules
 * swap semantics, detection.hpp:238-241).  The context keeps its own copy. */
int skv_set_rules(skv_ctx* ctx, const skv_rules* r);
/* cudaStream_t of the context (as void*). */
void* skv_stream(skv_ctx* ctx);

/* ------------------------------------------------------------------------------
 * Batch admission: phase L = skv_admit, phase C = skv_commit,
 * phase E = skv_epoch.  Replaces the per-request sequence of ServingSimulator::submit
 * (serving_sim.hpp:184-218): token_seq_digest (core.hpp:68-73),
 * RuleEngine::tier1_scan (detection.hpp:217), RadixCacheIndex::match_prefix
 * (cache_index.hpp:213-237), EntropyMonitor::record_access (monitor.hpp:50),
 * RadixCacheIndex::insert + resolve_block (cache_index.hpp:152-205, 321-343) and
 * EntropyMonitor::epoch_pass (monitor.hpp:85-99).
 * ------------------------------------------------------------------------------ */
typedef struct {
  const uint32_t* tokens;  /* concatenated prompts, TokenId = uint32 (core.hpp:65) */
  const uint64_t* offsets; /* n_prompts + 1 token offsets                          */
  const uint64_t* users;   /* UserId::value per prompt (core.hpp:129-135)          */
  const uint8_t* owners;   /* OwnerClass per prompt (0 Customer, 1 Business); NULL = Customer */
  uint32_t n_prompts;
  uint64_t n_tokens;
  int on_device;           /* 1: all pointers are device pointers (inputs resident in HBM) */
  /* optional, instead of tokens: the prompts' tokens as bytes -- the reference's ByteVocabulary
   * (core.hpp:92-101: TokenId = byte value), e.g. the prompt text itself.  A quarter of the
   * tokens' host->device copy; widened to TokenIds on the device.  tokens is then ignored. */
  const uint8_t* token_bytes;
} skv_batch;

typedef struct {
  /* per block, prompt-major, n_blocks = sum floor(L_p / B).  Any pointer may be NULL. */
  uint64_t* block_h;     /* chained prefix key h_b                          */
  uint64_t* block_d;     /* token_seq_digest of the block d_b               */
  uint8_t* label;        /* SKV_LABEL_PRIVATE / SKV_LABEL_PUBLIC (A.4)      */
  uint32_t* rule_mask;   /* window verdict, bit j = j-th enabled rule (A.3); word 0 of
                          * the mask (more words: skv_last_rule_masks)              */
  uint8_t* decision;     /* SKV_MISS / SKV_PUBLIC_HIT / SKV_OWNER_HIT (A.5) */
  /* per prompt */
  uint32_t* matched_blocks; /* longest visible prefix, in blocks            */
  uint8_t* lowest_tier;     /* MatchResult::lowest_tier (cache_index.hpp:234) */
  uint64_t* block_offsets;  /* n_prompts + 1                                 */
  int on_device;            /* 1: the pointers above are device pointers     */
  /* summary, always filled (host) */
  uint64_t n_blocks;
  uint64_t matched_total;
} skv_admit_out;

int skv_admit(skv_ctx* ctx, const skv_batch* batch, skv_admit_out* out);
/* The last admitted batch's full window rule masks: skv_mask_words(ctx) words per block,
 * word-major (out[w * n_blocks + b]); valid until the next skv_admit or skv_set_rules. */
int skv_last_rule_masks(skv_ctx* ctx, uint32_t* out, int on_device);
/* CUDA graphs for small batches (default on; SKV_GRAPHS=0 in the environment turns the default
 * off): a device-resident batch admitted without per-block outputs (no eviction, budgets,
 * replicated layer or prefetch) replays its admit, commit and epoch launches from graphs captured
 * once per buffer set; the per-step stamps come from a device-side step state.  Results are
 * identical either way; only the host issue cost differs. */
int skv_set_graphs(skv_ctx* ctx, int on);
/* Diagnostic (no reference counterpart; SURVEY D4 -- the monitor's flags use the reference's
 * u / h predicate): for every entry the last admitted batch matched, that batch's accesses, its
 * distinct users and the Shannon entropy in bits of its accesses over users, H = log2 T -
 * sum_u c_u log2 c_u / T.  Entries in slot order; *n_entries = all of them (the first cap are
 * written).  Valid until the next skv_admit. */
int skv_access_entropy(skv_ctx* ctx, uint64_t* h, uint64_t* d, uint64_t* accesses, uint64_t* users, double* bits,
                       size_t cap, size_t* n_entries);
/* mask words of the context's active rule set (skv_rules_mask_words of it) */
uint32_t skv_mask_words(const skv_ctx* ctx);
/* Cross-batch pipelining: stage the NEXT device-resident batch's digests and window
 * rule masks (stages 1-2, which read no index state) on a side stream, so they overlap
 * the pending batch's commit/epoch.  The next skv_admit with the same tokens/offsets
 * pointers and sizes consumes them; any other admit, or skv_set_rules, drops them.
 * A host batch is copied to the device asynchronously on the side stream, so the caller
 * must keep its host buffers (tokens, offsets, users, owners) alive and unchanged until the
 * consuming admit returns (a rewritten buffer would be admitted with stale stages 1-2).
 * Device batches must likewise stay unchanged until that admit; device batches whose tokens
 * are not 16-B aligned are ignored (admitted inline).  Results are identical with or
 * without prefetch; there is no reference counterpart (the reference admits one prompt at
 * a time). */
int skv_prefetch(skv_ctx* ctx, const skv_batch* next);
/* Host-input staging (end-to-end pipelining): queue the host->device copy of a HOST batch
 * (tokens or token bytes, offsets, users, owners) on a copy stream into one of three device
 * slots, so the copies of batches k+1..k+3 overlap the admission of batch k.  A later
 * skv_prefetch / skv_admit of the same batch (same pointers and sizes) reads the staged copy;
 * the caller keeps the host buffers unchanged until that admit returns.  A slot is reused once
 * the batch admitted from it is committed (or dropped); with every slot busy the call stages
 * nothing and the batch is copied inline later.  Pinned host memory makes the copy
 * asynchronous.  No reference counterpart (the reference has no device). */
int skv_stage(skv_ctx* ctx, const skv_batch* batch);
/* Insert the new blocks of the last admitted batch (first creator wins; intra-batch
 * duplicates are won by the lowest prompt index).  new_entries may be NULL.  A capacity
 * failure detected after the kernels ran (probe sequence or monitor set pool exhausted)
 * returns SKV_ERR_CAPACITY and leaves the context unusable for further batches (every
 * later batch call returns SKV_ERR_STATE naming the cause; skv_export still works). */
int skv_commit(skv_ctx* ctx, uint64_t* new_entries);

typedef struct {
  uint64_t h, d;          /* entry key                           */
  uint8_t action;         /* SKV_ACTION_*                        */
  uint8_t owner;          /* OwnerClass                          */
  double entropy_now, entropy_prev;
  uint64_t u_pre;
  uint64_t epoch;
} skv_event;

/* MonitorConfig (monitor.hpp:12-15) of the context's entropy monitor. */
int skv_set_monitor_config(skv_ctx* ctx, double entropy_jump, uint64_t u_pre_max);
/* advance_epoch + epoch_pass + roll.  Events are sorted by (h, d).  *n_events is the total
 * number of events; when it exceeds cap only the first cap are written and the whole list
 * stays retrievable with skv_last_events (nothing is lost: the epoch has been applied). */
int skv_epoch(skv_ctx* ctx, skv_event* events, size_t cap, size_t* n_events, uint64_t* epoch);
/* The events of the last skv_epoch (sorted by (h, d)); *n_events = their total count. */
int skv_last_events(skv_ctx* ctx, skv_event* events, size_t cap, size_t* n_events);
/* One step of the batch pipeline in one call, with one host synchronisation in the common case:
 * skv_admit(batch, out) -> skv_prefetch(prefetch_next) -> skv_commit -> skv_stage(stage_after) ->
 * skv_epoch.  The admit's output copies complete with the step's synchronisation (out's summary is
 * filled then); the epoch pass is queued right behind the commit and aborts itself on the device
 * when the commit failed or needs its ordered replay (it then runs after the replay).  Same
 * results and errors as the separate calls (A.1 with K = 1); prefetch_next / stage_after / out may
 * be NULL.  Eviction, budgets and the replicated layer take the separate calls' path. */
int skv_step(skv_ctx* ctx, const skv_batch* batch, skv_admit_out* out, const skv_batch* prefetch_next,
             const skv_batch* stage_after, uint64_t* new_entries, skv_event* events, size_t cap,
             size_t* n_events, uint64_t* epoch_out);

/* Label landing.  With pending != 0, skv_commit stores new entries
 * as PendingPrivate (visible to their creator only, like the reference's freshly inserted
 * nodes, cache_index.hpp:196-198) instead of the rule-tier labels, and the caller lands
 * the labels later, e.g. when an asynchronous detector finishes. */
int skv_set_label_policy(skv_ctx* ctx, int pending);
/* RadixCacheIndex::resolve_block (cache_index.hpp:321-343) per prompt: the classification
 * block of prompt p is its blocks [first_block[p], n_p) (keys prompt-major from block 0,
 * block_offsets as for skv_set_tiers), landed with labels[p]: Public labels every block of
 * the span without propagation; Private / Restricted label the span's top block and every
 * descendant.  Within one call, Public landings apply first, then Private, then
 * Restricted (so overlapping private landings resolve to the stricter label). */
int skv_resolve_blocks(skv_ctx* ctx, const uint64_t* h, const uint64_t* d, const uint32_t* block_offsets,
                       uint32_t n_prompts, const uint32_t* first_block, const uint8_t* labels);

/* Tier tags of existing entries (demote, cache_index.hpp:362-381): an entry's tier only
 * moves down HBM -> DRAM -> SSD, so it becomes max(current, tag).  Keys are given per
 * prompt, prompt-major from block 0 (the skv_admit_out layout): block_offsets has
 * n_prompts + 1 entries and the tags are per block. */
int skv_set_tiers(skv_ctx* ctx, const uint64_t* h, const uint64_t* d, const uint32_t* block_offsets,
                  uint32_t n_prompts, const uint8_t* tiers);

typedef struct {
  uint64_t h, d, creator;
  uint8_t label, owner, tier;
  uint64_t hit_cur, u_cnt, hit_pre, u_pre; /* AccessStats (access_stats.hpp:18-21) */
} skv_entry;
/* Export all live entries (parity dump; order unspecified). */
int skv_export(skv_ctx* ctx, skv_entry* out, size_t cap, size_t* n);
uint64_t skv_entry_count(skv_ctx* ctx);

/* Eviction (RadixCacheIndex::evict, cache_index.hpp:281-292,697-807; untiered mode).
 * skv_enable_eviction must precede the first admit: it allocates the per-entry access
 * epoch / node id bookkeeping.  skv_evict frees needed_blocks entries, one block each,
 * in the reference's victim order (unpinned HBM leaves, oldest access epoch first, then
 * Public before non-Public, then the smallest node id, repeatedly), leaving tombstones
 * that lookups treat as missing and a later insert of the same key revives as a fresh
 * entry.  With tiered_demotion (RadixCacheIndex::Config::tiered_demotion, lower tiers
 * unbounded) a victim is instead demoted HBM -> DRAM and stays a leaf, so the victims are
 * the smallest-key HBM leaves.  Writes the victims' keys (up to cap) and returns
 * SKV_ERR_CAPACITY, after freeing every candidate, when fewer than needed_blocks could
 * be freed. */
int skv_enable_eviction(skv_ctx* ctx, int tiered_demotion);
/* TierBudget (cache_index.hpp:26-55) in blocks, with the reference's insert-time make_room
 * (cache_index.hpp:183-190, 801-806) -- contract A.9: every prompt's matched path stays
 * pinned from its lookup until the batch's commit ends (ServingSimulator::submit pins,
 * serving_sim.hpp:195-215); the commit inserts the prompts in order, each first evicting unpinned
 * leaves in the reference's victim order until its new blocks fit the HBM budget; a prompt that
 * cannot make room is dropped (nothing inserted, CapacityExhausted in the reference -- listed by
 * skv_last_drops) and the commit continues.  With tiered demotion (skv_enable_eviction(ctx, 1))
 * a victim moves one tier down (HBM -> DRAM -> SSD) and a full lower tier first makes room the
 * same way, freeing from SSD (evict_or_demote, cache_index.hpp:732-766); skv_evict then cascades
 * too.  Needs skv_enable_eviction; call before the first admit.  skv_tier_usage: used / capacity
 * blocks per tier (HBM, DRAM, SSD). */
int skv_set_tier_budget(skv_ctx* ctx, uint64_t hbm_blocks, uint64_t dram_blocks, uint64_t ssd_blocks);
int skv_tier_usage(skv_ctx* ctx, uint64_t* used3, uint64_t* cap3);
/* Prompts (indices into the last committed batch, ascending) whose insert could not make room. */
int skv_last_drops(skv_ctx* ctx, uint32_t* prompts, size_t cap, size_t* n);
int skv_evict(skv_ctx* ctx, uint64_t needed_blocks, uint64_t epoch, uint64_t* n_evicted, uint64_t* victims_h,
              uint64_t* victims_d, size_t cap);
/* An admitted but uncommitted batch is dropped by skv_evict (its lookups and monitor records
 * stand; its commit would attach blocks to entries the eviction may free -- the reference pins
 * a request's path around insert), so a following skv_commit returns SKV_ERR_STATE. */

/* SURVEY A.8 evaluation leak flag of the last admitted batch (serving_sim.hpp:379-392 with
 * block_truth, workload.hpp:137-147): block b of prompt p leaks iff its label is Public and it
 * overlaps a planted span of p that is sensitive on its own (SpanSensitivity::Always).  The
 * caller passes only those spans: prompt p's are [span_off[p], span_off[p+1]) of span_begin /
 * span_end (token offsets within the prompt, end exclusive).  flags (per block, may be NULL). */
int skv_leak_flags(skv_ctx* ctx, const uint32_t* span_off, const uint64_t* span_begin, const uint64_t* span_end,
                   uint8_t* flags, uint64_t* n_leaks);

/* Per-stage device times of the last skv_admit / skv_commit (CUDA events, ms). */
typedef struct {
  float hash_scan_ms, chain_probe_ms, record_ms, admit_total_ms, commit_ms, epoch_ms;
  uint64_t matched_total, accesses, new_blocks, touched_entries;
  uint64_t replayed_entries;  /* entries whose user set crossed 64 in the batch (ordered replay) */
  uint32_t kernels_launched;  /* kernels of the last admit + commit + epoch */
  uint32_t prefetched;        /* 1: the last admit consumed stages 1-2 staged by skv_prefetch */
} skv_stage_times;
int skv_last_times(skv_ctx* ctx, skv_stage_times* out);

/* ------------------------------------------------------------------------------
 * Serving observables of the last skv_admit.  The probe records, per
 * matched block, its tier and whether the requesting user created it; this epilogue turns
 * them into the reference's per-request TTFT and reuse attribution.
 * ------------------------------------------------------------------------------ */
/* CostModel (serving_sim.hpp:25-57) */
typedef struct {
  double t_base_ms, c_prefill_ms;
  double tier_penalty_ms[3]; /* HBM, DRAM, SSD */
  double noise_sigma_ms;
  uint64_t seed;
} skv_cost_model;
void skv_cost_model_default(skv_cost_model* m);
/* CostModel::validate (serving_sim.hpp:35-42) -> SKV_ERR_CONFIG on a bad model. */
int skv_set_cost_model(skv_ctx* ctx, const skv_cost_model* m);
/* Per prompt of the last admitted batch: ttft_ms = CostModel::ttft(L_p, match,
 * request_id) (serving_sim.hpp:50-56), one KV handle of B tokens per matched block;
 * intra/inter_tokens = ServingSimulator::attribute_reuse (serving_sim.hpp:313-324).
 * request_ids may be NULL (= running admission index of the prompt).  Any output may be
 * NULL; on_device applies to request_ids and the outputs.  Valid until the next admit. */
int skv_admit_ttft(skv_ctx* ctx, const uint64_t* request_ids, double* ttft_ms, uint32_t* intra_tokens,
                   uint32_t* inter_tokens, int on_device);

/* ------------------------------------------------------------------------------
 * Per-call entry points of the reference-API facade (include/safekv/): the reference's
 * per-node operations on the device index, entries named by their keys (a facade NodeRef is
 * the key list of one insert's blocks).
 * ------------------------------------------------------------------------------ */
/* RadixCacheIndex::match_prefix (cache_index.hpp:213-237): an admit that records no accesses
 * (the reference's match only stamps access epochs) and leaves nothing to commit. */
int skv_lookup(skv_ctx* ctx, const skv_batch* batch, skv_admit_out* out);
/* RadixCacheIndex::insert (cache_index.hpp:152-205): admit without access records + commit. */
int skv_insert(skv_ctx* ctx, const skv_batch* batch, uint64_t* new_entries);
/* Entries by key (found[i] = 0 for a missing key; found may be NULL). */
int skv_get_entries(skv_ctx* ctx, const uint64_t* h, const uint64_t* d, size_t n, skv_entry* out, uint8_t* found);
/* set_label (cache_index.hpp:312-315, 654-685) on entries given root-first; with propagate a
 * Private / Restricted label also goes to every descendant of the last one (promotion to
 * Public never propagates).  *changed = entries whose label changed. */
int skv_label_entries(skv_ctx* ctx, const uint64_t* h, const uint64_t* d, size_t n, uint8_t label, int propagate,
                      size_t* changed);
/* record_access (cache_index.hpp:385-388, AccessStats::record) of (entry, user) pairs in order. */
int skv_record_accesses(skv_ctx* ctx, const uint64_t* h, const uint64_t* d, const uint64_t* users, size_t n);
/* roll_window (cache_index.hpp:390-393, AccessStats::roll) of the given entries. */
int skv_roll_entries(skv_ctx* ctx, const uint64_t* h, const uint64_t* d, size_t n);
/* EntropyMonitor::check_anomaly (monitor.hpp:56-81) on one entry: *ev gets the event values,
 * *fired = 1 (and the entry and its subtree are relabeled) when the predicate holds. */
int skv_check_anomaly(skv_ctx* ctx, uint64_t h, uint64_t d, uint64_t epoch, skv_event* ev, int* fired);

/* Per-call wrappers (batch of one, still on the device) for the facade:
 * RuleEngine::tier1_scan (detection.hpp:217) and token_seq_digest (core.hpp:68). */
/* rule_mask receives skv_mask_words(ctx) words (one for up to 32 enabled rules). */
int skv_tier1_scan(skv_ctx* ctx, const char* text, size_t len, uint32_t* rule_mask);
/* Tier-1 scan of n independent texts text[offsets[i] : offsets[i+1]] in one launch (the
 * DetectionPipeline drain's RuleEngine::tier1_scan per pending block, detection.hpp:547-552);
 * rule_masks[w * n + i] = word w of the enabled-rule mask of text i, as skv_tier1_scan. */
int skv_tier1_scan_batch(skv_ctx* ctx, const char* text, const uint64_t* offsets, uint32_t n, uint32_t* rule_masks);
int skv_token_seq_digest(skv_ctx* ctx, const uint32_t* tokens, size_t n, uint64_t* digest);

/* ------------------------------------------------------------------------------
 * Replicated layer (multi-GPU; north star: "each GPU holds a replica
 * of the index, and new-entry inserts and entropy counters are merged across GPUs").  Entries
 * at depth < depth (the first `depth` blocks of every prompt: system prompts, shared roots)
 * are replicated on every rank; deeper entries live on the rank skv_route_depth sends their
 * prompts to.  Per batch every rank runs admit -> commit -> skv_replica_export; the caller
 * all-gathers the exports (NCCL over NVLink; the accesses can stay in device memory) and every
 * rank runs skv_replica_apply on the same data: the entries merged to the lowest global prompt
 * id per key (first creator wins), the accesses as the raw concatenation of all ranks' exports,
 * merged on the device (per (entry, user) the lowest first prompt id and the summed count, then
 * replayed per entry in global prompt order).  The replicated entries therefore stay identical
 * everywhere and their AccessStats equal a single engine's, the order-dependent 64-user
 * saturation included.  The Python mirror is paper_2508_08438_b200.ReplicaGroup.  No reference
 * counterpart (the reference is single-process).
 * ------------------------------------------------------------------------------ */
typedef struct {
  uint64_t h, d;     /* entry key                                      */
  uint64_t ph, pd;   /* parent key, (0, 0) for a root                  */
  uint64_t creator;  /* UserId of the creating prompt                  */
  uint64_t gid;      /* global id of the creating prompt               */
  uint8_t label, owner, pad[6];
} skv_rep_entry;     /* 56 B */
typedef struct {
  uint64_t h, d;     /* entry key                                      */
  uint64_t user;     /* UserId                                         */
  uint64_t gid;      /* global id of the user's first accessing prompt */
  uint64_t count;    /* accesses                                       */
} skv_rep_access;    /* 40 B */
/* Before the first admit; not combinable with eviction. */
int skv_set_replicated_depth(skv_ctx* ctx, uint32_t depth);
/* After skv_commit: the replicated-layer entries the commit created (host) and the batch's
 * replicated-layer accesses aggregated per (entry, user) (device memory when accs_on_device).
 * prompt_gids[p] = global id of the last batch's prompt p (host).  When ecap / acap are too
 * small, returns SKV_ERR_CAPACITY with *n_ents / *n_accs set (call again: the export is
 * repeatable until skv_replica_apply). */
int skv_replica_export(skv_ctx* ctx, const uint64_t* prompt_gids, skv_rep_entry* ents, size_t ecap, size_t* n_ents,
                       skv_rep_access* accs, size_t acap, size_t* n_accs, int accs_on_device);
/* Apply every rank's export: ents = the merged entries (host), accs = all ranks' access exports
 * concatenated, unmerged (device memory when accs_on_device).  Ends the batch's sync. */
int skv_replica_apply(skv_ctx* ctx, const skv_rep_entry* ents, size_t n_ents, const skv_rep_access* accs,
                      size_t n_accs, int accs_on_device);

/* ------------------------------------------------------------------------------
 * Multi-GPU request router (host).  Entries at depth < depth (the
 * first `depth` blocks of every prompt) are replicated on every rank; an entry at depth
 * >= depth belongs to the rank of the key h_depth of its depth-`depth` ancestor.  A prompt
 * with more than `depth` full blocks is therefore routed by h_depth (a hash of the key of
 * its block `depth`), so every entry it can probe, record, insert or relabel below the
 * replicated layer lives on its rank; a prompt with at most `depth` blocks touches
 * replicated entries only and goes to prompt_id % world (prompt_ids may be NULL: index p).
 * depth = 0 is pure prefix-forest partitioning (route by the root block).  There is no
 * reference counterpart: the reference is single-process.
 * The synthetic workload generator of the bench and tests (workload/skv_gen.h) is NOT
 * part of this library.
 * ------------------------------------------------------------------------------ */
int skv_route(const uint32_t* tokens, const uint64_t* offsets, uint32_t n_prompts, uint32_t block_tokens,
              const uint64_t* prompt_ids, uint32_t world, uint32_t* rank_out);
int skv_route_depth(const uint32_t* tokens, const uint64_t* offsets, uint32_t n_prompts, uint32_t block_tokens,
                    uint32_t depth, const uint64_t* prompt_ids, uint32_t world, uint32_t* rank_out);

#ifdef __cplusplus
}
#endif
#endif /* SAFEKV_B200_H_ */
